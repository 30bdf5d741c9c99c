"""Summarise a cellbench A/B log: mean DistMesh / CVD cell-launch ms per (library, config).
python tools/ab_summary.py gpurun_out/<tag>_variants.jsonl"""
import json
import sys
from collections import defaultdict

agg = defaultdict(list)
for line in open(sys.argv[1]):
    if line.startswith("{"):
        d = json.loads(line)
        agg[(d["config"], d["lib"])].append((d["dm_ms"], d["cvd_ms"]))
for (cfg, lib), v in sorted(agg.items()):
    dm = sum(a for a, _ in v) / len(v)
    cvd = sum(b for _, b in v) / len(v)
    print(f"{cfg:8s} {lib:28s} dm {dm:7.3f} ms  cvd {cvd:7.3f} ms  (n={len(v)})")
