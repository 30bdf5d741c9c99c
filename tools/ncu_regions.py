"""Instruction / stall-sample shares of an ncu report by source region (needs -lineinfo):
python tools/ncu_regions.py rep.ncu-rep file.cu:a-b=name ...  (other lines grouped by file)"""
import collections, csv, io, subprocess, sys
rep = sys.argv[1]
regions = []
for spec in sys.argv[2:]:
    loc, name = spec.split("=")
    f, rng = loc.split(":")
    a, b = map(int, rng.split("-"))
    regions.append((f, a, b, name))
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
agg = collections.defaultdict(lambda: [0, 0])
path = ""
for r in rows:
    if r and r[0] == "File Path":
        path = r[1].split("/")[-1]; continue
    if not r or r[0] in ("Function Name", "Line No") or len(r) < 10 or r[2] != "-":
        continue
    try:
        line, smp, ins = int(r[0]), int(r[4]), int(r[7])
    except ValueError:
        continue
    key = path
    for f, a, b, name in regions:
        if f == path and a <= line <= b:
            key = name
            break
    agg[key][0] += ins
    agg[key][1] += smp
ti = sum(v[0] for v in agg.values()); ts = sum(v[1] for v in agg.values())
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{k:28s} inst {100*v[0]/ti:6.2f}%   stall samples {100*v[1]/ts:6.2f}%")
