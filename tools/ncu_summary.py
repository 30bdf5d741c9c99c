"""Summarise ncu outputs for profiles/ (run here, no GPU needed).

  python tools/ncu_summary.py launches gpurun_out/launches.csv   > profiles/<tag>_launches.txt
  python tools/ncu_summary.py full gpurun_out/prof.ncu-rep        > profiles/<tag>_ncu.txt

`launches`: per-kernel launch count, total / average device time and share of
the step (ncu --metrics gpu__time_duration.sum: cold-cache, serialised).
`full`: the counters SURVEY §8(d) asks for, per captured launch.
"""
import collections
import csv
import io
import re
import subprocess
import sys


def short(name):
    name = re.sub(r"\((tmg::|const |double|int|float|long|unsigned|__nv_).*", "", name)
    return name.replace("(anonymous namespace)::", "").replace("<unnamed>::", "").replace("void ", "")


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, mi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= mi:
            continue
        v = float(r[mi].replace(",", ""))
        v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "s": 1e6}[r[ui]]
        a = agg[short(r[ki])]
        a[0] += 1
        a[1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"# {path}: {sum(v[0] for v in agg.values())} launches, {tot / 1e3:.2f} ms total (cold-cache, serialised)")
    print(f"{'kernel':44s} {'n':>6s} {'total ms':>10s} {'share':>7s} {'avg us':>10s}")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k[:44]:44s} {v[0]:6d} {v[1] / 1e3:10.2f} {100 * v[1] / tot:6.1f}% {v[1] / v[0]:10.1f}")


WANT = [
    "gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum",
    "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
    "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum.per_cycle_elapsed",
    "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum.per_cycle_elapsed",
    "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum.per_cycle_elapsed", "sm__cycles_elapsed.avg",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio",
]


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units, data = rows[0], rows[1], rows[2:]
    print(f"# {path} (ncu --set full --clock-control none)")
    for d in data:
        print(f"## {short(d[h.index('Kernel Name')])}")
        for w in WANT:
            for i, x in enumerate(h):
                if x == w:
                    print(f"  {w:70s} {d[i]:>16s} {units[i]}")
        try:
            rate = sum(float(d[h.index(f"smsp__sass_thread_inst_executed_op_{o}_pred_on.sum.per_cycle_elapsed")])
                       for o in ("dfma", "dadd", "dmul"))
            cyc = float(d[h.index("sm__cycles_elapsed.avg")].replace(",", ""))
            print(f"  {'executed DP thread-instructions per launch (dfma+dadd+dmul)':70s} {rate * cyc:16.4e}")
            print(f"  {'  = per cycle, of the 148 x 64 = 9472 peak':70s} {rate:16.1f} ({100 * rate / 9472:.1f} %)")
        except (ValueError, IndexError):
            pass


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
