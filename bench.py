#!/usr/bin/env python3
"""Benchmark: points x iterations / s of the TriMe++ hot path (Delaunay from
bounded Voronoi cells + CVD/DistMesh update + treatment) on B200.

Workload (BASELINE.json metric "10^6 pts"): configs[2] = cfg3, the adaptive
annulus, N = 10^6 points, the hybrid schedule 30 DistMesh + 30 CVD
iterations.  One STEP = the whole schedule from the config's initial points
(60 iterations = 6e7 point-iterations); `value` = N * 60 * steps / time.

Timing: W untimed warm-up steps, then K timed steps bracketed by a barrier +
cuda.synchronize on both sides, CUDA events on the library's stream, max over
ranks; L2 flushed (256 MiB write) before every step; SM clocks sampled with
nvidia-smi during the timed region.  `e2e` repeats the measurement through
the public API with pinned HOST buffers: H2D of the step's input points and
D2H of the result (final points + triangle count) inside the timed region.

--impl reference: the CPU oracle (oracle/, plain C, 1 thread) on a bounded
sample of the same workload (one iteration per step, alternating DistMesh and
CVD), printed as a JSON line with "impl": "reference".

N > 1 (torchrun): the same mesh is split into N x-strips (x-quantiles of the
initial points), one per GPU; every iteration exchanges a ghost halo and the
migrating points with the neighbour strips over NCCL and all-reduces the two
DistMesh edge sums -> "scaling": "strong" (total work fixed).
`--strips` runs that path at N = 1 as well (smoke test of the code path).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

WORKLOAD = "cfg3: annulus 0.3<|x|<1, adaptive h=min(0.002+0.3|sdf|,0.02), rho=h^-2, N=1e6, 1024^2 grids, " \
           "hybrid 30 DistMesh + 30 CVD iterations per step"
METRIC = "points*iterations/s (Delaunay + CVD/DistMesh update), 10^6 pts"
UNIT = "pts*it/s"


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_rank{gpu_index}.csv")

    def start(self):
        try:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.close()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            p = [t.strip() for t in line.split(",")]
            if len(p) < 8:
                continue
            try:
                sm.append(float(p[0]))
                smax = float(p[1])
            except ValueError:
                continue
            for k, nm in enumerate(names):
                if p[4 + k].lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def flush_l2(buf):
    buf.add_(1.0)  # 256 MiB read+write > 126 MB L2


# ---------------------------------------------------------------- reference arm
def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import oracle as O
    from inputs import configs
    c = configs.load(3)
    fs = O.FieldSet.from_config(c)
    modes = ["dm", "cvd"]
    x, y, dp = c.x, c.y, None
    times = []
    total = args.warmup + args.steps
    for s in range(total):
        mode = modes[s % 2]
        t0 = time.perf_counter()
        r = O.iteration(fs, x, y, mode, d_prev=dp)
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            times.append(dt)
        x, y, dp = r.x, r.y, r.d_prev
    T = sum(times)
    value = c.n * len(times) / T
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * T / len(times),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "sample": "one oracle iteration per step (alternating DistMesh/CVD) "
                                                    "from the cfg3 initial points"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": f"{len(times)} single-threaded oracle iterations of cfg3 (1e6 points)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline_sample(pairs=2):
    """Oracle (as it stands, 1 thread) on a bounded sample: `pairs` x (one DistMesh
    then one CVD iteration) of cfg3 from its initial points (~10 s)."""
    import oracle as O
    from inputs import configs
    c = configs.load(3)
    fs = O.FieldSet.from_config(c)
    x, y, dp = c.x, c.y, None
    t0 = time.perf_counter()
    for _ in range(pairs):
        r = O.iteration(fs, x, y, "dm", d_prev=dp)
        r = O.iteration(fs, r.x, r.y, "cvd", d_prev=r.d_prev)
        x, y, dp = r.x, r.y, r.d_prev
    dt = time.perf_counter() - t0
    return {"value": 2 * pairs * c.n / dt, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"{pairs} x (1 DistMesh + 1 CVD) oracle iterations of cfg3 (1e6 points), single thread",
            "seconds": dt}


# ---------------------------------------------------------------- our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--strips", action="store_true", help="use the x-strip path even at N=1 (smoke test)")
    ap.add_argument("--n-opt", type=float, default=None, help="override tm_params.n_opt (tuning)")
    ap.add_argument("--cells", default="thread", choices=["thread", "group"],
                    help="cell kernel: one thread per cell (default) or 16-lane groups (A/B)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    import paper_2309_13824_b200 as T
    from inputs import configs

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    c = configs.load(3)
    n = c.n
    schedule = c.schedule  # 30 dm + 30 cvd
    iters = len(schedule)
    dev = torch.device("cuda", local)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    params = T.default_params()
    if args.cells == "group":
        params.flags |= T.TM_F_GROUP_CELLS
    if args.n_opt:
        params.n_opt = args.n_opt
    ctx = T.Context(local, params=params, stream=stream)
    box = c.box
    phi = torch.from_numpy(c.phi).to(dev)
    mu = torch.from_numpy(c.mu).to(dev)
    rho = torch.from_numpy(c.rho).to(dev)
    ctx.tm_set_domain(box, phi, mu, rho, n)
    x0 = torch.from_numpy(c.x).to(dev)
    y0 = torch.from_numpy(c.y).to(dev)
    bufs = T.IterBuffers.alloc(n, ctx.params.adj_stride, device=dev)
    X = [torch.empty(n, dtype=torch.float64, device=dev) for _ in range(2)]
    Y = [torch.empty(n, dtype=torch.float64, device=dev) for _ in range(2)]
    D = [torch.empty(n, dtype=torch.float64, device=dev) for _ in range(2)]
    flush = torch.empty(32 * 1024 * 1024, dtype=torch.float64, device=dev)
    ev_cells = []  # (start, end, mode) around every tm_voronoi_delaunay in the timed region

    def one_step_single(xin, yin, record=False):
        xc, yc, dc = xin, yin, None
        for it, mode in enumerate(schedule):
            xo, yo, do = X[it % 2], Y[it % 2], D[it % 2]
            ctx.tm_grid_bin(xc, yc)
            if record:
                e0 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
            if mode == "cvd":
                ctx.tm_voronoi_delaunay(bufs.tri, bufs.n_tri, None, None, dc, xo, yo, do, bufs.status)
            else:
                ctx.tm_voronoi_delaunay(bufs.tri, bufs.n_tri, bufs.adj, bufs.deg)
            if record:
                e1 = torch.cuda.Event(enable_timing=True)
                e1.record(stream)
                ev_cells.append((e0, e1, mode))
            if mode == "dm":
                ctx.tm_distmesh_sums(bufs.adj, bufs.deg, bufs.sums2)
                ctx.tm_distmesh_step(bufs.adj, bufs.deg, bufs.sums2, None, dc, xo, yo, do, bufs.status)
            xc, yc, dc = xo, yo, do
        return xc, yc

    # N > 1 (or --strips): x-strip decomposition of the same mesh: each rank owns the
    # points of one x-quantile strip; per iteration a ghost halo (W = 2 S_max) goes to both neighbours
    # over NCCL, the DistMesh edge sums are all-reduced, and points that left the strip migrate.
    strip_mode = world > 1 or args.strips
    if strip_mode:
        from paper_2309_13824_b200 import strips as S
        strips = S.Strips.from_quantiles(torch.from_numpy(c.x), world, box[0], box[2])
        st_init = S.split_initial(x0, y0, strips, rank)
        W = S.ghost_width(ctx.c, params.fac_voro_bound, float(c.mu.max()) if c.mu is not None else 1.0)
        comm = S.TorchP2P(rank, world, dev)
        backend = S.GpuStripBackend(ctx, params.adj_stride, keep_tri=False)
        n_own0 = st_init.x.shape[0]

    def one_step_strips(xin, yin, record=False):
        st = S.RankState(rank, xin, yin, st_init.gid, None)
        for mode in schedule:
            st = S.strip_iteration(st, strips, backend, comm.exchange, W, mode, allreduce=comm.allreduce_sum)
        return st.x, st.y

    one_step = one_step_strips if strip_mode else one_step_single
    xs0, ys0 = (st_init.x, st_init.y) if strip_mode else (x0, y0)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    # warm-up
    for _ in range(args.warmup):
        flush_l2(flush)
        one_step(xs0, ys0)
    ctx.tm_sync()
    # timed (device, inputs resident)
    sampler = ClockSampler(local)
    step_ms = []
    barrier()
    sampler.start()
    for _ in range(args.steps):
        flush_l2(flush)
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        one_step(xs0, ys0, record=True)
        s1.record(stream)
        s1.synchronize()
        step_ms.append(s0.elapsed_time(s1))
    barrier()
    clocks = sampler.stop()
    ctx.tm_sync()
    t_local = sum(step_ms) / 1e3
    t = torch.tensor([t_local], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_max = float(t.item())
    value = n * iters * args.steps / t_max  # all ranks together mesh the n points (strips at N > 1)

    # per-launch duration of the dominant kernel (k_cells), CUDA events on the launching stream
    cells_ms = {"dm": [], "cvd": []}
    for e0, e1, mode in ev_cells:
        cells_ms[mode].append(e0.elapsed_time(e1))

    # e2e through the public API with pinned host buffers
    e2e = None
    if not args.no_e2e:
        hx = xs0.cpu().pin_memory()  # this rank's input points (all of them at N=1)
        hy = ys0.cpu().pin_memory()
        n_in = hx.shape[0]
        rx = torch.empty(2 * n_in + 1024, dtype=torch.float64).pin_memory()
        ry = torch.empty(2 * n_in + 1024, dtype=torch.float64).pin_memory()
        rn = torch.empty(1, dtype=torch.int64).pin_memory()
        dx = torch.empty(n_in, dtype=torch.float64, device=dev)
        dy = torch.empty(n_in, dtype=torch.float64, device=dev)
        e2e_ms = []
        barrier()
        for _ in range(args.steps):
            flush_l2(flush)
            s0 = torch.cuda.Event(enable_timing=True)
            s1 = torch.cuda.Event(enable_timing=True)
            s0.record(stream)
            dx.copy_(hx, non_blocking=True)
            dy.copy_(hy, non_blocking=True)
            xf, yf = one_step(dx, dy)
            rx[:xf.shape[0]].copy_(xf, non_blocking=True)
            ry[:yf.shape[0]].copy_(yf, non_blocking=True)
            rn.copy_(bufs.n_tri, non_blocking=True)
            s1.record(stream)
            s1.synchronize()
            e2e_ms.append(s0.elapsed_time(s1))
        barrier()
        te = torch.tensor([sum(e2e_ms) / 1e3], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": n * iters * args.steps / float(te.item()), "unit": UNIT,
               "h2d_bytes_per_step": 2 * 8 * n, "d2h_bytes_per_step": 2 * 8 * n + 8}

    # algorithmic DP instructions of the dominant kernel: work counters from an
    # untimed counting pass over the same schedule (SURVEY §8(d) cost table)
    roof = None
    if rank == 0 and ev_cells:
        roof = roofline(T, c, ctx, cells_ms, params.flags, params.n_opt)

    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cpu = cpu_baseline_sample()
        # binning: k_bin_keys, k_bin_levels, 2 x (k_scan_tiles, k_scan_top, k_scan_add), k_leaf_keys,
        # k_perm_scatter, k_leaf_sort_perm, k_gather_sorted = 12; cells: k_cells_t + the retry pass = 2,
        # + k_output_t in CVD mode; DistMesh: k_dm_sums, k_dm_final, k_dm_step = 3
        launches_per_step = sum(17 if m == "dm" else 15 for m in schedule) + (
            7 * len(schedule) if strip_mode else 0)  # k_halo_pack; k_migrate_count, 3 scan kernels, scatter, unpack
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * t_max / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "n_points": n, "iterations_per_step": iters,
                       "schedule": "30 dm + 30 cvd",
                       "parallelism": f"x-strips{world} (NCCL halo + migration)" if strip_mode else "single",
                       "l2": "flushed before every step (256 MiB write); per-iteration working set ~90 MB"},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches_per_step * args.steps,
            "clocks": clocks,
            "cells_ms_per_launch": {k: (statistics.mean(v) if v else None) for k, v in cells_ms.items()},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")


def dp_peak():
    """fp64 ALU peak (DP thread-instructions/s) = SMs x 64 FP64 lanes x SM clock
    (B200: 148 SMs; profiling guide max clock 1965 MHz, MEASURED_PEAKS.json)."""
    mhz = 1965.0
    try:
        mhz = float(json.load(open(PEAKS)).get("sm_max_mhz", mhz))
    except Exception:
        pass
    meas = os.path.join(ROOT, "profiles", "fp64_peak.json")
    if os.path.exists(meas):
        try:
            m = json.load(open(meas))
            return float(m["dp_inst_per_s"]), "measured DFMA microbenchmark (tools/fp64_peak.cu, profiles/fp64_peak.json)"
        except Exception:
            pass
    return 148 * 64 * mhz * 1e6, f"derived 148 SMs x 64 FP64 lanes x {mhz:.0f} MHz"


def roofline(T, c, ctx, cells_ms, flags=0, n_opt=None):
    """achieved = algorithmic DP instructions per k_cells launch / mean launch time."""
    import torch
    p = T.default_params()
    p.flags |= T.TM_F_COUNT_WORK | flags
    if n_opt:
        p.n_opt = n_opt
    dev = torch.device("cuda", ctx.device)
    cc = T.Context(ctx.device, params=p)
    cc.tm_set_domain(c.box, torch.from_numpy(c.phi).to(dev), torch.from_numpy(c.mu).to(dev),
                     torch.from_numpy(c.rho).to(dev), c.n)
    bufs = T.IterBuffers.alloc(c.n, p.adj_stride, device=dev)
    xs = torch.from_numpy(c.x).to(dev)
    ys = torch.from_numpy(c.y).to(dev)
    xo, yo, do = torch.empty_like(xs), torch.empty_like(xs), torch.empty_like(xs)
    dc = None
    flops = {"dm": [], "cvd": []}
    wsum = {"dm": [0] * 11, "cvd": [0] * 11}
    for mode in c.schedule:
        cc.tm_grid_bin(xs, ys)
        if mode == "cvd":
            cc.tm_voronoi_delaunay(bufs.tri, bufs.n_tri, None, None, dc, xo, yo, do, bufs.status)
        else:
            cc.tm_voronoi_delaunay(bufs.tri, bufs.n_tri, bufs.adj, bufs.deg)
        w = cc.tm_work_counts()
        wsum[mode] = [a + b for a, b in zip(wsum[mode], [w.n_cells, w.n_cert, w.deg, w.verts, w.t_own, w.quad_tris,
                                                          w.ell, w.candidates, w.clips, w.exact_calls, w.retries])]
        # 4 n_cert + 5 deg V + 50 deg + 40 T_own + [6V+15 | 30 Q] + 20 (ELL/force cost is k_dm_step)
        f = 4 * w.n_cert + 5 * w.deg * (w.verts / max(w.n_cells, 1)) + 50 * w.deg + 40 * w.t_own
        if mode == "cvd":
            f += 30 * w.quad_tris + 20 * w.n_cells
        flops[mode].append(f)
        if mode == "dm":
            cc.tm_distmesh_sums(bufs.adj, bufs.deg, bufs.sums2)
            cc.tm_distmesh_step(bufs.adj, bufs.deg, bufs.sums2, None, dc, xo, yo, do, bufs.status)
        xs, ys, dc = xo.clone(), yo.clone(), do.clone()
    cc.tm_sync()
    cc.close()
    peak, how = dp_peak()
    traffic = None  # DRAM bytes per launch of the cell kernel from the committed ncu capture
    try:
        tj = json.load(open(os.path.join(ROOT, "profiles", "kcells_traffic.json")))
        nd = sum(1 for m in c.schedule if m == "dm")
        traffic = (nd * tj["dm_bytes"] + (len(c.schedule) - nd) * tj["cvd_bytes"]) / len(c.schedule)
    except Exception:
        pass
    tot_f = sum(flops["dm"]) + sum(flops["cvd"])
    tot_t = sum(sum(v) for v in cells_ms.values()) / max(1, len(cells_ms["dm"]) + len(cells_ms["cvd"]))
    nl = len(c.schedule)
    per_launch_f = tot_f / nl
    achieved = per_launch_f / (tot_t / 1e3)
    return {"bound": "alu", "achieved": achieved / 1e12, "peak": peak / 1e12, "unit": "T DP-inst/s",
            "frac": achieved / peak, "traffic": traffic, "traffic_unit": "bytes/launch (ncu dram read+write)",
            "kernel": "k_cells_t (S2+S3+S4a+S5 fused)",
            "algorithmic_dp_inst_per_launch": per_launch_f, "peak_source": how,
            "dp_inst_per_launch_by_mode": {k: (statistics.mean(v) if v else None) for k, v in flops.items()},
            "work_per_cell_by_mode": {m: {k: round(v / max(1, wsum[m][0]), 3) for k, v in zip(
                ["n_cells", "n_cert", "deg", "verts", "t_own", "quad_tris", "ell", "candidates", "clips",
                 "exact_calls", "retries"], wsum[m])} for m in wsum}}


if __name__ == "__main__":
    main()
