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
nvidia-smi during the timed region.  Every iteration is bracketed by events too:
the per-iteration time by mode is T_meas of SURVEY §8(d)'s per-iteration
roofline (T_roof from the kernel's own work counters, an untimed counting pass).

`e2e` repeats the measurement through the public API with pinned HOST buffers:
H2D of the step's input points, then D2H of the result -- the final points, the
triangle count and the final triangle list -- inside the timed region.

cfg5 leg (`cfg5`): the uniform scaling workload, 1.6e7 and
6.4e7 jittered points, 20 CVD iterations, ms/iteration and pts*it/s, so the
driver's 1..8-GPU runs carry the north_star scaling config as well.

cpu_baseline: the oracle (oracle/, plain C, as it stands) in a subprocess pinned
to one core (`taskset -c 0`), the first 3 iterations of each phase of the cfg3
schedule (3 DistMesh from the initial points, 3 CVD from the GPU's state after
the 30 DistMesh iterations), ~20 s.

--impl reference: the oracle on a bounded sample of the same workload (one
iteration per step, alternating DistMesh and CVD), pinned to one core, printed
as a JSON line with "impl": "reference".

N > 1 (torchrun): the same mesh is split into N x-strips (x-quantiles of the
initial points), one per GPU; every iteration exchanges a ghost halo and the
migrating points with the neighbour strips over NCCL and all-reduces the two
DistMesh edge sums -> "scaling": "strong" (total work fixed).
`--strips` runs that path at N = 1 as well.
"""
from __future__ import annotations

import argparse
import json
import os
import shutil
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

WORKLOAD = "cfg3: annulus 0.3<|x|<1, adaptive h=min(0.002+0.3|sdf|,0.02), rho=h^-2, N=1e6, 1024^2 grids, " \
           "hybrid 30 DistMesh + 30 CVD iterations per step"
METRIC = "points*iterations/s (Delaunay + CVD/DistMesh update), 10^6 pts"
UNIT = "pts*it/s"
PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
# SURVEY §8(d) compulsory HBM bytes per point and iteration, by stage
B_S1, B_FUSED, B_DM = 56.0, 69.0, 64.0


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def host_info():
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return model, os.cpu_count()


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


# ---------------------------------------------------------------- oracle timing (CPU)
def _pin_cmd():
    return ["taskset", "-c", "0"] if shutil.which("taskset") else []


def cpu_worker(path):
    """Child process: oracle iterations listed in the npz (pinned by the parent to core 0)."""
    if not _pin_cmd() and hasattr(os, "sched_setaffinity"):
        os.sched_setaffinity(0, {0})
    import oracle as O
    from inputs import configs
    z = np.load(path)
    c = configs.load(int(z["cfg"]))
    fs = O.FieldSet.from_config(c)
    out = []
    for ph in ("dm", "cvd"):
        x, y = z[f"{ph}_x"], z[f"{ph}_y"]
        dp = z[f"{ph}_dp"] if z[f"{ph}_has_dp"] else None
        for _ in range(int(z[f"{ph}_iters"])):
            t0 = time.perf_counter()
            r = O.iteration(fs, x, y, ph, d_prev=dp)
            out.append({"mode": ph, "s": time.perf_counter() - t0, "n": c.n})
            x, y, dp = r.x, r.y, r.d_prev
    print(json.dumps(out), flush=True)


def run_oracle_pinned(states: dict, cfg: int = 3):
    """Times the oracle in a child process on core 0; states: {mode: (x, y, d_prev|None, iters)}."""
    with tempfile.TemporaryDirectory() as td:
        f = os.path.join(td, "states.npz")
        kw = {"cfg": cfg}
        for ph in ("dm", "cvd"):
            x, y, dp, it = states.get(ph, (np.zeros(1), np.zeros(1), None, 0))
            kw.update({f"{ph}_x": x, f"{ph}_y": y, f"{ph}_dp": dp if dp is not None else np.zeros(1),
                       f"{ph}_has_dp": dp is not None, f"{ph}_iters": it})
        np.savez(f, **kw)
        cmd = _pin_cmd() + [sys.executable, os.path.abspath(__file__), "--cpu-worker", f]
        r = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT)
        if r.returncode != 0:
            raise RuntimeError(f"oracle worker failed: {r.stderr[-2000:]}")
        return json.loads(r.stdout.strip().splitlines()[-1])


def cpu_desc(sample):
    model, ncpu = host_info()
    pin = "taskset -c 0" if _pin_cmd() else "sched_setaffinity({0})"
    return {"cores": 1, "cores_available": ncpu, "cpu_model": model, "pinning": pin,
            "threads_note": f"1 of {ncpu} cores ({model}), single-threaded plain C oracle", "sample": sample}


# ---------------------------------------------------------------- reference arm
def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from inputs import configs
    c = configs.load(3)
    total = args.warmup + args.steps
    modes = ["dm", "cvd"]
    # one oracle iteration per step, alternating phases, chained from the config's points
    states = {"dm": (c.x, c.y, None, (total + 1) // 2), "cvd": (c.x, c.y, None, total // 2)}
    rec = run_oracle_pinned(states)
    # interleave in step order dm, cvd, dm, ... and drop the warm-up ones
    by = {m: [r for r in rec if r["mode"] == m] for m in modes}
    seq = [by[modes[s % 2]][s // 2] for s in range(total)]
    times = [r["s"] for r in seq[args.warmup:]]
    T = sum(times)
    value = c.n * len(times) / T
    d = cpu_desc(f"{len(times)} timed oracle iterations of cfg3 (1e6 points), one per step, alternating "
                 f"DistMesh/CVD from the config's points (after {args.warmup} warm-up ones)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * T / len(times),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "sample": "one oracle iteration per step (alternating DistMesh/CVD) "
                                                    "from the cfg3 initial points"},
        "cpu_baseline": dict(value=value, unit=UNIT, kind="oracle", **d),
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- roofline
def dp_peak():
    """fp64 ALU peak (DP thread-instructions/s): the measured DFMA microbenchmark
    (tools/fp64_peak.cu, profiles/fp64_peak.json), else 148 SMs x 64 lanes x clock."""
    meas = os.path.join(ROOT, "profiles", "fp64_peak.json")
    if os.path.exists(meas):
        try:
            m = json.load(open(meas))
            return float(m["dp_inst_per_s"]), "measured DFMA microbenchmark (tools/fp64_peak.cu, profiles/fp64_peak.json)"
        except Exception:
            pass
    mhz = 1965.0
    try:
        mhz = float(json.load(open(PEAKS)).get("sm_max_mhz", mhz))
    except Exception:
        pass
    return 148 * 64 * mhz * 1e6, f"derived 148 SMs x 64 FP64 lanes x {mhz:.0f} MHz"


def hbm_peak():
    try:
        return float(json.load(open(PEAKS))["hbm_gbs"]) * 1e9, "MEASURED_PEAKS.json hbm_gbs (copy)"
    except Exception:
        return 6.56e12, "SURVEY §8(d) 6560 GB/s"


def f_alg_cells(w, mode):
    """SURVEY §8(d) DP instructions of the fused cell kernel, summed over cells:
    4 n_cert + 5 deg V + 50 deg + 40 T_own + [6V+15 | 30 Q] + 20 (CVD update + projection test)."""
    n = max(w.n_cells, 1)
    f = 4 * w.n_cert + 5 * w.deg * (w.verts / n) + 50 * w.deg + 40 * w.t_own
    if mode == "cvd":
        f += 30 * w.quad_tris + 20 * w.n_cells  # quad_tris = V for uniform rho (the fan), Q otherwise
    return f


def count_work(T, c, ctx_device, schedule, dev):
    """Untimed TM_F_COUNT_WORK pass over the schedule (its own context): per iteration the
    oracle-pinned work counters of every cell (n_cert, deg, V, T_own, Q, E)."""
    import torch
    p = T.default_params()
    p.flags |= T.TM_F_COUNT_WORK
    cc = T.Context(ctx_device, params=p)
    to = lambda a: None if a is None else torch.from_numpy(a).to(dev)
    cc.tm_set_domain(c.box, to(c.phi), to(c.mu), to(c.rho), c.n)
    bufs = T.IterBuffers.alloc(c.n, p.adj_stride, device=dev)
    xs, ys = to(c.x), to(c.y)
    xo, yo, do = torch.empty_like(xs), torch.empty_like(xs), torch.empty_like(xs)
    dc = None
    per = []
    for mode in schedule:
        cc.tm_grid_bin(xs, ys)
        if mode == "cvd":
            cc.tm_voronoi_delaunay(bufs.tri, bufs.n_tri, None, None, dc, xo, yo, do, bufs.status)
        else:
            cc.tm_voronoi_delaunay(bufs.tri, bufs.n_tri, bufs.adj, bufs.deg)
        w = cc.tm_work_counts()
        per.append((mode, w))
        if mode == "dm":
            cc.tm_distmesh_sums(bufs.adj, bufs.deg, bufs.sums2)
            cc.tm_distmesh_step(bufs.adj, bufs.deg, bufs.sums2, None, dc, xo, yo, do, bufs.status)
        xs, ys, dc = xo.clone(), yo.clone(), do.clone()
    cc.tm_sync()
    cc.close()
    return per


def iteration_roof(mode, w, n, P, BW):
    """T_roof of one iteration: sum over stages of max(bytes/BW, DP/P_DP)."""
    fc = f_alg_cells(w, mode)
    t = n * B_S1 / BW + max(n * B_FUSED / BW, fc / P)
    if mode == "dm":
        t += max(n * B_DM / BW, 45.0 * w.ell / P)
    return t, fc


def roofline(per, cells_ms, it_ms):
    """Dominant kernel (k_cells_t, the fused S2-S5 launch): algorithmic DP instructions per
    launch / mean launch time (CUDA events on the launching stream).  Plus the per-iteration
    T_roof / T_meas of SURVEY §8(d) by iteration type."""
    P, how = dp_peak()
    BW, bw_how = hbm_peak()
    n = per[0][1].n_cells
    by = {"dm": [], "cvd": []}
    for mode, w in per:
        by[mode].append(iteration_roof(mode, w, n, P, BW))
    tot_f = sum(f for m in by for _, f in by[m])
    nl = sum(len(v) for v in by.values())
    tot_t = sum(sum(v) for v in cells_ms.values()) / max(1, sum(len(v) for v in cells_ms.values()))
    achieved = (tot_f / nl) / (tot_t / 1e3)
    traffic = None  # DRAM bytes per launch of the cell kernel from the committed ncu capture
    try:
        tj = json.load(open(os.path.join(ROOT, "profiles", "kcells_traffic.json")))
        nd = len(by["dm"])
        traffic = (nd * tj["dm_bytes"] + len(by["cvd"]) * tj["cvd_bytes"]) / nl
    except Exception:
        pass
    per_it = {}
    for m in ("dm", "cvd"):
        if not by[m] or not it_ms[m]:
            continue
        troof = statistics.mean(t for t, _ in by[m])
        tmeas = statistics.mean(it_ms[m]) / 1e3
        per_it[m] = {"T_roof_us": troof * 1e6, "T_meas_us": tmeas * 1e6, "frac": troof / tmeas,
                     "alg_dp_inst_cells": statistics.mean(f for _, f in by[m]),
                     "cells_ms": statistics.mean(cells_ms[m]) if cells_ms[m] else None}
    wsum = {m: [0] * 12 for m in ("dm", "cvd")}
    for mode, w in per:
        wsum[mode] = [a + b for a, b in zip(wsum[mode], [getattr(w, k) for k, _ in w._fields_])]
    names = [k for k, _ in per[0][1]._fields_]
    sched_roof = sum(t for m in by for t, _ in by[m])
    sched_meas = sum(sum(v) for v in it_ms.values()) / 1e3 / max(1, sum(len(v) for v in it_ms.values())) * nl
    return {"bound": "alu", "achieved": achieved / 1e12, "peak": P / 1e12, "unit": "T DP-inst/s",
            "frac": achieved / P, "traffic": traffic, "traffic_unit": "bytes/launch (ncu dram read+write)",
            "kernel": "k_cells_t (S2+S3 cells/Delaunay, S4a/S5 in k_output_t for CVD)",
            "algorithmic_dp_inst_per_launch": tot_f / nl, "peak_source": how, "hbm_peak_source": bw_how,
            "per_iteration": per_it,
            "schedule_T_roof_over_T_meas": sched_roof / sched_meas if sched_meas else None,
            "work_per_cell_by_mode": {m: {k: round(v / max(1, wsum[m][0]), 3) for k, v in zip(names, wsum[m])}
                                      for m in wsum if wsum[m][0]}}


# ---------------------------------------------------------------- the paper's E1 (context)
def run_paper_e1(T, dev, n=1_000_000):
    """The paper's uniform-square experiment end to end: Floyd-Steinberg initial points
    (init all), the paper's validity tests and controller, CVD and hybrid meshing to termination
    (NEXT-2..4).  Time per triangulation = wall time of the meshing loop (its per-iteration
    controller syncs included) / triangulations: the paper's metric; context for its
    28-thread 0.221 s (CVD) and 0.251 s (hybrid) per triangulation."""
    import time

    import torch
    from inputs import configs
    box = (0.0, 0.0, 1.0, 1.0)
    phi = torch.from_numpy(configs.box_phi(box, 1024)).to(dev)
    nxg, nyg = T.geometry_grid_dims(n, box)
    out = {"workload": "uniform unit square, N = 1e6, init all (fac_init = 1), validity Tests 1-3, "
                       "meshing to termination (P:705-745)"}
    for method in ("cvd", "hybrid"):
        ctx = T.Context(0, params=T.default_params(validity=1))
        ctx.tm_set_domain(box, phi, None, None, n)
        x, y, _, _ = T.initial_points(ctx, n, nxg, nyg, seed=3)
        ctx.tm_set_domain(box, phi, None, None, x.shape[0])
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = T.mesh(ctx, x, y, n_total=n, method=method, max_iterations=400)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        out[method] = {"triangulations": res.iterations, "seconds": dt, "s_per_triangulation": dt / res.iterations,
                       "end": res.history[-1]["action"], "n_tri": int(res.tri.shape[0]),
                       "half_mean_alpha": res.history[-1]["half_alpha"],
                       "paper_28_threads_s_per_triangulation": {"cvd": 0.220976, "hybrid": 0.250808}[method],
                       "paper_triangulations": {"cvd": 52, "hybrid": 57}[method]}
        ctx.close()
    return out


# ---------------------------------------------------------------- cfg5 leg
def run_cfg5(T, dev, stream, n, iters=20, count=True):
    """North-star scaling workload at N=1: jittered uniform square, n points, `iters` CVD
    iterations; one untimed pass, then one timed pass (events per iteration)."""
    import torch
    from inputs import configs
    c = configs.config5(n=n, iters=iters)
    ctx = T.Context(dev.index or 0, stream=stream)
    ctx.tm_set_domain(c.box, torch.from_numpy(c.phi).to(dev), None, None, c.n)
    x0, y0 = torch.from_numpy(c.x).to(dev), torch.from_numpy(c.y).to(dev)
    del c
    bufs = T.IterBuffers.alloc(n, 16, device=dev)
    X = [torch.empty(n, dtype=torch.float64, device=dev) for _ in range(2)]
    Y = [torch.empty_like(X[0]) for _ in range(2)]
    D = [torch.empty_like(X[0]) for _ in range(2)]

    def one(ev=None):
        xc, yc, dc = x0, y0, None
        for it in range(iters):
            if ev is not None:
                ev[it].record(stream)
            T.iterate(ctx, xc, yc, dc, "cvd", bufs, X[it % 2], Y[it % 2], D[it % 2])
            xc, yc, dc = X[it % 2], Y[it % 2], D[it % 2]
        if ev is not None:
            ev[iters].record(stream)
        return xc, yc, dc
    one()
    ctx.tm_sync()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(iters + 1)]
    torch.cuda.synchronize(dev)
    xl, yl, dl = one(ev)
    ev[-1].synchronize()
    its = [ev[k].elapsed_time(ev[k + 1]) for k in range(iters)]
    ctx.tm_sync()
    tot = sum(its) / 1e3
    out = {"n_points": n, "iterations": iters, "ms_per_iteration": statistics.mean(its),
           "value": n * iters / tot, "unit": UNIT}
    if count:
        p = T.default_params()
        p.flags |= T.TM_F_COUNT_WORK
        cc = T.Context(dev.index or 0, stream=stream, params=p)
        phi = torch.from_numpy(configs.box_phi((0.0, 0.0, 1.0, 1.0), 1024)).to(dev)
        cc.tm_set_domain((0.0, 0.0, 1.0, 1.0), phi, None, None, n)
        # warm lists on the last state, then the counted iteration on it
        for _ in range(2):
            cc.tm_grid_bin(xl, yl)
            cc.tm_voronoi_delaunay(bufs.tri, bufs.n_tri, None, None, dl, X[0], Y[0], D[0], bufs.status)
        w = cc.tm_work_counts()
        P, _ = dp_peak()
        BW, _ = hbm_peak()
        troof, fc = iteration_roof("cvd", w, n, P, BW)
        out["T_roof_us"] = troof * 1e6
        out["frac_per_iteration"] = troof / (its[-1] / 1e3)
        out["note"] = "T_roof of the last iteration's state vs its measured time (per GPU)"
        cc.close()
    ctx.close()
    return out


def run_cfg5_strips(T, dev, stream, n, rank, world, iters=20):
    """The north-star scaling workload on `world` ranks: cfg5's points split
    into equal-width x-strips (uniform density), each rank meshing its strip with the ghost-point
    halo and migration exchanged over NCCL every iteration; one untimed pass, then one timed pass
    between barriers; the time is the max over ranks (value = all ranks' points x iterations / t)."""
    import torch
    import torch.distributed as dist
    from inputs import configs
    from paper_2309_13824_b200 import strips as S
    c = configs.config5(n=n, iters=iters)
    params = T.default_params()
    ctx = T.Context(dev.index or 0, stream=stream, params=params)
    ctx.tm_set_domain(c.box, torch.from_numpy(c.phi).to(dev), None, None, c.n)
    strips = S.Strips(c.box[0], c.box[2], world)
    W = S.ghost_width(ctx.c, params.fac_voro_bound, 1.0)
    x0, y0 = torch.from_numpy(c.x).to(dev), torch.from_numpy(c.y).to(dev)
    del c
    cap_own, cap_msg = S.capacities(n, world, int(n * W) + 1)
    St = S.split_initial(x0, y0, strips, rank, cap_own, cap_msg)
    del x0, y0
    xo_, yo_, go_, _ = St.owned()
    x_own, y_own, g_own = xo_.clone(), yo_.clone(), go_.clone()
    counts0 = St.counts.clone()
    comm = S.TorchP2P(rank, world, dev)
    backend = S.GpuStripBackend(ctx, params.adj_stride)

    def one():
        St.reset(x_own, y_own, g_own, counts0)
        for _ in range(iters):
            S.strip_step(St, strips, backend, comm, W, "cvd")
    one()
    ctx.tm_sync()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    one()
    e1.record(stream)
    e1.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / 1e3], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ctx.tm_sync()
    tmax = float(t.item())
    ctx.close()
    return {"n_points": n, "iterations": iters, "ms_per_iteration": 1e3 * tmax / iters, "value": n * iters / tmax,
            "unit": UNIT, "ranks": world, "strips": "equal-width x-strips, NCCL halo + migration every iteration",
            "per_gpu_points": n // world}


# ---------------------------------------------------------------- our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cfg5", action="store_true")
    ap.add_argument("--no-paper-e1", action="store_true")
    ap.add_argument("--no-count", action="store_true",
                    help="skip the untimed work-counting pass of the roofline (ncu launch lists of the step alone)")
    ap.add_argument("--cfg5-sizes", default="16000000,64000000")
    ap.add_argument("--strips", action="store_true", help="use the x-strip path even at N=1")
    ap.add_argument("--flags", type=int, default=0, help="extra tm_params.flags (A/B)")
    ap.add_argument("--no-graph", action="store_true", help="issue every call eagerly (no CUDA Graph replay)")
    ap.add_argument("--cpu-worker", default=None, help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.cpu_worker:
        return cpu_worker(args.cpu_worker)
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
    params.flags |= args.flags
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
    ev_iter = []   # (start, end, mode) around every whole iteration in the timed region
    saved = {}

    def one_step_single(xin, yin, record=False, save=False):
        xc, yc, dc = xin, yin, None
        for it, mode in enumerate(schedule):
            xo, yo, do = X[it % 2], Y[it % 2], D[it % 2]
            if record:
                ei = torch.cuda.Event(enable_timing=True)
                ei.record(stream)
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
            if record:
                ej = torch.cuda.Event(enable_timing=True)
                ej.record(stream)
                ev_iter.append((ei, ej, mode))
            xc, yc, dc = xo, yo, do
            if save and it + 1 < len(schedule) and schedule[it + 1] != mode:  # phase change: keep the state
                saved["cvd"] = (xc.cpu().numpy(), yc.cpu().numpy(), dc.cpu().numpy())
        return xc, yc

    # N > 1 (or --strips): x-strip decomposition of the same mesh, the sync-free
    # protocol of paper_2309_13824_b200.strips (fixed-size messages, device counts)
    strip_mode = world > 1 or args.strips
    if strip_mode:
        from paper_2309_13824_b200 import strips as S
        strips = S.Strips.from_quantiles(torch.from_numpy(c.x), world, box[0], box[2])
        W = S.ghost_width(ctx.c, params.fac_voro_bound, float(c.mu.max()) if c.mu is not None else 1.0)
        # capacities: the owned share with slack; the messages sized from the initial halo
        # (a one-off measurement before timing: 4x the larger side, at most the owned capacity)
        cap_own, _ = S.capacities(n, world, 0)
        S0 = S.split_initial(x0, y0, strips, rank, cap_own, cap_own)
        lo_, hi_ = strips.bounds(rank)
        S.GpuStripBackend(ctx, params.adj_stride).halo_pack(S0, lo_, hi_, W)
        ghosts0 = max(S0.h_send[0].count(), S0.h_send[1].count())
        if world > 1:  # messages are fixed-size: every rank must size them alike (send/recv counts match)
            g_all = torch.tensor([ghosts0], dtype=torch.int64, device=dev)
            dist.all_reduce(g_all, op=dist.ReduceOp.MAX)
            ghosts0 = int(g_all.item())
        cap_msg = min(cap_own, 4 * ghosts0 + 4096)
        S0 = S.split_initial(x0, y0, strips, rank, cap_own, cap_msg)
        xo_, yo_, go_, _ = S0.owned()
        x_own, y_own, g_own = xo_.clone(), yo_.clone(), go_.clone()
        counts0 = S0.counts.clone()
        comm = S.TorchP2P(rank, world, dev)
        backend = S.GpuStripBackend(ctx, params.adj_stride)

    def one_step_strips(xin, yin, record=False, save=False):
        S0.reset(xin, yin, g_own, counts0)
        for mode in schedule:
            S.strip_step(S0, strips, backend, comm, W, mode)
        return S0.X, S0.Y  # owned points at [0, n_owned) (count on the device)

    one_step = one_step_strips if strip_mode else one_step_single
    xs0, ys0 = (x_own, y_own) if strip_mode else (x0, y0)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    # warm-up (the first one keeps the state at the DistMesh -> CVD switch for the CPU sample)
    for w_ in range(args.warmup):
        flush_l2(flush)
        one_step(xs0, ys0, save=(w_ == 0 and not strip_mode))
    ctx.tm_sync()
    # single path: the whole step (60 iterations, ~1000 launches) captured once as a CUDA Graph
    # and replayed (the inputs xs0/ys0 are the graph's input buffers; e2e copies into them)
    graph = None
    use_graph = not strip_mode and not args.no_graph
    if use_graph:
        graph = ctx.capture(lambda: one_step(xs0, ys0))
        graph.launch()  # one untimed replay
        ctx.tm_sync()

    def run_step(record=False):
        if graph is not None and not record:
            graph.launch()
            return X[(iters - 1) % 2], Y[(iters - 1) % 2]
        return one_step(xs0, ys0, record=record)
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
        run_step(record=not use_graph)
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

    if use_graph:  # per-iteration breakdown (T_meas by mode): one more step, eager, with events
        flush_l2(flush)
        one_step(xs0, ys0, record=True)
        ctx.tm_sync()
    cells_ms = {"dm": [], "cvd": []}
    for e0, e1, mode in ev_cells:
        cells_ms[mode].append(e0.elapsed_time(e1))
    it_ms = {"dm": [], "cvd": []}
    for e0, e1, mode in ev_iter:
        it_ms[mode].append(e0.elapsed_time(e1))

    # e2e through the public API with pinned host buffers: points in; points, triangle
    # count and triangle list out
    e2e = None
    if not args.no_e2e:
        hx = xs0.cpu().pin_memory()  # this rank's input points (all of them at N=1)
        hy = ys0.cpu().pin_memory()
        n_in = hx.shape[0]
        rx = torch.empty(2 * n_in + 1024, dtype=torch.float64).pin_memory()
        ry = torch.empty(2 * n_in + 1024, dtype=torch.float64).pin_memory()
        rn = torch.empty(1, dtype=torch.int64).pin_memory()
        rt = torch.empty(((backend.bufs if strip_mode else bufs).tri.shape[0], 3), dtype=torch.int32).pin_memory()
        rc = torch.empty(2, dtype=torch.int64).pin_memory()
        dx, dy = xs0, ys0  # the step's input buffers (the graph reads them)
        e2e_ms, d2h = [], []
        barrier()
        for _ in range(args.steps):
            flush_l2(flush)
            s0 = torch.cuda.Event(enable_timing=True)
            s1 = torch.cuda.Event(enable_timing=True)
            s0.record(stream)
            dx.copy_(hx, non_blocking=True)
            dy.copy_(hy, non_blocking=True)
            xf, yf = run_step()
            tb = backend.bufs if strip_mode else bufs
            rn.copy_(tb.n_tri, non_blocking=True)
            if strip_mode:
                rc.copy_(S0.counts, non_blocking=True)
            stream.synchronize()  # the caller needs the counts to size the copies
            npt = int(rc[0].item()) if strip_mode else xf.shape[0]
            nt = int(rn.item())
            rx[:npt].copy_(xf[:npt], non_blocking=True)
            ry[:npt].copy_(yf[:npt], non_blocking=True)
            if nt:
                rt[:nt].copy_(tb.tri[:nt], non_blocking=True)
            s1.record(stream)
            s1.synchronize()
            e2e_ms.append(s0.elapsed_time(s1))
            d2h.append(2 * 8 * npt + 8 + 12 * nt + (16 if strip_mode else 0))
        barrier()
        te = torch.tensor([sum(e2e_ms) / 1e3], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": n * iters * args.steps / float(te.item()), "unit": UNIT,
               "h2d_bytes_per_step": 2 * 8 * n_in, "d2h_bytes_per_step": int(statistics.mean(d2h)),
               "d2h": "final points (x, y), triangle count, final triangle list (int32 x3)"}

    roof = None
    if rank == 0 and ev_cells and not args.no_count:
        per = count_work(T, c, local, schedule, dev)
        roof = roofline(per, cells_ms, it_ms)

    cfg5 = None
    if not args.no_cfg5:
        cfg5 = {}
        for nn in [int(v) for v in args.cfg5_sizes.split(",") if v]:
            torch.cuda.empty_cache()
            cfg5[str(nn)] = (run_cfg5_strips(T, dev, stream, nn, rank, world) if strip_mode
                             else run_cfg5(T, dev, stream, nn))
        cfg5["workload"] = "cfg5: jittered uniform unit square, 20 CVD iterations per step (SURVEY §8(d) cfg5)"

    paper_e1 = None
    if not args.no_paper_e1 and world == 1 and not strip_mode:
        paper_e1 = run_paper_e1(T, dev)

    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline and "cvd" in saved:
            states = {"dm": (c.x, c.y, None, 3), "cvd": (*saved["cvd"], 3)}
            rec = run_oracle_pinned(states)
            tc = sum(r["s"] for r in rec)
            cpu = dict(value=len(rec) * n / tc, unit=UNIT, kind="oracle", seconds=tc,
                       per_iteration_s={m: [round(r["s"], 3) for r in rec if r["mode"] == m] for m in ("dm", "cvd")},
                       **cpu_desc("the first 3 iterations of each phase of the cfg3 schedule: 3 DistMesh from the "
                                  "config's points and 3 CVD from the GPU state after the 30 DistMesh iterations"))
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
                       "launch": "CUDA Graph replay of the whole step" if use_graph else "eager calls",
                       "schedule": "30 dm + 30 cvd",
                       "parallelism": f"x-strips{world} (NCCL halo + migration)" if strip_mode else "single",
                       "l2": "flushed before every step (256 MiB write); per-iteration working set ~90 MB"},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches_per_step * args.steps,
            "clocks": clocks,
            "ms_per_iteration": {m: (statistics.mean(v) if v else None) for m, v in it_ms.items()},
            "cells_ms_per_launch": {k: (statistics.mean(v) if v else None) for k, v in cells_ms.items()},
            "cfg5": cfg5,
            "paper_e1": paper_e1,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
