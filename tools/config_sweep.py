"""Per-config, per-iteration-type throughput and roofline fraction of the cell
kernel (SURVEY §8(d) "Evidence required": f per config and per iteration
type).  For each config: W warm-up iterations of its schedule, then T timed
iterations of each iteration type it uses (DistMesh / CVD) from the warmed
state; CUDA events around the whole iteration and around tm_voronoi_delaunay.
The algorithmic DP count comes from the kernel's own work counters (an
untimed TM_F_COUNT_WORK pass on the same state) with the §8(d) cost table.
Prints one JSON line per (config, mode).

  python tools/config_sweep.py [cfg ...]      (default: 1 2 3 4 5)
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2309_13824_b200 as T  # noqa: E402
from inputs import configs  # noqa: E402


def peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "profiles", "fp64_peak.json")))["dp_inst_per_s"])
    except Exception:
        return 148 * 64 * 1965e6


def f_alg(w, mode, adaptive):
    """SURVEY §8(d) per cell: 4 n_cert + 5 deg V + 50 deg + 40 T_own, plus for the fused CVD update
    [6 V + 15 (uniform rho) | 30 Q (adaptive quadrature)] + 20 (projection test); summed over cells."""
    n = max(w.n_cells, 1)
    f = 4 * w.n_cert + 5 * w.deg * (w.verts / n) + 50 * w.deg + 40 * w.t_own
    if mode == "cvd":
        f += (30 * w.quad_tris if adaptive else 6 * w.verts + 15 * n) + 20 * n
    return f


def run(k, warm=3, timed=5):
    c = configs.load(k)
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    to = lambda a: None if a is None else torch.from_numpy(a).to(dev)
    ctx = T.Context(0, stream=stream)
    ctx.tm_set_domain(c.box, to(c.phi), to(c.mu), to(c.rho), c.n)
    pc = T.default_params()
    pc.flags |= T.TM_F_COUNT_WORK
    cctx = T.Context(0, stream=stream, params=pc)
    cctx.tm_set_domain(c.box, to(c.phi), to(c.mu), to(c.rho), c.n)
    bufs = T.IterBuffers.alloc(c.n, ctx.params.adj_stride, device=dev)
    x, y, dp = to(c.x), to(c.y), None
    for mode in c.schedule[:warm]:
        xo, yo, do = torch.empty_like(x), torch.empty_like(x), torch.empty_like(x)
        T.iterate(ctx, x, y, dp, mode, bufs, xo, yo, do)
        x, y, dp = xo, yo, do
    out = []
    for mode in sorted(set(c.schedule)):
        it_ms, cell_ms = [], []
        xs, ys, ds = x, y, dp
        for r in range(timed):
            xo, yo, do = torch.empty_like(x), torch.empty_like(x), torch.empty_like(x)
            e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            e[0].record(stream)
            ctx.tm_grid_bin(xs, ys)
            e[1].record(stream)
            if mode == "cvd":
                ctx.tm_voronoi_delaunay(bufs.tri, bufs.n_tri, None, None, ds, xo, yo, do, bufs.status)
            else:
                ctx.tm_voronoi_delaunay(bufs.tri, bufs.n_tri, bufs.adj, bufs.deg)
            e[2].record(stream)
            if mode == "dm":
                ctx.tm_distmesh_sums(bufs.adj, bufs.deg, bufs.sums2)
                ctx.tm_distmesh_step(bufs.adj, bufs.deg, bufs.sums2, None, ds, xo, yo, do, bufs.status)
            e[3].record(stream)
            ctx.tm_sync()
            it_ms.append(e[0].elapsed_time(e[3]))
            cell_ms.append(e[1].elapsed_time(e[2]))
        # work counters on the same input state
        cctx.tm_grid_bin(xs, ys)
        xo2, yo2, do2 = torch.empty_like(x), torch.empty_like(x), torch.empty_like(x)
        if mode == "cvd":
            cctx.tm_voronoi_delaunay(bufs.tri, bufs.n_tri, None, None, ds, xo2, yo2, do2, bufs.status)
        else:
            cctx.tm_voronoi_delaunay(bufs.tri, bufs.n_tri, bufs.adj, bufs.deg)
        w = cctx.tm_work_counts()
        F = f_alg(w, mode, c.rho is not None)
        cm = sorted(cell_ms)[len(cell_ms) // 2]
        im = sorted(it_ms)[len(it_ms) // 2]
        P = peak()
        out.append({"config": c.name, "n": c.n, "mode": mode, "iteration_ms": round(im, 4), "cells_ms": round(cm, 4),
                    "pts_it_per_s": c.n / (im * 1e-3), "alg_dp_inst_per_launch": F,
                    "achieved_dp_inst_per_s": F / (cm * 1e-3), "peak_dp_inst_per_s": P,
                    "roofline_frac_cells": F / (cm * 1e-3) / P,
                    "work_per_cell": {kk: round(getattr(w, kk) / max(w.n_cells, 1), 3) for kk in
                                      ("n_cert", "deg", "verts", "t_own", "quad_tris", "candidates", "clips",
                                       "exact_calls")},
                    "retries": int(w.retries),
                    "lane_utilisation_search": w.candidates / max(1, 32 * w.warp_trips)})
        print(json.dumps(out[-1]), flush=True)
    ctx.close()
    cctx.close()
    return out


if __name__ == "__main__":
    ks = [int(a) for a in sys.argv[1:]] or [1, 2, 3, 4, 5]
    for k in ks:
        run(k)
