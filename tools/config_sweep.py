"""Per-config, per-iteration-type throughput and roofline fraction (SURVEY §8(d)
"Evidence required": f per config and per iteration type).

For each config and each iteration type of its schedule: W warm-up iterations of
that type from the config's points, then T timed CHAINED iterations (each from the
previous output, warm-start lists one move behind, as in the real schedule):
  * eager: CUDA events around each iteration and around tm_voronoi_delaunay;
  * graph: the same T-iteration chain captured once (tm_graph_*) and replayed.
The algorithmic work comes from the kernel's own counters (TM_F_COUNT_WORK) on the
last state, warm-started from the state before it, with the §8(d) cost table;
T_roof = S1 bytes / BW + max(fused bytes / BW, F_cells / P_DP) (+ DistMesh stage).
Prints one JSON line per (config, mode).

  python tools/config_sweep.py [cfg ...]      (default: 1 2 3 4 5)
"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2309_13824_b200 as T  # noqa: E402
from inputs import configs  # noqa: E402


def run(k, warm=4, timed=5):
    c = configs.load(k)
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    to = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    ctx = T.Context(0, stream=stream)
    ctx.tm_set_domain(c.box, to(c.phi), to(c.mu), to(c.rho), c.n)
    pc = T.default_params()
    pc.flags |= T.TM_F_COUNT_WORK
    cctx = T.Context(0, stream=stream, params=pc)
    cctx.tm_set_domain(c.box, to(c.phi), to(c.mu), to(c.rho), c.n)
    bufs = T.IterBuffers.alloc(c.n, ctx.params.adj_stride, device=dev)
    P, _ = bench.dp_peak()
    BW, _ = bench.hbm_peak()
    out = []
    for mode in sorted(set(c.schedule)):
        x, y, dp = to(c.x), to(c.y), None
        prev = (x, y, dp)
        for _ in range(warm):
            xo, yo, do = torch.empty_like(x), torch.empty_like(x), torch.empty_like(x)
            T.iterate(ctx, x, y, dp, mode, bufs, xo, yo, do)
            prev, (x, y, dp) = (x, y, dp), (xo, yo, do)
        B = [[torch.empty_like(x) for _ in range(3)] for _ in range(2)]

        def chain(record=None):
            xs, ys, ds = x, y, dp
            for t in range(timed):
                xo, yo, do = B[t % 2]
                if record is not None:
                    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
                    e[0].record(stream)
                ctx.tm_grid_bin(xs, ys)
                if record is not None:
                    e[1].record(stream)
                if mode == "cvd":
                    ctx.tm_voronoi_delaunay(bufs.tri, bufs.n_tri, None, None, ds, xo, yo, do, bufs.status)
                else:
                    ctx.tm_voronoi_delaunay(bufs.tri, bufs.n_tri, bufs.adj, bufs.deg)
                    ctx.tm_distmesh_sums(bufs.adj, bufs.deg, bufs.sums2)
                    ctx.tm_distmesh_step(bufs.adj, bufs.deg, bufs.sums2, None, ds, xo, yo, do, bufs.status)
                if record is not None:
                    e[2].record(stream)
                    record.append(e)
                xs, ys, ds = xo, yo, do
            return xs, ys, ds

        T.iterate(ctx, prev[0], prev[1], prev[2], mode, bufs, *B[1])  # warm lists of the state before
        rec = []
        chain(rec)
        ctx.tm_sync()
        it_ms = [a.elapsed_time(cc) for a, b, cc in rec]
        cell_ms = [b.elapsed_time(cc) for a, b, cc in rec]
        # the same chain as one CUDA Graph
        T.iterate(ctx, prev[0], prev[1], prev[2], mode, bufs, *B[1])
        g = ctx.capture(chain)
        g.launch()
        ctx.tm_sync()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for _ in range(3):
            g.launch()
        g1.record(stream)
        g1.synchronize()
        graph_ms = g0.elapsed_time(g1) / (3 * timed)
        g.close()
        # work counters of a warm-started launch: the counting context on S0, then on its output
        xo2, yo2, do2 = torch.empty_like(x), torch.empty_like(x), torch.empty_like(x)
        T.iterate(cctx, x, y, dp, mode, bufs, xo2, yo2, do2)
        cctx.tm_grid_bin(xo2, yo2)
        if mode == "cvd":
            cctx.tm_voronoi_delaunay(bufs.tri, bufs.n_tri, None, None, do2, *B[0], bufs.status)
        else:
            cctx.tm_voronoi_delaunay(bufs.tri, bufs.n_tri, bufs.adj, bufs.deg)
        w = cctx.tm_work_counts()
        troof, fc = bench.iteration_roof(mode, w, c.n, P, BW)
        im, cm = statistics.median(it_ms), statistics.median(cell_ms)
        nc = max(w.n_cells, 1)
        out.append({"config": c.name, "n": c.n, "mode": mode, "iteration_ms": round(im, 4),
                    "iteration_ms_graph": round(graph_ms, 4), "cells_and_update_ms": round(cm, 4),
                    "pts_it_per_s": c.n / (im * 1e-3), "pts_it_per_s_graph": c.n / (graph_ms * 1e-3),
                    "T_roof_us": troof * 1e6, "frac_iteration": troof / (min(im, graph_ms) * 1e-3),
                    "alg_dp_inst_cells": fc, "peak_dp_inst_per_s": P,
                    "work_per_cell": {kk: round(getattr(w, kk) / nc, 3) for kk in
                                      ("n_cert", "deg", "verts", "t_own", "quad_tris", "ell", "candidates", "clips",
                                       "retries")}})
        print(json.dumps(out[-1]), flush=True)
    ctx.close()
    cctx.close()
    return out


if __name__ == "__main__":
    ks = [int(a) for a in sys.argv[1:]] or [1, 2, 3, 4, 5]
    for k in ks:
        run(k)
