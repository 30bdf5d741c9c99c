"""Cell-kernel microbenchmark (tuning aid, not the bench contract).

cfg3 (10^6 points): W DistMesh warm-up iterations from the config's points,
then R timed tm_voronoi_delaunay launches in DistMesh mode (TRI|ELL) and R in
fused CVD mode (TRI|TREAT, adaptive quadrature) on the same sorted state;
CUDA events on the library stream.  Prints one JSON line.  The library is
$TRIME_LIB (default: the in-tree build), so compiled variants can be swept:
  TRIME_LIB=paper_2309_13824_b200/libtrime_gpu_v2.so python tools/cellbench.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2309_13824_b200 as T  # noqa: E402
from inputs import configs  # noqa: E402


def load_cfg(cfg):
    """3 (default) / 1..5: BASELINE configs; 'iid': 10^6 i.i.d. uniform points in the unit square
    (box SDF 1024^2, uniform density) -- isolates the point distribution from the adaptive grids."""
    if cfg == "iid":
        import numpy as np
        box = (0.0, 0.0, 1.0, 1.0)
        x, y = configs.random_points(1_000_000, 7, box)
        return configs.Config("iid1e6", x, y, box, configs.box_phi(box, 1024), None, None, ["dm", "cvd"])
    return configs.load(int(cfg))


def main(cfg=3, warm=3, reps=10, group=False, n_opt=None):
    c = load_cfg(cfg)
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    p = T.default_params()
    if group:
        p.flags |= T.TM_F_GROUP_CELLS
    if n_opt:
        p.n_opt = n_opt
    ctx = T.Context(0, stream=stream, params=p)
    ctx.tm_set_domain(c.box, torch.from_numpy(c.phi).to(dev),
                      None if c.mu is None else torch.from_numpy(c.mu).to(dev),
                      None if c.rho is None else torch.from_numpy(c.rho).to(dev), c.n)
    bufs = T.IterBuffers.alloc(c.n, ctx.params.adj_stride, device=dev)
    x, y = torch.from_numpy(c.x).to(dev), torch.from_numpy(c.y).to(dev)
    dp = None
    for _ in range(warm):
        xo, yo, do = torch.empty_like(x), torch.empty_like(x), torch.empty_like(x)
        T.iterate(ctx, x, y, dp, "dm", bufs, xo, yo, do)
        x, y, dp = xo, yo, do
    ctx.tm_grid_bin(x, y)
    xo, yo, do = torch.empty_like(x), torch.empty_like(x), torch.empty_like(x)
    out = {"lib": os.path.basename(T.LIB_PATH), "cells": "group" if group else "thread", "n_opt": p.n_opt,
           "config": c.name, "n": c.n}
    for mode in ("dm", "cvd"):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps + 1)]
        for r in range(reps + 1):
            ev[r][0].record(stream)
            if mode == "dm":
                ctx.tm_voronoi_delaunay(bufs.tri, bufs.n_tri, bufs.adj, bufs.deg)
            else:
                ctx.tm_voronoi_delaunay(bufs.tri, bufs.n_tri, None, None, dp, xo, yo, do, bufs.status)
            ev[r][1].record(stream)
        ctx.tm_sync()
        ms = [a.elapsed_time(b) for a, b in ev[1:]]
        out[f"{mode}_ms"] = sum(ms) / len(ms)
        out[f"{mode}_ms_min"] = min(ms)
        out[f"{mode}_n_tri"] = int(bufs.n_tri.item())
        out[f"{mode}_retries"] = int(ctx.tm_work_counts().retries)
    print(json.dumps(out), flush=True)
    ctx.close()


if __name__ == "__main__":
    nopts = [None]
    for a in sys.argv[1:]:
        if a.startswith("--n-opt="):
            nopts = [float(v) for v in a.split("=", 1)[1].split(",")]
    cfg = "3"
    for a in sys.argv[1:]:
        if a.startswith("--cfg="):
            cfg = a.split("=", 1)[1]
    for v in nopts:
        main(cfg=cfg, group="--group" in sys.argv, n_opt=v)
