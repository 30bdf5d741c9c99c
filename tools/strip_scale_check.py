"""Dry run of the driver's scaling run on ONE GPU: the bench's N = 2, 4, 8 strip set-ups (the same
strips, halo width and capacities as bench.py's cfg3 leg and run_cfg5_strips), with the P ranks run
as logical ranks through the loopback exchanger (strips.loopback_step; no rank waits on another).
Checks what a real N-GPU run could trip over: no latched capacity / overflow error on any rank over
the whole schedule, every point owned exactly once after every iteration, and the final state
against the single-domain run (CVD-only cfg5: bit-identical positions and the same triangle count;
cfg3: the same number of points, triangle count within 0.01 %).  Prints one JSON line per case.
  python tools/strip_scale_check.py [--cfg5-n 16000000]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2309_13824_b200 as T  # noqa: E402
from paper_2309_13824_b200 import strips as S  # noqa: E402
from inputs import configs  # noqa: E402


def single(c, schedule, dev, fields):
    ctx = T.Context(0)
    ctx.tm_set_domain(c.box, *fields, c.n)
    n = c.n
    bufs = T.IterBuffers.alloc(n, ctx.params.adj_stride, device=dev)
    X = [torch.empty(n, dtype=torch.float64, device=dev) for _ in range(2)]
    Y = [torch.empty(n, dtype=torch.float64, device=dev) for _ in range(2)]
    D = [torch.empty(n, dtype=torch.float64, device=dev) for _ in range(2)]
    xc, yc, dc = torch.from_numpy(c.x).to(dev), torch.from_numpy(c.y).to(dev), None
    for it, mode in enumerate(schedule):
        xo, yo, do = X[it % 2], Y[it % 2], D[it % 2]
        ctx.tm_grid_bin(xc, yc)
        if mode == "cvd":
            ctx.tm_voronoi_delaunay(bufs.tri, bufs.n_tri, None, None, dc, xo, yo, do, bufs.status)
        else:
            ctx.tm_voronoi_delaunay(bufs.tri, bufs.n_tri, bufs.adj, bufs.deg)
            ctx.tm_distmesh_sums(bufs.adj, bufs.deg, bufs.sums2)
            ctx.tm_distmesh_step(bufs.adj, bufs.deg, bufs.sums2, None, dc, xo, yo, do, bufs.status)
        xc, yc, dc = xo, yo, do
    ctx.tm_sync()
    out = (xc.cpu().numpy().copy(), yc.cpu().numpy().copy(), int(bufs.n_tri.item()))
    ctx.close()
    return out


def strips_run(c, schedule, P, dev, fields, quantiles, mu_max):
    params = T.default_params()
    backends = []
    for r in range(P):
        ctx = T.Context(0, params=params)
        cc, _ = ctx.tm_set_domain(c.box, *fields, c.n)
        backends.append(S.GpuStripBackend(ctx, params.adj_stride))
    n = c.n
    x0, y0 = torch.from_numpy(c.x).to(dev), torch.from_numpy(c.y).to(dev)
    W = S.ghost_width(cc, params.fac_voro_bound, mu_max)
    if quantiles:   # bench.py main(): cfg3
        strips = S.Strips.from_quantiles(torch.from_numpy(c.x), P, c.box[0], c.box[2])
        cap_own, _ = S.capacities(n, P, 0)
        g0 = 0
        for r in range(P):
            S0 = S.split_initial(x0, y0, strips, r, cap_own, cap_own)
            backends[r].halo_pack(S0, *strips.bounds(r), W)
            g0 = max(g0, S0.h_send[0].count(), S0.h_send[1].count())
        # fixed-size messages: one capacity for all ranks (the bench all-reduces the MAX)
        cap_msg = [min(cap_own, 4 * g0 + 4096)] * P
    else:           # run_cfg5_strips
        strips = S.Strips(c.box[0], c.box[2], P)
        cap_own, cm = S.capacities(n, P, int(n * W) + 1)
        cap_msg = [cm] * P
    states = [S.split_initial(x0, y0, strips, r, cap_own, cap_msg[r]) for r in range(P)]
    owned_max = 0
    for it, mode in enumerate(schedule):
        S.loopback_step(states, strips, backends, W, mode)
        if it % 10 == 9 or it == len(schedule) - 1:
            for b in backends:
                b.ctx.tm_sync()   # raises on a latched capacity error
            owned = [int(st.counts[0].item()) for st in states]
            assert sum(owned) == n, (it, owned)
            owned_max = max(owned_max, max(owned))
    import numpy as np
    xs, ys = np.empty(n), np.empty(n)
    seen = np.zeros(n, bool)
    ntri = 0
    for st, b in zip(states, backends):
        x, y, g, d = st.owned()
        gid = g.cpu().numpy().astype(np.int64)
        assert not seen[gid].any()
        seen[gid] = True
        xs[gid], ys[gid] = x.cpu().numpy(), y.cpu().numpy()
        ntri += int(b.triangles().shape[0])
    assert seen.all()
    for b in backends:
        b.ctx.close()
    return xs, ys, ntri, {"cap_own": cap_own, "cap_msg": cap_msg, "owned_max": owned_max, "W": W}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg5-n", type=int, default=16_000_000)
    ap.add_argument("--P", type=int, nargs="+", default=[2, 4, 8])
    a = ap.parse_args()
    import numpy as np
    dev = torch.device("cuda", 0)
    to = lambda v: None if v is None else torch.from_numpy(v).to(dev)
    for name, c, quant in (("cfg3", configs.load(3), True), ("cfg5", configs.config5(n=a.cfg5_n, iters=20), False)):
        schedule = list(c.schedule)
        fields = (to(c.phi), to(c.mu), to(c.rho))
        mu_max = float(c.mu.max()) if c.mu is not None else 1.0
        xr, yr, tr = single(c, schedule, dev, fields)
        for P in a.P:
            xs, ys, nt, info = strips_run(c, schedule, P, dev, fields, quant, mu_max)
            err = float(np.hypot(xs - xr, ys - yr).max())
            line = {"case": name, "n": c.n, "P": P, "iterations": len(schedule), "errors": 0,
                    "tri_single": tr, "tri_strips": nt, "max_pos_diff_vs_single": err,
                    "bit_identical": bool(np.array_equal(xs, xr) and np.array_equal(ys, yr)), **info}
            print(json.dumps(line), flush=True)
            if name == "cfg5":
                assert line["bit_identical"] and nt == tr, line
            else:
                assert abs(nt - tr) <= 1e-4 * tr, line


if __name__ == "__main__":
    main()
