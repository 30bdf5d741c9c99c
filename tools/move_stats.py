"""Per-iteration displacement statistics of a config's schedule (design aid for displacement-
certified candidate lists): quantiles of d_prev / h(p_old) and of the cumulative displacement
since iteration k0 over h.  python tools/move_stats.py --cfg 3"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2309_13824_b200 as T  # noqa: E402
from inputs import configs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int, default=3)
    a = ap.parse_args()
    c = configs.load(a.cfg)
    dev = torch.device("cuda", 0)
    ctx = T.Context(0)
    to = lambda v: None if v is None else torch.from_numpy(v).to(dev)
    ctx.tm_set_domain(c.box, to(c.phi), to(c.mu), to(c.rho), c.n)
    bufs = T.IterBuffers.alloc(c.n, ctx.params.adj_stride, device=dev)
    x, y = to(c.x), to(c.y)
    dp = None
    # h(p) from the domain: c * mu~(p); approximate by bilinear on the host grid via torch
    mu = to(c.mu) if c.mu is not None else None
    x0, y0, x1, y1 = c.box
    def h_of(px, py):
        if mu is None:
            return torch.full_like(px, ctx.c)
        ny, nx = mu.shape
        fx = (px - x0) / (x1 - x0) * (nx - 1); fy = (py - y0) / (y1 - y0) * (ny - 1)
        i = fx.floor().clamp(0, nx - 2).long(); j = fy.floor().clamp(0, ny - 2).long()
        s = fx - i; t = fy - j
        m = (1 - t) * ((1 - s) * mu[j, i] + s * mu[j, i + 1]) + t * ((1 - s) * mu[j + 1, i] + s * mu[j + 1, i + 1])
        return ctx.c * m
    anchor = None
    for it, mode in enumerate(c.schedule):
        xo, yo, do = torch.empty_like(x), torch.empty_like(x), torch.empty_like(x)
        T.iterate(ctx, x, y, dp, mode, bufs, xo, yo, do)
        h = h_of(x, y)
        r = do / h
        if anchor is None or it % 5 == 0:
            anchor = (x.clone(), y.clone(), it)
        cum = torch.hypot(xo - anchor[0], yo - anchor[1]) / h
        q = torch.tensor([0.5, 0.9, 0.99, 0.999, 1.0], device=dev, dtype=torch.float64)
        print(json.dumps({"it": it, "mode": mode, "d_over_h": [round(v, 5) for v in torch.quantile(r[:1000000][::7], q).tolist()],
                          "cum_since": anchor[2], "cum_over_h": [round(v, 5) for v in torch.quantile(cum[::7], q).tolist()]}))
        x, y, dp = xo, yo, do


if __name__ == "__main__":
    main()
