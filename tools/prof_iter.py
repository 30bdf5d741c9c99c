"""Driver for ncu captures: config `cfg`, `warm` warm-up iterations of the given mode
(the first one cold, the rest warm-started), then one iteration of each mode in `modes`.
The k_cells_t launches of the last iterations are the ones to capture (-k regex:k_cells_t
-s <warm> -c <len(modes)>).

  python tools/prof_iter.py --cfg 3 --warm 5 --warm-mode dm --modes dm cvd
"""
import argparse
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
    ap.add_argument("--n5", type=int, default=16_000_000)
    ap.add_argument("--warm", type=int, default=5)
    ap.add_argument("--warm-mode", default="dm")
    ap.add_argument("--modes", nargs="+", default=["dm", "cvd"])
    ap.add_argument("--flags", type=int, default=0)
    a = ap.parse_args()
    c = configs.load(a.cfg) if a.cfg != 5 else configs.config5(n=a.n5)
    dev = torch.device("cuda", 0)
    p = T.default_params()
    p.flags |= a.flags
    ctx = T.Context(0, params=p)
    to = lambda v: None if v is None else torch.from_numpy(v).to(dev)
    ctx.tm_set_domain(c.box, to(c.phi), to(c.mu), to(c.rho), c.n)
    bufs = T.IterBuffers.alloc(c.n, ctx.params.adj_stride, device=dev)
    x, y = to(c.x), to(c.y)
    dp = None
    for mode in [a.warm_mode] * a.warm + a.modes:
        xo, yo, do = torch.empty_like(x), torch.empty_like(x), torch.empty_like(x)
        T.iterate(ctx, x, y, dp, mode, bufs, xo, yo, do)
        x, y, dp = xo, yo, do
    ctx.tm_sync()
    w = ctx.tm_work_counts()
    print("ok", int(bufs.n_tri.item()), "retries", w.retries)


if __name__ == "__main__":
    main()
