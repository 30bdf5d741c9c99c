"""Small driver for ncu: cfg3 (10^6 points), W warm-up iterations of the hybrid
schedule, then one DistMesh and one CVD iteration (the launches to capture)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2309_13824_b200 as T  # noqa: E402
from inputs import configs  # noqa: E402


def main(cfg=3, warm=4):
    c = configs.load(cfg)
    dev = torch.device("cuda", 0)
    ctx = T.Context(0)
    ctx.tm_set_domain(c.box, torch.from_numpy(c.phi).to(dev),
                      None if c.mu is None else torch.from_numpy(c.mu).to(dev),
                      None if c.rho is None else torch.from_numpy(c.rho).to(dev), c.n)
    bufs = T.IterBuffers.alloc(c.n, ctx.params.adj_stride, device=dev)
    x, y = torch.from_numpy(c.x).to(dev), torch.from_numpy(c.y).to(dev)
    dp = None
    sched = ["dm"] * warm + ["dm", "cvd"]
    for mode in sched:
        xo, yo, do = torch.empty_like(x), torch.empty_like(x), torch.empty_like(x)
        T.iterate(ctx, x, y, dp, mode, bufs, xo, yo, do)
        x, y, dp = xo, yo, do
    ctx.tm_sync()
    print("ok", int(bufs.n_tri.item()))


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 3)
