"""Phase timing of one strip iteration at P=1 on cfg3 (diagnostic): halo pack,
exchange, cells (bin + cells + DistMesh), migrate, concatenation.  Each phase
is bracketed by torch.cuda.synchronize() (so the sum exceeds the pipelined
time); prints one JSON line of milliseconds per phase, averaged."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2309_13824_b200 as T  # noqa: E402
from paper_2309_13824_b200 import strips as S  # noqa: E402
from inputs import configs  # noqa: E402


def main(reps=6):
    c = configs.load(3)
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    ctx = T.Context(0, stream=stream)
    ctx.tm_set_domain(c.box, torch.from_numpy(c.phi).to(dev), torch.from_numpy(c.mu).to(dev),
                      torch.from_numpy(c.rho).to(dev), c.n)
    x0, y0 = torch.from_numpy(c.x).to(dev), torch.from_numpy(c.y).to(dev)
    strips = S.Strips(c.box[0], c.box[2], 1)
    st = S.split_initial(x0, y0, strips, 0)
    be = S.GpuStripBackend(ctx, keep_tri=False)
    comm = S.TorchP2P(0, 1, dev)
    W = S.ghost_width(ctx.c, 5.0, float(c.mu.max()))
    acc = {}

    def tick(name, t0):
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        acc[name] = acc.get(name, 0.0) + (t1 - t0) * 1e3
        return t1

    for it in range(reps + 1):
        if it == 1:
            acc.clear()
        mode = "dm" if it % 2 == 0 else "cvd"
        lo, hi = strips.bounds(0)
        t = time.perf_counter()
        h_lo, h_hi = be.halo(st, lo, hi, W)
        t = tick("halo", t)
        g_lo, g_hi = comm.exchange(h_lo, h_hi)
        t = tick("exchange", t)
        hnd, sums2 = be.cells_begin(st, [g_lo, g_hi], mode)
        t = tick("cells_begin", t)
        tri, xo, yo, do, status = be.cells_end(hnd, sums2)
        t = tick("cells_end", t)
        nst = S.RankState(0, xo, yo, st.gid, do, tri)
        keep, m_lo, m_hi = be.migrate(nst, lo, hi)
        t = tick("migrate", t)
        r_lo, r_hi = comm.exchange(m_lo, m_hi)
        t = tick("exchange2", t)
        parts = [keep] + [r for r in (r_lo, r_hi) if r is not None]
        st = S.RankState(0, torch.cat([p[0] for p in parts]).contiguous(), torch.cat([p[1] for p in parts]).contiguous(),
                         torch.cat([p[2] for p in parts]).contiguous(), torch.cat([p[3] for p in parts]).contiguous())
        t = tick("concat", t)
    print(json.dumps({k: round(v / reps, 3) for k, v in acc.items()}), flush=True)


if __name__ == "__main__":
    main()
