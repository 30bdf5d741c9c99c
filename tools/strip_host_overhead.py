"""Host-side cost of one strip iteration (diagnostic for the strong-scaled per-rank sizes): the
strip path at P = 1 on a cfg3-like point set of n points, `iters` DistMesh or CVD iterations:
  enqueue_us : host time to enqueue one iteration (no synchronisation inside the loop)
  wall_us    : device-complete time per iteration
If enqueue_us ~ wall_us the rank is launch-bound.  python tools/strip_host_overhead.py [n ...]"""
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


def main():
    sizes = [int(v) for v in sys.argv[1:]] or [125000, 250000, 500000]
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    for n in sizes:
        c = configs.config3(n=n, grid=1024)
        params = T.default_params()
        ctx = T.Context(0, stream=stream, params=params)
        to = lambda v: torch.from_numpy(v).to(dev)
        ctx.tm_set_domain(c.box, to(c.phi), to(c.mu), to(c.rho), c.n)
        strips = S.Strips(c.box[0], c.box[2], 1)
        W = S.ghost_width(ctx.c, params.fac_voro_bound, float(c.mu.max()))
        cap_own, cap_msg = S.capacities(c.n, 1, 4096)
        St = S.split_initial(to(c.x), to(c.y), strips, 0, cap_own, cap_msg)
        comm = S.TorchP2P(0, 1, dev)
        be = S.GpuStripBackend(ctx, params.adj_stride)
        for mode in ("dm", "cvd"):
            for _ in range(10):
                S.strip_step(St, strips, be, comm, W, mode)
            ctx.tm_sync()
            iters = 25  # ~600 launches: below the launch-queue depth, so the host never blocks
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            for _ in range(iters):
                S.strip_step(St, strips, be, comm, W, mode)
            t1 = time.perf_counter()
            torch.cuda.synchronize(dev)
            t2 = time.perf_counter()
            ctx.tm_sync()
            print(json.dumps({"n": c.n, "mode": mode, "enqueue_us": 1e6 * (t1 - t0) / iters,
                              "wall_us": 1e6 * (t2 - t0) / iters}), flush=True)
        ctx.close()


if __name__ == "__main__":
    main()
