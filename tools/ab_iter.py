"""A/B timing of one iteration type between two flag sets of the cell kernel, with a
bitwise cross-check of the two variants' outputs (they must agree exactly: the cell
search never changes a result, only how fast it is certified).

  python tools/ab_iter.py --cfg 3 --flags-b 8 [--warm 6] [--iters 5]

For the config: `warm` iterations of its schedule from its points (variant A), then
for each iteration type of the schedule `iters` timed iterations of A and of B from
that same state (CUDA events on the library stream around the whole iteration and
around tm_voronoi_delaunay).  Prints one JSON line per (cfg, mode).
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2309_13824_b200 as T  # noqa: E402
from inputs import configs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int, nargs="+", default=[3])
    ap.add_argument("--flags-a", type=int, default=0)
    ap.add_argument("--flags-b", type=int, default=T.TM_F_NO_WCERT)
    ap.add_argument("--warm", type=int, default=6)
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--n5", type=int, default=16_000_000)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    to = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    for k in args.cfg:
        c = configs.load(k) if k != 5 else configs.config5(n=args.n5)
        ctxs = {}
        for name, fl in (("A", args.flags_a), ("B", args.flags_b)):
            p = T.default_params()
            p.flags |= fl
            cx = T.Context(0, stream=stream, params=p)
            cx.tm_set_domain(c.box, to(c.phi), to(c.mu), to(c.rho), c.n)
            ctxs[name] = cx
        bufs = {n: T.IterBuffers.alloc(c.n, 16, device=dev) for n in ctxs}
        x, y, dp = to(c.x), to(c.y), None
        for mode in c.schedule[:args.warm]:
            xo, yo, do = torch.empty_like(x), torch.empty_like(x), torch.empty_like(x)
            T.iterate(ctxs["A"], x, y, dp, mode, bufs["A"], xo, yo, do)
            x, y, dp = xo, yo, do
        for mode in sorted(set(c.schedule)):
            res = {}
            outs = {}
            for name, cx in ctxs.items():
                b = bufs[name]
                xo, yo, do = torch.empty_like(x), torch.empty_like(x), torch.empty_like(x)
                # one untimed iteration on this state: fills the variant's warm-start lists
                T.iterate(cx, x, y, dp, mode, b, xo, yo, do)
                it_ms, cell_ms = [], []
                for _ in range(args.iters):
                    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
                    e0.record(stream)
                    cx.tm_grid_bin(x, y)
                    e1.record(stream)
                    if mode == "cvd":
                        cx.tm_voronoi_delaunay(b.tri, b.n_tri, None, None, dp, xo, yo, do, b.status)
                    else:
                        cx.tm_voronoi_delaunay(b.tri, b.n_tri, b.adj, b.deg)
                        cx.tm_distmesh_sums(b.adj, b.deg, b.sums2)
                        cx.tm_distmesh_step(b.adj, b.deg, b.sums2, None, dp, xo, yo, do, b.status)
                    e2.record(stream)
                    e2.synchronize()
                    it_ms.append(e0.elapsed_time(e2))
                    cell_ms.append(e1.elapsed_time(e2))
                cx.tm_sync()
                nt = int(b.n_tri.item())
                tri = np.sort(b.tri[:nt].cpu().numpy(), axis=1)
                tri = tri[np.lexsort(tri.T[::-1])]
                outs[name] = (xo.cpu().numpy(), yo.cpu().numpy(), do.cpu().numpy(), b.status.cpu().numpy(), tri)
                w = cx.tm_work_counts()
                res[name] = {"iteration_ms": float(np.median(it_ms)), "after_bin_ms": float(np.median(cell_ms)),
                             "retries": w.retries}
            A, B = outs["A"], outs["B"]
            same = {"x": bool(np.array_equal(A[0], B[0])), "y": bool(np.array_equal(A[1], B[1])),
                    "d_prev": bool(np.array_equal(A[2], B[2])), "status": bool(np.array_equal(A[3], B[3])),
                    "tri": bool(A[4].shape == B[4].shape and np.array_equal(A[4], B[4]))}
            print(json.dumps({"cfg": k, "n": c.n, "mode": mode, "flags_a": args.flags_a, "flags_b": args.flags_b,
                              "A": res["A"], "B": res["B"], "speedup_A_over_B":
                                  res["B"]["iteration_ms"] / res["A"]["iteration_ms"], "identical": same}), flush=True)


if __name__ == "__main__":
    main()
