"""A/B timing of one iteration type between two flag sets of the cell kernel, with a
bitwise cross-check of the two variants' outputs (they must agree exactly: the cell
search never changes a result, only how fast it is certified).

  python tools/ab_iter.py --cfg 3 --flags-b 8 [--warm 6] [--iters 5]

For the config: `warm` iterations of its schedule from its points, then for each
iteration type of the schedule and each variant: one untimed iteration from the state
before (so the warm-start lists come from a real previous iteration), then `iters` timed
CHAINED iterations (each from the previous output: the warm lists always lag one move
behind, as in the real schedule).  CUDA events around each iteration; the per-variant
median is reported, plus the warm-start work counters of a counted replay (TM_F_COUNT_WORK).
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
    ap.add_argument("--count", action="store_true", help="also report the work counters of variant A")
    ap.add_argument("--param-a", action="append", default=[], help="tm_params override for A, e.g. n_opt=4")
    ap.add_argument("--param-b", action="append", default=[], help="tm_params override for B")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    to = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    for k in args.cfg:
        c = configs.load(k) if k != 5 else configs.config5(n=args.n5)
        ctxs = {}
        for name, fl in (("A", args.flags_a), ("B", args.flags_b)) + ((("C", args.flags_a | T.TM_F_COUNT_WORK),)
                                                                        if args.count else ()):
            p = T.default_params()
            p.flags |= fl
            for kv in (args.param_b if name == "B" else args.param_a):
                kk, vv = kv.split("=")
                setattr(p, kk, type(getattr(p, kk))(float(vv)) if not isinstance(getattr(p, kk), int) else int(vv))
            cx = T.Context(0, stream=stream, params=p)
            cx.tm_set_domain(c.box, to(c.phi), to(c.mu), to(c.rho), c.n)
            ctxs[name] = cx
        bufs = T.IterBuffers.alloc(c.n, 16, device=dev)
        for mode in sorted(set(c.schedule)):
            # state after `warm` iterations of this mode from the config's points, and the one before
            x, y, dp = to(c.x), to(c.y), None
            prev = (x, y, dp)
            for _ in range(args.warm):
                xo, yo, do = torch.empty_like(x), torch.empty_like(x), torch.empty_like(x)
                T.iterate(ctxs["A"], x, y, dp, mode, bufs, xo, yo, do)
                prev = (x, y, dp)
                x, y, dp = xo, yo, do
            res, outs = {}, {}
            for name, cx in ctxs.items():
                xo, yo, do = torch.empty_like(x), torch.empty_like(x), torch.empty_like(x)
                T.iterate(cx, prev[0], prev[1], prev[2], mode, bufs, xo, yo, do)  # warm lists of the state before
                xc, yc, dc = x, y, dp
                it_ms, work = [], []
                for _ in range(args.iters):
                    xo, yo, do = torch.empty_like(x), torch.empty_like(x), torch.empty_like(x)
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    T.iterate(cx, xc, yc, dc, mode, bufs, xo, yo, do)
                    e1.record(stream)
                    e1.synchronize()
                    it_ms.append(e0.elapsed_time(e1))
                    if name == "C":
                        work.append(cx.tm_work_counts().as_dict())
                    xc, yc, dc = xo, yo, do
                cx.tm_sync()
                nt = int(bufs.n_tri.item())
                tri = np.sort(bufs.tri[:nt].cpu().numpy(), axis=1)
                tri = tri[np.lexsort(tri.T[::-1])]
                outs[name] = (xc.cpu().numpy(), yc.cpu().numpy(), dc.cpu().numpy(), bufs.status.cpu().numpy(), tri)
                res[name] = {"iteration_ms": float(np.median(it_ms)), "all_ms": [round(v, 4) for v in it_ms]}
                if work:
                    n = max(1, work[-1]["n_cells"])
                    res[name]["work_per_cell"] = {kk: round(v / n, 4) for kk, v in work[-1].items()}
            A, B = outs["A"], outs["B"]
            same = {"x": bool(np.array_equal(A[0], B[0])), "y": bool(np.array_equal(A[1], B[1])),
                    "d_prev": bool(np.array_equal(A[2], B[2])), "status": bool(np.array_equal(A[3], B[3])),
                    "tri": bool(A[4].shape == B[4].shape and np.array_equal(A[4], B[4]))}
            print(json.dumps({"cfg": k, "n": c.n, "mode": mode, "flags_a": args.flags_a, "flags_b": args.flags_b,
                              "A": res["A"], "B": res["B"], "C": res.get("C"),
                              "speedup_A_over_B": res["B"]["iteration_ms"] / res["A"]["iteration_ms"],
                              "identical": same}), flush=True)


if __name__ == "__main__":
    main()
