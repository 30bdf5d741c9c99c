"""The paper's uniform-square experiment end to end on the GPU (E1/E2; Table):
N_total = 10^6 points in the unit square, initial points by Floyd-Steinberg dithering on the
geometry grid (fac_init = 1 "init all", or 0.2 "point addition"), then meshing to termination with
the paper's validity tests and controller (CVD, DistMesh, hybrid).  Reports the number of
triangulations, the time per triangulation iteration (the paper's metric: wall time of the
whole meshing loop -- controller syncs included -- divided by the triangulations), and the final
mesh quality (triangles, median alpha).  Context, not a bench line.

  python tools/paper_e1.py [--n 1000000] [--methods cvd,dm,hybrid] [--schemes all,add]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2309_13824_b200 as T  # noqa: E402
from inputs import configs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--methods", default="cvd,dm,hybrid")
    ap.add_argument("--schemes", default="all,add")
    ap.add_argument("--grid", type=int, default=1024)
    ap.add_argument("--max-iterations", type=int, default=400)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    box = (0.0, 0.0, 1.0, 1.0)
    phi = torch.from_numpy(configs.box_phi(box, a.grid)).to(dev)
    nxg, nyg = T.geometry_grid_dims(a.n, box)
    for scheme in a.schemes.split(","):
        for method in a.methods.split(","):
            ctx = T.Context(0, params=T.default_params(validity=1))
            n_init = a.n if scheme == "all" else int(0.2 * a.n)
            ctx.tm_set_domain(box, phi, None, None, n_init)
            x, y, _, _ = T.initial_points(ctx, n_init, nxg, nyg, seed=3)
            ctx.tm_set_domain(box, phi, None, None, x.shape[0])
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            res = T.mesh(ctx, x, y, n_total=a.n, method=method, max_iterations=a.max_iterations)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            xs, ys = res.x.cpu().numpy(), res.y.cpu().numpy()
            t = res.tri.cpu().numpy()
            A = np.stack([xs[t[:, 0]], ys[t[:, 0]]], 1)
            B = np.stack([xs[t[:, 1]], ys[t[:, 1]]], 1)
            C = np.stack([xs[t[:, 2]], ys[t[:, 2]]], 1)
            la = np.linalg.norm(B - C, axis=1)
            lb = np.linalg.norm(A - C, axis=1)
            lc = np.linalg.norm(A - B, axis=1)
            cr = np.abs((B[:, 0] - A[:, 0]) * (C[:, 1] - A[:, 1]) - (B[:, 1] - A[:, 1]) * (C[:, 0] - A[:, 0]))
            s = 0.5 * (la + lb + lc)
            alpha = la * lb * lc * s / (2 * cr * cr)
            h = res.history
            print(json.dumps({
                "scheme": "init all" if scheme == "all" else "point addition", "method": method, "n_total": a.n,
                "n_init": int(x.shape[0]), "triangulations": res.iterations, "seconds": dt,
                "s_per_triangulation": dt / res.iterations, "end": h[-1]["action"],
                "switch_at": next((e["it"] for e in h if e["action"] == "switch"), None),
                "adds": [e["n_add"] for e in h if e["action"] == "add"],
                "n_tri": int(t.shape[0]), "median_alpha": float(np.median(alpha)),
                "half_mean_alpha": h[-1]["half_alpha"], "max_alpha": h[-1]["max_alpha"],
                "euler_boundary_b": int(2 * a.n - 2 - t.shape[0])}), flush=True)
            ctx.close()


if __name__ == "__main__":
    main()
