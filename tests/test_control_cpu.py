"""The library's controller (tm_control_init / tm_control_update: host code in libtrime_gpu.so,
no GPU needed) against the oracle's (oracle.Controller): identical
actions on scripted and random quality sequences."""
import ctypes

import numpy as np

import oracle as O


def _lib_step(T, ctl, q, moves):
    n = 1000
    s = T.tm_stats()
    s.n_tri = n
    s.sum_sqrt_alpha = np.sqrt(q[0]) * n
    s.sum_sqrt_beta = np.sqrt(q[1]) * n
    s.max_alpha = q[2]
    return ctl.update(s, moves), s


def test_library_controller_matches_oracle():
    import paper_2309_13824_b200 as T
    rng = np.random.default_rng(3)
    for method in ("cvd", "dm", "hybrid"):
        for trial in range(20):
            n_total = int(rng.integers(1000, 100000))
            n0 = int(n_total * rng.choice([0.2, 0.5, 1.0]))
            lib = T.Controller(n_total, n0, method)
            orc = O.Controller(n_total, n0, method=method if method != "dm" else "distmesh")
            qa, qb, am = 1.3, 1.6, 8.0
            for it in range(200):
                # shrinking relative changes: every branch gets reached
                f = 0.02 * np.exp(-it / 25.0) * rng.uniform(0.2, 1.5, 3)
                qa *= 1 - f[0]
                qb *= 1 - f[1]
                am *= 1 - f[2]
                moves = int(rng.integers(0, 3)) if it > 120 else 5
                (la, lk), s = _lib_step(T, lib, (qa, qb, am), moves)
                # the oracle sees the same 1/2-means the library derives from the sums
                na = (s.sum_sqrt_alpha / s.n_tri) ** 2
                nb = (s.sum_sqrt_beta / s.n_tri) ** 2
                od = orc.update(na, nb, s.max_alpha, moves)
                oa = od["action"]
                if oa == "terminate":
                    oa = "terminate_" + {"quality": "quality", "movement": "moves", "max_iterations": "cap"}[od["reason"]]
                assert (la, lk) == (oa, od["n_add"]), (method, trial, it, la, lk, od)
                assert lib.mode == ("cvd" if orc.mode == "cvd" else "dm")
                if la.startswith("terminate"):
                    break
