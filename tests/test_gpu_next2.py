"""GPU parity of the NEXT-2 / NEXT-3 rows against the oracle:
* the paper's validity Tests 1-3 (tm_params.validity = 1) inside full iterations:
  kept-triangle sets exactly equal, CVD bit for bit;
* the movement-termination count -- exact integer;
* tm_set_n_total: c and h_avg bit for bit against the oracle's normalisation at N;
* point addition: the same new points, bit for bit, and the same smallest ratio;
* meshing to termination (tm_control + mesh()): from fac_init * N_total points, every iteration
  checked against the oracle from the GPU's own state, every controller decision against the
  oracle controller fed with the oracle's quality of that state, every added point set against
  the oracle's point addition on the same mesh."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import oracle as O
from inputs import configs
from tests.gpu_util import GpuRunner, compare, to_dev


def _disk(n, seed, r=1.0):
    rng = np.random.default_rng(seed)
    P = rng.uniform(-r, r, (4 * n, 2))
    P = P[P[:, 0] ** 2 + P[:, 1] ** 2 < r * r][:n]
    return P[:, 0].copy(), P[:, 1].copy()


@pytest.mark.parametrize("k,modes", [(1, ["cvd", "dm"]), (2, ["dm"] * 4 + ["cvd"]), (3, ["dm"] * 3 + ["cvd"])])
def test_validity_tests_in_iterations(k, modes, cfg_cache):
    import paper_2309_13824_b200 as T
    c = cfg_cache(k)
    r = GpuRunner(c.box, c.phi, c.mu, c.rho, params=T.default_params(validity=1))
    fs = O.FieldSet.from_config(c)
    op = O.default_params(validity=1)
    x, y, dp = c.x, c.y, None
    for it, mode in enumerate(modes):
        g = r.iteration(x, y, mode, dp)
        o = O.iteration(fs, x, y, mode, d_prev=dp, params=op)
        compare(g, o, c.box, mode, ctx=f"cfg{k} it{it} {mode} validity=1")
        x, y, dp = g["x"], g["y"], g["d_prev"]


def test_validity_tests_decide_boundary_strip():
    """The smooth configs keep the same set under both readings (the octagon bound discards the
    triangles Tests 2-3 would decide).  inputs.configs.validity_strip() places points just outside
    (phi = +4e-4 <= geps) and inside (-2e-4) a straight boundary and a few outside (phi = 0.1):
    boundary triangles with centroids in (0, geps] and triangles decided by Test 3."""
    import paper_2309_13824_b200 as T
    box, phi, x, y = configs.validity_strip()
    r = GpuRunner(box, phi, params=T.default_params(validity=1))
    fs = O.FieldSet(box, phi)
    for mode in ("cvd", "dm"):
        g = r.iteration(x, y, mode)
        o = O.iteration(fs, x, y, mode, params=O.default_params(validity=1))
        o1 = O.iteration(fs, x, y, mode)
        assert o.info.n_degenerate == 0
        assert len(set(map(tuple, o.tri.tolist())) - set(map(tuple, o1.tri.tolist()))) > 0
        compare(g, o, box, mode, ctx=f"validity strip {mode}")


def test_move_count_matches_oracle(cfg_cache):
    c = cfg_cache(3)
    r = GpuRunner(c.box, c.phi, c.mu, c.rho)
    g = r.iteration(c.x, c.y, "dm")
    g2 = r.iteration(g["x"], g["y"], "cvd", g["d_prev"])
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    r.ctx.tm_move_count(to_dev(g["x"]), to_dev(g["y"]), to_dev(g2["d_prev"]), cnt)
    fs = O.FieldSet.from_config(c)
    oc, oh = O.domain(fs, c.n)
    exp = O.move_count(fs, oc, oh, g["x"], g["y"], g2["d_prev"])
    assert int(cnt.item()) == exp
    assert 0 < exp < c.n


def test_set_n_total_matches_oracle_normalisation(cfg_cache):
    c = cfg_cache(3)
    r = GpuRunner(c.box, c.phi, c.mu, c.rho)
    r.set_domain(c.n)
    fs = O.FieldSet.from_config(c)
    for n in (200_000, 320_000, 512_000, 1_000_000):
        gc, gh = r.ctx.tm_set_n_total(n)
        oc, oh = O.domain(fs, n)
        assert gc == oc and gh == oh, (n, gc, oc, gh, oh)


@pytest.mark.parametrize("k,frac", [(2, 0.3), (3, 0.6)])
def test_point_addition_matches_oracle(k, frac, cfg_cache):
    c = cfg_cache(k)
    n = 200_000 if k == 3 else c.n
    x, y = c.x[:n], c.y[:n]
    r = GpuRunner(c.box, c.phi, c.mu, c.rho, n_total=n)
    g = r.iteration(x, y, "dm")
    tri = g["tri"]
    kadd = int(frac * n)
    xn = torch.empty(kadd, dtype=torch.float64, device="cuda")
    yn = torch.empty_like(xn)
    rmin = r.ctx.tm_point_addition(to_dev(tri, torch.int32), len(tri), to_dev(x), to_dev(y), kadd, xn, yn)
    fs = O.FieldSet.from_config(c)
    oc, _ = O.domain(fs, n)
    assert r.ctx.c == oc
    ox, oy, orm = O.point_addition(fs, oc, tri, x, y, kadd)
    assert rmin == orm
    assert np.array_equal(xn.cpu().numpy(), ox) and np.array_equal(yn.cpu().numpy(), oy)


def _near_threshold(prev, cur, cp, tol=1e-9):
    """any controller comparison within tol (relative) of its threshold: a legitimate tie"""
    if prev is None:
        return False
    rel = [abs(c - p) / p for c, p in zip(cur, prev)]
    ths = [cp.t_add_quality, cp.t_switch_quality, cp.t_end_quality, cp.t_end_alpha_max]
    return any(abs(r - t) <= tol * t for r in rel for t in ths)


def _checker(ctx, fs, box, op, octl, st):
    """Per-iteration parity of mesh(): the oracle's iteration from the GPU's state (kept sets exact,
    positions within the bar, CVD bit for bit), the movement count, the controller decision (fed
    with the oracle's quality of that state; only exact ties may differ) and the added points."""
    def check(d):
        it, mode = d["it"], d["mode"]
        x, y = d["x"].cpu().numpy(), d["y"].cpu().numpy()
        n = len(x)
        if st["expect_new"] is not None:  # the points added after the previous iteration
            n0, ex, ey = st["expect_new"]
            assert np.array_equal(x[n0:], ex) and np.array_equal(y[n0:], ey), f"it{it}: added points differ"
            st["expect_new"] = None
        dpi = None if d["d_prev_in"] is None else d["d_prev_in"].cpu().numpy()
        o = O.iteration(fs, x, y, mode, d_prev=dpi, params=op, n_total=n)
        assert o.info.c == ctx.c and o.info.h_avg == ctx.h_avg
        g = {"tri": d["tri"].cpu().numpy(), "x": d["x_out"].cpu().numpy(), "y": d["y_out"].cpu().numpy(),
             "d_prev": d["d_prev_out"].cpu().numpy(), "status": d["status"].cpu().numpy()}
        compare({**g, "adj": None}, o, box, mode, ctx=f"mesh it{it} {mode}")
        omc = O.move_count(fs, o.info.c, o.info.h_avg, x, y, o.d_prev)
        assert omc == d["moves"], f"it{it}: move count {d['moves']} vs oracle {omc}"
        prev = octl.prev
        oq = O.quality_of(O.stats(o.tri, x, y))
        oa = octl.update(*oq, move_count=omc)
        if oa["action"] == "terminate":
            oa["action"] = "terminate_" + {"quality": "quality", "movement": "moves", "max_iterations": "cap"}[oa["reason"]]
        if oa["action"] != d["action"] or oa["n_add"] != d["n_add"]:
            assert _near_threshold(prev, oq, octl.cp), f"it{it}: GPU {d['action']} vs oracle {oa}"
            st["ties"] += 1
        if d["action"] == "add":
            ex, ey, _ = O.point_addition(fs, o.info.c, g["tri"], x, y, d["n_add"])
            st["expect_new"] = (n, ex, ey)
        st["its"] += 1
    return check


def test_mesh_to_termination_with_point_addition():
    """Unit disk, N_total = 2500 from fac_init = 0.2, hybrid DistMesh -> CVD, the paper's
    validity tests.  Every iteration is checked against the oracle from the GPU's state, every
    controller decision against the oracle controller fed with the oracle's quality of that state,
    every point addition against the oracle's on the same mesh; the run must add points up to
    N_total, switch to CVD and terminate."""
    import paper_2309_13824_b200 as T
    box = (-1.1, -1.1, 1.1, 1.1)
    phi = configs.disk_phi(box, 257)
    n_total = 2500
    x0, y0 = _disk(int(0.2 * n_total), 11)
    ctx = T.Context(0, params=T.default_params(validity=1))
    ctx.tm_set_domain(box, to_dev(phi), None, None, len(x0))
    fs = O.FieldSet(box, phi)
    octl = O.Controller(n_total, len(x0), method="hybrid")
    octl.cp.max_iterations = 400
    st = {"expect_new": None, "ties": 0, "its": 0}
    res = T.mesh(ctx, to_dev(x0), to_dev(y0), n_total=n_total, method="hybrid", max_iterations=400,
                 on_iteration=_checker(ctx, fs, box, O.default_params(validity=1), octl, st))
    acts = [h["action"] for h in res.history]
    assert acts[-1] in ("terminate_quality", "terminate_moves"), res.history[-1]
    assert res.x.shape[0] == n_total and st["ties"] == 0 and st["its"] == res.iterations
    assert "switch" in acts and acts.count("add") >= 3


def test_adaptive_mesh_to_termination(cfg_cache):
    """cfg3's adaptive annulus fields (rho = mu^-2, mu between 0.002 and 0.02) at N_total = 20000:
    Floyd-Steinberg initial points for fac_init = 0.2 (NEXT-4), then CVD meshing with point
    addition to termination, every iteration, decision and added point set checked against the
    oracle (the R_circ / h(g) ranking with non-uniform h, the rescaled c, the adaptive quadrature)."""
    import paper_2309_13824_b200 as T
    c = cfg_cache(3)
    n_total = 20_000
    n_init = int(0.2 * n_total)
    ctx = T.Context(0, params=T.default_params(validity=1))
    phi, mu, rho = to_dev(c.phi), to_dev(c.mu), to_dev(c.rho)
    ctx.tm_set_domain(c.box, phi, mu, rho, n_init)
    nxg, nyg = T.geometry_grid_dims(n_total, c.box)
    x, y, _, _ = T.initial_points(ctx, n_init, nxg, nyg, seed=9)
    ctx.tm_set_domain(c.box, phi, mu, rho, x.shape[0])
    fs = O.FieldSet.from_config(c)
    octl = O.Controller(n_total, x.shape[0], method="cvd")
    octl.cp.max_iterations = 300
    st = {"expect_new": None, "ties": 0, "its": 0}
    res = T.mesh(ctx, x, y, n_total=n_total, method="cvd", max_iterations=300,
                 on_iteration=_checker(ctx, fs, c.box, O.default_params(validity=1), octl, st))
    acts = [h["action"] for h in res.history]
    assert acts[-1] in ("terminate_quality", "terminate_moves"), acts[-3:]
    assert res.x.shape[0] == n_total and st["ties"] == 0 and acts.count("add") >= 3
