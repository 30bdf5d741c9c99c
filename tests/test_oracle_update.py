"""Pins for O4 (CVD centroid), O5 (DistMesh,
P:139-164), O6 (treatment), O7 (quality) and the
S0 normalisation (§8.0 'Local size')."""
import math

import numpy as np
import pytest

import oracle as O
from inputs import configs

BOX = (0.0, 0.0, 1.0, 1.0)


def unit_fields(n=64, rho=None, mu=None):
    return O.FieldSet(BOX, configs.box_phi(BOX, n), mu, rho)


def grid_xy(n=64, box=BOX):
    gx = configs.node_coords(box[0], box[2], n)
    gy = configs.node_coords(box[1], box[3], n)
    return np.meshgrid(gx, gy)


# ------------------------------------------------------------------ S0 / fields
def test_normalisation_uniform_unit_square():
    fs = unit_fields()
    for n in (1, 1000, 12345):
        c, havg = O.domain(fs, n)
        assert abs(c - n ** -0.5) <= 4e-16 * n ** -0.5
        assert havg == c


def test_bilinear_exact_for_bilinear_functions():
    X, Y = grid_xy(33)
    F = 0.3 + 1.7 * X - 0.9 * Y + 2.5 * X * Y
    fs = O.FieldSet(BOX, F)
    rng = np.random.default_rng(1)
    for _ in range(200):
        x, y = rng.random(2)
        v = O.field_value(fs, "phi", x, y)
        assert abs(v - (0.3 + 1.7 * x - 0.9 * y + 2.5 * x * y)) < 1e-14
        gx, gy = O.field_grad(fs, "phi", x, y)
        assert abs(gx - (1.7 + 2.5 * y)) < 1e-12 and abs(gy - (-0.9 + 2.5 * x)) < 1e-12


# ------------------------------------------------------------------ O4
def test_centroid_triangle_and_square_uniform():
    fs = unit_fields()
    px, py = np.array([0.1, 0.6, 0.2]), np.array([0.1, 0.2, 0.7])
    cx, cy, _ = O.cvd_polygon(fs, px, py, (0.3, 0.3), 0.1)
    assert abs(cx - px.mean()) < 1e-15 and abs(cy - py.mean()) < 1e-15
    sx, sy = np.array([0.2, 0.8, 0.8, 0.2]), np.array([0.3, 0.3, 0.9, 0.9])
    cx, cy, _ = O.cvd_polygon(fs, sx, sy, (0.5, 0.6), 0.1)
    assert abs(cx - 0.5) < 1e-15 and abs(cy - 0.6) < 1e-15


def test_centroid_linear_density_five_ninths():
    """rho = 1 + x on the unit square: x̄ = (5/6)/(3/2) = 5/9."""
    X, Y = grid_xy(17)
    fs = unit_fields(17, rho=1.0 + X)
    sx, sy = np.array([0.0, 1.0, 1.0, 0.0]), np.array([0.0, 0.0, 1.0, 1.0])
    h = 1.0
    for d_prev, eps in ((1e-9, 0.001), (0.05, 0.05)):
        cx, cy, lv = O.cvd_polygon(fs, sx, sy, (0.5, 0.5), h, d_prev)
        E = 1.0 * eps
        assert abs(cx - 5.0 / 9.0) < E and abs(cy - 0.5) < E
        assert lv >= (3 if eps < 0.01 else 1)
    # tighter tolerance needs at least as many levels
    _, _, lv_tight = O.cvd_polygon(fs, sx, sy, (0.5, 0.5), h, 1e-9)
    _, _, lv_loose = O.cvd_polygon(fs, sx, sy, (0.5, 0.5), h, 0.3)
    assert lv_tight >= lv_loose


def _second_moment(vx, vy):
    """∫_C |x|^2 dA for a polygon given relative to the generator (closed form)."""
    xs, ys = vx, vy
    x1, y1 = np.roll(xs, -1), np.roll(ys, -1)
    cr = xs * y1 - x1 * ys
    return float(np.sum(cr * (xs * xs + xs * x1 + x1 * x1 + ys * ys + ys * y1 + y1 * y1)) / 12.0)


def test_lloyd_energy_monotone_cfg1(cfg_cache):
    """E_CVD = Σ ∫_{V_i} |x - x_i|^2 non-increasing under Lloyd."""
    c = cfg_cache(1)
    fs = O.FieldSet.from_config(c)
    x, y, dp = c.x.copy(), c.y.copy(), None
    E_prev = None
    for it in range(10):
        cl = O.cells(fs, x, y)
        assert not np.any((cl.la >= -8) & (cl.la <= -1))  # octagons never bind (pin premise)
        E = sum(_second_moment(*cl.cell(i)[2:]) for i in range(c.n))
        if E_prev is not None:
            assert E <= E_prev * (1 + 1e-13)
        E_prev = E
        r = O.iteration(fs, x, y, "cvd", d_prev=dp)
        assert r.info.n_degenerate == 0
        x, y, dp = r.x, r.y, r.d_prev
    assert E_prev < 0.9 * sum(_second_moment(*O.cells(fs, c.x, c.y).cell(i)[2:]) for i in range(c.n))


def hex_lattice(m, jitter=0.0, seed=0):
    a = 1.0 / m
    pts = []
    for j in range(int(m / (math.sqrt(3) / 2)) + 1):
        for i in range(m + 1):
            px = (i + 0.5 * (j % 2)) * a
            py = j * a * math.sqrt(3) / 2
            if 0.0 < px < 1.0 and 0.0 < py < 1.0:
                pts.append((px, py))
    P = np.array(pts)
    rng = np.random.default_rng(seed)
    P = P + rng.uniform(-jitter, jitter, P.shape) * a
    return P[:, 0].copy(), P[:, 1].copy(), a


def test_hex_lattice_fixed_point():
    x, y, a = hex_lattice(30, jitter=1e-10)
    fs = unit_fields()
    r = O.iteration(fs, x, y, "cvd")
    interior = (x > 0.2) & (x < 0.8) & (y > 0.2) & (y < 0.8)
    assert np.max(np.hypot(r.x_hat - x, r.y_hat - y)[interior]) < 1e-8 * a
    r = O.iteration(fs, x, y, "dm")
    assert np.max(np.hypot(r.x_hat - x, r.y_hat - y)[interior]) < 1e-8 * a


# ------------------------------------------------------------------ O5
def test_distmesh_identities():
    rng = np.random.default_rng(5)
    n = 400
    x, y = rng.random(n), rng.random(n)
    tri, _ = O.delaunay(x, y)
    e = set()
    for t in tri.tolist():
        for k in range(3):
            a, b = t[k], t[(k + 1) % 3]
            e.add((min(a, b), max(a, b)))
    E = np.array(sorted(e), dtype=np.int32)
    X, Y = grid_xy()
    mu = 1.0 + 0.5 * X
    fs = unit_fields(mu=mu)
    xh, yh, fm = O.distmesh(fs, x, y, E)
    Fx, Fy = xh - x, yh - y
    assert abs(Fx.sum()) < 1e-13 * np.abs(Fx).sum() and abs(Fy.sum()) < 1e-13 * np.abs(Fy).sum()
    # l0 invariant under mu -> 7 mu (fac_mu rescales)
    xh7, yh7, fm7 = O.distmesh(unit_fields(mu=7.0 * mu), x, y, E)
    assert np.max(np.abs(xh7 - xh)) < 1e-14 and np.max(np.abs(yh7 - yh)) < 1e-14
    assert abs(fm7 * 7 - fm) < 1e-14 * fm
    # pure repulsion: with fscale tiny no edge is compressed -> no motion
    xh0, yh0, _ = O.distmesh(fs, x, y, E, params=O.default_params(fscale=0.01))
    assert np.array_equal(xh0, x) and np.array_equal(yh0, y)
    # fixed mask
    fixed = np.zeros(n, np.uint8)
    fixed[::3] = 1
    xf, yf, _ = O.distmesh(fs, x, y, E, fixed=fixed)
    assert np.array_equal(xf[::3], x[::3]) and np.array_equal(xf[1::3], xh[1::3])


def test_distmesh_closed_forms():
    fs = unit_fields()
    # single edge of length l, uniform mu: fac_mu = l, l0 = 1.2 l, f = 0.2 l
    x, y = np.array([0.4, 0.6]), np.array([0.5, 0.5])
    xh, yh, fm = O.distmesh(fs, x, y, np.array([[0, 1]], np.int32))
    l = 0.2
    assert abs(fm - l) < 1e-15
    assert abs(xh[0] - (0.4 - 0.2 * 0.2 * l)) < 1e-15 and abs(xh[1] - (0.6 + 0.2 * 0.2 * l)) < 1e-15
    # equilateral triangle side l: each vertex moves radially by dt*sqrt(3)*(l0-l)
    s = 0.1
    x = np.array([0.5, 0.5 + s, 0.5 + s / 2])
    y = np.array([0.5, 0.5, 0.5 + s * math.sqrt(3) / 2])
    E = np.array([[0, 1], [1, 2], [0, 2]], np.int32)
    xh, yh, _ = O.distmesh(fs, x, y, E)
    gx, gy = x.mean(), y.mean()
    for i in range(3):
        mv = math.hypot(xh[i] - x[i], yh[i] - y[i])
        assert abs(mv - 0.2 * math.sqrt(3) * 0.2 * s) < 1e-14
        # radial: displacement parallel to (p - g)
        assert abs((xh[i] - x[i]) * (y[i] - gy) - (yh[i] - y[i]) * (x[i] - gx)) < 1e-15


# ------------------------------------------------------------------ O6
def test_treat_linear_sdf_one_newton_step():
    X, Y = grid_xy(21)
    fs = O.FieldSet(BOX, X - 0.5)
    c, havg = O.domain(fs, 1)
    (qx, qy), dp, st = O.treat(fs, c, havg, (0.45, 0.5), (0.6, 0.5))
    assert st == 1 and abs(qx - 0.5) < 1e-15 and qy == 0.5
    assert abs(O.field_value(fs, "phi", qx, qy)) < 1e-15
    assert abs(dp - 0.05) < 1e-15


def test_treat_disk_projection():
    box = (-1.1, -1.1, 1.1, 1.1)
    fs = O.FieldSet(box, configs.disk_phi(box, 512))
    n = 100000
    c, havg = O.domain(fs, n)
    geps = 0.01 * min(c, havg)
    for ang in np.linspace(0, 2 * np.pi, 37):
        old = (0.999 * math.cos(ang), 0.999 * math.sin(ang))
        new = (1.001 * math.cos(ang), 1.001 * math.sin(ang))
        (qx, qy), dp, st = O.treat(fs, c, havg, old, new)
        assert st == 1
        assert abs(math.hypot(qx, qy) - 1.0) < 2e-5
        assert abs(O.field_value(fs, "phi", qx, qy)) <= geps


def test_treat_clamp_idempotent_fallback():
    fs = unit_fields()
    c, havg = O.domain(fs, 100)  # h = 0.1, T = 0.04
    (qx, qy), dp, st = O.treat(fs, c, havg, (0.5, 0.5), (0.7, 0.5))
    assert st == 4 and abs(qx - 0.54) < 1e-15 and abs(dp - 0.04) < 1e-15
    (q2x, q2y), dp2, st2 = O.treat(fs, c, havg, (qx, qy), (qx, qy))
    assert (q2x, q2y) == (qx, qy) and dp2 == 0.0 and st2 == 0
    # constant positive phi: Newton has no gradient -> fallback to p_old
    fs2 = O.FieldSet(BOX, np.full((8, 8), 0.3))
    (qx, qy), dp, st = O.treat(fs2, c, havg, (0.5, 0.5), (0.51, 0.5))
    assert st == 2 and (qx, qy) == (0.5, 0.5) and dp == 0.0


# ------------------------------------------------------------------ O7
def test_quality_worked_examples():
    al, be = O.triangle_quality((0, 0), (1, 0), (0.5, math.sqrt(3) / 2))
    assert abs(al - 1) < 1e-12 and abs(be - 1) < 1e-12
    al, be = O.triangle_quality((0, 0), (4, 0), (0, 3))  # 3-4-5
    assert abs(al - 1.25) < 1e-14 and abs(be - 5 / 3) < 1e-14
    al, be = O.triangle_quality((0, 0), (1, 0), (0, 1))  # isosceles right
    assert abs(al - (1 + math.sqrt(2)) / 2) < 1e-14
    tri = np.array([[0, 1, 2], [3, 4, 5]], np.int32)
    x = np.array([0, 1, 0.5, 0, 4, 0.0])
    y = np.array([0, 0, math.sqrt(3) / 2, 0, 0, 3.0])
    s = O.stats(tri, x, y)
    assert s[0] == 2 and abs(s[3] - 1.25) < 1e-14 and s[9] == 1 and s[10] == 2
    # 1/2-mean (Eq. 1/2 mean): ((1 + sqrt(1.25))/2)^2, and M_1/2 <= arithmetic mean
    assert abs(s[11] - ((1 + math.sqrt(1.25)) / 2) ** 2) < 1e-14
    assert s[11] <= s[5] / s[0]


def test_decision_margins_generic_inputs():
    """SURVEY §8(c) parity protocol: the oracle reports the floating decisions that fall
    within 1e-13 of their threshold (keep-rule box/octagon/phi tests, quadrature stop,
    treatment accept, Newton stop).  For the generic seeded inputs the report is empty
    (a non-empty one would explain, not excuse, a GPU/oracle mismatch)."""
    import oracle as O
    from inputs import configs
    c = configs.load(1)
    fs = O.FieldSet.from_config(c)
    x, y, dp = c.x, c.y, None
    for it in range(3):
        o = O.iteration(fs, x, y, "cvd", d_prev=dp)
        assert o.info.n_near_ties == 0 and o.info.n_degenerate == 0
        x, y, dp = o.x, o.y, o.d_prev
    o = O.iteration(fs, x, y, "dm", d_prev=dp)
    assert o.info.n_near_ties == 0
