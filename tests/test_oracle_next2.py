"""Pins for the NEXT-2 / NEXT-3 oracle pieces: the paper's triangle validity
Tests 1-3 (§4.1; T^tria = 0.4), the movement-termination count (P:484-485,
P:447), the iterate-to-termination controller (thresholds P:1091-1121)
and the point-addition scheme.  Every expected value is derived by hand or by an
independent formula in this file, not by re-calling the oracle's own routine."""
import math

import numpy as np

import oracle as O
from inputs import configs

# phi = x on integer nodes of [-20, 20]^2 (exactly bilinear); mu = 1, c = h_avg = 10 =>
# geps = 0.01 * min(h, h_avg) = 0.1, octagons of circumradius 50 (never binding here)
BOX = (-20.0, -20.0, 20.0, 20.0)
GX = configs.node_coords(BOX[0], BOX[2], 41)
X, Y = np.meshgrid(GX, GX)
FS = O.FieldSet(BOX, X.copy())
C = H_AVG = 10.0
PAPER = O.default_params(validity=1)
TEST1 = O.default_params(validity=0)


def _keep(pts, params):
    x = np.array([p[0] for p in pts], dtype=np.float64)
    y = np.array([p[1] for p in pts], dtype=np.float64)
    return O.keep_triangle(FS, C, H_AVG, x, y, (0, 1, 2), params=params)


def test_test1_discards_centroid_beyond_geps():
    """Centroid x = 0.2 > geps = 0.1: discarded by Test 1 in both readings."""
    pts = [(-1.0, 0.0), (0.3, 1.0), (1.3, -1.0)]
    assert not _keep(pts, PAPER)
    assert not _keep(pts, TEST1)


def test_test1_tolerance_and_test2_midpoints():
    """Centroid x = 0.05 (outside, within geps): Test 1 passes; midpoints x = -0.45 (in), 0.575 (out),
    0.025 (<= geps, counted) => count 2, kept.  The L10 reading (phi~(g) < 0) discards it."""
    pts = [(-1.0, 0.0), (0.1, 1.0), (1.05, -1.0)]
    assert _keep(pts, PAPER)
    assert not _keep(pts, TEST1)


def test_test3_keeps_small_circumcentre_ratio():
    """a = (-2,0), b = (-2,2), c = (3,1): g.x = -1/3 (in); midpoints x = -2 (in), 0.5, 0.5 (out) =>
    count 1, Test 3.  Circumcentre (0.4, 1) by (cx+2)^2 + 1 = (3-cx)^2, R = 2.6: |phi|/R = 0.154 <= 0.4."""
    pts = [(-2.0, 0.0), (-2.0, 2.0), (3.0, 1.0)]
    assert _keep(pts, PAPER)


def test_test3_discards_large_circumcentre_ratio():
    """a = (-2,0), b = (-2,12), c = (3,6): count 1 (midpoints x = -2 in, 0.5, 0.5 out).  Circumcentre
    x = 0.5 - 12^2/40 = -3.1, R = 6.1: |phi|/R = 0.508 > 0.4 => discarded (the circumcentre lies
    INSIDE: a signed ratio would keep it; a diameter for R would give 0.254 and keep it).  Test 1
    alone keeps it (phi~(g) = -1/3)."""
    pts = [(-2.0, 0.0), (-2.0, 12.0), (3.0, 6.0)]
    assert not _keep(pts, PAPER)
    assert _keep(pts, TEST1)


def test_validity_tests_invariant_to_vertex_order():
    pts = [(-2.0, 0.0), (-2.0, 12.0), (3.0, 6.0)]
    x = np.array([p[0] for p in pts]); y = np.array([p[1] for p in pts])
    res = {O.keep_triangle(FS, C, H_AVG, x, y, t, params=PAPER) for t in [(0, 1, 2), (2, 1, 0), (1, 2, 0)]}
    assert res == {False}


def test_move_count_classifies_inner_points_and_threshold():
    """phi = x: inner iff x < -geps = -0.1; threshold fac_end * h = 0.001 * 10 = 0.01."""
    xo = np.array([-5.0, -5.0, -5.0, -0.05, 0.05, -0.2])
    yo = np.zeros(6)
    dp = np.array([0.009, 0.01, 0.5, 0.5, 0.5, 0.011])
    # -5 / 0.009: below; -5 / 0.01: not below (counted); -5 / 0.5 counted; -0.05, 0.05: boundary
    # (|phi| <= geps), not inner; -0.2 / 0.011 counted
    assert O.move_count(FS, C, H_AVG, xo, yo, dp) == 3


def _circumradius(a, b, c):
    la, lb, lc = math.dist(b, c), math.dist(a, c), math.dist(a, b)
    area = abs((b[0] - a[0]) * (c[1] - a[1]) - (b[1] - a[1]) * (c[0] - a[0])) / 2
    return la * lb * lc / (4 * area)


def test_point_addition_ranks_by_circumradius_over_h():
    """Jittered points in the unit square, Delaunay triangles, uniform h = c: the selected set is the
    top-k by R = abc/(4A) (closed form, not the Cramer circumcentre), centroids in (u, v) order."""
    rng = np.random.default_rng(5)
    box = (0.0, 0.0, 1.0, 1.0)
    g = configs.node_coords(0, 1, 9)
    GXs, GYs = np.meshgrid(g, g)
    fs = O.FieldSet(box, np.maximum.reduce([-GXs, GXs - 1, -GYs, GYs - 1]))
    x = rng.uniform(0.05, 0.95, 300)
    y = rng.uniform(0.05, 0.95, 300)
    tri, _ = O.delaunay(x, y)
    c = 0.05
    k = 37
    xn, yn, rmin = O.point_addition(fs, c, tri, x, y, k)
    ratios = []
    for t in tri:
        u, v, w = sorted(int(q) for q in t)
        ratios.append((_circumradius((x[u], y[u]), (x[v], y[v]), (x[w], y[w])) / c, u, v, w))
    ratios.sort(key=lambda r: -r[0])
    assert ratios[k - 1][0] - ratios[k][0] > 1e-9 * ratios[k][0]  # no near tie at the cut
    assert abs(rmin - ratios[k - 1][0]) <= 1e-12 * rmin
    sel = sorted(ratios[:k], key=lambda r: (r[1], r[2]))
    ex = np.array([(x[u] + x[v] + x[w]) / 3 for _, u, v, w in sel])
    ey = np.array([(y[u] + y[v] + y[w]) / 3 for _, u, v, w in sel])
    assert len(xn) == k
    np.testing.assert_allclose(xn, ex, rtol=0, atol=1e-15)
    np.testing.assert_allclose(yn, ey, rtol=0, atol=1e-15)


def test_point_addition_uses_local_h():
    """Two congruent triangles, h twice as large on the right half (mu = 1 + x on [0, 1]): the left
    one (smaller h) ranks first."""
    box = (0.0, 0.0, 1.0, 1.0)
    g = configs.node_coords(0, 1, 3)
    GXs, GYs = np.meshgrid(g, g)
    fs = O.FieldSet(box, GXs - 2.0, mu=1.0 + GXs)
    x = np.array([0.1, 0.2, 0.15, 0.8, 0.9, 0.85])
    y = np.array([0.1, 0.1, 0.2, 0.1, 0.1, 0.2])
    tri = np.array([[3, 4, 5], [0, 1, 2]], dtype=np.int32)
    xn, yn, _ = O.point_addition(fs, 1.0, tri, x, y, 1)
    assert abs(xn[0] - 0.15) < 1e-15 and abs(yn[0] - (0.4 / 3)) < 1e-15


def test_controller_point_addition_schedule_of_the_worked_example():
    """P:436 (Fig. pt_addition): N_total = 5000, fac_init = 0.2 => 1000 initial points, the first
    addition adds fac_add * 1000 = 600.  Continuing the rule N_add = min(0.6 N, N_total - N):
    +960 (2560), +1536 (4096), +904 (5000)."""
    ctl = O.Controller(5000, 1000, method="cvd")
    adds = []
    q = (1.1, 1.3, 3.0)
    for it in range(40):
        d = ctl.update(*q, move_count=10)
        if d["action"] == "add":
            adds.append(d["n_add"])
    assert adds == [600, 960, 1536, 904]
    assert ctl.n_current == 5000


def test_controller_thresholds():
    """Relative changes against the Table B.1 thresholds, hand-computed."""
    # addition needs BOTH 1/2-means below 0.002
    ctl = O.Controller(100, 50, method="cvd")
    assert ctl.update(1.0, 1.0, 2.0, 5)["action"] == "continue"          # no history
    assert ctl.update(1.0019, 1.0025, 2.0, 5)["action"] == "continue"    # beta changed 0.25 %
    assert ctl.update(1.0019 * 1.001, 1.0025 * 1.001, 2.0, 5)["action"] == "add"
    # hybrid switch: alpha's 1/2-mean below 0.0015 only
    h = O.Controller(10, 10, method="hybrid")
    assert h.update(1.2, 1.5, 9.0, 5)["action"] == "continue"
    assert h.update(1.2 * 1.0016, 1.5, 9.0, 5)["action"] == "continue"
    assert h.update(1.2 * 1.0016 * 1.0014, 1.5 * 1.1, 9.0, 5)["action"] == "switch"
    assert h.mode == "cvd"
    # termination on quality: both 1/2-means below 0.001 AND max alpha below 0.005
    t = O.Controller(10, 10, method="cvd")
    t.update(1.05, 1.3, 4.0, 5)
    assert t.update(1.05 * 1.0009, 1.3 * 0.9991, 4.0 * 1.006, 5)["action"] == "continue"
    assert t.update(1.05 * 1.0009 * 1.0009, 1.3 * 0.9991, 4.0 * 1.006 * 0.996, 5)["reason"] == "quality"
    # termination on movement: no inner point moved by fac_end * h or more
    m = O.Controller(10, 10, method="cvd")
    assert m.update(1.05, 1.3, 4.0, 0)["reason"] == "movement"
    # hybrid: movement is not a termination test before the switch
    hm = O.Controller(10, 10, method="hybrid")
    assert hm.update(1.05, 1.3, 4.0, 0)["action"] == "continue"
