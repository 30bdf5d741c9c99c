"""Pins added in round 2 for oracle functions that no earlier test distinguished
from a plausible mistake (VERDICT r1 "What's weak" #2):

* ``or_domain``'s h_avg under a non-uniform sizing field (§8.0 "Local size",
  P:442 §3.7): closed forms on a half-plane shape and the survey's
  independently computed values for cfg3/cfg4;
* the adaptive-quadrature stop threshold E = sqrt(A) * max(d_prev/h, fac_end)
  (§4.2(2), reading L13) at h != 1;
* the DistMesh sizing evaluation point (reading L2: mu at the edge midpoint,
  P:149-153 Eq. size scaling);
* the Table B.1 defaults in both the oracle and the library.
"""
import ctypes
import json
import math
import os

import numpy as np
import pytest

import oracle as O
from inputs import configs

GOLD = os.path.join(os.path.dirname(__file__), "golden")
BOX = (0.0, 0.0, 1.0, 1.0)


def _grid(n, box=BOX):
    gx = configs.node_coords(box[0], box[2], n)
    gy = configs.node_coords(box[1], box[3], n)
    return np.meshgrid(gx, gy)


# ------------------------------------------------------------------ S0: c and h_avg
def test_domain_half_plane_linear_sizing_closed_form():
    """phi = x - 1/2 (inside: x < 1/2), mu = 1 + x on the unit square.
    c^2 N = ∫_{x<1/2} (1+x)^-2 dA = 1 - 1/1.5 = 1/3 and the mean of mu over the inside
    cells is 1.25, so h_avg = 1.25 c (h_i = sqrt(dx dy / n_i^E), n^E = rho^norm N
    with rho = mu^-2; h_avg = the mean of h over the inside cells).
    Mistakes this catches: mu^-1 instead of mu^-2 (c off by 18 %), outside cells in the
    mean (h_avg = 1.5 c), mean of 1/mu or of mu^-2 (h_avg != 1.25 c), cell count vs
    point count in the normalisation."""
    n = 1025
    X, Y = _grid(n)
    fs = O.FieldSet(BOX, X - 0.5, 1.0 + X)
    for N in (1, 1000, 10**6):
        c, havg = O.domain(fs, N)
        # midpoint rule on (1+x)^-2 over 512 columns of width 1/1024: error ~ dx^2/24 * 1.2
        assert abs(c * c * N - 1.0 / 3.0) < 2e-7, c * c * N
        assert abs(havg / c - 1.25) < 1e-12, havg / c


def test_domain_hole_excluded_from_h_avg():
    """An inside region with constant mu = 2 next to an outside region with mu = 1:
    only the inside cells count, so h_avg = 2c and c^2 N = area * 2^-2."""
    n = 513
    X, Y = _grid(n)
    phi = np.where(Y <= 0.25, -1.0, 1.0)  # inside: the 128 of 512 cell rows below y = 1/4
    mu = np.where(Y < 0.5, 2.0, 1.0)
    fs = O.FieldSet(BOX, phi, mu)
    c, havg = O.domain(fs, 100)
    assert abs(c * c * 100 - 0.25 / 4.0) < 1e-15
    assert abs(havg - 2.0 * c) < 1e-15


@pytest.mark.parametrize("k", [3, 4])
def test_domain_h_avg_matches_survey(k, cfg_cache):
    """SURVEY §8(c) 'Iteration-0 reference counts' (computed with numpy, independently of
    oracle/): c to 6 and h_avg to 4 significant digits, as printed."""
    gold = json.load(open(os.path.join(GOLD, "iter0_counts.json")))[f"cfg{k}"]
    c = cfg_cache(k)
    cc, havg = O.domain(O.FieldSet.from_config(c), c.n)
    assert abs(cc - gold["c"]) <= 0.5e-6 * 1.0001, (cc, gold["c"])
    assert abs(havg - gold["h_avg"]) <= 0.5e-6 * 1.0001, (havg, gold["h_avg"])


# ------------------------------------------------------------------ O4: quadrature stop
def _quad_setup():
    n = 65
    X, Y = _grid(n)
    rho = 1.0 + 20.0 * X * Y + 5.0 * X * X
    fs = O.FieldSet(BOX, configs.box_phi(BOX, n), None, rho)
    ang = np.arange(6) * (np.pi / 3) + 0.1
    px = 0.5 + 0.3 * np.cos(ang)
    py = 0.5 + 0.3 * np.sin(ang)
    return fs, px, py


def test_quadrature_level_nondecreasing_in_h():
    """E = sqrt(A) max(d_prev/h, fac_end): at fixed d_prev a larger local size
    h means a smaller tolerance, so the returned level can only grow with h.  A threshold
    written d_prev*h (or one ignoring h) fails this: it would shrink (or not move)."""
    fs, px, py = _quad_setup()
    d_prev = 2e-3
    hs = np.logspace(-3, 1, 25)
    lv = [O.cvd_polygon(fs, px, py, (0.5, 0.5), h, d_prev)[2] for h in hs]
    assert all(a <= b for a, b in zip(lv, lv[1:])), lv
    assert lv[-1] - lv[0] >= 2, lv  # the sweep crosses several levels
    # beyond h = d_prev / fac_end the floor fac_end = 0.001 binds: the level stops changing
    assert lv[-1] == O.cvd_polygon(fs, px, py, (0.5, 0.5), 1e3, d_prev)[2]


def test_quadrature_depends_on_ratio_d_prev_over_h():
    """Only d_prev/h enters: scaling both by the same factor keeps the level and
    the centroid; scaling d_prev alone changes the level."""
    fs, px, py = _quad_setup()
    base = O.cvd_polygon(fs, px, py, (0.5, 0.5), 0.01, 1e-4)
    for k in (0.25, 2.0, 8.0):
        r = O.cvd_polygon(fs, px, py, (0.5, 0.5), 0.01 * k, 1e-4 * k)
        assert r[2] == base[2] and abs(r[0] - base[0]) < 1e-15 and abs(r[1] - base[1]) < 1e-15
    loose = O.cvd_polygon(fs, px, py, (0.5, 0.5), 0.01, 1e-2)
    assert loose[2] < base[2]


# ------------------------------------------------------------------ O5: sizing at the edge midpoint
def test_distmesh_sizing_at_edge_midpoint():
    """Collinear chain p0 = 0.1, p1 = 0.3, p2 = 0.7 (y = 1/2), edges (0,1), (1,2), mu = 1 + x
    (exactly bilinear).  Reading L2 evaluates mu at the midpoints 0.2 and 0.5: mu = 1.2, 1.5.
    Hand derivation:
        fac_mu = sqrt((0.2^2 + 0.4^2) / (1.2^2 + 1.5^2)) = sqrt(0.2 / 3.69)
        l0_01 = 1.2 * 1.2 * fac_mu,  l0_12 = 1.5 * 1.2 * fac_mu  (both edges compressed)
        x0' = 0.1 - 0.2 (l0_01 - 0.2),  x1' = 0.3 + 0.2 (l0_01 - 0.2) - 0.2 (l0_12 - 0.4),
        x2' = 0.7 + 0.2 (l0_12 - 0.4).
    mu at an endpoint (x_a or x_b) or at the mean of the two mu values gives other numbers."""
    n = 33
    X, Y = _grid(n)
    fs = O.FieldSet(BOX, configs.box_phi(BOX, n), 1.0 + X)
    x = np.array([0.1, 0.3, 0.7])
    y = np.array([0.5, 0.5, 0.5])
    E = np.array([[0, 1], [1, 2]], np.int32)
    xh, yh, fm = O.distmesh(fs, x, y, E)
    fac_mu = math.sqrt(0.2 / 3.69)
    l0a, l0b = 1.44 * fac_mu, 1.8 * fac_mu
    assert abs(fm - fac_mu) < 1e-15
    want = [0.1 - 0.2 * (l0a - 0.2), 0.3 + 0.2 * (l0a - 0.2) - 0.2 * (l0b - 0.4), 0.7 + 0.2 * (l0b - 0.4)]
    assert np.max(np.abs(xh - np.array(want))) < 1e-15, (xh, want)
    assert np.array_equal(yh, y)


# ------------------------------------------------------------------ Table B.1 defaults
TABLE_FIELDS = ["fac_voro_bound", "fac_pt_mvmt", "fac_geps", "fac_end_mvmt", "newton_damping", "newton_max",
                "fscale"]


def test_oracle_defaults_are_table_b1():
    tb = json.load(open(os.path.join(GOLD, "table_b1.json")))
    p = O.default_params()
    for k in TABLE_FIELDS:
        assert getattr(p, k) == tb[k]["value"], k
    # readings where the paper is silent (SURVEY §8(c) ledger)
    assert p.dt_k == 0.2 and p.keep_tol == 0.0 and p.quad_max_level == 10  # L3, L10, L13
    assert p.t_circ == tb["t_tria_ccircum"]["value"] and p.fac_retria == tb["fac_retria_mvmt"]["value"]
    cp = O.ControlParams()
    for k in ["t_add_quality", "fac_add", "t_end_quality", "t_end_alpha_max", "t_switch_quality"]:
        assert getattr(cp, k) == tb[k]["value"], k


def test_library_defaults_are_table_b1():
    """tm_params_default (host function of libtrime_gpu.so; no GPU needed)."""
    import paper_2309_13824_b200 as T
    tb = json.load(open(os.path.join(GOLD, "table_b1.json")))
    p = T.tm_params()
    T.load_library().tm_params_default(ctypes.byref(p))
    for k in TABLE_FIELDS:
        assert getattr(p, k) == tb[k]["value"], k
    assert p.dt_k == 0.2 and p.keep_tol == 0.0 and p.quad_max_level == 10
    # documented deviation: the cell list holds 6 points per leaf, not the
    # paper's N_opt = 3.3 (tuned for Voro++ on CPUs); binning changes only the search (L24)
    assert tb["n_opt"]["value"] == 3.3 and p.n_opt == 6.0
