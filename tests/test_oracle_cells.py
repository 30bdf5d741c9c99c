"""Pins for O2 (bounded cells C_i = B ∩ Oct_i ∩ Vor(i), PAPER.md P:100,
P:491 with the L6 octagon reading) and O3 (keep rule)."""
import math

import numpy as np
import pytest

import oracle as O
from inputs import configs


def unit_fields(n=64, box=(0.0, 0.0, 1.0, 1.0)):
    return O.FieldSet(box, configs.box_phi(box, n))


def poly_area(vx, vy):
    return 0.5 * float(np.sum(vx * np.roll(vy, -1) - np.roll(vx, -1) * vy))


# ---------------------------------------------------------------- brute force
def octagon(px, py, S):
    ang = np.deg2rad(22.5 + 45.0 * np.arange(8))
    return [(px + S * math.cos(a), py + S * math.sin(a)) for a in ang]


def clip(poly, a, b, c):
    """keep a*x + b*y <= c (float Sutherland-Hodgman, unlabelled)"""
    out = []
    n = len(poly)
    for k in range(n):
        P, Q = poly[k], poly[(k + 1) % n]
        fp, fq = a * P[0] + b * P[1] - c, a * Q[0] + b * Q[1] - c
        if fp <= 0:
            out.append(P)
        if (fp < 0 < fq) or (fq < 0 < fp):
            t = fp / (fp - fq)
            out.append((P[0] + t * (Q[0] - P[0]), P[1] + t * (Q[1] - P[1])))
    return out


def brute_cell(i, x, y, S, box):
    poly = octagon(x[i], y[i], S[i])
    x0, y0, x1, y1 = box
    for (a, b, c) in ((1, 0, x1), (0, 1, y1), (-1, 0, -x0), (0, -1, -y0)):
        poly = clip(poly, a, b, c)
    for j in range(len(x)):
        if j == i:
            continue
        dx, dy = x[j] - x[i], y[j] - y[i]
        # |q-p_i|^2 <= |q-p_j|^2  <=>  dx*qx + dy*qy <= (|p_j|^2-|p_i|^2)/2
        poly = clip(poly, dx, dy, 0.5 * ((x[j] ** 2 + y[j] ** 2) - (x[i] ** 2 + y[i] ** 2)))
    return poly


@pytest.mark.parametrize("n,fac", [(300, 5.0), (300, 1.0), (150, 0.6)])
def test_all_pairs_bruteforce(n, fac):
    """Every oracle cell equals the O(N^2) all-pairs clipping of the same
    octagon ∩ box (SPEC acceptance #1 idea; octagon built from trig here)."""
    rng = np.random.default_rng(n + int(10 * fac))
    x, y = rng.random(n), rng.random(n)
    fs = unit_fields()
    p = O.default_params(fac_voro_bound=fac)
    cl = O.cells(fs, x, y, p)
    c, _ = O.domain(fs, n)
    S = np.full(n, fac * c)
    for i in range(n):
        la, lb, vx, vy = cl.cell(i)
        bp = brute_cell(i, x, y, S, (0, 0, 1, 1))
        # drop near-duplicate brute-force vertices (clip through an existing vertex)
        uniq = []
        for q in bp:
            if not uniq or math.dist(q, uniq[-1]) > 1e-13:
                uniq.append(q)
        if len(uniq) > 1 and math.dist(uniq[0], uniq[-1]) <= 1e-13:
            uniq.pop()
        assert len(uniq) == len(vx), i
        ov = list(zip((x[i] + vx).tolist(), (y[i] + vy).tolist()))
        for q in ov:  # every oracle vertex has a brute-force partner (bijection by count)
            assert min(math.dist(q, b) for b in uniq) < 1e-11


def test_area_sum_cfg1_no_octagon(cfg_cache):
    """Σ A(C_i) = A(B) when no octagon wall survives (SURVEY §8(c) O2 pin ii)."""
    c = cfg_cache(1)
    cl = O.cells(O.FieldSet.from_config(c), c.x, c.y)
    assert not np.any((cl.la >= -8) & (cl.la <= -1))
    tot = sum(poly_area(*cl.cell(i)[2:]) for i in range(c.n))
    assert abs(tot - 1.0) < 1e-13
    assert cl.info.n_degenerate == 0


def test_closed_forms():
    fs = unit_fields()
    # one point, octagon much larger than the box: cell = box (c = 1, S = 5)
    cl = O.cells(fs, [0.5], [0.5])
    la, lb, vx, vy = cl.cell(0)
    assert len(vx) == 4 and abs(poly_area(vx, vy) - 1.0) < 1e-15
    # one point, small octagon inside the box: regular octagon, area 2*sqrt(2)*S^2
    p = O.default_params(fac_voro_bound=0.2)
    cl = O.cells(fs, [0.5], [0.5], p)
    la, lb, vx, vy = cl.cell(0)
    assert len(vx) == 8 and set(la.tolist()) == set(range(-8, 0))
    assert abs(poly_area(vx, vy) - 2 * math.sqrt(2) * 0.2 ** 2) < 1e-15
    # two points (0.25,0.5),(0.75,0.5): shared edge x=0.5, areas 0.5 each
    cl = O.cells(fs, [0.25, 0.75], [0.5, 0.5])
    for i in range(2):
        la, lb, vx, vy = cl.cell(i)
        assert abs(poly_area(vx, vy) - 0.5) < 1e-15
        assert (1 - i) in la.tolist()


def test_jittered_lattice_areas():
    m = 20
    a = 1.0 / m
    rng = np.random.default_rng(3)
    g = (np.arange(m) + 0.5) * a
    X, Y = np.meshgrid(g, g)
    x = X.ravel() + rng.uniform(-1e-9, 1e-9, m * m) * a
    y = Y.ravel() + rng.uniform(-1e-9, 1e-9, m * m) * a
    cl = O.cells(unit_fields(), x, y)
    areas = np.array([poly_area(*cl.cell(i)[2:]) for i in range(m * m)])
    assert np.all(np.abs(areas - a * a) < 1e-8 * a * a)


def test_equidistance_and_duality():
    n = 2000
    rng = np.random.default_rng(9)
    x, y = rng.random(n), rng.random(n)
    fs = unit_fields()
    p = O.default_params(fac_voro_bound=1.2)  # octagons bind on many cells
    cl = O.cells(fs, x, y, p)
    c, _ = O.domain(fs, n)
    r = 1.2 * c * math.cos(math.pi / 8)
    tri, _ = O.delaunay(x, y)
    inc = {}
    for t in tri.tolist():
        for v in t:
            inc.setdefault(v, []).append(t)
    n_oct = 0
    for i in range(n):
        la, lb, vx, vy = cl.cell(i)
        n_oct += int(np.any((la >= -8) & (la <= -1)))
        pp = set()
        for k in range(len(vx)):
            if la[k] >= 0 and lb[k] >= 0:
                q = (x[i] + vx[k], y[i] + vy[k])
                d0 = math.dist(q, (x[i], y[i]))
                for j in (la[k], lb[k]):
                    assert abs(math.dist(q, (x[j], y[j])) - d0) <= 1e-12 * max(d0, 1e-300) + 1e-15
                pp.add(frozenset((i, int(la[k]), int(lb[k]))))
        # duality: triangles of D at i whose circumcentre is strictly inside B ∩ Oct_i
        exp = set()
        for t in inc.get(i, []):
            (ax, ay), (bx, by), (qx, qy) = [(x[v], y[v]) for v in t]
            d = 2 * ((bx - ax) * (qy - ay) - (by - ay) * (qx - ax))
            l1 = (bx - ax) ** 2 + (by - ay) ** 2
            l2 = (qx - ax) ** 2 + (qy - ay) ** 2
            cx = ax + ((qy - ay) * l1 - (by - ay) * l2) / d
            cy = ay + ((bx - ax) * l2 - (qx - ax) * l1) / d
            dx, dy = cx - x[i], cy - y[i]
            inside = (0 < cx < 1 and 0 < cy < 1 and abs(dx) < r and abs(dy) < r
                      and abs(dx + dy) < math.sqrt(2) * r and abs(dx - dy) < math.sqrt(2) * r)
            if inside:
                exp.add(frozenset(t))
        assert pp == exp, i
    assert n_oct > 100
