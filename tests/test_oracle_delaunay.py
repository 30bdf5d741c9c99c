"""Pins for O1 (Delaunay D by Bowyer-Watson), PAPER.md P:43 (unique
triangulation with empty circumcircles for points in general position)."""
import itertools
import json
import os
from fractions import Fraction as Fr

import numpy as np
import pytest

import oracle as O
from tests.test_oracle_predicates import incircle_fr, orient_fr


def _incircle_exactish(a, b, c, d):
    """float evaluation with a very loose error bound, Fraction fallback."""
    adx, ady = a[0] - d[0], a[1] - d[1]
    bdx, bdy = b[0] - d[0], b[1] - d[1]
    cdx, cdy = c[0] - d[0], c[1] - d[1]
    al, bl, cl = adx * adx + ady * ady, bdx * bdx + bdy * bdy, cdx * cdx + cdy * cdy
    det = al * (bdx * cdy - cdx * bdy) + bl * (cdx * ady - adx * cdy) + cl * (adx * bdy - bdx * ady)
    perm = al * (abs(bdx * cdy) + abs(cdx * bdy)) + bl * (abs(cdx * ady) + abs(adx * cdy)) + \
        cl * (abs(adx * bdy) + abs(bdx * ady))
    if abs(det) > 1e-12 * perm:
        return 1 if det > 0 else -1
    return incircle_fr(a, b, c, d)


def brute_force_delaunay(P):
    """O(n^4) enumeration: CCW triples whose circumcircle is empty."""
    n = len(P)
    out = set()
    for i, j, k in itertools.combinations(range(n), 3):
        o = orient_fr(P[i], P[j], P[k])
        if o == 0:
            continue
        a, b, c = (i, j, k) if o > 0 else (i, k, j)
        if all(_incircle_exactish(P[a], P[b], P[c], P[m]) <= 0 for m in range(n) if m not in (i, j, k)):
            out.add(tuple(sorted((i, j, k))))
    return out


@pytest.mark.parametrize("seed", range(12))
def test_brute_force_small(seed):
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(3, 26))
    x, y = rng.random(n), rng.random(n)
    P = list(zip(x.tolist(), y.tolist()))
    tri, nd = O.delaunay(x, y)
    assert nd == 0
    assert set(tuple(sorted(t)) for t in tri.tolist()) == brute_force_delaunay(P)
    for t in tri.tolist():
        assert t[0] == min(t)
        assert orient_fr(P[t[0]], P[t[1]], P[t[2]]) > 0


def hull_size_exact(P):
    """Andrew's monotone chain with exact orientation; strict hull vertices."""
    pts = sorted(set(P))
    def cross(o, a, b):
        return orient_fr(o, a, b)
    lower, upper = [], []
    for p in pts:
        while len(lower) >= 2 and cross(lower[-2], lower[-1], p) <= 0:
            lower.pop()
        lower.append(p)
    for p in reversed(pts):
        while len(upper) >= 2 and cross(upper[-2], upper[-1], p) <= 0:
            upper.pop()
        upper.append(p)
    return len(lower) + len(upper) - 2


@pytest.mark.parametrize("n,seed", [(200, 1), (2000, 2), (5000, 3)])
def test_euler(n, seed):
    rng = np.random.default_rng(seed)
    x, y = rng.random(n), rng.random(n)
    tri, _ = O.delaunay(x, y)
    h = hull_size_exact(list(zip(x.tolist(), y.tolist())))
    assert len(tri) == 2 * n - h - 2


def local_delaunay_certificate(x, y, tri):
    """Every triangle CCW; every interior edge locally Delaunay against the
    opposite vertex (exact on near-ties); triangle areas sum to the hull area.
    By the local-Delaunay lemma this certifies D."""
    T = tri.astype(np.int64)
    ax, ay = x[T[:, 0]], y[T[:, 0]]
    bx, by = x[T[:, 1]], y[T[:, 1]]
    cx, cy = x[T[:, 2]], y[T[:, 2]]
    cr = (bx - ax) * (cy - ay) - (by - ay) * (cx - ax)
    assert np.all(cr > 0)
    # edges -> (triangle, opposite vertex)
    e = {}
    for t, (a, b, c) in enumerate(T.tolist()):
        for (u, w, o) in ((a, b, c), (b, c, a), (c, a, b)):
            e[(u, w)] = o
    bad = 0
    for (u, w), o in e.items():
        if (w, u) in e and u < w:
            o2 = e[(w, u)]
            P = lambda i: (float(x[i]), float(y[i]))
            # triangle (u, w, o) is CCW; the opposite vertex o2 must not be inside
            if _incircle_exactish(P(u), P(w), P(o), P(o2)) > 0:
                bad += 1
    assert bad == 0
    # hull area by exact-ish shoelace of the boundary edges
    bnd = [(u, w) for (u, w) in e if (w, u) not in e]
    hull_area = sum(x[u] * y[w] - x[w] * y[u] for u, w in bnd) / 2.0
    assert abs(cr.sum() / 2.0 - hull_area) <= 1e-12 * abs(hull_area)


@pytest.mark.parametrize("n", [1000, 20000])
def test_local_certificate(n):
    rng = np.random.default_rng(n)
    x, y = rng.random(n), rng.random(n)
    tri, _ = O.delaunay(x, y)
    local_delaunay_certificate(x, y, tri)


def test_local_certificate_cfg2(cfg_cache):
    c = cfg_cache(2)
    tri, nd = O.delaunay(c.x, c.y)
    assert nd == 0
    local_delaunay_certificate(c.x, c.y, tri)


def test_qhull_crosscheck():
    from scipy.spatial import Delaunay
    rng = np.random.default_rng(77)
    x, y = rng.random(30000) * 2 - 1, rng.random(30000) * 2 - 1
    tri, _ = O.delaunay(x, y)
    q = Delaunay(np.c_[x, y]).simplices
    assert set(map(tuple, np.sort(tri, 1).tolist())) == set(map(tuple, np.sort(q, 1).tolist()))


def test_iter0_counts_cfg1_cfg2(cfg_cache):
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "iter0_counts.json")))
    for k in (1, 2):
        c = cfg_cache(k)
        r = O.iteration(O.FieldSet.from_config(c), c.x, c.y, c.schedule[0])
        g = gold[f"cfg{k}"]
        assert r.info.n_delaunay == g["D"]
        assert r.info.n_hull == g["hull"]
        assert r.info.n_kept == g["K"]
        assert abs(r.info.c - g["c"]) <= 2e-6 * g["c"]  # printed to 6 significant digits
        assert r.info.n_degenerate == 0


@pytest.mark.slow
def test_iter0_counts_cfg3_cfg4(cfg_cache):
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "iter0_counts.json")))
    for k in (3, 4):
        c = cfg_cache(k)
        r = O.iteration(O.FieldSet.from_config(c), c.x, c.y, "dm")
        g = gold[f"cfg{k}"]
        assert (r.info.n_delaunay, r.info.n_hull, r.info.n_kept) == (g["D"], g["hull"], g["K"])
        assert abs(r.info.c - g["c"]) <= 5e-6 * g["c"]
