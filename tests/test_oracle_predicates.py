"""Pins for the oracle's exact predicates against exact rational arithmetic.

The sign of orient2d / incircle for floating inputs is a plain definition on
rationals (every double is a dyadic rational); Python's fractions.Fraction
evaluates it exactly and shares nothing with oracle.c's big integers.
"""
from fractions import Fraction as Fr

import numpy as np
import pytest

import oracle as O


def orient_fr(a, b, c):
    a, b, c = [tuple(Fr(v) for v in p) for p in (a, b, c)]
    d = (b[0] - a[0]) * (c[1] - a[1]) - (b[1] - a[1]) * (c[0] - a[0])
    return (d > 0) - (d < 0)


def incircle_fr(a, b, c, d):
    P = [tuple(Fr(v) for v in p) for p in (a, b, c, d)]
    (ax, ay), (bx, by), (cx, cy), (dx, dy) = P
    m = [[ax - dx, ay - dy], [bx - dx, by - dy], [cx - dx, cy - dy]]
    lift = [r[0] * r[0] + r[1] * r[1] for r in m]
    det = (lift[0] * (m[1][0] * m[2][1] - m[2][0] * m[1][1])
           + lift[1] * (m[2][0] * m[0][1] - m[0][0] * m[2][1])
           + lift[2] * (m[0][0] * m[1][1] - m[1][0] * m[0][1]))
    return (det > 0) - (det < 0)


def test_random_quads():
    rng = np.random.default_rng(11)
    for _ in range(3000):
        P = rng.random((4, 2)) * rng.choice([1e-3, 1.0, 1e3]) + rng.choice([0.0, 1.0, -7.5])
        a, b, c, d = [tuple(p) for p in P]
        assert O.orient2d(a, b, c) == orient_fr(a, b, c)
        assert O.incircle(a, b, c, d) == incircle_fr(a, b, c, d)
        assert O.incircle(a, b, c, d, exact=True) == incircle_fr(a, b, c, d)


def _nudge(v, k):
    return float(np.nextafter(v, np.inf)) if k > 0 else (float(np.nextafter(v, -np.inf)) if k < 0 else v)


def test_near_degenerate_constructed():
    """Cocircular / collinear configurations perturbed by 0 or +-1 ulp: the
    floating filter cannot certify these, so the big-integer path decides."""
    rng = np.random.default_rng(12)
    n_zero = 0
    for t in range(400):
        cx, cy, r = rng.random() * 0.5 + 0.2, rng.random() * 0.5 + 0.2, 0.1 + rng.random() * 0.05
        ang = np.sort(rng.random(4) * 2 * np.pi)
        P = [(cx + r * np.cos(a), cy + r * np.sin(a)) for a in ang]
        # exact cocircular grid points (integers) in one of five trials
        if t % 5 == 0:
            P = [(3.0, 0.0), (0.0, 3.0), (-3.0, 0.0), (0.0, -3.0)]
        k = int(rng.integers(-1, 2))
        P[3] = (_nudge(P[3][0], k), P[3][1])
        a, b, c, d = P
        s = incircle_fr(a, b, c, d)
        n_zero += s == 0
        assert O.incircle(a, b, c, d) == s
        # collinear: midpoint-ish points
        q = (0.5 * (a[0] + b[0]), 0.5 * (a[1] + b[1]))
        q = (_nudge(q[0], k), q[1])
        assert O.orient2d(a, b, q) == orient_fr(a, b, q)
    assert n_zero > 0  # the exact-zero case was exercised


def test_extreme_exponents():
    a, b, c = (1e-300, 1e-300), (1.0, 2e-300), (3e-300, 1.0)
    assert O.orient2d(a, b, c) == orient_fr(a, b, c)
    d = (0.5, 0.5 + 1e-290)
    assert O.incircle(a, b, c, d) == incircle_fr(a, b, c, d)
