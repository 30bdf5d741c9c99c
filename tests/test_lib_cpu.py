"""CPU checks of the product library (no GPU): it builds, loads, exports every
symbol include/trime_gpu.h declares, and its host-callable hooks -- the very
same __host__ __device__ code the kernels run -- agree with exact rationals."""
import ctypes
import math
import os
import re
from fractions import Fraction as Fr

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2309_13824_b200 import load_library
    return load_library()


def declared_functions():
    src = open(os.path.join(ROOT, "include", "trime_gpu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tm_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol(lib):
    names = declared_functions()
    assert len(names) >= 18
    for n in names:
        assert hasattr(lib, n), n
    from paper_2309_13824_b200 import EXPORTED
    assert set(EXPORTED) == set(names)


def test_sm100a_cubin():
    import subprocess
    so = os.path.join(ROOT, "paper_2309_13824_b200", "libtrime_gpu.so")
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _dp(v):
    return (ctypes.c_double * len(v))(*v)


def incircle_fr(a, b, c, d):
    from tests.test_oracle_predicates import incircle_fr as f
    return f(a, b, c, d)


def test_host_incircle_exact_random(lib):
    rng = np.random.default_rng(21)
    for _ in range(1500):
        P = rng.random((4, 2)) * rng.choice([1e-4, 1.0, 10.0]) + rng.choice([0.0, 0.5, -3.0])
        a, b, c, d = [tuple(p) for p in P]
        assert lib.tm_host_incircle_exact(_dp(a), _dp(b), _dp(c), _dp(d)) == incircle_fr(a, b, c, d)


def test_host_incircle_exact_degenerate(lib):
    rng = np.random.default_rng(22)
    zeros = 0
    for t in range(300):
        if t % 3 == 0:
            s = float(rng.integers(1, 50))
            P = [(s, 0.0), (0.0, s), (-s, 0.0), (0.0, -s)]
        else:
            cx, cy, r = rng.random(3) + 0.1
            ang = rng.random(4) * 2 * np.pi
            P = [(cx + r * math.cos(a), cy + r * math.sin(a)) for a in ang]
        k = int(rng.integers(-1, 2))
        if k:  # 1-ulp nudge of a nonzero coordinate (expansions need no underflow: |v| = 0 or >= 2^-200)
            P[3] = (P[3][0], float(np.nextafter(P[3][1], k * np.inf)))
        a, b, c, d = P
        e = incircle_fr(a, b, c, d)
        zeros += e == 0
        assert lib.tm_host_incircle_exact(_dp(a), _dp(b), _dp(c), _dp(d)) == e
    assert zeros > 10


def test_host_cramer_symmetric_and_accurate(lib):
    rng = np.random.default_rng(23)
    for _ in range(500):
        A = rng.standard_normal(3)
        B = rng.standard_normal(3)
        xy1, xy2 = (ctypes.c_double * 2)(), (ctypes.c_double * 2)()
        lib.tm_host_cramer(_dp(A), _dp(B), xy1)
        lib.tm_host_cramer(_dp(B), _dp(A), xy2)
        assert tuple(xy1) == tuple(xy2)  # exactly symmetric (canonical)
        # exact rational intersection
        a = [Fr(float(v)) for v in A]
        b = [Fr(float(v)) for v in B]
        det = a[0] * b[1] - a[1] * b[0]
        x = (a[2] * b[1] - a[1] * b[2]) / det
        y = (a[0] * b[2] - a[2] * b[0]) / det
        cond = (abs(A[0] * B[1]) + abs(A[1] * B[0])) / abs(float(det))
        assert abs(xy1[0] - float(x)) <= 24 * cond * 2.2e-16 * (abs(float(x)) + abs(A[2] * B[1]) / abs(float(det)) + abs(A[1] * B[2]) / abs(float(det)))
        assert abs(xy1[1] - float(y)) <= 24 * cond * 2.2e-16 * (abs(float(y)) + abs(A[0] * B[2]) / abs(float(det)) + abs(A[2] * B[0]) / abs(float(det)))


def test_host_bilinear_exact_on_bilinear_field(lib):
    from inputs import configs
    n = 17
    gx = configs.node_coords(-1.0, 2.0, n)
    gy = configs.node_coords(0.5, 1.5, n)
    X, Y = np.meshgrid(gx, gy)
    F = np.ascontiguousarray(0.2 - 0.7 * X + 1.3 * Y + 0.9 * X * Y)
    rng = np.random.default_rng(1)
    for _ in range(200):
        x, y = -1.0 + 3.0 * rng.random(), 0.5 + rng.random()
        v = lib.tm_host_bilinear(n, n, -1.0, 0.5, 2.0, 1.5, F.ctypes.data_as(ctypes.c_void_p), x, y)
        assert abs(v - (0.2 - 0.7 * x + 1.3 * y + 0.9 * x * y)) < 1e-14


def test_host_bilinear_matches_oracle_bitwise(lib, cfg_cache):
    """Both sides implement the §8.0 canonical lookup; identical bits are the
    precondition for identical keep decisions."""
    import oracle as O
    c = cfg_cache(3)
    fs = O.FieldSet.from_config(c)
    phi = np.ascontiguousarray(c.phi)
    ny, nx = phi.shape
    for k in range(0, c.n, 997):
        x, y = float(c.x[k]), float(c.y[k])
        v = lib.tm_host_bilinear(nx, ny, *c.box, phi.ctypes.data_as(ctypes.c_void_p), x, y)
        assert v == O.field_value(fs, "phi", x, y)
