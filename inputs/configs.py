"""Seeded synthetic inputs for the five BASELINE.json configs.

This module is shared by the CPU oracle (``oracle/``) and the GPU path
(``paper_2309_13824_b200``).  It holds NONE of the method's arithmetic: it
only draws points and samples the user-supplied fields (signed distance
phi, relative sizing mu, density rho) on node-centred grids, i.e. the
*inputs* of the paper's problem statement (SDF: §3.1;
sizing field: §3.3; density rho = mu^-2: §3.4).

Recipes follow SURVEY.md §8(d) ("Synthetic inputs") exactly: numpy
``default_rng(seed)`` (PCG64), float64, rejection sampling in fixed batch
sizes (2**17 for cfg2, 2**20 for cfg3/cfg4) consumed in draw order and
truncated to N.  The paper's own workloads (uniform square P:705-747,
custom adaptive shape P:787-829) are stand-ins only: the custom contour is
not available, so cfg3/cfg4 are synthetic adaptive shapes.

Grids are node-centred, n x n over the box B=[x0,x1]x[y0,y1], row-major
``[ny][nx]`` with node k at ``x0 + k*(x1-x0)/(n-1)`` (reading L15).
"""
from __future__ import annotations

import dataclasses
import os
from typing import Optional

import numpy as np


@dataclasses.dataclass
class Config:
    """One workload: points + box + node grids + iteration schedule."""

    name: str
    x: np.ndarray              # float64 [N]
    y: np.ndarray              # float64 [N]
    box: tuple                 # (x0, y0, x1, y1)
    phi: np.ndarray            # float64 [ny, nx], < 0 inside
    mu: Optional[np.ndarray]   # float64 [ny, nx] relative sizing, None = uniform
    rho: Optional[np.ndarray]  # float64 [ny, nx] density, None = uniform
    schedule: list             # list of "cvd" / "dm", one per iteration

    @property
    def n(self) -> int:
        return int(self.x.shape[0])


def node_coords(lo: float, hi: float, n: int) -> np.ndarray:
    """Node coordinates lo + k*(hi-lo)/(n-1), last node pinned to hi."""
    step = (hi - lo) / (n - 1)
    c = lo + np.arange(n, dtype=np.float64) * step
    c[-1] = hi
    return c


def _grid(box, n):
    x0, y0, x1, y1 = box
    gx = node_coords(x0, x1, n)
    gy = node_coords(y0, y1, n)
    return np.meshgrid(gx, gy, indexing="xy")  # X[j,i] = gx[i], Y[j,i] = gy[j]


def _box_sdf(X, Y, lo=0.0, hi=1.0):
    # signed distance of the square [lo,hi]^2, exact inside (the only region used)
    inside = np.minimum(np.minimum(X - lo, hi - X), np.minimum(Y - lo, hi - Y))
    dx = np.maximum(np.maximum(lo - X, X - hi), 0.0)
    dy = np.maximum(np.maximum(lo - Y, Y - hi), 0.0)
    outside = np.sqrt(dx * dx + dy * dy)
    return np.where(inside >= 0.0, -inside, outside)


# ---------------------------------------------------------------- config 1
def config1(n: int = 1000) -> Config:
    """Unit square, i.i.d. uniform, 128^2 box SDF, 10 CVD (BASELINE configs[0])."""
    rng = np.random.default_rng(0)
    P = rng.random((n, 2))
    box = (0.0, 0.0, 1.0, 1.0)
    X, Y = _grid(box, 128)
    phi = _box_sdf(X, Y)
    return Config("cfg1", P[:, 0].copy(), P[:, 1].copy(), box, phi, None, None,
                  ["cvd"] * 10)


# ---------------------------------------------------------------- config 2
def config2(n: int = 100_000) -> Config:
    """Unit disk, 512^2 SDF over [-1.1,1.1]^2, 50 DistMesh (configs[1])."""
    rng = np.random.default_rng(1)
    keep = []
    got = 0
    while got < n:
        Q = rng.uniform(-1.0, 1.0, (2 ** 17, 2))
        Q = Q[Q[:, 0] ** 2 + Q[:, 1] ** 2 < 1.0]
        keep.append(Q)
        got += Q.shape[0]
    P = np.concatenate(keep)[:n]
    box = (-1.1, -1.1, 1.1, 1.1)
    X, Y = _grid(box, 512)
    phi = np.sqrt(X * X + Y * Y) - 1.0
    return Config("cfg2", P[:, 0].copy(), P[:, 1].copy(), box, phi, None, None,
                  ["dm"] * 50)


# ---------------------------------------------------------------- config 3
def _annulus_phi(X, Y):
    r = np.sqrt(X * X + Y * Y)
    return np.maximum(r - 1.0, 0.3 - r)


def _cfg3_mu(phi):
    return np.minimum(0.002 + 0.3 * np.abs(phi), 0.02)


def config3(n: int = 1_000_000, grid: int = 1024) -> Config:
    """Annulus 0.3<|x|<1, adaptive, 30 DistMesh + 30 CVD (configs[2])."""
    rng = np.random.default_rng(2)
    rho_max = 0.002 ** -2
    keep = []
    got = 0
    B = 2 ** 20
    while got < n:
        Q = rng.uniform(-1.0, 1.0, (B, 2))
        U = rng.random(B)
        r = np.sqrt(Q[:, 0] ** 2 + Q[:, 1] ** 2)
        phi = np.maximum(r - 1.0, 0.3 - r)
        rho = _cfg3_mu(phi) ** -2
        ok = (r > 0.3) & (r < 1.0) & (U < rho / rho_max)
        keep.append(Q[ok])
        got += int(ok.sum())
    P = np.concatenate(keep)[:n]
    box = (-1.1, -1.1, 1.1, 1.1)
    X, Y = _grid(box, grid)
    phi = _annulus_phi(X, Y)
    mu = _cfg3_mu(phi)
    rho = mu ** -2
    return Config("cfg3", P[:, 0].copy(), P[:, 1].copy(), box, phi, mu, rho,
                  ["dm"] * 30 + ["cvd"] * 30)


# ---------------------------------------------------------------- config 4
def _cfg4_phi(X, Y, dc, dr, hc, hr, chunk=1 << 18):
    flatx = X.reshape(-1)
    flaty = Y.reshape(-1)
    out = np.empty_like(flatx)
    for s in range(0, flatx.shape[0], chunk):
        px = flatx[s:s + chunk, None]
        py = flaty[s:s + chunk, None]
        dd = np.sqrt((px - dc[None, :, 0]) ** 2 + (py - dc[None, :, 1]) ** 2) - dr[None, :]
        dh = np.sqrt((px - hc[None, :, 0]) ** 2 + (py - hc[None, :, 1]) ** 2) - hr[None, :]
        # union of disks = min, minus holes = max(A, -B)
        out[s:s + chunk] = np.maximum(dd.min(axis=1), -dh.min(axis=1))
    return out.reshape(X.shape)


def _cfg4_mu(phi):
    return np.minimum(0.001 + 0.2 * np.abs(phi), 0.01)


def config4_shape():
    rng = np.random.default_rng(3)
    dc = rng.uniform(0.1, 0.9, (64, 2))
    dr = rng.uniform(0.03, 0.12, 64)
    hc = rng.uniform(0.1, 0.9, (32, 2))
    hr = rng.uniform(0.005, 0.03, 32)
    return rng, dc, dr, hc, hr


def config4(n: int = 1_000_000, grid: int = 2048) -> Config:
    """64 disks minus 32 holes, adaptive, 20 DistMesh + 20 CVD (configs[3])."""
    rng, dc, dr, hc, hr = config4_shape()
    rho_max = 0.001 ** -2
    keep = []
    got = 0
    B = 2 ** 20
    while got < n:
        Q = rng.uniform(-0.05, 1.05, (B, 2))
        U = rng.random(B)
        phi = _cfg4_phi(Q[:, 0], Q[:, 1], dc, dr, hc, hr)
        rho = _cfg4_mu(phi) ** -2
        ok = (phi < 0.0) & (U < rho / rho_max)
        keep.append(Q[ok])
        got += int(ok.sum())
    P = np.concatenate(keep)[:n]
    box = (-0.05, -0.05, 1.05, 1.05)
    X, Y = _grid(box, grid)
    phi = _cfg4_phi(X, Y, dc, dr, hc, hr)
    mu = _cfg4_mu(phi)
    rho = mu ** -2
    return Config("cfg4", P[:, 0].copy(), P[:, 1].copy(), box, phi, mu, rho,
                  ["dm"] * 20 + ["cvd"] * 20)


# ---------------------------------------------------------------- config 5
def config5(n: int = 16_000_000, grid: int = 1024, iters: int = 20) -> Config:
    """Jittered-uniform unit square for multi-GPU scaling (configs[4])."""
    s = int(round(np.sqrt(n)))
    assert s * s == n, "config 5 needs a square N"
    rng = np.random.default_rng(4)
    U = rng.random((n, 2))
    k = np.arange(n, dtype=np.int64)
    i = (k % s).astype(np.float64)
    j = (k // s).astype(np.float64)
    x = (i + U[:, 0]) / s
    y = (j + U[:, 1]) / s
    box = (0.0, 0.0, 1.0, 1.0)
    X, Y = _grid(box, grid)
    phi = _box_sdf(X, Y)
    return Config("cfg5", x, y, box, phi, None, None, ["cvd"] * iters)


_BUILDERS = {1: config1, 2: config2, 3: config3, 4: config4, 5: config5}


def _cache_dir():
    d = os.environ.get("TRIME_INPUT_CACHE",
                       os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                    ".cache", "inputs"))
    return d


def load(k: int, cache: bool = True, **kw) -> Config:
    """Build config k (1..5), optionally memoised as .npz under .cache/inputs.

    The cache is a pure speed-up (generation is deterministic); a missing or
    unreadable cache entry is regenerated.
    """
    if not cache or kw:
        return _BUILDERS[k](**kw)
    path = os.path.join(_cache_dir(), f"cfg{k}.npz")
    if os.path.exists(path):
        try:
            z = np.load(path, allow_pickle=False)
            mu = z["mu"] if z["has_mu"] else None
            rho = z["rho"] if z["has_rho"] else None
            return Config(str(z["name"]), z["x"], z["y"], tuple(z["box"].tolist()),
                          z["phi"], mu, rho, [str(s) for s in z["schedule"]])
        except Exception:
            pass
    c = _BUILDERS[k]()
    os.makedirs(_cache_dir(), exist_ok=True)
    tmp = path + f".tmp{os.getpid()}.npz"  # per process: the ranks of a multi-GPU run may build it at once
    np.savez(tmp, name=c.name, x=c.x, y=c.y, box=np.array(c.box), phi=c.phi,
             mu=c.mu if c.mu is not None else np.zeros(1),
             rho=c.rho if c.rho is not None else np.zeros(1),
             has_mu=c.mu is not None, has_rho=c.rho is not None,
             schedule=np.array(c.schedule))
    os.replace(tmp, path)
    return c


def random_points(n: int, seed: int, box=(0.0, 0.0, 1.0, 1.0)):
    """i.i.d. uniform points in a box (small parity/edge cases)."""
    rng = np.random.default_rng(seed)
    x0, y0, x1, y1 = box
    P = rng.random((n, 2))
    return x0 + P[:, 0] * (x1 - x0), y0 + P[:, 1] * (y1 - y0)


def box_phi(box, n):
    """Box SDF grid for the given box (used by small synthetic cases)."""
    X, Y = _grid(box, n)
    return _box_sdf(X, Y, box[0], box[2]) if box[0] == box[1] and box[2] == box[3] else \
        np.maximum(np.maximum(box[0] - X, X - box[2]), np.maximum(box[1] - Y, Y - box[3]))


def disk_phi(box, n, r=1.0):
    X, Y = _grid(box, n)
    return np.sqrt(X * X + Y * Y) - r


# ---------------------------------------------------------------- NEXT-2 test input
def validity_strip():
    """left half of the unit square (phi = x - 1/2, exactly bilinear on 33^2 nodes); a jittered
    interior lattice, a strip of points alternating just outside (phi = +4e-4 <= geps) and just
    inside (-2e-4) the boundary, and a few points outside (phi = 0.1): boundary triangles whose
    centroid lies in (0, geps] (Tests 1-2 keep, the L10 reading discards) and triangles decided
    by Test 3."""
    rng = np.random.default_rng(21)
    g = np.arange(0.03, 0.44, 0.05)
    X, Y = np.meshgrid(g, np.arange(0.03, 0.98, 0.05))
    xi = (X + rng.uniform(-0.01, 0.01, X.shape)).ravel(); yi = (Y + rng.uniform(-0.01, 0.01, Y.shape)).ravel()
    k = np.arange(0, 20)
    xo = 0.5004 + rng.uniform(-5e-5, 5e-5, k.size); yo = 0.30 + 0.02 * k + rng.uniform(-2e-3, 2e-3, k.size)
    xa = 0.4998 + rng.uniform(-5e-5, 5e-5, k.size - 1); ya = 0.31 + 0.02 * k[:-1] + rng.uniform(-2e-3, 2e-3, k.size - 1)
    xf = np.array([0.6, 0.62, 0.6]); yf = np.array([0.12, 0.80, 0.92])
    x = np.concatenate([xi, xo, xa, xf]); y = np.concatenate([yi, yo, ya, yf])
    box = (0.0, 0.0, 1.0, 1.0)
    gx = node_coords(0, 1, 33)
    PX, PY = np.meshgrid(gx, gx)
    return box, PX - 0.5, x, y
