"""CPU oracle for the TriMe++ hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product path (``paper_2309_13824_b200``) never imports it and shares no code
with it (see ``oracle/oracle.h``).

Thin ctypes wrapper over ``liboracle.so`` (plain C, built with
``-O2 -ffp-contract=off``); every arithmetic step lives in ``oracle.c`` and
cites PAPER.md there.  ``build()`` compiles it on demand.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass
from typing import Optional

import numpy as np

_DIR = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_DIR, "liboracle.so")
_lib = None

CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c11", "-fPIC", "-shared"]


def build(force: bool = False) -> str:
    src = os.path.join(_DIR, "oracle.c")
    hdr = os.path.join(_DIR, "oracle.h")
    if (not force and os.path.exists(_LIB_PATH)
            and os.path.getmtime(_LIB_PATH) >= max(os.path.getmtime(src), os.path.getmtime(hdr))):
        return _LIB_PATH
    tmp = _LIB_PATH + f".tmp{os.getpid()}"
    subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, src, "-lm"])
    os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


class Fields(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int32), ("ny", ctypes.c_int32),
                ("x0", ctypes.c_double), ("y0", ctypes.c_double),
                ("x1", ctypes.c_double), ("y1", ctypes.c_double),
                ("phi", ctypes.c_void_p), ("mu", ctypes.c_void_p), ("rho", ctypes.c_void_p)]


class Params(ctypes.Structure):
    _fields_ = [("fac_voro_bound", ctypes.c_double), ("fac_pt_mvmt", ctypes.c_double),
                ("fac_geps", ctypes.c_double), ("fac_end_mvmt", ctypes.c_double),
                ("newton_damping", ctypes.c_double), ("newton_max", ctypes.c_int32),
                ("quad_max_level", ctypes.c_int32), ("fscale", ctypes.c_double),
                ("dt_k", ctypes.c_double), ("keep_tol", ctypes.c_double),
                ("projection", ctypes.c_int32), ("trace_max", ctypes.c_int32), ("fac_retria", ctypes.c_double),
                ("validity", ctypes.c_int32), ("t_circ", ctypes.c_double)]


class Info(ctypes.Structure):
    _fields_ = [("c", ctypes.c_double), ("h_avg", ctypes.c_double), ("fac_mu", ctypes.c_double),
                ("sum_l2", ctypes.c_double), ("sum_mu2", ctypes.c_double),
                ("n_delaunay", ctypes.c_int64), ("n_kept", ctypes.c_int64),
                ("n_edges", ctypes.c_int64), ("n_degenerate", ctypes.c_int64),
                ("n_hull", ctypes.c_int64), ("n_near_ties", ctypes.c_int64)]


def default_params(**kw) -> Params:
    """Table B.1 defaults plus the L3/L10/L13 readings."""
    p = Params(fac_voro_bound=5.0, fac_pt_mvmt=0.4, fac_geps=0.01, fac_end_mvmt=0.001,
               newton_damping=1.0, newton_max=10, quad_max_level=10, fscale=1.2, dt_k=0.2,
               keep_tol=0.0, projection=0, trace_max=64, fac_retria=0.1,
               validity=0, t_circ=0.4)
    for k, v in kw.items():
        setattr(p, k, v)
    return p


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        D = ctypes.POINTER(ctypes.c_double)
        L.or_orient2d.restype = ctypes.c_int
        L.or_orient2d.argtypes = [D, D, D]
        L.or_orient2d_exact.restype = ctypes.c_int
        L.or_orient2d_exact.argtypes = [D, D, D]
        L.or_incircle.restype = ctypes.c_int
        L.or_incircle.argtypes = [D, D, D, D]
        L.or_incircle_exact.restype = ctypes.c_int
        L.or_incircle_exact.argtypes = [D, D, D, D]
        L.or_delaunay.restype = ctypes.c_int64
        L.or_delaunay.argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                  ctypes.c_int64, ctypes.POINTER(ctypes.c_int64)]
        L.or_field_value.restype = ctypes.c_double
        L.or_field_value.argtypes = [ctypes.POINTER(Fields), ctypes.c_void_p, ctypes.c_double, ctypes.c_double]
        L.or_field_grad.restype = None
        L.or_field_grad.argtypes = [ctypes.POINTER(Fields), ctypes.c_void_p, ctypes.c_double, ctypes.c_double,
                                    D, D]
        L.or_domain.restype = None
        L.or_domain.argtypes = [ctypes.POINTER(Fields), ctypes.c_int64, D, D]
        L.or_cells.restype = ctypes.c_int64
        L.or_cells.argtypes = [ctypes.POINTER(Fields), ctypes.POINTER(Params), ctypes.c_int64,
                               ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                               ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                               ctypes.POINTER(Info)]
        L.or_iteration.restype = ctypes.c_int
        L.or_iteration.argtypes = [ctypes.POINTER(Fields), ctypes.POINTER(Params), ctypes.c_int64, ctypes.c_int64,
                                   ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                                   ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64,
                                   ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                   ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(Info)]
        L.or_cvd_polygon.restype = None
        L.or_cvd_polygon.argtypes = [ctypes.POINTER(Fields), ctypes.POINTER(Params), ctypes.c_int,
                                     ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double, ctypes.c_double,
                                     ctypes.c_double, ctypes.c_double, D, D, ctypes.POINTER(ctypes.c_int)]
        L.or_distmesh.restype = None
        L.or_distmesh.argtypes = [ctypes.POINTER(Fields), ctypes.POINTER(Params), ctypes.c_int64,
                                  ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                  ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, D]
        L.or_treat.restype = ctypes.c_int
        L.or_treat.argtypes = [ctypes.POINTER(Fields), ctypes.POINTER(Params), ctypes.c_double,
                               ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                               ctypes.c_double, D, D, D]
        L.or_distmesh_lazy.restype = ctypes.c_int
        L.or_distmesh_lazy.argtypes = [ctypes.POINTER(Fields), ctypes.POINTER(Params), ctypes.c_int64, ctypes.c_int64,
                                       ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                       ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                       ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(ctypes.c_int32)]
        L.or_triangle_quality.restype = None
        L.or_triangle_quality.argtypes = [D, D, D, D, D]
        L.or_stats.restype = None
        L.or_stats.argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                               ctypes.c_void_p]
        L.or_keep_triangle.restype = ctypes.c_int
        L.or_keep_triangle.argtypes = [ctypes.POINTER(Fields), ctypes.POINTER(Params), ctypes.c_double,
                                       ctypes.c_double, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32,
                                       ctypes.c_int32, ctypes.c_int32]
        L.or_move_count.restype = ctypes.c_int64
        L.or_move_count.argtypes = [ctypes.POINTER(Fields), ctypes.POINTER(Params), ctypes.c_double, ctypes.c_double,
                                    ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        L.or_point_addition.restype = ctypes.c_int64
        L.or_point_addition.argtypes = [ctypes.POINTER(Fields), ctypes.c_double, ctypes.c_int64, ctypes.c_void_p,
                                        ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                        ctypes.c_void_p, D]
        I32P = ctypes.POINTER(ctypes.c_int32)
        L.or_geometry_grid_dims.restype = None
        L.or_geometry_grid_dims.argtypes = [ctypes.c_int64, ctypes.c_double, ctypes.c_int32, ctypes.c_double,
                                            ctypes.c_double, ctypes.c_double, ctypes.c_double, I32P, I32P]
        L.or_geometry_categories.restype = None
        L.or_geometry_categories.argtypes = [ctypes.POINTER(Fields), ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p]
        L.or_contour_sdf_point.restype = ctypes.c_double
        L.or_contour_sdf_point.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_double]
        L.or_contour_sdf.restype = None
        L.or_contour_sdf.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_double,
                                     ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_void_p]
        L.or_init_counts.restype = ctypes.c_int64
        L.or_init_counts.argtypes = [ctypes.POINTER(Fields), ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p,
                                     ctypes.c_double, ctypes.c_double, ctypes.c_void_p]
        L.or_init_points.restype = ctypes.c_int64
        L.or_init_points.argtypes = [ctypes.POINTER(Fields), ctypes.POINTER(Params), ctypes.c_double, ctypes.c_double,
                                     ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p, ctypes.c_uint64,
                                     ctypes.c_void_p, ctypes.c_void_p]
        L.or_boundary_points.restype = ctypes.c_int64
        L.or_boundary_points.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_double,
                                         ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64]
        L.or_medial_points.restype = ctypes.c_int64
        L.or_medial_points.argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double,
                                       ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                       ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p]
        L.or_sizing_field.restype = None
        L.or_sizing_field.argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                      ctypes.c_void_p, ctypes.c_double, ctypes.c_int32, ctypes.c_int32,
                                      ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                      ctypes.c_void_p, ctypes.c_void_p]
        L.or_adf_build.restype = ctypes.c_void_p
        L.or_adf_build.argtypes = [ctypes.POINTER(Fields), ctypes.POINTER(Params), ctypes.c_double, ctypes.c_double,
                                   ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                   ctypes.c_double, ctypes.c_double, ctypes.c_int32,
                                   ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)]
        L.or_adf_eval.restype = ctypes.c_double
        L.or_adf_eval.argtypes = [ctypes.c_void_p, ctypes.c_double, ctypes.c_double]
        L.or_adf_free.restype = None
        L.or_adf_free.argtypes = [ctypes.c_void_p]
        _lib = L
    return _lib


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _dptr(v):
    arr = (ctypes.c_double * len(v))(*[float(t) for t in v])
    return arr


class FieldSet:
    """Keeps the numpy grids alive while the C struct points into them."""

    def __init__(self, box, phi, mu=None, rho=None):
        self.phi = np.ascontiguousarray(phi, dtype=np.float64)
        self.mu = None if mu is None else np.ascontiguousarray(mu, dtype=np.float64)
        self.rho = None if rho is None else np.ascontiguousarray(rho, dtype=np.float64)
        ny, nx = self.phi.shape
        self.c = Fields(nx=nx, ny=ny, x0=box[0], y0=box[1], x1=box[2], y1=box[3],
                        phi=_p(self.phi), mu=_p(self.mu), rho=_p(self.rho))

    @classmethod
    def from_config(cls, cfg):
        return cls(cfg.box, cfg.phi, cfg.mu, cfg.rho)


# ------------------------------------------------------------------ predicates
def orient2d(a, b, c, exact=False) -> int:
    f = lib().or_orient2d_exact if exact else lib().or_orient2d
    return int(f(_dptr(a), _dptr(b), _dptr(c)))


def incircle(a, b, c, d, exact=False) -> int:
    f = lib().or_incircle_exact if exact else lib().or_incircle
    return int(f(_dptr(a), _dptr(b), _dptr(c), _dptr(d)))


# ------------------------------------------------------------------ O1
def delaunay(x, y):
    """Returns (tri int32 [T,3] CCW min-first, n_degenerate)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    n = x.shape[0]
    cap = 2 * n + 16
    tri = np.empty((cap, 3), dtype=np.int32)
    nd = ctypes.c_int64(0)
    t = lib().or_delaunay(n, _p(x), _p(y), _p(tri), cap, ctypes.byref(nd))
    if t < 0:
        raise RuntimeError("oracle Delaunay failed (n<3, collinear or duplicate points)")
    return tri[:t].copy(), int(nd.value)


# ------------------------------------------------------------------ fields
def field_value(fs: FieldSet, which: str, x: float, y: float) -> float:
    return float(lib().or_field_value(ctypes.byref(fs.c), _p(getattr(fs, which)), x, y))


def field_grad(fs: FieldSet, which: str, x: float, y: float):
    gx, gy = ctypes.c_double(), ctypes.c_double()
    lib().or_field_grad(ctypes.byref(fs.c), _p(getattr(fs, which)), x, y, ctypes.byref(gx), ctypes.byref(gy))
    return gx.value, gy.value


def domain(fs: FieldSet, n_total: int):
    c, h = ctypes.c_double(), ctypes.c_double()
    lib().or_domain(ctypes.byref(fs.c), n_total, ctypes.byref(c), ctypes.byref(h))
    return c.value, h.value


# ------------------------------------------------------------------ O2
@dataclass
class Cells:
    start: np.ndarray
    la: np.ndarray
    lb: np.ndarray
    vx: np.ndarray   # relative to the generator
    vy: np.ndarray
    info: Info

    def cell(self, i):
        s, e = self.start[i], self.start[i + 1]
        return self.la[s:e], self.lb[s:e], self.vx[s:e], self.vy[s:e]


def cells(fs: FieldSet, x, y, params: Optional[Params] = None) -> Cells:
    params = params or default_params()
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    n = x.shape[0]
    cap = 16 * n + 64
    while True:
        start = np.empty(n + 1, dtype=np.int64)
        la = np.empty(cap, dtype=np.int32)
        lb = np.empty(cap, dtype=np.int32)
        vx = np.empty(cap, dtype=np.float64)
        vy = np.empty(cap, dtype=np.float64)
        info = Info()
        t = lib().or_cells(ctypes.byref(fs.c), ctypes.byref(params), n, _p(x), _p(y), _p(start), _p(la),
                           _p(lb), _p(vx), _p(vy), cap, ctypes.byref(info))
        if t >= 0:
            return Cells(start, la[:t], lb[:t], vx[:t], vy[:t], info)
        cap = -t


# ------------------------------------------------------------------ one iteration
@dataclass
class IterResult:
    tri: np.ndarray          # kept triangles K [T,3], CCW, min index first
    edges: np.ndarray        # unique kept edges [E,2] (a<b)
    x_hat: np.ndarray
    y_hat: np.ndarray
    x: np.ndarray
    y: np.ndarray
    d_prev: np.ndarray
    status: np.ndarray
    counts: Optional[np.ndarray]
    info: Info


def iteration(fs: FieldSet, x, y, mode: str, d_prev=None, params: Optional[Params] = None,
              counts: bool = False, n_total: int = 0) -> IterResult:
    """One Delaunay + update + treatment iteration (mode 'cvd' or 'dm')."""
    params = params or default_params()
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    n = x.shape[0]
    tri_cap = 2 * n + 16
    tri = np.empty((tri_cap, 3), dtype=np.int32)
    edges = np.empty((3 * n + 16, 2), dtype=np.int32)
    xh = np.empty(n)
    yh = np.empty(n)
    xo = np.empty(n)
    yo = np.empty(n)
    dp = np.empty(n)
    st = np.empty(n, dtype=np.int8)
    cnt = np.zeros((n, 6), dtype=np.int64) if counts else None
    dpi = None if d_prev is None else np.ascontiguousarray(d_prev, dtype=np.float64)
    info = Info()
    rc = lib().or_iteration(ctypes.byref(fs.c), ctypes.byref(params), n, n_total, _p(x), _p(y), _p(dpi),
                            0 if mode == "cvd" else 1, _p(tri), tri_cap, _p(edges), edges.shape[0],
                            _p(xh), _p(yh), _p(xo), _p(yo), _p(dp), _p(st), _p(cnt), ctypes.byref(info))
    if rc != 0:
        raise RuntimeError(f"oracle iteration failed rc={rc}")
    return IterResult(tri[:info.n_kept].copy(), edges[:info.n_edges].copy(), xh, yh, xo, yo, dp, st, cnt, info)


# ------------------------------------------------------------------ pieces
def cvd_polygon(fs: FieldSet, px, py, g, h, d_prev=-1.0, params=None):
    params = params or default_params()
    px = np.ascontiguousarray(px, dtype=np.float64)
    py = np.ascontiguousarray(py, dtype=np.float64)
    cx, cy, lv = ctypes.c_double(), ctypes.c_double(), ctypes.c_int()
    lib().or_cvd_polygon(ctypes.byref(fs.c), ctypes.byref(params), px.shape[0], _p(px), _p(py), g[0], g[1],
                         h, d_prev, ctypes.byref(cx), ctypes.byref(cy), ctypes.byref(lv))
    return cx.value, cy.value, lv.value


def distmesh(fs: FieldSet, x, y, edges, fixed=None, params=None):
    params = params or default_params()
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    e = np.ascontiguousarray(edges, dtype=np.int32)
    fx = None if fixed is None else np.ascontiguousarray(fixed, dtype=np.uint8)
    xh = np.empty_like(x)
    yh = np.empty_like(y)
    fm = ctypes.c_double()
    lib().or_distmesh(ctypes.byref(fs.c), ctypes.byref(params), x.shape[0], _p(x), _p(y), e.shape[0], _p(e),
                      _p(fx), _p(xh), _p(yh), ctypes.byref(fm))
    return xh, yh, fm.value


def treat(fs: FieldSet, c, h_avg, old, new, params=None):
    params = params or default_params()
    xn, yn, dp = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    st = lib().or_treat(ctypes.byref(fs.c), ctypes.byref(params), c, h_avg, old[0], old[1], new[0], new[1],
                        ctypes.byref(xn), ctypes.byref(yn), ctypes.byref(dp))
    return (xn.value, yn.value), dp.value, int(st)


@dataclass
class LazyResult:
    x: np.ndarray
    y: np.ndarray
    d_prev: np.ndarray
    status: np.ndarray
    retria: bool


def distmesh_lazy(fs: FieldSet, x, y, edges, x_tria, y_tria, params=None, n_total: int = 0) -> LazyResult:
    """NEXT-1: one DistMesh update on the stale triangulation `edges` (Alg. 1), treatment,
    and the re-triangulation flag (any |p_new - p_tria| > fac_retria h(p_tria))."""
    params = params or default_params()
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    e = np.ascontiguousarray(edges, dtype=np.int32)
    xt = np.ascontiguousarray(x_tria, dtype=np.float64)
    yt = np.ascontiguousarray(y_tria, dtype=np.float64)
    n = x.shape[0]
    xo, yo, dp = np.empty(n), np.empty(n), np.empty(n)
    st = np.empty(n, dtype=np.int8)
    flag = ctypes.c_int32()
    lib().or_distmesh_lazy(ctypes.byref(fs.c), ctypes.byref(params), n, n_total, _p(x), _p(y), e.shape[0], _p(e),
                           _p(xt), _p(yt), _p(xo), _p(yo), _p(dp), _p(st), ctypes.byref(flag))
    return LazyResult(xo, yo, dp, st, bool(flag.value))


def triangle_quality(a, b, c):
    al, be = ctypes.c_double(), ctypes.c_double()
    lib().or_triangle_quality(_dptr(a), _dptr(b), _dptr(c), ctypes.byref(al), ctypes.byref(be))
    return al.value, be.value


def stats(tri, x, y):
    tri = np.ascontiguousarray(tri, dtype=np.int32)
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    out = np.zeros(12)
    lib().or_stats(tri.shape[0], _p(tri), _p(x), _p(y), _p(out))
    return out


# ---------------------------------------------------------------- NEXT-2 / NEXT-3
def keep_triangle(fs: FieldSet, c, h_avg, x, y, tri, params=None) -> bool:
    """O3 keep rule on one triangle (indices into x, y)."""
    params = params or default_params()
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    return bool(lib().or_keep_triangle(ctypes.byref(fs.c), ctypes.byref(params), c, h_avg, _p(x), _p(y),
                                       int(tri[0]), int(tri[1]), int(tri[2])))


def move_count(fs: FieldSet, c, h_avg, x_old, y_old, d_prev, params=None) -> int:
    """Inner points (phi~(p_old) < -geps) whose move is not below fac_end_mvmt*h(p_old)."""
    params = params or default_params()
    xo = np.ascontiguousarray(x_old, dtype=np.float64)
    yo = np.ascontiguousarray(y_old, dtype=np.float64)
    dp = np.ascontiguousarray(d_prev, dtype=np.float64)
    return int(lib().or_move_count(ctypes.byref(fs.c), ctypes.byref(params), c, h_avg, xo.shape[0], _p(xo), _p(yo),
                                   _p(dp)))


def point_addition(fs: FieldSet, c, tri, x, y, n_add):
    """centroids of the n_add triangles with the largest R_circ/h(g), in (u, v) order
    of their triangles (reading L46).  Returns (x_new, y_new, smallest selected ratio)."""
    tri = np.ascontiguousarray(tri, dtype=np.int32)
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    k = max(0, min(int(n_add), tri.shape[0]))
    xn, yn = np.empty(k), np.empty(k)
    r = ctypes.c_double(0.0)
    m = lib().or_point_addition(ctypes.byref(fs.c), c, tri.shape[0], _p(tri), _p(x), _p(y), k, _p(xn), _p(yn),
                                ctypes.byref(r))
    return xn[:m], yn[:m], r.value


@dataclass
class ControlParams:
    """Table B.1 thresholds of the meshing controller."""
    t_add_quality: float = 0.002     # P:1093  T^add_quality
    fac_add: float = 0.6             # P:1095  fac_add
    t_end_quality: float = 0.001     # P:1111  T^end_quality
    t_end_alpha_max: float = 0.005   # P:1113  T^end_alpha_max
    t_switch_quality: float = 0.0015 # P:1121  T^switch_quality
    max_iterations: int = 1000       # safety cap (paper silent)


class Controller:
    """The iterate-to-termination controller (NEXT-2, NEXT-3 trigger), step by step as the paper
    states it (reading L45):

    * quality of iteration n: the 1/2-means M_a, M_b of alpha and beta and max alpha over the kept
      triangles T_n at the positions p_n they were computed from (Eqs. aspect/edge ratios, 1/2-mean,
      P:415-427); relative change r(X) = |X_n - X_{n-1}| / X_{n-1} between consecutive iterations
      at the same N_current (the history restarts after a point addition);
    * N_current < N_total: add points when r(M_a) < T_add and r(M_b) < T_add, N_add =
      min(floor(fac_add N_current), N_total - N_current);
    * N_current = N_total, hybrid, still DistMesh: switch to CVD from the next iteration when
      r(M_a) < T_switch;
    * N_current = N_total, CVD (or DistMesh-only meshing): terminate when r(M_a) < T_end and
      r(M_b) < T_end and r(max alpha) < T_end_alpha, or when no inner point moved by at
      least fac_end h (move_count == 0).

    update() returns a dict {"action": "continue"|"add"|"switch"|"terminate", "n_add": k}."""

    def __init__(self, n_total, n_current, method="hybrid", cp: Optional[ControlParams] = None):
        self.cp = cp or ControlParams()
        self.n_total = int(n_total)
        self.n_current = int(n_current)
        self.method = method                       # "cvd", "distmesh", "hybrid"
        self.mode = "cvd" if method == "cvd" else "dm"
        self.prev = None
        self.iterations = 0

    @staticmethod
    def _rel(a, b):
        return abs(a - b) / b

    def update(self, half_alpha, half_beta, max_alpha, move_count):
        cp = self.cp
        self.iterations += 1
        cur = (float(half_alpha), float(half_beta), float(max_alpha))
        prev, self.prev = self.prev, cur
        if self.iterations >= cp.max_iterations:
            return {"action": "terminate", "n_add": 0, "reason": "max_iterations"}
        if self.n_current < self.n_total:
            if prev is not None and self._rel(cur[0], prev[0]) < cp.t_add_quality and \
                    self._rel(cur[1], prev[1]) < cp.t_add_quality:
                k = min(int(np.floor(cp.fac_add * self.n_current)), self.n_total - self.n_current)
                self.n_current += k
                self.prev = None
                return {"action": "add", "n_add": k}
            return {"action": "continue", "n_add": 0}
        if self.method == "hybrid" and self.mode == "dm":
            if prev is not None and self._rel(cur[0], prev[0]) < cp.t_switch_quality:
                self.mode = "cvd"
                return {"action": "switch", "n_add": 0}
            return {"action": "continue", "n_add": 0}
        if move_count == 0:
            return {"action": "terminate", "n_add": 0, "reason": "movement"}
        if prev is not None and self._rel(cur[0], prev[0]) < cp.t_end_quality and \
                self._rel(cur[1], prev[1]) < cp.t_end_quality and self._rel(cur[2], prev[2]) < cp.t_end_alpha_max:
            return {"action": "terminate", "n_add": 0, "reason": "quality"}
        return {"action": "continue", "n_add": 0}


def quality_of(st):
    """(1/2-mean alpha, 1/2-mean beta, max alpha) from stats() (Eq. 1/2-mean)."""
    n = st[0]
    return (st[1] / n) ** 2, (st[2] / n) ** 2, st[3]


# ---------------------------------------------------------------- NEXT-4
def geometry_grid_dims(n_total, box, n_opt=3.3, fac_grid=5):
    """P:338-346."""
    nx, ny = ctypes.c_int32(), ctypes.c_int32()
    lib().or_geometry_grid_dims(int(n_total), float(n_opt), int(fac_grid), box[0], box[1], box[2], box[3],
                                ctypes.byref(nx), ctypes.byref(ny))
    return nx.value, ny.value


def geometry_categories(fs: FieldSet, nxg, nyg):
    """[nyg, nxg] int8, 0 inner / 1 boundary / 2 outer."""
    cat = np.empty(nxg * nyg, dtype=np.int8)
    lib().or_geometry_categories(ctypes.byref(fs.c), int(nxg), int(nyg), _p(cat))
    return cat.reshape(nyg, nxg)


def contour_sdf(segs, nx, ny, box):
    """SDF of a closed clockwise loop of segments [n, 4] on the (ny, nx) node grid."""
    s = np.ascontiguousarray(segs, dtype=np.float64)
    phi = np.empty(nx * ny)
    lib().or_contour_sdf(_p(s), s.shape[0], int(nx), int(ny), box[0], box[1], box[2], box[3], _p(phi))
    return phi.reshape(ny, nx)


def contour_sdf_point(segs, x, y):
    s = np.ascontiguousarray(segs, dtype=np.float64)
    return lib().or_contour_sdf_point(_p(s), s.shape[0], float(x), float(y))


def init_counts(fs: FieldSet, cat, n_init, eta=0.5):
    """P:380-406 Floyd-Steinberg counts [nyg, nxg] and their total."""
    nyg, nxg = cat.shape
    c8 = np.ascontiguousarray(cat, dtype=np.int8)
    cnt = np.empty(nxg * nyg, dtype=np.int32)
    tot = lib().or_init_counts(ctypes.byref(fs.c), int(nxg), int(nyg), _p(c8), float(n_init), float(eta), _p(cnt))
    return cnt.reshape(nyg, nxg), int(tot)


def init_points(fs: FieldSet, counts, seed, c, h_avg, params=None):
    params = params or default_params()
    nyg, nxg = counts.shape
    cn = np.ascontiguousarray(counts, dtype=np.int32)
    n = int(cn.sum())
    x, y = np.empty(n), np.empty(n)
    lib().or_init_points(ctypes.byref(fs.c), ctypes.byref(params), c, h_avg, int(nxg), int(nyg), _p(cn), int(seed),
                         _p(x), _p(y))
    return x, y


def boundary_points(segs, d_s, geps_hat):
    """App. A: contour boundary points, trimmed to spacing >= d_s."""
    s = np.ascontiguousarray(segs, dtype=np.float64)
    cap = 16
    while True:
        x, y = np.empty(cap), np.empty(cap)
        n = lib().or_boundary_points(_p(s), s.shape[0], float(d_s), float(geps_hat), _p(x), _p(y), cap)
        if n >= 0:
            return x[:n].copy(), y[:n].copy()
        cap = -n


def medial_points(x, y, box, r_nei, n_thres=3):
    """Delaunay poles of the boundary points, trimmed by neighbour counts."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    mx, my = np.empty(2 * len(x) + 16), np.empty(2 * len(x) + 16)
    m = lib().or_medial_points(len(x), _p(x), _p(y), box[0], box[1], box[2], box[3], float(r_nei), int(n_thres),
                               _p(mx), _p(my))
    return mx[:m].copy(), my[:m].copy()


def sizing_field(sx, sy, mx, my, K, nx, ny, box):
    """Eq. sizing field: mu on the node grid and lfs at the boundary points."""
    sx, sy = np.ascontiguousarray(sx, dtype=np.float64), np.ascontiguousarray(sy, dtype=np.float64)
    mx, my = np.ascontiguousarray(mx, dtype=np.float64), np.ascontiguousarray(my, dtype=np.float64)
    mu = np.empty(nx * ny)
    lfs = np.empty(len(sx))
    lib().or_sizing_field(len(sx), _p(sx), _p(sy), len(mx), _p(mx), _p(my), float(K), int(nx), int(ny), box[0],
                          box[1], box[2], box[3], _p(mu), _p(lfs))
    return mu.reshape(ny, nx), lfs


class ADF:
    """quadtree ADFs of the contour's SDF on the boundary cells (cat == 1)."""

    def __init__(self, fs: FieldSet, c, h_avg, cat, segs, fac_etol=0.1, fac_pt=1.0, max_depth=10, params=None):
        params = params or default_params()
        nyg, nxg = cat.shape
        self._cat = np.ascontiguousarray(cat, dtype=np.int8)
        self._segs = np.ascontiguousarray(segs, dtype=np.float64)
        nn, nl = ctypes.c_int64(), ctypes.c_int64()
        self.h = lib().or_adf_build(ctypes.byref(fs.c), ctypes.byref(params), c, h_avg, nxg, nyg, _p(self._cat),
                                    _p(self._segs), self._segs.shape[0], fac_etol, fac_pt, max_depth,
                                    ctypes.byref(nn), ctypes.byref(nl))
        self.n_nodes, self.n_leaves = nn.value, nl.value

    def __call__(self, x, y):
        return lib().or_adf_eval(self.h, float(x), float(y))

    def __del__(self):
        try:
            lib().or_adf_free(self.h)
        except Exception:
            pass
