"""paper_2309_13824_b200 -- B200-native hot path of TriMe++ iterative meshing.

Thin ctypes binding over ``libtrime_gpu.so`` (``include/trime_gpu.h``): the
functions below keep the C names and only marshal arguments (torch CUDA
tensors -> device pointers, the current torch stream -> the context stream).
Every step of the iteration runs in the library's sm_100a kernels; there is
no CPU fallback -- importing this package on a machine without the built
library raises immediately, and calls fail loudly on a non-zero status.

PyTorch supplies device memory, streams and process groups only.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import Optional

import torch

from . import build as _build

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TRIME_LIB", os.path.join(_PKG, "libtrime_gpu.so"))

TM_OK, TM_E_ARG, TM_E_CUDA, TM_E_CAPACITY, TM_E_DUPLICATE, TM_E_OUTSIDE, TM_E_STATE, TM_E_DEGENERATE = range(8)
STATUS_NAMES = ["TM_OK", "TM_E_ARG", "TM_E_CUDA", "TM_E_CAPACITY", "TM_E_DUPLICATE", "TM_E_OUTSIDE",
                "TM_E_STATE", "TM_E_DEGENERATE"]
TM_F_TWO_LEVEL_BINS = 0x1
TM_F_COUNT_WORK = 0x2
TM_F_GROUP_CELLS = 0x4
TM_F_NO_WCERT = 0x8
TM_F_NO_PACKED_GRIDS = 0x10
TM_F_NO_DEEP_PASS = 0x20


class TmError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS_NAMES[code] if 0 <= code < len(STATUS_NAMES) else code}: {msg}")
        self.code = code


class tm_fields(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int32), ("ny", ctypes.c_int32),
                ("x0", ctypes.c_double), ("y0", ctypes.c_double),
                ("x1", ctypes.c_double), ("y1", ctypes.c_double),
                ("phi", ctypes.c_void_p), ("mu", ctypes.c_void_p), ("rho", ctypes.c_void_p)]


class tm_params(ctypes.Structure):
    _fields_ = [("n_opt", ctypes.c_double), ("fac_voro_bound", ctypes.c_double),
                ("fac_pt_mvmt", ctypes.c_double), ("fac_geps", ctypes.c_double),
                ("fac_end_mvmt", ctypes.c_double), ("newton_damping", ctypes.c_double),
                ("newton_max", ctypes.c_int32), ("quad_max_level", ctypes.c_int32),
                ("fscale", ctypes.c_double), ("dt_k", ctypes.c_double), ("keep_tol", ctypes.c_double),
                ("adj_stride", ctypes.c_int32), ("max_cell_vertices", ctypes.c_int32),
                ("flags", ctypes.c_uint32), ("projection", ctypes.c_int32), ("trace_max", ctypes.c_int32),
                ("fac_retria", ctypes.c_double), ("validity", ctypes.c_int32), ("t_circ", ctypes.c_double)]


class tm_stats(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in ("n_tri", "n_alpha_lt_1_2", "n_alpha_lt_2", "n_degenerate",
                                              "n_fallback", "n_overflow")] + \
               [(n, ctypes.c_double) for n in ("sum_sqrt_alpha", "sum_sqrt_beta", "max_alpha", "max_beta",
                                               "sum_alpha", "sum_alpha2", "sum_beta", "sum_beta2")]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


TM_METHOD_CVD, TM_METHOD_DISTMESH, TM_METHOD_HYBRID = 0, 1, 2
TM_ACT_NAMES = ["continue", "add", "switch", "terminate_quality", "terminate_moves", "terminate_cap"]


class tm_control(ctypes.Structure):
    _fields_ = [("n_total", ctypes.c_int64), ("n_current", ctypes.c_int64), ("method", ctypes.c_int32),
                ("mode", ctypes.c_int32), ("have_prev", ctypes.c_int32), ("iterations", ctypes.c_int32),
                ("prev", ctypes.c_double * 3), ("t_add_quality", ctypes.c_double), ("fac_add", ctypes.c_double),
                ("t_end_quality", ctypes.c_double), ("t_end_alpha_max", ctypes.c_double),
                ("t_switch_quality", ctypes.c_double), ("max_iterations", ctypes.c_int32)]


class tm_work(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in ("n_cells", "n_cert", "deg", "verts", "t_own", "quad_tris", "ell",
                                              "candidates", "clips", "exact_calls", "retries", "warp_trips")]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_lib = None
EXPORTED = ["tm_params_default", "tm_create", "tm_destroy", "tm_last_error", "tm_sync", "tm_set_domain",
            "tm_grid_bin", "tm_voronoi_delaunay", "tm_cvd_step", "tm_distmesh_sums", "tm_distmesh_step",
            "tm_project_sdf", "tm_mesh_stats", "tm_adjacency_export", "tm_work_counts", "tm_halo_pack",
            "tm_migrate_pack", "tm_grid_bin_dc", "tm_halo_pack_dc", "tm_migrate_pack_dc", "tm_append_points",
            "tm_graph_begin", "tm_graph_end", "tm_graph_launch", "tm_graph_destroy", "tm_refresh_positions",
            "tm_retria_check", "tm_move_count", "tm_set_n_total", "tm_point_addition", "tm_control_init",
            "tm_control_update", "tm_geometry_grid_dims", "tm_geometry_categories", "tm_contour_sdf",
            "tm_sdf_combine", "tm_init_points", "tm_boundary_points", "tm_medial_points", "tm_sizing_field",
            "tm_density_from_sizing", "tm_adf_build", "tm_adf_eval", "tm_x_histogram",
            "tm_host_incircle_exact", "tm_host_cramer", "tm_host_bilinear"]


def load_library(path: str = LIB_PATH, build_if_missing: bool = True):
    """Load libtrime_gpu.so (building it with nvcc if absent and allowed)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        if not build_if_missing:
            raise ImportError(f"{path} missing: run `python -m paper_2309_13824_b200.build`")
        _build.build()
    L = ctypes.CDLL(path)
    vp, i64, i32, dbl = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_double
    st = ctypes.c_int
    sig = {
        "tm_params_default": (None, [ctypes.POINTER(tm_params)]),
        "tm_create": (st, [ctypes.c_int, vp, ctypes.POINTER(tm_params), ctypes.POINTER(vp)]),
        "tm_destroy": (None, [vp]),
        "tm_last_error": (ctypes.c_char_p, [vp]),
        "tm_sync": (st, [vp]),
        "tm_set_domain": (st, [vp, ctypes.POINTER(tm_fields), i64, ctypes.POINTER(dbl), ctypes.POINTER(dbl)]),
        "tm_grid_bin": (st, [vp, vp, vp, i64, i64, vp]),
        "tm_voronoi_delaunay": (st, [vp, vp, i64, vp, vp, vp, vp, vp, vp, vp, vp]),
        "tm_cvd_step": (st, [vp, vp, vp, vp]),
        "tm_distmesh_sums": (st, [vp, vp, vp, vp]),
        "tm_distmesh_step": (st, [vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
        "tm_project_sdf": (st, [vp, vp, vp, vp, vp, i64, vp, vp, vp, vp]),
        "tm_mesh_stats": (st, [vp, vp, vp, vp, i64, ctypes.POINTER(tm_stats)]),
        "tm_adjacency_export": (st, [vp, vp, vp, vp, vp]),
        "tm_work_counts": (st, [vp, ctypes.POINTER(tm_work)]),
        "tm_move_count": (st, [vp, vp, vp, vp, i64, vp]),
        "tm_geometry_grid_dims": (None, [i64, dbl, i32, dbl, dbl, dbl, dbl, ctypes.POINTER(i32), ctypes.POINTER(i32)]),
        "tm_geometry_categories": (st, [vp, i32, i32, vp]),
        "tm_contour_sdf": (st, [vp, vp, i64, i32, i32, dbl, dbl, dbl, dbl, vp]),
        "tm_sdf_combine": (st, [vp, i32, vp, vp, i64, vp]),
        "tm_boundary_points": (st, [vp, vp, i64, dbl, dbl, vp, vp, i64, ctypes.POINTER(i64)]),
        "tm_medial_points": (st, [vp, vp, vp, i64, dbl, dbl, dbl, dbl, dbl, i32, vp, vp, i64, ctypes.POINTER(i64)]),
        "tm_density_from_sizing": (st, [vp, vp, i64, vp]),
        "tm_adf_build": (st, [vp, vp, i64, i32, i32, vp, dbl, dbl, i32, ctypes.POINTER(i64), ctypes.POINTER(i64)]),
        "tm_adf_eval": (st, [vp, vp, vp, i64, vp]),
        "tm_x_histogram": (st, [vp, vp, vp, i64, dbl, dbl, i32, vp]),
        "tm_sizing_field": (st, [vp, vp, vp, i64, vp, vp, i64, dbl, i32, i32, dbl, dbl, dbl, dbl, vp, vp]),
        "tm_init_points": (st, [vp, i32, i32, vp, dbl, dbl, ctypes.c_uint64, vp, vp, vp, i64, ctypes.POINTER(i64)]),
        "tm_set_n_total": (st, [vp, i64, ctypes.POINTER(dbl), ctypes.POINTER(dbl)]),
        "tm_point_addition": (st, [vp, vp, i64, vp, vp, i64, vp, vp, ctypes.POINTER(dbl)]),
        "tm_control_init": (None, [ctypes.POINTER(tm_control), i64, i64, i32]),
        "tm_control_update": (i32, [ctypes.POINTER(tm_control), ctypes.POINTER(tm_stats), i64,
                                    ctypes.POINTER(i64)]),
        "tm_halo_pack": (st, [vp, vp, vp, vp, i64, dbl, dbl, dbl, vp, vp, i64, vp]),
        "tm_migrate_pack": (st, [vp, vp, vp, vp, vp, i64, dbl, dbl, vp, vp, i64, vp]),
        "tm_grid_bin_dc": (st, [vp, vp, vp, i64, vp, vp]),
        "tm_halo_pack_dc": (st, [vp, vp, vp, vp, vp, i64, dbl, dbl, dbl, vp, vp, i64, vp, vp]),
        "tm_migrate_pack_dc": (st, [vp, vp, vp, vp, vp, vp, i64, dbl, dbl, vp, vp, i64, vp, vp]),
        "tm_append_points": (st, [vp, vp, vp, vp, vp, vp, i64, vp, vp, i64]),
        "tm_refresh_positions": (st, [vp, vp, vp]),
        "tm_retria_check": (st, [vp, vp, vp, vp]),
        "tm_graph_begin": (st, [vp]),
        "tm_graph_end": (st, [vp, ctypes.POINTER(vp)]),
        "tm_graph_launch": (st, [vp, vp]),
        "tm_graph_destroy": (None, [vp]),
        "tm_host_incircle_exact": (ctypes.c_int, [vp, vp, vp, vp]),
        "tm_host_cramer": (None, [vp, vp, vp]),
        "tm_host_bilinear": (dbl, [i32, i32, dbl, dbl, dbl, dbl, vp, dbl, dbl]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def _ptr(t: Optional[torch.Tensor]):
    if t is None:
        return None
    if not t.is_cuda:
        raise TmError(TM_E_ARG, "tensor must live on a CUDA device (no CPU fallback)")
    if not t.is_contiguous():
        raise TmError(TM_E_ARG, "tensor must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


def _addr(a):
    """A raw device address (int) or a CUDA tensor -> c_void_p."""
    if isinstance(a, torch.Tensor):
        return _ptr(a)
    return ctypes.c_void_p(int(a))


def default_params(**kw) -> tm_params:
    p = tm_params()
    load_library().tm_params_default(ctypes.byref(p))
    for k, v in kw.items():
        setattr(p, k, v)
    return p


class Context:
    """One tm_ctx bound to a CUDA device and a torch stream."""

    def __init__(self, device: int = 0, stream: Optional[torch.cuda.Stream] = None,
                 params: Optional[tm_params] = None):
        if not torch.cuda.is_available():
            raise TmError(TM_E_CUDA, "no CUDA device: the TriMe++ B200 path has no CPU fallback")
        self.L = load_library()
        self.device = device
        self.stream = stream or torch.cuda.current_stream(device)
        self.params = params or default_params()
        h = ctypes.c_void_p()
        rc = self.L.tm_create(device, ctypes.c_void_p(self.stream.cuda_stream), ctypes.byref(self.params),
                              ctypes.byref(h))
        if rc != TM_OK:
            raise TmError(rc, "tm_create failed")
        self.h = h
        self.c = None
        self.h_avg = None
        self._fields_keepalive = None

    def close(self):
        if getattr(self, "h", None):
            self.L.tm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc):
        if rc != TM_OK:
            msg = self.L.tm_last_error(self.h)
            raise TmError(rc, msg.decode() if msg else "")

    # ---------------------------------------------------------------- C names
    def tm_sync(self):
        self._check(self.L.tm_sync(self.h))

    def tm_set_domain(self, box, phi: torch.Tensor, mu=None, rho=None, n_total: int = 0):
        ny, nx = phi.shape
        f = tm_fields(nx=nx, ny=ny, x0=box[0], y0=box[1], x1=box[2], y1=box[3],
                      phi=_ptr(phi), mu=_ptr(mu), rho=_ptr(rho))
        c, ha = ctypes.c_double(), ctypes.c_double()
        self._check(self.L.tm_set_domain(self.h, ctypes.byref(f), int(n_total), ctypes.byref(c), ctypes.byref(ha)))
        self.c, self.h_avg = c.value, ha.value
        return self.c, self.h_avg

    def tm_grid_bin(self, x, y, n_owned: Optional[int] = None, gid=None):
        n = x.shape[0]
        self._check(self.L.tm_grid_bin(self.h, _ptr(x), _ptr(y), n, n if n_owned is None else n_owned, _ptr(gid)))

    def tm_voronoi_delaunay(self, tri, n_tri, adj=None, deg=None, d_prev=None, x_out=None, y_out=None,
                            d_prev_out=None, status=None):
        self._check(self.L.tm_voronoi_delaunay(self.h, _ptr(tri), tri.shape[0], _ptr(n_tri), _ptr(adj), _ptr(deg),
                                               _ptr(d_prev), _ptr(x_out), _ptr(y_out), _ptr(d_prev_out),
                                               _ptr(status)))

    def tm_cvd_step(self, d_prev, x_hat, y_hat):
        self._check(self.L.tm_cvd_step(self.h, _ptr(d_prev), _ptr(x_hat), _ptr(y_hat)))

    def tm_distmesh_sums(self, adj, deg, sums2):
        self._check(self.L.tm_distmesh_sums(self.h, _ptr(adj), _ptr(deg), _ptr(sums2)))

    def tm_distmesh_step(self, adj, deg, sums2, fixed, d_prev, x_out, y_out, d_prev_out, status):
        self._check(self.L.tm_distmesh_step(self.h, _ptr(adj), _ptr(deg), _ptr(sums2), _ptr(fixed), _ptr(d_prev),
                                            _ptr(x_out), _ptr(y_out), _ptr(d_prev_out), _ptr(status)))

    def tm_project_sdf(self, x_old, y_old, x_hat, y_hat, x_out, y_out, d_prev_out, status):
        self._check(self.L.tm_project_sdf(self.h, _ptr(x_old), _ptr(y_old), _ptr(x_hat), _ptr(y_hat),
                                          x_old.shape[0], _ptr(x_out), _ptr(y_out), _ptr(d_prev_out), _ptr(status)))

    def tm_mesh_stats(self, x, y, tri, n_tri: int) -> tm_stats:
        s = tm_stats()
        self._check(self.L.tm_mesh_stats(self.h, _ptr(x), _ptr(y), _ptr(tri), int(n_tri), ctypes.byref(s)))
        return s

    def tm_move_count(self, x_old, y_old, d_prev, d_count):
        self._check(self.L.tm_move_count(self.h, _ptr(x_old), _ptr(y_old), _ptr(d_prev), int(x_old.shape[0]),
                                         _ptr(d_count)))

    def tm_set_n_total(self, n_total: int):
        c, ha = ctypes.c_double(), ctypes.c_double()
        self._check(self.L.tm_set_n_total(self.h, int(n_total), ctypes.byref(c), ctypes.byref(ha)))
        self.c, self.h_avg = c.value, ha.value
        return self.c, self.h_avg

    def tm_point_addition(self, tri, n_tri: int, x, y, n_add: int, x_new, y_new) -> float:
        r = ctypes.c_double()
        self._check(self.L.tm_point_addition(self.h, _ptr(tri), int(n_tri), _ptr(x), _ptr(y), int(n_add),
                                             _ptr(x_new), _ptr(y_new), ctypes.byref(r)))
        return r.value

    def tm_geometry_categories(self, nxg: int, nyg: int, cat):
        self._check(self.L.tm_geometry_categories(self.h, int(nxg), int(nyg), _ptr(cat)))

    def tm_contour_sdf(self, segs, nx: int, ny: int, box, phi):
        self._check(self.L.tm_contour_sdf(self.h, _ptr(segs), int(segs.shape[0]), int(nx), int(ny), box[0], box[1],
                                          box[2], box[3], _ptr(phi)))

    def tm_sdf_combine(self, op: int, a, b, out):
        self._check(self.L.tm_sdf_combine(self.h, int(op), _ptr(a), _ptr(b), int(a.numel()), _ptr(out)))

    def tm_init_points(self, nxg: int, nyg: int, cat, n_init: float, eta: float, seed: int, counts, x=None, y=None,
                       cap: int = 0) -> int:
        n = ctypes.c_int64()
        self._check(self.L.tm_init_points(self.h, int(nxg), int(nyg), _ptr(cat), float(n_init), float(eta), int(seed),
                                          _ptr(counts), _ptr(x), _ptr(y), int(cap), ctypes.byref(n)))
        return int(n.value)

    def tm_adf_build(self, segs, nxg: int, nyg: int, cat, fac_etol=0.1, fac_pt=1.0, max_depth=10):
        nn, nl = ctypes.c_int64(), ctypes.c_int64()
        self._check(self.L.tm_adf_build(self.h, _ptr(segs), int(segs.shape[0]), int(nxg), int(nyg), _ptr(cat),
                                        float(fac_etol), float(fac_pt), int(max_depth), ctypes.byref(nn),
                                        ctypes.byref(nl)))
        return nn.value, nl.value

    def tm_adf_eval(self, x, y, out):
        self._check(self.L.tm_adf_eval(self.h, _ptr(x), _ptr(y), int(x.shape[0]), _ptr(out)))

    def tm_x_histogram(self, x, d_n_addr, cap: int, x0: float, x1: float, hist):
        self._check(self.L.tm_x_histogram(self.h, _ptr(x), None if d_n_addr is None else ctypes.c_void_p(int(d_n_addr)),
                                          int(cap), float(x0), float(x1), int(hist.shape[0]), _ptr(hist)))

    def tm_density_from_sizing(self, mu, rho):
        self._check(self.L.tm_density_from_sizing(self.h, _ptr(mu), int(mu.numel()), _ptr(rho)))

    def tm_adjacency_export(self, adj, deg, adj_out, deg_out):
        self._check(self.L.tm_adjacency_export(self.h, _ptr(adj), _ptr(deg), _ptr(adj_out), _ptr(deg_out)))

    def tm_work_counts(self) -> tm_work:
        w = tm_work()
        self._check(self.L.tm_work_counts(self.h, ctypes.byref(w)))
        return w

    def tm_halo_pack(self, x, y, gid, n_owned, lo, hi, width, send_lo, send_hi, cap, cnt2):
        self._check(self.L.tm_halo_pack(self.h, _ptr(x), _ptr(y), _ptr(gid), int(n_owned), lo, hi, width,
                                        _ptr(send_lo), _ptr(send_hi), int(cap), _ptr(cnt2)))

    def tm_migrate_pack(self, x, y, gid, d_prev, n_owned, lo, hi, out_lo, out_hi, cap, cnt3):
        self._check(self.L.tm_migrate_pack(self.h, _ptr(x), _ptr(y), _ptr(gid), _ptr(d_prev), int(n_owned), lo, hi,
                                           _ptr(out_lo), _ptr(out_hi), int(cap), _ptr(cnt3)))

    def tm_refresh_positions(self, x, y):
        self._check(self.L.tm_refresh_positions(self.h, _ptr(x), _ptr(y)))

    def tm_retria_check(self, x_new, y_new, flag):
        self._check(self.L.tm_retria_check(self.h, _ptr(x_new), _ptr(y_new), _ptr(flag)))

    # CUDA Graphs: record a sequence of calls once, replay it (same buffers, same arguments)
    def capture(self, fn) -> "Graph":
        """Run fn() under stream capture and return the instantiated graph.  fn must issue
        library calls (and torch work) on this context's stream only, must not synchronise
        and must not grow any buffer (run it once before, as a warm-up)."""
        self._check(self.L.tm_graph_begin(self.h))
        try:
            fn()
        except BaseException:
            g = ctypes.c_void_p()
            self.L.tm_graph_end(self.h, ctypes.byref(g))
            if g.value:
                self.L.tm_graph_destroy(g)
            raise
        g = ctypes.c_void_p()
        self._check(self.L.tm_graph_end(self.h, ctypes.byref(g)))
        return Graph(self, g)

    # device-count variants (strip path without host synchronisation); *_p arguments are raw
    # device addresses (int), e.g. a message header inside a byte buffer
    def tm_grid_bin_dc(self, x, y, cap_local, counts, gid):
        self._check(self.L.tm_grid_bin_dc(self.h, _ptr(x), _ptr(y), int(cap_local), _ptr(counts), _ptr(gid)))

    def tm_halo_pack_dc(self, x, y, gid, n_owned_p, cap_owned, lo, hi, width, send_lo_p, send_hi_p, cap, cnt_lo_p,
                        cnt_hi_p):
        self._check(self.L.tm_halo_pack_dc(self.h, _ptr(x), _ptr(y), _ptr(gid), _addr(n_owned_p), int(cap_owned), lo,
                                           hi, width, _addr(send_lo_p), _addr(send_hi_p), int(cap), _addr(cnt_lo_p),
                                           _addr(cnt_hi_p)))

    def tm_migrate_pack_dc(self, x, y, gid, d_prev, n_owned_p, cap_owned, lo, hi, out_lo_p, out_hi_p, cap, cnt_lo_p,
                           cnt_hi_p):
        self._check(self.L.tm_migrate_pack_dc(self.h, _ptr(x), _ptr(y), _ptr(gid), _ptr(d_prev), _addr(n_owned_p),
                                              int(cap_owned), lo, hi, _addr(out_lo_p), _addr(out_hi_p), int(cap),
                                              _addr(cnt_lo_p), _addr(cnt_hi_p)))

    def tm_append_points(self, x, y, gid, d_prev, count_p, cap, msg_p, msg_count_p, msg_cap):
        self._check(self.L.tm_append_points(self.h, _ptr(x), _ptr(y), _ptr(gid), _ptr(d_prev), _addr(count_p),
                                            int(cap), _addr(msg_p), _addr(msg_count_p), int(msg_cap)))


class Graph:
    """An instantiated capture of library calls (tm_graph); launch() replays it."""

    def __init__(self, ctx: "Context", handle):
        self.ctx, self.h = ctx, handle

    def launch(self):
        self.ctx._check(self.ctx.L.tm_graph_launch(self.ctx.h, self.h))

    def close(self):
        if self.h:
            self.ctx.L.tm_graph_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ------------------------------------------------------------------ driver
@dataclass
class IterBuffers:
    """Device buffers for one iteration on n points (allocated once)."""
    n: int
    tri: torch.Tensor
    n_tri: torch.Tensor
    adj: torch.Tensor
    deg: torch.Tensor
    sums2: torch.Tensor
    status: torch.Tensor

    @classmethod
    def alloc(cls, n: int, adj_stride: int = 16, device="cuda"):
        return cls(n=n,
                   tri=torch.empty((2 * n + 64, 3), dtype=torch.int32, device=device),
                   n_tri=torch.zeros(1, dtype=torch.int64, device=device),
                   adj=torch.empty((adj_stride, n), dtype=torch.int32, device=device),
                   deg=torch.empty(n, dtype=torch.uint8, device=device),
                   sums2=torch.empty(2, dtype=torch.float64, device=device),
                   status=torch.empty(n, dtype=torch.int8, device=device))


class LazyDistMesh:
    """NEXT-1: DistMesh with lazy re-triangulation (Alg. 1): the Voronoi/Delaunay
    step runs only in an iteration after some point moved more than fac_retria h since the
    last triangulation; the other iterations reuse its ELL rows at the current
    positions (tm_refresh_positions).  One 4-byte device-to-host read per iteration (the
    re-triangulation flag decides which calls the next iteration issues)."""

    def __init__(self, ctx: "Context", n: int):
        self.ctx = ctx
        self.bufs = IterBuffers.alloc(n, ctx.params.adj_stride)
        self.flag = torch.zeros(1, dtype=torch.int32, device="cuda")
        self.retria = True
        self.triangulations = 0

    def step(self, x, y, d_prev, x_out, y_out, d_prev_out):
        c, b = self.ctx, self.bufs
        if self.retria:
            c.tm_grid_bin(x, y)
            c.tm_voronoi_delaunay(b.tri, b.n_tri, b.adj, b.deg)
            self.triangulations += 1
        else:
            c.tm_refresh_positions(x, y)
        c.tm_distmesh_sums(b.adj, b.deg, b.sums2)
        c.tm_distmesh_step(b.adj, b.deg, b.sums2, None, d_prev, x_out, y_out, d_prev_out, b.status)
        self.flag.zero_()
        c.tm_retria_check(x_out, y_out, self.flag)
        self.retria = bool(self.flag.item())
        return self.retria


def iterate(ctx: Context, x, y, d_prev, mode: str, bufs: IterBuffers, x_out, y_out, d_prev_out):
    """One TriMe++ iteration (Procedure 1 + Alg. 2 or Alg. 1 with retriangulation
    every iteration, L5) on device tensors; all work is issued to ctx.stream.
    Returns nothing; triangles are in bufs.tri[:bufs.n_tri]."""
    ctx.tm_grid_bin(x, y)
    if mode == "cvd":
        ctx.tm_voronoi_delaunay(bufs.tri, bufs.n_tri, None, None, d_prev, x_out, y_out, d_prev_out, bufs.status)
    elif mode == "dm":
        ctx.tm_voronoi_delaunay(bufs.tri, bufs.n_tri, bufs.adj, bufs.deg)
        ctx.tm_distmesh_sums(bufs.adj, bufs.deg, bufs.sums2)
        ctx.tm_distmesh_step(bufs.adj, bufs.deg, bufs.sums2, None, d_prev, x_out, y_out, d_prev_out, bufs.status)
    else:
        raise ValueError(mode)


# ---------------------------------------------------------------- NEXT-2 / NEXT-3
class Controller:
    """The library's iterate-to-termination controller (tm_control_init / tm_control_update)."""

    def __init__(self, n_total: int, n_current: int, method: str = "hybrid"):
        self.L = load_library()
        self.c = tm_control()
        m = {"cvd": TM_METHOD_CVD, "dm": TM_METHOD_DISTMESH, "distmesh": TM_METHOD_DISTMESH,
             "hybrid": TM_METHOD_HYBRID}[method]
        self.L.tm_control_init(ctypes.byref(self.c), int(n_total), int(n_current), m)

    @property
    def mode(self) -> str:
        return "cvd" if self.c.mode == TM_METHOD_CVD else "dm"

    def update(self, stats: tm_stats, move_count: int):
        k = ctypes.c_int64(0)
        a = self.L.tm_control_update(ctypes.byref(self.c), ctypes.byref(stats), int(move_count), ctypes.byref(k))
        return TM_ACT_NAMES[a], int(k.value)


@dataclass
class MeshResult:
    x: torch.Tensor
    y: torch.Tensor
    tri: torch.Tensor
    iterations: int
    history: list


def mesh(ctx: Context, x, y, n_total: Optional[int] = None, method: str = "hybrid", max_iterations: int = 1000,
         on_iteration=None) -> MeshResult:
    """Mesh to termination (NEXT-2/NEXT-3): iterate (Procedure 1 +
    Alg. 1 or Alg. 2), read the quality of (T_n, p_n) and the movement count, and let the
    library's controller add points, switch DistMesh -> CVD, or stop.  x, y: the N_current
    initial points (device); n_total: N_total (default: no point addition).  ctx's domain must
    have been set for n_total = len(x) (c follows N_current).  Returns the final points, the
    last iteration's kept triangles (at the positions it was computed from) and a per-iteration
    history.  on_iteration(dict) runs after each iteration and decision, before points are added
    (tests: the iteration's inputs, outputs, triangles and the controller's action)."""
    n = int(x.shape[0])
    n_total = int(n_total or n)
    ctl = Controller(n_total, n, method)
    ctl.c.max_iterations = int(max_iterations)
    bufs = IterBuffers.alloc(n, ctx.params.adj_stride, device=x.device)
    cnt = torch.zeros(1, dtype=torch.int64, device=x.device)
    dp = None
    hist = []
    it = 0
    tri_last = None
    while True:
        mode = ctl.mode
        xo, yo, do = torch.empty_like(x), torch.empty_like(x), torch.empty_like(x)
        iterate(ctx, x, y, dp, mode, bufs, xo, yo, do)
        ctx.tm_move_count(x, y, do, cnt)
        nt = int(bufs.n_tri.item())
        st = ctx.tm_mesh_stats(x, y, bufs.tri, nt)
        action, k = ctl.update(st, int(cnt.item()))
        hist.append({"it": it, "mode": mode, "n": n, "n_tri": nt, "action": action, "n_add": k,
                     "half_alpha": (st.sum_sqrt_alpha / nt) ** 2, "half_beta": (st.sum_sqrt_beta / nt) ** 2,
                     "max_alpha": st.max_alpha, "moves": int(cnt.item())})
        if on_iteration is not None:
            on_iteration({"it": it, "mode": mode, "x": x, "y": y, "d_prev_in": dp, "x_out": xo, "y_out": yo,
                          "d_prev_out": do, "status": bufs.status[:n], "tri": bufs.tri[:nt], "action": action,
                          "n_add": k, "moves": int(cnt.item()), "stats": st})
        it += 1
        if action.startswith("terminate"):
            tri_last = bufs.tri[:nt].clone()
            x, y = xo, yo
            break
        if action == "add":
            x2 = torch.empty(n + k, dtype=x.dtype, device=x.device)
            y2 = torch.empty_like(x2)
            d2 = torch.full((n + k,), -1.0, dtype=x.dtype, device=x.device)  # new points: no previous move
            x2[:n].copy_(xo)
            y2[:n].copy_(yo)
            d2[:n].copy_(do)
            # centroids of the mesh (T_n, p_n) (reading L46)
            ctx.tm_point_addition(bufs.tri, nt, x, y, k, x2[n:], y2[n:])
            n += k
            ctx.tm_set_n_total(n)
            bufs = IterBuffers.alloc(n, ctx.params.adj_stride, device=x.device)
            x, y, dp = x2, y2, d2
        else:
            x, y, dp = xo, yo, do
    return MeshResult(x, y, tri_last, it, hist)


# ---------------------------------------------------------------- NEXT-4
def geometry_grid_dims(n_total: int, box, n_opt: float = 3.3, fac_grid: int = 5):
    """P:338-346 (host arithmetic of the library)."""
    nx, ny = ctypes.c_int32(), ctypes.c_int32()
    load_library().tm_geometry_grid_dims(int(n_total), float(n_opt), int(fac_grid), box[0], box[1], box[2], box[3],
                                         ctypes.byref(nx), ctypes.byref(ny))
    return nx.value, ny.value


def initial_points(ctx: Context, n_init: int, nxg: int, nyg: int, eta: float = 0.5, seed: int = 0):
    """geometry-grid categories, Floyd-Steinberg counts and the initial points (device)."""
    dev = torch.device("cuda", ctx.device)
    cat = torch.empty(nyg * nxg, dtype=torch.int8, device=dev)
    ctx.tm_geometry_categories(nxg, nyg, cat)
    counts = torch.empty(nyg * nxg, dtype=torch.int32, device=dev)
    n = ctx.tm_init_points(nxg, nyg, cat, n_init, eta, seed, counts)
    x = torch.empty(n, dtype=torch.float64, device=dev)
    y = torch.empty_like(x)
    ctx.tm_init_points(nxg, nyg, cat, n_init, eta, seed, counts, x, y, n)
    return x, y, cat.view(nyg, nxg), counts.view(nyg, nxg)


def automatic_sizing(ctx: Context, segs, box, nx: int, ny: int, K: float, d_s: float, geps_hat: float,
                     r_nei: float, n_thres: int = 3):
    """P:356-373 on the GPU: boundary points of the contour (App. A), their medial-axis poles
    (trimmed), lfs and the sizing field mu on the (ny, nx) node grid over box.  Returns
    (mu, (sx, sy), (mx, my), lfs) as device tensors."""
    dev = segs.device
    n = ctypes.c_int64()
    L = ctx.L
    ctx._check(L.tm_boundary_points(ctx.h, _ptr(segs), int(segs.shape[0]), float(d_s), float(geps_hat), None, None, 0,
                                    ctypes.byref(n)))
    sx = torch.empty(n.value, dtype=torch.float64, device=dev)
    sy = torch.empty_like(sx)
    ctx._check(L.tm_boundary_points(ctx.h, _ptr(segs), int(segs.shape[0]), float(d_s), float(geps_hat), _ptr(sx),
                                    _ptr(sy), n.value, ctypes.byref(n)))
    cap = 2 * sx.shape[0] + 16
    mx = torch.empty(cap, dtype=torch.float64, device=dev)
    my = torch.empty_like(mx)
    m = ctypes.c_int64()
    ctx._check(L.tm_medial_points(ctx.h, _ptr(sx), _ptr(sy), int(sx.shape[0]), box[0], box[1], box[2], box[3],
                                  float(r_nei), int(n_thres), _ptr(mx), _ptr(my), cap, ctypes.byref(m)))
    mx, my = mx[:m.value].contiguous(), my[:m.value].contiguous()
    mu = torch.empty(ny, nx, dtype=torch.float64, device=dev)
    lfs = torch.empty_like(sx)
    ctx._check(L.tm_sizing_field(ctx.h, _ptr(sx), _ptr(sy), int(sx.shape[0]), _ptr(mx), _ptr(my), int(mx.shape[0]),
                                 float(K), int(nx), int(ny), box[0], box[1], box[2], box[3], _ptr(mu), _ptr(lfs)))
    return mu, (sx, sy), (mx, my), lfs
