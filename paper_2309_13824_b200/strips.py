"""x-strip domain decomposition of one meshing iteration over P ranks
(the paper's MPI distribution is future work).

Rank r owns the points with x in [X_r, X_{r+1}).  Per iteration:
  1. halo: every rank sends the owned points within W of each strip edge to
     the neighbour across it (x, y, gid), W = 2 * S_max = 2 * fac_voro * h_max
     (a cell lies inside its octagon of circumradius S, so only points within
     2S can cut it);
  2. the rank bins owned + ghosts (tm_grid_bin with n_owned < n_local and the
     global ids) and computes cells for its OWNED points only; a triangle is
     emitted by the owner of its smallest-id vertex, so every triangle appears
     exactly once over all ranks;
  3. (DistMesh) the two edge sums are all-reduced (each edge counted by the
     rank owning its smaller-id endpoint);
  4. migrate: updated points that left the strip go to the neighbour.

The arithmetic runs in the backend (GpuStripBackend: the C-ABI kernels); the
exchange runs in an exchanger: TorchP2P (torch.distributed send/recv, NCCL
over NVLink on GPUs or gloo on CPU) or Loopback (P ranks inside one process,
for single-GPU emulation and tests).  This module only orchestrates.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional

import torch


@dataclass
class Strips:
    """P x-strips of [x0, x1): equal widths, or explicit interior cuts
    (e.g. x-quantiles of the points, for adaptive densities)."""
    x0: float
    x1: float
    P: int
    cuts: Optional[List[float]] = None  # P-1 increasing interior boundaries

    @classmethod
    def from_quantiles(cls, x: torch.Tensor, P: int, x0: float, x1: float) -> "Strips":
        if P == 1:
            return cls(x0, x1, 1)
        q = torch.quantile(x.double().cpu()[:: max(1, x.shape[0] // 1_000_000)],
                           torch.linspace(0, 1, P + 1, dtype=torch.float64)[1:-1])
        return cls(x0, x1, P, [float(v) for v in q])

    def _cut(self, k: int) -> float:
        if self.cuts is not None:
            return self.cuts[k - 1]
        return self.x0 + k * (self.x1 - self.x0) / self.P

    def bounds(self, r: int):
        lo = self._cut(r) if r > 0 else float("-inf")
        hi = self._cut(r + 1) if r < self.P - 1 else float("inf")
        return lo, hi

    def check_width(self, W: float):
        """Ghosts travel one strip only (to r-1 and r+1), so every interior strip must be at
        least as wide as the halo W = 2 S_max: a point two strips away is then at least W >=
        2 S_i from any cell it could otherwise cut (C_i lies in Oct_i, circumradius S_i).
        Narrower strips would silently lose cells and triangles -- fail loudly instead."""
        for r in range(1, self.P - 1):
            lo, hi = self.bounds(r)
            if not hi - lo >= W:
                raise ValueError(f"strip {r} of {self.P} is {hi - lo:.3g} wide, narrower than the halo width "
                                 f"W = {W:.3g}: use fewer strips (ghosts only reach the neighbouring strips)")

    def owner(self, x: torch.Tensor) -> torch.Tensor:
        if self.cuts is not None:
            c = torch.tensor(self.cuts, dtype=x.dtype, device=x.device)
            return torch.bucketize(x, c, right=True).to(torch.int64)
        w = (self.x1 - self.x0) / self.P
        return torch.clamp(((x - self.x0) / w).floor().to(torch.int64), 0, self.P - 1)


@dataclass
class RankState:
    """Owned points of one rank (device or host tensors)."""
    rank: int
    x: torch.Tensor
    y: torch.Tensor
    gid: torch.Tensor          # int32 global ids
    d_prev: Optional[torch.Tensor] = None
    tri: Optional[torch.Tensor] = None   # triangles emitted by this rank (global ids)
    extra: dict = field(default_factory=dict)


def split_initial(x, y, strips: Strips, rank: int, d_prev=None) -> RankState:
    own = strips.owner(x) == rank
    gid = torch.nonzero(own, as_tuple=False).flatten().to(torch.int32)
    return RankState(rank, x[own].contiguous(), y[own].contiguous(), gid.contiguous(),
                     None if d_prev is None else d_prev[own].contiguous())


# ---------------------------------------------------------------- exchangers
class TorchP2P:
    """Neighbour exchange with torch.distributed (NCCL or gloo): counts first,
    then the SoA payload, to ranks r-1 and r+1 (grouped send/recv)."""

    def __init__(self, rank: int, world: int, device):
        self.rank, self.world, self.device = rank, world, device

    def _pair(self, send: List[Optional[torch.Tensor]], recv_like):
        import torch.distributed as dist
        ops, recv = [], [None, None]
        nbr = [self.rank - 1, self.rank + 1]
        for side in (0, 1):
            if 0 <= nbr[side] < self.world:
                ops.append(dist.P2POp(dist.isend, send[side], nbr[side]))
                recv[side] = recv_like(side)
                ops.append(dist.P2POp(dist.irecv, recv[side], nbr[side]))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        return recv

    def exchange(self, to_lo: List[torch.Tensor], to_hi: List[torch.Tensor]):
        """to_lo/to_hi: lists of 1-D tensors of equal length (same dtypes on both sides).
        Returns (from_lo, from_hi) lists (None where there is no neighbour).  Two rounds:
        the element counts, then every array of a side packed into one byte buffer."""
        dev = self.device
        n = [torch.tensor([to_lo[0].shape[0]], dtype=torch.int64, device=dev),
             torch.tensor([to_hi[0].shape[0]], dtype=torch.int64, device=dev)]
        cnt = self._pair(n, lambda s: torch.empty(1, dtype=torch.int64, device=dev))
        dts = [t.dtype for t in to_lo]
        esz = [torch.empty(0, dtype=d).element_size() for d in dts]
        order = sorted(range(len(dts)), key=lambda i: -esz[i])  # widest first: every view stays aligned

        def pack(lst):
            if not lst[0].numel():
                return torch.empty(0, dtype=torch.uint8, device=dev)
            return torch.cat([lst[i].contiguous().view(torch.uint8) for i in order])
        k = [None if c is None else int(c.item()) for c in cnt]
        got = self._pair([pack(to_lo), pack(to_hi)],
                         lambda s: torch.empty(k[s] * sum(esz), dtype=torch.uint8, device=dev))
        out = [None, None]
        for side in (0, 1):
            if got[side] is None:
                continue
            parts, off = [None] * len(dts), 0
            for i in order:
                parts[i] = got[side][off:off + k[side] * esz[i]].view(dts[i])
                off += k[side] * esz[i]
            out[side] = parts
        return out[0], out[1]

    def allreduce_sum(self, t: torch.Tensor):
        import torch.distributed as dist
        if self.world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return t


class Loopback:
    """P ranks in one process: exchange() is called once per rank in order with
    the same call pattern; messages are parked until the matching rank reads."""

    def __init__(self, P: int):
        self.P = P
        self.box = {}

    def view(self, rank: int):
        return _LoopbackView(self, rank)


class _LoopbackView:
    def __init__(self, lb: Loopback, rank: int):
        self.lb, self.rank = lb, rank

    def post(self, tag, to_lo, to_hi):
        if self.rank > 0:
            self.lb.box[(tag, self.rank, self.rank - 1)] = [t.clone() for t in to_lo]
        if self.rank < self.lb.P - 1:
            self.lb.box[(tag, self.rank, self.rank + 1)] = [t.clone() for t in to_hi]

    def collect(self, tag):
        a = self.lb.box.pop((tag, self.rank - 1, self.rank), None)
        b = self.lb.box.pop((tag, self.rank + 1, self.rank), None)
        return a, b


# ---------------------------------------------------------------- backend (GPU)
class GpuStripBackend:
    """The per-rank arithmetic through the C ABI (no CPU work)."""

    def __init__(self, ctx, adj_stride=16, keep_tri=True, adaptive_halo=True):
        self.ctx = ctx
        self.adj_stride = adj_stride
        self.adaptive_halo = adaptive_halo  # per-point halo width from the Lipschitz bound of mu~
        self.keep_tri = keep_tri  # False: leave the triangles in the device buffers (no count readback)
        self.bufs = {}

    def _buf(self, name, numel, dtype, dev):
        """Persistent scratch (grown on demand): no per-iteration allocation."""
        b = self.bufs.get(name)
        if b is None or b.numel() < numel or b.device != dev:
            b = torch.empty(int(numel * 1.125) + 1024, dtype=dtype, device=dev)
            self.bufs[name] = b
        return b

    def halo(self, st: RankState, lo, hi, W):
        dev = st.x.device
        n = st.x.shape[0]
        cap = n
        send_lo = self._buf("send_lo", 3 * cap + 1, torch.float64, dev)
        send_hi = self._buf("send_hi", 3 * cap + 1, torch.float64, dev)
        cnt = self._buf("hcnt", 2, torch.int64, dev)[:2]
        self.ctx.tm_halo_pack(st.x, st.y, st.gid, n, lo if lo > -1e300 else -1e300, hi if hi < 1e300 else 1e300,
                              -W if self.adaptive_halo else W, send_lo, send_hi, cap, cnt)
        c = cnt.tolist()

        def seg(buf, k):
            return [buf[:k].clone(), buf[cap:cap + k].clone(),
                    buf[2 * cap:2 * cap + (k + 1) // 2 + 1].view(torch.int32)[:k].clone()]
        return seg(send_lo, c[0]), seg(send_hi, c[1])

    def cells_begin(self, st: RankState, ghosts, mode: str):
        """Bin owned + ghosts, compute the owned cells.  CVD completes here;
        DistMesh stops after pass 1 and returns its local edge sums."""
        import paper_2309_13824_b200 as T
        xs = [st.x] + [g[0] for g in ghosts if g is not None]
        ys = [st.y] + [g[1] for g in ghosts if g is not None]
        gs = [st.gid] + [g[2] for g in ghosts if g is not None]
        xl, yl, gl = torch.cat(xs).contiguous(), torch.cat(ys).contiguous(), torch.cat(gs).contiguous()
        n_own, n_loc = st.x.shape[0], xl.shape[0]
        ctx = self.ctx
        ctx.tm_grid_bin(xl, yl, n_own, gl)
        bufs = T.IterBuffers.alloc(n_loc, self.adj_stride, device=xl.device)
        h = {"bufs": bufs, "st": st, "mode": mode,
             "xo": torch.empty(n_own, dtype=torch.float64, device=xl.device)}
        h["yo"], h["do"] = torch.empty_like(h["xo"]), torch.empty_like(h["xo"])
        h["status"] = torch.empty(n_own, dtype=torch.int8, device=xl.device)
        if mode == "cvd":
            ctx.tm_voronoi_delaunay(bufs.tri, bufs.n_tri, None, None, st.d_prev, h["xo"], h["yo"], h["do"],
                                    h["status"])
            return h, None
        ctx.tm_voronoi_delaunay(bufs.tri, bufs.n_tri, bufs.adj, bufs.deg)
        ctx.tm_distmesh_sums(bufs.adj, bufs.deg, bufs.sums2)
        return h, bufs.sums2

    def cells_end(self, h, sums2=None):
        bufs, st = h["bufs"], h["st"]
        if h["mode"] == "dm":
            if sums2 is not None and sums2 is not bufs.sums2:
                bufs.sums2.copy_(sums2)
            self.ctx.tm_distmesh_step(bufs.adj, bufs.deg, bufs.sums2, None, st.d_prev, h["xo"], h["yo"], h["do"],
                                      h["status"])
        if not self.keep_tri:
            return None, h["xo"], h["yo"], h["do"], h["status"]
        nt = int(bufs.n_tri.item())
        return bufs.tri[:nt].clone(), h["xo"], h["yo"], h["do"], h["status"]

    def migrate(self, st: RankState, lo, hi):
        """Partition the updated owned points (stable, in place in st's arrays,
        which this iteration produced): kept ones stay at the front, leavers are
        packed for the neighbours."""
        dev = st.x.device
        n = st.x.shape[0]
        out_lo = self._buf("out_lo", 4 * n + 1, torch.float64, dev)
        out_hi = self._buf("out_hi", 4 * n + 1, torch.float64, dev)
        cnt = self._buf("mcnt", 3, torch.int64, dev)[:3]
        dp = st.d_prev if st.d_prev is not None else torch.zeros(n, dtype=torch.float64, device=dev)
        x, y, g = st.x, st.y, st.gid.clone()  # gid is shared with the previous state
        self.ctx.tm_migrate_pack(x, y, g, dp, n, lo if lo > -1e300 else -1e300, hi if hi < 1e300 else 1e300,
                                 out_lo, out_hi, n, cnt)
        k, a, b = cnt.tolist()

        def seg(buf, m):
            return [buf[:m].clone(), buf[n:n + m].clone(),
                    buf[2 * n:2 * n + (m + 1) // 2 + 1].view(torch.int32)[:m].clone(), buf[3 * n:3 * n + m].clone()]
        keep = [x[:k], y[:k], g[:k], dp[:k]]
        return keep, seg(out_lo, a), seg(out_hi, b)


# ---------------------------------------------------------------- one iteration
def ghost_width(c: float, fac_voro: float = 5.0, mu_max: float = 1.0) -> float:
    """W = 2 S_max, S = fac_voro * h, h = c * mu (reading L34)."""
    return 2.0 * fac_voro * c * mu_max


def strip_iteration(st: RankState, strips: Strips, backend, exchange, W: float, mode: str = "cvd",
                    allreduce=None) -> RankState:
    """One iteration on one rank.  `exchange(to_lo, to_hi) -> (from_lo, from_hi)`
    performs the neighbour exchange (collective over the ranks)."""
    strips.check_width(W)
    lo, hi = strips.bounds(st.rank)
    h_lo, h_hi = backend.halo(st, lo, hi, W)
    g_lo, g_hi = exchange(h_lo, h_hi)
    hnd, sums2 = backend.cells_begin(st, [g_lo, g_hi], mode)
    if sums2 is not None and allreduce is not None:
        allreduce(sums2)
    tri, xo, yo, do, status = backend.cells_end(hnd, sums2)
    nst = RankState(st.rank, xo, yo, st.gid, do, tri)
    nst.extra["status"] = status
    keep, m_lo, m_hi = backend.migrate(nst, lo, hi)
    r_lo, r_hi = exchange(m_lo, m_hi)
    parts = [keep] + [r for r in (r_lo, r_hi) if r is not None]
    out = RankState(st.rank, torch.cat([p[0] for p in parts]).contiguous(),
                    torch.cat([p[1] for p in parts]).contiguous(),
                    torch.cat([p[2] for p in parts]).contiguous(),
                    torch.cat([p[3] for p in parts]).contiguous(), tri)
    out.extra["status"] = status
    out.extra["n_ghosts"] = sum(0 if g is None else g[0].shape[0] for g in (g_lo, g_hi))
    out.extra["n_migrated_in"] = sum(0 if r is None else r[0].shape[0] for r in (r_lo, r_hi))
    return out


def loopback_iteration(states: List[RankState], strips: Strips, backends, W: float, mode: str = "cvd"):
    """All P ranks of one iteration inside one process (single-GPU emulation).
    Phases are run rank by rank with messages parked in a mailbox; the DistMesh
    sums are reduced across ranks between the two passes."""
    P = len(states)
    strips.check_width(W)
    lb = Loopback(P)
    views = [lb.view(r) for r in range(P)]
    halos = []
    for r, st in enumerate(states):
        lo, hi = strips.bounds(r)
        h_lo, h_hi = backends[r].halo(st, lo, hi, W)
        views[r].post("halo", h_lo, h_hi)
    for r in range(P):
        halos.append(views[r].collect("halo"))
    begun = [backends[r].cells_begin(st, list(halos[r]), mode) for r, st in enumerate(states)]
    total = None
    if mode == "dm":  # all-reduce of the two DistMesh sums across the ranks
        total = sum(b[1] for b in begun)
    results = [backends[r].cells_end(begun[r][0], total) for r in range(P)]
    migr = []
    for r, st in enumerate(states):
        tri, xo, yo, do, status = results[r]
        nst = RankState(r, xo, yo, st.gid, do, tri)
        lo, hi = strips.bounds(r)
        keep, m_lo, m_hi = backends[r].migrate(nst, lo, hi)
        views[r].post("mig", m_lo, m_hi)
        migr.append((keep, status, tri))
    out = []
    for r in range(P):
        keep, status, tri = migr[r]
        r_lo, r_hi = views[r].collect("mig")
        parts = [keep] + [p for p in (r_lo, r_hi) if p is not None]
        s = RankState(r, torch.cat([p[0] for p in parts]).contiguous(), torch.cat([p[1] for p in parts]).contiguous(),
                      torch.cat([p[2] for p in parts]).contiguous(), torch.cat([p[3] for p in parts]).contiguous(), tri)
        s.extra["status"] = status
        out.append(s)
    return out
