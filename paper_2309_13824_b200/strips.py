"""x-strip domain decomposition of one meshing iteration over P ranks
(the paper's MPI distribution is future work).

Rank r owns the points with x in [X_r, X_{r+1}).  Per iteration:
  1. halo: every rank sends the owned points within W of each strip edge to
     the neighbour across it (x, y, gid), W = 2 * S_max = 2 * fac_voro * h_max
     (a cell lies inside its octagon of circumradius S, so only points within
     2S can cut it); strips narrower than W are refused (Strips.check_width);
  2. the rank bins owned + ghosts (global ids) and computes cells for its OWNED
     points only; a triangle is emitted by the owner of its smallest-id vertex,
     so every triangle appears exactly once over all ranks;
  3. (DistMesh) the two edge sums are all-reduced (each edge counted by the
     rank owning its smaller-id endpoint);
  4. migrate: updated points that left the strip go to the neighbour.

No host synchronisation inside an iteration: every message has a FIXED size
(capacity `cap_msg`, an int64 count header followed by SoA segments), the
counts live on the device, and the library's device-count calls
(tm_halo_pack_dc, tm_append_points, tm_grid_bin_dc, tm_migrate_pack_dc) take
them from there.  All buffers are allocated once (StripState).  Overflow of a
capacity is latched by the library and raised at the next synchronising call.

The arithmetic runs in a backend (GpuStripBackend: the C ABI; the CPU test
double in tests/strip_cpu_backend.py); the exchange runs in an exchanger:
TorchP2P (torch.distributed send/recv, NCCL over NVLink on GPUs or gloo on
CPU) or the in-process loopback of `loopback_step`.  This module orchestrates.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional

import torch

HALO_SEGS, MIG_SEGS = 3, 4  # message segments: x | y | gid (| d_prev)


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


def rebalanced_cuts(strips: "Strips", hist, W: float, max_shift: float = 0.5) -> "Strips":
    """Re-balanced strips from a global histogram of the owned x (nb equal bins of [x0, x1)): cut k
    at the k/P quantile (linear inside its bin), each cut moved by at most `max_shift` of the
    narrower strip beside it -- so every point changes owner to a neighbouring strip only and the
    migration step can carry it -- and strips kept at least W wide.  Host arithmetic on the
    (all-reduced, identical on every rank) counts: every rank computes the same cuts."""
    P = strips.P
    if P == 1:
        return strips
    h = [int(v) for v in hist]
    nb = len(h)
    tot = sum(h)
    old = [strips._cut(k) for k in range(1, P)]
    edges = [strips.x0] + old + [strips.x1]
    cum = [0]
    for v in h:
        cum.append(cum[-1] + v)
    new = []
    b = 0
    for k in range(1, P):
        target = tot * k / P
        while b < nb - 1 and cum[b + 1] < target:
            b += 1
        frac = 0.0 if h[b] == 0 else (target - cum[b]) / h[b]
        q = strips.x0 + (b + min(max(frac, 0.0), 1.0)) * (strips.x1 - strips.x0) / nb
        lim = max_shift * min(edges[k] - edges[k - 1], edges[k + 1] - edges[k])
        new.append(min(max(q, old[k - 1] - lim), old[k - 1] + lim))
    for k in range(1, P - 1):  # keep the interior strips at least W wide (then keep the old cuts)
        if new[k] - new[k - 1] < W:
            return strips
    return Strips(strips.x0, strips.x1, P, new)


def rebalance(S: "StripState", strips: "Strips", backend, comm, W: float, nb: int = 1024) -> "Strips":
    """Periodic strip re-balancing, between iterations: the global histogram of the
    owned x (one all-reduce of nb counts), new cuts (rebalanced_cuts), then one migration step
    with the new bounds on the current points.  Synchronises once (the counts to the host)."""
    hist = backend.x_histogram(S, strips.x0, strips.x1, nb)
    comm.allreduce_sum(hist)
    new = rebalanced_cuts(strips, hist.cpu().tolist(), W)
    lo, hi = new.bounds(S.rank)
    S.swap()  # the current points into the update's arrays, where migrate_pack works
    backend.migrate_pack(S, lo, hi)
    comm.exchange(S.m_send[0], S.m_send[1], S.m_recv[0], S.m_recv[1])
    backend.append_migrants(S)
    S.swap()
    return new


def ghost_width(c: float, fac_voro: float = 5.0, mu_max: float = 1.0) -> float:
    """W = 2 S_max, S = fac_voro * h, h = c * mu (reading L34)."""
    return 2.0 * fac_voro * c * mu_max


class Msg:
    """A fixed-size strip message: int64 count header, then `segs` SoA segments of `cap`
    (doubles; the gid segment holds int32).  Sent and received whole: the receiver never
    needs the count on the host."""

    def __init__(self, cap: int, segs: int, device):
        self.cap, self.segs = cap, segs
        self.buf = torch.zeros(1 + segs * cap, dtype=torch.float64, device=device)

    @property
    def header(self) -> torch.Tensor:
        return self.buf[:1].view(torch.int64)

    def addr(self) -> int:
        return self.buf.data_ptr()

    def payload_addr(self) -> int:
        return self.buf.data_ptr() + 8

    def count(self) -> int:  # tests / diagnostics only (synchronises)
        return int(self.header.item())

    def segment(self, k: int, n: int, dtype=torch.float64) -> torch.Tensor:
        seg = self.buf[1 + k * self.cap: 1 + (k + 1) * self.cap]
        return seg.view(torch.int32)[:n] if dtype == torch.int32 else seg[:n]


class StripState:
    """Persistent per-rank state: owned points at [0, n_owned), ghosts after them, with
    device counts {n_owned, n_local}; the update's outputs in a second set of arrays (swapped
    after migration); the four halo and four migration messages."""

    def __init__(self, rank: int, x: torch.Tensor, y: torch.Tensor, gid: torch.Tensor, cap_own: int, cap_msg: int,
                 d_prev: Optional[torch.Tensor] = None):
        dev = x.device
        n = x.shape[0]
        if n > cap_own:
            raise ValueError(f"rank {rank}: {n} owned points exceed the capacity {cap_own}")
        self.rank, self.cap_own, self.cap_msg = rank, cap_own, cap_msg
        self.cap_local = cap_own + 2 * cap_msg
        f64 = dict(dtype=torch.float64, device=dev)
        self.X, self.Y, self.D = (torch.zeros(self.cap_local, **f64) for _ in range(3))
        self.Xo, self.Yo, self.Do = (torch.zeros(self.cap_local, **f64) for _ in range(3))
        self.G = torch.zeros(self.cap_local, dtype=torch.int32, device=dev)
        self.status = torch.zeros(self.cap_local, dtype=torch.int8, device=dev)
        self.X[:n], self.Y[:n], self.G[:n] = x, y, gid
        self.have_dprev = d_prev is not None
        if d_prev is not None:
            self.D[:n] = d_prev
        self.counts = torch.tensor([n, n], dtype=torch.int64, device=dev)  # n_owned, n_local
        self.h_send = [Msg(cap_msg, HALO_SEGS, dev) for _ in range(2)]
        self.h_recv = [Msg(cap_msg, HALO_SEGS, dev) for _ in range(2)]
        self.m_send = [Msg(cap_msg, MIG_SEGS, dev) for _ in range(2)]
        self.m_recv = [Msg(cap_msg, MIG_SEGS, dev) for _ in range(2)]
        self.extra = {}

    def reset(self, x: torch.Tensor, y: torch.Tensor, gid: torch.Tensor, counts: torch.Tensor):
        """Restart from the given owned points (device copies, no host sync): counts is a
        device int64[2] {n, n}."""
        n = x.shape[0]
        self.X[:n], self.Y[:n], self.G[:n] = x, y, gid
        self.counts.copy_(counts)
        self.have_dprev = False

    def swap(self):
        self.X, self.Xo = self.Xo, self.X
        self.Y, self.Yo = self.Yo, self.Y
        self.D, self.Do = self.Do, self.D
        self.have_dprev = True

    def owned(self):
        """The owned points (host-visible views; synchronises): x, y, gid, d_prev."""
        n = int(self.counts[0].item())
        return self.X[:n], self.Y[:n], self.G[:n], (self.D[:n] if self.have_dprev else None)


def split_initial(x, y, strips: Strips, rank: int, cap_own: int, cap_msg: int, d_prev=None) -> StripState:
    own = strips.owner(x) == rank
    gid = torch.nonzero(own, as_tuple=False).flatten().to(torch.int32)
    return StripState(rank, x[own].contiguous(), y[own].contiguous(), gid.contiguous(), cap_own, cap_msg,
                      None if d_prev is None else d_prev[own].contiguous())


def capacities(n_total: int, P: int, n_ghost_est: int, slack: float = 1.15):
    """Owned and message capacities: the owned share with slack for migration, and a halo
    message sized for the estimated ghosts per side (at most the owned capacity)."""
    cap_own = int(slack * n_total / P) + 1024
    cap_msg = min(cap_own, int(4 * n_ghost_est) + 4096)
    return cap_own, cap_msg


# ---------------------------------------------------------------- exchangers
class TorchP2P:
    """Neighbour exchange of fixed-size messages with torch.distributed (NCCL or gloo):
    one grouped send/recv round per exchange; with NCCL the waits are stream-ordered (the
    host does not block)."""

    def __init__(self, rank: int, world: int, device):
        self.rank, self.world, self.device = rank, world, device

    def exchange(self, send_lo: Msg, send_hi: Msg, recv_lo: Msg, recv_hi: Msg):
        import torch.distributed as dist
        ops = []
        if self.rank > 0:
            ops += [dist.P2POp(dist.isend, send_lo.buf, self.rank - 1),
                    dist.P2POp(dist.irecv, recv_lo.buf, self.rank - 1)]
        if self.rank < self.world - 1:
            ops += [dist.P2POp(dist.isend, send_hi.buf, self.rank + 1),
                    dist.P2POp(dist.irecv, recv_hi.buf, self.rank + 1)]
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()

    def allreduce_sum(self, t: torch.Tensor):
        import torch.distributed as dist
        if self.world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return t


# ---------------------------------------------------------------- backend (GPU)
class GpuStripBackend:
    """The per-rank arithmetic through the C ABI (no CPU work, no host synchronisation)."""

    def __init__(self, ctx, adj_stride=16, adaptive_halo=True):
        import paper_2309_13824_b200 as T
        self.T = T
        self.ctx = ctx
        self.adj_stride = adj_stride
        self.adaptive_halo = adaptive_halo  # per-point halo width from the Lipschitz bound of mu~
        self.bufs = None

    def _bufs(self, S: StripState):
        if self.bufs is None or self.bufs.n != S.cap_local:
            self.bufs = self.T.IterBuffers.alloc(S.cap_local, self.adj_stride, device=S.X.device)
        return self.bufs

    def halo_pack(self, S: StripState, lo, hi, W):
        self.ctx.tm_halo_pack_dc(S.X, S.Y, S.G, S.counts.data_ptr(), S.cap_own, lo, hi,
                                 -W if self.adaptive_halo else W, S.h_send[0].payload_addr(),
                                 S.h_send[1].payload_addr(), S.cap_msg, S.h_send[0].addr(), S.h_send[1].addr())

    def append_ghosts(self, S: StripState):
        S.counts[1:2].copy_(S.counts[0:1])
        for m in S.h_recv:
            self.ctx.tm_append_points(S.X, S.Y, S.G, None, S.counts.data_ptr() + 8, S.cap_local, m.payload_addr(),
                                      m.addr(), m.cap)

    def cells_begin(self, S: StripState, mode: str):
        """Bin owned + ghosts, compute the owned cells.  CVD completes here; DistMesh stops
        after pass 1 and returns its local edge sums (device)."""
        c = self.ctx
        b = self._bufs(S)
        c.tm_grid_bin_dc(S.X, S.Y, S.cap_local, S.counts, S.G)
        if mode == "cvd":
            c.tm_voronoi_delaunay(b.tri, b.n_tri, None, None, S.D if S.have_dprev else None, S.Xo, S.Yo, S.Do,
                                  S.status)
            return None
        c.tm_voronoi_delaunay(b.tri, b.n_tri, b.adj, b.deg)
        c.tm_distmesh_sums(b.adj, b.deg, b.sums2)
        return b.sums2

    def cells_end(self, S: StripState, mode: str, sums2=None):
        if mode != "dm":
            return
        b = self.bufs
        if sums2 is not None and sums2 is not b.sums2:
            b.sums2.copy_(sums2)
        self.ctx.tm_distmesh_step(b.adj, b.deg, b.sums2, None, S.D if S.have_dprev else None, S.Xo, S.Yo, S.Do,
                                  S.status)

    def migrate_pack(self, S: StripState, lo, hi):
        """Owned outputs that left the strip go to the messages; the rest are compacted in
        place (Xo, Yo, G, Do) and counts[0] becomes the kept count."""
        self.ctx.tm_migrate_pack_dc(S.Xo, S.Yo, S.G, S.Do, S.counts.data_ptr(), S.cap_own, lo, hi,
                                    S.m_send[0].payload_addr(), S.m_send[1].payload_addr(), S.cap_msg,
                                    S.m_send[0].addr(), S.m_send[1].addr())

    def append_migrants(self, S: StripState):
        for m in S.m_recv:
            self.ctx.tm_append_points(S.Xo, S.Yo, S.G, S.Do, S.counts.data_ptr(), S.cap_own, m.payload_addr(),
                                      m.addr(), m.cap)

    def x_histogram(self, S: StripState, x0: float, x1: float, nb: int) -> torch.Tensor:
        h = torch.empty(nb, dtype=torch.int64, device=S.X.device)
        self.ctx.tm_x_histogram(S.X, S.counts.data_ptr(), S.cap_own, x0, x1, h)
        return h

    def triangles(self):
        """This rank's emitted triangles (global ids; synchronises)."""
        nt = int(self.bufs.n_tri.item())
        return self.bufs.tri[:nt]


# ---------------------------------------------------------------- one iteration
def strip_step(S: StripState, strips: Strips, backend, comm, W: float, mode: str = "cvd"):
    """One iteration on one rank; `comm` is a TorchP2P (collective over the ranks)."""
    strips.check_width(W)
    lo, hi = strips.bounds(S.rank)
    backend.halo_pack(S, lo, hi, W)
    comm.exchange(S.h_send[0], S.h_send[1], S.h_recv[0], S.h_recv[1])
    backend.append_ghosts(S)
    sums2 = backend.cells_begin(S, mode)
    if sums2 is not None:
        comm.allreduce_sum(sums2)
    backend.cells_end(S, mode, sums2)
    backend.migrate_pack(S, lo, hi)
    comm.exchange(S.m_send[0], S.m_send[1], S.m_recv[0], S.m_recv[1])
    backend.append_migrants(S)
    S.swap()


def _loop_exchange(states: List[StripState], send, recv):
    """In-process exchange among logical ranks: rank r's low message to r-1's high slot."""
    P = len(states)
    for r, S in enumerate(states):
        if r > 0:
            recv(states[r - 1])[1].buf.copy_(send(S)[0].buf)
        if r < P - 1:
            recv(states[r + 1])[0].buf.copy_(send(S)[1].buf)


def loopback_rebalance(states: List[StripState], strips: Strips, backends, W: float, nb: int = 1024) -> Strips:
    """rebalance() for P logical ranks in one process (the histogram summed in place)."""
    total = None
    for r, S in enumerate(states):
        h = backends[r].x_histogram(S, strips.x0, strips.x1, nb)
        total = h if total is None else total + h
    new = rebalanced_cuts(strips, total.cpu().tolist(), W)
    for r, S in enumerate(states):
        S.swap()
        backends[r].migrate_pack(S, *new.bounds(r))
    _loop_exchange(states, lambda S: S.m_send, lambda S: S.m_recv)
    for r, S in enumerate(states):
        backends[r].append_migrants(S)
        S.swap()
    return new


def loopback_step(states: List[StripState], strips: Strips, backends, W: float, mode: str = "cvd"):
    """All P ranks of one iteration inside one process (single-GPU emulation): the same
    phases as strip_step, each run for every rank before the exchange that follows it; the
    DistMesh sums are reduced across ranks between the two passes."""
    strips.check_width(W)
    for r, S in enumerate(states):
        backends[r].halo_pack(S, *strips.bounds(r), W)
    _loop_exchange(states, lambda S: S.h_send, lambda S: S.h_recv)
    sums = []
    for r, S in enumerate(states):
        backends[r].append_ghosts(S)
        sums.append(backends[r].cells_begin(S, mode))
    total = None
    if mode == "dm":
        total = sums[0].clone()
        for s in sums[1:]:
            total += s
    for r, S in enumerate(states):
        backends[r].cells_end(S, mode, total)
        backends[r].migrate_pack(S, *strips.bounds(r))
    _loop_exchange(states, lambda S: S.m_send, lambda S: S.m_recv)
    for r, S in enumerate(states):
        backends[r].append_migrants(S)
        S.swap()
