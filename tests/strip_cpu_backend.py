"""CPU test double of paper_2309_13824_b200.strips.GpuStripBackend.

It implements the per-rank pieces of the sync-free strip protocol (fixed-size
messages with count headers, appends at device-style counts, cells of the owned
points with ghosts, in-place migration) with numpy and the oracle on CPU
tensors, so that the orchestration of paper_2309_13824_b200.strips -- what is
sent where, ghost completeness, ownership of emitted triangles, migration --
runs over real torch.distributed (gloo) on CPU.  CVD only (the DistMesh edge
sums of a rank are not separable in the oracle).  Test infrastructure only."""
import numpy as np
import torch

import oracle as O


def _write_msg(m, cols):
    k = len(cols[0])
    if k > m.cap:
        raise RuntimeError("strip message capacity exceeded")
    m.header[0] = k
    for s, c in enumerate(cols):
        m.segment(s, k, torch.int32 if c.dtype == torch.int32 else torch.float64).copy_(c)


def _read_msg(m, segs):
    k = m.count()
    out = [m.segment(s, k, torch.int32 if s == 2 else torch.float64).clone() for s in range(segs)]
    return k, out


class CpuStripBackend:
    def __init__(self, fs, n_total):
        self.fs = fs
        self.n_total = n_total
        self.tri = None

    def halo_pack(self, S, lo, hi, W):
        n = int(S.counts[0])
        x, y, g = S.X[:n], S.Y[:n], S.G[:n]
        for side, sel in enumerate((x < lo + W, x >= hi - W)):
            _write_msg(S.h_send[side], [x[sel], y[sel], g[sel]])

    def append_ghosts(self, S):
        S.counts[1] = S.counts[0]
        for m in S.h_recv:
            k, (x, y, g) = _read_msg(m, 3)
            b = int(S.counts[1])
            S.X[b:b + k], S.Y[b:b + k], S.G[b:b + k] = x, y, g
            S.counts[1] = b + k

    def cells_begin(self, S, mode):
        if mode != "cvd":
            raise NotImplementedError("the CPU double runs CVD only")
        n_own, n_loc = int(S.counts[0]), int(S.counts[1])
        xl, yl, gl = S.X[:n_loc].numpy(), S.Y[:n_loc].numpy(), S.G[:n_loc].numpy()
        dp = None
        if S.have_dprev:
            dp = np.concatenate([S.D[:n_own].numpy(), np.zeros(n_loc - n_own)])
        r = O.iteration(self.fs, xl, yl, mode, d_prev=dp, n_total=self.n_total)
        # triangles emitted by this rank: smallest global id is an owned point
        tg = gl[r.tri]
        owner_local = r.tri[np.arange(len(tg)), np.argmin(tg, axis=1)]
        tri = tg[owner_local < n_own]
        k = np.argmin(tri, axis=1)  # CCW with the smallest global id first
        self.tri = np.stack([tri[np.arange(len(tri)), (k + s) % 3] for s in range(3)], axis=1)
        S.Xo[:n_own] = torch.from_numpy(r.x[:n_own].copy())
        S.Yo[:n_own] = torch.from_numpy(r.y[:n_own].copy())
        S.Do[:n_own] = torch.from_numpy(r.d_prev[:n_own].copy())
        S.status[:n_own] = torch.from_numpy(r.status[:n_own].copy())
        return None

    def cells_end(self, S, mode, sums2=None):
        return None

    def migrate_pack(self, S, lo, hi):
        n = int(S.counts[0])
        x = S.Xo[:n]
        cols = [S.Xo[:n].clone(), S.Yo[:n].clone(), S.G[:n].clone(), S.Do[:n].clone()]
        keep = (x >= lo) & (x < hi)
        for side, sel in enumerate((x < lo, x >= hi)):
            _write_msg(S.m_send[side], [c[sel] for c in cols])
        k = int(keep.sum())
        S.Xo[:k], S.Yo[:k], S.G[:k], S.Do[:k] = (c[keep] for c in cols)
        S.counts[0] = k

    def append_migrants(self, S):
        for m in S.m_recv:
            k, (x, y, g, d) = _read_msg(m, 4)
            b = int(S.counts[0])
            S.Xo[b:b + k], S.Yo[b:b + k], S.G[b:b + k], S.Do[b:b + k] = x, y, g, d
            S.counts[0] = b + k

    def x_histogram(self, S, x0, x1, nb):
        n = int(S.counts[0])
        b = np.clip(np.floor((S.X[:n].numpy() - x0) / (x1 - x0) * nb).astype(np.int64), 0, nb - 1)
        return torch.from_numpy(np.bincount(b, minlength=nb).astype(np.int64))

    def triangles(self):
        return torch.from_numpy(self.tri.astype(np.int32))
