"""CPU test double of paper_2309_13824_b200.strips.GpuStripBackend.

It implements the per-rank pieces (halo selection, cells of the owned points
with ghosts, migration) with numpy and the oracle, so that the strip
protocol -- what is sent where, ghost completeness, ownership of emitted
triangles, migration -- can run over real torch.distributed (gloo) on CPU.
Test infrastructure only."""
import numpy as np
import torch

import oracle as O


class CpuStripBackend:
    def __init__(self, fs, n_total):
        self.fs = fs
        self.n_total = n_total

    def halo(self, st, lo, hi, W):
        x = st.x.numpy()
        sl = x < lo + W
        sh = x >= hi - W
        pick = lambda m: [st.x[torch.from_numpy(m)].clone(), st.y[torch.from_numpy(m)].clone(),
                          st.gid[torch.from_numpy(m)].clone()]
        return pick(sl), pick(sh)

    def cells_begin(self, st, ghosts, mode):
        xs = [st.x] + [g[0] for g in ghosts if g is not None]
        ys = [st.y] + [g[1] for g in ghosts if g is not None]
        gs = [st.gid] + [g[2] for g in ghosts if g is not None]
        xl, yl, gl = torch.cat(xs).numpy(), torch.cat(ys).numpy(), torch.cat(gs).numpy()
        n_own = st.x.shape[0]
        dp = None
        if st.d_prev is not None:
            dp = np.concatenate([st.d_prev.numpy(), np.zeros(len(xl) - n_own)])
        r = O.iteration(self.fs, xl, yl, mode, d_prev=dp, n_total=self.n_total)
        # triangles emitted by this rank: smallest global id is an owned point
        tg = gl[r.tri]
        owner_local = r.tri[np.arange(len(tg)), np.argmin(tg, axis=1)]
        keep = owner_local < n_own
        tri = tg[keep]
        # CCW with the smallest global id first
        k = np.argmin(tri, axis=1)
        tri = np.stack([tri[np.arange(len(tri)), (k + s) % 3] for s in range(3)], axis=1)
        return {"tri": tri, "r": r, "n_own": n_own, "st": st}, None

    def cells_end(self, h, sums2=None):
        r, n = h["r"], h["n_own"]
        return (torch.from_numpy(h["tri"].astype(np.int32)), torch.from_numpy(r.x[:n].copy()),
                torch.from_numpy(r.y[:n].copy()), torch.from_numpy(r.d_prev[:n].copy()),
                torch.from_numpy(r.status[:n].copy()))

    def migrate(self, st, lo, hi):
        x = st.x.numpy()
        k = (x >= lo) & (x < hi)
        a = x < lo
        b = x >= hi
        dp = st.d_prev if st.d_prev is not None else torch.zeros_like(st.x)
        sel = lambda m: [st.x[torch.from_numpy(m)].clone(), st.y[torch.from_numpy(m)].clone(),
                         st.gid[torch.from_numpy(m)].clone(), dp[torch.from_numpy(m)].clone()]
        return sel(k), sel(a), sel(b)
