"""Helpers shared by the -m gpu tests: run one GPU iteration through the C ABI
and compare it with the oracle on identical inputs."""
import numpy as np
import torch

import oracle as O


def to_dev(a, dtype=torch.float64):
    return torch.from_numpy(np.ascontiguousarray(a)).to(device="cuda", dtype=dtype)


class GpuRunner:
    def __init__(self, cfg_box, phi, mu=None, rho=None, n_total=None, params=None, flags=0):
        import paper_2309_13824_b200 as T
        self.T = T
        p = params or T.default_params()
        p.flags |= flags
        self.ctx = T.Context(0, params=p)
        self.box = cfg_box
        self.phi = to_dev(phi)
        self.mu = None if mu is None else to_dev(mu)
        self.rho = None if rho is None else to_dev(rho)
        self.n_total = n_total

    def set_domain(self, n):
        return self.ctx.tm_set_domain(self.box, self.phi, self.mu, self.rho, self.n_total or n)

    def iteration(self, x, y, mode, d_prev=None):
        """One GPU iteration from host arrays; returns numpy results."""
        T = self.T
        n = len(x)
        if self.ctx.c is None:
            self.set_domain(n)
        xd, yd = to_dev(x), to_dev(y)
        dp = None if d_prev is None else to_dev(d_prev)
        bufs = T.IterBuffers.alloc(n, self.ctx.params.adj_stride)
        xo = torch.empty(n, dtype=torch.float64, device="cuda")
        yo = torch.empty_like(xo)
        do = torch.empty_like(xo)
        T.iterate(self.ctx, xd, yd, dp, mode, bufs, xo, yo, do)
        self.ctx.tm_sync()
        nt = int(bufs.n_tri.item())
        out = {
            "tri": bufs.tri[:nt].cpu().numpy(),
            "x": xo.cpu().numpy(), "y": yo.cpu().numpy(), "d_prev": do.cpu().numpy(),
            "status": bufs.status.cpu().numpy(),
        }
        if mode == "dm":
            adj_o = torch.empty((n, self.ctx.params.adj_stride), dtype=torch.int32, device="cuda")
            deg_o = torch.empty(n, dtype=torch.uint8, device="cuda")
            self.ctx.tm_adjacency_export(bufs.adj, bufs.deg, adj_o, deg_o)
            out["adj"] = adj_o.cpu().numpy()
            out["deg"] = deg_o.cpu().numpy()
            out["sums2"] = bufs.sums2.cpu().numpy()
        return out


def tri_set(tri):
    t = np.asarray(tri, dtype=np.int64)
    return set(map(tuple, t.tolist()))


def edges_from_adj(adj, deg):
    E = set()
    for i in range(len(deg)):
        for k in range(int(deg[i])):
            a = int(adj[i, k])
            E.add((min(i, a), max(i, a)))
    return E


def compare(gpu, orc, box, mode, pos_tol=1e-12, ctx="", exact_cvd=True):
    """Assert the parity bar: identical kept-triangle set (CCW, min first),
    identical ELL edge set (DistMesh), positions within pos_tol*diam(B) (L14),
    identical status codes.  CVD positions are required to be BIT-identical
    (exact_cvd): both sides build every cell vertex by the same correctly rounded
    Cramer divisions and sum the centroid / quadrature in the same ring order
    without contraction (L25), so the only remaining freedom is none.  DistMesh
    positions differ by a few ulps (the force is a per-point gather on the GPU and
    an edge loop in the oracle: another summation order)."""
    gt = tri_set(gpu["tri"])
    ot = tri_set(orc.tri)
    assert len(gt) == len(gpu["tri"]), f"{ctx}: duplicate GPU triangles"
    missing, extra = ot - gt, gt - ot
    nt = getattr(orc.info, "n_near_ties", 0)
    assert not missing and not extra, f"{ctx}: triangle sets differ: {len(missing)} missing, {len(extra)} extra " \
                                      f"(e.g. {list(missing)[:3]} / {list(extra)[:3]}); oracle near ties: {nt}"
    diam = float(np.hypot(box[2] - box[0], box[3] - box[1]))
    err = np.hypot(gpu["x"] - orc.x, gpu["y"] - orc.y)
    k = int(np.argmax(err))
    assert err[k] <= pos_tol * diam, f"{ctx}: position error {err[k]:.3e} at {k} (tol {pos_tol * diam:.3e})"
    bad = np.nonzero(gpu["status"] != orc.status)[0]
    assert bad.size == 0, f"{ctx}: status differs at {bad[:5]} gpu={gpu['status'][bad[:5]]} or={orc.status[bad[:5]]}"
    derr = np.abs(gpu["d_prev"] - orc.d_prev)
    assert derr.max() <= pos_tol * diam, f"{ctx}: d_prev error {derr.max():.3e}"
    if mode == "cvd" and exact_cvd:
        nb = int(np.count_nonzero((gpu["x"] != orc.x) | (gpu["y"] != orc.y) | (gpu["d_prev"] != orc.d_prev)))
        assert nb == 0, f"{ctx}: {nb} CVD positions not bit-identical (max error {err[k]:.3e})"
    if mode == "dm" and gpu.get("adj") is not None:
        ge = edges_from_adj(gpu["adj"], gpu["deg"])
        oe = set(map(tuple, orc.edges.tolist()))
        assert ge == oe, f"{ctx}: ELL edges differ: {len(oe - ge)} missing {len(ge - oe)} extra"
    return float(err.max())
