"""x-strip decomposition on ONE GPU: P logical ranks run the
GPU strip backend (tm_halo_pack, ghost binning with global ids, owner-emits
triangles, tm_migrate_pack) through the Loopback exchanger.  The union of the
per-rank triangle sets must equal the oracle's single-domain result, every
triangle must be emitted exactly once and every point owned once, and the
owned positions must equal the oracle's update (CVD) / agree within the
parity bar (DistMesh, where the edge-sum reduction order differs)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import oracle as O
from inputs import configs


def _run(P, n, seed, modes, box=(0.0, 0.0, 1.0, 1.0)):
    import paper_2309_13824_b200 as T
    from paper_2309_13824_b200 import strips as S
    phi = configs.box_phi(box, 128)
    fs = O.FieldSet(box, phi)
    x, y = configs.random_points(n, seed, box)
    strips = S.Strips(box[0], box[2], P)
    dev = torch.device("cuda", 0)
    phid = torch.from_numpy(phi).to(dev)
    backends = []
    for r in range(P):
        ctx = T.Context(0)
        c, _ = ctx.tm_set_domain(box, phid, None, None, n)
        backends.append(S.GpuStripBackend(ctx))
    W = S.ghost_width(c, 5.0)
    xd, yd = torch.from_numpy(x).to(dev), torch.from_numpy(y).to(dev)
    states = [S.split_initial(xd, yd, strips, r) for r in range(P)]
    dp = None
    for it, mode in enumerate(modes):
        ref = O.iteration(fs, x, y, mode, d_prev=dp)
        states = S.loopback_iteration(states, strips, backends, W, mode)
        got, seen = [], np.zeros(n, bool)
        xs, ys, ds = np.empty(n), np.empty(n), np.empty(n)
        for st in states:
            gid = st.gid.cpu().numpy().astype(np.int64)
            assert not seen[gid].any()
            seen[gid] = True
            xs[gid], ys[gid], ds[gid] = st.x.cpu().numpy(), st.y.cpu().numpy(), st.d_prev.cpu().numpy()
            got += [tuple(t) for t in st.tri.cpu().numpy().tolist()]
        assert seen.all()
        assert len(got) == len(set(got)), "a triangle was emitted by two ranks"
        assert set(got) == set(map(tuple, ref.tri.tolist())), f"P={P} it={it} {mode}: triangle sets differ"
        diam = np.hypot(box[2] - box[0], box[3] - box[1])
        err = np.hypot(xs - ref.x, ys - ref.y).max()
        assert err <= 1e-12 * diam, f"P={P} it={it} {mode}: position error {err:.3e}"
        x, y, dp = ref.x, ref.y, ref.d_prev
        # continue from the oracle's state so that both sides start each iteration identically
        states = [S.split_initial(torch.from_numpy(x).to(dev), torch.from_numpy(y).to(dev), strips, r,
                                  d_prev=torch.from_numpy(dp).to(dev)) for r in range(P)]


@pytest.mark.parametrize("P", [2, 3, 8])
def test_gpu_strips_loopback_match_single_domain(P):
    _run(P, 20000, 21 + P, ["cvd", "dm", "cvd"])


def test_gpu_strips_adaptive_halo():
    """Adaptive sizing (an annulus like configs[2], 4x10^5 points -- enough that 2 fac c L < 1,
    c ~ N^-1/2, so the Lipschitz width applies): x-quantile strips with
    the per-point halo width from the Lipschitz bound of mu~ (tm_halo_pack width < 0).
    The union of the rank results equals the oracle's single-domain iteration, and the
    adaptive band sends fewer ghosts than the fixed 2 S_max band."""
    import paper_2309_13824_b200 as T
    from paper_2309_13824_b200 import strips as S
    c = configs.config3(n=400000, grid=512)
    n, P = c.n, 4
    fs = O.FieldSet.from_config(c)
    dev = torch.device("cuda", 0)
    to = lambda a: torch.from_numpy(a).to(dev)
    xd, yd = to(c.x), to(c.y)
    strips = S.Strips.from_quantiles(xd, P, c.box[0], c.box[2])
    results = {}
    for adaptive in (True, False):
        backends = []
        for r in range(P):
            ctx = T.Context(0)
            cc, _ = ctx.tm_set_domain(c.box, to(c.phi), to(c.mu), to(c.rho), n)
            backends.append(S.GpuStripBackend(ctx, adaptive_halo=adaptive))
        W = S.ghost_width(cc, 5.0, float(c.mu.max()))
        states = [S.split_initial(xd, yd, strips, r) for r in range(P)]
        ghosts = 0
        x, y, dp = c.x, c.y, None
        for mode in ("dm", "cvd"):
            ref = O.iteration(fs, x, y, mode, d_prev=dp)
            states = S.loopback_iteration(states, strips, backends, W, mode)
            got, xs, ys = [], np.empty(n), np.empty(n)
            for st in states:
                gid = st.gid.cpu().numpy().astype(np.int64)
                xs[gid], ys[gid] = st.x.cpu().numpy(), st.y.cpu().numpy()
                got += [tuple(t) for t in st.tri.cpu().numpy().tolist()]
            assert len(got) == len(set(got))
            assert set(got) == set(map(tuple, ref.tri.tolist())), f"adaptive={adaptive} {mode}: triangles differ"
            assert np.hypot(xs - ref.x, ys - ref.y).max() <= 1e-12 * 2.2 * np.sqrt(2)
            x, y, dp = ref.x, ref.y, ref.d_prev
            states = [S.split_initial(to(x), to(y), strips, r, d_prev=to(dp)) for r in range(P)]
            # ghosts sent for this state
            for r, st in enumerate(states):
                lo, hi = strips.bounds(r)
                h_lo, h_hi = backends[r].halo(st, lo, hi, W)
                ghosts += h_lo[0].shape[0] + h_hi[0].shape[0]
        results[adaptive] = ghosts
    assert results[True] < results[False], results
