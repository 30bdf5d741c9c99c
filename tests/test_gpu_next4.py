"""GPU parity of the NEXT-4 row (SURVEY §8(f) set-up pipeline) against the oracle, bit for bit:
geometry-grid categories, contour SDF and the set operations,
Floyd-Steinberg counts and initial points, and the whole pipeline contour -> SDF ->
geometry grid -> initial points -> meshing to termination."""
import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import oracle as O
from inputs import configs
from tests.gpu_util import to_dev


def _star(n_tips=7, m=24, r0=0.25, r1=0.45, c=(0.5, 0.5)):
    """A clockwise star-shaped loop: sharp convex tips and concave notches."""
    pts = []
    for k in range(n_tips * m):
        a = -2 * math.pi * k / (n_tips * m)  # clockwise
        f = 0.5 * (1 + math.cos(n_tips * a))
        r = r0 + (r1 - r0) * f ** 3
        pts.append((c[0] + r * math.cos(a), c[1] + r * math.sin(a)))
    return np.array([[*pts[k], *pts[(k + 1) % len(pts)]] for k in range(len(pts))])


def test_contour_sdf_and_set_operations_match_oracle():
    import paper_2309_13824_b200 as T
    ctx = T.Context(0)
    box = (0.0, 0.0, 1.0, 1.0)
    segs = _star()
    nx = ny = 193
    phi = torch.empty(ny, nx, dtype=torch.float64, device="cuda")
    ctx.tm_contour_sdf(to_dev(segs), nx, ny, box, phi)
    o = O.contour_sdf(segs, nx, ny, box)
    assert np.array_equal(phi.cpu().numpy(), o)
    # difference with a circle (the paper's custom shape is built this way)
    X, Y = np.meshgrid(configs.node_coords(0, 1, nx), configs.node_coords(0, 1, ny))
    circ = np.sqrt((X - 0.5) ** 2 + (Y - 0.7) ** 2) - 0.1
    out = torch.empty_like(phi)
    for op, ref in [(0, np.minimum(o, circ)), (1, np.maximum(o, -circ)), (2, np.maximum(o, circ))]:
        ctx.tm_sdf_combine(op, phi, to_dev(circ), out)
        assert np.array_equal(out.cpu().numpy(), ref), op


@pytest.mark.parametrize("k", [3, 4])
def test_categories_counts_and_points_match_oracle(k, cfg_cache):
    import paper_2309_13824_b200 as T
    c = cfg_cache(k)
    ctx = T.Context(0)
    n_init = 200_000
    ctx.tm_set_domain(c.box, to_dev(c.phi), to_dev(c.mu), to_dev(c.rho), n_init)
    nxg, nyg = T.geometry_grid_dims(c.n, c.box)
    assert (nxg, nyg) == O.geometry_grid_dims(c.n, c.box)
    x, y, cat, counts = T.initial_points(ctx, n_init, nxg, nyg, seed=5)
    fs = O.FieldSet.from_config(c)
    ocat = O.geometry_categories(fs, nxg, nyg)
    assert np.array_equal(cat.cpu().numpy(), ocat)
    ocnt, otot = O.init_counts(fs, ocat, n_init)
    # residuals reaching a cell with no valid later neighbour are dropped (the paper diffuses only
    # to valid cells): the total is N_init to within a few points
    assert np.array_equal(counts.cpu().numpy(), ocnt) and abs(otot - n_init) <= 1e-3 * n_init
    oc, oh = O.domain(fs, n_init)
    ox, oy = O.init_points(fs, ocnt, 5, oc, oh)
    assert np.array_equal(x.cpu().numpy(), ox) and np.array_equal(y.cpu().numpy(), oy)


def test_pipeline_contour_to_mesh():
    """contour -> SDF -> automatic sizing (boundary points, medial axis, lfs, mu; rho = mu^-2) ->
    geometry grid -> fac_init * N_total initial points -> hybrid meshing with point addition to
    termination (all on the GPU): every point ends inside or on the boundary, the mesh has N_total
    points, the triangle count obeys Euler's bound, and the mesh is finer where mu is smaller."""
    import paper_2309_13824_b200 as T
    ctx = T.Context(0, params=T.default_params(validity=1))
    box = (0.0, 0.0, 1.0, 1.0)
    n = 257
    segs = to_dev(_star())
    phi = torch.empty(n, n, dtype=torch.float64, device="cuda")
    ctx.tm_contour_sdf(segs, n, n, box, phi)
    n_total = 3000
    nxg, nyg = T.geometry_grid_dims(n_total, box)
    dxg = 1.0 / nxg
    mu, _, _, _ = T.automatic_sizing(ctx, segs, box, n, n, K=0.3, d_s=0.5 * dxg, geps_hat=0.01 * dxg,
                                     r_nei=2 * 3 * 0.5 * dxg)
    rho = torch.empty_like(mu)
    ctx.tm_density_from_sizing(mu, rho)
    n_init = int(0.2 * n_total)
    ctx.tm_set_domain(box, phi, mu, rho, n_init)
    x, y, cat, counts = T.initial_points(ctx, n_init, nxg, nyg, seed=1)
    ctx.tm_set_domain(box, phi, mu, rho, x.shape[0])
    res = T.mesh(ctx, x, y, n_total=n_total, method="hybrid", max_iterations=400)
    acts = [h["action"] for h in res.history]
    assert acts[-1] in ("terminate_quality", "terminate_moves"), acts[-5:]
    assert res.x.shape[0] == n_total
    fs = O.FieldSet(box, phi.cpu().numpy(), mu=mu.cpu().numpy())
    xs, ys = res.x.cpu().numpy(), res.y.cpu().numpy()
    _, ha = O.domain(fs, n_total)
    worst = max(O.field_value(fs, "phi", a, b) for a, b in zip(xs, ys))
    assert worst <= 0.01 * ha + 1e-12
    assert 0 < res.tri.shape[0] <= 2 * n_total - 2
    # edge length follows mu: the mean edge over mu at the edge midpoint is nearly constant
    t = res.tri.cpu().numpy()
    e = np.concatenate([t[:, [0, 1]], t[:, [1, 2]], t[:, [2, 0]]])
    L = np.hypot(xs[e[:, 0]] - xs[e[:, 1]], ys[e[:, 0]] - ys[e[:, 1]])
    m = np.array([O.field_value(fs, "mu", 0.5 * (xs[a] + xs[b]), 0.5 * (ys[a] + ys[b])) for a, b in e])
    r = L / m
    lo, hi = m < np.quantile(m, 0.25), m > np.quantile(m, 0.75)
    assert L[lo].mean() < L[hi].mean() and 0.6 < r[lo].mean() / r[hi].mean() < 1.6


def test_automatic_sizing_matches_oracle():
    """App. A + P:356-373 on the star contour: boundary points, medial points (poles of the
    library's own Delaunay, trimmed), lfs and the sizing field, bit for bit."""
    import paper_2309_13824_b200 as T
    ctx = T.Context(0)
    box = (0.0, 0.0, 1.0, 1.0)
    segs = _star()
    d_s, geps_hat, r_nei, K = 0.008, 5e-4, 2 * 3 * 0.008, 0.1
    mu, (sx, sy), (mx, my), lfs = T.automatic_sizing(ctx, to_dev(segs), box, 129, 129, K, d_s, geps_hat, r_nei)
    ox, oy = O.boundary_points(segs, d_s, geps_hat)
    assert np.array_equal(sx.cpu().numpy(), ox) and np.array_equal(sy.cpu().numpy(), oy)
    omx, omy = O.medial_points(ox, oy, box, r_nei, 3)
    assert len(omx) > 10
    assert np.array_equal(mx.cpu().numpy(), omx) and np.array_equal(my.cpu().numpy(), omy)
    omu, olfs = O.sizing_field(ox, oy, omx, omy, K, 129, 129, box)
    assert np.array_equal(lfs.cpu().numpy(), olfs)
    assert np.array_equal(mu.cpu().numpy(), omu)


def test_adf_matches_oracle():
    """ADF quadtrees on the star's boundary cells: the same node and leaf counts as the
    oracle's, and the same values, bit for bit, at random points of the boundary cells (NaN off
    them), for the paper's E_tol factor and a finer one."""
    import paper_2309_13824_b200 as T
    ctx = T.Context(0)
    box = (0.0, 0.0, 1.0, 1.0)
    segs = _star()
    n = 193
    phi = torch.empty(n, n, dtype=torch.float64, device="cuda")
    ctx.tm_contour_sdf(to_dev(segs), n, n, box, phi)
    ctx.tm_set_domain(box, phi, None, None, 5000)
    nxg, nyg = T.geometry_grid_dims(5000, box)
    cat = torch.empty(nyg * nxg, dtype=torch.int8, device="cuda")
    ctx.tm_geometry_categories(nxg, nyg, cat)
    fs = O.FieldSet(box, phi.cpu().numpy())
    oc, oh = O.domain(fs, 5000)
    ocat = cat.cpu().numpy().reshape(nyg, nxg)
    rng = np.random.default_rng(4)
    js, is_ = np.nonzero(ocat == 1)
    pick = rng.integers(0, len(js), 4000)
    d = 1.0 / nxg
    px = (is_[pick] + rng.random(4000)) * d
    py = (js[pick] + rng.random(4000)) * d
    px = np.concatenate([px, [0.5, 0.02]])
    py = np.concatenate([py, [0.5, 0.02]])  # an inner and an outer cell: NaN
    for fac_etol in (0.1, 0.01):
        nn, nl = ctx.tm_adf_build(to_dev(segs), nxg, nyg, cat, fac_etol=fac_etol, fac_pt=np.sqrt(0.2))
        oadf = O.ADF(fs, oc, oh, ocat, segs, fac_etol=fac_etol, fac_pt=np.sqrt(0.2))
        assert (nn, nl) == (oadf.n_nodes, oadf.n_leaves)
        out = torch.empty(len(px), dtype=torch.float64, device="cuda")
        ctx.tm_adf_eval(to_dev(px), to_dev(py), out)
        g = out.cpu().numpy()
        o = np.array([oadf(a, b) for a, b in zip(px, py)])
        assert np.array_equal(np.isnan(g), np.isnan(o))
        assert np.array_equal(g[~np.isnan(g)], o[~np.isnan(o)])
    assert np.isnan(g[-1]) and np.isnan(g[-2])
