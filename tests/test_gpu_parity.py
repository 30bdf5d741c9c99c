"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on
identical inputs, element by element.

Bar (BASELINE.json north_star): kept triangles bit-exact as sorted index
triples; ELL adjacency identical (DistMesh); positions and d_prev within
1e-12 * diam(B) after one update (reading L14); status codes identical.
Both sides take every discrete decision with the same canonical arithmetic
(L25) or exact predicates, so any mismatch is a bug, not rounding.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import oracle as O
from inputs import configs
from tests.gpu_util import GpuRunner, compare


def run_pair(c, x, y, mode, d_prev=None, params=None, oparams=None, runner=None):
    r = runner or GpuRunner(c.box, c.phi, c.mu, c.rho, params=params)
    g = r.iteration(x, y, mode, d_prev)
    o = O.iteration(O.FieldSet.from_config(c), x, y, mode, d_prev=d_prev, params=oparams)
    assert o.info.n_degenerate == 0
    return g, o, r


def test_cfg1_all_lloyd_iterations(cfg_cache):
    """configs[0]: 10 CVD iterations, parity at every iteration from the GPU's own state."""
    c = cfg_cache(1)
    r = GpuRunner(c.box, c.phi)
    x, y, dp = c.x, c.y, None
    for it in range(10):
        g = r.iteration(x, y, "cvd", dp)
        o = O.iteration(O.FieldSet.from_config(c), x, y, "cvd", d_prev=dp)
        compare(g, o, c.box, "cvd", ctx=f"cfg1 it{it}")
        x, y, dp = g["x"], g["y"], g["d_prev"]


def _protocol(c, check):
    """SURVEY §8(c) parity protocol: run the GPU through the config's whole schedule from
    its own state; at the iterations in `check` the oracle performs the same iteration
    from the identical input bits and the outputs are compared (triangles exact, ELL
    edges exact, positions within 1e-12 diam, status codes)."""
    r = GpuRunner(c.box, c.phi, c.mu, c.rho)
    fs = O.FieldSet.from_config(c)
    x, y, dp = c.x, c.y, None
    for it, mode in enumerate(c.schedule):
        g = r.iteration(x, y, mode, dp)
        if it in check:
            o = O.iteration(fs, x, y, mode, d_prev=dp)
            assert o.info.n_degenerate == 0
            compare(g, o, c.box, mode, ctx=f"{c.name} it{it} {mode}")
        x, y, dp = g["x"], g["y"], g["d_prev"]


def test_cfg2_distmesh(cfg_cache):
    """configs[1]: 50 DistMesh iterations on the disk; parity at {0, 1, 25, 49}."""
    c = cfg_cache(2)
    n = len(c.schedule)
    _protocol(c, {0, 1, n // 2, n - 1})


@pytest.mark.parametrize("k", [3, 4])
def test_adaptive_full_size_protocol(k, cfg_cache):
    """configs[2]/[3] at full size (10^6, adaptive): the whole hybrid schedule (30+30 /
    20+20 iterations, warm-started from the second iteration on); parity at the first two
    iterations, the last DistMesh and first CVD iteration (adaptive quadrature), and the
    last iteration."""
    c = cfg_cache(k)
    n = len(c.schedule)
    ndm = sum(1 for m in c.schedule if m == "dm")
    _protocol(c, {0, 1, ndm - 1, ndm, n - 1})


@pytest.mark.parametrize("n,seed", [(3, 1), (4, 2), (7, 3), (40, 4), (333, 5), (5000, 6)])
def test_small_random_ragged(n, seed):
    box = (0.0, 0.0, 1.0, 1.0)
    phi = configs.box_phi(box, 64)
    c = configs.Config("rand", *configs.random_points(n, seed, box), box, phi, None, None, ["cvd"])
    for mode in ("cvd", "dm"):
        g, o, _ = run_pair(c, c.x, c.y, mode)
        compare(g, o, box, mode, ctx=f"rand n={n} {mode}")


@pytest.mark.parametrize("fac", [0.6, 1.0, 2.0])
def test_octagon_binding(fac):
    """Small octagons (fac_voro_bound < 5) make the octagon walls bind on many
    cells and exercise the (wall, bisector) vertices and the octagon keep tests."""
    import paper_2309_13824_b200 as T
    box = (0.0, 0.0, 1.0, 1.0)
    phi = configs.box_phi(box, 64)
    x, y = configs.random_points(4000, 17, box)
    c = configs.Config("oct", x, y, box, phi, None, None, ["cvd"])
    for mode in ("cvd", "dm"):
        g, o, _ = run_pair(c, x, y, mode, params=T.default_params(fac_voro_bound=fac),
                           oparams=O.default_params(fac_voro_bound=fac))
        compare(g, o, box, mode, ctx=f"fac={fac} {mode}")


def test_points_on_bin_edges_and_box_boundary():
    """Points exactly on bin boundaries and on the box sides (L24)."""
    box = (0.0, 0.0, 1.0, 1.0)
    phi = configs.box_phi(box, 64)
    n = 2000
    rng = np.random.default_rng(8)
    x, y = rng.random(n), rng.random(n)
    import paper_2309_13824_b200 as T
    nb = int(np.ceil(np.sqrt(n / T.default_params().n_opt)))  # level-0 bins of the unit box
    k = rng.integers(1, nb, 300)
    x[:300] = k / nb  # on interior vertical bin edges (many collinear points: generic for Delaunay)
    # on the box sides: at most two per side (three collinear hull points are non-generic, L12)
    y[300:302] = 0.0
    y[302:304] = 1.0
    x[304:306] = 1.0
    x[306:308] = 0.0
    c = configs.Config("edges", x, y, box, phi, None, None, ["cvd"])
    for mode in ("cvd", "dm"):
        g, o, _ = run_pair(c, x, y, mode)
        compare(g, o, box, mode, ctx=f"edges {mode}")


def test_near_cocircular_forces_exact_path():
    """A square lattice jittered by ~1e-13 is nearly cocircular everywhere: the
    floating filters cannot decide and the exact expansion path must agree with
    the oracle's big integers."""
    import paper_2309_13824_b200 as T
    m = 40
    g1 = (np.arange(m) + 0.5) / m
    X, Y = np.meshgrid(g1, g1)
    box = (0.0, 0.0, 1.0, 1.0)
    phi = configs.box_phi(box, 64)
    for seed in range(20):  # a few-ulp jitter; retry the rare exactly-cocircular draw (L12)
        rng = np.random.default_rng(seed)
        ux = np.spacing(X.ravel()) * rng.integers(-20, 21, m * m)
        uy = np.spacing(Y.ravel()) * rng.integers(-20, 21, m * m)
        x, y = (X.ravel() + ux).copy(), (Y.ravel() + uy).copy()
        if O.iteration(O.FieldSet(box, phi), x, y, "cvd").info.n_degenerate == 0:
            break
    c = configs.Config("lattice", x, y, box, phi, None, None, ["cvd"])
    r = GpuRunner(box, phi, flags=T.TM_F_COUNT_WORK)
    g, o, _ = run_pair(c, x, y, "cvd", runner=r)
    compare(g, o, box, "cvd", ctx="lattice")
    w = r.ctx.tm_work_counts()
    assert w.exact_calls > 100


def test_work_counts_match_oracle(cfg_cache):
    """O8 work statistics: the GPU's own counters agree with the oracle's."""
    import paper_2309_13824_b200 as T
    c = cfg_cache(2)
    r = GpuRunner(c.box, c.phi, flags=T.TM_F_COUNT_WORK)
    g = r.iteration(c.x, c.y, "dm")
    w = r.ctx.tm_work_counts()
    o = O.iteration(O.FieldSet.from_config(c), c.x, c.y, "dm", counts=True)
    cnt = o.counts.sum(0)
    assert w.n_cells == c.n
    assert w.deg == cnt[1] and w.verts == cnt[2] and w.t_own == cnt[3] and w.ell == cnt[5]
    assert abs(w.n_cert - cnt[0]) <= 1e-4 * cnt[0]


def test_errors_are_loud():
    import paper_2309_13824_b200 as T
    import torch
    box = (0.0, 0.0, 1.0, 1.0)
    phi = configs.box_phi(box, 16)
    ctx = T.Context(0)
    x = torch.rand(100, dtype=torch.float64, device="cuda")
    y = torch.rand(100, dtype=torch.float64, device="cuda")
    with pytest.raises(T.TmError) as e:
        ctx.tm_grid_bin(x, y)
    assert e.value.code == T.TM_E_STATE
    ctx.tm_set_domain(box, torch.from_numpy(phi).cuda(), None, None, 100)
    # duplicates
    x2 = x.clone()
    y2 = y.clone()
    x2[7] = x2[3]
    y2[7] = y2[3]
    bufs = T.IterBuffers.alloc(100)
    ctx.tm_grid_bin(x2, y2)
    ctx.tm_voronoi_delaunay(bufs.tri, bufs.n_tri)
    with pytest.raises(T.TmError) as e:
        ctx.tm_sync()
    assert e.value.code == T.TM_E_DUPLICATE
    # outside the box
    ctx2 = T.Context(0)
    ctx2.tm_set_domain(box, torch.from_numpy(phi).cuda(), None, None, 100)
    x3 = x.clone()
    x3[0] = 1.5
    ctx2.tm_grid_bin(x3, y)
    with pytest.raises(T.TmError) as e:
        ctx2.tm_sync()
    assert e.value.code == T.TM_E_OUTSIDE
    # triangle capacity
    ctx3 = T.Context(0)
    ctx3.tm_set_domain(box, torch.from_numpy(phi).cuda(), None, None, 100)
    ctx3.tm_grid_bin(x, y)
    small = torch.empty((5, 3), dtype=torch.int32, device="cuda")
    nt = torch.zeros(1, dtype=torch.int64, device="cuda")
    ctx3.tm_voronoi_delaunay(small, nt)
    with pytest.raises(T.TmError) as e:
        ctx3.tm_sync()
    assert e.value.code == T.TM_E_CAPACITY
    need = int(nt.item())
    assert need > 5  # the required count is reported
    # the documented recovery: retry with the reported count on the SAME context -> TM_OK
    # (latched errors are cleared once reported)
    big = torch.empty((need, 3), dtype=torch.int32, device="cuda")
    ctx3.tm_voronoi_delaunay(big, nt)
    ctx3.tm_sync()
    assert int(nt.item()) == need
    # and a clean iteration after a duplicate error on the first context
    ctx.tm_grid_bin(x, y)
    ctx.tm_voronoi_delaunay(bufs.tri, bufs.n_tri)
    ctx.tm_sync()


def test_health_counters_per_sync():
    """n_fallback of tm_mesh_stats counts the projection fallbacks since the previous
    synchronising call, equal to the oracle's status & 2 count, iteration by iteration."""
    import torch
    import paper_2309_13824_b200 as T
    box = (0.0, 0.0, 1.0, 1.0)
    n = 513
    gx = configs.node_coords(0.0, 1.0, n)
    X, Y = np.meshgrid(gx, gx)
    # phi has a plateau (zero gradient) beyond x = 0.6: a point moved there cannot be projected
    phi = np.where(X > 0.6, 1.0, np.maximum(X - 0.6, configs.box_phi(box, n)))
    rng = np.random.default_rng(11)
    x = rng.random(3000) * 0.6
    y = rng.random(3000)
    fs = O.FieldSet(box, phi)
    r = GpuRunner(box, phi)
    r.set_domain(len(x))
    ctx = r.ctx
    bufs = T.IterBuffers.alloc(len(x))
    xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    dp = None
    seen = 0
    for it in range(2):
        o = O.iteration(fs, xd.cpu().numpy(), yd.cpu().numpy(), "cvd", d_prev=None if dp is None else dp.cpu().numpy())
        xo, yo, do = torch.empty_like(xd), torch.empty_like(xd), torch.empty_like(xd)
        T.iterate(ctx, xd, yd, dp, "cvd", bufs, xo, yo, do)
        nt = int(bufs.n_tri.item())
        s = ctx.tm_mesh_stats(xo, yo, bufs.tri, nt)
        want = int(np.count_nonzero(o.status & 2))
        assert s.n_fallback == want, (it, s.n_fallback, want)
        assert s.n_degenerate == 0 and s.n_overflow == 0
        seen += want
        xd, yd, dp = xo, yo, do
    assert seen > 0  # the case exercises the counter
    s = ctx.tm_mesh_stats(xd, yd, bufs.tri, 0)  # nothing since the last report
    assert s.n_fallback == 0


def test_standalone_project_and_cvd_step_match_fused(cfg_cache):
    """tm_cvd_step + tm_project_sdf (unfused) == fused tm_voronoi_delaunay CVD."""
    import torch
    import paper_2309_13824_b200 as T
    c = cfg_cache(1)
    r = GpuRunner(c.box, c.phi)
    g = r.iteration(c.x, c.y, "cvd")
    ctx = r.ctx
    x, y = torch.from_numpy(c.x).cuda(), torch.from_numpy(c.y).cuda()
    ctx.tm_grid_bin(x, y)
    xh, yh = torch.empty_like(x), torch.empty_like(y)
    ctx.tm_cvd_step(None, xh, yh)
    xo, yo, do = torch.empty_like(x), torch.empty_like(x), torch.empty_like(x)
    st = torch.empty(c.n, dtype=torch.int8, device="cuda")
    ctx.tm_project_sdf(x, y, xh, yh, xo, yo, do, st)
    ctx.tm_sync()
    assert np.array_equal(xo.cpu().numpy(), g["x"]) and np.array_equal(yo.cpu().numpy(), g["y"])
    assert np.array_equal(st.cpu().numpy(), g["status"])


def test_mesh_stats_match_oracle(cfg_cache):
    import torch
    c = cfg_cache(2)
    r = GpuRunner(c.box, c.phi)
    g = r.iteration(c.x, c.y, "dm")
    tri = torch.from_numpy(np.ascontiguousarray(g["tri"])).cuda()
    s = r.ctx.tm_mesh_stats(torch.from_numpy(c.x).cuda(), torch.from_numpy(c.y).cuda(), tri, len(g["tri"]))
    o = O.stats(g["tri"], c.x, c.y)
    assert s.n_tri == o[0] and s.n_alpha_lt_1_2 == o[9] and s.n_alpha_lt_2 == o[10]
    # per-triangle oracle values (O7), summed correctly rounded (math.fsum): the GPU's fixed
    # tree sum of n positive terms is within (log2 n + 2) eps of it, plus the per-term
    # rounding of alpha/beta (contracted on the GPU, a few eps relative each): 1e-14
    import math
    al, be = [], []
    for t in g["tri"]:
        a_, b_ = O.triangle_quality((c.x[t[0]], c.y[t[0]]), (c.x[t[1]], c.y[t[1]]), (c.x[t[2]], c.y[t[2]]))
        al.append(a_)
        be.append(b_)
    al, be = np.array(al), np.array(be)
    ref = {"sum_sqrt_alpha": math.fsum(np.sqrt(al)), "sum_sqrt_beta": math.fsum(np.sqrt(be)),
           "sum_alpha": math.fsum(al), "sum_alpha2": math.fsum(al * al), "sum_beta": math.fsum(be),
           "sum_beta2": math.fsum(be * be)}
    for k, v in ref.items():
        assert abs(getattr(s, k) - v) <= 1e-14 * v, (k, getattr(s, k), v)
    assert abs(s.max_alpha - al.max()) <= 1e-12 * al.max() and abs(s.max_beta - be.max()) <= 1e-13 * be.max()
    # deterministic (no atomics): the same bits on a second call
    s2 = r.ctx.tm_mesh_stats(torch.from_numpy(c.x).cuda(), torch.from_numpy(c.y).cuda(), tri, len(g["tri"]))
    assert s2.as_dict() == s.as_dict()


def test_determinism(cfg_cache):
    c = cfg_cache(2)
    r = GpuRunner(c.box, c.phi)
    a = r.iteration(c.x, c.y, "cvd")
    b = r.iteration(c.x, c.y, "cvd")
    assert np.array_equal(a["x"], b["x"]) and np.array_equal(a["y"], b["y"])
    assert tri_set_eq(a["tri"], b["tri"])


def tri_set_eq(a, b):
    from tests.gpu_util import tri_set
    return tri_set(a) == tri_set(b)


@pytest.mark.parametrize("cells", ["thread", "group"])
@pytest.mark.parametrize("k,mode", [(2, "dm"), (3, "dm"), (3, "cvd"), (4, "cvd")])
def test_both_cell_kernels_match_oracle(cells, k, mode, cfg_cache):
    """The thread-per-cell kernel (default) and the 16-lane group kernel
    (TM_F_GROUP_CELLS) both reproduce the oracle at iteration 0 of the
    full-size configs (the CVD case uses the adaptive quadrature on 3/4)."""
    import paper_2309_13824_b200 as T
    c = cfg_cache(k)
    p = T.default_params()
    if cells == "group":
        p.flags |= T.TM_F_GROUP_CELLS
    g, o, _ = run_pair(c, c.x, c.y, mode, params=p)
    compare(g, o, c.box, mode, ctx=f"cfg{k} {mode} {cells}")


def test_thread_kernel_overflow_retry():
    """Cells whose ring needs more slots than the thread kernel holds go to the
    32-lane retry pass: a point surrounded by a fine circle of 24 neighbours
    has a 24-gon cell; the result must still equal the oracle."""
    box = (0.0, 0.0, 1.0, 1.0)
    phi = configs.box_phi(box, 64)
    rng = np.random.default_rng(11)
    n0 = 3000
    x, y = rng.random(n0), rng.random(n0)
    keep = np.hypot(x - 0.5, y - 0.5) > 0.08
    x, y = x[keep], y[keep]
    ang = 2 * np.pi * (np.arange(24) + rng.uniform(-0.05, 0.05, 24)) / 24
    rad = 0.03 * (1 + rng.uniform(-1e-3, 1e-3, 24))
    x = np.concatenate([x, [0.5], 0.5 + rad * np.cos(ang)])
    y = np.concatenate([y, [0.5], 0.5 + rad * np.sin(ang)])
    c = configs.Config("ring24", x, y, box, phi, None, None, ["cvd"])
    import paper_2309_13824_b200 as T
    for mode in ("cvd", "dm"):
        g, o, _ = run_pair(c, x, y, mode, params=T.default_params(adj_stride=32))  # the 24-gon has 24 edges
        compare(g, o, box, mode, ctx=f"ring24 {mode}")


@pytest.mark.parametrize("n,it", [(16_000_000, 0), (16_000_000, 19), (64_000_000, 0), (64_000_000, 19)])
def test_cfg5_full_size_sampled_windows(n, it):
    """configs[4] at its full sizes (1.6e7 and 6.4e7 jittered-uniform points), at
    iteration 0 and at iteration n-1 = 19 of its 20-iteration CVD schedule (SURVEY §8(c)
    parity protocol): the GPU runs `it` iterations from the config's points (warm-started
    cell search), then one more; the oracle recomputes sampled windows of that last
    iteration's input.  A cell, its CVD update and the triangles around it
    depend only on points within a few h (the circumcircles of the Delaunay
    triangles are ~h), so for points farther than a margin of 10 h from a
    window edge (edges on the box sides need no margin) the oracle run on the
    window's points (with the global normalisation n_total = N) must give the
    GPU's positions, status codes and kept triangles exactly."""
    c = configs.config5(n=n)
    h = 1.0 / np.sqrt(n)
    r = GpuRunner(c.box, c.phi)
    X, Y, DP = c.x, c.y, None
    for _ in range(it):
        g = r.iteration(X, Y, "cvd", DP)
        X, Y, DP = g["x"], g["y"], g["d_prev"]
    g = r.iteration(X, Y, "cvd", DP)
    c = configs.Config(c.name, X, Y, c.box, c.phi, None, None, c.schedule)
    fs = O.FieldSet.from_config(c)
    rng = np.random.default_rng(50 + n % 7)
    w, m = 25 * h, 10 * h
    centers = [(w, w), (1 - w, 0.5), (0.5, 1 - w)] + [tuple(p) for p in rng.uniform(0, 1, (9, 2))]
    gtri = g["tri"].astype(np.int64)
    for cx, cy in centers:
        lo_x, hi_x, lo_y, hi_y = max(cx - w, 0.0), min(cx + w, 1.0), max(cy - w, 0.0), min(cy + w, 1.0)
        sel = np.nonzero((c.x >= lo_x) & (c.x <= hi_x) & (c.y >= lo_y) & (c.y <= hi_y))[0]
        ix0 = lo_x + (m if lo_x > 0.0 else -1.0)
        ix1 = hi_x - (m if hi_x < 1.0 else -1.0)
        iy0 = lo_y + (m if lo_y > 0.0 else -1.0)
        iy1 = hi_y - (m if hi_y < 1.0 else -1.0)
        xs, ys = c.x[sel], c.y[sel]
        inner = (xs > ix0) & (xs < ix1) & (ys > iy0) & (ys < iy1)
        o = O.iteration(fs, xs, ys, "cvd", n_total=n, d_prev=None if DP is None else DP[sel])
        assert o.info.n_degenerate == 0
        gi = sel[inner]
        # bit-identical CVD positions (same canonical arithmetic, see tests/gpu_util.compare)
        assert np.array_equal(g["x"][gi], o.x[inner]) and np.array_equal(g["y"][gi], o.y[inner]), \
            f"window {cx:.3f},{cy:.3f}: max position error " \
            f"{np.hypot(g['x'][gi] - o.x[inner], g['y'][gi] - o.y[inner]).max():.3e}"
        assert np.array_equal(g["status"][gi], o.status[inner])
        # triangles with all three vertices inner, in global ids
        inner_g = np.zeros(n, dtype=bool)
        inner_g[gi] = True
        gt = {tuple(t) for t in gtri[inner_g[gtri].all(1)].tolist()}
        ot_all = sel[np.asarray(o.tri, dtype=np.int64)]
        ot = {tuple(t) for t in ot_all[inner_g[ot_all].all(1)].tolist()}
        assert gt == ot, f"window {cx:.3f},{cy:.3f}: {len(ot - gt)} missing, {len(gt - ot)} extra"
        assert len(gt) > 1000


def test_cell_vertex_capacity_error_is_loud():
    """A cell with more vertices than the 32-lane retry pass can hold (a point ringed by 40
    near-cocircular neighbours) must latch TM_E_CAPACITY (reported by tm_sync), not
    return a wrong mesh silently (SURVEY §8(b) errors)."""
    import torch
    import paper_2309_13824_b200 as T
    box = (0.0, 0.0, 1.0, 1.0)
    rng = np.random.default_rng(12)
    x, y = rng.random(2000), rng.random(2000)
    keep = np.hypot(x - 0.5, y - 0.5) > 0.1
    x, y = x[keep], y[keep]
    m = 40
    ang = 2 * np.pi * (np.arange(m) + rng.uniform(-0.05, 0.05, m)) / m
    rad = 0.03 * (1 + rng.uniform(-1e-3, 1e-3, m))
    x = np.concatenate([x, [0.5], 0.5 + rad * np.cos(ang)])
    y = np.concatenate([y, [0.5], 0.5 + rad * np.sin(ang)])
    ctx = T.Context(0)
    ctx.tm_set_domain(box, torch.from_numpy(configs.box_phi(box, 64)).cuda(), None, None, len(x))
    xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    bufs = T.IterBuffers.alloc(len(x))
    ctx.tm_grid_bin(xd, yd)
    ctx.tm_voronoi_delaunay(bufs.tri, bufs.n_tri)
    with pytest.raises(T.TmError) as e:
        ctx.tm_sync()
    assert e.value.code == T.TM_E_CAPACITY


def test_cocircular_input_is_reported_degenerate():
    """Four exactly cocircular points (a square): the Delaunay triangulation is not unique
    (P:43 assumes general position, reading L12).  The exact predicates meet a zero and the
    library counts it in n_degenerate (tm_mesh_stats) -- parity is only promised when 0."""
    import torch
    import paper_2309_13824_b200 as T
    box = (0.0, 0.0, 1.0, 1.0)
    x = np.array([0.25, 0.75, 0.75, 0.25])
    y = np.array([0.25, 0.25, 0.75, 0.75])
    ctx = T.Context(0)
    ctx.tm_set_domain(box, torch.from_numpy(configs.box_phi(box, 64)).cuda(), None, None, 4)
    xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    bufs = T.IterBuffers.alloc(4)
    ctx.tm_grid_bin(xd, yd)
    ctx.tm_voronoi_delaunay(bufs.tri, bufs.n_tri)
    st = ctx.tm_mesh_stats(xd, yd, bufs.tri, int(bufs.n_tri.item()))
    assert st.n_degenerate > 0


@pytest.mark.parametrize("k", [1, 3, 5])
def test_domain_constants_bitwise(k, cfg_cache):
    """S0 (reading L7): c and h_avg come from a sequential row-major sum over the grid
    cells with phi~(centre) < 0 -- the same order as the oracle's definition, so the
    same bits (cfg5: 2048^2 cells, several staging tiles and a ragged last one)."""
    import torch
    import paper_2309_13824_b200 as T
    c = cfg_cache(k)
    dev = torch.device("cuda", 0)
    to = lambda a: None if a is None else torch.from_numpy(a).to(dev)
    ctx = T.Context(0)
    gc, gh = ctx.tm_set_domain(c.box, to(c.phi), to(c.mu), to(c.rho), c.n)
    ctx.close()
    oc, oh = O.domain(O.FieldSet.from_config(c), c.n)
    assert gc == oc and gh == oh, (gc, oc, gh, oh)


def test_graph_replay_equals_eager(cfg_cache):
    """A captured DistMesh + CVD iteration pair (tm_graph_begin/end) replays to the same
    bits as the eager calls; synchronising calls are refused while capturing."""
    import torch
    import paper_2309_13824_b200 as T
    c = cfg_cache(2)
    stream = torch.cuda.Stream()
    ctx = T.Context(0, stream=stream)
    with torch.cuda.stream(stream):
        ctx.tm_set_domain(c.box, torch.from_numpy(c.phi).cuda(), None, None, c.n)
        x0, y0 = torch.from_numpy(c.x).cuda(), torch.from_numpy(c.y).cuda()
        bufs = T.IterBuffers.alloc(c.n)
        X = [torch.empty_like(x0) for _ in range(6)]

        def two():
            T.iterate(ctx, x0, y0, None, "dm", bufs, X[0], X[1], X[2])
            T.iterate(ctx, X[0], X[1], X[2], "cvd", bufs, X[3], X[4], X[5])

        two()  # warm-up (allocations, warm-start lists)
        two()
        ctx.tm_sync()
        eager = [t.cpu().numpy().copy() for t in X] + [bufs.tri[:int(bufs.n_tri.item())].cpu().numpy().copy()]
        assert np.all(np.isfinite(eager[3]))
        g = ctx.capture(two)
        for t in X:
            t.zero_()
        g.launch()
        ctx.tm_sync()
        replay = [t.cpu().numpy() for t in X] + [bufs.tri[:int(bufs.n_tri.item())].cpu().numpy()]
        for a, b in zip(eager[:6], replay[:6]):
            assert np.array_equal(a, b)
        assert tri_set_eq(eager[6], replay[6])
        T.load_library().tm_graph_begin(ctx.h)
        with pytest.raises(T.TmError) as e:
            ctx.tm_sync()
        assert e.value.code == T.TM_E_STATE
        import ctypes
        h = ctypes.c_void_p()
        T.load_library().tm_graph_end(ctx.h, ctypes.byref(h))
        T.load_library().tm_graph_destroy(h)
        g.close()
