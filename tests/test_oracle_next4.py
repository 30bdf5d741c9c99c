"""Pins for the NEXT-4 oracle pieces (SURVEY §8(f) set-up pipeline): geometry grid size and
categories, contour SDF, Floyd-Steinberg point initialisation
(P:380-406).  Expected values are closed forms, the paper's worked numbers, or hand derivations."""
import math

import numpy as np

import oracle as O
from inputs import configs


def test_geometry_grid_of_the_worked_example():
    """N_total = 5000 (custom shape on the unit square, N_opt = 3.3, fac_grid = 5, Table B.1)
    gives a 195 x 195 geometry grid: lambda = sqrt(5000/3.3) = 38.92 -> 39 -> x5."""
    assert O.geometry_grid_dims(5000, (0.0, 0.0, 1.0, 1.0)) == (195, 195)
    # a 2 x 1 box: lambda = sqrt(N / (3.3 * 2)); n = (ceil(2 lambda), ceil(lambda)) x 5
    lam = math.sqrt(20000 / (3.3 * 2))
    assert O.geometry_grid_dims(20000, (0.0, 0.0, 2.0, 1.0)) == (5 * math.ceil(2 * lam), 5 * math.ceil(lam))


def test_library_geometry_grid_dims_matches():
    import paper_2309_13824_b200 as T
    for n, box in [(5000, (0, 0, 1, 1)), (10 ** 6, (-1, -1, 1, 1)), (777, (0, 0, 3, 0.5))]:
        assert T.geometry_grid_dims(n, box) == O.geometry_grid_dims(n, box)


def test_categories_of_a_half_plane():
    """phi = x - 1/2 (exactly bilinear): a cell is boundary iff |m_x - 1/2| <= l_diag (closed form
    per column), inner left of the band, outer right of it."""
    box = (0.0, 0.0, 1.0, 1.0)
    g = configs.node_coords(0, 1, 33)
    X, Y = np.meshgrid(g, g)
    fs = O.FieldSet(box, X - 0.5)
    nx, ny = 40, 25
    cat = O.geometry_categories(fs, nx, ny)
    dx, dy = 1 / nx, 1 / ny
    ld = math.hypot(dx, dy)
    for i in range(nx):
        m = (i + 0.5) * dx - 0.5
        exp = 1 if abs(m) <= ld else (0 if m < 0 else 2)
        assert (cat[:, i] == exp).all(), i


def _square(n_per_side=1, cw=True):
    P = [(0.0, 0.0), (0.0, 1.0), (1.0, 1.0), (1.0, 0.0)]  # clockwise
    if not cw:
        P = P[::-1]
    segs = []
    for k in range(4):
        a, b = np.array(P[k]), np.array(P[(k + 1) % 4])
        for q in range(n_per_side):
            segs.append([*(a + (b - a) * q / n_per_side), *(a + (b - a) * (q + 1) / n_per_side)])
    return np.array(segs)


def _square_sdf(x, y):
    dx = max(-x, x - 1.0)
    dy = max(-y, y - 1.0)
    if dx <= 0 and dy <= 0:
        return max(dx, dy)
    return math.hypot(max(dx, 0.0), max(dy, 0.0))


def test_contour_sdf_of_the_unit_square():
    """Closed form of the square's SDF (inside: minus the distance to the nearest side; outside:
    the distance to the square, rounded at the corners) on a node grid around it; splitting the
    sides into segments does not change it; a counter-clockwise loop flips the sign."""
    box = (-0.5, -0.5, 1.5, 1.5)
    phi = O.contour_sdf(_square(), 41, 41, box)
    phi5 = O.contour_sdf(_square(5), 41, 41, box)
    g = configs.node_coords(-0.5, 1.5, 41)
    for j in range(41):
        for i in range(41):
            e = _square_sdf(g[i], g[j])
            assert abs(phi[j, i] - e) <= 1e-15, (i, j, phi[j, i], e)
            assert abs(phi5[j, i] - e) <= 1e-15
    ccw = O.contour_sdf(_square(cw=False), 41, 41, box)
    inside = phi < -1e-12
    assert (ccw[inside] > 0).all()


def test_contour_sdf_of_an_l_shape():
    """L = [0,2]x[0,1] u [0,1]x[1,2] (clockwise).  Inside near the reflex corner (1,1) the closest
    boundary point is that corner (an endpoint of two segments: the averaged normal decides the
    sign); outside beyond the convex corner (2,1) too; elsewhere the nearest edge."""
    P = [(0, 0), (0, 2), (1, 2), (1, 1), (2, 1), (2, 0)]
    segs = np.array([[*P[k], *P[(k + 1) % 6]] for k in range(6)], dtype=float)
    assert abs(O.contour_sdf_point(segs, 0.9, 0.7) + math.hypot(0.1, 0.3)) < 1e-15  # inside, reflex corner
    assert abs(O.contour_sdf_point(segs, 2.3, 1.4) - math.hypot(0.3, 0.4)) < 1e-15  # outside, convex corner
    assert abs(O.contour_sdf_point(segs, 1.3, 1.4) - 0.3) < 1e-15                  # outside, edge x = 1
    assert abs(O.contour_sdf_point(segs, 0.5, 0.5) - (-0.5)) < 1e-15
    assert abs(O.contour_sdf_point(segs, 2.5, 0.5) - 0.5) < 1e-15


def _all_inner(n=9):
    box = (0.0, 0.0, 1.0, 1.0)
    g = configs.node_coords(0, 1, n)
    X, Y = np.meshgrid(g, g)
    return O.FieldSet(box, np.full_like(X, -10.0)), box


def test_init_counts_uniform_and_hand_worked():
    """All-inner grid, uniform density: N_init = 3 x cells puts exactly 3 in every cell.  A 2 x 2 grid
    with N_init = 2 (n_E = 1/2 each), by hand: top-left v = 1/2 -> 1, R = -1/2 to its 3 valid later
    neighbours (-1/6 each); top-right v = 1/3 -> 0, R = 1/3 to below-left and below (+1/6 each);
    bottom-left v = 1/2 -> 1 (R = -1/2 to its right); bottom-right v = 0 -> 0."""
    fs, box = _all_inner()
    cat = np.zeros((4, 5), dtype=np.int8)
    cnt, tot = O.init_counts(fs, cat, 3 * 20)
    assert tot == 60 and (cnt == 3).all()
    cat2 = np.zeros((2, 2), dtype=np.int8)
    cnt2, tot2 = O.init_counts(fs, cat2, 2)
    assert tot2 == 2
    assert cnt2[1, 0] == 1 and cnt2[1, 1] == 0 and cnt2[0, 0] == 1 and cnt2[0, 1] == 0


def test_init_counts_follow_density_and_band():
    """rho = 1 + 3 [x > 1/2] on the unit disk: the total is N_init within one point (dithering keeps
    the running residual bounded), the right half gets ~3/4 of the points, boundary cells beyond
    the eta band and outer cells get none."""
    box = (-1.1, -1.1, 1.1, 1.1)
    n = 129
    g = configs.node_coords(box[0], box[2], n)
    X, Y = np.meshgrid(g, g)
    phi = np.sqrt(X * X + Y * Y) - 1.0
    rho = 1.0 + 3.0 * (X > 0.0)
    fs = O.FieldSet(box, phi, rho=rho)
    nxg = nyg = 60
    cat = O.geometry_categories(fs, nxg, nyg)
    cnt, tot = O.init_counts(fs, cat, 20000.0)
    assert abs(tot - 20000) <= 1
    dxg = (box[2] - box[0]) / nxg
    mx = box[0] + (np.arange(nxg) + 0.5) * dxg
    right = cnt[:, mx > 0.02].sum() / tot
    assert 0.70 < right < 0.80
    phim = O.geometry_categories(fs, nxg, nyg)
    assert cnt[cat == 2].sum() == 0
    for j in range(nyg):
        for i in range(nxg):
            if cat[j, i] == 1:
                m = (box[0] + (i + 0.5) * dxg, box[1] + (j + 0.5) * dxg)
                if math.hypot(*m) - 1.0 > 0.5 * dxg + 1e-3:
                    assert cnt[j, i] == 0


def _splitmix_u01(seed, k, comp):
    M = (1 << 64) - 1
    z = (seed + (2 * k + comp + 1) * 0x9E3779B97F4A7C15) & M
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
    z ^= z >> 31
    return (z >> 11) * 2.0 ** -53


def test_init_points_in_their_cells_and_projected():
    box = (-1.1, -1.1, 1.1, 1.1)
    n = 129
    g = configs.node_coords(box[0], box[2], n)
    X, Y = np.meshgrid(g, g)
    fs = O.FieldSet(box, np.sqrt(X * X + Y * Y) - 1.0)
    nxg = nyg = 40
    cat = O.geometry_categories(fs, nxg, nyg)
    cnt, tot = O.init_counts(fs, cat, 3000.0)
    c, ha = O.domain(fs, tot)
    x, y = O.init_points(fs, cnt, 7, c, ha)
    assert len(x) == tot
    d = (box[2] - box[0]) / nxg
    geps = 0.01 * min(c, ha)
    k = 0
    for j in range(nyg - 1, -1, -1):
        for i in range(nxg):
            for q in range(cnt[j, i]):
                ex = box[0] + i * d + _splitmix_u01(7, k, 0) * d
                ey = box[1] + j * d + _splitmix_u01(7, k, 1) * d
                if O.field_value(fs, "phi", ex, ey) <= geps:
                    assert x[k] == ex and y[k] == ey  # the generator, bit for bit
                else:
                    assert abs(O.field_value(fs, "phi", x[k], y[k])) <= geps  # projected
                k += 1


def _circle(n=400, r=0.3, c=(0.5, 0.5)):
    P = [(c[0] + r * math.cos(-2 * math.pi * k / n), c[1] + r * math.sin(-2 * math.pi * k / n)) for k in range(n)]
    return np.array([[*P[k], *P[(k + 1) % n]] for k in range(n)])


def test_boundary_points_are_trimmed_to_spacing():
    """App. A: after trimming every point's nearest neighbour is at least d_s away,
    and a circle of perimeter 2 pi r keeps between 2 pi r / (2 d_s) and 2 pi r / d_s points."""
    segs = _circle(300)
    d_s = 0.01
    x, y = O.boundary_points(segs, d_s, 1e-3)
    P = np.stack([x, y], 1)
    D = np.sqrt(((P[:, None, :] - P[None, :, :]) ** 2).sum(-1)) + np.eye(len(x))
    assert D.min() >= d_s
    per = 2 * math.pi * 0.3
    assert per / (2 * d_s) <= len(x) <= per / d_s
    assert np.abs(np.hypot(x - 0.5, y - 0.5) - 0.3).max() < 1e-3  # on the boundary


def test_medial_axis_and_sizing_of_a_circle():
    """A circle's medial axis is its centre: the poles gather there, lfs(s) = r for every
    boundary point, and mu(x) = K (r - |x - c|) + r inside (Eq. sizing field)."""
    segs = _circle(300)
    x, y = O.boundary_points(segs, 0.01, 1e-3)
    box = (0.0, 0.0, 1.0, 1.0)
    mx, my = O.medial_points(x, y, box, r_nei=2 * 3 * 0.01, n_thres=3)
    assert len(mx) > 0 and np.hypot(mx - 0.5, my - 0.5).max() < 0.01
    K = 0.2
    mu, lfs = O.sizing_field(x, y, mx, my, K, 21, 21, box)
    assert np.abs(lfs - 0.3).max() < 0.01
    g = configs.node_coords(0, 1, 21)
    for j in range(21):
        for i in range(21):
            rho = math.hypot(g[i] - 0.5, g[j] - 0.5)
            if rho < 0.25:
                assert abs(mu[j, i] - (K * (0.3 - rho) + 0.3)) < 0.012, (i, j)


def test_lfs_of_a_thin_strip_is_its_half_thickness():
    """Rectangle [0.1, 0.9] x [0.45, 0.55] (clockwise): the medial axis of the long part is the
    centre line, so boundary points on the long sides away from the ends have lfs = 0.05."""
    P = [(0.1, 0.45), (0.1, 0.55), (0.9, 0.55), (0.9, 0.45)]
    segs = np.array([[*P[k], *P[(k + 1) % 4]] for k in range(4)])
    x, y = O.boundary_points(segs, 0.01, 1e-3)
    mx, my = O.medial_points(x, y, (0.0, 0.0, 1.0, 1.0), r_nei=0.06, n_thres=3)
    _, lfs = O.sizing_field(x, y, mx, my, 0.1, 5, 5, (0.0, 0.0, 1.0, 1.0))
    mid = (x > 0.3) & (x < 0.7)
    assert mid.sum() > 20
    assert np.abs(lfs[mid] - 0.05).max() < 0.006


def test_adf_on_straight_edges_needs_no_refinement_and_caps_depth():
    """P:457-472.  Inside a square, along an edge away from the corners, the SDF is linear, so the
    root's bilinear interpolant is exact at the 5 check points and the cell stays a single leaf;
    where the distance bends (corners) cells refine.  With a vanishing tolerance every boundary cell
    becomes a full tree of depth max_depth: (4^(d+1) - 1) / 3 nodes each."""
    segs = _square()
    box = (-0.5, -0.5, 1.5, 1.5)
    g = configs.node_coords(-0.5, 1.5, 65)
    X, Y = np.meshgrid(g, g)
    phi = O.contour_sdf(segs, 65, 65, box)
    fs = O.FieldSet(box, phi)
    nxg = nyg = 40
    cat = O.geometry_categories(fs, nxg, nyg)
    c, ha = O.domain(fs, 4000)
    adf = O.ADF(fs, c, ha, cat, segs)
    nb = int((cat == 1).sum())
    assert nb < adf.n_nodes  # some refinement (around the corners)
    # a boundary cell in the middle of the left edge (x = 0, y = 0.5), inside: a single leaf, exact
    d = 2.0 / nxg
    xs = [0.01, 0.02, 0.03]
    for x in xs:
        assert abs(adf(x, 0.5) - (-x)) < 1e-15
    # where the distance is linear the interpolant is exact (error 0 is never > E_tol): with a
    # vanishing tolerance only the curved cells refine, to the depth cap and no further
    full = O.ADF(fs, c, ha, cat, segs, fac_etol=1e-300, max_depth=3)
    assert nb < full.n_nodes <= nb * (1 + 4 + 16 + 64) and (full.n_nodes - nb) % 4 == 0
    segc = _circle(300)
    phic = O.contour_sdf(segc, 65, 65, box)
    fsc = O.FieldSet(box, phic)
    catc = O.geometry_categories(fsc, nxg, nyg)
    nbc = int((catc == 1).sum())
    fullc = O.ADF(fsc, c, ha, catc, segc, fac_etol=1e-300, max_depth=3)
    assert fullc.n_nodes == nbc * (1 + 4 + 16 + 64) and fullc.n_leaves == nbc * 64


def test_adf_error_bounded_on_a_circle():
    """A circle contour: the ADF agrees with the exact contour SDF within a few E_tol at random points
    of the boundary cells (E_tol bounds the error at each leaf's 5 check points), and a tighter
    tolerance refines more."""
    segs = _circle(300)
    box = (0.0, 0.0, 1.0, 1.0)
    phi = O.contour_sdf(segs, 129, 129, box)
    fs = O.FieldSet(box, phi)
    nxg = nyg = 50
    cat = O.geometry_categories(fs, nxg, nyg)
    c, ha = O.domain(fs, 5000)
    adf = O.ADF(fs, c, ha, cat, segs)
    fine = O.ADF(fs, c, ha, cat, segs, fac_etol=0.01)
    assert fine.n_nodes > adf.n_nodes
    etol = 0.1 * 0.01 * min(c, ha)
    rng = np.random.default_rng(2)
    d = 1.0 / nxg
    checked = 0
    for j, i in zip(*np.nonzero(cat == 1)):
        for _ in range(3):
            x, y = (i + rng.random()) * d, (j + rng.random()) * d
            assert abs(adf(x, y) - O.contour_sdf_point(segs, x, y)) <= 4 * etol
            checked += 1
    assert checked > 100
    assert math.isnan(adf(0.5, 0.5))  # an inner cell: no ADF
