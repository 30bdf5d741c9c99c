"""Pins for the NEXT-1 oracle pieces: the paper's treatment of escaped
points (Fig. 13: sphere tracing from an inner p_old; damped 2x2 Newton
projection with finite-difference derivatives from a boundary p_old) and the
lazy re-triangulation of Alg. 1 (threshold P:446 / P:1098)."""
import math

import numpy as np

import oracle as O
from inputs import configs

BOX = (0.0, 0.0, 1.0, 1.0)


def _grid(n, box=BOX):
    gx = configs.node_coords(box[0], box[2], n)
    gy = configs.node_coords(box[1], box[3], n)
    return np.meshgrid(gx, gy)


PAPER = dict(projection=1)


def test_sphere_tracing_planar_boundary_hits_the_segment():
    """phi = x - 1/2 (exactly bilinear).  From the inner p_old = (0.3, 0.4) toward p_new =
    (0.6, 0.55) the segment meets the boundary at (0.5, 0.5): sphere tracing must end on the
    segment, within geps of the boundary, approaching from inside (status 1 | 8)."""
    X, Y = _grid(33)
    fs = O.FieldSet(BOX, X - 0.5)
    c, havg = O.domain(fs, 1)
    p = O.default_params(**PAPER)
    (qx, qy), dp, st = O.treat(fs, c, havg, (0.3, 0.4), (0.6, 0.55), params=p)
    geps = 0.01 * min(c, havg)
    assert st & 8 and st & 1 and not st & 2
    assert abs(qx - 0.5) <= geps and qx <= 0.5 + 1e-15
    # on the segment: collinear with p_old -> p_new, and between them
    assert abs((qx - 0.3) * 0.15 - (qy - 0.4) * 0.3) < 1e-15
    assert 0.3 < qx < 0.6
    assert abs(qy - (0.4 + (qx - 0.3) * 0.5)) < 1e-15


def test_sphere_tracing_disk_matches_segment_circle_intersection():
    """Unit disk phi = |x| - 1 on a 513^2 grid: the traced point is the intersection of the
    segment with the circle (quadratic root), within geps + the grid's interpolation error."""
    box = (-1.5, -1.5, 1.5, 1.5)
    fs = O.FieldSet(box, configs.disk_phi(box, 513))
    c, havg = O.domain(fs, 5)  # h ~ 0.8: no move clamp for these short moves
    p = O.default_params(**PAPER)
    geps = 0.01 * min(c, havg)
    for (xo, yo), (xn, yn) in [((0.85, 0.2), (1.0, 0.25)), ((-0.3, 0.9), (-0.33, 1.02)), ((0.0, -0.95), (0.02, -1.04))]:
        (qx, qy), dp, st = O.treat(fs, c, havg, (xo, yo), (xn, yn), params=p)
        assert st & 8 and st & 1, st
        # analytic: |p_o + t (p_n - p_o)| = 1
        dx, dy = xn - xo, yn - yo
        a, b, cc = dx * dx + dy * dy, 2 * (xo * dx + yo * dy), xo * xo + yo * yo - 1
        t = (-b + math.sqrt(b * b - 4 * a * cc)) / (2 * a)
        ex, ey = xo + t * dx, yo + t * dy
        assert math.hypot(qx - ex, qy - ey) <= geps * 1.5 + 2e-5, (qx, qy, ex, ey)
        assert abs((qx - xo) * dy - (qy - yo) * dx) < 1e-14  # on the segment


def test_newton_projection_planar_one_step():
    """phi = x - 1/2, boundary p_old (|phi| <= geps): L(p) = [phi, (p - p_new) x grad phi]
    has the closest point (1/2, y_new) as root and the Newton step reaches it in one step
    (J = [[1, 0], [0, -1]] up to the finite-difference rounding of a linear field)."""
    X, Y = _grid(33)
    fs = O.FieldSet(BOX, X - 0.5)
    c, havg = O.domain(fs, 1)
    p = O.default_params(**PAPER)
    (qx, qy), dp, st = O.treat(fs, c, havg, (0.4995, 0.3), (0.6, 0.32), params=p)
    assert st & 1 and not st & 8 and not st & 2
    assert abs(qx - 0.5) < 1e-9 and abs(qy - 0.32) < 1e-9


def test_newton_projection_disk_closest_point():
    """Unit disk: from a boundary p_old, p_new outside projects to the closest circle point
    p_new / |p_new| (the normal direction), within geps and the grid error."""
    box = (-1.5, -1.5, 1.5, 1.5)
    fs = O.FieldSet(box, configs.disk_phi(box, 513))
    c, havg = O.domain(fs, 5)
    p = O.default_params(**PAPER)
    geps = 0.01 * min(c, havg)
    for ang in np.linspace(0.1, 6.0, 9):
        xo, yo = math.cos(ang), math.sin(ang)
        xn, yn = 1.03 * math.cos(ang + 0.01), 1.03 * math.sin(ang + 0.01)
        (qx, qy), dp, st = O.treat(fs, c, havg, (xo, yo), (xn, yn), params=p)
        assert st & 1 and not st & 8, st
        r = math.hypot(xn, yn)
        assert math.hypot(qx - xn / r, qy - yn / r) <= 2 * geps, ang
        assert abs(O.field_value(fs, "phi", qx, qy)) <= geps


def test_paper_projection_keeps_accepted_points_and_falls_back():
    """Points that stay inside are untouched by the projection mode; a point whose
    projection cannot succeed (constant positive phi: no boundary) falls back to p_old."""
    fs = O.FieldSet(BOX, configs.box_phi(BOX, 64))
    c, havg = O.domain(fs, 100)
    for proj in (0, 1):
        p = O.default_params(projection=proj)
        assert O.treat(fs, c, havg, (0.5, 0.5), (0.52, 0.5), params=p) == O.treat(fs, c, havg, (0.5, 0.5),
                                                                                  (0.52, 0.5))
    fs2 = O.FieldSet(BOX, np.full((8, 8), 0.3))
    (qx, qy), dp, st = O.treat(fs2, c, havg, (0.5, 0.5), (0.51, 0.5), params=O.default_params(**PAPER))
    assert st == 2 and (qx, qy) == (0.5, 0.5) and dp == 0.0


def test_lazy_distmesh_on_fresh_edges_equals_the_eager_iteration(cfg_cache):
    """With the edges of the current triangulation (x_tria = x), the lazy update is the
    eager DistMesh iteration bit for bit (same edges, same force loop, same treatment)."""
    c = cfg_cache(2)
    fs = O.FieldSet.from_config(c)
    r = O.iteration(fs, c.x, c.y, "dm")
    lz = O.distmesh_lazy(fs, c.x, c.y, r.edges, c.x, c.y)
    assert np.array_equal(lz.x, r.x) and np.array_equal(lz.y, r.y) and np.array_equal(lz.status, r.status)
    # the first DistMesh steps from random points move far more than 0.1 h: re-triangulate
    assert lz.retria


def test_lazy_retria_threshold_closed_form():
    """Two points, one edge of length l = 0.2, uniform mu, N = 2 in the unit square:
    h = c = 2^-1/2, each point moves dt (l0 - l) = 0.2 * 0.2 l = 0.008 (Eq. spring force,
    L1-L4).  fac_retria = 0.1: 0.008 < 0.0707, no re-triangulation; fac_retria = 0.01:
    0.008 > 0.00707, re-triangulation."""
    fs = O.FieldSet(BOX, configs.box_phi(BOX, 64))
    x, y = np.array([0.4, 0.6]), np.array([0.5, 0.5])
    E = np.array([[0, 1]], np.int32)
    lz = O.distmesh_lazy(fs, x, y, E, x, y)
    assert abs(lz.x[0] - (0.4 - 0.008)) < 1e-15 and abs(lz.x[1] - (0.6 + 0.008)) < 1e-15
    assert not lz.retria
    lz2 = O.distmesh_lazy(fs, x, y, E, x, y, params=O.default_params(fac_retria=0.01))
    assert lz2.retria
    # displacement counts from the triangulation, not from the last step: x_tria far away
    lz3 = O.distmesh_lazy(fs, x, y, E, x - 0.1, y)
    assert lz3.retria
