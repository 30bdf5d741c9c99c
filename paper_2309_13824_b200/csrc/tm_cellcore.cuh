// tm_cellcore.cuh -- pieces shared by the two cell kernels (16/32-lane groups in
// tm_cells.cu, one thread per cell in tm_cells_t.cu): kernel modes, the canonical
// line of a code, the point-point vertex filter constant, the leaf-ring
// enumeration of the cell list and the canonical keep rule.
#pragma once
#include "tm_internal.cuh"

namespace tmg {

// M_WCERT (thread kernel): warm clips from the previous neighbour lists, then warp-cooperative
// certification of each cell (tm_cells_t.cu); without it the flat nearest-first search
enum : int { M_TRI = 1, M_ELL = 2, M_TREAT = 4, M_HAT = 8, M_COUNT = 16, M_RETRY = 32, M_WCERT = 64 };

// the cell's lines are recomputed from their codes (canonical, so identical bits)
struct CellGeom {
    double px, py, r_oct, bx0, by0, bx1, by1;
};

__device__ __forceinline__ Line line_of(int code, const CellGeom &cg_, const CellArgs &A) {
    if (code >= 0) return bisector(csub(__ldg(A.xs + code), cg_.px), csub(__ldg(A.ys + code), cg_.py));
    return wall_line(code, cg_.px, cg_.py, cg_.r_oct, cg_.bx0, cg_.by0, cg_.bx1, cg_.by1);
}

// filter constant of a point-point vertex x = cramer(A, B) with inv = 1/det:
// K = e_v + 8 eps |v|_1, e_v a rigorous bound on |x - exact circumcentre|
// (Cramer evaluation rounding plus the rounding of d = fl(p - p_i)), x2 safety.
__device__ __forceinline__ double pp_filter_K(const Line &A, const Line &B, double x, double y, double inv) {
    double n1a = fabs(A.nx) + fabs(A.ny), n1b = fabs(B.nx) + fabs(B.ny);
    double m1 = fabs(x) + fabs(y);
    double ev = EPS * (10.0 * (A.r * n1b + B.r * n1a + m1 * n1a * n1b) * fabs(inv) * (1.0 + 8.0 * EPS) + 3.0 * m1);
    return ev + 8.0 * EPS * m1;
}

struct ClipStats {
    unsigned long long exact = 0, clips = 0;
};

// ring k leaf q -> (dx, dy), Chebyshev distance k, q in [0, 8k)
__device__ __forceinline__ void ring_bin(int k, int q, int &dx, int &dy) {
    int side = 2 * k + 1;
    if (q < side) { dx = q - k; dy = -k; return; }
    q -= side;
    if (q < side) { dx = q - k; dy = k; return; }
    q -= side;
    if (q < side - 2) { dx = -k; dy = q - k + 1; return; }
    q -= side - 2;
    dx = k; dy = q - k + 1;
}

// canonical keep rule (§8(a) S3; P:499-510 Test 1 in its L10 reading)
__device__ __forceinline__ bool in_oct(double cx, double cy, double qx, double qy, double r) {
    double dx = csub(cx, qx), dy = csub(cy, qy);
    double r2 = cmul(SQRT2, r);
    return fabs(dx) < r && fabs(dy) < r && fabs(cadd(dx, dy)) < r2 && fabs(csub(dx, dy)) < r2;
}

// geps(x) = fac_geps * min(h(x), h_avg), h(x) = c mu~(x)   (reading L20 evaluated at x)
static __device__ __forceinline__ double geps_at(const CellArgs &A, double x, double y) {
    const double h = A.mu ? cmul(A.c, bilinear(A.grid, A.mu, x, y, LdgLoad())) : A.c;
    return cmul(A.fac_geps, h < A.h_avg ? h : A.h_avg);
}

// NEXT-2: the paper's validity tests (reading L43) after the bounded-cell conditions:
// Test 1 discards iff phi~(g) > geps(g); Test 2 keeps iff >= 2 edge midpoints have phi~(m) <=
// geps(m); Test 3 keeps iff |phi~(c)| / R_circ <= t_circ.  Same operations as the oracle.
static __device__ __forceinline__ bool validity_tests(const CellArgs &A, double x0, double y0, double x1, double y1,
                                                      double x2, double y2, double gx, double gy, double ox, double oy,
                                                      double cx, double cy) {
    // inlined, scalars: a call (or an array argument) would cost every keep_tri a local-memory
    // frame, validity on or off (measured: +4..9 % per CVD iteration)
    if (bilinear(A.grid, A.phi, gx, gy, LdgLoad()) > geps_at(A, gx, gy)) return false;  // Test 1
    int count = 0;
    {   // Test 2: edges (u,v), (v,w), (w,u)
        const double mx0 = cmul(cadd(x0, x1), 0.5), my0 = cmul(cadd(y0, y1), 0.5);
        const double mx1 = cmul(cadd(x1, x2), 0.5), my1 = cmul(cadd(y1, y2), 0.5);
        const double mx2 = cmul(cadd(x2, x0), 0.5), my2 = cmul(cadd(y2, y0), 0.5);
        count += bilinear(A.grid, A.phi, mx0, my0, LdgLoad()) <= geps_at(A, mx0, my0) ? 1 : 0;
        count += bilinear(A.grid, A.phi, mx1, my1, LdgLoad()) <= geps_at(A, mx1, my1) ? 1 : 0;
        count += bilinear(A.grid, A.phi, mx2, my2, LdgLoad()) <= geps_at(A, mx2, my2) ? 1 : 0;
    }
    if (count >= 2) return true;
    const double R = sqrt(cadd(cmul(ox, ox), cmul(oy, oy)));  // Test 3
    return !(cdiv(fabs(bilinear(A.grid, A.phi, cx, cy, LdgLoad())), R) > A.t_circ);
}

// su,sv,sw: slots ordered by gid (u smallest); (ox,oy): canonical circumcentre relative to p_u
static __device__ __forceinline__ bool keep_tri(const CellArgs &A, int su, int sv, int sw, double ox, double oy) {
    const int s3[3] = {su, sv, sw};
    double X[3], Y[3];
#pragma unroll
    for (int k = 0; k < 3; k++) {
        X[k] = __ldg(A.xs + s3[k]);
        Y[k] = __ldg(A.ys + s3[k]);
    }
    const double cx = cadd(X[0], ox), cy = cadd(Y[0], oy);
    if (!(cx > A.grid.x0 && cx < A.grid.x1 && cy > A.grid.y0 && cy < A.grid.y1)) return false;
#pragma unroll
    for (int k = 0; k < 3; k++) {
        double r = cmul(cmul(A.fac_voro, __ldg(A.hs + s3[k])), COS_PI8);
        if (!in_oct(cx, cy, X[k], Y[k], r)) return false;
    }
    double gx = cdiv(cadd(cadd(X[0], X[1]), X[2]), 3.0);
    double gy = cdiv(cadd(cadd(Y[0], Y[1]), Y[2]), 3.0);
    if (A.validity) return validity_tests(A, X[0], Y[0], X[1], Y[1], X[2], Y[2], gx, gy, ox, oy, cx, cy);
    return bilinear(A.grid, A.phi, gx, gy, LdgLoad()) < A.keep_tol;
}

// ---- S4a adaptive quadrature over a ring stored in canonical order (shared by k_output_t
// and the group kernel, which gathers its ring into shared memory first)
// one longest-edge bisection of sub-triangle Q (Fig. 14): child `bit`
// (0: (a, m, c), 1: (m, b, c) with ab the longest edge, m its midpoint)
__device__ __forceinline__ void quad_split(const double Q[3][2], int bit, double C[3][2]) {
    double best = -1.0;
    int eidx = 0;
#pragma unroll
    for (int q = 0; q < 3; q++) {
        const int q1 = q == 2 ? 0 : q + 1;
        const double ddx = csub(Q[q1][0], Q[q][0]), ddy = csub(Q[q1][1], Q[q][1]);
        const double Lq = cadd(cmul(ddx, ddx), cmul(ddy, ddy));
        if (Lq > best) { best = Lq; eidx = q; }
    }
    // edge (a, b) = (Q[e], Q[e+1]), c the third vertex; selects, not indexing (registers)
    const double ax = eidx == 0 ? Q[0][0] : (eidx == 1 ? Q[1][0] : Q[2][0]);
    const double ay = eidx == 0 ? Q[0][1] : (eidx == 1 ? Q[1][1] : Q[2][1]);
    const double bx = eidx == 0 ? Q[1][0] : (eidx == 1 ? Q[2][0] : Q[0][0]);
    const double by = eidx == 0 ? Q[1][1] : (eidx == 1 ? Q[2][1] : Q[0][1]);
    const double cx = eidx == 0 ? Q[2][0] : (eidx == 1 ? Q[0][0] : Q[1][0]);
    const double cy = eidx == 0 ? Q[2][1] : (eidx == 1 ? Q[0][1] : Q[1][1]);
    const double mx = cmul(cadd(ax, bx), 0.5), my = cmul(cadd(ay, by), 0.5);
    if (bit) {
        C[0][0] = mx; C[0][1] = my; C[1][0] = bx; C[1][1] = by;
    } else {
        C[0][0] = ax; C[0][1] = ay; C[1][0] = mx; C[1][1] = my;
    }
    C[2][0] = cx; C[2][1] = cy;
}

// sub-triangle of fan triangle (0, a, b) reached by `levels` bisections along `path`
// (bit lev taken at level lev, from the top)
__device__ __forceinline__ void quad_descend(const double2 a, const double2 b, int levels, int64_t path,
                                             double Q[3][2]) {
    Q[0][0] = 0.0; Q[0][1] = 0.0; Q[1][0] = a.x; Q[1][1] = a.y; Q[2][0] = b.x; Q[2][1] = b.y;
    for (int lev = levels - 1; lev >= 0; lev--) {
        double C[3][2];
        quad_split(Q, (int)((path >> lev) & 1), C);
#pragma unroll
        for (int q = 0; q < 3; q++) { Q[q][0] = C[q][0]; Q[q][1] = C[q][1]; }
    }
}

// area and centroid of a sub-triangle, and its density corners
__device__ __forceinline__ void quad_leaf(const double Q[3][2], const CellArgs &A, double px, double py, double &At,
                                          double &qx, double &qy, double &ss, double &tt, double f[4]) {
    const double cr = csub(cmul(csub(Q[1][0], Q[0][0]), csub(Q[2][1], Q[0][1])),
                           cmul(csub(Q[1][1], Q[0][1]), csub(Q[2][0], Q[0][0])));
    At = cmul(0.5, cr);
    qx = div3(cadd(cadd(Q[0][0], Q[1][0]), Q[2][0]));
    qy = div3(cadd(cadd(Q[0][1], Q[1][1]), Q[2][1]));
    int gi, gj;
    grid_cell(A.grid, cadd(px, qx), cadd(py, qy), gi, gj, ss, tt);
    if (A.rho4) {  // packed corners (S0): one 32-byte sector per lookup, the same four values
        const double2 *c = reinterpret_cast<const double2 *>(A.rho4 + (int64_t)gj * (A.grid.nx - 1) + gi);
        const double2 lo = __ldg(c), hi = __ldg(c + 1);
        f[0] = lo.x;
        f[1] = lo.y;
        f[2] = hi.x;
        f[3] = hi.y;
        return;
    }
    const double *r0 = A.rho + (int64_t)gj * A.grid.nx + gi, *r1 = r0 + A.grid.nx;
    f[0] = __ldg(r0);
    f[1] = __ldg(r0 + 1);
    f[2] = __ldg(r1);
    f[3] = __ldg(r1 + 1);
}

// adaptive quadrature over a stored ring (ring order from the canonical vertex); the
// same sub-triangles and sums, in the same order, as quad_centroid_t.  Sub-triangles
// are taken two at a time with their density loads in flight together (the kernel is
// bound by the latency of those loads); below level 1 the two are siblings, so the
// descent to their parent is shared.
// Levels beyond `lmax` (< quad_max) are left to a later pass: returns false then, with (cx, cy) the
// centroid of level lmax (the later pass's previous level).
static __device__ bool quad_centroid_g(const double2 *rv, int64_t ns, int nv, double px, double py, double area,
                                       double h, double dprev, const CellArgs &A, double &cx, double &cy,
                                       unsigned long long &nq, int lmax) {
    double eps = dprev >= 0.0 ? cdiv(dprev, h) : A.fac_pt;
    if (eps < A.fac_end) eps = A.fac_end;
    const double E = cmul(sqrt(area), eps);
    double prevx = 0.0, prevy = 0.0;
    bool done = false;
    for (int L = 1; L <= A.quad_max; L++) {
        if (L > lmax) {  // the last level's centroid: the later pass continues from it
            cx = prevx;
            cy = prevy;
            return false;
        }
        const int depth = L - 1;
        const int64_t ntot = (int64_t)nv << depth;
        double sw = 0.0, swx = 0.0, swy = 0.0;
        for (int64_t t0 = 0; t0 < ntot; t0 += 2) {
            double At[2], qx[2], qy[2], ss[2], tt[2], f[2][4];
            if (depth == 0) {  // fan triangles t0, t0 + 1 (the last one again for odd nv)
#pragma unroll
                for (int u = 0; u < 2; u++) {
                    const int fi = (int)(t0 + u < ntot ? t0 + u : ntot - 1);
                    double Q[3][2];
                    quad_descend(rv[(int64_t)fi * ns], rv[(int64_t)(fi + 1 == nv ? 0 : fi + 1) * ns], 0, 0, Q);
                    quad_leaf(Q, A, px, py, At[u], qx[u], qy[u], ss[u], tt[u], f[u]);
                }
            } else {           // siblings t0, t0 + 1 of parent t0 / 2
                const int64_t par = t0 >> 1;
                const int fi = (int)(par >> (depth - 1));
                double Q[3][2];
                quad_descend(rv[(int64_t)fi * ns], rv[(int64_t)(fi + 1 == nv ? 0 : fi + 1) * ns], depth - 1,
                             par & (((int64_t)1 << (depth - 1)) - 1), Q);
#pragma unroll
                for (int u = 0; u < 2; u++) {
                    double C[3][2];
                    quad_split(Q, u, C);
                    quad_leaf(C, A, px, py, At[u], qx[u], qy[u], ss[u], tt[u], f[u]);
                }
            }
#pragma unroll
            for (int u = 0; u < 2; u++) {
                if (t0 + u >= ntot) break;
                const double rho = clerp(clerp(f[u][0], f[u][1], ss[u]), clerp(f[u][2], f[u][3], ss[u]), tt[u]);
                const double wgt = cmul(At[u], rho);
                sw = cadd(sw, wgt);
                swx = cadd(swx, cmul(wgt, qx[u]));
                swy = cadd(swy, cmul(wgt, qy[u]));
                nq++;
            }
        }
        const double curx = cdiv(swx, sw), cury = cdiv(swy, sw);
        const double dx = csub(prevx, curx), dy = csub(prevy, cury);
        const double dist = sqrt(cadd(cmul(dx, dx), cmul(dy, dy)));
        prevx = curx;
        prevy = cury;
        if (dist < E) {
            done = true;
            break;
        }
    }
    (void)done;  // converged, or the level cap of the method (L13) reached
    cx = prevx;
    cy = prevy;
    return true;
}

// S4a over a ring stored in canonical order rv[i * ns] (relative to p_i): the fan/shoelace
// sums in ring order, uncontracted, as the oracle's O4; non-uniform rho takes the
// adaptive quadrature.  Returns the centroid relative to p_i.
// lmax: see quad_centroid_g (false: the cell needs more quadrature levels than this pass does).
static __device__ bool ring_centroid(const double2 *rv, int64_t ns, int nv, double px, double py, double h,
                                     double dprev, const CellArgs &A, double &cx, double &cy, unsigned long long &nq,
                                     int lmax = 1 << 30) {
    double S2 = 0.0, sx = 0.0, sy = 0.0;
    for (int i = 0; i < nv; i++) {
        const double2 a = rv[(int64_t)i * ns], b = rv[(int64_t)(i + 1 == nv ? 0 : i + 1) * ns];
        const double cr = csub(cmul(a.x, b.y), cmul(b.x, a.y));
        S2 = cadd(S2, cr);
        sx = cadd(sx, cmul(cr, cadd(a.x, b.x)));
        sy = cadd(sy, cmul(cr, cadd(a.y, b.y)));
    }
    if (A.rho == nullptr) {
        cx = cdiv(sx, cmul(3.0, S2));
        cy = cdiv(sy, cmul(3.0, S2));
        nq += nv;
    } else {
        return quad_centroid_g(rv, ns, nv, px, py, cmul(0.5, S2), h, dprev, A, cx, cy, nq, lmax);
    }
    return true;
}

// thread-per-cell launcher (tm_cells_t.cu), explicitly instantiated for every mode
template <int MODE>
tm_status launch_cells_thread(tm_ctx *ctx, const CellArgs &a);

}  // namespace tmg
