// tm_cellcore.cuh -- pieces shared by the two cell kernels (16/32-lane groups in
// tm_cells.cu, one thread per cell in tm_cells_t.cu): kernel modes, the canonical
// line of a code, the point-point vertex filter constant, the leaf-ring
// enumeration of the cell list and the canonical keep rule.
#pragma once
#include "tm_internal.cuh"

namespace tmg {

enum : int { M_TRI = 1, M_ELL = 2, M_TREAT = 4, M_HAT = 8, M_COUNT = 16, M_RETRY = 32 };

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

static __device__ bool keep_tri(const CellArgs &A, int su, int sv, int sw, double cx, double cy) {
    // su,sv,sw: slots ordered by gid (u smallest); (cx,cy) canonical circumcentre (rel. p_u, made absolute)
    if (!(cx > A.grid.x0 && cx < A.grid.x1 && cy > A.grid.y0 && cy < A.grid.y1)) return false;
    const int s3[3] = {su, sv, sw};
    double X[3], Y[3];
#pragma unroll
    for (int k = 0; k < 3; k++) {
        X[k] = __ldg(A.xs + s3[k]);
        Y[k] = __ldg(A.ys + s3[k]);
        double r = cmul(cmul(A.fac_voro, __ldg(A.hs + s3[k])), COS_PI8);
        if (!in_oct(cx, cy, X[k], Y[k], r)) return false;
    }
    double gx = cdiv(cadd(cadd(X[0], X[1]), X[2]), 3.0);
    double gy = cdiv(cadd(cadd(Y[0], Y[1]), Y[2]), 3.0);
    return bilinear(A.grid, A.phi, gx, gy, LdgLoad()) < A.keep_tol;
}

// thread-per-cell launcher (tm_cells_t.cu), explicitly instantiated for every mode
template <int MODE>
tm_status launch_cells_thread(tm_ctx *ctx, const CellArgs &a);

}  // namespace tmg
