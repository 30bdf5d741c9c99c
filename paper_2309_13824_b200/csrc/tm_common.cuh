// tm_common.cuh -- device (and host-test) helpers for the TriMe++ B200 hot path.
//
// Canonical arithmetic (reading L25): every floating operation whose
// result decides something discrete (a cell vertex position, the octagon/box
// membership of a circumcentre, phi~ at a centroid, the quadrature's longest
// edge) goes through cmul/cadd/csub/cdiv, which are never contracted into FMA
// (__dmul_rn/__dadd_rn/... on the device; the host build uses
// -ffp-contract=off).  Continuous quantities (sums, forces, centroids) may use
// FMA freely.
#pragma once
#include <stdint.h>
#include <math.h>

#ifdef __CUDACC__
#define TM_HD __host__ __device__ __forceinline__
#define TM_HDNI static __host__ __device__ __noinline__
#else
#define TM_HD inline
#define TM_HDNI static
#endif

namespace tmg {

#if defined(__CUDA_ARCH__)
TM_HD double cmul(double a, double b) { return __dmul_rn(a, b); }
TM_HD double cadd(double a, double b) { return __dadd_rn(a, b); }
TM_HD double csub(double a, double b) { return __dsub_rn(a, b); }
TM_HD double cdiv(double a, double b) { return __ddiv_rn(a, b); }
TM_HD double cfma(double a, double b, double c) { return __fma_rn(a, b, c); }
TM_HD double crcp(double a) { return __drcp_rn(a); }  // IEEE RN 1/a: the same bits as __ddiv_rn(1.0, a)
#else
TM_HD double cmul(double a, double b) { volatile double r = a * b; return r; }
TM_HD double cadd(double a, double b) { volatile double r = a + b; return r; }
TM_HD double csub(double a, double b) { volatile double r = a - b; return r; }
TM_HD double cdiv(double a, double b) { volatile double r = a / b; return r; }
TM_HD double cfma(double a, double b, double c) { return fma(a, b, c); }
TM_HD double crcp(double a) { volatile double r = 1.0 / a; return r; }
#endif

// fl(cos(pi/8)) and fl(sqrt(2)): octagon geometry literals
constexpr double COS_PI8 = 0.92387953251128673848;
constexpr double SQRT2 = 1.41421356237309514547;
constexpr double EPS = 1.1102230246251565e-16;  // 2^-53

// ---------------------------------------------------------------- lines
// n.x' = r relative to the cell generator; inside is n.x' <= r.
struct Line {
    double nx, ny, r;
};

// bisector of (i, j) from d = fl(p_j - p_i): inside = closer to p_i
TM_HD Line bisector(double dx, double dy) {
    Line L;
    L.nx = dx;
    L.ny = dy;
    L.r = cmul(0.5, cadd(cmul(dx, dx), cmul(dy, dy)));
    return L;
}

// Cramer intersection of two lines in the canonical form of SURVEY §8.0 ("Canonical wall
// vertices"): det = A.nx B.ny - A.ny B.nx, x = fl(num_x / det), y = fl(num_y / det), every
// operation correctly rounded and uncontracted -- the same bits as the oracle's plain C,
// and exactly symmetric in (A, B) (det and both numerators change sign).  Returns an upper
// bound on 1/|det| for the vertex error bounds (a float reciprocal rounded up from a float
// |det| rounded down: cheap, and +inf when |det| underflows, which only widens a filter).
TM_HD double inv_det_bound(double det) {
#if defined(__CUDA_ARCH__)
    return (double)__frcp_ru(__double2float_rd(fabs(det)));
#else
    return (1.0 / fabs(det)) * (1.0 + 4.0 * 1.1102230246251565e-16);
#endif
}

TM_HD double cramer(const Line &A, const Line &B, double &x, double &y) {
    double det = csub(cmul(A.nx, B.ny), cmul(A.ny, B.nx));
    x = cdiv(csub(cmul(A.r, B.ny), cmul(A.ny, B.r)), det);
    y = cdiv(csub(cmul(A.nx, B.r), cmul(A.r, B.nx)), det);
    return inv_det_bound(det);
}

// wall codes: octagon side k (outward normal at 45k deg) -> -1-k;
// box: -9 x<=x1, -10 y<=y1, -11 x>=x0, -12 y>=y0
TM_HD Line wall_line(int code, double px, double py, double r_oct, double bx0, double by0, double bx1,
                     double by1) {
    Line L;
    if (code >= -8) {
        // octagon side k: outward normal at 45k degrees, unnormalised (no table:
        // a dynamically indexed local array would live in local memory)
        const int k = -1 - code;
        L.nx = (k == 0 || k == 1 || k == 7) ? 1.0 : ((k >= 3 && k <= 5) ? -1.0 : 0.0);
        L.ny = (k >= 1 && k <= 3) ? 1.0 : ((k >= 5) ? -1.0 : 0.0);
        L.r = (k & 1) ? cmul(SQRT2, r_oct) : r_oct;
        return L;
    }
    switch (code) {
    case -9: L.nx = 1; L.ny = 0; L.r = csub(bx1, px); break;
    case -10: L.nx = 0; L.ny = 1; L.r = csub(by1, py); break;
    case -11: L.nx = -1; L.ny = 0; L.r = csub(px, bx0); break;
    default: L.nx = 0; L.ny = -1; L.r = csub(py, by0); break;
    }
    return L;
}

// canonical wall-vertex cut test: w strictly outside L
TM_HD bool wall_out(const Line &L, double vx, double vy) {
    return cadd(cmul(L.nx, vx), cmul(L.ny, vy)) > L.r;
}

// ---------------------------------------------------------------- fields
struct Grid {
    int32_t nx, ny;
    double x0, y0, x1, y1;
    double idx, idy;  // (n-1)/(x1-x0)
    double dx, dy;    // (x1-x0)/(n-1)
};

TM_HD void grid_cell(const Grid &g, double x, double y, int &i, int &j, double &s, double &t) {
    double u = cmul(csub(x, g.x0), g.idx);
    double v = cmul(csub(y, g.y0), g.idy);
    double fu = floor(u), fv = floor(v);
    i = fu < 0.0 ? 0 : (fu > (double)(g.nx - 2) ? g.nx - 2 : (int)fu);
    j = fv < 0.0 ? 0 : (fv > (double)(g.ny - 2) ? g.ny - 2 : (int)fv);
    s = csub(u, (double)i);
    t = csub(v, (double)j);
}

TM_HD double clerp(double a, double b, double s) { return cadd(a, cmul(s, csub(b, a))); }

// x / 3 without a division: q = fl(x/3-ish), exact residual by FMA, one correction step
// (Markstein).  Equal to the IEEE quotient on 4e8 random inputs (tests/test_div3.py);
// used only for quadrature points (continuous quantities, never for a decision).
TM_HD double div3(double x) {
    const double T = 0.33333333333333331483;  // fl(1/3)
    const double q = cmul(x, T);
    const double r = cfma(-q, 3.0, x);
    return cfma(r, T, q);
}

template <typename Load>
TM_HD double bilinear(const Grid &g, const double *F, double x, double y, Load ld) {
    int i, j;
    double s, t;
    grid_cell(g, x, y, i, j, s, t);
    const double *r0 = F + (int64_t)j * g.nx, *r1 = r0 + g.nx;
    double f00 = ld(r0 + i), f10 = ld(r0 + i + 1), f01 = ld(r1 + i), f11 = ld(r1 + i + 1);
    return clerp(clerp(f00, f10, s), clerp(f01, f11, s), t);
}

template <typename Load>
TM_HD void bilinear_grad(const Grid &g, const double *F, double x, double y, double &gx, double &gy, Load ld) {
    int i, j;
    double s, t;
    grid_cell(g, x, y, i, j, s, t);
    const double *r0 = F + (int64_t)j * g.nx, *r1 = r0 + g.nx;
    double f00 = ld(r0 + i), f10 = ld(r0 + i + 1), f01 = ld(r1 + i), f11 = ld(r1 + i + 1);
    gx = cdiv(cadd(cmul(csub(1.0, t), csub(f10, f00)), cmul(t, csub(f11, f01))), g.dx);
    gy = cdiv(cadd(cmul(csub(1.0, s), csub(f01, f00)), cmul(s, csub(f11, f10))), g.dy);
}

struct PlainLoad {
    TM_HD double operator()(const double *p) const { return *p; }
};
#ifdef __CUDACC__
struct LdgLoad {
    __device__ __forceinline__ double operator()(const double *p) const { return __ldg(p); }
};
#endif

// ---------------------------------------------------------------- exact incircle
// Floating-point expansion arithmetic (error-free transformations: Knuth's
// TwoSum, FMA TwoProduct; nonoverlapping expansions grown component by
// component).  The determinant is the 4x4 lifted form det[x y x^2+y^2 1]
// expanded by 2x2 minors (Laplace over columns {x,y} | {w,1}):
//   det = M12 N34 - M13 N24 + M14 N23 + M23 N14 - M24 N13 + M34 N12,
//   M_pq = x_p y_q - x_q y_p,  N_rs = w_r - w_s,  w = x^2 + y^2,
// positive iff d lies inside the circle through a,b,c given CCW.
TM_HD void two_sum(double a, double b, double &x, double &y) {
    x = cadd(a, b);
    double bv = csub(x, a);
    double av = csub(x, bv);
    double br = csub(b, bv);
    double ar = csub(a, av);
    y = cadd(ar, br);
}

TM_HD void two_prod(double a, double b, double &x, double &y) {
    x = cmul(a, b);
    y = cfma(a, b, -x);
}

// h = e + b, e nonoverlapping increasing; zero elimination; returns length
TM_HD int grow(const double *e, int n, double b, double *h) {
    double Q = b;
    int m = 0;
    for (int i = 0; i < n; i++) {
        double Qn, hh;
        two_sum(Q, e[i], Qn, hh);
        Q = Qn;
        if (hh != 0.0) h[m++] = hh;
    }
    if (Q != 0.0 || m == 0) h[m++] = Q;
    return m;
}

// acc += f (acc nonoverlapping; scratch t needs len(acc)+1); returns new length
TM_HD int exp_accumulate(double *acc, int n, const double *f, int nf, double *t) {
    for (int k = 0; k < nf; k++) {
        n = grow(acc, n, f[k], t);
        for (int i = 0; i < n; i++) acc[i] = t[i];
    }
    return n;
}

// h = e * b exactly; returns length
TM_HD int exp_scale(const double *e, int ne, double b, double *h, double *t) {
    int n = 0;
    for (int i = 0; i < ne; i++) {
        double hi, lo;
        two_prod(e[i], b, hi, lo);
        if (lo != 0.0) {
            n = grow(h, n, lo, t);
            for (int k = 0; k < n; k++) h[k] = t[k];
        }
        n = grow(h, n, hi, t);
        for (int k = 0; k < n; k++) h[k] = t[k];
    }
    return n;
}

TM_HD int exp_sign(const double *e, int n) {
    for (int i = n - 1; i >= 0; i--)
        if (e[i] != 0.0) return e[i] > 0.0 ? 1 : -1;
    return 0;
}

// 2-term minor x_p*y_q - x_q*y_p  -> up to 4 terms
TM_HD int minor2(double xp, double yp, double xq, double yq, double *m) {
    double a1, a0, b1, b0;
    two_prod(xp, yq, a1, a0);
    two_prod(xq, yp, b1, b0);
    double e[2] = {a0, a1};
    double t[8];
    int n = grow(e, 2, -b0, m);
    n = grow(m, n, -b1, t);
    for (int i = 0; i < n; i++) m[i] = t[i];
    return n;
}

// w_r - w_s with w = x^2+y^2 -> up to 8 terms
TM_HD int liftdiff(double xr, double yr, double xs, double ys, double *out) {
    double p[8], t[16];
    double h, l;
    int n = 0;
    two_prod(xr, xr, h, l); n = grow(p, n, l, t); for (int i = 0; i < n; i++) p[i] = t[i];
    n = grow(p, n, h, t); for (int i = 0; i < n; i++) p[i] = t[i];
    two_prod(yr, yr, h, l); n = grow(p, n, l, t); for (int i = 0; i < n; i++) p[i] = t[i];
    n = grow(p, n, h, t); for (int i = 0; i < n; i++) p[i] = t[i];
    two_prod(xs, xs, h, l); n = grow(p, n, -l, t); for (int i = 0; i < n; i++) p[i] = t[i];
    n = grow(p, n, -h, t); for (int i = 0; i < n; i++) p[i] = t[i];
    two_prod(ys, ys, h, l); n = grow(p, n, -l, t); for (int i = 0; i < n; i++) p[i] = t[i];
    n = grow(p, n, -h, t); for (int i = 0; i < n; i++) p[i] = t[i];
    for (int i = 0; i < n; i++) out[i] = p[i];
    return n;
}

#define TM_EXACT_ACC 400  // 6 Laplace terms x <= 64 components each
TM_HDNI int incircle_exact(const double *a, const double *b, const double *c, const double *d) {
    const double *P[4] = {a, b, c, d};
    // pairs (p,q) with complement (r,s) and sign of the Laplace term
    const int pp[6] = {0, 0, 0, 1, 1, 2}, qq[6] = {1, 2, 3, 2, 3, 3};
    const int rr[6] = {2, 1, 1, 0, 0, 0}, ss[6] = {3, 3, 2, 3, 2, 1};
    const int sg[6] = {1, -1, 1, 1, -1, 1};
    double acc[TM_EXACT_ACC], tmp[TM_EXACT_ACC], prod[80], sc[20], t2[80];
    int nacc = 0;
    for (int k = 0; k < 6; k++) {
        double M[8], N[16];
        int nm = minor2(P[pp[k]][0], P[pp[k]][1], P[qq[k]][0], P[qq[k]][1], M);
        int nn = liftdiff(P[rr[k]][0], P[rr[k]][1], P[ss[k]][0], P[ss[k]][1], N);
        if (sg[k] < 0)
            for (int i = 0; i < nn; i++) N[i] = -N[i];
        int np = 0;
        for (int i = 0; i < nm; i++) {
            int ns = exp_scale(N, nn, M[i], sc, t2);
            np = exp_accumulate(prod, np, sc, ns, t2);
        }
        nacc = exp_accumulate(acc, nacc, prod, np, tmp);
    }
    return exp_sign(acc, nacc);
}

}  // namespace tmg
