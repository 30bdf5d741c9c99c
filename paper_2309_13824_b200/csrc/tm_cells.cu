// tm_cells.cu -- S2 bounded Voronoi cells, S3 Delaunay extraction + keep rule,
// fused S4a CVD centroid (uniform fan / adaptive quadrature) and S5 treatment.
//
// One thread group (G lanes of a warp) computes one cell C_i = B ∩ Oct_i ∩ Vor(i)
// (PAPER.md P:100 cell-based approach, Fig. 3; octagon bound P:491):
// lane k owns polygon vertex k (CCW).  Candidates come from rings of bins in
// increasing distance, are sorted by distance, and clip the polygon one at a
// time; the search stops when the next candidate/ring is at least 2*R_max away
// (reading L11).  A vertex is cut by j when it is strictly closer to p_j:
//   * point-point vertices (both labels are neighbours): exact incircle sign,
//     by a rigorous floating filter on the stored vertex and, when the filter
//     cannot decide, exact expansion arithmetic (tm_common.cuh);
//   * wall vertices (an octagon or box side among the labels): the canonical
//     contraction-free test n.x' > r (reading L25).
// Every vertex coordinate is the canonical Cramer intersection of its two
// lines, relative to p_i.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "tm_internal.cuh"

namespace cg = cooperative_groups;
using namespace tmg;

namespace {

constexpr int G = 32;            // lanes per cell (= max vertices)
constexpr int CELLS_PER_BLOCK = 4;
constexpr int BUF = 64;          // candidate buffer per cell

enum : int { M_TRI = 1, M_ELL = 2, M_TREAT = 4, M_HAT = 8, M_COUNT = 16 };

struct VState {
    int la, lb;              // incoming / outgoing line codes (slot >= 0 or wall < 0)
    double vx, vy;           // canonical coordinates relative to p_i
    double K;                // filter constant (pp vertex), < 0 for wall vertices
    double onx, ony, orr;    // outgoing line
};

struct CellSmem {
    int32_t cand[BUF];
    int32_t kj[BUF];
    double kd2[BUF];
    int32_t order[BUF];
};

__device__ __forceinline__ double warp_max(const cg::thread_block_tile<G> &g, double v) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v = fmax(v, g.shfl_xor(v, o));
    return v;
}
__device__ __forceinline__ double warp_sum(const cg::thread_block_tile<G> &g, double v) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v += g.shfl_xor(v, o);
    return v;
}
__device__ __forceinline__ int warp_isum(const cg::thread_block_tile<G> &g, int v) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v += g.shfl_xor(v, o);
    return v;
}

// filter constant of a point-point vertex x = cramer(A, B) (both bisectors):
// K = e_v + 8 eps |v|_1 with e_v a rigorous bound on |x - exact circumcentre|
// (evaluation rounding of Cramer plus the rounding of d = fl(p - p_i)), x2 safety.
__device__ __forceinline__ double pp_filter_K(const Line &A, const Line &B, double x, double y) {
    double det = fabs(A.nx * B.ny - A.ny * B.nx);
    double n1a = fabs(A.nx) + fabs(A.ny), n1b = fabs(B.nx) + fabs(B.ny);
    double m1 = fabs(x) + fabs(y);
    double ev = EPS * (10.0 * (A.r * n1b + B.r * n1a + m1 * n1a * n1b) / (det * (1.0 - 8.0 * EPS)) + 2.0 * m1);
    return ev + 8.0 * EPS * m1;
}

__device__ __forceinline__ double vertex_r2(const VState &v) {
    double m1 = fabs(v.vx) + fabs(v.vy);
    double K = v.K > 0.0 ? v.K : 0.0;
    return fma(v.vx, v.vx, v.vy * v.vy) + K * (2.0 * m1 + K);
}

__device__ __forceinline__ VState shfl_state(const cg::thread_block_tile<G> &g, const VState &v, int src) {
    VState w;
    w.la = g.shfl(v.la, src);
    w.lb = g.shfl(v.lb, src);
    w.vx = g.shfl(v.vx, src);
    w.vy = g.shfl(v.vy, src);
    w.K = g.shfl(v.K, src);
    w.onx = g.shfl(v.onx, src);
    w.ony = g.shfl(v.ony, src);
    w.orr = g.shfl(v.orr, src);
    return w;
}

// Clip the polygon by line `code` (>=0: bisector with slot code at d=(dx,dy);
// <0: wall).  Returns the new vertex count, -1 on overflow, -2 if inconsistent.
__device__ int clip_by(const cg::thread_block_tile<G> &g, VState &v, int nv, int code, const Line &L, double px,
                       double py, const CellArgs &A, unsigned long long &n_exact) {
    const int lane = g.thread_rank();
    const bool is_bis = code >= 0;
    bool out = false;
    if (lane < nv) {
        if (is_bis && v.K >= 0.0) {
            double del = fma(L.nx, v.vx, L.ny * v.vy) - L.r;
            double n1 = fabs(L.nx) + fabs(L.ny);
            double B = n1 * fma(8.0 * EPS, n1, v.K);
            if (del > B)
                out = true;
            else if (del >= -B) {
                double Pi[2] = {px, py};
                double Pa[2] = {__ldg(A.xs + v.la), __ldg(A.ys + v.la)};
                double Pb[2] = {__ldg(A.xs + v.lb), __ldg(A.ys + v.lb)};
                double Pj[2] = {__ldg(A.xs + code), __ldg(A.ys + code)};
                int s = incircle_exact(Pi, Pa, Pb, Pj);
                if (s == 0) atomicAdd(&A.st->n_degenerate, 1ull);
                out = s > 0;
                n_exact++;
            }
        } else {
            out = wall_out(L, v.vx, v.vy);
        }
    }
    const unsigned mask = g.ballot(out);
    if (mask == 0u) return nv;
    const unsigned full = nv >= 32 ? 0xffffffffu : ((1u << nv) - 1u);
    if (mask == full) return -2;
    const unsigned inm = full & ~mask;
    const unsigned rl = ((inm << 1) | (inm >> (nv - 1))) & full;  // bit k: vertex k-1 inside
    const unsigned rr = ((inm >> 1) | (inm << (nv - 1))) & full;  // bit k: vertex k+1 inside
    const unsigned sc = mask & rl, ec = mask & rr;
    if (__popc(sc) != 1 || __popc(ec) != 1) return -2;
    const int s = __ffs(sc) - 1, e = __ffs(ec) - 1;
    const int m = __popc(mask);
    const int nn = nv - m + 2;
    if (nn > G) return -1;
    const int ps = s == 0 ? nv - 1 : s - 1;
    // lines of the two cut edges: pred(s) -> s lies on lb(pred(s)); e -> succ(e) on lb(e)
    Line E1, E2;
    E1.nx = g.shfl(v.onx, ps); E1.ny = g.shfl(v.ony, ps); E1.r = g.shfl(v.orr, ps);
    E2.nx = g.shfl(v.onx, e); E2.ny = g.shfl(v.ony, e); E2.r = g.shfl(v.orr, e);
    const int c1 = g.shfl(v.lb, ps), c2 = g.shfl(v.lb, e);
    int src = lane >= 2 ? (e + lane - 1) % nv : 0;
    VState w = shfl_state(g, v, src);
    if (lane == 0) {
        w.la = c1; w.lb = code;
        cramer(E1, L, w.vx, w.vy);
        w.onx = L.nx; w.ony = L.ny; w.orr = L.r;
        w.K = (is_bis && c1 >= 0) ? pp_filter_K(E1, L, w.vx, w.vy) : -1.0;
    } else if (lane == 1) {
        w.la = code; w.lb = c2;
        cramer(L, E2, w.vx, w.vy);
        w.onx = E2.nx; w.ony = E2.ny; w.orr = E2.r;
        w.K = (is_bis && c2 >= 0) ? pp_filter_K(L, E2, w.vx, w.vy) : -1.0;
    }
    v = w;
    return nn;
}

// ring k bin q -> (dx, dy), Chebyshev distance k, q in [0, 8k)
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

__device__ bool keep_tri(const CellArgs &A, int su, int sv, int sw, double cx, double cy) {
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

// adaptive quadrature centroid (Fig. 14; reading L13), relative to p_i
__device__ void quad_centroid(const cg::thread_block_tile<G> &g, const VState &v, int nv, double px, double py,
                              double area, double h, double dprev, const CellArgs &A, double &cx, double &cy,
                              unsigned long long &nq) {
    const int lane = g.thread_rank();
    double eps = dprev >= 0.0 ? dprev / h : A.fac_pt;
    if (eps < A.fac_end) eps = A.fac_end;
    const double E = sqrt(area) * eps;
    double prevx = 0.0, prevy = 0.0;
    for (int L = 1; L <= A.quad_max; L++) {
        const int depth = L - 1;
        const int64_t nleaf = (int64_t)nv << depth;
        double sw = 0.0, swx = 0.0, swy = 0.0;
        for (int64_t base = 0; base < nleaf; base += G) {
            int64_t t = base + lane;
            bool valid = t < nleaf;
            int f = valid ? (int)(t >> depth) : 0;
            int f1 = f + 1 == nv ? 0 : f + 1;
            double x1 = g.shfl(v.vx, f), y1 = g.shfl(v.vy, f);
            double x2 = g.shfl(v.vx, f1), y2 = g.shfl(v.vy, f1);
            if (!valid) continue;
            double P[3][2] = {{0.0, 0.0}, {x1, y1}, {x2, y2}};
            int64_t path = t & (((int64_t)1 << depth) - 1);
            for (int lev = depth - 1; lev >= 0; lev--) {
                double best = -1.0;
                int eidx = 0;
#pragma unroll
                for (int k = 0; k < 3; k++) {
                    int k1 = k == 2 ? 0 : k + 1;
                    double dx = csub(P[k1][0], P[k][0]), dy = csub(P[k1][1], P[k][1]);
                    double Lk = cadd(cmul(dx, dx), cmul(dy, dy));
                    if (Lk > best) { best = Lk; eidx = k; }
                }
                int ia = eidx, ib = eidx == 2 ? 0 : eidx + 1, ic = ib == 2 ? 0 : ib + 1;
                double ax = P[ia][0], ay = P[ia][1], bx = P[ib][0], by = P[ib][1], qx = P[ic][0], qy = P[ic][1];
                double mx = cmul(cadd(ax, bx), 0.5), my = cmul(cadd(ay, by), 0.5);
                if ((path >> lev) & 1) {  // child 1 = (M, Pb, Pc)
                    P[0][0] = mx; P[0][1] = my; P[1][0] = bx; P[1][1] = by;
                } else {                  // child 0 = (Pa, M, Pc)
                    P[0][0] = ax; P[0][1] = ay; P[1][0] = mx; P[1][1] = my;
                }
                P[2][0] = qx; P[2][1] = qy;
            }
            double cr = csub(cmul(csub(P[1][0], P[0][0]), csub(P[2][1], P[0][1])),
                             cmul(csub(P[1][1], P[0][1]), csub(P[2][0], P[0][0])));
            double At = cmul(0.5, cr);
            double qx = cdiv(cadd(cadd(P[0][0], P[1][0]), P[2][0]), 3.0);
            double qy = cdiv(cadd(cadd(P[0][1], P[1][1]), P[2][1]), 3.0);
            double rho = bilinear(A.grid, A.rho, cadd(px, qx), cadd(py, qy), LdgLoad());
            double wgt = At * rho;
            sw += wgt;
            swx += wgt * qx;
            swy += wgt * qy;
            nq++;
        }
        sw = warp_sum(g, sw);
        swx = warp_sum(g, swx);
        swy = warp_sum(g, swy);
        double curx = swx / sw, cury = swy / sw;
        double dx = prevx - curx, dy = prevy - cury;
        double dist = sqrt(dx * dx + dy * dy);
        prevx = curx;
        prevy = cury;
        if (dist < E) break;
    }
    cx = prevx;
    cy = prevy;
}

template <int MODE>
__global__ void __launch_bounds__(G *CELLS_PER_BLOCK) k_cells(CellArgs A) {
    __shared__ CellSmem smem_all[CELLS_PER_BLOCK];
    cg::thread_block block = cg::this_thread_block();
    cg::thread_block_tile<G> g = cg::tiled_partition<G>(block);
    const int gib = threadIdx.x / G;
    CellSmem &sm = smem_all[gib];
    const int lane = g.thread_rank();
    const int64_t cell = (int64_t)blockIdx.x * CELLS_PER_BLOCK + gib;
    if (cell >= A.n_local) return;
    const int32_t orig = __ldg(A.perm + cell);
    if (orig >= A.n_owned) return;  // ghost point: no cell

    const double px = __ldg(A.xs + cell), py = __ldg(A.ys + cell);
    const double h = __ldg(A.hs + cell);
    const int32_t gi = __ldg(A.gids + cell);
    const double S = cmul(A.fac_voro, h);
    const double r_oct = cmul(S, COS_PI8);
    const double bx0 = A.grid.x0, by0 = A.grid.y0, bx1 = A.grid.x1, by1 = A.grid.y1;
    unsigned long long n_exact = 0, n_cand = 0, n_clip = 0, nq = 0;

    // ---- initial polygon: octagon (vertex k between sides k and k+1), then the box
    VState v;
    int nv = 8;
    {
        int k = lane & 7;
        v.la = -1 - k;
        v.lb = -1 - ((k + 1) & 7);
        Line La = wall_line(v.la, px, py, r_oct, bx0, by0, bx1, by1);
        Line Lb = wall_line(v.lb, px, py, r_oct, bx0, by0, bx1, by1);
        cramer(La, Lb, v.vx, v.vy);
        v.K = -1.0;
        v.onx = Lb.nx; v.ony = Lb.ny; v.orr = Lb.r;
    }
    bool failed = false;
    if (csub(px, bx0) < S || csub(bx1, px) < S || csub(py, by0) < S || csub(by1, py) < S) {
        const int box_codes[4] = {-9, -10, -11, -12};
        for (int b = 0; b < 4 && !failed; b++) {
            Line L = wall_line(box_codes[b], px, py, r_oct, bx0, by0, bx1, by1);
            int r = clip_by(g, v, nv, box_codes[b], L, px, py, A, n_exact);
            if (r < 0) failed = true; else nv = r;
        }
    }
    double R2 = warp_max(g, lane < nv ? vertex_r2(v) : 0.0);
    const double MARG = 1.0 + 1e-9;

    // ---- nearest-first ring search over bins (L11 stopping rule)
    const BinGeom &bg = A.bg;
    int hbx = (int)floor((px - bg.x0) * bg.isx), hby = (int)floor((py - bg.y0) * bg.isy);
    hbx = hbx < 0 ? 0 : (hbx >= bg.nbx ? bg.nbx - 1 : hbx);
    hby = hby < 0 ? 0 : (hby >= bg.nby ? bg.nby - 1 : hby);
    for (int k = 0; !failed; k++) {
        if (k > 0) {
            double dl = px - (bg.x0 + (hbx - k + 1) * bg.sx), dr = (bg.x0 + (hbx + k) * bg.sx) - px;
            double dd = py - (bg.y0 + (hby - k + 1) * bg.sy), du = (bg.y0 + (hby + k) * bg.sy) - py;
            double dmin = fmin(fmin(dl, dr), fmin(dd, du));
            if (dmin > 0.0 && dmin * dmin * (1.0 - 1e-9) >= 4.0 * R2 * MARG) break;
            if (hbx - k < 0 && hby - k < 0 && hbx + k >= bg.nbx && hby + k >= bg.nby) break;
        }
        const int nq_ring = k == 0 ? 1 : 8 * k;
        for (int q0 = 0; q0 < nq_ring && !failed; q0 += G) {
            int q = q0 + lane, st = 0, cnt = 0;
            if (q < nq_ring) {
                int dx = 0, dy = 0;
                if (k > 0) ring_bin(k, q, dx, dy);
                int bx = hbx + dx, by = hby + dy;
                if (bx >= 0 && bx < bg.nbx && by >= 0 && by < bg.nby) {
                    int b = by * bg.nbx + bx;
                    st = __ldg(A.bin_start + b);
                    cnt = __ldg(A.bin_start + b + 1) - st;
                }
            }
            int incl = cnt;
#pragma unroll
            for (int o = 1; o < G; o <<= 1) {
                int t = g.shfl_up(incl, o);
                if (lane >= o) incl += t;
            }
            const int total = g.shfl(incl, G - 1);
            const int excl = incl - cnt;
            for (int base = 0; base < total && !failed; base += BUF) {
                // gather this window of candidate slots into smem
                for (int t = 0; t < cnt; t++) {
                    int pos = excl + t - base;
                    if (pos >= 0 && pos < BUF) sm.cand[pos] = st + t;
                }
                g.sync();
                const int nwin = min(BUF, total - base);
                // distance filter + compaction
                const double thr = 4.0 * R2 * MARG;
                int nkeep = 0;
                for (int t0 = 0; t0 < nwin; t0 += G) {
                    int t = t0 + lane;
                    bool keep = false;
                    int j = 0;
                    double d2 = 0.0;
                    if (t < nwin) {
                        j = sm.cand[t];
                        if (j != (int)cell) {
                            double dx = __ldg(A.xs + j) - px, dy = __ldg(A.ys + j) - py;
                            d2 = dx * dx + dy * dy;
                            if (dx == 0.0 && dy == 0.0) atomicAdd(&A.st->n_duplicate, 1ull);
                            keep = d2 < thr && d2 > 0.0;
                        }
                        n_cand++;
                    }
                    unsigned km = g.ballot(keep);
                    if (keep) {
                        int pos = nkeep + __popc(km & ((1u << lane) - 1u));
                        sm.kj[pos] = j;
                        sm.kd2[pos] = d2;
                    }
                    nkeep += __popc(km);
                }
                g.sync();
                // rank sort by (d2, slot)
                for (int t = lane; t < nkeep; t += G) {
                    double dt = sm.kd2[t];
                    int jt = sm.kj[t], r = 0;
                    for (int u = 0; u < nkeep; u++) {
                        double du = sm.kd2[u];
                        r += (du < dt) || (du == dt && sm.kj[u] < jt);
                    }
                    sm.order[r] = t;
                }
                g.sync();
                for (int r = 0; r < nkeep; r++) {
                    int t = sm.order[r];
                    double d2 = sm.kd2[t];
                    if (d2 >= 4.0 * R2 * MARG) break;  // sorted: the rest are farther
                    int j = sm.kj[t];
                    double dx = csub(__ldg(A.xs + j), px), dy = csub(__ldg(A.ys + j), py);
                    Line L = bisector(dx, dy);
                    int nn = clip_by(g, v, nv, j, L, px, py, A, n_exact);
                    if (nn < 0) {
                        failed = true;
                        if (lane == 0) atomicAdd(nn == -1 ? &A.st->n_overflow : &A.st->n_degenerate, 1ull);
                        break;
                    }
                    nv = nn;
                    R2 = warp_max(g, lane < nv ? vertex_r2(v) : 0.0);
                    n_clip++;
                }
                g.sync();
            }
        }
    }
    if (failed) {
        // leave the point where it is; counted in n_overflow / n_degenerate
        if ((MODE & M_TREAT) && lane == 0) {
            A.x_out[orig] = px; A.y_out[orig] = py; A.d_prev_out[orig] = 0.0; A.status[orig] = 2;
        }
        if ((MODE & M_HAT) && lane == 0) { A.x_hat[orig] = px; A.y_hat[orig] = py; }
        if ((MODE & M_ELL) && lane == 0) A.deg[cell] = 0;
        return;
    }

    const bool active = lane < nv;
    // ---- S3: Delaunay triangles at point-point vertices + keep rule
    bool kept = false;
    int t_own = 0;
    if (MODE & (M_TRI | M_ELL)) {
        bool pp = active && v.la >= 0 && v.lb >= 0;
        bool owned = false;
        if (pp) {
            int32_t ga = __ldg(A.gids + v.la), gb = __ldg(A.gids + v.lb);
            owned = gi < ga && gi < gb;
            if (owned) {
                int sv = ga < gb ? v.la : v.lb, sw = ga < gb ? v.lb : v.la;
                kept = keep_tri(A, (int)cell, sv, sw, cadd(px, v.vx), cadd(py, v.vy));
            } else if (MODE & M_ELL) {
                // canonical circumcentre relative to the smallest-id vertex
                int s3[3] = {(int)cell, v.la, v.lb};
                int32_t g3[3] = {gi, ga, gb};
                // sort the three by gid
                for (int a = 0; a < 2; a++)
                    for (int b = 0; b < 2 - a; b++)
                        if (g3[b] > g3[b + 1]) {
                            int32_t tg = g3[b]; g3[b] = g3[b + 1]; g3[b + 1] = tg;
                            int ts = s3[b]; s3[b] = s3[b + 1]; s3[b + 1] = ts;
                        }
                double ux = __ldg(A.xs + s3[0]), uy = __ldg(A.ys + s3[0]);
                Line B1 = bisector(csub(__ldg(A.xs + s3[1]), ux), csub(__ldg(A.ys + s3[1]), uy));
                Line B2 = bisector(csub(__ldg(A.xs + s3[2]), ux), csub(__ldg(A.ys + s3[2]), uy));
                double ox, oy;
                cramer(B1, B2, ox, oy);
                kept = keep_tri(A, s3[0], s3[1], s3[2], cadd(ux, ox), cadd(uy, oy));
            }
        }
        if (MODE & M_TRI) {
            bool emit = owned && kept;
            unsigned em = g.ballot(emit);
            t_own = __popc(em);
            unsigned long long base = 0;
            if (lane == 0 && em) base = atomicAdd(A.n_tri, (unsigned long long)t_own);
            base = g.shfl(base, 0);
            if (emit) {
                unsigned long long idx = base + __popc(em & ((1u << lane) - 1u));
                if ((int64_t)idx < A.tri_cap) {
                    A.tri[3 * idx] = gi;
                    A.tri[3 * idx + 1] = __ldg(A.gids + v.la);
                    A.tri[3 * idx + 2] = __ldg(A.gids + v.lb);
                } else if (__popc(em & ((1u << lane) - 1u)) == 0) {
                    atomicAdd(&A.st->n_tri_overflow, 1ull);
                }
            }
        }
    }
    // ---- DistMesh ELL row: neighbour a (incoming bisector of vertex k) borders a kept triangle
    int ell = 0;
    if (MODE & M_ELL) {
        bool kprev = g.shfl((int)kept, lane == 0 ? nv - 1 : lane - 1) != 0;
        bool nb = active && v.la >= 0 && (kept || kprev);
        unsigned nm = g.ballot(nb);
        ell = __popc(nm);
        if (nb) {
            int pos = __popc(nm & ((1u << lane) - 1u));
            if (pos < A.adj_stride) A.adj[(int64_t)pos * A.n_local + cell] = v.la;
        }
        if (lane == 0) {
            A.deg[cell] = (uint8_t)(ell < A.adj_stride ? ell : A.adj_stride);
            if (ell > A.adj_stride) atomicAdd(&A.st->n_adj_overflow, 1ull);
        }
    }
    // ---- S4a: centroid of C_i (relative to p_i)
    double cx = 0.0, cy = 0.0;
    if (MODE & (M_TREAT | M_HAT)) {
        int nx1 = lane + 1 == nv ? 0 : lane + 1;
        double x1 = g.shfl(v.vx, nx1), y1 = g.shfl(v.vy, nx1);
        double cr = active ? v.vx * y1 - x1 * v.vy : 0.0;
        double S2 = warp_sum(g, cr);
        if (A.rho == nullptr) {
            double sx = warp_sum(g, active ? cr * (v.vx + x1) : 0.0);
            double sy = warp_sum(g, active ? cr * (v.vy + y1) : 0.0);
            cx = sx / (3.0 * S2);
            cy = sy / (3.0 * S2);
            nq += nv;
        } else {
            double dp = A.d_prev ? __ldg(A.d_prev + orig) : -1.0;
            quad_centroid(g, v, nv, px, py, 0.5 * S2, h, dp, A, cx, cy, nq);
        }
        if ((MODE & M_HAT) && lane == 0) {
            A.x_hat[orig] = px + cx;
            A.y_hat[orig] = py + cy;
        }
        // ---- S5 fused treatment (Alg. 2 line "project it back")
        if ((MODE & M_TREAT) && lane == 0) {
            double qx, qy, dpo;
            int s = treat_point(A.grid, A.phi, h, A.h_avg, A.fac_pt, A.fac_geps, A.damping, A.newton_max, px, py,
                                px + cx, py + cy, qx, qy, dpo, LdgLoad());
            A.x_out[orig] = qx;
            A.y_out[orig] = qy;
            A.d_prev_out[orig] = dpo;
            A.status[orig] = (int8_t)s;
            if (s & 2) atomicAdd(&A.st->n_fallback, 1ull);
        }
    }
    // ---- O8 work counters (TM_F_COUNT_WORK)
    if (MODE & M_COUNT) {
        // n_cert: points within 2R of p_i for the final cell (rescan of the bins)
        double R2f = R2;
        int ncert = 0;
        double rad = 2.0 * sqrt(R2f);
        int bxa = max(0, (int)floor((px - rad - bg.x0) * bg.isx)), bxb = min(bg.nbx - 1, (int)floor((px + rad - bg.x0) * bg.isx));
        int bya = max(0, (int)floor((py - rad - bg.y0) * bg.isy)), byb = min(bg.nby - 1, (int)floor((py + rad - bg.y0) * bg.isy));
        for (int by = bya; by <= byb; by++) {
            int s0 = __ldg(A.bin_start + by * bg.nbx + bxa), s1 = __ldg(A.bin_start + by * bg.nbx + bxb + 1);
            for (int s = s0 + lane; s < s1; s += G) {
                double dx = __ldg(A.xs + s) - px, dy = __ldg(A.ys + s) - py;
                ncert += (s != (int)cell) && (dx * dx + dy * dy < rad * rad);
            }
        }
        ncert = warp_isum(g, ncert);
        int degc = warp_isum(g, active && v.lb >= 0 ? 1 : 0);
        unsigned long long ex = n_exact, ca = n_cand;
        for (int o = G / 2; o > 0; o >>= 1) {
            ex += g.shfl_xor(ex, o);
            ca += g.shfl_xor(ca, o);
        }
        unsigned long long nqs = nq;
        for (int o = G / 2; o > 0; o >>= 1) nqs += g.shfl_xor(nqs, o);
        if (lane == 0) {
            atomicAdd(&A.st->work[0], 1ull);
            atomicAdd(&A.st->work[1], (unsigned long long)ncert);
            atomicAdd(&A.st->work[2], (unsigned long long)degc);
            atomicAdd(&A.st->work[3], (unsigned long long)nv);
            atomicAdd(&A.st->work[4], (unsigned long long)t_own);
            atomicAdd(&A.st->work[5], (A.rho == nullptr) ? (unsigned long long)nv : nqs);
            atomicAdd(&A.st->work[6], (unsigned long long)ell);
            atomicAdd(&A.st->work[7], ca);
            atomicAdd(&A.st->work[8], n_clip);
            atomicAdd(&A.st->work[9], ex);
        }
    }
}

template <int MODE>
tm_status launch_cells(tm_ctx *ctx, const CellArgs &a) {
    unsigned blocks = (unsigned)((ctx->n_local + CELLS_PER_BLOCK - 1) / CELLS_PER_BLOCK);
    k_cells<MODE><<<blocks, G * CELLS_PER_BLOCK, 0, ctx->stream>>>(a);
    return tm_internal_check_launch(ctx, "k_cells");
}

template <int BASE>
tm_status dispatch_count(tm_ctx *ctx, const CellArgs &a) {
    if (ctx->p.flags & TM_F_COUNT_WORK) return launch_cells<BASE | M_COUNT>(ctx, a);
    return launch_cells<BASE>(ctx, a);
}

}  // namespace

extern "C" tm_status tm_voronoi_delaunay(tm_ctx *ctx, int32_t *tri, int64_t tri_cap, int64_t *n_tri, int32_t *adj,
                                         uint8_t *deg, const double *d_prev, double *x_out, double *y_out,
                                         double *d_prev_out, int8_t *status) {
    if (!ctx) return TM_E_ARG;
    if (!ctx->have_bins) TM_FAIL(ctx, TM_E_STATE, "tm_voronoi_delaunay before tm_grid_bin");
    if (!tri || !n_tri || tri_cap < 0) TM_FAIL(ctx, TM_E_ARG, "tri/n_tri required");
    if ((adj == nullptr) != (deg == nullptr)) TM_FAIL(ctx, TM_E_ARG, "adj and deg must be given together");
    bool treat = x_out != nullptr;
    if (treat && (!y_out || !d_prev_out || !status)) TM_FAIL(ctx, TM_E_ARG, "fused CVD needs x_out,y_out,d_prev_out,status");
    TM_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
    CellArgs a;
    tm_internal_fill_cell_args(ctx, &a);
    a.tri = tri; a.tri_cap = tri_cap; a.n_tri = (unsigned long long *)n_tri;
    a.adj = adj; a.deg = deg;
    a.d_prev = d_prev; a.x_out = x_out; a.y_out = y_out; a.d_prev_out = d_prev_out; a.status = status;
    TM_CUDA_TRY(ctx, cudaMemsetAsync(n_tri, 0, sizeof(int64_t), ctx->stream));
    if (ctx->p.flags & TM_F_COUNT_WORK)
        TM_CUDA_TRY(ctx, cudaMemsetAsync(ctx->dst->work, 0, sizeof(ctx->dst->work), ctx->stream));
    tm_status s;
    if (treat && adj) s = dispatch_count<M_TRI | M_ELL | M_TREAT>(ctx, a);
    else if (treat) s = dispatch_count<M_TRI | M_TREAT>(ctx, a);
    else if (adj) s = dispatch_count<M_TRI | M_ELL>(ctx, a);
    else s = dispatch_count<M_TRI>(ctx, a);
    if (s == TM_OK) ctx->have_cells = true;
    return s;
}

extern "C" tm_status tm_cvd_step(tm_ctx *ctx, const double *d_prev, double *x_hat, double *y_hat) {
    if (!ctx) return TM_E_ARG;
    if (!ctx->have_bins) TM_FAIL(ctx, TM_E_STATE, "tm_cvd_step before tm_grid_bin");
    if (!x_hat || !y_hat) TM_FAIL(ctx, TM_E_ARG, "x_hat/y_hat required");
    TM_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
    CellArgs a;
    tm_internal_fill_cell_args(ctx, &a);
    a.d_prev = d_prev; a.x_hat = x_hat; a.y_hat = y_hat;
    if (ctx->p.flags & TM_F_COUNT_WORK)
        TM_CUDA_TRY(ctx, cudaMemsetAsync(ctx->dst->work, 0, sizeof(ctx->dst->work), ctx->stream));
    return dispatch_count<M_HAT>(ctx, a);
}
