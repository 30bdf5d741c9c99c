// tm_cells_t.cu -- thread-per-cell cell kernel (the default S2-S5 path).
//
// Same method and the same canonical arithmetic as the group kernel (S2 bounded
// cell by half-plane clipping, P:100 / Fig. 3; octagon bound P:491; S3 keep rule
// P:499-510 in reading L10; S4a centroid P:203-207 / P:537-553; S5 treatment),
// but one THREAD computes one cell C_i = B ∩ Oct_i ∩ Vor(i):
//   * the polygon is a linked ring of up to TM_VMAX vertex slots in shared
//     memory, laid out [slot][thread] so that every slot access of a warp is
//     bank-conflict free whatever slot each thread touches (TB*8 B rows);
//     a clip rewrites two slots and two links, never moves vertices;
//   * a vertex slot holds its canonical coordinates relative to p_i (fp64),
//     its filter constant K (float, rounded up; < 0 marks a wall vertex), the
//     code of its incoming line (the outgoing line is the incoming line of the
//     next slot) and its ring links;
//   * candidates are visited leaf by leaf: the home leaf, the 8 neighbouring
//     leaves nearest-first, then rings >= 2; a leaf (or ring) whose distance
//     from p_i is at least 2 R_max is skipped (reading L11);
//   * a cell that needs more than TM_VMAX slots is handed to the 32-lane group
//     kernel (retry list), which holds up to 32 vertices.
// Work is independent per thread, so the fp64 pipe sees 32 cells per warp
// instead of 2, and no shuffle/ballot sits on the per-candidate critical path.

#include <cuda_runtime.h>
#include <climits>
#include <algorithm>

#include "tm_cellcore.cuh"

using namespace tmg;

#ifndef TM_TB
#define TM_TB 128
#endif
#ifndef TM_VMAX
#define TM_VMAX 10
#endif
#ifndef TM_TMINB
#define TM_TMINB 5
#endif
#ifndef TM_OUT_MINB
#define TM_OUT_MINB 6  // min resident 128-thread blocks per SM for k_output_t (80-register cap: r3h A/B)
#endif
#ifndef TM_CVD_SPLIT
#define TM_CVD_SPLIT 1  // 1: CVD centroid, quadrature, treatment in a second kernel over stored rings;
                        // 2: triangles and ELL rows there too (all modes)
#endif
#ifndef TM_K_DOUBLE
#define TM_K_DOUBLE 0  // filter constants as float (rounded up): less shared memory, more L1
#endif
#ifndef TM_R2_CACHE
#define TM_R2_CACHE 1  // cache each vertex's r^2 bound in shared memory
#endif
#ifndef TM_GROUP_SHIFT
#define TM_GROUP_SHIFT 2  // measured: 1, 2, 3 all ~5 % faster than per-leaf groups, 2 best; whole-warp 3x slower
#endif
#ifndef TM_THREAD_EXACT
#define TM_THREAD_EXACT 0  // 0: cells with an undecided filter go to the 32-lane group kernel (rare)
#endif

namespace {

// which outputs leave k_cells_t for k_output_t (measured per mode, round 2): CVD's centroid,
// quadrature and treatment always; DistMesh's triangles and ELL rows (-6 % per DistMesh
// iteration on cfg3/cfg4); CVD's triangles stay (+4 % if moved)
__host__ __device__ constexpr bool split_tris(int mode) {
    return !(mode & M_COUNT) && (TM_CVD_SPLIT >= 2 || ((mode & M_ELL) && TM_CVD_SPLIT >= 1));
}
__host__ __device__ constexpr bool split_rings(int mode) {
    return !(mode & M_COUNT) && ((TM_CVD_SPLIT >= 1 && (mode & (M_TREAT | M_HAT))) || split_tris(mode));
}

constexpr int TB = TM_TB;
constexpr int VMAX = TM_VMAX;
// TM_HISLOT: slots >= VLO are tested only by threads whose ring uses one (slots are handed out
// lowest-free first, so rings rarely reach them); the masks below make this exactly equivalent
#ifndef TM_BLOCK_ORDER
#define TM_BLOCK_ORDER 0
#endif
#ifndef TM_HISLOT
#define TM_HISLOT 0
#endif
constexpr int VLO = (TM_HISLOT && VMAX > 8) ? 8 : VMAX;
static_assert(VMAX <= 31, "slot masks are 32-bit");
static_assert(VMAX <= TM_NBR, "warm-start rows hold at most TM_NBR neighbours per point (ADVICE r1)");
static_assert(TB <= 256 && (TB & (TB - 1)) == 0, "balancing keys hold the lane slot in 8 bits");
#if TM_K_DOUBLE
typedef double KT;  // filter constant storage
#else
typedef float KT;   // rounded up: still a valid bound
#endif
constexpr size_t TSMEM = (size_t)VMAX * TB * (16 + sizeof(KT) + (TM_R2_CACHE ? 4 : 0) + 4 + 1 + 1);

// per-warp staging of the warm-certification phase (M_WCERT), after the rings: the warp's
// cells (generator, prefilter data, ring masks, slot) and the queue of (cell, point) pairs
struct WarpQ {
    double cx[32], cy[32];
    float4 cf[32];  // the group's cells relative to the group origin (float) and a (2 R_max)^2
                    // bound rounded up with margin: a conservative prefilter, never the decision
    unsigned used[32], wall[32];
    int qj[64];
    uint8_t qc[64];
};
constexpr size_t TSMEM_W = TSMEM + (TB / 32) * sizeof(WarpQ);
static_assert(TSMEM_W + 1024 <= 228 * 1024 / TM_TMINB, "5 blocks per SM must fit the shared memory");

// this thread's view of the block's slot arrays (element k at [k * TB])
struct TPoly {
    double2 *v;     // canonical coordinates relative to p_i
    KT *K;          // filter constant of a point-point vertex (< 0: wall vertex)
    float *r2;      // conservative squared distance from p_i (rounded up), if TM_R2_CACHE
    int *la;        // incoming line code
    uint8_t *prv, *nxt;
    unsigned used;  // occupied slots
    unsigned wall;  // slots holding a wall vertex (an octagon or box side among its lines)
    unsigned long long lmask;  // bit (slot & 63) of every warm-start candidate clipped (a filter):
                               // only those can reach the clip test twice
};

__device__ __forceinline__ TPoly tpoly_bind(unsigned char *smem, int tid) {
    TPoly P;
    double2 *v = reinterpret_cast<double2 *>(smem);
    KT *K = reinterpret_cast<KT *>(v + VMAX * TB);
    float *r2 = reinterpret_cast<float *>(K + VMAX * TB);
    int *la = reinterpret_cast<int *>(r2 + (TM_R2_CACHE ? VMAX * TB : 0));
    uint8_t *prv = reinterpret_cast<uint8_t *>(la + VMAX * TB);
    uint8_t *nxt = prv + VMAX * TB;
    P.v = v + tid; P.K = K + tid; P.r2 = r2 + tid; P.la = la + tid; P.prv = prv + tid; P.nxt = nxt + tid;
    P.used = 0;
    P.wall = 0;
    P.lmask = 0;
    return P;
}

__device__ __forceinline__ float vertex_r2f_t(double vx, double vy, double K) {
    double m1 = fabs(vx) + fabs(vy);
    K = K > 0.0 ? K : 0.0;
    double r2 = fma(vx, vx, vy * vy) + K * (2.0 * m1 + K);
    return __double2float_ru(r2 * (1.0 + 1e-12));
}

__device__ __forceinline__ float poly_R2(const TPoly &P) {
    float r = 0.f;
#pragma unroll
    for (int k = 0; k < VMAX; k++) {
#if TM_R2_CACHE
        const float rk = P.r2[k * TB];
#else
        const double2 vv = P.v[k * TB];
        const float rk = vertex_r2f_t(vv.x, vv.y, (double)P.K[k * TB]);
#endif
        r = fmaxf(r, ((P.used >> k) & 1u) ? rk : 0.f);
    }
    return r;
}

__device__ __forceinline__ void set_r2(TPoly &P, int k, double x, double y, double K) {
#if TM_R2_CACHE
    P.r2[k * TB] = vertex_r2f_t(x, y, K);
#endif
}

__device__ __forceinline__ KT store_K(double K) {
#if TM_K_DOUBLE
    return K;
#else
    return K < 0.0 ? -1.f : __double2float_ru(K);
#endif
}

// Clip the ring by line L (code >= 0: bisector with slot `code`; < 0: wall).
// Returns 0 ok, -1 out of slots (or undecided filter, see TM_THREAD_EXACT),
// -2 inconsistent.  The decisions are exactly those of clip_by (group kernel):
// exact incircle sign for point-point vertices (floating filter, expansion
// fallback), canonical test for wall vertices.  All VMAX slots are tested,
// unrolled and branch-free (unused slots are masked out): no divergence between
// threads with rings of different sizes, full ILP.
__device__ __forceinline__ int clip_t(TPoly &P, int code, const Line &L, const CellGeom &cgm, const CellArgs &A,
                                      ClipStats &cs) {
    const bool is_bis = code >= 0;
    const double n1 = fabs(L.nx) + fabs(L.ny);
    const double c8 = 8.0 * EPS * n1 * n1;  // filter bound |d|_1 (K + 8 eps |d|_1) = n1 K + c8
    unsigned out = 0, unc = 0;
    // L already bounds the ring (a warm-start neighbour met again): no cut.  lmask filters;
    // the full check over the ring's lines runs on a filter hit only
    if (is_bis && ((P.lmask >> (code & 63)) & 1ull)) {
        unsigned dup = 0;
#pragma unroll
        for (int k = 0; k < VMAX; k++) dup |= (unsigned)(P.la[k * TB] == code) << k;
        if (dup & P.used) return 0;
    }
    if (is_bis) {
#pragma unroll
        for (int k = 0; k < VLO; k++) {  // point-point filter on every slot (masked below)
            const double2 vv = P.v[k * TB];
            const double del = fma(L.nx, vv.x, L.ny * vv.y) - L.r;
            const double B = fma(n1, (double)P.K[k * TB], c8);
            out |= (unsigned)(del > B) << k;
            unc |= (unsigned)(del <= B && del >= -B) << k;
        }
        if (VLO < VMAX && (P.used >> VLO)) {
#pragma unroll
            for (int k = VLO; k < VMAX; k++) {
                const double2 vv = P.v[k * TB];
                const double del = fma(L.nx, vv.x, L.ny * vv.y) - L.r;
                const double B = fma(n1, (double)P.K[k * TB], c8);
                out |= (unsigned)(del > B) << k;
                unc |= (unsigned)(del <= B && del >= -B) << k;
            }
        }
    }
    // wall vertices (and every vertex when L is a wall): the canonical test (L25); interior
    // cells have none once their neighbours bound them
    const unsigned wset = is_bis ? (P.wall & P.used) : P.used;
    out &= P.used & ~wset;
    unc &= P.used & ~wset;
    for (unsigned m = wset; m; m &= m - 1) {
        const int k = __ffs(m) - 1;
        const double2 vv = P.v[k * TB];
        out |= (unsigned)wall_out(L, vv.x, vv.y) << k;
    }
    // undecided point-point vertices (rare): exact incircle sign, outside the hot
    // loop -- or, with TM_THREAD_EXACT=0, the whole cell goes to the group kernel
#if TM_THREAD_EXACT
    for (; unc; unc &= unc - 1) {
        const int k = __ffs(unc) - 1;
        const int a = P.la[k * TB], b = P.la[P.nxt[k * TB] * TB];
        double Pi[2] = {cgm.px, cgm.py};
        double Pa[2] = {__ldg(A.xs + a), __ldg(A.ys + a)};
        double Pb[2] = {__ldg(A.xs + b), __ldg(A.ys + b)};
        double Pj[2] = {__ldg(A.xs + code), __ldg(A.ys + code)};
        const int sg = incircle_exact(Pi, Pa, Pb, Pj);
        if (sg == 0) atomicAdd(&A.st->n_degenerate, 1ull);
        out |= (unsigned)(sg > 0) << k;
        cs.exact++;
    }
#else
    if (unc) return -1;
#endif
    if (out == 0u) return 0;
    if (out == P.used) return -2;
    int s = -1, e = -1, ns = 0, ne_ = 0;
    for (unsigned m = out; m; m &= m - 1) {
        const int k = __ffs(m) - 1;
        if (!((out >> P.prv[k * TB]) & 1u)) { s = k; ns++; }
        if (!((out >> P.nxt[k * TB]) & 1u)) { e = k; ne_++; }
    }
    if (ns != 1 || ne_ != 1) return -2;
    int sB = e;
    if (__popc(out) == 1) {
        const unsigned fr = ~P.used & ((1u << VMAX) - 1u);
        if (fr == 0u) return -1;
        sB = __ffs(fr) - 1;
    }
    const int ne = P.nxt[e * TB];
    const int c1 = P.la[s * TB];   // line into s: the edge ps -> s
    const int c2 = P.la[ne * TB];  // line out of e = line into ne
    {   // A = (c1, L) in slot s
        const Line E1 = line_of(c1, cgm, A);
        double x, y;
        const double inv = cramer(E1, L, x, y);
        const bool ppv = is_bis && c1 >= 0;
        const double Kn = ppv ? pp_filter_K(E1, L, x, y, inv) : -1.0;
        P.v[s * TB] = make_double2(x, y);
        P.K[s * TB] = store_K(Kn);
        set_r2(P, s, x, y, Kn);
        P.wall = ppv ? (P.wall & ~(1u << s)) : (P.wall | (1u << s));
        P.nxt[s * TB] = (uint8_t)sB;
    }
    {   // B = (L, c2) in slot sB
        const Line E2 = line_of(c2, cgm, A);
        double x, y;
        const double inv = cramer(L, E2, x, y);
        const bool ppv = is_bis && c2 >= 0;
        const double Kn = ppv ? pp_filter_K(L, E2, x, y, inv) : -1.0;
        P.v[sB * TB] = make_double2(x, y);
        P.K[sB * TB] = store_K(Kn);
        set_r2(P, sB, x, y, Kn);
        P.wall = ppv ? (P.wall & ~(1u << sB)) : (P.wall | (1u << sB));
        P.la[sB * TB] = code;
        P.prv[sB * TB] = (uint8_t)s;
        P.nxt[sB * TB] = (uint8_t)ne;
    }
    P.prv[ne * TB] = (uint8_t)sB;
    P.used = (P.used & ~out) | (1u << s) | (1u << sB);
    cs.clips++;
    return 0;
}

// leaf range [st, st+cnt) of virtual leaf (vx, vy) at the home resolution rh
// (coarser leaves only at the virtual leaf closest to (ux, uy)); as the group kernel
// (hb, hoff): the home level-0 bin and its first leaf -- most ring-1 leaves lie in the
// home bin, whose level is rh: their range then costs one dependent load, not two
__device__ __forceinline__ void vleaf_range(const CellArgs &A, int vx, int vy, int rh, int ux, int uy, int hb,
                                            int hoff, int &st, int &cnt) {
    const BinGeom &bg = A.bg;
    st = 0;
    cnt = 0;
    const int bx = vx >> rh, by = vy >> rh;
    const int b = by * bg.nbx + bx;
    const bool home = b == hb;
    const int rb = home ? rh : __ldg(A.rlev + b);
    const int off = home ? hoff : __ldg(A.leaf_off + b);
    if (rb >= rh) {
        const int sh = 2 * (rb - rh);
        const int mlo = (int)morton2((uint32_t)(vx - (bx << rh)), (uint32_t)(vy - (by << rh))) << sh;
        st = __ldg(A.leaf_start + off + mlo);
        cnt = __ldg(A.leaf_start + off + mlo + (1 << sh)) - st;
    } else {
        const int d = rh - rb;
        const int Lx = vx >> d, Ly = vy >> d;
        const int rx = min(max(ux, Lx << d), ((Lx + 1) << d) - 1);
        const int ry = min(max(uy, Ly << d), ((Ly + 1) << d) - 1);
        if (rx == vx && ry == vy) {
            const int mm = (int)morton2((uint32_t)(Lx - (bx << rb)), (uint32_t)(Ly - (by << rb)));
            st = __ldg(A.leaf_start + off + mm);
            cnt = __ldg(A.leaf_start + off + mm + 1) - st;
        }
    }
}

struct SearchCtx {
    double px, py;
    int cell;
    unsigned long long n_cand;
};

// squared distance from p to the rectangle of virtual leaf (vx, vy)
__device__ __forceinline__ double leaf_d2(const BinGeom &bg, double lsx, double lsy, int vx, int vy, double px,
                                          double py) {
    const double lx = bg.x0 + vx * lsx, ly = bg.y0 + vy * lsy;
    const double gx = fmax(fmax(lx - px, px - (lx + lsx)), 0.0);
    const double gy = fmax(fmax(ly - py, py - (ly + lsy)), 0.0);
    return gx * gx + gy * gy;
}

__device__ __forceinline__ void cswap(unsigned &a, unsigned &b) {
    const unsigned lo = min(a, b), hi = max(a, b);
    a = lo;
    b = hi;
}

// adaptive quadrature centroid (Fig. 14; reading L13), one thread,
// relative to p_i; same sub-triangle construction as quad_centroid
__device__ void quad_centroid_t(const TPoly &P, int start, int nv, double px, double py, double area, double h,
                                double dprev, const CellArgs &A, double &cx, double &cy, unsigned long long &nq) {
    double eps = dprev >= 0.0 ? cdiv(dprev, h) : A.fac_pt;
    if (eps < A.fac_end) eps = A.fac_end;
    const double E = cmul(sqrt(area), eps);
    double prevx = 0.0, prevy = 0.0;
    for (int L = 1; L <= A.quad_max; L++) {
        const int depth = L - 1;
        double sw = 0.0, swx = 0.0, swy = 0.0;
        int k = start;
        for (int f = 0; f < nv; f++) {
            const int kn = P.nxt[k * TB];
            const double x1 = P.v[k * TB].x, y1 = P.v[k * TB].y;
            const double x2 = P.v[kn * TB].x, y2 = P.v[kn * TB].y;
            k = kn;
            const int64_t nleaf = (int64_t)1 << depth;
            for (int64_t path = 0; path < nleaf; path++) {
                double Q[3][2] = {{0.0, 0.0}, {x1, y1}, {x2, y2}};
                for (int lev = depth - 1; lev >= 0; lev--) {
                    double best = -1.0;
                    int eidx = 0;
#pragma unroll
                    for (int q = 0; q < 3; q++) {
                        const int q1 = q == 2 ? 0 : q + 1;
                        const double ddx = csub(Q[q1][0], Q[q][0]), ddy = csub(Q[q1][1], Q[q][1]);
                        const double Lq = cadd(cmul(ddx, ddx), cmul(ddy, ddy));
                        if (Lq > best) { best = Lq; eidx = q; }
                    }
                    const int ia = eidx, ib = eidx == 2 ? 0 : eidx + 1, ic = ib == 2 ? 0 : ib + 1;
                    const double ax = Q[ia][0], ay = Q[ia][1], bx = Q[ib][0], by = Q[ib][1];
                    const double qx = Q[ic][0], qy = Q[ic][1];
                    const double mx = cmul(cadd(ax, bx), 0.5), my = cmul(cadd(ay, by), 0.5);
                    if ((path >> lev) & 1) {
                        Q[0][0] = mx; Q[0][1] = my; Q[1][0] = bx; Q[1][1] = by;
                    } else {
                        Q[0][0] = ax; Q[0][1] = ay; Q[1][0] = mx; Q[1][1] = my;
                    }
                    Q[2][0] = qx; Q[2][1] = qy;
                }
                const double cr = csub(cmul(csub(Q[1][0], Q[0][0]), csub(Q[2][1], Q[0][1])),
                                       cmul(csub(Q[1][1], Q[0][1]), csub(Q[2][0], Q[0][0])));
                const double At = cmul(0.5, cr);
                const double qx = div3(cadd(cadd(Q[0][0], Q[1][0]), Q[2][0]));
                const double qy = div3(cadd(cadd(Q[0][1], Q[1][1]), Q[2][1]));
                const double rho = bilinear(A.grid, A.rho, cadd(px, qx), cadd(py, qy), LdgLoad());
                const double wgt = cmul(At, rho);
                sw = cadd(sw, wgt);
                swx = cadd(swx, cmul(wgt, qx));
                swy = cadd(swy, cmul(wgt, qy));
                nq++;
            }
        }
        const double curx = cdiv(swx, sw), cury = cdiv(swy, sw);
        const double dx = csub(prevx, curx), dy = csub(prevy, cury);
        const double dist = sqrt(cadd(cmul(dx, dx), cmul(dy, dy)));
        prevx = curx;
        prevy = cury;
        if (dist < E) break;
    }
    cx = prevx;
    cy = prevy;
}

// stored rings: k_cells_t writes them in CVD mode, k_output_t reads them
struct RingBuf {
    double2 *v;                // [i * n_local + cell] (slot-major), ring order from the canonical vertex
    int *la;                   // incoming line code of ring vertex i
    uint8_t *n;                // vertices, 0 = no ring (ghost, failed, or retried)
};

// initial ring B ∩ Oct_i: the octagon (vertex k between sides k and k+1), clipped by the box
// sides it crosses.  Returns the clip status (0 ok).
__device__ __forceinline__ int init_ring(TPoly &P, const CellGeom &g, double S, const CellArgs &A, ClipStats &cs) {
#pragma unroll
    for (int k = 0; k < 8; k++) {
        // consecutive octagon sides have det = 1 exactly, so the canonical Cramer vertex is
        // the numerators themselves (x / 1 = x): no division
        const Line La = wall_line(-1 - k, g.px, g.py, g.r_oct, g.bx0, g.by0, g.bx1, g.by1);
        const Line Lb = wall_line(-1 - ((k + 1) & 7), g.px, g.py, g.r_oct, g.bx0, g.by0, g.bx1, g.by1);
        const double x = csub(cmul(La.r, Lb.ny), cmul(La.ny, Lb.r));
        const double y = csub(cmul(La.nx, Lb.r), cmul(La.r, Lb.nx));
        P.v[k * TB] = make_double2(x, y);
        P.K[k * TB] = store_K(-1.0);
        set_r2(P, k, x, y, -1.0);
        P.la[k * TB] = -1 - k;
        P.prv[k * TB] = (uint8_t)((k + 7) & 7);
        P.nxt[k * TB] = (uint8_t)((k + 1) & 7);
    }
    P.used = 0xffu;
    P.wall = 0xffu;
    int fail = 0;
    if (csub(g.px, g.bx0) < S || csub(g.bx1, g.px) < S || csub(g.py, g.by0) < S || csub(g.by1, g.py) < S) {
        for (int b = 0; b < 4 && !fail; b++) {
            const int code = -9 - b;
            fail = clip_t(P, code, wall_line(code, g.px, g.py, g.r_oct, g.bx0, g.by0, g.bx1, g.by1), g, A, cs);
        }
    }
    return fail;
}

// Keep rule fast path (S3, P:499-510 in reading L10): every Delaunay triangle around p_i is kept
// when the cell is deep inside -- then the canonical keep_tri would return true for each of them,
// so it need not run.  The triangle (i, a, b) of a point-point ring vertex has its exact
// circumcentre c within R_i of p_i (R_i: the rounded-up max vertex distance plus error bound
// the search uses) and |p_x - c| = |p_i - c| for x in {i, a, b}; its centroid lies within
// 4 R_i / 3 of p_i (|p_a - p_i| <= 2 R_i).  So it is kept if
//   * c stays inside B: p_i farther than R_i from every box side;
//   * c is in the three octagons: R_i below their inradius r_x = fac h(p_x) cos(pi/8), with
//     h(p_x) >= h(p_i) - c L_mu 2 R_i (h = c mu~, mu~ L_mu-Lipschitz);
//   * phi~(g) < keep_tol: phi~(p_i) + L_phi 4 R_i / 3 < keep_tol (phi~ L_phi-Lipschitz).
// All with relative margins (1e-9 .. 1e-6) far above the canonical arithmetic's rounding.
__device__ __forceinline__ bool interior_keeps_all_R(const CellArgs &A, double px, double py, double h, double R) {
    const Grid &g = A.grid;
    if (!(px - g.x0 > R * (1.0 + 1e-9) + 1e-300 && g.x1 - px > R * (1.0 + 1e-9) && py - g.y0 > R * (1.0 + 1e-9) &&
          g.y1 - py > R * (1.0 + 1e-9)))
        return false;
    const double hmin = (h - A.c * A.lip_mu * 2.0 * R) * (1.0 - 1e-9);
    if (!(R < A.fac_voro * hmin * COS_PI8 * (1.0 - 1e-9))) return false;
    const double ph = bilinear(g, A.phi, px, py, LdgLoad());
    // validity 1 (Tests 1-3): every midpoint (within 2R of p_i) and centroid inside keeps the triangle
    if (A.validity) return ph + A.lip_phi * 2.0 * R * (1.0 + 1e-6) + 1e-12 * (1.0 + fabs(ph)) < 0.0;
    return ph + A.lip_phi * (4.0 / 3.0) * R * (1.0 + 1e-6) + 1e-12 * (1.0 + fabs(ph)) < A.keep_tol;
}

__device__ __forceinline__ bool interior_keeps_all(const TPoly &P, const CellArgs &A, double px, double py, double h) {
    if (P.wall & P.used) return false;
    return interior_keeps_all_R(A, px, py, h, sqrt((double)poly_R2(P)) * (1.0 + 1e-9));
}

#ifndef TM_WMINB
#define TM_WMINB 5  // min resident blocks per SM of the warm-certification kernels (register cap)
#endif

template <int MODE>
__global__ void __launch_bounds__(TB, (MODE & M_WCERT) ? TM_WMINB : TM_TMINB) k_cells_t(CellArgs A, int32_t *retry_list,
                                                          unsigned long long *retry_cnt, RingBuf R) {
    // output split: this kernel stores the ring and k_output_t computes the centroid, quadrature
    // and treatment (CVD), or the triangles and ELL rows (DistMesh) -- a smaller kernel body
    // (instruction cache) for the search
    constexpr bool CSPLIT = split_rings(MODE);
    constexpr bool TSPLIT = split_tris(MODE);
    extern __shared__ __align__(16) unsigned char tsmem[];
    const int tid = threadIdx.x;
    // TM_BLOCK_ORDER=1: blocks taken from both ends of the sorted order first (the first and last
    // bin rows hold the boundary arcs, whose octagon-bounded cells are the slow ones), the middle last
#if TM_BLOCK_ORDER == 1
    const unsigned bid = (blockIdx.x & 1u) ? gridDim.x - 1u - (blockIdx.x >> 1) : (blockIdx.x >> 1);
#else
    const unsigned bid = blockIdx.x;
#endif
    const int64_t cell = (int64_t)bid * TB + tid;
    const int lane = tid & 31;
    TPoly P = tpoly_bind(tsmem, tid);
    bool live = false;
    int32_t orig = 0;
    const int64_t n_live = live_local(A);
    if (cell < n_live) {
        orig = __ldg(A.perm + cell);
        live = orig < live_owned(A);
    }
    // ---- per-cell results consumed by the warp-collective emission below
    int t_own = 0;
    unsigned keptmask = 0;  // slots whose (owned) point-point vertex is a kept triangle
    int32_t gi = 0, nid = 0;
    ClipStats cs;
    unsigned long long nq = 0;
    SearchCtx sc;
    sc.n_cand = 0;
    int fail = 0;
    double px = 0.0, py = 0.0, h = 0.0;
    CellGeom cgm = {};
    // search state (kept outside `if (live)` so that the whole warp runs the
    // flat candidate loop below in lockstep)
    float R2 = 0.f;
    const double MARG = 1.0 + 1e-9;
    const BinGeom &bg = A.bg;
    int rh = 0, ux = 0, uy = 0, nlx = 0, nly = 0, hb = 0, hoff = 0;
    double lsx = 0.0, lsy = 0.0;
    unsigned key[8];
    // candidate iterator: phase (0 ring 1, 1 rings >= 2 clipped to a box, 2 done), ring-1 position
    // (phase 1: ring rk, side 0-3, cursor cvx up to cend along it; cvy / cfix the fixed row / column)
    int wi = 0, wn = 0;  // warm-start cursor (phase -1)
    int ph = 2, rr = 0, t = 0, tend = 0, cvx = 0, cvy = 0, cend = -1, cfix = 0, rk = 1, side = 4, kmax = 0;
    int bxa = 0, bxb = -1, bya = 0, byb = -1;
    double r_oct = 0.0;
    if (live) {
        px = __ldg(A.xs + cell);
        py = __ldg(A.ys + cell);
        h = __ldg(A.hs + cell);
        gi = __ldg(A.gids + cell);
        nid = A.nbr_by_gid ? gi : orig;  // warm-start key (gid on strips, else caller index)
        if (nid < 0 || (int64_t)nid >= A.nbr_keys) nid = -1;  // outside the key space: no warm start
        sc.px = px; sc.py = py; sc.cell = (int)cell;
        const double S = cmul(A.fac_voro, h);
        r_oct = cmul(S, COS_PI8);
        const double bx0 = A.grid.x0, by0 = A.grid.y0, bx1 = A.grid.x1, by1 = A.grid.y1;
        cgm = {px, py, r_oct, bx0, by0, bx1, by1};
        // the flat search starts from B ∩ Oct_i; the warm path only when its direct
        // construction fails (phase A below)
        if constexpr (!(MODE & M_WCERT)) fail = init_ring(P, cgm, S, A, cs);
        R2 = poly_R2(P);
        // ---- candidate order over the two-level cell list (L11 stopping rule)
        int hbx = (int)floor((px - bg.x0) * bg.isx), hby = (int)floor((py - bg.y0) * bg.isy);
        hbx = hbx < 0 ? 0 : (hbx >= bg.nbx ? bg.nbx - 1 : hbx);
        hby = hby < 0 ? 0 : (hby >= bg.nby ? bg.nby - 1 : hby);
        hb = hby * bg.nbx + hbx;
        rh = __ldg(A.rlev + hb);
        hoff = __ldg(A.leaf_off + hb);
        ux = leaf_coord(px, bg.x0, bg.isx, bg.nbx, rh);
        uy = leaf_coord(py, bg.y0, bg.isy, bg.nby, rh);
        nlx = bg.nbx << rh;
        nly = bg.nby << rh;
        lsx = bg.sx * pow2neg(rh);
        lsy = bg.sy * pow2neg(rh);
        if constexpr (!(MODE & M_WCERT)) {
            // ring 1: the 8 neighbours nearest first (keys: d2 as float bits, low 3 bits = index)
            const double gl = px - (bg.x0 + ux * lsx), gr = (bg.x0 + (ux + 1) * lsx) - px;
            const double gd = py - (bg.y0 + uy * lsy), gu = (bg.y0 + (uy + 1) * lsy) - py;
            const int ddx[8] = {-1, 1, 0, 0, -1, 1, -1, 1};
            const int ddy[8] = {0, 0, -1, 1, -1, -1, 1, 1};
    #pragma unroll
            for (int q = 0; q < 8; q++) {
                const double gx = fmax(ddx[q] < 0 ? gl : (ddx[q] > 0 ? gr : 0.0), 0.0);
                const double gy = fmax(ddy[q] < 0 ? gd : (ddy[q] > 0 ? gu : 0.0), 0.0);
                const float d2 = __double2float_rd(gx * gx + gy * gy);
                key[q] = (__float_as_uint(fmaxf(d2, 0.f)) & ~7u) | (unsigned)q;
            }
            // 19-comparator sorting network for 8 keys
            cswap(key[0], key[2]); cswap(key[1], key[3]); cswap(key[4], key[6]); cswap(key[5], key[7]);
            cswap(key[0], key[4]); cswap(key[1], key[5]); cswap(key[2], key[6]); cswap(key[3], key[7]);
            cswap(key[0], key[1]); cswap(key[2], key[3]); cswap(key[4], key[5]); cswap(key[6], key[7]);
            cswap(key[2], key[4]); cswap(key[3], key[5]);
            cswap(key[1], key[4]); cswap(key[3], key[6]);
            cswap(key[1], key[2]); cswap(key[3], key[4]); cswap(key[5], key[6]);
            // ring 0: the home leaf first
            int st, cnt;
            vleaf_range(A, ux, uy, rh, ux, uy, hb, hoff, st, cnt);
            t = st;
            tend = st + cnt;
            // warm start: the cell's neighbours of the previous launch on the same point set
            // (caller ids) are clipped first -- the ring is then nearly final and R_max small
            // before the search; the search still certifies the cell (L11), so the result
            // does not depend on them
            wn = (A.warm && A.nbr_cnt && nid >= 0) ? min((int)A.nbr_cnt[nid], TM_NBR) : 0;
            ph = fail ? 2 : (wn > 0 ? -1 : 0);
            rr = 0;
            if (ph == -1) { cvx = t; cend = tend; t = tend = 0; }  // home range parked until the warm list ends
            if (ph == 2) t = tend;
        } else {
            wn = (A.warm && A.nbr_cnt && nid >= 0) ? min((int)A.nbr_cnt[nid], TM_NBR) : 0;
        }
    }
    unsigned trips = 0;
    if constexpr (!(MODE & M_WCERT)) {
    // ---- flat candidate loop: one candidate per thread per trip, the warp
    // re-converges every trip (a per-thread nested loop lets lanes drift apart)
    // the iterator: advance to this thread's next candidate slot (-1 when done)
    auto next_cand = [&]() -> int {
        int j = -1;
        if (t < tend) return t++;  // common case first: the next point of the current leaf
        while (ph < 2) {
            if (ph < 0) {
                if (wi >= wn) { ph = 0; t = cvx; tend = cend; cvx = 0; cend = -1; continue; }
                const int id = A.nbr[(int64_t)nid * TM_NBR + wi++];
                if (id < 0 || (int64_t)id >= A.nbr_keys) continue;
                const int js = A.inv_perm[id];  // stale for a gid not binned here: checked
                if (js < 0 || (int64_t)js >= n_live || (A.nbr_by_gid && __ldg(A.gids + js) != id)) continue;
                j = js;
                P.lmask |= 1ull << (j & 63);
                break;
            }
            if (t < tend) { j = t++; break; }
            const float lim = 4.0f * R2 * (float)MARG;
            if (ph == 0) {  // ring 1, sorted
                if (rr >= 8) {
                    // then rings k >= 2, each clipped to the box of leaves that can hold
                    // a point closer than 2 R_max (L11)
                    const double rad = 2.0 * sqrt((double)R2 * MARG) * (1.0 + 1e-6);
                    const double sxl = bg.isx * (double)(1 << rh), syl = bg.isy * (double)(1 << rh);
                    bxa = max(0, (int)floor((px - rad - bg.x0) * sxl));
                    bxb = min(nlx - 1, (int)floor((px + rad - bg.x0) * sxl));
                    bya = max(0, (int)floor((py - rad - bg.y0) * syl));
                    byb = min(nly - 1, (int)floor((py + rad - bg.y0) * syl));
                    kmax = max(max(ux - bxa, bxb - ux), max(uy - bya, byb - uy));
                    ph = 1;
                    rk = 1;
                    side = 4;  // -> start ring 2
                    continue;
                }
                unsigned kq = key[0];
#pragma unroll
                for (int u = 1; u < 8; u++)
                    if (rr == u) kq = key[u];
                rr++;
                if (__uint_as_float(kq & ~7u) * (1.0f - 1e-6f) >= lim) { rr = 8; continue; }  // the rest are farther
                const int q = (int)(kq & 7u);
                const int vx = ux + (q == 0 || q == 4 || q == 6 ? -1 : (q == 1 || q == 5 || q == 7 ? 1 : 0));
                const int vy = uy + (q == 2 || q == 4 || q == 5 ? -1 : (q == 3 || q == 6 || q == 7 ? 1 : 0));
                if (vx < 0 || vx >= nlx || vy < 0 || vy >= nly) continue;
                int st, cnt;
                vleaf_range(A, vx, vy, rh, ux, uy, hb, hoff, st, cnt);
                t = st;
                tend = st + cnt;
            } else {        // rings >= 2, side by side, clipped to the box; leaf-level pruning
                if (cvx > cend) {  // next side
                    if (++side >= 4) {
                        rk++;
                        if (rk > kmax) { ph = 2; break; }
                        const double dl = px - (bg.x0 + (ux - rk + 1) * lsx), dr = (bg.x0 + (ux + rk) * lsx) - px;
                        const double dd = py - (bg.y0 + (uy - rk + 1) * lsy), du = (bg.y0 + (uy + rk) * lsy) - py;
                        const double dmin = fmin(fmin(dl, dr), fmin(dd, du));
                        if (dmin > 0.0 && dmin * dmin * (1.0 - 1e-9) >= 4.0 * (double)R2 * MARG) { ph = 2; break; }
                        side = 0;
                    }
                    // side 0: bottom row, 1: top row, 2: left column, 3: right column
                    if (side < 2) {
                        cvy = side == 0 ? uy - rk : uy + rk;
                        cvx = max(ux - rk, bxa);
                        cend = (cvy < bya || cvy > byb) ? cvx - 1 : min(ux + rk, bxb);
                    } else {
                        cfix = side == 2 ? ux - rk : ux + rk;
                        cvx = max(uy - rk + 1, bya);
                        cend = (cfix < bxa || cfix > bxb) ? cvx - 1 : min(uy + rk - 1, byb);
                    }
                    continue;
                }
                const int vx = side < 2 ? cvx : cfix, vy = side < 2 ? cvy : cvx;
                cvx++;
                if (leaf_d2(bg, lsx, lsy, vx, vy, px, py) * (1.0 - 1e-9) >= 4.0 * (double)R2 * MARG) continue;
                int st, cnt;
                vleaf_range(A, vx, vy, rh, ux, uy, hb, hoff, st, cnt);
                t = st;
                tend = st + cnt;
            }
        }
        return j;
    };
    double lim2 = 4.0 * (double)R2 * MARG;  // (2 R_max)^2 with margin, updated with R_max
    // ---- (C) flat candidate loop
    int j = next_cand();
    double xj = 0.0, yj = 0.0;
    if (j >= 0) { xj = __ldg(A.xs + j); yj = __ldg(A.ys + j); }
    for (;;) {
        if (!__any_sync(0xffffffffu, j >= 0)) break;
        trips++;
        // one candidate per thread per trip (skipping far candidates inside the iterator,
        // or testing several per step, lets single lanes run alone: measured slower);
        // the next candidate is fetched before this one is clipped (its load overlaps the
        // clip; leaf pruning then uses the R_max before the clip, which is conservative)
        const int cj = j;
        const double cxj = xj, cyj = yj;
        j = next_cand();
        if (j >= 0) { xj = __ldg(A.xs + j); yj = __ldg(A.ys + j); }
        if (cj >= 0) {
            sc.n_cand++;
            const double dx = csub(cxj, px), dy = csub(cyj, py);
            const double d2 = dx * dx + dy * dy;
            if (d2 < lim2 && cj != (int)cell) {
                if (dx == 0.0 && dy == 0.0) {
                    atomicAdd(&A.st->n_duplicate, 1ull);
                } else {
                    const unsigned long long c0 = cs.clips;
                    fail = clip_t(P, cj, bisector(dx, dy), cgm, A, cs);
                    if (fail) { ph = 2; j = -1; t = tend; }
                    else if (cs.clips != c0) { R2 = poly_R2(P); lim2 = 4.0 * (double)R2 * MARG; }
                }
            }
        }
    }
    } else {
        // ---- (A) warm clips, one thread per cell: the cell's neighbours of the previous
        // launch on the same point set (ids -> slots of this binning; a stale id fails the
        // check).  Every lane clips about the same number (~6) of lines: uniform work.
        if (live && !fail) {
            if (wn == 0) fail = -1;  // no warm list: the 32-lane pass computes the cell from scratch
            if (!fail) fail = init_ring(P, cgm, cmul(A.fac_voro, h), A, cs);
            for (int w = 0; w < wn && !fail; w++) {
                const int id = A.nbr[(int64_t)nid * TM_NBR + w];
                if (id < 0 || (int64_t)id >= A.nbr_keys) continue;
                const int js = A.inv_perm[id];
                if (js < 0 || (int64_t)js >= n_live || js == (int)cell ||
                    (A.nbr_by_gid && __ldg(A.gids + js) != id))
                    continue;
                const double dx = csub(__ldg(A.xs + js), px), dy = csub(__ldg(A.ys + js), py);
                if (dx == 0.0 && dy == 0.0) {
                    atomicAdd(&A.st->n_duplicate, 1ull);
                    continue;
                }
                fail = clip_t(P, js, bisector(dx, dy), cgm, A, cs);
            }
            R2 = poly_R2(P);
        }
        // ---- (B) certification (L11), warp-cooperative: every point within 2 R_max of p_c must be
        // tested against cell c's warm ring.  The warp's cells are grouped by home leaf (cells are
        // sorted by leaf); per group the lanes enumerate, once, the leaves of the union of the
        // cells' 2 R_max boxes, take one candidate point each and distance-test it against every
        // cell of the group.  The near (cell, point) pairs go to a per-warp queue; 32 at a time
        // the lanes test one pair each against that cell's ring (shared memory).  A point that
        // does not cut a ring cannot cut any later (smaller) ring, so only the rare cutters are
        // clipped, by the cell's own lane, in any order: the cell is the same (exact topology).
        WarpQ &W = reinterpret_cast<WarpQ *>(tsmem + TSMEM)[tid >> 5];
        const int wbase = tid & ~31;
        const bool act = live && !fail;
        W.cx[lane] = px;
        W.cy[lane] = py;
        W.used[lane] = act ? P.used : 0u;
        W.wall[lane] = P.wall;
        const unsigned todo = __ballot_sync(0xffffffffu, act);
        __syncwarp();
        const unsigned lt = (1u << lane) - 1u;
        int qn = 0;
        // test the first m queued pairs (one per lane), clip the cutters, drop the tested pairs
        auto flush = [&](int m) {
            __syncwarp();
            int cq = 0, jq = 0;
            double dxq = 0.0, dyq = 0.0;
            bool flq = false;
            if (lane < m) {
                jq = W.qj[lane];
                cq = W.qc[lane];
                const unsigned usedq = (int64_t)jq != (int64_t)bid * TB + wbase + cq ? W.used[cq] : 0u;
                if (usedq) {
                    dxq = csub(__ldg(A.xs + jq), W.cx[cq]);
                    dyq = csub(__ldg(A.ys + jq), W.cy[cq]);
                }
                if (usedq && dxq == 0.0 && dyq == 0.0) {
                    atomicAdd(&A.st->n_duplicate, 1ull);
                } else if (usedq) {
                    const Line L = bisector(dxq, dyq);
                    const double n1 = fabs(L.nx) + fabs(L.ny);
                    const double c8 = 8.0 * EPS * n1 * n1;
                    const TPoly Pq = tpoly_bind(tsmem, wbase + cq);
                    const unsigned wallq = W.wall[cq];
                    unsigned hit = 0u, isl = 0u;
#pragma unroll
                    for (int k = 0; k < VLO; k++) {  // all slots, masked: no divergence between rings
                        const double2 vv = Pq.v[k * TB];
                        isl |= (unsigned)(Pq.la[k * TB] == jq) << k;
                        const double del = fma(L.nx, vv.x, L.ny * vv.y) - L.r;
                        const bool o = ((wallq >> k) & 1u) ? wall_out(L, vv.x, vv.y)
                                                           : del > -fma(n1, (double)Pq.K[k * TB], c8);
                        hit |= (unsigned)o << k;
                    }
                    if (VLO < VMAX && (usedq >> VLO)) {
#pragma unroll
                        for (int k = VLO; k < VMAX; k++) {
                            const double2 vv = Pq.v[k * TB];
                            isl |= (unsigned)(Pq.la[k * TB] == jq) << k;
                            const double del = fma(L.nx, vv.x, L.ny * vv.y) - L.r;
                            const bool o = ((wallq >> k) & 1u) ? wall_out(L, vv.x, vv.y)
                                                               : del > -fma(n1, (double)Pq.K[k * TB], c8);
                            hit |= (unsigned)o << k;
                        }
                    }
                    // cut or undecided, and not a line of the ring (a line already bounding it never cuts)
                    flq = (hit & usedq) && !(isl & usedq);
                }
            }
            __syncwarp();
            // drop the tested pairs (qn - m < 32 remain)
            int rj = 0, rc = 0;
            const bool mv = lane < qn - m;
            if (mv) { rj = W.qj[m + lane]; rc = W.qc[m + lane]; }
            __syncwarp();
            if (mv) { W.qj[lane] = rj; W.qc[lane] = (uint8_t)rc; }
            qn -= m;
            // cutters (rare): in rounds, the lowest flagged lane of every cell clips that cell --
            // cells differ between the round's leaders, so they clip in parallel.  The ring's
            // masks live in shared memory during the certification; the owners reload them after.
            unsigned fb = __ballot_sync(0xffffffffu, flq);
            while (fb) {
                const unsigned same = __match_any_sync(0xffffffffu, flq ? cq : -1 - lane);
                if (flq && __ffs(same) - 1 == lane) {
                    const int ct = wbase + cq;  // thread (and ring) of cell cq in this block
                    TPoly Pc = tpoly_bind(tsmem, ct);
                    Pc.used = W.used[cq];
                    Pc.wall = W.wall[cq];
                    if (Pc.used) {
                        const double roc =
                            cmul(cmul(A.fac_voro, __ldg(A.hs + (int64_t)bid * TB + ct)), COS_PI8);
                        const CellGeom gc = {W.cx[cq], W.cy[cq], roc, A.grid.x0, A.grid.y0, A.grid.x1, A.grid.y1};
                        const int fc = clip_t(Pc, jq, bisector(dxq, dyq), gc, A, cs);
                        W.used[cq] = fc ? 0u : Pc.used;  // 0: the cell failed, its code in wall
                        W.wall[cq] = fc ? (unsigned)fc : Pc.wall;
                    }
                    flq = false;
                }
                __syncwarp();
                fb = __ballot_sync(0xffffffffu, flq);
            }
        };
        // groups: runs of lanes with the same home leaf (blocks of 2^TM_GROUP_SHIFT leaves per side)
        const unsigned long long lkey = ((unsigned long long)rh << 48) |
                                        ((unsigned long long)(unsigned)(ux >> TM_GROUP_SHIFT) << 24) |
                                        (unsigned)(uy >> TM_GROUP_SHIFT);
        const unsigned long long lprev = __shfl_up_sync(0xffffffffu, lkey, 1);
        for (unsigned hm = __ballot_sync(0xffffffffu, lane == 0 || lkey != lprev); hm;) {
            const int g0 = __ffs(hm) - 1;
            hm &= hm - 1;
            const int g1 = hm ? __ffs(hm) - 1 : 32;
            const unsigned gmask = (g1 == 32 ? 0xffffffffu : ((1u << g1) - 1u)) & ~((1u << g0) - 1u);
            const unsigned gact = gmask & todo;
            if (!gact) continue;
            const int rhg = __shfl_sync(0xffffffffu, rh, g0), uxg = __shfl_sync(0xffffffffu, ux, g0);
            const int uyg = __shfl_sync(0xffffffffu, uy, g0), hbg = __shfl_sync(0xffffffffu, hb, g0);
            const int hoffg = __shfl_sync(0xffffffffu, hoff, g0);
            const double lsxg = bg.sx * pow2neg(rhg), lsyg = bg.sy * pow2neg(rhg);
            const double sxl = bg.isx * (double)(1 << rhg), syl = bg.isy * (double)(1 << rhg);
            const int nlxg = bg.nbx << rhg, nlyg = bg.nby << rhg;
            // union of the group's leaf boxes that can hold a point closer than 2 R_max
            int bxa = INT_MAX, bxb = INT_MIN, bya = INT_MAX, byb = INT_MIN;
            if ((gact >> lane) & 1u) {
                const double rad = 2.0 * sqrt((double)R2 * MARG) * (1.0 + 1e-6);
                bxa = max(0, (int)floor((px - rad - bg.x0) * sxl));
                bxb = min(nlxg - 1, (int)floor((px + rad - bg.x0) * sxl));
                bya = max(0, (int)floor((py - rad - bg.y0) * syl));
                byb = min(nlyg - 1, (int)floor((py + rad - bg.y0) * syl));
            }
            bxa = __reduce_min_sync(0xffffffffu, bxa);
            bxb = __reduce_max_sync(0xffffffffu, bxb);
            bya = __reduce_min_sync(0xffffffffu, bya);
            byb = __reduce_max_sync(0xffffffffu, byb);
            // float prefilter data relative to the group origin (the first cell): distances of a
            // few h are exact to ~1e-7 relative, far inside the 1e-4 margin of the bound
            const double ox = __shfl_sync(0xffffffffu, px, g0), oy = __shfl_sync(0xffffffffu, py, g0);
            if ((gact >> lane) & 1u)
                W.cf[lane] = make_float4((float)(px - ox), (float)(py - oy),
                                         __double2float_ru(4.0 * (double)R2 * MARG * (1.0 + 1e-4)), 0.f);
            __syncwarp();
            const float lxf = (float)(bg.x0 - ox), lyf = (float)(bg.y0 - oy);
            const int nLx = bxb - bxa + 1, nL = nLx * (byb - bya + 1);
            for (int l0 = 0; l0 < nL; l0 += 32) {
                const int l = l0 + lane;
                int st = 0, cnt = 0;
                if (l < nL) {
                    const int vy = l / nLx, vx = bxa + (l - vy * nLx), vyy = bya + vy;
                    // the rectangle to test: the virtual leaf, or -- in a coarser bin -- the whole
                    // coarse leaf, which vleaf_range returns once, at its virtual leaf closest to the
                    // group's first home leaf (inside the union box, which holds that leaf); a group
                    // spanning several home leaves must test the coarse leaf as a whole
                    int x0l = vx, y0l = vyy, span = 1;
                    bool canon = true;
                    {
                        const int b = (vyy >> rhg) * bg.nbx + (vx >> rhg);
                        const int rb = b == hbg ? rhg : __ldg(A.rlev + b);
                        if (rb < rhg) {
                            const int d = rhg - rb, Lx = vx >> d, Ly = vyy >> d;
                            const int rx = min(max(uxg, Lx << d), ((Lx + 1) << d) - 1);
                            const int ry = min(max(uyg, Ly << d), ((Ly + 1) << d) - 1);
                            canon = rx == vx && ry == vyy;
                            x0l = Lx << d;
                            y0l = Ly << d;
                            span = 1 << d;
                        }
                    }
                    if (canon) {
                        // any cell of the group within reach (float, conservative: the leaf is widened
                        // by 1e-5 of its size, the bound carries a 1e-4 margin)
                        const float ax = lxf + (float)(x0l * lsxg), ay = lyf + (float)(y0l * lsyg);
                        const float wx = (float)(span * lsxg), wy = (float)(span * lsyg), ex = 1e-5f * wx,
                                    ey = 1e-5f * wy;
                        bool need = false;
                        for (unsigned m = gact; m; m &= m - 1) {
                            const int c = __ffs(m) - 1;
                            const float4 q = W.cf[c];
                            const float gx = fmaxf(fmaxf(ax - ex - q.x, q.x - (ax + wx + ex)), 0.f);
                            const float gy = fmaxf(fmaxf(ay - ey - q.y, q.y - (ay + wy + ey)), 0.f);
                            need |= gx * gx + gy * gy < q.z;
                        }
                        if (need) vleaf_range(A, vx, vyy, rhg, uxg, uyg, hbg, hoffg, st, cnt);
                    }
                }
                int incl = cnt;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int u = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += u;
                }
                const int tot = __shfl_sync(0xffffffffu, incl, 31);
                if ((gact >> lane) & 1u) sc.n_cand += (unsigned long long)tot;
                for (int base = 0; base < tot; base += 32) {
                    trips++;
                    const int tt = base + lane;
                    int k = 0;  // leaf of candidate tt: the leaves whose inclusive count is <= tt
#pragma unroll
                    for (int s = 16; s > 0; s >>= 1)
                        if (__shfl_sync(0xffffffffu, incl, k + s - 1) <= tt) k += s;
                    const int kk = k < 31 ? k : 31;
                    const int stk = __shfl_sync(0xffffffffu, st, kk);
                    const int exk = __shfl_sync(0xffffffffu, incl - cnt, kk);
                    const bool valid = tt < tot;
                    const int j = stk + (tt - exk);
                    float xjf = 3e38f, yjf = 3e38f;
                    if (valid) { xjf = (float)(__ldg(A.xs + j) - ox); yjf = (float)(__ldg(A.ys + j) - oy); }
                    // the group's cells near this lane's candidate, as a mask (conservative: a few
                    // extra pairs are harmless, the ring test decides; the cell's own point and exact
                    // duplicates are sorted out there) ...
                    unsigned nm = 0u;
                    for (unsigned m = gact; m; m &= m - 1) {
                        const int c = __ffs(m) - 1;
                        const float4 q = W.cf[c];
                        const float dx = xjf - q.x, dy = yjf - q.y;
                        nm |= (unsigned)(fmaf(dx, dx, dy * dy) < q.z) << c;
                    }
                    // ... queued one pair per lane per round (rounds = the most near cells of a lane)
                    for (;;) {
                        const unsigned b = __ballot_sync(0xffffffffu, nm != 0u);
                        if (!b) break;
                        if (nm) {
                            const int pos = qn + __popc(b & lt);
                            W.qj[pos] = j;
                            W.qc[pos] = (uint8_t)(__ffs(nm) - 1);
                            nm &= nm - 1;
                        }
                        qn += __popc(b);
                        if (qn >= 32) flush(32);
                    }
                }
            }
        }
        if (qn > 0) flush(qn);
        __syncwarp();
        if (act) {  // the certified ring (or the failure) back to its owner
            if (W.used[lane]) {
                P.used = W.used[lane];
                P.wall = W.wall[lane];
            } else {
                fail = (int)W.wall[lane];
            }
        }
    }
    if (live) {
        if (fail == -1) {
            // more than VMAX slots (or an undecided filter without TM_THREAD_EXACT):
            // the 32-lane group kernel redoes this cell
            const unsigned long long k = atomicAdd(retry_cnt, 1ull);
            retry_list[k] = (int32_t)cell;
            if (A.nbr_cnt && nid >= 0) A.nbr_cnt[nid] = 0;
            live = false;
        } else if (fail) {
            if (A.nbr_cnt && nid >= 0) A.nbr_cnt[nid] = 0;
            atomicAdd(&A.st->n_degenerate, 1ull);
            if (MODE & M_TREAT) {
                A.x_out[orig] = px; A.y_out[orig] = py; A.d_prev_out[orig] = 0.0; A.status[orig] = 2;
            }
            if (MODE & M_HAT) { A.x_hat[orig] = px; A.y_hat[orig] = py; }
            if (MODE & M_ELL) A.deg[cell] = 0;
            live = false;
        }
    }
    // canonical start vertex: the smallest (incoming, outgoing) line pair with points named
    // by their ids (gid / caller index, walls by their negative codes) -- the oracle's
    // canonical rotation (O2).  Every ring traversal below (neighbour lists, ELL rows,
    // centroid and quadrature sums) is then independent of the clipping order AND of the
    // binning, so the sums run in the oracle's order (bit-identical CVD, L25)
    int start = 0;
    if (live) {
        long long best = LLONG_MAX;
        for (unsigned m = P.used; m; m &= m - 1) {  // used slots only: a free slot's link is garbage
            const int k = __ffs(m) - 1;
            const int la = P.la[k * TB], lb = P.la[P.nxt[k * TB] * TB];
            const long long key = ((long long)(la >= 0 ? __ldg(A.gids + la) : la) << 32) |
                                  (unsigned)(lb >= 0 ? __ldg(A.gids + lb) : lb);
            if (key < best) { best = key; start = k; }
        }
    }
    const int nv = live ? __popc(P.used) : 0;
    // neighbour list for the next launch's warm start (point ids, ring order)
    if (live && A.nbr && nid >= 0) {
        int k = start, c = 0;
        for (int q = 0; q < nv; q++) {
            const int a = P.la[k * TB];
            if (a >= 0) A.nbr[(int64_t)nid * TM_NBR + c++] = A.nbr_by_gid ? __ldg(A.gids + a) : __ldg(A.perm + a);
            k = P.nxt[k * TB];
        }
        A.nbr_cnt[nid] = (uint8_t)c;
    }
    // ---- S3: Delaunay triangles at point-point vertices + keep rule; ELL rows
    int ell = 0;
    if (!TSPLIT && live && (MODE & (M_TRI | M_ELL))) {
        unsigned keptall = 0;  // for the ELL: kept, owned or not
        const bool all_in = interior_keeps_all(P, A, px, py, h);
        int k = start;
        for (int c = 0; c < nv; c++) {
            const int kn = P.nxt[k * TB];
            const int a = P.la[k * TB], b = P.la[kn * TB];
            if (a >= 0 && b >= 0) {
                const int32_t ga = __ldg(A.gids + a), gb = __ldg(A.gids + b);
                if (all_in) {
                    keptall |= 1u << k;
                    if (gi < ga && gi < gb) keptmask |= 1u << k;
                } else if (gi < ga && gi < gb) {
                    const int sv = ga < gb ? a : b, sw = ga < gb ? b : a;
                    if (keep_tri(A, (int)cell, sv, sw, P.v[k * TB].x, P.v[k * TB].y)) {
                        keptmask |= 1u << k;
                        keptall |= 1u << k;
                    }
                } else if (MODE & M_ELL) {
                    int s3[3] = {(int)cell, a, b};
                    int32_t g3[3] = {gi, ga, gb};
                    for (int u = 0; u < 2; u++)
                        for (int w = 0; w < 2 - u; w++)
                            if (g3[w] > g3[w + 1]) {
                                int32_t tg = g3[w]; g3[w] = g3[w + 1]; g3[w + 1] = tg;
                                int ts = s3[w]; s3[w] = s3[w + 1]; s3[w + 1] = ts;
                            }
                    const double uxx = __ldg(A.xs + s3[0]), uyy = __ldg(A.ys + s3[0]);
                    const Line B1 = bisector(csub(__ldg(A.xs + s3[1]), uxx), csub(__ldg(A.ys + s3[1]), uyy));
                    const Line B2 = bisector(csub(__ldg(A.xs + s3[2]), uxx), csub(__ldg(A.ys + s3[2]), uyy));
                    double ox, oy;
                    cramer(B1, B2, ox, oy);
                    if (keep_tri(A, s3[0], s3[1], s3[2], ox, oy)) keptall |= 1u << k;
                }
            }
            k = kn;
        }
        if (!(MODE & M_TRI)) keptmask = 0;
        t_own = __popc(keptmask);
        if (MODE & M_ELL) {
            // neighbour a = incoming line of slot k borders a kept triangle at k or at prev(k)
            k = start;
            for (int c = 0; c < nv; c++) {
                const int a = P.la[k * TB];
                const int kp = P.prv[k * TB];
                if (a >= 0 && (((keptall >> k) & 1u) || ((keptall >> kp) & 1u))) {
                    if (ell < A.adj_stride) A.adj[(int64_t)ell * A.n_local + cell] = a;
                    ell++;
                }
                k = P.nxt[k * TB];
            }
            A.deg[cell] = (uint8_t)(ell < A.adj_stride ? ell : A.adj_stride);
            if (ell > A.adj_stride) atomicAdd(&A.st->n_adj_overflow, 1ull);
        }
    }
    if (!TSPLIT && (MODE & M_TRI)) {
        // warp-aggregated allocation of the owned kept triangles
        __syncwarp();
        int incl = t_own;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        const int tot = __shfl_sync(0xffffffffu, incl, 31);
        unsigned long long base = 0;
        if (lane == 31 && tot > 0) base = atomicAdd(A.n_tri, (unsigned long long)tot);
        base = __shfl_sync(0xffffffffu, base, 31) + (unsigned long long)(incl - t_own);
        for (unsigned m = keptmask; m; m &= m - 1) {
            const int k = __ffs(m) - 1;
            const int a = P.la[k * TB], b = P.la[P.nxt[k * TB] * TB];
            if ((int64_t)base < A.tri_cap) {
                A.tri[3 * base] = gi;
                A.tri[3 * base + 1] = __ldg(A.gids + a);
                A.tri[3 * base + 2] = __ldg(A.gids + b);
            } else {
                atomicAdd(&A.st->n_tri_overflow, 1ull);
            }
            base++;
        }
    }
    if (CSPLIT && cell < A.n_local) {
        if (live) {
            double2 *rv = R.v + cell;
            int *rl = R.la + cell;
            int k = start;
            for (int i = 0; i < nv; i++) {
                rv[(int64_t)i * A.n_local] = P.v[k * TB];  // slot-major: a warp's stores coalesce
                rl[(int64_t)i * A.n_local] = P.la[k * TB];
                k = P.nxt[k * TB];
            }
        }
        R.n[cell] = (uint8_t)(live ? nv : 0);
    }
    // ---- S4a centroid of C_i (relative to p_i) and S5 treatment
    if (!CSPLIT && live && (MODE & (M_TREAT | M_HAT))) {
        double S2 = 0.0, sx = 0.0, sy = 0.0;
        int k = start;
        for (int c = 0; c < nv; c++) {
            const int kn = P.nxt[k * TB];
            const double x0 = P.v[k * TB].x, y0 = P.v[k * TB].y, x1 = P.v[kn * TB].x, y1 = P.v[kn * TB].y;
            const double cr = csub(cmul(x0, y1), cmul(x1, y0));
            S2 = cadd(S2, cr);
            sx = cadd(sx, cmul(cr, cadd(x0, x1)));
            sy = cadd(sy, cmul(cr, cadd(y0, y1)));
            k = kn;
        }
        double cx, cy;
        if (A.rho == nullptr) {
            cx = cdiv(sx, cmul(3.0, S2));
            cy = cdiv(sy, cmul(3.0, S2));
            nq += nv;
        } else {
            const double dp = A.d_prev ? __ldg(A.d_prev + orig) : -1.0;
            quad_centroid_t(P, start, nv, px, py, cmul(0.5, S2), h, dp, A, cx, cy, nq);
        }
        if (MODE & M_HAT) {
            A.x_hat[orig] = px + cx;
            A.y_hat[orig] = py + cy;
        }
        if (MODE & M_TREAT) {
            double qx, qy, dpo;
            const int s = treat_point(A.grid, A.phi, h, A.h_avg, A.fac_pt, A.fac_geps, A.damping, A.newton_max, px,
                                      py, px + cx, py + cy, qx, qy, dpo, LdgLoad(), A.projection, A.trace_max);
            A.x_out[orig] = qx;
            A.y_out[orig] = qy;
            A.d_prev_out[orig] = dpo;
            A.status[orig] = (int8_t)s;
            if (s & 2) atomicAdd(&A.st->n_fallback, 1ull);
        }
    }
    // ---- O8 work counters (TM_F_COUNT_WORK)
    if ((MODE & M_COUNT) && lane == 0) atomicAdd(&A.st->work[10], (unsigned long long)trips);
    if ((MODE & M_COUNT) && live) {
        const float R2f = poly_R2(P);
        const double rad = 2.0 * sqrt((double)R2f);
        const BinGeom &bg = A.bg;
        int ncert = 0;
        const int bxa = max(0, (int)floor((px - rad - bg.x0) * bg.isx));
        const int bxb = min(bg.nbx - 1, (int)floor((px + rad - bg.x0) * bg.isx));
        const int bya = max(0, (int)floor((py - rad - bg.y0) * bg.isy));
        const int byb = min(bg.nby - 1, (int)floor((py + rad - bg.y0) * bg.isy));
        for (int by = bya; by <= byb; by++) {
            const int s0 = __ldg(A.leaf_start + __ldg(A.leaf_off + by * bg.nbx + bxa));
            const int s1 = __ldg(A.leaf_start + __ldg(A.leaf_off + by * bg.nbx + bxb + 1));
            for (int s = s0; s < s1; s++) {
                const double dx = __ldg(A.xs + s) - px, dy = __ldg(A.ys + s) - py;
                ncert += (s != (int)cell) && (dx * dx + dy * dy < rad * rad);
            }
        }
        int degc = 0;
        for (unsigned m = P.used; m; m &= m - 1) {
            const int k = __ffs(m) - 1;
            degc += P.la[P.nxt[k * TB] * TB] >= 0 ? 1 : 0;
        }
        atomicAdd(&A.st->work[0], 1ull);
        atomicAdd(&A.st->work[1], (unsigned long long)ncert);
        atomicAdd(&A.st->work[2], (unsigned long long)degc);
        atomicAdd(&A.st->work[3], (unsigned long long)nv);
        atomicAdd(&A.st->work[4], (unsigned long long)t_own);
        atomicAdd(&A.st->work[5], (A.rho == nullptr) ? (unsigned long long)nv : nq);
        atomicAdd(&A.st->work[6], (unsigned long long)ell);
        atomicAdd(&A.st->work[7], sc.n_cand);
        atomicAdd(&A.st->work[8], cs.clips);
        atomicAdd(&A.st->work[9], cs.exact);
    }
}


// outputs of every stored ring: S3 triangles + keep rule and ELL rows, S4a centroid,
// S5 treatment, warm-start neighbour lists, O8 counters -- one thread per cell
#ifndef TM_QLEV1
#define TM_QLEV1 2  // quadrature levels done by k_output_t; deeper cells go to k_output_deep
#endif
#ifndef TM_DEEP_G
#define TM_DEEP_G 8  // lanes per deep cell in k_output_deep
#endif

// S4a result -> x_hat (tm_cvd_step) or S5 treatment (fused CVD update), caller order
template <int MODE>
__device__ __forceinline__ void cell_update(const CellArgs &A, int32_t orig, double px, double py, double h,
                                            double cx, double cy) {
    if (MODE & M_HAT) {
        A.x_hat[orig] = px + cx;
        A.y_hat[orig] = py + cy;
    }
    if (MODE & M_TREAT) {
        double qx, qy, dpo;
        const int s = treat_point(A.grid, A.phi, h, A.h_avg, A.fac_pt, A.fac_geps, A.damping, A.newton_max, px, py,
                                  px + cx, py + cy, qx, qy, dpo, LdgLoad(), A.projection, A.trace_max);
        A.x_out[orig] = qx;
        A.y_out[orig] = qy;
        A.d_prev_out[orig] = dpo;
        A.status[orig] = (int8_t)s;
        if (s & 2) atomicAdd(&A.st->n_fallback, 1ull);
    }
}

// the cells whose adaptive quadrature needs more than TM_QLEV1 levels, compacted, G lanes per
// cell: the lanes compute the sub-triangle terms of a level G at a time (descent, area,
// centroid, density lookup, the products w, w qx, w qy), the group's first lane adds them in
// sub-triangle order -- the same operations in the same order as k_output_t and the oracle
// (bit-identical), with the long serial chain of lookups of a deep cell cut G-fold
template <int MODE, int G>
__global__ void __launch_bounds__(128) k_output_deep(CellArgs A, RingBuf R, const int32_t *list,
                                                     const double2 *list_xy, const unsigned long long *cnt) {
    const int64_t n = (int64_t)*cnt;
    const int gl = threadIdx.x % G;  // lane in the group
    const unsigned gmask = (G == 32 ? 0xffffffffu : ((1u << G) - 1u) << ((threadIdx.x & 31) & ~(G - 1)));
    const int64_t ngroups = (int64_t)gridDim.x * (blockDim.x / G);
    for (int64_t it = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G; it < n; it += ngroups) {
        const int64_t cell = list[it];
        const int nv = (int)R.n[cell];
        const int32_t orig = __ldg(A.perm + cell);
        const double px = __ldg(A.xs + cell), py = __ldg(A.ys + cell), h = __ldg(A.hs + cell);
        const double2 *rv = R.v + cell;
        const int64_t ns = A.n_local;
        // area by the shoelace in ring order (every lane the same, as ring_centroid)
        double S2 = 0.0;
        for (int i = 0; i < nv; i++) {
            const double2 a = rv[(int64_t)i * ns], b = rv[(int64_t)(i + 1 == nv ? 0 : i + 1) * ns];
            S2 = cadd(S2, csub(cmul(a.x, b.y), cmul(b.x, a.y)));
        }
        const double dprev = A.d_prev ? __ldg(A.d_prev + orig) : -1.0;
        double eps = dprev >= 0.0 ? cdiv(dprev, h) : A.fac_pt;
        if (eps < A.fac_end) eps = A.fac_end;
        const double E = cmul(sqrt(cmul(0.5, S2)), eps);
        // levels 1..TM_QLEV1 were summed by k_output_t (same operations): continue from its centroid
        const double2 pv = list_xy[it];
        double prevx = pv.x, prevy = pv.y;
        unsigned long long nq = 0;
        for (int L = TM_QLEV1 + 1; L <= A.quad_max; L++) {
            const int depth = L - 1;
            const int64_t ntot = (int64_t)nv << depth;
            double sw = 0.0, swx = 0.0, swy = 0.0;
            for (int64_t base = 0; base < ntot; base += G) {
                const int64_t t = base + gl;
                double w = 0.0, wx = 0.0, wy = 0.0;
                if (t < ntot) {
                    const int fi = (int)(t >> depth);
                    double Q[3][2];
                    quad_descend(rv[(int64_t)fi * ns], rv[(int64_t)(fi + 1 == nv ? 0 : fi + 1) * ns], depth,
                                 t & (((int64_t)1 << depth) - 1), Q);
                    double At, qx, qy, ss, tt, f[4];
                    quad_leaf(Q, A, px, py, At, qx, qy, ss, tt, f);
                    const double rho = clerp(clerp(f[0], f[1], ss), clerp(f[2], f[3], ss), tt);
                    w = cmul(At, rho);
                    wx = cmul(w, qx);
                    wy = cmul(w, qy);
                }
                const int m = (int)(ntot - base < G ? ntot - base : G);
                for (int k = 0; k < m; k++) {  // in sub-triangle order
                    const double a = __shfl_sync(gmask, w, k, G), b = __shfl_sync(gmask, wx, k, G),
                                 c = __shfl_sync(gmask, wy, k, G);
                    sw = cadd(sw, a);
                    swx = cadd(swx, b);
                    swy = cadd(swy, c);
                }
                nq += (unsigned long long)m;
            }
            const double curx = cdiv(swx, sw), cury = cdiv(swy, sw);
            const double dx = csub(prevx, curx), dy = csub(prevy, cury);
            const double dist = sqrt(cadd(cmul(dx, dx), cmul(dy, dy)));
            prevx = curx;
            prevy = cury;
            if (dist < E) break;
        }
        if (gl == 0) {
            cell_update<MODE>(A, orig, px, py, h, prevx, prevy);
            if (MODE & M_COUNT) atomicAdd(&A.st->work[5], nq);
        }
    }
}

template <int MODE>
__global__ void __launch_bounds__(128, TM_OUT_MINB) k_output_t(CellArgs A, RingBuf R, int32_t *deep_list,
                                                               double2 *deep_xy, unsigned long long *deep_cnt) {
    const int64_t cell = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const int nv = cell < A.n_local ? (int)R.n[cell] : 0;
    const bool live = nv > 0;
    // rings are slot-major ([i][cell]): the loads of a warp for the same i coalesce
    const double2 *rv0 = R.v + cell;
    const int *rl0 = R.la + cell;
    const int64_t ns = A.n_local;
    auto RV = [&](int i) { return rv0[(int64_t)i * ns]; };
    auto RL = [&](int i) { return rl0[(int64_t)i * ns]; };
    int32_t orig = 0, gi = 0, nid = 0;
    double px = 0.0, py = 0.0, h = 0.0;
    if (live) {
        orig = __ldg(A.perm + cell);
        px = __ldg(A.xs + cell);
        py = __ldg(A.ys + cell);
        h = __ldg(A.hs + cell);
        gi = __ldg(A.gids + cell);
        nid = A.nbr_by_gid ? gi : orig;
        if (nid < 0 || (int64_t)nid >= A.nbr_keys) nid = -1;
    }
    if (live && A.nbr && nid >= 0) {
        int c = 0;
        for (int i = 0; i < nv; i++) {
            const int a = RL(i);
            if (a >= 0) A.nbr[(int64_t)nid * TM_NBR + c++] = A.nbr_by_gid ? __ldg(A.gids + a) : __ldg(A.perm + a);
        }
        A.nbr_cnt[nid] = (uint8_t)c;
    }
    int t_own = 0, ell = 0;
    unsigned keptmask = 0;
    if (live && (MODE & (M_TRI | M_ELL))) {
        unsigned keptall = 0;
        // keep-rule fast path (see interior_keeps_all): no wall line in the ring, and R from the
        // stored vertices with a 1e-9 margin (far above their error bound)
        bool all_in = true;
        double R2 = 0.0;
        for (int i = 0; i < nv; i++) {
            const double2 v = RV(i);
            R2 = fmax(R2, v.x * v.x + v.y * v.y);
            all_in = all_in && RL(i) >= 0;
        }
        all_in = all_in && interior_keeps_all_R(A, px, py, h, sqrt(R2) * (1.0 + 1e-9));
        for (int i = 0; i < nv; i++) {
            const int a = RL(i), b = RL(i + 1 == nv ? 0 : i + 1);
            if (a >= 0 && b >= 0) {
                const int32_t ga = __ldg(A.gids + a), gb = __ldg(A.gids + b);
                if (all_in) {
                    keptall |= 1u << i;
                    if (gi < ga && gi < gb) keptmask |= 1u << i;
                } else if (gi < ga && gi < gb) {
                    const int sv = ga < gb ? a : b, sw = ga < gb ? b : a;
                    const double2 v = RV(i);
                    if (keep_tri(A, (int)cell, sv, sw, v.x, v.y)) {
                        keptmask |= 1u << i;
                        keptall |= 1u << i;
                    }
                } else if (MODE & M_ELL) {
                    int s3[3] = {(int)cell, a, b};
                    int32_t g3[3] = {gi, ga, gb};
                    for (int u = 0; u < 2; u++)
                        for (int w = 0; w < 2 - u; w++)
                            if (g3[w] > g3[w + 1]) {
                                int32_t tg = g3[w]; g3[w] = g3[w + 1]; g3[w + 1] = tg;
                                int ts = s3[w]; s3[w] = s3[w + 1]; s3[w + 1] = ts;
                            }
                    const double uxx = __ldg(A.xs + s3[0]), uyy = __ldg(A.ys + s3[0]);
                    const Line B1 = bisector(csub(__ldg(A.xs + s3[1]), uxx), csub(__ldg(A.ys + s3[1]), uyy));
                    const Line B2 = bisector(csub(__ldg(A.xs + s3[2]), uxx), csub(__ldg(A.ys + s3[2]), uyy));
                    double ox, oy;
                    cramer(B1, B2, ox, oy);
                    if (keep_tri(A, s3[0], s3[1], s3[2], ox, oy)) keptall |= 1u << i;
                }
            }
        }
        if (!(MODE & M_TRI)) keptmask = 0;
        t_own = __popc(keptmask);
        if (MODE & M_ELL) {
            for (int i = 0; i < nv; i++) {
                const int a = RL(i);
                const int ip = i == 0 ? nv - 1 : i - 1;
                if (a >= 0 && (((keptall >> i) & 1u) || ((keptall >> ip) & 1u))) {
                    if (ell < A.adj_stride) A.adj[(int64_t)ell * A.n_local + cell] = a;
                    ell++;
                }
            }
            A.deg[cell] = (uint8_t)(ell < A.adj_stride ? ell : A.adj_stride);
            if (ell > A.adj_stride) atomicAdd(&A.st->n_adj_overflow, 1ull);
        }
    }
    if (MODE & M_TRI) {
        int incl = t_own;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int tt = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += tt;
        }
        const int tot = __shfl_sync(0xffffffffu, incl, 31);
        unsigned long long base = 0;
        if (lane == 31 && tot > 0) base = atomicAdd(A.n_tri, (unsigned long long)tot);
        base = __shfl_sync(0xffffffffu, base, 31) + (unsigned long long)(incl - t_own);
        for (unsigned m = keptmask; m; m &= m - 1) {
            const int i = __ffs(m) - 1;
            const int a = RL(i), b = RL(i + 1 == nv ? 0 : i + 1);
            if ((int64_t)base < A.tri_cap) {
                A.tri[3 * base] = gi;
                A.tri[3 * base + 1] = __ldg(A.gids + a);
                A.tri[3 * base + 2] = __ldg(A.gids + b);
            } else {
                atomicAdd(&A.st->n_tri_overflow, 1ull);
            }
            base++;
        }
    }
    unsigned long long nq = 0;
    if (live && (MODE & (M_TREAT | M_HAT))) {
        double cx, cy;
        // levels beyond TM_QLEV1: deferred to k_output_deep over a compacted list, so that the
        // few cells that refine deep do not hold their whole warp (lane divergence)
        unsigned long long nq1 = 0;
        const bool done = ring_centroid(rv0, ns, nv, px, py, h, A.d_prev ? __ldg(A.d_prev + orig) : -1.0, A, cx, cy,
                                        nq1, deep_list ? TM_QLEV1 : (1 << 30));
        nq += nq1;
        if (done) {
            cell_update<MODE>(A, orig, px, py, h, cx, cy);
        } else {
            const unsigned long long k = atomicAdd(deep_cnt, 1ull);
            deep_list[k] = (int32_t)cell;
            deep_xy[k] = make_double2(cx, cy);  // the level-TM_QLEV1 centroid
        }
    }    if ((MODE & M_COUNT) && live) {
        float R2f = 0.f;
        for (int i = 0; i < nv; i++) R2f = fmaxf(R2f, vertex_r2f_t(RV(i).x, RV(i).y, -1.0));
        const double rad = 2.0 * sqrt((double)R2f);
        const BinGeom &bg = A.bg;
        int ncert = 0;
        const int bxa = max(0, (int)floor((px - rad - bg.x0) * bg.isx));
        const int bxb = min(bg.nbx - 1, (int)floor((px + rad - bg.x0) * bg.isx));
        const int bya = max(0, (int)floor((py - rad - bg.y0) * bg.isy));
        const int byb = min(bg.nby - 1, (int)floor((py + rad - bg.y0) * bg.isy));
        for (int by = bya; by <= byb; by++) {
            const int s0 = __ldg(A.leaf_start + __ldg(A.leaf_off + by * bg.nbx + bxa));
            const int s1 = __ldg(A.leaf_start + __ldg(A.leaf_off + by * bg.nbx + bxb + 1));
            for (int s = s0; s < s1; s++) {
                const double dx = __ldg(A.xs + s) - px, dy = __ldg(A.ys + s) - py;
                ncert += (s != (int)cell) && (dx * dx + dy * dy < rad * rad);
            }
        }
        int degc = 0;
        for (int i = 0; i < nv; i++) degc += RL(i + 1 == nv ? 0 : i + 1) >= 0 ? 1 : 0;
        atomicAdd(&A.st->work[0], 1ull);
        atomicAdd(&A.st->work[1], (unsigned long long)ncert);
        atomicAdd(&A.st->work[2], (unsigned long long)degc);
        atomicAdd(&A.st->work[3], (unsigned long long)nv);
        atomicAdd(&A.st->work[4], (unsigned long long)t_own);
        atomicAdd(&A.st->work[5], (A.rho == nullptr) ? (unsigned long long)nv : nq);
        atomicAdd(&A.st->work[6], (unsigned long long)ell);
    }
}

}  // namespace

namespace tmg {

template <int MODE>
static tm_status launch_cells_thread_impl(tm_ctx *ctx, const CellArgs &a) {
    static bool attr_set = false;  // per instantiation
    constexpr size_t smem = (MODE & M_WCERT) ? TSMEM_W : TSMEM;
    if (!attr_set) {
        TM_CUDA_TRY(ctx, cudaFuncSetAttribute(k_cells_t<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr_set = true;
    }
    constexpr bool CSPLIT = split_rings(MODE);
    constexpr int OMODE = split_tris(MODE) ? (MODE & (M_TRI | M_ELL | M_TREAT | M_HAT)) : (MODE & (M_TREAT | M_HAT));
    RingBuf R = {};
    if (CSPLIT) {
        if (ctx->n_local > ctx->cap_ring) {
            cudaFree(ctx->ring_v); cudaFree(ctx->ring_la); cudaFree(ctx->ring_n);
            ctx->ring_v = ctx->ring_la = ctx->ring_n = nullptr;
            const int64_t c = ctx->n_local + ctx->n_local / 8 + 1024;
            TM_CUDA_TRY(ctx, cudaMalloc(&ctx->ring_v, c * VMAX * sizeof(double2)));
            TM_CUDA_TRY(ctx, cudaMalloc(&ctx->ring_la, c * VMAX * sizeof(int)));
            TM_CUDA_TRY(ctx, cudaMalloc(&ctx->ring_n, c * sizeof(uint8_t) + 64));
            ctx->cap_ring = c;
        }
        R.v = (double2 *)ctx->ring_v;
        R.la = (int *)ctx->ring_la;
        R.n = (uint8_t *)ctx->ring_n;
    }
    const unsigned blocks = (unsigned)((ctx->n_local + TB - 1) / TB);
    k_cells_t<MODE><<<blocks, TB, smem, ctx->stream>>>(a, ctx->retry_list, ctx->retry_cnt, R);
    tm_status s = tm_internal_check_launch(ctx, "k_cells_t");
    if (s != TM_OK || !CSPLIT) return s;
    CellArgs b = a;
    b.nbr = nullptr;  // the neighbour lists were written by k_cells_t
    const bool deep = b.rho != nullptr && (OMODE & (M_TREAT | M_HAT)) && !(ctx->p.flags & TM_F_NO_DEEP_PASS);
    if (deep) {
        if (!ctx->deep_cnt) TM_CUDA_TRY(ctx, cudaMalloc(&ctx->deep_cnt, sizeof(unsigned long long)));
        if (ctx->cap_deep < ctx->n_local) {
            cudaFree(ctx->deep_list);
            cudaFree(ctx->deep_xy);
            ctx->deep_list = nullptr;
            ctx->deep_xy = nullptr;
            ctx->cap_deep = 0;
            TM_CUDA_TRY(ctx, cudaMalloc(&ctx->deep_list, ctx->cap_ring * sizeof(int32_t)));
            TM_CUDA_TRY(ctx, cudaMalloc(&ctx->deep_xy, ctx->cap_ring * sizeof(double2)));
            ctx->cap_deep = ctx->cap_ring;
        }
        TM_CUDA_TRY(ctx, cudaMemsetAsync(ctx->deep_cnt, 0, sizeof(unsigned long long), ctx->stream));
    }
    k_output_t<OMODE><<<(unsigned)((ctx->n_local + 127) / 128), 128, 0, ctx->stream>>>(
        b, R, deep ? ctx->deep_list : nullptr, ctx->deep_xy, ctx->deep_cnt);
    s = tm_internal_check_launch(ctx, "k_output_t");
    if (s != TM_OK || !deep) return s;
    k_output_deep<OMODE, TM_DEEP_G><<<148 * 8, 128, 0, ctx->stream>>>(b, R, ctx->deep_list, ctx->deep_xy,
                                                                      ctx->deep_cnt);
    return tm_internal_check_launch(ctx, "k_output_deep");
}

// warm-started launches (neighbour lists of the previous launch on the same point set)
// certify the warm rings warp-cooperatively (M_WCERT); cold ones run the flat search
template <int MODE>
tm_status launch_cells_thread(tm_ctx *ctx, const CellArgs &a) {
    if (a.warm && !(ctx->p.flags & TM_F_NO_WCERT)) return launch_cells_thread_impl<MODE | M_WCERT>(ctx, a);
    return launch_cells_thread_impl<MODE>(ctx, a);
}

#define TM_INST(M) template tm_status launch_cells_thread<M>(tm_ctx *, const CellArgs &);
TM_INST(M_TRI) TM_INST(M_TRI | M_ELL) TM_INST(M_TRI | M_TREAT) TM_INST(M_TRI | M_ELL | M_TREAT) TM_INST(M_HAT)
TM_INST(M_TRI | M_COUNT) TM_INST(M_TRI | M_ELL | M_COUNT) TM_INST(M_TRI | M_TREAT | M_COUNT)
TM_INST(M_TRI | M_ELL | M_TREAT | M_COUNT) TM_INST(M_HAT | M_COUNT)
#undef TM_INST

}  // namespace tmg
