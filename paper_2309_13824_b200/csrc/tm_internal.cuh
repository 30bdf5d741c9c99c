// tm_internal.cuh -- context layout and kernel argument blocks shared by the
// .cu files of libtrime_gpu.so.  Not part of the public ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "../../include/trime_gpu.h"
#include "tm_common.cuh"

namespace tmg {

constexpr int TM_NBR = 12;  // warm-start neighbours kept per point (= thread-kernel slot capacity)

// device-resident health counters and work counters (one per context)
struct DevState {
    unsigned long long n_degenerate;   // exact zeros + inconsistent clips
    unsigned long long n_overflow;     // cells over the vertex capacity
    unsigned long long n_duplicate;    // bitwise-equal point pairs met
    unsigned long long n_outside;      // points outside B / NaN
    unsigned long long n_tri_overflow; // triangles beyond tri_cap
    unsigned long long n_adj_overflow; // ELL rows beyond adj_stride
    unsigned long long n_fallback;     // projection fallbacks
    unsigned long long n_strip_overflow; // strip messages / appends beyond their capacity
    unsigned long long work[11];       // tm_work fields n_cells .. exact_calls, then warp_trips
};

struct BinGeom {
    int32_t nbx, nby;
    double x0, y0;   // bin grid origin (= box origin)
    double sx, sy;   // level-0 bin size
    double isx, isy; // 1/size
};

// Two-level cell list: level-0 bin b (row-major) holds 4^rlev[b] leaves in
// Morton order; leaf_start is indexed by leaf_off[b] + morton index.
constexpr int MAX_SUBLEVEL = 5;

__host__ __device__ __forceinline__ uint32_t part1by1(uint32_t v) {
    v &= 0x0000ffffu;
    v = (v | (v << 8)) & 0x00ff00ffu;
    v = (v | (v << 4)) & 0x0f0f0f0fu;
    v = (v | (v << 2)) & 0x33333333u;
    v = (v | (v << 1)) & 0x55555555u;
    return v;
}
__host__ __device__ __forceinline__ uint32_t morton2(uint32_t x, uint32_t y) { return part1by1(x) | (part1by1(y) << 1); }

// 2^-r for 0 <= r <= MAX_SUBLEVEL, exactly: leaf sizes bg.sx * 2^-r are the same bits as
// bg.sx / 2^r (scaling by a power of two is exact), without a DP division
__host__ __device__ __forceinline__ double pow2neg(int r) {
#if defined(__CUDA_ARCH__)
    return __longlong_as_double((long long)(1023 - r) << 52);
#else
    return 1.0 / (double)(1 << r);
#endif
}

// leaf coordinate of x at depth r (consistent between binning and search):
// floor((x-x0)*isx*2^r) clamped into the level-0 bin floor((x-x0)*isx)
__device__ __forceinline__ int leaf_coord(double x, double x0, double is, int nb, int r) {
    int b = (int)floor((x - x0) * is);
    b = b < 0 ? 0 : (b >= nb ? nb - 1 : b);
    int u = (int)floor((x - x0) * is * (double)(1 << r));
    int lo = b << r, hi = ((b + 1) << r) - 1;
    return u < lo ? lo : (u > hi ? hi : u);
}

// everything a cell kernel reads or writes
struct CellArgs {
    const double *xs, *ys, *hs;
    const int32_t *perm, *gids;
    const int32_t *inv_perm;   // point id -> sorted slot (this binning; stale for absent gids)
    int32_t *nbr;              // warm start: per caller index, the cell's neighbours (caller ids) of the
    uint8_t *nbr_cnt;          //   last cell launch on the same point set; nbr_cnt[i] entries (<= TM_NBR)
    int32_t warm;              // 1: read nbr/nbr_cnt before the search (they are written back either way)
    int32_t nbr_by_gid;        // ids are gids (strips), else caller indices
    int64_t nbr_keys;          // size of the id space (n_total with gids, else n_local)
    const uint8_t *rlev;
    const int32_t *leaf_off, *leaf_start;
    BinGeom bg;
    int64_t n_local, n_owned;  // capacity (array stride) and owned bound; the live counts are
    const int64_t *dcnt;       // device {n_owned, n_local} when binned by tm_grid_bin_dc, else NULL
    Grid grid;
    const double *phi, *mu, *rho;
    const double4 *rho4;     // rho's grid cells with their 4 corners packed (f00, f10, f01, f11), or NULL
    double c, h_avg;
    double lip_mu, lip_phi;  // Lipschitz constants of mu~ and phi~ (0 for uniform mu)
    double fac_voro, fac_pt, fac_geps, fac_end, damping, keep_tol;
    int32_t newton_max, quad_max;
    int32_t projection, trace_max;  // treatment scheme (NEXT-1), see treat_point
    int32_t validity;               // keep rule: 0 Test 1 (L10), 1 the paper's Tests 1-3 (NEXT-2)
    double t_circ;
    // outputs
    int32_t *tri;
    int64_t tri_cap;
    unsigned long long *n_tri;
    int32_t *adj;
    uint8_t *deg;
    int32_t adj_stride;
    const double *d_prev;
    double *x_out, *y_out, *d_prev_out;
    int8_t *status;
    double *x_hat, *y_hat;
    DevState *st;
};

}  // namespace tmg

struct tm_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    tm_params p;
    char err[512] = {0};
    // domain (S0)
    bool have_domain = false;
    tmg::Grid grid;
    double c = 0, h_avg = 0;
    double dom_sums[3] = {0, 0, 0};  // S0 sums: sum mu~^-2, sum mu~, count over the inside cells
    double lip_mu = 0;  // Lipschitz constant of mu~ (0 for uniform sizing): adaptive halo widths
    double lip_phi = 0; // Lipschitz constant of phi~ (keep-rule fast path)
    int64_t n_total = 0;
    double *phi = nullptr, *mu = nullptr, *rho = nullptr;
    double4 *rho4 = nullptr;  // packed corners of rho (S0, one sector per bilinear lookup)
    size_t grid_bytes = 0;
    tmg::BinGeom bg;
    // sorted state (S1)
    bool have_bins = false;
    int64_t n_local = 0, n_owned = 0, cap_points = 0, cap_bins = 0;
    double *xs = nullptr, *ys = nullptr, *hs = nullptr;
    int32_t *perm = nullptr, *gids = nullptr, *key = nullptr, *rank = nullptr;
    // warm start of the cell search (previous iteration's neighbours, caller ids; single domain only)
    int32_t *nbr = nullptr;
    uint8_t *nbr_cnt = nullptr;
    int32_t *inv_id = nullptr;  // point id -> slot of the last binning
    int64_t cap_nbr = 0, nbr_n = -1;
    bool have_gid = false;
    int32_t *bin_count = nullptr, *block_sums = nullptr;
    uint8_t *rlev = nullptr;
    int32_t *leaf_off = nullptr, *leaf_count = nullptr, *leaf_start = nullptr;
    int64_t cap_block_sums = 0, cap_leaves = 0;
    // DistMesh scratch
    double *partials = nullptr;
    int64_t cap_partials = 0;
    // stats scratch
    double *stat_acc = nullptr;
    // cells of the 16-lane pass that need the 32-lane retry pass
    int32_t *retry_list = nullptr;
    unsigned long long *retry_cnt = nullptr;
    int64_t cap_retry = 0;
    // CVD split: stored rings (slot-major, see tm_cells_t.cu RingBuf)
    void *ring_v = nullptr, *ring_la = nullptr, *ring_n = nullptr;
    int64_t cap_ring = 0;
    // cells whose adaptive quadrature goes deeper than k_output_t's levels (k_output_deep)
    int32_t *deep_list = nullptr;
    double2 *deep_xy = nullptr;  // their level-TM_QLEV1 centroid (k_output_deep continues from it)
    unsigned long long *deep_cnt = nullptr;
    int64_t cap_deep = 0;
    // strip migration scratch (stable partition)
    double *mig_keep = nullptr;
    int32_t *mig_cnt = nullptr, *mig_off = nullptr;
    int64_t cap_mig = 0, cap_mig_blk = 0;
    // device health counters
    tmg::DevState *dst = nullptr;
    bool have_cells = false;
    const int64_t *dcnt = nullptr;  // device {n_owned, n_local} of the last tm_grid_bin_dc, else NULL
    bool capturing = false;         // tm_graph_begin .. tm_graph_end
    const int32_t *gids_in = nullptr;  // the caller's gid array of the last tm_grid_bin (or NULL)
    // positions and h of the last triangulation with adjacency (lazy re-triangulation, NEXT-1)
    double *xs_tria = nullptr, *ys_tria = nullptr, *hs_tria = nullptr;
    int64_t cap_tria = 0;
    bool have_tria = false;
    int64_t *scratch_n = nullptr;   // device scratch count (migration source size)
    // ADF quadtrees on the boundary geometry cells (NEXT-4, tm_setup.cu)
    void *adf_nodes = nullptr;      // AdfNode pool
    int32_t *adf_root = nullptr;    // per geometry cell: root node or -1
    int64_t adf_cap = 0, adf_n = 0;
    int32_t adf_nxg = 0, adf_nyg = 0;
};

#define TM_CUDA_TRY(ctx, call)                                                                       \
    do {                                                                                             \
        cudaError_t e_ = (call);                                                                     \
        if (e_ != cudaSuccess) {                                                                     \
            snprintf((ctx)->err, sizeof((ctx)->err), "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                     __FILE__, __LINE__);                                                            \
            return TM_E_CUDA;                                                                        \
        }                                                                                            \
    } while (0)

#define TM_FAIL(ctx, code, ...)                                   \
    do {                                                          \
        snprintf((ctx)->err, sizeof((ctx)->err), __VA_ARGS__);    \
        return (code);                                            \
    } while (0)

// live counts of the binned point set: host values, or device ones (tm_grid_bin_dc: the
// multi-GPU strip path learns its ghost and migrant counts on the device, no host sync)
__device__ __forceinline__ int64_t live_local(const tmg::CellArgs &A) { return A.dcnt ? __ldg(A.dcnt + 1) : A.n_local; }
__device__ __forceinline__ int64_t live_owned(const tmg::CellArgs &A) { return A.dcnt ? __ldg(A.dcnt) : A.n_owned; }

// internal helpers implemented in tm_api.cu
tm_status tm_internal_fill_cell_args(tm_ctx *ctx, tmg::CellArgs *a);
tm_status tm_internal_check_launch(tm_ctx *ctx, const char *what);
void tm_internal_set_n_total(tm_ctx *ctx, int64_t n_total);

namespace tmg {

// NEXT-1: the paper's projection of escaped points (Fig. 13), the same operations
// in the same order as the oracle (canonical, uncontracted: identical bits).
// Sphere tracing from the inner p_old toward p_new: q <- q + |phi~(q)| u, a step never
// passing p_new, until |phi~(q)| <= geps, at most trace_max steps (L39).
// results by value (a reference output would take the caller's variables' addresses: a local-memory
// frame in every kernel that can reach the treatment, projection used or not)
struct ProjResult {
    double x, y;
    bool ok;
};

template <typename Load>
__device__ __forceinline__ ProjResult sphere_trace(const Grid &g, const double *phi, double xo, double yo, double xn,
                                                double yn, double geps, int trace_max, Load ld) {
    const double dx = csub(xn, xo), dy = csub(yn, yo);
    const double len = sqrt(cadd(cmul(dx, dx), cmul(dy, dy)));
    const double ux = cdiv(dx, len), uy = cdiv(dy, len);
    double qx = xo, qy = yo, s = 0.0;
    for (int k = 0; k < trace_max; k++) {
        const double v = bilinear(g, phi, qx, qy, ld);
        if (fabs(v) <= geps) return ProjResult{qx, qy, true};
        double r = fabs(v);
        if (cadd(s, r) > len) r = csub(len, s);
        s = cadd(s, r);
        qx = cadd(qx, cmul(r, ux));
        qy = cadd(qy, cmul(r, uy));
    }
    return ProjResult{qx, qy, fabs(bilinear(g, phi, qx, qy, ld)) <= geps};
}

// Damped Newton projection: L(p) = [phi~(p), (p - p_new) x grad phi~(p)] = 0 from
// p_new, the Jacobian of Eq. projection_Newton_Jacobian with central finite differences of step
// deps (L36, L41), p <- p - alpha J^-1 L clamped into B, until |phi~| <= geps.
template <typename Load>
__device__ __forceinline__ ProjResult newton_project(const Grid &g, const double *phi, double xn, double yn, double geps,
                                                  double deps, double damping, int newton_max, Load ld) {
    double x = xn, y = yn;
    bool ok = false;
    for (int k = 0; k < newton_max; k++) {
        const double d = deps;
        const double f0 = bilinear(g, phi, x, y, ld);
        const double xp = cadd(x, d), xm = csub(x, d), yp = cadd(y, d), ym = csub(y, d);
        const double fxp = bilinear(g, phi, xp, y, ld), fxm = bilinear(g, phi, xm, y, ld);
        const double fyp = bilinear(g, phi, x, yp, ld), fym = bilinear(g, phi, x, ym, ld);
        const double fpp = bilinear(g, phi, xp, yp, ld), fpm = bilinear(g, phi, xp, ym, ld);
        const double fmp = bilinear(g, phi, xm, yp, ld), fmm = bilinear(g, phi, xm, ym, ld);
        const double fx = cdiv(csub(fxp, fxm), cmul(2.0, d)), fy = cdiv(csub(fyp, fym), cmul(2.0, d));
        const double dd = cmul(d, d);
        const double fxx = cdiv(cadd(csub(fxp, cmul(2.0, f0)), fxm), dd);
        const double fyy = cdiv(cadd(csub(fyp, cmul(2.0, f0)), fym), dd);
        const double fxy = cdiv(cadd(csub(csub(fpp, fpm), fmp), fmm), cmul(cmul(4.0, d), d));
        const double L1 = f0;
        const double ex = csub(x, xn), ey = csub(y, yn);
        const double L2 = csub(cmul(ex, fy), cmul(ey, fx));
        const double J11 = fx, J12 = fy;
        const double J21 = csub(cadd(fy, cmul(ex, fxy)), cmul(ey, fxx));
        const double J22 = cadd(csub(-fx, cmul(ey, fxy)), cmul(ex, fyy));
        const double det = csub(cmul(J11, J22), cmul(J12, J21));
        if (!(det != 0.0)) break;
        const double sx = cdiv(csub(cmul(L1, J22), cmul(J12, L2)), det);
        const double sy = cdiv(csub(cmul(J11, L2), cmul(J21, L1)), det);
        const double nx = csub(x, cmul(damping, sx)), ny = csub(y, cmul(damping, sy));
        x = nx < g.x0 ? g.x0 : (nx > g.x1 ? g.x1 : nx);
        y = ny < g.y0 ? g.y0 : (ny > g.y1 ? g.y1 : ny);
        if (fabs(bilinear(g, phi, x, y, ld)) <= geps) {
            ok = true;
            break;
        }
    }
    return ProjResult{x, y, ok};
}

// S5 treatment of one point (L20-L22); returns status.
// projection 0: the L22 reading (1-D gradient Newton from p_new); 1: the paper's Fig. 13
// (sphere tracing from an inner p_old, status + 8; 2x2 FD Newton from a boundary p_old).
template <typename Load>
__device__ __forceinline__ int treat_point(const Grid &g, const double *phi, double h, double h_avg,
                                           double fac_pt, double fac_geps, double damping, int newton_max,
                                           double xo, double yo, double xh, double yh, double &qx_out,
                                           double &qy_out, double &dprev, Load ld, int projection = 0,
                                           int trace_max = 64) {
    int status = 0;
    double T = cmul(fac_pt, h);
    double dx = csub(xh, xo), dy = csub(yh, yo);
    double len = sqrt(cadd(cmul(dx, dx), cmul(dy, dy)));
    if (len > T) {
        double sc = cdiv(T, len);
        dx = cmul(dx, sc);
        dy = cmul(dy, sc);
        status |= 4;
    }
    double qx = fmin(fmax(cadd(xo, dx), g.x0), g.x1);
    double qy = fmin(fmax(cadd(yo, dy), g.y0), g.y1);
    const double hm = h < h_avg ? h : h_avg;
    double geps = cmul(fac_geps, hm);
    double ph = bilinear(g, phi, qx, qy, ld);
    if (!(ph <= geps) && projection == 1) {
        const double po = bilinear(g, phi, xo, yo, ld);
        ProjResult r;
        if (po < -geps) {
            r = sphere_trace(g, phi, xo, yo, qx, qy, geps, trace_max, ld);
            status |= 8;
        } else {
            r = newton_project(g, phi, qx, qy, geps, cmul(1.4901161193847656e-08, hm), damping, newton_max, ld);
        }
        const bool ok = r.ok;
        if (ok) {
            qx = r.x;
            qy = r.y;
            status |= 1;
        } else {
            qx = xo;
            qy = yo;
            status = (status & 4) | 2;
        }
    } else if (!(ph <= geps)) {
        bool ok = false;
        for (int it = 0; it < newton_max; it++) {
            double gx, gy;
            bilinear_grad(g, phi, qx, qy, gx, gy, ld);
            double g2 = cadd(cmul(gx, gx), cmul(gy, gy));
            if (!(g2 > 0.0)) break;
            double stp = cdiv(cmul(damping, ph), g2);
            qx = fmin(fmax(csub(qx, cmul(stp, gx)), g.x0), g.x1);
            qy = fmin(fmax(csub(qy, cmul(stp, gy)), g.y0), g.y1);
            ph = bilinear(g, phi, qx, qy, ld);
            if (fabs(ph) <= geps) {
                ok = true;
                break;
            }
        }
        if (ok)
            status |= 1;
        else {
            qx = xo;
            qy = yo;
            status = (status & 4) | 2;
        }
    }
    qx_out = qx;
    qy_out = qy;
    double ex = csub(qx, xo), ey = csub(qy, yo);
    dprev = sqrt(cadd(cmul(ex, ex), cmul(ey, ey)));
    return status;
}

}  // namespace tmg
