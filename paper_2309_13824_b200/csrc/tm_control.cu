// tm_control.cu -- NEXT-2 / NEXT-3 of SURVEY §8(f): the iterate-to-termination controller
// (thresholds Table B.1), its movement input (P:484-485,
// P:447), the point-addition scheme and the resolution update of the adaptive
// quantities.  Readings L43-L46.
#include <cuda_runtime.h>
#include <math.h>

#include <cub/cub.cuh>

#include "tm_internal.cuh"

using namespace tmg;

namespace {

// inner points (phi~(p_old) < -geps(p_old), P:410 / L38) whose move d_prev is not below
// T_end = fac_end_mvmt * h(p_old); integer count, warp-aggregated atomics (exact)
__global__ void k_move_count(int64_t n, const double *__restrict__ xo, const double *__restrict__ yo,
                             const double *__restrict__ dp, Grid g, const double *__restrict__ phi,
                             const double *__restrict__ mu, double c, double h_avg, double fac_geps, double fac_end,
                             unsigned long long *__restrict__ count) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool big = false;
    if (i < n) {
        const double x = xo[i], y = yo[i];
        const double h = mu ? cmul(c, bilinear(g, mu, x, y, LdgLoad())) : c;
        const double geps = cmul(fac_geps, h < h_avg ? h : h_avg);
        const double ph = bilinear(g, phi, x, y, LdgLoad());
        big = ph < -geps && !(dp[i] < cmul(fac_end, h));
    }
    const unsigned b = __ballot_sync(0xffffffffu, big);
    if ((threadIdx.x & 31) == 0 && b) atomicAdd(count, (unsigned long long)__popc(b));
}

// point addition keys: per triangle {u < v < w} (caller indices), the ratio R_circ / h(g) (the
// canonical circumcentre of the keep rule, R = |c - p_u|, g = ((p_u + p_v) + p_w) / 3, h = c mu~(g)),
// as a descending-order key, and the (u, v) tie key; operations as the oracle's
__global__ void k_pa_keys(int64_t nt, const int32_t *__restrict__ tri, const double *__restrict__ x,
                          const double *__restrict__ y, Grid g, const double *__restrict__ mu, double c,
                          unsigned long long *__restrict__ kr, unsigned long long *__restrict__ kuv,
                          int32_t *__restrict__ idx, double *__restrict__ gxy) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nt) return;
    int32_t q0 = tri[3 * t], q1 = tri[3 * t + 1], q2 = tri[3 * t + 2], s;
    if (q0 > q1) { s = q0; q0 = q1; q1 = s; }
    if (q1 > q2) { s = q1; q1 = q2; q2 = s; }
    if (q0 > q1) { s = q0; q0 = q1; q1 = s; }
    const double xu = x[q0], yu = y[q0], xv = x[q1], yv = y[q1], xw = x[q2], yw = y[q2];
    const Line A = bisector(csub(xv, xu), csub(yv, yu)), B = bisector(csub(xw, xu), csub(yw, yu));
    double ox, oy;
    cramer(A, B, ox, oy);
    const double R = sqrt(cadd(cmul(ox, ox), cmul(oy, oy)));
    const double gx = cdiv(cadd(cadd(xu, xv), xw), 3.0), gy = cdiv(cadd(cadd(yu, yv), yw), 3.0);
    const double h = mu ? cmul(c, bilinear(g, mu, gx, gy, LdgLoad())) : c;
    const double r = cdiv(R, h);
    // r >= 0 (finite or +inf): its bits order like unsigned integers; descending = complement
    kr[t] = ~(unsigned long long)__double_as_longlong(r);
    kuv[t] = ((unsigned long long)(uint32_t)q0 << 32) | (uint32_t)q1;
    idx[t] = (int32_t)t;
    gxy[2 * t] = gx;
    gxy[2 * t + 1] = gy;
}

__global__ void k_pa_gather_uv(int64_t k, const int32_t *__restrict__ idx, const unsigned long long *__restrict__ kuv,
                               unsigned long long *__restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < k) out[i] = kuv[idx[i]];
}

__global__ void k_pa_write(int64_t k, const int32_t *__restrict__ idx, const double *__restrict__ gxy,
                           double *__restrict__ xn, double *__restrict__ yn) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= k) return;
    const int32_t t = idx[i];
    xn[i] = gxy[2 * t];
    yn[i] = gxy[2 * t + 1];
}

struct DevBuf {  // scratch owned by one call
    void *p = nullptr;
    ~DevBuf() { cudaFree(p); }
};

}  // namespace

extern "C" tm_status tm_move_count(tm_ctx *ctx, const double *x_old, const double *y_old, const double *d_prev,
                                   int64_t n, int64_t *d_count) {
    if (!ctx) return TM_E_ARG;
    if (!ctx->have_domain) TM_FAIL(ctx, TM_E_STATE, "tm_move_count before tm_set_domain");
    if (!x_old || !y_old || !d_prev || !d_count || n < 0) TM_FAIL(ctx, TM_E_ARG, "bad arguments to tm_move_count");
    TM_CUDA_TRY(ctx, cudaMemsetAsync(d_count, 0, sizeof(int64_t), ctx->stream));
    if (n == 0) return TM_OK;
    k_move_count<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(
        n, x_old, y_old, d_prev, ctx->grid, ctx->phi, ctx->mu, ctx->c, ctx->h_avg, ctx->p.fac_geps,
        ctx->p.fac_end_mvmt, reinterpret_cast<unsigned long long *>(d_count));
    return tm_internal_check_launch(ctx, "k_move_count");
}

extern "C" tm_status tm_set_n_total(tm_ctx *ctx, int64_t n_total, double *c_out, double *h_avg_out) {
    if (!ctx) return TM_E_ARG;
    if (!ctx->have_domain) TM_FAIL(ctx, TM_E_STATE, "tm_set_n_total before tm_set_domain");
    if (ctx->capturing) TM_FAIL(ctx, TM_E_STATE, "tm_set_n_total while capturing a graph");
    if (n_total < 1) TM_FAIL(ctx, TM_E_ARG, "n_total %lld", (long long)n_total);
    tm_internal_set_n_total(ctx, n_total);
    if (c_out) *c_out = ctx->c;
    if (h_avg_out) *h_avg_out = ctx->h_avg;
    return TM_OK;
}

extern "C" tm_status tm_point_addition(tm_ctx *ctx, const int32_t *tri, int64_t n_tri, const double *x,
                                       const double *y, int64_t n_add, double *x_new, double *y_new,
                                       double *ratio_min) {
    if (!ctx) return TM_E_ARG;
    if (!ctx->have_domain) TM_FAIL(ctx, TM_E_STATE, "tm_point_addition before tm_set_domain");
    if (ctx->capturing) TM_FAIL(ctx, TM_E_STATE, "tm_point_addition while capturing a graph");
    if (n_tri < 0 || n_add < 0 || n_add > n_tri || (n_tri > 0 && (!tri || !x || !y)) || (n_add > 0 && (!x_new || !y_new)) ||
        n_tri >= (int64_t)INT32_MAX)
        TM_FAIL(ctx, TM_E_ARG, "bad arguments to tm_point_addition (n_tri %lld, n_add %lld)", (long long)n_tri,
                (long long)n_add);
    if (ratio_min) *ratio_min = 0.0;
    if (n_add == 0) return TM_OK;
    TM_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
    const int nt = (int)n_tri, k = (int)n_add;
    DevBuf b_kr, b_kr2, b_kuv, b_kuv2, b_idx, b_idx2, b_gxy, b_tmp;
    TM_CUDA_TRY(ctx, cudaMalloc(&b_kr.p, (size_t)nt * 8));
    TM_CUDA_TRY(ctx, cudaMalloc(&b_kr2.p, (size_t)nt * 8));
    TM_CUDA_TRY(ctx, cudaMalloc(&b_kuv.p, (size_t)nt * 8));
    TM_CUDA_TRY(ctx, cudaMalloc(&b_kuv2.p, (size_t)nt * 8));
    TM_CUDA_TRY(ctx, cudaMalloc(&b_idx.p, (size_t)nt * 4));
    TM_CUDA_TRY(ctx, cudaMalloc(&b_idx2.p, (size_t)nt * 4));
    TM_CUDA_TRY(ctx, cudaMalloc(&b_gxy.p, (size_t)nt * 16));
    auto *kr = (unsigned long long *)b_kr.p, *kr2 = (unsigned long long *)b_kr2.p;
    auto *kuv = (unsigned long long *)b_kuv.p, *kuv2 = (unsigned long long *)b_kuv2.p;
    auto *idx = (int32_t *)b_idx.p, *idx2 = (int32_t *)b_idx2.p;
    auto *gxy = (double *)b_gxy.p;
    k_pa_keys<<<(unsigned)((nt + 255) / 256), 256, 0, ctx->stream>>>(nt, tri, x, y, ctx->grid, ctx->mu, ctx->c, kr, kuv,
                                                                   idx, gxy);
    tm_status s = tm_internal_check_launch(ctx, "k_pa_keys");
    if (s != TM_OK) return s;
    // (1) canonical order of the triangles by (u, v) -- unique per triangle (a directed edge
    // belongs to one triangle), so the result does not depend on the emission order;
    // (2) stable sort by the ratio, descending (ties keep the (u, v) order);
    // (3) the first k by (u, v) again: the order the new points are written in
    size_t need = 0, n2 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, need, kuv, kuv2, idx, idx2, nt, 0, 64, ctx->stream);
    cub::DeviceRadixSort::SortPairs(nullptr, n2, kr, kr2, idx, idx2, nt, 0, 64, ctx->stream);
    need = need > n2 ? need : n2;
    TM_CUDA_TRY(ctx, cudaMalloc(&b_tmp.p, need + 16));
    TM_CUDA_TRY(ctx, cub::DeviceRadixSort::SortPairs(b_tmp.p, need, kuv, kuv2, idx, idx2, nt, 0, 64, ctx->stream));
    // ratio keys in the canonical order
    k_pa_gather_uv<<<(unsigned)((nt + 255) / 256), 256, 0, ctx->stream>>>(nt, idx2, kr, kr2);
    TM_CUDA_TRY(ctx, cub::DeviceRadixSort::SortPairs(b_tmp.p, need, kr2, kr, idx2, idx, nt, 0, 64, ctx->stream));
    // idx[0..k) = the selected triangles; kr[k-1] = the smallest selected ratio (complemented)
    unsigned long long klast = 0;
    TM_CUDA_TRY(ctx, cudaMemcpyAsync(&klast, kr + (k - 1), 8, cudaMemcpyDeviceToHost, ctx->stream));
    k_pa_gather_uv<<<(unsigned)((k + 255) / 256), 256, 0, ctx->stream>>>(k, idx, kuv, kr2);
    TM_CUDA_TRY(ctx, cub::DeviceRadixSort::SortPairs(b_tmp.p, need, kr2, kuv2, idx, idx2, k, 0, 64, ctx->stream));
    k_pa_write<<<(unsigned)((k + 255) / 256), 256, 0, ctx->stream>>>(k, idx2, gxy, x_new, y_new);
    if ((s = tm_internal_check_launch(ctx, "k_pa_write")) != TM_OK) return s;
    TM_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));  // the scratch is freed on return
    if (ratio_min) {
        const unsigned long long bits = ~klast;
        memcpy(ratio_min, &bits, sizeof(double));
    }
    return TM_OK;
}

// ---- the controller (host) ----------------------------------------
extern "C" void tm_control_init(tm_control *c, int64_t n_total, int64_t n_current, int32_t method) {
    memset(c, 0, sizeof(*c));
    c->n_total = n_total;
    c->n_current = n_current;
    c->method = method;
    c->mode = method == TM_METHOD_CVD ? TM_METHOD_CVD : TM_METHOD_DISTMESH;
    c->t_add_quality = 0.002;
    c->fac_add = 0.6;
    c->t_end_quality = 0.001;
    c->t_end_alpha_max = 0.005;
    c->t_switch_quality = 0.0015;
    c->max_iterations = 1000;     // safety cap (paper silent)
}

static double rel_change(double a, double b) { return fabs(a - b) / b; }

extern "C" int32_t tm_control_update(tm_control *c, const tm_stats *s, int64_t move_count, int64_t *n_add) {
    if (n_add) *n_add = 0;
    const double n = (double)s->n_tri;
    const double ma = s->sum_sqrt_alpha / n, mb = s->sum_sqrt_beta / n;
    const double cur[3] = {ma * ma, mb * mb, s->max_alpha};  // Eq. 1/2-mean
    double prev[3] = {c->prev[0], c->prev[1], c->prev[2]};
    const int had = c->have_prev;
    c->prev[0] = cur[0];
    c->prev[1] = cur[1];
    c->prev[2] = cur[2];
    c->have_prev = 1;
    c->iterations++;
    if (c->iterations >= c->max_iterations) return TM_ACT_TERMINATE_CAP;
    if (c->n_current < c->n_total) {
        if (had && rel_change(cur[0], prev[0]) < c->t_add_quality && rel_change(cur[1], prev[1]) < c->t_add_quality) {
            int64_t k = (int64_t)floor(c->fac_add * (double)c->n_current);
            if (k > c->n_total - c->n_current) k = c->n_total - c->n_current;
            c->n_current += k;
            c->have_prev = 0;  // the history restarts at the new resolution
            if (n_add) *n_add = k;
            return TM_ACT_ADD;
        }
        return TM_ACT_CONTINUE;
    }
    if (c->method == TM_METHOD_HYBRID && c->mode == TM_METHOD_DISTMESH) {
        if (had && rel_change(cur[0], prev[0]) < c->t_switch_quality) {
            c->mode = TM_METHOD_CVD;
            return TM_ACT_SWITCH;
        }
        return TM_ACT_CONTINUE;
    }
    if (move_count == 0) return TM_ACT_TERMINATE_MOVES;
    if (had && rel_change(cur[0], prev[0]) < c->t_end_quality && rel_change(cur[1], prev[1]) < c->t_end_quality &&
        rel_change(cur[2], prev[2]) < c->t_end_alpha_max)
        return TM_ACT_TERMINATE_QUALITY;
    return TM_ACT_CONTINUE;
}
