// tm_api.cu -- context, S0 domain, S1 binning, S5 standalone treatment, S6
// statistics, S7 halo/migration packing and host-side hooks of libtrime_gpu.so.
#include <cuda_runtime.h>
#include <math.h>
#include <stddef.h>
#include <stdlib.h>

#include <algorithm>
#include <new>

#include "tm_internal.cuh"

using namespace tmg;

// ============================================================================ params / ctx
extern "C" void tm_params_default(tm_params *p) {
    p->n_opt = 6.0;            // P:1077 gives 3.3 for Voro++; 6 suits the GPU cell search
    p->fac_voro_bound = 5.0;
    p->fac_pt_mvmt = 0.4;
    p->fac_geps = 0.01;
    p->fac_end_mvmt = 0.001;
    p->newton_damping = 1.0;
    p->newton_max = 10;
    p->quad_max_level = 10;    // L13
    p->fscale = 1.2;
    p->dt_k = 0.2;             // L3
    p->keep_tol = 0.0;         // L10
    p->adj_stride = 16;
    p->max_cell_vertices = 32;
    p->flags = TM_F_TWO_LEVEL_BINS;
    p->projection = 0;         // L22 (north_star "gradient projection"); 1 = the paper's Fig. 13
    p->trace_max = 64;         // L39
    p->fac_retria = 0.1;
    p->validity = 0;           // L10 (north_star Test 1); 1 = the paper's Tests 1-3 (NEXT-2)
    p->t_circ = 0.4;
}

extern "C" tm_status tm_create(int device, void *cuda_stream, const tm_params *p, tm_ctx **out) {
    if (!out) return TM_E_ARG;
    *out = nullptr;
    tm_ctx *ctx = new (std::nothrow) tm_ctx();
    if (!ctx) return TM_E_ARG;
    ctx->device = device;
    ctx->stream = (cudaStream_t)cuda_stream;
    if (p)
        ctx->p = *p;
    else
        tm_params_default(&ctx->p);
    if (ctx->p.max_cell_vertices != 32 || ctx->p.adj_stride < 1 || ctx->p.adj_stride > 255 ||
        ctx->p.quad_max_level < 1 || ctx->p.quad_max_level > 20 || ctx->p.newton_max < 0 ||
        (ctx->p.projection != 0 && ctx->p.projection != 1) || ctx->p.trace_max < 0) {
        delete ctx;
        return TM_E_ARG;
    }
    if (cudaSetDevice(device) != cudaSuccess || cudaMalloc(&ctx->dst, sizeof(DevState)) != cudaSuccess ||
        cudaMalloc(&ctx->stat_acc, 16 * sizeof(double)) != cudaSuccess ||
        cudaMemsetAsync(ctx->dst, 0, sizeof(DevState), ctx->stream) != cudaSuccess) {
        cudaGetLastError();
        delete ctx;
        return TM_E_CUDA;
    }
    *out = ctx;
    return TM_OK;
}

static void free_points(tm_ctx *c) {
    cudaFree(c->xs); cudaFree(c->ys); cudaFree(c->hs);
    cudaFree(c->perm); cudaFree(c->gids); cudaFree(c->key); cudaFree(c->rank);
    c->xs = c->ys = c->hs = nullptr;
    c->perm = c->gids = c->key = c->rank = nullptr;
    c->cap_points = 0;
}

extern "C" void tm_destroy(tm_ctx *ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    free_points(ctx);
    cudaFree(ctx->bin_count); cudaFree(ctx->rlev); cudaFree(ctx->leaf_off); cudaFree(ctx->block_sums);
    cudaFree(ctx->leaf_count); cudaFree(ctx->leaf_start);
    cudaFree(ctx->phi); cudaFree(ctx->mu); cudaFree(ctx->rho); cudaFree(ctx->rho4);
    cudaFree(ctx->partials); cudaFree(ctx->stat_acc); cudaFree(ctx->dst);
    cudaFree(ctx->retry_list); cudaFree(ctx->retry_cnt);
    cudaFree(ctx->mig_keep); cudaFree(ctx->mig_cnt); cudaFree(ctx->mig_off);
    cudaFree(ctx->nbr); cudaFree(ctx->nbr_cnt); cudaFree(ctx->inv_id);
    cudaFree(ctx->ring_v); cudaFree(ctx->ring_la); cudaFree(ctx->ring_n);
    cudaFree(ctx->deep_list); cudaFree(ctx->deep_xy); cudaFree(ctx->deep_cnt); cudaFree(ctx->scratch_n);
    cudaFree(ctx->xs_tria); cudaFree(ctx->ys_tria); cudaFree(ctx->hs_tria);
    cudaFree(ctx->adf_nodes); cudaFree(ctx->adf_root);
    delete ctx;
}

extern "C" const char *tm_last_error(const tm_ctx *ctx) { return ctx ? ctx->err : "null context"; }

tm_status tm_internal_check_launch(tm_ctx *ctx, const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) TM_FAIL(ctx, TM_E_CUDA, "%s: launch failed: %s", what, cudaGetErrorString(e));
    return TM_OK;
}

// Latched device errors (DevState, first seven fields) -> status.  The health and error
// counters accumulate from one synchronising call (tm_sync, tm_mesh_stats) to the next,
// which reports them and then clears them, so a caller that retries after an error
// (e.g. a larger tri_cap after TM_E_CAPACITY) is not stuck with a stale error.
static tm_status report_latched(tm_ctx *ctx, const DevState &s) {
    if (s.n_outside) TM_FAIL(ctx, TM_E_OUTSIDE, "%llu point(s) are NaN or outside the box B", s.n_outside);
    if (s.n_duplicate) TM_FAIL(ctx, TM_E_DUPLICATE, "%llu bitwise-duplicate point pair(s)", s.n_duplicate);
    if (s.n_overflow)
        TM_FAIL(ctx, TM_E_CAPACITY, "%llu cell(s) exceeded the %d-vertex capacity", s.n_overflow,
                ctx->p.max_cell_vertices);
    if (s.n_tri_overflow) TM_FAIL(ctx, TM_E_CAPACITY, "triangle buffer too small (tri_cap)");
    if (s.n_adj_overflow) TM_FAIL(ctx, TM_E_CAPACITY, "ELL row wider than adj_stride=%d", ctx->p.adj_stride);
    if (s.n_strip_overflow)
        TM_FAIL(ctx, TM_E_CAPACITY, "%llu strip halo/migration message(s) or append(s) beyond capacity",
                s.n_strip_overflow);
    return TM_OK;
}

static tm_status clear_latched(tm_ctx *ctx) {
    TM_CUDA_TRY(ctx, cudaMemsetAsync(ctx->dst, 0, offsetof(DevState, work), ctx->stream));
    return TM_OK;
}

extern "C" tm_status tm_sync(tm_ctx *ctx) {
    if (!ctx) return TM_E_ARG;
    if (ctx->capturing) TM_FAIL(ctx, TM_E_STATE, "tm_sync while capturing a graph");
    TM_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
    TM_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    DevState s;
    TM_CUDA_TRY(ctx, cudaMemcpy(&s, ctx->dst, sizeof(s), cudaMemcpyDeviceToHost));
    const tm_status r = report_latched(ctx, s);
    const tm_status c = clear_latched(ctx);
    return r != TM_OK ? r : c;
}

// ============================================================================ S0
// c and h_avg by a deterministic sequential sum in row-major cell order
// (identical operation order to the oracle's definition, §8.0 "Local size").
// S0 sums (reading L7): the per-cell terms are evaluated in parallel, then summed by
// one thread in row-major order, so that c and h_avg keep the bits of the sequential
// definition (the oracle's order) -- the sums are sequential, the bilinear work is not.
__global__ void k_domain_terms(Grid g, const double *phi, const double *mu, double *w, double *m) {
    const int64_t ncx = g.nx - 1, ncy = g.ny - 1;
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= ncx * ncy) return;
    const int64_t j = k / ncx, i = k % ncx;
    const double *p0 = phi + j * g.nx, *p1 = p0 + g.nx;
    const double ph = clerp(clerp(p0[i], p0[i + 1], 0.5), clerp(p1[i], p1[i + 1], 0.5), 0.5);
    if (!(ph < 0.0)) {
        w[k] = -1.0;  // outside: skipped by the sum
        return;
    }
    double mm = 1.0;
    if (mu) {
        const double *m0 = mu + j * g.nx, *m1 = m0 + g.nx;
        mm = clerp(clerp(m0[i], m0[i + 1], 0.5), clerp(m1[i], m1[i + 1], 0.5), 0.5);
    }
    w[k] = cdiv(1.0, cmul(mm, mm));
    m[k] = mm;
}

// S0 sums in row-major order, one adder (the oracle's order, so the same bits): the block's
// other warps stage the next tile of terms in shared memory while thread 0 adds the current
// one -- the adds then wait on shared-memory loads, not on DRAM round trips
constexpr int DS_TILE = 1024;
__global__ void __launch_bounds__(256) k_domain_sums(int64_t n, const double *__restrict__ w,
                                                     const double *__restrict__ m, double *out3) {
    __shared__ double tw[2][DS_TILE], tm[2][DS_TILE];
    const int tid = threadIdx.x;
    auto stage = [&](int buf, int64_t base, int t0, int stride) {
        for (int i = t0; i < DS_TILE; i += stride) {
            const int64_t k = base + i;
            tw[buf][i] = k < n ? w[k] : -1.0;  // padding: w < 0 is skipped like an outside cell
            tm[buf][i] = k < n ? m[k] : 0.0;
        }
    };
    stage(0, 0, tid, blockDim.x);
    __syncthreads();
    double sum_w = 0.0, sum_mu = 0.0, cnt = 0.0;
    const int64_t ntiles = (n + DS_TILE - 1) / DS_TILE;
    for (int64_t t = 0; t < ntiles; t++) {
        const int b = (int)(t & 1);
        if (tid >= 32) {
            if (t + 1 < ntiles) stage(b ^ 1, (t + 1) * DS_TILE, tid - 32, blockDim.x - 32);
        } else if (tid == 0) {
#pragma unroll 16
            for (int i = 0; i < DS_TILE; i++) {
                const double wk = tw[b][i];
                if (wk < 0.0) continue;
                sum_w = cadd(sum_w, wk);
                sum_mu = cadd(sum_mu, tm[b][i]);
                cnt += 1.0;
            }
        }
        __syncthreads();
    }
    if (tid == 0) {
        out3[0] = sum_w;
        out3[1] = sum_mu;
        out3[2] = cnt;
    }
}

// Lipschitz constant of the bilinear interpolant mu~ (continuous, bilinear per cell):
// max over cells of |grad| <= sqrt(gx^2 + gy^2), gx = max(|f10-f00|,|f11-f01|)/dx, gy
// likewise; kept as the bits of a positive double (atomicMax on the integer view)
// the four corners of every grid cell contiguous: (f00, f10, f01, f11) of cell (i, j)
__global__ void k_pack_corners(Grid g, const double *__restrict__ f, double4 *__restrict__ out) {
    const int64_t ncx = g.nx - 1, ncy = g.ny - 1;
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= ncx * ncy) return;
    const int64_t j = k / ncx, i = k % ncx;
    const double *r0 = f + j * g.nx, *r1 = r0 + g.nx;
    out[k] = make_double4(r0[i], r0[i + 1], r1[i], r1[i + 1]);
}

__global__ void k_lipschitz(Grid g, const double *mu, unsigned long long *out) {
    const int64_t ncx = g.nx - 1, ncy = g.ny - 1;
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= ncx * ncy) return;
    const int64_t j = k / ncx, i = k % ncx;
    const double *r0 = mu + j * g.nx, *r1 = r0 + g.nx;
    const double gx = fmax(fabs(r0[i + 1] - r0[i]), fabs(r1[i + 1] - r1[i])) / g.dx;
    const double gy = fmax(fabs(r1[i] - r0[i]), fabs(r1[i + 1] - r0[i + 1])) / g.dy;
    const double L = sqrt(gx * gx + gy * gy) * (1.0 + 1e-12);
    atomicMax(out, (unsigned long long)__double_as_longlong(L));
}

extern "C" tm_status tm_set_domain(tm_ctx *ctx, const tm_fields *f, int64_t n_total, double *c_out,
                                   double *h_avg_out) {
    if (ctx && ctx->capturing) TM_FAIL(ctx, TM_E_STATE, "tm_set_domain while capturing a graph");
    if (!ctx || !f || !f->phi) return ctx ? (snprintf(ctx->err, sizeof(ctx->err), "null argument"), TM_E_ARG) : TM_E_ARG;
    if (f->nx < 2 || f->ny < 2 || !(f->x1 > f->x0) || !(f->y1 > f->y0) || n_total < 1)
        TM_FAIL(ctx, TM_E_ARG, "bad domain: grid %dx%d, box [%g,%g]x[%g,%g], n_total %lld", f->nx, f->ny, f->x0,
                f->x1, f->y0, f->y1, (long long)n_total);
    TM_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
    size_t nb = (size_t)f->nx * f->ny * sizeof(double);
    if (nb != ctx->grid_bytes) {
        cudaFree(ctx->phi); cudaFree(ctx->mu); cudaFree(ctx->rho);
        ctx->phi = ctx->mu = ctx->rho = nullptr;
        TM_CUDA_TRY(ctx, cudaMalloc(&ctx->phi, nb));
        TM_CUDA_TRY(ctx, cudaMalloc(&ctx->mu, nb));
        TM_CUDA_TRY(ctx, cudaMalloc(&ctx->rho, nb));
        ctx->grid_bytes = nb;
    }
    TM_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->phi, f->phi, nb, cudaMemcpyDeviceToDevice, ctx->stream));
    if (f->mu) TM_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->mu, f->mu, nb, cudaMemcpyDeviceToDevice, ctx->stream));
    if (f->rho) TM_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->rho, f->rho, nb, cudaMemcpyDeviceToDevice, ctx->stream));
    Grid g;
    g.nx = f->nx; g.ny = f->ny;
    g.x0 = f->x0; g.y0 = f->y0; g.x1 = f->x1; g.y1 = f->y1;
    g.idx = cdiv((double)(f->nx - 1), csub(f->x1, f->x0));
    g.idy = cdiv((double)(f->ny - 1), csub(f->y1, f->y0));
    g.dx = cdiv(csub(f->x1, f->x0), (double)(f->nx - 1));
    g.dy = cdiv(csub(f->y1, f->y0), (double)(f->ny - 1));
    ctx->grid = g;
    bool has_mu = f->mu != nullptr, has_rho = f->rho != nullptr;
    double *d3, *terms;
    const int64_t ncell = (int64_t)(g.nx - 1) * (g.ny - 1);
    TM_CUDA_TRY(ctx, cudaMalloc(&d3, 3 * sizeof(double)));
    TM_CUDA_TRY(ctx, cudaMalloc(&terms, 2 * ncell * sizeof(double)));
    k_domain_terms<<<(unsigned)((ncell + 255) / 256), 256, 0, ctx->stream>>>(g, ctx->phi, has_mu ? ctx->mu : nullptr,
                                                                             terms, terms + ncell);
    k_domain_sums<<<1, 256, 0, ctx->stream>>>(ncell, terms, terms + ncell, d3);
    tm_status s = tm_internal_check_launch(ctx, "k_domain_sums");
    if (s != TM_OK) { cudaFree(d3); cudaFree(terms); return s; }
    double h3[3];
    cudaError_t e = cudaMemcpyAsync(h3, d3, sizeof(h3), cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    cudaFree(d3);
    cudaFree(terms);
    if (e != cudaSuccess) TM_FAIL(ctx, TM_E_CUDA, "set_domain: %s", cudaGetErrorString(e));
    if (!(h3[2] > 0)) TM_FAIL(ctx, TM_E_ARG, "the SDF grid has no cell with phi < 0");
    // c = sqrt( sum_w * (dx*dy) / N ),  h_avg = c * (sum_mu / count)   (same order as the definition)
    // Lipschitz constants of the bilinear interpolants of mu (adaptive halo widths) and phi
    // (keep-rule fast path of the cell kernels)
    {
        unsigned long long *dl;
        TM_CUDA_TRY(ctx, cudaMalloc(&dl, 2 * sizeof(unsigned long long)));
        TM_CUDA_TRY(ctx, cudaMemsetAsync(dl, 0, 2 * sizeof(unsigned long long), ctx->stream));
        if (has_mu) k_lipschitz<<<(unsigned)((ncell + 255) / 256), 256, 0, ctx->stream>>>(g, ctx->mu, dl);
        k_lipschitz<<<(unsigned)((ncell + 255) / 256), 256, 0, ctx->stream>>>(g, ctx->phi, dl + 1);
        unsigned long long hl[2] = {0, 0};
        cudaError_t e2 = cudaMemcpyAsync(hl, dl, sizeof(hl), cudaMemcpyDeviceToHost, ctx->stream);
        if (e2 == cudaSuccess) e2 = cudaStreamSynchronize(ctx->stream);
        cudaFree(dl);
        if (e2 != cudaSuccess) TM_FAIL(ctx, TM_E_CUDA, "set_domain: %s", cudaGetErrorString(e2));
        double L[2];
        memcpy(L, hl, sizeof(L));
        ctx->lip_mu = has_mu ? L[0] : 0.0;
        ctx->lip_phi = L[1];
    }
    ctx->dom_sums[0] = h3[0];
    ctx->dom_sums[1] = h3[1];
    ctx->dom_sums[2] = h3[2];
    ctx->c = sqrt(cdiv(cmul(h3[0], cmul(g.dx, g.dy)), (double)n_total));
    ctx->h_avg = cmul(ctx->c, cdiv(h3[1], h3[2]));
    if (!has_mu) { cudaFree(ctx->mu); ctx->mu = nullptr; ctx->grid_bytes = 0; }
    if (!has_rho) { cudaFree(ctx->rho); ctx->rho = nullptr; ctx->grid_bytes = 0; }
    // S0 packing: each grid cell's four corners of rho contiguous, 32 bytes,
    // so the quadrature's bilinear lookups cost one sector instead of two rows
    cudaFree(ctx->rho4);
    ctx->rho4 = nullptr;
    if (has_rho) {
        TM_CUDA_TRY(ctx, cudaMalloc(&ctx->rho4, (size_t)ncell * sizeof(double4)));
        k_pack_corners<<<(unsigned)((ncell + 255) / 256), 256, 0, ctx->stream>>>(g, ctx->rho, ctx->rho4);
        TM_CUDA_TRY(ctx, cudaGetLastError());
    }
    tm_internal_set_n_total(ctx, n_total);
    ctx->have_domain = true;
    ctx->nbr_n = -1;
    ctx->have_bins = false;
    ctx->have_cells = false;
    if (c_out) *c_out = ctx->c;
    if (h_avg_out) *h_avg_out = ctx->h_avg;
    return TM_OK;
}

// c = sqrt( sum_w * (dx*dy) / N ), h_avg = c * (sum_mu / count) for N = n_total, and the level-0
// bins for N points: N_opt points per bin on average (P:343 without fac_grid; Listing P:651-654).
// Point addition (NEXT-3) calls it with N_current: the adaptive quantities follow the resolution
// (reading L44: recomputed for N_current = scaled by sqrt(N_old / N_current) up to rounding)
void tm_internal_set_n_total(tm_ctx *ctx, int64_t n_total) {
    const Grid &g = ctx->grid;
    ctx->c = sqrt(cdiv(cmul(ctx->dom_sums[0], cmul(g.dx, g.dy)), (double)n_total));
    ctx->h_avg = cmul(ctx->c, cdiv(ctx->dom_sums[1], ctx->dom_sums[2]));
    ctx->n_total = n_total;
    double Lx = g.x1 - g.x0, Ly = g.y1 - g.y0;
    double lam = sqrt((double)n_total / (ctx->p.n_opt * Lx * Ly));
    int32_t nbx = (int32_t)ceil(lam * Lx), nby = (int32_t)ceil(lam * Ly);
    if (nbx < 1) nbx = 1;
    if (nby < 1) nby = 1;
    ctx->bg.nbx = nbx; ctx->bg.nby = nby;
    ctx->bg.x0 = g.x0; ctx->bg.y0 = g.y0;
    ctx->bg.sx = Lx / nbx; ctx->bg.sy = Ly / nby;
    ctx->bg.isx = nbx / Lx; ctx->bg.isy = nby / Ly;
    ctx->nbr_n = -1;  // warm-start lists are keyed by a point set of the old size
    ctx->have_bins = false;
    ctx->have_cells = false;
}

// ============================================================================ S1
__global__ void k_bin_keys(const double *__restrict__ x, const double *__restrict__ y, int64_t n, BinGeom bg,
                           double bx0, double by0, double bx1, double by1, int32_t *__restrict__ key,
                           int32_t *__restrict__ count, DevState *st, const int64_t *dn) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (dn ? dn[1] : n)) return;
    double px = x[i], py = y[i];
    if (!(px >= bx0 && px <= bx1 && py >= by0 && py <= by1)) {
        atomicAdd(&st->n_outside, 1ull);
        px = fmin(fmax(px == px ? px : bx0, bx0), bx1);
        py = fmin(fmax(py == py ? py : by0, by0), by1);
    }
    int bx = (int)floor((px - bg.x0) * bg.isx), by = (int)floor((py - bg.y0) * bg.isy);
    bx = bx < 0 ? 0 : (bx >= bg.nbx ? bg.nbx - 1 : bx);
    by = by < 0 ? 0 : (by >= bg.nby ? bg.nby - 1 : by);
    int32_t k = by * bg.nbx + bx;
    key[i] = k;
    atomicAdd(&count[k], 1);
}

// level of every level-0 bin: r = 0 if count <= 4*N_opt, else the smallest
// r <= MAX_SUBLEVEL with 4^r >= count/N_opt (SURVEY §8(a) S1 two-level list)
__global__ void k_bin_levels(const int32_t *__restrict__ count, int64_t nb, double n_opt, int two_level,
                             uint8_t *__restrict__ rlev, int32_t *__restrict__ nleaf) {
    int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= nb) return;
    double c = (double)count[b];
    int r = 0;
    if (two_level && c > 4.0 * n_opt) {
        r = 1;
        while (r < MAX_SUBLEVEL && (double)(1 << (2 * r)) * n_opt < c) r++;
    }
    rlev[b] = (uint8_t)r;
    nleaf[b] = 1 << (2 * r);
}

// leaf key (level-0 bin, Morton sub-index) and rank within the leaf
__global__ void k_leaf_keys(const double *__restrict__ x, const double *__restrict__ y, int64_t n, BinGeom bg,
                            double bx0, double by0, double bx1, double by1, int32_t *__restrict__ key,
                            const uint8_t *__restrict__ rlev, const int32_t *__restrict__ leaf_off,
                            int32_t *__restrict__ leaf_count, int32_t *__restrict__ rank, const int64_t *dn) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (dn ? dn[1] : n)) return;
    double px = fmin(fmax(x[i] == x[i] ? x[i] : bx0, bx0), bx1);
    double py = fmin(fmax(y[i] == y[i] ? y[i] : by0, by0), by1);
    int32_t b = key[i];
    int r = rlev[b];
    int32_t leaf = leaf_off[b];
    if (r > 0) {
        int bxi = b % bg.nbx, byi = b / bg.nbx;
        int ux = leaf_coord(px, bg.x0, bg.isx, bg.nbx, r) - (bxi << r);
        int uy = leaf_coord(py, bg.y0, bg.isy, bg.nby, r) - (byi << r);
        leaf += (int32_t)morton2((uint32_t)ux, (uint32_t)uy);
    }
    key[i] = leaf;
    rank[i] = atomicAdd(&leaf_count[leaf], 1);
}

// exclusive scan: per-block (1024 threads x 4 items)
constexpr int SCAN_T = 1024, SCAN_ITEMS = 4, SCAN_TILE = SCAN_T * SCAN_ITEMS;

__device__ __forceinline__ int32_t block_exclusive_scan(int32_t v, int32_t *smem_warp, int32_t &total) {
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int32_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) smem_warp[w] = incl;
    __syncthreads();
    if (w == 0) {
        int32_t s = lane < (int)(blockDim.x >> 5) ? smem_warp[lane] : 0;
        int32_t si = s;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int32_t t = __shfl_up_sync(0xffffffffu, si, o);
            if (lane >= o) si += t;
        }
        smem_warp[lane] = si - s;
        if (lane == 31) smem_warp[32] = si;
    }
    __syncthreads();
    total = smem_warp[32];
    int32_t r = smem_warp[w] + incl - v;
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(SCAN_T) k_scan_tiles(const int32_t *__restrict__ in, int32_t *__restrict__ out,
                                                       int32_t *__restrict__ tile_sums, int64_t n) {
    __shared__ int32_t sw[33];
    int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
    int32_t v[SCAN_ITEMS], s = 0;
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; k++) {
        v[k] = (base + k < n) ? in[base + k] : 0;
        s += v[k];
    }
    int32_t total;
    int32_t ex = block_exclusive_scan(s, sw, total);
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; k++) {
        if (base + k < n) out[base + k] = ex;
        ex += v[k];
    }
    if (threadIdx.x == 0) tile_sums[blockIdx.x] = total;
}

// single block: exclusive scan of tile sums in place, grand total to *total_out
__global__ void __launch_bounds__(SCAN_T) k_scan_top(int32_t *tile_sums, int64_t ntiles, int32_t *total_out) {
    __shared__ int32_t sw[33];
    int32_t carry = 0;
    for (int64_t b0 = 0; b0 < ntiles; b0 += SCAN_T) {
        int64_t i = b0 + threadIdx.x;
        int32_t v = i < ntiles ? tile_sums[i] : 0;
        int32_t total;
        int32_t ex = block_exclusive_scan(v, sw, total);
        if (i < ntiles) tile_sums[i] = ex + carry;
        carry += total;
    }
    if (threadIdx.x == 0) *total_out = carry;
}

__global__ void k_scan_add(int32_t *out, const int32_t *tile_sums, int64_t n) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    out[i] += tile_sums[i / SCAN_TILE];
}

// S1 tail: the slot of every point is its leaf's start plus its rank in the leaf; the
// ranks come from atomics (arbitrary order), so each leaf's caller indices are then
// sorted (4-byte keys only) and the point data gathered once into slot order with
// coalesced stores: the in-leaf order is the caller order, deterministic.
__global__ void k_perm_scatter(int64_t n, const int32_t *__restrict__ key, const int32_t *__restrict__ rank,
                               const int32_t *__restrict__ start, int32_t *__restrict__ perm, const int64_t *dn) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (dn ? dn[1] : n)) return;
    perm[(int64_t)start[key[i]] + rank[i]] = (int32_t)i;
}

__global__ void k_leaf_sort_perm(const int32_t *__restrict__ leaf_start, int64_t nleaves, int32_t *__restrict__ perm,
                                 const int32_t *__restrict__ gid, int64_t nkey, int32_t *__restrict__ inv_id) {
    const int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= nleaves) return;
    const int s = leaf_start[l], e = leaf_start[l + 1];
    for (int a = s + 1; a < e; a++) {
        const int32_t pk = perm[a];
        int b = a - 1;
        while (b >= s && perm[b] > pk) {
            perm[b + 1] = perm[b];
            b--;
        }
        perm[b + 1] = pk;
    }
    // point id (gid if given, else caller index) -> slot, for the warm start
    for (int a = s; a < e; a++) {
        const int32_t id = gid ? gid[perm[a]] : perm[a];
        if (id >= 0 && (int64_t)id < nkey) inv_id[id] = a;  // gids outside [0, n_total): no warm start
    }
}

__global__ void k_gather_sorted(const double *__restrict__ x, const double *__restrict__ y,
                                const int32_t *__restrict__ gid, int64_t n, const int32_t *__restrict__ perm,
                                double bx0, double by0, double bx1, double by1, Grid g, const double *__restrict__ mu,
                                double c, double *__restrict__ xs, double *__restrict__ ys, double *__restrict__ hs,
                                int32_t *__restrict__ gids, const int64_t *dn) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= (dn ? dn[1] : n)) return;
    const int32_t i = perm[s];
    double px = x[i], py = y[i];
    px = fmin(fmax(px == px ? px : bx0, bx0), bx1);
    py = fmin(fmax(py == py ? py : by0, by0), by1);
    xs[s] = px;
    ys[s] = py;
    hs[s] = mu ? cmul(c, bilinear(g, mu, px, py, LdgLoad())) : c;  // h(p) = c mu~(p) (§8.0 "Local size")
    gids[s] = gid ? gid[i] : i;
}

static tm_status ensure_points(tm_ctx *ctx, int64_t n) {
    if (n <= ctx->cap_points) return TM_OK;
    free_points(ctx);
    int64_t cap = n + n / 8 + 1024;
    TM_CUDA_TRY(ctx, cudaMalloc(&ctx->xs, cap * sizeof(double)));
    TM_CUDA_TRY(ctx, cudaMalloc(&ctx->ys, cap * sizeof(double)));
    TM_CUDA_TRY(ctx, cudaMalloc(&ctx->hs, cap * sizeof(double)));
    TM_CUDA_TRY(ctx, cudaMalloc(&ctx->perm, cap * sizeof(int32_t)));
    TM_CUDA_TRY(ctx, cudaMalloc(&ctx->gids, cap * sizeof(int32_t)));
    TM_CUDA_TRY(ctx, cudaMalloc(&ctx->key, cap * sizeof(int32_t)));
    TM_CUDA_TRY(ctx, cudaMalloc(&ctx->rank, cap * sizeof(int32_t)));
    ctx->cap_points = cap;
    return TM_OK;
}

static tm_status ensure_bins(tm_ctx *ctx, int64_t nb, int64_t nleaves) {
    int64_t ntiles = (std::max(nb, nleaves) + SCAN_TILE - 1) / SCAN_TILE;
    if (nb + 1 > ctx->cap_bins) {
        cudaFree(ctx->bin_count); cudaFree(ctx->rlev); cudaFree(ctx->leaf_off);
        ctx->bin_count = nullptr; ctx->rlev = nullptr; ctx->leaf_off = nullptr;
        TM_CUDA_TRY(ctx, cudaMalloc(&ctx->bin_count, (nb + 1) * sizeof(int32_t)));
        TM_CUDA_TRY(ctx, cudaMalloc(&ctx->rlev, (nb + 1) * sizeof(uint8_t)));
        TM_CUDA_TRY(ctx, cudaMalloc(&ctx->leaf_off, (nb + 1) * sizeof(int32_t)));
        ctx->cap_bins = nb + 1;
    }
    if (nleaves + 1 > ctx->cap_leaves) {
        cudaFree(ctx->leaf_count); cudaFree(ctx->leaf_start);
        ctx->leaf_count = ctx->leaf_start = nullptr;
        TM_CUDA_TRY(ctx, cudaMalloc(&ctx->leaf_count, (nleaves + 1) * sizeof(int32_t)));
        TM_CUDA_TRY(ctx, cudaMalloc(&ctx->leaf_start, (nleaves + 1) * sizeof(int32_t)));
        ctx->cap_leaves = nleaves + 1;
    }
    if (ntiles > ctx->cap_block_sums) {
        cudaFree(ctx->block_sums);
        ctx->block_sums = nullptr;
        TM_CUDA_TRY(ctx, cudaMalloc(&ctx->block_sums, ntiles * sizeof(int32_t)));
        ctx->cap_block_sums = ntiles;
    }
    return TM_OK;
}

static tm_status ensure_scan_scratch(tm_ctx *ctx, int64_t n) {
    const int64_t ntiles = (n + SCAN_TILE - 1) / SCAN_TILE;
    if (ntiles > ctx->cap_block_sums) {
        cudaFree(ctx->block_sums);
        ctx->block_sums = nullptr;
        TM_CUDA_TRY(ctx, cudaMalloc(&ctx->block_sums, ntiles * sizeof(int32_t)));
        ctx->cap_block_sums = ntiles;
    }
    return TM_OK;
}

// exclusive scan of n int32 values into out[0..n], out[n] = total
static tm_status scan_counts(tm_ctx *ctx, const int32_t *in, int32_t *out, int64_t n) {
    int64_t ntiles = (n + SCAN_TILE - 1) / SCAN_TILE;
    k_scan_tiles<<<(unsigned)ntiles, SCAN_T, 0, ctx->stream>>>(in, out, ctx->block_sums, n);
    k_scan_top<<<1, SCAN_T, 0, ctx->stream>>>(ctx->block_sums, ntiles, out + n);
    k_scan_add<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(out, ctx->block_sums, n);
    return tm_internal_check_launch(ctx, "scan");
}

// n_local: the number of points, or with dcnt (device {n_owned, n_local}) the capacity of x/y/gid
static tm_status grid_bin_impl(tm_ctx *ctx, const double *x, const double *y, int64_t n_local, int64_t n_owned,
                               const int32_t *gid, const int64_t *dcnt) {
    if (!ctx) return TM_E_ARG;
    if (!ctx->have_domain) TM_FAIL(ctx, TM_E_STATE, "tm_grid_bin before tm_set_domain");
    if (!x || !y) TM_FAIL(ctx, TM_E_ARG, "null x/y");
    if (n_local < 3 || n_owned < 1 || n_owned > n_local || n_local >= (int64_t)INT32_MAX)
        TM_FAIL(ctx, TM_E_ARG, "bad sizes n_local=%lld n_owned=%lld", (long long)n_local, (long long)n_owned);
    TM_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
    tm_status s = ensure_points(ctx, n_local);
    if (s != TM_OK) return s;
    int64_t nb = (int64_t)ctx->bg.nbx * ctx->bg.nby;
    // leaves: 4^r per bin; for r > 0, 4^r < 4 count / N_opt, so the total is below nb + 4 N / N_opt
    int64_t nleaves_max = nb + (int64_t)ceil(4.0 * (double)n_local / ctx->p.n_opt) + 1;
    if ((s = ensure_bins(ctx, nb, nleaves_max)) != TM_OK) return s;
    // warm start (tm_cells_t.cu): neighbour lists and the id -> slot map are keyed by point id,
    // the gid when given (strips: ids are global and stable while local positions change),
    // else the caller index; the key space is n_total resp. n_local
    const int64_t nkey = gid ? ctx->n_total : n_local;
    if (nkey != ctx->nbr_n || (gid != nullptr) != ctx->have_gid) ctx->nbr_n = -1;  // warm start invalid
    if (nkey > ctx->cap_nbr) {
        cudaFree(ctx->nbr);
        cudaFree(ctx->nbr_cnt);
        cudaFree(ctx->inv_id);
        ctx->nbr = nullptr;
        ctx->nbr_cnt = nullptr;
        ctx->inv_id = nullptr;
        const int64_t c = nkey + nkey / 8 + 1024;
        TM_CUDA_TRY(ctx, cudaMalloc(&ctx->nbr, c * TM_NBR * sizeof(int32_t)));
        TM_CUDA_TRY(ctx, cudaMalloc(&ctx->nbr_cnt, c * sizeof(uint8_t)));
        TM_CUDA_TRY(ctx, cudaMalloc(&ctx->inv_id, c * sizeof(int32_t)));
        TM_CUDA_TRY(ctx, cudaMemsetAsync(ctx->nbr_cnt, 0, c * sizeof(uint8_t), ctx->stream));
        ctx->cap_nbr = c;
        ctx->nbr_n = -1;
    }
    TM_CUDA_TRY(ctx, cudaMemsetAsync(ctx->bin_count, 0, nb * sizeof(int32_t), ctx->stream));
    const Grid &g = ctx->grid;
    unsigned blocks = (unsigned)((n_local + 255) / 256);
    k_bin_keys<<<blocks, 256, 0, ctx->stream>>>(x, y, n_local, ctx->bg, g.x0, g.y0, g.x1, g.y1, ctx->key,
                                                ctx->bin_count, ctx->dst, dcnt);
    if ((s = tm_internal_check_launch(ctx, "k_bin_keys")) != TM_OK) return s;
    // per-bin level and number of leaves (reuses leaf_count as scratch), scan -> leaf_off
    k_bin_levels<<<(unsigned)((nb + 255) / 256), 256, 0, ctx->stream>>>(
        ctx->bin_count, nb, ctx->p.n_opt, (ctx->p.flags & TM_F_TWO_LEVEL_BINS) ? 1 : 0, ctx->rlev, ctx->leaf_count);
    if ((s = scan_counts(ctx, ctx->leaf_count, ctx->leaf_off, nb)) != TM_OK) return s;
    TM_CUDA_TRY(ctx, cudaMemsetAsync(ctx->leaf_count, 0, nleaves_max * sizeof(int32_t), ctx->stream));
    k_leaf_keys<<<blocks, 256, 0, ctx->stream>>>(x, y, n_local, ctx->bg, g.x0, g.y0, g.x1, g.y1, ctx->key, ctx->rlev,
                                                 ctx->leaf_off, ctx->leaf_count, ctx->rank, dcnt);
    if ((s = tm_internal_check_launch(ctx, "k_leaf_keys")) != TM_OK) return s;
    if ((s = scan_counts(ctx, ctx->leaf_count, ctx->leaf_start, nleaves_max)) != TM_OK) return s;
    k_perm_scatter<<<blocks, 256, 0, ctx->stream>>>(n_local, ctx->key, ctx->rank, ctx->leaf_start, ctx->perm, dcnt);
    k_leaf_sort_perm<<<(unsigned)((nleaves_max + 255) / 256), 256, 0, ctx->stream>>>(ctx->leaf_start, nleaves_max,
                                                                                   ctx->perm, gid, nkey, ctx->inv_id);
    ctx->gids_in = gid;
    k_gather_sorted<<<blocks, 256, 0, ctx->stream>>>(x, y, gid, n_local, ctx->perm, g.x0, g.y0, g.x1, g.y1, g, ctx->mu,
                                                     ctx->c, ctx->xs, ctx->ys, ctx->hs, ctx->gids, dcnt);
    if ((s = tm_internal_check_launch(ctx, "k_gather_sorted")) != TM_OK) return s;
    ctx->have_gid = gid != nullptr;
    ctx->n_local = n_local;
    ctx->n_owned = n_owned;
    ctx->dcnt = dcnt;
    ctx->have_bins = true;
    ctx->have_cells = false;
    return TM_OK;
}

extern "C" tm_status tm_grid_bin(tm_ctx *ctx, const double *x, const double *y, int64_t n_local, int64_t n_owned,
                                 const int32_t *gid) {
    return grid_bin_impl(ctx, x, y, n_local, n_owned, gid, nullptr);
}

extern "C" tm_status tm_grid_bin_dc(tm_ctx *ctx, const double *x, const double *y, int64_t cap_local,
                                    const int64_t *d_counts, const int32_t *gid) {
    if (!ctx) return TM_E_ARG;
    if (!d_counts || !gid) TM_FAIL(ctx, TM_E_ARG, "tm_grid_bin_dc needs device counts and global ids");
    return grid_bin_impl(ctx, x, y, cap_local, cap_local, gid, d_counts);
}

tm_status tm_internal_fill_cell_args(tm_ctx *ctx, CellArgs *a) {
    memset(a, 0, sizeof(*a));
    a->xs = ctx->xs; a->ys = ctx->ys; a->hs = ctx->hs;
    a->perm = ctx->perm; a->gids = ctx->gids; a->inv_perm = ctx->inv_id;
    a->nbr = ctx->nbr;
    a->nbr_cnt = ctx->nbr_cnt;
    a->nbr_by_gid = ctx->have_gid ? 1 : 0;
    a->nbr_keys = ctx->have_gid ? ctx->n_total : ctx->n_local;
    a->warm = (a->nbr && ctx->nbr_n == a->nbr_keys) ? 1 : 0;
    a->rlev = ctx->rlev; a->leaf_off = ctx->leaf_off; a->leaf_start = ctx->leaf_start;
    a->bg = ctx->bg;
    a->n_local = ctx->n_local; a->n_owned = ctx->n_owned;
    a->dcnt = ctx->dcnt;
    a->grid = ctx->grid;
    a->phi = ctx->phi; a->mu = ctx->mu; a->rho = ctx->rho;
    a->rho4 = (ctx->p.flags & TM_F_NO_PACKED_GRIDS) ? nullptr : ctx->rho4;
    a->c = ctx->c; a->h_avg = ctx->h_avg;
    a->lip_mu = ctx->lip_mu; a->lip_phi = ctx->lip_phi;
    a->fac_voro = ctx->p.fac_voro_bound; a->fac_pt = ctx->p.fac_pt_mvmt;
    a->fac_geps = ctx->p.fac_geps; a->fac_end = ctx->p.fac_end_mvmt;
    a->damping = ctx->p.newton_damping; a->keep_tol = ctx->p.keep_tol;
    a->validity = ctx->p.validity; a->t_circ = ctx->p.t_circ;
    a->newton_max = ctx->p.newton_max; a->quad_max = ctx->p.quad_max_level;
    a->projection = ctx->p.projection; a->trace_max = ctx->p.trace_max;
    a->adj_stride = ctx->p.adj_stride;
    a->st = ctx->dst;
    return TM_OK;
}

// ============================================================================ S5 standalone
__global__ void k_project(Grid g, const double *__restrict__ phi, const double *__restrict__ mu, double c,
                          double h_avg, double fac_pt, double fac_geps, double damping, int newton_max,
                          const double *__restrict__ xo, const double *__restrict__ yo,
                          const double *__restrict__ xh, const double *__restrict__ yh, int64_t n,
                          double *__restrict__ x_out, double *__restrict__ y_out, double *__restrict__ d_out,
                          int8_t *__restrict__ status, DevState *st, int projection, int trace_max) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double px = xo[i], py = yo[i];
    double h = mu ? cmul(c, bilinear(g, mu, px, py, LdgLoad())) : c;
    double qx, qy, dp;
    int s = treat_point(g, phi, h, h_avg, fac_pt, fac_geps, damping, newton_max, px, py, xh[i], yh[i], qx, qy, dp,
                        LdgLoad(), projection, trace_max);
    x_out[i] = qx;
    y_out[i] = qy;
    d_out[i] = dp;
    status[i] = (int8_t)s;
    if (s & 2) atomicAdd(&st->n_fallback, 1ull);
}

extern "C" tm_status tm_project_sdf(tm_ctx *ctx, const double *x_old, const double *y_old, const double *x_hat,
                                    const double *y_hat, int64_t n, double *x_out, double *y_out,
                                    double *d_prev_out, int8_t *status) {
    if (!ctx) return TM_E_ARG;
    if (!ctx->have_domain) TM_FAIL(ctx, TM_E_STATE, "tm_project_sdf before tm_set_domain");
    if (!x_old || !y_old || !x_hat || !y_hat || !x_out || !y_out || !d_prev_out || !status || n < 0)
        TM_FAIL(ctx, TM_E_ARG, "null argument to tm_project_sdf");
    if (n == 0) return TM_OK;
    TM_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
    k_project<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(
        ctx->grid, ctx->phi, ctx->mu, ctx->c, ctx->h_avg, ctx->p.fac_pt_mvmt, ctx->p.fac_geps,
        ctx->p.newton_damping, ctx->p.newton_max, x_old, y_old, x_hat, y_hat, n, x_out, y_out, d_prev_out,
        status, ctx->dst, ctx->p.projection, ctx->p.trace_max);
    return tm_internal_check_launch(ctx, "k_project");
}

// ============================================================================ S6
// acc layout: 0 n, 1 sum sqrt a, 2 sum sqrt b, 3 max a, 4 max b, 5 sum a, 6 sum a2, 7 sum b, 8 sum b2,
//             9 #a<1.2, 10 #a<2
// Deterministic: every block reduces its STATS_T triangles by a fixed shuffle tree and a
// fixed warp order into one row of partials; one block then reduces the rows in a fixed
// order (each thread a fixed stride of rows, then the same tree).  No atomics: the sums
// have the same bits on every run (no atomics on results).
constexpr int STATS_T = 256, STATS_K = 11;

__device__ __forceinline__ double stats_op(int k, double a, double b) { return (k == 3 || k == 4) ? fmax(a, b) : a + b; }

// block-wide fixed-order reduction of v[STATS_K]; result valid in thread 0
__device__ __forceinline__ void stats_block_reduce(double v[STATS_K], double (*sm)[STATS_T / 32]) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < STATS_K; k++) {
        double x = v[k];
        for (int o = 16; o > 0; o >>= 1) x = stats_op(k, x, __shfl_xor_sync(0xffffffffu, x, o));
        if (lane == 0) sm[k][w] = x;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < STATS_K; k++) {
            double x = sm[k][0];
            for (int ww = 1; ww < STATS_T / 32; ww++) x = stats_op(k, x, sm[k][ww]);
            v[k] = x;
        }
    }
}

__global__ void __launch_bounds__(STATS_T) k_stats(const double *__restrict__ x, const double *__restrict__ y,
                                                   const int32_t *__restrict__ tri, int64_t nt,
                                                   double *__restrict__ part) {
    __shared__ double sm[STATS_K][STATS_T / 32];
    const int64_t t = (int64_t)blockIdx.x * STATS_T + threadIdx.x;
    double v[STATS_K] = {0};
    if (t < nt) {
        int32_t a = tri[3 * t], b = tri[3 * t + 1], c = tri[3 * t + 2];
        double ax = x[a], ay = y[a], bx = x[b], by = y[b], cx = x[c], cy = y[c];
        double la = sqrt((bx - cx) * (bx - cx) + (by - cy) * (by - cy));
        double lb = sqrt((ax - cx) * (ax - cx) + (ay - cy) * (ay - cy));
        double lc = sqrt((ax - bx) * (ax - bx) + (ay - by) * (ay - by));
        double cr = (bx - ax) * (cy - ay) - (by - ay) * (cx - ax);
        double s = 0.5 * (la + lb + lc);
        double al = (la * lb * lc * s) / (2.0 * cr * cr);  // R/(2 r_in), Eq. aspect ratio
        double be = fmax(la, fmax(lb, lc)) / fmin(la, fmin(lb, lc));
        v[0] = 1; v[1] = sqrt(al); v[2] = sqrt(be); v[3] = al; v[4] = be;
        v[5] = al; v[6] = al * al; v[7] = be; v[8] = be * be; v[9] = al < 1.2; v[10] = al < 2.0;
    }
    stats_block_reduce(v, sm);
    if (threadIdx.x == 0)
        for (int k = 0; k < STATS_K; k++) part[(int64_t)k * gridDim.x + blockIdx.x] = v[k];
}

__global__ void __launch_bounds__(STATS_T) k_stats_final(const double *__restrict__ part, int64_t nb,
                                                         double *__restrict__ acc) {
    __shared__ double sm[STATS_K][STATS_T / 32];
    double v[STATS_K];
#pragma unroll
    for (int k = 0; k < STATS_K; k++) {
        double x = 0.0;
        for (int64_t b = threadIdx.x; b < nb; b += STATS_T) x = stats_op(k, x, part[k * nb + b]);
        v[k] = x;
    }
    stats_block_reduce(v, sm);
    if (threadIdx.x == 0)
        for (int k = 0; k < STATS_K; k++) acc[k] = v[k];
}

extern "C" tm_status tm_mesh_stats(tm_ctx *ctx, const double *x, const double *y, const int32_t *tri,
                                   int64_t n_tri, tm_stats *out) {
    if (!ctx) return TM_E_ARG;
    if (ctx->capturing) TM_FAIL(ctx, TM_E_STATE, "tm_mesh_stats while capturing a graph");
    if (!x || !y || (!tri && n_tri > 0) || !out || n_tri < 0) TM_FAIL(ctx, TM_E_ARG, "null argument to tm_mesh_stats");
    TM_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
    TM_CUDA_TRY(ctx, cudaMemsetAsync(ctx->stat_acc, 0, 16 * sizeof(double), ctx->stream));
    if (n_tri > 0) {
        const int64_t nb = (n_tri + STATS_T - 1) / STATS_T;
        if (nb * STATS_K > ctx->cap_partials) {  // cap_partials counts doubles (shared with DistMesh)
            cudaFree(ctx->partials);
            ctx->partials = nullptr;
            const int64_t c = (nb + nb / 8 + 64) * STATS_K;
            TM_CUDA_TRY(ctx, cudaMalloc(&ctx->partials, (size_t)c * sizeof(double)));
            ctx->cap_partials = c;
        }
        k_stats<<<(unsigned)nb, STATS_T, 0, ctx->stream>>>(x, y, tri, n_tri, ctx->partials);
        k_stats_final<<<1, STATS_T, 0, ctx->stream>>>(ctx->partials, nb, ctx->stat_acc);
        tm_status s = tm_internal_check_launch(ctx, "k_stats");
        if (s != TM_OK) return s;
    }
    double acc[16];
    DevState ds;
    TM_CUDA_TRY(ctx, cudaMemcpyAsync(acc, ctx->stat_acc, sizeof(acc), cudaMemcpyDeviceToHost, ctx->stream));
    TM_CUDA_TRY(ctx, cudaMemcpyAsync(&ds, ctx->dst, sizeof(ds), cudaMemcpyDeviceToHost, ctx->stream));
    TM_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    memset(out, 0, sizeof(*out));
    out->n_tri = (int64_t)acc[0];
    out->sum_sqrt_alpha = acc[1]; out->sum_sqrt_beta = acc[2];
    out->max_alpha = acc[3]; out->max_beta = acc[4];
    out->sum_alpha = acc[5]; out->sum_alpha2 = acc[6]; out->sum_beta = acc[7]; out->sum_beta2 = acc[8];
    out->n_alpha_lt_1_2 = (int64_t)acc[9]; out->n_alpha_lt_2 = (int64_t)acc[10];
    out->n_degenerate = (int64_t)ds.n_degenerate;
    out->n_fallback = (int64_t)ds.n_fallback;
    out->n_overflow = (int64_t)ds.n_overflow;
    const tm_status r = report_latched(ctx, ds);
    const tm_status c = clear_latched(ctx);
    return r != TM_OK ? r : c;
}

extern "C" tm_status tm_work_counts(tm_ctx *ctx, tm_work *out) {
    if (!ctx || !out) return TM_E_ARG;
    if (ctx->capturing) TM_FAIL(ctx, TM_E_STATE, "tm_work_counts while capturing a graph");
    TM_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
    DevState ds;
    TM_CUDA_TRY(ctx, cudaMemcpyAsync(&ds, ctx->dst, sizeof(ds), cudaMemcpyDeviceToHost, ctx->stream));
    TM_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    int64_t *o = (int64_t *)out;
    for (int k = 0; k < 10; k++) o[k] = (int64_t)ds.work[k];
    unsigned long long rc = 0;
    if (ctx->retry_cnt) {
        TM_CUDA_TRY(ctx, cudaMemcpyAsync(&rc, ctx->retry_cnt, sizeof(rc), cudaMemcpyDeviceToHost, ctx->stream));
        TM_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    }
    out->retries = (int64_t)rc;
    out->warp_trips = (int64_t)ds.work[10];
    return TM_OK;
}

// ============================================================================ exports
__global__ void k_adj_export(const int32_t *__restrict__ adj, const uint8_t *__restrict__ deg,
                             const int32_t *__restrict__ perm, const int32_t *__restrict__ gids, int64_t n_local,
                             int64_t n_owned, const int64_t *dcnt, int stride, int32_t *__restrict__ adj_out,
                             uint8_t *__restrict__ deg_out) {
    int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= (dcnt ? dcnt[1] : n_local)) return;
    int32_t o = perm[s];
    if (o >= (dcnt ? dcnt[0] : n_owned)) return;
    int d = deg[s];
    deg_out[o] = (uint8_t)d;
    for (int k = 0; k < stride; k++)
        adj_out[(int64_t)o * stride + k] = k < d ? gids[adj[(int64_t)k * n_local + s]] : -1;
}

extern "C" tm_status tm_adjacency_export(tm_ctx *ctx, const int32_t *adj, const uint8_t *deg, int32_t *adj_out,
                                         uint8_t *deg_out) {
    if (!ctx) return TM_E_ARG;
    if (!ctx->have_bins) TM_FAIL(ctx, TM_E_STATE, "tm_adjacency_export before tm_grid_bin");
    if (!adj || !deg || !adj_out || !deg_out) TM_FAIL(ctx, TM_E_ARG, "null argument to tm_adjacency_export");
    TM_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
    k_adj_export<<<(unsigned)((ctx->n_local + 255) / 256), 256, 0, ctx->stream>>>(
        adj, deg, ctx->perm, ctx->gids, ctx->n_local, ctx->n_owned, ctx->dcnt, ctx->p.adj_stride, adj_out, deg_out);
    return tm_internal_check_launch(ctx, "k_adj_export");
}

// ============================================================================ S7 packing
static double strip_edge(double v) { return v < -1e300 ? -1e300 : (v > 1e300 ? 1e300 : v); }

// Halo selection.  A point j of this strip can cut the cell of a point i
// across the edge only if |p_j - p_i| < 2 S_i (C_i lies in Oct_i).  With w > 0 the band
// is the fixed width w = 2 S_max.  With w < 0 the width is per point: S = fac h and h =
// c mu~ is Lipschitz with constant c L, so S_i <= S_j + fac c L d and d < 2 S_i implies
// d < 2 S_j / (1 - 2 fac c L) when 2 fac c L < 1; the band is the smaller of that and |w|.
// n: the owned count, or with dn the device one (*dn) and n the capacity.
__global__ void k_halo_pack(const double *__restrict__ x, const double *__restrict__ y,
                            const int32_t *__restrict__ gid, int64_t n, const int64_t *dn, double lo, double hi,
                            double w, Grid g, const double *__restrict__ mu, double c, double fac, double lip,
                            double *send_lo, double *send_hi, int64_t cap, unsigned long long *cnt_lo,
                            unsigned long long *cnt_hi) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const bool in_n = i < (dn ? *dn : n);
    const double px = in_n ? x[i] : 0.0;
    double wi = w;
    if (w < 0.0) {
        const double k = 2.0 * fac * c * lip;
        if (k < 1.0 && in_n) {
            const double h = mu ? c * bilinear(g, mu, px, y[i], LdgLoad()) : c;
            wi = fmin(2.0 * fac * h / (1.0 - k) * (1.0 + 1e-9), -w);  // both bounds hold: take the tighter
        } else {
            wi = -w;
        }
    }
    // two bands (a point can be in both when the strip is narrower than 2w);
    // one atomic per warp and band
#pragma unroll
    for (int side = 0; side < 2; side++) {
        const bool sel = in_n && (side == 0 ? px < lo + wi : px >= hi - wi);
        const unsigned m = __ballot_sync(0xffffffffu, sel);
        if (!m) continue;
        unsigned long long base = 0;
        if (lane == __ffs(m) - 1) base = atomicAdd(side == 0 ? cnt_lo : cnt_hi, (unsigned long long)__popc(m));
        base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
        if (sel) {
            const unsigned long long k = base + __popc(m & ((1u << lane) - 1u));
            double *dst = side == 0 ? send_lo : send_hi;
            if ((int64_t)k < cap) {
                dst[k] = px;
                dst[cap + k] = y[i];
                ((int32_t *)(dst + 2 * cap))[k] = gid ? gid[i] : (int32_t)i;
            }
        }
    }
}

static tm_status halo_pack_impl(tm_ctx *ctx, const double *x, const double *y, const int32_t *gid, int64_t n,
                                const int64_t *dn, double lo, double hi, double width, double *send_lo,
                                double *send_hi, int64_t cap, int64_t *cnt_lo, int64_t *cnt_hi) {
    TM_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
    TM_CUDA_TRY(ctx, cudaMemsetAsync(cnt_lo, 0, sizeof(int64_t), ctx->stream));
    TM_CUDA_TRY(ctx, cudaMemsetAsync(cnt_hi, 0, sizeof(int64_t), ctx->stream));
    if (n == 0) return TM_OK;
    if (width < 0.0 && !ctx->have_domain) TM_FAIL(ctx, TM_E_STATE, "adaptive halo width needs tm_set_domain");
    k_halo_pack<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(
        x, y, gid, n, dn, strip_edge(lo), strip_edge(hi), width, ctx->grid, ctx->mu, ctx->c, ctx->p.fac_voro_bound,
        ctx->lip_mu, send_lo, send_hi, cap, (unsigned long long *)cnt_lo, (unsigned long long *)cnt_hi);
    return tm_internal_check_launch(ctx, "k_halo_pack");
}

extern "C" tm_status tm_halo_pack(tm_ctx *ctx, const double *x, const double *y, const int32_t *gid,
                                  int64_t n_owned, double strip_lo, double strip_hi, double width, double *send_lo,
                                  double *send_hi, int64_t cap, int64_t *cnt2) {
    if (!ctx) return TM_E_ARG;
    if (!x || !y || !send_lo || !send_hi || !cnt2 || n_owned < 0 || cap < 0)
        TM_FAIL(ctx, TM_E_ARG, "null argument to tm_halo_pack");
    return halo_pack_impl(ctx, x, y, gid, n_owned, nullptr, strip_lo, strip_hi, width, send_lo, send_hi, cap, cnt2,
                          cnt2 + 1);
}

extern "C" tm_status tm_halo_pack_dc(tm_ctx *ctx, const double *x, const double *y, const int32_t *gid,
                                     const int64_t *d_n_owned, int64_t cap_owned, double strip_lo, double strip_hi,
                                     double width, double *send_lo, double *send_hi, int64_t cap, int64_t *cnt_lo,
                                     int64_t *cnt_hi) {
    if (!ctx) return TM_E_ARG;
    if (!x || !y || !d_n_owned || !send_lo || !send_hi || !cnt_lo || !cnt_hi || cap_owned < 0 || cap < 0)
        TM_FAIL(ctx, TM_E_ARG, "null argument to tm_halo_pack_dc");
    return halo_pack_impl(ctx, x, y, gid, cap_owned, d_n_owned, strip_lo, strip_hi, width, send_lo, send_hi, cap,
                          cnt_lo, cnt_hi);
}

// Stable 3-way partition of the owned points after an update (SURVEY §8(e)
// step 4): category 0 stays, 1 leaves to the lower strip, 2 to the upper one.
// Per-block counts -> exclusive scan -> per-block ranks by warp ballots: the
// order inside every category is the input order (deterministic, no atomics).
// n: the owned count, or with dn the device one (*dn; n = capacity).
constexpr int MIG_T = 256;

__device__ __forceinline__ int mig_cat(double px, double lo, double hi) {
    return px < lo ? 1 : (px >= hi ? 2 : 0);
}

__global__ void __launch_bounds__(MIG_T) k_migrate_count(const double *__restrict__ x, int64_t n, const int64_t *dn,
                                                         double lo, double hi, int32_t *__restrict__ bc, int64_t nblk) {
    __shared__ int sc[3];
    if (threadIdx.x < 3) sc[threadIdx.x] = 0;
    __syncthreads();
    const int64_t i = (int64_t)blockIdx.x * MIG_T + threadIdx.x;
    const int c = i < (dn ? *dn : n) ? mig_cat(x[i], lo, hi) : -1;
#pragma unroll
    for (int cc = 0; cc < 3; cc++) {
        const unsigned m = __ballot_sync(0xffffffffu, c == cc);
        if ((threadIdx.x & 31) == 0 && m) atomicAdd(&sc[cc], __popc(m));
    }
    __syncthreads();
    if (threadIdx.x < 3) bc[threadIdx.x * nblk + blockIdx.x] = sc[threadIdx.x];
}

__global__ void __launch_bounds__(MIG_T) k_migrate_scatter(const double *__restrict__ x, const double *__restrict__ y,
                                                           const int32_t *__restrict__ gid,
                                                           const double *__restrict__ dp, int64_t n,
                                                           const int64_t *dn, double lo, double hi,
                                                           const int32_t *__restrict__ off, int64_t nblk,
                                                           double *keep, double *out_lo, double *out_hi, int64_t cap,
                                                           unsigned long long *c0, unsigned long long *c1,
                                                           unsigned long long *c2) {
    __shared__ int wc[3][MIG_T / 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t i = (int64_t)blockIdx.x * MIG_T + threadIdx.x;
    const int c = i < (dn ? *dn : n) ? mig_cat(x[i], lo, hi) : -1;
    int rank = 0;
#pragma unroll
    for (int cc = 0; cc < 3; cc++) {
        const unsigned m = __ballot_sync(0xffffffffu, c == cc);
        if (c == cc) rank = __popc(m & ((1u << lane) - 1u));
        if (lane == 0) wc[cc][w] = __popc(m);
    }
    __syncthreads();
    if (c >= 0) {
        for (int ww = 0; ww < w; ww++) rank += wc[c][ww];
        const int64_t pos = (int64_t)(off[c * nblk + blockIdx.x] - off[c * nblk]) + rank;
        double *dst = c == 0 ? keep : (c == 1 ? out_lo : out_hi);
        const int64_t cc_cap = c == 0 ? n : cap;
        if (pos < cc_cap) {
            dst[pos] = x[i];
            dst[cc_cap + pos] = y[i];
            ((int32_t *)(dst + 2 * cc_cap))[pos] = gid[i];
            dst[3 * cc_cap + pos] = dp ? dp[i] : 0.0;
        }
    }
    if (blockIdx.x == 0 && threadIdx.x < 3) {
        unsigned long long *dcnt = threadIdx.x == 0 ? c0 : (threadIdx.x == 1 ? c1 : c2);
        *dcnt = (unsigned long long)(off[(threadIdx.x + 1) * nblk] - off[threadIdx.x * nblk]);
    }
}

__global__ void k_migrate_unpack(const double *keep, int64_t n, const unsigned long long *cnt, double *x, double *y,
                                 int32_t *gid, double *dp) {
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= (int64_t)cnt[0]) return;
    x[k] = keep[k];
    y[k] = keep[n + k];
    gid[k] = ((const int32_t *)(keep + 2 * n))[k];
    if (dp) dp[k] = keep[3 * n + k];
}

// n: count (host) or capacity with dn (device count, read before anything is written: the
// kept count may be written to the same location, c_kept == dn is allowed)
static tm_status migrate_impl(tm_ctx *ctx, double *x, double *y, int32_t *gid, double *d_prev, int64_t n,
                              const int64_t *dn, double lo, double hi, double *out_lo, double *out_hi, int64_t cap,
                              int64_t *c_kept, int64_t *c_lo, int64_t *c_hi) {
    TM_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
    if (!dn) {
        TM_CUDA_TRY(ctx, cudaMemsetAsync(c_kept, 0, sizeof(int64_t), ctx->stream));
        TM_CUDA_TRY(ctx, cudaMemsetAsync(c_lo, 0, sizeof(int64_t), ctx->stream));
        TM_CUDA_TRY(ctx, cudaMemsetAsync(c_hi, 0, sizeof(int64_t), ctx->stream));
    }
    if (n == 0) return TM_OK;
    const int64_t nblk = (n + MIG_T - 1) / MIG_T;
    if (n > ctx->cap_mig) {
        cudaFree(ctx->mig_keep);
        ctx->mig_keep = nullptr;
        const int64_t c = n + n / 8 + 1024;
        TM_CUDA_TRY(ctx, cudaMalloc(&ctx->mig_keep, 4 * c * sizeof(double)));
        ctx->cap_mig = c;
    }
    if (3 * nblk + 1 > ctx->cap_mig_blk) {
        cudaFree(ctx->mig_cnt);
        cudaFree(ctx->mig_off);
        ctx->mig_cnt = ctx->mig_off = nullptr;
        const int64_t c = 3 * nblk + 1 + 1024;
        TM_CUDA_TRY(ctx, cudaMalloc(&ctx->mig_cnt, c * sizeof(int32_t)));
        TM_CUDA_TRY(ctx, cudaMalloc(&ctx->mig_off, c * sizeof(int32_t)));
        ctx->cap_mig_blk = c;
    }
    const int64_t *src_n = nullptr;
    if (dn) {  // the source count, copied: the kept count may overwrite *dn
        if (!ctx->scratch_n) TM_CUDA_TRY(ctx, cudaMalloc(&ctx->scratch_n, 2 * sizeof(int64_t)));
        TM_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->scratch_n, dn, sizeof(int64_t), cudaMemcpyDeviceToDevice, ctx->stream));
        src_n = ctx->scratch_n;
    }
    tm_status s = ensure_scan_scratch(ctx, 3 * nblk);
    if (s != TM_OK) return s;
    // keep is n-strided: the scatter writes [x | y | gid | d_prev] segments of stride n
    k_migrate_count<<<(unsigned)nblk, MIG_T, 0, ctx->stream>>>(x, n, src_n, lo, hi, ctx->mig_cnt, nblk);
    if ((s = scan_counts(ctx, ctx->mig_cnt, ctx->mig_off, 3 * nblk)) != TM_OK) return s;
    k_migrate_scatter<<<(unsigned)nblk, MIG_T, 0, ctx->stream>>>(
        x, y, gid, d_prev, n, src_n, lo, hi, ctx->mig_off, nblk, ctx->mig_keep, out_lo, out_hi, cap,
        (unsigned long long *)c_kept, (unsigned long long *)c_lo, (unsigned long long *)c_hi);
    k_migrate_unpack<<<(unsigned)nblk, MIG_T, 0, ctx->stream>>>(ctx->mig_keep, n, (const unsigned long long *)c_kept,
                                                                x, y, gid, d_prev);
    return tm_internal_check_launch(ctx, "k_migrate");
}

extern "C" tm_status tm_migrate_pack(tm_ctx *ctx, double *x, double *y, int32_t *gid, double *d_prev,
                                     int64_t n_owned, double strip_lo, double strip_hi, double *out_lo,
                                     double *out_hi, int64_t cap, int64_t *cnt3) {
    if (!ctx) return TM_E_ARG;
    if (!x || !y || !gid || !out_lo || !out_hi || !cnt3 || n_owned < 0 || cap < 0)
        TM_FAIL(ctx, TM_E_ARG, "null argument to tm_migrate_pack");
    return migrate_impl(ctx, x, y, gid, d_prev, n_owned, nullptr, strip_edge(strip_lo), strip_edge(strip_hi), out_lo,
                        out_hi, cap, cnt3, cnt3 + 1, cnt3 + 2);
}

extern "C" tm_status tm_migrate_pack_dc(tm_ctx *ctx, double *x, double *y, int32_t *gid, double *d_prev,
                                        int64_t *d_n_owned, int64_t cap_owned, double strip_lo, double strip_hi,
                                        double *out_lo, double *out_hi, int64_t cap, int64_t *cnt_lo,
                                        int64_t *cnt_hi) {
    if (!ctx) return TM_E_ARG;
    if (!x || !y || !gid || !d_n_owned || !out_lo || !out_hi || !cnt_lo || !cnt_hi || cap_owned < 0 || cap < 0)
        TM_FAIL(ctx, TM_E_ARG, "null argument to tm_migrate_pack_dc");
    return migrate_impl(ctx, x, y, gid, d_prev, cap_owned, d_n_owned, strip_edge(strip_lo), strip_edge(strip_hi),
                        out_lo, out_hi, cap, d_n_owned, cnt_lo, cnt_hi);
}

// Append a received strip message (segments [x | y | gid (| d_prev)] of capacity msg_cap,
// *msg_count entries) after the *d_count points of x/y/gid(/d_prev) (capacity cap), then
// advance *d_count: all on the device (no host sync).  Beyond a capacity nothing is written
// and TM_E_CAPACITY is latched.
__global__ void k_append(double *__restrict__ x, double *__restrict__ y, int32_t *__restrict__ gid,
                         double *__restrict__ dp, const int64_t *d_count, int64_t cap, const double *__restrict__ src,
                         const int64_t *src_count, int64_t src_cap) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t k = *src_count, base = *d_count;
    if (i >= k || i >= src_cap || base + i >= cap) return;
    x[base + i] = src[i];
    y[base + i] = src[src_cap + i];
    gid[base + i] = ((const int32_t *)(src + 2 * src_cap))[i];
    if (dp) dp[base + i] = src[3 * src_cap + i];
}

__global__ void k_append_count(int64_t *d_count, int64_t cap, const int64_t *src_count, int64_t src_cap,
                               DevState *st) {
    const int64_t k = *src_count, base = *d_count;
    if (k > src_cap || base + k > cap) atomicAdd(&st->n_strip_overflow, 1ull);
    *d_count = min(base + min(k, src_cap), cap);
}

extern "C" tm_status tm_append_points(tm_ctx *ctx, double *x, double *y, int32_t *gid, double *d_prev,
                                      int64_t *d_count, int64_t cap, const double *msg, const int64_t *msg_count,
                                      int64_t msg_cap) {
    if (!ctx) return TM_E_ARG;
    if (!x || !y || !gid || !d_count || !msg || !msg_count || cap < 0 || msg_cap < 0)
        TM_FAIL(ctx, TM_E_ARG, "null argument to tm_append_points");
    TM_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
    if (msg_cap > 0)
        k_append<<<(unsigned)((msg_cap + 255) / 256), 256, 0, ctx->stream>>>(x, y, gid, d_prev, d_count, cap, msg,
                                                                          msg_count, msg_cap);
    k_append_count<<<1, 1, 0, ctx->stream>>>(d_count, cap, msg_count, msg_cap, ctx->dst);
    return tm_internal_check_launch(ctx, "k_append");
}

// ============================================================================ NEXT-1: lazy re-triangulation
extern "C" tm_status tm_refresh_positions(tm_ctx *ctx, const double *x, const double *y) {
    if (!ctx) return TM_E_ARG;
    if (!ctx->have_bins) TM_FAIL(ctx, TM_E_STATE, "tm_refresh_positions before tm_grid_bin");
    if (!x || !y) TM_FAIL(ctx, TM_E_ARG, "null x/y");
    if (ctx->dcnt) TM_FAIL(ctx, TM_E_STATE, "tm_refresh_positions on a device-count binning");
    TM_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
    const Grid &g = ctx->grid;
    // the binning's gather with the same permutation: sorted positions and h(p) of the new
    // positions, slots (and so the ELL rows) unchanged
    k_gather_sorted<<<(unsigned)((ctx->n_local + 255) / 256), 256, 0, ctx->stream>>>(
        x, y, ctx->have_gid ? ctx->gids_in : nullptr, ctx->n_local, ctx->perm, g.x0, g.y0, g.x1, g.y1, g, ctx->mu,
        ctx->c, ctx->xs, ctx->ys, ctx->hs, ctx->gids, nullptr);
    return tm_internal_check_launch(ctx, "k_gather_sorted");
}

__global__ void k_retria(const double *__restrict__ x, const double *__restrict__ y, const int32_t *__restrict__ perm,
                         const double *__restrict__ xt, const double *__restrict__ yt,
                         const double *__restrict__ ht, int64_t n, int64_t n_owned, double fac, int32_t *flag) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool big = false;
    if (s < n) {
        const int32_t i = perm[s];
        if (i < n_owned) {
            // movement since the triangulation vs T_retria = fac h(p_tria), as the oracle
            const double ex = csub(x[i], xt[s]), ey = csub(y[i], yt[s]);
            big = sqrt(cadd(cmul(ex, ex), cmul(ey, ey))) > cmul(fac, ht[s]);
        }
    }
    if (__any_sync(0xffffffffu, big) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

extern "C" tm_status tm_retria_check(tm_ctx *ctx, const double *x_new, const double *y_new, int32_t *flag) {
    if (!ctx) return TM_E_ARG;
    if (!x_new || !y_new || !flag) TM_FAIL(ctx, TM_E_ARG, "null argument to tm_retria_check");
    if (!ctx->have_tria) TM_FAIL(ctx, TM_E_STATE, "tm_retria_check before a triangulation with adjacency");
    TM_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
    k_retria<<<(unsigned)((ctx->n_local + 255) / 256), 256, 0, ctx->stream>>>(
        x_new, y_new, ctx->perm, ctx->xs_tria, ctx->ys_tria, ctx->hs_tria, ctx->n_local, ctx->n_owned,
        ctx->p.fac_retria, flag);
    return tm_internal_check_launch(ctx, "k_retria");
}

// ============================================================================ CUDA Graphs
struct tm_graph {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
};

extern "C" tm_status tm_graph_begin(tm_ctx *ctx) {
    if (!ctx) return TM_E_ARG;
    if (ctx->capturing) TM_FAIL(ctx, TM_E_STATE, "tm_graph_begin while capturing");
    TM_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
    if (!ctx->stream) TM_FAIL(ctx, TM_E_ARG, "graph capture needs a non-default stream");
    TM_CUDA_TRY(ctx, cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
    ctx->capturing = true;
    return TM_OK;
}

extern "C" tm_status tm_graph_end(tm_ctx *ctx, tm_graph **out) {
    if (!ctx || !out) return TM_E_ARG;
    if (!ctx->capturing) TM_FAIL(ctx, TM_E_STATE, "tm_graph_end without tm_graph_begin");
    ctx->capturing = false;
    tm_graph *g = new (std::nothrow) tm_graph();
    if (!g) return TM_E_ARG;
    cudaError_t e = cudaStreamEndCapture(ctx->stream, &g->graph);
    if (e == cudaSuccess) e = cudaGraphInstantiate(&g->exec, g->graph, 0);
    if (e != cudaSuccess) {
        if (g->graph) cudaGraphDestroy(g->graph);
        delete g;
        cudaGetLastError();
        TM_FAIL(ctx, TM_E_CUDA, "graph capture failed: %s", cudaGetErrorString(e));
    }
    *out = g;
    return TM_OK;
}

extern "C" tm_status tm_graph_launch(tm_ctx *ctx, tm_graph *g) {
    if (!ctx || !g) return TM_E_ARG;
    TM_CUDA_TRY(ctx, cudaGraphLaunch(g->exec, ctx->stream));
    return TM_OK;
}

extern "C" void tm_graph_destroy(tm_graph *g) {
    if (!g) return;
    if (g->exec) cudaGraphExecDestroy(g->exec);
    if (g->graph) cudaGraphDestroy(g->graph);
    delete g;
}

extern "C" int tm_host_incircle_exact(const double *a, const double *b, const double *c, const double *d) {
    return tmg::incircle_exact(a, b, c, d);
}

extern "C" void tm_host_cramer(const double *A3, const double *B3, double *xy) {
    Line A = {A3[0], A3[1], A3[2]}, B = {B3[0], B3[1], B3[2]};
    cramer(A, B, xy[0], xy[1]);
}

extern "C" double tm_host_bilinear(int32_t nx, int32_t ny, double x0, double y0, double x1, double y1,
                                   const double *F, double x, double y) {
    Grid g;
    g.nx = nx; g.ny = ny; g.x0 = x0; g.y0 = y0; g.x1 = x1; g.y1 = y1;
    g.idx = cdiv((double)(nx - 1), csub(x1, x0));
    g.idy = cdiv((double)(ny - 1), csub(y1, y0));
    g.dx = cdiv(csub(x1, x0), (double)(nx - 1));
    g.dy = cdiv(csub(y1, y0), (double)(ny - 1));
    return bilinear(g, F, x, y, PlainLoad());
}

// ============================================================================ S7: strip re-balancing input
// histogram of the owned x over nb equal bins of [x0, x1) (x below x0 in bin 0, at or above x1 in the
// last): integer counts, exact
__global__ void k_x_histogram(const double *__restrict__ x, const int64_t *__restrict__ d_n, int64_t n_host,
                              double x0, double x1, int32_t nb, unsigned long long *__restrict__ hist) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t n = d_n ? d_n[0] : n_host;
    if (i >= n) return;
    int b = (int)floor((x[i] - x0) / (x1 - x0) * (double)nb);
    b = b < 0 ? 0 : (b >= nb ? nb - 1 : b);
    atomicAdd(hist + b, 1ull);
}

extern "C" tm_status tm_x_histogram(tm_ctx *ctx, const double *x, const int64_t *d_n, int64_t cap, double x0,
                                    double x1, int32_t nb, int64_t *hist) {
    if (!ctx) return TM_E_ARG;
    if (!x || !hist || nb < 1 || cap < 0 || !(x1 > x0)) TM_FAIL(ctx, TM_E_ARG, "bad arguments to tm_x_histogram");
    TM_CUDA_TRY(ctx, cudaMemsetAsync(hist, 0, (size_t)nb * sizeof(int64_t), ctx->stream));
    if (cap == 0) return TM_OK;
    k_x_histogram<<<(unsigned)((cap + 255) / 256), 256, 0, ctx->stream>>>(x, d_n, cap, x0, x1, nb,
                                                                         reinterpret_cast<unsigned long long *>(hist));
    return tm_internal_check_launch(ctx, "k_x_histogram");
}
