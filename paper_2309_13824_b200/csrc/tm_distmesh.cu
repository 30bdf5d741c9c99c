// tm_distmesh.cu -- S4b DistMesh truss-force update (§2.2 Eqs.
// spring force P:141-146, size scaling P:150-153 in reading L1/L2, forward
// Euler P:160-163; parallel structure P:619-621) with the S5 treatment fused.
//
// The paper's OpenMP version loops over edges with a reduction for the two
// global sums and `omp atomic` force scatters.  Here the forces are
// a per-point GATHER over the ELL adjacency written by the cell kernel (each
// point sums its own incident edges), so there are no atomics and the result is
// deterministic; the two sums are a fixed-order block-tree reduction.
#include <cuda_runtime.h>

#include "tm_internal.cuh"

using namespace tmg;

namespace {

constexpr int DM_T = 256;
constexpr int DM_U = 4;  // edges gathered per group

__device__ __forceinline__ double mu_at(const Grid &g, const double *mu, double x, double y) {
    return mu ? bilinear(g, mu, x, y, LdgLoad()) : 1.0;
}

// pass 1: per-block partial sums of l^2 and mu~(m)^2 over edges (i,a) with gid_i < gid_a
__global__ void __launch_bounds__(DM_T) k_dm_sums(const double *__restrict__ xs, const double *__restrict__ ys,
                                                  const int32_t *__restrict__ perm, const int32_t *__restrict__ gids,
                                                  const int32_t *__restrict__ adj, const uint8_t *__restrict__ deg,
                                                  int64_t n_local, int64_t n_owned, const int64_t *dcnt, Grid g,
                                                  const double *__restrict__ mu, double *__restrict__ partials) {
    __shared__ double red[2][DM_T / 32];
    int64_t s = (int64_t)blockIdx.x * DM_T + threadIdx.x;
    double l2 = 0.0, m2 = 0.0;
    const int64_t n_live = dcnt ? dcnt[1] : n_local, n_own = dcnt ? dcnt[0] : n_owned;
    if (s < n_live && perm[s] < n_own) {
        const double xi = xs[s], yi = ys[s];
        const int32_t gi = gids[s];
        const int d = deg[s];
        // edges in groups of DM_U: all index and position loads of a group are issued
        // before any arithmetic (memory-level parallelism for the gathers)
        for (int k0 = 0; k0 < d; k0 += DM_U) {
            int a[DM_U];
#pragma unroll
            for (int u = 0; u < DM_U; u++) a[u] = (k0 + u < d) ? adj[(int64_t)(k0 + u) * n_local + s] : s;
            double xa[DM_U], ya[DM_U];
            int32_t ga[DM_U];
#pragma unroll
            for (int u = 0; u < DM_U; u++) {
                xa[u] = __ldg(xs + a[u]);
                ya[u] = __ldg(ys + a[u]);
                ga[u] = __ldg(gids + a[u]);
            }
#pragma unroll
            for (int u = 0; u < DM_U; u++) {
                if (k0 + u < d && gi < ga[u]) {
                    const double dx = xi - xa[u], dy = yi - ya[u];
                    l2 += dx * dx + dy * dy;
                    const double m = mu_at(g, mu, cmul(cadd(xi, xa[u]), 0.5), cmul(cadd(yi, ya[u]), 0.5));
                    m2 += m * m;
                }
            }
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        l2 += __shfl_xor_sync(0xffffffffu, l2, o);
        m2 += __shfl_xor_sync(0xffffffffu, m2, o);
    }
    int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) { red[0][w] = l2; red[1][w] = m2; }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, b = 0.0;
        for (int k = 0; k < DM_T / 32; k++) { a += red[0][k]; b += red[1][k]; }
        partials[2 * blockIdx.x] = a;
        partials[2 * blockIdx.x + 1] = b;
    }
}

// fixed-order final sum of the block partials (one block)
__global__ void __launch_bounds__(DM_T) k_dm_final(const double *__restrict__ partials, int64_t nblk,
                                                   double *__restrict__ sums2) {
    __shared__ double red[2][DM_T];
    double a = 0.0, b = 0.0;
    for (int64_t k = threadIdx.x; k < nblk; k += DM_T) {
        a += partials[2 * k];
        b += partials[2 * k + 1];
    }
    red[0][threadIdx.x] = a;
    red[1][threadIdx.x] = b;
    __syncthreads();
    for (int o = DM_T / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
            red[0][threadIdx.x] += red[0][threadIdx.x + o];
            red[1][threadIdx.x] += red[1][threadIdx.x + o];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        sums2[0] = red[0][0];
        sums2[1] = red[1][0];
    }
}

// pass 2: F_i = Σ_a max(l0 - l, 0) (p_i - p_a)/l, x_hat = p + dt_k F, then S5
__global__ void __launch_bounds__(DM_T) k_dm_step(CellArgs A, const int32_t *__restrict__ adj,
                                                  const uint8_t *__restrict__ deg, const double *__restrict__ sums2,
                                                  const uint8_t *__restrict__ fixed, double fscale, double dt_k) {
    int64_t s = (int64_t)blockIdx.x * DM_T + threadIdx.x;
    if (s >= live_local(A)) return;
    int32_t orig = A.perm[s];
    if (orig >= live_owned(A)) return;
    double fac_mu = sqrt(sums2[0] / sums2[1]);
    double xi = A.xs[s], yi = A.ys[s];
    double Fx = 0.0, Fy = 0.0;
    const int d = deg[s];
    for (int k0 = 0; k0 < d; k0 += DM_U) {  // gathers issued per group (see k_dm_sums)
        int a[DM_U];
#pragma unroll
        for (int u = 0; u < DM_U; u++) a[u] = (k0 + u < d) ? adj[(int64_t)(k0 + u) * A.n_local + s] : (int)s;
        double xa[DM_U], ya[DM_U];
#pragma unroll
        for (int u = 0; u < DM_U; u++) {
            xa[u] = __ldg(A.xs + a[u]);
            ya[u] = __ldg(A.ys + a[u]);
        }
#pragma unroll
        for (int u = 0; u < DM_U; u++) {
            if (k0 + u >= d) continue;
            const double dx = xi - xa[u], dy = yi - ya[u];
            const double l = sqrt(dx * dx + dy * dy);
            const double l0 = mu_at(A.grid, A.mu, cmul(cadd(xi, xa[u]), 0.5), cmul(cadd(yi, ya[u]), 0.5)) * fscale * fac_mu;
            if (l < l0) {
                const double fm = l0 - l;  // spring stiffness k = 1 (L3): only dt*k enters
                Fx += fm * (dx / l);
                Fy += fm * (dy / l);
            }
        }
    }
    double xh = xi, yh = yi;
    if (!(fixed && fixed[orig])) {
        xh = xi + dt_k * Fx;
        yh = yi + dt_k * Fy;
    }
    double qx, qy, dpo;
    int st = treat_point(A.grid, A.phi, A.hs[s], A.h_avg, A.fac_pt, A.fac_geps, A.damping, A.newton_max, xi, yi, xh,
                         yh, qx, qy, dpo, LdgLoad(), A.projection, A.trace_max);
    A.x_out[orig] = qx;
    A.y_out[orig] = qy;
    A.d_prev_out[orig] = dpo;
    A.status[orig] = (int8_t)st;
    if (st & 2) atomicAdd(&A.st->n_fallback, 1ull);
}

}  // namespace

extern "C" tm_status tm_distmesh_sums(tm_ctx *ctx, const int32_t *adj, const uint8_t *deg, double *sums2) {
    if (!ctx) return TM_E_ARG;
    if (!ctx->have_cells) TM_FAIL(ctx, TM_E_STATE, "tm_distmesh_sums before tm_voronoi_delaunay");
    if (!adj || !deg || !sums2) TM_FAIL(ctx, TM_E_ARG, "null argument to tm_distmesh_sums");
    TM_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
    int64_t nblk = (ctx->n_local + DM_T - 1) / DM_T;
    if (2 * nblk > ctx->cap_partials) {  // cap_partials counts doubles (shared with tm_mesh_stats)
        cudaFree(ctx->partials);
        ctx->partials = nullptr;
        TM_CUDA_TRY(ctx, cudaMalloc(&ctx->partials, 2 * nblk * sizeof(double)));
        ctx->cap_partials = 2 * nblk;
    }
    k_dm_sums<<<(unsigned)nblk, DM_T, 0, ctx->stream>>>(ctx->xs, ctx->ys, ctx->perm, ctx->gids, adj, deg,
                                                        ctx->n_local, ctx->n_owned, ctx->dcnt, ctx->grid, ctx->mu,
                                                        ctx->partials);
    k_dm_final<<<1, DM_T, 0, ctx->stream>>>(ctx->partials, nblk, sums2);
    return tm_internal_check_launch(ctx, "k_dm_sums");
}

extern "C" tm_status tm_distmesh_step(tm_ctx *ctx, const int32_t *adj, const uint8_t *deg, const double *sums2,
                                      const uint8_t *fixed, const double *d_prev, double *x_out, double *y_out,
                                      double *d_prev_out, int8_t *status) {
    (void)d_prev;
    if (!ctx) return TM_E_ARG;
    if (!ctx->have_cells) TM_FAIL(ctx, TM_E_STATE, "tm_distmesh_step before tm_voronoi_delaunay");
    if (!adj || !deg || !sums2 || !x_out || !y_out || !d_prev_out || !status)
        TM_FAIL(ctx, TM_E_ARG, "null argument to tm_distmesh_step");
    TM_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
    CellArgs a;
    tm_internal_fill_cell_args(ctx, &a);
    a.x_out = x_out; a.y_out = y_out; a.d_prev_out = d_prev_out; a.status = status;
    int64_t nblk = (ctx->n_local + DM_T - 1) / DM_T;
    k_dm_step<<<(unsigned)nblk, DM_T, 0, ctx->stream>>>(a, adj, deg, sums2, fixed, ctx->p.fscale, ctx->p.dt_k);
    return tm_internal_check_launch(ctx, "k_dm_step");
}
