// tm_setup.cu -- NEXT-4 of SURVEY §8(f): the set-up pipeline before meshing.
//   * geometry grid size and cell categories (§3.2);
//   * contour SDF from a closed clockwise loop of line segments with a segment grid and the
//     outward layer search (§3.1), and the SDF set operations;
//   * point initialisation by Floyd-Steinberg dithering of the expected counts (§3.5)
//     and the projection of outside initial points.
// Readings L47-L48.  Every floating decision uses the canonical uncontracted
// operations (cadd/cmul/..., L25), the same operations in the same order as the oracle.
#include <cuda_runtime.h>
#include <math.h>

#include <algorithm>
#include <vector>

#include "tm_internal.cuh"

using namespace tmg;

namespace {

struct DevBuf {
    void *p = nullptr;
    ~DevBuf() { cudaFree(p); }
};

// geometry grid cell categories: 1 boundary iff |phi~(m)| <= l_diag, else 0 inner iff phi~(m) < 0,
// else 2 outer
__global__ void k_geo_categories(Grid g, const double *__restrict__ phi, int32_t nxg, int32_t nyg, double dx,
                                 double dy, double ld, int8_t *__restrict__ cat) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= (int64_t)nxg * nyg) return;
    const int32_t i = (int32_t)(c % nxg), j = (int32_t)(c / nxg);
    const double mx = cadd(g.x0, cmul(cadd((double)i, 0.5), dx)), my = cadd(g.y0, cmul(cadd((double)j, 0.5), dy));
    const double s = bilinear(g, phi, mx, my, LdgLoad());
    cat[c] = (int8_t)(fabs(s) <= ld ? 1 : (s < 0.0 ? 0 : 2));
}

// ---- contour SDF
__device__ __forceinline__ void seg_closest(const double *s, double px, double py, double &d2, double &t_out) {
    const double ax = s[0], ay = s[1], bx = s[2], by = s[3];
    const double ex = csub(bx, ax), ey = csub(by, ay);
    const double t = cdiv(cadd(cmul(csub(px, ax), ex), cmul(csub(py, ay), ey)), cadd(cmul(ex, ex), cmul(ey, ey)));
    double qx, qy, tt;
    if (t <= 0.0) { qx = ax; qy = ay; tt = 0.0; }
    else if (t >= 1.0) { qx = bx; qy = by; tt = 1.0; }
    else { qx = cadd(ax, cmul(t, ex)); qy = cadd(ay, cmul(t, ey)); tt = t; }
    const double dx = csub(px, qx), dy = csub(py, qy);
    d2 = cadd(cmul(dx, dx), cmul(dy, dy));
    t_out = tt;
}

__device__ __forceinline__ void seg_normal(const double *s, double &nx, double &ny) {
    const double ex = csub(s[2], s[0]), ey = csub(s[3], s[1]);
    const double l = sqrt(cadd(cmul(ex, ex), cmul(ey, ey)));
    nx = cdiv(ey, l);
    ny = cdiv(-ex, l);
}

struct SegGrid {
    int32_t nx, ny;
    double x0, y0, dx, dy, dmin;  // cell size, min(dx, dy)
    const int32_t *start, *ids;   // CSR: segments whose bounding box meets the cell
};

// |sdf| by the outward layer search: layers of cells at Chebyshev distance l around
// the node's cell until no segment in a further layer can be closer (lower bound (l-1) dmin,
// strictly: tied segments are still examined); sign from the inward normal, ties by the
// smallest segment index
__global__ void k_contour_sdf(const double *__restrict__ segs, int64_t n_seg, SegGrid G, int32_t nx, int32_t ny,
                              double x0, double y0, double x1, double y1, double *__restrict__ phi) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= (int64_t)nx * ny) return;
    const int32_t i = (int32_t)(c % nx), j = (int32_t)(c / nx);
    const double px = cadd(x0, cmul((double)i, cdiv(csub(x1, x0), (double)(nx - 1))));
    const double py = cadd(y0, cmul((double)j, cdiv(csub(y1, y0), (double)(ny - 1))));
    int ci = (int)floor((px - G.x0) / G.dx), cj = (int)floor((py - G.y0) / G.dy);
    ci = ci < 0 ? 0 : (ci >= G.nx ? G.nx - 1 : ci);
    cj = cj < 0 ? 0 : (cj >= G.ny ? G.ny - 1 : cj);
    int64_t best = -1;
    double bd = 0.0, bt = 0.0;
    const int lmax = max(max(ci, G.nx - 1 - ci), max(cj, G.ny - 1 - cj));
    for (int l = 0; l <= lmax; l++) {
        if (best >= 0 && l >= 1) {
            const double lb = (double)(l - 1) * G.dmin * (1.0 - 1e-12);
            if (lb * lb > bd) break;
        }
        for (int b = cj - l; b <= cj + l; b++) {
            if (b < 0 || b >= G.ny) continue;
            const bool edge_row = b == cj - l || b == cj + l;
            for (int a = ci - l; a <= ci + l; a += edge_row ? 1 : 2 * l) {
                if (a >= 0 && a < G.nx) {
                    const int64_t cc = (int64_t)b * G.nx + a;
                    for (int32_t q = G.start[cc]; q < G.start[cc + 1]; q++) {
                        const int32_t k = G.ids[q];
                        double d2, t;
                        seg_closest(segs + 4 * (int64_t)k, px, py, d2, t);
                        if (best < 0 || d2 < bd || (d2 == bd && k < best)) { best = k; bd = d2; bt = t; }
                    }
                }
                if (l == 0) break;
            }
        }
    }
    if (best < 0) {  // no segment at all
        phi[c] = 0.0;
        return;
    }
    const double *s = segs + 4 * best;
    double nxv, nyv;
    seg_normal(s, nxv, nyv);
    double qx, qy;
    if (bt == 0.0 || bt == 1.0) {
        const int64_t o = bt == 0.0 ? (best + n_seg - 1) % n_seg : (best + 1) % n_seg;
        double mx, my;
        seg_normal(segs + 4 * o, mx, my);
        nxv = cmul(cadd(nxv, mx), 0.5);
        nyv = cmul(cadd(nyv, my), 0.5);
        qx = bt == 0.0 ? s[0] : s[2];
        qy = bt == 0.0 ? s[1] : s[3];
    } else {
        qx = cadd(s[0], cmul(bt, csub(s[2], s[0])));
        qy = cadd(s[1], cmul(bt, csub(s[3], s[1])));
    }
    const double d = sqrt(bd);
    const double side = cadd(cmul(csub(px, qx), nxv), cmul(csub(py, qy), nyv));
    phi[c] = side > 0.0 ? -d : d;
}

__global__ void k_density(const double *__restrict__ mu, int64_t n, double *__restrict__ rho) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) rho[i] = cdiv(1.0, cmul(mu[i], mu[i]));  // Eq. density sizing relationship
}

__global__ void k_sdf_combine(int op, const double *__restrict__ a, const double *__restrict__ b, int64_t n,
                              double *__restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double u = a[i], v = b[i];
    out[i] = op == 0 ? fmin(u, v) : (op == 1 ? fmax(u, -v) : fmax(u, v));
}

// ---- point initialisation
__global__ void k_cell_rho(Grid g, const double *__restrict__ phi, const double *__restrict__ rho, int32_t nxg,
                           int32_t nyg, double dx, double dy, double *__restrict__ out_phi, double *__restrict__ out_rho) {
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= (int64_t)nxg * nyg) return;
    const int32_t i = (int32_t)(c % nxg), j = (int32_t)(c / nxg);
    const double mx = cadd(g.x0, cmul(cadd((double)i, 0.5), dx)), my = cadd(g.y0, cmul(cadd((double)j, 0.5), dy));
    out_phi[c] = bilinear(g, phi, mx, my, LdgLoad());
    out_rho[c] = rho ? bilinear(g, rho, mx, my, LdgLoad()) : 1.0;
}

__device__ __forceinline__ double u01(uint64_t seed, uint64_t k, int comp) {
    uint64_t z = seed + (2u * k + (uint64_t)comp + 1u) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z = z ^ (z >> 31);
    return cmul((double)(z >> 11), 1.1102230246251565e-16);
}

// point k of the loop order: its cell by binary search over the exclusive prefix of the counts
// (cells in the loop order), then the cell-uniform position and, outside the tolerance, the
// projection onto the boundary (the treatment's 2x2 damped Newton, P:402 -> P:575-605)
__global__ void k_init_points(int64_t n_pts, const int64_t *__restrict__ off, int64_t n_cells,
                              const int32_t *__restrict__ cell_of_rank, Grid g, const double *__restrict__ phi,
                              const double *__restrict__ mu, double c, double h_avg, double fac_geps, double damping,
                              int newton_max, int32_t nxg, double dx, double dy, uint64_t seed,
                              double *__restrict__ x, double *__restrict__ y) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n_pts) return;
    int64_t lo = 0, hi = n_cells - 1;  // last rank r with off[r] <= k
    while (lo < hi) {
        const int64_t mid = (lo + hi + 1) >> 1;
        if (off[mid] <= k) lo = mid; else hi = mid - 1;
    }
    const int32_t cc = cell_of_rank[lo];
    const int32_t i = cc % nxg, j = cc / nxg;
    const double cx0 = cadd(g.x0, cmul((double)i, dx)), cy0 = cadd(g.y0, cmul((double)j, dy));
    double px = cadd(cx0, cmul(u01(seed, (uint64_t)k, 0), dx));
    double py = cadd(cy0, cmul(u01(seed, (uint64_t)k, 1), dy));
    const double h = mu ? cmul(c, bilinear(g, mu, px, py, LdgLoad())) : c;
    const double hm = h < h_avg ? h : h_avg;
    const double geps = cmul(fac_geps, hm);
    if (bilinear(g, phi, px, py, LdgLoad()) > geps) {
        const ProjResult r =
            newton_project(g, phi, px, py, geps, cmul(1.4901161193847656e-08, hm), damping, newton_max, LdgLoad());
        if (r.ok) {
            px = r.x;
            py = r.y;
        }
    }
    x[k] = px;
    y[k] = py;
}

}  // namespace

extern "C" void tm_geometry_grid_dims(int64_t n_total, double n_opt, int32_t fac_grid, double x0, double y0,
                                      double x1, double y1, int32_t *nx, int32_t *ny) {
    const double lx = x1 - x0, ly = y1 - y0;
    const double lam = sqrt((double)n_total / (n_opt * (lx * ly)));
    *nx = fac_grid * (int32_t)ceil(lam * lx);
    *ny = fac_grid * (int32_t)ceil(lam * ly);
}

extern "C" tm_status tm_geometry_categories(tm_ctx *ctx, int32_t nxg, int32_t nyg, int8_t *cat) {
    if (!ctx) return TM_E_ARG;
    if (!ctx->have_domain) TM_FAIL(ctx, TM_E_STATE, "tm_geometry_categories before tm_set_domain");
    if (nxg < 1 || nyg < 1 || !cat) TM_FAIL(ctx, TM_E_ARG, "bad geometry grid %dx%d", nxg, nyg);
    const Grid &g = ctx->grid;
    const double dx = cdiv(csub(g.x1, g.x0), (double)nxg), dy = cdiv(csub(g.y1, g.y0), (double)nyg);
    const double ld = sqrt(cadd(cmul(dx, dx), cmul(dy, dy)));
    const int64_t n = (int64_t)nxg * nyg;
    k_geo_categories<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(g, ctx->phi, nxg, nyg, dx, dy, ld, cat);
    return tm_internal_check_launch(ctx, "k_geo_categories");
}

extern "C" tm_status tm_contour_sdf(tm_ctx *ctx, const double *segs, int64_t n_seg, int32_t nx, int32_t ny, double x0,
                                    double y0, double x1, double y1, double *phi) {
    if (!ctx) return TM_E_ARG;
    if (ctx->capturing) TM_FAIL(ctx, TM_E_STATE, "tm_contour_sdf while capturing a graph");
    if (!segs || n_seg < 3 || nx < 2 || ny < 2 || !phi || !(x1 > x0) || !(y1 > y0) || n_seg >= (int64_t)INT32_MAX)
        TM_FAIL(ctx, TM_E_ARG, "bad arguments to tm_contour_sdf");
    TM_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
    // segment grid (host; the loop has few segments): n = ceil(L / mean segment length)
    std::vector<double> hs((size_t)n_seg * 4);
    TM_CUDA_TRY(ctx, cudaMemcpyAsync(hs.data(), segs, hs.size() * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    TM_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    double bx0 = x0, by0 = y0, bx1 = x1, by1 = y1, lsum = 0.0;
    for (int64_t k = 0; k < n_seg; k++) {
        const double *s = &hs[4 * k];
        bx0 = std::min(bx0, std::min(s[0], s[2])); bx1 = std::max(bx1, std::max(s[0], s[2]));
        by0 = std::min(by0, std::min(s[1], s[3])); by1 = std::max(by1, std::max(s[1], s[3]));
        lsum += sqrt((s[2] - s[0]) * (s[2] - s[0]) + (s[3] - s[1]) * (s[3] - s[1]));
    }
    const double lbar = lsum / (double)n_seg;
    if (!(lbar > 0.0)) TM_FAIL(ctx, TM_E_ARG, "degenerate contour");
    SegGrid G;
    G.nx = std::max(1, std::min(4096, (int)ceil((bx1 - bx0) / lbar)));
    G.ny = std::max(1, std::min(4096, (int)ceil((by1 - by0) / lbar)));
    G.x0 = bx0; G.y0 = by0;
    G.dx = (bx1 - bx0) / G.nx; G.dy = (by1 - by0) / G.ny;
    G.dmin = std::min(G.dx, G.dy);
    const int64_t ncell = (int64_t)G.nx * G.ny;
    std::vector<int32_t> cnt(ncell + 1, 0);
    auto cell_range = [&](const double *s, int &a0, int &a1, int &b0, int &b1) {
        a0 = (int)floor((std::min(s[0], s[2]) - G.x0) / G.dx); a1 = (int)floor((std::max(s[0], s[2]) - G.x0) / G.dx);
        b0 = (int)floor((std::min(s[1], s[3]) - G.y0) / G.dy); b1 = (int)floor((std::max(s[1], s[3]) - G.y0) / G.dy);
        a0 = std::max(0, std::min(G.nx - 1, a0 - 1)); a1 = std::max(0, std::min(G.nx - 1, a1 + 1));
        b0 = std::max(0, std::min(G.ny - 1, b0 - 1)); b1 = std::max(0, std::min(G.ny - 1, b1 + 1));
    };
    for (int64_t k = 0; k < n_seg; k++) {
        int a0, a1, b0, b1;
        cell_range(&hs[4 * k], a0, a1, b0, b1);
        for (int b = b0; b <= b1; b++)
            for (int a = a0; a <= a1; a++) cnt[(int64_t)b * G.nx + a + 1]++;
    }
    for (int64_t cc = 0; cc < ncell; cc++) cnt[cc + 1] += cnt[cc];
    std::vector<int32_t> ids(cnt[ncell]), fill(cnt.begin(), cnt.end() - 1);
    for (int64_t k = 0; k < n_seg; k++) {
        int a0, a1, b0, b1;
        cell_range(&hs[4 * k], a0, a1, b0, b1);
        for (int b = b0; b <= b1; b++)
            for (int a = a0; a <= a1; a++) ids[fill[(int64_t)b * G.nx + a]++] = (int32_t)k;
    }
    DevBuf dst, dids;
    TM_CUDA_TRY(ctx, cudaMalloc(&dst.p, cnt.size() * sizeof(int32_t)));
    TM_CUDA_TRY(ctx, cudaMalloc(&dids.p, std::max<size_t>(1, ids.size()) * sizeof(int32_t)));
    TM_CUDA_TRY(ctx, cudaMemcpyAsync(dst.p, cnt.data(), cnt.size() * sizeof(int32_t), cudaMemcpyHostToDevice, ctx->stream));
    if (!ids.empty())
        TM_CUDA_TRY(ctx, cudaMemcpyAsync(dids.p, ids.data(), ids.size() * sizeof(int32_t), cudaMemcpyHostToDevice, ctx->stream));
    G.start = (const int32_t *)dst.p;
    G.ids = (const int32_t *)dids.p;
    const int64_t n = (int64_t)nx * ny;
    k_contour_sdf<<<(unsigned)((n + 127) / 128), 128, 0, ctx->stream>>>(segs, n_seg, G, nx, ny, x0, y0, x1, y1, phi);
    tm_status s = tm_internal_check_launch(ctx, "k_contour_sdf");
    if (s != TM_OK) return s;
    TM_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));  // the segment grid is freed on return
    return TM_OK;
}

extern "C" tm_status tm_sdf_combine(tm_ctx *ctx, int32_t op, const double *a, const double *b, int64_t n, double *out) {
    if (!ctx) return TM_E_ARG;
    if (op < 0 || op > 2 || !a || !b || !out || n < 0) TM_FAIL(ctx, TM_E_ARG, "bad arguments to tm_sdf_combine");
    if (n == 0) return TM_OK;
    k_sdf_combine<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(op, a, b, n, out);
    return tm_internal_check_launch(ctx, "k_sdf_combine");
}

extern "C" tm_status tm_init_points(tm_ctx *ctx, int32_t nxg, int32_t nyg, const int8_t *cat, double n_init,
                                    double eta, uint64_t seed, int32_t *counts, double *x, double *y, int64_t cap,
                                    int64_t *n_out) {
    if (!ctx) return TM_E_ARG;
    if (!ctx->have_domain) TM_FAIL(ctx, TM_E_STATE, "tm_init_points before tm_set_domain");
    if (ctx->capturing) TM_FAIL(ctx, TM_E_STATE, "tm_init_points while capturing a graph");
    if (nxg < 1 || nyg < 1 || !cat || !counts || !n_out || !(n_init >= 0.0) || cap < 0)
        TM_FAIL(ctx, TM_E_ARG, "bad arguments to tm_init_points");
    TM_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
    const Grid &g = ctx->grid;
    const double dx = cdiv(csub(g.x1, g.x0), (double)nxg), dy = cdiv(csub(g.y1, g.y0), (double)nyg);
    const int64_t nc = (int64_t)nxg * nyg;
    DevBuf dphi, drho;
    TM_CUDA_TRY(ctx, cudaMalloc(&dphi.p, nc * sizeof(double)));
    TM_CUDA_TRY(ctx, cudaMalloc(&drho.p, nc * sizeof(double)));
    k_cell_rho<<<(unsigned)((nc + 255) / 256), 256, 0, ctx->stream>>>(g, ctx->phi, ctx->rho, nxg, nyg, dx, dy,
                                                                     (double *)dphi.p, (double *)drho.p);
    tm_status s = tm_internal_check_launch(ctx, "k_cell_rho");
    if (s != TM_OK) return s;
    std::vector<double> hphi(nc), hrho(nc);
    std::vector<int8_t> hcat(nc);
    TM_CUDA_TRY(ctx, cudaMemcpyAsync(hphi.data(), dphi.p, nc * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    TM_CUDA_TRY(ctx, cudaMemcpyAsync(hrho.data(), drho.p, nc * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    TM_CUDA_TRY(ctx, cudaMemcpyAsync(hcat.data(), cat, nc, cudaMemcpyDeviceToHost, ctx->stream));
    TM_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    // Floyd-Steinberg over the valid cells (serial by the method: the residual of a cell is known
    // only after its predecessors; host code): rows from the top, each left to right (L47)
    const double band = cmul(eta, dx < dy ? dx : dy);
    std::vector<uint8_t> valid(nc, 0);
    double S = 0.0;
    for (int32_t j = nyg - 1; j >= 0; j--)
        for (int32_t i = 0; i < nxg; i++) {
            const int64_t c = (int64_t)j * nxg + i;
            valid[c] = hcat[c] == 0 || (hcat[c] == 1 && hphi[c] <= band);
            if (valid[c]) S = cadd(S, hrho[c]);
        }
    std::vector<double> acc(nc, 0.0);
    std::vector<int32_t> hcnt(nc, 0), rank_cell;
    std::vector<int64_t> off;
    int64_t tot = 0;
    for (int32_t j = nyg - 1; j >= 0; j--)
        for (int32_t i = 0; i < nxg; i++) {
            const int64_t c = (int64_t)j * nxg + i;
            if (!valid[c]) continue;
            const double v = cadd(cmul(cdiv(hrho[c], S), n_init), acc[c]);
            double r = floor(cadd(v, 0.5));
            if (r < 0.0) r = 0.0;
            hcnt[c] = (int32_t)r;
            if (hcnt[c] > 0) {
                rank_cell.push_back((int32_t)c);
                off.push_back(tot);
            }
            tot += hcnt[c];
            const double R = csub(v, r);
            const int ni[4] = {i + 1, i - 1, i, i + 1}, nj[4] = {j, j - 1, j - 1, j - 1};
            int m = 0;
            for (int q = 0; q < 4; q++)
                if (ni[q] >= 0 && ni[q] < nxg && nj[q] >= 0 && valid[(int64_t)nj[q] * nxg + ni[q]]) m++;
            if (m == 0) continue;
            const double w = cdiv(R, (double)m);
            for (int q = 0; q < 4; q++)
                if (ni[q] >= 0 && ni[q] < nxg && nj[q] >= 0 && valid[(int64_t)nj[q] * nxg + ni[q]]) {
                    double &a = acc[(int64_t)nj[q] * nxg + ni[q]];
                    a = cadd(a, w);
                }
        }
    TM_CUDA_TRY(ctx, cudaMemcpyAsync(counts, hcnt.data(), nc * sizeof(int32_t), cudaMemcpyHostToDevice, ctx->stream));
    *n_out = tot;
    if (tot > cap || !x || !y || tot == 0) {
        TM_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
        if (x && y && tot > cap) TM_FAIL(ctx, TM_E_CAPACITY, "tm_init_points: %lld points, capacity %lld", (long long)tot,
                               (long long)cap);
        return TM_OK;
    }
    DevBuf doff, drank;
    TM_CUDA_TRY(ctx, cudaMalloc(&doff.p, off.size() * sizeof(int64_t)));
    TM_CUDA_TRY(ctx, cudaMalloc(&drank.p, rank_cell.size() * sizeof(int32_t)));
    TM_CUDA_TRY(ctx, cudaMemcpyAsync(doff.p, off.data(), off.size() * sizeof(int64_t), cudaMemcpyHostToDevice, ctx->stream));
    TM_CUDA_TRY(ctx, cudaMemcpyAsync(drank.p, rank_cell.data(), rank_cell.size() * sizeof(int32_t),
                                     cudaMemcpyHostToDevice, ctx->stream));
    k_init_points<<<(unsigned)((tot + 127) / 128), 128, 0, ctx->stream>>>(
        tot, (const int64_t *)doff.p, (int64_t)off.size(), (const int32_t *)drank.p, g, ctx->phi, ctx->mu, ctx->c,
        ctx->h_avg, ctx->p.fac_geps, ctx->p.newton_damping, ctx->p.newton_max, nxg, dx, dy, seed, x, y);
    if ((s = tm_internal_check_launch(ctx, "k_init_points")) != TM_OK) return s;
    TM_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    return TM_OK;
}

// ---- automatic sizing (App. A)
namespace {

// poles: per boundary point s the farthest circumcentre of its Delaunay triangles (pass 0), then
// the farthest in the half-space opposite to v1 (pass 1); ties by the triangle's (u, v) key.
// Deterministic in two steps: max of the squared distance (bits of a non-negative double order
// as unsigned integers), then the min key among the triangles attaining it.
__global__ void k_pole_circ(int64_t nt, const int32_t *__restrict__ tri, const double *__restrict__ x,
                            const double *__restrict__ y, double *__restrict__ cxy, uint64_t *__restrict__ key,
                            int32_t *__restrict__ su) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nt) return;
    int32_t q0 = tri[3 * t], q1 = tri[3 * t + 1], q2 = tri[3 * t + 2], s;
    if (q0 > q1) { s = q0; q0 = q1; q1 = s; }
    if (q1 > q2) { s = q1; q1 = q2; q2 = s; }
    if (q0 > q1) { s = q0; q0 = q1; q1 = s; }
    const Line A = bisector(csub(x[q1], x[q0]), csub(y[q1], y[q0])), B = bisector(csub(x[q2], x[q0]), csub(y[q2], y[q0]));
    double ox, oy;
    cramer(A, B, ox, oy);
    cxy[2 * t] = cadd(x[q0], ox);
    cxy[2 * t + 1] = cadd(y[q0], oy);
    key[t] = ((uint64_t)(uint32_t)q0 << 32) | (uint32_t)q1;
    su[3 * t] = q0; su[3 * t + 1] = q1; su[3 * t + 2] = q2;
}

__device__ __forceinline__ bool pole_ok(int pass, const double *cxy, int64_t t, const double *x, const double *y,
                                        int32_t s, const int64_t *b1, double &dd) {
    const double ex = csub(cxy[2 * t], x[s]), ey = csub(cxy[2 * t + 1], y[s]);
    dd = cadd(cmul(ex, ex), cmul(ey, ey));
    if (pass == 0) return true;
    const int64_t t1 = b1[s];
    if (t1 < 0) return false;
    const double fx = csub(cxy[2 * t1], x[s]), fy = csub(cxy[2 * t1 + 1], y[s]);
    return cadd(cmul(ex, fx), cmul(ey, fy)) < 0.0;
}

__global__ void k_pole_max(int64_t nt, int pass, const double *__restrict__ cxy, const int32_t *__restrict__ su,
                           const double *__restrict__ x, const double *__restrict__ y, double bx0, double by0,
                           double bx1, double by1, const int64_t *__restrict__ b1, unsigned long long *__restrict__ dmax) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nt) return;
    const double cx = cxy[2 * t], cy = cxy[2 * t + 1];
    if (!(cx > bx0 && cx < bx1 && cy > by0 && cy < by1)) return;
    for (int k = 0; k < 3; k++) {
        const int32_t s = su[3 * t + k];
        double dd;
        if (pole_ok(pass, cxy, t, x, y, s, b1, dd)) atomicMax(dmax + s, (unsigned long long)__double_as_longlong(dd));
    }
}

__global__ void k_pole_arg(int64_t nt, int pass, const double *__restrict__ cxy, const int32_t *__restrict__ su,
                           const uint64_t *__restrict__ key, const double *__restrict__ x, const double *__restrict__ y,
                           double bx0, double by0, double bx1, double by1, const int64_t *__restrict__ b1,
                           const unsigned long long *__restrict__ dmax, unsigned long long *__restrict__ kmin) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nt) return;
    const double cx = cxy[2 * t], cy = cxy[2 * t + 1];
    if (!(cx > bx0 && cx < bx1 && cy > by0 && cy < by1)) return;
    for (int k = 0; k < 3; k++) {
        const int32_t s = su[3 * t + k];
        double dd;
        if (pole_ok(pass, cxy, t, x, y, s, b1, dd) && (unsigned long long)__double_as_longlong(dd) == dmax[s])
            atomicMin(kmin + s, (unsigned long long)key[t]);
    }
}

// triangle index of the winning key per point (keys are unique per triangle)
__global__ void k_pole_pick(int64_t nt, int pass, const double *__restrict__ cxy, const int32_t *__restrict__ su,
                            const uint64_t *__restrict__ key, const double *__restrict__ x, const double *__restrict__ y,
                            double bx0, double by0, double bx1, double by1, const int64_t *__restrict__ b1,
                            const unsigned long long *__restrict__ dmax, const unsigned long long *__restrict__ kmin,
                            int64_t *__restrict__ best) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nt) return;
    const double cx = cxy[2 * t], cy = cxy[2 * t + 1];
    if (!(cx > bx0 && cx < bx1 && cy > by0 && cy < by1)) return;
    for (int k = 0; k < 3; k++) {
        const int32_t s = su[3 * t + k];
        double dd;
        if (pole_ok(pass, cxy, t, x, y, s, b1, dd) && (unsigned long long)__double_as_longlong(dd) == dmax[s] &&
            kmin[s] == key[t])
            best[s] = t;
    }
}

// medial points kept iff >= n_thres OTHER medial points lie strictly within r_nei (brute force)
__global__ void k_medial_trim(int64_t m, const double *__restrict__ mx, const double *__restrict__ my, double r2,
                              int32_t n_thres, uint8_t *__restrict__ keep) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    int64_t c = 0;
    for (int64_t j = 0; j < m; j++) {
        if (j == i) continue;
        const double dx = csub(mx[j], mx[i]), dy = csub(my[j], my[i]);
        c += cadd(cmul(dx, dx), cmul(dy, dy)) < r2 ? 1 : 0;
    }
    keep[i] = c >= n_thres;
}

__global__ void k_lfs(int64_t ns, const double *__restrict__ sx, const double *__restrict__ sy, int64_t nm,
                      const double *__restrict__ mx, const double *__restrict__ my, double *__restrict__ lfs) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= ns) return;
    double b = -1.0;
    for (int64_t j = 0; j < nm; j++) {
        const double dx = csub(mx[j], sx[i]), dy = csub(my[j], sy[i]);
        const double d = sqrt(cadd(cmul(dx, dx), cmul(dy, dy)));
        if (b < 0.0 || d < b) b = d;
    }
    lfs[i] = b;
}

// mu(node) = min_s [K |node - s| + lfs(s)]: the boundary points staged in shared memory by tiles
__global__ void k_sizing(int64_t ns, const double *__restrict__ sx, const double *__restrict__ sy,
                         const double *__restrict__ lfs, double K, int32_t nx, int32_t ny, double x0, double y0,
                         double x1, double y1, double *__restrict__ mu) {
    __shared__ double tx[256], ty[256], tl[256];
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool live = c < (int64_t)nx * ny;
    const int32_t i = live ? (int32_t)(c % nx) : 0, j = live ? (int32_t)(c / nx) : 0;
    const double px = cadd(x0, cmul((double)i, cdiv(csub(x1, x0), (double)(nx - 1))));
    const double py = cadd(y0, cmul((double)j, cdiv(csub(y1, y0), (double)(ny - 1))));
    double b = -1.0;
    for (int64_t base = 0; base < ns; base += 256) {
        __syncthreads();
        const int64_t q = base + threadIdx.x;
        if (threadIdx.x < 256 && q < ns) { tx[threadIdx.x] = sx[q]; ty[threadIdx.x] = sy[q]; tl[threadIdx.x] = lfs[q]; }
        __syncthreads();
        const int m = (int)(ns - base < 256 ? ns - base : 256);
        for (int k = 0; k < m; k++) {  // in boundary-point order: min is order independent anyway
            const double dx = csub(px, tx[k]), dy = csub(py, ty[k]);
            const double v = cadd(cmul(K, sqrt(cadd(cmul(dx, dx), cmul(dy, dy)))), tl[k]);
            if (b < 0.0 || v < b) b = v;
        }
    }
    if (live) mu[c] = b;
}

// |sdf| of the contour at one point (host; the trimming loop is serial by the method)
double host_contour_sdf_abs(const std::vector<double> &S, double px, double py) {
    const int64_t n = (int64_t)S.size() / 4;
    double bd = -1.0;
    for (int64_t k = 0; k < n; k++) {
        const double *s = &S[4 * k];
        const double ex = csub(s[2], s[0]), ey = csub(s[3], s[1]);
        const double t = cdiv(cadd(cmul(csub(px, s[0]), ex), cmul(csub(py, s[1]), ey)), cadd(cmul(ex, ex), cmul(ey, ey)));
        double qx, qy;
        if (t <= 0.0) { qx = s[0]; qy = s[1]; }
        else if (t >= 1.0) { qx = s[2]; qy = s[3]; }
        else { qx = cadd(s[0], cmul(t, ex)); qy = cadd(s[1], cmul(t, ey)); }
        const double dx = csub(px, qx), dy = csub(py, qy);
        const double d2 = cadd(cmul(dx, dx), cmul(dy, dy));
        if (bd < 0.0 || d2 < bd) bd = d2;
    }
    return sqrt(bd);
}

}  // namespace

extern "C" tm_status tm_boundary_points(tm_ctx *ctx, const double *segs, int64_t n_seg, double d_s, double geps_hat,
                                        double *x, double *y, int64_t cap, int64_t *n_out) {
    if (!ctx) return TM_E_ARG;
    if (ctx->capturing) TM_FAIL(ctx, TM_E_STATE, "tm_boundary_points while capturing a graph");
    if (!segs || n_seg < 3 || !(d_s > 0.0) || !(geps_hat >= 0.0) || !n_out || cap < 0)
        TM_FAIL(ctx, TM_E_ARG, "bad arguments to tm_boundary_points");
    TM_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
    std::vector<double> S((size_t)n_seg * 4);
    TM_CUDA_TRY(ctx, cudaMemcpyAsync(S.data(), segs, S.size() * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    TM_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    std::vector<double> px, py;
    for (int64_t k = 0; k < n_seg; k++) {  // App. A: start points, evenly spaced points on long segments
        const double *s = &S[4 * k];
        const double ex = csub(s[2], s[0]), ey = csub(s[3], s[1]);
        const double len = sqrt(cadd(cmul(ex, ex), cmul(ey, ey)));
        px.push_back(s[0]);
        py.push_back(s[1]);
        if (len > d_s) {
            const int64_t m = (int64_t)floor(cdiv(len, d_s)) + 1;
            for (int64_t q = 1; q < m; q++) {
                const double t = cdiv((double)q, (double)m);
                px.push_back(cadd(s[0], cmul(t, ex)));
                py.push_back(cadd(s[1], cmul(t, ey)));
            }
        }
    }
    const int64_t n = (int64_t)px.size();
    std::vector<uint8_t> alive(n, 1);
    const double ds2 = cmul(d_s, d_s);
    for (bool changed = true; changed;) {  // the trimming sweeps (serial by the method)
        changed = false;
        for (int64_t i = 0; i < n; i++) {
            while (alive[i]) {
                int64_t best = -1;
                double bd = 0.0;
                for (int64_t j = 0; j < n; j++) {
                    if (j == i || !alive[j]) continue;
                    const double dx = csub(px[j], px[i]), dy = csub(py[j], py[i]);
                    const double d2 = cadd(cmul(dx, dx), cmul(dy, dy));
                    if (best >= 0 && !(d2 < bd)) continue;
                    const double mx = cmul(cadd(px[i], px[j]), 0.5), my = cmul(cadd(py[i], py[j]), 0.5);
                    if (!(host_contour_sdf_abs(S, mx, my) <= geps_hat)) continue;
                    best = j;
                    bd = d2;
                }
                if (best < 0 || !(bd < ds2)) break;
                px[i] = cmul(cadd(px[i], px[best]), 0.5);
                py[i] = cmul(cadd(py[i], py[best]), 0.5);
                alive[best] = 0;
                changed = true;
            }
        }
    }
    std::vector<double> ox, oy;
    for (int64_t i = 0; i < n; i++)
        if (alive[i]) { ox.push_back(px[i]); oy.push_back(py[i]); }
    *n_out = (int64_t)ox.size();
    if (!x || !y) return TM_OK;
    if ((int64_t)ox.size() > cap) TM_FAIL(ctx, TM_E_CAPACITY, "tm_boundary_points: %lld points, capacity %lld",
                                          (long long)ox.size(), (long long)cap);
    TM_CUDA_TRY(ctx, cudaMemcpyAsync(x, ox.data(), ox.size() * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    TM_CUDA_TRY(ctx, cudaMemcpyAsync(y, oy.data(), oy.size() * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    TM_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    return TM_OK;
}

extern "C" tm_status tm_medial_points(tm_ctx *ctx, const double *x, const double *y, int64_t n, double x0, double y0,
                                      double x1, double y1, double r_nei, int32_t n_thres, double *mx, double *my,
                                      int64_t cap, int64_t *n_out) {
    if (!ctx) return TM_E_ARG;
    if (ctx->capturing) TM_FAIL(ctx, TM_E_STATE, "tm_medial_points while capturing a graph");
    if (!x || !y || n < 3 || !(x1 > x0) || !(y1 > y0) || !mx || !my || !n_out || n >= (int64_t)INT32_MAX / 2)
        TM_FAIL(ctx, TM_E_ARG, "bad arguments to tm_medial_points");
    TM_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
    // the Delaunay triangles of the boundary points by the library's own cell kernel on a second
    // context: phi = -1 on a 2x2 grid over the box, one point's worth of h (c = sqrt(area)) and a
    // large octagon factor, so cells are Voronoi cells clipped by the box only, and keep_tol =
    // +inf: every triangle with its circumcentre strictly inside the box ("an
    // unbounded-cell variant of S2")
    tm_params p2 = ctx->p;
    p2.fac_voro_bound = 1e3;
    p2.keep_tol = 1e300;
    p2.validity = 0;
    p2.flags = TM_F_TWO_LEVEL_BINS;
    tm_ctx *c2 = nullptr;
    tm_status s = tm_create(ctx->device, ctx->stream, &p2, &c2);
    if (s != TM_OK) TM_FAIL(ctx, s, "tm_medial_points: context");
    struct Guard { tm_ctx *c; ~Guard() { tm_destroy(c); } } guard{c2};
    DevBuf dphi, dtri, dnt;
    const double m1[4] = {-1.0, -1.0, -1.0, -1.0};
    TM_CUDA_TRY(ctx, cudaMalloc(&dphi.p, sizeof(m1)));
    TM_CUDA_TRY(ctx, cudaMemcpyAsync(dphi.p, m1, sizeof(m1), cudaMemcpyHostToDevice, ctx->stream));
    tm_fields f = {2, 2, x0, y0, x1, y1, (const double *)dphi.p, nullptr, nullptr};
    if ((s = tm_set_domain(c2, &f, 1, nullptr, nullptr)) != TM_OK) TM_FAIL(ctx, s, "tm_medial_points: %s", c2->err);
    if ((s = tm_grid_bin(c2, x, y, n, n, nullptr)) != TM_OK) TM_FAIL(ctx, s, "tm_medial_points: %s", c2->err);
    const int64_t tcap = 2 * n + 64;
    TM_CUDA_TRY(ctx, cudaMalloc(&dtri.p, tcap * 3 * sizeof(int32_t)));
    TM_CUDA_TRY(ctx, cudaMalloc(&dnt.p, sizeof(int64_t)));
    s = tm_voronoi_delaunay(c2, (int32_t *)dtri.p, tcap, (int64_t *)dnt.p, nullptr, nullptr, nullptr, nullptr, nullptr,
                            nullptr, nullptr);
    if (s == TM_OK) s = tm_sync(c2);
    if (s != TM_OK) TM_FAIL(ctx, s, "tm_medial_points: %s", c2->err);
    int64_t nt = 0;
    TM_CUDA_TRY(ctx, cudaMemcpy(&nt, dnt.p, sizeof(int64_t), cudaMemcpyDeviceToHost));
    DevBuf dc, dk, ds, dmax, dkmin, db1, db2;
    TM_CUDA_TRY(ctx, cudaMalloc(&dc.p, std::max<int64_t>(nt, 1) * 2 * sizeof(double)));
    TM_CUDA_TRY(ctx, cudaMalloc(&dk.p, std::max<int64_t>(nt, 1) * sizeof(uint64_t)));
    TM_CUDA_TRY(ctx, cudaMalloc(&ds.p, std::max<int64_t>(nt, 1) * 3 * sizeof(int32_t)));
    TM_CUDA_TRY(ctx, cudaMalloc(&dmax.p, n * sizeof(unsigned long long)));
    TM_CUDA_TRY(ctx, cudaMalloc(&dkmin.p, n * sizeof(unsigned long long)));
    TM_CUDA_TRY(ctx, cudaMalloc(&db1.p, n * sizeof(int64_t)));
    TM_CUDA_TRY(ctx, cudaMalloc(&db2.p, n * sizeof(int64_t)));
    const unsigned gt = (unsigned)((std::max<int64_t>(nt, 1) + 255) / 256);
    auto *cxy = (double *)dc.p;
    auto *key = (uint64_t *)dk.p;
    auto *su = (int32_t *)ds.p;
    if (nt > 0) k_pole_circ<<<gt, 256, 0, ctx->stream>>>(nt, (const int32_t *)dtri.p, x, y, cxy, key, su);
    int64_t *bb[2] = {(int64_t *)db1.p, (int64_t *)db2.p};
    for (int pass = 0; pass < 2; pass++) {
        TM_CUDA_TRY(ctx, cudaMemsetAsync(dmax.p, 0, n * sizeof(unsigned long long), ctx->stream));
        TM_CUDA_TRY(ctx, cudaMemsetAsync(dkmin.p, 0xff, n * sizeof(unsigned long long), ctx->stream));
        TM_CUDA_TRY(ctx, cudaMemsetAsync(bb[pass], 0xff, n * sizeof(int64_t), ctx->stream));
        if (nt > 0) {
            k_pole_max<<<gt, 256, 0, ctx->stream>>>(nt, pass, cxy, su, x, y, x0, y0, x1, y1, bb[0],
                                                    (unsigned long long *)dmax.p);
            k_pole_arg<<<gt, 256, 0, ctx->stream>>>(nt, pass, cxy, su, key, x, y, x0, y0, x1, y1, bb[0],
                                                    (const unsigned long long *)dmax.p, (unsigned long long *)dkmin.p);
            k_pole_pick<<<gt, 256, 0, ctx->stream>>>(nt, pass, cxy, su, key, x, y, x0, y0, x1, y1, bb[0],
                                                     (const unsigned long long *)dmax.p,
                                                     (const unsigned long long *)dkmin.p, bb[pass]);
        }
        if ((s = tm_internal_check_launch(ctx, "k_pole")) != TM_OK) return s;
    }
    // gather v1, v2 per boundary point in order (host: a compaction of 2n candidates)
    std::vector<int64_t> h1(n), h2(n);
    std::vector<double> hc(2 * std::max<int64_t>(nt, 1));
    TM_CUDA_TRY(ctx, cudaMemcpyAsync(h1.data(), bb[0], n * sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    TM_CUDA_TRY(ctx, cudaMemcpyAsync(h2.data(), bb[1], n * sizeof(int64_t), cudaMemcpyDeviceToHost, ctx->stream));
    if (nt > 0) TM_CUDA_TRY(ctx, cudaMemcpyAsync(hc.data(), cxy, nt * 2 * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    TM_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    std::vector<double> vx, vy;
    for (int64_t i = 0; i < n; i++) {
        if (h1[i] >= 0) { vx.push_back(hc[2 * h1[i]]); vy.push_back(hc[2 * h1[i] + 1]); }
        if (h2[i] >= 0) { vx.push_back(hc[2 * h2[i]]); vy.push_back(hc[2 * h2[i] + 1]); }
    }
    const int64_t m = (int64_t)vx.size();
    int64_t kept = 0;
    if (m > 0) {
        DevBuf dvx, dvy, dkeep;
        TM_CUDA_TRY(ctx, cudaMalloc(&dvx.p, m * sizeof(double)));
        TM_CUDA_TRY(ctx, cudaMalloc(&dvy.p, m * sizeof(double)));
        TM_CUDA_TRY(ctx, cudaMalloc(&dkeep.p, m));
        TM_CUDA_TRY(ctx, cudaMemcpyAsync(dvx.p, vx.data(), m * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        TM_CUDA_TRY(ctx, cudaMemcpyAsync(dvy.p, vy.data(), m * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        k_medial_trim<<<(unsigned)((m + 255) / 256), 256, 0, ctx->stream>>>(m, (const double *)dvx.p, (const double *)dvy.p,
                                                                           cmul(r_nei, r_nei), n_thres, (uint8_t *)dkeep.p);
        if ((s = tm_internal_check_launch(ctx, "k_medial_trim")) != TM_OK) return s;
        std::vector<uint8_t> hk(m);
        TM_CUDA_TRY(ctx, cudaMemcpyAsync(hk.data(), dkeep.p, m, cudaMemcpyDeviceToHost, ctx->stream));
        TM_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
        std::vector<double> kx, ky;
        for (int64_t i = 0; i < m; i++)
            if (hk[i]) { kx.push_back(vx[i]); ky.push_back(vy[i]); }
        kept = (int64_t)kx.size();
        if (kept > cap) TM_FAIL(ctx, TM_E_CAPACITY, "tm_medial_points: %lld points, capacity %lld", (long long)kept,
                                (long long)cap);
        if (kept > 0) {
            TM_CUDA_TRY(ctx, cudaMemcpyAsync(mx, kx.data(), kept * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
            TM_CUDA_TRY(ctx, cudaMemcpyAsync(my, ky.data(), kept * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        }
        TM_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    }
    *n_out = kept;
    return TM_OK;
}

extern "C" tm_status tm_sizing_field(tm_ctx *ctx, const double *sx, const double *sy, int64_t ns, const double *mx,
                                     const double *my, int64_t nm, double K, int32_t nx, int32_t ny, double x0,
                                     double y0, double x1, double y1, double *mu, double *lfs) {
    if (!ctx) return TM_E_ARG;
    if (!sx || !sy || ns < 1 || !mx || !my || nm < 1 || nx < 2 || ny < 2 || !mu || !lfs || !(K >= 0.0))
        TM_FAIL(ctx, TM_E_ARG, "bad arguments to tm_sizing_field");
    k_lfs<<<(unsigned)((ns + 255) / 256), 256, 0, ctx->stream>>>(ns, sx, sy, nm, mx, my, lfs);
    const int64_t nn = (int64_t)nx * ny;
    k_sizing<<<(unsigned)((nn + 255) / 256), 256, 0, ctx->stream>>>(ns, sx, sy, lfs, K, nx, ny, x0, y0, x1, y1, mu);
    return tm_internal_check_launch(ctx, "k_sizing");
}

extern "C" tm_status tm_density_from_sizing(tm_ctx *ctx, const double *mu, int64_t n, double *rho) {
    if (!ctx) return TM_E_ARG;
    if (!mu || !rho || n < 0) TM_FAIL(ctx, TM_E_ARG, "bad arguments to tm_density_from_sizing");
    if (n == 0) return TM_OK;
    k_density<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(mu, n, rho);
    return tm_internal_check_launch(ctx, "k_density");
}

// ---- ADF quadtrees on the boundary geometry cells (after Frisken et al.; reading L48)
namespace {

struct AdfNode {
    double x0, y0, x1, y1, f[4];  // bounds and the exact SDF at the corners (f00, f10, f01, f11)
    int32_t child;                 // first of 4 consecutive children, or -1 (leaf)
    int32_t pad;
};

// exact SDF of the contour at one point: brute force over the segments, the same operations and
// tie rule (smallest segment index) as the oracle's or_contour_sdf_point
__device__ double contour_sdf_bf(const double *__restrict__ segs, int64_t n_seg, double px, double py) {
    int64_t best = -1;
    double bd = 0.0, bt = 0.0;
    for (int64_t k = 0; k < n_seg; k++) {
        double d2, t;
        seg_closest(segs + 4 * k, px, py, d2, t);
        if (best < 0 || d2 < bd) { best = k; bd = d2; bt = t; }
    }
    const double *s = segs + 4 * best;
    double nxv, nyv;
    seg_normal(s, nxv, nyv);
    double qx, qy;
    if (bt == 0.0 || bt == 1.0) {
        const int64_t o = bt == 0.0 ? (best + n_seg - 1) % n_seg : (best + 1) % n_seg;
        double mx, my;
        seg_normal(segs + 4 * o, mx, my);
        nxv = cmul(cadd(nxv, mx), 0.5);
        nyv = cmul(cadd(nyv, my), 0.5);
        qx = bt == 0.0 ? s[0] : s[2];
        qy = bt == 0.0 ? s[1] : s[3];
    } else {
        qx = cadd(s[0], cmul(bt, csub(s[2], s[0])));
        qy = cadd(s[1], cmul(bt, csub(s[3], s[1])));
    }
    const double d = sqrt(bd);
    return cadd(cmul(csub(px, qx), nxv), cmul(csub(py, qy), nyv)) > 0.0 ? -d : d;
}

__device__ __forceinline__ double adf_lerp2(const double *f, double s, double t) {
    return clerp(clerp(f[0], f[1], s), clerp(f[2], f[3], s), t);
}

__device__ void adf_fill(AdfNode &d, double x0, double y0, double x1, double y1, const double *segs, int64_t ns) {
    d.x0 = x0; d.y0 = y0; d.x1 = x1; d.y1 = y1; d.child = -1; d.pad = 0;
    d.f[0] = contour_sdf_bf(segs, ns, x0, y0);
    d.f[1] = contour_sdf_bf(segs, ns, x1, y0);
    d.f[2] = contour_sdf_bf(segs, ns, x0, y1);
    d.f[3] = contour_sdf_bf(segs, ns, x1, y1);
}

// one thread per boundary cell, depth-first with an explicit stack; nodes from a pool (a node
// beyond the capacity is counted but not written: the host rebuilds with the exact size)
__global__ void k_adf_build(int32_t nxg, int32_t nyg, const int8_t *__restrict__ cat, Grid g,
                            const double *__restrict__ mu, double c, double h_avg, double fac_geps, double dx,
                            double dy, const double *__restrict__ segs, int64_t n_seg, double fac_etol, double fac_pt,
                            int max_depth, AdfNode *__restrict__ pool, int64_t cap,
                            unsigned long long *__restrict__ count, int32_t *__restrict__ root) {
    const int64_t cc = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (cc >= (int64_t)nxg * nyg) return;
    root[cc] = -1;
    if (cat[cc] != 1) return;
    const int32_t i = (int32_t)(cc % nxg), j = (int32_t)(cc / nxg);
    const double mx = cadd(g.x0, cmul(cadd((double)i, 0.5), dx)), my = cadd(g.y0, cmul(cadd((double)j, 0.5), dy));
    const double h = mu ? cmul(c, bilinear(g, mu, mx, my, LdgLoad())) : c;
    const double etol = cmul(cmul(fac_etol, cmul(fac_geps, h < h_avg ? h : h_avg)), fac_pt);
    const unsigned long long r = atomicAdd(count, 1ull);
    if ((int64_t)r >= cap) return;
    AdfNode nd;
    adf_fill(nd, cadd(g.x0, cmul((double)i, dx)), cadd(g.y0, cmul((double)j, dy)),
             cadd(g.x0, cmul((double)(i + 1), dx)), cadd(g.y0, cmul((double)(j + 1), dy)), segs, n_seg);
    pool[r] = nd;
    root[cc] = (int32_t)r;
    int64_t stk[64];
    int8_t dep[64];
    int sp = 0;
    stk[sp] = (int64_t)r;
    dep[sp++] = 0;
    while (sp > 0) {
        const int64_t k = stk[--sp];
        const int depth = dep[sp];
        if (depth >= max_depth) continue;
        const AdfNode d = pool[k];
        const double xm = cmul(cadd(d.x0, d.x1), 0.5), ym = cmul(cadd(d.y0, d.y1), 0.5);
        const double px[5] = {xm, xm, d.x0, d.x1, xm}, py[5] = {d.y0, d.y1, ym, ym, ym};
        const double ps[5] = {0.5, 0.5, 0.0, 1.0, 0.5}, pt[5] = {0.0, 1.0, 0.5, 0.5, 0.5};
        double err = 0.0;
        for (int q = 0; q < 5; q++) {
            const double e = fabs(csub(adf_lerp2(d.f, ps[q], pt[q]), contour_sdf_bf(segs, n_seg, px[q], py[q])));
            if (e > err) err = e;
        }
        if (!(err > etol)) continue;
        const unsigned long long c0 = atomicAdd(count, 4ull);
        if ((int64_t)c0 + 4 > cap) continue;
        AdfNode ch;
        adf_fill(ch, d.x0, d.y0, xm, ym, segs, n_seg); pool[c0] = ch;
        adf_fill(ch, xm, d.y0, d.x1, ym, segs, n_seg); pool[c0 + 1] = ch;
        adf_fill(ch, d.x0, ym, xm, d.y1, segs, n_seg); pool[c0 + 2] = ch;
        adf_fill(ch, xm, ym, d.x1, d.y1, segs, n_seg); pool[c0 + 3] = ch;
        pool[k].child = (int32_t)c0;
        for (int q = 3; q >= 0; q--) {
            stk[sp] = (int64_t)c0 + q;
            dep[sp++] = (int8_t)(depth + 1);
        }
    }
}

__global__ void k_adf_eval(int64_t n, const double *__restrict__ x, const double *__restrict__ y, int32_t nxg,
                           int32_t nyg, double x0, double y0, double dx, double dy, const AdfNode *__restrict__ pool,
                           const int32_t *__restrict__ root, double *__restrict__ out) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const double px = x[p], py = y[p];
    const int i = (int)floor(cdiv(csub(px, x0), dx)), j = (int)floor(cdiv(csub(py, y0), dy));
    double v = __longlong_as_double(0x7ff8000000000000ll);  // NaN: not a boundary cell
    if (i >= 0 && j >= 0 && i < nxg && j < nyg) {
        int64_t k = root[(int64_t)j * nxg + i];
        if (k >= 0) {
            while (pool[k].child >= 0) {
                const AdfNode &d = pool[k];
                const double xm = cmul(cadd(d.x0, d.x1), 0.5), ym = cmul(cadd(d.y0, d.y1), 0.5);
                k = d.child + (px >= xm ? 1 : 0) + (py >= ym ? 2 : 0);
            }
            const AdfNode &d = pool[k];
            v = adf_lerp2(d.f, cdiv(csub(px, d.x0), csub(d.x1, d.x0)), cdiv(csub(py, d.y0), csub(d.y1, d.y0)));
        }
    }
    out[p] = v;
}

__global__ void k_adf_leaves(int64_t n, const AdfNode *__restrict__ pool, unsigned long long *__restrict__ leaves) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool leaf = k < n && pool[k].child < 0;
    const unsigned b = __ballot_sync(0xffffffffu, leaf);
    if ((threadIdx.x & 31) == 0 && b) atomicAdd(leaves, (unsigned long long)__popc(b));
}

}  // namespace

extern "C" tm_status tm_adf_build(tm_ctx *ctx, const double *segs, int64_t n_seg, int32_t nxg, int32_t nyg,
                                  const int8_t *cat, double fac_etol, double fac_pt, int32_t max_depth,
                                  int64_t *n_nodes, int64_t *n_leaves) {
    if (!ctx) return TM_E_ARG;
    if (!ctx->have_domain) TM_FAIL(ctx, TM_E_STATE, "tm_adf_build before tm_set_domain");
    if (ctx->capturing) TM_FAIL(ctx, TM_E_STATE, "tm_adf_build while capturing a graph");
    if (!segs || n_seg < 3 || nxg < 1 || nyg < 1 || !cat || max_depth < 0 || max_depth > 20)
        TM_FAIL(ctx, TM_E_ARG, "bad arguments to tm_adf_build");
    TM_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
    const Grid &g = ctx->grid;
    const double dx = cdiv(csub(g.x1, g.x0), (double)nxg), dy = cdiv(csub(g.y1, g.y0), (double)nyg);
    const int64_t nc = (int64_t)nxg * nyg;
    if (ctx->adf_nxg * (int64_t)ctx->adf_nyg < nc || !ctx->adf_root) {
        cudaFree(ctx->adf_root);
        ctx->adf_root = nullptr;
        TM_CUDA_TRY(ctx, cudaMalloc(&ctx->adf_root, nc * sizeof(int32_t)));
    }
    ctx->adf_nxg = nxg;
    ctx->adf_nyg = nyg;
    DevBuf dcnt;
    TM_CUDA_TRY(ctx, cudaMalloc(&dcnt.p, 2 * sizeof(unsigned long long)));
    // an overflowing build undercounts (the subtrees of unwritten nodes are not explored): grow and
    // rebuild until the whole forest fits
    for (int attempt = 0; attempt < 12; attempt++) {
        if (ctx->adf_cap < 1024) {
            cudaFree(ctx->adf_nodes);
            ctx->adf_nodes = nullptr;
            TM_CUDA_TRY(ctx, cudaMalloc(&ctx->adf_nodes, 65536 * sizeof(AdfNode)));
            ctx->adf_cap = 65536;
        }
        TM_CUDA_TRY(ctx, cudaMemsetAsync(dcnt.p, 0, 2 * sizeof(unsigned long long), ctx->stream));
        k_adf_build<<<(unsigned)((nc + 127) / 128), 128, 0, ctx->stream>>>(
            nxg, nyg, cat, g, ctx->mu, ctx->c, ctx->h_avg, ctx->p.fac_geps, dx, dy, segs, n_seg, fac_etol, fac_pt,
            max_depth, (AdfNode *)ctx->adf_nodes, ctx->adf_cap, (unsigned long long *)dcnt.p, ctx->adf_root);
        tm_status s = tm_internal_check_launch(ctx, "k_adf_build");
        if (s != TM_OK) return s;
        unsigned long long used = 0;
        TM_CUDA_TRY(ctx, cudaMemcpyAsync(&used, dcnt.p, sizeof(used), cudaMemcpyDeviceToHost, ctx->stream));
        TM_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
        if ((int64_t)used <= ctx->adf_cap) {
            ctx->adf_n = (int64_t)used;
            break;
        }
        if (attempt == 11) TM_FAIL(ctx, TM_E_CAPACITY, "tm_adf_build: more than %llu nodes", used);
        cudaFree(ctx->adf_nodes);
        ctx->adf_nodes = nullptr;
        const int64_t cap = 2 * (int64_t)used + 1024;
        TM_CUDA_TRY(ctx, cudaMalloc(&ctx->adf_nodes, cap * sizeof(AdfNode)));
        ctx->adf_cap = cap;
    }
    k_adf_leaves<<<(unsigned)((ctx->adf_n + 255) / 256), 256, 0, ctx->stream>>>(
        ctx->adf_n, (const AdfNode *)ctx->adf_nodes, (unsigned long long *)dcnt.p + 1);
    unsigned long long lv = 0;
    TM_CUDA_TRY(ctx, cudaMemcpyAsync(&lv, (unsigned long long *)dcnt.p + 1, sizeof(lv), cudaMemcpyDeviceToHost,
                                     ctx->stream));
    TM_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    if (n_nodes) *n_nodes = ctx->adf_n;
    if (n_leaves) *n_leaves = (int64_t)lv;
    return TM_OK;
}

extern "C" tm_status tm_adf_eval(tm_ctx *ctx, const double *x, const double *y, int64_t n, double *out) {
    if (!ctx) return TM_E_ARG;
    if (!ctx->adf_nodes || !ctx->adf_root || ctx->adf_nxg < 1) TM_FAIL(ctx, TM_E_STATE, "tm_adf_eval before tm_adf_build");
    if (!x || !y || !out || n < 0) TM_FAIL(ctx, TM_E_ARG, "bad arguments to tm_adf_eval");
    if (n == 0) return TM_OK;
    const Grid &g = ctx->grid;
    const double dx = cdiv(csub(g.x1, g.x0), (double)ctx->adf_nxg), dy = cdiv(csub(g.y1, g.y0), (double)ctx->adf_nyg);
    k_adf_eval<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(n, x, y, ctx->adf_nxg, ctx->adf_nyg, g.x0, g.y0,
                                                                      dx, dy, (const AdfNode *)ctx->adf_nodes,
                                                                      ctx->adf_root, out);
    return tm_internal_check_launch(ctx, "k_adf_eval");
}
