// tm_cells.cu -- S2 bounded Voronoi cells, S3 Delaunay extraction + keep rule,
// fused S4a CVD centroid (uniform fan / adaptive quadrature) and S5 treatment.
//
// A group of G lanes (G = 16: two cells per warp; G = 32 for the retry pass)
// computes one cell C_i = B ∩ Oct_i ∩ Vor(i) (PAPER.md P:100 cell-based approach,
// Fig. 3; octagon bound P:491).  The polygon is a linked ring: every
// vertex stays in the lane that created it (prev/next lane links, free-lane
// allocation), so a clip moves no vertex data between lanes.  Each lane keeps
// the vertex's two lines (incoming/outgoing), its canonical coordinates
// relative to p_i and its filter constant.
//
// Candidates come from rings of leaves of the two-level cell list, nearest
// first by a group-wide select-min, until the next one is at least 2*R_max
// away (reading L11; R_max is re-reduced after every effective clip).  A vertex is cut by j when it is strictly closer to p_j:
//   * point-point vertices: exact incircle sign, by a rigorous floating filter
//     on the stored vertex and exact expansion arithmetic when undecided;
//   * wall vertices (an octagon or box side among the labels): the canonical
//     contraction-free test n.x' > r (reading L25).
// Every vertex coordinate is the canonical Cramer intersection of its lines.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <climits>

#include "tm_cellcore.cuh"

namespace cg = cooperative_groups;
using namespace tmg;

namespace {

constexpr int BLOCK = 128;
#ifndef TM_MINB
#define TM_MINB 1  // min resident blocks per SM for the 16-lane kernel (register cap); tuning knob
#endif


struct VState {
    int la, lb;      // incoming / outgoing line codes (slot >= 0, wall < 0)
    int prev, next;  // ring links (lanes of the group)
    double vx, vy;   // canonical coordinates relative to p_i
    double K;        // filter constant of a point-point vertex, < 0 for wall vertices
};


template <int G>
using Tile = cg::thread_block_tile<G>;

template <int G>
__device__ __forceinline__ float tile_maxf(const Tile<G> &g, float v) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v = fmaxf(v, g.shfl_xor(v, o));
    return v;
}
template <int G>
__device__ __forceinline__ double tile_sum(const Tile<G> &g, double v) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v += g.shfl_xor(v, o);
    return v;
}
template <int G>
__device__ __forceinline__ unsigned long long tile_min_u64(const Tile<G> &g, unsigned long long v) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) {
        unsigned long long w = g.shfl_xor(v, o);
        v = w < v ? w : v;
    }
    return v;
}
template <int G>
__device__ __forceinline__ int tile_isum(const Tile<G> &g, int v) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v += g.shfl_xor(v, o);
    return v;
}


// conservative squared distance bound of a vertex from p_i (float, rounded up)
__device__ __forceinline__ float vertex_r2f(const VState &v) {
    double m1 = fabs(v.vx) + fabs(v.vy);
    double K = v.K > 0.0 ? v.K : 0.0;
    double r2 = fma(v.vx, v.vx, v.vy * v.vy) + K * (2.0 * m1 + K);
    return __double2float_ru(r2 * (1.0 + 1e-12));
}


// Clip the ring by line L (code >= 0: bisector with slot `code`; < 0: wall).
// valid: lane mask of the ring (uniform).  Returns 0 ok, -1 overflow, -2 inconsistent.
template <int G>
__device__ int clip_by(const Tile<G> &g, VState &v, unsigned &valid, int code, const Line &L, const CellGeom &cgm,
                       const CellArgs &A, ClipStats &cs) {
    const int lane = g.thread_rank();
    const bool is_bis = code >= 0;
    const bool act = (valid >> lane) & 1u;
    bool out = false;
    if (act) {
        if (is_bis && v.K >= 0.0) {
            double del = fma(L.nx, v.vx, L.ny * v.vy) - L.r;
            double n1 = fabs(L.nx) + fabs(L.ny);
            double B = n1 * fma(8.0 * EPS, n1, v.K);
            if (del > B)
                out = true;
            else if (del >= -B) {
                double Pi[2] = {cgm.px, cgm.py};
                double Pa[2] = {__ldg(A.xs + v.la), __ldg(A.ys + v.la)};
                double Pb[2] = {__ldg(A.xs + v.lb), __ldg(A.ys + v.lb)};
                double Pj[2] = {__ldg(A.xs + code), __ldg(A.ys + code)};
                int s = incircle_exact(Pi, Pa, Pb, Pj);
                if (s == 0) atomicAdd(&A.st->n_degenerate, 1ull);
                out = s > 0;
                cs.exact++;
            }
        } else {
            out = wall_out(L, v.vx, v.vy);
        }
    }
    const unsigned mask = g.ballot(out);
    if (mask == 0u) return 0;
    if (mask == valid) return -2;
    // run start s: out with prev in; run end e: out with next in
    const bool is_s = out && !((mask >> v.prev) & 1u);
    const bool is_e = out && !((mask >> v.next) & 1u);
    const unsigned sm = g.ballot(is_s), em = g.ballot(is_e);
    if (__popc(sm) != 1 || __popc(em) != 1) return -2;
    const int s = __ffs(sm) - 1, e = __ffs(em) - 1;
    int laneB = e;
    if (__popc(mask) == 1) {
        const unsigned fr = ~valid & (G == 32 ? 0xffffffffu : ((1u << G) - 1u));
        if (fr == 0u) return -1;
        laneB = __ffs(fr) - 1;
    }
    const int ps = g.shfl(v.prev, s), ne = g.shfl(v.next, e);
    const int c2 = g.shfl(v.lb, e);  // B's outgoing line = outgoing line of e
    if (lane == s) {  // A = (line into s, L): the edge ps -> s lies on s's incoming line
        const Line E1 = line_of(v.la, cgm, A);
        double inv = cramer(E1, L, v.vx, v.vy);
        v.K = (is_bis && v.la >= 0) ? pp_filter_K(E1, L, v.vx, v.vy, inv) : -1.0;
        v.lb = code;
        v.prev = ps;
        v.next = laneB;
    } else if (lane == laneB) {  // B = (L, line out of e)
        const Line E2 = line_of(c2, cgm, A);
        double inv = cramer(L, E2, v.vx, v.vy);
        v.K = (is_bis && c2 >= 0) ? pp_filter_K(L, E2, v.vx, v.vy, inv) : -1.0;
        v.la = code;
        v.lb = c2;
        v.prev = s;
        v.next = ne;
    }
    if (lane == ps && lane != s) v.next = s;
    if (lane == ne && lane != laneB) v.prev = laneB;
    valid = (valid & ~mask) | (1u << s) | (1u << laneB);
    cs.clips++;
    return 0;
}

// ascending bitonic sort of the 2G keys (element c*G + lane held as key[c])
template <int G>
__device__ __forceinline__ void bitonic_sort2(const Tile<G> &g, unsigned long long key[2]) {
    const int lane = g.thread_rank();
#pragma unroll
    for (int k = 2; k <= 2 * G; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j == G) {  // partner is the other slot of the same lane
                const bool up = ((lane & k) == 0);  // j == G only when k == 2G: always ascending
                unsigned long long a = key[0], b = key[1];
                unsigned long long mn = a < b ? a : b, mx = a < b ? b : a;
                key[0] = up ? mn : mx;
                key[1] = up ? mx : mn;
            } else {
#pragma unroll
                for (int c = 0; c < 2; c++) {
                    const int e = c * G + lane;
                    const unsigned long long o = g.shfl_xor(key[c], j);
                    const bool up = ((e & k) == 0);
                    const bool lower = (lane & j) == 0;  // e < partner
                    const unsigned long long mn = key[c] < o ? key[c] : o, mx = key[c] < o ? o : key[c];
                    key[c] = (lower == up) ? mn : mx;
                }
            }
        }
    }
}


template <int G>
__device__ __forceinline__ float fresh_R2(const Tile<G> &g, const VState &v, unsigned valid) {
    return tile_maxf<G>(g, ((valid >> g.thread_rank()) & 1u) ? vertex_r2f(v) : 0.0f);
}

// One cell per G-lane group; in the retry pass (M_RETRY) the cells come from the
// overflow list of the G=16 pass and the grid is persistent.
template <int G, int MODE>
__global__ void __launch_bounds__(BLOCK, (G == 16 ? TM_MINB : 1)) k_cells(CellArgs A, int32_t *retry_list, unsigned long long *retry_cnt) {
    constexpr int CPB = BLOCK / G;
    __shared__ int32_t sbuf_all[CPB][2 * G];
    __shared__ double2 ring_smem[CPB][G];  // a finished ring in canonical order (S4a, lane 0)
    cg::thread_block block = cg::this_thread_block();
    Tile<G> g = cg::tiled_partition<G>(block);
    const int lane = g.thread_rank();
    const int gib = threadIdx.x / G;
    int32_t *sbuf = sbuf_all[gib];
    const int64_t nitems = (MODE & M_RETRY) ? (int64_t)*retry_cnt : live_local(A);
    const int64_t stride = (MODE & M_RETRY) ? (int64_t)gridDim.x * CPB : 0;
    for (int64_t item = (int64_t)blockIdx.x * CPB + gib; item < nitems; item += stride) {
        const int64_t cell = (MODE & M_RETRY) ? (int64_t)retry_list[item] : item;
        const int32_t orig = __ldg(A.perm + cell);
        if (orig < live_owned(A)) {
            const double px = __ldg(A.xs + cell), py = __ldg(A.ys + cell);
            const double h = __ldg(A.hs + cell);
            const int32_t gi = __ldg(A.gids + cell);
            const double S = cmul(A.fac_voro, h);
            const double r_oct = cmul(S, COS_PI8);
            const double bx0 = A.grid.x0, by0 = A.grid.y0, bx1 = A.grid.x1, by1 = A.grid.y1;
            ClipStats cs;
            unsigned long long n_cand = 0, nq = 0;

            const CellGeom cgm = {px, py, r_oct, bx0, by0, bx1, by1};
            // ---- initial ring: octagon, vertex k between sides k and k+1
            VState v;
            unsigned valid = 0xffu;
            {
                int k = lane & 7;
                v.la = -1 - k;
                v.lb = -1 - ((k + 1) & 7);
                v.prev = (k + 7) & 7;
                v.next = (k + 1) & 7;
                cramer(wall_line(v.la, px, py, r_oct, bx0, by0, bx1, by1),
                       wall_line(v.lb, px, py, r_oct, bx0, by0, bx1, by1), v.vx, v.vy);
                v.K = -1.0;
            }
            int fail = 0;
            if (csub(px, bx0) < S || csub(bx1, px) < S || csub(py, by0) < S || csub(by1, py) < S) {
                const int box_codes[4] = {-9, -10, -11, -12};
                for (int b = 0; b < 4 && !fail; b++) {
                    Line L = wall_line(box_codes[b], px, py, r_oct, bx0, by0, bx1, by1);
                    fail = clip_by<G>(g, v, valid, box_codes[b], L, cgm, A, cs);
                }
            }
            float R2 = fresh_R2<G>(g, v, valid);
            const double MARG = 1.0 + 1e-9;

            // ---- nearest-first search over the two-level cell list (L11 stopping rule)
            const BinGeom &bg = A.bg;
            int hbx = (int)floor((px - bg.x0) * bg.isx), hby = (int)floor((py - bg.y0) * bg.isy);
            hbx = hbx < 0 ? 0 : (hbx >= bg.nbx ? bg.nbx - 1 : hbx);
            hby = hby < 0 ? 0 : (hby >= bg.nby ? bg.nby - 1 : hby);
            const int rh = __ldg(A.rlev + hby * bg.nbx + hbx);
            const int ux = leaf_coord(px, bg.x0, bg.isx, bg.nbx, rh), uy = leaf_coord(py, bg.y0, bg.isy, bg.nby, rh);
            const int nlx = bg.nbx << rh, nly = bg.nby << rh;
            const double lsx = bg.sx * pow2neg(rh), lsy = bg.sy * pow2neg(rh);
            for (int k = 1; !fail; k++) {
                if (k > 1) {
                    double dl = px - (bg.x0 + (ux - k + 1) * lsx), dr = (bg.x0 + (ux + k) * lsx) - px;
                    double dd = py - (bg.y0 + (uy - k + 1) * lsy), du = (bg.y0 + (uy + k) * lsy) - py;
                    double dmin = fmin(fmin(dl, dr), fmin(dd, du));
                    if (dmin > 0.0) {
                        if (dmin * dmin * (1.0 - 1e-9) >= 4.0 * (double)R2 * MARG) break;
                    }
                    if (ux - k < 0 && uy - k < 0 && ux + k >= nlx && uy + k >= nly) break;
                }
                const int nq_ring = k == 1 ? 9 : 8 * k;
                for (int q0 = 0; q0 < nq_ring && !fail; q0 += G) {
                    // leaf ranges of this chunk of the ring
                    int q = q0 + lane, st = 0, cnt = 0;
                    if (q < nq_ring) {
                        int dx, dy;
                        if (k == 1) { dx = q % 3 - 1; dy = q / 3 - 1; }
                        else ring_bin(k, q, dx, dy);
                        int vx = ux + dx, vy = uy + dy;
                        if (vx >= 0 && vx < nlx && vy >= 0 && vy < nly) {
                            int bx = vx >> rh, by = vy >> rh;
                            int b = by * bg.nbx + bx;
                            int rb = __ldg(A.rlev + b);
                            int off = __ldg(A.leaf_off + b);
                            if (rb >= rh) {
                                int sh = 2 * (rb - rh);
                                int mlo = (int)morton2((uint32_t)(vx - (bx << rh)), (uint32_t)(vy - (by << rh))) << sh;
                                st = __ldg(A.leaf_start + off + mlo);
                                cnt = __ldg(A.leaf_start + off + mlo + (1 << sh)) - st;
                            } else {
                                int d = rh - rb;
                                int Lx = vx >> d, Ly = vy >> d;
                                int rx = min(max(ux, Lx << d), ((Lx + 1) << d) - 1);
                                int ry = min(max(uy, Ly << d), ((Ly + 1) << d) - 1);
                                if (rx == vx && ry == vy) {
                                    int mm = (int)morton2((uint32_t)(Lx - (bx << rb)), (uint32_t)(Ly - (by << rb)));
                                    st = __ldg(A.leaf_start + off + mm);
                                    cnt = __ldg(A.leaf_start + off + mm + 1) - st;
                                }
                            }
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
                    for (int base = 0; base < total && !fail; base += 2 * G) {
                        // stage the window's candidate slots through shared memory
                        for (int t = max(0, base - excl); t < cnt && excl + t < base + 2 * G; t++)
                            sbuf[excl + t - base] = st + t;
                        g.sync();
                        unsigned long long key[2];
#pragma unroll
                        for (int c = 0; c < 2; c++) {
                            const int t = base + c * G + lane;
                            key[c] = ~0ull;
                            if (t < total) {
                                const int j = sbuf[c * G + lane];
                                n_cand++;
                                if (j != (int)cell) {
                                    double dx = __ldg(A.xs + j) - px, dy = __ldg(A.ys + j) - py;
                                    double d2 = dx * dx + dy * dy;
                                    if (dx == 0.0 && dy == 0.0) atomicAdd(&A.st->n_duplicate, 1ull);
                                    if (d2 > 0.0 && d2 < 4.0 * (double)R2 * MARG)
                                        key[c] = ((unsigned long long)__float_as_uint(__double2float_ru(d2)) << 32) |
                                                 (unsigned)j;
                                }
                            }
                        }
                        g.sync();
                        // nearest first: one bitonic sort of the window, keys (d2 rounded up, slot)
                        bitonic_sort2<G>(g, key);
                        for (int r = 0; r < 2 * G; r++) {
                            const unsigned long long kr = g.shfl(r < G ? key[0] : key[1], r & (G - 1));
                            if (kr == ~0ull) break;
                            // keys round d2 up and are sorted: stop when this one is clearly beyond 2 R_max
                            if ((double)__uint_as_float((unsigned)(kr >> 32)) >= 4.0 * (double)R2 * (1.0 + 1e-5)) break;
                            const int j = (int)(kr & 0xffffffffu);
                            const double dx = csub(__ldg(A.xs + j), px), dy = csub(__ldg(A.ys + j), py);
                            if (dx * dx + dy * dy >= 4.0 * (double)R2 * MARG) continue;
                            const unsigned long long c0 = cs.clips;
                            fail = clip_by<G>(g, v, valid, j, bisector(dx, dy), cgm, A, cs);
                            if (fail) break;
                            if (cs.clips != c0) R2 = fresh_R2<G>(g, v, valid);  // R_max only shrinks
                        }
                    }
                }
            }
            if (fail == -1 && !(MODE & M_RETRY)) {
                // more than G vertices: hand the cell to the 32-lane retry pass
                if (lane == 0) {
                    unsigned long long k = atomicAdd(retry_cnt, 1ull);
                    retry_list[k] = (int32_t)cell;
                }
            } else if (fail) {
                if (lane == 0) atomicAdd(fail == -1 ? &A.st->n_overflow : &A.st->n_degenerate, 1ull);
                if ((MODE & M_TREAT) && lane == 0) {
                    A.x_out[orig] = px; A.y_out[orig] = py; A.d_prev_out[orig] = 0.0; A.status[orig] = 2;
                }
                if ((MODE & M_HAT) && lane == 0) { A.x_hat[orig] = px; A.y_hat[orig] = py; }
                if ((MODE & M_ELL) && lane == 0) A.deg[cell] = 0;
            } else {
                const bool active = (valid >> lane) & 1u;
                const int nv = __popc(valid);
                // ---- S3: Delaunay triangles at point-point vertices + keep rule
                bool kept = false;
                int t_own = 0;
                if (MODE & (M_TRI | M_ELL)) {
                    const bool pp = active && v.la >= 0 && v.lb >= 0;
                    bool owned = false;
                    if (pp) {
                        const int32_t ga = __ldg(A.gids + v.la), gb = __ldg(A.gids + v.lb);
                        owned = gi < ga && gi < gb;
                        if (owned) {
                            const int sv = ga < gb ? v.la : v.lb, sw = ga < gb ? v.lb : v.la;
                            kept = keep_tri(A, (int)cell, sv, sw, v.vx, v.vy);
                        } else if (MODE & M_ELL) {
                            // canonical circumcentre relative to the smallest-id vertex
                            int s3[3] = {(int)cell, v.la, v.lb};
                            int32_t g3[3] = {gi, ga, gb};
                            for (int a = 0; a < 2; a++)
                                for (int b = 0; b < 2 - a; b++)
                                    if (g3[b] > g3[b + 1]) {
                                        int32_t tg = g3[b]; g3[b] = g3[b + 1]; g3[b + 1] = tg;
                                        int ts = s3[b]; s3[b] = s3[b + 1]; s3[b + 1] = ts;
                                    }
                            const double uxx = __ldg(A.xs + s3[0]), uyy = __ldg(A.ys + s3[0]);
                            const Line B1 = bisector(csub(__ldg(A.xs + s3[1]), uxx), csub(__ldg(A.ys + s3[1]), uyy));
                            const Line B2 = bisector(csub(__ldg(A.xs + s3[2]), uxx), csub(__ldg(A.ys + s3[2]), uyy));
                            double ox, oy;
                            cramer(B1, B2, ox, oy);
                            kept = keep_tri(A, s3[0], s3[1], s3[2], ox, oy);
                        }
                    }
                    if (MODE & M_TRI) {
                        const bool emit = owned && kept;
                        const unsigned em = g.ballot(emit);
                        t_own = __popc(em);
                        unsigned long long base = 0;
                        if (lane == 0 && em) base = atomicAdd(A.n_tri, (unsigned long long)t_own);
                        base = g.shfl(base, 0);
                        if (emit) {
                            const unsigned long long idx = base + __popc(em & ((1u << lane) - 1u));
                            if ((int64_t)idx < A.tri_cap) {
                                A.tri[3 * idx] = gi;
                                A.tri[3 * idx + 1] = __ldg(A.gids + v.la);
                                A.tri[3 * idx + 2] = __ldg(A.gids + v.lb);
                            } else {
                                atomicAdd(&A.st->n_tri_overflow, 1ull);
                            }
                        }
                    }
                }
                // canonical ring order (from the smallest (incoming, outgoing) line pair, points
                // named by their ids, as k_cells_t and the oracle): the ELL row, the warm-start
                // neighbour list and the centroid sums below all walk the ring in this order, so
                // every output is independent of which kernel computed the cell
                const long long ckey =
                    active ? (((long long)(v.la >= 0 ? __ldg(A.gids + v.la) : v.la) << 32) |
                              (unsigned)(v.lb >= 0 ? __ldg(A.gids + v.lb) : v.lb))
                           : LLONG_MAX;
                const unsigned long long kmin = tile_min_u64<G>(g, (unsigned long long)ckey ^ 0x8000000000000000ull);
                const int cstart =
                    __ffs(g.ballot(active && ((unsigned long long)ckey ^ 0x8000000000000000ull) == kmin)) - 1;
                // ---- DistMesh ELL row: neighbour a (incoming bisector of a vertex) borders a kept triangle
                int ell = 0;
                if (MODE & M_ELL) {
                    const bool kprev = g.shfl((int)kept, v.prev) != 0;
                    const bool nb = active && v.la >= 0 && (kept || kprev);
                    int walk = cstart;
                    for (int q = 0; q < nv; q++) {
                        const bool nbq = g.shfl((int)nb, walk) != 0;
                        const int aq = g.shfl(v.la, walk);
                        if (nbq) {
                            if (lane == 0 && ell < A.adj_stride) A.adj[(int64_t)ell * A.n_local + cell] = aq;
                            ell++;
                        }
                        walk = g.shfl(v.next, walk);
                    }
                    if (lane == 0) {
                        A.deg[cell] = (uint8_t)(ell < A.adj_stride ? ell : A.adj_stride);
                        if (ell > A.adj_stride) atomicAdd(&A.st->n_adj_overflow, 1ull);
                    }
                }
                // ---- warm-start neighbour list for the next launch (ids, canonical ring order,
                // at most TM_NBR: a hint only, the next launch certifies its cells either way)
                {
                    const int32_t nid = A.nbr_by_gid ? gi : orig;
                    if (A.nbr && A.nbr_cnt && nid >= 0 && (int64_t)nid < A.nbr_keys) {
                        int walk = cstart, cnt = 0;
                        for (int q = 0; q < nv; q++) {
                            const int aq = g.shfl(v.la, walk);
                            if (aq >= 0) {
                                if (lane == 0 && cnt < TM_NBR)
                                    A.nbr[(int64_t)nid * TM_NBR + cnt] = A.nbr_by_gid ? __ldg(A.gids + aq) : __ldg(A.perm + aq);
                                cnt++;
                            }
                            walk = g.shfl(v.next, walk);
                        }
                        if (lane == 0) A.nbr_cnt[nid] = (uint8_t)(cnt < TM_NBR ? cnt : TM_NBR);
                    }
                }
                // ---- S4a: centroid of C_i (relative to p_i)
                if (MODE & (M_TREAT | M_HAT)) {
                    // gather the ring in canonical order and let lane 0 sum it sequentially: the
                    // same operations in the same order as k_output_t and the oracle's O4
                    int walk = cstart;
                    double2 *rb = ring_smem[threadIdx.x / G];
                    for (int q = 0; q < nv; q++) {
                        const double wx = g.shfl(v.vx, walk), wy = g.shfl(v.vy, walk);
                        if (lane == 0) rb[q] = make_double2(wx, wy);
                        walk = g.shfl(v.next, walk);
                    }
                    g.sync();
                    double cx = 0.0, cy = 0.0;
                    if (lane == 0)
                        ring_centroid(rb, 1, nv, px, py, h, A.d_prev ? __ldg(A.d_prev + orig) : -1.0, A, cx, cy, nq);
                    g.sync();
                    if ((MODE & M_HAT) && lane == 0) {
                        A.x_hat[orig] = px + cx;
                        A.y_hat[orig] = py + cy;
                    }
                    // ---- S5 fused treatment (Alg. 2: project escaped centroids back)
                    if ((MODE & M_TREAT) && lane == 0) {
                        double qx, qy, dpo;
                        const int s = treat_point(A.grid, A.phi, h, A.h_avg, A.fac_pt, A.fac_geps, A.damping,
                                                  A.newton_max, px, py, px + cx, py + cy, qx, qy, dpo, LdgLoad(),
                                                  A.projection, A.trace_max);
                        A.x_out[orig] = qx;
                        A.y_out[orig] = qy;
                        A.d_prev_out[orig] = dpo;
                        A.status[orig] = (int8_t)s;
                        if (s & 2) atomicAdd(&A.st->n_fallback, 1ull);
                    }
                }
                // ---- O8 work counters (TM_F_COUNT_WORK)
                if (MODE & M_COUNT) {
                    const float R2f = fresh_R2<G>(g, v, valid);
                    const double rad = 2.0 * sqrt((double)R2f);
                    int ncert = 0;
                    const int bxa = max(0, (int)floor((px - rad - bg.x0) * bg.isx));
                    const int bxb = min(bg.nbx - 1, (int)floor((px + rad - bg.x0) * bg.isx));
                    const int bya = max(0, (int)floor((py - rad - bg.y0) * bg.isy));
                    const int byb = min(bg.nby - 1, (int)floor((py + rad - bg.y0) * bg.isy));
                    for (int by = bya; by <= byb; by++) {
                        const int s0 = __ldg(A.leaf_start + __ldg(A.leaf_off + by * bg.nbx + bxa));
                        const int s1 = __ldg(A.leaf_start + __ldg(A.leaf_off + by * bg.nbx + bxb + 1));
                        for (int s = s0 + lane; s < s1; s += G) {
                            const double dx = __ldg(A.xs + s) - px, dy = __ldg(A.ys + s) - py;
                            ncert += (s != (int)cell) && (dx * dx + dy * dy < rad * rad);
                        }
                    }
                    ncert = tile_isum<G>(g, ncert);
                    const int degc = tile_isum<G>(g, active && v.lb >= 0 ? 1 : 0);
                    unsigned long long ex = cs.exact, ca = n_cand, nqs = nq, cl = cs.clips;
                    for (int o = G / 2; o > 0; o >>= 1) {
                        ex += g.shfl_xor(ex, o);
                        ca += g.shfl_xor(ca, o);
                        nqs += g.shfl_xor(nqs, o);
                    }
                    if (lane == 0) {
                        atomicAdd(&A.st->work[0], 1ull);
                        atomicAdd(&A.st->work[1], (unsigned long long)ncert);
                        atomicAdd(&A.st->work[2], (unsigned long long)degc);
                        atomicAdd(&A.st->work[3], (unsigned long long)nv);
                        atomicAdd(&A.st->work[4], (unsigned long long)t_own);
                        atomicAdd(&A.st->work[5], (A.rho == nullptr) ? (unsigned long long)nv : nqs);
                        atomicAdd(&A.st->work[6], (unsigned long long)ell);
                        atomicAdd(&A.st->work[7], ca);
                        atomicAdd(&A.st->work[8], cl);
                        atomicAdd(&A.st->work[9], ex);
                    }
                }
            }
        }
        if (!(MODE & M_RETRY)) break;
    }
}

template <int MODE>
tm_status launch_cells(tm_ctx *ctx, const CellArgs &a) {
    TM_CUDA_TRY(ctx, cudaMemsetAsync(ctx->retry_cnt, 0, sizeof(unsigned long long), ctx->stream));
    tm_status s;
    if (ctx->p.flags & TM_F_GROUP_CELLS) {
        // 16-lane group per cell (two cells per warp)
        constexpr int G = 16;
        const unsigned blocks = (unsigned)((ctx->n_local + (BLOCK / G) - 1) / (BLOCK / G));
        k_cells<G, MODE><<<blocks, BLOCK, 0, ctx->stream>>>(a, ctx->retry_list, ctx->retry_cnt);
        s = tm_internal_check_launch(ctx, "k_cells");
    } else {
        // one thread per cell, polygon ring in shared memory (tm_cells_t.cu)
        s = launch_cells_thread<MODE>(ctx, a);
    }
    if (s != TM_OK) return s;
    // cells that needed more than 16 vertices at some point: persistent 32-lane retry pass
    k_cells<32, MODE | M_RETRY><<<148 * 2, BLOCK, 0, ctx->stream>>>(a, ctx->retry_list, ctx->retry_cnt);
    return tm_internal_check_launch(ctx, "k_cells_retry");
}

template <int BASE>
tm_status dispatch_count(tm_ctx *ctx, const CellArgs &a) {
    if (ctx->p.flags & TM_F_COUNT_WORK) return launch_cells<BASE | M_COUNT>(ctx, a);
    return launch_cells<BASE>(ctx, a);
}

tm_status ensure_retry(tm_ctx *ctx) {
    if (!ctx->retry_cnt) TM_CUDA_TRY(ctx, cudaMalloc(&ctx->retry_cnt, sizeof(unsigned long long)));
    if (ctx->cap_retry >= ctx->n_local) return TM_OK;
    cudaFree(ctx->retry_list);
    ctx->retry_list = nullptr;
    TM_CUDA_TRY(ctx, cudaMalloc(&ctx->retry_list, ctx->cap_points * sizeof(int32_t)));
    ctx->cap_retry = ctx->cap_points;
    return TM_OK;
}

}  // namespace

extern "C" tm_status tm_voronoi_delaunay(tm_ctx *ctx, int32_t *tri, int64_t tri_cap, int64_t *n_tri, int32_t *adj,
                                         uint8_t *deg, const double *d_prev, double *x_out, double *y_out,
                                         double *d_prev_out, int8_t *status) {
    if (!ctx) return TM_E_ARG;
    if (!ctx->have_bins) TM_FAIL(ctx, TM_E_STATE, "tm_voronoi_delaunay before tm_grid_bin");
    if (!tri || !n_tri || tri_cap < 0) TM_FAIL(ctx, TM_E_ARG, "tri/n_tri required");
    if ((adj == nullptr) != (deg == nullptr)) TM_FAIL(ctx, TM_E_ARG, "adj and deg must be given together");
    const bool treat = x_out != nullptr;
    if (treat && (!y_out || !d_prev_out || !status))
        TM_FAIL(ctx, TM_E_ARG, "fused CVD needs x_out,y_out,d_prev_out,status");
    TM_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
    tm_status s = ensure_retry(ctx);
    if (s != TM_OK) return s;
    CellArgs a;
    tm_internal_fill_cell_args(ctx, &a);
    a.tri = tri; a.tri_cap = tri_cap; a.n_tri = (unsigned long long *)n_tri;
    a.adj = adj; a.deg = deg;
    a.d_prev = d_prev; a.x_out = x_out; a.y_out = y_out; a.d_prev_out = d_prev_out; a.status = status;
    TM_CUDA_TRY(ctx, cudaMemsetAsync(n_tri, 0, sizeof(int64_t), ctx->stream));
    if (ctx->p.flags & TM_F_COUNT_WORK)
        TM_CUDA_TRY(ctx, cudaMemsetAsync(ctx->dst->work, 0, sizeof(ctx->dst->work), ctx->stream));
    if (treat && adj) s = dispatch_count<M_TRI | M_ELL | M_TREAT>(ctx, a);
    else if (treat) s = dispatch_count<M_TRI | M_TREAT>(ctx, a);
    else if (adj) s = dispatch_count<M_TRI | M_ELL>(ctx, a);
    else s = dispatch_count<M_TRI>(ctx, a);
    if (s == TM_OK) {
        ctx->have_cells = true;
        // neighbour lists written (thread kernel only): warm start for the next launch
        ctx->nbr_n = (a.nbr && !(ctx->p.flags & TM_F_GROUP_CELLS)) ? a.nbr_keys : -1;
    }
    if (s == TM_OK && adj && !ctx->dcnt) {
        // positions and h of this triangulation, for tm_retria_check (NEXT-1, Alg. 1)
        if (ctx->cap_tria < ctx->n_local) {
            cudaFree(ctx->xs_tria); cudaFree(ctx->ys_tria); cudaFree(ctx->hs_tria);
            ctx->xs_tria = ctx->ys_tria = ctx->hs_tria = nullptr;
            const int64_t c = ctx->cap_points;
            TM_CUDA_TRY(ctx, cudaMalloc(&ctx->xs_tria, c * sizeof(double)));
            TM_CUDA_TRY(ctx, cudaMalloc(&ctx->ys_tria, c * sizeof(double)));
            TM_CUDA_TRY(ctx, cudaMalloc(&ctx->hs_tria, c * sizeof(double)));
            ctx->cap_tria = c;
        }
        const size_t nb = (size_t)ctx->n_local * sizeof(double);
        TM_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->xs_tria, ctx->xs, nb, cudaMemcpyDeviceToDevice, ctx->stream));
        TM_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->ys_tria, ctx->ys, nb, cudaMemcpyDeviceToDevice, ctx->stream));
        TM_CUDA_TRY(ctx, cudaMemcpyAsync(ctx->hs_tria, ctx->hs, nb, cudaMemcpyDeviceToDevice, ctx->stream));
        ctx->have_tria = true;
    }
    return s;
}

extern "C" tm_status tm_cvd_step(tm_ctx *ctx, const double *d_prev, double *x_hat, double *y_hat) {
    if (!ctx) return TM_E_ARG;
    if (!ctx->have_bins) TM_FAIL(ctx, TM_E_STATE, "tm_cvd_step before tm_grid_bin");
    if (!x_hat || !y_hat) TM_FAIL(ctx, TM_E_ARG, "x_hat/y_hat required");
    TM_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
    tm_status s = ensure_retry(ctx);
    if (s != TM_OK) return s;
    CellArgs a;
    tm_internal_fill_cell_args(ctx, &a);
    a.d_prev = d_prev; a.x_hat = x_hat; a.y_hat = y_hat;
    if (ctx->p.flags & TM_F_COUNT_WORK)
        TM_CUDA_TRY(ctx, cudaMemsetAsync(ctx->dst->work, 0, sizeof(ctx->dst->work), ctx->stream));
    s = dispatch_count<M_HAT>(ctx, a);
    if (s == TM_OK) ctx->nbr_n = (a.nbr && !(ctx->p.flags & TM_F_GROUP_CELLS)) ? a.nbr_keys : -1;
    return s;
}
