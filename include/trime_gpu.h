/*
 * trime_gpu.h -- C ABI of libtrime_gpu.so, the B200 (sm_100a) hot path of one
 * TriMe++ meshing iteration (arXiv 2309.13824; PAPER.md cited as P:<line>).
 *
 * The paper's problem statement (P:117-119 Procedure 1, Alg. 2,
 * P:168-195 Alg. 1): points + a signed-distance grid + a sizing/density field
 * go in; the Delaunay triangles of the current points (obtained from
 * Voronoi cells built by half-plane clipping) and the updated
 * points (CVD centroid P:203-207, or DistMesh truss force P:139-164, then the
 * boundary treatment P:570-605) come out.
 *
 * CONVENTIONS (all entry points)
 *  - Pointers are DEVICE pointers unless annotated "host".  The caller owns
 *    every I/O buffer; the context owns its scratch, its copies of the grids
 *    and the sorted state of the last tm_grid_bin (freed by tm_destroy).
 *  - Every call is stream-ordered on the context's stream and never blocks the
 *    host, except where annotated "synchronises".  Nothing aborts or exits:
 *    every function returns a tm_status; tm_last_error() explains the last
 *    failure.  Asynchronous device-side failures (capacity overflow, duplicate
 *    or outside points, CUDA faults) are latched in the context and reported
 *    by the next synchronising call (tm_sync, tm_mesh_stats), which then clears
 *    them: after TM_E_CAPACITY the caller retries with the reported size on the
 *    same context and gets TM_OK.
 *  - Point-indexed outputs are in the CALLER's input order; triangle vertex
 *    indices are caller indices, or gid[] values when gid was given to
 *    tm_grid_bin.  The DistMesh ELL adjacency (adj/deg) is the exception: it is
 *    laid out by the context's sorted slot order and holds sorted slots; use
 *    tm_adjacency_export() to obtain caller-order rows of caller indices.
 *  - Call order is a state machine (TM_E_STATE otherwise):
 *      tm_set_domain -> tm_grid_bin -> { tm_voronoi_delaunay | tm_cvd_step }
 *      -> [ tm_distmesh_sums -> tm_distmesh_step ] -> [ tm_project_sdf ]
 *    tm_grid_bin must be repeated whenever the points change.
 *  - Precision: IEEE binary64 round-to-nearest; decision-relevant arithmetic
 *    is contraction-free (reading L25); exact incircle decisions
 *    (floating filter + exact expansion arithmetic).  Inputs must be generic
 *    (no four cocircular Delaunay points, L12); exact predicate zeros are
 *    counted in tm_stats.n_degenerate.
 *  - Threading: a context is bound to one device and one stream and is not
 *    thread-safe; several contexts may coexist.
 */
#ifndef TRIME_GPU_H
#define TRIME_GPU_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct tm_ctx tm_ctx;

typedef enum {
    TM_OK = 0,
    TM_E_ARG = 1,        /* NULL pointer, N < 3, grid < 2x2, bad size            */
    TM_E_CUDA = 2,       /* launch / allocation / asynchronous CUDA failure      */
    TM_E_CAPACITY = 3,   /* tri_cap, adj_stride or cell vertex capacity exceeded */
    TM_E_DUPLICATE = 4,  /* two bitwise-equal points (bisector undefined, L26)   */
    TM_E_OUTSIDE = 5,    /* a point is NaN or outside the closed box B           */
    TM_E_STATE = 6,      /* call out of the documented order                     */
    TM_E_DEGENERATE = 7  /* inconsistent cell clip (non-generic input, L12)      */
} tm_status;

/* Node-centred grids over B = [x0,x1] x [y0,y1], row-major [ny][nx], node k at
 * x0 + k*(x1-x0)/(nx-1) (L15).  Bilinear lookup with cell index clamped
 * (SURVEY §8.0).  All three are DEVICE pointers; the context copies them. */
typedef struct {
    int32_t nx, ny;
    double x0, y0, x1, y1;
    const double *phi;   /* required: signed distance, < 0 inside  */
    const double *mu;    /* relative sizing mu(x); NULL = uniform   */
    const double *rho;   /* CVD density rho(x);   NULL = uniform    */
} tm_fields;

/* Defaults = PAPER.md Table B.1 where the paper gives one. */
typedef struct {
    double n_opt;              /* 6.0   mean points per leaf (3.3 for Voro++)   */
    double fac_voro_bound;     /* 5     P:1116 octagon circumradius S = fac*h (L6)      */
    double fac_pt_mvmt;        /* 0.4   P:1102 move clamp T_pt = fac*h(p_old)           */
    double fac_geps;           /* 0.01  P:1104 geps = fac*min(h, h_avg)                 */
    double fac_end_mvmt;       /* 0.001 P:1100 quadrature error floor                   */
    double newton_damping;     /* 1                                          */
    int32_t newton_max;        /* 10                                          */
    int32_t quad_max_level;    /* 10    L13 (paper silent)                              */
    double fscale;             /* 1.2   P:147 fac_F                                     */
    double dt_k;               /* 0.2   L3: Delta t * k (paper silent)                  */
    double keep_tol;           /* 0.0   L10: keep t iff phi~(centroid) < keep_tol       */
    int32_t adj_stride;        /* 16    ELL row width for DistMesh                      */
    int32_t max_cell_vertices; /* 32    cell vertex capacity (one warp lane per vertex) */
    uint32_t flags;            /* TM_F_* below                                          */
    /* NEXT-1 */
    int32_t projection;        /* 0     escaped points: L22 gradient Newton from p_new;
                                  1     the paper's Fig. 13: sphere tracing from an
                                        inner p_old (status |= 8), 2x2 damped Newton with FD
                                        derivatives from a boundary p_old                       */
    int32_t trace_max;         /* 64    sphere-tracing step cap (L39)                           */
    double fac_retria;         /* 0.1   P:1098 lazy re-triangulation threshold fac * h (Alg. 1) */
    /* NEXT-2 */
    int32_t validity;          /* 0     keep rule: L10 Test 1 (phi~(g) < keep_tol);
                                  1     the paper's Tests 1-3 (reading L43): discard iff
                                        phi~(g) > geps(g); keep iff >= 2 edge midpoints have
                                        phi~(m) <= geps(m); else keep iff |phi~(c_circ)|/R_circ <= t_circ */
    double t_circ;             /* 0.4   P:1118 circumcentre test threshold T^tria_ccircum        */
} tm_params;

#define TM_F_TWO_LEVEL_BINS 0x1u  /* split dense bins into 2^r x 2^r sub-bins (adaptive rho) */
#define TM_F_COUNT_WORK     0x2u  /* accumulate per-cell work counters (tm_work_counts)       */
#define TM_F_GROUP_CELLS    0x4u  /* cells by 16-lane groups instead of one thread per cell  */
#define TM_F_NO_WCERT       0x8u  /* warm-started launches: flat search instead of warm clips +
                                     warp-cooperative certification (A/B and tests)        */
#define TM_F_NO_PACKED_GRIDS 0x10u /* bilinear rho lookups from the node grid rows instead of the
                                      packed 4-corner cells of tm_set_domain (A/B and tests)   */
#define TM_F_NO_DEEP_PASS   0x20u  /* one output pass for every quadrature depth instead of
                                      deferring deep cells to a compacted pass (A/B, tests) */

/* Mesh quality (alpha = R_circ/(2 R_in), beta = l_max/l_min) and
 * the health counters accumulated since the previous synchronising call
 * (tm_sync / tm_mesh_stats, which read and clear them). */
typedef struct {
    int64_t n_tri, n_alpha_lt_1_2, n_alpha_lt_2;
    int64_t n_degenerate;   /* exact predicate zeros + inconsistent clips        */
    int64_t n_fallback;     /* points whose projection failed (status & 2)       */
    int64_t n_overflow;     /* cells that exceeded the vertex capacity           */
    double sum_sqrt_alpha, sum_sqrt_beta, max_alpha, max_beta;
    double sum_alpha, sum_alpha2, sum_beta, sum_beta2;
} tm_stats;

/* Algorithmic work of the last tm_voronoi_delaunay / tm_cvd_step launch
 * (only with TM_F_COUNT_WORK).  Sums over cells. */
typedef struct {
    int64_t n_cells, n_cert, deg, verts, t_own, quad_tris, ell, candidates, clips, exact_calls;
    int64_t retries;    /* cells the thread kernel handed to the 32-lane pass (any flags)           */
    int64_t warp_trips; /* thread kernel: candidate-loop trips summed over warps (x32 = lane slots) */
} tm_work;

void tm_params_default(tm_params *p);

/* Create a context on `device` that issues all work on `cuda_stream`
 * (a cudaStream_t; NULL = legacy default stream).  *out receives the handle. */
tm_status tm_create(int device, void *cuda_stream, const tm_params *p, tm_ctx **out);
void tm_destroy(tm_ctx *ctx);
const char *tm_last_error(const tm_ctx *ctx);
/* host: blocks until the stream is idle, then reports (and clears) latched device
 * errors. synchronises */
tm_status tm_sync(tm_ctx *ctx);

/* S0: copy the grids, compute
 * h(x) = c*mu~(x) with c = sqrt( ∫_{phi~<0} mu~^-2 dA / n_total ) (midpoint
 * rule over grid cells, row-major sequential sum) and h_avg = mean h over those
 * cells; size the level-0 bins for n_total points.  c_out/h_avg_out are host
 * pointers (may be NULL).  synchronises */
tm_status tm_set_domain(tm_ctx *ctx, const tm_fields *f, int64_t n_total, double *c_out, double *h_avg_out);

/* S1 (container insert P:651-655): counting-sort points into the
 * uniform bin grid (average occupancy n_opt), splitting dense bins when
 * TM_F_TWO_LEVEL_BINS.  x,y: n_local caller-order coordinates; the first
 * n_owned are owned, the rest are ghosts (multi-GPU halo) that are binned but
 * get no cell.  gid: global ids (NULL = identity).  Points must lie in B
 * (TM_E_OUTSIDE, latched). */
tm_status tm_grid_bin(tm_ctx *ctx, const double *x, const double *y, int64_t n_local, int64_t n_owned,
                      const int32_t *gid);

/* S2+S3: bounded Voronoi cell of every owned point by
 * nearest-first half-plane clipping of B ∩ Oct_i, then Delaunay extraction:
 * triangle {i,a,b} (i the smallest id) is written once, CCW with the smallest
 * id first, iff its circumcentre lies strictly inside B and all three octagons
 * and phi~(centroid) < keep_tol.  tri: int32[3*tri_cap]; n_tri: device int64
 * receiving the count (required count on overflow, TM_E_CAPACITY latched).
 * adj/deg (both or neither): DistMesh ELL rows (sorted-slot layout, width
 * adj_stride).  If x_out is non-NULL the CVD update is fused (S4a+S5, Alg. 2):
 * d_prev (caller order, NULL => first iteration, eps_c = fac_pt_mvmt, L13) in,
 * treated positions x_out/y_out, d_prev_out and status out (caller order;
 * status 0 accepted, 1 projected, 2 fallback to p_old, +4 move clamped). */
tm_status tm_voronoi_delaunay(tm_ctx *ctx, int32_t *tri, int64_t tri_cap, int64_t *n_tri,
                              int32_t *adj, uint8_t *deg,
                              const double *d_prev, double *x_out, double *y_out,
                              double *d_prev_out, int8_t *status);

/* S4a alone: density-weighted centroid x_hat of every
 * owned cell (recomputes the cells of the last tm_grid_bin), caller order. */
tm_status tm_cvd_step(tm_ctx *ctx, const double *d_prev, double *x_hat, double *y_hat);

/* S4b pass 1 (Eq. size scaling P:150-153, L1-L2): sums2[0] = Σ l_e^2,
 * sums2[1] = Σ mu~(m_e)^2 over unique kept edges owned by this rank (edge owned
 * by its smaller-id endpoint), deterministic fixed-order reduction. sums2: device
 * double[2].  For multi-GPU, all-reduce sums2 before pass 2. */
tm_status tm_distmesh_sums(tm_ctx *ctx, const int32_t *adj, const uint8_t *deg, double *sums2);

/* S4b pass 2 + S5 (Eqs. spring force, Euler P:141-163): per-point
 * gather F_i = Σ_a max(l0-l,0)(p_i-p_a)/l with l0 = mu~(m)*fscale*sqrt(s0/s1),
 * x_hat = p + dt_k*F (p if fixed[i], caller order, NULL = none), then the
 * treatment as in tm_voronoi_delaunay.  Outputs caller order. */
tm_status tm_distmesh_step(tm_ctx *ctx, const int32_t *adj, const uint8_t *deg, const double *sums2,
                           const uint8_t *fixed, const double *d_prev,
                           double *x_out, double *y_out, double *d_prev_out, int8_t *status);

/* S5 alone (L20-L22): clamp the move to
 * fac_pt_mvmt*h(p_old), clamp into B, accept if phi~ <= geps, else <= newton_max
 * gradient-Newton steps q -= phi~ grad/|grad|^2 (clamped into B) until
 * |phi~| <= geps, else fall back to p_old.  All arrays length n, any order. */
tm_status tm_project_sdf(tm_ctx *ctx, const double *x_old, const double *y_old, const double *x_hat,
                         const double *y_hat, int64_t n, double *x_out, double *y_out, double *d_prev_out,
                         int8_t *status);

/* S6: quality of n_tri triangles (caller indices into x,y) and the
 * health counters since the previous synchronising call; returns a latched
 * error like tm_sync (out is filled either way).  The sums are fixed-order tree
 * reductions (no atomics): bitwise reproducible.  out: host.  synchronises */
tm_status tm_mesh_stats(tm_ctx *ctx, const double *x, const double *y, const int32_t *tri, int64_t n_tri,
                        tm_stats *out);

/* NEXT-1, Alg. 1: DistMesh iterations on a stale triangulation.
 * tm_refresh_positions: new positions (caller order, the point set of the last tm_grid_bin)
 *   replace the binned ones without re-binning -- the ELL rows of the last triangulation
 *   then act on the current positions (tm_distmesh_sums / tm_distmesh_step).
 * tm_retria_check: *flag (device int32) |= 1 iff some point's position x_new/y_new (caller
 *   order) is farther than fac_retria * h(p_tria) from its position p_tria at the last
 *   tm_voronoi_delaunay with adj (re-triangulate in the next iteration). */
tm_status tm_refresh_positions(tm_ctx *ctx, const double *x, const double *y);
tm_status tm_retria_check(tm_ctx *ctx, const double *x_new, const double *y_new, int32_t *flag);

/* Copy of the ELL adjacency in caller order with caller ids (tests/export):
 * adj_out int32[n_owned*adj_stride], deg_out uint8[n_owned] (device). */
tm_status tm_adjacency_export(tm_ctx *ctx, const int32_t *adj, const uint8_t *deg, int32_t *adj_out,
                              uint8_t *deg_out);

/* Work counters of the last cell launch (TM_F_COUNT_WORK).  out: host. synchronises */
tm_status tm_work_counts(tm_ctx *ctx, tm_work *out);

/* ---- S7 multi-GPU strips; the exchange itself is NCCL ------ */
/* Pack the owned points with x < strip_lo + w into send_lo and those with
 * x >= strip_hi - w into send_hi, each as SoA segments [x | y | gid] of
 * capacity cap (doubles, doubles, int32).  Counts go to cnt2 (device int64[2]).
 * width > 0: w = width for every point (2 S_max, reading L34).  width < 0:
 * per point w_j = min(2 S_j / (1 - 2 fac c L), -width), L the Lipschitz
 * constant of mu~ (computed by tm_set_domain), which bounds the octagon radius
 * of any point across the edge; w = -width when 2 fac c L >= 1. */
tm_status tm_halo_pack(tm_ctx *ctx, const double *x, const double *y, const int32_t *gid, int64_t n_owned,
                       double strip_lo, double strip_hi, double width, double *send_lo, double *send_hi,
                       int64_t cap, int64_t *cnt2);
/* Partition owned points after an update: points with x < strip_lo go to
 * out_lo, x >= strip_hi to out_hi (SoA [x|y|gid|d_prev] segments of capacity
 * cap), the rest are compacted in place at the front of x/y/gid/d_prev.
 * cnt3 (device int64[3]) = kept, to_lo, to_hi. */
tm_status tm_migrate_pack(tm_ctx *ctx, double *x, double *y, int32_t *gid, double *d_prev, int64_t n_owned,
                          double strip_lo, double strip_hi, double *out_lo, double *out_hi, int64_t cap,
                          int64_t *cnt3);

/* ---- device-count variants: the strip path without host synchronisation --------
 * The ghost and migrant counts of a strip iteration are known only on the device (they
 * arrive with the NCCL messages).  These calls take them from device memory, so one
 * iteration issues no host sync; array arguments are then CAPACITIES (host, fixed).
 *
 * tm_grid_bin_dc: as tm_grid_bin, with d_counts = device int64[2] {n_owned, n_local}
 * (the first n_owned of the n_local points are owned) and cap_local >= n_local the
 * capacity of x/y/gid (gid required).  Every later call of the iteration (cells,
 * DistMesh passes, adjacency export) uses these live counts; ELL rows and rings are
 * strided by cap_local. */
tm_status tm_grid_bin_dc(tm_ctx *ctx, const double *x, const double *y, int64_t cap_local, const int64_t *d_counts,
                         const int32_t *gid);
/* tm_halo_pack with the owned count *d_n_owned (device) and capacity cap_owned; the two
 * counts go to cnt_lo / cnt_hi (device int64, e.g. the headers of the two messages).
 * Counts beyond cap are still counted (the receiver's tm_append_points latches the
 * overflow, TM_E_CAPACITY at the next synchronising call). */
tm_status tm_halo_pack_dc(tm_ctx *ctx, const double *x, const double *y, const int32_t *gid,
                          const int64_t *d_n_owned, int64_t cap_owned, double strip_lo, double strip_hi,
                          double width, double *send_lo, double *send_hi, int64_t cap, int64_t *cnt_lo,
                          int64_t *cnt_hi);
/* tm_migrate_pack with the owned count *d_n_owned (device, capacity cap_owned): the kept
 * count is written back to *d_n_owned, the leaver counts to cnt_lo / cnt_hi. */
tm_status tm_migrate_pack_dc(tm_ctx *ctx, double *x, double *y, int32_t *gid, double *d_prev, int64_t *d_n_owned,
                             int64_t cap_owned, double strip_lo, double strip_hi, double *out_lo, double *out_hi,
                             int64_t cap, int64_t *cnt_lo, int64_t *cnt_hi);
/* Append a received message -- segments [x | y | gid (int32) | d_prev] of capacity
 * msg_cap holding *msg_count entries (d_prev: NULL = no such segment) -- after the
 * *d_count points of x/y/gid/d_prev (capacity cap), and advance *d_count; overflow
 * latches TM_E_CAPACITY.  Device pointers, no host sync. */
tm_status tm_append_points(tm_ctx *ctx, double *x, double *y, int32_t *gid, double *d_prev, int64_t *d_count,
                           int64_t cap, const double *msg, const int64_t *msg_count, int64_t msg_cap);

/* Strip re-balancing input (S7): hist[b] (device int64, nb entries) = the number of the first
 * *d_n (device; NULL: cap) points of x (device) with x in bin b of nb equal bins of [x0, x1)
 * (clamped into the first / last bin).  Exact counts; asynchronous. */
tm_status tm_x_histogram(tm_ctx *ctx, const double *x, const int64_t *d_n, int64_t cap, double x0, double x1,
                         int32_t nb, int64_t *hist);

/* ---- CUDA Graphs: capture a sequence of the calls above once, replay it many times ----
 * tm_graph_begin starts capturing the context's stream (thread-local capture mode);
 * every call until tm_graph_end is recorded instead of run (its status reports argument
 * and state errors as usual).  Synchronising calls (tm_sync, tm_set_domain, tm_mesh_stats,
 * tm_work_counts) are refused with TM_E_STATE while capturing.  Buffers must not grow
 * during a capture: run the same sequence once before (warm-up).  A replay repeats the
 * recorded kernels with the recorded arguments (same buffers) on the context's stream. */
/* ---- NEXT-2 / NEXT-3: meshing to termination ------------------------------ */
/* Movement termination input (T^end_mvmt,i = fac_end_mvmt * h_i): *d_count
 * (device int64) = the number of inner points -- phi~(p_old) < -geps(p_old), the tagging rule of
 * P:410 (reading L38) -- whose move d_prev[i] (= |p_new - p_old|, L32) is NOT below
 * fac_end_mvmt * h(p_old).  x_old, y_old, d_prev: device, caller order, n entries.  Asynchronous;
 * exact (integer count). */
tm_status tm_move_count(tm_ctx *ctx, const double *x_old, const double *y_old, const double *d_prev, int64_t n,
                        int64_t *d_count);

/* Resolution update after point addition (reading L44): c, h_avg and the level-0 bins are
 * recomputed for N = n_total from the sums of tm_set_domain (equal to scaling the adaptive
 * quantities by sqrt(N_old / N_current) up to rounding).  Invalidates the warm start.  c_out /
 * h_avg_out: host, may be NULL.  Host arithmetic only. */
tm_status tm_set_n_total(tm_ctx *ctx, int64_t n_total, double *c_out, double *h_avg_out);

/* Point addition (§3.6, after Alliez et al.; reading L46): rank the n_tri triangles
 * (caller indices into x, y: the mesh T_n at its positions p_n) by R_circ / h(g) -- R_circ the
 * distance from p_u (u the smallest index) to the canonical circumcentre of the keep rule, g =
 * ((p_u + p_v) + p_w) / 3 with u < v < w, h(g) = c mu~(g) -- and write the centroids g of the
 * n_add largest (ties by (u, v) ascending) to x_new/y_new (device, n_add entries) in (u, v)
 * ascending order of their triangles.  *ratio_min (host, may be NULL) = the smallest selected
 * ratio.  0 <= n_add <= n_tri.  Uses scratch memory of ~56 bytes per triangle.  synchronises */
tm_status tm_point_addition(tm_ctx *ctx, const int32_t *tri, int64_t n_tri, const double *x, const double *y,
                            int64_t n_add, double *x_new, double *y_new, double *ratio_min);

/* The iterate-to-termination controller (host state machine; P:483-485, P:430, P:555,
 * thresholds Table B.1; reading L45).  After each iteration n, tm_control_update
 * takes the quality of the mesh (T_n, p_n) from tm_mesh_stats -- M_a, M_b the 1/2-means of
 * alpha and beta (Eq. 1/2-mean), A = max alpha -- and the movement count, compares them
 * with the previous iteration at the same N_current (relative changes r(X) = |X_n - X_{n-1}| /
 * X_{n-1}), and returns the action:
 *   N_current < N_total:            ADD (n_add = min(floor(fac_add N_current), N_total - N_current))
 *                                   when r(M_a) < T_add and r(M_b) < T_add;
 *   hybrid, still DistMesh:         SWITCH to CVD when r(M_a) < T_switch;
 *   otherwise:                      TERMINATE_MOVES when move_count == 0,
 *                                   TERMINATE_QUALITY when r(M_a), r(M_b) < T_end and
 *                                   r(A) < T_end_alpha;
 *   any:                            TERMINATE_CAP after max_iterations updates. */
#define TM_METHOD_CVD 0
#define TM_METHOD_DISTMESH 1
#define TM_METHOD_HYBRID 2
#define TM_ACT_CONTINUE 0
#define TM_ACT_ADD 1
#define TM_ACT_SWITCH 2
#define TM_ACT_TERMINATE_QUALITY 3
#define TM_ACT_TERMINATE_MOVES 4
#define TM_ACT_TERMINATE_CAP 5
typedef struct {
    int64_t n_total, n_current;
    int32_t method;            /* TM_METHOD_*                                   */
    int32_t mode;              /* current: TM_METHOD_CVD or TM_METHOD_DISTMESH   */
    int32_t have_prev, iterations;
    double prev[3];            /* M_a, M_b, max alpha of the previous iteration  */
    double t_add_quality;      /* 0.002 */
    double fac_add;            /* 0.6 */
    double t_end_quality;      /* 0.001 */
    double t_end_alpha_max;    /* 0.005 */
    double t_switch_quality;   /* 0.0015 P:1121 */
    int32_t max_iterations;    /* 1000   safety cap (paper silent) */
} tm_control;
void tm_control_init(tm_control *c, int64_t n_total, int64_t n_current, int32_t method);
/* returns TM_ACT_*; *n_add (host, may be NULL) receives the points to add for TM_ACT_ADD */
int32_t tm_control_update(tm_control *c, const tm_stats *s, int64_t move_count, int64_t *n_add);

/* ---- NEXT-4: the set-up pipeline ---------------------------------------------- */
/* Geometry grid size: lambda = sqrt(N_total / (N_opt A)), n = ceil(lambda L),
 * n_geo = fac_grid * n per axis (N_total = 5000 on the unit square, N_opt = 3.3,
 * fac_grid = 5 -> 195 x 195).  Host arithmetic. */
void tm_geometry_grid_dims(int64_t n_total, double n_opt, int32_t fac_grid, double x0, double y0, double x1,
                           double y1, int32_t *nx, int32_t *ny);
/* Geometry grid cell categories over the domain box of tm_set_domain, nxg x nyg cells:
 * cat[j*nxg+i] (device int8) = 1 (boundary) iff |phi~(m)| <= l_diag (m the midpoint, l_diag the
 * cell diagonal), else 0 (inner) iff phi~(m) < 0, else 2 (outer).  Asynchronous. */
tm_status tm_geometry_categories(tm_ctx *ctx, int32_t nxg, int32_t nyg, int8_t *cat);
/* Contour SDF: segs (device, n_seg x {x1, y1, x2, y2}) a closed loop in clockwise
 * order (segment k ends where k+1 starts; the last closes on the first).  phi (device, [ny][nx]
 * at the nodes x0 + i (x1-x0)/(nx-1), y likewise) = the distance to the closest segment point p*
 * (found by the outward layer search in a segment grid of ~mean-segment-length cells),
 * negative iff (p - p*).n > 0 for the inward normal n (right-hand normal of the clockwise
 * direction, averaged over both segments at a shared endpoint); ties of the distance:
 * the smallest segment index (reading L48).  synchronises */
tm_status tm_contour_sdf(tm_ctx *ctx, const double *segs, int64_t n_seg, int32_t nx, int32_t ny, double x0,
                         double y0, double x1, double y1, double *phi);
/* SDF set operations, elementwise on device arrays: op 0 union min(a,b),
 * 1 difference max(a,-b), 2 intersection max(a,b).  Asynchronous. */
tm_status tm_sdf_combine(tm_ctx *ctx, int32_t op, const double *a, const double *b, int64_t n, double *out);
/* Point initialisation (reading L47).  cat: the categories of tm_geometry_categories.
 * Valid cells: inner, and boundary cells with phi~(m) <= eta min(dx, dy) (eta 0.5).
 * Expected counts n_E = rho_norm * n_init with rho = rho~(m) (1 without rho) normalised over the
 * valid cells; Floyd-Steinberg dithering over the valid cells, rows from the top (largest y),
 * each left to right: count = max(0, floor(v + 1/2)) of v = n_E + received residual, the residual
 * spread equally over the valid not-yet-visited neighbours among right, below-left, below,
 * below-right (serial by construction: host code).  counts (device int32 [nyg][nxg]) receives the
 * counts and *n_out (host) their total.  Then, if x, y are given and cap >= total, point k (loop
 * order of cells, then within the cell) is cell-uniform from the counter-based generator
 * splitmix64(seed + (2k + comp + 1) * 0x9E3779B97F4A7C15) >> 11 * 2^-53 (comp 0: x, 1: y) and, if
 * phi~ > geps there, projected onto the boundary by the treatment's 2x2 damped Newton.
 * TM_E_CAPACITY if cap is too small (*n_out tells the size).  synchronises */
tm_status tm_init_points(tm_ctx *ctx, int32_t nxg, int32_t nyg, const int8_t *cat, double n_init, double eta,
                         uint64_t seed, int32_t *counts, double *x, double *y, int64_t cap, int64_t *n_out);

/* Automatic sizing (App. A; reading L48).
 * tm_boundary_points: boundary points of a closed contour (segs as for tm_contour_sdf): every
 *   segment's start point and, on a segment longer than d_s, the points a + (q/m)(b - a),
 *   q = 1..m-1, m = floor(len/d_s) + 1; then the serial trimming sweeps of App. A: for each point
 *   in order, its closest other point whose midpoint with it has |sdf| <= geps_hat is merged into
 *   the midpoint while closer than d_s; sweeps repeat until nothing changes.  *n_out (host) = the
 *   count; x, y (device, cap entries) receive the points when given.  synchronises
 * tm_medial_points: the medial-axis approximation of boundary points x, y (device, n): the
 *   Delaunay triangles with circumcentre strictly inside the box, from the library's own cell
 *   kernel with an octagon larger than the box (an unbounded-cell variant of S2); per point the
 *   farthest circumcentre v1 and the farthest v2 with (v2 - s).(v1 - s) < 0 (ties by the
 *   triangle's two smallest indices); v1, v2 in point order, kept iff >= n_thres other medial
 *   points lie strictly within r_nei.  mx, my (device, cap); *n_out (host).  synchronises
 * tm_sizing_field: lfs(s) = the distance to the nearest medial point, and
 *   mu = min_s [K |x - s| + lfs(s)] (Eq. sizing field) at the nodes of the [ny][nx] grid
 *   over the box (device mu; lfs device, ns entries).  Asynchronous. */
tm_status tm_boundary_points(tm_ctx *ctx, const double *segs, int64_t n_seg, double d_s, double geps_hat, double *x,
                             double *y, int64_t cap, int64_t *n_out);
tm_status tm_medial_points(tm_ctx *ctx, const double *x, const double *y, int64_t n, double x0, double y0, double x1,
                           double y1, double r_nei, int32_t n_thres, double *mx, double *my, int64_t cap,
                           int64_t *n_out);
tm_status tm_sizing_field(tm_ctx *ctx, const double *sx, const double *sy, int64_t ns, const double *mx,
                          const double *my, int64_t nm, double K, int32_t nx, int32_t ny, double x0, double y0,
                          double x1, double y1, double *mu, double *lfs);

/* Adaptive distance field on the boundary geometry cells (after Frisken et al.; L48):
 * tm_adf_build: per boundary cell (cat == 1 from tm_geometry_categories on an nxg x nyg grid) a
 *   top-down quadtree whose nodes hold the contour's exact SDF (segs as tm_contour_sdf) at their
 *   corners; a node splits into 4 while the largest error of its bilinear interpolant at the 4
 *   edge midpoints and the centre exceeds E_tol = fac_etol * geps_i * fac_pt (fac_etol 0.1,
 *   P:1107; geps_i = fac_geps min(h(m_i), h_avg); fac_pt = sqrt(N_current / N_total)) and its
 *   depth is below max_depth (10).  The trees live in the context; *n_nodes / *n_leaves
 *   (host, may be NULL) report their size.  synchronises
 * tm_adf_eval: out[i] (device) = the ADF at (x[i], y[i]) (device): descend to the leaf holding the
 *   point (x >= a node's mid line goes right / up), bilinear in its corners; NaN outside the
 *   boundary cells.  Asynchronous. */
tm_status tm_adf_build(tm_ctx *ctx, const double *segs, int64_t n_seg, int32_t nxg, int32_t nyg, const int8_t *cat,
                       double fac_etol, double fac_pt, int32_t max_depth, int64_t *n_nodes, int64_t *n_leaves);
tm_status tm_adf_eval(tm_ctx *ctx, const double *x, const double *y, int64_t n, double *out);

/* rho = 1 / mu^2 elementwise (Eq. density sizing relationship), device arrays. Asynchronous. */
tm_status tm_density_from_sizing(tm_ctx *ctx, const double *mu, int64_t n, double *rho);

typedef struct tm_graph tm_graph;
tm_status tm_graph_begin(tm_ctx *ctx);
tm_status tm_graph_end(tm_ctx *ctx, tm_graph **out);
tm_status tm_graph_launch(tm_ctx *ctx, tm_graph *g);
void tm_graph_destroy(tm_graph *g);

/* ---- host-side predicate hooks (no GPU needed; same code as the kernels) -- */
/* sign of incircle(a,b,c,d) (>0: d inside circle(a,b,c), a,b,c CCW) by the
 * kernels' exact expansion arithmetic, and by the kernels' full filtered path */
int tm_host_incircle_exact(const double *a, const double *b, const double *c, const double *d);
/* kernels' canonical Cramer vertex and keep-rule arithmetic, for CPU tests */
void tm_host_cramer(const double *A3, const double *B3, double *xy);
double tm_host_bilinear(int32_t nx, int32_t ny, double x0, double y0, double x1, double y1, const double *F,
                        double x, double y);

#ifdef __cplusplus
}
#endif
#endif
