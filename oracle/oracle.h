/*
 * oracle.h -- plain, slow, single-threaded CPU oracle for the TriMe++ hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, headers or constants with the CUDA path
 * (paper_2309_13824_b200/csrc, include/trime_gpu.h); both follow PAPER.md
 * (/root/reference/PAPER.md, cited as P:<line>) and the readings listed in
 * DESIGN.md / SURVEY.md §8(c) (cited as L<k>).
 *
 * Compiled with -O2 -ffp-contract=off (no fast-math): every expression is
 * evaluated in IEEE binary64 round-to-nearest exactly in source order (L25).
 */
#ifndef TRIME_ORACLE_H
#define TRIME_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int32_t nx, ny;              /* node grid size, >= 2 each            */
    double x0, y0, x1, y1;       /* box B = grid domain (L8, L15)        */
    const double *phi;           /* [ny][nx] signed distance, <0 inside  */
    const double *mu;            /* [ny][nx] relative sizing or NULL     */
    const double *rho;           /* [ny][nx] density or NULL             */
} or_fields;

typedef struct {
    double fac_voro_bound;  /* 5     P:1116 octagon circumradius S = fac*h     */
    double fac_pt_mvmt;     /* 0.4   P:1102 move clamp T_pt = fac*h            */
    double fac_geps;        /* 0.01  P:1104 geps = fac*min(h, h_avg)           */
    double fac_end_mvmt;    /* 0.001 P:1100 quadrature error floor             */
    double newton_damping;  /* 1                                    */
    int32_t newton_max;     /* 10                                    */
    int32_t quad_max_level; /* 10    L13                                       */
    double fscale;          /* 1.2                                     */
    double dt_k;            /* 0.2   L3                                        */
    double keep_tol;        /* 0.0   L10                                       */
    /* NEXT-1: the paper's treatment of escaped points, Fig. 13:
     * 0 = the L22 reading (gradient Newton from p_new), 1 = sphere tracing from an inner
     * p_old / damped 2x2 Newton on L(p) with FD derivatives from a boundary p_old
     * (Eqs. projection_*) */
    int32_t projection;
    int32_t trace_max;      /* 64    sphere-tracing step cap (paper silent, L39)            */
    double fac_retria;      /* 0.1   P:1098 lazy re-triangulation threshold fac * h (Alg. 1) */
    /* NEXT-2: the triangle validity tests, P:499-521 (§4.1).
     * 0 = Test 1 only in the L10 reading (keep iff phi~(g) < keep_tol);
     * 1 = the paper's Tests 1-3 (reading L43): discard iff phi~(g) > geps(g) (Test 1); keep iff
     *     at least two edge midpoints have phi~(m) <= geps(m) (Test 2); otherwise keep iff
     *     |phi~(c_circ)| / R_circ <= t_circ (Test 3).  geps(x) = fac_geps * min(h(x), h_avg). */
    int32_t validity;
    double t_circ;          /* 0.4   P:1118 circumcentre test threshold T^tria_ccircum          */
} or_params;

typedef struct {
    double c;              /* h(x) = c * mu~(x) normalisation (§8.0)  */
    double h_avg;          /* mean h over inside grid cells   */
    double fac_mu;         /* DistMesh scaling (Eq. size scaling)     */
    double sum_l2, sum_mu2;
    int64_t n_delaunay;    /* |D|                                      */
    int64_t n_kept;        /* |K|                                      */
    int64_t n_edges;       /* unique kept edges                        */
    int64_t n_degenerate;  /* exact predicate zeros / invariant faults */
    int64_t n_hull;        /* convex hull vertices of the input        */
    int64_t n_near_ties;   /* floating decisions within 1e-13 of their threshold (report) */
} or_info;

/* ---- exact predicates (sign only: -1, 0, +1) ---------------------------- */
int or_orient2d(const double *a, const double *b, const double *c);
int or_incircle(const double *a, const double *b, const double *c, const double *d);
/* same, forcing the big-integer path (no floating filter) */
int or_orient2d_exact(const double *a, const double *b, const double *c);
int or_incircle_exact(const double *a, const double *b, const double *c, const double *d);

/* ---- O1: Delaunay triangulation by Bowyer-Watson ------------------------ */
/* writes CCW triples (3*ntri ints); returns ntri, or -(needed) if cap too
 * small, or -1 on failure (n<3, all collinear, duplicates). */
int64_t or_delaunay(int64_t n, const double *x, const double *y,
                    int32_t *tri, int64_t cap, int64_t *n_degenerate);

/* ---- fields (§8.0 bilinear lookup) -------------------------------------- */
double or_field_value(const or_fields *f, const double *F, double x, double y);
void or_field_grad(const or_fields *f, const double *F, double x, double y, double *gx, double *gy);
/* S0: c and h_avg (§8.0 "Local size") */
void or_domain(const or_fields *f, int64_t n_total, double *c_out, double *h_avg_out);

/* ---- O2: bounded cells ---------------------------------------------------- */
/* Computes C_i for every point.  Output CSR: cell_start[n+1]; per vertex
 * labels la/lb (neighbour id >= 0, wall codes < 0) and coordinates RELATIVE
 * to p_i.  Vertices CCW from the smallest (la,lb) tuple.  Returns total
 * vertex count, or -(needed) if vcap too small. */
int64_t or_cells(const or_fields *f, const or_params *p, int64_t n,
                 const double *x, const double *y,
                 int64_t *cell_start, int32_t *la, int32_t *lb,
                 double *vx, double *vy, int64_t vcap, or_info *info);

/* ---- one full iteration (O1..O6) --------------------------------------- */
/* mode 0 = CVD (Alg. 2), 1 = DistMesh (Alg. 1 with retriangulation every
 * iteration, L5).  d_prev may be NULL (=> eps_c = fac_pt_mvmt, L13).
 * n_total: the N of the h normalisation (0 => n; a strip of a larger set passes the global N).
 * Outputs: kept triangles K (CCW, min index first) and, for DistMesh, unique
 * kept edges (a<b); proposals x_hat/y_hat; treated x_out/y_out, d_prev_out,
 * status (0 accepted, 1 projected, 2 fallback, +4 clamped).
 * counts (nullable) = int64[n][6]: n_cert, deg, V, T_own, Q, E  (O8). */
int or_iteration(const or_fields *f, const or_params *p, int64_t n, int64_t n_total,
                 const double *x, const double *y, const double *d_prev, int mode,
                 int32_t *tri, int64_t tri_cap,
                 int32_t *edges, int64_t edge_cap,
                 double *x_hat, double *y_hat,
                 double *x_out, double *y_out, double *d_prev_out, int8_t *status,
                 int64_t *counts, or_info *info);

/* ---- pieces exposed for pin tests -------------------------------------- */
/* O4 on a single convex polygon given by absolute CCW vertices (generator g) */
void or_cvd_polygon(const or_fields *f, const or_params *p, int nv, const double *px, const double *py,
                    double gx, double gy, double h, double d_prev, double *cx, double *cy, int *levels);
/* O5 on an explicit edge list */
void or_distmesh(const or_fields *f, const or_params *p, int64_t n, const double *x, const double *y,
                 int64_t ne, const int32_t *edges, const uint8_t *fixed,
                 double *x_hat, double *y_hat, double *fac_mu);
/* O6 treatment of one point */
int or_treat(const or_fields *f, const or_params *p, double c, double h_avg,
             double xo, double yo, double xh, double yh, double *xn, double *yn, double *dprev);
/* NEXT-1, Alg. 1 lines 7-11 with P:446: one DistMesh update on a STALE
 * triangulation -- forces over the unique edges of the last triangulation at the current
 * positions (O5), the treatment (O6), and the re-triangulation test: *retria = 1 iff some
 * point's displacement since that triangulation exceeds fac_retria * h(p_tria) (L40).
 * x_tria/y_tria: the positions the edges were computed at.  Returns 0. */
int or_distmesh_lazy(const or_fields *f, const or_params *p, int64_t n, int64_t n_total,
                     const double *x, const double *y, int64_t ne, const int32_t *edges,
                     const double *x_tria, const double *y_tria,
                     double *x_out, double *y_out, double *d_prev_out, int8_t *status, int32_t *retria);
/* O7 quality of one triangle and reductions over a list */
void or_triangle_quality(const double *a, const double *b, const double *c, double *alpha, double *beta);
void or_stats(int64_t n_tri, const int32_t *tri, const double *x, const double *y, double *out12);

/* ---- NEXT-2 / NEXT-3 ------------------------------------- */
/* keep rule O3 on one triangle (any vertex order), for pin tests */
int or_keep_triangle(const or_fields *f, const or_params *p, double c, double h_avg, const double *x,
                     const double *y, int32_t u, int32_t v, int32_t w);
/* inner points (phi~(p_old) < -geps) whose move d_prev is not below fac_end_mvmt*h(p_old) */
int64_t or_move_count(const or_fields *f, const or_params *p, double c, double h_avg, int64_t n,
                      const double *x_old, const double *y_old, const double *d_prev);
/* point addition: centroids of the n_add triangles of largest R_circ/h(g), in (u,v)
 * order; ratio_out[0] = smallest selected ratio.  Returns the count written. */
int64_t or_point_addition(const or_fields *f, double c, int64_t n_tri, const int32_t *tri, const double *x,
                          const double *y, int64_t n_add, double *x_new, double *y_new, double *ratio_out);

/* ---- NEXT-4: set-up pipeline ------------------------------ */
void or_geometry_grid_dims(int64_t n_total, double n_opt, int32_t fac_grid, double x0, double y0, double x1,
                           double y1, int32_t *nx, int32_t *ny);
/* cat[j*nxg+i]: 0 inner, 1 boundary (|phi~(m)| <= l_diag), 2 outer; box = the fields' box */
void or_geometry_categories(const or_fields *f, int32_t nxg, int32_t nyg, int8_t *cat);
/* SDF of a closed clockwise segment loop, brute force over the segments */
double or_contour_sdf_point(const double *segs, int64_t n_seg, double px, double py);
void or_contour_sdf(const double *segs, int64_t n_seg, int32_t nx, int32_t ny, double x0, double y0, double x1,
                    double y1, double *phi);
/* Floyd-Steinberg counts (reading L47); returns the total */
int64_t or_init_counts(const or_fields *f, int32_t nxg, int32_t nyg, const int8_t *cat, double n_init, double eta,
                       int32_t *counts);
/* the initial points of the counts (counter-based generator, projection P:402); returns the count */
int64_t or_init_points(const or_fields *f, const or_params *p, double c, double h_avg, int32_t nxg, int32_t nyg,
                       const int32_t *counts, uint64_t seed, double *x, double *y);

/* automatic sizing (App. A): boundary points of a contour, trimmed (returns the count,
 * -needed if cap is short); medial points by Delaunay poles, trimmed by neighbour counts; sizing */
int64_t or_boundary_points(const double *segs, int64_t n_seg, double d_s, double geps_hat, double *x, double *y,
                           int64_t cap);
int64_t or_medial_points(int64_t n, const double *x, const double *y, double x0, double y0, double x1, double y1,
                         double r_nei, int32_t n_thres, double *mx, double *my);
void or_sizing_field(int64_t ns, const double *sx, const double *sy, int64_t nm, const double *mx, const double *my,
                     double K, int32_t nx, int32_t ny, double x0, double y0, double x1, double y1, double *mu,
                     double *lfs);

/* ADF quadtrees on the boundary cells; handle freed by or_adf_free; eval NaN off them */
void *or_adf_build(const or_fields *f, const or_params *p, double c, double h_avg, int32_t nxg, int32_t nyg,
                   const int8_t *cat, const double *segs, int64_t n_seg, double fac_etol, double fac_pt,
                   int32_t max_depth, int64_t *n_nodes, int64_t *n_leaves);
double or_adf_eval(const void *h, double x, double y);
void or_adf_free(void *h);

#ifdef __cplusplus
}
#endif
#endif
