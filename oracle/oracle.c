/*
 * oracle.c -- plain, slow, single-threaded CPU oracle for one iteration of the
 * TriMe++ hot path (arXiv 2309.13824).  TEST INFRASTRUCTURE: see oracle.h.
 *
 * PAPER.md citations are "P:<line>"; readings of silent/garbled passages are
 * SURVEY.md §8(c) ledger entries "L<k>", restated in DESIGN.md.
 *
 *   O1  Delaunay D by Bowyer-Watson, exact predicates     P:43, P:118 (Proc. 1)
 *   O2  bounded cells C_i = B ∩ Oct_i ∩ Vor(i)
 *   O3  kept triangles K (Test 1 centroid form)
 *   O4  CVD centroid, adaptive quadrature
 *   O5  DistMesh force step
 *   O6  point treatment / projection
 *   O7  quality statistics
 *
 * Exact arithmetic: a double is m*2^e with m a 53-bit integer; all coordinates
 * entering a predicate are scaled to the smallest exponent and the determinant
 * is evaluated with schoolbook big integers (no floating point at all).
 */
#include "oracle.h"

#include <float.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_DIE(...) do { fprintf(stderr, "oracle: " __VA_ARGS__); fputc('\n', stderr); abort(); } while (0)

static int64_t g_degenerate = 0; /* exact zeros met by predicates / invariant faults */
/* decision-margin report (SURVEY §8(c) parity protocol): floating decisions -- keep-rule
 * box/octagon/phi tests, quadrature stop, treatment accept and Newton stop -- whose two
 * sides differ by at most 1e-13 of the decision's own scale.  Reporting only: no result
 * depends on it. */
static int64_t g_near = 0;
static void near_tie(double a, double b, double scale) {
    if (fabs(a - b) <= 1e-13 * fabs(scale)) g_near++;
}

/* ========================================================================== */
/* Big integers: sign-magnitude, 32-bit limbs, little endian.                  */
/* ========================================================================== */
#define BI_LIMBS 176 /* 5632 bits: enough for degree-4 products of any finite doubles' differences within ~1300-bit spans */

typedef struct {
    int sign;   /* -1, 0, +1 */
    int n;      /* used limbs */
    uint32_t d[BI_LIMBS];
} bigint;

static void bi_zero(bigint *a) { a->sign = 0; a->n = 0; }

static void bi_trim(bigint *a) {
    while (a->n > 0 && a->d[a->n - 1] == 0) a->n--;
    if (a->n == 0) a->sign = 0;
}

/* |a| cmp |b| */
static int bi_cmp_mag(const bigint *a, const bigint *b) {
    if (a->n != b->n) return a->n < b->n ? -1 : 1;
    for (int i = a->n - 1; i >= 0; i--)
        if (a->d[i] != b->d[i]) return a->d[i] < b->d[i] ? -1 : 1;
    return 0;
}

/* r = |a| + |b| (magnitudes) */
static void bi_add_mag(bigint *r, const bigint *a, const bigint *b) {
    int n = a->n > b->n ? a->n : b->n;
    uint64_t carry = 0;
    if (n + 1 > BI_LIMBS) ORACLE_DIE("bigint overflow (add)");
    for (int i = 0; i < n; i++) {
        uint64_t s = carry;
        if (i < a->n) s += a->d[i];
        if (i < b->n) s += b->d[i];
        r->d[i] = (uint32_t)s;
        carry = s >> 32;
    }
    r->d[n] = (uint32_t)carry;
    r->n = n + 1;
}

/* r = |a| - |b|, requires |a| >= |b| */
static void bi_sub_mag(bigint *r, const bigint *a, const bigint *b) {
    int64_t borrow = 0;
    for (int i = 0; i < a->n; i++) {
        int64_t s = (int64_t)a->d[i] - borrow - (i < b->n ? (int64_t)b->d[i] : 0);
        borrow = 0;
        if (s < 0) { s += ((int64_t)1 << 32); borrow = 1; }
        r->d[i] = (uint32_t)s;
    }
    r->n = a->n;
}

static void bi_add(bigint *r, const bigint *a, const bigint *b) {
    bigint t;
    if (a->sign == 0) { *r = *b; return; }
    if (b->sign == 0) { *r = *a; return; }
    if (a->sign == b->sign) {
        bi_add_mag(&t, a, b);
        t.sign = a->sign;
    } else {
        int c = bi_cmp_mag(a, b);
        if (c == 0) { bi_zero(r); return; }
        if (c > 0) { bi_sub_mag(&t, a, b); t.sign = a->sign; }
        else       { bi_sub_mag(&t, b, a); t.sign = b->sign; }
    }
    bi_trim(&t);
    *r = t;
}

static void bi_neg(bigint *a) { a->sign = -a->sign; }

static void bi_sub(bigint *r, const bigint *a, const bigint *b) {
    bigint nb = *b;
    bi_neg(&nb);
    bi_add(r, a, &nb);
}

static void bi_mul(bigint *r, const bigint *a, const bigint *b) {
    bigint t;
    if (a->sign == 0 || b->sign == 0) { bi_zero(r); return; }
    if (a->n + b->n > BI_LIMBS) ORACLE_DIE("bigint overflow (mul)");
    memset(t.d, 0, sizeof(uint32_t) * (size_t)(a->n + b->n));
    for (int i = 0; i < a->n; i++) {
        uint64_t carry = 0;
        for (int j = 0; j < b->n; j++) {
            uint64_t cur = (uint64_t)a->d[i] * b->d[j] + t.d[i + j] + carry;
            t.d[i + j] = (uint32_t)cur;
            carry = cur >> 32;
        }
        int k = i + b->n;
        while (carry) {
            uint64_t cur = (uint64_t)t.d[k] + carry;
            t.d[k] = (uint32_t)cur;
            carry = cur >> 32;
            k++;
        }
    }
    t.n = a->n + b->n;
    t.sign = a->sign * b->sign;
    bi_trim(&t);
    *r = t;
}

/* decompose finite v = m * 2^e with |m| < 2^53 integer; returns e (unused if v==0) */
static int dbl_decompose(double v, int64_t *m) {
    int E;
    double f = frexp(v, &E);            /* v = f * 2^E, 0.5 <= |f| < 1 */
    double mi = ldexp(f, 53);            /* exact: integer-valued */
    *m = (int64_t)mi;
    return E - 53;
}

/* bigint = v * 2^(-emin), exact (requires exponent(v) >= emin) */
static void bi_from_double(bigint *r, double v, int emin) {
    int64_t m;
    if (v == 0.0) { bi_zero(r); return; }
    int e = dbl_decompose(v, &m);
    int sh = e - emin;
    if (sh < 0) ORACLE_DIE("internal: negative shift");
    uint64_t mag = (uint64_t)(m < 0 ? -m : m);
    int limb = sh / 32, bit = sh % 32;
    int need = limb + 3;
    if (need > BI_LIMBS) ORACLE_DIE("coordinate exponent span too large for the big-integer oracle");
    memset(r->d, 0, sizeof(uint32_t) * (size_t)need);
    /* place 64-bit mag shifted by bit into limbs limb..limb+2 */
    uint64_t lo = mag << bit;
    uint64_t hi = bit ? (mag >> (64 - bit)) : 0;
    r->d[limb] = (uint32_t)lo;
    r->d[limb + 1] = (uint32_t)(lo >> 32);
    r->d[limb + 2] = (uint32_t)hi;
    r->n = need;
    r->sign = m < 0 ? -1 : 1;
    bi_trim(r);
}

static int min_exponent(const double *v, int k) {
    int emin = 1 << 30;
    for (int i = 0; i < k; i++) {
        if (v[i] == 0.0) continue;
        if (!isfinite(v[i])) ORACLE_DIE("non-finite coordinate");
        int64_t m;
        int e = dbl_decompose(v[i], &m);
        if (e < emin) emin = e;
    }
    return emin == (1 << 30) ? 0 : emin;
}

/* ========================================================================== */
/* Exact predicates                                                            */
/* ========================================================================== */
/* orient2d(a,b,c) = sign of (bx-ax)(cy-ay) - (by-ay)(cx-ax): >0 iff a,b,c CCW */
int or_orient2d_exact(const double *a, const double *b, const double *c) {
    double v[6] = {a[0], a[1], b[0], b[1], c[0], c[1]};
    int emin = min_exponent(v, 6);
    bigint A[6], t1, t2, u, w, det;
    for (int i = 0; i < 6; i++) bi_from_double(&A[i], v[i], emin);
    bi_sub(&t1, &A[2], &A[0]); /* bx-ax */
    bi_sub(&t2, &A[5], &A[1]); /* cy-ay */
    bi_mul(&u, &t1, &t2);
    bi_sub(&t1, &A[3], &A[1]); /* by-ay */
    bi_sub(&t2, &A[4], &A[0]); /* cx-ax */
    bi_mul(&w, &t1, &t2);
    bi_sub(&det, &u, &w);
    return det.sign;
}

/* incircle(a,b,c,d) = sign of det | a-d, |a-d|^2 ; b-d ... ; c-d ... |:
 * >0 iff d lies strictly inside the circle through a,b,c when a,b,c are CCW. */
int or_incircle_exact(const double *a, const double *b, const double *c, const double *d) {
    double v[8] = {a[0], a[1], b[0], b[1], c[0], c[1], d[0], d[1]};
    int emin = min_exponent(v, 8);
    bigint P[8];
    for (int i = 0; i < 8; i++) bi_from_double(&P[i], v[i], emin);
    bigint adx, ady, bdx, bdy, cdx, cdy;
    bi_sub(&adx, &P[0], &P[6]); bi_sub(&ady, &P[1], &P[7]);
    bi_sub(&bdx, &P[2], &P[6]); bi_sub(&bdy, &P[3], &P[7]);
    bi_sub(&cdx, &P[4], &P[6]); bi_sub(&cdy, &P[5], &P[7]);
    bigint t1, t2, alift, blift, clift;
    bi_mul(&t1, &adx, &adx); bi_mul(&t2, &ady, &ady); bi_add(&alift, &t1, &t2);
    bi_mul(&t1, &bdx, &bdx); bi_mul(&t2, &bdy, &bdy); bi_add(&blift, &t1, &t2);
    bi_mul(&t1, &cdx, &cdx); bi_mul(&t2, &cdy, &cdy); bi_add(&clift, &t1, &t2);
    bigint m1, m2, m3, s;
    bi_mul(&t1, &bdx, &cdy); bi_mul(&t2, &cdx, &bdy); bi_sub(&m1, &t1, &t2); /* bdx*cdy - cdx*bdy */
    bi_mul(&t1, &cdx, &ady); bi_mul(&t2, &adx, &cdy); bi_sub(&m2, &t1, &t2); /* cdx*ady - adx*cdy */
    bi_mul(&t1, &adx, &bdy); bi_mul(&t2, &bdx, &ady); bi_sub(&m3, &t1, &t2); /* adx*bdy - bdx*ady */
    bigint det;
    bi_mul(&det, &alift, &m1);
    bi_mul(&s, &blift, &m2); bi_add(&det, &det, &s);
    bi_mul(&s, &clift, &m3); bi_add(&det, &det, &s);
    return det.sign;
}

/* Floating filters with Shewchuk's static forward-error bounds (Shewchuk 1997,
 * "Adaptive precision floating-point arithmetic and fast robust geometric
 * predicates": orient2d (3+16eps)eps, incircle (10+96eps)eps), each taken
 * with an extra safety factor; anything not certified goes to the big-integer
 * path.  Pinned against exact rationals in tests/test_oracle_predicates.py. */
static const double OR_EPS = 1.1102230246251565e-16; /* 2^-53 */

/* counted = 0: an exact zero is legitimate (collinear points met by the
 * point-location walk or the ghost test, which handle it explicitly) */
static int orient2d_impl(const double *a, const double *b, const double *c, int counted) {
    double detl = (b[0] - a[0]) * (c[1] - a[1]);
    double detr = (b[1] - a[1]) * (c[0] - a[0]);
    double det = detl - detr;
    double detsum = fabs(detl) + fabs(detr);
    double bound = 8.0 * OR_EPS * detsum;
    if (det > bound) return 1;
    if (-det > bound) return -1;
    int s = or_orient2d_exact(a, b, c);
    if (s == 0 && counted) g_degenerate++;
    return s;
}

int or_orient2d(const double *a, const double *b, const double *c) { return orient2d_impl(a, b, c, 1); }
static int orient_walk(const double *a, const double *b, const double *c) { return orient2d_impl(a, b, c, 0); }

int or_incircle(const double *a, const double *b, const double *c, const double *d) {
    double adx = a[0] - d[0], ady = a[1] - d[1];
    double bdx = b[0] - d[0], bdy = b[1] - d[1];
    double cdx = c[0] - d[0], cdy = c[1] - d[1];
    double bdxcdy = bdx * cdy, cdxbdy = cdx * bdy;
    double cdxady = cdx * ady, adxcdy = adx * cdy;
    double adxbdy = adx * bdy, bdxady = bdx * ady;
    double alift = adx * adx + ady * ady;
    double blift = bdx * bdx + bdy * bdy;
    double clift = cdx * cdx + cdy * cdy;
    double det = alift * (bdxcdy - cdxbdy) + blift * (cdxady - adxcdy) + clift * (adxbdy - bdxady);
    double perm = (fabs(bdxcdy) + fabs(cdxbdy)) * alift + (fabs(cdxady) + fabs(adxcdy)) * blift +
                  (fabs(adxbdy) + fabs(bdxady)) * clift;
    double bound = 24.0 * OR_EPS * perm;
    if (det > bound) return 1;
    if (-det > bound) return -1;
    int s = or_incircle_exact(a, b, c, d);
    if (s == 0) g_degenerate++;
    return s;
}

/* ========================================================================== */
/* O1: Bowyer-Watson with ghost triangles                                       */
/* ========================================================================== */
#define GHOST (-1)

typedef struct {
    int32_t v[3];  /* CCW; a ghost triangle has v[2] == GHOST, its finite edge v0->v1 faces outside */
    int32_t n[3];  /* n[k] = triangle across the edge v[k+1]->v[k+2] */
    int32_t alive;
} bw_tri;

typedef struct {
    const double *x, *y;
    bw_tri *t;
    int64_t nt, cap;
    int32_t *freelist;
    int64_t nfree, freecap;
    int32_t last;
    /* scratch */
    int32_t *stack, *cavity, *mark;
    int64_t stackcap, markcap;
    uint64_t rng;
} bw_state;

static uint64_t bw_rand(bw_state *s) {
    s->rng ^= s->rng << 13; s->rng ^= s->rng >> 7; s->rng ^= s->rng << 17;
    return s->rng;
}

static void pt(const bw_state *s, int32_t i, double *out) { out[0] = s->x[i]; out[1] = s->y[i]; }

static int32_t bw_new(bw_state *s, int32_t a, int32_t b, int32_t c) {
    int32_t id;
    if (s->nfree > 0) id = s->freelist[--s->nfree];
    else {
        if (s->nt == s->cap) {
            s->cap = s->cap ? s->cap * 2 : 1024;
            s->t = (bw_tri *)realloc(s->t, sizeof(bw_tri) * (size_t)s->cap);
            s->mark = (int32_t *)realloc(s->mark, sizeof(int32_t) * (size_t)s->cap);
            if (!s->t || !s->mark) ORACLE_DIE("out of memory");
            for (int64_t k = s->nt; k < s->cap; k++) s->mark[k] = 0;
        }
        id = (int32_t)s->nt++;
    }
    /* normalise: ghost vertex last */
    int32_t v[3] = {a, b, c};
    if (v[0] == GHOST) { v[0] = b; v[1] = c; v[2] = a; }
    else if (v[1] == GHOST) { v[0] = c; v[1] = a; v[2] = b; }
    s->t[id].v[0] = v[0]; s->t[id].v[1] = v[1]; s->t[id].v[2] = v[2];
    s->t[id].n[0] = s->t[id].n[1] = s->t[id].n[2] = -1;
    s->t[id].alive = 1;
    s->mark[id] = 0;
    return id;
}

static void bw_free(bw_state *s, int32_t id) {
    s->t[id].alive = 0;
    if (s->nfree == s->freecap) {
        s->freecap = s->freecap ? s->freecap * 2 : 1024;
        s->freelist = (int32_t *)realloc(s->freelist, sizeof(int32_t) * (size_t)s->freecap);
        if (!s->freelist) ORACLE_DIE("out of memory");
    }
    s->freelist[s->nfree++] = id;
}

/* index k of the directed edge u->w in triangle t, or -1 */
static int edge_index(const bw_tri *t, int32_t u, int32_t w) {
    for (int k = 0; k < 3; k++)
        if (t->v[(k + 1) % 3] == u && t->v[(k + 2) % 3] == w) return k;
    return -1;
}

/* Is p (index q) in conflict with triangle id, i.e. strictly inside its
 * circumcircle (real) or strictly beyond its hull edge (ghost)? */
static int bw_conflict(bw_state *s, int32_t id, int32_t q) {
    const bw_tri *t = &s->t[id];
    double P[2], A[2], B[2], C[2];
    pt(s, q, P);
    if (t->v[2] == GHOST) {
        pt(s, t->v[0], A); pt(s, t->v[1], B);
        int o = orient_walk(A, B, P);
        if (o > 0) return 1;
        if (o < 0) return 0;
        /* collinear with the hull edge: conflict iff strictly inside the segment */
        double lo = A[0] < B[0] ? A[0] : B[0], hi = A[0] < B[0] ? B[0] : A[0];
        double loy = A[1] < B[1] ? A[1] : B[1], hiy = A[1] < B[1] ? B[1] : A[1];
        if (A[0] != B[0]) return P[0] > lo && P[0] < hi;
        return P[1] > loy && P[1] < hiy;
    }
    pt(s, t->v[0], A); pt(s, t->v[1], B); pt(s, t->v[2], C);
    return or_incircle(A, B, C, P) > 0;
}

/* visibility walk from s->last to a triangle in conflict with q */
static int32_t bw_locate(bw_state *s, int32_t q) {
    int32_t cur = s->last;
    double P[2], A[2], B[2];
    pt(s, q, P);
    int64_t steps = 0;
    for (;;) {
        if (++steps > 4 * s->nt + 100) break; /* should not happen on a Delaunay triangulation */
        const bw_tri *t = &s->t[cur];
        if (t->v[2] == GHOST) {
            if (bw_conflict(s, cur, q)) return cur;
            /* walk onto the adjacent real triangle */
            cur = t->n[2];
            continue;
        }
        int start = (int)(bw_rand(s) % 3), moved = 0;
        for (int kk = 0; kk < 3; kk++) {
            int k = (start + kk) % 3;
            pt(s, t->v[(k + 1) % 3], A);
            pt(s, t->v[(k + 2) % 3], B);
            if (orient_walk(A, B, P) < 0) { cur = t->n[k]; moved = 1; break; }
        }
        if (!moved) {
            if (bw_conflict(s, cur, q)) return cur;
            /* p on the boundary of cur but not in conflict: degenerate; fall back */
            break;
        }
    }
    for (int64_t id = 0; id < s->nt; id++)
        if (s->t[id].alive && bw_conflict(s, (int32_t)id, q)) return (int32_t)id;
    return -1;
}

static void bw_link(bw_state *s, int32_t a, int32_t u, int32_t w, int32_t b) {
    int k = edge_index(&s->t[a], u, w);
    if (k < 0) ORACLE_DIE("internal: link edge missing");
    s->t[a].n[k] = b;
}

static int bw_insert(bw_state *s, int32_t q) {
    int32_t seed = bw_locate(s, q);
    if (seed < 0) return -1;
    /* BFS over conflicting triangles */
    int64_t ncav = 0, nstack = 0;
    s->stack[nstack++] = seed;
    s->mark[seed] = 1;
    while (nstack) {
        int32_t id = s->stack[--nstack];
        s->cavity[ncav++] = id;
        for (int k = 0; k < 3; k++) {
            int32_t nb = s->t[id].n[k];
            if (nb < 0 || s->mark[nb]) continue;
            if (bw_conflict(s, nb, q)) {
                s->mark[nb] = 1;
                if (nstack >= s->stackcap) ORACLE_DIE("cavity too large");
                s->stack[nstack++] = nb;
            }
        }
        if (ncav + 3 >= s->stackcap) ORACLE_DIE("cavity too large");
    }
    /* boundary edges: (u, w, outer triangle) */
    int64_t nb_edges = 0;
    int32_t *eu = s->stack, *ew = s->stack + s->stackcap / 3, *eo = s->stack + 2 * (s->stackcap / 3);
    for (int64_t c = 0; c < ncav; c++) {
        int32_t id = s->cavity[c];
        for (int k = 0; k < 3; k++) {
            int32_t nb = s->t[id].n[k];
            if (nb >= 0 && s->mark[nb]) continue;
            if (nb_edges >= s->stackcap / 3) ORACLE_DIE("cavity boundary too large");
            eu[nb_edges] = s->t[id].v[(k + 1) % 3];
            ew[nb_edges] = s->t[id].v[(k + 2) % 3];
            eo[nb_edges] = nb;
            nb_edges++;
        }
    }
    for (int64_t c = 0; c < ncav; c++) { s->mark[s->cavity[c]] = 0; bw_free(s, s->cavity[c]); }
    /* new triangles (u, w, q); remember which new triangle starts at u */
    int32_t *newt = s->cavity; /* reuse */
    for (int64_t e = 0; e < nb_edges; e++) {
        int32_t id = bw_new(s, eu[e], ew[e], q);
        newt[e] = id;
        int32_t o = eo[e];
        bw_link(s, id, eu[e], ew[e], o);
        if (o >= 0) bw_link(s, o, ew[e], eu[e], id);
    }
    /* internal links: triangle on (u,w) has edge w->q, matched by the triangle starting at w (edge q->w) */
    for (int64_t e = 0; e < nb_edges; e++) {
        int32_t w = ew[e], partner = -1;
        for (int64_t f = 0; f < nb_edges; f++)
            if (eu[f] == w) { partner = newt[f]; break; }
        if (partner < 0) ORACLE_DIE("internal: cavity boundary not closed");
        bw_link(s, newt[e], w, q, partner);
        bw_link(s, partner, q, w, newt[e]);
    }
    s->last = newt[0];
    for (int64_t e = 0; e < nb_edges; e++)
        if (s->t[newt[e]].v[2] != GHOST) { s->last = newt[e]; break; }
    return 0;
}

/* Hilbert index of (xi, yi) on a 2^16 x 2^16 grid */
static uint64_t hilbert_d(uint32_t xi, uint32_t yi) {
    uint64_t d = 0;
    uint32_t n = 1u << 16;
    for (uint32_t s = n / 2; s > 0; s /= 2) {
        uint32_t rx = (xi & s) > 0, ry = (yi & s) > 0;
        d += (uint64_t)s * s * ((3 * rx) ^ ry);
        if (ry == 0) {
            if (rx == 1) { xi = n - 1 - xi; yi = n - 1 - yi; }
            uint32_t t = xi; xi = yi; yi = t;
        }
    }
    return d;
}

typedef struct { uint64_t key; int32_t idx; } keyidx;
static int cmp_keyidx(const void *a, const void *b) {
    const keyidx *p = (const keyidx *)a, *q = (const keyidx *)b;
    if (p->key != q->key) return p->key < q->key ? -1 : 1;
    return p->idx < q->idx ? -1 : (p->idx > q->idx);
}

static int bw_build(bw_state *s, int64_t n, const double *x, const double *y) {
    memset(s, 0, sizeof(*s));
    s->x = x; s->y = y; s->rng = 0x9E3779B97F4A7C15ull;
    s->stackcap = 3 * 65536;
    s->stack = (int32_t *)malloc(sizeof(int32_t) * (size_t)s->stackcap);
    s->cavity = (int32_t *)malloc(sizeof(int32_t) * (size_t)s->stackcap);
    if (!s->stack || !s->cavity) ORACLE_DIE("out of memory");
    /* insertion order: Hilbert curve over the bounding box */
    double xmin = x[0], xmax = x[0], ymin = y[0], ymax = y[0];
    for (int64_t i = 1; i < n; i++) {
        if (x[i] < xmin) xmin = x[i];
        if (x[i] > xmax) xmax = x[i];
        if (y[i] < ymin) ymin = y[i];
        if (y[i] > ymax) ymax = y[i];
    }
    double sx = xmax > xmin ? 65535.0 / (xmax - xmin) : 0.0, sy = ymax > ymin ? 65535.0 / (ymax - ymin) : 0.0;
    keyidx *ord = (keyidx *)malloc(sizeof(keyidx) * (size_t)n);
    for (int64_t i = 0; i < n; i++) {
        uint32_t xi = (uint32_t)((x[i] - xmin) * sx), yi = (uint32_t)((y[i] - ymin) * sy);
        ord[i].key = hilbert_d(xi, yi);
        ord[i].idx = (int32_t)i;
    }
    qsort(ord, (size_t)n, sizeof(keyidx), cmp_keyidx);
    /* first triangle: first two points + first point not collinear with them */
    int32_t a = ord[0].idx, b = ord[1].idx, c = -1;
    int64_t cpos = -1;
    double A[2], B[2], C[2];
    pt(s, a, A); pt(s, b, B);
    if (A[0] == B[0] && A[1] == B[1]) { free(ord); return -2; }
    for (int64_t k = 2; k < n; k++) {
        pt(s, ord[k].idx, C);
        if (orient_walk(A, B, C) != 0) { c = ord[k].idx; cpos = k; break; }
    }
    if (c < 0) { free(ord); return -1; }
    pt(s, c, C);
    if (orient_walk(A, B, C) < 0) { int32_t t = a; a = b; b = t; }
    int32_t T = bw_new(s, a, b, c);
    int32_t G0 = bw_new(s, c, b, GHOST), G1 = bw_new(s, a, c, GHOST), G2 = bw_new(s, b, a, GHOST);
    bw_link(s, T, b, c, G0); bw_link(s, G0, c, b, T);
    bw_link(s, T, c, a, G1); bw_link(s, G1, a, c, T);
    bw_link(s, T, a, b, G2); bw_link(s, G2, b, a, T);
    /* ghost-ghost: edge (x -> GHOST) of one with (GHOST -> x) of another */
    int32_t G[3] = {G0, G1, G2};
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) {
            if (i == j) continue;
            int32_t u = s->t[G[i]].v[1]; /* edge v1 -> GHOST */
            if (s->t[G[j]].v[0] == u) { bw_link(s, G[i], u, GHOST, G[j]); bw_link(s, G[j], GHOST, u, G[i]); }
        }
    s->last = T;
    for (int64_t k = 2; k < n; k++) {
        if (k == cpos) continue;
        int32_t q = ord[k].idx;
        if (bw_insert(s, q) != 0) { free(ord); return -3; }
    }
    free(ord);
    return 0;
}

static void bw_destroy(bw_state *s) {
    free(s->t); free(s->freelist); free(s->stack); free(s->cavity); free(s->mark);
    memset(s, 0, sizeof(*s));
}

int64_t or_delaunay(int64_t n, const double *x, const double *y, int32_t *tri, int64_t cap, int64_t *n_degenerate) {
    if (n < 3) return -1;
    int64_t deg0 = g_degenerate;
    bw_state s;
    int rc = bw_build(&s, n, x, y);
    if (rc != 0) { bw_destroy(&s); return -1; }
    int64_t cnt = 0;
    for (int64_t id = 0; id < s.nt; id++) {
        if (!s.t[id].alive || s.t[id].v[2] == GHOST) continue;
        if (cnt < cap) {
            /* rotate so the smallest index comes first (CCW kept) */
            int32_t *v = s.t[id].v, r = 0;
            if (v[1] < v[r]) r = 1;
            if (v[2] < v[r]) r = 2;
            tri[3 * cnt + 0] = v[r]; tri[3 * cnt + 1] = v[(r + 1) % 3]; tri[3 * cnt + 2] = v[(r + 2) % 3];
        }
        cnt++;
    }
    bw_destroy(&s);
    if (n_degenerate) *n_degenerate = g_degenerate - deg0;
    return cnt <= cap ? cnt : -cnt;
}

/* ========================================================================== */
/* Fields: canonical bilinear lookup                   */
/* ========================================================================== */
static void cell_of(const or_fields *f, double x, double y, int *i, int *j, double *s, double *t) {
    double idx = (double)(f->nx - 1) / (f->x1 - f->x0);
    double idy = (double)(f->ny - 1) / (f->y1 - f->y0);
    double u = (x - f->x0) * idx;
    double v = (y - f->y0) * idy;
    double fu = floor(u), fv = floor(v);
    int ii = fu < 0.0 ? 0 : (fu > (double)(f->nx - 2) ? f->nx - 2 : (int)fu);
    int jj = fv < 0.0 ? 0 : (fv > (double)(f->ny - 2) ? f->ny - 2 : (int)fv);
    *i = ii; *j = jj;
    *s = u - (double)ii;
    *t = v - (double)jj;
}

static double lerp(double a, double b, double s) { return a + s * (b - a); }

double or_field_value(const or_fields *f, const double *F, double x, double y) {
    int i, j;
    double s, t;
    cell_of(f, x, y, &i, &j, &s, &t);
    const double *r0 = F + (int64_t)j * f->nx, *r1 = F + (int64_t)(j + 1) * f->nx;
    return lerp(lerp(r0[i], r0[i + 1], s), lerp(r1[i], r1[i + 1], s), t);
}

void or_field_grad(const or_fields *f, const double *F, double x, double y, double *gx, double *gy) {
    int i, j;
    double s, t;
    cell_of(f, x, y, &i, &j, &s, &t);
    const double *r0 = F + (int64_t)j * f->nx, *r1 = F + (int64_t)(j + 1) * f->nx;
    double f00 = r0[i], f10 = r0[i + 1], f01 = r1[i], f11 = r1[i + 1];
    double dx = (f->x1 - f->x0) / (double)(f->nx - 1);
    double dy = (f->y1 - f->y0) / (double)(f->ny - 1);
    *gx = ((1.0 - t) * (f10 - f00) + t * (f11 - f01)) / dx;
    *gy = ((1.0 - s) * (f01 - f00) + s * (f11 - f10)) / dy;
}

static double mu_at(const or_fields *f, double x, double y) {
    return f->mu ? or_field_value(f, f->mu, x, y) : 1.0;
}
static double rho_at(const or_fields *f, double x, double y) {
    return f->rho ? or_field_value(f, f->rho, x, y) : 1.0;
}

/* S0 (§8.0 "Local size"): h(x) = c*mu~(x), c = sqrt( ∫_{phi~<0} mu~^-2 dA / N ),
 * midpoint rule over grid cells whose centre has phi~ < 0, rows then columns;
 * the centre value is the bilinear form at s = t = 1/2.  h_avg = mean of h over
 * those cells. */
void or_domain(const or_fields *f, int64_t n_total, double *c_out, double *h_avg_out) {
    double sum_w = 0.0, sum_mu = 0.0;
    int64_t cnt = 0;
    for (int j = 0; j < f->ny - 1; j++)
        for (int i = 0; i < f->nx - 1; i++) {
            const double *p0 = f->phi + (int64_t)j * f->nx, *p1 = f->phi + (int64_t)(j + 1) * f->nx;
            double ph = lerp(lerp(p0[i], p0[i + 1], 0.5), lerp(p1[i], p1[i + 1], 0.5), 0.5);
            if (!(ph < 0.0)) continue;
            double m = 1.0;
            if (f->mu) {
                const double *m0 = f->mu + (int64_t)j * f->nx, *m1 = f->mu + (int64_t)(j + 1) * f->nx;
                m = lerp(lerp(m0[i], m0[i + 1], 0.5), lerp(m1[i], m1[i + 1], 0.5), 0.5);
            }
            sum_w += 1.0 / (m * m);
            sum_mu += m;
            cnt++;
        }
    double dx = (f->x1 - f->x0) / (double)(f->nx - 1);
    double dy = (f->y1 - f->y0) / (double)(f->ny - 1);
    double c = sqrt(sum_w * (dx * dy) / (double)n_total);
    *c_out = c;
    *h_avg_out = cnt ? c * (sum_mu / (double)cnt) : c;
}

/* ========================================================================== */
/* O2: bounded cells by labelled clipping                                      */
/* ========================================================================== */
static const double OR_COS_PI8 = 0.92387953251128673848; /* cos(pi/8) */
static const double OR_SQRT2 = 1.41421356237309514547;    /* fl(sqrt(2)) */

/* line n.x' = r in coordinates relative to the cell's generator; inside n.x' <= r */
typedef struct { double nx, ny, r; } line2;

/* wall codes: octagon sides k=0..7 -> -1-k ; box: -9 (x<=x1), -10 (y<=y1), -11 (x>=x0), -12 (y>=y0) */
typedef struct {
    const or_fields *f;
    const double *x, *y;
    int32_t i;
    double px, py;
    double r_oct;     /* S*cos(pi/8), S = fac*h(p_i) */
} cellctx;

static line2 line_of(const cellctx *C, int32_t code) {
    line2 L;
    if (code >= 0) {
        L.nx = C->x[code] - C->px;
        L.ny = C->y[code] - C->py;
        L.r = 0.5 * (L.nx * L.nx + L.ny * L.ny);
        return L;
    }
    static const double onx[8] = {1, 1, 0, -1, -1, -1, 0, 1};
    static const double ony[8] = {0, 1, 1, 1, 0, -1, -1, -1};
    if (code >= -8) {
        int k = -1 - code;
        L.nx = onx[k]; L.ny = ony[k];
        L.r = (k % 2 == 0) ? C->r_oct : OR_SQRT2 * C->r_oct;
        return L;
    }
    switch (code) {
    case -9:  L.nx = 1;  L.ny = 0;  L.r = C->f->x1 - C->px; break;
    case -10: L.nx = 0;  L.ny = 1;  L.r = C->f->y1 - C->py; break;
    case -11: L.nx = -1; L.ny = 0;  L.r = C->px - C->f->x0; break;
    default:  L.nx = 0;  L.ny = -1; L.r = C->py - C->f->y0; break;
    }
    return L;
}

/* Cramer intersection of two lines, relative coordinates, in the form SURVEY §8.0
 * "Canonical wall vertices" writes down: det = n_a.x n_b.y - n_a.y n_b.x,
 * x' = (r_a n_b.y - n_a.y r_b)/det, y' = (n_a.x r_b - r_a n_b.x)/det (correctly rounded
 * divisions).  Exactly symmetric in (A, B): det and both numerators change sign. */
static void cramer(line2 A, line2 B, double *x, double *y) {
    double det = A.nx * B.ny - A.ny * B.nx;
    *x = (A.r * B.ny - A.ny * B.r) / det;
    *y = (A.nx * B.r - A.r * B.nx) / det;
}

typedef struct { int32_t la, lb; double x, y; } cvert;

#define OR_MAXV 512

/* j cuts v?  pp vertices: exact incircle (i, la, lb) vs j, orientation checked;
 * wall vertices: canonical floating test n.x' > r (L25). */
static int vertex_out(const cellctx *C, const cvert *v, int32_t code, line2 L) {
    if (code >= 0 && v->la >= 0 && v->lb >= 0) {
        double Pi[2] = {C->px, C->py}, Pa[2] = {C->x[v->la], C->y[v->la]};
        double Pb[2] = {C->x[v->lb], C->y[v->lb]}, Pj[2] = {C->x[code], C->y[code]};
        int o = or_orient2d(Pi, Pa, Pb);
        if (o <= 0) g_degenerate++;
        int ic = or_incircle(Pi, Pa, Pb, Pj);
        return ic * o > 0;
    }
    double lhs = L.nx * v->x + L.ny * v->y;
    return lhs > L.r;
}

/* Sutherland-Hodgman clip of poly (in place) by line 'code'. returns new count or -1 */
static int clip_poly(const cellctx *C, cvert *poly, int nv, int32_t code, cvert *tmp) {
    line2 L = line_of(C, code);
    int out[OR_MAXV];
    int any = 0, all = 1;
    for (int k = 0; k < nv; k++) {
        out[k] = vertex_out(C, &poly[k], code, L);
        any |= out[k];
        all &= out[k];
    }
    if (!any) return nv;
    if (all) { g_degenerate++; return -1; }
    int transitions = 0;
    for (int k = 0; k < nv; k++) transitions += out[k] != out[(k + 1) % nv];
    if (transitions != 2) g_degenerate++;
    int m = 0;
    for (int k = 0; k < nv; k++) {
        const cvert *a = &poly[k], *b = &poly[(k + 1) % nv];
        int32_t e = a->lb; /* line of edge a->b */
        if (!out[k] && !out[(k + 1) % nv]) {
            tmp[m++] = *b;
        } else if (!out[k] && out[(k + 1) % nv]) {
            cvert w; w.la = e; w.lb = code; cramer(line_of(C, e), L, &w.x, &w.y); tmp[m++] = w;
        } else if (out[k] && !out[(k + 1) % nv]) {
            cvert w; w.la = code; w.lb = e; cramer(L, line_of(C, e), &w.x, &w.y); tmp[m++] = w;
            tmp[m++] = *b;
        }
        if (m >= OR_MAXV - 2) ORACLE_DIE("cell vertex overflow");
    }
    memcpy(poly, tmp, sizeof(cvert) * (size_t)m);
    return m;
}

static int label_less(const cvert *a, const cvert *b) {
    if (a->la != b->la) return a->la < b->la;
    return a->lb < b->lb;
}

/* rotate so the smallest (la,lb) tuple is first (CCW order kept) */
static void canonical_rotate(cvert *poly, int nv, cvert *tmp) {
    int s = 0;
    for (int k = 1; k < nv; k++) if (label_less(&poly[k], &poly[s])) s = k;
    for (int k = 0; k < nv; k++) tmp[k] = poly[(s + k) % nv];
    memcpy(poly, tmp, sizeof(cvert) * (size_t)nv);
}

static double h_of(const or_fields *f, double c, double x, double y) { return c * mu_at(f, x, y); }

static double r_oct_of(const or_fields *f, const or_params *p, double c, double x, double y) {
    double h = h_of(f, c, x, y);
    double S = p->fac_voro_bound * h;
    return S * OR_COS_PI8;
}

/* B ∩ Oct_i ∩ ⋂_{j in nbrs} H_ij  (O2) */
static int build_cell(const cellctx *C, const int32_t *nbrs, int nn, cvert *poly, cvert *tmp) {
    int nv = 8;
    for (int k = 0; k < 8; k++) {
        poly[k].la = -1 - k;
        poly[k].lb = -1 - ((k + 1) % 8);
        cramer(line_of(C, poly[k].la), line_of(C, poly[k].lb), &poly[k].x, &poly[k].y);
    }
    static const int32_t box_codes[4] = {-9, -10, -11, -12};
    for (int b = 0; b < 4; b++) {
        nv = clip_poly(C, poly, nv, box_codes[b], tmp);
        if (nv < 0) return -1;
    }
    for (int k = 0; k < nn; k++) {
        nv = clip_poly(C, poly, nv, nbrs[k], tmp);
        if (nv < 0) return -1;
    }
    canonical_rotate(poly, nv, tmp);
    return nv;
}

/* ---------------------------------------------------------------------------
 * Delaunay adjacency (CSR over vertices) from the triangle list
 * ------------------------------------------------------------------------- */
typedef struct { int64_t *start; int32_t *nb; } csr;

static int cmp_i32(const void *a, const void *b) {
    int32_t p = *(const int32_t *)a, q = *(const int32_t *)b;
    return p < q ? -1 : (p > q);
}

static csr build_neighbours(int64_t n, int64_t nt, const int32_t *tri) {
    csr g;
    g.start = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
    for (int64_t t = 0; t < nt; t++)
        for (int k = 0; k < 3; k++) g.start[tri[3 * t + k] + 1] += 2;
    for (int64_t i = 0; i < n; i++) g.start[i + 1] += g.start[i];
    g.nb = (int32_t *)malloc(sizeof(int32_t) * (size_t)(g.start[n] + 1));
    int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    for (int64_t i = 0; i < n; i++) fill[i] = g.start[i];
    for (int64_t t = 0; t < nt; t++)
        for (int k = 0; k < 3; k++) {
            int32_t a = tri[3 * t + k];
            g.nb[fill[a]++] = tri[3 * t + (k + 1) % 3];
            g.nb[fill[a]++] = tri[3 * t + (k + 2) % 3];
        }
    /* sort + unique per row, compact */
    int64_t w = 0;
    for (int64_t i = 0; i < n; i++) {
        int64_t s = g.start[i], e = g.start[i + 1];
        qsort(g.nb + s, (size_t)(e - s), sizeof(int32_t), cmp_i32);
        int64_t row = w;
        for (int64_t k = s; k < e; k++)
            if (k == s || g.nb[k] != g.nb[k - 1]) g.nb[w++] = g.nb[k];
        g.start[i] = row;
    }
    g.start[n] = w;
    free(fill);
    return g;
}

int64_t or_cells(const or_fields *f, const or_params *p, int64_t n, const double *x, const double *y,
                 int64_t *cell_start, int32_t *la, int32_t *lb, double *vx, double *vy, int64_t vcap,
                 or_info *info) {
    int64_t deg0 = g_degenerate;
    int64_t cap = 2 * n + 16;
    int32_t *tri = (int32_t *)malloc(sizeof(int32_t) * 3 * (size_t)cap);
    int64_t nt;
    csr g;
    if (n < 3) {
        /* fewer than 3 points: every other point is a neighbour */
        nt = 0;
        g.start = (int64_t *)calloc((size_t)n + 1, sizeof(int64_t));
        g.nb = (int32_t *)malloc(sizeof(int32_t) * 4);
        for (int64_t i = 0; i < n; i++) {
            g.start[i + 1] = g.start[i];
            for (int64_t j = 0; j < n; j++)
                if (j != i) g.nb[g.start[i + 1]++] = (int32_t)j;
        }
    } else {
        nt = or_delaunay(n, x, y, tri, cap, NULL);
        if (nt < 0) { free(tri); return 0; }
        g = build_neighbours(n, nt, tri);
    }
    double c, havg;
    or_domain(f, n, &c, &havg);
    cvert poly[OR_MAXV], tmp[OR_MAXV];
    int64_t tot = 0;
    for (int64_t i = 0; i < n; i++) {
        cellctx C = {f, x, y, (int32_t)i, x[i], y[i], r_oct_of(f, p, c, x[i], y[i])};
        int nv = build_cell(&C, g.nb + g.start[i], (int)(g.start[i + 1] - g.start[i]), poly, tmp);
        if (nv < 0) nv = 0;
        cell_start[i] = tot;
        for (int k = 0; k < nv; k++) {
            if (tot < vcap) { la[tot] = poly[k].la; lb[tot] = poly[k].lb; vx[tot] = poly[k].x; vy[tot] = poly[k].y; }
            tot++;
        }
    }
    cell_start[n] = tot;
    if (info) {
        info->c = c; info->h_avg = havg; info->n_delaunay = nt;
        info->n_degenerate = g_degenerate - deg0;
    }
    free(tri); free(g.start); free(g.nb);
    return tot <= vcap ? tot : -tot;
}

/* ========================================================================== */
/* O3: keep rule                                                               */
/* ========================================================================== */
static int in_octagon(double cx, double cy, double qx, double qy, double r) {
    double dx = cx - qx, dy = cy - qy;
    double r2 = OR_SQRT2 * r;
    return fabs(dx) < r && fabs(dy) < r && fabs(dx + dy) < r2 && fabs(dx - dy) < r2;
}

/* geps(x) = fac_geps * min(h(x), h_avg)   (reading L20 evaluated at x) */
static double geps_at(const or_fields *f, const or_params *p, double c, double h_avg, double x, double y) {
    const double h = c * (f->mu ? or_field_value(f, f->mu, x, y) : 1.0);
    return p->fac_geps * (h < h_avg ? h : h_avg);
}

/* NEXT-2: the paper's validity tests on a triangle whose circumcentre passed the bounded-cell
 * conditions (§4.1, reading L43).  (ox, oy): canonical circumcentre relative to p_u.
 *   Test 1: the centroid g; discard iff phi~(g) > geps(g).
 *   Test 2: count the edge midpoints m with phi~(m) <= geps(m); valid iff >= 2.
 *   Test 3: otherwise discard iff |phi~(c_circ)| / R_circ > T^tria. */
static int validity_tests(const or_fields *f, const or_params *p, double c, double h_avg, const double *x,
                          const double *y, int32_t u, int32_t v, int32_t w, double ox, double oy) {
    const double gx = ((x[u] + x[v]) + x[w]) / 3.0, gy = ((y[u] + y[v]) + y[w]) / 3.0;
    const double pg = or_field_value(f, f->phi, gx, gy), eg = geps_at(f, p, c, h_avg, gx, gy);
    near_tie(pg, eg, eg);
    if (pg > eg) return 0;                                   /* Test 1: centroid outside */
    const int32_t q[3] = {u, v, w};
    int count = 0;
    for (int k = 0; k < 3; k++) {                            /* Test 2: edges (u,v), (v,w), (w,u) */
        const int32_t a = q[k], b = q[(k + 1) % 3];
        const double mx = (x[a] + x[b]) * 0.5, my = (y[a] + y[b]) * 0.5;
        const double pm = or_field_value(f, f->phi, mx, my), em = geps_at(f, p, c, h_avg, mx, my);
        near_tie(pm, em, em);
        if (pm <= em) count++;
    }
    if (count >= 2) return 1;
    const double R = sqrt(ox * ox + oy * oy);                /* Test 3: circumcentre */
    const double pc = or_field_value(f, f->phi, x[u] + ox, y[u] + oy);
    near_tie(fabs(pc) / R, p->t_circ, 1.0);
    return !(fabs(pc) / R > p->t_circ);
}

/* t = {u<v<w}: keep iff c_t strictly in B and in all three octagons and phi~(g_t) < tau
 * (validity 0, L10), or the paper's Tests 1-3 (validity 1, NEXT-2) */
static int keep_triangle(const or_fields *f, const or_params *p, double c, double h_avg, const double *x,
                         const double *y, int32_t u, int32_t v, int32_t w) {
    /* canonical circumcentre relative to p_u, as the Cramer intersection of the two bisectors */
    line2 A, B;
    A.nx = x[v] - x[u]; A.ny = y[v] - y[u]; A.r = 0.5 * (A.nx * A.nx + A.ny * A.ny);
    B.nx = x[w] - x[u]; B.ny = y[w] - y[u]; B.r = 0.5 * (B.nx * B.nx + B.ny * B.ny);
    double ox, oy;
    cramer(A, B, &ox, &oy);
    double cx = x[u] + ox, cy = y[u] + oy;
    const double Lb = (f->x1 - f->x0) + (f->y1 - f->y0);
    near_tie(cx, f->x0, Lb); near_tie(cx, f->x1, Lb); near_tie(cy, f->y0, Lb); near_tie(cy, f->y1, Lb);
    if (!(cx > f->x0 && cx < f->x1 && cy > f->y0 && cy < f->y1)) return 0;
    int32_t q[3] = {u, v, w};
    for (int k = 0; k < 3; k++) {
        const double r = r_oct_of(f, p, c, x[q[k]], y[q[k]]);
        const double dx = cx - x[q[k]], dy = cy - y[q[k]];
        near_tie(fabs(dx), r, r); near_tie(fabs(dy), r, r);
        near_tie(fabs(dx + dy), OR_SQRT2 * r, r); near_tie(fabs(dx - dy), OR_SQRT2 * r, r);
        if (!in_octagon(cx, cy, x[q[k]], y[q[k]], r)) return 0;
    }
    if (p->validity) return validity_tests(f, p, c, h_avg, x, y, u, v, w, ox, oy);
    double gx = ((x[u] + x[v]) + x[w]) / 3.0, gy = ((y[u] + y[v]) + y[w]) / 3.0;
    const double ph = or_field_value(f, f->phi, gx, gy);
    near_tie(ph, p->keep_tol, sqrt(ox * ox + oy * oy));
    return ph < p->keep_tol;
}

/* ========================================================================== */
/* O4: CVD centroid (quadrature P:537-553, L13)                      */
/* ========================================================================== */
typedef struct { double ax, ay, bx, by, cx, cy; } qtri;

static void quad_accumulate(const or_fields *f, double gx0, double gy0, qtri t, int depth,
                            double *sw, double *swx, double *swy, int64_t *nq) {
    if (depth == 0) {
        double cr = (t.bx - t.ax) * (t.cy - t.ay) - (t.by - t.ay) * (t.cx - t.ax);
        double A = 0.5 * cr;
        double qx = ((t.ax + t.bx) + t.cx) / 3.0, qy = ((t.ay + t.by) + t.cy) / 3.0;
        double r = rho_at(f, gx0 + qx, gy0 + qy);
        double wgt = A * r;
        *sw += wgt; *swx += wgt * qx; *swy += wgt * qy;
        (*nq)++;
        return;
    }
    /* split at the midpoint of the longest edge: first of (e01,e12,e20) under strict > */
    double P[3][2] = {{t.ax, t.ay}, {t.bx, t.by}, {t.cx, t.cy}};
    double best = -1.0;
    int e = 0;
    for (int k = 0; k < 3; k++) {
        double dx = P[(k + 1) % 3][0] - P[k][0], dy = P[(k + 1) % 3][1] - P[k][1];
        double L = dx * dx + dy * dy;
        if (L > best) { best = L; e = k; }
    }
    double *Pa = P[e], *Pb = P[(e + 1) % 3], *Pc = P[(e + 2) % 3];
    double mx = (Pa[0] + Pb[0]) * 0.5, my = (Pa[1] + Pb[1]) * 0.5;
    qtri c0 = {Pa[0], Pa[1], mx, my, Pc[0], Pc[1]};
    qtri c1 = {mx, my, Pb[0], Pb[1], Pc[0], Pc[1]};
    quad_accumulate(f, gx0, gy0, c0, depth - 1, sw, swx, swy, nq);
    quad_accumulate(f, gx0, gy0, c1, depth - 1, sw, swx, swy, nq);
}

/* polygon given RELATIVE to generator (gx,gy); returns relative centroid */
static void cvd_rel(const or_fields *f, const or_params *p, int nv, const double *px, const double *py,
                    double gx, double gy, double h, double d_prev, double *cx, double *cy, int *levels,
                    int64_t *nq) {
    if (!f->rho) {
        /* uniform density: exact polygon centroid by the fan from the generator */
        double A2 = 0.0, sx = 0.0, sy = 0.0;
        for (int k = 0; k < nv; k++) {
            int k1 = (k + 1) % nv;
            double cr = px[k] * py[k1] - px[k1] * py[k];
            A2 += cr;
            sx += cr * (px[k] + px[k1]);
            sy += cr * (py[k] + py[k1]);
        }
        *cx = sx / (3.0 * A2);
        *cy = sy / (3.0 * A2);
        if (levels) *levels = 1;
        if (nq) *nq += nv;
        return;
    }
    double area2 = 0.0;
    for (int k = 0; k < nv; k++) {
        int k1 = (k + 1) % nv;
        area2 += px[k] * py[k1] - px[k1] * py[k];
    }
    double area = 0.5 * area2;
    double eps = d_prev >= 0.0 ? d_prev / h : p->fac_pt_mvmt;
    if (eps < p->fac_end_mvmt) eps = p->fac_end_mvmt;
    double E = sqrt(area) * eps;
    double prevx = 0.0, prevy = 0.0; /* c^_0 = generator */
    int L;
    for (L = 1; L <= p->quad_max_level; L++) {
        double sw = 0.0, swx = 0.0, swy = 0.0;
        for (int k = 0; k < nv; k++) {
            int k1 = (k + 1) % nv;
            qtri t = {0.0, 0.0, px[k], py[k], px[k1], py[k1]};
            quad_accumulate(f, gx, gy, t, L - 1, &sw, &swx, &swy, nq);
        }
        double curx = swx / sw, cury = swy / sw;
        double dx = prevx - curx, dy = prevy - cury;
        double dist = sqrt(dx * dx + dy * dy);
        prevx = curx; prevy = cury;
        near_tie(dist, E, E);
        if (dist < E) break;        /* |c^_{L-1} - c^_L| < E  -> return c^_L */
    }
    if (L > p->quad_max_level) L = p->quad_max_level;
    *cx = prevx; *cy = prevy;
    if (levels) *levels = L;
}

void or_cvd_polygon(const or_fields *f, const or_params *p, int nv, const double *px, const double *py,
                    double gx, double gy, double h, double d_prev, double *cx, double *cy, int *levels) {
    double rx[OR_MAXV], ry[OR_MAXV];
    for (int k = 0; k < nv; k++) { rx[k] = px[k] - gx; ry[k] = py[k] - gy; }
    int64_t nq = 0;
    cvd_rel(f, p, nv, rx, ry, gx, gy, h, d_prev, cx, cy, levels, &nq);
    *cx = gx + *cx;
    *cy = gy + *cy;
}

/* ========================================================================== */
/* O5: DistMesh (Eqs. spring force, size scaling, Euler; L1-L4)                */
/* ========================================================================== */
void or_distmesh(const or_fields *f, const or_params *p, int64_t n, const double *x, const double *y,
                 int64_t ne, const int32_t *edges, const uint8_t *fixed,
                 double *x_hat, double *y_hat, double *fac_mu_out) {
    double sum_l2 = 0.0, sum_mu2 = 0.0;
    for (int64_t e = 0; e < ne; e++) {
        int32_t a = edges[2 * e], b = edges[2 * e + 1];
        double dx = x[a] - x[b], dy = y[a] - y[b];
        double mx = (x[a] + x[b]) * 0.5, my = (y[a] + y[b]) * 0.5;
        double m = mu_at(f, mx, my);
        sum_l2 += dx * dx + dy * dy;
        sum_mu2 += m * m;
    }
    double fac_mu = sqrt(sum_l2 / sum_mu2);
    if (fac_mu_out) *fac_mu_out = fac_mu;
    double *Fx = (double *)calloc((size_t)n, sizeof(double));
    double *Fy = (double *)calloc((size_t)n, sizeof(double));
    for (int64_t e = 0; e < ne; e++) {
        int32_t a = edges[2 * e], b = edges[2 * e + 1];
        double dx = x[a] - x[b], dy = y[a] - y[b];
        double l = sqrt(dx * dx + dy * dy);
        double mx = (x[a] + x[b]) * 0.5, my = (y[a] + y[b]) * 0.5;
        double l0 = mu_at(f, mx, my) * p->fscale * fac_mu;
        if (l < l0) {
            double fm = l0 - l; /* k = 1 (L3): only dt*k enters */
            double ux = dx / l, uy = dy / l;
            Fx[a] += fm * ux; Fy[a] += fm * uy;   /* repulsive: pushes a away from b */
            Fx[b] -= fm * ux; Fy[b] -= fm * uy;
        }
    }
    for (int64_t i = 0; i < n; i++) {
        if (fixed && fixed[i]) { x_hat[i] = x[i]; y_hat[i] = y[i]; continue; }
        x_hat[i] = x[i] + p->dt_k * Fx[i];
        y_hat[i] = y[i] + p->dt_k * Fy[i];
    }
    free(Fx); free(Fy);
}

/* ========================================================================== */
/* O6: treatment of the updated point (L20-L22) */
/* ========================================================================== */
static double clampd(double v, double lo, double hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* NEXT-1: the paper's projection of escaped points (Fig. 13).
 * Sphere tracing ([hart1995]): from the inner p_old toward p_new, step by the circle of
 * radius |sdf(q)| around the current point q, q <- q + |sdf(q)| u (u the unit direction of the
 * segment, a step never passing p_new), until |sdf(q)| <= geps; at most trace_max steps (L39). */
static int sphere_trace(const or_fields *f, const or_params *p, double xo, double yo, double xn, double yn,
                        double geps, double *qx_out, double *qy_out) {
    double dx = xn - xo, dy = yn - yo;
    double len = sqrt(dx * dx + dy * dy);
    double ux = dx / len, uy = dy / len;
    double qx = xo, qy = yo, s = 0.0;
    for (int k = 0; k < p->trace_max; k++) {
        double v = or_field_value(f, f->phi, qx, qy);
        near_tie(fabs(v), geps, geps);
        if (fabs(v) <= geps) { *qx_out = qx; *qy_out = qy; return 1; }
        double r = fabs(v);
        if (s + r > len) r = len - s;
        s = s + r;
        qx = qx + r * ux;
        qy = qy + r * uy;
    }
    double v = or_field_value(f, f->phi, qx, qy);
    *qx_out = qx; *qy_out = qy;
    return fabs(v) <= geps;
}

/* Finite-difference derivatives of sdf~ with step d ("approximated with the finite
 * difference method of step size deps"): central differences (reading L41). */
static void fd_derivs(const or_fields *f, double x, double y, double d, double *fx, double *fy,
                      double *fxx, double *fyy, double *fxy) {
    const double *F = f->phi;
    double f0 = or_field_value(f, F, x, y);
    double fxp = or_field_value(f, F, x + d, y), fxm = or_field_value(f, F, x - d, y);
    double fyp = or_field_value(f, F, x, y + d), fym = or_field_value(f, F, x, y - d);
    double fpp = or_field_value(f, F, x + d, y + d), fpm = or_field_value(f, F, x + d, y - d);
    double fmp = or_field_value(f, F, x - d, y + d), fmm = or_field_value(f, F, x - d, y - d);
    *fx = (fxp - fxm) / (2.0 * d);
    *fy = (fyp - fym) / (2.0 * d);
    *fxx = ((fxp - 2.0 * f0) + fxm) / (d * d);
    *fyy = ((fyp - 2.0 * f0) + fym) / (d * d);
    *fxy = (((fpp - fpm) - fmp) + fmm) / (4.0 * d * d);
}

/* Point projection by the damped Newton method: solve
 * L(p) = [sdf(p), (p - p_new) x grad sdf(p)] = 0 (Eq. projection_point_requirement, written
 * with the gradient at p as its Jacobian Eq. projection_Newton_Jacobian requires, L36), from
 * p_new, p <- p - alpha J^-1 L (Eq. projection_pt_update), clamped into B, until
 * |sdf(p)| <= geps or newton_max steps. */
static int newton_project(const or_fields *f, const or_params *p, double xn, double yn, double geps,
                          double deps, double *qx_out, double *qy_out) {
    double x = xn, y = yn;
    int ok = 0;
    for (int k = 0; k < p->newton_max; k++) {
        double fx, fy, fxx, fyy, fxy;
        fd_derivs(f, x, y, deps, &fx, &fy, &fxx, &fyy, &fxy);
        double L1 = or_field_value(f, f->phi, x, y);
        double ex = x - xn, ey = y - yn;
        double L2 = ex * fy - ey * fx;
        double J11 = fx, J12 = fy;
        double J21 = (fy + ex * fxy) - ey * fxx;
        double J22 = (-fx - ey * fxy) + ex * fyy;
        double det = J11 * J22 - J12 * J21;
        if (!(det != 0.0)) break;
        double sx = (L1 * J22 - J12 * L2) / det;
        double sy = (J11 * L2 - J21 * L1) / det;
        x = clampd(x - p->newton_damping * sx, f->x0, f->x1);
        y = clampd(y - p->newton_damping * sy, f->y0, f->y1);
        double v = or_field_value(f, f->phi, x, y);
        near_tie(fabs(v), geps, geps);
        if (fabs(v) <= geps) { ok = 1; break; }
    }
    *qx_out = x; *qy_out = y;
    return ok;
}

int or_treat(const or_fields *f, const or_params *p, double c, double h_avg,
             double xo, double yo, double xh, double yh, double *xn, double *yn, double *dprev) {
    int status = 0;
    double h = h_of(f, c, xo, yo);
    double T = p->fac_pt_mvmt * h;
    double dx = xh - xo, dy = yh - yo;
    double len = sqrt(dx * dx + dy * dy);
    if (len > T) {
        double sc = T / len;
        dx = dx * sc; dy = dy * sc;
        status |= 4;
    }
    double qx = clampd(xo + dx, f->x0, f->x1), qy = clampd(yo + dy, f->y0, f->y1);
    double hm = h < h_avg ? h : h_avg;
    double geps = p->fac_geps * hm;
    double ph = or_field_value(f, f->phi, qx, qy);
    near_tie(ph, geps, geps);
    if (!(ph <= geps)) {
        int ok = 0;
        if (p->projection == 1) {
            /* Fig. 13: an inner p_old (sdf < -geps) is sphere-traced toward p_new;
             * a boundary (or outside) p_old projects p_new by the 2x2 damped Newton method */
            double po = or_field_value(f, f->phi, xo, yo);
            double px_, py_;
            if (po < -geps) {
                ok = sphere_trace(f, p, xo, yo, qx, qy, geps, &px_, &py_);
                status |= 8;
            } else {
                double deps = 1.4901161193847656e-08 * hm;  /* sqrt(DBL_EPSILON) min(h, h_avg) */
                ok = newton_project(f, p, qx, qy, geps, deps, &px_, &py_);
            }
            qx = px_; qy = py_;
        } else {
            for (int it = 0; it < p->newton_max; it++) {
                double gx, gy;
                or_field_grad(f, f->phi, qx, qy, &gx, &gy);
                double g2 = gx * gx + gy * gy;
                if (!(g2 > 0.0)) break;
                double st = p->newton_damping * ph / g2;
                qx = clampd(qx - st * gx, f->x0, f->x1);
                qy = clampd(qy - st * gy, f->y0, f->y1);
                ph = or_field_value(f, f->phi, qx, qy);
                near_tie(fabs(ph), geps, geps);
                if (fabs(ph) <= geps) { ok = 1; break; }
            }
        }
        if (ok) status |= 1;
        else { qx = xo; qy = yo; status = (status & 4) | 2; }
    }
    *xn = qx; *yn = qy;
    double ex = qx - xo, ey = qy - yo;
    *dprev = sqrt(ex * ex + ey * ey);
    return status;
}

int or_distmesh_lazy(const or_fields *f, const or_params *p, int64_t n, int64_t n_total,
                     const double *x, const double *y, int64_t ne, const int32_t *edges,
                     const double *x_tria, const double *y_tria,
                     double *x_out, double *y_out, double *d_prev_out, int8_t *status, int32_t *retria) {
    double c, h_avg;
    or_domain(f, n_total > 0 ? n_total : n, &c, &h_avg);
    double *xh = (double *)malloc(sizeof(double) * (size_t)n);
    double *yh = (double *)malloc(sizeof(double) * (size_t)n);
    or_distmesh(f, p, n, x, y, ne, edges, NULL, xh, yh, NULL);
    int32_t flag = 0;
    for (int64_t i = 0; i < n; i++) {
        status[i] = (int8_t)or_treat(f, p, c, h_avg, x[i], y[i], xh[i], yh[i], &x_out[i], &y_out[i], &d_prev_out[i]);
        /* movement since the last triangulation against T_retria = fac_retria h(p_tria) */
        double ex = x_out[i] - x_tria[i], ey = y_out[i] - y_tria[i];
        double d = sqrt(ex * ex + ey * ey);
        double T = p->fac_retria * h_of(f, c, x_tria[i], y_tria[i]);
        near_tie(d, T, T);
        if (d > T) flag = 1;
    }
    *retria = flag;
    free(xh); free(yh);
    return 0;
}

/* ========================================================================== */
/* O7: quality (Eqs. aspect/edge ratios, 1/2-mean)                             */
/* ========================================================================== */
void or_triangle_quality(const double *a, const double *b, const double *c, double *alpha, double *beta) {
    double la = sqrt((b[0] - c[0]) * (b[0] - c[0]) + (b[1] - c[1]) * (b[1] - c[1]));
    double lb = sqrt((a[0] - c[0]) * (a[0] - c[0]) + (a[1] - c[1]) * (a[1] - c[1]));
    double lc = sqrt((a[0] - b[0]) * (a[0] - b[0]) + (a[1] - b[1]) * (a[1] - b[1]));
    double cross = (b[0] - a[0]) * (c[1] - a[1]) - (b[1] - a[1]) * (c[0] - a[0]);
    double s = 0.5 * (la + lb + lc);
    /* R = la lb lc / (4A), r_in = A/s, A = |cross|/2  =>  alpha = R/(2 r_in) = la lb lc s / (2 cross^2) */
    *alpha = (la * lb * lc * s) / (2.0 * cross * cross);
    double mx = la > lb ? (la > lc ? la : lc) : (lb > lc ? lb : lc);
    double mn = la < lb ? (la < lc ? la : lc) : (lb < lc ? lb : lc);
    *beta = mx / mn;
}

/* out12: n, sum sqrt(alpha), sum sqrt(beta), max alpha, max beta, sum alpha, sum alpha^2,
 *        sum beta, sum beta^2, #(alpha<1.2), #(alpha<2), half-mean alpha */
void or_stats(int64_t n_tri, const int32_t *tri, const double *x, const double *y, double *o) {
    for (int k = 0; k < 12; k++) o[k] = 0.0;
    for (int64_t t = 0; t < n_tri; t++) {
        double A[2] = {x[tri[3 * t]], y[tri[3 * t]]}, B[2] = {x[tri[3 * t + 1]], y[tri[3 * t + 1]]};
        double C[2] = {x[tri[3 * t + 2]], y[tri[3 * t + 2]]};
        double al, be;
        or_triangle_quality(A, B, C, &al, &be);
        o[0] += 1.0; o[1] += sqrt(al); o[2] += sqrt(be);
        if (al > o[3]) o[3] = al;
        if (be > o[4]) o[4] = be;
        o[5] += al; o[6] += al * al; o[7] += be; o[8] += be * be;
        o[9] += al < 1.2; o[10] += al < 2.0;
    }
    if (o[0] > 0) { double m = o[1] / o[0]; o[11] = m * m; }
}

/* ========================================================================== */
/* One iteration                                                                */
/* ========================================================================== */
typedef struct { int32_t a, b; } edge2;
static int cmp_edge(const void *p, const void *q) {
    const edge2 *a = (const edge2 *)p, *b = (const edge2 *)q;
    if (a->a != b->a) return a->a < b->a ? -1 : 1;
    return a->b < b->b ? -1 : (a->b > b->b);
}

/* number of points within distance 2R of p_i (O8 n_cert), via a coarse uniform grid */
typedef struct { int nbx, nby; double x0, y0, sx, sy; int64_t *start; int32_t *idx; } cgrid;

static cgrid cgrid_build(int64_t n, const double *x, const double *y, const or_fields *f) {
    cgrid g;
    g.nbx = (int)ceil(sqrt((double)n / 3.3)); if (g.nbx < 1) g.nbx = 1;
    g.nby = g.nbx;
    g.x0 = f->x0; g.y0 = f->y0;
    g.sx = (f->x1 - f->x0) / g.nbx; g.sy = (f->y1 - f->y0) / g.nby;
    int64_t nb = (int64_t)g.nbx * g.nby;
    g.start = (int64_t *)calloc((size_t)nb + 1, sizeof(int64_t));
    g.idx = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    int32_t *key = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    for (int64_t i = 0; i < n; i++) {
        int bx = (int)((x[i] - g.x0) / g.sx), by = (int)((y[i] - g.y0) / g.sy);
        bx = bx < 0 ? 0 : (bx >= g.nbx ? g.nbx - 1 : bx);
        by = by < 0 ? 0 : (by >= g.nby ? g.nby - 1 : by);
        key[i] = by * g.nbx + bx;
        g.start[key[i] + 1]++;
    }
    for (int64_t b = 0; b < nb; b++) g.start[b + 1] += g.start[b];
    int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (size_t)nb);
    for (int64_t b = 0; b < nb; b++) fill[b] = g.start[b];
    for (int64_t i = 0; i < n; i++) g.idx[fill[key[i]]++] = (int32_t)i;
    free(fill); free(key);
    return g;
}

static int64_t cgrid_count(const cgrid *g, const double *x, const double *y, double px, double py, double rad) {
    int bx0 = (int)floor((px - rad - g->x0) / g->sx), bx1 = (int)floor((px + rad - g->x0) / g->sx);
    int by0 = (int)floor((py - rad - g->y0) / g->sy), by1 = (int)floor((py + rad - g->y0) / g->sy);
    if (bx0 < 0) bx0 = 0;
    if (by0 < 0) by0 = 0;
    if (bx1 >= g->nbx) bx1 = g->nbx - 1;
    if (by1 >= g->nby) by1 = g->nby - 1;
    int64_t c = 0;
    for (int by = by0; by <= by1; by++)
        for (int bx = bx0; bx <= bx1; bx++) {
            int64_t b = (int64_t)by * g->nbx + bx;
            for (int64_t k = g->start[b]; k < g->start[b + 1]; k++) {
                int32_t j = g->idx[k];
                double dx = x[j] - px, dy = y[j] - py;
                if (dx * dx + dy * dy < rad * rad) c++;
            }
        }
    return c - 1; /* exclude the point itself */
}

int or_iteration(const or_fields *f, const or_params *p, int64_t n, int64_t n_total, const double *x,
                 const double *y, const double *d_prev, int mode, int32_t *tri_out, int64_t tri_cap, int32_t *edges_out,
                 int64_t edge_cap, double *x_hat, double *y_hat, double *x_out, double *y_out,
                 double *d_prev_out, int8_t *status, int64_t *counts, or_info *info) {
    int64_t deg0 = g_degenerate, near0 = g_near;
    or_info inf;
    memset(&inf, 0, sizeof(inf));
    or_domain(f, n_total > 0 ? n_total : n, &inf.c, &inf.h_avg);
    double c = inf.c;
    /* O1 */
    int64_t cap = 2 * n + 16;
    int32_t *D = (int32_t *)malloc(sizeof(int32_t) * 3 * (size_t)cap);
    int64_t nd = or_delaunay(n, x, y, D, cap, NULL);
    if (nd < 0) { free(D); return -1; }
    inf.n_delaunay = nd;
    inf.n_hull = 2 * n - 2 - nd; /* Euler: T = 2n - h - 2 */
    /* O3 */
    int64_t nk = 0;
    int32_t *own = counts ? (int32_t *)calloc((size_t)n, sizeof(int32_t)) : NULL;
    for (int64_t t = 0; t < nd; t++) {
        int32_t u = D[3 * t], v = D[3 * t + 1], w = D[3 * t + 2]; /* u is the min, CCW */
        int32_t lo = v < w ? v : w, hi = v < w ? w : v;
        if (keep_triangle(f, p, c, inf.h_avg, x, y, u, lo, hi)) {
            if (nk < tri_cap) { tri_out[3 * nk] = u; tri_out[3 * nk + 1] = v; tri_out[3 * nk + 2] = w; }
            if (own) own[u]++;
            nk++;
        }
    }
    inf.n_kept = nk;
    if (nk > tri_cap) { free(D); free(own); return -2; }
    /* unique kept edges */
    edge2 *E = (edge2 *)malloc(sizeof(edge2) * 3 * (size_t)(nk + 1));
    for (int64_t t = 0; t < nk; t++)
        for (int k = 0; k < 3; k++) {
            int32_t a = tri_out[3 * t + k], b = tri_out[3 * t + (k + 1) % 3];
            E[3 * t + k].a = a < b ? a : b;
            E[3 * t + k].b = a < b ? b : a;
        }
    qsort(E, (size_t)(3 * nk), sizeof(edge2), cmp_edge);
    int64_t ne = 0;
    for (int64_t k = 0; k < 3 * nk; k++)
        if (k == 0 || E[k].a != E[k - 1].a || E[k].b != E[k - 1].b) E[ne++] = E[k];
    inf.n_edges = ne;
    if (edges_out) {
        if (ne > edge_cap) { free(D); free(own); free(E); return -3; }
        for (int64_t k = 0; k < ne; k++) { edges_out[2 * k] = E[k].a; edges_out[2 * k + 1] = E[k].b; }
    }
    int32_t *erow = NULL;
    if (counts) {
        erow = (int32_t *)calloc((size_t)n, sizeof(int32_t));
        for (int64_t k = 0; k < ne; k++) { erow[E[k].a]++; erow[E[k].b]++; }
    }
    /* O2 + O4 (CVD) or O5 (DistMesh) */
    csr g = build_neighbours(n, nd, D);
    cgrid cg;
    if (counts) cg = cgrid_build(n, x, y, f);
    cvert poly[OR_MAXV], tmp[OR_MAXV];
    double rx[OR_MAXV], ry[OR_MAXV];
    if (mode == 0 || counts) {
        for (int64_t i = 0; i < n; i++) {
            cellctx C = {f, x, y, (int32_t)i, x[i], y[i], r_oct_of(f, p, c, x[i], y[i])};
            int nv = build_cell(&C, g.nb + g.start[i], (int)(g.start[i + 1] - g.start[i]), poly, tmp);
            if (nv < 3) { g_degenerate++; if (mode == 0) { x_hat[i] = x[i]; y_hat[i] = y[i]; } continue; }
            int64_t nq = 0;
            if (mode == 0) {
                for (int k = 0; k < nv; k++) { rx[k] = poly[k].x; ry[k] = poly[k].y; }
                double h = h_of(f, c, x[i], y[i]);
                double dp = d_prev ? d_prev[i] : -1.0;
                double cx, cy;
                cvd_rel(f, p, nv, rx, ry, x[i], y[i], h, dp, &cx, &cy, NULL, &nq);
                x_hat[i] = x[i] + cx;
                y_hat[i] = y[i] + cy;
            }
            if (counts) {
                double R2 = 0.0;
                int64_t deg = 0;
                for (int k = 0; k < nv; k++) {
                    double r2 = poly[k].x * poly[k].x + poly[k].y * poly[k].y;
                    if (r2 > R2) R2 = r2;
                    if (poly[k].lb >= 0) deg++;
                }
                int64_t *cc = counts + 6 * i;
                cc[0] = cgrid_count(&cg, x, y, x[i], y[i], 2.0 * sqrt(R2));
                cc[1] = deg; cc[2] = nv; cc[3] = own[i]; cc[4] = nq; cc[5] = erow[i];
            }
        }
    }
    if (mode == 1) or_distmesh(f, p, n, x, y, ne, (const int32_t *)E, NULL, x_hat, y_hat, &inf.fac_mu);
    if (mode == 1) {
        double sl = 0, sm = 0;
        for (int64_t k = 0; k < ne; k++) {
            double dx = x[E[k].a] - x[E[k].b], dy = y[E[k].a] - y[E[k].b];
            double m = mu_at(f, (x[E[k].a] + x[E[k].b]) * 0.5, (y[E[k].a] + y[E[k].b]) * 0.5);
            sl += dx * dx + dy * dy; sm += m * m;
        }
        inf.sum_l2 = sl; inf.sum_mu2 = sm;
    }
    /* O6 */
    for (int64_t i = 0; i < n; i++)
        status[i] = (int8_t)or_treat(f, p, c, inf.h_avg, x[i], y[i], x_hat[i], y_hat[i], &x_out[i], &y_out[i],
                                     &d_prev_out[i]);
    inf.n_degenerate = g_degenerate - deg0;
    inf.n_near_ties = g_near - near0;
    if (info) *info = inf;
    free(D); free(own); free(E); free(erow); free(g.start); free(g.nb);
    if (counts) { free(cg.start); free(cg.idx); }
    return 0;
}

/* ========================================================================== */
/* NEXT-2 / NEXT-3: controller inputs and point addition          */
/* ========================================================================== */
/* the keep rule (O3) on one triangle, for pin tests: u, v, w any order */
int or_keep_triangle(const or_fields *f, const or_params *p, double c, double h_avg, const double *x,
                     const double *y, int32_t u, int32_t v, int32_t w) {
    int32_t q[3] = {u, v, w};
    for (int a = 0; a < 2; a++)
        for (int b = 0; b < 2 - a; b++)
            if (q[b] > q[b + 1]) { int32_t t = q[b]; q[b] = q[b + 1]; q[b + 1] = t; }
    return keep_triangle(f, p, c, h_avg, x, y, q[0], q[1], q[2]);
}

/* Movement termination input (P:447 T^end_mvmt,i = fac_end * h_i): the number of
 * inner points whose move in this iteration is NOT below its local threshold.  A point is
 * inner iff phi~(p_old) < -geps(p_old) (the tagging rule P:410, reading L38); its move is
 * d_prev = |p_new - p_old| (L32) and its threshold fac_end_mvmt * h(p_old).  Meshing may
 * terminate on movements iff the count is 0. */
int64_t or_move_count(const or_fields *f, const or_params *p, double c, double h_avg, int64_t n,
                      const double *x_old, const double *y_old, const double *d_prev) {
    int64_t cnt = 0;
    for (int64_t i = 0; i < n; i++) {
        const double h = h_of(f, c, x_old[i], y_old[i]);
        const double geps = p->fac_geps * (h < h_avg ? h : h_avg);
        const double ph = or_field_value(f, f->phi, x_old[i], y_old[i]);
        if (!(ph < -geps)) continue;                     /* boundary or outside point */
        if (!(d_prev[i] < p->fac_end_mvmt * h)) cnt++;
    }
    return cnt;
}

/* Point addition (§3.6, after Alliez et al.): rank the triangles by
 * R_circum / h(g) and add one point at the centroid g of each of the n_add largest.
 * Reading L46: a triangle is taken as {u < v < w} (caller indices); its circumcentre is the
 * canonical Cramer intersection of the bisectors of (u,v) and (u,w) relative to p_u (as in the
 * keep rule), R = |c - p_u|, g = ((p_u + p_v) + p_w) / 3, h(g) = c mu~(g).  Ties of the ratio
 * are broken by (u, v) ascending; the new points are written in (u, v) ascending order of their
 * triangles.  Returns the number written (min(n_add, n_tri)). */
typedef struct { double r; int32_t u, v; double gx, gy; } pa_item;
static int cmp_pa_rank(const void *a, const void *b) {
    const pa_item *A = (const pa_item *)a, *B = (const pa_item *)b;
    if (A->r != B->r) return A->r > B->r ? -1 : 1;
    if (A->u != B->u) return A->u < B->u ? -1 : 1;
    return A->v < B->v ? -1 : (A->v > B->v);
}
static int cmp_pa_uv(const void *a, const void *b) {
    const pa_item *A = (const pa_item *)a, *B = (const pa_item *)b;
    if (A->u != B->u) return A->u < B->u ? -1 : 1;
    return A->v < B->v ? -1 : (A->v > B->v);
}
int64_t or_point_addition(const or_fields *f, double c, int64_t n_tri, const int32_t *tri, const double *x,
                          const double *y, int64_t n_add, double *x_new, double *y_new, double *ratio_out) {
    if (n_add > n_tri) n_add = n_tri;
    if (n_add <= 0) return 0;
    pa_item *it = (pa_item *)malloc(sizeof(pa_item) * (size_t)n_tri);
    for (int64_t t = 0; t < n_tri; t++) {
        int32_t q[3] = {tri[3 * t], tri[3 * t + 1], tri[3 * t + 2]};
        for (int a = 0; a < 2; a++)
            for (int b = 0; b < 2 - a; b++)
                if (q[b] > q[b + 1]) { int32_t s = q[b]; q[b] = q[b + 1]; q[b + 1] = s; }
        const int32_t u = q[0], v = q[1], w = q[2];
        line2 A, B;
        A.nx = x[v] - x[u]; A.ny = y[v] - y[u]; A.r = 0.5 * (A.nx * A.nx + A.ny * A.ny);
        B.nx = x[w] - x[u]; B.ny = y[w] - y[u]; B.r = 0.5 * (B.nx * B.nx + B.ny * B.ny);
        double ox, oy;
        cramer(A, B, &ox, &oy);
        const double R = sqrt(ox * ox + oy * oy);
        const double gx = ((x[u] + x[v]) + x[w]) / 3.0, gy = ((y[u] + y[v]) + y[w]) / 3.0;
        const double h = h_of(f, c, gx, gy);
        it[t].r = R / h; it[t].u = u; it[t].v = v; it[t].gx = gx; it[t].gy = gy;
    }
    qsort(it, (size_t)n_tri, sizeof(pa_item), cmp_pa_rank);
    if (ratio_out) ratio_out[0] = it[n_add - 1].r;  /* the smallest selected ratio */
    qsort(it, (size_t)n_add, sizeof(pa_item), cmp_pa_uv);
    for (int64_t k = 0; k < n_add; k++) { x_new[k] = it[k].gx; y_new[k] = it[k].gy; }
    free(it);
    return n_add;
}

/* ========================================================================== */
/* NEXT-4: the set-up pipeline                                   */
/* ========================================================================== */
/* Geometry grid size: lambda = sqrt(N/(N_opt A)), n = ceil(lambda L), n_geo = fac n. */
void or_geometry_grid_dims(int64_t n_total, double n_opt, int32_t fac_grid, double x0, double y0, double x1,
                           double y1, int32_t *nx, int32_t *ny) {
    const double lx = x1 - x0, ly = y1 - y0;
    const double lam = sqrt((double)n_total / (n_opt * (lx * ly)));
    *nx = fac_grid * (int32_t)ceil(lam * lx);
    *ny = fac_grid * (int32_t)ceil(lam * ly);
}

/* Cell categories: m the cell midpoint, l_diag its diagonal; boundary (1) iff
 * |sdf(m)| <= l_diag, else inner (0) iff sdf(m) < 0, else outer (2).  sdf = phi~ (bilinear). */
void or_geometry_categories(const or_fields *f, int32_t nxg, int32_t nyg, int8_t *cat) {
    const double dx = (f->x1 - f->x0) / (double)nxg, dy = (f->y1 - f->y0) / (double)nyg;
    const double ld = sqrt(dx * dx + dy * dy);
    for (int32_t j = 0; j < nyg; j++)
        for (int32_t i = 0; i < nxg; i++) {
            const double mx = f->x0 + ((double)i + 0.5) * dx, my = f->y0 + ((double)j + 0.5) * dy;
            const double s = or_field_value(f, f->phi, mx, my);
            cat[(int64_t)j * nxg + i] = (int8_t)(fabs(s) <= ld ? 1 : (s < 0.0 ? 0 : 2));
        }
}

/* Contour SDF by brute force over all segments: |sdf(p)| = min over segments of the
 * distance to the closest point p* (an endpoint or the foot on the segment, Fig. (c)); the sign
 * is that of -(p - p*).n with n the inward normal of the clockwise loop (right-hand normal of
 * the direction), averaged over the two incident segments when p* is a shared endpoint (Fig.
 * (b)).  Ties of the distance: the smallest segment index.  segs: n_seg x (x1, y1, x2, y2),
 * consecutive and closed (segment k ends where k+1 starts, the last where the first starts).
 * phi: [ny][nx] at the nodes x_i = x0 + i (x1 - x0)/(nx - 1). */
static void seg_closest(const double *s, double px, double py, double *d2, double *t_out) {
    const double ax = s[0], ay = s[1], bx = s[2], by = s[3];
    const double ex = bx - ax, ey = by - ay;
    const double t = ((px - ax) * ex + (py - ay) * ey) / (ex * ex + ey * ey);
    double qx, qy, tt;
    if (t <= 0.0) { qx = ax; qy = ay; tt = 0.0; }
    else if (t >= 1.0) { qx = bx; qy = by; tt = 1.0; }
    else { qx = ax + t * ex; qy = ay + t * ey; tt = t; }
    const double dx = px - qx, dy = py - qy;
    *d2 = dx * dx + dy * dy;
    *t_out = tt;
}
static void seg_normal(const double *s, double *nx, double *ny) {
    const double ex = s[2] - s[0], ey = s[3] - s[1];
    const double l = sqrt(ex * ex + ey * ey);
    *nx = ey / l;
    *ny = -ex / l;
}
double or_contour_sdf_point(const double *segs, int64_t n_seg, double px, double py) {
    int64_t best = -1;
    double bd = 0.0, bt = 0.0;
    for (int64_t k = 0; k < n_seg; k++) {
        double d2, t;
        seg_closest(segs + 4 * k, px, py, &d2, &t);
        if (best < 0 || d2 < bd) { best = k; bd = d2; bt = t; }
    }
    const double *s = segs + 4 * best;
    double nx, ny;
    seg_normal(s, &nx, &ny);
    double qx, qy;
    if (bt == 0.0 || bt == 1.0) {  /* endpoint: average with the incident segment */
        const int64_t o = bt == 0.0 ? (best + n_seg - 1) % n_seg : (best + 1) % n_seg;
        double mx, my;
        seg_normal(segs + 4 * o, &mx, &my);
        nx = (nx + mx) * 0.5;
        ny = (ny + my) * 0.5;
        qx = bt == 0.0 ? s[0] : s[2];
        qy = bt == 0.0 ? s[1] : s[3];
    } else {
        const double ex = s[2] - s[0], ey = s[3] - s[1];
        qx = s[0] + bt * ex;
        qy = s[1] + bt * ey;
    }
    const double d = sqrt(bd);
    const double side = (px - qx) * nx + (py - qy) * ny;
    return side > 0.0 ? -d : d;
}
void or_contour_sdf(const double *segs, int64_t n_seg, int32_t nx, int32_t ny, double x0, double y0, double x1,
                    double y1, double *phi) {
    for (int32_t j = 0; j < ny; j++)
        for (int32_t i = 0; i < nx; i++) {
            const double px = x0 + (double)i * ((x1 - x0) / (double)(nx - 1));
            const double py = y0 + (double)j * ((y1 - y0) / (double)(ny - 1));
            phi[(int64_t)j * nx + i] = or_contour_sdf_point(segs, n_seg, px, py);
        }
}

/* Point initialisation counts: valid cells = inner cells and the boundary cells whose
 * midpoint has sdf(m) <= eta min(dx, dy); rho_i = rho~(m) (1 without rho); rho_norm = rho_i /
 * sum_valid rho (summed in the loop order); n_E = rho_norm N_init.  Floyd-Steinberg (reading L47):
 * rows from the top (largest y) down, each row left to right; v = n_E + received residual,
 * count = max(0, floor(v + 1/2)), R = v - count, R / m to each of the m valid not-yet-visited
 * neighbours among right, below-left, below, below-right.  cat from or_geometry_categories.
 * counts: [nyg][nxg].  Returns the total. */
int64_t or_init_counts(const or_fields *f, int32_t nxg, int32_t nyg, const int8_t *cat, double n_init, double eta,
                       int32_t *counts) {
    const double dx = (f->x1 - f->x0) / (double)nxg, dy = (f->y1 - f->y0) / (double)nyg;
    const double band = eta * (dx < dy ? dx : dy);
    const int64_t nc = (int64_t)nxg * nyg;
    uint8_t *valid = (uint8_t *)calloc((size_t)nc, 1);
    double *rho = (double *)calloc((size_t)nc, sizeof(double));
    double *acc = (double *)calloc((size_t)nc, sizeof(double));
    double S = 0.0;
    for (int32_t j = nyg - 1; j >= 0; j--)
        for (int32_t i = 0; i < nxg; i++) {
            const int64_t c = (int64_t)j * nxg + i;
            const double mx = f->x0 + ((double)i + 0.5) * dx, my = f->y0 + ((double)j + 0.5) * dy;
            int v = cat[c] == 0;
            if (cat[c] == 1) v = or_field_value(f, f->phi, mx, my) <= band;
            valid[c] = (uint8_t)v;
            if (v) {
                rho[c] = f->rho ? or_field_value(f, f->rho, mx, my) : 1.0;
                S += rho[c];
            }
        }
    int64_t tot = 0;
    for (int32_t j = nyg - 1; j >= 0; j--)
        for (int32_t i = 0; i < nxg; i++) {
            const int64_t c = (int64_t)j * nxg + i;
            counts[c] = 0;
            if (!valid[c]) continue;
            const double v = (rho[c] / S) * n_init + acc[c];
            double r = floor(v + 0.5);
            if (r < 0.0) r = 0.0;
            counts[c] = (int32_t)r;
            tot += counts[c];
            const double R = v - r;
            const int ni[4] = {i + 1, i - 1, i, i + 1}, nj[4] = {j, j - 1, j - 1, j - 1};
            int m = 0;
            for (int q = 0; q < 4; q++)
                if (ni[q] >= 0 && ni[q] < nxg && nj[q] >= 0 && valid[(int64_t)nj[q] * nxg + ni[q]]) m++;
            if (m == 0) continue;
            const double w = R / (double)m;
            for (int q = 0; q < 4; q++)
                if (ni[q] >= 0 && ni[q] < nxg && nj[q] >= 0 && valid[(int64_t)nj[q] * nxg + ni[q]])
                    acc[(int64_t)nj[q] * nxg + ni[q]] += w;
        }
    free(valid); free(rho); free(acc);
    return tot;
}

/* Counter-based uniform numbers shared by both sides' point generation (reading L47): splitmix64
 * of seed + (2 k + comp + 1) * 0x9E3779B97F4A7C15, the top 53 bits scaled by 2^-53. */
static double or_u01(uint64_t seed, uint64_t k, int comp) {
    uint64_t z = seed + (2u * k + (uint64_t)comp + 1u) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z = z ^ (z >> 31);
    return (double)(z >> 11) * 1.1102230246251565e-16;
}

/* The points: counts[c] uniform points in cell c, cells in the loop order of
 * or_init_counts, point k (global index in that order) at (cx0 + u dx, cy0 + v dy) with
 * u = or_u01(seed, k, 0), v = or_u01(seed, k, 1).  A point outside the boundary tolerance
 * (phi~ > geps = fac_geps min(h, h_avg)) is projected onto the boundary by the damped 2x2 Newton
 * method of the treatment (P:402 -> P:575-605; deps = sqrt(eps) min(h, h_avg)); if that fails it
 * stays (reading L47).  Returns the number written. */
int64_t or_init_points(const or_fields *f, const or_params *p, double c, double h_avg, int32_t nxg, int32_t nyg,
                       const int32_t *counts, uint64_t seed, double *x, double *y) {
    const double dx = (f->x1 - f->x0) / (double)nxg, dy = (f->y1 - f->y0) / (double)nyg;
    int64_t k = 0;
    for (int32_t j = nyg - 1; j >= 0; j--)
        for (int32_t i = 0; i < nxg; i++) {
            const int64_t cc = (int64_t)j * nxg + i;
            const double cx0 = f->x0 + (double)i * dx, cy0 = f->y0 + (double)j * dy;
            for (int32_t q = 0; q < counts[cc]; q++, k++) {
                double px = cx0 + or_u01(seed, (uint64_t)k, 0) * dx;
                double py = cy0 + or_u01(seed, (uint64_t)k, 1) * dy;
                const double h = h_of(f, c, px, py);
                const double hm = h < h_avg ? h : h_avg;
                const double geps = p->fac_geps * hm;
                if (or_field_value(f, f->phi, px, py) > geps) {
                    double qx, qy;
                    if (newton_project(f, p, px, py, geps, 1.4901161193847656e-08 * hm, &qx, &qy)) { px = qx; py = qy; }
                }
                x[k] = px;
                y[k] = py;
            }
        }
    return k;
}

/* ---- NEXT-4: automatic sizing (App. A) ---------------------------- */
/* Boundary points from a contour (App. A): every segment's start point, and on a segment
 * longer than d_s the points a + (q/m)(b - a), q = 1..m-1, m = floor(len/d_s) + 1 (spacing below
 * d_s).  Then the trimming loop (reading L48): over the points in their order, find
 * the closest OTHER point whose midpoint m with p_i has |sdf(m)| <= geps_hat; if it is closer than
 * d_s, delete it and move p_i to m (and look again), else p_i is done; sweeps repeat until a sweep
 * changes nothing.  sdf is the contour's (or_contour_sdf_point).  Returns the count (<= cap). */
int64_t or_boundary_points(const double *segs, int64_t n_seg, double d_s, double geps_hat, double *x, double *y,
                           int64_t cap) {
    int64_t n = 0;
    for (int64_t k = 0; k < n_seg; k++) {
        const double *s = segs + 4 * k;
        const double ex = s[2] - s[0], ey = s[3] - s[1];
        const double len = sqrt(ex * ex + ey * ey);
        if (n < cap) { x[n] = s[0]; y[n] = s[1]; }
        n++;
        if (len > d_s) {
            const int64_t m = (int64_t)floor(len / d_s) + 1;
            for (int64_t q = 1; q < m; q++) {
                const double t = (double)q / (double)m;
                if (n < cap) { x[n] = s[0] + t * ex; y[n] = s[1] + t * ey; }
                n++;
            }
        }
    }
    if (n > cap) return -n;
    uint8_t *alive = (uint8_t *)malloc((size_t)(n > 0 ? n : 1));
    for (int64_t i = 0; i < n; i++) alive[i] = 1;
    for (int changed = 1; changed;) {
        changed = 0;
        for (int64_t i = 0; i < n; i++) {
            while (alive[i]) {
                int64_t best = -1;
                double bd = 0.0;
                for (int64_t j = 0; j < n; j++) {
                    if (j == i || !alive[j]) continue;
                    const double dx = x[j] - x[i], dy = y[j] - y[i];
                    const double d2 = dx * dx + dy * dy;
                    if (best >= 0 && !(d2 < bd)) continue;
                    const double mx = (x[i] + x[j]) * 0.5, my = (y[i] + y[j]) * 0.5;
                    if (!(fabs(or_contour_sdf_point(segs, n_seg, mx, my)) <= geps_hat)) continue;
                    best = j;
                    bd = d2;
                }
                if (best < 0 || !(bd < d_s * d_s)) break;
                x[i] = (x[i] + x[best]) * 0.5;
                y[i] = (y[i] + y[best]) * 0.5;
                alive[best] = 0;
                changed = 1;
            }
        }
    }
    int64_t m = 0;
    for (int64_t i = 0; i < n; i++)
        if (alive[i]) { x[m] = x[i]; y[m] = y[i]; m++; }
    free(alive);
    return m;
}

/* Medial-axis approximation (after Amenta et al.): for each boundary point s its
 * Voronoi vertices are the circumcentres of its Delaunay triangles (canonical Cramer relative to
 * the smallest index, as the keep rule); v1 = the farthest from s, v2 = the farthest among those
 * with (v - s).(v1 - s) < 0; distance ties by the smallest (u, v) of the triangle (reading L48).
 * Only triangles whose circumcentre lies inside the box [x0,x1]x[y0,y1] count (a bounded diagram).
 * Writes up to 2 points per boundary point into mx/my (v1 then v2, boundary points in order).
 * Trimming: a medial point is kept iff at least n_thres OTHER medial points lie within
 * r_nei (strictly closer).  Returns the kept count; med_x/med_y compacted. */
int64_t or_medial_points(int64_t n, const double *x, const double *y, double x0, double y0, double x1, double y1,
                         double r_nei, int32_t n_thres, double *mx, double *my) {
    int64_t cap = 2 * n + 16;
    int32_t *D = (int32_t *)malloc(sizeof(int32_t) * 3 * (size_t)cap);
    int64_t nd = or_delaunay(n, x, y, D, cap, NULL);
    if (nd < 0) { free(D); return -1; }
    double *cx = (double *)malloc(sizeof(double) * (size_t)(nd > 0 ? nd : 1));
    double *cy = (double *)malloc(sizeof(double) * (size_t)(nd > 0 ? nd : 1));
    int32_t *su = (int32_t *)malloc(sizeof(int32_t) * 3 * (size_t)(nd > 0 ? nd : 1));
    for (int64_t t = 0; t < nd; t++) {
        int32_t q[3] = {D[3 * t], D[3 * t + 1], D[3 * t + 2]};
        for (int a = 0; a < 2; a++)
            for (int b = 0; b < 2 - a; b++)
                if (q[b] > q[b + 1]) { int32_t s_ = q[b]; q[b] = q[b + 1]; q[b + 1] = s_; }
        line2 A, B;
        A.nx = x[q[1]] - x[q[0]]; A.ny = y[q[1]] - y[q[0]]; A.r = 0.5 * (A.nx * A.nx + A.ny * A.ny);
        B.nx = x[q[2]] - x[q[0]]; B.ny = y[q[2]] - y[q[0]]; B.r = 0.5 * (B.nx * B.nx + B.ny * B.ny);
        double ox, oy;
        cramer(A, B, &ox, &oy);
        cx[t] = x[q[0]] + ox;
        cy[t] = y[q[0]] + oy;
        su[3 * t] = q[0]; su[3 * t + 1] = q[1]; su[3 * t + 2] = q[2];
    }
    /* per point: the best triangle for v1, then for v2 */
    int64_t *b1 = (int64_t *)malloc(sizeof(int64_t) * (size_t)n), *b2 = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    double *d1 = (double *)malloc(sizeof(double) * (size_t)n), *d2 = (double *)malloc(sizeof(double) * (size_t)n);
    for (int64_t i = 0; i < n; i++) { b1[i] = b2[i] = -1; d1[i] = d2[i] = 0.0; }
#define OR_TKEY(t) (((uint64_t)(uint32_t)su[3 * (t)] << 32) | (uint32_t)su[3 * (t) + 1])
    for (int pass = 0; pass < 2; pass++)
        for (int64_t t = 0; t < nd; t++) {
            if (!(cx[t] > x0 && cx[t] < x1 && cy[t] > y0 && cy[t] < y1)) continue;
            for (int k = 0; k < 3; k++) {
                const int32_t s = su[3 * t + k];
                const double ex = cx[t] - x[s], ey = cy[t] - y[s];
                const double dd = ex * ex + ey * ey;
                int64_t *bb = pass ? b2 : b1;
                double *db = pass ? d2 : d1;
                if (pass) {
                    if (b1[s] < 0) continue;
                    const double fx = cx[b1[s]] - x[s], fy = cy[b1[s]] - y[s];
                    if (!(ex * fx + ey * fy < 0.0)) continue;
                }
                if (bb[s] < 0 || dd > db[s] || (dd == db[s] && OR_TKEY(t) < OR_TKEY(bb[s]))) { bb[s] = t; db[s] = dd; }
            }
        }
#undef OR_TKEY
    int64_t m = 0;
    for (int64_t i = 0; i < n; i++) {
        if (b1[i] >= 0) { mx[m] = cx[b1[i]]; my[m] = cy[b1[i]]; m++; }
        if (b2[i] >= 0) { mx[m] = cx[b2[i]]; my[m] = cy[b2[i]]; m++; }
    }
    uint8_t *keep = (uint8_t *)malloc((size_t)(m > 0 ? m : 1));
    for (int64_t i = 0; i < m; i++) {
        int64_t c = 0;
        for (int64_t j = 0; j < m; j++) {
            if (j == i) continue;
            const double dx = mx[j] - mx[i], dy = my[j] - my[i];
            if (dx * dx + dy * dy < r_nei * r_nei) c++;
        }
        keep[i] = c >= n_thres;
    }
    int64_t k = 0;
    for (int64_t i = 0; i < m; i++)
        if (keep[i]) { mx[k] = mx[i]; my[k] = my[i]; k++; }
    free(D); free(cx); free(cy); free(su); free(b1); free(b2); free(d1); free(d2); free(keep);
    return k;
}

/* Sizing field (Eq. sizing field): lfs(s) = distance from s to the nearest medial point
 * (P:373); mu(x) = min_s [K |x - s| + lfs(s)] at the nodes of the [ny][nx] grid over the box
 * (reading L48: the node grid of the bilinear fields instead of geometry-grid midpoints). */
void or_sizing_field(int64_t ns, const double *sx, const double *sy, int64_t nm, const double *mx, const double *my,
                     double K, int32_t nx, int32_t ny, double x0, double y0, double x1, double y1, double *mu,
                     double *lfs) {
    for (int64_t i = 0; i < ns; i++) {
        double b = -1.0;
        for (int64_t j = 0; j < nm; j++) {
            const double dx = mx[j] - sx[i], dy = my[j] - sy[i];
            const double d = sqrt(dx * dx + dy * dy);
            if (b < 0.0 || d < b) b = d;
        }
        lfs[i] = b;
    }
    for (int32_t j = 0; j < ny; j++)
        for (int32_t i = 0; i < nx; i++) {
            const double px = x0 + (double)i * ((x1 - x0) / (double)(nx - 1));
            const double py = y0 + (double)j * ((y1 - y0) / (double)(ny - 1));
            double b = -1.0;
            for (int64_t s = 0; s < ns; s++) {
                const double dx = px - sx[s], dy = py - sy[s];
                const double v = K * sqrt(dx * dx + dy * dy) + lfs[s];
                if (b < 0.0 || v < b) b = v;
            }
            mu[(int64_t)j * nx + i] = b;
        }
}

/* ---- NEXT-4: adaptive distance field on the boundary cells (after Frisken et al.) --- */
/* Top-down quadtree per boundary geometry cell: a node holds the exact SDF of the shape input (the
 * contour, or_contour_sdf_point) at its 4 corners; it is subdivided into 4 children while the
 * largest error of its bilinear interpolant at the 4 edge midpoints and the centre exceeds E_tol
 * and its depth (root 0) is below max_depth.  E_tol = fac_etol * geps_i * fac_pt, geps_i =
 * fac_geps * min(h(m_i), h_avg) at the cell midpoint m_i, fac_pt = sqrt(N_current / N_total).
 * Evaluation: descend to the leaf holding p (x >= the node's mid line goes right/up), bilinear
 * interpolation of its corners.  Reading L48. */
typedef struct { double x0, y0, x1, y1, f[4]; int32_t child; } or_adf_node;
typedef struct { or_adf_node *nodes; int64_t n, cap; int32_t *root; int32_t nxg, nyg; double x0, y0, dx, dy; } or_adf;

static double adf_lerp2(const double *f, double s, double t) {
    return lerp(lerp(f[0], f[1], s), lerp(f[2], f[3], s), t);
}
static int64_t adf_push(or_adf *A, double x0, double y0, double x1, double y1, const double *segs, int64_t ns) {
    if (A->n == A->cap) {
        A->cap = A->cap ? 2 * A->cap : 1024;
        A->nodes = (or_adf_node *)realloc(A->nodes, sizeof(or_adf_node) * (size_t)A->cap);
    }
    or_adf_node *d = &A->nodes[A->n];
    d->x0 = x0; d->y0 = y0; d->x1 = x1; d->y1 = y1; d->child = -1;
    d->f[0] = or_contour_sdf_point(segs, ns, x0, y0);
    d->f[1] = or_contour_sdf_point(segs, ns, x1, y0);
    d->f[2] = or_contour_sdf_point(segs, ns, x0, y1);
    d->f[3] = or_contour_sdf_point(segs, ns, x1, y1);
    return A->n++;
}
static void adf_refine(or_adf *A, int64_t k, int depth, double etol, int max_depth, const double *segs, int64_t ns) {
    or_adf_node nd = A->nodes[k];
    if (depth >= max_depth) return;
    const double xm = (nd.x0 + nd.x1) * 0.5, ym = (nd.y0 + nd.y1) * 0.5;
    const double px[5] = {xm, xm, nd.x0, nd.x1, xm}, py[5] = {nd.y0, nd.y1, ym, ym, ym};
    const double ps[5] = {0.5, 0.5, 0.0, 1.0, 0.5}, pt[5] = {0.0, 1.0, 0.5, 0.5, 0.5};
    double err = 0.0;
    for (int q = 0; q < 5; q++) {
        const double e = fabs(adf_lerp2(nd.f, ps[q], pt[q]) - or_contour_sdf_point(segs, ns, px[q], py[q]));
        if (e > err) err = e;
    }
    if (!(err > etol)) return;
    const int64_t c0 = adf_push(A, nd.x0, nd.y0, xm, ym, segs, ns);
    adf_push(A, xm, nd.y0, nd.x1, ym, segs, ns);
    adf_push(A, nd.x0, ym, xm, nd.y1, segs, ns);
    adf_push(A, xm, ym, nd.x1, nd.y1, segs, ns);
    A->nodes[k].child = (int32_t)c0;
    for (int q = 0; q < 4; q++) adf_refine(A, c0 + q, depth + 1, etol, max_depth, segs, ns);
}
/* builds the ADF of every boundary cell (cat == 1); returns the node count and the leaf count */
void *or_adf_build(const or_fields *f, const or_params *p, double c, double h_avg, int32_t nxg, int32_t nyg,
                   const int8_t *cat, const double *segs, int64_t n_seg, double fac_etol, double fac_pt,
                   int32_t max_depth, int64_t *n_nodes, int64_t *n_leaves) {
    or_adf *A = (or_adf *)calloc(1, sizeof(or_adf));
    A->nxg = nxg; A->nyg = nyg; A->x0 = f->x0; A->y0 = f->y0;
    A->dx = (f->x1 - f->x0) / (double)nxg; A->dy = (f->y1 - f->y0) / (double)nyg;
    A->root = (int32_t *)malloc(sizeof(int32_t) * (size_t)nxg * (size_t)nyg);
    for (int32_t j = 0; j < nyg; j++)
        for (int32_t i = 0; i < nxg; i++) {
            const int64_t cc = (int64_t)j * nxg + i;
            A->root[cc] = -1;
            if (cat[cc] != 1) continue;
            const double cx0 = f->x0 + (double)i * A->dx, cy0 = f->y0 + (double)j * A->dy;
            const double cx1 = f->x0 + (double)(i + 1) * A->dx, cy1 = f->y0 + (double)(j + 1) * A->dy;
            const double mx = f->x0 + ((double)i + 0.5) * A->dx, my = f->y0 + ((double)j + 0.5) * A->dy;
            const double h = h_of(f, c, mx, my);
            const double geps = p->fac_geps * (h < h_avg ? h : h_avg);
            const double etol = fac_etol * geps * fac_pt;
            const int64_t r = adf_push(A, cx0, cy0, cx1, cy1, segs, n_seg);
            A->root[cc] = (int32_t)r;
            adf_refine(A, r, 0, etol, max_depth, segs, n_seg);
        }
    int64_t leaves = 0;
    for (int64_t k = 0; k < A->n; k++) leaves += A->nodes[k].child < 0;
    *n_nodes = A->n;
    *n_leaves = leaves;
    return A;
}
/* ADF value at (x, y) if it lies in a boundary cell, else NaN */
double or_adf_eval(const void *h, double x, double y) {
    const or_adf *A = (const or_adf *)h;
    int i = (int)floor((x - A->x0) / A->dx), j = (int)floor((y - A->y0) / A->dy);
    if (i < 0 || j < 0 || i >= A->nxg || j >= A->nyg) return NAN;
    int64_t k = A->root[(int64_t)j * A->nxg + i];
    if (k < 0) return NAN;
    while (A->nodes[k].child >= 0) {
        const or_adf_node *d = &A->nodes[k];
        const double xm = (d->x0 + d->x1) * 0.5, ym = (d->y0 + d->y1) * 0.5;
        k = d->child + (x >= xm ? 1 : 0) + (y >= ym ? 2 : 0);
    }
    const or_adf_node *d = &A->nodes[k];
    return adf_lerp2(d->f, (x - d->x0) / (d->x1 - d->x0), (y - d->y0) / (d->y1 - d->y0));
}
void or_adf_free(void *h) {
    or_adf *A = (or_adf *)h;
    if (!A) return;
    free(A->nodes); free(A->root); free(A);
}
