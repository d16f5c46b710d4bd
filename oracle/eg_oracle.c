/*
 * oracle/eg_oracle.c -- CPU ORACLE for the extremum-graph hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_2303_02724_b200/) never imports, links or executes
 * it, and the two share no code: no headers, no tables, no helpers.
 *
 * A plain, slow, single-threaded transcription of arXiv 2303.02724
 * (/root/reference/PAPER.md, cited as P:<line>), in the paper's order:
 *
 *   O1 order       P:184  simulated perturbation.  Reading L1:
 *                         u < v  iff  f[u] < f[v] or (f[u] == f[v] and u < v),
 *                         IEEE compares (so -0 == +0), NaN rejected (L2).
 *   O2 link        P:104-138  Freudenthal tessellation; the link of v is every
 *                         in-domain q with GridAdjacency(v, q) (Alg. 1, with
 *                         p != q, reading L6), truncated at the boundary (L3).
 *                         CSR: the neighbour list N(v) (reading L14).
 *   O3 upper link  P:144  U = { u in Lk(v) : v < u }.
 *   O4 gradient    P:186  "the vertex with the highest scalar value in the
 *                         upper link"; computed for every non-maximum (L4).
 *   O5 components  P:184-186  union-find over the link edges whose two ends
 *                         are both in U; an edge between link vertices a, b
 *                         exists iff GridAdjacency(a, b) (grid) or b in N(a)
 *                         (CSR).  beta0+ = number of components.
 *                         UpperLinkRep = highest vertex of a component.
 *   O6 class       P:147-159 (Table 1)  maximum iff beta0+ = 0,
 *                         (n-1)-saddle iff beta0+ >= 2 (L5).
 *   O7 labels      P:192-208 (Alg. 2)  follow gradient(u) until a maximum;
 *                         the walk is memoised so that every vertex gets the
 *                         maximum its path reaches.
 *   O8 arcs        P:219, P:260  for every saddle (ascending) and every
 *                         upper-link component: m = label[rep]; the multiset
 *                         of m is reduced to unique (s, m) with multiplicity
 *                         (L7).  Raw (s, rep, m) triples are kept as well.
 *
 *   O10 minimum graph  P:62, "computes both maximum and minimum graph".
 *                         Reading L11: the minimum graph (minima, 1-saddles,
 *                         descending arcs) is the maximum graph under the
 *                         REVERSED total order -- O1 with u and v swapped
 *                         (ego_set_order(1)); every other step is unchanged.
 *
 * Parity status: every function below is pinned by tests/test_oracle_pins.py
 * (closed forms, Euler invariant, literal brute force, golden examples); the
 * CSR path on kNN graphs is pinned only by brute force on small graphs and
 * the clique Euler identity ("parity partially unpinned" in DESIGN.md).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define EGO_OK 0
#define EGO_ERR_INVALID 1
#define EGO_ERR_NAN 2
#define EGO_ERR_OOM 3

#define EGO_MAX_DIM 8

typedef struct {
    int64_t n;            /* number of vertices */
    int64_t *ptr;         /* [n] gradient(v), v itself for a maximum   (O4) */
    int64_t *label;       /* [n] maximum reached by the ascending path (O7) */
    int32_t *beta;        /* [n] beta0+ of every vertex               (O5) */
    int64_t n_max;
    int64_t *maxima;      /* ascending */
    int64_t n_saddle;
    int64_t *saddles;     /* ascending */
    int32_t *saddle_beta;
    int64_t n_arc;
    int64_t *arc_s, *arc_m;
    int32_t *arc_mult;
    int64_t n_raw;
    int64_t *raw_s, *raw_rep, *raw_m;
} ego_result;

/* ---------------------------------------------------------------- O1 order */

static int g_reverse = 0;   /* O10: 1 = the reversed order (minimum graph) */

void ego_set_order(int reverse) { g_reverse = reverse != 0; }

static int less(const float *f, int64_t u, int64_t v) {
    /* P:184 simulated perturbation, lower index = lower (L1). */
    if (g_reverse) { const int64_t t = u; u = v; v = t; }
    return f[u] < f[v] || (f[u] == f[v] && u < v);
}

static int any_nan(const float *f, int64_t n) {
    for (int64_t i = 0; i < n; ++i)
        if (isnan(f[i])) return 1;
    return 0;
}

/* ------------------------------------------------------------- grid domain */

typedef struct {
    int ndim;
    int64_t dims[EGO_MAX_DIM];    /* axis 0 fastest (L9) */
    int64_t stride[EGO_MAX_DIM];
    int64_t n;
} grid_t;

static int grid_init(grid_t *g, int ndim, const int64_t *dims) {
    if (ndim < 1 || ndim > EGO_MAX_DIM) return EGO_ERR_INVALID;
    g->ndim = ndim;
    int64_t n = 1;
    for (int i = 0; i < ndim; ++i) {
        if (dims[i] < 1) return EGO_ERR_INVALID;
        if (n > INT64_MAX / dims[i]) return EGO_ERR_INVALID;
        g->dims[i] = dims[i];
        g->stride[i] = n;
        n *= dims[i];
    }
    g->n = n;
    return EGO_OK;
}

static void delinearize(const grid_t *g, int64_t v, int64_t *c) {
    for (int i = 0; i < g->ndim; ++i) c[i] = (v / g->stride[i]) % g->dims[i];
}

/* Alg. 1 GridAdjacency, literally: collect the set U of
 * component-wise differences p_i - q_i; adjacent iff U is a subset of {0,1}
 * or of {0,-1}.  As printed the test also passes for p == q (U = {0}); the
 * edge set excludes it (reading L6). */
int ego_grid_adjacent(int ndim, const int64_t *p, const int64_t *q) {
    int has_pos1 = 0, has_neg1 = 0, has_other = 0, has_nonzero = 0;
    for (int i = 0; i < ndim; ++i) {
        int64_t d = p[i] - q[i];
        if (d == 1) has_pos1 = 1;
        else if (d == -1) has_neg1 = 1;
        else if (d != 0) has_other = 1;
        if (d != 0) has_nonzero = 1;
    }
    if (!has_nonzero) return 0;                /* p == q: not an edge (L6) */
    if (has_other) return 0;
    int subset01 = !has_neg1;                  /* U subset of {0, 1}  */
    int subset0m1 = !has_pos1;                 /* U subset of {0, -1} */
    return subset01 || subset0m1;
}

/* O2: the link of v = every in-domain vertex q with GridAdjacency(v, q).
 * Candidates are q = v + d, d in {-1,0,1}^n (Alg. 1 can only accept those);
 * the domain boundary truncates the link (L3).  Output in ascending id. */
static int64_t grid_link(const grid_t *g, int64_t v, int64_t *out) {
    int64_t cv[EGO_MAX_DIM], cq[EGO_MAX_DIM];
    delinearize(g, v, cv);
    int64_t total = 1;
    for (int i = 0; i < g->ndim; ++i) total *= 3;
    int64_t cnt = 0;
    for (int64_t t = 0; t < total; ++t) {
        int64_t r = t, q = 0, inside = 1;
        for (int i = 0; i < g->ndim; ++i) {
            int64_t d = (r % 3) - 1;
            r /= 3;
            cq[i] = cv[i] + d;
            if (cq[i] < 0 || cq[i] >= g->dims[i]) inside = 0;
        }
        if (!inside) continue;
        if (!ego_grid_adjacent(g->ndim, cv, cq)) continue;
        for (int i = 0; i < g->ndim; ++i) q += cq[i] * g->stride[i];
        out[cnt++] = q;
    }
    /* ascending ids (insertion sort: at most 2(2^n - 1) entries) */
    for (int64_t i = 1; i < cnt; ++i) {
        int64_t x = out[i], j = i - 1;
        while (j >= 0 && out[j] > x) { out[j + 1] = out[j]; --j; }
        out[j + 1] = x;
    }
    return cnt;
}

int64_t ego_grid_link(int ndim, const int64_t *dims, int64_t v, int64_t *out) {
    grid_t g;
    if (grid_init(&g, ndim, dims) != EGO_OK) return -1;
    if (v < 0 || v >= g.n) return -1;
    return grid_link(&g, v, out);
}

static int grid_edge(const grid_t *g, int64_t a, int64_t b) {
    int64_t ca[EGO_MAX_DIM], cb[EGO_MAX_DIM];
    delinearize(g, a, ca);
    delinearize(g, b, cb);
    return ego_grid_adjacent(g->ndim, ca, cb);
}

/* ----------------------------------------------------------- CSR domain */

typedef struct {
    int64_t n;
    const int64_t *row_ptr;
    const int32_t *col_idx;
} csr_t;

static int64_t csr_link(const csr_t *c, int64_t v, int64_t *out) {
    int64_t cnt = 0;
    for (int64_t k = c->row_ptr[v]; k < c->row_ptr[v + 1]; ++k) out[cnt++] = c->col_idx[k];
    return cnt;
}

static int csr_edge(const csr_t *c, int64_t a, int64_t b) {
    /* b in N(a), by binary search in the sorted neighbour list */
    int64_t lo = c->row_ptr[a], hi = c->row_ptr[a + 1];
    while (lo < hi) {
        int64_t mid = lo + (hi - lo) / 2;
        if (c->col_idx[mid] < b) lo = mid + 1;
        else hi = mid;
    }
    return lo < c->row_ptr[a + 1] && c->col_idx[lo] == b;
}

/* ------------------------------------------------------- union-find (O5) */

static int64_t uf_find(int64_t *parent, int64_t x) {
    while (parent[x] != x) {            /* path halving */
        parent[x] = parent[parent[x]];
        x = parent[x];
    }
    return x;
}

static void uf_union(int64_t *parent, int64_t *size, int64_t a, int64_t b) {
    a = uf_find(parent, a);
    b = uf_find(parent, b);
    if (a == b) return;
    if (size[a] < size[b]) { int64_t t = a; a = b; b = t; }
    parent[b] = a;
    size[a] += size[b];
}

/* ------------------------------------------- per-vertex classification */

typedef struct {
    int is_grid;
    const grid_t *g;
    const csr_t *c;
    const float *f;
    int64_t cap;        /* max link size */
    int64_t *link, *up, *parent, *size, *rep;
} work_t;

static int64_t wk_link(work_t *w, int64_t v) {
    return w->is_grid ? grid_link(w->g, v, w->link) : csr_link(w->c, v, w->link);
}
static int wk_edge(work_t *w, int64_t a, int64_t b) {
    return w->is_grid ? grid_edge(w->g, a, b) : csr_edge(w->c, a, b);
}

/* O3..O5 for one vertex.  Returns beta0+; *ptr_out = gradient (O4);
 * w->rep[0..beta) = UpperLinkRep, ascending. */
static int64_t classify_vertex(work_t *w, int64_t v, int64_t *ptr_out) {
    const float *f = w->f;
    int64_t nl = wk_link(w, v);
    int64_t nu = 0;
    for (int64_t i = 0; i < nl; ++i)                    /* O3 upper link */
        if (less(f, v, w->link[i])) w->up[nu++] = w->link[i];

    int64_t best = v;                                   /* O4 gradient */
    for (int64_t i = 0; i < nu; ++i)
        if (less(f, best, w->up[i])) best = w->up[i];
    *ptr_out = best;

    for (int64_t i = 0; i < nu; ++i) { w->parent[i] = i; w->size[i] = 1; }
    for (int64_t a = 0; a < nu; ++a)                    /* O5 union-find */
        for (int64_t b = a + 1; b < nu; ++b)
            if (wk_edge(w, w->up[a], w->up[b])) uf_union(w->parent, w->size, a, b);

    int64_t beta = 0;
    for (int64_t i = 0; i < nu; ++i) {                  /* roots -> components */
        if (uf_find(w->parent, i) != i) continue;
        int64_t r = -1;                                 /* UpperLinkRep: highest member */
        for (int64_t j = 0; j < nu; ++j)
            if (uf_find(w->parent, j) == i && (r < 0 || less(f, r, w->up[j]))) r = w->up[j];
        w->rep[beta++] = r;
    }
    for (int64_t i = 1; i < beta; ++i) {                /* ascending reps */
        int64_t x = w->rep[i], j = i - 1;
        while (j >= 0 && w->rep[j] > x) { w->rep[j + 1] = w->rep[j]; --j; }
        w->rep[j + 1] = x;
    }
    return beta;
}

static int work_alloc(work_t *w, int64_t cap) {
    w->cap = cap < 1 ? 1 : cap;
    w->link = malloc(sizeof(int64_t) * w->cap);
    w->up = malloc(sizeof(int64_t) * w->cap);
    w->parent = malloc(sizeof(int64_t) * w->cap);
    w->size = malloc(sizeof(int64_t) * w->cap);
    w->rep = malloc(sizeof(int64_t) * w->cap);
    return (w->link && w->up && w->parent && w->size && w->rep) ? EGO_OK : EGO_ERR_OOM;
}

static void work_free(work_t *w) {
    free(w->link); free(w->up); free(w->parent); free(w->size); free(w->rep);
}

static int64_t grid_link_cap(const grid_t *g) {
    int64_t c = 1;
    for (int i = 0; i < g->ndim; ++i) c *= 3;
    return c;
}

static int64_t csr_link_cap(const csr_t *c) {
    int64_t m = 0;
    for (int64_t v = 0; v < c->n; ++v) {
        int64_t d = c->row_ptr[v + 1] - c->row_ptr[v];
        if (d > m) m = d;
    }
    return m;
}

/* ------------------------------------------------- whole-domain driver */

void ego_free(ego_result *r) {
    if (!r) return;
    free(r->ptr); free(r->label); free(r->beta);
    free(r->maxima); free(r->saddles); free(r->saddle_beta);
    free(r->arc_s); free(r->arc_m); free(r->arc_mult);
    free(r->raw_s); free(r->raw_rep); free(r->raw_m);
    memset(r, 0, sizeof(*r));
}

static int cmp_i64(const void *a, const void *b) {
    int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
    return (x > y) - (x < y);
}

/* O7 (Alg. 2 "follow gradient(u) until u is a maximum"): for
 * v = 0..n-1 whose label is unset, walk v, ptr[v], ptr[ptr[v]], ... pushing
 * onto `stack` until a maximum (ptr[x] == x) or a labelled vertex, then give
 * the whole stack that label (memoised, O(n) in total).  `stack` holds n. */
static void labels_from_ptr(int64_t n, const int64_t *ptr, int64_t *label, int64_t *stack) {
    for (int64_t v = 0; v < n; ++v) label[v] = -1;
    for (int64_t v = 0; v < n; ++v) {
        if (label[v] >= 0) continue;
        int64_t sp = 0, x = v;
        while (label[x] < 0 && ptr[x] != x) { stack[sp++] = x; x = ptr[x]; }
        int64_t m = label[x] >= 0 ? label[x] : x;
        label[x] = m;
        while (sp > 0) label[stack[--sp]] = m;
    }
}

static int run_all(work_t *w, int64_t n, ego_result *out) {
    memset(out, 0, sizeof(*out));
    out->n = n;
    out->ptr = malloc(sizeof(int64_t) * (n ? n : 1));
    out->label = malloc(sizeof(int64_t) * (n ? n : 1));
    out->beta = malloc(sizeof(int32_t) * (n ? n : 1));
    int64_t *stack = malloc(sizeof(int64_t) * (n ? n : 1));
    if (!out->ptr || !out->label || !out->beta || !stack) { free(stack); ego_free(out); return EGO_ERR_OOM; }

    /* O3..O6 for every vertex in index order */
    int64_t n_max = 0, n_sad = 0, n_raw = 0;
    for (int64_t v = 0; v < n; ++v) {
        int64_t p;
        int64_t b = classify_vertex(w, v, &p);
        out->ptr[v] = p;
        out->beta[v] = (int32_t)b;
        if (b == 0) ++n_max;
        if (b >= 2) { ++n_sad; n_raw += b; }
    }

    /* O7: labels by following the gradient (Alg. 2), memoised */
    labels_from_ptr(n, out->ptr, out->label, stack);
    free(stack);

    /* O6 / O9 node lists, ascending */
    out->n_max = n_max;
    out->n_saddle = n_sad;
    out->maxima = malloc(sizeof(int64_t) * (n_max ? n_max : 1));
    out->saddles = malloc(sizeof(int64_t) * (n_sad ? n_sad : 1));
    out->saddle_beta = malloc(sizeof(int32_t) * (n_sad ? n_sad : 1));
    out->raw_s = malloc(sizeof(int64_t) * (n_raw ? n_raw : 1));
    out->raw_rep = malloc(sizeof(int64_t) * (n_raw ? n_raw : 1));
    out->raw_m = malloc(sizeof(int64_t) * (n_raw ? n_raw : 1));
    out->arc_s = malloc(sizeof(int64_t) * (n_raw ? n_raw : 1));
    out->arc_m = malloc(sizeof(int64_t) * (n_raw ? n_raw : 1));
    out->arc_mult = malloc(sizeof(int32_t) * (n_raw ? n_raw : 1));
    int64_t *ms = malloc(sizeof(int64_t) * w->cap);
    if (!out->maxima || !out->saddles || !out->saddle_beta || !out->raw_s || !out->raw_rep ||
        !out->raw_m || !out->arc_s || !out->arc_m || !out->arc_mult || !ms) {
        free(ms); ego_free(out); return EGO_ERR_OOM;
    }
    int64_t im = 0, is = 0;
    for (int64_t v = 0; v < n; ++v) {
        if (out->beta[v] == 0) out->maxima[im++] = v;
        if (out->beta[v] >= 2) { out->saddles[is] = v; out->saddle_beta[is] = out->beta[v]; ++is; }
    }

    /* O8 arcs: per saddle, m = label[UpperLinkRep(C)] for each component C */
    int64_t ir = 0, ia = 0;
    for (int64_t k = 0; k < n_sad; ++k) {
        int64_t s = out->saddles[k], p;
        int64_t b = classify_vertex(w, s, &p);
        for (int64_t c = 0; c < b; ++c) {
            int64_t rep = w->rep[c];
            out->raw_s[ir] = s; out->raw_rep[ir] = rep; out->raw_m[ir] = out->label[rep]; ++ir;
            ms[c] = out->label[rep];
        }
        qsort(ms, (size_t)b, sizeof(int64_t), cmp_i64);
        for (int64_t c = 0; c < b;) {
            int64_t e = c;
            while (e < b && ms[e] == ms[c]) ++e;
            out->arc_s[ia] = s; out->arc_m[ia] = ms[c]; out->arc_mult[ia] = (int32_t)(e - c); ++ia;
            c = e;
        }
    }
    free(ms);
    out->n_raw = ir;
    out->n_arc = ia;
    return EGO_OK;
}

int ego_grid(int ndim, const int64_t *dims, const float *f, ego_result *out) {
    grid_t g;
    memset(out, 0, sizeof(*out));
    if (grid_init(&g, ndim, dims) != EGO_OK) return EGO_ERR_INVALID;
    if (any_nan(f, g.n)) return EGO_ERR_NAN;
    work_t w = {1, &g, NULL, f, 0, 0, 0, 0, 0, 0};
    if (work_alloc(&w, grid_link_cap(&g)) != EGO_OK) { work_free(&w); return EGO_ERR_OOM; }
    int rc = run_all(&w, g.n, out);
    work_free(&w);
    return rc;
}

int ego_csr(int64_t nv, const int64_t *row_ptr, const int32_t *col_idx, const float *f, ego_result *out) {
    memset(out, 0, sizeof(*out));
    if (nv < 0) return EGO_ERR_INVALID;
    if (any_nan(f, nv)) return EGO_ERR_NAN;
    csr_t c = {nv, row_ptr, col_idx};
    work_t w = {0, NULL, &c, f, 0, 0, 0, 0, 0, 0};
    if (work_alloc(&w, csr_link_cap(&c)) != EGO_OK) { work_free(&w); return EGO_ERR_OOM; }
    int rc = run_all(&w, nv, out);
    work_free(&w);
    return rc;
}

/* ---------------------------------------------- range entry points
 * The same steps as run_all, split for domains too big for one thread in a
 * test (C3 has 2^30 vertices): O3..O6 of the vertices [v0, v1) -- every
 * vertex is classified on its own, so disjoint ranges may be classified by
 * separate processes (oracle/__init__.py: grid_parallel / csr_parallel) --
 * and O7 over the assembled gradient array.  Each call is single-threaded and
 * runs exactly classify_vertex / labels_from_ptr; nothing is re-derived.
 * ptr / beta are indexed v - v0.  For every saddle (beta0+ >= 2), ascending,
 * its UpperLinkReps (ascending) are appended to (rep_s, rep_r) while fewer
 * than `cap` are stored; *n_rep counts all of them (> cap: call again with
 * room). */
static int range_common(work_t *w, int64_t v0, int64_t v1, int64_t *ptr, int32_t *beta,
                        int64_t *rep_s, int64_t *rep_r, int64_t cap, int64_t *n_rep) {
    int64_t k = 0;
    for (int64_t v = v0; v < v1; ++v) {
        int64_t p;
        int64_t b = classify_vertex(w, v, &p);
        ptr[v - v0] = p;
        beta[v - v0] = (int32_t)b;
        if (b >= 2)
            for (int64_t c = 0; c < b; ++c, ++k)
                if (k < cap) { rep_s[k] = v; rep_r[k] = w->rep[c]; }
    }
    *n_rep = k;
    return EGO_OK;
}

int ego_grid_range(int ndim, const int64_t *dims, const float *f, int64_t v0, int64_t v1, int64_t *ptr,
                   int32_t *beta, int64_t *rep_s, int64_t *rep_r, int64_t cap, int64_t *n_rep) {
    grid_t g;
    if (grid_init(&g, ndim, dims) != EGO_OK || v0 < 0 || v1 < v0 || v1 > g.n) return EGO_ERR_INVALID;
    for (int64_t v = v0; v < v1; ++v)
        if (isnan(f[v])) return EGO_ERR_NAN;
    work_t w = {1, &g, NULL, f, 0, 0, 0, 0, 0, 0};
    if (work_alloc(&w, grid_link_cap(&g)) != EGO_OK) { work_free(&w); return EGO_ERR_OOM; }
    int rc = range_common(&w, v0, v1, ptr, beta, rep_s, rep_r, cap, n_rep);
    work_free(&w);
    return rc;
}

int ego_csr_range(int64_t nv, const int64_t *row_ptr, const int32_t *col_idx, const float *f, int64_t v0,
                  int64_t v1, int64_t *ptr, int32_t *beta, int64_t *rep_s, int64_t *rep_r, int64_t cap,
                  int64_t *n_rep) {
    if (nv < 0 || v0 < 0 || v1 < v0 || v1 > nv) return EGO_ERR_INVALID;
    for (int64_t v = v0; v < v1; ++v)
        if (isnan(f[v])) return EGO_ERR_NAN;
    csr_t c = {nv, row_ptr, col_idx};
    work_t w = {0, NULL, &c, f, 0, 0, 0, 0, 0, 0};
    if (work_alloc(&w, csr_link_cap(&c)) != EGO_OK) { work_free(&w); return EGO_ERR_OOM; }
    int rc = range_common(&w, v0, v1, ptr, beta, rep_s, rep_r, cap, n_rep);
    work_free(&w);
    return rc;
}

/* O7 over a whole gradient array (the ptr of every vertex, e.g. assembled
 * from ego_*_range calls). */
int ego_labels(int64_t n, const int64_t *ptr, int64_t *label) {
    if (n < 0) return EGO_ERR_INVALID;
    for (int64_t v = 0; v < n; ++v)
        if (ptr[v] < 0 || ptr[v] >= n) return EGO_ERR_INVALID;
    int64_t *stack = malloc(sizeof(int64_t) * (n ? n : 1));
    if (!stack) return EGO_ERR_OOM;
    labels_from_ptr(n, ptr, label, stack);
    free(stack);
    return EGO_OK;
}

/* ------------------------------------------ single-vertex entry points
 * For sampled parity at sizes where the whole-domain oracle is too slow:
 * classify one vertex (O3..O5), or walk its ascending path (Alg. 2) to the
 * maximum, computing the gradient of each visited vertex on the fly. */

static int vertex_common(work_t *w, int64_t v, int64_t *ptr, int32_t *beta, int64_t *reps, int32_t cap) {
    int64_t p;
    int64_t b = classify_vertex(w, v, &p);
    *ptr = p;
    *beta = (int32_t)b;
    for (int64_t i = 0; i < b && i < cap; ++i) reps[i] = w->rep[i];
    return EGO_OK;
}

int ego_grid_vertex(int ndim, const int64_t *dims, const float *f, int64_t v,
                    int64_t *ptr, int32_t *beta, int64_t *reps, int32_t cap) {
    grid_t g;
    if (grid_init(&g, ndim, dims) != EGO_OK || v < 0 || v >= g.n) return EGO_ERR_INVALID;
    work_t w = {1, &g, NULL, f, 0, 0, 0, 0, 0, 0};
    if (work_alloc(&w, grid_link_cap(&g)) != EGO_OK) { work_free(&w); return EGO_ERR_OOM; }
    int rc = vertex_common(&w, v, ptr, beta, reps, cap);
    work_free(&w);
    return rc;
}

int ego_csr_vertex(int64_t nv, const int64_t *row_ptr, const int32_t *col_idx, const float *f, int64_t v,
                   int64_t *ptr, int32_t *beta, int64_t *reps, int32_t cap) {
    if (v < 0 || v >= nv) return EGO_ERR_INVALID;
    csr_t c = {nv, row_ptr, col_idx};
    work_t w = {0, NULL, &c, f, 0, 0, 0, 0, 0, 0};
    int64_t deg = row_ptr[v + 1] - row_ptr[v];
    if (work_alloc(&w, deg) != EGO_OK) { work_free(&w); return EGO_ERR_OOM; }
    int rc = vertex_common(&w, v, ptr, beta, reps, cap);
    work_free(&w);
    return rc;
}

/* Alg. 2 inner loop from v: u <- gradient(u) until u in M. */
int64_t ego_grid_walk(int ndim, const int64_t *dims, const float *f, int64_t v, int64_t *steps) {
    grid_t g;
    if (grid_init(&g, ndim, dims) != EGO_OK || v < 0 || v >= g.n) return -1;
    int64_t nl_cap = grid_link_cap(&g);
    int64_t *link = malloc(sizeof(int64_t) * nl_cap);
    if (!link) return -1;
    int64_t u = v, k = 0;
    for (;;) {
        int64_t nl = grid_link(&g, u, link), best = u;
        for (int64_t i = 0; i < nl; ++i)
            if (less(f, best, link[i])) best = link[i];
        if (best == u) break;           /* u is a maximum */
        u = best;
        ++k;
    }
    free(link);
    if (steps) *steps = k;
    return u;
}

int64_t ego_csr_walk(int64_t nv, const int64_t *row_ptr, const int32_t *col_idx, const float *f, int64_t v,
                     int64_t *steps) {
    if (v < 0 || v >= nv) return -1;
    int64_t u = v, k = 0;
    for (;;) {
        int64_t best = u;
        for (int64_t e = row_ptr[u]; e < row_ptr[u + 1]; ++e)
            if (less(f, best, col_idx[e])) best = col_idx[e];
        if (best == u) break;
        u = best;
        ++k;
    }
    if (steps) *steps = k;
    return u;
}

/* ------------------------------------------------- Euler diagnostics
 * chi(Lk+(v)) of the induced upper link.  The Freudenthal triangulation is a
 * flag complex, so the induced subcomplex on U is the clique complex of the
 * induced graph (pin "Euler").  chi = sum_k (-1)^(k+1) #k-cliques. */

static int64_t clique_chi(work_t *w, const int64_t *cand, int64_t nc, int depth) {
    /* cliques extending the current one by a vertex from cand (all of which
     * are adjacent to every current member and ordered ascending) */
    int64_t chi = 0;
    int64_t *next = malloc(sizeof(int64_t) * (nc ? nc : 1));
    for (int64_t i = 0; i < nc; ++i) {
        chi += (depth % 2 == 1) ? 1 : -1;   /* a clique of size `depth` */
        int64_t m = 0;
        for (int64_t j = i + 1; j < nc; ++j)
            if (wk_edge(w, cand[i], cand[j])) next[m++] = cand[j];
        if (m) {
            int64_t *sub = malloc(sizeof(int64_t) * m);
            memcpy(sub, next, sizeof(int64_t) * m);
            chi += clique_chi(w, sub, m, depth + 1);
            free(sub);
        }
    }
    free(next);
    return chi;
}

static int64_t chi_upper(work_t *w, int64_t v) {
    int64_t nl = wk_link(w, v), nu = 0;
    for (int64_t i = 0; i < nl; ++i)
        if (less(w->f, v, w->link[i])) w->up[nu++] = w->link[i];
    int64_t *u = malloc(sizeof(int64_t) * (nu ? nu : 1));
    memcpy(u, w->up, sizeof(int64_t) * nu);
    int64_t chi = clique_chi(w, u, nu, 1);
    free(u);
    return chi;
}

/* sum over all vertices of (1 - chi(Lk+(v))) -- equals chi(domain) (Banchoff). */
int ego_grid_euler(int ndim, const int64_t *dims, const float *f, int64_t *sum_out) {
    grid_t g;
    if (grid_init(&g, ndim, dims) != EGO_OK) return EGO_ERR_INVALID;
    work_t w = {1, &g, NULL, f, 0, 0, 0, 0, 0, 0};
    if (work_alloc(&w, grid_link_cap(&g)) != EGO_OK) { work_free(&w); return EGO_ERR_OOM; }
    int64_t s = 0;
    for (int64_t v = 0; v < g.n; ++v) s += 1 - chi_upper(&w, v);
    work_free(&w);
    *sum_out = s;
    return EGO_OK;
}

int ego_csr_euler(int64_t nv, const int64_t *row_ptr, const int32_t *col_idx, const float *f, int64_t *sum_out) {
    csr_t c = {nv, row_ptr, col_idx};
    work_t w = {0, NULL, &c, f, 0, 0, 0, 0, 0, 0};
    if (work_alloc(&w, csr_link_cap(&c)) != EGO_OK) { work_free(&w); return EGO_ERR_OOM; }
    int64_t s = 0;
    for (int64_t v = 0; v < nv; ++v) s += 1 - chi_upper(&w, v);
    work_free(&w);
    *sum_out = s;
    return EGO_OK;
}

/* chi of the whole clique complex of the graph restricted to the full link of
 * v (used by the flag-complex pin: an interior Freudenthal link is an
 * (n-1)-sphere).  Also returns the number of link edges and maximal cliques. */
int ego_grid_link_stats(int ndim, const int64_t *dims, int64_t v, int64_t *n_link, int64_t *n_edges,
                        int64_t *chi) {
    grid_t g;
    if (grid_init(&g, ndim, dims) != EGO_OK || v < 0 || v >= g.n) return EGO_ERR_INVALID;
    work_t w = {1, &g, NULL, NULL, 0, 0, 0, 0, 0, 0};
    if (work_alloc(&w, grid_link_cap(&g)) != EGO_OK) { work_free(&w); return EGO_ERR_OOM; }
    int64_t nl = grid_link(&g, v, w.link), ne = 0;
    for (int64_t a = 0; a < nl; ++a)
        for (int64_t b = a + 1; b < nl; ++b) ne += grid_edge(&g, w.link[a], w.link[b]);
    int64_t *cand = malloc(sizeof(int64_t) * (nl ? nl : 1));
    memcpy(cand, w.link, sizeof(int64_t) * nl);
    *chi = clique_chi(&w, cand, nl, 1);
    free(cand);
    *n_link = nl;
    *n_edges = ne;
    work_free(&w);
    return EGO_OK;
}
