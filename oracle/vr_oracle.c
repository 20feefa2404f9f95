/*
 * vr_oracle.c -- CPU ORACLE for the Vietoris-Rips filtration build.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_1809_04424_b200/, libvrb.so) never links, imports
 * or executes it, and shares no code, header, table or helper with it.
 *
 * Plain, slow, single-threaded, obviously-correct C, written from the paper
 * (/root/reference/PAPER.md, cited as P:<line>) and the readings A1..A14 of
 * SURVEY.md section 8(c), restated in DESIGN.md "Readings".  Built with
 *     gcc -O2 -ffp-contract=off -fno-fast-math   (x86-64 SSE2, FLT_EVAL_METHOD 0)
 * so every double operation is one IEEE-754 binary64 round-to-nearest op.
 *
 * Steps:
 *   1 distances        P:107-110 (sec 2.1), reading A5  -> or_length
 *   2 cap              P:109-110, reading A1 -> or_new
 *   3 ranks            P:929-941 (sec 4.5), readings A2,A3,A4,A14 -> or_new, or_sortperm
 *   4 vertices         P:267, P:286 (filt 0, index order)
 *   5 cliques          P:111-113 (sec 2.1), reading A6 -> or_build_simplices
 *   6 order            P:251, reading A4 -> or_build_simplices
 *   7 boundary CSC     P:205, reading A7 -> or_build_simplices
 *   8 barcodes         Algorithm 1, Algorithm 2 P:229-248,
 *                      Pers/Barcode P:251-260, Fig.4 caption P:286,
 *                      clearing P:302, readings A8,A9,A10,A13 -> or_barcodes
 * SURVEY 8(f) rows built beyond the path:
 *   F3 inputs          distance matrix P:351-353 -> or_new_dm; latlon2euc
 *                      P:383-408 -> or_latlon2euc
 *   F4 blockprodsum    S = D + C E over GF(2), sec. 4.6 P:986-1022 -> or_blockprodsum
 *   (F1, dimension-0 bars, is checked against or_barcodes.)
 * plus per-filtration-level helpers used for sampled parity at full size
 * (or_filt_hist, or_simplices_at_filt): the same definitions, evaluated for
 * one filtration level at a time.
 *
 * Parity pins: tests/test_oracle_pins.py.
 */
#pragma STDC FP_CONTRACT OFF

#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define NONE32 0xFFFFFFFFu

/* ------------------------------------------------------------------------ */
/* growable arrays                                                          */
/* ------------------------------------------------------------------------ */
typedef struct { uint32_t* a; int64_t n, cap; } vec32;

static void v32_push(vec32* v, uint32_t x) {
    if (v->n == v->cap) {
        v->cap = v->cap ? 2 * v->cap : 16;
        v->a = (uint32_t*)realloc(v->a, (size_t)v->cap * sizeof(uint32_t));
    }
    v->a[v->n++] = x;
}

/* ------------------------------------------------------------------------ */
/* Step 1: Euclidean length with a fixed fold (reading A5).      */
/*   acc = +0.0; for c in 0..d-1: t = x_ic - x_jc; acc = acc + t*t;        */
/*   len = sqrt(acc)   (correctly rounded, sqrtsd)                          */
/* ------------------------------------------------------------------------ */
double or_length(const double* X, int32_t d, int64_t i, int64_t j) {
    double acc = 0.0;
    for (int32_t c = 0; c < d; ++c) {
        double t = X[i * d + c] - X[j * d + c];
        acc = acc + t * t;
    }
    return sqrt(acc);
}

/* ------------------------------------------------------------------------ */
/* Step 3 literal: sortperm (sec 4.5; Fig. GPU_sortperm).  */
/* perm = stable ascending argsort (0-based); dense = 1 + #distinct values  */
/* strictly below (reading A3).                                             */
/* ------------------------------------------------------------------------ */
typedef struct { double v; int64_t i; } vi_rec;

static int cmp_vi(const void* pa, const void* pb) {
    const vi_rec* a = (const vi_rec*)pa;
    const vi_rec* b = (const vi_rec*)pb;
    if (a->v < b->v) return -1;
    if (a->v > b->v) return 1;
    return (a->i > b->i) - (a->i < b->i);
}

void or_sortperm(const double* v, int64_t n, int64_t* perm, uint32_t* dense) {
    vi_rec* r = (vi_rec*)malloc((size_t)(n ? n : 1) * sizeof(vi_rec));
    for (int64_t i = 0; i < n; ++i) { r[i].v = v[i]; r[i].i = i; }
    qsort(r, (size_t)n, sizeof(vi_rec), cmp_vi);
    uint32_t rank = 0;
    for (int64_t p = 0; p < n; ++p) {
        if (p == 0 || r[p].v != r[p - 1].v) rank++;
        perm[p] = r[p].i;
        if (dense) dense[r[p].i] = rank;
    }
    free(r);
}

/* ------------------------------------------------------------------------ */
/* Context: the edge level (steps 1-4) plus optional simplices of dim 2, 3. */
/* ------------------------------------------------------------------------ */
typedef struct {
    int64_t n;
    int32_t d;
    double radius;
    int32_t strict;
    double* X;
    /* edges in filtration order (pos order) */
    int64_t E;
    uint32_t* ev;       /* 2E: (i, j), i < j */
    uint32_t* efilt;    /* E: dense rank, 1-based */
    double* elen;       /* E */
    int64_t nvals;
    double* vor;        /* nvals: value_of_rank[f-1] */
    uint32_t* posmat;   /* n*n: position of edge {i,j}, NONE32 if not kept */
    /* upper neighbour lists N+(v) ascending (built from posmat) */
    int64_t* up_off;    /* n+1 */
    uint32_t* up_nbr;
    /* simplices, index by dimension k = 2, 3 */
    int64_t N[4];
    uint32_t* sv[4];    /* (k+1) * N[k] vertices, filtration order */
    uint32_t* sf[4];    /* N[k] filt */
    uint32_t* rows[4];  /* (k+1) * N[k] boundary rows, ascending */
} or_ctx;

typedef struct { double len; uint32_t i, j; } edge_rec;

static int cmp_edge(const void* pa, const void* pb) {
    const edge_rec* a = (const edge_rec*)pa;
    const edge_rec* b = (const edge_rec*)pb;
    if (a->len < b->len) return -1;
    if (a->len > b->len) return 1;
    if (a->i != b->i) return a->i < b->i ? -1 : 1;
    if (a->j != b->j) return a->j < b->j ? -1 : 1;
    return 0;
}

/* Steps 1-4.  Returns NULL on allocation failure. */
/* Steps 1-4 from either a point cloud X (n x d) or a distance matrix D (n x n,
 * D != NULL): "x is either a point cloud ... or a square symmetric matrix
 * (typically a pairwise distance matrix)" (sec. 3).
 * With D the length of edge (i, j), i < j, is the upper-triangle entry
 * D[i][j] (+0.0, so a -0.0 entry is the length +0.0). */
static or_ctx* or_new_impl(const double* X, const double* D, int64_t n, int32_t d, double radius, int32_t strict) {
    or_ctx* c = (or_ctx*)calloc(1, sizeof(or_ctx));
    if (!c) return NULL;
    c->n = n; c->d = d; c->radius = radius; c->strict = strict;
    c->X = (double*)malloc((size_t)(n * d ? n * d : 1) * sizeof(double));
    if (X) memcpy(c->X, X, (size_t)(n * d) * sizeof(double));

    /* Steps 1-2: every pair i < j, keep iff len <= r (len < r when strict). */
    int64_t cap = 1024, E = 0;
    edge_rec* er = (edge_rec*)malloc((size_t)cap * sizeof(edge_rec));
    for (int64_t i = 0; i < n; ++i) {
        for (int64_t j = i + 1; j < n; ++j) {
            double len = D ? D[i * n + j] + 0.0 : or_length(c->X, d, i, j);
            int keep = strict ? (len < radius) : (len <= radius);
            if (!keep) continue;
            if (E == cap) { cap *= 2; er = (edge_rec*)realloc(er, (size_t)cap * sizeof(edge_rec)); }
            er[E].len = len; er[E].i = (uint32_t)i; er[E].j = (uint32_t)j;
            E++;
        }
    }
    /* Step 3: sort by (len, i, j); dense rank = 1 + #distinct lengths below. */
    qsort(er, (size_t)E, sizeof(edge_rec), cmp_edge);
    c->E = E;
    c->ev = (uint32_t*)malloc((size_t)(2 * E + 1) * sizeof(uint32_t));
    c->efilt = (uint32_t*)malloc((size_t)(E + 1) * sizeof(uint32_t));
    c->elen = (double*)malloc((size_t)(E + 1) * sizeof(double));
    c->vor = (double*)malloc((size_t)(E + 1) * sizeof(double));
    uint32_t rank = 0;
    for (int64_t p = 0; p < E; ++p) {
        if (p == 0 || er[p].len != er[p - 1].len) {
            rank++;
            c->vor[rank - 1] = er[p].len;
        }
        c->ev[2 * p] = er[p].i;
        c->ev[2 * p + 1] = er[p].j;
        c->efilt[p] = rank;
        c->elen[p] = er[p].len;
    }
    c->nvals = rank;
    free(er);

    /* position table of every kept edge */
    c->posmat = (uint32_t*)malloc((size_t)(n * n ? n * n : 1) * sizeof(uint32_t));
    if (!c->posmat) return c;
    for (int64_t q = 0; q < n * n; ++q) c->posmat[q] = NONE32;
    for (int64_t p = 0; p < E; ++p) {
        int64_t i = c->ev[2 * p], j = c->ev[2 * p + 1];
        c->posmat[i * n + j] = (uint32_t)p;
        c->posmat[j * n + i] = (uint32_t)p;
    }
    /* upper neighbour lists, ascending */
    c->up_off = (int64_t*)calloc((size_t)(n + 1), sizeof(int64_t));
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = i + 1; j < n; ++j)
            if (c->posmat[i * n + j] != NONE32) c->up_off[i + 1]++;
    for (int64_t i = 0; i < n; ++i) c->up_off[i + 1] += c->up_off[i];
    c->up_nbr = (uint32_t*)malloc((size_t)(c->up_off[n] + 1) * sizeof(uint32_t));
    for (int64_t i = 0; i < n; ++i) {
        int64_t w = c->up_off[i];
        for (int64_t j = i + 1; j < n; ++j)
            if (c->posmat[i * n + j] != NONE32) c->up_nbr[w++] = (uint32_t)j;
    }
    return c;
}

or_ctx* or_new(const double* X, int64_t n, int32_t d, double radius, int32_t strict) {
    return or_new_impl(X, NULL, n, d, radius, strict);
}

or_ctx* or_new_dm(const double* D, int64_t n, double radius, int32_t strict) {
    return or_new_impl(NULL, D, n, 0, radius, strict);
}

/* latlon2euc (sec. 3): spherical coordinates in degrees on the
 * unit sphere -> Euclidean (cos(lat) cos(lon), cos(lat) sin(lon), sin(lat)).
 * P:403-407 prints (34.983, 63.1333) -> (0.370265, 0.730885, 0.573333). */
void or_latlon2euc(const double* latlon, int64_t n, double* xyz) {
    const double deg = 3.14159265358979323846 / 180.0;
    for (int64_t i = 0; i < n; ++i) {
        double la = latlon[2 * i] * deg, lo = latlon[2 * i + 1] * deg;
        xyz[3 * i] = cos(la) * cos(lo);
        xyz[3 * i + 1] = cos(la) * sin(lo);
        xyz[3 * i + 2] = sin(la);
    }
}

void or_free(or_ctx* c) {
    if (!c) return;
    free(c->X); free(c->ev); free(c->efilt); free(c->elen); free(c->vor);
    free(c->posmat); free(c->up_off); free(c->up_nbr);
    for (int k = 0; k < 4; ++k) { free(c->sv[k]); free(c->sf[k]); free(c->rows[k]); }
    free(c);
}

int64_t or_n_edges(const or_ctx* c) { return c->E; }
int64_t or_n_vals(const or_ctx* c) { return c->nvals; }

void or_get_edges(const or_ctx* c, uint32_t* ev, uint32_t* efilt, double* elen, double* vor) {
    if (ev) memcpy(ev, c->ev, (size_t)(2 * c->E) * sizeof(uint32_t));
    if (efilt) memcpy(efilt, c->efilt, (size_t)c->E * sizeof(uint32_t));
    if (elen) memcpy(elen, c->elen, (size_t)c->E * sizeof(double));
    if (vor) memcpy(vor, c->vor, (size_t)c->nvals * sizeof(double));
}

/* position of edge {i,j}, or -1 */
int64_t or_edge_pos(const or_ctx* c, int64_t i, int64_t j) {
    uint32_t p = c->posmat[i * c->n + j];
    return p == NONE32 ? -1 : (int64_t)p;
}

static uint32_t edge_filt(const or_ctx* c, uint32_t a, uint32_t b) {
    return c->efilt[c->posmat[(int64_t)a * c->n + b]];
}

static int adjacent(const or_ctx* c, uint32_t a, uint32_t b) {
    return c->posmat[(int64_t)a * c->n + b] != NONE32;
}

/* ------------------------------------------------------------------------ */
/* Steps 5-7 for one dimension k (2 or 3); dimension k-1 must exist.        */
/* ------------------------------------------------------------------------ */
typedef struct { uint32_t filt; uint32_t v[4]; } simp_rec;
static int g_cmp_len;   /* number of vertices compared by cmp_simp */

static int cmp_simp(const void* pa, const void* pb) {
    const simp_rec* a = (const simp_rec*)pa;
    const simp_rec* b = (const simp_rec*)pb;
    if (a->filt != b->filt) return a->filt < b->filt ? -1 : 1;
    for (int t = 0; t < g_cmp_len; ++t)
        if (a->v[t] != b->v[t]) return a->v[t] < b->v[t] ? -1 : 1;
    return 0;
}

static int cmp_lex(const void* pa, const void* pb) {
    const simp_rec* a = (const simp_rec*)pa;
    const simp_rec* b = (const simp_rec*)pb;
    for (int t = 0; t < g_cmp_len; ++t)
        if (a->v[t] != b->v[t]) return a->v[t] < b->v[t] ? -1 : 1;
    return 0;
}

/* Lex-sorted lookup table of dim-(k-1) simplices: v[] = vertices, filt = pos. */
static simp_rec* face_table(const or_ctx* c, int32_t km1, int64_t* count) {
    int64_t N = c->N[km1];
    simp_rec* t = (simp_rec*)malloc((size_t)(N ? N : 1) * sizeof(simp_rec));
    const uint32_t* V = km1 == 1 ? c->ev : c->sv[km1];
    for (int64_t q = 0; q < N; ++q) {
        memset(&t[q], 0, sizeof(simp_rec));
        for (int s = 0; s <= km1; ++s) t[q].v[s] = V[q * (km1 + 1) + s];
        t[q].filt = (uint32_t)q;
    }
    g_cmp_len = km1 + 1;
    qsort(t, (size_t)N, sizeof(simp_rec), cmp_lex);
    *count = N;
    return t;
}

static uint32_t face_pos(const simp_rec* tab, int64_t N, int32_t len, const uint32_t* v) {
    simp_rec key;
    memset(&key, 0, sizeof(key));
    for (int s = 0; s < len; ++s) key.v[s] = v[s];
    g_cmp_len = len;
    const simp_rec* hit = (const simp_rec*)bsearch(&key, tab, (size_t)N, sizeof(simp_rec), cmp_lex);
    return hit ? hit->filt : NONE32;
}

/* Returns the number of k-simplices, or -1 on bad arguments. */
int64_t or_build_simplices(or_ctx* c, int32_t k) {
    if (k < 2 || k > 3) return -1;
    if (k == 3 && !c->sv[2]) return -1;
    c->N[1] = c->E;
    int64_t cap = 1024, N = 0;
    simp_rec* s = (simp_rec*)malloc((size_t)cap * sizeof(simp_rec));
    /* Step 5: all (k+1)-tuples v0 < ... < vk whose every pair is an edge,
     * by neighbour-list loops; filt = max edge filt (A3). */
    for (int64_t i = 0; i < c->n; ++i) {
        for (int64_t a = c->up_off[i]; a < c->up_off[i + 1]; ++a) {
            uint32_t j = c->up_nbr[a];
            for (int64_t b = c->up_off[j]; b < c->up_off[j + 1]; ++b) {
                uint32_t l = c->up_nbr[b];
                if (!adjacent(c, (uint32_t)i, l)) continue;
                if (k == 2) {
                    uint32_t f = edge_filt(c, (uint32_t)i, j);
                    if (edge_filt(c, (uint32_t)i, l) > f) f = edge_filt(c, (uint32_t)i, l);
                    if (edge_filt(c, j, l) > f) f = edge_filt(c, j, l);
                    if (N == cap) { cap *= 2; s = (simp_rec*)realloc(s, (size_t)cap * sizeof(simp_rec)); }
                    memset(&s[N], 0, sizeof(simp_rec));
                    s[N].filt = f; s[N].v[0] = (uint32_t)i; s[N].v[1] = j; s[N].v[2] = l;
                    N++;
                } else {
                    for (int64_t q = c->up_off[l]; q < c->up_off[l + 1]; ++q) {
                        uint32_t m = c->up_nbr[q];
                        if (!adjacent(c, (uint32_t)i, m) || !adjacent(c, j, m)) continue;
                        uint32_t vv[4] = {(uint32_t)i, j, l, m};
                        uint32_t f = 0;
                        for (int x = 0; x < 4; ++x)
                            for (int y = x + 1; y < 4; ++y) {
                                uint32_t g = edge_filt(c, vv[x], vv[y]);
                                if (g > f) f = g;
                            }
                        if (N == cap) { cap *= 2; s = (simp_rec*)realloc(s, (size_t)cap * sizeof(simp_rec)); }
                        memset(&s[N], 0, sizeof(simp_rec));
                        s[N].filt = f;
                        for (int x = 0; x < 4; ++x) s[N].v[x] = vv[x];
                        N++;
                    }
                }
            }
        }
    }
    /* Step 6: sort by (filt, v0, ..., vk) (reading A4). */
    g_cmp_len = k + 1;
    qsort(s, (size_t)N, sizeof(simp_rec), cmp_simp);
    free(c->sv[k]); free(c->sf[k]); free(c->rows[k]);
    c->N[k] = N;
    c->sv[k] = (uint32_t*)malloc((size_t)((k + 1) * N + 1) * sizeof(uint32_t));
    c->sf[k] = (uint32_t*)malloc((size_t)(N + 1) * sizeof(uint32_t));
    c->rows[k] = (uint32_t*)malloc((size_t)((k + 1) * N + 1) * sizeof(uint32_t));
    for (int64_t q = 0; q < N; ++q) {
        c->sf[k][q] = s[q].filt;
        for (int x = 0; x <= k; ++x) c->sv[k][q * (k + 1) + x] = s[q].v[x];
    }
    free(s);
    /* Step 7: column q = ascending positions of its k+1 faces (A7). */
    int64_t NF;
    simp_rec* tab = face_table(c, k - 1, &NF);
    for (int64_t q = 0; q < N; ++q) {
        uint32_t r[4];
        for (int t = 0; t <= k; ++t) {
            uint32_t f[3];
            int w = 0;
            for (int x = 0; x <= k; ++x)
                if (x != t) f[w++] = c->sv[k][q * (k + 1) + x];
            r[t] = face_pos(tab, NF, k, f);
        }
        for (int x = 1; x <= k; ++x)            /* insertion sort, ascending */
            for (int y = x; y > 0 && r[y - 1] > r[y]; --y) {
                uint32_t tmp = r[y]; r[y] = r[y - 1]; r[y - 1] = tmp;
            }
        for (int x = 0; x <= k; ++x) c->rows[k][q * (k + 1) + x] = r[x];
    }
    free(tab);
    return N;
}

void or_get_simplices(const or_ctx* c, int32_t k, uint32_t* verts, uint32_t* filt, uint32_t* rows) {
    int64_t N = c->N[k];
    if (verts) memcpy(verts, c->sv[k], (size_t)((k + 1) * N) * sizeof(uint32_t));
    if (filt) memcpy(filt, c->sf[k], (size_t)N * sizeof(uint32_t));
    if (rows) memcpy(rows, c->rows[k], (size_t)((k + 1) * N) * sizeof(uint32_t));
}

/* ------------------------------------------------------------------------ */
/* Sampled parity at full size: the same definitions, one level at a time.  */
/* ------------------------------------------------------------------------ */

/* hist[f] = number of k-simplices (k = 2, 3) with filt f, f in 0..nvals.   */
/* Same enumeration as step 5, without storing the simplices.              */
void or_filt_hist(const or_ctx* c, int32_t k, uint64_t* hist) {
    memset(hist, 0, (size_t)(c->nvals + 1) * sizeof(uint64_t));
    for (int64_t i = 0; i < c->n; ++i) {
        for (int64_t a = c->up_off[i]; a < c->up_off[i + 1]; ++a) {
            uint32_t j = c->up_nbr[a];
            uint32_t fij = edge_filt(c, (uint32_t)i, j);
            for (int64_t b = c->up_off[j]; b < c->up_off[j + 1]; ++b) {
                uint32_t l = c->up_nbr[b];
                uint32_t pil = c->posmat[i * c->n + l];
                if (pil == NONE32) continue;
                uint32_t f = fij;
                if (c->efilt[pil] > f) f = c->efilt[pil];
                uint32_t fjl = edge_filt(c, j, l);
                if (fjl > f) f = fjl;
                if (k == 2) { hist[f]++; continue; }
                for (int64_t q = c->up_off[l]; q < c->up_off[l + 1]; ++q) {
                    uint32_t m = c->up_nbr[q];
                    uint32_t pim = c->posmat[i * c->n + m];
                    uint32_t pjm = c->posmat[(int64_t)j * c->n + m];
                    if (pim == NONE32 || pjm == NONE32) continue;
                    uint32_t g = f;
                    if (c->efilt[pim] > g) g = c->efilt[pim];
                    if (c->efilt[pjm] > g) g = c->efilt[pjm];
                    uint32_t flm = edge_filt(c, l, m);
                    if (flm > g) g = flm;
                    hist[g]++;
                }
            }
        }
    }
}

/* All k-simplices (k = 2, 3) with filt == f, in lex order, with their      */
/* boundary rows when k == 2 (edge positions, ascending).  Every such       */
/* simplex contains an edge of filt f (filt = max edge filt), so it is      */
/* found by extending each edge of level f.  Returns the count (may exceed  */
/* cap, in which case only cap are written).                                */
int64_t or_simplices_at_filt(const or_ctx* c, int32_t k, uint32_t f,
                             uint32_t* verts, uint32_t* rows, int64_t cap) {
    int64_t scap = 64, N = 0;
    simp_rec* s = (simp_rec*)malloc((size_t)scap * sizeof(simp_rec));
    for (int64_t p = 0; p < c->E; ++p) {
        if (c->efilt[p] != f) continue;
        uint32_t a = c->ev[2 * p], b = c->ev[2 * p + 1];
        for (uint32_t x = 0; x < (uint32_t)c->n; ++x) {
            if (x == a || x == b) continue;
            if (!adjacent(c, a, x) || !adjacent(c, b, x)) continue;
            if (edge_filt(c, a, x) > f || edge_filt(c, b, x) > f) continue;
            if (k == 2) {
                uint32_t v[3] = {a, b, x};
                for (int q = 1; q < 3; ++q)
                    for (int y = q; y > 0 && v[y - 1] > v[y]; --y) { uint32_t t = v[y]; v[y] = v[y - 1]; v[y - 1] = t; }
                if (N == scap) { scap *= 2; s = (simp_rec*)realloc(s, (size_t)scap * sizeof(simp_rec)); }
                memset(&s[N], 0, sizeof(simp_rec));
                s[N].filt = f; s[N].v[0] = v[0]; s[N].v[1] = v[1]; s[N].v[2] = v[2];
                N++;
            } else {
                for (uint32_t y = x + 1; y < (uint32_t)c->n; ++y) {
                    if (y == a || y == b) continue;
                    if (!adjacent(c, a, y) || !adjacent(c, b, y) || !adjacent(c, x, y)) continue;
                    if (edge_filt(c, a, y) > f || edge_filt(c, b, y) > f || edge_filt(c, x, y) > f) continue;
                    uint32_t v[4] = {a, b, x, y};
                    for (int q = 1; q < 4; ++q)
                        for (int z = q; z > 0 && v[z - 1] > v[z]; --z) { uint32_t t = v[z]; v[z] = v[z - 1]; v[z - 1] = t; }
                    if (N == scap) { scap *= 2; s = (simp_rec*)realloc(s, (size_t)scap * sizeof(simp_rec)); }
                    memset(&s[N], 0, sizeof(simp_rec));
                    s[N].filt = f;
                    for (int z = 0; z < 4; ++z) s[N].v[z] = v[z];
                    N++;
                }
            }
        }
    }
    /* lex order, duplicates removed (a simplex with several level-f edges is
     * reached once per such edge) */
    g_cmp_len = k + 1;
    qsort(s, (size_t)N, sizeof(simp_rec), cmp_lex);
    int64_t U = 0;
    for (int64_t q = 0; q < N; ++q)
        if (U == 0 || cmp_lex(&s[U - 1], &s[q]) != 0) s[U++] = s[q];
    for (int64_t q = 0; q < U && q < cap; ++q) {
        for (int z = 0; z <= k; ++z) verts[q * (k + 1) + z] = s[q].v[z];
        if (k == 2 && rows) {
            uint32_t r[3] = {c->posmat[(int64_t)s[q].v[0] * c->n + s[q].v[1]],
                             c->posmat[(int64_t)s[q].v[0] * c->n + s[q].v[2]],
                             c->posmat[(int64_t)s[q].v[1] * c->n + s[q].v[2]]};
            for (int x = 1; x < 3; ++x)
                for (int y = x; y > 0 && r[y - 1] > r[y]; --y) { uint32_t t = r[y]; r[y] = r[y - 1]; r[y - 1] = t; }
            for (int x = 0; x < 3; ++x) rows[q * 3 + x] = r[x];
        }
    }
    free(s);
    return U;
}

/* ------------------------------------------------------------------------ */
/* Step 8: barcodes by textbook GF(2) reduction.                            */
/* ------------------------------------------------------------------------ */
/* Column j of D_k as a sorted index vector (rows ascending). */
static void column_of(const or_ctx* c, int32_t k, int64_t j, vec32* out) {
    out->n = 0;
    if (k == 1) {
        v32_push(out, c->ev[2 * j]);
        v32_push(out, c->ev[2 * j + 1]);
    } else {
        for (int x = 0; x <= k; ++x) v32_push(out, c->rows[k][j * (k + 1) + x]);
    }
}

/* a <- a + b over GF(2): symmetric difference of two ascending vectors. */
static void gf2_add(vec32* a, const vec32* b, vec32* tmp) {
    tmp->n = 0;
    int64_t x = 0, y = 0;
    while (x < a->n || y < b->n) {
        if (y >= b->n || (x < a->n && a->a[x] < b->a[y])) v32_push(tmp, a->a[x++]);
        else if (x >= a->n || b->a[y] < a->a[x]) v32_push(tmp, b->a[y++]);
        else { x++; y++; }
    }
    vec32 t = *a; *a = *tmp; *tmp = t;
}

static int64_t ncols_of(const or_ctx* c, int32_t k) { return k == 1 ? c->E : c->N[k]; }
static int64_t nrows_of(const or_ctx* c, int32_t k) { return k == 1 ? c->n : (k == 2 ? c->E : c->N[2]); }
static uint32_t filt_of(const or_ctx* c, int32_t k, int64_t q) {
    if (k == 0) return 0;                 /* vertices: filt 0 (step 4) */
    if (k == 1) return c->efilt[q];
    return c->sf[k][q];
}

/* Textbook reduction of the columns R[0..nc) (each an ascending row-index  */
/* vector over GF(2)) with nr rows.  method 0: pHcol (Algorithm 1,          */
/* P:210-227; V update reading A10).  method 1: pHrow (Algorithm 2,         */
/* P:229-248; reading A10: clear each later column of `indices` against    */
/* p = indices[0]).  pivot_row[r] = the column whose reduced low is r, or  */
/* -1.  zero[j] = 1 iff column j reduced to zero.                          */
static void reduce_core(vec32* R, int64_t nc, int64_t nr, int method,
                        int64_t* pivot_row, uint8_t* zero) {
    vec32 tmp = {0, 0, 0};
    for (int64_t r = 0; r < nr; ++r) pivot_row[r] = -1;
    if (method == 0) {
        for (int64_t j = 0; j < nc; ++j) {
            /* while exists j' < j with low(j') == low(j): R_j += R_j' */
            while (R[j].n > 0 && pivot_row[R[j].a[R[j].n - 1]] >= 0)
                gf2_add(&R[j], &R[pivot_row[R[j].a[R[j].n - 1]]], &tmp);
            if (R[j].n > 0) pivot_row[R[j].a[R[j].n - 1]] = j;
        }
    } else {
        /* rows from the bottom: indices = [j | low(j) == i], p = indices[0] */
        for (int64_t i = nr - 1; i >= 0; --i) {
            int64_t p = -1;
            for (int64_t j = 0; j < nc; ++j) {
                if (R[j].n == 0 || R[j].a[R[j].n - 1] != (uint32_t)i) continue;
                if (p < 0) p = j;
                else gf2_add(&R[j], &R[p], &tmp);
            }
            if (p >= 0) pivot_row[i] = p;
        }
    }
    for (int64_t j = 0; j < nc; ++j) zero[j] = R[j].n == 0;
    free(tmp.a);
}

/* Generic entry: reduce an arbitrary GF(2) CSC matrix (rows ascending in   */
/* each column).  Used to pin the pivot -> bar mapping on Fig. 4.   */
void or_reduce(int64_t nr, int64_t nc, const int64_t* colptr, const uint32_t* rowval,
               int32_t method, int64_t* pivot_row, uint8_t* zero) {
    vec32* R = (vec32*)calloc((size_t)(nc ? nc : 1), sizeof(vec32));
    for (int64_t j = 0; j < nc; ++j)
        for (int64_t q = colptr[j]; q < colptr[j + 1]; ++q) v32_push(&R[j], rowval[q]);
    reduce_core(R, nc, nr, method, pivot_row, zero);
    for (int64_t j = 0; j < nc; ++j) free(R[j].a);
    free(R);
}

/* F4: blockprodsum (sec. 4.6, Fig. BlkProdSum): S = D + C E    */
/* over GF(2) ("using the modulo-2 operation"), all CSC.   */
/* Column j of S is the mod-2 sum of column j of D and the columns C[:, i]  */
/* for every i in column j of E, written out as a dense 0/1 accumulator of  */
/* nr entries per column (textbook, no blocking).  Returns nnz(S); the      */
/* caller sizes s_rowval with an upper bound or calls twice (s_rowval NULL  */
/* counts only).  s_colptr has nc + 1 entries; rows ascending.              */
int64_t or_blockprodsum(int64_t nr, int64_t nc,
                        const int64_t* d_colptr, const uint32_t* d_rowval,
                        const int64_t* c_colptr, const uint32_t* c_rowval,
                        const int64_t* e_colptr, const uint32_t* e_rowval,
                        int64_t* s_colptr, uint32_t* s_rowval) {
    uint8_t* acc = (uint8_t*)calloc((size_t)(nr ? nr : 1), 1);
    int64_t nnz = 0;
    if (s_colptr) s_colptr[0] = 0;
    for (int64_t j = 0; j < nc; ++j) {
        for (int64_t q = d_colptr[j]; q < d_colptr[j + 1]; ++q) acc[d_rowval[q]] ^= 1;
        for (int64_t q = e_colptr[j]; q < e_colptr[j + 1]; ++q) {
            uint32_t i = e_rowval[q];
            for (int64_t t = c_colptr[i]; t < c_colptr[i + 1]; ++t) acc[c_rowval[t]] ^= 1;
        }
        for (int64_t r = 0; r < nr; ++r) {
            if (acc[r]) {
                if (s_rowval) s_rowval[nnz] = (uint32_t)r;
                nnz++;
                acc[r] = 0;
            }
        }
        if (s_colptr) s_colptr[j + 1] = nnz;
    }
    free(acc);
    return nnz;
}

/* Reduce D_k of the context; cleared[j] != 0 marks columns zeroed          */
/* beforehand (clearing).                                            */
static void reduce_dim(const or_ctx* c, int32_t k, int method, const uint8_t* cleared,
                       int64_t* pivot_row, uint8_t* zero) {
    int64_t nc = ncols_of(c, k), nr = nrows_of(c, k);
    vec32* R = (vec32*)calloc((size_t)(nc ? nc : 1), sizeof(vec32));
    for (int64_t j = 0; j < nc; ++j)
        if (!(cleared && cleared[j])) column_of(c, k, j, &R[j]);
    reduce_core(R, nc, nr, method, pivot_row, zero);
    for (int64_t j = 0; j < nc; ++j) free(R[j].a);
    free(R);
}

/* Bars (dim, birth filt, death filt or -1 = infinity) of dims 0..maxdim.   */
/* method: 0 pHcol, 1 pHrow, 2 pHcol with clearing.                  */
/* Pair from pivot (low, j) of D_k: dim k-1, birth filt_{k-1}[low], death   */
/* filt_k[j] (Fig. 4 caption P:286; reading A13).  Essential: dim-k simplex */
/* whose column reduced to zero and which is no pivot row of D_{k+1}        */
/* (reading A8).  Bars of zero real length (value(birth) == value(death),  */
/* filt 0 -> 0.0) dropped unless keep_zero (reading A9).                    */
/* Needs simplices built up to dimension maxdim + 1.  With top != 0 the    */
/* unkilled cycles of the top dimension K = maxdim + 1 are reported too (as */
/* dim-K infinite bars; used by the Euler pin P11).  Returns bar count.     */
int64_t or_barcodes(const or_ctx* c, int32_t maxdim, int32_t method, int32_t keep_zero,
                    int32_t top, int64_t* out, int64_t cap) {
    int32_t K = maxdim + 1;
    int64_t* piv[5] = {0};
    uint8_t* zero[5] = {0};
    uint8_t* cleared[5] = {0};
    for (int32_t k = K; k >= 1; --k) {
        int64_t nc = ncols_of(c, k), nr = nrows_of(c, k);
        piv[k] = (int64_t*)malloc((size_t)(nr ? nr : 1) * sizeof(int64_t));
        zero[k] = (uint8_t*)malloc((size_t)(nc ? nc : 1));
        if (method == 2 && k < K) {
            cleared[k] = (uint8_t*)calloc((size_t)(nc ? nc : 1), 1);
            for (int64_t r = 0; r < nc; ++r)
                if (piv[k + 1][r] >= 0) cleared[k][r] = 1;
        }
        reduce_dim(c, k, method == 1 ? 1 : 0, cleared[k], piv[k], zero[k]);
        if (cleared[k])     /* a cleared column is zero in the reduced matrix */
            for (int64_t r = 0; r < nc; ++r) if (cleared[k][r]) zero[k][r] = 1;
    }
    int64_t nb = 0;
#define EMIT(D, B, DE) do { if (nb < cap) { out[3*nb] = (D); out[3*nb+1] = (B); out[3*nb+2] = (DE); } nb++; } while (0)
    for (int32_t k = 1; k <= K; ++k) {
        int64_t nr = nrows_of(c, k);
        for (int64_t r = 0; r < nr; ++r) {
            int64_t j = piv[k][r];
            if (j < 0) continue;
            uint32_t b = filt_of(c, k - 1, r), dth = filt_of(c, k, j);
            /* zero length in real values: filt 0 -> 0.0, f -> value_of_rank[f-1] */
            double vb = b ? c->vor[b - 1] : 0.0, vd = dth ? c->vor[dth - 1] : 0.0;
            if (vb == vd && !keep_zero) continue;
            EMIT(k - 1, b, dth);
        }
    }
    for (int32_t k = 0; k <= (top ? K : maxdim); ++k) {
        int64_t ns = k == 0 ? c->n : ncols_of(c, k);
        for (int64_t q = 0; q < ns; ++q) {
            int z = k == 0 ? 1 : zero[k][q];
            if (!z) continue;
            if (k + 1 <= K && piv[k + 1][q] >= 0) continue;
            EMIT(k, filt_of(c, k, q), -1);
        }
    }
#undef EMIT
    for (int k = 0; k < 5; ++k) { free(piv[k]); free(zero[k]); free(cleared[k]); }
    return nb;
}
