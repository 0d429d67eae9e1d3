/*
 * oracle.c -- plain, slow, obviously-correct CPU Min-Sum decoder.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_2507_10424_b200/) never links, imports or calls it,
 * and this file shares no code, header, table or constant with the CUDA path.
 *
 * Citations: "P:n" = line n of the paper text (PAPER.md, arXiv 2507.10424),
 * "S:n" = line n of SPEC.md.  Readings of ambiguous passages (A1..A20) are
 * listed in DESIGN.md section "Readings of the paper".
 *
 * What it computes (Algorithm 1, with the pre-loop check of
 * Listing 1), per frame, entirely in REAL arithmetic:
 *
 *   N_i = ascending columns j with H(i,j)=1
 *   M_j = ascending rows    i with H(i,j)=1
 *   s_j = r_j ; eta_{i,j} = 0 ; k = 0
 *   pre-check: b = slice(s); H.b == 0 -> (true, 0)  (reading A9)
 *   while k < L:
 *     CN  eta_{i,j} = min_{k in N_i, k!=j} |x_k| * prod_{k!=j} sign(x_k),
 *         x_k = s_k - eta^prev_{i,k}                (Eq. eta_update)
 *         sign(0) = +1                              (reading A12)
 *         times (-1)^{d_i} under the CORRECTED rule  (reading A1)
 *     BN  s_j = (sum over i in M_j ascending of eta_{i,j}) + r_j
 *                                                  (Eq. lambda_j; order A14)
 *     k = k + 1
 *     b = slice(s): b_j = 1 iff s_j > 0             (Eq. slice)
 *     H.b == 0 (mod 2) -> isCodeword
 *
 * The check-node update is the literal leave-one-out definition of
 * Eq. eta_update: an O(d_i^2) brute-force minimum and sign product per edge.
 * It deliberately does NOT use Observation 1/2; the CUDA path does,
 * and the two must agree exactly (Observations 1 and 2 are exact identities).
 *
 * Compiled twice: REAL=float (parity reference, fp32 as the kernel computes;
 * see DESIGN.md "precision") and REAL=double (fp64 shadow for drift reports).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#ifndef REAL
#define REAL float
#endif
#ifndef SFX
#define SFX f32
#endif
#define CAT2(a, b) a##_##b
#define CAT(a, b) CAT2(a, b)
#define NAME(x) CAT(x, SFX)

/* flags -- same meaning as documented in oracle/__init__.py */
#define ORACLE_SIGN_PAPER_LITERAL 1 /* drop the (-1)^{d_i} factor (reading A1) */
#define ORACLE_NO_EARLY_STOP 2      /* no pre-check, no early exit; exactly L bodies */

/* ------------------------------------------------------------------------ */
/* Tanner graph of H, built from the list of ones of H.   */
/* ------------------------------------------------------------------------ */
typedef struct {
    int m, n;
    int64_t E;
    int64_t *row_ptr; /* N_i = row_col[row_ptr[i] .. row_ptr[i+1]) ascending */
    int32_t *row_col;
    int64_t *col_ptr; /* M_j = col_row[col_ptr[j] .. col_ptr[j+1]) ascending */
    int32_t *col_row;
    int64_t *col_edge; /* position of (i,j) inside row storage, for eta_{i,j} */
} graph_t;

static int cmp_i32(const void *a, const void *b) {
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return (x > y) - (x < y);
}

static void graph_free(graph_t *g) {
    free(g->row_ptr); free(g->row_col); free(g->col_ptr); free(g->col_row); free(g->col_edge);
    memset(g, 0, sizeof(*g));
}

/* returns 0, or -1 (index out of range), -2 (duplicate one), -3 (row degree < 2) */
static int graph_build(graph_t *g, const int32_t *rows, const int32_t *cols, int64_t nnz, int m, int n) {
    memset(g, 0, sizeof(*g));
    g->m = m; g->n = n; g->E = nnz;
    g->row_ptr = calloc((size_t)m + 1, sizeof(int64_t));
    g->col_ptr = calloc((size_t)n + 1, sizeof(int64_t));
    g->row_col = malloc(sizeof(int32_t) * (size_t)(nnz > 0 ? nnz : 1));
    g->col_row = malloc(sizeof(int32_t) * (size_t)(nnz > 0 ? nnz : 1));
    g->col_edge = malloc(sizeof(int64_t) * (size_t)(nnz > 0 ? nnz : 1));
    for (int64_t t = 0; t < nnz; t++) {
        if (rows[t] < 0 || rows[t] >= m || cols[t] < 0 || cols[t] >= n) { graph_free(g); return -1; }
        g->row_ptr[rows[t] + 1]++;
        g->col_ptr[cols[t] + 1]++;
    }
    for (int i = 0; i < m; i++) g->row_ptr[i + 1] += g->row_ptr[i];
    for (int j = 0; j < n; j++) g->col_ptr[j + 1] += g->col_ptr[j];
    int64_t *fill = calloc((size_t)(m > n ? m : n) + 1, sizeof(int64_t));
    for (int64_t t = 0; t < nnz; t++) {
        int i = rows[t];
        g->row_col[g->row_ptr[i] + fill[i]++] = cols[t];
    }
    /* N_i in ascending column order */
    for (int i = 0; i < m; i++) {
        int64_t a = g->row_ptr[i], b = g->row_ptr[i + 1];
        qsort(g->row_col + a, (size_t)(b - a), sizeof(int32_t), cmp_i32);
        for (int64_t e = a + 1; e < b; e++)
            if (g->row_col[e] == g->row_col[e - 1]) { free(fill); graph_free(g); return -2; }
        if (b - a < 2) { free(fill); graph_free(g); return -3; }
    }
    /* M_j: walking rows in ascending order visits each column's rows ascending */
    memset(fill, 0, sizeof(int64_t) * ((size_t)(m > n ? m : n) + 1));
    for (int i = 0; i < m; i++)
        for (int64_t e = g->row_ptr[i]; e < g->row_ptr[i + 1]; e++) {
            int j = g->row_col[e];
            int64_t slot = g->col_ptr[j] + fill[j]++;
            g->col_row[slot] = i;
            g->col_edge[slot] = e;
        }
    free(fill);
    return 0;
}

/* H.b over GF(2): syndrome_i = XOR_{j in N_i} b_j.  Returns #unsatisfied. */
static int syndrome_weight(const graph_t *g, const uint8_t *b) {
    int w = 0;
    for (int i = 0; i < g->m; i++) {
        int acc = 0;
        for (int64_t e = g->row_ptr[i]; e < g->row_ptr[i + 1]; e++) acc ^= b[g->row_col[e]];
        w += acc;
    }
    return w;
}

/* sign(x) with sign(0) = +1.  -0.0 is not < 0, so it is +1 too (A12). */
static REAL sign_of(REAL x) { return (x < (REAL)0) ? (REAL)-1 : (REAL)1; }

/*
 * Check-node update of one row, Eq. eta_update, literal leave-one-out:
 *   eta_j = min_{k != j} |x_k| * prod_{k != j} sign(x_k)
 * multiplied by (-1)^d under the CORRECTED sign rule (reading A1: the paper's
 * "strictly positive means 1" convention).
 */
static void check_node(const REAL *x, int d, int literal, REAL *eta) {
    for (int j = 0; j < d; j++) {
        REAL mag = (REAL)INFINITY;
        REAL sgn = (REAL)1;
        for (int k = 0; k < d; k++) {
            if (k == j) continue;
            REAL a = (REAL)fabs((double)x[k]);
            if (a < mag) mag = a;
            sgn = sgn * sign_of(x[k]);
        }
        if (!literal && (d & 1)) sgn = -sgn;
        eta[j] = sgn * mag;
    }
}

/* exported for the SPEC check-node examples */
void NAME(oracle_check_node)(const REAL *x, int d, int flags, REAL *eta) {
    check_node(x, d, flags & ORACLE_SIGN_PAPER_LITERAL, eta);
}

static void decode_frame(const graph_t *g, const float *r_in, int L, int T, int flags, REAL *s, REAL *r, REAL *eta,
                         REAL *xbuf, REAL *ebuf, uint8_t *b, uint8_t *bits_out, int32_t *iters_out,
                         uint8_t *conv_out, REAL *post_out) {
    const int m = g->m, n = g->n;
    const int literal = flags & ORACLE_SIGN_PAPER_LITERAL;
    const int early = !(flags & ORACLE_NO_EARLY_STOP);
    /* initial state: lambda_j = r(j), eta = 0 */
    for (int j = 0; j < n; j++) { r[j] = (REAL)r_in[j]; s[j] = r[j]; }
    for (int64_t e = 0; e < g->E; e++) eta[e] = (REAL)0;
    int k = 0, is_codeword = 0;
    for (int j = 0; j < n; j++) b[j] = (s[j] > (REAL)0) ? 1 : 0; /* Eq. slice */
    if (early && syndrome_weight(g, b) == 0) is_codeword = 1;   /* pre-loop check */
    while (k < L && !is_codeword) {
        /* check nodes: every row from the previous iteration's s and eta */
        for (int i = 0; i < m; i++) {
            int64_t a = g->row_ptr[i];
            int d = (int)(g->row_ptr[i + 1] - a);
            for (int p = 0; p < d; p++) xbuf[p] = s[g->row_col[a + p]] - eta[a + p]; /* lambda_k - eta^prev_{i,k} */
            check_node(xbuf, d, literal, ebuf);
            for (int p = 0; p < d; p++) eta[a + p] = ebuf[p];
        }
        /* bit nodes: lambda_j = r(j) + sum_{i in M_j} eta_{i,j}; ascending rows, then + r (A14) */
        for (int j = 0; j < n; j++) {
            REAL acc = (REAL)0;
            for (int64_t t = g->col_ptr[j]; t < g->col_ptr[j + 1]; t++) acc = acc + eta[g->col_edge[t]];
            s[j] = acc + r[j];
        }
        k = k + 1;
        for (int j = 0; j < n; j++) b[j] = (s[j] > (REAL)0) ? 1 : 0;
        /* the codeword test runs every T bodies and after the last one ("Termination was checked for
           every 6 iterations"; SPEC checkEvery); T = 1 is Alg. 1 */
        if (early && (k % T == 0 || k == L) && syndrome_weight(g, b) == 0) is_codeword = 1;
    }
    if (!early) is_codeword = (syndrome_weight(g, b) == 0);
    for (int j = 0; j < n; j++) bits_out[j] = b[j];
    *iters_out = k;
    *conv_out = (uint8_t)is_codeword;
    if (post_out) for (int j = 0; j < n; j++) post_out[j] = s[j];
    (void)m;
}

/*
 * Decode `frames` independent frames r[f*n .. f*n+n) with the same H given as
 * its list of ones (rows[t], cols[t]), t < nnz, 0-based.  check_every = T >= 1: the
 * codeword test after loop body k runs when k % T == 0 or k == L (the pre-loop test always).  Outputs as in
 * Alg. 1's KwOut: bits, k, isCodeword, plus the soft vector s.
 * Returns 0 or a negative graph_build error.  threads <= 0 -> library default.
 */
int NAME(oracle_decode)(const int32_t *rows, const int32_t *cols, int64_t nnz, int m, int n, const float *r,
                        int64_t frames, int L, int check_every, int flags, int threads, uint8_t *bits_out,
                        int32_t *iters_out, uint8_t *conv_out, REAL *post_out) {
    if (check_every < 1) return -4;
    graph_t g;
    int rc = graph_build(&g, rows, cols, nnz, m, n);
    if (rc) return rc;
    int maxd = 0;
    for (int i = 0; i < m; i++) {
        int d = (int)(g.row_ptr[i + 1] - g.row_ptr[i]);
        if (d > maxd) maxd = d;
    }
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#pragma omp parallel
#endif
    {
        REAL *s = malloc(sizeof(REAL) * (size_t)n), *rr = malloc(sizeof(REAL) * (size_t)n);
        REAL *eta = malloc(sizeof(REAL) * (size_t)(g.E > 0 ? g.E : 1));
        REAL *xb = malloc(sizeof(REAL) * (size_t)maxd), *eb = malloc(sizeof(REAL) * (size_t)maxd);
        uint8_t *b = malloc((size_t)n);
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 1)
#endif
        for (int64_t f = 0; f < frames; f++)
            decode_frame(&g, r + f * n, L, check_every, flags, s, rr, eta, xb, eb, b, bits_out + f * n, iters_out + f,
                         conv_out + f, post_out ? post_out + f * n : NULL);
        free(s); free(rr); free(eta); free(xb); free(eb); free(b);
    }
    graph_free(&g);
    return 0;
}

/* H.b for a batch of hard vectors; out[f] = number of unsatisfied checks */
int NAME(oracle_syndrome)(const int32_t *rows, const int32_t *cols, int64_t nnz, int m, int n, const uint8_t *b,
                          int64_t frames, int32_t *out) {
    graph_t g;
    /* syndrome is defined for any H (no degree requirement): build without the degree gate */
    memset(&g, 0, sizeof(g));
    int rc = graph_build(&g, rows, cols, nnz, m, n);
    if (rc == -3) {
        /* degree < 2 rows are legal for a plain H.b; recompute directly from the list of ones */
        for (int64_t f = 0; f < frames; f++) {
            int32_t w = 0;
            uint8_t *acc = calloc((size_t)m, 1);
            for (int64_t t = 0; t < nnz; t++) acc[rows[t]] ^= b[f * n + cols[t]];
            for (int i = 0; i < m; i++) w += acc[i];
            free(acc);
            out[f] = w;
        }
        return 0;
    }
    if (rc) return rc;
    for (int64_t f = 0; f < frames; f++) out[f] = syndrome_weight(&g, b + f * n);
    graph_free(&g);
    return 0;
}

int NAME(oracle_max_threads)(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
