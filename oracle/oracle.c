/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY.  The plain, slow, serial CPU oracle for
 * the rank-k Cholesky modification of arXiv 1011.1173 (Walder, "Rank k Cholesky
 * Up/Down-dating on the GPU: gpucholmodV0.2").
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * leg may load this library.  The product path (paper_1011_1173_b200/) never
 * links, imports or calls it, and shares no code, header or constant with it.
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -fPIC -shared
 *        oracle.c -o liboracle.so -lm
 * (-ffp-contract=off keeps every multiply and add separately rounded so that the
 *  two loop orderings of Algorithm 1 give bit-identical results, PAPER.md
 *  Sec. 2 / SPEC.md line 183.)
 *
 * Storage (reading R7): L is upper triangular, column-major with
 * leading dimension ldl; element (i,j), i <= j, lives at L[i + j*ldl]; the
 * strictly lower part is never read or written.  V is n x k column-major with
 * leading dimension n (update vector e is V[e*n .. e*n+n-1]).
 *
 * Everything is fp64 except gcmo_modify_a_f32 (the paper's single-precision runs).
 * Indices below are 0-based; the paper's are 1-based.
 *
 * Functions and the passages they follow:
 *   gcmo_compute        PAPER.md lines 44-49, function Compute
 *   gcmo_apply          PAPER.md lines 52-54, function Apply (2nd line reads the
 *                       NEW L_ij: sequential assignment, reading R2)
 *   gcmo_modify_a       PAPER.md lines 24-30, CholeskyModifyA, with the inner
 *                       loop moved BEFORE Compute (erratum, R1) and the
 *                       rank-k loop of lines 14/73/86 (all k rotations of row j,
 *                       in order e = 0..k-1, per L element; R3)
 *   gcmo_modify_b       PAPER.md lines 34-40, CholeskyModifyB, run as k
 *                       sequential rank-1 sweeps
 *   gcmo_chol_upper     textbook Cholesky A = L^T L (the paper's "LAPACK
 *                       algorithm"), used for brute force.
 *
 * Failure reporting (R5/R6, not in the paper): Compute fails when
 * !(L_ii^2 + sigma*V_i^2 > 0) (code 1, "indefinite downdate"); a pivot with
 * !(L_ii > 0) on entry to row i is code 2 ("non-positive pivot").  After a
 * failure the sweep continues with NaN so that every later quantity of the same
 * and later update columns is NaN; the reported failure is the
 * lexicographically smallest (e, i), which is what k sequential rank-1 calls
 * would report first.
 *
 * Parity pins: see tests/test_oracle.py and DESIGN.md section "Oracle pins".
 */
#include <math.h>
#include <stdint.h>
#include <stddef.h>

typedef struct {
    int32_t code; /* 0 ok, 1 indefinite downdate, 2 non-positive pivot on entry */
    int32_t col;  /* e of the first failure (lexicographic (e, row)) */
    int64_t row;  /* row/column index i of the first failure */
} gcmo_info_t;

static void info_record(gcmo_info_t *info, int32_t code, int64_t e, int64_t i) {
    if (!info) return;
    if (info->code == 0 || e < info->col || (e == info->col && i < info->row)) {
        info->code = code;
        info->col = (int32_t)e;
        info->row = i;
    }
}

/* Compute (PAPER.md 44-49):
 *   w <- sqrt(L_ii^2 + sigma V_i^2); c <- w / L_ii; s <- V_i / L_ii; L_ii <- w
 * Returns 0 on success, 1 if the radicand is not > 0 (then w = NaN). */
int gcmo_compute(double *c, double *s, double *Lii, double Vi, int sigma) {
    double d = *Lii;
    double x = d * d + (double)sigma * (Vi * Vi);
    int bad = !(x > 0.0);
    double w = bad ? NAN : sqrt(x);
    *c = w / d;
    *s = Vi / d;
    *Lii = w;
    return bad;
}

/* Apply (PAPER.md 52-54):
 *   L_ij <- (L_ij + sigma s V_j) / c
 *   V_j  <- c V_j - s L_ij            (the L_ij just written) */
void gcmo_apply(double c, double s, double *Lij, double *Vj, int sigma) {
    double l = (*Lij + (double)sigma * s * (*Vj)) / c;
    *Lij = l;
    *Vj = c * (*Vj) - s * l;
}

#define LIJ(i, j) L[(size_t)(i) + (size_t)(j) * (size_t)ldl]
#define VIE(i, e) V[(size_t)(i) + (size_t)(e) * (size_t)n]

/* CholeskyModifyA, rank k (dependency-corrected, R1):
 *   for i = 0..n-1:                                  (column i, PAPER.md 25)
 *     for j = 0..i-1: for e = 0..k-1:                (PAPER.md 27-28)
 *        Apply(c[j][e], s[j][e], L_ji, V_ie)
 *     for e = 0..k-1: Compute(c[i][e], s[i][e], L_ii, V_ie)   (PAPER.md 26)
 * cs_c / cs_s: caller-provided n*k scratch (row-major [i][e]), also an output
 * so tests can pin the coefficient ranges. */
int gcmo_modify_a(double *L, int64_t n, int64_t ldl, double *V, int64_t k, int sigma,
                  double *cs_c, double *cs_s, gcmo_info_t *info) {
    if (info) { info->code = 0; info->col = 0; info->row = 0; }
    for (int64_t i = 0; i < n; ++i) {
        for (int64_t j = 0; j < i; ++j)
            for (int64_t e = 0; e < k; ++e)
                gcmo_apply(cs_c[j * k + e], cs_s[j * k + e], &LIJ(j, i), &VIE(i, e), sigma);
        if (!(LIJ(i, i) > 0.0)) {
            info_record(info, 2, 0, i);
            LIJ(i, i) = NAN;
        }
        for (int64_t e = 0; e < k; ++e) {
            if (gcmo_compute(&cs_c[i * k + e], &cs_s[i * k + e], &LIJ(i, i), VIE(i, e), sigma))
                info_record(info, 1, e, i);
        }
    }
    return info ? info->code : 0;
}

/* CholeskyModifyB, as k sequential rank-1 sweeps:
 *   for e = 0..k-1: for i = 0..n-1:
 *     Compute(c_i, s_i, L_ii, V_ie)                  (PAPER.md 36)
 *     for j = i+1..n-1: Apply(c_i, s_i, L_ij, V_je)  (PAPER.md 37-38)
 * V_ie on exit is the value Compute consumed (it is never written after). */
int gcmo_modify_b(double *L, int64_t n, int64_t ldl, double *V, int64_t k, int sigma,
                  double *cs_c, double *cs_s, gcmo_info_t *info) {
    if (info) { info->code = 0; info->col = 0; info->row = 0; }
    for (int64_t e = 0; e < k; ++e) {
        for (int64_t i = 0; i < n; ++i) {
            if (e == 0 && !(LIJ(i, i) > 0.0)) {
                info_record(info, 2, 0, i);
                LIJ(i, i) = NAN;
            }
            double c, s;
            if (gcmo_compute(&c, &s, &LIJ(i, i), VIE(i, e), sigma))
                info_record(info, 1, e, i);
            cs_c[i * k + e] = c;
            cs_s[i * k + e] = s;
            for (int64_t j = i + 1; j < n; ++j)
                gcmo_apply(c, s, &LIJ(i, j), &VIE(j, e), sigma);
        }
    }
    return info ? info->code : 0;
}

/* Single precision (the paper's Figs. 2-3 ran fp32 and fp64, PAPER.md 111): the same
 * CholeskyModifyA (PAPER.md 24-30 with the inner loop before Compute, R1), Compute
 * (44-49) and Apply (52-54) with every quantity a float.  Separate functions, written out,
 * so the fp64 oracle above stays exactly as pinned. */
static int compute_f32(float *c, float *s, float *Lii, float Vi, int sigma) {
    float d = *Lii;
    float x = d * d + (float)sigma * (Vi * Vi);
    int bad = !(x > 0.0f);
    float w = bad ? NAN : sqrtf(x);
    *c = w / d;
    *s = Vi / d;
    *Lii = w;
    return bad;
}
static void apply_f32(float c, float s, float *Lij, float *Vj, int sigma) {
    float l = (*Lij + (float)sigma * s * (*Vj)) / c;
    *Lij = l;
    *Vj = c * (*Vj) - s * l;
}
int gcmo_modify_a_f32(float *L, int64_t n, int64_t ldl, float *V, int64_t k, int sigma, float *cs_c, float *cs_s,
                      gcmo_info_t *info) {
    if (info) { info->code = 0; info->col = 0; info->row = 0; }
    for (int64_t i = 0; i < n; ++i) {
        for (int64_t j = 0; j < i; ++j)
            for (int64_t e = 0; e < k; ++e)
                apply_f32(cs_c[j * k + e], cs_s[j * k + e], &LIJ(j, i), &VIE(i, e), sigma);
        if (!(LIJ(i, i) > 0.0f)) {
            info_record(info, 2, 0, i);
            LIJ(i, i) = NAN;
        }
        for (int64_t e = 0; e < k; ++e) {
            if (compute_f32(&cs_c[i * k + e], &cs_s[i * k + e], &LIJ(i, i), VIE(i, e), sigma))
                info_record(info, 1, e, i);
        }
    }
    return info ? info->code : 0;
}

/* Textbook (left-looking, column-by-column) Cholesky of a symmetric positive
 * definite A, upper factor: A = L^T L.  Reads the upper triangle of A
 * (column-major, lda), writes the upper triangle of L (column-major, ldl).
 *   L_ij = (A_ij - sum_{m<i} L_mi L_mj) / L_ii      (i < j)
 *   L_jj = sqrt(A_jj - sum_{m<j} L_mj^2)
 * Returns 0, or 1 + the index of the first non-positive pivot. */
int64_t gcmo_chol_upper(const double *A, int64_t n, int64_t lda, double *L, int64_t ldl) {
    for (int64_t j = 0; j < n; ++j) {
        for (int64_t i = 0; i < j; ++i) {
            double acc = A[(size_t)i + (size_t)j * (size_t)lda];
            for (int64_t m = 0; m < i; ++m) acc -= LIJ(m, i) * LIJ(m, j);
            LIJ(i, j) = acc / LIJ(i, i);
        }
        double acc = A[(size_t)j + (size_t)j * (size_t)lda];
        for (int64_t m = 0; m < j; ++m) acc -= LIJ(m, j) * LIJ(m, j);
        if (!(acc > 0.0)) return 1 + j;
        LIJ(j, j) = sqrt(acc);
    }
    return 0;
}
