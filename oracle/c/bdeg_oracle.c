/* CPU ORACLE (C variant) — test infrastructure only.
 *
 * Same brute force as oracle/subdivision.py, for sizes
 * the Fraction version cannot reach in seconds.  Linked only by
 * oracle/native.py; never by the product library.  Shares no code with
 * paper_1501_02237_b200/csrc.
 *
 * Input: K-vectors v_0..v_{N-1} (point-major, int64) and lifts w_l
 * (homogeneous coordinates; for the generic case v = (1, a), see
 * oracle/points.py).  For every K-subset sigma (colex rank order, rank =
 * sum_i C(c_i, i+1)) in [rank_begin, rank_end):
 *   D      = det V_sigma                        (Z1 reading of P:690-695)
 *   h~_t   = det(M with column t replaced by w_sigma), M rows = v_c
 *            (Cramer's rule: h~ = D h, h . v_c = w_c for c in sigma)
 *   delta~_l = D w_l - h~ . v_l = D (w_l - h . v_l)
 *   sigma is a lower facet (a cell) iff sign(delta~_l) = sign(D) for every
 *   other l (strict, reading Z3); no wrong sign but some zero = tie.
 * Determinants by textbook fraction-free (Bareiss) elimination in __int128
 * with every product and sum overflow-checked; an overflow sets status 1.
 */
#include <stdint.h>
#include <string.h>

#define MAXK 33
#define MAXN 128

typedef __int128 i128;

static __thread int g_overflow;   /* per calling thread */

static i128 cmul(i128 a, i128 b) {
    i128 r;
    if (__builtin_mul_overflow(a, b, &r)) { g_overflow = 1; return 0; }
    return r;
}
static i128 csub(i128 a, i128 b) {
    i128 r;
    if (__builtin_sub_overflow(a, b, &r)) { g_overflow = 1; return 0; }
    return r;
}

/* det of the n x n matrix a (destroyed), Bareiss with row pivoting */
static i128 det_bareiss(int n, i128 a[MAXK][MAXK]) {
    i128 prev = 1;
    int sign = 1;
    for (int k = 0; k < n - 1; k++) {
        if (a[k][k] == 0) {
            int p = -1;
            for (int i = k + 1; i < n; i++) if (a[i][k] != 0) { p = i; break; }
            if (p < 0) return 0;
            for (int j = 0; j < n; j++) { i128 t = a[k][j]; a[k][j] = a[p][j]; a[p][j] = t; }
            sign = -sign;
        }
        for (int i = k + 1; i < n; i++) {
            for (int j = k + 1; j < n; j++) {
                i128 num = csub(cmul(a[k][k], a[i][j]), cmul(a[i][k], a[k][j]));
                a[i][j] = num / prev;      /* exact (Bareiss) */
            }
        }
        prev = a[k][k];
    }
    return sign > 0 ? a[n - 1][n - 1] : -a[n - 1][n - 1];
}

static uint64_t binom_u64(int n, int k) {
    if (k < 0 || k > n) return 0;
    if (k > n - k) k = n - k;
    unsigned __int128 r = 1;
    for (int i = 1; i <= k; i++) r = r * (unsigned)(n - k + i) / (unsigned)i;
    return (uint64_t)r;
}

/* colex unrank: largest c with C(c, i+1) <= r, from the top element down */
static void unrank(uint64_t r, int K, int *c) {
    for (int i = K - 1; i >= 0; i--) {
        int x = i;
        while (binom_u64(x + 1, i + 1) <= r) x++;
        c[i] = x;
        r -= binom_u64(x, i + 1);
    }
}

static int next_comb(int *c, int K, int N) {
    for (int i = 0; i < K; i++) {
        int limit = (i + 1 < K) ? c[i + 1] : N;
        if (c[i] + 1 < limit) {
            c[i]++;
            for (int t = 0; t < i; t++) c[t] = t;
            return 1;
        }
    }
    return 0;
}

/* out[0..6]: volume lo 64 bits, volume hi 64 bits, cells, singular,
 * candidates, ties, status (0 ok, 1 overflow, 2 bad args) */
int bdeg_oracle_enumerate(int K, int N, const int64_t *V, const int64_t *w,
                          uint64_t rank_begin, uint64_t rank_end, int64_t *out) {
    memset(out, 0, 7 * sizeof(int64_t));
    if (K < 1 || K > MAXK - 1 || N < K || N > MAXN) { out[6] = 2; return 2; }
    uint64_t total = binom_u64(N, K);
    if (rank_end > total) rank_end = total;
    if (rank_begin >= rank_end) return 0;
    g_overflow = 0;
    int c[MAXK];
    unrank(rank_begin, K, c);
    unsigned __int128 vol = 0;
    uint64_t cells = 0, singular = 0, cand = 0, ties = 0;
    i128 M[MAXK][MAXK], h[MAXK];
    for (uint64_t r = rank_begin; r < rank_end; r++) {
        cand++;
        for (int i = 0; i < K; i++)
            for (int t = 0; t < K; t++) M[i][t] = V[(int64_t)c[i] * K + t];
        i128 D = det_bareiss(K, M);
        if (D == 0) {
            singular++;
        } else {
            for (int t = 0; t < K; t++) {          /* Cramer: h~_t */
                for (int i = 0; i < K; i++)
                    for (int u = 0; u < K; u++)
                        M[i][u] = (u == t) ? (i128)w[c[i]] : (i128)V[(int64_t)c[i] * K + u];
                h[t] = det_bareiss(K, M);
            }
            int bad = 0, zero = 0, ci = 0;
            for (int l = 0; l < N && !bad; l++) {
                if (ci < K && c[ci] == l) { ci++; continue; }
                i128 s = cmul(D, (i128)w[l]);
                for (int t = 0; t < K; t++) s = csub(s, cmul(h[t], (i128)V[(int64_t)l * K + t]));
                if (s == 0) zero = 1;
                else if ((s > 0) != (D > 0)) bad = 1;
            }
            if (!bad) {
                if (zero) ties++;
                else { cells++; vol += (unsigned __int128)(D > 0 ? D : -D); }
            }
        }
        if (g_overflow) { out[6] = 1; return 1; }
        if (r + 1 < rank_end) next_comb(c, K, N);
    }
    out[0] = (int64_t)(uint64_t)vol;
    out[1] = (int64_t)(uint64_t)(vol >> 64);
    out[2] = (int64_t)cells;
    out[3] = (int64_t)singular;
    out[4] = (int64_t)cand;
    out[5] = (int64_t)ties;
    return 0;
}
