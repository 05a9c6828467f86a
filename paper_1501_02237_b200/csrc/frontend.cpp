// Host front end of libbdeg: Smith Normal Form, parametrisation matrix P_0,
// consistency, LLL reduction of P_0 and the lifted point configuration.
//
// PAPER.md §2-§3: P A Q = diag(d_1..d_r, 0) with P, Q unimodular (eq. smith,
// P:213-228); #components = |prod d_j| (Prop. 1); P_0 = last n-r rows
// of P, Q_0 = last m-r columns of Q (eq. rank-decomp); consistent
// iff b^{Q_0} = 1 (eq. consistency); deg V = NVol(conv(cols P_0 u 0))
// (Prop. 4).
//
// The diagonalisation uses Euclidean elimination (repeated integer-quotient
// row/column subtraction with a minimum-modulus pivot), the unimodular
// reduction of P:569-585; the divisibility chain is not needed.
// All arithmetic is checked __int128; overflow is reported, never wrapped.
#include "bdeg_internal.h"

#include <algorithm>
#include <cmath>
#include <complex>
#include <map>

namespace bdeg {

namespace {

struct Overflow {};

inline i128 cadd(i128 a, i128 b) {
    i128 r;
    if (__builtin_add_overflow(a, b, &r)) throw Overflow();
    return r;
}
inline i128 cmul(i128 a, i128 b) {
    i128 r;
    if (__builtin_mul_overflow(a, b, &r)) throw Overflow();
    return r;
}
inline i128 iabs(i128 a) { return a < 0 ? -a : a; }

// floor division for i128
inline i128 fdiv(i128 a, i128 b) {
    i128 q = a / b;
    if ((a % b != 0) && ((a < 0) != (b < 0))) q -= 1;
    return q;
}

typedef std::vector<std::vector<i128>> Mat;

// row_dst += f * row_src on matrix X (rows)
void row_axpy(Mat &X, int dst, int src, i128 f) {
    if (f == 0) return;
    for (size_t j = 0; j < X[dst].size(); ++j) X[dst][j] = cadd(X[dst][j], cmul(f, X[src][j]));
}
void col_axpy(Mat &X, int dst, int src, i128 f) {
    if (f == 0) return;
    for (size_t i = 0; i < X.size(); ++i) X[i][dst] = cadd(X[i][dst], cmul(f, X[i][src]));
}

// Diagonalise M (n x m) in place; P (n x n) and Q (m x m) accumulate the
// unimodular row / column operations so that P * A * Q = M.  Returns rank.
int smith_euclid(Mat &M, Mat &P, Mat &Q) {
    const int n = (int)M.size();
    const int m = n ? (int)M[0].size() : 0;
    int t = 0;
    for (; t < std::min(n, m); ++t) {
        for (;;) {
            // minimum-modulus non-zero entry of the trailing block
            int bi = -1, bj = -1;
            i128 best = 0;
            for (int i = t; i < n; ++i)
                for (int j = t; j < m; ++j)
                    if (M[i][j] != 0 && (bi < 0 || iabs(M[i][j]) < best)) { best = iabs(M[i][j]); bi = i; bj = j; }
            if (bi < 0) return t;
            if (bi != t) { std::swap(M[bi], M[t]); std::swap(P[bi], P[t]); }
            if (bj != t) {
                for (auto &row : M) std::swap(row[bj], row[t]);
                for (auto &row : Q) std::swap(row[bj], row[t]);
            }
            bool clean = true;
            const i128 piv = M[t][t];
            for (int i = t + 1; i < n; ++i) {
                if (M[i][t] == 0) continue;
                i128 q = fdiv(M[i][t], piv);
                row_axpy(M, i, t, -q);
                row_axpy(P, i, t, -q);
                if (M[i][t] != 0) clean = false;    // remainder smaller than |piv|
            }
            for (int j = t + 1; j < m; ++j) {
                if (M[t][j] == 0) continue;
                i128 q = fdiv(M[t][j], piv);
                col_axpy(M, j, t, -q);
                col_axpy(Q, j, t, -q);
                if (M[t][j] != 0) clean = false;
            }
            if (clean) break;   // row t and column t are zero off the pivot
        }
    }
    return t;
}

// LLL reduction (delta = 0.99) of the rows of B, with exact integer basis
// operations (the Gram-Schmidt data is long double and only steers the
// choice of unimodular steps, so the result spans the same lattice exactly).
void lll_rows(Mat &B) {
    const int d = (int)B.size();
    if (d <= 1) return;
    const int n = (int)B[0].size();
    typedef long double R;
    std::vector<std::vector<R>> bs(d, std::vector<R>(n)), mu(d, std::vector<R>(d, 0));
    std::vector<R> bb(d);
    auto gso = [&]() {
        for (int i = 0; i < d; ++i) {
            for (int t = 0; t < n; ++t) bs[i][t] = (R)B[i][t];
            for (int j = 0; j < i; ++j) {
                R dot = 0;
                for (int t = 0; t < n; ++t) dot += (R)B[i][t] * bs[j][t];
                mu[i][j] = bb[j] > 0 ? dot / bb[j] : 0;
                for (int t = 0; t < n; ++t) bs[i][t] -= mu[i][j] * bs[j][t];
            }
            bb[i] = 0;
            for (int t = 0; t < n; ++t) bb[i] += bs[i][t] * bs[i][t];
        }
    };
    gso();
    int k = 1, guard = 0;
    while (k < d && guard++ < 200000) {
        for (int j = k - 1; j >= 0; --j) {
            R q = std::nearbyint(mu[k][j]);
            if (q != 0) {
                row_axpy(B, k, j, -(i128)q);
                gso();
            }
        }
        if (bb[k] >= (0.99L - mu[k][k - 1] * mu[k][k - 1]) * bb[k - 1]) {
            ++k;
        } else {
            std::swap(B[k], B[k - 1]);
            gso();
            k = std::max(k - 1, 1);
        }
    }
}

}  // namespace

uint64_t derive_seed(uint64_t seed, int attempt) {
    if (attempt == 0) return seed;
    SplitMix64 g(seed ^ ((uint64_t)attempt * 0x9E3779B97F4A7C15ull));
    return g.next();
}

bool smith_factors(int n, int m, const int64_t *A, int &rank, u128 &prod, std::string &err) {
    try {
        Mat M(n, std::vector<i128>(m)), P(n, std::vector<i128>(n, 0)), Q(m, std::vector<i128>(m, 0));
        for (int i = 0; i < n; ++i) {
            P[i][i] = 1;
            for (int j = 0; j < m; ++j) M[i][j] = A[(size_t)i * m + j];
        }
        for (int j = 0; j < m; ++j) Q[j][j] = 1;
        rank = smith_euclid(M, P, Q);
        prod = 1;
        for (int t = 0; t < rank; ++t) {
            const i128 d = iabs(M[t][t]);
            if (d != 0 && prod > (((u128)1 << 127) / (u128)d)) { err = "component count beyond 2^127"; return false; }
            prod *= (u128)d;
        }
    } catch (const Overflow &) {
        err = "Smith form of the residual: __int128 overflow";
        return false;
    }
    return true;
}

bool analyze_system(int n, int m, const int64_t *A, const double *b_re, const double *b_im,
                    bool lll, FrontEnd &fe, std::string &err) {
    fe = FrontEnd();
    fe.n = n;
    fe.m = m;
    try {
        Mat M(n, std::vector<i128>(m)), P(n, std::vector<i128>(n, 0)), Q(m, std::vector<i128>(m, 0));
        for (int i = 0; i < n; ++i) {
            P[i][i] = 1;
            for (int j = 0; j < m; ++j) M[i][j] = A[(size_t)i * m + j];
        }
        for (int j = 0; j < m; ++j) Q[j][j] = 1;
        const int r = smith_euclid(M, P, Q);
        fe.rank = r;
        fe.dim = n - r;
        u128 comps = 1;
        for (int j = 0; j < r; ++j) {
            u128 a = (u128)iabs(M[j][j]);
            if (a != 0 && comps > (~(u128)0) / a) throw Overflow();
            comps *= a;
        }
        fe.components = comps;
        // consistency b^{Q_0} = 1 for each of the m - r columns of Q_0
        fe.consistent = true;
        for (int k = r; k < m; ++k) {
            std::complex<long double> acc(1.0L, 0.0L);
            for (int i = 0; i < m; ++i) {
                i128 e = Q[i][k];
                if (e == 0) continue;
                std::complex<long double> bi(b_re ? b_re[i] : 1.0, b_im ? b_im[i] : 0.0);
                if (e < 0) { bi = 1.0L / bi; e = -e; }
                std::complex<long double> pw(1.0L, 0.0L);
                while (e) {                   // exact-exponent repeated squaring
                    if (e & 1) pw *= bi;
                    bi *= bi;
                    e >>= 1;
                }
                acc *= pw;
            }
            long double dev = std::abs(acc - std::complex<long double>(1.0L, 0.0L));
            if (dev > 1e-8L * std::max((long double)1.0L, std::abs(acc))) fe.consistent = false;
        }
        fe.P0.assign(P.begin() + r, P.end());
        if (lll) lll_rows(fe.P0);
        bool homog = true;
        for (int j = 0; j < m && homog; ++j) {
            int64_t s = 0;
            for (int i = 0; i < n; ++i) s += A[(size_t)i * m + j];
            if (s != 0) homog = false;
        }
        fe.homogeneous = homog;
    } catch (Overflow &) {
        err = "integer overflow in the Smith normal form (entries beyond 127 bits)";
        return false;
    }
    return true;
}

void build_points(const FrontEnd &fe, const int64_t *lifting, bool homog_shortcut,
                  int &K, int &N, std::vector<int64_t> &V, std::vector<int64_t> &w,
                  std::vector<int> &point_of_var, int &origin_index) {
    const int d = fe.dim, n = fe.n;
    std::map<std::vector<i128>, int> index;
    std::vector<std::vector<i128>> pts;
    std::vector<int64_t> lifts;
    point_of_var.assign(n, -1);
    int64_t origin_lift = lifting[n];
    std::vector<int> zero_vars;
    for (int j = 0; j < n; ++j) {
        std::vector<i128> c(d);
        bool zero = true;
        for (int i = 0; i < d; ++i) {
            c[i] = fe.P0[i][j];
            if (c[i] != 0) zero = false;
        }
        if (zero) {
            origin_lift = std::min(origin_lift, lifting[j]);
            zero_vars.push_back(j);
            continue;
        }
        auto it = index.find(c);
        if (it == index.end()) {
            index[c] = (int)pts.size();
            point_of_var[j] = (int)pts.size();
            pts.push_back(c);
            lifts.push_back(lifting[j]);
        } else {
            point_of_var[j] = it->second;
            lifts[it->second] = std::min(lifts[it->second], lifting[j]);
        }
    }
    const bool homog = fe.homogeneous && homog_shortcut;
    V.clear();
    w.clear();
    if (homog) {
        K = d;
        N = (int)pts.size();
        for (int l = 0; l < N; ++l) {
            for (int i = 0; i < d; ++i) V.push_back((int64_t)pts[l][i]);
            w.push_back(lifts[l]);
        }
        origin_index = -1;
    } else {
        K = d + 1;
        N = (int)pts.size() + 1;
        for (int l = 0; l < N - 1; ++l) {
            V.push_back(1);
            for (int i = 0; i < d; ++i) V.push_back((int64_t)pts[l][i]);
            w.push_back(lifts[l]);
        }
        V.push_back(1);
        for (int i = 0; i < d; ++i) V.push_back(0);
        w.push_back(origin_lift);
        origin_index = N - 1;
        for (int j : zero_vars) point_of_var[j] = origin_index;
    }
}

}  // namespace bdeg
