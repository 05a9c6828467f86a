// libbdeg device code (sm_100a): rank-space enumeration of the K-subsets of
// a lifted point configuration with exact fraction-free elimination, the
// warp-cooperative lower-facet test and the exact volume reduction.
//
// What is computed (§4): every K-subset sigma (colex rank order) is
// a candidate simplex; D = det V_sigma is its normalised volume (eq.
// simplex-vol, reading Z1); sigma is a cell of the regular
// subdivision iff the lower-face system I(sigma) (eq. lower-face,
// P:782-792) holds strictly, i.e. sign det[[V_sig, v_l],[w_sig, w_l]] =
// sign D for every other point l; the degree is sum |D| over cells
// (Prop. 4).
//
// How (DESIGN.md §"Kernel"): one warp owns one *block* = all candidates
// sharing their top T = K-1-S indices (c_{S+1} < ... < c_{K-1}); lanes own
// points (point l in lane l%32, slot l/32).  The block prefix is eliminated
// once (Bareiss, fraction-free, Sylvester's identity) in per-warp shared
// scratch; the remaining S prefix indices are walked depth-first with the
// elimination state in registers.  After the full (K-1)-prefix P has been
// eliminated, every point l reduces to a 2-vector (x_l, y_l) with
// x_l = +-det V_{P u l} and y_l its lift minor, and for sigma = P u {j}:
//     cell  <=>  kappa * x_j * (x_j y_l - x_l y_j) > 0   for all l not in sigma
// (kappa = sign of the last pivot).  So the <= 2 cells per prefix are the
// unique extreme slopes y/x of the two half-planes x>0 / x<0; they are found
// with one REDUX per half-plane on monotone float keys and then verified
// exactly against every lane (ballot/any).
#include "bdeg_internal.h"

#include <cuda_runtime.h>
#include <atomic>

namespace bdeg {

static std::atomic<uint64_t> g_launches{0};
uint64_t launch_counter_add(uint64_t k) { return g_launches.fetch_add(k) + k; }

namespace dev {

constexpr unsigned FULL = 0xffffffffu;
constexpr int kWarps = 8;           // warps per CTA

template <int TIER> struct VT;
template <> struct VT<0> { typedef int32_t T; };
template <> struct VT<1> { typedef int64_t T; };

// Exact division by a known divisor d != 0: shift out the 2-adic part, then
// multiply by the inverse of the odd part mod 2^64.  Exact whenever the
// dividend is a multiple of d and the quotient fits (Bareiss guarantees the
// former; the callers check the latter).
struct Div {
    uint64_t inv;
    int64_t d;
    int tz;
    int unit;   // +1: d == 1, -1: d == -1, 0: general
};

__device__ __forceinline__ Div make_div(int64_t d) {
    Div r;
    r.d = d;
    r.unit = (d == 1) ? 1 : (d == -1 ? -1 : 0);
    r.tz = __ffsll(d) - 1;
    const uint64_t o = (uint64_t)(d >> r.tz);
    uint64_t x = o;                        // correct to 3 bits
#pragma unroll
    for (int i = 0; i < 5; ++i) x *= 2 - o * x;   // Newton: 6, 12, 24, 48, 96 bits
    r.inv = x;
    return r;
}

// tier 0: |values| < 2^31, numerators exact in int64
__device__ __forceinline__ int64_t qdiv64(int64_t num, const Div &dv) {
    if (dv.unit == 1) return num;
    if (dv.unit == -1) return -num;
    return (int64_t)((uint64_t)(num >> dv.tz) * dv.inv);
}
__device__ __forceinline__ bool fits31(int64_t v) {  // |v| <= 2^31 - 1
    return (uint64_t)(v + 0x7FFFFFFFll) <= 0xFFFFFFFEull;
}
// tier 1: |values| < 2^62, numerators exact in int128; the quotient is
// verified by multiplying back (detects any value beyond the int64 tier).
__device__ __forceinline__ int64_t qdiv128(i128 num, const Div &dv, bool &ovf) {
    int64_t q;
    if (dv.unit != 0) {
        const i128 t = dv.unit > 0 ? num : -num;
        q = (int64_t)t;
        ovf |= ((i128)q != t);
    } else {
        q = (int64_t)((uint64_t)(num >> dv.tz) * dv.inv);
        ovf |= ((i128)q * (i128)dv.d != num);
    }
    const int64_t lim = (int64_t)1 << 62;
    ovf |= (q >= lim) || (q <= -lim);
    return q;
}

template <typename T>
__device__ __forceinline__ T shfl(T v, int src) {
    return __shfl_sync(FULL, v, src);
}
template <>
__device__ __forceinline__ int64_t shfl<int64_t>(int64_t v, int src) {
    return (int64_t)__shfl_sync(FULL, (long long)v, src);
}

// order-preserving map float -> uint32 (finite values)
__device__ __forceinline__ uint32_t ford(float f) {
    uint32_t b = __float_as_uint(f);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

struct Acc {
    uint64_t vol_lo, vol_hi, cells, singular, cand, ties, updates, leaves;
    __device__ void zero() { vol_lo = vol_hi = cells = singular = cand = ties = updates = leaves = 0; }
    __device__ void add_vol(uint64_t v) {
        uint64_t t = vol_lo + v;
        vol_hi += (t < vol_lo);
        vol_lo = t;
    }
    __device__ void add(const Acc &o) {
        add_vol(o.vol_lo);
        vol_hi += o.vol_hi;
        cells += o.cells; singular += o.singular; cand += o.cand; ties += o.ties;
        updates += o.updates; leaves += o.leaves;
    }
};

struct Ctx {
    const uint64_t *B;   // binomial table in smem
    int N, K, lane;
    uint64_t rb, re;
    bool partial;
    __device__ __forceinline__ uint64_t C(int n, int k) const { return B[n * kBinomCols + k]; }
    // |[base, base+size) n [rb, re)|
    __device__ __forceinline__ uint64_t isect(uint64_t base, uint64_t size) const {
        if (!partial) return size;
        uint64_t lo = base > rb ? base : rb;
        uint64_t hi = base + size < re ? base + size : re;
        return hi > lo ? hi - lo : 0;
    }
};

// ------------------------------------------------------------------ leaf
// x, y: leaf 2-vectors of this lane's points; c1 = smallest prefix index;
// base = rank of candidate (j = 0, P); inP = prefix point mask; kappa = sign
// of the last pivot.  Counts the candidates P u {j}, j in [0, c1) n range.
template <int NPL>
__device__ __forceinline__ void leaf_test(const int64_t (&x)[NPL], const int64_t (&y)[NPL], int c1,
                                          uint64_t base, uint64_t inP, int kappa, const Ctx &cx, Acc &acc) {
    int jlo = 0, jhi = c1;
    if (cx.partial) {
        if (cx.rb > base) jlo = (cx.rb - base >= (uint64_t)c1) ? c1 : (int)(cx.rb - base);
        if (cx.re < base + (uint64_t)c1) jhi = (cx.re <= base) ? 0 : (int)(cx.re - base);
        if (jlo >= jhi) return;
    }
    acc.cand += (uint64_t)(jhi - jlo);
    acc.leaves += 1;
    int64_t yk[NPL];
    bool valid[NPL], cnt[NPL];
    bool bad0 = false, small = true, wide = false;
    unsigned sing = 0;
#pragma unroll
    for (int q = 0; q < NPL; ++q) {
        const int l = cx.lane + 32 * q;
        valid[q] = (l < cx.N) && !((inP >> l) & 1ull);
        cnt[q] = (l >= jlo) && (l < jhi);
        yk[q] = kappa > 0 ? y[q] : -y[q];
        sing += __popc(__ballot_sync(FULL, cnt[q] && x[q] == 0));
        bad0 |= valid[q] && x[q] == 0 && yk[q] < 0;
        const uint64_t ax = (uint64_t)(x[q] < 0 ? -x[q] : x[q]);
        const uint64_t ay = (uint64_t)(yk[q] < 0 ? -yk[q] : yk[q]);
        if (valid[q]) {
            small &= (ax < (1ull << 24)) && (ay < (1ull << 24));
            wide |= (ax >= (1ull << 53)) || (ay >= (1ull << 53));
        }
    }
    acc.singular += sing;
    if (__any_sync(FULL, bad0)) return;          // a point in span(P) strictly below
    uint64_t candmask = 0;
    const bool anywide = __any_sync(FULL, wide);
    if (!anywide) {
        const bool allsmall = __all_sync(FULL, small);
        uint32_t kp[NPL], km[NPL];
        uint32_t mp = 0xFFFFFFFFu, mm = 0xFFFFFFFFu;
#pragma unroll
        for (int q = 0; q < NPL; ++q) {
            kp[q] = km[q] = 0xFFFFFFFFu;
            if (valid[q] && x[q] != 0) {
                // slope y'/x, correctly rounded => monotone in the exact rational
                float f = allsmall ? __fdiv_rn((float)yk[q], (float)x[q])
                                   : __double2float_rn(__ddiv_rn((double)yk[q], (double)x[q]));
                const uint32_t o = ford(f);
                if (x[q] > 0) kp[q] = o; else km[q] = ~o;
            }
            mp = min(mp, kp[q]);
            mm = min(mm, km[q]);
        }
        mp = __reduce_min_sync(FULL, mp);        // min slope over x > 0
        mm = __reduce_min_sync(FULL, mm);        // max slope over x < 0 (complemented)
        // both cells need  max_{x<0} slope < min_{x>0} slope ; float '>' is exact '>'
        if (mp != 0xFFFFFFFFu && mm != 0xFFFFFFFFu && (~mm) > mp) return;
#pragma unroll
        for (int q = 0; q < NPL; ++q) {
            const bool c = cnt[q] && ((kp[q] == mp && mp != 0xFFFFFFFFu) || (km[q] == mm && mm != 0xFFFFFFFFu));
            candmask |= (uint64_t)__ballot_sync(FULL, c) << (32 * q);
        }
    } else {
        // values beyond 2^53: no float keys, verify every countable j exactly
#pragma unroll
        for (int q = 0; q < NPL; ++q)
            candmask |= (uint64_t)__ballot_sync(FULL, cnt[q] && x[q] != 0) << (32 * q);
    }
    while (candmask) {
        const int j = __ffsll((long long)candmask) - 1;
        candmask &= candmask - 1;
        const int js = j >> 5, jl = j & 31;
        int64_t xs = x[0], ys = yk[0];
        if (NPL > 1 && js == 1) { xs = x[NPL - 1]; ys = yk[NPL - 1]; }
        const int64_t xj = shfl<int64_t>(xs, jl);
        const int64_t yj = shfl<int64_t>(ys, jl);
        bool bad = false, zero = false;
#pragma unroll
        for (int q = 0; q < NPL; ++q) {
            const int l = cx.lane + 32 * q;
            if (valid[q] && l != j) {
                i128 c = (i128)xj * yk[q] - (i128)x[q] * yj;
                if (xj < 0) c = -c;
                bad |= c < 0;
                zero |= c == 0;
            }
        }
        if (__any_sync(FULL, bad)) continue;
        if (__any_sync(FULL, zero)) {
            acc.ties += 1;                         // would-be cell on a tie (reading Z3)
        } else {
            acc.cells += 1;
            acc.add_vol((uint64_t)(xj < 0 ? -xj : xj));   // |x_j| = |det V_sigma|
        }
    }
}

// --------------------------------------------------------- one elimination step
// st: R rows (R-1 V rows, then the lift row) of this lane's points.  Pivot
// column values colv (uniform), pivot row pr, pivot value piv, previous
// pivot divisor dv.  Output: R-1 rows (other V rows in order, lift row last):
//     a'_{o,l} = (piv * a_{o,l} - a_{o,p} * a_{pr,l}) / prev      (Bareiss)
template <int TIER, int NPL, int R, typename OT>
__device__ __forceinline__ void elim_step(const typename VT<TIER>::T (&st)[NPL][R],
                                          const typename VT<TIER>::T (&colv)[R], int pr,
                                          typename VT<TIER>::T piv, const Div &dv,
                                          OT (&out)[NPL][R - 1], bool &ovf) {
    typedef typename VT<TIER>::T V;
#pragma unroll
    for (int q = 0; q < NPL; ++q) {
        V prow = st[q][0];
#pragma unroll
        for (int r = 1; r < R - 1; ++r) if (pr == r) prow = st[q][r];
#pragma unroll
        for (int o = 0; o < R - 1; ++o) {
            V s, cs;
            if (o == R - 2) { s = st[q][R - 1]; cs = colv[R - 1]; }
            else { s = (o < pr) ? st[q][o] : st[q][o + 1]; cs = (o < pr) ? colv[o] : colv[o + 1]; }
            if constexpr (TIER == 0) {
                const int64_t num = (int64_t)piv * (int64_t)s - (int64_t)cs * (int64_t)prow;
                const int64_t v = qdiv64(num, dv);
                if constexpr (sizeof(OT) == 4) ovf |= !fits31(v);
                out[q][o] = (OT)v;
            } else {
                const i128 num = (i128)piv * (i128)s - (i128)cs * (i128)prow;
                out[q][o] = (OT)qdiv128(num, dv, ovf);
            }
        }
    }
}

template <int TIER, int NPL, int R>
__device__ __forceinline__ void fetch_col(const typename VT<TIER>::T (&st)[NPL][R], int c,
                                          typename VT<TIER>::T (&colv)[R]) {
    typedef typename VT<TIER>::T V;
    const int src = c & 31;
    const bool hi = (c >> 5) != 0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        V mine = st[0][r];
        if (NPL > 1 && hi) mine = st[NPL - 1][r];
        colv[r] = shfl<V>(mine, src);
    }
}

// ------------------------------------------------------------ inner DFS
// State with R >= 3 rows (R-1 remaining V rows + lift).  Chooses c_i,
// i = R-2, in [i, cbound) in colex order; base = rank contribution of the
// indices above; prev = previous pivot.
template <int TIER, int NPL, int R>
__device__ __forceinline__ void inner_dfs(const typename VT<TIER>::T (&st)[NPL][R], int cbound,
                                          uint64_t base, uint64_t inP, int64_t prev, const Ctx &cx,
                                          Acc &acc, bool &ovf) {
    typedef typename VT<TIER>::T V;
    constexpr int i = R - 2;
    const Div dv = make_div(prev);
    for (int c = i; c < cbound; ++c) {
        const uint64_t nb = base + cx.C(c, i + 1);
        const uint64_t ns = cx.C(c, i);
        if (cx.partial && cx.isect(nb, ns) == 0) continue;
        V colv[R];
        fetch_col<TIER, NPL, R>(st, c, colv);
        int pr = -1;
#pragma unroll
        for (int r = R - 2; r >= 0; --r) if (colv[r] != 0) pr = r;
        if (pr < 0) {                        // prefix dependent: whole subtree singular
            const uint64_t k = cx.isect(nb, ns);
            acc.singular += k;
            acc.cand += k;
            continue;
        }
        V piv = colv[0];
#pragma unroll
        for (int r = 1; r < R - 1; ++r) if (pr == r) piv = colv[r];
        acc.updates += (uint64_t)(R - 1) * cx.N;
        if constexpr (R == 3) {
            int64_t out[NPL][2];
            elim_step<TIER, NPL, R, int64_t>(st, colv, pr, piv, dv, out, ovf);
            if constexpr (TIER == 1) {
                if (__any_sync(FULL, ovf)) { ovf = true; return; }
            }
            int64_t xx[NPL], yy[NPL];
#pragma unroll
            for (int q = 0; q < NPL; ++q) { xx[q] = out[q][0]; yy[q] = out[q][1]; }
            leaf_test<NPL>(xx, yy, c, nb, inP | (1ull << c), piv > 0 ? 1 : -1, cx, acc);
        } else {
            V out[NPL][R - 1];
            elim_step<TIER, NPL, R, V>(st, colv, pr, piv, dv, out, ovf);
            if (__any_sync(FULL, ovf)) { ovf = true; return; }
            inner_dfs<TIER, NPL, R - 1>(out, c, nb, inP | (1ull << c), (int64_t)piv, cx, acc, ovf);
            if (ovf) return;
        }
    }
}

// ------------------------------------------------------------ one block
// Block id -> top tuple (colex over T-subsets of {0..N-S-2}, shifted by S+1),
// prefix elimination in shared scratch, then the register DFS.
template <int TIER, int NPL, int S>
__device__ void process_block(uint64_t blk, const int64_t *Lsm, int64_t *scr, const Ctx &cx0,
                              int T, Acc &acc, bool &ovf) {
    typedef typename VT<TIER>::T V;
    const int lane = cx0.lane;
    const int K = cx0.K, N = cx0.N;
    constexpr int NP = 32 * NPL;
    // --- unrank the top tuple: lane t (< T) holds c_{S+1+t}
    int mytop = 0;
    {
        uint64_t r = blk;
        for (int t = T - 1; t >= 0; --t) {
            // largest u with C(u, t+1) <= r  (u < N-S-1)
            uint32_t m0 = __ballot_sync(FULL, lane < N - S - 1 && cx0.C(lane, t + 1) <= r);
            uint32_t m1 = __ballot_sync(FULL, lane + 32 < N - S - 1 && cx0.C(lane + 32, t + 1) <= r);
            const int u = m1 ? 32 + 31 - __clz(m1) : 31 - __clz(m0);
            r -= cx0.C(u, t + 1);
            if (lane == t) mytop = u + S + 1;
        }
    }
    // rank base and size of the block
    uint64_t term = (lane < T) ? cx0.C(mytop, S + 2 + lane) : 0;
#pragma unroll
    for (int o = 16; o; o >>= 1) term += __shfl_xor_sync(FULL, term, o);
    const uint64_t bbase = term;
    const int ctop = T > 0 ? __shfl_sync(FULL, mytop, 0) : N;
    const uint64_t bsize = cx0.C(ctop, S + 1);
    Ctx cx = cx0;
    {
        const uint64_t lo = bbase > cx0.rb ? bbase : cx0.rb;
        const uint64_t hi = bbase + bsize < cx0.re ? bbase + bsize : cx0.re;
        if (hi <= lo) return;
        cx.partial = (lo != bbase) || (hi != bbase + bsize);
    }
    uint64_t inP = 0;
    {
        const uint64_t bit = (lane < T) ? (1ull << mytop) : 0ull;
        const unsigned lo = __reduce_or_sync(FULL, (unsigned)bit);
        const unsigned hi = __reduce_or_sync(FULL, (unsigned)(bit >> 32));
        inP = ((uint64_t)hi << 32) | lo;
    }
    // --- prefix elimination in shared scratch: scr[i*NP + l], rows 0..K
    __syncwarp();
    for (int i = 0; i <= K; ++i)
#pragma unroll
        for (int q = 0; q < NPL; ++q) {
            const int l = lane + 32 * q;
            scr[i * NP + l] = (l < N) ? Lsm[l * (K + 1) + i] : 0;
        }
    __syncwarp();
    uint64_t alive = (K >= 64) ? ~0ull : ((1ull << K) - 1);
    int64_t prev = 1;
    for (int t = 0; t < T; ++t) {
        const int p = __shfl_sync(FULL, mytop, T - 1 - t);   // pivot order c_{K-1}, c_{K-2}, ...
        const bool nz = (lane < K) && ((alive >> lane) & 1ull) && scr[lane * NP + p] != 0;
        const unsigned bal = __ballot_sync(FULL, nz);
        if (bal == 0) {                                       // dependent block prefix
            const uint64_t k = cx.isect(bbase, bsize);
            acc.singular += k;
            acc.cand += k;
            return;
        }
        const int r = __ffs(bal) - 1;
        const int64_t piv = scr[r * NP + p];
        const Div dv = make_div(prev);
        bool o = false;
        for (int i = 0; i <= K; ++i) {
            if (i == r || (i < K && !((alive >> i) & 1ull))) continue;
            const int64_t ci = scr[i * NP + p];
#pragma unroll
            for (int q = 0; q < NPL; ++q) {
                const int l = lane + 32 * q;
                if (l == p) continue;
                const i128 num = (i128)piv * scr[i * NP + l] - (i128)ci * scr[r * NP + l];
                const int64_t v = qdiv128(num, dv, o);
                scr[i * NP + l] = v;
            }
        }
        acc.updates += (uint64_t)(K - t) * N;
        if (__any_sync(FULL, o)) { ovf = true; return; }     // beyond the int64 tier
        alive &= ~(1ull << r);
        prev = piv;
        __syncwarp();
    }
    // --- registers: remaining S+1 V rows (ascending) then the lift row
    V st[NPL][S + 2];
    bool o = false;
    {
        int k = 0;
        for (int i = 0; i < K; ++i) {
            if (!((alive >> i) & 1ull)) continue;
#pragma unroll
            for (int kk = 0; kk < S + 1; ++kk)
                if (kk == k)
#pragma unroll
                    for (int q = 0; q < NPL; ++q) {
                        const int64_t v = scr[i * NP + lane + 32 * q];
                        if (TIER == 0) o |= !fits31(v);
                        st[q][kk] = (V)v;
                    }
            ++k;
        }
#pragma unroll
        for (int q = 0; q < NPL; ++q) {
            const int64_t v = scr[K * NP + lane + 32 * q];
            if (TIER == 0) o |= !fits31(v);
            st[q][S + 1] = (V)v;
        }
    }
    if (__any_sync(FULL, o)) { ovf = true; return; }
    if constexpr (S == 0) {
        // the block is a single leaf: prefix = the top tuple, c1 = ctop
        int64_t xx[NPL], yy[NPL];
#pragma unroll
        for (int q = 0; q < NPL; ++q) { xx[q] = (int64_t)st[q][0]; yy[q] = (int64_t)st[q][S + 1]; }
        leaf_test<NPL>(xx, yy, ctop, bbase, inP, prev > 0 ? 1 : -1, cx, acc);
    } else {
        inner_dfs<TIER, NPL, S + 2>(st, ctop, bbase, inP, prev, cx, acc, ovf);
    }
}

// ------------------------------------------------------------ TMA staging
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

template <int TIER, int NPL, int S>
__global__ void __launch_bounds__(kWarps * 32)
k_enumerate(LaunchArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int K = a.P.K, N = a.P.N, T = a.P.T;
    const uint32_t lbytes = (uint32_t)(((K + 1) * N * 8 + 15) & ~15);
    const uint32_t bbytes = kBinomRows * kBinomCols * 8;
    int64_t *Lsm = reinterpret_cast<int64_t *>(smem);
    uint64_t *Bsm = reinterpret_cast<uint64_t *>(smem + lbytes);
    unsigned long long *red = reinterpret_cast<unsigned long long *>(smem + lbytes + bbytes);
    uint64_t *mbar = reinterpret_cast<uint64_t *>(smem + lbytes + bbytes + kWarps * 16 * 8);
    int64_t *scr_all = reinterpret_cast<int64_t *>(smem + lbytes + bbytes + kWarps * 16 * 8 + 16);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    // stage the lifted matrix and the binomial table once per CTA (TMA bulk copy)
    if (threadIdx.x == 0) {
        const uint32_t mb = smem_u32(mbar);
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(lbytes + bbytes)
                     : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(Lsm)),
            "l"(a.P.L), "r"(lbytes), "r"(mb)
            : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(Bsm)),
            "l"(a.P.binom), "r"(bbytes), "r"(mb)
            : "memory");
    }
    __syncthreads();
    {
        const uint32_t mb = smem_u32(mbar);
        uint32_t done = 0;
        while (!done) {
            asm volatile(
                "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                : "=r"(done)
                : "r"(mb)
                : "memory");
        }
    }

    Ctx cx;
    cx.B = Bsm;
    cx.N = N;
    cx.K = K;
    cx.lane = lane;
    cx.rb = a.rank_begin;
    cx.re = a.rank_end;
    cx.partial = true;
    int64_t *scr = scr_all + (size_t)warp * (K + 1) * 32 * NPL;

    Acc wacc;
    wacc.zero();
    unsigned long long n_ovf = 0, n_fatal = 0, n_qfull = 0, n_blocks = 0;
    const uint64_t span = a.blk_last - a.blk_first + 1;
    const uint64_t nwork = a.replay ? (uint64_t)min((unsigned long long)a.ovf_cap, *a.ovf_count)
                                    : (span > a.blk_offset ? (span - a.blk_offset + a.blk_stride - 1) / a.blk_stride : 0);
    for (;;) {
        unsigned long long idx = 0;
        if (lane == 0) idx = atomicAdd(a.counter, 1ull);
        idx = __shfl_sync(FULL, idx, 0);
        if (idx >= nwork) break;
        const uint64_t blk = a.replay ? a.ovf_queue[idx] : (a.blk_last - (a.blk_offset + idx * a.blk_stride));
        Acc bacc;
        bacc.zero();
        bool ovf = false;
        process_block<TIER, NPL, S>(blk, Lsm, scr, cx, T, bacc, ovf);
        ovf = __any_sync(FULL, ovf);
        ++n_blocks;
        if (ovf) {
            if (TIER == 0) {
                ++n_ovf;
                if (lane == 0) {
                    const unsigned long long pos = atomicAdd(a.ovf_count, 1ull);
                    if (pos < a.ovf_cap) a.ovf_queue[pos] = blk;
                    else ++n_qfull;
                }
                n_qfull = __shfl_sync(FULL, n_qfull, 0);
            } else {
                ++n_fatal;
            }
        } else {
            wacc.add(bacc);
        }
    }
    // warp totals are uniform across lanes: lane 0 publishes, CTA reduces
    if (lane == 0) {
        unsigned long long *w = red + warp * 16;
        w[0] = wacc.vol_lo & 0xFFFFFFFFull;
        w[1] = wacc.vol_lo >> 32;
        w[2] = wacc.vol_hi & 0xFFFFFFFFull;
        w[3] = wacc.vol_hi >> 32;
        w[SLOT_CELLS] = wacc.cells;
        w[SLOT_SINGULAR] = wacc.singular;
        w[SLOT_CAND] = wacc.cand;
        w[SLOT_TIES] = wacc.ties;
        w[SLOT_OVF_BLOCKS] = n_ovf;
        w[SLOT_FATAL] = n_fatal;
        w[SLOT_QFULL] = n_qfull;
        w[SLOT_BLOCKS] = n_blocks;
        w[SLOT_UPDATES] = wacc.updates;
        w[SLOT_LEAVES] = wacc.leaves;
        w[14] = 0;
        w[15] = 0;
    }
    __syncthreads();
    if (threadIdx.x < kNSlots) {
        unsigned long long s = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) s += red[w * 16 + threadIdx.x];
        // limbs: each CTA adds < 2^35 per limb slot (8 warps x 2^32)
        if (s) atomicAdd(a.slots + threadIdx.x, s);
    }
}

}  // namespace dev

size_t enumerate_smem_bytes(int K, int N, int warps) {
    const size_t lbytes = ((size_t)(K + 1) * N * 8 + 15) & ~(size_t)15;
    const size_t bbytes = kBinomRows * kBinomCols * 8;
    const int npl = N > 32 ? 2 : 1;
    return lbytes + bbytes + (size_t)warps * 16 * 8 + 16 + (size_t)warps * (K + 1) * 32 * npl * 8;
}

int kernel_warps_per_cta() { return dev::kWarps; }

typedef void (*KernFn)(LaunchArgs);

static KernFn pick(int tier, int npl, int S) {
#define BDEG_K(T_, P_, S_) \
    if (tier == T_ && npl == P_ && S == S_) return dev::k_enumerate<T_, P_, S_>;
    BDEG_K(0, 1, 0) BDEG_K(0, 1, 1) BDEG_K(0, 1, 2) BDEG_K(0, 1, 3)
    BDEG_K(0, 2, 0) BDEG_K(0, 2, 1) BDEG_K(0, 2, 2) BDEG_K(0, 2, 3)
    BDEG_K(1, 1, 0) BDEG_K(1, 1, 1) BDEG_K(1, 1, 2) BDEG_K(1, 1, 3)
    BDEG_K(1, 2, 0) BDEG_K(1, 2, 1) BDEG_K(1, 2, 2) BDEG_K(1, 2, 3)
#undef BDEG_K
    return nullptr;
}

int enumerate_max_ctas_per_sm(const LaunchArgs &a) {
    const int npl = a.P.N > 32 ? 2 : 1;
    KernFn f = pick(a.tier, npl, a.P.S);
    if (!f) return 1;
    const size_t smem = enumerate_smem_bytes(a.P.K, a.P.N, dev::kWarps);
    cudaFuncSetAttribute((const void *)f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, f, dev::kWarps * 32, smem) != cudaSuccess) return 1;
    return n > 0 ? n : 1;
}

int launch_enumerate(const LaunchArgs &a) {
    const int npl = a.P.N > 32 ? 2 : 1;
    KernFn f = pick(a.tier, npl, a.P.S);
    if (!f) return (int)cudaErrorInvalidValue;
    const size_t smem = enumerate_smem_bytes(a.P.K, a.P.N, dev::kWarps);
    cudaError_t e = cudaFuncSetAttribute((const void *)f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return (int)e;
    f<<<a.grid, dev::kWarps * 32, smem, (cudaStream_t)a.stream>>>(a);
    launch_counter_add(1);
    return (int)cudaGetLastError();
}

}  // namespace bdeg
