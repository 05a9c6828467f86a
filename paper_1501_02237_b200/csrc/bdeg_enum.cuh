// libbdeg device code (sm_100a), shared by the per-tier translation units
// bdeg_enum_t{0,1,2,3}.cu (compiled in parallel) and bdeg_kernels.cu.
//
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
#pragma once
#include "bdeg_internal.h"

#include <cuda_runtime.h>
#include <type_traits>

namespace bdeg {
namespace dev {

constexpr unsigned FULL = 0xffffffffu;
constexpr int kWarps = 4;           // warps per CTA

// Arithmetic tiers (value storage of the K "V" rows / of the lift row):
//   0: int32 / int32, |v| < 2^31, products and numerators exact in int64
//   1: int32 / int64, |V| < 2^Bv, |L| < 2^Bl with Bv + Bl <= 61 and
//      2 Bv <= 61 (runtime bounds), numerators exact in int64
//   2: int64 / int64, |v| < 2^62, numerators in int128, quotients verified
// Tiers 0/1 check every stored value against its bound; a block that leaves
// its tier is re-run in tier 2 (replay launch).
template <int TIER> struct Tr;
template <> struct Tr<0> { typedef int32_t VV; typedef int32_t VL; };
// tier 3 = tier 0 for a plan whose V-minors are all < 2^31 by Hadamard's
// bound (host-proved): V-row range checks are omitted, the lift
// row is still checked
template <> struct Tr<3> { typedef int32_t VV; typedef int32_t VL; };
template <> struct Tr<1> { typedef int32_t VV; typedef int64_t VL; };
template <> struct Tr<2> { typedef int64_t VV; typedef int64_t VL; };

// Exact division by a known divisor d != 0: shift out the 2-adic part, then
// multiply by the inverse of the odd part mod 2^64.  Exact whenever the
// dividend is a multiple of d (Bareiss guarantees it) and the quotient fits.
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
    r.tz = 0;
    r.inv = d < 0 ? ~0ull : 1ull;   // d = +-1: (num >> 0) * inv is the quotient, branch-free
    if (r.unit == 0) {
        r.tz = __ffsll(d) - 1;
        const uint64_t o = (uint64_t)(d >> r.tz);
        uint64_t x = (3 * o) ^ 2;                      // correct to 5 bits
#pragma unroll
        for (int i = 0; i < 4; ++i) x *= 2 - o * x;    // 10, 20, 40, 80 bits
        r.inv = x;
    }
    return r;
}

__device__ __forceinline__ int64_t qdiv64(int64_t num, const Div &dv) {
    if (dv.unit == 1) return num;
    if (dv.unit == -1) return -num;
    return (int64_t)((uint64_t)(num >> dv.tz) * dv.inv);
}
// Exact quotient known to fit int32 (tiers 0/1, V rows): only the low word
// of (num >> tz) times the odd inverse is needed; one wide multiply-back
// verifies the result (flags any quotient outside int32, or INT32_MIN).
__device__ __forceinline__ int32_t qdiv32(int64_t num, const Div &dv, bool &ovf) {
    int32_t q;
    if (dv.unit != 0) {
        const int64_t t = dv.unit > 0 ? num : -num;
        q = (int32_t)t;
        ovf |= (int64_t)q != t;
    } else {
        q = (int32_t)((uint32_t)(num >> dv.tz) * (uint32_t)dv.inv);
        ovf |= (int64_t)q * dv.d != num;
    }
    ovf |= q == INT32_MIN;
    return q;
}
// |v| < lim  (lim a power of two <= 2^62)
__device__ __forceinline__ bool inside(int64_t v, int64_t lim) {
    return (uint64_t)(v + (lim - 1)) <= (uint64_t)(2 * (lim - 1));
}
// |num| < b  (b >= 1)
__device__ __forceinline__ bool within(int64_t num, int64_t b) {
    return (uint64_t)(num + (b - 1)) <= (uint64_t)(2 * (b - 1));
}
// Exact quotient whose range was established from the numerator (|num| <
// L * |d| implies |q| < L): no multiply-back is needed.
__device__ __forceinline__ int32_t qdiv32u(int64_t num, const Div &dv) {
    return (int32_t)((uint32_t)(num >> dv.tz) * (uint32_t)dv.inv);   // also d = +-1 (tz 0, inv +-1)
}
// same for an int64 quotient (tier-1 lift row), branch-free
__device__ __forceinline__ int64_t qdiv64u(int64_t num, const Div &dv) {
    return (int64_t)((uint64_t)(num >> dv.tz) * dv.inv);
}
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
    ovf |= !inside(q, (int64_t)1 << 62);
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

__device__ __forceinline__ float rcp_approx(float x) {   // MUFU.RCP, |x| >= 1 here
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
// signed 32 x 32 -> 64 (IMAD.WIDE) and multiply-add
__device__ __forceinline__ int64_t mulw(int32_t a, int32_t b) {
    int64_t r;
    asm("mul.wide.s32 %0, %1, %2;" : "=l"(r) : "r"(a), "r"(b));
    return r;
}
__device__ __forceinline__ int64_t madw(int32_t a, int32_t b, int64_t c) {
    int64_t r;
    asm("mad.wide.s32 %0, %1, %2, %3;" : "=l"(r) : "r"(a), "r"(b), "l"(c));
    return r;
}
// a float the compiler cannot trace back to its integer source (keeps the
// sign tests as single FSETPs instead of 64-bit integer compares)
__device__ __forceinline__ float opaque(float x) {
    float r;
    asm("mov.b32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float unford(uint32_t o) {   // inverse of ford
    return __uint_as_float((o & 0x80000000u) ? (o & 0x7FFFFFFFu) : ~o);
}

// Per-item accumulators (warp-uniform: every lane holds the same values).
// The item counts its NON-singular candidates (nonsing); its singular count is
// then |item| - nonsing, so dependent subtrees (no pivot: every candidate
// below singular) cost nothing at all -- no subtree-size bookkeeping.
struct Acc {
    uint64_t vol_lo, vol_hi, nonsing, cand, updates;
    uint32_t cells, ties, leaves, dead;
    __device__ void zero() { vol_lo = vol_hi = nonsing = cand = updates = 0; cells = ties = leaves = dead = 0; }
    __device__ void add_vol(uint64_t v) {
        uint64_t t = vol_lo + v;
        vol_hi += (t < vol_lo);
        vol_lo = t;
    }
};
// Per-warp totals.
struct WAcc {
    uint64_t vol_lo, vol_hi, cells, singular, cand, ties, updates, leaves, dead;
    __device__ void zero() { vol_lo = vol_hi = cells = singular = cand = ties = updates = leaves = dead = 0; }
    __device__ void add(const Acc &o) {
        uint64_t t = vol_lo + o.vol_lo;
        vol_hi += (t < vol_lo) + o.vol_hi;
        vol_lo = t;
        cells += o.cells; singular += o.cand - o.nonsing; cand += o.cand; ties += o.ties;
        updates += o.updates; leaves += o.leaves; dead += o.dead;
    }
};

struct Ctx {
    const uint64_t *B;   // binomial table in smem
    const LaunchArgs *A; // the kernel's (grid-constant) arguments: rarely used fields
    int N, K, lane;
    int64_t limV, limL;  // tier-1 bounds (exclusive)
    uint64_t nmask;      // points 0..N-1
    int D, kd, fmin;     // item depth, K - D, smallest forced DFS level
    int mytop;           // this lane's entry of the item tuple: c_{kd + lane} (lane < D)
    uint64_t irb, ire;   // the item's candidates n [rank_begin, rank_end)
    bool deg_only;       // skip cell-dead subtrees (singular count becomes an upper bound)
    bool dead_full;      // full mode: find cell-dead subtrees too (their leaves only count non-singular j)
    bool partial;        // the item is cut by the rank range
    __device__ __forceinline__ uint64_t C(int n, int k) const { return B[n * kBinomCols + k]; }
    // |[base, base+size) n [irb, ire)| (subtrees below the item level lie inside the item)
    __device__ __forceinline__ uint64_t isect(uint64_t base, uint64_t size) const {
        if (!partial) return size;
        uint64_t lo = base > irb ? base : irb;
        uint64_t hi = base + size < ire ? base + size : ire;
        return hi > lo ? hi - lo : 0;
    }
    // optional emission of a found cell
    __device__ __forceinline__ void emit(uint64_t mask, uint64_t vol) const {
        if (A->cells_out && lane == 0) {
            const unsigned long long pos = atomicAdd(A->cells_cnt, 1ull);
            if (pos < A->cells_cap) {
                A->cells_out[2 * pos] = mask;
                A->cells_out[2 * pos + 1] = vol;
            }
        }
    }
};

// ------------------------------------------------------------------ leaf
// After the whole (K-1)-prefix P is eliminated every point l is a 2-vector
// (x_l, y_l) = g * (+-det V_{P u l}, lift minor) for a common non-zero g.
// With kappa = sign(last pivot) * sign(g), sigma = P u {j} is a cell iff
//     sign(x_j) * (x_j * yk_l - x_l * yk_j) > 0   for every l not in sigma,
// yk = kappa * y (DESIGN.md §"Leaf test").  So only the unique extreme
// slopes yk/x of the half-planes x > 0 (min) and x < 0 (max) can be cells:
// found with REDUX over approximate float keys (error << margin), then
// verified exactly (int128) against every lane.  |det| = |x_j| / |g|.
constexpr uint32_t kKeyMargin = 64;   // key units (ulps); the fp32 key error is < 8

template <int NPL>
__device__ __forceinline__ void leaf_test(const int64_t (&x)[NPL], const int64_t (&y)[NPL], int c1,
                                          uint64_t base, uint64_t inP, int kappa, uint64_t gabs,
                                          const Ctx &cx, Acc &acc) {
    int jlo = 0, jhi = c1;
    if (cx.partial) {
        if (cx.irb > base) jlo = (cx.irb - base >= (uint64_t)c1) ? c1 : (int)(cx.irb - base);
        if (cx.ire < base + (uint64_t)c1) jhi = (cx.ire <= base) ? 0 : (int)(cx.ire - base);
        if (jlo >= jhi) return;
    }
    acc.leaves += 1;
    // warp-uniform point masks: countable j in [jlo, jhi); valid l = not in P, < N
    const uint64_t cntm = ((jhi >= 64) ? ~0ull : ((1ull << jhi) - 1)) & ~((1ull << jlo) - 1);
    const uint64_t valm = ~inP & cx.nmask;
    const uint32_t lanebit = 1u << cx.lane;
    int64_t yk[NPL];
    uint32_t kp = 0xFFFFFFFFu, km = 0xFFFFFFFFu;
    uint32_t kq[NPL];
    unsigned sing = 0;
    bool bad0 = false;
#pragma unroll
    for (int q = 0; q < NPL; ++q) {
        const uint32_t vq = (uint32_t)(valm >> (32 * q));
        const bool v = (vq & lanebit) != 0;
        yk[q] = kappa > 0 ? y[q] : -y[q];
        const bool zx = x[q] == 0;
        sing += __popc(__ballot_sync(FULL, !zx) & (uint32_t)(cntm >> (32 * q)));   // non-singular
        bad0 |= v && zx && yk[q] < 0;
        // slope key yk/x (approximate; error << kKeyMargin key units)
        const uint32_t o = ford(__fdividef((float)yk[q], (float)x[q]));
        kq[q] = o;
        if (v && x[q] > 0) kp = min(kp, o);
        if (v && x[q] < 0) km = min(km, ~o);
    }
    acc.nonsing += sing;
    if (__any_sync(FULL, bad0)) return;          // a point of span(P) lies strictly below
    const uint32_t mp = __reduce_min_sync(FULL, kp);   // ~ min slope over x > 0
    const uint32_t mm = __reduce_min_sync(FULL, km);   // ~ max slope over x < 0 (complemented)
    // both cells need  max_{x<0} slope < min_{x>0} slope
    if (mp != 0xFFFFFFFFu && mm != 0xFFFFFFFFu && (~mm) > mp + 2 * kKeyMargin) return;
    uint64_t candmask = 0;
#pragma unroll
    for (int q = 0; q < NPL; ++q) {
        const bool c = (x[q] > 0 && kq[q] <= mp + kKeyMargin) || (x[q] < 0 && (~kq[q]) <= mm + kKeyMargin);
        candmask |= (uint64_t)__ballot_sync(FULL, c) << (32 * q);
    }
    candmask &= cntm;
    while (candmask) {
        const int j = __ffsll((long long)candmask) - 1;
        candmask &= candmask - 1;
        const int jl = j & 31;
        int64_t xs = x[0], ys = yk[0];
        if (NPL > 1 && (j >> 5)) { xs = x[NPL - 1]; ys = yk[NPL - 1]; }
        const int64_t xj = shfl<int64_t>(xs, jl);
        const int64_t yj = shfl<int64_t>(ys, jl);
        bool bad = false, zero = false;
#pragma unroll
        for (int q = 0; q < NPL; ++q) {
            const int l = cx.lane + 32 * q;
            if (((valm >> l) & 1ull) && l != j) {
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
            const uint64_t vol = (uint64_t)(xj < 0 ? -xj : xj) / gabs;   // |det V_sigma|
            acc.add_vol(vol);
            cx.emit(inP | (1ull << j), vol);
        }
    }
}

// --------------------------------------------------------- elimination
// State of this lane's points: sv[q][0..RV-1] (remaining V rows), sl[q] (lift).
// Pivot column values cv[.], cl; pivot row pr; pivot piv; previous pivot dv:
//     a'_{o,l} = (piv * a_{o,l} - a_{o,p} * a_{pr,l}) / prev      (Bareiss)
template <int TIER, int NPL, int RV>
__device__ __forceinline__ void elim_step(const typename Tr<TIER>::VV (&sv)[NPL][RV],
                                          const typename Tr<TIER>::VL (&sl)[NPL],
                                          const typename Tr<TIER>::VV (&cv)[RV],
                                          typename Tr<TIER>::VL cl, int pr, typename Tr<TIER>::VV piv,
                                          const Div &dv, int64_t bV, int64_t bL, const Ctx &cx,
                                          typename Tr<TIER>::VV (&ov)[NPL][RV - 1],
                                          typename Tr<TIER>::VL (&ol)[NPL], bool &ovf) {
    typedef typename Tr<TIER>::VV VV;
    typedef typename Tr<TIER>::VL VL;
#pragma unroll
    for (int q = 0; q < NPL; ++q) {
        VV prow = sv[q][0];
#pragma unroll
        for (int r = 1; r < RV; ++r) if (pr == r) prow = sv[q][r];
#pragma unroll
        for (int o = 0; o < RV - 1; ++o) {
            const VV s = (o < pr) ? sv[q][o] : sv[q][o + 1];
            const VV cs = (o < pr) ? cv[o] : cv[o + 1];
            if constexpr (TIER == 2) {
                ov[q][o] = qdiv128((i128)piv * s - (i128)cs * prow, dv, ovf);
            } else {
                // |num| < bV = L |prev|  <=>  |quotient| < L (tier bound)
                const int64_t num = madw(piv, s, mulw(-cs, prow));
                if constexpr (TIER != 3) ovf |= !within(num, bV);
                ov[q][o] = qdiv32u(num, dv);
            }
        }
        if constexpr (TIER == 2) {
            ol[q] = qdiv128((i128)piv * sl[q] - (i128)cl * prow, dv, ovf);
        } else if constexpr (TIER == 0 || TIER == 3) {
            const int64_t num = madw(piv, sl[q], mulw(-cl, prow));
            ovf |= !within(num, bL);
            ol[q] = qdiv32u(num, dv);
        } else {
            const int64_t num = (int64_t)piv * (int64_t)sl[q] - (int64_t)cl * (int64_t)prow;
            ovf |= !within(num, bL);
            ol[q] = (VL)qdiv64u(num, dv);
        }
    }
}

template <int TIER, int NPL, int RV>
__device__ __forceinline__ void fetch_col(const typename Tr<TIER>::VV (&sv)[NPL][RV],
                                          const typename Tr<TIER>::VL (&sl)[NPL], int c,
                                          typename Tr<TIER>::VV (&cv)[RV], typename Tr<TIER>::VL &cl) {
    typedef typename Tr<TIER>::VV VV;
    typedef typename Tr<TIER>::VL VL;
    const int src = c & 31;
    const bool hi = NPL > 1 && (c >> 5) != 0;
#pragma unroll
    for (int r = 0; r < RV; ++r) cv[r] = shfl<VV>(hi ? sv[NPL - 1][r] : sv[0][r], src);
    cl = shfl<VL>(hi ? sl[NPL - 1] : sl[0], src);
}

// ------------------------------------------------------------ leaf level
// Tiers 0/1: the DFS level that picks c_1 (two V rows u, v and the lift z
// remain) fused with the leaf test.  For pivot point c the leaf 2-vectors are
//   X_l = piv*s_l - cs*prow_l,   Y_l = kappa'*(piv*z_l - z_c*prow_l)
// (prow = pivot row, s = the other V row), i.e. prev * (true Bareiss values):
// no division is needed, since slopes and cross-product signs are invariant
// under the common factor prev, whose sign is folded into kappa'
// (= sign(piv) * sign(prev)).  |det| = |X_j| / |prev| for the (rare) cells.
// Cell-dead test of a DFS node (P:913-929 monotonicity, in determinant
// form).  If a point l outside the prefix has all remaining V-row values 0
// (v_l lies in the span of the prefix vectors), its lift residual y_l only
// gets multiplied by pivot ratios further down: at any leaf of this subtree
// the facet test reads sign(g) * y_l with g the node's last pivot.  A
// negative value means l lies strictly below every hyperplane through the
// prefix: no cell exists in the subtree (only the non-singular count remains).
template <int TIER, int NPL, int RV>
__device__ __forceinline__ bool node_dead(const typename Tr<TIER>::VV (&sv)[NPL][RV],
                                          const typename Tr<TIER>::VL (&sl)[NPL], uint64_t inP,
                                          int64_t g, const Ctx &cx) {
    bool below = false;
#pragma unroll
    for (int q = 0; q < NPL; ++q) {
        const int l = cx.lane + 32 * q;
        bool zero = true;
#pragma unroll
        for (int r = 0; r < RV; ++r) zero &= sv[q][r] == 0;
        const bool neg = (g > 0) ? (sl[q] < 0) : (sl[q] > 0);
        below |= zero && neg && l < cx.N && !((inP >> l) & 1ull);
    }
    return __any_sync(FULL, below);
}

// Leaf level, tiers 0/1/3 (round 2 rewrite).  Invariant: every point that
// cannot enter a candidate here -- the prefix P (pivot columns are zeroed),
// lanes >= N, and c itself -- has u = v = z = 0, so it yields X = Y = 0:
// never a slope, never "below", never counted (j < c < min P).  No per-point
// validity masks are needed on the hot path; the rare exact verification
// rebuilds them.
//   X_l = u_c v_l - v_c u_l                (cross product: the 1-D quotient
//                                            by c; negating every X leaves the
//                                            cell test and |X| unchanged)
//   Y_l = kappa' (e_c z_l - z_c e_l)       (e = the row of the pivot: u if
//                                            u_c != 0, else v)
// and with the sign-free key k_l = Y_l / |X_l| the two half-planes need
//   min_{X>0} k  and  min_{X<0} k  with  min_{X>0} k + min_{X<0} k >= 0
// (the max slope over X<0 is -min_{X<0} k).  Keys are fp32 with a relative
// error < 2^-21; the reductions are CREDUX.MIN.F32 and every margin is
// relative (kRelMargin), so exactness rests on the int128 verification.
constexpr float kRelMargin = 3.0517578125e-05f;   // 2^-15

__device__ __forceinline__ float redux_min_f32(float v) {
    float r;
    asm volatile("redux.sync.min.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(v));
    return r;
}
// bits [lo, hi) of a 32-bit word, 0 <= lo <= hi <= 32
__device__ __forceinline__ uint32_t bits_range(int lo, int hi) {
    const uint32_t h = hi >= 32 ? 0xFFFFFFFFu : ((1u << hi) - 1u);
    const uint32_t l = lo >= 32 ? 0xFFFFFFFFu : ((1u << lo) - 1u);
    return h & ~l;
}

template <int TIER, int NPL, bool R>
__device__ __forceinline__ void leaf_level(const typename Tr<TIER>::VV (&sv)[NPL][2],
                                           const typename Tr<TIER>::VL (&sl)[NPL], int lo, int hi,
                                           uint64_t base, uint64_t inP, int64_t prev, const Ctx &cx,
                                           Acc &acc, bool dead) {
    typedef typename Tr<TIER>::VV VV;
    typedef typename Tr<TIER>::VL VL;
    const bool gneg = prev < 0;
    const float INFF = __int_as_float(0x7f800000);
    if (hi <= lo) return;
    if (!R) {                                  // whole leaves: counters per parent
        const uint64_t nl = (uint64_t)(hi - lo);
        acc.leaves += (uint32_t)nl;
        acc.updates += 2ull * cx.N * nl;
    }
    // X of this lane's slot-q point for the leaf with pivot column (uc, vc)
    auto xval = [&](const VV uc, const VV nvc, const int q) -> int64_t {
        return madw(uc, sv[q][1], mulw(nvc, sv[q][0]));
    };
    // rejected: a point strictly below (-> -inf) or min_{X>0} k + min_{X<0} k < 0
    // beyond the key error
    auto rejected = [&](const float mp, const float mm) {
        return mp == -INFF || (mp + mm < -(fabsf(mp) + fabsf(mm)) * kRelMargin);
    };
    // Y of a point (e = the pivot row's entry, z = lift) for the leaf's (pz, ncz)
    auto yval = [&](const VV pz, const VL ncz, const VV el, const VL zl) -> int64_t {
        if constexpr (TIER == 0 || TIER == 3) return madw(pz, zl, mulw(ncz, el));
        else return (int64_t)pz * (int64_t)zl + (int64_t)ncz * (int64_t)el;
    };
    struct Ev {
        int64_t X, Y;
        float fx, key;
    };
    // One leaf c, held in slot SC (compile time: the loop below is split at 32).
    auto leaf = [&](auto SCC, const int c) {
        constexpr int SC = decltype(SCC)::value;
        int jlo = 0, jhi = c;
        if constexpr (R) {
            const uint64_t nb = base + (uint64_t)c * (uint64_t)(c - 1) / 2;   // + C(c, 2)
            if (cx.irb > nb) jlo = (cx.irb - nb >= (uint64_t)c) ? c : (int)(cx.irb - nb);
            if (cx.ire < nb + (uint64_t)c) jhi = (cx.ire <= nb) ? 0 : (int)(cx.ire - nb);
            if (jlo >= jhi) return;
            acc.leaves += 1;
            acc.updates += 2ull * cx.N;
        }
        const int src = c & 31;
        const VV uc = shfl<VV>(sv[SC][0], src);
        const VV vc = shfl<VV>(sv[SC][1], src);
        const VL zc = shfl<VL>(sl[SC], src);
        if ((uc | vc) == 0) return;                // dependent prefix: every j singular
        // countable j per slot (uniform masks)
        const uint32_t m0 = R ? bits_range(jlo, jhi < 32 ? jhi : 32) : (SC == 0 ? bits_range(0, c) : 0xFFFFFFFFu);
        const uint32_t m1 = (NPL > 1 && SC == 1)
                                ? (R ? bits_range(jlo > 32 ? jlo - 32 : 0, jhi > 32 ? jhi - 32 : 0)
                                     : bits_range(0, c - 32))
                                : 0u;
        const uint32_t n0 = m0, n1 = m1;
        const VV nvc = -vc;
        if (dead) {                                // no cell below: non-singular count only
            unsigned sd = __popc(__ballot_sync(FULL, xval(uc, nvc, 0) != 0) & n0);
            if constexpr (NPL > 1 && SC == 1) sd += __popc(__ballot_sync(FULL, xval(uc, nvc, 1) != 0) & n1);
            acc.nonsing += sd;
            acc.dead += 1;
            return;
        }
        const bool p0 = uc != 0;
        const VV ec = p0 ? uc : vc;
        const bool kneg = (ec < 0) != gneg;
        const VV pz = kneg ? (VV)-ec : ec;
        const VL ncz = kneg ? zc : (VL)-zc;
        Ev ev[NPL];
        float fp = INFF, fm = INFF;
        bool bad0 = false;
        unsigned nons = 0;
        auto eval = [&](const int q) {
            ev[q].X = xval(uc, nvc, q);
            ev[q].Y = yval(pz, ncz, p0 ? sv[q][0] : sv[q][1], sl[q]);
            ev[q].fx = opaque((float)ev[q].X);
            const float fy = opaque((float)ev[q].Y);
            const bool zer = ev[q].fx == 0.0f;
            bad0 |= zer && fy < 0.0f;
            ev[q].key = fy * rcp_approx(fabsf(ev[q].fx));
            fp = fminf(fp, ev[q].fx > 0.0f ? ev[q].key : INFF);
            fm = fminf(fm, ev[q].fx < 0.0f ? ev[q].key : INFF);
        };
        eval(0);
        nons += __popc(__ballot_sync(FULL, ev[0].fx != 0.0f) & n0);
        if constexpr (NPL == 2) {
            // Early rejection on points 0..31 alone: a violation among a subset of
            // the points is one of the whole set (its min over X > 0 can only
            // drop, its max over X < 0 only rise); slot 1 is evaluated for the
            // few leaves that survive, and for the count when c > 32.
            const float mp0 = redux_min_f32(bad0 ? -INFF : fp);
            const float mm0 = redux_min_f32(fm);
            if (rejected(mp0, mm0)) {
                if constexpr (SC == 1) nons += __popc(__ballot_sync(FULL, xval(uc, nvc, 1) != 0) & n1);
                acc.nonsing += nons;
                return;
            }
            eval(1);
            nons += __popc(__ballot_sync(FULL, ev[1].fx != 0.0f) & n1);
        }
        acc.nonsing += nons;
        const float mp = redux_min_f32(bad0 ? -INFF : fp);
        const float mm = redux_min_f32(fm);
        if (rejected(mp, mm)) return;
        const float tp = mp + fabsf(mp) * kRelMargin;
        const float tm = mm + fabsf(mm) * kRelMargin;
        uint64_t candmask = 0;
#pragma unroll
        for (int q = 0; q < NPL; ++q) {
            const bool cd = (ev[q].fx > 0.0f && ev[q].key <= tp) || (ev[q].fx < 0.0f && ev[q].key <= tm);
            candmask |= (uint64_t)(__ballot_sync(FULL, cd) & (q == 0 ? m0 : m1)) << (32 * q);
        }
        const uint64_t gabs = (uint64_t)(prev < 0 ? -prev : prev);
        while (candmask) {                         // exact verification (int128)
            const int j = __ffsll((long long)candmask) - 1;
            candmask &= candmask - 1;
            const int jl = j & 31;
            const bool js = NPL > 1 && (j >> 5) != 0;
            const int64_t xj = shfl<int64_t>(js ? ev[NPL - 1].X : ev[0].X, jl);
            const int64_t yj = shfl<int64_t>(js ? ev[NPL - 1].Y : ev[0].Y, jl);
            bool bad = false, zero = false;
#pragma unroll
            for (int q = 0; q < NPL; ++q) {
                const int l = cx.lane + 32 * q;
                if (l < cx.N && !((inP >> l) & 1ull) && l != c && l != j) {
                    i128 cr = (i128)xj * ev[q].Y - (i128)ev[q].X * yj;
                    if (xj < 0) cr = -cr;
                    bad |= cr < 0;
                    zero |= cr == 0;
                }
            }
            if (__any_sync(FULL, bad)) continue;
            if (__any_sync(FULL, zero)) {
                acc.ties += 1;                     // would-be cell on a tie (reading Z3)
            } else {
                acc.cells += 1;
                const uint64_t vol = (uint64_t)(xj < 0 ? -xj : xj) / gabs;   // |det V_sigma|
                acc.add_vol(vol);
                cx.emit(inP | (1ull << c) | (1ull << j), vol);
            }
        }
    };
    const int mid = hi < 32 ? hi : 32;
    for (int c = lo; c < mid; ++c) leaf(std::integral_constant<int, 0>{}, c);
    if constexpr (NPL == 2)
        for (int c = lo > 32 ? lo : 32; c < hi; ++c) leaf(std::integral_constant<int, 1>{}, c);
}

// ------------------------------------------------------------ inner DFS
// RV >= 2 remaining V rows.  Chooses c_i, i = RV-1, in [i, cbound) in colex
// order; base = rank contribution of the indices above; prev = last pivot.
template <int TIER, int NPL, int RV, bool R>
__device__ __forceinline__ void inner_dfs(const typename Tr<TIER>::VV (&sv)[NPL][RV],
                                          const typename Tr<TIER>::VL (&sl)[NPL], int cbound,
                                          uint64_t base, uint64_t inP, int64_t prev, const Ctx &cx,
                                          Acc &acc, bool &ovf, bool dead) {
    typedef typename Tr<TIER>::VV VV;
    typedef typename Tr<TIER>::VL VL;
    constexpr int i = RV - 1;
    int lo = i, hi = cbound;
    if (i >= cx.fmin) {                      // forced level: c_i is fixed by the work item
        lo = __shfl_sync(FULL, cx.mytop, i - cx.kd);
        hi = lo + 1;
    }
    if constexpr (RV == 2 && TIER != 2) {
        leaf_level<TIER, NPL, R>(sv, sl, lo, hi, base, inP, prev, cx, acc, dead);
        return;
    }
    Div dv;
    int64_t bV = 0, bL = 0;   // numerator bounds: tier bound x |prev| (tiers 0/1)
    if constexpr (RV > 2 || TIER == 2) dv = make_div(prev);
    if constexpr (TIER != 2) {
        const int64_t ap = prev < 0 ? -prev : prev;
        bV = ((TIER == 0 || TIER == 3) ? (int64_t)INT32_MAX : cx.limV) * ap;
        bL = ((TIER == 0 || TIER == 3) ? (int64_t)INT32_MAX : cx.limL) * ap;
    }
    for (int c = lo; c < hi; ++c) {
        // rank bookkeeping only for rank-range launches (R): whole items need
        // the subtree size for dependent prefixes only
        const uint64_t nb = R ? base + cx.C(c, i + 1) : 0;
        if constexpr (R) {
            if (cx.isect(nb, cx.C(c, i)) == 0) continue;
        }
        VV cv[RV];
        VL cl;
        fetch_col<TIER, NPL, RV>(sv, sl, c, cv, cl);
        int pr = -1;
#pragma unroll
        for (int r = RV - 1; r >= 0; --r) if (cv[r] != 0) pr = r;
        if (pr < 0) continue;                // prefix dependent: whole subtree singular
        VV piv = cv[0];
#pragma unroll
        for (int r = 1; r < RV; ++r) if (pr == r) piv = cv[r];
        acc.updates += (uint64_t)RV * cx.N;
        if constexpr (RV == 2) {
            // last prefix index: the leaf 2-vectors
            int64_t xx[NPL], yy[NPL];
            const VV cs = pr == 0 ? cv[1] : cv[0];
            {
#pragma unroll
                for (int q = 0; q < NPL; ++q) {
                    const VV prow = pr == 0 ? sv[q][0] : sv[q][1];
                    const VV s = pr == 0 ? sv[q][1] : sv[q][0];
                    xx[q] = qdiv128((i128)piv * s - (i128)cs * prow, dv, ovf);
                    yy[q] = qdiv128((i128)piv * sl[q] - (i128)cl * prow, dv, ovf);
                }
                if (__any_sync(FULL, ovf)) { ovf = true; return; }
                leaf_test<NPL>(xx, yy, c, nb, inP | (1ull << c), piv > 0 ? 1 : -1, 1, cx, acc);
            }
        } else {
            VV ov[NPL][RV - 1];
            VL ol[NPL];
            // overflow is voted once per item (the item is discarded and replayed);
            // loops are index-bounded, so garbage values cannot hang the warp
            elim_step<TIER, NPL, RV>(sv, sl, cv, cl, pr, piv, dv, bV, bL, cx, ov, ol, ovf);
            const uint64_t cinP = inP | (1ull << c);
            // cell-dead subtree: degree-only skips it; full mode keeps
            // walking it for the non-singular count but its leaves skip the facet test
            const bool cdead = dead || (cx.dead_full || cx.deg_only) &&
                                           node_dead<TIER, NPL, RV - 1>(ov, ol, cinP, (int64_t)piv, cx);
            if (cdead && cx.deg_only) continue;  // no cell in the subtree: skip it
            inner_dfs<TIER, NPL, RV - 1, R>(ov, ol, c, nb, cinP, (int64_t)piv, cx, acc, ovf, cdead);
        }
    }
}

// ------------------------------------------------------------ one work item
// Colex unranking of r over cnt-subsets of {0..M-1} (M <= 64): lane
// lane_off + t receives element t + shift.  Warp-parallel: one ballot pair
// per element finds the largest x with C(x, t+1) <= r.
__device__ __forceinline__ void unrank_lanes(uint64_t r, int cnt, int M, int shift, int lane_off,
                                             const Ctx &cx, int &mytop) {
    const int lane = cx.lane;
    for (int t = cnt - 1; t >= 0; --t) {
        const uint32_t m0 = __ballot_sync(FULL, lane < M && cx.C(lane, t + 1) <= r);
        const uint32_t m1 = __ballot_sync(FULL, lane + 32 < M && cx.C(lane + 32, t + 1) <= r);
        const int u = m1 ? 32 + 31 - __clz(m1) : 31 - __clz(m0);
        r -= cx.C(u, t + 1);
        if (lane == t + lane_off) mytop = u + shift;
    }
}

// Queue position -> item depth D and tuple (lane t < D holds c_{K-D+t}).
__device__ __forceinline__ int decode_item(uint64_t pos, const LaunchArgs &a, const Ctx &cx, int &mytop) {
    const int K = cx.K, N = cx.N;
    if (a.mode == 0) {                       // base-depth colex id (rank-range calls)
        const int D = a.P.D;
        unrank_lanes(a.blk_last - pos, D, N - (K - D), K - D, 0, cx, mytop);
        return D;
    }
    if (pos < a.n_split) {                   // an item split to a finer depth
        const uint64_t e = a.split[pos];
        const int D = (int)(e >> 58);
        unrank_lanes(e & ((1ull << 58) - 1), D, N - (K - D), K - D, 0, cx, mytop);
        return D;
    }
    const int D = a.P.D;                     // grouped base-depth item
    if (D == 0) return 0;
    const uint64_t q = pos - a.n_split;
    // group g: the last with grp_cum[g] <= q (g < n_grp <= 64)
    const int lane = cx.lane;
    const bool c0 = lane < a.n_grp && a.grp_cum[lane] <= q;
    const bool c1 = lane + 32 < a.n_grp && a.grp_cum[lane + 32] <= q;
    const uint32_t b0 = __ballot_sync(FULL, c0), b1 = __ballot_sync(FULL, c1);
    const int g = b1 ? 32 + 31 - __clz(b1) : 31 - __clz(b0);
    const int u = (int)a.grp_u[g];
    if (lane == 0) mytop = u;
    // the rest: a (D-1)-subset of {u+1..N-1}
    unrank_lanes(q - a.grp_cum[g], D - 1, N - u - 1, u + 1, 1, cx, mytop);
    return D;
}

// The item (depth D, tuple in mytop) covers the contiguous colex ranks below
// its tuple.  The T = K-1-S largest entries are eliminated in shared scratch
// (tier-2 arithmetic); the other D-T are "forced" levels of the S-level
// register DFS, which walks the rest.
template <int TIER, int NPL, int S, bool R>
__device__ void process_item(int D, int mytop, const int64_t *Lsm, int64_t *scr, const Ctx &cx0,
                             Acc &acc, bool &ovf) {
    typedef typename Tr<TIER>::VV VV;
    typedef typename Tr<TIER>::VL VL;
    const int lane = cx0.lane;
    const int K = cx0.K, N = cx0.N;
    const int kd = K - D;
    constexpr int NP = 32 * NPL;
    const int T = K - 1 - S;
    // item rank range: sum over all D entries; size C(c_{kd}, kd)
    uint64_t tall = (lane < D) ? cx0.C(mytop, kd + lane + 1) : 0;
    uint64_t ttop = (lane < D && lane >= D - T) ? tall : 0;    // the T smem entries only
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        tall += __shfl_xor_sync(FULL, tall, o);
        ttop += __shfl_xor_sync(FULL, ttop, o);
    }
    const int cfirst = D > 0 ? __shfl_sync(FULL, mytop, 0) : N;
    const uint64_t isize = cx0.C(cfirst, kd);
    Ctx cx = cx0;
    cx.mytop = mytop;
    cx.D = D;
    cx.kd = kd;
    cx.fmin = (D > T) ? kd : S + 1;
    {
        // effective range = item n [rb, re); the item's candidate count is its
        // size, its singular count |item| - non-singular (Acc).
        const uint64_t rb = cx0.A->rank_begin, re = cx0.A->rank_end;
        const uint64_t lo = tall > rb ? tall : rb;
        const uint64_t hi = tall + isize < re ? tall + isize : re;
        if (hi <= lo) return;
        cx.irb = lo;
        cx.ire = hi;
        cx.partial = (lo != tall) || (hi != tall + isize);
        acc.cand = hi - lo;                   // the item's candidates: a contiguous colex interval
    }
    uint64_t inP = 0;
    {
        const uint64_t bit = (lane < D && lane >= D - T) ? (1ull << mytop) : 0ull;
        const unsigned lo = __reduce_or_sync(FULL, (unsigned)bit);
        const unsigned hi = __reduce_or_sync(FULL, (unsigned)(bit >> 32));
        inP = ((uint64_t)hi << 32) | lo;
    }
    // --- elimination of the T largest entries in shared scratch: scr[i*NP + l], rows 0..K
    int64_t prev = 1;
    uint64_t alive = (1ull << K) - 1;
    if (T > 0) {
        __syncwarp();
        for (int i = 0; i <= K; ++i)
#pragma unroll
            for (int q = 0; q < NPL; ++q) {
                const int l = lane + 32 * q;
                scr[i * NP + l] = (l < N) ? Lsm[l * (K + 1) + i] : 0;
            }
        __syncwarp();
        for (int t = 0; t < T; ++t) {
            const int p = __shfl_sync(FULL, mytop, D - 1 - t);   // pivot order c_{K-1}, c_{K-2}, ...
            const bool nz = (lane < K) && ((alive >> lane) & 1ull) && scr[lane * NP + p] != 0;
            const unsigned bal = __ballot_sync(FULL, nz);
            if (bal == 0) return;                                 // dependent prefix: all singular
            const int r = __ffs(bal) - 1;
            const int64_t piv = scr[r * NP + p];
            const Div dv = make_div(prev);
            bool o = false;
            // tiers 0/1: every value obeys the tier bound (|V| < LV, |lift| < LL,
            // checked), so numerators are exact in int64 and |num| < L |prev|
            // <=> |quotient| < L; tier 2: int128 numerators, quotients verified
            const int64_t ap = prev < 0 ? -prev : prev;
            const int64_t bV = ((TIER == 0 || TIER == 3) ? (int64_t)INT32_MAX : cx.limV) * ap;
            const int64_t bL = ((TIER == 0 || TIER == 3) ? (int64_t)INT32_MAX : cx.limL) * ap;
            for (int i = 0; i <= K; ++i) {
                if (i == r || (i < K && !((alive >> i) & 1ull))) continue;
                const int64_t ci = scr[i * NP + p];
                const int64_t b = i < K ? bV : bL;
#pragma unroll
                for (int q = 0; q < NPL; ++q) {
                    const int l = lane + 32 * q;
                    if (l == p) continue;
                    if constexpr (TIER == 2) {
                        const i128 num = (i128)piv * scr[i * NP + l] - (i128)ci * scr[r * NP + l];
                        scr[i * NP + l] = qdiv128(num, dv, o);
                    } else {
                        const int64_t num = piv * scr[i * NP + l] - ci * scr[r * NP + l];
                        if (TIER != 3 || i == K) o |= !within(num, b);
                        scr[i * NP + l] = qdiv64u(num, dv);
                    }
                }
            }
            acc.updates += (uint64_t)(K - t) * N;
            if (__any_sync(FULL, o)) { ovf = true; return; }     // beyond the int64 tier
            alive &= ~(1ull << r);
            prev = piv;
            __syncwarp();
            // the pivot column is 0 below the pivot (Bareiss); store it, so that
            // prefix points carry all-zero rows into the register DFS (leaf invariant)
            for (int i = lane; i <= K; i += 32)
                if (i != r) scr[i * NP + p] = 0;
            __syncwarp();
        }
    }
    // --- registers: remaining S+1 V rows (ascending) then the lift row
    VV sv[NPL][S + 1];
    VL sl[NPL];
    bool o = false;
    if (T > 0) {
        int k = 0;
        for (int i = 0; i < K; ++i) {
            if (!((alive >> i) & 1ull)) continue;
#pragma unroll
            for (int kk = 0; kk < S + 1; ++kk)
                if (kk == k)
#pragma unroll
                    for (int q = 0; q < NPL; ++q) {
                        const int64_t v = scr[i * NP + lane + 32 * q];
                        if constexpr (TIER == 0 || TIER == 3) o |= !inside(v, (int64_t)1 << 31);
                        if constexpr (TIER == 1) o |= !inside(v, cx.limV);
                        sv[q][kk] = (VV)v;
                    }
            ++k;
        }
#pragma unroll
        for (int q = 0; q < NPL; ++q) {
            const int64_t v = scr[K * NP + lane + 32 * q];
            if constexpr (TIER == 0 || TIER == 3) o |= !inside(v, (int64_t)1 << 31);
            if constexpr (TIER == 1) o |= !inside(v, cx.limL);
            sl[q] = (VL)v;
        }
    } else {                                   // S = K-1: straight from the staged matrix
#pragma unroll
        for (int q = 0; q < NPL; ++q) {
            const int l = lane + 32 * q;
#pragma unroll
            for (int kk = 0; kk < S + 1; ++kk) {
                const int64_t v = (l < N) ? Lsm[l * (K + 1) + kk] : 0;
                if constexpr (TIER == 0 || TIER == 3) o |= !inside(v, (int64_t)1 << 31);
                if constexpr (TIER == 1) o |= !inside(v, cx.limV);
                sv[q][kk] = (VV)v;
            }
            const int64_t v = (l < N) ? Lsm[l * (K + 1) + K] : 0;
            if constexpr (TIER == 0 || TIER == 3) o |= !inside(v, (int64_t)1 << 31);
            if constexpr (TIER == 1) o |= !inside(v, cx.limL);
            sl[q] = (VL)v;
        }
    }
    if (__any_sync(FULL, o)) { ovf = true; return; }
    const int ctop = T > 0 ? __shfl_sync(FULL, mytop, D - T) : N;   // c_{S+1}
    if constexpr (S == 0) {
        // the item is a single leaf: prefix = the tuple, c1 = ctop; the
        // shared-memory values are the true minors (divided), so g = 1
        int64_t xx[NPL], yy[NPL];
#pragma unroll
        for (int q = 0; q < NPL; ++q) { xx[q] = (int64_t)sv[q][0]; yy[q] = (int64_t)sl[q]; }
        leaf_test<NPL>(xx, yy, ctop, ttop, inP, prev > 0 ? 1 : -1, 1, cx, acc);
    } else {
        const bool dead = (cx.dead_full || cx.deg_only) && node_dead<TIER, NPL, S + 1>(sv, sl, inP, prev, cx);
        if (dead && cx.deg_only) return;
        inner_dfs<TIER, NPL, S + 1, R>(sv, sl, ctop, ttop, inP, prev, cx, acc, ovf, dead);
    }
}

// ------------------------------------------------------------ TMA staging
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

template <int TIER, int NPL, int S, bool R>
// Occupancy: <= 128 registers (4 CTAs of 4 warps per SM) at every DFS depth;
// for S >= 5 this spills some of the deeper DFS state to local memory, which
// measured faster than 168 registers at 3 CTAs (W_{2,6} 266.8 -> 254.5 ms,
// tools/ab_bench.sh).
#ifndef BDEG_MIN_BLOCKS
#define BDEG_MIN_BLOCKS 4
#endif
__global__ void __launch_bounds__(kWarps * 32, BDEG_MIN_BLOCKS)
k_enumerate(const __grid_constant__ LaunchArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    // a replay with nothing marked by the launch before it (the common case)
    if (a.replay && a.replay_gate && *(volatile const unsigned long long *)a.replay_gate == 0) return;
    const int K = a.P.K, N = a.P.N, T = a.P.T;
    (void)T;
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
    cx.A = &a;
    cx.partial = true;
    cx.limV = (int64_t)1 << a.bits_v;
    cx.limL = (int64_t)1 << a.bits_l;
    cx.nmask = (N >= 64) ? ~0ull : ((1ull << N) - 1);
    int64_t *scr = scr_all + (size_t)warp * (K + 1) * 32 * NPL;

    cx.D = a.P.D;
    cx.deg_only = a.degree_only != 0;
    cx.dead_full = a.dead_full != 0;
    cx.kd = K - a.P.D;
    cx.fmin = S + 1;
    cx.mytop = 0;
    WAcc wacc;
    wacc.zero();
    unsigned long long n_ovf = 0, n_fatal = 0, n_qfull = 0, n_blocks = 0;
    if (a.reset_next && blockIdx.x == 0 && threadIdx.x == 0) *a.reset_next = 0ull;   // next step's tail counter
    // queue acquisition state (lane 0): static interleaved positions, then the
    // cross-GPU tail `grab` positions per atomic
    bool tail = false;
    uint64_t tcur = 0, tend = 0;
    unsigned long long rbits = 0, rword = 0;     // replay: the bitmap word being drained
    for (;;) {
        if (a.stop_on_cell && *(volatile unsigned long long *)a.cells_cnt > 0) break;
        unsigned long long pos = ~0ull;
        if (lane == 0) {
            if (a.replay) {
                while (rbits == 0) {
                    rword = atomicAdd(a.counter, 1ull);
                    if (rword >= a.ovf_words) break;
                    rbits = a.replay_bits[rword];
                    if (rbits) a.replay_bits[rword] = 0ull;   // clean for the next step
                }
                if (rbits) {
                    pos = rword * 64 + (unsigned long long)(__ffsll((long long)rbits) - 1);
                    rbits &= rbits - 1;
                }
            } else {
                if (!tail) {
                    const unsigned long long i = atomicAdd(a.counter, 1ull);
                    const uint64_t p = (uint64_t)a.rank + i * (uint64_t)a.world;
                    if (p < a.n_static) pos = p;
                    else tail = true;
                }
                if (tail && a.gcounter) {
                    if (tcur >= tend) {
                        const unsigned long long g = a.system_counter ? atomicAdd_system(a.gcounter, a.grab)
                                                                      : atomicAdd(a.gcounter, a.grab);
                        tcur = a.n_static + g;
                        tend = min(tcur + a.grab, a.n_items);
                    }
                    if (tcur < tend) pos = tcur++;
                }
            }
        }
        pos = __shfl_sync(FULL, pos, 0);
        if (pos == ~0ull) break;
        int mytop = 0;
        const int D = decode_item(pos, a, cx, mytop);
        Acc bacc;
        bacc.zero();
        bool ovf = false;
        process_item<TIER, NPL, S, R>(D, mytop, Lsm, scr, cx, bacc, ovf);
        ovf = __any_sync(FULL, ovf);
        ++n_blocks;
        if (ovf) {
            // the item is redone by the next tier: narrow -> tier 2 -> tier 4 (int128)
            if ((pos >> 6) < a.ovf_words) {
                if (TIER != 2) ++n_ovf;
                else ++n_fatal;
                if (lane == 0) atomicOr(a.mark_bits + (pos >> 6), 1ull << (pos & 63));
            } else {
                ++n_qfull;                       // beyond the bitmap: the host redoes the space
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
        w[SLOT_FATAL] = 0;
        w[SLOT_QFULL] = n_qfull;
        w[SLOT_BLOCKS] = n_blocks;
        w[SLOT_UPDATES] = wacc.updates;
        w[SLOT_LEAVES] = wacc.leaves;
        w[14] = wacc.dead;
        w[SLOT_WIDE] = n_fatal;            // tier 2 -> tier 4 hand-offs
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

typedef void (*KernFn)(LaunchArgs);
// per-tier kernel selection (bdeg_enum_t<T>.cu): R = rank-range launch (mode 0)
KernFn pick_t0(int npl, int S, bool ranged);
KernFn pick_t1(int npl, int S, bool ranged);
KernFn pick_t2(int npl, int S, bool ranged);
KernFn pick_t3(int npl, int S, bool ranged);

}  // namespace bdeg
