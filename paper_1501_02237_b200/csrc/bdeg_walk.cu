// libbdeg device code: output-sensitive enumeration of the
// regular subdivision by walking its cells (§4.2 "pivoting",
// P:969-1039, and the graph view of §4.3), on B200.
//
// The paper pivots with LP phase one in floating point.  Here a pivot is the
// exact warp-wide ridge test of the enumeration kernel: for a cell C and a
// point p of C, the ridge R = C \ {p} (K-1 points) is eliminated
// (fraction-free, Bareiss, shared-memory scratch, int64 values / int128
// products), every point l reduces to (x_l, y_l), and the cells containing R
// are the extreme slopes of the half-planes x > 0 and x < 0 (the same
// Sylvester-identity test as bdeg_kernels.cu).  C is one of them; the other,
// if any, is the neighbour across R.  The dual graph of a triangulation of a
// convex polytope is connected, so a breadth-first walk from one cell
// (P:1117-1125 FIFO) reaches every cell exactly once; discovered cells are
// deduplicated in an open-addressing hash set of 64-bit point masks (the
// paper's KnownNodes, without collisions: full keys).
// Volumes are computed at the end, one exact determinant per cell.
#include "bdeg_internal.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

namespace bdeg {
namespace walk {

constexpr unsigned FULL = 0xffffffffu;
constexpr int kWarps = 4;

struct Div {
    uint64_t inv;
    int64_t d;
    int tz, unit;
};

__device__ __forceinline__ Div make_div(int64_t d) {
    Div r;
    r.d = d;
    r.unit = (d == 1) ? 1 : (d == -1 ? -1 : 0);
    r.tz = 0;
    r.inv = 1;
    if (r.unit == 0) {
        r.tz = __ffsll(d) - 1;
        const uint64_t o = (uint64_t)(d >> r.tz);
        uint64_t x = (3 * o) ^ 2;
#pragma unroll
        for (int i = 0; i < 4; ++i) x *= 2 - o * x;
        r.inv = x;
    }
    return r;
}

// exact quotient of a Bareiss numerator, verified; |q| < 2^62
__device__ __forceinline__ int64_t qdiv(i128 num, const Div &dv, bool &ovf) {
    int64_t q;
    if (dv.unit != 0) {
        const i128 t = dv.unit > 0 ? num : -num;
        q = (int64_t)t;
        ovf |= (i128)q != t;
    } else {
        q = (int64_t)((uint64_t)(num >> dv.tz) * dv.inv);
        ovf |= (i128)q * (i128)dv.d != num;
    }
    const int64_t lim = (int64_t)1 << 62;
    ovf |= q >= lim || q <= -lim;
    return q;
}

__device__ __forceinline__ uint32_t ford(float f) {
    uint32_t b = __float_as_uint(f);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

__device__ __forceinline__ uint64_t mix64(uint64_t z) {   // SplitMix64 finaliser as hash
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// t-th set bit (t >= 0) of a 64-bit mask
__device__ __forceinline__ int nth_bit(uint64_t m, int t) {
    const uint32_t lo = (uint32_t)m, hi = (uint32_t)(m >> 32);
    const int pl = __popc(lo);
    return t < pl ? (int)__fns(lo, 0, t + 1) : 32 + (int)__fns(hi, 0, t + 1 - pl);
}

// Cell / ridge masks over up to 128 points (bit l = point l).
struct M128 {
    uint64_t lo, hi;
};
__device__ __forceinline__ bool mbit(const M128 &m, int l) {
    return ((l < 64 ? m.lo >> l : m.hi >> (l - 64)) & 1ull) != 0;
}
__device__ __forceinline__ M128 mclear(M128 m, int l) {
    if (l < 64) m.lo &= ~(1ull << l); else m.hi &= ~(1ull << (l - 64));
    return m;
}
__device__ __forceinline__ M128 mset(M128 m, int l) {
    if (l < 64) m.lo |= 1ull << l; else m.hi |= 1ull << (l - 64);
    return m;
}
__device__ __forceinline__ int mpopc(const M128 &m) { return __popcll(m.lo) + __popcll(m.hi); }
__device__ __forceinline__ int mnth(const M128 &m, int t) {
    const int pl = __popcll(m.lo);
    return t < pl ? nth_bit(m.lo, t) : 64 + nth_bit(m.hi, t - pl);
}
__device__ __forceinline__ int mtop(const M128 &m) {
    return m.hi ? 127 - __clzll((long long)m.hi) : 63 - __clzll((long long)m.lo);
}
__device__ __forceinline__ uint64_t mhash(const M128 &m) { return mix64(m.lo ^ mix64(m.hi + 0x9E3779B97F4A7C15ull)); }

// 128-bit compare-and-swap (sm_90+: ATOMG.E.CAS.128)
__device__ __forceinline__ M128 cas128(M128 *addr, M128 cmp, M128 val) {
    M128 old;
    asm volatile("{\n\t.reg .b128 c, n, o;\n\t"
                 "mov.b128 c, {%2, %3};\n\t"
                 "mov.b128 n, {%4, %5};\n\t"
                 "atom.global.cas.b128 o, [%6], c, n;\n\t"
                 "mov.b128 {%0, %1}, o;\n\t}"
                 : "=l"(old.lo), "=l"(old.hi)
                 : "l"(cmp.lo), "l"(cmp.hi), "l"(val.lo), "l"(val.hi), "l"(addr)
                 : "memory");
    return old;
}

__device__ __forceinline__ int64_t qdiv64(int64_t num, const Div &dv) {
    if (dv.unit == 1) return num;
    if (dv.unit == -1) return -num;
    return (int64_t)((uint64_t)(num >> dv.tz) * dv.inv);
}
__device__ __forceinline__ bool inside(int64_t v, int64_t lim) {
    return (uint64_t)(v + (lim - 1)) <= (uint64_t)(2 * (lim - 1));
}
// exact quotient known (from |num| < L |d|) to satisfy |q| < L <= 2^31
__device__ __forceinline__ int32_t qdiv32u(int64_t num, const Div &dv) {
    if (dv.unit != 0) return (int32_t)(dv.unit > 0 ? num : -num);
    return (int32_t)((uint32_t)(num >> dv.tz) * (uint32_t)dv.inv);
}

// Eliminate the pivot columns of `piv_mask` (ascending order) from the lifted
// matrix in the warp's scratch scr[i*NP + l] (rows 0..K, K = lift row).
// Afterwards the single alive V row is *vrow; values are the true minors.
// WIDE = false: int64 numerators, every stored value checked against
// |V| < limV, |lift| < limL (limV * limL <= 2^61, limV^2 <= 2^61: numerators
// exact) — ovf set if a value leaves the bounds; WIDE = true: int128
// numerators, quotients verified, |v| < 2^62.
// Returns false if the pivots are linearly dependent.
template <int NPL, bool WIDE>
__device__ bool eliminate(const int64_t *Lsm, int64_t *scr, int K, int N, M128 piv_mask, int lane,
                          int *vrow, int64_t *last_piv, bool &ovf, int64_t limV, int64_t limL) {
    constexpr int NP = 32 * NPL;
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
    const int T = mpopc(piv_mask);
    for (int t = 0; t < T; ++t) {
        const int p = mnth(piv_mask, t);
        const bool nz = lane < K && ((alive >> lane) & 1ull) && scr[lane * NP + p] != 0;
        const unsigned bal = __ballot_sync(FULL, nz);
        if (bal == 0) return false;
        const int r = __ffs(bal) - 1;
        const int64_t piv = scr[r * NP + p];
        const Div dv = make_div(prev);
        int64_t prow[NPL];
#pragma unroll
        for (int q = 0; q < NPL; ++q) prow[q] = scr[r * NP + lane + 32 * q];
        for (int i = 0; i <= K; ++i) {
            if (i == r || (i < K && !((alive >> i) & 1ull))) continue;
            const int64_t ci = scr[i * NP + p];
            const int64_t lim = i < K ? limV : limL;
#pragma unroll
            for (int q = 0; q < NPL; ++q) {
                const int l = lane + 32 * q;
                if (l == p) continue;
                if constexpr (WIDE) {
                    scr[i * NP + l] = qdiv((i128)piv * scr[i * NP + l] - (i128)ci * prow[q], dv, ovf);
                } else {
                    const int64_t v = qdiv64(piv * scr[i * NP + l] - ci * prow[q], dv);
                    ovf |= !inside(v, lim);
                    scr[i * NP + l] = v;
                }
            }
        }
        alive &= ~(1ull << r);
        prev = piv;
        __syncwarp();
        if constexpr (!WIDE) {
            if (__any_sync(FULL, ovf)) return true;       // caller redoes it wide
        }
    }
    *vrow = __ffsll((long long)alive) - 1;
    *last_piv = prev;
    return true;
}

template <int NPL>
__device__ __forceinline__ bool eliminate_auto(const int64_t *Lsm, int64_t *scr, int K, int N, M128 piv_mask,
                                               int lane, int *vrow, int64_t *last_piv, bool &ovf, int64_t limV,
                                               int64_t limL) {
    if (limV > 0) {
        bool o = false;
        const bool ok = eliminate<NPL, false>(Lsm, scr, K, N, piv_mask, lane, vrow, last_piv, o, limV, limL);
        if (!__any_sync(FULL, o)) return ok;
    }
    return eliminate<NPL, true>(Lsm, scr, K, N, piv_mask, lane, vrow, last_piv, ovf, 0, 0);
}

struct WalkArgs {
    const int64_t *L;             // lifted matrix, column-major (K+1) x N
    int K, N;
    const M128 *cur;                  // frontier (cell masks)
    uint64_t ncur;
    M128 *next;                       // next frontier
    unsigned long long *next_cnt;
    M128 *table;                      // hash set of cell masks ({0,0} = empty)
    uint64_t cap;                     // power of two
    uint8_t *tags;                    // per-slot level tag (mod 256)
    uint8_t tag;                      // tag of the next level's cells
    uint64_t next_cap;                // capacity of `next`
    unsigned long long *counter;      // work counter
    int64_t limV, limL;               // int64 fast-path bounds (0: always int128)
    int narrow;                       // D&C walk with int32 storage (tier-0 plans)
    int vsafe;                        // V-minors < 2^31 by Hadamard (host): no V-row range checks
    M128 *ovfl;                       // narrow: cells that left int32 (redone in int64)
    unsigned long long *ovfl_cnt;
    uint64_t ovfl_cap;
    unsigned long long *vol;          // D&C walk: [4 limbs of sum |det|, cells] of this level
    unsigned long long *stats;        // [0] ridges tested, [1] ties, [2] inconsistent,
                                      // [3] table full, [4] overflow, [5] boundary ridges,
                                      // [6] cells redone with int128 numerators (D&C walk)
    int grid;
    void *stream;
    // sharded walk: the hash set is split over `world` ranks,
    // cell m is owned by rank owner(m); neighbours owned elsewhere are
    // appended to `remote` and exchanged after the level (all-to-all)
    int world, rank;
    M128 *remote;
    unsigned long long *remote_cnt;
    uint64_t remote_cap;
};

// owner rank of a cell (low half of the hash; the table slot uses the high half)
__device__ __forceinline__ int owner_of(const M128 &m, int world) {
    return (int)((uint32_t)mhash(m) % (uint32_t)world);
}

// Insert key (linear probing); true if it was new.  tags (optional): the
// slot's walk level (mod 256) is recorded beside it, so a level's cells can be
// re-collected from the table (frontier overflow).
__device__ __forceinline__ bool insert(M128 *table, uint64_t cap, M128 key, bool &full,
                                       uint8_t *tags = nullptr, uint8_t tag = 0) {
    uint64_t h = __umul64hi(mhash(key), cap);            // any table size (range reduction)
    const M128 empty = {0, 0};
    const uint64_t max_probe = cap < 4096 ? cap : 4096;   // load <= 3/4: short probes
    for (uint64_t probe = 0; probe < max_probe; ++probe) {
        const M128 old = cas128(table + h, empty, key);
        if (old.lo == 0 && old.hi == 0) {
            if (tags) tags[h] = tag;
            return true;
        }
        if (old.lo == key.lo && old.hi == key.hi) return false;
        h = (h + 1 == cap) ? 0 : h + 1;
    }
    full = true;
    return false;
}

// One pivot: cell `m`, drop its t-th point p, find the neighbour across the
// ridge R = m \ {p}.
template <int NPL>
__global__ void __launch_bounds__(kWarps * 32) k_walk(WalkArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int K = a.K, N = a.N;
    int64_t *Lsm = reinterpret_cast<int64_t *>(smem);
    const int lsz = (K + 1) * N;
    for (int i = threadIdx.x; i < lsz; i += blockDim.x) Lsm[i] = a.L[i];
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int NP = 32 * NPL;
    int64_t *scr = reinterpret_cast<int64_t *>(smem + ((lsz * 8 + 15) & ~15)) + (size_t)warp * (K + 1) * NP;
    unsigned long long st[6] = {0, 0, 0, 0, 0, 0};
    const uint64_t nwork = a.ncur * (uint64_t)K;
    for (;;) {
        unsigned long long idx = 0;
        if (lane == 0) idx = atomicAdd(a.counter, 1ull);
        idx = __shfl_sync(FULL, idx, 0);
        if (idx >= nwork) break;
        const M128 m = a.cur[idx / K];
        const int p = mnth(m, (int)(idx % K));
        const M128 ridge = mclear(m, p);
        bool ovf = false;
        int vr = 0;
        int64_t g = 1;
        ++st[0];
        if (!eliminate_auto<NPL>(Lsm, scr, K, N, ridge, lane, &vr, &g, ovf, a.limV, a.limL)) { ++st[2]; continue; }
        int64_t x[NPL], yk[NPL];
        bool valid[NPL];
        const int kappa = g > 0 ? 1 : -1;
#pragma unroll
        for (int q = 0; q < NPL; ++q) {
            const int l = lane + 32 * q;
            x[q] = scr[vr * NP + l];
            yk[q] = kappa > 0 ? scr[K * NP + l] : -scr[K * NP + l];
            valid[q] = l < N && !mbit(ridge, l);
        }
        if (__any_sync(FULL, ovf)) { ++st[4]; continue; }
        // side of the current cell's point p; the neighbour is on the other side
        int64_t xps = x[0];
#pragma unroll
        for (int q = 1; q < NPL; ++q) if ((p >> 5) == q) xps = x[q];
        const int64_t xp = __shfl_sync(FULL, (long long)xps, p & 31);
        if (xp == 0) { ++st[2]; continue; }
        const bool want_pos = xp < 0;
        // points of span(R) strictly below: R is no lower ridge -> inconsistent
        bool bad0 = false;
        uint32_t kk = 0xFFFFFFFFu;
        uint32_t key[NPL];
#pragma unroll
        for (int q = 0; q < NPL; ++q) {
            bad0 |= valid[q] && x[q] == 0 && yk[q] < 0;
            const uint32_t o = ford(__fdividef((float)yk[q], (float)x[q]));
            key[q] = want_pos ? o : ~o;          // min slope (x > 0) or max slope (x < 0)
            const bool side = want_pos ? x[q] > 0 : x[q] < 0;
            if (valid[q] && side) kk = min(kk, key[q]);
        }
        if (__any_sync(FULL, bad0)) { ++st[2]; continue; }
        const uint32_t mk = __reduce_min_sync(FULL, kk);
        if (mk == 0xFFFFFFFFu) { ++st[5]; continue; }      // boundary ridge
        uint32_t cand[NPL];
#pragma unroll
        for (int q = 0; q < NPL; ++q) {
            const bool side = want_pos ? x[q] > 0 : x[q] < 0;
            cand[q] = __ballot_sync(FULL, valid[q] && side && key[q] <= mk + 64u);
        }
        int found = -1;
        bool tie = false;
        for (int cq = 0; cq < NPL; ++cq)
        while (cand[cq]) {
            const int j = 32 * cq + __ffs(cand[cq]) - 1;
            cand[cq] &= cand[cq] - 1;
            int64_t xs = x[0], ys = yk[0];
#pragma unroll
            for (int q = 1; q < NPL; ++q) if ((j >> 5) == q) { xs = x[q]; ys = yk[q]; }
            const int64_t xj = __shfl_sync(FULL, (long long)xs, j & 31);
            const int64_t yj = __shfl_sync(FULL, (long long)ys, j & 31);
            bool bad = false, zero = false;
#pragma unroll
            for (int q = 0; q < NPL; ++q) {
                const int l = lane + 32 * q;
                if (valid[q] && l != j) {
                    i128 c = (i128)xj * yk[q] - (i128)x[q] * yj;
                    if (xj < 0) c = -c;
                    bad |= c < 0;
                    zero |= c == 0;
                }
            }
            if (__any_sync(FULL, bad)) continue;
            if (__any_sync(FULL, zero)) { tie = true; continue; }
            found = j;
        }
        if (tie) ++st[1];
        if (found < 0) { if (!tie) ++st[5]; continue; }
        if (lane == 0) {
            const M128 nm = mset(ridge, found);
            bool full = false;
            if (a.world > 1 && owner_of(nm, a.world) != a.rank) {
                const unsigned long long pos = atomicAdd(a.remote_cnt, 1ull);
                if (pos < a.remote_cap) a.remote[pos] = nm;
            } else if (insert(a.table, a.cap, nm, full, a.tags, a.tag)) {
                const unsigned long long pos = atomicAdd(a.next_cnt, 1ull);
                if (pos < a.next_cap) a.next[pos] = nm;   // else re-collected by tag
            }
            if (full) ++st[3];
        }
    }
    if (lane == 0)
        for (int i = 0; i < 6; ++i)
            if (st[i]) atomicAdd(a.stats + i, st[i]);
}

// ------------------------------------------------------------------------
// Divide-and-conquer leave-one-out elimination (one warp per cell).  A node
// holds the cell's points [a, b) still to be eliminated, in a row-compacted
// buffer whose other K - (b - a) cell points are eliminated; its children
// eliminate one half and recurse into the other.  The K leaves are the K
// ridges; total pivot steps O(K log K) instead of O(K^2) from scratch.
// Buffers: rows [0, R-1) are the alive V rows, row R-1 the lift row.

// ridge test on a 2-row state (x = remaining V row, y = lift row); inserts the
// neighbour across the ridge (cell minus p) into the hash set / next frontier
template <int NPL, typename T>
__device__ __forceinline__ int64_t ridge_step(const T *bx, const T *by, int64_t g, M128 ridge, int p,
                                           int N, int lane, const WalkArgs &a, unsigned long long (&st)[6],
                                           int &nb) {
    nb = -1;
    int64_t x[NPL], yk[NPL];
    bool valid[NPL];
    const int kappa = g > 0 ? 1 : -1;
#pragma unroll
    for (int q = 0; q < NPL; ++q) {
        const int l = lane + 32 * q;
        x[q] = (int64_t)bx[l];
        yk[q] = kappa > 0 ? (int64_t)by[l] : -(int64_t)by[l];
        valid[q] = l < N && !mbit(ridge, l);
    }
    ++st[0];
    int64_t xps = x[0];
#pragma unroll
    for (int q = 1; q < NPL; ++q) if ((p >> 5) == q) xps = x[q];
    const int64_t xp = __shfl_sync(FULL, (long long)xps, p & 31);
    if (xp == 0) { ++st[2]; return 0; }
    const bool want_pos = xp < 0;                 // the neighbour is on the other side
    bool bad0 = false;
    uint32_t kk = 0xFFFFFFFFu;
    uint32_t key[NPL];
#pragma unroll
    for (int q = 0; q < NPL; ++q) {
        bad0 |= valid[q] && x[q] == 0 && yk[q] < 0;
        const uint32_t o = ford(__fdividef((float)yk[q], (float)x[q]));
        key[q] = want_pos ? o : ~o;
        const bool side = want_pos ? x[q] > 0 : x[q] < 0;
        if (valid[q] && side) kk = min(kk, key[q]);
    }
    if (__any_sync(FULL, bad0)) { ++st[2]; return xp; }
    const uint32_t mk = __reduce_min_sync(FULL, kk);
    if (mk == 0xFFFFFFFFu) { ++st[5]; return xp; }          // boundary ridge
    int found = -1;
    bool tie = false;
#pragma unroll
    for (int cq = 0; cq < NPL; ++cq) {
        const bool side = want_pos ? x[cq] > 0 : x[cq] < 0;
        uint32_t cand = __ballot_sync(FULL, valid[cq] && side && key[cq] <= mk + 64u);
        while (cand) {
            const int j = 32 * cq + __ffs(cand) - 1;
            cand &= cand - 1;
            const int64_t xj = __shfl_sync(FULL, (long long)x[cq], j & 31);
            const int64_t yj = __shfl_sync(FULL, (long long)yk[cq], j & 31);
            bool bad = false, zero = false;
#pragma unroll
            for (int q = 0; q < NPL; ++q) {
                const int l = lane + 32 * q;
                if (valid[q] && l != j) {
                    i128 c = (i128)xj * yk[q] - (i128)x[q] * yj;
                    if (xj < 0) c = -c;
                    bad |= c < 0;
                    zero |= c == 0;
                }
            }
            if (__any_sync(FULL, bad)) continue;
            if (__any_sync(FULL, zero)) { tie = true; continue; }
            found = j;
        }
    }
    if (tie) ++st[1];
    if (found < 0) { if (!tie) ++st[5]; return xp; }
    nb = found;                                   // inserted by dc_cell, batched per cell
    return xp;
}

// Insert the neighbours found by a cell's ridge tests, one per lane (lane t
// holds ridge t's neighbour point, or -1): up to K concurrent 128-bit CAS
// probes instead of K serial ones, and one warp-aggregated frontier append.
__device__ __forceinline__ void insert_neighbours(M128 m, int my_p, int my_nb, int lane, const WalkArgs &a,
                                                  unsigned long long (&st)[6]) {
    bool isnew = false, full = false, isremote = false;
    M128 nm = {0, 0};
    if (my_nb >= 0) {
        nm = mset(mclear(m, my_p), my_nb);
        if (a.world > 1 && owner_of(nm, a.world) != a.rank) isremote = true;
        else isnew = insert(a.table, a.cap, nm, full, a.tags, a.tag);
    }
    const unsigned rmask = __ballot_sync(FULL, isremote);
    if (rmask) {                                  // owned by another rank: exchanged after the level
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(a.remote_cnt, (unsigned long long)__popc(rmask));
        base = __shfl_sync(FULL, base, 0);
        if (isremote) {
            const unsigned long long pos = base + __popc(rmask & ((1u << lane) - 1));
            if (pos < a.remote_cap) a.remote[pos] = nm;
        }
    }
    const unsigned nmask = __ballot_sync(FULL, isnew);
    if (nmask) {
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(a.next_cnt, (unsigned long long)__popc(nmask));
        base = __shfl_sync(FULL, base, 0);
        if (isnew) {
            const unsigned long long pos = base + __popc(nmask & ((1u << lane) - 1));
            if (pos < a.next_cap) a.next[pos] = nm;   // else re-collected by tag
        }
    }
    st[3] += __popc(__ballot_sync(FULL, full));
}

// Eliminate pivot column p: rows of src (R rows, V rows [0, R-1), lift row
// R-1) -> dst with R-1 rows, row-compacted (the last V row takes the pivot
// row's slot, the lift row moves down one).  src == dst is allowed: each lane
// touches only its own columns, column p's multipliers are read up front and
// rows are visited in increasing order.  Column p is written too (it becomes
// exactly 0): stale values there would feed later steps' inexact divisions
// and raise false overflow flags.  R <= 32.
// T = int32_t (narrow, tier-0 plans): int32 storage, int64 numerators; the
// range check is on the numerator, |num| < L |prev| <=> |quotient| < L, so
// no multiply-back is needed (L = limV for V rows, limL for the lift row).
template <int NPL, bool WIDE, typename T = int64_t, bool VSAFE = false>
__device__ __forceinline__ bool dc_eliminate(const T *src, T *dst, int &R, int p, int64_t &prev,
                                             int lane, bool &ovf, int64_t limV, int64_t limL) {
    constexpr int NP = 32 * NPL;
    constexpr bool NARROW = sizeof(T) == 4;
    __syncwarp();
    const T cl = lane < R ? src[lane * NP + p] : 0;
    const unsigned bal = __ballot_sync(FULL, lane < R - 1 && cl != 0);
    if (bal == 0) return false;
    const int r = __ffs(bal) - 1;
    const Div dv = make_div(prev);
    T prow[NPL];
#pragma unroll
    for (int q = 0; q < NPL; ++q) prow[q] = src[r * NP + lane + 32 * q];
    if constexpr (NARROW) {
        const int32_t piv = __shfl_sync(FULL, (int32_t)cl, r);
        const int64_t ap = prev < 0 ? -prev : prev;
        const int64_t bV = limV * ap, bL = limL * ap;
        // branch-free exact quotient: for d = +-1, tz = 0 and inv = d^-1 = d
        const int tz = dv.unit != 0 ? 0 : dv.tz;
        const uint32_t inv = dv.unit > 0 ? 1u : (dv.unit < 0 ? 0xFFFFFFFFu : (uint32_t)dv.inv);
        __syncwarp();
        // rows in increasing order (in place: see above); V rows keep their slot
        // except the last one, which takes the pivot row's; the lift row moves
        // to R-2 — no per-row selects in the loops
        auto row = [&](int i, int o, int64_t b, bool chk) {
            const int32_t ci = __shfl_sync(FULL, (int32_t)cl, i);
            const int64_t b1 = b - 1, b2 = 2 * (b - 1);
#pragma unroll
            for (int q = 0; q < NPL; ++q) {
                const int l = lane + 32 * q;
                const int64_t num = (int64_t)piv * (int64_t)src[i * NP + l] - (int64_t)ci * (int64_t)prow[q];
                if (chk) ovf |= (uint64_t)(num + b1) > (uint64_t)b2;
                dst[o * NP + l] = (int32_t)((uint32_t)(num >> tz) * inv);
            }
        };
        // V rows need no check when Hadamard bounds every V-minor below 2^31
        const bool cv = !VSAFE;
        for (int i = 0; i < r; ++i) row(i, i, bV, cv);
        for (int i = r + 1; i < R - 2; ++i) row(i, i, bV, cv);
        if (r != R - 2) row(R - 2, r, bV, cv);
        row(R - 1, R - 2, bL, true);
        --R;
        prev = piv;
        return true;
    }
    const int64_t piv = __shfl_sync(FULL, (long long)cl, r);
    __syncwarp();   // every lane has read column p before its owner rewrites it
    // same row order and slot mapping as the narrow path, without per-row selects
    auto row = [&](int i, int o, int64_t lim) {
        const int64_t ci = __shfl_sync(FULL, (long long)cl, i);
#pragma unroll
        for (int q = 0; q < NPL; ++q) {
            const int l = lane + 32 * q;
            int64_t v;
            if constexpr (WIDE) {
                v = qdiv((i128)piv * src[i * NP + l] - (i128)ci * prow[q], dv, ovf);
            } else {
                v = qdiv64(piv * src[i * NP + l] - ci * prow[q], dv);
                ovf |= !inside(v, lim);
            }
            dst[o * NP + l] = v;
        }
    };
    for (int i = 0; i < r; ++i) row(i, i, limV);
    for (int i = r + 1; i < R - 2; ++i) row(i, i, limV);
    if (r != R - 2) row(R - 2, r, limV);
    row(R - 1, R - 2, limL);
    --R;
    prev = piv;
    return true;
}

constexpr int kDcDepth = 7;   // K <= 31: ceil(log2 31) + 1 levels

// per-depth row offsets (depth >= 1; depth 0 is the shared L) and their total
__host__ __device__ inline int dc_offsets(int K, int *roff) {
    int g = K, rows = K + 1, off = 0;
    for (int d = 0; d <= kDcDepth; ++d) {
        if (roff) roff[d] = off;
        if (d > 0) off += rows;
        rows -= g / 2;
        g = (g + 1) / 2;
        if (rows < 2) rows = 2;
    }
    return off;
}

// All K ridges of cell m; false on int64 overflow (the caller retries WIDE).
// vol = |det| of the cell (the pivot x_p of the first leaf).  Lsm: row-major
// (K+1) x NP lifted matrix = the depth-0 buffer.
template <int NPL, bool WIDE, typename T = int64_t, bool VSAFE = false>
__device__ bool dc_cell(const T *Lsm, T *bufs, const int *roff, int K, int N, M128 m, int lane,
                        const WalkArgs &a, unsigned long long (&st)[6], int64_t limV, int64_t limL,
                        uint64_t &vol) {
    constexpr int NP = 32 * NPL;
    int pts[32];                      // the cell's points, ascending
    {
        int n = 0;
        uint64_t w = m.lo;
        while (w) { pts[n++] = __ffsll((long long)w) - 1; w &= w - 1; }
        w = m.hi;
        while (w) { pts[n++] = 64 + __ffsll((long long)w) - 1; w &= w - 1; }
    }
    int A[kDcDepth], Bn[kDcDepth], stage[kDcDepth], R[kDcDepth];
    int64_t prev[kDcDepth];
    int d = 0;
    A[0] = 0; Bn[0] = K; stage[0] = 0; R[0] = K + 1; prev[0] = 1;
    bool ovf = false;
    vol = 0;
    int my_p = -1, my_nb = -1;        // lane t: ridge t's dropped point and neighbour
    while (d >= 0) {
        const T *Bd = d == 0 ? Lsm : bufs + (size_t)roff[d] * NP;
        if (Bn[d] - A[d] == 1) {
            int nb;
            const int64_t xp = ridge_step<NPL, T>(Bd, Bd + NP, prev[d], mclear(m, pts[A[d]]), pts[A[d]], N, lane,
                                                  a, st, nb);
            if (lane == A[d]) { my_p = pts[A[d]]; my_nb = nb; }
            if (A[d] == 0) vol = (uint64_t)(xp < 0 ? -xp : xp);
            --d;
            continue;
        }
        if (stage[d] == 2) { --d; continue; }
        const int mid = (A[d] + Bn[d]) / 2;
        const int e0 = stage[d] == 0 ? mid : A[d];       // eliminate [e0, e1)
        const int e1 = stage[d] == 0 ? Bn[d] : mid;
        T *C = bufs + (size_t)roff[d + 1] * NP;
        int Rc = R[d];
        int64_t pc = prev[d];
        for (int t = e0; t < e1; ++t) {
            if (!dc_eliminate<NPL, WIDE, T, VSAFE>(t == e0 ? Bd : C, C, Rc, pts[t], pc, lane, ovf, limV, limL)) {
                ++st[2];
                insert_neighbours(m, my_p, my_nb, lane, a, st);
                return true;
            }
            if (__any_sync(FULL, ovf)) return false;   // nothing inserted: the caller redoes the cell
        }
        A[d + 1] = stage[d] == 0 ? A[d] : mid;
        Bn[d + 1] = stage[d] == 0 ? mid : Bn[d];
        stage[d] += 1;
        ++d;
        stage[d] = 0;
        R[d] = Rc;
        prev[d] = pc;
    }
    insert_neighbours(m, my_p, my_nb, lane, a, st);
    return true;
}

// One warp per cell of the frontier (walk level); also sums |det| and counts
// the level's cells (each cell is in exactly one frontier).
// T = int32_t: narrow storage (tier-0 plans, values |v| < 2^30 / lifts < 2^31);
// a cell whose values leave int32 goes to a.ovfl and is redone by the int64
// kernel (neighbours it already inserted were found from checked values).
template <int NPL, typename T = int64_t, bool VSAFE = false>
__global__ void __launch_bounds__(512) k_walk_dc(WalkArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr int NP = 32 * NPL;
    constexpr bool NARROW = sizeof(T) == 4;
    const int K = a.K, N = a.N;
    T *Lsm = reinterpret_cast<T *>(smem);                           // row-major (K+1) x NP
    for (int t = threadIdx.x; t < (K + 1) * NP; t += blockDim.x) {
        const int i = t / NP, l = t - i * NP;
        Lsm[t] = l < N ? (T)a.L[(size_t)l * (K + 1) + i] : 0;
    }
    int roff[kDcDepth + 1];
    const int rows_total = dc_offsets(K, roff);
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // roff[d] for d >= 1 counts from roff[1] = 0
    T *bufs = Lsm + (size_t)(K + 1) * NP + (size_t)warp * rows_total * NP;
    unsigned long long st[6] = {0, 0, 0, 0, 0, 0};
    uint64_t lo = 0, hi = 0, cells = 0, fallbacks = 0;
    for (;;) {
        unsigned long long idx = 0;
        if (lane == 0) idx = atomicAdd(a.counter, 1ull);
        idx = __shfl_sync(FULL, idx, 0);
        if (idx >= a.ncur) break;
        const M128 m = a.cur[idx];
        uint64_t v = 0;
        if constexpr (NARROW) {
            if (!dc_cell<NPL, false, T, VSAFE>(Lsm, bufs, roff, K, N, m, lane, a, st, a.limV, a.limL, v)) {
                if (lane == 0) {
                    const unsigned long long pos = atomicAdd(a.ovfl_cnt, 1ull);
                    if (pos < a.ovfl_cap) a.ovfl[pos] = m;
                }
                continue;
            }
        } else {
            bool done = false;
            if (a.limV > 0) done = dc_cell<NPL, false>(Lsm, bufs, roff, K, N, m, lane, a, st, a.limV, a.limL, v);
            fallbacks += !done;
            if (!done && !dc_cell<NPL, true>(Lsm, bufs, roff, K, N, m, lane, a, st, 0, 0, v)) {
                ++st[4];
                continue;
            }
        }
        const uint64_t t = lo + v;
        hi += t < lo;
        lo = t;
        ++cells;
    }
    if (lane == 0) {
        for (int i = 0; i < 6; ++i)
            if (st[i]) atomicAdd(a.stats + i, st[i]);
        atomicAdd(a.vol + 0, lo & 0xFFFFFFFFull);
        atomicAdd(a.vol + 1, lo >> 32);
        atomicAdd(a.vol + 2, hi & 0xFFFFFFFFull);
        atomicAdd(a.vol + 3, hi >> 32);
        atomicAdd(a.vol + 4, cells);
        if (fallbacks) atomicAdd(a.stats + 6, fallbacks);   // cells redone in int128
    }
}

// |det| of every cell in the table (one warp per cell) into 4 limbs + count
template <int NPL>
__global__ void __launch_bounds__(kWarps * 32) k_cellvol(const int64_t *L, int K, int N,
                                                          const M128 *table, uint64_t cap,
                                                          unsigned long long *out /* [4 limbs, cells, ovf] */,
                                                          unsigned long long *counter, int64_t limV, int64_t limL) {
    extern __shared__ __align__(16) unsigned char smem[];
    int64_t *Lsm = reinterpret_cast<int64_t *>(smem);
    const int lsz = (K + 1) * N;
    for (int i = threadIdx.x; i < lsz; i += blockDim.x) Lsm[i] = L[i];
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int NP = 32 * NPL;
    int64_t *scr = reinterpret_cast<int64_t *>(smem + ((lsz * 8 + 15) & ~15)) + (size_t)warp * (K + 1) * NP;
    uint64_t lo = 0, hi = 0, cells = 0, ovfs = 0;
    const uint64_t chunk = 256;
    for (;;) {
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(counter, chunk);
        base = __shfl_sync(FULL, base, 0);
        if (base >= cap) break;
        for (uint64_t s = base; s < base + chunk && s < cap; ++s) {
            const M128 m = table[s];
            if (m.lo == 0 && m.hi == 0) continue;
            const int top = mtop(m);
            bool ovf = false;
            int vr = 0;
            int64_t g = 1;
            if (!eliminate_auto<NPL>(Lsm, scr, K, N, mclear(m, top), lane, &vr, &g, ovf, limV, limL)) {
                ++ovfs;
                continue;
            }
            const int64_t d = scr[vr * NP + top];            // +-det of the cell (column top)
            if (__any_sync(FULL, ovf)) { ++ovfs; continue; }
            const uint64_t v = (uint64_t)(d < 0 ? -d : d);
            const uint64_t t = lo + v;
            hi += t < lo;
            lo = t;
            ++cells;
        }
    }
    if (lane == 0) {
        atomicAdd(out + 0, lo & 0xFFFFFFFFull);
        atomicAdd(out + 1, lo >> 32);
        atomicAdd(out + 2, hi & 0xFFFFFFFFull);
        atomicAdd(out + 3, hi >> 32);
        atomicAdd(out + 4, cells);
        atomicAdd(out + 5, ovfs);
    }
}

// Re-insert the cells of `old` into `tab`.  keep_n > 0: only the cells of
// the keep_n consecutive levels starting at tag keep0 (mod 256) survive —
// the breadth-first window: a neighbour of a level-L cell lies in level
// L-1, L or L+1 (BFS distances of adjacent cells differ by <= 1), so older
// levels are never looked up again (the paper's hash table
// P:1134-1162 keeps every face).
__global__ void k_rehash(const M128 *old, const uint8_t *old_tags, uint64_t oldcap, M128 *tab, uint8_t *tags,
                         uint64_t cap, unsigned long long *full_flag, uint8_t keep0, int keep_n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < oldcap; i += (uint64_t)gridDim.x * blockDim.x) {
        const M128 k = old[i];
        if (k.lo == 0 && k.hi == 0) continue;
        if (keep_n > 0 && (uint8_t)(old_tags[i] - keep0) >= (unsigned)keep_n) continue;
        bool full = false;
        insert(tab, cap, k, full, tags, old_tags[i]);
        if (full) atomicAdd(full_flag, 1ull);
    }
}

// insert a list of cells (one level of the walk, tagged) into the table
__global__ void k_insert_list(const M128 *list, uint64_t n, M128 *tab, uint8_t *tags, uint64_t cap, uint8_t tag,
                              unsigned long long *full_flag) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        bool full = false;
        insert(tab, cap, list[i], full, tags, tag);
        if (full) atomicAdd(full_flag, 1ull);
    }
}

// the cells of one level (by tag) into out[0, *cnt)
__global__ void k_collect(const M128 *tab, const uint8_t *tags, uint64_t cap, uint8_t tag, M128 *out,
                          unsigned long long *cnt) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < cap; i += (uint64_t)gridDim.x * blockDim.x) {
        if (tags[i] != tag) continue;
        const M128 k = tab[i];
        if (k.lo == 0 && k.hi == 0) continue;
        out[atomicAdd(cnt, 1ull)] = k;
    }
}

// received cells (owned here): insert with the level tag, new ones join the
// next frontier (re-collected by tag if it overflows)
__global__ void k_insert_recv(const M128 *list, uint64_t n, M128 *tab, uint8_t *tags, uint64_t cap, uint8_t tag,
                              M128 *next, unsigned long long *next_cnt, uint64_t next_cap,
                              unsigned long long *full_flag) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        bool full = false;
        if (insert(tab, cap, list[i], full, tags, tag)) {
            const unsigned long long pos = atomicAdd(next_cnt, 1ull);
            if (pos < next_cap) next[pos] = list[i];
        }
        if (full) atomicAdd(full_flag, 1ull);
    }
}

// counting sort of the remote cells by owner: counts, then scatter into
// per-owner segments [off[o], off[o] + cnt[o])
__global__ void k_owner_count(const M128 *list, uint64_t n, int world, unsigned long long *cnt) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        atomicAdd(cnt + owner_of(list[i], world), 1ull);
}
__global__ void k_owner_scatter(const M128 *list, uint64_t n, int world, unsigned long long *cursor, M128 *out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        out[atomicAdd(cursor + owner_of(list[i], world), 1ull)] = list[i];
}

}  // namespace walk

int launch_insert_recv(const void *list, uint64_t n, void *tab, uint8_t *tags, uint64_t cap, uint8_t tag, void *next,
                       unsigned long long *next_cnt, uint64_t next_cap, unsigned long long *full_flag, void *stream) {
    if (n == 0) return 0;
    const int grid = (int)std::min<uint64_t>((n + 255) / 256, 4096);
    walk::k_insert_recv<<<grid, 256, 0, (cudaStream_t)stream>>>((const walk::M128 *)list, n, (walk::M128 *)tab, tags,
                                                                cap, tag, (walk::M128 *)next, next_cnt, next_cap,
                                                                full_flag);
    launch_counter_add(1);
    return (int)cudaGetLastError();
}

int launch_owner_count(const void *list, uint64_t n, int world, unsigned long long *cnt, void *stream) {
    if (n == 0) return 0;
    const int grid = (int)std::min<uint64_t>((n + 255) / 256, 4096);
    walk::k_owner_count<<<grid, 256, 0, (cudaStream_t)stream>>>((const walk::M128 *)list, n, world, cnt);
    launch_counter_add(1);
    return (int)cudaGetLastError();
}

int launch_owner_scatter(const void *list, uint64_t n, int world, unsigned long long *cursor, void *out,
                         void *stream) {
    if (n == 0) return 0;
    const int grid = (int)std::min<uint64_t>((n + 255) / 256, 4096);
    walk::k_owner_scatter<<<grid, 256, 0, (cudaStream_t)stream>>>((const walk::M128 *)list, n, world, cursor,
                                                                  (walk::M128 *)out);
    launch_counter_add(1);
    return (int)cudaGetLastError();
}

// host copy of the device hash of a 128-bit cell mask (for seeding the table)
static uint64_t hmix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
uint64_t walk_hash(uint64_t lo, uint64_t hi) { return hmix(lo ^ hmix(hi + 0x9E3779B97F4A7C15ull)); }

int launch_rehash(const void *old, const uint8_t *old_tags, uint64_t oldcap, void *tab, uint8_t *tags, uint64_t cap,
                  unsigned long long *full_flag, void *stream, uint8_t keep0, int keep_n) {
    walk::k_rehash<<<1184, 256, 0, (cudaStream_t)stream>>>((const walk::M128 *)old, old_tags, oldcap,
                                                           (walk::M128 *)tab, tags, cap, full_flag, keep0, keep_n);
    launch_counter_add(1);
    return (int)cudaGetLastError();
}

int launch_insert_list(const void *list, uint64_t n, void *tab, uint8_t *tags, uint64_t cap, uint8_t tag,
                       unsigned long long *full_flag, void *stream) {
    if (n == 0) return 0;
    walk::k_insert_list<<<1184, 256, 0, (cudaStream_t)stream>>>((const walk::M128 *)list, n, (walk::M128 *)tab,
                                                                tags, cap, tag, full_flag);
    launch_counter_add(1);
    return (int)cudaGetLastError();
}

int launch_collect(const void *tab, const uint8_t *tags, uint64_t cap, uint8_t tag, void *out,
                   unsigned long long *cnt, void *stream) {
    walk::k_collect<<<1184, 256, 0, (cudaStream_t)stream>>>((const walk::M128 *)tab, tags, cap, tag,
                                                            (walk::M128 *)out, cnt);
    launch_counter_add(1);
    return (int)cudaGetLastError();
}

static int npl_of(int N) { return (N + 31) / 32; }

size_t walk_smem_bytes(int K, int N) {
    return (((size_t)(K + 1) * N * 8 + 15) & ~(size_t)15) + (size_t)walk::kWarps * (K + 1) * 32 * npl_of(N) * 8;
}

// D&C walk kernel when it fits (K <= 31, >= 2 warps' buffers in shared
// memory); *fused = 1 then (the launch also summed the level's volumes).
template <int NPL>
static int walk_npl(const walk::WalkArgs &a, int grid, size_t smem, int *fused) {
    if (a.narrow && a.K <= 31 && !std::getenv("BDEG_WALK_SCRATCH")) {
        const size_t lb = (size_t)(a.K + 1) * 32 * NPL * 4;
        const size_t pw = (size_t)walk::dc_offsets(a.K, nullptr) * 32 * NPL * 4;
        const size_t budget = 227 * 1024;
        const int nw = lb + pw > budget ? 0 : (int)std::min<size_t>(16, (budget - lb) / pw);
        if (nw >= 2) {
            const size_t dsmem = lb + (size_t)nw * pw;
            auto kern = a.vsafe ? walk::k_walk_dc<NPL, int32_t, true> : walk::k_walk_dc<NPL, int32_t, false>;
            cudaError_t e = cudaFuncSetAttribute((const void *)kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)dsmem);
            if (e != cudaSuccess) return (int)e;
            int dev = 0, sms = 148;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            const int per_sm = std::max<int>(1, (int)((228 * 1024) / (dsmem + 1024)));
            kern<<<sms * per_sm, nw * 32, dsmem, (cudaStream_t)a.stream>>>(a);
            *fused = 2;
            return (int)cudaGetLastError();
        }
    }
    const size_t lbytes = (size_t)(a.K + 1) * 32 * NPL * 8;
    const size_t per_warp = (size_t)walk::dc_offsets(a.K, nullptr) * 32 * NPL * 8;
    const size_t budget = 227 * 1024;
    const int nw = lbytes + per_warp > budget ? 0 : (int)std::min<size_t>(16, (budget - lbytes) / per_warp);
    *fused = 0;
    // per-ridge elimination from scratch: A/B reference, K > 31, or buffers beyond smem
    if (std::getenv("BDEG_WALK_SCRATCH") || a.K > 31 || nw < 2) {
        cudaError_t e = cudaFuncSetAttribute((const void *)walk::k_walk<NPL>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return (int)e;
        walk::k_walk<NPL><<<grid, walk::kWarps * 32, smem, (cudaStream_t)a.stream>>>(a);
        return (int)cudaGetLastError();
    }
    const size_t dsmem = lbytes + (size_t)nw * per_warp;
    cudaError_t e = cudaFuncSetAttribute((const void *)walk::k_walk_dc<NPL>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsmem);
    if (e != cudaSuccess) return (int)e;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int per_sm = std::max<int>(1, (int)((228 * 1024) / (dsmem + 1024)));
    walk::k_walk_dc<NPL><<<sms * per_sm, nw * 32, dsmem, (cudaStream_t)a.stream>>>(a);
    *fused = 1;
    return (int)cudaGetLastError();
}

int launch_walk(const int64_t *L, int K, int N, const void *cur, uint64_t ncur, void *next,
                unsigned long long *next_cnt, void *table, uint64_t cap, unsigned long long *counter,
                unsigned long long *stats, int grid, void *stream, int64_t limV, int64_t limL,
                unsigned long long *vol, int *fused, uint8_t *tags, unsigned tag, uint64_t next_cap,
                int narrow, void *ovfl, unsigned long long *ovfl_cnt, uint64_t ovfl_cap, int vsafe,
                int world, int rank, void *remote, unsigned long long *remote_cnt, uint64_t remote_cap) {
    walk::WalkArgs a;
    a.world = world;
    a.rank = rank;
    a.remote = (walk::M128 *)remote;
    a.remote_cnt = remote_cnt;
    a.remote_cap = remote_cap;
    a.narrow = narrow;
    a.vsafe = vsafe;
    a.ovfl = (walk::M128 *)ovfl;
    a.ovfl_cnt = ovfl_cnt;
    a.ovfl_cap = ovfl_cap;
    a.vol = vol;
    a.tags = tags;
    a.tag = (uint8_t)tag;
    a.next_cap = next_cap;
    a.limV = limV;
    a.limL = limL;
    a.L = L; a.K = K; a.N = N; a.cur = (const walk::M128 *)cur; a.ncur = ncur; a.next = (walk::M128 *)next;
    a.next_cnt = next_cnt; a.table = (walk::M128 *)table; a.cap = cap; a.counter = counter; a.stats = stats;
    a.grid = grid; a.stream = stream;
    const size_t smem = walk_smem_bytes(K, N);
    int rc;
    switch (npl_of(N)) {
        case 1: rc = walk_npl<1>(a, grid, smem, fused); break;
        case 2: rc = walk_npl<2>(a, grid, smem, fused); break;
        case 3: rc = walk_npl<3>(a, grid, smem, fused); break;
        default: rc = walk_npl<4>(a, grid, smem, fused); break;
    }
    launch_counter_add(1);
    return rc;
}

template <int NPL>
static int cellvol_npl(const int64_t *L, int K, int N, const void *table, uint64_t cap, unsigned long long *out,
                       unsigned long long *counter, int grid, void *stream, int64_t limV, int64_t limL, size_t smem) {
    cudaError_t e = cudaFuncSetAttribute((const void *)walk::k_cellvol<NPL>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return (int)e;
    walk::k_cellvol<NPL><<<grid, walk::kWarps * 32, smem, (cudaStream_t)stream>>>(
        L, K, N, (const walk::M128 *)table, cap, out, counter, limV, limL);
    return (int)cudaGetLastError();
}

int launch_cellvol(const int64_t *L, int K, int N, const void *table, uint64_t cap, unsigned long long *out,
                   unsigned long long *counter, int grid, void *stream, int64_t limV, int64_t limL) {
    const size_t smem = walk_smem_bytes(K, N);
    int rc;
    switch (npl_of(N)) {
        case 1: rc = cellvol_npl<1>(L, K, N, table, cap, out, counter, grid, stream, limV, limL, smem); break;
        case 2: rc = cellvol_npl<2>(L, K, N, table, cap, out, counter, grid, stream, limV, limL, smem); break;
        case 3: rc = cellvol_npl<3>(L, K, N, table, cap, out, counter, grid, stream, limV, limL, smem); break;
        default: rc = cellvol_npl<4>(L, K, N, table, cap, out, counter, grid, stream, limV, limL, smem); break;
    }
    launch_counter_add(1);
    return rc;
}

}  // namespace bdeg
