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

// Eliminate the pivot columns of `piv_mask` (ascending order) from the lifted
// matrix in the warp's scratch scr[i*NP + l] (rows 0..K, K = lift row).
// Afterwards the single alive V row is *vrow; values are the true minors.
// Returns false if the pivots are linearly dependent.
template <int NPL>
__device__ bool eliminate(const int64_t *Lsm, int64_t *scr, int K, int N, uint64_t piv_mask, int lane,
                          int *vrow, int64_t *last_piv, bool &ovf) {
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
    const int T = __popcll(piv_mask);
    for (int t = 0; t < T; ++t) {
        const int p = nth_bit(piv_mask, t);
        const bool nz = lane < K && ((alive >> lane) & 1ull) && scr[lane * NP + p] != 0;
        const unsigned bal = __ballot_sync(FULL, nz);
        if (bal == 0) return false;
        const int r = __ffs(bal) - 1;
        const int64_t piv = scr[r * NP + p];
        const Div dv = make_div(prev);
        for (int i = 0; i <= K; ++i) {
            if (i == r || (i < K && !((alive >> i) & 1ull))) continue;
            const int64_t ci = scr[i * NP + p];
#pragma unroll
            for (int q = 0; q < NPL; ++q) {
                const int l = lane + 32 * q;
                if (l == p) continue;
                scr[i * NP + l] = qdiv((i128)piv * scr[i * NP + l] - (i128)ci * scr[r * NP + l], dv, ovf);
            }
        }
        alive &= ~(1ull << r);
        prev = piv;
        __syncwarp();
    }
    *vrow = __ffsll((long long)alive) - 1;
    *last_piv = prev;
    return true;
}

struct WalkArgs {
    const int64_t *L;             // lifted matrix, column-major (K+1) x N
    int K, N;
    const unsigned long long *cur;    // frontier (cell masks)
    uint64_t ncur;
    unsigned long long *next;         // next frontier
    unsigned long long *next_cnt;
    unsigned long long *table;        // hash set of cell masks (0 = empty)
    uint64_t cap;                     // power of two
    unsigned long long *counter;      // work counter
    unsigned long long *stats;        // [0] ridges tested, [1] ties, [2] inconsistent,
                                      // [3] table full, [4] overflow, [5] boundary ridges
    int grid;
    void *stream;
};

__device__ __forceinline__ bool insert(unsigned long long *table, uint64_t cap, uint64_t key, bool &full) {
    uint64_t h = mix64(key) & (cap - 1);
    for (uint64_t probe = 0; probe < cap; ++probe) {
        const unsigned long long old = atomicCAS(table + h, 0ull, (unsigned long long)key);
        if (old == 0ull) return true;
        if (old == key) return false;
        h = (h + 1) & (cap - 1);
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
    const uint64_t nmask = (N >= 64) ? ~0ull : ((1ull << N) - 1);
    unsigned long long st[6] = {0, 0, 0, 0, 0, 0};
    const uint64_t nwork = a.ncur * (uint64_t)K;
    for (;;) {
        unsigned long long idx = 0;
        if (lane == 0) idx = atomicAdd(a.counter, 1ull);
        idx = __shfl_sync(FULL, idx, 0);
        if (idx >= nwork) break;
        const uint64_t m = a.cur[idx / K];
        const int p = nth_bit(m, (int)(idx % K));
        const uint64_t ridge = m & ~(1ull << p);
        bool ovf = false;
        int vr = 0;
        int64_t g = 1;
        ++st[0];
        if (!eliminate<NPL>(Lsm, scr, K, N, ridge, lane, &vr, &g, ovf)) { ++st[2]; continue; }
        int64_t x[NPL], yk[NPL];
        bool valid[NPL];
        const int kappa = g > 0 ? 1 : -1;
#pragma unroll
        for (int q = 0; q < NPL; ++q) {
            const int l = lane + 32 * q;
            x[q] = scr[vr * NP + l];
            yk[q] = kappa > 0 ? scr[K * NP + l] : -scr[K * NP + l];
            valid[q] = ((nmask & ~ridge) >> l) & 1ull;
        }
        if (__any_sync(FULL, ovf)) { ++st[4]; continue; }
        // side of the current cell's point p; the neighbour is on the other side
        const int64_t xp = __shfl_sync(FULL, (long long)(p >= 32 && NPL > 1 ? x[NPL - 1] : x[0]), p & 31);
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
        uint64_t cand = 0;
#pragma unroll
        for (int q = 0; q < NPL; ++q) {
            const bool side = want_pos ? x[q] > 0 : x[q] < 0;
            cand |= (uint64_t)__ballot_sync(FULL, valid[q] && side && key[q] <= mk + 64u) << (32 * q);
        }
        int found = -1;
        bool tie = false;
        while (cand) {
            const int j = __ffsll((long long)cand) - 1;
            cand &= cand - 1;
            const bool js = NPL > 1 && j >= 32;
            const int64_t xj = __shfl_sync(FULL, (long long)(js ? x[NPL - 1] : x[0]), j & 31);
            const int64_t yj = __shfl_sync(FULL, (long long)(js ? yk[NPL - 1] : yk[0]), j & 31);
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
            const uint64_t nm = ridge | (1ull << found);
            bool full = false;
            if (insert(a.table, a.cap, nm, full)) {
                const unsigned long long pos = atomicAdd(a.next_cnt, 1ull);
                a.next[pos] = nm;
            }
            if (full) ++st[3];
        }
    }
    if (lane == 0)
        for (int i = 0; i < 6; ++i)
            if (st[i]) atomicAdd(a.stats + i, st[i]);
}

// |det| of every cell in the table (one warp per cell) into 4 limbs + count
template <int NPL>
__global__ void __launch_bounds__(kWarps * 32) k_cellvol(const int64_t *L, int K, int N,
                                                          const unsigned long long *table, uint64_t cap,
                                                          unsigned long long *out /* [4 limbs, cells, ovf] */,
                                                          unsigned long long *counter) {
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
            const uint64_t m = table[s];
            if (m == 0) continue;
            const int top = 63 - __clzll((long long)m);
            bool ovf = false;
            int vr = 0;
            int64_t g = 1;
            if (!eliminate<NPL>(Lsm, scr, K, N, m & ~(1ull << top), lane, &vr, &g, ovf)) { ++ovfs; continue; }
            const int64_t d = scr[vr * NP + top];            // +-det of the cell
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

__global__ void k_rehash(const unsigned long long *old, uint64_t oldcap, unsigned long long *tab, uint64_t cap,
                         unsigned long long *full_flag) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < oldcap; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t k = old[i];
        if (k == 0) continue;
        bool full = false;
        insert(tab, cap, k, full);
        if (full) atomicAdd(full_flag, 1ull);
    }
}

}  // namespace walk

uint64_t walk_hash(uint64_t key) {          // host copy of the device hash (for seeding)
    uint64_t z = key;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

int launch_rehash(const unsigned long long *old, uint64_t oldcap, unsigned long long *tab, uint64_t cap,
                  unsigned long long *full_flag, void *stream) {
    walk::k_rehash<<<1184, 256, 0, (cudaStream_t)stream>>>(old, oldcap, tab, cap, full_flag);
    launch_counter_add(1);
    return (int)cudaGetLastError();
}

size_t walk_smem_bytes(int K, int N) {
    const int npl = N > 32 ? 2 : 1;
    return (((size_t)(K + 1) * N * 8 + 15) & ~(size_t)15) + (size_t)walk::kWarps * (K + 1) * 32 * npl * 8;
}

int launch_walk(const int64_t *L, int K, int N, const unsigned long long *cur, uint64_t ncur,
                unsigned long long *next, unsigned long long *next_cnt, unsigned long long *table, uint64_t cap,
                unsigned long long *counter, unsigned long long *stats, int grid, void *stream) {
    walk::WalkArgs a;
    a.L = L; a.K = K; a.N = N; a.cur = cur; a.ncur = ncur; a.next = next; a.next_cnt = next_cnt;
    a.table = table; a.cap = cap; a.counter = counter; a.stats = stats; a.grid = grid; a.stream = stream;
    const size_t smem = walk_smem_bytes(K, N);
    cudaError_t e;
    if (N > 32) {
        e = cudaFuncSetAttribute((const void *)walk::k_walk<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return (int)e;
        walk::k_walk<2><<<grid, walk::kWarps * 32, smem, (cudaStream_t)stream>>>(a);
    } else {
        e = cudaFuncSetAttribute((const void *)walk::k_walk<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return (int)e;
        walk::k_walk<1><<<grid, walk::kWarps * 32, smem, (cudaStream_t)stream>>>(a);
    }
    launch_counter_add(1);
    return (int)cudaGetLastError();
}

int launch_cellvol(const int64_t *L, int K, int N, const unsigned long long *table, uint64_t cap,
                   unsigned long long *out, unsigned long long *counter, int grid, void *stream) {
    const size_t smem = walk_smem_bytes(K, N);
    cudaError_t e;
    if (N > 32) {
        e = cudaFuncSetAttribute((const void *)walk::k_cellvol<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return (int)e;
        walk::k_cellvol<2><<<grid, walk::kWarps * 32, smem, (cudaStream_t)stream>>>(L, K, N, table, cap, out, counter);
    } else {
        e = cudaFuncSetAttribute((const void *)walk::k_cellvol<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return (int)e;
        walk::k_cellvol<1><<<grid, walk::kWarps * 32, smem, (cudaStream_t)stream>>>(L, K, N, table, cap, out, counter);
    }
    launch_counter_add(1);
    return (int)cudaGetLastError();
}

}  // namespace bdeg
