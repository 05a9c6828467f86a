// libbdeg host side of the enumeration kernels: launch bookkeeping, kernel
// selection and the tier-4 (int128-value) replay kernel.  The k_enumerate
// template lives in bdeg_enum.cuh, instantiated per tier in bdeg_enum_t*.cu.
#include "bdeg_enum.cuh"

#include <atomic>
#include <map>
#include <mutex>

namespace bdeg {

static std::atomic<uint64_t> g_launches{0};
uint64_t launch_counter_add(uint64_t k) { return g_launches.fetch_add(k) + k; }

namespace dev {

// ------------------------------------------------------------ tier 4
// int128 values with exact 256-bit intermediates (the
// wider path of the overflow chain; the paper lost exactness on large
// instances).  Rare by construction (only items whose values
// left int64 in tier 2 arrive here), so it trades speed for simplicity: one
// warp per candidate, lanes = points (2 slots), the K pivots of the
// candidate eliminated from scratch over the whole (K+1) x N lifted matrix
// in shared memory (Bareiss, P:687-695 reading Z1), then the sign test of
// the lift row: sigma is a cell iff every other point's
// lifted minor has the sign of det V_sigma.  Every quotient is checked to
// stay below 2^125 in magnitude (|num| < 2^125 |prev|), else the item is
// fatal (BDEG_E_TOO_LARGE).
typedef unsigned __int128 u128d;

struct S256 { uint64_t w[4]; };   // two's complement, little-endian limbs

__device__ __forceinline__ S256 mul_s128(i128 a, i128 b) {
    const bool neg = (a < 0) != (b < 0);
    const u128d x = a < 0 ? (u128d)(-a) : (u128d)a;
    const u128d y = b < 0 ? (u128d)(-b) : (u128d)b;
    const uint64_t x0 = (uint64_t)x, x1 = (uint64_t)(x >> 64), y0 = (uint64_t)y, y1 = (uint64_t)(y >> 64);
    const u128d p00 = (u128d)x0 * y0, p01 = (u128d)x0 * y1, p10 = (u128d)x1 * y0, p11 = (u128d)x1 * y1;
    S256 r;
    r.w[0] = (uint64_t)p00;
    u128d mid = (p00 >> 64) + (uint64_t)p01 + (uint64_t)p10;
    r.w[1] = (uint64_t)mid;
    u128d hi = (mid >> 64) + (p01 >> 64) + (p10 >> 64) + (uint64_t)p11;
    r.w[2] = (uint64_t)hi;
    r.w[3] = (uint64_t)(hi >> 64) + (uint64_t)(p11 >> 64);
    if (neg) {                                  // two's complement negation
        uint64_t c = 1;
        for (int i = 0; i < 4; ++i) {
            const uint64_t v = ~r.w[i] + c;
            c = (c && v == 0) ? 1 : 0;
            r.w[i] = v;
        }
    }
    return r;
}

__device__ __forceinline__ S256 sub256(const S256 &a, const S256 &b) {
    S256 r;
    uint64_t borrow = 0;
    for (int i = 0; i < 4; ++i) {
        const uint64_t d = a.w[i] - b.w[i];
        const uint64_t d2 = d - borrow;
        borrow = (a.w[i] < b.w[i]) || (d < borrow) ? 1 : 0;
        r.w[i] = d2;
    }
    return r;
}

__device__ __forceinline__ u128d inv128_odd(u128d o) {
    u128d x = o;                                // correct to 3 bits
    for (int i = 0; i < 6; ++i) x *= (u128d)2 - o * x;
    return x;
}

// exact (a*b - c*d) / e, e != 0, quotient required to satisfy |q| < 2^125
__device__ __forceinline__ i128 bareiss_wide(i128 a, i128 b, i128 c, i128 d, i128 e, bool &ovf) {
    const S256 num = sub256(mul_s128(a, b), mul_s128(c, d));
    const bool neg = (int64_t)num.w[3] < 0;
    S256 m = num;                               // |num|
    if (neg) {
        uint64_t cy = 1;
        for (int i = 0; i < 4; ++i) {
            const uint64_t v = ~m.w[i] + cy;
            cy = (cy && v == 0) ? 1 : 0;
            m.w[i] = v;
        }
    }
    // bound = |e| << 125 (|e| < 2^126: fits in 251 bits)
    const u128d ae = e < 0 ? (u128d)(-e) : (u128d)e;
    S256 bd;
    bd.w[0] = 0;
    bd.w[1] = (uint64_t)(ae << 61);
    bd.w[2] = (uint64_t)(ae >> 3);
    bd.w[3] = (uint64_t)(ae >> 67);
    bool lt = false, decided = false;
    for (int i = 3; i >= 0 && !decided; --i)
        if (m.w[i] != bd.w[i]) { lt = m.w[i] < bd.w[i]; decided = true; }
    if (!lt) { ovf = true; return 0; }
    // exact division: shift out e's 2-adic part, multiply by the odd inverse mod 2^128
    const uint64_t elo = (uint64_t)(u128d)e, ehi = (uint64_t)((u128d)e >> 64);
    const int tz = elo ? __ffsll((long long)elo) - 1 : 64 + __ffsll((long long)ehi) - 1;
    // (num >> tz) low 128 bits (arithmetic shift of the 256-bit value)
    u128d lo = ((u128d)num.w[1] << 64) | num.w[0];
    u128d hi = ((u128d)num.w[3] << 64) | num.w[2];
    u128d sh;
    if (tz == 0) sh = lo;
    else if (tz < 128) sh = (lo >> tz) | (hi << (128 - tz));
    else sh = (u128d)((i128)hi >> (tz - 128));
    const u128d o = (u128d)(e >> tz);
    return (i128)(sh * inv128_odd(o));
}

__global__ void __launch_bounds__(kWarps * 32, 1)
k_enumerate_wide(const __grid_constant__ LaunchArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    if (a.replay_gate && *(volatile const unsigned long long *)a.replay_gate == 0) return;
    const int K = a.P.K, N = a.P.N;
    const uint32_t lbytes = (uint32_t)(((K + 1) * N * 8 + 15) & ~15);
    const uint32_t bbytes = kBinomRows * kBinomCols * 8;
    int64_t *Lsm = reinterpret_cast<int64_t *>(smem);
    uint64_t *Bsm = reinterpret_cast<uint64_t *>(smem + lbytes);
    unsigned long long *red = reinterpret_cast<unsigned long long *>(smem + lbytes + bbytes);
    i128 *scr_all = reinterpret_cast<i128 *>(smem + lbytes + bbytes + kWarps * 16 * 8);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (uint32_t i = threadIdx.x; i < (uint32_t)((K + 1) * N); i += blockDim.x) Lsm[i] = a.P.L[i];
    for (uint32_t i = threadIdx.x; i < (uint32_t)(kBinomRows * kBinomCols); i += blockDim.x) Bsm[i] = a.P.binom[i];
    __syncthreads();
    constexpr int NP = 64;
    i128 *M = scr_all + (size_t)warp * (K + 1) * NP;
    Ctx cx;
    cx.B = Bsm;
    cx.N = N;
    cx.K = K;
    cx.lane = lane;
    cx.A = &a;
    cx.partial = true;
    cx.nmask = (N >= 64) ? ~0ull : ((1ull << N) - 1);
    cx.D = a.P.D;
    cx.kd = K - a.P.D;
    cx.fmin = 0;
    cx.mytop = 0;
    cx.deg_only = false;
    cx.dead_full = false;
    uint64_t vol_lo = 0, vol_hi = 0, cells = 0, singular = 0, cand = 0, ties = 0, items = 0, fatal = 0;
    unsigned long long rbits = 0, rword = 0;
    for (;;) {
        unsigned long long pos = ~0ull;
        if (lane == 0) {
            while (rbits == 0) {
                rword = atomicAdd(a.counter, 1ull);
                if (rword >= a.ovf_words) break;
                rbits = a.replay_bits[rword];
                if (rbits) a.replay_bits[rword] = 0ull;
            }
            if (rbits) {
                pos = rword * 64 + (unsigned long long)(__ffsll((long long)rbits) - 1);
                rbits &= rbits - 1;
            }
        }
        pos = __shfl_sync(FULL, pos, 0);
        if (pos == ~0ull) break;
        int mytop = 0;
        const int D = decode_item(pos, a, cx, mytop);
        const int kd = K - D;
        uint64_t tall = (lane < D) ? cx.C(mytop, kd + lane + 1) : 0;
#pragma unroll
        for (int o = 16; o; o >>= 1) tall += __shfl_xor_sync(FULL, tall, o);
        const int cfirst = D > 0 ? __shfl_sync(FULL, mytop, 0) : N;
        const uint64_t isize = cx.C(cfirst, kd);
        const uint64_t rb = tall > a.rank_begin ? tall : a.rank_begin;
        const uint64_t re = tall + isize < a.rank_end ? tall + isize : a.rank_end;
        ++items;
        bool item_bad = false;
        uint64_t i_vol_lo = 0, i_vol_hi = 0, i_cells = 0, i_sing = 0, i_ties = 0;
        for (uint64_t r = rb; r < re && !item_bad; ++r) {
            int myc = 0;                                   // lane t < K: c_t of rank r
            unrank_lanes(r, K, N, 0, 0, cx, myc);
            uint64_t inS = 0;
            {
                const uint64_t bit = lane < K ? (1ull << myc) : 0ull;
                const unsigned lo = __reduce_or_sync(FULL, (unsigned)bit);
                const unsigned hi = __reduce_or_sync(FULL, (unsigned)(bit >> 32));
                inS = ((uint64_t)hi << 32) | lo;
            }
            __syncwarp();
            for (int i = 0; i <= K; ++i)
                for (int q = 0; q < 2; ++q) {
                    const int l = lane + 32 * q;
                    M[i * NP + l] = (l < N) ? (i128)Lsm[l * (K + 1) + i] : (i128)0;
                }
            __syncwarp();
            i128 prev = 1;
            uint64_t alive = (K >= 64) ? ~0ull : ((1ull << K) - 1);
            bool sing = false, o = false;
            for (int t = K - 1; t >= 0; --t) {
                const int c = __shfl_sync(FULL, myc, t);
                const bool nz = lane < K && ((alive >> lane) & 1ull) && M[lane * NP + c] != 0;
                const unsigned bal = __ballot_sync(FULL, nz);
                if (bal == 0) { sing = true; break; }
                const int pr = __ffs(bal) - 1;
                const i128 piv = M[pr * NP + c];
                for (int i = 0; i <= K; ++i) {
                    if (i == pr || (i < K && !((alive >> i) & 1ull))) continue;
                    const i128 ci = M[i * NP + c];
                    i128 nv[2];
                    for (int q = 0; q < 2; ++q) {
                        const int l = lane + 32 * q;
                        nv[q] = bareiss_wide(piv, M[i * NP + l], ci, M[pr * NP + l], prev, o);
                    }
                    __syncwarp();                          // every lane has read column c of row i
                    for (int q = 0; q < 2; ++q) M[i * NP + lane + 32 * q] = nv[q];
                    __syncwarp();
                }
                if (__any_sync(FULL, o)) break;
                alive &= ~(1ull << pr);
                prev = piv;
            }
            if (__any_sync(FULL, o)) { item_bad = true; break; }
            if (sing) { ++i_sing; continue; }
            // lift row vs det: cell iff sign(y_l) = sign(prev) for all l not in sigma
            bool bad = false, zero = false;
            for (int q = 0; q < 2; ++q) {
                const int l = lane + 32 * q;
                if (l < N && !((inS >> l) & 1ull)) {
                    const i128 y = M[K * NP + l];
                    bad |= (y < 0) != (prev < 0) && y != 0;
                    zero |= y == 0;
                }
            }
            if (__any_sync(FULL, bad)) continue;
            if (__any_sync(FULL, zero)) { ++i_ties; continue; }
            ++i_cells;
            const u128d v = prev < 0 ? (u128d)(-prev) : (u128d)prev;
            const uint64_t t0 = i_vol_lo + (uint64_t)v;
            i_vol_hi += (uint64_t)(v >> 64) + (t0 < i_vol_lo);
            i_vol_lo = t0;
            if (a.cells_out && lane == 0 && (v >> 64) == 0) {
                const unsigned long long at = atomicAdd(a.cells_cnt, 1ull);
                if (at < a.cells_cap) { a.cells_out[2 * at] = inS; a.cells_out[2 * at + 1] = (uint64_t)v; }
            }
        }
        if (item_bad) { ++fatal; continue; }        // beyond int128: BDEG_E_TOO_LARGE
        const uint64_t t0 = vol_lo + i_vol_lo;
        vol_hi += i_vol_hi + (t0 < vol_lo);
        vol_lo = t0;
        cells += i_cells;
        singular += i_sing;
        ties += i_ties;
        cand += re > rb ? re - rb : 0;
    }
    if (lane == 0) {
        unsigned long long *w = red + warp * 16;
        w[0] = vol_lo & 0xFFFFFFFFull;
        w[1] = vol_lo >> 32;
        w[2] = vol_hi & 0xFFFFFFFFull;
        w[3] = vol_hi >> 32;
        w[SLOT_CELLS] = cells;
        w[SLOT_SINGULAR] = singular;
        w[SLOT_CAND] = cand;
        w[SLOT_TIES] = ties;
        w[SLOT_OVF_BLOCKS] = 0;
        w[SLOT_FATAL] = fatal;
        w[SLOT_QFULL] = 0;
        w[SLOT_BLOCKS] = items;
        w[SLOT_UPDATES] = 0;
        w[SLOT_LEAVES] = 0;
        w[14] = 0;
        w[SLOT_WIDE] = 0;
    }
    __syncthreads();
    if (threadIdx.x < kNSlots) {
        unsigned long long s = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) s += red[w * 16 + threadIdx.x];
        if (s) atomicAdd(a.slots + threadIdx.x, s);
    }
}

}  // namespace dev

size_t enumerate_wide_smem_bytes(int K, int N) {
    const size_t lbytes = ((size_t)(K + 1) * N * 8 + 15) & ~(size_t)15;
    const size_t bbytes = kBinomRows * kBinomCols * 8;
    return lbytes + bbytes + (size_t)dev::kWarps * 16 * 8 + (size_t)dev::kWarps * (K + 1) * 64 * 16;
}

size_t enumerate_smem_bytes(int K, int N, int warps) {
    const size_t lbytes = ((size_t)(K + 1) * N * 8 + 15) & ~(size_t)15;
    const size_t bbytes = kBinomRows * kBinomCols * 8;
    const int npl = N > 32 ? 2 : 1;
    return lbytes + bbytes + (size_t)warps * 16 * 8 + 16 + (size_t)warps * (K + 1) * 32 * npl * 8;
}

int kernel_warps_per_cta() { return dev::kWarps; }

static KernFn pick(int tier, int npl, int S, bool ranged) {
    switch (tier) {
        case 0: return pick_t0(npl, S, ranged);
        case 1: return pick_t1(npl, S, ranged);
        case 2: return pick_t2(npl, S, ranged);
        case 3: return pick_t3(npl, S, ranged);
        default: return nullptr;
    }
}

// cudaFuncSetAttribute(max dynamic smem) once per (kernel, size): the value
// only ever grows, so remember the largest one set per kernel
static std::mutex g_attr_mu;
static std::map<std::pair<int, KernFn>, size_t> g_attr;   // (device, kernel) -> smem set

static cudaError_t ensure_smem_attr(KernFn f, size_t smem) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_attr_mu);
    auto it = g_attr.find({dev, f});
    if (it != g_attr.end() && it->second >= smem) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute((const void *)f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess) g_attr[{dev, f}] = smem;
    return e;
}

int enumerate_max_ctas_per_sm(const LaunchArgs &a) {
    const int npl = a.P.N > 32 ? 2 : 1;
    KernFn f = pick(a.tier, npl, a.P.S, a.mode == 0);
    if (!f) return 1;
    const size_t smem = enumerate_smem_bytes(a.P.K, a.P.N, dev::kWarps);
    ensure_smem_attr(f, smem);
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, f, dev::kWarps * 32, smem) != cudaSuccess) return 1;
    return n > 0 ? n : 1;
}

int launch_enumerate_wide(const LaunchArgs &a) {
    KernFn f = dev::k_enumerate_wide;
    const size_t smem = enumerate_wide_smem_bytes(a.P.K, a.P.N);
    cudaError_t e = ensure_smem_attr(f, smem);
    if (e != cudaSuccess) return (int)e;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    f<<<sms, dev::kWarps * 32, smem, (cudaStream_t)a.stream>>>(a);
    launch_counter_add(1);
    return (int)cudaGetLastError();
}

int launch_enumerate(const LaunchArgs &a) {
    const int npl = a.P.N > 32 ? 2 : 1;
    KernFn f = pick(a.tier, npl, a.P.S, a.mode == 0);
    if (!f) return (int)cudaErrorInvalidValue;
    const size_t smem = enumerate_smem_bytes(a.P.K, a.P.N, dev::kWarps);
    cudaError_t e = ensure_smem_attr(f, smem);
    if (e != cudaSuccess) return (int)e;
    f<<<a.grid, dev::kWarps * 32, smem, (cudaStream_t)a.stream>>>(a);
    launch_counter_add(1);
    return (int)cudaGetLastError();
}

}  // namespace bdeg
