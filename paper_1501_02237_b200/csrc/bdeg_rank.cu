// libbdeg device code: the front end at scale — the paper's
// GPU row reduction of the exponent matrix (§3; Tables
// 1-2), rebuilt for B200 as ONE cooperative persistent kernel
// per matrix: no host round trip per column, grid-wide barriers between the
// pivot search and the elimination of each column.
//
//   rank_modp:  Gaussian elimination over GF(p), p < 2^31 (any non-zero
//               pivot).  rank_p(A) <= rank_Q(A), equal unless p divides every
//               maximal non-zero minor.
//   smith_unimodular: exact elimination over Z with unit pivots only (an
//               entry +-1): each such pivot is an invariant factor 1 of the
//               Smith form, so SNF(A) = I_k (+) SNF(residual),
//               where the residual is the block of unused rows x columns that
//               had non-zero entries but no unit pivot.  The host finishes the
//               (small) residual with the exact Euclidean SNF.  This gives the
//               EXACT rank (dimension d = n - r, Prop. 1) and the component
//               count |prod d_j| for n in the thousands.
//
// Layout: row-major n x m in HBM (the paper's Table 2 sizes: n = 4800 fits in
// L2 for GF(p); int64 entries for Z).  Column j: phase 1 finds the first
// unused row with an admissible pivot (atomicMin, per-column slot, so no
// reset barrier is needed); phase 2 clears column j from every other unused
// row (one CTA per row, coalesced along the row).
#include "bdeg_internal.h"

#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <vector>

namespace cg = cooperative_groups;

namespace bdeg {
namespace rk {

constexpr int kThreads = 256;

__device__ __forceinline__ uint32_t mulmod(uint32_t a, uint32_t b, uint32_t p) {
    return (uint32_t)(((uint64_t)a * b) % p);
}
__device__ uint32_t powmod(uint32_t a, uint32_t e, uint32_t p) {
    uint32_t r = 1;
    while (e) {
        if (e & 1) r = mulmod(r, a, p);
        a = mulmod(a, a, p);
        e >>= 1;
    }
    return r;
}

// GF(p).  best[j] = n (host-initialised), used[i] = 0, out[0] = rank.
__global__ void __launch_bounds__(kThreads) k_rank_modp(uint32_t *M, int n, int m, uint32_t p, int *best,
                                                        int *used, int *out) {
    cg::grid_group grid = cg::this_grid();
    __shared__ uint32_t s_a;
    int rank = 0;
    for (int j = 0; j < m && rank < n; ++j) {
        for (int i = (int)grid.thread_rank(); i < n; i += (int)grid.size())
            if (!used[i] && M[(size_t)i * m + j] != 0) atomicMin(best + j, i);
        grid.sync();
        const int r = *(volatile int *)(best + j);
        if (r >= n) continue;                       // uniform across the grid
        const uint32_t *prow = M + (size_t)r * m;
        const uint32_t inv = powmod(prow[j], p - 2, p);
        for (int i = blockIdx.x; i < n; i += gridDim.x) {
            if (i == r || used[i]) continue;
            uint32_t *row = M + (size_t)i * m;
            if (threadIdx.x == 0) s_a = row[j];
            __syncthreads();                        // every thread sees a before anyone writes row[j]
            const uint32_t a = s_a;
            __syncthreads();
            if (a == 0) continue;
            const uint32_t f = mulmod(a, inv, p);
            for (int t = j + threadIdx.x; t < m; t += blockDim.x) {
                const uint32_t s = mulmod(f, prow[t], p);
                const uint32_t x = row[t];
                row[t] = x >= s ? x - s : x + p - s;
            }
        }
        if (blockIdx.x == 0 && threadIdx.x == 0) used[r] = 1;
        ++rank;
        grid.sync();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = rank;
}

// Z, unit pivots.  best[j] = n, nz[j] = 0, used[i] = 0 (host-initialised).
// out: [0] unit pivots, [1] overflow flag, [2] first deferred column (m if none).
__global__ void __launch_bounds__(kThreads) k_smith_unimodular(int64_t *M, int n, int m, int *best, int *nz,
                                                               int *used, int *out) {
    cg::grid_group grid = cg::this_grid();
    __shared__ int64_t s_a;
    int pivots = 0, first_def = m;
    const int64_t LIM = (int64_t)1 << 61;
    for (int j = 0; j < m && pivots < n; ++j) {
        for (int i = (int)grid.thread_rank(); i < n; i += (int)grid.size()) {
            if (used[i]) continue;
            const int64_t v = M[(size_t)i * m + j];
            if (v == 1 || v == -1) atomicMin(best + j, i);
            if (v != 0) nz[j] = 1;                  // benign race: any writer stores 1
        }
        grid.sync();
        const int r = *(volatile int *)(best + j);
        if (r >= n) {                               // no unit pivot: defer (or all zero)
            if (*(volatile int *)(nz + j) && j < first_def) first_def = j;
            continue;
        }
        const int64_t *prow = M + (size_t)r * m;
        const int64_t sgn = prow[j];                // +-1: the multiplier is a * sgn
        const int k0 = first_def < j ? first_def : j;
        for (int i = blockIdx.x; i < n; i += gridDim.x) {
            if (i == r || used[i]) continue;
            int64_t *row = M + (size_t)i * m;
            if (threadIdx.x == 0) s_a = row[j];
            __syncthreads();
            const int64_t a = s_a;
            __syncthreads();
            if (a == 0) continue;
            const int64_t f = a * sgn;
            bool ovf = f >= LIM || f <= -LIM;
            for (int t = k0 + threadIdx.x; t < m; t += blockDim.x) {
                const int64_t b = prow[t];
                if (b == 0) continue;
                // |f|, |b| < 2^61 and |f b| < 2^61 checked in 128-bit
                const __int128 prod = (__int128)f * b;
                const __int128 nv = (__int128)row[t] - prod;
                if (nv >= LIM || nv <= -LIM) ovf = true;
                row[t] = (int64_t)nv;
            }
            if (ovf) out[1] = 1;
        }
        if (blockIdx.x == 0 && threadIdx.x == 0) used[r] = 1;
        ++pivots;
        grid.sync();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        out[0] = pivots;
        out[2] = first_def;
    }
}

}  // namespace rk

namespace {

int coop_grid(const void *fn, int device) {
    int sms = 0, per = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, rk::kThreads, 0);
    return sms * (per > 0 ? per : 1);
}

}  // namespace

// rank of A (row-major int64 n x m) modulo the prime p; -1 on CUDA error
long long rank_modp(const int64_t *A, int n, int m, uint32_t p, int device, void *stream) {
    if (cudaSetDevice(device) != cudaSuccess) return -1;
    cudaStream_t st = (cudaStream_t)stream;
    std::vector<uint32_t> h((size_t)n * m);
    for (size_t i = 0; i < h.size(); ++i) {
        int64_t v = A[i] % (int64_t)p;
        if (v < 0) v += p;
        h[i] = (uint32_t)v;
    }
    char *d = nullptr;
    const size_t mb = h.size() * 4, bb = (size_t)m * 4, ub = (size_t)n * 4;
    if (cudaMalloc(&d, mb + bb + ub + 16) != cudaSuccess) return -1;
    uint32_t *dM = (uint32_t *)d;
    int *best = (int *)(d + mb), *used = (int *)(d + mb + bb), *out = (int *)(d + mb + bb + ub);
    std::vector<int> init(m, n);
    cudaMemcpyAsync(dM, h.data(), mb, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(best, init.data(), bb, cudaMemcpyHostToDevice, st);
    cudaMemsetAsync(used, 0, ub + 16, st);
    int nn = n, mm = m;
    uint32_t pp = p;
    void *args[] = {&dM, &nn, &mm, &pp, &best, &used, &out};
    const int grid = coop_grid((const void *)rk::k_rank_modp, device);
    cudaError_t e = cudaLaunchCooperativeKernel((const void *)rk::k_rank_modp, grid, rk::kThreads, args, 0, st);
    launch_counter_add(1);
    int r = -1;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&r, out, 4, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaFree(d);
    return e == cudaSuccess ? r : -1;
}

// Exact unit-pivot elimination on the GPU; returns 0 on success, 1 on an
// entry beyond 2^61 (caller falls back / reports), -1 on CUDA error.  On
// success *pivots = unit pivots and `residual` = the rows never used x the
// columns deferred (non-zero in unused rows but without a unit pivot), as a
// dense row-major int64 matrix (res_rows x res_cols).
int smith_unimodular(const int64_t *A, int n, int m, int device, void *stream, long long *pivots,
                     std::vector<int64_t> &residual, int &res_rows, int &res_cols) {
    if (cudaSetDevice(device) != cudaSuccess) return -1;
    cudaStream_t st = (cudaStream_t)stream;
    char *d = nullptr;
    const size_t mb = (size_t)n * m * 8, bb = (size_t)m * 4, ub = (size_t)n * 4;
    if (cudaMalloc(&d, mb + 2 * bb + ub + 16) != cudaSuccess) return -1;
    int64_t *dM = (int64_t *)d;
    int *best = (int *)(d + mb), *nz = (int *)(d + mb + bb), *used = (int *)(d + mb + 2 * bb);
    int *out = (int *)(d + mb + 2 * bb + ub);
    std::vector<int> init(m, n);
    cudaMemcpyAsync(dM, A, mb, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(best, init.data(), bb, cudaMemcpyHostToDevice, st);
    cudaMemsetAsync(nz, 0, bb, st);
    cudaMemsetAsync(used, 0, ub + 16, st);
    int nn = n, mm = m;
    void *args[] = {&dM, &nn, &mm, &best, &nz, &used, &out};
    const int grid = coop_grid((const void *)rk::k_smith_unimodular, device);
    cudaError_t e =
        cudaLaunchCooperativeKernel((const void *)rk::k_smith_unimodular, grid, rk::kThreads, args, 0, st);
    launch_counter_add(1);
    int h_out[3] = {0, 0, 0};
    std::vector<int> h_used(n), h_best(m), h_nz(m);
    if (e == cudaSuccess) e = cudaMemcpyAsync(h_out, out, 12, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(h_used.data(), used, ub, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(h_best.data(), best, bb, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(h_nz.data(), nz, bb, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) { cudaFree(d); return -1; }
    if (h_out[1]) { cudaFree(d); return 1; }
    *pivots = h_out[0];
    std::vector<int> rows, cols;
    for (int i = 0; i < n; ++i) if (!h_used[i]) rows.push_back(i);
    // deferred columns: non-zero in unused rows at their turn, no unit pivot
    // (a column whose turn came after the pivots ran out counts as deferred
    // if it has any non-zero entry left: checked on the host copy)
    std::vector<int64_t> hM;
    if (!rows.empty()) {
        hM.resize((size_t)n * m);
        if (cudaMemcpy(hM.data(), dM, mb, cudaMemcpyDeviceToHost) != cudaSuccess) { cudaFree(d); return -1; }
        for (int j = 0; j < m; ++j) {
            if (h_best[j] < n) continue;            // a unit pivot column: zero in every unused row
            bool any = false;
            for (int i : rows) if (hM[(size_t)i * m + j] != 0) { any = true; break; }
            if (any) cols.push_back(j);
        }
    }
    cudaFree(d);
    res_rows = (int)rows.size();
    res_cols = (int)cols.size();
    residual.assign((size_t)res_rows * res_cols, 0);
    for (int a = 0; a < res_rows; ++a)
        for (int b = 0; b < res_cols; ++b) residual[(size_t)a * res_cols + b] = hM[(size_t)rows[a] * m + cols[b]];
    return 0;
}

}  // namespace bdeg
