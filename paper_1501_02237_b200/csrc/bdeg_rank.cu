// libbdeg device code: front end at scale.  Rank of the
// exponent matrix A (n x m) by Gaussian row reduction modulo a 31-bit prime on
// the GPU — the paper's GPU row reduction used for the Smith form and the
// dimensions of Tables 1-2 (§3, Table tab:mspace-dim-long,
// P:1623-1636), rebuilt for B200.  rank_p(A) <= rank_Q(A) for every prime p,
// with equality unless p divides all maximal non-zero minors; the host takes
// the maximum over two primes (probabilistic, pinned by Table 2).
//
// Layout: row-major n x m uint32 residues in HBM.  Step j (column j): one
// kernel finds the first row >= r with a non-zero entry (atomicMin), the host
// swaps it to row r (device copy), and one kernel eliminates column j from
// every row below with a non-zero entry (one CTA per row, coalesced along the
// row; rows with a zero in column j exit at once).
#include "bdeg_internal.h"

#include <cuda_runtime.h>

#include <vector>

namespace bdeg {
namespace rk {

__device__ __forceinline__ uint32_t mulmod(uint32_t a, uint32_t b, uint32_t p) {
    return (uint32_t)(((uint64_t)a * b) % p);
}

__global__ void k_find_pivot(const uint32_t *M, int n, int m, int r, int j, int *best) {
    for (int i = r + blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        if (M[(size_t)i * m + j] != 0) atomicMin(best, i);
}

__global__ void k_swap_rows(uint32_t *M, int m, int a, int b) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < m; t += gridDim.x * blockDim.x) {
        const uint32_t x = M[(size_t)a * m + t];
        M[(size_t)a * m + t] = M[(size_t)b * m + t];
        M[(size_t)b * m + t] = x;
    }
}

// rows i > r: row_i <- row_i - (a_ij / a_rj) row_r  (columns >= j)
__global__ void k_eliminate(uint32_t *M, int n, int m, int r, int j, uint32_t p, uint32_t inv_piv) {
    for (int i = r + 1 + blockIdx.x; i < n; i += gridDim.x) {
        uint32_t *row = M + (size_t)i * m;
        const uint32_t a = row[j];
        // every thread has read the pivot-column entry before any thread of
        // the block overwrites it (t == j below); `a` is block-uniform
        __syncthreads();
        if (a == 0) continue;
        const uint32_t f = mulmod(a, inv_piv, p);
        const uint32_t *prow = M + (size_t)r * m;
        for (int t = j + threadIdx.x; t < m; t += blockDim.x) {
            const uint32_t s = mulmod(f, prow[t], p);
            const uint32_t x = row[t];
            row[t] = x >= s ? x - s : x + p - s;
        }
    }
}

}  // namespace rk

static uint32_t powmod(uint32_t a, uint32_t e, uint32_t p) {
    uint64_t r = 1, b = a % p;
    while (e) {
        if (e & 1) r = r * b % p;
        b = b * b % p;
        e >>= 1;
    }
    return (uint32_t)r;
}

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
    uint32_t *d = nullptr;
    int *best = nullptr;
    if (cudaMalloc(&d, h.size() * 4 + 16) != cudaSuccess) return -1;
    best = (int *)((char *)d + h.size() * 4);
    cudaMemcpyAsync(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice, st);
    int r = 0;
    for (int j = 0; j < m && r < n; ++j) {
        const int big = n;
        cudaMemcpyAsync(best, &big, 4, cudaMemcpyHostToDevice, st);
        rk::k_find_pivot<<<(n - r + 255) / 256, 256, 0, st>>>(d, n, m, r, j, best);
        int piv_row = n;
        uint32_t piv = 0;
        cudaMemcpyAsync(&piv_row, best, 4, cudaMemcpyDeviceToHost, st);
        if (cudaStreamSynchronize(st) != cudaSuccess) { cudaFree(d); return -1; }
        if (piv_row >= n) continue;
        if (piv_row != r) rk::k_swap_rows<<<(m + 255) / 256, 256, 0, st>>>(d, m, piv_row, r);
        cudaMemcpyAsync(&piv, d + (size_t)r * m + j, 4, cudaMemcpyDeviceToHost, st);
        if (cudaStreamSynchronize(st) != cudaSuccess) { cudaFree(d); return -1; }
        const uint32_t inv = powmod(piv, p - 2, p);
        const int rows = n - r - 1;
        if (rows > 0) rk::k_eliminate<<<rows < 4096 ? rows : 4096, 128, 0, st>>>(d, n, m, r, j, p, inv);
        launch_counter_add(3);
        ++r;
    }
    cudaError_t e = cudaStreamSynchronize(st);
    cudaFree(d);
    return e == cudaSuccess ? r : -1;
}

}  // namespace bdeg
