// Integer-pipe peak microbenchmark for the roofline denominator (SURVEY §8.d
// "Peak to measure (do not assume)").  Measures warp-instructions issued per
// SM clock for the integer instruction classes the enumeration kernel uses:
//   IADD3 / LOP3 / SHF / ISETP   (ALU pipe)
//   IMAD                         (FMA pipe)
//   IADD3 + IMAD interleaved     (both pipes: the SM's integer issue ceiling)
// Each thread runs 8 independent dependency chains (ILP) at full occupancy
// (TLP), one resident wave on every SM; cycles come from %clock64 on the SM
// (so the result is per clock, independent of the clock rate), and the SASS
// of every loop body is checked with cuobjdump (tools/intpipe_sass.txt) so
// that instructions are counted exactly.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o intpipe_bench tools/intpipe_bench.cu
//   ./intpipe_bench  > profiles/r2_intpipe_peaks.json
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>
#include <vector>

constexpr int kIters = 4096;
constexpr int kChains = 8;

enum Op { IADD3, LOP3, IMAD, IMADW, MIX, SHF, ISETP, MIX_REUSE, MIX3, LOP3_REUSE };

template <int OP>
__global__ void __launch_bounds__(256) k_pipe(uint32_t *out, unsigned long long *cyc, uint32_t seed) {
    uint32_t r[kChains], s[kChains];
#pragma unroll
    for (int j = 0; j < kChains; ++j) {
        r[j] = seed ^ (threadIdx.x * 2654435761u + j);
        s[j] = seed + 7 * j + threadIdx.x;
    }
    uint64_t w[kChains];
#pragma unroll
    for (int j = 0; j < kChains; ++j) w[j] = r[j];
    __syncthreads();
    const unsigned long long t0 = clock64();
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int j = 0; j < kChains; ++j) {
            if constexpr (OP == IADD3) {
                asm volatile("{ .reg .u32 t; add.u32 t, %0, %1; add.u32 %0, t, %2; }" : "+r"(r[j]) : "r"(s[j]), "r"(s[(j + 3) & 7]));
            } else if constexpr (OP == LOP3) {
                asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(r[j]) : "r"(s[j]), "r"(s[(j + 3) & 7]));
            } else if constexpr (OP == IMAD) {
                asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(r[j]) : "r"(s[j]), "r"(s[(j + 3) & 7]));
            } else if constexpr (OP == IMADW) {
                asm volatile("{ .reg .u32 lo, hi; mov.b64 {lo, hi}, %0; mul.wide.s32 %0, lo, %1; }" : "+l"(w[j]) : "r"(s[j]));
            } else if constexpr (OP == MIX) {
                if (j & 1) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(r[j]) : "r"(s[j]), "r"(s[(j + 3) & 7]));
                else asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(r[j]) : "r"(s[j]), "r"(s[(j + 3) & 7]));
            } else if constexpr (OP == SHF) {
                asm volatile("shf.l.wrap.b32 %0, %0, %1, %2;" : "+r"(r[j]) : "r"(s[j]), "r"(s[(j + 3) & 7]));
            } else if constexpr (OP == MIX_REUSE) {   // IMAD / LOP3 sharing two loop-invariant sources
                if (j & 1) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(r[j]) : "r"(s[0]), "r"(s[1]));
                else asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(r[j]) : "r"(s[0]), "r"(s[1]));
            } else if constexpr (OP == MIX3) {        // IMAD : LOP3 : IADD3 = 3 : 3 : 2 (chain j mod 3)
                if (j % 3 == 0) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(r[j]) : "r"(s[0]), "r"(s[1]));
                else if (j % 3 == 1) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(r[j]) : "r"(s[0]), "r"(s[1]));
                else asm volatile("{ .reg .u32 t; add.u32 t, %0, %1; add.u32 %0, t, %2; }" : "+r"(r[j]) : "r"(s[0]), "r"(s[1]));
            } else if constexpr (OP == LOP3_REUSE) {
                asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(r[j]) : "r"(s[0]), "r"(s[1]));
            } else {   // ISETP feeding a select (the facet tests' compare + select pattern)
                asm volatile("{ .reg .pred p; setp.lt.s32 p, %0, %1; selp.u32 %0, %2, %0, p; }" : "+r"(r[j]) : "r"(s[j]), "r"(s[(j + 3) & 7]));
            }
        }
    }
    const unsigned long long t1 = clock64();
    uint32_t acc = 0;
#pragma unroll
    for (int j = 0; j < kChains; ++j) acc ^= r[j] ^ (uint32_t)w[j] ^ (uint32_t)(w[j] >> 32);
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
static void run(const char *name, const char *pipe, double sass_per_op, int sms, int blocks_per_sm, bool last) {
    const int grid = sms * blocks_per_sm, block = 256;
    uint32_t *out;
    unsigned long long *cyc;
    cudaMalloc(&out, (size_t)grid * block * 4);
    cudaMalloc(&cyc, (size_t)grid * 8);
    k_pipe<OP><<<grid, block>>>(out, cyc, 1);   // warm-up
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_pipe<OP><<<grid, block>>>(out, cyc, 2);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    std::vector<unsigned long long> c(grid);
    cudaMemcpy(c.data(), cyc, (size_t)grid * 8, cudaMemcpyDeviceToHost);
    unsigned long long cmax = 0;
    for (auto x : c) cmax = x > cmax ? x : cmax;
    // warp-instructions per SM over the timed loop (SASS count per op = sass_per_op)
    const double warp_inst_per_sm = (double)blocks_per_sm * (block / 32) * kIters * kChains * sass_per_op;
    const double per_clk = warp_inst_per_sm / (double)cmax;
    const double ghz = (double)cmax / (ms * 1e6);
    printf("  \"%s\": {\"pipe\": \"%s\", \"warp_inst_per_clk_per_sm\": %.4f, \"lane_ops_per_clk_per_sm\": %.2f, "
           "\"cycles\": %llu, \"ms\": %.4f, \"implied_sm_ghz\": %.4f}%s\n",
           name, pipe, per_clk, 32.0 * per_clk, cmax, ms, ghz, last ? "" : ",");
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    cudaDeviceProp prop;
    cudaGetDeviceProperties(&prop, 0);
    const int sms = prop.multiProcessorCount;
    const int bps = 8;   // 8 x 256 threads = 64 warps per SM (full occupancy)
    printf("{\n  \"gpu\": \"%s\", \"sms\": %d, \"blocks_per_sm\": %d, \"threads_per_block\": 256, "
           "\"chains_per_thread\": %d, \"iters\": %d,\n", prop.name, sms, bps, kChains, kIters);
    run<IADD3>("iadd3", "alu", 1.0, sms, bps, false);
    run<LOP3>("lop3", "alu", 1.0, sms, bps, false);
    run<SHF>("shf", "alu", 1.0, sms, bps, false);
    run<ISETP>("isetp_sel", "alu", 2.0, sms, bps, false);
    run<IMAD>("imad", "fma", 1.0, sms, bps, false);
    run<MIX>("imad_lop3_mix", "alu+fma", 1.0, sms, bps, false);
    run<MIX_REUSE>("imad_lop3_mix_reuse", "alu+fma", 1.0, sms, bps, false);
    run<MIX3>("imad_lop3_iadd3_mix", "alu+fma", 1.0, sms, bps, false);
    run<LOP3_REUSE>("lop3_reuse", "alu", 1.0, sms, bps, true);
    printf("}\n");
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
