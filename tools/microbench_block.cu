// Ceiling of the block-product structure: back-to-back acc_mul<C> / acc_sqr<C> on register
// operands (no memory traffic), at a given number of resident 128-thread CTAs per SM.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2410_18129_b200/csrc/mp_block.cuh"
using namespace mpb;
__device__ unsigned long long g_cyc[4096];
template <int C, int MODE>
__global__ void __launch_bounds__(128) k_blk(uint32_t* out, uint32_t seed, int iters) {
    uint32_t x[C], y[C], W[2 * C + 1];
#pragma unroll
    for (int i = 0; i < C; i++) { x[i] = seed * (i + 3) + threadIdx.x; y[i] = seed ^ (i * 77 + threadIdx.x); }
#pragma unroll
    for (int i = 0; i <= 2 * C; i++) W[i] = 0;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
        if (MODE == 0) acc_mul<C>(W, x, y);
        else if (MODE == 1) acc_sqr<C>(W, x);
        else { uint32_t E[2 * C], O[2 * C]; bp_mul<C>(x, y, E, O);
#pragma unroll
               for (int i = 0; i < 2 * C; i++) W[i & 7] ^= E[i] ^ O[i]; }
        x[it & (C - 1)] ^= W[C];  // loop-carried dependence keeps the work live
#pragma unroll
        for (int i = 0; i <= C; i++) W[i] = W[i + C];
    }
    __syncthreads();
    long long t1 = clock64();
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i <= 2 * C; i++) s ^= W[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) g_cyc[blockIdx.x] = t1 - t0;
}
template <int C, int MODE>
void run(const char* name, int blocks_per_sm, double prods_per_iter) {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t* d; cudaMalloc(&d, sizeof(uint32_t) * 128 * sms * blocks_per_sm);
    const int iters = 400;
    for (int r = 0; r < 2; r++) k_blk<C, MODE><<<sms * blocks_per_sm, 128>>>(d, 7 + r, iters);
    cudaDeviceSynchronize();
    unsigned long long cyc[4096]; cudaMemcpyFromSymbol(cyc, g_cyc, sizeof(unsigned long long) * sms * blocks_per_sm);
    unsigned long long mx = 0; for (int i = 0; i < sms * blocks_per_sm; i++) mx = cyc[i] > mx ? cyc[i] : mx;
    double per_clk = prods_per_iter * iters * 128.0 * blocks_per_sm / (double)mx;
    printf("%-28s C=%2d ctas/SM=%d  products/clk/SM=%.2f  (%.1f%% of 32)\n", name, C, blocks_per_sm, per_clk, per_clk / 32 * 100);
    cudaFree(d);
}
int main() {
    for (int b : {1, 2, 3, 4}) {
        run<16, 0>("acc_mul (products+merge)", b, 256);
        run<16, 2>("bp_mul only", b, 256);
        run<16, 1>("acc_sqr", b, 136);
    }
    for (int b : {3, 5, 6}) { run<8, 0>("acc_mul (products+merge)", b, 64); run<8, 1>("acc_sqr", b, 36); }
    return 0;
}
