// Ceiling of the block-product structure: back-to-back acc_mul<C> / acc_sqr<C> on register
// operands (no memory traffic), at a given number of resident 128-thread CTAs per SM.
//   MODE 0: acc_mul, operands depend on the previous window (serialised iterations)
//   MODE 1: acc_sqr, same dependence
//   MODE 3: acc_mul, independent operands (the real engine: operands come from memory)
//   MODE 4: acc_mul, independent operands, two block products per iteration (merge of the
//           first can overlap the products of the second inside one basic block)
//   MODE 5: acc_sqr, independent operands
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
        else if (MODE == 3) acc_mul<C>(W, x, y);
        else if (MODE == 4) { acc_mul<C>(W, x, y); acc_mul<C>(W, y, x); }
        else if (MODE == 5) acc_sqr<C>(W, x);
        else if (MODE == 6) acc_mul2<C>(W, x, y);
        if (MODE <= 1) x[it & (C - 1)] ^= W[C];
        else { x[it & (C - 1)] += 0x9E3779B9u; y[(it + 3) & (C - 1)] ^= 0x85EBCA6Bu; }
#pragma unroll
        for (int i = 0; i <= C; i++) W[i] = W[i + C];
#pragma unroll
        for (int i = C + 1; i <= 2 * C; i++) W[i] = 0;
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
    printf("%-40s C=%2d ctas/SM=%d  products/clk/SM=%.2f  (%.1f%% of 32)\n", name, C, blocks_per_sm, per_clk, per_clk / 32 * 100);
    cudaFree(d);
}
int main() {
    for (int b : {2, 3}) {
        run<16, 0>("acc_mul dependent", b, 256);
        run<16, 3>("acc_mul independent", b, 256);
        run<16, 6>("acc_mul2 independent", b, 256);
        run<16, 1>("acc_sqr dependent", b, 136);
        run<16, 5>("acc_sqr independent", b, 136);
    }
    return 0;
}
