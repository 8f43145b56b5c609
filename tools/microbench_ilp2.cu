// Two independent operands per thread (V = 2): does interleaving the block products of two
// operands (separate windows, separate x / y) raise the product pipe rate over one operand per
// thread?  Same structure as microbench_block.cu MODE 3 (acc_mul on fresh operands every
// iteration + the window shift), V copies per thread; run at 1..4 CTAs/SM.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2410_18129_b200/csrc/mp_block.cuh"
using namespace mpb;
__device__ unsigned long long g_cyc[4096];

template <int C, int V, int MODE>
__global__ void __launch_bounds__(128) k_v(uint32_t* out, uint32_t seed, int iters) {
    uint32_t x[V][C], y[V][C], W[V][2 * C + 1];
#pragma unroll
    for (int v = 0; v < V; v++) {
#pragma unroll
        for (int i = 0; i < C; i++) { x[v][i] = seed * (i + 3 + v) + threadIdx.x; y[v][i] = seed ^ (i * 77 + threadIdx.x + v); }
#pragma unroll
        for (int i = 0; i <= 2 * C; i++) W[v][i] = 0;
    }
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int v = 0; v < V; v++) {
            if (MODE == 0) acc_mul<C>(W[v], x[v], y[v]);
            else acc_sqr<C>(W[v], x[v]);
        }
#pragma unroll
        for (int v = 0; v < V; v++) {
            x[v][0] += 0x9E3779B9u + W[v][C];  // compile-time indices: operands stay in registers
            y[v][3] ^= 0x85EBCA6Bu;
#pragma unroll
            for (int i = 0; i <= C; i++) W[v][i] = W[v][i + C];
#pragma unroll
            for (int i = C + 1; i <= 2 * C; i++) W[v][i] = 0;
        }
    }
    __syncthreads();
    long long t1 = clock64();
    uint32_t s = 0;
#pragma unroll
    for (int v = 0; v < V; v++)
#pragma unroll
        for (int i = 0; i <= 2 * C; i++) s ^= W[v][i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) g_cyc[blockIdx.x] = t1 - t0;
}
template <int C, int V, int MODE>
void run(const char* name, int bps, double prods) {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t* d; cudaMalloc(&d, sizeof(uint32_t) * 128 * sms * bps);
    const int iters = 400;
    for (int r = 0; r < 2; r++) k_v<C, V, MODE><<<sms * bps, 128>>>(d, 7 + r, iters);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); return; }
    unsigned long long cyc[4096]; cudaMemcpyFromSymbol(cyc, g_cyc, sizeof(unsigned long long) * sms * bps);
    unsigned long long mx = 0; for (int i = 0; i < sms * bps; i++) mx = cyc[i] > mx ? cyc[i] : mx;
    cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, k_v<C, V, MODE>);
    double per_clk = prods * V * iters * 128.0 * bps / (double)mx;
    printf("{\"kernel\": \"%s\", \"V\": %d, \"ctas_per_sm\": %d, \"warps_per_sm\": %d, \"operand_streams_per_sm\": %d, \"regs\": %d, \"local_bytes\": %zu, \"products_per_clk_sm\": %.2f, \"pct_of_32\": %.1f}\n",
           name, V, bps, 4 * bps, 4 * bps * V, fa.numRegs, fa.localSizeBytes, per_clk, per_clk / 32 * 100);
    cudaFree(d);
}
int main() {
    for (int b : {1, 2, 3, 4}) run<16, 1, 0>("acc_mul", b, 256);
    for (int b : {1, 2, 3}) run<16, 2, 0>("acc_mul", b, 256);
    for (int b : {1, 2}) run<16, 3, 0>("acc_mul", b, 256);
    for (int b : {1, 2, 3, 4}) run<16, 1, 1>("acc_sqr", b, 136);
    for (int b : {1, 2, 3}) run<16, 2, 1>("acc_sqr", b, 136);
    return 0;
}
