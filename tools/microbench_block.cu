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

// Accumulate model: persistent even/odd accumulators and per-position carry catchers.
//   E[p]      words at positions p = 0..2C-1 (pairs at even positions)
//   O[k]      word at position k+1, k = 0..2C-3 (pairs at odd positions)
//   K[k]      carry counts at position C+k, k = 0..C
// Every row chain is an exact multi-word addition whose final carry is caught in K, so many
// block products accumulate with no per-block merge.
template <int C>
__device__ __forceinline__ void acca_mul(uint32_t (&E)[2 * C], uint32_t (&O)[2 * C - 2], uint32_t (&K)[C + 1],
                                         const uint32_t (&x)[C], const uint32_t (&y)[C]) {
#pragma unroll
    for (int i = 0; i < C; i++) {
        {
            const int j0 = i & 1;
#pragma unroll
            for (int j = j0; j < C; j += 2) {
                if (j == j0) pr_first(E[i + j], E[i + j + 1], x[j], y[i]);
                else pr_next(E[i + j], E[i + j + 1], x[j], y[i]);
            }
            const int jl = (C - 1 - j0) & ~1 | j0;  // last j with j == j0 (mod 2)
            absorb(K[i + (j0 == 0 ? C - 2 : C - 1) + 2 - C]);
            (void)jl;
        }
        {
            const int j0 = (i & 1) ^ 1;
#pragma unroll
            for (int j = j0; j < C; j += 2) {
                if (j == j0) pr_first(O[i + j - 1], O[i + j], x[j], y[i]);
                else pr_next(O[i + j - 1], O[i + j], x[j], y[i]);
            }
            absorb(K[i + (j0 == 0 ? C - 2 : C - 1) + 2 - C]);
        }
    }
}
// V = E + O*2^32(shifted) + K*2^(32C): low C words to out (xor sink), the top C+1 words become
// the next column's E[0..C]; O and K restart at zero.
template <int C>
__device__ __forceinline__ uint32_t acca_merge(uint32_t (&E)[2 * C], uint32_t (&O)[2 * C - 2], uint32_t (&K)[C + 1]) {
    uint32_t top = 0;
    add_first(E[1], O[0]);
#pragma unroll
    for (int k = 1; k < 2 * C - 2; k++) add_next(E[k + 1], O[k]);
    add_next(E[2 * C - 1], 0u);
    absorb(top);
    add_first(E[C], K[0]);
#pragma unroll
    for (int k = 1; k < C; k++) add_next(E[C + k], K[k]);
    add_end(top, K[C]);
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < C; k++) s ^= E[k];
#pragma unroll
    for (int k = 0; k < C; k++) E[k] = E[k + C];
    E[C] = top;
#pragma unroll
    for (int k = C + 1; k < 2 * C; k++) E[k] = 0;
#pragma unroll
    for (int k = 0; k < 2 * C - 2; k++) O[k] = 0;
#pragma unroll
    for (int k = 0; k <= C; k++) K[k] = 0;
    return s;
}

template <int C, int PER>
__global__ void __launch_bounds__(128) k_acca(uint32_t* out, uint32_t seed, int iters) {
    uint32_t x[C], y[C], E[2 * C], O[2 * C - 2], K[C + 1];
#pragma unroll
    for (int i = 0; i < C; i++) { x[i] = seed * (i + 3) + threadIdx.x; y[i] = seed ^ (i * 77 + threadIdx.x); }
#pragma unroll
    for (int i = 0; i < 2 * C; i++) E[i] = 0;
#pragma unroll
    for (int i = 0; i < 2 * C - 2; i++) O[i] = 0;
#pragma unroll
    for (int i = 0; i <= C; i++) K[i] = 0;
    uint32_t sink = 0;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
#pragma unroll 1
        for (int b = 0; b < PER; b++) {
            acca_mul<C>(E, O, K, x, y);
            x[0] += 0x9E3779B9u; y[C - 1] ^= 0x85EBCA6Bu;
        }
        sink ^= acca_merge<C>(E, O, K);
    }
    __syncthreads();
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = sink ^ E[0] ^ O[3] ^ K[2];
    if (threadIdx.x == 0) g_cyc[blockIdx.x] = t1 - t0;
}

// exactness of the accumulate model: PER block products of random blocks vs a plain schoolbook
template <int C, int PER>
__global__ void k_acca_check(const uint32_t* xs, const uint32_t* ys, uint32_t* out) {
    uint32_t x[C], y[C], E[2 * C], O[2 * C - 2], K[C + 1];
    for (int i = 0; i < 2 * C; i++) E[i] = 0;
    for (int i = 0; i < 2 * C - 2; i++) O[i] = 0;
    for (int i = 0; i <= C; i++) K[i] = 0;
    const int t = threadIdx.x;
    for (int b = 0; b < PER; b++) {
        for (int i = 0; i < C; i++) { x[i] = xs[(t * PER + b) * C + i]; y[i] = ys[(t * PER + b) * C + i]; }
        acca_mul<C>(E, O, K, x, y);
    }
    // full value, no shift: E + O + K
    uint32_t top = 0;
    add_first(E[1], O[0]);
    for (int k = 1; k < 2 * C - 2; k++) add_next(E[k + 1], O[k]);
    add_next(E[2 * C - 1], 0u);
    absorb(top);
    add_first(E[C], K[0]);
    for (int k = 1; k < C; k++) add_next(E[C + k], K[k]);
    add_end(top, K[C]);
    for (int k = 0; k < 2 * C; k++) out[t * (2 * C + 1) + k] = E[k];
    out[t * (2 * C + 1) + 2 * C] = top;
}

template <int C, int PER>
void check_acca() {
    const int T = 64;
    static uint32_t hx[T * PER * C], hy[T * PER * C], ho[T * (2 * C + 1)];
    srand(7);
    for (int i = 0; i < T * PER * C; i++) {
        hx[i] = ((uint32_t)rand() << 16) ^ (uint32_t)rand();
        hy[i] = ((uint32_t)rand() << 16) ^ (uint32_t)rand();
        if (i % 3 == 0) hx[i] = 0xFFFFFFFFu;
        if (i % 2 == 0) hy[i] = 0xFFFFFFFFu;
    }
    uint32_t *dx, *dy, *dout;
    cudaMalloc(&dx, sizeof hx); cudaMalloc(&dy, sizeof hy); cudaMalloc(&dout, sizeof ho);
    cudaMemcpy(dx, hx, sizeof hx, cudaMemcpyHostToDevice); cudaMemcpy(dy, hy, sizeof hy, cudaMemcpyHostToDevice);
    k_acca_check<C, PER><<<1, T>>>(dx, dy, dout);
    cudaMemcpy(ho, dout, sizeof ho, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int t = 0; t < T; t++) {
        unsigned long long acc[2 * C + 2] = {0};
        for (int b = 0; b < PER; b++)
            for (int i = 0; i < C; i++)
                for (int j = 0; j < C; j++) {
                    unsigned long long p = (unsigned long long)hx[(t * PER + b) * C + j] * hy[(t * PER + b) * C + i];
                    acc[i + j] += (uint32_t)p;
                    acc[i + j + 1] += p >> 32;
                }
        unsigned long long c = 0;
        for (int k = 0; k <= 2 * C; k++) {
            unsigned long long v = acc[k] + c;
            if ((uint32_t)v != ho[t * (2 * C + 1) + k]) bad++;
            c = v >> 32;
        }
    }
    printf("acca exactness C=%d PER=%d: mismatched words %d\n", C, PER, bad);
    cudaFree(dx); cudaFree(dy); cudaFree(dout);
}
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
template <int C, int PER>
void run_acca(const char* name, int blocks_per_sm) {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t* d; cudaMalloc(&d, sizeof(uint32_t) * 128 * sms * blocks_per_sm);
    const int iters = 100;
    for (int r = 0; r < 2; r++) k_acca<C, PER><<<sms * blocks_per_sm, 128>>>(d, 7 + r, iters);
    cudaDeviceSynchronize();
    unsigned long long cyc[4096]; cudaMemcpyFromSymbol(cyc, g_cyc, sizeof(unsigned long long) * sms * blocks_per_sm);
    unsigned long long mx = 0; for (int i = 0; i < sms * blocks_per_sm; i++) mx = cyc[i] > mx ? cyc[i] : mx;
    double per_clk = (double)C * C * PER * iters * 128.0 * blocks_per_sm / (double)mx;
    cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, k_acca<C, PER>);
    printf("%-40s C=%2d ctas/SM=%d regs=%d products/clk/SM=%.2f  (%.1f%% of 32)\n", name, C, blocks_per_sm, fa.numRegs, per_clk, per_clk / 32 * 100);
    cudaFree(d);
}

int main() {
    check_acca<16, 3>();
    check_acca<8, 5>();
    for (int b : {2, 3, 4}) {
        run_acca<16, 1>("acca_mul, merge every block", b);
        run_acca<16, 2>("acca_mul, merge every 2 blocks", b);
        run_acca<16, 4>("acca_mul, merge every 4 blocks", b);
    }
    for (int b : {4, 6, 8}) run_acca<8, 4>("acca_mul C=8, merge every 4", b);
    for (int b : {2, 3}) {
        run<16, 0>("acc_mul dependent", b, 256);
        run<16, 3>("acc_mul independent", b, 256);
        run<16, 6>("acc_mul2 independent", b, 256);
        run<16, 1>("acc_sqr dependent", b, 136);
        run<16, 5>("acc_sqr independent", b, 136);
    }
    return 0;
}
