// K0 integer-pipe microbenchmark for sm_100a (hard part H6).
//
// Measures warp-instruction throughput per SM per clock (in-kernel clock64) of
//   IMAD (lo), IMAD.HI.U32, IMAD.WIDE.U32, IMAD.WIDE.U32.X carry chains,
//   IADD3(.X) carry adds, the unfused lo/hi/carry product form, DFMA,
// and the dependent latency of an IMAD.WIDE.U32.X chain.  One CTA of 1024
// threads per SM (x 148), every thread runs K independent chains so the pipe,
// not latency, is the limit.  Output: one JSON object on stdout.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench_int microbench_int.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int ITERS = 256;

__device__ unsigned long long g_cycles[1024];

template <int K>
__global__ void k_imad_lo(uint32_t* out, uint32_t seed) {
    uint32_t x[K];
#pragma unroll
    for (int k = 0; k < K; k++) x[k] = threadIdx.x * (k + 3) + seed;
    uint32_t m = seed | 1;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < ITERS; it++) {
#pragma unroll
        for (int k = 0; k < K; k++) asm volatile("mad.lo.u32 %0, %0, %1, %0;" : "+r"(x[k]) : "r"(m));
    }
    __syncthreads();
    long long t1 = clock64();
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < K; k++) s ^= x[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
}

template <int K>
__global__ void k_imad_hi(uint32_t* out, uint32_t seed) {
    uint32_t x[K];
#pragma unroll
    for (int k = 0; k < K; k++) x[k] = threadIdx.x * (k + 3) + seed;
    uint32_t m = seed | 0x80000001u;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < ITERS; it++) {
#pragma unroll
        for (int k = 0; k < K; k++) asm volatile("mad.hi.u32 %0, %0, %1, %0;" : "+r"(x[k]) : "r"(m));
    }
    __syncthreads();
    long long t1 = clock64();
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < K; k++) s ^= x[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
}

// IMAD.WIDE.U32 (no carry): acc64 = x * m + acc64
template <int K>
__global__ void k_imad_wide(uint32_t* out, uint32_t seed) {
    unsigned long long acc[K];
    uint32_t x[K];
#pragma unroll
    for (int k = 0; k < K; k++) { acc[k] = threadIdx.x + k; x[k] = threadIdx.x * (k + 7) + seed; }
    uint32_t m = seed | 1;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < ITERS; it++) {
#pragma unroll
        for (int k = 0; k < K; k++) asm volatile("{ .reg .u32 lo; cvt.u32.u64 lo, %0; mad.wide.u32 %0, lo, %1, %0; }" : "+l"(acc[k]) : "r"(m));
    }
    __syncthreads();
    long long t1 = clock64();
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < K; k++) s ^= (uint32_t)(acc[k] ^ (acc[k] >> 32));
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
}

// IMAD.WIDE.U32.X carry chains: C independent accumulators of 2*P words, each iteration is one
// chain of P products  mad.lo.cc / madc.hi.cc  over aligned pairs (ptxas fuses each pair).
template <int C, int P>
__global__ void k_wide_chain(uint32_t* out, uint32_t seed) {
    uint32_t acc[C][2 * P + 2];
    uint32_t a[P];
#pragma unroll
    for (int j = 0; j < P; j++) a[j] = threadIdx.x * (j + 5) + seed;
#pragma unroll
    for (int c = 0; c < C; c++)
#pragma unroll
        for (int j = 0; j < 2 * P + 2; j++) acc[c][j] = c + j;
    uint32_t b = seed | 3;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < ITERS; it++) {
#pragma unroll
        for (int c = 0; c < C; c++) {
            asm volatile("mad.lo.cc.u32 %0, %2, %3, %0; madc.hi.cc.u32 %1, %2, %3, %1;" : "+r"(acc[c][0]), "+r"(acc[c][1]) : "r"(a[0]), "r"(b));
#pragma unroll
            for (int j = 1; j < P; j++)
                asm volatile("madc.lo.cc.u32 %0, %2, %3, %0; madc.hi.cc.u32 %1, %2, %3, %1;" : "+r"(acc[c][2 * j]), "+r"(acc[c][2 * j + 1]) : "r"(a[j]), "r"(b));
            asm volatile("addc.u32 %0, %0, 0;" : "+r"(acc[c][2 * P]));
        }
        b += 0x9E3779B9u;
    }
    __syncthreads();
    long long t1 = clock64();
    uint32_t s = 0;
#pragma unroll
    for (int c = 0; c < C; c++)
#pragma unroll
        for (int j = 0; j < 2 * P + 2; j++) s ^= acc[c][j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
}

// Unfused product form: lo chain then hi chain into the same accumulator (CGBN style).
template <int C, int P>
__global__ void k_lohi_chain(uint32_t* out, uint32_t seed) {
    uint32_t acc[C][P + 2];
    uint32_t a[P];
#pragma unroll
    for (int j = 0; j < P; j++) a[j] = threadIdx.x * (j + 5) + seed;
#pragma unroll
    for (int c = 0; c < C; c++)
#pragma unroll
        for (int j = 0; j < P + 2; j++) acc[c][j] = c + j;
    uint32_t b = seed | 3;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < ITERS; it++) {
#pragma unroll
        for (int c = 0; c < C; c++) {
            asm volatile("mad.lo.cc.u32 %0, %1, %2, %0;" : "+r"(acc[c][0]) : "r"(a[0]), "r"(b));
#pragma unroll
            for (int j = 1; j < P; j++) asm volatile("madc.lo.cc.u32 %0, %1, %2, %0;" : "+r"(acc[c][j]) : "r"(a[j]), "r"(b));
            asm volatile("addc.u32 %0, %0, 0;" : "+r"(acc[c][P]));
            asm volatile("mad.hi.cc.u32 %0, %1, %2, %0;" : "+r"(acc[c][1]) : "r"(a[0]), "r"(b));
#pragma unroll
            for (int j = 1; j < P; j++) asm volatile("madc.hi.cc.u32 %0, %1, %2, %0;" : "+r"(acc[c][j + 1]) : "r"(a[j]), "r"(b));
            asm volatile("addc.u32 %0, %0, 0;" : "+r"(acc[c][P + 1]));
        }
        b += 0x9E3779B9u;
    }
    __syncthreads();
    long long t1 = clock64();
    uint32_t s = 0;
#pragma unroll
    for (int c = 0; c < C; c++)
#pragma unroll
        for (int j = 0; j < P + 2; j++) s ^= acc[c][j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
}

// ALU carry adds: add.cc / addc.cc chains
template <int C, int P>
__global__ void k_addc(uint32_t* out, uint32_t seed) {
    uint32_t acc[C][P];
#pragma unroll
    for (int c = 0; c < C; c++)
#pragma unroll
        for (int j = 0; j < P; j++) acc[c][j] = threadIdx.x * (c + j + 1) + seed;
    uint32_t b = seed | 3;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < ITERS; it++) {
#pragma unroll
        for (int c = 0; c < C; c++) {
            asm volatile("add.cc.u32 %0, %0, %1;" : "+r"(acc[c][0]) : "r"(b));
#pragma unroll
            for (int j = 1; j < P; j++) asm volatile("addc.cc.u32 %0, %0, %1;" : "+r"(acc[c][j]) : "r"(b));
        }
        b += 0x9E3779B9u;
    }
    __syncthreads();
    long long t1 = clock64();
    uint32_t s = 0;
#pragma unroll
    for (int c = 0; c < C; c++)
#pragma unroll
        for (int j = 0; j < P; j++) s ^= acc[c][j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
}

template <int K>
__global__ void k_dfma(uint32_t* out, uint32_t seed) {
    double x[K];
#pragma unroll
    for (int k = 0; k < K; k++) x[k] = (double)(threadIdx.x + k + seed);
    double m = 1.0000001, c = 0.5;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < ITERS; it++) {
#pragma unroll
        for (int k = 0; k < K; k++) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(x[k]) : "d"(m), "d"(c));
    }
    __syncthreads();
    long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int k = 0; k < K; k++) s += x[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = (uint32_t)s;
    if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
}

// dependent latency of an IMAD.WIDE.U32.X chain: one thread runs k_wide_chain<1,8>
template <typename F>
static int run(const char* name, F kern, double ops_per_thread, int threads, uint32_t* d_out, int sms, int first) {
    for (int rep = 0; rep < 2; rep++) {
        kern<<<sms, threads>>>(d_out, 12345u + rep);
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
    }
    unsigned long long cyc[1024];
    CK(cudaMemcpyFromSymbol(cyc, g_cycles, sizeof(unsigned long long) * sms));
    unsigned long long mx = 0, mn = ~0ull;
    for (int i = 0; i < sms; i++) { if (cyc[i] > mx) mx = cyc[i]; if (cyc[i] < mn) mn = cyc[i]; }
    double per_clk = ops_per_thread * threads / (double)mx;  // thread-ops per SM per clock
    printf("%s  \"%s\": {\"thread_ops_per_clk_per_sm\": %.2f, \"cycles_max\": %llu, \"cycles_min\": %llu}",
           first ? "" : ",\n", name, per_clk, mx, mn);
    return 0;
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
    uint32_t* d_out;
    CK(cudaMalloc(&d_out, sizeof(uint32_t) * 1024 * sms));
    printf("{\"sms\": %d, \"clock_rate_khz\": %d,\n", sms, clk);
    const int T = 1024;
    run("imad_lo", k_imad_lo<8>, 8.0 * ITERS, T, d_out, sms, 1);
    run("imad_hi", k_imad_hi<8>, 8.0 * ITERS, T, d_out, sms, 0);
    run("imad_wide", k_imad_wide<8>, 8.0 * ITERS, T, d_out, sms, 0);
    run("wide_chain_products", k_wide_chain<2, 8>, 2.0 * 8 * ITERS, 512, d_out, sms, 0);
    run("wide_chain_products_c4", k_wide_chain<4, 4>, 4.0 * 4 * ITERS, 512, d_out, sms, 0);
    run("lohi_chain_products", k_lohi_chain<2, 8>, 2.0 * 8 * ITERS, 512, d_out, sms, 0);
    run("addc_ops", k_addc<4, 8>, 4.0 * 8 * ITERS, T, d_out, sms, 0);
    run("dfma", k_dfma<8>, 8.0 * ITERS, T, d_out, sms, 0);
    {
        k_wide_chain<1, 8><<<1, 32>>>(d_out, 7);
        CK(cudaDeviceSynchronize());
        k_wide_chain<1, 8><<<1, 32>>>(d_out, 7);
        CK(cudaDeviceSynchronize());
        unsigned long long c;
        CK(cudaMemcpyFromSymbol(&c, g_cycles, sizeof(c)));
        printf(",\n  \"wide_chain_latency_cycles_per_product\": %.2f", c / (ITERS * 8.0));
        k_lohi_chain<1, 8><<<1, 32>>>(d_out, 7);
        CK(cudaDeviceSynchronize());
        CK(cudaMemcpyFromSymbol(&c, g_cycles, sizeof(c)));
        printf(",\n  \"lohi_chain_latency_cycles_per_product\": %.2f", c / (ITERS * 8.0));
    }
    printf("\n}\n");
    return 0;
}
