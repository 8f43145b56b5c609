// FP64 pipe rates on sm_100a for the radix-2^52 product split (tools/microbench_dfma.cu):
// DFMA (rn), DFMA.RZ, DADD, the 3-op split sequence alone, and the split plus the 64-bit
// integer accumulation, each with K independent streams per thread (throughput, not latency).
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ unsigned long long g_cyc[8192];
constexpr int ITERS = 256, K = 8;

template <int MODE>
__global__ void __launch_bounds__(256, 1) k_fp(double* out, double seed) {
    double a[K], b[K], c[K];
    uint64_t acc[K];
#pragma unroll
    for (int k = 0; k < K; k++) {
        a[k] = seed * (k + 1) + threadIdx.x;
        b[k] = seed + 3 * k;
        c[k] = 0;
        acc[k] = 0;
    }
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < ITERS; it++) {
#pragma unroll
        for (int k = 0; k < K; k++) {
            if (MODE == 0) c[k] = __fma_rn(a[k], b[k], c[k]);
            if (MODE == 1) c[k] = __fma_rz(a[k], b[k], c[k]);
            if (MODE == 2) c[k] = __dadd_rn(c[k], a[k]);
            if (MODE == 3 || MODE == 4) {  // the product split; a[k] varies so nothing is loop-invariant
                const double hi = __fma_rz(a[k], b[k], 0x1p104);
                const double sub = __dsub_rn(0x1.0000000000001p104, hi);
                const double lo = __fma_rn(a[k], b[k], sub);
                if (MODE == 3) { c[k] = __dadd_rn(c[k], lo); a[k] = hi; }
                else { acc[k] += (uint64_t)__double_as_longlong(lo) + (uint64_t)__double_as_longlong(hi); a[k] = lo; }
            }
            if (MODE == 6 || MODE == 7 || MODE == 8) {
                const double hi = __fma_rz(a[k], b[k], 0x1p104);
                const double sub = __dsub_rn(0x1.0000000000001p104, hi);
                const double lo = __fma_rn(a[k], b[k], sub);
                if (MODE == 6) { acc[k] += (uint64_t)__double_as_longlong(lo); c[k] = __longlong_as_double(__double_as_longlong(c[k]) + __double_as_longlong(hi)); }
                if (MODE == 7) acc[k] += (uint32_t)__double_as_longlong(lo) + (uint32_t)__double_as_longlong(hi);
                if (MODE == 8) acc[k] += (uint32_t)__double_as_longlong(lo);
                a[k] = lo;
            }
            if (MODE == 9) {  // split, no accumulation at all beyond the chain (3 fp64 ops)
                const double hi = __fma_rz(a[k], b[k], 0x1p104);
                const double sub = __dsub_rn(0x1.0000000000001p104, hi);
                a[k] = __fma_rn(a[k], b[k], sub);
            }
            if (MODE == 5) {  // split with an fma-form subtraction: sub = fma(hi, -1, c2)
                const double hi = __fma_rz(a[k], b[k], 0x1p104);
                const double sub = __fma_rn(hi, -1.0, 0x1.0000000000001p104);
                const double lo = __fma_rn(a[k], b[k], sub);
                acc[k] += (uint64_t)__double_as_longlong(lo) + (uint64_t)__double_as_longlong(hi);
                a[k] = lo;
            }
        }
    }
    __syncthreads();
    long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int k = 0; k < K; k++) s += c[k] + a[k] + (double)acc[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) g_cyc[blockIdx.x] = t1 - t0;
}

template <int MODE>
int run(const char* name, double ops_per_k, int ctas) {
    int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const int n = sms * ctas;
    double* d; CK(cudaMalloc(&d, sizeof(double) * 256 * n));
    for (int r = 0; r < 2; r++) k_fp<MODE><<<n, 256>>>(d, 1.5 + r);
    CK(cudaDeviceSynchronize());
    static unsigned long long cyc[8192];
    CK(cudaMemcpyFromSymbol(cyc, g_cyc, sizeof(unsigned long long) * n));
    unsigned long long mx = 0;
    for (int i = 0; i < n; i++) mx = cyc[i] > mx ? cyc[i] : mx;
    const double per = ops_per_k * K * ITERS * 256.0 * ctas / (double)mx;
    printf("{\"op\": \"%s\", \"ctas_per_sm\": %d, \"thread_ops_per_clk_per_sm\": %.2f}\n", name, ctas, per);
    cudaFree(d);
    return 0;
}

int main() {
    for (int c : {2, 4, 8}) {
        run<0>("dfma_rn", 1, c);
        run<1>("dfma_rz", 1, c);
        run<2>("dadd", 1, c);
        run<3>("split_fp_only (4 fp64 ops: rz, dadd, rn, dadd)", 4, c);
        run<4>("split+int64 acc (3 fp64 ops per product)", 3, c);
        run<5>("split with fma-form sub + int64 acc (3 fp64 ops)", 3, c);
        run<6>("split + two 2-input int64 adds", 3, c);
        run<7>("split + one 32-bit IADD3", 3, c);
        run<8>("split + one 32-bit IADD", 3, c);
        run<9>("split only (3 fp64 ops)", 3, c);
    }
    return 0;
}
