// Radix-2^52 FP64 block-product microbenchmark for sm_100a.
//
// A 52x52-bit word product a*b (a, b < 2^52 held exactly as doubles) is split with two FMAs:
//   hi = fma_rz(a, b, 2^104)            -> bits(hi) = (1127 << 52) | floor(ab / 2^52)
//   lo = fma_rn(a, b, (2^104 + 2^52) - hi)  -> bits(lo) = (1075 << 52) | (ab mod 2^52)
// (the subtraction is exact by Sterbenz; lo lies in [2^52, 2^53) so its ulp is 1).  The raw
// bit patterns are summed as 64-bit integers into column accumulators; the exponent bias only
// touches bits 52..63 and is removed per column at normalisation.  This measures the C x C
// block product on register operands (products per clock per SM) and checks it exactly
// against a host __int128 schoolbook.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ void dprod(double a, double b, uint64_t& clo, uint64_t& chi) {
    const double hi = __fma_rz(a, b, 0x1p104);
    const double sub = __dsub_rn(0x1.0000000000001p104, hi);
    const double lo = __fma_rn(a, b, sub);
    clo += (uint64_t)__double_as_longlong(lo);
    chi += (uint64_t)__double_as_longlong(hi);
}

template <int C>
__device__ __forceinline__ void dblk(uint64_t (&W)[2 * C], const double (&x)[C], const double (&y)[C]) {
#pragma unroll
    for (int i = 0; i < C; i++)
#pragma unroll
        for (int j = 0; j < C; j++) dprod(x[i], y[j], W[i + j], W[i + j + 1]);
}

__device__ unsigned long long g_cyc[8192];

template <int C>
__global__ void __launch_bounds__(128) k_bench(uint64_t* out, int iters) {
    double x[C], y[C];
    uint64_t W[2 * C];
#pragma unroll
    for (int i = 0; i < C; i++) {
        x[i] = (double)((threadIdx.x * 977u + i * 131u) & 0xFFFFFu) * 1024.0 + 12345.0;
        y[i] = (double)((threadIdx.x * 313u + i * 7u) & 0xFFFFFu) * 2048.0 + 777.0;
    }
#pragma unroll
    for (int i = 0; i < 2 * C; i++) W[i] = 0;
    uint64_t sink = 0;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
        dblk<C>(W, x, y);
#pragma unroll
        for (int i = 0; i < C; i++) x[i] = __dadd_rn(x[i], 1.0);  // every product changes (C extra DADD)
#pragma unroll
        for (int i = 0; i < C; i++) { sink ^= W[i]; W[i] = W[i + C]; }  // low columns are "stored"
#pragma unroll
        for (int i = C; i < 2 * C; i++) W[i] = 0;
    }
    __syncthreads();
    long long t1 = clock64();
    uint64_t s = sink;
#pragma unroll
    for (int i = 0; i < 2 * C; i++) s ^= W[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) g_cyc[blockIdx.x] = t1 - t0;
}

// exactness: one block product per thread on given limbs, normalised to 52-bit limbs
template <int C>
__global__ void k_check(const uint64_t* xa, const uint64_t* ya, uint64_t* out) {
    const int t = threadIdx.x;
    double x[C], y[C];
    for (int i = 0; i < C; i++) { x[i] = (double)xa[t * C + i]; y[i] = (double)ya[t * C + i]; }
    uint64_t W[2 * C];
    for (int i = 0; i < 2 * C; i++) W[i] = 0;
    dblk<C>(W, x, y);
    // bias: column k holds n_lo(k) lo patterns and n_hi(k) = n_lo(k-1) hi patterns
    uint64_t carry = 0;
    for (int k = 0; k < 2 * C; k++) {
        const int nlo = k <= 2 * C - 2 ? (k < C ? k + 1 : 2 * C - 1 - k) : 0;
        const int km = k - 1;
        const int nhi = km >= 0 ? (km < C ? km + 1 : 2 * C - 1 - km) : 0;
        const uint64_t bias = ((uint64_t)((nlo * 1075u + nhi * 1127u) & 0xFFFu)) << 52;
        const uint64_t v = W[k] - bias + carry;
        out[t * 2 * C + k] = v & ((1ull << 52) - 1);
        carry = v >> 52;
    }
}

template <int C>
void check() {
    const int T = 64;
    uint64_t hx[T * C], hy[T * C], ho[T * 2 * C];
    srand(12345);
    auto r52 = [] { return (((uint64_t)rand() << 40) ^ ((uint64_t)rand() << 20) ^ (uint64_t)rand()) & ((1ull << 52) - 1); };
    for (int i = 0; i < T * C; i++) {
        hx[i] = r52(); hy[i] = r52();
        if (i % 7 == 0) hx[i] = (1ull << 52) - 1;
        if (i % 5 == 0) hy[i] = (1ull << 52) - 1;
    }
    uint64_t *dx, *dy, *dout;
    CK(cudaMalloc(&dx, sizeof hx)); CK(cudaMalloc(&dy, sizeof hy)); CK(cudaMalloc(&dout, sizeof ho));
    CK(cudaMemcpy(dx, hx, sizeof hx, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dy, hy, sizeof hy, cudaMemcpyHostToDevice));
    k_check<C><<<1, T>>>(dx, dy, dout);
    CK(cudaMemcpy(ho, dout, sizeof ho, cudaMemcpyDeviceToHost));
    int bad = 0;
    for (int t = 0; t < T; t++) {
        unsigned __int128 col[2 * C + 1] = {0};
        for (int i = 0; i < C; i++)
            for (int j = 0; j < C; j++) {
                unsigned __int128 p = (unsigned __int128)hx[t * C + i] * hy[t * C + j];
                col[i + j] += p & ((1ull << 52) - 1);
                col[i + j + 1] += p >> 52;
            }
        unsigned __int128 c = 0;
        for (int k = 0; k < 2 * C; k++) {
            unsigned __int128 v = col[k] + c;
            if ((uint64_t)(v & ((1ull << 52) - 1)) != ho[t * 2 * C + k]) bad++;
            c = v >> 52;
        }
    }
    printf("{\"check\": \"C=%d dfma block product vs __int128\", \"threads\": %d, \"mismatched_limbs\": %d}\n", C, T, bad);
    cudaFree(dx); cudaFree(dy); cudaFree(dout);
}

template <int C>
void run(int ctas_per_sm) {
    int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const int n = sms * ctas_per_sm, iters = 200;
    uint64_t* d; CK(cudaMalloc(&d, sizeof(uint64_t) * 128 * n));
    for (int r = 0; r < 2; r++) k_bench<C><<<n, 128>>>(d, iters);
    CK(cudaDeviceSynchronize());
    static unsigned long long cyc[8192];
    CK(cudaMemcpyFromSymbol(cyc, g_cyc, sizeof(unsigned long long) * n));
    unsigned long long mx = 0;
    for (int i = 0; i < n; i++) mx = cyc[i] > mx ? cyc[i] : mx;
    const double p52 = (double)C * C * iters * 128.0 * ctas_per_sm / (double)mx;
    const double eq32 = p52 * (52.0 * 52.0) / (32.0 * 32.0);
    cudaFuncAttributes fa; CK(cudaFuncGetAttributes(&fa, k_bench<C>));
    printf("{\"C\": %d, \"ctas_per_sm\": %d, \"regs\": %d, \"p52_per_clk_sm\": %.2f, \"dfma_per_clk_sm\": %.2f, "
           "\"eq32_products_per_clk_sm\": %.2f, \"vs_imad_wide_peak_32\": %.3f}\n",
           C, ctas_per_sm, fa.numRegs, p52, 3 * p52, eq32, eq32 / 32.0);
    cudaFree(d);
}

int main() {
    check<8>();
    check<4>();
    for (int b : {2, 4, 6, 8}) run<8>(b);
    for (int b : {4, 8, 12}) run<4>(b);
    for (int b : {2, 3, 4}) run<12>(b);
    return 0;
}
