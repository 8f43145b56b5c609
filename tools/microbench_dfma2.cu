// Radix-2^52 FP64 block-product microbenchmark, v2: the column-window form the
// DFMA engine uses.  Each 52x52-bit product a*b (a, b < 2^52 exact in doubles) is split by
//   hi = fma_rz(a, b, 2^104)                 bits(hi) = (1127 << 52) | floor(ab / 2^52)
//   lo = fma_rn(a, b, (2^104 + 2^52) - hi)    bits(lo) = (1075 << 52) | (ab mod 2^52)
// and the raw patterns of a block column are summed into 64-bit column accumulators with
// THREE-input adds (IADD3 + IADD3.X with two carry predicates: 2 ALU instructions per 2 patterns),
// i.e. 3 FP64 + 2 ALU instructions per product.  The exponent biases are removed once per column.
// Measures products per clock per SM (CUDA events over the whole grid, at the sampled clock) for
// C x C blocks at several occupancies, and checks exactness against a host __int128 schoolbook.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                                    \
    do {                                                                                         \
        cudaError_t e = (x);                                                                     \
        if (e != cudaSuccess) {                                                                  \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));            \
            exit(1);                                                                             \
        }                                                                                        \
    } while (0)

__device__ __forceinline__ void dprod(double a, double b, uint64_t& lo, uint64_t& hi) {
    const double h = __fma_rz(a, b, 0x1p104);
    const double sub = __dsub_rn(0x1.0000000000001p104, h);
    const double l = __fma_rn(a, b, sub);
    lo = (uint64_t)__double_as_longlong(l);
    hi = (uint64_t)__double_as_longlong(h);
}

// W[0..2C] += x*y as raw patterns (biased), column by column, 3-input adds.
template <int C>
__device__ __forceinline__ void dblk(uint64_t (&W)[2 * C + 1], const double (&x)[C], const double (&y)[C]) {
    uint64_t ph[C];
    int nph = 0;
#pragma unroll
    for (int p = 0; p < 2 * C - 1; p++) {
        uint64_t t[2 * C];
        int n = 0;
        uint64_t nh[C];
        int nn = 0;
#pragma unroll
        for (int i = 0; i < C; i++) {
            const int j = p - i;
            if (j >= 0 && j < C) {
                uint64_t lo, hi;
                dprod(x[i], y[j], lo, hi);
                t[n++] = lo;
                nh[nn++] = hi;
            }
        }
#pragma unroll
        for (int i = 0; i < nph; i++) t[n++] = ph[i];
        uint64_t s = W[p];
#pragma unroll
        for (int i = 0; i + 1 < n; i += 2) s = s + t[i] + t[i + 1];
        if (n & 1) s += t[n - 1];
        W[p] = s;
#pragma unroll
        for (int i = 0; i < nn; i++) ph[i] = nh[i];
        nph = nn;
    }
    uint64_t s = W[2 * C - 1];
#pragma unroll
    for (int i = 0; i + 1 < nph; i += 2) s = s + ph[i] + ph[i + 1];
    if (nph & 1) s += ph[nph - 1];
    W[2 * C - 1] = s;
}

template <int C>
__global__ void __launch_bounds__(128) k_bench(uint64_t* out, int iters) {
    double x[C], y[C];
    uint64_t W[2 * C + 1];
#pragma unroll
    for (int i = 0; i < C; i++) {
        x[i] = (double)((threadIdx.x * 977u + i * 131u) & 0xFFFFFu) * 1024.0 + 12345.0;
        y[i] = (double)((threadIdx.x * 313u + i * 7u) & 0xFFFFFu) * 2048.0 + 777.0;
    }
#pragma unroll
    for (int i = 0; i <= 2 * C; i++) W[i] = 0;
    uint64_t sink = 0;
    for (int it = 0; it < iters; it++) {
        dblk<C>(W, x, y);
#pragma unroll
        for (int i = 0; i < C; i++) x[i] = __dadd_rn(x[i], 1.0);
#pragma unroll
        for (int i = 0; i < C; i++) {
            sink ^= W[i];
            W[i] = W[i + C];
        }
#pragma unroll
        for (int i = C; i <= 2 * C; i++) W[i] = 0;
    }
    uint64_t s = sink;
#pragma unroll
    for (int i = 0; i <= 2 * C; i++) s ^= W[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int C>
__global__ void k_check(const uint64_t* xa, const uint64_t* ya, uint64_t* out) {
    const int t = threadIdx.x;
    double x[C], y[C];
    for (int i = 0; i < C; i++) {
        x[i] = (double)xa[t * C + i];
        y[i] = (double)ya[t * C + i];
    }
    uint64_t W[2 * C + 1];
    for (int i = 0; i <= 2 * C; i++) W[i] = 0;
    dblk<C>(W, x, y);
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
    static uint64_t hx[T * C], hy[T * C], ho[T * 2 * C];
    srand(12345 + C);
    auto r52 = [] {
        return (((uint64_t)rand() << 40) ^ ((uint64_t)rand() << 20) ^ (uint64_t)rand()) & ((1ull << 52) - 1);
    };
    for (int i = 0; i < T * C; i++) {
        hx[i] = r52();
        hy[i] = r52();
        if (i % 7 == 0) hx[i] = (1ull << 52) - 1;
        if (i % 5 == 0) hy[i] = (1ull << 52) - 1;
    }
    uint64_t *dx, *dy, *dout;
    CK(cudaMalloc(&dx, sizeof hx));
    CK(cudaMalloc(&dy, sizeof hy));
    CK(cudaMalloc(&dout, sizeof ho));
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
    printf("{\"check\": \"C=%d dfma2 block product vs __int128\", \"threads\": %d, \"mismatched_limbs\": %d}\n", C, T,
           bad);
    cudaFree(dx);
    cudaFree(dy);
    cudaFree(dout);
}

template <int C>
void run(int ctas_per_sm, int clk_mhz) {
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const int n = sms * ctas_per_sm, iters = 400;
    uint64_t* d;
    CK(cudaMalloc(&d, sizeof(uint64_t) * 128 * n));
    k_bench<C><<<n, 128>>>(d, iters);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    const int reps = 5;
    for (int r = 0; r < reps; r++) k_bench<C><<<n, 128>>>(d, iters);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double prods = (double)C * C * iters * 128.0 * n * reps;
    const double p52 = prods / (ms * 1e-3) / (sms * (double)clk_mhz * 1e6);
    cudaFuncAttributes fa;
    CK(cudaFuncGetAttributes(&fa, k_bench<C>));
    printf("{\"C\": %d, \"ctas_per_sm\": %d, \"warps_per_sm\": %d, \"regs\": %d, \"ms\": %.3f, \"p52_per_clk_sm\": %.2f, "
           "\"fp64_ops_per_clk_sm\": %.1f, \"eq32_products_per_clk_sm\": %.2f, \"vs_imad_wide_31.1\": %.3f, \"clk_mhz\": %d}\n",
           C, ctas_per_sm, 4 * ctas_per_sm, fa.numRegs, ms, p52, 3 * p52, p52 * 2704.0 / 1024.0,
           p52 * 2704.0 / 1024.0 / 31.1, clk_mhz);
    cudaFree(d);
}

int main(int argc, char** argv) {
    const int clk = argc > 1 ? atoi(argv[1]) : 1965;
    check<8>();
    check<4>();
    check<6>();
    for (int b : {1, 2, 3, 4, 6}) run<8>(b, clk);
    for (int b : {2, 4, 8}) run<4>(b, clk);
    for (int b : {2, 3, 4}) run<6>(b, clk);
    for (int b : {1, 2, 3}) run<12>(b, clk);
    return 0;
}
