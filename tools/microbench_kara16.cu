// Register-level one-level Karatsuba inside the 16-limb block product, against
// the engine's schoolbook block (acc_mul<16>, mp_block.cuh), on register operands.
//
//   schoolbook  W[0..32] += x*y: 256 fused IMAD.WIDE.U32.X products + the even/odd merge (63 adds)
//   karatsuba   x = x0 + x1 X, y = y0 + y1 X (X = 2^256, 8-limb halves):
//               D0 = x0 y0, D2 = x1 y1, Dm = |x0 - x1| |y0 - y1|, s = sign(x0 - x1) sign(y0 - y1)
//               W += D0 + (D0 + D2 - s Dm) X + D2 X^2   (192 products, the subtractive form of
//               P:L239-258 with reading A4: every half stays 8 limbs, the sign is a mask)
// Both are checked equal on random and all-ones operands, then timed with independent operands
// per iteration (the engine's situation: operands come from memory) at 1..4 CTAs of 128 threads
// per SM.  Rate = 256 (schoolbook-equivalent) products per block per clock per SM.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "../paper_2410_18129_b200/csrc/mp_block.cuh"
using namespace mpb;

#define CK(x)                                                                                    \
    do {                                                                                         \
        cudaError_t e = (x);                                                                     \
        if (e != cudaSuccess) {                                                                  \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));            \
            exit(1);                                                                             \
        }                                                                                        \
    } while (0)

// P[0..16) = a*b exactly for 8-limb a, b (E/O block product, odd array folded in)
__device__ __forceinline__ void mul8(const uint32_t (&a)[8], const uint32_t (&b)[8], uint32_t (&P)[16]) {
    uint32_t E[16], O[16];
    bp_mul<8>(a, b, E, O);
    fold_odd<8>(E, O);
#pragma unroll
    for (int i = 0; i < 16; i++) P[i] = E[i];
}
// d = |u - v| (8 limbs), returns 1 if u < v; branch-free (mask negation)
__device__ __forceinline__ uint32_t absdiff8(const uint32_t* u, const uint32_t* v, uint32_t (&d)[8]) {
#pragma unroll
    for (int i = 0; i < 8; i++) d[i] = u[i];
    sub_first(d[0], v[0]);
#pragma unroll
    for (int i = 1; i < 8; i++) sub_next(d[i], v[i]);
    const uint32_t b = bc_save();
    const uint32_t m = 0u - b;
#pragma unroll
    for (int i = 0; i < 8; i++) d[i] ^= m;
    add_first(d[0], b);
#pragma unroll
    for (int i = 1; i < 8; i++) add_next(d[i], 0u);
    return b;
}
// W[0..32] += x*y by one level of Karatsuba on 8-limb halves
__device__ __forceinline__ void acc_kara16(uint32_t (&W)[33], const uint32_t (&x)[16], const uint32_t (&y)[16]) {
    uint32_t x0[8], x1[8], y0[8], y1[8];
#pragma unroll
    for (int i = 0; i < 8; i++) { x0[i] = x[i]; x1[i] = x[8 + i]; y0[i] = y[i]; y1[i] = y[8 + i]; }
    uint32_t D0[16], D2[16], Dm[16], dx[8], dy[8];
    mul8(x0, y0, D0);
    mul8(x1, y1, D2);
    const uint32_t sx = absdiff8(x0, x1, dx), sy = absdiff8(y0, y1, dy);
    mul8(dx, dy, Dm);
    // mid = D0 + D2 - s*Dm (17 words, >= 0); subtract iff the signs agree (s = +1)
    const uint32_t m = 0u - ((sx ^ sy ^ 1u) & 1u);
    uint32_t mid[17];
#pragma unroll
    for (int i = 0; i < 16; i++) mid[i] = D0[i];
    mid[16] = 0;
    add_first(mid[0], D2[0]);
#pragma unroll
    for (int i = 1; i < 16; i++) add_next(mid[i], D2[i]);
    absorb(mid[16]);
    cc_restore(m & 1u);  // two's complement: + ~Dm + 1 when subtracting
#pragma unroll
    for (int i = 0; i < 16; i++) add_next(mid[i], Dm[i] ^ m);
    add_end(mid[16], m);
    // W += D0 + mid X + D2 X^2
    add_first(W[0], D0[0]);
#pragma unroll
    for (int i = 1; i < 16; i++) add_next(W[i], D0[i]);
#pragma unroll
    for (int i = 16; i < 32; i++) add_next(W[i], D2[i - 16]);
    absorb(W[32]);
    add_first(W[8], mid[0]);
#pragma unroll
    for (int i = 1; i < 17; i++) add_next(W[8 + i], mid[i]);
#pragma unroll
    for (int i = 25; i < 32; i++) add_next(W[i], 0u);
    absorb(W[32]);
}

template <int KARA>
__global__ void k_check(const uint32_t* xs, const uint32_t* ys, uint32_t* out) {
    const int t = threadIdx.x;
    uint32_t x[16], y[16], W[33];
    for (int i = 0; i < 16; i++) { x[i] = xs[t * 16 + i]; y[i] = ys[t * 16 + i]; }
    for (int i = 0; i < 33; i++) W[i] = (i < 20) ? xs[t * 16 + (i & 15)] ^ 0x5a5a5a5au : 0u;  // non-zero window
    if (KARA) acc_kara16(W, x, y);
    else acc_mul<16>(W, x, y);
    for (int i = 0; i < 33; i++) out[t * 33 + i] = W[i];
}

// independent operands per iteration (as in the engine); the window shifts down by 16 words
template <int KARA>
__global__ void __launch_bounds__(128) k_bench(uint32_t* out, uint32_t seed, int iters) {
    uint32_t x[16], y[16], W[33];
#pragma unroll
    for (int i = 0; i < 16; i++) {
        x[i] = seed * 2654435761u + threadIdx.x * 97u + i * 1013u;
        y[i] = seed * 40503u + threadIdx.x * 31u + i * 7919u;
    }
#pragma unroll
    for (int i = 0; i < 33; i++) W[i] = 0;
    uint32_t sink = 0;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 16; i++) { x[i] += (uint32_t)it; y[i] ^= (uint32_t)it * 0x9e3779b9u; }
        if (KARA) acc_kara16(W, x, y);
        else acc_mul<16>(W, x, y);
#pragma unroll
        for (int i = 0; i < 16; i++) sink ^= W[i];
#pragma unroll
        for (int i = 0; i <= 16; i++) W[i] = W[i + 16];
#pragma unroll
        for (int i = 17; i < 33; i++) W[i] = 0;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = sink ^ W[0];
}

int main(int argc, char** argv) {
    const int clk = argc > 1 ? atoi(argv[1]) : 1965;
    const int T = 128;
    static uint32_t hx[T * 16], hy[T * 16], h0[T * 33], h1[T * 33];
    srand(2410);
    for (int i = 0; i < T * 16; i++) {
        hx[i] = (uint32_t)rand() * 2654435761u ^ (uint32_t)rand();
        hy[i] = (uint32_t)rand() * 40503u ^ (uint32_t)rand();
        if ((i / 16) % 5 == 0) hx[i] = 0xFFFFFFFFu;  // all-ones rows (carry worst case)
        if ((i / 16) % 7 == 0) hy[i] = 0xFFFFFFFFu;
        if ((i / 16) % 11 == 1) hx[i] = (i % 16 < 8) ? 0u : 0xFFFFFFFFu;  // x0 < x1
    }
    uint32_t *dx, *dy, *dout;
    CK(cudaMalloc(&dx, sizeof hx)); CK(cudaMalloc(&dy, sizeof hy)); CK(cudaMalloc(&dout, sizeof h0));
    CK(cudaMemcpy(dx, hx, sizeof hx, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dy, hy, sizeof hy, cudaMemcpyHostToDevice));
    k_check<0><<<1, T>>>(dx, dy, dout);
    CK(cudaMemcpy(h0, dout, sizeof h0, cudaMemcpyDeviceToHost));
    k_check<1><<<1, T>>>(dx, dy, dout);
    CK(cudaMemcpy(h1, dout, sizeof h1, cudaMemcpyDeviceToHost));
    int bad = 0;
    for (int i = 0; i < T * 33; i++) bad += h0[i] != h1[i];
    printf("{\"check\": \"kara16 == schoolbook acc_mul<16> (window += x*y)\", \"rows\": %d, \"mismatched_words\": %d}\n", T, bad);
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    for (int kara = 0; kara < 2; kara++) {
        for (int b : {1, 2, 3, 4}) {
            const int n = sms * b, iters = 2000;
            uint32_t* d;
            CK(cudaMalloc(&d, sizeof(uint32_t) * 128 * n));
            auto launch = [&] {
                if (kara) k_bench<1><<<n, 128>>>(d, 7, iters);
                else k_bench<0><<<n, 128>>>(d, 7, iters);
            };
            launch();
            CK(cudaDeviceSynchronize());
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0); cudaEventCreate(&e1);
            cudaEventRecord(e0);
            for (int r = 0; r < 3; r++) launch();
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double blocks = (double)iters * 128.0 * n * 3;
            const double per_clk = blocks * 256.0 / (ms * 1e-3) / (sms * (double)clk * 1e6);
            cudaFuncAttributes fa;
            CK(cudaFuncGetAttributes(&fa, kara ? (const void*)k_bench<1> : (const void*)k_bench<0>));
            printf("{\"block\": \"%s\", \"ctas_per_sm\": %d, \"regs\": %d, \"ms\": %.3f, "
                   "\"schoolbook_equiv_products_per_clk_sm\": %.2f}\n",
                   kara ? "karatsuba 3 x 8x8" : "schoolbook 16x16", b, fa.numRegs, ms, per_clk);
            cudaFree(d);
        }
    }
    return 0;
}
