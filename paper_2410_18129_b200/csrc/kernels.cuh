// kernels.cuh -- the templated sm_100a kernels of libmpb.so and their launchers.
// Instantiated per shape (C, NB) in inst_L*.cu so the fully unrolled compiles run in
// parallel; api.cu holds the C ABI and only sees the Launch<C, NB> declarations.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "launch.h"
#include "mp_mont.cuh"

namespace mpb {

constexpr int kThreads = 128;

MPB_DEVI size_t tid_global() { return (size_t)blockIdx.x * blockDim.x + threadIdx.x; }
// word-sliced accessor for operand k of an array with `count` operands
MPB_DEVI GArr garr(uint32_t* base, size_t count, size_t k) { return GArr{reinterpret_cast<uint4*>(base) + k, count}; }
MPB_DEVI GIn gin(const uint32_t* base, size_t count, size_t k) {
    return GIn{reinterpret_cast<const uint4*>(base) + k, count};
}
// word i of operand k (32-bit access)
MPB_DEVI uint32_t word_at(const uint32_t* base, size_t count, size_t k, int i) {
    return __ldg(base + ((size_t)(i >> 2) * count + k) * 4 + (i & 3));
}

// ------------------------------------------------------------ product kernels
template <int C, int NB, bool SQR>
__global__ void __launch_bounds__(kThreads) k_mp_mul(const uint32_t* __restrict__ a, const uint32_t* __restrict__ b,
                                                     uint32_t* __restrict__ c, size_t count) {
    const size_t k = tid_global();
    if (k >= count) return;
    ph_product<C, NB, SQR>(gin(a, count, k), gin(SQR ? a : b, count, k), garr(c, count, k));
}

// workspace for the mont kernels: T (2L) then Q (L), word-sliced with stride count
template <int C, int NB, bool TRUNC, bool SQR>
__global__ void __launch_bounds__(kThreads) k_mont_mul(const uint32_t* __restrict__ a, const uint32_t* __restrict__ b,
                                                       const uint32_t* __restrict__ N, const uint32_t* __restrict__ NP,
                                                       uint32_t* __restrict__ c, size_t count, uint32_t* ws) {
    constexpr int L = C * NB;
    const size_t k = tid_global();
    if (k >= count) return;
    const GArr T = garr(ws, count, k);
    const GArr Q = garr(ws + (size_t)2 * L * count, count, k);
    mont_mul<C, NB, TRUNC, SQR>(gin(a, count, k), gin(SQR ? a : b, count, k), gin(N, count, k), gin(NP, count, k), T,
                                Q, garr(c, count, k));
}

template <int C, int NB, bool TRUNC>
__global__ void __launch_bounds__(kThreads) k_mont_redc(const uint32_t* __restrict__ Tin, const uint32_t* __restrict__ N,
                                                        const uint32_t* __restrict__ NP, uint32_t* __restrict__ c,
                                                        size_t count, uint32_t* ws) {
    constexpr int L = C * NB;
    const size_t k = tid_global();
    if (k >= count) return;
    const GArr T = garr(ws, count, k);
    const GArr Q = garr(ws + (size_t)2 * L * count, count, k);
    const GIn Ti = gin(Tin, count, k);
#pragma unroll 1
    for (int q = 0; q < 2 * L / 4; q++) T.st(q, Ti.ld(q));
    mont_redc<C, NB, TRUNC>(gin(N, count, k), gin(NP, count, k), T, Q, garr(c, count, k));
}

// ------------------------------------------------------------------- modexp
// workspace per operand (word-sliced, stride count): G (2^w * L) | Y (L) | T (2L) | Q (L) | S (L)
template <int C, int NB, bool TRUNC>
__global__ void __launch_bounds__(kThreads) k_modexp(const uint32_t* __restrict__ N, const uint32_t* __restrict__ NP,
                                                     const uint32_t* __restrict__ R2, const uint32_t* __restrict__ base,
                                                     const uint32_t* __restrict__ exp, uint32_t* __restrict__ out,
                                                     size_t count, int bits, int w, uint32_t* ws) {
    constexpr int L = C * NB;
    const size_t k = tid_global();
    if (k >= count) return;
    const int nent = 1 << w;
    uint32_t* p = ws;
    const GArr G = garr(p, count, k);
    p += (size_t)nent * L * count;
    const GArr Y = garr(p, count, k);
    p += (size_t)L * count;
    const GArr T = garr(p, count, k);
    p += (size_t)2 * L * count;
    const GArr Q = garr(p, count, k);
    p += (size_t)L * count;
    const GArr S = garr(p, count, k);
    const GIn Nn = gin(N, count, k), NPn = gin(NP, count, k), R2n = gin(R2, count, k), Bn = gin(base, count, k);
    auto Gent = [&](int e) { return GArr{G.p + (size_t)e * (L / 4) * count, count}; };

    // G[0] = R mod N = REDC(R^2)  (Montgomery one, SURVEY A11 "1 = R mod N")
#pragma unroll 1
    for (int q = 0; q < L / 4; q++) {
        T.st(q, R2n.ld(q));
        T.st(L / 4 + q, make_uint4(0, 0, 0, 0));
    }
    mont_redc<C, NB, TRUNC>(Nn, NPn, T, Q, Gent(0));
    // G[1] = base * R mod N = MontMul(base, R^2);  G[i] = MontMul(G[i-1], G[1])
    if (nent > 1) mont_mul<C, NB, TRUNC, false>(Bn, R2n, Nn, NPn, T, Q, Gent(1));
#pragma unroll 1
    for (int e = 2; e < nent; e++) mont_mul<C, NB, TRUNC, false>(Gent(e - 1), Gent(1), Nn, NPn, T, Q, Gent(e));

    // windows are LSB-aligned: window j covers exponent bits [j*w, j*w + w)
    const int nwin = (bits + w - 1) / w;
    auto window = [&](int j) -> uint32_t {
        const int pos = j * w;
        const int wi = pos >> 5, off = pos & 31;
        uint32_t v = word_at(exp, count, k, wi) >> off;
        if (off + w > 32 && wi + 1 < L) v |= word_at(exp, count, k, wi + 1) << (32 - off);
        return v & ((1u << w) - 1u);
    };
    // Y = G[top window] (the top partial window initialises Y; no epilogue)
    ct_select<L>(G, nent, window(nwin - 1), Y);
#pragma unroll 1
    for (int j = nwin - 2; j >= 0; j--) {
#pragma unroll 1
        for (int s = 0; s < w; s++) mont_mul<C, NB, TRUNC, true>(Y, Y, Nn, NPn, T, Q, Y);
        ct_select<L>(G, nent, window(j), S);
        mont_mul<C, NB, TRUNC, false>(Y, S, Nn, NPn, T, Q, Y);
    }
    // leave the Montgomery domain: out = REDC(Y)
#pragma unroll 1
    for (int q = 0; q < L / 4; q++) {
        T.st(q, Y.ld(q));
        T.st(L / 4 + q, make_uint4(0, 0, 0, 0));
    }
    mont_redc<C, NB, TRUNC>(Nn, NPn, T, Q, garr(out, count, k));
}


inline unsigned grid_for(size_t n) { return (unsigned)((n + kThreads - 1) / kThreads); }

template <int C, int NB>
void Launch<C, NB>::mp_mul(const uint32_t* a, const uint32_t* b, uint32_t* c, size_t count, bool sqr, cudaStream_t s) {
    if (sqr) k_mp_mul<C, NB, true><<<grid_for(count), kThreads, 0, s>>>(a, a, c, count);
    else k_mp_mul<C, NB, false><<<grid_for(count), kThreads, 0, s>>>(a, b, c, count);
}
template <int C, int NB>
void Launch<C, NB>::mont_mul(const uint32_t* a, const uint32_t* b, const uint32_t* N, const uint32_t* NP, uint32_t* c,
                             size_t count, bool trunc, bool sqr, uint32_t* ws, cudaStream_t s) {
    const unsigned g = grid_for(count);
    if (trunc) {
        if (sqr) k_mont_mul<C, NB, true, true><<<g, kThreads, 0, s>>>(a, a, N, NP, c, count, ws);
        else k_mont_mul<C, NB, true, false><<<g, kThreads, 0, s>>>(a, b, N, NP, c, count, ws);
    } else {
        if (sqr) k_mont_mul<C, NB, false, true><<<g, kThreads, 0, s>>>(a, a, N, NP, c, count, ws);
        else k_mont_mul<C, NB, false, false><<<g, kThreads, 0, s>>>(a, b, N, NP, c, count, ws);
    }
}
template <int C, int NB>
void Launch<C, NB>::mont_redc(const uint32_t* T, const uint32_t* N, const uint32_t* NP, uint32_t* c, size_t count,
                              bool trunc, uint32_t* ws, cudaStream_t s) {
    if (trunc) k_mont_redc<C, NB, true><<<grid_for(count), kThreads, 0, s>>>(T, N, NP, c, count, ws);
    else k_mont_redc<C, NB, false><<<grid_for(count), kThreads, 0, s>>>(T, N, NP, c, count, ws);
}
template <int C, int NB>
void Launch<C, NB>::modexp(const uint32_t* N, const uint32_t* NP, const uint32_t* R2, const uint32_t* base,
                           const uint32_t* exp, uint32_t* out, size_t count, int bits, int window, bool trunc,
                           uint32_t* ws, cudaStream_t s) {
    if (trunc) k_modexp<C, NB, true><<<grid_for(count), kThreads, 0, s>>>(N, NP, R2, base, exp, out, count, bits, window, ws);
    else k_modexp<C, NB, false><<<grid_for(count), kThreads, 0, s>>>(N, NP, R2, base, exp, out, count, bits, window, ws);
}

}  // namespace mpb
