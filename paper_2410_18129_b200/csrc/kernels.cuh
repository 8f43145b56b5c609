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
// resident CTAs per SM the modexp kernel is compiled for (register budget 65536 / (128 * minb))
template <int C>
__host__ __device__ constexpr int modexp_min_blocks() { return C >= 12 ? 3 : 5; }
// entries of the CT table scan kept in flight per step (register budget)
template <int C>
__host__ __device__ constexpr int select_unroll() {
#ifdef MPB_SEL_U
    return MPB_SEL_U;
#else
    return 4;  // measured best at L = 64 (U = 4 entries x 4 chunks in flight; 8 x 4 and 1 x 8 are slower)
#endif
}

MPB_DEVI size_t tid_global() { return (size_t)blockIdx.x * blockDim.x + threadIdx.x; }
// word-sliced accessor for operand k of an array with `count` operands
MPB_DEVI Arr arr(const uint32_t* base, size_t count, size_t k) {
    return Arr{reinterpret_cast<char*>(const_cast<uint32_t*>(base)) + k * 16, (uint32_t)(count * 16)};
}
// this thread's staging area in dynamic shared memory (2 buffers x 2 blocks x C/4 chunks)
template <int C>
MPB_DEVI Stage stage() {
    extern __shared__ uint4 smem_stage[];
    return Stage{(uint32_t)__cvta_generic_to_shared(smem_stage + threadIdx.x), (uint32_t)(blockDim.x * 16)};
}
template <int C>
constexpr size_t stage_bytes() { return (size_t)kThreads * 4 * (C / 4) * 16; }
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
    uint32_t orlo = 0, tl1 = 0;
    const Arr C_ = arr(c, count, k);
    engine<C, NB, true>(SQR ? PH_SQR : PH_MUL, arr(a, count, k), arr(SQR ? a : b, count, k), C_, C_, C_, C_, orlo,
                        tl1, stage<C>());
}

// workspace for the mont kernels: T (2L) then Q (L), word-sliced with stride count
template <int C, int NB, bool TRUNC, bool SQR>
__global__ void __launch_bounds__(kThreads) k_mont_mul(const uint32_t* __restrict__ a, const uint32_t* __restrict__ b,
                                                       const uint32_t* __restrict__ N, const uint32_t* __restrict__ NP,
                                                       uint32_t* __restrict__ c, size_t count, uint32_t* ws) {
    constexpr int L = C * NB;
    const size_t k = tid_global();
    if (k >= count) return;
    const Arr T = arr(ws, count, k), Q = arr(ws + (size_t)2 * L * count, count, k);
    mont_op<C, NB, TRUNC>(SQR ? MODE_SQR : MODE_MUL, arr(a, count, k), arr(SQR ? a : b, count, k), arr(N, count, k),
                          arr(NP, count, k), T, Q, arr(c, count, k), stage<C>());
}

template <int C, int NB, bool TRUNC>
__global__ void __launch_bounds__(kThreads) k_mont_redc(const uint32_t* __restrict__ Tin, const uint32_t* __restrict__ N,
                                                        const uint32_t* __restrict__ NP, uint32_t* __restrict__ c,
                                                        size_t count, uint32_t* ws) {
    constexpr int L = C * NB;
    const size_t k = tid_global();
    if (k >= count) return;
    const Arr T = arr(ws, count, k), Q = arr(ws + (size_t)2 * L * count, count, k);
    const Arr Ti = arr(Tin, count, k);
#pragma unroll 1
    for (int q = 0; q < 2 * L / 4; q++) T.st(q, Ti.ld(q));
    mont_op<C, NB, TRUNC>(MODE_REDC, T, T, arr(N, count, k), arr(NP, count, k), T, Q, arr(c, count, k), stage<C>());
}

// ------------------------------------------------------------------- modexp
// alg:8FWExp as one flat, public schedule of operations so that the kernel
// holds a single instance of the Montgomery engine:
//   op 0             G[0] = REDC(R^2) = R mod N               (Montgomery one)
//   op 1             G[1] = MontMul(base, R^2)
//   op e < 2^w       G[e] = MontMul(G[e-1], G[1])
//   op 2^w           Y = CTsel(G, top window)                  (windows LSB-aligned, A11)
//   then per window j = W-2 .. 0:  w x Y = MontSqr(Y),  S = CTsel(G, window j)
//                                  (P:L765-766),  Y = MontMul(Y, S)
//   last op          out = REDC(Y)
// workspace per operand (word-sliced, stride count): G (2^w * L) | Y (L) | T (2L) | Q (L) | S (L)
template <int C, int NB, bool TRUNC>
__global__ void __launch_bounds__(kThreads, modexp_min_blocks<C>()) k_modexp(const uint32_t* __restrict__ N, const uint32_t* __restrict__ NP,
                                                     const uint32_t* __restrict__ R2, const uint32_t* __restrict__ base,
                                                     const uint32_t* __restrict__ exp, uint32_t* __restrict__ out,
                                                     size_t count, int bits, int w, uint32_t* ws) {
    constexpr int L = C * NB, Q4 = L / 4;
    const size_t k = tid_global();
    if (k >= count) return;
    const int nent = 1 << w;
    uint32_t* p = ws;
    const Arr G = arr(p, count, k);
    p += (size_t)nent * L * count;
    const Arr Y = arr(p, count, k);
    p += (size_t)L * count;
    const Arr T = arr(p, count, k);
    p += (size_t)2 * L * count;
    const Arr Q = arr(p, count, k);
    p += (size_t)L * count;
    const Arr S = arr(p, count, k);
    const Arr Nn = arr(N, count, k), NPn = arr(NP, count, k), R2n = arr(R2, count, k), Bn = arr(base, count, k);
    const Arr On = arr(out, count, k);
    const Stage sg = stage<C>();

    const int nwin = (bits + w - 1) / w;
    const int per_win = w + 2;
    const int n_ops = nent + 1 + (nwin - 1) * per_win + 1;
#pragma unroll 1
    for (int op = 0; op < n_ops; op++) {
        int mode = MODE_MUL;
        bool select = false;
        int win = 0;
        Arr X = Y, B = Y, O = Y;
        if (op == 0) {
            mode = MODE_REDC; X = R2n; O = G;
        } else if (op < nent) {
            X = op == 1 ? Bn : G.at((op - 1) * Q4);
            B = op == 1 ? R2n : G.at(Q4);
            O = G.at(op * Q4);
        } else if (op == nent) {
            select = true; win = nwin - 1; O = Y;
        } else if (op == n_ops - 1) {
            mode = MODE_REDC; X = Y; O = On;
        } else {
            const int r = (op - nent - 1) % per_win;
            win = nwin - 2 - (op - nent - 1) / per_win;
            if (r < w) {
                mode = MODE_SQR;
            } else if (r == w) {
                select = true; O = S;
            } else {
                B = S;
            }
        }
        if (select) {
            // w bits of the exponent at public position win*w (may straddle two words)
            const int pos = win * w, wi = pos >> 5, off = pos & 31;
            uint32_t v = word_at(exp, count, k, wi) >> off;
            if (off + w > 32 && wi + 1 < L) v |= word_at(exp, count, k, wi + 1) << (32 - off);
            ct_select<L, select_unroll<C>()>(G, nent, v & ((1u << w) - 1u), O);
            continue;
        }
        if (mode == MODE_REDC) {  // T = X zero-extended to 2L limbs
#pragma unroll 1
            for (int q = 0; q < Q4; q++) {
                T.st(q, X.ld(q));
                T.st(Q4 + q, make_uint4(0, 0, 0, 0));
            }
        }
        mont_op<C, NB, TRUNC>(mode, X, B, Nn, NPn, T, Q, O, sg);
    }
}

inline unsigned grid_for(size_t n) { return (unsigned)((n + kThreads - 1) / kThreads); }

template <int C, int NB>
void Launch<C, NB>::mp_mul(const uint32_t* a, const uint32_t* b, uint32_t* c, size_t count, bool sqr, cudaStream_t s) {
    if (sqr) k_mp_mul<C, NB, true><<<grid_for(count), kThreads, stage_bytes<C>(), s>>>(a, a, c, count);
    else k_mp_mul<C, NB, false><<<grid_for(count), kThreads, stage_bytes<C>(), s>>>(a, b, c, count);
}
template <int C, int NB>
void Launch<C, NB>::mont_mul(const uint32_t* a, const uint32_t* b, const uint32_t* N, const uint32_t* NP, uint32_t* c,
                             size_t count, bool trunc, bool sqr, uint32_t* ws, cudaStream_t s) {
    const unsigned g = grid_for(count);
    if (trunc) {
        if (sqr) k_mont_mul<C, NB, true, true><<<g, kThreads, stage_bytes<C>(), s>>>(a, a, N, NP, c, count, ws);
        else k_mont_mul<C, NB, true, false><<<g, kThreads, stage_bytes<C>(), s>>>(a, b, N, NP, c, count, ws);
    } else {
        if (sqr) k_mont_mul<C, NB, false, true><<<g, kThreads, stage_bytes<C>(), s>>>(a, a, N, NP, c, count, ws);
        else k_mont_mul<C, NB, false, false><<<g, kThreads, stage_bytes<C>(), s>>>(a, b, N, NP, c, count, ws);
    }
}
template <int C, int NB>
void Launch<C, NB>::mont_redc(const uint32_t* T, const uint32_t* N, const uint32_t* NP, uint32_t* c, size_t count,
                              bool trunc, uint32_t* ws, cudaStream_t s) {
    if (trunc) k_mont_redc<C, NB, true><<<grid_for(count), kThreads, stage_bytes<C>(), s>>>(T, N, NP, c, count, ws);
    else k_mont_redc<C, NB, false><<<grid_for(count), kThreads, stage_bytes<C>(), s>>>(T, N, NP, c, count, ws);
}
template <int C, int NB>
void Launch<C, NB>::modexp(const uint32_t* N, const uint32_t* NP, const uint32_t* R2, const uint32_t* base,
                           const uint32_t* exp, uint32_t* out, size_t count, int bits, int window, bool trunc,
                           uint32_t* ws, cudaStream_t s) {
    if (trunc) k_modexp<C, NB, true><<<grid_for(count), kThreads, stage_bytes<C>(), s>>>(N, NP, R2, base, exp, out, count, bits, window, ws);
    else k_modexp<C, NB, false><<<grid_for(count), kThreads, stage_bytes<C>(), s>>>(N, NP, R2, base, exp, out, count, bits, window, ws);
}

}  // namespace mpb
