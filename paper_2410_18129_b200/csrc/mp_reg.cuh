// mp_reg.cuh -- register-resident CIOS Montgomery multiplication for L <= 32 limbs (1024 bits).
//
// alg:8BlockMontRed (the CIOS-style interleaved Montgomery multiplication) word by word,
// exactly as the paper writes it -- digit 2^32, m_i = (Y mod 2^32) n0' mod 2^32 with n0' = N'[0]
// (reading A10) -- but with the whole accumulator, the multiplicand and the modulus in REGISTERS:
// rows fully unrolled, no scratch traffic.  Every word product is one fused IMAD.WIDE.U32.X
// (mp_block.cuh), which needs its two destination words to be an even-aligned register pair, so
// the accumulator is split by the parity of the product's position p (lo at p, hi at p+1):
//     Y = U + V * 2^32,   U[k] = word k   (pairs at even p),   V[k] = word k+1  (pairs at odd p)
// (the row-by-row counterpart of the block engine's E/O arrays, mp_block.cuh).  Row i adds a_i * B
// and then m_i * N, each as two carry chains (one per array) starting at position i; a chain's
// carry propagates to position i+L+1, which bounds every partial value: U, V <= U + V < 2^(32(i+L+1)+2).
// The words below position i are never touched again, so they are dropped instead of shifted
// (full unroll: the compiler renames).  Word i of Y is (U[i] + V[i-1] + cin) with cin the carry
// out of word i-1; m_i makes it 0 mod 2^32 and its carry becomes the next cin.  After L rows
// Y / 2^(32L) < 2N (inputs < N) is merged into L+1 words and one masked subtraction of N gives the
// canonical result (A5 / A14).  Constant time: one straight-line instruction sequence.
#pragma once
#include <cstdint>

#include "mp_block.cuh"

namespace mpb {
namespace reg {

// U/V += x * Y  (row at position base i): the two parity chains, carries propagated to i+L+1.
// U indices are positions; V indices are positions - 1.
template <int L, int I>
MPB_DEVI void row(uint32_t (&U)[2 * L + 2], uint32_t (&V)[2 * L + 2], uint32_t x, const uint32_t (&Y)[L]) {
    // U chain: positions p = I + j even
    {
        constexpr int j0 = I & 1;
        constexpr int jl = ((L - 1 - j0) & ~1) + j0;  // last j of this parity
#pragma unroll
        for (int j = j0; j < L; j += 2) pr_chain_rt(j == j0, false, U[I + j], U[I + j + 1], x, Y[j]);
        // carry out of the top pair (I+jl, I+jl+1): propagate to position I+L+1
        constexpr int q0 = I + jl + 2;
        if (q0 == I + L + 1) {
            absorb(U[q0]);
        } else {
#pragma unroll
            for (int q = q0; q <= I + L + 1; q++) {
                if (q == I + L + 1) asm volatile("addc.u32 %0, %0, 0;" : "+r"(U[q]));
                else asm volatile("addc.cc.u32 %0, %0, 0;" : "+r"(U[q]));
            }
        }
    }
    // V chain: positions p = I + j odd, stored at V[p - 1]
    {
        constexpr int j0 = (I & 1) ^ 1;
        constexpr int jl = ((L - 1 - j0) & ~1) + j0;
#pragma unroll
        for (int j = j0; j < L; j += 2) pr_chain_rt(j == j0, false, V[I + j - 1], V[I + j], x, Y[j]);
        constexpr int q0 = I + jl + 2;  // next position after the top pair
        if (q0 == I + L + 1) {
            absorb(V[q0 - 1]);
        } else {
#pragma unroll
            for (int q = q0; q <= I + L + 1; q++) {
                if (q == I + L + 1) asm volatile("addc.u32 %0, %0, 0;" : "+r"(V[q - 1]));
                else asm volatile("addc.cc.u32 %0, %0, 0;" : "+r"(V[q - 1]));
            }
        }
    }
}

// OUT = a * b * 2^(-32L) mod N, canonical, for a, b < N.  a_i comes from `aw(i)` (a functor: the
// caller streams it from shared memory); b, N in registers; n0p = -N^-1 mod 2^32.
template <int L, int I, class AW>
MPB_DEVI void rows(uint32_t (&U)[2 * L + 2], uint32_t (&V)[2 * L + 2], uint32_t& cin, const AW& aw,
                   const uint32_t (&b)[L], const uint32_t (&N)[L], uint32_t n0p) {
    if constexpr (I < L) {
        row<L, I>(U, V, aw(I), b);
        // word I of Y: U[I] + V[I-1] + cin (V[I-1] = word I of the odd array)
        uint32_t w = U[I] + cin;
        if constexpr (I >= 1) w += V[I - 1];
        const uint32_t m = w * n0p;
        row<L, I>(U, V, m, N);
        // the carry out of word I (its value is now 0 mod 2^32)
        uint32_t lo = U[I], c = 0;
        asm volatile("add.cc.u32 %0, %0, %2;\n\taddc.u32 %1, 0, 0;" : "+r"(lo), "+r"(c) : "r"(cin));
        if constexpr (I >= 1) {
            asm volatile("add.cc.u32 %0, %0, %2;\n\taddc.u32 %1, %1, 0;" : "+r"(lo), "+r"(c) : "r"(V[I - 1]));
        }
        cin = c;
        rows<L, I + 1>(U, V, cin, aw, b, N, n0p);
    }
}

template <int L, class AW>
MPB_DEVI void montmul(const AW& aw, const uint32_t (&b)[L], const uint32_t (&N)[L], uint32_t n0p, uint32_t (&out)[L]) {
    uint32_t U[2 * L + 2], V[2 * L + 2];
#pragma unroll
    for (int k = 0; k < 2 * L + 2; k++) { U[k] = 0; V[k] = 0; }
    uint32_t cin = 0;
    rows<L, 0>(U, V, cin, aw, b, N, n0p);
    // Y = positions L .. 2L: U[L + k] + V[L + k - 1] + carries, L + 1 words (< 2N)
    uint32_t y[L + 1];
#pragma unroll
    for (int k = 0; k <= L; k++) y[k] = U[L + k];
    add_first(y[0], cin);
#pragma unroll
    for (int k = 1; k <= L; k++) add_next(y[k], 0u);
    add_first(y[0], V[L - 1]);
#pragma unroll
    for (int k = 1; k < L; k++) add_next(y[k], V[L + k - 1]);
    add_end(y[L], V[2 * L - 1]);
    // canonical: y >= N ? y - N : y (mask)
    uint32_t d[L];
#pragma unroll
    for (int k = 0; k < L; k++) d[k] = y[k];
    sub_first(d[0], N[0]);
#pragma unroll
    for (int k = 1; k < L; k++) sub_next(d[k], N[k]);
    uint32_t top = y[L];
    asm volatile("subc.u32 %0, %0, 0;" : "+r"(top));  // y[L] - borrow: 0 (y >= N) or -1 (y < N)
    const uint32_t m = 0u - (top == 0u ? 1u : 0u);      // all ones: take y - N
#pragma unroll
    for (int k = 0; k < L; k++) out[k] = (d[k] & m) | (y[k] & ~m);
}

}  // namespace reg
}  // namespace mpb
