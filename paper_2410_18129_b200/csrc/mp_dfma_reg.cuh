// mp_dfma_reg.cuh -- register-resident radix-2^52 CIOS Montgomery multiplication on the FP64 pipe
// for D = 20 limbs (1024-bit operands, R = 2^1040 >= 4N).
//
// alg:8BlockMontRed word by word in the paper's own radix and form: per row i,
// Y += a_i * B (madd52lo / madd52hi into Y[j], Y[j+1]), m_i = (Y[0] mod 2^52) n0' mod 2^52,
// Y += m_i * N, Y >>= 52 -- with the madd52 halves produced by exact FP64 FMAs (mp_dfma.cuh) and
// summed as raw bit patterns into LAZY 64-bit accumulators: no carry chain anywhere.  The exponent
// biases only touch bits 52..63, so Y[0] mod 2^52 (all m_i needs) is exact as accumulated; the bias
// of the word shifted out is a compile-time constant (the number of halves it received) and is
// removed just before its carry (>> 52) moves up.  Rows fully unrolled: b and N as doubles and the
// accumulator window live in registers; each row has 2D independent products.  Outputs stay in the
// redundant range [0, 2N) (R >= 4N); the exponentiation subtracts N once at the end.
#pragma once
#include <cstdint>

#include "mp_dfma.cuh"

namespace mpb {
namespace d52r {

using d52::dbits;
using d52::kBH;
using d52::kBL;
using d52::kM52;
using d52::to_d;

// halves received by accumulator position p (absolute) from rows 0 .. r-1 of a D-limb CIOS:
// row i adds lo(a_i b_j) + lo(m_i n_j) at i + j and hi(...) at i + j + 1
template <int D>
__host__ __device__ constexpr uint64_t bias_pos(int p, int rows) {
    uint64_t nl = 0, nh = 0;
    for (int i = 0; i < rows; i++) {
        const int j = p - i, jh = p - i - 1;
        if (j >= 0 && j < D) nl += 2;
        if (jh >= 0 && jh < D) nh += 2;
    }
    return nl * kBL + nh * kBH;
}

template <int D, int I, class AW>
MPB_DEVI void rows(uint64_t (&Y)[2 * D + 2], uint64_t& cin, const AW& aw, const double (&b)[D], const double (&n)[D],
                   double n0p) {
    if constexpr (I < D) {
        const double a = aw(I);
        // m_I = (Y[I] + lo(a b_0) + cin) mod 2^52 * n0' mod 2^52  (biases vanish mod 2^52)
        uint64_t lo0, hi0;
        d52::prod(a, b[0], lo0, hi0);
        const uint64_t y0 = (Y[I] + lo0 + cin) & kM52;
        uint64_t ml, mh;
        d52::prod(to_d(y0), n0p, ml, mh);
        const double m = to_d(ml & kM52);
        // each product pair consumed at once (few live patterns; the 2D products are independent)
        {
            uint64_t l2, h2;
            d52::prod(m, n[0], l2, h2);
            Y[I] = Y[I] + lo0 + l2;
            Y[I + 1] = Y[I + 1] + hi0 + h2;
        }
#pragma unroll
        for (int j = 1; j < D; j++) {
            uint64_t l1, h1, l2, h2;
            d52::prod(a, b[j], l1, h1);
            d52::prod(m, n[j], l2, h2);
            Y[I + j] = Y[I + j] + l1 + l2;
            Y[I + j + 1] = Y[I + j + 1] + h1 + h2;
        }
        // word I is now 0 mod 2^52: remove its bias, carry the rest up (with the incoming carry)
        constexpr uint64_t bias = bias_pos<D>(I, I + 1);
        const uint64_t v = Y[I] - bias + cin;  // exact: the true value is < 2^64
        cin = v >> 52;
        rows<D, I + 1>(Y, cin, aw, b, n, n0p);
    }
}

// out = a b 2^(-52D) mod N in [0, 2N) as D normalised 52-bit limbs (doubles), for a, b < 2N.
// aw(i): a_i as a double; b, n in registers; n0p = -N^-1 mod 2^52 (as a double).
template <int D, class AW>
MPB_DEVI void montmul(const AW& aw, const double (&b)[D], const double (&n)[D], double n0p, double (&out)[D]) {
    uint64_t Y[2 * D + 2];
#pragma unroll
    for (int k = 0; k < 2 * D + 2; k++) Y[k] = 0;
    uint64_t cin = 0;
    rows<D, 0>(Y, cin, aw, b, n, n0p);
    // normalise positions D .. 2D (the last row left its top halves at 2D)
#pragma unroll
    for (int k = 0; k < D; k++) {
        const uint64_t v = Y[D + k] - bias_pos<D>(D + k, D) + cin;
        out[k] = to_d(v & kM52);
        cin = v >> 52;
    }
    // (the value is < 2N < 2^(52D): nothing remains above)
}

}  // namespace d52r
}  // namespace mpb
