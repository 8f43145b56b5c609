// mp_setup.cuh -- Montgomery constants on the device through the block engine
// (the paper's "precomputed values" N' = (-N)^-1 mod R and R^2 mod N).
//
//   N^-1 mod R   Newton / Hensel lifting x <- x * (2 - N*x) mod R from x = N^-1 mod 2^32; each step
//                doubles the number of correct low bits, so ceil(log2 L) steps reach 32L bits.  Both
//                products are low-half block products (engine PH_Q).  N' = -x mod R.
//   R^2 mod N    y = 2^(nbits-1) < N, doubled (32L - nbits + 1) + c times = 2^c * R mod N (Montgomery
//                form of 2^c), then squared s times with Montgomery squarings (each squaring maps
//                2^a * R to 2^(2a) * R), where 32L = c * 2^s with c odd: 2^(c * 2^s) * R = R^2 mod N.
// Modular doublings are constant time (shift, subtract, mask select).  Untimed support path.
#pragma once
#include "mp_kara.cuh"

namespace mpb {

// X <- 2X mod N (X < N), nb blocks; D: nb-block scratch.  Branch-free.
template <int C>
MPB_DEVI void mod_double(const Arr& X, const Arr& N, const Arr& D, int nb) {
    uint32_t sh = 0, borrow = 0;
#pragma unroll 1
    for (int j = 0; j < nb; j++) {
        uint32_t x[C], n[C], d[C];
        ldb<C>(X, j, x);
        ldb<C>(N, j, n);
#pragma unroll
        for (int i = 0; i < C; i++) {
            const uint32_t v = x[i];
            x[i] = (v << 1) | sh;
            sh = v >> 31;
            d[i] = x[i];
        }
        bc_restore(borrow);
#pragma unroll
        for (int i = 0; i < C; i++) sub_next(d[i], n[i]);
        borrow = bc_save();
        stb<C>(X, j, x);  // 2X mod 2^(32L)
        stb<C>(D, j, d);  // 2X - N
    }
    const uint32_t m = 0u - ((sh | (borrow ^ 1u)) & 1u);  // take 2X - N iff 2X >= N
#pragma unroll 1
    for (int j = 0; j < nb; j++) {
        uint32_t x[C], d[C];
        ldb<C>(X, j, x);
        ldb<C>(D, j, d);
#pragma unroll
        for (int i = 0; i < C; i++) x[i] = (d[i] & m) | (x[i] & ~m);
        stb<C>(X, j, x);
    }
}

// scratch per operand (blocks): X (nb), Y (nb), T (2nb), Q (nb), D (nb)  = 6 nb blocks
template <int C>
MPB_DEVI void setup_one(int nb, const Arr& N, const Arr& NP, const Arr& R2, const Arr& W, const Stage& sg,
                        uint32_t n0, int nbits) {
    constexpr int Q4 = C / 4;
    const int L = C * nb;
    const Arr X = W, Y = W.at(nb * Q4), T = W.at(2 * nb * Q4), Q = W.at(4 * nb * Q4), D = W.at(5 * nb * Q4);
    uint32_t ol[2] = {0, 0};
    // ---- N^-1 mod R
    uint32_t inv = n0;  // correct to 3 bits for odd n0; 5 Newton steps reach 32 bits
#pragma unroll
    for (int it = 0; it < 5; it++) inv *= 2u - n0 * inv;
#pragma unroll 1
    for (int q = 0; q < nb * Q4; q++) X.st(q, make_uint4(q == 0 ? inv : 0u, 0, 0, 0));
    int steps = 0;
    while ((32 << steps) < 32 * L) steps++;
#pragma unroll 1
    for (int it = 0; it < steps; it++) {
        engine_call<C, true>(PH_Q, nb, N, X, Y, Y, Y, Y, ol, sg);  // Y = N*X mod R
        // Y = 2 - Y mod R = ~Y + 3
        uint32_t c = 0;
#pragma unroll 1
        for (int j = 0; j < nb; j++) {
            uint32_t y[C];
            ldb<C>(Y, j, y);
#pragma unroll
            for (int i = 0; i < C; i++) y[i] = ~y[i];
            if (j == 0) {
                add_first(y[0], 3u);
            } else {
                cc_restore(c);
                add_next(y[0], 0u);
            }
#pragma unroll
            for (int i = 1; i < C; i++) add_next(y[i], 0u);
            c = cc_save();
            stb<C>(Y, j, y);
        }
        engine_call<C, true>(PH_Q, nb, X, Y, T, T, T, T, ol, sg);  // T = X*Y mod R
#pragma unroll 1
        for (int q = 0; q < nb * Q4; q++) X.st(q, T.ld(q));
    }
    // N' = -X mod R = ~X + 1
    {
        uint32_t c = 0;
#pragma unroll 1
        for (int j = 0; j < nb; j++) {
            uint32_t x[C];
            ldb<C>(X, j, x);
#pragma unroll
            for (int i = 0; i < C; i++) x[i] = ~x[i];
            if (j == 0) {
                add_first(x[0], 1u);
            } else {
                cc_restore(c);
                add_next(x[0], 0u);
            }
#pragma unroll
            for (int i = 1; i < C; i++) add_next(x[i], 0u);
            c = cc_save();
            stb<C>(NP, j, x);
        }
    }
    // ---- R^2 mod N
    int c_odd = 32 * L, s = 0;
    while ((c_odd & 1) == 0) {
        c_odd >>= 1;
        s++;
    }
#pragma unroll 1
    for (int q = 0; q < nb * Q4; q++) {
        const int w0 = 4 * q, bit = nbits - 1;
        const int wi = bit >> 5;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (wi == w0) v.x = 1u << (bit & 31);
        if (wi == w0 + 1) v.y = 1u << (bit & 31);
        if (wi == w0 + 2) v.z = 1u << (bit & 31);
        if (wi == w0 + 3) v.w = 1u << (bit & 31);
        Y.st(q, v);
    }
    const int doublings = 32 * L - nbits + 1 + c_odd;
#pragma unroll 1
    for (int d = 0; d < doublings; d++) mod_double<C>(Y, N, D, nb);  // Y = 2^c_odd * R mod N
#pragma unroll 1
    for (int it = 0; it < s; it++) {  // Montgomery squarings: Y = MontSqr(Y)
        ol[0] = ol[1] = 0;
        engine_call<C, true>(PH_SQR, nb, Y, Y, T, T, T, T, ol, sg);
        engine_call<C, true>(PH_Q, nb, T, NP, Q, T, N, Y, ol, sg);
        engine_call<C, true>(PH_HI, nb, Q, N, Q, T, N, Y, ol, sg);
    }
#pragma unroll 1
    for (int q = 0; q < nb * Q4; q++) R2.st(q, Y.ld(q));
}

}  // namespace mpb
