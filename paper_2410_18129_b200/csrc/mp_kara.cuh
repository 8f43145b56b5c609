// mp_kara.cuh -- block-level subtractive Karatsuba (1 and 2 levels) on the block engine.
//
// PAPER.md L239-258 (section 3): A*B = D0 + X(D0 + D2 - D1') + X^2 D2 with the middle term from
// one half-size product.  The paper's additive form (a_l + a_h)(b_l + b_h) needs a carry bit
// per half; on 32-bit limbs the subtractive form keeps every half-size operand exactly h blocks:
//     Dm = |a0 - a1| * |b0 - b1|,  mid = D0 + D2 - s*Dm,  s = sign(a0 - a1) * sign(b0 - b1)
// (mid = a0*b1 + a1*b0 >= 0 always; SURVEY 8(c) A4 reading).  Splits are block-aligned
// (A19): a0 has h0 = ceil(nb/2) blocks, a1 the remaining h1 <= h0 (so an odd block count,
// e.g. 11 blocks at 4154 bits, splits 6 + 5).  Two levels apply the split again to each of
// the three half-size products (the paper's "double Karatsuba": 9 elementary
// products).  Squaring uses Dm = (a0 - a1)^2 and always subtracts.
//
// Everything is branch-free on data: the sign only builds masks; all loops run on public
// block counts.  Half-size products go through one non-inlined engine call so the block
// primitives exist once in the code.
#pragma once
#include "mp_mont.cuh"

namespace mpb {

// DST[0..2nb) = X*Y (or X^2) through the engine -- one shared, non-inlined instance.
template <int C>
__device__ __noinline__ void engine_product(bool sqr, int nb, Arr X, Arr Y, Arr DST, Stage sg) {
    uint32_t orlo = 0, tl1 = 0;
    engine<C, true>(sqr ? PH_SQR : PH_MUL, nb, X, Y, DST, DST, DST, DST, orlo, tl1, sg);
}

// D[0..h0) = |A[0..h0) - A[h0..h0+h1)| (the high part zero-extended); returns 1 if low < high.
template <int C>
MPB_DEVI uint32_t kara_absdiff(const Arr& A, int h0, int h1, const Arr& D) {
    uint32_t borrow = 0;
#pragma unroll 1
    for (int j = 0; j < h0; j++) {
        uint32_t x[C], y[C];
        ldb<C>(A, j, x);
        if (j < h1) {
            ldb<C>(A, h0 + j, y);
        } else {
#pragma unroll
            for (int i = 0; i < C; i++) y[i] = 0;
        }
        bc_restore(borrow);
#pragma unroll
        for (int i = 0; i < C; i++) sub_next(x[i], y[i]);
        borrow = bc_save();
        stb<C>(D, j, x);
    }
    // conditional two's-complement negation (x ^ m) + (m & 1), m = -borrow: a mask, no branch
    const uint32_t m = 0u - borrow;
    uint32_t carry = m & 1u;
#pragma unroll 1
    for (int j = 0; j < h0; j++) {
        uint32_t x[C];
        ldb<C>(D, j, x);
#pragma unroll
        for (int i = 0; i < C; i++) x[i] ^= m;
        cc_restore(carry);
#pragma unroll
        for (int i = 0; i < C; i++) add_next(x[i], 0u);
        carry = cc_save();
        stb<C>(D, j, x);
    }
    return borrow;
}

// OUT holds D0 (blocks 0..2h0) and D2 (blocks 2h0..2h0+2h1); M holds Dm (2h0 blocks).
// mid = D0 + D2 -/+ Dm is formed in M, then OUT += mid * X (X = 2^(32*C*h0)).
// m: all ones to subtract Dm, zero to add it (built from the signs as a mask, never a branch).
template <int C>
MPB_DEVI void kara_combine(const Arr& OUT, const Arr& M, int nb, int h0, int h1, uint32_t m) {
    uint32_t c1 = 0, c2 = m & 1u;
#pragma unroll 1
    for (int j = 0; j < 2 * h0; j++) {
        uint32_t t[C], d2[C], dm[C];
        ldb<C>(OUT, j, t);
        if (j < 2 * h1) {
            ldb<C>(OUT, 2 * h0 + j, d2);
        } else {
#pragma unroll
            for (int i = 0; i < C; i++) d2[i] = 0;
        }
        ldb<C>(M, j, dm);
        cc_restore(c1);
#pragma unroll
        for (int i = 0; i < C; i++) add_next(t[i], d2[i]);
        c1 = cc_save();
        cc_restore(c2);
#pragma unroll
        for (int i = 0; i < C; i++) add_next(t[i], dm[i] ^ m);
        c2 = cc_save();
        stb<C>(M, j, t);
    }
    const uint32_t top = c1 + c2 + m;  // the extra word of mid: 0 or 1 (mid < 2 X^2)
    uint32_t c = 0;
#pragma unroll 1
    for (int j = h0; j < 2 * nb; j++) {
        const int jj = j - h0;
        uint32_t x[C], y[C];
        ldb<C>(OUT, j, x);
        if (jj < 2 * h0) {
            ldb<C>(M, jj, y);
        } else {
#pragma unroll
            for (int i = 0; i < C; i++) y[i] = 0;
            if (jj == 2 * h0) y[0] = top;
        }
        cc_restore(c);
#pragma unroll
        for (int i = 0; i < C; i++) add_next(x[i], y[i]);
        c = cc_save();
        stb<C>(OUT, j, x);
    }
}

// Scratch blocks kmul<C, LEVEL> needs for nb blocks.
__host__ __device__ constexpr int kara_scratch_blocks(int nb, int level) {
    return level <= 0 || nb < 2 ? 0 : 4 * ((nb + 1) / 2) + kara_scratch_blocks((nb + 1) / 2, level - 1);
}

// OUT[0..2nb) = A*B (SQR: A^2) with LEVEL levels of Karatsuba; S: kara_scratch_blocks(nb, LEVEL) blocks.
template <int C, int LEVEL>
MPB_DEVI void kmul(bool sqr, int nb, const Arr& A, const Arr& B, const Arr& OUT, const Arr& S, const Stage& sg) {
    if constexpr (LEVEL <= 0) {
        engine_product<C>(sqr, nb, A, B, OUT, sg);
    } else {
    if (nb < 2) {
        engine_product<C>(sqr, nb, A, B, OUT, sg);
        return;
    }
    constexpr int Q = C / 4;  // chunks per block
    const int h0 = (nb + 1) / 2, h1 = nb - h0;
    const Arr da = S, db = S.at(h0 * Q), M = S.at(2 * h0 * Q), sub = S.at(4 * h0 * Q);
    const uint32_t sa = kara_absdiff<C>(A, h0, h1, da);
    const uint32_t sb = sqr ? sa : kara_absdiff<C>(B, h0, h1, db);
    kmul<C, LEVEL - 1>(sqr, h0, A, B, OUT, sub, sg);                                        // D0 = a0*b0
    kmul<C, LEVEL - 1>(sqr, h1, A.at(h0 * Q), B.at(h0 * Q), OUT.at(2 * h0 * Q), sub, sg);    // D2 = a1*b1
    kmul<C, LEVEL - 1>(sqr, h0, da, sqr ? da : db, M, sub, sg);                              // Dm
    const uint32_t m = sqr ? 0xFFFFFFFFu : 0u - ((sa ^ sb ^ 1u) & 1u);  // subtract iff signs agree
    kara_combine<C>(OUT, M, nb, h0, h1, m);
    }
}

}  // namespace mpb

namespace mpb {

// One shared, non-inlined engine entry (setup and other support kernels).
template <int C, bool TRUNC>
__device__ __noinline__ void engine_call(int ph, int nb, Arr AX, Arr AY, Arr DST, Arr T, Arr N, Arr OUT, uint32_t* ol,
                                         Stage sg) {
    uint32_t orlo = ol[0], tl1 = ol[1];
    engine<C, TRUNC>(ph, nb, AX, AY, DST, T, N, OUT, orlo, tl1, sg);
    ol[0] = orlo;
    ol[1] = tl1;
}

}  // namespace mpb

namespace mpb {

// Montgomery operation whose product phase (T = X*B or X^2) uses KLEV levels of block Karatsuba
// (Karatsuba inside MontMul/MontSqr); the reduction phases stay on the engine.
// KS: kara_scratch_blocks(NB, KLEV) blocks of scratch.  KLEV = 0 is mont_op.
template <int C, bool TRUNC, int KLEV, class AR = Arr>
MPB_DEVI void mont_op_k(int mode, int NB, const AR& X, const AR& B, const AR& N, const AR& NP, const AR& T,
                        const AR& Q, const AR& OUT, const AR& KS, const Stage& sg) {
    if constexpr (KLEV == 0) {
        mont_op<C, TRUNC>(mode, NB, X, B, N, NP, T, Q, OUT, sg);
    } else {
        if (mode != MODE_REDC) kmul<C, KLEV>(mode == MODE_SQR, NB, X, B, T, KS, sg);
        mont_op<C, TRUNC>(MODE_REDC, NB, X, B, N, NP, T, Q, OUT, sg);
    }
}

// Any REDC mode: RM = 0 full (alg:8MontRed), 1 truncated (alg:trunc_montred), 2 CIOS
// (alg:8BlockMontRed, schoolbook only: the reduction is interleaved with the product rows).
// CIOS uses T as its Y scratch and Q as its m scratch; REDC(X) is MontMul(X, 1).
template <int C, int RM, int KLEV, class AR = Arr>
MPB_DEVI void mont_op_rm(int mode, int NB, const AR& X, const AR& B, const AR& N, const AR& NP, const AR& T,
                         const AR& Q, const AR& OUT, const AR& KS, const Stage& sg) {
    if constexpr (RM == 2) {
        static_assert(KLEV == 0, "CIOS interleaves reduction and product rows: schoolbook only");
        cios_op<C>(NB, X, B, mode == MODE_REDC, N, NP, T, Q, OUT);
    } else {
        mont_op_k<C, RM == 1, KLEV>(mode, NB, X, B, N, NP, T, Q, OUT, KS, sg);
    }
}

}  // namespace mpb
