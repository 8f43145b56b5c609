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
// ------------------------------------------------ truncated-Karatsuba REDC (f1)
// floor(x*y / 2^(32 C nb)) for nb-block x, y, given K = word C*nb-1 of (x*y mod 2^(32 C nb)):
// Theorem 2's truncated high part (corners of block column nb-2, truncated high blocks of column
// nb-1, the exact carry [S mod 2^32 > K], full blocks above) -- PH_HI's walk without T, emit, select.
template <int C>
__device__ __noinline__ void trunc_high_product(int nb, Arr X, Arr Y, uint32_t K, Arr DST) {
    uint32_t W[2 * C + 1];
    w_zero<C>(W);
#pragma unroll 1
    for (int s = 0; s + 2 <= nb; s++) {
        const uint32_t xw = X.ld(s * (C / 4) + C / 4 - 1).w, yw = Y.ld((nb - 2 - s) * (C / 4) + C / 4 - 1).w;
        asm volatile("mad.hi.cc.u32 %0, %2, %3, %0;\n\taddc.u32 %1, %1, 0;" : "+r"(W[0]), "+r"(W[1]) : "r"(xw), "r"(yw));
    }
#pragma unroll 1
    for (int s = 0; s < nb; s++) {
        uint32_t x[C], y[C];
        ldb<C>(X, s, x);
        ldb<C>(Y, nb - 1 - s, y);
        acc_hi<C>(W, x, y);
    }
    {
        const uint32_t corr = W[0] > K ? 1u : 0u;
#pragma unroll
        for (int i = 0; i < 2 * C; i++) W[i] = W[i + 1];
        W[2 * C] = 0;
        add_first(W[0], corr);
#pragma unroll
        for (int i = 1; i <= C; i++) add_next(W[i], 0u);
        absorb(W[C + 1]);
    }
#pragma unroll 1
    for (int k = nb; k <= 2 * nb - 2; k++) {
#pragma unroll 1
        for (int s = k - nb + 1; s < nb; s++) {
            uint32_t x[C], y[C];
            ldb<C>(X, s, x);
            ldb<C>(Y, k - s, y);
            acc_mul<C>(W, x, y);
        }
        stb<C>(DST, k - nb, W);
        w_shift<C>(W);
    }
    stb<C>(DST, nb - 1, W);
}

// The high part of the Montgomery reduction, floor(q N / R), by the paper's truncated Karatsuba
// (trunc(A B) = 2^t (D2l + D1h - D0h - D2h) + 2^(3t/2) D2h, computed "with the same kind
// of carry evaluation" as the truncated schoolbook), in the subtractive form (reading A4) with the
// exact carries derived from the known low half Lam = q N mod R = (-T) mod R:
//   halves of h = NB/2 blocks, X = 2^(32 C h):  D2 = q1 N1 (full), D0h = floor(q0 N0 / X) (Theorem 2,
//   K0 = word of Lam_l), Dm = |q0 - q1| |N0 - N1|, sigma = +1 iff the two differences have the same
//   sign (mid = D0 + D2 - sigma Dm), V = D0h + Lam_l + D2l - Lam_h, Dml = sigma V mod X,
//   Dmh = floor(Dm / X) (Theorem 2, K = top word of Dml), c = floor(V / X) + [sigma = -1, V mod X != 0],
//   floor(q N / R) = D2 + D0h + D2h - sigma Dmh + c.
// Then C = floor(T/R) + that + c_add, D = C - N, canonical by a mask (as PH_HI).  Block products:
// h^2 + 2 (h^2/2 + h) -- the truncated schoolbook high part's (2h)^2/2 + 2h; the linear passes are the
// extra cost.  NB even.  S: 6 NB blocks of scratch (word-sliced, like T).
template <int C>
__device__ __noinline__ void kara_trunc_high(int NB, Arr T, Arr Q, Arr N, Arr OUT, Arr S, Stage sg) {
    constexpr int Q4 = C / 4;
    const int h = NB / 2;
    const Arr LAM = S, D2 = S.at(NB * Q4), D0H = S.at(2 * NB * Q4), DML = S.at((2 * NB + h) * Q4),
              DQ = S.at((2 * NB + 2 * h) * Q4), DN = S.at((2 * NB + 3 * h) * Q4), DMH = S.at((2 * NB + 4 * h) * Q4);
    // Lam = (0 - T_low) mod R; c_add = [T mod R != 0] = the final borrow
    uint32_t bw = 0;
#pragma unroll 1
    for (int j = 0; j < NB; j++) {
        uint32_t t[C], z[C];
        ldb<C>(T, j, t);
#pragma unroll
        for (int i = 0; i < C; i++) z[i] = 0;
        bc_restore(bw);
#pragma unroll
        for (int i = 0; i < C; i++) sub_next(z[i], t[i]);
        bw = bc_save();
        stb<C>(LAM, j, z);
    }
    const uint32_t cadd = bw;
    engine_product<C>(false, h, Q.at(h * Q4), N.at(h * Q4), D2, sg);                 // D2 = q1 N1
    trunc_high_product<C>(h, Q, N, LAM.ld((h * C - 1) / 4).w, D0H);                   // D0h
    const uint32_t sq = kara_absdiff<C>(Q, h, h, DQ), sn = kara_absdiff<C>(N, h, h, DN);
    const int64_t sigma = sq == sn ? 1 : -1;  // (a mask-like value: no branch depends on it)
    // V = D0h + Lam_l + D2_l - Lam_h (signed carry), Dml = sigma V mod X
    int64_t cv = 0;
    uint32_t vnz = 0;
#pragma unroll 1
    for (int j = 0; j < h; j++) {
        uint32_t a[C], b[C], d[C], e[C], v[C];
        ldb<C>(D0H, j, a);
        ldb<C>(LAM, j, b);
        ldb<C>(D2, j, d);
        ldb<C>(LAM, h + j, e);
#pragma unroll
        for (int i = 0; i < C; i++) {
            const int64_t sm = (int64_t)a[i] + (int64_t)b[i] + (int64_t)d[i] - (int64_t)e[i] + cv;
            v[i] = (uint32_t)sm;
            cv = sm >> 32;  // arithmetic: floor
            vnz |= v[i];
        }
        stb<C>(DML, j, v);
    }
    {  // Dml = sigma == -1 ? (-V mod X) : V  (two's complement under a mask)
        const uint32_t m = sigma < 0 ? 0xFFFFFFFFu : 0u;
        uint32_t cy = m & 1u;
#pragma unroll 1
        for (int j = 0; j < h; j++) {
            uint32_t v[C];
            ldb<C>(DML, j, v);
#pragma unroll
            for (int i = 0; i < C; i++) v[i] ^= m;
            cc_restore(cy);
#pragma unroll
            for (int i = 0; i < C; i++) add_next(v[i], 0u);
            cy = cc_save();
            stb<C>(DML, j, v);
        }
    }
    const int64_t c = cv + ((sigma < 0 && vnz != 0u) ? 1 : 0);
    trunc_high_product<C>(h, DQ, DN, DML.ld((h * C - 1) / 4).w, DMH);                 // Dmh
    // H = D2 + (D0h + D2h - sigma Dmh + c); C = T_hi + H + c_add into T[NB..2NB), D = C - N into OUT
    int64_t ch = c;
    uint32_t cyc = cadd, borrow = 0;
#pragma unroll 1
    for (int j = 0; j < NB; j++) {
        uint32_t d2[C], th[C], n[C], hv[C];
        ldb<C>(D2, j, d2);
        ldb<C>(T, NB + j, th);
        ldb<C>(N, j, n);
        if (j < h) {
            uint32_t a[C], e[C], f[C];
            ldb<C>(D0H, j, a);
            ldb<C>(D2, h + j, e);
            ldb<C>(DMH, j, f);
#pragma unroll
            for (int i = 0; i < C; i++) {
                const int64_t sm = (int64_t)d2[i] + (int64_t)a[i] + (int64_t)e[i] - sigma * (int64_t)f[i] + ch;
                hv[i] = (uint32_t)sm;
                ch = sm >> 32;
            }
        } else {
#pragma unroll
            for (int i = 0; i < C; i++) {
                const int64_t sm = (int64_t)d2[i] + ch;
                hv[i] = (uint32_t)sm;
                ch = sm >> 32;
            }
        }
        cc_restore(cyc);  // C block = T_hi block + H block + carry
#pragma unroll
        for (int i = 0; i < C; i++) add_next(th[i], hv[i]);
        cyc = cc_save();
        stb<C>(T, NB + j, th);
        bc_restore(borrow);  // D block = C block - N block
#pragma unroll
        for (int i = 0; i < C; i++) sub_next(th[i], n[i]);
        borrow = bc_save();
        stb<C>(OUT, j, th);
    }
    final_select<C>(NB, T, OUT, cyc, borrow);
}

// Scratch blocks of kara_trunc_high for nb blocks (6 nb; mirrored by kara_redc_scratch_blocks_host).
__host__ __device__ constexpr int kara_redc_scratch_blocks(int nb) { return 6 * nb; }

template <int C, bool TRUNC, int KLEV, class AR = Arr>
MPB_DEVI void mont_op_k(int mode, int NB, const AR& X, const AR& B, const AR& N, const AR& NP, const AR& T,
                        const AR& Q, const AR& OUT, const AR& KS, const Stage& sg) {
    if constexpr (KLEV == 0) {
        mont_op<C, TRUNC>(mode, NB, X, B, N, NP, T, Q, OUT, sg);
    } else {
        if (mode != MODE_REDC) kmul<C, KLEV>(mode == MODE_SQR, NB, X, B, T, KS, sg);
        if (TRUNC && (NB & 1) == 0 && NB >= 2) {
            // q = T N' mod R (schoolbook low half, PH_Q), then the truncated-Karatsuba high part
            uint32_t ol[2] = {0u, 0u};
            engine_call<C, true>(PH_Q, NB, T, NP, Q, T, N, OUT, ol, sg);
            kara_trunc_high<C>(NB, T, Q, N, OUT, KS.at(kara_scratch_blocks(NB, KLEV) * (C / 4)), sg);
        } else {
            mont_op<C, TRUNC>(MODE_REDC, NB, X, B, N, NP, T, Q, OUT, sg);
        }
    }
}

#ifndef MPB_CIOS_SQR
#define MPB_CIOS_SQR 1  // 0: CIOS squares through the multiplication rows (A/B builds)
#endif
// Any REDC mode: RM = 0 full (alg:8MontRed), 1 truncated (alg:trunc_montred), 2 CIOS
// (alg:8BlockMontRed, schoolbook only: the reduction is interleaved with the product rows).
// CIOS uses T as its Y scratch and Q as its m scratch; REDC(X) is MontMul(X, 1).
template <int C, int RM, int KLEV, class AR = Arr>
MPB_DEVI void mont_op_rm(int mode, int NB, const AR& X, const AR& B, const AR& N, const AR& NP, const AR& T,
                         const AR& Q, const AR& OUT, const AR& KS, const Stage& sg) {
    if constexpr (RM == 2) {
        static_assert(KLEV == 0, "CIOS interleaves reduction and product rows: schoolbook only");
        cios_op<C>(NB, X, B, mode == MODE_REDC, N, NP, T, Q, OUT, mode == MODE_SQR && MPB_CIOS_SQR);
    } else {
        mont_op_k<C, RM == 1, KLEV>(mode, NB, X, B, N, NP, T, Q, OUT, KS, sg);
    }
}

}  // namespace mpb
