// mp_mont.cuh -- per-thread blocked schoolbook products, Montgomery reduction
// (full = alg:8MontRed, truncated = alg:trunc_montred) and the constant-time
// fixed-window exponentiation (alg:8FWExp) on sm_100a.
//
// A number of L = NB*C 32-bit limbs is NB blocks of C limbs.  Every product is
// computed block column by block column (product scanning over blocks): for
// block column k the window W[0..2C] (registers) accumulates every C x C block
// product with s + t = k (mp_block.cuh), then its low C words are final and are
// stored, and the window shifts down by C words.  Big numbers live in memory
// behind an accessor (word-sliced: chunk q of this thread's number at base +
// q*stride, 16-byte chunks), so block loops are ordinary rolled loops and the
// register footprint is independent of L.
//
// Paper mapping:
//   ph_product        T = X*B or X^2              alg:8SBmul / alg:8SBsqu  (L140-209)
//   ph_q              q = T*N' mod R              alg:montred line 1       (L402, L425)
//   ph_hi_trunc       C = floor(T/R) + qnhat + c_add
//                     qnhat from the partial products of weight >= L-1  alg:trunc_montred,
//                     Theorems 1-2 (L418-542), read as SURVEY 8(c) A6/A7
//   ph_hi_full        C = (T + q*N)/R             alg:8MontRed lines 2-3   (L352-354)
//   final select      C -= N if C >= N (mask)     canonical output
//   modexp            table G, CT masked scan, w squarings + 1 multiply per window
//                                                  alg:8FWExp (L742-778), A11 reading
// No branch, address or trip count depends on secret data (operands, exponent):
// loops depend on (L, w, bits) only, selections use masks.
#pragma once
#include <cstdint>

#include "mp_block.cuh"

namespace mpb {

// ----------------------------------------------------------------- accessors
// Global memory, word-sliced: chunk q of operand k at base[q*stride + k] (uint4 units).
struct GArr {
    uint4* p;
    size_t stride;
    MPB_DEVI uint4 ld(int q) const { return p[(size_t)q * stride]; }
    MPB_DEVI void st(int q, uint4 v) const { p[(size_t)q * stride] = v; }
};
// Read-only global input (non-coherent path).
struct GIn {
    const uint4* p;
    size_t stride;
    MPB_DEVI uint4 ld(int q) const { return __ldg(p + (size_t)q * stride); }
};

template <int C, class A>
MPB_DEVI void ldb(const A& a, int blk, uint32_t (&x)[C]) {
#pragma unroll
    for (int q = 0; q < C / 4; q++) {
        uint4 v = a.ld(blk * (C / 4) + q);
        x[4 * q] = v.x; x[4 * q + 1] = v.y; x[4 * q + 2] = v.z; x[4 * q + 3] = v.w;
    }
}
template <int C, int N, class A>
MPB_DEVI void stb(const A& a, int blk, const uint32_t (&x)[N]) {
    static_assert(N >= C, "");
#pragma unroll
    for (int q = 0; q < C / 4; q++) a.st(blk * (C / 4) + q, make_uint4(x[4 * q], x[4 * q + 1], x[4 * q + 2], x[4 * q + 3]));
}

template <int C>
MPB_DEVI void w_zero(uint32_t (&W)[2 * C + 1]) {
#pragma unroll
    for (int i = 0; i <= 2 * C; i++) W[i] = 0;
}
template <int C>
MPB_DEVI void w_shift(uint32_t (&W)[2 * C + 1]) {  // W >>= 32C
#pragma unroll
    for (int i = 0; i <= C; i++) W[i] = W[i + C];
#pragma unroll
    for (int i = C + 1; i <= 2 * C; i++) W[i] = 0;
}

// --------------------------------------------------------------- phase 1
// T[0..2L) = X*B (SQR: X^2).  alg:8SBmul / alg:8SBsqu, blocked.
template <int C, int NB, bool SQR, class AX, class AB, class AT>
MPB_DEVI void ph_product(const AX& X, const AB& B, const AT& T) {
    uint32_t W[2 * C + 1];
    w_zero<C>(W);
#pragma unroll 1
    for (int k = 0; k < 2 * NB - 1; k++) {
        const int s_lo = k - NB + 1 > 0 ? k - NB + 1 : 0;
        const int s_hi = k < NB - 1 ? k : NB - 1;
        if (SQR) {
#pragma unroll 1
            for (int s = s_lo; 2 * s <= k; s++) {
                const int t = k - s;
                uint32_t x[C];
                ldb<C>(X, s, x);
                if (s < t) {
                    uint32_t y[C];
                    ldb<C>(X, t, y);
                    acc_mul2<C>(W, x, y);
                } else {
                    acc_sqr<C>(W, x);
                }
            }
        } else {
#pragma unroll 1
            for (int s = s_lo; s <= s_hi; s++) {
                uint32_t x[C], y[C];
                ldb<C>(X, s, x);
                ldb<C>(B, k - s, y);
                acc_mul<C>(W, x, y);
            }
        }
        stb<C>(T, k, W);
        w_shift<C>(W);
    }
    stb<C>(T, 2 * NB - 1, W);
}

// --------------------------------------------------------------- phase 2
// Q = (T mod R) * N' mod R; also returns orlo = OR of T[0..L-2] and tl1 = T[L-1]
// (for c_add, eq:c_add P:L459-461, and b, K of the A6/A7 reading).
template <int C, int NB, class AT, class ANP, class AQ>
MPB_DEVI void ph_q(const AT& T, const ANP& NP, const AQ& Q, uint32_t& orlo, uint32_t& tl1) {
    uint32_t W[2 * C + 1];
    w_zero<C>(W);
    orlo = 0;
    tl1 = 0;
#pragma unroll 1
    for (int k = 0; k < NB; k++) {
#pragma unroll 1
        for (int s = 0; s <= k; s++) {
            uint32_t x[C], y[C];
            ldb<C>(T, s, x);
            ldb<C>(NP, k - s, y);
            if (s == k) {  // first (and only) time block T_k is loaded with t == 0
#pragma unroll
                for (int i = 0; i < C - 1; i++) orlo |= x[i];
                if (k == NB - 1) tl1 = x[C - 1];
                else orlo |= x[C - 1];
            }
            if (k < NB - 1) acc_mul<C>(W, x, y);
            else acc_lo<C>(W, x, y);
        }
        stb<C>(Q, k, W);
        w_shift<C>(W);
    }
}

// ------------------------------------------------ shared tail: C, D = C - N
// Block j of H (window words 0..C-1) becomes block j of C = T_hi + H + carry (truncated) or
// of C itself (full); C is parked in T block NB+j and D = C - N - borrow goes to OUT block j.
template <int C, int NB, bool ADD_THI, class AT, class AN, class AOUT>
MPB_DEVI void emit_block(const uint32_t (&W)[2 * C + 1], int j, const AT& T, const AN& N, const AOUT& OUT,
                         uint32_t& carry, uint32_t& borrow) {
    uint32_t c[C];
#pragma unroll
    for (int i = 0; i < C; i++) c[i] = W[i];
    if (ADD_THI) {
        uint32_t t[C];
        ldb<C>(T, NB + j, t);
        cc_restore(carry);
#pragma unroll
        for (int i = 0; i < C; i++) add_next(c[i], t[i]);
        carry = cc_save();
    }
    stb<C>(T, NB + j, c);
    uint32_t n[C];
    ldb<C>(N, j, n);
    bc_restore(borrow);
#pragma unroll
    for (int i = 0; i < C; i++) sub_next(c[i], n[i]);
    borrow = bc_save();
    stb<C>(OUT, j, c);
}

// OUT = (ctop || !borrow) ? D : C, with D in OUT and C in T[NB..2NB) -- a mask, no branch.
template <int C, int NB, class AT, class AOUT>
MPB_DEVI void final_select(const AT& T, const AOUT& OUT, uint32_t ctop, uint32_t borrow) {
    const uint32_t m = 0u - ((ctop | (borrow ^ 1u)) & 1u);  // all ones: take D = C - N
#pragma unroll 1
    for (int j = 0; j < NB; j++) {
#pragma unroll
        for (int q = 0; q < C / 4; q++) {
            uint4 d = OUT.ld(j * (C / 4) + q);
            uint4 c = T.ld((NB + j) * (C / 4) + q);
            d.x = (d.x & m) | (c.x & ~m);
            d.y = (d.y & m) | (c.y & ~m);
            d.z = (d.z & m) | (c.z & ~m);
            d.w = (d.w & m) | (c.w & ~m);
            OUT.st(j * (C / 4) + q, d);
        }
    }
}

// ------------------------------------------------------ phase 3, truncated
// alg:trunc_montred lines 2-4: C = floor(T/R) + qnhat + c_add with
//   qnhat = floor(S'/2^32) + [S mod 2^32 > K],  S' = sum of partial products of weight >= L-1
//   (lo of i+j = L-1 and up, hi of i+j = L-2 and up), K = (-T[L-1] - b) mod 2^32,
//   b = [T mod 2^{32(L-1)} != 0], c_add = [T mod R != 0].
template <int C, int NB, class AQ, class AN, class AT, class AOUT>
MPB_DEVI void ph_hi_trunc(const AQ& Q, const AN& N, const AT& T, const AOUT& OUT, uint32_t orlo, uint32_t tl1) {
    const uint32_t b = orlo != 0u ? 1u : 0u;
    const uint32_t c_add = (orlo | tl1) != 0u ? 1u : 0u;
    const uint32_t K = 0u - tl1 - b;
    uint32_t W[2 * C + 1];
    w_zero<C>(W);
    // corners: block column NB-2 contributes hi(q_s[C-1] * N_t[C-1]) at global position L-1
#pragma unroll 1
    for (int s = 0; s + 2 <= NB; s++) {
        const uint4 qv = Q.ld(s * (C / 4) + C / 4 - 1);
        const uint4 nv = N.ld((NB - 2 - s) * (C / 4) + C / 4 - 1);
        asm volatile("mad.hi.cc.u32 %0, %2, %3, %0;\n\taddc.u32 %1, %1, 0;" : "+r"(W[0]), "+r"(W[1]) : "r"(qv.w), "r"(nv.w));
    }
    // block column NB-1: truncated high parts, relative to global position L-1
#pragma unroll 1
    for (int s = 0; s < NB; s++) {
        uint32_t x[C], y[C];
        ldb<C>(Q, s, x);
        ldb<C>(N, NB - 1 - s, y);
        acc_hi<C>(W, x, y);
    }
    // exact carry out of column L-1 (eq:TqN / eq:qnhat under the A6/A7 reading)
    const uint32_t corr = W[0] > K ? 1u : 0u;
#pragma unroll
    for (int i = 0; i < 2 * C; i++) W[i] = W[i + 1];
    W[2 * C] = 0;
    add_first(W[0], corr);
#pragma unroll
    for (int i = 1; i <= C; i++) add_next(W[i], 0u);
    absorb(W[C + 1]);
    // block columns NB .. 2NB-2 (global offset k*C), full block products
    uint32_t carry = c_add, borrow = 0;
#pragma unroll 1
    for (int k = NB; k < 2 * NB - 1; k++) {
#pragma unroll 1
        for (int s = k - NB + 1; s < NB; s++) {
            uint32_t x[C], y[C];
            ldb<C>(Q, s, x);
            ldb<C>(N, k - s, y);
            acc_mul<C>(W, x, y);
        }
        emit_block<C, NB, true>(W, k - NB, T, N, OUT, carry, borrow);
        w_shift<C>(W);
    }
    emit_block<C, NB, true>(W, NB - 1, T, N, OUT, carry, borrow);
    final_select<C, NB>(T, OUT, carry, borrow);
}

// ----------------------------------------------------------- phase 3, full
// alg:8MontRed lines 2-3: C = (T + q*N) / R with the whole q*N product.
template <int C, int NB, class AQ, class AN, class AT, class AOUT>
MPB_DEVI void ph_hi_full(const AQ& Q, const AN& N, const AT& T, const AOUT& OUT) {
    uint32_t W[2 * C + 1];
    w_zero<C>(W);
    uint32_t carry = 0, borrow = 0;
#pragma unroll 1
    for (int k = 0; k < 2 * NB; k++) {
        if (k < 2 * NB - 1) {
            const int s_lo = k - NB + 1 > 0 ? k - NB + 1 : 0;
            const int s_hi = k < NB - 1 ? k : NB - 1;
#pragma unroll 1
            for (int s = s_lo; s <= s_hi; s++) {
                uint32_t x[C], y[C];
                ldb<C>(Q, s, x);
                ldb<C>(N, k - s, y);
                acc_mul<C>(W, x, y);
            }
        }
        {  // + T block k, carry through the whole window
            uint32_t t[C];
            ldb<C>(T, k, t);
            add_first(W[0], t[0]);
#pragma unroll
            for (int i = 1; i < C; i++) add_next(W[i], t[i]);
#pragma unroll
            for (int i = C; i < 2 * C; i++) add_next(W[i], 0u);
            absorb(W[2 * C]);
        }
        if (k >= NB) emit_block<C, NB, false>(W, k - NB, T, N, OUT, carry, borrow);
        w_shift<C>(W);
    }
    final_select<C, NB>(T, OUT, W[0], borrow);
}

// ------------------------------------------------------------ compositions
// OUT = X*B*R^-1 mod N (SQR: X^2*R^-1 mod N), canonical.  T: 2L-word scratch, Q: L-word scratch.
template <int C, int NB, bool TRUNC, bool SQR, class AX, class AB, class AN, class ANP, class AT, class AQ, class AOUT>
MPB_DEVI void mont_mul(const AX& X, const AB& B, const AN& N, const ANP& NP, const AT& T, const AQ& Q, const AOUT& OUT) {
    ph_product<C, NB, SQR>(X, B, T);
    uint32_t orlo, tl1;
    ph_q<C, NB>(T, NP, Q, orlo, tl1);
    if (TRUNC) ph_hi_trunc<C, NB>(Q, N, T, OUT, orlo, tl1);
    else ph_hi_full<C, NB>(Q, N, T, OUT);
}

// OUT = T*R^-1 mod N for the 2L-word T held in scratch T (T is consumed).
template <int C, int NB, bool TRUNC, class AN, class ANP, class AT, class AQ, class AOUT>
MPB_DEVI void mont_redc(const AN& N, const ANP& NP, const AT& T, const AQ& Q, const AOUT& OUT) {
    uint32_t orlo, tl1;
    ph_q<C, NB>(T, NP, Q, orlo, tl1);
    if (TRUNC) ph_hi_trunc<C, NB>(Q, N, T, OUT, orlo, tl1);
    else ph_hi_full<C, NB>(Q, N, T, OUT);
}

// ---------------------------------------------------------- CT table select
// OUT = G[idx] by a masked scan of every entry ("constant-time batch selection").
// Entry e, chunk q lives at chunk index e*(L/4) + q of accessor G.
template <int L, class AG, class AOUT>
MPB_DEVI void ct_select(const AG& G, int nent, uint32_t idx, const AOUT& OUT) {
    uint4 acc[L / 4];
#pragma unroll
    for (int q = 0; q < L / 4; q++) acc[q] = make_uint4(0, 0, 0, 0);
#pragma unroll 1
    for (int e = 0; e < nent; e++) {
        const uint32_t x = (uint32_t)e ^ idx;
        const uint32_t m = 0u - ((x - 1u) >> 31);  // all ones iff e == idx (x < 2^31)
#pragma unroll
        for (int q = 0; q < L / 4; q++) {
            const uint4 v = G.ld(e * (L / 4) + q);
            acc[q].x |= v.x & m;
            acc[q].y |= v.y & m;
            acc[q].z |= v.z & m;
            acc[q].w |= v.w & m;
        }
    }
#pragma unroll
    for (int q = 0; q < L / 4; q++) OUT.st(q, acc[q]);
}

}  // namespace mpb
