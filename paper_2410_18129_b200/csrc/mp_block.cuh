// mp_block.cuh -- per-thread C x C limb block products on sm_100a.
//
// The paper's batch schoolbook kernels (alg:8SBmul / alg:8SBsqu)
// word-slice 8 operands across the lanes of a zmm register and multiply 52-bit
// words with VPMADD52LO/HI.  The B200 analog used here: one operand per thread
// (the warp is the "batch"), 32-bit limbs, and every 32x32->64 word product is
// ONE fused `IMAD.WIDE.U32.X` (carry in and out through a predicate).  ptxas
// emits that instruction for a PTX pair `mad{c}.lo.cc` / `madc.hi.cc` whose two
// destination words form an even-aligned register pair (measured in
// tools/microbench_int.cu: 31 products/clk/SM = the 2-IMAD-per-product roofline;
// the unfused lo/hi form reaches only 19).  A product at word position p lands on
// words (p, p+1); to keep every pair aligned the accumulator is split into
//   E : pairs starting at even positions   (E[k] = word k)
//   O : pairs starting at odd positions    (O[k] = word k+1)
// and E + O*2^32 is the value (the GPU counterpart of the paper's deferred
// mask52 carry pass).  Inside one row the E chain and the O chain
// each run as one carry chain; the top of each chain either ends on a word that
// is provably fresh, or absorbs its carry into a word that holds at most a carry
// bit (see the bounds in DESIGN.md section 5.2), so no carry is ever dropped.
//
// All loops are over compile-time bounds and are fully unrolled: register
// arrays stay in registers.  Nothing here branches on data.
#pragma once
#include <cstdint>

#define MPB_DEVI __device__ __forceinline__

namespace mpb {

// ------------------------------------------------------------ PTX primitives
// (lo,hi) += a*b, no carry in, carry out to CC
MPB_DEVI void pr_first(uint32_t& lo, uint32_t& hi, uint32_t a, uint32_t b) {
    asm volatile("mad.lo.cc.u32 %0, %2, %3, %0;\n\tmadc.hi.cc.u32 %1, %2, %3, %1;" : "+r"(lo), "+r"(hi) : "r"(a), "r"(b));
}
// (lo,hi) += a*b + CC, carry out to CC
MPB_DEVI void pr_next(uint32_t& lo, uint32_t& hi, uint32_t a, uint32_t b) {
    asm volatile("madc.lo.cc.u32 %0, %2, %3, %0;\n\tmadc.hi.cc.u32 %1, %2, %3, %1;" : "+r"(lo), "+r"(hi) : "r"(a), "r"(b));
}
// (lo,hi) += a*b + CC, no carry out (caller proves the pair cannot overflow)
MPB_DEVI void pr_next_end(uint32_t& lo, uint32_t& hi, uint32_t a, uint32_t b) {
    asm volatile("madc.lo.cc.u32 %0, %2, %3, %0;\n\tmadc.hi.u32 %1, %2, %3, %1;" : "+r"(lo), "+r"(hi) : "r"(a), "r"(b));
}
// (lo,hi) += a*b, no carry in, no carry out
MPB_DEVI void pr_only(uint32_t& lo, uint32_t& hi, uint32_t a, uint32_t b) {
    asm volatile("mad.lo.cc.u32 %0, %2, %3, %0;\n\tmadc.hi.u32 %1, %2, %3, %1;" : "+r"(lo), "+r"(hi) : "r"(a), "r"(b));
}
// (lo,hi) = a*b  (fresh)
MPB_DEVI void pr_set(uint32_t& lo, uint32_t& hi, uint32_t a, uint32_t b) {
    asm("mul.lo.u32 %0, %2, %3;\n\tmul.hi.u32 %1, %2, %3;" : "=r"(lo), "=r"(hi) : "r"(a), "r"(b));
}
// w += CC (no carry out)
MPB_DEVI void absorb(uint32_t& w) { asm volatile("addc.u32 %0, %0, 0;" : "+r"(w)); }
// lo-only products
MPB_DEVI void lo_next_end(uint32_t& d, uint32_t a, uint32_t b) {
    asm volatile("madc.lo.u32 %0, %1, %2, %0;" : "+r"(d) : "r"(a), "r"(b));
}
MPB_DEVI void lo_only(uint32_t& d, uint32_t a, uint32_t b) {
    asm volatile("mad.lo.u32 %0, %1, %2, %0;" : "+r"(d) : "r"(a), "r"(b));
}
MPB_DEVI uint32_t lo_set(uint32_t a, uint32_t b) { return a * b; }
// plain add chains
MPB_DEVI void add_first(uint32_t& d, uint32_t s) { asm volatile("add.cc.u32 %0, %0, %1;" : "+r"(d) : "r"(s)); }
MPB_DEVI void add_next(uint32_t& d, uint32_t s) { asm volatile("addc.cc.u32 %0, %0, %1;" : "+r"(d) : "r"(s)); }
MPB_DEVI void add_end(uint32_t& d, uint32_t s) { asm volatile("addc.u32 %0, %0, %1;" : "+r"(d) : "r"(s)); }
MPB_DEVI void sub_first(uint32_t& d, uint32_t s) { asm volatile("sub.cc.u32 %0, %0, %1;" : "+r"(d) : "r"(s)); }
MPB_DEVI void sub_next(uint32_t& d, uint32_t s) { asm volatile("subc.cc.u32 %0, %0, %1;" : "+r"(d) : "r"(s)); }
// CC <- (c != 0) for a saved carry bit c in {0,1}
MPB_DEVI void cc_restore(uint32_t c) {
    uint32_t t;
    asm volatile("add.cc.u32 %0, %1, 0xFFFFFFFF;" : "=r"(t) : "r"(c));
}
// CC <- borrow flag for a saved borrow bit b in {0,1}  (0 - b sets borrow iff b != 0)
MPB_DEVI void bc_restore(uint32_t b) {
    uint32_t t;
    asm volatile("sub.cc.u32 %0, 0, %1;" : "=r"(t) : "r"(b));
}
MPB_DEVI uint32_t cc_save() {  // returns CC as 0/1, clears nothing it needs
    uint32_t c;
    asm volatile("addc.u32 %0, 0, 0;" : "=r"(c));
    return c;
}
MPB_DEVI uint32_t bc_save() {  // borrow as 0/1
    uint32_t b;
    asm volatile("subc.u32 %0, 0, 0;" : "=r"(b));
    return b & 1u;
}

// emit one pair of a chain with compile-time position in the chain
template <bool FIRST, bool LAST_NOCC>
MPB_DEVI void pr_chain(uint32_t& lo, uint32_t& hi, uint32_t a, uint32_t b) {
    if (FIRST && LAST_NOCC) pr_only(lo, hi, a, b);
    else if (FIRST) pr_first(lo, hi, a, b);
    else if (LAST_NOCC) pr_next_end(lo, hi, a, b);
    else pr_next(lo, hi, a, b);
}
MPB_DEVI void pr_chain_rt(bool first, bool last_nocc, uint32_t& lo, uint32_t& hi, uint32_t a, uint32_t b) {
    // all arguments are compile-time constants after unrolling; the branches fold away
    if (first && last_nocc) pr_only(lo, hi, a, b);
    else if (first) pr_first(lo, hi, a, b);
    else if (last_nocc) pr_next_end(lo, hi, a, b);
    else pr_next(lo, hi, a, b);
}

// ----------------------------------------------------------- block products
// Full product x*y of C-limb blocks: value = E[0..2C) + O[0..2C-1)*2^32.
template <int C>
MPB_DEVI void bp_mul(const uint32_t (&x)[C], const uint32_t (&y)[C], uint32_t (&E)[2 * C], uint32_t (&O)[2 * C]) {
    static_assert(C % 2 == 0, "even block");
#pragma unroll
    for (int j = 0; j < C; j++) {  // row 0 writes fresh pairs, no chains
        if ((j & 1) == 0) pr_set(E[j], E[j + 1], x[j], y[0]);
        else pr_set(O[j - 1], O[j], x[j], y[0]);
    }
#pragma unroll
    for (int k = C; k < 2 * C; k++) { E[k] = 0; O[k] = 0; }
#pragma unroll
    for (int i = 1; i < C; i++) {
        {  // E chain: j == i (mod 2); absorbing iff i even (top pair at i+C-2)
            const int j0 = i & 1;
            const bool absorb_e = (i & 1) == 0;
#pragma unroll
            for (int j = j0; j < C; j += 2)
                pr_chain_rt(j == j0, (j + 2 >= C) && !absorb_e, E[i + j], E[i + j + 1], x[j], y[i]);
            if (absorb_e) absorb(E[i + C]);
        }
        {  // O chain: j == i+1 (mod 2); absorbing iff i odd
            const int j0 = (i & 1) ^ 1;
            const bool absorb_o = (i & 1) == 1;
#pragma unroll
            for (int j = j0; j < C; j += 2)
                pr_chain_rt(j == j0, (j + 2 >= C) && !absorb_o, O[i + j - 1], O[i + j], x[j], y[i]);
            if (absorb_o) absorb(O[i + C - 1]);
        }
    }
}

// Off-diagonal half of x^2: value = E + O*2^32 = sum_{i<j} x_i x_j 2^{32(i+j)}  (2C-1 words)
template <int C>
MPB_DEVI void bp_sqr_offdiag(const uint32_t (&x)[C], uint32_t (&E)[2 * C], uint32_t (&O)[2 * C]) {
    static_assert(C % 2 == 0, "even block");
#pragma unroll
    for (int k = 0; k < 2 * C; k++) { E[k] = 0; O[k] = 0; }
#pragma unroll
    for (int j = 1; j < C; j++) {  // row 0, fresh
        if ((j & 1) == 0) pr_set(E[j], E[j + 1], x[j], x[0]);
        else pr_set(O[j - 1], O[j], x[j], x[0]);
    }
#pragma unroll
    for (int i = 1; i < C - 1; i++) {
        {  // E chain: j == i (mod 2), j >= i+2
            const int j0 = i + 2;
            const bool absorb_e = (i & 1) == 0;
#pragma unroll
            for (int j = j0; j < C; j += 2)
                pr_chain_rt(j == j0, (j + 2 >= C) && !absorb_e, E[i + j], E[i + j + 1], x[j], x[i]);
            if (absorb_e && j0 < C) absorb(E[i + C]);
        }
        {  // O chain: j == i+1 (mod 2), j >= i+1
            const int j0 = i + 1;
            const bool absorb_o = (i & 1) == 1;
#pragma unroll
            for (int j = j0; j < C; j += 2)
                pr_chain_rt(j == j0, (j + 2 >= C) && !absorb_o, O[i + j - 1], O[i + j], x[j], x[i]);
            if (absorb_o && j0 < C) absorb(O[i + C - 1]);
        }
    }
}

// Low half: value = E[0..C) + O[0..C-1)*2^32 == x*y (mod 2^{32C}); the top column is lo-only.
template <int C>
MPB_DEVI void bp_lo(const uint32_t (&x)[C], const uint32_t (&y)[C], uint32_t (&E)[2 * C], uint32_t (&O)[2 * C]) {
    static_assert(C % 2 == 0, "even block");
#pragma unroll
    for (int j = 0; j < C - 1; j++) {  // row 0 fresh (positions j)
        if ((j & 1) == 0) pr_set(E[j], E[j + 1], x[j], y[0]);
        else pr_set(O[j - 1], O[j], x[j], y[0]);
    }
    O[C - 2] = lo_set(x[C - 1], y[0]);  // position C-1, lo only
    O[C - 1] = 0;
#pragma unroll
    for (int i = 1; i < C; i++) {
        {  // E chain: even positions p = i+j <= C-2, last pair ends without carry out
            const int j0 = i & 1;
#pragma unroll
            for (int j = j0; i + j <= C - 2; j += 2)
                pr_chain_rt(j == j0, (i + j + 2 > C - 2), E[i + j], E[i + j + 1], x[j], y[i]);
        }
        {  // O chain: odd positions p <= C-3 as pairs, then the lo-only product at p = C-1
            const int j0 = (i & 1) ^ 1;
            bool first = true;
#pragma unroll
            for (int j = j0; i + j <= C - 3; j += 2) {
                pr_chain_rt(j == j0, false, O[i + j - 1], O[i + j], x[j], y[i]);
                first = false;
            }
            const int jl = C - 1 - i;  // p = C-1
            if (first) lo_only(O[C - 2], x[jl], y[i]);
            else lo_next_end(O[C - 2], x[jl], y[i]);
        }
    }
}

// Truncated high part (Theorem 2, per block), relative to position C-1:
//   R = sum_{i+j>=C-1} x_i y_j 2^{32(i+j-C+1)} + sum_{i+j=C-2} hi(x_i y_j)
// value = E[0..C+1) + O[1..C+2)*2^0  with O[k] at relative position k-1 (O[0] is a dummy lo word).
template <int C>
MPB_DEVI void bp_hi(const uint32_t (&x)[C], const uint32_t (&y)[C], uint32_t (&E)[2 * C], uint32_t (&O)[2 * C]) {
    static_assert(C % 2 == 0 && C >= 4, "even block >= 4");
#pragma unroll
    for (int k = 0; k < C + 2; k++) { E[k] = 0; O[k] = 0; }
    pr_set(O[0], O[1], x[C - 2], y[0]);  // row 0: hi-only product at p' = -1 (lo is the dummy)
    pr_set(E[0], E[1], x[C - 1], y[0]);  // p' = 0
#pragma unroll
    for (int i = 1; i < C; i++) {
        {  // E chain: p' = i+j-C+1 in {0, 2, 4, ...}  (j = C-1-i, C+1-i, ...); absorbing iff i odd
            const bool absorb_e = (i & 1) == 1;
            const int j0 = C - 1 - i;
#pragma unroll
            for (int j = j0; j < C; j += 2) {
                const int p = i + j - C + 1;
                pr_chain_rt(j == j0, (j + 2 >= C) && !absorb_e, E[p], E[p + 1], x[j], y[i]);
            }
            if (absorb_e) absorb(E[i + 1]);
        }
        {  // O chain: p' in {-1, 1, 3, ...}; p' = -1 is the hi-only product; absorbing iff i even
            const bool absorb_o = (i & 1) == 0;
            const int j0 = (C - 2 - i >= 0) ? (C - 2 - i) : (C - i);
            if (C - 2 - i >= 0) O[0] = 0;  // dummy lo of the p' = -1 pair must start at 0
#pragma unroll
            for (int j = j0; j < C; j += 2) {
                const int p = i + j - C + 1;
                pr_chain_rt(j == j0, (j + 2 >= C) && !absorb_o, O[p + 1], O[p + 2], x[j], y[i]);
            }
            if (absorb_o) absorb(O[i + 2]);
        }
    }
}

// ------------------------------------------------------------ window adds
// W[OFF .. OFF+LEN) += S[SOFF .. SOFF+LEN), then propagate the carry into W[OFF+LEN] (if any).
template <int OFF, int LEN, int SOFF, int WN, int SN>
MPB_DEVI void w_add(uint32_t (&W)[WN], const uint32_t (&S)[SN]) {
    static_assert(OFF + LEN <= WN && SOFF + LEN <= SN, "range");
    add_first(W[OFF], S[SOFF]);
#pragma unroll
    for (int k = 1; k < LEN; k++) add_next(W[OFF + k], S[SOFF + k]);
    if (OFF + LEN < WN) absorb(W[OFF + LEN < WN ? OFF + LEN : 0]);
}
// same, but the carry out of the last word is dropped (mod 2^{32(OFF+LEN)})
template <int OFF, int LEN, int SOFF, int WN, int SN>
MPB_DEVI void w_add_trunc(uint32_t (&W)[WN], const uint32_t (&S)[SN]) {
    static_assert(OFF + LEN <= WN && SOFF + LEN <= SN, "range");
    if (LEN == 1) {
        W[OFF] += S[SOFF];
        return;
    }
    add_first(W[OFF], S[SOFF]);
#pragma unroll
    for (int k = 1; k < LEN - 1; k++) add_next(W[OFF + k], S[SOFF + k]);
    add_end(W[OFF + LEN - 1], S[SOFF + LEN - 1]);
}

// W[0..2C] += x*y
template <int C>
MPB_DEVI void acc_mul(uint32_t (&W)[2 * C + 1], const uint32_t (&x)[C], const uint32_t (&y)[C]) {
    uint32_t E[2 * C], O[2 * C];
    bp_mul<C>(x, y, E, O);
    w_add<0, 2 * C, 0>(W, E);
    w_add<1, 2 * C - 1, 0>(W, O);
}
// E[1..2C) += O[0..2C-1)  (fold the odd-aligned array into the even one: one carry chain)
template <int C>
MPB_DEVI void fold_odd(uint32_t (&E)[2 * C], const uint32_t (&O)[2 * C]) {
    add_first(E[1], O[0]);
#pragma unroll
    for (int k = 2; k < 2 * C - 1; k++) add_next(E[k], O[k - 1]);
    add_end(E[2 * C - 1], O[2 * C - 2]);
}
// W[0..2C] += 2*S for a 2C-word S (shift by one bit with funnel shifts: no carry chain)
template <int C>
MPB_DEVI void w_add_double(uint32_t (&W)[2 * C + 1], const uint32_t (&S)[2 * C]) {
    uint32_t D[2 * C];
    D[0] = S[0] << 1;
#pragma unroll
    for (int k = 1; k < 2 * C; k++) D[k] = __funnelshift_l(S[k - 1], S[k], 1);
    const uint32_t top = S[2 * C - 1] >> 31;
    add_first(W[0], D[0]);
#pragma unroll
    for (int k = 1; k < 2 * C; k++) add_next(W[k], D[k]);
    add_end(W[2 * C], top);
}
// W[0..2C] += 2*x*y
template <int C>
MPB_DEVI void acc_mul2(uint32_t (&W)[2 * C + 1], const uint32_t (&x)[C], const uint32_t (&y)[C]) {
    uint32_t E[2 * C], O[2 * C];
    bp_mul<C>(x, y, E, O);
    fold_odd<C>(E, O);  // E = x*y exactly (< 2^{64C})
    w_add_double<C>(W, E);
}
// W[0..2C] += x^2 = D + 2*S with D the diagonal squares (added first: its products and chain do
// not depend on the off-diagonal rows, so ptxas can overlap them) and S the off-diagonal sum.
template <int C>
MPB_DEVI void acc_sqr(uint32_t (&W)[2 * C + 1], const uint32_t (&x)[C]) {
    uint32_t E[2 * C], O[2 * C];
    bp_sqr_offdiag<C>(x, E, O);
    fold_odd<C>(E, O);  // S = sum_{i<j} x_i x_j 2^{32(i+j)} < 2^{64C-1}
    // E = 2S (funnel shifts, top down, in place; 2S < 2^{64C}), then + the diagonal squares x_i^2
    // at the even-aligned pairs (2i, 2i+1) as ONE fused carry chain: 2S + D = x^2 < 2^{64C}, so the
    // chain ends without a carry; one merge into the window
#pragma unroll
    for (int k = 2 * C - 1; k >= 1; k--) E[k] = __funnelshift_l(E[k - 1], E[k], 1);
    E[0] <<= 1;
    pr_first(E[0], E[1], x[0], x[0]);
#pragma unroll
    for (int i = 1; i < C - 1; i++) pr_next(E[2 * i], E[2 * i + 1], x[i], x[i]);
    pr_next_end(E[2 * C - 2], E[2 * C - 1], x[C - 1], x[C - 1]);
    w_add<0, 2 * C, 0>(W, E);
}
// W[0..C) += x*y mod 2^{32C}
template <int C>
MPB_DEVI void acc_lo(uint32_t (&W)[2 * C + 1], const uint32_t (&x)[C], const uint32_t (&y)[C]) {
    uint32_t E[2 * C], O[2 * C];
    bp_lo<C>(x, y, E, O);
    w_add_trunc<0, C, 0>(W, E);
    w_add_trunc<1, C - 1, 0>(W, O);
}
// W[0..C+1] += truncated high part (relative to block position C-1)
template <int C>
MPB_DEVI void acc_hi(uint32_t (&W)[2 * C + 1], const uint32_t (&x)[C], const uint32_t (&y)[C]) {
    uint32_t E[2 * C], O[2 * C];
    bp_hi<C>(x, y, E, O);
    w_add<0, C + 1, 0>(W, E);
    w_add<0, C + 1, 1>(W, O);
}

// ------------------------------------------------ register-level Karatsuba block
// W[0..2C] += TW * x*y (TW = 1 or 2: the squaring's off-diagonal blocks count twice) by ONE level
// of subtractive Karatsuba on the halves (H = C/2 limbs, X = 2^(32H); SURVEY 8(f) f1
// with reading A4):  D0 = x0 y0, D2 = x1 y1, Dm = |x0 - x1| |y0 - y1|, s = sign(x0-x1) sign(y0-y1),
//   x*y = D0 + (D0 + D2 - s Dm) X + D2 X^2
// 3 H x H block products (3C^2/4 fused products instead of C^2) with shorter carry chains; the
// sign only builds masks.  Measured on register operands (tools/microbench_kara16.cu, C = 16):
// 28.8 vs 22.9 schoolbook-equivalent products per clock per SM at 12 warps, bit-identical.
template <int H>
MPB_DEVI void kara_half_product(const uint32_t (&a)[H], const uint32_t (&b)[H], uint32_t (&P)[2 * H]) {
    uint32_t E[2 * H], O[2 * H];
    bp_mul<H>(a, b, E, O);
    fold_odd<H>(E, O);
#pragma unroll
    for (int i = 0; i < 2 * H; i++) P[i] = E[i];
}
template <int H>
MPB_DEVI uint32_t kara_absdiff(const uint32_t* u, const uint32_t* v, uint32_t (&d)[H]) {
#pragma unroll
    for (int i = 0; i < H; i++) d[i] = u[i];
    sub_first(d[0], v[0]);
#pragma unroll
    for (int i = 1; i < H; i++) sub_next(d[i], v[i]);
    const uint32_t b = bc_save();
    const uint32_t m = 0u - b;
#pragma unroll
    for (int i = 0; i < H; i++) d[i] ^= m;
    add_first(d[0], b);
#pragma unroll
    for (int i = 1; i < H; i++) add_next(d[i], 0u);
    return b;
}
template <int C, int TW>
MPB_DEVI void acc_kara(uint32_t (&W)[2 * C + 1], const uint32_t (&x)[C], const uint32_t (&y)[C]) {
    static_assert(C % 4 == 0, "halves must be even blocks");
    constexpr int H = C / 2;
    uint32_t dx[H], dy[H];
    const uint32_t sx = kara_absdiff<H>(x, x + H, dx), sy = kara_absdiff<H>(y, y + H, dy);
    uint32_t D[2 * C];  // D0 | D2 (= D0 + D2 X^2, 2C words)
    {
        uint32_t x0[H], y0[H], x1[H], y1[H], P[2 * H];
#pragma unroll
        for (int i = 0; i < H; i++) { x0[i] = x[i]; y0[i] = y[i]; x1[i] = x[H + i]; y1[i] = y[H + i]; }
        kara_half_product<H>(x0, y0, P);
#pragma unroll
        for (int i = 0; i < 2 * H; i++) D[i] = P[i];
        kara_half_product<H>(x1, y1, P);
#pragma unroll
        for (int i = 0; i < 2 * H; i++) D[2 * H + i] = P[i];
    }
    // mid = D0 + D2 - s Dm  (C + 1 words, >= 0: it is x0 y1 + x1 y0)
    uint32_t mid[C + 1];
#pragma unroll
    for (int i = 0; i < C; i++) mid[i] = D[i];
    mid[C] = 0;
    add_first(mid[0], D[C]);
#pragma unroll
    for (int i = 1; i < C; i++) add_next(mid[i], D[C + i]);
    absorb(mid[C]);
#pragma unroll
    for (int t = 0; t < TW; t++) {  // W += D0 + D2 X^2
        add_first(W[0], D[0]);
#pragma unroll
        for (int i = 1; i < 2 * C; i++) add_next(W[i], D[i]);
        absorb(W[2 * C]);
    }
    {
        uint32_t P[2 * H];
        kara_half_product<H>(dx, dy, P);
        const uint32_t m = 0u - ((sx ^ sy ^ 1u) & 1u);  // all ones: subtract Dm (the signs agree)
        cc_restore(m & 1u);                               // two's complement: + ~Dm + 1
#pragma unroll
        for (int i = 0; i < 2 * H; i++) add_next(mid[i], P[i] ^ m);
        add_end(mid[C], m);
    }
#pragma unroll
    for (int t = 0; t < TW; t++) {  // W += mid X  (words H .. H + C, carry to the top)
        add_first(W[H], mid[0]);
#pragma unroll
        for (int i = 1; i <= C; i++) add_next(W[H + i], mid[i]);
#pragma unroll
        for (int i = H + C + 1; i < 2 * C; i++) add_next(W[i], 0u);
        absorb(W[2 * C]);
    }
}

}  // namespace mpb
