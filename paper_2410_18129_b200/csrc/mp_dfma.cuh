// mp_dfma.cuh -- radix-2^52 Montgomery arithmetic on the FP64 pipe.
//
// The paper's own radix (section 2): numbers are D limbs of 52 bits and every
// 52 x 52-bit word product is split into a low and a high 52-bit half that are added, WITHOUT carry
// propagation, into 64-bit column accumulators -- the paper's VPMADD52LUQ / VPMADD52HUQ
// (madd52lo / madd52hi) with its deferred normalisation (the "mask52" pass).  On the
// B200 the split is two exact FP64 fused multiply-adds on limbs held as doubles:
//   hi = fma_rz(a, b, 2^104)                 bits(hi) = (1127 << 52) | floor(ab / 2^52)
//   lo = fma_rn(a, b, (2^104 + 2^52) - hi)    bits(lo) = (1075 << 52) | (ab mod 2^52)
// (ab < 2^104 keeps 2^104 + ab in one binade, ulp 2^52, so the RZ sum is exact up to the floor; the
// subtraction is exact by Sterbenz; lo lies in [2^52, 2^53), ulp 1).  The raw bit patterns are summed
// as 64-bit integers with three-input adds (IADD3 + IADD3.X: two patterns per two ALU instructions),
// the exponent biases -- a compile-time constant per column position -- folded into the same adds.
// Per product: 3 FP64 + 2 ALU instructions and no carry chain (the IMAD path's bound is its serial
// carry chains).  A column holds at most ~4D patterns < 2^52 each, so a 64-bit
// accumulator never overflows; it is normalised (carry-propagated into 52-bit limbs) once, when its
// block column is final.
//
// The Montgomery machinery mirrors the 32-bit engine (mp_mont.cuh): product scanning over C x C
// blocks with a register window, the three phases T = X*B (or X^2), q = T*N' mod R, and
// (T + q*N)/R -- full (alg:8MontRed) or truncated (alg:trunc_montred, with
// Theorem 2's exact correction in radix 2^52: products of weight >= D-1, the high
// halves of weight D-2, carry = floor(S / 2^52) + [S mod 2^52 > K], K = (-T[D-1] - b) mod 2^52).
// R = 2^(52D) >= 4N, so operands stay in the redundant range [0, 2N) and no operation needs the
// conditional subtraction (allowed when the radix exceeds bits + 2); the
// exponentiation subtracts once at the end.  Limbs are doubles in the warp-tiled workspace (two
// per 16-byte chunk, kernels.cuh ArrT), staged per block product by cp.async.
//
// Constant time: every loop bound and address depends on (D, w, bits) only; FP64 latency does not
// depend on the values (all values are integers of at most 105 bits: no subnormals).
#pragma once
#include <cstdint>

#include "mp_mont.cuh"

namespace mpb {
namespace d52 {

constexpr uint64_t kM52 = (1ull << 52) - 1;
constexpr uint64_t kBL = 1075ull << 52;  // pattern bias of a lo half, and of an exact limb v as 2^52 + v
constexpr uint64_t kBH = 1127ull << 52;  // pattern bias of a hi half

MPB_DEVI uint64_t dbits(double d) { return (uint64_t)__double_as_longlong(d); }
// an exact 52-bit integer as a double: (2^52 + v) - 2^52
MPB_DEVI double to_d(uint64_t v) { return __dsub_rn(__longlong_as_double((long long)(v | kBL)), 0x1p52); }
// a limb held as a double, as its pattern (2^52 + v): bias kBL, value v
MPB_DEVI uint64_t limb_pat(double d) { return dbits(__dadd_rn(d, 0x1p52)); }

MPB_DEVI void prod(double a, double b, uint64_t& lo, uint64_t& hi) {
    const double h = __fma_rz(a, b, 0x1p104);
    const double l = __fma_rn(a, b, __dsub_rn(0x1.0000000000001p104, h));
    lo = dbits(l);
    hi = dbits(h);
}
MPB_DEVI uint64_t prod_hi(double a, double b) { return dbits(__fma_rz(a, b, 0x1p104)); }

// ------------------------------------------------------------ block kinds
// Which halves of product (i, j) of a C x C block a kind keeps:
//   FULL   all products                                         (x*y)
//   LOW    i+j <= C-1, the lo half only at i+j = C-1             (x*y mod 2^(52C))
//   HIGH   i+j >= C-1, plus the hi half of i+j = C-2             (truncated high part, Theorem 2)
//   UPPER  i < j (x == y)                                        (off-diagonal half of a square)
//   SQUARE i == j                                                (the diagonal squares)
enum { K_FULL = 0, K_LOW = 1, K_HIGH = 2, K_UPPER = 3, K_SQUARE = 4 };
template <int C, int KIND>
__host__ __device__ constexpr bool keep_lo(int i, int j) {
    return KIND == K_FULL ? true
         : KIND == K_LOW  ? i + j <= C - 1
         : KIND == K_HIGH ? i + j >= C - 1
         : KIND == K_UPPER ? i < j
                           : i == j;
}
template <int C, int KIND>
__host__ __device__ constexpr bool keep_hi(int i, int j) {
    return KIND == K_FULL ? true
         : KIND == K_LOW  ? i + j <= C - 2
         : KIND == K_HIGH ? i + j >= C - 2
         : KIND == K_UPPER ? i < j
                           : i == j;
}
// number of lo / hi halves a kind puts at absolute position p (lo of i+j = p, hi of i+j = p-1)
template <int C, int KIND>
__host__ __device__ constexpr uint64_t bias_at(int p) {
    uint64_t nl = 0, nh = 0;
    for (int i = 0; i < C; i++) {
        const int j = p - i, jh = p - 1 - i;
        if (j >= 0 && j < C && keep_lo<C, KIND>(i, j)) nl++;
        if (jh >= 0 && jh < C && keep_hi<C, KIND>(i, jh)) nh++;
    }
    return nl * kBL + nh * kBH;
}

// W[OFF + p - SH] += the kept halves of x*y at absolute position p (minus their exponent biases),
// for every p with a kept half.  Product (i, j) is computed at column p = i + j; its hi half is held
// for column p + 1, so at most C hi patterns are live.  Sums use three-input adds.
template <int C, int KIND, int OFF, int SH, int WN>
MPB_DEVI void blk(uint64_t (&W)[WN], const double (&x)[C], const double (&y)[C]) {
    uint64_t ph[C];
    int nph = 0;
#pragma unroll
    for (int p = 0; p < 2 * C; p++) {
        uint64_t t[2 * C + 1];
        int n = 0;
        uint64_t nh[C];
        int nn = 0;
#pragma unroll
        for (int i = 0; i < C; i++) {
            const int j = p - i;
            if (j >= 0 && j < C) {
                const bool kl = keep_lo<C, KIND>(i, j), kh = keep_hi<C, KIND>(i, j);
                if (kl) {
                    uint64_t lo, hi;
                    prod(x[i], y[j], lo, hi);
                    t[n++] = lo;
                    if (kh) nh[nn++] = hi;
                } else if (kh) {
                    nh[nn++] = prod_hi(x[i], y[j]);
                }
            }
        }
#pragma unroll
        for (int i = 0; i < nph; i++) t[n++] = ph[i];
        if (n > 0) {
            const int w = OFF + p - SH;
            if (w >= 0 && w < WN) {
                t[n++] = 0ull - bias_at<C, KIND>(p);
                uint64_t s = W[w];
#pragma unroll
                for (int i = 0; i + 1 < n; i += 2) s = s + t[i] + t[i + 1];
                if (n & 1) s += t[n - 1];
                W[w] = s;
            }
        }
#pragma unroll
        for (int i = 0; i < nn; i++) ph[i] = nh[i];
        nph = nn;
    }
}

// W[0..2C) += 2*F for a fresh 2C-position block sum F (squaring: off-diagonal products count twice)
template <int C, int WN>
MPB_DEVI void add_twice(uint64_t (&W)[WN], const uint64_t (&F)[2 * C]) {
#pragma unroll
    for (int p = 0; p < 2 * C; p++) W[p] = W[p] + F[p] + F[p];
}

// ----------------------------------------------------------------- accessors
// Tiled arrays of doubles: chunk q (16 bytes = limbs 2q, 2q+1) of this thread at A.addr(q).
MPB_DEVI void unpack2(const uint4 v, double& a, double& b) {
    a = __hiloint2double((int)v.y, (int)v.x);
    b = __hiloint2double((int)v.w, (int)v.z);
}
MPB_DEVI uint4 pack2(double a, double b) {
    return make_uint4((uint32_t)__double2loint(a), (uint32_t)__double2hiint(a), (uint32_t)__double2loint(b),
                      (uint32_t)__double2hiint(b));
}
template <int C>
MPB_DEVI void ldd(const ArrT& A, int blk_i, double (&x)[C]) {
#pragma unroll
    for (int q = 0; q < C / 2; q++) unpack2(A.ld(blk_i * (C / 2) + q), x[2 * q], x[2 * q + 1]);
}
template <int C>
MPB_DEVI void std_(const ArrT& A, int blk_i, const double (&x)[C]) {
#pragma unroll
    for (int q = 0; q < C / 2; q++) A.st(blk_i * (C / 2) + q, pack2(x[2 * q], x[2 * q + 1]));
}

// Normalise window positions 0..C-1 (lazy, bias-free) into 52-bit limbs with carry propagation;
// the carry out is added to W[C].  Returns the limbs as doubles in d.
template <int C, int WN>
MPB_DEVI void normalize(uint64_t (&W)[WN], double (&d)[C], uint64_t cin = 0) {
    uint64_t c = cin;
#pragma unroll
    for (int i = 0; i < C; i++) {
        const uint64_t v = W[i] + c;
        d[i] = to_d(v & kM52);
        c = v >> 52;
    }
    W[C] += c;
}
template <int C, int WN>
MPB_DEVI void shift(uint64_t (&W)[WN]) {
#pragma unroll
    for (int i = 0; i < WN; i++) W[i] = i + C < WN ? W[i + C] : 0ull;
}

// -------------------------------------------------------------- the engine
// Phases as mp_mont.cuh: PH_MUL / PH_SQR  DST = AX*AY (AX^2), 2D limbs, normalised
//                        PH_Q             DST = (AX mod R)*AY mod R (AX = T, AY = N'), also
//                                         orlo = [T mod 2^(52(D-1)) != 0], tl1 = T[D-1]
//                        PH_HI            OUT = (T + AX*AY)/R, AX = q, AY = N (TRUNC: Theorem 2)
template <int C, int NB, bool TRUNC>
MPB_DEVI void engine(int ph, const ArrT& AX, const ArrT& AY, const ArrT& DST, const ArrT& T, const ArrT& OUT,
                     uint32_t& orlo, uint64_t& tl1, const Stage& sg) {
    constexpr int WN = 2 * C + 1;
    constexpr int QB = C / 2;  // chunks per block
    uint64_t W[WN];
#pragma unroll
    for (int i = 0; i < WN; i++) W[i] = 0;
    const bool sqr = ph == PH_SQR;
    const bool hi_trunc = TRUNC && ph == PH_HI;
    int k0 = 0, k1 = 2 * NB - 1;
    if (ph == PH_Q) k1 = NB;
    uint64_t carry = 0;  // PH_HI: carry into the next emitted block
    uint64_t K = 0;
    if (hi_trunc) {
        k0 = NB - 1;
        // corners: block column NB-2 contributes hi(q_s[C-1] * N_t[C-1]) at position D-1 (window 0)
#pragma unroll 1
        for (int s = 0; s + 2 <= NB; s++) {
            const uint4 qa = AX.ld(s * QB + QB - 1), na = AY.ld((NB - 2 - s) * QB + QB - 1);
            double q0, q1, n0, n1;
            unpack2(qa, q0, q1);
            unpack2(na, n0, n1);
            W[0] = W[0] + prod_hi(q1, n1) - kBH;
        }
        const uint64_t b = orlo != 0u ? 1ull : 0ull;
        carry = (orlo != 0u || tl1 != 0ull) ? 1ull : 0ull;  // c_add = [T mod R != 0]
        K = (0ull - tl1 - b) & kM52;                          // K = (-T[D-1] - b) mod 2^52
    }
    auto issue = [&](int kk, int ss, int buf) {
        const uint32_t base = sg.base + (uint32_t)(buf * 2 * QB) * kStageCS;
        const char* bx = reinterpret_cast<const char*>(AX.addr(ss * QB));
#pragma unroll
        for (int q = 0; q < QB; q++) cp_async16(base + q * kStageCS, bx + q * 512);
        if (!(sqr && 2 * ss == kk)) {
            const char* by = reinterpret_cast<const char*>(AY.addr((kk - ss) * QB));
#pragma unroll
            for (int q = 0; q < QB; q++) cp_async16(base + (QB + q) * kStageCS, by + q * 512);
        }
        cp_commit();
    };
    int k = k0, s = k0 - NB + 1 > 0 ? k0 - NB + 1 : 0;
    int s_hi = sqr ? (k >> 1) : (k < NB - 1 ? k : NB - 1);
    issue(k, s, 0);
    int buf = 0;
#pragma unroll 1
    while (k < k1) {
        int nk = k, ns = s + 1, ns_hi = s_hi;
        if (ns > s_hi) {
            nk = k + 1;
            ns = nk - NB + 1 > 0 ? nk - NB + 1 : 0;
            ns_hi = sqr ? (nk >> 1) : (nk < NB - 1 ? nk : NB - 1);
        }
        const bool more = nk < k1;
        if (more) {
            issue(nk, ns, buf ^ 1);
            cp_wait<1>();
        } else {
            cp_wait<0>();
        }
        const int t = k - s;
        const bool diag = sqr && s == t;
        double x[C], y[C];
        {
            const uint32_t base = sg.base + (uint32_t)(buf * 2 * QB) * kStageCS;
#pragma unroll
            for (int q = 0; q < QB; q++) unpack2(lds128(base + q * kStageCS), x[2 * q], x[2 * q + 1]);
            if (!diag) {
#pragma unroll
                for (int q = 0; q < QB; q++) unpack2(lds128(base + (QB + q) * kStageCS), y[2 * q], y[2 * q + 1]);
            }
        }
        buf ^= 1;
        if (ph == PH_Q && t == 0) {  // block T_k is seen with t == 0 exactly once
            uint32_t o = 0;
#pragma unroll
            for (int i = 0; i < C - 1; i++) o |= (uint32_t)__double2hiint(x[i]) | (uint32_t)__double2loint(x[i]);
            if (k == NB - 1) {
                tl1 = limb_pat(x[C - 1]) & kM52;
            } else {
                o |= (uint32_t)__double2hiint(x[C - 1]) | (uint32_t)__double2loint(x[C - 1]);
            }
            orlo |= o;
        }
        const bool lo_col = ph == PH_Q && k == NB - 1;
        const bool hi_col = hi_trunc && k == NB - 1;
        if (diag) {
            uint64_t F[2 * C];
#pragma unroll
            for (int i = 0; i < 2 * C; i++) F[i] = 0;
            blk<C, K_UPPER, 0, 0>(F, x, x);
            add_twice<C>(W, F);
            blk<C, K_SQUARE, 0, 0>(W, x, x);
        } else if (lo_col) {
            blk<C, K_LOW, 0, 0>(W, x, y);
        } else if (hi_col) {
            blk<C, K_HIGH, 0, C - 1>(W, x, y);
        } else if (sqr) {  // s < t: the product counts twice
            uint64_t F[2 * C];
#pragma unroll
            for (int i = 0; i < 2 * C; i++) F[i] = 0;
            blk<C, K_FULL, 0, 0>(F, x, y);
            add_twice<C>(W, F);
        } else {
            blk<C, K_FULL, 0, 0>(W, x, y);
        }
        if (nk != k) {  // ---- end of block column k
            if (ph != PH_HI) {
                double d[C];
                normalize<C>(W, d);
                std_<C>(DST, k, d);
                shift<C>(W);
            } else if (TRUNC && k == NB - 1) {
                // window 0 = position D-1: exact carry out of it (Theorem 2 in radix 2^52)
                const uint64_t S = W[0];
                const uint64_t corr = (S & kM52) > K ? 1ull : 0ull;
#pragma unroll
                for (int i = 0; i + 1 < WN; i++) W[i] = W[i + 1];
                W[WN - 1] = 0;
                W[0] += (S >> 52) + corr + carry;  // + c_add
                carry = 0;
            } else {
                // + T block k (as integers), normalise; k >= NB: block k-NB of the result
                double tb[C];
                ldd<C>(T, k, tb);
#pragma unroll
                for (int i = 0; i < C; i++) W[i] = W[i] + limb_pat(tb[i]) - kBL;
                double d[C];
                normalize<C>(W, d, carry);
                carry = 0;
                if (k >= NB) std_<C>(OUT, k - NB, d);
                shift<C>(W);
            }
        }
        k = nk;
        s = ns;
        s_hi = ns_hi;
    }
    if (ph == PH_MUL || ph == PH_SQR) {
        double d[C];
        normalize<C>(W, d);
        std_<C>(DST, 2 * NB - 1, d);
    }
    if (ph == PH_HI) {  // the top block: + T block 2NB-1 (+ the truncated path's pending carry)
        double tb[C];
        ldd<C>(T, 2 * NB - 1, tb);
#pragma unroll
        for (int i = 0; i < C; i++) W[i] = W[i] + limb_pat(tb[i]) - kBL;
        double d[C];
        normalize<C>(W, d, carry);
        std_<C>(OUT, NB - 1, d);
    }
}

enum { MODE_MUL = 0, MODE_SQR = 1, MODE_REDC = 2, MODE_LO = 3 };
// OUT = X*B*R^-1 mod N (MUL), X^2*R^-1 (SQR), T*R^-1 for T already in scratch (REDC), in [0, 2N)
// for inputs in [0, 2N).  MODE_LO: OUT = X*B mod R (one low-half product; setup only).  One
// engine call site for every phase (the kernel's instruction footprint stays small).
template <int C, int NB, bool TRUNC>
MPB_DEVI void mont_op(int mode, const ArrT& X, const ArrT& B, const ArrT& N, const ArrT& NP, const ArrT& T,
                      const ArrT& Q, const ArrT& OUT, const Stage& sg) {
    uint32_t orlo = 0;
    uint64_t tl1 = 0;
    const int s0 = mode == MODE_REDC || mode == MODE_LO ? 1 : 0, s1 = mode == MODE_LO ? 2 : 3;
#pragma unroll 1
    for (int step = s0; step < s1; step++) {
        const int ph = step == 0 ? (mode == MODE_SQR ? PH_SQR : PH_MUL) : (step == 1 ? PH_Q : PH_HI);
        const bool lo = mode == MODE_LO;
        const ArrT ax = step == 0 || lo ? X : (step == 1 ? T : Q);
        const ArrT ay = step == 0 || lo ? B : (step == 1 ? NP : N);
        const ArrT dst = lo ? OUT : (step == 0 ? T : Q);
        engine<C, NB, TRUNC>(ph, ax, ay, dst, T, OUT, orlo, tl1, sg);
    }
}

// ------------------------------------------------------------ conversions
// 32-bit limbs (word-sliced ABI array, L limbs) -> D limbs of 52 bits (tiled doubles)
template <int D>
MPB_DEVI void from32(const Arr& A, int L, const ArrT& OUT) {
#pragma unroll 1
    for (int j = 0; j < D; j += 2) {
        double v[2];
#pragma unroll
        for (int u = 0; u < 2; u++) {
            const int b = 52 * (j + u), q = b >> 5, r = b & 31;
            uint64_t x = 0;
#pragma unroll
            for (int e = 0; e < 3; e++) {
                const int wi = q + e;
                uint32_t w = 0;
                if (wi < L) {
                    const uint4 c = A.ld(wi >> 2);
                    const int m = wi & 3;
                    w = m == 0 ? c.x : (m == 1 ? c.y : (m == 2 ? c.z : c.w));
                }
                const int sh = 32 * e - r;  // position of word wi relative to bit b
                if (sh >= 0) x |= sh < 64 ? (uint64_t)w << sh : 0ull;
                else x |= (uint64_t)(w >> (-sh));
            }
            v[u] = to_d(x & kM52);
        }
        OUT.st(j / 2, pack2(v[0], v[1]));
    }
}
// D normalised limbs of 52 bits (value < 2^(32L)) -> 32-bit limbs (word-sliced ABI array)
template <int D>
MPB_DEVI void to32(const ArrT& A, int L, const Arr& OUT) {
#pragma unroll 1
    for (int q4 = 0; q4 < L / 4; q4++) {
        uint32_t w[4];
#pragma unroll
        for (int m = 0; m < 4; m++) {
            const int b = 32 * (4 * q4 + m), j = b / 52, r = b - 52 * j;
            uint64_t x = 0;
#pragma unroll
            for (int e = 0; e < 2; e++) {
                const int lj = j + e;
                uint64_t limb = 0;
                if (lj < D) {
                    double a, c;
                    unpack2(A.ld(lj >> 1), a, c);
                    limb = limb_pat((lj & 1) ? c : a) & kM52;
                }
                const int sh = 52 * e - r;
                if (sh >= 0) x |= sh < 64 ? limb << sh : 0ull;
                else x |= limb >> (-sh);
            }
            w[m] = (uint32_t)x;
        }
        OUT.st(q4, make_uint4(w[0], w[1], w[2], w[3]));
    }
}
// OUT = (c0 - A) mod 2^(52D) on normalised limbs (setup: 2 - y, and the negation of N^-1)
template <int D>
MPB_DEVI void sub_from(uint64_t c0, const ArrT& A, const ArrT& OUT) {
    uint64_t borrow = 0;
#pragma unroll 1
    for (int q = 0; q < D / 2; q++) {
        double a[2], r[2];
        unpack2(A.ld(q), a[0], a[1]);
#pragma unroll
        for (int u = 0; u < 2; u++) {
            const uint64_t c = (q == 0 && u == 0) ? c0 : 0ull;
            const uint64_t v = c - (limb_pat(a[u]) & kM52) - borrow;  // in (-2^53, 2^52)
            r[u] = to_d(v & kM52);
            borrow = (v >> 63) & 1ull;
        }
        OUT.st(q, pack2(r[0], r[1]));
    }
}
// a constant: limb bit `bit` set (bit < 52D), all else zero
template <int D>
MPB_DEVI void set_pow2(int bit, const ArrT& OUT) {
#pragma unroll 1
    for (int q = 0; q < D / 2; q++) {
        const int j0 = 2 * q, j1 = 2 * q + 1;
        const double a = j0 == bit / 52 ? to_d(1ull << (bit % 52)) : 0.0;
        const double b = j1 == bit / 52 ? to_d(1ull << (bit % 52)) : 0.0;
        OUT.st(q, pack2(a, b));
    }
}
template <int D>
MPB_DEVI void copy(const ArrT& A, const ArrT& OUT) {
#pragma unroll 1
    for (int q = 0; q < D / 2; q++) OUT.st(q, A.ld(q));
}
// canonical: OUT = A >= N ? A - N : A for A < 2N (normalised limbs), by a mask
template <int D>
MPB_DEVI void final_sub(const ArrT& A, const ArrT& N, const ArrT& TMP, const ArrT& OUT) {
    uint64_t borrow = 0;
#pragma unroll 1
    for (int q = 0; q < D / 2; q++) {
        double a[2], n[2], r[2];
        unpack2(A.ld(q), a[0], a[1]);
        unpack2(N.ld(q), n[0], n[1]);
#pragma unroll
        for (int u = 0; u < 2; u++) {
            const uint64_t v = (limb_pat(a[u]) & kM52) - (limb_pat(n[u]) & kM52) - borrow;
            r[u] = to_d(v & kM52);
            borrow = (v >> 63) & 1ull;
        }
        TMP.st(q, pack2(r[0], r[1]));
    }
    const uint32_t m = 0u - (uint32_t)(borrow ^ 1ull);  // all ones: A >= N, take A - N
#pragma unroll 1
    for (int q = 0; q < D / 2; q++) {
        const uint4 d = TMP.ld(q), a = A.ld(q);
        OUT.st(q, make_uint4((d.x & m) | (a.x & ~m), (d.y & m) | (a.y & ~m), (d.z & m) | (a.z & ~m),
                             (d.w & m) | (a.w & ~m)));
    }
}

}  // namespace d52
}  // namespace mpb
