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

// Y = positions L .. 2L of the finished rows (U[L + k] + V[L + k - 1] + cin, L + 1 words, < 2N),
// then one masked subtraction of N: the canonical result.
template <int L>
MPB_DEVI void finish(const uint32_t (&U)[2 * L + 2], const uint32_t (&V)[2 * L + 2], uint32_t cin, const uint32_t (&N)[L],
                     uint32_t (&out)[L]) {
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
    finish<L>(U, V, cin, N, out);
}

// ---------------------------------------------------------------------------------------------------
// MontSqr with SQUARING ROWS in the same CIOS order.  a^2 = sum_i a_i M_i 2^(32i) with
// M_i = a_i + 2 sum_{j>i} a_j 2^(32(j-i)) (the textbook symmetric square: each cross product once,
// doubled), so row i is a_i times the words j = i .. L of
//     M[i] = a_i,  M[i+1] = D[i+1] with bit 0 cleared,  M[j] = D[j] (j > i+1),   D = 2a (L+1 words)
// at positions i + j >= 2i.  Row i never reaches below position 2i >= i, so word i is complete when
// m_i is formed, exactly as in CIOS; the reduction rows are montmul's.  L(L+1)/2 + L a-products
// instead of L^2 (560 + 1024 reduction products instead of 2048 at L = 32).  Bounds: rows r <= i
// sum to < 2a 2^(32(i+1)) <= 2^(32(i+L+1)+1) and the reductions to < N 2^(32i), so no chain carries
// past position i+L+1, the top of the window (as in montmul).
template <int L, int I>
MPB_DEVI void row_sq(uint32_t (&U)[2 * L + 2], uint32_t (&V)[2 * L + 2], uint32_t x, const uint32_t (&D)[L + 1]) {
    {  // U chain: j = I, I+2, .. <= L (positions 2I, 2I+2, ..)
        constexpr int jl = L - ((L - I) & 1);
#pragma unroll
        for (int j = I; j <= L; j += 2)
            pr_chain_rt(j == I, j == jl && jl == L, U[I + j], U[I + j + 1], x, j == I ? x : D[j]);
        if constexpr (jl < L) absorb(U[I + L + 1]);
    }
    {  // V chain: j = I+1, I+3, .. <= L (positions 2I+1, ..; V index = position - 1)
        constexpr int jl = L - ((L - I - 1) & 1);
#pragma unroll
        for (int j = I + 1; j <= L; j += 2)
            pr_chain_rt(j == I + 1, j == jl && jl == L, V[I + j - 1], V[I + j], x, j == I + 1 ? (D[j] & ~1u) : D[j]);
        if constexpr (jl < L) absorb(V[I + L]);
    }
}

template <int L, int I, class AW>
MPB_DEVI void rows_sq(uint32_t (&U)[2 * L + 2], uint32_t (&V)[2 * L + 2], uint32_t& cin, const AW& aw,
                      const uint32_t (&D)[L + 1], const uint32_t (&N)[L], uint32_t n0p) {
    if constexpr (I < L) {
        row_sq<L, I>(U, V, aw(I), D);
        uint32_t w = U[I] + cin;
        if constexpr (I >= 1) w += V[I - 1];
        const uint32_t m = w * n0p;
        row<L, I>(U, V, m, N);
        uint32_t lo = U[I], c = 0;
        asm volatile("add.cc.u32 %0, %0, %2;\n\taddc.u32 %1, 0, 0;" : "+r"(lo), "+r"(c) : "r"(cin));
        if constexpr (I >= 1) {
            asm volatile("add.cc.u32 %0, %0, %2;\n\taddc.u32 %1, %1, 0;" : "+r"(lo), "+r"(c) : "r"(V[I - 1]));
        }
        cin = c;
        rows_sq<L, I + 1>(U, V, cin, aw, D, N, n0p);
    }
}

// out = a^2 * 2^(-32L) mod N canonical, a < N: aw(i) = a_i, D = 2a (double_words)
template <int L, class AW>
MPB_DEVI void montsqr(const AW& aw, const uint32_t (&D)[L + 1], const uint32_t (&N)[L], uint32_t n0p, uint32_t (&out)[L]) {
    uint32_t U[2 * L + 2], V[2 * L + 2];
#pragma unroll
    for (int k = 0; k < 2 * L + 2; k++) { U[k] = 0; V[k] = 0; }
    uint32_t cin = 0;
    rows_sq<L, 0>(U, V, cin, aw, D, N, n0p);
    finish<L>(U, V, cin, N, out);
}

// B = 2a as L+1 words (the squaring rows' multiplicand)
template <int L>
MPB_DEVI void double_words(const uint32_t (&a)[L], uint32_t (&B)[L + 1]) {
    B[0] = a[0] << 1;
#pragma unroll
    for (int q = 1; q < L; q++) B[q] = __funnelshift_l(a[q - 1], a[q], 1);
    B[L] = a[L - 1] >> 31;
}

}  // namespace reg
}  // namespace mpb

namespace mpb {
namespace reg {

// ===================================================================================================
// Register-resident truncated Montgomery multiplication / squaring (alg:trunc_montred, P:L418-431,
// with Theorem 2's exact correction at word granularity, reading A6/A7) for L = 32.
// SOS order as the block engine: T = a*b (or a^2), q = (T mod R) N' mod R, C = floor(T/R) +
// floor(q N / R) + c_add, canonical by one masked subtraction.  Rows fully unrolled; the row
// multiplier comes from registers or a per-thread shared-memory slot, the multiplicand is in
// registers; accumulators split by pair parity (U: pairs at even positions, U index = position;
// V: pairs at odd positions, V index = position - 1) so every fused product writes an even-aligned
// register pair.  N, N' and T's high half live in per-thread shared memory between phases.
// ===================================================================================================

// U/V += x * M[j] for j in [J0, J1), product j at positions P0 + j (lo) / P0 + j + 1 (hi):
//   HIF:  product J0 keeps only its hi half (its lo goes to a dummy word zeroed first)
//   LOL:  product J1-1 keeps only its lo half, and nothing carries out of its position (mod R)
//   TOP:  last position a carry may reach (the final add of every chain ends there without carry)
template <int P0, int J0, int J1, bool HIF, bool LOL, int TOP, int NU, int LM>
MPB_DEVI void grow(uint32_t (&U)[NU], uint32_t (&V)[NU], uint32_t x, const uint32_t (&M)[LM]) {
#pragma unroll
    for (int par = 0; par < 2; par++) {
        // products of this chain: j in [J0, J1) with (P0 + j) % 2 == par
        int first = -1, last = -1;
#pragma unroll
        for (int j = J0; j < J1; j++)
            if (((P0 + j) & 1) == par) {
                if (first < 0) first = j;
                last = j;
            }
        if (first < 0) continue;
#pragma unroll
        for (int j = J0; j < J1; j++) {
            if (((P0 + j) & 1) != par) continue;
            const int p = P0 + j;
            uint32_t& lo = par == 0 ? U[p] : V[p - 1];
            uint32_t& hi = par == 0 ? U[p + 1] : V[p];
            const bool isfirst = j == first, islast = j == last;
            if (HIF && j == J0) lo = 0u;  // dummy lo: the word is never read as a result
            if (LOL && j == J1 - 1) {
                // lo half only, at the top position: madc.lo without carry out
                if (isfirst) lo_only(lo, x, M[j]);
                else lo_next_end(lo, x, M[j]);
            } else {
                // a pair whose hi word is at TOP ends the chain without carry out
                const bool nocc = islast && (p + 1 >= TOP);
                pr_chain_rt(isfirst, nocc, lo, hi, x, M[j]);
                if (islast && p + 1 < TOP) {  // carry out: propagate to TOP
#pragma unroll
                    for (int q = p + 2; q <= TOP; q++) {
                        uint32_t& w = par == 0 ? U[q] : V[q - 1];  // the chain's own array
                        if (q == TOP) asm volatile("addc.u32 %0, %0, 0;" : "+r"(w));
                        else asm volatile("addc.cc.u32 %0, %0, 0;" : "+r"(w));
                    }
                }
            }
        }
    }
}

// T[p] = U[p] + V[p-1] + c (word p of the merged accumulator), c <- its carry (0..2)
// (P is a compile-time constant after unrolling: the arrays stay in registers)
template <int NU>
MPB_DEVI uint32_t merge_word(const uint32_t (&U)[NU], const uint32_t (&V)[NU], int P, uint32_t& c) {
    uint32_t t = U[P], cc = 0;
    asm volatile("add.cc.u32 %0, %0, %2;\n\taddc.u32 %1, 0, 0;" : "+r"(t), "+r"(cc) : "r"(c));
    if (P >= 1) {
        asm volatile("add.cc.u32 %0, %0, %2;\n\taddc.u32 %1, %1, 0;" : "+r"(t), "+r"(cc) : "r"(V[P >= 1 ? P - 1 : 0]));
    }
    c = cc;
    return t;
}

// ---- T = a * b (a_i from aw, b in registers): T[0..32) to t_lo (registers), T[32..64) to th (smem slot)
template <int L, int I, class AW, class TH>
MPB_DEVI void mul_rows(uint32_t (&U)[2 * L + 2], uint32_t (&V)[2 * L + 2], uint32_t& c, const AW& aw,
                       const uint32_t (&b)[L], uint32_t (&tlo)[L], const TH& th) {
    if constexpr (I < L) {
        grow<I, 0, L, false, false, I + L, 2 * L + 2, L>(U, V, aw(I), b);
        tlo[I] = merge_word(U, V, I, c);
        mul_rows<L, I + 1>(U, V, c, aw, b, tlo, th);
    } else {
#pragma unroll
        for (int k = 0; k < L; k++) th(k, merge_word(U, V, L + k, c));
    }
}

// ---- T = x^2: off-diagonal rows (x_i x_j, i < j), merged progressively into o[], then
// T = 2 o + sum x_i^2 4^i (funnel shifts, one fused chain of the diagonal squares)
template <int L, int I>
MPB_DEVI void sqr_rows(uint32_t (&U)[2 * L + 2], uint32_t (&V)[2 * L + 2], uint32_t& c, const uint32_t (&x)[L],
                       uint32_t (&o)[2 * L]) {
    if constexpr (I < L - 1) {
        grow<I, I + 1, L, false, false, I + L, 2 * L + 2, L>(U, V, x[I], x);
        // positions 2I+1 and 2I+2 are final (the next row starts at 2I+3)
        o[2 * I + 1] = merge_word(U, V, 2 * I + 1, c);
        o[2 * I + 2] = merge_word(U, V, 2 * I + 2, c);
        sqr_rows<L, I + 1>(U, V, c, x, o);
    } else {
        o[2 * L - 1] = merge_word(U, V, 2 * L - 1, c);  // the last position (2L-1 = 63)
    }
}
template <int L, class TH>
MPB_DEVI void sqr_T(const uint32_t (&x)[L], uint32_t (&tlo)[L], const TH& th) {
    uint32_t U[2 * L + 2], V[2 * L + 2];
#pragma unroll
    for (int k = 0; k < 2 * L + 2; k++) { U[k] = 0; V[k] = 0; }
    uint32_t o[2 * L];
    o[0] = 0;
    uint32_t c = 0;
    sqr_rows<L, 0>(U, V, c, x, o);
    // T = 2 o + D:  t[k] = (o[k] << 1) | (o[k-1] >> 31), then the squares at (2i, 2i+1)
    uint32_t t[2 * L];
#pragma unroll
    for (int k = 2 * L - 1; k >= 1; k--) t[k] = __funnelshift_l(o[k - 1], o[k], 1);
    t[0] = o[0] << 1;
    pr_first(t[0], t[1], x[0], x[0]);
#pragma unroll
    for (int i = 1; i < L - 1; i++) pr_next(t[2 * i], t[2 * i + 1], x[i], x[i]);
    pr_next_end(t[2 * L - 2], t[2 * L - 1], x[L - 1], x[L - 1]);
#pragma unroll
    for (int k = 0; k < L; k++) tlo[k] = t[k];
#pragma unroll
    for (int k = 0; k < L; k++) th(k, t[L + k]);
}

// ---- q = T_low * N' mod R: rows over N'[j] (from np(j)), multiplicand T_low (registers)
template <int L, int J, class NPW>
MPB_DEVI void q_rows(uint32_t (&U)[L + 2], uint32_t (&V)[L + 2], uint32_t& c, const NPW& np, const uint32_t (&tlo)[L],
                     uint32_t (&q)[L]) {
    if constexpr (J < L) {
        // row J: N'[J] * T_low[i] for i = 0 .. L-1-J at positions J + i (top position L-1 lo only)
        grow<J, 0, L - J, false, true, L - 1, L + 2, L>(U, V, np(J), tlo);
        q[J] = merge_word(U, V, J, c);
        q_rows<L, J + 1>(U, V, c, np, tlo, q);
    }
}

// ---- H = floor(q N / R) by Theorem 2 (products of weight >= L-1, hi halves of weight L-2, exact
// carry out of column L-1), then C = T_high + H + c_add and the masked subtraction of N.
// Rows over N[j] (from nw(j)), multiplicand q (registers).  Positions L-2 .. 2L-1.
template <int L, int J, class NW>
MPB_DEVI void h_rows(uint32_t (&U)[2 * L + 2], uint32_t (&V)[2 * L + 2], const NW& nw, const uint32_t (&q)[L]) {
    if constexpr (J < L) {
        if constexpr (J == L - 1) {
            // q_i N_{L-1} for all i >= 0: positions L-1+i, no hi-only product (i = -1 absent)
            grow<J, 0, L, false, false, J + L, 2 * L + 2, L>(U, V, nw(J), q);
        } else {
            // i from L-2-J (hi only: position L-2 is the dummy lo) to L-1
            grow<J, L - 2 - J, L, true, false, J + L, 2 * L + 2, L>(U, V, nw(J), q);
        }
        h_rows<L, J + 1>(U, V, nw, q);
    }
}

template <int L, class TH, class NW>
MPB_DEVI void trunc_reduce(const uint32_t (&tlo)[L], const TH& thr, const NW& nw, const uint32_t (&q)[L], uint32_t (&out)[L]) {
    uint32_t U[2 * L + 2], V[2 * L + 2];
#pragma unroll
    for (int k = 0; k < 2 * L + 2; k++) { U[k] = 0; V[k] = 0; }
    h_rows<L, 0>(U, V, nw, q);
    // b = [T mod 2^(32(L-1)) != 0], c_add = [T mod R != 0], K = (-T[L-1] - b) mod 2^32
    uint32_t orlo = 0;
#pragma unroll
    for (int k = 0; k < L - 1; k++) orlo |= tlo[k];
    const uint32_t b = orlo != 0u ? 1u : 0u;
    const uint32_t cadd = (orlo | tlo[L - 1]) != 0u ? 1u : 0u;
    const uint32_t K = 0u - tlo[L - 1] - b;
    // S = word L-1 of the included partial products: U[L-1] + V[L-2] (their higher carries are in the chains)
    uint32_t s = U[L - 1], sc = 0;
    asm volatile("add.cc.u32 %0, %0, %2;\n\taddc.u32 %1, 0, 0;" : "+r"(s), "+r"(sc) : "r"(V[L - 2]));
    const uint32_t corr = s > K ? 1u : 0u;  // exact carry out of column L-1 (Theorem 2)
    uint32_t cin = sc + corr + cadd;
    // C[k] = U[L+k] + V[L+k-1] + T_high[k] + carries
    uint32_t y[L + 1];
#pragma unroll
    for (int k = 0; k < L; k++) {
        uint32_t t = merge_word(U, V, L + k, cin);
        uint32_t cc = 0;
        asm volatile("add.cc.u32 %0, %0, %2;\n\taddc.u32 %1, 0, 0;" : "+r"(t), "+r"(cc) : "r"(thr(k)));
        cin += cc;
        y[k] = t;
    }
    y[L] = cin + U[2 * L] + V[2 * L - 1];
    // canonical: y >= N ? y - N : y
    uint32_t d[L], n[L];
#pragma unroll
    for (int k = 0; k < L; k++) { d[k] = y[k]; n[k] = nw(k); }
    sub_first(d[0], n[0]);
#pragma unroll
    for (int k = 1; k < L; k++) sub_next(d[k], n[k]);
    uint32_t top = y[L];
    asm volatile("subc.u32 %0, %0, 0;" : "+r"(top));
    const uint32_t m = 0u - (top == 0u ? 1u : 0u);
#pragma unroll
    for (int k = 0; k < L; k++) out[k] = (d[k] & m) | (y[k] & ~m);
}

// The whole truncated Montgomery operation: out = x^2 R^-1 mod N (sqr, x = b) or a b R^-1 mod N.
// aw(i): a_i; npw(j): N'[j]; nw(j): N[j]; thw(k, v) / thr(k): store / load word k of T_high.
// The product phase is the only part that differs; the reduction (q, H, C) is one shared instance.
template <int L, class AW, class NPW, class NW, class THW, class THR>
MPB_DEVI void montmul_trunc(bool sqr, const AW& aw, const uint32_t (&b)[L], const NPW& npw, const NW& nw,
                            const THW& thw, const THR& thr, uint32_t (&out)[L]) {
    uint32_t tlo[L];
    if (sqr) {
        sqr_T<L>(b, tlo, thw);
    } else {
        uint32_t U[2 * L + 2], V[2 * L + 2];
#pragma unroll
        for (int k = 0; k < 2 * L + 2; k++) { U[k] = 0; V[k] = 0; }
        uint32_t c = 0;
        mul_rows<L, 0>(U, V, c, aw, b, tlo, thw);
    }
    uint32_t q[L];
    {
        uint32_t U[L + 2], V[L + 2];
#pragma unroll
        for (int k = 0; k < L + 2; k++) { U[k] = 0; V[k] = 0; }
        uint32_t c = 0;
        q_rows<L, 0>(U, V, c, npw, tlo, q);
    }
    trunc_reduce<L>(tlo, thr, nw, q, out);
}

}  // namespace reg
}  // namespace mpb
