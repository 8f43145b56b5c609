// mp_coop.cuh -- warp-cooperative operands: G = 2, 4 or 8 adjacent lanes of a warp per operand
// (north_star (b); sm_100a).
//
// The one-thread-per-operand engine (mp_mont.cuh) needs one resident thread per operand, so a batch
// much smaller than the resident capacity leaves SMs idle (Launch::modexp uses G lanes for small
// >= 3072-bit batches: 1.71x at 2 048 x 4096-bit operands with 8 lanes).  The G
// lanes Gm .. Gm+G-1 own operand m (role r = lane mod G) and split the block products of every
// block column: in iteration i of column k, role r takes the pair s = s_lo + G*i + r (PH_SQR: the
// off-diagonal pairs, then one iteration for the diagonal block, which role 0 computes and the
// others run on a zero block).  A role without a pair in an iteration multiplies a zero block, so
// all lanes always execute the same instructions.  At the end of a column the lanes sum their
// windows by a shuffle butterfly (log2 G rounds of 33 shuffles and one 33-word add chain), so all
// hold the column total and run the column action (store, truncated-REDC correction, emit)
// identically; only role 0 stores and reads the T blocks the phase rewrites, and the other roles
// clear their carry-in so the next column counts it once.  Per operand the product work is split
// G ways; the column actions are repeated in every lane.  Same results as the single-thread
// engine; constant time in the same sense (public schedule).
#pragma once
#include "mp_mont.cuh"

namespace mpb {

// W (2C+1 words) = the sum of the G lanes' windows (butterfly over lanes xor 1, 2, .., G/2): every
// lane of the group ends with the same total.  Partial sums never exceed the total (all terms are
// non-negative parts of one column sum), so the window cannot overflow.
template <int C, int G>
MPB_DEVI void coop_window_sum(uint32_t (&W)[2 * C + 1], unsigned mask) {
#pragma unroll
    for (int m = 1; m < G; m <<= 1) {
        uint32_t o[2 * C + 1];
#pragma unroll
        for (int i = 0; i <= 2 * C; i++) o[i] = __shfl_xor_sync(mask, W[i], m);
        add_first(W[0], o[0]);
#pragma unroll
        for (int i = 1; i < 2 * C; i++) add_next(W[i], o[i]);
        add_end(W[2 * C], o[2 * C]);
    }
}
template <int G>
MPB_DEVI uint32_t coop_or(uint32_t v, unsigned mask) {
#pragma unroll
    for (int m = 1; m < G; m <<= 1) v |= __shfl_xor_sync(mask, v, m);
    return v;
}

// G lanes per operand (G = 2, 4, 8): role r in [0, G) takes the pairs s = s_lo + G*i + r of each
// block column; role 0 alone carries the column's carry-in, stores, and reads T blocks the phase
// rewrites (see the invariant at the column end).
template <int C, bool TRUNC, int G = 2, class AR = Arr>
MPB_DEVI void engine_coop(int ph, int NB, const AR& AX, const AR& AY, const AR& DST, const AR& T, const AR& N,
                          const AR& OUT, uint32_t& orlo, uint32_t& tl1, const Stage& sg, uint32_t role,
                          unsigned mask) {
    uint32_t W[2 * C + 1];
    w_zero<C>(W);
    uint32_t carry = 0, borrow = 0;
    const bool sqr = ph == PH_SQR;
    const bool hi_trunc = TRUNC && ph == PH_HI;
    const uint32_t keep = role ? 0u : 0xFFFFFFFFu;  // role 0 keeps the carry-in / one-off terms
    int k0 = 0, k1 = 2 * NB - 1;
    if (ph == PH_Q) k1 = NB;
    if (ph == PH_HI && TRUNC) {
        k0 = NB - 1;
        const uint32_t b = orlo != 0u ? 1u : 0u;
        carry = (orlo | tl1) != 0u ? 1u : 0u;  // c_add = [T mod R != 0]
#pragma unroll 1
        for (int s0 = 0; s0 + 2 <= NB; s0 += 4) {  // corners (role 0 only: role 1 adds zeros)
            uint32_t qw[4], nw[4];
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const int s = s0 + u;
                qw[u] = nw[u] = 0;
                if (s + 2 <= NB) {
                    qw[u] = AX.ld(s * (C / 4) + C / 4 - 1).w & keep;
                    nw[u] = AY.ld((NB - 2 - s) * (C / 4) + C / 4 - 1).w;
                }
            }
#pragma unroll
            for (int u = 0; u < 4; u++)
                asm volatile("mad.hi.cc.u32 %0, %2, %3, %0;\n\taddc.u32 %1, %1, 0;"
                             : "+r"(W[0]), "+r"(W[1]) : "r"(qw[u]), "r"(nw[u]));
        }
        orlo = 0u - tl1 - b;  // reuse: K = (-T[L-1] - b) mod 2^32
    }
    // column k: pairs s in [s_lo, s_hi] (PH_SQR: off-diagonal s < t only) split by role, plus the
    // diagonal iteration for even k in PH_SQR
    auto s_lo_of = [&](int k) { return k - NB + 1 > 0 ? k - NB + 1 : 0; };
    auto s_hi_of = [&](int k) { return sqr ? ((k - 1) >> 1) : (k < NB - 1 ? k : NB - 1); };
    auto iters_of = [&](int k) {
        const int n = s_hi_of(k) - s_lo_of(k) + 1;
        return (n > 0 ? (n + G - 1) / G : 0) + ((sqr && !(k & 1)) ? 1 : 0);
    };
    // this role's pair in iteration it of column k: s (a valid block index), valid, diagonal
    auto pair_of = [&](int k, int it, int& s, bool& valid, bool& diag) {
        diag = sqr && !(k & 1) && it == iters_of(k) - 1;
        if (diag) {
            s = k >> 1;
            valid = role == 0;
        } else {
            s = s_lo_of(k) + G * it + (int)role;
            valid = s <= s_hi_of(k);
            if (!valid) s = s_lo_of(k);
        }
    };
    const char* const axp = AX.p;
    const char* const ayp = AY.p;
    const uint32_t sbx = AX.sb, sby = AY.sb;
    auto issue = [&](int kk, int it, int buf) {
        int ss;
        bool valid, dg;
        pair_of(kk, it, ss, valid, dg);
        const uint32_t b = sg.base + (uint32_t)(buf * 2 * (C / 4)) * kStageCS;
        if constexpr (AR::kSBC != 0) {  // warp tile: one address per block, immediate row offsets
            const char* bx = reinterpret_cast<const char*>(AX.addr(ss * (C / 4)));
#pragma unroll
            for (int q = 0; q < C / 4; q++) cp_async16(b + q * kStageCS, bx + q * AR::kSBC);
            if (!dg) {
                const char* by = reinterpret_cast<const char*>(AY.addr((kk - ss) * (C / 4)));
#pragma unroll
                for (int q = 0; q < C / 4; q++) cp_async16(b + (C / 4 + q) * kStageCS, by + q * AR::kSBC);
            }
        } else {
            const uint32_t cx = (uint32_t)ss * (C / 4), cy = (uint32_t)(kk - ss) * (C / 4);
#pragma unroll
            for (int q = 0; q < C / 4; q++) cp_async16(b + q * kStageCS, chunk_addr(axp, cx + q, sbx));
            if (!dg) {
#pragma unroll
                for (int q = 0; q < C / 4; q++)
                    cp_async16(b + (C / 4 + q) * kStageCS, chunk_addr(ayp, cy + q, sby));
            }
        }
        cp_commit();
    };
    int k = k0, it = 0;
    issue(k, it, 0);
    int buf = 0;
#pragma unroll 1
    while (k < k1) {
        int nk = k, nit = it + 1;
        if (nit >= iters_of(k)) {
            nk = k + 1;
            nit = 0;
        }
        const bool more = nk < k1;
        if (more) {
            issue(nk, nit, buf ^ 1);
            cp_wait<1>();
        } else {
            cp_wait<0>();
        }
        int s;
        bool valid, diag;
        pair_of(k, it, s, valid, diag);
        const int t = k - s;
        const uint32_t vm = valid ? 0xFFFFFFFFu : 0u;  // an idle role multiplies a zero block
        uint32_t x[C], y[C];
        {
            const uint32_t b = sg.base + (uint32_t)(buf * 2 * (C / 4)) * kStageCS;
#pragma unroll
            for (int q = 0; q < C / 4; q++) {
                const uint4 v = lds128(b + q * kStageCS);
                x[4 * q] = v.x & vm; x[4 * q + 1] = v.y & vm; x[4 * q + 2] = v.z & vm; x[4 * q + 3] = v.w & vm;
            }
            if (!diag) {
#pragma unroll
                for (int q = 0; q < C / 4; q++) {
                    const uint4 v = lds128(b + (C / 4 + q) * kStageCS);
                    y[4 * q] = v.x; y[4 * q + 1] = v.y; y[4 * q + 2] = v.z; y[4 * q + 3] = v.w;
                }
            }
        }
        buf ^= 1;
        if (ph == PH_Q && t == 0 && valid) {  // block T_k (one of the roles sees it)
#pragma unroll
            for (int i = 0; i < C - 1; i++) orlo |= x[i];
            if (k == NB - 1) tl1 = x[C - 1];
            else orlo |= x[C - 1];
        }
        const bool lo_col = ph == PH_Q && k == NB - 1;
        const bool hi_col = hi_trunc && k == NB - 1;
        if (diag) {
            acc_sqr<C>(W, x);
        } else if (lo_col) {
            acc_lo<C>(W, x, y);
        } else if (hi_col) {
            acc_hi<C>(W, x, y);
        } else {
            uint32_t E[2 * C], O[2 * C];
            bp_mul<C>(x, y, E, O);
            w_add<0, 2 * C, 0>(W, E);
            w_add<1, 2 * C - 1, 0>(W, O);
            if (sqr) {  // s < t: the product counts twice
                w_add<0, 2 * C, 0>(W, E);
                w_add<1, 2 * C - 1, 0>(W, O);
            }
        }
        if (nk != k) {  // ---- end of block column k: both lanes hold the column total
            // Invariant: only role 0 stores (DST, T, OUT) and only role 0 reads T blocks that this
            // phase rewrites; role 1's column results are discarded (its window is cleared below)
            // and the phase ends with __syncwarp, so no lane reads a block the other is storing.
            coop_window_sum<C, G>(W, mask);
            if (ph != PH_HI) {
                if (role == 0) stb<C>(DST, k, W);
                w_shift<C>(W);
            } else if (TRUNC) {
                if (k == NB - 1) {
                    const uint32_t corr = W[0] > orlo ? 1u : 0u;
#pragma unroll
                    for (int i = 0; i < 2 * C; i++) W[i] = W[i + 1];
                    W[2 * C] = 0;
                    add_first(W[0], corr);
#pragma unroll
                    for (int i = 1; i <= C; i++) add_next(W[i], 0u);
                    absorb(W[C + 1]);
                } else {
                    emit_block<C>(W, k - NB, NB, true, T, N, OUT, carry, borrow, role == 0);
                    w_shift<C>(W);
                }
            } else {
                uint32_t tb[C];
                if (role == 0) {
                    ldb<C>(T, k, tb);
                } else {
#pragma unroll
                    for (int i = 0; i < C; i++) tb[i] = 0;
                }
                add_first(W[0], tb[0]);
#pragma unroll
                for (int i = 1; i < C; i++) add_next(W[i], tb[i]);
#pragma unroll
                for (int i = C; i < 2 * C; i++) add_next(W[i], 0u);
                absorb(W[2 * C]);
                if (k >= NB) emit_block<C>(W, k - NB, NB, false, T, N, OUT, carry, borrow, role == 0);
                w_shift<C>(W);
            }
#pragma unroll
            for (int i = 0; i <= 2 * C; i++) W[i] &= keep;  // the carry-in lives in role 0 only
        }
        k = nk;
        it = nit;
    }
    // the top of the walk: only role 0's window is non-zero; make every lane hold it
    coop_window_sum<C, G>(W, mask);
    if ((ph == PH_MUL || ph == PH_SQR) && role == 0) stb<C>(DST, 2 * NB - 1, W);
    if (ph == PH_Q) {  // every role needs c_add / the correction inputs
        orlo = coop_or<G>(orlo, mask);
        tl1 = coop_or<G>(tl1, mask);
    }
    if (ph == PH_HI) {
        if (TRUNC) {
            emit_block<C>(W, NB - 1, NB, true, T, N, OUT, carry, borrow, role == 0);
        } else {
            uint32_t tb[C];
            if (role == 0) {
                ldb<C>(T, 2 * NB - 1, tb);
            } else {
#pragma unroll
                for (int i = 0; i < C; i++) tb[i] = 0;
            }
            add_first(W[0], tb[0]);
#pragma unroll
            for (int i = 1; i < C; i++) add_next(W[i], tb[i]);
            add_next(W[C], 0u);
            emit_block<C>(W, NB - 1, NB, false, T, N, OUT, carry, borrow, role == 0);
        }
        final_select<C>(NB, T, OUT, TRUNC ? carry : W[C], borrow, role == 0);
    }
    __syncwarp(mask);  // both lanes' stores are visible to both before the next phase
}

template <int C, bool TRUNC, int G = 2, class AR = Arr>
MPB_DEVI void mont_op_coop(int mode, int NB, const AR& X, const AR& B, const AR& N, const AR& NP, const AR& T,
                           const AR& Q, const AR& OUT, const Stage& sg, uint32_t role, unsigned mask) {
    uint32_t orlo = 0, tl1 = 0;
#pragma unroll 1
    for (int step = mode == MODE_REDC ? 1 : 0; step < 3; step++) {
        const int ph = step == 0 ? (mode == MODE_SQR ? PH_SQR : PH_MUL) : (step == 1 ? PH_Q : PH_HI);
        const AR ax = step == 0 ? X : (step == 1 ? T : Q);
        const AR ay = step == 0 ? B : (step == 1 ? NP : N);
        const AR dst = step == 0 ? T : Q;
        engine_coop<C, TRUNC, G>(ph, NB, ax, ay, dst, T, N, OUT, orlo, tl1, sg, role, mask);
    }
}

}  // namespace mpb
