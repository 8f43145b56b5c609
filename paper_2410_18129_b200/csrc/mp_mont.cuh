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

#ifdef MPB_CORR_COUNT
// DEBUG builds only (csrc/debug/corr_count.cu -> libmpb_corr.so, a test artefact): how many times
// the exact carry correction of Theorem 2 ([S mod 2^32 > K]) evaluated to 1.  The
// counting branch depends on secret data, so no shipped build defines MPB_CORR_COUNT.
static __device__ unsigned long long g_corr_count;
#endif

// ----------------------------------------------------------------- accessors
// Word-sliced global array: chunk q (4 limbs, 16 bytes) of this thread's number at p + q*sb
// (sb = count * 16 bytes).  The chunk address is one IMAD.WIDE.U32 (32-bit q times 32-bit sb
// plus the 64-bit base).
// p + idx * sb as ONE mad.wide.u32 (32 x 32 -> 64 plus the 64-bit base)
MPB_DEVI char* chunk_addr(const char* p, uint32_t idx, uint32_t sb) {
    uint64_t a;
    asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(a) : "r"(idx), "r"(sb), "l"(reinterpret_cast<uint64_t>(p)));
    return reinterpret_cast<char*>(a);
}
// tm (optional): the TMA tensor map describing the whole array (bits 0..3: map index + 1, 0 = none)
// and this view's first chunk row in it (bits 4..31); see k_modexp / TmaMaps in kernels.cuh.
// SBC = 0: word-sliced array with the run-time stride sb (the ABI layout, DESIGN 5.6).
// SBC = kTileSB: warp-tiled workspace array (the exponentiation's internal arrays, DESIGN 5.6):
// the 32 operands of a warp tile keep chunk q of all 32 numbers in one 512-byte row, rows of one
// tile contiguous, so chunk q of this thread's number is at p + q * 512 -- a compile-time stride,
// and every chunk of a block is an immediate offset from one address.
template <uint32_t SBC>
struct ArrS {
    static constexpr uint32_t kSBC = SBC;
    char* p;
    uint32_t sb;
    uint32_t tm;
    MPB_DEVI uint4* addr(int q) const {
        if constexpr (SBC != 0) return reinterpret_cast<uint4*>(p + (ptrdiff_t)q * (ptrdiff_t)SBC);
        else return reinterpret_cast<uint4*>(chunk_addr(p, (uint32_t)q, sb));
    }
    MPB_DEVI uint4 ld(int q) const { return *addr(q); }
    MPB_DEVI uint4 ld_stream(int q) const { return __ldcs(addr(q)); }  // evict-first (table scans)
    MPB_DEVI void st(int q, uint4 v) const { *addr(q) = v; }
    MPB_DEVI ArrS at(int chunk) const {
        if constexpr (SBC != 0) return ArrS{p + (ptrdiff_t)chunk * (ptrdiff_t)SBC, sb, tm};
        else return ArrS{p + (size_t)(uint32_t)chunk * sb, sb, tm + ((uint32_t)chunk << 4)};
    }
};
constexpr uint32_t kTileSB = 512;  // one chunk row of a warp tile: 32 operands x 16 bytes
using Arr = ArrS<0>;
using ArrT = ArrS<kTileSB>;

// Per-thread shared-memory staging for the operand blocks of the next block product
// (double buffered, filled by cp.async while the current block product runs).
// Chunk c of this thread lives at base + c*cs bytes (cs = blockDim * 16: conflict-free LDS.128).
struct Stage {
    uint32_t base;
    uint32_t cs;
    // TMA path (engine<.., TMA = true>): this warp's tile stage, its two mbarriers, the warp's first
    // operand index and the kernel's tensor maps
    uint32_t tbase;
    uint32_t tbar;
    uint32_t kw;
    uint32_t amask;  // the warp's active lanes
    const void* maps;
};
// ---- TMA (cp.async.bulk.tensor) + mbarrier primitives
MPB_DEVI void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
MPB_DEVI void mbar_arrive_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
MPB_DEVI void mbar_wait(uint32_t bar, uint32_t phase) {
    uint32_t ok;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(bar), "r"(phase)
            : "memory");
    } while (!ok);
}
// 2-D tile of a word-sliced array: c0 = word offset (4 x operand index), c1 = chunk row
MPB_DEVI void tma_load_2d(uint32_t dst, const void* map, int c0, int c1, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            dst),
        "l"(map), "r"(c0), "r"(c1), "r"(bar)
        : "memory");
}
// Threads per CTA of every engine kernel (kernels.cuh kThreads): the stage stride blockDim * 16
// is then a compile-time constant and every staging address is base + immediate.
#ifdef MPB_THREADS
constexpr uint32_t kStageThreads = MPB_THREADS;
#else
constexpr uint32_t kStageThreads = 128;
#endif
constexpr uint32_t kStageCS = kStageThreads * 16;
MPB_DEVI void cp_async16(uint32_t saddr, const void* g) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(saddr), "l"(g) : "memory");
}
MPB_DEVI void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
MPB_DEVI void cp_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
MPB_DEVI uint4 lds128(uint32_t saddr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(saddr));
    return v;
}

template <int C, class AR = Arr>
MPB_DEVI void ldb(const AR& a, int blk, uint32_t (&x)[C]) {
#pragma unroll
    for (int q = 0; q < C / 4; q++) {
        uint4 v = a.ld(blk * (C / 4) + q);
        x[4 * q] = v.x; x[4 * q + 1] = v.y; x[4 * q + 2] = v.z; x[4 * q + 3] = v.w;
    }
}
template <int C, int N, class AR = Arr>
MPB_DEVI void stb(const AR& a, int blk, const uint32_t (&x)[N]) {
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

// ------------------------------------------------ shared tail: C, D = C - N
// Block j of H (window words 0..C-1) becomes block j of C = T_hi + H + carry (truncated) or
// of C itself (full); C is parked in T block NB+j and D = C - N - borrow goes to OUT block j.
// wr = false (the idle lane of a cooperative pair, mp_coop.cuh): nothing is stored and T is not
// read (zeros instead) -- that lane's results are discarded, and reading T here would race with
// the partner lane's store of the same block.
template <int C, class AR = Arr>
MPB_DEVI void emit_block(const uint32_t (&W)[2 * C + 1], int j, int NB, bool add_thi, const AR& T, const AR& N,
                         const AR& OUT, uint32_t& carry, uint32_t& borrow, bool wr = true) {
    uint32_t c[C];
#pragma unroll
    for (int i = 0; i < C; i++) c[i] = W[i];
    if (add_thi) {
        uint32_t t[C];
        if (wr) {
            ldb<C>(T, NB + j, t);
        } else {
#pragma unroll
            for (int i = 0; i < C; i++) t[i] = 0;
        }
        cc_restore(carry);
#pragma unroll
        for (int i = 0; i < C; i++) add_next(c[i], t[i]);
        carry = cc_save();
    }
    if (wr) stb<C>(T, NB + j, c);
    uint32_t n[C];
    ldb<C>(N, j, n);
    bc_restore(borrow);
#pragma unroll
    for (int i = 0; i < C; i++) sub_next(c[i], n[i]);
    borrow = bc_save();
    if (wr) stb<C>(OUT, j, c);
}

// OUT = (ctop || !borrow) ? D : C, with D in OUT and C in T[NB..2NB) -- a mask, no branch.
// Two blocks per step so that 4*(C/4) loads are in flight (the data was just written: L2 latency).
template <int C, class AR = Arr>
MPB_DEVI void final_select(int NB, const AR& T, const AR& OUT, uint32_t ctop, uint32_t borrow, bool wr = true) {
    const uint32_t m = 0u - ((ctop | (borrow ^ 1u)) & 1u);  // all ones: take D = C - N
    constexpr int Q = C / 4;
#pragma unroll 1
    for (int j = 0; j < NB; j += 2) {
        uint4 d[2 * Q], c[2 * Q];
        const bool two = j + 1 < NB;
#pragma unroll
        for (int q = 0; q < 2 * Q; q++) {
            if (q < Q || two) {
                d[q] = OUT.ld(j * Q + q);
                c[q] = T.ld((NB + j) * Q + q);
            }
        }
#pragma unroll
        for (int q = 0; q < 2 * Q; q++) {
            if (q < Q || two) {
                uint4 r;
                r.x = (d[q].x & m) | (c[q].x & ~m);
                r.y = (d[q].y & m) | (c[q].y & ~m);
                r.z = (d[q].z & m) | (c[q].z & ~m);
                r.w = (d[q].w & m) | (c[q].w & ~m);
                if (wr) OUT.st(j * Q + q, r);
            }
        }
    }
}

// ------------------------------------------------------------ the engine
// One generic block-column engine runs every phase of every Montgomery operation, so each
// block primitive exists once in a kernel's code (the hot loop stays inside the instruction
// cache).  Phases:
//   PH_MUL / PH_SQR  DST = AX*AY (AX^2): alg:8SBmul / alg:8SBsqu, blocked
//   PH_Q             DST = (AX mod R)*AY mod R, AX = T, AY = N'             (alg:montred l.1)
//                    also orlo = OR T[0..L-2], tl1 = T[L-1] (eq:c_add; A6)
//   PH_HI            AX = q, AY = N.  TRUNC: alg:trunc_montred lines 2-4 with
//                    qnhat from the partial products of weight >= L-1 and the exact carry
//                    correction [S mod 2^32 > K] (Theorem 2).
//                    FULL: alg:8MontRed lines 2-3, C = (T + q*N)/R.
//                    Then D = C - N and a masked select give the canonical result in OUT.
enum { PH_MUL = 0, PH_SQR = 1, PH_Q = 2, PH_HI = 3 };
// Full (non-diagonal, non-truncated) block products by one level of register Karatsuba
// (acc_kara) instead of the C x C schoolbook block, for C = 16 and at least KARA_MIN_NB blocks per
// number.  Measured (same box, one thread per operand, truncated REDC): 4096 bits +5.7 %, 3072 bits
// +2.3 %, 2048 bits +1.7 %, 1024 bits -2.9 %.  2048 bits keeps the schoolbook
// blocks: its gain is within 2 % and the schoolbook kernel is the roofline-reported headline.
// MPB_KARA_BLOCK = 0 disables it (tuning builds).
#ifndef MPB_KARA_BLOCK
#define MPB_KARA_BLOCK 1
#endif
#ifndef MPB_KARA_MIN_NB
#define MPB_KARA_MIN_NB 6
#endif
#ifndef MPB_KARA_C12
#define MPB_KARA_C12 1  // C = 12 blocks (4108 / 4154 bits): measured +1.4 % alone, +10.5 % with one wave
#endif
template <int C>
__host__ __device__ constexpr bool kara_blocks() {
    return MPB_KARA_BLOCK && (C == 16 || (C == 12 && MPB_KARA_C12));
}
enum { OP_MUL = 0, OP_MUL2 = 1, OP_SQR = 2, OP_LO = 3, OP_HI = 4 };

// TMA: the operand blocks of a pair are loaded per WARP as 2-D tiles (C/4 chunk rows x 32 operands
// = (C/4) * 512 bytes) by one lane with cp.async.bulk.tensor, completing on the warp's mbarrier for
// that buffer; the pair walk is identical in every lane, so the tile coordinates are warp-uniform.
// tph: the two buffers' mbarrier phase bits (carried across calls).
template <int C, bool TRUNC, bool TMA = false, class AR = Arr>
MPB_DEVI void engine(int ph, int NB, const AR& AX, const AR& AY, const AR& DST, const AR& T, const AR& N,
                     const AR& OUT, uint32_t& orlo, uint32_t& tl1, const Stage& sg, uint32_t* tph = nullptr) {
    uint32_t W[2 * C + 1];
    w_zero<C>(W);
    uint32_t carry = 0, borrow = 0;
    const bool sqr = ph == PH_SQR;
    const bool hi_trunc = TRUNC && ph == PH_HI;
    // block columns k0 .. k1-1; pairs (k, s) with s in [max(0, k-NB+1), min(k, NB-1)] (SQR: s <= k/2)
    int k0 = 0, k1 = 2 * NB - 1;
    if (ph == PH_Q) k1 = NB;
    if (ph == PH_HI) {
        if (TRUNC) {
            k0 = NB - 1;
            const uint32_t b = orlo != 0u ? 1u : 0u;
            carry = (orlo | tl1) != 0u ? 1u : 0u;  // c_add = [T mod R != 0]
            // corners: block column NB-2 contributes hi(q_s[C-1] * N_t[C-1]) at position L-1
#pragma unroll 1
            for (int s0 = 0; s0 + 2 <= NB; s0 += 4) {  // 4 corners per step: loads in flight together
                uint32_t qw[4], nw[4];
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    const int s = s0 + u;
                    qw[u] = nw[u] = 0;
                    if (s + 2 <= NB) {
                        qw[u] = AX.ld(s * (C / 4) + C / 4 - 1).w;
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
        // FULL: k1 = 2NB-1 here; the empty top column 2NB-1 is finished after the loop
    }
    // One linear walk over the pairs: (k, s) is the pair being computed, (nk, ns) the next one,
    // whose operand blocks are prefetched (cp.async, double buffered) while (k, s) runs.
    const char* const axp = AX.p;
    const char* const ayp = AY.p;
    const uint32_t sbx = AX.sb, sby = AY.sb;  // arrays may hold different operand counts
    constexpr uint32_t kTile = (C / 4) * 512u;  // one operand block of 32 operands
    const uint32_t lane = threadIdx.x & 31u;
    if constexpr (TMA) {
        // AX / AY were written (generic proxy) by earlier phases of this warp; make those writes
        // visible to the async proxy before the first tile load of this phase
        asm volatile("fence.proxy.async;" ::: "memory");
        __syncwarp(sg.amask);
    }
    auto issue = [&](int kk, int ss, int buf) {
        if constexpr (TMA) {
            const bool dg = sqr && 2 * ss == kk;
            const uint32_t dst = sg.tbase + (uint32_t)buf * 2u * kTile;
            const uint32_t bar = sg.tbar + (uint32_t)buf * 8u;
            __syncwarp(sg.amask);  // every lane has read this buffer's previous tiles (two pairs ago)
            if (lane == 0) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_arrive_tx(bar, dg ? kTile : 2u * kTile);
                const char* maps = static_cast<const char*>(sg.maps);
                tma_load_2d(dst, maps + ((AX.tm & 15u) - 1u) * 128u, (int)(4u * sg.kw),
                            (int)((AX.tm >> 4) + (uint32_t)ss * (C / 4)), bar);
                if (!dg)
                    tma_load_2d(dst + kTile, maps + ((AY.tm & 15u) - 1u) * 128u, (int)(4u * sg.kw),
                                (int)((AY.tm >> 4) + (uint32_t)(kk - ss) * (C / 4)), bar);
            }
        } else {
            const uint32_t b = sg.base + (uint32_t)(buf * 2 * (C / 4)) * kStageCS;
            if constexpr (AR::kSBC != 0) {  // warp tile: one address per block, immediate row offsets
                const char* bx = reinterpret_cast<const char*>(AX.addr(ss * (C / 4)));
#pragma unroll
                for (int q = 0; q < C / 4; q++) cp_async16(b + q * kStageCS, bx + q * AR::kSBC);
                if (!(sqr && 2 * ss == kk)) {
                    const char* by = reinterpret_cast<const char*>(AY.addr((kk - ss) * (C / 4)));
#pragma unroll
                    for (int q = 0; q < C / 4; q++) cp_async16(b + (C / 4 + q) * kStageCS, by + q * AR::kSBC);
                }
            } else {
                const uint32_t cx = (uint32_t)ss * (C / 4), cy = (uint32_t)(kk - ss) * (C / 4);
#pragma unroll
                for (int q = 0; q < C / 4; q++) cp_async16(b + q * kStageCS, chunk_addr(axp, cx + q, sbx));
                if (!(sqr && 2 * ss == kk)) {
#pragma unroll
                    for (int q = 0; q < C / 4; q++)
                        cp_async16(b + (C / 4 + q) * kStageCS, chunk_addr(ayp, cy + q, sby));
                }
            }
            cp_commit();
        }
    };
    int k = k0, s = k0 - NB + 1 > 0 ? k0 - NB + 1 : 0;
    int s_hi = sqr ? (k >> 1) : (k < NB - 1 ? k : NB - 1);
    issue(k, s, 0);
    int buf = 0;
#pragma unroll 1
    while (k < k1) {
        // next pair
        int nk = k, ns = s + 1, ns_hi = s_hi;
        if (ns > s_hi) {
            nk = k + 1;
            ns = nk - NB + 1 > 0 ? nk - NB + 1 : 0;
            ns_hi = sqr ? (nk >> 1) : (nk < NB - 1 ? nk : NB - 1);
        }
        const bool more = nk < k1;
        if constexpr (TMA) {
            if (more) issue(nk, ns, buf ^ 1);
            mbar_wait(sg.tbar + (uint32_t)buf * 8u, (*tph >> buf) & 1u);
            *tph ^= 1u << buf;
        } else {
            if (more) {
                issue(nk, ns, buf ^ 1);
                cp_wait<1>();
            } else {
                cp_wait<0>();
            }
        }
        const int t = k - s;
        const bool diag = sqr && s == t;
        uint32_t x[C], y[C];
        {
            // cp.async stage: chunk c of this thread at base + c * kStageCS; TMA tile: row c of the
            // warp's tile, this lane's 16 bytes at + lane * 16 (both conflict-free LDS.128)
            const uint32_t b = TMA ? sg.tbase + (uint32_t)buf * 2u * kTile + lane * 16u
                                   : sg.base + (uint32_t)(buf * 2 * (C / 4)) * kStageCS;
            constexpr uint32_t rs = TMA ? 512u : kStageCS;
            constexpr uint32_t yo = TMA ? kTile : (C / 4) * kStageCS;
#pragma unroll
            for (int q = 0; q < C / 4; q++) {
                const uint4 v = lds128(b + q * rs);
                x[4 * q] = v.x; x[4 * q + 1] = v.y; x[4 * q + 2] = v.z; x[4 * q + 3] = v.w;
            }
            if (!diag) {
#pragma unroll
                for (int q = 0; q < C / 4; q++) {
                    const uint4 v = lds128(b + yo + q * rs);
                    y[4 * q] = v.x; y[4 * q + 1] = v.y; y[4 * q + 2] = v.z; y[4 * q + 3] = v.w;
                }
            }
        }
        buf ^= 1;
        if (ph == PH_Q && t == 0) {  // block T_k is loaded with t == 0 exactly once
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
        } else if (kara_blocks<C>() && NB >= MPB_KARA_MIN_NB) {  // register Karatsuba block (acc_kara)
            if (sqr) acc_kara<C, 2>(W, x, y);  // s < t: the product counts twice
            else acc_kara<C, 1>(W, x, y);
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
        if (nk != k) {  // ---- end of block column k
            if (ph != PH_HI) {
                stb<C>(DST, k, W);
                w_shift<C>(W);
            } else if (TRUNC) {
                if (k == NB - 1) {
                    // exact carry out of column L-1: floor(S/2^32) + [S mod 2^32 > K]
                    const uint32_t corr = W[0] > orlo ? 1u : 0u;
#ifdef MPB_CORR_COUNT
                    if (corr) atomicAdd(&g_corr_count, 1ull);
#endif
#pragma unroll
                    for (int i = 0; i < 2 * C; i++) W[i] = W[i + 1];
                    W[2 * C] = 0;
                    add_first(W[0], corr);
#pragma unroll
                    for (int i = 1; i <= C; i++) add_next(W[i], 0u);
                    absorb(W[C + 1]);
                } else {
                    emit_block<C>(W, k - NB, NB, true, T, N, OUT, carry, borrow);
                    w_shift<C>(W);
                }
            } else {
                uint32_t tb[C];  // + T block k, carried through the whole window
                ldb<C>(T, k, tb);
                add_first(W[0], tb[0]);
#pragma unroll
                for (int i = 1; i < C; i++) add_next(W[i], tb[i]);
#pragma unroll
                for (int i = C; i < 2 * C; i++) add_next(W[i], 0u);
                absorb(W[2 * C]);
                if (k >= NB) emit_block<C>(W, k - NB, NB, false, T, N, OUT, carry, borrow);
                w_shift<C>(W);
            }
        }
        k = nk;
        s = ns;
        s_hi = ns_hi;
    }
    if (ph == PH_MUL || ph == PH_SQR) stb<C>(DST, 2 * NB - 1, W);
    if (ph == PH_HI) {
        if (TRUNC) {
            emit_block<C>(W, NB - 1, NB, true, T, N, OUT, carry, borrow);
        } else {  // empty top column 2NB-1: + T block 2NB-1, emit the last block of C
            uint32_t tb[C];
            ldb<C>(T, 2 * NB - 1, tb);
            add_first(W[0], tb[0]);
#pragma unroll
            for (int i = 1; i < C; i++) add_next(W[i], tb[i]);
            add_next(W[C], 0u);
            emit_block<C>(W, NB - 1, NB, false, T, N, OUT, carry, borrow);
        }
        final_select<C>(NB, T, OUT, TRUNC ? carry : W[C], borrow);
    }
}

// Montgomery operation through the engine (single call site for all phases).
//   mode MUL:  OUT = X*B*R^-1 mod N      mode SQR: OUT = X^2*R^-1 mod N
//   mode REDC: OUT = T*R^-1 mod N for the 2L-word T already in scratch T
enum { MODE_MUL = 0, MODE_SQR = 1, MODE_REDC = 2 };

template <int C, bool TRUNC, bool TMA = false, class AR = Arr>
MPB_DEVI void mont_op(int mode, int NB, const AR& X, const AR& B, const AR& N, const AR& NP, const AR& T, const AR& Q,
                      const AR& OUT, const Stage& sg, uint32_t* tph = nullptr) {
    uint32_t orlo = 0, tl1 = 0;
#pragma unroll 1
    for (int step = mode == MODE_REDC ? 1 : 0; step < 3; step++) {
        const int ph = step == 0 ? (mode == MODE_SQR ? PH_SQR : PH_MUL) : (step == 1 ? PH_Q : PH_HI);
        const AR ax = step == 0 ? X : (step == 1 ? T : Q);
        const AR ay = step == 0 ? B : (step == 1 ? NP : N);
        const AR dst = step == 0 ? T : Q;
        engine<C, TRUNC, TMA>(ph, NB, ax, ay, dst, T, N, OUT, orlo, tl1, sg, tph);
    }
}

// ------------------------------------------------- CIOS (third REDC mode)
// alg:8BlockMontRed, the CIOS-inspired interleaved Montgomery multiplication, with
// the paper's machine word (52 bits, one VPMADD52 lane) replaced by the engine's block of C limbs:
// digit d = 2^{32C}, m_i = (Y mod d) * N' mod d (only the low block of N', the block analog of
// n0'), then Y <- (Y + m_i N) / d.  Per row i the block pass t = 0..NB-1 computes
//   Z_t = carry + Y_t + a_i B_t + m_i N_t,  Y_{t-1} <- Z_t mod d,  carry <- Z_t / d
// (block 0 of Z vanishes by the choice of m_i).  Y < 2N throughout, so Y has L limbs plus a top
// word; the result is canonicalised by one masked conditional subtraction.  B_ONE: B = 1 (used
// for REDC(X) = MontMul(X, 1) in the exponentiation).  Scratch: Y (L limbs), M (C limbs).
// SQR (MontSqr, B unused): squaring rows at block granularity -- row i adds a_i^2 at pass t = i
// and 2 a_i a_t at passes t > i (nothing below): each cross block product once, doubled, the
// diagonal blocks as symmetric squares (a^2 = sum_i a_i^2 d^(2i) + 2 sum_{i<t} a_i a_t d^(i+t)).
// Pass t < i of row i touches only blocks >= t where row i's a-part starts at block i, so block 0
// of Z (m_i) is complete as in CIOS.  Rows r <= i add < 2a d^(i+1) in all, so Y < 2a + N < 3N
// between rows (the top word holds 0..2) and < 2N at the end.  NB(NB-1)/2 full and NB square
// blocks instead of NB^2 full blocks for the a-part (2 080 instead of 4 096 products at 2048 bits).
template <int C, class AR = Arr>
MPB_DEVI void cios_op(int NB, const AR& X, const AR& B, bool b_one, const AR& N, const AR& NP, const AR& Y,
                      const AR& M, const AR& OUT, bool sqr = false) {
    uint32_t ytop = 0;
#pragma unroll 1
    for (int i = 0; i < NB; i++) {
        uint32_t W[2 * C + 1];
        w_zero<C>(W);
#pragma unroll 1
        for (int t = 0; t < NB; t++) {
            if (i > 0) {  // + Y_t (Y = 0 before the first row)
                uint32_t yt[C];
                ldb<C>(Y, t, yt);
                w_add<0, C, 0>(W, yt);
            }
            if (!sqr) {  // + a_i * B_t
                uint32_t x[C], y[C];
                ldb<C>(X, i, x);
                if (b_one) {
#pragma unroll
                    for (int k = 0; k < C; k++) y[k] = 0;
                    y[0] = t == 0 ? 1u : 0u;
                } else {
                    ldb<C>(B, t, y);
                }
                acc_mul<C>(W, x, y);
            } else if (t == i) {  // squaring row: + a_i^2
                uint32_t x[C];
                ldb<C>(X, i, x);
                acc_sqr<C>(W, x);
            } else if (t > i) {  // squaring row: + 2 a_i a_t
                uint32_t x[C], y[C];
                ldb<C>(X, i, x);
                ldb<C>(X, t, y);
                acc_mul2<C>(W, x, y);
            }
            if (t == 0) {  // m_i = (Z mod d) * N' mod d  (low-half block product)
                uint32_t z[C], np[C], E[2 * C], O[2 * C];
#pragma unroll
                for (int k = 0; k < C; k++) z[k] = W[k];
                ldb<C>(NP, 0, np);
                bp_lo<C>(z, np, E, O);
                uint32_t m[C];
#pragma unroll
                for (int k = 0; k < C; k++) m[k] = E[k];
                w_add_trunc<1, C - 1, 0>(m, O);
                stb<C>(M, 0, m);
            }
            {  // + m_i * N_t
                uint32_t m[C], n[C];
                ldb<C>(M, 0, m);
                ldb<C>(N, t, n);
                acc_mul<C>(W, m, n);
            }
            if (t > 0) stb<C>(Y, t - 1, W);  // block 0 of Z_0 is zero
            w_shift<C>(W);
        }
        // W[0..C] = the top of Z (positions L .. L+C); add the old top bit of Y at position L
        add_first(W[0], ytop);
#pragma unroll
        for (int k = 1; k <= C; k++) add_next(W[k], 0u);
        stb<C>(Y, NB - 1, W);
        ytop = W[C];
    }
    // canonical: OUT = (ytop || Y >= N) ? Y - N : Y, by a mask
    uint32_t borrow = 0;
#pragma unroll 1
    for (int j = 0; j < NB; j++) {
        uint32_t c[C], n[C];
        ldb<C>(Y, j, c);
        ldb<C>(N, j, n);
        bc_restore(borrow);
#pragma unroll
        for (int k = 0; k < C; k++) sub_next(c[k], n[k]);
        borrow = bc_save();
        stb<C>(OUT, j, c);
    }
    const uint32_t msk = 0u - ((ytop | (borrow ^ 1u)) & 1u);
#pragma unroll 1
    for (int j = 0; j < NB; j++) {
#pragma unroll
        for (int q = 0; q < C / 4; q++) {
            uint4 d = OUT.ld(j * (C / 4) + q);
            const uint4 y = Y.ld(j * (C / 4) + q);
            d.x = (d.x & msk) | (y.x & ~msk);
            d.y = (d.y & msk) | (y.y & ~msk);
            d.z = (d.z & msk) | (y.z & ~msk);
            d.w = (d.w & msk) | (y.w & ~msk);
            OUT.st(j * (C / 4) + q, d);
        }
    }
}

// ---------------------------------------------------------- CT table select
#ifdef MPB_PLANTED_BRANCH
#define MPB_PLANTED 1
#else
#define MPB_PLANTED 0
#endif
// OUT = G[idx] by a masked scan of every entry ("constant-time batch selection").
// Entry e, chunk q lives at chunk index e*(L/4) + q of G.  The scan is bound by DRAM latency
// (the tables of all resident operands exceed L2), so it keeps U entries x GRP chunks of
// loads in flight per step; accumulators stay in registers at every L.
// part / nparts: this thread scans chunk groups part, part + nparts, ... (cooperative operands
// split the scan between their lanes; every entry is still read in full by the operand's lanes).
template <int U, int GRP, class AR = Arr>
MPB_DEVI void ct_select(const AR& G, int L, int nent, uint32_t idx, const AR& OUT, int part = 0, int nparts = 1) {
    const int Q4 = L / 4;
    if constexpr (AR::kSBC != 0) {
        // warp tile: every load of a step is an immediate offset from one address, and with whole
        // steps (nent % U == 0, Q4 % GRP == 0: the tiled sizes at w >= 2) no load needs a guard
        if (!MPB_PLANTED && nent % U == 0 && Q4 % GRP == 0) {
            constexpr int RW = AR::kSBC / 16;  // uint4 per chunk row
#pragma unroll 1
            for (int g0 = part * GRP; g0 < Q4; g0 += nparts * GRP) {
                uint4 acc[GRP];
#pragma unroll
                for (int q = 0; q < GRP; q++) acc[q] = make_uint4(0, 0, 0, 0);
#pragma unroll 1
                for (int e0 = 0; e0 < nent; e0 += U) {
                    const uint4* eb = G.addr(e0 * Q4 + g0);
                    uint4 v[U][GRP];
#pragma unroll
                    for (int u = 0; u < U; u++)
#pragma unroll
                        for (int q = 0; q < GRP; q++) v[u][q] = __ldcs(eb + (u * Q4 + q) * RW);
#pragma unroll
                    for (int u = 0; u < U; u++) {
                        const uint32_t x = (uint32_t)(e0 + u) ^ idx;
                        const uint32_t m = 0u - ((x - 1u) >> 31);  // all ones iff e == idx
#pragma unroll
                        for (int q = 0; q < GRP; q++) {
                            acc[q].x |= v[u][q].x & m;
                            acc[q].y |= v[u][q].y & m;
                            acc[q].z |= v[u][q].z & m;
                            acc[q].w |= v[u][q].w & m;
                        }
                    }
                }
                uint4* ob = OUT.addr(g0);
#pragma unroll
                for (int q = 0; q < GRP; q++) ob[q * RW] = acc[q];
            }
            return;
        }
    }
#pragma unroll 1
    for (int g0 = part * GRP; g0 < Q4; g0 += nparts * GRP) {
        uint4 acc[GRP];
#pragma unroll
        for (int q = 0; q < GRP; q++) acc[q] = make_uint4(0, 0, 0, 0);
#pragma unroll 1
        for (int e0 = 0; e0 < nent; e0 += U) {
            uint4 v[U][GRP];
#pragma unroll
            for (int u = 0; u < U; u++)
#pragma unroll
                for (int q = 0; q < GRP; q++)
#ifdef MPB_PLANTED_BRANCH  // NEGATIVE CONTROL ONLY (tools/ct_check.py): secret-dependent branch + address
                    v[u][q] = ((uint32_t)(e0 + u) == idx && g0 + q < Q4) ? G.ld_stream((e0 + u) * Q4 + g0 + q)
                                                                         : make_uint4(0, 0, 0, 0);
#else
                    v[u][q] = (e0 + u < nent && g0 + q < Q4) ? G.ld_stream((e0 + u) * Q4 + g0 + q)
                                                              : make_uint4(0, 0, 0, 0);
#endif
#pragma unroll
            for (int u = 0; u < U; u++) {
                const uint32_t x = (uint32_t)(e0 + u) ^ idx;
                const uint32_t m = 0u - ((x - 1u) >> 31);  // all ones iff e == idx (x < 2^31)
#pragma unroll
                for (int q = 0; q < GRP; q++) {
                    acc[q].x |= v[u][q].x & m;
                    acc[q].y |= v[u][q].y & m;
                    acc[q].z |= v[u][q].z & m;
                    acc[q].w |= v[u][q].w & m;
                }
            }
        }
#pragma unroll
        for (int q = 0; q < GRP; q++)
            if (g0 + q < Q4) OUT.st(g0 + q, acc[q]);
    }
}

}  // namespace mpb
