// kernels.cuh -- the templated sm_100a kernels of libmpb.so and their launchers.
// Templated on the block size C only; the block count nb = L / C is a runtime argument.
// Instantiated once per C in inst_C*.cu; api.cu holds the C ABI and sees only launch.h.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <type_traits>

#include "launch.h"
#include "mp_kara.cuh"
#include "mp_coop.cuh"
#include "mp_mont.cuh"
#include "mp_setup.cuh"

namespace mpb {

#ifdef MPB_THREADS
constexpr int kThreads = MPB_THREADS;
#else
constexpr int kThreads = 128;
#endif

static_assert(kThreads == (int)kStageThreads, "the engine's stage stride assumes blockDim == kThreads");

// resident CTAs per SM the heavy kernels are compiled for (register budget 65536 / (128 * minb))
template <int C>
__host__ __device__ constexpr int min_blocks() {
#ifdef MPB_MINB
    return MPB_MINB;
#else
    return C >= 12 ? 3 : 5;
#endif
}
// entries of the CT table scan kept in flight per step (x 4 chunks); measured best at L = 64
template <int C>
__host__ __device__ constexpr int select_unroll() {
#ifdef MPB_SEL_U
    return MPB_SEL_U;
#else
    return 4;
#endif
}
// chunks per entry loaded per step of the table scan (x select_unroll entries in flight): 32 loads
// in the tiled C = 16 kernels (+0.6 % over 16 at L = 64); 16 elsewhere (the C < 12 kernels have 102
// registers, the generic-NB ones spill with 32, the cooperative lanes split the groups)
template <int C, bool TILE>
__host__ __device__ constexpr int select_group() {
#ifdef MPB_SEL_G
    return MPB_SEL_G;
#else
    return C == 16 && TILE ? 8 : 4;
#endif
}
// dynamic shared memory: 2 buffers x 2 operand blocks x C/4 chunks of 16 bytes per thread (as
// per-thread cp.async chunks or as per-warp TMA tiles), then two mbarriers per warp
template <int C>
constexpr size_t stage_bytes() { return (size_t)kThreads * 4 * (C / 4) * 16 + (kThreads / 32) * 16; }

// TMA tensor maps of the exponentiation's arrays (2-D: 4*count words x chunk rows)
enum { TM_N = 1, TM_NP, TM_R2, TM_BASE, TM_G, TM_Y, TM_T, TM_Q, TM_S, TM_COUNT = 9 };
struct TmaMaps {
    CUtensorMap m[TM_COUNT];
};

MPB_DEVI size_t tid_global() { return (size_t)blockIdx.x * blockDim.x + threadIdx.x; }
// word-sliced accessor for operand k of an array with `count` operands
MPB_DEVI Arr arr(const uint32_t* base, size_t count, size_t k) {
    return Arr{reinterpret_cast<char*>(const_cast<uint32_t*>(base)) + k * 16, (uint32_t)(count * 16)};
}
// this thread's staging area in dynamic shared memory
MPB_DEVI Stage stage() {
    extern __shared__ __align__(128) uint4 smem_stage[];
    return Stage{(uint32_t)__cvta_generic_to_shared(smem_stage + threadIdx.x), (uint32_t)(blockDim.x * 16)};
}
// TMA staging: this warp's 2 x 2 tiles and its two mbarriers (initialised here); kw = the warp's
// first operand.  Every lane of the warp calls this (lane 0 of the active ones initialises).
template <int C>
MPB_DEVI Stage stage_tma(size_t kw, const TmaMaps* maps) {
    extern __shared__ __align__(128) uint4 smem_stage[];
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(smem_stage);
    const uint32_t warp = threadIdx.x >> 5;
    constexpr uint32_t tile = (C / 4) * 512u;
    Stage sg{};
    sg.tbase = base + warp * 4u * tile;
    sg.tbar = base + (uint32_t)kThreads * 4u * (C / 4) * 16u + warp * 16u;
    sg.kw = (uint32_t)kw;
    sg.amask = __activemask();
    sg.maps = maps;
    if ((threadIdx.x & 31u) == 0) {
        mbar_init(sg.tbar, 1);
        mbar_init(sg.tbar + 8, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp(sg.amask);
    return sg;
}
// word i of operand k (32-bit access)
MPB_DEVI uint32_t word_at(const uint32_t* base, size_t count, size_t k, int i) {
    return __ldg(base + ((size_t)(i >> 2) * count + k) * 4 + (i & 3));
}

// ------------------------------------------------------------ product kernels
// c = a*b (SQR: a^2): schoolbook through the engine, or LEVELS of block Karatsuba (mp_kara.cuh).
// ws: kara_scratch_blocks(nb, LEVELS) blocks per operand (word-sliced, stride count).
template <int C, bool SQR, int LEVELS>
__global__ void __launch_bounds__(kThreads) k_mp_mul(const uint32_t* __restrict__ a, const uint32_t* __restrict__ b,
                                                     uint32_t* __restrict__ c, size_t count, int nb, uint32_t* ws) {
    const size_t k = tid_global();
    if (k >= count) return;
    const Arr A = arr(a, count, k), B = arr(SQR ? a : b, count, k), Cc = arr(c, count, k);
    if (LEVELS == 0) {
        uint32_t orlo = 0, tl1 = 0;
        engine<C, true>(SQR ? PH_SQR : PH_MUL, nb, A, B, Cc, Cc, Cc, Cc, orlo, tl1, stage());
    } else {
        kmul<C, LEVELS>(SQR, nb, A, B, Cc, arr(ws, count, k), stage());
    }
}

// workspace for the mont kernels: T (2L) then Q (L), word-sliced with stride count.
// RM: 0 full, 1 truncated, 2 CIOS (mont_op_rm).
template <int C, int RM, bool SQR, int NBT>
__global__ void __launch_bounds__(kThreads) k_mont_mul(const uint32_t* __restrict__ a, const uint32_t* __restrict__ b,
                                                       const uint32_t* __restrict__ N, const uint32_t* __restrict__ NP,
                                                       uint32_t* __restrict__ c, size_t count, int nb_rt, uint32_t* ws) {
    const size_t k = tid_global();
    if (k >= count) return;
    const int nb = NBT ? NBT : nb_rt;
    const size_t L = (size_t)C * nb;
    const Arr T = arr(ws, count, k), Q = arr(ws + 2 * L * count, count, k);
    const Arr A = arr(a, count, k);
    mont_op_rm<C, RM, 0>(SQR ? MODE_SQR : MODE_MUL, nb, A, SQR ? A : arr(b, count, k), arr(N, count, k),
                         arr(NP, count, k), T, Q, arr(c, count, k), Q, stage());
}

template <int C, bool TRUNC>
__global__ void __launch_bounds__(kThreads) k_mont_redc(const uint32_t* __restrict__ Tin, const uint32_t* __restrict__ N,
                                                        const uint32_t* __restrict__ NP, uint32_t* __restrict__ c,
                                                        size_t count, int nb, uint32_t* ws) {
    const size_t k = tid_global();
    if (k >= count) return;
    const size_t L = (size_t)C * nb;
    const Arr T = arr(ws, count, k), Q = arr(ws + 2 * L * count, count, k);
    const Arr Ti = arr(Tin, count, k);
#pragma unroll 1
    for (int q = 0; q < (int)(2 * L / 4); q++) T.st(q, Ti.ld(q));
    mont_op<C, TRUNC>(MODE_REDC, nb, T, T, arr(N, count, k), arr(NP, count, k), T, Q, arr(c, count, k), stage());
}

#ifndef MPB_LOCKSTEP
#define MPB_LOCKSTEP 0
#endif
#ifndef MPB_TBL_PF
#define MPB_TBL_PF 0  // L2 bulk prefetch of the window table this many squarings before its scan (0: off)
#endif

// warp-tiled view of operand k in an array of nch chunks per operand (DESIGN 5.6)
MPB_DEVI ArrT tarr(uint32_t* base, int nch, size_t k) {
    char* p = reinterpret_cast<char*>(base) + (k >> 5) * ((size_t)nch * kTileSB) + (k & 31) * 16;
    return ArrT{p, kTileSB, 0u};
}

// Stand-alone REDC for the compile-time block counts (the hot sizes): the same engine
// instantiation as the exponentiation's REDC / MontMul reduction phases inside k_modexp -- the
// warp-tiled ArrT accessor, NB a compile-time constant -- so the adversarial REDC families
// (tests/adversarial.py; Theorem 2's exact carry correction) reach the code that ships.
// Workspace: T (2L) | Q (L) | N (L) | N' (L) | OUT (L), warp tiles over count rounded up to 32.
template <int C, bool TRUNC, int NBT>
__global__ void __launch_bounds__(kThreads, min_blocks<C>()) k_mont_redc_tiled(
    const uint32_t* __restrict__ Tin, const uint32_t* __restrict__ N, const uint32_t* __restrict__ NP,
    uint32_t* __restrict__ c, size_t count, uint32_t* ws) {
    const size_t k = tid_global();
    if (k >= count) return;
    constexpr int Q4 = C * NBT / 4;
    const size_t cpad = (count + 31) & ~(size_t)31;
    uint32_t* p = ws;
    auto take = [&](int nch) {
        const ArrT a = tarr(p, nch, k);
        p += cpad * (size_t)nch * 4;
        return a;
    };
    const ArrT T = take(2 * Q4), Q = take(Q4), Nt = take(Q4), NPt = take(Q4), O = take(Q4);
    const Arr Tk = arr(Tin, count, k), Nn = arr(N, count, k), NPn = arr(NP, count, k), On = arr(c, count, k);
#pragma unroll 1
    for (int q = 0; q < 2 * Q4; q++) T.st(q, Tk.ld(q));
#pragma unroll 1
    for (int q = 0; q < Q4; q++) {
        Nt.st(q, Nn.ld(q));
        NPt.st(q, NPn.ld(q));
    }
    mont_op<C, TRUNC, false, ArrT>(MODE_REDC, NBT, T, T, Nt, NPt, T, Q, O, stage());
#pragma unroll 1
    for (int q = 0; q < Q4; q++) On.st(q, O.ld(q));
}

// ------------------------------------------------------------------- modexp
// alg:8FWExp as one flat, public schedule of operations so that the kernel
// holds a single instance of the Montgomery engine:
//   op 0             G[0] = REDC(R^2) = R mod N               (Montgomery one)
//   op 1             G[1] = MontMul(base, R^2)
//   op e < 2^w       G[e] = MontMul(G[e-1], G[1])
//   op 2^w           Y = CTsel(G, top window)                  (windows LSB-aligned, A11)
//   then per window j = W-2 .. 0:  w x Y = MontSqr(Y),  S = CTsel(G, window j)
//                                  (P:L765-766),  Y = MontMul(Y, S)
//   last op          out = REDC(Y)
// workspace: TILE (compile-time block count, schoolbook products, cp.async staging: the hot
// sizes) -- warp-tiled arrays (ArrT, DESIGN 5.6) over cpad = count rounded up to 32 operands:
//   G (2^w * L) | Y (L) | T (2L) | Q (L) | S (L) | N (L) | N' (L)
// with N, N', base and R^2 copied in from the word-sliced inputs and the result copied out, so
// every engine array has the compile-time chunk stride.  Otherwise (generic block count,
// Karatsuba products, TMA tiles) -- word-sliced arrays, stride count: G | Y | T | Q | S |
// Karatsuba scratch (kara_scratch_blocks(nb, KLEV) blocks; KLEV = algo levels for the products).
// The whole exponentiation of operand k (of `count`, the arrays' stride).  LANES > 1: that many lanes
// per operand (mp_coop.cuh), role = lane mod LANES, mask = the active lanes of the warp.
#ifndef MPB_TILE
#define MPB_TILE 1
#endif
#ifndef MPB_ONEWAVE_C12
#define MPB_ONEWAVE_C12 1  // 4108 bits: the 4-CTA one-wave instance too (measured, DESIGN 5.3b)
#endif
// tiled for the compile-time block counts (the hot sizes); the generic-NB kernels run measurably
// slower with it (1536 / 2560 / 4108 bits: 5-20 %) and keep the word-sliced workspace
__host__ __device__ constexpr bool modexp_tiled(int KLEV, bool TMA, int NBT) {
    return MPB_TILE && KLEV == 0 && !TMA && NBT != 0;
}
template <int C, int RM, int NBT, int KLEV, int LANES, bool TMA = false>
MPB_DEVI void modexp_body(const uint32_t* N, const uint32_t* NP, const uint32_t* R2, const uint32_t* base,
                          const uint32_t* exp, uint32_t* out, size_t count, size_t k, int nb_rt, int bits, int w,
                          uint32_t* ws, uint32_t role, unsigned mask, const TmaMaps* maps = nullptr) {
    constexpr bool TILE = modexp_tiled(KLEV, TMA, NBT);
    constexpr bool COOP = LANES > 1;
    using A = std::conditional_t<TILE, ArrT, Arr>;
    const int nb = NBT ? NBT : nb_rt;  // compile-time block count for the hot sizes
    const int L = C * nb, Q4 = L / 4;
    const int nent = 1 << w;
    const Arr Nn = arr(N, count, k), NPn = arr(NP, count, k), R2n = arr(R2, count, k), Bn = arr(base, count, k);
    const Arr On = arr(out, count, k);
    Stage sg = stage();
    uint32_t tph = 0;  // TMA: mbarrier phase bits of the two tile buffers
    A Gt, Yt, Tt, Qt, St, Nt, NPt, R2t, Bt, KS;
    if constexpr (TILE) {
        const size_t cpad = (count + 31) & ~(size_t)31;
        uint32_t* p = ws;
        auto take = [&](int nch) {
            const ArrT a = tarr(p, nch, k);
            p += cpad * (size_t)nch * 4;
            return a;
        };
        Gt = take(nent * Q4);
        Yt = take(Q4);
        Tt = take(2 * Q4);
        Qt = take(Q4);
        St = take(Q4);
        Nt = take(Q4);
        NPt = take(Q4);
        KS = St;   // unused (schoolbook)
        Bt = Yt;   // base, then Y
        R2t = St;  // R^2, then S
        if (!COOP || role == 0) {
#pragma unroll 1
            for (int q = 0; q < Q4; q++) {
                Nt.st(q, Nn.ld(q));
                NPt.st(q, NPn.ld(q));
                Bt.st(q, Bn.ld(q));
                R2t.st(q, R2n.ld(q));
            }
        }
        if constexpr (COOP) __syncwarp(mask);
    } else {
        uint32_t* p = ws;
        Gt = arr(p, count, k);
        p += (size_t)nent * L * count;
        Yt = arr(p, count, k);
        p += (size_t)L * count;
        Tt = arr(p, count, k);
        p += (size_t)2 * L * count;
        Qt = arr(p, count, k);
        p += (size_t)L * count;
        St = arr(p, count, k);
        p += (size_t)L * count;
        KS = arr(p, count, k);  // Karatsuba scratch (KLEV > 0)
        Nt = Nn; NPt = NPn; R2t = R2n; Bt = Bn;
        if constexpr (TMA) {  // the same arrays, tagged with their tensor maps
            sg = stage_tma<C>(k - (threadIdx.x & 31u), maps);
            Gt.tm = TM_G; Yt.tm = TM_Y; Tt.tm = TM_T; Qt.tm = TM_Q; St.tm = TM_S;
            Nt.tm = TM_N; NPt.tm = TM_NP; R2t.tm = TM_R2; Bt.tm = TM_BASE;
        }
    }
    const A G = Gt, Y = Yt, T = Tt, Q = Qt;
    // the result: word-sliced output directly, or (TILE) S then copied out
    A Ofin;
    if constexpr (TILE) Ofin = St;
    else Ofin = On;

    const int nwin = (bits + w - 1) / w;
    const int per_win = w + 2;
    const int n_ops = nent + 1 + (nwin - 1) * per_win + 1;
#pragma unroll 1
    for (int op = 0; op < n_ops; op++) {
#if MPB_LOCKSTEP
        // keep the CTA's warps in step (the warp scheduler favours some warps; a CTA whose warps
        // drift apart ends at its slowest warp's time).  Public schedule: a barrier every
        // MPB_LOCKSTEP operations.
        if constexpr (!COOP) {
            if (op % MPB_LOCKSTEP == 0) __syncthreads();
        }
#endif
        int mode = MODE_MUL;
        bool select = false;
        int win = 0;
        A X = Yt, B = Yt, O = Yt;
        if (op == 0) {
            mode = MODE_REDC; X = R2t; O = Gt;
        } else if (op < nent) {
            X = op == 1 ? Bt : Gt.at((op - 1) * Q4);
            B = op == 1 ? R2t : Gt.at(Q4);
            O = Gt.at(op * Q4);
        } else if (op == nent) {
            select = true; win = nwin - 1; O = Yt;
        } else if (op == n_ops - 1) {
            mode = MODE_REDC; X = Yt; O = Ofin;
        } else {
            const int r = (op - nent - 1) % per_win;
            win = nwin - 2 - (op - nent - 1) / per_win;
            if (r < w) {
                mode = MODE_SQR;
            } else if (r == w) {
                select = true; O = St;
            } else {
                B = St;
            }
        }
        if (select) {
            // w bits of the exponent at public position win*w (may straddle two words)
            const int pos = win * w, wi = pos >> 5, off = pos & 31;
            uint32_t v = word_at(exp, count, k, wi) >> off;
            if (off + w > 32 && wi + 1 < L) v |= word_at(exp, count, k, wi + 1) << (32 - off);
            if constexpr (COOP) {  // the lanes of an operand scan alternate chunk groups of every entry
                ct_select<select_unroll<C>(), 4>(G, L, nent, v & ((1u << w) - 1u), O, (int)role, LANES);
                __syncwarp(mask);
            } else {
                ct_select<select_unroll<C>(), select_group<C, TILE>()>(G, L, nent, v & ((1u << w) - 1u), O);
            }
            continue;
        }
#if MPB_TBL_PF
        // L2 bulk prefetch of this warp's window table (one contiguous region of the warp tile:
        // nent * Q4 chunk rows x 512 bytes), issued MPB_TBL_PF squarings before the CT scan of a
        // window so its HBM reads spread over compute-bound squarings instead of arriving in one
        // burst.  Public addresses and a public schedule: always the whole table.
        if constexpr (TILE && !COOP) {
            if (op > nent && op < n_ops - 1 && (op - nent - 1) % per_win == w - MPB_TBL_PF) {
                const uint32_t lane = threadIdx.x & 31u;
                const char* tb = reinterpret_cast<const char*>(G.p) - lane * 16u;  // tile base
                const uint32_t tbytes = (uint32_t)nent * (uint32_t)Q4 * kTileSB;
#if MPB_TBL_PF_ONE  // one lane, one bulk prefetch of MPB_TBL_PF_ONE / 32 of the table
                if (lane == 0)
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(tb),
                                 "r"(tbytes / 32u * (uint32_t)MPB_TBL_PF_ONE)
                                 : "memory");
#else
                const uint32_t piece = tbytes / 32u;  // multiple of 16: nent * Q4 * 16
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(tb + lane * piece), "r"(piece)
                             : "memory");
#endif
            }
        }
#endif
        if (RM != 2 && mode == MODE_REDC) {  // T = X zero-extended to 2L limbs (CIOS: MontMul(X, 1))
            if (!COOP || role == 0) {  // one writer per operand
#pragma unroll 1
                for (int q = 0; q < Q4; q++) {
                    T.st(q, X.ld(q));
                    T.st(Q4 + q, make_uint4(0, 0, 0, 0));
                }
            }
            if constexpr (COOP) __syncwarp(mask);
        }
        if constexpr (COOP) {
            static_assert(RM != 2 && KLEV == 0, "cooperative operands: truncated or full REDC, schoolbook");
            mont_op_coop<C, RM == 1, LANES>(mode, nb, X, B, Nt, NPt, T, Q, O, sg, role, mask);
        } else if constexpr (TMA) {
            static_assert(RM != 2 && KLEV == 0, "TMA operand tiles: truncated or full REDC, schoolbook");
            mont_op<C, RM == 1, true>(mode, nb, X, B, Nt, NPt, Tt, Qt, O, sg, &tph);
        } else {
            mont_op_rm<C, RM, KLEV>(mode, nb, X, B, Nt, NPt, T, Q, O, KS, sg);
        }
    }
    if constexpr (TILE) {  // the result, S (warp tile) -> out (word-sliced)
        if constexpr (COOP) __syncwarp(mask);
        if (!COOP || role == 0) {
#pragma unroll 1
            for (int q = 0; q < Q4; q++) On.st(q, Ofin.ld(q));
        }
    }
}

#ifdef MPB_CTA_TIMES
static __device__ unsigned long long g_cta_t0[1 << 14], g_cta_t1[1 << 14];
static __device__ uint32_t g_cta_sm[1 << 14];
#endif
// One thread per operand: operands k_ofs .. k_ofs + n_run - 1 of a batch of `count`.
template <int C, int RM, int NBT, int KLEV, int MINB = min_blocks<C>()>
__global__ void __launch_bounds__(kThreads, MINB) k_modexp(
    const uint32_t* __restrict__ N, const uint32_t* __restrict__ NP, const uint32_t* __restrict__ R2,
    const uint32_t* __restrict__ base, const uint32_t* __restrict__ exp, uint32_t* __restrict__ out, size_t count,
    size_t k_ofs, size_t n_run, int nb_rt, int bits, int w, uint32_t* ws) {
    const size_t t = tid_global();
#ifdef MPB_CTA_TIMES  // DIAGNOSTIC builds only (tools/cta_times.cu): per-CTA start / end / SM
    if (threadIdx.x == 0) {
        unsigned long long t0;
        uint32_t sm;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
        g_cta_t0[blockIdx.x] = t0;
        g_cta_sm[blockIdx.x] = sm;
    }
#endif
    if (t >= n_run) return;
    modexp_body<C, RM, NBT, KLEV, 1>(N, NP, R2, base, exp, out, count, k_ofs + t, nb_rt, bits, w, ws, 0u,
                                     0xFFFFFFFFu);
#ifdef MPB_CTA_TIMES
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    atomicMax(&g_cta_t1[blockIdx.x], t1);
#endif
}

// One thread per operand, operand blocks loaded as per-warp TMA tiles (engine<.., TMA = true>).
template <int C, int RM, int NBT>
__global__ void __launch_bounds__(kThreads, min_blocks<C>()) k_modexp_tma(
    const uint32_t* __restrict__ N, const uint32_t* __restrict__ NP, const uint32_t* __restrict__ R2,
    const uint32_t* __restrict__ base, const uint32_t* __restrict__ exp, uint32_t* __restrict__ out, size_t count,
    size_t k_ofs, size_t n_run, int nb_rt, int bits, int w, uint32_t* ws, const __grid_constant__ TmaMaps maps) {
    const size_t t = tid_global();
    if (t >= n_run) return;
    modexp_body<C, RM, NBT, 0, 1, true>(N, NP, R2, base, exp, out, count, k_ofs + t, nb_rt, bits, w, ws, 0u,
                                        0xFFFFFFFFu, &maps);
}

// LANES (2, 4, 8) lanes per operand (mp_coop.cuh): >= 3072-bit batches too small to fill the
// GPU with one thread per operand, and the tail of a batch after its whole waves (Launch::modexp).
template <int C, int RM, int NBT, int LANES>
__global__ void __launch_bounds__(kThreads, min_blocks<C>()) k_modexp_coop(
    const uint32_t* __restrict__ N, const uint32_t* __restrict__ NP, const uint32_t* __restrict__ R2,
    const uint32_t* __restrict__ base, const uint32_t* __restrict__ exp, uint32_t* __restrict__ out, size_t count,
    size_t k_ofs, size_t n_run, int nb_rt, int bits, int w, uint32_t* ws) {
    static_assert(LANES == 2 || LANES == 4 || LANES == 8, "lanes per operand");
    const size_t t = tid_global();
    if (t / LANES >= n_run) return;
    // lanes of this warp that own an operand: groups are never split (32 % LANES == 0)
    const size_t wbase = t & ~(size_t)31;
    const size_t lanes = LANES * n_run - wbase;
    const unsigned mask = lanes >= 32 ? 0xFFFFFFFFu : ((1u << lanes) - 1u);
    modexp_body<C, RM, NBT, 0, LANES>(N, NP, R2, base, exp, out, count, k_ofs + t / LANES, nb_rt, bits, w, ws,
                                      (uint32_t)(t % LANES), mask);
}

// ------------------------------------------------------------------- setup
// N' = (-N)^-1 mod R and R^2 mod N (mp_setup.cuh); workspace 6L words per operand.
template <int C>
__global__ void __launch_bounds__(kThreads) k_setup(const uint32_t* __restrict__ N, uint32_t* __restrict__ NP,
                                                    uint32_t* __restrict__ R2, size_t count, int nb, int pub_bits,
                                                    uint32_t* ws) {
    const size_t k = tid_global();
    if (k >= count) return;
    const int L = C * nb;
    int nbits = pub_bits;  // the public bit length (CRT primes: bits/2, never read from the secret)
    if (nbits <= 0) {      // a public modulus: its bit length from its top limbs
        int top = L - 1;
        while (top > 0 && word_at(N, count, k, top) == 0) top--;
        nbits = 32 * top + (32 - __clz(word_at(N, count, k, top)));
    }
    setup_one<C>(nb, arr(N, count, k), arr(NP, count, k), arr(R2, count, k), arr(ws, count, k), stage(),
                 word_at(N, count, k, 0), nbits);
}

// ------------------------------------------------------------------ CRT-RSA
// Batched CRT-RSA private-key operation (the paper's motivating use; SURVEY
// 8(f) f4): three launches around the half-size exponentiation.  Arrays of n2 = 2*count operands
// hold the p-items at 0..count-1 and the q-items at count..2count-1 (word-sliced, stride n2).
//   k_crt_reduce    B_j = c mod P_j = MontMul(REDC(c), R^2 mod P_j)   (REDC needs c < P_j * R)
//   (modexp)        M_j = B_j^E_j mod P_j                              (mont_batch_modexp_ct)
//   k_crt_recombine m = m_q + q * (qinv * (m_p - m_q) mod p)           (Garner)
// Every step is a fixed sequence of block operations and masked selects (constant time).
template <int C>
__global__ void __launch_bounds__(kThreads) k_crt_reduce(const uint32_t* __restrict__ c, int Lc,
                                                         const uint32_t* __restrict__ PQ, const uint32_t* __restrict__ NPQ,
                                                         const uint32_t* __restrict__ R2Q, uint32_t* __restrict__ B,
                                                         size_t count, int nb, uint32_t* ws) {
    const size_t n2 = 2 * count;
    const size_t j = tid_global();
    if (j >= n2) return;
    const size_t k = j < count ? j : j - count;
    const int Lh = C * nb;
    const Arr T = arr(ws, n2, j), Q = arr(ws + (size_t)2 * Lh * n2, n2, j), X = arr(ws + (size_t)3 * Lh * n2, n2, j);
    const Arr Cc = arr(c, count, k);
#pragma unroll 1
    for (int q = 0; q < 2 * Lh / 4; q++) T.st(q, q < Lc / 4 ? Cc.ld(q) : make_uint4(0, 0, 0, 0));
    const Arr N = arr(PQ, n2, j), NP = arr(NPQ, n2, j);
    const Stage sg = stage();
    mont_op<C, true>(MODE_REDC, nb, T, T, N, NP, T, Q, X, sg);                    // X = c R^-1 mod P_j
    mont_op<C, true>(MODE_MUL, nb, X, arr(R2Q, n2, j), N, NP, T, Q, arr(B, n2, j), sg);  // B = c mod P_j
}

template <int C>
__global__ void __launch_bounds__(kThreads) k_crt_recombine(const uint32_t* __restrict__ M, const uint32_t* __restrict__ PQ,
                                                            const uint32_t* __restrict__ NPQ, const uint32_t* __restrict__ R2Q,
                                                            const uint32_t* __restrict__ qinv, uint32_t* __restrict__ out,
                                                            int Lo, size_t count, int nb, uint32_t* ws) {
    const size_t k = tid_global();
    if (k >= count) return;
    const size_t n2 = 2 * count;
    const int Lh = C * nb;
    const Arr mp = arr(M, n2, k), mq = arr(M, n2, count + k), P = arr(PQ, n2, k), Qm = arr(PQ, n2, count + k);
    const Arr NPp = arr(NPQ, n2, k), R2p = arr(R2Q, n2, k), QI = arr(qinv, count, k);
    uint32_t* w = ws;
    const Arr T = arr(w, count, k);
    w += (size_t)2 * Lh * count;
    const Arr Qs = arr(w, count, k);
    w += (size_t)Lh * count;
    const Arr X = arr(w, count, k);
    w += (size_t)Lh * count;
    const Arr H = arr(w, count, k);
    w += (size_t)Lh * count;
    const Arr PR = arr(w, count, k);  // 2Lh limbs
    const Stage sg = stage();
    // X = m_q - p; then X = borrow ? m_q : X   (m_q < q < 2p, so m_q mod p needs one subtraction)
    uint32_t bw = 0;
#pragma unroll 1
    for (int b = 0; b < nb; b++) {
        uint32_t u[C], v[C];
        ldb<C>(mq, b, u);
        ldb<C>(P, b, v);
        bc_restore(bw);
#pragma unroll
        for (int i = 0; i < C; i++) sub_next(u[i], v[i]);
        bw = bc_save();
        stb<C>(X, b, u);
    }
    {
        const uint32_t keep = 0u - bw;  // all ones: m_q < p, keep m_q
#pragma unroll 1
        for (int b = 0; b < nb; b++) {
            uint32_t u[C], v[C];
            ldb<C>(X, b, u);
            ldb<C>(mq, b, v);
#pragma unroll
            for (int i = 0; i < C; i++) u[i] = (v[i] & keep) | (u[i] & ~keep);
            stb<C>(X, b, u);
        }
    }
    // X = m_p - X; if that borrowed, X += p
    bw = 0;
#pragma unroll 1
    for (int b = 0; b < nb; b++) {
        uint32_t u[C], v[C];
        ldb<C>(mp, b, u);
        ldb<C>(X, b, v);
        bc_restore(bw);
#pragma unroll
        for (int i = 0; i < C; i++) sub_next(u[i], v[i]);
        bw = bc_save();
        stb<C>(X, b, u);
    }
    {
        const uint32_t addp = 0u - bw;
        uint32_t cy = 0;
#pragma unroll 1
        for (int b = 0; b < nb; b++) {
            uint32_t u[C], v[C];
            ldb<C>(X, b, u);
            ldb<C>(P, b, v);
            cc_restore(cy);
#pragma unroll
            for (int i = 0; i < C; i++) add_next(u[i], v[i] & addp);
            cy = cc_save();
            stb<C>(X, b, u);
        }
    }
    mont_op<C, true>(MODE_MUL, nb, X, QI, P, NPp, T, Qs, H, sg);   // H = d qinv R^-1 mod p
    mont_op<C, true>(MODE_MUL, nb, H, R2p, P, NPp, T, Qs, X, sg);  // X = h = d qinv mod p
    {
        uint32_t orlo = 0, tl1 = 0;
        engine<C, true>(PH_MUL, nb, X, Qm, PR, PR, PR, PR, orlo, tl1, sg);  // PR = h q (2Lh limbs)
    }
    // out = PR + m_q  (< p q: the top 2Lh - Lo limbs are zero)
    const Arr O = arr(out, count, k);
    uint32_t cy = 0;
#pragma unroll 1
    for (int b = 0; b < 2 * nb; b++) {
        uint32_t u[C], v[C];
        ldb<C>(PR, b, u);
        if (b < nb) {
            ldb<C>(mq, b, v);
        } else {
#pragma unroll
            for (int i = 0; i < C; i++) v[i] = 0;
        }
        cc_restore(cy);
#pragma unroll
        for (int i = 0; i < C; i++) add_next(u[i], v[i]);
        cy = cc_save();
#pragma unroll
        for (int q = 0; q < C / 4; q++)
            if ((b * C) / 4 + q < Lo / 4) O.st((b * C) / 4 + q, make_uint4(u[4 * q], u[4 * q + 1], u[4 * q + 2], u[4 * q + 3]));
    }
}

// ---------------------------------------------------------------- launchers
// stage buffers above the 48 KB default need the per-kernel opt-in (only with MPB_THREADS > 128 builds)
template <class K>
inline void smem_optin(K* k, size_t sm) {
    if (sm > 48 * 1024) cudaFuncSetAttribute((const void*)k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
}
template <int C>
void Launch<C>::setup(const uint32_t* N, uint32_t* NP, uint32_t* R2, size_t count, int nb, int pub_bits,
                      uint32_t* ws, cudaStream_t s) {
    smem_optin(k_setup<C>, stage_bytes<C>());
    k_setup<C><<<(unsigned)((count + kThreads - 1) / kThreads), kThreads, stage_bytes<C>(), s>>>(N, NP, R2, count, nb,
                                                                                               pub_bits, ws);
}

inline unsigned grid_for(size_t n) { return (unsigned)((n + kThreads - 1) / kThreads); }

template <int C>
void Launch<C>::mp_mul(const uint32_t* a, const uint32_t* b, uint32_t* c, size_t count, int nb, bool sqr, int levels,
                       uint32_t* ws, cudaStream_t s) {
    const unsigned g = grid_for(count);
    const size_t sm = stage_bytes<C>();
    if (sqr) {
        if (levels >= 2) k_mp_mul<C, true, 2><<<g, kThreads, sm, s>>>(a, a, c, count, nb, ws);
        else if (levels == 1) k_mp_mul<C, true, 1><<<g, kThreads, sm, s>>>(a, a, c, count, nb, ws);
        else k_mp_mul<C, true, 0><<<g, kThreads, sm, s>>>(a, a, c, count, nb, ws);
    } else {
        if (levels >= 2) k_mp_mul<C, false, 2><<<g, kThreads, sm, s>>>(a, b, c, count, nb, ws);
        else if (levels == 1) k_mp_mul<C, false, 1><<<g, kThreads, sm, s>>>(a, b, c, count, nb, ws);
        else k_mp_mul<C, false, 0><<<g, kThreads, sm, s>>>(a, b, c, count, nb, ws);
    }
}
// compile-time block counts of the hot sizes (1024/2048/3072/4096 bits at C = 16; 4108 at C = 12)
template <int C, typename F>
void with_nb(int nb, F&& f) {
    if constexpr (C == 16) {
        switch (nb) {
            case 2: return f(std::integral_constant<int, 2>{});
            case 4: return f(std::integral_constant<int, 4>{});
            case 6: return f(std::integral_constant<int, 6>{});
            case 8: return f(std::integral_constant<int, 8>{});
            default: break;
        }
    } else if constexpr (C == 12) {
        if (nb == 11) return f(std::integral_constant<int, 11>{});
    } else if constexpr (C == 8) {
        switch (nb) {
            case 4: return f(std::integral_constant<int, 4>{});  // 1024 bits with MPB_BLOCK=8 (tuning)
            case 8: return f(std::integral_constant<int, 8>{});
            case 16: return f(std::integral_constant<int, 16>{});
            default: break;
        }
    }
    f(std::integral_constant<int, 0>{});
}

template <int C>
void Launch<C>::mont_mul(const uint32_t* a, const uint32_t* b, const uint32_t* N, const uint32_t* NP, uint32_t* c,
                         size_t count, int nb, int redc, bool sqr, uint32_t* ws, cudaStream_t s) {
    const unsigned g = grid_for(count);
    const size_t sm = stage_bytes<C>();
    with_nb<C>(nb, [&](auto NBc) {
        constexpr int NBT = decltype(NBc)::value;
        auto go = [&](auto RMc) {
            constexpr int RM = decltype(RMc)::value;
            if (sqr) k_mont_mul<C, RM, true, NBT><<<g, kThreads, sm, s>>>(a, a, N, NP, c, count, nb, ws);
            else k_mont_mul<C, RM, false, NBT><<<g, kThreads, sm, s>>>(a, b, N, NP, c, count, nb, ws);
        };
        if (redc == 2) go(std::integral_constant<int, 2>{});
        else if (redc == 1) go(std::integral_constant<int, 1>{});
        else go(std::integral_constant<int, 0>{});
    });
}
template <int C>
void Launch<C>::crt_reduce(const uint32_t* c, int Lc, const uint32_t* PQ, const uint32_t* NPQ, const uint32_t* R2Q,
                           uint32_t* B, size_t count, int nb, uint32_t* ws, cudaStream_t s) {
    k_crt_reduce<C><<<grid_for(2 * count), kThreads, stage_bytes<C>(), s>>>(c, Lc, PQ, NPQ, R2Q, B, count, nb, ws);
}
template <int C>
void Launch<C>::crt_recombine(const uint32_t* M, const uint32_t* PQ, const uint32_t* NPQ, const uint32_t* R2Q,
                              const uint32_t* qinv, uint32_t* out, int Lo, size_t count, int nb, uint32_t* ws,
                              cudaStream_t s) {
    k_crt_recombine<C><<<grid_for(count), kThreads, stage_bytes<C>(), s>>>(M, PQ, NPQ, R2Q, qinv, out, Lo, count, nb,
                                                                          ws);
}
template <int C>
void Launch<C>::mont_redc(const uint32_t* T, const uint32_t* N, const uint32_t* NP, uint32_t* c, size_t count, int nb,
                          bool trunc, uint32_t* ws, cudaStream_t s) {
    const size_t sm = stage_bytes<C>();
    with_nb<C>(nb, [&](auto NBc) {
        constexpr int NBT = decltype(NBc)::value;
        if constexpr (NBT != 0 && MPB_TILE) {  // the exponentiation's tiled, compile-time-NB engine
            if (trunc) k_mont_redc_tiled<C, true, NBT><<<grid_for(count), kThreads, sm, s>>>(T, N, NP, c, count, ws);
            else k_mont_redc_tiled<C, false, NBT><<<grid_for(count), kThreads, sm, s>>>(T, N, NP, c, count, ws);
        } else {
            if (trunc) k_mont_redc<C, true><<<grid_for(count), kThreads, sm, s>>>(T, N, NP, c, count, nb, ws);
            else k_mont_redc<C, false><<<grid_for(count), kThreads, sm, s>>>(T, N, NP, c, count, nb, ws);
        }
    });
}
// One-thread or cooperative kernel (small >= 3072-bit batches); MPB_COOP=0 / 1 forces never /
// always (tuning and tests).
// TMA tensor map of a word-sliced array: 2-D, dim 0 = 4*count uint32 words (all operands' chunk
// rows), dim 1 = rows (chunks per operand), row stride count*16 bytes; box = 128 words (one warp's
// 32 operands) x box_rows (one block); out-of-range operands read as zero.
inline bool encode_tile_map(CUtensorMap* m, const uint32_t* base, size_t count, int rows, int box_rows) {
    using Fn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                            const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                            CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static Fn fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return (Fn) nullptr;
        return (Fn)f;
    }();
    if (!fn) return false;
    const cuuint64_t dims[2] = {(cuuint64_t)count * 4, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)count * 16};
    const cuuint32_t box[2] = {128, (cuuint32_t)box_rows};
    const cuuint32_t estr[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<uint32_t*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// MPB_TMA=1 selects the TMA operand tiles (tests and measurements)
inline int tma_policy() {
    static int v = [] {
        const char* e = getenv("MPB_TMA");
        return e ? atoi(e) : -1;
    }();
    return v;
}
// MPB_ONEWAVE=0: no one-CTA-per-SM instances for one-wave batches (tests and A/B measurements)
inline int onewave_policy() {
    static int v = [] {
        const char* e = getenv("MPB_ONEWAVE");
        return e ? atoi(e) : 1;
    }();
    return v;
}
// MPB_COOP: unset = the measured policy; 0 = always one thread per operand; 1 or 2 / 4 / 8 =
// always 2 / 2 / 4 / 8 lanes per operand (tests and tuning)
inline int coop_policy() {
    static int v = [] {
        const char* e = getenv("MPB_COOP");
        return e ? atoi(e) : -1;
    }();
    return v;
}
// MPB_COOP_TAIL = 2 / 4 / 8: lanes per operand of an (opt-in) cooperative tail after the whole
// waves of a large batch (unset = no cooperative tail, the measured policy)
inline int coop_tail_lanes() {
    static int v = [] {
        const char* e = getenv("MPB_COOP_TAIL");
        return e ? atoi(e) : -1;
    }();
    return v;
}
template <int C>
void Launch<C>::modexp(const uint32_t* N, const uint32_t* NP, const uint32_t* R2, const uint32_t* base,
                       const uint32_t* exp, uint32_t* out, size_t count, int nb, int bits, int window, int redc,
                       int levels, uint32_t* ws, cudaStream_t s) {
    const size_t sm = stage_bytes<C>();
    with_nb<C>(nb, [&](auto NBc) {
        constexpr int NBT = decltype(NBc)::value;
        auto single = [&](size_t k0, size_t n) {
            if (n == 0) return;
            if constexpr ((C == 16 && (NBT == 2 || NBT == 4 || NBT == 6 || NBT == 8)) || (C == 12 && NBT == 11)) {
                // A batch that fits one wave: one CTA of <= 384 (<= 448 at 4096 bits) threads per SM,
                // the batch spread evenly over the SMs (inst_W384.cu / inst_W448.cu).
                // Measured: 2^16 x 4096 bits 49.4 K vs 46.1 K/s (4 x 128-thread CTAs per SM),
                // 56 832 x 2048 bits 398 K vs 365 K/s (3 x 128).
                if (levels == 0 && onewave_policy() != 0) {
                    int dev = 0, sms = 148;
                    if (cudaGetDevice(&dev) == cudaSuccess)
                        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
                    const size_t per = (n + (size_t)sms - 1) / (size_t)sms;
                    const unsigned thr = (unsigned)((per + 31) / 32 * 32);
                    const unsigned gw = (unsigned)((n + thr - 1) / thr);
                    if (thr <= 384 && ::mpb_modexp_w384(N, NP, R2, base, exp, out, count, k0, n, C, nb, bits,
                                                        window, redc, ws, gw, thr, s))
                        return;
                    if ((NBT == 8 || NBT == 11) && thr <= 448 &&
                        ::mpb_modexp_w448(N, NP, R2, base, exp, out, count, k0, n, C, nb, bits, window, redc, ws,
                                          gw, thr, s))
                        return;
                }
            }
            const unsigned g = grid_for(n);
            if (redc == 2) {  // CIOS: schoolbook rows only
                k_modexp<C, 2, NBT, 0><<<g, kThreads, sm, s>>>(N, NP, R2, base, exp, out, count, k0, n, nb, bits,
                                                              window, ws);
                return;
            }
            auto go = [&](auto KL) {
                constexpr int KLEV = decltype(KL)::value;
                if (redc == 1) {
                    smem_optin(k_modexp<C, 1, NBT, KLEV>, sm);
                    k_modexp<C, 1, NBT, KLEV><<<g, kThreads, sm, s>>>(N, NP, R2, base, exp, out, count, k0, n, nb,
                                                                     bits, window, ws);
                } else {
                    smem_optin(k_modexp<C, 0, NBT, KLEV>, sm);
                    k_modexp<C, 0, NBT, KLEV><<<g, kThreads, sm, s>>>(N, NP, R2, base, exp, out, count, k0, n, nb,
                                                                     bits, window, ws);
                }
            };
            // Karatsuba product phases are compiled for the large shapes only (f1); elsewhere schoolbook
            if constexpr (NBT == 0 || NBT == 8 || NBT == 11) {
                if (levels >= 2) return go(std::integral_constant<int, 2>{});
                if (levels == 1) return go(std::integral_constant<int, 1>{});
            }
            if constexpr ((C == 16 && NBT == 8) || (C == 12 && NBT == 11 && MPB_ONEWAVE_C12)) {
                // 4096 bits: a batch that needs two waves at 3 CTAs per SM but fits ONE wave at 4
                // (128 registers, a few spills) runs the 4-CTA instance -- config 4 (2^16 operands,
                // 1.15 waves at 3 CTAs): 46.1 K vs 44.3 K/s measured; many-wave batches keep 3 CTAs
                // (the 4-CTA instance is slower per operand).  DESIGN.md 5.3b.
                int dev = 0, sms = 148;
                if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
                const size_t w3 = (size_t)sms * kThreads * min_blocks<C>(), w4 = (size_t)sms * kThreads * 4;
                if (n > w3 && n <= w4 && min_blocks<C>() < 4 && redc != 2) {
                    if (redc == 1)
                        k_modexp<C, 1, NBT, 0, 4><<<g, kThreads, sm, s>>>(N, NP, R2, base, exp, out, count, k0, n, nb,
                                                                          bits, window, ws);
                    else
                        k_modexp<C, 0, NBT, 0, 4><<<g, kThreads, sm, s>>>(N, NP, R2, base, exp, out, count, k0, n, nb,
                                                                          bits, window, ws);
                    return;
                }
            }
            go(std::integral_constant<int, 0>{});
        };
        auto coop = [&](size_t k0, size_t n, int lanes) {
            if (n == 0) return;
            const unsigned g = grid_for((size_t)lanes * n);
            auto go = [&](auto LC) {
                constexpr int LN = decltype(LC)::value;
                if (redc == 1)
                    k_modexp_coop<C, 1, NBT, LN><<<g, kThreads, sm, s>>>(N, NP, R2, base, exp, out, count, k0, n, nb,
                                                                        bits, window, ws);
                else
                    k_modexp_coop<C, 0, NBT, LN><<<g, kThreads, sm, s>>>(N, NP, R2, base, exp, out, count, k0, n, nb,
                                                                        bits, window, ws);
            };
            if (lanes >= 8) go(std::integral_constant<int, 8>{});
            else if (lanes == 4) go(std::integral_constant<int, 4>{});
            else go(std::integral_constant<int, 2>{});
        };
        const int pol = coop_policy();
        if (redc != 2 && levels == 0 && pol <= 0 && tma_policy() == 1) {
            // opt-in (MPB_TMA=1): one thread per operand with per-warp TMA operand tiles -- correct,
            // but 10 % slower than the cp.async.ca stage, whose operand blocks re-hit in L1
            // (DESIGN.md 5.3); falls back when the tensor maps cannot be encoded
            TmaMaps maps;
            const int L = C * nb;
            const uint32_t* arrs[TM_COUNT] = {N, NP, R2, base, ws, ws + (size_t)(1 << window) * L * count,
                                              ws + (size_t)((1 << window) + 1) * L * count,
                                              ws + (size_t)((1 << window) + 3) * L * count,
                                              ws + (size_t)((1 << window) + 4) * L * count};
            const int rows[TM_COUNT] = {L / 4, L / 4, L / 4, L / 4, (1 << window) * L / 4, L / 4, 2 * L / 4, L / 4,
                                        L / 4};
            bool ok = true;
            for (int i = 0; i < TM_COUNT && ok; i++) ok = encode_tile_map(&maps.m[i], arrs[i], count, rows[i], C / 4);
            if (ok) {
                const unsigned g = grid_for(count);
                if (redc == 1)
                    k_modexp_tma<C, 1, NBT><<<g, kThreads, sm, s>>>(N, NP, R2, base, exp, out, count, 0, count, nb,
                                                                   bits, window, ws, maps);
                else
                    k_modexp_tma<C, 0, NBT><<<g, kThreads, sm, s>>>(N, NP, R2, base, exp, out, count, 0, count, nb,
                                                                   bits, window, ws, maps);
                return;
            }
        }
        if (redc == 2 || levels > 0 || pol == 0) return single(0, count);
        if (pol == 1 || pol == 2 || pol == 4 || pol == 8) return coop(0, count, pol == 1 ? 2 : pol);  // forced
        // Measured: cooperative lanes pay for >= 3072-bit operands at low occupancy;
        // at 1024/2048 bits they do not.
        if (C * nb < 96) return single(0, count);
        int dev = 0, sms = 148;
        if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const size_t wave = (size_t)sms * kThreads * min_blocks<C>();  // one-thread operands resident at once
        const int tl = coop_tail_lanes();
        // Small batches: as many lanes per operand as keep the cooperative launch within one
        // (8 lanes) or two (4 lanes) CTAs per SM.  Measured at 4096 bits: 2 048
        // operands 3.5 / 4.1 / 5.5 / 6.0 K/s with 1 / 2 / 4 / 8 lanes; 8 192 operands 13.5 / 15.9 /
        // 16.9 / 8.9 K/s (8 lanes there would need 3.5 CTAs per SM).
        if (8 * count <= (size_t)sms * kThreads) return coop(0, count, 8);
        if (4 * count <= (size_t)2 * sms * kThreads) return coop(0, count, 4);
        if (2 * count <= (size_t)sms * kThreads) return coop(0, count, 2);
        // (opt-in, MPB_COOP_TAIL = 2 / 4 / 8) whole waves one thread per operand, then the tail with
        // several lanes per operand.  Measured at 2^16 x 4096 bits: 41.9 K/s without,
        // 39.6 / 40.3 / 31.8 K/s with a 2 / 4 / 8-lane tail -- the one-thread tail, which starts as the
        // last whole wave drains and runs a few warps per SM, is faster; so it stays the default.
        const size_t full = count / wave * wave, rest = count - full;
        if (tl <= 1 || full == 0 || rest == 0) return single(0, count);
        single(0, full);
        coop(full, rest, tl);
    });
}

}  // namespace mpb
