// inst_R32.cu -- the register-resident CIOS exponentiation for 1024-bit operands (mp_reg.cuh).
//
// mont_batch_modexp_ct with redc = MPB_REDC_CIOS and L = 32 limbs (897..1024 bits) runs this kernel:
// alg:8FWExp on alg:8BlockMontRed MontMuls whose accumulator, multiplicand
// and modulus live in registers (mp_reg.cuh); the a operand of each MontMul is streamed from a
// per-thread shared-memory slot (one LDS per row), the 2^w-entry table lives in the warp-tiled
// workspace and is read by the masked full scan.  One flat public schedule with a single
// MontMul call site, as k_modexp: the kernel is one straight-line MontMul plus control.
#include "kernels.cuh"
#include "mp_reg.cuh"

#ifndef MPB_REG_MINB
#define MPB_REG_MINB 3
#endif

namespace mpb {

#ifndef MPB_SCAN_U
#define MPB_SCAN_U 1  // entries per step
#endif
#ifndef MPB_SCAN_G
#define MPB_SCAN_G 8  // chunks (uint4) per group
#endif
#ifndef MPB_SCAN_LD
#define MPB_SCAN_LD 0  // 0 evict-first (__ldcs), 1 default caching (__ldg)
#endif

// The CT masked full-table scan of a warp-tiled table of nent entries x Q4 chunks into a
// per-thread shared-memory slot (word q at slot[q * blockDim]): every entry is read in full with a
// mask, no address or branch depends on idx.  U entries x GR chunks in flight per step.
template <int Q4, int U = MPB_SCAN_U, int GR = (MPB_SCAN_G < Q4 ? MPB_SCAN_G : Q4)>
MPB_DEVI void scan_to_slot(const ArrT& G, int nent, uint32_t idx, uint32_t* slot) {
    static_assert(Q4 % GR == 0, "whole chunk groups");
#pragma unroll 1
    for (int g0 = 0; g0 < Q4; g0 += GR) {
        uint4 acc[GR];
#pragma unroll
        for (int q = 0; q < GR; q++) acc[q] = make_uint4(0, 0, 0, 0);
#pragma unroll 1
        for (int e0 = 0; e0 < nent; e0 += U) {
            uint4 v[U][GR];
#pragma unroll
            for (int u = 0; u < U; u++)
#pragma unroll
                for (int q = 0; q < GR; q++) {
                    const int c = (e0 + u) * Q4 + g0 + q;
#if MPB_SCAN_LD == 1
                    v[u][q] = e0 + u < nent ? __ldg(G.addr(c)) : make_uint4(0, 0, 0, 0);
#else
                    v[u][q] = e0 + u < nent ? G.ld_stream(c) : make_uint4(0, 0, 0, 0);
#endif
                }
#pragma unroll
            for (int u = 0; u < U; u++) {
                const uint32_t x = (uint32_t)(e0 + u) ^ idx;
                const uint32_t m = 0u - ((x - 1u) >> 31);  // all ones iff e == idx
#pragma unroll
                for (int q = 0; q < GR; q++) {
                    acc[q].x |= v[u][q].x & m;
                    acc[q].y |= v[u][q].y & m;
                    acc[q].z |= v[u][q].z & m;
                    acc[q].w |= v[u][q].w & m;
                }
            }
        }
#pragma unroll
        for (int q = 0; q < GR; q++) {
            const int w0 = 4 * (g0 + q);
            slot[(w0) * kThreads] = acc[q].x;
            slot[(w0 + 1) * kThreads] = acc[q].y;
            slot[(w0 + 2) * kThreads] = acc[q].z;
            slot[(w0 + 3) * kThreads] = acc[q].w;
        }
    }
}

template <int L>
__global__ void __launch_bounds__(kThreads, MPB_REG_MINB) k_modexp_reg(
    const uint32_t* __restrict__ N, const uint32_t* __restrict__ NP, const uint32_t* __restrict__ R2,
    const uint32_t* __restrict__ base, const uint32_t* __restrict__ exp, uint32_t* __restrict__ out, size_t count,
    int bits, int w, uint32_t* ws, int sqr_rows) {
    const size_t k = tid_global();
    if (k >= count) return;
    constexpr int Q4 = L / 4;
    const int nent = 1 << w;
    extern __shared__ __align__(16) uint32_t smem_a[];  // word q of this thread at q * blockDim + tid
    uint32_t* const sa = smem_a + threadIdx.x;
    const ArrT G = tarr(ws, nent * Q4, k);
    const Arr Nn = arr(N, count, k), R2n = arr(R2, count, k), Bn = arr(base, count, k), On = arr(out, count, k);
    uint32_t n[L];
    ldb<L>(Nn, 0, n);
    const uint32_t n0p = word_at(NP, count, k, 0);  // n0' = N'[0] (reading A10)
    auto aw = [&](int i) { return sa[i * kThreads]; };
    auto a_from_regs = [&](const uint32_t (&x)[L]) {
#pragma unroll
        for (int q = 0; q < L; q++) sa[q * kThreads] = x[q];
    };
    auto a_from_mem = [&](const auto& A) {
#pragma unroll
        for (int q = 0; q < Q4; q++) {
            const uint4 v = A.ld(q);
            sa[(4 * q) * kThreads] = v.x;
            sa[(4 * q + 1) * kThreads] = v.y;
            sa[(4 * q + 2) * kThreads] = v.z;
            sa[(4 * q + 3) * kThreads] = v.w;
        }
    };
    const int nwin = (bits + w - 1) / w;
    auto window = [&](int win) {
        const int pos = win * w, wi = pos >> 5, off = pos & 31;
        uint32_t v = word_at(exp, count, k, wi) >> off;
        if (off + w > 32 && wi + 1 < L) v |= word_at(exp, count, k, wi + 1) << (32 - off);
        return v & ((1u << w) - 1u);
    };
    // CT masked full-table scan into the a slot
    auto select = [&](uint32_t idx) { scan_to_slot<Q4>(G, nent, idx, sa); };
    // Flat schedule (public): op 0 G[0] = MontMul(R2, 1) (Montgomery one), op 1 G[1] = MontMul(base, R2),
    // op e < 2^w G[e] = MontMul(G[e-1], G[1]); then Y = G[top window]; per window w squarings, select,
    // one multiplication; last op out = MontMul(Y, 1).
    uint32_t y[L];
#pragma unroll
    for (int q = 0; q < L; q++) y[q] = 0;
    const int per_win = w + 1;
    const int n_ops = nent + (nwin - 1) * per_win + 1;
#pragma unroll 1
    for (int op = 0; op < n_ops; op++) {
        uint32_t b[L + 1];  // the multiplicand (words 0 .. L-1) or, for a squaring, D = 2Y (L+1 words)
        uint32_t(&bl)[L] = *reinterpret_cast<uint32_t(*)[L]>(b);
        int store_e = -1;
        bool b_one = false, b_y = true, sqr = false;
        if (op < nent) {
            store_e = op;
            if (op == 0) {
                a_from_mem(R2n);
                b_one = true;
            } else if (op == 1) {
                a_from_mem(Bn);
                ldb<L>(R2n, 0, bl);
                b_y = false;
            } else {
                a_from_mem(G.at((op - 1) * Q4));
                ldb<L>(G.at(Q4), 0, bl);
                b_y = false;
            }
        } else if (op == n_ops - 1) {
            a_from_regs(y);
            b_one = true;
        } else {
            const int r = (op - nent) % per_win, win = nwin - 2 - (op - nent) / per_win;
            if (r < w) {  // squaring: a = Y, squaring rows over B = 2Y
                a_from_regs(y);
                sqr = sqr_rows != 0;
            } else {
                select(window(win));  // multiplication by the selected entry
            }
        }
        if (b_one) {
#pragma unroll
            for (int q = 0; q < L; q++) b[q] = q == 0 ? 1u : 0u;
        } else if (sqr) {
            reg::double_words<L>(y, b);
        } else if (b_y) {
#pragma unroll
            for (int q = 0; q < L; q++) b[q] = y[q];
        }
        if (sqr) reg::montsqr<L>(aw, b, n, n0p, y);  // two call sites: MontSqr rows and MontMul rows
        else reg::montmul<L>(aw, bl, n, n0p, y);
        if (store_e >= 0) stb<L>(G.at(store_e * Q4), 0, y);
        if (op == nent - 1) {  // after the table: Y = G[top window]
            select(window(nwin - 1));
#pragma unroll
            for (int q = 0; q < L; q++) y[q] = aw(q);
        }
    }
    stb<L>(On, 0, y);
}

// Stand-alone CIOS MontMul / MontSqr at L = 32 (mont_batch_mul / mont_batch_sqr, redc = CIOS):
// c = a b 2^(-1024) mod N canonical, the register-resident row loop of mp_reg.cuh.
template <int L>
__global__ void __launch_bounds__(kThreads, MPB_REG_MINB) k_mont_mul_reg(
    const uint32_t* __restrict__ a, const uint32_t* __restrict__ b, const uint32_t* __restrict__ N,
    const uint32_t* __restrict__ NP, uint32_t* __restrict__ c, size_t count, bool sqr) {
    const size_t k = tid_global();
    if (k >= count) return;
    extern __shared__ __align__(16) uint32_t smem_a[];
    uint32_t* const sa = smem_a + threadIdx.x;
    const Arr A = arr(a, count, k);
#pragma unroll
    for (int q = 0; q < L / 4; q++) {
        const uint4 v = A.ld(q);
        sa[(4 * q) * kThreads] = v.x;
        sa[(4 * q + 1) * kThreads] = v.y;
        sa[(4 * q + 2) * kThreads] = v.z;
        sa[(4 * q + 3) * kThreads] = v.w;
    }
    uint32_t bb[L + 1], n[L], y[L];
    ldb<L>(arr(sqr ? a : b, count, k), 0, y);
    ldb<L>(arr(N, count, k), 0, n);
    const uint32_t n0p = word_at(NP, count, k, 0);
    auto aw = [&](int i) { return sa[i * kThreads]; };
    if (sqr) {
        reg::double_words<L>(y, bb);
        reg::montsqr<L>(aw, bb, n, n0p, y);
    } else {
        reg::montmul<L>(aw, y, n, n0p, y);
    }
    stb<L>(arr(c, count, k), 0, y);
}

// Stand-alone TRUNCATED MontMul / MontSqr at L = 32 (mont_batch_mul / mont_batch_sqr, redc =
// truncated): reg::montmul_trunc (alg:trunc_montred, with Theorem 2's correction at word
// granularity), one operation per thread, squaring and multiplication as separate instantiations
// (SQR compile-time).  Per-thread shared memory: the a operand, N, N', T's high half.
template <int L, bool SQR>
__global__ void __launch_bounds__(kThreads, MPB_REG_MINB) k_mont_mul_rtr(
    const uint32_t* __restrict__ a, const uint32_t* __restrict__ b, const uint32_t* __restrict__ N,
    const uint32_t* __restrict__ NP, uint32_t* __restrict__ c, size_t count) {
    const size_t k = tid_global();
    if (k >= count) return;
    constexpr int Q4 = L / 4;
    constexpr int SL = L * kThreads;
    extern __shared__ __align__(16) uint32_t smem_a[];
    uint32_t* const sa = smem_a + threadIdx.x;
    uint32_t* const sn = sa + SL;
    uint32_t* const snp = sa + 2 * SL;
    uint32_t* const sth = sa + 3 * SL;
    auto to_slot = [&](uint32_t* slot, const Arr& A) {
#pragma unroll
        for (int q = 0; q < Q4; q++) {
            const uint4 v = A.ld(q);
            slot[(4 * q) * kThreads] = v.x;
            slot[(4 * q + 1) * kThreads] = v.y;
            slot[(4 * q + 2) * kThreads] = v.z;
            slot[(4 * q + 3) * kThreads] = v.w;
        }
    };
    to_slot(sa, arr(a, count, k));
    to_slot(sn, arr(N, count, k));
    to_slot(snp, arr(NP, count, k));
    auto aw = [&](int i) { return sa[i * kThreads]; };
    auto nw = [&](int j) { return sn[j * kThreads]; };
    auto npw = [&](int j) { return snp[j * kThreads]; };
    auto thw = [&](int i, uint32_t v) { sth[i * kThreads] = v; };
    auto thr = [&](int i) { return sth[i * kThreads]; };
    uint32_t bb[L], y[L];
    ldb<L>(arr(SQR ? a : b, count, k), 0, bb);
    reg::montmul_trunc<L>(SQR, aw, bb, npw, nw, thw, thr, y);
    stb<L>(arr(c, count, k), 0, y);
}

// Register-resident TRUNCATED exponentiation at L = 32 (mont_batch_modexp_ct, redc = truncated):
// reg::montmul_trunc (alg:trunc_montred + Theorem 2 at word granularity) as MontSqr and MontMul
// instances, one call site each, inside the same flat public schedule as k_modexp_reg.  Per-thread
// shared memory (word q of thread t at q * blockDim + t): the a operand, N, N', T's high half.
template <int L>
__global__ void __launch_bounds__(kThreads, MPB_REG_MINB) k_modexp_rtr(
    const uint32_t* __restrict__ N, const uint32_t* __restrict__ NP, const uint32_t* __restrict__ R2,
    const uint32_t* __restrict__ base, const uint32_t* __restrict__ exp, uint32_t* __restrict__ out, size_t count,
    int bits, int w, uint32_t* ws) {
    const size_t k = tid_global();
    if (k >= count) return;
    constexpr int Q4 = L / 4;
    constexpr int SL = L * kThreads;  // words per shared-memory region
    const int nent = 1 << w;
    extern __shared__ __align__(16) uint32_t smem_a[];
    uint32_t* const sa = smem_a + threadIdx.x;  // a operand
    uint32_t* const sn = sa + SL;               // N
    uint32_t* const snp = sa + 2 * SL;          // N'
    uint32_t* const sth = sa + 3 * SL;          // T high half
    const ArrT G = tarr(ws, nent * Q4, k);
    const Arr Nn = arr(N, count, k), NPn = arr(NP, count, k), R2n = arr(R2, count, k), Bn = arr(base, count, k),
              On = arr(out, count, k);
    auto to_slot = [&](uint32_t* slot, const auto& A) {
#pragma unroll
        for (int q = 0; q < Q4; q++) {
            const uint4 v = A.ld(q);
            slot[(4 * q) * kThreads] = v.x;
            slot[(4 * q + 1) * kThreads] = v.y;
            slot[(4 * q + 2) * kThreads] = v.z;
            slot[(4 * q + 3) * kThreads] = v.w;
        }
    };
    to_slot(sn, Nn);
    to_slot(snp, NPn);
    auto aw = [&](int i) { return sa[i * kThreads]; };
    auto nw = [&](int j) { return sn[j * kThreads]; };
    auto npw = [&](int j) { return snp[j * kThreads]; };
    auto thw = [&](int i, uint32_t v) { sth[i * kThreads] = v; };
    auto thr = [&](int i) { return sth[i * kThreads]; };
    const int nwin = (bits + w - 1) / w;
    auto window = [&](int win) {
        const int pos = win * w, wi = pos >> 5, off = pos & 31;
        uint32_t v = word_at(exp, count, k, wi) >> off;
        if (off + w > 32 && wi + 1 < L) v |= word_at(exp, count, k, wi + 1) << (32 - off);
        return v & ((1u << w) - 1u);
    };
    auto select = [&](uint32_t idx) { scan_to_slot<Q4>(G, nent, idx, sa); };  // CT masked scan
    uint32_t y[L];
#pragma unroll
    for (int q = 0; q < L; q++) y[q] = 0;
    const int per_win = w + 1;
    const int n_ops = nent + (nwin - 1) * per_win + 1;
#pragma unroll 1
    for (int op = 0; op < n_ops; op++) {
        uint32_t b[L];
        int store_e = -1;
        bool b_one = false, b_y = true, sqr = false;
        if (op < nent) {
            store_e = op;
            if (op == 0) {
                to_slot(sa, R2n);
                b_one = true;
            } else if (op == 1) {
                to_slot(sa, Bn);
                ldb<L>(R2n, 0, b);
                b_y = false;
            } else {
                to_slot(sa, G.at((op - 1) * Q4));
                ldb<L>(G.at(Q4), 0, b);
                b_y = false;
            }
        } else if (op == n_ops - 1) {
#pragma unroll
            for (int q = 0; q < L; q++) sa[q * kThreads] = y[q];
            b_one = true;
        } else {
            const int r = (op - nent) % per_win, win = nwin - 2 - (op - nent) / per_win;
            if (r < w) sqr = true;
            else select(window(win));
        }
        if (b_one) {
#pragma unroll
            for (int q = 0; q < L; q++) b[q] = q == 0 ? 1u : 0u;
        } else if (b_y) {
#pragma unroll
            for (int q = 0; q < L; q++) b[q] = y[q];
        }
        reg::montmul_trunc<L>(sqr, aw, b, npw, nw, thw, thr, y);
        if (store_e >= 0) stb<L>(G.at(store_e * Q4), 0, y);
        if (op == nent - 1) {
            select(window(nwin - 1));
#pragma unroll
            for (int q = 0; q < L; q++) y[q] = aw(q);
        }
    }
    stb<L>(On, 0, y);
}

bool launch_modexp_rtr(const uint32_t* N, const uint32_t* NP, const uint32_t* R2, const uint32_t* base,
                       const uint32_t* exp, uint32_t* out, size_t count, int bits, int window, uint32_t* ws,
                       cudaStream_t s) {
    if (4 * ((bits + 127) / 128) != 32) return false;
    const unsigned g = (unsigned)((count + kThreads - 1) / kThreads);
    const size_t sm = (size_t)kThreads * 32 * 4 * 4;  // a, N, N', T_high
    // 64 KB of dynamic shared memory needs the opt-in on every device the kernel runs on (per call:
    // a static would set it for the first device only)
    if (cudaFuncSetAttribute(k_modexp_rtr<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) != cudaSuccess)
        return false;
    k_modexp_rtr<32><<<g, kThreads, sm, s>>>(N, NP, R2, base, exp, out, count, bits, window, ws);
    return true;
}

bool launch_mont_mul_rtr(const uint32_t* a, const uint32_t* b, const uint32_t* N, const uint32_t* NP, uint32_t* c,
                         size_t count, int bits, bool sqr, cudaStream_t s) {
    if (4 * ((bits + 127) / 128) != 32) return false;
    const unsigned g = (unsigned)((count + kThreads - 1) / kThreads);
    const size_t sm = (size_t)kThreads * 32 * 4 * 4;  // a, N, N', T_high
    if (sqr) {
        if (cudaFuncSetAttribute(k_mont_mul_rtr<32, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) !=
            cudaSuccess)
            return false;
        k_mont_mul_rtr<32, true><<<g, kThreads, sm, s>>>(a, a, N, NP, c, count);
    } else {
        if (cudaFuncSetAttribute(k_mont_mul_rtr<32, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) !=
            cudaSuccess)
            return false;
        k_mont_mul_rtr<32, false><<<g, kThreads, sm, s>>>(a, b, N, NP, c, count);
    }
    return true;
}

// MPB_REG_SQR=0 runs MontSqr through the multiplication rows (A/B); default: squaring rows
static int reg_sqr_rows() {
    static int v = [] {
        const char* e = getenv("MPB_REG_SQR");
        return e ? atoi(e) : 1;
    }();
    return v;
}

bool launch_mont_mul_reg(const uint32_t* a, const uint32_t* b, const uint32_t* N, const uint32_t* NP, uint32_t* c,
                         size_t count, int bits, cudaStream_t s) {
    if (4 * ((bits + 127) / 128) != 32) return false;
    const unsigned g = (unsigned)((count + kThreads - 1) / kThreads);
    k_mont_mul_reg<32><<<g, kThreads, (size_t)kThreads * 32 * 4, s>>>(a, b, N, NP, c, count,
                                                                    a == b && reg_sqr_rows());
    return true;
}

bool launch_modexp_reg(const uint32_t* N, const uint32_t* NP, const uint32_t* R2, const uint32_t* base,
                       const uint32_t* exp, uint32_t* out, size_t count, int bits, int window, uint32_t* ws,
                       cudaStream_t s) {
    if (4 * ((bits + 127) / 128) != 32) return false;
    const unsigned g = (unsigned)((count + kThreads - 1) / kThreads);
    k_modexp_reg<32><<<g, kThreads, (size_t)kThreads * 32 * 4, s>>>(N, NP, R2, base, exp, out, count, bits, window,
                                                                  ws, reg_sqr_rows());
    return true;
}

}  // namespace mpb
