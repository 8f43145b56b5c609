// inst_D52.cu -- the radix-2^52 FP64 exponentiation (mp_dfma.cuh), selected by
// mont_batch_modexp_ct with algo = MPB_ALGO_RADIX52.  Same ABI, same inputs (32-bit word-sliced
// N, N', R^2 mod N, base, exp) and the same canonical result as the 32-bit kernels; only the
// internal radix differs.
#include "kernels.cuh"
#include "mp_dfma.cuh"
#include "mp_dfma_reg.cuh"

#ifndef MPB_D52_MINB
#define MPB_D52_MINB 3  // resident 128-thread CTAs per SM the radix-2^52 kernel is compiled for
#endif
#ifndef MPB_D52_C40
#define MPB_D52_C40 8  // block size of the 2048-bit (D = 40) instance (tuning: 4)
#endif

namespace mpb {

// Internal constants from the ABI's 32-bit ones (R32 = 2^(32L), R52 = 2^(52D)):
//   N'52 = -N^-1 mod R52 by one Newton step from N'32: x0 = -N'32 (= N^-1 mod R32),
//          x1 = x0 (2 - N x0) mod R52 (exact to 2^(64L) >= R52), N'52 = -x1
//   R52^2 mod N = MontSqr52(MontMul52(R2_32, 2^k)), k = 130 D - 64 L  (0 <= k <= bits - 2):
//          MontMul52(a, b) = a b 2^(-52D), so 2^(64L + k - 52D) squared is 2^(128L + 2k - 156D) = 2^(104D)
// Then alg:8FWExp exactly as k_modexp: G[0] = REDC(R^2), G[1] = MontMul(base, R^2),
// G[e] = MontMul(G[e-1], G[1]), top window by CT select, w squarings + select + multiply per window,
// REDC, and one masked subtraction to [0, N) at the end (operands live in [0, 2N), R52 >= 4N).
// Workspace (warp tiles over count rounded up to 32, D/2 chunks of 16 bytes per number):
//   G (2^w numbers) | Y | T (2 numbers) | Q | S | N | N' | X
template <int C, int NB, bool TRUNC>
MPB_DEVI void modexp_d52_body(const uint32_t* N, const uint32_t* NP, const uint32_t* R2, const uint32_t* base,
                              const uint32_t* exp, uint32_t* out, size_t count, size_t k, int L, int bits, int w,
                              uint32_t* ws) {
    namespace d = d52;
    constexpr int D = C * NB, QD = D / 2;
    const int nent = 1 << w;
    const size_t cpad = (count + 31) & ~(size_t)31;
    uint32_t* p = ws;
    auto take = [&](int nch) {
        const ArrT a = tarr(p, nch, k);
        p += cpad * (size_t)nch * 4;
        return a;
    };
    const ArrT G = take(nent * QD), Y = take(QD), T = take(2 * QD), Q = take(QD), S = take(QD), Nt = take(QD),
               NPt = take(QD), X = take(QD);
    const Stage sg = stage();
    auto zext_to_T = [&](const ArrT& a) {  // T = a zero-extended to 2D limbs (REDC input)
#pragma unroll 1
        for (int q = 0; q < QD; q++) {
            T.st(q, a.ld(q));
            T.st(QD + q, make_uint4(0, 0, 0, 0));
        }
    };
    const int nwin = (bits + w - 1) / w;
    auto window = [&](int win) {
        const int pos = win * w, wi = pos >> 5, off = pos & 31;
        uint32_t v = word_at(exp, count, k, wi) >> off;
        if (off + w > 32 && wi + 1 < L) v |= word_at(exp, count, k, wi + 1) << (32 - off);
        return v & ((1u << w) - 1u);
    };
    // One flat public schedule with a single Montgomery call site (as k_modexp):
    //   0  S = N x0 mod R52 (LO)          1  Y = x0 (2 - S) mod R52 (LO)
    //   2  Y = MontMul(R2_32, 2^k)         3  S = MontSqr(Y) = R52^2 mod N
    //   4  G[0] = REDC(S)                  5  G[1] = MontMul(base, S)
    //   4 + e (e = 2 .. 2^w - 1)  G[e] = MontMul(G[e-1], G[1])
    //   then per window: w x MontSqr(Y), select, MontMul(Y, S); the top window selects the start
    //   last  S = REDC(Y), canonical, back to 32-bit limbs
    const int n_pre = 4 + nent;
    const int per_win = w + 1;
    const int n_ops = n_pre + (nwin - 1) * per_win + 1;
#pragma unroll 1
    for (int op = 0; op < n_ops; op++) {
        int mode = d::MODE_MUL;
        ArrT A = Y, B = S, O = Y;
        if (op < n_pre) {
            if (op == 0) {
                d::from32<D>(arr(N, count, k), L, Nt);
                d::from32<D>(arr(NP, count, k), L, X);
                d::sub_from<D>(0, X, X);  // x0 = -N'32 mod R52 (= N^-1 mod R32)
                mode = d::MODE_LO; A = Nt; B = X; O = S;
            } else if (op == 1) {
                d::sub_from<D>(2, S, S);
                mode = d::MODE_LO; A = X; B = S; O = Y;  // x1 = N^-1 mod R52
            } else if (op == 2) {
                d::sub_from<D>(0, Y, NPt);  // N'52 = -x1
                d::from32<D>(arr(R2, count, k), L, X);
                d::set_pow2<D>(130 * D - 64 * L, S);
                A = X; B = S; O = Y;
            } else if (op == 3) {
                mode = d::MODE_SQR; A = Y; B = Y; O = S;
            } else if (op == 4) {
                zext_to_T(S);
                mode = d::MODE_REDC; A = T; B = T; O = G;
            } else if (op == 5) {
                d::from32<D>(arr(base, count, k), L, X);
                A = X; B = S; O = G.at(QD);
            } else {
                const int e = op - 4;
                A = G.at((e - 1) * QD); B = G.at(QD); O = G.at(e * QD);
            }
            if (op == n_pre - 1) {  // after the table: the top window selects the start value
                d::mont_op<C, NB, TRUNC>(mode, A, B, Nt, NPt, T, Q, O, sg);
                ct_select<4, 4>(G, 2 * D, nent, window(nwin - 1), Y);
                continue;
            }
        } else if (op == n_ops - 1) {
            zext_to_T(Y);
            mode = d::MODE_REDC; A = T; B = T; O = S;
        } else {
            const int r = (op - n_pre) % per_win, win = nwin - 2 - (op - n_pre) / per_win;
            if (r < w) {
                mode = d::MODE_SQR; A = Y; B = Y; O = Y;
            } else {
                ct_select<4, 4>(G, 2 * D, nent, window(win), S);
                A = Y; B = S; O = Y;
            }
        }
        d::mont_op<C, NB, TRUNC>(mode, A, B, Nt, NPt, T, Q, O, sg);
    }
    // ---- canonical [0, N), back to 32-bit limbs
    d::final_sub<D>(S, Nt, Q, X);
    d::to32<D>(X, L, arr(out, count, k));
}

template <int C, int NB, bool TRUNC>
__global__ void __launch_bounds__(kThreads, MPB_D52_MINB) k_modexp_d52(const uint32_t* __restrict__ N, const uint32_t* __restrict__ NP,
                                                          const uint32_t* __restrict__ R2, const uint32_t* __restrict__ base,
                                                          const uint32_t* __restrict__ exp, uint32_t* __restrict__ out,
                                                          size_t count, int L, int bits, int w, uint32_t* ws) {
    const size_t k = tid_global();
    if (k >= count) return;
    modexp_d52_body<C, NB, TRUNC>(N, NP, R2, base, exp, out, count, k, L, bits, w, ws);
}

// Hybrid (MPB_ALGO_HYBRID, 2048 bits): ONE kernel whose CTAs take either arithmetic -- in every
// group of three consecutive CTAs, two run the 32-bit IMAD exponentiation (k_modexp<16, RM, 4, 0>'s
// body, operands 0 .. n32-1) and one the radix-2^52 FP64 exponentiation (operands n32 .. count-1),
// so an SM's three resident CTAs mix the two and the IMAD (fmaheavy) and FP64 pipes work at the
// same time.  Same results operand by operand (each operand runs one complete, constant-time
// exponentiation).  ws32: the 32-bit path's tiled workspace for `count`; ws52: the radix-2^52 one.
template <int RM>
__global__ void __launch_bounds__(kThreads, 3) k_modexp_hybrid(
    const uint32_t* __restrict__ N, const uint32_t* __restrict__ NP, const uint32_t* __restrict__ R2,
    const uint32_t* __restrict__ base, const uint32_t* __restrict__ exp, uint32_t* __restrict__ out, size_t count,
    size_t n32, int L, int bits, int w, uint32_t* ws32, uint32_t* ws52) {
    const unsigned g = blockIdx.x / 3, r = blockIdx.x % 3;
    if (r < 2) {
        const size_t k = ((size_t)(2 * g + r)) * kThreads + threadIdx.x;
        if (k >= n32) return;
        modexp_body<16, RM, 4, 0, 1>(N, NP, R2, base, exp, out, count, k, 4, bits, w, ws32, 0u, 0xFFFFFFFFu);
    } else {
        const size_t k = n32 + (size_t)g * kThreads + threadIdx.x;
        if (k >= count) return;
        modexp_d52_body<8, 5, RM == 1>(N, NP, R2, base, exp, out, count, k, L, bits, w, ws52);
    }
}

// Register-resident radix-2^52 exponentiation at 1024 bits (D = 20; mp_dfma_reg.cuh): alg:8FWExp on
// alg:8BlockMontRed rows in the paper's radix with lazy FP64-split accumulators in registers.  The
// 52-bit constants come from the 32-bit inputs in the kernel: n0' = -N^-1 mod 2^52 by Newton in 64-bit
// integers, R52^2 = MontSqr52(MontMul52(R2_32, 2^k)), k = 130 D - 64 L (as k_modexp_d52).  Flat public
// schedule, one MontMul call site; the a operand streams from a per-thread shared-memory slot.
// Workspace (tiled, D/2 chunks per number): G (2^w numbers) | RR.
template <int D>
__global__ void __launch_bounds__(kThreads, 3) k_modexp_d52r(const uint32_t* __restrict__ N, const uint32_t* __restrict__ R2,
                                                           const uint32_t* __restrict__ base, const uint32_t* __restrict__ exp,
                                                           uint32_t* __restrict__ out, size_t count, int L, int bits, int w,
                                                           uint32_t* ws) {
    namespace d = d52;
    const size_t k = tid_global();
    if (k >= count) return;
    constexpr int QD = D / 2;
    const int nent = 1 << w;
    const size_t cpad = (count + 31) & ~(size_t)31;
    const ArrT G = tarr(ws, nent * QD, k);
    const ArrT RRt = tarr(ws + cpad * (size_t)(nent * QD) * 4, QD, k);
    extern __shared__ __align__(16) double smem_d[];
    double* const sa = smem_d + threadIdx.x;  // double j of this thread at j * blockDim
    const Arr Nn = arr(N, count, k), R2n = arr(R2, count, k), Bn = arr(base, count, k), On = arr(out, count, k);
    // 32-bit word-sliced number -> D limbs of 52 bits (doubles), in registers
    auto from32 = [&](const Arr& A, double (&x)[D]) {
#pragma unroll
        for (int j = 0; j < D; j++) {
            const int b0 = 52 * j, q = b0 >> 5, r = b0 & 31;
            uint64_t v = 0;
#pragma unroll
            for (int e = 0; e < 3; e++) {
                const int wi = q + e;
                uint32_t wv = 0;
                if (wi < L) {
                    const uint4 c = A.ld(wi >> 2);
                    const int m = wi & 3;
                    wv = m == 0 ? c.x : (m == 1 ? c.y : (m == 2 ? c.z : c.w));
                }
                const int sh = 32 * e - r;
                if (sh >= 0) v |= sh < 64 ? (uint64_t)wv << sh : 0ull;
                else v |= (uint64_t)(wv >> (-sh));
            }
            x[j] = d::to_d(v & d::kM52);
        }
    };
    auto ld_num = [&](const ArrT& A, double (&x)[D]) {
#pragma unroll
        for (int q = 0; q < QD; q++) d::unpack2(A.ld(q), x[2 * q], x[2 * q + 1]);
    };
    auto st_num = [&](const ArrT& A, const double (&x)[D]) {
#pragma unroll
        for (int q = 0; q < QD; q++) A.st(q, d::pack2(x[2 * q], x[2 * q + 1]));
    };
    auto a_set = [&](const double (&x)[D]) {
#pragma unroll
        for (int j = 0; j < D; j++) sa[j * kThreads] = x[j];
    };
    auto aw = [&](int i) { return sa[i * kThreads]; };
    double n[D];
    from32(Nn, n);
    double n0p;
    {  // n0' = -N^-1 mod 2^52: Newton on the low 52 bits of N (an odd 64-bit integer)
        const uint64_t n0 = d::limb_pat(n[0]) & d::kM52;
        uint64_t x = n0;  // correct to 3 bits (odd n0: n0 * n0 = 1 mod 8)
#pragma unroll
        for (int it = 0; it < 5; it++) x = x * (2ull - n0 * x);
        n0p = d::to_d((0ull - x) & d::kM52);
    }
    const int nwin = (bits + w - 1) / w;
    auto window = [&](int win) {
        const int pos = win * w, wi = pos >> 5, off = pos & 31;
        uint32_t v = word_at(exp, count, k, wi) >> off;
        if (off + w > 32 && wi + 1 < L) v |= word_at(exp, count, k, wi + 1) << (32 - off);
        return v & ((1u << w) - 1u);
    };
    auto select = [&](uint32_t idx) {  // CT masked full-table scan into the a slot
        uint4 acc[QD];
#pragma unroll
        for (int q = 0; q < QD; q++) acc[q] = make_uint4(0, 0, 0, 0);
#pragma unroll 1
        for (int e = 0; e < nent; e++) {
            const uint32_t x = (uint32_t)e ^ idx;
            const uint32_t m = 0u - ((x - 1u) >> 31);
            const ArrT Ge = G.at(e * QD);
#pragma unroll
            for (int q = 0; q < QD; q++) {
                const uint4 v = Ge.ld_stream(q);
                acc[q].x |= v.x & m;
                acc[q].y |= v.y & m;
                acc[q].z |= v.z & m;
                acc[q].w |= v.w & m;
            }
        }
#pragma unroll
        for (int q = 0; q < QD; q++) {
            double u, v;
            d::unpack2(acc[q], u, v);
            sa[(2 * q) * kThreads] = u;
            sa[(2 * q + 1) * kThreads] = v;
        }
    };
    // schedule: 0 Y = MontMul(R2_32, 2^k); 1 RR = MontSqr(Y); 2 G[0] = MontMul(RR, 1); 3 G[1] =
    // MontMul(base, RR); 2 + e: G[e] = MontMul(G[e-1], G[1]); top window; windows; last MontMul(Y, 1)
    double y[D];
#pragma unroll
    for (int j = 0; j < D; j++) y[j] = 0.0;
    const int n_pre = nent + 2;
    const int per_win = w + 1;
    const int n_ops = n_pre + (nwin - 1) * per_win + 1;
#pragma unroll 1
    for (int op = 0; op < n_ops; op++) {
        double b[D];
        int kind = 0;  // 0: b = y, 1: b = one, 2: b loaded
        const ArrT* store = nullptr;
        ArrT dst = G;
        if (op == 0) {
            double x[D];
            from32(R2n, x);
            a_set(x);
            const int kk = 130 * D - 64 * L;
#pragma unroll
            for (int j = 0; j < D; j++) b[j] = j == kk / 52 ? d::to_d(1ull << (kk % 52)) : 0.0;
            kind = 2;
        } else if (op == 1) {
            a_set(y);
            dst = RRt; store = &dst;
        } else if (op == 2) {
            double x[D];
            ld_num(RRt, x);
            a_set(x);
            kind = 1;
            dst = G; store = &dst;
        } else if (op == 3) {
            double x[D];
            from32(Bn, x);
            a_set(x);
            ld_num(RRt, b);
            kind = 2;
            dst = G.at(QD); store = &dst;
        } else if (op < n_pre) {
            const int e = op - 2;
            double x[D];
            ld_num(G.at((e - 1) * QD), x);
            a_set(x);
            ld_num(G.at(QD), b);
            kind = 2;
            dst = G.at(e * QD); store = &dst;
        } else if (op == n_ops - 1) {
            a_set(y);
            kind = 1;
        } else {
            const int r = (op - n_pre) % per_win, win = nwin - 2 - (op - n_pre) / per_win;
            if (r < w) a_set(y);
            else select(window(win));
        }
        if (kind == 0) {
#pragma unroll
            for (int j = 0; j < D; j++) b[j] = y[j];
        } else if (kind == 1) {
#pragma unroll
            for (int j = 0; j < D; j++) b[j] = j == 0 ? 1.0 : 0.0;
        }
        d52r::montmul<D>(aw, b, n, n0p, y);
        if (store) st_num(*store, y);
        if (op == n_pre - 1) {  // after the table: Y = G[top window]
            select(window(nwin - 1));
#pragma unroll
            for (int j = 0; j < D; j++) y[j] = aw(j);
        }
    }
    // canonical [0, N): y - N if y >= N (y <= N after the final REDC), back to 32-bit limbs
    uint64_t yl[D], dl[D];
    uint64_t borrow = 0;
#pragma unroll
    for (int j = 0; j < D; j++) {
        yl[j] = d::limb_pat(y[j]) & d::kM52;
        const uint64_t v = yl[j] - (d::limb_pat(n[j]) & d::kM52) - borrow;
        dl[j] = v & d::kM52;
        borrow = (v >> 63) & 1ull;
    }
    const uint64_t m = 0ull - (borrow ^ 1ull);  // all ones: y >= N
#pragma unroll
    for (int j = 0; j < D; j++) yl[j] = (dl[j] & m) | (yl[j] & ~m);
#pragma unroll 1
    for (int q4 = 0; q4 < L / 4; q4++) {
        uint32_t wv[4];
#pragma unroll
        for (int mm = 0; mm < 4; mm++) {
            const int b0 = 32 * (4 * q4 + mm), j = b0 / 52, r = b0 - 52 * j;
            uint64_t x = 0;
#pragma unroll
            for (int e = 0; e < D; e++) {  // (compile-time select of limbs j, j+1 without dynamic indexing)
                if (e == j) x |= yl[e] >> r;
                if (e == j + 1) x |= yl[e] << (52 - r);
            }
            wv[mm] = (uint32_t)x;
        }
        On.st(q4, make_uint4(wv[0], wv[1], wv[2], wv[3]));
    }
}

size_t d52r_workspace_bytes(size_t count, int bits, int window) {
    if (4 * ((bits + 127) / 128) != 32 || d52_digits(bits) != 20) return 0;
    const size_t cpad = (count + 31) & ~(size_t)31;
    return cpad * 10 * 16 * (size_t)((1 << window) + 1);
}

bool launch_modexp_d52r(const uint32_t* N, const uint32_t* R2, const uint32_t* base, const uint32_t* exp,
                        uint32_t* out, size_t count, int bits, int window, uint32_t* ws, cudaStream_t s) {
    if (!d52r_workspace_bytes(1, bits, window)) return false;
    const unsigned g = (unsigned)((count + kThreads - 1) / kThreads);
    k_modexp_d52r<20><<<g, kThreads, (size_t)kThreads * 20 * 8, s>>>(N, R2, base, exp, out, count, 32, bits, window,
                                                                    ws);
    return true;
}

// (C, NB) instances: 1024 (4, 5) D = 20; 2048 (8, 5) D = 40; 3072 (8, 8) D = 64; 4096 / 4108 (8, 10) D = 80
int d52_digits(int bits) {
    const int L = 4 * ((bits + 127) / 128);
    for (int D : {20, 40, 64, 80}) {
        const int kk = 130 * D - 64 * L;
        if (52 * D >= bits + 2 && kk >= 0 && kk <= bits - 2) return D;
    }
    return 0;
}

size_t d52_workspace_bytes(size_t count, int bits, int window) {
    const int D = d52_digits(bits);
    if (!D) return 0;
    const size_t cpad = (count + 31) & ~(size_t)31;
    return cpad * (size_t)(D / 2) * 16 * (size_t)((1 << window) + 8);
}

// 32-bit share of a hybrid launch: MPB_HYBRID_FRAC (0..1, tuning) or 2/3 (two of three CTAs)
static double hybrid_frac32() {
    static double v = [] {
        const char* e = getenv("MPB_HYBRID_FRAC");
        const double f = e ? atof(e) : 2.0 / 3.0;
        return f > 0.0 && f < 1.0 ? f : 2.0 / 3.0;
    }();
    return v;
}

size_t hybrid_workspace_bytes(size_t count, int bits, int window) {
    if (bits <= 1920 || bits > 2048) return 0;  // L = 64 limbs (NB = 4 of C = 16) and D = 40
    const size_t cpad = (count + 31) & ~(size_t)31;
    const size_t ws32 = cpad * 64 * (size_t)((1 << window) + 7) * 4;
    return ws32 + d52_workspace_bytes(count, bits, window) + 256;
}

bool launch_modexp_hybrid(const uint32_t* N, const uint32_t* NP, const uint32_t* R2, const uint32_t* base,
                          const uint32_t* exp, uint32_t* out, size_t count, int bits, int window, bool trunc,
                          uint32_t* ws, cudaStream_t s) {
    if (!hybrid_workspace_bytes(count, bits, window) || d52_digits(bits) != 40) return false;
    const size_t cpad = (count + 31) & ~(size_t)31;
    uint32_t* ws32 = ws;
    uint32_t* ws52 = ws + ((cpad * 64 * (size_t)((1 << window) + 7) + 63) & ~(size_t)63);
    // 32-bit operands: a whole number of 128-thread CTAs
    size_t n32 = (size_t)(hybrid_frac32() * (double)count) / kThreads * kThreads;
    if (n32 > count) n32 = count;
    const size_t c32 = (n32 + kThreads - 1) / kThreads, c52 = (count - n32 + kThreads - 1) / kThreads;
    const size_t groups = ((c32 + 1) / 2 > c52 ? (c32 + 1) / 2 : c52);
    const unsigned g = (unsigned)(3 * groups);
    const size_t sm = (size_t)kThreads * 4 * 4 * 16 + (kThreads / 32) * 16;
    if (trunc) k_modexp_hybrid<1><<<g, kThreads, sm, s>>>(N, NP, R2, base, exp, out, count, n32, 64, bits, window, ws32, ws52);
    else k_modexp_hybrid<0><<<g, kThreads, sm, s>>>(N, NP, R2, base, exp, out, count, n32, 64, bits, window, ws32, ws52);
    return true;
}

bool launch_modexp_d52(const uint32_t* N, const uint32_t* NP, const uint32_t* R2, const uint32_t* base,
                       const uint32_t* exp, uint32_t* out, size_t count, int bits, int window, bool trunc,
                       uint32_t* ws, cudaStream_t s) {

    const int L = 4 * ((bits + 127) / 128);
    const unsigned g = (unsigned)((count + kThreads - 1) / kThreads);
    const size_t sm = (size_t)kThreads * 4 * 4 * 16;  // 2 buffers x 2 blocks x (C/2 <= 4) chunks
    auto go = [&](auto Cc, auto NBc) {
        constexpr int C = decltype(Cc)::value, NBv = decltype(NBc)::value;
        if (trunc) k_modexp_d52<C, NBv, true><<<g, kThreads, sm, s>>>(N, NP, R2, base, exp, out, count, L, bits, window, ws);
        else k_modexp_d52<C, NBv, false><<<g, kThreads, sm, s>>>(N, NP, R2, base, exp, out, count, L, bits, window, ws);
        return true;
    };
    switch (d52_digits(bits)) {
        case 20: return go(std::integral_constant<int, 4>{}, std::integral_constant<int, 5>{});
#if MPB_D52_C40 == 4
        case 40: return go(std::integral_constant<int, 4>{}, std::integral_constant<int, 10>{});
#else
        case 40: return go(std::integral_constant<int, 8>{}, std::integral_constant<int, 5>{});
#endif
        case 64: return go(std::integral_constant<int, 8>{}, std::integral_constant<int, 8>{});
        case 80: return go(std::integral_constant<int, 8>{}, std::integral_constant<int, 10>{});
        default: return false;
    }
}

}  // namespace mpb
