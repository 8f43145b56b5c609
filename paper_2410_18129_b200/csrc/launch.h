// launch.h -- host-side launchers of the templated kernels.  One explicit instantiation per
// block size C (limbs per block; C in {16, 12, 8, 4}); the block count nb = L / C is a runtime
// argument, so any limb count that C divides is served by the same code.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace mpb {

template <int C>
struct Launch {
    // c = a*b (sqr: a^2), 2L limbs; levels = Karatsuba levels (0 = schoolbook); ws: scratch
    static void mp_mul(const uint32_t* a, const uint32_t* b, uint32_t* c, size_t count, int nb, bool sqr, int levels,
                       uint32_t* ws, cudaStream_t s);
    // redc: 0 full, 1 truncated, 2 CIOS
    static void mont_mul(const uint32_t* a, const uint32_t* b, const uint32_t* N, const uint32_t* NP, uint32_t* c,
                         size_t count, int nb, int redc, bool sqr, uint32_t* ws, cudaStream_t s);
    static void mont_redc(const uint32_t* T, const uint32_t* N, const uint32_t* NP, uint32_t* c, size_t count, int nb,
                          bool trunc, uint32_t* ws, cudaStream_t s);
    // CRT-RSA (k_crt_reduce / k_crt_recombine in kernels.cuh); nb = blocks of the half size
    static void crt_reduce(const uint32_t* c, int Lc, const uint32_t* PQ, const uint32_t* NPQ, const uint32_t* R2Q,
                           uint32_t* B, size_t count, int nb, uint32_t* ws, cudaStream_t s);
    static void crt_recombine(const uint32_t* M, const uint32_t* PQ, const uint32_t* NPQ, const uint32_t* R2Q,
                              const uint32_t* qinv, uint32_t* out, int Lo, size_t count, int nb, uint32_t* ws,
                              cudaStream_t s);
    // N' = (-N)^-1 mod R and R^2 mod N; ws: 6L words per operand.  pub_bits > 0: every modulus has
    // exactly this (public) bit length (CRT primes: the schedule must not depend on a secret
    // length); 0: each modulus's bit length is read from its top limbs (public moduli)
    static void setup(const uint32_t* N, uint32_t* NP, uint32_t* R2, size_t count, int nb, int pub_bits,
                      uint32_t* ws, cudaStream_t s);
    // levels: Karatsuba levels of the product phases (0 = schoolbook)
    static void modexp(const uint32_t* N, const uint32_t* NP, const uint32_t* R2, const uint32_t* base,
                       const uint32_t* exp, uint32_t* out, size_t count, int nb, int bits, int window, int redc,
                       int levels, uint32_t* ws, cudaStream_t s);
};

#define MPB_BLOCKS(X) X(16) X(12) X(8) X(4)
#define MPB_EXTERN(C) extern template struct Launch<C>;
MPB_BLOCKS(MPB_EXTERN)
#undef MPB_EXTERN

// radix-2^52 FP64 exponentiation (inst_D52.cu, mp_dfma.cuh): digits D for a size (0 = unsupported),
// its workspace, and the launch (false if the size is unsupported)
int d52_digits(int bits);
size_t d52_workspace_bytes(size_t count, int bits, int window);
bool launch_modexp_d52(const uint32_t* N, const uint32_t* NP, const uint32_t* R2, const uint32_t* base,
                       const uint32_t* exp, uint32_t* out, size_t count, int bits, int window, bool trunc,
                       uint32_t* ws, cudaStream_t s);

// register-resident radix-2^52 CIOS exponentiation at 1024 bits (inst_D52.cu, mp_dfma_reg.cuh)
size_t d52r_workspace_bytes(size_t count, int bits, int window);
bool launch_modexp_d52r(const uint32_t* N, const uint32_t* R2, const uint32_t* base, const uint32_t* exp,
                        uint32_t* out, size_t count, int bits, int window, uint32_t* ws, cudaStream_t s);

// hybrid 2048-bit exponentiation: 32-bit IMAD CTAs and radix-2^52 FP64 CTAs in one launch
size_t hybrid_workspace_bytes(size_t count, int bits, int window);
bool launch_modexp_hybrid(const uint32_t* N, const uint32_t* NP, const uint32_t* R2, const uint32_t* base,
                          const uint32_t* exp, uint32_t* out, size_t count, int bits, int window, bool trunc,
                          uint32_t* ws, cudaStream_t s);

// register-resident CIOS exponentiation for L = 32 limbs (inst_R32.cu, mp_reg.cuh); false if L != 32
bool launch_modexp_reg(const uint32_t* N, const uint32_t* NP, const uint32_t* R2, const uint32_t* base,
                       const uint32_t* exp, uint32_t* out, size_t count, int bits, int window, uint32_t* ws,
                       cudaStream_t s);

// register-resident TRUNCATED exponentiation for L = 32 limbs (inst_R32.cu)
bool launch_modexp_rtr(const uint32_t* N, const uint32_t* NP, const uint32_t* R2, const uint32_t* base,
                       const uint32_t* exp, uint32_t* out, size_t count, int bits, int window, uint32_t* ws,
                       cudaStream_t s);
bool launch_mont_mul_reg(const uint32_t* a, const uint32_t* b, const uint32_t* N, const uint32_t* NP, uint32_t* c,
                         size_t count, int bits, cudaStream_t s);
// stand-alone register-resident TRUNCATED MontMul / MontSqr for L = 32 (inst_R32.cu); false if L != 32
bool launch_mont_mul_rtr(const uint32_t* a, const uint32_t* b, const uint32_t* N, const uint32_t* NP, uint32_t* c,
                         size_t count, int bits, bool sqr, cudaStream_t s);

// scratch blocks of the Karatsuba product (mirror of mp_kara.cuh kara_scratch_blocks)
inline int kara_scratch_blocks_host(int nb, int level) {
    return level <= 0 || nb < 2 ? 0 : 4 * ((nb + 1) / 2) + kara_scratch_blocks_host((nb + 1) / 2, level - 1);
}

// block size used for a limb count: the largest of 16, 12, 8, 4 dividing L
inline int block_for(int L) { return L % 16 == 0 ? 16 : (L % 12 == 0 ? 12 : (L % 8 == 0 ? 8 : 4)); }

}  // namespace mpb

// One-wave exponentiation instances (inst_W384.cu, inst_W448.cu): the same
// k_modexp code compiled for one CTA of up to 384 (168 registers) or 448 (128 registers) threads
// per SM, launched as `grid` CTAs of `threads` (a multiple of 32) threads on stream s.  A batch
// that fits one wave runs faster this way than as several 128-thread CTAs per SM, whose warps the
// scheduler serves unevenly (the launch ends with its most starved CTA).  false: the block count
// (C, nb) or redc is not compiled in that unit (the caller falls back).
bool mpb_modexp_w384(const uint32_t* N, const uint32_t* NP, const uint32_t* R2, const uint32_t* base,
                     const uint32_t* exp, uint32_t* out, size_t count, size_t k0, size_t n, int C, int nb,
                     int bits, int window, int redc, uint32_t* ws, unsigned grid, unsigned threads, cudaStream_t s);
bool mpb_modexp_w448(const uint32_t* N, const uint32_t* NP, const uint32_t* R2, const uint32_t* base,
                     const uint32_t* exp, uint32_t* out, size_t count, size_t k0, size_t n, int C, int nb,
                     int bits, int window, int redc, uint32_t* ws, unsigned grid, unsigned threads, cudaStream_t s);
