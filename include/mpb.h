/*
 * mpb.h -- C ABI of libmpb.so: batched constant-time Montgomery arithmetic on NVIDIA B200
 * (sm_100a), the data-parallel hot path of arXiv 2410.18129 (PAPER.md in the reference).
 *
 * Numbers.  Unsigned integers in 32-bit limbs, little-endian (a GMP-style
 * 64-bit little-endian word array is byte-identical).  L = mpb_limbs(bits) = 4*ceil(bits/128)
 * limbs per operand, R = 2^(32L).  Any bits in 1..16384 is supported (L <= 512); larger is
 * MPB_EUNSUPPORTED.  Kernels work on blocks of C = 16, 12, 8 or 4 limbs (the largest that
 * divides L); 1024/2048/3072/4096 bits use C = 16, 4108/4154 bits (L = 132) use C = 12.
 *
 * Layout ("word-sliced", the B200 form of the paper's Table 1 word slicing):
 * every device array argument below holds `count` operands of `nlimbs` limbs as
 *     limb i of operand k at  uint32 index  ((i/4)*count + k)*4 + (i%4)
 * i.e. 16-byte chunks of 4 consecutive limbs, chunk-major, operand-minor: one uint4 load
 * per thread per chunk, a warp reads 512 contiguous bytes.  mpb_layout_expand/contract
 * convert from/to the operand-major layout (operand k's limbs contiguous), the paper's
 * `expand`/`contract`.
 *
 * Calls.  All pointers are DEVICE pointers, 16-byte aligned, owned by the caller; the library
 * never allocates or frees them and keeps no state between calls except the thread-local
 * error string.  Work is enqueued on `stream` (a cudaStream_t, 0 = legacy default) and the
 * call returns immediately; kernel faults surface at the caller's next synchronisation.
 * count == 0 is a no-op returning MPB_OK.  Outputs must not alias inputs.
 *
 * Preconditions NOT checked on the device (no host sync; violations give unspecified
 * output, never a fault): N odd, 1 < N < 2^bits; a, b, base < N; T < N*R; exp < 2^bits;
 * Nprime == (-N)^-1 mod R; R2 == R^2 mod N.  Modular outputs are canonical, in [0, N),
 * for both REDC modes; `redc` and `algo` never change a result, only speed.
 *
 * Errors.  MPB_EINVAL: null / misaligned / aliasing pointer, redc or algo out of range,
 * window not in 1..6, workspace too small (SPEC "shape"/"usage" errors).  MPB_EUNSUPPORTED:
 * bits out of range, count > 2^27 operands per call (SPEC "configuration error").  MPB_ECUDA: launch failure; text via mpb_last_error().
 */
#ifndef PAPER_2410_18129_MPB_H
#define PAPER_2410_18129_MPB_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum { MPB_OK = 0, MPB_EINVAL = -1, MPB_EUNSUPPORTED = -2, MPB_ECUDA = -3 } mpb_status;
/* FULL: alg:8MontRed; TRUNCATED: alg:trunc_montred (Theorems 1-2);
 * CIOS: alg:8BlockMontRed, reduction interleaved with the rows of a schoolbook
 * multiplication at the engine's block granularity (digit 2^(32C), uses only the low block of
 * Nprime).  CIOS applies to mont_batch_mul/sqr and the exponentiation (schoolbook only), not
 * to a stand-alone mont_batch_redc (MPB_EUNSUPPORTED).  At 1024 bits CIOS runs a register-resident
 * kernel with the paper's 32-bit word digit (n0' = Nprime limb 0).  MontSqr under CIOS uses squaring
 * rows (each cross product once, doubled, at word or block granularity); the result is the same
 * value a^2 R^-1 mod N (at 1024 bits mont_batch_mul with a == b, the same pointer, also takes the
 * squaring rows). */
enum { MPB_REDC_FULL = 0, MPB_REDC_TRUNCATED = 1, MPB_REDC_CIOS = 2 };
/* AUTO = schoolbook: on sm_100a the blocked schoolbook engine beat every Karatsuba variant at every
 * measured size, so there is no crossover to select; KARATSUBA = one level,
 * KARATSUBA2 = two levels, explicit requests only. */
enum { MPB_ALGO_AUTO = 0, MPB_ALGO_SCHOOLBOOK = 1, MPB_ALGO_KARATSUBA = 2, MPB_ALGO_KARATSUBA2 = 3, MPB_ALGO_RADIX52 = 4,
       MPB_ALGO_HYBRID = 5 };
/* RADIX52 (mont_batch_modexp_ct only): the exponentiation runs internally on 52-bit limbs held in
 * doubles, every word product split exactly into its low and high 52-bit halves by two FP64 fused
 * multiply-adds (the paper's own radix and madd52lo/hi) and summed without carries;
 * Montgomery reduction modulo 2^(52D) with truncated or full REDC, or -- at 1024 bits only -- CIOS
 * (a register-resident kernel, the paper's word-level alg:8BlockMontRed in its own radix).  Same inputs (the
 * 32-bit N', R^2 mod N: the 52-bit constants are derived in the kernel), same canonical result.
 * Sizes: bits with a D in {20, 40, 64, 80} such that 52D >= bits + 2 and 0 <= 130D - 64L <= bits - 2
 * (1024, 2048, 3072, 4096 and 4108 bits among them); other sizes MPB_EUNSUPPORTED.
 * HYBRID (mont_batch_modexp_ct, 1921..2048 bits): one launch whose CTAs run either the 32-bit
 * schoolbook exponentiation or the RADIX52 one on disjoint operand ranges, so the integer-multiply
 * and FP64 pipes of an SM work at the same time; truncated or full REDC. */

/* L(bits) = 4*ceil(bits/128); 0 if bits <= 0. */
int mpb_limbs(int bits);
/* 1 if bits is supported (1..16384). */
int mpb_supported(int bits);

/* Layout: operand-major (count x limbs) <-> word-sliced.  limbs % 4 == 0. */
int mpb_layout_expand(const uint32_t* src_opmajor, uint32_t* dst, size_t count, int limbs, void* stream);
int mpb_layout_contract(const uint32_t* src, uint32_t* dst_opmajor, size_t count, int limbs, void* stream);

/* c = a*b, c has 2L limbs (word-sliced with 2L limbs).  Schoolbook (alg:8SBmul)
 * or block-aligned subtractive Karatsuba with 1 or 2 levels.  workspace:
 * mp_batch_workspace(count, bits, algo) bytes (0 for schoolbook: ws may then be NULL). */
int mp_batch_mul(const uint32_t* a, const uint32_t* b, uint32_t* c, size_t count, int bits, int algo,
                 void* workspace, size_t workspace_bytes, void* stream);
/* c = a^2, c has 2L limbs.  alg:8SBsqu, or Karatsuba squaring. */
int mp_batch_sqr(const uint32_t* a, uint32_t* c, size_t count, int bits, int algo, void* workspace,
                 size_t workspace_bytes, void* stream);
size_t mp_batch_workspace(size_t count, int bits, int algo);

/* c = a*b*R^-1 mod N (canonical).  redc = MPB_REDC_TRUNCATED (alg:trunc_montred),
 * MPB_REDC_FULL (alg:8MontRed) or MPB_REDC_CIOS (alg:8BlockMontRed).  Nprime is the full (-N)^-1 mod R (limb 0 is
 * the n0' of CIOS).  workspace: mont_batch_workspace(count, bits) bytes of device memory. */
int mont_batch_mul(const uint32_t* a, const uint32_t* b, const uint32_t* N, const uint32_t* Nprime,
                   uint32_t* c, size_t count, int bits, int redc, void* workspace, size_t workspace_bytes,
                   void* stream);
/* c = a^2*R^-1 mod N (canonical). */
int mont_batch_sqr(const uint32_t* a, const uint32_t* N, const uint32_t* Nprime, uint32_t* c, size_t count,
                   int bits, int redc, void* workspace, size_t workspace_bytes, void* stream);
/* c = T*R^-1 mod N for T < N*R given with 2L limbs (word-sliced with 2L limbs).  alg:montred.
 * At 1024/2048/3072/4096/4108 bits this runs the exponentiation's own engine instantiation
 * (compile-time block count, warp-tiled workspace), so it exercises the code mont_batch_modexp_ct
 * ships.  workspace: mont_batch_workspace(count, bits) bytes. */
int mont_batch_redc(const uint32_t* T, const uint32_t* N, const uint32_t* Nprime, uint32_t* c, size_t count,
                    int bits, int redc, void* workspace, size_t workspace_bytes, void* stream);
size_t mont_batch_workspace(size_t count, int bits);

/* out = base^exp mod N, constant-time fixed-window left-to-right exponentiation
 * (alg:8FWExp): 2^window-entry table in Montgomery form, windows LSB-aligned,
 * the top partial window selects the start value, then per window `window` Montgomery
 * squarings, a masked full-table scan and one Montgomery multiplication.
 * exp has L limbs and `bits` significant bits (zero padded); timing depends on
 * (count, bits, window, redc) only.  window in 1..6.  exp = 0 gives 1 (0^0 = 1).
 * For >= 3072-bit operands, small batches run with 8, 4 or 2 lanes of a warp per operand (8 while
 * 8*count <= SMs*128, 4 while 4*count <= SMs*256, 2 while 2*count <= SMs*128), block products of
 * every block column split between the lanes and their windows summed by shuffles (the result is
 * the same; only the schedule differs).  A batch that fits one wave on the device (count <= SMs*384,
 * or SMs*448 at 4096 / 4108 bits) runs one thread per operand as one CTA of 32*ceil(ceil(count/SMs)/32)
 * threads per SM, the same kernel code compiled for that block size; the
 * environment variable MPB_ONEWAVE=0, read once per process, disables this (tests, A/B). */
int mont_batch_modexp_ct(const uint32_t* N, const uint32_t* Nprime, const uint32_t* R2, const uint32_t* base,
                         const uint32_t* exp, uint32_t* out, size_t count, int bits, int window, int redc,
                         int algo, void* workspace, size_t workspace_bytes, void* stream);
size_t mont_batch_modexp_ct_workspace(size_t count, int bits, int window, int algo);

/* Montgomery constants: Nprime = (-N)^-1 mod R, R2 = R^2 mod N ("precomputed values").
 * The schedule (number of modular doublings) depends on each modulus's bit length, read from its
 * top limbs: moduli are public here.  (rsa_batch_crt_ct, whose primes are secret, runs the same
 * kernel with the public length bits/2 instead.) */
int mont_batch_setup(const uint32_t* N, uint32_t* Nprime, uint32_t* R2, size_t count, int bits,
                     void* workspace, size_t workspace_bytes, void* stream);
size_t mont_batch_setup_workspace(size_t count, int bits);

/* Batched CRT-RSA private-key operation (the paper's motivating use, P:L20 / P:L28; SURVEY
 * 8(f) f4): m = c^d mod pq computed as m_p = (c mod p)^dp mod p, m_q = (c mod q)^dq mod q by one
 * constant-time exponentiation over the 2*count half-size operands, then Garner's recombination
 * m = m_q + q * (qinv * (m_p - m_q) mod p).  bits = modulus size (even, >= 128); c and m have
 * mpb_limbs(bits) limbs, p, q, dp, dq, qinv have mpb_limbs(bits/2) limbs (word-sliced, `count`
 * operands each).  Preconditions (not checked on the device): p, q odd with exactly bits/2 bits,
 * qinv = q^-1 mod p, c < p*q, dp, dq < 2^(bits/2).  The Montgomery setup of p and q uses the public
 * length bits/2, never one read from the primes; a prime of any other length violates the
 * precondition and gives a wrong result (and Garner's single masked subtraction assumes q < 2p).  redc selects the REDC mode of the
 * exponentiation.  workspace: rsa_batch_crt_workspace(count, bits, window) bytes.
 * MPB_EUNSUPPORTED for count > 2^26 (the half-size exponentiation runs 2*count operands). */
int rsa_batch_crt_ct(const uint32_t* c, const uint32_t* p, const uint32_t* q, const uint32_t* dp, const uint32_t* dq,
                     const uint32_t* qinv, uint32_t* m, size_t count, int bits, int window, int redc,
                     void* workspace, size_t workspace_bytes, void* stream);
size_t rsa_batch_crt_workspace(size_t count, int bits, int window);

/* End-to-end convenience over HOST buffers (operand-major, L limbs each; exp L limbs):
 * allocates device memory (stream-ordered, from the library's OWN per-device memory pool, created
 * on first use and kept with an unlimited release threshold so repeated calls reuse the
 * allocation; the device's default pool is not touched), copies in, runs setup + modexp, copies
 * out, synchronises.  Returns MPB_OK or an error; blocking.  Host buffers should be pinned for
 * the copies to be asynchronous. */
int mpb_modexp_host(const uint32_t* N, const uint32_t* base, const uint32_t* exp, uint32_t* out, size_t count,
                    int bits, int window, int redc, void* stream);

/* Thread-local text of the last error ("" if none). */
const char* mpb_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
