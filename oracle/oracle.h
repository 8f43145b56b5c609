/*
 * oracle.h -- plain, slow, obviously-correct CPU oracle for the hot path of
 * arXiv 2410.18129 (batched constant-time fixed-window Montgomery modexp).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library.  It
 * shares no code, header, table or constant generator with the CUDA path
 * (paper_2410_18129_b200/csrc), and neither side includes the other.
 *
 * Numbers are little-endian arrays of 32-bit limbs with an
 * explicit limb count.  Every function computes a plain mathematical
 * definition; none of them uses Montgomery arithmetic except the two
 * "paper route" functions at the bottom, which follow the paper's algorithms
 * step by step so tests can check the paper's readings against the
 * definitions.
 *
 * Return codes: 0 = ok, -1 = invalid argument (division by zero, no inverse,
 * size mismatch).
 */
#ifndef PAPER_2410_18129_ORACLE_H
#define PAPER_2410_18129_ORACLE_H
#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* c[0..na+nb) = a * b  (schoolbook; the result of PAPER.md L140-168, alg:8SBmul). */
void o_mul(const uint32_t* a, int na, const uint32_t* b, int nb, uint32_t* c);
/* c[0..2n) = a * a  (the result of PAPER.md L177-209, alg:8SBsqu). */
void o_sqr(const uint32_t* a, int n, uint32_t* c);
/* Knuth algorithm D: a = q*b + r, 0 <= r < b.  q has na limbs, r has nb limbs. */
int o_divmod(const uint32_t* a, int na, const uint32_t* b, int nb, uint32_t* q, uint32_t* r);
/* x = a^-1 mod m by the extended Euclidean algorithm; -1 if gcd(a,m) != 1. x has nm limbs. */
int o_inv_mod(const uint32_t* a, int na, const uint32_t* m, int nm, uint32_t* x);
/* x, y, g with a*x - b*y = g = gcd(a, b) (x in [0,b), y >= 0); all have n limbs.  Bezout pin. */
int o_egcd(const uint32_t* a, const uint32_t* b, int n, uint32_t* x, uint32_t* y, uint32_t* g);
/* Montgomery constants: Nprime = (-N)^-1 mod R, R2 = R^2 mod N, R = 2^(32L). */
int o_setup(const uint32_t* N, int L, uint32_t* Nprime, uint32_t* R2);
/* c = a*b*R^-1 mod N, canonical, computed as (a*b mod N)*(R^-1 mod N) mod N. */
int o_montmul(const uint32_t* a, const uint32_t* b, const uint32_t* N, int L, uint32_t* c);
/* c = T*R^-1 mod N for a 2L-limb T (the Ensure line of alg:montred). */
int o_redc(const uint32_t* T, const uint32_t* N, int L, uint32_t* c);
/* out = base^e mod N, e has ebits bits (e_limbs = ceil(ebits/32)); left-to-right binary
 * square-and-multiply reduced by o_divmod (the Ensure line of alg:8FWExp). */
int o_modexp(const uint32_t* base, const uint32_t* e, int ebits, const uint32_t* N, int L, uint32_t* out);
/* Miller-Rabin with `rounds` bases drawn from splitmix64(seed); 1 = probable prime. */
int o_is_probable_prime(const uint32_t* n, int L, int rounds, uint64_t seed);
/* Random prime of exactly `bits` bits (top bit and bit 0 set) from splitmix64(seed). */
int o_gen_prime(int bits, uint64_t seed, uint32_t* out);

/* ---- paper routes, step by step (used only to pin the paper's readings) ---- */
/* alg:montred: q = T*N' mod R; C = (T + q*N)/R.  C has L+1 limbs, C < 2N. */
int o_montred_classic(const uint32_t* T, const uint32_t* N, const uint32_t* Nprime, int L, uint32_t* C);
/* alg:trunc_montred with Theorem 2 read as SURVEY 8(c) A6/A7:
 * qnhat = floor(q*N/R) from the partial products of weight >= L-1, the hi halves of weight
 * L-2 and the exact carry correction; C = floor(T/R) + qnhat + c_add.  C has L+1 limbs.
 * Also returns qnhat (L+1 limbs) when qnhat_out != NULL. */
int o_montred_truncated(const uint32_t* T, const uint32_t* N, const uint32_t* Nprime, int L,
                        uint32_t* C, uint32_t* qnhat_out);

/* alg:8BlockMontRed, CIOS in 32-bit words with n0' = N' mod 2^32 only:
 * C = a*B*R^-1 mod N up to one N (C < 2N), L+1 limbs; -1 if a low word fails to vanish. */
int o_montmul_cios(const uint32_t* a, const uint32_t* B, const uint32_t* N, uint32_t n0p, int L, uint32_t* C);

/* Batched CRT-RSA private-key operation: c_p = c mod p, c_q = c mod q,
 * m_p = c_p^dp mod p, m_q = c_q^dq mod q, h = qinv*(m_p - m_q) mod p, m = m_q + h*q.
 * c, m: 2*Lh limbs; p, q, dp, dq, qinv: Lh limbs; ebits = exponent bits of dp, dq. */
int o_rsa_crt(const uint32_t* c, const uint32_t* p, const uint32_t* q, const uint32_t* dp, const uint32_t* dq,
              const uint32_t* qinv, int Lh, int ebits, uint32_t* m);

/* ---- batch drivers (pthreads over independent items; operand-major arrays) ---- */
int o_batch_modexp(const uint32_t* base, const uint32_t* e, int ebits, const uint32_t* N, int L,
                   uint32_t* out, size_t count, int threads);
int o_batch_montmul(const uint32_t* a, const uint32_t* b, const uint32_t* N, int L,
                    uint32_t* c, size_t count, int threads);

#ifdef __cplusplus
}
#endif
#endif
