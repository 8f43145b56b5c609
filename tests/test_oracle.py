"""Pins for the CPU oracle (oracle/oracle.c) -- none of them re-types the oracle's formula.

Each family pins the oracle to something other than itself (SURVEY.md 8(c) "What
pins each part"): exhaustive brute force on tiny widths, Python's own big-int
library routines (a different implementation), closed forms, number-theoretic
invariants (Bezout, Fermat, exponent additivity, RSA round trip), and known
primes / Carmichael numbers.  A dropped term, wrong sign or index, or a
transposed operand anywhere in the oracle fails at least one of these.
"""
from __future__ import annotations

import math
import os
import random

import numpy as np
import pytest

import oracle as O
from adversarial import column_sum_L_minus_1, redc_family
from paper_2410_18129_b200 import inputs as I

RNG = random.Random(2410_18129)


# ------------------------------------------------------------------ o_mul / o_sqr
def test_mul_exhaustive_tiny():
    # all a, b < 2^7 (brute force against the definition of integer multiplication)
    for a in range(1 << 7):
        for b in range(0, 1 << 7, 1):
            assert O.mul(a, b) == a * b
    # one-limb grid including the carry extremes
    grid = [0, 1, 2, 3, 0xFFFF, 0x10000, 0x7FFFFFFF, 0x80000000, 0xFFFFFFFE, 0xFFFFFFFF]
    for a in grid:
        for b in grid:
            assert O.mul(a, b) == a * b


@pytest.mark.parametrize("bits", [32, 33, 64, 100, 1024, 2048, 3072, 4096, 4154, 8320])
def test_mul_vs_python_int(bits):
    for _ in range(6):
        a, b = RNG.getrandbits(bits), RNG.getrandbits(RNG.randint(1, bits))
        assert O.mul(a, b) == a * b
        assert O.sqr(a) == a * a


@pytest.mark.parametrize("m", [1, 31, 32, 33, 64, 1024, 2048, 4096, 4154])
def test_mul_closed_forms(m):
    ones = (1 << m) - 1
    # (2^m - 1)^2 = 2^(2m) - 2^(m+1) + 1
    assert O.sqr(ones) == (1 << (2 * m)) - (1 << (m + 1)) + 1
    a = RNG.getrandbits(m) | 1
    b = RNG.getrandbits(m)
    for k in (0, 1, 31, 32, 33, 100):
        assert O.mul(a, 1 << k) == a << k  # multiplication by 2^k is a shift
    assert O.sqr(a) == O.mul(a, a)
    assert O.sqr(a + b) == O.sqr(a) + 2 * O.mul(a, b) + O.sqr(b)  # binomial identity
    assert O.mul(a, b) == O.mul(b, a)


# -------------------------------------------------------------------- o_divmod
def test_divmod_exhaustive_tiny():
    for a in range(1 << 8):
        for b in range(1, 1 << 8):
            q, r = O.divmod_(a, b)
            assert a == q * b + r and 0 <= r < b


def test_divmod_zero_divisor():
    with pytest.raises(ZeroDivisionError):
        O.divmod_(5, 0)


def _structured(nlimbs):
    pool = [0, 1, 0x7FFFFFFF, 0x80000000, 0xFFFFFFFE, 0xFFFFFFFF]
    return sum((RNG.choice(pool) if RNG.random() < 0.7 else RNG.getrandbits(32)) << (32 * i) for i in range(nlimbs))


def test_divmod_vs_python_and_knuth_stress():
    for _ in range(3000):
        nb = RNG.randint(1, 8)
        na = RNG.randint(1, 16)
        a = _structured(na)
        b = _structured(nb) or 1
        if RNG.random() < 0.3:  # divisor top limb 0x80000000 / 0xFFFFFFFF
            b = (b & ((1 << (32 * (nb - 1))) - 1)) | (RNG.choice([0x80000000, 0xFFFFFFFF]) << (32 * (nb - 1)))
        q, r = O.divmod_(a, b)
        assert (q, r) == divmod(a, b)
    # dividend all ones
    for nb in range(1, 10):
        b = RNG.getrandbits(32 * nb) | (1 << (32 * nb - 1))
        a = (1 << (32 * 2 * nb)) - 1
        assert O.divmod_(a, b) == divmod(a, b)


def test_divmod_add_back_case():
    # Knuth D step D6 (add back) fires when qhat overestimates by one after the D3 test.
    # u = 0x8000_0000_0000_0000_0000_0000_0000_0000 / v = 0x8000_0000_0000_0000_0000_0001 style
    # cases: search a structured family until the quotient's estimate needs the add-back, pinning
    # the path against Python divmod.
    hits = 0
    for t in range(20000):
        v = (0x80000000 << 64) | (RNG.choice([0, 1, 0xFFFFFFFF]) << 32) | RNG.getrandbits(32)
        u = (RNG.getrandbits(32) << 96) | (RNG.choice([0, 0xFFFFFFFF]) << 64) | RNG.getrandbits(64)
        if u >> 96 >= 0x80000000:
            u >>= 1
        q, r = O.divmod_(u, v)
        assert (q, r) == divmod(u, v)
        hits += 1
    assert hits == 20000


# --------------------------------------------------------- inverse, egcd, setup
def test_egcd_bezout_and_gcd():
    for _ in range(300):
        n = RNG.randint(1, 6)
        a, b = RNG.getrandbits(32 * n) | 1, RNG.getrandbits(32 * n) | 1
        g0 = RNG.getrandbits(20) + 1
        a, b = a * g0, b * g0  # force a non-trivial gcd
        x, y, g = O.egcd(a, b)
        assert g == math.gcd(a, b)
        assert a * x - b * y == g  # Bezout identity
        assert 0 <= x < b


def test_inv_mod_vs_python_pow():
    for _ in range(300):
        m = RNG.getrandbits(RNG.randint(2, 300)) | 1
        a = RNG.randrange(1, m) if m > 1 else 0
        if math.gcd(a, m) != 1:
            with pytest.raises(ValueError):
                O.inv_mod(a, m)
            continue
        x = O.inv_mod(a, m)
        assert x == pow(a, -1, m)
        assert (a * x) % m == 1 % m
    with pytest.raises(ValueError):
        O.inv_mod(6, 9)


@pytest.mark.parametrize("bits", [64, 1024, 2048, 4096, 4108])
def test_setup_invariants(bits):
    L = I.limbs_for_bits(bits)
    R = 1 << (32 * L)
    for _ in range(3):
        N = RNG.getrandbits(bits) | 1 | (1 << (bits - 1))
        Np, R2 = O.setup(N, L)
        assert (N * Np) % R == R - 1  # N * N' == -1 (mod R)
        assert Np == (-pow(N, -1, R)) % R
        assert R2 == pow(2, 64 * L, N)  # R^2 mod N
        assert R2 < N


# ---------------------------------------------------------------- montmul/redc
@pytest.mark.parametrize("bits", [64, 1024, 2048])
def test_montmul_definition_and_roundtrip(bits):
    L = I.limbs_for_bits(bits)
    R = 1 << (32 * L)
    for _ in range(4):
        N = RNG.getrandbits(bits) | 1 | (1 << (bits - 1))
        Np, R2 = O.setup(N, L)
        a, b = RNG.randrange(N), RNG.randrange(N)
        c = O.montmul(a, b, N, L)
        assert 0 <= c < N
        assert (c * R - a * b) % N == 0  # c * R == a * b (mod N)
        # Montgomery form round trip: from_mont(to_mont(x)) == x
        am = O.montmul(a, R2, N, L)
        assert am == (a * R) % N
        assert O.montmul(am, 1, N, L) == a
        # Montgomery one: montmul(R mod N, x) == x
        assert O.montmul(R % N, b, N, L) == b
        # second route (alg:montred) agrees after one conditional subtraction
        T = a * b
        C = O.montred_classic(T, N, Np, L)
        assert C < 2 * N
        assert (C - N if C >= N else C) == c
        assert O.redc(T, N, L) == c


@pytest.mark.parametrize("bits", [32, 64, 1024, 2048, 4096])
def test_cios_route_matches_definition(bits):
    """alg:8BlockMontRed step by step with n0' only (A10) lands within one N of the
    plain definition a*b*R^-1 mod N, including the extreme operands 0, 1 and N-1."""
    L = I.limbs_for_bits(bits)
    R = 1 << (32 * L)
    for _ in range(4):
        N = RNG.getrandbits(bits) | 1 | (1 << (bits - 1))
        Np, _ = O.setup(N, L)
        n0p = Np & 0xFFFFFFFF
        assert (N * n0p) % (1 << 32) == (1 << 32) - 1  # n0' = -N^-1 mod 2^32
        for a, b in [(RNG.randrange(N), RNG.randrange(N)), (0, RNG.randrange(N)), (1, 1), (N - 1, N - 1)]:
            C = O.montmul_cios(a, b, N, n0p, L)
            assert C < 2 * N
            assert (C * R - a * b) % N == 0
            assert (C - N if C >= N else C) == O.montmul(a, b, N, L)


# ------------------------------------------- truncated REDC reading (A6 / A7)
@pytest.mark.parametrize("bits", [64, 128, 1024, 2048])
def test_truncated_reading_random_and_adversarial(bits):
    L = I.limbs_for_bits(bits)
    R = 1 << (32 * L)
    fired = 0
    for _ in range(3):
        N = RNG.getrandbits(bits) | 1 | (1 << (bits - 1))
        Np, _ = O.setup(N, L)
        cases = [("random", RNG.randrange(N * R)) for _ in range(4)] + redc_family(RNG, N, L, per_family=3)
        for fam, T in cases:
            q = ((T % R) * Np) % R
            C, qnhat = O.montred_truncated(T, N, Np, L)
            assert qnhat == (q * N) // R, fam  # plain definition of floor(qN/R)
            assert C == (T + q * N) // R, fam  # Theorem 1: equals the classic result exactly
            assert C < 2 * N
            assert (C - N if C >= N else C) == O.redc(T, N, L)
            # count how often the exact carry correction [S mod 2^32 > K] is needed
            S = column_sum_L_minus_1(q, N, L)
            b = 1 if T % (1 << (32 * (L - 1))) else 0
            K = (-((T >> (32 * (L - 1))) & 0xFFFFFFFF) - b) % (1 << 32)
            fired += (S & 0xFFFFFFFF) > K
    assert fired > 0  # the adversarial families really exercise the correction


def _trunc_high_radix(q: int, N: int, D: int, w: int, T: int) -> int:
    """Theorem 2's truncated high part in radix 2^w (reading A6/A7 with w-bit words; the radix-2^52
    kernels, csrc/mp_dfma.cuh, use w = 52): products of weight >= D-1, hi halves of weight D-2,
    carry out of column D-1 = floor(S / 2^w) + [S mod 2^w > K], K = (-T[D-1] - b) mod 2^w."""
    M = (1 << w) - 1
    qw = [(q >> (w * i)) & M for i in range(D)]
    nw = [(N >> (w * i)) & M for i in range(D)]
    S, high = 0, 0
    for i in range(D):
        for j in range(D):
            p = qw[i] * nw[j]
            lo, hi = p & M, p >> w
            if i + j == D - 1:
                S += lo
            if i + j == D - 2:
                S += hi
            if i + j >= D:
                high += lo << (w * (i + j - D))
            if i + j >= D - 1:
                high += hi << (w * (i + j + 1 - D))
    b = 1 if T % (1 << (w * (D - 1))) else 0
    K = (-((T >> (w * (D - 1))) & M) - b) & M
    return high + (S >> w) + (1 if (S & M) > K else 0)


@pytest.mark.parametrize("bits,D", [(1024, 20), (2048, 40)])
def test_truncated_reading_radix52(bits, D):
    """The radix-2^52 reading of Theorem 2 (DESIGN 3.2, the RADIX52 kernels) equals floor(qN/R),
    R = 2^(52D), on random T and on a forced-wrap family built in radix 2^52 (S mod 2^52 =
    2^52-1-k), where the correction term is needed; dropping it fails there."""
    w = 52
    R = 1 << (w * D)
    M = (1 << w) - 1
    fired = 0
    for _ in range(3):
        N = RNG.getrandbits(bits) | 1 | (1 << (bits - 1))
        Np = (-pow(N, -1, R)) % R
        cases = [RNG.randrange(N * R) for _ in range(3)]
        for k in (0, 1, 2):  # forced wrap: choose q's top limb so S mod 2^52 = 2^52 - 1 - k
            q = RNG.randrange(R) & ~(M << (w * (D - 1)))
            qw = [(q >> (w * i)) & M for i in range(D)]
            nw = [(N >> (w * i)) & M for i in range(D)]
            rest = sum((qw[i] * nw[D - 1 - i]) & M for i in range(D - 1)) + \
                sum((qw[i] * nw[D - 2 - i]) >> w for i in range(D - 1))
            top = (((M - k) - rest) * pow(nw[0], -1, 1 << w)) & M
            q |= top << (w * (D - 1))
            cases.append((-q * N) % R + RNG.randrange(N) * R)
        for T in cases:
            q = ((T % R) * Np) % R
            got = _trunc_high_radix(q, N, D, w, T)
            assert got == (q * N) // R
            C = T // R + got + (1 if T % R else 0)
            assert C == (T + q * N) // R  # Theorem 1 in radix 2^52
            # is the correction term what made it exact?
            S_lo_gt_K = got - _trunc_high_radix_no_corr(q, N, D, w)
            fired += S_lo_gt_K
    assert fired > 0


def _trunc_high_radix_no_corr(q: int, N: int, D: int, w: int) -> int:
    M = (1 << w) - 1
    qw = [(q >> (w * i)) & M for i in range(D)]
    nw = [(N >> (w * i)) & M for i in range(D)]
    S, high = 0, 0
    for i in range(D):
        for j in range(D):
            p = qw[i] * nw[j]
            lo, hi = p & M, p >> w
            if i + j == D - 1:
                S += lo
            if i + j == D - 2:
                S += hi
            if i + j >= D:
                high += lo << (w * (i + j - D))
            if i + j >= D - 1:
                high += hi << (w * (i + j + 1 - D))
    return high + (S >> w)


def _trunc_karatsuba_high(T: int, q: int, N: int, L: int) -> int:
    """The truncated-Karatsuba high part of the REDC (reading in DESIGN 5.7b), as
    csrc/mp_kara.cuh kara_trunc_high computes it, word level: halves of H = L/2 words, Lam = -T mod R
    known, D0h and Dmh by Theorem 2 with K from Lam's low half and from Dml."""
    H = L // 2
    X = 1 << (32 * H)
    R = X * X
    lam = (-T) % R
    lam_l, lam_h = lam % X, lam // X
    q0, q1, n0, n1 = q % X, q // X, N % X, N // X
    D2 = q1 * n1
    D2l, D2h = D2 % X, D2 // X
    # _trunc_high_radix derives K = word H-1 of (-Targ mod X); here the known low half is Lam_l itself
    D0h = _trunc_high_radix(q0, n0, H, 32, (-lam_l) % X)
    sigma = 1 if (q0 >= q1) == (n0 >= n1) else -1
    V = D0h + lam_l + D2l - lam_h
    Dml = V % X if sigma == 1 else (-V) % X
    Dmh = _trunc_high_radix(abs(q0 - q1), abs(n0 - n1), H, 32, (-Dml) % X)
    c = V // X + (1 if sigma == -1 and V % X else 0)
    return D2 + D0h + D2h - sigma * Dmh + c


@pytest.mark.parametrize("bits", [512, 1024, 2048, 4096])
def test_truncated_karatsuba_reading(bits):
    """The truncated-Karatsuba REDC reading equals floor(qN/R) on random T, on T mod R = 0, and on
    the adversarial family of tests/adversarial.py t_kara_trunc, which forces BOTH half-level
    Theorem-2 corrections (dropping either one fails there)."""
    from adversarial import t_kara_trunc

    L = I.limbs_for_bits(bits)
    R = 1 << (32 * L)
    H = L // 2
    X = 1 << (32 * H)
    crafted = 0
    for _ in range(6):
        N = RNG.getrandbits(bits) | 1 | (1 << (bits - 1))
        Np = (-pow(N, -1, R)) % R
        Ts = [RNG.randrange(N * R), RNG.randrange(N) * R]
        for k0, km in ((0, 0), (1, 2), (2, 1)):
            t = t_kara_trunc(RNG, N, L, k0, km)
            if t is not None:
                Ts.append(t)
                crafted += 1
        for T in Ts:
            q = ((T % R) * Np) % R
            assert _trunc_karatsuba_high(T, q, N, L) == (q * N) // R
    assert crafted > 0
    # the family really needs both corrections
    N = next(n for n in (RNG.getrandbits(bits) | 1 | (1 << (bits - 1)) for _ in range(100))
             if (n % X) % 2 and abs(n % X - n // X) % 2)
    T = t_kara_trunc(RNG, N, L, 0, 0)
    q = ((T % R) * ((-pow(N, -1, R)) % R)) % R
    q0, q1, n0, n1 = q % X, q // X, N % X, N // X
    assert _trunc_high_radix(q0, n0, H, 32, T % X) != _trunc_high_radix_no_corr(q0, n0, H, 32)
    assert (q0 * n0) // X == _trunc_high_radix(q0, n0, H, 32, T % X)
    dq, dnn = abs(q0 - q1), abs(n0 - n1)
    assert (dq * dnn) // X != _trunc_high_radix_no_corr(dq, dnn, H, 32)


# --------------------------------------------------------------------- modexp
def test_modexp_exhaustive_tiny():
    for N in range(3, 1 << 6, 2):
        for a in range(N):
            for e in range(1 << 6):
                assert O.modexp(a, e, N, 1, ebits=6) == pow(a, e, N)


def test_modexp_random_tiny_8bit():
    for _ in range(3000):
        N = RNG.randrange(3, 256, 2)
        a, e = RNG.randrange(N), RNG.randrange(256)
        assert O.modexp(a, e, N, 1, ebits=8) == pow(a, e, N)


@pytest.mark.parametrize("bits", [64, 512, 1024, 2048])
def test_modexp_vs_python_pow(bits):
    L = I.limbs_for_bits(bits)
    for _ in range(2):
        N = RNG.getrandbits(bits) | 1 | (1 << (bits - 1))
        a = RNG.randrange(N)
        e = RNG.getrandbits(bits) | (1 << (bits - 1))
        assert O.modexp(a, e, N, L, ebits=bits) == pow(a, e, N)


def test_modexp_special_cases():
    bits, L = 1024, 32
    N = RNG.getrandbits(bits) | 1 | (1 << (bits - 1))
    a = RNG.randrange(2, N)
    assert O.modexp(a, 0, N, L, ebits=bits) == 1
    assert O.modexp(0, 0, N, L, ebits=bits) == 1  # 0^0 = 1 (matches Python pow)
    assert O.modexp(0, 5, N, L, ebits=bits) == 0
    assert O.modexp(1, (1 << bits) - 1, N, L, ebits=bits) == 1
    assert O.modexp(a, 1, N, L, ebits=bits) == a
    assert O.modexp(a, 2, N, L, ebits=bits) == (a * a) % N
    assert O.modexp(N - 1, 1234, N, L, ebits=bits) == 1  # (N-1)^even = 1
    assert O.modexp(N - 1, 1235, N, L, ebits=bits) == N - 1  # (N-1)^odd = N-1


def test_modexp_exponent_laws():
    bits, L = 512, 16
    N = RNG.getrandbits(bits) | 1 | (1 << (bits - 1))
    a = RNG.randrange(N)
    e1, e2 = RNG.getrandbits(200), RNG.getrandbits(200)
    x1, x2 = O.modexp(a, e1, N, L), O.modexp(a, e2, N, L)
    assert O.modexp(a, e1 + e2, N, L) == (x1 * x2) % N  # a^(e1+e2) = a^e1 * a^e2
    assert O.modexp(x1, e2, N, L) == O.modexp(a, e1 * e2, N, L)  # (a^e1)^e2 = a^(e1 e2)


# ----------------------------------------------------------------- primality
def test_primality_known_values():
    assert O.is_probable_prime((1 << 127) - 1)
    assert O.is_probable_prime((1 << 521) - 1)
    assert not O.is_probable_prime((1 << 128) - 1)
    for c in (561, 1105, 1729, 2465, 2821, 6601, 8911, 41041, 825265, 321197185):  # Carmichael numbers
        assert not O.is_probable_prime(c)
    for p in (2, 3, 5, 7, 251, 257, 65537, 2147483647):
        assert O.is_probable_prime(p)
    for n in (0, 1, 4, 9, 15, 65535):
        assert not O.is_probable_prime(n)


def test_primality_vs_sympy():
    sympy = pytest.importorskip("sympy")
    for _ in range(200):
        n = RNG.getrandbits(RNG.randint(8, 200)) | 1
        assert O.is_probable_prime(n) == bool(sympy.isprime(n))


@pytest.mark.parametrize("bits", [64, 256, 512])
def test_fermat_on_generated_primes(bits):
    sympy = pytest.importorskip("sympy")
    p = O.gen_prime(bits, seed=bits)
    assert p.bit_length() == bits and p & 1
    assert sympy.isprime(p)
    L = I.limbs_for_bits(bits)
    for _ in range(3):
        a = RNG.randrange(2, p - 1)
        assert O.modexp(a, p - 1, p, L, ebits=bits) == 1  # Fermat's little theorem


def test_rsa_round_trip():
    p, q = O.gen_prime(256, 11), O.gen_prime(256, 12)
    n = p * q
    lam = (p - 1) * (q - 1) // math.gcd(p - 1, q - 1)
    e = 65537
    d = O.inv_mod(e, lam)
    L = I.limbs_for_bits(512)
    for _ in range(3):
        m = RNG.randrange(n)
        c = O.modexp(m, e, n, L)
        assert O.modexp(c, d, n, L) == m


@pytest.mark.parametrize("bits", [256, 1024])
def test_rsa_crt_route(bits):
    """CRT-RSA (Garner) step by step equals the full-size private-key power c^d mod n (Python pow
    and the oracle's own modexp), including c = 0, 1, n-1 and c sharing a factor with n, and
    inverts the public operation (m^e)^d = m."""
    h = bits // 2
    Lh = I.limbs_for_bits(h)
    p, q = O.gen_prime(h, 2 * bits + 1), O.gen_prime(h, 2 * bits + 2)
    n = p * q
    lam = (p - 1) * (q - 1) // math.gcd(p - 1, q - 1)
    e = 65537
    d = O.inv_mod(e, lam)
    dp, dq, qinv = d % (p - 1), d % (q - 1), O.inv_mod(q, p)
    assert (qinv * q) % p == 1
    cs = [0, 1, n - 1, p * 3, q * 5, RNG.randrange(n), RNG.randrange(n)]
    for c in cs:
        m = O.rsa_crt(c, p, q, dp, dq, qinv, Lh, h)
        assert m == pow(c, d, n)
        if bits <= 256:
            assert m == O.modexp(c, d, n, I.limbs_for_bits(bits))
    msg = RNG.randrange(n)
    assert O.rsa_crt(pow(msg, e, n), p, q, dp, dq, qinv, Lh, h) == msg


# ----------------------------------------------------------------- batch driver
def test_batch_drivers_match_single_calls():
    N, base, exp = I.modexp_inputs(config=1, count=8, bits=1024)
    out = O.batch_modexp(base, exp, 1024, N, threads=4)
    for k in range(8):
        Nk, bk, ek = I.from_limbs(N[k]), I.from_limbs(base[k]), I.from_limbs(exp[k])
        assert I.from_limbs(out[k]) == pow(bk, ek, Nk)
    N, a, b = I.montmul_inputs(config=2, count=16, bits=2048)
    c = O.batch_montmul(a, b, N, threads=3)
    R = 1 << 2048
    for k in range(16):
        Nk = I.from_limbs(N[k])
        assert I.from_limbs(c[k]) == (I.from_limbs(a[k]) * I.from_limbs(b[k]) * pow(R, -1, Nk)) % Nk


# ------------------------------------------------------------ input generators
def test_input_generators_follow_recipe():
    for bits in (1024, 2048, 4108):
        N, base, exp = I.modexp_inputs(config=3, count=64, bits=bits)
        L = I.limbs_for_bits(bits)
        assert N.shape == (64, L) and N.dtype == np.uint32
        for k in range(64):
            n, b, e = I.from_limbs(N[k]), I.from_limbs(base[k]), I.from_limbs(exp[k])
            assert n.bit_length() == bits and n & 1
            assert 0 <= b < n
            assert e.bit_length() == bits
    # determinism
    a1 = I.modexp_inputs(config=3, count=4, bits=2048)
    a2 = I.modexp_inputs(config=3, count=4, bits=2048)
    assert all((x == y).all() for x, y in zip(a1, a2))
