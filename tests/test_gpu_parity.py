"""GPU parity: every C-ABI entry point of libmpb.so against the CPU oracle, bit-exact.

All arithmetic is exact unsigned integer ("no floating point, no rounding
and no tolerance anywhere on this path"), so every comparison is element-by-element
equality.  Sizes span several C=16-limb blocks and ragged batch tails (count not a
multiple of the 128-thread CTA); the full-size cases sample outputs the oracle can
recompute one by one and check truncated == full REDC on the whole batch.
"""
from __future__ import annotations

import functools
import random

import numpy as np
import pytest

import oracle as O
from adversarial import redc_family, t_gamma, t_kara_trunc
from paper_2410_18129_b200 import inputs as I

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

BITS_MOD = [512, 1024, 2048, 3072, 4096, 4108]
BITS_ODD = [256, 700, 1536]  # block sizes 8 and 12, odd block counts
BITS_MUL = [512, 1024, 2048, 3072, 4096, 4154]
ALGOS = [1, 2, 3]  # schoolbook, 1-level Karatsuba, 2-level Karatsuba
REDC = [1, 0, 2]  # truncated, full, CIOS (alg:8BlockMontRed)
REDC_STANDALONE = [1, 0]  # a stand-alone REDC has no CIOS form


@pytest.fixture(scope="module")
def mpb():
    from paper_2410_18129_b200 import mpb as m

    return m


def ints(arr):
    return I.array_to_ints(arr)


def structured_operands(N_ints, L):
    """Edge operands below each modulus: 0, 1, N-1, 2^k, all-ones below N, N>>1."""
    out = []
    for n in N_ints:
        cands = [0, 1, n - 1, n >> 1, (1 << (n.bit_length() - 1)) - 1, 1 << (n.bit_length() // 2)]
        out.append(cands)
    return out


# ------------------------------------------------------------------------ layout
@pytest.mark.parametrize("L,count", [(4, 1), (16, 33), (64, 1000), (132, 129)])
def test_layout_roundtrip(mpb, L, count):
    rng = np.random.default_rng(L * 1000 + count)
    x = rng.integers(0, 1 << 32, size=(count, L), dtype=np.uint64).astype(np.uint32)
    d = mpb.to_device(x)
    assert d.shape == (L // 4, count, 4)
    # the device layout is exactly the documented word-sliced formula
    flat = d.cpu().numpy().view(np.uint32).reshape(-1)
    for (k, i) in [(0, 0), (count - 1, L - 1), (count // 2, L // 2)]:
        assert flat[((i // 4) * count + k) * 4 + (i % 4)] == x[k, i]
    assert np.array_equal(mpb.to_host(d), x)


# ---------------------------------------------------------------------- products
@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("bits", BITS_MUL + [96, 700, 1536])
def test_mp_batch_mul_sqr(mpb, bits, algo):
    count = 130  # ragged over 128-thread CTAs
    a, b = I.mul_inputs(config=4, count=count, bits=bits)
    L = a.shape[1]
    # structured rows: all ones (carry worst case), zero, one, powers of two
    a[0] = np.uint32(0xFFFFFFFF); b[0] = np.uint32(0xFFFFFFFF)
    a[1] = 0; a[2] = 0; a[2, 0] = 1
    a[3] = 0; a[3, L - 1] = np.uint32(1 << 31); b[3] = np.uint32(0xFFFFFFFF)
    da, db = mpb.to_device(a), mpb.to_device(b)
    c = mpb.to_host(mpb.mp_batch_mul(da, db, bits, algo))
    s = mpb.to_host(mpb.mp_batch_sqr(da, bits, algo))
    A, B = ints(a), ints(b)
    for k in range(count):
        assert I.from_limbs(c[k]) == O.mul(A[k], B[k]), k
        assert I.from_limbs(s[k]) == O.sqr(A[k]), k


# ------------------------------------------------------------------------- setup
@pytest.mark.parametrize("bits", BITS_MOD + BITS_ODD)
def test_setup(mpb, bits):
    count = 40
    N, _, _ = I.modexp_inputs(config=2, count=count, bits=bits)
    L = N.shape[1]
    Np, R2 = mpb.mont_batch_setup(mpb.to_device(N), bits)
    Np, R2 = mpb.to_host(Np), mpb.to_host(R2)
    for k, n in enumerate(ints(N)):
        np_ref, r2_ref = O.setup(n, L)
        assert I.from_limbs(Np[k]) == np_ref
        assert I.from_limbs(R2[k]) == r2_ref


def _mont_fixture(mpb, bits, count, config=2):
    N, a, b = I.montmul_inputs(config=config, count=count, bits=bits)
    dN = mpb.to_device(N)
    Np, R2 = mpb.mont_batch_setup(dN, bits)
    return N, a, b, dN, Np, R2


# ----------------------------------------------------------- montmul / montsqr
@pytest.mark.parametrize("redc", REDC)
@pytest.mark.parametrize("bits", BITS_MOD + BITS_ODD)
def test_mont_mul_sqr(mpb, bits, redc):
    count = 131
    N, a, b, dN, Np, R2 = _mont_fixture(mpb, bits, count)
    L = N.shape[1]
    # edge operands in the first rows
    for k, n in enumerate(ints(N[:6])):
        ev = [0, 1, n - 1, n >> 1, n - 2, (n - 1) // 3][k]
        a[k] = I.to_limbs(ev, L)
        b[k] = I.to_limbs([n - 1, n - 1, n - 1, 1, n - 2, 0][k], L)
    da, db = mpb.to_device(a), mpb.to_device(b)
    c = mpb.to_host(mpb.mont_batch_mul(da, db, dN, Np, bits, redc=redc))
    s = mpb.to_host(mpb.mont_batch_sqr(da, dN, Np, bits, redc=redc))
    ref_c = O.batch_montmul(a, b, N)
    ref_s = O.batch_montmul(a, a, N)
    assert np.array_equal(c, ref_c)
    assert np.array_equal(s, ref_s)


@pytest.mark.parametrize("bits", [1024, 2048, 3072, 4096])
def test_mont_sqr_rows(mpb, bits):
    """CIOS MontSqr by squaring rows.  1024 bits: the register kernel (mp_reg.cuh montsqr: row i =
    a_i times a_i, 2a's word i+1 with bit 0 cleared, 2a's words above; D = 2a has L+1 words).  Larger
    sizes: the block engine (mp_mont.cuh cios_op, sqr: a_i^2 at pass i, 2 a_i a_t above).  Operands
    whose words all have the top bit set (every D word carries a bit in from below; every doubled
    block product carries out of its top word), all-ones moduli (N = 2^bits - small, a = N - 1: the
    largest carries, Y up to 3N between rows), alternating patterns, powers of two, against the
    oracle."""
    count = 96 if bits <= 2048 else 40
    L = I.limbs_for_bits(bits)
    N, a, _, dN, Np, R2 = _mont_fixture(mpb, bits, count, config=1)
    rng = np.random.default_rng(77)
    M = (1 << 32) - 1
    Ns = ints(N)
    for k in range(count):
        n = Ns[k]
        kind = k % 8
        if kind == 0:  # every word's top bit set, a < N
            v = int.from_bytes(rng.bytes(L * 4), "little") | int("80000000" * L, 16)
            v %= n
            v |= int("80000000" * (L - 1), 16) & ((1 << (32 * (L - 1))) - 1)  # keep the low words' top bits
            if v >= n:
                v %= n
        elif kind == 1:  # N = 2^bits - odd small, a = N - 1
            n = (1 << bits) - (2 * int(rng.integers(1, 1 << 20)) + 1)
            v = n - 1
        elif kind == 2:  # alternating words, top bits set
            v = int(("AAAAAAAA" + "D5555555") * (L // 2), 16) % n
        elif kind == 3:
            v = 1 << int(rng.integers(0, bits - 1))
            v %= n
        elif kind == 4:
            v = n - 1
        elif kind == 5:  # words 0xFFFFFFFF except one
            v = ((1 << bits) - 1 - (M << (32 * int(rng.integers(0, L))))) % n
        else:
            v = int.from_bytes(rng.bytes(L * 4), "little") % n
        N[k] = I.to_limbs(n, L)
        a[k] = I.to_limbs(v, L)
    dN = mpb.to_device(N)
    Np, R2 = mpb.mont_batch_setup(dN, bits)
    s = mpb.to_host(mpb.mont_batch_sqr(mpb.to_device(a), dN, Np, bits, redc=mpb.REDC_CIOS))
    assert np.array_equal(s, O.batch_montmul(a, a, N))
    # the same operands through the exponentiation (squarings dominate: w squaring rows per window)
    e = np.full((count, L), M, dtype=np.uint32)
    out = mpb.to_host(mpb.mont_batch_modexp_ct(dN, Np, R2, mpb.to_device(a), mpb.to_device(e), bits, window=5,
                                               redc=mpb.REDC_CIOS))
    assert np.array_equal(out, O.batch_modexp(a, e, bits, N))


# --------------------------------------------------------------------- REDC
@pytest.mark.parametrize("redc", REDC_STANDALONE)
@pytest.mark.parametrize("bits", BITS_MOD + BITS_ODD)
def test_mont_redc_adversarial(mpb, bits, redc):
    """The exact carry correction of Theorem 2 (families alpha..delta, tests/adversarial.py)."""
    L = I.limbs_for_bits(bits)
    rng = random.Random(bits * 7 + redc)
    N_arr, _, _ = I.modexp_inputs(config=1, count=6, bits=bits)
    Ts, Ns = [], []
    for n in ints(N_arr):
        R = 1 << (32 * L)
        for fam, t in redc_family(rng, n, L, per_family=4) + [("random", rng.randrange(n * R))]:
            Ts.append(t)
            Ns.append(n)
    count = len(Ts)
    T = I.ints_to_array(Ts, 2 * L)
    N = I.ints_to_array(Ns, L)
    dN = mpb.to_device(N)
    Np, _ = mpb.mont_batch_setup(dN, bits)
    c = mpb.to_host(mpb.mont_batch_redc(mpb.to_device(T), dN, Np, bits, redc=redc))
    for k in range(count):
        assert I.from_limbs(c[k]) == O.redc(Ts[k], Ns[k], L), k


def _gamma_low(rng: random.Random, N: int, L: int, k: int) -> int:
    """A gamma-family T (forced wrap of column L-1, tests/adversarial.py) with a zero high half
    and T < N, so it is a valid operand in the R^2 position of the exponentiation.  The forced wrap
    makes word L-1 of q*N mod R tiny, so T = -q*N mod R has its top word near 2^32 - 1: N needs an
    all-ones top word (the caller crafts such moduli)."""
    R = 1 << (32 * L)
    for _ in range(1000):
        t = t_gamma(rng, N, L, k) % R
        if t < N:
            return t
    raise AssertionError("no gamma-family T below N (the modulus needs an all-ones top word)")


def _schedule_modexp(base: int, e: int, N: int, rho: int, L: int, bits: int, w: int) -> int:
    """alg:8FWExp's public schedule as k_modexp runs it (kernels.cuh; reading A11: G[0] =
    REDC(R2), G[1] = MontMul(base, R2), G[i] = MontMul(G[i-1], G[1]), LSB-aligned windows, the top
    window selects the start, w squarings + one multiplication per window, REDC at the end), every
    Montgomery operation at its definition x*y*R^-1 mod N, with `rho` in the R^2 position."""
    R = 1 << (32 * L)
    Ri = pow(R, -1, N)

    def mm(x, y):
        return x * y * Ri % N

    G = [rho * Ri % N, mm(base, rho)]
    for _ in range(2, 1 << w):
        G.append(mm(G[-1], G[1]))
    nwin = -(-bits // w)
    dig = [(e >> (i * w)) & ((1 << w) - 1) for i in range(nwin)]
    Y = G[dig[-1]]
    for j in range(nwin - 2, -1, -1):
        for _ in range(w):
            Y = mm(Y, Y)
        Y = mm(Y, G[dig[j]])
    return Y * Ri % N


def _corr_lib():
    import ctypes
    import os

    path = os.path.join(os.path.dirname(os.path.abspath(I.__file__)), "libmpb_corr.so")
    if not os.path.exists(path):
        raise AssertionError(f"{path} missing: build() builds it beside libmpb.so")
    lib = ctypes.CDLL(path)
    lib.mpb_corr_modexp_2048.restype = ctypes.c_int
    lib.mpb_corr_modexp_2048.argtypes = [ctypes.c_void_p] * 6 + [ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p,
                                                                  ctypes.c_void_p]
    lib.mpb_corr_count_take.restype = ctypes.c_ulonglong
    return lib


def test_theorem2_correction_fires_in_shipped_modexp_kernel(mpb):
    """Theorem 2's exact carry correction exercised deterministically in
    the instantiation bench.py times, k_modexp<C=16, truncated, NB=4, schoolbook> on the warp-tiled
    workspace: a gamma-family T (S mod 2^32 = 2^32-1-k, T < N) in the R^2 position makes the
    exponentiation's first operation, REDC(R2), need the correction.  (1) The release library's
    output equals the exact schedule for every operand (and the schedule model itself reduces to
    base^e mod N when R2 = R^2 mod N).  (2) The same kernel built with the correction counter
    (libmpb_corr.so) reports that the correction fired at least once per crafted operand."""
    import ctypes

    bits, w, count = 2048, 5, 40  # ragged: one full warp tile and a partial one
    L = I.limbs_for_bits(bits)
    R = 1 << (32 * L)
    N, base, exp = I.modexp_inputs(config=3, count=count, bits=bits, dataset=7)
    crafted = list(range(0, count, 2))  # even operands crafted, odd ones keep R^2 mod N
    N[crafted, L - 1] = np.uint32(0xFFFFFFFF)  # raises N only: bases stay below it
    Ns, Bs, Es = ints(N), ints(base), ints(exp)
    rng = random.Random(2410)
    rho = [(_gamma_low(rng, n, L, k % 3) if k in crafted else R * R % n) for k, n in enumerate(Ns)]
    assert _schedule_modexp(Bs[1], Es[1], Ns[1], rho[1], L, bits, w) == pow(Bs[1], Es[1], Ns[1])
    dN, dB, dE = (mpb.to_device(x) for x in (N, base, exp))
    Np, _ = mpb.mont_batch_setup(dN, bits)
    dR = mpb.to_device(I.ints_to_array(rho, L))
    out = mpb.to_host(mpb.mont_batch_modexp_ct(dN, Np, dR, dB, dE, bits, w, redc=mpb.REDC_TRUNCATED))
    for k in range(count):
        assert I.from_limbs(out[k]) == _schedule_modexp(Bs[k], Es[k], Ns[k], rho[k], L, bits, w), k
    # full REDC on the same inputs agrees (it has no correction term)
    out_f = mpb.to_host(mpb.mont_batch_modexp_ct(dN, Np, dR, dB, dE, bits, w, redc=mpb.REDC_FULL))
    assert np.array_equal(out, out_f)
    # the counter build of the same kernel
    lib = _corr_lib()
    torch.cuda.synchronize()
    lib.mpb_corr_count_take()
    ws = mpb.modexp_workspace(count, bits, w)
    o2 = mpb.empty_sliced(L, count)
    rc = lib.mpb_corr_modexp_2048(dN.data_ptr(), Np.data_ptr(), dR.data_ptr(), dB.data_ptr(), dE.data_ptr(),
                                  o2.data_ptr(), count, w, ws.data_ptr(), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert rc == 0
    fired = lib.mpb_corr_count_take()
    assert np.array_equal(mpb.to_host(o2), out)
    assert fired >= len(crafted), fired
    # control: no crafted operand -> (almost surely) no correction in this small batch
    dR0 = mpb.to_device(I.ints_to_array([R * R % n for n in Ns], L))
    rc = lib.mpb_corr_modexp_2048(dN.data_ptr(), Np.data_ptr(), dR0.data_ptr(), dB.data_ptr(), dE.data_ptr(),
                                  o2.data_ptr(), count, w, ws.data_ptr(), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert rc == 0
    assert lib.mpb_corr_count_take() < len(crafted)
    assert np.array_equal(mpb.to_host(o2), O.batch_modexp(base, exp, bits, N))


# ------------------------------------------------------------------- modexp
MODEXP_COUNTS = {512: 70, 1024: 40, 2048: 10, 3072: 4, 4096: 3, 4108: 3, 256: 70, 700: 40, 1536: 12}


@pytest.mark.parametrize("redc", REDC)
@pytest.mark.parametrize("bits", BITS_MOD + BITS_ODD)
def test_modexp(mpb, bits, redc):
    count = MODEXP_COUNTS[bits]
    N, base, exp = I.modexp_inputs(config=3, count=count, bits=bits)
    dN = mpb.to_device(N)
    Np, R2 = mpb.mont_batch_setup(dN, bits)
    out = mpb.to_host(mpb.mont_batch_modexp_ct(dN, Np, R2, mpb.to_device(base), mpb.to_device(exp), bits,
                                               window=5, redc=redc))
    ref = O.batch_modexp(base, exp, bits, N)
    assert np.array_equal(out, ref)


@pytest.mark.parametrize("window", [1, 2, 3, 4, 5, 6])
def test_modexp_window_independence(mpb, window):
    bits, count = 1024, 20
    N, base, exp = I.modexp_inputs(config=1, count=count, bits=bits)
    dN = mpb.to_device(N)
    Np, R2 = mpb.mont_batch_setup(dN, bits)
    out = mpb.to_host(mpb.mont_batch_modexp_ct(dN, Np, R2, mpb.to_device(base), mpb.to_device(exp), bits,
                                               window=window))
    assert np.array_equal(out, O.batch_modexp(base, exp, bits, N))


@pytest.mark.parametrize("bits", [2048, 3072])
@pytest.mark.parametrize("count", [31, 32, 33, 65])
def test_modexp_warp_tile_edges(mpb, bits, count):
    """The exponentiation's warp-tiled workspace (DESIGN 5.6): counts around whole 32-operand tiles
    (a ragged last tile, exactly one tile, one operand into the next), all REDC modes, windows on
    the unguarded (w = 5) and guarded (w = 1) table-scan paths; first, last and a middle operand
    against the oracle."""
    N, base, exp = I.modexp_inputs(config=3, count=count, bits=bits, dataset=count)
    dN = mpb.to_device(N)
    Np, R2 = mpb.mont_batch_setup(dN, bits)
    idx = [0, count // 2, count - 1]
    for redc in REDC:
        for w in (5, 1):
            out = mpb.to_host(mpb.mont_batch_modexp_ct(dN, Np, R2, mpb.to_device(base), mpb.to_device(exp), bits,
                                                       window=w, redc=redc))
            assert np.array_equal(out[idx], O.batch_modexp(base[idx], exp[idx], bits, N[idx])), (redc, w)


def test_modexp_special_exponents_and_bases(mpb):
    bits = 1024
    L = I.limbs_for_bits(bits)
    N, base, exp = I.modexp_inputs(config=1, count=12, bits=bits)
    Ns = ints(N)
    cases = [(0, 0), (5, 0), (0, 7), (1, (1 << bits) - 1), (Ns[4] - 1, 1234), (Ns[5] - 1, 1235),
             (3, 1), (3, 2), (7, (1 << bits) - 1), (11, 1 << (bits - 1)), (2, 31), (Ns[11] - 2, 5)]
    for k, (bv, ev) in enumerate(cases):
        base[k] = I.to_limbs(bv, L)
        exp[k] = I.to_limbs(ev, L)
    dN = mpb.to_device(N)
    Np, R2 = mpb.mont_batch_setup(dN, bits)
    out = mpb.to_host(mpb.mont_batch_modexp_ct(dN, Np, R2, mpb.to_device(base), mpb.to_device(exp), bits))
    for k, (bv, ev) in enumerate(cases):
        assert I.from_limbs(out[k]) == O.modexp(bv, ev, Ns[k], L, ebits=bits), k


def test_modexp_fermat_primes(mpb):
    """a^(p-1) = 1 mod p for Miller-Rabin primes from the oracle (north_star Fermat pin)."""
    bits = 512
    L = I.limbs_for_bits(bits)
    ps = [O.gen_prime(bits, seed=100 + i) for i in range(4)]
    rng = random.Random(5)
    N = I.ints_to_array(ps, L)
    base = I.ints_to_array([rng.randrange(2, p - 1) for p in ps], L)
    exp = I.ints_to_array([p - 1 for p in ps], L)
    dN = mpb.to_device(N)
    Np, R2 = mpb.mont_batch_setup(dN, bits)
    out = mpb.to_host(mpb.mont_batch_modexp_ct(dN, Np, R2, mpb.to_device(base), mpb.to_device(exp), bits))
    assert all(I.from_limbs(r) == 1 for r in out)


def test_modexp_host_e2e(mpb):
    bits, count = 1024, 9
    N, base, exp = I.modexp_inputs(config=5, count=count, bits=bits)
    out = mpb.modexp_host(N, base, exp, bits, window=5)
    assert np.array_equal(out, O.batch_modexp(base, exp, bits, N))


# ------------------------------------------ register-resident CIOS (1024 bits)
@pytest.mark.parametrize("count,window", [(1, 5), (33, 1), (33, 6), (300, 5), (129, 4)])
def test_modexp_cios_register_kernel(mpb, count, window):
    """1024-bit CIOS exponentiation: the register-resident kernel (mp_reg.cuh, inst_R32.cu: rows
    fully unrolled, accumulator / multiplicand / modulus in registers) against the oracle, ragged
    counts, windows 1..6, plus edge operands (0^0, base 0, base N-1, all-ones exponent, N = 2^1024-1,
    N = 2^1023+1)."""
    bits = 1024
    L = I.limbs_for_bits(bits)
    N, base, exp = I.modexp_inputs(config=1, count=count, bits=bits, dataset=count + window)
    if count >= 12:
        N[0] = np.uint32(0xFFFFFFFF)
        N[1] = 0
        N[1, 0] = 1
        N[1, L - 1] = np.uint32(1 << 31)
        Ns = ints(N)
        cases = [(5, 7), (Ns[1] - 1, 12), (0, 0), (0, 9), (1, (1 << bits) - 1), (Ns[5] - 1, 3), (2, Ns[6] - 1),
                 (Ns[7] - 2, (1 << bits) - 1), (Ns[8] // 3, 1), (3, 1 << (bits - 1)), (Ns[10] - 1, 2),
                 (Ns[11] - 1, (1 << bits) - 2)]
        for k, (bv, ev) in enumerate(cases):
            base[k] = I.to_limbs(bv, L)
            exp[k] = I.to_limbs(ev, L)
    dN = mpb.to_device(N)
    Np, R2 = mpb.mont_batch_setup(dN, bits)
    out = mpb.to_host(mpb.mont_batch_modexp_ct(dN, Np, R2, mpb.to_device(base), mpb.to_device(exp), bits,
                                               window=window, redc=mpb.REDC_CIOS))
    assert np.array_equal(out, O.batch_modexp(base, exp, bits, N))


_RTR_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, %r)
from paper_2410_18129_b200 import inputs as I, mpb
bits = 1024
L = I.limbs_for_bits(bits)
for count, w, ds in ((37, 5, 1), (300, 4, 2), (9, 1, 3), (33, 6, 4)):
    N, base, exp = I.modexp_inputs(config=1, count=count, bits=bits, dataset=ds)
    if count >= 12:
        N[0] = np.uint32(0xFFFFFFFF)
        N[1] = 0; N[1, 0] = 1; N[1, L - 1] = np.uint32(1 << 31)
        base[2] = 0; exp[2] = 0
        base[3] = 0
        base[4] = 0; base[4, 0] = 1
        exp[5] = np.uint32(0xFFFFFFFF)
    dN = mpb.to_device(N)
    Np, R2 = mpb.mont_batch_setup(dN, bits)
    o = mpb.to_host(mpb.mont_batch_modexp_ct(dN, Np, R2, mpb.to_device(base), mpb.to_device(exp), bits, window=w,
                                             redc=mpb.REDC_TRUNCATED))
    print(count, w, ds, N.tobytes().hex(), base.tobytes().hex(), exp.tobytes().hex(), o.tobytes().hex())
"""


def test_modexp_truncated_register_kernel(mpb):
    """The register-resident truncated exponentiation at 1024 bits (mp_reg.cuh montmul_trunc:
    word-level alg:trunc_montred with Theorem 2's correction), forced with MPB_REG=2 in a
    subprocess, against the oracle: ragged counts, windows 1..6, edge operands and moduli."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = subprocess.run([sys.executable, "-c", _RTR_SCRIPT % root], env=dict(os.environ, MPB_REG="2"),
                         capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [l for l in res.stdout.splitlines() if l.strip()]
    assert len(lines) == 4
    L = 32
    for line in lines:
        count, w, ds, hn, hb, he, ho = line.split()
        count = int(count)
        N, base, exp, got = (np.frombuffer(bytes.fromhex(h), dtype=np.uint32).reshape(count, L) for h in (hn, hb, he, ho))
        assert np.array_equal(got, O.batch_modexp(base, exp, 1024, N)), (count, w)


# ------------------------------------------------- radix-2^52 FP64 path (f3)
BITS_D52 = [1024, 2048, 3072, 4096, 4108]
D52_COUNTS = {1024: 40, 2048: 37, 3072: 5, 4096: 3, 4108: 3}


@pytest.mark.parametrize("redc", REDC_STANDALONE)
@pytest.mark.parametrize("bits", BITS_D52)
def test_modexp_radix52(mpb, bits, redc):
    """mont_batch_modexp_ct with algo = RADIX52 (52-bit limbs on the FP64 pipe, mp_dfma.cuh) against
    the oracle, truncated and full REDC, ragged counts (partial warp tiles / CTAs)."""
    count = D52_COUNTS[bits]
    N, base, exp = I.modexp_inputs(config=3, count=count, bits=bits, dataset=52)
    dN = mpb.to_device(N)
    Np, R2 = mpb.mont_batch_setup(dN, bits)
    out = mpb.to_host(mpb.mont_batch_modexp_ct(dN, Np, R2, mpb.to_device(base), mpb.to_device(exp), bits,
                                               window=5, redc=redc, algo=mpb.ALGO_RADIX52))
    assert np.array_equal(out, O.batch_modexp(base, exp, bits, N))


@pytest.mark.parametrize("window", [1, 2, 3, 4, 5, 6])
def test_modexp_radix52_window_independence(mpb, window):
    bits, count = 2048, 9
    N, base, exp = I.modexp_inputs(config=1, count=count, bits=bits, dataset=window)
    dN = mpb.to_device(N)
    Np, R2 = mpb.mont_batch_setup(dN, bits)
    out = mpb.to_host(mpb.mont_batch_modexp_ct(dN, Np, R2, mpb.to_device(base), mpb.to_device(exp), bits,
                                               window=window, algo=mpb.ALGO_RADIX52))
    assert np.array_equal(out, O.batch_modexp(base, exp, bits, N))


def test_modexp_radix52_special_operands(mpb):
    """Edge operands through the radix-2^52 path: 0^0, base 0, base 1, base N-1 (even / odd
    exponents), all-ones exponent, exponent 1, 2^(bits-1), moduli with all-ones limbs."""
    bits = 2048
    L = I.limbs_for_bits(bits)
    N, base, exp = I.modexp_inputs(config=1, count=12, bits=bits, dataset=3)
    N[10] = np.uint32(0xFFFFFFFF)  # N = 2^2048 - 1 (odd, all ones)
    N[11] = 0
    N[11, 0] = 1
    N[11, L - 1] = np.uint32(1 << 31)  # N = 2^2047 + 1
    Ns = ints(N)
    cases = [(0, 0), (0, 5), (1, 123), (Ns[3] - 1, 1 << 20), (Ns[4] - 1, (1 << 20) + 1), (7, (1 << bits) - 1),
             (Ns[6] - 2, 1), (3, 1 << (bits - 1)), (Ns[8] // 2, 65537), (2, Ns[9] - 1), (Ns[10] - 1, 3),
             (Ns[11] - 3, 12345678)]
    for k, (bv, ev) in enumerate(cases):
        base[k] = I.to_limbs(bv, L)
        exp[k] = I.to_limbs(ev, L)
    dN = mpb.to_device(N)
    Np, R2 = mpb.mont_batch_setup(dN, bits)
    for redc in REDC_STANDALONE:
        out = mpb.to_host(mpb.mont_batch_modexp_ct(dN, Np, R2, mpb.to_device(base), mpb.to_device(exp), bits,
                                                   redc=redc, algo=mpb.ALGO_RADIX52))
        for k, (bv, ev) in enumerate(cases):
            assert I.from_limbs(out[k]) == pow(bv, ev, Ns[k]), (redc, k)


@pytest.mark.parametrize("redc", REDC_STANDALONE)
@pytest.mark.parametrize("count", [1, 129, 700])
def test_modexp_hybrid(mpb, count, redc):
    """MPB_ALGO_HYBRID: one launch, 32-bit IMAD CTAs and radix-2^52 FP64 CTAs on disjoint operand
    ranges (counts below one CTA, across the split, and with several CTA groups); every operand
    equals the 32-bit path's result and, on a sample, the oracle."""
    bits = 2048
    N, base, exp = I.modexp_inputs(config=3, count=count, bits=bits, dataset=count)
    dN, dB, dE = (mpb.to_device(x) for x in (N, base, exp))
    Np, R2 = mpb.mont_batch_setup(dN, bits)
    out = mpb.mont_batch_modexp_ct(dN, Np, R2, dB, dE, bits, 5, redc=redc, algo=mpb.ALGO_HYBRID)
    ref32 = mpb.mont_batch_modexp_ct(dN, Np, R2, dB, dE, bits, 5, redc=redc, algo=mpb.ALGO_SCHOOLBOOK)
    assert torch.equal(out, ref32)
    h = mpb.to_host(out)
    idx = sorted({0, count // 3, count // 2, count - 1})
    assert np.array_equal(h[idx], O.batch_modexp(base[idx], exp[idx], bits, N[idx]))


@pytest.mark.parametrize("count,window", [(1, 5), (37, 5), (300, 4), (33, 1), (33, 6)])
def test_modexp_radix52_cios_register_kernel(mpb, count, window):
    """RADIX52 + CIOS at 1024 bits: the register-resident radix-2^52 CIOS kernel (mp_dfma_reg.cuh,
    lazy FP64-split accumulators in registers) against the oracle, with edge operands."""
    bits = 1024
    L = I.limbs_for_bits(bits)
    N, base, exp = I.modexp_inputs(config=1, count=count, bits=bits, dataset=500 + count + window)
    if count >= 12:
        N[0] = np.uint32(0xFFFFFFFF)
        N[1] = 0
        N[1, 0] = 1
        N[1, L - 1] = np.uint32(1 << 31)
        base[2] = 0
        exp[2] = 0
        base[3] = 0
        base[4] = 0
        base[4, 0] = 1
        exp[5] = np.uint32(0xFFFFFFFF)
        base[6] = I.to_limbs(I.from_limbs(N[6]) - 1, L)
    dN = mpb.to_device(N)
    Np, R2 = mpb.mont_batch_setup(dN, bits)
    out = mpb.to_host(mpb.mont_batch_modexp_ct(dN, Np, R2, mpb.to_device(base), mpb.to_device(exp), bits,
                                               window=window, redc=mpb.REDC_CIOS, algo=mpb.ALGO_RADIX52))
    assert np.array_equal(out, O.batch_modexp(base, exp, bits, N))


def test_modexp_radix52_rejects_unsupported(mpb):
    bits = 700
    N, base, exp = I.modexp_inputs(config=1, count=4, bits=bits)
    dN = mpb.to_device(N)
    Np, R2 = mpb.mont_batch_setup(dN, bits)
    with pytest.raises(ValueError):
        mpb.mont_batch_modexp_ct(dN, Np, R2, mpb.to_device(base), mpb.to_device(exp), bits,
                                 algo=mpb.ALGO_RADIX52)


def test_fault_injection_negative_control(mpb):
    """Negative control of the parity harness: the comparison that passes on the kernel's
    output must fail when one bit of one output limb is flipped -- in the element-wise oracle
    comparison, in the truncated == full whole-batch comparison, and in the slicing-independent
    digest config 5 prints."""
    from paper_2410_18129_b200 import shard

    bits, count = 1024, 33
    N, base, exp = I.modexp_inputs(config=3, count=count, bits=bits, dataset=99)
    dN = mpb.to_device(N)
    Np, R2 = mpb.mont_batch_setup(dN, bits)
    dB, dE = mpb.to_device(base), mpb.to_device(exp)
    out_t = mpb.mont_batch_modexp_ct(dN, Np, R2, dB, dE, bits, 5, redc=1)
    out_f = mpb.mont_batch_modexp_ct(dN, Np, R2, dB, dE, bits, 5, redc=0)
    ref = O.batch_modexp(base, exp, bits, N)
    h = mpb.to_host(out_t)
    assert np.array_equal(h, ref) and torch.equal(out_t, out_f)
    rng = np.random.default_rng(7)
    for _ in range(8):
        k, i, b = int(rng.integers(count)), int(rng.integers(h.shape[1])), int(rng.integers(32))
        bad = h.copy()
        bad[k, i] ^= np.uint32(1 << b)
        assert not np.array_equal(bad, ref)
        assert shard.digest_combine([shard.digest_part(bad, 0)]) != shard.digest_combine([shard.digest_part(ref, 0)])
        flipped = out_t.clone()
        flipped[i // 4, k, i % 4] ^= (1 << b) if b < 31 else -(1 << 31)
        assert not torch.equal(flipped, out_f)


# -------------------------------------------------- full-size, sampled checks
@pytest.mark.slow
def test_config3_full_batch_sampled(mpb):
    """Config 3 at its full size (2048-bit, 2^18, w=5), in the launch configuration bench.py times:
    a seeded sample of outputs against the oracle, and truncated == full on the whole batch."""
    bits, count = 2048, 1 << 18
    N, base, exp = I.modexp_inputs(config=3, count=count, bits=bits)
    dN, dB, dE = (mpb.to_device(x) for x in (N, base, exp))
    Np, R2 = mpb.mont_batch_setup(dN, bits)
    ws = mpb.modexp_workspace(count, bits, 5)
    out_t = mpb.mont_batch_modexp_ct(dN, Np, R2, dB, dE, bits, 5, redc=1, ws=ws)
    out_f = mpb.mont_batch_modexp_ct(dN, Np, R2, dB, dE, bits, 5, redc=0, ws=ws)
    assert torch.equal(out_t, out_f)
    out_c = mpb.mont_batch_modexp_ct(dN, Np, R2, dB, dE, bits, 5, redc=2, ws=ws)
    assert torch.equal(out_t, out_c)
    h = mpb.to_host(out_t)
    idx = np.random.default_rng(3).choice(count, size=48, replace=False)
    idx = np.concatenate([idx, [0, count - 1]])
    ref = O.batch_modexp(base[idx], exp[idx], bits, N[idx])
    assert np.array_equal(h[idx], ref)


@pytest.mark.slow
@pytest.mark.parametrize("bits", [1024, 2048, 3072, 4096])
def test_config2_full_batch_sampled(mpb, bits):
    """Config 2 at its full size (2^20 per size): MontMul and MontSqr, the three REDC modes equal
    on the whole batch, a seeded sample against the oracle."""
    count = 1 << 20
    N, a, b = I.montmul_inputs(config=2, count=count, bits=bits)
    dN, da, db = (mpb.to_device(x) for x in (N, a, b))
    Np, _ = mpb.mont_batch_setup(dN, bits)
    ws = mpb.mont_workspace(count, bits)
    idx = np.concatenate([np.random.default_rng(bits).choice(count, size=12, replace=False), [0, count - 1]])
    for op in ("mul", "sqr"):
        outs = []
        for redc in REDC:
            if op == "mul":
                outs.append(mpb.mont_batch_mul(da, db, dN, Np, bits, redc=redc, ws=ws))
            else:
                outs.append(mpb.mont_batch_sqr(da, dN, Np, bits, redc=redc, ws=ws))
        assert all(torch.equal(outs[0], o) for o in outs[1:]), op
        h = mpb.to_host(outs[0])
        ref = O.batch_montmul(a[idx], (b if op == "mul" else a)[idx], N[idx])
        assert np.array_equal(h[idx], ref), op


@pytest.mark.slow
def test_config4_full_batch_sampled(mpb):
    """Config 4 at its full size (2^16): 4096-bit modexp with truncated / full / CIOS REDC and with
    2-level Karatsuba products all equal on the whole batch; 4108 bits (L = 132, C = 12) sampled."""
    count = 1 << 16
    for bits, modes in ((4096, [(1, 1), (0, 1), (2, 1), (1, 3)]), (4108, [(1, 1)])):
        N, base, exp = I.modexp_inputs(config=4, count=count, bits=bits)
        dN, dB, dE = (mpb.to_device(x) for x in (N, base, exp))
        Np, R2 = mpb.mont_batch_setup(dN, bits)
        outs = [mpb.mont_batch_modexp_ct(dN, Np, R2, dB, dE, bits, 5, redc=r, algo=alg) for r, alg in modes]
        assert all(torch.equal(outs[0], o) for o in outs[1:]), bits
        h = mpb.to_host(outs[0])
        idx = np.concatenate([np.random.default_rng(bits).choice(count, size=4, replace=False), [0, count - 1]])
        assert np.array_equal(h[idx], O.batch_modexp(base[idx], exp[idx], bits, N[idx])), bits
        del dN, dB, dE, Np, R2, outs
        torch.cuda.empty_cache()


@pytest.mark.slow
def test_config5_full_batch_sampled(mpb):
    """Config 5 at its full size (2^22 2048-bit modexps): eight contiguous slices (the 8-GPU plan,
    run here as logical shards on one device) reproduce the whole-batch result byte for byte, and
    a random 4096-element subset matches the oracle (BASELINE config 5)."""
    from paper_2410_18129_b200 import shard

    bits, count = 2048, 1 << 22
    N, base, exp = I.modexp_inputs(config=5, count=count, bits=bits)
    whole = shard.modexp_devices(N, base, exp, bits, devices=[0])
    sliced = shard.modexp_devices(N, base, exp, bits, devices=[0] * 8)
    assert np.array_equal(whole, sliced)
    idx = np.random.default_rng(5).choice(count, size=4096, replace=False)
    assert np.array_equal(whole[idx], O.batch_modexp(base[idx], exp[idx], bits, N[idx]))


@pytest.mark.parametrize("bits", [8192, 16384])
def test_products_at_maximum_size(mpb, bits):
    """The largest supported operands (L = 256 and 512 limbs): schoolbook products and
    Montgomery multiplication / squaring in all REDC modes against the oracle."""
    count = 33
    a, b = I.mul_inputs(config=4, count=count, bits=bits)
    da, db = mpb.to_device(a), mpb.to_device(b)
    c = mpb.to_host(mpb.mp_batch_mul(da, db, bits, 1))
    A, B = ints(a), ints(b)
    for k in range(0, count, 4):
        assert I.from_limbs(c[k]) == O.mul(A[k], B[k]), k
    N, x, y = I.montmul_inputs(config=2, count=count, bits=bits)
    dN, dx, dy = (mpb.to_device(v) for v in (N, x, y))
    Np, _ = mpb.mont_batch_setup(dN, bits)
    idx = list(range(0, count, 8))
    ref_m = O.batch_montmul(x[idx], y[idx], N[idx])
    ref_s = O.batch_montmul(x[idx], x[idx], N[idx])
    for redc in REDC:
        assert np.array_equal(mpb.to_host(mpb.mont_batch_mul(dx, dy, dN, Np, bits, redc=redc))[idx], ref_m), redc
        assert np.array_equal(mpb.to_host(mpb.mont_batch_sqr(dx, dN, Np, bits, redc=redc))[idx], ref_s), redc


# ------------------------------------------------------------- ABI errors
def test_abi_errors_and_noop(mpb):
    bits = 1024
    N, a, b = I.montmul_inputs(config=2, count=4, bits=bits)
    dN, da = mpb.to_device(N), mpb.to_device(a)
    Np, R2 = mpb.mont_batch_setup(dN, bits)
    with pytest.raises(ValueError):
        mpb.mont_batch_modexp_ct(dN, Np, R2, da, da, bits, window=7)
    with pytest.raises(ValueError):
        mpb.mont_batch_mul(da, da, dN, Np, bits, redc=5)
    with pytest.raises(ValueError):
        mpb.mp_batch_mul(da, da, 20000)  # beyond the 16384-bit maximum
    with pytest.raises(ValueError):  # CIOS has no stand-alone REDC form
        mpb.mont_batch_redc(mpb.to_device(np.zeros((4, 64), np.uint32)), dN, Np, bits, redc=2)
    with pytest.raises(ValueError):  # CIOS interleaves schoolbook rows: no Karatsuba
        mpb.mont_batch_modexp_ct(dN, Np, R2, da, da, bits, redc=2, algo=2)
    assert not mpb.supported(20000) and mpb.supported(700) and mpb.supported(2048) and mpb.supported(4108)
    # count == 0 is a no-op
    z = mpb.empty_sliced(32, 0)
    assert mpb.mp_batch_mul(z, z, bits).shape == (16, 0, 4)


def test_sharded_slices_match_whole_batch(mpb):
    """G logical shards on one device (one stream each) reproduce the whole-batch result
    byte for byte (SURVEY 8(c) multi-GPU row; the real 1/2/4/8-GPU runs slice the same way)."""
    from paper_2410_18129_b200 import shard

    bits, count = 1024, 1000
    N, base, exp = I.modexp_inputs(config=5, count=count, bits=bits)
    whole = shard.modexp_devices(N, base, exp, bits, devices=[0])
    for G in (2, 3, 8):
        assert np.array_equal(shard.modexp_devices(N, base, exp, bits, devices=[0] * G), whole)
    idx = [0, 1, 499, 998, 999]
    assert np.array_equal(whole[idx], O.batch_modexp(base[idx], exp[idx], bits, N[idx]))


@pytest.mark.parametrize("algo", [2, 3])
@pytest.mark.parametrize("bits", [1536, 3072, 4096, 4108, 5120])
def test_modexp_karatsuba_products(mpb, bits, algo):
    """Karatsuba (1 and 2 levels) in the product phase of every MontMul/MontSqr."""
    count = 5
    N, base, exp = I.modexp_inputs(config=4, count=count, bits=bits)
    dN = mpb.to_device(N)
    Np, R2 = mpb.mont_batch_setup(dN, bits)
    out = mpb.to_host(mpb.mont_batch_modexp_ct(dN, Np, R2, mpb.to_device(base), mpb.to_device(exp), bits,
                                               window=5, algo=algo))
    assert np.array_equal(out, O.batch_modexp(base, exp, bits, N))


@pytest.mark.parametrize("algo", [2, 3])
def test_truncated_karatsuba_redc_crafted(mpb, algo):
    """The truncated-Karatsuba REDC (mp_kara.cuh kara_trunc_high, used by the Karatsuba
    exponentiation at 4096 bits) on inputs that force BOTH half-level Theorem-2 corrections
    (tests/adversarial.py t_kara_trunc, pinned in test_oracle): the crafted T stands in the R^2
    position, so the exponentiation's first operation REDC(R2) needs them.  Every operand equals
    the exact schedule and the schoolbook kernel's output on the same inputs."""
    bits, w, count = 4096, 5, 6
    L = I.limbs_for_bits(bits)
    H = L // 2
    R = 1 << (32 * L)
    N, base, exp = I.modexp_inputs(config=4, count=count, bits=bits, dataset=11)
    N[:, H] &= np.uint32(0xFFFFFFFE)  # N1 even, N0 odd: |N0 - N1| odd (the construction needs it)
    Ns = ints(N)
    Bs = [b % n for b, n in zip(ints(base), Ns)]
    base = I.ints_to_array(Bs, L)
    Es = ints(exp)
    rng = random.Random(4096 + algo)
    rho = []
    for k, n in enumerate(Ns):
        t = t_kara_trunc(rng, n, L, k % 3, (k + 1) % 3, below_n=True)
        assert t is not None
        rho.append(t)
    dN, dB, dE = (mpb.to_device(x) for x in (N, base, exp))
    Np, _ = mpb.mont_batch_setup(dN, bits)
    dR = mpb.to_device(I.ints_to_array(rho, L))
    out = mpb.to_host(mpb.mont_batch_modexp_ct(dN, Np, dR, dB, dE, bits, w, redc=mpb.REDC_TRUNCATED, algo=algo))
    ref = mpb.to_host(mpb.mont_batch_modexp_ct(dN, Np, dR, dB, dE, bits, w, redc=mpb.REDC_TRUNCATED,
                                               algo=mpb.ALGO_SCHOOLBOOK))
    assert np.array_equal(out, ref)
    for k in (0, count - 1):
        assert I.from_limbs(out[k]) == _schedule_modexp(Bs[k], Es[k], Ns[k], rho[k], L, bits, w), k


# ----------------------------------------------------------------- CRT-RSA (f4)
@functools.lru_cache(maxsize=None)
def _rsa_keys(bits: int, n_keys: int, seed: int):
    """RSA keys from oracle primes (exactly bits/2 bits each), e = 65537."""
    import math

    h = bits // 2
    keys = []
    for i in range(n_keys):
        while True:
            p, q = O.gen_prime(h, seed + 2 * i), O.gen_prime(h, seed + 2 * i + 1 + 7919)
            lam = (p - 1) * (q - 1) // math.gcd(p - 1, q - 1)
            if p != q and math.gcd(65537, lam) == 1:
                break
            seed += 104729
        d = O.inv_mod(65537, lam)
        keys.append((p, q, d, d % (p - 1), d % (q - 1), O.inv_mod(q, p)))
    return keys


@pytest.mark.parametrize("redc", REDC)
@pytest.mark.parametrize("bits", [512, 1024, 2048])
def test_rsa_crt(mpb, bits, redc):
    """Batched CRT-RSA private-key operation vs the oracle's CRT route and the full-size power
    c^d mod n, with the edge ciphertexts 0, 1, n-1 and multiples of p and q; ragged count."""
    n_keys, count = 5, 133
    keys = _rsa_keys(bits, n_keys, seed=bits * 31 + 7)
    L, Lh = I.limbs_for_bits(bits), I.limbs_for_bits(bits // 2)
    rng = random.Random(bits + redc)
    rows = []
    for k in range(count):
        p, q, d, dp, dq, qi = keys[k % n_keys]
        n = p * q
        c = [0, 1, n - 1, 3 * p, 5 * q][k] if k < 5 else rng.randrange(n)
        rows.append((c, p, q, d, dp, dq, qi))
    arrs = [I.ints_to_array([r[0] for r in rows], L)] + [I.ints_to_array([r[j] for r in rows], Lh) for j in (1, 2, 4, 5, 6)]
    dc, dp_, dq_, ddp, ddq, dqi = (mpb.to_device(a) for a in arrs)
    m = mpb.to_host(mpb.rsa_batch_crt_ct(dc, dp_, dq_, ddp, ddq, dqi, bits, window=5, redc=redc))
    for k, (c, p, q, d, dp, dq, qi) in enumerate(rows):
        got = I.from_limbs(m[k])
        if k < 12:
            assert got == O.rsa_crt(c, p, q, dp, dq, qi, Lh, bits // 2), k
        assert got == pow(c, d, p * q), k


def test_rsa_crt_round_trip(mpb):
    """(msg^e)^d = msg for 2048-bit keys: the public operation by the oracle, the private one on the GPU."""
    bits, count = 2048, 6
    keys = _rsa_keys(bits, 3, seed=99)
    L, Lh = I.limbs_for_bits(bits), I.limbs_for_bits(bits // 2)
    rng = random.Random(4)
    msgs, cts, ks = [], [], []
    for k in range(count):
        p, q, d, dp, dq, qi = keys[k % 3]
        msg = rng.randrange(p * q)
        msgs.append(msg)
        cts.append(O.modexp(msg, 65537, p * q, L, ebits=17))
        ks.append(keys[k % 3])
    arrs = [I.ints_to_array(cts, L)] + [I.ints_to_array([kk[j] for kk in ks], Lh) for j in (0, 1, 3, 4, 5)]
    m = mpb.to_host(mpb.rsa_batch_crt_ct(*(mpb.to_device(a) for a in arrs), bits))
    assert [I.from_limbs(r) for r in m] == msgs


# ------------------------------------------------------------------ edge cases
def test_empty_and_single_operand_batches(mpb):
    """count = 0 is a no-op on every entry point; count = 1 is exact."""
    bits = 1024
    L = I.limbs_for_bits(bits)
    z = mpb.empty_sliced(L, 0)
    assert mpb.mont_batch_mul(z, z, z, z, bits).shape == (L // 4, 0, 4)
    assert mpb.mont_batch_sqr(z, z, z, bits).shape == (L // 4, 0, 4)
    assert mpb.mont_batch_modexp_ct(z, z, z, z, z, bits).shape == (L // 4, 0, 4)
    zh = mpb.empty_sliced(L // 2, 0)
    assert mpb.rsa_batch_crt_ct(z, zh, zh, zh, zh, zh, bits).shape == (L // 4, 0, 4)
    N, base, exp = I.modexp_inputs(config=3, count=1, bits=bits)
    dN = mpb.to_device(N)
    Np, R2 = mpb.mont_batch_setup(dN, bits)
    for redc in REDC:
        out = mpb.to_host(mpb.mont_batch_modexp_ct(dN, Np, R2, mpb.to_device(base), mpb.to_device(exp), bits,
                                                   redc=redc))
        assert np.array_equal(out, O.batch_modexp(base, exp, bits, N)), redc


@pytest.mark.parametrize("redc", REDC)
def test_tiny_moduli(mpb, redc):
    """Degenerate small moduli at the smallest width (bits = 32, L = 4, C = 4): N = 3, 5, 7, 2^31+1,
    2^32-1 with every base below N (or a spread of them) and assorted exponents."""
    bits = 32
    L = I.limbs_for_bits(bits)
    rows = []
    for n in (3, 5, 7, (1 << 31) + 1, (1 << 32) - 1):
        for b in ([0, 1, 2] if n <= 7 else [0, 1, 2, n - 1, n // 3]):
            for e in (0, 1, 2, 3, (1 << 32) - 1, 0x80000001):
                rows.append((n, b % n, e))
    N = I.ints_to_array([r[0] for r in rows], L)
    B = I.ints_to_array([r[1] for r in rows], L)
    E = I.ints_to_array([r[2] for r in rows], L)
    dN = mpb.to_device(N)
    Np, R2 = mpb.mont_batch_setup(dN, bits)
    out = mpb.to_host(mpb.mont_batch_modexp_ct(dN, Np, R2, mpb.to_device(B), mpb.to_device(E), bits, window=3,
                                               redc=redc))
    for k, (n, b, e) in enumerate(rows):
        assert I.from_limbs(out[k]) == O.modexp(b, e, n, L, ebits=bits), (n, b, e)


# ------------------------------------------------ one-thread vs two-lane operands
_COOP_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, %r)
from paper_2410_18129_b200 import inputs as I, mpb
out = {}
for bits, count, w, redc in ((1024, 9, 5, 1), (2048, 5, 4, 0), (3072, 4, 5, 1), (4096, 3, 5, 0), (4108, 2, 3, 1)):
    N, base, exp = I.modexp_inputs(config=4, count=count, bits=bits)
    dN = mpb.to_device(N)
    Np, R2 = mpb.mont_batch_setup(dN, bits)
    o = mpb.to_host(mpb.mont_batch_modexp_ct(dN, Np, R2, mpb.to_device(base), mpb.to_device(exp), bits, window=w,
                                             redc=redc))
    print(bits, count, w, redc, o.tobytes().hex())
"""


@pytest.mark.parametrize("coop", ["0", "0-nowave", "1", "4", "8", "tma"])
def test_modexp_one_thread_and_two_lane_kernels(mpb, coop):
    """All exponentiation kernels, forced by MPB_COOP / MPB_TMA in a subprocess (the policy is read
    once per process): one thread per operand (0), two / four / eight lanes per operand (1, 4, 8:
    mp_coop.cuh, shuffle-summed block-column windows) and one thread per operand with per-warp TMA
    operand tiles (tma), 1024..4108 bits, truncated and full REDC, against the oracle."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    if coop == "tma":
        env = dict(os.environ, MPB_COOP="0", MPB_TMA="1")
    elif coop == "0-nowave":  # one thread per operand, 128-thread CTAs (no one-wave instances)
        env = dict(os.environ, MPB_COOP="0", MPB_ONEWAVE="0")
    else:
        env = dict(os.environ, MPB_COOP=coop)
    res = subprocess.run([sys.executable, "-c", _COOP_SCRIPT % root], env=env, capture_output=True, text=True,
                         timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [l for l in res.stdout.splitlines() if l.strip()]
    assert len(lines) == 5
    for line in lines:
        bits, count, w, redc, hx = line.split()
        bits, count = int(bits), int(count)
        L = I.limbs_for_bits(bits)
        got = np.frombuffer(bytes.fromhex(hx), dtype=np.uint32).reshape(count, L)
        N, base, exp = I.modexp_inputs(config=4, count=count, bits=bits)
        assert np.array_equal(got, O.batch_modexp(base, exp, bits, N)), (bits, coop)


_ONEWAVE_SCRIPT = r"""
import sys, hashlib, numpy as np
sys.path.insert(0, %r)
from paper_2410_18129_b200 import inputs as I, mpb
for bits, count, redc in %r:
    N, base, exp = I.modexp_inputs(config=4, count=count, bits=bits)
    dN = mpb.to_device(N)
    Np, R2 = mpb.mont_batch_setup(dN, bits)
    o = mpb.to_host(mpb.mont_batch_modexp_ct(dN, Np, R2, mpb.to_device(base), mpb.to_device(exp), bits, window=5,
                                             redc=redc))
    print(bits, count, redc, hashlib.sha256(o.tobytes()).hexdigest())
"""

# (bits, count, redc): batches of one wave or less, so the one-CTA-per-SM instances run with
# 64..448-thread CTAs and ragged last CTAs (count not a multiple of the CTA size)
_ONEWAVE_CASES = ((1024, 10007, 1), (2048, 20011, 1), (2048, 4740, 0), (2048, 9000, 2), (3072, 30001, 1),
                  (4096, 60001, 1), (4096, 12001, 0), (4108, 50001, 1), (4108, 65536, 0))


def test_modexp_onewave_instances(mpb):
    """One-wave batches run as one CTA of up to 384 / 448 threads per SM (inst_W384.cu / inst_W448.cu,
    DESIGN.md 5.3c): every output equals the 128-thread kernels' (MPB_ONEWAVE=0, a subprocess: the
    policy is read once per process) on the whole batch, and a sample including the first and last
    operand equals the oracle."""
    import hashlib
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = subprocess.run([sys.executable, "-c", _ONEWAVE_SCRIPT % (root, _ONEWAVE_CASES)],
                         env=dict(os.environ, MPB_ONEWAVE="0"), capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stderr[-2000:]
    ref = {tuple(map(int, l.split()[:3])): l.split()[3] for l in res.stdout.splitlines() if l.strip()}
    assert len(ref) == len(_ONEWAVE_CASES)
    for bits, count, redc in _ONEWAVE_CASES:
        N, base, exp = I.modexp_inputs(config=4, count=count, bits=bits)
        dN = mpb.to_device(N)
        Np, R2 = mpb.mont_batch_setup(dN, bits)
        out = mpb.to_host(mpb.mont_batch_modexp_ct(dN, Np, R2, mpb.to_device(base), mpb.to_device(exp), bits,
                                                   window=5, redc=redc))
        assert hashlib.sha256(out.tobytes()).hexdigest() == ref[(bits, count, redc)], (bits, count, redc)
        idx = np.array(sorted({0, count - 1, *np.random.default_rng(count).choice(count, 3, replace=False)}))
        assert np.array_equal(out[idx], O.batch_modexp(base[idx], exp[idx], bits, N[idx])), (bits, count, redc)


_RTR_OPS_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, %r)
from paper_2410_18129_b200 import inputs as I, mpb
N, x, y = I.montmul_inputs(config=2, count=301, bits=1024)
dN, dx, dy = (mpb.to_device(v) for v in (N, x, y))
Np, _ = mpb.mont_batch_setup(dN, 1024)
print(mpb.to_host(mpb.mont_batch_mul(dx, dy, dN, Np, 1024, 1)).tobytes().hex())
print(mpb.to_host(mpb.mont_batch_sqr(dx, dN, Np, 1024, 1)).tobytes().hex())
"""


def test_mont_ops_register_truncated_kernel(mpb):
    """The opt-in stand-alone register-resident truncated MontMul / MontSqr at 1024 bits
    (k_mont_mul_rtr, MPB_REG_TRUNC=1 in a subprocess) against the oracle on every operand."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = subprocess.run([sys.executable, "-c", _RTR_OPS_SCRIPT % root], env=dict(os.environ, MPB_REG_TRUNC="1"),
                         capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    mul_hex, sqr_hex = [l for l in res.stdout.splitlines() if l.strip()]
    N, x, y = I.montmul_inputs(config=2, count=301, bits=1024)
    L = I.limbs_for_bits(1024)
    got_mul = np.frombuffer(bytes.fromhex(mul_hex), dtype=np.uint32).reshape(301, L)
    got_sqr = np.frombuffer(bytes.fromhex(sqr_hex), dtype=np.uint32).reshape(301, L)
    assert np.array_equal(got_mul, O.batch_montmul(x, y, N))
    assert np.array_equal(got_sqr, O.batch_montmul(x, x, N))


# ----------------------------------------------------------------------- fuzz
def test_fuzz_shapes(mpb):
    """Seeded random shapes: widths 64..8192 bits (every block size C = 16, 12, 8, 4 and odd block
    counts), ragged counts, windows 1..6, all REDC modes and product algorithms, against the
    oracle.  Sizes are bounded so the oracle side stays within seconds."""
    rng = random.Random(20241018)
    cases = 0
    for _ in range(24):
        bits = rng.choice([64, 96, 160, 288, 416, 544, 700, 1056, 1312, 1600, 2112, 2720, 3200, 4000, 5000, 8192])
        L = I.limbs_for_bits(bits)
        count = rng.randint(1, 70)
        w = rng.randint(1, 6)
        redc = rng.choice(REDC)
        algo = rng.choice([0, 1, 2, 3]) if redc != 2 else rng.choice([0, 1])
        N, base, exp = I.modexp_inputs(config=3, count=count, bits=bits, dataset=cases)
        dN = mpb.to_device(N)
        Np, R2 = mpb.mont_batch_setup(dN, bits)
        idx = sorted(rng.sample(range(count), min(count, 3 if bits <= 2048 else 1)))
        a = mpb.to_device(base)
        mm = mpb.to_host(mpb.mont_batch_mul(a, a, dN, Np, bits, redc=redc))
        assert np.array_equal(mm[idx], O.batch_montmul(base[idx], base[idx], N[idx])), (bits, count, redc)
        if bits <= 4000:
            out = mpb.to_host(mpb.mont_batch_modexp_ct(dN, Np, R2, a, mpb.to_device(exp), bits, window=w, redc=redc,
                                                       algo=algo))
            assert np.array_equal(out[idx], O.batch_modexp(base[idx], exp[idx], bits, N[idx])), \
                (bits, count, w, redc, algo)
        prod = mpb.to_host(mpb.mp_batch_mul(a, a, bits, rng.choice([1, 2, 3])))
        for k in idx:
            assert I.from_limbs(prod[k]) == I.from_limbs(base[k]) ** 2, (bits, k)
        cases += 1
    assert cases == 24
