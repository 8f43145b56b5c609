"""ctypes wrapper around oracle/liboracle.so -- the plain CPU oracle.

TEST INFRASTRUCTURE ONLY: only tests/, ``__graft_entry__.smoke()`` and
bench.py's ``cpu_baseline`` / ``--impl reference`` leg may import this
package.  The product path (``paper_2410_18129_b200``) never imports it and
shares no code with it; both sides take their inputs from
``paper_2410_18129_b200.inputs`` (seeded generators and int<->limb plumbing,
no arithmetic of the method).

Every function here is a thin marshalling layer over oracle/oracle.c; the
citations for what each computes are in oracle/oracle.h.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from paper_2410_18129_b200.inputs import from_limbs, to_limbs

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

_u32p = ctypes.POINTER(ctypes.c_uint32)


def build(force: bool = False) -> str:
    """Compile oracle.c into liboracle.so with gcc (plain -O2, no vector tricks)."""
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(
            ["gcc", "-O2", "-std=c99", "-fPIC", "-shared", "-Wall", "-o", _LIB_PATH, src, "-lpthread"]
        )
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        i, sz, u64 = ctypes.c_int, ctypes.c_size_t, ctypes.c_uint64
        sigs = {
            "o_mul": (None, [_u32p, i, _u32p, i, _u32p]),
            "o_sqr": (None, [_u32p, i, _u32p]),
            "o_divmod": (i, [_u32p, i, _u32p, i, _u32p, _u32p]),
            "o_inv_mod": (i, [_u32p, i, _u32p, i, _u32p]),
            "o_egcd": (i, [_u32p, _u32p, i, _u32p, _u32p, _u32p]),
            "o_setup": (i, [_u32p, i, _u32p, _u32p]),
            "o_montmul": (i, [_u32p, _u32p, _u32p, i, _u32p]),
            "o_redc": (i, [_u32p, _u32p, i, _u32p]),
            "o_modexp": (i, [_u32p, _u32p, i, _u32p, i, _u32p]),
            "o_is_probable_prime": (i, [_u32p, i, i, u64]),
            "o_gen_prime": (i, [i, u64, _u32p]),
            "o_montred_classic": (i, [_u32p, _u32p, _u32p, i, _u32p]),
            "o_montred_truncated": (i, [_u32p, _u32p, _u32p, i, _u32p, _u32p]),
            "o_montmul_cios": (i, [_u32p, _u32p, _u32p, ctypes.c_uint32, i, _u32p]),
            "o_rsa_crt": (i, [_u32p, _u32p, _u32p, _u32p, _u32p, _u32p, i, i, _u32p]),
            "o_batch_modexp": (i, [_u32p, _u32p, i, _u32p, i, _u32p, sz, i]),
            "o_batch_montmul": (i, [_u32p, _u32p, _u32p, i, _u32p, sz, i]),
        }
        for name, (res, args) in sigs.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _arr(x: int, n: int) -> np.ndarray:
    return np.ascontiguousarray(to_limbs(x, n), dtype=np.uint32)


def _p(a: np.ndarray):
    assert a.dtype == np.uint32 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_u32p)


def _limbs_for(*xs: int) -> int:
    return max(1, max((int(x).bit_length() + 31) // 32 for x in xs))


# ------------------------------------------------------------ int interface
def mul(a: int, b: int) -> int:
    na, nb = _limbs_for(a), _limbs_for(b)
    A, B, C = _arr(a, na), _arr(b, nb), np.zeros(na + nb, np.uint32)
    lib().o_mul(_p(A), na, _p(B), nb, _p(C))
    return from_limbs(C)


def sqr(a: int) -> int:
    n = _limbs_for(a)
    A, C = _arr(a, n), np.zeros(2 * n, np.uint32)
    lib().o_sqr(_p(A), n, _p(C))
    return from_limbs(C)


def divmod_(a: int, b: int) -> tuple[int, int]:
    na, nb = _limbs_for(a), _limbs_for(b)
    A, B = _arr(a, na), _arr(b, nb)
    Q, R = np.zeros(na, np.uint32), np.zeros(nb, np.uint32)
    if lib().o_divmod(_p(A), na, _p(B), nb, _p(Q), _p(R)) != 0:
        raise ZeroDivisionError("o_divmod: division by zero")
    return from_limbs(Q), from_limbs(R)


def inv_mod(a: int, m: int) -> int:
    n = _limbs_for(a, m)
    A, M, X = _arr(a, n), _arr(m, n), np.zeros(n, np.uint32)
    if lib().o_inv_mod(_p(A), n, _p(M), n, _p(X)) != 0:
        raise ValueError("not invertible")
    return from_limbs(X)


def egcd(a: int, b: int) -> tuple[int, int, int]:
    """(x, y, g) with a*x - b*y = g = gcd(a, b)."""
    n = _limbs_for(a, b)
    A, B = _arr(a, n), _arr(b, n)
    X, Y, G = (np.zeros(n, np.uint32) for _ in range(3))
    if lib().o_egcd(_p(A), _p(B), n, _p(X), _p(Y), _p(G)) != 0:
        raise ValueError("egcd failed")
    return from_limbs(X), from_limbs(Y), from_limbs(G)


def setup(N: int, L: int) -> tuple[int, int]:
    """(N', R^2 mod N) for R = 2^(32L)."""
    Nn, NP, R2 = _arr(N, L), np.zeros(L, np.uint32), np.zeros(L, np.uint32)
    if lib().o_setup(_p(Nn), L, _p(NP), _p(R2)) != 0:
        raise ValueError("N not invertible mod R")
    return from_limbs(NP), from_limbs(R2)


def montmul(a: int, b: int, N: int, L: int) -> int:
    A, B, Nn, C = _arr(a, L), _arr(b, L), _arr(N, L), np.zeros(L, np.uint32)
    if lib().o_montmul(_p(A), _p(B), _p(Nn), L, _p(C)) != 0:
        raise ValueError("o_montmul failed")
    return from_limbs(C)


def redc(T: int, N: int, L: int) -> int:
    Tt, Nn, C = _arr(T, 2 * L), _arr(N, L), np.zeros(L, np.uint32)
    if lib().o_redc(_p(Tt), _p(Nn), L, _p(C)) != 0:
        raise ValueError("o_redc failed")
    return from_limbs(C)


def modexp(base: int, e: int, N: int, L: int, ebits: int | None = None) -> int:
    if ebits is None:
        ebits = max(1, int(e).bit_length())
    eL = (ebits + 31) // 32
    B, E, Nn, Y = _arr(base, L), _arr(e, eL), _arr(N, L), np.zeros(L, np.uint32)
    if lib().o_modexp(_p(B), _p(E), ebits, _p(Nn), L, _p(Y)) != 0:
        raise ValueError("o_modexp failed")
    return from_limbs(Y)


def is_probable_prime(n: int, rounds: int = 40, seed: int = 1) -> bool:
    L = _limbs_for(n)
    return bool(lib().o_is_probable_prime(_p(_arr(n, L)), L, rounds, seed))


def gen_prime(bits: int, seed: int) -> int:
    L = (bits + 31) // 32
    out = np.zeros(L, np.uint32)
    if lib().o_gen_prime(bits, seed, _p(out)) != 0:
        raise ValueError("bits too small")
    return from_limbs(out)


def montred_classic(T: int, N: int, Nprime: int, L: int) -> int:
    Tt, Nn, NP, C = _arr(T, 2 * L), _arr(N, L), _arr(Nprime, L), np.zeros(L + 1, np.uint32)
    if lib().o_montred_classic(_p(Tt), _p(Nn), _p(NP), L, _p(C)) != 0:
        raise ValueError("T + qN not divisible by R")
    return from_limbs(C)


def montred_truncated(T: int, N: int, Nprime: int, L: int) -> tuple[int, int]:
    """(C, qnhat) of alg:trunc_montred under the SURVEY A6/A7 reading."""
    Tt, Nn, NP = _arr(T, 2 * L), _arr(N, L), _arr(Nprime, L)
    C, Q = np.zeros(L + 1, np.uint32), np.zeros(L + 1, np.uint32)
    lib().o_montred_truncated(_p(Tt), _p(Nn), _p(NP), L, _p(C), _p(Q))
    return from_limbs(C), from_limbs(Q)


def montmul_cios(a: int, b: int, N: int, n0p: int, L: int) -> int:
    """alg:8BlockMontRed word by word: a*b*R^-1 mod N up to one N (< 2N)."""
    A, B, Nn, C = _arr(a, L), _arr(b, L), _arr(N, L), np.zeros(L + 1, np.uint32)
    if lib().o_montmul_cios(_p(A), _p(B), _p(Nn), n0p, L, _p(C)) != 0:
        raise ValueError("a low word of Y + q*N did not vanish")
    return from_limbs(C)


def rsa_crt(c: int, p: int, q: int, dp: int, dq: int, qinv: int, Lh: int, ebits: int) -> int:
    """CRT-RSA private-key operation (Garner), step by step: m = c^d mod pq."""
    m = np.zeros(2 * Lh, np.uint32)
    args = [_arr(c, 2 * Lh), _arr(p, Lh), _arr(q, Lh), _arr(dp, Lh), _arr(dq, Lh), _arr(qinv, Lh)]
    if lib().o_rsa_crt(*[_p(a) for a in args], Lh, ebits, _p(m)) != 0:
        raise ValueError("invalid CRT-RSA operands")
    return from_limbs(m)


# ---------------------------------------------------------- batch interface
def batch_modexp(base: np.ndarray, e: np.ndarray, ebits: int, N: np.ndarray, threads: int | None = None) -> np.ndarray:
    """Operand-major uint32 arrays: base, N (count, L); e (count, ceil(ebits/32))."""
    base, e, N = (np.ascontiguousarray(x, dtype=np.uint32) for x in (base, e, N))
    count, L = N.shape
    eL = (ebits + 31) // 32
    assert e.shape[0] == count and e.shape[1] >= eL
    e = np.ascontiguousarray(e[:, :eL])  # the limbs holding the ebits-bit exponent
    out = np.zeros((count, L), np.uint32)
    th = threads or os.cpu_count() or 1
    if lib().o_batch_modexp(_p(base), _p(e), ebits, _p(N), L, _p(out), count, th) != 0:
        raise ValueError("o_batch_modexp failed")
    return out


def batch_montmul(a: np.ndarray, b: np.ndarray, N: np.ndarray, threads: int | None = None) -> np.ndarray:
    a, b, N = (np.ascontiguousarray(x, dtype=np.uint32) for x in (a, b, N))
    count, L = N.shape
    out = np.zeros((count, L), np.uint32)
    th = threads or os.cpu_count() or 1
    if lib().o_batch_montmul(_p(a), _p(b), _p(N), L, _p(out), count, th) != 0:
        raise ValueError("o_batch_montmul failed")
    return out
