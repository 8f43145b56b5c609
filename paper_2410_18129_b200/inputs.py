"""Seeded synthetic inputs and int <-> limb plumbing.

This is the ONE module shared by the oracle side (oracle/, tests/) and the
CUDA side (the binding, bench.py).  It holds none of the method's arithmetic:
only random draws, bit masks, a limb-wise comparison for rejection sampling,
and format conversions.

Recipe: the paper measures on random
operands ("50 random data sets") and names no dataset, so these
synthetic draws *are* the workload family:
  * generator  numpy.random.Generator(PCG64(24101812900 + config + 1000*dataset))
  * N          `bits` uniform random bits, bit bits-1 and bit 0 forced (odd, exact length)
  * base, a, b uniform in [0, N) by rejection (redraw rows that are >= N)
  * exp        `bits` uniform random bits with bit bits-1 forced (full length)
All arrays are operand-major little-endian uint32 limbs, shape (count, L),
L = limbs_for_bits(bits) = 4*ceil(bits/128) (SURVEY 8 notation).
"""
from __future__ import annotations

import numpy as np

SEED_BASE = 24101812900


def limbs_for_bits(bits: int) -> int:
    """L = 4*ceil(bits/128): 32-bit limbs, a multiple of 4 (one uint4 per 4 limbs)."""
    if bits <= 0:
        raise ValueError("bits must be positive")
    return 4 * ((bits + 127) // 128)


def rng_for(config: int, dataset: int = 0) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(SEED_BASE + config + 1000 * dataset))


# ------------------------------------------------------------- conversions
def to_limbs(x: int, n: int) -> np.ndarray:
    x = int(x)
    if x < 0:
        raise ValueError("negative")
    if x >> (32 * n):
        raise ValueError(f"value does not fit in {n} limbs")
    return np.frombuffer(x.to_bytes(4 * n, "little"), dtype="<u4").astype(np.uint32)


def from_limbs(a) -> int:
    a = np.ascontiguousarray(np.asarray(a, dtype=np.uint32))
    return int.from_bytes(a.astype("<u4").tobytes(), "little")


def ints_to_array(xs, n: int) -> np.ndarray:
    out = np.zeros((len(xs), n), np.uint32)
    for k, x in enumerate(xs):
        out[k] = to_limbs(x, n)
    return out


def array_to_ints(arr) -> list[int]:
    arr = np.asarray(arr, dtype=np.uint32)
    return [from_limbs(row) for row in arr]


# ---------------------------------------------------------------- draws
def _random_bits(rng: np.random.Generator, count: int, bits: int, L: int) -> np.ndarray:
    x = rng.integers(0, 1 << 32, size=(count, L), dtype=np.uint64).astype(np.uint32)
    full, rem = divmod(bits, 32)
    if full < L:
        x[:, full + (1 if rem else 0):] = 0
        if rem:
            x[:, full] &= np.uint32((1 << rem) - 1)
    return x


def less_than(x: np.ndarray, N: np.ndarray) -> np.ndarray:
    """Row-wise x < N for operand-major limb arrays (compared from the top limb)."""
    diff = x != N
    any_diff = diff.any(axis=1)
    L = x.shape[1]
    top = L - 1 - np.argmax(diff[:, ::-1], axis=1)
    rows = np.arange(x.shape[0])
    return any_diff & (x[rows, top] < N[rows, top])


def gen_moduli(rng: np.random.Generator, count: int, bits: int, L: int | None = None) -> np.ndarray:
    L = L or limbs_for_bits(bits)
    N = _random_bits(rng, count, bits, L)
    N[:, (bits - 1) // 32] |= np.uint32(1 << ((bits - 1) % 32))
    N[:, 0] |= np.uint32(1)
    return N


def gen_below(rng: np.random.Generator, N: np.ndarray, bits: int) -> np.ndarray:
    """Uniform in [0, N) per row by rejection (acceptance >= 1/2 since N >= 2^(bits-1))."""
    count, L = N.shape
    out = _random_bits(rng, count, bits, L)
    bad = ~less_than(out, N)
    while bad.any():
        idx = np.nonzero(bad)[0]
        out[idx] = _random_bits(rng, len(idx), bits, L)
        bad[idx] = ~less_than(out[idx], N[idx])
    return out


def gen_exponents(rng: np.random.Generator, count: int, bits: int, L: int | None = None) -> np.ndarray:
    L = L or limbs_for_bits(bits)
    e = _random_bits(rng, count, bits, L)
    e[:, (bits - 1) // 32] |= np.uint32(1 << ((bits - 1) % 32))
    return e


def modexp_inputs(config: int, count: int, bits: int, dataset: int = 0):
    """(N, base, exp) for a modexp batch: shapes (count, L)."""
    rng = rng_for(config, dataset)
    L = limbs_for_bits(bits)
    N = gen_moduli(rng, count, bits, L)
    base = gen_below(rng, N, bits)
    exp = gen_exponents(rng, count, bits, L)
    return N, base, exp


CHUNK = 1 << 16  # operands per independently seeded chunk of a sliced global batch (config 5)


def modexp_inputs_range(config: int, start: int, stop: int, bits: int, chunk: int = CHUNK):
    """Operands [start, stop) of a global modexp batch drawn chunk by chunk: chunk c (operands
    c*chunk .. (c+1)*chunk-1) is modexp_inputs(config, chunk, bits, dataset=c).  A rank generates
    only the chunks its slice touches, and every slicing of the global batch sees the same operands
    (config 5: "generated once and sliced", G-invariance)."""
    if not 0 <= start <= stop:
        raise ValueError("need 0 <= start <= stop")
    L = limbs_for_bits(bits)
    parts = ([], [], [])
    for c in range(start // chunk, (stop + chunk - 1) // chunk):
        lo, hi = max(start, c * chunk) - c * chunk, min(stop, (c + 1) * chunk) - c * chunk
        for p, x in zip(parts, modexp_inputs(config, chunk, bits, dataset=c)):
            p.append(x[lo:hi])
    if not parts[0]:
        z = np.zeros((0, L), np.uint32)
        return z, z.copy(), z.copy()
    return tuple(np.concatenate(p) for p in parts)


def montmul_inputs(config: int, count: int, bits: int, dataset: int = 0):
    """(N, a, b) for a Montgomery multiply/square batch: shapes (count, L)."""
    rng = rng_for(config, dataset)
    L = limbs_for_bits(bits)
    N = gen_moduli(rng, count, bits, L)
    a = gen_below(rng, N, bits)
    b = gen_below(rng, N, bits)
    return N, a, b


def mul_inputs(config: int, count: int, bits: int, dataset: int = 0):
    """(a, b) uniform `bits`-bit operands for the plain batch multiply/square."""
    rng = rng_for(config, dataset)
    L = limbs_for_bits(bits)
    return _random_bits(rng, count, bits, L), _random_bits(rng, count, bits, L)
