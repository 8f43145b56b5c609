"""Adversarial inputs for the truncated REDC (SURVEY.md 8(c) "GPU truncated REDC" row).

Random T almost never exercises the exact carry correction of Theorem 2
(PAPER.md L473-542): it fires with probability ~2L/2^32.
These builders construct T = some 2L-limb value with T < N*R for the families

  alpha  c_add = 0:           T mod R = 0
  beta   the A6 trap:         T[0..L-2] = 0, T[L-1] != 0
  gamma  forced wrap:         q chosen so that S mod 2^32 = 2^32-1-k (k in 0,1,2),
                              T mod R = (-q*N) mod R, floor(T/R) uniform in [0, N)
  delta  extremes:            T = 0 and T = N*R - 1

They are INPUT constructions (plain Python ints, no oracle, no CUDA) and are
used by both the oracle pins and the GPU parity tests.
"""
from __future__ import annotations

import random


def column_sum_L_minus_1(q: int, N: int, L: int) -> int:
    """S = sum_{i+j=L-1} lo(q_i N_j) + sum_{i+j=L-2} hi(q_i N_j) (eq:qn)."""
    M = (1 << 32) - 1
    qw = [(q >> (32 * i)) & M for i in range(L)]
    nw = [(N >> (32 * i)) & M for i in range(L)]
    S = 0
    for i in range(L):
        j = L - 1 - i
        if 0 <= j < L:
            S += (qw[i] * nw[j]) & M
        j = L - 2 - i
        if 0 <= j < L:
            S += (qw[i] * nw[j]) >> 32
    return S


def t_alpha(rng: random.Random, N: int, L: int) -> int:
    R = 1 << (32 * L)
    return rng.randrange(N) * R


def t_beta(rng: random.Random, N: int, L: int) -> int:
    R = 1 << (32 * L)
    return rng.randrange(N) * R + rng.randrange(1, 1 << 32) * (1 << (32 * (L - 1)))


def t_gamma(rng: random.Random, N: int, L: int, k: int) -> int:
    R = 1 << (32 * L)
    M = (1 << 32) - 1
    q = rng.randrange(R)
    q &= ~(M << (32 * (L - 1)))  # clear q[L-1]
    rest = column_sum_L_minus_1(q, N, L) & M
    target = (M - k) & M
    n0_inv = pow(N & M, -1, 1 << 32)
    q_top = ((target - rest) * n0_inv) & M
    q |= q_top << (32 * (L - 1))
    assert column_sum_L_minus_1(q, N, L) & M == target
    t_lo = (-q * N) % R
    return rng.randrange(N) * R + t_lo


def t_delta(N: int, L: int) -> list[int]:
    R = 1 << (32 * L)
    return [0, N * R - 1]


def redc_family(rng: random.Random, N: int, L: int, per_family: int = 4) -> list[tuple[str, int]]:
    out = []
    for _ in range(per_family):
        out.append(("alpha", t_alpha(rng, N, L)))
        out.append(("beta", t_beta(rng, N, L)))
        for k in (0, 1, 2):
            out.append((f"gamma{k}", t_gamma(rng, N, L, k)))
    for t in t_delta(N, L):
        out.append(("delta", t))
    return out


# ----------------------------------------------- truncated-Karatsuba REDC (f1) families
def craft_half(rng: random.Random, y: int, H: int, k: int) -> int:
    """x (H words) with column H-1 of x*y forced: S mod 2^32 = 2^32-1-k (S = lo halves of weight H-1 +
    hi halves of weight H-2, the Theorem-2 column of an H-word product).  Needs y odd."""
    M = (1 << 32) - 1
    x = rng.getrandbits(32 * H) & ~(M << (32 * (H - 1)))
    xw = [(x >> (32 * i)) & M for i in range(H)]
    yw = [(y >> (32 * i)) & M for i in range(H)]
    rest = sum((xw[i] * yw[H - 1 - i]) & M for i in range(H - 1)) + \
        sum((xw[i] * yw[H - 2 - i]) >> 32 for i in range(H - 1))
    top = (((M - k) - rest) * pow(yw[0], -1, 1 << 32)) & M
    return x | (top << (32 * (H - 1)))


def t_kara_trunc(rng: random.Random, N: int, L: int, k0: int, km: int, below_n: bool = False):
    """A REDC input T whose q = T N' mod R makes BOTH half-level corrections of the truncated-
    Karatsuba REDC necessary: q0 * N0 and |q0 - q1| * |N0 - N1| each get a forced-wrap Theorem-2
    column (halves of H = L/2 words).  below_n: T < N (a valid operand in the R^2 position).
    Returns None when N's halves do not allow it (N0 or |N0 - N1| even)."""
    H = L // 2
    X = 1 << (32 * H)
    R = X * X
    n0, n1 = N % X, N // X
    dn = abs(n0 - n1)
    if n0 % 2 == 0 or dn % 2 == 0:
        return None
    for _ in range(2000):
        q0 = craft_half(rng, n0, H, k0)
        dq = craft_half(rng, dn, H, km)
        if dq > q0:
            continue
        q = q0 + (q0 - dq) * X
        t_lo = (-q * N) % R
        if below_n:
            if t_lo < N:
                return t_lo
            continue
        return t_lo + rng.randrange(N) * R
    return None
