"""One small call of every kernel family (a smoke of all launch paths; compute-sanitizer is closed on
the GPU pool): layout, products (3 algorithms),
Montgomery ops (3 REDC modes), REDC, setup, modexp (3 REDC modes, Karatsuba), CRT-RSA."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2410_18129_b200 import inputs as I  # noqa: E402
from paper_2410_18129_b200 import mpb  # noqa: E402

for bits, count in ((1024, 37), (4096, 5), (4108, 3)):
    a, b = I.mul_inputs(config=4, count=count, bits=bits)
    da, db = mpb.to_device(a), mpb.to_device(b)
    for algo in (1, 2, 3):
        mpb.mp_batch_mul(da, db, bits, algo)
        mpb.mp_batch_sqr(da, bits, algo)
    N, x, y = I.montmul_inputs(config=2, count=count, bits=bits)
    dN, dx, dy = (mpb.to_device(v) for v in (N, x, y))
    Np, R2 = mpb.mont_batch_setup(dN, bits)
    for redc in (0, 1, 2):
        mpb.mont_batch_mul(dx, dy, dN, Np, bits, redc=redc)
        mpb.mont_batch_sqr(dx, dN, Np, bits, redc=redc)
    L = I.limbs_for_bits(bits)
    T = mpb.to_device(np.zeros((count, 2 * L), np.uint32))
    mpb.mont_batch_redc(T, dN, Np, bits, redc=1)
    _, base, exp = I.modexp_inputs(config=3, count=count, bits=bits)
    for redc in (0, 1, 2):
        mpb.mont_batch_modexp_ct(dN, Np, R2, mpb.to_device(base), mpb.to_device(exp), bits, window=4, redc=redc)
    if bits >= 4096:
        mpb.mont_batch_modexp_ct(dN, Np, R2, mpb.to_device(base), mpb.to_device(exp), bits, window=4, algo=3)
torch.cuda.synchronize()
# CRT-RSA with synthetic odd "primes" of the right size (memory behaviour only; values unchecked)
bits, count = 1024, 9
h = bits // 2
Lh, L = I.limbs_for_bits(h), I.limbs_for_bits(bits)
rng = np.random.default_rng(1)
pq = [int.from_bytes(rng.bytes(h // 8), "little") | 1 | (1 << (h - 1)) for _ in range(2 * count)]
p, q = pq[:count], pq[count:]
c = [int.from_bytes(rng.bytes(bits // 8 - 1), "little") for _ in range(count)]
arrs = [I.ints_to_array(c, L)] + [I.ints_to_array(v, Lh) for v in (p, q, p, q, p)]
mpb.rsa_batch_crt_ct(*(mpb.to_device(v) for v in arrs), bits)
torch.cuda.synchronize()
print("sanitize run ok")
