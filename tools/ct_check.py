"""Constant-time evidence driver (SURVEY.md 8(d) "CT evidence").

Runs ONE modexp launch (2048-bit, w = 5, truncated) over a batch whose exponents all belong to
one class -- 'zero' (every window 0 apart from the forced top bit), 'ones' (all bits set),
'random' -- with the SAME moduli and bases.  Under ncu, the warp-level SASS instruction counts,
branch counts and load/store counts of k_modexp must be identical across classes; a build with
-DMPB_PLANTED_BRANCH (secret-dependent table loads) is the negative control that must differ.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2410_18129_b200 import inputs as I  # noqa: E402
from paper_2410_18129_b200 import mpb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cls", choices=["zero", "ones", "random"], required=True)
ap.add_argument("--count", type=int, default=148 * 128)
ap.add_argument("--bits", type=int, default=2048)
ap.add_argument("--algo", type=int, default=0)  # 4 = radix-2^52 kernel
ap.add_argument("--redc", type=int, default=1)  # 2 = CIOS (1024 bits: the register kernel)
a = ap.parse_args()
N, base, exp = I.modexp_inputs(config=3, count=a.count, bits=a.bits)
L = N.shape[1]
if a.cls == "zero":
    exp[:] = 0
    exp[:, (a.bits - 1) // 32] = np.uint32(1 << ((a.bits - 1) % 32))  # full length, all other windows 0
elif a.cls == "ones":
    exp[:] = np.uint32(0xFFFFFFFF)
    if a.bits % 32:
        exp[:, (a.bits - 1) // 32] = np.uint32((1 << (a.bits % 32)) - 1)
    exp[:, (a.bits + 31) // 32:] = 0
dN, dB, dE = (mpb.to_device(x) for x in (N, base, exp))
Np, R2 = mpb.mont_batch_setup(dN, a.bits)
out = mpb.mont_batch_modexp_ct(dN, Np, R2, dB, dE, a.bits, 5, a.redc, algo=a.algo)
torch.cuda.synchronize()
print("ok", a.cls, int(mpb.to_host(out)[0, 0]))
