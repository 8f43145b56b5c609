"""Profiling driver: one setup + one modexp launch (for ncu / compute-sanitizer runs)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2410_18129_b200 import inputs as I  # noqa: E402
from paper_2410_18129_b200 import mpb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--bits", type=int, default=2048)
ap.add_argument("--count", type=int, default=148 * 128 * 2)
ap.add_argument("--window", type=int, default=5)
ap.add_argument("--redc", type=int, default=1)
ap.add_argument("--op", default="modexp", choices=["modexp", "montmul", "montsqr"])
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--algo", type=int, default=0)
a = ap.parse_args()
N, base, exp = I.modexp_inputs(config=3, count=a.count, bits=a.bits)
dN, dB, dE = (mpb.to_device(x) for x in (N, base, exp))
Np, R2 = mpb.mont_batch_setup(dN, a.bits)
for _ in range(a.reps):
    if a.op == "modexp":
        out = mpb.mont_batch_modexp_ct(dN, Np, R2, dB, dE, a.bits, a.window, a.redc, algo=a.algo)
    elif a.op == "montmul":
        out = mpb.mont_batch_mul(dB, dE, dN, Np, a.bits, a.redc)
    else:
        out = mpb.mont_batch_sqr(dB, dN, Np, a.bits, a.redc)
torch.cuda.synchronize()
print("ok", a.op, a.bits, a.count)
