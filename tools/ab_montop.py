"""A/B of stand-alone MontMul / MontSqr (config 2 shape: 2^20 operands, inputs resident): mean
CUDA-event time of 10 launches after 2 warm-ups, ops/s, IMAD fraction on the algorithm's count,
and a seeded sample against the oracle.  The kernel choice comes from the environment.

  MPB_REG_TRUNC=1 python tools/ab_montop.py --bits 1024 --redc 1
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402  (parity sample only)
from bench import imad_counts  # noqa: E402
from paper_2410_18129_b200 import inputs as I  # noqa: E402
from paper_2410_18129_b200 import mpb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--bits", type=int, default=1024)
ap.add_argument("--redc", type=int, default=1)
ap.add_argument("--count", type=int, default=1 << 20)
a = ap.parse_args()
N, x, y = I.montmul_inputs(config=2, count=a.count, bits=a.bits)
dN, dx, dy = (mpb.to_device(v) for v in (N, x, y))
Np, _ = mpb.mont_batch_setup(dN, a.bits)
L = I.limbs_for_bits(a.bits)
cnt = imad_counts(L, a.redc)
idx = np.concatenate([np.random.default_rng(1).choice(a.count, 12, replace=False), [0, a.count - 1]])
for op in ("mul", "sqr"):
    fn = (lambda: mpb.mont_batch_mul(dx, dy, dN, Np, a.bits, a.redc)) if op == "mul" else \
        (lambda: mpb.mont_batch_sqr(dx, dN, Np, a.bits, a.redc))
    out = fn()
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ops = a.count * 10 / (e0.elapsed_time(e1) / 1e3)
    h = mpb.to_host(out)
    ref = O.batch_montmul(x[idx], (x if op == "sqr" else y)[idx], N[idx])
    print(json.dumps({"bits": a.bits, "redc": a.redc, "op": op, "env_reg_trunc": os.environ.get("MPB_REG_TRUNC", "0"),
                      "ops_per_s": ops, "imad_frac": ops * cnt[op] / (148 * 64 * 1.965e9),
                      "parity_sample": bool(np.array_equal(h[idx], ref))}))
