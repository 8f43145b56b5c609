"""A/B timing of mont_batch_modexp_ct variants on one GPU (tuning tool; bench.py is the contract).

  python tools/bench_algo.py --bits 2048 --count 262144 --algos 0,4 --redc 1 [--reps 3] [--check 16]

For each algo: mean CUDA-event time of `reps` launches after one warm-up, modexp/s, and (if
--check > 0) a seeded sample of outputs against the oracle plus equality with the first algo's
output on the whole batch.  One JSON line per algo.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2410_18129_b200 import inputs as I  # noqa: E402
from paper_2410_18129_b200 import mpb  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bits", type=int, default=2048)
    ap.add_argument("--count", type=int, default=1 << 18)
    ap.add_argument("--window", type=int, default=5)
    ap.add_argument("--algos", default="0,4")
    ap.add_argument("--redc", type=int, default=1)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--check", type=int, default=16)
    a = ap.parse_args()
    bits, count = a.bits, a.count
    N, base, exp = I.modexp_inputs(config=3, count=count, bits=bits)
    dN, dB, dE = (mpb.to_device(x) for x in (N, base, exp))
    Np, R2 = mpb.mont_batch_setup(dN, bits)
    first = None
    for algo in (int(x) for x in a.algos.split(",")):
        ws = mpb.modexp_workspace(count, bits, a.window, algo)
        out = mpb.empty_sliced(I.limbs_for_bits(bits), count)

        def run():
            mpb.mont_batch_modexp_ct(dN, Np, R2, dB, dE, bits, a.window, a.redc, algo=algo, ws=ws, out=out)

        run()
        torch.cuda.synchronize()
        s = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(a.reps):
            run()
        e1.record(s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        line = {"bits": bits, "count": count, "window": a.window, "redc": a.redc, "algo": algo, "ms": ms,
                "modexp_per_s": count / (ms / 1000.0)}
        if a.check > 0:
            import oracle as O

            h = mpb.to_host(out)
            idx = np.unique(np.concatenate([np.random.default_rng(1).choice(count, size=min(a.check, count),
                                                                            replace=False), [0, count - 1]]))
            line["oracle_sample_ok"] = bool(np.array_equal(h[idx], O.batch_modexp(base[idx], exp[idx], bits, N[idx])))
            if first is None:
                first = h
            else:
                line["equals_first_algo_on_all"] = bool(np.array_equal(h, first))
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
