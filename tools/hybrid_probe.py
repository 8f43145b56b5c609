"""Do the FP64 (radix-2^52) and IMAD (radix-2^32) exponentiations overlap on one SM?

One-wave probe at 2048 bits: a CTAs/SM of the radix-2^52 kernel (algo 4) and b CTAs/SM of the
32-bit kernel (algo 0), a + b = 3 (the register-limited residency of both), launched concurrently
on two streams (radix-2^52 first, so every SM holds a of its CTAs and b of the other's).  Prints
the concurrent time, each kernel alone, and modexp/s of the mix -- if the two pipes (FP64, IMAD)
overlap, the mix beats the pure 32-bit wave.

  python tools/hybrid_probe.py [--bits 2048]
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


def setup(count, bits, dataset):
    N, base, exp = I.modexp_inputs(config=3, count=count, bits=bits, dataset=dataset)
    dN, dB, dE = (mpb.to_device(x) for x in (N, base, exp))
    Np, R2 = mpb.mont_batch_setup(dN, bits)
    return dN, Np, R2, dB, dE


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bits", type=int, default=2048)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    bits = a.bits
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    per = sms * 128
    s0, s1 = torch.cuda.Stream(), torch.cuda.Stream()
    for nd, ni in ((0, 3), (3, 0), (1, 2), (2, 1)):
        cd, ci = nd * per, ni * per
        D = setup(cd, bits, 1) if cd else None
        M = setup(ci, bits, 2) if ci else None
        wsd = mpb.modexp_workspace(cd, bits, 5, 4) if cd else None
        wsi = mpb.modexp_workspace(ci, bits, 5, 0) if ci else None
        L = I.limbs_for_bits(bits)
        od = mpb.empty_sliced(L, cd) if cd else None
        oi = mpb.empty_sliced(L, ci) if ci else None

        def run_d():
            mpb.mont_batch_modexp_ct(*D, bits, 5, 1, algo=4, ws=wsd, out=od)

        def run_i():
            mpb.mont_batch_modexp_ct(*M, bits, 5, 1, algo=0, ws=wsi, out=oi)

        def timed(fn_pairs):
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            cur = torch.cuda.current_stream()
            e0.record(cur)
            ends = []
            for st, fn in fn_pairs:
                st.wait_event(e0)
                with torch.cuda.stream(st):
                    fn()
                ev = torch.cuda.Event()
                ev.record(st)
                ends.append(ev)
            for ev in ends:
                cur.wait_event(ev)
            e1.record(cur)
            torch.cuda.synchronize()
            return e0.elapsed_time(e1)

        pairs = []
        if cd:
            pairs.append((s1, run_d))
        if ci:
            pairs.append((s0, run_i))
        timed(pairs)  # warm-up
        t_mix = min(timed(pairs) for _ in range(a.reps))
        t_d = min(timed([(s1, run_d)]) for _ in range(a.reps)) if cd else 0.0
        t_i = min(timed([(s0, run_i)]) for _ in range(a.reps)) if ci else 0.0
        print(json.dumps({"bits": bits, "ctas_per_sm_radix52": nd, "ctas_per_sm_radix32": ni, "count_radix52": cd,
                          "count_radix32": ci, "ms_concurrent": t_mix, "ms_radix52_alone": t_d,
                          "ms_radix32_alone": t_i, "modexp_per_s_mix": (cd + ci) / (t_mix / 1000.0)}), flush=True)
        del D, M, wsd, wsi, od, oi
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
