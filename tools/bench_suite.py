"""Measure every BASELINE.json config on one B200 (bench.py times config 3 only).

Prints one JSON object per measurement; each carries the algorithmic IMAD count, the
roofline fraction (148 SMs x 64 IMAD/clk x 1965 MHz = 18.61 T IMAD/s) and, where cheap,
a parity verdict against the oracle on a seeded sample.

  python tools/bench_suite.py [--configs 1,2,3,4,5,6,7,8,9] [--reps 3]
      (6 = CRT-RSA; 7 = config 3 under the paper's timing protocol, SURVEY 8(d);
       8 = radix-2^52 FP64 and hybrid exponentiations, f3; 9 = small 4096-bit batches, cooperative lanes)
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import oracle as O  # noqa: E402  (parity samples only)
from bench import imad_counts, kara_saved_imad, modexp_imad  # noqa: E402
from paper_2410_18129_b200 import inputs as I  # noqa: E402
from paper_2410_18129_b200 import mpb  # noqa: E402

PEAK = 148 * 64 * 1.965e9


def timeit(fn, reps: int, warmup: int = 2) -> float:
    """Mean CUDA-event time (ms) of fn over reps, after warmup."""
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def emit(d: dict) -> None:
    print(json.dumps(d), flush=True)


def sample_idx(count: int, n: int = 16, seed: int = 0) -> np.ndarray:
    rng = np.random.default_rng(seed)
    idx = rng.choice(count, size=min(n, count), replace=False)
    return np.unique(np.concatenate([idx, [0, count - 1]]))


def config1(reps):
    bits, count = 1024, 8
    N, base, exp = I.modexp_inputs(config=1, count=count, bits=bits)
    _, a, b = I.montmul_inputs(config=1, count=count, bits=bits)
    dN, dB, dE, da, db = (mpb.to_device(x) for x in (N, base, exp, a, b))
    Np, R2 = mpb.mont_batch_setup(dN, bits)
    ref_exp = O.batch_modexp(base, exp, bits, N)
    for redc, name in ((1, "truncated"), (0, "full"), (2, "cios")):
        ws = mpb.modexp_workspace(count, bits, 5)
        out = mpb.empty_sliced(32, count)
        ms = timeit(lambda: mpb.mont_batch_modexp_ct(dN, Np, R2, dB, dE, bits, 5, redc, ws=ws, out=out), reps)
        ok = bool(np.array_equal(mpb.to_host(out), ref_exp))
        mws = mpb.mont_workspace(count, bits)
        mm = mpb.to_host(mpb.mont_batch_mul(da, db, dN, Np, bits, redc, ws=mws))
        ms2 = mpb.to_host(mpb.mont_batch_sqr(da, dN, Np, bits, redc, ws=mws))
        ok_m = bool(np.array_equal(mm, O.batch_montmul(a, b, N)) and np.array_equal(ms2, O.batch_montmul(a, a, N)))
        emit({"config": 1, "op": "modexp", "bits": bits, "count": count, "window": 5, "redc": name,
              "latency_us": 1000 * ms, "parity_modexp": ok, "parity_montmul_montsqr": ok_m})


def config2(reps, sizes=(1024, 2048, 3072, 4096)):
    count = 1 << 20
    for bits in sizes:
        L = I.limbs_for_bits(bits)
        N, a, b = I.montmul_inputs(config=2, count=count, bits=bits)
        dN, da, db = (mpb.to_device(x) for x in (N, a, b))
        Np, _ = mpb.mont_batch_setup(dN, bits)
        ws = mpb.mont_workspace(count, bits)
        idx = sample_idx(count)
        for redc, name in ((1, "truncated"), (0, "full"), (2, "cios")):
            res = {}
            for op in ("mul", "sqr"):
                if op == "mul":
                    fn = lambda: mpb.mont_batch_mul(da, db, dN, Np, bits, redc, ws=ws)  # noqa: E731
                else:
                    fn = lambda: mpb.mont_batch_sqr(da, dN, Np, bits, redc, ws=ws)  # noqa: E731
                ms = timeit(fn, reps)
                out = mpb.to_host(fn())
                ref = O.batch_montmul(a[idx], (b if op == "mul" else a)[idx], N[idx])
                imad = imad_counts(L, redc)[op] * count
                imad_own = imad - kara_saved_imad(L, redc)[op] * count
                bytes_io = (5 if op == "mul" else 4) * L * 4 * count
                emit({"config": 2, "op": f"mont_{op}", "bits": bits, "count": count, "redc": name,
                      "ms": ms, "ops_per_s": count / (ms / 1e3), "imad_frac": imad_own / (ms / 1e3) / PEAK,
                      "imad_frac_schoolbook_basis": imad / (ms / 1e3) / PEAK,
                      "io_gbs": bytes_io / (ms / 1e3) / 1e9, "parity_sample": bool(np.array_equal(out[idx], ref))})
                res[op] = ms
            torch.cuda.synchronize()
        del dN, da, db, Np, ws
        torch.cuda.empty_cache()


def modexp_run(config, bits, count, reps, redcs=((1, "truncated"), (0, "full"), (2, "cios")), check=8, algo=0):
    N, base, exp = I.modexp_inputs(config=config, count=count, bits=bits)
    dN, dB, dE = (mpb.to_device(x) for x in (N, base, exp))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    Np, R2 = mpb.mont_batch_setup(dN, bits)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t0
    ws = mpb.modexp_workspace(count, bits, 5, algo)
    L = I.limbs_for_bits(bits)
    outs = {}
    idx = sample_idx(count, check)
    for redc, name in redcs:
        out = mpb.empty_sliced(L, count)
        ms = timeit(lambda: mpb.mont_batch_modexp_ct(dN, Np, R2, dB, dE, bits, 5, redc, algo=algo, ws=ws, out=out),
                    reps, 1)
        outs[name] = out
        h = mpb.to_host(out)
        ok = bool(np.array_equal(h[idx], O.batch_modexp(base[idx], exp[idx], bits, N[idx])))
        imad = modexp_imad(bits, 5, redc) * count
        imad_own = modexp_imad(bits, 5, redc, own=algo in (0, 1)) * count
        emit({"config": config, "op": "modexp", "bits": bits, "count": count, "window": 5, "redc": name,
              "algo": ["auto", "schoolbook", "karatsuba", "karatsuba2", "radix52", "hybrid"][algo], "ms": ms,
              "modexp_per_s": count / (ms / 1e3), "imad_frac": imad_own / (ms / 1e3) / PEAK,
              "imad_frac_schoolbook_basis": imad / (ms / 1e3) / PEAK,
              "setup_s": setup_s, "parity_sample": ok, "sample": len(idx)})
    if len(outs) >= 2:
        emit({"config": config, "bits": bits, "all_redc_modes_equal_on_whole_batch":
              bool(all(torch.equal(outs["truncated"], o) for o in outs.values()))})
    del dN, dB, dE, Np, R2, ws, outs
    torch.cuda.empty_cache()


def products(bits, count, reps):
    L = I.limbs_for_bits(bits)
    a, b = I.mul_inputs(config=4, count=count, bits=bits)
    da, db = mpb.to_device(a), mpb.to_device(b)
    idx = sample_idx(count, 8)
    for algo, name in ((mpb.ALGO_SCHOOLBOOK, "schoolbook"), (mpb.ALGO_KARATSUBA, "karatsuba")):
        for op in ("mul", "sqr"):
            try:
                fn = (lambda: mpb.mp_batch_mul(da, db, bits, algo)) if op == "mul" else (lambda: mpb.mp_batch_sqr(da, bits, algo))
                ms = timeit(fn, reps)
                out = mpb.to_host(fn())
            except ValueError as e:
                emit({"config": 4, "op": f"mp_{op}", "bits": bits, "algo": name, "unavailable": str(e)})
                continue
            ok = all(I.from_limbs(out[k]) == O.mul(I.from_limbs(a[k]), I.from_limbs((b if op == "mul" else a)[k]))
                     for k in idx)
            imad = (2 * L * L if op == "mul" else L * L + L) * count
            emit({"config": 4, "op": f"mp_{op}", "bits": bits, "count": count, "algo": name, "ms": ms,
                  "ops_per_s": count / (ms / 1e3), "imad_frac_schoolbook_basis": imad / (ms / 1e3) / PEAK,
                  "parity_sample": ok})


def rsa_crt(bits, count, reps, n_keys=16):
    """Batched CRT-RSA private-key operations: keys from oracle primes, a pool of
    n_keys keys cycled over the batch (every item has its own ciphertext; the kernels' work per
    item does not depend on which key it uses)."""
    import math
    import random

    h = bits // 2
    L, Lh = I.limbs_for_bits(bits), I.limbs_for_bits(h)
    keys = []
    for i in range(n_keys):
        p, q = O.gen_prime(h, 1000 + 2 * i), O.gen_prime(h, 5000 + 2 * i)
        lam = (p - 1) * (q - 1) // math.gcd(p - 1, q - 1)
        d = O.inv_mod(65537, lam)
        keys.append((p, q, d % (p - 1), d % (q - 1), O.inv_mod(q, p), d))
    rng = random.Random(bits)
    sel = [keys[k % n_keys] for k in range(count)]
    cts = [rng.randrange(kk[0] * kk[1]) for kk in sel]
    arrs = [I.ints_to_array(cts, L)] + [I.ints_to_array([kk[j] for kk in sel], Lh) for j in range(5)]
    dev = [mpb.to_device(a) for a in arrs]
    ws = mpb.rsa_workspace(count, bits, 5)
    out = mpb.empty_sliced(L, count)
    for redc, name in ((1, "truncated"), (0, "full"), (2, "cios")):
        ms = timeit(lambda: mpb.rsa_batch_crt_ct(*dev, bits, 5, redc, ws=ws, out=out), reps, 1)
        h_out = mpb.to_host(out)
        idx = sample_idx(count, 8)
        ok = all(I.from_limbs(h_out[k]) == pow(cts[k], sel[k][5], sel[k][0] * sel[k][1]) for k in idx)
        imad = 2 * modexp_imad(h, 5, redc) * count
        emit({"config": "crt-rsa", "op": "rsa_private_crt", "bits": bits, "count": count, "window": 5, "redc": name,
              "ms": ms, "ops_per_s": count / (ms / 1e3), "imad_frac_modexp_basis": imad / (ms / 1e3) / PEAK,
              "keys_in_pool": n_keys, "parity_sample_vs_pow": ok, "sample": len(idx)})
    del dev, ws, out
    torch.cuda.empty_cache()


def config5_e2e(bits=2048, count=1 << 22, window=5):
    """Config 5 end to end on one GPU: mpb_modexp_host over PINNED host buffers --
    H2D of N / base / exp, layout expand, setup, modexp, contract, D2H -- timed by the host clock
    around the blocking call (one untimed warm-up call sizes the memory pool)."""
    import ctypes

    N, base, exp = I.modexp_inputs(config=5, count=count, bits=bits)
    hN, hB, hE = (torch.from_numpy(x.view(np.int32)).pin_memory() for x in (N, base, exp))
    hO = torch.empty_like(hN).pin_memory()
    stream = torch.cuda.current_stream()

    def call():
        rc = mpb._lib.mpb_modexp_host(hN.data_ptr(), hB.data_ptr(), hE.data_ptr(), hO.data_ptr(), count, bits, window,
                                      1, ctypes.c_void_p(stream.cuda_stream))
        assert rc == 0, mpb._lib.mpb_last_error()

    call()
    t0 = time.perf_counter()
    call()
    dt = time.perf_counter() - t0
    out = hO.numpy().view(np.uint32)
    idx = sample_idx(count, 8, seed=5)
    ok = bool(np.array_equal(out[idx], O.batch_modexp(base[idx], exp[idx], bits, N[idx])))
    L = I.limbs_for_bits(bits)
    emit({"config": 5, "op": "modexp_e2e_pinned", "bits": bits, "count": count, "window": window, "s": dt,
          "modexp_per_s": count / dt, "h2d_bytes": 3 * count * L * 4, "d2h_bytes": count * L * 4,
          "parity_sample": ok})


def paper_protocol(bits=2048, count=1 << 18, datasets=5, launches=10, warmup=3):
    """SURVEY 8(d) timing protocol, adapted from P:L614-621: 3 warm-up launches, then for each of
    D = 5 seeded datasets the minimum over 10 launches (CUDA events around the kernel only);
    reports the mean of the minimums (the paper's statistic) and the median of all launches."""
    mins, alls = [], []
    for d in range(datasets):
        N, base, exp = I.modexp_inputs(config=3, count=count, bits=bits, dataset=d)
        dN, dB, dE = (mpb.to_device(x) for x in (N, base, exp))
        Np, R2 = mpb.mont_batch_setup(dN, bits)
        ws = mpb.modexp_workspace(count, bits, 5)
        out = mpb.empty_sliced(I.limbs_for_bits(bits), count)
        fn = lambda: mpb.mont_batch_modexp_ct(dN, Np, R2, dB, dE, bits, 5, 1, ws=ws, out=out)  # noqa: E731
        if d == 0:
            for _ in range(warmup):
                fn()
        ts = []
        for _ in range(launches):
            ts.append(timeit(fn, 1, 0))
        mins.append(min(ts))
        alls += ts
        idx = sample_idx(count, 4, seed=d)
        ok = bool(np.array_equal(mpb.to_host(out)[idx], O.batch_modexp(base[idx], exp[idx], bits, N[idx])))
        emit({"protocol": "paper", "dataset": d, "min_ms": min(ts), "max_ms": max(ts), "parity_sample": ok})
        del dN, dB, dE, Np, R2, ws, out
        torch.cuda.empty_cache()
    mean_min = float(np.mean(mins))
    emit({"protocol": "paper (P:L614-621 adapted)", "bits": bits, "count": count, "window": 5, "redc": "truncated",
          "datasets": datasets, "launches_per_dataset": launches, "mean_of_min_ms": mean_min,
          "median_ms": float(np.median(alls)), "modexp_per_s_at_mean_of_min": count / (mean_min / 1e3),
          "imad_frac_at_mean_of_min": modexp_imad(bits, 5, 1) * count / (mean_min / 1e3) / PEAK})


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4,5")
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    cfgs = {int(c) for c in args.configs.split(",")}
    emit({"device": torch.cuda.get_device_name(), "peak_imad_per_s": PEAK})
    if 1 in cfgs:
        config1(args.reps)
    if 2 in cfgs:
        config2(args.reps)
    if 3 in cfgs:
        modexp_run(3, 2048, 1 << 18, args.reps)
    if 4 in cfgs:
        modexp_run(4, 4096, 1 << 16, args.reps)
        modexp_run(4, 4108, 1 << 16, 1, redcs=((1, "truncated"),))
        for algo in (2, 3):
            modexp_run(4, 4096, 1 << 16, args.reps, redcs=((1, "truncated"),), algo=algo)
        products(4096, 1 << 16, args.reps)
        products(4154, 1 << 16, args.reps)
    if 5 in cfgs:
        modexp_run(5, 2048, 1 << 22, 1, redcs=((1, "truncated"),), check=64)
        config5_e2e()
    if 8 in cfgs:  # radix-2^52 FP64 exponentiation and the hybrid launch, vs the IMAD path
        modexp_run(3, 2048, 1 << 18, args.reps, redcs=((1, "truncated"), (0, "full")), algo=4)
        modexp_run(3, 2048, 1 << 18, args.reps, redcs=((1, "truncated"),), algo=5)
        modexp_run(2, 1024, 1 << 20, args.reps, redcs=((1, "truncated"), (2, "cios")), algo=4)
        modexp_run(4, 4096, 1 << 16, 1, redcs=((1, "truncated"),), algo=4)
    if 9 in cfgs:  # small 4096-bit batches: the 8 / 4 / 2-lane cooperative policy (north_star (b))
        for n in (2048, 8192, 16384):
            modexp_run(4, 4096, n, args.reps, redcs=((1, "truncated"),), check=4)
    if 7 in cfgs:  # the paper's timing statistic on config 3
        paper_protocol()
    if 6 in cfgs:  # CRT-RSA (not a BASELINE config: SURVEY 8(f) f4)
        rsa_crt(2048, 1 << 17, args.reps)
        rsa_crt(4096, 1 << 14, args.reps)


if __name__ == "__main__":
    main()
