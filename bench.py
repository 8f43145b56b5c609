#!/usr/bin/env python
"""bench.py -- batched constant-time 2048-bit modexp on B200 (arXiv 2410.18129 hot path).

A "step" is one pass of the whole hot path over one batch: mont_batch_modexp_ct on
BASELINE.json config 3 (2048-bit moduli, window 5, truncated REDC, batch 2^18 per GPU;
table build, the 409 windows of squarings / masked table scans / multiplications, and the
exit REDC all inside one kernel).  Inputs are resident in HBM before timing starts; the
per-step working set (inputs 320 MiB + window tables and scratch 2.4 GiB) is larger than
the 126 MB L2, so no explicit flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload config3|config5]

N > 1: one rank per GPU, under torchrun or -- when WORLD_SIZE is unset -- started here by
torch.multiprocessing (launcher.spawn); NCCL only for the barrier and the max over ranks.
Default (config3): each rank takes its own 2^18 batch (independent units, no data-path
collective; weak scaling).  --workload config5: one 2^22 batch split into contiguous slices
(strong scaling), with the oracle check of a seeded 4096-element subset and a slicing-independent
digest of all outputs in the line (G-invariance across runs with 1/2/4/8 GPUs).
`--impl reference` times the plain CPU oracle (oracle/, test infrastructure) on the host
cores on bounded samples of the same workload -- the reference arm of this tier.
Extra keys, measured on rank 0 AFTER the timed region and outside it: `modmul` (config 2 at 2048
bits: MontMul / MontSqr per second, 2^20 operands) and `config4` (4096-bit modexp, 2^16 operands,
the one-CTA-per-SM instance; `--no-config4` skips it).  In an ncu launch list of this command those
are the k_mont_mul and mpb_w448::k_modexp launches; the step is k_modexp<16, 1, 4, 0, 3>.
Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2410_18129_b200 import inputs as I  # noqa: E402

BASELINE = json.load(open(os.path.join(ROOT, "BASELINE.json")))
METRIC = BASELINE["metric"]
UNIT = "modexp/s"
BITS, WINDOW, COUNT, CONFIG = 2048, 5, 1 << 18, 3
COUNT5 = 1 << 22  # config 5: whole-box batch
SMS, IMAD_PER_CLK_SM = 148, 64  # K0-measured 63.6 (profiles/r01_microbench_int.json)
K0_PRODUCTS_PER_CLK_SM = 31.1  # measured fused IMAD.WIDE.U32.X chain rate (profiles/r01_microbench_int.json)


# ------------------------------------------------------------------ roofline
def block_for(L: int) -> int:
    """Limbs per block of the kernels (the largest of 16, 12, 8, 4 dividing L)."""
    return next(c for c in (16, 12, 8, 4) if L % c == 0)


def imad_counts(L: int, redc: int) -> dict:
    """Algorithmic IMAD per operation: a 32x32->64 word product = 2 IMAD,
    a lo-only product = 1; the hi-only products of column L-2 count 1 each.
    redc: 1 truncated, 0 full, 2 CIOS (alg:8BlockMontRed at digit 2^(32C): per row of C limbs,
    2CL products for a_i*B, 2CL for m_i*N and a C x C low-half product of C^2 IMAD, so
    4L^2 + LC for a multiplication or a squaring; REDC is MontMul(X, 1).  At L = 32 the
    register-resident kernel (csrc/mp_reg.cuh) uses the paper's word digit: C = 1, 4L^2 + L.
    MontSqr uses squaring rows (each cross product once, doubled): at block granularity
    NB(NB-1)/2 full blocks + NB symmetric C x C squares = L^2 + L for the a-part, so 3L^2 + L + LC;
    the register kernel's word rows also multiply by the top word of 2a: 3L^2 + 4L)."""
    if redc == 2:
        C = 1 if L == 32 else block_for(L)  # 1024 bits: the register-resident kernel's 32-bit digit
        mul = redc_ = 4 * L * L + L * C
        sqr = 3 * L * L + 4 * L if L == 32 else 3 * L * L + L + L * C
    elif redc:
        mul, sqr, redc_ = 4 * L * L + 2 * L - 1, 3 * L * L + 3 * L - 1, 2 * L * L + 2 * L - 1
    else:
        mul, sqr, redc_ = 5 * L * L, 4 * L * L + L, 3 * L * L
    return {"mul": mul, "sqr": sqr, "redc": redc_}


KARA_MIN_NB = 6  # csrc/mp_mont.cuh: full 16-limb blocks by register Karatsuba from 6 blocks (3072 bits) up


def kara_saved_imad(L: int, redc: int) -> dict:
    """IMAD the engine's register-Karatsuba blocks (mp_block.cuh acc_kara: 3 half-size products,
    3C^2/4 instead of C^2 word products) do NOT execute per operation, for the sizes where the engine
    uses them (C = 16 or 12, NB = L/C >= KARA_MIN_NB; truncated or full REDC).  Kara blocks: PH_MUL all NB^2,
    PH_SQR the NB(NB-1)/2 off-diagonal ones, PH_Q the NB(NB-1)/2 below its top column, PH_HI the
    NB(NB-1)/2 above column NB-1 (truncated) or all NB^2 (full); each saves C^2/4 products (C^2/2 IMAD)."""
    C = block_for(L)
    NB = L // C
    if redc == 2 or C not in (16, 12) or NB < KARA_MIN_NB:
        return {"mul": 0, "sqr": 0, "redc": 0}
    tri = NB * (NB - 1) // 2
    hi = tri if redc else NB * NB
    per = 2 * (C * C // 4)
    return {"mul": per * (NB * NB + tri + hi), "sqr": per * (tri + tri + hi), "redc": per * (tri + hi)}


def modexp_imad(bits: int, w: int, redc: int, own: bool = False) -> int:
    """(W-1)*w MontSqr + (W-1) + (2^w - 1) MontMul + 2 REDC.  own=True: the
    products the kernel's own algorithm executes (minus the register-Karatsuba savings, which get
    no credit: SURVEY 8(d) "each configuration reports its own algorithm's count")."""
    L = I.limbs_for_bits(bits)
    W = -(-bits // w)
    c = dict(imad_counts(L, int(redc)))
    if own:
        k = kara_saved_imad(L, int(redc))
        c = {op: c[op] - k[op] for op in c}
    return (W - 1) * w * c["sqr"] + ((W - 1) + (1 << w) - 1) * c["mul"] + 2 * c["redc"]


NCU_CAPTURE = "r02_ncu_modexp.json"  # the committed `ncu --set full` summary of this launch


def ncu_traffic():
    """(TB per launch, note): dram__bytes_read.sum + dram__bytes_write.sum of k_modexp from the
    committed `ncu --set full` capture of this same launch (a timed run cannot be profiled), or
    (None, note) when no capture of this launch shape is committed."""
    for name in (NCU_CAPTURE, "r01_v7_ncu_modexp.json"):
        try:
            d = json.load(open(os.path.join(ROOT, "profiles", name)))
            if d.get("operands_per_launch") == COUNT:
                return d["dram_bytes_per_launch"] / 1e12, (
                    f"from profiles/{name} (ncu --set full of this launch shape, NOT measured in this run); "
                    f"algorithmic table-scan bytes 0.881 TB per launch")
        except Exception:
            pass
    return None, "no committed ncu capture of this launch"


# -------------------------------------------------------------------- clocks
class ClockSampler:
    """Samples SM clock and throttle reasons with NVML during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index: int, period: float = 0.1):
        self.index, self.period = index, period
        self.samples, self.reasons = [], set()
        self._stop = threading.Event()
        self.max_mhz = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nvml = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nvml.nvmlDeviceGetClockInfo(self.h, self.nvml.NVML_CLOCK_SM))
                r = self.nvml.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nvml:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nvml:
            self.t.join()

    def summary(self) -> dict:
        med = float(np.median(self.samples)) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ------------------------------------------------------------- CPU baseline
def cpu_oracle_sample(target_s: float = 12.0, config: int = CONFIG, dataset: int = 0) -> dict:
    """The plain oracle (oracle/, as it stands) on all host cores over a bounded sample of the
    same workload (first operands of the config-3 batch); sample sized to ~target_s of wall time."""
    import oracle as O

    cores = os.cpu_count() or 1
    N, base, exp = I.modexp_inputs(config=config, count=cores, bits=BITS, dataset=dataset)
    t0 = time.perf_counter()
    O.batch_modexp(base, exp, BITS, N, threads=cores)  # probe: one item per core
    probe = time.perf_counter() - t0
    n = cores * max(1, int(target_s / max(probe, 1e-3)))
    N, base, exp = I.modexp_inputs(config=config, count=n, bits=BITS, dataset=dataset)
    t0 = time.perf_counter()
    O.batch_modexp(base, exp, BITS, N, threads=cores)
    dt = time.perf_counter() - t0
    return {"value": n / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"first {n} operands of the config-3 batch (2048-bit, w=5 workload; oracle = "
                      f"left-to-right binary square-and-multiply with Knuth-D reduction), {dt:.1f} s wall"}


# ---------------------------------------------------------------- reference
def run_reference(args, rank: int, world: int) -> None:
    if rank != 0:
        return
    import oracle as O

    cores = os.cpu_count() or 1
    per_step = max(cores, 2 * cores)
    N, base, exp = I.modexp_inputs(config=CONFIG, count=per_step, bits=BITS)
    for _ in range(args.warmup):
        O.batch_modexp(base[:cores], exp[:cores], BITS, N[:cores], threads=cores)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        O.batch_modexp(base, exp, BITS, N, threads=cores)
    dt = time.perf_counter() - t0
    value = args.steps * per_step / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * dt / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": config_dict(world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": f"{per_step} operands of the config-3 batch per step on {cores} host threads"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_dict(world: int, c5: bool = False) -> dict:
    if c5:
        return {"workload": "BASELINE config 5: one 2^22-operand batch of 2048-bit constant-time fixed-window "
                            "modexps (window 5, truncated REDC) split into contiguous slices across the GPUs "
                            "(random odd moduli with top bit set, bases in [0,N), full-length exponents; "
                            "chunk-seeded so every slicing sees the same operands)",
                "bits": BITS, "window": WINDOW, "redc": "truncated", "count_per_gpu": COUNT5 // world,
                "global_batch": COUNT5, "parallelism": f"independent slices x{world}",
                "l2": "no flush: per-step working set (inputs >= 640 MiB + tables/scratch >= 5 GiB) > 126 MB L2"}
    return {"workload": "BASELINE config 3: 2048-bit constant-time fixed-window modexp, window 5, truncated "
                        "REDC, batch 2^18 per GPU (random odd moduli with top bit set, bases in [0,N), "
                        "full-length exponents)",
            "bits": BITS, "window": WINDOW, "redc": "truncated", "count_per_gpu": COUNT,
            "global_batch": COUNT * world, "parallelism": f"independent slices x{world}",
            "l2": "no flush: per-step working set (inputs 320 MiB + tables/scratch 2.5 GiB) > 126 MB L2"}


# ------------------------------------------------------------------- ours
def run_ours(args) -> None:
    import torch

    from paper_2410_18129_b200 import mpb, shard
    from paper_2410_18129_b200.launcher import Ranks

    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    # MPB_BENCH_SHARE_GPU=1 (launcher check only, never a scaling number): every rank on device 0,
    # gloo for the barrier and the reductions -- exercises the multi-rank path on a one-GPU box
    share = os.environ.get("MPB_BENCH_SHARE_GPU") == "1"
    if share:
        local_rank = 0
    torch.cuda.set_device(local_rank)
    rk = Ranks("gloo" if share else "nccl", device=torch.device("cuda", local_rank))
    rank, world = rk.rank, rk.world
    if world != args.gpus:
        raise SystemExit(f"bench.py: {world} rank(s) running but --gpus {args.gpus}")
    c5 = args.workload == "config5"
    L = I.limbs_for_bits(BITS)
    if c5:  # strong scaling: one global 2^22 batch, contiguous slices (shard.plan)
        a0, b0 = shard.rank_slice(COUNT5, rank, world)
        N, base, exp = I.modexp_inputs_range(5, a0, b0, BITS)
    else:  # weak scaling: 2^18 operands per rank (dataset = rank)
        a0, b0 = 0, COUNT
        N, base, exp = I.modexp_inputs(config=CONFIG, count=COUNT, bits=BITS, dataset=rank)
    count = b0 - a0

    def barrier():
        rk.barrier()
        torch.cuda.synchronize()

    dN, dB, dE = (mpb.to_device(x) for x in (N, base, exp))
    Np, R2 = mpb.mont_batch_setup(dN, BITS)
    ws = mpb.modexp_workspace(count, BITS, WINDOW)
    out = mpb.empty_sliced(L, count)
    stream = torch.cuda.current_stream()

    def step():
        mpb.mont_batch_modexp_ct(dN, Np, R2, dB, dE, BITS, WINDOW, mpb.REDC_TRUNCATED, ws=ws, out=out)

    for _ in range(args.warmup):
        step()
    barrier()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    with ClockSampler(local_rank) as clocks:
        ev[0].record(stream)
        for i in range(args.steps):
            step()
            ev[i + 1].record(stream)
        barrier()
    per_launch_ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(args.steps)]
    total_ms = rk.max(ev[0].elapsed_time(ev[-1]))  # the slowest rank's device time
    dev_out = mpb.to_host(out)

    # end to end through the public host-buffer call (pinned host memory, H2D + setup + modexp + D2H)
    e2e_steps = max(1, min(args.steps, 3))
    hN, hB, hE = (torch.from_numpy(x.view(np.int32)).pin_memory() for x in (N, base, exp))
    hO = torch.empty_like(hN).pin_memory()

    def e2e_call():
        mpb.modexp_host_ptrs(hN.data_ptr(), hB.data_ptr(), hE.data_ptr(), hO.data_ptr(), count, BITS, WINDOW,
                             mpb.REDC_TRUNCATED, stream.cuda_stream)

    e2e_call()  # warm-up: the first call sizes the library's memory pool
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_call()
    barrier()
    e2e_s = rk.max(time.perf_counter() - t0)
    ok_e2e = rk.sum(0 if np.array_equal(hO.numpy().view(np.uint32), dev_out) else 1) == 0

    # config 2 at 2048 bits (BASELINE metric's "modmul/s"): MontMul and MontSqr, truncated REDC, 2^20
    # operands, inputs resident, mean CUDA-event time of 5 launches after one warm-up (not the
    # exponentiation's timed region)
    modmul = None
    if rank == 0 and not c5:
        n2 = 1 << 20
        N2, a2, b2 = I.montmul_inputs(config=2, count=n2, bits=BITS)
        dN2, da2, db2 = (mpb.to_device(x) for x in (N2, a2, b2))
        Np2, _ = mpb.mont_batch_setup(dN2, BITS)
        ws2 = mpb.mont_workspace(n2, BITS)
        o2 = mpb.empty_sliced(L, n2)

        def per_s(fn, reps=5):
            fn()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(stream)
            for _ in range(reps):
                fn()
            e1.record(stream)
            torch.cuda.synchronize()
            return n2 * reps / (e0.elapsed_time(e1) / 1000.0)

        lib, sz = mpb._lib, ws2.numel() * 4
        mm = per_s(lambda: lib.mont_batch_mul(da2.data_ptr(), db2.data_ptr(), dN2.data_ptr(), Np2.data_ptr(),
                                              o2.data_ptr(), n2, BITS, mpb.REDC_TRUNCATED, ws2.data_ptr(), sz,
                                              stream.cuda_stream))
        ms_ = per_s(lambda: lib.mont_batch_sqr(da2.data_ptr(), dN2.data_ptr(), Np2.data_ptr(), o2.data_ptr(), n2,
                                               BITS, mpb.REDC_TRUNCATED, ws2.data_ptr(), sz, stream.cuda_stream))
        c2 = imad_counts(L, 1)
        modmul = {"workload": "BASELINE config 2 at 2048 bits: 2^20 operands, truncated REDC, inputs resident",
                  "modmul_per_s": mm, "modsqr_per_s": ms_, "unit": "op/s",
                  "frac_modmul": mm * c2["mul"] / (SMS * IMAD_PER_CLK_SM * 1965e6),
                  "frac_modsqr": ms_ * c2["sqr"] / (SMS * IMAD_PER_CLK_SM * 1965e6)}
        del dN2, da2, db2, Np2, ws2, o2

    # config 4 (4096-bit modexp, w = 5, truncated REDC, 2^16 operands: one wave, one 448-thread CTA
    # per SM): mean CUDA-event time of 2 launches after one warm-up (not the headline's
    # timed region)
    config4 = None
    if rank == 0 and not c5 and not args.no_config4:
        b4, n4 = 4096, 1 << 16
        N4, B4, E4 = I.modexp_inputs(config=4, count=n4, bits=b4)
        dN4, dB4, dE4 = (mpb.to_device(x) for x in (N4, B4, E4))
        Np4, R24 = mpb.mont_batch_setup(dN4, b4)
        ws4 = mpb.modexp_workspace(n4, b4, WINDOW, 0)
        o4 = mpb.empty_sliced(I.limbs_for_bits(b4), n4)

        def run4():
            mpb.mont_batch_modexp_ct(dN4, Np4, R24, dB4, dE4, b4, WINDOW, mpb.REDC_TRUNCATED, ws=ws4, out=o4)

        run4()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(torch.cuda.current_stream())
        for _ in range(2):
            run4()
        e1.record(torch.cuda.current_stream())
        torch.cuda.synchronize()
        r4 = n4 * 2 / (e0.elapsed_time(e1) / 1000.0)
        peak = SMS * IMAD_PER_CLK_SM * 1965e6
        config4 = {"workload": "BASELINE config 4: 4096-bit CT modexp, w = 5, truncated REDC, 2^16 operands "
                               "(register-Karatsuba blocks, one 448-thread CTA per SM)",
                   "modexp_per_s": r4, "unit": "modexp/s",
                   "frac_own_count": r4 * modexp_imad(b4, WINDOW, 1, own=True) / peak,
                   "frac_schoolbook_basis": r4 * modexp_imad(b4, WINDOW, 1) / peak,
                   "parity": "tests/test_gpu_parity.py::test_config4_full_batch_sampled (same inputs)"}
        del dN4, dB4, dE4, Np4, R24, ws4, o4

    extra = {}
    if modmul:
        extra["modmul"] = modmul
    if config4:
        extra["config4"] = config4
    if c5:  # parity on the seeded 4096-element subset of the global batch + G-invariant digest
        import oracle as O

        sub = np.sort(np.random.default_rng(5).choice(COUNT5, size=4096, replace=False))
        mine = sub[(sub >= a0) & (sub < b0)] - a0
        cores = max(1, (os.cpu_count() or 1) // world)
        bad = 0
        if len(mine):
            ref = O.batch_modexp(base[mine], exp[mine], BITS, N[mine], threads=cores)
            bad = int((ref != dev_out[mine]).any(axis=1).sum())
        bad = rk.sum(bad)
        dig = shard.digest_combine(rk.gather_objects(shard.digest_part(dev_out, a0)))
        extra = {"oracle_subset": {"checked": 4096, "mismatches": bad, "seed": 5},
                 "digest": dig, "g_invariant_digest_of": f"all {COUNT5} outputs in global order"}

    if rank == 0:
        ms = total_ms / args.steps
        total = COUNT5 if c5 else world * COUNT
        value = total / (ms / 1000.0)
        kern_ms = float(np.mean(per_launch_ms))
        imad = modexp_imad(BITS, WINDOW, True) * count
        clk = clocks.summary()
        f_max = (clk["sm_max_mhz"] or 1965) * 1e6
        peak = SMS * IMAD_PER_CLK_SM * f_max
        peak_k0 = SMS * 2 * K0_PRODUCTS_PER_CLK_SM * f_max
        achieved = imad / (kern_ms / 1000.0)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong" if c5 else "weak",
            "vs_baseline": None, "dtype": "u32", "data": "synthetic", "config": config_dict(world, c5),
            "roofline": {
                "bound": "imad", "pipe": "fmaheavy (IMAD.WIDE.U32.X: one fused 32x32->64 product = 2 IMAD)",
                "kernel": "k_modexp<C=16, truncated REDC, NB=4, schoolbook>",
                "achieved": achieved / 1e12, "peak": peak / 1e12, "unit": "TIMAD/s", "frac": achieved / peak,
                "peak_basis": f"nominal: {SMS} SMs x {IMAD_PER_CLK_SM} IMAD/clk/SM x {f_max/1e6:.0f} MHz "
                              "(MEASURED_PEAKS.json has no integer peak; the profiling guide gives no integer fallback)",
                "peak_k0": peak_k0 / 1e12, "frac_k0": achieved / peak_k0,
                "peak_k0_basis": f"measured fused-chain rate {K0_PRODUCTS_PER_CLK_SM} products/clk/SM "
                                 "(profiles/r01_microbench_int.json) x 2 IMAD x SMs x clock",
                "frac_at_sampled_clock": (achieved / (SMS * IMAD_PER_CLK_SM * clk["sm_mhz"] * 1e6)
                                          if clk["sm_mhz"] else None),
                "imad_per_modexp": modexp_imad(BITS, WINDOW, True),
                "traffic": ncu_traffic()[0], "traffic_unit": "TB per launch",
                "traffic_source": ncu_traffic()[1],
            },
            "clocks": clk,
            "e2e": {"value": total * e2e_steps / e2e_s, "unit": UNIT,
                    "h2d_bytes_per_step": 3 * total * L * 4, "d2h_bytes_per_step": total * L * 4,
                    "includes": "pinned H2D of N/base/exp, layout expand, mont_batch_setup, modexp, contract, D2H",
                    "matches_device_result": bool(ok_e2e)},
            "gpu_launches": args.steps,
            "kernel_ms": {"mean": kern_ms, "min": float(np.min(per_launch_ms)), "max": float(np.max(per_launch_ms))},
            **extra,
        }
        if share:
            line["shared_gpu"] = ("MPB_BENCH_SHARE_GPU=1: all ranks on device 0 with gloo -- a check of the "
                                  "multi-rank launcher and slicing, NOT a multi-GPU measurement")
        if not args.no_cpu_baseline and world == 1:
            line["cpu_baseline"] = cpu_oracle_sample()
        print(json.dumps(line), flush=True)
    rk.close()


def _rank_main(args) -> None:
    if args.impl == "reference":
        run_reference(args, int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", args.gpus)))
    else:
        run_ours(args)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-config4", action="store_true", help="skip the extra config-4 (4096-bit) measurement")
    ap.add_argument("--workload", default="config3", choices=["config3", "config5"],
                    help="config3: 2^18 operands per GPU (weak scaling, the default); config5: one 2^22 batch "
                         "split across the GPUs (strong scaling), oracle subset + G-invariant digest")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.gpus < 1:
        raise SystemExit("--gpus must be >= 1")
    if args.impl == "ours" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # started as `python bench.py --gpus N` without torchrun: start the N ranks here
        import torch

        from paper_2410_18129_b200.launcher import spawn

        have = torch.cuda.device_count()
        if have < args.gpus and os.environ.get("MPB_BENCH_SHARE_GPU") != "1":
            raise SystemExit(f"bench.py: --gpus {args.gpus} but only {have} CUDA device(s) visible")
        spawn(args.gpus, _rank_main, args)
        return
    _rank_main(args)


if __name__ == "__main__":
    main()
