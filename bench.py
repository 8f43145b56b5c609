#!/usr/bin/env python
"""bench.py -- batched constant-time 2048-bit modexp on B200 (arXiv 2410.18129 hot path).

A "step" is one pass of the whole hot path over one batch: mont_batch_modexp_ct on
BASELINE.json config 3 (2048-bit moduli, window 5, truncated REDC, batch 2^18 per GPU;
table build, the 409 windows of squarings / masked table scans / multiplications, and the
exit REDC all inside one kernel).  Inputs are resident in HBM before timing starts; the
per-step working set (inputs 320 MiB + window tables and scratch 2.4 GiB) is larger than
the 126 MB L2, so no explicit flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 runs under torchrun, one rank per GPU: each rank takes its own 2^18 slice
(independent units, no data-path collective; weak scaling), timing is the max over ranks.
`--impl reference` times the plain CPU oracle (oracle/, test infrastructure) on the host
cores on bounded samples of the same workload -- the reference arm of this tier.
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
SMS, IMAD_PER_CLK_SM = 148, 64  # K0-measured 63.6 (profiles/r01_microbench_int.json)


# ------------------------------------------------------------------ roofline
def block_for(L: int) -> int:
    """Limbs per block of the kernels (the largest of 16, 12, 8, 4 dividing L)."""
    return next(c for c in (16, 12, 8, 4) if L % c == 0)


def imad_counts(L: int, redc: int) -> dict:
    """Algorithmic IMAD per operation: a 32x32->64 word product = 2 IMAD,
    a lo-only product = 1; the hi-only products of column L-2 count 1 each.
    redc: 1 truncated, 0 full, 2 CIOS (alg:8BlockMontRed at digit 2^(32C): per row of C limbs,
    2CL products for a_i*B, 2CL for m_i*N and a C x C low-half product of C^2 IMAD, so
    4L^2 + LC for a multiplication or a squaring; REDC is MontMul(X, 1))."""
    if redc == 2:
        C = block_for(L)
        mul = sqr = redc_ = 4 * L * L + L * C
    elif redc:
        mul, sqr, redc_ = 4 * L * L + 2 * L - 1, 3 * L * L + 3 * L - 1, 2 * L * L + 2 * L - 1
    else:
        mul, sqr, redc_ = 5 * L * L, 4 * L * L + L, 3 * L * L
    return {"mul": mul, "sqr": sqr, "redc": redc_}


def modexp_imad(bits: int, w: int, redc: int) -> int:
    """(W-1)*w MontSqr + (W-1) + (2^w - 1) MontMul + 2 REDC."""
    L = I.limbs_for_bits(bits)
    W = -(-bits // w)
    c = imad_counts(L, int(redc))
    return (W - 1) * w * c["sqr"] + ((W - 1) + (1 << w) - 1) * c["mul"] + 2 * c["redc"]


def ncu_traffic():
    """dram__bytes_read.sum + dram__bytes_write.sum per k_modexp launch (TB), from the committed
    `ncu --set full` capture of this exact launch (profiles/r01_v7_ncu_modexp.json), else None."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "r01_v7_ncu_modexp.json")))
        if d.get("operands_per_launch") == COUNT:
            return d["dram_bytes_per_launch"] / 1e12
    except Exception:
        pass
    return None


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


def config_dict(world: int) -> dict:
    return {"workload": "BASELINE config 3: 2048-bit constant-time fixed-window modexp, window 5, truncated "
                        "REDC, batch 2^18 per GPU (random odd moduli with top bit set, bases in [0,N), "
                        "full-length exponents)",
            "bits": BITS, "window": WINDOW, "redc": "truncated", "count_per_gpu": COUNT,
            "global_batch": COUNT * world, "parallelism": f"independent slices x{world}",
            "l2": "no flush: per-step working set (inputs 320 MiB + tables/scratch 2.5 GiB) > 126 MB L2"}


# ------------------------------------------------------------------- ours
def run_ours(args, rank: int, world: int, local_rank: int) -> None:
    import torch

    from paper_2410_18129_b200 import mpb

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))

    def barrier():
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    L = I.limbs_for_bits(BITS)
    N, base, exp = I.modexp_inputs(config=CONFIG, count=COUNT, bits=BITS, dataset=rank)
    dN, dB, dE = (mpb.to_device(x) for x in (N, base, exp))
    Np, R2 = mpb.mont_batch_setup(dN, BITS)
    ws = mpb.modexp_workspace(COUNT, BITS, WINDOW)
    out = mpb.empty_sliced(L, COUNT)
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
    total_ms = ev[0].elapsed_time(ev[-1])
    t = torch.tensor([total_ms], device="cuda")
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())

    # end to end through the public host-buffer call (pinned host memory, H2D + setup + modexp + D2H)
    e2e_steps = max(1, min(args.steps, 3))
    hN, hB, hE = (torch.from_numpy(x.view(np.int32)).pin_memory() for x in (N, base, exp))
    hO = torch.empty_like(hN).pin_memory()
    import ctypes

    lib = mpb._lib

    def e2e_call():
        rc = lib.mpb_modexp_host(hN.data_ptr(), hB.data_ptr(), hE.data_ptr(), hO.data_ptr(), COUNT, BITS, WINDOW,
                                 mpb.REDC_TRUNCATED, ctypes.c_void_p(stream.cuda_stream))
        if rc != 0:
            raise RuntimeError(lib.mpb_last_error().decode())

    e2e_call()  # warm-up: the first call sizes the stream-ordered memory pool
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_call()
    barrier()
    e2e_s = time.perf_counter() - t0
    te = torch.tensor([e2e_s], device="cuda")
    if dist:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_s = float(te.item())
    ok_e2e = np.array_equal(hO.numpy().view(np.uint32)[:4], mpb.to_host(out)[:4])

    if rank == 0:
        ms = total_ms / args.steps
        value = world * COUNT / (ms / 1000.0)
        kern_ms = float(np.mean(per_launch_ms))
        imad = modexp_imad(BITS, WINDOW, True) * COUNT
        clk = clocks.summary()
        f_max = (clk["sm_max_mhz"] or 1965) * 1e6
        peak = SMS * IMAD_PER_CLK_SM * f_max
        achieved = imad / (kern_ms / 1000.0)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u32", "data": "synthetic", "config": config_dict(world),
            "roofline": {
                "bound": "alu", "kernel": "k_modexp<C=16, truncated REDC, NB=4, schoolbook>",
                "achieved": achieved / 1e12, "peak": peak / 1e12, "unit": "TIMAD/s", "frac": achieved / peak,
                "traffic_unit": "TB per launch (DRAM, ncu; algorithmic table-scan bytes 0.88 TB)",
                "traffic": ncu_traffic(),
                "peak_basis": f"{SMS} SMs x {IMAD_PER_CLK_SM} IMAD/clk/SM (K0 measured 63.6) x {f_max/1e6:.0f} MHz",
                "frac_at_sampled_clock": (achieved / (SMS * IMAD_PER_CLK_SM * clk["sm_mhz"] * 1e6)
                                          if clk["sm_mhz"] else None),
                "imad_per_modexp": modexp_imad(BITS, WINDOW, True),
            },
            "clocks": clk,
            "e2e": {"value": world * COUNT * e2e_steps / e2e_s, "unit": UNIT,
                    "h2d_bytes_per_step": 3 * COUNT * L * 4, "d2h_bytes_per_step": COUNT * L * 4,
                    "includes": "pinned H2D of N/base/exp, layout expand, mont_batch_setup, modexp, contract, D2H",
                    "matches_device_result": bool(ok_e2e)},
            "gpu_launches": args.steps,
            "kernel_ms": {"mean": kern_ms, "min": float(np.min(per_launch_ms)), "max": float(np.max(per_launch_ms))},
        }
        if not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_oracle_sample()
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", args.gpus if args.impl == "reference" else 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
