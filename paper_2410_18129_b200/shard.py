"""Batch sharding across GPUs: every operand is an independent unit, so a
global batch is cut into contiguous slices, one per device/rank, with no collective on the data
path.  Results return by device-to-host copies only.

* ``plan(count, world)``           contiguous slices, sizes differ by at most one (the remainder
                                   goes to the last slices), identical on every rank.
* ``rank_slice(count, rank, world)``  this rank's (start, stop).
* ``modexp_devices(...)``          one process driving several GPUs: one stream per device, the
                                   slices run concurrently, outputs are written into the global
                                   host array at each slice's offset.
* ``gather_to_rank0(...)``         multi-process convenience (torch.distributed, any backend):
                                   rank 0 receives every slice's output as host bytes.  Not part
                                   of the timed path.
"""
from __future__ import annotations

import numpy as np


def plan(count: int, world: int) -> list[tuple[int, int]]:
    """Contiguous slices [start, stop) for `world` shards of `count` units."""
    if world < 1:
        raise ValueError("world must be >= 1")
    if count < 0:
        raise ValueError("count must be >= 0")
    base, rem = divmod(count, world)
    out, start = [], 0
    for r in range(world):
        n = base + (1 if r >= world - rem else 0)
        out.append((start, start + n))
        start += n
    assert start == count
    return out


def rank_slice(count: int, rank: int, world: int) -> tuple[int, int]:
    return plan(count, world)[rank]


def modexp_devices(N: np.ndarray, base: np.ndarray, exp: np.ndarray, bits: int, devices: list[int],
                   window: int = 5, redc: int = 1) -> np.ndarray:
    """Global operand-major batch -> results, computed on `devices` (one slice each, concurrently)."""
    import torch

    from . import mpb

    count = N.shape[0]
    out = np.empty_like(N)
    work = []
    for dev, (a, b) in zip(devices, plan(count, len(devices))):
        if b == a:
            continue
        with torch.cuda.device(dev):
            s = torch.cuda.Stream(dev)
            with torch.cuda.stream(s):
                dN, dB, dE = (mpb.to_device(np.ascontiguousarray(x[a:b]), f"cuda:{dev}") for x in (N, base, exp))
                Np, R2 = mpb.mont_batch_setup(dN, bits)
                res = mpb.mont_batch_modexp_ct(dN, Np, R2, dB, dE, bits, window, redc)
                host = mpb.layout_contract(res).to("cpu", non_blocking=True)
            work.append((dev, s, host, a, b))
    for dev, s, host, a, b in work:
        s.synchronize()
        out[a:b] = host.numpy().view(np.uint32)
    return out


def gather_to_rank0(local: np.ndarray, count: int, rank: int, world: int, group=None):
    """Every rank passes its slice's output (operand-major uint32); rank 0 gets the global array."""
    import torch.distributed as dist

    parts = [None] * world if rank == 0 else None
    dist.gather_object(np.ascontiguousarray(local), parts, dst=0, group=group)
    if rank != 0:
        return None
    L = local.shape[1]
    out = np.empty((count, L), np.uint32)
    for r, (a, b) in enumerate(plan(count, world)):
        out[a:b] = parts[r]
    return out
