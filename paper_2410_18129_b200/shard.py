"""Batch sharding across GPUs: every operand is an independent unit, so a
global batch is cut into contiguous slices, one per device/rank, with no collective on the data
path.  Results return by device-to-host copies only.

* ``plan(count, world)``           contiguous slices, sizes differ by at most one (the remainder
                                   goes to the last slices), identical on every rank.
* ``rank_slice(count, rank, world)``  this rank's (start, stop).
* ``modexp_devices(...)``          one process driving several GPUs: pinned host buffers, one
                                   host thread and stream per device, the slices' copies and
                                   kernels run concurrently, outputs land in the global host
                                   array at each slice's offset.
* ``digest_part / digest_combine`` a slicing-independent digest of a global result (G-invariance
                                   of config 5 across runs with different GPU counts).
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
    """Global operand-major batch -> results, computed on `devices` (one contiguous slice each).

    The batch is copied once into pinned host memory; one host thread per device then runs the
    public host-buffer call (mpb_modexp_host: async H2D of its slice, setup, modexp, D2H into the
    pinned output at the slice offset) on that device's own stream, so the devices' copies and
    kernels overlap (ctypes releases the GIL during the call)."""
    import threading

    import torch

    from . import mpb

    count, L = N.shape
    if count == 0:
        return np.empty_like(N)
    pin = [torch.from_numpy(np.ascontiguousarray(x, dtype=np.uint32).view(np.int32)).pin_memory()
           for x in (N, base, exp)]
    hout = torch.empty((count, L), dtype=torch.int32).pin_memory()
    errs: list[BaseException] = []

    def run(dev: int, a: int, b: int) -> None:
        # a failed slice is retried once on its device (a transient launch or copy error must not
        # lose the whole batch); a second failure is re-raised in the caller
        for attempt in range(2):
            try:
                torch.cuda.set_device(dev)
                s = torch.cuda.Stream(dev)
                mpb.modexp_host_ptrs(*(t[a:b].data_ptr() for t in (*pin, hout)), b - a, bits, window, redc,
                                     s.cuda_stream)
                return
            except BaseException as e:
                if attempt == 1:
                    errs.append(e)

    threads = [threading.Thread(target=run, args=(dev, a, b))
               for dev, (a, b) in zip(devices, plan(count, len(devices))) if b > a]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errs:
        raise errs[0]
    return hout.numpy().view(np.uint32).copy()


def digest_part(out: np.ndarray, start: int) -> int:
    """Order-sensitive 64-bit digest of rows start .. start+len(out)-1 of a global operand-major
    result; parts of disjoint slices combine by addition mod 2^64 (digest_combine), so the digest
    of the whole batch is the same for every slicing (config 5 G-invariance across 1/2/4/8 GPUs).
    Plumbing only (a mixing hash), not part of the method."""
    out = np.ascontiguousarray(out, dtype=np.uint32)
    n = out.shape[0]
    if n == 0:
        return 0
    w = out.view(np.uint64) if out.shape[1] % 2 == 0 else out.astype(np.uint64)
    with np.errstate(over="ignore"):
        h = np.full(n, 0x243F6A8885A308D3, np.uint64)
        for i in range(w.shape[1]):
            h = (h ^ w[:, i]) * np.uint64(0x100000001B3)
            h ^= h >> np.uint64(29)
        h ^= (np.arange(start, start + n, dtype=np.uint64) + np.uint64(1)) * np.uint64(0x9E3779B97F4A7C15)
        h = (h ^ (h >> np.uint64(31))) * np.uint64(0xBF58476D1CE4E5B9)
        h ^= h >> np.uint64(32)
        return int(h.sum(dtype=np.uint64))


def digest_combine(parts) -> str:
    return f"{sum(int(p) for p in parts) % (1 << 64):016x}"


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
