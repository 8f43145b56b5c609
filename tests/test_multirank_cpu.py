"""Multi-rank path on CPU (gloo, world size 2): the shard plan, the per-rank slices and the
gather give byte-identical results to the single-rank run (G-invariance, SURVEY 8(c) last row).
The per-slice compute is the CPU oracle standing in for the GPU kernel (no GPU here); the GPU
kernel's own G-invariance is covered by test_gpu_parity (slices of one batch == the batch)."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2410_18129_b200 import inputs as I
from paper_2410_18129_b200 import shard


@pytest.mark.parametrize("count,world", [(0, 1), (1, 2), (7, 2), (8, 8), (10, 4), (4194304, 8), (5, 8)])
def test_plan_covers_batch_contiguously(count, world):
    p = shard.plan(count, world)
    assert len(p) == world
    assert p[0][0] == 0 and p[-1][1] == count
    sizes = [b - a for a, b in p]
    assert all(p[i][1] == p[i + 1][0] for i in range(world - 1))
    assert max(sizes) - min(sizes) <= 1
    assert sizes == sorted(sizes)  # remainder on the last slices
    assert [shard.rank_slice(count, r, world) for r in range(world)] == p


def test_plan_rejects_bad_args():
    with pytest.raises(ValueError):
        shard.plan(4, 0)
    with pytest.raises(ValueError):
        shard.plan(-1, 2)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, count, bits, q):
    import oracle as O

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    N, base, exp = I.modexp_inputs(config=5, count=count, bits=bits)  # same global batch on every rank
    a, b = shard.rank_slice(count, rank, world)
    local = O.batch_modexp(base[a:b], exp[a:b], bits, N[a:b], threads=1)
    full = shard.gather_to_rank0(local, count, rank, world)
    if rank == 0:
        q.put(full)
    dist.destroy_process_group()


def test_two_rank_gloo_gather_is_g_invariant():
    count, bits, world = 11, 512, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, count, bits, q)) for r in range(world)]
    for p in procs:
        p.start()
    full = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    import oracle as O

    N, base, exp = I.modexp_inputs(config=5, count=count, bits=bits)
    assert np.array_equal(full, O.batch_modexp(base, exp, bits, N, threads=2))

