"""bench.py's multi-rank launcher on CPU (gloo, world size 2): launcher.spawn starts the ranks
with the environment bench.py reads, Ranks gives the barrier / max / sum / gather it uses, and a
config-5-style run (one chunk-seeded global batch, contiguous slices, slicing-independent digest)
gives the same digest and the same outputs as one rank.  The per-slice compute is the CPU
oracle standing in for the GPU kernel (no GPU here)."""
from __future__ import annotations

import json
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_2410_18129_b200 import inputs as I
from paper_2410_18129_b200 import launcher, shard

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BITS, COUNT, CHUNK = 512, 11, 4


def _worker(out_path: str) -> None:
    import oracle as O

    rk = launcher.Ranks("gloo")
    assert rk.world == int(os.environ["WORLD_SIZE"]) and rk.rank == int(os.environ["RANK"])
    a, b = shard.rank_slice(COUNT, rk.rank, rk.world)
    N, base, exp = I.modexp_inputs_range(5, a, b, BITS, chunk=CHUNK)
    local = O.batch_modexp(base, exp, BITS, N, threads=1)
    rk.barrier()
    slowest = rk.max(float(rk.rank + 1))
    nitems = rk.sum(b - a)
    dig = shard.digest_combine(rk.gather_objects(shard.digest_part(local, a)))
    full = shard.gather_to_rank0(local, COUNT, rk.rank, rk.world) if rk.world > 1 else local
    if rk.rank == 0:
        json.dump({"world": rk.world, "slowest": slowest, "nitems": nitems, "digest": dig,
                   "full": full.tolist()}, open(out_path, "w"))
    rk.close()


@pytest.mark.parametrize("world", [1, 2])
def test_spawned_ranks_gloo_config5_style(world, tmp_path):
    out = tmp_path / f"w{world}.json"
    launcher.spawn(world, _worker, str(out))
    r = json.load(open(out))
    assert r["world"] == world
    assert r["slowest"] == float(world)  # max over ranks
    assert r["nitems"] == COUNT  # every operand counted once
    import oracle as O

    N, base, exp = I.modexp_inputs_range(5, 0, COUNT, BITS, chunk=CHUNK)
    ref = O.batch_modexp(base, exp, BITS, N, threads=2)
    assert np.array_equal(np.array(r["full"], dtype=np.uint32), ref)
    assert r["digest"] == shard.digest_combine([shard.digest_part(ref, 0)])


def test_chunked_inputs_are_slicing_independent():
    whole = I.modexp_inputs_range(5, 0, 23, 256, chunk=5)
    assert whole[0].shape == (23, I.limbs_for_bits(256))
    for a, b in [(0, 0), (0, 5), (3, 9), (5, 10), (7, 23), (22, 23)]:
        part = I.modexp_inputs_range(5, a, b, 256, chunk=5)
        for x, y in zip(part, whole):
            assert np.array_equal(x, y[a:b])
    # chunk c is exactly the dataset-c draw of the plain generator
    c1 = I.modexp_inputs(5, 5, 256, dataset=1)
    for x, y in zip(c1, whole):
        assert np.array_equal(x, y[5:10])


def test_digest_is_slicing_independent_and_order_sensitive():
    rng = np.random.default_rng(1)
    x = rng.integers(0, 1 << 32, size=(37, 8), dtype=np.uint64).astype(np.uint32)
    d1 = shard.digest_combine([shard.digest_part(x, 0)])
    for world in (2, 3, 8):
        parts = [shard.digest_part(x[a:b], a) for a, b in shard.plan(37, world)]
        assert shard.digest_combine(parts) == d1
    y = x.copy()
    y[[3, 4]] = y[[4, 3]]  # swapped rows
    assert shard.digest_combine([shard.digest_part(y, 0)]) != d1
    y = x.copy()
    y[10, 7] ^= 1  # one flipped bit
    assert shard.digest_combine([shard.digest_part(y, 0)]) != d1


def test_bench_refuses_more_gpus_than_visible():
    """`python bench.py --gpus 2` starts the ranks itself, and refuses (instead of silently timing
    one GPU) when fewer devices are visible -- here, with no GPU at all."""
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env["CUDA_VISIBLE_DEVICES"] = ""
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1"],
                       capture_output=True, text=True, env=env, timeout=300)
    assert p.returncode != 0
    assert "only 0 CUDA device" in (p.stdout + p.stderr)
