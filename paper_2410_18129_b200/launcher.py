"""One process per GPU: start N ranks on this node and give each the
torch.distributed plumbing bench.py needs -- a barrier and max/sum reductions over ranks.
No data-path collective: every operand is an independent unit (north_star (c)).

* ``spawn(world, fn, *args)``  start `world` processes (spawn start method), each with RANK,
                               LOCAL_RANK, WORLD_SIZE, MASTER_ADDR=127.0.0.1 and a free
                               MASTER_PORT in its environment, then run fn(*args); raises if a
                               rank exits non-zero.  Used when bench.py is started as
                               `python bench.py --gpus N` without torchrun.
* ``Ranks(backend)``           this process's rank/world from the environment; init the
                               process group when world > 1 ("nccl" on GPUs, "gloo" on CPU).
"""
from __future__ import annotations

import os
import socket


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _entry(rank: int, world: int, port: int, fn, args) -> None:
    os.environ.update(RANK=str(rank), LOCAL_RANK=str(rank), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1",
                      MASTER_PORT=str(port))
    fn(*args)


def spawn(world: int, fn, *args) -> None:
    """Run fn(*args) in `world` fresh processes (one per GPU), rank from the environment."""
    import torch.multiprocessing as mp

    if world < 1:
        raise ValueError("world must be >= 1")
    mp.start_processes(_entry, args=(world, free_port(), fn, args), nprocs=world, join=True, start_method="spawn")


class Ranks:
    """rank / world / local_rank from the environment (torchrun or spawn); process group when world > 1."""

    def __init__(self, backend: str = "nccl", device=None):
        self.rank = int(os.environ.get("RANK", 0))
        self.world = int(os.environ.get("WORLD_SIZE", 1))
        self.local_rank = int(os.environ.get("LOCAL_RANK", 0))
        self.backend = backend
        self.dist = None
        if self.world > 1:
            import torch.distributed as dist

            kw = {"device_id": device} if (backend == "nccl" and device is not None) else {}
            dist.init_process_group(backend, **kw)
            self.dist = dist

    def _tensor(self, v, dtype):
        import torch

        dev = f"cuda:{self.local_rank}" if self.backend == "nccl" else "cpu"
        return torch.tensor([v], dtype=dtype, device=dev)

    def barrier(self) -> None:
        if self.dist:
            self.dist.barrier()

    def max(self, v: float) -> float:
        """max over ranks (device time of the slowest rank)."""
        if not self.dist:
            return float(v)
        import torch

        t = self._tensor(float(v), torch.float64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def sum(self, v: int) -> int:
        if not self.dist:
            return int(v)
        import torch

        t = self._tensor(int(v), torch.int64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM)
        return int(t.item())

    def gather_objects(self, obj):
        """every rank's obj, in rank order, on every rank (small objects only)."""
        if not self.dist:
            return [obj]
        out = [None] * self.world
        self.dist.all_gather_object(out, obj)
        return out

    def close(self) -> None:
        if self.dist:
            self.dist.destroy_process_group()
            self.dist = None
