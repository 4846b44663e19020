"""Multi-GPU partitioning of the hot path: independent replicas.

Sessions are the only unit that shards: a session's lookahead step is one
dependent chain of layers, and sessions share no state beyond the server's
session table (server.hpp:75-76).  So N GPUs run N engine replicas, one
process per GPU, and sessions are assigned to GPUs at prompt time
(round-robin, sticky afterwards).  There is no data-path collective; the
process group is only used for barriers and for reducing the measurement
(max over ranks for time, sum for tokens).  The backend is NCCL on GPUs and
gloo on CPU (used by the tests).
"""
from __future__ import annotations

import os
from dataclasses import dataclass


@dataclass
class Group:
    world: int = 1
    rank: int = 0
    local: int = 0
    backend: str = "none"

    @property
    def device(self) -> str:
        return f"cuda:{self.local}" if self.backend == "nccl" else "cpu"


def setup(backend: str | None = None) -> Group:
    """Join the process group described by torchrun's env (WORLD_SIZE, RANK,
    LOCAL_RANK, MASTER_ADDR/PORT).  world == 1 needs no group."""
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws == 1:
        return Group(1, 0, local, "none")
    import torch
    import torch.distributed as dist
    if backend is None:
        backend = "nccl" if torch.cuda.is_available() else "gloo"
    if backend == "nccl":
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group(backend)
    return Group(ws, rank, local, backend)


def teardown(g: Group) -> None:
    if g.world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def barrier(g: Group) -> None:
    if g.world == 1:
        return
    import torch
    import torch.distributed as dist
    if g.backend == "nccl":
        dist.barrier(device_ids=[g.local])
        torch.cuda.synchronize(g.local)
    else:
        dist.barrier()


def _reduce(g: Group, x: float, op_name: str) -> float:
    if g.world == 1:
        return float(x)
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64, device=g.device)
    dist.all_reduce(t, op=getattr(dist.ReduceOp, op_name))
    return float(t.item())


def max_over_ranks(g: Group, x: float) -> float:
    """Device time of a multi-GPU run = the slowest rank's."""
    return _reduce(g, x, "MAX")


def sum_over_ranks(g: Group, x: float) -> float:
    return _reduce(g, x, "SUM")


def assign_sessions(n_sessions: int, world: int) -> list[list[int]]:
    """Round-robin session -> GPU map (sticky after the prompt)."""
    if n_sessions < 0 or world < 1:
        raise ValueError("n_sessions must be >= 0 and world >= 1")
    return [list(range(r, n_sessions, world)) for r in range(world)]


def session_id(rank: int, index: int, prefix: str = "bench") -> str:
    return f"{prefix}-r{rank}-s{index}"
