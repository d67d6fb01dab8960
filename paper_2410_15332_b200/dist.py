"""Multi-GPU plumbing for the data-parallel link path: one process per GPU,
independent requests sharded r -> rank r mod world, no collective on the data path.  Timing
uses a barrier on both sides of the timed region and the max over ranks.  torch.distributed is
plumbing only (NCCL on GPUs, gloo in the CPU tests)."""
from __future__ import annotations

import os
from typing import List, Sequence, Tuple, TypeVar

T = TypeVar("T")


def env_rank() -> Tuple[int, int, int]:
    """(rank, world, local_rank) from the torchrun environment (defaults: single process)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard(items: Sequence[T], rank: int, world: int) -> List[T]:
    """Request r goes to rank r mod world (deterministic, disjoint, covering)."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    return [x for i, x in enumerate(items) if i % world == rank]


def init(backend: str, device_id=None) -> None:
    import torch.distributed as dist
    if not dist.is_initialized():
        kw = {"device_id": device_id} if device_id is not None else {}
        dist.init_process_group(backend, **kw)


def barrier() -> None:
    import torch.distributed as dist
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.barrier()


def max_over_ranks(value: float, device=None) -> float:
    """Max of a scalar over all ranks (the whole-job time of a multi-GPU step)."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def tp_connect(engine, group=None) -> None:
    """Exchange the engines' CUDA IPC arena handles across the tensor-parallel group and wire the peer
    pointers of the fused all-reduce (every rank of `group` calls this once, in rank order)."""
    import torch.distributed as dist
    mine = engine.ipc_handle()
    allh = [None] * dist.get_world_size(group)
    dist.all_gather_object(allh, mine, group=group)
    engine.tp_connect(allh)
