"""Block sharding over GPUs: one process per GPU, no data-path collective.

FaSE blocks are independent (the reference runs them as order-independent
jobs, ``pkg/src/fase/conceal.py:3-7``), so N ranks take contiguous block
ranges and never exchange data while extrapolating. The only collective is
the optional result gather at the end (NCCL on GPUs, gloo in the CPU tests).
"""

from __future__ import annotations

import os


def block_range(n_blocks: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [lo, hi) share of ``n_blocks`` for ``rank``; sizes differ by <= 1."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank {rank} of world {world}")
    base, extra = divmod(n_blocks, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def dist_env() -> tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment (1 process: 0, 1, 0)."""
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def gather_blocks(tensor, lo: int, hi: int, n_blocks: int, group=None):
    """All-gather per-rank block rows [lo, hi) into an (n_blocks, ...) tensor.

    Ranks pad their shard to the largest shard size so one all_gather moves
    everything (NCCL for CUDA tensors, gloo for CPU tensors).
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    sizes = [block_range(n_blocks, r, world) for r in range(world)]
    width = max(h - l for l, h in sizes)
    pad = torch.zeros((width,) + tuple(tensor.shape[1:]), dtype=tensor.dtype, device=tensor.device)
    pad[: hi - lo] = tensor
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([p[: h - l] for p, (l, h) in zip(parts, sizes)], dim=0)
