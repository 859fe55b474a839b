"""Multi-process sharding on CPU (gloo, world_size 2): block ranges are disjoint,
cover the batch, and the result gather reassembles rank shards in order.

The GPU path uses the same helpers with NCCL; no rank waits on another while
extrapolating (blocks are independent), so the only collective is the gather.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2204_14194_b200.shard import block_range, gather_blocks
from paper_2204_14194_b200 import workloads as wl


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n_blocks, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = block_range(n_blocks, rank, world)
    # each rank produces its shard from the shared seeded generator
    sig = torch.from_numpy(wl.block_signals(1, hi - lo, 8, 8, first=lo)).reshape(hi - lo, -1)
    sel = torch.arange(lo, hi, dtype=torch.int32)[:, None].repeat(1, 3)
    full_sig = gather_blocks(sig, lo, hi, n_blocks)
    full_sel = gather_blocks(sel, lo, hi, n_blocks)
    t = torch.tensor([float(rank + 1)])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)  # the bench's max-over-ranks timing
    if rank == 0:
        out_q.put((full_sig.numpy(), full_sel.numpy(), float(t)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n_blocks", [7, 16])
def test_gloo_world2_shards_and_gather(n_blocks):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_blocks, q)) for r in range(2)]
    for p in procs:
        p.start()
    sig, sel, tmax = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = wl.block_signals(1, n_blocks, 8, 8).reshape(n_blocks, -1)
    assert np.array_equal(sig, want)
    assert np.array_equal(sel[:, 0], np.arange(n_blocks))
    assert tmax == 2.0
