"""Block sharding over GPUs: one process per GPU, results gathered to one rank.

FaSE blocks are independent (the reference runs them as order-independent
jobs, ``pkg/src/fase/conceal.py:3-7,234-245``), so N ranks take contiguous
block ranges of ONE batch (or of one frame's lossy tiles) and never exchange
data while extrapolating. The only data-path collective is the result gather
(BASELINE north_star: "NCCL is used only to gather results"):

- every rank writes its shard's results into one contiguous byte *arena*
  (coefficients (n, I) float64 | lost samples (n, L) float64 | selections
  (n, I) int32, rows padded to the largest shard);
- one ``gather`` per batch moves every arena to the root rank (NCCL over
  NVLink on GPUs, gloo on CPU in the tests), where the per-rank views of the
  gathered buffer are the batch's results in block order, without a copy.

Frames: each rank conceals its share of the lossy tiles on the full frame;
the root pastes the other ranks' tiles from their gathered (selections,
coefficients) -- the paste is order-independent (each block writes only its
own tile, ``conceal.py:144-148``).
"""

from __future__ import annotations

import os

import numpy as np


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


def _world(group=None) -> tuple[int, int]:
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return 0, 1
    return dist.get_rank(group), dist.get_world_size(group)


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


def assemble_row_panels(G, n_rows: int, build_panel, finish=None, group=None):
    """Cooperative build of an (n_rows, ld) table: rank r fills its row panel
    ``block_range(n_rows, r, N)`` with ``build_panel(G, lo, hi)``, one broadcast
    per rank (panel sizes differ by at most one row) hands every panel to every
    rank, and ``finish(G)`` completes the table locally (the Gram build mirrors
    the upper triangle). SURVEY 8(e): each GPU computes 1/N of the row panels
    instead of the whole table."""
    import torch.distributed as dist

    rank, world = _world(group)
    lo, hi = block_range(n_rows, rank, world)
    build_panel(G, lo, hi)
    if world > 1:
        for r in range(world):
            l, h = block_range(n_rows, r, world)
            if h > l:
                dist.broadcast(G[l:h], src=r if group is None else dist.get_global_rank(group, r),
                               group=group)
    if finish is not None:
        finish(G)
    return G


def build_gram_tables_sharded(dictionary, weight, device=None, group=None):
    """``build_gram_tables`` with the table rows split over the ranks: each rank
    builds its row panel of the non-symmetric product on the tensor cores
    (``fast.gram_panel_into``), the panels are broadcast (NCCL over NVLink),
    and every rank mirrors the upper triangle and derives D. The result is
    bit-identical to the single-GPU table (entries i <= j are computed the
    same way, the mirror copies them). Dictionaries off the Ozaki table path
    (complex, small K) build the whole table on every rank."""
    import torch

    from . import _native
    from .fast import (GramTable, _device_vector, build_gram_tables, gram_panel_into,
                       gram_panel_worthwhile, gram_support, resolve_device)

    dev = resolve_device(device)
    w = np.asarray(weight, dtype=np.float64).ravel()
    K, M = len(dictionary), dictionary.area
    _, world = _world(group)
    if world == 1 or not dictionary.is_real or w.size != M:
        return build_gram_tables(dictionary, weight, device=dev)
    w_dev = _device_vector(w, dictionary.ld, dev)
    support = gram_support(w_dev, M)
    if not gram_panel_worthwhile(K, int(support[0].numel())):
        return build_gram_tables(dictionary, weight, device=dev)
    phi = dictionary.device_matrix(dev)
    G = torch.zeros((K, _native.table_ld(K)), dtype=torch.float64, device=dev)
    assemble_row_panels(
        G, K, lambda g, lo, hi: gram_panel_into(phi, w_dev, K, M, g, lo, hi, support),
        finish=lambda g: _native.mirror_upper(g, K), group=group)
    D = torch.empty(K, dtype=torch.float64, device=dev)
    alive = torch.zeros(1, dtype=torch.int32, device=dev)
    _native.gram_finish(G, K, D, alive)
    return GramTable(G=G, D=D, source=(dictionary, w.copy()), n_alive=int(alive.item()))


class ResultArena:
    """Per-rank result rows of a sharded batch in one contiguous byte buffer.

    Layout (8-byte aligned): coefficients (width, I) float64, then lost
    samples (width, L) float64 (L = 0 for frames, whose results are pasted),
    then selections (width, I) int32. ``width`` is the largest shard, so every
    rank's arena has the same size and one gather moves them all.
    """

    def __init__(self, n_blocks: int, iterations: int, n_lost: int, device, world: int,
                 rank: int, root: int = 0, slots: int = 1, complex_coef: bool = False):
        import torch

        self.cw = 2 if complex_coef else 1  # float64 words per coefficient
        self.n_blocks, self.I, self.L = n_blocks, iterations, n_lost
        self.world, self.rank, self.root = world, rank, root
        self.ranges = [block_range(n_blocks, r, world) for r in range(world)]
        self.lo, self.hi = self.ranges[rank]
        self.width = max(h - l for l, h in self.ranges)
        w, I, L, cw = self.width, iterations, n_lost, self.cw
        self.offsets = (0, 8 * w * I * cw, 8 * w * (I * cw + L))
        self.nbytes = 8 * w * (I * cw + L) + 4 * w * I
        self.nbytes += (-self.nbytes) % 8
        self.device = device
        self.bufs = [torch.zeros(self.nbytes, dtype=torch.uint8, device=device)
                     for _ in range(slots)]
        if world == 1:  # one process: the arena is the gathered buffer
            self.gathered = [b.view(1, -1) for b in self.bufs]
        else:
            self.gathered = ([torch.zeros((world, self.nbytes), dtype=torch.uint8, device=device)
                              for _ in range(slots)] if rank == root else None)

    def views(self, buf, n: int | None = None):
        """(selected (n, I) int32, coefficients (n, I) float64, lost (n, L) float64)
        views of one arena (n defaults to the width)."""
        import torch

        n = self.width if n is None else n
        w, I, L = self.width, self.I, self.L
        o_c, o_l, o_s = self.offsets
        coef = buf[o_c:o_l].view(torch.float64).view(w, I * self.cw)[:n]
        if self.cw == 2:
            coef = torch.view_as_complex(coef.view(n, I, 2))
        lost = buf[o_l:o_s].view(torch.float64).view(w, max(L, 0))[:n]
        sel = buf[o_s:o_s + 4 * w * I].view(torch.int32).view(w, I)[:n]
        return sel, coef, lost

    def local(self, slot: int = 0):
        """This rank's shard views (n = its own block count)."""
        return self.views(self.bufs[slot], self.hi - self.lo)

    def gather(self, slot: int = 0, group=None):
        """Collect every rank's arena on the root (no-op for one process)."""
        if self.world == 1:
            return
        import torch.distributed as dist

        parts = list(self.gathered[slot].unbind(0)) if self.rank == self.root else None
        dist.gather(self.bufs[slot], gather_list=parts, dst=self.root, group=group)

    def shards(self, slot: int = 0, gathered=None):
        """On the root: [(lo, hi, selected, coefficients, lost)] per rank, views
        of the gathered buffer (or of ``gathered``, e.g. its host copy)."""
        g = self.gathered[slot] if gathered is None else gathered
        return [(lo, hi, *self.views(g[r], hi - lo)) for r, (lo, hi) in enumerate(self.ranges)]

    def assemble(self, slot: int = 0, gathered=None):
        """(selected (B, I), coefficients (B, I), lost (B, L)) concatenated in block
        order (a copy; tests and host consumers)."""
        import torch

        parts = self.shards(slot, gathered)
        return tuple(torch.cat([p[k] for p in parts], dim=0) for k in (2, 3, 4))


class ShardedBatch:
    """One shared-geometry batch of ``n_blocks`` blocks sharded over the ranks.

    Rank r extrapolates ``block_range(n_blocks, r, N)`` through its own
    ``ExtrapolationPlan`` (writing into its result arena); ``run`` then gathers
    the arenas to the root in one collective. Timing a step as the max over
    ranks of (extrapolate + gather) is the strong-scaling cost of the batch.
    """

    def __init__(self, dictionary, mask, n_blocks: int, config, tables, device,
                 products: str = "auto", recursion: str = "exact", root: int = 0, group=None):
        from .fast import ExtrapolationPlan

        self.rank, self.world = _world(group)
        self.group, self.root = group, root
        probe = np.asarray(mask, dtype=bool)
        n_lost = int(probe.sum())
        self.arena = ResultArena(n_blocks, config.iterations, max(n_lost, 1), device, self.world,
                                 self.rank, root, slots=2, complex_coef=not dictionary.is_real)
        self.lo, self.hi = self.arena.lo, self.arena.hi
        sel, coef, lost = self.arena.local(0)
        self.plan = ExtrapolationPlan(dictionary, mask, self.hi - self.lo, config, tables,
                                      device=device, products=products, recursion=recursion,
                                      outputs={"selected": sel, "coefficients": coef, "lost": lost})
        self.n_blocks = n_blocks

    @property
    def is_root(self) -> bool:
        return self.rank == self.root

    def run(self, signals=None):
        """Extrapolate this rank's shard (``signals``: its (n, M, N) rows) and
        gather every shard to the root. Enqueued on the current stream."""
        self.plan.run(signals)
        self.arena.gather(0, self.group)
        return self

    def results(self):
        """On the root: per-rank (lo, hi, selected, coefficients, lost) views."""
        return self.arena.shards(0)

    def host_arena(self):
        """A pinned host buffer for the root's gathered arena (run_host_stream)."""
        import torch

        return torch.empty((self.world, self.arena.nbytes), dtype=torch.uint8, pin_memory=True)

    def run_host_stream(self, host_inputs, host_arenas):
        """End to end over a sequence of batches: each rank uploads its shard of
        every batch (pinned (n, M, N) float64), extrapolates it, the shards are
        gathered on the root, and the root reads the gathered arena back into
        ``host_arenas[i]`` (pinned, from ``host_arena``; ignored on other ranks).
        Consecutive batches alternate between two compute streams as in
        ``ExtrapolationPlan.run_host_stream``."""
        import torch

        plan = self.plan
        sel1, coef1, lost1 = self.arena.local(1)
        slot1 = (sel1, torch.empty_like(plan.projections), coef1, lost1)

        def finish(slot, hout):
            self.arena.gather(slot, self.group)
            return [(hout, self.arena.gathered[slot])] if self.is_root else []

        outs = host_arenas if self.is_root else [None] * len(host_inputs)
        return plan.run_host_stream(host_inputs, outs, slot_outputs=slot1, finish=finish)


class ShardedFrame:
    """The lossy tiles of frames of one geometry sharded over the ranks.

    Every rank holds the whole frame (its tiles' areas reach into the
    neighbours) and conceals tiles ``block_range(L, r, N)`` with its own
    ``FrameEngine``; the (selections, coefficients) arenas are gathered to the
    root, which pastes the other ranks' tiles into its frame.
    """

    def __init__(self, engine, grid, corners, root: int = 0, group=None):
        import torch

        self.engine, self.grid = engine, grid
        self.rank, self.world = _world(group)
        self.group, self.root = group, root
        L = int(corners.shape[0])
        self.arena = ResultArena(L, engine.config.iterations, 0, engine.device, self.world,
                                 self.rank, root, slots=2,
                                 complex_coef=getattr(engine, "complex", False))
        self.lo, self.hi = self.arena.lo, self.arena.hi
        self.corners = corners
        self.local_corners = corners[self.lo:self.hi].contiguous()
        self.rank_corners = [corners[lo:hi].contiguous() for lo, hi in self.arena.ranges]
        self.n_blocks = L
        self._torch = torch

    @property
    def is_root(self) -> bool:
        return self.rank == self.root

    def _paste_others(self, out, slot: int):
        from . import _native

        if not self.is_root or self.world == 1:
            return
        eng = self.engine
        paste = _native.frame_paste_complex if getattr(eng, "complex", False) else _native.frame_paste
        for r, (lo, hi, sel, coef, _) in enumerate(self.arena.shards(slot)):
            if r == self.rank or hi == lo:
                continue
            paste(eng.phi, sel, coef, eng.config.iterations, self.grid, eng.tile, eng.support,
                  self.rank_corners[r], out)

    def run(self, frame, out=None, slot: int = 0):
        """Conceal this rank's tiles of ``frame`` (device float64) into ``out``,
        gather, and (root) paste every other rank's tiles. Enqueued."""
        sel, coef, _ = self.arena.local(slot)
        res = self.engine.run(frame, self.grid, self.local_corners, out=out, slot=slot,
                              outputs=(sel, coef))
        self.arena.gather(slot, self.group)
        self._paste_others(res.patched, slot)
        return res

    def run_host_stream(self, frames_u8, outs, lost):
        """End to end: every rank uploads each pinned uint8 frame, conceals its
        tiles, the results are gathered and the root pastes the rest and reads
        the restored float64 frame back into ``outs[i]`` (root only)."""

        def finish(slot, f64, hout):
            self.arena.gather(slot, self.group)
            self._paste_others(f64, slot)
            return [(hout, f64)] if self.is_root else []

        sels = [self.arena.local(s)[:2] for s in (0, 1)]
        return self.engine.run_host_stream(frames_u8, outs, self.grid, self.local_corners, lost,
                                           slot_outputs=sels, finish=finish)
