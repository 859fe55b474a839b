"""Frame concealment over many loss blocks at once (BASELINE configs 2 and 3).

The reference conceals an image tile by tile (``pkg/src/fase/conceal.py:111-245``):
area = tile +- support, weight from every lost pixel inside the area, FaSE,
then only the tile's own lost pixels are pasted back (``conceal.py:144-148``).
Here all lossy tiles of a frame form ONE batch with fixed-size areas
(out-of-frame samples are unavailable, BASELINE config 2: "lost and
unavailable samples set to zero"). Interior tiles give exactly the reference's
per-tile result; border tiles differ from the reference's *clipped* areas by
design.

``FrameEngine`` is the device pipeline for the usual case of whole-tile
(macroblock) losses. Because every area sits at the same offset to the tile
grid, the area splits into the same *cells* (rectangles cut by tile lines and
frame edges) for every block, and each cell is entirely available or entirely
unavailable in any block. So the tables are frame-independent:
- G0 is the table of the weight without the own tile;
- C_c is the table of cell c alone.
A block's table is G0 - sum of its unavailable cells' tables, applied row by row
inside the recursion kernel. Per frame, only kernels run:
1. area extraction;
2. per-block cell lists;
3. normalizers;
4. the DMMA GEMM for the initial products;
5. the recursion;
6. paste into the frame.
"""

from __future__ import annotations

import math
import os
import time

import numpy as np

from . import _native
from .dictionary import Dictionary, parse_dict_spec
from .errors import ParameterError, ShapeError, UnsupportedDictionaryError
from .fast import ChunkedTables, fase_extrapolate_batch, resolve_device
from .grid import ExtrapConfig, as_mask, base_weight, psnr_over_region
from .model import BatchResult
from .workloads import frame_areas

REPORT_SCHEMA = "fase-b200-conceal-report/1"


def lossy_tiles(lost: np.ndarray, block: tuple[int, int]) -> np.ndarray:
    """(L, 2) top-left corners of full tiles that contain a lost pixel, row-major."""
    bh, bw = block
    h, w = lost.shape
    rows, cols = h // bh, w // bw
    tiles = lost[: rows * bh, : cols * bw].reshape(rows, bh, cols, bw).any(axis=(1, 3))
    r, c = np.nonzero(tiles)
    return np.stack([r * bh, c * bw], axis=1).astype(np.int64)


def tile_grid(lost: np.ndarray, tile: int):
    """Tile loss grid (Ty, Tx) uint8 if losses are whole full tiles, else None."""
    h, w = lost.shape
    ty, tx = h // tile, w // tile
    full = lost[: ty * tile, : tx * tile].reshape(ty, tile, tx, tile)
    anyl = full.any(axis=(1, 3))
    if not np.array_equal(full.all(axis=(1, 3)), anyl):
        return None
    if lost[ty * tile:, :].any() or lost[:, tx * tile:].any():
        return None
    return anyl.astype(np.uint8)


def _cuts(n: int, tile: int, support: int, area: int) -> list[int]:
    """Area coordinates where the tile grid or a frame edge crosses, for any tile row."""
    cuts = {0, area}
    for i in range(1, area):
        if (i - support) % tile == 0:
            cuts.add(i)
    for r0 in range(0, (n // tile) * tile, tile):
        for edge in (support - r0, n - r0 + support):
            if 0 < edge < area:
                cuts.add(edge)
    return sorted(cuts)


# device bytes the frame engine may spend on precomposed base tables (at most
# half the free memory): config 3 takes 78 GB for all cell triples on a B200
COMPOSE_BUDGET = 96 << 30
# longest-processing-time-first dispatch of the frame recursion (fase_block_order);
# FASE_BLOCK_ORDER=0 keeps the row-major tile order (measurement)
BLOCK_ORDER = os.environ.get("FASE_BLOCK_ORDER", "1") != "0"


class FrameEngine:
    """Device pipeline concealing the lossy tiles of frames of one geometry."""

    def __init__(self, dictionary: Dictionary, frame_shape: tuple[int, int], tile: int,
                 support: int, config: ExtrapConfig = ExtrapConfig(), device=None,
                 compose: str = "auto"):
        """``compose``: precomposed base tables for the first chunks of a block's
        cell list -- "none", "singles" (G0 - C_c for every cell), "pairs" (also
        G0 - C_c1 - C_c2 for every cell pair), "triples" or "auto" (the deepest
        that fits the memory budget COMPOSE_BUDGET). Composition
        runs in list order, so every variant streams bit-identical rows; the
        composed ones stream one or two fewer rows per block-iteration
        (triples: config 2 2.22 -> 1.10 rows, config 3 5.95 -> 3.10)."""
        import torch

        self.device = dev = resolve_device(device)
        a = tile + 2 * support
        if dictionary.shape != (a, a):
            raise ShapeError(f"dictionary area {dictionary.shape} vs extrapolation area {(a, a)}")
        # complex dictionaries (the reference's default `dft`, conceal.py:169):
        # conjugate-split Phi, tables of rows of conj(C), the complex recursion
        # and paste (iterate_complex.cu, fase_frame_paste_complex)
        self.complex = cplx = not dictionary.is_real
        self.dictionary, self.config = dictionary, config
        self.H, self.W = frame_shape
        self.tile, self.support, self.A = tile, support, a
        K, M = len(dictionary), a * a
        self.K, self.M = K, M
        rows = _cuts(self.H, tile, support, a)
        cols = _cuts(self.W, tile, support, a)
        cells = [(i0, i1, j0, j1) for i0, i1 in zip(rows[:-1], rows[1:])
                 for j0, j1 in zip(cols[:-1], cols[1:])]
        own = [c for c in cells if c[0] >= support and c[1] <= support + tile
               and c[2] >= support and c[3] <= support + tile]
        self.cells = [c for c in cells if c not in own]
        base = base_weight(a, a, config.rho_hat)
        w0 = base.copy()
        w0[support:support + tile, support:support + tile] = 0.0
        self.phi = phi = dictionary.device_matrix(dev)
        ld = dictionary.ld
        from .fast import _device_vector, _gram_on_device
        t0 = time.perf_counter()
        self.G0 = _gram_on_device(phi, _device_vector(w0.ravel(), ld, dev), K, M, dev,
                                  complex_rows=cplx)
        ldg = self.G0.shape[1]
        self.tables = torch.zeros((max(len(self.cells), 1), K, ldg), dtype=self.G0.dtype,
                                  device=dev)
        flat_base = base.ravel()
        for c, (i0, i1, j0, j1) in enumerate(self.cells):
            ii, jj = np.meshgrid(np.arange(i0, i1), np.arange(j0, j1), indexing="ij")
            samples = (ii * a + jj).ravel()
            cols_t = torch.from_numpy(samples.astype(np.int64)).to(dev)
            width = samples.size + (samples.size & 1)
            sub = torch.zeros((phi.shape[0], width), dtype=torch.float64, device=dev)
            sub[:, : samples.size] = phi.index_select(1, cols_t)
            wj = torch.zeros(width, dtype=torch.float64, device=dev)
            wj[: samples.size] = torch.from_numpy(flat_base[samples]).to(dev)
            (_native.gram_complex if cplx else _native.gram)(sub, wj, K, samples.size,
                                                             self.tables[c])
        self.bases, self.compose = self._compose_bases(compose)
        # dense initial products on the tcgen05 tensor cores (Ozaki digit planes);
        # complex sets: separable DFT row ranges through the complex transform
        self._oz_phi = None
        self._cparts = dictionary.device_cfactors(dev) if cplx else []
        if not (self._cparts if cplx else dictionary.device_factors(dev)):
            from .fast import ozaki_worthwhile

            if ozaki_worthwhile(4096, phi.shape[0]):
                self._oz_phi = _native.OzakiOperand(phi.shape[0], M, 64, dev).split(phi[:, :ld])
        torch.cuda.current_stream(dev).synchronize()
        self.table_seconds = time.perf_counter() - t0
        self.stride = self.tables[0].numel()
        # diagonals of G0 and of every cell table for the per-frame normalizers:
        # contiguous, L2-resident reads instead of one sector per diagonal element
        # (complex tables: the real diagonal, exactly what fase_block_normalizers
        # reads from a complex table with its complex stride)
        self._diag_G0 = self.G0.diagonal()[:K].real.contiguous()
        self._diag_tabs = self.tables.diagonal(dim1=1, dim2=2)[:, :K].real.contiguous()
        self.cell_rep = torch.tensor([[c[0], c[2]] for c in self.cells] or [[0, 0]],
                                     dtype=torch.int32, device=dev)
        self.base_w = torch.from_numpy(flat_base.copy()).to(dev)
        self._buf = {}

    def _compose_bases(self, mode: str):
        """(bases, compose map): bases[0] is G0 and bases[p] = G0 - C_c1 - ... - C_ck
        for ascending cell prefixes up to the mode's depth (singles 1, pairs 2,
        triples 3), composed element by element in list order (IEEE
        subtraction, as the recursion kernel composes rows). The map is indexed
        by the prefix padded with its last cell (fase_iterate_args.compose)."""
        import itertools

        import torch

        depths = {"none": 0, "singles": 1, "pairs": 2, "triples": 3}
        if mode != "auto" and mode not in depths:
            raise ParameterError(f"compose must be auto or one of {sorted(depths)}, got {mode!r}")
        n = len(self.cells)

        def n_bases(depth):
            return 1 + sum(math.comb(n, k) for k in range(1, depth + 1))

        if mode == "auto":
            table = self.G0.numel() * self.G0.element_size()
            budget = min(COMPOSE_BUDGET, torch.cuda.mem_get_info(self.device)[0] // 2)
            mode = next((m for m in ("triples", "pairs", "singles")
                         if n_bases(depths[m]) * table <= budget), "none")
        depth = depths[mode] if n else 0
        self.compose_mode = mode if depth else None
        if not depth:
            return None, None
        K, ldg = self.G0.shape
        bases = torch.empty((n_bases(depth), K, ldg), dtype=self.G0.dtype, device=self.device)
        bases[0].copy_(self.G0)
        cmap = np.zeros((n,) * depth, dtype=np.int32)
        index = {(): 0}
        p = 1
        for k in range(1, depth + 1):
            for pre in itertools.combinations(range(n), k):
                torch.sub(bases[index[pre[:-1]]], self.tables[pre[-1]], out=bases[p])
                index[pre] = p
                cmap[pre + (pre[-1],) * (depth - k)] = p
                p += 1
        self.G0 = bases[0]  # one allocation: base p at G0 + p * stride
        return bases, torch.from_numpy(cmap).to(self.device)

    def _buffers(self, L: int, slot: int = 0):
        import torch

        key = (L, slot)
        if key not in self._buf:
            dev, K, I = self.device, self.K, self.config.iterations
            ldx = self.M + (self.M & 1)
            vdt = torch.complex128 if self.complex else torch.float64
            self._buf = {k: v for k, v in self._buf.items() if k[0] == L}  # one batch size kept
            self._buf[key] = dict(
                X=torch.empty((L, ldx), dtype=torch.float64, device=dev),
                R0=torch.empty((L, K + (K & 1)), dtype=vdt, device=dev),
                D=torch.empty((L, self.G0.shape[1]), dtype=torch.float64, device=dev),
                alive=torch.empty(L, dtype=torch.int32, device=dev),
                counts=torch.empty(L, dtype=torch.int32, device=dev),
                order=torch.empty(L, dtype=torch.int32, device=dev),
                ids=torch.zeros((L, max(len(self.cells), 1)), dtype=torch.int32, device=dev),
                sel=torch.empty((L, I), dtype=torch.int32, device=dev),
                proj=torch.empty((L, I), dtype=vdt, device=dev),
                coef=torch.empty((L, I), dtype=vdt, device=dev),
                max_imag=torch.zeros(L, dtype=torch.float64, device=dev) if self.complex else None,
            )
            from .fast import ozaki_worthwhile

            if self._oz_phi is not None and ozaki_worthwhile(L, self.phi.shape[0]):
                self._buf[key]["oz"] = _native.OzakiOperand(L, self.M, 128, dev)
        return self._buf[key]

    @property
    def launches_per_frame(self) -> int:
        """areas, cells, normalizers, products (one per separable part or one GEMM),
        iterate, paste"""
        if self.complex and self._cparts:
            from .fast import _ranges

            return 5 + len(self._cparts) + len(_ranges(self._uncovered()))
        factors = None if self.complex else self.dictionary.device_factors(self.device)
        if factors:
            return 5 + (1 if len(factors) <= 8 else len(factors))
        return 5 + (2 if any("oz" in b for b in self._buf.values()) else 1)

    def _uncovered(self):
        flags = np.ones(self.K, dtype=bool)
        for rre, _, cre, _, row0 in self._cparts:
            flags[row0: row0 + rre.shape[0] * cre.shape[0]] = False
        return flags

    def _products(self, b):
        """R0 of the frame's areas from the weighted areas X (frame_areas)."""
        from .fast import _ranges, _real_view

        X, R0 = b["X"], b["R0"]
        if self.complex:
            if self._cparts:  # conj(E) X conj(F)^T per separable part; the rest by GEMM
                try:
                    for rre, rim, cre, cim, row0 in self._cparts:
                        _native.sep_products_complex(rre, rim, cre, cim, X, self.A, self.A, R0,
                                                     row0)
                    uncovered = self._uncovered()
                except UnsupportedDictionaryError:  # area too large for the transform
                    uncovered = np.ones(self.K, dtype=bool)
                Rv = _real_view(R0)
                for lo, hi in _ranges(uncovered):
                    _native.gemm_nt(X[:, : self.M], self.phi[2 * lo: 2 * hi, : self.M], Rv[:, 2 * lo:])
            elif self._oz_phi is not None and "oz" in b:
                _native.ozaki_gemm(b["oz"].split(X), self._oz_phi, _real_view(R0))
            else:
                _native.gemm_nt(X[:, : self.M], self.phi[:, : self.M], _real_view(R0))
            return
        factors = self.dictionary.device_factors(self.device)
        if factors:
            try:
                if len(factors) <= 8:  # separable parts on DMMA, one launch
                    _native.sep_products_batch(factors, X, None, self.A, self.A, R0)
                else:  # rows X cols^T per part (csrc/separable.cu)
                    for rows, cols, row0 in factors:
                        _native.sep_products(rows, cols, X, self.A, self.A, R0, row0)
                return
            except UnsupportedDictionaryError:  # area too large for the transform
                pass
        if self._oz_phi is not None and "oz" in b:
            _native.ozaki_gemm(b["oz"].split(X), self._oz_phi, R0)
        else:
            _native.gemm_nt(X[:, : self.M], self.phi[:, : self.M], R0)

    def run(self, frame, grid, corners, out=None, slot: int = 0, outputs=None) -> BatchResult:
        """Conceal one frame: ``frame`` (H, W) float64, ``grid`` (H/tile, W/tile)
        uint8 tile loss map, ``corners`` (L, 2) int32 lossy-tile corners, all on
        the device. The restored frame is written to ``out`` (default: a copy of
        ``frame``). Enqueued on the current stream; no host synchronization.
        ``slot`` picks one of two work-buffer sets (two frames in flight).
        ``outputs``: optional caller-owned (selected (L, I) int32, coefficients
        (L, I) float64) device buffers to write instead of the engine's (views
        of a result arena a collective gathers, ``shard.ShardedFrame``)."""
        L = int(corners.shape[0])
        if out is None:
            out = frame.clone()
        if L == 0:
            return BatchResult(selected=None, projections=None, coefficients=None, patched=out)
        b = self._buffers(L, slot)
        if outputs is not None:
            import torch

            sel, coef = outputs
            I = self.config.iterations
            cdt = torch.complex128 if self.complex else torch.float64
            if (tuple(sel.shape) != (L, I) or sel.dtype != torch.int32 or tuple(coef.shape) != (L, I)
                    or coef.dtype != cdt or not (sel.is_contiguous() and coef.is_contiguous())):
                raise ShapeError(f"outputs must be contiguous (L, I) int32 / {cdt} buffers")
            b = dict(b, sel=sel, coef=coef)
        cfg, K = self.config, self.K
        _native.frame_areas(frame, grid, self.tile, self.support, corners, self.base_w, b["X"])
        _native.frame_cells(grid, self.H, self.W, self.tile, self.support, corners, self.cell_rep,
                            b["counts"], b["ids"])
        _native.block_normalizers(self._diag_G0, self._diag_tabs, K, b["counts"], b["ids"], K,
                                  b["D"], b["alive"])
        self._products(b)
        # costliest blocks first (chunk rows beyond the precomposed base), so the
        # last wave of CTAs holds the cheap ones; a schedule only, results unchanged
        order = None
        if BLOCK_ORDER:
            depth = self.compose.dim() if self.compose is not None else 0
            _native.block_order(b["counts"], depth, b["order"])
            order = b["order"]
        (_native.iterate_complex if self.complex else _native.iterate)(
            self.G0, b["D"], b["R0"], K, cfg.iterations, cfg.gamma, b["sel"], b["proj"], b["coef"],
            chunk_tables=self.tables, chunk_stride=self.stride, chunk_count=b["counts"],
            chunk_ids=b["ids"], compose=self.compose, base_stride=self.G0.numel(), order=order)
        if self.complex:
            _native.frame_paste_complex(self.phi, b["sel"], b["coef"], cfg.iterations, grid,
                                        self.tile, self.support, corners, out, b["max_imag"])
        else:
            _native.frame_paste(self.phi, b["sel"], b["coef"], cfg.iterations, grid, self.tile,
                                self.support, corners, out)
        return BatchResult(selected=b["sel"], projections=b["proj"], coefficients=b["coef"],
                           patched=out, dictionary=self.dictionary,
                           shape=(self.A, self.A), max_imag=b["max_imag"])

    def run_host_stream(self, frames_u8, outs, grid, corners, lost, *, slot_outputs=None,
                        finish=None):
        """End to end over a sequence of frames with one loss pattern: pinned
        uint8 frames in, restored float64 frames (pinned) out. Frames alternate
        between two compute streams with their own buffers; uploads and
        read-backs run on their own streams, overlapped with the neighbouring
        frames' kernels. ``grid`` / ``corners`` / ``lost`` (H x W bool) live on
        the device. Enqueued; the caller's stream waits for the last read-back.
        ``slot_outputs`` optionally gives per-slot (selected, coefficients)
        buffers for ``run``; ``finish(slot, frame, hout)``, called on the
        slot's compute stream after ``run``, returns the (host, device) copies
        to make instead of the default frame read-back (``shard.ShardedFrame``)."""
        import torch

        dev = self.device
        cs = torch.cuda.current_stream(dev)
        H, W = self.H, self.W
        if not hasattr(self, "_pipe"):
            self._pipe = {"h2d": torch.cuda.Stream(dev), "d2h": torch.cuda.Stream(dev),
                          "comp": [torch.cuda.Stream(dev), torch.cuda.Stream(dev)],
                          "u8": [torch.empty((H, W), dtype=torch.uint8, device=dev) for _ in range(2)],
                          "f64": [torch.empty((H, W), dtype=torch.float64, device=dev)
                                  for _ in range(2)]}
        p = self._pipe
        start = torch.cuda.Event()
        start.record(cs)
        for st in (p["h2d"], p["d2h"], *p["comp"]):
            st.wait_event(start)
        ev_in = [torch.cuda.Event(), torch.cuda.Event()]
        ev_used = [None, None]
        ev_out = [None, None]
        for i, (hin, hout) in enumerate(zip(frames_u8, outs)):
            s = i % 2
            with torch.cuda.stream(p["h2d"]):
                if ev_used[s] is not None:
                    p["h2d"].wait_event(ev_used[s])
                p["u8"][s].copy_(hin, non_blocking=True)
                ev_in[s].record(p["h2d"])
            c = p["comp"][s]
            with torch.cuda.stream(c):
                c.wait_event(ev_in[s])
                if ev_out[s] is not None:
                    c.wait_event(ev_out[s])
                f64 = p["f64"][s]
                _native.frame_widen(p["u8"][s], lost, f64)  # widen + zero the lost pixels
                ev_used[s] = torch.cuda.Event()
                ev_used[s].record(c)
                self.run(f64, grid, corners, out=f64, slot=s,
                         outputs=None if slot_outputs is None else slot_outputs[s])
                copies = [(hout, f64)] if finish is None else finish(s, f64, hout)
                done = torch.cuda.Event()
                done.record(c)
            with torch.cuda.stream(p["d2h"]):
                p["d2h"].wait_event(done)
                for dst, src in copies:
                    dst.copy_(src, non_blocking=True)
                ev_out[s] = torch.cuda.Event()
                ev_out[s].record(p["d2h"])
        for e in ev_out:
            if e is not None:
                cs.wait_event(e)
        return outs

    def dead_blocks(self) -> int:
        """Blocks of the last run whose every atom was degenerate (syncs)."""
        for b in self._buf.values():
            return int((b["alive"] == 0).sum().item())
        return 0


class FramePlan:
    """Host-built geometry for arbitrary (not tile-aligned) loss masks."""

    def __init__(self, image, lost, block: int, support: int, device):
        import torch

        self.device = device
        img = np.asarray(image, dtype=np.float64)
        self.lost = as_mask(lost)
        if img.ndim != 2 or img.shape != self.lost.shape:
            raise ShapeError(f"image {img.shape} vs mask {self.lost.shape}")
        if block < 1 or support < 0:
            raise ParameterError(f"block must be >= 1 and support >= 0 (got {block}, {support})")
        self.shape = img.shape
        self.block = block
        self.support = support
        self.corners = lossy_tiles(self.lost, (block, block))
        damaged = img.copy()
        damaged[self.lost] = 0.0
        signals, masks = frame_areas(damaged, self.lost, self.corners, block, support)
        self.masks = masks
        self.signals = torch.from_numpy(signals).to(device)
        a = block + 2 * support
        h, w = self.shape
        idx, dst, ptr = [], [], [0]
        for (r0, c0) in self.corners:
            tile = self.lost[r0:r0 + block, c0:c0 + block]
            tr, tc = np.nonzero(tile)
            idx.append(((tr + support) * a + (tc + support)).astype(np.int32))
            dst.append(((r0 + tr) * w + (c0 + tc)).astype(np.int64))
            ptr.append(ptr[-1] + len(tr))
        self.idx = torch.from_numpy(np.concatenate(idx) if idx else np.zeros(0, np.int32)).to(device)
        self.dst = torch.from_numpy(np.concatenate(dst) if dst else np.zeros(0, np.int64)).to(device)
        self.ptr = torch.from_numpy(np.asarray(ptr, dtype=np.int32)).to(device)
        self.frame = torch.from_numpy(damaged).to(device)

    @property
    def n_blocks(self) -> int:
        return len(self.corners)


def conceal_frame(image, lost_mask, *, dictionary: Dictionary | None = None,
                  dict_spec: str = "union:dct+had", config: ExtrapConfig = ExtrapConfig(),
                  block: int = 16, support: int = 16, reference=None, engine=None, device=None):
    """Conceal every lossy ``block`` x ``block`` tile of a frame on the GPU.

    Whole-tile losses take the FrameEngine pipeline (pass ``engine`` to reuse
    its frame-independent tables across frames); other masks take the general
    per-block path. Returns (restored float64 frame as a device tensor, report).
    """
    import torch

    dev = resolve_device(device)
    t0 = time.perf_counter()
    img = np.asarray(image, dtype=np.float64)
    lost = as_mask(lost_mask)
    if img.shape != lost.shape or img.ndim != 2:
        raise ShapeError(f"image {img.shape} vs mask {lost.shape}")
    a = block + 2 * support
    if dictionary is None:
        dictionary = parse_dict_spec(dict_spec, a, a)
    grid = tile_grid(lost, block)  # whole-tile losses: the FrameEngine (real and complex sets)
    damaged = img.copy()
    damaged[lost] = 0.0
    if grid is not None:
        if engine is None:
            engine = FrameEngine(dictionary, img.shape, block, support, config, dev)
        corners = lossy_tiles(lost, (block, block)).astype(np.int32)
        frame = torch.from_numpy(damaged).to(dev)
        res = engine.run(frame, torch.from_numpy(grid).to(dev), torch.from_numpy(corners).to(dev))
        out = res.patched
        n_blocks = len(corners)
    else:
        plan = FramePlan(img, lost, block, support, dev)
        out = plan.frame.clone()
        n_blocks = plan.n_blocks
        res = None
        if plan.n_blocks:
            tables = ChunkedTables(dictionary, plan.masks, config.rho_hat, dev)
            res = fase_extrapolate_batch(plan.signals, plan.masks, dictionary, tables, config,
                                         patch=False, device=dev)
            synth = _native.synth_paste if dictionary.is_real else _native.synth_paste_complex
            synth(dictionary.device_matrix(dev), res.selected, res.coefficients,
                  config.iterations, plan.idx, out.view(-1), idx_ptr=plan.ptr, dst=plan.dst)
    torch.cuda.current_stream(dev).synchronize()
    report = {
        "schema": REPORT_SCHEMA,
        "image": {"height": img.shape[0], "width": img.shape[1]},
        "settings": {"dict": dict_spec, "iterations": config.iterations, "gamma": config.gamma,
                     "rho": config.rho_hat, "block": [block, block], "support": support,
                     "pipeline": "frame-engine" if grid is not None else "per-block-masks"},
        "lost_pixels": int(lost.sum()),
        "blocks": int(n_blocks),
        "seconds": time.perf_counter() - t0,
    }
    if reference is not None and lost.any():
        report["psnr_db"] = psnr_over_region(np.asarray(reference, dtype=np.float64),
                                             out.cpu().numpy(), lost)
    report["result"] = res
    return out, report


# ----------------------------------------------------------------- reference semantics

DEFAULT_SUPPORT = 24               # conceal.py:37
REFERENCE_REPORT_SCHEMA = "fase-conceal-report/1"


def _block_json(row, col, height, width, area, lost, seconds, psnr, max_imag, sel, coef):
    """One entry of the report's ``blocks`` list (BlockResult.to_json, conceal.py:55-70)."""
    return {
        "row": int(row), "col": int(col), "height": int(height), "width": int(width),
        "area": [int(x) for x in area], "lost": int(lost), "seconds": float(seconds),
        "psnr_db": psnr, "max_imag": float(max_imag),
        "trace": [{"atom": int(k), "coefficient": [float(c.real), float(c.imag)]}
                  for k, c in zip(sel, coef)],
    }


def conceal_image(image, lost_mask, *, dict_spec: str = "dft",
                  config: ExtrapConfig = ExtrapConfig(), block: tuple[int, int] | None = None,
                  support: int = DEFAULT_SUPPORT, tables=None, use_fft: bool = False,
                  single_thread: bool = False, reference=None, device=None):
    """Fill the lost samples of an image and report what happened -- the
    reference's ``conceal_image`` (``conceal.py:167-270``) on the GPU.

    Same tiling, same clipped extrapolation areas (tile +- ``support``, cut at
    the image border), same per-area dictionaries and weights, same paste of
    each tile's own lost pixels, same report (schema ``fase-conceal-report/1``).
    Instead of one job per tile, all tiles whose areas share a shape run as one
    batch: identical geometries share a table, differing ones use chunked
    per-block tables (``fase_extrapolate_batch``). ``tables`` serves every
    group whose provenance matches (counted once, as ``tables_reused``);
    ``use_fft`` builds shared tables through the transform shortcut where
    every atom is frequency-tagged (initial products of exponential atoms are
    always computed as separable transforms). ``single_thread`` is accepted for
    signature compatibility (blocks are independent; results do not depend on
    it). A block's ``seconds`` is its share of its batch's wall time.

    Returns:
        (restored float64 image (host), JSON-ready report dict).
    """
    import torch

    from .fast import GramTable, build_gram_tables
    from .grid import build_weight_field
    from .transform import fft_gram_table

    img = np.asarray(image, dtype=np.float64)
    if img.ndim != 2 or img.size == 0:
        raise ShapeError(f"image must be non-empty 2-D, got shape {img.shape}")
    lost = as_mask(lost_mask)
    if lost.shape != img.shape:
        raise ShapeError(f"image {img.shape} vs mask {lost.shape}")
    ref = None
    if reference is not None:
        ref = np.asarray(reference, dtype=np.float64)
        if ref.shape != img.shape:
            raise ShapeError(f"image {img.shape} vs reference {ref.shape}")
    if support < 0:
        raise ParameterError(f"support margin must be >= 0, got {support}")
    h_img, w_img = img.shape
    if block is None:
        tiles = [(0, 0, h_img, w_img)]
        grid = None
    else:
        bh, bw = block
        if bh < 1 or bw < 1:
            raise ParameterError(f"block must be at least 1x1, got {bh}x{bw}")
        tiles = [(r0, c0, min(bh, h_img - r0), min(bw, w_img - c0))
                 for r0 in range(0, h_img, bh) for c0 in range(0, w_img, bw)]
        grid = [bh, bw]
    jobs = [t for t in tiles if lost[t[0]:t[0] + t[2], t[1]:t[1] + t[3]].any()]

    started = time.perf_counter()
    out = img.copy()
    entries = [None] * len(jobs)
    reused = 0
    if jobs:
        dev = resolve_device(device)
        # clipped areas (conceal.py:119-124), grouped by shape
        areas = []
        for r0, c0, bh_, bw_ in jobs:
            a_r0, a_c0 = max(0, r0 - support), max(0, c0 - support)
            a_r1, a_c1 = min(h_img, r0 + bh_ + support), min(w_img, c0 + bw_ + support)
            areas.append((a_r0, a_c0, a_r1, a_c1))
        groups: dict = {}
        for j, (a_r0, a_c0, a_r1, a_c1) in enumerate(areas):
            groups.setdefault((a_r1 - a_r0, a_c1 - a_c0), []).append(j)
        for shape, members in groups.items():
            t_g = time.perf_counter()
            d = parse_dict_spec(dict_spec, *shape)
            sig = np.stack([img[a[0]:a[2], a[1]:a[3]] for a in (areas[j] for j in members)])
            msk = np.stack([lost[a[0]:a[2], a[1]:a[3]] for a in (areas[j] for j in members)])
            shared = bool((msk == msk[0]).all())
            tab = None
            if shared:
                w = build_weight_field(msk[0], config.rho_hat)
                if isinstance(tables, GramTable) and tables.matches(d, w):
                    tab = tables
                    reused = 1
                elif use_fft and len(d.tagged_indices()) == len(d):
                    tab = fft_gram_table(w, d, device=dev)
                else:
                    tab = build_gram_tables(d, w, device=dev)
                masks_arg = msk[0]
            else:
                masks_arg = msk
            res = fase_extrapolate_batch(sig, masks_arg, d, tab, config, device=dev)
            patched = res.patched.cpu().numpy()
            sel = res.selected.cpu().numpy()
            coef = res.coefficients.cpu().numpy().astype(np.complex128)
            mi = (res.max_imag.cpu().numpy() if res.max_imag is not None
                  else np.zeros(len(members)))
            each = (time.perf_counter() - t_g) / len(members)
            for i, j in enumerate(members):
                r0, c0, bh_, bw_ = jobs[j]
                a_r0, a_c0, a_r1, a_c1 = areas[j]
                tile_lost = lost[r0:r0 + bh_, c0:c0 + bw_]
                rel = patched[i][r0 - a_r0:r0 - a_r0 + bh_, c0 - a_c0:c0 - a_c0 + bw_]
                out[r0:r0 + bh_, c0:c0 + bw_][tile_lost] = rel[tile_lost]
                psnr = None
                if ref is not None:
                    psnr = psnr_over_region(ref[r0:r0 + bh_, c0:c0 + bw_],
                                            out[r0:r0 + bh_, c0:c0 + bw_], tile_lost)
                entries[j] = _block_json(r0, c0, bh_, bw_, (a_r0, a_c0, a_r1 - a_r0, a_c1 - a_c0),
                                         tile_lost.sum(), each, psnr, mi[i], sel[i], coef[i])
        torch.cuda.current_stream(dev).synchronize()
    total_seconds = time.perf_counter() - started
    overall_psnr = None
    if ref is not None and lost.any():
        overall_psnr = psnr_over_region(ref, out, lost)
    report = {
        "schema": REFERENCE_REPORT_SCHEMA,
        "image": {"height": h_img, "width": w_img},
        "settings": {"dict": dict_spec, "iterations": config.iterations, "gamma": config.gamma,
                     "rho": config.rho_hat, "block": grid, "support": support, "fft": use_fft},
        "lost_pixels": int(lost.sum()),
        "blocks": entries,
        "tables_reused": reused,
        "psnr_db": overall_psnr,
        "max_imag": max((e["max_imag"] for e in entries), default=0.0),
        "seconds": total_seconds,
    }
    return out, report
