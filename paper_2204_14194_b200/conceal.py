"""Frame concealment over many loss blocks at once (BASELINE configs 2 and 3).

The reference conceals an image tile by tile (``pkg/src/fase/conceal.py:111-245``):
area = tile +- support, weight from every lost pixel inside the area, FaSE,
then only the tile's own lost pixels are pasted back (``conceal.py:144-148``).
Here all lossy tiles of a frame form ONE batch: fixed-size areas (out-of-frame
samples are masked as unavailable, BASELINE config 2: "lost and unavailable
samples set to zero"), chunked per-block tables, one recursion launch, and one
synthesis kernel that pastes straight into the device frame. Interior tiles
give exactly the reference's per-tile result; border tiles differ from the
reference's *clipped* areas by design.
"""

from __future__ import annotations

import time

import numpy as np

from . import _native
from .dictionary import Dictionary, parse_dict_spec
from .errors import ParameterError, ShapeError
from .fast import ChunkedTables, fase_extrapolate_batch, resolve_device
from .grid import ExtrapConfig, as_mask, psnr_over_region
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


class FramePlan:
    """Device-side geometry of one damaged frame: areas, masks, paste targets."""

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
        # paste targets: each tile's own lost pixels (area index -> frame index)
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
                  block: int = 16, support: int = 16, reference=None, tables=None,
                  plan: FramePlan | None = None, device=None):
    """Conceal every lossy ``block`` x ``block`` tile of a frame on the GPU.

    Returns (restored float64 frame as a device tensor, report dict). Pass a
    prebuilt ``plan`` / ``tables`` to reuse geometry across frames with the
    same loss pattern.
    """
    import torch

    dev = resolve_device(device)
    t0 = time.perf_counter()
    if plan is None:
        plan = FramePlan(image, lost_mask, block, support, dev)
    a = plan.block + 2 * plan.support
    if dictionary is None:
        dictionary = parse_dict_spec(dict_spec, a, a)
    if dictionary.shape != (a, a):
        raise ShapeError(f"dictionary area {dictionary.shape} vs extrapolation area {(a, a)}")
    out = plan.frame.clone()
    if plan.n_blocks:
        if tables is None:
            tables = ChunkedTables(dictionary, plan.masks, config.rho_hat, dev)
        res = fase_extrapolate_batch(plan.signals, plan.masks, dictionary, tables, config,
                                     patch=False, device=dev)
        phi = dictionary.device_matrix(dev)
        _native.synth_paste(phi, res.selected, res.coefficients, config.iterations, plan.idx,
                            out.view(-1), idx_ptr=plan.ptr, dst=plan.dst)
    else:
        res = None
    torch.cuda.current_stream(dev).synchronize()
    report = {
        "schema": REPORT_SCHEMA,
        "image": {"height": plan.shape[0], "width": plan.shape[1]},
        "settings": {"dict": dict_spec if dictionary is None else dictionary.families[0],
                     "iterations": config.iterations, "gamma": config.gamma,
                     "rho": config.rho_hat, "block": [plan.block, plan.block],
                     "support": plan.support},
        "lost_pixels": int(plan.lost.sum()),
        "blocks": int(plan.n_blocks),
        "seconds": time.perf_counter() - t0,
    }
    if reference is not None and plan.lost.any():
        report["psnr_db"] = psnr_over_region(np.asarray(reference, dtype=np.float64),
                                             out.cpu().numpy(), plan.lost)
    report["result"] = res
    return out, report
