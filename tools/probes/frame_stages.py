"""Per-stage device time of one FrameEngine frame (configs 2 / 3): every
library call inside engine.run is bracketed with CUDA events."""
import sys
from collections import defaultdict

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2204_14194_b200 import _native, workloads as wl  # noqa: E402
from paper_2204_14194_b200.conceal import FrameEngine, lossy_tiles, tile_grid  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 3
dev = torch.device("cuda:0")
w = wl.WORKLOADS[cid]
d = w.dictionary()
case = wl.frame_case(w)
engine = FrameEngine(d, case.frame.shape, case.mb, case.support, w.config, device=dev)
grid = torch.from_numpy(tile_grid(case.lost, case.mb)).to(dev)
corners = torch.from_numpy(lossy_tiles(case.lost, (case.mb, case.mb)).astype(np.int32)).to(dev)
damaged = torch.from_numpy(case.damaged()).to(dev)
out = damaged.clone()
for _ in range(3):
    engine.run(damaged, grid, corners, out=out)
torch.cuda.synchronize()

events = []


def wrap(obj, name):
    fn = getattr(obj, name)

    def inner(*a, **k):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = fn(*a, **k)
        e1.record()
        events.append((name, e0, e1))
        return r
    setattr(obj, name, inner)


for n in ("frame_areas", "frame_cells", "block_normalizers", "sep_products_batch", "sep_products",
          "ozaki_gemm", "gemm_nt", "iterate", "frame_paste"):
    wrap(_native, n)
wrap(_native.OzakiOperand, "split")
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
tot = defaultdict(float)
n = 5
for _ in range(n):
    _native.l2_flush(flush)
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record()
    engine.run(damaged, grid, corners, out=out)
    f1.record()
    torch.cuda.synchronize()
    tot["frame"] += f0.elapsed_time(f1)
for name, e0, e1 in events:
    tot[name] += e0.elapsed_time(e1)
print(f"config {cid}, {int(corners.shape[0])} blocks: " +
      ", ".join(f"{k} {v / n:.3f} ms" for k, v in tot.items()))
