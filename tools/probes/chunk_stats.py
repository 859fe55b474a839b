"""Chunked-path counters of one frame run (needs a library built with
-DFASE_ITERATE_STATS, passed through FASE_B200_LIB)."""
import ctypes
import sys

import numpy as np
import torch

from paper_2204_14194_b200 import _native
from paper_2204_14194_b200 import workloads as wl
from paper_2204_14194_b200.conceal import FrameEngine, lossy_tiles, tile_grid

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 3
w = wl.WORKLOADS[cid]
case = wl.frame_case(w)
eng = FrameEngine(w.dictionary(), case.frame.shape, case.mb, case.support, w.config, device="cuda:0")
grid = torch.from_numpy(tile_grid(case.lost, case.mb)).cuda()
corners = torch.from_numpy(lossy_tiles(case.lost, (case.mb, case.mb)).astype(np.int32)).cuda()
dmg = torch.from_numpy(case.damaged()).cuda()
lib = _native.load()
out = (ctypes.c_ulonglong * 8)()
eng.run(dmg, grid, corners)
lib.fase_iterate_stats(out)  # reset
eng.run(dmg, grid, corners)
torch.cuda.synchronize()
lib.fase_iterate_stats(out)
n = out[0]
print(f"config {cid}: block-iterations {n}, copies issued {out[1] / n:.3f}, held hits {out[2] / n:.3f}, "
      f"mispredicted copies {out[3] / n:.3f}, held misses w/o copy {out[5] / n:.3f}, "
      f"remaining chunks per iteration {out[4] / n:.3f}, on predicted copies {out[6] / max(1, out[1] - out[3]):.3f}")
