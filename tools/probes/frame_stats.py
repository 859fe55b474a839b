"""Selection statistics of a frame config on the GPU: immediate re-selection
rate and remaining chunk-list lengths after the precomposed bases."""
import sys

import numpy as np
import torch

from paper_2204_14194_b200 import workloads as wl
from paper_2204_14194_b200.conceal import FrameEngine, lossy_tiles, tile_grid

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 3
w = wl.WORKLOADS[cid]
case = wl.frame_case(w)
eng = FrameEngine(w.dictionary(), case.frame.shape, case.mb, case.support, w.config, device="cuda:0")
grid = torch.from_numpy(tile_grid(case.lost, case.mb)).cuda()
corners = torch.from_numpy(lossy_tiles(case.lost, (case.mb, case.mb)).astype(np.int32)).cuda()
res = eng.run(torch.from_numpy(case.damaged()).cuda(), grid, corners)
torch.cuda.synchronize()
sel = res.selected.cpu().numpy()
rep = (sel[:, 1:] == sel[:, :-1]).mean()
counts = eng._buffers(int(corners.shape[0]))["counts"].cpu().numpy()
depth = eng.compose.dim() if eng.compose is not None else 0
rem = counts - np.minimum(counts, depth)
print(f"config {cid}: blocks {sel.shape[0]}, immediate re-selection {rep:.3f}, "
      f"unique atoms per block {np.mean([len(set(r)) for r in sel]) / sel.shape[1]:.3f}")
print("list lengths", np.bincount(counts).tolist(), "remaining after compose", np.bincount(rem).tolist())
