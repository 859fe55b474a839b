"""Mispredicted row copies of the shared-geometry recursion (library built
with -DFASE_ITERATE_STATS, passed through FASE_B200_LIB)."""
import ctypes
import sys

import torch

from paper_2204_14194_b200 import ExtrapolationPlan, _native, build_gram_tables, build_weight_field
from paper_2204_14194_b200 import workloads as wl

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 1
w = wl.WORKLOADS[cid]
d = w.dictionary()
mask = wl.central_loss_mask(*w.area, *w.loss)
dev = torch.device("cuda", 0)
tables = build_gram_tables(d, build_weight_field(mask, w.config.rho_hat), device=dev)
plan = ExtrapolationPlan(d, mask, w.n_blocks, w.config, tables, device=dev)
sig = torch.from_numpy(wl.block_signals(cid, w.n_blocks, *w.area)).to(dev)
lib = _native.load()
out = (ctypes.c_ulonglong * 8)()
plan.run(sig)
lib.fase_iterate_stats(out)
plan.run(sig)
lib.fase_iterate_stats(out)
print(f"config {cid}: block-iterations {out[0]}, mispredicted copies {out[3] / max(1, out[0]):.4f}")
