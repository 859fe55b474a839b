"""Per-phase cycle stamps of the recursion kernel (experiment build FASE_EXP=5)."""
import os, sys
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2204_14194_b200 import ExtrapolationPlan, _native, workloads as wl, build_gram_tables, build_weight_field
w = wl.WORKLOADS[1]
d = w.dictionary()
mask = wl.central_loss_mask(48, 48, 16, 16)
dev = torch.device("cuda:0")
t = build_gram_tables(d, build_weight_field(mask, 0.8), device=dev)
plan = ExtrapolationPlan(d, mask, 1024, w.config, t, device=dev)
sig = torch.from_numpy(wl.block_signals(1, 1024, 48, 48)).to(dev)
plan.run(sig)
torch.cuda.synchronize()
B, I, K = 1024, 200, len(d)
stamps = torch.zeros(B * I * 8, dtype=torch.int64, device=dev)
R_out = stamps.view(torch.float64)
for rep in range(2):
    _native.iterate(plan.G, plan.D, plan.R0, K, I, 0.5, plan.selected, plan.projections,
                    plan.coefficients, R_out=R_out.view(B, -1) if False else None)
torch.cuda.synchronize()
# direct call with R_out (ldr must be >= K: use a (B, I*8) view as doubles)
R_out2 = stamps.view(torch.float64).view(B, I * 8)
import ctypes
args = _native.IterateArgs(G0=plan.G.data_ptr(), ldg=plan.G.stride(0), D=plan.D.data_ptr(), ldd=0,
                           R0=plan.R0.data_ptr(), ldr=plan.R0.stride(0), R_out=R_out2.data_ptr(),
                           K=K, B=B, I=I, gamma=0.5, sel=plan.selected.data_ptr(),
                           proj=plan.projections.data_ptr(), coef=plan.coefficients.data_ptr(),
                           ldo=plan.selected.stride(0))
lib = _native.load()
s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
s.record()
st = lib.fase_iterate(ctypes.byref(args), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
e.record(); torch.cuda.synchronize()
print("status", st, "ms", s.elapsed_time(e))
ts = stamps.view(B, I, 8).cpu().numpy().astype(np.float64)
names = ["A->sync1", "sync1->pre_sync2", "pre_sync2->post_sync2", "post_sync2->tma_ready", "tma_ready->update_done", "update_done->next"]
for blk in (0, 300, 700, 1000):
    x = ts[blk]
    seg = np.stack([x[:, 1] - x[:, 0], x[:, 2] - x[:, 1], x[:, 3] - x[:, 2], x[:, 4] - x[:, 3], x[:, 5] - x[:, 4]], axis=1)
    nxt = x[1:, 0] - x[:-1, 5]
    med = np.median(seg[5:], axis=0)
    print(blk, "per-iteration cycles (median):", dict(zip(names, [int(v) for v in med])), "next:", int(np.median(nxt[5:])), "total", int(np.median(x[6:, 0] - x[5:-1, 0])))
