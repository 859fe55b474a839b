"""Scaled recursion with the synthesis fused in vs recursion + fase_synth_paste."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2204_14194_b200 import ExtrapolationPlan, _native, build_gram_tables, build_weight_field  # noqa: E402
from paper_2204_14194_b200 import workloads as wl  # noqa: E402

dev = torch.device("cuda:0")
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def timed(fn, n=8):
    out = []
    for _ in range(2):
        fn()
    for _ in range(n):
        _native.l2_flush(flush)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1))
    return float(np.median(out))


for cid in [int(c) for c in (sys.argv[1:] or ["1", "4", "0"])]:
    w = wl.WORKLOADS[cid]
    d = w.dictionary()
    mask = wl.central_loss_mask(*w.area, *w.loss)
    t = build_gram_tables(d, build_weight_field(mask, w.config.rho_hat), device=dev)
    B, K, I, g = w.n_blocks, len(d), w.config.iterations, w.config.gamma
    p = ExtrapolationPlan(d, mask, B, w.config, t, device=dev, recursion="scaled")
    sig = torch.from_numpy(wl.block_signals(cid, B, *w.area)).to(dev)
    p.run(sig)
    torch.cuda.synchronize()
    Gs = p.Gs
    lost2 = torch.zeros_like(p.lost)
    sel2, proj2, coef2 = (torch.empty_like(x) for x in (p.selected, p.projections, p.coefficients))

    def split():
        _native.iterate_scaled(Gs, p.D, p.R0, K, I, g, p.selected, p.projections, p.coefficients)
        _native.synth_paste(p.phi_lost, p.selected, p.coefficients, I, p.lost_seq, p.lost,
                            n_shared=p.n_lost, dst=p.lost_pos)

    def fused():
        _native.iterate_scaled(Gs, p.D, p.R0, K, I, g, sel2, proj2, coef2, phi_lost=p.phi_lost,
                               n_lost=p.n_lost, lost=lost2)

    ts, tf = timed(split), timed(fused)
    print(f"c{cid}: capacity {_native.scaled_synth_capacity(K, B)} (n_lost {p.n_lost}); "
          f"recursion + synth {ts:.4f} ms, fused {tf:.4f} ms ({ts / tf:.3f}x); "
          f"selections equal {torch.equal(sel2, p.selected)}, lost bit-identical "
          f"{torch.equal(lost2[:, :p.n_lost], p.lost[:, :p.n_lost])}")
