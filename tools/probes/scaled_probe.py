"""Exact vs scaled recursion (fase_iterate vs fase_iterate_scaled) on the
shared-geometry configs: time per launch (L2 flushed), selections identical,
max coefficient deviation; alternative scaled shapes via FASE_SCALED_VARIANT."""
import os
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
    plan = ExtrapolationPlan(d, mask, B, w.config, t, device=dev)
    sig = torch.from_numpy(wl.block_signals(cid, B, *w.area)).to(dev)
    plan.run(sig)
    torch.cuda.synchronize()
    Gs = torch.empty_like(plan.G)
    _native.scale_columns(plan.G, plan.D, K, Gs)
    sel2, proj2, coef2 = (torch.empty_like(x) for x in (plan.selected, plan.projections,
                                                        plan.coefficients))

    def exact():
        _native.iterate(plan.G, plan.D, plan.R0, K, I, g, plan.selected, plan.projections,
                        plan.coefficients)

    def scaled():
        _native.iterate_scaled(Gs, plan.D, plan.R0, K, I, g, sel2, proj2, coef2)

    te = timed(exact)
    for var in [None] + (["256x18x3", "128x36x4", "256x20x4"] if cid == 1 else
                         ["128x64x2", "128x64x3"] if cid == 4 else []):
        if var:
            os.environ["FASE_SCALED_VARIANT"] = var
        else:
            os.environ.pop("FASE_SCALED_VARIANT", None)
        ts = timed(scaled)
        same = (sel2 == plan.selected).all(dim=1)
        nsame = int(same.sum())
        cdev = ((coef2 - plan.coefficients).abs().amax(dim=1) /
                plan.coefficients.abs().amax(dim=1))[same].max().item() if nsame else float("nan")
        first = [int(torch.nonzero(sel2[b] != plan.selected[b])[0]) for b in
                 torch.nonzero(~same).flatten().tolist()[:8]]
        print(f"c{cid} K={K} B={B}: exact {te:.4f} ms, scaled[{var or 'default'}] {ts:.4f} ms "
              f"({te / ts:.3f}x); identical blocks {nsame}/{B}, first divergences {first}, "
              f"max coef rel dev (identical blocks) {cdev:.2e}")
    os.environ.pop("FASE_SCALED_VARIANT", None)
