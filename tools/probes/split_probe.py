"""Config-1 step: one 1,024-block plan vs two half plans on two streams, and the
recursion alone at several batch sizes (wave quantization of the step)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2204_14194_b200 import ExtrapolationPlan, _native, build_gram_tables, build_weight_field  # noqa: E402
from paper_2204_14194_b200 import workloads as wl  # noqa: E402

dev = torch.device("cuda:0")
w = wl.WORKLOADS[1]
d = w.dictionary()
mask = wl.central_loss_mask(48, 48, 16, 16)
t = build_gram_tables(d, build_weight_field(mask, 0.8), device=dev)
K, I = len(d), w.config.iterations
sig = torch.from_numpy(wl.block_signals(1, 1024, 48, 48)).to(dev)
full = ExtrapolationPlan(d, mask, 1024, w.config, t, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def timed(fn, n=10):
    out = []
    for _ in range(3):
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


print(f"full plan.run: {timed(lambda: full.run(sig)):.4f} ms")
for nb in (1024, 888, 592, 444, 296, 148, 136):
    def it(nb=nb):
        _native.iterate(full.G, full.D, full.R0[:nb], K, I, 0.5, full.selected[:nb],
                        full.projections[:nb], full.coefficients[:nb])
    print(f"iterate B={nb}: {timed(it):.4f} ms")

for split in (512, 592, 444):
    a = ExtrapolationPlan(d, mask, split, w.config, t, device=dev)
    b = ExtrapolationPlan(d, mask, 1024 - split, w.config, t, device=dev)
    sa, sb = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def two():
        cs = torch.cuda.current_stream()
        ev = torch.cuda.Event()
        ev.record(cs)
        sa.wait_event(ev)
        sb.wait_event(ev)
        with torch.cuda.stream(sa):
            a.run(sig[:split])
        with torch.cuda.stream(sb):
            b.run(sig[split:])
        for s in (sa, sb):
            e = torch.cuda.Event()
            e.record(s)
            cs.wait_event(e)

    ms = timed(two)
    ok = torch.equal(torch.cat([a.selected, b.selected]), full.selected) and \
        torch.equal(torch.cat([a.lost, b.lost]), full.lost)
    print(f"two plans {split}+{1024 - split} on two streams: {ms:.4f} ms  identical={ok}")
