"""Config-1 step with the scaled recursion: one launch of 1,024 blocks vs a
full first wave (592 = 148 x 4 blocks) followed by the remainder, with the
first wave's synthesis on a side stream overlapping the remainder's recursion."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2204_14194_b200 import ExtrapolationPlan, _native, build_gram_tables, build_weight_field  # noqa: E402
from paper_2204_14194_b200 import workloads as wl  # noqa: E402

dev = torch.device("cuda:0")
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
w = wl.WORKLOADS[1]
d = w.dictionary()
mask = wl.central_loss_mask(48, 48, 16, 16)
t = build_gram_tables(d, build_weight_field(mask, 0.8), device=dev)
B, K, I, g = w.n_blocks, len(d), w.config.iterations, w.config.gamma
p = ExtrapolationPlan(d, mask, B, w.config, t, device=dev, recursion="scaled")
sig = torch.from_numpy(wl.block_signals(1, B, 48, 48)).to(dev)
side = torch.cuda.Stream(dev)


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


def synth(lo, hi):
    _native.synth_paste(p.phi_lost, p.selected[lo:hi], p.coefficients[lo:hi], I, p.lost_seq,
                        p.lost[lo:hi], n_shared=p.n_lost, dst=p.lost_pos)


def iterate(lo, hi):
    _native.iterate_scaled(p.Gs, p.D, p.R0[lo:hi], K, I, g, p.selected[lo:hi],
                           p.projections[lo:hi], p.coefficients[lo:hi])


def plain():
    p.run(sig)


def split(A):
    def fn():
        cs = torch.cuda.current_stream()
        p.F[:, :p.M].copy_(sig.reshape(B, -1), non_blocking=True)
        p._products(p.F)
        iterate(0, A)
        ev = torch.cuda.Event()
        ev.record(cs)
        side.wait_event(ev)
        with torch.cuda.stream(side):
            synth(0, A)
        iterate(A, B)
        synth(A, B)
        ev2 = torch.cuda.Event()
        ev2.record(side)
        cs.wait_event(ev2)
    return fn


ref = None
tp = timed(plain)
ref = (p.selected.clone(), p.lost.clone())
print(f"one launch: {tp:.4f} ms")
for A in (592, 444, 296):
    ts = timed(split(A))
    ok = torch.equal(ref[0], p.selected) and torch.equal(ref[1], p.lost)
    print(f"split at {A}: {ts:.4f} ms ({tp / ts:.3f}x) identical={ok}")
