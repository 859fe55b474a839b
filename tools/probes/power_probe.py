"""Clocks and power per phase of the config-4 step (measurement probe).

Runs each phase back to back for ~3 s with nvidia-smi sampling clocks, power
and throttle reasons: the scaled recursion alone, the Ozaki products alone,
the synthesis alone, and whole steps. Prints one JSON line per phase (ms per
launch from CUDA events, median SM clock, median power, reasons seen).

    python tools/probes/power_probe.py [--config 4] [--seconds 3]
"""
import argparse
import json
import os
import subprocess
import sys
import time

sys.path.insert(0, os.getcwd())
import numpy as np
import torch

from paper_2204_14194_b200 import ShardedBatch, _native, build_gram_tables, build_weight_field
from paper_2204_14194_b200 import workloads as wl

REASONS = {0x1: "gpu_idle", 0x2: "app_clocks", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
           0x20: "sw_thermal", 0x40: "hw_thermal", 0x80: "hw_power_brake"}


def sample(fn, seconds, label):
    path = f"gpurun_out/power_{label}.csv"
    os.makedirs("gpurun_out", exist_ok=True)
    fh = open(path, "w")
    proc = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,power.draw,"
                             "clocks_event_reasons.active,temperature.gpu",
                             "--format=csv,noheader,nounits", "-lms", "20"], stdout=fh)
    time.sleep(0.3)
    skip = len(open(path).read().splitlines())
    ev = []
    t0 = time.time()
    n = 0
    while time.time() - t0 < seconds:
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        ev.append((a, b))
        n += 1
        if n % 8 == 0:
            torch.cuda.synchronize()
    torch.cuda.synchronize()
    end = len(open(path).read().splitlines())
    proc.terminate()
    proc.wait()
    fh.close()
    ms = [a.elapsed_time(b) for a, b in ev]
    sm, pw, rs = [], [], set()
    for line in open(path).read().splitlines()[skip:end]:
        p = [x.strip() for x in line.split(",")]
        try:
            sm.append(float(p[0]))
            pw.append(float(p[1]))
            m = int(p[2], 16)
        except (ValueError, IndexError):
            continue
        rs |= {v for k, v in REASONS.items() if m & k}
    half = len(ms) // 2  # steady state: the second half
    return {"phase": label, "launches": len(ms), "ms_median": float(np.median(ms[half:])),
            "ms_first": float(np.median(ms[:max(1, half // 4)])),
            "sm_mhz_median": float(np.median(sm)) if sm else None,
            "sm_mhz_min": float(np.min(sm)) if sm else None,
            "power_w_median": float(np.median(pw)) if pw else None,
            "reasons": sorted(rs), "samples": len(sm)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--seconds", type=float, default=3.0)
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    _native.load()
    w = wl.WORKLOADS[args.config]
    d = w.dictionary()
    K, I = len(d), w.config.iterations
    mask = wl.central_loss_mask(*w.area, *w.loss)
    tables = build_gram_tables(d, build_weight_field(mask, w.config.rho_hat), device=dev)
    sb = ShardedBatch(d, mask, w.n_blocks, w.config, tables, dev, recursion="scaled")
    plan = sb.plan
    sig = torch.from_numpy(wl.block_signals(args.config, w.n_blocks, *w.area)).to(dev)
    sig = sig.reshape(w.n_blocks, -1)
    plan.run(sig)
    torch.cuda.synchronize()

    def rec():
        _native.iterate_scaled(plan.Gs, plan.D, plan.R0, K, I, w.config.gamma, plan.selected,
                               plan.projections, plan.coefficients)

    def prod():
        plan._products(sig)

    def step():
        plan.run(sig)

    time.sleep(2.0)
    for label, fn in (("recursion", rec), ("products", prod), ("step", step), ("recursion2", rec)):
        print(json.dumps(sample(fn, args.seconds, label)), flush=True)
        time.sleep(2.0)


if __name__ == "__main__":
    main()
