#!/usr/bin/env python
"""FaSE throughput on B200: extrapolated blocks/s (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl b200|reference]

A *step* is one pass of the hot path over one batch: BASELINE config 4 by
default (the largest single-GPU config, the one the "blocks/s at 1/2/4/8 B200"
metric is quoted on) -- 4,096 independent 64x64 areas with a centred 24x24
loss, 8,192 unit-norm Gaussian atoms, 500 iterations, rho 0.85, FP64. Per
step: batched initial products (tcgen05 Ozaki digit planes over the support),
the FaSE recursion, synthesis of the lost samples, and the result gather. The
shared Gram table is built once before the clock, exactly as the reference's
own benchmark does (pkg/src/fase/bench.py:6-9,118-119); its build time is
reported as ``gram_ms``. ``--config 0..3`` selects the other BASELINE configs.

``value``: device-resident throughput (signals already in HBM), CUDA events
per step on the launching stream, L2 flushed (256 MiB write) between steps.
``e2e``: the same batch through ShardedBatch.run_host_stream -- pinned host
signals -> device, kernels, gather, selections / coefficients / lost samples
-> pinned host -- all inside the timed region. After the clock the timed
outputs are classified against the reference-written batch fixture
(``parity_vs_reference``).

Multi-GPU (torchrun): one process per GPU; the ONE batch (or the frame's lossy
tiles) is sharded by contiguous block ranges (shard.block_range) and the
per-rank results are gathered to rank 0 with one NCCL gather per step, inside
the timed region (strong scaling); time = max over ranks.

--impl reference: the reference algorithm's CPU path (the oracle port of the
pure-Python reference, oracle/fase_oracle.py) on all host cores, one process
per core with one BLAS thread each; each step is a bounded sample of the same
workload.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

from paper_2204_14194_b200 import workloads as wl  # noqa: E402
from paper_2204_14194_b200.shard import dist_env  # noqa: E402

HBM_FALLBACK_GBS = 6650.0
FP64_FALLBACK_TFLOPS = 35.4
REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x40: "sw_thermal_slowdown",
           0x80: "hw_thermal_slowdown", 0x100: "hw_power_brake_slowdown",
           0x2: "applications_clocks_setting", 0x20: "sync_boost"}


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)  # ~0.17 s timed: several clock samples
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4, choices=[0, 1, 2, 3, 4])
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=12.0,
                    help="target wall seconds of the bounded CPU-baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--products", default="auto", choices=["auto", "gemm", "separable", "ozaki"],
                    help="initial products: separable transforms (separable dictionaries) or "
                         "the dense DMMA GEMM")
    ap.add_argument("--recursion", default="auto", choices=["auto", "exact", "scaled"],
                    help="shared-geometry recursion: exact (bit-identical to the reference loop) "
                         "or scaled (column-scaled table, no normalizers in the loop); auto = "
                         "scaled for real dictionaries")
    ap.add_argument("--compose", default=None, choices=["none", "singles", "pairs", "triples"],
                    help="frame configs: precomposed base tables (default: the engine's)")
    ap.add_argument("--l2-hint", default="off", choices=["on", "off"],
                    help="shared-geometry recursion: L2 residency hint for the most frequently "
                         "selected rows, tuned on a separate (never timed) batch (measured: "
                         "L2 hits 67 -> 74%%, DRAM reads -17%%, no speed-up; off by default)")
    ap.add_argument("--dict", default=None,
                    help="override the dictionary spec of a shared-geometry config (0, 1, 4), "
                         "e.g. 'dft' (the reference's default, complex-valued)")
    ap.add_argument("--blocks", type=int, default=None,
                    help="override the batch size of a shared-geometry config (the first B "
                         "blocks), e.g. one rank's shard of a multi-GPU run measured on one GPU")
    args = ap.parse_args()
    if args.dict and not wl.WORKLOADS[args.config].shared_geometry:
        ap.error("--dict applies to the shared-geometry configs 0, 1 and 4")
    if args.blocks is not None and (args.blocks < 1 or not wl.WORKLOADS[args.config].shared_geometry):
        ap.error("--blocks takes a positive batch size for the shared-geometry configs 0, 1 and 4")
    return args


def bench_dictionary(w, spec):
    """The workload's dictionary, or ``spec`` over the same area."""
    if not spec:
        return w.dictionary()
    from paper_2204_14194_b200 import parse_dict_spec

    return parse_dict_spec(spec, *w.area)


# ----------------------------------------------------------------- CPU reference


_CPU = {}


def _cpu_worker(args):
    """Extrapolate blocks [first, first+n) of the workload with the oracle port.

    Shared geometry (configs 0/1/4): tables prebuilt once, as the reference's
    bench does. Frame configs (2/3): per block weight -> Gram table -> FaSE ->
    paste, the reference's own frame path (conceal.py:132-141) minus its
    unbounded table cache.
    """
    cid, first, n = args
    from threadpoolctl import threadpool_limits

    from oracle import fase_oracle as orc

    w = wl.WORKLOADS[cid]
    vals, tables = _CPU["vals"], _CPU["tables"]
    nb = _CPU["n_blocks"]
    with threadpool_limits(limits=1):
        t0 = time.perf_counter()
        for i in range(n):
            b = (first + i) % nb
            if tables is not None:  # signals generated before the clock
                sig = _CPU["signals"][b % len(_CPU["signals"])]
                mask = _CPU["mask"]
            else:
                sig, mask = _CPU["signals"][b], _CPU["masks"][b]
            orc.extrapolate_block(sig, mask, vals, w.config.gamma, w.config.iterations,
                                  w.config.rho_hat, tables=tables)
        return n, time.perf_counter() - t0


def cpu_prepare(cid: int, spec=None):
    from oracle import fase_oracle as orc

    w = wl.WORKLOADS[cid]
    d = bench_dictionary(w, spec)
    vals = d.values
    if w.shared_geometry:
        mask = wl.central_loss_mask(*w.area, *w.loss)
        tables = orc.gram(vals.reshape(len(vals), -1), orc.weight_field(mask, w.config.rho_hat))
        # a pool of the workload's own blocks, generated outside the timed loop
        _CPU.update(vals=vals, mask=mask, tables=tables, n_blocks=w.n_blocks,
                    signals=wl.block_signals(cid, min(w.n_blocks, 256), *w.area))
    else:
        case = wl.frame_case(w)
        signals, masks = wl.frame_areas(case.damaged(), case.lost, case.corners, case.mb,
                                        case.support)
        # spread the sample over the frame: every 7th block
        order = np.arange(len(masks))[::7]
        _CPU.update(vals=vals, tables=None, signals=signals[order], masks=masks[order],
                    n_blocks=len(order))


def cpu_sample(cid: int, seconds: float, pool, procs: int, per_block_s: float):
    """One bounded sample: every worker extrapolates ~seconds worth of blocks."""
    n = max(1, int(seconds / max(per_block_s, 1e-4)))
    t0 = time.perf_counter()
    out = pool.map(_cpu_worker, [(cid, p * n, n) for p in range(procs)])
    wall = time.perf_counter() - t0
    blocks = sum(o[0] for o in out)
    return blocks / wall, blocks, wall


def cpu_baseline(cid: int, seconds: float, steps: int = 1, warmup: int = 0, spec=None):
    import multiprocessing as mp

    cpu_prepare(cid, spec)
    procs = os.cpu_count() or 1
    # calibrate one block on one core
    n1, t1 = _cpu_worker((cid, 0, 1))
    per_block = t1 / n1
    ctx = mp.get_context("fork")
    with ctx.Pool(procs) as pool:
        for _ in range(warmup):
            cpu_sample(cid, seconds, pool, procs, per_block)
        vals = [cpu_sample(cid, seconds, pool, procs, per_block) for _ in range(steps)]
    rate = float(np.median([v[0] for v in vals]))
    blocks, wall = vals[-1][1], vals[-1][2]
    return {"value": rate, "unit": "blocks/s", "cores": procs, "kind": "port",
            "ms_per_sample": float(np.median([v[2] for v in vals])) * 1e3,
            "sample": (f"{blocks} blocks of config {cid} per step ({procs} processes x 1 BLAS "
                       f"thread, ~{wall:.1f} s wall), oracle/fase_oracle.py port of the reference "
                       f"fase_extrapolate+apply_model with tables prebuilt; 1-core "
                       f"{1.0 / per_block:.1f} blocks/s")}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    w = wl.WORKLOADS[args.config]
    # bounded samples: the whole --steps/--warmup run stays within ~2.5 minutes
    seconds = max(1.0, min(args.cpu_seconds, 150.0 / max(1, args.steps + args.warmup)))
    base = cpu_baseline(args.config, seconds, steps=args.steps, warmup=args.warmup,
                        spec=args.dict)
    line = {
        "impl": "reference", "metric": "extrapolated blocks/s", "value": base["value"],
        "unit": "blocks/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        # one step = one bounded sample of the workload on the host cores
        "ms_per_step": base["ms_per_sample"], "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64" if bench_dictionary(w, args.dict).is_real else "c128",
        "data": "synthetic (seeded, BASELINE Appendix-A generators)",
        "config": workload_config(w, args.gpus, args.dict), "cpu_baseline": base,
        "e2e": {"value": base["value"], "unit": "blocks/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- GPU arm


def workload_config(w, n_gpus, spec=None):
    cfg = {"workload": w.name + (f" with dictionary {spec}" if spec else ""), "area": list(w.area),
           "K": len(bench_dictionary(w, spec)) if spec else w.n_atoms,
           "M": w.area[0] * w.area[1], "iterations": w.config.iterations, "gamma": w.config.gamma,
           "rho": w.config.rho_hat, "dictionary": spec or w.dict_spec,
           "l2": "flushed between timed steps (256 MiB write)",
           "parallelism": f"dp{n_gpus}: one batch sharded by block ranges, results gathered "
                          f"to rank 0 (NCCL gather, inside the timed region)"
                          if n_gpus > 1 else "dp1"}
    if w.shared_geometry:
        cfg.update(blocks=w.n_blocks, loss=f"{w.loss[0]}x{w.loss[1]} centred",
                   tables="shared Gram prebuilt before the clock (reference bench.py:118-119)")
    else:
        cfg.update(frame=list(w.frame), macroblock=w.macroblock, support=w.support,
                   loss=f"{w.loss_fraction:.0%} of full macroblocks",
                   tables="frame-independent cell tables prebuilt (G0 + one per area cell); "
                          "per-frame cell lists, normalizers, products, recursion, paste timed",
                   parallelism=f"dp{n_gpus}: the frame's lossy tiles sharded by ranges, results "
                               f"gathered to rank 0 which pastes them (NCCL gather, timed)"
                               if n_gpus > 1 else "dp1")
    return cfg


class ClockSampler:
    def __init__(self, gpu_id: str):
        self.gpu_id = gpu_id
        self.proc = None
        self.path = ROOT / "gpurun_out" / f"clocks_{os.getpid()}.csv"

    def __enter__(self):
        try:
            self.path.parent.mkdir(exist_ok=True)
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", self.gpu_id,
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,power.draw",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=self.fh, stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
            return self
        # the timed region starts only once the sampler is producing lines
        t0 = time.time()
        while time.time() - t0 < 5.0 and self.proc.poll() is None:
            if self.path.stat().st_size > 0:
                break
            time.sleep(0.02)
        self.skip = len(self.path.read_text().splitlines())  # idle samples before the region
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            # a region shorter than the 20 ms sampling period may hold no sample:
            # then wait (<= 0.2 s) for the first one after it, flagged as such
            self.region_lines = len(self.path.read_text().splitlines())
            t0 = time.time()
            while (self.region_lines <= getattr(self, "skip", 0) and time.time() - t0 < 0.2
                   and self.proc.poll() is None):
                time.sleep(0.005)
                if len(self.path.read_text().splitlines()) > self.region_lines:
                    break
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.fh.close()

    def summary(self):
        if self.proc is None or not self.path.exists():
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, smax, reasons = [], None, set()
        lines = self.path.read_text().splitlines()
        skip = getattr(self, "skip", 0)
        end = getattr(self, "region_lines", len(lines))
        in_region = end > skip
        for line in (lines[skip:end] if in_region else lines[skip:skip + 1]):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 3:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
                mask = int(parts[2], 16)
            except ValueError:
                continue
            for bit, name in REASONS.items():
                if mask & bit:
                    reasons.add(name)
        out = {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax,
               "reasons": sorted(reasons), "samples": len(sm)}
        if not in_region:
            out["note"] = "timed region shorter than the 20 ms sampling period: first sample after it"
        return out


def measured_peaks():
    hbm, src = HBM_FALLBACK_GBS, "fallback"
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            hbm, src = float(json.loads(p.read_text())["hbm_gbs"]), "measured"
        except (KeyError, ValueError):
            pass
    fp64, fsrc = FP64_FALLBACK_TFLOPS, "cuBLAS DGEMM 8192^3 measured r01"
    q = ROOT / "profiles" / "r01_fp64_peak.json"
    if q.exists():
        fp64 = float(json.loads(q.read_text())["dgemm_8192_tflops"])
    return hbm, src, fp64, fsrc


def measured_l2():
    """(GB/s, lts__throughput % at that rate, source): the L2 -> SM read
    bandwidth measured on this pool's B200 with tools/probes/l2_probe.cu, taken
    under ncu in round 2 (profiles/r02_l2_peak_ncu.json: the probe's best
    L2-resident stream registers ~54.4% lts__throughput, the reachable ceiling),
    else the round-1 plain run; None if neither exists."""
    q = ROOT / "profiles" / "r02_l2_peak_ncu.json"
    try:
        s = json.loads(q.read_text())["summary"]
        return (s["l2_read_peak_gbs"], s["at_lts_throughput_pct"],
                "tools/probes/l2_probe.cu under ncu (profiles/r02_l2_peak_ncu.json): lts__t_sectors_op_read "
                "bytes / time of the best L2-resident read stream")
    except (OSError, ValueError, KeyError):
        pass
    q = ROOT / "profiles" / "r01_l2_peak.json"
    try:
        res = json.loads(q.read_text())["results"]
        best = max(r["read_gbs"] for r in res if r["mb"] <= 96)
        return best, None, "tools/probes/l2_probe.cu: ld.global.cg 16-byte reads of L2-resident buffers"
    except (OSError, ValueError, KeyError):
        return None


def ncu_traffic(kernel: str, tag: str):
    """DRAM bytes per launch of ``kernel`` from the committed ncu capture of the
    same workload (profiles/ncu_summary.json, key "<tag>/<kernel>"), or None."""
    p = ROOT / "profiles" / "ncu_summary.json"
    if not p.exists():
        return None
    try:
        return json.loads(p.read_text()).get(f"{tag}/{kernel}", {}).get("dram_bytes_per_launch")
    except ValueError:
        return None


def ncu_profile(kernel: str, tag: str):
    """The committed ncu counters of ``kernel`` for workload ``tag`` beyond DRAM
    bytes (L2 throughput, issue activity, instructions per warp-iteration)."""
    p = ROOT / "profiles" / "ncu_summary.json"
    if not p.exists():
        return None
    try:
        rec = json.loads(p.read_text()).get(f"{tag}/{kernel}", {})
    except ValueError:
        return None
    keep = {k: v for k, v in rec.items() if k != "dram_bytes_per_launch"}
    return keep or None


def l2_roofline(achieved_gbs, prof=None, warps_per_block=None, blocks=None, iters=None):
    """The recursion's row stream against the measured L2 read bandwidth: with
    most rows L2 hits, L2 -> SM bandwidth, not HBM, bounds the kernel. ``prof``
    (the committed ncu counters of the same kernel) adds the ncu-side
    fractions: its lts__throughput over the probe's, and its L2 -> SM crossbar
    bytes (= the algorithmic row bytes) at ncu's own duration."""
    m = measured_l2()
    if m is None:
        return None
    peak, probe_lts, src = m
    out = {"bound": "l2", "achieved": achieved_gbs, "peak": peak, "unit": "GB/s",
           "frac": achieved_gbs / peak, "peak_source": src,
           "note": "same algorithmic bytes as roofline (one table row per block-iteration)"}
    if prof:
        if prof.get("lts_throughput_pct") and probe_lts:
            out["ncu_lts_throughput_pct"] = prof["lts_throughput_pct"]
            out["probe_lts_throughput_pct"] = probe_lts
            out["ncu_frac_of_probe"] = prof["lts_throughput_pct"] / probe_lts
        if prof.get("xbar_read_bytes_per_launch") and prof.get("duration_ms"):
            out["ncu_xbar_read_gbs"] = prof["xbar_read_bytes_per_launch"] / (prof["duration_ms"] * 1e-3) / 1e9
            out["ncu_xbar_frac"] = out["ncu_xbar_read_gbs"] / peak
        if prof.get("warp_instructions") and warps_per_block and blocks and iters:
            out["warp_instructions_per_warp_iteration"] = (
                prof["warp_instructions"] / (warps_per_block * blocks * iters))
    return out


def ozaki_roofline(plan, flops_fp64, seconds, fp64_peak, fp64_src):
    """Initial products on the tcgen05 INT8 tensor cores (Ozaki digit planes):
    the executed int8 MMA work against the INT8 dense peak (2x the measured
    BF16 dense peak in MEASURED_PEAKS.json), with the FP64-equivalent rate."""
    a, b = plan._ozaki
    s = a.slices
    pairs = s * (s + 1) // 2
    ops = 2.0 * pairs * a.rows * b.rows * a.kp
    # measured on this pool's B200 with an issue-only tcgen05.mma kind::i8 probe
    # (tools/probes/i8_peak_probe.cu, profiles/r02_int8_peak.json); fallback:
    # the nominal dense INT8 (= FP8) rate of B200_PROFILING.md
    i8_peak, src = 4500.0, "nominal B200 dense INT8 (= FP8) tensor rate, B200_PROFILING.md"
    q = ROOT / "profiles" / "r02_int8_peak.json"
    if q.exists():
        try:
            rec = json.loads(q.read_text())
            i8_peak = max(float(rec["tops_n128"]), float(rec["tops_n256"]))
            src = ("measured: issue-only tcgen05.mma kind::i8 M=128 N=128/256 on every SM "
                   "(tools/probes/i8_peak_probe.cu, profiles/r02_int8_peak.json)")
        except (KeyError, ValueError):
            pass
    return {"bound": "tensor", "kernel": "ozaki_gemm_kernel (tcgen05.mma kind::i8, "
            f"{s} digit planes, {pairs} pairs) over the support samples",
            "achieved": ops / seconds / 1e12, "peak": i8_peak, "unit": "TOPS (int8)",
            "frac": ops / seconds / 1e12 / i8_peak, "ms_per_launch": seconds * 1e3,
            "peak_source": src, "fp64_equivalent_tflops": flops_fp64 / seconds / 1e12,
            "fp64_peak_tflops": fp64_peak, "fp64_peak_source": fp64_src,
            "note": "ms includes the digit-split kernel (support gather and weights fused) "
                    "of the batch"}


def parity_vs_reference(cid, sel, coef, lost, n_lost, name=None):
    """Classify the timed outputs against the reference-written batch fixture
    (tests/golden/<name or c{cid}>_batch.npz, make_batch_golden.py) after the clock:
    identical sequences, legitimate near-tie stops (the GPU's atom is one the
    reference's tie rule could pick under a 1e-9 relative Delta-E change),
    failures; coefficient / lost-sample deviation on the run scale."""
    p = ROOT / "tests" / "golden" / f"{name or f'c{cid}'}_batch.npz"
    if not p.exists():
        return None
    z = np.load(p)
    blocks = z["blocks"]
    ties = {}
    for i, t, k in z["ties"]:
        ties.setdefault((int(i), int(t)), set()).add(int(k))
    out = {"fixture": p.name, "blocks_checked": int(len(blocks)), "identical": 0, "near_tie": 0,
           "failure": 0}
    worst_c = worst_l = 0.0
    has_coef = "coefficients" in z.files  # selections-only fixtures (c4all)
    # (NpzFile members decompress on every access: load each array once)
    z_sel = z["selected"]
    z_coef = z["coefficients"] if has_coef else None
    z_lost = z["lost"] if has_coef else None
    z_lost_n = z["lost_n"] if has_coef else None
    for i, b in enumerate(blocks):
        if int(b) >= len(sel):  # a smaller batch (--blocks): the fixture blocks it holds
            out["blocks_checked"] -= 1
            continue
        g = sel[int(b)].astype(np.int64)
        want = z_sel[i].astype(np.int64)
        diff = np.flatnonzero(g != want)
        stop = int(diff[0]) if diff.size else len(g)
        if diff.size == 0:
            out["identical"] += 1
        elif int(g[stop]) in ties.get((i, stop), ()):
            out["near_tie"] += 1
        else:
            out["failure"] += 1
            continue
        if not has_coef:
            continue
        sc = max(float(np.abs(z_coef[i]).max()), 1e-300)
        worst_c = max(worst_c, float(np.abs(coef[int(b)][:stop] - z_coef[i][:stop])
                                     .max(initial=0.0)) / sc)
        if diff.size == 0 and lost is not None:
            n = int(z_lost_n[i])
            want_l = z_lost[i][:n]
            worst_l = max(worst_l, float(np.abs(lost[int(b)][:n] - want_l).max(initial=0.0))
                          / max(float(np.abs(want_l).max()), 1e-300))
    out.update(max_coef_rel_dev=worst_c, max_lost_rel_dev=worst_l,
               rule="selection bit-exact except legitimate near-ties (1e-9 rel. Delta-E); "
                    "coefficients / samples within 1e-6 of the run scale")
    return out


def run_gpu(args):
    import torch
    import torch.distributed as dist

    from paper_2204_14194_b200 import ShardedBatch, _native, build_gram_tables, build_weight_field
    from paper_2204_14194_b200.shard import build_gram_tables_sharded
    from paper_2204_14194_b200.fast import gram_into, gram_support

    rank, world, local = dist_env()
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # before CUDA init (fork-safe)
        cpu = cpu_baseline(args.config, args.cpu_seconds, spec=args.dict)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    _native.load()

    w = wl.WORKLOADS[args.config]
    d = bench_dictionary(w, args.dict)
    cplx = not d.is_real
    K, M, I, B_total = len(d), w.area[0] * w.area[1], w.config.iterations, args.blocks or w.n_blocks
    mask = wl.central_loss_mask(*w.area, *w.loss)
    d.device_matrix(dev)
    # the shared table, outside the timed region (reference bench.py:118-119):
    # under torchrun every rank builds 1/N of its rows on the tensor cores and
    # the row panels are broadcast (bit-identical to one GPU's
    # table); one GPU builds it whole
    tables = build_gram_tables_sharded(d, build_weight_field(mask, w.config.rho_hat), device=dev)
    # auto: the scaled recursion (complex: union:dft+bdft 2.31 -> 1.84 ms; dft
    # 48^2 0.994 -> 0.830 ms at four CTAs per SM), except for batches of at most
    # one block per SM, where the bit-exact recursion with the synthesis fused
    # in is the faster one (config 0: 113.9 vs 118.1 us per step)
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    n_lost = int(mask.sum())
    latency_exact = (not cplx and B_total <= n_sm and world == 1
                     and 0 < n_lost <= _native.synth_capacity(K, B_total))
    recursion = args.recursion if args.recursion != "auto" else (
        "exact" if latency_exact else "scaled")
    if cplx and world > 1:
        raise SystemExit("complex dictionaries: single GPU only in the bench")
    # ONE batch of B_total blocks, rank r taking block_range(B_total, r, N)
    sb = ShardedBatch(d, mask, B_total, w.config, tables, dev, products=args.products,
                      recursion=recursion)
    plan = sb.plan
    B, lo = sb.hi - sb.lo, sb.lo
    if recursion == "scaled":
        scaled_fn = _native.iterate_complex_scaled if cplx else _native.iterate_scaled

        def iterate(G, D, R0, K, I, gamma, sel, proj, coef):
            scaled_fn(plan.Gs, D, R0, K, I, gamma, sel, proj, coef)
    else:
        iterate = _native.iterate_complex if cplx else _native.iterate
    synth_extra = {"max_imag": plan.max_imag} if cplx else {}
    synth = _native.synth_paste_complex if cplx else _native.synth_paste
    # one more table build, kernels only, for the reported Gram time
    G2 = torch.zeros_like(plan.G)
    D2 = torch.empty_like(plan.D)
    gws = torch.empty((int(_native.load().fase_gram_complex_workspace(K, plan.phi.shape[1]))
                       if cplx else K * plan.phi.shape[1] * 8) // 8 + 2,
                      dtype=torch.float64, device=dev)
    support = None if cplx else gram_support(plan.W, M)

    def build_table():
        if cplx:
            _native.gram_complex(plan.phi, plan.W, K, M, G2, ws=gws)
            _native.gram_finish_complex(G2, K, D2)
            return "dmma"
        path = gram_into(plan.phi, plan.W, K, M, G2, support)
        _native.gram_finish(G2, K, D2)
        return path

    # warm build first (operand buffers come from the caching allocator, as in
    # a process that builds tables repeatedly), then the timed one
    build_table()
    torch.cuda.synchronize()
    g0 = torch.cuda.Event(enable_timing=True)
    g1 = torch.cuda.Event(enable_timing=True)
    g0.record()
    gram_path = build_table()
    g1.record()
    torch.cuda.synchronize()
    gram_ms = g0.elapsed_time(g1)
    assert torch.equal(G2, plan.G) and torch.equal(D2, plan.D), "Gram build is not deterministic"
    del G2, D2, gws
    fft_gram_ms = None
    if cplx and len(d.tagged_indices()) == K:  # transform-shortcut table (fft_gram_table)
        from paper_2204_14194_b200 import fft_gram_table

        wfield = build_weight_field(mask, w.config.rho_hat)
        fft_gram_table(wfield, d, device=dev)  # warm (factor upload)
        g0.record()
        fft_gram_table(wfield, d, device=dev)
        g1.record()
        torch.cuda.synchronize()
        fft_gram_ms = g0.elapsed_time(g1)

    # this rank's shard of batch 0 (timed device-resident and e2e) and of a
    # second batch (blocks B_total + ...) the e2e stream alternates with
    host = torch.from_numpy(wl.block_signals(args.config, B, *w.area, first=lo)).pin_memory()
    host2 = torch.from_numpy(wl.block_signals(args.config, B, *w.area,
                                              first=B_total + lo)).pin_memory()
    dev_sig = host.to(dev)
    sig_view = dev_sig.reshape(B, -1)
    if plan.F.shape[1] != M:  # odd areas: the kernels read the padded layout
        plan.F[:, :M].copy_(sig_view)
        sig_view = plan.F
    harena = [sb.host_arena(), sb.host_arena()] if sb.is_root else [None, None]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    # L2 residency hint: the rows a separate batch (blocks 2*B_total + ..., never
    # timed) selects most often are copied evict_last, the others evict_first
    l2_hint = None
    if args.l2_hint == "on" and not cplx:
        tune = torch.from_numpy(wl.block_signals(args.config, B, *w.area,
                                                 first=2 * B_total + lo)).to(dev)
        plan.run(tune)
        torch.cuda.synchronize()
        n_hot = plan.tune_l2(plan.selected)
        G_ = plan.Gs if plan.Gs is not None else plan.G
        l2_hint = {"hot_rows": n_hot, "hot_bytes": n_hot * G_.shape[1] * 8,
                   "hot_share_of_tuning_selections": plan.l2_hot_share,
                   "tuned_on": f"blocks {2 * B_total + lo}..{2 * B_total + lo + B - 1} (never timed)",
                   "policy": "staged-row TMA copies: hot rows L2::evict_last, others L2::evict_first"}
        del tune
    for _ in range(max(args.warmup, 0)):
        sb.run(dev_sig)
    sb.run_host_stream([host, host2] * max(args.warmup, 1), harena * max(args.warmup, 1))
    torch.cuda.synchronize()

    def timed_e2e():
        """All K steps through ShardedBatch.run_host_stream (copies overlapped
        with compute): shard H2D, extrapolate, gather to the root, root D2H of
        the gathered results; one event pair around the whole sequence."""
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        ins = [host if i % 2 == 0 else host2 for i in range(args.steps)]
        out = [harena[i % 2] for i in range(args.steps)]
        e0.record(stream)
        sb.run_host_stream(ins, out)
        e1.record(stream)
        return [[e0, e1]]

    def timed(steps, split=False):
        """``steps`` device-resident steps, each between two events (L2 flushed
        before each). ``split``: also events between the stages -- a separate,
        untimed diagnostic pass, since an event between two kernels serializes
        them (the latency shapes' programmatic dependent launch) and adds its
        own gap to a ~100 us step."""
        evs = []
        for _ in range(steps):
            _native.l2_flush(flush)
            e = [torch.cuda.Event(enable_timing=True) if split or i in (0, 4) else None
                 for i in range(5)]
            e[0].record(stream)
            plan._products(sig_view)  # signals resident in HBM, read in place
            if split:
                e[1].record(stream)
            if plan.fused_synth:  # recursion with the synthesis inside
                plan._iterate_synth(plan.selected, plan.projections, plan.coefficients,
                                    plan.lost)
                if split:
                    e[2].record(stream)
            else:
                iterate(plan.G, plan.D, plan.R0, K, I, w.config.gamma, plan.selected,
                        plan.projections, plan.coefficients)
                if split:
                    e[2].record(stream)
                if cplx:
                    synth(plan.phi_lost, plan.selected, plan.coefficients, I, plan.lost_seq,
                          plan.lost, n_shared=plan.n_lost, dst=plan.lost_pos, **synth_extra)
                else:  # the plan's synthesis (Ozaki product or per-block paste)
                    plan._synth(plan.selected, plan.coefficients, plan.lost)
            if split:
                e[3].record(stream)
            sb.arena.gather(0)  # results of every rank to the root (NCCL; no-op at N=1)
            e[4].record(stream)
            evs.append(e)
        return evs

    gpu_id = str(local)
    try:
        uuid = torch.cuda.get_device_properties(dev).uuid
        gpu_id = f"GPU-{uuid}"
    except AttributeError:
        pass
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(gpu_id) as clocks:
        t_wall0 = time.perf_counter()
        ev_dev = timed(args.steps)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ev_e2e = timed_e2e()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t_wall = time.perf_counter() - t_wall0
    dev_ms = [e[0].elapsed_time(e[4]) for e in ev_dev]
    # the stage split: a separate pass after the clock (stage events inside the
    # timed steps would serialize the kernels they sit between)
    ev_split = timed(min(args.steps, 20), split=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    init_ms = [e[0].elapsed_time(e[1]) for e in ev_split]
    iter_ms = [e[1].elapsed_time(e[2]) for e in ev_split]
    synth_ms = [e[2].elapsed_time(e[3]) for e in ev_split]
    gather_ms = [e[3].elapsed_time(e[4]) for e in ev_split]
    e2e_ms = [e[0].elapsed_time(e[1]) for e in ev_e2e]
    tot = torch.tensor([sum(dev_ms), sum(e2e_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    dev_total_s, e2e_total_s = tot[0].item() / 1e3, tot[1].item() / 1e3

    # correctness guard on the timed outputs (not timed): range / finiteness on
    # every rank; on the root, the gathered batch against the reference fixture
    sel = plan.selected
    assert int(sel.min()) >= 0 and int(sel.max()) < K, "selection out of range"
    assert torch.isfinite(plan.lost).all(), "non-finite reconstruction"
    parity = None
    fixture = None if not args.dict else ("dft1" if args.dict == "dft" and args.config == 1 else "")
    if sb.is_root and fixture != "":
        g_sel, g_coef, g_lost = (x.cpu().numpy() for x in sb.arena.assemble(0))
        parity = parity_vs_reference(args.config, g_sel, g_coef, g_lost, plan.n_lost, fixture)
        if parity is not None and parity["failure"]:
            raise RuntimeError(f"timed outputs diverge from the reference: {parity}")
        if args.config == 4 and not args.dict:  # all 4,096 selected sequences
            every = parity_vs_reference(4, g_sel, g_coef, g_lost, plan.n_lost, "c4all")
            if every is not None:
                if every["failure"]:
                    raise RuntimeError(f"timed selections diverge from the reference: {every}")
                parity["all_blocks_selections"] = {k: every[k] for k in (
                    "fixture", "blocks_checked", "identical", "near_tie", "failure")}
    agreement = None
    if recursion == "scaled":
        # the same shard through the exact (reference-bit-identical) recursion
        sel_x, proj_x, coef_x = (torch.empty_like(x) for x in (plan.selected, plan.projections,
                                                               plan.coefficients))
        (_native.iterate_complex if cplx else _native.iterate)(
            plan.G, plan.D, plan.R0, K, I, w.config.gamma, sel_x, proj_x, coef_x)
        same = (sel_x == plan.selected).all(dim=1)
        dev_c = ((coef_x - plan.coefficients).abs().amax(dim=1)
                 / coef_x.abs().amax(dim=1).clamp_min(1e-300))
        agreement = {"blocks_identical_selections": int(same.sum()), "blocks": B,
                     "max_coef_rel_dev": float(dev_c[same].max()) if bool(same.any()) else None,
                     "vs": "fase_iterate (exact) on the same R0 / table"}
    dropin = None
    if rank == 0 and world == 1 and not cplx:
        dropin = time_dropin(w, d, mask, tables, dev)

    if rank == 0:
        hbm, hsrc, fp64, fsrc = measured_peaks()
        it_s = float(np.mean(iter_ms)) / 1e3
        bytes_iter = (16.0 if cplx else 8.0) * K * B * I
        achieved = bytes_iter / it_s / 1e9
        init_s = float(np.mean(init_ms)) / 1e3
        flops_init = (4.0 if cplx else 2.0) * K * M * B
        if plan._support is not None:  # contraction over the support samples only
            flops_init = (4.0 if cplx else 2.0) * K * int(plan._support[0].shape[0]) * B
        factors = d.device_factors(dev) if plan.products in ("auto", "separable") else None
        mr, nc = w.area
        if factors:  # executed flops of the separable form
            flops_sep = sum(2.0 * B * (r.shape[0] * mr * nc + r.shape[0] * nc * c.shape[0])
                            for r, c, _ in factors)
        elif cplx and plan.products_method.startswith("separable"):
            # complex transforms: [Cn; Sn] X^T (2 Lc x Mr x Nc), then 2 Lr x Lc x 2 Mr;
            # rows outside the separable ranges (if any) go through the DMMA GEMM
            cparts = d.device_cfactors(dev)
            flops_sep = sum(2.0 * B * (2 * c.shape[0] * mr * nc + 4 * r.shape[0] * c.shape[0] * mr)
                            for r, _, c, _, _ in cparts)
            covered = sum(r.shape[0] * c.shape[0] for r, _, c, _, _ in cparts)
            flops_sep += 4.0 * (K - covered) * M * B
            factors = cparts
        step_ms = dev_total_s / args.steps * 1e3
        tag = ("dft" if args.dict == "dft" else f"c{args.config}") + (
            "-scaled" if recursion == "scaled" else "")
        kname = "fase_iterate_complex_kernel" if cplx else "fase_iterate_kernel"
        line = {
            "metric": "extrapolated blocks/s",
            "value": B_total * args.steps / dev_total_s,
            "unit": "blocks/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": step_ms,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "c128" if cplx else "f64",
            "data": "synthetic (seeded BASELINE Appendix-A generators; random atoms: none)",
            "config": dict(workload_config(w, world, args.dict),
                           **({"blocks": B_total, "blocks_note": "--blocks: the first B blocks of "
                               "the workload's batch"} if args.blocks else {})),
            "e2e": {"value": B_total * args.steps / e2e_total_s, "unit": "blocks/s",
                    "h2d_bytes_per_step": int(host.numel() * 8) * world,
                    "d2h_bytes_per_step": sb.arena.nbytes * world,
                    "ms_per_step": e2e_total_s / args.steps * 1e3,
                    "api": "ShardedBatch.run_host_stream (ExtrapolationPlan per rank): pinned host "
                           "shard in, extrapolation, result gather to rank 0, rank-0 D2H of the "
                           "gathered selections / coefficients / lost samples, every step; copies "
                           "on side streams overlapped with compute; no L2 flush (per-step input "
                           "comes over PCIe)"},
            "roofline": roofline_recursion(achieved, hbm, hsrc, kname, tag, recursion, bytes_iter,
                                           it_s, cplx, B, I),
            "roofline_l2": l2_roofline(achieved, ncu_profile(kname, tag), 8, B, I),
            "roofline_init": (ozaki_roofline(plan, flops_init, init_s, fp64, fsrc)
                              if plan._ozaki is not None else
                              {"bound": "tensor", "kernel": "dgemm_nt_kernel (DMMA FP64)"
                               + (" over the support samples" if plan._support is not None else ""),
                               "achieved": flops_init / init_s / 1e12, "peak": fp64,
                               "unit": "TFLOP/s", "frac": flops_init / init_s / 1e12 / fp64,
                               "ms_per_launch": init_s * 1e3, "peak_source": fsrc}
                              if not factors else
                              {"bound": "tensor" if not cplx else "fp64",
                               "kernel": ("sep_products_dmma_kernel (separable transforms on DMMA, "
                                          "weights fused, all parts in one launch)") if not cplx else
                                         "weigh_kernel + sep_products_complex_kernel (separable "
                                         "transforms, FP64 FMA)",
                               "achieved": flops_sep / init_s / 1e12, "peak": fp64,
                               "unit": "TFLOP/s", "frac": flops_sep / init_s / 1e12 / fp64,
                               "ms_per_launch": init_s * 1e3, "peak_source": fsrc,
                               "dense_equivalent_tflops": flops_init / init_s / 1e12,
                               "note": "executed flops of rows X cols^T per part; the dense "
                                       "GEMM form (--products gemm) does 24x more work"}),
            "products": plan.products_method,
            "recursion": recursion,
            "fused_synth": plan.fused_synth,
            "synthesis": ("ozaki (sparse models x Phi_lost^T, %d digit planes)" % plan._synth_oz[0].slices
                          if plan._synth_oz is not None else ("fused" if plan.fused_synth else "paste")),
            "l2_hint": l2_hint,
            "parity_vs_reference": parity,
            "recursion_agreement": agreement,
            "stage_ms": {"init_products": float(np.mean(init_ms)), "iterate": float(np.mean(iter_ms)),
                         "synth": float(np.mean(synth_ms)), "gather": float(np.mean(gather_ms))},
            "stage_ms_pass": f"{len(ev_split)} untimed steps after the clock with events between "
                             "the stages (the timed steps carry events at their ends only)",
            "shard": {"blocks_total": B_total, "blocks_rank0": B, "ranks": world,
                      "gather_bytes_per_rank": sb.arena.nbytes,
                      "collective": "torch.distributed.gather (NCCL) of one result arena per "
                                    "rank, inside the timed region" if world > 1 else
                                    "none (one rank)"},
            "gram_ms": gram_ms,
            "gram_path": gram_path,
            "fft_gram_ms": fft_gram_ms,
            "gram_tflops": (4 if cplx else 1) * K * (K + 1) * M / (gram_ms * 1e-3) / 1e12,
            "gram_fp64_frac": (4 if cplx else 1) * K * (K + 1) * M / (gram_ms * 1e-3) / 1e12 / fp64,
            "gpu_launches": args.steps * (plan.launches_per_run + 1) + args.steps * plan.launches_per_run,
            "e2e_dropin": dropin,
            "clocks": clocks.summary(),
            "wall_s": t_wall,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def time_dropin(w, d, mask, tables, dev):
    """One batch through the drop-in ``fase_extrapolate_batch`` (host numpy in,
    host results out, per-call validation / provenance check / uploads /
    allocations): the host overhead of the reference-facing call next to the
    prepared-plan figure. Warm once, then time one call (wall clock around a
    synchronizing call)."""
    import torch

    from paper_2204_14194_b200 import fase_extrapolate_batch

    sig = wl.block_signals(w.cid, w.n_blocks, *w.area)
    res = fase_extrapolate_batch(sig, mask, d, tables, w.config, device=dev, recursion="scaled")
    torch.cuda.synchronize()
    res.to_host()  # warm the pinned staging buffers
    t0 = time.perf_counter()
    res = fase_extrapolate_batch(sig, mask, d, tables, w.config, device=dev, recursion="scaled")
    host = res.to_host()
    t = time.perf_counter() - t0
    return {"value": w.n_blocks / t, "unit": "blocks/s", "ms_per_call": t * 1e3,
            "api": "fase_extrapolate_batch(host numpy signals, mask, dictionary, tables, config) "
                   "+ BatchResult.to_host() (selected, coefficients, patched areas through "
                   "reusable pinned buffers): per-call validation, pageable upload, kernels, "
                   "read-back",
            "h2d_bytes": int(sig.nbytes),
            "d2h_bytes": int(sum(v.nbytes for v in host.values() if v is not None))}


def roofline_recursion(achieved, hbm, hsrc, kname, tag, recursion, bytes_iter, it_s, cplx, B, I):
    """The recursion against HBM: ``achieved`` counts the algorithmic bytes (one
    table row per block-iteration); most rows are L2 hits, so the
    DRAM bytes ncu measured for the same kernel (``traffic``) are reported with
    their own rate and fraction (``dram_*``) -- the honest HBM figure."""
    traffic = ncu_traffic(kname, tag)
    prof = ncu_profile(kname, tag)
    out = {"bound": "hbm", "kernel": kname + (" (scaled: column-scaled table)"
                                              if recursion == "scaled" else ""),
           "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
           "traffic": traffic, "algorithmic_bytes_per_launch": bytes_iter,
           "ms_per_launch": it_s * 1e3, "peak_source": hsrc,
           "note": ("16*K" if cplx else "8*K") + " bytes per block-iteration (one table row); "
                   "rows mostly hit L2, so achieved/frac exceed what DRAM serves: dram_gbs / "
                   "dram_frac are the ncu DRAM bytes of the same kernel over the live time"}
    if traffic:
        out["dram_gbs"] = traffic / it_s / 1e9
        out["dram_frac"] = traffic / it_s / 1e9 / hbm
    if prof:
        out["ncu"] = prof
    return out


def run_gpu_frame(args):
    """Configs 2/3: one step = conceal one damaged frame (all lossy macroblocks),
    the lossy tiles sharded over the ranks (ShardedFrame: every rank conceals
    block_range(L, r, N) of the tiles, results gathered to rank 0, which pastes
    the other ranks' tiles)."""
    import torch
    import torch.distributed as dist

    from paper_2204_14194_b200 import ShardedFrame, _native
    from paper_2204_14194_b200.conceal import FrameEngine, lossy_tiles, tile_grid

    rank, world, local = dist_env()
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.config, args.cpu_seconds)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    _native.load()
    w = wl.WORKLOADS[args.config]
    d = w.dictionary()
    case = wl.frame_case(w)
    K, M, I = len(d), w.area[0] * w.area[1], w.config.iterations
    engine = FrameEngine(d, case.frame.shape, case.mb, case.support, w.config, device=dev,
                         **({"compose": args.compose} if args.compose else {}))
    grid_h = tile_grid(case.lost, case.mb)
    corners_h = lossy_tiles(case.lost, (case.mb, case.mb)).astype(np.int32)
    L_total = len(corners_h)
    frame_u8 = torch.from_numpy(case.frame).pin_memory()
    lost_h = torch.from_numpy(case.lost)
    grid = torch.from_numpy(grid_h).to(dev)
    corners = torch.from_numpy(corners_h).to(dev)
    sf = ShardedFrame(engine, grid, corners)
    L = sf.hi - sf.lo
    damaged = torch.from_numpy(case.damaged()).to(dev)
    out = damaged.clone()
    out_host = torch.empty(out.shape, dtype=torch.float64, pin_memory=True)
    out_host2 = torch.empty(out.shape, dtype=torch.float64, pin_memory=True)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    lost_dev = lost_h.to(dev)
    for _ in range(max(args.warmup, 1)):
        sf.run(damaged, out=out)
    torch.cuda.synchronize()
    if engine.dead_blocks():
        raise RuntimeError("a block had every atom degenerate")
    sf.run_host_stream([frame_u8] * 2, [out_host, out_host2], lost_dev)
    torch.cuda.synchronize()
    if sf.is_root and (not torch.equal(out_host, out_host2) or not torch.equal(out_host, out.cpu())):
        raise RuntimeError("pipelined frames differ from the single-frame run")
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    gpu_id = str(local)
    try:
        gpu_id = f"GPU-{torch.cuda.get_device_properties(dev).uuid}"
    except AttributeError:
        pass
    dev_ms, e2e_ms = [], []
    with ClockSampler(gpu_id) as clocks:
        t_wall0 = time.perf_counter()
        for _ in range(args.steps):
            _native.l2_flush(flush)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            sf.run(damaged, out=out)  # this rank's tiles + gather (+ root paste)
            e1.record(stream)
            dev_ms.append((e0, e1))
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        # end to end: K frames through ShardedFrame.run_host_stream (uploads,
        # kernels, gather and root read-backs of neighbouring frames
        # overlapped); one event pair around the whole sequence
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        sf.run_host_stream([frame_u8] * args.steps, [out_host, out_host2] * args.steps, lost_dev)
        e1.record(stream)
        e2e_ms.append((e0, e1))
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t_wall = time.perf_counter() - t_wall0
    dev_t = sum(a.elapsed_time(b) for a, b in dev_ms) / 1e3
    e2e_t = sum(a.elapsed_time(b) for a, b in e2e_ms) / 1e3
    tot = torch.tensor([dev_t, e2e_t], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    dev_t, e2e_t = tot.tolist()
    parity = None
    if sf.is_root:
        g_sel, g_coef, _ = (x.cpu().numpy() for x in sf.arena.assemble(0))
        parity = parity_vs_reference(args.config, g_sel, g_coef, None, 0)
        if parity is not None and parity["failure"]:
            raise RuntimeError(f"timed outputs diverge from the reference: {parity}")
        every = parity_vs_reference(args.config, g_sel, g_coef, None, 0, f"c{args.config}all")
        if every is not None:  # every block of the frame: selected sequences
            if every["failure"]:
                raise RuntimeError(f"timed selections diverge from the reference: {every}")
            parity["all_blocks_selections"] = {k: every[k] for k in (
                "fixture", "blocks_checked", "identical", "near_tie", "failure")}
    # kernel split of this rank's tiles, for the roofline
    b = engine._buffers(L)
    engine.run(damaged, grid, sf.local_corners, out=out)
    torch.cuda.synchronize()
    counts = b["counts"].float()
    # rows streamed per block-iteration: the base row plus the chunks left after
    # the precomposed bases (the first one or two cells of a list)
    absorbed = {None: 0, "singles": 1, "pairs": 2, "triples": 3}[engine.compose_mode]
    mean_rows = 1.0 + float((counts - counts.clamp(max=absorbed)).mean())
    # recursion alone (same inputs as the last run)
    ev_i0 = torch.cuda.Event(enable_timing=True)
    ev_i1 = torch.cuda.Event(enable_timing=True)
    ev_i0.record(stream)
    _native.iterate(engine.G0, b["D"], b["R0"], K, I, w.config.gamma, b["sel"], b["proj"], b["coef"],
                    chunk_tables=engine.tables, chunk_stride=engine.stride,
                    chunk_count=b["counts"], chunk_ids=b["ids"], compose=engine.compose,
                    base_stride=engine.G0.numel())
    ev_i1.record(stream)
    torch.cuda.synchronize()
    it_s = ev_i0.elapsed_time(ev_i1) / 1e3
    if rank == 0:
        hbm, hsrc, fp64, fsrc = measured_peaks()
        # SURVEY 8(d) unit: one FP64 table row (8 K bytes) per block-iteration;
        # the chunked tables stream (1 + unavailable cells) rows for it
        bytes_iter = 8.0 * K * L * I
        achieved = bytes_iter / it_s / 1e9
        streamed = bytes_iter * mean_rows
        traffic = ncu_traffic("fase_iterate_kernel", f"c{args.config}")
        line = {
            "metric": "extrapolated blocks/s", "value": L_total * args.steps / dev_t,
            "unit": "blocks/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dev_t / args.steps * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic frame (seeded BASELINE Appendix-A generator)",
            "config": dict(workload_config(w, world), blocks_per_frame=L_total,
                           cells=len(engine.cells), mean_rows_per_iteration=mean_rows,
                           composed_bases=engine.compose_mode),
            "e2e": {"value": L_total * args.steps / e2e_t, "unit": "blocks/s",
                    "h2d_bytes_per_step": int(case.frame.nbytes) * world,
                    "d2h_bytes_per_step": int(out_host.numel() * 8),
                    "ms_per_step": e2e_t / args.steps * 1e3,
                    "api": "ShardedFrame.run_host_stream (FrameEngine per rank): pinned uint8 frame "
                           "in on every rank, its tiles concealed, results gathered to rank 0 "
                           "(pastes the rest), restored float64 frame (pinned) out every step; "
                           "neighbouring frames' copies and kernels overlapped; no L2 flush"},
            "roofline": {"bound": "hbm", "kernel": "fase_iterate_kernel (chunked rows)",
                         "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                         "traffic": traffic,
                         "dram_gbs": traffic / it_s / 1e9 if traffic else None,
                         "dram_frac": traffic / it_s / 1e9 / hbm if traffic else None,
                         "algorithmic_bytes_per_launch": bytes_iter,
                         "ms_per_launch": it_s * 1e3, "peak_source": hsrc,
                         "streamed_bytes_per_launch": streamed,
                         "streamed_gbs": streamed / it_s / 1e9,
                         "ncu": ncu_profile("fase_iterate_kernel", f"c{args.config}"),
                         "note": "achieved counts 8*K bytes (one table row) per block-iteration, "
                                 "the SURVEY 8(d) unit; the per-block table G0 - sum C_cell "
                                 "streams one base row (G0 or a precomposed G0 - C_c1 (- C_c2)) "
                                 "plus the remaining unavailable cells' rows for it "
                                 "(streamed_*), served largely from L2"},
            "parity_vs_reference": parity,
            "shard": {"blocks_total": L_total, "blocks_rank0": L, "ranks": world,
                      "gather_bytes_per_rank": sf.arena.nbytes},
            "table_build_s": engine.table_seconds,
            "gpu_launches": args.steps * (engine.launches_per_frame + 1) + args.steps * engine.launches_per_frame,
            "clocks": clocks.summary(), "wall_s": t_wall, "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse_args()
    if args.impl == "reference":
        run_reference(args)
    elif wl.WORKLOADS[args.config].shared_geometry:
        run_gpu(args)
    else:
        run_gpu_frame(args)


if __name__ == "__main__":
    main()
