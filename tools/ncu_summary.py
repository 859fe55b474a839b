"""Summarise ncu reports (read here, captured on the B200 via gpurun).

    python tools/ncu_summary.py OUT_PREFIX REPORT.ncu-rep|REPORT.raw.csv [...] [--launches launches.csv]

Writes OUT_PREFIX.md (human summary) and merges per-kernel DRAM traffic into
profiles/ncu_summary.json under "<tag>/<kernel>", tag = the suffix after
"_ncu_" in OUT_PREFIX (c1, c4, dft ...); bench.py reads it for the roofline
"traffic" key of the matching config.
"""

from __future__ import annotations

import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit rate"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput % peak"),
    ("lts__t_bytes.sum", "L2 slice traffic (`lts__t_bytes`)"),
    ("l1tex__m_xbar2l1tex_read_bytes.sum", "L2 -> SM read bytes over the crossbar"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput % peak"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active %"),
    ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
     "tensor pipe active, realtime % of elapsed (tcgen05)"),
    ("sm__inst_executed_pipe_tensor_subpipe_imma.avg.pct_of_peak_sustained_active",
     "IMMA subpipe instructions % peak"),
    ("sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
     "tensor memory (smem operand / TMEM) cycles active %"),
    ("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
     "DMMA subpipe instructions % peak"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe active %"),
    ("sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active", "shared pipe active %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall: barrier"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall: wait"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
     "stall: long scoreboard"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
     "stall: short scoreboard"),
    ("smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
     "stall: math pipe"),
]


def raw_rows(rep: str):
    """Rows of a report's raw page: from the .ncu-rep (ncu -i), or from a CSV
    already exported with ``ncu -i REP --page raw --csv`` on the GPU box."""
    if rep.endswith(".csv"):
        out = Path(rep).read_text()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [(dict(zip(hdr, r)), dict(zip(hdr, units))) for r in rows[2:]]


def to_bytes(val: str, unit: str) -> float:
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    return float(val.replace(",", "")) * scale.get(unit, 1)


def short(name: str) -> str:
    for key in ("fase_iterate_complex_kernel", "fase_iterate_kernel", "dgemm_nt_kernel",
                "synth_paste_complex_kernel", "synth_paste_pair_kernel", "synth_paste_kernel",
                "scale_columns_kernel", "gram_finish_kernel",
                "weigh_gather_kernel", "weigh_kernel", "sep_products_complex_kernel",
                "sep_products_dmma_kernel",
                "sep_products_kernel", "ozaki_gemm_kernel", "ozaki_split_kernel",
                "block_normalizers_kernel", "basis_outer_kernel", "flush_kernel",
                "frame_areas_kernel", "frame_cells_kernel", "frame_paste_kernel"):
        if key in name:
            return key
    return name[:60]


def main():
    args = sys.argv[1:]
    launches = None
    if "--launches" in args:
        i = args.index("--launches")
        launches = args[i + 1]
        del args[i:i + 2]
    out, reps = args[0], args[1:]
    lines = [f"# ncu summary ({Path(out).name})", ""]
    js_path = ROOT / "profiles" / "ncu_summary.json"
    js = json.loads(js_path.read_text()) if js_path.exists() else {}
    for rep in reps:
        for row, unit in raw_rows(rep):
            name = row["Kernel Name"]
            lines.append(f"## `{name}`  ({Path(rep).name})")
            lines.append("")
            lines.append("| metric | value |")
            lines.append("|---|---|")
            for key, label in METRICS:
                if key in row and row[key] != "":
                    lines.append(f"| {label} (`{key}`) | {row[key]} {unit.get(key, '')} |")
            lines.append("")
            traffic = to_bytes(row["dram__bytes_read.sum"], unit["dram__bytes_read.sum"]) + \
                to_bytes(row["dram__bytes_write.sum"], unit["dram__bytes_write.sum"])
            tag = Path(out).name.split("_ncu_")[-1]  # e.g. profiles/r01_ncu_c1 -> c1
            rec = {"dram_bytes_per_launch": traffic, "report": Path(rep).name,
                   "duration_ms": float(row["gpu__time_duration.sum"].replace(",", "")) *
                   (1e-3 if unit["gpu__time_duration.sum"] == "us" else 1.0)}
            for key, field in (("l1tex__m_xbar2l1tex_read_bytes.sum", "xbar_read_bytes_per_launch"),
                               ("lts__t_bytes.sum", "lts_bytes_per_launch")):
                if row.get(key):
                    rec[field] = to_bytes(row[key], unit[key])
            for key, field in (("lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts_throughput_pct"),
                               ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_pct"),
                               ("smsp__inst_executed.sum", "warp_instructions"),
                               ("lts__t_sector_hit_rate.pct", "l2_hit_pct")):
                if row.get(key):
                    rec[field] = float(row[key].replace(",", ""))
            js[f"{tag}/{short(name)}"] = rec
    if launches:
        lines.append("## launch list (cold-cache, serialised: compare shares, not absolutes)")
        lines.append("")
        tot = {}
        for row in csv.DictReader(l for l in open(launches) if not l.startswith("==")):
            if row.get("Metric Name") != "gpu__time_duration.sum":
                continue
            v = float(row["Metric Value"].replace(",", ""))
            if row.get("Metric Unit") == "us":
                v *= 1e3
            elif row.get("Metric Unit") == "ms":
                v *= 1e6
            k = short(row["Kernel Name"])
            tot.setdefault(k, [0, 0.0])
            tot[k][0] += 1
            tot[k][1] += v
        s = sum(v[1] for v in tot.values()) or 1.0
        lines.append("| kernel | launches | total ns | share |")
        lines.append("|---|---|---|---|")
        for k, (n, v) in sorted(tot.items(), key=lambda x: -x[1][1]):
            lines.append(f"| {k} | {n} | {v:.0f} | {v / s * 100:.1f}% |")
        lines.append("")
    Path(out + ".md").write_text("\n".join(lines))
    js_path.write_text(json.dumps(js, indent=1))
    print("\n".join(lines))


if __name__ == "__main__":
    main()
