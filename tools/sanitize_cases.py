"""Small invocations of every kernel family, for compute-sanitizer.

    compute-sanitizer --tool memcheck  python tools/sanitize_cases.py [--case NAME]
    compute-sanitizer --tool racecheck python tools/sanitize_cases.py
    compute-sanitizer --tool synccheck python tools/sanitize_cases.py

(tools/sanitize.sh runs all three and writes the logs.) Each case is sized to
select one kernel variant (the dispatch rules in csrc/iterate.cu,
csrc/iterate_complex.cu, fast.py) at the smallest shape that reaches it, so the
tools finish in minutes. A case prints one line; any CUDA fault raises.
"""

from __future__ import annotations

import argparse
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2204_14194_b200 import (  # noqa: E402
    Dictionary,
    ExtrapConfig,
    ExtrapolationPlan,
    build_gram_tables,
    build_weight_field,
    fase_extrapolate_batch,
    parse_dict_spec,
)
from paper_2204_14194_b200 import workloads as wl  # noqa: E402

DEV = torch.device("cuda", 0)
SMS = torch.cuda.get_device_properties(DEV).multi_processor_count if torch.cuda.is_available() else 148


def sig(b, m, n, seed=0):
    return np.random.default_rng(seed).uniform(0.0, 255.0, (b, m, n))


def per_block_masks(b, m, n, seed=1):
    """Centred loss plus a random neighbour cell per block: per-block geometries."""
    rng = np.random.default_rng(seed)
    base = wl.central_loss_mask(m, n, m // 3, n // 3)
    out = np.repeat(base[None], b, axis=0)
    for i in range(b):
        r, c = rng.integers(0, m - 2), rng.integers(0, n - 2)
        out[i, r:r + 2, c:c + 2] = True
    return out


def gauss(k, m, n, seed=3):
    v = np.random.default_rng(seed).standard_normal((k, m, n))
    return Dictionary(v / np.linalg.norm(v.reshape(k, -1), axis=1)[:, None, None])


def case_exact_plain():
    """fase_iterate_kernel, shared geometry, more blocks than SMs (3-4 CTAs/SM shapes)."""
    d = parse_dict_spec("union:dct+had", 12, 12)
    mask = wl.central_loss_mask(12, 12, 4, 4)
    r = fase_extrapolate_batch(sig(SMS + 12, 12, 12), mask, d, None, ExtrapConfig(12), device=DEV)
    return r.selected


def case_exact_latency():
    """Latency variant (at most one block per SM), K = 2304."""
    d = parse_dict_spec("dct", 48, 48)
    mask = wl.central_loss_mask(48, 48, 16, 16)
    return fase_extrapolate_batch(sig(2, 48, 48), mask, d, None, ExtrapConfig(6), device=DEV).selected


def case_exact_paired():
    """Paired blocks (two blocks per 512-thread CTA sharing D), 4608 < K <= 8192."""
    d = gauss(5000, 8, 8)
    mask = wl.central_loss_mask(8, 8, 3, 3)
    return fase_extrapolate_batch(sig(SMS + 2, 8, 8), mask, d, None, ExtrapConfig(5),
                                  device=DEV).selected


def case_exact_regs():
    """512-thread variant with R and D in registers (K > 5120, few blocks)."""
    d = gauss(6000, 8, 8)
    mask = wl.central_loss_mask(8, 8, 3, 3)
    return fase_extrapolate_batch(sig(3, 8, 8), mask, d, None, ExtrapConfig(5), device=DEV).selected


def case_record():
    """R logged after every iteration (record_products)."""
    d = parse_dict_spec("union:dct+wht", 8, 8)
    mask = wl.central_loss_mask(8, 8, 4, 4)
    r = fase_extrapolate_batch(sig(3, 8, 8), mask, d, None, ExtrapConfig(10), device=DEV,
                               record_products=True)
    return r.selected


def case_scaled():
    """fase_iterate_scaled at full occupancy and the fused-synthesis variant."""
    d = parse_dict_spec("union:dct+had", 12, 12)
    mask = wl.central_loss_mask(12, 12, 4, 4)
    cfg = ExtrapConfig(12)
    t = build_gram_tables(d, build_weight_field(mask, cfg.rho_hat), device=DEV)
    for b in (SMS + 12, 3):  # plain, fused synthesis (latency shape)
        p = ExtrapolationPlan(d, mask, b, cfg, t, device=DEV, recursion="scaled")
        p.run(torch.from_numpy(sig(b, 12, 12)).to(DEV))
    return p.selected


def case_scaled_large():
    """Scaled 256 x 32 shape (K = 8192 capacity, two CTAs per SM) and Ozaki products."""
    d = gauss(6000, 16, 16)
    mask = wl.central_loss_mask(16, 16, 6, 6)
    cfg = ExtrapConfig(4)
    t = build_gram_tables(d, build_weight_field(mask, cfg.rho_hat), device=DEV)
    p = ExtrapolationPlan(d, mask, SMS + 4, cfg, t, device=DEV, recursion="scaled",
                          products="ozaki")
    p.run(torch.from_numpy(sig(SMS + 4, 16, 16)).to(DEV))
    return p.selected


def case_chunked():
    """Per-block geometries: chunk tables, the chunked recursion, block normalizers."""
    d = parse_dict_spec("union:dct+had", 12, 12)
    masks = per_block_masks(20, 12, 12)
    return fase_extrapolate_batch(sig(20, 12, 12), masks, d, None, ExtrapConfig(12),
                                  device=DEV).selected


def case_frame():
    """FrameEngine: areas, cells, normalizers, precomposed bases, held rows, paste."""
    from paper_2204_14194_b200.conceal import FrameEngine, lossy_tiles, tile_grid

    d = parse_dict_spec("union:rdft+brdft", 16, 16)
    rng = np.random.default_rng(5)
    h, w, mb = 64, 96, 8
    img = rng.uniform(0, 255, (h, w))
    lost = np.zeros((h, w), dtype=bool)
    for ty, tx in [(0, 0), (0, 1), (3, 5), (4, 5), (7, 11), (2, 0), (5, 8)]:
        lost[ty * mb:(ty + 1) * mb, tx * mb:(tx + 1) * mb] = True
    img[lost] = 0.0
    eng = FrameEngine(d, (h, w), mb, 4, ExtrapConfig(20), device=DEV, compose="triples")
    grid = torch.from_numpy(tile_grid(lost, mb)).to(DEV)
    corners = torch.from_numpy(lossy_tiles(lost, (mb, mb)).astype(np.int32)).to(DEV)
    return eng.run(torch.from_numpy(img).to(DEV), grid, corners).selected


def case_complex():
    """Complex recursion: exact (shared and chunked), scaled, paired; complex Gram / synthesis."""
    d = parse_dict_spec("dft", 8, 8)
    mask = wl.central_loss_mask(8, 8, 3, 3)
    cfg = ExtrapConfig(10)
    fase_extrapolate_batch(sig(SMS + 3, 8, 8), mask, d, None, cfg, device=DEV)
    fase_extrapolate_batch(sig(6, 8, 8), per_block_masks(6, 8, 8), d, None, cfg, device=DEV)
    u = parse_dict_spec("union:dft+bdft", 48, 48)  # K = 4608 complex
    m48 = wl.central_loss_mask(48, 48, 16, 16)
    fase_extrapolate_batch(sig(SMS + 2, 48, 48), m48, u, None, ExtrapConfig(3), device=DEV)
    r = fase_extrapolate_batch(sig(4, 48, 48), m48, u, None, ExtrapConfig(3), device=DEV,
                               recursion="scaled")
    return r.selected


def case_products():
    """Initial products: separable DMMA (batch), per-part separable, DMMA GEMM, complex separable."""
    mask = wl.central_loss_mask(16, 16, 6, 6)
    cfg = ExtrapConfig(3)
    for spec, prod in (("union:dct+had", "separable"), ("union:dct+had", "gemm"),
                       ("dct", None), ("union:dct+dft", None)):
        d = parse_dict_spec(spec, 16, 16)
        fase_extrapolate_batch(sig(SMS + 1, 16, 16), mask, d, None, cfg, device=DEV,
                               **({"recursion": "exact"} if prod is None else {}))
        if prod:
            t = build_gram_tables(d, build_weight_field(mask, cfg.rho_hat), device=DEV)
            p = ExtrapolationPlan(d, mask, 9, cfg, t, device=DEV, products=prod)
            p.run(torch.from_numpy(sig(9, 16, 16)).to(DEV))
    return None


def case_gram():
    """Gram tables: DMMA (small K), Ozaki symmetric (K >= 2048), transform shortcut."""
    from paper_2204_14194_b200 import fft_gram_table

    mask = wl.central_loss_mask(16, 16, 6, 6)
    w = build_weight_field(mask, 0.8)
    build_gram_tables(parse_dict_spec("union:dct+wht", 16, 16), w, device=DEV)
    build_gram_tables(gauss(2100, 16, 16), w, device=DEV)
    fft_gram_table(w, parse_dict_spec("dft", 16, 16), device=DEV)
    return None


CASES = {k[5:]: v for k, v in globals().items() if k.startswith("case_")}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", default="all", choices=["all", *CASES])
    args = ap.parse_args()
    names = list(CASES) if args.case == "all" else [args.case]
    for name in names:
        t0 = time.perf_counter()
        CASES[name]()
        torch.cuda.synchronize()
        print(f"case {name}: ok ({time.perf_counter() - t0:.1f} s)", flush=True)


if __name__ == "__main__":
    main()
