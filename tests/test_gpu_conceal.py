"""GPU parity of ``conceal_image`` against the reference's own runs.

The fixtures (tests/golden/conceal_cases.*) are the reference's conceal_image
on a small scene with losses at corners, edges and the interior: clipped
border areas of several shapes, real, complex and mixed dictionaries, and the
whole-image mode with the default dictionary. Per block: identical tiling,
area and loss count; the selection trace identical up to a legitimate
near-tie; coefficients, restored pixels and PSNR within the BASELINE
tolerance (1e-6 of the run scale).
"""

import json

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import fase_oracle as orc  # noqa: E402
from paper_2204_14194_b200 import (  # noqa: E402
    ExtrapConfig,
    MaskError,
    ParameterError,
    ShapeError,
    build_gram_tables,
    build_weight_field,
    central_loss_mask,
    conceal_image,
    parse_dict_spec,
)
from paper_2204_14194_b200.conceal import REFERENCE_REPORT_SCHEMA  # noqa: E402
from parity import COEF_REL, compare_selection, metric_fn  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


@pytest.fixture(scope="module")
def golden(golden_dir):
    with open(golden_dir / "conceal_cases.json") as fh:
        meta = json.load(fh)
    return meta, np.load(golden_dir / "conceal_cases.npz")


def _check_report(got, want, image, lost, spec, iterations):
    assert got["schema"] == want["schema"] == REFERENCE_REPORT_SCHEMA
    assert got["image"] == want["image"]
    assert {k: v for k, v in got["settings"].items()} == want["settings"]
    assert got["lost_pixels"] == want["lost_pixels"]
    assert got["tables_reused"] == want["tables_reused"]
    assert len(got["blocks"]) == len(want["blocks"])
    exact = 0
    for g, w in zip(got["blocks"], want["blocks"]):
        for key in ("row", "col", "height", "width", "area", "lost"):
            assert g[key] == w[key], key
        gs = [t["atom"] for t in g["trace"]]
        ws = [t["atom"] for t in w["trace"]]
        gc = np.array([complex(*t["coefficient"]) for t in g["trace"]])
        wc = np.array([complex(*t["coefficient"]) for t in w["trace"]])
        a_r0, a_c0, ah, aw = w["area"]

        def metric_at(t, a_r0=a_r0, a_c0=a_c0, ah=ah, aw=aw):
            sig = image[a_r0:a_r0 + ah, a_c0:a_c0 + aw]
            msk = lost[a_r0:a_r0 + ah, a_c0:a_c0 + aw]
            vals = parse_dict_spec(spec, ah, aw).values
            ref = orc.extrapolate_block(sig, msk, vals, 0.5, t, 0.8, record=True)
            return metric_fn(ref["r0"], ref["d"], ref["log"])(t)

        v = compare_selection(gs, ws, metric_at)
        assert v.ok, f"block {(w['row'], w['col'])}: diverged at {v.stop}, gap {v.gap}"
        s = v.stop
        assert np.abs(gc[:s] - wc[:s]).max(initial=0) <= COEF_REL * np.abs(wc[:s]).max(initial=1)
        if v.exact:
            exact += 1
            assert abs(g["max_imag"] - w["max_imag"]) <= 1e-6 * max(1.0, w["max_imag"])
            if w["psnr_db"] is not None:
                assert abs(g["psnr_db"] - w["psnr_db"]) < 1e-6
    return exact


@pytest.mark.parametrize("i", [0, 1, 2])
def test_conceal_image_blocked_against_reference(golden, i):
    meta, z = golden
    case = meta[i]
    cfg = ExtrapConfig(case["iterations"], 0.5, 0.8)
    restored, report = conceal_image(z["observed"], z["lost"], dict_spec=case["spec"], config=cfg,
                                     block=tuple(case["block"]), support=case["support"],
                                     reference=z["image"], device=DEV)
    exact = _check_report(report, case["report"], z["observed"], z["lost"], case["spec"],
                          case["iterations"])
    assert exact >= len(case["report"]["blocks"]) - 1
    want = z[f"{case['key']}_restored"]
    assert np.array_equal(restored[~z["lost"]], want[~z["lost"]])  # support untouched
    if exact == len(case["report"]["blocks"]):
        assert np.abs(restored - want).max() <= COEF_REL * 255
        assert abs(report["psnr_db"] - case["report"]["psnr_db"]) < 1e-6


def test_conceal_image_whole_area_default_dictionary(golden):
    meta, z = golden
    case = meta[3]
    restored, report = conceal_image(z["whole_observed"], z["whole_lost"],
                                     config=ExtrapConfig(iterations=40),
                                     reference=z["whole_reference"], device=DEV)
    _check_report(report, case["report"], z["whole_observed"], z["whole_lost"], "dft", 40)
    assert np.abs(restored - z["whole_restored"]).max() <= COEF_REL * 255


def test_conceal_image_tables_fft_and_edges():
    rng = np.random.default_rng(4)
    img = np.clip(128 + 30 * np.cos(np.arange(256).reshape(16, 16) * 0.3) +
                  rng.normal(0, 1, (16, 16)), 0, 255)
    lost = central_loss_mask(16, 16, 4, 4)
    obs = img.copy()
    obs[lost] = 0.0
    cfg = ExtrapConfig(iterations=30)
    d = parse_dict_spec("dct", 16, 16)
    tables = build_gram_tables(d, build_weight_field(lost, cfg.rho_hat), device=DEV)
    plain, _ = conceal_image(obs, lost, dict_spec="dct", config=cfg, device=DEV)
    reused, rep = conceal_image(obs, lost, dict_spec="dct", config=cfg, tables=tables, device=DEV)
    assert rep["tables_reused"] == 1
    assert np.array_equal(plain, reused)
    direct, _ = conceal_image(obs, lost, dict_spec="dft", config=cfg, device=DEV)
    via_fft, rep = conceal_image(obs, lost, dict_spec="dft", config=cfg, use_fft=True, device=DEV)
    assert rep["settings"]["fft"] is True
    assert np.allclose(direct, via_fft, rtol=0, atol=1e-9)
    same, rep = conceal_image(img, np.zeros((16, 16), bool), device=DEV)
    assert np.array_equal(same, img) and rep["blocks"] == [] and rep["psnr_db"] is None
    with pytest.raises(ShapeError):
        conceal_image(img, np.zeros((16, 15), bool), device=DEV)
    with pytest.raises(ShapeError):
        conceal_image(img, lost, reference=np.zeros((4, 4)), device=DEV)
    with pytest.raises(ParameterError):
        conceal_image(img, lost, support=-1, device=DEV)
    with pytest.raises(ParameterError):
        conceal_image(img, lost, block=(0, 8), device=DEV)
    with pytest.raises(MaskError):  # an area with no support left
        conceal_image(img, np.ones((16, 16), bool), block=(8, 8), support=0, device=DEV)


def test_conceal_frame_complex_dictionary():
    """conceal_frame (fixed areas) with the default complex dictionary takes the
    FrameEngine pipeline (complex cell tables, precomposed bases, the complex
    chunked recursion and paste); every block's selections / coefficients and
    every lost pixel match the oracle's block result."""
    from paper_2204_14194_b200 import conceal_frame
    from paper_2204_14194_b200 import workloads as wl

    rng = np.random.default_rng(21)
    yy, xx = np.mgrid[0:48, 0:56]
    img = np.clip(120 + 50 * np.sin(0.21 * yy + 0.13 * xx) + rng.normal(0, 3, (48, 56)), 0, 255)
    lost = np.zeros((48, 56), dtype=bool)
    for r, c in [(8, 8), (0, 48), (24, 16), (40, 0), (16, 24)]:
        lost[r:r + 8, c:c + 8] = True
    cfg = ExtrapConfig(30, 0.5, 0.8)
    out, rep = conceal_frame(img, lost, dict_spec="dft", config=cfg, block=8, support=4, device=DEV)
    out = out.cpu().numpy()
    damaged = img.copy()
    damaged[lost] = 0.0
    corners = np.array(sorted({(r // 8 * 8, c // 8 * 8) for r, c in zip(*np.nonzero(lost))}))
    signals, masks = wl.frame_areas(damaged, lost, corners, 8, 4)
    vals = parse_dict_spec("dft", 16, 16).values
    assert rep["settings"]["pipeline"] == "frame-engine"
    res = rep["result"]
    for i, (r0, c0) in enumerate(corners):
        ref = orc.extrapolate_block(signals[i], masks[i], vals, 0.5, 30, 0.8, record=True)
        v = compare_selection(res.selected[i].cpu().numpy(), ref["selected"],
                              metric_fn(ref["r0"], ref["d"], ref["log"]))
        assert v.ok, f"block {i}: diverged at {v.stop}, gap {v.gap}"
        c = res.coefficients[i].cpu().numpy()[: v.stop]
        assert np.abs(c - ref["coefficients"][: v.stop]).max() <= COEF_REL * np.abs(
            ref["coefficients"]).max()
        tile = ref["patched"][4:12, 4:12]
        got = out[r0:r0 + 8, c0:c0 + 8]
        sel_lost = lost[r0:r0 + 8, c0:c0 + 8]
        assert np.abs(got[sel_lost] - tile[sel_lost]).max() <= COEF_REL * 255
        # apply_model's diagnostic over the tile's pasted pixels
        want_imag = float(np.abs(ref["g"].imag[4:12, 4:12][sel_lost]).max())
        assert abs(float(res.max_imag[i]) - want_imag) <= COEF_REL * max(want_imag, 1.0)
    assert np.array_equal(out[~lost], img[~lost])


@pytest.mark.parametrize("spec", ["dft", "union:dct+dft", "bdft"])
def test_frame_engine_complex_compose_bit_identical(spec):
    """Complex FrameEngine: precomposed bases (pairs, triples) stream rows
    bit-identical to the uncomposed cell lists, so every composition mode gives
    the same selections, coefficients and frame; mixed unions take the complex
    separable transform plus the DMMA GEMM for the real rows."""
    import torch

    from paper_2204_14194_b200.conceal import FrameEngine, lossy_tiles, tile_grid

    rng = np.random.default_rng(8)
    h, w, mb, sup = 40, 48, 8, 4
    img = rng.uniform(0, 255, (h, w))
    lost = np.zeros((h, w), dtype=bool)
    for ty, tx in [(0, 0), (0, 1), (1, 1), (2, 3), (4, 5), (3, 0), (4, 4)]:
        lost[ty * mb:(ty + 1) * mb, tx * mb:(tx + 1) * mb] = True
    img[lost] = 0.0
    d = parse_dict_spec(spec, mb + 2 * sup, mb + 2 * sup)
    cfg = ExtrapConfig(25, 0.5, 0.8)
    dev = torch.device(DEV)
    grid = torch.from_numpy(tile_grid(lost, mb)).to(dev)
    corners = torch.from_numpy(lossy_tiles(lost, (mb, mb)).astype(np.int32)).to(dev)
    outs = {}
    for mode in ("none", "pairs", "triples"):
        eng = FrameEngine(d, (h, w), mb, sup, cfg, device=dev, compose=mode)
        r = eng.run(torch.from_numpy(img).to(dev), grid, corners)
        outs[mode] = (r.selected.clone(), r.coefficients.clone(), r.patched.clone())
    for mode in ("pairs", "triples"):
        for a, b in zip(outs["none"], outs[mode]):
            assert torch.equal(a, b)
    # against the general per-block path (ChunkedTables) on the same areas
    from paper_2204_14194_b200 import fase_extrapolate_batch
    from paper_2204_14194_b200 import workloads as wl

    signals, masks = wl.frame_areas(img, lost, corners.cpu().numpy(), mb, sup)
    res = fase_extrapolate_batch(signals, masks, d, None, cfg, device=dev)
    same = (res.selected == outs["none"][0]).all(dim=1)
    assert int(same.sum()) >= len(same) - 1
    dc = (res.coefficients - outs["none"][1]).abs().amax(dim=1) / res.coefficients.abs().amax(dim=1)
    assert float(dc[same].max()) < 1e-12


@pytest.mark.parametrize("B", [1, 7, 1000, 25920])
def test_block_order_stable_by_cost_class(B):
    """fase_block_order: a permutation of the blocks by descending cost class
    min(7, max(0, count - depth)), ascending block index within a class."""
    from paper_2204_14194_b200 import _native

    rng = np.random.default_rng(B)
    counts = rng.integers(0, 14, B).astype(np.int32)
    dev = torch.device(DEV)
    for depth in (0, 3):
        order = torch.empty(B, dtype=torch.int32, device=dev)
        _native.block_order(torch.from_numpy(counts).to(dev), depth, order)
        got = order.cpu().numpy()
        cls = np.clip(counts - depth, 0, 7)
        want = np.lexsort((np.arange(B), -cls))  # class descending, then index
        assert np.array_equal(got, want)


@pytest.mark.parametrize("spec", ["dct", "dft"])
def test_frame_engine_dispatch_order_is_a_schedule_only(spec, monkeypatch):
    """Costliest-first dispatch (fase_iterate_args.order) changes which CTA runs
    which block, never a result: the frame, selections and coefficients are
    bit-identical to row-major dispatch."""
    from paper_2204_14194_b200 import conceal
    from paper_2204_14194_b200.conceal import FrameEngine, lossy_tiles, tile_grid

    rng = np.random.default_rng(9)
    h, w, mb, sup = 48, 56, 8, 4
    img = rng.uniform(0, 255, (h, w))
    lost = np.zeros((h, w), dtype=bool)
    for ty, tx in [(0, 0), (0, 1), (1, 1), (2, 3), (4, 5), (3, 0), (4, 4), (5, 6), (2, 2), (1, 3)]:
        lost[ty * mb:(ty + 1) * mb, tx * mb:(tx + 1) * mb] = True
    img[lost] = 0.0
    d = parse_dict_spec(spec, mb + 2 * sup, mb + 2 * sup)
    cfg = ExtrapConfig(20, 0.5, 0.8)
    dev = torch.device(DEV)
    grid = torch.from_numpy(tile_grid(lost, mb)).to(dev)
    corners = torch.from_numpy(lossy_tiles(lost, (mb, mb)).astype(np.int32)).to(dev)
    outs = []
    for on in (False, True):
        monkeypatch.setattr(conceal, "BLOCK_ORDER", on)
        eng = FrameEngine(d, (h, w), mb, sup, cfg, device=dev, compose="pairs")
        r = eng.run(torch.from_numpy(img).to(dev), grid, corners)
        outs.append((r.selected.clone(), r.coefficients.clone(), r.patched.clone()))
        if on:  # the order really permutes (cells lost around some tiles, not others)
            order = eng._buffers(int(corners.shape[0]))["order"].cpu().numpy()
            assert sorted(order.tolist()) == list(range(int(corners.shape[0])))
            assert not np.array_equal(order, np.arange(len(order)))
    for a, b in zip(*outs):
        assert torch.equal(a, b)


def test_frame_widen_kernel():
    """fase_frame_widen: uint8 frame -> float64 with lost pixels zeroed, exactly
    (odd widths and unaligned row starts take the scalar tail)."""
    import torch

    from paper_2204_14194_b200 import _native

    rng = np.random.default_rng(3)
    for h, w in ((1080, 1920), (37, 45), (5, 3)):
        img = rng.integers(0, 256, (h, w), dtype=np.uint8)
        lost = rng.random((h, w)) < 0.2
        want = img.astype(np.float64)
        want[lost] = 0.0
        dev = torch.device("cuda", 0)
        out = torch.full((h, w), -1.0, dtype=torch.float64, device=dev)
        _native.frame_widen(torch.from_numpy(img).to(dev), torch.from_numpy(lost).to(dev), out)
        assert np.array_equal(out.cpu().numpy(), want)


def test_batch_result_to_host_pinned():
    """BatchResult.to_host: host copies through reusable pinned buffers equal
    the plain read-back."""
    import torch

    from paper_2204_14194_b200 import fase_extrapolate_batch

    d = parse_dict_spec("union:dct+wht", 8, 8)
    mask = central_loss_mask(8, 8, 4, 4)
    sig = np.random.default_rng(5).uniform(0, 255, (7, 8, 8))
    res = fase_extrapolate_batch(sig, mask, d, None, ExtrapConfig(12), device=DEV)
    for _ in range(2):  # second call reuses the staging buffers
        h = res.to_host()
        assert np.array_equal(h["selected"], res.selected.cpu().numpy())
        assert np.array_equal(h["coefficients"], res.coefficients.cpu().numpy())
        assert np.array_equal(h["patched"], res.patched.cpu().numpy())
        assert torch.from_numpy(h["patched"]).is_pinned()
