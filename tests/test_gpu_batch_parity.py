"""Parity on the BENCHMARKED batches, against reference-written fixtures.

``tests/golden/make_batch_golden.py`` ran the unmodified reference over the
blocks ``bench.py`` times (all 1,024 config-1 blocks, 256 config-4 blocks, 256
config-3 and 128 config-2 frame blocks covering every edge / corner /
neighbour-loss class) and stored, per block, the selected sequence, the
coefficients, the reconstructed lost samples and the reference's near-tie sets.

Here the bench's own device paths run the same batches -- ``ExtrapolationPlan``
(exact and scaled recursions) for the shared-geometry configs, ``FrameEngine``
for the frames -- and every block is classified per SURVEY 8(c) step 2:

- ``identical``: the whole selected sequence equals the reference's;
- ``near_tie``: the first divergence is at an iteration where the GPU's atom
  is one the reference's tie rule could pick if Delta-E moved by 1e-9 relative
  (BASELINE north_star; ``make_batch_golden.near_ties``), read off the
  reference's own per-iteration R vectors;
- ``failure``: anything else.

Coefficients must match to 1e-6 of the run scale up to the first divergence,
reconstructed samples to 1e-6 on identical blocks. The counts are printed and
written to ``gpurun_out/batch_parity.json``; the test fails on any failure.
"""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np
import pytest

from paper_2204_14194_b200 import workloads as wl

from parity import COEF_REL  # noqa: E402

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
GOLD = Path(__file__).resolve().parent / "golden"
REPORT = ROOT / "gpurun_out" / "batch_parity.json"


def classify(got_sel, got_coef, z, rows=None, got_lost=None):
    """Per-block verdicts against a batch fixture; ``rows[i]`` is the row of
    fixture block i in the GPU outputs (default: i)."""
    want_sel = z["selected"].astype(np.int64)
    want_coef = z["coefficients"] if "coefficients" in z.files else None  # selections-only fixtures
    # (NpzFile members decompress on every access: load each array once)
    z_lost = z["lost"] if want_coef is not None else None
    z_lost_n = z["lost_n"] if want_coef is not None else None
    z_blocks = z["blocks"]
    ties = {}
    for i, t, k in z["ties"]:
        ties.setdefault((int(i), int(t)), set()).add(int(k))
    counts = {"identical": 0, "near_tie": 0, "failure": 0, "blocks": len(want_sel)}
    stops, failures, worst_coef, worst_lost = [], [], 0.0, 0.0
    for i in range(len(want_sel)):
        r = i if rows is None else int(rows[i])
        g = np.asarray(got_sel[r], dtype=np.int64)
        diff = np.flatnonzero(g != want_sel[i])
        stop = int(diff[0]) if diff.size else len(g)
        if diff.size == 0:
            counts["identical"] += 1
        elif int(g[stop]) in ties.get((i, stop), ()):
            counts["near_tie"] += 1
            stops.append(stop)
        else:
            counts["failure"] += 1
            failures.append((int(z_blocks[i]), stop, int(g[stop]), int(want_sel[i][stop])))
            continue
        if want_coef is None:
            continue
        c = np.asarray(got_coef[r])[:stop]
        scale = max(np.abs(want_coef[i]).max(), 1e-300)
        dev = float(np.abs(c - want_coef[i][:stop]).max(initial=0.0)) / scale
        worst_coef = max(worst_coef, dev)
        if diff.size == 0 and got_lost is not None:
            n = int(z_lost_n[i])
            want = z_lost[i][:n]
            got = np.asarray(got_lost(i, r))
            worst_lost = max(worst_lost, float(np.abs(got - want).max(initial=0.0))
                             / max(np.abs(want).max(initial=0.0), 1e-300))
    counts.update(near_tie_stops=sorted(stops), failures=failures[:10],
                  max_coef_rel_dev=worst_coef, max_lost_rel_dev=worst_lost,
                  tie_iterations_in_reference=len({(int(a), int(b)) for a, b, _ in z["ties"]}))
    return counts


def _report(key, counts):
    REPORT.parent.mkdir(exist_ok=True)
    data = json.loads(REPORT.read_text()) if REPORT.exists() else {}
    data[key] = counts
    REPORT.write_text(json.dumps(data, indent=1))
    print(f"\n[batch parity] {key}: {counts['identical']} identical, {counts['near_tie']} "
          f"near-tie stops, {counts['failure']} failures of {counts['blocks']} blocks; "
          f"coef dev {counts['max_coef_rel_dev']:.2e}, lost dev {counts['max_lost_rel_dev']:.2e}")


def _check(counts):
    assert counts["failure"] == 0, f"non-tie divergences: {counts['failures']}"
    assert counts["max_coef_rel_dev"] < COEF_REL
    assert counts["max_lost_rel_dev"] < COEF_REL


@pytest.mark.parametrize("recursion", ["exact", "scaled"])
@pytest.mark.parametrize("cid", [1, 4])
def test_shared_batch_against_reference(cid, recursion):
    """The bench's ExtrapolationPlan over the full config batch (c1: 1,024
    blocks; c4: 4,096 blocks, the first 256 pinned by the reference)."""
    import torch

    from paper_2204_14194_b200 import ExtrapolationPlan, build_gram_tables, build_weight_field

    z = np.load(GOLD / f"c{cid}_batch.npz")
    w = wl.WORKLOADS[cid]
    dev = torch.device("cuda", 0)
    d = w.dictionary()
    mask = wl.central_loss_mask(*w.area, *w.loss)
    tables = build_gram_tables(d, build_weight_field(mask, w.config.rho_hat), device=dev)
    assert int(tables.provenance) == int(z["provenance"])
    plan = ExtrapolationPlan(d, mask, w.n_blocks, w.config, tables, device=dev,
                             recursion=recursion)
    sig = torch.from_numpy(wl.block_signals(cid, w.n_blocks, *w.area)).to(dev)
    plan.run(sig)
    torch.cuda.synchronize()
    lost = plan.lost.cpu().numpy()
    counts = classify(plan.selected.cpu().numpy(), plan.coefficients.cpu().numpy(), z,
                      got_lost=lambda i, r: lost[r, : plan.n_lost])
    counts["recursion"] = recursion
    _report(f"c{cid}-{recursion}", counts)
    _check(counts)
    if cid == 4:  # every one of the 4,096 blocks: selected sequences vs the reference
        za = np.load(GOLD / "c4all_batch.npz")
        assert len(za["blocks"]) == w.n_blocks
        counts = classify(plan.selected.cpu().numpy(), plan.coefficients.cpu().numpy(), za)
        counts["recursion"] = recursion
        _report(f"c4all-{recursion}", counts)
        assert counts["failure"] == 0, f"non-tie divergences: {counts['failures']}"


@pytest.mark.parametrize("cid", [3, 2])
def test_frame_batch_against_reference(cid):
    """The bench's FrameEngine over the whole frame (per-block geometries,
    precomposed bases, held rows); the reference pins the fixture blocks,
    including frame edges, corners and neighbour losses."""
    import torch

    from paper_2204_14194_b200.conceal import FrameEngine, lossy_tiles, tile_grid

    z = np.load(GOLD / f"c{cid}_batch.npz")
    w = wl.WORKLOADS[cid]
    dev = torch.device("cuda", 0)
    case = wl.frame_case(w)
    engine = FrameEngine(w.dictionary(), case.frame.shape, case.mb, case.support, w.config,
                         device=dev)
    grid = torch.from_numpy(tile_grid(case.lost, case.mb)).to(dev)
    corners_h = lossy_tiles(case.lost, (case.mb, case.mb))
    assert np.array_equal(corners_h, case.corners)
    assert int(z["n_blocks"]) == len(corners_h)
    corners = torch.from_numpy(corners_h.astype(np.int32)).to(dev)
    damaged = torch.from_numpy(case.damaged()).to(dev)
    res = engine.run(damaged, grid, corners)
    torch.cuda.synchronize()
    out = res.patched.cpu().numpy()
    _, masks = wl.frame_areas(case.damaged(), case.lost, case.corners, case.mb, case.support)
    mb, s, a = case.mb, case.support, case.area
    own = np.zeros((a, a), dtype=bool)
    own[s:s + mb, s:s + mb] = True
    blocks = z["blocks"]
    z_lost, z_lost_n = z["lost"], z["lost_n"]

    def got_lost(i, r):
        # the fixture's lost samples are in area-mask order; the frame holds
        # the own tile's pixels (conceal.py:144-148 pastes only those)
        b = int(blocks[i])
        sel = own[masks[b]]
        r0, c0 = case.corners[b]
        full = z_lost[i][: int(z_lost_n[i])].copy()
        full[sel] = out[r0:r0 + mb, c0:c0 + mb].ravel()  # row-major = mask order
        return full

    counts = classify(res.selected.cpu().numpy(), res.coefficients.cpu().numpy(), z,
                      rows=blocks, got_lost=got_lost)
    counts["classes_covered"] = int(len({tuple(c) for c in z["classes"]}))
    _report(f"c{cid}-frame", counts)
    _check(counts)
    # every block of the frame: selected sequences vs the reference
    za = np.load(GOLD / f"c{cid}all_batch.npz")
    assert np.array_equal(za["blocks"], np.arange(len(corners_h)))
    counts = classify(res.selected.cpu().numpy(), res.coefficients.cpu().numpy(), za)
    _report(f"c{cid}all-frame", counts)
    assert counts["failure"] == 0, f"non-tie divergences: {counts['failures']}"


@pytest.mark.parametrize("recursion", ["exact", "scaled"])
def test_dft_batch_against_reference(recursion):
    """The reference's default (complex) dictionary ``dft`` on the config-1
    batch (bench.py --dict dft): 1,024 blocks through ExtrapolationPlan, the
    first 256 pinned by the reference (complex coefficients)."""
    import torch

    from paper_2204_14194_b200 import (ExtrapolationPlan, build_gram_tables, build_weight_field,
                                       parse_dict_spec)

    z = np.load(GOLD / "dft1_batch.npz")
    w = wl.WORKLOADS[1]
    dev = torch.device("cuda", 0)
    d = parse_dict_spec("dft", *w.area)
    mask = wl.central_loss_mask(*w.area, *w.loss)
    tables = build_gram_tables(d, build_weight_field(mask, w.config.rho_hat), device=dev)
    assert int(tables.provenance) == int(z["provenance"])
    plan = ExtrapolationPlan(d, mask, w.n_blocks, w.config, tables, device=dev,
                             recursion=recursion)
    sig = torch.from_numpy(wl.block_signals(1, w.n_blocks, *w.area)).to(dev)
    plan.run(sig)
    torch.cuda.synchronize()
    lost = plan.lost.cpu().numpy()
    counts = classify(plan.selected.cpu().numpy(), plan.coefficients.cpu().numpy(), z,
                      got_lost=lambda i, r: lost[r, : plan.n_lost])
    counts["recursion"] = recursion
    _report(f"dft1-{recursion}", counts)
    _check(counts)
