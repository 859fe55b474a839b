"""Generate the golden fixtures under tests/golden/ FROM THE REFERENCE ITSELF.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the unmodified reference package from /root/reference/pkg/src and
calls its public API (weights, dictionaries, Gram tables, fase_extrapolate,
se_extrapolate, apply_model) on inputs produced by this repo's seeded
generators (paper_2204_14194_b200.workloads), then stores inputs' seeds and the
reference outputs as small .npz files. Nothing at test / bench time reads
/root/reference: the GPU box only sees these fixtures.

Custom BASELINE families (DCT u Hadamard-48, real DFT u sign, Gaussian) are
handed to the reference as ``fase.Dictionary(values)`` -- the reference's own
container for numerically defined atoms (dictionary.py:59-85).
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

import fase  # noqa: E402  (the reference)

from paper_2204_14194_b200 import workloads as wl  # noqa: E402
from paper_2204_14194_b200.dictionary import parse_dict_spec  # noqa: E402


def ref_dictionary(spec: str, m: int, n: int):
    """Reference Dictionary for a spec; custom kinds via Dictionary(values)."""
    try:
        return fase.parse_dict_spec(spec, m, n)
    except ValueError:
        ours = parse_dict_spec(spec, m, n)
        return fase.Dictionary(ours.real_values())


def run_block(d, signal, mask, cfg, tables=None, record=False):
    w = fase.build_weight_field(mask, cfg.rho_hat)
    if tables is None:
        tables = fase.build_gram_tables(d, w)
    r0 = fase.initial_scalar_products(signal, w, d)
    model, trace = fase.fase_extrapolate(signal, mask, d, tables, cfg, record_products=record)
    patched, max_imag = fase.apply_model(signal, model, mask)
    out = {
        "r0": r0.real.copy(),
        "selected": np.asarray(trace.selected, dtype=np.int64),
        "projections": trace.projections.real.copy(),
        "coefficients": trace.coefficients.real.copy(),
        "patched_lost": patched[mask].copy(),
        "max_imag": np.float64(max_imag),
        "d": tables.d.copy(),
    }
    if record:
        out["products"] = np.stack([p.real for p in trace.products])
    return out, tables


def small_cases():
    cases = []
    specs = [("dct", 8, 8, (4, 4)), ("wht", 8, 8, (4, 4)), ("union:dct+wht", 8, 8, (4, 4)),
             ("union:dct+had", 12, 12, (4, 4)), ("dct", 16, 16, (8, 8)),
             ("union:rdft+brdft", 8, 8, (2, 2)), ("had", 12, 12, (4, 6)), ("dct", 6, 10, (2, 4))]
    out = {}
    for i, (spec, m, n, loss) in enumerate(specs):
        d = ref_dictionary(spec, m, n)
        mask = wl.central_loss_mask(m, n, *loss)
        cfg = fase.ExtrapConfig(iterations=40, gamma=[0.5, 1.0, 0.25][i % 3], rho_hat=0.8)
        signal = np.random.default_rng([2204, i]).uniform(0.0, 255.0, (m, n))
        res, tables = run_block(d, signal, mask, cfg, record=True)
        _, se_trace = fase.se_extrapolate(signal, mask, d, cfg)
        key = f"case{i}"
        out[f"{key}_signal"] = signal
        out[f"{key}_mask"] = mask
        out[f"{key}_gram"] = tables.c.real.copy()
        out[f"{key}_se_selected"] = np.asarray(se_trace.selected, dtype=np.int64)
        out[f"{key}_se_coefficients"] = se_trace.coefficients.real.copy()
        for k, v in res.items():
            out[f"{key}_{k}"] = v
        cases.append({"key": key, "spec": spec, "m": m, "n": n, "loss": list(loss),
                      "iterations": cfg.iterations, "gamma": cfg.gamma, "rho_hat": cfg.rho_hat,
                      "provenance": str(tables.provenance),
                      "content_hash": str(d.content_hash())})
    np.savez_compressed(HERE / "small_cases.npz", **out)
    return cases


def complex_cases():
    """Complex dictionaries (the reference's default ``dft`` and its relatives)."""
    specs = [("dft", 8, 8, (4, 4)), ("bdft", 8, 8, (4, 4)), ("union:dft+bdft", 6, 6, (2, 2)),
             ("union:dct+dft", 8, 8, (4, 4)), ("dft", 6, 10, (2, 4)), ("bdft", 12, 12, (4, 4)),
             ("union:wht+dft", 16, 16, (8, 8))]
    cases, out = [], {}
    for i, (spec, m, n, loss) in enumerate(specs):
        d = fase.parse_dict_spec(spec, m, n)
        mask = wl.central_loss_mask(m, n, *loss)
        cfg = fase.ExtrapConfig(iterations=40, gamma=[0.5, 1.0, 0.25][i % 3], rho_hat=0.8)
        signal = np.random.default_rng([2204, 100 + i]).uniform(0.0, 255.0, (m, n))
        w = fase.build_weight_field(mask, cfg.rho_hat)
        tables = fase.build_gram_tables(d, w)
        r0 = fase.initial_scalar_products(signal, w, d)
        model, trace = fase.fase_extrapolate(signal, mask, d, tables, cfg, record_products=True)
        patched, max_imag = fase.apply_model(signal, model, mask)
        key = f"z{i}"
        out.update({f"{key}_signal": signal, f"{key}_mask": mask, f"{key}_gram": tables.c,
                    f"{key}_d": tables.d, f"{key}_r0": r0,
                    f"{key}_selected": np.asarray(trace.selected, dtype=np.int64),
                    f"{key}_projections": trace.projections, f"{key}_coefficients": trace.coefficients,
                    f"{key}_products": np.stack(trace.products),
                    f"{key}_patched_lost": patched[mask], f"{key}_max_imag": np.float64(max_imag)})
        cases.append({"key": key, "spec": spec, "m": m, "n": n, "loss": list(loss),
                      "iterations": cfg.iterations, "gamma": cfg.gamma, "rho_hat": cfg.rho_hat,
                      "provenance": str(tables.provenance), "content_hash": str(d.content_hash())})
    np.savez_compressed(HERE / "complex_cases.npz", **out)
    return cases


def complex_blocks(n_blocks: int = 3):
    """The reference's default dictionary (dft) on the config-1 area and loss."""
    w1 = wl.WORKLOADS[1]
    m, n = w1.area
    d = fase.parse_dict_spec("dft", m, n)
    mask = wl.central_loss_mask(m, n, *w1.loss)
    cfg = fase.ExtrapConfig(w1.config.iterations, w1.config.gamma, w1.config.rho_hat)
    sig = wl.block_signals(1, n_blocks, m, n)
    w = fase.build_weight_field(mask, cfg.rho_hat)
    tables = fase.build_gram_tables(d, w)
    out = {"blocks": np.arange(n_blocks), "d": tables.d.copy(), "provenance": np.uint64(tables.provenance),
           "gram_diag": tables.c.diagonal().real.copy(), "gram_row0": tables.c[0].copy(),
           "gram_row777": tables.c[777].copy()}
    t0 = time.time()
    for b in range(n_blocks):
        r0 = fase.initial_scalar_products(sig[b], w, d)
        model, trace = fase.fase_extrapolate(sig[b], mask, d, tables, cfg)
        patched, max_imag = fase.apply_model(sig[b], model, mask)
        out.update({f"b{b}_r0": r0, f"b{b}_selected": np.asarray(trace.selected, dtype=np.int64),
                    f"b{b}_projections": trace.projections, f"b{b}_coefficients": trace.coefficients,
                    f"b{b}_patched_lost": patched[mask], f"b{b}_max_imag": np.float64(max_imag)})
    np.savez_compressed(HERE / "dft48_blocks.npz", **out)
    return {"spec": "dft", "area": [m, n], "blocks": n_blocks, "seconds": time.time() - t0}


def transform_cases():
    """The reference's transform shortcuts (fft_initial_products / fft_gram_table)."""
    out, rec = {}, []
    for i, (spec, m, n) in enumerate([("dft", 8, 8), ("dft", 4, 6), ("union:dct+dft", 8, 8),
                                      ("dft", 12, 12)]):
        d = fase.parse_dict_spec(spec, m, n)
        mask = wl.central_loss_mask(m, n, m // 2, n // 2)
        w = fase.build_weight_field(mask, 0.8)
        s = np.random.default_rng([2204, 200 + i]).uniform(0.0, 255.0, (m, n))
        out[f"t{i}_signal"] = s
        out[f"t{i}_w"] = w
        out[f"t{i}_products"] = fase.fft_initial_products(s, w, d, min_tagged=1)
        if len(d.tagged_indices()) == len(d):
            t = fase.fft_gram_table(w, d)
            out[f"t{i}_gram"] = t.c
            out[f"t{i}_d"] = t.d
        rec.append({"key": f"t{i}", "spec": spec, "m": m, "n": n})
    np.savez_compressed(HERE / "transform_cases.npz", **out)
    return rec


def conceal_cases():
    """The reference's conceal_image (clipped border areas, per-tile paste, report)."""
    rng = np.random.default_rng(22042)
    h, w = 37, 45
    yy, xx = np.mgrid[0:h, 0:w]
    img = 128 + 40 * np.cos(0.31 * yy + 0.17 * xx) + 25 * np.sin(0.11 * yy - 0.27 * xx + 1.0)
    img = np.clip(img + rng.normal(0, 2, (h, w)), 0, 255)
    lost = np.zeros((h, w), dtype=bool)
    lost[0:5, 0:6] = True        # top-left corner tile (clipped area)
    lost[10:14, 18:23] = True    # interior
    lost[30:37, 40:45] = True    # bottom-right partial tile
    lost[17:20, 0:3] = True      # left edge
    observed = img.copy()
    observed[lost] = 0.0
    out, meta = {}, []
    runs = [("dct", (8, 8), 4, 30), ("dft", (8, 8), 4, 30), ("union:dct+dft", (12, 10), 3, 20)]
    for i, (spec, block, support, iters) in enumerate(runs):
        cfg = fase.ExtrapConfig(iterations=iters, gamma=0.5, rho_hat=0.8)
        restored, report = fase.conceal_image(observed, lost, dict_spec=spec, config=cfg,
                                              block=block, support=support, reference=img,
                                              single_thread=True)
        out[f"k{i}_restored"] = restored
        for b in report["blocks"]:
            b.pop("seconds")
        report.pop("seconds")
        meta.append({"key": f"k{i}", "spec": spec, "block": list(block), "support": support,
                     "iterations": iters, "report": report})
    # whole image as one area (block=None), the reference's default dictionary
    small = img[:16, :16].copy()
    lost16 = fase.central_loss_mask(16, 16, 4, 4)
    obs16 = small.copy()
    obs16[lost16] = 0.0
    restored, report = fase.conceal_image(obs16, lost16, config=fase.ExtrapConfig(iterations=40),
                                          reference=small)
    out["whole_restored"] = restored
    out["whole_observed"] = obs16
    out["whole_reference"] = small
    out["whole_lost"] = lost16
    for b in report["blocks"]:
        b.pop("seconds")
    report.pop("seconds")
    meta.append({"key": "whole", "spec": "dft", "block": None, "support": 24, "iterations": 40,
                 "report": report})
    out["image"] = img
    out["observed"] = observed
    out["lost"] = lost
    np.savez_compressed(HERE / "conceal_cases.npz", **out)
    with open(HERE / "conceal_cases.json", "w") as fh:
        json.dump(meta, fh)
    return [m["key"] for m in meta]


def complex_arithmetic():
    """numpy's complex128 product and abs on this host (the oracle's semantics)."""
    rng = np.random.default_rng(22041)
    n = 4099
    x = (rng.standard_normal(n) + 1j * rng.standard_normal(n)) * 10.0 ** rng.integers(-4, 5, n)
    y = (rng.standard_normal(n) + 1j * rng.standard_normal(n)) * 10.0 ** rng.integers(-4, 5, n)
    x[::7] = x[::7].real
    y[3::11] = 1j * y[3::11].imag
    c = complex(rng.standard_normal(), rng.standard_normal())
    np.savez_compressed(HERE / "complex_arith.npz", x=x, y=y, c=np.complex128(c), xy=x * y,
                        cy=c * np.conj(y), absx=np.abs(x))


def weights_and_hashes():
    rec = {"weights": [], "hashes": []}
    arrays = {}
    for i, (m, n, rho, loss) in enumerate([(3, 3, 0.5, (1, 1)), (48, 48, 0.8, (16, 16)),
                                           (64, 64, 0.85, (24, 24)), (32, 32, 0.8, (8, 8)),
                                           (5, 7, 0.3, (1, 3))]):
        mask = wl.central_loss_mask(m, n, *loss)
        arrays[f"w{i}"] = fase.build_weight_field(mask, rho)
        arrays[f"mask{i}"] = mask
        rec["weights"].append({"key": f"w{i}", "rho": rho})
    for spec, m, n in [("dct", 4, 4), ("wht", 8, 8), ("dft", 4, 4), ("bdft", 4, 4),
                       ("union:dct+wht", 8, 8), ("dct", 48, 48), ("dft", 6, 5),
                       ("union:dct+had", 48, 48), ("union:rdft+brdft", 32, 32),
                       ("union:dct+had", 12, 12)]:
        d = ref_dictionary(spec, m, n)
        rec["hashes"].append({"spec": spec, "m": m, "n": n, "K": len(d),
                              "content_hash": str(d.content_hash())})
    g = wl.WORKLOADS[4].dictionary()
    rec["hashes"].append({"spec": wl.WORKLOADS[4].dict_spec, "m": 64, "n": 64, "K": len(g),
                          "content_hash": str(fase.Dictionary(g.real_values()).content_hash())})
    np.savez_compressed(HERE / "weights.npz", **arrays)
    return rec


def shared_config_blocks(cid: int, blocks):
    w = wl.WORKLOADS[cid]
    m, n = w.area
    d = ref_dictionary(w.dict_spec, m, n)
    mask = wl.central_loss_mask(m, n, *w.loss)
    cfg = fase.ExtrapConfig(w.config.iterations, w.config.gamma, w.config.rho_hat)
    sig = wl.block_signals(cid, max(blocks) + 1, m, n)
    tables = None
    out = {"blocks": np.asarray(blocks)}
    t0 = time.time()
    for b in blocks:
        res, tables = run_block(d, sig[b], mask, cfg, tables=tables)
        for k, v in res.items():
            if k == "d":
                continue
            out[f"b{b}_{k}"] = v
    out["d"] = tables.d.copy()
    out["gram_diag"] = tables.c.diagonal().real.copy()
    out["provenance"] = np.uint64(tables.provenance)
    np.savez_compressed(HERE / f"c{cid}_blocks.npz", **out)
    return {"config": cid, "blocks": list(blocks), "seconds": time.time() - t0}


def frame_config_blocks(cid: int, picks: int):
    w = wl.WORKLOADS[cid]
    case = wl.frame_case(w)
    signals, masks = wl.frame_areas(case.damaged(), case.lost, case.corners, case.mb, case.support)
    # cover the per-block geometries: most neighbour losses (interior), frame
    # edges / corners (out-of-frame samples), both at once, and a plain block
    h, wd = case.frame.shape
    a = case.area
    oof = np.empty(len(masks), dtype=np.int64)
    for i, (r, c) in enumerate(case.corners):
        rr = np.arange(r - case.support, r - case.support + a)
        cc = np.arange(c - case.support, c - case.support + a)
        inside = ((rr >= 0) & (rr < h))[:, None] & ((cc >= 0) & (cc < wd))[None, :]
        oof[i] = a * a - inside.sum()
    neigh = masks.reshape(len(masks), -1).sum(axis=1) - oof - case.mb * case.mb
    interior = np.flatnonzero(oof == 0)
    chosen = [0]
    chosen += list(interior[np.argsort(-neigh[interior], kind="stable")[:2]])
    both = np.flatnonzero((oof > 0) & (neigh > 0))
    if both.size:
        chosen.append(int(both[np.argmax(neigh[both])]))
    chosen.append(int(np.argmax(oof)))
    plain = np.flatnonzero((oof == 0) & (neigh == 0))
    if plain.size:
        chosen.append(int(plain[len(plain) // 2]))
    chosen = sorted(set(int(x) for x in chosen))[:picks]
    m, n = w.area
    d = ref_dictionary(w.dict_spec, m, n)
    cfg = fase.ExtrapConfig(w.config.iterations, w.config.gamma, w.config.rho_hat)
    out = {"blocks": np.asarray(chosen, dtype=np.int64), "n_blocks": np.int64(len(masks)),
           "lost_total": np.int64(case.lost.sum())}
    t0 = time.time()
    for b in chosen:
        res, _ = run_block(d, signals[b], masks[b], cfg)
        for k, v in res.items():
            out[f"b{b}_{k}"] = v
        out[f"b{b}_mask"] = masks[b]
        out[f"b{b}_signal_sum"] = np.float64(signals[b].sum())
    np.savez_compressed(HERE / f"c{cid}_blocks.npz", **out)
    return {"config": cid, "blocks": [int(x) for x in chosen], "seconds": time.time() - t0}


def fgrm_fixture():
    """A small table file written by the reference's own save_gram_table."""
    d = fase.parse_dict_spec("union:dct+wht", 4, 4)
    w = fase.build_weight_field(wl.central_loss_mask(4, 4, 2, 2), 0.8)
    t = fase.build_gram_tables(d, w)
    fase.save_gram_table(t, HERE / "ref_tables.fgrm")
    return {"spec": "union:dct+wht", "m": 4, "n": 4, "provenance": str(t.provenance)}


def main():
    meta = {"generator": "tests/golden/make_golden.py",
            "reference": "/root/reference/pkg (fase 0.1.0, unmodified)",
            "numpy": np.__version__}
    meta.update(weights_and_hashes())
    meta["small_cases"] = small_cases()
    meta["complex_cases"] = complex_cases()
    meta["transform_cases"] = transform_cases()
    meta["conceal_cases"] = conceal_cases()
    complex_arithmetic()
    meta["fgrm"] = fgrm_fixture()
    meta["c0"] = shared_config_blocks(0, [0])
    meta["c1"] = shared_config_blocks(1, [0, 1, 2, 3])
    meta["c4"] = shared_config_blocks(4, [0, 1])
    meta["c3"] = frame_config_blocks(3, 6)
    meta["c2"] = frame_config_blocks(2, 4)
    meta["dft48"] = complex_blocks()
    with open(HERE / "golden.json", "w") as fh:
        json.dump(meta, fh, indent=1)
    print(json.dumps({k: v for k, v in meta.items() if k.startswith("c")}, indent=1))


if __name__ == "__main__":
    main()
