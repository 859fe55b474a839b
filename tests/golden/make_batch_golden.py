"""Batch-scale golden fixtures FROM THE REFERENCE ITSELF (the benchmarked batches).

Run in the build container (where /root/reference exists):

    python tests/golden/make_batch_golden.py [--procs 8] [--only c1,c4,c3,c2]

The unmodified reference (``/root/reference/pkg/src``) runs ``fase_extrapolate``
+ ``apply_model`` on the exact blocks ``bench.py`` times:

- c1: all 1,024 blocks of the config-1 batch (shared table);
- c4: blocks 0..255 of the config-4 batch (shared table);
- c3: 256 of the 25,920 frame blocks, every edge / corner / neighbour-loss class
  first, then an even stride over the frame (per-block tables);
- c2: 128 of the 804 frame blocks, chosen the same way;
- dft1: blocks 0..255 of the config-1 batch with the reference's default
  (complex) dictionary ``dft`` (K = 2304; complex coefficients);
- c4all / c2all / c3all: EVERY block of the config-4 batch / config-2 frame /
  config-3 frame, selected sequences and near-tie sets only (coefficients and
  samples are pinned on the samples above). Not in the default --only list
  for c3all (about 25 minutes on 8 cores).

Per block it stores the selected sequence (int16), the coefficients, the
reconstructed lost samples (mask order) and the reference's NEAR-TIE SETS: for
every iteration t where a 1e-9 relative perturbation of Delta-E = (|R|*D)^2
(BASELINE north_star) could change the tie rule's pick, the records (block, t,
k) of every atom k it could pick (see ``near_ties``), read off the reference's
own per-iteration R vectors (``record_products``, ``fast.py:251-252``). A GPU
sequence that first diverges at t is a legitimate near-tie stop iff its atom at
t is in that set; anything else is a failure.

Blocks are spread over worker processes (one BLAS thread each); shared tables
are built once in the parent and inherited through fork. Nothing at test time
reads /root/reference: the GPU box only sees the .npz files.
"""

from __future__ import annotations

import argparse
import json
import multiprocessing as mp
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

TIE_REL = 1e-9
_G = {}


def ref_dictionary(spec: str, m: int, n: int):
    try:
        return fase.parse_dict_spec(spec, m, n)
    except ValueError:
        return fase.Dictionary(parse_dict_spec(spec, m, n).real_values())


def near_ties(r0, log, d, selected):
    """[(t, k)]: the atoms k the tie rule could pick at iteration t if every
    metric moved by up to 1e-9 relative Delta-E of the top (the BASELINE
    near-tie tolerance), for iterations where that is more than one atom.

    The reference picks the lowest index with metric >= top - q, q the running
    tie quantum (``reference.py:58-85``). With delta = 0.5e-9 * top on the
    metric scale (1e-9 on Delta-E = metric^2): atoms >= top - q + delta are
    surely eligible, atoms >= top - q - delta possibly; the possible picks are
    the possibly-eligible atoms at or below the lowest surely-eligible index.
    With q ~ 1e-13 * top this is the plain top-two rule (every atom within 1e-9
    relative Delta-E of the top); once q has grown past delta it also covers
    atoms sitting on the threshold.
    """
    out = []
    dead = d == 0
    q = 0.0
    for t in range(len(selected)):
        r = r0 if t == 0 else log[t - 1]
        m = np.abs(r) * d
        m[dead] = -np.inf
        top = m.max()
        q = max(q, 1e-13 * top if np.isfinite(top) and top > 0 else 0.0)
        delta = 0.5 * TIE_REL * top
        sure = np.flatnonzero(m >= top - q + delta)
        maybe = np.flatnonzero(m >= top - q - delta)
        if sure.size:
            maybe = maybe[maybe <= sure[0]]
        assert int(selected[t]) in set(maybe.tolist())
        if maybe.size > 1:
            out.extend((t, int(k)) for k in maybe)
    return out


def _block(args):
    """One block through the reference: shared tables from the parent, or its own."""
    i, signal, mask = args
    from threadpoolctl import threadpool_limits

    d, cfg, tables = _G["d"], _G["cfg"], _G["tables"]
    with threadpool_limits(limits=1):
        w = fase.build_weight_field(mask, cfg.rho_hat)
        if tables is None:
            tables = fase.build_gram_tables(d, w)
        r0 = fase.initial_scalar_products(signal, w, d)
        model, trace = fase.fase_extrapolate(signal, mask, d, tables, cfg, record_products=True)
        patched, _ = fase.apply_model(signal, model, mask)
        ties = near_ties(r0, trace.products, tables.d, trace.selected)
    coef = trace.coefficients if _G.get("complex") else trace.coefficients.real.copy()
    return (i, np.asarray(trace.selected, dtype=np.int16), coef, patched[mask].real.copy(), ties)


def _run(jobs, procs):
    out = [None] * len(jobs)
    with mp.get_context("fork").Pool(procs) as pool:
        for res in pool.imap_unordered(_block, jobs, chunksize=4):
            out[res[0]] = res
    return out


def _pack(name, blocks, results, extra, selections_only=False):
    n = len(blocks)
    sel = np.stack([r[1] for r in results])
    if selections_only:  # whole batches: the selected sequences and near-tie sets only
        ties = np.array([(i, t, k) for i, r in enumerate(results) for t, k in r[4]],
                        dtype=np.int32).reshape(-1, 3)
        np.savez_compressed(HERE / f"{name}_batch.npz", blocks=np.asarray(blocks, dtype=np.int32),
                            selected=sel, ties=ties, **extra)
        return {"blocks": n, "iterations": int(sel.size), "selections_only": True,
                "tie_iterations": len({(int(a), int(b)) for a, b, _ in ties}) if len(ties) else 0,
                "file": f"{name}_batch.npz"}
    coef = np.stack([r[2] for r in results])
    lost = [r[3] for r in results]
    nl = max(len(x) for x in lost)
    lost_arr = np.full((n, nl), np.nan)
    lost_n = np.zeros(n, dtype=np.int32)
    for i, x in enumerate(lost):
        lost_arr[i, : len(x)] = x
        lost_n[i] = len(x)
    ties = np.array([(i, t, k) for i, r in enumerate(results) for t, k in r[4]],
                    dtype=np.int32).reshape(-1, 3)
    np.savez_compressed(HERE / f"{name}_batch.npz", blocks=np.asarray(blocks, dtype=np.int32),
                        selected=sel, coefficients=coef, lost=lost_arr, lost_n=lost_n,
                        ties=ties, **extra)
    tie_iters = len({(int(a), int(b)) for a, b, _ in ties}) if len(ties) else 0
    return {"blocks": n, "tie_iterations": tie_iters,
            "iterations": int(sel.size), "file": f"{name}_batch.npz"}


def shared_batch(cid: int, n_blocks: int, procs: int, spec: str | None = None, name=None,
                 selections_only=False):
    w = wl.WORKLOADS[cid]
    m, n = w.area
    d = ref_dictionary(spec or w.dict_spec, m, n)
    mask = wl.central_loss_mask(m, n, *w.loss)
    cfg = fase.ExtrapConfig(w.config.iterations, w.config.gamma, w.config.rho_hat)
    t0 = time.time()
    tables = fase.build_gram_tables(d, fase.build_weight_field(mask, cfg.rho_hat))
    t_tab = time.time() - t0
    _G.update(d=d, cfg=cfg, tables=tables, complex=bool(spec) and not np.isrealobj(d.values))
    sig = wl.block_signals(cid, n_blocks, m, n)
    blocks = list(range(n_blocks))
    t0 = time.time()
    res = _run([(i, sig[b], mask) for i, b in enumerate(blocks)], procs)
    rec = _pack(name or f"c{cid}", blocks, res, {"provenance": np.uint64(tables.provenance)},
                selections_only)
    rec.update(table_seconds=t_tab, seconds=time.time() - t0)
    _G.clear()
    return rec


def block_classes(case, masks):
    """Per block: (out-of-frame sides bitmask, number of other lost samples) --
    the geometry classes the per-block tables depend on."""
    h, wd = case.frame.shape
    a, s = case.area, case.support
    keys = []
    for i, (r, c) in enumerate(case.corners):
        sides = (int(r - s < 0) | int(r - s + a > h) << 1 | int(c - s < 0) << 2
                 | int(c - s + a > wd) << 3)
        rr = np.arange(r - s, r - s + a)
        cc = np.arange(c - s, c - s + a)
        inside = ((rr >= 0) & (rr < h))[:, None] & ((cc >= 0) & (cc < wd))[None, :]
        other = int(masks[i].sum()) - int(a * a - inside.sum()) - case.mb * case.mb
        keys.append((sides, other // (case.mb * case.mb // 4)))
    return keys


def frame_batch(cid: int, picks: int, procs: int, name=None, selections_only=False):
    w = wl.WORKLOADS[cid]
    case = wl.frame_case(w)
    signals, masks = wl.frame_areas(case.damaged(), case.lost, case.corners, case.mb, case.support)
    keys = block_classes(case, masks)
    by_class = {}
    for i, k in enumerate(keys):
        by_class.setdefault(k, []).append(i)
    chosen = []
    for rnd in range(3):  # one block of every class, then a second, then a third
        chosen += [v[rnd] for v in by_class.values() if len(v) > rnd]
    chosen = chosen[:picks] if picks < len(keys) else list(range(len(keys)))
    taken = set(chosen)
    rest = [i for i in range(len(keys)) if i not in taken]
    need = min(picks, len(keys)) - len(chosen)
    if need > 0:
        chosen += [rest[j] for j in np.linspace(0, len(rest) - 1, need).astype(int)]
    blocks = sorted(set(chosen))
    m, n = w.area
    d = ref_dictionary(w.dict_spec, m, n)
    cfg = fase.ExtrapConfig(w.config.iterations, w.config.gamma, w.config.rho_hat)
    _G.update(d=d, cfg=cfg, tables=None)
    t0 = time.time()
    res = _run([(i, signals[b], masks[b]) for i, b in enumerate(blocks)], procs)
    rec = _pack(name or f"c{cid}", blocks, res, {"n_blocks": np.int64(len(masks)),
                                                 "classes": np.asarray([keys[b] for b in blocks],
                                                                       dtype=np.int32)},
                selections_only)
    rec.update(seconds=time.time() - t0, classes=len(set(keys)),
               classes_covered=len({keys[b] for b in blocks}))
    _G.clear()
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--procs", type=int, default=mp.cpu_count())
    ap.add_argument("--only", default="c1,c4,c3,c2,dft1,c4all,c2all")
    args = ap.parse_args()
    todo = args.only.split(",")
    meta_path = HERE / "batch_golden.json"
    meta = json.loads(meta_path.read_text()) if meta_path.exists() else {}
    meta.update(generator="tests/golden/make_batch_golden.py",
                reference="/root/reference/pkg (fase 0.1.0, unmodified)",
                numpy=np.__version__, tie_rel=TIE_REL)
    if "c1" in todo:
        meta["c1"] = shared_batch(1, wl.WORKLOADS[1].n_blocks, args.procs)
        print("c1", meta["c1"], flush=True)
    if "c4" in todo:
        meta["c4"] = shared_batch(4, 256, args.procs)
        print("c4", meta["c4"], flush=True)
    if "c3" in todo:
        meta["c3"] = frame_batch(3, 256, args.procs)
        print("c3", meta["c3"], flush=True)
    if "c2" in todo:
        meta["c2"] = frame_batch(2, 128, args.procs)
        print("c2", meta["c2"], flush=True)
    if "c4all" in todo:  # every block of the config-4 batch: selections + near-tie sets
        meta["c4all"] = shared_batch(4, wl.WORKLOADS[4].n_blocks, args.procs, name="c4all",
                                     selections_only=True)
        print("c4all", meta["c4all"], flush=True)
    for cid, key in ((2, "c2all"), (3, "c3all")):  # every frame block: selections + ties
        if key in todo:
            meta[key] = frame_batch(cid, 10 ** 9, args.procs, name=key, selections_only=True)
            print(key, meta[key], flush=True)
    if "dft1" in todo:  # the reference's default dictionary on the config-1 batch
        meta["dft1"] = shared_batch(1, 256, args.procs, spec="dft", name="dft1")
        print("dft1", meta["dft1"], flush=True)
    meta_path.write_text(json.dumps(meta, indent=1))


if __name__ == "__main__":
    main()
