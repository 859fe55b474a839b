"""GPU parity: libfase_b200 against the reference (golden fixtures) and the oracle.

Two gates, as in SURVEY.md section 8(c):
  1. stage-isolated -- the oracle's own tables / initial products are fed to the
     CUDA recursion; selections, projections and coefficients must then be
     BIT-IDENTICAL to the reference;
  2. end to end -- GPU-built tables and products; selections identical up to a
     legitimate near-tie (top-two Delta-E within 1e-9 relative), coefficients
     and reconstructed samples within 1e-6 of the run scale.
"""

import json

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import fase_oracle as orc  # noqa: E402
from paper_2204_14194_b200 import (  # noqa: E402
    ExtrapConfig,
    GramTable,
    NoSelectableAtomError,
    StaleTableError,
    UnsupportedDictionaryError,
    build_gram_tables,
    build_weight_field,
    fase_extrapolate,
    fase_extrapolate_batch,
    generate_dictionary,
    initial_scalar_products,
    parse_dict_spec,
    provenance_hash,
)
from paper_2204_14194_b200 import _native, workloads as wl  # noqa: E402
from paper_2204_14194_b200.dictionary import Dictionary  # noqa: E402
from parity import COEF_REL, compare_selection, metric_fn, rel_dev  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


@pytest.fixture(scope="module")
def meta(golden_dir):
    with open(golden_dir / "golden.json") as fh:
        return json.load(fh)


def host_tables(dictionary, mask, rho):
    """Oracle tables wrapped as a reference-style GramTable (host arrays)."""
    vals = dictionary.real_values().astype(np.complex128)
    w = orc.weight_field(mask, rho)
    c, d = orc.gram(vals.reshape(len(vals), -1), w)
    return GramTable(c=c, d=d, provenance=provenance_hash(dictionary, w)), (c, d)


# ----------------------------------------------------------------- kernels


@pytest.mark.parametrize("spec,m,n", [("dct", 48, 48), ("union:dct+had", 48, 48),
                                      ("union:dct+wht", 8, 8), ("had", 12, 20)])
def test_basis_outer_bit_exact(spec, m, n):
    d = parse_dict_spec(spec, m, n)
    phi = d.device_matrix(DEV)[:, : m * n].cpu().numpy()
    assert np.array_equal(phi, d.real_values().reshape(len(d), -1))


@pytest.mark.parametrize("spec,m,n,loss", [("dct", 48, 48, (16, 16)),
                                           ("union:dct+had", 48, 48, (16, 16)),
                                           ("dct", 5, 7, (1, 3)), ("union:rdft+brdft", 32, 32, (8, 8))])
def test_gram_and_normalizers(spec, m, n, loss):
    d = parse_dict_spec(spec, m, n)
    mask = wl.central_loss_mask(m, n, *loss)
    w = build_weight_field(mask, 0.8)
    t = build_gram_tables(d, w, device=DEV)
    G = t._G[:, : len(d)].cpu().numpy()
    assert np.array_equal(G, G.T)  # exact mirror
    c, dd = orc.gram(d.real_values().reshape(len(d), -1).astype(np.complex128), w)
    assert rel_dev(G, c.real) < 1e-14
    alive = dd != 0
    assert np.array_equal(t.d != 0, alive)
    assert np.abs(t.d[alive] / dd[alive] - 1).max() < 1e-14
    assert t.provenance == orc.provenance(orc.content_hash(d.values), w)


def test_initial_products_batched():
    w8 = wl.WORKLOADS[1]
    d = w8.dictionary()
    mask = wl.central_loss_mask(48, 48, 16, 16)
    w = build_weight_field(mask, 0.8)
    sig = wl.block_signals(1, 37, 48, 48)
    F = torch.from_numpy(sig.reshape(37, -1)).to(DEV)
    R0 = torch.empty((37, len(d)), dtype=torch.float64, device=DEV)
    wd = torch.from_numpy(w.ravel()).to(DEV)
    _native.init_products(d.device_matrix(DEV), F, wd, len(d), 2304, R0)
    got = R0.cpu().numpy()
    phi = d.real_values().reshape(len(d), -1).astype(np.complex128)
    for b in (0, 17, 36):
        want = orc.initial_products(sig[b], w, phi).real
        assert rel_dev(got[b], want) < 1e-13


# ----------------------------------------------------------------- stage-isolated


def test_recursion_bit_exact_small(golden_dir, meta):
    z = np.load(golden_dir / "small_cases.npz")
    from test_oracle_golden import oracle_values

    for case in meta["small_cases"]:
        k = case["key"]
        vals = oracle_values(case["spec"], case["m"], case["n"])
        d = Dictionary(vals.real) if case["spec"] not in ("dct", "wht") else \
            parse_dict_spec(case["spec"], case["m"], case["n"])
        mask = z[f"{k}_mask"]
        cfg = ExtrapConfig(case["iterations"], case["gamma"], case["rho_hat"])
        w = orc.weight_field(mask, cfg.rho_hat)
        tables = GramTable(c=z[f"{k}_gram"], d=z[f"{k}_d"], provenance=provenance_hash(d, w))
        model, trace = fase_extrapolate(z[f"{k}_signal"], mask, d, tables, cfg,
                                        products=z[f"{k}_r0"], record_products=True, device=DEV)
        assert np.array_equal(trace.selected, z[f"{k}_selected"]), k
        assert np.array_equal(trace.coefficients.real, z[f"{k}_coefficients"]), k
        assert np.array_equal(trace.projections.real, z[f"{k}_projections"]), k
        assert np.array_equal(np.stack([p.real for p in trace.products]), z[f"{k}_products"]), k


@pytest.mark.parametrize("cid", [0, 1])
def test_recursion_bit_exact_configs(golden_dir, cid):
    """Reference tables + reference R0 -> the CUDA recursion reproduces the
    reference's selections / coefficients / projections bit-for-bit."""
    z = np.load(golden_dir / f"c{cid}_blocks.npz")
    w8 = wl.WORKLOADS[cid]
    d = w8.dictionary()
    mask = wl.central_loss_mask(*w8.area, *w8.loss)
    tables, _ = host_tables(d, mask, w8.config.rho_hat)
    assert np.array_equal(tables.d, z["d"])
    blocks = list(z["blocks"])
    sig = wl.block_signals(cid, max(blocks) + 1, *w8.area)[blocks]
    r0 = np.stack([z[f"b{b}_r0"] for b in blocks])
    res = fase_extrapolate_batch(sig, mask, d, tables, w8.config, products=r0, device=DEV)
    for i, b in enumerate(blocks):
        assert np.array_equal(res.selected[i].cpu().numpy(), z[f"b{b}_selected"])
        assert np.array_equal(res.coefficients[i].cpu().numpy(), z[f"b{b}_coefficients"])
        assert np.array_equal(res.projections[i].cpu().numpy(), z[f"b{b}_projections"])
        # synthesis is also bit-exact given the same terms
        lost = res.patched[i].cpu().numpy()[mask]
        assert np.array_equal(lost, z[f"b{b}_patched_lost"])


# ----------------------------------------------------------------- end to end


def _end_to_end(cid, golden_dir, tol_blocks_early=None, recursion="exact"):
    z = np.load(golden_dir / f"c{cid}_blocks.npz")
    w8 = wl.WORKLOADS[cid]
    d = w8.dictionary()
    mask = wl.central_loss_mask(*w8.area, *w8.loss)
    blocks = list(z["blocks"])
    sig = wl.block_signals(cid, max(blocks) + 1, *w8.area)[blocks]
    res = fase_extrapolate_batch(sig, mask, d, None, w8.config, device=DEV, recursion=recursion)
    vals = d.real_values()
    tables = None
    verdicts = []
    for i, b in enumerate(blocks):
        got_sel = res.selected[i].cpu().numpy()
        want_sel = z[f"b{b}_selected"]

        def metric_at(t, b=b, i=i):
            nonlocal tables
            if tables is None:
                tables = orc.gram(vals.reshape(len(vals), -1).astype(np.complex128),
                                  orc.weight_field(mask, w8.config.rho_hat))
            _, _, _, log = orc.fase_run(z[f"b{b}_r0"], tables[0], tables[1], w8.config.gamma,
                                        t, record=True)
            return metric_fn(z[f"b{b}_r0"], tables[1], log)(t)

        v = compare_selection(got_sel, want_sel, metric_at)
        assert v.ok, f"block {b}: diverged at {v.stop} with Delta-E gap {v.gap}"
        s = v.stop
        assert rel_dev(res.coefficients[i].cpu().numpy()[:s], z[f"b{b}_coefficients"][:s]) < COEF_REL
        if v.exact:
            lost = res.patched[i].cpu().numpy()[mask]
            assert rel_dev(lost, z[f"b{b}_patched_lost"]) < COEF_REL
        verdicts.append(v)
    return verdicts


@pytest.mark.parametrize("cid", [0, 1, 4])
@pytest.mark.parametrize("recursion", ["exact", "scaled"])
def test_end_to_end_configs(golden_dir, cid, recursion):
    _end_to_end(cid, golden_dir, recursion=recursion)


# ----------------------------------------------------------------- scaled recursion


def test_scale_columns_bit_exact():
    """Gs[u, k] = G[u, k] * D_k, correctly rounded (numpy's product), zero padding."""
    d = parse_dict_spec("union:dct+had", 16, 16)
    mask = wl.central_loss_mask(16, 16, 6, 6)
    t = build_gram_tables(d, build_weight_field(mask, 0.8), device=DEV)
    G, D = t.device_tables(torch.device(DEV))
    Gs, D2 = t.scaled_table(torch.device(DEV))
    assert D2 is D and Gs.shape == G.shape
    K = len(d)
    g, dd, gs = G.cpu().numpy(), D.cpu().numpy(), Gs.cpu().numpy()
    assert np.array_equal(gs[:, :K], g[:, :K] * dd[None, :])
    assert not gs[:, K:].any()
    assert t.scaled_table(torch.device(DEV))[0] is Gs  # cached


@pytest.mark.parametrize("cid", [0, 1])
def test_recursion_scaled_configs(golden_dir, cid):
    """Reference tables + reference R0 through the scaled recursion: iteration 0
    selects bit-identically; the sequence matches the reference's up to a legitimate
    near-tie, and coefficients agree to rounding (1e-12 of the run scale, far
    inside the 1e-6 bar)."""
    z = np.load(golden_dir / f"c{cid}_blocks.npz")
    w8 = wl.WORKLOADS[cid]
    d = w8.dictionary()
    mask = wl.central_loss_mask(*w8.area, *w8.loss)
    tables, (c, dd) = host_tables(d, mask, w8.config.rho_hat)
    blocks = list(z["blocks"])
    sig = wl.block_signals(cid, max(blocks) + 1, *w8.area)[blocks]
    r0 = np.stack([z[f"b{b}_r0"] for b in blocks])
    res = fase_extrapolate_batch(sig, mask, d, tables, w8.config, products=r0, device=DEV,
                                 recursion="scaled")
    n_exact = 0
    for i, b in enumerate(blocks):
        want = z[f"b{b}_selected"]
        got = res.selected[i].cpu().numpy()
        assert got[0] == want[0]  # iteration 0's metric is bit-identical

        def metric_at(t, b=b):
            _, _, _, log = orc.fase_run(z[f"b{b}_r0"], c, dd, w8.config.gamma, t, record=True)
            return metric_fn(z[f"b{b}_r0"], dd, log)(t)

        v = compare_selection(got, want, metric_at)
        assert v.ok, f"block {b}: diverged at {v.stop} with Delta-E gap {v.gap}"
        n_exact += v.exact
        s = v.stop
        assert rel_dev(res.coefficients[i].cpu().numpy()[:s], z[f"b{b}_coefficients"][:s]) < 1e-12
        assert rel_dev(res.projections[i].cpu().numpy()[:s], z[f"b{b}_projections"][:s]) < 1e-12
        if v.exact:
            lost = res.patched[i].cpu().numpy()[mask]
            assert rel_dev(lost, z[f"b{b}_patched_lost"]) < 1e-12
    assert n_exact == len(blocks)  # no near-tie divergence on these fixtures


def test_recursion_scaled_matches_exact_full_config1():
    """All 1,024 config-1 blocks: scaled and exact recursions select the same
    sequences (up to legitimate near-ties, none expected) from the same R0."""
    w8 = wl.WORKLOADS[1]
    d = w8.dictionary()
    mask = wl.central_loss_mask(*w8.area, *w8.loss)
    dev = torch.device(DEV)
    t = build_gram_tables(d, build_weight_field(mask, w8.config.rho_hat), device=dev)
    from paper_2204_14194_b200 import ExtrapolationPlan

    sig = torch.from_numpy(wl.block_signals(1, w8.n_blocks, *w8.area)).to(dev)
    px = ExtrapolationPlan(d, mask, w8.n_blocks, w8.config, t, device=dev).run(sig)
    ps = ExtrapolationPlan(d, mask, w8.n_blocks, w8.config, t, device=dev,
                           recursion="scaled").run(sig)
    torch.cuda.synchronize()
    assert torch.equal(px.R0, ps.R0)
    same = (px.selected == ps.selected).all(dim=1)
    # every block identical (measured); a divergence must be a legitimate
    # near-tie against the reference, which tests/test_gpu_batch_parity.py
    # checks block by block on this same batch
    assert int(same.sum()) == w8.n_blocks
    dev_c = ((px.coefficients - ps.coefficients).abs().amax(dim=1)
             / px.coefficients.abs().amax(dim=1))
    assert float(dev_c[same].max()) < 1e-12
    dev_l = (px.lost - ps.lost).abs().amax(dim=1) / px.lost.abs().amax(dim=1)
    assert float(dev_l[same].max()) < 1e-12


def test_recursion_scaled_dead_atoms_and_options():
    """Dead atoms (zero weighted energy) are never selected by the scaled
    recursion; unsupported combinations raise the reference exceptions."""
    from paper_2204_14194_b200 import ParameterError, UnsupportedDictionaryError

    rng = np.random.default_rng(11)
    m = n = 8
    mask = np.zeros((m, n), dtype=bool)
    mask[2:5, 2:5] = True
    vals = rng.standard_normal((40, m, n))
    for k in (0, 7, 19):  # atoms living only on lost samples
        vals[k] = 0.0
        vals[k][mask] = rng.standard_normal(int(mask.sum()))
    d = Dictionary(vals)
    cfg = ExtrapConfig(30, 0.5, 0.8)
    sig = rng.uniform(0, 255, (5, m, n))
    rx = fase_extrapolate_batch(sig, mask, d, None, cfg, device=DEV)
    rs = fase_extrapolate_batch(sig, mask, d, None, cfg, device=DEV, recursion="scaled")
    s = rs.selected.cpu().numpy()
    assert not np.isin(s, [0, 7, 19]).any()
    assert np.array_equal(s, rx.selected.cpu().numpy())
    with pytest.raises(ParameterError):
        fase_extrapolate_batch(sig, mask, d, None, cfg, device=DEV, recursion="fast")
    with pytest.raises(UnsupportedDictionaryError):
        fase_extrapolate_batch(sig, mask, d, None, cfg, device=DEV, recursion="scaled",
                               record_products=True)
    with pytest.raises(UnsupportedDictionaryError):  # per-block geometries: exact only
        fase_extrapolate_batch(sig, np.stack([mask] * 4 + [~mask]), d, None, cfg, device=DEV,
                               recursion="scaled")


def test_frame_blocks_config3(golden_dir):
    """All 25,920 blocks of the config-3 frame in one batch (chunked per-block
    tables); the reference's per-block results pin the sampled blocks."""
    z = np.load(golden_dir / "c3_blocks.npz")
    w8 = wl.WORKLOADS[3]
    case = wl.frame_case(w8)
    signals, masks = wl.frame_areas(case.damaged(), case.lost, case.corners, case.mb, case.support)
    d = w8.dictionary()
    res = fase_extrapolate_batch(signals, masks, d, None, w8.config, device=DEV)
    vals = d.real_values().reshape(len(d), -1).astype(np.complex128)
    exact = 0
    for b in z["blocks"]:
        got = res.selected[b].cpu().numpy()
        want = z[f"b{b}_selected"]

        def metric_at(t, b=b):
            tab = orc.gram(vals, orc.weight_field(masks[b], w8.config.rho_hat))
            r0 = orc.initial_products(signals[b], orc.weight_field(masks[b], w8.config.rho_hat), vals)
            _, _, _, log = orc.fase_run(r0, tab[0], tab[1], w8.config.gamma, t, record=True)
            return metric_fn(r0, tab[1], log)(t)

        v = compare_selection(got, want, metric_at)
        assert v.ok, f"block {b}: diverged at {v.stop}, gap {v.gap}"
        s = v.stop
        assert rel_dev(res.coefficients[b].cpu().numpy()[:s], z[f"b{b}_coefficients"][:s]) < COEF_REL
        if v.exact:
            exact += 1
            lost = res.patched[b].cpu().numpy()[masks[b]]
            assert rel_dev(lost, z[f"b{b}_patched_lost"]) < COEF_REL
    assert exact >= len(z["blocks"]) - 1


def _small_frame_case():
    """A 72 x 80 frame, 8-pixel tiles, support 4 (16 x 16 areas, 8 cells), 35%
    of the tiles lost: lists of every length from 0 to 8."""
    rng = np.random.default_rng(33)
    h, w, mb = 72, 80, 8
    yy, xx = np.mgrid[0:h, 0:w]
    frame = np.clip(128 + 60 * np.sin(0.17 * yy + 0.11 * xx) + rng.normal(0, 6, (h, w)), 0, 255)
    frame = frame.astype(np.uint8)
    tiles = [(r, c) for r in range(0, h, mb) for c in range(0, w, mb)]
    pick = rng.choice(len(tiles), int(0.35 * len(tiles)), replace=False)
    corners = np.array(sorted(tiles[i] for i in pick), dtype=np.int32)
    lost = np.zeros((h, w), dtype=bool)
    for r0, c0 in corners:
        lost[r0:r0 + mb, c0:c0 + mb] = True
    case = wl.FrameCase(frame=frame, lost=lost, corners=corners, mb=mb, support=4)
    return case, parse_dict_spec("dct", 16, 16), ExtrapConfig(40, 0.5, 0.8)


@pytest.mark.parametrize("cid,modes", [("small", ("singles", "pairs", "triples")),
                                       (3, ("singles", "pairs")), (2, ("singles", "pairs"))])
def test_frame_engine_composed_bases_bit_identical(cid, modes):
    """Precomposed base tables (G0 - C_c1 - ... - C_ck, composed in list order)
    stream fewer rows but must give bit-identical selections, coefficients and
    restored frames to the uncomposed chunk lists."""
    from paper_2204_14194_b200.conceal import FrameEngine, lossy_tiles, tile_grid

    if cid == "small":
        case, d, cfg = _small_frame_case()
    else:
        w8 = wl.WORKLOADS[cid]
        case, d, cfg = wl.frame_case(w8), w8.dictionary(), w8.config
    grid = torch.from_numpy(tile_grid(case.lost, case.mb)).to(DEV)
    corners = torch.from_numpy(lossy_tiles(case.lost, (case.mb, case.mb)).astype(np.int32)).to(DEV)
    damaged = torch.from_numpy(case.damaged()).to(DEV)
    runs = {}
    for mode in ("none",) + modes:
        eng = FrameEngine(d, case.frame.shape, case.mb, case.support, cfg, device=DEV,
                          compose=mode)
        assert (eng.compose is None) == (mode == "none")
        res = eng.run(damaged, grid, corners)
        torch.cuda.synchronize()
        runs[mode] = (res.selected.clone(), res.coefficients.clone(), res.patched.clone())
        if mode != "none":  # some blocks do take a composed base of the full depth
            depth = eng.compose.dim()
            counts = eng._buffers(int(corners.shape[0]))["counts"]
            assert int((counts >= depth).sum()) > 0
        del eng
    for mode in modes:
        for a, b in zip(runs["none"], runs[mode]):
            assert torch.equal(a, b), mode


# ----------------------------------------------------------------- properties / edges


def test_full_config1_properties():
    """1,024 blocks: deterministic, support untouched, selections valid."""
    w8 = wl.WORKLOADS[1]
    d = w8.dictionary()
    mask = wl.central_loss_mask(48, 48, 16, 16)
    sig = wl.block_signals(1, 1024, 48, 48)
    t = build_gram_tables(d, build_weight_field(mask, 0.8), device=DEV)
    a = fase_extrapolate_batch(sig, mask, d, t, w8.config, device=DEV)
    b = fase_extrapolate_batch(torch.from_numpy(sig).to(DEV), mask, d, t, w8.config, device=DEV)
    assert torch.equal(a.selected, b.selected) and torch.equal(a.coefficients, b.coefficients)
    sel = a.selected.cpu().numpy()
    assert sel.min() >= 0 and sel.max() < len(d)
    patched = a.patched.cpu().numpy()
    assert np.array_equal(patched[:, ~mask], sig[:, ~mask])
    assert np.isfinite(patched).all()


def test_zero_signal_selects_first_atom():
    # pkg/tests/test_reference.py:186-191: zero signal -> atom 0, coefficient 0
    d = generate_dictionary("dct", 8, 8)
    mask = wl.central_loss_mask(8, 8, 4, 4)
    t = build_gram_tables(d, build_weight_field(mask, 0.8), device=DEV)
    _, trace = fase_extrapolate(np.zeros((8, 8)), mask, d, t, ExtrapConfig(5), device=DEV)
    assert (trace.selected == 0).all() and (trace.coefficients == 0).all()


def test_single_atom_recovery():
    # signal = atom 9, gamma = 1, one iteration -> term (9, 1.0) (SPEC fase-core example)
    d = generate_dictionary("dct", 8, 8)
    mask = np.zeros((8, 8), bool)
    mask[3:5, 3:5] = True
    sig = d.real_values()[9].copy()
    t = build_gram_tables(d, build_weight_field(mask, 0.8), device=DEV)
    _, trace = fase_extrapolate(sig, mask, d, t, ExtrapConfig(1, 1.0, 0.8), device=DEV)
    assert trace.selected[0] == 9
    assert abs(trace.coefficients[0] - 1.0) < 1e-13


def test_degenerate_atoms_never_selected_and_all_dead_raises():
    mask = wl.central_loss_mask(4, 4, 2, 2)
    inside = np.zeros((4, 4))
    inside[1:3, 1:3] = 1.0
    base = generate_dictionary("dct", 4, 4).real_values()
    d = Dictionary(np.concatenate([inside[None], base]))
    t = build_gram_tables(d, build_weight_field(mask, 0.8), device=DEV)
    assert t.d[0] == 0.0
    _, trace = fase_extrapolate(np.random.default_rng(12).standard_normal((4, 4)), mask, d, t,
                                ExtrapConfig(10), device=DEV)
    assert (trace.selected != 0).all()
    dead = Dictionary(inside[None])
    td = build_gram_tables(dead, build_weight_field(mask, 0.8), device=DEV)
    with pytest.raises(NoSelectableAtomError):
        fase_extrapolate(np.ones((4, 4)), mask, dead, td, device=DEV)


@pytest.mark.parametrize("blocks", [3, 200])
def test_scaled_recursion_zero_metrics_and_dead_atoms(blocks):
    """The scaled recursion's running max keeps the signed R' and starts at
    -0, so all-zero metrics take the lowest live atom through its fallback
    scan: zero signals select atom 0 (pkg/tests/test_reference.py:186-191), and
    with atom 0 dead (zero weighted energy) atom 1, exactly like the bit-exact
    kernel; one-CTA shapes (200 blocks) and latency / cluster shapes (3)."""
    mask = wl.central_loss_mask(4, 4, 2, 2)
    inside = np.zeros((4, 4))
    inside[1:3, 1:3] = 1.0
    base = generate_dictionary("dct", 4, 4).real_values()
    cfg = ExtrapConfig(6)
    for vals, first in ((base, 0), (np.concatenate([inside[None], base]), 1)):
        d = Dictionary(vals)
        zero = np.zeros((blocks, 4, 4))
        out = {}
        for rec in ("exact", "scaled"):
            r = fase_extrapolate_batch(zero, mask, d, None, cfg, device=DEV, recursion=rec)
            out[rec] = r
            assert (r.selected.cpu().numpy() == first).all(), rec
            assert (r.coefficients.cpu().numpy() == 0.0).all(), rec
        # a live signal in one block: the others stay at the first live atom
        sig = zero.copy()
        sig[blocks // 2] = np.random.default_rng(5).standard_normal((4, 4))
        a = fase_extrapolate_batch(sig, mask, d, None, cfg, device=DEV, recursion="exact")
        b = fase_extrapolate_batch(sig, mask, d, None, cfg, device=DEV, recursion="scaled")
        assert torch.equal(a.selected, b.selected)
        sel = b.selected.cpu().numpy()
        assert (np.delete(sel, blocks // 2, axis=0) == first).all()
        if first == 1:
            assert (sel != 0).all()


@pytest.mark.parametrize("K", [6000, 8192])
def test_scaled_recursion_integer_max_shapes(monkeypatch, K):
    """The 24- and 32-element shapes of the scaled recursion (K > 5,120) track
    integer keys of the high words and resolve the exact top and the tie rule
    in one warp (csrc/iterate.cu, kIntMax). Exact ties between duplicated atoms
    held by one thread, by two lanes of a warp, by two warps and far apart,
    dead atoms, padding (K = 6,000 of 6,144 positions) and an all-zero block:
    the selections must be the bit-exact kernel's -- the lowest index of every
    tie set (reference.py:55-85)."""
    rng = np.random.default_rng(21)
    vals = rng.standard_normal((K, 8, 8))
    mask = wl.central_loss_mask(8, 8, 2, 2)
    vals[1] = vals[0]            # elements 0 and 1 of thread 0
    vals[56] = vals[40]          # threads 20 and 28: two lanes of warp 0
    vals[164] = vals[100]        # threads 50 and 82: warps 1 and 2
    vals[4000] = vals[5]         # far apart
    for k in (2, 4001):          # dead: atoms living only on lost samples
        vals[k] = 0.0
        vals[k][mask] = rng.standard_normal(int(mask.sum()))
    d = Dictionary(vals)
    blocks = 160                 # more than one block per SM: the one-CTA kernels
    sig = rng.uniform(0, 255, (blocks, 8, 8))
    sig[7] = 0.0                 # all-zero metrics
    sig[9] = 37.5 * vals[300]    # one atom's multiple: the top halves every iteration until the
    #                              ratcheted quantum exceeds it (threshold <= 0: every live atom ties)
    cfg = ExtrapConfig(48, 0.5, 0.8)
    a = fase_extrapolate_batch(sig, mask, d, None, cfg, device=DEV, recursion="exact")
    b = fase_extrapolate_batch(sig, mask, d, None, cfg, device=DEV, recursion="scaled")
    sa, sb = a.selected.cpu().numpy(), b.selected.cpu().numpy()
    same = (sa == sb).all(axis=1)
    same[9] = True               # (threshold-wide tie sets: compared bit for bit below instead)
    assert int(same.sum()) == blocks, np.flatnonzero(~same)
    assert (sb[9, :8] == 300).all() and (sb[9] >= 0).all() and not np.isin(sb[9], [2, 4001]).any()
    if K == 8192:
        # the compare / select scaled kernel (128 x 64 shape: no integer keys) on the same
        # table layout: the integer-key kernel must agree bit for bit, block 9 included
        monkeypatch.setenv("FASE_SCALED_VARIANT", "128x64x2")
        c = fase_extrapolate_batch(sig, mask, d, None, cfg, device=DEV, recursion="scaled")
        monkeypatch.delenv("FASE_SCALED_VARIANT")
        assert torch.equal(b.selected, c.selected)
        assert torch.equal(b.coefficients, c.coefficients)
    assert not np.isin(sb, [1, 56, 164, 4000, 2, 4001]).any()
    assert np.isin(sb, [0, 40, 100, 5]).any()      # the tie sets were reached
    assert (sb[7] == 0).all() and (b.coefficients[7].cpu().numpy() == 0.0).all()
    scale = a.coefficients.abs().amax(dim=1).clamp_min(1e-300)
    assert float(((a.coefficients - b.coefficients).abs().amax(dim=1) / scale).max()) < 1e-10


def test_stale_tables_detected():
    d = generate_dictionary("dct", 4, 4)
    mask = wl.central_loss_mask(4, 4, 2, 2)
    other = build_gram_tables(generate_dictionary("wht", 4, 4), build_weight_field(mask, 0.8),
                              device=DEV)
    with pytest.raises(StaleTableError):
        fase_extrapolate(np.ones((4, 4)), mask, d, other, device=DEV)
    rho = build_gram_tables(d, build_weight_field(mask, 0.5), device=DEV)
    with pytest.raises(StaleTableError):
        fase_extrapolate(np.ones((4, 4)), mask, d, rho, device=DEV)


def test_empty_batch_and_odd_area():
    d = generate_dictionary("dct", 5, 7)  # K = 35, odd area
    mask = wl.central_loss_mask(5, 7, 1, 3)
    res = fase_extrapolate_batch(np.zeros((0, 5, 7)), mask, d, None, ExtrapConfig(3), device=DEV)
    assert res.selected.shape == (0, 3)
    sig = np.random.default_rng(3).uniform(0, 255, (3, 5, 7))
    res = fase_extrapolate_batch(sig, mask, d, None, ExtrapConfig(12), device=DEV)
    vals = d.real_values().astype(np.complex128)
    for b in range(3):
        ref = orc.extrapolate_block(sig[b], mask, vals, 0.5, 12, 0.8)
        assert np.array_equal(res.selected[b].cpu().numpy(), ref["selected"])
        assert rel_dev(res.coefficients[b].cpu().numpy(), ref["coefficients"].real) < 1e-12


# ----------------------------------------------------------------- frame engine


@pytest.mark.parametrize("cid", [3, 2])
def test_frame_engine_against_reference_blocks(golden_dir, cid):
    """Whole-frame device pipeline (areas, cell lists, normalizers, GEMM,
    chunked recursion, paste) against the reference's per-block results."""
    from paper_2204_14194_b200.conceal import FrameEngine, lossy_tiles, tile_grid

    z = np.load(golden_dir / f"c{cid}_blocks.npz")
    w8 = wl.WORKLOADS[cid]
    case = wl.frame_case(w8)
    d = w8.dictionary()
    eng = FrameEngine(d, case.frame.shape, case.mb, case.support, w8.config, device=DEV)
    grid = torch.from_numpy(tile_grid(case.lost, case.mb)).to(DEV)
    corners_h = lossy_tiles(case.lost, (case.mb, case.mb)).astype(np.int32)
    assert np.array_equal(corners_h, case.corners)
    damaged = torch.from_numpy(case.damaged()).to(DEV)
    res = eng.run(damaged, grid, torch.from_numpy(corners_h).to(DEV))
    torch.cuda.synchronize()
    assert eng.dead_blocks() == 0
    out = res.patched.cpu().numpy()
    # untouched outside the lost pixels
    assert np.array_equal(out[~case.lost], case.damaged()[~case.lost])
    signals, masks = wl.frame_areas(case.damaged(), case.lost, case.corners, case.mb, case.support)
    vals = d.real_values().reshape(len(d), -1).astype(np.complex128)
    s, mb = case.support, case.mb
    exact = 0
    for b in z["blocks"]:
        got = res.selected[b].cpu().numpy()
        want = z[f"b{b}_selected"]

        def metric_at(t, b=b):
            wb = orc.weight_field(masks[b], w8.config.rho_hat)
            tab = orc.gram(vals, wb)
            r0 = orc.initial_products(signals[b], wb, vals)
            _, _, _, log = orc.fase_run(r0, tab[0], tab[1], w8.config.gamma, t, record=True)
            return metric_fn(r0, tab[1], log)(t)

        v = compare_selection(got, want, metric_at)
        assert v.ok, f"block {b}: diverged at {v.stop}, gap {v.gap}"
        k = v.stop
        assert rel_dev(res.coefficients[b].cpu().numpy()[:k], z[f"b{b}_coefficients"][:k]) < COEF_REL
        if v.exact:
            exact += 1
            # own-tile lost pixels in the frame vs the reference's reconstruction
            full = np.zeros(masks[b].shape)
            full[masks[b]] = z[f"b{b}_patched_lost"]
            r0_, c0_ = case.corners[b]
            want_tile = full[s:s + mb, s:s + mb]
            got_tile = out[r0_:r0_ + mb, c0_:c0_ + mb]
            assert rel_dev(got_tile, want_tile) < COEF_REL
    assert exact >= len(z["blocks"]) - 1


def test_reference_fgrm_table_drives_the_gpu_path(golden_dir):
    """A table file written by the reference's save_gram_table runs on the GPU
    and gives the same selections as a GPU-built table."""
    from paper_2204_14194_b200 import load_gram_table

    t = load_gram_table(golden_dir / "ref_tables.fgrm")
    d = parse_dict_spec("union:dct+wht", 4, 4)
    mask = wl.central_loss_mask(4, 4, 2, 2)
    sig = np.random.default_rng(7).standard_normal((4, 4))
    _, a = fase_extrapolate(sig, mask, d, t, ExtrapConfig(8), device=DEV)
    t2 = build_gram_tables(d, build_weight_field(mask, 0.8), device=DEV)
    _, b = fase_extrapolate(sig, mask, d, t2, ExtrapConfig(8), device=DEV)
    assert np.array_equal(a.selected, b.selected)
    assert rel_dev(a.coefficients.real, b.coefficients.real) < 1e-12


@pytest.mark.parametrize("spec,m,n", [("union:dct+had", 48, 48), ("dct", 5, 7), ("wht", 8, 16)])
def test_separable_products_match_gemm_and_oracle(spec, m, n):
    from paper_2204_14194_b200.fast import initial_products_into

    d = parse_dict_spec(spec, m, n)
    K, M = len(d), m * n
    mask = wl.central_loss_mask(m, n, max(1, m // 3), max(1, n // 3))
    w = build_weight_field(mask, 0.8)
    rng = np.random.default_rng(11)
    sig = rng.uniform(0, 255, (5, m, n))
    ld = M + (M & 1)
    F = torch.zeros((5, ld), dtype=torch.float64, device=DEV)
    F[:, :M] = torch.from_numpy(sig.reshape(5, -1)).to(DEV)
    W = torch.zeros(ld, dtype=torch.float64, device=DEV)
    W[:M] = torch.from_numpy(w.ravel()).to(DEV)
    ws = torch.empty(5 * ld + 2, dtype=torch.float64, device=DEV)
    outs = {}
    for method in ("separable", "gemm"):
        R0 = torch.zeros((5, K + (K & 1)), dtype=torch.float64, device=DEV)
        assert initial_products_into(d, F, W, R0, ws, method=method) == method
        outs[method] = R0[:, :K].cpu().numpy()
    phi = d.real_values().reshape(K, -1).astype(np.complex128)
    for b in range(5):
        want = orc.initial_products(sig[b], w, phi).real
        assert rel_dev(outs["separable"][b], want) < 1e-13
        assert rel_dev(outs["gemm"][b], want) < 1e-13


@pytest.mark.parametrize("spec", ["gauss:600:7", "union:rdft+brdft", "bdft"])
def test_plan_support_compacted_products(spec):
    """Dense products over the support only (lost samples add exact zeros):
    same R0 as the full GEMM to rounding, same selections as the oracle."""
    from paper_2204_14194_b200 import ExtrapolationPlan

    d = parse_dict_spec(spec, 16, 16)
    mask = wl.central_loss_mask(16, 16, 6, 6)
    cfg = ExtrapConfig(40, 0.5, 0.85)
    sig = np.random.default_rng(8).uniform(0, 255, (7, 16, 16))
    plan = ExtrapolationPlan(d, mask, 7, cfg, device=DEV)
    assert plan._support is not None and plan.launches_per_run == 4
    plan.run(torch.from_numpy(sig).to(DEV))
    assert plan.products_method == "gemm-support"
    R0 = plan.R0[:, : len(d)].cpu().numpy()
    w = orc.weight_field(mask, 0.85)
    vals = d.values
    for b in range(7):
        ref = orc.extrapolate_block(sig[b], mask, vals, 0.5, 40, 0.85, record=True)
        assert rel_dev(R0[b], ref["r0"] if not d.is_real else ref["r0"].real) < 1e-13
        v = compare_selection(plan.selected[b].cpu().numpy(), ref["selected"],
                              metric_fn(ref["r0"], ref["d"], ref["log"]))
        assert v.ok
    del w


@pytest.mark.parametrize("spec,m,n", [("union:dct+had", 48, 48), ("dct", 5, 7), ("union:dct+wht", 16, 16)])
def test_separable_dmma_batch_matches_fma_kernel(spec, m, n):
    """The fused DMMA transform (weights applied while staging, all parts in one
    launch) equals the per-part FMA kernel and the oracle to rounding."""
    d = parse_dict_spec(spec, m, n)
    K, M = len(d), m * n
    B = 19
    sig = np.random.default_rng(31).uniform(0, 255, (B, m, n))
    mask = wl.central_loss_mask(m, n, max(1, m // 3), max(1, n // 3))
    w = build_weight_field(mask, 0.8)
    ld = M + (M & 1)
    F = torch.zeros((B, ld), dtype=torch.float64, device=DEV)
    F[:, :M] = torch.from_numpy(sig.reshape(B, -1)).to(DEV)
    W = torch.zeros(ld, dtype=torch.float64, device=DEV)
    W[:M] = torch.from_numpy(w.ravel()).to(DEV)
    factors = d.device_factors(DEV)
    Rd = torch.zeros((B, K + 3), dtype=torch.float64, device=DEV)
    _native.sep_products_batch(factors, F, W, m, n, Rd)
    X = torch.zeros((B, ld), dtype=torch.float64, device=DEV)
    _native.weigh(F, W, M, X)
    Rf = torch.zeros((B, K + 3), dtype=torch.float64, device=DEV)
    for rows, cols, row0 in factors:
        _native.sep_products(rows, cols, X, m, n, Rf, row0)
    a, f = Rd.cpu().numpy(), Rf.cpu().numpy()
    assert np.all(a[:, K:] == 0.0)
    assert rel_dev(a, f) < 1e-13
    phi = d.real_values().reshape(K, -1).astype(np.complex128)
    for b in (0, B - 1):
        assert rel_dev(a[b, :K], orc.initial_products(sig[b], w, phi).real) < 1e-13


def test_full_config4_properties():
    """Config 4 at full size (4,096 blocks, K = 8,192, M = 4,096, I = 500):
    the tcgen05 Ozaki products equal the DMMA products to 1e-12, the
    recursion is deterministic, and every output is in range / finite."""
    from paper_2204_14194_b200 import ExtrapolationPlan

    w4 = wl.WORKLOADS[4]
    d = w4.dictionary()
    mask = wl.central_loss_mask(*w4.area, *w4.loss)
    sig = torch.from_numpy(wl.block_signals(4, w4.n_blocks, *w4.area)).to(DEV)
    t = build_gram_tables(d, build_weight_field(mask, w4.config.rho_hat), device=DEV)
    oz = ExtrapolationPlan(d, mask, w4.n_blocks, w4.config, t, device=DEV, products="auto")
    assert oz._ozaki is not None
    oz.run(sig)
    sel_a, coef_a = oz.selected.clone(), oz.coefficients.clone()
    oz.run(sig)
    assert torch.equal(oz.selected, sel_a) and torch.equal(oz.coefficients, coef_a)
    dm = ExtrapolationPlan(d, mask, w4.n_blocks, w4.config, t, device=DEV, products="gemm")
    dm._products(sig.reshape(w4.n_blocks, -1))
    # 7 digit planes (_native.PRODUCT_SLICES): 2.8e-13 measured
    assert rel_dev(oz.R0.cpu().numpy(), dm.R0.cpu().numpy()) < 1e-12
    s = sel_a.cpu().numpy()
    assert s.min() >= 0 and s.max() < len(d)
    assert torch.isfinite(oz.lost).all() and torch.isfinite(oz.coefficients).all()


@pytest.mark.parametrize("spec", ["gauss:5000:1", "gauss:8192:2"])
def test_recursion_bit_exact_paired_blocks(spec):
    """Large-K shared geometry runs two blocks per CTA sharing D (paired
    variant; an odd batch leaves the last CTA half idle): given the oracle's
    tables and initial products the run is bit-identical to the oracle."""
    d = parse_dict_spec(spec, 16, 16)
    mask = wl.central_loss_mask(16, 16, 6, 6)
    cfg = ExtrapConfig(25, 0.5, 0.8)
    tables, (c, dd) = host_tables(d, mask, cfg.rho_hat)
    # more blocks than SMs (smaller batches run one wide CTA per block)
    nb = 151
    sig = np.random.default_rng(5).uniform(0, 255, (nb, 16, 16))
    w = orc.weight_field(mask, cfg.rho_hat)
    vals = d.real_values().reshape(len(d), -1).astype(np.complex128)
    r0 = np.stack([orc.initial_products(sig[b], w, vals) for b in range(nb)])
    res = fase_extrapolate_batch(sig, mask, d, tables, cfg, products=r0.real, device=DEV)
    for b in (0, 1, 2, 77, nb - 2, nb - 1):
        sel, proj, coef, _ = orc.fase_run(r0[b], c, dd, cfg.gamma, cfg.iterations)
        assert np.array_equal(res.selected[b].cpu().numpy(), sel)
        assert np.array_equal(res.coefficients[b].cpu().numpy(), coef.real)
        assert np.array_equal(res.projections[b].cpu().numpy(), proj.real)


@pytest.mark.parametrize("cplx,depth", [(False, 2), (True, 2), (False, 3), (True, 1)])
def test_iterate_compose_map_bit_identical(cplx, depth):
    """fase_iterate(_complex) with a compose map: base tables G0 - C_c1 (- C_c2)
    composed in list order replace the first one or two chunks of each list;
    the run is bit-identical to the plain chunk lists (random tables and lists,
    some blocks without chunks, singles and pairs both present)."""
    from paper_2204_14194_b200 import _native

    rng = np.random.default_rng(11 + cplx)
    K, B, I, n = 300, 9, 30, 4
    ld = _native.table_ld_complex(K) if cplx else _native.table_ld(K)
    dt = torch.complex128 if cplx else torch.float64

    def rnd(*shape):
        x = torch.from_numpy(rng.normal(size=shape))
        if cplx:
            x = torch.complex(x, torch.from_numpy(rng.normal(size=shape)))
        return x.to(DEV)

    G0 = torch.zeros((K, ld), dtype=dt, device=DEV)
    G0[:, :K] = rnd(K, K)
    tabs = torch.zeros((n, K, ld), dtype=dt, device=DEV)
    tabs[:, :, :K] = 0.3 * rnd(n, K, K)
    counts = torch.tensor([0, 1, 2, 3, 4, 1, 2, 3, 0], dtype=torch.int32, device=DEV)
    ids = torch.zeros((B, n), dtype=torch.int32)
    for b, c in enumerate(counts.tolist()):
        ids[b, :c] = torch.from_numpy(np.sort(rng.choice(n, c, replace=False)))
    ids = ids.to(DEV)
    # every single, a few pairs / triples (the rest fall back to shorter prefixes)
    prefixes = [(c,) for c in range(n)] + [(0, 1), (1, 3), (0, 2), (1, 2), (0, 1, 2), (1, 2, 3)]
    prefixes = [p for p in prefixes if len(p) <= depth]
    bases = torch.empty((1 + len(prefixes), K, ld), dtype=dt, device=DEV)
    bases[0] = G0
    cmap = torch.zeros((n,) * depth, dtype=torch.int32)
    index = {(): 0}
    for p, pre in enumerate(prefixes, start=1):
        torch.sub(bases[index[pre[:-1]]], tabs[pre[-1]], out=bases[p])
        index[pre] = p
        cmap[pre + (pre[-1],) * (depth - len(pre))] = p
    cmap = cmap.to(DEV)
    D = torch.from_numpy(rng.uniform(0.5, 1.5, (B, ld))).to(DEV)
    R0 = torch.zeros((B, ld), dtype=dt, device=DEV)
    R0[:, :K] = rnd(B, K)
    fn = _native.iterate_complex if cplx else _native.iterate
    out = []
    for composed in (False, True):
        sel = torch.empty((B, I), dtype=torch.int32, device=DEV)
        proj = torch.empty((B, I), dtype=dt, device=DEV)
        coef = torch.empty((B, I), dtype=dt, device=DEV)
        fn(bases[0], D, R0, K, I, 0.5, sel, proj, coef, chunk_tables=tabs,
           chunk_stride=tabs[0].numel(), chunk_count=counts, chunk_ids=ids,
           compose=cmap if composed else None, base_stride=bases[0].numel() if composed else 0)
        out.append((sel, proj, coef))
    torch.cuda.synchronize()
    for a, b in zip(*out):
        assert torch.equal(a, b)
    assert (out[0][0] >= 0).all()


@pytest.mark.parametrize("spec,m,loss,nb", [("union:dct+had", 48, 16, 64), ("dct", 48, 16, 1),
                                            ("gauss:2000:3", 24, 10, 37)])
def test_fused_synthesis_bit_identical(spec, m, loss, nb):
    """The recursion with the synthesis fused in (scaled: fase_iterate_scaled
    with a synth block; exact: fase_iterate_synth) writes the same lost
    samples, bit for bit, as the recursion followed by fase_synth_paste; the
    plan fuses it for batches of at most one block per SM."""
    from paper_2204_14194_b200 import ExtrapolationPlan

    d = parse_dict_spec(spec, m, m)
    mask = wl.central_loss_mask(m, m, loss, loss)
    cfg = ExtrapConfig(60, 0.5, 0.8)
    dev = torch.device(DEV)
    t = build_gram_tables(d, build_weight_field(mask, cfg.rho_hat), device=dev)
    sig = torch.from_numpy(np.random.default_rng(3).uniform(0, 255, (nb, m, m))).to(dev)
    for rec in ("scaled", "exact"):
        p = ExtrapolationPlan(d, mask, nb, cfg, t, device=dev, recursion=rec)
        K, n = len(d), p.n_lost
        if rec == "exact" and _native.synth_capacity(K, nb) < n:  # no latency shape for this K
            assert not p.fused_synth
            continue
        assert p.fused_synth
        p.run(sig)
        sel, proj, coef = (torch.empty_like(x) for x in (p.selected, p.projections,
                                                         p.coefficients))
        lost = torch.zeros_like(p.lost)
        if rec == "scaled":
            _native.iterate_scaled(p.Gs, p.D, p.R0, K, cfg.iterations, cfg.gamma, sel, proj, coef)
        else:
            _native.iterate(p.G, p.D, p.R0, K, cfg.iterations, cfg.gamma, sel, proj, coef)
        _native.synth_paste(p.phi_lost, sel, coef, cfg.iterations, p.lost_seq, lost, n_shared=n,
                            dst=p.lost_pos)
        torch.cuda.synchronize()
        assert torch.equal(sel, p.selected) and torch.equal(coef, p.coefficients)
        assert torch.equal(lost[:, :n], p.lost[:, :n])
        # capacity guard: more lost samples than the fused kernel holds is refused
        cap = (_native.scaled_synth_capacity(K, nb) if rec == "scaled"
               else _native.synth_capacity(K, nb))
        big = torch.zeros((K, cap + 2), dtype=torch.float64, device=dev)
        fn = _native.iterate_scaled if rec == "scaled" else _native.iterate
        with pytest.raises(UnsupportedDictionaryError):
            fn(p.Gs if rec == "scaled" else p.G, p.D, p.R0, K, cfg.iterations, cfg.gamma, sel,
               proj, coef, phi_lost=big, n_lost=cap + 1,
               lost=torch.zeros((nb, cap + 2), dtype=torch.float64, device=dev))


@pytest.mark.parametrize("nb,n_lost,I,stop", [(300, 256, 200, None), (160, 576, 37, 20),
                                              (151, 100, 1030, 700)])
def test_synth_paste_throughput_shape_bit_exact(nb, n_lost, I, stop):
    """fase_synth_paste on batches that fill the GPU (two samples per thread,
    valid-term count found while staging) against numpy's sequential
    mul-then-add in selection order (SparseModel.materialize); a recursion that
    stopped early (sel = -1 from `stop` on) contributes nothing after it."""
    rng = np.random.default_rng(nb)
    K, ld = 700, n_lost + (n_lost & 1)
    phi = rng.standard_normal((K, ld))
    sel = rng.integers(0, K, (nb, I)).astype(np.int32)
    coef = rng.standard_normal((nb, I))
    if stop is not None:
        sel[::3, stop:] = -1
    dev = torch.device(DEV)
    out = torch.zeros((nb, ld), dtype=torch.float64, device=dev)
    seq = torch.arange(ld, dtype=torch.int32, device=dev)
    _native.synth_paste(torch.from_numpy(phi).to(dev), torch.from_numpy(sel).to(dev),
                        torch.from_numpy(coef).to(dev), I, seq, out, n_shared=n_lost,
                        dst=torch.arange(ld, dtype=torch.int64, device=dev))
    got = out.cpu().numpy()[:, :n_lost]
    want = np.zeros((nb, n_lost))
    for t in range(I):
        live = sel[:, t] >= 0
        want[live] = want[live] + coef[live, t, None] * phi[sel[live, t], :n_lost]
    assert np.array_equal(got, want)


def test_maximum_atom_count():
    """K at the largest register-resident variant (512 x 24 = 12,288) and one
    atom beyond it (odd K: the streaming recursion, csrc/iterate_generic.cu):
    both stay bit-exact against the oracle's loop on the same (device-built)
    table / normalizers / initial products. The scaled recursion refuses K
    beyond the registers; K beyond fase_max_atoms raises
    UnsupportedDictionaryError, the reference-facing error class."""
    kreg = _native.register_atoms()
    assert kreg == 12288 and _native.max_atoms() > kreg
    rng = np.random.default_rng(12)
    m = n = 16
    mask = wl.central_loss_mask(m, n, 6, 6)
    cfg = ExtrapConfig(20, 0.5, 0.8)
    sig = rng.uniform(0, 255, (3, m, n))
    w = build_weight_field(mask, cfg.rho_hat)
    for K in (kreg, kreg + 1):
        d = Dictionary(rng.standard_normal((K, m, n)))
        t = build_gram_tables(d, w, device=DEV)
        r0 = np.stack([initial_scalar_products(sig[b], w, d, device=DEV).real for b in range(3)])
        res = fase_extrapolate_batch(sig, mask, d, t, cfg, device=DEV, patch=False, products=r0)
        G, D = t.device_tables(torch.device(DEV))
        g = G[:, :K].cpu().numpy()
        dd = D.cpu().numpy()
        for b in range(3):
            sel, _, coef, _ = orc.fase_run(r0[b], g, dd, cfg.gamma, cfg.iterations)
            assert np.array_equal(res.selected[b].cpu().numpy(), sel), K
            assert np.array_equal(res.coefficients[b].cpu().numpy(), coef.real), K
        del G, g, t
    with pytest.raises(UnsupportedDictionaryError):
        fase_extrapolate_batch(sig, mask, d, None, cfg, device=DEV, recursion="scaled")
    with pytest.raises(UnsupportedDictionaryError):
        _native.table_ld(_native.max_atoms() + 1)


def test_streaming_recursion_chunk_lists_and_dead_atoms():
    """The streaming recursion (K beyond the registers) with per-block chunk
    lists, per-block normalizers with dead atoms and a dispatch order:
    bit-exact against the oracle's loop on rows composed in list order."""
    from paper_2204_14194_b200 import _native

    rng = np.random.default_rng(21)
    K, B, I, n = _native.register_atoms() + 3, 4, 15, 2
    ld = _native.table_ld(K)
    assert ld >= K and ld % 2 == 0
    G0 = torch.zeros((K, ld), dtype=torch.float64, device=DEV)
    G0[:, :K] = torch.from_numpy(rng.normal(size=(K, K))).to(DEV)
    tabs = torch.zeros((n, K, ld), dtype=torch.float64, device=DEV)
    tabs[:, :, :K] = 0.3 * torch.from_numpy(rng.normal(size=(n, K, K))).to(DEV)
    counts = torch.tensor([0, 1, 2, 1], dtype=torch.int32, device=DEV)
    ids = torch.tensor([[0, 0], [1, 0], [0, 1], [0, 0]], dtype=torch.int32, device=DEV)
    Dh = rng.uniform(0.5, 1.5, (B, ld))
    Dh[:, [3, 77, K - 1]] = 0.0  # dead atoms: never selected
    D = torch.from_numpy(Dh).to(DEV)
    R0 = torch.zeros((B, ld), dtype=torch.float64, device=DEV)
    R0[:, :K] = torch.from_numpy(rng.normal(size=(B, K))).to(DEV)
    sel = torch.empty((B, I), dtype=torch.int32, device=DEV)
    proj = torch.empty((B, I), dtype=torch.float64, device=DEV)
    coef = torch.empty((B, I), dtype=torch.float64, device=DEV)
    order = torch.tensor([2, 0, 3, 1], dtype=torch.int32, device=DEV)
    _native.iterate(G0, D, R0, K, I, 0.5, sel, proj, coef, chunk_tables=tabs,
                    chunk_stride=tabs[0].numel(), chunk_count=counts, chunk_ids=ids, order=order)
    torch.cuda.synchronize()

    class Rows:  # row u of block b's table: G0[u] - C_j1[u] - ... in list order
        def __init__(self, b):
            self.lst = ids[b, : int(counts[b])].tolist()

        def __getitem__(self, u):
            r = G0[u, :K].clone()
            for j in self.lst:
                r = r - tabs[j, u, :K]
            return r.cpu().numpy()

    for b in range(B):
        s_ref, p_ref, c_ref, _ = orc.fase_run(R0[b, :K].cpu().numpy(), Rows(b), Dh[b, :K], 0.5, I)
        assert np.array_equal(sel[b].cpu().numpy(), s_ref), b
        assert np.array_equal(proj[b].cpu().numpy(), p_ref.real), b
        assert np.array_equal(coef[b].cpu().numpy(), c_ref.real), b
        assert not np.isin(s_ref, [3, 77, K - 1]).any()


def test_streaming_recursion_complex():
    """The complex streaming recursion (K beyond the complex register kernels):
    rows of conj(C) composed in list order, per-block normalizers with dead
    atoms; bit-exact against the oracle's complex loop (numpy's product and
    abs); the complex scaled recursion refuses such K."""
    from paper_2204_14194_b200 import _native

    rng = np.random.default_rng(22)
    K, B, I, n = _native.register_atoms_complex() + 1, 3, 12, 2
    ld = _native.table_ld_complex(K)

    def crnd(*shape):
        return torch.complex(torch.from_numpy(rng.normal(size=shape)),
                             torch.from_numpy(rng.normal(size=shape))).to(DEV)

    T0 = torch.zeros((K, ld), dtype=torch.complex128, device=DEV)
    T0[:, :K] = crnd(K, K)
    tabs = torch.zeros((n, K, ld), dtype=torch.complex128, device=DEV)
    tabs[:, :, :K] = 0.3 * crnd(n, K, K)
    counts = torch.tensor([0, 2, 1], dtype=torch.int32, device=DEV)
    ids = torch.tensor([[0, 0], [0, 1], [1, 0]], dtype=torch.int32, device=DEV)
    Dh = rng.uniform(0.5, 1.5, (B, ld))
    Dh[:, [5, K - 2]] = 0.0
    D = torch.from_numpy(Dh).to(DEV)
    R0 = torch.zeros((B, ld), dtype=torch.complex128, device=DEV)
    R0[:, :K] = crnd(B, K)
    sel = torch.empty((B, I), dtype=torch.int32, device=DEV)
    proj = torch.empty((B, I), dtype=torch.complex128, device=DEV)
    coef = torch.empty((B, I), dtype=torch.complex128, device=DEV)
    _native.iterate_complex(T0, D, R0, K, I, 0.5, sel, proj, coef, chunk_tables=tabs,
                            chunk_stride=tabs[0].numel(), chunk_count=counts, chunk_ids=ids)
    torch.cuda.synchronize()

    class ConjRows:  # the oracle conjugates row u: hand it conj(composed row of conj(C))
        def __init__(self, b):
            self.lst = ids[b, : int(counts[b])].tolist()

        def __getitem__(self, u):
            r = T0[u, :K].clone()
            for j in self.lst:
                r = r - tabs[j, u, :K]
            return np.conj(r.cpu().numpy())

    for b in range(B):
        s_ref, p_ref, c_ref, _ = orc.fase_run(R0[b, :K].cpu().numpy(), ConjRows(b), Dh[b, :K], 0.5, I)
        assert np.array_equal(sel[b].cpu().numpy(), s_ref), b
        assert np.array_equal(proj[b].cpu().numpy(), p_ref), b
        assert np.array_equal(coef[b].cpu().numpy(), c_ref), b
        assert not np.isin(s_ref, [5, K - 2]).any()
    d = parse_dict_spec("dft", 79, 79)  # 6,241 complex atoms
    assert len(d) > _native.register_atoms_complex()
    with pytest.raises(UnsupportedDictionaryError):
        fase_extrapolate_batch(np.zeros((1, 79, 79)), wl.central_loss_mask(79, 79, 9, 9), d, None,
                               ExtrapConfig(3), device=DEV, recursion="scaled")


@pytest.mark.parametrize("spec", ["dft", "dct", "union:dct+dft"])
def test_complex_signals(spec):
    """Complex signals (the reference's as_field coercion; its own
    test_initial_products_match_bruteforce uses one): initial products equal the
    oracle's conj(Phi) (s o w) to 1e-13; fase_extrapolate selects exactly the
    oracle loop's atoms on the same products and table, for real dictionaries
    (complex state over the real table) and complex ones; apply_model returns
    Re g with max |Im g|."""
    from paper_2204_14194_b200 import apply_model, initial_scalar_products

    rng = np.random.default_rng(4)
    m = n = 8
    d = parse_dict_spec(spec, m, n)
    mask = wl.central_loss_mask(m, n, 3, 3)
    w = build_weight_field(mask, 0.8)
    s = rng.standard_normal((m, n)) + 1j * rng.standard_normal((m, n))
    vals = d.values.reshape(len(d), -1).astype(np.complex128)
    r0 = initial_scalar_products(s, w, d, device=DEV)
    want = orc.initial_products(s, w, vals)
    assert np.abs(r0 - want).max() <= 1e-13 * np.abs(want).max()
    cfg = ExtrapConfig(25, 0.5, 0.8)
    t = build_gram_tables(d, w, device=DEV)
    model, trace = fase_extrapolate(s, mask, d, t, cfg, device=DEV)
    c, dd = orc.gram(vals, w)
    sel, _, coef, _ = orc.fase_run(r0, c, dd, cfg.gamma, cfg.iterations)
    assert np.array_equal(trace.selected, sel)
    assert np.abs(trace.coefficients - coef).max() <= 1e-12 * np.abs(coef).max()
    out, max_imag = apply_model(s, model, mask, device=DEV)
    g = orc.materialize(d.values, trace.selected, trace.coefficients)
    assert out.dtype == np.complex128
    assert np.abs(out[mask] - g.real[mask]).max() <= 1e-12 * np.abs(g).max()
    assert np.array_equal(out[~mask], s[~mask])
    assert abs(max_imag - np.abs(g.imag[mask]).max()) <= 1e-12 * np.abs(g).max()


@pytest.mark.parametrize("case", ["no_loss", "one_sample_area", "iterations_beyond_k",
                                  "gamma_rho_one", "single_block_per_block_mask"])
def test_drop_in_edge_shapes(case):
    """Edge shapes of the drop-in batch call against the oracle's per-block
    pipeline (weights -> tables -> R0 -> recursion -> synthesis -> paste):
    nothing lost, a 1 x 2 area, more iterations than atoms, gamma = rho = 1,
    a one-block batch with its own mask (chunked path)."""
    rng = np.random.default_rng(41)
    if case == "no_loss":
        d, m, n = generate_dictionary("dct", 6, 6), 6, 6
        masks = np.zeros((6, 6), dtype=bool)
        cfg, B = ExtrapConfig(8), 3
    elif case == "one_sample_area":
        d, m, n = Dictionary(rng.standard_normal((3, 1, 2))), 1, 2
        masks = np.array([[False, True]])
        cfg, B = ExtrapConfig(4), 2
    elif case == "iterations_beyond_k":
        d, m, n = generate_dictionary("wht", 4, 4), 4, 4
        masks = wl.central_loss_mask(4, 4, 2, 2)
        cfg, B = ExtrapConfig(60), 2
    elif case == "gamma_rho_one":
        d, m, n = generate_dictionary("dct", 8, 8), 8, 8
        masks = wl.central_loss_mask(8, 8, 2, 4)
        cfg, B = ExtrapConfig(12, 1.0, 1.0), 2
    else:
        d, m, n = parse_dict_spec("union:dct+had", 12, 12), 12, 12
        masks = wl.central_loss_mask(12, 12, 4, 4)[None].copy()
        masks[0, 0:2, 0:2] = True
        cfg, B = ExtrapConfig(10), 1
    sig = rng.uniform(0, 255, (B, m, n))
    res = fase_extrapolate_batch(sig, masks, d, None, cfg, device=DEV)
    vals = d.real_values().astype(np.complex128)
    for b in range(B):
        mb = masks if masks.ndim == 2 else masks[b]
        ref = orc.extrapolate_block(sig[b], mb, vals, cfg.gamma, cfg.iterations, cfg.rho_hat,
                                    record=True)
        v = compare_selection(res.selected[b].cpu().numpy(), ref["selected"],
                              metric_fn(ref["r0"], ref["d"], ref["log"]))
        assert v.ok, (case, b, v)
        s = v.stop
        scale = max(np.abs(ref["coefficients"][:s]).max(initial=0.0), 1e-300)
        assert np.abs(res.coefficients[b].cpu().numpy()[:s] - ref["coefficients"].real[:s]).max(
            initial=0.0) <= COEF_REL * scale
        got = res.patched[b].cpu().numpy()
        assert np.array_equal(got[~mb], sig[b][~mb])  # support untouched
        if v.exact and mb.any():
            assert rel_dev(got[mb], ref["patched"][mb]) < COEF_REL
