"""GPU parity for complex-valued dictionaries (dft, bdft and unions with them).

The reference's default dictionary is ``dft`` (cli.py:61, conceal.py:171);
these tests hold the complex kernels (csrc/iterate_complex.cu, the complex
Gram / synthesis in csrc/dgemm.cu and csrc/capi.cu) to the same two gates as
the real path:
  1. stage-isolated -- the reference's own tables and initial products drive
     the CUDA recursion; selections, projections, coefficients and the R
     vector after every iteration must be BIT-IDENTICAL to the reference;
  2. end to end -- GPU-built tables and products; selections identical up to a
     legitimate near-tie, coefficients and samples within 1e-6 of the run scale.
"""

import json

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import fase_oracle as orc  # noqa: E402
from paper_2204_14194_b200 import (  # noqa: E402
    ExtrapConfig,
    ExtrapolationPlan,
    GramTable,
    NoSelectableAtomError,
    apply_model,
    build_gram_tables,
    build_weight_field,
    fase_extrapolate,
    fase_extrapolate_batch,
    initial_scalar_products,
    parse_dict_spec,
    provenance_hash,
)
from paper_2204_14194_b200 import workloads as wl  # noqa: E402
from paper_2204_14194_b200.dictionary import Dictionary  # noqa: E402
from paper_2204_14194_b200.model import SparseModel  # noqa: E402
from parity import COEF_REL, compare_selection, metric_fn, rel_dev  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


@pytest.fixture(scope="module")
def meta(golden_dir):
    with open(golden_dir / "golden.json") as fh:
        return json.load(fh)


@pytest.fixture(scope="module")
def cases(golden_dir):
    return np.load(golden_dir / "complex_cases.npz")


# ----------------------------------------------------------------- kernels


@pytest.mark.parametrize("spec,m,n,loss", [("dft", 8, 8, (4, 4)), ("union:dft+bdft", 6, 6, (2, 2)),
                                           ("bdft", 12, 12, (4, 4)), ("dft", 48, 48, (16, 16)),
                                           ("union:dct+dft", 5, 7, (1, 3))])
def test_complex_gram_and_normalizers(spec, m, n, loss):
    d = parse_dict_spec(spec, m, n)
    assert not d.is_real
    mask = wl.central_loss_mask(m, n, *loss)
    w = build_weight_field(mask, 0.8)
    t = build_gram_tables(d, w, device=DEV)
    assert t.is_complex
    k = len(d)
    T = t._G[:, :k].cpu().numpy()           # rows of conj(C)
    assert np.array_equal(T, np.conj(T.T))  # exactly Hermitian
    assert np.all(np.signbit(np.diagonal(T).imag)) and np.all(np.diagonal(T).imag == 0)
    assert np.all(t._G[:, k:].cpu().numpy() == 0)  # zero padding
    c, dd = orc.gram(d.values.reshape(k, -1), w)
    assert rel_dev(np.conj(T), c) < 1e-14
    alive = dd != 0
    assert np.array_equal(t.d != 0, alive)
    assert np.abs(t.d[alive] / dd[alive] - 1).max() < 1e-14
    assert np.allclose(t.c, c, rtol=0, atol=1e-14 * np.abs(c).max())


def test_complex_initial_products():
    d = parse_dict_spec("union:dft+bdft", 16, 16)
    mask = wl.central_loss_mask(16, 16, 6, 6)
    w = build_weight_field(mask, 0.8)
    sig = np.random.default_rng(5).uniform(0, 255, (16, 16))
    got = initial_scalar_products(sig, w, d, device=DEV)
    want = orc.initial_products(sig, w, d.values.reshape(len(d), -1))
    assert rel_dev(got.real, want.real) < 1e-13 and rel_dev(got.imag, want.imag) < 1e-13


# ----------------------------------------------------------------- stage-isolated


def test_complex_recursion_bit_exact(cases, meta):
    """Reference tables + reference R0 -> bit-identical selections, projections,
    coefficients and R after every iteration (numpy's fused complex product and
    scaled abs, restated in csrc/common.cuh)."""
    for case in meta["complex_cases"]:
        k = case["key"]
        d = parse_dict_spec(case["spec"], case["m"], case["n"])
        assert d.content_hash() == int(case["content_hash"]), k
        mask = cases[f"{k}_mask"]
        cfg = ExtrapConfig(case["iterations"], case["gamma"], case["rho_hat"])
        w = build_weight_field(mask, cfg.rho_hat)
        tables = GramTable(c=cases[f"{k}_gram"], d=cases[f"{k}_d"], provenance=provenance_hash(d, w))
        model, trace = fase_extrapolate(cases[f"{k}_signal"], mask, d, tables, cfg,
                                        products=cases[f"{k}_r0"], record_products=True, device=DEV)
        assert np.array_equal(trace.selected, cases[f"{k}_selected"]), k
        assert np.array_equal(trace.projections, cases[f"{k}_projections"]), k
        assert np.array_equal(trace.coefficients, cases[f"{k}_coefficients"]), k
        assert np.array_equal(np.stack(trace.products), cases[f"{k}_products"]), k
        # synthesis is bit-exact too given the same terms, max |Im g| included
        patched, max_imag = apply_model(cases[f"{k}_signal"], model, mask, device=DEV)
        assert np.array_equal(patched[mask], cases[f"{k}_patched_lost"]), k
        assert max_imag == cases[f"{k}_max_imag"], k


def test_complex_synthesis_matches_materialize(cases, meta):
    case = meta["complex_cases"][2]
    k = case["key"]
    d = parse_dict_spec(case["spec"], case["m"], case["n"])
    terms = [(int(u), complex(c)) for u, c in zip(cases[f"{k}_selected"],
                                                  cases[f"{k}_coefficients"])]
    model = SparseModel(shape=d.shape, terms=terms, dictionary=d)
    full = np.ones(d.shape, dtype=bool)
    full[0, 0] = False
    patched, mi = apply_model(np.zeros(d.shape), model, full, device=DEV)
    g = orc.materialize(d.values, cases[f"{k}_selected"], cases[f"{k}_coefficients"])
    assert np.array_equal(patched[full], g.real[full])
    assert mi == np.abs(g.imag[full]).max()


# ----------------------------------------------------------------- end to end


def _check_block(got_sel, got_coef, want_sel, want_coef, metric_at):
    v = compare_selection(got_sel, want_sel, metric_at)
    assert v.ok, f"diverged at {v.stop} with Delta-E gap {v.gap}"
    s = v.stop
    scale = np.abs(want_coef[:s]).max()
    assert np.abs(got_coef[:s] - want_coef[:s]).max() <= COEF_REL * scale
    return v


@pytest.mark.parametrize("recursion", ["exact", "scaled"])
def test_dft48_end_to_end(golden_dir, recursion):
    """The reference's default dictionary on the config-1 geometry, GPU-built
    tables and products, against the reference's own results."""
    z = np.load(golden_dir / "dft48_blocks.npz")
    w1 = wl.WORKLOADS[1]
    m, n = w1.area
    d = parse_dict_spec("dft", m, n)
    mask = wl.central_loss_mask(m, n, *w1.loss)
    blocks = list(z["blocks"])
    sig = wl.block_signals(1, len(blocks), m, n)
    res = fase_extrapolate_batch(sig, mask, d, None, w1.config, device=DEV, recursion=recursion)
    tabs = None
    for b in blocks:
        def metric_at(t, b=b):
            nonlocal tabs
            if tabs is None:
                tabs = orc.gram(d.values.reshape(len(d), -1), orc.weight_field(mask, 0.8))
            _, _, _, log = orc.fase_run(z[f"b{b}_r0"], tabs[0], tabs[1], 0.5, t, record=True)
            return metric_fn(z[f"b{b}_r0"], tabs[1], log)(t)

        v = _check_block(res.selected[b].cpu().numpy(), res.coefficients[b].cpu().numpy(),
                         z[f"b{b}_selected"], z[f"b{b}_coefficients"], metric_at)
        if v.exact:
            lost = res.patched[b].cpu().numpy()[mask]
            assert rel_dev(lost, z[f"b{b}_patched_lost"]) < COEF_REL
            assert abs(float(res.max_imag[b]) - z[f"b{b}_max_imag"]) <= COEF_REL * np.abs(lost).max()


@pytest.mark.parametrize("spec,m,n", [("union:dft+bdft", 16, 16), ("union:wht+dft", 16, 16),
                                      ("bdft", 9, 7)])
@pytest.mark.parametrize("recursion", ["exact", "scaled"])
def test_complex_batch_against_oracle(spec, m, n, recursion):
    d = parse_dict_spec(spec, m, n)
    mask = wl.central_loss_mask(m, n, m // 3, n // 3)
    sig = np.random.default_rng(11).uniform(0, 255, (5, m, n))
    cfg = ExtrapConfig(60, 0.5, 0.8)
    res = fase_extrapolate_batch(sig, mask, d, None, cfg, device=DEV, recursion=recursion)
    vals = d.values
    for b in range(5):
        ref = orc.extrapolate_block(sig[b], mask, vals, 0.5, 60, 0.8, record=True)

        def metric_at(t, ref=ref):
            return metric_fn(ref["r0"], ref["d"], ref["log"])(t)

        v = _check_block(res.selected[b].cpu().numpy(), res.coefficients[b].cpu().numpy(),
                         ref["selected"], ref["coefficients"], metric_at)
        if v.exact:
            assert rel_dev(res.patched[b].cpu().numpy()[mask], ref["patched"][mask]) < COEF_REL


def test_complex_per_block_masks_chunked():
    """Per-block geometries with a complex dictionary: chunked complex tables."""
    d = parse_dict_spec("dft", 12, 12)
    rng = np.random.default_rng(17)
    masks = np.zeros((6, 12, 12), dtype=bool)
    for b in range(6):
        masks[b, 4:8, 4:8] = True
        r, c = rng.integers(0, 9, 2)
        masks[b, r:r + 3, c:c + 3] |= bool(b % 2)
    sig = rng.uniform(0, 255, (6, 12, 12))
    cfg = ExtrapConfig(40, 0.5, 0.8)
    res = fase_extrapolate_batch(sig, masks, d, None, cfg, device=DEV)
    for b in range(6):
        ref = orc.extrapolate_block(sig[b], masks[b], d.values, 0.5, 40, 0.8, record=True)

        def metric_at(t, ref=ref):
            return metric_fn(ref["r0"], ref["d"], ref["log"])(t)

        v = _check_block(res.selected[b].cpu().numpy(), res.coefficients[b].cpu().numpy(),
                         ref["selected"], ref["coefficients"], metric_at)
        if v.exact:
            assert rel_dev(res.patched[b].cpu().numpy()[masks[b]], ref["patched"][masks[b]]) < COEF_REL


def test_complex_plan_matches_batch():
    d = parse_dict_spec("dft", 16, 16)
    mask = wl.central_loss_mask(16, 16, 6, 6)
    cfg = ExtrapConfig(50, 0.5, 0.8)
    sig = np.random.default_rng(23).uniform(0, 255, (9, 16, 16))
    plan = ExtrapolationPlan(d, mask, 9, cfg, device=DEV)
    plan.run(torch.from_numpy(sig).to(DEV))
    res = fase_extrapolate_batch(sig, mask, d, plan.tables, cfg, device=DEV)
    assert torch.equal(plan.selected, res.selected)
    assert torch.equal(plan.coefficients, res.coefficients)
    assert torch.equal(plan.lost, res.patched.reshape(9, -1)[:, torch.from_numpy(mask.ravel()).to(DEV)])
    host = plan.host_buffers()
    pinned = torch.from_numpy(sig).pin_memory()
    plan.run_host_stream([pinned, pinned], [host, plan.host_buffers()])
    torch.cuda.synchronize()
    assert torch.equal(host["coefficients"], res.coefficients.cpu())


def test_complex_zero_signal_and_dead_atoms():
    # zero signal: every metric is 0 -> the lowest live atom, coefficient 0 (untrusted-proxy path)
    d = parse_dict_spec("dft", 8, 8)
    mask = wl.central_loss_mask(8, 8, 4, 4)
    t = build_gram_tables(d, build_weight_field(mask, 0.8), device=DEV)
    _, trace = fase_extrapolate(np.zeros((8, 8)), mask, d, t, ExtrapConfig(5), device=DEV)
    assert (trace.selected == 0).all() and (trace.coefficients == 0).all()
    # an atom living only on the loss is never selected; all-dead raises
    inside = np.zeros((4, 4), dtype=np.complex128)
    inside[1:3, 1:3] = 1.0 + 1.0j
    base = parse_dict_spec("dft", 4, 4).values
    dd = Dictionary(np.concatenate([inside[None], base]))
    m4 = wl.central_loss_mask(4, 4, 2, 2)
    td = build_gram_tables(dd, build_weight_field(m4, 0.8), device=DEV)
    assert td.d[0] == 0.0
    _, trace = fase_extrapolate(np.random.default_rng(2).standard_normal((4, 4)), m4, dd, td,
                                ExtrapConfig(10), device=DEV)
    assert (trace.selected != 0).all()
    dead = Dictionary(inside[None])
    tdead = build_gram_tables(dead, build_weight_field(m4, 0.8), device=DEV)
    with pytest.raises(NoSelectableAtomError):
        fase_extrapolate(np.ones((4, 4)), m4, dead, tdead, device=DEV)


def test_complex_large_k_variant():
    """K = 4608 complex (union:dft+bdft 48x48) through the 512-thread variant."""
    d = parse_dict_spec("union:dft+bdft", 48, 48)
    mask = wl.central_loss_mask(48, 48, 16, 16)
    sig = wl.block_signals(1, 2, 48, 48)
    cfg = ExtrapConfig(30, 0.5, 0.8)
    res = fase_extrapolate_batch(sig, mask, d, None, cfg, device=DEV)
    for b in range(2):
        ref = orc.extrapolate_block(sig[b], mask, d.values, 0.5, 30, 0.8, record=True)

        def metric_at(t, ref=ref):
            return metric_fn(ref["r0"], ref["d"], ref["log"])(t)

        _check_block(res.selected[b].cpu().numpy(), res.coefficients[b].cpu().numpy(),
                     ref["selected"], ref["coefficients"], metric_at)


@pytest.mark.parametrize("copies", [3, 70])
def test_many_exact_ties_lowest_index(copies):
    """Atoms repeated `copies` times tie exactly in every metric: the lowest
    index must win (reference.py:58-73). 70 copies overflow the complex
    kernel's 64-entry candidate list and take its exact fallback pass; the
    real kernel sees the same ties in its tie pass."""
    rng = np.random.default_rng(copies)
    for cplx in (True, False):
        base = parse_dict_spec("dft" if cplx else "dct", 6, 6).values[:12]
        if not cplx:
            base = base.real
        vals = np.concatenate([np.repeat(base[:1], copies, axis=0), base[1:]])
        d = Dictionary(vals)
        mask = wl.central_loss_mask(6, 6, 2, 2)
        sig = rng.uniform(0, 255, (3, 6, 6))
        res = fase_extrapolate_batch(sig, mask, d, None, ExtrapConfig(15, 0.5, 0.8), device=DEV)
        for b in range(3):
            ref = orc.extrapolate_block(sig[b], mask, d.values, 0.5, 15, 0.8)
            got = res.selected[b].cpu().numpy()
            assert np.array_equal(got, ref["selected"]), (cplx, b, got, ref["selected"])
            assert got.min() >= 0 and not np.any((got > 0) & (got < copies))  # only the first copy


@pytest.mark.parametrize("k_rand,copies", [(2930, 70), (4500, 3)])
def test_complex_recursion_bit_exact_paired_blocks(k_rand, copies):
    """Shared geometries with 2304 < K <= 5120 complex atoms run two blocks per
    CTA sharing D^2 (paired variant; an odd batch leaves the last half idle).
    With the oracle's tables and initial products every block is
    bit-identical to the oracle -- including exact ties among `copies`
    repeated atoms (70 overflow the candidate list: the exact fallback pass
    with its extra barriers)."""
    rng = np.random.default_rng(k_rand)
    m = n = 12
    base = rng.normal(size=(k_rand, m, n)) + 1j * rng.normal(size=(k_rand, m, n))
    vals = np.concatenate([np.repeat(base[:1], copies, axis=0), base[1:]])
    d = Dictionary(vals)
    mask = wl.central_loss_mask(m, n, 4, 4)
    cfg = ExtrapConfig(20, 0.5, 0.8)
    w = orc.weight_field(mask, cfg.rho_hat)
    phi = d.values.reshape(len(d), -1)
    c, dd = orc.gram(phi, w)
    tables = GramTable(c=c, d=dd, provenance=provenance_hash(d, build_weight_field(mask, cfg.rho_hat)))
    nb = 151  # more blocks than SMs (smaller batches are not paired)
    sig = rng.uniform(0, 255, (nb, m, n))
    r0 = np.stack([orc.initial_products(sig[b], w, phi) for b in range(nb)])
    res = fase_extrapolate_batch(sig, mask, d, tables, cfg, products=r0, device=DEV)
    for b in (0, 1, 2, nb - 2, nb - 1):
        sel, proj, coef, _ = orc.fase_run(r0[b], c, dd, cfg.gamma, cfg.iterations)
        got = res.selected[b].cpu().numpy()
        assert np.array_equal(got, sel), b
        assert np.array_equal(res.coefficients[b].cpu().numpy(), coef), b
        assert np.array_equal(res.projections[b].cpu().numpy(), proj), b


def test_complex_scaled_matches_exact_and_dead_atoms():
    """The scaled complex recursion: the same selections as the exact kernel on
    the config-1 geometry with the default dictionary (coefficients to
    rounding); a zero signal selects the lowest live atom with coefficient 0;
    dead atoms are never selected."""
    w1 = wl.WORKLOADS[1]
    m, n = w1.area
    d = parse_dict_spec("dft", m, n)
    mask = wl.central_loss_mask(m, n, *w1.loss)
    sig = wl.block_signals(1, 200, m, n)
    rx = fase_extrapolate_batch(sig, mask, d, None, w1.config, device=DEV)
    rs = fase_extrapolate_batch(sig, mask, d, None, w1.config, device=DEV, recursion="scaled")
    same = (rx.selected == rs.selected).all(dim=1)
    assert int(same.sum()) >= 198
    cx, cs = rx.coefficients[same], rs.coefficients[same]
    assert float(((cx - cs).abs().amax(dim=1) / cx.abs().amax(dim=1)).max()) < 1e-12
    d8 = parse_dict_spec("dft", 8, 8)
    m8 = wl.central_loss_mask(8, 8, 4, 4)
    r0 = fase_extrapolate_batch(np.zeros((2, 8, 8)), m8, d8, None, ExtrapConfig(5), device=DEV,
                                recursion="scaled")
    assert (r0.selected.cpu().numpy() == 0).all() and (r0.coefficients.cpu().numpy() == 0).all()
    inside = np.zeros((4, 4), dtype=np.complex128)
    inside[1:3, 1:3] = 1.0 + 1.0j
    dd = Dictionary(np.concatenate([inside[None], parse_dict_spec("dft", 4, 4).values]))
    m4 = wl.central_loss_mask(4, 4, 2, 2)
    r = fase_extrapolate_batch(np.random.default_rng(2).standard_normal((3, 4, 4)), m4, dd, None,
                               ExtrapConfig(10), device=DEV, recursion="scaled")
    assert (r.selected.cpu().numpy() != 0).all()


def test_maximum_atom_count_complex():
    """K at the largest register-resident complex variant: the exact complex
    recursion is bit-exact against the oracle's loop on the same device-built
    table, normalizers and initial products (one atom more runs the streaming
    recursion: test_gpu_parity.py::test_streaming_recursion_complex); K beyond
    fase_max_atoms_complex raises UnsupportedDictionaryError."""
    from paper_2204_14194_b200 import (ExtrapConfig, UnsupportedDictionaryError, _native,
                                       build_gram_tables, build_weight_field,
                                       fase_extrapolate_batch, initial_scalar_products)

    kmax = _native.register_atoms_complex()
    rng = np.random.default_rng(21)
    m = n = 16
    mask = wl.central_loss_mask(m, n, 6, 6)
    vals = rng.standard_normal((kmax, m, n)) + 1j * rng.standard_normal((kmax, m, n))
    d = Dictionary(vals)
    cfg = ExtrapConfig(15, 0.5, 0.8)
    sig = rng.uniform(0, 255, (2, m, n))
    w = build_weight_field(mask, cfg.rho_hat)
    t = build_gram_tables(d, w, device=DEV)
    r0 = np.stack([initial_scalar_products(sig[b], w, d, device=DEV) for b in range(2)])
    res = fase_extrapolate_batch(sig, mask, d, t, cfg, device=DEV, patch=False, products=r0)
    G, D = t.device_tables(torch.device(DEV), complex_rows=True)
    c = np.conj(G[:, :kmax].cpu().numpy())
    dd = D.cpu().numpy()
    for b in range(2):
        sel, _, coef, _ = orc.fase_run(r0[b], c, dd, cfg.gamma, cfg.iterations)
        assert np.array_equal(res.selected[b].cpu().numpy(), sel)
        assert np.array_equal(res.coefficients[b].cpu().numpy(), coef)
    with pytest.raises(UnsupportedDictionaryError):
        _native.table_ld_complex(_native.max_atoms_complex() + 1)


def test_large_area_products_fall_back_to_gemm():
    """dft over a 72 x 72 area (5,184 atoms): the complex separable transform's
    factor tables exceed shared memory, so the products take the dense GEMM for
    every row (the library refuses the transform before launching); R0 matches
    the oracle, and the batch entry point runs end to end."""
    from paper_2204_14194_b200.fast import initial_products_into  # noqa: F401

    d = parse_dict_spec("dft", 72, 72)
    mask = wl.central_loss_mask(72, 72, 8, 8)
    w = build_weight_field(mask, 0.8)
    sig = np.random.default_rng(31).uniform(0, 255, (72, 72))
    got = initial_scalar_products(sig, w, d, device=DEV)
    want = orc.initial_products(sig, w, d.values.reshape(len(d), -1))
    assert rel_dev(got.real, want.real) < 1e-13 and rel_dev(got.imag, want.imag) < 1e-13
    r = fase_extrapolate_batch(np.stack([sig, sig[::-1]]), mask, d, None, ExtrapConfig(5),
                               device=DEV)
    assert r.selected.shape == (2, 5) and (r.selected >= 0).all()


def test_large_area_real_products_fall_back_to_gemm():
    """dct over a 112 x 112 area (12,544 atoms: also past the register kernels):
    the real separable transform does not fit shared memory either, the dense
    products take over; R0 matches the oracle and a short batch runs end to end
    through the streaming recursion."""
    d = parse_dict_spec("dct", 112, 112)
    mask = wl.central_loss_mask(112, 112, 16, 16)
    w = build_weight_field(mask, 0.8)
    sig = np.random.default_rng(32).uniform(0, 255, (112, 112))
    got = initial_scalar_products(sig, w, d, device=DEV)
    want = orc.initial_products(sig, w, d.values.reshape(len(d), -1))
    assert rel_dev(got.real, want.real) < 1e-13
    r = fase_extrapolate_batch(sig[None], mask, d, None, ExtrapConfig(3), device=DEV)
    assert (r.selected >= 0).all()
