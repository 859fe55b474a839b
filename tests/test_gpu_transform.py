"""GPU parity of the transform shortcuts (reference transform.py) and of the
separable complex initial products (csrc/separable.cu).

Mirrors the reference's own test strategy for the shortcuts (pkg/tests/
test_transform.py): shortcut == direct path to rounding, exact Hermitian
tables, untagged atoms rejected, general tag layouts, and tables that drive the
fast path to the same selections -- plus the reference's own shortcut outputs
(tests/golden/transform_cases.npz).
"""

import json

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import fase_oracle as orc  # noqa: E402
from paper_2204_14194_b200 import (  # noqa: E402
    Dictionary,
    ExtrapConfig,
    ExtrapolationPlan,
    UnsupportedDictionaryError,
    build_gram_tables,
    build_weight_field,
    fase_extrapolate,
    fase_extrapolate_batch,
    fft_gram_table,
    fft_initial_products,
    generate_dictionary,
    initial_scalar_products,
    parse_dict_spec,
)
from paper_2204_14194_b200 import _native, workloads as wl  # noqa: E402
from paper_2204_14194_b200.fast import initial_products_into  # noqa: E402
from parity import rel_dev  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def _w(m, n):
    return build_weight_field(wl.central_loss_mask(m, n, m // 2, n // 2), 0.8)


@pytest.mark.parametrize("shape", [(4, 4), (8, 8), (4, 6), (6, 4), (48, 48)])
def test_fft_products_match_direct(shape):
    m, n = shape
    d = generate_dictionary("dft", m, n)
    w = _w(m, n)
    s = np.random.default_rng(m * 100 + n).uniform(0, 255, shape)
    fast = fft_initial_products(s, w, d, min_tagged=1, device=DEV)
    direct = orc.initial_products(s, w, d.values.reshape(len(d), -1))
    assert rel_dev(fast, direct) < 1e-13


def test_fft_products_mixed_and_fallback():
    d = parse_dict_spec("union:dct+dft", 8, 8)
    w = _w(8, 8)
    s = np.random.default_rng(5).standard_normal((8, 8))
    fast = fft_initial_products(s, w, d, min_tagged=1, device=DEV)
    direct = orc.initial_products(s, w, d.values.reshape(len(d), -1))
    assert rel_dev(fast, direct) < 1e-13
    small = generate_dictionary("dft", 4, 4)  # 16 tagged atoms < FFT_MIN_TAGGED: direct path
    w4 = _w(4, 4)
    s4 = s[:4, :4]
    assert np.array_equal(fft_initial_products(s4, w4, small, device=DEV),
                          initial_scalar_products(s4, w4, small, device=DEV))


@pytest.mark.parametrize("shape", [(4, 4), (8, 8), (4, 6), (48, 48)])
def test_fft_gram_matches_direct(shape):
    m, n = shape
    d = generate_dictionary("dft", m, n)
    w = _w(m, n)
    via_fft = fft_gram_table(w, d, device=DEV)
    direct = build_gram_tables(d, w, device=DEV)
    assert rel_dev(via_fft.c, direct.c) < 1e-13
    alive = direct.d != 0
    assert np.array_equal(via_fft.d != 0, alive)
    assert np.abs(via_fft.d[alive] / direct.d[alive] - 1).max() < 1e-12
    assert via_fft.provenance == direct.provenance
    T = via_fft._G[:, : len(d)].cpu().numpy()
    assert np.array_equal(T, np.conj(T.T))
    assert np.all(np.diagonal(T).imag == 0)


def test_fft_gram_against_reference(golden_dir):
    with open(golden_dir / "golden.json") as fh:
        meta = json.load(fh)
    z = np.load(golden_dir / "transform_cases.npz")
    for case in meta["transform_cases"]:
        k, m, n = case["key"], case["m"], case["n"]
        d = parse_dict_spec(case["spec"], m, n)
        got = fft_initial_products(z[f"{k}_signal"], z[f"{k}_w"], d, min_tagged=1, device=DEV)
        assert rel_dev(got, z[f"{k}_products"]) < 1e-13, k
        if f"{k}_gram" in z:
            t = fft_gram_table(z[f"{k}_w"], d, device=DEV)
            assert rel_dev(t.c, z[f"{k}_gram"]) < 1e-13, k
            assert np.abs(t.d - z[f"{k}_d"]).max() <= 1e-13 * np.abs(z[f"{k}_d"]).max(), k


def test_fft_gram_rejects_untagged_and_general_layout():
    w = np.ones((4, 4))
    with pytest.raises(UnsupportedDictionaryError):
        fft_gram_table(w, generate_dictionary("dct", 4, 4), device=DEV)
    with pytest.raises(UnsupportedDictionaryError):
        fft_gram_table(w, parse_dict_spec("union:dct+dft", 4, 4), device=DEV)
    base = generate_dictionary("dft", 4, 4)
    order = np.random.default_rng(3).permutation(16)
    shuffled = Dictionary(base.values[order], families=[base.families[k] for k in order],
                          freqs=[base.freqs[k] for k in order])
    w = _w(4, 4)
    t = fft_gram_table(w, shuffled, device=DEV)
    direct = build_gram_tables(shuffled, w, device=DEV)
    assert rel_dev(t.c, direct.c) < 1e-13
    assert np.array_equal(t.c, np.conj(t.c.T))


def test_fft_tables_drive_the_fast_path():
    d = generate_dictionary("dft", 8, 8)
    mask = wl.central_loss_mask(8, 8, 4, 4)
    w = build_weight_field(mask, 0.8)
    s = np.random.default_rng(9).standard_normal((8, 8))
    cfg = ExtrapConfig(iterations=25)
    _, via_fft = fase_extrapolate(s, mask, d, fft_gram_table(w, d, device=DEV), cfg, device=DEV)
    _, direct = fase_extrapolate(s, mask, d, build_gram_tables(d, w, device=DEV), cfg, device=DEV)
    assert np.array_equal(via_fft.selected, direct.selected)
    assert np.allclose(via_fft.coefficients, direct.coefficients, rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("spec,m,n", [("dft", 48, 48), ("union:dct+dft", 16, 16),
                                      ("union:dft+bdft", 12, 12), ("union:wht+dft", 16, 16),
                                      ("dft", 5, 7)])
def test_batched_complex_products_separable_vs_gemm(spec, m, n):
    """Separable complex transforms (with GEMM for the non-separable rows) equal
    the dense conjugate-split GEMM and the oracle to rounding."""
    d = parse_dict_spec(spec, m, n)
    mask = wl.central_loss_mask(m, n, m // 3, n // 3)
    w = build_weight_field(mask, 0.8)
    B = 37
    sig = np.random.default_rng(1).uniform(0, 255, (B, m, n))
    M, K = m * n, len(d)
    ld = M + (M & 1)
    F = torch.zeros((B, ld), dtype=torch.float64, device=DEV)
    F[:, :M] = torch.from_numpy(sig.reshape(B, -1)).to(DEV)
    W = torch.zeros(ld, dtype=torch.float64, device=DEV)
    W[:M] = torch.from_numpy(w.ravel()).to(DEV)
    ws = torch.empty(max(_native.init_products_workspace(M, B) // 8, 2), dtype=torch.float64,
                     device=DEV)
    Rs = torch.zeros((B, K), dtype=torch.complex128, device=DEV)
    Rg = torch.zeros((B, K), dtype=torch.complex128, device=DEV)
    how = initial_products_into(d, F, W, Rs, ws, method="auto")
    assert how.startswith("separable")
    assert initial_products_into(d, F, W, Rg, ws, method="gemm") == "gemm"
    a, g = Rs.cpu().numpy(), Rg.cpu().numpy()
    assert rel_dev(a, g) < 1e-13
    phi = d.values.reshape(K, -1)
    for b in (0, 36):
        assert rel_dev(a[b], orc.initial_products(sig[b], w, phi)) < 1e-13


def test_plan_uses_separable_complex_products():
    d = generate_dictionary("dft", 16, 16)
    mask = wl.central_loss_mask(16, 16, 6, 6)
    cfg = ExtrapConfig(40, 0.5, 0.8)
    sig = np.random.default_rng(2).uniform(0, 255, (6, 16, 16))
    plan = ExtrapolationPlan(d, mask, 6, cfg, device=DEV)
    plan.run(torch.from_numpy(sig).to(DEV))
    assert plan.products_method == "separable"
    ref = fase_extrapolate_batch(sig, mask, d, plan.tables, cfg, device=DEV)
    assert torch.equal(plan.selected, ref.selected)


# ----------------------------------------------------------------- tcgen05 Ozaki products


@pytest.mark.parametrize("slices", [8, 7])
@pytest.mark.parametrize("M,N,Kd,kind", [(300, 200, 131, "uniform"), (1000, 333, 777, "wide"),
                                         (256, 128, 64, "zeros"), (130, 65, 4000, "signal")])
def test_ozaki_gemm_matches_fp64(M, N, Kd, kind, slices):
    """tcgen05 INT8 digit-plane contraction == FP64 contraction to rounding:
    with 8 planes the error is within 1e-15 of sum |x y| (the DMMA GEMM
    measures 1.7e-16 - 2.8e-16 on the same data; rows with a wide dynamic range
    lose low digits of their small entries, so the bound is a few ulp, not
    one); 7 planes (the batched products' setting) drop 7 more bits: 2^7 x."""
    rng = np.random.default_rng(M * 7 + N)
    if kind == "wide":
        X = rng.standard_normal((M, Kd)) * 10.0 ** rng.integers(-3, 4, (M, 1))
        Y = rng.standard_normal((N, Kd)) * 10.0 ** rng.integers(-3, 4, (1, Kd))
    elif kind == "signal":
        X = rng.uniform(0, 255, (M, Kd)) * 0.8 ** rng.uniform(0, 30, Kd)
        Y = rng.standard_normal((N, Kd)) / 64
    else:
        X = rng.uniform(-1, 1, (M, Kd))
        Y = rng.uniform(-1, 1, (N, Kd))
    if kind == "zeros":
        X[::3] = 0.0
        Y[:, ::5] = 0.0
    ld = Kd + (Kd & 1)
    Xd = torch.zeros((M, ld), dtype=torch.float64, device=DEV)
    Xd[:, :Kd] = torch.from_numpy(X)
    Yd = torch.zeros((N, ld), dtype=torch.float64, device=DEV)
    Yd[:, :Kd] = torch.from_numpy(Y)
    a = _native.OzakiOperand(M, Kd, 128, DEV, slices).split(Xd)
    b = _native.OzakiOperand(N, Kd, 64, DEV, slices).split(Yd)
    C = torch.full((M, N + 3), 7.0, dtype=torch.float64, device=DEV)
    _native.ozaki_gemm(a, b, C)
    c = C.cpu().numpy()
    assert np.all(c[:, N:] == 7.0)  # nothing written past the valid columns
    XL, YL = X.astype(np.longdouble), Y.astype(np.longdouble)
    rows = rng.integers(0, M, 60)
    cols = rng.integers(0, N, 60)
    ref = np.array([np.dot(XL[i], YL[j]) for i, j in zip(rows, cols)])
    scale = np.array([np.dot(np.abs(XL[i]), np.abs(YL[j])) for i, j in zip(rows, cols)])
    err = np.abs(c[rows, cols] - ref) / np.maximum(scale, 1e-300)
    assert float(err.max()) < 1e-15 * 2.0 ** (7 * (8 - slices))
    if kind == "zeros":
        assert np.all(c[::3, :N] == 0.0)


@pytest.mark.parametrize("rows,K,L,iters", [(300, 700, 130, 40), (129, 2000, 64, 1500)])
def test_ozaki_sparse_synthesis_matches_dense(rows, K, L, iters):
    """fase_ozaki_split_sparse + fase_ozaki_gemm == V Phi_lost^T for sparse
    models with repeated atoms (inside one 32-term window and across 1,024-term
    staging windows), stopped runs (sel = -1 tails), an empty model and out-of-
    range atoms: within the truncation bound of 7 planes (every operand entry
    carries 49 bits of its row's scale, so |err| <= 2 nnz 2^-49 max|v_r|
    max|phi_i|, plus the dropped plane pairs), deterministic from run to run."""
    rng = np.random.default_rng(rows + K)
    sel = rng.integers(0, K, (rows, iters)).astype(np.int32)
    coef = rng.standard_normal((rows, iters)) * 10.0 ** rng.uniform(-4, 2, (rows, iters))
    sel[0, 1:9] = sel[0, 0]          # repeats inside a window
    sel[1, 5] = sel[1, min(iters - 1, 1030)]  # across windows (long models)
    sel[2, iters // 2:] = -1         # a run that stopped (NoSelectableAtom)
    sel[3, :] = -1                   # an empty model
    sel[4, 3] = K + 5                # out of range: no term
    phi = rng.standard_normal((K, L)) / 16
    V = np.zeros((rows, K))
    for r in range(rows):
        for t in range(iters):
            if 0 <= sel[r, t] < K:
                V[r, sel[r, t]] += coef[r, t]
    want = V.astype(np.longdouble) @ phi.astype(np.longdouble)
    nnz = (V != 0).sum(axis=1)
    bound = ((nnz + 1) * 2.0 ** -47 * np.abs(V).max(axis=1))[:, None] * np.abs(phi).max(axis=0)[None, :]
    phi_t = torch.from_numpy(np.ascontiguousarray(phi.T)).to(DEV)
    b = _native.OzakiOperand(L, K, 64, DEV, 7).split(phi_t)
    sel_d = torch.from_numpy(sel).to(DEV)
    coef_d = torch.from_numpy(coef).to(DEV)
    outs = []
    for _ in range(2):
        a = _native.OzakiOperand(rows, K, 128, DEV, 7).split_sparse(sel_d, coef_d, iters)
        C = torch.full((rows, L + 1), 3.0, dtype=torch.float64, device=DEV)
        _native.ozaki_gemm(a, b, C)
        outs.append(C.cpu().numpy())
    c = outs[0]
    assert np.array_equal(outs[0], outs[1])
    assert np.all(c[:, L] == 3.0)
    assert np.all(c[3, :L] == 0.0)
    assert np.all(np.abs(c[:, :L] - want) <= bound)


def test_plan_ozaki_synthesis(monkeypatch):
    """The plan's synthesis as one Ozaki product (FASE_SYNTH=ozaki forces it
    on a small batch; config 4 takes it by size): the same selections and
    coefficients as the per-block paste, lost samples within 1e-12 of the
    paste's, and of the oracle's for sampled blocks."""
    d = parse_dict_spec("gauss:900:3", 16, 16)
    mask = wl.central_loss_mask(16, 16, 6, 6)
    cfg = ExtrapConfig(30, 0.5, 0.85)
    sig = np.random.default_rng(21).uniform(0, 255, (300, 16, 16))
    sig_d = torch.from_numpy(sig).to(DEV)
    monkeypatch.setenv("FASE_SYNTH", "paste")
    ref = ExtrapolationPlan(d, mask, 300, cfg, device=DEV).run(sig_d)
    assert ref._synth_oz is None
    monkeypatch.setenv("FASE_SYNTH", "ozaki")
    oz = ExtrapolationPlan(d, mask, 300, cfg, device=DEV).run(sig_d)
    assert oz._synth_oz is not None and oz.launches_per_run == ref.launches_per_run + 1
    torch.cuda.synchronize()
    assert torch.equal(oz.selected, ref.selected)
    assert torch.equal(oz.coefficients, ref.coefficients)
    assert rel_dev(oz.lost.cpu().numpy(), ref.lost.cpu().numpy()) < 1e-12
    for b in (0, 150, 299):
        want = orc.extrapolate_block(sig[b], mask, d.values, 0.5, 30, 0.85)
        assert rel_dev(oz.lost[b].cpu().numpy(), want["patched"][mask].real) < 1e-12


@pytest.mark.parametrize("spec", ["gauss:700:5", "bdft"])
def test_plan_ozaki_products(spec):
    """The plan's tcgen05 path (weigh-gather, digit split, INT8 MMAs; 7 digit
    planes, _native.PRODUCT_SLICES) reproduces the reference's initial
    products to 1e-12 and its selections."""
    d = parse_dict_spec(spec, 16, 16)
    mask = wl.central_loss_mask(16, 16, 6, 6)
    cfg = ExtrapConfig(40, 0.5, 0.85)
    sig = np.random.default_rng(9).uniform(0, 255, (150, 16, 16))
    plan = ExtrapolationPlan(d, mask, 150, cfg, device=DEV, products="ozaki")
    assert plan._ozaki is not None and plan.launches_per_run == 4
    plan.run(torch.from_numpy(sig).to(DEV))
    assert plan.products_method == "ozaki-support"
    R0 = plan.R0[:, : len(d)].cpu().numpy()
    ref_plan = ExtrapolationPlan(d, mask, 150, cfg, device=DEV, products="gemm")
    ref_plan.run(torch.from_numpy(sig).to(DEV))
    assert rel_dev(R0, ref_plan.R0[:, : len(d)].cpu().numpy()) < 1e-12
    for b in (0, 77, 149):
        ref = orc.extrapolate_block(sig[b], mask, d.values, 0.5, 40, 0.85, record=True)
        assert rel_dev(R0[b], ref["r0"] if not d.is_real else ref["r0"].real) < 1e-12
        from parity import compare_selection, metric_fn

        v = compare_selection(plan.selected[b].cpu().numpy(), ref["selected"],
                              metric_fn(ref["r0"], ref["d"], ref["log"]))
        assert v.ok


def test_batch_api_uses_ozaki_for_large_dense_batches():
    """fase_extrapolate_batch on a batch that fills the GPU with a dense
    dictionary takes the tcgen05 products (support samples only): R0 and the
    selections still match the oracle."""
    from paper_2204_14194_b200 import fase_extrapolate_batch
    from parity import compare_selection, metric_fn

    d = parse_dict_spec("gauss:2560:4", 16, 16)
    mask = wl.central_loss_mask(16, 16, 6, 6)
    cfg = ExtrapConfig(20, 0.5, 0.8)
    sig = np.random.default_rng(12).uniform(0, 255, (2048, 16, 16))
    from paper_2204_14194_b200.fast import ozaki_worthwhile

    assert ozaki_worthwhile(2048, len(d))
    res = fase_extrapolate_batch(sig, mask, d, None, cfg, record_products=True, device=DEV)
    vals = d.values
    for b in (0, 1000, 2047):
        ref = orc.extrapolate_block(sig[b], mask, vals, 0.5, 20, 0.8, record=True)
        v = compare_selection(res.selected[b].cpu().numpy(), ref["selected"],
                              metric_fn(ref["r0"], ref["d"], ref["log"]))
        assert v.ok
        assert rel_dev(res.coefficients[b].cpu().numpy()[: v.stop], ref["coefficients"].real[: v.stop]) < 1e-9


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_gram_row_panels_bit_identical(world):
    """The multi-GPU table build (shard.build_gram_tables_sharded): each rank's
    row panel of the non-symmetric Ozaki product, assembled and mirrored
    (fase_mirror_upper), equals the single-GPU symmetric table bit for bit --
    here the N ranks' panels are built one after another on one GPU."""
    from paper_2204_14194_b200 import _native
    from paper_2204_14194_b200.fast import _device_vector, gram_into, gram_panel_into, gram_support
    from paper_2204_14194_b200.shard import block_range

    d = parse_dict_spec("gauss:2304:7", 24, 24)
    mask = wl.central_loss_mask(24, 24, 8, 8)
    w = build_weight_field(mask, 0.85)
    K, M = len(d), d.area
    dev = torch.device(DEV)
    phi = d.device_matrix(dev)
    w_dev = _device_vector(w.ravel(), d.ld, dev)
    support = gram_support(w_dev, M)
    ld = _native.table_ld(K)
    G1 = torch.zeros((K, ld), dtype=torch.float64, device=dev)
    assert gram_into(phi, w_dev, K, M, G1, support) == "ozaki"
    G2 = torch.full((K, ld), float("nan"), dtype=torch.float64, device=dev)
    G2[:, K:] = 0.0
    for r in range(world):
        lo, hi = block_range(K, r, world)
        gram_panel_into(phi, w_dev, K, M, G2, lo, hi, support)
    _native.mirror_upper(G2, K)
    torch.cuda.synchronize()
    assert torch.equal(G1, G2)
