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
