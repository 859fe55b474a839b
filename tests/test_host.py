"""Host-side logic of the drop-in API (no GPU): weights, dictionaries,
provenance, chunk planning, workloads, sharding."""

import json

import numpy as np
import pytest

from paper_2204_14194_b200 import (
    Dictionary,
    ExtrapConfig,
    MaskError,
    ParameterError,
    ShapeError,
    build_weight_field,
    build_weight_fields,
    chunk_plan,
    generate_dictionary,
    hadamard_matrix,
    load_dictionary,
    parse_dict_spec,
    provenance_hash,
    psnr_over_region,
    save_dictionary,
    union_dictionaries,
)
from paper_2204_14194_b200 import workloads as wl
from paper_2204_14194_b200.errors import FormatError, NativeLibraryError
from paper_2204_14194_b200.shard import block_range


@pytest.fixture(scope="module")
def meta(golden_dir):
    with open(golden_dir / "golden.json") as fh:
        return json.load(fh)


# ----------------------------------------------------------------- config / weights


@pytest.mark.parametrize("kw", [dict(iterations=0), dict(iterations=2.5), dict(gamma=0.0),
                                dict(gamma=1.5), dict(rho_hat=0.0), dict(rho_hat=1.01),
                                dict(iterations=True)])
def test_config_validation(kw):
    with pytest.raises(ParameterError):
        ExtrapConfig(**kw)


def test_weights_match_reference_golden(golden_dir, meta):
    z = np.load(golden_dir / "weights.npz")
    for rec in meta["weights"]:
        k = rec["key"]
        mask = z["mask" + k[1:]]
        assert np.array_equal(build_weight_field(mask, rec["rho"]), z[k])


def test_batched_weights_bit_identical():
    rng = np.random.default_rng(1)
    masks = rng.random((5, 9, 7)) < 0.3
    ws = build_weight_fields(masks, 0.77)
    for b in range(5):
        assert np.array_equal(ws[b], build_weight_field(masks[b], 0.77))


def test_weight_errors():
    with pytest.raises(MaskError):
        build_weight_field(np.ones((3, 3), bool), 0.8)
    with pytest.raises(ParameterError):
        build_weight_field(np.zeros((3, 3), bool), 0.0)
    with pytest.raises(ShapeError):
        build_weight_field(np.zeros(9, bool), 0.8)
    with pytest.raises(MaskError):
        build_weight_fields(np.ones((2, 3, 3), bool), 0.8)


def test_psnr_sentinels():
    a = np.full((4, 4), 10.0)
    reg = np.ones((4, 4), bool)
    assert psnr_over_region(a, a, reg) == 99.0
    assert psnr_over_region(a, a + 1.0, reg) == pytest.approx(20 * np.log10(255.0))
    with pytest.raises(ParameterError):
        psnr_over_region(a, a, np.zeros((4, 4), bool))


# ----------------------------------------------------------------- dictionaries


def test_content_hashes_match_reference(meta):
    for rec in meta["hashes"]:
        if rec["spec"].startswith("gauss"):
            continue
        d = parse_dict_spec(rec["spec"], rec["m"], rec["n"])
        assert len(d) == rec["K"]
        assert d.content_hash() == int(rec["content_hash"]), rec["spec"]


@pytest.mark.slow
def test_gaussian_dictionary_hash(meta):
    rec = [h for h in meta["hashes"] if h["spec"].startswith("gauss")][0]
    d = wl.WORKLOADS[4].dictionary()
    assert len(d) == 8192
    assert d.content_hash() == int(rec["content_hash"])


def test_provenance_matches_reference(meta):
    for case in meta["small_cases"]:
        d = parse_dict_spec(case["spec"], case["m"], case["n"])
        mask = wl.central_loss_mask(case["m"], case["n"], *case["loss"])
        w = build_weight_field(mask, case["rho_hat"])
        assert provenance_hash(d, w) == int(case["provenance"]), case["spec"]


@pytest.mark.parametrize("order", [1, 2, 4, 12, 20, 24, 40, 44, 48, 64, 96])
def test_hadamard_orders(order):
    h = hadamard_matrix(order)
    assert h.shape == (order, order)
    assert set(np.unique(h)) <= {-1.0, 1.0}
    assert np.array_equal(h @ h.T, order * np.eye(order))
    assert (h[0] == 1).all()


def test_hadamard_unknown_order():
    with pytest.raises(ParameterError):
        hadamard_matrix(6)


def test_real_dft_family():
    d = parse_dict_spec("union:rdft+brdft", 32, 32)
    assert len(d) == 2048 and d.is_real
    v = d.real_values()
    assert np.isin(v[1024:], (-1.0, 0.0, 1.0)).all()
    norms = np.sqrt((v.reshape(2048, -1) ** 2).sum(axis=1))
    assert (norms > 0).all()
    # rank of the cos/sin part is the full area
    assert np.linalg.matrix_rank(v[:1024].reshape(1024, -1)) == 1024


def test_union_and_specs():
    u = union_dictionaries([generate_dictionary("dct", 4, 4), generate_dictionary("wht", 4, 4)])
    assert len(u) == 32 and u.is_separable
    with pytest.raises(ParameterError):
        parse_dict_spec("union:dct", 4, 4)
    with pytest.raises(ParameterError):
        parse_dict_spec("nope", 4, 4)
    with pytest.raises(ParameterError):
        generate_dictionary("wht", 6, 4)
    with pytest.raises(ShapeError):
        union_dictionaries([generate_dictionary("dct", 4, 4), generate_dictionary("dct", 4, 5)])
    with pytest.raises(ParameterError):
        Dictionary(np.zeros((2, 3, 3)))
    d = parse_dict_spec("gauss:16:3", 4, 4)
    assert len(d) == 16 and np.allclose((d.matrix() ** 2).sum(axis=1), 1.0)


def test_dictionary_values_and_complex():
    d = generate_dictionary("dct", 4, 4)
    assert d.values.dtype == np.complex128 and d.values.shape == (16, 4, 4)
    dft = generate_dictionary("dft", 4, 4)
    assert not dft.is_real and dft.freqs[5] == (1, 1)
    with pytest.raises(ParameterError):
        dft.real_values()


def test_fdic_round_trip(tmp_path):
    d = parse_dict_spec("union:dct+had", 4, 4)
    p = tmp_path / "d.fdic"
    save_dictionary(d, p)
    e = load_dictionary(p)
    assert np.array_equal(e.real_values(), d.real_values())
    assert e.content_hash() == d.content_hash()
    p.write_bytes(b"junk\n")
    with pytest.raises(FormatError):
        load_dictionary(p)


# ----------------------------------------------------------------- per-block geometry


def test_chunk_plan_partitions_samples():
    rng = np.random.default_rng(5)
    base = np.zeros((6, 6), bool)
    base[2:4, 2:4] = True
    patches = [np.s_[0:2, 0:2], np.s_[0:2, 4:6], np.s_[4:6, 0:3]]
    masks = np.repeat(base[None], 10, axis=0)
    for b in range(10):
        for p in patches:
            if rng.random() < 0.5:
                masks[b][p] = True
    plan = chunk_plan(masks)
    assert plan.base_lost.reshape(6, 6)[2:4, 2:4].all()
    seen = np.concatenate(plan.classes) if plan.classes else np.zeros(0, int)
    assert len(seen) == len(set(seen.tolist()))
    # every block's mask = base lost + exactly its listed classes
    for b in range(10):
        rebuilt = plan.base_lost.copy()
        for j in plan.ids[plan.ptr[b]:plan.ptr[b + 1]]:
            rebuilt[plan.classes[j]] = True
        assert np.array_equal(rebuilt, masks[b].ravel())
    assert plan.n_classes <= len(patches)


def test_frame_geometry_config2_and_3():
    for cid, n_expected in ((2, 804), (3, 25920)):
        w = wl.WORKLOADS[cid]
        case = wl.frame_case(w)
        assert case.n_blocks == n_expected
        assert case.lost.sum() == n_expected * w.macroblock ** 2
    w = wl.WORKLOADS[3]
    case = wl.frame_case(w)
    sig, masks = wl.frame_areas(case.damaged(), case.lost, case.corners[:50], case.mb, case.support)
    plan = chunk_plan(masks)
    assert plan.n_classes <= 25  # area sliced by macroblock / frame boundaries
    assert (masks[:, 12:20, 12:20]).all()  # the own macroblock is always lost
    assert (sig[masks] == 0).all()


def test_block_signals_deterministic():
    a = wl.block_signals(1, 3, 48, 48, first=5)
    b = wl.block_signals(1, 8, 48, 48)
    assert np.array_equal(a, b[5:8])
    assert a.min() >= 0 and a.max() <= 255


def test_block_range_covers_everything():
    for n in (0, 1, 7, 1024, 25920):
        for world in (1, 2, 3, 8):
            spans = [block_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            sizes = [h - l for l, h in spans]
            assert max(sizes) - min(sizes) <= 1


def test_gpu_entry_points_refuse_without_cuda():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2204_14194_b200 import fase_extrapolate_batch

    d = generate_dictionary("dct", 4, 4)
    with pytest.raises(NativeLibraryError):
        fase_extrapolate_batch(np.zeros((1, 4, 4)), np.eye(4, dtype=bool), d)


# ----------------------------------------------------------------- FGRM table files


def test_fgrm_reads_reference_file_and_round_trips(golden_dir, meta, tmp_path):
    from paper_2204_14194_b200 import load_gram_table, save_gram_table

    rec = meta["fgrm"]
    t = load_gram_table(golden_dir / "ref_tables.fgrm")
    d = parse_dict_spec(rec["spec"], rec["m"], rec["n"])
    w = build_weight_field(wl.central_loss_mask(4, 4, 2, 2), 0.8)
    assert t.size == len(d) == 32
    assert t.provenance == int(rec["provenance"]) == provenance_hash(d, w)
    out = tmp_path / "t.fgrm"
    save_gram_table(t, out)
    assert out.stat().st_size == 24 + 16 * 32 * 32 + 8 * 32
    back = load_gram_table(out)
    # values survive (a signed zero in an imaginary part may not: loading
    # forms re + 1j*im, in the reference as here)
    assert np.array_equal(back.c, t.c) and np.array_equal(back.d, t.d)
    assert back.provenance == t.provenance
    again = tmp_path / "t2.fgrm"
    save_gram_table(back, again)
    assert again.read_bytes() == out.read_bytes()


def test_fgrm_rejects_bad_files(golden_dir, tmp_path):
    from paper_2204_14194_b200 import load_gram_table

    blob = (golden_dir / "ref_tables.fgrm").read_bytes()
    bad = tmp_path / "bad.fgrm"
    for payload in (b"GARBAGE!" + blob[8:], blob + b"\0", blob[:-8], blob[:20]):
        bad.write_bytes(payload)
        with pytest.raises(FormatError):
            load_gram_table(bad)


def test_central_loss_mask_errors():
    """Same ParameterError conditions as the reference (verify.py:37-49)."""
    assert wl.central_loss_mask(48, 48, 16, 16)[16:32, 16:32].all()
    assert wl.central_loss_mask(4, 4, 4, 3).sum() == 12
    for bad in ((4, 4, 4, 4), (4, 4, 0, 2), (4, 4, 5, 1), (3, 5, 1, 6)):
        with pytest.raises(ParameterError):
            wl.central_loss_mask(*bad)


def test_complex_signal_rejected_with_boundary_error():
    """A complex signal with a non-zero imaginary part is refused with
    UnsupportedDictionaryError (the GPU path takes real images); one with a
    zero imaginary part is the real field."""
    from paper_2204_14194_b200.errors import UnsupportedDictionaryError
    from paper_2204_14194_b200.grid import as_real_field

    z = np.arange(6.0).reshape(2, 3) + 0j
    assert np.array_equal(as_real_field(z), z.real)
    with pytest.raises(UnsupportedDictionaryError):
        as_real_field(z + 1j)
    with pytest.raises(ShapeError):
        as_real_field(np.zeros(3))


def test_bench_parity_classifier(golden_dir):
    """bench.parity_vs_reference (the post-clock check of the timed outputs):
    the reference's own outputs classify as identical; a swap at an iteration
    with a near-tie set is a near-tie stop; any other swap is a failure."""
    import bench

    z = np.load(golden_dir / "c3_batch.npz")
    n = int(z["n_blocks"])
    I = z["selected"].shape[1]
    sel = np.zeros((n, I), dtype=np.int32)
    coef = np.zeros((n, I))
    sel[z["blocks"]] = z["selected"]
    coef[z["blocks"]] = z["coefficients"]
    out = bench.parity_vs_reference(3, sel, coef, None, 0)
    assert out["identical"] == len(z["blocks"]) and out["failure"] == 0
    assert out["max_coef_rel_dev"] == 0.0
    i, t, k = (int(x) for x in z["ties"][0])
    want = int(z["selected"][i][t])
    alt = next(int(kk) for ii, tt, kk in z["ties"] if ii == i and tt == t and kk != want)
    s2 = sel.copy()
    s2[z["blocks"][i], t] = alt
    out = bench.parity_vs_reference(3, s2, coef, None, 0)
    assert out["near_tie"] == 1 and out["failure"] == 0
    tied = {(int(a), int(b)) for a, b, _ in z["ties"]}
    j, tj = next((j, tt) for j in range(len(z["blocks"])) for tt in range(I) if (j, tt) not in tied)
    s3 = sel.copy()
    s3[z["blocks"][j], tj] = (int(z["selected"][j][tj]) + 1) % 2048
    out = bench.parity_vs_reference(3, s3, coef, None, 0)
    assert out["failure"] == 1
