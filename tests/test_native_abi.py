"""The C-ABI library loads without a GPU and exports every declared entry point.

No compute is launched here: only host-side entry points (version / capacity
queries) and argument validation paths that return before touching CUDA.
"""

import ctypes
import re
from pathlib import Path

import pytest

from paper_2204_14194_b200 import _build, _native, errors

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "fase_b200.h"


@pytest.fixture(scope="module")
def lib():
    _build.build()
    return _native.load()


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"FASE_API\s+[\w\s\*]*?\b(fase_\w+)\s*\(", text)))


def test_header_declares_the_abi():
    names = declared_symbols()
    assert "fase_iterate" in names and "fase_gram" in names and "fase_synth_paste" in names
    assert set(names) == set(_native.EXPORTS)


def test_every_declared_symbol_is_exported(lib):
    raw = ctypes.CDLL(str(_native.library_path()))
    for name in declared_symbols():
        assert hasattr(raw, name), name


def test_host_queries(lib):
    assert lib.fase_abi_version() == (3 << 16)  # 3.0: fase_iterate_args.order
    assert lib.fase_max_atoms() >= 8192
    assert lib.fase_gram_workspace(4608, 2304) == 8 * 4608 * 2304
    assert lib.fase_init_products_workspace(35, 3) == 8 * 3 * 36
    # rows padded to the kernel variant's capacity, never shorter than K, even
    for k in (1, 35, 2048, 2304, 4608, 8192):
        ld = _native.table_ld(k)
        assert ld >= k and ld % 2 == 0
    assert _native.table_ld(4608) == 4608 and _native.table_ld(8192) == 8192
    assert _native.table_ld(2048) == 2048
    with pytest.raises(errors.UnsupportedDictionaryError):
        _native.table_ld(lib.fase_max_atoms() + 1)
    # complex tables: leading dimensions in complex elements
    assert lib.fase_max_atoms_complex() >= 4608
    for k in (1, 64, 2304, 4608):
        assert _native.table_ld_complex(k) >= k
    assert _native.table_ld_complex(2304) == 2304 and _native.table_ld_complex(4608) == 4608
    with pytest.raises(errors.UnsupportedDictionaryError):
        _native.table_ld_complex(lib.fase_max_atoms_complex() + 1)
    # complex Gram workspace: w2, P o w2 and Q (K x 2 ldphi each), Re / Im (K x K)
    assert lib.fase_gram_complex_workspace(64, 64) == 8 * (128 + 2 * 64 * 128 + 2 * 64 * 64)


def test_status_codes_and_messages(lib):
    # argument errors are reported before any CUDA call
    assert lib.fase_iterate(None, None) == -2
    assert b"null argument" in lib.fase_last_error()
    assert lib.fase_gram(None, 0, None, 0, 0, None, 0, None, 0, None) == -1
    assert lib.fase_init_products(None, 0, None, 0, None, 0, 4, 4, -1, None, 0, None, 0,
                                  None) == -1
    assert lib.fase_synth_paste(None, 0, None, None, 0, 0, 1, None, None, 0, None, None, 0,
                                None) == -1
    args = _native.IterateArgs(K=4, B=1, I=1, gamma=2.0)
    assert lib.fase_iterate(ctypes.byref(args), None) == -2
    assert b"gamma" in lib.fase_last_error()
    assert lib.fase_iterate_complex(ctypes.byref(args), None) == -2
    assert lib.fase_iterate_complex(None, None) == -2
    assert lib.fase_gram_complex(None, 0, None, 0, 0, None, 0, None, 0, None) == -1
    assert lib.fase_synth_paste_complex(None, 0, None, None, 0, 0, 1, None, None, 0, None, None, 0,
                                        None, None) == -1
    # transform shortcuts, support gather, tcgen05 Ozaki products
    assert lib.fase_sep_products_complex(None, None, 0, 4, None, None, 4, 4, None, 16, 1, None, 16,
                                         0, None) == -1
    assert lib.fase_fft_gram(None, 4, 4, None, None, 17, None, 17, None) == -1  # K > M*N
    assert b"canonical" in lib.fase_last_error()
    assert lib.fase_weigh_gather(None, 8, None, None, 2, 4, None, 2, None) == -1  # ldo < 4
    assert lib.fase_ozaki_split(None, 64, None, None, 4, 64, 9, None, 64, 8, None, None) == -1
    assert b"slices=9" in lib.fase_last_error()
    assert lib.fase_ozaki_split(None, 64, None, None, 4, 70, 8, None, 64, 8, None, None) == -1
    assert lib.fase_ozaki_gemm(None, 128, None, 100, None, 64, None, 50, 96, 8, None, 50,
                               None) == -1  # kp not a multiple of 64
    assert lib.fase_ozaki_gemm(None, 64, None, 100, None, 64, None, 50, 64, 8, None, 50,
                               None) == -1  # A rows not padded to 128
    assert b"padded" in lib.fase_last_error()
    # scaled recursion: same argument checks; shared geometry only
    assert lib.fase_iterate_scaled(None, None, None) == -2
    args = _native.IterateArgs(K=4, B=1, I=1, gamma=2.0)
    assert lib.fase_iterate_scaled(ctypes.byref(args), None, None) == -2
    fake = 1 << 20  # aligned, never dereferenced: validation returns first
    args = _native.IterateArgs(G0=fake, ldg=4, D=fake, R0=fake, ldr=4, K=4, B=1, I=1, gamma=0.5,
                               sel=fake, proj=fake, coef=fake, ldo=1, chunk_count=fake)
    assert lib.fase_iterate_scaled(ctypes.byref(args), None, None) == -8
    assert b"shared geometry only" in lib.fase_last_error()
    args = _native.IterateArgs(G0=fake, ldg=4, D=fake, R0=fake, ldr=4, K=4, B=1, I=1, gamma=0.5,
                               sel=fake, proj=fake, coef=fake, ldo=1, R_out=fake)
    assert lib.fase_iterate_scaled(ctypes.byref(args), None, None) == -8
    syn = _native.SynthFused(phi=fake, ldphi=3, n_lost=3, out=fake, ldout=3)  # odd ldphi
    args = _native.IterateArgs(G0=fake, ldg=4, D=fake, R0=fake, ldr=4, K=4, B=1, I=1, gamma=0.5,
                               sel=fake, proj=fake, coef=fake, ldo=1)
    assert lib.fase_iterate_scaled(ctypes.byref(args), ctypes.byref(syn), None) == -1
    assert b"fused-synthesis" in lib.fase_last_error()
    assert lib.fase_iterate_scaled_synth_capacity(4608, 1024) >= 256
    assert lib.fase_iterate_scaled_synth_capacity(0, 1) == 0
    assert lib.fase_scale_columns(None, 4, None, 4, 4, None, 4, None) == -1
    assert lib.fase_scale_columns(fake, 4, fake, 4, 4, fake, 5, None) == -1  # odd lds
    # empty batches are a no-op, not an error
    args = _native.IterateArgs(K=4, B=0, I=1, gamma=0.5)
    assert lib.fase_iterate(ctypes.byref(args), None) == 0
    assert lib.fase_iterate_scaled(ctypes.byref(args), None, None) == 0
    assert lib.fase_iterate_complex_scaled(ctypes.byref(args), None) == 0
    assert lib.fase_iterate_complex_scaled(None, None) == -2
    assert lib.fase_ozaki_gemm(None, 128, None, 0, None, 64, None, 50, 64, 8, None, 50, None) == 0


def test_status_maps_to_reference_exceptions(lib):
    assert _native._STATUS[-1] is errors.ShapeError
    assert _native._STATUS[-2] is errors.ParameterError
    assert _native._STATUS[-6] is errors.NoSelectableAtomError
    assert _native._STATUS[-7] is errors.StaleTableError
    assert all(issubclass(c, ValueError) for c in _native._STATUS.values())
    lib.fase_iterate(None, None)
    with pytest.raises(errors.ParameterError):
        _native._check(-2)


def test_iterate_args_layout_matches_header():
    # the ctypes mirror must have the header's field order
    text = HEADER.read_text()
    end = text.index("} fase_iterate_args;")
    body = text[text.rindex("typedef struct {", 0, end):end]
    fields = re.findall(r"\b(\w+);", body)
    assert fields == [f for f, _ in _native.IterateArgs._fields_]


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    monkeypatch.setattr(_native, "_lib", None)
    monkeypatch.setenv("FASE_B200_LIB", str(tmp_path / "nope.so"))
    with pytest.raises(errors.NativeLibraryError):
        _native.load()
