"""ctypes binding of libfase_b200.so (the C ABI in include/fase_b200.h).

torch tensors are used as device buffers only: this module passes raw
``data_ptr()`` values, leading dimensions and the current CUDA stream. A
missing or unloadable library raises NativeLibraryError -- there is no CPU or
eager fallback for any entry point.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

from . import errors

_LIB_PATH = Path(__file__).resolve().parent / "libfase_b200.so"
_lib = None

_STATUS = {
    -1: errors.ShapeError,
    -2: errors.ParameterError,
    -3: errors.MaskError,
    -4: errors.FormatError,
    -5: errors.DegenerateAtomError,
    -6: errors.NoSelectableAtomError,
    -7: errors.StaleTableError,
    -8: errors.UnsupportedDictionaryError,
}

EXPORTS = (
    "fase_last_error", "fase_abi_version", "fase_max_atoms", "fase_table_ld", "fase_basis_outer",
    "fase_gram", "fase_gram_workspace", "fase_gemm_nt", "fase_init_products_workspace",
    "fase_gram_finish", "fase_init_products", "fase_block_normalizers", "fase_iterate",
    "fase_synth_paste", "fase_l2_flush", "fase_frame_areas", "fase_frame_cells",
    "fase_frame_paste", "fase_weigh", "fase_sep_products", "fase_gram_complex_workspace",
    "fase_gram_complex", "fase_max_atoms_complex", "fase_table_ld_complex", "fase_iterate_complex",
    "fase_synth_paste_complex", "fase_sep_products_complex", "fase_fft_gram", "fase_weigh_gather",
    "fase_ozaki_split", "fase_ozaki_split_sparse", "fase_ozaki_gemm", "fase_ozaki_gram", "fase_sep_products_batch",
    "fase_iterate_scaled", "fase_scale_columns", "fase_iterate_scaled_synth_capacity",
    "fase_iterate_complex_scaled", "fase_frame_widen", "fase_frame_paste_complex",
    "fase_iterate_synth", "fase_iterate_synth_capacity", "fase_block_order",
    "fase_iterate_register_atoms", "fase_iterate_complex_register_atoms", "fase_mirror_upper",
)

ABI_MAJOR = 3  # fase_abi_version() >> 16 of the library this binding matches
_vp = ctypes.c_void_p
_i32 = ctypes.c_int
_i64 = ctypes.c_int64
_f64 = ctypes.c_double


class SepPart(ctypes.Structure):
    """Mirror of ``fase_sep_part`` (include/fase_b200.h)."""

    _fields_ = [("rows", _vp), ("Lr", _i32), ("cols", _vp), ("Lc", _i32), ("col0", _i64)]


class SynthFused(ctypes.Structure):
    """Mirror of ``fase_synth_fused`` (include/fase_b200.h)."""

    _fields_ = [("phi", _vp), ("ldphi", _i64), ("n_lost", _i32), ("out", _vp), ("ldout", _i64)]


class IterateArgs(ctypes.Structure):
    """Mirror of ``fase_iterate_args`` (include/fase_b200.h)."""

    _fields_ = [
        ("G0", _vp), ("ldg", _i64), ("chunk_tables", _vp), ("chunk_stride", _i64),
        ("chunk_count", _vp), ("chunk_ids", _vp), ("chunk_list_ld", _i64), ("D", _vp),
        ("ldd", _i64), ("R0", _vp),
        ("ldr", _i64), ("R_out", _vp), ("R_log", _vp), ("K", _i32), ("B", _i32), ("I", _i32),
        ("gamma", _f64), ("sel", _vp), ("proj", _vp), ("coef", _vp), ("ldo", _i64),
        ("compose", _vp), ("n_compose", _i32), ("compose_depth", _i32), ("base_stride", _i64),
        ("l2_hot", _vp), ("order", _vp),
    ]


def library_path() -> Path:
    return Path(os.environ.get("FASE_B200_LIB", _LIB_PATH))


def load():
    """Load the shared library once; NativeLibraryError if it is absent or broken."""
    global _lib
    if _lib is not None:
        return _lib
    path = library_path()
    if not path.exists():
        raise errors.NativeLibraryError(
            f"{path} is missing: run `python -m paper_2204_14194_b200._build` "
            "(or __graft_entry__.build()) -- there is no CPU fallback")
    try:
        lib = ctypes.CDLL(str(path))
    except OSError as exc:
        raise errors.NativeLibraryError(f"cannot load {path}: {exc}") from exc
    lib.fase_last_error.restype = ctypes.c_char_p
    lib.fase_last_error.argtypes = []
    lib.fase_abi_version.restype = _i32
    if lib.fase_abi_version() >> 16 != ABI_MAJOR:  # IterateArgs must match the library's struct
        raise errors.NativeLibraryError(
            f"{path}: ABI {lib.fase_abi_version() >> 16}.{lib.fase_abi_version() & 0xffff}, this "
            f"package needs {ABI_MAJOR}.x: rebuild with `python -m paper_2204_14194_b200._build`")
    lib.fase_max_atoms.restype = _i32
    lib.fase_iterate_register_atoms.restype = _i32
    lib.fase_iterate_complex_register_atoms.restype = _i32
    lib.fase_table_ld.restype = _i32
    lib.fase_table_ld.argtypes = [_i32]
    lib.fase_gram_workspace.restype = ctypes.c_size_t
    lib.fase_gram_workspace.argtypes = [_i32, _i32]
    lib.fase_init_products_workspace.restype = ctypes.c_size_t
    lib.fase_init_products_workspace.argtypes = [_i32, _i32]
    lib.fase_gram_complex_workspace.restype = ctypes.c_size_t
    lib.fase_gram_complex_workspace.argtypes = [_i32, _i64]
    lib.fase_max_atoms_complex.restype = _i32
    lib.fase_table_ld_complex.restype = _i32
    lib.fase_table_ld_complex.argtypes = [_i32]
    sigs = {
        "fase_basis_outer": [_vp, _i32, _i32, _vp, _i32, _i32, _vp, _i64, _i64, _vp],
        "fase_gram": [_vp, _i64, _vp, _i32, _i32, _vp, _i64, _vp, ctypes.c_size_t, _vp],
        "fase_gemm_nt": [_vp, _i64, _vp, _i64, _i32, _i32, _i32, _vp, _i64, _i32, _vp],
        "fase_gram_finish": [_vp, _i64, _i32, _vp, _vp, _vp],
        "fase_init_products": [_vp, _i64, _vp, _i64, _vp, _i64, _i32, _i32, _i32, _vp, _i64, _vp,
                               ctypes.c_size_t, _vp],
        "fase_block_normalizers": [_vp, _i64, _vp, _i64, _vp, _vp, _i64, _i32, _i32, _vp, _i64,
                                   _vp, _vp],
        "fase_iterate": [ctypes.POINTER(IterateArgs), _vp],
        "fase_iterate_scaled": [ctypes.POINTER(IterateArgs), ctypes.POINTER(SynthFused), _vp],
        "fase_iterate_scaled_synth_capacity": [_i32, _i32],
        "fase_iterate_synth": [ctypes.POINTER(IterateArgs), ctypes.POINTER(SynthFused), _vp],
        "fase_iterate_synth_capacity": [_i32, _i32],
        "fase_scale_columns": [_vp, _i64, _vp, _i32, _i32, _vp, _i64, _vp],
        "fase_iterate_complex_scaled": [ctypes.POINTER(IterateArgs), _vp],
        "fase_iterate_complex": [ctypes.POINTER(IterateArgs), _vp],
        "fase_gram_complex": [_vp, _i64, _vp, _i32, _i32, _vp, _i64, _vp, ctypes.c_size_t, _vp],
        "fase_synth_paste_complex": [_vp, _i64, _vp, _vp, _i64, _i32, _i32, _vp, _vp, _i32, _vp,
                                     _vp, _i64, _vp, _vp],
        "fase_sep_products_complex": [_vp, _vp, _i32, _i32, _vp, _vp, _i32, _i32, _vp, _i64, _i32,
                                      _vp, _i64, _i64, _vp],
        "fase_fft_gram": [_vp, _i32, _i32, _vp, _vp, _i32, _vp, _i64, _vp],
        "fase_weigh_gather": [_vp, _i64, _vp, _vp, _i32, _i32, _vp, _i64, _vp],
        "fase_sep_products_batch": [ctypes.POINTER(SepPart), _i32, _i32, _i32, _vp, _i64, _vp,
                                    _i64, _i32, _vp, _i64, _vp],
        "fase_ozaki_split": [_vp, _i64, _vp, _vp, _i32, _i32, _i32, _vp, _i64, _i32, _vp, _vp],
        "fase_ozaki_split_sparse": [_vp, _i64, _vp, _i64, _i32, _i32, _i32, _i32, _vp, _i64, _i32,
                                    _vp, _vp],
        "fase_ozaki_gemm": [_vp, _i32, _vp, _i32, _vp, _i32, _vp, _i32, _i64, _i32, _vp, _i64,
                            _vp],
        "fase_ozaki_gram": [_vp, _i32, _vp, _vp, _i32, _vp, _i32, _i64, _i32, _vp, _i64, _vp],
        "fase_synth_paste": [_vp, _i64, _vp, _vp, _i64, _i32, _i32, _vp, _vp, _i32, _vp, _vp,
                             _i64, _vp],
        "fase_l2_flush": [_vp, ctypes.c_size_t, _vp],
        "fase_weigh": [_vp, _i64, _vp, _i64, _i32, _i32, _vp, _i64, _vp],
        "fase_sep_products": [_vp, _i32, _i32, _vp, _i32, _i32, _vp, _i64, _i32, _vp, _i64, _i64,
                              _vp],
        "fase_frame_areas": [_vp, _i64, _vp, _i64, _i32, _i32, _i32, _i32, _vp, _i32, _vp, _vp,
                             _i64, _vp],
        "fase_frame_cells": [_vp, _i64, _i32, _i32, _i32, _i32, _vp, _i32, _vp, _i32, _vp, _vp,
                             _i64, _vp],
        "fase_frame_paste": [_vp, _i64, _vp, _vp, _i64, _i32, _vp, _i64, _i32, _i32, _i32, _i32,
                             _vp, _i32, _vp, _i64, _vp],
        "fase_frame_widen": [_vp, _i64, _vp, _i64, _i32, _i32, _vp, _i64, _vp],
        "fase_block_order": [_vp, _i32, _i32, _vp, _vp],
        "fase_mirror_upper": [_vp, _i64, _i32, _vp],
        "fase_frame_paste_complex": [_vp, _i64, _vp, _vp, _i64, _i32, _vp, _i64, _i32, _i32, _i32,
                                     _i32, _vp, _i32, _vp, _i64, _vp, _vp],
    }
    for name, args in sigs.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = _i32
    _lib = lib
    return lib


def _check(status: int) -> None:
    if status == 0:
        return
    msg = _lib.fase_last_error().decode("utf-8", "replace")
    cls = _STATUS.get(status)
    if cls is None:
        raise errors.NativeLibraryError(f"libfase_b200 status {status}: {msg}")
    raise cls(msg)


def _stream(tensor) -> int:
    import torch

    return torch.cuda.current_stream(tensor.device).cuda_stream


def _ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def _require(t, name, dtype=None, ndim=None):
    import torch

    if t is None:
        raise errors.ShapeError(f"{name} is required")
    if not t.is_cuda:
        raise errors.NativeLibraryError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if dtype is not None and t.dtype != dtype:
        raise errors.ShapeError(f"{name} must be {dtype}, got {t.dtype}")
    if ndim is not None and t.dim() != ndim:
        raise errors.ShapeError(f"{name} must be {ndim}-D, got shape {tuple(t.shape)}")
    if t.dim() >= 1 and t.stride(-1) != 1:
        raise errors.ShapeError(f"{name} must be contiguous in its last dimension")
    return t


def _ld(t) -> int:
    return t.stride(0) if t.dim() == 2 else 0


# ----------------------------------------------------------------- entry points


def basis_outer(rows, cols, phi, row0: int) -> None:
    import torch

    lib = load()
    _require(rows, "rows", torch.float64, 2)
    _require(cols, "cols", torch.float64, 2)
    _require(phi, "phi", torch.float64, 2)
    lr, mr = rows.shape
    lc, nc = cols.shape
    _check(lib.fase_basis_outer(_ptr(rows), lr, mr, _ptr(cols), lc, nc, _ptr(phi), _ld(phi),
                                row0, _stream(phi)))


def _workspace(nbytes: int, device, ws=None):
    """A 16-byte-aligned device scratch of at least ``nbytes`` (reused when given)."""
    import torch

    if ws is not None and ws.numel() * ws.element_size() >= nbytes:
        return ws
    return torch.empty(max(nbytes // 8, 2), dtype=torch.float64, device=device)


def gram(phi, w, K: int, M: int, G, ws=None) -> None:
    import torch

    lib = load()
    _require(phi, "phi", torch.float64, 2)
    _require(w, "w", torch.float64, 1)
    _require(G, "G", torch.float64, 2)
    need = int(lib.fase_gram_workspace(K, M))
    ws = _workspace(need, G.device, ws)
    _check(lib.fase_gram(_ptr(phi), _ld(phi), _ptr(w), K, M, _ptr(G), _ld(G), _ptr(ws),
                         ws.numel() * 8, _stream(G)))


def init_products_workspace(M: int, B: int) -> int:
    return int(load().fase_init_products_workspace(M, B))


def gemm_nt(A, B, C, variant: int = 0) -> None:
    """C = A @ B.T in FP64 (all 2-D, contiguous rows)."""
    import torch

    lib = load()
    for t, n in ((A, "A"), (B, "B"), (C, "C")):
        _require(t, n, torch.float64, 2)
    _check(lib.fase_gemm_nt(_ptr(A), _ld(A), _ptr(B), _ld(B), A.shape[0], B.shape[0], A.shape[1],
                            _ptr(C), _ld(C), variant, _stream(C)))


def gram_finish(G, K: int, D, n_alive=None) -> None:
    import torch

    lib = load()
    _require(G, "G", torch.float64, 2)
    _require(D, "D", torch.float64, 1)
    _check(lib.fase_gram_finish(_ptr(G), _ld(G), K, _ptr(D), _ptr(n_alive), _stream(G)))


def init_products(phi, f, w, K: int, M: int, R0, ws=None) -> None:
    """R0[b] = (f[b] o w[b or shared]) @ phi.T ; f, R0 2-D; w 1-D (shared) or 2-D."""
    import torch

    lib = load()
    _require(phi, "phi", torch.float64, 2)
    _require(f, "f", torch.float64, 2)
    _require(w, "w", torch.float64)
    _require(R0, "R0", torch.float64, 2)
    ldw = _ld(w) if w.dim() == 2 else 0
    B = f.shape[0]
    ws = _workspace(int(lib.fase_init_products_workspace(M, B)), R0.device, ws)
    _check(lib.fase_init_products(_ptr(phi), _ld(phi), _ptr(f), _ld(f), _ptr(w), ldw, K, M, B,
                                  _ptr(R0), _ld(R0), _ptr(ws), ws.numel() * 8, _stream(R0)))


def block_normalizers(G0, chunk_tables, chunk_stride: int, chunk_count, chunk_ids, K: int,
                      D, n_alive) -> None:
    """D of B per-block geometries; chunk_ids is (B, L) with chunk_count[b] valid entries.
    ``G0`` 1-D: the tables are given as their diagonals (G0 (K,), chunk_tables
    (n, chunk_stride) rows of diagonals), read contiguously."""
    import torch

    lib = load()
    _require(G0, "G0", torch.float64)
    _require(D, "D", torch.float64, 2)
    list_ld = _ld(chunk_ids) if chunk_ids is not None else 0
    _check(lib.fase_block_normalizers(_ptr(G0), _ld(G0), _ptr(chunk_tables), chunk_stride,
                                      _ptr(chunk_count), _ptr(chunk_ids), list_ld, K, D.shape[0],
                                      _ptr(D), _ld(D), _ptr(n_alive), _stream(D)))


def _hot_ptr(l2_hot, K: int):
    """Device pointer of an L2 hot-row mask (int32 words, bit u of word u // 32), or None."""
    import torch

    if l2_hot is None:
        return None
    _require(l2_hot, "l2_hot", torch.int32, 1)
    if l2_hot.numel() * 32 < K:
        raise errors.ShapeError(f"l2_hot holds {l2_hot.numel() * 32} bits, K = {K}")
    return _ptr(l2_hot)


def synth_capacity(K: int, B: int) -> int:
    """Lost samples the exact recursion with fused synthesis can carry (0: n/a)."""
    return int(load().fase_iterate_synth_capacity(K, B))


def _order_ptr(order, B: int):
    import torch

    if order is None:
        return None
    _require(order, "order", torch.int32, 1)
    if order.shape[0] != B:
        raise errors.ShapeError(f"order must hold one entry per block ({B}), got {order.shape[0]}")
    return _ptr(order)


def mirror_upper(G, K: int) -> None:
    """G[i, j] <- G[j, i] for i > j (fase_mirror_upper), in place."""
    import torch

    lib = load()
    _require(G, "G", torch.float64, 2)
    _check(lib.fase_mirror_upper(_ptr(G), _ld(G), K, _stream(G)))


def block_order(counts, depth: int, order) -> None:
    """order <- blocks by descending cost class min(7, max(0, counts - depth)),
    stable (fase_block_order): the dispatch order of a chunked recursion."""
    import torch

    lib = load()
    _require(counts, "counts", torch.int32, 1)
    _require(order, "order", torch.int32, 1)
    if order.shape[0] != counts.shape[0]:
        raise errors.ShapeError("order and counts must have one entry per block")
    _check(lib.fase_block_order(_ptr(counts), counts.shape[0], depth, _ptr(order),
                                _stream(counts)))


def iterate(G0, D, R0, K: int, iterations: int, gamma: float, sel, proj, coef, *,
            chunk_tables=None, chunk_stride: int = 0, chunk_count=None, chunk_ids=None,
            R_out=None, R_log=None, compose=None, base_stride: int = 0, l2_hot=None,
            phi_lost=None, n_lost: int = 0, lost=None, order=None) -> None:
    """The recursion (fase_iterate). ``compose`` (int32 device table n^depth,
    depth 1..3) with ``base_stride`` selects precomposed base tables at
    G0 + p * base_stride for the longest prefix of each block's chunk list.
    ``order`` (int32 (B,) device permutation, optional): CTA i runs block
    order[i] (a schedule only; ``block_order``)."""
    import torch

    lib = load()
    _require(G0, "G0", torch.float64, 2)
    _require(D, "D", torch.float64)
    _require(R0, "R0", torch.float64, 2)
    _require(sel, "sel", torch.int32, 2)
    _require(proj, "proj", torch.float64, 2)
    _require(coef, "coef", torch.float64, 2)
    if R_out is None and phi_lost is None and K > register_atoms():
        # beyond the registers the streaming recursion works in R_out
        R_out = torch.empty_like(R0)
    args = IterateArgs(
        G0=_ptr(G0), ldg=_ld(G0), chunk_tables=_ptr(chunk_tables), chunk_stride=chunk_stride,
        chunk_count=_ptr(chunk_count), chunk_ids=_ptr(chunk_ids),
        chunk_list_ld=_ld(chunk_ids) if chunk_ids is not None else 0, D=_ptr(D),
        ldd=_ld(D) if D.dim() == 2 else 0, R0=_ptr(R0), ldr=_ld(R0), R_out=_ptr(R_out),
        R_log=_ptr(R_log), K=K, B=R0.shape[0], I=iterations, gamma=gamma, sel=_ptr(sel),
        proj=_ptr(proj), coef=_ptr(coef), ldo=_ld(sel), compose=_ptr(compose),
        n_compose=compose.shape[0] if compose is not None else 0,
        compose_depth=compose.dim() if compose is not None else 0, base_stride=base_stride,
        l2_hot=_hot_ptr(l2_hot, K), order=_order_ptr(order, R0.shape[0]))
    if compose is not None:
        _require(compose, "compose", torch.int32)
        if compose.dim() > 3 or any(x != compose.shape[0] for x in compose.shape):
            raise errors.ShapeError("compose must be an n, n x n or n x n x n table")
    if proj.stride(0) != args.ldo or coef.stride(0) != args.ldo:
        raise errors.ShapeError("sel / proj / coef must share one leading dimension")
    if phi_lost is not None:  # the synthesis fused in (fase_iterate_synth)
        _require(phi_lost, "phi_lost", torch.float64, 2)
        _require(lost, "lost", torch.float64, 2)
        syn = SynthFused(phi=_ptr(phi_lost), ldphi=_ld(phi_lost), n_lost=n_lost, out=_ptr(lost),
                         ldout=_ld(lost))
        _check(lib.fase_iterate_synth(ctypes.byref(args), ctypes.byref(syn), _stream(R0)))
        return
    _check(lib.fase_iterate(ctypes.byref(args), _stream(R0)))


def scale_columns(G, D, K: int, Gs) -> None:
    """Gs[u, k] = G[u, k] * D[k] (fase_scale_columns): the scaled recursion's
    table. Complex tables (rows of conj(C), complex128) are scaled as their real
    view with D repeated per (re, im) pair."""
    import torch

    lib = load()
    if G.is_complex():
        _require(G, "G", torch.complex128, 2)
        _require(Gs, "Gs", torch.complex128, 2)
        _require(D, "D", torch.float64, 1)
        Gr, Gsr = torch.view_as_real(G).reshape(G.shape[0], -1), \
            torch.view_as_real(Gs).reshape(Gs.shape[0], -1)
        D2 = D[:K].repeat_interleave(2).contiguous()
        if Gs.shape[0] < K:
            raise errors.ShapeError(f"Gs has {Gs.shape[0]} rows, need {K}")
        _check(lib.fase_scale_columns(_ptr(Gr), Gr.stride(0), _ptr(D2), K, 2 * K, _ptr(Gsr),
                                      Gsr.stride(0), _stream(Gs)))
        return
    _require(G, "G", torch.float64, 2)
    _require(D, "D", torch.float64, 1)
    _require(Gs, "Gs", torch.float64, 2)
    if Gs.shape[0] < K:
        raise errors.ShapeError(f"Gs has {Gs.shape[0]} rows, need {K}")
    _check(lib.fase_scale_columns(_ptr(G), _ld(G), _ptr(D), K, K, _ptr(Gs), _ld(Gs), _stream(Gs)))


def iterate_complex_scaled(Gs, D, R0, K: int, iterations: int, gamma: float, sel, proj,
                           coef) -> None:
    """The complex scaled recursion (fase_iterate_complex_scaled) over the
    column-scaled complex table ``Gs``; R0 (B, ldr) complex128, D unscaled."""
    import torch

    lib = load()
    _require(Gs, "Gs", torch.complex128, 2)
    _require(D, "D", torch.float64, 1)
    _require(R0, "R0", torch.complex128, 2)
    _require(sel, "sel", torch.int32, 2)
    _require(proj, "proj", torch.complex128, 2)
    _require(coef, "coef", torch.complex128, 2)
    args = IterateArgs(G0=_ptr(Gs), ldg=_ld(Gs), D=_ptr(D), ldd=0, R0=_ptr(R0), ldr=_ld(R0), K=K,
                       B=R0.shape[0], I=iterations, gamma=gamma, sel=_ptr(sel), proj=_ptr(proj),
                       coef=_ptr(coef), ldo=_ld(sel))
    if proj.stride(0) != args.ldo or coef.stride(0) != args.ldo:
        raise errors.ShapeError("sel / proj / coef must share one leading dimension")
    _check(lib.fase_iterate_complex_scaled(ctypes.byref(args), _stream(R0)))


def scaled_synth_capacity(K: int, B: int) -> int:
    """Most lost samples the scaled recursion can synthesize in-kernel for (K, B)."""
    return int(load().fase_iterate_scaled_synth_capacity(K, B))


def iterate_scaled(Gs, D, R0, K: int, iterations: int, gamma: float, sel, proj, coef, *,
                   phi_lost=None, n_lost: int = 0, lost=None, l2_hot=None) -> None:
    """The scaled recursion (fase_iterate_scaled) over a column-scaled shared
    table ``Gs`` (scale_columns); R0 and D unscaled, as for ``iterate``.
    With ``phi_lost`` (K, ld) and ``lost`` (B, >= n_lost) the synthesis of the
    n_lost packed lost samples is fused in (bit-identical to synth_paste)."""
    import torch

    lib = load()
    _require(Gs, "Gs", torch.float64, 2)
    _require(D, "D", torch.float64, 1)
    _require(R0, "R0", torch.float64, 2)
    _require(sel, "sel", torch.int32, 2)
    _require(proj, "proj", torch.float64, 2)
    _require(coef, "coef", torch.float64, 2)
    args = IterateArgs(G0=_ptr(Gs), ldg=_ld(Gs), D=_ptr(D), ldd=0, R0=_ptr(R0), ldr=_ld(R0), K=K,
                       B=R0.shape[0], I=iterations, gamma=gamma, sel=_ptr(sel), proj=_ptr(proj),
                       coef=_ptr(coef), ldo=_ld(sel), l2_hot=_hot_ptr(l2_hot, K))
    if proj.stride(0) != args.ldo or coef.stride(0) != args.ldo:
        raise errors.ShapeError("sel / proj / coef must share one leading dimension")
    syn = None
    if phi_lost is not None:
        _require(phi_lost, "phi_lost", torch.float64, 2)
        _require(lost, "lost", torch.float64, 2)
        syn = ctypes.byref(SynthFused(phi=_ptr(phi_lost), ldphi=_ld(phi_lost), n_lost=n_lost,
                                      out=_ptr(lost), ldout=_ld(lost)))
    _check(lib.fase_iterate_scaled(ctypes.byref(args), syn, _stream(R0)))


def synth_paste(phi, sel, coef, iterations: int, idx, out, *, idx_ptr=None, n_shared: int = 0,
                dst=None) -> None:
    import torch

    lib = load()
    _require(phi, "phi", torch.float64, 2)
    _require(idx, "idx", torch.int32, 1)
    _require(out, "out", torch.float64)
    B = sel.shape[0]
    ldout = _ld(out) if out.dim() == 2 else 0
    _check(lib.fase_synth_paste(_ptr(phi), _ld(phi), _ptr(sel), _ptr(coef), _ld(sel), iterations,
                                B, _ptr(idx_ptr), _ptr(idx), n_shared, _ptr(dst), _ptr(out),
                                ldout, _stream(out)))


# ---- complex dictionaries: phi2 is the (2K, ld) conjugate-split matrix; tables,
# products, projections and coefficients are complex128 tensors whose leading
# dimensions count complex elements.


def _require_complex(t, name, ndim=None):
    import torch

    return _require(t, name, torch.complex128, ndim)


def gram_complex(phi2, w, K: int, M: int, T, ws=None) -> None:
    """T[u, l] = conj(C[u, l]) with C = conj(Phi) W Phi^T (T: complex128 (K, ldt))."""
    import torch

    lib = load()
    _require(phi2, "phi2", torch.float64, 2)
    _require(w, "w", torch.float64, 1)
    _require_complex(T, "T", 2)
    need = int(lib.fase_gram_complex_workspace(K, _ld(phi2)))
    ws = _workspace(need, T.device, ws)
    _check(lib.fase_gram_complex(_ptr(phi2), _ld(phi2), _ptr(w), K, M, _ptr(T), _ld(T), _ptr(ws),
                                 ws.numel() * 8, _stream(T)))


def gram_finish_complex(T, K: int, D, n_alive=None) -> None:
    """D from the (real) diagonal of a complex table."""
    import torch

    lib = load()
    _require_complex(T, "T", 2)
    _require(D, "D", torch.float64, 1)
    _check(lib.fase_gram_finish(_ptr(T), 2 * _ld(T) + 1, K, _ptr(D), _ptr(n_alive), _stream(T)))


def block_normalizers_complex(T0, chunk_tables, chunk_stride: int, chunk_count, chunk_ids, K: int,
                              D, n_alive) -> None:
    """Per-block D of complex chunked tables (chunk_stride in complex elements)."""
    import torch

    lib = load()
    _require_complex(T0, "T0", 2)
    _require(D, "D", torch.float64, 2)
    list_ld = _ld(chunk_ids) if chunk_ids is not None else 0
    _check(lib.fase_block_normalizers(_ptr(T0), 2 * _ld(T0) + 1, _ptr(chunk_tables),
                                      2 * chunk_stride, _ptr(chunk_count), _ptr(chunk_ids),
                                      list_ld, K, D.shape[0], _ptr(D), _ld(D), _ptr(n_alive),
                                      _stream(D)))


def iterate_complex(T, D, R0, K: int, iterations: int, gamma: float, sel, proj, coef, *,
                    chunk_tables=None, chunk_stride: int = 0, chunk_count=None, chunk_ids=None,
                    R_out=None, R_log=None, compose=None, base_stride: int = 0,
                    order=None) -> None:
    import torch

    lib = load()
    _require_complex(T, "T", 2)
    _require(D, "D", torch.float64)
    _require_complex(R0, "R0", 2)
    _require(sel, "sel", torch.int32, 2)
    _require_complex(proj, "proj", 2)
    _require_complex(coef, "coef", 2)
    if R_out is None and K > register_atoms_complex():
        # beyond the registers the streaming recursion works in R_out
        R_out = torch.empty_like(R0)
    args = IterateArgs(
        G0=_ptr(T), ldg=_ld(T), chunk_tables=_ptr(chunk_tables), chunk_stride=chunk_stride,
        chunk_count=_ptr(chunk_count), chunk_ids=_ptr(chunk_ids),
        chunk_list_ld=_ld(chunk_ids) if chunk_ids is not None else 0, D=_ptr(D),
        ldd=_ld(D) if D.dim() == 2 else 0, R0=_ptr(R0), ldr=_ld(R0), R_out=_ptr(R_out),
        R_log=_ptr(R_log), K=K, B=R0.shape[0], I=iterations, gamma=gamma, sel=_ptr(sel),
        proj=_ptr(proj), coef=_ptr(coef), ldo=_ld(sel), compose=_ptr(compose),
        n_compose=compose.shape[0] if compose is not None else 0,
        compose_depth=compose.dim() if compose is not None else 0, base_stride=base_stride,
        order=_order_ptr(order, R0.shape[0]))
    if compose is not None:
        _require(compose, "compose", torch.int32)
        if compose.dim() > 3 or any(x != compose.shape[0] for x in compose.shape):
            raise errors.ShapeError("compose must be an n, n x n or n x n x n table")
    if proj.stride(0) != args.ldo or coef.stride(0) != args.ldo:
        raise errors.ShapeError("sel / proj / coef must share one leading dimension")
    _check(lib.fase_iterate_complex(ctypes.byref(args), _stream(R0)))


def synth_paste_complex(phi2, sel, coef, iterations: int, idx, out, *, idx_ptr=None,
                        n_shared: int = 0, dst=None, max_imag=None) -> None:
    import torch

    lib = load()
    _require(phi2, "phi2", torch.float64, 2)
    _require(idx, "idx", torch.int32, 1)
    _require(out, "out", torch.float64)
    _require_complex(coef, "coef", 2)
    B = sel.shape[0]
    ldout = _ld(out) if out.dim() == 2 else 0
    _check(lib.fase_synth_paste_complex(_ptr(phi2), _ld(phi2), _ptr(sel), _ptr(coef), _ld(sel),
                                        iterations, B, _ptr(idx_ptr), _ptr(idx), n_shared,
                                        _ptr(dst), _ptr(out), ldout, _ptr(max_imag),
                                        _stream(out)))


def sep_products_complex(rows_re, rows_im, cols_re, cols_im, X, M_rows: int, N_cols: int, R0,
                         col0: int) -> None:
    """R0[b, col0 + u*Lc + v] = (conj(E) X_b conj(F)^T)[u, v], E = rows_re + i rows_im,
    F = cols_re + i cols_im (R0 complex128)."""
    import torch

    lib = load()
    for t, n in ((rows_re, "rows_re"), (rows_im, "rows_im"), (cols_re, "cols_re"),
                 (cols_im, "cols_im"), (X, "X")):
        _require(t, n, torch.float64, 2)
    _require_complex(R0, "R0", 2)
    _check(lib.fase_sep_products_complex(_ptr(rows_re), _ptr(rows_im), rows_re.shape[0], M_rows,
                                         _ptr(cols_re), _ptr(cols_im), cols_re.shape[0], N_cols,
                                         _ptr(X), _ld(X), X.shape[0], _ptr(R0), _ld(R0), col0,
                                         _stream(R0)))


def fft_gram(spec, M: int, N: int, mu, eta, K: int, T) -> None:
    """Complex table rows conj(C) gathered from the spectrum of the weight
    (spec: complex128 (M*N,) or (1, M*N)); mu/eta int32 tags or None (canonical)."""
    lib = load()
    _require_complex(T, "T", 2)
    _check(lib.fase_fft_gram(_ptr(spec), M, N, _ptr(mu), _ptr(eta), K, _ptr(T), _ld(T),
                             _stream(T)))


def max_atoms_complex() -> int:
    return int(load().fase_max_atoms_complex())


def register_atoms_complex() -> int:
    """Largest complex K whose recursion keeps R in registers."""
    return int(load().fase_iterate_complex_register_atoms())


def table_ld_complex(K: int) -> int:
    ld = int(load().fase_table_ld_complex(K))
    if ld <= 0:
        raise errors.UnsupportedDictionaryError(f"K={K} exceeds the complex iteration kernel's "
                                                f"{max_atoms_complex()} atoms")
    return ld


def frame_areas(frame, grid, tile: int, support: int, corners, base_w, X) -> None:
    import torch

    lib = load()
    _require(frame, "frame", torch.float64, 2)
    _require(grid, "grid", torch.uint8, 2)
    _require(corners, "corners", torch.int32, 2)
    _require(base_w, "base_w", torch.float64, 1)
    _require(X, "X", torch.float64, 2)
    H, W = frame.shape
    _check(lib.fase_frame_areas(_ptr(frame), _ld(frame), _ptr(grid), _ld(grid), H, W, tile,
                                support, _ptr(corners), corners.shape[0], _ptr(base_w), _ptr(X),
                                _ld(X), _stream(X)))


def frame_cells(grid, H: int, W: int, tile: int, support: int, corners, cell_rep, counts,
                ids) -> None:
    import torch

    lib = load()
    _require(grid, "grid", torch.uint8, 2)
    _require(corners, "corners", torch.int32, 2)
    _require(cell_rep, "cell_rep", torch.int32, 2)
    _require(counts, "counts", torch.int32, 1)
    _require(ids, "ids", torch.int32, 2)
    _check(lib.fase_frame_cells(_ptr(grid), _ld(grid), H, W, tile, support, _ptr(corners),
                                corners.shape[0], _ptr(cell_rep), cell_rep.shape[0],
                                _ptr(counts), _ptr(ids), _ld(ids), _stream(ids)))


def frame_paste(phi, sel, coef, iterations: int, grid, tile: int, support: int, corners,
                out) -> None:
    import torch

    lib = load()
    _require(phi, "phi", torch.float64, 2)
    _require(out, "out", torch.float64, 2)
    H, W = out.shape
    _check(lib.fase_frame_paste(_ptr(phi), _ld(phi), _ptr(sel), _ptr(coef), _ld(sel), iterations,
                                _ptr(grid), _ld(grid), H, W, tile, support, _ptr(corners),
                                corners.shape[0], _ptr(out), _ld(out), _stream(out)))


def frame_paste_complex(phi2, sel, coef, iterations: int, grid, tile: int, support: int,
                        corners, out, max_imag=None) -> None:
    import torch

    lib = load()
    _require(phi2, "phi2", torch.float64, 2)
    _require(out, "out", torch.float64, 2)
    _require_complex(coef, "coef", 2)
    H, W = out.shape
    _check(lib.fase_frame_paste_complex(_ptr(phi2), _ld(phi2), _ptr(sel), _ptr(coef), _ld(sel),
                                        iterations, _ptr(grid), _ld(grid), H, W, tile, support,
                                        _ptr(corners), corners.shape[0], _ptr(out), _ld(out),
                                        _ptr(max_imag), _stream(out)))


def frame_widen(frame_u8, lost, out) -> None:
    """out = lost ? 0 : float64(frame_u8) (H x W; lost bool / uint8, nonzero = lost)."""
    import torch

    lib = load()
    _require(frame_u8, "frame_u8", torch.uint8, 2)
    _require(out, "out", torch.float64, 2)
    if not lost.is_cuda:
        raise errors.NativeLibraryError("lost must be a CUDA tensor (no CPU fallback)")
    if lost.dtype not in (torch.bool, torch.uint8) or lost.dim() != 2 or lost.stride(1) != 1:
        raise errors.ShapeError("lost must be a row-major (H, W) bool / uint8 tensor")
    H, W = out.shape
    if tuple(frame_u8.shape) != (H, W) or tuple(lost.shape) != (H, W):
        raise errors.ShapeError(f"frame {tuple(frame_u8.shape)} / lost {tuple(lost.shape)} vs {(H, W)}")
    _check(lib.fase_frame_widen(_ptr(frame_u8), _ld(frame_u8), _ptr(lost), lost.stride(0), H, W,
                                _ptr(out), _ld(out), _stream(out)))


def weigh(x, w, M: int, out) -> None:
    """out[b, :M] = x[b, :M] * w[(b or shared), :M] (one rounding per sample)."""
    import torch

    lib = load()
    _require(x, "x", torch.float64, 2)
    _require(w, "w", torch.float64)
    _require(out, "out", torch.float64, 2)
    ldw = _ld(w) if w.dim() == 2 else 0
    _check(lib.fase_weigh(_ptr(x), _ld(x), _ptr(w), ldw, x.shape[0], M, _ptr(out), _ld(out),
                          _stream(out)))


def weigh_gather(x, idx, w, out) -> None:
    """out[b, i] = x[b, idx[i]] * w[i] (i < len(idx)), zero pad to even width."""
    import torch

    lib = load()
    _require(x, "x", torch.float64, 2)
    _require(idx, "idx", torch.int32, 1)
    _require(w, "w", torch.float64, 1)
    _require(out, "out", torch.float64, 2)
    _check(lib.fase_weigh_gather(_ptr(x), _ld(x), _ptr(idx), _ptr(w), x.shape[0], idx.shape[0],
                                 _ptr(out), _ld(out), _stream(out)))


# Digit planes per FP64 operand. Shared tables keep 8 (56 bits of each row's
# scale: the DMMA table to a few ulp). The batched initial products use 7 (49
# bits, 28 plane pairs instead of 36): config 4 R0 within 2.8e-13 of the DMMA
# products (max |dR0| / max |R0|), every one of the 4,096 selected sequences
# still identical to the reference's, coefficients within 3.4e-13 of it, and
# the products 2.74 -> 2.28 ms (259.6K -> 269.1K blocks/s; 6 planes: 1.94 ms
# but 3.1e-11, too little margin for the 1e-9 near-tie rule after 500 updates;
# profiles/r02d/ab_slices.txt). FASE_PRODUCT_SLICES overrides (6-8).
OZAKI_SLICES = 8
PRODUCT_SLICES = int(os.environ.get("FASE_PRODUCT_SLICES", "7"))


class OzakiOperand:
    """Digit planes of an FP64 operand (rows x kd) for the tcgen05 INT8 path."""

    def __init__(self, rows: int, kd: int, row_align: int, device, slices: int = OZAKI_SLICES):
        import torch

        self.rows, self.kd, self.slices = rows, kd, slices
        self.kp = (kd + 63) // 64 * 64
        self.rows_pad = (max(rows, 1) + row_align - 1) // row_align * row_align
        # every byte of the valid rows is written by split(); the padding rows only
        # feed output rows that are never stored, so no zero fill is needed
        self.planes = torch.empty((slices, self.rows_pad, self.kp), dtype=torch.int8, device=device)
        self.exps = torch.zeros(self.rows_pad, dtype=torch.int32, device=device)

    def split(self, x, idx=None, w=None) -> "OzakiOperand":
        """Planes of x (rows x kd), or of x[:, idx] * w when a support gather
        and weights are given (idx int32 (kd,), w float64 (kd,))."""
        import torch

        lib = load()
        _require(x, "x", torch.float64, 2)
        if idx is not None:
            _require(idx, "idx", torch.int32, 1)
        if w is not None:
            _require(w, "w", torch.float64, 1)
        _check(lib.fase_ozaki_split(_ptr(x), _ld(x), _ptr(idx), _ptr(w), self.rows, self.kd,
                                    self.slices, _ptr(self.planes), self.kp, self.rows_pad,
                                    _ptr(self.exps), _stream(x)))
        return self


    def split_sparse(self, sel, coef, iters: int) -> "OzakiOperand":
        """Planes of the dense coefficient rows of sparse models: row r is
        sum_t coef[r, t] e_{sel[r, t]} over t < iters (sel int32 (rows, >= iters),
        coef float64 (rows, >= iters); sel < 0 adds nothing), kd = atoms."""
        import torch

        lib = load()
        _require(sel, "sel", torch.int32, 2)
        _require(coef, "coef", torch.float64, 2)
        if sel.shape[0] < self.rows or coef.shape[0] < self.rows:
            raise errors.ShapeError("split_sparse: fewer model rows than operand rows")
        _check(lib.fase_ozaki_split_sparse(_ptr(sel), _ld(sel), _ptr(coef), _ld(coef), self.rows,
                                           iters, self.kd, self.slices, _ptr(self.planes),
                                           self.kp, self.rows_pad, _ptr(self.exps),
                                           _stream(coef)))
        return self


def ozaki_gemm(a: OzakiOperand, b: OzakiOperand, C) -> None:
    """C[:a.rows, :b.rows] = X Y^T from the digit planes (C float64, 2-D)."""
    import torch

    lib = load()
    _require(C, "C", torch.float64, 2)
    if a.kp != b.kp or a.slices != b.slices:
        raise errors.ShapeError("operands were split with different K padding / plane counts")
    _check(lib.fase_ozaki_gemm(_ptr(a.planes), a.rows_pad, _ptr(a.exps), a.rows,
                               _ptr(b.planes), b.rows_pad, _ptr(b.exps), b.rows, a.kp,
                               a.slices, _ptr(C), _ld(C), _stream(C)))


def ozaki_gram(a: "OzakiOperand", b: "OzakiOperand", G) -> None:
    """Bit-symmetric G = X Y^T (X = Phi o w planes, Y = Phi planes, same K rows)."""
    import torch

    lib = load()
    _require(G, "G", torch.float64, 2)
    if a.kp != b.kp or a.slices != b.slices or a.rows != b.rows:
        raise errors.ShapeError("Gram operands must share K, the K padding and the plane count")
    _check(lib.fase_ozaki_gram(_ptr(a.planes), a.rows_pad, _ptr(a.exps), _ptr(b.planes),
                               b.rows_pad, _ptr(b.exps), a.rows, a.kp, a.slices, _ptr(G), _ld(G),
                               _stream(G)))


def sep_products_batch(factors, F, W, M_rows: int, N_cols: int, R0) -> None:
    """All separable parts [(rows, cols, col0)] of F o W (W None: F already
    weighted; 1-D W shared) on the FP64 tensor cores, one launch."""
    import torch

    lib = load()
    _require(F, "F", torch.float64, 2)
    _require(R0, "R0", torch.float64, 2)
    if W is not None:
        _require(W, "W", torch.float64)
    parts = (SepPart * len(factors))()
    for i, (rows, cols, col0) in enumerate(factors):
        _require(rows, "rows", torch.float64, 2)
        _require(cols, "cols", torch.float64, 2)
        parts[i] = SepPart(_ptr(rows), rows.shape[0], _ptr(cols), cols.shape[0], col0)
    ldw = _ld(W) if (W is not None and W.dim() == 2) else 0
    _check(lib.fase_sep_products_batch(parts, len(factors), M_rows, N_cols, _ptr(F), _ld(F),
                                       _ptr(W), ldw, F.shape[0], _ptr(R0), _ld(R0), _stream(R0)))


def sep_products(rows, cols, X, M_rows: int, N_cols: int, R0, col0: int) -> None:
    """R0[b, col0 + u*Lc + v] = (rows X_b cols^T)[u, v] for one separable part."""
    import torch

    lib = load()
    _require(rows, "rows", torch.float64, 2)
    _require(cols, "cols", torch.float64, 2)
    _require(X, "X", torch.float64, 2)
    _require(R0, "R0", torch.float64, 2)
    _check(lib.fase_sep_products(_ptr(rows), rows.shape[0], M_rows, _ptr(cols), cols.shape[0],
                                 N_cols, _ptr(X), _ld(X), X.shape[0], _ptr(R0), _ld(R0), col0,
                                 _stream(R0)))


def l2_flush(buf) -> None:
    lib = load()
    _check(lib.fase_l2_flush(_ptr(buf), buf.numel() * buf.element_size(), _stream(buf)))


def max_atoms() -> int:
    return int(load().fase_max_atoms())


def register_atoms() -> int:
    """Largest K whose recursion keeps R in registers (the tuned kernels); larger
    real dictionaries run the streaming recursion (exact only)."""
    return int(load().fase_iterate_register_atoms())


def table_ld(K: int) -> int:
    """Row stride (zero-padded) the recursion kernel needs for a K-atom table."""
    ld = int(load().fase_table_ld(K))
    if ld <= 0:
        raise errors.UnsupportedDictionaryError(f"K={K} exceeds the iteration kernel's "
                                                f"{max_atoms()} atoms")
    return ld
