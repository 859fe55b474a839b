"""FaSE on the B200: Gram tables, initial products, the recursion, synthesis.

Drop-in for the reference's fast path (``pkg/src/fase/fast.py``): the same
names, arguments, return types and error classes --
``GramTable``, ``provenance_hash``, ``build_gram_tables``,
``initial_scalar_products``, ``fase_extrapolate``, ``apply_model`` -- plus the
batched entry point the BASELINE configs need, ``fase_extrapolate_batch``.

Every numeric step runs in libfase_b200.so (csrc/); this module only
validates arguments, hashes provenance on the host (blake2b, as the
reference), builds the host-side weight field (bit-exact ``rho ** dist``), and
moves buffers. There is no CPU fallback: without CUDA or the library every
entry point raises NativeLibraryError.

Per-block geometries (``masks`` of shape (B, M, N)) use *chunked tables*:
samples are grouped into classes by their lost/kept pattern across the batch;
G0 is the table of the weight that keeps every sample some block keeps, and
C_j the table restricted to class j. Block b's table is
G0 - sum_{j lost in b} C_j, applied row by row inside the recursion kernel,
so per-block tables are never materialized.
"""

from __future__ import annotations

import functools
import hashlib
import os
import struct
from dataclasses import dataclass

import numpy as np

from . import _native
from .dictionary import Dictionary
from .errors import (
    MaskError,
    NativeLibraryError,
    NoSelectableAtomError,
    ParameterError,
    ShapeError,
    StaleTableError,
    UnsupportedDictionaryError,
)
from .grid import (
    ExtrapConfig,
    as_mask,
    as_real_field,
    base_weight,
    build_weight_field,
)
from .model import BatchResult, SparseModel

# Chunked per-block tables beyond this many bytes switch to one table per
# distinct geometry (see _run_grouped).
CHUNK_TABLE_BUDGET = 48 << 30


def _round_up(x: int, to: int) -> int:
    return (x + to - 1) // to * to


def _torch():
    import torch

    return torch


@functools.lru_cache(maxsize=1)
def _cuda_available() -> bool:
    return bool(_torch().cuda.is_available())


def resolve_device(device=None):
    torch = _torch()
    if not _cuda_available():
        raise NativeLibraryError("a CUDA device is required: the FaSE hot path has no CPU fallback")
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    dev = torch.device(device)
    if dev.type != "cuda":
        raise NativeLibraryError(f"device {dev} is not a CUDA device (no CPU fallback)")
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    return dev


def provenance_hash(dictionary: Dictionary, weight) -> int:
    """blake2b-64 binding a table to (dictionary, weight) (``fast.py:87-94``)."""
    w = np.ascontiguousarray(weight, dtype=np.float64).ravel()
    h = hashlib.blake2b(digest_size=8)
    h.update(b"gram-tables/1")
    h.update(struct.pack("<2Q", dictionary.content_hash(), w.size))
    h.update(w.tobytes())
    return int.from_bytes(h.digest(), "little")


class GramTable:
    """Weighted cross-energies C = conj(Phi) W Phi^T and normalizers D of one weight.

    Reference-compatible construction ``GramTable(c, d, provenance)`` from host
    arrays (``fast.py:55-85``), or device-born from ``build_gram_tables``.
    On the device a real table is a (K, ldg) float64 matrix, exactly
    symmetric; a complex table is a (K, ldt) complex128 matrix holding
    conj(C) row by row (the recursion's update operand), exactly Hermitian.
    Rows are zero-padded to the recursion kernel's capacity.
    """

    def __init__(self, c=None, d=None, provenance: int = 0, *, G=None, D=None, n_alive=None,
                 source=None):
        # ``source`` = (dictionary, weight) of a table built here: the
        # provenance digest (a blake2b pass over every atom) is computed only
        # when someone asks for it, and ``matches`` recognizes the same pair
        # without hashing
        self._provenance = None if source is not None else int(provenance)
        self._source = source
        self._G = G
        self._D = D
        self._host_c = None
        self._host_d = None
        self._uploaded = {}
        if G is None:
            c = np.asarray(c)
            d = np.asarray(d)
            if c.ndim != 2 or c.shape[0] != c.shape[1]:
                raise ShapeError(f"table must be square, got {c.shape}")
            if d.shape != (c.shape[0],):
                raise ShapeError(f"{d.shape[0] if d.ndim == 1 else d.shape} normalizers for a "
                                 f"{c.shape[0]}-atom table")
            self._host_c = c
            self._host_d = np.asarray(d, dtype=np.float64)
            self._k = c.shape[0]
            self._n_alive = int(np.count_nonzero(self._host_d))
            self._complex = bool(np.iscomplexobj(c) and np.any(c.imag != 0))
        else:
            self._k = int(G.shape[0])
            self._n_alive = int(n_alive) if n_alive is not None else None
            self._complex = bool(G.is_complex())

    @property
    def provenance(self) -> int:
        if self._provenance is None:
            self._provenance = provenance_hash(*self._source)
        return self._provenance

    def matches(self, dictionary: Dictionary, weight) -> bool:
        """True when this table was built for (dictionary, weight): the
        reference's provenance comparison (``fast.py:198-208``)."""
        if self._source is not None and self._source[0] is dictionary:
            w = np.asarray(weight, dtype=np.float64).ravel()
            if w.shape == self._source[1].shape and np.array_equal(w, self._source[1]):
                return True
        return self.provenance == provenance_hash(dictionary, weight)

    @property
    def size(self) -> int:
        return self._k

    @property
    def is_complex(self) -> bool:
        """True when the table carries imaginary parts (complex dictionaries)."""
        return self._complex

    @property
    def n_alive(self) -> int:
        if self._n_alive is None:
            self._n_alive = int((self._D != 0).sum().item())
        return self._n_alive

    @property
    def d(self) -> np.ndarray:
        if self._host_d is None:
            self._host_d = self._D.cpu().numpy()
        return self._host_d

    @property
    def c(self) -> np.ndarray:
        """Host complex128 (K, K) copy (downloads a device table on first use)."""
        if self._host_c is None:
            if self._G.is_complex():
                self._host_c = np.conj(self._G[:, : self._k].cpu().numpy())
            else:
                self._host_c = self._G[:, : self._k].cpu().numpy().astype(np.complex128)
        return self._host_c

    def degenerate(self) -> np.ndarray:
        return self.d == 0.0

    def device_tables(self, device, complex_rows: bool = False):
        """(G, D) on ``device`` in the layout the recursion needs.

        ``complex_rows=False``: real (K, table_ld(K)) float64 table -- raises
        UnsupportedDictionaryError when the table has imaginary content.
        ``complex_rows=True``: (K, table_ld_complex(K)) complex128 rows of
        conj(C). Host-born or other-layout tables are converted once and cached.
        """
        torch = _torch()
        k = self._k
        if self._G is not None:
            if self._G.device != device:
                raise ShapeError(f"table lives on {self._G.device}, run requested on {device}")
            if self._G.is_complex() == complex_rows:
                return self._G, self._D
        key = (device.type, device.index, complex_rows)
        if key not in self._uploaded:
            if complex_rows:
                T = torch.zeros((k, _native.table_ld_complex(k)), dtype=torch.complex128,
                                device=device)
                if self._G is not None:  # a real device table: conj(C) = C
                    T[:, :k].copy_(self._G[:, :k])
                else:
                    T[:, :k].copy_(torch.from_numpy(np.conj(np.asarray(self._host_c,
                                                                       dtype=np.complex128))))
                self._uploaded[key] = (T, self._D if self._D is not None else
                                       torch.from_numpy(self._host_d.copy()).to(device))
            else:
                if self._complex:
                    raise UnsupportedDictionaryError(
                        "this table has imaginary parts: run it with a complex dictionary")
                c = self._host_c if self._G is None else np.conj(
                    self._G[:, :k].cpu().numpy())
                c = np.asarray(c.real if np.iscomplexobj(c) else c, dtype=np.float64)
                G = torch.zeros((k, _native.table_ld(k)), dtype=torch.float64, device=device)
                G[:, :k].copy_(torch.from_numpy(np.ascontiguousarray(c)))
                D = self._D if self._D is not None else torch.from_numpy(self._host_d.copy()).to(device)
                self._uploaded[key] = (G, D)
        return self._uploaded[key]

    def scaled_table(self, device, complex_rows: bool = False):
        """(Gs, D): the column-scaled table Gs[u, k] = G[u, k] * D_k of the
        scaled recursion (``fase_iterate_scaled``; complex rows of conj(C) for
        ``fase_iterate_complex_scaled``), built on the device once and cached
        (one more table of the layout ``device_tables`` gives)."""
        torch = _torch()
        key = (device.type, device.index, "scaled", complex_rows)
        if key not in self._uploaded:
            G, D = self.device_tables(device, complex_rows=complex_rows)
            Gs = torch.empty_like(G)
            _native.scale_columns(G, D, self._k, Gs)
            self._uploaded[key] = (Gs, D)
        return self._uploaded[key]


RECURSIONS = ("exact", "scaled")


def _check_recursion(recursion: str, cplx: bool, shared: bool = True, record: bool = False):
    """Validate the ``recursion`` option of the batch entry points.

    ``exact``: fase_iterate(_complex), bit-identical to the reference given
    the same tables and initial products. ``scaled``: fase_iterate(_complex)
    _scaled over the column-scaled table (shared geometries; ~1.25x faster at
    config 1): selections identical except within a few ulp of a tie,
    coefficients to rounding -- the north-star parity bar, not bit-identity.
    """
    if recursion not in RECURSIONS:
        raise ParameterError(f"recursion must be one of {RECURSIONS}, got {recursion!r}")
    if recursion == "scaled" and (not shared or record):
        raise UnsupportedDictionaryError(
            "the scaled recursion runs shared-geometry batches without product logs")


def _check_large_k(recursion: str, K: int, cplx: bool):
    """Real dictionaries beyond the register kernels run the streaming exact
    recursion (csrc/iterate_generic.cu); the scaled one needs R in registers."""
    reg = _native.register_atoms_complex() if cplx else _native.register_atoms()
    if recursion == "scaled" and K > reg:
        raise UnsupportedDictionaryError(
            f"the scaled recursion holds at most {reg} atoms (K={K}); use recursion='exact'")


def _device_vector(x: np.ndarray, length: int, device):
    torch = _torch()
    out = torch.zeros(length, dtype=torch.float64, device=device)
    out[: x.size].copy_(torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64).ravel()))
    return out


def gram_support(w_dev, M: int):
    """(support indices int32, support weights) of a device weight vector."""
    torch = _torch()
    support = torch.nonzero(w_dev[:M] != 0).flatten()
    return support.to(torch.int32), w_dev.index_select(0, support).contiguous()


def gram_into(phi, w_dev, K: int, M: int, G, support=None) -> str:
    """The real weighted Gram table G = (Phi o w) Phi^T into G (K, ld), exactly
    symmetric; returns the path used. Large tables go to the tcgen05 Ozaki path
    over the support samples (digit planes of Phi o w and Phi gathered in one
    pass each); small ones to the DMMA GEMM. ``support``: gram_support(w_dev, M)
    when the caller has it (saves a device sync)."""
    sidx, w_s = support if support is not None else gram_support(w_dev, M)
    n_s = int(sidx.numel())
    if K >= 2048 and n_s >= 256:
        a = _native.OzakiOperand(K, n_s, 128, G.device).split(phi, sidx, w_s)
        b = _native.OzakiOperand(K, n_s, 64, G.device).split(phi, sidx)
        _native.ozaki_gram(a, b, G)
        return "ozaki"
    _native.gram(phi, w_dev, K, M, G)
    return "dmma"


def gram_panel_worthwhile(K: int, n_support: int) -> bool:
    """Row panels reproduce the single-GPU table bit for bit on the Ozaki path
    (exact integer accumulation, the same per-element epilogue whatever the
    tile), which is the one large tables take (``gram_into``)."""
    return K >= 2048 and n_support >= 256


def gram_panel_into(phi, w_dev, K: int, M: int, G, r0: int, r1: int, support=None) -> None:
    """Rows r0..r1 of the non-symmetric product (Phi o w) Phi^T into G[r0:r1]
    on the tcgen05 Ozaki path: every entry (i, j) with i <= j is bit-identical
    to the single-GPU symmetric build (``gram_into``), so assembling all panels
    and mirroring the upper triangle (``_native.mirror_upper``) gives that
    table exactly (multi-GPU table build, ``shard.build_gram_tables_sharded``)."""
    sidx, w_s = support if support is not None else gram_support(w_dev, M)
    n_s = int(sidx.numel())
    if not gram_panel_worthwhile(K, n_s):
        raise ParameterError("row panels need the Ozaki table path (K >= 2048, >= 256 support "
                             "samples)")
    if not (0 <= r0 <= r1 <= K):
        raise ShapeError(f"panel rows {r0}..{r1} outside 0..{K}")
    if r1 == r0:
        return
    a = _native.OzakiOperand(r1 - r0, n_s, 128, G.device).split(phi[r0:r1], sidx, w_s)
    b = _native.OzakiOperand(K, n_s, 64, G.device).split(phi, sidx)
    _native.ozaki_gemm(a, b, G[r0:r1])


def _gram_on_device(phi, w_dev, K: int, M: int, device, complex_rows: bool = False):
    """Real (K, table_ld) table, or complex (K, table_ld_complex) rows of conj(C)
    from the conjugate-split matrix of a complex dictionary."""
    torch = _torch()
    if complex_rows:
        T = torch.zeros((K, _native.table_ld_complex(K)), dtype=torch.complex128, device=device)
        _native.gram_complex(phi, w_dev, K, M, T)
        return T
    G = torch.zeros((K, _native.table_ld(K)), dtype=torch.float64, device=device)
    gram_into(phi, w_dev, K, M, G)
    return G


def _real_view(R):
    """(B, 2*ld) float64 view of a complex128 (B, ld) tensor (same storage)."""
    torch = _torch()
    return torch.view_as_real(R).reshape(R.shape[0], -1)


def initial_products_into(dictionary: Dictionary, F, W, R0, ws, *, method: str = "auto") -> str:
    """R0[b] = (F[b] o W) Phi^T on the device; returns the method used.

    ``separable``: for separable dictionaries (DCT / WHT / Hadamard parts) the
    weighted area X = F o W is transformed as rows X cols^T per part (csrc/
    separable.cu) -- the same identity as the reference's FFT shortcut for DFT
    atoms (transform.py:43-69), 24x fewer flops at 48 x 48. ``gemm``: one DMMA
    GEMM against the dense Phi. ``auto`` picks separable when available.
    """
    K, M = len(dictionary), dictionary.area
    dev = R0.device
    if R0.is_complex():
        # conj(Phi) (F o W) = [Re Phi; -Im Phi] (F o W): the conjugate-split
        # matrix as 2K real atoms writes (re, im) pairs straight into R0.
        # Separable row ranges (DFT exponentials) go through the complex
        # transform instead (fft_initial_products' identity, transform.py:43-69).
        parts = dictionary.device_cfactors(dev) if method in ("auto", "separable") else []
        if method == "separable" and not parts:
            raise UnsupportedDictionaryError("separable initial products need separable atoms")
        if not parts:
            _native.init_products(dictionary.device_matrix(dev), F, W, 2 * K, M, _real_view(R0),
                                  ws=ws)
            return "gemm"
        B = F.shape[0]
        ldx = M + (M & 1)
        X = ws[: B * ldx].view(B, ldx)
        _native.weigh(F, W, M, X)
        m, n = dictionary.shape
        covered = np.zeros(K, dtype=bool)
        try:
            for rre, rim, cre, cim, row0 in parts:
                _native.sep_products_complex(rre, rim, cre, cim, X, m, n, R0, row0)
                covered[row0: row0 + rre.shape[0] * cre.shape[0]] = True
        except UnsupportedDictionaryError:
            # areas whose factor tables exceed shared memory (about 71 x 71 and
            # up; the library refuses before launching): every row by GEMM
            if method == "separable":
                raise
            covered[:] = False
        phi2 = dictionary.device_matrix(dev)
        Rv = _real_view(R0)
        for lo, hi in _ranges(~covered):  # the remaining rows: one DMMA GEMM each
            _native.gemm_nt(X, phi2[2 * lo: 2 * hi], Rv[:, 2 * lo:])
        return "separable" if covered.all() else "separable+gemm"
    factors = dictionary.device_factors(dev) if method in ("auto", "separable") else None
    if method == "separable" and factors is None:
        raise UnsupportedDictionaryError("separable initial products need a separable dictionary")
    if factors is None:
        _native.init_products(dictionary.device_matrix(dev), F, W, K, M, R0, ws=ws)
        return "gemm"
    m, n = dictionary.shape
    try:
        if len(factors) <= 8:  # weights fused, all parts in one DMMA launch
            _native.sep_products_batch(factors, F, W, m, n, R0)
            return "separable"
        B = F.shape[0]
        ldx = M + (M & 1)
        X = ws[: B * ldx].view(B, ldx)
        _native.weigh(F, W, M, X)
        for rows, cols, row0 in factors:
            _native.sep_products(rows, cols, X, m, n, R0, row0)
        return "separable"
    except UnsupportedDictionaryError:
        # areas too large for the shared-memory transform (refused before
        # launching): the dense products cover every row
        if method == "separable":
            raise
        _native.init_products(dictionary.device_matrix(dev), F, W, K, M, R0, ws=ws)
        return "gemm"


def ozaki_worthwhile(rows: int, cols: int) -> bool:
    """Dense FP64 products go to the tcgen05 Ozaki path when the output has at
    least one 128 x 64 tile per SM (measured 2x DMMA at config-4 size and 2.6x
    on an 8-GPU shard of it, 512 x 8192: 0.40 vs 1.02 ms; smaller outputs stay
    on DMMA, whose tiles fill the GPU sooner)."""
    return rows >= 256 and cols >= 512 and ((rows + 127) // 128) * ((cols + 63) // 64) >= 148


def _ranges(flags: np.ndarray):
    """[(lo, hi)] runs of True in a boolean vector."""
    f = np.concatenate([[False], np.asarray(flags, dtype=bool), [False]])
    edges = np.flatnonzero(f[1:] != f[:-1])
    return list(zip(edges[0::2], edges[1::2]))


def build_gram_tables(dictionary: Dictionary, weight, *, block: int = 256, counter=None,
                      device=None) -> GramTable:
    """C and D for one (dictionary, weight) pair (``fast.py:109-142``).

    Upper-triangle DMMA tiles mirrored exactly (``C == C.T`` bit-for-bit),
    then D = 1/sqrt(diag) with the 1e-12 relative degeneracy cutoff.
    ``block`` is accepted for signature compatibility (the device tile is
    fixed); it must still be positive.
    """
    torch = _torch()
    w = np.asarray(weight, dtype=np.float64).ravel()
    if w.size != dictionary.area:
        raise ShapeError(f"weight has {w.size} samples, atoms have {dictionary.area}")
    if block < 1:
        raise ShapeError(f"block must be positive, got {block}")
    dev = resolve_device(device)
    K, M = len(dictionary), dictionary.area
    phi = dictionary.device_matrix(dev)
    cplx = not dictionary.is_real
    G = _gram_on_device(phi, _device_vector(w, dictionary.ld, dev), K, M, dev, cplx)
    D = torch.empty(K, dtype=torch.float64, device=dev)
    alive = torch.zeros(1, dtype=torch.int32, device=dev)
    (_native.gram_finish_complex if cplx else _native.gram_finish)(G, K, D, alive)
    if counter is not None:
        counter.table_pair_products(M, (K * K + K) // 2)
        counter.table_normalizers(K)
    return GramTable(G=G, D=D, source=(dictionary, w.copy()), n_alive=int(alive.item()))


def _complex_field(signal):
    """The signal as a 2-D complex128 field when it carries a non-zero imaginary
    part (``grid.as_field``'s coercion, ``grid.py:26-33``), else None."""
    arr = np.asarray(signal)
    if not np.iscomplexobj(arr) or not np.any(arr.imag != 0):
        return None
    if arr.ndim != 2:
        raise ShapeError(f"field must be 2-D, got shape {arr.shape}")
    if arr.size == 0:
        raise ShapeError("field must be non-empty")
    return np.ascontiguousarray(arr, dtype=np.complex128)


def initial_scalar_products(signal, weight, dictionary: Dictionary, *, counter=None,
                            device=None) -> np.ndarray:
    """R0_k = sum s * w * phi_k over the area (``fast.py:145-157``), on the GPU.

    A complex signal s = a + ib (the reference coerces with ``as_field``) gives
    R0(a) + i R0(b): the real path twice, combined in complex arithmetic."""
    torch = _torch()
    cs = _complex_field(signal)
    if cs is not None:
        ra = initial_scalar_products(cs.real, weight, dictionary, device=device)
        rb = initial_scalar_products(cs.imag, weight, dictionary, device=device)
        if counter is not None:
            counter.fase_initial(cs.size, len(dictionary))
        return ra + 1j * rb
    s = as_real_field(signal)
    w = np.asarray(weight, dtype=np.float64)
    if w.shape != s.shape:
        raise ShapeError(f"signal {s.shape} vs weight {w.shape}")
    if dictionary.shape != s.shape:
        raise ShapeError(f"signal {s.shape} vs dictionary area {dictionary.shape}")
    dev = resolve_device(device)
    K = len(dictionary)
    phi = dictionary.device_matrix(dev)
    f = _device_vector(s, dictionary.ld, dev).reshape(1, -1)
    wd = _device_vector(w, dictionary.ld, dev)
    if dictionary.is_real:
        R0 = torch.empty((1, _round_up(K, 2)), dtype=torch.float64, device=dev)
        _native.init_products(phi, f, wd, K, dictionary.area, R0)
    else:
        R0 = torch.empty((1, K), dtype=torch.complex128, device=dev)
        _native.init_products(phi, f, wd, 2 * K, dictionary.area, _real_view(R0))
    if counter is not None:
        counter.fase_initial(s.size, K)
    return R0[0, :K].cpu().numpy().astype(np.complex128)


# ----------------------------------------------------------------- batches


def _signals_on_device(signals, dictionary: Dictionary, device):
    """(B, ld) float64 device matrix of the block signals (a view when possible)."""
    torch = _torch()
    m, n = dictionary.shape
    area = m * n
    if isinstance(signals, torch.Tensor):
        if signals.dim() != 3 or tuple(signals.shape[1:]) != (m, n):
            raise ShapeError(f"signals {tuple(signals.shape)} vs dictionary area {(m, n)}")
        if signals.dtype != torch.float64:
            raise ShapeError(f"signals must be float64, got {signals.dtype}")
        flat = signals.to(device).reshape(signals.shape[0], area)
    else:
        arr = np.asarray(signals)
        if np.iscomplexobj(arr):
            if np.any(arr.imag != 0):
                raise UnsupportedDictionaryError("complex signals are not supported on the GPU path")
            arr = arr.real
        if arr.ndim != 3 or arr.shape[1:] != (m, n):
            raise ShapeError(f"signals {arr.shape} vs dictionary area {(m, n)}")
        flat = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float64).reshape(-1, area))
        flat = flat.to(device, non_blocking=True)
    if area % 2 == 0 and flat.is_contiguous():
        return flat
    out = torch.zeros((flat.shape[0], dictionary.ld), dtype=torch.float64, device=device)
    out[:, :area].copy_(flat)
    return out


@dataclass
class ChunkPlan:
    """Sample classes of a batch of per-block masks (host side).

    base_lost: (M,) lost in every block; classes: list of sample-index arrays
    of the mixed classes; ptr/ids: CSR of the classes each block loses.
    """

    base_lost: np.ndarray
    classes: list
    ptr: np.ndarray
    ids: np.ndarray

    @property
    def n_classes(self) -> int:
        return len(self.classes)


def chunk_plan(masks: np.ndarray) -> ChunkPlan:
    """Group samples by their lost/kept pattern across the batch."""
    b = masks.shape[0]
    flat = masks.reshape(b, -1)
    lost_any = flat.any(axis=0)
    lost_all = flat.all(axis=0)
    mixed = np.flatnonzero(lost_any & ~lost_all)
    if mixed.size == 0:
        classes, member = [], np.zeros((b, 0), dtype=bool)
    else:
        packed = np.packbits(flat[:, mixed], axis=0).T  # (n_mixed, ceil(B/8))
        _, first, inverse = np.unique(packed, axis=0, return_index=True, return_inverse=True)
        inverse = inverse.ravel()
        classes = [mixed[inverse == j] for j in range(len(first))]
        member = flat[:, mixed[first]]  # (B, n_classes): block loses class j
    counts = member.sum(axis=1)
    ptr = np.zeros(b + 1, dtype=np.int32)
    np.cumsum(counts, out=ptr[1:])
    ids = np.nonzero(member)[1].astype(np.int32)
    return ChunkPlan(base_lost=lost_all, classes=classes, ptr=ptr, ids=ids)


class ChunkedTables:
    """Device tables for a batch of per-block geometries: G0 and the class tables."""

    def __init__(self, dictionary: Dictionary, masks: np.ndarray, rho_hat: float, device):
        torch = _torch()
        self.device = device
        self.rho_hat = rho_hat
        m, n = dictionary.shape
        K, M = len(dictionary), m * n
        self.plan = chunk_plan(masks)
        base = base_weight(m, n, rho_hat).ravel()
        w0 = base.copy()
        w0[self.plan.base_lost] = 0.0
        phi = dictionary.device_matrix(device)
        self.complex = cplx = not dictionary.is_real
        self.G0 = _gram_on_device(phi, _device_vector(w0, dictionary.ld, device), K, M, device,
                                  cplx)
        ldg = self.G0.shape[1]
        nc = self.plan.n_classes
        self.tables = torch.zeros((max(nc, 1), K, ldg), dtype=self.G0.dtype, device=device)
        for j, samples in enumerate(self.plan.classes):
            cols = torch.from_numpy(samples.astype(np.int64)).to(device)
            width = _round_up(len(samples), 2)
            sub = torch.zeros((phi.shape[0], width), dtype=torch.float64, device=device)
            sub[:, : len(samples)] = phi.index_select(1, cols)
            wj = torch.zeros(width, dtype=torch.float64, device=device)
            wj[: len(samples)] = torch.from_numpy(base[samples]).to(device)
            (_native.gram_complex if cplx else _native.gram)(sub, wj, K, len(samples),
                                                             self.tables[j])
        counts = np.diff(self.plan.ptr).astype(np.int32)
        lists = np.zeros((len(counts), max(1, int(counts.max(initial=0)))), dtype=np.int32)
        for b in np.flatnonzero(counts):
            lists[b, : counts[b]] = self.plan.ids[self.plan.ptr[b]:self.plan.ptr[b + 1]]
        self.counts = torch.from_numpy(counts).to(device)
        self.ids = torch.from_numpy(lists).to(device)
        self.masks = masks
        self._dictionary = dictionary

    @property
    def key(self):
        """(dictionary content hash, mask shape, mask digest, rho_hat): an
        identity for caching these tables (hashed on first use)."""
        return (self._dictionary.content_hash(), self.masks.shape, hashlib.blake2b(
            np.packbits(self.masks).tobytes(), digest_size=16).hexdigest(), self.rho_hat)

    @staticmethod
    def table_bytes(dictionary: Dictionary, masks: np.ndarray) -> int:
        plan = chunk_plan(masks)
        k = len(dictionary)
        return (plan.n_classes + 1) * k * _round_up(k, 2) * (8 if dictionary.is_real else 16)


def _validate_masks(masks, dictionary: Dictionary, n_blocks: int):
    m, n = dictionary.shape
    arr = np.asarray(masks, dtype=bool)
    if arr.ndim == 2:
        if arr.shape != (m, n):
            raise ShapeError(f"mask {arr.shape} vs dictionary area {(m, n)}")
        if arr.all():
            raise MaskError("loss mask marks every sample lost; nothing to extrapolate from")
        return arr, True
    if arr.ndim != 3 or arr.shape != (n_blocks, m, n):
        raise ShapeError(f"masks {arr.shape} vs ({n_blocks}, {m}, {n})")
    full = arr.reshape(n_blocks, -1).all(axis=1)
    if full.any():
        raise MaskError(f"block {int(np.flatnonzero(full)[0])}: every sample is lost")
    if n_blocks > 0 and (arr == arr[0]).all():
        return arr[0], True
    return arr, False


def fase_extrapolate_batch(signals, masks, dictionary: Dictionary, tables=None,
                           config: ExtrapConfig = ExtrapConfig(), *, products=None,
                           record_products: bool = False, patch: bool = True,
                           device=None, recursion: str = "exact",
                           _complex_state: bool = False) -> BatchResult:
    """Run FaSE on B independent blocks; equals B calls of ``fase_extrapolate``.

    Args:
        signals: (B, M, N) float64 -- numpy (host) or torch (any device).
        masks: (M, N) shared loss mask, or (B, M, N) per-block masks.
        dictionary: atoms over the (M, N) area (real-valued).
        tables: shared geometry -- a GramTable for the shared weight (built
            when None; StaleTableError on a provenance mismatch); per-block
            geometry -- None or a ChunkedTables built for these masks.
        config: iterations / gamma / rho_hat.
        products: optional (B, K) initial products (skips the GEMM).
        record_products: keep R after every iteration (B, I, K) -- test use.
        patch: produce the patched (B, M, N) areas.
        recursion: "exact" (bit-identical to the reference's loop) or
            "scaled" (real shared geometries; see ``_check_recursion``).

    Returns:
        BatchResult with device tensors.
    """
    torch = _torch()
    dev = resolve_device(device)
    F = _signals_on_device(signals, dictionary, dev)
    B = F.shape[0]
    K, M = len(dictionary), dictionary.area
    # (_complex_state: complex initial products with a real dictionary -- a
    # complex signal -- run the complex recursion over the real table; no synthesis)
    cplx = not dictionary.is_real or _complex_state
    if _complex_state and (patch or products is None):
        raise ParameterError("_complex_state needs given products and patch=False")
    kmax = _native.max_atoms_complex() if cplx else _native.max_atoms()
    if K > kmax:
        raise UnsupportedDictionaryError(f"K={K} exceeds the iteration kernel's {kmax}")
    _check_large_k(recursion, K, cplx)
    mask, shared = _validate_masks(masks, dictionary, B)
    _check_recursion(recursion, cplx, shared, record_products)
    I = config.iterations
    phi = dictionary.device_matrix(dev)

    chunk_args = {}
    if shared:
        w = build_weight_field(mask, config.rho_hat)
        if tables is None:
            tables = build_gram_tables(dictionary, w, device=dev)
        elif not isinstance(tables, GramTable):
            raise StaleTableError("per-block tables given for a shared geometry")
        if tables.size != K:
            raise StaleTableError(f"tables hold {tables.size} atoms, dictionary has {K}")
        if not tables.matches(dictionary, w):
            raise StaleTableError("table provenance mismatch: tables were built for a different "
                                  "dictionary/weight combination")
        if tables.n_alive == 0:
            raise NoSelectableAtomError("every atom has zero weighted energy")
        G, D = tables.device_tables(dev, complex_rows=cplx)
        W = _device_vector(w, dictionary.ld, dev)
        lost_idx = np.flatnonzero(mask.ravel()).astype(np.int32)
    else:
        if tables is None:
            if ChunkedTables.table_bytes(dictionary, mask) > CHUNK_TABLE_BUDGET:
                return _run_grouped(F, mask, dictionary, config, dev, patch)
            tables = ChunkedTables(dictionary, mask, config.rho_hat, dev)
        elif not isinstance(tables, ChunkedTables) or tables.masks.shape != mask.shape or \
                not np.array_equal(tables.masks, mask) or tables.rho_hat != config.rho_hat:
            raise StaleTableError("chunked tables were built for other masks / rho_hat")
        G = tables.G0
        D = torch.empty((B, G.shape[1]), dtype=torch.float64, device=dev)
        alive = torch.empty(B, dtype=torch.int32, device=dev)
        stride = tables.tables[0].numel()
        (_native.block_normalizers_complex if cplx else _native.block_normalizers)(
            G, tables.tables, stride, tables.counts, tables.ids, K, D, alive)
        dead = torch.nonzero(alive == 0)
        if dead.numel():
            raise NoSelectableAtomError(f"block {int(dead[0, 0])}: every atom has zero weighted energy")
        chunk_args = dict(chunk_tables=tables.tables, chunk_stride=stride,
                          chunk_count=tables.counts, chunk_ids=tables.ids)
        base = torch.from_numpy(base_weight(*dictionary.shape, config.rho_hat).ravel()).to(dev)
        mdev = torch.from_numpy(mask.reshape(B, -1)).to(dev)
        W = torch.zeros((B, F.shape[1]), dtype=torch.float64, device=dev)
        W[:, :M] = torch.where(mdev, torch.zeros((), dtype=torch.float64, device=dev), base)
        lost_idx = None

    ldr = _round_up(K, 2)
    vdt = torch.complex128 if cplx else torch.float64
    if products is None:
        R0 = torch.empty((B, ldr), dtype=vdt, device=dev)
        dense = not (dictionary.device_cfactors(dev) if cplx else dictionary.device_factors(dev))
        rows = phi.shape[0]
        if shared and dense and ozaki_worthwhile(B, rows):
            # large dense batches: support samples only, on the tcgen05 Ozaki path
            sidx, w_s = gram_support(W, M)
            n_s = int(sidx.numel())
            ns = _native.PRODUCT_SLICES
            a = _native.OzakiOperand(B, n_s, 128, dev, ns).split(F, sidx, w_s)
            b = _native.OzakiOperand(rows, n_s, 64, dev, ns).split(phi, sidx)
            _native.ozaki_gemm(a, b, _real_view(R0) if cplx else R0)
        else:
            ws = torch.empty(max(_native.init_products_workspace(M, B) // 8, 2),
                             dtype=torch.float64, device=dev)
            initial_products_into(dictionary, F, W, R0, ws)
    else:
        R0 = _products_on_device(products, B, K, ldr, dev, cplx)
    sel = torch.empty((B, I), dtype=torch.int32, device=dev)
    proj = torch.empty((B, I), dtype=vdt, device=dev)
    coef = torch.empty((B, I), dtype=vdt, device=dev)
    R_log = torch.empty((B, I, ldr), dtype=vdt, device=dev) if record_products else None
    if recursion == "scaled":
        Gs, _ = tables.scaled_table(dev, complex_rows=cplx)
        (_native.iterate_complex_scaled if cplx else _native.iterate_scaled)(
            Gs, D, R0, K, I, config.gamma, sel, proj, coef)
    else:
        (_native.iterate_complex if cplx else _native.iterate)(
            G, D, R0, K, I, config.gamma, sel, proj, coef, R_log=R_log, **chunk_args)

    patched = None
    max_imag = torch.zeros(B, dtype=torch.float64, device=dev) if cplx else None
    if patch:
        patched = F[:, :M].clone() if F.shape[1] != M else F.clone()
        extra = {"max_imag": max_imag} if cplx else {}
        synth = _native.synth_paste_complex if cplx else _native.synth_paste
        if shared:
            if lost_idx.size:
                idx = torch.from_numpy(lost_idx).to(dev)
                synth(phi, sel, coef, I, idx, patched, n_shared=int(lost_idx.size), **extra)
        else:
            flat = mask.reshape(B, -1)
            counts = flat.sum(axis=1)
            ptr = np.zeros(B + 1, dtype=np.int32)
            np.cumsum(counts, out=ptr[1:])
            idx = np.nonzero(flat)[1].astype(np.int32)
            if idx.size:
                synth(phi, sel, coef, I, torch.from_numpy(idx).to(dev), patched,
                      idx_ptr=torch.from_numpy(ptr).to(dev), **extra)
        patched = patched.reshape(B, *dictionary.shape)
    prods = R_log[:, :, :K] if R_log is not None else None
    return BatchResult(selected=sel, projections=proj, coefficients=coef, patched=patched,
                       products=prods, dictionary=dictionary, shape=dictionary.shape,
                       max_imag=max_imag)


def _bound_output(outputs: dict, key: str, shape, dtype, dev):
    """A caller-owned output buffer, checked against what the kernels write."""
    t = outputs[key]
    if tuple(t.shape) != tuple(shape) or t.dtype != dtype or t.device != dev:
        raise ShapeError(f"output {key}: {tuple(t.shape)} {t.dtype} on {t.device}, expected "
                         f"{tuple(shape)} {dtype} on {dev}")
    if not t.is_contiguous():
        raise ShapeError(f"output {key} must be contiguous")
    return t


class ExtrapolationPlan:
    """A prepared shared-geometry batch: validate, hash and build tables once,
    then ``run`` only enqueues the three kernels (initial products, recursion,
    synthesis) on the current stream -- no host work, no synchronization.

    Outputs live in preallocated device buffers: ``selected`` (B, I) int32,
    ``coefficients`` / ``projections`` (B, I) float64 and ``lost`` (B, L)
    float64, the reconstructed lost samples in row-major mask order.
    ``run_host`` is the end-to-end form: pinned host signals in, pinned host
    results out, copies on the same stream.
    """

    def __init__(self, dictionary: Dictionary, mask, n_blocks: int,
                 config: ExtrapConfig = ExtrapConfig(), tables: GramTable | None = None,
                 device=None, products: str = "auto", recursion: str = "exact",
                 outputs: dict | None = None):
        """``outputs``: optional caller-owned device buffers ``selected`` (B, I)
        int32, ``coefficients`` (B, I) and ``lost`` (B, max(L, 1)) float64 the
        kernels write instead of plan-owned ones (e.g. views of one contiguous
        result arena that a collective gathers, ``shard.ShardedBatch``)."""
        torch = _torch()
        self.device = dev = resolve_device(device)
        self.complex = cplx = not dictionary.is_real
        _check_recursion(recursion, cplx)
        self.recursion = recursion
        self.dictionary = dictionary
        self.config = config
        mask = as_mask(mask)
        if mask.shape != dictionary.shape:
            raise ShapeError(f"mask {mask.shape} vs dictionary area {dictionary.shape}")
        w = build_weight_field(mask, config.rho_hat)
        if tables is None:
            tables = build_gram_tables(dictionary, w, device=dev)
        if tables.size != len(dictionary):
            raise StaleTableError(f"tables hold {tables.size} atoms, dictionary has {len(dictionary)}")
        if not tables.matches(dictionary, w):
            raise StaleTableError("table provenance mismatch")
        if tables.n_alive == 0:
            raise NoSelectableAtomError("every atom has zero weighted energy")
        self.tables = tables
        K, M, I = len(dictionary), dictionary.area, config.iterations
        kmax = _native.max_atoms_complex() if cplx else _native.max_atoms()
        if K > kmax:
            raise UnsupportedDictionaryError(f"K={K} exceeds the iteration kernel's {kmax}")
        _check_large_k(recursion, K, cplx)
        self.G, self.D = tables.device_tables(dev, complex_rows=cplx)
        # the scaled recursion reads the column-scaled table instead of G
        self.Gs = tables.scaled_table(dev, complex_rows=cplx)[0] if recursion == "scaled" else None
        self.K, self.M, self.I, self.B = K, M, I, int(n_blocks)
        self.phi = dictionary.device_matrix(dev)
        self.W = _device_vector(w, dictionary.ld, dev)
        ldf = M if M % 2 == 0 else dictionary.ld
        self.F = torch.zeros((self.B, ldf), dtype=torch.float64, device=dev)
        vdt = torch.complex128 if cplx else torch.float64
        self.R0 = torch.empty((self.B, _round_up(K, 2)), dtype=vdt, device=dev)
        self.ws = torch.empty(max(_native.init_products_workspace(M, self.B) // 8, 2),
                              dtype=torch.float64, device=dev)
        self.products = products
        self.selected = torch.empty((self.B, I), dtype=torch.int32, device=dev)
        self.projections = torch.empty((self.B, I), dtype=vdt, device=dev)
        self.coefficients = torch.empty((self.B, I), dtype=vdt, device=dev)
        if outputs is not None:
            self.selected = _bound_output(outputs, "selected", (self.B, I), torch.int32, dev)
            self.coefficients = _bound_output(outputs, "coefficients", (self.B, I), vdt, dev)
        self.max_imag = torch.zeros(self.B, dtype=torch.float64, device=dev) if cplx else None
        lost = np.flatnonzero(mask.ravel()).astype(np.int32)
        self.n_lost = int(lost.size)
        self.lost_idx = torch.from_numpy(lost if lost.size else np.zeros(1, np.int32)).to(dev)
        self.lost_pos = torch.arange(max(self.n_lost, 1), dtype=torch.int64, device=dev)
        self.lost = torch.zeros((self.B, max(self.n_lost, 1)), dtype=torch.float64, device=dev)
        if outputs is not None:
            self.lost = _bound_output(outputs, "lost", (self.B, max(self.n_lost, 1)),
                                      torch.float64, dev)
        # Phi restricted to the lost samples (synthesis reads only these; the
        # compact copy stays L2-resident where the full matrix would not)
        nl = max(self.n_lost, 1)
        self.phi_lost = torch.zeros((self.phi.shape[0], nl + (nl & 1)), dtype=torch.float64,
                                    device=dev)
        if self.n_lost:
            self.phi_lost[:, : self.n_lost] = self.phi.index_select(1, self.lost_idx.long())
        self.lost_seq = torch.arange(nl, dtype=torch.int32, device=dev)
        # scaled recursion, batches of at most one block per SM (latency bound):
        # the synthesis runs inside the recursion (config 0: 0.112 -> 0.099 ms);
        # at full occupancy the separate kernel is faster (fused: c1 -6%, c4 -4%)
        # (the exact recursion fuses it too: fase_iterate_synth; config 0 exact
        # recursion + separate synthesis 87.7 + 16.9 us)
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        self.fused_synth = bool(
            not cplx and self.n_lost and self.B <= sms
            and self.n_lost <= (_native.scaled_synth_capacity(K, self.B) if self.Gs is not None
                                else _native.synth_capacity(K, self.B)))
        if cplx:
            cparts = dictionary.device_cfactors(dev) if products in ("auto", "separable") else []
            n_prod = 1 + (len(cparts) + len(_ranges(self._uncovered(cparts))) if cparts else 1)
        else:
            factors = dictionary.device_factors(dev) if products in ("auto", "separable") else None
            n_prod = (1 if len(factors) <= 8 else 1 + len(factors)) if factors else 2
        # Dense products over the support only: the lost samples have weight 0
        # and add exact zeros, so Phi's support columns are gathered once and
        # each run contracts over them (fase_weigh_gather + one DMMA GEMM).
        self._support = None
        self._ozaki = None
        dense = (cplx and not cparts) or (not cplx and not factors)
        support = np.flatnonzero(w.ravel() != 0.0).astype(np.int32)
        if dense and products in ("auto", "gemm", "ozaki"):
            n_s = support.size
            phi_s = torch.zeros((self.phi.shape[0], n_s + (n_s & 1)), dtype=torch.float64,
                                device=dev)
            sidx = torch.from_numpy(support).to(dev)
            phi_s[:, :n_s] = self.phi.index_select(1, sidx.long())
            w_s = torch.from_numpy(np.ascontiguousarray(w.ravel()[support])).to(dev)
            self._support = (sidx, w_s, phi_s,
                             torch.empty((self.B, n_s + (n_s & 1)), dtype=torch.float64,
                                         device=dev))
            n_prod = 2
            # FP64 products on the tcgen05 tensor cores (Ozaki digit planes,
            # csrc/ozaki.cu) for batches that fill the GPU; Phi's planes once here
            if products == "ozaki" or (products == "auto" and ozaki_worthwhile(self.B, phi_s.shape[0])):
                rows = phi_s.shape[0]
                ns = _native.PRODUCT_SLICES
                self._ozaki = (_native.OzakiOperand(self.B, n_s, 128, dev, ns),
                               _native.OzakiOperand(rows, n_s, 64, dev, ns).split(phi_s))
                n_prod = 2
        # Synthesis of the lost samples as one Ozaki product, g = V Phi_lost^T,
        # V the batch's sparse models scattered to dense coefficient rows
        # (fase_ozaki_split_sparse), when the B x L output fills the GPU with
        # one 128 x 64 tile per SM (config 4: 4,096 x 576): the per-block
        # gathers of phi rows stream 9.5 GB from L2 per batch, the product reads
        # Phi_lost's planes once per tile. Real dictionaries; FASE_SYNTH=paste
        # keeps the per-block kernel (measurement knob).
        self._synth_oz = None
        synth_mode = os.environ.get("FASE_SYNTH", "auto")
        if (not cplx and self.n_lost and not self.fused_synth and K <= 16384
                and synth_mode != "paste"
                and (synth_mode == "ozaki" or ozaki_worthwhile(self.B, self.n_lost))):
            ns = _native.PRODUCT_SLICES
            phi_t = self.phi_lost[:K, : self.n_lost].t().contiguous()
            self._synth_oz = (_native.OzakiOperand(self.B, K, 128, dev, ns),
                              _native.OzakiOperand(self.n_lost, K, 64, dev, ns).split(phi_t))
            torch.cuda.current_stream(dev).synchronize()  # phi_t freed after its split
            del phi_t
        # (weigh +) products + iterate + synth (split + product on the Ozaki path)
        n_synth = (2 if self._synth_oz is not None else 1) if self.n_lost and not self.fused_synth else 0
        self.launches_per_run = n_prod + 1 + n_synth

    def _scratch(self, slot: int = 0) -> dict:
        """Per-slot work buffers (R0, products scratch, max |Im g|): slot 0 is the
        plan's own, slot 1 lets a second batch run concurrently (run_host_stream)."""
        torch = _torch()
        if slot == 0:
            return {"R0": self.R0, "ws": self.ws,
                    "X": self._support[3] if self._support is not None else None,
                    "oz": self._ozaki[0] if self._ozaki is not None else None,
                    "soz": self._synth_oz[0] if self._synth_oz is not None else None,
                    "max_imag": self.max_imag}
        if not hasattr(self, "_slot1"):
            oz = None
            if self._ozaki is not None:
                a = self._ozaki[0]
                oz = _native.OzakiOperand(a.rows, a.kd, 128, self.device, a.slices)
            self._slot1 = {
                "R0": torch.empty_like(self.R0), "ws": torch.empty_like(self.ws),
                "X": torch.empty_like(self._support[3]) if self._support is not None else None,
                "oz": oz,
                "soz": (_native.OzakiOperand(self.B, self.K, 128, self.device,
                                             self._synth_oz[0].slices)
                        if self._synth_oz is not None else None),
                "max_imag": torch.zeros_like(self.max_imag) if self.max_imag is not None else None}
        return self._slot1

    def _products(self, F, slot: int = 0):
        """R0 for signals F (device, (B, ldf)): the support-compacted GEMM when
        the products are dense, else initial_products_into."""
        sc = self._scratch(slot)
        if self._support is None:
            return initial_products_into(self.dictionary, F, self.W, sc["R0"], sc["ws"],
                                         method=self.products)
        sidx, w_s, phi_s, _ = self._support
        out = _real_view(sc["R0"]) if self.complex else sc["R0"]
        if self._ozaki is not None:  # gather, weigh and split in one pass
            _native.ozaki_gemm(sc["oz"].split(F, sidx, w_s), self._ozaki[1], out)
            return "ozaki-support"
        _native.weigh_gather(F, sidx, w_s, sc["X"])
        _native.gemm_nt(sc["X"], phi_s, out)
        return "gemm-support"

    def _uncovered(self, cparts):
        flags = np.ones(self.K, dtype=bool)
        for rre, _, cre, _, row0 in cparts:
            flags[row0: row0 + rre.shape[0] * cre.shape[0]] = False
        return flags

    def tune_l2(self, selected, fraction: float = 0.5):
        """L2 residency hint from a previous batch's selections (host work, once):
        the most frequently selected atoms whose table rows fill ``fraction`` of
        the L2 are marked hot; the recursion copies their rows with an L2
        evict_last policy and every other row evict_first
        (``fase_iterate_args.l2_hot``). Results are unchanged (a cache hint).
        ``selected``: (B', I) int32 selections (host or device); None clears."""
        torch = _torch()
        if selected is None:
            self.l2_hot = None
            self.l2_hot_rows = 0
            return 0
        sel = np.asarray(selected.cpu() if hasattr(selected, "cpu") else selected).ravel()
        sel = sel[(sel >= 0) & (sel < self.K)]
        counts = np.bincount(sel, minlength=self.K)
        G = self.Gs if self.Gs is not None else self.G
        row_bytes = G.shape[1] * G.element_size()
        l2 = torch.cuda.get_device_properties(self.device).L2_cache_size
        n_hot = min(int(fraction * l2 // row_bytes), int((counts > 0).sum()))
        hot = np.argsort(-counts, kind="stable")[:n_hot]
        words = np.zeros((self.K + 31) // 32, dtype=np.uint32)
        np.bitwise_or.at(words, hot // 32, (np.uint32(1) << (hot % 32).astype(np.uint32)))
        self.l2_hot = torch.from_numpy(words.view(np.int32)).to(self.device)
        self.l2_hot_rows = int(n_hot)
        self.l2_hot_share = float(counts[hot].sum() / max(counts.sum(), 1))
        return n_hot

    def _iterate_synth(self, sel, proj, coef, lost, slot: int = 0):
        sc = self._scratch(slot)
        if self.complex:
            if self.Gs is not None:
                _native.iterate_complex_scaled(self.Gs, self.D, sc["R0"], self.K, self.I,
                                               self.config.gamma, sel, proj, coef)
            else:
                _native.iterate_complex(self.G, self.D, sc["R0"], self.K, self.I,
                                        self.config.gamma, sel, proj, coef)
            if self.n_lost:
                _native.synth_paste_complex(self.phi_lost, sel, coef, self.I, self.lost_seq, lost,
                                            n_shared=self.n_lost, dst=self.lost_pos,
                                            max_imag=sc["max_imag"])
            return
        hot = getattr(self, "l2_hot", None)
        if self.fused_synth and self.Gs is not None:
            _native.iterate_scaled(self.Gs, self.D, sc["R0"], self.K, self.I, self.config.gamma,
                                   sel, proj, coef, phi_lost=self.phi_lost, n_lost=self.n_lost,
                                   lost=lost, l2_hot=hot)
            return
        if self.fused_synth:
            _native.iterate(self.G, self.D, sc["R0"], self.K, self.I, self.config.gamma, sel, proj,
                            coef, l2_hot=hot, phi_lost=self.phi_lost, n_lost=self.n_lost, lost=lost)
            return
        if self.Gs is not None:
            _native.iterate_scaled(self.Gs, self.D, sc["R0"], self.K, self.I, self.config.gamma,
                                   sel, proj, coef, l2_hot=hot)
        else:
            _native.iterate(self.G, self.D, sc["R0"], self.K, self.I, self.config.gamma, sel,
                            proj, coef, l2_hot=hot)
        self._synth(sel, coef, lost, slot)

    def _synth(self, sel, coef, lost, slot: int = 0):
        """Lost samples of real models (separate from the recursion): the Ozaki
        product when the plan set it up, else fase_synth_paste (bit-exact
        sequential order)."""
        if not self.n_lost:
            return
        if self._synth_oz is not None:
            a = self._scratch(slot)["soz"].split_sparse(sel, coef, self.I)
            _native.ozaki_gemm(a, self._synth_oz[1], lost)
            return
        _native.synth_paste(self.phi_lost, sel, coef, self.I, self.lost_seq, lost,
                            n_shared=self.n_lost, dst=self.lost_pos)

    def run(self, signals=None):
        """Enqueue one batch. ``signals``: None (use ``self.F`` as filled by the
        caller) or a (B, M, N) / (B, M) float64 tensor on any device. A
        contiguous float64 tensor on the plan's device whose rows already have
        the kernels' layout (even area) is read in place and must stay unchanged
        until the batch completes; anything else is copied asynchronously into
        ``self.F``."""
        F = self.F
        if signals is not None:
            src = signals.reshape(self.B, -1)
            torch = _torch()
            if (src.device == self.device and src.dtype == torch.float64 and src.is_contiguous()
                    and F.shape[1] == self.M and src.data_ptr() % 16 == 0):
                F = src  # already in the kernels' layout: read in place, no copy
            else:
                F[:, : self.M].copy_(src, non_blocking=True)
        self.products_method = self._products(F)
        self._iterate_synth(self.selected, self.projections, self.coefficients, self.lost)
        return self

    def host_buffers(self):
        """Pinned host buffers matching the outputs (for ``run_host``)."""
        torch = _torch()
        return {
            "selected": torch.empty(tuple(self.selected.shape), dtype=torch.int32, pin_memory=True),
            "coefficients": torch.empty(tuple(self.coefficients.shape),
                                        dtype=self.coefficients.dtype, pin_memory=True),
            "lost": torch.empty(tuple(self.lost.shape), dtype=torch.float64, pin_memory=True),
        }

    def run_host(self, host_signals, out: dict):
        """H2D of pinned ``host_signals`` (B, M, N), the batch, D2H of selections,
        coefficients and lost samples into pinned ``out`` -- all on one stream."""
        self.run(host_signals)
        out["selected"].copy_(self.selected, non_blocking=True)
        out["coefficients"].copy_(self.coefficients, non_blocking=True)
        out["lost"].copy_(self.lost, non_blocking=True)
        return out

    def run_host_stream(self, host_inputs, host_outputs, *, slot_outputs=None, finish=None):
        """End-to-end over a sequence of batches with copies and batches overlapped.

        ``host_inputs[i]`` (pinned (B, M, N) float64) goes in and
        ``host_outputs[i]`` (pinned dicts from ``host_buffers``) comes back, for
        every i. Consecutive batches alternate between two compute streams with
        their own device buffers, so batch i+1's copy-in, products and first
        recursion CTAs fill the SMs that batch i's last wave leaves idle;
        copies run on their own streams; events order every buffer reuse.
        Everything is enqueued; the caller's stream waits for the last results.

        ``slot_outputs`` optionally gives the second slot's device outputs
        (selected, projections, coefficients, lost); ``finish(slot, hout)``,
        called on the slot's compute stream after its kernels, replaces the
        default read-back: it returns the (host destination, device source)
        pairs to copy (``shard.ShardedBatch`` gathers the ranks' results there
        and reads back the gathered arena on the root rank only).
        """
        torch = _torch()
        dev = self.device
        cs = torch.cuda.current_stream(dev)
        if not hasattr(self, "_pipe"):
            self._scratch(1)
            self._pipe = {
                "h2d": torch.cuda.Stream(dev), "d2h": torch.cuda.Stream(dev),
                "comp": [torch.cuda.Stream(dev), torch.cuda.Stream(dev)],
                "F": [self.F, torch.zeros_like(self.F)],
                "out": [(self.selected, self.projections, self.coefficients, self.lost),
                        tuple(slot_outputs) if slot_outputs is not None else
                        tuple(torch.empty_like(x) for x in (self.selected, self.projections,
                                                            self.coefficients, self.lost))],
            }
        p = self._pipe
        h2d, d2h, comp = p["h2d"], p["d2h"], p["comp"]
        start = torch.cuda.Event()
        start.record(cs)  # nothing below starts before the caller's prior work
        for st in (h2d, d2h, comp[0], comp[1]):
            st.wait_event(start)
        ev_in = [torch.cuda.Event(), torch.cuda.Event()]
        ev_used = [None, None]     # compute finished reading F[slot]
        ev_out = [None, None]      # results of slot copied back
        for i, (hin, hout) in enumerate(zip(host_inputs, host_outputs)):
            s = i % 2
            F = p["F"][s]
            sel, proj, coef, lost = p["out"][s]
            with torch.cuda.stream(h2d):
                if ev_used[s] is not None:
                    h2d.wait_event(ev_used[s])
                F[:, : self.M].copy_(hin.reshape(self.B, -1), non_blocking=True)
                ev_in[s].record(h2d)
            c = comp[s]
            with torch.cuda.stream(c):
                c.wait_event(ev_in[s])
                if ev_out[s] is not None:
                    c.wait_event(ev_out[s])
                self._products(F, s)
                ev_used[s] = torch.cuda.Event()
                ev_used[s].record(c)
                self._iterate_synth(sel, proj, coef, lost, s)
                if finish is not None:
                    copies = finish(s, hout)
                else:
                    copies = [(hout["selected"], sel), (hout["coefficients"], coef),
                              (hout["lost"], lost)]
                done = torch.cuda.Event()
                done.record(c)
            with torch.cuda.stream(d2h):
                d2h.wait_event(done)
                for dst, src in copies:
                    dst.copy_(src, non_blocking=True)
                ev_out[s] = torch.cuda.Event()
                ev_out[s].record(d2h)
        # the caller's stream waits for the last copies
        for e in ev_out:
            if e is not None:
                cs.wait_event(e)
        return host_outputs

    def bytes_h2d(self) -> int:
        return self.B * self.M * 8

    def bytes_d2h(self) -> int:
        return (self.selected.numel() * 4 + self.coefficients.numel() * self.coefficients.element_size()
                + self.lost.numel() * 8)


def _products_on_device(products, B: int, K: int, ldr: int, device, cplx: bool = False):
    torch = _torch()
    if isinstance(products, torch.Tensor):
        p = products.to(device)
        if p.is_complex() and not cplx:
            if torch.any(p.imag != 0):
                raise UnsupportedDictionaryError("complex products for a real dictionary")
            p = p.real
    else:
        arr = np.asarray(products)
        if cplx:
            p = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.complex128)).to(device)
        else:
            if np.iscomplexobj(arr):
                if np.any(arr.imag != 0):
                    raise UnsupportedDictionaryError("complex products for a real dictionary")
                arr = arr.real
            p = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float64)).to(device)
    p = p.reshape(-1, K) if p.dim() == 1 else p
    if tuple(p.shape) != (B, K):
        raise ShapeError(f"products shape {tuple(p.shape)}, expected ({B}, {K})")
    R0 = torch.zeros((B, ldr), dtype=torch.complex128 if cplx else torch.float64, device=device)
    R0[:, :K].copy_(p)
    return R0


def _run_grouped(F, masks, dictionary, config, dev, patch):
    """One table per distinct geometry (fallback when chunk tables would not fit)."""
    torch = _torch()
    B = F.shape[0]
    flat = masks.reshape(B, -1)
    uniq, inverse = np.unique(flat, axis=0, return_inverse=True)
    inverse = inverse.ravel()
    I = config.iterations
    vdt = torch.float64 if dictionary.is_real else torch.complex128
    sel = torch.empty((B, I), dtype=torch.int32, device=dev)
    proj = torch.empty((B, I), dtype=vdt, device=dev)
    coef = torch.empty((B, I), dtype=vdt, device=dev)
    max_imag = None if dictionary.is_real else torch.zeros(B, dtype=torch.float64, device=dev)
    patched = F[:, : dictionary.area].clone() if patch else None
    for g in range(uniq.shape[0]):
        rows = np.flatnonzero(inverse == g)
        ridx = torch.from_numpy(rows).to(dev)
        sub = fase_extrapolate_batch(F.index_select(0, ridx).reshape(-1, *dictionary.shape),
                                     uniq[g].reshape(dictionary.shape), dictionary, None, config,
                                     patch=patch, device=dev)
        sel[ridx] = sub.selected
        proj[ridx] = sub.projections
        coef[ridx] = sub.coefficients
        if max_imag is not None:
            max_imag[ridx] = sub.max_imag
        if patch:
            patched[ridx] = sub.patched.reshape(len(rows), -1)
    if patch:
        patched = patched.reshape(B, *dictionary.shape)
    return BatchResult(selected=sel, projections=proj, coefficients=coef, patched=patched,
                       dictionary=dictionary, shape=dictionary.shape, max_imag=max_imag)


# ----------------------------------------------------------------- single block


def fase_extrapolate(signal, mask, dictionary: Dictionary, tables: GramTable,
                     config: ExtrapConfig = ExtrapConfig(), *, products=None,
                     record_products: bool = False, counter=None, device=None):
    """Scalar-product recursion for one area (``fast.py:160-264``).

    Same checks in the same order as the reference: shapes, atom count,
    provenance (StaleTableError), all-degenerate (NoSelectableAtomError).
    Returns (SparseModel, IterationTrace) with host arrays.
    """
    cs = _complex_field(signal)  # complex signals: products R0(re) + i R0(im)
    s = as_real_field(signal) if cs is None else np.ascontiguousarray(cs.real)
    mask = as_mask(mask)
    if mask.shape != s.shape:
        raise ShapeError(f"signal {s.shape} vs mask {mask.shape}")
    if dictionary.shape != s.shape:
        raise ShapeError(f"signal {s.shape} vs dictionary area {dictionary.shape}")
    if tables.size != len(dictionary):
        raise StaleTableError(f"tables hold {tables.size} atoms, dictionary has {len(dictionary)}")
    w = build_weight_field(mask, config.rho_hat)
    if not tables.matches(dictionary, w):
        raise StaleTableError("table provenance mismatch: tables were built for a different "
                              "dictionary/weight combination")
    if tables.n_alive == 0:
        raise NoSelectableAtomError("every atom has zero weighted energy")
    if products is not None:
        p = np.asarray(products)
        if p.shape != (len(dictionary),):
            raise ShapeError(f"products shape {p.shape}, expected ({len(dictionary)},)")
        products = p.reshape(1, -1)
    elif cs is not None:
        products = initial_scalar_products(cs, w, dictionary, device=device).reshape(1, -1)
    cstate = (dictionary.is_real and products is not None and np.iscomplexobj(products)
              and bool(np.any(np.asarray(products).imag != 0)))
    res = fase_extrapolate_batch(s[None], mask, dictionary, tables, config, products=products,
                                 record_products=record_products, patch=False, device=device,
                                 _complex_state=cstate)
    model, trace = res.block(0)
    if counter is not None:
        if products is None:
            counter.fase_initial(s.size, len(dictionary))
        for _ in range(config.iterations):
            counter.fase_selection(len(dictionary))
            counter.fase_update(s.size, len(dictionary))
    return model, trace


def apply_model(signal, model: SparseModel, mask, *, device=None):
    """Replace lost samples by Re(g) (``fast.py:267-286``); g on the GPU.

    Returns (patched float64 field, max |Im g| over lost samples) -- the latter
    is exactly 0.0 for real dictionaries.
    """
    torch = _torch()
    s = np.asarray(signal)
    mask = as_mask(mask)
    if s.shape != mask.shape:
        raise ShapeError(f"signal {s.shape} vs mask {mask.shape}")
    if tuple(model.shape) != s.shape:
        raise ShapeError(f"signal {s.shape} vs model area {model.shape}")
    out = s.astype(np.complex128 if np.iscomplexobj(s) else np.float64, copy=True)
    if not mask.any():
        return out, 0.0
    if len(model.terms) == 0:
        out[mask] = 0.0
        return out, 0.0
    dictionary = model.dictionary
    coefs = np.array([c for _, c in model.terms], dtype=np.complex128)
    dev = resolve_device(device)
    phi = dictionary.device_matrix(dev)
    sel = torch.tensor([[int(k) for k, _ in model.terms]], dtype=torch.int32, device=dev)
    idx = np.flatnonzero(mask.ravel()).astype(np.int32)
    g = torch.zeros((1, s.size), dtype=torch.float64, device=dev)
    if dictionary.is_real:
        # g = sum c * phi with real atoms: Re g and Im g are the real synthesis
        # of Re c and Im c (numpy's complex product with a zero imaginary part
        # rounds each component once, as here); complex coefficients come from
        # complex signals
        coef = torch.from_numpy(coefs.real.reshape(1, -1).copy()).to(dev)
        idx_d = torch.from_numpy(idx).to(dev)
        _native.synth_paste(phi, sel, coef, len(model.terms), idx_d, g, n_shared=int(idx.size))
        max_imag = 0.0
        if np.any(coefs.imag != 0):
            gi = torch.zeros_like(g)
            ci = torch.from_numpy(coefs.imag.reshape(1, -1).copy()).to(dev)
            _native.synth_paste(phi, sel, ci, len(model.terms), idx_d, gi, n_shared=int(idx.size))
            max_imag = float(gi.abs().max().item())
    else:
        coef = torch.from_numpy(coefs.reshape(1, -1).copy()).to(dev)
        mi = torch.zeros(1, dtype=torch.float64, device=dev)
        _native.synth_paste_complex(phi, sel, coef, len(model.terms),
                                    torch.from_numpy(idx).to(dev), g, n_shared=int(idx.size),
                                    max_imag=mi)
        max_imag = float(mi.item())
    out[mask] = g.cpu().numpy().ravel()[idx]
    return out, max_imag


# ----------------------------------------------------------------- FGRM files
#
# Layout of the reference's table files (fast.py:289-328): "FGRM v1\n", u64 LE
# K, u64 LE provenance, K*K complex entries row-major as (re, im) f64 LE, then
# K f64 LE entries of D -- exactly 24 + 16*K^2 + 8*K bytes.

_FGRM_MAGIC = b"FGRM v1\n"


def save_gram_table(tables: GramTable, path) -> None:
    """Write a table in the FGRM layout (device tables are downloaded once)."""
    k = tables.size
    c = tables.c
    d = np.asarray(tables.d, dtype="<f8")
    with open(path, "wb") as fh:
        fh.write(_FGRM_MAGIC)
        fh.write(struct.pack("<2Q", k, tables.provenance))
        step = max(1, (1 << 22) // max(1, k))
        for lo in range(0, k, step):
            blk = c[lo:lo + step]
            pairs = np.empty(blk.shape + (2,), dtype="<f8")
            pairs[..., 0] = blk.real
            pairs[..., 1] = blk.imag if np.iscomplexobj(blk) else 0.0
            fh.write(pairs.tobytes())
        fh.write(d.tobytes())


def load_gram_table(path) -> GramTable:
    """Read an FGRM file (e.g. written by the reference's ``fase tables``);
    FormatError on any layout violation. The table is uploaded on first use."""
    from .errors import FormatError

    with open(path, "rb") as fh:
        blob = fh.read()
    if len(blob) < 24 or blob[:8] != _FGRM_MAGIC:
        raise FormatError(f"{path}: not an FGRM v1 file")
    k, prov = struct.unpack_from("<2Q", blob, 8)
    if k < 1:
        raise FormatError(f"{path}: atom count must be positive, got {k}")
    if len(blob) != 24 + 16 * k * k + 8 * k:
        raise FormatError(f"{path}: {len(blob)} bytes, layout implies {24 + 16 * k * k + 8 * k}")
    pairs = np.frombuffer(blob, dtype="<f8", count=2 * k * k, offset=24).reshape(k, k, 2)
    c = pairs[..., 0] + 1j * pairs[..., 1]
    d = np.frombuffer(blob, dtype="<f8", count=k, offset=24 + 16 * k * k).copy()
    return GramTable(c=c, d=d, provenance=int(prov))
