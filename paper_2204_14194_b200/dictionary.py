"""Basis-function dictionaries and their HBM-resident matrix Phi.

A dictionary is an ordered set of K atoms over an M x N area. The API keeps the
reference's names and semantics (``pkg/src/fase/dictionary.py:50-219``):
``Dictionary(values, families, freqs)``, ``generate_dictionary``,
``union_dictionaries``, ``parse_dict_spec``, FDIC file I/O, and a blake2b
``content_hash`` over the complex128 bytes so provenance hashes agree with the
reference for the same atoms.

What changes is where the atoms live. Separable families (DCT, WHT, Hadamard)
are kept as two small 1-D factor tables and expanded on the device by
``fase_basis_outer`` -- one correctly-rounded multiply per atom sample, which
is exactly the reference's ``np.einsum("um,vn->uvmn")`` outer product
(``dictionary.py:167-178``). Non-separable real families (the real DFT of
config 3, the Gaussian set of config 4, user arrays) are built on the host and
uploaded once. Phi is stored on the device as a (K, ld) float64 row-per-atom
matrix, ``ld`` = M rounded up to a multiple of 4 with zero padding.

Families added for the BASELINE configs, which the reference cannot express:

* ``had`` -- +-1 Hadamard atoms of any order with a known construction
  (Sylvester for powers of two, Paley I for q+1 with q prime = 3 mod 4, and
  their Kronecker products). ``had`` at 48 x 48 is Paley I with q = 47; row 0
  is all ones, so its DC atom is proportional to DCT atom 0 (the structural
  tie the selection rule exists for, ``reference.py:38-54``).
* ``rdft`` -- real 2-D DFT: cos atoms of one representative per conjugate
  frequency pair (self-conjugate frequencies included) then sin atoms of the
  non-self-conjugate representatives; K = M*N. Values are the real / imaginary
  parts of the reference's own complex DFT atoms (``dictionary.py:126-131``).
* ``brdft`` -- ``rdft`` sign-binarized with the reference's 1e-12 snap
  (``dictionary.py:36,142-147``).
* ``gauss`` -- K i.i.d. N(0,1) atoms from a fixed seed, each divided by its
  L2 norm (config 4).
"""

from __future__ import annotations

import hashlib
import struct
from collections import OrderedDict
from dataclasses import dataclass

import numpy as np

from .errors import FormatError, ParameterError, ShapeError

GENERATED_KINDS = ("dft", "dct", "wht", "bdft", "had", "rdft", "brdft")
BINARIZE_SNAP = 1e-12
_FDIC_MAGIC = "FDIC v1"


@dataclass(frozen=True)
class Atom:
    """One atom: its (M, N) values, optional DFT frequency tag, family label."""

    values: np.ndarray
    freq: tuple[int, int] | None = None
    family: str = "custom"


@dataclass(frozen=True)
class _SeparablePart:
    """K_p = Lr * Lc atoms phi[u*Lc + v][m, n] = rows[u, m] * cols[v, n]."""

    rows: np.ndarray  # (Lr, M) float64
    cols: np.ndarray  # (Lc, N) float64

    @property
    def size(self) -> int:
        return self.rows.shape[0] * self.cols.shape[0]

    def materialize(self) -> np.ndarray:
        lr, m = self.rows.shape
        lc, n = self.cols.shape
        return np.einsum("um,vn->uvmn", self.rows, self.cols).reshape(lr * lc, m, n)


def _round_up(x: int, to: int) -> int:
    return (x + to - 1) // to * to


def _complex_bytes_hash(arr: np.ndarray) -> int:
    h = hashlib.blake2b(digest_size=8)
    k, m, n = arr.shape
    h.update(struct.pack("<3Q", k, m, n))
    h.update(arr.view(np.float64).tobytes())
    return int.from_bytes(h.digest(), "little")


class Dictionary:
    """Ordered atom set over an M x N area.

    ``Dictionary(values, families=None, freqs=None)`` accepts any (K, M, N)
    array like the reference (``dictionary.py:59-85``): all-real input is kept
    as float64 (the GPU path's type), anything with a non-zero imaginary part
    as complex128 (handled by the oracle; the GPU path raises
    UnsupportedDictionaryError for it). Identically-zero atoms are rejected.
    """

    def __init__(self, values=None, families=None, freqs=None, *, _parts=None, _shape=None):
        if _parts is not None:
            self._parts = list(_parts)
            self._dense = None
            k = sum(p.size for p in self._parts)
            self._shape = tuple(_shape)
            self._is_real = True
        else:
            arr = np.asarray(values)
            if arr.ndim != 3 or min(arr.shape) < 1:
                raise ShapeError(f"dictionary values must be (K, M, N) with K >= 1, got {arr.shape}")
            early_hash = None
            if np.iscomplexobj(arr) and np.any(arr.imag != 0):
                dense = np.array(arr, dtype=np.complex128, order="C", copy=True)
                self._is_real = False
            else:
                if np.iscomplexobj(arr):
                    # hash the caller's exact complex bytes (signed zeros included)
                    early_hash = _complex_bytes_hash(
                        np.ascontiguousarray(arr, dtype=np.complex128))
                dense = np.array(arr.real if np.iscomplexobj(arr) else arr,
                                 dtype=np.float64, order="C", copy=True)
                self._is_real = True
            k = dense.shape[0]
            nonzero = dense.reshape(k, -1).any(axis=1)
            if not nonzero.all():
                raise ParameterError(f"atom {int(np.flatnonzero(~nonzero)[0])} is identically zero")
            dense.setflags(write=False)
            self._dense = dense
            self._parts = None
            self._shape = (dense.shape[1], dense.shape[2])
        self._k = k
        if families is None:
            families = ("custom",) * k
        elif isinstance(families, str):
            families = (families,) * k
        else:
            families = tuple(families)
        if len(families) != k:
            raise ShapeError(f"{len(families)} family labels for {k} atoms")
        if freqs is None:
            freqs = (None,) * k
        else:
            freqs = tuple(None if f is None else (int(f[0]), int(f[1])) for f in freqs)
        if len(freqs) != k:
            raise ShapeError(f"{len(freqs)} frequency tags for {k} atoms")
        self.families = families
        self.freqs = freqs
        self._content_hash: int | None = None if _parts is not None else early_hash
        self._device_cache: dict = {}
        # complex sets: row ranges that are separable products rows[u,m]*cols[v,n]
        # with complex factors (DFT exponentials, or real parts of a mixed union):
        # [(first atom, rows (Lr, M) complex, cols (Lc, N) complex)]
        self._cfactors: list = []

    # -- introspection ------------------------------------------------------

    def __len__(self) -> int:
        return self._k

    @property
    def shape(self) -> tuple[int, int]:
        return self._shape

    @property
    def area(self) -> int:
        return self._shape[0] * self._shape[1]

    @property
    def is_real(self) -> bool:
        return self._is_real

    @property
    def is_separable(self) -> bool:
        return self._parts is not None

    def real_values(self) -> np.ndarray:
        """(K, M, N) float64 host values (materialized on demand for separable sets)."""
        if not self._is_real:
            raise ParameterError("dictionary is complex-valued")
        if self._dense is None:
            dense = np.concatenate([p.materialize() for p in self._parts], axis=0)
            dense.setflags(write=False)
            self._dense = dense
        return self._dense

    @property
    def values(self) -> np.ndarray:
        """(K, M, N) complex128 values, as the reference exposes them."""
        if self._is_real:
            out = self.real_values().astype(np.complex128)
        else:
            out = self._dense.copy()
        out.setflags(write=False)
        return out

    def matrix(self) -> np.ndarray:
        """(K, M*N) row-per-atom host matrix (float64 for real sets)."""
        src = self.real_values() if self._is_real else self._dense
        return src.reshape(self._k, -1)

    def atom(self, k: int) -> Atom:
        src = self.real_values() if self._is_real else self._dense
        return Atom(values=src[k], freq=self.freqs[k], family=self.families[k])

    def __iter__(self):
        return (self.atom(k) for k in range(len(self)))

    def tagged_indices(self) -> np.ndarray:
        return np.array([k for k, f in enumerate(self.freqs) if f is not None], dtype=np.intp)

    def content_hash(self) -> int:
        """blake2b-64 of (K, M, N) and the complex128 atom bytes.

        Same digest as the reference's ``Dictionary.content_hash``
        (``dictionary.py:111-120``): for real sets the complex128 stream is
        re-created in chunks with +0.0 imaginary parts.
        """
        if self._content_hash is None:
            h = hashlib.blake2b(digest_size=8)
            m, n = self._shape
            h.update(struct.pack("<3Q", self._k, m, n))
            if self._is_real:
                flat = self.real_values().reshape(self._k, -1)
                step = max(1, (1 << 22) // max(1, flat.shape[1]))
                for lo in range(0, self._k, step):
                    blk = flat[lo:lo + step]
                    pair = np.zeros(blk.shape + (2,), dtype=np.float64)
                    pair[..., 0] = blk
                    h.update(pair.tobytes())
            else:
                h.update(np.ascontiguousarray(self._dense).view(np.float64).tobytes())
            self._content_hash = int.from_bytes(h.digest(), "little")
        return self._content_hash

    # -- device side --------------------------------------------------------

    @property
    def ld(self) -> int:
        """Leading dimension of the device Phi (area rounded up to 4 samples)."""
        return _round_up(self.area, 4)

    def device_factors(self, device):
        """[(rows (Lr, M) , cols (Lc, N), first atom)] on ``device`` for separable
        sets (cached), or None."""
        import torch

        if self._parts is None:
            return None
        dev = torch.device(device)
        key = ("factors", dev.type, dev.index)
        if key not in self._device_cache:
            out, row = [], 0
            for p in self._parts:
                out.append((torch.from_numpy(np.ascontiguousarray(p.rows)).to(dev),
                            torch.from_numpy(np.ascontiguousarray(p.cols)).to(dev), row))
                row += p.size
            self._device_cache[key] = out
        return self._device_cache[key]

    def device_cfactors(self, device):
        """[(rows_re, rows_im, cols_re, cols_im, first atom)] on ``device`` for the
        separable row ranges of a complex set (cached); [] when there are none."""
        import torch

        if self._is_real or not self._cfactors:
            return []
        dev = torch.device(device)
        key = ("cfactors", dev.type, dev.index)
        if key not in self._device_cache:
            def up(a):
                return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(dev)

            self._device_cache[key] = [(up(r.real), up(r.imag), up(c.real), up(c.imag), row0)
                                       for row0, r, c in self._cfactors]
        return self._device_cache[key]

    def device_matrix(self, device):
        """Phi in HBM, cached per device: (K, ld) float64 for real sets, and
        for complex sets the (2K, ld) conjugate-split matrix -- row 2k =
        Re phi_k, row 2k+1 = -Im phi_k (include/fase_b200.h, "Complex-valued
        dictionaries").

        Separable parts are expanded by the native outer-product kernel;
        dense atoms are uploaded.
        """
        import torch

        from . import _native

        dev = torch.device(device)
        key = (dev.type, dev.index)
        cached = self._device_cache.get(key)
        if cached is not None:
            return cached
        m, n = self._shape
        if not self._is_real:
            flat = self._dense.reshape(self._k, -1)
            split = np.zeros((2 * self._k, self.ld), dtype=np.float64)
            split[0::2, : m * n] = flat.real
            split[1::2, : m * n] = -flat.imag
            phi = torch.from_numpy(split).to(dev)
            self._device_cache[key] = phi
            return phi
        phi = torch.zeros((self._k, self.ld), dtype=torch.float64, device=dev)
        if self._parts is not None:
            row = 0
            for p in self._parts:
                rows = torch.from_numpy(np.ascontiguousarray(p.rows)).to(dev)
                cols = torch.from_numpy(np.ascontiguousarray(p.cols)).to(dev)
                _native.basis_outer(rows, cols, phi, row)
                row += p.size
        else:
            host = torch.from_numpy(np.array(self._dense.reshape(self._k, -1), copy=True))
            phi[:, : m * n].copy_(host.to(dev))
        self._device_cache[key] = phi
        return phi


# -- 1-D factor tables --------------------------------------------------------


def dct_rows(length: int) -> np.ndarray:
    """Orthonormal DCT-II rows (``dictionary.py:134-139``): row u at sample m is
    cos(pi*(2m+1)*u/(2L)), scaled by sqrt(1/L) for u=0 and sqrt(2/L) otherwise."""
    angles = np.pi * (2.0 * np.arange(length) + 1.0) / (2.0 * length)
    table = np.cos(np.outer(np.arange(length), angles))
    table[0] *= np.sqrt(1.0 / length)
    table[1:] *= np.sqrt(2.0 / length)
    return table


def sylvester_hadamard(order: int) -> np.ndarray:
    """Natural-order Sylvester matrix (what scipy.linalg.hadamard returns)."""
    if order < 1 or order & (order - 1):
        raise ParameterError(f"Sylvester construction needs a power of two, got {order}")
    h = np.ones((1, 1), dtype=np.float64)
    while h.shape[0] < order:
        h = np.block([[h, h], [h, -h]])
    return h


def _is_prime(q: int) -> bool:
    if q < 2:
        return False
    f = 2
    while f * f <= q:
        if q % f == 0:
            return False
        f += 1
    return True


def paley_hadamard(order: int) -> np.ndarray:
    """Paley construction I for order = q + 1, q prime with q = 3 (mod 4).

    Q[i, j] = chi(j - i) (Legendre symbol mod q), S = [[0, 1^T], [-1, Q]],
    H = I + S. Row 0 is all ones.
    """
    q = order - 1
    if not (_is_prime(q) and q % 4 == 3):
        raise ParameterError(f"Paley I needs order-1 prime and = 3 mod 4, got order {order}")
    squares = {(x * x) % q for x in range(1, q)}
    chi = np.array([0.0] + [1.0 if a in squares else -1.0 for a in range(1, q)])
    idx = np.arange(q)
    jac = chi[(idx[None, :] - idx[:, None]) % q]
    s = np.zeros((order, order))
    s[0, 1:] = 1.0
    s[1:, 0] = -1.0
    s[1:, 1:] = jac
    return np.eye(order) + s


def hadamard_matrix(order: int) -> np.ndarray:
    """+-1 Hadamard matrix of the given order with a normalized all-ones row 0."""
    if order >= 1 and order & (order - 1) == 0:
        return sylvester_hadamard(order)
    p2 = 1
    rest = order
    while rest % 2 == 0 and rest > 0:
        try:
            core = paley_hadamard(rest)
            return np.kron(sylvester_hadamard(p2), core) if p2 > 1 else core
        except ParameterError:
            rest //= 2
            p2 *= 2
    try:
        core = paley_hadamard(rest)
        return np.kron(sylvester_hadamard(p2), core) if p2 > 1 else core
    except ParameterError:
        raise ParameterError(f"no Hadamard construction known here for order {order}") from None


def _dft_exponentials(m_rows: int, n_cols: int):
    """Complex DFT atoms exactly as the reference forms them (``dictionary.py:126-131``)."""
    em = np.exp(2j * np.pi * np.outer(np.arange(m_rows), np.arange(m_rows)) / m_rows)
    en = np.exp(2j * np.pi * np.outer(np.arange(n_cols), np.arange(n_cols)) / n_cols)
    atoms = np.einsum("um,vn->uvmn", em, en).reshape(m_rows * n_cols, m_rows, n_cols)
    tags = [(mu, eta) for mu in range(m_rows) for eta in range(n_cols)]
    return atoms, tags, (em, en)


def _sign_snapped(x: np.ndarray) -> np.ndarray:
    y = np.array(x, dtype=np.float64, copy=True)
    y[np.abs(y) < BINARIZE_SNAP] = 0.0
    return np.sign(y)


def _binarize_complex(values: np.ndarray) -> np.ndarray:
    """Componentwise sign with snap (``dictionary.py:142-147``)."""
    return _sign_snapped(values.real) + 1j * _sign_snapped(values.imag)


def real_dft_atoms(m_rows: int, n_cols: int) -> np.ndarray:
    """(M*N, M, N) real DFT set: cos of pair representatives, then sin of the
    non-self-conjugate representatives (see module docstring)."""
    atoms, _, _ = _dft_exponentials(m_rows, n_cols)
    mu = np.arange(m_rows * n_cols) // n_cols
    eta = np.arange(m_rows * n_cols) % n_cols
    partner = ((m_rows - mu) % m_rows) * n_cols + (n_cols - eta) % n_cols
    k = np.arange(m_rows * n_cols)
    cos_idx = k[k <= partner]
    sin_idx = k[k < partner]
    out = np.concatenate([atoms.real[cos_idx], atoms.imag[sin_idx]], axis=0)
    assert out.shape[0] == m_rows * n_cols
    return np.ascontiguousarray(out)


def generate_dictionary(kind: str, m_rows: int, n_cols: int) -> Dictionary:
    """One family over an M x N area, K = M*N atoms, k = u*N + v order.

    Reference families ``dft, dct, wht, bdft`` follow
    ``dictionary.py:150-179``; ``had, rdft, brdft`` are the BASELINE
    additions described in the module docstring.

    Raises:
        ParameterError: unknown kind, size < 1, or no construction for the size.
    """
    if m_rows < 1 or n_cols < 1:
        raise ParameterError(f"area must be at least 1x1, got {m_rows}x{n_cols}")
    if kind == "dft":
        atoms, tags, (em, en) = _dft_exponentials(m_rows, n_cols)
        d = Dictionary(atoms, families="dft", freqs=tags)
        d._cfactors = [(0, em, en)]
        return d
    if kind == "bdft":
        atoms, _, _ = _dft_exponentials(m_rows, n_cols)
        return Dictionary(_binarize_complex(atoms), families="bdft")
    if kind == "dct":
        part = _SeparablePart(dct_rows(m_rows), dct_rows(n_cols))
        return Dictionary(_parts=[part], _shape=(m_rows, n_cols), families="dct")
    if kind == "wht":
        if m_rows & (m_rows - 1) or n_cols & (n_cols - 1):
            raise ParameterError(f"wht needs power-of-two sizes, got {m_rows}x{n_cols}")
        part = _SeparablePart(sylvester_hadamard(m_rows), sylvester_hadamard(n_cols))
        return Dictionary(_parts=[part], _shape=(m_rows, n_cols), families="wht")
    if kind == "had":
        part = _SeparablePart(hadamard_matrix(m_rows), hadamard_matrix(n_cols))
        return Dictionary(_parts=[part], _shape=(m_rows, n_cols), families="had")
    if kind == "rdft":
        return Dictionary(real_dft_atoms(m_rows, n_cols), families="rdft")
    if kind == "brdft":
        return Dictionary(_sign_snapped(real_dft_atoms(m_rows, n_cols)), families="brdft")
    raise ParameterError(f"unknown dictionary kind {kind!r}; expected one of {GENERATED_KINDS}")


def gaussian_dictionary(n_atoms: int, m_rows: int, n_cols: int, seed: int) -> Dictionary:
    """K unit-norm atoms with i.i.d. N(0,1) samples from ``default_rng(seed)`` (config 4)."""
    if n_atoms < 1 or m_rows < 1 or n_cols < 1:
        raise ParameterError("gaussian dictionary needs K, M, N >= 1")
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((n_atoms, m_rows * n_cols))
    norms = np.sqrt(np.einsum("ij,ij->i", x, x))
    x /= norms[:, None]
    return Dictionary(x.reshape(n_atoms, m_rows, n_cols), families="gauss")


def union_dictionaries(parts) -> Dictionary:
    """Concatenate dictionaries over one area, keeping order and tags
    (``dictionary.py:182-194``). Separable parts stay separable."""
    parts = list(parts)
    if not parts:
        raise ParameterError("union of zero dictionaries")
    shape = parts[0].shape
    for p in parts[1:]:
        if p.shape != shape:
            raise ShapeError(f"cannot union areas {shape} and {p.shape}")
    families = tuple(f for p in parts for f in p.families)
    freqs = tuple(f for p in parts for f in p.freqs)
    if all(p.is_separable for p in parts):
        sep = [q for p in parts for q in p._parts]
        return Dictionary(_parts=sep, _shape=shape, families=families, freqs=freqs)
    if all(p.is_real for p in parts):
        values = np.concatenate([p.real_values() for p in parts], axis=0)
        return Dictionary(values, families=families, freqs=freqs)
    values = np.concatenate([p.values for p in parts], axis=0)
    out = Dictionary(values, families=families, freqs=freqs)
    row = 0
    for p in parts:  # separable row ranges survive the union
        if p.is_separable:
            for q in p._parts:
                out._cfactors.append((row, q.rows.astype(np.complex128),
                                      q.cols.astype(np.complex128)))
                row += q.size
            continue
        out._cfactors.extend((row + r0, a, b) for r0, a, b in p._cfactors)
        row += len(p)
    return out


# Generated dictionaries are immutable and deterministic in (spec, M, N): the
# most recent ones are kept, so repeated calls (one per area shape in every
# conceal_image call) reuse the atoms, their content hash and device copies.
_SPEC_CACHE: "OrderedDict[tuple, Dictionary]" = OrderedDict()
_SPEC_CACHE_SIZE = 8


def parse_dict_spec(spec: str, m_rows: int, n_cols: int) -> Dictionary:
    """Resolve ``kind`` | ``union:a+b[+c]`` | ``file:PATH`` | ``gauss:K:SEED``
    against an M x N area (``dictionary.py:197-219`` plus the gauss form).
    Generated (non-file) dictionaries are memoized per (spec, M, N)."""
    spec = spec.strip()
    if spec.startswith("file:"):
        return _parse_dict_spec(spec, m_rows, n_cols)
    key = (spec, int(m_rows), int(n_cols))
    hit = _SPEC_CACHE.get(key)
    if hit is not None:
        _SPEC_CACHE.move_to_end(key)
        return hit
    d = _parse_dict_spec(spec, m_rows, n_cols)
    _SPEC_CACHE[key] = d
    while len(_SPEC_CACHE) > _SPEC_CACHE_SIZE:
        _SPEC_CACHE.popitem(last=False)
    return d


def _parse_dict_spec(spec: str, m_rows: int, n_cols: int) -> Dictionary:
    if spec.startswith("file:"):
        loaded = load_dictionary(spec[5:])
        if loaded.shape != (m_rows, n_cols):
            raise ShapeError(f"dictionary file covers {loaded.shape[0]}x{loaded.shape[1]}, "
                             f"area is {m_rows}x{n_cols}")
        return loaded
    if spec.startswith("gauss:"):
        try:
            _, k, seed = spec.split(":")
            return gaussian_dictionary(int(k), m_rows, n_cols, int(seed))
        except ValueError as exc:
            if isinstance(exc, ParameterError):
                raise
            raise ParameterError(f"gauss spec must be 'gauss:K:SEED', got {spec!r}") from None
    if spec.startswith("union:"):
        names = [part.strip() for part in spec[6:].split("+")]
        if len(names) < 2 or any(not name for name in names):
            raise ParameterError(f"union spec needs '+'-joined family names, got {spec!r}")
        return union_dictionaries(generate_dictionary(name, m_rows, n_cols) for name in names)
    return generate_dictionary(spec, m_rows, n_cols)


# -- FDIC files (layout of ``dictionary.py:222-286``) ---------------------------


def save_dictionary(dictionary: Dictionary, path) -> None:
    """Write ``FDIC v1 M N K real|complex\\n`` then K*M*N (re, im) float64 LE pairs."""
    m, n = dictionary.shape
    flag = "real" if dictionary.is_real else "complex"
    vals = dictionary.real_values() if dictionary.is_real else dictionary._dense
    with open(path, "wb") as fh:
        fh.write(f"{_FDIC_MAGIC} {m} {n} {len(dictionary)} {flag}\n".encode("ascii"))
        flat = vals.reshape(-1)
        step = 1 << 22
        for lo in range(0, flat.size, step):
            blk = flat[lo:lo + step]
            pair = np.empty((blk.size, 2), dtype="<f8")
            pair[:, 0] = blk.real
            pair[:, 1] = blk.imag if np.iscomplexobj(blk) else 0.0
            fh.write(pair.tobytes())


def load_dictionary(path) -> Dictionary:
    """Read an FDIC file; FormatError on any layout violation."""
    with open(path, "rb") as fh:
        header = fh.readline(256)
        payload = fh.read()
    try:
        text = header.decode("ascii")
    except UnicodeDecodeError as exc:
        raise FormatError(f"{path}: header is not ASCII") from exc
    if not text.endswith("\n"):
        raise FormatError(f"{path}: unterminated header line")
    fields = text.split()
    if len(fields) != 6 or " ".join(fields[:2]) != _FDIC_MAGIC:
        raise FormatError(f"{path}: expected '{_FDIC_MAGIC} M N K complex|real' header")
    try:
        m, n, k = int(fields[2]), int(fields[3]), int(fields[4])
    except ValueError as exc:
        raise FormatError(f"{path}: non-integer dimension in header") from exc
    flag = fields[5]
    if flag not in ("complex", "real"):
        raise FormatError(f"{path}: value flag must be 'complex' or 'real', got {flag!r}")
    if m < 1 or n < 1 or k < 1:
        raise FormatError(f"{path}: dimensions must be positive, got M={m} N={n} K={k}")
    if len(payload) != k * m * n * 16:
        raise FormatError(f"{path}: payload holds {len(payload)} bytes, header implies "
                          f"{k * m * n * 16}")
    pairs = np.frombuffer(payload, dtype="<f8").reshape(k * m * n, 2)
    if flag == "real" and pairs[:, 1].any():
        raise FormatError(f"{path}: flagged 'real' but carries nonzero imaginary parts")
    if pairs[:, 1].any():
        values = (pairs[:, 0] + 1j * pairs[:, 1]).reshape(k, m, n)
    else:
        values = pairs[:, 0].reshape(k, m, n).copy()
    zero = ~values.reshape(k, -1).any(axis=1)
    if zero.any():
        raise FormatError(f"{path}: atom {int(np.flatnonzero(zero)[0])} is identically zero")
    return Dictionary(values, families="file")
