"""Transform shortcuts for frequency-tagged dictionaries, on the GPU.

Drop-in for the reference's ``pkg/src/fase/transform.py`` (same names,
arguments, fallbacks and errors):

* ``fft_initial_products`` -- initial scalar products of the tagged atoms as
  one 2-D DFT of s*w evaluated at their (mu, eta) bins (transform.py:43-69).
  Here the DFT of the weighted area is the separable complex transform of
  csrc/separable.cu (conj(E) X conj(F)^T with the dictionary's own exponential
  factors) -- at 48 x 48 two small matrix products per block beat an FFT on a
  GPU and keep the atoms' exact factor values. Untagged atoms are evaluated
  directly (the DMMA GEMM); below ``min_tagged`` tagged atoms the whole call
  defers to ``initial_scalar_products``, as in the reference.
* ``fft_gram_table`` -- the (K, K) table gathered from the symmetrized
  spectrum of the weight (transform.py:84-110): one small transform plus a
  pure HBM write stream instead of (K^2 + K)/2 area sums.

Results agree with the direct path to rounding, as in the reference.
"""

from __future__ import annotations

import numpy as np

from . import _native
from .dictionary import Dictionary
from .errors import ShapeError, UnsupportedDictionaryError
from .fast import GramTable, initial_scalar_products, resolve_device
from .grid import as_real_field

FFT_MIN_TAGGED = 64


def _torch():
    import torch

    return torch


def _tags(dictionary: Dictionary):
    tagged = dictionary.tagged_indices()
    mu = np.array([dictionary.freqs[k][0] for k in tagged], dtype=np.int64)
    eta = np.array([dictionary.freqs[k][1] for k in tagged], dtype=np.int64)
    return tagged, mu, eta


_FACTORS: dict = {}


def _grid_factors(m_rows: int, n_cols: int, device):
    """The reference's exponential factors exp(2j pi u m / M) (dictionary.py:127-128),
    uploaded once per (area, device)."""
    torch = _torch()
    key = (m_rows, n_cols, device.type, device.index)
    if key not in _FACTORS:
        em = np.exp(2j * np.pi * np.outer(np.arange(m_rows), np.arange(m_rows)) / m_rows)
        en = np.exp(2j * np.pi * np.outer(np.arange(n_cols), np.arange(n_cols)) / n_cols)

        def up(a):
            return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(device)

        _FACTORS[key] = (up(em.real), up(em.imag), up(en.real), up(en.imag))
    return _FACTORS[key]


def weighted_spectra(x, m_rows: int, n_cols: int, device=None):
    """fft2 of B real (M, N) areas on the device: (B, M*N) complex128, bin
    (a, b) at a*N + b (the unnormalized forward DFT numpy's fft2 computes)."""
    torch = _torch()
    dev = resolve_device(device)
    X = torch.as_tensor(np.asarray(x, dtype=np.float64) if not isinstance(x, torch.Tensor) else x,
                        device=dev).reshape(-1, m_rows * n_cols)
    if (m_rows * n_cols) % 2:
        Xp = torch.zeros((X.shape[0], m_rows * n_cols + 1), dtype=torch.float64, device=dev)
        Xp[:, : m_rows * n_cols] = X
        X = Xp
    X = X.contiguous()
    out = torch.empty((X.shape[0], m_rows * n_cols), dtype=torch.complex128, device=dev)
    rre, rim, cre, cim = _grid_factors(m_rows, n_cols, dev)
    _native.sep_products_complex(rre, rim, cre, cim, X, m_rows, n_cols, out, 0)
    return out


def fft_initial_products(signal, weight, dictionary: Dictionary, *,
                         min_tagged: int = FFT_MIN_TAGGED, device=None) -> np.ndarray:
    """Initial scalar products with every tagged atom read off one 2-D DFT of
    s*w (``transform.py:43-69``); untagged atoms directly. Host (K,) complex128."""
    s = as_real_field(signal)
    w = np.asarray(weight, dtype=np.float64)
    if w.shape != s.shape:
        raise ShapeError(f"signal {s.shape} vs weight {w.shape}")
    if dictionary.shape != s.shape:
        raise ShapeError(f"signal {s.shape} vs dictionary area {dictionary.shape}")
    tagged, mu, eta = _tags(dictionary)
    if tagged.size < min_tagged:
        return initial_scalar_products(s, w, dictionary, device=device)
    m, n = s.shape
    spec = weighted_spectra((s * w)[None], m, n, device=device)[0].cpu().numpy()
    products = np.empty(len(dictionary), dtype=np.complex128)
    products[tagged] = spec[(mu % m) * n + (eta % n)]
    rest = np.setdiff1d(np.arange(len(dictionary)), tagged)
    if rest.size:
        direct = initial_scalar_products(s, w, dictionary, device=device)
        products[rest] = direct[rest]
    return products


def fft_gram_table(weight, dictionary: Dictionary, *, device=None) -> GramTable:
    """C and D gathered from the symmetrized spectrum of the weight
    (``transform.py:84-110``); every atom must carry a frequency tag.

    Raises:
        UnsupportedDictionaryError: at least one atom is untagged.
    """
    torch = _torch()
    w = np.asarray(weight, dtype=np.float64)
    m, n = dictionary.shape
    if w.shape != (m, n):
        raise ShapeError(f"weight {w.shape} vs dictionary area {(m, n)}")
    tagged, mu, eta = _tags(dictionary)
    k = len(dictionary)
    if tagged.size != k:
        raise UnsupportedDictionaryError(
            f"fft table build needs frequency tags on all atoms; {k - tagged.size} of {k} lack one")
    dev = resolve_device(device)
    spec = weighted_spectra(w[None], m, n, device=dev)
    mu, eta = mu % m, eta % n
    canonical = k == m * n and np.array_equal(mu, np.arange(k) // n) and \
        np.array_equal(eta, np.arange(k) % n)
    T = torch.zeros((k, _native.table_ld_complex(k)), dtype=torch.complex128, device=dev)
    if canonical:
        _native.fft_gram(spec, m, n, None, None, k, T)
    else:
        mu_d = torch.from_numpy(mu.astype(np.int32)).to(dev)
        eta_d = torch.from_numpy(eta.astype(np.int32)).to(dev)
        _native.fft_gram(spec, m, n, mu_d, eta_d, k, T)
    D = torch.empty(k, dtype=torch.float64, device=dev)
    alive = torch.zeros(1, dtype=torch.int32, device=dev)
    _native.gram_finish_complex(T, k, D, alive)
    return GramTable(G=T, D=D, source=(dictionary, np.asarray(w, dtype=np.float64).ravel().copy()),
                     n_alive=int(alive.item()))


__all__ = ["FFT_MIN_TAGGED", "fft_gram_table", "fft_initial_products", "weighted_spectra"]
