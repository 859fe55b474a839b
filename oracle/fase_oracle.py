"""CPU oracle for the FaSE hot path -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.

A numpy restatement of the reference algorithm (``/root/reference/pkg/src/fase``),
in complex128 exactly as the reference computes, so that on the same numpy /
OpenBLAS build it reproduces the reference's outputs bit-for-bit. That claim is
pinned by ``tests/test_oracle_golden.py`` against fixtures produced by the
reference itself (``tests/golden/make_golden.py``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this module, and only as the checker / the timed CPU reference;
the product package never touches it (``tests/test_boundary.py`` checks that).

Every function cites the reference lines it restates.
"""

from __future__ import annotations

import hashlib
import math
import struct

import numpy as np

DEGENERACY_RTOL = 1e-12      # reference.py:36
SELECTION_TIE_RTOL = 1e-13   # reference.py:55
BINARIZE_SNAP = 1e-12        # dictionary.py:36


# ----------------------------------------------------------------- complex128 scalar semantics
#
# The reference's complex arithmetic is numpy's. On the build host (numpy 2.x,
# AVX-512 / FMA3 loops) the contiguous complex128 product and abs evaluate as
# below; tests/test_oracle_golden.py checks these statements against numpy and
# against tests/golden/complex_arith.npz, and the CUDA kernels implement the
# same sequences (csrc/common.cuh: np_cmul, np_cabs).


def _fma(a: float, b: float, c: float) -> float:
    """Correctly rounded a*b + c (exact rational arithmetic, then one rounding)."""
    from fractions import Fraction

    return float(Fraction(a) * Fraction(b) + Fraction(c))


def cmul_fused(x: complex, y: complex) -> complex:
    """x*y as numpy's loop computes it: (fma(xr, yr, -(xi*yi)), fma(xr, yi, xi*yr))."""
    return complex(_fma(x.real, y.real, -(x.imag * y.imag)),
                   _fma(x.real, y.imag, x.imag * y.real))


def cabs_scaled(z: complex) -> float:
    """|z| as numpy's loop computes it: larger * sqrt(fma(r, r, 1)), r = smaller / larger."""
    a, b = abs(z.real), abs(z.imag)
    hi, lo = max(a, b), min(a, b)
    if hi == 0.0:
        return 0.0
    r = lo / hi
    return math.sqrt(_fma(r, r, 1.0)) * hi


# ----------------------------------------------------------------- weighting


def weight_field(mask: np.ndarray, rho_hat: float) -> np.ndarray:
    """rho_hat ** distance-to-centre on support, 0.0 on lost (grid.py:75-99)."""
    mask = np.asarray(mask, dtype=bool)
    m_rows, n_cols = mask.shape
    dm = np.arange(m_rows, dtype=np.float64) - (m_rows - 1) / 2.0
    dn = np.arange(n_cols, dtype=np.float64) - (n_cols - 1) / 2.0
    w = rho_hat ** np.hypot(dm[:, None], dn[None, :])
    w[mask] = 0.0
    return w


def central_mask(m_rows: int, n_cols: int, loss_rows: int, loss_cols: int) -> np.ndarray:
    """Centred loss block at ((M-l)//2, (N-l)//2) (verify.py:37-49)."""
    mask = np.zeros((m_rows, n_cols), dtype=bool)
    r0 = (m_rows - loss_rows) // 2
    c0 = (n_cols - loss_cols) // 2
    mask[r0:r0 + loss_rows, c0:c0 + loss_cols] = True
    return mask


# ----------------------------------------------------------------- atoms


def dct_table(length: int) -> np.ndarray:
    """Orthonormal DCT-II 1-D rows (dictionary.py:134-139)."""
    ang = np.pi * (2.0 * np.arange(length) + 1.0) / (2.0 * length)
    t = np.cos(np.outer(np.arange(length), ang))
    t[0] *= np.sqrt(1.0 / length)
    t[1:] *= np.sqrt(2.0 / length)
    return t


def sylvester(order: int) -> np.ndarray:
    """Natural-order Walsh-Hadamard, the matrix scipy.linalg.hadamard builds
    (dictionary.py:173-178)."""
    h = np.array([[1.0]])
    while h.shape[0] < order:
        h = np.vstack([np.hstack([h, h]), np.hstack([h, -h])])
    return h


def outer_atoms(rows: np.ndarray, cols: np.ndarray) -> np.ndarray:
    """Separable atoms rows[u,m]*cols[v,n] at k = u*Lc + v (dictionary.py:167-178)."""
    lr, m = rows.shape
    lc, n = cols.shape
    return np.einsum("um,vn->uvmn", rows, cols).reshape(lr * lc, m, n).astype(np.complex128)


def dft_atoms(m_rows: int, n_cols: int) -> np.ndarray:
    """exp(+j2pi mu m/M) exp(+j2pi eta n/N) at k = mu*N + eta (dictionary.py:126-131)."""
    em = np.exp(2j * np.pi * np.outer(np.arange(m_rows), np.arange(m_rows)) / m_rows)
    en = np.exp(2j * np.pi * np.outer(np.arange(n_cols), np.arange(n_cols)) / n_cols)
    return np.einsum("um,vn->uvmn", em, en).reshape(m_rows * n_cols, m_rows, n_cols)


def binarize(values: np.ndarray) -> np.ndarray:
    """Componentwise sign after snapping |x| < 1e-12 to 0 (dictionary.py:142-147)."""
    re = np.array(values.real, dtype=np.float64, copy=True)
    im = np.array(values.imag, dtype=np.float64, copy=True)
    re[np.abs(re) < BINARIZE_SNAP] = 0.0
    im[np.abs(im) < BINARIZE_SNAP] = 0.0
    return np.sign(re) + 1j * np.sign(im)


def family(kind: str, m_rows: int, n_cols: int) -> np.ndarray:
    """The four reference families as (K, M, N) complex128 (dictionary.py:150-179)."""
    if kind == "dct":
        return outer_atoms(dct_table(m_rows), dct_table(n_cols))
    if kind == "wht":
        return outer_atoms(sylvester(m_rows), sylvester(n_cols))
    if kind == "dft":
        return dft_atoms(m_rows, n_cols)
    if kind == "bdft":
        return binarize(dft_atoms(m_rows, n_cols))
    raise ValueError(kind)


# ----------------------------------------------------------------- hashing


def content_hash(values: np.ndarray) -> int:
    """blake2b-64 over (K, M, N) and the complex128 bytes (dictionary.py:111-120)."""
    v = np.ascontiguousarray(values, dtype=np.complex128)
    h = hashlib.blake2b(digest_size=8)
    h.update(struct.pack("<3Q", *v.shape))
    h.update(v.view(np.float64).tobytes())
    return int.from_bytes(h.digest(), "little")


def provenance(dict_hash: int, weight: np.ndarray) -> int:
    """Table provenance over the dictionary hash and the weight bytes (fast.py:87-94)."""
    w = np.ascontiguousarray(weight, dtype=np.float64).ravel()
    h = hashlib.blake2b(digest_size=8)
    h.update(b"gram-tables/1")
    h.update(struct.pack("<2Q", dict_hash, w.size))
    h.update(w.tobytes())
    return int.from_bytes(h.digest(), "little")


# ----------------------------------------------------------------- tables


def gram(phi: np.ndarray, weight: np.ndarray, block: int = 256):
    """Weighted cross-energy table C and normalizers D.

    Upper-triangle row panels of ``conj(phi)*w @ phi.T``, then an exact
    conjugate mirror of the strict lower triangle, then a real diagonal and
    D = 1/sqrt(diag) with the 1e-12 relative degeneracy cutoff
    (fast.py:109-142 and fast.py:97-106).
    """
    w = np.asarray(weight, dtype=np.float64).ravel()
    phi = np.asarray(phi, dtype=np.complex128)
    k = phi.shape[0]
    c = np.empty((k, k), dtype=np.complex128)
    starts = list(range(0, k, block))
    for lo in starts:
        hi = min(lo + block, k)
        c[lo:hi, lo:] = (np.conj(phi[lo:hi]) * w) @ phi[lo:].T
    for lo in starts:
        hi = min(lo + block, k)
        c[hi:, lo:hi] = np.conj(c[lo:hi, hi:]).T
        tile = c[lo:hi, lo:hi]
        il = np.tril_indices(hi - lo, k=-1)
        tile[il] = np.conj(tile.T[il])
    diag = c.diagonal().real.copy()
    np.fill_diagonal(c, diag)
    top = float(diag.max(initial=0.0))
    d = np.zeros(k, dtype=np.float64)
    if top > 0.0:
        keep = diag > DEGENERACY_RTOL * top
        d[keep] = 1.0 / np.sqrt(diag[keep])
    return c, d


def initial_products(signal: np.ndarray, weight: np.ndarray, phi: np.ndarray) -> np.ndarray:
    """R0 = conj(Phi @ conj(s*w)) -- one zgemv (fast.py:145-157)."""
    s = np.ascontiguousarray(signal, dtype=np.complex128)
    w = np.asarray(weight, dtype=np.float64)
    return np.conj(np.asarray(phi, dtype=np.complex128) @ np.conj((s * w).ravel()))


# ----------------------------------------------------------------- selection


def tie_quantum(metric: np.ndarray) -> float:
    """1e-13 * max(metric), or 0 when the max is not finite-positive (reference.py:76-85)."""
    top = float(np.max(metric))
    if not math.isfinite(top) or top <= 0.0:
        return 0.0
    return SELECTION_TIE_RTOL * top


def select(metric: np.ndarray, quantum: float) -> int:
    """Lowest index within ``quantum`` of the max; -inf never ties (reference.py:58-73)."""
    u = int(np.argmax(metric))
    if quantum > 0.0 and math.isfinite(metric[u]):
        return int(np.argmax(metric >= metric[u] - quantum))
    return u


# ----------------------------------------------------------------- transform shortcuts


def fft_products(signal: np.ndarray, weight: np.ndarray, phi: np.ndarray, tags) -> np.ndarray:
    """Initial products of tagged atoms from fft2(s*w) at (mu, eta); untagged
    atoms directly (transform.py:43-69, without the min_tagged fallback)."""
    s = np.asarray(signal)
    m, n = s.shape
    out = np.empty(phi.shape[0], dtype=np.complex128)
    spec = np.fft.fft2(s * weight)
    rest = []
    for k, t in enumerate(tags):
        if t is None:
            rest.append(k)
        else:
            out[k] = spec[t[0] % m, t[1] % n]
    if rest:
        out[rest] = np.conj(phi[rest] @ np.conj((s * weight).ravel()))
    return out


def fft_gram(weight: np.ndarray, tags, m: int, n: int):
    """Table from the symmetrized spectrum of the weight, gathered at tag
    differences, then _finish_tables (transform.py:84-110)."""
    spec = np.fft.fft2(weight)
    mirror = spec[np.ix_((-np.arange(m)) % m, (-np.arange(n)) % n)]
    spec = 0.5 * (spec + np.conj(mirror))
    mu = np.array([t[0] for t in tags]) % m
    eta = np.array([t[1] for t in tags]) % n
    c = spec[(mu[:, None] - mu[None, :]) % m, (eta[:, None] - eta[None, :]) % n]
    diag = c.diagonal().real.copy()
    np.fill_diagonal(c, diag)
    top = float(diag.max(initial=0.0))
    d = np.zeros(diag.shape)
    if top > 0.0:
        alive = diag > DEGENERACY_RTOL * top
        d[alive] = 1.0 / np.sqrt(diag[alive])
    return c, d


# ----------------------------------------------------------------- iteration


def fase_run(r0: np.ndarray, c: np.ndarray, d: np.ndarray, gamma: float, iterations: int,
             record: bool = False):
    """The scalar-product recursion (fast.py:224-255).

    Returns (selected int64[I], projections complex[I], coefficients complex[I],
    product log list | None). No division inside the loop.
    """
    r = np.array(r0, dtype=np.complex128, copy=True)
    dead = d == 0.0
    any_dead = bool(dead.any())
    sel = np.empty(iterations, dtype=np.int64)
    proj = np.empty(iterations, dtype=np.complex128)
    coef = np.empty(iterations, dtype=np.complex128)
    log = [] if record else None
    q = 0.0
    for t in range(iterations):
        metric = np.abs(r) * d
        if any_dead:
            metric[dead] = -np.inf
        q = max(q, tie_quantum(metric))
        u = select(metric, q)
        p = r[u] * (d[u] * d[u])
        cu = complex(gamma * p)
        r -= cu * np.conj(c[u])
        sel[t] = u
        proj[t] = p
        coef[t] = cu
        if log is not None:
            log.append(r.copy())
    return sel, proj, coef, log


def se_run(signal: np.ndarray, mask: np.ndarray, phi: np.ndarray, gamma: float,
           iterations: int, rho_hat: float):
    """Explicit-residual Selective Extrapolation (reference.py:141-284).

    Recomputes every weighted projection from the residual each iteration.
    Returns (selected, projections, coefficients).
    """
    w = weight_field(mask, rho_hat).ravel()
    phi = np.asarray(phi, dtype=np.complex128)
    energies = np.empty(phi.shape[0])
    step = max(1, (1 << 22) // max(1, phi.shape[1]))
    for lo in range(0, phi.shape[0], step):
        b = phi[lo:lo + step]
        energies[lo:lo + step] = (b.real ** 2 + b.imag ** 2) @ w
    top = float(energies.max())
    if top <= 0.0:
        raise ValueError("every atom has zero weighted energy")
    alive = energies > DEGENERACY_RTOL * top
    root = np.sqrt(energies)
    r = np.ascontiguousarray(signal, dtype=np.complex128).ravel().copy()
    sel = np.empty(iterations, dtype=np.int64)
    proj = np.empty(iterations, dtype=np.complex128)
    coef = np.empty(iterations, dtype=np.complex128)
    q = 0.0
    for t in range(iterations):
        numer = np.conj(phi @ np.conj(r * w))
        p = np.zeros(phi.shape[0], dtype=np.complex128)
        np.divide(numer, energies, out=p, where=alive)
        metric = np.abs(p) * root
        metric[~alive] = -np.inf
        q = max(q, tie_quantum(metric))
        u = select(metric, q)
        cu = complex(gamma * p[u])
        r -= cu * phi[u]
        sel[t] = u
        proj[t] = p[u]
        coef[t] = cu
    return sel, proj, coef


# ----------------------------------------------------------------- synthesis


def materialize(values: np.ndarray, selected, coefficients) -> np.ndarray:
    """g = sum of c_t * phi_{u_t}, accumulated in selection order (reference.py:120-125)."""
    values = np.asarray(values, dtype=np.complex128)
    g = np.zeros(values.shape[1:], dtype=np.complex128)
    for u, cu in zip(selected, coefficients):
        g += complex(cu) * values[int(u)]
    return g


def apply(signal: np.ndarray, g: np.ndarray, mask: np.ndarray):
    """Paste Re(g) on lost samples; report max |Im g| over them (fast.py:267-286)."""
    s = np.asarray(signal)
    mask = np.asarray(mask, dtype=bool)
    out = s.astype(np.complex128 if np.iscomplexobj(s) else np.float64, copy=True)
    if not mask.any():
        return out, 0.0
    out[mask] = g.real[mask]
    return out, float(np.abs(g.imag[mask]).max())


# ----------------------------------------------------------------- one block


def extrapolate_block(signal, mask, values, gamma, iterations, rho_hat, tables=None,
                      record=False):
    """weight -> tables -> R0 -> recursion -> synthesis -> paste for one area
    (the per-block body of conceal.py:132-148 with fixed areas).

    ``values`` is (K, M, N); ``tables`` optionally a prebuilt (C, D) pair.
    Returns a dict with every intermediate the parity tests compare.
    """
    values = np.asarray(values)
    k = values.shape[0]
    phi = values.reshape(k, -1)
    w = weight_field(mask, rho_hat)
    if tables is None:
        tables = gram(phi, w)
    c, d = tables
    if (d == 0.0).all():
        raise ValueError("every atom has zero weighted energy")
    r0 = initial_products(signal, w, phi)
    sel, proj, coef, log = fase_run(r0, c, d, gamma, iterations, record=record)
    g = materialize(values, sel, coef)
    patched, max_imag = apply(np.asarray(signal, dtype=np.float64), g, mask)
    return {"weight": w, "r0": r0, "selected": sel, "projections": proj,
            "coefficients": coef, "log": log, "g": g, "patched": patched,
            "max_imag": max_imag, "d": d}
