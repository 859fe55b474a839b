"""Result types shared by every extrapolation entry point.

``IterationTrace`` and ``SparseModel`` keep the reference's field names and
semantics (``pkg/src/fase/reference.py:88-125``) so code written against the
reference reads results the same way. ``BatchResult`` is the batched form
returned by ``fase_extrapolate_batch``; it holds device tensors and converts
to per-block ``(SparseModel, IterationTrace)`` pairs on request.

The selection constants are the reference's (``reference.py:36,55``); the
device kernels hard-code the same values (csrc/iterate.cu, csrc/capi.cu).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

DEGENERACY_RTOL = 1e-12
SELECTION_TIE_RTOL = 1e-13


@dataclass
class IterationTrace:
    """Per-iteration record: selected atom, raw projection, applied coefficient.

    ``products`` holds the R vector after every iteration when recording was
    requested (the fast path never materializes residual fields, so
    ``residuals`` stays None, as in the reference's fast path).
    """

    selected: np.ndarray
    projections: np.ndarray
    coefficients: np.ndarray
    residuals: list | None = None
    products: list | None = None

    def __len__(self) -> int:
        return len(self.selected)


@dataclass
class SparseModel:
    """g = sum of c * phi_k over the selected terms, in selection order."""

    shape: tuple[int, int]
    terms: list
    dictionary: object

    def materialize(self) -> np.ndarray:
        """Evaluate g over the full area on the host (reference.py:120-125 order)."""
        vals = self.dictionary.values
        g = np.zeros(self.shape, dtype=np.complex128)
        for k, c in self.terms:
            g += c * vals[k]
        return g


_PINNED = {}  # (shape, dtype) -> pinned host staging buffer of BatchResult.to_host


@dataclass
class BatchResult:
    """Outcome of one batched run over B blocks (device tensors).

    selected: (B, I) int32; projections, coefficients: (B, I) float64
    (complex128 for complex dictionaries); patched: (B, M, N) float64 areas
    with lost samples replaced (Re g), or None; products: (B, I, K) record of R
    when requested, else None; max_imag: (B,) max |Im g| over each block's
    lost samples for complex dictionaries (apply_model's diagnostic), else None.
    """

    selected: object
    projections: object
    coefficients: object
    patched: object = None
    products: object = None
    dictionary: object = None
    shape: tuple[int, int] | None = None
    max_imag: object = None

    def __len__(self) -> int:
        return int(self.selected.shape[0])

    def to_host(self, fields=("selected", "coefficients", "patched")) -> dict:
        """Host numpy copies of the named fields through reusable pinned staging
        buffers (one per shape / dtype, kept across calls): a read-back at
        PCIe rate instead of a pageable copy into fresh, page-faulting memory
        (config 4's 134 MB of patched areas: 61 ms pageable). The arrays are
        views of the staging buffers, valid until the next ``to_host`` with
        the same shape and dtype; copy them to keep them longer."""
        import torch

        out, pending = {}, []
        for name in fields:
            t = getattr(self, name)
            if t is None:
                out[name] = None
                continue
            key = (tuple(t.shape), t.dtype)
            buf = _PINNED.get(key)
            if buf is None:
                buf = _PINNED[key] = torch.empty(key[0], dtype=key[1], pin_memory=True)
            buf.copy_(t, non_blocking=True)
            pending.append((name, buf))
        if pending:
            torch.cuda.current_stream(self.selected.device).synchronize()
        for name, buf in pending:
            out[name] = buf.numpy()
        return out

    def block(self, b: int) -> tuple[SparseModel, IterationTrace]:
        """Per-block reference-style (model, trace) pair (host copies)."""
        sel = self.selected[b].cpu().numpy().astype(np.intp)
        proj = self.projections[b].cpu().numpy().astype(np.complex128)
        coef = self.coefficients[b].cpu().numpy().astype(np.complex128)
        prods = None
        if self.products is not None:
            prods = [p.astype(np.complex128) for p in self.products[b].cpu().numpy()]
        terms = [(int(k), complex(c)) for k, c in zip(sel, coef)]
        model = SparseModel(shape=self.shape, terms=terms, dictionary=self.dictionary)
        trace = IterationTrace(selected=sel, projections=proj, coefficients=coef, products=prods)
        return model, trace
