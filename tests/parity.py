"""Parity helpers shared by the CPU and GPU tests (test infrastructure).

The BASELINE acceptance rule (BASELINE.json north_star): the selected
sequence must be bit-exact except where the top-two Delta-E = metric^2 differ
by less than 1e-9 relative; coefficients and reconstructed samples within
1e-6 relative (FP64). Deviations are measured against the run scale, as the
reference's own harness does (``pkg/src/fase/verify.py:52-54``).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

TIE_REL = 1e-9        # top-two Delta-E gap below which a divergence is allowed
COEF_REL = 1e-6       # run-scale coefficient / sample tolerance (BASELINE)


def rel_dev(a, b) -> float:
    """max |a - b| / max(|a|, |b|) (real or complex)."""
    a = np.asarray(a)
    b = np.asarray(b)
    if not (np.iscomplexobj(a) or np.iscomplexobj(b)):
        a = a.astype(np.float64)
        b = b.astype(np.float64)
    scale = max(float(np.abs(a).max(initial=0.0)), float(np.abs(b).max(initial=0.0)), 1e-300)
    return float(np.abs(a - b).max(initial=0.0)) / scale


@dataclass
class SeqVerdict:
    exact: bool          # whole sequence identical
    ok: bool             # identical, or diverged only at a legitimate near-tie
    stop: int            # first diverging iteration (== len when exact)
    gap: float | None    # relative Delta-E gap at the divergence


def compare_selection(got, want, metric_at) -> SeqVerdict:
    """Compare selection sequences; ``metric_at(t)`` gives the reference
    metric vector |R|*D before iteration t (only called at a divergence)."""
    got = np.asarray(got).astype(np.int64)
    want = np.asarray(want).astype(np.int64)
    diff = np.flatnonzero(got != want)
    if diff.size == 0:
        return SeqVerdict(True, True, len(want), None)
    t = int(diff[0])
    m = np.asarray(metric_at(t), dtype=np.float64)
    e1 = m[want[t]] ** 2
    e2 = m[got[t]] ** 2
    gap = abs(e1 - e2) / max(e1, e2, 1e-300)
    return SeqVerdict(False, gap < TIE_REL, t, gap)


def metric_fn(r0, d, log):
    """metric_at(t) from a reference run: R before iteration t is r0 or log[t-1]."""
    r0 = np.asarray(r0)
    d = np.asarray(d)

    def at(t):
        r = r0 if t == 0 else np.asarray(log[t - 1])
        m = np.abs(r) * d
        m[d == 0] = -np.inf
        return m

    return at
