"""The cluster recursion (csrc/iterate_cluster.cu): one block split over a
thread-block cluster of 4 or 8 CTAs, for batches of at most one CTA per SM.

It is dispatched by default where it measured faster (K > 4608, clusters of
8: the config-4 geometry, so the small-batch config-4 parity tests exercise
it) and on request (FASE_CLUSTER=4 / 8) elsewhere. Here it is pinned directly
against the one-CTA-per-block kernels (FASE_CLUSTER=0): same inputs,
bit-identical selections, projections, coefficients and synthesized samples,
exact and scaled recursions, fused synthesis, dead atoms and the
all-degenerate stop.
"""

from __future__ import annotations

import os

import numpy as np
import pytest
import torch

from paper_2204_14194_b200 import (
    Dictionary,
    ExtrapConfig,
    ExtrapolationPlan,
    build_gram_tables,
    build_weight_field,
    fase_extrapolate_batch,
)
from paper_2204_14194_b200 import workloads as wl

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0)


def _both(fn, cs="4"):
    """fn() with the cluster path forced on (FASE_CLUSTER=cs) and off (=0)."""
    os.environ["FASE_CLUSTER"] = cs
    on = [x.clone() for x in fn()]
    os.environ["FASE_CLUSTER"] = "0"
    try:
        off = [x.clone() for x in fn()]
    finally:
        os.environ.pop("FASE_CLUSTER", None)
    return on, off


@pytest.mark.parametrize("cid,blocks", [(0, 1), (0, 37), (1, 2), (1, 30), (4, 1), (4, 18)])
@pytest.mark.parametrize("recursion", ["exact", "scaled"])
def test_cluster_matches_single_cta(cid, blocks, recursion):
    w = wl.WORKLOADS[cid]
    d = w.dictionary()
    mask = wl.central_loss_mask(*w.area, *w.loss)
    cfg = ExtrapConfig(min(w.config.iterations, 120), w.config.gamma, w.config.rho_hat)
    t = build_gram_tables(d, build_weight_field(mask, cfg.rho_hat), device=DEV)
    sig = torch.from_numpy(wl.block_signals(cid, blocks, *w.area)).to(DEV)

    def run():
        p = ExtrapolationPlan(d, mask, blocks, cfg, t, device=DEV, recursion=recursion)
        p.run(sig)
        torch.cuda.synchronize()
        return [p.selected, p.projections, p.coefficients, p.lost]

    on, off = _both(run, "8" if len(d) > 4608 else "4")
    for a, b in zip(on, off):
        assert torch.equal(a, b)


def test_cluster_fused_synthesis_and_dead_atoms():
    """Atoms living only on lost samples (zero weighted energy) are never
    selected; the fused synthesis equals the separate kernel's output."""
    rng = np.random.default_rng(4)
    m = n = 16
    mask = wl.central_loss_mask(m, n, 6, 6)
    vals = rng.standard_normal((700, m, n))
    for k in (0, 5, 333, 699):
        vals[k] = 0.0
        vals[k][mask] = rng.standard_normal(int(mask.sum()))
    d = Dictionary(vals)
    cfg = ExtrapConfig(60, 0.5, 0.8)
    sig = rng.uniform(0, 255, (5, m, n))
    for rec in ("exact", "scaled"):
        on, off = _both(lambda: [r for r in (lambda x: (x.selected, x.coefficients, x.patched))(
            fase_extrapolate_batch(sig, mask, d, None, cfg, device=DEV, recursion=rec))])
        for a, b in zip(on, off):
            assert torch.equal(a, b)
        assert not np.isin(on[0].cpu().numpy(), [0, 5, 333, 699]).any()


def test_cluster_all_degenerate_stops():
    """Every atom dead in one block: the kernel marks the rest of the sequence
    (-1) and the batch API raises NoSelectableAtomError, as without clusters."""
    from paper_2204_14194_b200 import NoSelectableAtomError

    m = n = 8
    mask = wl.central_loss_mask(m, n, 4, 4)
    vals = np.zeros((64, m, n))
    for k in range(64):
        vals[k][mask] = np.random.default_rng(k).standard_normal(int(mask.sum()))
    d = Dictionary(vals)
    with pytest.raises(NoSelectableAtomError):
        fase_extrapolate_batch(np.ones((2, m, n)), mask, d, None, ExtrapConfig(5), device=DEV)
