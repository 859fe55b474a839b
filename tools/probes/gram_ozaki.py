"""Gram build: DMMA symmetric GEMM vs tcgen05 Ozaki (planes pre-split / with split)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2204_14194_b200 import _native, build_weight_field, workloads as wl  # noqa: E402

dev = torch.device("cuda", 0)
for cid in (1, 4):
    w8 = wl.WORKLOADS[cid]
    d = w8.dictionary()
    K, M = len(d), w8.area[0] * w8.area[1]
    phi = d.device_matrix(dev)
    w = build_weight_field(wl.central_loss_mask(*w8.area, *w8.loss), w8.config.rho_hat).ravel()
    wd = torch.zeros(phi.shape[1], dtype=torch.float64, device=dev)
    wd[:M] = torch.from_numpy(w).to(dev)
    sup = torch.nonzero(wd[:M] != 0).flatten()
    sidx, ws = sup.to(torch.int32), wd.index_select(0, sup).contiguous()
    n_s = int(sup.numel())
    G1 = torch.zeros((K, _native.table_ld(K)), dtype=torch.float64, device=dev)
    G2 = torch.zeros_like(G1)
    gws = torch.empty(K * phi.shape[1] + 2, dtype=torch.float64, device=dev)
    a = _native.OzakiOperand(K, n_s, 128, dev)
    b = _native.OzakiOperand(K, n_s, 64, dev)

    def t(fn, n=5):
        fn(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(n):
            fn()
        e1.record(); torch.cuda.synchronize()
        return e0.elapsed_time(e1) / n

    td = t(lambda: _native.gram(phi, wd, K, M, G1, ws=gws))
    ts = t(lambda: (a.split(phi, sidx, ws), b.split(phi, sidx)))
    tg = t(lambda: _native.ozaki_gram(a, b, G2))
    g1, g2 = G1[:, :K].cpu().numpy(), G2[:, :K].cpu().numpy()
    print(f"c{cid} K={K} M={M} support={n_s}: dmma {td:.3f} ms, ozaki split {ts:.3f} + gram {tg:.3f} ms; "
          f"sym {np.array_equal(g2, g2.T)}; rel diff {np.abs(g1 - g2).max() / np.abs(g1).max():.2e}")

    # the bench's timed sequence: support, fresh operands, split, gram, finish
    from paper_2204_14194_b200.fast import gram_into, gram_support  # noqa: E402
    D2 = torch.empty(K, dtype=torch.float64, device=dev)
    tsup = t(lambda: gram_support(wd, M))
    tall = t(lambda: gram_into(phi, wd, K, M, G2))
    tfin = t(lambda: _native.gram_finish(G2, K, D2))
    print(f"c{cid}: gram_support {tsup:.3f} ms, gram_into (alloc+split+gram) {tall:.3f} ms, finish {tfin:.3f} ms")
