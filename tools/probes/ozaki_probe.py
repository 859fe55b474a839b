"""Ozaki (tcgen05 INT8) FP64 contraction vs DMMA vs extended-precision reference."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2204_14194_b200 import _native  # noqa: E402

dev = torch.device("cuda", 0)
for (M, N, Kd, kind) in [(256, 128, 200, "uniform"), (4096, 8192, 3520, "c4"), (1000, 333, 777, "wide")]:
    rng = np.random.default_rng(M + N + Kd)
    if kind == "c4":
        X = rng.uniform(0, 255, (M, Kd)) * rng.uniform(0, 1, Kd)
        Y = rng.standard_normal((N, Kd)) / 64.0
    elif kind == "wide":
        X = rng.standard_normal((M, Kd)) * 10.0 ** rng.integers(-3, 4, (M, 1))
        Y = rng.standard_normal((N, Kd)) * 10.0 ** rng.integers(-3, 4, (1, Kd))
    else:
        X = rng.uniform(-1, 1, (M, Kd))
        Y = rng.uniform(-1, 1, (N, Kd))
    ld = Kd + (Kd & 1)
    Xd = torch.zeros((M, ld), dtype=torch.float64, device=dev); Xd[:, :Kd] = torch.from_numpy(X)
    Yd = torch.zeros((N, ld), dtype=torch.float64, device=dev); Yd[:, :Kd] = torch.from_numpy(Y)
    a = _native.OzakiOperand(M, Kd, 128, dev).split(Xd)
    b = _native.OzakiOperand(N, Kd, 64, dev).split(Yd)
    C = torch.zeros((M, N), dtype=torch.float64, device=dev)
    _native.ozaki_gemm(a, b, C)
    Cg = torch.zeros((M, N), dtype=torch.float64, device=dev)
    _native.gemm_nt(Xd, Yd, Cg)
    torch.cuda.synchronize()
    c, cg = C.cpu().numpy(), Cg.cpu().numpy()
    rows = rng.integers(0, M, 40); cols = rng.integers(0, N, 40)
    XL, YL = X.astype(np.longdouble), Y.astype(np.longdouble)
    ref = np.array([np.dot(XL[i], YL[j]) for i, j in zip(rows, cols)])
    scale = np.array([np.dot(np.abs(XL[i]), np.abs(YL[j])) for i, j in zip(rows, cols)])
    eo = np.abs(c[rows, cols] - ref) / scale
    eg = np.abs(cg[rows, cols] - ref) / scale
    print(f"{kind} M={M} N={N} K={Kd}: ozaki err/sum|xy| max {float(eo.max()):.2e}, dgemm {float(eg.max()):.2e}; "
          f"ozaki vs dgemm rel {float(np.abs(c - cg).max() / np.abs(cg).max()):.2e}")
    for name, fn in (("ozaki", lambda: (_native.OzakiOperand.split(a, Xd), _native.ozaki_gemm(a, b, C))),
                     ("ozaki-gemm-only", lambda: _native.ozaki_gemm(a, b, C)),
                     ("dmma", lambda: _native.gemm_nt(Xd, Yd, Cg))):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        print(f"   {name}: {ms:.3f} ms, FP64-equivalent {2 * M * N * Kd / ms / 1e9:.1f} TFLOP/s")
