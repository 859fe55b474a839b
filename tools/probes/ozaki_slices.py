import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2204_14194_b200 import _native
dev = torch.device("cuda", 0)
M, N, Kd = 4096, 8192, 3520
rng = np.random.default_rng(1)
Xd = torch.from_numpy(rng.uniform(0, 255, (M, Kd))).to(dev)
Yd = torch.from_numpy(rng.standard_normal((N, Kd)) / 64).to(dev)
C = torch.zeros((M, N), dtype=torch.float64, device=dev)
for s in (6, 7, 8):
    a = _native.OzakiOperand(M, Kd, 128, dev, slices=s).split(Xd)
    b = _native.OzakiOperand(N, Kd, 64, dev, slices=s).split(Yd)
    for _ in range(2): _native.ozaki_gemm(a, b, C)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): _native.ozaki_gemm(a, b, C)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    pairs = s * (s + 1) // 2
    print(f"s={s}: {ms:.3f} ms; int8 {pairs * 2 * M * N * Kd / ms / 1e9:.0f} TOPS; bytes/stage {s * 12} KB")
