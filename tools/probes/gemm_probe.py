"""Time the DMMA GEMM variants against cuBLAS on the c1 init-products shape."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2204_14194_b200 import _native
M, N, K = 1024, 4608, 2304
a = torch.randn(M, K, dtype=torch.float64, device="cuda")
b = torch.randn(N, K, dtype=torch.float64, device="cuda")
w = torch.rand(K, dtype=torch.float64, device="cuda")
ref = (a * w) @ b.T
def t(fn, n=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(n):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); e.synchronize(); best = min(best, s.elapsed_time(e))
    return best
for v in (0, 1):
    c = torch.empty(M, N, dtype=torch.float64, device="cuda")
    ms = t(lambda: _native.gemm_nt(a, b, c, v))
    err = ((c - a @ b.T).abs().max() / (a @ b.T).abs().max()).item()
    print(f"plain variant {v}: {ms:.3f} ms {2*M*N*K/ms/1e9:.2f} TF  relerr {err:.2e}")
c = torch.empty(M, N, dtype=torch.float64, device="cuda")
ms = t(lambda: _native.init_products(b, a, w, N, K, c))
print(f"scaled (init_products): {ms:.3f} ms {2*M*N*K/ms/1e9:.2f} TF  relerr {((c-ref).abs().max()/ref.abs().max()).item():.2e}")
ms = t(lambda: a @ b.T)
print(f"cublas: {ms:.3f} ms {2*M*N*K/ms/1e9:.2f} TF")
