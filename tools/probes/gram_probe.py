"""Time the Gram build pieces on the c1 shape (weigh, symmetric GEMM, finish)."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2204_14194_b200 import _native, workloads as wl, build_weight_field
w8 = wl.WORKLOADS[1]
d = w8.dictionary()
K, M = len(d), 2304
phi = d.device_matrix("cuda:0")
mask = wl.central_loss_mask(48, 48, 16, 16)
w = torch.from_numpy(build_weight_field(mask, 0.8).ravel()).cuda()
G = torch.zeros(K, _native.table_ld(K), dtype=torch.float64, device="cuda")
ws = torch.empty(K * M + 2, dtype=torch.float64, device="cuda")
def t(fn, n=5):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(n):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); e.synchronize(); best = min(best, s.elapsed_time(e))
    return best
ms = t(lambda: _native.gram(phi, w, K, M, G, ws=ws))
print(f"fase_gram: {ms:.3f} ms  {K*(K+1)*M/ms/1e9:.2f} TF(alg)")
pw = (phi[:, :M] * w).contiguous()
C = torch.empty(K, K, dtype=torch.float64, device="cuda")
ms = t(lambda: _native.gemm_nt(pw, phi, C))
print(f"full (non-sym) gemm_nt KxKxM: {ms:.3f} ms {2*K*K*M/ms/1e9:.2f} TF")
ms = t(lambda: torch.matmul(pw, phi[:, :M].T))
print(f"cublas KxKxM: {ms:.3f} ms {2*K*K*M/ms/1e9:.2f} TF")
