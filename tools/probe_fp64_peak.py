"""Measure the FP64 roofline denominators on the B200 box.

cuBLAS DGEMM (CUBLAS_COMPUTE_64F via torch.matmul on float64) at 8192^3, best
of 10 with CUDA events, plus a float64 copy bandwidth probe. Writes
gpurun_out/fp64_peak.json. Used only to set the FP64 denominator that
MEASURED_PEAKS.json does not carry.
"""
import json
import os
import torch

def main():
    dev = torch.device("cuda:0")
    torch.manual_seed(0)
    out = {"gpu": torch.cuda.get_device_name(0)}
    for n in (4096, 8192):
        a = torch.randn(n, n, dtype=torch.float64, device=dev)
        b = torch.randn(n, n, dtype=torch.float64, device=dev)
        for _ in range(3):
            torch.matmul(a, b)
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(10):
            s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
            s.record(); torch.matmul(a, b); e.record(); e.synchronize()
            best = min(best, s.elapsed_time(e))
        out[f"dgemm_{n}_tflops"] = 2 * n**3 / (best * 1e-3) / 1e12
        out[f"dgemm_{n}_ms"] = best
    # NT-shaped (both operands contraction-contiguous), like the Gram
    k, m = 4608, 2304
    phi = torch.randn(k, m, dtype=torch.float64, device=dev)
    for _ in range(3):
        phi @ phi.T
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); phi @ phi.T; e.record(); e.synchronize()
        best = min(best, s.elapsed_time(e))
    out["dgemm_gram_4608x2304_tflops"] = 2 * k * k * m / (best * 1e-3) / 1e12
    x = torch.empty(1 << 28, dtype=torch.float64, device=dev)
    y = torch.empty_like(x)
    for _ in range(3):
        y.copy_(x)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); y.copy_(x); e.record(); e.synchronize()
        best = min(best, s.elapsed_time(e))
    out["copy_gbs"] = 2 * x.numel() * 8 / (best * 1e-3) / 1e9
    props = torch.cuda.get_device_properties(0)
    out["sms"] = props.multi_processor_count
    out["l2_bytes"] = getattr(props, "L2_cache_size", None)
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/fp64_peak.json", "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out))

if __name__ == "__main__":
    main()
