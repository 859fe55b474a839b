// L2 -> SM read bandwidth on the B200 (the bound of the table-row streams of
// the recursion and the synthesis, whose working sets are L2-resident).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_probe l2_probe.cu && ./l2_probe
//
// Every CTA streams a buffer of S bytes with 16-byte ld.global.cg loads (L2
// only, no L1 reuse), 8 loads in flight per thread, for several passes; the
// result is the total bytes read / kernel time (CUDA events, best of 5).
// S below the L2 capacity measures L2 bandwidth, S = 2 GiB measures DRAM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint4 ld_cg(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

__global__ void __launch_bounds__(512) read_kernel(const uint4* buf, size_t n, int passes,
                                                   unsigned* sink) {
  unsigned acc = 0;
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (int p = 0; p < passes; ++p) {
    // rotate the start so consecutive passes do not hit the same lines first
    const size_t off = (static_cast<size_t>(p) * 7919 * blockDim.x) % n;
    for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += 8 * stride) {
      uint4 v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        size_t k = i + j * stride;
        if (k < n) {
          k += off;
          if (k >= n) k -= n;
          v[j] = ld_cg(buf + k);
        } else {
          v[j] = make_uint4(0, 0, 0, 0);
        }
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) acc ^= v[j].x ^ v[j].y ^ v[j].z ^ v[j].w;
    }
  }
  if (acc == 0x12345678u) *sink = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned* sink;
  cudaMalloc(&sink, 4);
  const size_t sizes_mb[] = {8, 16, 32, 48, 64, 96, 2048};
  printf("{\"sms\": %d, \"results\": [", sms);
  bool first = true;
  for (size_t mb : sizes_mb) {
    const size_t bytes = mb << 20;
    const size_t n = bytes / sizeof(uint4);
    uint4* buf;
    cudaMalloc(&buf, bytes);
    cudaMemset(buf, 1, bytes);
    const int passes = mb >= 1024 ? 4 : static_cast<int>(8192 / mb);
    const int grid = sms * 4;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    read_kernel<<<grid, 512>>>(buf, n, 1, sink);  // warm (fills L2)
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0);
      read_kernel<<<grid, 512>>>(buf, n, passes, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    const double gbs = static_cast<double>(bytes) * passes / (best * 1e-3) / 1e9;
    printf("%s{\"mb\": %zu, \"passes\": %d, \"ms\": %.4f, \"read_gbs\": %.1f}", first ? "" : ", ", mb,
           passes, best, gbs);
    first = false;
    cudaFree(buf);
  }
  printf("]}\n");
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
