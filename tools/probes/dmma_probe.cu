// DMMA (mma.sync m8n8k4 f64) issue-rate probe: registers only, no memory.
#include <cstdio>
#include <cuda_runtime.h>
template <int ACC>
__global__ void dmma_loop(double* out, int iters) {
  double c[ACC][2];
  double a = threadIdx.x * 1e-3, b = 1.0 + blockIdx.x * 1e-6;
  for (int i = 0; i < ACC; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int i = 0; i < ACC; ++i) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int ACC>
void run(int blocks, int threads) {
  double* out;
  cudaMalloc(&out, sizeof(double) * blocks * threads);
  int iters = 4096;
  dmma_loop<ACC><<<blocks, threads>>>(out, 16);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  dmma_loop<ACC><<<blocks, threads>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double flops = 512.0 * ACC * iters * (double)blocks * (threads / 32);
  printf("ACC=%2d blocks=%4d threads=%4d : %.2f TFLOP/s\n", ACC, blocks, threads, flops / (ms * 1e-3) / 1e12);
  cudaFree(out);
}
int main() {
  for (int t : {128, 256, 512, 1024}) { run<16>(148, t); run<32>(148, t); }
  run<8>(148 * 4, 256); run<16>(148 * 2, 512);
  return 0;
}
