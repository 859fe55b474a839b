// Issue-only tcgen05.mma kind::i8 probe: the dense INT8 tensor peak of this B200
// (the denominator of the Ozaki products' roofline, bench.py roofline_init).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o i8_peak_probe i8_peak_probe.cu
//   ./i8_peak_probe            -> one JSON line
//
// One CTA per SM; one thread issues back-to-back 128 x N x 32 int8 MMAs from
// fixed (zeroed) shared-memory operands into TMEM, alternating two accumulators,
// then commits to an mbarrier. No loads, no epilogue: the tensor pipe alone.
// ops = 2 * 128 * N * 32 per MMA; best of 5 timed launches (CUDA events).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint64_t umma_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return static_cast<uint64_t>((addr >> 4) & 0x3FFF) |
         (static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

template <int N>
__global__ void __launch_bounds__(128, 1) i8_issue_kernel(int iters, int* sink) {
  constexpr int BM = 128, BK = 64;
  __shared__ __align__(1024) uint8_t a[BM * BK];
  __shared__ __align__(1024) uint8_t b[N * BK];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x;
  for (int i = tid; i < BM * BK / 16; i += blockDim.x) reinterpret_cast<uint4*>(a)[i] = make_uint4(0, 0, 0, 0);
  for (int i = tid; i < N * BK / 16; i += blockDim.x) reinterpret_cast<uint4*>(b)[i] = make_uint4(0, 0, 0, 0);
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     smem_u32(&tmem_base)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 32) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n");
  }
  asm volatile("fence.proxy.async.shared::cta;\n");
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    // kind::i8, int32 accumulate, signed A/B, K-major, M = 128, N
    const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
                           (static_cast<uint32_t>(BM >> 4) << 24);
    const uint32_t sa = smem_u32(a), sb = smem_u32(b);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int ks = 0; ks < BK / 32; ++ks) {
        const uint64_t ad = umma_desc(sa + ks * 256, 128, 8 * BK);
        const uint64_t bd = umma_desc(sb + ks * 256, 128, 8 * BK);
        const uint32_t dst = tmem + static_cast<uint32_t>((it & 1) * 256);
        const uint32_t acc = it > 1 ? 1u : 0u;
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(dst),
            "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
      }
    }
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
            smem_u32(&bar)));
  }
  __syncwarp();
  {
    uint32_t done = 0;
    while (!done) {
      asm volatile(
          "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0, 1, 0, p;\n}\n"
          : "=r"(done) : "r"(smem_u32(&bar)));
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  uint32_t v;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];\n" : "=r"(v) : "r"(tmem + ((tid >> 5) << 21)));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n");
  if (v == 0x7fffffff) *sink = v;
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512));
}

template <int N>
double run(int sms, int iters, int* sink) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  i8_issue_kernel<N><<<sms, 128>>>(iters / 10, sink);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    i8_issue_kernel<N><<<sms, 128>>>(iters, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double ops = 2.0 * 128 * N * 64 * static_cast<double>(iters) * sms;  // 2 MMAs of K=32
  return ops / (best * 1e-3) / 1e12;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int* sink;
  cudaMalloc(&sink, 4);
  const int iters = 20000;
  const double t64 = run<64>(sms, iters, sink);
  const double t128 = run<128>(sms, iters, sink);
  const double t256 = run<256>(sms, iters, sink);
  cudaError_t err = cudaDeviceSynchronize();
  printf("{\"probe\": \"tcgen05.mma.cta_group::1.kind::i8 issue-only, M=128, K=32\", \"sms\": %d, "
         "\"tops_n64\": %.1f, \"tops_n128\": %.1f, \"tops_n256\": %.1f, \"status\": \"%s\"}\n",
         sms, t64, t128, t256, cudaGetErrorString(err));
  return err == cudaSuccess ? 0 : 1;
}
