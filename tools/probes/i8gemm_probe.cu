// Probe: tcgen05 kind::i8 GEMM on sm_100a (C[int32] = A[int8, MxK] . B[int8, NxK]^T),
// the building block of the FP64-by-INT8 (Ozaki) products. Validates the
// shared-memory / instruction descriptors and the TMEM epilogue against a CPU
// reference, and reports int8 TOPS.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o i8gemm_probe i8gemm_probe.cu
//   ./i8gemm_probe [M N K]
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess) {                                                         \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__);     \
      exit(1);                                                                       \
    }                                                                                \
  } while (0)

constexpr int BM = 128, BN = 64, BKB = 64;  // tile rows, cols, K bytes per stage
constexpr int STAGES = 4;
constexpr int A_STAGE = BM * BKB, B_STAGE = BN * BKB;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// K-major, no swizzle: core matrices of 8 rows x 16 B; LBO = next core along K,
// SBO = next 8-row group. Version 1 (sm_100).
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return static_cast<uint64_t>((addr >> 4) & 0x3FFF) |
         (static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

constexpr uint32_t kIdesc = (2u << 4) | (1u << 7) | (1u << 10) | (uint32_t(BN >> 3) << 17) |
                            (uint32_t(BM >> 4) << 24);

__device__ __forceinline__ void cp_async16(uint32_t s, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(g));
}

__global__ void __launch_bounds__(128, 1) i8gemm(const int8_t* __restrict__ A, const int8_t* __restrict__ B,
                                                 int32_t* __restrict__ C, int M, int N, int K) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_STAGE;
  __shared__ __align__(8) uint64_t mbar[STAGES];
  __shared__ __align__(8) uint64_t done_bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int nk = K / BKB;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base)),
                 "r"(64));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&mbar[s])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&done_bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = tmem_base;

  auto load = [&](int kb, int st) {
    // A: 128 rows x 4 chunks of 16 B; B: 64 rows x 4 chunks
    for (int c = tid; c < BM * 4; c += 128) {
      const int r = c >> 2, kc = c & 3;
      const uint32_t off = (r >> 3) * 512 + kc * 128 + (r & 7) * 16;
      cp_async16(smem_u32(sA + st * A_STAGE + off), A + static_cast<int64_t>(m0 + r) * K + kb * BKB + kc * 16);
    }
    for (int c = tid; c < BN * 4; c += 128) {
      const int r = c >> 2, kc = c & 3;
      const uint32_t off = (r >> 3) * 512 + kc * 128 + (r & 7) * 16;
      cp_async16(smem_u32(sB + st * B_STAGE + off), B + static_cast<int64_t>(n0 + r) * K + kb * BKB + kc * 16);
    }
    asm volatile("cp.async.commit_group;\n");
  };

  uint32_t phase[STAGES] = {0, 0, 0, 0};
  for (int s = 0; s < STAGES - 1 && s < nk; ++s) load(s, s);
  for (int kb = 0; kb < nk; ++kb) {
    const int st = kb % STAGES;
    // loads of stage kb complete (groups are issued in order)
    if (kb + STAGES - 1 <= nk) asm volatile("cp.async.wait_group %0;\n" ::"n"(STAGES - 2));
    else asm volatile("cp.async.wait_group 0;\n");
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;\n");
      for (int s = 0; s < 2; ++s) {
        const uint64_t ad = smem_desc(smem_u32(sA + st * A_STAGE) + s * 256, 128, 512);
        const uint64_t bd = smem_desc(smem_u32(sB + st * B_STAGE) + s * 256, 128, 512);
        const uint32_t acc = (kb | s) ? 1u : 0u;
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
            "l"(ad), "l"(bd), "r"(kIdesc), "r"(acc));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
          smem_u32(&mbar[st])));
    }
    // refill the stage used STAGES-1 iterations ahead once its MMAs are done
    const int nkb = kb + STAGES - 1;
    if (nkb < nk) {
      const int nst = nkb % STAGES;
      if (nkb >= STAGES) {  // the previous occupant (iteration nkb - STAGES) must be consumed
        asm volatile(
            "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
                smem_u32(&mbar[nst])),
            "r"(phase[nst]));
        phase[nst] ^= 1;
      }
      load(nkb, nst);
    }
  }
  if (tid == 0)
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
        smem_u32(&done_bar)));
  asm volatile("{\n.reg .pred p;\nW2_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W2_%=;\n}\n" ::"r"(
      smem_u32(&done_bar)));
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  // epilogue: warp w reads TMEM lanes 32w..32w+31 (tile rows), 64 columns
  uint32_t v[16];
  const int row = m0 + warp * 32 + (tid & 31);
  for (int c0 = 0; c0 < BN; c0 += 16) {
    const uint32_t taddr = tmem + (static_cast<uint32_t>(warp * 32) << 16) + c0;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n");
    for (int j = 0; j < 16; ++j) C[static_cast<int64_t>(row) * N + n0 + c0 + j] = static_cast<int32_t>(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(64));
}

int main(int argc, char** argv) {
  int M = argc > 3 ? atoi(argv[1]) : 1024, N = argc > 3 ? atoi(argv[2]) : 1024, K = argc > 3 ? atoi(argv[3]) : 1024;
  std::vector<int8_t> a(size_t(M) * K), b(size_t(N) * K);
  srand(1);
  for (auto& x : a) x = int8_t(rand() % 255 - 127);
  for (auto& x : b) x = int8_t(rand() % 255 - 127);
  int8_t *dA, *dB;
  int32_t* dC;
  CK(cudaMalloc(&dA, a.size()));
  CK(cudaMalloc(&dB, b.size()));
  CK(cudaMalloc(&dC, sizeof(int32_t) * M * N));
  CK(cudaMemcpy(dA, a.data(), a.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, b.data(), b.size(), cudaMemcpyHostToDevice));
  const size_t smem = STAGES * (A_STAGE + B_STAGE);
  CK(cudaFuncSetAttribute(i8gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  dim3 grid(N / BN, M / BM);
  i8gemm<<<grid, 128, smem>>>(dA, dB, dC, M, N, K);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<int32_t> c(size_t(M) * N);
  CK(cudaMemcpy(c.data(), dC, sizeof(int32_t) * c.size(), cudaMemcpyDeviceToHost));
  long bad = 0;
  for (int i = 0; i < M; i += 37)
    for (int j = 0; j < N; j += 11) {
      int64_t s = 0;
      for (int k = 0; k < K; ++k) s += int(a[size_t(i) * K + k]) * int(b[size_t(j) * K + k]);
      if (s != c[size_t(i) * N + j]) {
        if (bad < 5) printf("mismatch (%d,%d): %lld vs %d\n", i, j, (long long)s, c[size_t(i) * N + j]);
        ++bad;
      }
    }
  printf("check: %ld mismatches\n", bad);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  const int reps = 20;
  for (int r = 0; r < reps; ++r) i8gemm<<<grid, 128, smem>>>(dA, dB, dC, M, N, K);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("M=%d N=%d K=%d: %.3f ms/launch, %.1f TOPS\n", M, N, K, ms / reps, 2.0 * M * N * K / (ms / reps * 1e-3) / 1e12);
  return bad != 0;
}
