// Shared helpers of libfase_b200: status plumbing and small device utilities.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>

#include "fase_b200.h"

namespace fase {

// Thread-local message of the last failing call (fase_last_error()).
void set_error(const char* fmt, ...);

inline int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return FASE_ERR_CUDA;
  }
  return FASE_OK;
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

__host__ __device__ inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// ---- device helpers --------------------------------------------------------

// Checked build (-DFASE_BOUNDS, tools/build_exp.sh bounds): data-derived
// indices are asserted in range and every mbarrier wait is bounded (a TMA whose
// expect_tx does not match the bytes delivered would hang; here it traps).
// compute-sanitizer is closed on this GPU pool, so this build plus the
// determinism / operand-integrity runs of tools/sanitize_cases.py stand in.
#ifdef FASE_BOUNDS
#define FASE_ASSERT(cond)                                                               \
  do {                                                                                  \
    if (!(cond)) {                                                                      \
      printf("FASE_BOUNDS %s:%d block %d thread %d: %s\n", __FILE__, __LINE__,           \
             static_cast<int>(blockIdx.x), static_cast<int>(threadIdx.x), #cond);       \
      __trap();                                                                         \
    }                                                                                   \
  } while (0)
#else
#define FASE_ASSERT(cond) \
  do {                    \
  } while (0)
#endif


// Correctly rounded multiply / subtract, never contracted into an FMA: the
// reference's numpy arithmetic rounds the product and the difference
// separately.
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }

// Max of a signed 64-bit key over the warp, from two 32-bit redux.sync steps.
__device__ __forceinline__ long long warp_max_i64(long long v) {
  const int hi = static_cast<int>(v >> 32);
  const unsigned lo = static_cast<unsigned>(v);
  const int mhi = __reduce_max_sync(0xffffffffu, hi);
  const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
  return (static_cast<long long>(mhi) << 32) | static_cast<long long>(mlo);
}

// g + sum_t coef[t] * phi[sel[t] * ldphi + m] for t ascending, stopping at the
// first sel < 0 (a block whose atoms were all degenerate): the reference's
// sequential summation order (SparseModel.materialize, reference.py:120-125).
// Atom values are fetched 8 terms at a time (independent loads in flight), then
// accumulated strictly in order. G: loads in flight (more for small, latency-
// bound batches).
template <int G = 8>
__device__ __forceinline__ double synth_terms(const double* __restrict__ phi, int64_t ldphi,
                                              const int32_t* s_sel, const double* s_coef,
                                              int len, int m, double g) {
  for (int t0 = 0; t0 < len; t0 += G) {
    double v[G];
#pragma unroll
    for (int j = 0; j < G; ++j) {
      const int t = t0 + j;
      const int u = t < len ? s_sel[t] : -1;
      FASE_ASSERT(u >= -1);
      v[j] = u >= 0 ? __ldg(phi + static_cast<int64_t>(u) * ldphi + m) : 0.0;
    }
#pragma unroll
    for (int j = 0; j < G; ++j) {
      const int t = t0 + j;
      if (t >= len || s_sel[t] < 0) return g;
      g = __dadd_rn(g, __dmul_rn(s_coef[t], v[j]));
    }
  }
  return g;
}

// ---- complex128 arithmetic exactly as numpy evaluates it --------------------
// (numpy 2.x contiguous complex loops, checked bit-for-bit against np on the
// build host: tests/golden/complex_arith.npz)
//
// product x * y = (fma(xr, yr, -(xi*yi)), fma(xr, yi, xi*yr)): the first
// operand's real part enters both fused multiply-adds.
__device__ __forceinline__ double2 np_cmul(double xr, double xi, double yr, double yi) {
  return make_double2(__fma_rn(xr, yr, -__dmul_rn(xi, yi)), __fma_rn(xr, yi, __dmul_rn(xi, yr)));
}

// |z| = larger * sqrt(fma(r, r, 1)), r = smaller / larger (0 when both vanish).
__device__ __forceinline__ double np_cabs(double re, double im) {
  const double a = fabs(re), b = fabs(im);
  const double hi = fmax(a, b), lo = fmin(a, b);
  if (hi == 0.0) return 0.0;
  const double r = __ddiv_rn(lo, hi);
  return __dmul_rn(__dsqrt_rn(__fma_rn(r, r, 1.0)), hi);
}

// ---- call-free correctly rounded division / square root on a narrow range ---
// The IEEE __ddiv_rn / __dsqrt_rn carry slow-path subroutine calls for special
// operands; inlined in a register-resident kernel, every call site forces the
// caller's live registers around it. These variants cover only normal operands
// in a fixed binade (the callers scale exactly into it) and are checked
// bit-for-bit against the IEEE operations (tools/probes/cabs_probe.cu).

// RN(a / b) for 1 <= b < 2 and 2^-61 <= a < 2: hardware reciprocal estimate, two
// Newton steps, one fused correction of the quotient (Markstein).
__device__ __forceinline__ double div_rn_unit(double a, double b) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(b));
  double e = __fma_rn(-b, y, 1.0);
  y = __fma_rn(y, e, y);
  e = __fma_rn(-b, y, 1.0);
  y = __fma_rn(y, e, y);
  const double q = __dmul_rn(a, y);
  const double r = __fma_rn(-b, q, a);
  return __fma_rn(r, y, q);
}

// RN(sqrt(t)) for 1 <= t <= 2: reciprocal square-root estimate, coupled
// Newton iterations for sqrt and 1/(2 sqrt), one fused final correction.
__device__ __forceinline__ double sqrt_rn_unit(double t) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(t));
  double s = __dmul_rn(t, y);
  double h = 0.5 * y;
  double e = __fma_rn(-s, h, 0.5);
  s = __fma_rn(s, e, s);
  h = __fma_rn(h, e, h);
  e = __fma_rn(-s, h, 0.5);
  s = __fma_rn(s, e, s);
  h = __fma_rn(h, e, h);
  const double d = __fma_rn(-s, s, t);
  return __fma_rn(d, h, s);
}

// np_cabs without subroutine calls: identical results for finite inputs.
// lo <= hi * 2^-61 gives r^2 < 2^-122, so fma(r, r, 1) == 1 and |z| == hi.
// Otherwise both are scaled by the same power of two (exact) into hi in [1, 2).
__device__ __forceinline__ double np_cabs_fast(double re, double im) {
  const double a = fabs(re), b = fabs(im);
  const double hi = fmax(a, b), lo = fmin(a, b);
  if (hi == 0.0) return 0.0;
  if (lo <= hi * 0x1p-61) return hi;
  long long hb = __double_as_longlong(hi);
  double hs = hi, ls = lo;
  if ((hb >> 52) == 0) {  // subnormal: lift by 2^64 first (exact)
    hs *= 0x1p64;
    ls *= 0x1p64;
    hb = __double_as_longlong(hs);
  }
  const int ex = static_cast<int>(hb >> 52) - 1023;  // hs in [2^ex, 2^(ex+1))
  // 2^-ex as a double (ex in [-1022 - 64, 1023]; split in two factors to stay normal)
  const int e1 = -ex / 2, e2 = -ex - e1;
  const double f1 = __longlong_as_double(static_cast<long long>(e1 + 1023) << 52);
  const double f2 = __longlong_as_double(static_cast<long long>(e2 + 1023) << 52);
  hs = (hs * f1) * f2;
  ls = (ls * f1) * f2;
  const double r = div_rn_unit(ls, hs);
  return __dmul_rn(sqrt_rn_unit(__fma_rn(r, r, 1.0)), hi);
}

__device__ __forceinline__ double2 ldg2(const double* p) {
  return __ldg(reinterpret_cast<const double2*>(p));
}

// ld.global.nc as a volatile asm: stays where it is written relative to other
// volatile asm (e.g. an mbarrier wait), so a batch of loads issued before a
// wait is not hoisted into one long-lived register block by the compiler.
__device__ __forceinline__ double2 ldg2_here(const double* p) {
  double2 v;
  asm volatile("ld.global.nc.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}

__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];\n" ::"l"(p));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
// 8-byte async copy (L1-allocating); src_bytes 0 writes zeros
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }

// ---- mbarrier + TMA 1-D bulk copy (cp.async.bulk), sm_90+ / sm_100a ---------

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

// Make barrier initialization visible to the async (TMA) proxy.
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}

// Proxy fence before a TMA refill of a staging buffer (measurement knob):
// the buffer's previous generic-proxy reads are already ordered by the block
// barrier between them and the issue, and generic WRITES (row composition) are
// followed by their own fence, so the issue-time fence only orders what is
// already ordered (FASE_ISSUE_FENCE=0 drops it)
// Scaled recursion variants (bits; see iterate.cu): 1 signed running max,
// 2 D prefetch, 4 fused update (iterate.cu and iterate_cluster.cu), 8 tie-dump
// shortcut, 16 issue-warp offset, 32 integer running max (24-32 elements per thread)
#ifndef FASE_SCALED_LEAN
#define FASE_SCALED_LEAN 45
#endif
#ifndef FASE_ISSUE_FENCE
#define FASE_ISSUE_FENCE 1
#endif
__device__ __forceinline__ void fence_before_refill() {
#if FASE_ISSUE_FENCE
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
#endif
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

// One-thread bulk copy global -> shared; completion is signalled on `bar`.
__device__ __forceinline__ void tma_load_1d(void* smem_dst, const void* gmem_src, unsigned bytes,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::
          "r"(smem_u32(smem_dst)),
      "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// The same bulk copy with an L2 cache-policy hint (createpolicy): rows marked
// hot (fase_iterate_args.l2_hot) are copied evict_last, the others evict_first.
__device__ __forceinline__ void tma_load_1d_hint(void* smem_dst, const void* gmem_src, unsigned bytes,
                                                 uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], "
      "%2, [%3], %4;\n" ::"r"(smem_u32(smem_dst)),
      "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

__device__ __forceinline__ uint64_t l2_policy(bool keep) {
  uint64_t p;
  if (keep)
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
  else
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}

#ifdef FASE_BOUNDS
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  for (long long spin = 0;; ++spin) {
    unsigned done;
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (done) return;
    FASE_ASSERT(spin < (1ll << 26));  // ~seconds: a transfer that never completes
  }
}
#else
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
#endif
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

}  // namespace fase
