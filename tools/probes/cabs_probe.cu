// Bit-for-bit check of the call-free div / sqrt / |z| (csrc/common.cuh) against
// the IEEE operations on random and targeted operands.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../include -I../../paper_2204_14194_b200/csrc -o cabs_probe cabs_probe.cu
#include <cstdio>
#include <cstdlib>

#include "common.cuh"

namespace fase {
void set_error(const char*, ...) {}
}
using namespace fase;

__device__ unsigned long long g_bad[4];
__device__ unsigned long long g_first[4][3];

__device__ __forceinline__ unsigned long long mix(unsigned long long x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33;
  return x;
}

__device__ void report(int which, double a, double b, double got) {
  const unsigned long long n = atomicAdd(&g_bad[which], 1ULL);
  if (n == 0) {
    g_first[which][0] = __double_as_longlong(a);
    g_first[which][1] = __double_as_longlong(b);
    g_first[which][2] = __double_as_longlong(got);
  }
}

__global__ void probe(unsigned long long base, int per_thread) {
  const unsigned long long tid = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
  for (int i = 0; i < per_thread; ++i) {
    const unsigned long long s = mix(base + tid * per_thread + i);
    const unsigned long long s2 = mix(s ^ 0x9e3779b97f4a7c15ULL);
    // division: b in [1, 2), a in [2^-61, 2) with random mantissas; mode bits pick hard cases
    double b = __longlong_as_double((1023LL << 52) | (s & 0xFFFFFFFFFFFFFULL));
    if ((s2 & 15) == 0) b = __longlong_as_double((1023LL << 52) | 0xFFFFFFFFFFFFFULL - (s2 >> 60));
    const int ea = -(int)((s2 >> 8) % 62);
    double a = __longlong_as_double((long long)(1023 + ea) << 52 | (s2 & 0xFFFFFFFFFFFFFULL) ^ (s >> 12));
    if ((s2 & 0x70) == 0x10) {  // a = b * q for q a midpoint-ish value
      const double q = __longlong_as_double((1022LL << 52) | (s2 & 0xFFFFFFFFFFFFEULL) | 1);
      a = __dmul_rn(b, q);
    }
    if (a < 2.0 && a >= 0x1p-61 && div_rn_unit(a, b) != __ddiv_rn(a, b)) report(0, a, b, div_rn_unit(a, b));
    // sqrt on [1, 2]
    const double t = __longlong_as_double((1023LL << 52) | (s & 0xFFFFFFFFFFFFFULL));
    if (sqrt_rn_unit(t) != __dsqrt_rn(t)) report(1, t, 0, sqrt_rn_unit(t));
    if (sqrt_rn_unit(2.0) != __dsqrt_rn(2.0)) report(1, 2.0, 0, sqrt_rn_unit(2.0));
    // |z| over the full finite range, equal magnitudes, zeros, tiny ratios
    const int e1 = (int)(s2 % 2046) + 1, e2 = (int)((s2 >> 11) % 2046) + 1;
    double re = __longlong_as_double((long long)e1 << 52 | (s & 0xFFFFFFFFFFFFFULL));
    double im = __longlong_as_double((long long)e2 << 52 | (s2 & 0xFFFFFFFFFFFFFULL));
    switch ((s >> 56) & 7) {
      case 0: im = re; break;
      case 1: im = 0.0; break;
      case 2: im = re * 0x1p-30; break;
      case 3: re = __longlong_as_double(s & 0xFFFFFFFFFFFFFULL); break;  // subnormal
      case 4: im = re * (1.0 + 0x1p-52 * (s2 & 7)); break;
      case 5: re = re * 0x1p-600; im = im * 0x1p-600; break;
      default: break;
    }
    if ((s >> 55) & 1) re = -re;
    if ((s >> 54) & 1) im = -im;
    if (__double_as_longlong(np_cabs_fast(re, im)) != __double_as_longlong(np_cabs(re, im)))
      report(2, re, im, np_cabs_fast(re, im));
    // the recursion's operating range: |z| ~ 1e-3 .. 1e7, ratio anything
    const double re2 = (double)(s % 10000000) * 1e-3 * ((s >> 63) ? -1 : 1) + 1e-9 * (s2 & 1023);
    const double im2 = (double)(s2 % 10000000) * 1e-3 * ((s2 >> 63) ? -1 : 1);
    if (__double_as_longlong(np_cabs_fast(re2, im2)) != __double_as_longlong(np_cabs(re2, im2)))
      report(3, re2, im2, np_cabs_fast(re2, im2));
  }
}

int main(int argc, char** argv) {
  const int rounds = argc > 1 ? atoi(argv[1]) : 16;
  const int blocks = 148 * 8, threads = 256, per = 256;
  for (int r = 0; r < rounds; ++r) probe<<<blocks, threads>>>((unsigned long long)r * blocks * threads * per, per);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 2; }
  unsigned long long bad[4], first[4][3];
  cudaMemcpyFromSymbol(bad, g_bad, sizeof(bad));
  cudaMemcpyFromSymbol(first, g_first, sizeof(first));
  const double n = (double)rounds * blocks * threads * per;
  const char* names[4] = {"div_rn_unit", "sqrt_rn_unit", "np_cabs_fast (full range)", "np_cabs_fast (operating range)"};
  int rc = 0;
  for (int i = 0; i < 4; ++i) {
    printf("%-32s %.3g cases, %llu mismatches", names[i], n, bad[i]);
    if (bad[i]) {
      double x[3]; memcpy(x, first[i], sizeof(x));
      printf("  first: %.17g %.17g -> %.17g", x[0], x[1], x[2]);
      rc = 1;
    }
    printf("\n");
  }
  return rc;
}
