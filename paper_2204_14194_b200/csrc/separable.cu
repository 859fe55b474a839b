// Initial products for separable dictionaries, as two small transforms.
//
// For atoms phi[u*Lc + v](m, n) = rows[u, m] * cols[v, n] (DCT, WHT, Hadamard
// families: dictionary.py:167-178) the initial products of a weighted area X
// (R0_k = sum_{m,n} X[m,n] phi_k[m,n], fast.py:145-157) factor as
//
//   R0[u*Lc + v] = sum_m rows[u, m] * ( sum_n X[m, n] * cols[v, n] )  =  (rows X cols^T)[u, v]
//
// so one block costs 2 * (Lr*Mr*Nc + Lr*Nc*Lc) flops instead of the
// 2 * Lr*Lc*Mr*Nc of the dense contraction (24x fewer at 48 x 48). The same
// identity underlies the reference's FFT shortcut for DFT atoms
// (transform.py:43-69); here it covers the real separable families. Summation
// order differs from the dense GEMM, so results agree to rounding (the parity
// tests hold them to the same tolerance as the GEMM path).
//

#include "common.cuh"

namespace fase {
namespace {

constexpr int kSepThreads = 256;  // a 16 x 16 thread grid

// C[i][j] = sum_l A[i*lda + l] * B[j*ldb + l] for i < ni, j < nj (shared memory
// operands), each thread owning a kMaxTile x kMaxTile register tile of rows
// ty + 16*a and columns tx + 16*c, so every loaded value feeds kMaxTile FMAs.
template <int kMaxTile>
__device__ __forceinline__ void smem_nt(const double* A, int lda, const double* B, int ldb, int ni,
                                        int nj, int nl, double* C, int ldc, int64_t cstride_i = -1) {
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  for (int i0 = 0; i0 < ni; i0 += 16 * kMaxTile) {
    for (int j0 = 0; j0 < nj; j0 += 16 * kMaxTile) {
      double acc[kMaxTile][kMaxTile];
#pragma unroll
      for (int a = 0; a < kMaxTile; ++a)
#pragma unroll
        for (int c = 0; c < kMaxTile; ++c) acc[a][c] = 0.0;
      for (int l = 0; l < nl; ++l) {
        double av[kMaxTile], bv[kMaxTile];
#pragma unroll
        for (int a = 0; a < kMaxTile; ++a) {
          const int i = i0 + ty + 16 * a;
          av[a] = i < ni ? A[i * lda + l] : 0.0;
        }
#pragma unroll
        for (int c = 0; c < kMaxTile; ++c) {
          const int j = j0 + tx + 16 * c;
          bv[c] = j < nj ? B[j * ldb + l] : 0.0;
        }
#pragma unroll
        for (int a = 0; a < kMaxTile; ++a)
#pragma unroll
          for (int c = 0; c < kMaxTile; ++c) acc[a][c] = fma(av[a], bv[c], acc[a][c]);
      }
#pragma unroll
      for (int a = 0; a < kMaxTile; ++a) {
        const int i = i0 + ty + 16 * a;
#pragma unroll
        for (int c = 0; c < kMaxTile; ++c) {
          const int j = j0 + tx + 16 * c;
          if (i < ni && j < nj) {
            if (cstride_i < 0)
              C[i * ldc + j] = acc[a][c];
            else
              C[static_cast<int64_t>(i) * cstride_i + j] = acc[a][c];
          }
        }
      }
    }
  }
}

// One CTA per (block, slice of `rpc` output rows u).
//   step 1: T^T[v][m] = sum_n cols[v][n] X[m][n]      (Lc x Mr)
//   step 2: out[u][v] = sum_m rows[u][m] T^T[v][m]     (rpc x Lc)
// T is formed by every slice (rpc = Lr when the batch alone fills the GPU, so
// once per block; small batches split rows for parallelism). Shared pitches
// are odd so a warp's strided reads spread over the banks.
template <int kTile>
__global__ void __launch_bounds__(kSepThreads) sep_products_kernel(
    const double* __restrict__ rows, int Lr, int Mr, const double* __restrict__ cols, int Lc,
    int Nc, const double* __restrict__ X, int64_t ldx, double* __restrict__ R0, int64_t ldr,
    int64_t col0, int rpc) {
  extern __shared__ __align__(16) double sm[];
  const int pn = Nc | 1, pm = Mr | 1;
  double* sX = sm;              // Mr x pn
  double* sC = sX + Mr * pn;    // Lc x pn
  double* sT = sC + Lc * pn;    // Lc x pm   (T transposed)
  double* sR = sT + Lc * pm;    // rpc x pm
  const int b = blockIdx.x;
  const int u0 = blockIdx.y * rpc;
  const int nu = min(rpc, Lr - u0);
  const double* xb = X + static_cast<int64_t>(b) * ldx;
  for (int i = threadIdx.x; i < Mr * Nc; i += kSepThreads) sX[(i / Nc) * pn + i % Nc] = xb[i];
  for (int i = threadIdx.x; i < Lc * Nc; i += kSepThreads) sC[(i / Nc) * pn + i % Nc] = cols[i];
  for (int i = threadIdx.x; i < nu * Mr; i += kSepThreads)
    sR[(i / Mr) * pm + i % Mr] = rows[static_cast<int64_t>(u0) * Mr + i];
  __syncthreads();
  smem_nt<kTile>(sC, pn, sX, pn, Lc, Mr, Nc, sT, pm);
  __syncthreads();
  smem_nt<kTile>(sR, pm, sT, pm, nu, Lc, Mr,
          R0 + static_cast<int64_t>(b) * ldr + col0 + static_cast<int64_t>(u0) * Lc, 0, Lc);
}

}  // namespace
}  // namespace fase

using namespace fase;

extern "C" int fase_sep_products(const double* rows, int Lr, int Mr, const double* cols, int Lc,
                                 int Nc, const double* X, int64_t ldx, int B, double* R0,
                                 int64_t ldr, int64_t col0, void* stream) {
  if (Lr < 1 || Mr < 1 || Lc < 1 || Nc < 1 || B < 0 || ldx < static_cast<int64_t>(Mr) * Nc ||
      col0 < 0 || ldr < col0 + static_cast<int64_t>(Lr) * Lc) {
    set_error("fase_sep_products: bad sizes (Lr=%d Mr=%d Lc=%d Nc=%d B=%d)", Lr, Mr, Lc, Nc, B);
    return FASE_ERR_SHAPE;
  }
  if (B == 0) return FASE_OK;
  if (!rows || !cols || !X || !R0) {
    set_error("fase_sep_products: null pointer");
    return FASE_ERR_SHAPE;
  }
  const int rpc = B >= 148 ? Lr : (Lr < 8 ? Lr : 8);
  const size_t smem =
      sizeof(double) * (static_cast<size_t>(Mr + Lc) * (Nc | 1) +
                        static_cast<size_t>(Lc + rpc) * (Mr | 1));
  if (smem > 200 * 1024) {
    set_error("fase_sep_products: factor tables too large for shared memory (%zu bytes)", smem);
    return FASE_ERR_UNSUPPORTED;
  }
  // register tile: 16 x 16 threads cover the larger of the two product shapes
  const int span = (Lr > Lc ? (Lr > Mr ? Lr : Mr) : (Lc > Mr ? Lc : Mr));
  const int tile = span <= 32 ? 2 : (span <= 48 ? 3 : 4);
  auto kern = tile == 2 ? sep_products_kernel<2> : (tile == 3 ? sep_products_kernel<3>
                                                              : sep_products_kernel<4>);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) {
    set_error("fase_sep_products: cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    return FASE_ERR_CUDA;
  }
  dim3 grid(B, (Lr + rpc - 1) / rpc);
  kern<<<grid, kSepThreads, smem, as_stream(stream)>>>(rows, Lr, Mr, cols, Lc, Nc, X, ldx, R0, ldr,
                                                        col0, rpc);
  return check_launch("fase_sep_products");
}
