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
// store(i, j, value) writes one result.
template <int kMaxTile, class Store>
__device__ __forceinline__ void smem_nt_f(const double* A, int lda, const double* B, int ldb, int ni,
                                          int nj, int nl, Store store) {
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
          if (i < ni && j < nj) store(i, j, acc[a][c]);
        }
      }
    }
  }
}

template <int kMaxTile>
__device__ __forceinline__ void smem_nt(const double* A, int lda, const double* B, int ldb, int ni,
                                        int nj, int nl, double* C, int ldc, int64_t cstride_i = -1) {
  smem_nt_f<kMaxTile>(A, lda, B, ldb, ni, nj, nl, [&](int i, int j, double v) {
    if (cstride_i < 0)
      C[i * ldc + j] = v;
    else
      C[static_cast<int64_t>(i) * cstride_i + j] = v;
  });
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

// Complex separable parts (DFT exponentials, dictionary.py:126-131, or real
// parts of a complex union): atoms phi[u*Lc + v](m, n) = E[u, m] * F[v, n] with
// E = Cm + i Sm, F = Cn + i Sn, and a real weighted area X:
//   R0[u*Lc + v] = sum_{m,n} conj(E[u,m]) conj(F[v,n]) X[m,n] = (conj(E) X conj(F)^T)[u, v]
// -- fft2(X) at (u, v) for the full exponential grid, the reference's
// fft_initial_products identity (transform.py:43-69). As real contractions:
//   step 1: [T1; T2] = [Cn; Sn] X^T                       (2 Lc x Mr)
//   step 2: Re = [Cm | -Sm] [T1 | T2]^T, Im = [-Sm | -Cm] [T1 | T2]^T
// (contraction depth 2 Mr), written interleaved into the complex R0. X and the
// column factors are dead after step 1, so the row operand reuses their space.
template <int kTile>
__global__ void __launch_bounds__(kSepThreads) sep_products_complex_kernel(
    const double* __restrict__ rows_re, const double* __restrict__ rows_im, int Lr, int Mr,
    const double* __restrict__ cols_re, const double* __restrict__ cols_im, int Lc, int Nc,
    const double* __restrict__ X, int64_t ldx, double2* __restrict__ R0, int64_t ldr, int64_t col0,
    int rpc) {
  extern __shared__ __align__(16) double sm[];
  const int pn = Nc | 1, p2m = (2 * Mr) | 1;
  double* sB = sm;                 // Lc x p2m: row v = [T1^T[v, :] | T2^T[v, :]]
  double* sX = sB + Lc * p2m;      // Mr x pn        (step 1)
  double* sC = sX + Mr * pn;       // 2Lc x pn: [Cn; Sn]
  double* sA = sX;                 // 2rpc x p2m     (step 2, reuses sX / sC)
  const int b = blockIdx.x;
  const int u0 = blockIdx.y * rpc;
  const int nu = min(rpc, Lr - u0);
  const double* xb = X + static_cast<int64_t>(b) * ldx;
  for (int i = threadIdx.x; i < Mr * Nc; i += kSepThreads) sX[(i / Nc) * pn + i % Nc] = xb[i];
  for (int i = threadIdx.x; i < Lc * Nc; i += kSepThreads) {
    sC[(i / Nc) * pn + i % Nc] = cols_re[i];
    sC[(Lc + i / Nc) * pn + i % Nc] = cols_im[i];
  }
  __syncthreads();
  smem_nt_f<kTile>(sC, pn, sX, pn, 2 * Lc, Mr, Nc, [&](int i, int j, double v) {
    if (i < Lc)
      sB[i * p2m + j] = v;
    else
      sB[(i - Lc) * p2m + Mr + j] = v;
  });
  __syncthreads();
  for (int i = threadIdx.x; i < nu * Mr; i += kSepThreads) {
    const int u = i / Mr, m = i % Mr;
    const int64_t g = static_cast<int64_t>(u0 + u) * Mr + m;
    const double cm = rows_re[g], sn = rows_im[g];
    sA[u * p2m + m] = cm;              // Re row: [Cm | -Sm]
    sA[u * p2m + Mr + m] = -sn;
    sA[(nu + u) * p2m + m] = -sn;      // Im row: [-Sm | -Cm]
    sA[(nu + u) * p2m + Mr + m] = -cm;
  }
  __syncthreads();
  double* out = reinterpret_cast<double*>(R0 + static_cast<int64_t>(b) * ldr + col0 +
                                          static_cast<int64_t>(u0) * Lc);
  smem_nt_f<kTile>(sA, p2m, sB, p2m, 2 * nu, Lc, 2 * Mr, [&](int i, int j, double v) {
    if (i < nu)
      out[2 * (i * Lc + j)] = v;
    else
      out[2 * ((i - nu) * Lc + j) + 1] = v;
  });
}

// Transform-shortcut Gram table (fft_gram_table, transform.py:84-110): with
// What = fft2(w) (spec, M x N complex, e.g. from fase_sep_products_complex),
// S = (What + conj(What[-a, -b])) / 2 is exactly Hermitian-symmetric and
//   C(k, l) = S[(mu_k - mu_l) mod M, (eta_k - eta_l) mod N],
// so the stored row of conj(C) is T[k, l] = S[(mu_l - mu_k) mod M, (eta_l - eta_k) mod N],
// with the diagonal forced real (_finish_tables). S is staged in shared memory;
// each thread writes one 16-byte entry (the build is a pure HBM write stream).
__global__ void __launch_bounds__(256) fft_gram_kernel(const double2* __restrict__ spec, int M,
                                                      int N, const int32_t* __restrict__ mu,
                                                      const int32_t* __restrict__ eta, int K,
                                                      double2* __restrict__ T, int64_t ldt) {
  extern __shared__ __align__(16) double2 s_s[];
  const int MN = M * N;
  for (int i = threadIdx.x; i < MN; i += blockDim.x) {
    const int a = i / N, c = i % N;
    const int j = ((M - a) % M) * N + (N - c) % N;
    const double2 x = spec[i], y = spec[j];
    s_s[i] = make_double2(0.5 * (x.x + y.x), 0.5 * (x.y - y.y));
  }
  __syncthreads();
  const int64_t total = static_cast<int64_t>(K) * ldt;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int k = static_cast<int>(e / ldt);
    const int l = static_cast<int>(e - static_cast<int64_t>(k) * ldt);
    double2 v = make_double2(0.0, 0.0);
    if (l < K) {
      const int mk = mu ? mu[k] : k / N, ek = eta ? eta[k] : k % N;
      const int ml = mu ? mu[l] : l / N, el = eta ? eta[l] : l % N;
      const int a = ((ml - mk) % M + M) % M, c = ((el - ek) % N + N) % N;
      v = s_s[a * N + c];
      if (k == l) v = make_double2(v.x, -0.0);
    }
    T[e] = v;
  }
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

extern "C" int fase_sep_products_complex(const double* rows_re, const double* rows_im, int Lr,
                                         int Mr, const double* cols_re, const double* cols_im,
                                         int Lc, int Nc, const double* X, int64_t ldx, int B,
                                         double* R0, int64_t ldr, int64_t col0, void* stream) {
  if (Lr < 1 || Mr < 1 || Lc < 1 || Nc < 1 || B < 0 || ldx < static_cast<int64_t>(Mr) * Nc ||
      col0 < 0 || ldr < col0 + static_cast<int64_t>(Lr) * Lc) {
    set_error("fase_sep_products_complex: bad sizes (Lr=%d Mr=%d Lc=%d Nc=%d B=%d)", Lr, Mr, Lc,
              Nc, B);
    return FASE_ERR_SHAPE;
  }
  if (B == 0) return FASE_OK;
  if (!rows_re || !rows_im || !cols_re || !cols_im || !X || !R0 || !aligned16(R0)) {
    set_error("fase_sep_products_complex: null or misaligned pointer");
    return FASE_ERR_SHAPE;
  }
  const int p2m = (2 * Mr) | 1, pn = Nc | 1;
  const int rpc = B >= 148 ? Lr : (Lr < 8 ? Lr : 8);
  const size_t step1 = static_cast<size_t>(Mr + 2 * Lc) * pn;
  const size_t step2 = static_cast<size_t>(2 * rpc) * p2m;
  const size_t smem = sizeof(double) * (static_cast<size_t>(Lc) * p2m + (step1 > step2 ? step1 : step2));
  if (smem > 200 * 1024) {
    set_error("fase_sep_products_complex: factor tables too large for shared memory (%zu bytes)",
              smem);
    return FASE_ERR_UNSUPPORTED;
  }
  const int span = 2 * (Lr > Lc ? (Lr > Mr ? Lr : Mr) : (Lc > Mr ? Lc : Mr));
  const int tile = span <= 32 ? 2 : (span <= 48 ? 3 : 4);
  auto kern = tile == 2 ? sep_products_complex_kernel<2>
                        : (tile == 3 ? sep_products_complex_kernel<3> : sep_products_complex_kernel<4>);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) {
    set_error("fase_sep_products_complex: cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    return FASE_ERR_CUDA;
  }
  dim3 grid(B, (Lr + rpc - 1) / rpc);
  kern<<<grid, kSepThreads, smem, as_stream(stream)>>>(rows_re, rows_im, Lr, Mr, cols_re, cols_im,
                                                        Lc, Nc, X, ldx,
                                                        reinterpret_cast<double2*>(R0), ldr, col0,
                                                        rpc);
  return check_launch("fase_sep_products_complex");
}

extern "C" int fase_fft_gram(const double* spec, int M, int N, const int32_t* mu,
                             const int32_t* eta, int K, double* T, int64_t ldt, void* stream) {
  if (M < 1 || N < 1 || K < 1 || ldt < K || (!mu) != (!eta)) {
    set_error("fase_fft_gram: bad sizes or tags (M=%d N=%d K=%d)", M, N, K);
    return FASE_ERR_SHAPE;
  }
  if (!mu && K > M * N) {
    set_error("fase_fft_gram: %d canonical tags exceed the %dx%d frequency grid", K, M, N);
    return FASE_ERR_SHAPE;
  }
  if (!spec || !T || !aligned16(spec) || !aligned16(T)) {
    set_error("fase_fft_gram: null or misaligned pointer");
    return FASE_ERR_SHAPE;
  }
  const size_t smem = sizeof(double2) * static_cast<size_t>(M) * N;
  if (smem > 200 * 1024) {
    set_error("fase_fft_gram: %dx%d spectrum exceeds shared memory", M, N);
    return FASE_ERR_UNSUPPORTED;
  }
  cudaError_t e = cudaFuncSetAttribute(fft_gram_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) {
    set_error("fase_fft_gram: cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    return FASE_ERR_CUDA;
  }
  const int64_t total = static_cast<int64_t>(K) * ldt;
  const int64_t blocks = (total + 255) / 256;
  fft_gram_kernel<<<static_cast<unsigned>(blocks < 148 * 4 ? blocks : 148 * 4), 256, smem,
                    as_stream(stream)>>>(reinterpret_cast<const double2*>(spec), M, N, mu, eta, K,
                                         reinterpret_cast<double2*>(T), ldt);
  return check_launch("fase_fft_gram");
}
