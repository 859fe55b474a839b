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

#include <cstdlib>

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

// ---- the same transforms on the FP64 tensor cores (DMMA), all parts fused ----
//
// One CTA per block: X = F o W (weights applied while staging, one rounding per
// sample as fase_weigh) stays in shared memory and every separable part runs
// two small NT contractions on mma.sync.m8n8k4.f64:
//   T[v][m] = sum_n cols[v][n] X[m][n],   out[u][v] = sum_m rows[u][m] T[v][m].
// Each warp owns 16 x 16 output macro-tiles (2 x 2 fragments, operands reused
// across the fragment pair); the factor tables are read through L1 (shared by
// every block); shared rows are padded to 4 (mod 16) doubles like the GEMM's.

constexpr int kSepMaxParts = 8;

struct SepPartsArg {
  const double* rows[kSepMaxParts];
  const double* cols[kSepMaxParts];
  int lr[kSepMaxParts];
  int lc[kSepMaxParts];
  int64_t col0[kSepMaxParts];
  int n;
  int stage;  // small batches: factor tables staged in shared memory (fits)
};

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// acc[i][j] (8x8 fragment (i, j) of the macro-tile at rows r0, cols c0) of
// C[r][c] = sum_k A(r, k) B(c, k), k < kk (a multiple of 4); A / B fetched by
// the given functors (zero outside their extents).
template <class FA, class FB>
__device__ __forceinline__ void macro_nt(FA fa, FB fb, int r0, int c0, int kk, double (&acc)[2][2][2]) {
  const int lane = threadIdx.x & 31, fr = lane >> 2, fc = lane & 3;
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  // operands of step k + 4 are fetched while step k's four MMAs run
  double a0 = fa(r0 + fr, fc), a1 = fa(r0 + 8 + fr, fc);
  double b0 = fb(c0 + fr, fc), b1 = fb(c0 + 8 + fr, fc);
#pragma unroll 4
  for (int k = 0; k < kk; k += 4) {
    const bool more = k + 4 < kk;
    const double na0 = more ? fa(r0 + fr, k + 4 + fc) : 0.0;
    const double na1 = more ? fa(r0 + 8 + fr, k + 4 + fc) : 0.0;
    const double nb0 = more ? fb(c0 + fr, k + 4 + fc) : 0.0;
    const double nb1 = more ? fb(c0 + 8 + fr, k + 4 + fc) : 0.0;
    dmma884(acc[0][0][0], acc[0][0][1], a0, b0);
    dmma884(acc[0][1][0], acc[0][1][1], a0, b1);
    dmma884(acc[1][0][0], acc[1][0][1], a1, b0);
    dmma884(acc[1][1][0], acc[1][1][1], a1, b1);
    a0 = na0;
    a1 = na1;
    b0 = nb0;
    b1 = nb1;
  }
}

// MINB 4 for batches that fill the GPU: four CTAs per SM (56 registers, no
// spills; three at 70 registers), config-1 products 0.080 -> 0.074 ms. Small
// batches keep the unconstrained allocation (latency: config 0 0.021 ms
// against 0.031 ms at 56 registers), and (kStage) copy their part's factor
// tables into shared memory with async copies issued alongside the area's
// loads: one round of memory latency, where the operand stream's one-step
// prefetch waited on a cold line every few k-steps.
template <int MINB>
__global__ void __launch_bounds__(288, MINB) sep_products_dmma_kernel(
    const SepPartsArg parts, int Mr, int Nc, const double* __restrict__ F, int64_t ldf,
    const double* __restrict__ W, int64_t ldw, double* __restrict__ R0, int64_t ldr) {
  extern __shared__ __align__(16) double sm[];
  constexpr bool kStage = MINB == 1;
  // small batches: release a programmatic dependent (the latency recursion)
  // now, so it is scheduled while these products run (it waits for them)
  if constexpr (MINB == 1) asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  const int b = blockIdx.x;
  const int warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int lane = threadIdx.x & 31, fr = lane >> 2, fc = lane & 3;
  const int Mp = (Mr + 15) & ~15, Nk = (Nc + 3) & ~3, Mk = (Mr + 3) & ~3;
  const int sx = Nk + ((4 - Nk) & 15), st = Mk + ((4 - Mk) & 15);  // strides = 4 (mod 16)
  double* sX = sm;                   // Mp x sx: X[m][n], zero padded
  double* sT = sm + Mp * sx;         // Lcp x st: T[v][m]
  int lcp_max = 16;
  for (int p = 0; p < parts.n; ++p) lcp_max = max(lcp_max, (parts.lc[p] + 15) & ~15);
  double* sC = sT + lcp_max * st;    // kStage: cols of this CTA's part, Lcp x sx
  double* sR = sC + lcp_max * sx;    // kStage: its slice of rows, 16*per x st
  const double* f = F + static_cast<int64_t>(b) * ldf;
  const double* w = W ? W + static_cast<int64_t>(b) * ldw : nullptr;
  // small batches split the work over gridDim.y CTAs per block: part p =
  // y / splits, and a slice of 16-row groups of u for product 2 (T is formed by
  // every slice of the part)
  const int splits = gridDim.y > 1 ? static_cast<int>(gridDim.y) / parts.n : 1;
  const int p_first = gridDim.y > 1 ? static_cast<int>(blockIdx.y) / splits : 0;
  const int p_last = gridDim.y > 1 ? p_first + 1 : parts.n;
  const int slice = gridDim.y > 1 ? static_cast<int>(blockIdx.y) % splits : 0;
  // kStage (one part per CTA): the part's cols and the rows of its u slice,
  // zero padded, as async copies in flight with the area's loads below
  const bool stage = kStage && parts.stage && p_last == p_first + 1;
  int u_lo = 0;
  if (stage) {
    const int p = p_first, Lr = parts.lr[p], Lc = parts.lc[p];
    const int tm_all = ((Lr + 15) & ~15) / 16, per = (tm_all + splits - 1) / splits;
    u_lo = slice * per * 16;
    const int u_n = max(0, min(tm_all * 16, u_lo + per * 16) - u_lo);
    const double* cols = parts.cols[p];
    const double* rows = parts.rows[p];
    const int nc = ((Lc + 15) & ~15) * sx, nr = u_n * st;
    for (int i = threadIdx.x; i < nc; i += blockDim.x) {
      const int v = i / sx, n = i - v * sx;
      const bool in = v < Lc && n < Nc;
      cp_async8(sC + i, in ? cols + v * Nc + n : cols, in ? 8 : 0);
    }
    for (int i = threadIdx.x; i < nr; i += blockDim.x) {
      const int uu = i / st, m = i - uu * st, u = u_lo + uu;
      const bool in = u < Lr && m < Mr;
      cp_async8(sR + i, in ? rows + u * Mr + m : rows, in ? 8 : 0);
    }
    cp_async_commit();
  }
  // zero the padding, then stage the area with independent loads in flight
  for (int i = threadIdx.x; i < Mp * sx; i += blockDim.x) {
    const int m = i / sx, n = i - m * sx;
    if (m >= Mr || n >= Nc) sX[i] = 0.0;
  }
  const int area = Mr * Nc;
  for (int i0 = 0; i0 < area; i0 += 4 * static_cast<int>(blockDim.x)) {
    double v[4], wv[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int i = i0 + j * blockDim.x + threadIdx.x;
      v[j] = i < area ? __ldg(f + i) : 0.0;
      wv[j] = (w && i < area) ? __ldg(w + i) : 1.0;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int i = i0 + j * blockDim.x + threadIdx.x;
      if (i < area) {
        const int m = i / Nc;
        sX[m * sx + (i - m * Nc)] = w ? __dmul_rn(v[j], wv[j]) : v[j];
      }
    }
  }
  if (stage) cp_async_wait<0>();
  for (int p = p_first; p < p_last; ++p) {
    const double* rows = parts.rows[p];
    const double* cols = parts.cols[p];
    const int Lr = parts.lr[p], Lc = parts.lc[p];
    const int Lcp = (Lc + 15) & ~15, Lrp = (Lr + 15) & ~15;
    __syncthreads();  // sX staged / previous part's sT consumed
    // T[v][m] = sum_n cols[v][n] X[m][n]
    {
      auto fa = [&](int v, int n) {
        if (stage) return sC[v * sx + n];
        return (v < Lc && n < Nc) ? __ldg(cols + v * Nc + n) : 0.0;
      };
      auto fb = [&](int m, int n) { return sX[m * sx + n]; };
      const int tm = Lcp / 16, tn = Mp / 16;
      for (int t = warp; t < tm * tn; t += nwarps) {
        const int r0 = (t / tn) * 16, c0 = (t % tn) * 16;
        double acc[2][2][2];
        macro_nt(fa, fb, r0, c0, Nk, acc);
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int v = r0 + 8 * i + fr, m = c0 + 8 * j + 2 * fc + e;
              if (m < st) sT[v * st + m] = (m < Mr) ? acc[i][j][e] : 0.0;
            }
      }
    }
    __syncthreads();
    // out[u][v] = sum_m rows[u][m] T[v][m]  ->  R0[b, col0 + u*Lc + v]
    {
      auto fa = [&](int u, int m) {
        if (stage) return sR[(u - u_lo) * st + m];
        return (u < Lr && m < Mr) ? __ldg(rows + u * Mr + m) : 0.0;
      };
      auto fb = [&](int v, int m) { return sT[v * st + m]; };
      const int tm_all = Lrp / 16, tn = Lcp / 16;
      const int per = (tm_all + splits - 1) / splits;  // 16-row groups of u per slice
      const int tm_lo = slice * per, tm = max(0, min(tm_all, tm_lo + per) - tm_lo);
      double* out = R0 + static_cast<int64_t>(b) * ldr + parts.col0[p];
      for (int t = warp; t < tm * tn; t += nwarps) {
        const int r0 = (tm_lo + t / tn) * 16, c0 = (t % tn) * 16;
        double acc[2][2][2];
        macro_nt(fa, fb, r0, c0, Mk, acc);
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int u = r0 + 8 * i + fr, v = c0 + 8 * j + 2 * fc + e;
              if (u < Lr && v < Lc) out[u * Lc + v] = acc[i][j][e];
            }
      }
    }
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

extern "C" int fase_sep_products_batch(const fase_sep_part* parts, int n_parts, int Mr, int Nc,
                                       const double* F, int64_t ldf, const double* W, int64_t ldw,
                                       int B, double* R0, int64_t ldr, void* stream) {
  if (n_parts < 1 || n_parts > kSepMaxParts || Mr < 1 || Nc < 1 || B < 0 ||
      ldf < static_cast<int64_t>(Mr) * Nc || (W && ldw != 0 && ldw < static_cast<int64_t>(Mr) * Nc)) {
    set_error("fase_sep_products_batch: bad sizes (parts=%d Mr=%d Nc=%d B=%d)", n_parts, Mr, Nc, B);
    return FASE_ERR_SHAPE;
  }
  if (B == 0) return FASE_OK;
  if (!parts || !F || !R0) {
    set_error("fase_sep_products_batch: null pointer");
    return FASE_ERR_SHAPE;
  }
  SepPartsArg a{};
  a.n = n_parts;
  int lcp_max = 16;
  for (int p = 0; p < n_parts; ++p) {
    const fase_sep_part& q = parts[p];
    if (!q.rows || !q.cols || q.Lr < 1 || q.Lc < 1 || q.col0 < 0 ||
        ldr < q.col0 + static_cast<int64_t>(q.Lr) * q.Lc) {
      set_error("fase_sep_products_batch: part %d: bad factors / output range", p);
      return FASE_ERR_SHAPE;
    }
    a.rows[p] = q.rows;
    a.cols[p] = q.cols;
    a.lr[p] = q.Lr;
    a.lc[p] = q.Lc;
    a.col0[p] = q.col0;
    lcp_max = (q.Lc + 15) / 16 * 16 > lcp_max ? (q.Lc + 15) / 16 * 16 : lcp_max;
  }
  const int Mp = (Mr + 15) / 16 * 16, Nk = (Nc + 3) / 4 * 4, Mk = (Mr + 3) / 4 * 4;
  const int sx = Nk + ((4 - Nk) & 15), st = Mk + ((4 - Mk) & 15);
  size_t smem = sizeof(double) * (static_cast<size_t>(Mp) * sx + static_cast<size_t>(lcp_max) * st);
  if (smem > 200 * 1024) {
    set_error("fase_sep_products_batch: area %dx%d too large for shared memory", Mr, Nc);
    return FASE_ERR_UNSUPPORTED;
  }
  auto kernel = B < 148 ? sep_products_dmma_kernel<1> : sep_products_dmma_kernel<4>;
  // batches smaller than the GPU: one CTA per (block, part, slice of u)
  int splits = 1;
  if (B < 148) {
    const int lr_min_groups = (parts[0].Lr + 15) / 16;
    splits = lr_min_groups < 4 ? lr_min_groups : 4;
    if (splits < 1) splits = 1;
    // staged factor tables: cols Lcp x sx, the rows of a u slice 16*per x st
    int per_max = 1;
    for (int p = 0; p < n_parts; ++p) {
      const int tm_all = (parts[p].Lr + 15) / 16, per = (tm_all + splits - 1) / splits;
      per_max = per > per_max ? per : per_max;
    }
    const size_t staged = smem + sizeof(double) * (static_cast<size_t>(lcp_max) * sx +
                                                   static_cast<size_t>(16 * per_max) * st);
    if (staged <= 200 * 1024) {  // else the factors stream from global memory
      smem = staged;
      a.stage = 1;
    }
  }
  cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) {
    set_error("fase_sep_products_batch: cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    return FASE_ERR_CUDA;
  }
  const dim3 grid(B, B < 148 ? n_parts * splits : 1);
  kernel<<<grid, 288, smem, as_stream(stream)>>>(a, Mr, Nc, F, ldf, W, ldw, R0, ldr);
  return check_launch("fase_sep_products_batch");
}
