// FP64 tensor-core (DMMA) contractions of the FaSE correlation stage.
//
//   C[i, j] = sum_k A[i, k] * B[j, k]        ("NT": both operands contraction-contiguous)
//
// Used for the weighted Gram table G = (Phi o w) Phi^T (build_gram_tables,
// reference fast.py:109-142) and the batched initial products
// R0 = (F o W) Phi^T (initial_scalar_products, fast.py:145-157, one zgemv per
// block in the reference). The weighted operand is formed first by a streaming
// kernel (one correctly rounded multiply per sample, the rounding structure of
// the reference's `conj(phi)*w` / `s*w` before its BLAS call); folding the
// multiply into the GEMM's shared-memory stage was measured 23% slower
// (0.88 vs 0.72 ms on the config-1 shape) because it adds a barrier and a
// shared-memory round trip per k-tile.
//
// Why DMMA and not tcgen05: tcgen05.mma has no f64 kind on sm_100a
// (SURVEY.md section 0, item 7); FP64 on Blackwell's tensor cores is the
// warp-level `mma.sync ... .f64` path, which ptxas lowers to DMMA.8x8x4.
// Measured DMMA issue peak on the B200: 37 TFLOP/s (tools/probes/dmma_probe.cu).
//
// Tiling: BK = 16, 3-stage cp.async ring; main tile 64 x 128 with 4 warps of
// 32 x 64 (4 x 8 DMMA 8x8 accumulators, 64 FP64 registers) and two CTAs per
// SM, so one CTA's k-tile barrier is covered by the other; a 128 x 128 /
// 8-warp tile is kept as fase_gemm_nt variant 1 for comparison. Shared rows are
// padded to 20 doubles: the 8x4 fragment a half-warp reads then hits 16
// distinct 8-byte bank pairs.
// Symmetric mode (Gram) computes tiles with bm <= bn only and writes each
// accumulator to (i, j) and (j, i): the table is bit-symmetric.

#include "common.cuh"

namespace fase {
namespace {

constexpr int BK = 16;
constexpr int LDS = BK + 4;
constexpr int STAGES = 3;

struct GemmParams {
  const double* A;
  int64_t lda;
  const double* B;
  int64_t ldb;
  double* C;
  int64_t ldc;
  int m_rows;
  int n_rows;
  int kdim;
};

__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// BM x BN CTA tile, warps of WM x WN (a grid of BM/WM x BN/WN warps),
// MINB resident CTAs per SM.
template <int BM, int BN, int WM, int WN, int MINB>
struct Tile {
  static constexpr int kBM = BM, kBN = BN, kWM = WM, kWN = WN;
  static constexpr int kWarpsM = BM / WM, kWarpsN = BN / WN;
  static constexpr int kThreads = 32 * kWarpsM * kWarpsN;
  static constexpr int kMinBlocks = MINB;
  static constexpr size_t kSmem = sizeof(double) * STAGES * LDS * (BM + BN);
};
using TileBig = Tile<128, 128, 64, 32, 1>;   // 8 warps, 1 CTA / SM
using TileSmall = Tile<64, 128, 32, 64, 2>;  // 4 warps, 2 CTAs / SM

template <class T, bool kSym>
__global__ void __launch_bounds__(T::kThreads, T::kMinBlocks) dgemm_nt_kernel(const GemmParams p) {
  constexpr int BM = T::kBM, BN = T::kBN, NTH = T::kThreads;
  constexpr int MI = T::kWM / 8, NI = T::kWN / 8;
  extern __shared__ __align__(16) double smem[];
  double* As = smem;
  double* Bs = As + STAGES * BM * LDS;

  const int bm = blockIdx.y;
  const int bn = blockIdx.x;
  if (kSym && bm * BM >= (bn + 1) * BN) return;  // entirely below the diagonal
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int wm = warp / T::kWarpsN;
  const int wn = warp % T::kWarpsN;
  const int row0 = bm * BM;
  const int col0 = bn * BN;
  const int ktiles = (p.kdim + BK - 1) / BK;

  auto load_rows = [&](double* dst, const double* src, int64_t ld, int rows_total, int row_base,
                       int nrows, int k0) {
    constexpr int kChunksPerRow = BK / 2;
#pragma unroll
    for (int i = 0; i < (nrows * kChunksPerRow + NTH - 1) / NTH; ++i) {
      const int idx = tid + i * NTH;
      if (idx < nrows * kChunksPerRow) {
        const int r = idx / kChunksPerRow;
        const int kc = (idx % kChunksPerRow) * 2;
        const int k = k0 + kc;
        int kb = (p.kdim - k) * 8;
        kb = kb < 0 ? 0 : (kb > 16 ? 16 : kb);
        const int gr = row_base + r;
        const int nb = gr < rows_total ? kb : 0;
        const double* g = nb ? src + static_cast<int64_t>(gr) * ld + k : src;
        cp_async16(dst + r * LDS + kc, g, nb);
      }
    }
  };
  auto load_stage = [&](int stage, int kt) {
    load_rows(As + stage * BM * LDS, p.A, p.lda, p.m_rows, row0, BM, kt * BK);
    load_rows(Bs + stage * BN * LDS, p.B, p.ldb, p.n_rows, col0, BN, kt * BK);
  };

  double acc[MI][NI][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < ktiles) load_stage(s, s);
    cp_async_commit();
  }

  const int fr = lane >> 2;
  const int fc = lane & 3;
  for (int kt = 0; kt < ktiles; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    const int st = kt % STAGES;
    const int nk = kt + STAGES - 1;
    if (nk < ktiles) load_stage(nk % STAGES, nk);
    cp_async_commit();

    const double* as = As + st * BM * LDS + (wm * T::kWM + fr) * LDS + fc;
    const double* bs = Bs + st * BN * LDS + (wn * T::kWN + fr) * LDS + fc;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double a[MI], b[NI];
#pragma unroll
      for (int i = 0; i < MI; ++i) a[i] = as[i * 8 * LDS + kk];
#pragma unroll
      for (int j = 0; j < NI; ++j) b[j] = bs[j * 8 * LDS + kk];
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
  }
  cp_async_wait<0>();

  const bool vec_ok = ((p.ldc & 1) == 0) && aligned16(p.C);
#pragma unroll
  for (int i = 0; i < MI; ++i) {
    const int r = row0 + wm * T::kWM + i * 8 + fr;
#pragma unroll
    for (int j = 0; j < NI; ++j) {
      const int c = col0 + wn * T::kWN + j * 8 + fc * 2;
      if (!kSym) {
        if (r < p.m_rows) {
          double* dst = p.C + static_cast<int64_t>(r) * p.ldc + c;
          if (vec_ok && c + 1 < p.n_rows) {
            *reinterpret_cast<double2*>(dst) = make_double2(acc[i][j][0], acc[i][j][1]);
          } else {
            if (c < p.n_rows) dst[0] = acc[i][j][0];
            if (c + 1 < p.n_rows) dst[1] = acc[i][j][1];
          }
        }
      } else {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int cc = c + e;
          if (r < p.m_rows && cc < p.n_rows && r <= cc) {
            p.C[static_cast<int64_t>(r) * p.ldc + cc] = acc[i][j][e];
            p.C[static_cast<int64_t>(cc) * p.ldc + r] = acc[i][j][e];
          }
        }
      }
    }
  }
}

// Small batches (B <= kGemvMax, e.g. config 0's single block): one warp per
// atom row streams phi[k, :] once and dots it with every block's weighted
// signal (L2/L1-resident), instead of a GEMM tile that would be almost empty.
constexpr int kGemvMax = 8;

__global__ void gemv_rows_kernel(const double* __restrict__ X, int64_t ldx, int B,
                                 const double* __restrict__ phi, int64_t ldphi, int K, int M,
                                 double* __restrict__ R0, int64_t ldr) {
  const int lane = threadIdx.x & 31;
  const int warps = blockDim.x >> 5;
  for (int k = blockIdx.x * warps + (threadIdx.x >> 5); k < K; k += gridDim.x * warps) {
    double acc[kGemvMax];
#pragma unroll
    for (int b = 0; b < kGemvMax; ++b) acc[b] = 0.0;
    const double* row = phi + static_cast<int64_t>(k) * ldphi;
    for (int m = 2 * lane; m < M; m += 64) {
      const double2 pv = ldg2(row + m);  // even leading dimensions: the pair exists
      const bool pair = m + 1 < M;       // the odd tail's partner is never used
#pragma unroll
      for (int b = 0; b < kGemvMax; ++b) {
        if (b < B) {
          const double2 xv = ldg2(X + b * ldx + m);
          acc[b] = fma(pv.x, xv.x, acc[b]);
          if (pair) acc[b] = fma(pv.y, xv.y, acc[b]);
        }
      }
    }
#pragma unroll
    for (int b = 0; b < kGemvMax; ++b) {
      double v = acc[b];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0 && b < B) R0[b * ldr + k] = v;
    }
  }
}

// out[b*ldo + m] = x[b*ldx + m] * w[b*ldw + m]  (ldw == 0: one shared weight row);
// one correctly rounded multiply per sample, 16-byte accesses.
__global__ void weigh_kernel(const double* __restrict__ x, int64_t ldx, const double* __restrict__ w,
                             int64_t ldw, int rows, int M, double* __restrict__ out, int64_t ldo) {
  const int pairs = (M + 1) / 2;
  const int64_t total = static_cast<int64_t>(rows) * pairs;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int b = static_cast<int>(i / pairs);
    const int m = 2 * static_cast<int>(i - static_cast<int64_t>(b) * pairs);
    const double2 xv = *reinterpret_cast<const double2*>(x + b * ldx + m);
    const double2 wv = *reinterpret_cast<const double2*>(w + b * ldw + m);
    double2 o;
    o.x = mul_rn(xv.x, wv.x);
    o.y = m + 1 < M ? mul_rn(xv.y, wv.y) : 0.0;
    *reinterpret_cast<double2*>(out + b * ldo + m) = o;
  }
}

// out[b*ldo + i] = x[b*ldx + idx[i]] * w[i] for i < n (zero pad to even n): the
// weighted operand restricted to the samples with nonzero weight (lost samples
// contribute exact zeros to every product, so the contraction skips them).
__global__ void weigh_gather_kernel(const double* __restrict__ x, int64_t ldx,
                                    const int32_t* __restrict__ idx, const double* __restrict__ w,
                                    int rows, int n, double* __restrict__ out, int64_t ldo) {
  const int np = (n + 1) / 2 * 2;
  const int64_t total = static_cast<int64_t>(rows) * np;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int b = static_cast<int>(e / np);
    const int i = static_cast<int>(e - static_cast<int64_t>(b) * np);
    out[b * ldo + i] = i < n ? mul_rn(__ldg(x + b * ldx + __ldg(idx + i)), __ldg(w + i)) : 0.0;
  }
}

template <class T, bool kSym>
int launch(const GemmParams& p, cudaStream_t stream, const char* what) {
  // per-device attributes; cheap enough to set on every launch
  cudaError_t e = cudaFuncSetAttribute(dgemm_nt_kernel<T, kSym>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(T::kSmem));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(dgemm_nt_kernel<T, kSym>,
                             cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (e != cudaSuccess) {
    set_error("%s: cudaFuncSetAttribute: %s", what, cudaGetErrorString(e));
    return FASE_ERR_CUDA;
  }
  dim3 grid((p.n_rows + T::kBN - 1) / T::kBN, (p.m_rows + T::kBM - 1) / T::kBM);
  dgemm_nt_kernel<T, kSym><<<grid, T::kThreads, T::kSmem, stream>>>(p);
  return check_launch(what);
}

// The tile used by the library entry points (see tools/probes/gemm_probe.py).
using TileMain = TileSmall;

int launch_weigh(const double* x, int64_t ldx, const double* w, int64_t ldw, int rows, int M,
                 double* out, int64_t ldo, cudaStream_t stream, const char* what) {
  const int64_t total = static_cast<int64_t>(rows) * ((M + 1) / 2);
  const int threads = 256;
  const int64_t blocks = (total + threads - 1) / threads;
  weigh_kernel<<<static_cast<unsigned>(blocks < 148 * 16 ? blocks : 148 * 16), threads, 0,
                 stream>>>(x, ldx, w, ldw, rows, M, out, ldo);
  return check_launch(what);
}

bool operand_ok(const double* ptr, int64_t ld) { return ptr && aligned16(ptr) && (ld % 2 == 0); }

// ---- complex tables ---------------------------------------------------------
//
// A complex dictionary lives on the device in the conjugate-split layout:
// row 2k = Re phi_k, row 2k+1 = -Im phi_k (each ldphi doubles). Read as K rows
// of 2*ldphi doubles, row k is P_k = [A_k | -B_k] (phi = A + iB), so with
// w2 = [w | w] the Gram table C = conj(Phi) W Phi^T (fast.py:129-131) is
//   Re C = (P o w2) P^T,   Im C = (P o w2) Q^T,   Q_l = [B_l | A_l],
// two real DMMA contractions of depth 2*ldphi. Both run in symmetric mode
// (tiles bm <= bn only); the pack kernel reads the upper triangle and emits
// the table row by row as conj(C[u, :]) -- the operand of the recursion's
// update (fast.py:246) -- mirroring the strict lower triangle exactly like
// the reference's Hermitian fill (fast.py:132-137) and forcing a real
// diagonal (_finish_tables, fast.py:97-100).

// w2[i] = w[i mod ldphi] for i mod ldphi < M, else 0
__global__ void dup_weight_kernel(const double* __restrict__ w, int M, int64_t ldphi,
                                  double* __restrict__ w2) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < 2 * ldphi;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t m = i < ldphi ? i : i - ldphi;
    w2[i] = m < M ? w[m] : 0.0;
  }
}

// Q_k = [-(P_k second half) | P_k first half] = [B_k | A_k]
__global__ void swap_halves_kernel(const double* __restrict__ P, int K, int64_t ldphi,
                                   double* __restrict__ Q) {
  const int64_t total = static_cast<int64_t>(K) * 2 * ldphi;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t k = i / (2 * ldphi);
    const int64_t c = i - k * 2 * ldphi;
    const double* row = P + k * 2 * ldphi;
    Q[i] = c < ldphi ? -row[ldphi + c] : row[c - ldphi];
  }
}

// T[u, l] = conj(C[u, l]) for l < ldt (zero past K): u < l (Re[u,l], -Im[u,l]);
// u > l (Re[l,u], Im[l,u]); u == l (Re[u,u], -0.0). 32 x 32 tiles, the
// transposed Im tile staged through shared memory.
__global__ void hermitian_pack_kernel(const double* __restrict__ re, const double* __restrict__ im,
                                      int64_t ldk, int K, double2* __restrict__ T, int64_t ldt) {
  __shared__ double s_im_t[32][33];
  const int u0 = blockIdx.y * 32, l0 = blockIdx.x * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  // Im[l0 + i, u0 + tx] for the tile's lower part (u > l): transposed read
  for (int i = ty; i < 32; i += 8) {
    const int l = l0 + i, u = u0 + tx;
    s_im_t[i][tx] = (l < K && u < K && l < u) ? im[static_cast<int64_t>(l) * ldk + u] : 0.0;
  }
  __syncthreads();
  for (int i = ty; i < 32; i += 8) {
    const int u = u0 + i, l = l0 + tx;
    if (u >= K || l >= ldt) continue;
    double2 v;
    if (l >= K) {
      v = make_double2(0.0, 0.0);
    } else if (u < l) {
      v = make_double2(re[static_cast<int64_t>(u) * ldk + l], -im[static_cast<int64_t>(u) * ldk + l]);
    } else if (u > l) {
      v = make_double2(re[static_cast<int64_t>(u) * ldk + l], s_im_t[tx][i]);  // Re bit-symmetric
    } else {
      v = make_double2(re[static_cast<int64_t>(u) * ldk + u], -0.0);
    }
    T[static_cast<int64_t>(u) * ldt + l] = v;
  }
}

size_t complex_gram_parts(int K, int64_t ldphi, size_t* off) {
  const size_t row = 2 * static_cast<size_t>(ldphi);
  const size_t ldk = (static_cast<size_t>(K) + 1) / 2 * 2;
  size_t o = 0;
  off[0] = o; o += row;                                 // w2
  off[1] = o; o += static_cast<size_t>(K) * row;        // P o w2
  off[2] = o; o += static_cast<size_t>(K) * row;        // Q
  off[3] = o; o += static_cast<size_t>(K) * ldk;        // Re C
  off[4] = o; o += static_cast<size_t>(K) * ldk;        // Im C
  return o * sizeof(double);
}

}  // namespace
}  // namespace fase

using namespace fase;

extern "C" size_t fase_gram_workspace(int K, int M) {
  return K < 1 || M < 1 ? 0 : sizeof(double) * static_cast<size_t>(K) * ((M + 1) / 2 * 2);
}

extern "C" size_t fase_init_products_workspace(int M, int B) {
  return M < 1 || B < 1 ? 0 : sizeof(double) * static_cast<size_t>(B) * ((M + 1) / 2 * 2);
}

extern "C" int fase_gram(const double* phi, int64_t ldphi, const double* w, int K, int M, double* G,
                         int64_t ldg, void* ws, size_t ws_bytes, void* stream) {
  if (K < 1 || M < 1) {
    set_error("fase_gram: K and M must be positive (K=%d, M=%d)", K, M);
    return FASE_ERR_SHAPE;
  }
  if (!operand_ok(phi, ldphi) || ldphi < M || !w || !aligned16(w) || !G || ldg < K) {
    set_error("fase_gram: bad operand (null, misaligned, odd or short leading dimension)");
    return FASE_ERR_SHAPE;
  }
  if (!ws || !aligned16(ws) || ws_bytes < fase_gram_workspace(K, M)) {
    set_error("fase_gram: workspace must hold fase_gram_workspace(K, M) bytes");
    return FASE_ERR_SHAPE;
  }
  double* pw = static_cast<double*>(ws);
  const int64_t ldw = (M + 1) / 2 * 2;
  const cudaStream_t s = as_stream(stream);
  int st = launch_weigh(phi, ldphi, w, 0, K, M, pw, ldw, s, "fase_gram (weigh)");
  if (st != FASE_OK) return st;
  GemmParams p{pw, ldw, phi, ldphi, G, ldg, K, K, M};
  return launch<TileMain, true>(p, s, "fase_gram");
}

extern "C" int fase_init_products(const double* phi, int64_t ldphi, const double* f, int64_t ldf,
                                  const double* w, int64_t ldw, int K, int M, int B, double* R0,
                                  int64_t ldr, void* ws, size_t ws_bytes, void* stream) {
  if (K < 1 || M < 1 || B < 0) {
    set_error("fase_init_products: bad sizes (K=%d, M=%d, B=%d)", K, M, B);
    return FASE_ERR_SHAPE;
  }
  if (B == 0) return FASE_OK;
  if (!operand_ok(phi, ldphi) || ldphi < M || !operand_ok(f, ldf) || ldf < M || !w ||
      !aligned16(w) || (ldw != 0 && (ldw % 2 || ldw < M)) || !R0 || ldr < K) {
    set_error("fase_init_products: bad operand (null, misaligned, odd or short leading dimension)");
    return FASE_ERR_SHAPE;
  }
  if (!ws || !aligned16(ws) || ws_bytes < fase_init_products_workspace(M, B)) {
    set_error("fase_init_products: workspace must hold fase_init_products_workspace(M, B) bytes");
    return FASE_ERR_SHAPE;
  }
  double* fw = static_cast<double*>(ws);
  const int64_t ldfw = (M + 1) / 2 * 2;
  const cudaStream_t s = as_stream(stream);
  int st = launch_weigh(f, ldf, w, ldw, B, M, fw, ldfw, s, "fase_init_products (weigh)");
  if (st != FASE_OK) return st;
  if (B <= kGemvMax) {
    const int threads = 256;
    const int blocks = (K + threads / 32 - 1) / (threads / 32);
    gemv_rows_kernel<<<blocks < 148 * 8 ? blocks : 148 * 8, threads, 0, s>>>(
        fw, ldfw, B, phi, ldphi, K, M, R0, ldr);
    return check_launch("fase_init_products (gemv)");
  }
  GemmParams p{fw, ldfw, phi, ldphi, R0, ldr, B, K, M};
  return launch<TileMain, false>(p, s, "fase_init_products");
}

extern "C" int fase_gemm_nt(const double* A, int64_t lda, const double* B, int64_t ldb, int M,
                            int N, int Kd, double* C, int64_t ldc, int variant, void* stream) {
  if (M < 0 || N < 0 || Kd < 1) {
    set_error("fase_gemm_nt: bad sizes (M=%d, N=%d, K=%d)", M, N, Kd);
    return FASE_ERR_SHAPE;
  }
  if (M == 0 || N == 0) return FASE_OK;
  if (!operand_ok(A, lda) || !operand_ok(B, ldb) || lda < Kd || ldb < Kd || !C || ldc < N) {
    set_error("fase_gemm_nt: bad operand (null, misaligned, odd or short leading dimension)");
    return FASE_ERR_SHAPE;
  }
  GemmParams p{A, lda, B, ldb, C, ldc, M, N, Kd};
  return variant == 1 ? launch<TileBig, false>(p, as_stream(stream), "fase_gemm_nt")
                      : launch<TileMain, false>(p, as_stream(stream), "fase_gemm_nt");
}

extern "C" int fase_weigh(const double* x, int64_t ldx, const double* w, int64_t ldw, int rows,
                          int M, double* out, int64_t ldo, void* stream) {
  if (rows < 0 || M < 1 || ldx < M || ldo < M || (ldw != 0 && ldw < M) || (ldx & 1) ||
      (ldo & 1) || (ldw & 1)) {
    set_error("fase_weigh: bad sizes or odd leading dimension (rows=%d, M=%d)", rows, M);
    return FASE_ERR_SHAPE;
  }
  if (rows == 0) return FASE_OK;
  if (!x || !w || !out || !aligned16(x) || !aligned16(w) || !aligned16(out)) {
    set_error("fase_weigh: null or misaligned pointer");
    return FASE_ERR_SHAPE;
  }
  return launch_weigh(x, ldx, w, ldw, rows, M, out, ldo, as_stream(stream), "fase_weigh");
}

extern "C" size_t fase_gram_complex_workspace(int K, int64_t ldphi) {
  size_t off[5];
  return K < 1 || ldphi < 1 ? 0 : complex_gram_parts(K, ldphi, off);
}

extern "C" int fase_gram_complex(const double* phi2, int64_t ldphi, const double* w, int K, int M,
                                 double* T, int64_t ldt, void* ws, size_t ws_bytes, void* stream) {
  if (K < 1 || M < 1) {
    set_error("fase_gram_complex: K and M must be positive (K=%d, M=%d)", K, M);
    return FASE_ERR_SHAPE;
  }
  if (!operand_ok(phi2, ldphi) || ldphi < M || !w || !T || !aligned16(T) || ldt < K) {
    set_error("fase_gram_complex: bad operand (null, misaligned, odd or short leading dimension)");
    return FASE_ERR_SHAPE;
  }
  size_t off[5];
  if (!ws || !aligned16(ws) || ws_bytes < complex_gram_parts(K, ldphi, off)) {
    set_error("fase_gram_complex: workspace must hold fase_gram_complex_workspace(K, ldphi) bytes");
    return FASE_ERR_SHAPE;
  }
  double* base = static_cast<double*>(ws);
  double* w2 = base + off[0];
  double* pw = base + off[1];
  double* qm = base + off[2];
  double* cre = base + off[3];
  double* cim = base + off[4];
  const int64_t row = 2 * ldphi;
  const int64_t ldk = (K + 1) / 2 * 2;
  const cudaStream_t s = as_stream(stream);
  dup_weight_kernel<<<(static_cast<unsigned>(row) + 255) / 256, 256, 0, s>>>(w, M, ldphi, w2);
  int st = check_launch("fase_gram_complex (weights)");
  if (st != FASE_OK) return st;
  st = launch_weigh(phi2, row, w2, 0, K, static_cast<int>(row), pw, row, s, "fase_gram_complex (weigh)");
  if (st != FASE_OK) return st;
  const int64_t total = static_cast<int64_t>(K) * row;
  swap_halves_kernel<<<static_cast<unsigned>(total / 256 + 1 < 148 * 16 ? total / 256 + 1 : 148 * 16),
                       256, 0, s>>>(phi2, K, ldphi, qm);
  st = check_launch("fase_gram_complex (swap)");
  if (st != FASE_OK) return st;
  GemmParams pr{pw, row, phi2, row, cre, ldk, K, K, static_cast<int>(row)};
  st = launch<TileMain, true>(pr, s, "fase_gram_complex (re)");
  if (st != FASE_OK) return st;
  GemmParams pi{pw, row, qm, row, cim, ldk, K, K, static_cast<int>(row)};
  st = launch<TileMain, true>(pi, s, "fase_gram_complex (im)");
  if (st != FASE_OK) return st;
  dim3 grid(static_cast<unsigned>((ldt + 31) / 32), static_cast<unsigned>((K + 31) / 32));
  hermitian_pack_kernel<<<grid, dim3(32, 8), 0, s>>>(cre, cim, ldk, K, reinterpret_cast<double2*>(T),
                                                     ldt);
  return check_launch("fase_gram_complex (pack)");
}

extern "C" int fase_weigh_gather(const double* x, int64_t ldx, const int32_t* idx, const double* w,
                                 int rows, int n, double* out, int64_t ldo, void* stream) {
  if (rows < 0 || n < 1 || ldo < (n + 1) / 2 * 2) {
    set_error("fase_weigh_gather: bad sizes (rows=%d, n=%d, ldo=%lld)", rows, n,
              static_cast<long long>(ldo));
    return FASE_ERR_SHAPE;
  }
  if (rows == 0) return FASE_OK;
  if (!x || !idx || !w || !out) {
    set_error("fase_weigh_gather: null pointer");
    return FASE_ERR_SHAPE;
  }
  const int64_t total = static_cast<int64_t>(rows) * ((n + 1) / 2 * 2);
  const int64_t blocks = (total + 255) / 256;
  weigh_gather_kernel<<<static_cast<unsigned>(blocks < 148 * 16 ? blocks : 148 * 16), 256, 0,
                        as_stream(stream)>>>(x, ldx, idx, w, rows, n, out, ldo);
  return check_launch("fase_weigh_gather");
}
