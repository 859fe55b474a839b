// C ABI plumbing plus the small kernels of libfase_b200: basis expansion,
// table normalizers, model synthesis / paste, L2 flush.

#include <cstdarg>
#include <cstring>

#include "common.cuh"

namespace fase {

namespace {
thread_local char g_last_error[512] = "";
}

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
}

namespace {

// phi[(row0 + u*Lc + v) * ld + m*Nc + n] = rows[u, m] * cols[v, n]
// (reference dictionary.py:167-178: one rounded product per sample).
__global__ void basis_outer_kernel(const double* __restrict__ rows, int Lr, int Mr,
                                   const double* __restrict__ cols, int Lc, int Nc,
                                   double* __restrict__ phi, int64_t ld, int64_t row0) {
  const int64_t area = static_cast<int64_t>(Mr) * Nc;
  const int64_t total = static_cast<int64_t>(Lr) * Lc * area;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t atom = i / area;
    const int64_t s = i - atom * area;
    const int u = static_cast<int>(atom / Lc);
    const int v = static_cast<int>(atom - static_cast<int64_t>(u) * Lc);
    const int m = static_cast<int>(s / Nc);
    const int n = static_cast<int>(s - static_cast<int64_t>(m) * Nc);
    phi[(row0 + atom) * ld + s] = mul_rn(rows[u * Mr + m], cols[v * Nc + n]);
  }
}

// Block-wide max of non-negative doubles (fmax is exact).
template <int NT>
__device__ double block_max(double v, double* scratch) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  double m = scratch[0];
#pragma unroll
  for (int w = 1; w < NT / 32; ++w) m = fmax(m, scratch[w]);
  return m;
}

template <int NT>
__device__ int block_sum(int v, int* scratch) {
  v = __reduce_add_sync(0xffffffffu, v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  int s = 0;
#pragma unroll
  for (int w = 0; w < NT / 32; ++w) s += scratch[w];
  return s;
}

// D from a table diagonal: _finish_tables (reference fast.py:97-106).
// 1.0 / sqrt(x): IEEE sqrt and division, both correctly rounded like numpy's.
__device__ __forceinline__ double normalizer(double diag, double top) {
  return (top > 0.0 && diag > mul_rn(1e-12, top)) ? 1.0 / sqrt(diag) : 0.0;
}

constexpr int kFinishThreads = 1024;

__global__ void __launch_bounds__(kFinishThreads) gram_finish_kernel(const double* __restrict__ G,
                                                                     int64_t ldg, int K,
                                                                     double* __restrict__ D,
                                                                     int32_t* n_alive) {
  __shared__ double s_m[kFinishThreads / 32];
  __shared__ int s_n[kFinishThreads / 32];
  double m = 0.0;
  for (int k = threadIdx.x; k < K; k += kFinishThreads) m = fmax(m, G[k * ldg + k]);
  const double top = block_max<kFinishThreads>(m, s_m);
  int alive = 0;
  for (int k = threadIdx.x; k < K; k += kFinishThreads) {
    const double dk = normalizer(G[k * ldg + k], top);
    D[k] = dk;
    alive += dk != 0.0;
  }
  alive = block_sum<kFinishThreads>(alive, s_n);
  if (n_alive && threadIdx.x == 0) *n_alive = alive;
}

// Column-scaled table of the scaled recursion: Gs[u, k] = G[u, k] * D_k for
// k < K (0 for dead atoms, D_k == 0), zero padding up to lds. One CTA streams
// rows; 16-byte loads and stores.
__global__ void __launch_bounds__(256) scale_columns_kernel(const double* __restrict__ G,
                                                            int64_t ldg, const double* __restrict__ D,
                                                            int rows, int K, double* __restrict__ Gs,
                                                            int64_t lds) {
  const int pairs = static_cast<int>(lds / 2);
  for (int64_t u = blockIdx.x; u < rows; u += gridDim.x) {
    const double* g = G + u * ldg;
    double* o = Gs + u * lds;
    for (int p = threadIdx.x; p < pairs; p += blockDim.x) {
      const int k = 2 * p;
      double2 v = make_double2(0.0, 0.0);
      if (k < K) v.x = mul_rn(g[k], D[k]);
      if (k + 1 < K) v.y = mul_rn(g[k + 1], D[k + 1]);
      reinterpret_cast<double2*>(o)[p] = v;
    }
  }
}

constexpr int kNormThreads = 256;

__device__ __forceinline__ double chunk_diag(const double* G0, int64_t ldg, const double* tabs,
                                             int64_t stride, const int32_t* ids, int nch, int k) {
  const int64_t off = static_cast<int64_t>(k) * ldg + k;
  double x = G0[off];
  for (int c = 0; c < nch; ++c) x = sub_rn(x, tabs[static_cast<int64_t>(ids[c]) * stride + off]);
  return x;
}

__global__ void __launch_bounds__(kNormThreads) block_normalizers_kernel(
    const double* __restrict__ G0, int64_t ldg, const double* __restrict__ tabs, int64_t stride,
    const int32_t* __restrict__ counts, const int32_t* __restrict__ ids, int64_t list_ld, int K,
    double* __restrict__ D, int64_t ldd, int32_t* n_alive) {
  __shared__ double s_m[kNormThreads / 32];
  __shared__ int s_n[kNormThreads / 32];
  const int b = blockIdx.x;
  const int nch = counts ? counts[b] : 0;
  const int32_t* my = ids ? ids + static_cast<int64_t>(b) * list_ld : nullptr;
  double m = 0.0;
  for (int k = threadIdx.x; k < K; k += kNormThreads)
    m = fmax(m, chunk_diag(G0, ldg, tabs, stride, my, nch, k));
  const double top = block_max<kNormThreads>(m, s_m);
  double* Db = D + static_cast<int64_t>(b) * ldd;
  int alive = 0;
  for (int k = threadIdx.x; k < K; k += kNormThreads) {
    const double dk = normalizer(chunk_diag(G0, ldg, tabs, stride, my, nch, k), top);
    Db[k] = dk;
    alive += dk != 0.0;
  }
  alive = block_sum<kNormThreads>(alive, s_n);
  if (n_alive && threadIdx.x == 0) n_alive[b] = alive;
}

// g = sum_t coef_t * phi[sel_t, m] in selection order: SparseModel.materialize
// (reference.py:120-125) restricted to the lost samples, then the paste of
// apply_model (fast.py:267-286). Selection terms are staged in shared memory.
constexpr int kSynthThreads = 256;
constexpr int kSynthChunk = 1024;

template <int G>
__global__ void __launch_bounds__(kSynthThreads) synth_paste_kernel(
    const double* __restrict__ phi, int64_t ldphi, const int32_t* __restrict__ sel,
    const double* __restrict__ coef, int64_t ldo, int I, const int32_t* __restrict__ idx_ptr,
    const int32_t* __restrict__ idx, int n_shared, const int64_t* __restrict__ dst,
    double* __restrict__ out, int64_t ldout) {
  __shared__ int32_t s_sel[kSynthChunk];
  __shared__ double s_coef[kSynthChunk];
  const int b = blockIdx.x;
  const int lo = idx_ptr ? idx_ptr[b] : 0;
  const int n = idx_ptr ? idx_ptr[b + 1] - lo : n_shared;
  const int32_t* my_idx = idx + lo;
  const int32_t* my_sel = sel + static_cast<int64_t>(b) * ldo;
  const double* my_coef = coef + static_cast<int64_t>(b) * ldo;
  for (int base = 0; base < n; base += kSynthThreads) {
    const int i = base + threadIdx.x;
    const int m = i < n ? my_idx[i] : 0;
    double g = 0.0;
    for (int t0 = 0; t0 < I; t0 += kSynthChunk) {
      const int len = min(kSynthChunk, I - t0);
      __syncthreads();
      for (int t = threadIdx.x; t < len; t += kSynthThreads) {
        s_sel[t] = my_sel[t0 + t];
        s_coef[t] = my_coef[t0 + t];
      }
      __syncthreads();
      if (i < n) g = synth_terms<G>(phi, ldphi, s_sel, s_coef, len, m, g);
    }
    if (i < n) out[(dst ? dst[lo + i] : static_cast<int64_t>(m)) + static_cast<int64_t>(b) * ldout] = g;
  }
}

// Throughput shape for batches that fill the GPU: 128 threads per block, two
// samples per thread (m0 = idx[base + tid], m1 = idx[base + 128 + tid]) sharing
// each term's row address, coefficient and selection loads, with two
// independent accumulation chains per thread. The number of valid terms of a
// chunk (up to the first sel < 0, where the recursion stopped) is found while
// staging, so the term loop carries no per-term checks. Each sample's sum is
// still accumulated strictly in selection order (bit-identical output).
constexpr int kSynthPairThreads = 128;

template <int G>
__global__ void __launch_bounds__(kSynthPairThreads) synth_paste_pair_kernel(
    const double* __restrict__ phi, int64_t ldphi, const int32_t* __restrict__ sel,
    const double* __restrict__ coef, int64_t ldo, int I, const int32_t* __restrict__ idx_ptr,
    const int32_t* __restrict__ idx, int n_shared, const int64_t* __restrict__ dst,
    double* __restrict__ out, int64_t ldout) {
  __shared__ int32_t s_sel[kSynthChunk];
  __shared__ double s_coef[kSynthChunk];
  __shared__ int s_len;
  const int b = blockIdx.x;
  const int tid = static_cast<int>(threadIdx.x);
  const int lo = idx_ptr ? idx_ptr[b] : 0;
  const int n = idx_ptr ? idx_ptr[b + 1] - lo : n_shared;
  const int32_t* my_idx = idx + lo;
  const int32_t* my_sel = sel + static_cast<int64_t>(b) * ldo;
  const double* my_coef = coef + static_cast<int64_t>(b) * ldo;
  for (int base = 0; base < n; base += 2 * kSynthPairThreads) {
    const int i0 = base + tid, i1 = base + kSynthPairThreads + tid;
    const int m0 = i0 < n ? my_idx[i0] : 0;
    const int m1 = i1 < n ? my_idx[i1] : m0;
    double g0 = 0.0, g1 = 0.0;
    for (int t0 = 0; t0 < I; t0 += kSynthChunk) {
      const int len = min(kSynthChunk, I - t0);
      __syncthreads();
      if (tid == 0) s_len = len;
      __syncthreads();
      for (int t = tid; t < len; t += kSynthPairThreads) {
        const int u = my_sel[t0 + t];
        s_sel[t] = u;
        s_coef[t] = my_coef[t0 + t];
        if (u < 0) atomicMin(&s_len, t);
      }
      __syncthreads();
      const int lv = s_len;
      for (int tb = 0; tb < lv; tb += G) {
        double v0[G], v1[G];
#pragma unroll
        for (int j = 0; j < G; ++j) {
          const int t = tb + j;
          if (t < lv) {
            const double* row = phi + static_cast<int64_t>(s_sel[t]) * ldphi;
            v0[j] = __ldg(row + m0);
            v1[j] = __ldg(row + m1);
          }
        }
#pragma unroll
        for (int j = 0; j < G; ++j) {
          const int t = tb + j;
          if (t < lv) {
            const double c = s_coef[t];
            g0 = __dadd_rn(g0, __dmul_rn(c, v0[j]));
            g1 = __dadd_rn(g1, __dmul_rn(c, v1[j]));
          }
        }
      }
      if (lv < len) break;  // the recursion stopped: no later terms
    }
    const int64_t ob = static_cast<int64_t>(b) * ldout;
    if (i0 < n) out[(dst ? dst[lo + i0] : static_cast<int64_t>(m0)) + ob] = g0;
    if (i1 < n) out[(dst ? dst[lo + i1] : static_cast<int64_t>(m1)) + ob] = g1;
  }
}

// Complex dictionaries (conjugate-split rows: phi2[2u] = Re phi_u,
// phi2[2u+1] = -Im phi_u): g = sum_t coef_t * phi_{sel_t} with numpy's fused
// complex product (np_cmul), accumulated in selection order
// (reference.py:120-125); Re g is pasted (fast.py:282) and max |Im g| over the
// block's samples goes to max_imag[b] (apply_model's diagnostic, fast.py:284).
__global__ void __launch_bounds__(kSynthThreads) synth_paste_complex_kernel(
    const double* __restrict__ phi2, int64_t ldphi, const int32_t* __restrict__ sel,
    const double* __restrict__ coef, int64_t ldo, int I, const int32_t* __restrict__ idx_ptr,
    const int32_t* __restrict__ idx, int n_shared, const int64_t* __restrict__ dst,
    double* __restrict__ out, int64_t ldout, double* __restrict__ max_imag) {
  __shared__ int32_t s_sel[kSynthChunk];
  __shared__ double2 s_coef[kSynthChunk];
  __shared__ double s_m[kSynthThreads / 32];
  const int b = blockIdx.x;
  const int lo = idx_ptr ? idx_ptr[b] : 0;
  const int n = idx_ptr ? idx_ptr[b + 1] - lo : n_shared;
  const int32_t* my_idx = idx + lo;
  const int32_t* my_sel = sel + static_cast<int64_t>(b) * ldo;
  const double* my_coef = coef + 2 * static_cast<int64_t>(b) * ldo;
  double imax = 0.0;
  for (int base = 0; base < n; base += kSynthThreads) {
    const int i = base + threadIdx.x;
    const int m = i < n ? my_idx[i] : 0;
    double gr = 0.0, gi = 0.0;
    bool done = false;
    for (int t0 = 0; t0 < I; t0 += kSynthChunk) {
      const int len = min(kSynthChunk, I - t0);
      __syncthreads();
      for (int t = threadIdx.x; t < len; t += kSynthThreads) {
        s_sel[t] = my_sel[t0 + t];
        s_coef[t] = make_double2(my_coef[2 * (t0 + t)], my_coef[2 * (t0 + t) + 1]);
      }
      __syncthreads();
      if (i < n && !done) {
        for (int t = 0; t < len; ++t) {
          const int u = s_sel[t];
          if (u < 0) {  // block without selectable atoms: terms end here
            done = true;
            break;
          }
          const double pr = __ldg(phi2 + (2 * static_cast<int64_t>(u)) * ldphi + m);
          const double pi = -__ldg(phi2 + (2 * static_cast<int64_t>(u) + 1) * ldphi + m);
          const double2 c = s_coef[t];
          const double2 x = np_cmul(c.x, c.y, pr, pi);
          gr = add_rn(gr, x.x);
          gi = add_rn(gi, x.y);
        }
      }
    }
    if (i < n) {
      out[(dst ? dst[lo + i] : static_cast<int64_t>(m)) + static_cast<int64_t>(b) * ldout] = gr;
      imax = fmax(imax, fabs(gi));
    }
  }
  if (max_imag) {
    const double v = block_max<kSynthThreads>(imax, s_m);
    if (threadIdx.x == 0) max_imag[b] = v;
  }
}

__global__ void flush_kernel(uint4* buf, size_t n, unsigned salt) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    buf[i] = make_uint4(salt, salt ^ 1u, salt ^ 2u, static_cast<unsigned>(i));
}

// G[i, j] <- G[j, i] for i > j (32 x 32 tiles through shared memory): the
// lower triangle of a table whose rows were built as independent panels
// (multi-GPU table build) becomes the exact mirror of the upper one, as the
// single-GPU symmetric build writes it
__global__ void __launch_bounds__(256) mirror_upper_kernel(double* __restrict__ G, int64_t ldg,
                                                           int K) {
  __shared__ double tile[32][33];
  const int tiles = (K + 31) / 32;
  for (int64_t tt = blockIdx.x; tt < static_cast<int64_t>(tiles) * tiles; tt += gridDim.x) {
    const int bi = static_cast<int>(tt / tiles), bj = static_cast<int>(tt % tiles);
    if (bi < bj) continue;  // destination tiles on or below the diagonal
    __syncthreads();
    // read the source tile (rows bj*32.., cols bi*32..) of the upper triangle
    for (int e = threadIdx.x; e < 1024; e += blockDim.x) {
      const int r = bj * 32 + (e >> 5), c = bi * 32 + (e & 31);
      tile[e >> 5][e & 31] = (r < K && c < K) ? G[static_cast<int64_t>(r) * ldg + c] : 0.0;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < 1024; e += blockDim.x) {
      const int r = bi * 32 + (e >> 5), c = bj * 32 + (e & 31);
      if (r < K && c < K && r > c) G[static_cast<int64_t>(r) * ldg + c] = tile[e & 31][e >> 5];
    }
  }
}
}  // namespace
}  // namespace fase

using namespace fase;

extern "C" const char* fase_last_error(void) { return g_last_error; }

// 2.0: fase_iterate_args gained l2_hot (round 2) -- callers built against 1.x
// pass a shorter argument block
// 3.0: fase_iterate_args.order (dispatch order) appended
extern "C" int fase_abi_version(void) { return (3 << 16) | 0; }

extern "C" int fase_basis_outer(const double* rows, int Lr, int Mr, const double* cols, int Lc,
                                int Nc, double* phi, int64_t ldphi, int64_t row0, void* stream) {
  if (Lr < 1 || Mr < 1 || Lc < 1 || Nc < 1 || row0 < 0 || ldphi < static_cast<int64_t>(Mr) * Nc) {
    set_error("fase_basis_outer: bad sizes (Lr=%d Mr=%d Lc=%d Nc=%d ld=%lld)", Lr, Mr, Lc, Nc,
              static_cast<long long>(ldphi));
    return FASE_ERR_SHAPE;
  }
  if (!rows || !cols || !phi) {
    set_error("fase_basis_outer: null pointer");
    return FASE_ERR_SHAPE;
  }
  const int64_t total = static_cast<int64_t>(Lr) * Lc * Mr * Nc;
  const int threads = 256;
  const int64_t blocks = (total + threads - 1) / threads;
  basis_outer_kernel<<<static_cast<unsigned>(blocks < 148 * 64 ? blocks : 148 * 64), threads, 0,
                       as_stream(stream)>>>(rows, Lr, Mr, cols, Lc, Nc, phi, ldphi, row0);
  return check_launch("fase_basis_outer");
}

extern "C" int fase_gram_finish(const double* G, int64_t ldg, int K, double* D, int32_t* n_alive,
                                void* stream) {
  if (K < 1 || ldg < K || !G || !D) {
    set_error("fase_gram_finish: bad operand (K=%d)", K);
    return FASE_ERR_SHAPE;
  }
  gram_finish_kernel<<<1, kFinishThreads, 0, as_stream(stream)>>>(G, ldg, K, D, n_alive);
  return check_launch("fase_gram_finish");
}

extern "C" int fase_scale_columns(const double* G, int64_t ldg, const double* D, int rows, int K,
                                  double* Gs, int64_t lds, void* stream) {
  if (rows < 1 || K < 1 || ldg < K || lds < K || (lds & 1) || !G || !D || !Gs || !aligned16(Gs)) {
    set_error("fase_scale_columns: bad operand (rows=%d, K=%d, ldg=%lld, lds=%lld)", rows, K,
              static_cast<long long>(ldg), static_cast<long long>(lds));
    return FASE_ERR_SHAPE;
  }
  scale_columns_kernel<<<min(rows, 148 * 8), 256, 0, as_stream(stream)>>>(G, ldg, D, rows, K, Gs,
                                                                          lds);
  return check_launch("fase_scale_columns");
}

extern "C" int fase_block_normalizers(const double* G0, int64_t ldg, const double* chunk_tables,
                                      int64_t chunk_stride, const int32_t* chunk_count,
                                      const int32_t* chunk_ids, int64_t chunk_list_ld, int K,
                                      int B, double* D, int64_t ldd, int32_t* n_alive,
                                      void* stream) {
  // ldg == 0: G0 and the chunk tables are given as their diagonals
  // (G0[k], chunk_tables[id * chunk_stride + k]), e.g. extracted once per table
  // set -- contiguous reads instead of one sector per diagonal element
  if (K < 1 || B < 0 || (ldg != 0 && ldg < K) || ldd < K || !G0 || !D) {
    set_error("fase_block_normalizers: bad operand (K=%d, B=%d)", K, B);
    return FASE_ERR_SHAPE;
  }
  if (chunk_count && (!chunk_ids || !chunk_tables)) {
    set_error("fase_block_normalizers: chunk list without chunk tables");
    return FASE_ERR_SHAPE;
  }
  if (B == 0) return FASE_OK;
  block_normalizers_kernel<<<B, kNormThreads, 0, as_stream(stream)>>>(
      G0, ldg, chunk_tables, chunk_stride, chunk_count, chunk_ids, chunk_list_ld, K, D, ldd,
      n_alive);
  return check_launch("fase_block_normalizers");
}

extern "C" int fase_synth_paste(const double* phi, int64_t ldphi, const int32_t* sel,
                                const double* coef, int64_t ldo, int I, int B,
                                const int32_t* idx_ptr, const int32_t* idx, int n_shared,
                                const int64_t* dst, double* out, int64_t ldout, void* stream) {
  if (I < 1 || B < 0 || ldo < I || (!idx_ptr && n_shared < 0)) {
    set_error("fase_synth_paste: bad sizes (I=%d, B=%d)", I, B);
    return FASE_ERR_SHAPE;
  }
  if (B == 0 || (!idx_ptr && n_shared == 0)) return FASE_OK;
  if (!phi || !sel || !coef || !idx || !out) {
    set_error("fase_synth_paste: null pointer");
    return FASE_ERR_SHAPE;
  }
  // a batch that cannot fill the GPU is latency-bound: keep more atom values in
  // flight; larger batches take the two-samples-per-thread shape
  if (B < 148) {
    synth_paste_kernel<32><<<B, kSynthThreads, 0, as_stream(stream)>>>(
        phi, ldphi, sel, coef, ldo, I, idx_ptr, idx, n_shared, dst, out, ldout);
  } else {
    synth_paste_pair_kernel<8><<<B, kSynthPairThreads, 0, as_stream(stream)>>>(
        phi, ldphi, sel, coef, ldo, I, idx_ptr, idx, n_shared, dst, out, ldout);
  }
  return check_launch("fase_synth_paste");
}

extern "C" int fase_synth_paste_complex(const double* phi2, int64_t ldphi, const int32_t* sel,
                                        const double* coef, int64_t ldo, int I, int B,
                                        const int32_t* idx_ptr, const int32_t* idx, int n_shared,
                                        const int64_t* dst, double* out, int64_t ldout,
                                        double* max_imag, void* stream) {
  if (I < 1 || B < 0 || ldo < I || (!idx_ptr && n_shared < 0)) {
    set_error("fase_synth_paste_complex: bad sizes (I=%d, B=%d)", I, B);
    return FASE_ERR_SHAPE;
  }
  if (B == 0) return FASE_OK;
  if (!phi2 || !sel || !coef || (!idx && (idx_ptr || n_shared > 0)) || !out) {
    set_error("fase_synth_paste_complex: null pointer");
    return FASE_ERR_SHAPE;
  }
  synth_paste_complex_kernel<<<B, kSynthThreads, 0, as_stream(stream)>>>(
      phi2, ldphi, sel, coef, ldo, I, idx_ptr, idx, n_shared, dst, out, ldout, max_imag);
  return check_launch("fase_synth_paste_complex");
}

extern "C" int fase_mirror_upper(double* G, int64_t ldg, int K, void* stream) {
  if (K < 0 || ldg < K) {
    set_error("fase_mirror_upper: bad sizes (K=%d, ldg=%lld)", K, static_cast<long long>(ldg));
    return FASE_ERR_SHAPE;
  }
  if (K < 2) return FASE_OK;
  if (!G) {
    set_error("fase_mirror_upper: null table");
    return FASE_ERR_SHAPE;
  }
  const int64_t tiles = static_cast<int64_t>((K + 31) / 32) * ((K + 31) / 32);
  const int grid = static_cast<int>(tiles < 148 * 8 ? tiles : 148 * 8);
  mirror_upper_kernel<<<grid, 256, 0, as_stream(stream)>>>(G, ldg, K);
  return check_launch("fase_mirror_upper");
}

extern "C" int fase_l2_flush(void* buf, size_t bytes, void* stream) {
  if (!buf || bytes < 16) {
    set_error("fase_l2_flush: need a buffer of at least 16 bytes");
    return FASE_ERR_SHAPE;
  }
  static unsigned salt = 0;
  flush_kernel<<<148 * 8, 512, 0, as_stream(stream)>>>(static_cast<uint4*>(buf), bytes / 16,
                                                       ++salt);
  return check_launch("fase_l2_flush");
}
