// FP64 contractions on the 5th-generation tensor cores: the Ozaki scheme with
// tcgen05 INT8 MMAs (kind::i8, int32 accumulators in TMEM).
//
// FP64 has no tcgen05 kind on sm_100a; DMMA (csrc/dgemm.cu) tops out near
// 37 TFLOP/s. Splitting every FP64 row into s signed 7-bit digits,
//   x[r, k] = 2^e_r * sum_{i=1..s} a_i[r, k] 2^{-7i}  (+ |residual| < 2^{e_r - 7s}),
// turns C = X Y^T into integer products of digit matrices:
//   C[r, c] ~= 2^{e_r + f_c} * sum_{d=2..s+1} 2^{-7d} * sum_{i+j=d} (A_i B_j^T)[r, c],
// keeping the pairs i + j <= s + 1 (the dropped pairs lie below 2^{-7(s+2)} of
// the leading term). Every A_i B_j^T is an exact int8 x int8 -> int32
// contraction (|sum| <= Kd * 127^2 * s < 2^31 for Kd <= 16384), pairs of one
// diagonal d share one TMEM accumulator, and the epilogue combines the s
// diagonals in FP64 from the smallest weight up and applies the row scales.
//
// Used for the dense initial products R0 = (F o W) Phi^T over the support
// (initial_scalar_products, fast.py:145-157): the digit planes of Phi are cut
// once per plan, those of the weighted signals once per batch.
//
// Kernel: one CTA per 128 x 64 output tile, 256 threads. Digit planes are
// stored in global memory already in the K-major, no-swizzle UMMA layout
// (8-row x 16-byte core matrices, grouped per 64-byte K block), so a tile's
// slab of one plane is one contiguous run: a stage (s planes of a 128 x 64-byte
// A slab and a 64 x 64-byte B slab) arrives by 2s TMA bulk copies issued by one
// thread, completing on the stage's full mbarrier. Another thread issues the
// MMAs -- digit i of A against the stacked digits 0..s-1-i of B, up to N = 256
// per instruction, so each A digit is read from shared memory once or twice per
// K step instead of s - i times (the smem operand bandwidth, not the tensor
// pipe, bounded the one-pair-per-MMA form) -- and commits to the stage's empty
// mbarrier. TMEM holds s accumulators of 64 columns; all eight
// warps run the epilogue.

#include <climits>
#include <cstdlib>

#include "common.cuh"

namespace fase {
namespace {

constexpr int OZ_BM = 128, OZ_BN = 64, OZ_BK = 64;  // rows, cols, K bytes per stage
constexpr int OZ_THREADS = 256;
constexpr int OZ_STAGES = 2;  // (32-byte stages x 4 measured 5% slower)
constexpr int OZ_RG = 8 * OZ_BK;  // bytes of one 8-row group of a slab (UMMA SBO)
constexpr int OZ_MAX_SLICES = 8;

__device__ __forceinline__ uint64_t umma_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return static_cast<uint64_t>((addr >> 4) & 0x3FFF) |
         (static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);  // version 1
}

// kind::i8: int32 accumulate (c_format 2), signed A / B (format 1), K-major,
// M = OZ_BM (bits 24-28, >> 4); N (bits 17-22, >> 3) is set per instruction
constexpr uint32_t kOzIdescBase = (2u << 4) | (1u << 7) | (1u << 10) |
                                  (static_cast<uint32_t>(OZ_BM >> 4) << 24);

// Byte offset of (row r, K byte k) inside one digit plane, in the UMMA-ready
// tiled layout: [K block of OZ_BK B][8-row group][16-byte K chunk][row % 8][16 B].
// A tile's slab (all rows of the tile for one K block) is then one contiguous
// run of bytes, fetched by a single 1-D TMA bulk copy.
__device__ __forceinline__ int64_t plane_offset(int r, int64_t k, int64_t rows_pad) {
  return (k / OZ_BK) * (rows_pad * OZ_BK) + static_cast<int64_t>(r >> 3) * OZ_RG +
         ((k >> 4) % (OZ_BK / 16)) * 128 + (r & 7) * 16 + (k & 15);
}

// Digit planes of one FP64 row per CTA: v[k] = x[r, idx[k]] * w[k] (idx / w
// optional: the weighted operand restricted to the support, rounded once like
// fase_weigh_gather) is staged in shared memory with coalesced loads; e is the
// smallest integer with max|v| < 2^e; then each thread cuts 16 consecutive k
// into s truncated base-2^7 digits of v * 2^-e (each step exact) and stores one
// 16-byte chunk per plane.
constexpr int OZ_SPLIT_THREADS = 256;

// Cut the staged row s_v (kp values, one pad per 16) into S digit planes of
// row r: e = smallest integer with max|v| < 2^e (m = max|v| over the row, block-
// uniform), then each thread cuts 16 consecutive k into S truncated base-2^7
// digits of v * 2^-e (each step exact) and stores one 16-byte chunk per plane.
template <int S, class Get>
__device__ __forceinline__ void cut_row_planes(Get get, double m, int r, int64_t kp,
                                               int64_t rows_pad, int64_t plane_stride,
                                               int8_t* __restrict__ planes,
                                               int32_t* __restrict__ exps) {
  const int tid = threadIdx.x;
  const int chunks = static_cast<int>(kp >> 4);
  const int e = m > 0.0 ? ilogb(m) + 1 : 0;
  if (tid == 0) exps[r] = e;
  for (int c = tid; c < chunks; c += OZ_SPLIT_THREADS) {
    uint32_t packed[S][4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
#pragma unroll
      for (int i = 0; i < S; ++i) packed[i][q] = 0u;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        double y = get(c, 4 * q + b);
        if (y == 0.0) continue;  // all digits 0 (most entries of sparse model rows)
        y = scalbn(y, -e);       // |y| < 1, exact
#pragma unroll
        for (int i = 0; i < S; ++i) {
          y = y * 128.0;               // exact
          const double t = trunc(y);  // |t| <= 127
          y -= t;                      // exact
          packed[i][q] |= (static_cast<uint32_t>(static_cast<int>(t)) & 0xffu) << (8 * b);
        }
      }
    }
    const int64_t off = plane_offset(r, 16 * static_cast<int64_t>(c), rows_pad);
#pragma unroll
    for (int i = 0; i < S; ++i)
      *reinterpret_cast<uint4*>(planes + i * plane_stride + off) =
          make_uint4(packed[i][0], packed[i][1], packed[i][2], packed[i][3]);
  }
}

// block-wide max of the per-thread m (s_max: OZ_SPLIT_THREADS / 32 slots)
__device__ __forceinline__ double block_max_abs(double m, double* s_max) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) s_max[warp] = m;
  __syncthreads();
  m = s_max[0];
#pragma unroll
  for (int i = 1; i < OZ_SPLIT_THREADS / 32; ++i) m = fmax(m, s_max[i]);
  return m;
}

// Digit planes of one FP64 row per CTA: v[k] = x[r, idx[k]] * w[k] (idx / w
// optional: the weighted operand restricted to the support, rounded once like
// fase_weigh_gather) is staged in shared memory with coalesced loads, then cut.
template <int S>
__global__ void __launch_bounds__(OZ_SPLIT_THREADS) ozaki_split_kernel(
    const double* __restrict__ x, int64_t ldx, const int32_t* __restrict__ idx,
    const double* __restrict__ w, int rows, int kd, int8_t* __restrict__ planes, int64_t kp,
    int64_t rows_pad, int64_t plane_stride, int32_t* __restrict__ exps) {
  extern __shared__ double s_v[];  // kp + kp/16 (one pad per 16 against bank conflicts)
  __shared__ double s_max[OZ_SPLIT_THREADS / 32];
  const int tid = threadIdx.x;
  for (int r = blockIdx.x; r < rows; r += gridDim.x) {
    const double* xr = x + static_cast<int64_t>(r) * ldx;
    double m = 0.0;
    // eight independent gathers in flight per thread (the index loads, then
    // the values: one dependent global round trip per eight elements)
    constexpr int U = 8;
    for (int k0 = tid; k0 < kp; k0 += U * OZ_SPLIT_THREADS) {
      int col[U];
      double v[U], wk[U];
#pragma unroll
      for (int j = 0; j < U; ++j) {
        const int k = k0 + j * OZ_SPLIT_THREADS;
        col[j] = k < kd ? (idx ? __ldg(idx + k) : k) : -1;
        wk[j] = (w && k < kd) ? __ldg(w + k) : 1.0;
      }
#pragma unroll
      for (int j = 0; j < U; ++j) v[j] = col[j] >= 0 ? __ldg(xr + col[j]) : 0.0;
#pragma unroll
      for (int j = 0; j < U; ++j) {
        const int k = k0 + j * OZ_SPLIT_THREADS;
        if (w) v[j] = mul_rn(v[j], wk[j]);
        if (k < kp) {
          s_v[k + (k >> 4)] = v[j];
          m = fmax(m, fabs(v[j]));
        }
      }
    }
    m = block_max_abs(m, s_max);
    cut_row_planes<S>([&](int c, int j) { return s_v[17 * c + j]; }, m, r, kp, rows_pad,
                      plane_stride, planes, exps);
    __syncthreads();  // s_v / s_max reused by the next row
  }
}

// Digit planes of sparse rows: row r is the dense coefficient vector of the
// sparse model of block r, v[sel[r, t]] += coef[r, t] over its `iters` terms
// (terms with sel < 0 -- a run stopped by degeneracy -- or sel >= kd add
// nothing). Synthesis of the lost samples of a shared geometry is then one
// Ozaki product g = V Phi_lost^T (fase_ozaki_gemm).
// Shared memory holds a slot map (kp int32: the term that first names atom k,
// or -1) and the terms, not the dense row, so several CTAs share an SM. Every
// term claims its atom (atomicMin of the term index); when no atom is named
// twice each slot's value is its term's coefficient; repeated terms are
// flagged in a bit mask, and one thread walks the set bits in term order,
// adding each into its atom's first occurrence -- the same sums in the same
// order as a sequential scatter, on every run. The cut reads v[k] through the
// map.
template <int S>
__global__ void __launch_bounds__(OZ_SPLIT_THREADS) ozaki_split_sparse_kernel(
    const int32_t* __restrict__ sel, int64_t ldsel, const double* __restrict__ coef,
    int64_t ldcoef, int rows, int iters, int kd, int8_t* __restrict__ planes, int64_t kp,
    int64_t rows_pad, int64_t plane_stride, int32_t* __restrict__ exps) {
  extern __shared__ double s_dyn[];
  double* s_val = s_dyn;                                   // iters values
  int* s_u = reinterpret_cast<int*>(s_val + iters);        // iters atoms
  int* s_slot = reinterpret_cast<int*>(                    // kp slots, 16-byte aligned
      (reinterpret_cast<uintptr_t>(s_u + iters) + 15) & ~static_cast<uintptr_t>(15));
  unsigned* s_rep = reinterpret_cast<unsigned*>(s_slot + kp);  // (iters + 31) / 32 words
  __shared__ double s_max[OZ_SPLIT_THREADS / 32];
  __shared__ int s_dup;
  const int tid = threadIdx.x;
  const int rep_words = (iters + 31) >> 5;
  for (int r = blockIdx.x; r < rows; r += gridDim.x) {
    for (int k = 4 * tid; k < kp; k += 4 * OZ_SPLIT_THREADS)
      *reinterpret_cast<int4*>(s_slot + k) = make_int4(INT_MAX, INT_MAX, INT_MAX, INT_MAX);
    for (int i = tid; i < rep_words; i += OZ_SPLIT_THREADS) s_rep[i] = 0u;
    if (tid == 0) s_dup = 0;
    const int32_t* sr = sel + static_cast<int64_t>(r) * ldsel;
    const double* cr = coef + static_cast<int64_t>(r) * ldcoef;
    for (int t = tid; t < iters; t += OZ_SPLIT_THREADS) {
      const int u = __ldg(sr + t);
      s_u[t] = (u >= 0 && u < kd) ? u : -1;
      s_val[t] = __ldg(cr + t);
    }
    __syncthreads();
    for (int t = tid; t < iters; t += OZ_SPLIT_THREADS)
      if (s_u[t] >= 0) atomicMin(s_slot + s_u[t], t);
    __syncthreads();
    for (int t = tid; t < iters; t += OZ_SPLIT_THREADS)
      if (s_u[t] >= 0 && s_slot[s_u[t]] != t) {
        atomicOr(s_rep + (t >> 5), 1u << (t & 31));
        s_dup = 1;
      }
    __syncthreads();
    if (s_dup) {  // repeated atoms: each added, in term order, into the first occurrence
      if (tid == 0)
        for (int i = 0; i < rep_words; ++i)
          for (unsigned bits = s_rep[i]; bits; bits &= bits - 1u) {
            const int t = 32 * i + __ffs(bits) - 1;
            const int o = s_slot[s_u[t]];
            s_val[o] = s_val[o] + s_val[t];
            s_u[t] = -1;  // folded into its first occurrence
          }
      __syncthreads();
    }
    double m = 0.0;
    for (int t = tid; t < iters; t += OZ_SPLIT_THREADS)
      if (s_u[t] >= 0) m = fmax(m, fabs(s_val[t]));
    m = block_max_abs(m, s_max);
    cut_row_planes<S>(
        [&](int c, int j) {
          const int o = s_slot[16 * c + j];
          return o == INT_MAX ? 0.0 : s_val[o];
        },
        m, r, kp, rows_pad, plane_stride, planes, exps);
    __syncthreads();  // shared arrays reused by the next row
  }
}

template <int S>
__global__ void __launch_bounds__(OZ_THREADS, 1) ozaki_gemm_kernel(
    const int8_t* __restrict__ A, int64_t a_plane, const int32_t* __restrict__ ea,
    const int8_t* __restrict__ B, int64_t b_plane, const int32_t* __restrict__ eb, int64_t kp,
    int m_valid, int n_valid, int rows_a_pad, int rows_b_pad, double* __restrict__ C, int64_t ldc,
    int group_m, int sym) {
  constexpr int A_SLAB = OZ_BM * OZ_BK, B_SLAB = OZ_BN * OZ_BK;
  constexpr int STAGE = S * (A_SLAB + B_SLAB);
  constexpr int TMEM_COLS = 512;
  static_assert(S * OZ_BN <= TMEM_COLS, "one 64-column accumulator per diagonal");
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t full_bar[OZ_STAGES];
  __shared__ __align__(8) uint64_t empty_bar[OZ_STAGES];
  __shared__ __align__(8) uint64_t done_bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  // grouped raster: CTAs in flight cover group_m M-tiles x a band of N-tiles,
  // so each A / B slab is read by a bounded number of concurrent CTAs
  int tm, tn;
  {
    const int mt = (m_valid + OZ_BM - 1) / OZ_BM, nt = (n_valid + OZ_BN - 1) / OZ_BN;
    const int pid = blockIdx.x;
    const int per_group = group_m * nt;
    const int first_m = (pid / per_group) * group_m;
    const int gm = min(mt - first_m, group_m);
    tm = first_m + (pid % per_group) % gm;
    tn = (pid % per_group) / gm;
  }
  const int m0 = tm * OZ_BM, n0 = tn * OZ_BN;
  const int nk = static_cast<int>(kp / OZ_BK);
  // symmetric mode (Gram tables): only tiles holding entries r <= c; each such
  // entry is written to (r, c) and (c, r), so the table is bit-symmetric
  if (sym && m0 >= n0 + OZ_BN) return;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     smem_u32(&tmem_base)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 32) {
    for (int s = 0; s < OZ_STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    mbar_init(&done_bar, 1);
    fence_mbar_init();
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = tmem_base;
  const uint32_t sbase = smem_u32(smem);

  // warp-specialized pipeline: thread 0 streams slabs with TMA bulk copies
  // (one per digit plane), thread 32 issues the MMAs; full / empty mbarriers
  const int64_t a_kblock = static_cast<int64_t>(rows_a_pad) * OZ_BK;  // bytes per K block of a plane
  const int64_t b_kblock = static_cast<int64_t>(rows_b_pad) * OZ_BK;
  if (tid == 0) {
    for (int kb = 0; kb < nk; ++kb) {
      const int st = kb % OZ_STAGES;
      mbar_wait(&empty_bar[st], ((kb / OZ_STAGES) & 1) ^ 1);
      mbar_arrive_expect_tx(&full_bar[st], STAGE);
      uint8_t* sa = smem + st * STAGE;
      uint8_t* sb = sa + S * A_SLAB;
#pragma unroll
      for (int p = 0; p < S; ++p) {
        tma_load_1d(sa + p * A_SLAB, A + p * a_plane + kb * a_kblock + static_cast<int64_t>(m0 >> 3) * OZ_RG,
                    A_SLAB, &full_bar[st]);
        tma_load_1d(sb + p * B_SLAB, B + p * b_plane + kb * b_kblock + static_cast<int64_t>(n0 >> 3) * OZ_RG,
                    B_SLAB, &full_bar[st]);
      }
    }
  } else if (tid == 32) {
    for (int kb = 0; kb < nk; ++kb) {
      const int st = kb % OZ_STAGES;
      mbar_wait(&full_bar[st], (kb / OZ_STAGES) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n");
      const uint32_t sa = sbase + st * STAGE, sb = sa + S * A_SLAB;
#pragma unroll
      for (int ks = 0; ks < OZ_BK / 32; ++ks) {  // K = 32 per MMA
#pragma unroll
        for (int i = 0; i < S; ++i) {
          // digit i of A against digits j = 0 .. S-1-i of B in one wide MMA per
          // group of up to 4 planes: the B planes sit back to back in shared
          // memory (a uniform 64n-row operand) and their diagonals i + j are
          // consecutive 64-column TMEM blocks, so A is read once per group
#pragma unroll
          for (int jb = 0; jb < S - i; jb += 4) {
            const int nj = (S - i - jb) < 4 ? (S - i - jb) : 4;
            const uint64_t ad = umma_desc(sa + i * A_SLAB + ks * 256, 128, OZ_RG);
            const uint64_t bd = umma_desc(sb + jb * B_SLAB + ks * 256, 128, OZ_RG);
            const uint32_t idesc = kOzIdescBase | (static_cast<uint32_t>((nj * OZ_BN) >> 3) << 17);
            const uint32_t acc = (kb > 0 || ks > 0 || i > 0) ? 1u : 0u;  // digit 0 of A inits every diagonal
            const uint32_t dst = tmem + static_cast<uint32_t>((i + jb) * OZ_BN);
            asm volatile(
                "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(dst),
                "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
          }
        }
      }
      asm volatile(
          "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
              smem_u32(&empty_bar[st])));
    }
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
            smem_u32(&done_bar)));
  }
  __syncwarp();
  mbar_wait(&done_bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;\n");

  // epilogue: warp w reads lanes 32(w%4).. (tile rows) and columns half (w/4)
  const int row = m0 + (warp & 3) * 32 + (tid & 31);
  const int cbase = (warp >> 2) * (OZ_BN / 2);
  const int er = row < m_valid ? ea[row] : 0;
  for (int c0 = 0; c0 < OZ_BN / 2; c0 += 8) {
    double sum[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) sum[j] = 0.0;
#pragma unroll
    for (int d = S - 1; d >= 0; --d) {  // smallest weight first
      uint32_t v[8];
      const uint32_t taddr = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16) +
                             static_cast<uint32_t>(d * OZ_BN + cbase + c0);
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
            "=r"(v[7])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;\n");
      const double w = scalbn(1.0, -7 * (d + 2));
#pragma unroll
      for (int j = 0; j < 8; ++j) sum[j] = fma(static_cast<double>(static_cast<int32_t>(v[j])), w, sum[j]);
    }
    if (row < m_valid) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int col = n0 + cbase + c0 + j;
        if (col >= n_valid) continue;
        const double v = scalbn(sum[j], er + eb[col]);
        if (!sym) {
          C[static_cast<int64_t>(row) * ldc + col] = v;
        } else if (row <= col) {
          C[static_cast<int64_t>(row) * ldc + col] = v;
          C[static_cast<int64_t>(col) * ldc + row] = v;
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem),
                 "r"(TMEM_COLS));
}

}  // namespace
}  // namespace fase

using namespace fase;

extern "C" int fase_ozaki_split(const double* x, int64_t ldx, const int32_t* idx, const double* w,
                                int rows, int kd, int slices, int8_t* planes, int64_t kp,
                                int rows_pad, int32_t* exps, void* stream) {
  if (rows < 0 || kd < 1 || slices < 6 || slices > OZ_MAX_SLICES || kp < kd || kp % OZ_BK || kp > 16384 ||
      (!idx && ldx < kd) || rows_pad < rows || rows_pad % 8) {
    set_error("fase_ozaki_split: bad sizes (rows=%d kd=%d slices=%d kp=%lld rows_pad=%d)", rows,
              kd, slices, static_cast<long long>(kp), rows_pad);
    return FASE_ERR_SHAPE;
  }
  if (rows == 0) return FASE_OK;
  if (!x || !planes || !exps || !aligned16(planes)) {
    set_error("fase_ozaki_split: null or misaligned pointer");
    return FASE_ERR_SHAPE;
  }
  const dim3 grid(rows < 148 * 8 ? rows : 148 * 8);
  const int64_t stride = static_cast<int64_t>(rows_pad) * kp;
  const size_t smem = sizeof(double) * static_cast<size_t>(kp + kp / 16);
  auto run = [&](auto kern) -> cudaError_t {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    kern<<<grid, OZ_SPLIT_THREADS, smem, as_stream(stream)>>>(x, ldx, idx, w, rows, kd, planes,
                                                               kp, rows_pad, stride, exps);
    return cudaSuccess;
  };
  cudaError_t e = slices == 8 ? run(ozaki_split_kernel<8>)
                              : (slices == 7 ? run(ozaki_split_kernel<7>) : run(ozaki_split_kernel<6>));
  if (e != cudaSuccess) {
    set_error("fase_ozaki_split: cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    return FASE_ERR_CUDA;
  }
  return check_launch("fase_ozaki_split");
}

extern "C" int fase_ozaki_split_sparse(const int32_t* sel, int64_t ldsel, const double* coef,
                                       int64_t ldcoef, int rows, int iters, int kd, int slices,
                                       int8_t* planes, int64_t kp, int rows_pad, int32_t* exps,
                                       void* stream) {
  if (rows < 0 || iters < 0 || kd < 1 || slices < 6 || slices > OZ_MAX_SLICES || kp < kd ||
      kp % OZ_BK || kp > 16384 || ldsel < iters || ldcoef < iters || rows_pad < rows ||
      rows_pad % 8) {
    set_error("fase_ozaki_split_sparse: bad sizes (rows=%d iters=%d kd=%d slices=%d kp=%lld)",
              rows, iters, kd, slices, static_cast<long long>(kp));
    return FASE_ERR_SHAPE;
  }
  if (rows == 0) return FASE_OK;
  if ((iters > 0 && (!sel || !coef)) || !planes || !exps || !aligned16(planes)) {
    set_error("fase_ozaki_split_sparse: null or misaligned pointer");
    return FASE_ERR_SHAPE;
  }
  const dim3 grid(rows < 148 * 8 ? rows : 148 * 8);
  const int64_t stride = static_cast<int64_t>(rows_pad) * kp;
  const size_t smem = static_cast<size_t>(iters) * 12 + 16 + 4 * static_cast<size_t>(kp) +
                      4 * static_cast<size_t>((iters + 31) / 32);
  if (smem > 200 * 1024) {
    set_error("fase_ozaki_split_sparse: %d terms x %lld atoms exceed shared memory", iters,
              static_cast<long long>(kp));
    return FASE_ERR_SHAPE;
  }
  auto run = [&](auto kern) -> cudaError_t {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    kern<<<grid, OZ_SPLIT_THREADS, smem, as_stream(stream)>>>(sel, ldsel, coef, ldcoef, rows,
                                                               iters, kd, planes, kp, rows_pad,
                                                               stride, exps);
    return cudaSuccess;
  };
  cudaError_t e = slices == 8 ? run(ozaki_split_sparse_kernel<8>)
                              : (slices == 7 ? run(ozaki_split_sparse_kernel<7>)
                                             : run(ozaki_split_sparse_kernel<6>));
  if (e != cudaSuccess) {
    set_error("fase_ozaki_split_sparse: cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    return FASE_ERR_CUDA;
  }
  return check_launch("fase_ozaki_split_sparse");
}

static int ozaki_gemm_impl(const int8_t* a_planes, int a_rows_pad, const int32_t* ea, int m_rows,
                           const int8_t* b_planes, int b_rows_pad, const int32_t* eb, int n_rows,
                           int64_t kp, int slices, double* C, int64_t ldc, int sym, void* stream);

extern "C" int fase_ozaki_gemm(const int8_t* a_planes, int a_rows_pad, const int32_t* ea,
                               int m_rows, const int8_t* b_planes, int b_rows_pad,
                               const int32_t* eb, int n_rows, int64_t kp, int slices, double* C,
                               int64_t ldc, void* stream) {
  return ozaki_gemm_impl(a_planes, a_rows_pad, ea, m_rows, b_planes, b_rows_pad, eb, n_rows, kp,
                         slices, C, ldc, 0, stream);
}

extern "C" int fase_ozaki_gram(const int8_t* a_planes, int a_rows_pad, const int32_t* ea,
                               const int8_t* b_planes, int b_rows_pad, const int32_t* eb, int K,
                               int64_t kp, int slices, double* G, int64_t ldg, void* stream) {
  return ozaki_gemm_impl(a_planes, a_rows_pad, ea, K, b_planes, b_rows_pad, eb, K, kp, slices, G,
                         ldg, 1, stream);
}

static int ozaki_gemm_impl(const int8_t* a_planes, int a_rows_pad, const int32_t* ea, int m_rows,
                           const int8_t* b_planes, int b_rows_pad, const int32_t* eb, int n_rows,
                           int64_t kp, int slices, double* C, int64_t ldc, int sym, void* stream) {
  if (m_rows < 0 || n_rows < 0 || kp < OZ_BK || kp % OZ_BK || slices < 1 ||
      slices > OZ_MAX_SLICES || ldc < n_rows || kp > 16384) {  // int32 headroom, split smem
    set_error("fase_ozaki_gemm: bad sizes (M=%d N=%d kp=%lld slices=%d)", m_rows, n_rows,
              static_cast<long long>(kp), slices);
    return FASE_ERR_SHAPE;
  }
  if (m_rows == 0 || n_rows == 0) return FASE_OK;
  const int mt = (m_rows + OZ_BM - 1) / OZ_BM, nt = (n_rows + OZ_BN - 1) / OZ_BN;
  if (!a_planes || !b_planes || !ea || !eb || !C || a_rows_pad < mt * OZ_BM ||
      a_rows_pad % OZ_BM || b_rows_pad < nt * OZ_BN || b_rows_pad % OZ_BN ||
      !aligned16(a_planes) || !aligned16(b_planes)) {
    set_error("fase_ozaki_gemm: planes must hold rows padded to %d (A) / %d (B), 16-byte aligned",
              OZ_BM, OZ_BN);
    return FASE_ERR_SHAPE;
  }
  const int64_t a_plane = static_cast<int64_t>(a_rows_pad) * kp;
  const int64_t b_plane = static_cast<int64_t>(b_rows_pad) * kp;
  auto launch = [&](auto kern, int s) -> int {
    const size_t smem = static_cast<size_t>(OZ_STAGES) * s * (OZ_BM + OZ_BN) * OZ_BK;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) {
      set_error("fase_ozaki_gemm: cudaFuncSetAttribute: %s", cudaGetErrorString(e));
      return FASE_ERR_CUDA;
    }
    const char* env = getenv("FASE_OZAKI_GROUP_M");
    int group_m = env ? atoi(env) : 8;
    if (group_m < 1) group_m = 1;
    kern<<<nt * mt, OZ_THREADS, smem, as_stream(stream)>>>(a_planes, a_plane, ea, b_planes, b_plane,
                                                            eb, kp, m_rows, n_rows, a_rows_pad,
                                                            b_rows_pad, C, ldc, group_m, sym);
    return check_launch("fase_ozaki_gemm");
  };
  switch (slices) {
    case 8: return launch(ozaki_gemm_kernel<8>, 8);
    case 7: return launch(ozaki_gemm_kernel<7>, 7);
    case 6: return launch(ozaki_gemm_kernel<6>, 6);
    default:
      set_error("fase_ozaki_gemm: %d digit planes not instantiated (6-8)", slices);
      return FASE_ERR_UNSUPPORTED;
  }
}
