// Frame concealment kernels: area extraction, per-block cell lists, paste.
//
// Reference per-tile path: pkg/src/fase/conceal.py:111-148 -- area = tile +-
// support, weight from every lost pixel in the area, FaSE, then only the
// tile's own lost pixels are written back. Here every lossy tile of a frame is
// one block of a batch; areas have a fixed size A = tile + 2*support and
// out-of-frame samples count as unavailable (BASELINE configs 2/3).
//
// Losses are whole tiles (macroblocks), described by a tile-level loss grid
// (Ty x Tx bytes); a pixel (y, x) is lost iff it lies in a full tile whose grid
// entry is set. Pixels past the last full tile row / column (e.g. the 8-row
// bottom strip of 1080p at 16-pixel tiles) are kept.

#include <algorithm>

#include "common.cuh"

namespace fase {
namespace {

struct FrameGeom {
  int H, W, tile, support, A, Ty, Tx;
};

// 1 = unavailable (outside the frame or lost), 0 = support sample
__device__ __forceinline__ int unavailable(const FrameGeom& g, const uint8_t* __restrict__ grid,
                                           int64_t ldgrid, int y, int x) {
  if (y < 0 || x < 0 || y >= g.H || x >= g.W) return 1;
  const int ty = y / g.tile, tx = x / g.tile;
  if (ty >= g.Ty || tx >= g.Tx) return 0;
  return grid[ty * ldgrid + tx] != 0;
}

// X[b, i*A + j] = frame(y, x) * base_w[i*A + j] on support samples, 0 elsewhere
// (the reference's s * w with s = 0 on lost pixels and w = 0 off support),
// y = r0 - support + i, x = c0 - support + j. One rounded multiply per sample.
__global__ void frame_areas_kernel(FrameGeom g, const double* __restrict__ frame, int64_t ldf,
                                   const uint8_t* __restrict__ grid, int64_t ldgrid,
                                   const int32_t* __restrict__ corners, int L,
                                   const double* __restrict__ base_w, double* __restrict__ X,
                                   int64_t ldx) {
  const int M = g.A * g.A;
  const int64_t total = static_cast<int64_t>(L) * M;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int b = static_cast<int>(idx / M);
    const int m = static_cast<int>(idx - static_cast<int64_t>(b) * M);
    const int i = m / g.A, j = m - (m / g.A) * g.A;
    FASE_ASSERT(corners[2 * b] >= 0 && corners[2 * b] < g.H && corners[2 * b + 1] >= 0 &&
                corners[2 * b + 1] < g.W);
    const int y = corners[2 * b] - g.support + i;
    const int x = corners[2 * b + 1] - g.support + j;
    double v = 0.0;
    if (!unavailable(g, grid, ldgrid, y, x)) v = mul_rn(frame[y * ldf + x], base_w[m]);
    X[b * ldx + m] = v;
  }
}

// counts[b] / ids[b, :] = the candidate cells (area rectangles, given by one
// representative sample each) that are unavailable for block b, in cell order.
__global__ void frame_cells_kernel(FrameGeom g, const uint8_t* __restrict__ grid, int64_t ldgrid,
                                   const int32_t* __restrict__ corners, int L,
                                   const int32_t* __restrict__ cell_rep, int n_cells,
                                   int32_t* __restrict__ counts, int32_t* __restrict__ ids,
                                   int64_t ids_ld) {
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < L; b += gridDim.x * blockDim.x) {
    const int y0 = corners[2 * b] - g.support, x0 = corners[2 * b + 1] - g.support;
    int n = 0;
    for (int c = 0; c < n_cells; ++c) {
      if (unavailable(g, grid, ldgrid, y0 + cell_rep[2 * c], x0 + cell_rep[2 * c + 1]))
        ids[b * ids_ld + n++] = c;
    }
    counts[b] = n;
  }
}

// g = sum_t coef_t * phi[sel_t, m] (selection order; SparseModel.materialize,
// reference.py:120-125) for the tile's own lost pixels, written into the frame
// (conceal.py:144-148).
constexpr int kPasteThreads = 256;
constexpr int kPasteChunk = 1024;

__global__ void __launch_bounds__(kPasteThreads) frame_paste_kernel(
    FrameGeom g, const double* __restrict__ phi, int64_t ldphi, const int32_t* __restrict__ sel,
    const double* __restrict__ coef, int64_t ldo, int I, const uint8_t* __restrict__ grid,
    int64_t ldgrid, const int32_t* __restrict__ corners, double* __restrict__ out, int64_t ldout) {
  __shared__ int32_t s_sel[kPasteChunk];
  __shared__ double s_coef[kPasteChunk];
  const int b = blockIdx.x;
  const int r0 = corners[2 * b], c0 = corners[2 * b + 1];
  FASE_ASSERT(r0 >= 0 && c0 >= 0 && r0 < g.H && c0 < g.W);
  const int n = g.tile * g.tile;
  const int32_t* my_sel = sel + static_cast<int64_t>(b) * ldo;
  const double* my_coef = coef + static_cast<int64_t>(b) * ldo;
  for (int base = 0; base < n; base += kPasteThreads) {
    const int p = base + threadIdx.x;
    const int i = p / g.tile, j = p - (p / g.tile) * g.tile;
    const bool mine = p < n && r0 + i < g.H && c0 + j < g.W &&
                      unavailable(g, grid, ldgrid, r0 + i, c0 + j);
    const int m = (g.support + i) * g.A + g.support + j;
    double acc = 0.0;
    for (int t0 = 0; t0 < I; t0 += kPasteChunk) {
      const int len = min(kPasteChunk, I - t0);
      __syncthreads();
      for (int t = threadIdx.x; t < len; t += kPasteThreads) {
        s_sel[t] = my_sel[t0 + t];
        s_coef[t] = my_coef[t0 + t];
      }
      __syncthreads();
      if (mine) acc = synth_terms(phi, ldphi, s_sel, s_coef, len, m, acc);
    }
    if (mine) out[static_cast<int64_t>(r0 + i) * ldout + c0 + j] = acc;
  }
}

// Complex dictionaries (conjugate-split rows phi2[2u] = Re phi_u, phi2[2u+1] =
// -Im phi_u; coef interleaved complex): g = sum_t coef_t * phi_{sel_t} with
// numpy's complex product, accumulated in selection order (reference.py:120-125,
// as synth_paste_complex); Re g is pasted (fast.py:282) and max |Im g| over the
// tile goes to max_imag[b] when given (apply_model's diagnostic).
__global__ void __launch_bounds__(kPasteThreads) frame_paste_complex_kernel(
    FrameGeom g, const double* __restrict__ phi2, int64_t ldphi, const int32_t* __restrict__ sel,
    const double* __restrict__ coef, int64_t ldo, int I, const uint8_t* __restrict__ grid,
    int64_t ldgrid, const int32_t* __restrict__ corners, double* __restrict__ out, int64_t ldout,
    double* __restrict__ max_imag) {
  __shared__ int32_t s_sel[kPasteChunk];
  __shared__ double2 s_coef[kPasteChunk];
  __shared__ double s_m[kPasteThreads / 32];
  const int b = blockIdx.x;
  const int r0 = corners[2 * b], c0 = corners[2 * b + 1];
  FASE_ASSERT(r0 >= 0 && c0 >= 0 && r0 < g.H && c0 < g.W);
  const int n = g.tile * g.tile;
  const int32_t* my_sel = sel + static_cast<int64_t>(b) * ldo;
  const double* my_coef = coef + 2 * static_cast<int64_t>(b) * ldo;
  double imax = 0.0;
  for (int base = 0; base < n; base += kPasteThreads) {
    const int p = base + threadIdx.x;
    const int i = p / g.tile, j = p - (p / g.tile) * g.tile;
    const bool mine = p < n && r0 + i < g.H && c0 + j < g.W &&
                      unavailable(g, grid, ldgrid, r0 + i, c0 + j);
    const int m = (g.support + i) * g.A + g.support + j;
    double gr = 0.0, gi = 0.0;
    bool done = false;
    for (int t0 = 0; t0 < I; t0 += kPasteChunk) {
      const int len = min(kPasteChunk, I - t0);
      __syncthreads();
      for (int t = threadIdx.x; t < len; t += kPasteThreads) {
        s_sel[t] = my_sel[t0 + t];
        s_coef[t] = make_double2(my_coef[2 * (t0 + t)], my_coef[2 * (t0 + t) + 1]);
      }
      __syncthreads();
      if (mine && !done) {
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
    if (mine) {
      out[static_cast<int64_t>(r0 + i) * ldout + c0 + j] = gr;
      imax = fmax(imax, fabs(gi));
    }
  }
  if (max_imag) {
    for (int o = 16; o > 0; o >>= 1) imax = fmax(imax, __shfl_xor_sync(0xffffffffu, imax, o));
    if ((threadIdx.x & 31) == 0) s_m[threadIdx.x >> 5] = imax;
    __syncthreads();
    if (threadIdx.x == 0) {
      double v = 0.0;
      for (int w = 0; w < kPasteThreads / 32; ++w) v = fmax(v, s_m[w]);
      max_imag[b] = v;
    }
  }
}

bool geom_ok(const FrameGeom& g) {
  return g.H > 0 && g.W > 0 && g.tile > 0 && g.support >= 0 && g.A == g.tile + 2 * g.support &&
         g.Ty == g.H / g.tile && g.Tx == g.W / g.tile;
}

}  // namespace
}  // namespace fase

using namespace fase;

extern "C" int fase_frame_areas(const double* frame, int64_t ldf, const uint8_t* grid,
                                int64_t ldgrid, int H, int W, int tile, int support,
                                const int32_t* corners, int L, const double* base_w, double* X,
                                int64_t ldx, void* stream) {
  const FrameGeom g{H, W, tile, support, tile + 2 * support, H / tile, W / tile};
  if (!geom_ok(g) || L < 0 || ldf < W || ldgrid < g.Tx || ldx < g.A * g.A) {
    set_error("fase_frame_areas: bad geometry (H=%d W=%d tile=%d support=%d)", H, W, tile, support);
    return FASE_ERR_SHAPE;
  }
  if (L == 0) return FASE_OK;
  if (!frame || !grid || !corners || !base_w || !X) {
    set_error("fase_frame_areas: null pointer");
    return FASE_ERR_SHAPE;
  }
  const int64_t total = static_cast<int64_t>(L) * g.A * g.A;
  const int64_t blocks = (total + 255) / 256;
  frame_areas_kernel<<<static_cast<unsigned>(blocks < 148 * 32 ? blocks : 148 * 32), 256, 0,
                       as_stream(stream)>>>(g, frame, ldf, grid, ldgrid, corners, L, base_w, X,
                                            ldx);
  return check_launch("fase_frame_areas");
}

extern "C" int fase_frame_cells(const uint8_t* grid, int64_t ldgrid, int H, int W, int tile,
                                int support, const int32_t* corners, int L,
                                const int32_t* cell_rep, int n_cells, int32_t* counts,
                                int32_t* ids, int64_t ids_ld, void* stream) {
  const FrameGeom g{H, W, tile, support, tile + 2 * support, H / tile, W / tile};
  if (!geom_ok(g) || L < 0 || n_cells < 0 || ids_ld < (n_cells > 0 ? n_cells : 1) ||
      ldgrid < g.Tx) {
    set_error("fase_frame_cells: bad geometry or list stride");
    return FASE_ERR_SHAPE;
  }
  if (L == 0) return FASE_OK;
  if (!grid || !corners || !counts || !ids || (n_cells && !cell_rep)) {
    set_error("fase_frame_cells: null pointer");
    return FASE_ERR_SHAPE;
  }
  frame_cells_kernel<<<(L + 255) / 256, 256, 0, as_stream(stream)>>>(
      g, grid, ldgrid, corners, L, cell_rep, n_cells, counts, ids, ids_ld);
  return check_launch("fase_frame_cells");
}

extern "C" int fase_frame_paste(const double* phi, int64_t ldphi, const int32_t* sel,
                                const double* coef, int64_t ldo, int I, const uint8_t* grid,
                                int64_t ldgrid, int H, int W, int tile, int support,
                                const int32_t* corners, int L, double* out, int64_t ldout,
                                void* stream) {
  const FrameGeom g{H, W, tile, support, tile + 2 * support, H / tile, W / tile};
  if (!geom_ok(g) || L < 0 || I < 1 || ldo < I || ldout < W || ldgrid < g.Tx) {
    set_error("fase_frame_paste: bad geometry or sizes");
    return FASE_ERR_SHAPE;
  }
  if (L == 0) return FASE_OK;
  if (!phi || !sel || !coef || !grid || !corners || !out) {
    set_error("fase_frame_paste: null pointer");
    return FASE_ERR_SHAPE;
  }
  frame_paste_kernel<<<L, kPasteThreads, 0, as_stream(stream)>>>(
      g, phi, ldphi, sel, coef, ldo, I, grid, ldgrid, corners, out, ldout);
  return check_launch("fase_frame_paste");
}

namespace fase {
namespace {
// frame_widen: out = lost ? 0 : double(u8), 8 pixels per thread (8-byte loads of
// the uint8 frame and the loss mask, four 16-byte stores)
__global__ void __launch_bounds__(256) frame_widen_kernel(const uint8_t* __restrict__ u8, int64_t ldu,
                                                          const uint8_t* __restrict__ lost,
                                                          int64_t ldl, int H, int W,
                                                          double* __restrict__ out, int64_t ldo) {
  const int per_row = (W + 7) / 8;
  const int64_t total = static_cast<int64_t>(H) * per_row;
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int y = static_cast<int>(idx / per_row);
    const int x0 = static_cast<int>(idx - static_cast<int64_t>(y) * per_row) * 8;
    const uint8_t* src = u8 + y * ldu + x0;
    const uint8_t* lm = lost + y * ldl + x0;
    double* dst = out + y * ldo + x0;
    const bool vec = x0 + 8 <= W && aligned16(dst) && (reinterpret_cast<uintptr_t>(src) & 7u) == 0 &&
                     (reinterpret_cast<uintptr_t>(lm) & 7u) == 0;
    if (vec) {
      const uint2 pv = *reinterpret_cast<const uint2*>(src);
      const uint2 lv = *reinterpret_cast<const uint2*>(lm);
      double v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const unsigned pw = i < 4 ? pv.x : pv.y, lw = i < 4 ? lv.x : lv.y;
        const unsigned sh = 8u * (i & 3);
        v[i] = ((lw >> sh) & 0xffu) ? 0.0 : static_cast<double>((pw >> sh) & 0xffu);
      }
#pragma unroll
      for (int i = 0; i < 8; i += 2) *reinterpret_cast<double2*>(dst + i) = make_double2(v[i], v[i + 1]);
    } else {
      for (int i = 0; i < 8 && x0 + i < W; ++i) dst[i] = lm[i] ? 0.0 : static_cast<double>(src[i]);
    }
  }
}
}  // namespace
}  // namespace fase

extern "C" int fase_frame_paste_complex(const double* phi2, int64_t ldphi, const int32_t* sel,
                                        const double* coef, int64_t ldo, int I,
                                        const uint8_t* grid, int64_t ldgrid, int H, int W,
                                        int tile, int support, const int32_t* corners, int L,
                                        double* out, int64_t ldout, double* max_imag,
                                        void* stream) {
  const FrameGeom g{H, W, tile, support, tile + 2 * support, H / tile, W / tile};
  if (!geom_ok(g) || L < 0 || I < 1 || ldo < I || ldout < W || ldgrid < g.Tx) {
    set_error("fase_frame_paste_complex: bad geometry or sizes");
    return FASE_ERR_SHAPE;
  }
  if (L == 0) return FASE_OK;
  if (!phi2 || !sel || !coef || !grid || !corners || !out) {
    set_error("fase_frame_paste_complex: null pointer");
    return FASE_ERR_SHAPE;
  }
  frame_paste_complex_kernel<<<L, kPasteThreads, 0, as_stream(stream)>>>(
      g, phi2, ldphi, sel, coef, ldo, I, grid, ldgrid, corners, out, ldout, max_imag);
  return check_launch("fase_frame_paste_complex");
}

namespace fase {
namespace {
// Dispatch order of a chunked recursion (longest processing time first): the
// blocks by descending cost class, stable. One CTA: each thread counts the
// classes of a contiguous range of blocks, a scan per class (descending) over
// the threads gives every (class, thread) its first output slot, and each
// thread writes its range again in index order.
constexpr int kOrderThreads = 1024, kOrderClasses = 8;
__global__ void __launch_bounds__(kOrderThreads) block_order_kernel(const int32_t* __restrict__ counts,
                                                                    int B, int depth,
                                                                    int32_t* __restrict__ order) {
  __shared__ int s_hist[kOrderClasses][kOrderThreads];
  __shared__ int s_tot[kOrderClasses];
  __shared__ int s_warp[kOrderThreads / 32];
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int per = (B + kOrderThreads - 1) / kOrderThreads;
  const int lo = min(B, t * per), hi = min(B, lo + per);
  auto cls = [&](int b) {
    const int r = counts[b] - depth;
    return r <= 0 ? 0 : (r >= kOrderClasses - 1 ? kOrderClasses - 1 : r);
  };
  int h[kOrderClasses];
#pragma unroll
  for (int c = 0; c < kOrderClasses; ++c) h[c] = 0;
  for (int b = lo; b < hi; ++b) {
    const int c = cls(b);
#pragma unroll
    for (int k = 0; k < kOrderClasses; ++k) h[k] += (k == c);
  }
  // exclusive scan over threads, one class at a time (descending classes first)
  int base = 0;
  for (int c = kOrderClasses - 1; c >= 0; --c) {
    int v = h[c];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int n = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += n;
    }
    if (lane == 31) s_warp[warp] = v;
    __syncthreads();
    if (warp == 0) {
      int w = s_warp[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int n = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += n;
      }
      s_warp[lane] = w;  // inclusive over warps
      if (lane == 31) s_tot[c] = w;
    }
    __syncthreads();
    const int before = (warp > 0 ? s_warp[warp - 1] : 0) + v - h[c];
    s_hist[c][t] = base + before;
    base += s_tot[c];
    __syncthreads();
  }
  int pos[kOrderClasses];
#pragma unroll
  for (int c = 0; c < kOrderClasses; ++c) pos[c] = s_hist[c][t];
  for (int b = lo; b < hi; ++b) {
    const int c = cls(b);
#pragma unroll
    for (int k = 0; k < kOrderClasses; ++k)
      if (k == c) order[pos[k]++] = b;
  }
}
}  // namespace
}  // namespace fase

extern "C" int fase_block_order(const int32_t* counts, int B, int depth, int32_t* order,
                                void* stream) {
  if (B < 0 || depth < 0) {
    set_error("fase_block_order: bad sizes (B=%d, depth=%d)", B, depth);
    return FASE_ERR_SHAPE;
  }
  if (B == 0) return FASE_OK;
  if (!counts || !order) {
    set_error("fase_block_order: null pointer");
    return FASE_ERR_SHAPE;
  }
  fase::block_order_kernel<<<1, fase::kOrderThreads, 0, as_stream(stream)>>>(counts, B, depth,
                                                                             order);
  return check_launch("fase_block_order");
}

extern "C" int fase_frame_widen(const uint8_t* frame_u8, int64_t ldu, const uint8_t* lost,
                                int64_t ldl, int H, int W, double* out, int64_t ldout,
                                void* stream) {
  if (H < 0 || W < 0 || ldu < W || ldl < W || ldout < W) {
    set_error("fase_frame_widen: bad sizes");
    return FASE_ERR_SHAPE;
  }
  if (H == 0 || W == 0) return FASE_OK;
  if (!frame_u8 || !lost || !out) {
    set_error("fase_frame_widen: null pointer");
    return FASE_ERR_SHAPE;
  }
  const int64_t work = static_cast<int64_t>(H) * ((W + 7) / 8);
  const int blocks = static_cast<int>(std::min<int64_t>((work + 255) / 256, 148 * 16));
  frame_widen_kernel<<<blocks, 256, 0, as_stream(stream)>>>(frame_u8, ldu, lost, ldl, H, W, out,
                                                           ldout);
  return check_launch("fase_frame_widen");
}
