// The FaSE recursion: one persistent CTA per loss block.
//
// Reference: fase_extrapolate's loop (pkg/src/fase/fast.py:224-255) with the
// selection rule of pkg/src/fase/reference.py:55-85. Per iteration:
//
//   metric_k = |R_k| * D_k               (D_k == 0: never selectable)
//   q        = max(q, 1e-13 * max_k metric_k)        (tie quantum ratchet)
//   u        = lowest k with metric_k >= max - q
//   p        = R_u * (D_u * D_u);  c = gamma * p     (no division)
//   R_k     <- R_k - c * row_u[k]                     (mul, then sub: no FMA)
//
// Every operation is a single correctly rounded IEEE op in the same order as
// the reference's numpy code, so given the same R0 / table / D the selected
// sequence and coefficients are bit-identical.
//
// Layout: thread t owns the element pairs k = 2*(j*NT + t) + {0,1},
// j < EPT/2, so one table row is streamed with coalesced 16-byte loads (a
// warp reads 512 contiguous bytes per j). R and D stay in registers for the
// whole run; nothing but the table rows comes from memory inside the loop.
//
// Reductions: metric values are non-negative doubles, so their IEEE bit
// patterns order like int64; a dead atom is the key -1. The block max is two
// 32-bit redux.sync steps per warp plus one shared-memory exchange; the tie
// pass is a 32-bit redux.sync min over candidate indices, executed only by
// warps whose own max reaches the threshold (warp-uniform skip). Two
// __syncthreads per iteration.
//
// Per-block geometries: row_u = G0[u,:] - sum_{j in chunks(b)} C_j[u,:]
// (chunk tables of sample classes that are lost in some blocks and not in
// others). The subtraction order is the
// chunk-list order, identical to fase_block_normalizers' diagonal.

#include <climits>

#include "common.cuh"

namespace fase {
namespace {

constexpr unsigned kNone = 0xffffffffu;

__device__ __forceinline__ long long metric_key(double r, double d) {
  return d != 0.0 ? __double_as_longlong(mul_rn(fabs(r), d)) : -1LL;
}

template <int NT, int EPT, int MINB>
__global__ void __launch_bounds__(NT, MINB) fase_iterate_kernel(const fase_iterate_args a) {
  constexpr int EP = EPT / 2;
  constexpr int NW = NT / 32;
  __shared__ long long s_max[NW];
  __shared__ unsigned s_u[NW];
  __shared__ double s_r[NW];
  __shared__ double s_d[NW];

  const int b = blockIdx.x;
  const int t = threadIdx.x;
  const int lane = t & 31;
  const int warp = t >> 5;
  const int K = a.K;

  const double* D = a.D + (a.ldd ? static_cast<int64_t>(b) * a.ldd : 0);
  const double* R0 = a.R0 + static_cast<int64_t>(b) * a.ldr;
  const int32_t* cids = nullptr;
  int nch = 0;
  if (a.chunk_ptr) {
    const int lo = a.chunk_ptr[b];
    nch = a.chunk_ptr[b + 1] - lo;
    cids = a.chunk_ids + lo;
  }

  double r[EP][2], d[EP][2];
  long long lmax = -1;
#pragma unroll
  for (int j = 0; j < EP; ++j) {
    const int k = 2 * (j * NT + t);
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const bool in = k + e < K;
      r[j][e] = in ? R0[k + e] : 0.0;
      d[j][e] = in ? D[k + e] : 0.0;
      lmax = max(lmax, metric_key(r[j][e], d[j][e]));
    }
  }

  int32_t* sel = a.sel + static_cast<int64_t>(b) * a.ldo;
  double* proj = a.proj + static_cast<int64_t>(b) * a.ldo;
  double* coef = a.coef + static_cast<int64_t>(b) * a.ldo;
  double q = 0.0;

  for (int it = 0; it < a.I; ++it) {
    // ---- block max of the metric keys
    const long long wmax = warp_max_i64(lmax);
    if (lane == 0) s_max[warp] = wmax;
    __syncthreads();
    long long top_key = s_max[0];
#pragma unroll
    for (int w = 1; w < NW; ++w) top_key = max(top_key, s_max[w]);
    const double top = __longlong_as_double(top_key);
    // tie_quantum: only a finite, strictly positive top moves the ratchet
    if (top_key > 0 && top_key < 0x7ff0000000000000LL) q = fmax(q, mul_rn(1e-13, top));
    const double thr = q > 0.0 ? sub_rn(top, q) : top;

    // ---- lowest index reaching the threshold
    unsigned cand = kNone;
    double cr = 0.0, cd = 0.0;
    if (wmax >= 0 && __longlong_as_double(wmax) >= thr) {
#pragma unroll
      for (int j = 0; j < EP; ++j) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          if (cand == kNone && d[j][e] != 0.0 && mul_rn(fabs(r[j][e]), d[j][e]) >= thr) {
            cand = static_cast<unsigned>(2 * (j * NT + t) + e);
            cr = r[j][e];
            cd = d[j][e];
          }
        }
      }
    }
    const unsigned wmin = __reduce_min_sync(0xffffffffu, cand);
    if (wmin == kNone) {
      if (lane == 0) s_u[warp] = kNone;
    } else if (cand == wmin) {
      s_u[warp] = cand;
      s_r[warp] = cr;
      s_d[warp] = cd;
    }
    __syncthreads();
    unsigned u = s_u[0];
    int uw = 0;
#pragma unroll
    for (int w = 1; w < NW; ++w) {
      const unsigned v = s_u[w];
      if (v < u) {
        u = v;
        uw = w;
      }
    }
    const double ru = s_r[uw];
    const double du = s_d[uw];
    const double p = mul_rn(ru, mul_rn(du, du));
    const double c = mul_rn(a.gamma, p);
    if (t == 0) {
      sel[it] = static_cast<int32_t>(u);
      proj[it] = p;
      coef[it] = c;
    }

    // ---- stream row u (minus chunk rows) and apply the rank-1 update
    const double* row = a.G0 + static_cast<int64_t>(u) * a.ldg;
    double g[EP][2];
#pragma unroll
    for (int j = 0; j < EP; ++j) {
      const int k = 2 * (j * NT + t);
      if (k < K) {
        const double2 v = ldg2(row + k);
        g[j][0] = v.x;
        g[j][1] = v.y;
      } else {
        g[j][0] = g[j][1] = 0.0;
      }
    }
    for (int ch = 0; ch < nch; ++ch) {
      const double* crow = a.chunk_tables + static_cast<int64_t>(cids[ch]) * a.chunk_stride +
                           static_cast<int64_t>(u) * a.ldg;
#pragma unroll
      for (int j = 0; j < EP; ++j) {
        const int k = 2 * (j * NT + t);
        if (k < K) {
          const double2 v = ldg2(crow + k);
          g[j][0] = sub_rn(g[j][0], v.x);
          g[j][1] = sub_rn(g[j][1], v.y);
        }
      }
    }
    lmax = -1;
#pragma unroll
    for (int j = 0; j < EP; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        r[j][e] = sub_rn(r[j][e], mul_rn(c, g[j][e]));
        lmax = max(lmax, metric_key(r[j][e], d[j][e]));
      }
    }
    if (a.R_log) {
      double* dst = a.R_log + (static_cast<int64_t>(b) * a.I + it) * a.ldr;
#pragma unroll
      for (int j = 0; j < EP; ++j) {
        const int k = 2 * (j * NT + t);
        if (k < K) dst[k] = r[j][0];
        if (k + 1 < K) dst[k + 1] = r[j][1];
      }
    }
  }

  if (a.R_out) {
    double* dst = a.R_out + static_cast<int64_t>(b) * a.ldr;
#pragma unroll
    for (int j = 0; j < EP; ++j) {
      const int k = 2 * (j * NT + t);
      if (k < K) dst[k] = r[j][0];
      if (k + 1 < K) dst[k + 1] = r[j][1];
    }
  }
}

using KernelFn = void (*)(const fase_iterate_args);

struct Variant {
  int nt;
  int ept;
  KernelFn fn;
};

#define FASE_V(NT, EPT, MINB) {NT, EPT, fase_iterate_kernel<NT, EPT, MINB>}
// Ordered by capacity NT*EPT; the first variant that holds K is used. R and D
// live in registers (4 registers per owned atom), which caps K at 512 x 24.
const Variant kVariants[] = {
    FASE_V(128, 2, 4),   FASE_V(128, 4, 4),   FASE_V(128, 6, 4),   FASE_V(128, 8, 4),
    FASE_V(256, 6, 3),   FASE_V(256, 8, 3),   FASE_V(256, 10, 3),  FASE_V(256, 12, 2),
    FASE_V(256, 14, 2),  FASE_V(256, 16, 2),  FASE_V(256, 18, 2),  FASE_V(256, 20, 2),
    FASE_V(512, 12, 1),  FASE_V(512, 14, 1),  FASE_V(512, 16, 1),  FASE_V(512, 18, 1),
    FASE_V(512, 20, 1),  FASE_V(512, 24, 1),
};
#undef FASE_V

const Variant* pick_variant(int K) {
  for (const Variant& v : kVariants)
    if (v.nt * v.ept >= K) return &v;
  return nullptr;
}

}  // namespace
}  // namespace fase

using namespace fase;

extern "C" int fase_max_atoms(void) {
  const Variant& last = kVariants[sizeof(kVariants) / sizeof(kVariants[0]) - 1];
  return last.nt * last.ept;
}

extern "C" int fase_iterate(const fase_iterate_args* args, void* stream) {
  if (!args) {
    set_error("fase_iterate: null argument block");
    return FASE_ERR_PARAMETER;
  }
  const fase_iterate_args& a = *args;
  if (a.K < 1 || a.B < 0 || a.I < 1) {
    set_error("fase_iterate: bad sizes (K=%d, B=%d, I=%d)", a.K, a.B, a.I);
    return FASE_ERR_SHAPE;
  }
  if (!(a.gamma > 0.0 && a.gamma <= 1.0)) {
    set_error("fase_iterate: gamma must lie in (0, 1], got %g", a.gamma);
    return FASE_ERR_PARAMETER;
  }
  if (a.B == 0) return FASE_OK;
  if (!a.G0 || !aligned16(a.G0) || a.ldg < a.K || (a.ldg & 1) || !a.D || !a.R0 ||
      a.ldr < a.K || (a.ldd != 0 && a.ldd < a.K) || !a.sel || !a.proj || !a.coef || a.ldo < a.I) {
    set_error("fase_iterate: bad operand (null, misaligned, odd or short leading dimension)");
    return FASE_ERR_SHAPE;
  }
  if (a.chunk_ptr && (!a.chunk_ids || !a.chunk_tables || !aligned16(a.chunk_tables) ||
                      (a.chunk_stride & 1))) {
    set_error("fase_iterate: chunk tables given without ids / aligned storage");
    return FASE_ERR_SHAPE;
  }
  const Variant* v = pick_variant(a.K);
  if (!v) {
    set_error("fase_iterate: K=%d exceeds the largest kernel variant (%d atoms)", a.K,
              fase_max_atoms());
    return FASE_ERR_UNSUPPORTED;
  }
  v->fn<<<a.B, v->nt, 0, as_stream(stream)>>>(a);
  return check_launch("fase_iterate");
}
