// The FaSE recursion for dictionaries larger than the register-resident
// kernels hold (K > fase_iterate_register_atoms(), real tables): R streams
// through global memory instead of living in registers.
//
// Reference: fase_extrapolate's loop (pkg/src/fase/fast.py:238-255) with the
// tie rule of pkg/src/fase/reference.py:55-85, the same arithmetic as
// csrc/iterate.cu (one correctly rounded IEEE operation at a time, numpy's
// order), so selections, projections and coefficients are bit-identical to
// the register kernels and to the reference given the same R0 / table / D.
//
// One 1024-thread CTA per block. The working vector R is the caller's R_out
// (B x ldr, written with R0 first). Per iteration, thread t visits k = t,
// t + 1024, ... once: it applies the previous iteration's update
//   R_k <- R_k - c * row_u[k],  row_u = base[u] - sum of the block's chunk rows
// and folds |R_k| * D_k into its running max (lowest index on equal maxima).
// The block max and its lowest index come from the same three-step redux
// exchange as the register kernels; the tie pass re-reads R and D only in
// threads whose own max reaches the threshold. Bound: latency of the global
// passes (R read + write, D and the row per element): this is the capability
// path for large K, not the tuned one.

#include <climits>
#include <cstdlib>

#include "common.cuh"

namespace fase {
namespace {

constexpr int kGenThreads = 1024;
constexpr int kGenWarps = kGenThreads / 32;
constexpr unsigned kGenNone = 0xffffffffu;

__global__ void __launch_bounds__(kGenThreads, 1) fase_iterate_generic_kernel(const fase_iterate_args a) {
  __shared__ long long s_key[kGenWarps];
  __shared__ unsigned s_arg[kGenWarps];
  __shared__ unsigned s_u[kGenWarps];
  const int slot = static_cast<int>(blockIdx.x);
  const int b = a.order ? __ldg(a.order + slot) : slot;
  const int t = static_cast<int>(threadIdx.x), lane = t & 31, warp = t >> 5;
  const int K = a.K;
  const double kDead = __longlong_as_double(static_cast<long long>(0xfff0000000000000ULL));
  const double* D = a.D + (a.ldd ? static_cast<int64_t>(b) * a.ldd : 0);
  const double* R0 = a.R0 + static_cast<int64_t>(b) * a.ldr;
  double* R = a.R_out + static_cast<int64_t>(b) * a.ldr;
  int32_t* sel = a.sel + static_cast<int64_t>(b) * a.ldo;
  double* proj = a.proj + static_cast<int64_t>(b) * a.ldo;
  double* coef = a.coef + static_cast<int64_t>(b) * a.ldo;
  const int64_t ldg = a.ldg;

  // this block's base table and remaining chunk list (as csrc/iterate.cu)
  const int32_t* cids = nullptr;
  int nch = 0;
  const double* G0b = a.G0;
  if (a.chunk_count) {
    nch = a.chunk_count[b];
    cids = a.chunk_ids + static_cast<int64_t>(b) * a.chunk_list_ld;
    if (a.compose && nch > 0) {
      for (int k = min(nch, a.compose_depth); k >= 1; --k) {
        int64_t idx = 0;
        for (int d = 0; d < a.compose_depth; ++d) {
          FASE_ASSERT(cids[min(d, k - 1)] >= 0 && cids[min(d, k - 1)] < a.n_compose);
          idx = idx * a.n_compose + cids[min(d, k - 1)];
        }
        const int p = a.compose[idx];
        if (p > 0) {
          G0b += static_cast<int64_t>(p) * a.base_stride;
          cids += k;
          nch -= k;
          break;
        }
      }
    }
  }
  auto dval = [&](int k) {
    const double d = __ldg(D + k);
    return d != 0.0 ? d : kDead;
  };

  // the block-wide max of the threads' (best, barg): redux per warp, one
  // shared exchange, every warp reduces the slots
  auto block_max = [&](double best, unsigned barg, long long& top_key, unsigned& top_arg) {
    const long long key = __double_as_longlong(best);
    const int kh = static_cast<int>(key >> 32);
    const unsigned kl = static_cast<unsigned>(key);
    const int wh = __reduce_max_sync(0xffffffffu, kh);
    const unsigned wl = __reduce_max_sync(0xffffffffu, kh == wh ? kl : 0u);
    const unsigned wa = __reduce_min_sync(0xffffffffu, (kh == wh && kl == wl) ? barg : kGenNone);
    if (lane == 0) {
      s_key[warp] = (static_cast<long long>(wh) << 32) | wl;
      s_arg[warp] = wa;
    }
    __syncthreads();
    const long long sk = s_key[lane];
    const unsigned sa = s_arg[lane];
    const int h = static_cast<int>(sk >> 32);
    const unsigned l = static_cast<unsigned>(sk);
    const int bh = __reduce_max_sync(0xffffffffu, h);
    const unsigned bl = __reduce_max_sync(0xffffffffu, h == bh ? l : 0u);
    top_arg = __reduce_min_sync(0xffffffffu, (h == bh && l == bl) ? sa : kGenNone);
    top_key = (static_cast<long long>(bh) << 32) | bl;
  };

  // iteration 0's metrics from R0 (R <- R0)
  double best = kDead;
  unsigned barg = kGenNone;
  for (int k = t; k < K; k += kGenThreads) {
    const double r = R0[k];
    R[k] = r;
    const double m = mul_rn(fabs(r), dval(k));
    if (m > best) {
      best = m;
      barg = static_cast<unsigned>(k);
    }
  }
  double q = 0.0;
  for (int it = 0; it < a.I; ++it) {
    long long top_key;
    unsigned top_arg;
    block_max(best, barg, top_key, top_arg);
    if (top_key < 0) {  // every atom degenerate (NoSelectableAtomError): mark and stop
      for (int k = it + t; k < a.I; k += kGenThreads) {
        sel[k] = -1;
        proj[k] = 0.0;
        coef[k] = 0.0;
      }
      return;
    }
    const double top = __longlong_as_double(top_key);
    {  // the ratchet; a +0 top leaves it (1e-13 * 0), a +inf one must not move it
      const double qn = mul_rn(1e-13, top);
      q = qn < __longlong_as_double(0x7ff0000000000000LL) ? fmax(q, qn) : q;
    }
    const double thr = sub_rn(top, q);  // (q == 0: exactly top)
    // lowest index reaching the threshold: only threads whose max reaches it
    unsigned cand = kGenNone;
    if (best >= thr) {
      for (int k = t; k < K && cand == kGenNone; k += kGenThreads)
        if (mul_rn(fabs(R[k]), dval(k)) >= thr) cand = static_cast<unsigned>(k);
    }
    const unsigned wmin = __reduce_min_sync(0xffffffffu, cand);
    if (lane == 0) s_u[warp] = wmin;
    __syncthreads();
    const unsigned u = __reduce_min_sync(0xffffffffu, s_u[lane]);
    FASE_ASSERT(u < static_cast<unsigned>(K));
    const double ru = R[u];
    const double du = __ldg(D + u);
    const double p = mul_rn(ru, mul_rn(du, du));
    const double c = mul_rn(a.gamma, p);
    if (t == 0) {
      sel[it] = static_cast<int32_t>(u);
      proj[it] = p;
      coef[it] = c;
    }
    __syncthreads();  // every thread has read R[u] and s_u before R and the slots change
    // R <- R - c * row_u, fused with the next iteration's running max
    const double* grow = G0b + static_cast<int64_t>(u) * ldg;
    best = kDead;
    barg = kGenNone;
    for (int k = t; k < K; k += kGenThreads) {
      double g = __ldg(grow + k);
      for (int ch = 0; ch < nch; ++ch)
        g = sub_rn(g, __ldg(a.chunk_tables + static_cast<int64_t>(cids[ch]) * a.chunk_stride +
                            static_cast<int64_t>(u) * ldg + k));
      const double r = sub_rn(R[k], mul_rn(c, g));
      R[k] = r;
      const double m = mul_rn(fabs(r), dval(k));
      if (m > best) {
        best = m;
        barg = static_cast<unsigned>(k);
      }
    }
  }
}

// Complex tables (rows of conj(C), csrc/iterate_complex.cu's arithmetic: numpy's
// complex product and hypot, one rounding at a time): the same streaming loop
// with R complex (interleaved) in R_out and the exact metric |R| * D per element.
__global__ void __launch_bounds__(kGenThreads, 1) fase_iterate_generic_complex_kernel(const fase_iterate_args a) {
  __shared__ long long s_key[kGenWarps];
  __shared__ unsigned s_arg[kGenWarps];
  __shared__ unsigned s_u[kGenWarps];
  const int slot = static_cast<int>(blockIdx.x);
  const int b = a.order ? __ldg(a.order + slot) : slot;
  const int t = static_cast<int>(threadIdx.x), lane = t & 31, warp = t >> 5;
  const int K = a.K;
  const double kDead = __longlong_as_double(static_cast<long long>(0xfff0000000000000ULL));
  const double* D = a.D + (a.ldd ? static_cast<int64_t>(b) * a.ldd : 0);
  const double2* R0 = reinterpret_cast<const double2*>(a.R0) + static_cast<int64_t>(b) * a.ldr;
  double2* R = reinterpret_cast<double2*>(a.R_out) + static_cast<int64_t>(b) * a.ldr;
  int32_t* sel = a.sel + static_cast<int64_t>(b) * a.ldo;
  double* proj = a.proj + 2 * static_cast<int64_t>(b) * a.ldo;
  double* coef = a.coef + 2 * static_cast<int64_t>(b) * a.ldo;
  const int64_t ldg = a.ldg;  // complex elements
  const double2* C = reinterpret_cast<const double2*>(a.chunk_tables);

  const int32_t* cids = nullptr;
  int nch = 0;
  const double2* G0b = reinterpret_cast<const double2*>(a.G0);
  if (a.chunk_count) {
    nch = a.chunk_count[b];
    cids = a.chunk_ids + static_cast<int64_t>(b) * a.chunk_list_ld;
    if (a.compose && nch > 0) {
      for (int k = min(nch, a.compose_depth); k >= 1; --k) {
        int64_t idx = 0;
        for (int d = 0; d < a.compose_depth; ++d) {
          FASE_ASSERT(cids[min(d, k - 1)] >= 0 && cids[min(d, k - 1)] < a.n_compose);
          idx = idx * a.n_compose + cids[min(d, k - 1)];
        }
        const int p = a.compose[idx];
        if (p > 0) {
          G0b += static_cast<int64_t>(p) * a.base_stride;
          cids += k;
          nch -= k;
          break;
        }
      }
    }
  }
  auto metric = [&](double2 r, int k) {
    const double d = __ldg(D + k);
    return mul_rn(np_cabs_fast(r.x, r.y), d != 0.0 ? d : kDead);
  };
  auto block_max = [&](double best, unsigned barg, long long& top_key) {
    const long long key = __double_as_longlong(best);
    const int kh = static_cast<int>(key >> 32);
    const unsigned kl = static_cast<unsigned>(key);
    const int wh = __reduce_max_sync(0xffffffffu, kh);
    const unsigned wl = __reduce_max_sync(0xffffffffu, kh == wh ? kl : 0u);
    if (lane == 0) s_key[warp] = (static_cast<long long>(wh) << 32) | wl;
    __syncthreads();
    const long long sk = s_key[lane];
    const int h = static_cast<int>(sk >> 32);
    const unsigned l = static_cast<unsigned>(sk);
    const int bh = __reduce_max_sync(0xffffffffu, h);
    const unsigned bl = __reduce_max_sync(0xffffffffu, h == bh ? l : 0u);
    top_key = (static_cast<long long>(bh) << 32) | bl;
  };

  double best = kDead;
  unsigned barg = kGenNone;
  for (int k = t; k < K; k += kGenThreads) {
    const double2 r = R0[k];
    R[k] = r;
    const double m = metric(r, k);
    if (m > best) {
      best = m;
      barg = static_cast<unsigned>(k);
    }
  }
  double q = 0.0;
  for (int it = 0; it < a.I; ++it) {
    long long top_key;
    block_max(best, barg, top_key);
    if (top_key < 0) {  // every atom degenerate: mark and stop
      for (int k = it + t; k < a.I; k += kGenThreads) {
        sel[k] = -1;
        proj[2 * k] = proj[2 * k + 1] = 0.0;
        coef[2 * k] = coef[2 * k + 1] = 0.0;
      }
      return;
    }
    const double top = __longlong_as_double(top_key);
    {  // the ratchet; a +0 top leaves it (1e-13 * 0), a +inf one must not move it
      const double qn = mul_rn(1e-13, top);
      q = qn < __longlong_as_double(0x7ff0000000000000LL) ? fmax(q, qn) : q;
    }
    const double thr = sub_rn(top, q);  // (q == 0: exactly top)
    unsigned cand = kGenNone;
    if (best >= thr) {
      for (int k = t; k < K && cand == kGenNone; k += kGenThreads)
        if (metric(R[k], k) >= thr) cand = static_cast<unsigned>(k);
    }
    const unsigned wmin = __reduce_min_sync(0xffffffffu, cand);
    if (lane == 0) s_u[warp] = wmin;
    __syncthreads();
    const unsigned u = __reduce_min_sync(0xffffffffu, s_u[lane]);
    FASE_ASSERT(u < static_cast<unsigned>(K));
    const double2 ru = R[u];
    const double du = __ldg(D + u);
    const double d2u = mul_rn(du, du);
    const double pr = mul_rn(ru.x, d2u), pi = mul_rn(ru.y, d2u);
    const double cr = mul_rn(a.gamma, pr), ci = mul_rn(a.gamma, pi);
    if (t == 0) {
      sel[it] = static_cast<int32_t>(u);
      proj[2 * it] = pr;
      proj[2 * it + 1] = pi;
      coef[2 * it] = cr;
      coef[2 * it + 1] = ci;
    }
    __syncthreads();
    const double2* grow = G0b + static_cast<int64_t>(u) * ldg;
    best = kDead;
    barg = kGenNone;
    for (int k = t; k < K; k += kGenThreads) {
      double2 g = grow[k];
      for (int ch = 0; ch < nch; ++ch) {
        const double2 v = C[static_cast<int64_t>(cids[ch]) * a.chunk_stride +
                            static_cast<int64_t>(u) * ldg + k];
        g.x = sub_rn(g.x, v.x);
        g.y = sub_rn(g.y, v.y);
      }
      const double2 x = np_cmul(cr, ci, g.x, g.y);
      double2 r = R[k];
      r.x = sub_rn(r.x, x.x);
      r.y = sub_rn(r.y, x.y);
      R[k] = r;
      const double m = metric(r, k);
      if (m > best) {
        best = m;
        barg = static_cast<unsigned>(k);
      }
    }
  }
}

}  // namespace

// the register-resident kernels' capacity (csrc/iterate.cu)
int iterate_register_atoms();

int launch_iterate_generic_complex(const fase_iterate_args& a, int reg_atoms, cudaStream_t stream) {
  if (!a.R_out || a.R_log) {
    set_error("fase_iterate_complex: K=%d exceeds the register kernels' %d atoms: the streaming "
              "recursion needs R_out (B x ldr, may alias R0) as its working vector and takes "
              "no R_log", a.K, reg_atoms);
    return a.R_log ? FASE_ERR_UNSUPPORTED : FASE_ERR_SHAPE;
  }
  fase_iterate_generic_complex_kernel<<<a.B, kGenThreads, 0, stream>>>(a);
  return check_launch("fase_iterate_complex (streaming, large K)");
}

int launch_iterate_generic(const fase_iterate_args& a, cudaStream_t stream) {
  if (!a.R_out || a.R_log) {
    set_error("fase_iterate: K=%d exceeds the register kernels' %d atoms: the streaming "
              "recursion needs R_out (B x ldr, may alias R0) as its working vector and takes "
              "no R_log", a.K, iterate_register_atoms());
    return a.R_log ? FASE_ERR_UNSUPPORTED : FASE_ERR_SHAPE;
  }
  fase_iterate_generic_kernel<<<a.B, kGenThreads, 0, stream>>>(a);
  return check_launch("fase_iterate (streaming, large K)");
}

}  // namespace fase
