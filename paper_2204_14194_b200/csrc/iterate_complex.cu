// The FaSE recursion for complex-valued dictionaries (dft, bdft, their unions,
// complex file dictionaries): one persistent CTA per loss block.
//
// Reference: the same loop as the real kernel (fast.py:224-255, selection
// reference.py:55-85) in complex128:
//
//   metric_k = |R_k| * D_k                  np.abs: hypot as numpy evaluates it
//   q        = max(q, 1e-13 * max metric);  u = lowest k with metric_k >= max - q
//   p        = R_u * (D_u * D_u);  c = gamma * p
//   R_k     <- R_k - c * conj(C[u, k])       numpy's fused complex multiply
//
// The table handed in stores conj(C[u, :]) row by row (fase_gram_complex), so
// the update streams one 16-byte complex per element. Every operation is the
// one numpy performs (common.cuh: np_cmul, np_cabs), so given the same R0,
// table and D the run is bit-identical to the reference.
//
// Selection without a hypot per element and iteration: the update pass keeps a
// cheap proxy P_k = (re^2 + im^2) * D_k^2 and its running max. The exact metric
// differs from sqrt(P_k) by a few ulp (<= 8 * 2^-53 relative), so only elements
// with P_k above a conservative bound of the threshold (margins 2^-40) can be
// the maximum or reach the threshold. Those candidates (normally the predicted
// atom plus its structural twins, e.g. a conjugate-frequency partner) get the
// exact metric and land in a short shared list; after the second barrier every
// warp resolves the list redundantly (exact max, tie quantum, lowest index), so
// an iteration still has two barriers. A single candidate is the selection
// outright; its exact metric is needed only while the tie quantum can move. An overflowing list, or proxies too
// small / large to trust, fall back to an exact pass over all elements.
//
// Layout: thread t owns complex elements k = j*NT + t, j < EP (R in registers,
// D^2 in shared memory or registers; D itself only for exact metrics, from
// global memory), so a table row streams with
// coalesced 16-byte loads; the predicted row is staged by TMA as in the real
// kernel, and per-block geometries compose rows G0[u] - sum C_j[u] the same way.
// Leading dimensions (ldg, ldr, ldo, chunk_stride) count complex elements.

#include <climits>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"

namespace fase {
namespace {

constexpr unsigned kNone = 0xffffffffu;
constexpr int kCap = 64;  // candidate list capacity
// scaled recursion: the update as fused multiply-adds (measurement knob)
#ifndef FASE_CSCALED_FMA
#define FASE_CSCALED_FMA 1
#endif

// NB == 2 (shared geometry, D^2 in shared memory): one CTA runs two blocks on
// its two NT-thread halves (own staged row, candidate list, named barriers)
// that share one copy of D^2, as in the real kernel's paired variants.
//
// kScaled (fase_iterate_complex_scaled, shared geometry): as the real scaled
// recursion -- the table rows are column-scaled, conj(C)[u, k] * D_k, and the
// state is R'_k = R_k * D_k, so the proxy is |R'|^2 and the exact metric
// |R'| (np.abs of the scaled value) with no normalizers in the loop;
// p = R'_u * D_u. Dead atoms hold NaN. Selections match the exact kernel up
// to ties within the rounding of the scaled operands.
template <int NT, int EP, int MINB, bool kDsmem, bool kChunked, bool kRecord, int NB,
          bool kScaled = false>
__global__ void __launch_bounds__(NT * NB, MINB) fase_iterate_complex_kernel(const fase_iterate_args a) {
  constexpr int NW = NT / 32;
  constexpr int kSeg = EP < 3 ? EP : 3;
  static_assert(NB == 1 || (kDsmem && !kChunked), "paired blocks share one D^2 in shared memory");
  static_assert(!kScaled || (!kDsmem && !kChunked && !kRecord && NB == 1),
                "the scaled recursion keeps no normalizers and has one block per CTA");

  __shared__ long long s_key_all[NB][NW];
  __shared__ unsigned s_arg_all[NB][NW];
  __shared__ int s_cnt_all[NB][2];
  __shared__ double s_cm_all[NB][kCap];            // candidate exact metric
  __shared__ unsigned s_ck_all[NB][kCap];          // candidate index
  __shared__ __align__(16) double2 s_cr_all[NB][kCap];  // candidate R
  __shared__ double s_cd_all[NB][kCap];            // candidate D
  __shared__ __align__(8) uint64_t s_bar_all[NB][kSeg];
  extern __shared__ double2 s_dyn[];

  const int half = NB == 1 ? 0 : static_cast<int>(threadIdx.x) / NT;
  long long* s_key = s_key_all[half];
  unsigned* s_arg = s_arg_all[half];
  int* s_cnt = s_cnt_all[half];
  double* s_cm = s_cm_all[half];
  unsigned* s_ck = s_ck_all[half];
  double2* s_cr = s_cr_all[half];
  double* s_cd = s_cd_all[half];
  uint64_t* s_bar = s_bar_all[half];
  double2* s_row = s_dyn + half * EP * NT;  // staged row: element j*NT + t
  double* s_D2 = reinterpret_cast<double*>(s_dyn + NB * EP * NT);  // kDsmem: D^2 per element

  // the block of this CTA slot: slot order, or (per-block geometries) the
  // caller's dispatch order (shared geometries ignore it: equal-cost blocks, and
  // a loaded block index costs a register, csrc/iterate.cu)
  const int slot = static_cast<int>(blockIdx.x) * NB + half;
  const int b = (kChunked && a.order && slot < a.B) ? __ldg(a.order + slot) : slot;
  const int t = static_cast<int>(threadIdx.x) - half * NT;
  const int lane = t & 31;
  const int warp = t >> 5;
  const int K = a.K;
  const double kDead = __longlong_as_double(static_cast<long long>(0xfff0000000000000ULL));
  const bool active = NB == 1 || slot < a.B;
  auto block_sync = [&]() {  // the whole CTA, or this block's half
    if constexpr (NB == 1)
      __syncthreads();
    else
      asm volatile("bar.sync %0, %1;\n" ::"r"(1 + half), "r"(NT) : "memory");
  };

  if (t == 0) {
    for (int sg = 0; sg < kSeg; ++sg) mbar_init(&s_bar[sg], 1);
    fence_mbar_init();
    s_cnt[0] = 0;
    s_cnt[1] = 0;
  }

  const double* D = a.D + (a.ldd ? static_cast<int64_t>(b) * a.ldd : 0);
  const double* R0 = a.R0 + 2 * static_cast<int64_t>(active ? b : 0) * a.ldr;
  const int32_t* cids = nullptr;
  int nch = 0;
  const double* G0 = a.G0;  // this block's base table
  if (kChunked) {
    nch = a.chunk_count[b];
    cids = a.chunk_ids + static_cast<int64_t>(b) * a.chunk_list_ld;
    if (a.compose && nch > 0) {  // precomposed base for the longest listed prefix
      for (int k = min(nch, a.compose_depth); k >= 1; --k) {
        int64_t idx = 0;
        for (int d = 0; d < a.compose_depth; ++d) {
          FASE_ASSERT(cids[min(d, k - 1)] >= 0 && cids[min(d, k - 1)] < a.n_compose);
          idx = idx * a.n_compose + cids[min(d, k - 1)];
        }
        const int p = a.compose[idx];
        if (p > 0) {
          G0 += 2 * static_cast<int64_t>(p) * a.base_stride;
          cids += k;
          nch -= k;
          break;
        }
      }
    }
  }

  double r[EP][2];
  double dreg[(kDsmem || kScaled) ? 1 : EP];
  auto d2 = [&](int j) -> double {  // D^2 of element j; dead: -inf
    if constexpr (kDsmem)
      return s_D2[j * NT + t];
    else
      return dreg[j];
  };
  // D itself is only needed for exact metrics (candidates, the exact pass):
  // read from global memory (L2-resident) there
  auto dval = [&](int j) -> double {
    const int k = j * NT + t;
    const double dk = k < K ? D[k] : 0.0;
    return dk != 0.0 ? dk : kDead;
  };
  auto proxy = [](double re, double im, double d2) {
    if constexpr (kScaled)
      return __fma_rn(re, re, mul_rn(im, im));
    else
      return mul_rn(__fma_rn(re, re, mul_rn(im, im)), d2);
  };
  auto d2_if = [&](int j) -> double {
    if constexpr (kScaled)
      return 1.0;
    else
      return d2(j);
  };
  // the exact metric |R| * D (scaled: |R'|)
  auto emetric = [](double re, double im, double d) {
    if constexpr (kScaled)
      return np_cabs_fast(re, im);
    else
      return mul_rn(np_cabs_fast(re, im), d);
  };
  double best = kDead;
  unsigned barg = kNone;
#pragma unroll
  for (int j = 0; j < EP; ++j) {
    const int k = j * NT + t;
    r[j][0] = k < K ? R0[2 * k] : 0.0;
    r[j][1] = k < K ? R0[2 * k + 1] : 0.0;
    const double dk = k < K ? D[k] : 0.0;
    const double dsq = dk != 0.0 ? mul_rn(dk, dk) : kDead;
    if constexpr (kScaled) {
      const double kNaN = __longlong_as_double(0x7ff8000000000000LL);
      r[j][0] = dk != 0.0 ? mul_rn(r[j][0], dk) : kNaN;
      r[j][1] = dk != 0.0 ? mul_rn(r[j][1], dk) : kNaN;
    } else if constexpr (kDsmem) {
      if (half == 0) s_D2[j * NT + t] = dsq;
    } else
      dreg[j] = dsq;
    const double pk = proxy(r[j][0], r[j][1], dsq);
    if (pk > best) {
      best = pk;
      barg = static_cast<unsigned>(k);
    }
  }
  if constexpr (NB > 1) {
    __syncthreads();  // the shared D^2 (written by half 0) is complete
    if (!active) return;
  }

  int32_t* sel = a.sel + static_cast<int64_t>(b) * a.ldo;
  double* proj = a.proj + 2 * static_cast<int64_t>(b) * a.ldo;
  double* coef = a.coef + 2 * static_cast<int64_t>(b) * a.ldo;
  const int64_t ldg2x = 2 * a.ldg;  // row stride in doubles
  double q = 0.0;

  for (int it = 0; it < a.I; ++it) {
    // ---- warp max of the proxy and the lowest index attaining it
    {
      const long long key = __double_as_longlong(best);
      const int kh = static_cast<int>(key >> 32);
      const unsigned kl = static_cast<unsigned>(key);
      const int wh = __reduce_max_sync(0xffffffffu, kh);
      const unsigned wl = __reduce_max_sync(0xffffffffu, kh == wh ? kl : 0u);
      const unsigned wa = __reduce_min_sync(0xffffffffu, (kh == wh && kl == wl) ? barg : kNone);
      if (lane == 0) {
        s_key[warp] = (static_cast<long long>(wh) << 32) | wl;
        s_arg[warp] = wa;
      }
    }
    block_sync();
    if (t == 0) s_cnt[(it + 1) & 1] = 0;  // next iteration's list (last read before this barrier)
    long long top_key, wkey;
    unsigned guess;
    {
      const long long sk = lane < NW ? s_key[lane] : LLONG_MIN;
      const unsigned sa = lane < NW ? s_arg[lane] : kNone;
      wkey = s_key[warp];
      const int h = static_cast<int>(sk >> 32);
      const unsigned l = static_cast<unsigned>(sk);
      const int bh = __reduce_max_sync(0xffffffffu, h);
      const unsigned bl = __reduce_max_sync(0xffffffffu, h == bh ? l : 0u);
      guess = __reduce_min_sync(0xffffffffu, (h == bh && l == bl) ? sa : kNone);
      top_key = (static_cast<long long>(bh) << 32) | bl;
    }
    if (top_key < 0) {  // every atom degenerate (NoSelectableAtomError): mark and stop
      for (int k = it + t; k < a.I; k += NT) {
        sel[k] = -1;
        proj[2 * k] = proj[2 * k + 1] = 0.0;
        coef[2 * k] = coef[2 * k + 1] = 0.0;
      }
      return;
    }
    if (t == 0) {
      FASE_ASSERT(guess < static_cast<unsigned>(K));
      fence_before_refill();
      const double* grow = G0 + static_cast<int64_t>(guess) * ldg2x;
#pragma unroll
      for (int sg = 0; sg < kSeg; ++sg) {
        const int j0 = sg * EP / kSeg, j1 = (sg + 1) * EP / kSeg;
        const unsigned bytes = static_cast<unsigned>((j1 - j0) * NT * sizeof(double2));
        mbar_arrive_expect_tx(&s_bar[sg], bytes);
        tma_load_1d(s_row + j0 * NT, grow + 2 * j0 * NT, bytes, &s_bar[sg]);
      }
    }

    // ---- candidates: P_k >= a lower bound of thr^2 (conservative margins)
    const double pmax = __longlong_as_double(top_key);
    // proxies outside [2^-900, 2^900] lose the relative accuracy the bound needs
    const bool trusted = pmax >= 0x1p-900 && pmax <= 0x1p+900;
    double pc = 0.0, top_hi = 0.0;
    if (trusted) {
      const double s = sqrt(pmax);
      const double top_lo = s * (1.0 - 0x1p-40);
      top_hi = s * (1.0 + 0x1p-40);
      const double thr_lo = top_lo - fmax(q, 1e-13 * top_hi) * (1.0 + 0x1p-40);
      pc = thr_lo > 0.0 ? thr_lo * thr_lo * (1.0 - 0x1p-40) : 0.0;
    }
    if (trusted && pc > 0.0 && wkey >= 0 && __longlong_as_double(wkey) >= pc) {  // warp-uniform
#pragma unroll
      for (int j = 0; j < EP; ++j) {
        if (proxy(r[j][0], r[j][1], d2_if(j)) >= pc) {  // exact metric after the barrier
          const int slot = atomicAdd(&s_cnt[it & 1], 1);
          if (slot < kCap) {
            s_ck[slot] = static_cast<unsigned>(j * NT + t);
            s_cr[slot] = make_double2(r[j][0], r[j][1]);
            s_cd[slot] = dval(j);
          }
        }
      }
    }
    block_sync();
    const int cnt = s_cnt[it & 1];

    unsigned u;
    double2 ru;
    double du;
    if (trusted && pc > 0.0 && cnt == 1) {
      // ---- the common case: one candidate, so it is the maximum and the
      // selection. Its exact metric matters only if the tie quantum can move
      // (1e-13 * top > q), which the proxy's upper bound rules out after the
      // first iterations.
      u = s_ck[0];
      ru = s_cr[0];
      du = s_cd[0];
      if (mul_rn(1e-13, top_hi) > q) {
        const double top = emetric(ru.x, ru.y, du);
        if (top > 0.0 && top < __longlong_as_double(0x7ff0000000000000LL)) q = fmax(q, mul_rn(1e-13, top));
      }
    } else if (trusted && pc > 0.0 && cnt >= 2 && cnt <= kCap) {
      // ---- resolve the list in every warp: exact max, quantum, lowest index
      // one lane per entry: exact metric (entries past 32 are rare)
      long long mk = LLONG_MIN;
      double m0 = -1.0;
      for (int l = lane; l < cnt; l += 32) {
        const double2 rv = s_cr[l];
        const double m = emetric(rv.x, rv.y, s_cd[l]);
        if (l == lane) m0 = m;
        else s_cm[l] = m;
        const long long v = __double_as_longlong(m);  // metrics of candidates are >= 0
        mk = v > mk ? v : mk;
      }
      const double top = __longlong_as_double(warp_max_i64(mk));
      if (top > 0.0 && top < __longlong_as_double(0x7ff0000000000000LL)) q = fmax(q, mul_rn(1e-13, top));
      const double thr = q > 0.0 ? sub_rn(top, q) : top;
      unsigned ub = kNone;
      int ib = 0;
      for (int l = lane; l < cnt; l += 32) {
        const unsigned kk = (l == lane ? m0 : s_cm[l]) >= thr ? s_ck[l] : kNone;
        if (kk < ub) {
          ub = kk;
          ib = l;
        }
      }
      u = __reduce_min_sync(0xffffffffu, ub);
      const int src = __ffs(__ballot_sync(0xffffffffu, ub == u)) - 1;
      ib = __shfl_sync(0xffffffffu, ib, src);
      ru = s_cr[ib];
      du = s_cd[ib];
    } else {
      // ---- exact pass over every element (block-uniform branch). One rolled
      // loop per pass: element jj is picked out of the register array with
      // selects, so the division / square root appear once in the code.
      auto element = [&](int jj, double& re, double& im, double& d) {
        re = 0.0;
        im = 0.0;
#pragma unroll
        for (int j = 0; j < EP; ++j)
          if (j == jj) {
            re = r[j][0];
            im = r[j][1];
          }
        d = dval(jj);
      };
      double mb = kDead;
#pragma unroll 1
      for (int jj = 0; jj < EP; ++jj) {
        double re, im, d;
        element(jj, re, im, d);
        const double m = emetric(re, im, d);  // dead: -inf or NaN
        mb = m > mb ? m : mb;
      }
      const long long wk = warp_max_i64(__double_as_longlong(mb));
      if (lane == 0) s_key[warp] = wk;
      block_sync();
      long long tk = LLONG_MIN;
#pragma unroll
      for (int w = 0; w < NW; ++w) tk = s_key[w] > tk ? s_key[w] : tk;
      const double top = __longlong_as_double(tk);
      if (tk > 0 && tk < 0x7ff0000000000000LL) q = fmax(q, mul_rn(1e-13, top));
      const double thr = q > 0.0 ? sub_rn(top, q) : top;
      unsigned cand = kNone;
      double2 rv = make_double2(0.0, 0.0);
      double dv = 0.0;
#pragma unroll 1
      for (int jj = 0; jj < EP; ++jj) {
        double re, im, d;
        element(jj, re, im, d);
        if (cand == kNone && emetric(re, im, d) >= thr) {
          cand = static_cast<unsigned>(jj * NT + t);
          rv = make_double2(re, im);
          dv = d;
        }
      }
      // exchange through the candidate arrays: s_key / s_arg are rewritten by
      // fast warps before the next first barrier, the list only after it
      const unsigned wmin = __reduce_min_sync(0xffffffffu, cand);
      if (lane == 0) s_ck[warp] = wmin;
      if (cand != kNone && cand == wmin) {
        s_cr[warp] = rv;
        s_cd[warp] = dv;
      }
      block_sync();
      const unsigned su = lane < NW ? s_ck[lane] : kNone;
      u = __reduce_min_sync(0xffffffffu, su);
      const int uw = __ffs(__ballot_sync(0xffffffffu, su == u)) - 1;
      ru = s_cr[uw];
      du = s_cd[uw];
    }

    FASE_ASSERT(u < static_cast<unsigned>(K));
    const double d2u = kScaled ? du : mul_rn(du, du);  // scaled: p = R'_u * D_u
    const double pr = mul_rn(ru.x, d2u), pi = mul_rn(ru.y, d2u);
    const double cr = mul_rn(a.gamma, pr), ci = mul_rn(a.gamma, pi);
    if (t == 0) {
      sel[it] = static_cast<int32_t>(u);
      proj[2 * it] = pr;
      proj[2 * it + 1] = pi;
      coef[2 * it] = cr;
      coef[2 * it + 1] = ci;
    }

    auto wait_all = [&]() {
#pragma unroll
      for (int sg = 0; sg < kSeg; ++sg) mbar_wait(&s_bar[sg], it & 1);
    };
    // ---- R <- R - c * conj(C[u, :]) fused with the next running max of the proxy
    auto update = [&](auto row_elem, auto staged) {
      best = kDead;
      barg = kNone;
#pragma unroll
      for (int j = 0; j < EP; ++j) {
        if constexpr (decltype(staged)::value) {
#pragma unroll
          for (int sg = 0; sg < kSeg; ++sg)
            if (j == sg * EP / kSeg) mbar_wait(&s_bar[sg], it & 1);
        }
        const double2 g = row_elem(j);
        if constexpr (kScaled && FASE_CSCALED_FMA) {
          // scaled recursion: R' - c * row fused (two roundings per component
          // instead of numpy's three)
          r[j][0] = __fma_rn(ci, g.y, __fma_rn(-cr, g.x, r[j][0]));
          r[j][1] = __fma_rn(-ci, g.x, __fma_rn(-cr, g.y, r[j][1]));
        } else {
          const double2 x = np_cmul(cr, ci, g.x, g.y);
          r[j][0] = sub_rn(r[j][0], x.x);
          r[j][1] = sub_rn(r[j][1], x.y);
        }
        const double pk = proxy(r[j][0], r[j][1], d2_if(j));
        if (pk > best) {
          best = pk;
          barg = static_cast<unsigned>(j * NT + t);
        }
      }
    };
    using Staged = std::true_type;
    using Direct = std::false_type;
    if (kChunked && nch > 0) {
      wait_all();
      if (u != guess) {
        const double* urow = G0 + static_cast<int64_t>(u) * ldg2x + 2 * t;
#pragma unroll 4
        for (int j = 0; j < EP; ++j) s_row[j * NT + t] = ldg2(urow + 2 * j * NT);
      }
      for (int ch = 0; ch < nch; ++ch) {
        const double* crow = a.chunk_tables + 2 * static_cast<int64_t>(cids[ch]) * a.chunk_stride +
                             static_cast<int64_t>(u) * ldg2x + 2 * t;
#pragma unroll 4
        for (int j = 0; j < EP; ++j) {
          const double2 v = ldg2(crow + 2 * j * NT);
          double2 g = s_row[j * NT + t];
          g.x = sub_rn(g.x, v.x);
          g.y = sub_rn(g.y, v.y);
          s_row[j * NT + t] = g;
        }
      }
      update([&](int j) { return s_row[j * NT + t]; }, Direct{});
      fence_proxy_async_smem();
    } else if (u == guess) {
      update([&](int j) { return s_row[j * NT + t]; }, Staged{});
    } else {
      wait_all();
      const double* urow = G0 + static_cast<int64_t>(u) * ldg2x + 2 * t;
      update([&](int j) { return ldg2(urow + 2 * j * NT); }, Direct{});
    }
    if (kRecord) {
      double* dst = a.R_log + 2 * ((static_cast<int64_t>(b) * a.I + it) * a.ldr);
#pragma unroll
      for (int j = 0; j < EP; ++j) {
        const int k = j * NT + t;
        if (k < K) *reinterpret_cast<double2*>(dst + 2 * k) = make_double2(r[j][0], r[j][1]);
      }
    }
  }

  if (a.R_out) {
    double* dst = a.R_out + 2 * static_cast<int64_t>(b) * a.ldr;
#pragma unroll
    for (int j = 0; j < EP; ++j) {
      const int k = j * NT + t;
      if (k < K) *reinterpret_cast<double2*>(dst + 2 * k) = make_double2(r[j][0], r[j][1]);
    }
  }
}

using KernelFn = void (*)(const fase_iterate_args);

struct Variant {
  int nt;
  int ep;  // complex elements per thread
  bool dsmem;
  KernelFn plain;
  KernelFn chunked;
  KernelFn record;
  int nb = 1;  // blocks per CTA (2: paired blocks sharing D^2)
};

#define FASE_CV(NT, EP, MINB, DS)                                      \
  {NT,                                                                  \
   EP,                                                                  \
   DS,                                                                  \
   fase_iterate_complex_kernel<NT, EP, MINB, DS, false, false, 1>,         \
   fase_iterate_complex_kernel<NT, EP, MINB, DS, true, false, 1>,          \
   fase_iterate_complex_kernel<NT, EP, MINB, DS, false, true, 1>}
// Ordered by capacity NT*EP (complex elements); the first that holds K is used.
// The exact metric uses call-free division / square root (np_cabs_fast), so
// the 256-thread shapes fit three CTAs per SM like the real kernel (the IEEE
// operations' slow-path calls cost 40 registers and 2 CTAs/SM: 1.25 ms against
// 1.02 ms per config-1 step with the default dictionary).
const Variant kVariants[] = {
    FASE_CV(128, 1, 4, false), FASE_CV(128, 2, 4, false), FASE_CV(128, 4, 4, false),
    FASE_CV(128, 8, 4, true),  FASE_CV(256, 5, 3, true),  FASE_CV(256, 6, 3, true),
    FASE_CV(256, 7, 3, true),  FASE_CV(256, 8, 3, true),  FASE_CV(256, 9, 3, true),
    FASE_CV(256, 10, 2, true), FASE_CV(512, 6, 1, true),  FASE_CV(512, 8, 1, true),
    FASE_CV(512, 9, 1, true),  FASE_CV(512, 10, 1, true), FASE_CV(512, 12, 1, true),
};
// Paired blocks for shared geometries, same capacity as the 512-thread default
// (so the same table layout): two blocks in flight per SM instead of one.
#define FASE_CVP(NT, EP)                                                                   \
  {NT, EP, true, fase_iterate_complex_kernel<NT, EP, 1, true, false, false, 2>, nullptr, nullptr, 2}
const Variant kPairVariants[] = {
    FASE_CVP(256, 12), FASE_CVP(256, 16), FASE_CVP(256, 18), FASE_CVP(256, 20),
};
#undef FASE_CVP
// Alternative residency for measurement (FASE_ITERATE_COMPLEX_VARIANT=NTxEPxMINB;
// same capacity as the default variant for K).
struct ExtraVariant {
  int minb;
  Variant v;
};
const ExtraVariant kExtraVariants[] = {
    {2, FASE_CV(256, 7, 2, true)}, {2, FASE_CV(256, 8, 2, true)}, {2, FASE_CV(256, 9, 2, true)},
    {4, FASE_CV(256, 9, 4, true)},
};
#undef FASE_CV

// Scaled recursion: no D^2 in shared memory; ordered by capacity like
// kVariants (same table layout), 256-thread shapes up to 5120 atoms (two
// blocks per SM where the exact kernel needs paired 512-thread CTAs).
#define FASE_CS(NT, EP, MINB) \
  {NT, EP, false, fase_iterate_complex_kernel<NT, EP, MINB, false, false, false, 1, true>, nullptr, nullptr}
// The 256-thread shapes up to 2304 atoms run four CTAs per SM (64 registers,
// a few spilled): 1,024 blocks then take two waves of 592 slots instead of
// three of 444 (`dft` 48^2, config-1 batch: 1.018 -> 0.830 ms per recursion,
// tools/ab_complex.sh; the exact kernel, with D^2 in shared memory, was slower
// at four CTAs: 0.994 -> 1.198 ms).
const Variant kScaledVariants[] = {
    FASE_CS(128, 1, 4),  FASE_CS(128, 2, 4),  FASE_CS(128, 4, 4),  FASE_CS(128, 8, 4),
    FASE_CS(256, 5, 4),  FASE_CS(256, 6, 4),  FASE_CS(256, 7, 4),  FASE_CS(256, 8, 4),
    FASE_CS(256, 9, 4),  FASE_CS(256, 10, 2), FASE_CS(256, 12, 2), FASE_CS(256, 16, 2),
    FASE_CS(256, 18, 2), FASE_CS(256, 20, 2), FASE_CS(512, 12, 1),
};
// alternative residency of the scaled shapes (FASE_COMPLEX_SCALED_VARIANT=NTxEPxMINB)
const ExtraVariant kScaledExtra[] = {
    {3, FASE_CS(256, 9, 3)}, {3, FASE_CS(256, 8, 3)}, {3, FASE_CS(256, 10, 3)},
};
#undef FASE_CS

const Variant* pick_variant(int K) {
  for (const Variant& v : kVariants)
    if (v.nt * v.ep >= K) return &v;
  return nullptr;
}

const Variant* override_variant(int K, const Variant* dflt) {
  const char* env = getenv("FASE_ITERATE_COMPLEX_VARIANT");
  if (!env || !dflt) return dflt;
  int nt = 0, ep = 0, minb = 0;
  if (sscanf(env, "%dx%dx%d", &nt, &ep, &minb) != 3) return dflt;
  for (const ExtraVariant& x : kExtraVariants)
    if (x.minb == minb && x.v.nt == nt && x.v.ep == ep && nt * ep >= K &&
        nt * ep <= dflt->nt * dflt->ep)
      return &x.v;
  return dflt;
}

}  // namespace
}  // namespace fase

using namespace fase;

namespace fase {
// csrc/iterate_generic.cu: R streamed through global memory (K beyond the registers)
int launch_iterate_generic_complex(const fase_iterate_args& a, int reg_atoms, cudaStream_t stream);
}
namespace {
constexpr int kGenericMaxAtomsComplex = 1 << 20;
int complex_register_atoms() {
  const Variant& last = kVariants[sizeof(kVariants) / sizeof(kVariants[0]) - 1];
  return last.nt * last.ep;
}
}  // namespace

extern "C" int fase_max_atoms_complex(void) { return kGenericMaxAtomsComplex; }

extern "C" int fase_iterate_complex_register_atoms(void) { return complex_register_atoms(); }

extern "C" int fase_table_ld_complex(int K) {
  if (K < 1 || K > kGenericMaxAtomsComplex) return 0;
  const Variant* v = pick_variant(K);
  return v ? v->nt * v->ep : K;  // beyond the registers: unpadded (16-byte elements)
}

extern "C" int fase_iterate_complex(const fase_iterate_args* args, void* stream) {
  if (!args) {
    set_error("fase_iterate_complex: null argument block");
    return FASE_ERR_PARAMETER;
  }
  const fase_iterate_args& a = *args;
  if (a.K < 1 || a.B < 0 || a.I < 1) {
    set_error("fase_iterate_complex: bad sizes (K=%d, B=%d, I=%d)", a.K, a.B, a.I);
    return FASE_ERR_SHAPE;
  }
  if (!(a.gamma > 0.0 && a.gamma <= 1.0)) {
    set_error("fase_iterate_complex: gamma must lie in (0, 1], got %g", a.gamma);
    return FASE_ERR_PARAMETER;
  }
  if (a.B == 0) return FASE_OK;
  if (!a.G0 || !aligned16(a.G0) || a.ldg < a.K || !a.D || !a.R0 || !aligned16(a.R0) ||
      a.ldr < a.K || (a.ldd != 0 && a.ldd < a.K) || !a.sel || !a.proj || !a.coef || a.ldo < a.I ||
      (a.R_out && !aligned16(a.R_out)) || (a.R_log && !aligned16(a.R_log))) {
    set_error("fase_iterate_complex: bad operand (null, misaligned or short leading dimension)");
    return FASE_ERR_SHAPE;
  }
  if (a.chunk_count && (!a.chunk_ids || !a.chunk_tables || !aligned16(a.chunk_tables))) {
    set_error("fase_iterate_complex: chunk tables given without ids / aligned storage");
    return FASE_ERR_SHAPE;
  }
  if (a.compose && (!a.chunk_count || a.n_compose < 1 || a.compose_depth < 1 ||
                    a.compose_depth > 3 || a.base_stride < a.ldg * a.K)) {
    set_error("fase_iterate_complex: compose table needs chunk lists, n_compose >= 1, depth 1..3 "
              "and base_stride >= ldg*K");
    return FASE_ERR_SHAPE;
  }
  if (a.chunk_count && a.R_log) {
    set_error("fase_iterate_complex: R_log recording is not available with chunked tables");
    return FASE_ERR_UNSUPPORTED;
  }
  if (!pick_variant(a.K) && a.K <= kGenericMaxAtomsComplex) {  // the streaming recursion
    if (a.ldg < a.K || (a.chunk_count && a.chunk_stride < a.ldg * a.K)) {
      set_error("fase_iterate_complex: table rows shorter than K (ldg=%lld)",
                static_cast<long long>(a.ldg));
      return FASE_ERR_SHAPE;
    }
    return launch_iterate_generic_complex(a, complex_register_atoms(), as_stream(stream));
  }
  const Variant* v = override_variant(a.K, pick_variant(a.K));
  if (!v) {
    set_error("fase_iterate_complex: K=%d exceeds the largest kernel variant (%d atoms)", a.K,
              complex_register_atoms());
    return FASE_ERR_UNSUPPORTED;
  }
  if (a.ldg < v->nt * v->ep || (a.chunk_count && a.chunk_stride < a.ldg * a.K)) {
    set_error("fase_iterate_complex: table rows must be zero-padded to fase_table_ld_complex(K)=%d "
              "(ldg=%lld)", v->nt * v->ep, static_cast<long long>(a.ldg));
    return FASE_ERR_SHAPE;
  }
  int sms = 148;
  {
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess)
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  if (!a.chunk_count && !a.R_log && a.ldd == 0 && a.B > sms) {
    // FASE_ITERATE_PAIR: 0 disables pairing (measurement); batches of at most
    // one block per SM are not paired (pairs would halve the CTAs)
    const char* env = getenv("FASE_ITERATE_PAIR");
    if (!env || atoi(env) != 0)
      for (const Variant& pv : kPairVariants)
        if (pv.nt * pv.ep == v->nt * v->ep) v = &pv;
  }
  KernelFn fn = a.chunk_count ? v->chunked : (a.R_log ? v->record : v->plain);
  const size_t smem = static_cast<size_t>(v->nt) * v->ep *
                      (v->nb * sizeof(double2) + (v->dsmem ? sizeof(double) : 0));
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e == cudaSuccess) e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (e != cudaSuccess) {
    set_error("fase_iterate_complex: cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    return FASE_ERR_CUDA;
  }
  fn<<<(a.B + v->nb - 1) / v->nb, v->nt * v->nb, smem, as_stream(stream)>>>(a);
  return check_launch("fase_iterate_complex");
}

extern "C" int fase_iterate_complex_scaled(const fase_iterate_args* args, void* stream) {
  if (!args) {
    set_error("fase_iterate_complex_scaled: null argument block");
    return FASE_ERR_PARAMETER;
  }
  const fase_iterate_args& a = *args;
  if (a.K < 1 || a.B < 0 || a.I < 1) {
    set_error("fase_iterate_complex_scaled: bad sizes (K=%d, B=%d, I=%d)", a.K, a.B, a.I);
    return FASE_ERR_SHAPE;
  }
  if (!(a.gamma > 0.0 && a.gamma <= 1.0)) {
    set_error("fase_iterate_complex_scaled: gamma must lie in (0, 1], got %g", a.gamma);
    return FASE_ERR_PARAMETER;
  }
  if (a.B == 0) return FASE_OK;
  if (!a.G0 || !aligned16(a.G0) || a.ldg < a.K || !a.D || !a.R0 || !aligned16(a.R0) ||
      a.ldr < a.K || !a.sel || !a.proj || !a.coef || a.ldo < a.I) {
    set_error("fase_iterate_complex_scaled: bad operand (null, misaligned or short leading "
              "dimension)");
    return FASE_ERR_SHAPE;
  }
  if (a.chunk_count || a.compose || a.ldd != 0 || a.R_out || a.R_log) {
    set_error("fase_iterate_complex_scaled: shared geometry only (no chunk tables, per-block D, "
              "R_out or R_log)");
    return FASE_ERR_UNSUPPORTED;
  }
  const Variant* dflt = pick_variant(a.K);
  const Variant* v = nullptr;
  for (const Variant& sv : kScaledVariants)
    if (sv.nt * sv.ep >= a.K) {
      v = &sv;
      break;
    }
  if (const char* env = getenv("FASE_COMPLEX_SCALED_VARIANT")) {
    int nt = 0, ep = 0, minb = 0;
    if (v && dflt && sscanf(env, "%dx%dx%d", &nt, &ep, &minb) == 3)
      for (const ExtraVariant& x : kScaledExtra)
        if (x.minb == minb && x.v.nt == nt && x.v.ep == ep && nt * ep >= a.K &&
            nt * ep <= dflt->nt * dflt->ep)
          v = &x.v;
  }
  if (!dflt || !v) {
    set_error("fase_iterate_complex_scaled: K=%d exceeds the largest kernel variant (%d atoms)",
              a.K, complex_register_atoms());
    return FASE_ERR_UNSUPPORTED;
  }
  if (a.ldg < v->nt * v->ep) {
    set_error("fase_iterate_complex_scaled: table rows must be zero-padded to "
              "fase_table_ld_complex(K)=%d (ldg=%lld)", dflt->nt * dflt->ep,
              static_cast<long long>(a.ldg));
    return FASE_ERR_SHAPE;
  }
  const size_t smem = static_cast<size_t>(v->nt) * v->ep * sizeof(double2);
  cudaError_t e = cudaFuncSetAttribute(v->plain, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(v->plain, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (e != cudaSuccess) {
    set_error("fase_iterate_complex_scaled: cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    return FASE_ERR_CUDA;
  }
  v->plain<<<a.B, v->nt, smem, as_stream(stream)>>>(a);
  return check_launch("fase_iterate_complex_scaled");
}
