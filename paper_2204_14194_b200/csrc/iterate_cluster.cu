// The FaSE recursion for latency-bound batches: ONE block split over a
// thread-block cluster of CS CTAs (hard part 5).
//
// Same loop and arithmetic as fase_iterate_kernel (pkg/src/fase/fast.py:238-255,
// tie rule reference.py:55-85), exact or scaled, but the K atoms of a block are
// cut into CS contiguous slices, one per CTA of the cluster (on CS SMs). Each
// CTA keeps its slice of R (and D) in registers and TMA-stages only its slice
// of the selected table row, so a row arrives CS times faster and the update is
// CS times shorter. The two block-wide decisions of an iteration become
// cluster-wide exchanges over distributed shared memory:
//
//   A. each CTA's exact max |R|*D and the lowest index attaining it;
//   B. each CTA's lowest index reaching the tie threshold, with its R (and D).
//
// An exchange is one 16- or 32-byte st.async push from every CTA into every
// CTA's slot array, completing transaction bytes on the receiver's mbarrier
// (no cluster-wide barrier in the loop: a receiver waits only for its own
// mbarrier, ~one DSMEM latency). Slots and mbarriers are double buffered by
// iteration parity; a CTA cannot run two iterations ahead of a peer because
// every iteration needs the peer's pushes, so a slot is never overwritten
// before it has been read. Every CTA derives the same top, threshold, tie
// quantum and selection from the same slots, so the cluster stays in lockstep
// without further synchronization; CTA rank 0 writes the outputs.

#include <climits>
#include <cstdlib>

#include "common.cuh"

namespace fase {

int sm_count_cluster();

namespace {

constexpr unsigned kNoneC = 0xffffffffu;

__device__ __forceinline__ unsigned cluster_ctarank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}

// shared::cluster address of `p` (a shared variable of this CTA) in CTA `rank`
__device__ __forceinline__ unsigned peer_addr(const void* p, unsigned rank) {
  unsigned a;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(a) : "r"(smem_u32(p)), "r"(rank));
  return a;
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile(
      "barrier.cluster.arrive.release.aligned;\n"
      "barrier.cluster.wait.acquire.aligned;\n" ::
          : "memory");
}

// 16 bytes into a peer's shared memory; completes 16 transaction bytes on the
// peer's mbarrier `bar` (both shared::cluster addresses)
__device__ __forceinline__ void push16(unsigned dst, unsigned bar, uint32_t x, uint32_t y, uint32_t z,
                                       uint32_t w) {
  asm volatile(
      "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];\n" ::
          "r"(dst),
      "r"(x), "r"(y), "r"(z), "r"(w), "r"(bar)
      : "memory");
}

__device__ __forceinline__ void mbar_wait_acq_cluster(uint64_t* bar, unsigned parity) {
#ifdef FASE_BOUNDS
  for (long long spin = 0;; ++spin) {
    unsigned done;
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (done) return;
    FASE_ASSERT(spin < (1ll << 26));
  }
#else
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAITC_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAITC_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
#endif
}

__device__ __forceinline__ uint32_t lo32(double v) {
  return static_cast<uint32_t>(__double_as_longlong(v));
}
__device__ __forceinline__ uint32_t hi32(double v) {
  return static_cast<uint32_t>(static_cast<unsigned long long>(__double_as_longlong(v)) >> 32);
}
__device__ __forceinline__ double mk_double(uint32_t lo, uint32_t hi) {
  return __longlong_as_double(static_cast<long long>((static_cast<unsigned long long>(hi) << 32) | lo));
}

template <int NT, int EP, int CS, bool kScaled, int SYN>
__global__ void __cluster_dims__(CS, 1, 1) __launch_bounds__(NT, 1)
    fase_iterate_cluster_kernel(const fase_iterate_args a, const fase_synth_fused syn) {
  constexpr int NW = NT / 32;
  constexpr int KS = 2 * NT * EP;  // elements per CTA slice
  constexpr int kSeg = EP < 3 ? EP : 3;
  static_assert(NT % 32 == 0 && NW <= 32, "whole warps, at most 32");
  static_assert(SYN == 0 || kScaled, "fused synthesis runs with the scaled recursion");
  __shared__ __align__(16) double2 s_row[EP * NT];
  __shared__ __align__(16) double s_phi[SYN > 0 ? SYN * NT : 2];
  __shared__ __align__(8) uint64_t s_bar[kSeg];   // staged row segments (TMA)
  __shared__ __align__(8) uint64_t s_xbar[2][2];  // exchange [A|B][iteration parity]
  __shared__ __align__(16) uint4 s_xa[2][CS];     // A: key lo, key hi, arg, -
  __shared__ __align__(16) uint4 s_xb[2][CS][2];  // B: cand, -, r lo, r hi | d lo, d hi, -, -
  __shared__ long long s_key[NW];
  __shared__ unsigned s_arg[NW];
  __shared__ unsigned s_u[NW];
  __shared__ double s_r[NW];
  __shared__ double s_d[NW];
  __shared__ __align__(16) double s_dump[NW][2 * EP];
  __shared__ __align__(16) double s_dumpd[kScaled ? 1 : NW][2 * EP];

  const unsigned rank = cluster_ctarank();
  const int b = static_cast<int>(blockIdx.x) / CS;
  const int t = static_cast<int>(threadIdx.x);
  const int lane = t & 31, warp = t >> 5;
  const int K = a.K;
  const int k0 = static_cast<int>(rank) * KS;  // first element of this CTA's slice
  const double kDead = __longlong_as_double(static_cast<long long>(0xfff0000000000000ULL));

  if (t == 0) {
    for (int sg = 0; sg < kSeg; ++sg) mbar_init(&s_bar[sg], 1);
    for (int x = 0; x < 2; ++x)
      for (int p = 0; p < 2; ++p) mbar_init(&s_xbar[x][p], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  cluster_sync_all();  // every CTA's mbarriers exist before any push

  // fused synthesis: CTA `rank` owns lost samples [ls0, ls1), thread t the
  // samples ls0 + t + s*NT
  const int LS = SYN > 0 ? (((syn.n_lost + CS - 1) / CS + 1) & ~1) : 0;
  const int ls0 = SYN > 0 ? min(syn.n_lost, static_cast<int>(rank) * LS) : 0;
  const int ls1 = SYN > 0 ? min(syn.n_lost, ls0 + LS) : 0;
  double gacc[SYN > 0 ? SYN : 1];
#pragma unroll
  for (int i = 0; i < (SYN > 0 ? SYN : 1); ++i) gacc[i] = 0.0;

  const double* R0 = a.R0 + static_cast<int64_t>(b) * a.ldr;
  double r[EP][2];
  double dreg[kScaled ? 1 : EP][2];
  double best = kDead;
  unsigned barg = kNoneC;
#pragma unroll
  for (int j = 0; j < EP; ++j) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int k = k0 + 2 * (j * NT + t) + e;
      const double d = k < K ? a.D[k] : 0.0;
      double m;
      if constexpr (kScaled) {
        r[j][e] = d != 0.0 ? mul_rn(R0[k], d) : __longlong_as_double(0x7ff8000000000000LL);
        m = fabs(r[j][e]);
      } else {
        r[j][e] = k < K ? R0[k] : 0.0;
        dreg[j][e] = d != 0.0 ? d : kDead;
        m = mul_rn(fabs(r[j][e]), dreg[j][e]);
      }
      if (m > best) {
        best = m;
        barg = static_cast<unsigned>(k);
      }
    }
  }

  int32_t* sel = a.sel + static_cast<int64_t>(b) * a.ldo;
  double* proj = a.proj + static_cast<int64_t>(b) * a.ldo;
  double* coef = a.coef + static_cast<int64_t>(b) * a.ldo;
  double q = 0.0;
  bool dead = false;

  for (int it = 0; it < a.I; ++it) {
    const int par = it & 1;
    const unsigned xpar = static_cast<unsigned>(it >> 1) & 1u;
    // ---- A: this CTA's exact max and lowest index, pushed to every CTA
    {
      const long long key = __double_as_longlong(best);
      const int kh = static_cast<int>(key >> 32);
      const unsigned kl = static_cast<unsigned>(key);
      const int wh = __reduce_max_sync(0xffffffffu, kh);
      const unsigned wl = __reduce_max_sync(0xffffffffu, kh == wh ? kl : 0u);
      const unsigned wa = __reduce_min_sync(0xffffffffu, (kh == wh && kl == wl) ? barg : kNoneC);
      if (lane == 0) {
        s_key[warp] = (static_cast<long long>(wh) << 32) | wl;
        s_arg[warp] = wa;
      }
    }
    __syncthreads();
    long long wkey = s_key[warp];
    if (warp == 0) {
      const long long sk = lane < NW ? s_key[lane] : LLONG_MIN;
      const unsigned sa = lane < NW ? s_arg[lane] : kNoneC;
      const int h = static_cast<int>(sk >> 32);
      const unsigned l = static_cast<unsigned>(sk);
      const int bh = __reduce_max_sync(0xffffffffu, h);
      const unsigned bl = __reduce_max_sync(0xffffffffu, h == bh ? l : 0u);
      const unsigned ga = __reduce_min_sync(0xffffffffu, (h == bh && l == bl) ? sa : kNoneC);
      if (lane < CS) {  // lane p pushes this CTA's record into CTA p
        push16(peer_addr(&s_xa[par][rank], lane), peer_addr(&s_xbar[0][par], lane), bl,
               static_cast<uint32_t>(bh), ga, 0u);
      }
      if (lane == 0) mbar_arrive_expect_tx(&s_xbar[0][par], CS * 16);
    }
    mbar_wait_acq_cluster(&s_xbar[0][par], xpar);
    long long top_key = LLONG_MIN;
    unsigned guess = kNoneC;
#pragma unroll
    for (int p = 0; p < CS; ++p) {
      const uint4 v = s_xa[par][p];
      const long long k = (static_cast<long long>(static_cast<int>(v.y)) << 32) | v.x;
      if (k > top_key || (k == top_key && v.z < guess)) {
        top_key = k;
        guess = v.z;
      }
    }
    if (top_key < 0) {  // every atom degenerate: mark and stop (all CTAs agree)
      if (rank == 0)
        for (int k = it + t; k < a.I; k += NT) {
          sel[k] = -1;
          proj[k] = 0.0;
          coef[k] = 0.0;
        }
      dead = true;
      break;
    }
    FASE_ASSERT(guess < static_cast<unsigned>(K));
    // stage this CTA's slice of the likely selection's row (and its lost
    // samples' phi values) while the tie pass and exchange B run
    if (t == 0) {
      fence_proxy_async_smem();
      const double* grow = a.G0 + static_cast<int64_t>(guess) * a.ldg + k0;
#pragma unroll
      for (int sg = 0; sg < kSeg; ++sg) {
        const int j0 = sg * EP / kSeg, j1 = (sg + 1) * EP / kSeg;
        const unsigned bytes = static_cast<unsigned>((j1 - j0) * NT * sizeof(double2));
        const unsigned pb = (SYN > 0 && sg == kSeg - 1 && ls1 > ls0)
                                ? static_cast<unsigned>(((ls1 - ls0) * sizeof(double) + 15) & ~size_t{15})
                                : 0u;
        mbar_arrive_expect_tx(&s_bar[sg], bytes + pb);
        tma_load_1d(s_row + j0 * NT, grow + 2 * j0 * NT, bytes, &s_bar[sg]);
        if (pb) tma_load_1d(s_phi, syn.phi + static_cast<int64_t>(guess) * syn.ldphi + ls0, pb, &s_bar[sg]);
      }
    }
    const double top = __longlong_as_double(top_key);
    {  // the ratchet; a +0 top leaves it (1e-13 * 0), a +inf one must not move it
      const double qn = mul_rn(1e-13, top);
      q = qn < __longlong_as_double(0x7ff0000000000000LL) ? fmax(q, qn) : q;
    }
    const double thr = sub_rn(top, q);  // (q == 0: exactly top)

    // ---- B: this CTA's lowest index reaching the threshold, with R (and D)
    unsigned cand = kNoneC;
    if (wkey >= 0 && __longlong_as_double(wkey) >= thr) {  // warp-uniform
#pragma unroll
      for (int j = EP - 1; j >= 0; --j) {
#pragma unroll
        for (int e = 1; e >= 0; --e) {
          const double m = kScaled ? fabs(r[j][e]) : mul_rn(fabs(r[j][e]), dreg[j][kScaled ? 0 : e]);
          if (m >= thr) cand = static_cast<unsigned>(k0 + 2 * (j * NT + t) + e);
        }
      }
    }
    const unsigned wmin = __reduce_min_sync(0xffffffffu, cand);
    if (wmin == kNoneC) {
      if (lane == 0) s_u[warp] = kNoneC;
    } else if (cand == wmin) {
#pragma unroll
      for (int j = 0; j < EP; ++j) {
        *reinterpret_cast<double2*>(&s_dump[warp][2 * j]) = make_double2(r[j][0], r[j][1]);
        if constexpr (!kScaled)
          *reinterpret_cast<double2*>(&s_dumpd[warp][2 * j]) = make_double2(dreg[j][0], dreg[j][1]);
      }
      const int loc = static_cast<int>(cand) - k0;
      const int jj = (loc / 2 - t) / NT;
      const int ee = loc & 1;
      s_u[warp] = cand;
      s_r[warp] = s_dump[warp][2 * jj + ee];
      s_d[warp] = kScaled ? a.D[cand] : s_dumpd[kScaled ? 0 : warp][2 * jj + ee];
    }
    __syncthreads();
    if (warp == 0) {
      const unsigned su = lane < NW ? s_u[lane] : kNoneC;
      const unsigned cu = __reduce_min_sync(0xffffffffu, su);
      const int cw = cu == kNoneC ? 0 : __ffs(__ballot_sync(0xffffffffu, su == cu)) - 1;
      const double rv = cu == kNoneC ? 0.0 : s_r[cw];
      const double dv = cu == kNoneC ? 0.0 : s_d[cw];
      if (lane < CS) {
        const unsigned dst = peer_addr(&s_xb[par][rank][0], lane);
        const unsigned bar = peer_addr(&s_xbar[1][par], lane);
        push16(dst, bar, cu, 0u, lo32(rv), hi32(rv));
        push16(dst + 16, bar, lo32(dv), hi32(dv), 0u, 0u);
      }
      if (lane == 0) mbar_arrive_expect_tx(&s_xbar[1][par], CS * 32);
    }
    mbar_wait_acq_cluster(&s_xbar[1][par], xpar);
    unsigned u = kNoneC;
    double ru = 0.0, du = 0.0;
#pragma unroll
    for (int p = 0; p < CS; ++p) {
      const uint4 v0 = s_xb[par][p][0];
      if (v0.x < u) {
        const uint4 v1 = s_xb[par][p][1];
        u = v0.x;
        ru = mk_double(v0.z, v0.w);
        du = mk_double(v1.x, v1.y);
      }
    }
    FASE_ASSERT(u < static_cast<unsigned>(K));
    const double p = kScaled ? mul_rn(ru, du) : mul_rn(ru, mul_rn(du, du));
    const double c = mul_rn(a.gamma, p);
    if (rank == 0 && t == 0) {
      sel[it] = static_cast<int32_t>(u);
      proj[it] = p;
      coef[it] = c;
    }

    // ---- rank-1 update of this slice fused with the next running max
    best = kDead;
    barg = kNoneC;
    auto step = [&](int j, double2 g) {
      if constexpr (kScaled && (FASE_SCALED_LEAN & 4)) {  // as the one-CTA scaled kernel
        r[j][0] = __fma_rn(-c, g.x, r[j][0]);
        r[j][1] = __fma_rn(-c, g.y, r[j][1]);
      } else {
        r[j][0] = sub_rn(r[j][0], mul_rn(c, g.x));
        r[j][1] = sub_rn(r[j][1], mul_rn(c, g.y));
      }
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const double m = kScaled ? fabs(r[j][e]) : mul_rn(fabs(r[j][e]), dreg[j][kScaled ? 0 : e]);
        if (m > best) {
          best = m;
          barg = static_cast<unsigned>(k0 + 2 * (j * NT + t) + e);
        }
      }
    };
    const unsigned spar = static_cast<unsigned>(it) & 1u;
    if (u == guess) {
#pragma unroll
      for (int j = 0; j < EP; ++j) {
#pragma unroll
        for (int sg = 0; sg < kSeg; ++sg)
          if (j == sg * EP / kSeg) mbar_wait(&s_bar[sg], spar);
        step(j, s_row[j * NT + t]);
      }
      if constexpr (SYN > 0) {
#pragma unroll
        for (int i = 0; i < SYN; ++i)
          if (ls0 + t + i * NT < ls1) gacc[i] = add_rn(gacc[i], mul_rn(c, s_phi[t + i * NT]));
      }
    } else {
#pragma unroll
      for (int sg = 0; sg < kSeg; ++sg) mbar_wait(&s_bar[sg], spar);  // retire the copy
      const double* urow = a.G0 + static_cast<int64_t>(u) * a.ldg + k0 + 2 * t;
#pragma unroll
      for (int j = 0; j < EP; ++j) step(j, ldg2(urow + 2 * j * NT));
      if constexpr (SYN > 0) {
        const double* prow = syn.phi + static_cast<int64_t>(u) * syn.ldphi;
#pragma unroll
        for (int i = 0; i < SYN; ++i) {
          const int li = ls0 + t + i * NT;
          if (li < ls1) gacc[i] = add_rn(gacc[i], mul_rn(c, __ldg(prow + li)));
        }
      }
    }
  }
  (void)dead;
  if constexpr (SYN > 0) {
    double* o = syn.out + static_cast<int64_t>(b) * syn.ldout;
#pragma unroll
    for (int i = 0; i < SYN; ++i) {
      const int li = ls0 + t + i * NT;
      if (li < ls1) o[li] = gacc[i];
    }
  }
  cluster_sync_all();  // no CTA leaves while a peer may still push into it
}

using ClusterFn = void (*)(const fase_iterate_args, const fase_synth_fused);

struct ClusterShape {
  int nt, ep, cs;
  ClusterFn exact, scaled, scaled_syn;
};

#define FASE_CL(NT, EP, CS)                                                                  \
  {NT, EP, CS, fase_iterate_cluster_kernel<NT, EP, CS, false, 0>,                           \
   fase_iterate_cluster_kernel<NT, EP, CS, true, 0>, fase_iterate_cluster_kernel<NT, EP, CS, true, 1>}
// by capacity CS * 2 * NT * EP; a shape is used when its capacity holds K and
// fits the table rows' padding (fase_table_ld(K) >= capacity)
const ClusterShape kClusterShapes[] = {
    FASE_CL(64, 2, 4),   // 1024
    FASE_CL(96, 3, 4),   // 2304 (config 0)
    FASE_CL(128, 3, 4),  // 3072
    FASE_CL(192, 3, 4),  // 4608
    FASE_CL(128, 4, 8),  // 8192
};
#undef FASE_CL

}  // namespace

// Launches the cluster recursion when it applies (shared geometry, no R logs,
// a batch whose clusters fit on the SMs at once, a shape holding K within the
// table padding); returns 1 when it does not apply. FASE_CLUSTER=0 disables
// it (measurement), FASE_CLUSTER=N forces cluster size N where available.
int launch_iterate_cluster(const fase_iterate_args& a, const fase_synth_fused* syn, bool scaled,
                           cudaStream_t stream) {
  const char* env = getenv("FASE_CLUSTER");
  const int want = env && *env ? atoi(env) : -1;
  if (want == 0) return 1;
  if (a.chunk_count || a.R_log || a.R_out || a.ldd != 0 || a.compose) return 1;
  const ClusterShape* sh = nullptr;
  for (const ClusterShape& s : kClusterShapes) {
    const int cap = s.cs * 2 * s.nt * s.ep;
    if (cap >= a.K && a.ldg >= cap && (want < 0 || want == s.cs)) {
      sh = &s;
      break;
    }
  }
  // default: only where it measured faster than the one-CTA latency variants
  // (tools/probes/cluster_probe.py: K = 8192 over 8 CTAs 1.39 vs 1.51 us per
  // scaled iteration, 1.54 vs 1.81 exact; at K <= 4608 the two exchanges per
  // iteration cost more than the shorter row fetch saves: 1.45 vs 0.97 us)
  if (sh && want < 0 && sh->cs < 8) return 1;
  if (!sh) return 1;
  if (static_cast<int64_t>(a.B) * sh->cs > sm_count_cluster()) return 1;  // one wave, one CTA per SM
  if (syn && syn->n_lost > sh->cs * sh->nt) return 1;
  ClusterFn fn = scaled ? (syn ? sh->scaled_syn : sh->scaled) : sh->exact;
  fn<<<a.B * sh->cs, sh->nt, 0, stream>>>(a, syn ? *syn : fase_synth_fused{});
  return check_launch("fase_iterate (cluster)");
}

// synthesis capacity of the cluster path for (K, B), 0 when it does not apply
int cluster_synth_capacity(int K, int64_t ldg, int B) {
  const char* env = getenv("FASE_CLUSTER");
  const int want = env && *env ? atoi(env) : -1;
  if (want == 0) return 0;
  for (const ClusterShape& s : kClusterShapes) {
    const int cap = s.cs * 2 * s.nt * s.ep;
    if (cap >= K && ldg >= cap && (want < 0 || want == s.cs)) {
      if (want < 0 && s.cs < 8) return 0;  // (as launch_iterate_cluster's default)
      return static_cast<int64_t>(B) * s.cs <= sm_count_cluster() ? s.cs * s.nt : 0;
    }
  }
  return 0;
}

}  // namespace fase
