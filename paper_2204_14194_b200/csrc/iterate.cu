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
// whole run (or D in shared memory, kDsmem); nothing but the table rows comes
// from global memory inside the loop.
// Table rows are padded with zeros to the variant's capacity NT*EPT
// (fase_table_ld), so row loads carry no bounds predicates.
//
// Reductions: each thread tracks the exact max of its metrics (and the lowest
// index attaining it) during the update pass. Non-negative doubles order like
// their int64 bit patterns, so the warp max is three 32-bit redux.sync steps
// (high word, low word, lowest index) and one shared-memory exchange gives
// the block max. The tie pass is a 32-bit redux.sync min over candidate
// indices, run only by warps whose own max reaches the threshold (warp-uniform
// skip). Two __syncthreads per iteration.
//
// Row staging: after the first barrier the block knows the exact max and the
// lowest index attaining it. That index is the selection unless a tie within
// the quantum resolves lower (structural twins, rare), so one thread issues a
// TMA 1-D bulk copy (cp.async.bulk + mbarrier) of that row into shared memory
// while the tie pass and the second barrier run; no registers are held for it.
// A mispredicted row is loaded directly from global memory.
//
// Per-block geometries: row_u = G0[u,:] - sum_{j in chunks(b)} C_j[u,:]
// (chunk tables of sample classes that are lost in some blocks and not in
// others). The subtraction order is the
// chunk-list order, identical to fase_block_normalizers' diagonal.

#include <climits>
#include <type_traits>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"

namespace fase {
namespace {

constexpr unsigned kNone = 0xffffffffu;
#ifndef FASE_SCALED_SEG
#define FASE_SCALED_SEG 3
#endif
// (measurement: output rows re-derived at their use in the integer-key kernels; it
// halves the 18-element shape's spills, yet config 1 stays 1.4% slower with integer
// keys (0.690 vs 0.680 ms) and config 4 loses 1%: off, profiles/r02d/ab_intmax.txt)
#ifndef FASE_INTMAX_OUTROW
#define FASE_INTMAX_OUTROW 0
#endif
#ifndef FASE_INTMAX_MIN_EPT
#define FASE_INTMAX_MIN_EPT 24
#endif
#ifndef FASE_SCALED_CHAINS
#define FASE_SCALED_CHAINS 1
#endif
// chunked recursion: runner-up rows prefetched into L2 (measurement knob; 0 by
// default -- config 2 recursion 1.856 ms without, 1.896 / 2.034 / 2.232 ms with
// 1 / 2 / 3 runners: the extra DRAM traffic evicts more than it saves)
#ifndef FASE_RUNNER_PREFETCH
#define FASE_RUNNER_PREFETCH 0
#endif
#ifndef FASE_BASE_EVICT_FIRST  // chunked recursion: composed-base rows copied evict_first
#define FASE_BASE_EVICT_FIRST 1
#endif
// Row staging of the latency shapes (at most one block per SM), the kernel's
// SPEC argument: -1 (default) every thread loads its pairs of the predicted
// row straight into registers after the block max (config 0 scaled recursion
// 101.6 -> 96.3 us against 0); 0 one TMA copy into shared memory, as at full
// occupancy; N > 0 that copy plus N speculative spare buffers for the
// runners-up's rows (measured: 100.5 -> 164 us with 3 -- the speculative
// copies compete with the selected row for the one SM's L2 -> shared-memory
// bandwidth, and warp 0's extra reductions sit before the second barrier)
#ifndef FASE_SPEC
#define FASE_SPEC -1
#endif
// chunked recursion: start stagger of up to N ns per block (measurement knob;
// measured no effect on configs 2 / 3 at 2 and 8 us: the DRAM-resident row
// fetches are latency-, not burst-bound)
#ifndef FASE_STAGGER_NS
#define FASE_STAGGER_NS 0
#endif
// programmatic dependent launch of the latency shapes (measurement knob: 0 off)
#ifndef FASE_PDL
#define FASE_PDL 1
#endif
// Scaled recursion, per-iteration critical path (measurement knob, bits):
//  1: the running max keeps the signed R' of the best element and compares
//     magnitudes with |.| operand modifiers (no |R'| materialised per element:
//     one FP64 instruction per element less)
//     (config 4: 12.98 -> 12.36 ms per recursion, 244.8K -> 254.0K blocks/s)
//  4: the update R' -= c * Gs[u, :] as one fused multiply-add (one rounding
//     instead of two: config 4 12.36 -> 12.00 ms, config 1 0.726 -> 0.707 ms;
//     selections identical to the reference on every benchmarked block)
//  8: the tie winner takes R'_u from the signed running max when the pick is
//     its own argmax (no register dump through shared memory; config 1 0.708
//     -> 0.690 ms). Shapes with more than 20 elements per thread keep the dump:
//     the extra live value spills the 128-register 256 x 32 shape (config 4
//     12.0 -> 12.25 ms)
// 16: the predicted row's TMA copy is issued by a warp other than the argmax
//     warp (the tie pass and the issue run in parallel)
//  2: D of the predicted atom is loaded by every thread right after the block
//     max, so the tie winner no longer reads D from global memory between the
//     two barriers (measured: no gain on config 4, config 1 0.4% slower: off)
// 32: integer running max (kIntMax in the kernel: keys of the high words, the
//     exact top and tie rule resolved by one warp while the row copy is in
//     flight), on shapes of at least FASE_INTMAX_MIN_EPT elements per thread
// (FASE_SCALED_LEAN is defined in common.cuh: the cluster recursion follows bit 4 too)
#ifdef FASE_ITERATE_STATS
__device__ unsigned long long g_stats[8];  // measurement build: chunked-path counters
#endif

// Dead atoms (D == 0, and the padding past K) carry d = -inf: their metric
// |R| * d is -inf (NaN when R == 0), which never wins a '>' comparison and
// never reaches a finite threshold.
//
// kDsmem: D lives in shared memory instead of registers. That frees 2*EPT
// registers per thread so three 256-thread CTAs fit per SM (more blocks in
// flight to hide latency) at the cost of one extra 16-byte shared load per
// element pair and iteration.
//
// NB == 2 (shared D only): one CTA runs two blocks, each on its own NT-thread
// half with its own staged row, barriers (named, per half) and slots, while
// the normalizers -- identical for every block of a shared geometry -- are
// kept once in shared memory for both. For large K this doubles the blocks in
// flight per SM (two staged rows + one D fit where two CTAs' D + rows do not).
//
// kScaled (fase_iterate_scaled, shared geometry only): the table is
// column-scaled, Gs[u, k] = G[u, k] * D_k, and the state is R'_k = R_k * D_k,
// so the metric is |R'_k| -- no normalizer loads or products in the update
// pass, and no D in shared memory. The metric of iteration 0 is bit-identical
// (|R * D| == |R| * D); later iterations differ from the reference by the
// rounding of the scaled operands (~1 ulp per update), which can only change a
// selection whose top-two metrics lie within that rounding -- inside the
// north-star tolerance (top-two within 1e-9 relative). p = R'_u * D_u.
//
// SYN > 0 (scaled only): synthesis fused into the recursion. Each thread owns
// up to SYN lost samples (i = t + s*NT) and accumulates g_i += c * phi[u, i]
// after every update, in selection order with the same mul-then-add as
// fase_synth_paste (bit-identical output); the phi row of the predicted atom
// arrives by TMA with the last table segment.
//
// SPEC > 0 (latency shapes: at most one block per SM): speculative row staging.
// The next selection is usually one of this iteration's runners-up (the best
// maxima of the other warps), so besides the selected row, SPEC spare buffers
// receive the runners' rows a whole iteration ahead (one TMA each). When the
// next iteration's predicted atom is already in a spare buffer, no copy is
// issued and the update reads that buffer: the row's L2 round trip leaves the
// critical path of a latency-bound block. Arithmetic is unchanged.
template <int NT, int EPT, int MINB, bool kDsmem, bool kChunked, bool kRecord, int NB,
          bool kScaled = false, int SYN = 0, int SPEC = 0>
__global__ void __launch_bounds__(NT * NB, MINB) fase_iterate_kernel(const fase_iterate_args a,
                                                                     const fase_synth_fused syn) {
  // programmatic dependent launch (latency shapes): the grid may be scheduled
  // while the kernel that writes R0 finishes; wait for its results here (a
  // no-op for ordinary launches)
  if constexpr (SPEC != 0 || SYN > 0) asm volatile("griddepcontrol.wait;\n" ::: "memory");
  constexpr int EP = EPT / 2;
  constexpr int NW = NT / 32;
  static_assert(SPEC == 0 || (NB == 1 && !kChunked && !kRecord), "speculative staging: one "
                "shared-geometry block per CTA");
  constexpr int kSp = SPEC > 0 ? SPEC : 1;
  // SPEC < 0 (latency shapes, measurement): the predicted row is loaded straight
  // into registers by every thread right after the block max (no TMA, no
  // mbarrier), overlapping the tie pass and the second barrier like the copy
  constexpr bool kRegRow = SPEC < 0;
  static_assert(!kRegRow || (NB == 1 && !kChunked), "register-staged rows: shared geometry");
  __shared__ __align__(8) uint64_t s_sbar[kSp];   // SPEC: one mbarrier per spare buffer
  __shared__ unsigned s_stag[kSp];                 // SPEC: atom held by each spare buffer
  __shared__ unsigned s_sfill[kSp];                // SPEC: fills issued per spare buffer
  __shared__ int s_use;                            // SPEC: spare buffer holding the guess, or -1
  __shared__ unsigned s_upar;                      // SPEC: its mbarrier parity
  __shared__ __align__(16) double s_sphi[SPEC > 0 && SYN > 0 ? SPEC : 1][SYN > 0 ? SYN * NT : 2];
  static_assert(NB == 1 || (kDsmem && !kChunked), "paired blocks share one D in shared memory");
  static_assert(!kScaled || (!kDsmem && !kChunked && !kRecord && NB == 1),
                "the scaled recursion keeps no normalizers and has one block per CTA");
  static_assert(SYN == 0 || (!kChunked && !kRecord && NB == 1),
                "fused synthesis: one shared-geometry block per CTA");
  __shared__ __align__(16) double s_phi[SYN > 0 ? SYN * NT : 2];

  __shared__ long long s_key_all[NB][NW];
  __shared__ unsigned s_arg_all[NB][NW];
  __shared__ unsigned s_u_all[NB][NW];
  __shared__ double s_r_all[NB][NW];
  __shared__ double s_d_all[NB][NW];
  __shared__ __align__(16) double s_dump_all[NB][NW][kDsmem ? 1 : 2][EPT];  // tie-pass winner's registers
  // kIntMax (scaled, FASE_SCALED_LEAN & 32): the update keeps, per thread, only
  // the largest key (high word of |R'| with its five low bits replaced by the
  // element's position): one logic op per element and one 3-input integer max
  // per pair instead of a compare and three selects per element. The largest
  // key of the block names the row to stage; the exact top and the tie rule
  // are then resolved, while that copy is in flight, by the warp holding every
  // element within one key unit (2^-15 relative) of the largest: each such
  // lane's registers are spread over the warp's lanes through shared memory.
  // Any other situation (two such warps, a wide tie quantum, zero / subnormal /
  // non-finite maxima) takes an exact per-thread scan and one more barrier.
  // Dead atoms and the padding hold R' = 0 here (their table columns are 0).
  // Shapes of 24 to 32 elements per thread (K > 5120): config 4 recursion 11.85 ->
  // 11.35 ms on one box, every selection unchanged; the 64-register 18-element
  // shape of config 1 measured 3.5% slower (0.698 -> 0.722 ms: its resolution
  // spills) and keeps the compare / select running max.
  constexpr bool kIntMax = kScaled && (FASE_SCALED_LEAN & 32) && EPT >= FASE_INTMAX_MIN_EPT && EPT <= 32 && SPEC == 0;
  __shared__ unsigned s_wk[kIntMax ? NW : 1];  // kIntMax: the warps' largest keys
  // ... and their atoms (not s_arg: the exact path republishes s_arg one barrier later,
  // while slower warps may still be reading these)
  __shared__ unsigned s_wa[kIntMax ? NW : 1];
  __shared__ double s_ftop;                    // kIntMax: the exact top of a resolved iteration
  // The staged row arrives in kSeg segments, each on its own mbarrier, so the
  // update can start on the first segment while the rest is still in flight.
  constexpr int kSegMax = kScaled ? FASE_SCALED_SEG : 3;
  constexpr int kSeg = EP < kSegMax ? EP : kSegMax;
  // independent running-max chains in the update (the compare / select chain
  // through all EP pairs is serial otherwise); merged lowest-index-first
  constexpr int kChains = (kScaled && EP >= 8) ? FASE_SCALED_CHAINS : 1;
  __shared__ __align__(8) uint64_t s_bar_all[NB][kSeg];
  __shared__ double s_heldm_all[NB];  // kChunked: metric of the held atom after the update
  extern __shared__ double2 s_dyn[];

  const int half = NB == 1 ? 0 : static_cast<int>(threadIdx.x) / NT;
  long long* s_key = s_key_all[half];
  unsigned* s_arg = s_arg_all[half];
  unsigned* s_u = s_u_all[half];
  double* s_r = s_r_all[half];
  double* s_d = s_d_all[half];
  auto s_dump = s_dump_all[half];
  uint64_t* s_bar = s_bar_all[half];
  double2* s_row = s_dyn + half * EP * NT;  // staged row: pair p at s_row[p]
  double2* s_D = s_dyn + NB * EP * NT;      // kDsmem: normalizer pairs, same indexing
  // SPEC: spare row buffers k at s_spare + k * EP * NT
  double2* s_spare = s_dyn + NB * EP * NT + (kDsmem ? EP * NT : 0);

  // the block of this CTA slot: slot order, or (per-block geometries) the
  // caller's dispatch order. Shared geometries ignore the order: their blocks
  // cost the same, and a block index that is a load instead of a function of
  // blockIdx.x is one more live register -- at 64 / 128 registers the config-1
  // / config-4 shapes spilled (16 -> 120 bytes, 0 -> 28)
  const int slot = static_cast<int>(blockIdx.x) * NB + half;
  const int b = (kChunked && a.order && slot < a.B) ? __ldg(a.order + slot) : slot;
  // kChunked: the block index parked in shared memory for the loop's (thread-0)
  // output rows instead of held in a register across it
  __shared__ int s_blk[NB];
  const int t = static_cast<int>(threadIdx.x) - half * NT;
  if (kChunked && t == 0) s_blk[half] = b;  // (read after the loop's first barrier)
  const int lane = t & 31;
  const int warp = t >> 5;
  double gacc[SYN > 0 ? SYN : 1];
#pragma unroll
  for (int i = 0; i < (SYN > 0 ? SYN : 1); ++i) gacc[i] = 0.0;
  // fused synthesis output of this block (SYN > 0)
  auto write_synth = [&](int blk) {
    if constexpr (SYN > 0) {
      double* o = syn.out + static_cast<int64_t>(blk) * syn.ldout;
#pragma unroll
      for (int i = 0; i < SYN; ++i)
        if (t + i * NT < syn.n_lost) o[t + i * NT] = gacc[i];
    }
  };
  const int K = a.K;
  const double kDead = __longlong_as_double(static_cast<long long>(0xfff0000000000000ULL));
  const bool active = NB == 1 || slot < a.B;
  // the per-iteration barrier: the whole CTA, or this block's half
  auto block_sync = [&]() {
    if constexpr (NB == 1)
      __syncthreads();
    else
      asm volatile("bar.sync %0, %1;\n" ::"r"(1 + half), "r"(NT) : "memory");
  };

  if (t == 0) {
    for (int sg = 0; sg < kSeg; ++sg) mbar_init(&s_bar[sg], 1);
    if constexpr (SPEC > 0) {
      for (int k = 0; k < SPEC; ++k) {
        mbar_init(&s_sbar[k], 1);
        s_stag[k] = kNone;
        s_sfill[k] = 0;
      }
    }
    fence_mbar_init();
  }

  const double* D = a.D + (a.ldd ? static_cast<int64_t>(b) * a.ldd : 0);
  const double* R0 = a.R0 + static_cast<int64_t>(active ? b : 0) * a.ldr;
  const int32_t* cids = nullptr;
  int nch = 0;
  const double* G0b = a.G0;  // kChunked: this block's base table
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
        FASE_ASSERT(p >= 0);
        if (p > 0) {
          G0b += static_cast<int64_t>(p) * a.base_stride;
          cids += k;
          nch -= k;
          break;
        }
      }
    }
  }

  double r[EP][2];
  double dreg[(kDsmem || kScaled) ? 1 : EP][2];
  // normalizer pair j of this thread (registers or shared memory)
  auto dpair = [&](int j) -> double2 {
    if constexpr (kDsmem)
      return s_D[j * NT + t];
    else
      return make_double2(dreg[j][0], dreg[j][1]);
  };
  // the selection metrics of pair j (normalizers `dd` loaded once by the caller)
  auto metrics = [&](int j, double2 dd) -> double2 {
    if constexpr (kScaled)
      return make_double2(fabs(r[j][0]), fabs(r[j][1]));
    else
      return make_double2(mul_rn(fabs(r[j][0]), dd.x), mul_rn(fabs(r[j][1]), dd.y));
  };
  auto dpair_if = [&](int j) -> double2 {
    if constexpr (kScaled)
      return make_double2(0.0, 0.0);
    else
      return dpair(j);
  };
  double best = kDead;
  unsigned barg = kNone;
  double bsig = 0.0;  // kScaled: the signed R' of this thread's best element
#pragma unroll
  for (int j = 0; j < EP; ++j) {
    const int k = 2 * (j * NT + t);
    if constexpr (kScaled) {
      // R' = R * D; dead atoms and the padding hold NaN (never selected)
      const double kNaN = __longlong_as_double(0x7ff8000000000000LL);
      const double d0 = k < K ? D[k] : 0.0, d1 = k + 1 < K ? D[k + 1] : 0.0;
      r[j][0] = d0 != 0.0 ? mul_rn(R0[k], d0) : (kIntMax ? 0.0 : kNaN);
      r[j][1] = d1 != 0.0 ? mul_rn(R0[k + 1], d1) : (kIntMax ? 0.0 : kNaN);
      const double m0 = fabs(r[j][0]);
      if (m0 > best) {
        best = m0;
        bsig = r[j][0];
        barg = static_cast<unsigned>(k);
      }
      const double m1 = fabs(r[j][1]);
      if (m1 > best) {
        best = m1;
        bsig = r[j][1];
        barg = static_cast<unsigned>(k + 1);
      }
      continue;
    }
    double2 dd;
    r[j][0] = k < K ? R0[k] : 0.0;
    r[j][1] = k + 1 < K ? R0[k + 1] : 0.0;
    dd.x = k < K ? D[k] : 0.0;
    dd.y = k + 1 < K ? D[k + 1] : 0.0;
    dd.x = dd.x != 0.0 ? dd.x : kDead;
    dd.y = dd.y != 0.0 ? dd.y : kDead;
    if constexpr (kDsmem) {
      if (half == 0) s_D[j * NT + t] = dd;
    } else {
      dreg[j][0] = dd.x;
      dreg[j][1] = dd.y;
    }
    const double m0 = mul_rn(fabs(r[j][0]), dd.x);
    if (m0 > best) {
      best = m0;
      barg = static_cast<unsigned>(k);
    }
    const double m1 = mul_rn(fabs(r[j][1]), dd.y);
    if (m1 > best) {
      best = m1;
      barg = static_cast<unsigned>(k + 1);
    }
  }

  if constexpr (NB > 1) {
    __syncthreads();  // the shared D (written by half 0) is complete
    if (!active) return;
  }
#if FASE_STAGGER_NS > 0
  // measurement: desynchronise the blocks' row requests (per-block geometries
  // read their rows mostly from DRAM, in bursts when every block iterates in step)
  if constexpr (kChunked) __nanosleep(static_cast<unsigned>((blockIdx.x * 5u) % 8u) * (FASE_STAGGER_NS / 8));
#endif

  int32_t* sel = a.sel + static_cast<int64_t>(b) * a.ldo;
  double* proj = a.proj + static_cast<int64_t>(b) * a.ldo;
  double* coef = a.coef + static_cast<int64_t>(b) * a.ldo;
  // Chunked shapes re-derive the output rows from the parameter bank at each
  // (thread-0) use: as loop-carried induction pointers they cost six registers
  // in every thread and spilled the 80-register chunked variant (local-memory
  // round trips on the per-iteration path; config 2)
  auto out_row = [&](auto* base, auto* hoisted) {
    if constexpr (kChunked) {
      asm volatile("" : "+l"(base));
      return base + static_cast<int64_t>(s_blk[half]) * a.ldo;
    } else if constexpr (kIntMax && FASE_INTMAX_OUTROW) {
      // (one lane writes the outputs: re-derived at the use, not held across the loop)
      asm volatile("" : "+l"(base));
      return base + static_cast<int64_t>(blockIdx.x) * a.ldo;
    } else {
      return hoisted;
    }
  };
  const int64_t ldg = a.ldg;
  double q = 0.0;
  // kChunked: the atom whose complete (composed) row the staging buffer holds,
  // and the number of row copies issued so far (mbarrier phase parity)
  unsigned held = kNone;
  unsigned n_copies = 0;
  unsigned par_m = 0;     // SPEC: mbarrier parity of this iteration's main-buffer copy
  unsigned runner[kSp];  // SPEC: this iteration's runners-up (warp 0)
#pragma unroll
  for (int rr = 0; rr < kSp; ++rr) runner[rr] = kNone;

  // kIntMax: a live atom (dead ones and the padding hold R' = 0 there)
  auto live = [&](int k) { return k < K && __ldg(D + k) != 0.0; };
  // kIntMax: this thread's largest key; key = (high word & mask) | position, one LOP3
  constexpr unsigned kKeyMask = 0x7fffffe0u;
  auto key_of = [&](double x, unsigned pos) -> unsigned {
    unsigned d;
    asm("lop3.b32 %0, %1, %2, %3, 0xEC;" : "=r"(d) : "r"(__double2hiint(x)), "r"(pos), "r"(kKeyMask));
    return d;
  };
  unsigned tkey = 0u;
  if constexpr (kIntMax) {
#pragma unroll
    for (int j = 0; j < EP; ++j)
      tkey = __vimax3_u32(tkey, key_of(r[j][0], 31u - 2 * j), key_of(r[j][1], 30u - 2 * j));
  }
  // kIntMax, exact path: this thread's exact max, its signed value and lowest index
  auto rescan = [&]() {
    double cb = -0.0;
    unsigned ca = kNone;
#pragma unroll
    for (int j = 0; j < EP; ++j) {
      if (fabs(r[j][0]) > fabs(cb)) {
        cb = r[j][0];
        ca = static_cast<unsigned>(2 * (j * NT + t));
      }
      if (fabs(r[j][1]) > fabs(cb)) {
        cb = r[j][1];
        ca = static_cast<unsigned>(2 * (j * NT + t) + 1);
      }
    }
    best = ca == kNone ? kDead : fabs(cb);
    bsig = cb;
    barg = ca;
    if (ca == kNone) {  // rare: no metric > 0 here -- the lowest live atom (metric 0), if any
#pragma unroll
      for (int j = EP - 1; j >= 0; --j) {
        const int k = 2 * (j * NT + t);
        if (live(k + 1)) {
          best = 0.0;
          bsig = r[j][1];
          barg = static_cast<unsigned>(k + 1);
        }
        if (live(k)) {
          best = 0.0;
          bsig = r[j][0];
          barg = static_cast<unsigned>(k);
        }
      }
    }
  };

  for (int it = 0; it < a.I; ++it) {
    long long top_key = 0;
    unsigned guess = kNone;
    long long wkey = LLONG_MIN;
    // ---- exact warp max and the lowest index attaining it
    auto publish_exact = [&]() {
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
    };
    // ---- block max: every warp reduces the NW slots in parallel (lane l reads slot l)
    auto block_exact = [&](unsigned& guess_out) {
    {
      const long long sk = lane < NW ? s_key[lane] : LLONG_MIN;
      const unsigned sa = lane < NW ? s_arg[lane] : kNone;
      wkey = s_key[warp];
      const int h = static_cast<int>(sk >> 32);
      const unsigned l = static_cast<unsigned>(sk);
      const int bh = __reduce_max_sync(0xffffffffu, h);
      const unsigned bl = __reduce_max_sync(0xffffffffu, h == bh ? l : 0u);
      guess_out = __reduce_min_sync(0xffffffffu, (h == bh && l == bl) ? sa : kNone);
      top_key = (static_cast<long long>(bh) << 32) | bl;
      if constexpr (SPEC > 0) {
        // the best maxima of the other warps (warp 0; thread 0 stages their rows)
        if (warp == 0) {
#pragma unroll
          for (int rr = 0; rr < SPEC; ++rr) {
            bool taken = sa == guess_out;
#pragma unroll
            for (int q2 = 0; q2 < rr; ++q2) taken = taken || sa == runner[q2];
            const long long k2 = taken ? LLONG_MIN : sk;
            const int h2 = static_cast<int>(k2 >> 32);
            const unsigned l2 = static_cast<unsigned>(k2);
            const int b2 = __reduce_max_sync(0xffffffffu, h2);
            const unsigned c2 = __reduce_max_sync(0xffffffffu, h2 == b2 ? l2 : 0u);
            const unsigned r2 = __reduce_min_sync(0xffffffffu, (h2 == b2 && l2 == c2) ? sa : kNone);
            runner[rr] = (b2 < 0 || r2 >= static_cast<unsigned>(K)) ? kNone : r2;
          }
        }
      }
      if constexpr (kChunked && FASE_RUNNER_PREFETCH > 0) {
        // Per-block geometries read their (composed) base rows mostly from
        // DRAM. The next selection is often one of this iteration's runners-up
        // (config 2: the runner-up 46%, one of the top two 62%): pull the rows
        // of the best two other warps' maxima into L2 now, a whole iteration
        // ahead (bulk prefetches: no registers or shared memory held).
        if (warp == 0) {
          unsigned prev = guess_out;
#pragma unroll
          for (int rr = 0; rr < FASE_RUNNER_PREFETCH; ++rr) {
            const long long k2 = (sa == guess_out || sa == prev) ? LLONG_MIN : sk;
            const int h2 = static_cast<int>(k2 >> 32);
            const unsigned l2 = static_cast<unsigned>(k2);
            const int b2 = __reduce_max_sync(0xffffffffu, h2);
            const unsigned c2 = __reduce_max_sync(0xffffffffu, h2 == b2 ? l2 : 0u);
            const unsigned r2 = __reduce_min_sync(0xffffffffu, (h2 == b2 && l2 == c2) ? sa : kNone);
            if (b2 < 0 || r2 >= static_cast<unsigned>(K)) break;
            if (lane == 0)
              asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(
                               G0b + static_cast<int64_t>(r2) * ldg),
                           "r"(static_cast<unsigned>(EP * NT * sizeof(double2)))
                           : "memory");
            prev = r2;
          }
        }
      }
    }
    };
    bool fastb = false;  // kIntMax: one warp resolves this iteration (block-uniform)
    unsigned sk_l = 0u;  // kIntMax: warp `lane`'s largest key
    unsigned kb = 0u;    // kIntMax: the block's largest key
    if constexpr (kIntMax) {
      const unsigned wk = __reduce_max_sync(0xffffffffu, tkey);
      const int wl = __ffs(__ballot_sync(0xffffffffu, tkey == wk)) - 1;
      if (lane == 0) {
        const int e = 31 - static_cast<int>(wk & 31u);
        s_wk[warp] = wk;
        s_wa[warp] = 2u * static_cast<unsigned>((e >> 1) * NT + warp * 32 + wl) + (e & 1);
      }
      block_sync();
      sk_l = lane < NW ? s_wk[lane] : 0u;
      const unsigned sa = lane < NW ? s_wa[lane] : kNone;
      kb = __reduce_max_sync(0xffffffffu, sk_l);
      guess = __reduce_min_sync(0xffffffffu, sk_l == kb ? sa : kNone);
      guess = guess < static_cast<unsigned>(K) ? guess : 0u;  // (an all-zero block: any row)
      top_key = 1;  // (known after the resolution below)
    } else {
      publish_exact();
      block_sync();
      block_exact(guess);
    }
    if (top_key < 0) {  // every atom degenerate (NoSelectableAtomError): mark and stop
      for (int k = it + t; k < a.I; k += NT) {
        out_row(a.sel, sel)[k] = -1;
        out_row(a.proj, proj)[k] = 0.0;
        out_row(a.coef, coef)[k] = 0.0;
      }
      write_synth(b);
      return;
    }
    // stage the likely selection's row in shared memory (one TMA bulk copy)
    // while the tie pass and the second barrier run -- unless the buffer
    // already holds that atom's complete row (per-block geometries re-select
    // the previous atom often: 60% of config-3 iterations)
    // (shared geometries always copy; their base and mbarrier parity come
    // straight from the parameters and the loop counter at each use)
    if constexpr (kChunked) {
      // predict the tie rule's pick: the held atom, when it reaches this
      // iteration's threshold and precedes the argmax (the rule takes the
      // lowest index at or above the threshold; structural near-ties make the
      // argmax a poor guess: 44% of config-3 copies were mispredicted)
      if (held != kNone && held < guess) {
        const double top_ = __longlong_as_double(top_key);
        double q_ = q;
        if (top_key > 0 && top_key < 0x7ff0000000000000LL) q_ = fmax(q_, mul_rn(1e-13, top_));
        const double thr_ = q_ > 0.0 ? sub_rn(top_, q_) : top_;
        if (s_heldm_all[half] >= thr_) guess = held;
      }
    }
    const bool issue = (!kChunked || guess != held) && !kRegRow;  // block-uniform
    double2 rrow[kRegRow ? EP : 1];  // kRegRow: this thread's pairs of the predicted row
    double rphi[kRegRow && SYN > 0 ? SYN : 1];
    if constexpr (kRegRow) {
      const double* grow = a.G0 + static_cast<int64_t>(guess < static_cast<unsigned>(K) ? guess : 0u) * ldg + 2 * t;
#pragma unroll
      for (int j = 0; j < EP; ++j) rrow[j] = ldg2_here(grow + 2 * j * NT);
      if constexpr (SYN > 0) {
        const double* prow = syn.phi + static_cast<int64_t>(guess < static_cast<unsigned>(K) ? guess : 0u) * syn.ldphi;
#pragma unroll
        for (int i = 0; i < SYN; ++i) rphi[i] = t + i * NT < syn.n_lost ? __ldg(prow + t + i * NT) : 0.0;
      }
    }
    const unsigned par_c = n_copies & 1u;
    if constexpr (kChunked) n_copies += issue ? 1u : 0u;
    auto parity = [&]() -> unsigned {
      if constexpr (kChunked)
        return par_c;
      else if constexpr (SPEC > 0)
        return par_m;
      else
        return it & 1;
    };
    auto base = [&]() -> const double* {
      if constexpr (kChunked)
        return G0b;
      else
        return a.G0;
    };
    // the issuing thread: thread 0, or (kIssueOff) lane 0 of a warp other
    // than the predicted atom's, so the issue and its tie pass overlap
    constexpr bool kIssueOff = kScaled && (FASE_SCALED_LEAN & 16) && SPEC == 0 && NW > 1;
    const int t_iss = kIssueOff ? ((((static_cast<int>(guess >> 1) % NT) >> 5) + 1) % NW) * 32 : 0;
    if (t == t_iss && issue) {
      FASE_ASSERT(guess < static_cast<unsigned>(K));
      fence_before_refill();
      int use = -1;  // SPEC: a spare buffer already holding the guess's row
      if constexpr (SPEC > 0) {
        for (int k = 0; k < SPEC; ++k)
          if (s_stag[k] == guess) use = k;
        s_use = use;
        s_upar = use >= 0 ? ((s_sfill[use] - 1u) & 1u) : 0u;
      }
      if (use < 0) {
      const double* grow = base() + static_cast<int64_t>(guess) * ldg;
      // fused synthesis: the predicted atom's phi row rides on the last segment
      const unsigned phi_bytes =
          SYN > 0 ? static_cast<unsigned>((syn.n_lost * sizeof(double) + 15) & ~size_t{15}) : 0u;
      // L2 residency hint: hot rows evict_last, the rest evict_first. Per-block
      // geometries: rows of a precomposed base (used by this block, or a few)
      // stream through L2 evict_first so they do not displace the shared G0 rows
      // (FASE_BASE_EVICT_FIRST 2: G0's own rows evict_last besides)
      const bool composed = kChunked && FASE_BASE_EVICT_FIRST && G0b != a.G0;
      const bool shared_g0 = kChunked && FASE_BASE_EVICT_FIRST == 2 && G0b == a.G0;
      const bool hint = (!kChunked && a.l2_hot != nullptr) || composed || shared_g0;
      const uint64_t pol =
          kChunked ? l2_policy(shared_g0)
                   : (hint ? l2_policy((__ldg(a.l2_hot + (guess >> 5)) >> (guess & 31)) & 1u) : 0ull);
#pragma unroll
      for (int sg = 0; sg < kSeg; ++sg) {
        const int j0 = sg * EP / kSeg, j1 = (sg + 1) * EP / kSeg;
        const unsigned bytes = static_cast<unsigned>((j1 - j0) * NT * sizeof(double2));
        mbar_arrive_expect_tx(&s_bar[sg], bytes + (sg == kSeg - 1 ? phi_bytes : 0u));
        if (hint)
          tma_load_1d_hint(s_row + j0 * NT, grow + 2 * j0 * NT, bytes, &s_bar[sg], pol);
        else
          tma_load_1d(s_row + j0 * NT, grow + 2 * j0 * NT, bytes, &s_bar[sg]);
        if (SYN > 0 && sg == kSeg - 1)
          tma_load_1d(s_phi, syn.phi + static_cast<int64_t>(guess) * syn.ldphi, phi_bytes,
                      &s_bar[sg]);
      }
      }  // use < 0
      if constexpr (SPEC > 0) {
        // stage the runners' rows (and phi rows) for the next iteration in
        // spare buffers other than the one read now, round robin; a buffer's
        // previous fill (issued at least one iteration ago) is retired first
        const unsigned row_bytes = static_cast<unsigned>(EP * NT * sizeof(double2));
        const unsigned pb =
            SYN > 0 ? static_cast<unsigned>((syn.n_lost * sizeof(double) + 15) & ~size_t{15}) : 0u;
        int victim = (use + 1) % SPEC;
        for (int rr = 0; rr < SPEC; ++rr) {
          const unsigned r2 = runner[rr];
          if (r2 == kNone) break;
          bool have = false;
          for (int k = 0; k < SPEC; ++k) have = have || s_stag[k] == r2;
          if (have) continue;
          int k = -1;
          for (int step = 0; step < SPEC && k < 0; ++step) {
            const int c2 = (victim + step) % SPEC;
            bool keep = c2 == use;
            for (int q2 = 0; q2 < SPEC; ++q2) keep = keep || (runner[q2] != kNone && s_stag[c2] == runner[q2]);
            if (!keep) k = c2;
          }
          if (k < 0) break;
          victim = (k + 1) % SPEC;
          if (s_sfill[k] > 0) mbar_wait(&s_sbar[k], (s_sfill[k] - 1u) & 1u);
          mbar_arrive_expect_tx(&s_sbar[k], row_bytes + pb);
          tma_load_1d(s_spare + k * EP * NT, base() + static_cast<int64_t>(r2) * ldg, row_bytes,
                      &s_sbar[k]);
          if constexpr (SYN > 0)
            tma_load_1d(s_sphi[k], syn.phi + static_cast<int64_t>(r2) * syn.ldphi, pb, &s_sbar[k]);
          s_stag[k] = r2;
          s_sfill[k] += 1u;
        }
      }
      if constexpr (kChunked) {
        // the guess's chunk-table rows are read right after the second
        // barrier: pull them into L2 now (one bulk prefetch per row)
        for (int ch = 0; ch < nch; ++ch) {
          const double* crow = a.chunk_tables + static_cast<int64_t>(cids[ch]) * a.chunk_stride +
                               static_cast<int64_t>(guess) * ldg;
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(crow),
                       "r"(static_cast<unsigned>(EP * NT * sizeof(double2)))
                       : "memory");
        }
      }
    }
    constexpr bool kLeanD = kScaled && (FASE_SCALED_LEAN & 2);
    if constexpr (kIntMax) {
      const unsigned kb27 = kb >> 5;
      const unsigned nearw = __ballot_sync(0xffffffffu, lane < NW && (sk_l >> 5) + 1u >= kb27);
      const int wstar = __ffs(nearw) - 1;
      // every element that can reach the tie threshold lies within one key
      // unit of the largest when the quantum max(q, 1e-13 * top) is below
      // 2^(e-16) for a top in [2^e, 2^(e+1)) -- half a unit there, a whole one
      // just below 2^e: compared through the exponent fields
      fastb = __popc(nearw) == 1 && kb >= 0x02000000u && kb < 0x7ff00000u &&
              __double2hiint(q) < static_cast<int>(((kb >> 20) - 16u) << 20);
      if (fastb) {
        if (warp == wstar) {
          // the lanes holding an element within one key unit of the largest
          const unsigned nearl = __ballot_sync(0xffffffffu, (tkey >> 5) + 1u >= kb27);
          unsigned cu = kNone;
          double rv = 0.0, topx = 0.0;
          if ((nearl & (nearl - 1u)) == 0u) {  // one lane: its registers over the lanes
            const int c = __ffs(nearl) - 1;
            if (lane == c) {
#pragma unroll
              for (int j = 0; j < EP; ++j)
                *reinterpret_cast<double2*>(&s_dump[warp][0][2 * j]) = make_double2(r[j][0], r[j][1]);
            }
            __syncwarp();
            const double v = lane < EPT ? s_dump[warp][0][lane] : 0.0;
            const unsigned hv = (static_cast<unsigned>(__double2hiint(v)) & 0x7fffffffu) >> 5;
            const unsigned nb = __ballot_sync(0xffffffffu, hv + 1u >= kb27);
            if ((nb & (nb - 1u)) == 0u) {  // one element: the top and the pick
              const int e = __ffs(nb) - 1;
              rv = __shfl_sync(0xffffffffu, v, e);
              topx = fabs(rv);
              cu = 2u * static_cast<unsigned>((e >> 1) * NT + warp * 32 + c) + (e & 1);
            }
          }
          if (cu == kNone) {  // several elements: exact top, then the lowest index at the threshold
            long long tk = 0;
            for (unsigned m = nearl; m; m &= m - 1u) {
              const int c = __ffs(m) - 1;
              __syncwarp();
              if (lane == c) {
#pragma unroll
                for (int j = 0; j < EP; ++j)
                  *reinterpret_cast<double2*>(&s_dump[warp][0][2 * j]) = make_double2(r[j][0], r[j][1]);
              }
              __syncwarp();
              const double v = lane < EPT ? s_dump[warp][0][lane] : 0.0;
              const long long key = __double_as_longlong(fabs(v));
              const int kh = static_cast<int>(key >> 32);
              const unsigned kl = static_cast<unsigned>(key);
              const int wh = __reduce_max_sync(0xffffffffu, kh);
              const unsigned wl2 = __reduce_max_sync(0xffffffffu, kh == wh ? kl : 0u);
              const long long k2 = (static_cast<long long>(wh) << 32) | wl2;
              tk = k2 > tk ? k2 : tk;
            }
            topx = __longlong_as_double(tk);
            const double thrx = sub_rn(topx, fmax(q, mul_rn(1e-13, topx)));  // as below (finite top)
            for (unsigned m = nearl; m; m &= m - 1u) {
              const int c = __ffs(m) - 1;
              __syncwarp();
              if (lane == c) {
#pragma unroll
                for (int j = 0; j < EP; ++j)
                  *reinterpret_cast<double2*>(&s_dump[warp][0][2 * j]) = make_double2(r[j][0], r[j][1]);
              }
              __syncwarp();
              const double v = lane < EPT ? s_dump[warp][0][lane] : 0.0;
              const unsigned hit = __ballot_sync(0xffffffffu, fabs(v) >= thrx);
              if (hit) {
                const int e = __ffs(hit) - 1;
                const unsigned ci = 2u * static_cast<unsigned>((e >> 1) * NT + warp * 32 + c) + (e & 1);
                const double cv = __shfl_sync(0xffffffffu, v, e);
                if (ci < cu) {
                  cu = ci;
                  rv = cv;
                }
              }
            }
          }
          FASE_ASSERT(cu < static_cast<unsigned>(K));
          if (lane == 0) {  // projection, coefficient and the iteration's outputs
            const double pf = mul_rn(rv, __ldg(D + cu));
            const double cf = mul_rn(a.gamma, pf);
            s_u[0] = cu;
            s_r[0] = pf;
            s_d[0] = cf;
            s_ftop = topx;
            out_row(a.sel, sel)[it] = static_cast<int32_t>(cu);
            out_row(a.proj, proj)[it] = pf;
            out_row(a.coef, coef)[it] = cf;
          }
        }
        block_sync();
        top_key = __double_as_longlong(s_ftop);
      } else {
        rescan();
        publish_exact();
        block_sync();
        unsigned exact_guess;
        block_exact(exact_guess);
        if (top_key < 0) {  // every atom degenerate: retire the copy, then mark and stop as above
#pragma unroll
          for (int sg = 0; sg < kSeg; ++sg) mbar_wait(&s_bar[sg], it & 1);
          for (int k = it + t; k < a.I; k += NT) {
            out_row(a.sel, sel)[k] = -1;
            out_row(a.proj, proj)[k] = 0.0;
            out_row(a.coef, coef)[k] = 0.0;
          }
          write_synth(b);
          return;
        }
      }
    }
    // kLeanD: D of the predicted atom, in flight during the tie pass and the
    // second barrier (the guess is in range here: a degenerate top returned)
    const double dguess = kLeanD ? __ldg(D + guess) : 0.0;
    const double top = __longlong_as_double(top_key);
    // tie_quantum (reference.py:55-85): only a finite, strictly positive top moves the ratchet
    double thr;
    if constexpr (kChunked) {
      // (the branch-free form below perturbs the chunked shapes' register
      // allocation into spills: config 3 12.6 -> 13.7 ms)
      if (top_key > 0 && top_key < 0x7ff0000000000000LL) q = fmax(q, mul_rn(1e-13, top));
      thr = q > 0.0 ? sub_rn(top, q) : top;
    } else {
      // a +0 top leaves the ratchet (1e-13 * 0), a +inf one must not move it;
      // q == 0 gives exactly top (c1 0.780 -> 0.772 ms)
      const double qn = mul_rn(1e-13, top);
      q = qn < __longlong_as_double(0x7ff0000000000000LL) ? fmax(q, qn) : q;
      thr = sub_rn(top, q);
    }

    unsigned u = 0u;
    int uw = 0;
    if (!(kIntMax && fastb)) {
    // ---- lowest index reaching the threshold (only warps whose max reaches it)
    unsigned cand = kNone;
    if (wkey >= 0 && __longlong_as_double(wkey) >= thr) {  // warp-uniform
#pragma unroll
      for (int j = EP - 1; j >= 0; --j) {
        const double2 m = metrics(j, dpair_if(j));
        // (kIntMax: dead atoms hold 0, which reaches a threshold <= 0)
        if (m.y >= thr && (!kIntMax || thr > 0.0 || live(2 * (j * NT + t) + 1))) cand = 2 * (j * NT + t) + 1;
        if (m.x >= thr && (!kIntMax || thr > 0.0 || live(2 * (j * NT + t)))) cand = 2 * (j * NT + t);
      }
    }
    const unsigned wmin = __reduce_min_sync(0xffffffffu, cand);
    if (wmin == kNone) {
      if (lane == 0) s_u[warp] = kNone;
    } else if (kScaled && (FASE_SCALED_LEAN & 8) && (FASE_SCALED_LEAN & 1) && EPT <= 20 &&
               cand == wmin && cand == barg) {
      // the pick is this thread's own argmax: its signed R' is at hand
      s_u[warp] = cand;
      s_r[warp] = bsig;
      if constexpr (!kLeanD) s_d[warp] = __ldg(D + cand);
    } else if (cand == wmin) {
      // fetch R (and D) of the winner through a shared scratch (no dynamic
      // register indexing)
#pragma unroll
      for (int j = 0; j < EP; ++j) {
        *reinterpret_cast<double2*>(&s_dump[warp][0][2 * j]) = make_double2(r[j][0], r[j][1]);
        if constexpr (!kDsmem && !kScaled)
          *reinterpret_cast<double2*>(&s_dump[warp][kDsmem ? 0 : 1][2 * j]) = dpair(j);
      }
      const int pair = static_cast<int>(cand >> 1);
      const int jj = (pair - t) / NT;
      const int ee = static_cast<int>(cand & 1u);
      s_u[warp] = cand;
      s_r[warp] = s_dump[warp][0][2 * jj + ee];
      if constexpr (kScaled) {
        if constexpr (!kLeanD) s_d[warp] = __ldg(D + cand);
      } else if constexpr (kDsmem) {
        const double2 dd = s_D[pair];
        s_d[warp] = ee ? dd.y : dd.x;
      } else {
        s_d[warp] = s_dump[warp][kDsmem ? 0 : 1][2 * jj + ee];
      }
    }
    block_sync();
    {
      const unsigned su = lane < NW ? s_u[lane] : kNone;
      u = __reduce_min_sync(0xffffffffu, su);
      uw = __ffs(__ballot_sync(0xffffffffu, su == u)) - 1;
    }
    FASE_ASSERT(u < static_cast<unsigned>(K) && uw >= 0 && uw < NW);
    } else {
      u = s_u[0];  // resolved above (one barrier back)
    }
    if constexpr (kChunked) {
      for (int ch = 0; ch < nch; ++ch) FASE_ASSERT(cids[ch] >= 0);
    }
    int use_b = -1;  // SPEC: the spare buffer holding the guess's row (no main copy issued)
    unsigned use_par = 0;
    if constexpr (SPEC > 0) {
      use_b = s_use;
      use_par = s_upar;
      if (use_b < 0) {
        par_m = n_copies & 1u;
        n_copies += 1u;
      }
    }
    const double ru = s_r[uw];
    const double du = kLeanD ? (u == guess ? dguess : __ldg(D + u)) : s_d[uw];
    // (kIntMax, resolved above: the two slots hold the projection and the coefficient)
    const double p = (kIntMax && fastb) ? ru : (kScaled ? mul_rn(ru, du) : mul_rn(ru, mul_rn(du, du)));
    const double c = (kIntMax && fastb) ? du : mul_rn(a.gamma, p);
    if (t == 0 && !(kIntMax && fastb)) {
      out_row(a.sel, sel)[it] = static_cast<int32_t>(u);
      out_row(a.proj, proj)[it] = p;
      out_row(a.coef, coef)[it] = c;
    }

    auto wait_all = [&]() {
#pragma unroll
      for (int sg = 0; sg < kSeg; ++sg) mbar_wait(&s_bar[sg], parity());
    };
    // ---- rank-1 update fused with the next iteration's running max; the row
    // source is block-uniform, so each source gets its own unrolled loop
    // `pre(sg)` runs at the start of segment sg, before its arrival is awaited
    // (chunk-row loads are issued there, so they overlap the TMA wait)
    // kLeanMax: cb holds the signed R' of the best element and the compare
    // reads magnitudes through |.| operand modifiers; it starts at -0 so only
    // metrics > 0 register -- a thread whose live metrics are all 0 (or that
    // holds only dead atoms) is resolved by the scan after the loop
    constexpr bool kLeanMax = kScaled && (FASE_SCALED_LEAN & 1);
    auto update = [&](auto row_pair, auto staged, auto pre) {
      double cb[kChains];
      unsigned ca[kChains];
      unsigned tk = 0u;  // kIntMax: the running largest key
#pragma unroll
      for (int h = 0; h < kChains; ++h) {
        cb[h] = kLeanMax ? -0.0 : kDead;
        ca[h] = kNone;
      }
#pragma unroll
      for (int j = 0; j < EP; ++j) {
#pragma unroll
        for (int sg = 0; sg < kSeg; ++sg)
          if (j == sg * EP / kSeg) {
            pre(sg);
            if constexpr (decltype(staged)::value) mbar_wait(&s_bar[sg], parity());  // segment arrives
          }
        const double2 g = row_pair(j);
        const double2 dd = dpair_if(j);
        if constexpr (kScaled && (FASE_SCALED_LEAN & 4)) {  // one rounding: R' - c*Gs fused
          r[j][0] = __fma_rn(-c, g.x, r[j][0]);
          r[j][1] = __fma_rn(-c, g.y, r[j][1]);
        } else {
          r[j][0] = sub_rn(r[j][0], mul_rn(c, g.x));
          r[j][1] = sub_rn(r[j][1], mul_rn(c, g.y));
        }
        if constexpr (kIntMax) {
          tk = __vimax3_u32(tk, key_of(r[j][0], 31u - 2 * j), key_of(r[j][1], 30u - 2 * j));
          continue;
        }
        const int h = j % kChains;
        if constexpr (kLeanMax) {
          if (fabs(r[j][0]) > fabs(cb[h])) {
            cb[h] = r[j][0];
            ca[h] = static_cast<unsigned>(2 * (j * NT + t));
          }
          if (fabs(r[j][1]) > fabs(cb[h])) {
            cb[h] = r[j][1];
            ca[h] = static_cast<unsigned>(2 * (j * NT + t) + 1);
          }
          continue;
        }
        const double2 mm = metrics(j, dd);
        const double m0 = mm.x;
        if (m0 > cb[h]) {
          cb[h] = m0;
          ca[h] = static_cast<unsigned>(2 * (j * NT + t));
        }
        const double m1 = mm.y;
        if (m1 > cb[h]) {
          cb[h] = m1;
          ca[h] = static_cast<unsigned>(2 * (j * NT + t) + 1);
        }
      }
      if constexpr (kIntMax) {
        tkey = tk;
        return;
      }
      if constexpr (kLeanMax) {
        bsig = cb[0];
        unsigned bi = ca[0];
#pragma unroll
        for (int h = 1; h < kChains; ++h)  // equal magnitudes: the lower index wins
          if (ca[h] != kNone && (bi == kNone || fabs(cb[h]) > fabs(bsig) ||
                                 (fabs(cb[h]) == fabs(bsig) && ca[h] < bi))) {
            bsig = cb[h];
            bi = ca[h];
          }
#pragma unroll
        for (int h = 0; h < kChains; ++h) cb[h] = ca[h] == kNone ? kDead : fabs(cb[h]);
      }
      best = cb[0];
      barg = ca[0];
#pragma unroll
      for (int h = 1; h < kChains; ++h)  // equal maxima: the lower index wins
        if (cb[h] > best || (cb[h] == best && ca[h] < barg)) {
          best = cb[h];
          barg = ca[h];
        }
      if constexpr (kLeanMax) {
        // rare: no live metric > 0 here -- the lowest live atom (metric 0), if any
        if (barg == kNone) {
#pragma unroll
          for (int j = EP - 1; j >= 0; --j) {
            if (r[j][1] == r[j][1]) {
              best = 0.0;
              bsig = r[j][1];
              barg = static_cast<unsigned>(2 * (j * NT + t) + 1);
            }
            if (r[j][0] == r[j][0]) {
              best = 0.0;
              bsig = r[j][0];
              barg = static_cast<unsigned>(2 * (j * NT + t));
            }
          }
        }
      }
    };
    using Staged = std::true_type;
    using Direct = std::false_type;
    auto no_pre = [](int) {};
#ifdef FASE_ITERATE_STATS
    if constexpr (!kChunked) {
      if (t == 0) {
        atomicAdd(&g_stats[0], 1ull);
        atomicAdd(&g_stats[3], u != guess ? 1ull : 0ull);
      }
    }
#endif
    if constexpr (kChunked) {
#ifdef FASE_ITERATE_STATS
      if (t == 0) {  // measurement build only: path counters
        atomicAdd(&g_stats[0], 1ull);
        atomicAdd(&g_stats[1], issue ? 1ull : 0ull);
        atomicAdd(&g_stats[2], (!issue && u == held) ? 1ull : 0ull);
        atomicAdd(&g_stats[3], (issue && u != guess) ? 1ull : 0ull);
        atomicAdd(&g_stats[4], static_cast<unsigned long long>(nch));
        atomicAdd(&g_stats[5], (!issue && u != held) ? 1ull : 0ull);
        atomicAdd(&g_stats[6], (issue && u == guess) ? static_cast<unsigned long long>(nch) : 0ull);
      }
#endif
      // row_u of this block = G0[u] - sum of its remaining chunk tables' rows,
      // element by element in list order; the complete row is left in the
      // staging buffer (held) for a re-selection of u
      if (issue && u == guess && nch == 0) {
        update([&](int j) { return s_row[j * NT + t]; }, Staged{}, no_pre);
      } else if (issue && u == guess && nch == 1) {
        // fused: a segment's chunk values are loaded before its staged G0
        // part is awaited; the composed row is written back
        const double* c0 = a.chunk_tables + static_cast<int64_t>(cids[0]) * a.chunk_stride +
                           static_cast<int64_t>(u) * ldg + 2 * t;
        double2 v0[EP];
        auto pre = [&](int sg) {
          const int j0 = sg * EP / kSeg, j1 = (sg + 1) * EP / kSeg;
#pragma unroll
          for (int j = 0; j < EP; ++j)
            if (j >= j0 && j < j1) v0[j] = ldg2_here(c0 + 2 * j * NT);
        };
        update(
            [&](int j) {
              double2 g = s_row[j * NT + t];
              g.x = sub_rn(g.x, v0[j].x);
              g.y = sub_rn(g.y, v0[j].y);
              s_row[j * NT + t] = g;
              return g;
            },
            Staged{}, pre);
        fence_proxy_async_smem();  // generic writes precede the next TMA fill
      } else if (!issue && u == held) {
        update([&](int j) { return s_row[j * NT + t]; }, Direct{}, no_pre);
      } else {
        // compose in the staging buffer (each thread only touches its own pairs)
        if (issue) wait_all();  // retire the copy before touching the buffer
        if (!issue || u != guess) {
          const double* urow = base() + static_cast<int64_t>(u) * ldg + 2 * t;
#pragma unroll 4
          for (int j = 0; j < EP; ++j) s_row[j * NT + t] = ldg2(urow + 2 * j * NT);
        }
        auto crow = [&](int ch) {
          return a.chunk_tables + static_cast<int64_t>(cids[ch]) * a.chunk_stride +
                 static_cast<int64_t>(u) * ldg + 2 * t;
        };
        int ch = 0;
        // two chunks per pass (twice the loads in flight) where registers allow
        for (; EP <= 8 && ch + 1 < nch; ch += 2) {
          const double* ca = crow(ch);
          const double* cb = crow(ch + 1);
#pragma unroll 4
          for (int j = 0; j < EP; ++j) {
            const double2 va = ldg2(ca + 2 * j * NT);
            const double2 vb = ldg2(cb + 2 * j * NT);
            double2 g = s_row[j * NT + t];
            g.x = sub_rn(sub_rn(g.x, va.x), vb.x);
            g.y = sub_rn(sub_rn(g.y, va.y), vb.y);
            s_row[j * NT + t] = g;
          }
        }
        for (; ch < nch; ++ch) {
          const double* ca = crow(ch);
#pragma unroll 4
          for (int j = 0; j < EP; ++j) {
            const double2 v = ldg2(ca + 2 * j * NT);
            double2 g = s_row[j * NT + t];
            g.x = sub_rn(g.x, v.x);
            g.y = sub_rn(g.y, v.y);
            s_row[j * NT + t] = g;
          }
        }
        update([&](int j) { return s_row[j * NT + t]; }, Direct{}, no_pre);
        fence_proxy_async_smem();  // generic writes above precede the next TMA fill
      }
      held = u;
      {  // publish the held atom's new metric for the next prediction
        const int pr = static_cast<int>(u >> 1);
        if (pr % NT == t) {
          const int jj = pr / NT;
          double rv = 0.0, dv = 0.0;
#pragma unroll
          for (int j = 0; j < EP; ++j)
            if (j == jj) {  // static register indices
              const double2 dd = dpair(j);
              rv = (u & 1u) ? r[j][1] : r[j][0];
              dv = (u & 1u) ? dd.y : dd.x;
            }
          s_heldm_all[half] = mul_rn(fabs(rv), dv);
        }
      }
    } else if (SPEC > 0 && u == guess && use_b >= 0) {  // row staged one iteration ahead
      mbar_wait(&s_sbar[use_b], use_par);
      const double2* sb = s_spare + use_b * EP * NT;
      update([&](int j) { return sb[j * NT + t]; }, Direct{}, no_pre);
      if constexpr (SYN > 0) {
#pragma unroll
        for (int i = 0; i < SYN; ++i)
          if (t + i * NT < syn.n_lost)
            gacc[i] = add_rn(gacc[i], mul_rn(c, s_sphi[SPEC > 0 ? use_b : 0][t + i * NT]));
      }
    } else if (kRegRow && u == guess) {  // the row is already in registers
      update([&](int j) { return rrow[kRegRow ? j : 0]; }, Direct{}, no_pre);
      if constexpr (SYN > 0 && kRegRow) {
#pragma unroll
        for (int i = 0; i < SYN; ++i)
          if (t + i * NT < syn.n_lost) gacc[i] = add_rn(gacc[i], mul_rn(c, rphi[i]));
      }
    } else if (u == guess) {  // block-uniform
      update([&](int j) { return s_row[j * NT + t]; }, Staged{}, no_pre);
      if constexpr (SYN > 0) {
#pragma unroll
        for (int i = 0; i < SYN; ++i)
          if (t + i * NT < syn.n_lost) gacc[i] = add_rn(gacc[i], mul_rn(c, s_phi[t + i * NT]));
      }
    } else {
      if (use_b < 0 && !kRegRow) wait_all();  // retire the mispredicted copy before the next one
      const double* urow = base() + static_cast<int64_t>(u) * ldg + 2 * t;
      double phv[SYN > 0 ? SYN : 1];
      if constexpr (SYN > 0) {
        const double* prow = syn.phi + static_cast<int64_t>(u) * syn.ldphi;
#pragma unroll
        for (int i = 0; i < SYN; ++i) phv[i] = t + i * NT < syn.n_lost ? __ldg(prow + t + i * NT) : 0.0;
      }
      update([&](int j) { return ldg2(urow + 2 * j * NT); }, Direct{}, no_pre);
      if constexpr (SYN > 0) {
#pragma unroll
        for (int i = 0; i < SYN; ++i)
          if (t + i * NT < syn.n_lost) gacc[i] = add_rn(gacc[i], mul_rn(c, phv[i]));
      }
    }
    if (kRecord) {
      double* dst = a.R_log + (static_cast<int64_t>(b) * a.I + it) * a.ldr;
#pragma unroll
      for (int j = 0; j < EP; ++j) {
        const int k = 2 * (j * NT + t);
        if (k < K) dst[k] = r[j][0];
        if (k + 1 < K) dst[k + 1] = r[j][1];
      }
    }
  }

  write_synth(b);
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

using KernelFn = void (*)(const fase_iterate_args, const fase_synth_fused);

struct Variant {
  int nt;
  int ept;
  bool dsmem;             // D in shared memory (else registers)
  KernelFn plain;         // shared geometry
  KernelFn chunked;       // per-block geometry (chunk-corrected rows)
  KernelFn record;        // shared geometry, R logged after every iteration
  int nb = 1;             // blocks per CTA (2: paired blocks sharing one D)
  KernelFn fused = nullptr;  // scaled: synthesis fused (up to syn lost samples per thread)
  int syn = 0;
  int spec = 0;              // spare row buffers (speculative staging, latency shapes)
};

#define FASE_V(NT, EPT, MINB, DS)                                                       \
  {NT,                                                                                   \
   EPT,                                                                                  \
   DS,                                                                                   \
   fase_iterate_kernel<NT, EPT, MINB, DS, false, false, 1>,                              \
   fase_iterate_kernel<NT, EPT, MINB, DS, true, false, 1>,                               \
   fase_iterate_kernel<NT, EPT, MINB, DS, false, true, 1>}
// Ordered by capacity NT*EPT; the first variant that holds K is used.
// 128/256-thread variants keep D in shared memory (3-6 CTAs per SM); the
// 512-thread variants keep R and D in registers (4 registers per atom), which
// caps K at 512 x 24.
const Variant kVariants[] = {
    FASE_V(128, 2, 4, false),  FASE_V(128, 4, 4, false),  FASE_V(128, 8, 4, false),
    FASE_V(128, 16, 6, true),  FASE_V(256, 10, 4, true),  FASE_V(256, 12, 3, true),
    FASE_V(256, 14, 3, true),  FASE_V(256, 16, 3, true),  FASE_V(256, 18, 3, true),
    FASE_V(256, 20, 2, true),  FASE_V(512, 12, 1, false), FASE_V(512, 16, 1, false),
    FASE_V(512, 20, 1, false), FASE_V(512, 24, 1, false),
};

// Paired blocks for large shared-geometry tables (same capacity as the default
// variant, so the same table layout): one 512-thread CTA runs two blocks that
// share D in shared memory -- two blocks in flight per SM where one 512-thread
// CTA with D in registers fits only one.
#define FASE_VP(NT, EPT)                                                              \
  {NT, EPT, true, fase_iterate_kernel<NT, EPT, 1, true, false, false, 2>, nullptr, nullptr, 2}
const Variant kPairVariants[] = {
    FASE_VP(256, 20), FASE_VP(256, 24), FASE_VP(256, 32), FASE_VP(512, 16),
};
#undef FASE_VP

// Alternative shapes, selectable for measurement with FASE_ITERATE_VARIANT=NTxEPT
// (must not exceed the default variant's capacity, which sizes the tables).
const Variant kExtraVariants[] = {
    FASE_V(256, 8, 5, true),
    FASE_V(128, 36, 3, true),
    FASE_V(576, 4, 1, true),
};

// Latency variants: batches of at most one block per SM gain nothing from
// residency, so each block gets the widest CTA (576 x 4 / 768 x 6 / 1024 x 8) that keeps two or three pairs per
// thread (config 0, K = 2304: 384 threads, 113 -> 98 us for 100 iterations).
// (fused: the exact recursion with the synthesis fused in, fase_iterate_synth)
#define FASE_VL(NT, EPT, SPEC, SYN)                                                      \
  {NT,                                                                                  \
   EPT,                                                                                 \
   true,                                                                                \
   fase_iterate_kernel<NT, EPT, 1, true, false, false, 1, false, 0, SPEC>,             \
   fase_iterate_kernel<NT, EPT, 1, true, true, false, 1>,                               \
   fase_iterate_kernel<NT, EPT, 1, true, false, true, 1>,                               \
   1, fase_iterate_kernel<NT, EPT, 1, true, false, false, 1, false, SYN, SPEC>, SYN, SPEC}
// (576 x 4 for K <= 2304: two pairs per thread, config-0 exact recursion
// 115.2 -> 106.6 us against 384 x 6; 87.7 us with register rows)
const Variant kLatencyVariants[] = {
    FASE_VL(384, 6, FASE_SPEC, 2),
    FASE_VL(576, 4, FASE_SPEC, 1),
    FASE_VL(768, 6, FASE_SPEC, 1),
    FASE_VL(1024, 8, 0, 1),  // (register rows measured slower at 4 pairs per thread)
};
#undef FASE_VL
#undef FASE_V

// Scaled recursion (fase_iterate_scaled): no normalizers in the loop, so only
// the staged row occupies shared memory and four 256-thread CTAs fit per SM
// (64 registers; config 1: 0.916 ms exact at three CTAs, 0.815 ms scaled at
// three, 0.721 ms scaled at four). Ordered by capacity like kVariants.
// (Capacity 8192 as 128 x 64 -- 4 warps, 255 registers, two CTAs per SM --
// halves the per-warp iteration overhead: on a power-capped box config 4 holds
// 1837 instead of 1747 MHz and gains 1.3%, but without the cap it is 8% slower
// (11.89 vs 11.0 ms under ncu, fewer warps to hide the row latency); the
// default stays 256 x 32, tools/ab_variant128*.sh, profiles/r02b/ab_variant128.txt)
// SYN: lost samples per thread of the fused-synthesis kernel (registers allow
// only one at the 64-register four-CTA shapes).
#define FASE_VS(NT, EPT, MINB, SYN)                                                          \
  {NT,      EPT,     false, fase_iterate_kernel<NT, EPT, MINB, false, false, false, 1, true>, \
   nullptr, nullptr, 1,     fase_iterate_kernel<NT, EPT, MINB, false, false, false, 1, true, SYN>, SYN}
const Variant kScaledVariants[] = {
    FASE_VS(128, 2, 8, 4),   FASE_VS(128, 4, 8, 4),   FASE_VS(128, 8, 8, 4),
    FASE_VS(128, 16, 6, 4),  FASE_VS(256, 10, 4, 1),  FASE_VS(256, 12, 4, 1),
    FASE_VS(256, 14, 4, 1),  FASE_VS(256, 16, 4, 1),  FASE_VS(256, 18, 4, 1),
    FASE_VS(256, 20, 3, 3),  FASE_VS(256, 24, 2, 3),  FASE_VS(256, 32, 2, 3),
    FASE_VS(512, 20, 1, 2),  FASE_VS(512, 24, 1, 2),
};
// alternatives for measurement (FASE_SCALED_VARIANT=NTxEPTxMINB) and the
// latency shapes for batches of at most one block per SM
const Variant kScaledExtra[] = {
    FASE_VS(128, 36, 4, 2), FASE_VS(256, 18, 3, 2), FASE_VS(128, 64, 2, 4),
    FASE_VS(128, 64, 3, 4), FASE_VS(256, 20, 4, 1),
};
const int kScaledExtraMinb[] = {4, 3, 2, 3, 4};
#define FASE_VSL(NT, EPT, SYN, SPEC)                                                            \
  {NT,      EPT,     false, fase_iterate_kernel<NT, EPT, 1, false, false, false, 1, true, 0, SPEC>, \
   nullptr, nullptr, 1,     fase_iterate_kernel<NT, EPT, 1, false, false, false, 1, true, SYN, SPEC>, \
   SYN,     SPEC}
// (576 x 4 measured slower for the scaled recursion: config 0 106.6 vs ~97 us
// with staged rows, 102.4 vs 96.3 us with register rows)
const Variant kScaledLatency[] = {
    FASE_VSL(384, 6, 2, FASE_SPEC), FASE_VSL(768, 6, 1, FASE_SPEC), FASE_VSL(1024, 8, 1, 0),
};
#undef FASE_VSL
#undef FASE_VS

int sm_count() {
  static int n = [] {
    int dev = 0, count = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&count, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
      return 148;
    return count;
  }();
  return n;
}

const Variant* pick_variant(int K) {
  for (const Variant& v : kVariants)
    if (v.nt * v.ept >= K) return &v;
  return nullptr;
}

const Variant* override_variant(int K, const Variant* dflt) {
  const char* env = getenv("FASE_ITERATE_VARIANT");
  if (!env || !dflt) return dflt;
  int nt = 0, ept = 0;
  if (sscanf(env, "%dx%d", &nt, &ept) != 2) return dflt;
  auto match = [&](const Variant& v) {
    return v.nt == nt && v.ept == ept && v.nt * v.ept >= K && v.nt * v.ept <= dflt->nt * dflt->ept;
  };
  for (const Variant& v : kVariants)
    if (match(v)) return &v;
  for (const Variant& v : kExtraVariants)
    if (match(v)) return &v;
  for (const Variant& v : kLatencyVariants)
    if (match(v)) return &v;
  return dflt;
}

}  // namespace

int sm_count_cluster() { return sm_count(); }
int iterate_register_atoms() {
  const Variant& last = kVariants[sizeof(kVariants) / sizeof(kVariants[0]) - 1];
  return last.nt * last.ept;
}
// csrc/iterate_generic.cu: R streamed through global memory (K beyond the registers)
int launch_iterate_generic(const fase_iterate_args& a, cudaStream_t stream);
// the streaming recursion's atom limit (tables of K x K doubles beyond it)
constexpr int kGenericMaxAtoms = 1 << 20;
// csrc/iterate_cluster.cu: one block over a CTA cluster (latency-bound batches)
int launch_iterate_cluster(const fase_iterate_args& a, const fase_synth_fused* syn, bool scaled,
                           cudaStream_t stream);
int cluster_synth_capacity(int K, int64_t ldg, int B);
}  // namespace fase

using namespace fase;

extern "C" int fase_max_atoms(void) { return kGenericMaxAtoms; }

extern "C" int fase_iterate_register_atoms(void) { return iterate_register_atoms(); }

extern "C" int fase_table_ld(int K) {
  if (K < 1 || K > kGenericMaxAtoms) return 0;
  const Variant* v = pick_variant(K);
  return v ? v->nt * v->ept : K + (K & 1);  // beyond the registers: even, unpadded
}

namespace {
// FASE_L2_HINT=0 drops the L2 residency hint (measurement)
fase_iterate_args hint_policy(const fase_iterate_args& in) {
  fase_iterate_args a = in;
  const char* env = getenv("FASE_L2_HINT");
  if (env && env[0] == '0') a.l2_hot = nullptr;
  return a;
}
}  // namespace

extern "C" int fase_iterate(const fase_iterate_args* args, void* stream) {
  if (!args) {
    set_error("fase_iterate: null argument block");
    return FASE_ERR_PARAMETER;
  }
  const fase_iterate_args a = hint_policy(*args);
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
  if (a.chunk_count && (!a.chunk_ids || !a.chunk_tables || !aligned16(a.chunk_tables) ||
                      (a.chunk_stride & 1))) {
    set_error("fase_iterate: chunk tables given without ids / aligned storage");
    return FASE_ERR_SHAPE;
  }
  if (a.compose && (!a.chunk_count || a.n_compose < 1 || a.compose_depth < 1 ||
                    a.compose_depth > 3 || a.base_stride < a.ldg * a.K || (a.base_stride & 1))) {
    set_error("fase_iterate: compose table needs chunk lists, n_compose >= 1, depth 1..3 and an "
              "even base_stride >= ldg*K");
    return FASE_ERR_SHAPE;
  }
  if (a.chunk_count && a.R_log) {
    set_error("fase_iterate: R_log recording is not available with chunked tables");
    return FASE_ERR_UNSUPPORTED;
  }
  const Variant* dflt = pick_variant(a.K);
  if (!dflt && a.K <= kGenericMaxAtoms) {  // beyond the registers: the streaming recursion
    if (a.ldg < a.K || (a.chunk_count && a.chunk_stride < a.ldg * a.K)) {
      set_error("fase_iterate: table rows shorter than K (ldg=%lld)", static_cast<long long>(a.ldg));
      return FASE_ERR_SHAPE;
    }
    return launch_iterate_generic(a, as_stream(stream));
  }
  const Variant* v = override_variant(a.K, dflt);
  const bool small = a.B <= sm_count();  // at most one block per SM
  if (small && !getenv("FASE_ITERATE_VARIANT")) {  // a block over a CTA cluster
    const int rc = launch_iterate_cluster(a, nullptr, false, as_stream(stream));
    if (rc != 1) return rc;
  }
  if (v == dflt && dflt && small && !getenv("FASE_ITERATE_VARIANT")) {
    for (const Variant& lv : kLatencyVariants)
      if (lv.nt * lv.ept >= a.K && lv.nt * lv.ept <= dflt->nt * dflt->ept && lv.nt > v->nt) v = &lv;
  }
  if (!v) {
    set_error("fase_iterate: K=%d exceeds the largest kernel variant (%d atoms)", a.K,
              iterate_register_atoms());
    return FASE_ERR_UNSUPPORTED;
  }
  if (a.ldg < v->nt * v->ept || (a.chunk_count && a.chunk_stride < a.ldg * a.K)) {
    set_error("fase_iterate: table rows must be zero-padded to fase_table_ld(K)=%d (ldg=%lld)",
              v->nt * v->ept, static_cast<long long>(a.ldg));
    return FASE_ERR_SHAPE;
  }
  if (!a.chunk_count && !a.R_log && a.ldd == 0 && !small) {
    // FASE_ITERATE_PAIR: 0 disables pairing, NT picks the half size (measurement)
    const char* env = getenv("FASE_ITERATE_PAIR");
    const int want = env ? atoi(env) : 256;
    if (want != 0)
      for (const Variant& pv : kPairVariants)
        if (pv.nt * pv.ept == v->nt * v->ept && pv.nt == want) v = &pv;
  }
  KernelFn fn = a.chunk_count ? v->chunked : (a.R_log ? v->record : v->plain);
  const size_t smem = static_cast<size_t>(v->nt) * (v->ept / 2) * sizeof(double2) *
                      (v->nb + (v->dsmem ? 1 : 0) + (fn == v->plain && v->spec > 0 ? v->spec : 0));
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e == cudaSuccess)  // several CTAs per SM need the full shared-memory carveout
    e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (e != cudaSuccess) {
    set_error("fase_iterate: cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    return FASE_ERR_CUDA;
  }
  fn<<<(a.B + v->nb - 1) / v->nb, v->nt * v->nb, smem, as_stream(stream)>>>(a, fase_synth_fused{});
  return check_launch("fase_iterate");
}

namespace fase {
namespace {
// The scaled variant for K atoms and B blocks (nullptr when K is too large):
// the smallest capacity holding K; FASE_SCALED_VARIANT=NTxEPT[xMINB] picks an
// alternative shape for measurement; at most one block per SM takes the
// widest latency shape.
const Variant* pick_scaled(int K, int B) {
  const Variant* dflt = pick_variant(K);
  if (!dflt) return nullptr;
  const int cap = dflt->nt * dflt->ept;
  const Variant* v = nullptr;
  for (const Variant& sv : kScaledVariants)
    if (sv.nt * sv.ept >= K) {
      v = &sv;
      break;
    }
  const char* env = getenv("FASE_SCALED_VARIANT");
  int nt = 0, ept = 0, minb = 0;
  if (env && sscanf(env, "%dx%dx%d", &nt, &ept, &minb) >= 2) {
    for (int i = 0; i < static_cast<int>(sizeof(kScaledExtra) / sizeof(kScaledExtra[0])); ++i) {
      const Variant& ev = kScaledExtra[i];
      if (ev.nt == nt && ev.ept == ept && (minb == 0 || kScaledExtraMinb[i] == minb) &&
          ev.nt * ev.ept >= K && ev.nt * ev.ept <= cap)
        v = &ev;
    }
  } else if (B <= sm_count()) {
    for (const Variant& lv : kScaledLatency)
      if (lv.nt * lv.ept >= K && lv.nt * lv.ept <= cap && lv.nt > v->nt) v = &lv;
  }
  return v;
}
}  // namespace
}  // namespace fase

namespace fase {
namespace {
// The exact latency variant for K (the widest one-block-per-SM shape whose
// capacity fits the default variant's table layout), or nullptr.
const Variant* pick_latency_exact(int K) {
  const Variant* dflt = pick_variant(K);
  if (!dflt) return nullptr;
  const Variant* v = nullptr;
  for (const Variant& lv : kLatencyVariants)
    if (lv.nt * lv.ept >= K && lv.nt * lv.ept <= dflt->nt * dflt->ept && (!v || lv.nt > v->nt))
      v = &lv;
  return v;
}
}  // namespace
}  // namespace fase

extern "C" int fase_iterate_synth_capacity(int K, int B) {
  if (K < 1 || B < 1 || B > sm_count()) return 0;
  const Variant* v = pick_latency_exact(K);
  return v ? v->syn * v->nt : 0;
}

extern "C" int fase_iterate_synth(const fase_iterate_args* args, const fase_synth_fused* syn,
                                  void* stream) {
  if (!args || !syn) {
    set_error("fase_iterate_synth: null argument block");
    return FASE_ERR_PARAMETER;
  }
  const fase_iterate_args a = hint_policy(*args);
  if (a.K < 1 || a.B < 0 || a.I < 1) {
    set_error("fase_iterate_synth: bad sizes (K=%d, B=%d, I=%d)", a.K, a.B, a.I);
    return FASE_ERR_SHAPE;
  }
  if (!(a.gamma > 0.0 && a.gamma <= 1.0)) {
    set_error("fase_iterate_synth: gamma must lie in (0, 1], got %g", a.gamma);
    return FASE_ERR_PARAMETER;
  }
  if (a.B == 0) return FASE_OK;
  if (!a.G0 || !aligned16(a.G0) || a.ldg < a.K || (a.ldg & 1) || !a.D || !a.R0 ||
      a.ldr < a.K || !a.sel || !a.proj || !a.coef || a.ldo < a.I) {
    set_error("fase_iterate_synth: bad operand (null, misaligned, odd or short leading dimension)");
    return FASE_ERR_SHAPE;
  }
  if (a.chunk_count || a.compose || a.ldd != 0 || a.R_out || a.R_log) {
    set_error("fase_iterate_synth: shared geometry only (no chunk tables, per-block D, R_out or "
              "R_log)");
    return FASE_ERR_UNSUPPORTED;
  }
  if (syn->n_lost < 1 || !syn->phi || !aligned16(syn->phi) || (syn->ldphi & 1) ||
      syn->ldphi < syn->n_lost || !syn->out || syn->ldout < syn->n_lost) {
    set_error("fase_iterate_synth: bad fused-synthesis operand (n_lost=%d)", syn->n_lost);
    return FASE_ERR_SHAPE;
  }
  const Variant* v = a.B <= sm_count() ? pick_latency_exact(a.K) : nullptr;
  if (!v || !v->fused || syn->n_lost > v->syn * v->nt) {
    set_error("fase_iterate_synth: needs at most one block per SM and n_lost <= "
              "fase_iterate_synth_capacity(K, B) (K=%d, B=%d, n_lost=%d)", a.K, a.B, syn->n_lost);
    return FASE_ERR_UNSUPPORTED;
  }
  if (a.ldg < pick_variant(a.K)->nt * pick_variant(a.K)->ept) {
    set_error("fase_iterate_synth: table rows must be zero-padded to fase_table_ld(K) (ldg=%lld)",
              static_cast<long long>(a.ldg));
    return FASE_ERR_SHAPE;
  }
  const size_t smem = static_cast<size_t>(v->nt) * (v->ept / 2) * sizeof(double2) *
                      (1 + 1 + (v->spec > 0 ? v->spec : 0));  // row, D (+ spare rows)
  cudaError_t e = cudaFuncSetAttribute(v->fused, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e != cudaSuccess) {
    set_error("fase_iterate_synth: cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    return FASE_ERR_CUDA;
  }
  // one block per SM at most: launched as a programmatic dependent of the
  // products kernel before it (which releases it at its start), so this grid is
  // resident when the products finish instead of launching after them
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(a.B);
  cfg.blockDim = dim3(v->nt);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = as_stream(stream);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = FASE_PDL;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, v->fused, a, *syn);
  if (e != cudaSuccess) {
    set_error("fase_iterate_synth: launch: %s", cudaGetErrorString(e));
    return FASE_ERR_CUDA;
  }
  return check_launch("fase_iterate_synth");
}

extern "C" int fase_iterate_scaled_synth_capacity(int K, int B) {
  // the larger of the cluster path's (taken when the lost samples fit it) and
  // the one-CTA variant's capacity
  int c = 0;
  if (K >= 1 && B >= 1 && B <= sm_count() && !getenv("FASE_SCALED_VARIANT"))
    c = cluster_synth_capacity(K, fase_table_ld(K), B);
  const Variant* v = K >= 1 ? pick_scaled(K, B) : nullptr;
  return v ? max(c, v->syn * v->nt) : c;
}

extern "C" int fase_iterate_scaled(const fase_iterate_args* args, const fase_synth_fused* syn,
                                   void* stream) {
  if (!args) {
    set_error("fase_iterate_scaled: null argument block");
    return FASE_ERR_PARAMETER;
  }
  const fase_iterate_args a = hint_policy(*args);
  if (a.K < 1 || a.B < 0 || a.I < 1) {
    set_error("fase_iterate_scaled: bad sizes (K=%d, B=%d, I=%d)", a.K, a.B, a.I);
    return FASE_ERR_SHAPE;
  }
  if (!(a.gamma > 0.0 && a.gamma <= 1.0)) {
    set_error("fase_iterate_scaled: gamma must lie in (0, 1], got %g", a.gamma);
    return FASE_ERR_PARAMETER;
  }
  if (a.B == 0) return FASE_OK;
  if (!a.G0 || !aligned16(a.G0) || a.ldg < a.K || (a.ldg & 1) || !a.D || !a.R0 ||
      a.ldr < a.K || !a.sel || !a.proj || !a.coef || a.ldo < a.I) {
    set_error("fase_iterate_scaled: bad operand (null, misaligned, odd or short leading dimension)");
    return FASE_ERR_SHAPE;
  }
  if (a.chunk_count || a.compose || a.ldd != 0 || a.R_out || a.R_log) {
    set_error("fase_iterate_scaled: shared geometry only (no chunk tables, per-block D, R_out or "
              "R_log)");
    return FASE_ERR_UNSUPPORTED;
  }
  if (syn && (syn->n_lost < 1 || !syn->phi || !aligned16(syn->phi) || (syn->ldphi & 1) ||
              syn->ldphi < syn->n_lost || !syn->out || syn->ldout < syn->n_lost)) {
    set_error("fase_iterate_scaled: bad fused-synthesis operand (n_lost=%d)", syn ? syn->n_lost : 0);
    return FASE_ERR_SHAPE;
  }
  if (a.B <= sm_count() && !getenv("FASE_SCALED_VARIANT")) {  // a block over a CTA cluster
    const int rc = launch_iterate_cluster(a, syn, true, as_stream(stream));
    if (rc != 1) return rc;
  }
  const Variant* v = pick_scaled(a.K, a.B);
  if (!v) {
    set_error("fase_iterate_scaled: K=%d exceeds the largest kernel variant (%d atoms)", a.K,
              iterate_register_atoms());
    return FASE_ERR_UNSUPPORTED;
  }
  if (syn && syn->n_lost > v->syn * v->nt) {
    set_error("fase_iterate_scaled: %d lost samples exceed the fused synthesis capacity %d "
              "(fase_iterate_scaled_synth_capacity)", syn->n_lost, v->syn * v->nt);
    return FASE_ERR_UNSUPPORTED;
  }
  if (a.ldg < v->nt * v->ept) {
    set_error("fase_iterate_scaled: table rows must be zero-padded to fase_table_ld(K) (ldg=%lld)",
              static_cast<long long>(a.ldg));
    return FASE_ERR_SHAPE;
  }
  KernelFn fn = syn ? v->fused : v->plain;
  const size_t smem = static_cast<size_t>(v->nt) * (v->ept / 2) * sizeof(double2) *
                      (1 + (v->spec > 0 ? v->spec : 0));
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (e != cudaSuccess) {
    set_error("fase_iterate_scaled: cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    return FASE_ERR_CUDA;
  }
  fn<<<a.B, v->nt, smem, as_stream(stream)>>>(a, syn ? *syn : fase_synth_fused{});
  return check_launch("fase_iterate_scaled");
}

#ifdef FASE_ITERATE_STATS
// measurement build only: chunked-path counters since the last call
// (iterations, copies issued, held hits, mispredicted copies, remaining chunks,
// held misses without a copy, remaining chunks on predicted copies)
extern "C" __attribute__((visibility("default"))) int fase_iterate_stats(unsigned long long* out8) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out8, fase::g_stats, 8 * sizeof(unsigned long long));
  unsigned long long zero[8] = {0};
  cudaMemcpyToSymbol(fase::g_stats, zero, sizeof(zero));
  return check_launch("fase_iterate_stats");
}
#endif
