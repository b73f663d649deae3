// Shared device code of the thread-per-replica Detector kernels
// (pass_small_kernel in pipeline.cu, pass_wide_kernel in pass_wide.cu): the
// launch parameters, TMA staging of a CTA's offsets / documents, and the
// compile-time 1F1B / ZBH walks.
#pragma once

#include <algorithm>
#include <type_traits>
#include <utility>

#include <math_constants.h>

#include "common.cuh"
#include "wavefront.cuh"

namespace rh {

struct PassParams {
  rh_pipe_shape sh;
  rh_cost_model m;
  rh_segments sg;
  rh_trace tr;
  rh_pass_out out;
  double thr;
  int pw, log_pw;  // lanes per pipeline
  int lpi;         // lanes per iteration = D * pw
  int ipb;         // iterations per CTA
  int mmax;        // micro-batches per replica (smem row length)
  int vec4;        // device_time rows are float4-aligned
  // thread-per-replica kernel only
  const unsigned long long* sched;  // level table (sched_table)
  const int32_t* sched_off;         // [mmax+2] first level word of each micro-batch count
  const int32_t* sched_peak;        // [mmax+1] peak in-flight forward chunks on any stage
  int region_off;            // smem offset of the document / base-cost region
  int doc_stage;             // documents that fit in that region
  int pf_stride;             // resident CTA slots: CTA b prefetches CTA b + pf_stride (0: off)
  // wide kernel smem (byte offsets): base costs [mmax][TW] doubles, ratio *
  // layers [ipb][3][P] doubles, then a union of {offsets (ipb*M+1 int32,
  // 16 B slack) + documents (doc_stage int32)} and {hops [2][P][TW] doubles}
  int w_base, w_rl, w_union, w_docs;
  const double* wtab;  // wide kernel: per-launch transposed segment table (wide_prep)
  int q32;         // micro-batch sum l^2 in 32-bit integers (exactness checked per micro-batch)
  int static_max;  // largest micro-batch count walked by the unrolled code
  int steady;      // m >= P: the steady-state loop walk (walk_steady)
  // lane kernel only: level table (lane_table), NULL = closed-form walk
  const uint16_t* ltab;
  const int32_t *ltab_off, *ltab_nlev, *ltab_peak;  // [mmax+1] each
};

// ---- TMA bulk staging (cp.async.bulk + mbarrier, sm_90+ / sm_100a)
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // visible to the TMA unit
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; "
        "selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
}
// L2 prefetch of [p, p + bytes), trimmed inward to 16-byte alignment (a hint:
// nothing outside the range is touched)
__device__ __forceinline__ void prefetch_l2(const void* p, size_t bytes) {
  const uintptr_t a = (reinterpret_cast<uintptr_t>(p) + 15) & ~uintptr_t(15);
  const uintptr_t b = (reinterpret_cast<uintptr_t>(p) + bytes) & ~uintptr_t(15);
  if (b > a)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"((unsigned)(b - a))
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Stage n ints at src into shared memory: the 16-byte-aligned interior by
// one TMA bulk copy (issued by thread 0, completing on `bar`), the ragged
// head / tail words by plain loads -- nothing outside [src, src+n) is read.
// `dst_base` is 16-byte aligned with 16 spare bytes; the returned pointer is
// dst_base shifted by src's misalignment so the interior lines up.  Returns
// the bytes the TMA will deliver (for the barrier's expect_tx).
struct StagePlan {
  int32_t* dst;
  int head, tail;      // words loaded by threads at the front / back
  unsigned tx_bytes;   // bytes delivered by the bulk copy
};
__device__ __forceinline__ StagePlan stage_plan(unsigned char* dst_base, const int32_t* src,
                                                int n) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(src);
  StagePlan sp;
  sp.dst = reinterpret_cast<int32_t*>(dst_base + (a & 15));
  const uintptr_t a16 = (a + 15) & ~uintptr_t(15), b = a + 4 * (uintptr_t)n,
                  b16 = b & ~uintptr_t(15);
  if (b16 > a16) {
    sp.head = (int)((a16 - a) / 4);
    sp.tail = (int)((b - b16) / 4);
    sp.tx_bytes = (unsigned)(b16 - a16);
  } else {  // too short for a bulk copy: threads load everything
    sp.head = n;
    sp.tail = 0;
    sp.tx_bytes = 0;
  }
  return sp;
}
__device__ __forceinline__ void stage_issue(const StagePlan& sp, const int32_t* src,
                                            uint64_t* bar) {
  if (sp.tx_bytes) bulk_g2s(sp.dst + sp.head, src + sp.head, sp.tx_bytes, bar);
}
__device__ __forceinline__ void stage_edges(const StagePlan& sp, const int32_t* src, int n) {
  for (int q = threadIdx.x; q < sp.head + sp.tail; q += blockDim.x) {
    const int k = q < sp.head ? q : n - sp.tail + (q - sp.head);
    sp.dst[k] = __ldg(src + k);
  }
}

// sched_table entry: one 64-bit word per DAG level, 16 bits per stage:
// 0 = idle, else kind (1 F, 2 B / BW, 3 W) | j << 2
enum : unsigned { kOpF = 1, kOpB = 2, kOpW = 3 };

// A shared-memory load the compiler must not keep in a register across uses
// (ld.volatile: neither nvcc nor ptxas merges it with an earlier load of the
// same address).  The wide walks reload their per-stage constants and base
// costs per chunk instead of pinning hundreds of registers.
__device__ __forceinline__ double lds_nc(const double* p) {
  double v;
  asm volatile("ld.volatile.shared.f64 %0, [%1];" : "=d"(v) : "r"((uint32_t)__cvta_generic_to_shared(p)));
  return v;
}

// Walk arguments of the thread-per-replica kernels.  A walk reads the
// per-stage constants through accessors -- rlF/rlB/rlW(s) (ratio * layers),
// sp/inv(s) (stage speed and its exact reciprocal), hf/hb(s) (hop weights) --
// and updates fin[s] (the chain's last finish) and ssum[s] (its cost sum).
// Every index is a compile-time constant after unrolling, so register arrays
// stay in registers.
//
// WalkArgs (pass_small_kernel, P <= 4): everything in registers.
#ifndef RH_SMALL_SLOWMASK
#define RH_SMALL_SLOWMASK 0  // A/B knob: measured slower for the P <= 4 walks (40.0 vs 37.5 us)
#endif
template <int P, int TW>
struct WalkArgs {
  static constexpr int kStride = TW;  // CTA width: base costs live [j][thread]
  static constexpr bool kSlowMask = RH_SMALL_SLOWMASK != 0;
  const double* bt;  // base costs of this thread: bt[j * kStride]
  const double (&rlF_)[P];
  const double (&rlB_)[P];
  const double (&rlW_)[P];
  const double (&sp_)[P];
  const double (&inv_)[P];  // recip_of(sp): exact division by div_fast
  const double (&hf_)[P];
  const double (&hb_)[P];
  double (&fin)[P];
  double (&ssum)[P];
  // warp-uniform: bit s = some replica of the warp runs stage s slower than
  // 1.0; the other stages skip the division (x / 1.0 == x exactly)
  unsigned slow;
  __device__ __forceinline__ static double ld(const double* p) { return *p; }
  __device__ __forceinline__ double rlF(int s) const { return rlF_[s]; }
  __device__ __forceinline__ double rlB(int s) const { return rlB_[s]; }
  __device__ __forceinline__ double rlW(int s) const { return rlW_[s]; }
  __device__ __forceinline__ double sp(int s) const { return sp_[s]; }
  __device__ __forceinline__ double inv(int s) const { return inv_[s]; }
  __device__ __forceinline__ double hf(int s) const { return hf_[s]; }
  __device__ __forceinline__ double hb(int s) const { return hb_[s]; }
  __device__ __forceinline__ bool is_slow(int s) const { return (slow >> s) & 1u; }
};

// One chunk of stage s: c = (rl * b) [/ speed], start = max(chain finish,
// dependency finish + hop), finish = start + c (pipeline.py:275-291).
// (rl * b) / sp exactly as __ddiv_rn; SAFE: the walk's operand ranges were
// checked up front (div_fast), otherwise every division is __ddiv_rn.
// nodep: the chunk has no data dependency (stage 0's F, the last stage's B,
// every W; dep == 0.0), so start = chain finish -- a finish is a sum of
// non-negative costs from +0.0, never -0.0 or NaN, so max(fin, 0.0) == fin;
// stated explicitly because the compiler must otherwise keep the NaN-aware
// max (5 instructions instead of none).
template <bool SAFE, class WA>
__device__ __forceinline__ double chunk(const WA& a, int s, double rl, double b, double dep,
                                        bool nodep = false) {
  const double x = __dmul_rn(rl, b);
  double c = x;
  if constexpr (WA::kSlowMask) {
    if (!SAFE)
      c = __ddiv_rn(x, a.sp(s));
    else if (a.is_slow(s))  // warp-uniform
      c = div_fast(x, a.sp(s), a.inv(s));
  } else {
    c = SAFE ? div_fast(x, a.sp(s), a.inv(s)) : __ddiv_rn(x, a.sp(s));
  }
  const double st = (nodep || a.fin[s] > dep) ? a.fin[s] : dep;
  a.fin[s] = __dadd_rn(st, c);
  a.ssum[s] = __dadd_rn(a.ssum[s], c);
  return a.fin[s];
}

// Dynamic walk over the level table: kWords 64-bit words per level (16 bits
// per stage: 0 idle, else kind | j << 2); stages in descending order.
template <int P, int ZBH, bool SAFE, class WA>
__device__ __forceinline__ void walk_table(const WA& a, const unsigned long long* lv,
                                           const unsigned long long* lv_end) {
  constexpr int kWords = (P + 3) / 4;
  double lastF[P], lastB[P];
#pragma unroll
  for (int s = 0; s < P; ++s) lastF[s] = lastB[s] = 0.0;
  for (; lv < lv_end; lv += kWords) {
    unsigned long long words[kWords];
#pragma unroll
    for (int w = 0; w < kWords; ++w) words[w] = __ldg(lv + w);
#pragma unroll
    for (int s = P - 1; s >= 0; --s) {
      const unsigned code = (unsigned)(words[s / 4] >> (16 * (s % 4))) & 0xffffu;
      if (code == 0) continue;
      const unsigned kind = code & 3u;
      const bool isF = kind == kOpF, isB = kind == kOpB;
      const double dF = s > 0 ? __dadd_rn(lastF[s > 0 ? s - 1 : 0], a.hf(s)) : 0.0;
      const double dB = s < P - 1 ? __dadd_rn(lastB[s < P - 1 ? s + 1 : 0], a.hb(s)) : 0.0;
      const double nf = chunk<SAFE>(a, s, isF ? a.rlF(s) : (isB || !ZBH ? a.rlB(s) : a.rlW(s)),
                                    WA::ld(a.bt + (code >> 2) * WA::kStride), isF ? dF : (isB ? dB : 0.0));
      lastF[s] = isF ? nf : lastF[s];
      lastB[s] = isB ? nf : lastB[s];
    }
  }
}

// The chunk of stage s at DAG level t for MM micro-batches (ChainLevels::at,
// the inverse of the wavefront.cuh closed forms).  Evaluated on compile-time
// constants inside walk_static, so it folds away.
__host__ __device__ __forceinline__ constexpr int op_at(int P, int MM, int zbh, int t, int s,
                                                       int& j) {
  return ChainLevels{s, P, MM, (P - 1 - s) < MM ? (P - 1 - s) : MM}.at(t, zbh != 0, j);
}
// compile-time kind / micro-batch of stage s at level t
__host__ __device__ constexpr int op_kind_c(int P, int MM, int zbh, int t, int s) {
  int j = 0;
  return op_at(P, MM, zbh, t, s, j);
}
__host__ __device__ constexpr int op_j_c(int P, int MM, int zbh, int t, int s) {
  int j = 0;
  op_at(P, MM, zbh, t, s, j);
  return j;
}

// Upper bound on the DAG levels of an MM-micro-batch replica (levels past the
// last chunk are idle and fold away).
__host__ __device__ constexpr int n_levels(int P, int MM) { return 2 * P + 3 * MM + 2; }

// Fully unrolled walk for a compile-time micro-batch count: every op, its
// kind and j are constants, so a chunk is ~8 instructions with no dispatch.
template <int P, int ZBH, int MM, class WA>
__device__ __forceinline__ void walk_static(const WA& a);

// One (level T, stage S) slot of a compile-time walk: kind and j are
// constants, so a chunk is ~8 instructions and an idle slot is nothing.
template <int P, int ZBH, int MM, int T, int S, bool COOL, bool MASK, class WA>
__device__ __forceinline__ void walk_slot(const WA& a, const double* bt_fb, const double* bt_w,
                                          double (&lastF)[P], double (&lastB)[P], int mlim) {
  constexpr int kind = op_kind_c(P, MM, ZBH, T, S);
  constexpr int j = op_j_c(P, MM, ZBH, T, S);
  if constexpr (kind == 0) {
    return;
  } else {
    if (MASK && j >= mlim) return;  // (masked 1F1B walk: m < P)
    if constexpr (kind == kOpF) {
      const double dep = S > 0 ? __dadd_rn(lastF[S > 0 ? S - 1 : 0], a.hf(S)) : 0.0;
      lastF[S] = chunk<true>(a, S, a.rlF(S), WA::ld(bt_fb + j * WA::kStride), dep, S == 0);
    } else if constexpr (kind == kOpB) {
      const double dep = S < P - 1 ? __dadd_rn(lastB[S < P - 1 ? S + 1 : 0], a.hb(S)) : 0.0;
      lastB[S] = chunk<true>(a, S, a.rlB(S), WA::ld(bt_fb + j * WA::kStride), dep, S == P - 1);
    } else if constexpr (!(COOL && j >= P - 1 - S)) {
      chunk<true>(a, S, a.rlW(S), WA::ld(bt_w + j * WA::kStride), 0.0, true);
    }
  }
}

// All stages of level T, descending (fold over the stage sequence).
template <int P, int ZBH, int MM, int T, bool COOL, bool MASK, class WA, int... I>
__device__ __forceinline__ void walk_level(const WA& a, const double* bt_fb, const double* bt_w,
                                           double (&lastF)[P], double (&lastB)[P], int mlim,
                                           std::integer_sequence<int, I...>) {
  (walk_slot<P, ZBH, MM, T, P - 1 - I, COOL, MASK>(a, bt_fb, bt_w, lastF, lastB, mlim), ...);
}

template <int P, int ZBH, int MM, int T0, bool COOL, bool MASK, class WA, int... L>
__device__ __forceinline__ void walk_level_seq(const WA& a, const double* bt_fb,
                                               const double* bt_w, double (&lastF)[P],
                                               double (&lastB)[P], int mlim,
                                               std::integer_sequence<int, L...>) {
  (walk_level<P, ZBH, MM, T0 + L, COOL, MASK>(a, bt_fb, bt_w, lastF, lastB, mlim,
                                              std::make_integer_sequence<int, P>()),
   ...);
}

// Levels [T0, T1) of the MM-micro-batch walk, with the chain state passed in:
// F / B chunks read micro-batch j at bt_fb[j * WA::kStride], W chunks (ZBH)
// at bt_w[j * WA::kStride] (callers shift the pointers to re-base j); with
// COOL the W chunks of the chain's tail (j >= P-1-s) are left to the caller.
// Expanded at compile time (template folds, not a pragma-unrolled loop: the
// long pipelines' walks exceed the unroller's budget, and a loop would
// evaluate the level formulas at run time).
template <int P, int ZBH, int MM, int T0, int T1, bool COOL, class WA, bool MASK = false>
__device__ __forceinline__ void walk_levels(const WA& a, const double* bt_fb,
                                            const double* bt_w, double (&lastF)[P],
                                            double (&lastB)[P], int mlim = MM) {
  walk_level_seq<P, ZBH, MM, T0, COOL, MASK>(a, bt_fb, bt_w, lastF, lastB, mlim,
                                             std::make_integer_sequence<int, T1 - T0>());
}

// Fully unrolled walk for a compile-time micro-batch count: every op, its
// kind and j are constants, so a chunk is ~8 instructions with no dispatch.
template <int P, int ZBH, int MM, class WA>
__device__ __forceinline__ void walk_static(const WA& a) {
  double lastF[P], lastB[P];
#pragma unroll
  for (int s = 0; s < P; ++s) lastF[s] = lastB[s] = 0.0;
  walk_levels<P, ZBH, MM, 0, n_levels(P, MM), false>(a, a.bt, a.bt, lastF, lastB);
}

// Walk for any m >= P micro-batches with a compact steady state.  The level
// pattern of m >= P micro-batches is: levels [0, 2P-1) as for m = P
// (warm-up: every j involved is < P); then m - P level pairs in which every
// stage does one F and one B -- at level 2P-1+2k even stages do B_{k+s/2}
// and odd stages F_{P+k-(s+1)/2}, at the next level even stages do
// F_{P+k-s/2} and odd stages B_{k+(s+1)/2}; then the cool-down, the m = P
// pattern from level 2P-1 on with every F / B j shifted by m - P.  ZBH: the
// cool-down's W chunks with j < P-1-s keep their j, and each stage's chain
// ends with W_j for j = P-1-s .. m-1, walked last (a W chunk feeds only its
// own stage's chain, so only the per-stage chain order matters for it).
// The F / B order (stages descending within a level) and every stage's chain
// order equal the level-ordered walk's; checked against the closed-form
// levels for P <= 8, m < 40 (1F1B) and m < 30 (ZBH).  The steady pair is a
// loop whose body stays in the instruction cache; warm-up and cool-down are
// unrolled.
template <int P, int ZBH, class WA>
__device__ __forceinline__ void walk_steady(const WA& a, int m) {
  double lastF[P], lastB[P];
#pragma unroll
  for (int s = 0; s < P; ++s) lastF[s] = lastB[s] = 0.0;
  walk_levels<P, ZBH, P, 0, 2 * P - 1, false>(a, a.bt, a.bt, lastF, lastB);
  const double* bk = a.bt;
  for (int k = 0; k < m - P; ++k, bk += WA::kStride) {
#pragma unroll
    for (int s = P - 1; s >= 0; --s) {  // level 2P-1+2k
      if (s % 2 == 0) {
        const double dep = s < P - 1 ? __dadd_rn(lastB[s < P - 1 ? s + 1 : 0], a.hb(s)) : 0.0;
        lastB[s] = chunk<true>(a, s, a.rlB(s), WA::ld(bk + (s / 2) * WA::kStride), dep, s == P - 1);
      } else {
        const double dep = __dadd_rn(lastF[s > 0 ? s - 1 : 0], a.hf(s));
        lastF[s] = chunk<true>(a, s, a.rlF(s), WA::ld(bk + (P - (s + 1) / 2) * WA::kStride), dep);
      }
    }
#pragma unroll
    for (int s = P - 1; s >= 0; --s) {  // level 2P+2k
      if (s % 2 == 0) {
        const double dep = s > 0 ? __dadd_rn(lastF[s > 0 ? s - 1 : 0], a.hf(s)) : 0.0;
        lastF[s] = chunk<true>(a, s, a.rlF(s), WA::ld(bk + (P - s / 2) * WA::kStride), dep, s == 0);
      } else {
        const double dep = s < P - 1 ? __dadd_rn(lastB[s < P - 1 ? s + 1 : 0], a.hb(s)) : 0.0;
        lastB[s] = chunk<true>(a, s, a.rlB(s), WA::ld(bk + ((s + 1) / 2) * WA::kStride), dep,
                               s == P - 1);
      }
    }
  }
  walk_levels<P, ZBH, P, 2 * P - 1, n_levels(P, P), true>(a, a.bt + (m - P) * WA::kStride,
                                                          a.bt, lastF, lastB);
  if (ZBH) {
#pragma unroll
    for (int s = P - 1; s >= 0; --s)
      for (int j = P - 1 - s; j < m; ++j)
        chunk<true>(a, s, a.rlW(s), WA::ld(a.bt + j * WA::kStride), 0.0, true);
  }
}

constexpr int kStaticMaxMB = 12;  // RH_STATIC_MAX_MB-style cap on the unrolled walks (m < P in practice)

// Replicas with m >= P take walk_steady, so the kernels carry unrolled walks
// only for m < P (less code competing for the instruction cache); the level
// table covers the rest.
template <int P, int ZBH, int MM = 1, class WA>
__device__ __forceinline__ bool walk_static_dispatch(const WA& a, int mm) {
  if constexpr (MM > P - 1) {
    return false;
  } else {
    if (mm == MM) {
      walk_static<P, ZBH, MM>(a);
      return true;
    }
    return walk_static_dispatch<P, ZBH, MM + 1>(a, mm);
  }
}

// Shared-memory layout of the thread-per-replica kernels:
//   [it_ms | it_st][q: ipb*M int64][off: 16 + 4*(ipb*M+1)][documents -> base costs]
struct CtaStage {
  double* it_ms;
  unsigned* it_st;
  unsigned long long* s_q;
  double* base_t;
  int n_it, n_mb;
};

__device__ __forceinline__ CtaStage cta_layout(const PassParams& p, unsigned char* smem_raw) {
  CtaStage c;
  const int M = p.sh.micro_batches;
  c.it_ms = reinterpret_cast<double*>(smem_raw);
  c.it_st = reinterpret_cast<unsigned*>(c.it_ms + p.ipb);
  const int it_bytes = ((p.ipb * 12 + 15) / 16) * 16;
  c.s_q = reinterpret_cast<unsigned long long*>(smem_raw + it_bytes);
  c.base_t = reinterpret_cast<double*>(smem_raw + p.region_off);
  const int64_t it0 = (int64_t)blockIdx.x * p.ipb;
  c.n_it = (int)min((int64_t)p.ipb, p.tr.n_iter - it0);
  c.n_mb = c.n_it * M;
  return c;
}

// Phase A of the CTA staging: thread 0 arms the mbarrier and issues the TMA
// bulk copies of the offsets and (when they fit) the documents; everybody
// loads the ragged edges.  Per-thread loads issued between stage_begin and
// stage_finish overlap the copies.
struct StageState {
  StagePlan so, sd;
  const int32_t* g_off;
  int32_t d_lo;
  int n_doc;
  bool staged;
};

__device__ __forceinline__ StageState stage_begin(const PassParams& p, unsigned char* smem_raw,
                                                  const CtaStage& c, uint64_t* bar) {
  const int M = p.sh.micro_batches;
  const int it_bytes = ((p.ipb * 12 + 15) / 16) * 16;
  int32_t* s_off_raw = reinterpret_cast<int32_t*>(
      smem_raw + ((it_bytes + 8 * (size_t)p.ipb * M + 15) & ~size_t(15)));
  StageState g;
  const int64_t it0 = (int64_t)blockIdx.x * p.ipb;
  g.g_off = p.tr.mb_off + it0 * M;
  g.d_lo = __ldg(g.g_off);
  g.n_doc = __ldg(g.g_off + c.n_mb) - g.d_lo;
  g.staged = g.n_doc <= p.doc_stage;
  g.so = stage_plan(reinterpret_cast<unsigned char*>(s_off_raw), g.g_off, c.n_mb + 1);
  g.sd = g.staged ? stage_plan(reinterpret_cast<unsigned char*>(c.base_t), p.tr.doc_len + g.d_lo,
                               g.n_doc)
                  : StagePlan{nullptr, 0, 0, 0u};
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_arrive_expect_tx(bar, g.so.tx_bytes + g.sd.tx_bytes);
    stage_issue(g.so, g.g_off, bar);
    if (g.staged) stage_issue(g.sd, p.tr.doc_len + g.d_lo, bar);
  }
  // nobody may poll the barrier before thread 0 has initialised it (the word
  // may still hold a previous CTA's state)
  __syncthreads();
  stage_edges(g.so, g.g_off, c.n_mb + 1);
  if (g.staged) stage_edges(g.sd, p.tr.doc_len + g.d_lo, g.n_doc);
  return g;
}

// Phase B: wait for the copies, then Q_j = sum l^2, one thread per
// micro-batch, into s_q; the document buffer is dead afterwards.
__device__ __forceinline__ void stage_finish(const PassParams& p, const CtaStage& c,
                                             const StageState& g, uint64_t* bar) {
  mbar_wait(bar, 0);  // the bulk copies have landed
  __syncthreads();    // ... and so have the threads' edge words
  const int32_t* s_off = g.so.dst;
  const int32_t* s_doc = g.sd.dst;
  if (p.q32 && g.staged) {
    // 32-bit integer sums: whenever sum l < 2^16, sum l^2 <= (sum l)^2 < 2^32
    // is exact (a packed micro-batch holds N = token_budget tokens); a
    // micro-batch above that is redone in 64-bit
    for (int mb = threadIdx.x; mb < c.n_mb; mb += blockDim.x) {
      const int32_t k0 = s_off[mb] - g.d_lo, k1 = s_off[mb + 1] - g.d_lo;
      const int32_t nd = k1 - k0;
      uint32_t q = 0, sl = 0;
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const uint32_t l = t < nd ? (uint32_t)s_doc[k0 + t] : 0u;
        q += l * l;
        sl += l;
      }
      for (int32_t k = k0 + 4; k < k1; ++k) {
        const uint32_t l = (uint32_t)s_doc[k];
        q += l * l;
        sl += l;
      }
      unsigned long long q64 = q;
      if (sl >= 65536u || nd < 0) {
        q64 = 0;
        for (int32_t k = k0; k < k1; ++k) {
          const long long l = s_doc[k];
          q64 += (unsigned long long)(l * l);
        }
      }
      c.s_q[mb] = q64;
    }
  } else {
  for (int mb = threadIdx.x; mb < c.n_mb; mb += blockDim.x) {
    const int32_t k0 = s_off[mb] - g.d_lo, k1 = s_off[mb + 1] - g.d_lo;
    unsigned long long q = 0;
    if (g.staged) {
      // packed bins hold few documents (C2: 2.4 on average, at most 4): the
      // first four are summed branch-free with predicated loads
      const int32_t nd = k1 - k0;
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const long long l = t < nd ? s_doc[k0 + t] : 0;
        q += (unsigned long long)(l * l);
      }
      for (int32_t k = k0 + 4; k < k1; ++k) {
        const long long l = s_doc[k];
        q += (unsigned long long)(l * l);
      }
    } else {  // too many documents to stage: straight from global memory
      for (int32_t k = k0; k < k1; ++k) {
        const long long l = __ldg(p.tr.doc_len + g.d_lo + k);
        q += (unsigned long long)(l * l);
      }
    }
    c.s_q[mb] = q;
  }
  }
  __syncthreads();  // sums complete; the document buffer is dead from here
}


// pass_wide_kernel (pass_wide.cu): CTA width and the kernel for (P, schedule,
// detect), nullptr when P has no instantiation
// (128-thread CTAs of 4 iterations at 4 CTAs/SM: trace R 2.76 -> 2.72 ms, within
// noise of the per-CTA overheads; 96: 2.93 ms)
constexpr int kWideThreads = 64;
void* wide_kernel_ptr(int P, int zbh, int detect);
size_t wide_tab_bytes(int n_seg, int P);
int wide_prep(const rh_segments& sg, int D, int P, double* tab, cudaStream_t stream);

}  // namespace rh
