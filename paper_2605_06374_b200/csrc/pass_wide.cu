// pass_wide_kernel: the thread-per-replica Detector pass for long 1F1B
// pipelines (5 <= P <= 16, D <= 64) -- SURVEY §8(d)'s trace R and the C3-C5
// shapes -- where a lane per stage (pass_kernel) idles half its DAG levels
// and pays ~45 instructions of level bookkeeping per lane per level.
//
// One THREAD walks one replica pipeline: the chain state (finish and cost
// sum of every stage) lives in registers, and the chunks
// are visited in a topological order that is a few short loops with the
// stage index unrolled at compile time:
//
//   warm-up, by DAG level L = 0..P-1 (four loops over quarters of the
//   levels, each holding only the stages it can touch), stages descending:
//       F_{L-s}(s)                    if s <= L and L-s < m
//   main loop, for i = 0..m-1, stages descending:
//       B_i(s)                        (dependency B_i(s+1): same i, done)
//       F_{P-s+i}(s)                  if P-s+i < m  (dependency
//                                     F_{P-s+i}(s-1): previous i, not yet
//                                     overwritten -- s-1 comes later)
//   walked two steps at a time, step i+1 two stages behind step i, so the two
//   B chains interleave (two_steps).
//
// Each stage's chunks come out in its 1F1B chain order (warm-up Fs, then
// (B_i, F_{w+1+i}) pairs, then the B tail -- pipeline.py:92-126) and every
// chunk after its DAG predecessors, so starts, finishes and chain-order cost
// sums equal the level-ordered walk's bit for bit (any topological order of
// Eq. 2's max/+ relaxation gives the same values).  The loop bodies are a
// few hundred instructions (the unrolled 512-chunk walk streamed 480 KB of
// SASS through a 32 KB instruction cache).
//
// Shared memory per CTA (~27 KB for trace R: 8 CTAs / SM): base costs
// [j][thread], the iteration's ratio * layers and the TMA-staged offsets +
// documents.  Hop weights and stage speeds come from a per-launch transposed
// copy of the segment tables (wide_prep_kernel) that L1 holds for every CTA
// of the SM; speeds are read only on the stages some replica of the warp runs
// slow (a warp-uniform branch; x / 1.0 == x exactly otherwise).
#include "walks.cuh"

namespace rh {

// ld.volatile.shared at a 32-bit shared address plus a compile-time offset
// (folded into the instruction): never cached in a register by the compiler,
// so the per-stage constants cost a load per use instead of pinning ~100
// registers across the walk.
template <int OFF>
__device__ __forceinline__ double lds_at(uint32_t a) {
  double v;
  asm volatile("ld.volatile.shared.f64 %0, [%1+%2];" : "=d"(v) : "r"(a), "n"(OFF));
  return v;
}
__device__ __forceinline__ double lds_rt(uint32_t a) {
  double v;
  asm volatile("ld.volatile.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}
// the same for the L1-resident segment table (read-only global memory)
template <int OFF>
__device__ __forceinline__ double ldg_at(const double* a) {
  double v;
  // volatile: a plain load lets ptxas hoist every table read of the walk
  // (1.5 KB of spills per thread, 2x slower)
  asm volatile("ld.global.nc.f64 %0, [%1+%2];" : "=d"(v) : "l"(a), "n"(OFF));
  return v;
}

// Per-launch transposed segment table (wide_prep_kernel):
//   tab[seg][k][s][kWideTabW], k = 0 hop into stage s on the forward path
//   (hop_fwd[s-1], 0 for s = 0), 1 hop into s on the backward path
//   (hop_bwd[s], 0 for s = P-1), 2 pow2_recip(speed), 3 speed,
//   4 recip_of(speed).
// Replica d of a warp reads column d: every walk load is coalesced, and the
// table of a segment (the same for all its iterations) stays in L1 for every
// CTA of the SM -- shared memory keeps only the per-replica base costs.
constexpr int kWideTabW = 64;
constexpr int kWideTabK = 5;
__device__ __forceinline__ size_t wide_tab_index(int seg, int k, int s, int d, int P) {
  return (((size_t)seg * kWideTabK + k) * P + s) * kWideTabW + d;
}

// 1/b when b is a power of two whose reciprocal is a normal double, else 0:
// then x / b == x * (1/b) exactly for every x (both are the real x * 2^-e,
// rounded once), so the division is one multiply.
__device__ __forceinline__ double pow2_recip(double b) {
  const unsigned long long u = __double_as_longlong(b);
  const int e = (int)((u >> 52) & 0x7ff);
  const bool pow2 = (u >> 63) == 0 && (u & 0xfffffffffffffull) == 0 && e >= 1 && e <= 2045;
  return pow2 ? 1.0 / b : 0.0;
}

// Per (segment, replica) summary of its stage speeds, one word (P <= 16):
// bits 0-15 the stages not at 1.0, kSpRange every such speed in the
// hoisted-reciprocal range, kSpPow2 every such speed a power of two, kSpStop
// some speed <= 0 -- one load in the kernel instead of P.
enum : uint32_t { kSpRange = 1u << 16, kSpPow2 = 1u << 17, kSpStop = 1u << 18 };

__global__ void wide_prep_kernel(const rh_segments sg, int D, int P, double* tab) {
  {
    uint32_t* flags = reinterpret_cast<uint32_t*>(tab + (size_t)sg.n_seg * kWideTabK * P * kWideTabW);
    const int64_t nr = (int64_t)sg.n_seg * D;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nr;
         r += (int64_t)gridDim.x * blockDim.x) {
      const int d = (int)(r % D), seg = (int)(r / D);
      uint32_t w = kSpRange | kSpPow2;
      for (int s = 0; s < P; ++s) {
        const double sp = sg.speed[r * P + s];
        if (sp != 1.0) {
          w |= 1u << s;
          if (!(sp >= 0x1p-100 && sp <= 0x1p100)) w &= ~kSpRange;  // recip_of(sp) == 0
          if (pow2_recip(sp) == 0.0) w &= ~kSpPow2;
        }
        if (sp <= 0.0) w |= kSpStop;
      }
      flags[(size_t)seg * kWideTabW + d] = w;
    }
  }
  const int64_t n = (int64_t)sg.n_seg * D * P;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int s = (int)(i % P), d = (int)((i / P) % D), seg = (int)(i / ((int64_t)P * D));
    const int64_t g = ((int64_t)seg * D + d) * P + s;  // [seg][d][s]
    const double sp = sg.speed[g];
    tab[wide_tab_index(seg, 0, s, d, P)] = s > 0 ? sg.hop_fwd[g - 1] : 0.0;
    tab[wide_tab_index(seg, 1, s, d, P)] = s < P - 1 ? sg.hop_bwd[g] : 0.0;
    tab[wide_tab_index(seg, 2, s, d, P)] = pow2_recip(sp);
    tab[wide_tab_index(seg, 3, s, d, P)] = sp;
    tab[wide_tab_index(seg, 4, s, d, P)] = recip_of(sp);
  }
}

// How a walk divides a chunk's cost by a slow stage's speed: kDivScale, every
// slow speed of the warp is a power of two (one exact multiply); kDivFast, the
// hoisted-reciprocal form (operands range-checked); kDivExact, __ddiv_rn.
enum { kDivScale = 0, kDivFast = 1, kDivExact = 2 };

// One replica's walk: shared addresses of its base costs [j][TW] and its
// iteration's ratio * layers [rlF: P][rlB: P]; its column of the segment
// table; the chain state (finish and cost sum of every stage) in registers.
// A stage's last F finish is never kept apart from its chain finish: when
// F(S) reads stage S-1's last F, that F is stage S-1's latest chunk (warm-up:
// its chunk of the previous DAG level; main loop: the previous step's, S-1 not
// yet visited this step), so fin[S-1] is that finish -- 2P doubles of state.
template <int P, int TW, int MODE>
struct WideWalk {
  uint32_t bt, rl;   // shared addresses (this thread's column / iteration row)
  const double* tb;  // this replica's column of the segment table
  unsigned slow;  // warp-uniform: bit s = some replica of the warp runs stage s slow
  double fin[P], ssum[P];

  template <int K, int S>
  __device__ __forceinline__ double tab() const {
    return ldg_at<(K * P + S) * kWideTabW * 8>(tb);
  }
  // start = max(chain finish, dependency finish + hop); finish = start + c;
  // cost sum in chain order (pipeline.py:275-291, 446-453)
  // NODEP: no data dependency (dep == 0.0): start = chain finish (a finish
  // is a sum of non-negative costs from +0.0; see walks.cuh chunk())
  template <int S, bool NODEP = false>
  __device__ __forceinline__ double step(double c, double dep) {
    const double st = (NODEP || fin[S] > dep) ? fin[S] : dep;
    fin[S] = __dadd_rn(st, c);
    ssum[S] = __dadd_rn(ssum[S], c);
    return fin[S];
  }
  // one chunk of cost c = (rl * b) / speed, exactly as __ddiv_rn (MODE: one
  // multiply by 1/speed for power-of-two speeds, the hoisted-reciprocal form
  // after the kernel's operand-range check, or __ddiv_rn out of line),
  // skipped on unit-speed stages (x / 1.0 == x).  ptxas predicates the
  // division (no branch): a
  // branch per chunk -- warp-uniform, or around an IEEE division -- splits
  // the walk into basic blocks it cannot interleave, and measured slower
  // (trace R 376 -> 442-480 us per 10^4 iterations).
  template <int S, bool NODEP = false>
  __device__ __forceinline__ double chunk(double rl_, double b_, double dep) {
    double c = __dmul_rn(rl_, b_);
    if (slow & (1u << S)) {  // warp-uniform
      if (MODE == kDivScale) {
        c = __dmul_rn(c, tab<2, S>());
      } else {
        const double sp = tab<3, S>();
        c = MODE == kDivExact ? div_slow(c, sp) : div_fast(c, sp, tab<4, S>());
      }
    }
    return step<S, NODEP>(c, dep);
  }
  // warm-up in DAG-level order: level L holds F_{L-S}(S) for every S <= L
  // (j = L - S < m); they are independent (F_{L-S}(S) needs stage S-1's chunk
  // of level L-1 and stage S's own), so a level is up to P-way ILP where the
  // stage-ascending triangle is one serial chain per step.  Stages descend so
  // fin[S-1] still holds level L-1's finish.
  template <int S>
  __device__ __forceinline__ void warm(int L, int m, uint32_t brow) {
    if (L >= S && L - S < m) {
      const double dep = S > 0 ? __dadd_rn(fin[S > 0 ? S - 1 : 0], tab<0, S>()) : 0.0;
      chunk<S, S == 0>(lds_at<S * 8>(rl), lds_at<-S * TW * 8>(brow), dep);
    }
  }
  template <int... I>
  __device__ __forceinline__ void warm_all(int L, int m, uint32_t brow, std::integer_sequence<int, I...>) {
    constexpr int NS = sizeof...(I);
    (warm<NS - 1 - I>(L, m, brow), ...);  // S = NS-1, ..., 0
  }
  // levels [L0, L1) touch stages S <= L < L1 only: a quarter of the levels per
  // loop, each loop's body holding just the stages it can touch
  template <int Q>
  __device__ __forceinline__ void warm_quarter(int m) {
    constexpr int L0 = Q * P / 4, L1 = (Q + 1) * P / 4;
#pragma unroll 1
    for (int L = L0; L < L1; ++L)
      warm_all(L, m, bt + (uint32_t)(L * TW * 8), std::make_integer_sequence<int, L1>());
  }
  // main-loop slot (stages descending): B_i(S), then F_{P-S+i}(S) if it exists
  // (tried branch-free, a missing F costing +0.0 from a predicated load:
  // 423 -> 459 us per 10^4 trace-R iterations)
  template <int S>
  __device__ __forceinline__ void pair(int i, int m, double bi, double& nB) {
    const double depB = S < P - 1 ? __dadd_rn(nB, tab<1, S>()) : 0.0;
    nB = chunk<S, S == P - 1>(lds_at<(P + S) * 8>(rl), bi, depB);
    if (i < m - P + S) {
      const double bF = lds_rt(bt + (uint32_t)((P - S + i) * TW * 8));
      const double dep = S > 0 ? __dadd_rn(fin[S > 0 ? S - 1 : 0], tab<0, S>()) : 0.0;
      chunk<S, S == 0>(lds_at<S * 8>(rl), bF, dep);
    }
  }
  template <int... I>
  __device__ __forceinline__ void pair_all(int i, int m, double bi,
                                           std::integer_sequence<int, I...>) {
    double nB = 0.0;  // B_i of the stage above
    (pair<P - 1 - I>(i, m, bi, nB), ...);  // S = P-1, ..., 0
  }
  // Two main-loop steps at once, step i+1 two stages behind step i: at tick T
  // step i does stage P-1-T and step i+1 stage P+1-T.  Every read still sees
  // what the sequential order gives it (step i+1's B(s) follows step i's
  // chunks of stage s, done two ticks before; its F(s) reads stage s-1 after
  // step i, done the tick before and not yet touched by step i+1; step i reads
  // stages step i+1 reaches only later), and the two B chains interleave:
  // trace R 2.69 -> 2.58 ms.  (Three or four steps: register spills, 2.67 /
  // 3.89 ms.)
  template <int S>
  __device__ __forceinline__ void half_b(double bi, double& nB) {
    const double depB = S < P - 1 ? __dadd_rn(nB, tab<1, S>()) : 0.0;
    nB = chunk<S, S == P - 1>(lds_at<(P + S) * 8>(rl), bi, depB);
  }
  template <int S>
  __device__ __forceinline__ void half_f(int i, int m) {
    if (i < m - P + S) {
      const double bF = lds_rt(bt + (uint32_t)((P - S + i) * TW * 8));
      const double dep = S > 0 ? __dadd_rn(fin[S > 0 ? S - 1 : 0], tab<0, S>()) : 0.0;
      chunk<S, S == 0>(lds_at<S * 8>(rl), bF, dep);
    }
  }
  template <int T>
  __device__ __forceinline__ void tick(int i, int m, double b0, double b1, double& n0, double& n1) {
    constexpr int SA = P - 1 - T, SB = P + 1 - T;
    if constexpr (SA >= 0) half_b<SA>(b0, n0);
    if constexpr (SB >= 0 && SB < P) half_b<SB>(b1, n1);
    if constexpr (SA >= 0) half_f<SA>(i, m);
    if constexpr (SB >= 0 && SB < P) half_f<SB>(i + 1, m);
  }
  template <int... T>
  __device__ __forceinline__ void two_steps(int i, int m, double b0, double b1,
                                            std::integer_sequence<int, T...>) {
    double n0 = 0.0, n1 = 0.0;
    (tick<T>(i, m, b0, b1, n0, n1), ...);
  }
  // (Tried: the next stage's table / shared loads issued before this stage's
  // chunk (software-pipelined operands): spills, 352 -> 362-388 us.)
  // (Round 2 tried K groups of stages skewed by one loop step each: the
  // per-group validity and slow-stage branches kept the compiler from
  // interleaving them, 463 -> 520 us per 10^4 iterations; with the division
  // predicated and the steps skewed two stages apart it pays, above.
  // A level-ordered walk -- the P chunks of a DAG level are independent --
  // issued more, not faster: tools/walkbench.cu, 1.57 -> 2.1 ms branch-free.)
  __device__ __forceinline__ void walk(int m) {
#pragma unroll
    for (int s = 0; s < P; ++s) fin[s] = ssum[s] = 0.0;
    warm_quarter<0>(m);  // (the stage-ascending triangle per j: 350 -> 344 us)
    warm_quarter<1>(m);
    warm_quarter<2>(m);
    warm_quarter<3>(m);
    int i = 0;
#pragma unroll 1
    for (; i + 1 < m; i += 2)
      two_steps(i, m, lds_rt(bt + (uint32_t)(i * TW * 8)), lds_rt(bt + (uint32_t)((i + 1) * TW * 8)),
                std::make_integer_sequence<int, P + 2>());
    if (i < m)  // odd m: the last step alone
      pair_all(i, m, lds_rt(bt + (uint32_t)(i * TW * 8)), std::make_integer_sequence<int, P>());
  }
};

#ifdef RH_WIDE_TRACE
// debug build only (tools/wide_trace.py): per CTA, thread 0's globaltimer at
// the phase boundaries of pass_wide_kernel
__device__ unsigned long long g_wtrace[4096 * 8];
__device__ __forceinline__ void wmark(int k) {
  if (threadIdx.x == 0 && blockIdx.x < 4096) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_wtrace[blockIdx.x * 8 + k] = t;
  }
}
#define RH_WMARK(k) wmark(k)
#else
#define RH_WMARK(k) ((void)0)
#endif

// CTAs per SM the register budget targets: with the hop / speed tables in L1
// and the chain state at 2P doubles, 8 CTAs (16 warps) fit every P <= 16 in
// 128 registers; shared memory (base costs + staging, ~27 KB for trace R)
// allows the same.  (tools/walkbench.cu: 10 -> 16 warps per SM took the
// trace-R walk from 1.57 to 1.03 ms; more warps than that did not help.)
#ifndef RH_WIDE_DTPF
#define RH_WIDE_DTPF 2  // device-time L2 prefetch: 0 CTA start, 1 none, 2 before the walk
#endif
#ifndef RH_WIDE_DT_UNROLL
#define RH_WIDE_DT_UNROLL 8
#endif
constexpr int kWideDtUnroll = RH_WIDE_DT_UNROLL;  // device-time rows in flight per thread
#ifdef RH_WIDE_MINB
constexpr int kWideMinBlocks = RH_WIDE_MINB;  // A/B builds
#else
constexpr int kWideMinBlocks = 8;
#endif

template <int P, int DETECT>
__global__ void __launch_bounds__(kWideThreads, kWideMinBlocks) pass_wide_kernel(const PassParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int TW = kWideThreads;
  const int tid = threadIdx.x;
  const int D = p.sh.dp, M = p.sh.micro_batches, T = p.sh.tp;
  const int li = tid / D, d = tid - li * D;
  const int64_t it0 = (int64_t)blockIdx.x * p.ipb;
  const int64_t it = it0 + li;
  const int n_it = (int)min((int64_t)p.ipb, p.tr.n_iter - it0);
  const bool on = li < n_it;
  double* it_ms = reinterpret_cast<double*>(smem_raw);
  unsigned* it_st = reinterpret_cast<unsigned*>(it_ms + p.ipb);
  double* base_t = reinterpret_cast<double*>(smem_raw + p.w_base);
  double* s_rl = reinterpret_cast<double*>(smem_raw + p.w_rl);
  __shared__ uint64_t s_bar;
  RH_WMARK(0);
  if (tid < p.ipb) {
    it_ms[tid] = 0.0;
    it_st[tid] = 0u;
  }
  // ---- the replica's segment: its loads are issued first, so their latency
  // overlaps the staging below (consumed after its barrier)
  const int seg = on && p.tr.seg ? __ldg(p.tr.seg + it) : 0;
  // ---- TMA staging of the CTA's micro-batch offsets and documents
  const int n_mb = n_it * M;
  const int32_t* g_off = p.tr.mb_off + it0 * M;
  const int32_t d_lo = __ldg(g_off), n_doc = __ldg(g_off + n_mb) - d_lo;
  int m0 = 0, md = 0;
  if (on) {
    const int32_t* ms = p.sg.mb_start + (int64_t)seg * (D + 1);
    m0 = __ldg(ms + d);
    md = __ldg(ms + d + 1) - m0;
  }
  const double* tb = p.wtab + wide_tab_index(seg, 0, 0, d, P);
  const uint32_t spw =
      on ? __ldg(reinterpret_cast<const uint32_t*>(p.wtab + (size_t)p.sg.n_seg * kWideTabK * P * kWideTabW) +
                 (size_t)seg * kWideTabW + d)
         : kSpRange | kSpPow2;
  // this thread's first ratio * layers entry (stage d)
  const int32_t L_d = on && d < P ? __ldg(p.sg.layers + (int64_t)seg * P + d) : 0;
  const bool staged = n_doc <= p.doc_stage;
  const StagePlan so = stage_plan(smem_raw + p.w_union, g_off, n_mb + 1);
  const StagePlan sd = staged ? stage_plan(smem_raw + p.w_docs, p.tr.doc_len + d_lo, n_doc)
                              : StagePlan{nullptr, 0, 0, 0u};
  if (tid == 0) {
    mbar_init(&s_bar, 1);
    mbar_arrive_expect_tx(&s_bar, so.tx_bytes + sd.tx_bytes);
    stage_issue(so, g_off, &s_bar);
    if (staged) stage_issue(sd, p.tr.doc_len + d_lo, &s_bar);
#if RH_WIDE_DTPF == 0
    if (DETECT)  // reduced after the walk: pull the rows into L2 now
      prefetch_l2(p.tr.device_time + it0 * D * P * T, 4 * (size_t)n_it * D * P * T);
#endif
    const int64_t nb = (int64_t)blockIdx.x + p.pf_stride;
    if (p.pf_stride > 0 && nb < gridDim.x) {  // the next wave's inputs
      const int64_t pf_it = nb * p.ipb;
      const int pf_nmb = (int)min((int64_t)p.ipb, p.tr.n_iter - pf_it) * M;
      const int32_t lo = __ldg(p.tr.mb_off + pf_it * M);
      const int32_t hi = __ldg(p.tr.mb_off + pf_it * M + pf_nmb);
      prefetch_l2(p.tr.mb_off + pf_it * M, 4 * (size_t)(pf_nmb + 1));
      prefetch_l2(p.tr.doc_len + lo, 4 * (size_t)(hi - lo));
    }
  }
  __syncthreads();  // the barrier is initialised before anybody polls it
  stage_edges(so, g_off, n_mb + 1);
  if (staged) stage_edges(sd, p.tr.doc_len + d_lo, n_doc);
  // ---- per-replica inputs (overlap the copies)
  if (on)  // the iteration's ratio * layers (the same for all its replicas)
    for (int s = d; s < P; s += D) {
      const double L = (double)(s == d ? L_d : __ldg(p.sg.layers + (int64_t)seg * P + s));
      s_rl[li * 2 * P + s] = __dmul_rn(p.m.ratio_f, L);
      s_rl[li * 2 * P + P + s] = __dmul_rn(__dadd_rn(p.m.ratio_b, p.m.ratio_w), L);
    }
  // the replica's speed summary (wide_prep_kernel): slow stages, divisor range,
  // power-of-two slow speeds, a stopped stage
  bool stopped = (spw & kSpStop) != 0, safe = (spw & kSpRange) != 0;
  const bool pow2 = (spw & kSpPow2) != 0;
  unsigned slow = spw & 0xffffu;
  bool link_bad = false;  // the segment's exercised-link test, issued before the wait
  if (DETECT && on && p.sg.link_off && p.sg.link_max) {  // one compare (segment maximum)
    link_bad = __ldg(p.sg.link_max + seg) > p.thr;
  } else if (DETECT && on && p.sg.link_off) {  // exercised-link ratios, split over the replicas
    const int32_t q0 = __ldg(p.sg.link_off + seg), q1 = __ldg(p.sg.link_off + seg + 1);
    int32_t q = q0 + d;
    for (; q + 3 * D < q1; q += 4 * D) {
      const double a = __ldg(p.sg.link_ratio + q), b = __ldg(p.sg.link_ratio + q + D),
                   c = __ldg(p.sg.link_ratio + q + 2 * D), e = __ldg(p.sg.link_ratio + q + 3 * D);
      link_bad = link_bad || a > p.thr || b > p.thr || c > p.thr || e > p.thr;
    }
    for (; q < q1; q += D) link_bad = link_bad || __ldg(p.sg.link_ratio + q) > p.thr;
  }
  RH_WMARK(1);
  mbar_wait(&s_bar, 0);  // the bulk copies have landed
  __syncthreads();       // ... and so have the threads' edge words
  RH_WMARK(2);
  // ---- Q_j = sum l^2 and base costs alpha*N + beta*Q_j, one thread per replica
  if (md > p.mmax) md = -1;
  const int m = md > 0 ? md : 0;
  double b_lo = CUDART_INF, b_hi = 0.0;  // base-cost range (non-zero minimum)
  if (m > 0) {
    const double lin = __dmul_rn(p.m.alpha, (double)p.sh.token_budget);
    const int32_t* s_off = so.dst + li * M + m0;
    const auto put = [&](int j, double q) {
      const double b = __dadd_rn(lin, __dmul_rn(p.m.beta, q));
      base_t[j * TW + tid] = b;
      b_hi = b > b_hi ? b : b_hi;
      if (b > 0.0 && b < b_lo) b_lo = b;
    };
    if (staged) {
      // 32-bit sums, the first 4 documents of a micro-batch unrolled: whenever
      // sum l < 2^16, sum l^2 <= (sum l)^2 < 2^32 is exact; a micro-batch above
      // that (or with a negative length) is redone in 64-bit.  Two
      // micro-batches per step, their heads side by side (independent chains)
      const int32_t* doc = sd.dst;
      const auto redo = [&](int32_t k0, int32_t k1) {
        unsigned long long q = 0;
        for (int32_t k = k0; k < k1; ++k) {
          const long long l = doc[k];
          q += (unsigned long long)(l * l);
        }
        return (double)(long long)q;
      };
      int32_t kb = s_off[0] - d_lo;
      for (int j = 0; j < m; j += 2) {
        const bool two = j + 1 < m;
        const int32_t k0 = kb, k1 = s_off[j + 1] - d_lo, k2 = two ? s_off[j + 2] - d_lo : k1;
        kb = k2;
        const int32_t na = k1 - k0, nb = k2 - k1;
        uint32_t qa = 0, sa = 0, qb = 0, sb = 0;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const uint32_t la = t < na ? (uint32_t)doc[k0 + t] : 0u;
          const uint32_t lb = t < nb ? (uint32_t)doc[k1 + t] : 0u;
          qa += la * la;
          sa += la;
          qb += lb * lb;
          sb += lb;
        }
        for (int32_t k = k0 + 4; k < k1; ++k) {
          const uint32_t l = (uint32_t)doc[k];
          qa += l * l;
          sa += l;
        }
        for (int32_t k = k1 + 4; k < k2; ++k) {
          const uint32_t l = (uint32_t)doc[k];
          qb += l * l;
          sb += l;
        }
        put(j, sa >= 65536u || na < 0 ? redo(k0, k1) : (double)qa);
        if (two) put(j + 1, sb >= 65536u || nb < 0 ? redo(k1, k2) : (double)qb);
      }
    } else {
      for (int j = 0; j < m; ++j) {
        const int32_t k0 = s_off[j] - d_lo, k1 = s_off[j + 1] - d_lo;
        unsigned long long q = 0;
        for (int32_t k = k0; k < k1; ++k) {
          const long long l = __ldg(p.tr.doc_len + d_lo + k);
          q += (unsigned long long)(l * l);
        }
        put(j, (double)(long long)q);
      }
    }
  }
  RH_WMARK(7);
  if (m == 0) {  // nothing runs: no speeds, no costs
    slow = 0;
    stopped = false;
    safe = true;
  }
  const double* rl = s_rl + li * 2 * P;
  __syncthreads();  // ratio * layers visible
  if (slow && m > 0) {  // exact hoisted-reciprocal division needs in-range operands
    double r_lo = CUDART_INF, r_hi = 0.0;
#pragma unroll
    for (int s = 0; s < P; ++s) {
      const double f = rl[s], bw = rl[P + s];
      r_hi = f > r_hi ? f : r_hi;
      r_hi = bw > r_hi ? bw : r_hi;
      if (f > 0.0 && f < r_lo) r_lo = f;
      if (bw > 0.0 && bw < r_lo) r_lo = bw;
    }
    safe = safe && div_range_ok(r_lo * b_lo, r_hi * b_hi);
  }
  const int mm = stopped ? 0 : m;
  const bool over = p.sh.capacity > 0 && mm > 0 && __ldg(p.sched_peak + mm) > p.sh.capacity;
  const unsigned wslow = __reduce_or_sync(0xffffffffu, mm > 0 ? slow : 0u);
  double fin[P], ssum[P];
#pragma unroll
  for (int s = 0; s < P; ++s) fin[s] = ssum[s] = 0.0;
  // (Tried: a warp whose replicas all walk the same micro-batch count taking
  // that count from a warp reduction, so ptxas sees uniform loop bounds and
  // validity tests -- no gain, 481 vs 481 us.)
  RH_WMARK(3);
  const uint32_t a_bt = smem_u32(base_t + tid), a_rl = smem_u32(rl);
#if RH_WIDE_DTPF == 2
  // the rows the epilogue reduces: pulled into L2 as the walk starts (at the
  // CTA's start they were partly evicted again by the time the walk ended:
  // DRAM reads 1.4x the algorithmic bytes; trace R 3.00 -> 2.96 ms)
  if (DETECT && tid == 0)
    prefetch_l2(p.tr.device_time + it0 * D * P * T, 4 * (size_t)n_it * D * P * T);
#endif
#ifdef RH_WIDE_NO_POW2
  const bool wpow2 = false;
#else
  const bool wpow2 = __all_sync(0xffffffffu, pow2 || mm == 0);
#endif
  // A warp whose replicas all walk the same micro-batch count takes that count
  // from a warp reduction (CREDUX, a uniform register): ptxas then knows the
  // loop bounds and chunk-validity tests are warp-uniform and drops the
  // divergence bookkeeping (BSSY/BSYNC) around every chunk (2.775 -> 2.685 ms)
  const int mu = __reduce_min_sync(0xffffffffu, mm);
  const bool wuni = __all_sync(0xffffffffu, mm == mu);
#ifdef RH_WIDE_NOWALK
  if (mm > 0 && p.thr < -1.0) {
#else
  if (mm > 0) {
#endif
    if (wpow2) {  // every slow speed of the warp a power of two (0.5, 0.25, ...)
      WideWalk<P, TW, kDivScale> w{a_bt, a_rl, tb, wslow, {}, {}};
      if (wuni)
        w.walk(mu);
      else
        w.walk(mm);
#pragma unroll
      for (int s = 0; s < P; ++s) fin[s] = w.fin[s], ssum[s] = w.ssum[s];
    } else if (safe) {
      WideWalk<P, TW, kDivFast> w{a_bt, a_rl, tb, wslow, {}, {}};
      w.walk(mm);  // (a uniform-count instance here: no change; mixed counts in trace R)
#pragma unroll
      for (int s = 0; s < P; ++s) fin[s] = w.fin[s], ssum[s] = w.ssum[s];
    } else {  // operands outside the hoisted-reciprocal range
      WideWalk<P, TW, kDivExact> w{a_bt, a_rl, tb, wslow, {}, {}};
      w.walk(mm);
#pragma unroll
      for (int s = 0; s < P; ++s) fin[s] = w.fin[s], ssum[s] = w.ssum[s];
    }
  }
  RH_WMARK(4);
  // ---- replica makespan, validation, iteration reductions
  unsigned bits = 0;
  uint32_t flags = 0;  // bit s: stage s flagged
  // measured stage times (max over the TP group's device times, float4
  // loads) land in the staging region, dead since the base costs: a register
  // array indexed in a partially unrolled loop would live in local memory
  float* s_meas = reinterpret_cast<float*>(smem_raw + p.w_union);
  if (on) {
    double g = 0.0;
#pragma unroll
    for (int s = 0; s < P; ++s) g = fmax(g, fin[s]);
    if (md < 0) bits |= RH_IT_OVERFLOW;
    if (stopped && m > 0) bits |= RH_IT_STOPPED;
    if (over) bits |= RH_IT_CAPACITY;
    if (p.sh.has_allreduce && D > 1) g = __dadd_rn(g, __ldg(p.sg.allreduce + (int64_t)seg * D + d));
    atomic_max_nonneg(it_ms + li, g);
    if (DETECT && md >= 0) {
      const float* dt = p.tr.device_time + (it * D + d) * P * (int64_t)T;
      if (p.vec4 && T == 8) {
#pragma unroll kWideDtUnroll
        for (int s = 0; s < P; ++s) {
          const float4 v = __ldg(reinterpret_cast<const float4*>(dt + s * 8));
          const float4 w = __ldg(reinterpret_cast<const float4*>(dt + s * 8 + 4));
          s_meas[s * TW + tid] = fmaxf(fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w)),
                                       fmaxf(fmaxf(w.x, w.y), fmaxf(w.z, w.w)));
        }
      } else {
#pragma unroll 4
        for (int s = 0; s < P; ++s) {
          float mx = 0.0f;
          if (p.vec4) {
            for (int q = 0; q < T; q += 4) {
              const float4 v = __ldg(reinterpret_cast<const float4*>(dt + s * T + q));
              mx = fmaxf(mx, fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w)));
            }
          } else {
            for (int q = 0; q < T; ++q) mx = fmaxf(mx, __ldg(dt + s * T + q));
          }
          s_meas[s * TW + tid] = mx;
        }
      }
#pragma unroll
      for (int s = 0; s < P; ++s) {
        const double ms_d = (double)s_meas[s * TW + tid];
        if (!(ssum[s] <= 0.0 || ms_d <= 0.0) && ms_d > __dmul_rn(p.thr, ssum[s])) {
          flags |= 1u << s;
          bits |= RH_IT_STAGE_FLAG;
        }
      }
    }
    if (link_bad) bits |= RH_IT_LINK_FLAG;
    if (bits) atomicOr(it_st + li, bits);
  }
  RH_WMARK(5);
  __syncthreads();
  if (!on) return;
  const unsigned st_bits = it_st[li];
  const bool dead = (st_bits & (RH_IT_STOPPED | RH_IT_OVERFLOW)) != 0;
  // a replica's P outputs are contiguous: vector stores when P and the
  // caller's pointer allow (4 flags per u32, float4 severities, double2 costs)
  const int64_t o0 = (it * D + d) * P;
  const auto al = [](const void* q, unsigned a) { return (reinterpret_cast<uintptr_t>(q) & (a - 1)) == 0; };
  if (p.out.stage_cost) {
    if (P % 2 == 0 && al(p.out.stage_cost, 16)) {
#pragma unroll
      for (int s = 0; s < P; s += 2)
        *reinterpret_cast<double2*>(p.out.stage_cost + o0 + s) =
            dead ? make_double2(0.0, 0.0) : make_double2(ssum[s], ssum[s + 1 < P ? s + 1 : s]);
    } else {
#pragma unroll
      for (int s = 0; s < P; ++s) p.out.stage_cost[o0 + s] = dead ? 0.0 : ssum[s];
    }
  }
  if (DETECT) {
    const uint32_t fl = dead ? 0u : flags;
    if (p.out.stage_flag) {
      if (P % 4 == 0 && al(p.out.stage_flag, 4)) {
#pragma unroll
        for (int s = 0; s < P; s += 4)
          *reinterpret_cast<uint32_t*>(p.out.stage_flag + o0 + s) =
              ((fl >> s) & 1u) | (((fl >> (s + 1)) & 1u) << 8) | (((fl >> (s + 2)) & 1u) << 16) |
              (((fl >> (s + 3)) & 1u) << 24);
      } else {
#pragma unroll
        for (int s = 0; s < P; ++s) p.out.stage_flag[o0 + s] = (fl >> s) & 1u;
      }
    }
    if (p.out.severity) {
      float sev[P];
#pragma unroll
      for (int s = 0; s < P; ++s)
        sev[s] = ((fl >> s) & 1u) ? (float)__ddiv_rn(ssum[s], (double)s_meas[s * TW + tid]) : 0.0f;
      if (P % 4 == 0 && al(p.out.severity, 16)) {
#pragma unroll
        for (int s = 0; s < P; s += 4)
          *reinterpret_cast<float4*>(p.out.severity + o0 + s) =
              make_float4(sev[s], sev[(s + 1) % P], sev[(s + 2) % P], sev[(s + 3) % P]);
      } else {
#pragma unroll
        for (int s = 0; s < P; ++s) p.out.severity[o0 + s] = sev[s];
      }
    }
  }
  if (d == 0) {
    unsigned st = st_bits;
    double ms = dead ? 0.0 : it_ms[li];
    if (dead) st &= (RH_IT_STOPPED | RH_IT_OVERFLOW);
    if (DETECT && !dead) {
      const double obs = __ldg(p.tr.observed + it);
      if (ms <= 0.0 || obs > __dmul_rn(p.thr, ms)) st |= RH_IT_ESCALATE;
    }
    p.out.makespan[it] = ms;
    p.out.status[it] = (uint8_t)st;
  }
  RH_WMARK(6);
}

template <int DETECT>
static void* wide_kernel_t(int P) {
  switch (P) {
#define RH_WIDE_CASE(n) \
  case n:               \
    return (void*)pass_wide_kernel<n, DETECT>;
    RH_WIDE_CASE(5)
    RH_WIDE_CASE(6)
    RH_WIDE_CASE(7)
    RH_WIDE_CASE(8)
    RH_WIDE_CASE(9)
    RH_WIDE_CASE(10)
    RH_WIDE_CASE(11)
    RH_WIDE_CASE(12)
    RH_WIDE_CASE(13)
    RH_WIDE_CASE(14)
    RH_WIDE_CASE(15)
    RH_WIDE_CASE(16)
#undef RH_WIDE_CASE
    default: return nullptr;
  }
}

void* wide_kernel_ptr(int P, int zbh, int detect) {
  if (zbh) return nullptr;  // ZBH long pipelines: the lane kernel
  return detect ? wide_kernel_t<1>(P) : wide_kernel_t<0>(P);
}

#ifdef RH_WIDE_TRACE
extern "C" int rh_debug_wide_trace(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, g_wtrace, sizeof(g_wtrace)) == cudaSuccess ? 0 : 1;
}
#endif

size_t wide_tab_bytes(int n_seg, int P) {
  return (size_t)n_seg * kWideTabK * P * kWideTabW * 8 + (size_t)n_seg * kWideTabW * 4;
}

int wide_prep(const rh_segments& sg, int D, int P, double* tab, cudaStream_t stream) {
  const int64_t n = (int64_t)sg.n_seg * D * P;
  if (n == 0) return RH_OK;
  const int blocks = (int)std::min<int64_t>((n + 255) / 256, 1024);
  wide_prep_kernel<<<blocks, 256, 0, stream>>>(sg, D, P, tab);
  RH_CUDA(cudaGetLastError());
  return RH_OK;
}

}  // namespace rh
