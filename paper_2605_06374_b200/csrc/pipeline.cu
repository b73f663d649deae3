// Fused pipeline predictor + Detector residual pass (rh_pipeline_batch,
// rh_detect_batch, rh_detect_batch_host).
//
// What it computes, per iteration i of the batch:
//   Q_j   = sum of squared doc lengths of micro-batch j      (workload.py:83-85)
//   c(v)  = ((ratio(kind)*L_s) * (alpha*N + beta*Q_j)) / p   (workload.py:88-98)
//   start(v) = max(finish(chain predecessor), finish(data predecessor) + hop)
//   makespan = max_d ( max_s finish(last chunk of (d,s)) + AR_d )
//              — the critical path of build_dag's canonical DAG
//              (pipeline.py:129-292), evaluated as a wavefront
//   stage_cost[d][s] = sum of c(v) over the (d,s) chain, in chain order
//              (pipeline.py:446-453)
//   detect: filter verdict observed > thr*makespan (detector.py:111-116) and
//           per-(d,s) flag measured > thr*stage_cost, severity
//           stage_cost/measured (detector.py:127-158), measured = max over
//           the group's member device times (float4 loads).
//
// Two mappings (launch_pass picks one per launch):
//   pass_small_kernel (P <= 4, D <= 128): one THREAD per replica pipeline,
//     all stage state in registers, chunks in DAG-level order (steady-state
//     loop walk for 1F1B, fully unrolled for small micro-batch counts, level
//     table otherwise); see below.
//   pass_kernel (P <= 32): one replica pipeline = `pw` lanes (pw =
//     next_pow2(P), lane s = stage s); each lane walks its chain with the
//     branch-free static level walk of wavefront.cuh, neighbours exchange the
//     last F / B finish by warp shuffle.
// In both, all D pipelines of an iteration sit in one CTA and reduce the
// makespan through shared memory.  All fp64 ops use explicit _rn
// intrinsics: no FMA contraction anywhere.
#include <algorithm>
#include <type_traits>
#include <utility>

#include <math_constants.h>

#include "common.cuh"
#include "wavefront.cuh"
#include "walks.cuh"

namespace rh {

// Lane walk driven by a host-built level table (lane_table): for the
// replica's micro-batch count mm, codes[t * P + s] is stage s's chunk at DAG
// level t (0 idle, else kind | j << 2).  Same arithmetic and exchange as
// chain_walk, without the closed-form level bookkeeping.
template <int ZBH>
__device__ __forceinline__ void chain_walk_table(int s, int P, int pw, int mm,
                                                 const uint16_t* codes, int n_lev,
                                                 const double* base, double rlF, double rlB,
                                                 double rlW, double sp, double hopf,
                                                 double hopb, double& fin, double& ssum) {
  const bool unit = sp == 1.0;
  const double inv = unit ? 1.0 : recip_of(sp);
  const int T = __reduce_max_sync(0xffffffffu, mm > 0 ? n_lev : 0);
  const double hF = s > 0 ? hopf : 0.0, hB = s < P - 1 ? hopb : 0.0;
  const bool getF = s > 0, getB = s < P - 1;
  const bool mine = mm > 0 && s < P;
  double lastF = 0.0, lastB = 0.0;
  for (int t = 0; t < T; ++t) {
    const double nF = __shfl_up_sync(0xffffffffu, lastF, 1, pw);
    const double nB = __shfl_down_sync(0xffffffffu, lastB, 1, pw);
    const unsigned code = (mine && t < n_lev) ? (unsigned)__ldg(codes + t * P + s) : 0u;
    const unsigned kind = code & 3u;
    const bool doF = kind == 1u, doB = kind == 2u, act = kind != 0u;
    const double dF = getF ? __dadd_rn(nF, hF) : 0.0;
    const double dB = getB ? __dadd_rn(nB, hB) : 0.0;
    const double dep = doF ? dF : (doB ? dB : 0.0);
    const double rl = doF ? rlF : (doB || !ZBH ? rlB : rlW);
    double c = __dmul_rn(rl, base[code >> 2]);
    if (!unit) c = div_recip(c, sp, inv);
    const double st = fin > dep ? fin : dep;  // max (no NaNs on this path)
    const double nf = __dadd_rn(st, c);
    fin = act ? nf : fin;
    ssum = act ? __dadd_rn(ssum, c) : ssum;
    lastF = doF ? nf : lastF;
    lastB = doB ? nf : lastB;
  }
}

// MAXT = launch bound: 256 for the common case (more registers per lane),
// 1024 when one iteration needs D*pw > 256 lanes.
template <int ZBH, int DETECT, int MAXT>
__global__ void __launch_bounds__(MAXT) pass_kernel(const PassParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tid = threadIdx.x;
  const int P = p.sh.pp, D = p.sh.dp, M = p.sh.micro_batches, T = p.sh.tp;
  const int li = tid / p.lpi;
  const int within = tid - li * p.lpi;
  const int d = within >> p.log_pw;
  const int s = within & (p.pw - 1);
  const int64_t it = (int64_t)blockIdx.x * p.ipb + li;
  const bool iter_ok = li < p.ipb && it < p.tr.n_iter;
  const bool lane_on = iter_ok && s < P;
  const unsigned gmask = p.pw == 32 ? 0xffffffffu
                                    : (((1u << p.pw) - 1u) << (tid & 31 & ~(p.pw - 1)));

  double* it_ms = reinterpret_cast<double*>(smem_raw);
  unsigned* it_st = reinterpret_cast<unsigned*>(it_ms + p.ipb);
  const int it_bytes = ((p.ipb * 12 + 15) / 16) * 16;
  // per pipeline: base cost alpha*N + beta*Q_j of its micro-batches
  double* gbase = reinterpret_cast<double*>(smem_raw + it_bytes) +
                  (size_t)(tid >> p.log_pw) * p.mmax;

  if (tid < p.ipb) {
    it_ms[tid] = 0.0;
    it_st[tid] = 0u;
  }

  int seg = 0, m0 = 0, md = 0;
  if (iter_ok) {
    seg = p.tr.seg ? p.tr.seg[it] : 0;
    const int32_t* ms = p.sg.mb_start + (int64_t)seg * (D + 1);
    m0 = ms[d];
    md = ms[d + 1] - m0;
    if (md > p.mmax) md = -1;  // overflow: flagged below
  }
  // base cost alpha*N + beta*Q_j of the replica's micro-batches; the pw lanes
  // of the pipeline split the micro-batches between them
  if (iter_ok && md > 0) {
    const int64_t mb0 = it * M + m0;
    const double lin = __dmul_rn(p.m.alpha, (double)p.sh.token_budget);
    for (int jj = s; jj < md; jj += p.pw) {
      const int32_t a = __ldg(p.tr.mb_off + mb0 + jj);
      const int32_t b = __ldg(p.tr.mb_off + mb0 + jj + 1);
      long long q = 0;
      for (int32_t k = a; k < b; ++k) {
        const long long l = __ldg(p.tr.doc_len + k);
        q += l * l;
      }
      gbase[jj] = __dadd_rn(lin, __dmul_rn(p.m.beta, (double)q));
    }
  }

  double sp = 1.0, rlF = 0.0, rlB = 0.0, rlW = 0.0, hopf = 0.0, hopb = 0.0;
  int n_chain = 0, w = 0;
  bool stopped = false;
  if (lane_on && md > 0) {
    const int64_t gs = ((int64_t)seg * D + d) * P + s;
    sp = __ldg(p.sg.speed + gs);
    const double L = (double)__ldg(p.sg.layers + (int64_t)seg * P + s);
    rlF = __dmul_rn(p.m.ratio_f, L);
    rlB = __dmul_rn(ZBH ? p.m.ratio_b : __dadd_rn(p.m.ratio_b, p.m.ratio_w), L);
    rlW = __dmul_rn(p.m.ratio_w, L);
    if (s > 0) hopf = __ldg(p.sg.hop_fwd + gs - 1);
    if (s < P - 1) hopb = __ldg(p.sg.hop_bwd + gs);
    w = min(P - 1 - s, md);
    n_chain = (ZBH ? 3 : 2) * md;
    if (sp <= 0.0) {  // completeness violated (pipeline.py:408-415)
      stopped = true;
      n_chain = 0;
    }
  }
  __syncthreads();  // base costs visible; iteration slots initialised
  // a stopped stage invalidates the whole iteration (the reference raises
  // before building any DAG); its pipeline neighbours must not wait on it
  const unsigned bad = __ballot_sync(0xffffffffu, stopped) & gmask;
  if (bad) n_chain = 0;

  // ---------------------------------------------------------- wavefront
  double fin = 0.0, ssum = 0.0;
  bool over = false, hung = false;
  if (p.ltab) {  // level table: codes per (level, stage), peak in-flight per count
    const int mm = n_chain > 0 ? md : 0;
    const int mi = mm > 0 ? mm : 0;
    chain_walk_table<ZBH>(s, P, p.pw, mm, p.ltab + __ldg(p.ltab_off + mi),
                          __ldg(p.ltab_nlev + mi), gbase, rlF, rlB, rlW, sp, hopf, hopb, fin,
                          ssum);
    over = p.sh.capacity > 0 && mm > 0 && __ldg(p.ltab_peak + mi) > p.sh.capacity;
  } else {
    chain_walk<ZBH>(s, P, p.pw, md, w, n_chain, gbase, rlF, rlB, rlW, sp, hopf, hopb,
                    p.sh.capacity, p.mmax, fin, ssum, over, hung);
  }

  // ------------------------------------------------------ reductions
  double gmax = fin;
  for (int off = p.pw >> 1; off > 0; off >>= 1)
    gmax = fmax(gmax, __shfl_xor_sync(0xffffffffu, gmax, off));
  const unsigned ovf = __ballot_sync(0xffffffffu, over) & gmask;
  const unsigned hang = __ballot_sync(0xffffffffu, hung) & gmask;

  uint8_t flag = 0;
  float sev = 0.0f;
  if (DETECT && lane_on && md >= 0) {
    const float* dt = p.tr.device_time + ((it * D + d) * P + s) * (int64_t)T;
    float mx = 0.0f;
    if (p.vec4) {
      for (int t = 0; t < T; t += 4) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(dt + t));
        mx = fmaxf(mx, fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w)));
      }
    } else {
      for (int t = 0; t < T; ++t) mx = fmaxf(mx, __ldg(dt + t));
    }
    const double meas = (double)mx;
    if (!(ssum <= 0.0 || meas <= 0.0) && meas > __dmul_rn(p.thr, ssum)) {
      flag = 1;
      sev = (float)__ddiv_rn(ssum, meas);
    }
  }
  if (iter_ok) {
    unsigned bits = 0;
    if (s == 0) {
      if (md < 0 || hang) bits |= RH_IT_OVERFLOW;
      if (bad) bits |= RH_IT_STOPPED;
      if (ovf) bits |= RH_IT_CAPACITY;
      double msd = gmax;
      if (p.sh.has_allreduce && D > 1)
        msd = __dadd_rn(gmax, __ldg(p.sg.allreduce + (int64_t)seg * D + d));
      atomic_max_nonneg(it_ms + li, msd);
    }
    if (flag) bits |= RH_IT_STAGE_FLAG;
    if (DETECT && p.sg.link_off && p.sg.link_max) {  // one compare (segment maximum)
      if (within == 0 && __ldg(p.sg.link_max + seg) > p.thr) bits |= RH_IT_LINK_FLAG;
    } else if (DETECT && p.sg.link_off) {  // exercised-link ratios, split over the lanes
      const int32_t q0 = __ldg(p.sg.link_off + seg), q1 = __ldg(p.sg.link_off + seg + 1);
      for (int32_t q = q0 + within; q < q1; q += p.lpi)
        if (__ldg(p.sg.link_ratio + q) > p.thr) bits |= RH_IT_LINK_FLAG;
    }
    if (bits) atomicOr(it_st + li, bits);
  }
  __syncthreads();

  if (!iter_ok) return;
  const unsigned st_bits = it_st[li];
  const bool dead = (st_bits & (RH_IT_STOPPED | RH_IT_OVERFLOW)) != 0;
  if (lane_on) {
    const int64_t o = (it * D + d) * P + s;
    if (p.out.stage_cost) p.out.stage_cost[o] = dead ? 0.0 : ssum;
    if (DETECT) {
      if (p.out.stage_flag) p.out.stage_flag[o] = dead ? 0 : flag;
      if (p.out.severity) p.out.severity[o] = dead ? 0.0f : sev;
    }
  }
  if (within == 0) {
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
}

// ---------------------------------------------------------------------------
// Small-P variant (P <= 4, D <= 128): one THREAD per replica pipeline.
//
// Op order.  The thread executes its replica's chunks in DAG-level order
// (wavefront.cuh closed forms), inside a level by DESCENDING stage: for
// 1F1B with m >= P an unrolled warm-up and cool-down around a loop over the
// steady F/B level pairs (walk_steady); for smaller m (and ZBH up to 12)
// fully unrolled at compile time (walk_static); otherwise from a level table
// (sched_table).  With every stage's state in registers
// (P is a template parameter) the dependencies then read straight from the
// neighbours' registers:
//   * F(s,j) needs F(s-1,j) (one level earlier); stage s-1's next F may sit
//     on the same level as F(s,j), but in descending order it runs after;
//   * B(s,j) needs B(s+1,j) (one level earlier); B levels of neighbouring
//     stages have opposite parity, so no B of stage s+1 shares its level.
// That is exactly the level-synchronous wavefront, without per-level tests.
//
// Quadratic loads.  Thread 0 stages the CTA's micro-batch offsets and
// documents into shared memory with TMA bulk copies (cp.async.bulk completing
// on an mbarrier); l^2 is summed one thread per micro-batch; each thread then
// turns its replica's sums into base costs stored [j][thread] (conflict-free
// reads in the walk), aliasing the dead document buffer.  Thread 0 also
// prefetches into L2 the inputs of the CTA that takes over its slot in the
// next wave (cp.async.bulk.prefetch.L2).
//
// Division by a stage speed: exact hoisted-reciprocal form (div_fast) after a
// once-per-replica operand-range check (wavefront.cuh).
#ifndef RH_SMALL_THREADS
#define RH_SMALL_THREADS 128
#endif
constexpr int kSmallThreads = RH_SMALL_THREADS;
#ifndef RH_SMALL_MIN_BLOCKS
#define RH_SMALL_MIN_BLOCKS 5
#endif
constexpr int kSmallMinBlocks = RH_SMALL_MIN_BLOCKS;  // CTAs per SM the register budget targets
// narrow CTA width, used when dp <= kSmallNarrow (min blocks scale up to keep
// the per-thread register budget of the wide kernel)
constexpr int kSmallNarrow = kSmallThreads / 2;

#ifdef RH_DETECT_TRACE
// debug build only (tools/detect_trace.py): per CTA, warp 0's globaltimer at
// the phase boundaries of pass_small_kernel, and the SM it ran on
__device__ unsigned long long g_dtrace[4096 * 8];
__device__ __forceinline__ void dmark(int k) {
  if (threadIdx.x == 0 && blockIdx.x < 4096) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_dtrace[blockIdx.x * 8 + k] = t;
    if (k == 0) {
      unsigned sm;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
      g_dtrace[blockIdx.x * 8 + 7] = sm;
    }
  }
}
#define RH_DMARK(k) dmark(k)
#else
#define RH_DMARK(k) ((void)0)
#endif

template <int P, int ZBH, int DETECT, int TW>
__global__ void __launch_bounds__(TW, (ZBH ? 4 : kSmallMinBlocks) * (kSmallThreads / TW)) pass_small_kernel(const PassParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tid = threadIdx.x;
  const int D = p.sh.dp, M = p.sh.micro_batches, T = p.sh.tp;
  const int li = tid / D, d = tid - li * D;
  const int64_t it = (int64_t)blockIdx.x * p.ipb + li;
  const CtaStage cs = cta_layout(p, smem_raw);
  double* it_ms = cs.it_ms;
  unsigned* it_st = cs.it_st;
  unsigned long long* s_q = cs.s_q;
  double* base_t = cs.base_t;
  const int n_it = cs.n_it;
  const bool on = li < n_it;
  __shared__ uint64_t s_bar;
  RH_DMARK(0);
  if (tid < p.ipb) {
    it_ms[tid] = 0.0;
    it_st[tid] = 0u;
  }
  // ---- staging by TMA; the per-thread loads below run meanwhile
  const int seg = on && p.tr.seg ? __ldg(p.tr.seg + it) : 0;
  // the CTA that will run in this slot's next wave: its inputs are pulled into
  // L2 now, while this wave is latency-bound and HBM is mostly idle
  const int64_t nb = (int64_t)blockIdx.x + p.pf_stride;
  const bool pf = tid == 0 && p.pf_stride > 0 && nb < gridDim.x;
  int64_t pf_it = 0;
  int pf_nmb = 0;
  int32_t pf_lo = 0, pf_hi = 0;
  if (pf) {
    pf_it = nb * p.ipb;
    pf_nmb = (int)min((int64_t)p.ipb, p.tr.n_iter - pf_it) * M;
    pf_lo = __ldg(p.tr.mb_off + pf_it * M);
    pf_hi = __ldg(p.tr.mb_off + pf_it * M + pf_nmb);
  }
  // the replica's segment tables and device-time rows: loads issued before
  // the staging's barrier so their latency overlaps it (consumed after)
  int m0 = 0, md = 0;
  double rlF[P], rlB[P], rlW[P], sp[P], hf[P], hb[P], fin[P], ssum[P];
  int32_t Ls[P];
  float meas[P];
  float4 dtv[P];
  const bool pre4 = DETECT && on && p.vec4 && T == 4;
  if (on) {
    const int32_t* ms = p.sg.mb_start + (int64_t)seg * (D + 1);
    m0 = __ldg(ms + d);
    md = __ldg(ms + d + 1) - m0;
  }
#pragma unroll
  for (int s = 0; s < P; ++s) {
    const int64_t gs = ((int64_t)seg * D + d) * P + s;
    sp[s] = 1.0;
    hf[s] = hb[s] = 0.0;
    Ls[s] = 0;
    if (on) {
      sp[s] = __ldg(p.sg.speed + gs);
      Ls[s] = __ldg(p.sg.layers + (int64_t)seg * P + s);
      if (s > 0) hf[s] = __ldg(p.sg.hop_fwd + gs - 1);
      if (s < P - 1) hb[s] = __ldg(p.sg.hop_bwd + gs);
    }
    if (pre4)
      dtv[s] = __ldg(reinterpret_cast<const float4*>(p.tr.device_time +
                                                     ((it * D + d) * P + s) * (int64_t)4));
  }
  const bool use_lmax = DETECT && on && p.sg.link_off && p.sg.link_max;
  const double lmax = use_lmax ? __ldg(p.sg.link_max + seg) : 0.0;
  const StageState sg_state = stage_begin(p, smem_raw, cs, &s_bar);
#pragma unroll
  for (int s = 0; s < P; ++s) {
    rlF[s] = rlB[s] = rlW[s] = 0.0;
    if (on) {
      const double L = (double)Ls[s];
      rlF[s] = __dmul_rn(p.m.ratio_f, L);
      rlB[s] = __dmul_rn(ZBH ? p.m.ratio_b : __dadd_rn(p.m.ratio_b, p.m.ratio_w), L);
      rlW[s] = __dmul_rn(p.m.ratio_w, L);
    }
    fin[s] = ssum[s] = 0.0;
    // measured stage time: max over the TP group's device times
    meas[s] = 0.0f;
    if (pre4) {
      meas[s] = fmaxf(0.0f, fmaxf(fmaxf(dtv[s].x, dtv[s].y), fmaxf(dtv[s].z, dtv[s].w)));
    } else if (DETECT && on) {
      const float* dt = p.tr.device_time + ((it * D + d) * P + s) * (int64_t)T;
      float mx = 0.0f;
      if (p.vec4) {
        for (int q = 0; q < T; q += 4) {
          const float4 v = __ldg(reinterpret_cast<const float4*>(dt + q));
          mx = fmaxf(mx, fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w)));
        }
      } else {
        for (int q = 0; q < T; ++q) mx = fmaxf(mx, __ldg(dt + q));
      }
      meas[s] = mx;
    }
  }
  // the segment's exercised-link test: one compare against the segment's
  // maximum ratio, else a scan (4 independent load chains)
  bool link_bad = false;
  if (use_lmax) {
    link_bad = lmax > p.thr;  // any ratio > thr <=> max > thr
  } else if (DETECT && on && p.sg.link_off) {
    const int32_t q0 = __ldg(p.sg.link_off + seg), q1 = __ldg(p.sg.link_off + seg + 1);
    int32_t q = q0 + d;
    for (; q + 3 * D < q1; q += 4 * D) {
      const double a0 = __ldg(p.sg.link_ratio + q), a1 = __ldg(p.sg.link_ratio + q + D),
                   a2 = __ldg(p.sg.link_ratio + q + 2 * D), a3 = __ldg(p.sg.link_ratio + q + 3 * D);
      link_bad = link_bad || a0 > p.thr || a1 > p.thr || a2 > p.thr || a3 > p.thr;
    }
    for (; q < q1; q += D) link_bad = link_bad || __ldg(p.sg.link_ratio + q) > p.thr;
  }
  RH_DMARK(1);
  if (pf) {
    prefetch_l2(p.tr.mb_off + pf_it * M, 4 * (size_t)(pf_nmb + 1));
    prefetch_l2(p.tr.doc_len + pf_lo, 4 * (size_t)(pf_hi - pf_lo));
    if (DETECT)
      prefetch_l2(p.tr.device_time + pf_it * D * P * T, 4 * (size_t)(pf_nmb / M) * D * P * T);
  }
#ifdef RH_DETECT_TRACE
  mbar_wait(&s_bar, 0);  // (trace build: time the copies' wait apart from the sums)
  RH_DMARK(5);
#endif
  stage_finish(p, cs, sg_state, &s_bar);
  RH_DMARK(2);
  if (md > p.mmax) md = -1;
  // division by a unit speed is exact for any numerator (div_fast(a, 1, 1)
  // == a): only replicas with a slower stage need the operand-range check
  bool all_unit = true;
#pragma unroll
  for (int s = 0; s < P; ++s) all_unit = all_unit && sp[s] == 1.0;
  double b_lo = CUDART_INF, b_hi = 0.0;  // base-cost range (non-zero minimum)
  if (md > 0) {
    const double lin = __dmul_rn(p.m.alpha, (double)p.sh.token_budget);
    const unsigned long long* q = s_q + li * M + m0;
    // rotated start: neighbouring replicas' runs are md words apart, so
    // reading them in step would hit the same banks
    int j = d % md;
    for (int k = 0; k < md; ++k, j = j + 1 == md ? 0 : j + 1) {
      const double b = __dadd_rn(lin, __dmul_rn(p.m.beta, (double)(long long)q[j]));
      base_t[j * TW + tid] = b;
      if (!all_unit) {  // (finite, non-negative: plain compares)
        b_hi = b > b_hi ? b : b_hi;
        if (b > 0.0 && b < b_lo) b_lo = b;
      }
    }
  }
  const int m = md > 0 ? md : 0;
  bool stopped = false;
#pragma unroll
  for (int s = 0; s < P; ++s) {
    if (m == 0) {  // nothing runs: no speeds, no costs
      sp[s] = 1.0;
      rlF[s] = rlB[s] = rlW[s] = 0.0;
    }
    if (sp[s] <= 0.0) stopped = true;
  }
  // ---- the replica's chunks, level by level
  const int mm = stopped ? 0 : m;
  // activation capacity: the in-flight count along a chain is fixed by the
  // schedule, so its peak per micro-batch count is precomputed
  // (the peak is compared in the epilogue: its load's latency hides behind the walk)
  const int32_t peak = p.sh.capacity > 0 && mm > 0 ? __ldg(p.sched_peak + mm) : 0;
  const double* bt = base_t + tid;
  // exact division by a hoisted reciprocal when every numerator rl * b of the
  // walk and every divisor are in range (always, in practice); otherwise the
  // table walk divides with __ddiv_rn
  double inv[P];
  bool safe = true;
#pragma unroll
  for (int s = 0; s < P; ++s) inv[s] = sp[s] == 1.0 ? 1.0 : recip_of(sp[s]);
  if (!all_unit) {
    double r_lo = CUDART_INF, r_hi = 0.0;
#pragma unroll
    for (int s = 0; s < P; ++s) {
      safe = safe && inv[s] != 0.0;
      const double rs[3] = {rlF[s], rlB[s], ZBH ? rlW[s] : rlB[s]};
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        r_hi = rs[k] > r_hi ? rs[k] : r_hi;
        if (rs[k] > 0.0 && rs[k] < r_lo) r_lo = rs[k];
      }
    }
    safe = safe && div_range_ok(r_lo * b_lo, r_hi * b_hi);
  }
  // warp-uniform: the stages any replica of the warp runs slow (only those
  // divide; x / 1.0 == x exactly)
  unsigned slow = 0;
#pragma unroll
  for (int s = 0; s < P; ++s)
    if (mm > 0 && sp[s] != 1.0) slow |= 1u << s;
  slow = __reduce_or_sync(0xffffffffu, slow);
  WalkArgs<P, TW> wa{bt, rlF, rlB, rlW, sp, inv, hf, hb, fin, ssum, slow};
  RH_DMARK(3);
  if (mm > 0) {
    // the level table is read only by the table walks
    auto lv = [&](int k) { return p.sched + __ldg(p.sched_off + mm + k); };
    if (!safe)
      walk_table<P, ZBH, false>(wa, lv(0), lv(1));
    else if (mm >= P && p.steady)
      walk_steady<P, ZBH>(wa, mm);
    else if (mm > p.static_max || !walk_static_dispatch<P, ZBH>(wa, mm))
      walk_table<P, ZBH, true>(wa, lv(0), lv(1));
  }
  RH_DMARK(4);
  __syncthreads();  // iteration slots initialised before the reductions
  // ---- replica makespan, validation, iteration reductions
  uint8_t flag[P];
  float sev[P];
  unsigned bits = 0;
  if (on) {
    double g = 0.0;
#pragma unroll
    for (int s = 0; s < P; ++s) g = fmax(g, fin[s]);
    if (md < 0) bits |= RH_IT_OVERFLOW;
    if (stopped && m > 0) bits |= RH_IT_STOPPED;
    if (p.sh.capacity > 0 && mm > 0 && peak > p.sh.capacity) bits |= RH_IT_CAPACITY;
    if (p.sh.has_allreduce && D > 1)
      g = __dadd_rn(g, __ldg(p.sg.allreduce + (int64_t)seg * D + d));
    atomic_max_nonneg(it_ms + li, g);
#pragma unroll
    for (int s = 0; s < P; ++s) {
      flag[s] = 0;
      sev[s] = 0.0f;
      if (DETECT && md >= 0) {
        const double ms_d = (double)meas[s];
        if (!(ssum[s] <= 0.0 || ms_d <= 0.0) && ms_d > __dmul_rn(p.thr, ssum[s])) {
          flag[s] = 1;
          sev[s] = (float)__ddiv_rn(ssum[s], ms_d);
          bits |= RH_IT_STAGE_FLAG;
        }
      }
    }
    if (link_bad) bits |= RH_IT_LINK_FLAG;
    if (bits) atomicOr(it_st + li, bits);
  }
  __syncthreads();
  if (!on) return;
  const unsigned st_bits = it_st[li];
  const bool dead = (st_bits & (RH_IT_STOPPED | RH_IT_OVERFLOW)) != 0;
#pragma unroll
  for (int s = 0; s < P; ++s) {
    const int64_t o = (it * D + d) * P + s;
    if (p.out.stage_cost) p.out.stage_cost[o] = dead ? 0.0 : ssum[s];
    if (DETECT) {
      if (p.out.stage_flag) p.out.stage_flag[o] = dead ? 0 : flag[s];
      if (p.out.severity) p.out.severity[o] = dead ? 0.0f : sev[s];
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
  RH_DMARK(6);
}

// Level table for (P, schedule, mmax): for every micro-batch count
// mm = 0..mmax, kWords = ceil(P/4) 64-bit words per DAG level holding each
// stage's chunk at that level, 16 bits per stage (wavefront.cuh closed forms;
// a chain has at most one chunk per level).  Device layout [off: mmax+2
// int32 (word offsets) | peak: mmax+1 int32, padded to 8 B][level words].
// Built once per context.
static int sched_table(rh_ctx* ctx, int P, int zbh, int mmax,
                       const unsigned long long** lv_out, const int32_t** off_out,
                       const int32_t** peak_out) {
  const int W = (P + 3) / 4;
  // [off: mmax+2][peak: mmax+1] int32, padded to 8 B, then the level words
  const size_t off_words = ((size_t)(2 * mmax + 3) + 1) & ~size_t(1);
  auto view = [&](void* dev) {
    *off_out = static_cast<const int32_t*>(dev);
    *peak_out = *off_out + (mmax + 2);
    *lv_out = reinterpret_cast<const unsigned long long*>(*off_out + off_words);
  };
  std::lock_guard<std::mutex> lock(ctx->sched_mu);
  for (const auto& t : ctx->sched) {
    if (t.pp == P && t.zbh == zbh && t.mmax == mmax) {
      view(t.dev);
      return RH_OK;
    }
  }
  std::vector<int32_t> o(off_words, 0);
  std::vector<unsigned long long> v;
  for (int mm = 0; mm <= mmax; ++mm) {
    o[mm] = (int32_t)v.size();
    if (mm == 0) continue;
    const size_t base = v.size();
    auto put = [&](int level, int s, unsigned kind, int j) {
      const size_t at = base + (size_t)level * W + s / 4;
      if (at >= v.size()) v.resize(base + (size_t)(level + 1) * W, 0ull);
      v[at] |= (unsigned long long)(kind | ((unsigned)j << 2)) << (16 * (s % 4));
    };
    for (int s = 0; s < P; ++s) {
      const ChainLevels lv{s, P, mm, std::min(P - 1 - s, mm)};
      for (int j = 0; j < mm; ++j) {
        put(lv.F(j), s, kOpF, j);
        put(lv.B(j), s, kOpB, j);
        if (zbh) put(lv.W(j), s, kOpW, j);
      }
    }
    // peak in-flight forward chunks (F done, its B not yet) on any stage
    int peak = 0;
    for (int s = 0; s < P; ++s) {
      int live = 0;
      for (size_t t = base + s / 4; t < v.size(); t += W) {
        const unsigned kind = (unsigned)(v[t] >> (16 * (s % 4))) & 3u;
        if (kind == kOpF) peak = std::max(peak, ++live);
        if (kind == kOpB) --live;
      }
    }
    o[mmax + 2 + mm] = peak;
  }
  o[mmax + 1] = (int32_t)v.size();
  const size_t bytes = sizeof(int32_t) * off_words + sizeof(unsigned long long) * (v.size() + 1);
  void* dev = nullptr;
  RH_CUDA(cudaMalloc(&dev, bytes));
  RH_CUDA(cudaMemcpy(dev, o.data(), sizeof(int32_t) * off_words, cudaMemcpyHostToDevice));
  if (!v.empty())
    RH_CUDA(cudaMemcpy(static_cast<int32_t*>(dev) + off_words, v.data(),
                       sizeof(unsigned long long) * v.size(), cudaMemcpyHostToDevice));
  ctx->sched.push_back({P, zbh, mmax, dev});
  view(dev);
  return RH_OK;
}

// Level table of the lane kernel for (P, schedule, mmax): for every count
// mm = 0..mmax, uint16 codes [level][stage] (0 idle, else kind | j << 2), the
// level count and the peak in-flight forward chunks on any stage.  Device
// layout [off | nlev | peak: (mmax+1) int32 each, padded to 16 B][codes].
// Built once per context; returns ok = false when it would be too large.
static int lane_table(rh_ctx* ctx, int P, int zbh, int mmax, const uint16_t** codes,
                      const int32_t** off, const int32_t** nlev, const int32_t** peak,
                      bool* ok) {
  const size_t head = ((3 * (size_t)(mmax + 1) * 4) + 15) & ~size_t(15);
  auto view = [&](void* dev) {
    const int32_t* b = static_cast<const int32_t*>(dev);
    *off = b;
    *nlev = b + (mmax + 1);
    *peak = b + 2 * (mmax + 1);
    *codes = reinterpret_cast<const uint16_t*>(static_cast<const char*>(dev) + head);
  };
  std::lock_guard<std::mutex> lock(ctx->sched_mu);
  const int key_p = 1000 + P;  // distinct from sched_table's entries
  for (const auto& t : ctx->sched)
    if (t.pp == key_p && t.zbh == zbh && t.mmax == mmax) {
      view(t.dev);
      *ok = true;
      return RH_OK;
    }
  // size first: levels(mm) <= 2P + 3mm per count
  size_t words = 0;
  for (int mm = 1; mm <= mmax; ++mm) words += (size_t)(2 * P + 3 * mm + 2) * P;
  if (words * 2 > (64u << 20) || mmax >= (1 << 14)) {
    *ok = false;
    return RH_OK;
  }
  std::vector<int32_t> o(mmax + 1, 0), nl(mmax + 1, 0), pk(mmax + 1, 0);
  std::vector<uint16_t> v;
  for (int mm = 1; mm <= mmax; ++mm) {
    o[mm] = (int32_t)v.size();
    int t_end = 0;
    for (int s2 = 0; s2 < P; ++s2)
      t_end = std::max(t_end, ChainLevels{s2, P, mm, std::min(P - 1 - s2, mm)}.end(zbh));
    v.resize(v.size() + (size_t)t_end * P, 0);
    std::vector<int> live(P, 0);
    int peak_mm = 0;
    for (int s2 = 0; s2 < P; ++s2) {
      const ChainLevels lv{s2, P, mm, std::min(P - 1 - s2, mm)};
      for (int t = 0; t < t_end; ++t) {
        int j = 0;
        const int kind = lv.at(t, zbh, j);
        if (!kind) continue;
        v[o[mm] + (size_t)t * P + s2] = (uint16_t)(kind | (j << 2));
        if (kind == kOpF) peak_mm = std::max(peak_mm, ++live[s2]);
        if (kind == kOpB) --live[s2];
      }
    }
    nl[mm] = t_end;
    pk[mm] = peak_mm;
  }
  const size_t bytes = head + 2 * std::max<size_t>(1, v.size());
  std::vector<char> stage(bytes, 0);
  memcpy(stage.data(), o.data(), 4 * o.size());
  memcpy(stage.data() + 4 * (mmax + 1), nl.data(), 4 * nl.size());
  memcpy(stage.data() + 8 * (mmax + 1), pk.data(), 4 * pk.size());
  if (!v.empty()) memcpy(stage.data() + head, v.data(), 2 * v.size());
  void* dev = nullptr;
  RH_CUDA(cudaMalloc(&dev, bytes));
  RH_CUDA(cudaMemcpy(dev, stage.data(), bytes, cudaMemcpyHostToDevice));
  ctx->sched.push_back({key_p, zbh, mmax, dev});
  view(dev);
  *ok = true;
  return RH_OK;
}

template <int ZBH, int DETECT, int TW>
static void* small_kernel_w(int P) {
  switch (P) {
    case 1: return (void*)pass_small_kernel<1, ZBH, DETECT, TW>;
    case 2: return (void*)pass_small_kernel<2, ZBH, DETECT, TW>;
    case 3: return (void*)pass_small_kernel<3, ZBH, DETECT, TW>;
    default: return (void*)pass_small_kernel<4, ZBH, DETECT, TW>;
  }
}

template <int ZBH, int DETECT>
static void* small_kernel(int P, int tw) {
  return tw == kSmallNarrow ? small_kernel_w<ZBH, DETECT, kSmallNarrow>(P)
                            : small_kernel_w<ZBH, DETECT, kSmallThreads>(P);
}

static int next_pow2(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}

int launch_pass(rh_ctx* ctx, const rh_pipe_shape* sh, const rh_cost_model* m,
                const rh_segments* sg, const rh_trace* tr, double thr, int detect,
                const rh_pass_out* out, cudaStream_t stream) {
  if (!ctx || !sh || !m || !sg || !tr || !out || !out->makespan || !out->status) {
    set_error("pass: NULL argument");
    return RH_E_INVALID;
  }
  const int P = sh->pp, D = sh->dp, M = sh->micro_batches;
  if (P < 1 || D < 1 || M < 1 || sh->tp < 1 || sh->token_budget < 1 ||
      (sh->schedule != RH_SCHED_1F1B && sh->schedule != RH_SCHED_ZBH)) {
    set_error("pass: invalid shape pp=%d dp=%d tp=%d M=%d N=%d schedule=%d", P, D,
              sh->tp, M, sh->token_budget, sh->schedule);
    return RH_E_INVALID;
  }
  if (tr->n_iter == 0) return RH_OK;
  DeviceGuard guard(ctx);
  if (!tr->mb_off || !tr->doc_len || !sg->layers || !sg->mb_start || !sg->speed ||
      !sg->hop_fwd || !sg->hop_bwd || (sh->has_allreduce && D > 1 && !sg->allreduce) ||
      (detect && (!tr->device_time || !tr->observed))) {
    set_error("pass: missing trace/segment array");
    return RH_E_INVALID;
  }
  if (P > 32) {
    set_error("pass: pp=%d exceeds the 32-stage envelope", P);
    return RH_E_SHAPE;
  }
  PassParams p;
  p.sh = *sh;
  p.m = *m;
  p.sg = *sg;
  p.tr = *tr;
  p.out = *out;
  p.thr = thr;
  p.pw = next_pow2(P);
  p.log_pw = 0;
  while ((1 << p.log_pw) < p.pw) ++p.log_pw;
  p.lpi = D * p.pw;
  if (p.lpi > 1024) {
    set_error("pass: dp*next_pow2(pp) = %d exceeds 1024 lanes per CTA", p.lpi);
    return RH_E_SHAPE;
  }
  p.mmax = sh->max_mb_per_replica > 0 ? sh->max_mb_per_replica : M;
  p.vec4 = (sh->tp % 4 == 0) && ((reinterpret_cast<uintptr_t>(tr->device_time) & 15) == 0);
  if (P <= 4 && D <= kSmallThreads && p.mmax < 16384 && !getenv("RH_FORCE_LANE_KERNEL")) {
    // thread-per-replica kernel for short pipelines
    // narrow CTAs when a replica set fits: twice the CTAs per SM at the same
    // register budget, so more of them overlap their setup latency
    const int tw = (D <= kSmallNarrow && !getenv("RH_SMALL_WIDE")) ? kSmallNarrow : kSmallThreads;
    p.ipb = std::max(1, tw / D);
    const int threads = p.ipb * D;
    // j is stored in 14 bits of a level word
    const int it_bytes = ((p.ipb * 12 + 15) / 16) * 16;
    // [it_ms|it_st] [q: ipb*M int64] [off: 16 + 4*(ipb*M+1)] [docs -> base costs]
    const size_t off_base = (it_bytes + 8 * (size_t)p.ipb * M + 15) & ~size_t(15);
    const size_t head = off_base + 16 + 4 * (size_t)(p.ipb * M + 1);
    p.region_off = (int)((head + 15) & ~size_t(15));
    // the region holds the staged documents (+16 B for the TMA alignment
    // shift), later the base costs
    const size_t region =
        std::max<size_t>(128 * (size_t)tw + 16, (size_t)tw * p.mmax * 8);
    p.doc_stage = (int)((region - 16) / 4);
#ifdef RH_STATIC_MAX_MB
    p.static_max = RH_STATIC_MAX_MB;  // A/B builds: 0 = always the level-table walk
#else
    p.static_max = kStaticMaxMB;
#endif
    p.steady = getenv("RH_NO_STEADY_WALK") ? 0 : 1;
    p.q32 = getenv("RH_NO_Q32") ? 0 : 1;
    p.ltab = nullptr;
    const size_t smem = p.region_off + region;
    if (smem <= ctx->smem_optin && smem <= 56 * 1024) {
      const bool zbh = sh->schedule == RH_SCHED_ZBH;
      if (int e = sched_table(ctx, P, zbh, p.mmax, &p.sched, &p.sched_off, &p.sched_peak))
        return e;
      const int64_t blocks = (tr->n_iter + p.ipb - 1) / p.ipb;
      void* kern = zbh ? (detect ? small_kernel<1, 1>(P, tw) : small_kernel<1, 0>(P, tw))
                       : (detect ? small_kernel<0, 1>(P, tw) : small_kernel<0, 0>(P, tw));
      if (int e = ensure_smem(ctx, kern, smem)) return e;
      {
        int occ = 0;
        RH_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem));
        p.pf_stride = getenv("RH_NO_L2_PREFETCH") ? 0 : occ * ctx->num_sms;
      }
      void* args[] = {&p};
      RH_CUDA(cudaLaunchKernel(kern, dim3((unsigned)blocks), dim3(threads), args, smem, stream));
      RH_CHECK_LAUNCH(ctx);
      return RH_OK;
    }
  }
  if (P >= 5 && P <= 16 && D <= kWideThreads && p.mmax < 16384 && !getenv("RH_FORCE_LANE_KERNEL")) {
    const bool zbh = sh->schedule == RH_SCHED_ZBH;
    void* kern = wide_kernel_ptr(P, zbh ? 1 : 0, detect);
    if (kern) {
      constexpr int tw = kWideThreads;
      p.ipb = std::max(1, tw / D);
      auto al = [](size_t x) { return (x + 15) & ~size_t(15); };
      const size_t it_bytes = al((size_t)p.ipb * 12);
      p.w_base = (int)it_bytes;
      p.w_rl = (int)al(p.w_base + (size_t)tw * p.mmax * 8);
      // [rl: ipb][2][P] doubles, then the staged offsets and documents (the
      // hop / speed tables live in L1: wide_prep's transposed copy)
      p.w_union = (int)al(p.w_rl + (size_t)p.ipb * 2 * P * 8);
      const size_t off_bytes = al(16 + 4 * ((size_t)p.ipb * M + 1));
      p.w_docs = (int)(p.w_union + off_bytes);
      // documents: ~3.5 per micro-batch (a CTA with more reads them from L2)
      // (the region later holds the measured stage times [P][TW] floats)
      const size_t docs = al(std::max<size_t>(16 + 14 * (size_t)p.ipb * M,
                                              (size_t)P * tw * 4 > off_bytes ? (size_t)P * tw * 4 - off_bytes : 0));
      p.doc_stage = (int)((docs - 16) / 4);
      const size_t smem = p.w_docs + docs;
      if (smem <= ctx->smem_optin) {
        if (int e = sched_table(ctx, P, zbh, p.mmax, &p.sched, &p.sched_off, &p.sched_peak))
          return e;
        const int64_t blocks = (tr->n_iter + p.ipb - 1) / p.ipb;
        {
          void* tab = nullptr;
          if (int e = workspace(ctx, wide_tab_bytes(std::max(sg->n_seg, 1), P), &tab, 6, stream)) return e;
          if (int e = wide_prep(*sg, D, P, static_cast<double*>(tab), stream)) return e;
          p.wtab = static_cast<const double*>(tab);
        }
        if (int e = ensure_smem(ctx, kern, smem)) return e;
        int occ = 0;
        RH_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, tw, smem));
        p.pf_stride = getenv("RH_NO_L2_PREFETCH") ? 0 : occ * ctx->num_sms;
        void* args[] = {&p};
        RH_CUDA(cudaLaunchKernel(kern, dim3((unsigned)blocks), dim3(tw), args, smem, stream));
        RH_CHECK_LAUNCH(ctx);
        return RH_OK;
      }
    }
  }
  p.ipb = std::max(1, 256 / p.lpi);
  const int threads = ((p.ipb * p.lpi + 31) / 32) * 32;
  {
    bool ok = false;
    if (int e = lane_table(ctx, P, sh->schedule == RH_SCHED_ZBH, p.mmax, &p.ltab, &p.ltab_off,
                           &p.ltab_nlev, &p.ltab_peak, &ok))
      return e;
    if (!ok) p.ltab = nullptr;
  }
  const int it_bytes = ((p.ipb * 12 + 15) / 16) * 16;
  const size_t smem = it_bytes + (size_t)(threads / p.pw) * p.mmax * 8;
  if (smem > ctx->smem_optin) {
    set_error("pass: %zu bytes of shared memory needed (max_mb_per_replica=%d, pp=%d); "
              "limit %zu", smem, p.mmax, P, ctx->smem_optin);
    return RH_E_SHAPE;
  }
  const int64_t blocks = (tr->n_iter + p.ipb - 1) / p.ipb;
  if (blocks > 0x7fffffff) {
    set_error("pass: too many iterations");
    return RH_E_SHAPE;
  }
  void (*kern)(const PassParams);
  const bool big = threads > 256;
  if (sh->schedule == RH_SCHED_ZBH)
    kern = detect ? (big ? pass_kernel<1, 1, 1024> : pass_kernel<1, 1, 256>)
                  : (big ? pass_kernel<1, 0, 1024> : pass_kernel<1, 0, 256>);
  else
    kern = detect ? (big ? pass_kernel<0, 1, 1024> : pass_kernel<0, 1, 256>)
                  : (big ? pass_kernel<0, 0, 1024> : pass_kernel<0, 0, 256>);
  if (int e = ensure_smem(ctx, (const void*)kern, smem)) return e;
  kern<<<(unsigned)blocks, threads, smem, stream>>>(p);
  RH_CHECK_LAUNCH(ctx);
  return RH_OK;
}

// ------------------------------------------------------------------ host I/O

// Packed trace -> int32 CSR for iterations [i0, i0 + gridDim.x): one block per
// iteration scans its micro-batch document counts (absolute offsets from
// iter_doc) and widens its document lengths.
constexpr int kExpandThreads = 128;

__global__ void __launch_bounds__(kExpandThreads) expand_kernel(
    int64_t i0, int64_t n, int M, const int32_t* __restrict__ iter_doc,
    const uint8_t* __restrict__ mb_docs, const uint16_t* __restrict__ doc16,
    int32_t* __restrict__ off, int32_t* __restrict__ doc) {
  __shared__ int s_w[kExpandThreads / 32];
  const int64_t i = i0 + blockIdx.x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int carry = iter_doc[i];
  for (int j0 = 0; j0 < M; j0 += kExpandThreads) {
    const int j = j0 + threadIdx.x;
    const int c = j < M ? (int)mb_docs[i * M + j] : 0;
    int x = c;  // inclusive block scan
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_w[wid] = x;
    __syncthreads();
    int pre = 0, tot = 0;
    for (int w = 0; w < kExpandThreads / 32; ++w) {
      if (w < wid) pre += s_w[w];
      tot += s_w[w];
    }
    if (j < M) off[i * M + j] = carry + pre + x - c;
    carry += tot;
    __syncthreads();
  }
  // the end offset of this iteration's last micro-batch (the next iteration's
  // block writes the same value as its start)
  if (threadIdx.x == 0) off[(i + 1) * M] = iter_doc[i + 1];
  const int32_t d0 = iter_doc[i], d1 = iter_doc[i + 1];
  for (int32_t k = d0 + threadIdx.x; k < d1; k += kExpandThreads) doc[k] = doc16[k];
}

namespace {
struct Carver {
  char* base;
  size_t off = 0;
  template <class T>
  T* take(size_t n) {
    off = (off + 255) & ~size_t(255);
    T* r = reinterpret_cast<T*>(base + off);
    off += n * sizeof(T);
    return r;
  }
};
}  // namespace

// Chunks of the host pass: H2D of chunk k+1 overlaps the kernels of chunk k.
// The first and last chunks are small (RH_HOST_EDGE of the iterations each,
// default 12 %): compute starts early, and what remains after the last byte
// has crossed PCIe -- that chunk's kernels and read-back, the screen -- is
// short.  RH_HOST_CHUNKS forces a count of equal chunks (A/B runs).
static int host_chunks(int64_t n) {
  static const int force = getenv("RH_HOST_CHUNKS") ? atoi(getenv("RH_HOST_CHUNKS")) : 0;
  const int cap = force > 0 ? std::min(force, rh_ctx::kChunkEvents) : 3;
  return (int)std::max<int64_t>(1, std::min<int64_t>(cap, n / 1024));
}
// first iteration of chunk c (c = n_chunks: n)
static int64_t chunk_start(int64_t n, int c, int n_chunks) {
  static const int force = getenv("RH_HOST_CHUNKS") ? atoi(getenv("RH_HOST_CHUNKS")) : 0;
  static const double edge = getenv("RH_HOST_EDGE") ? atof(getenv("RH_HOST_EDGE")) : 0.12;
  if (c <= 0) return 0;
  if (c >= n_chunks) return n;
  if (force > 0 || n_chunks < 3) return n * c / n_chunks;
  // small first and last chunks, the middle ones equal
  const int64_t e = (int64_t)(edge * (double)n);
  if (c == n_chunks - 1) return n - e;
  return e + (n - 2 * e) * (c - 1) / (n_chunks - 2);
}

// The host pass's small inputs -- segment tables and the screen history --
// travel as ONE copy: they are gathered into a pinned staging buffer of the
// context on every call (a few KB of host memcpy) and the pass (or its
// captured graph) copies the staging buffer to the device.  Separate
// cudaMemcpyAsync calls cost ~5 us of DMA setup each.
struct SmallLayout {
  size_t layers, mbs, speed, hf, hb, ar, loff, lr, lmax, hist, bytes;
};
static SmallLayout small_layout(const rh_pipe_shape* sh, const rh_segments* sg) {
  const int64_t P = sh->pp, D = sh->dp, G = D * P, S = sg->n_seg;
  const int64_t n_links = sg->link_off ? sg->link_off[S] : 0;
  SmallLayout L;
  Carver c{nullptr};
  L.layers = (size_t)(uintptr_t)c.take<int32_t>(S * P);
  L.mbs = (size_t)(uintptr_t)c.take<int32_t>(S * (D + 1));
  L.speed = (size_t)(uintptr_t)c.take<double>(S * G);
  L.hf = (size_t)(uintptr_t)c.take<double>(S * G);
  L.hb = (size_t)(uintptr_t)c.take<double>(S * G);
  L.ar = (size_t)(uintptr_t)c.take<double>(S * D);
  L.loff = (size_t)(uintptr_t)c.take<int32_t>(S + 1);
  L.lr = (size_t)(uintptr_t)c.take<double>(n_links + 1);
  L.lmax = (size_t)(uintptr_t)c.take<double>(S + 1);
  L.hist = (size_t)(uintptr_t)c.take<double>(64);
  L.bytes = (c.off + 255) & ~size_t(255);
  return L;
}

static int fill_small_stage(rh_ctx* ctx, const rh_pipe_shape* sh, const rh_segments* sg,
                            const rh_screen_params* screen, int64_t series_len,
                            const double* hist) {
  const SmallLayout L = small_layout(sh, sg);
  if (L.bytes > ctx->host_stage_bytes) {
    // a captured graph may still copy from the old buffer: retire it
    if (ctx->host_stage) ctx->host_stage_retired.push_back(ctx->host_stage);
    ctx->host_stage = nullptr;
    ctx->host_stage_bytes = 0;
    RH_CUDA(cudaMallocHost(&ctx->host_stage, L.bytes + L.bytes / 2 + 4096));
    ctx->host_stage_bytes = L.bytes + L.bytes / 2 + 4096;
    std::lock_guard<std::mutex> lock(ctx->ws_mu);
    ++ctx->ws_epoch;
  }
  char* h = static_cast<char*>(ctx->host_stage);
  const int64_t P = sh->pp, D = sh->dp, G = D * P, S = sg->n_seg;
  const int64_t n_links = sg->link_off ? sg->link_off[S] : 0;
  auto put = [&](size_t off, const void* src, size_t bytes) {
    if (src && bytes) memcpy(h + off, src, bytes);
  };
  put(L.layers, sg->layers, 4 * S * P);
  put(L.mbs, sg->mb_start, 4 * S * (D + 1));
  put(L.speed, sg->speed, 8 * S * G);
  put(L.hf, sg->hop_fwd, 8 * S * G);
  put(L.hb, sg->hop_bwd, 8 * S * G);
  put(L.ar, sg->allreduce, 8 * S * D);
  put(L.loff, sg->link_off, 4 * (S + 1));
  put(L.lr, sg->link_ratio, 8 * n_links);
  put(L.lmax, sg->link_max, 8 * S);
  const int64_t hcount = screen ? std::min<int64_t>(series_len, screen->window) : 0;
  put(L.hist, hist, 8 * std::min<int64_t>(hcount, 64));
  return RH_OK;
}

// RH_HOST_TRACE=1 (debug aid, tools/e2e_timeline.py): timing events at the
// host pass's milestones, printed to stderr after every call.  The events are
// pooled and reused, so a captured graph re-records the ones it baked in.
struct HostTrace {
  const bool on = getenv("RH_HOST_TRACE") != nullptr;  // fixed at load: no per-call writes
  std::vector<cudaEvent_t> pool;
  std::vector<const char*> names;  // of the last enqueue (= the captured graph's)
  void begin() {
    if (on) names.clear();
  }
  void mark(const char* what, cudaStream_t st) {
    if (!on) return;
    if (names.size() == pool.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      pool.push_back(e);
    }
    cudaEventRecord(pool[names.size()], st);
    names.push_back(what);
  }
  void dump() {
    if (!on) return;
    for (size_t k = 0; k < names.size(); ++k) {
      float ms = 0.f;
      const cudaError_t e = cudaEventElapsedTime(&ms, pool[0], pool[k]);
      fprintf(stderr, "rh_host_trace %-16s %9.1f us %s\n", names[k], 1e3 * ms,
              e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
  }
};
static HostTrace g_htrace;

// Host-buffer Detector pass over an int32 trace (tr) or a packed one (pk):
// enqueues copies, kernels and read-backs on `stream` (+ the copy stream).
int enqueue_host_pass(rh_ctx* ctx, const rh_pipe_shape* sh, const rh_cost_model* m,
                const rh_segments* sg, const rh_trace* tr_in, const rh_trace_packed* pk,
                double thr, const rh_screen_params* screen, int64_t series_len,
                const double* hist, const uint8_t* reset, const rh_pass_out* out,
                uint8_t* outcome, int64_t* series_len_out, cudaStream_t stream) {
  if (!ctx || !sh || !sg || !out || (!tr_in && !pk) || (tr_in && !tr_in->mb_off) ||
      (pk && (!pk->iter_doc || !pk->mb_docs || !pk->doc_len)) ||
      (screen && series_len > 0 && !hist)) {
    set_error("detect_host: NULL argument (or series_len > 0 without hist)");
    return RH_E_INVALID;
  }
  const int P = sh->pp, D = sh->dp, T = sh->tp, M = sh->micro_batches;
  // the int32 view of the trace (its CSR arrays are rebuilt on the device
  // when the trace is packed)
  rh_trace tv{};
  if (pk) {
    tv.n_iter = pk->n_iter;
    tv.seg = pk->seg;
    tv.device_time = pk->device_time;
    tv.observed = pk->observed;
  } else {
    tv = *tr_in;
  }
  const rh_trace* tr = &tv;
  const int64_t n = tr->n_iter, G = (int64_t)D * P, S = sg->n_seg;
  if (n == 0) return RH_OK;
  const int64_t n_docs = pk ? pk->iter_doc[n] : tr->mb_off[n * M];
  const int64_t n_links = sg->link_off ? sg->link_off[S] : 0;
  size_t need = 0;
  {
    Carver c{nullptr};
    c.take<int32_t>(n);
    c.take<int32_t>(n * M + 1);
    c.take<int32_t>(n_docs);
    c.take<float>(n * G * T);
    c.take<double>(n);
    c.take<char>(small_layout(sh, sg).bytes);
    c.take<double>(n);
    c.take<uint8_t>(n);
    c.take<double>(n * G);
    c.take<uint8_t>(n * G);
    c.take<float>(n * G);
    c.take<uint8_t>(n);
    c.take<uint8_t>(n);
    c.take<int64_t>(1);
    if (pk) {
      c.take<int32_t>(n + 1);
      c.take<uint8_t>(n * M);
      c.take<uint16_t>(n_docs);
    }
    need = c.off + 256;
  }
  void* ws = nullptr;
  int rc = workspace(ctx, need, &ws, 0, stream);
  if (rc) return rc;
  Carver c{static_cast<char*>(ws)};
  // device buffers: every trace array lands at its own offsets, so the
  // absolute CSR offsets of mb_off stay valid for any chunk of iterations
  int32_t* d_seg = tr->seg ? c.take<int32_t>(n) : nullptr;
  int32_t* d_off = c.take<int32_t>(n * M + 1);
  int32_t* d_doc = c.take<int32_t>(n_docs);
  float* d_dt = c.take<float>(n * G * T);
  double* d_obs = c.take<double>(n);
  rh_segments dsg = *sg;
  const SmallLayout SL = small_layout(sh, sg);
  char* d_small = c.take<char>(SL.bytes);
  int32_t* d_layers = reinterpret_cast<int32_t*>(d_small + SL.layers);
  int32_t* d_mbs = reinterpret_cast<int32_t*>(d_small + SL.mbs);
  double* d_speed = reinterpret_cast<double*>(d_small + SL.speed);
  double* d_hf = reinterpret_cast<double*>(d_small + SL.hf);
  double* d_hb = reinterpret_cast<double*>(d_small + SL.hb);
  double* d_ar = reinterpret_cast<double*>(d_small + SL.ar);
  int32_t* d_loff = reinterpret_cast<int32_t*>(d_small + SL.loff);
  double* d_lr = reinterpret_cast<double*>(d_small + SL.lr);
  double* d_lmax = reinterpret_cast<double*>(d_small + SL.lmax);
  double* d_hist = reinterpret_cast<double*>(d_small + SL.hist);
  rh_pass_out dout = {};
  dout.makespan = c.take<double>(n);
  dout.status = c.take<uint8_t>(n);
  dout.stage_cost = out->stage_cost ? c.take<double>(n * G) : nullptr;
  dout.stage_flag = out->stage_flag ? c.take<uint8_t>(n * G) : nullptr;
  dout.severity = out->severity ? c.take<float>(n * G) : nullptr;
  uint8_t* d_reset = c.take<uint8_t>(n);
  uint8_t* d_outcome = c.take<uint8_t>(n);
  int64_t* d_len = c.take<int64_t>(1);
  int32_t* d_idoc = pk ? c.take<int32_t>(n + 1) : nullptr;
  uint8_t* d_cnt = pk ? c.take<uint8_t>(n * M) : nullptr;
  uint16_t* d_doc16 = pk ? c.take<uint16_t>(n_docs) : nullptr;
  auto cp = [&](void* dst, const void* src, size_t bytes, cudaMemcpyKind kind,
                cudaStream_t st) -> int {
    if (!src || !bytes) return RH_OK;
    RH_CUDA(cudaMemcpyAsync(dst, src, bytes, kind, st));
    return RH_OK;
  };
  const auto H2D = cudaMemcpyHostToDevice;
  const auto D2H = cudaMemcpyDeviceToHost;
  if (!ctx->copy_stream)
    RH_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
  if (!ctx->side_stream)
    RH_CUDA(cudaStreamCreateWithFlags(&ctx->side_stream, cudaStreamNonBlocking));
  if (!ctx->side_ev) RH_CUDA(cudaEventCreateWithFlags(&ctx->side_ev, cudaEventDisableTiming));
  const int n_chunks = host_chunks(n);
  for (int k = 0; k < n_chunks; ++k) {
    if (!ctx->chunk_ev[k])
      RH_CUDA(cudaEventCreateWithFlags(&ctx->chunk_ev[k], cudaEventDisableTiming));
    if (!ctx->done_ev[k])
      RH_CUDA(cudaEventCreateWithFlags(&ctx->done_ev[k], cudaEventDisableTiming));
  }
  if (!ctx->d2h_stream)
    RH_CUDA(cudaStreamCreateWithFlags(&ctx->d2h_stream, cudaStreamNonBlocking));
  if (!ctx->d2h_ev) RH_CUDA(cudaEventCreateWithFlags(&ctx->d2h_ev, cudaEventDisableTiming));
  // every copy runs on the copy stream, which must not overwrite buffers
  // earlier work on `stream` reads
  RH_CUDA(cudaEventRecord(ctx->chunk_ev[0], stream));
  RH_CUDA(cudaStreamWaitEvent(ctx->copy_stream, ctx->chunk_ev[0], 0));
  cudaStream_t cs = ctx->copy_stream, ds = ctx->d2h_stream;
  // segment tables + screen history: one copy of the staging buffer that
  // detect_host filled for this call (fill_small_stage)
  if ((rc = cp(d_small, ctx->host_stage, SL.bytes, H2D, cs))) return rc;
  dsg.layers = d_layers;
  dsg.mb_start = d_mbs;
  dsg.speed = d_speed;
  dsg.hop_fwd = d_hf;
  dsg.hop_bwd = d_hb;
  dsg.allreduce = sg->allreduce ? d_ar : nullptr;
  dsg.link_off = sg->link_off ? d_loff : nullptr;
  dsg.link_ratio = sg->link_off ? d_lr : nullptr;
  dsg.link_max = sg->link_off && sg->link_max ? d_lmax : nullptr;
  const int64_t h = screen ? std::min<int64_t>(series_len, screen->window) : 0;
  if (screen && h > 64) {
    set_error("detector_pass_host: window > 64");
    return RH_E_INVALID;
  }
  // the screen's inputs are tiny: copy them first and start its input-only
  // half (rh_screen_prepare) on the side stream while the trace streams in
  if (screen && reset && (rc = cp(d_reset, reset, n, H2D, cs))) return rc;
  if ((rc = cp(d_obs, tr->observed, 8 * n, H2D, cs))) return rc;
  if (screen) {
    RH_CUDA(cudaEventRecord(ctx->side_ev, cs));
    RH_CUDA(cudaStreamWaitEvent(ctx->side_stream, ctx->side_ev, 0));
    if ((rc = rh_screen_prepare(ctx, screen, series_len, d_hist, n, d_obs,
                                reset ? d_reset : nullptr, ctx->side_stream)))
      return rc;
  }
  // chunked pipeline: chunk k+1 crosses PCIe on the copy stream while chunk k
  // is processed on the caller's stream and chunk k-1's results come back on
  // the read-back stream
  g_htrace.mark("chunks start", cs);
  for (int k = 0; k < n_chunks; ++k) {
    const int64_t i0 = chunk_start(n, k, n_chunks), i1 = chunk_start(n, k + 1, n_chunks);
    const int64_t ni = i1 - i0;
    const int64_t o0 = pk ? pk->iter_doc[i0] : tr->mb_off[i0 * M];
    const int64_t o1 = pk ? pk->iter_doc[i1] : tr->mb_off[i1 * M];
    // this chunk's index arrays (segment ids, offsets or packed counts), then
    // its bulky device times and documents
    if ((rc = cp(d_seg ? d_seg + i0 : nullptr, tr->seg ? tr->seg + i0 : nullptr, 4 * ni, H2D, cs)))
      return rc;
    if (pk) {
      if ((rc = cp(d_idoc + i0, pk->iter_doc + i0, 4 * (ni + 1), H2D, cs)) ||
          (rc = cp(d_cnt + i0 * M, pk->mb_docs + i0 * M, ni * M, H2D, cs)))
        return rc;
    } else if ((rc = cp(d_off + i0 * M, tr->mb_off + i0 * M, 4 * (ni * M + 1), H2D, cs))) {
      return rc;
    }
    if ((rc = cp(d_dt + i0 * G * T, tr->device_time + i0 * G * T, 4 * ni * G * T, H2D, cs)))
      return rc;
    if (pk) {
      if ((rc = cp(d_doc16 + o0, pk->doc_len + o0, 2 * (o1 - o0), H2D, cs))) return rc;
    } else if ((rc = cp(d_doc + o0, tr->doc_len + o0, 4 * (o1 - o0), H2D, cs))) {
      return rc;
    }
    RH_CUDA(cudaEventRecord(ctx->chunk_ev[k], cs));
    g_htrace.mark("h2d chunk", cs);
    RH_CUDA(cudaStreamWaitEvent(stream, ctx->chunk_ev[k], 0));
    if (pk) {  // rebuild this chunk's int32 CSR
      expand_kernel<<<(unsigned)ni, kExpandThreads, 0, stream>>>(i0, n, M, d_idoc, d_cnt,
                                                                 d_doc16, d_off, d_doc);
      RH_CHECK_LAUNCH(ctx);
    }
    rh_trace ct = *tr;
    ct.n_iter = ni;
    ct.seg = d_seg ? d_seg + i0 : nullptr;
    ct.mb_off = d_off + i0 * M;
    ct.doc_len = d_doc;
    ct.device_time = d_dt + i0 * G * T;
    ct.observed = d_obs + i0;
    rh_pass_out co = dout;
    co.makespan += i0;
    co.status += i0;
    if (co.stage_cost) co.stage_cost += i0 * G;
    if (co.stage_flag) co.stage_flag += i0 * G;
    if (co.severity) co.severity += i0 * G;
    rc = launch_pass(ctx, sh, m, &dsg, &ct, thr, 1, &co, stream);
    if (rc) return rc;
    RH_CUDA(cudaEventRecord(ctx->done_ev[k], stream));
    g_htrace.mark("detect chunk", stream);
    RH_CUDA(cudaStreamWaitEvent(ds, ctx->done_ev[k], 0));
    if ((rc = cp(out->makespan + i0, co.makespan, 8 * ni, D2H, ds)) ||
        (rc = cp(out->status + i0, co.status, ni, D2H, ds)) ||
        (out->stage_cost && (rc = cp(out->stage_cost + i0 * G, co.stage_cost, 8 * ni * G, D2H, ds))) ||
        (out->stage_flag && (rc = cp(out->stage_flag + i0 * G, co.stage_flag, ni * G, D2H, ds))) ||
        (out->severity && (rc = cp(out->severity + i0 * G, co.severity, 4 * ni * G, D2H, ds))))
      return rc;
    g_htrace.mark("d2h chunk", ds);
  }
  if (screen) {
    rc = rh_screen(ctx, screen, series_len, d_hist, n, d_obs, dout.status,
                   reset ? d_reset : nullptr, d_outcome, d_len, stream);
    if (rc) return rc;
    if (outcome)
      RH_CUDA(cudaMemcpyAsync(outcome, d_outcome, n, D2H, stream));
    if (series_len_out)
      RH_CUDA(cudaMemcpyAsync(series_len_out, d_len, sizeof(int64_t), D2H, stream));
    g_htrace.mark("screen+out", stream);
  }
  // the caller's stream covers the read-backs
  RH_CUDA(cudaEventRecord(ctx->d2h_ev, ds));
  RH_CUDA(cudaStreamWaitEvent(stream, ctx->d2h_ev, 0));
  return RH_OK;
}

// Everything that shapes the enqueued work of a host pass: the graph key.
// Buffer CONTENTS are not part of it (memcpy nodes read them at replay), but
// the chunk boundaries' document offsets are, because they size the copies.
static std::vector<uint64_t> host_pass_key(const rh_pipe_shape* sh, const rh_cost_model* m,
                                           const rh_segments* sg, const rh_trace* tr,
                                           const rh_trace_packed* pk, double thr,
                                           const rh_screen_params* screen, int64_t series_len,
                                           const double* hist, const uint8_t* reset,
                                           const rh_pass_out* out, uint8_t* outcome,
                                           int64_t* series_len_out, cudaStream_t stream) {
  std::vector<uint64_t> k;
  auto raw = [&](const void* p, size_t n) {
    const size_t w = (n + 7) / 8;
    const size_t at = k.size();
    k.resize(at + w, 0);
    memcpy(k.data() + at, p, n);
  };
  raw(sh, sizeof(*sh));
  raw(m, sizeof(*m));
  raw(sg, sizeof(*sg));
  raw(out, sizeof(*out));
  if (tr) raw(tr, sizeof(*tr));
  if (pk) raw(pk, sizeof(*pk));
  if (screen) raw(screen, sizeof(*screen));
  raw(&thr, sizeof(thr));
  k.push_back((uint64_t)series_len);
  k.push_back((uint64_t)(uintptr_t)hist);
  k.push_back((uint64_t)(uintptr_t)reset);
  k.push_back((uint64_t)(uintptr_t)outcome);
  k.push_back((uint64_t)(uintptr_t)series_len_out);
  k.push_back((uint64_t)(uintptr_t)stream);
  k.push_back(pk ? 1 : 0);
  k.push_back(screen ? 1 : 0);
  const int64_t n = pk ? pk->n_iter : tr->n_iter;
  const int M = sh->micro_batches;
  k.push_back(sg->link_off ? (uint64_t)sg->link_off[sg->n_seg] : 0);
  const int n_chunks = host_chunks(n);
  for (int c = 0; c <= n_chunks; ++c) {
    const int64_t i = chunk_start(n, c, n_chunks);
    k.push_back((uint64_t)(pk ? pk->iter_doc[i] : tr->mb_off[i * M]));
  }
  return k;
}

// The host pass replays a CUDA graph: the first call with a given key runs
// directly (sizing every workspace and table), the second captures and
// instantiates it, later calls are one cudaGraphLaunch -- instead of ~60
// copy / event / launch API calls.  A failed capture just runs directly.
int detect_host(rh_ctx* ctx, const rh_pipe_shape* sh, const rh_cost_model* m,
                const rh_segments* sg, const rh_trace* tr, const rh_trace_packed* pk,
                double thr, const rh_screen_params* screen, int64_t series_len,
                const double* hist, const uint8_t* reset, const rh_pass_out* out,
                uint8_t* outcome, int64_t* series_len_out, cudaStream_t stream) {
  if (!ctx || !sh || !sg || !out || (!tr && !pk) || (tr && !tr->mb_off) ||
      (pk && (!pk->iter_doc || !pk->mb_docs || !pk->doc_len))) {
    set_error("detect_host: NULL argument");
    return RH_E_INVALID;
  }
  if (screen && series_len > 0 && !hist) {
    set_error("detect_host: series_len = %lld but hist is NULL", (long long)series_len);
    return RH_E_INVALID;
  }
  if ((pk ? pk->n_iter : tr->n_iter) == 0) return RH_OK;
  DeviceGuard guard(ctx);
  if (int rc = fill_small_stage(ctx, sh, sg, screen, series_len, hist)) return rc;
  auto& g = ctx->host_graph;
  std::vector<uint64_t> key = host_pass_key(sh, m, sg, tr, pk, thr, screen, series_len, hist,
                                            reset, out, outcome, series_len_out, stream);
  // the captured graph bakes in workspace pointers: any reallocation since
  // (by this or another call on the context) invalidates it
  {
    std::lock_guard<std::mutex> lock(ctx->ws_mu);
    key.push_back(ctx->ws_epoch);
  }
  const bool same = key == g.key;
  if (same && g.exec) {
    RH_CUDA(cudaGraphLaunch(g.exec, stream));
    RH_CUDA(cudaStreamSynchronize(stream));
    g_htrace.dump();
    return RH_OK;
  }
  if (!same) {
    if (g.exec) cudaGraphExecDestroy(g.exec);
    g.exec = nullptr;
    g.key = std::move(key);
    g.failed = false;
  } else if (!g.failed && !getenv("RH_NO_GRAPH")) {
    cudaGraph_t graph = nullptr;
    if (cudaStreamBeginCapture(stream, cudaStreamCaptureModeRelaxed) == cudaSuccess) {
      g_htrace.begin();
      g_htrace.mark("call", stream);
      const int rc = enqueue_host_pass(ctx, sh, m, sg, tr, pk, thr, screen, series_len, hist,
                                       reset, out, outcome, series_len_out, stream);
      g_htrace.mark("end", stream);
      const cudaError_t e = cudaStreamEndCapture(stream, &graph);
      if (rc == RH_OK && e == cudaSuccess && graph &&
          cudaGraphInstantiate(&g.exec, graph, 0) == cudaSuccess) {
        cudaGraphDestroy(graph);
        RH_CUDA(cudaGraphLaunch(g.exec, stream));
        RH_CUDA(cudaStreamSynchronize(stream));
        return RH_OK;
      }
      if (graph) cudaGraphDestroy(graph);
      g.exec = nullptr;
    }
    cudaGetLastError();  // clear a capture failure; run directly below
    g.failed = true;
  }
  g_htrace.begin();
  g_htrace.mark("call", stream);
  if (int rc = enqueue_host_pass(ctx, sh, m, sg, tr, pk, thr, screen, series_len, hist, reset,
                                 out, outcome, series_len_out, stream))
    return rc;
  g_htrace.mark("end", stream);
  RH_CUDA(cudaStreamSynchronize(stream));
  g_htrace.dump();
  return RH_OK;
}

}  // namespace rh

extern "C" {

int rh_pipeline_batch(rh_ctx* ctx, const rh_pipe_shape* shape, const rh_cost_model* model,
                      const rh_segments* segs, const rh_trace* trace,
                      const rh_pass_out* out, void* stream) {
  return rh::launch_pass(ctx, shape, model, segs, trace, 0.0, 0, out, rh::as_stream(stream));
}

int rh_detect_batch(rh_ctx* ctx, const rh_pipe_shape* shape, const rh_cost_model* model,
                    const rh_segments* segs, const rh_trace* trace, double threshold,
                    const rh_pass_out* out, void* stream) {
  return rh::launch_pass(ctx, shape, model, segs, trace, threshold, 1, out,
                         rh::as_stream(stream));
}

int rh_detector_pass_host(rh_ctx* ctx, const rh_pipe_shape* shape, const rh_cost_model* model,
                          const rh_segments* segs, const rh_trace* trace, double threshold,
                          const rh_screen_params* screen, int64_t series_len,
                          const double* hist, const uint8_t* reset, const rh_pass_out* out,
                          uint8_t* outcome, int64_t* series_len_out, void* stream) {
  return rh::detect_host(ctx, shape, model, segs, trace, nullptr, threshold, screen,
                         series_len, hist, reset, out, outcome, series_len_out,
                         rh::as_stream(stream));
}

int rh_detector_pass_host_packed(rh_ctx* ctx, const rh_pipe_shape* shape,
                                 const rh_cost_model* model, const rh_segments* segs,
                                 const rh_trace_packed* trace, double threshold,
                                 const rh_screen_params* screen, int64_t series_len,
                                 const double* hist, const uint8_t* reset,
                                 const rh_pass_out* out, uint8_t* outcome,
                                 int64_t* series_len_out, void* stream) {
  return rh::detect_host(ctx, shape, model, segs, nullptr, trace, threshold, screen,
                         series_len, hist, reset, out, outcome, series_len_out,
                         rh::as_stream(stream));
}

}  // extern "C"

#ifdef RH_DETECT_TRACE
extern "C" int rh_debug_detect_trace(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, rh::g_dtrace, sizeof(rh::g_dtrace)) == cudaSuccess ? 0 : 1;
}
#endif
