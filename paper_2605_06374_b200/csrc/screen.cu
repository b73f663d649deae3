// Change-point screen + DetectorState.observe state machine (rh_screen).
//
// Reference semantics (detector.py:94-108, 198-271): per iteration, append
// the observed time to the series, test it against the median/MAD of the
// previous `window` entries, run the workload-aware filter on candidates
// (or on every iteration while the window refills), escalate to validation,
// and POP the newest entry when the candidate is benign or the escalation is
// unconfirmed.  Because pops change later windows, the reference is a
// sequential scan.
//
// B200 formulation: the pop decision of iteration i is a pure function of
// the kept-set of earlier iterations.  We solve the triangular system
//     kept[i] = f_i(kept[0..i-1])
// by Jacobi iteration on the whole GPU: start from kept = all, recompute
// every decision in parallel from the previous round's kept-set, repeat
// until no decision changes.  The fixpoint is unique and equal to the
// sequential answer (induction on i); each round fixes at least one more
// leading decision, so it terminates, and in practice pops are sparse and it
// converges in 3 rounds.
//
// One persistent cooperative launch, one grid barrier per round.  A warp owns
// a fixed set of iterations and keeps their constants (observation, status,
// reset, the 32 preceding observations, last decision) in shared memory
// across rounds.  Per round and iteration, the warp
//   * scans the previous round's state bytes (bit 0 = popped, bit 1 =
//     changed in that round) backwards from i, 32 at a time with ballots,
//     until it has found the last `window` kept entries or reached the reset;
//     the kept lanes drop their observation straight into the warp's window
//     slots in shared memory, so no global prefix sum / compaction exists;
//   * skips the decision when no change lies inside that window span (or,
//     while the series is short, since the reset): it cannot differ;
//   * otherwise takes the median and MAD by lane-parallel rank selection over
//     the window in shared memory and applies the filter / validation bits.
// The kept-state is double-buffered, so every round reads one consistent
// kept-set (pure Jacobi) while writing the next.
#include <algorithm>

#include "common.cuh"

namespace rh {

constexpr int kScanThreads = 128;  // reset_scan_kernel block (= bres granularity)
#ifndef RH_SCREEN_THREADS
#define RH_SCREEN_THREADS 512
#endif
#ifndef RH_SCREEN_BPS
#define RH_SCREEN_BPS 2
#endif
constexpr int kScreenThreads = RH_SCREEN_THREADS;  // A/B builds may override both
constexpr int kScreenWarps = kScreenThreads / 32;
constexpr int kScreenBlocksPerSm = RH_SCREEN_BPS;
constexpr int kMaxWindow = 64;

struct ScreenArgs {
  int w;
  int fe;  // filter enabled
  double kappa;
  int64_t len0;
  int h;  // visible history entries
  const double* hist;
  int64_t n;
  const double* obs;
  const uint8_t* st;
  const uint8_t* reset;
  uint8_t* outcome;
  int64_t* len_out;
  // scratch
  int32_t* R;                      // [n] last reset index <= i, or -1
  int32_t* bres;                   // [n/128] last reset inside each scan block
  uint8_t* state;                  // [2][n] bit0 popped, bit1 changed in that round
  uint8_t* c0;                     // [n] round-0 verdicts (round0_kernel)
  // control words (workspace slot 3 of the stream): zero when a launch starts, and the
  // launch leaves them zero again (no memset per call; graph-replay safe)
  unsigned* cnt;             // [3] barrier words per round (rotating): arrivals + changed blocks << 16
  unsigned long long* kcnt;  // [3] kept entries since the last reset, per round
  unsigned* bar;             // [2] unused (reserved)
  unsigned* ticket;          // [1] blocks finished
  void* prep_buf;            // host side: the slot-2 buffer launch_prepare filled
};

// Grid barrier of Jacobi round `round`, carrying the round's "anything
// changed" bit: thread 0 of every block adds 1 (+ 1 << 16 when the block
// changed a decision) to the round's word with release semantics and polls it
// with acquire loads until every block has arrived.  One fire-and-forget
// atomic and one polling round trip per block; the poll's value is the
// round's verdict, so no separate counter read follows.  Words rotate over
// three rounds: the word of round r + 1 was last polled before barrier r - 1
// and is zeroed by block 0 before it arrives at barrier r.
__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ bool grid_barrier_any(unsigned* words, int round, unsigned nblocks,
                                                 bool changed, unsigned* s_any) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned* w = words + round % 3;
    red_release_add(w, 1u + (changed ? 0x10000u : 0u));
    unsigned v;
    do {
      v = ld_acquire(w);
    } while ((v & 0xffffu) < nblocks);
    *s_any = v >> 16;
  }
  __syncthreads();
  return *s_any != 0;
}

// statistics.median of the w values in a[] (shared memory, warp-visible):
// lane-parallel rank selection.  Slot q's rank is the number of entries that
// sort before it (ties broken by slot index, i.e. a stable sort), so exactly
// one slot holds each rank; the slots of rank w/2-1 and w/2 are the middle.
// Every lane reads every entry as a shared-memory broadcast, so the w loads
// are independent and pipeline, unlike a sorting network's dependent stages.
__device__ __forceinline__ double warp_median(const double* a, int w, double* sel) {
  const int lane = threadIdx.x & 31;
  for (int q = lane; q < w; q += 32) {
    const double v = a[q];
    int rank = 0;
#pragma unroll 4
    for (int p = 0; p < w; ++p) {
      const double u = a[p];
      rank += (u < v) | ((u == v) & (p < q));
    }
    if (rank == (w >> 1)) sel[1] = v;
    if (rank == (w >> 1) - 1) sel[0] = v;
  }
  __syncwarp();
  const double hi = sel[1];
  return (w & 1) ? hi : __ddiv_rn(__dadd_rn(sel[0], hi), 2.0);
}

// last reset index <= i: block-local inclusive max-scan, one element per
// thread; block summaries land in bres and are folded in by screen_kernel
__global__ void __launch_bounds__(kScanThreads) reset_scan_kernel(ScreenArgs a) {
  __shared__ int sm[32];
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int x = (i < a.n && a.reset[i]) ? (int)i : -1;
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x = max(x, y);
  }
  if (lane == 31) sm[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int t = lane < (int)(blockDim.x >> 5) ? sm[lane] : -1;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t = max(t, y);
    }
    sm[lane] = t;
  }
  __syncthreads();
  if (wid) x = max(x, sm[wid - 1]);
  if (i < a.n) a.R[i] = x;
  if (threadIdx.x == 0) a.bres[blockIdx.x] = sm[(blockDim.x >> 5) - 1];
}

// Per-warp shared scratch: the window, its deviations, the median selection.
struct WarpScratch {
  double win[kMaxWindow];
  double dev[kMaxWindow];
  double sel[2];
};

// Window part of one Jacobi step for iteration i, executed by a whole warp
// (uniform result).  x is the iteration's observation; ob (optional) holds
// obs[i-32+lane] so the common single-chunk window needs no global gather.
// skip = no change of the previous round lies where it could reach i.
struct WindowTest {
  bool skip, cand, refill_len;  // refill_len: series still at most `window` long
};

// Round-0 pop decision of iteration j from its prepared verdict bits and
// status (the filter / validation logic of outcome_of, without the outcome).
__device__ __forceinline__ unsigned pop0_of(unsigned c0, unsigned stb, int fe) {
  const bool cand = c0 & 1u, refill = !cand && fe && (c0 & 2u);
  if (!(cand || refill)) return 0u;
  if (fe && !(stb & RH_IT_ESCALATE)) return cand ? 1u : 0u;
  return (stb & (RH_IT_STAGE_FLAG | RH_IT_LINK_FLAG)) ? 0u : 1u;
}

// state byte of iteration j in the previous round: bit 0 popped, bit 1
// changed.  from_c0: that round is round 0, rebuilt on the fly from the
// prepared verdicts (changed == popped, since round 0 starts from kept = all).
__device__ __forceinline__ unsigned prev_state(const ScreenArgs& a, const uint8_t* cur,
                                               bool first_round, bool from_c0, int64_t j) {
  if (first_round) return 0u;
  if (from_c0) return pop0_of(__ldg(a.c0 + j), __ldg(a.st + j), a.fe) * 3u;
  return (unsigned)__ldcg(cur + j);
}

__device__ __forceinline__ WindowTest window_test(const ScreenArgs& a, int64_t i, int r, double x,
                                                  const double* ob, const uint8_t* cur,
                                                  bool first_round, WarpScratch& ws,
                                                  bool from_c0 = false, int sv0 = -1) {
  const int lane = threadIdx.x & 31;
  const int w = a.w;
  const int64_t first = r >= 0 ? r : 0;
  // backward scan for the last w kept entries in [first, i)
  int found = 0;
  bool any_chg = first_round;
  for (int64_t hi = i; hi > first && found < w; hi -= 32) {
    const int64_t j = hi - 32 + lane;
    const bool in = j >= first;
    // sv0: this lane's state byte of the first chunk, preloaded by the caller
    const unsigned sv = !in ? 1u
                            : (hi == i && sv0 >= 0 ? (unsigned)sv0
                                                   : prev_state(a, cur, first_round, from_c0, j));
    const bool kept = !(sv & 1u);
    const unsigned km = __ballot_sync(0xffffffffu, kept);
    const unsigned cm = __ballot_sync(0xffffffffu, (sv & 2u) != 0u);
    // rank of this lane's kept entry counted from i downwards (0 = newest)
    const int rank = found + __popc(km >> lane) - 1;
    if (kept && rank < w) ws.win[w - 1 - rank] = (ob && hi == i) ? ob[lane] : a.obs[j];
    const int cnt = __popc(km);
    if (found + cnt >= w) {
      // the window starts at the kept lane of rank w-1: changes below it
      // cannot reach iteration i
      const int pos = __ffs(__ballot_sync(0xffffffffu, kept && rank == w - 1)) - 1;
      any_chg |= (cm >> pos) != 0u;
      found = w;
    } else {
      found += cnt;
      any_chg |= cm != 0u;
    }
  }
  WindowTest t{false, false, false};
  if (!any_chg) {
    __syncwarp();
    t.skip = true;
    return t;
  }
  // kept entries since the reset: exact below w, which is all the length
  // thresholds need
  const int64_t len = (r >= 0 ? found : a.len0 + found) + 1;
  if (len >= w + 1) {
    const int need = w - found;  // > 0 only without a reset: history entries
    for (int q = lane; q < need; q += 32) ws.win[q] = a.hist[a.h - need + q];
    __syncwarp();
    const double med = warp_median(ws.win, w, ws.sel);
    for (int q = lane; q < w; q += 32) ws.dev[q] = fabs(__dsub_rn(ws.win[q], med));
    __syncwarp();
    const double mad = warp_median(ws.dev, w, ws.sel);
    t.cand = fabs(__dsub_rn(x, med)) > __dmul_rn(a.kappa, mad);
  }
  t.refill_len = len <= w;
  __syncwarp();  // the scratch is reused by the warp's next iteration
  return t;
}

// Filter / validation part (detector.py:223-271): the pop decision and the
// outcome bits from the screen verdict and the iteration's status bits.
__device__ __forceinline__ unsigned outcome_of(bool cand, bool refill_len, unsigned stb, int fe,
                                               uint8_t& oc_out) {
  const bool refill = !cand && fe && refill_len;
  bool pop = false;
  uint8_t oc = 0;
  if (cand || refill) {
    oc = cand ? RH_SC_CANDIDATE : 0;
    bool done = false;
    if (fe) {
      oc |= RH_SC_FILTERED;
      if (!(stb & RH_IT_ESCALATE)) {
        if (cand) {
          pop = true;
          oc |= RH_SC_POPPED;
        }
        done = true;
      }
    }
    if (!done) {
      oc |= RH_SC_ESCALATED;
      if (!(stb & (RH_IT_STAGE_FLAG | RH_IT_LINK_FLAG))) {
        pop = true;
        oc |= RH_SC_POPPED;
      } else {
        oc |= RH_SC_CONFIRMED;
      }
    }
  }
  oc_out = oc;
  return pop ? 1u : 0u;
}

// One DetectorState.observe (detector.py:198-271) in one launch: validate
// the (replica, stage) times and the exercised-link ratios when asked
// (detector.py:127-158: flag = measured > thr * expected, severity =
// expected / measured; links: ratio > thr, severity 1 / ratio), fold the
// flags into the iteration's status, then warp 0 screens the new observation
// against the carried series (the window test of window_test with no
// earlier iteration in the batch: the window is the history itself).
constexpr int kObserveThreads = 256;
__global__ void __launch_bounds__(kObserveThreads) observe_kernel(
    int w, int fe, double kappa, int64_t series_len, const double* __restrict__ hist, int h,
    double x, unsigned escalate, int do_validate, int n_stage, const double* __restrict__ meas,
    const double* __restrict__ expd, int n_link, const double* __restrict__ lr, double thr,
    uint8_t* __restrict__ s_flag, double* __restrict__ s_sev, uint8_t* __restrict__ l_flag,
    double* __restrict__ l_sev, uint8_t* __restrict__ outcome, int64_t* __restrict__ len_out) {
  __shared__ WarpScratch ws;
  int stage_hit = 0, link_hit = 0;
  if (do_validate) {
    for (int i = threadIdx.x; i < n_stage; i += blockDim.x) {
      const double m = meas[i], e = expd[i];
      const bool f = !(e <= 0.0 || m <= 0.0) && m > __dmul_rn(thr, e);
      s_flag[i] = f ? 1 : 0;
      s_sev[i] = f ? __ddiv_rn(e, m) : 0.0;
      stage_hit |= f;
    }
    for (int i = threadIdx.x; i < n_link; i += blockDim.x) {
      const double r = lr[i];
      const bool f = r > thr;
      l_flag[i] = f ? 1 : 0;
      l_sev[i] = f ? __ddiv_rn(1.0, r) : 0.0;
      link_hit |= f;
    }
  }
  stage_hit = __syncthreads_or(stage_hit);
  link_hit = __syncthreads_or(link_hit);
  if (threadIdx.x >= 32) return;
  const unsigned stb = (escalate ? RH_IT_ESCALATE : 0u) | (stage_hit ? RH_IT_STAGE_FLAG : 0u) |
                       (link_hit ? RH_IT_LINK_FLAG : 0u);
  const int lane = threadIdx.x;
  const int64_t len = series_len + 1;  // the series after appending x
  bool cand = false;
  if (len >= w + 1) {  // detect_change_point: the previous w values
    for (int q = lane; q < w; q += 32) ws.win[q] = hist[h - w + q];
    __syncwarp();
    const double med = warp_median(ws.win, w, ws.sel);
    for (int q = lane; q < w; q += 32) ws.dev[q] = fabs(__dsub_rn(ws.win[q], med));
    __syncwarp();
    const double mad = warp_median(ws.dev, w, ws.sel);
    cand = fabs(__dsub_rn(x, med)) > __dmul_rn(kappa, mad);
  }
  uint8_t oc;
  const unsigned pop = outcome_of(cand, len <= w, stb, fe, oc);
  if (lane == 0) {
    *outcome = oc;
    *len_out = len - (int64_t)pop;
  }
}

// Round 0 (kept = all) of every iteration, one warp each over the whole GPU:
// folds the reset index and runs the window test, which in this round only
// depends on the inputs.  c0 = cand | refill_len << 1.
constexpr int kRound0Threads = 256;

__global__ void __launch_bounds__(kRound0Threads) round0_kernel(ScreenArgs a) {
  __shared__ WarpScratch s_ws[kRound0Threads / 32];
  const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (i >= a.n) return;
  const int lane = threadIdx.x & 31;
  const double x = a.obs[i];
  int r = a.R[i];
  if (r < 0 && a.reset) {  // fold in the resets of earlier scan blocks
    const int nb = (int)(i / kScanThreads);
    for (int b = lane; b < nb; b += 32) r = max(r, a.bres[b]);
    for (int o = 16; o > 0; o >>= 1) r = max(r, __shfl_xor_sync(0xffffffffu, r, o));
  }
  const WindowTest t = window_test(a, i, r, x, nullptr, nullptr, true, s_ws[threadIdx.x >> 5]);
  if (lane == 0) {
    a.R[i] = r;
    a.c0[i] = (uint8_t)((t.cand ? 1 : 0) | (t.refill_len ? 2 : 0));
  }
}

// What a warp keeps across rounds for each of its first kCache iterations.
constexpr int kCache = 4;
struct IterCache {
  double x;
  int32_t r;
  uint8_t st;
  uint8_t pop;
};

struct ScreenSmem {
  WarpScratch ws[kScreenWarps];
  double ob[kScreenWarps][kCache][32];
  IterCache it[kScreenWarps][kCache];
  unsigned long long kcnt;
  unsigned cnt;
};

#ifdef RH_SCREEN_TRACE
// debug build only (tools/screen_trace.py): per round, block 0's timestamps
// around the barrier and the slowest block's compute time
__device__ unsigned long long g_trace_t[3 * 32];
__device__ unsigned long long g_trace_slow[32];
__device__ unsigned g_trace_chg[32];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
extern "C" int rh_debug_screen_trace(unsigned long long* t, unsigned long long* slow,
                                     unsigned* chg) {
  cudaMemcpyFromSymbol(t, g_trace_t, sizeof(g_trace_t));
  cudaMemcpyFromSymbol(slow, g_trace_slow, sizeof(g_trace_slow));
  cudaMemcpyFromSymbol(chg, g_trace_chg, sizeof(g_trace_chg));
  return 0;
}
#endif

__global__ void __launch_bounds__(kScreenThreads) screen_kernel(const ScreenArgs a) {
  // dynamic shared memory (ScreenSmem): per-warp scratch, the 32 preceding
  // observations and the constants of each cached iteration
  extern __shared__ __align__(16) unsigned char screen_smem[];
  ScreenSmem& sm = *reinterpret_cast<ScreenSmem*>(screen_smem);
  WarpScratch* s_ws = sm.ws;
  auto& s_ob = sm.ob;
  auto& s_it = sm.it;
  unsigned& s_cnt = sm.cnt;
  __shared__ unsigned s_any;
  unsigned long long& s_kcnt = sm.kcnt;
  // the series length at the end counts kept entries from the last reset on
  const int32_t r_last = __ldg(a.R + (a.n - 1));
  const int64_t first_last = r_last >= 0 ? r_last : 0;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t gw = (int64_t)blockIdx.x * kScreenWarps + wid;
  const int64_t n_warps = (int64_t)gridDim.x * kScreenWarps;

  int round = 0;
  for (;; ++round) {
    const uint8_t* cur = a.state + (size_t)(round & 1) * a.n;
    uint8_t* nxt = a.state + (size_t)((round + 1) & 1) * a.n;
    if (threadIdx.x == 0) {
      s_cnt = 0;
      s_kcnt = 0;
    }
    __syncthreads();
#ifdef RH_SCREEN_TRACE
    const unsigned long long t_start = gtimer();
#endif
    unsigned changes = 0, kept = 0;
    auto process = [&](int64_t i, int k, bool cached, int sv0) {
      int r;
      double x;
      unsigned stb, old;
      unsigned pop;
      if (round == 0) {
        // First cooperative round = Jacobi round 1, reading round 0's state on
        // the fly from the prepared verdicts (no barrier for round 0 itself).
        // Cache what later rounds need.
        x = a.obs[i];
        stb = a.st[i];
        r = a.R[i];
        const unsigned c0 = a.c0[i];
        if (cached) {
          const int64_t j = i - 32 + lane;
          s_ob[wid][k][lane] = j >= 0 ? a.obs[j] : 0.0;
        }
        __syncwarp();
        uint8_t oc0;
        old = outcome_of(c0 & 1u, (c0 & 2u) != 0u, stb, a.fe, oc0);
        const WindowTest t = window_test(a, i, r, x, cached ? s_ob[wid][k] : nullptr, cur, false,
                                         s_ws[wid], true, sv0);
        uint8_t oc = oc0;
        pop = old;
        if (!t.skip) pop = outcome_of(t.cand, t.refill_len, stb, a.fe, oc);
        if (lane == 0) {
          a.outcome[i] = oc;
          if (cached) s_it[wid][k] = IterCache{x, r, (uint8_t)stb, 0};
        }
      } else {
        if (cached) {
          const IterCache c = s_it[wid][k];
          x = c.x;
          r = c.r;
          stb = c.st;
          old = c.pop;
        } else {
          x = a.obs[i];
          stb = a.st[i];
          r = __ldcg(a.R + i);
          old = __ldcg(cur + i) & 1u;
        }
        const WindowTest t = window_test(a, i, r, x, cached ? s_ob[wid][k] : nullptr, cur, false,
                                         s_ws[wid], false, sv0);
        if (t.skip) {
          pop = old;
        } else {
          uint8_t oc;
          pop = outcome_of(t.cand, t.refill_len, stb, a.fe, oc);
          if (lane == 0) a.outcome[i] = oc;
        }
      }
      const unsigned changed = pop != old;
      if (lane == 0) {
        nxt[i] = (uint8_t)(pop | (changed << 1));
        if (cached) s_it[wid][k].pop = (uint8_t)pop;
      }
      changes += changed;
      kept += (!pop && i >= first_last) ? 1u : 0u;
    };
    // the first window chunk of every cached iteration is loaded up front, so
    // those round trips overlap instead of queueing behind each other
    int pre[kCache];
#pragma unroll
    for (int k = 0; k < kCache; ++k) {
      const int64_t i = gw + k * n_warps, j = i - 32 + lane;
      pre[k] = -1;
      if (i < a.n && j >= 0)
        pre[k] = (int)(round == 0 ? pop0_of(__ldg(a.c0 + j), __ldg(a.st + j), a.fe) * 3u
                                  : (unsigned)__ldcg(cur + j));
    }
#pragma unroll
    for (int k = 0; k < kCache; ++k) {
      const int64_t i = gw + k * n_warps;
      if (i < a.n) process(i, k, true, pre[k]);
    }
    for (int64_t i = gw + kCache * n_warps; i < a.n; i += n_warps) process(i, kCache, false, -1);
    if (lane == 0 && changes) atomicAdd(&s_cnt, changes);
    if (lane == 0 && kept) atomicAdd(&s_kcnt, (unsigned long long)kept);
    // the next round's counters were last read before this round began
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      a.cnt[(round + 1) % 3] = 0;
      a.kcnt[(round + 1) % 3] = 0;
    }
    __syncthreads();
    if (threadIdx.x == 0 && s_kcnt) atomicAdd(a.kcnt + round % 3, s_kcnt);
#ifdef RH_SCREEN_TRACE
    const unsigned long long t_arrive = gtimer();
    if (threadIdx.x == 0 && round < 32) atomicMax(&g_trace_slow[round], t_arrive - t_start);
#endif
    const bool any = grid_barrier_any(a.cnt, round, gridDim.x, s_cnt != 0, &s_any);
#ifdef RH_SCREEN_TRACE
    if (blockIdx.x == 0 && threadIdx.x == 0 && round < 32) {
      g_trace_t[3 * round] = t_start;
      g_trace_t[3 * round + 1] = t_arrive;
      g_trace_t[3 * round + 2] = gtimer();
      g_trace_chg[round] = __ldcg(a.cnt + round % 3) >> 16;
    }
#endif
    if (!any) break;  // fixpoint: nothing changed
  }
  // final series length: kept entries since the last reset (+ history), as
  // counted in the round that changed nothing
  if (threadIdx.x == 0) {
    const unsigned long long total = __ldcg(a.kcnt + round % 3);
    if (blockIdx.x == 0 && a.len_out)
      *a.len_out = r_last >= 0 ? (int64_t)total : a.len0 + (int64_t)total;
    // the last block out leaves the control words zero for the next launch
    __threadfence();
    if (atomicAdd(a.ticket, 1u) == gridDim.x - 1) {
      for (int q = 0; q < 3; ++q) {
        a.cnt[q] = 0;
        a.kcnt[q] = 0;
      }
      *a.ticket = 0;
    }
  }
}

}  // namespace rh

using namespace rh;

namespace {

// Workspace carve shared by rh_screen_prepare and rh_screen.
struct PrepLayout {
  size_t oR, oRes, oC0, bytes;
  explicit PrepLayout(int64_t n) {
    size_t b = 0;
    auto take = [&](size_t n_bytes) {
      const size_t o = b;
      b = (b + n_bytes + 255) & ~size_t(255);
      return o;
    };
    oR = take(sizeof(int32_t) * n);
    oRes = take(sizeof(int32_t) * ((n + kScanThreads - 1) / kScanThreads));
    oC0 = take((size_t)n);
    bytes = b;
  }
};

int check_screen_args(const rh_ctx* ctx, const rh_screen_params* params, int64_t series_len,
                      const double* hist, int64_t n, const double* observed) {
  if (!ctx || !params || n < 0 || series_len < 0 || params->window < 1 ||
      params->window > kMaxWindow || (n && !observed) || (series_len > 0 && !hist)) {
    set_error("rh_screen: invalid arguments (window must be 1..%d)", kMaxWindow);
    return RH_E_INVALID;
  }
  if (n >= 0x7fffffff) {
    set_error("rh_screen: batch too large");
    return RH_E_SHAPE;
  }
  return RH_OK;
}

void fill_inputs(ScreenArgs& a, const rh_screen_params* params, int64_t series_len,
                 const double* hist, int64_t n, const double* observed, const uint8_t* reset) {
  a = ScreenArgs{};
  a.w = params->window;
  a.fe = params->filter_enabled != 0;
  a.kappa = params->kappa;
  a.len0 = series_len;
  a.h = (int)std::min<int64_t>(series_len, params->window);
  a.hist = hist;
  a.n = n;
  a.obs = observed;
  a.reset = reset;
}

// reset indices + round-0 verdicts into the slot-2 workspace
int launch_prepare(rh_ctx* ctx, ScreenArgs& a, cudaStream_t st) {
  const PrepLayout L(a.n);
  void* ws = nullptr;
  if (int rc = workspace(ctx, L.bytes, &ws, 2, st)) return rc;
  a.prep_buf = ws;
  char* base = static_cast<char*>(ws);
  a.R = reinterpret_cast<int32_t*>(base + L.oR);
  a.bres = reinterpret_cast<int32_t*>(base + L.oRes);
  a.c0 = reinterpret_cast<uint8_t*>(base + L.oC0);
  const int64_t grid0 = (a.n + kScanThreads - 1) / kScanThreads;
  if (a.reset) {
    reset_scan_kernel<<<(unsigned)grid0, kScanThreads, 0, st>>>(a);
    RH_CHECK_LAUNCH(ctx);
  } else {
    RH_CUDA(cudaMemsetAsync(a.R, 0xff, sizeof(int32_t) * a.n, st));  // no resets: all -1
  }
  const int64_t grid_r0 = (a.n * 32 + kRound0Threads - 1) / kRound0Threads;
  round0_kernel<<<(unsigned)grid_r0, kRound0Threads, 0, st>>>(a);
  RH_CHECK_LAUNCH(ctx);
  return RH_OK;
}

}  // namespace

extern "C" int rh_screen_prepare(rh_ctx* ctx, const rh_screen_params* params,
                                 int64_t series_len, const double* hist, int64_t n,
                                 const double* observed, const uint8_t* reset, void* stream) {
  if (int rc = check_screen_args(ctx, params, series_len, hist, n, observed)) return rc;
  DeviceGuard guard(ctx);
  std::lock_guard<std::mutex> lock(ctx->prep_mu);
  ctx->prep.valid = false;
  if (n == 0) return RH_OK;
  cudaStream_t st = as_stream(stream);
  // the previous rh_screen may still read the slot-2 results (inside a graph
  // capture the fork from the capturing stream already orders us after it)
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  RH_CUDA(cudaStreamIsCapturing(st, &cap));
  if (ctx->prep.consumed_recorded && cap == cudaStreamCaptureStatusNone)
    RH_CUDA(cudaStreamWaitEvent(st, ctx->prep.consumed, 0));
  ScreenArgs a;
  fill_inputs(a, params, series_len, hist, n, observed, reset);
  if (int rc = launch_prepare(ctx, a, st)) return rc;
  if (!ctx->prep.done) RH_CUDA(cudaEventCreateWithFlags(&ctx->prep.done, cudaEventDisableTiming));
  RH_CUDA(cudaEventRecord(ctx->prep.done, st));
  auto& pr = ctx->prep;
  pr.window = params->window;
  pr.filter_enabled = params->filter_enabled;
  pr.kappa = params->kappa;
  pr.series_len = series_len;
  pr.n = n;
  pr.hist = hist;
  pr.observed = observed;
  pr.reset = reset;
  pr.buf = a.prep_buf;
  pr.valid = true;
  return RH_OK;
}

extern "C" int rh_screen(rh_ctx* ctx, const rh_screen_params* params, int64_t series_len,
                         const double* hist, int64_t n, const double* observed,
                         const uint8_t* it_status, const uint8_t* reset, uint8_t* outcome,
                         int64_t* series_len_out, void* stream) {
  if (int rc = check_screen_args(ctx, params, series_len, hist, n, observed)) return rc;
  if (n && (!it_status || !outcome)) {
    set_error("rh_screen: invalid arguments (NULL status / outcome)");
    return RH_E_INVALID;
  }
  cudaStream_t st = as_stream(stream);
  DeviceGuard guard(ctx);
  std::lock_guard<std::mutex> lock(ctx->prep_mu);
  const auto& pr = ctx->prep;
  const bool prepared = pr.valid && pr.window == params->window &&
                        pr.filter_enabled == params->filter_enabled && pr.kappa == params->kappa &&
                        pr.series_len == series_len && pr.n == n && pr.hist == hist &&
                        pr.observed == observed && pr.reset == reset;
  // a pending prepare may still be writing the slot-2 results: whether or not
  // they are usable here, nothing below may touch them before it finishes
  const bool pending = pr.valid;
  ctx->prep.valid = false;  // one use
  if (pending) RH_CUDA(cudaStreamWaitEvent(as_stream(stream), ctx->prep.done, 0));
  if (n == 0) {
    if (series_len_out)
      RH_CUDA(cudaMemcpyAsync(series_len_out, &series_len, sizeof(int64_t),
                              cudaMemcpyHostToDevice, st));
    return RH_OK;
  }
  int& occ = ctx->screen_occ;  // cached occupancy of the cooperative kernel
  if (occ < 0) {
    RH_CUDA(cudaFuncSetAttribute((void*)screen_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)sizeof(ScreenSmem)));
    RH_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (void*)screen_kernel,
                                                          kScreenThreads, sizeof(ScreenSmem)));
  }
  if (occ < 1) {
    set_error("rh_screen: kernel does not fit on an SM");
    return RH_E_SHAPE;
  }
  // co-resident CTAs (cooperative launch), about one warp per 2 iterations
  int blocks = ctx->num_sms * std::min(occ, kScreenBlocksPerSm);
  blocks = (int)std::max<int64_t>(
      1, std::min<int64_t>(blocks, (n + 2 * kScreenWarps - 1) / (2 * kScreenWarps)));
  ScreenArgs a;
  fill_inputs(a, params, series_len, hist, n, observed, reset);
  a.st = it_status;
  a.outcome = outcome;
  a.len_out = series_len_out;
  if (prepared) {
    const PrepLayout L(n);
    char* pbase = static_cast<char*>(pr.buf);
    a.R = reinterpret_cast<int32_t*>(pbase + L.oR);
    a.bres = reinterpret_cast<int32_t*>(pbase + L.oRes);
    a.c0 = reinterpret_cast<uint8_t*>(pbase + L.oC0);
  } else if (int rc = launch_prepare(ctx, a, st)) {
    return rc;
  }
  // control words: a dedicated per-stream block, zeroed on allocation (the
  // kernel leaves it zero); kept-state: the slot-1 workspace
  void* ctrl = nullptr;
  if (int rc = workspace(ctx, 256, &ctrl, 3, st, /*zero=*/true)) return rc;
  char* cb = static_cast<char*>(ctrl);
  a.kcnt = reinterpret_cast<unsigned long long*>(cb);       // 24 B
  a.cnt = reinterpret_cast<unsigned*>(cb + 32);             // 12 B
  a.bar = reinterpret_cast<unsigned*>(cb + 64);             // 8 B
  a.ticket = reinterpret_cast<unsigned*>(cb + 96);          // 4 B
  void* ws = nullptr;
  if (int rc = workspace(ctx, 2 * (size_t)n + 256, &ws, 1, st)) return rc;
  a.state = static_cast<uint8_t*>(ws);
  void* kargs[] = {&a};
  RH_CUDA(cudaLaunchCooperativeKernel((void*)screen_kernel, dim3(blocks), dim3(kScreenThreads),
                                      kargs, sizeof(ScreenSmem), st));
  RH_CHECK_LAUNCH(ctx);
  if (!ctx->prep.consumed)
    RH_CUDA(cudaEventCreateWithFlags(&ctx->prep.consumed, cudaEventDisableTiming));
  RH_CUDA(cudaEventRecord(ctx->prep.consumed, st));
  ctx->prep.consumed_recorded = true;
  return RH_OK;
}

extern "C" int rh_observe_host(rh_ctx* ctx, const rh_screen_params* params, int64_t series_len,
                               const double* hist, double observed, int32_t escalate,
                               int32_t do_validate, int32_t n_stage, const double* measured,
                               const double* expected, int32_t n_link, const double* link_ratio,
                               double threshold, uint8_t* stage_flag, double* stage_sev,
                               uint8_t* link_flag, double* link_sev, uint8_t* outcome,
                               int64_t* series_len_out) {
  if (!ctx || !params || series_len < 0 || params->window < 1 || params->window > kMaxWindow ||
      (series_len > 0 && !hist) || !outcome || !series_len_out || n_stage < 0 || n_link < 0 ||
      (do_validate && ((n_stage && (!measured || !expected || !stage_flag || !stage_sev)) ||
                       (n_link && (!link_ratio || !link_flag || !link_sev))))) {
    set_error("rh_observe_host: invalid arguments");
    return RH_E_INVALID;
  }
  DeviceGuard guard(ctx);
  const int h = (int)std::min<int64_t>(series_len, params->window);
  const bool v = do_validate != 0;
  HostCall c;
  const size_t oh = c.in(h ? hist : nullptr, 8 * (size_t)h);
  const size_t om = c.in(v ? measured : nullptr, v ? 8 * (size_t)n_stage : 0),
               oe = c.in(v ? expected : nullptr, v ? 8 * (size_t)n_stage : 0),
               ol = c.in(v ? link_ratio : nullptr, v ? 8 * (size_t)n_link : 0);
  const size_t osf = c.out(v ? stage_flag : nullptr, v ? (size_t)n_stage : 0),
               oss = c.out(v ? stage_sev : nullptr, v ? 8 * (size_t)n_stage : 0),
               olf = c.out(v ? link_flag : nullptr, v ? (size_t)n_link : 0),
               ols = c.out(v ? link_sev : nullptr, v ? 8 * (size_t)n_link : 0),
               ooc = c.out(outcome, 1), olen = c.out(series_len_out, 8);
  return c.run(ctx, [&](char* din, char* dout, cudaStream_t st) -> int {
    observe_kernel<<<1, kObserveThreads, 0, st>>>(
        params->window, params->filter_enabled != 0, params->kappa, series_len,
        reinterpret_cast<const double*>(din + oh), h, observed, escalate ? 1u : 0u, v ? 1 : 0,
        n_stage, reinterpret_cast<const double*>(din + om),
        reinterpret_cast<const double*>(din + oe), n_link,
        reinterpret_cast<const double*>(din + ol), threshold,
        reinterpret_cast<uint8_t*>(dout + osf), reinterpret_cast<double*>(dout + oss),
        reinterpret_cast<uint8_t*>(dout + olf), reinterpret_cast<double*>(dout + ols),
        reinterpret_cast<uint8_t*>(dout + ooc), reinterpret_cast<int64_t*>(dout + olen));
    RH_CHECK_LAUNCH(ctx);
    return RH_OK;
  });
}
