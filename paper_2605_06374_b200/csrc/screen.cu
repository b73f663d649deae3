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
// by Jacobi iteration on the whole grid: start from kept = all, recompute
// every decision in parallel from the current kept-set (prefix sums +
// compaction give each iteration its window in O(window)), repeat until no
// decision changes.  The fixpoint of this system is unique and equal to the
// sequential answer (induction on i); each round fixes at least one more
// leading decision, so it terminates, and in practice pops are sparse and it
// converges in 2-3 rounds.  One cooperative launch; rounds are separated by
// a grid barrier (the blocks are co-resident by construction).
#include <algorithm>

#include "common.cuh"

namespace rh {

constexpr int kScreenThreads = 128;
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
  int32_t* R;        // [n] last reset index <= i, or -1
  int32_t* Pk;       // [n+1] exclusive count of kept before i
  int32_t* Cc;       // [n+1] exclusive count of changed decisions before i
  int32_t* Kidx;     // [n] compacted position -> iteration index
  double* Vk;        // [n] compacted kept observations
  uint8_t* pop;      // [n] current pop decisions
  uint8_t* chg;      // [n] decision changed in the last round
  int32_t* bsum;     // [2*blocks] per-block (kept, changed)
  int32_t* bres;     // [blocks] last reset in block chunk
  unsigned* bar;     // [2] barrier count, generation
};

__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* gen = bar + 1;
    const unsigned g = *gen;
    __threadfence();
    if (atomicAdd(bar, 1u) == nblocks - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*gen == g) {
      }
    }
    __threadfence();
  }
  __syncthreads();
}

// exclusive block scan of two ints per thread; returns the block totals
__device__ int2 block_exclusive_scan2(int2 v, int2* out_excl, int2* smem) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int2 x = v;
  for (int o = 1; o < 32; o <<= 1) {
    const int a = __shfl_up_sync(0xffffffffu, x.x, o);
    const int b = __shfl_up_sync(0xffffffffu, x.y, o);
    if (lane >= o) {
      x.x += a;
      x.y += b;
    }
  }
  if (lane == 31) smem[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int2 t = lane < (int)(blockDim.x >> 5) ? smem[lane] : make_int2(0, 0);
    for (int o = 1; o < 32; o <<= 1) {
      const int a = __shfl_up_sync(0xffffffffu, t.x, o);
      const int b = __shfl_up_sync(0xffffffffu, t.y, o);
      if (lane >= o) {
        t.x += a;
        t.y += b;
      }
    }
    smem[lane] = t;  // inclusive warp totals
  }
  __syncthreads();
  const int2 off = wid ? smem[wid - 1] : make_int2(0, 0);
  *out_excl = make_int2(off.x + x.x - v.x, off.y + x.y - v.y);
  const int2 total = smem[(blockDim.x >> 5) - 1];
  __syncthreads();
  return total;
}

__device__ __forceinline__ void sort_small(double* a, int n) {
  for (int i = 1; i < n; ++i) {
    const double v = a[i];
    int j = i - 1;
    while (j >= 0 && a[j] > v) {
      a[j + 1] = a[j];
      --j;
    }
    a[j + 1] = v;
  }
}

// statistics.median on a sorted array
__device__ __forceinline__ double median_sorted(const double* a, int n) {
  return (n & 1) ? a[n >> 1] : __ddiv_rn(__dadd_rn(a[(n >> 1) - 1], a[n >> 1]), 2.0);
}

// odd-even transposition sort, fully unrolled: the array stays in registers
template <int W>
__device__ __forceinline__ void sort_net(double (&a)[W]) {
#pragma unroll
  for (int r = 0; r < W; ++r) {
#pragma unroll
    for (int i = r & 1; i + 1 < W; i += 2) {
      const double lo = fmin(a[i], a[i + 1]);
      const double hi = fmax(a[i], a[i + 1]);
      a[i] = lo;
      a[i + 1] = hi;
    }
  }
}

template <int W>
__device__ __forceinline__ double median_net(const double (&a)[W]) {
  if (W & 1) return a[W >> 1];
  return __ddiv_rn(__dadd_rn(a[(W >> 1) - 1], a[W >> 1]), 2.0);
}

// |x - median| > kappa * MAD over a window (statistics.median semantics)
template <int W>
__device__ __forceinline__ bool outlier_fixed(const double* win_src, bool cg, double x,
                                              double kappa) {
  double v[W], d[W];
#pragma unroll
  for (int q = 0; q < W; ++q) v[q] = cg ? __ldcg(win_src + q) : win_src[q];
#pragma unroll
  for (int q = 0; q < W; ++q) d[q] = v[q];
  sort_net<W>(d);
  const double med = median_net<W>(d);
#pragma unroll
  for (int q = 0; q < W; ++q) d[q] = fabs(__dsub_rn(v[q], med));
  sort_net<W>(d);
  const double mad = median_net<W>(d);
  return fabs(__dsub_rn(x, med)) > __dmul_rn(kappa, mad);
}

__device__ __noinline__ bool outlier_generic(const double* win, int w, double x, double kappa) {
  double dev[kMaxWindow];
  for (int q = 0; q < w; ++q) dev[q] = win[q];
  sort_small(dev, w);
  const double med = median_sorted(dev, w);
  for (int q = 0; q < w; ++q) dev[q] = fabs(__dsub_rn(win[q], med));
  sort_small(dev, w);
  const double mad = median_sorted(dev, w);
  return fabs(__dsub_rn(x, med)) > __dmul_rn(kappa, mad);
}

// Pop decision + outcome bits of iteration i under the current kept-set.
// identity: every earlier iteration is kept (round 0: positions == indices).
// Returns false (and leaves outputs alone) when the iteration is provably
// unaffected by the last round's changes.
template <int WF>
__device__ bool decide(const ScreenArgs& a, int64_t i, bool identity, uint8_t& oc_out,
                       bool& pop) {
  const int w = WF > 0 ? WF : a.w;
  const int32_t r = a.R[i];
  const int64_t pb = identity ? i : __ldcg(a.Pk + i);
  const int64_t base = r >= 0 ? (identity ? r : __ldcg(a.Pk + r)) : 0;
  const int64_t nk = pb - base;
  if (!identity) {
    // only changes inside the window span -- or, while the series is short,
    // anywhere since the reset (length thresholds) -- can alter the decision
    const int64_t first = r >= 0 ? r : 0;
    const int32_t ci = __ldcg(a.Cc + i);
    const int32_t c_all = ci - __ldcg(a.Cc + first);
    if (c_all == 0) return false;
    if (nk - c_all >= w + 2) {
      const int64_t lb = __ldcg(a.Kidx + (pb - w));
      if (ci - __ldcg(a.Cc + lb) == 0) return false;
    }
  }
  const int64_t len = (r >= 0 ? nk : a.len0 + nk) + 1;
  const double x = a.obs[i];
  const double* V = identity ? a.obs : a.Vk;
  bool cand = false;
  if (len >= w + 1) {
    if (nk >= w && WF > 0) {
      cand = outlier_fixed<(WF > 0 ? WF : 1)>(V + (pb - w), !identity, x, a.kappa);
    } else {
      double win[kMaxWindow];
      int c = 0;
      if (nk < w) {  // only without a reset: the window starts in the history
        for (int q = a.h - (w - (int)nk); q < a.h; ++q) win[c++] = a.hist[q];
        for (int64_t q = base; q < pb; ++q) win[c++] = identity ? V[q] : __ldcg(V + q);
      } else {
        for (int64_t q = pb - w; q < pb; ++q) win[c++] = identity ? V[q] : __ldcg(V + q);
      }
      cand = outlier_generic(win, w, x, a.kappa);
    }
  }
  const bool refill = !cand && a.fe && len <= w;
  pop = false;
  uint8_t oc = 0;
  if (cand || refill) {
    oc = cand ? RH_SC_CANDIDATE : 0;
    const uint8_t st = a.st[i];
    bool done = false;
    if (a.fe) {
      oc |= RH_SC_FILTERED;
      if (!(st & RH_IT_ESCALATE)) {
        if (cand) {
          pop = true;
          oc |= RH_SC_POPPED;
        }
        done = true;
      }
    }
    if (!done) {
      oc |= RH_SC_ESCALATED;
      if (!(st & (RH_IT_STAGE_FLAG | RH_IT_LINK_FLAG))) {
        pop = true;
        oc |= RH_SC_POPPED;
      } else {
        oc |= RH_SC_CONFIRMED;
      }
    }
  }
  oc_out = oc;
  return true;
}

// last reset index <= i: block-local inclusive max-scan, one element per
// thread; block summaries land in bres and are folded in by round0_kernel
__global__ void __launch_bounds__(kScreenThreads) reset_scan_kernel(ScreenArgs a) {
  __shared__ int sm[32];
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int x = (i < a.n && a.reset && a.reset[i]) ? (int)i : -1;
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

// round 0 on every SM: each iteration decided as if all earlier were kept
template <int WF>
__global__ void __launch_bounds__(kScreenThreads) round0_kernel(ScreenArgs a) {
  __shared__ int s_prev;
  if (threadIdx.x < 32) {
    int m = -1;
    for (unsigned b = threadIdx.x; b < blockIdx.x; b += 32) m = max(m, a.bres[b]);
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0) s_prev = m;
  }
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n) return;
  if (a.R[i] < s_prev) a.R[i] = s_prev;
  uint8_t oc;
  bool p;
  decide<WF>(a, i, true, oc, p);
  a.outcome[i] = oc;
  a.pop[i] = p;
  a.chg[i] = p;
}

template <int WF>
__global__ void __launch_bounds__(kScreenThreads) screen_kernel(const ScreenArgs a) {
  __shared__ int2 sm2[32];
  __shared__ int s_pref_k, s_pref_c, s_total_c;
  const unsigned nb = gridDim.x;
  const int64_t per_block = (a.n + nb - 1) / nb;
  const int64_t b0 = (int64_t)blockIdx.x * per_block;
  const int64_t b1 = min(a.n, b0 + per_block);
  const int64_t per_thread = (per_block + blockDim.x - 1) / blockDim.x;
  const int64_t t0 = min(b1, b0 + (int64_t)threadIdx.x * per_thread);
  const int64_t t1 = min(b1, t0 + per_thread);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;

  for (int64_t round = 1; round <= a.n + 2; ++round) {
    // ---- phase A: kept / changed counts
    int2 cnt = make_int2(0, 0);
    for (int64_t i = t0; i < t1; ++i) {
      cnt.x += a.pop[i] ? 0 : 1;
      cnt.y += a.chg[i];
    }
    int2 excl;
    const int2 tot = block_exclusive_scan2(cnt, &excl, sm2);
    if (threadIdx.x == 0) {
      a.bsum[2 * blockIdx.x] = tot.x;
      a.bsum[2 * blockIdx.x + 1] = tot.y;
    }
    grid_barrier(a.bar, nb);
    // ---- phase B: global prefixes + compaction
    if (wid == 0) {
      int pk = 0, pc = 0, tc = 0;
      for (unsigned b = lane; b < nb; b += 32) {
        const int k = __ldcg(a.bsum + 2 * b), c = __ldcg(a.bsum + 2 * b + 1);
        if (b < blockIdx.x) {
          pk += k;
          pc += c;
        }
        tc += c;
      }
      for (int o = 16; o > 0; o >>= 1) {
        pk += __shfl_xor_sync(0xffffffffu, pk, o);
        pc += __shfl_xor_sync(0xffffffffu, pc, o);
        tc += __shfl_xor_sync(0xffffffffu, tc, o);
      }
      if (lane == 0) {
        s_pref_k = pk;
        s_pref_c = pc;
        s_total_c = tc;
      }
    }
    __syncthreads();
    {
      int64_t pos = (int64_t)s_pref_k + excl.x;
      int32_t cc = s_pref_c + excl.y;
      for (int64_t i = t0; i < t1; ++i) {
        a.Pk[i] = (int32_t)pos;
        a.Cc[i] = cc;
        cc += a.chg[i];
        if (!a.pop[i]) {
          a.Vk[pos] = a.obs[i];
          a.Kidx[pos] = (int32_t)i;
          ++pos;
        }
      }
      if (t1 == a.n && t1 > t0) {
        a.Pk[a.n] = (int32_t)pos;
        a.Cc[a.n] = cc;
      }
    }
    if (s_total_c == 0) break;  // fixpoint: the last round changed nothing
    grid_barrier(a.bar, nb);
    // ---- phase C: re-decide the iterations the changes can reach
    for (int64_t i = t0; i < t1; ++i) {
      uint8_t oc;
      bool p;
      uint8_t changed = 0;
      if (decide<WF>(a, i, false, oc, p)) {
        a.outcome[i] = oc;
        changed = (uint8_t)p != a.pop[i];
        a.pop[i] = p;
      }
      a.chg[i] = changed;
    }
  }
  // final series length (Pk reflects the fixpoint decisions)
  if (a.len_out && t1 == a.n && t1 > t0) {
    const int64_t last = a.n - 1;
    const int32_t r = a.R[last];
    const int64_t kept_total = a.Pk[last] + (a.pop[last] ? 0 : 1);
    *a.len_out = r >= 0 ? kept_total - __ldcg(a.Pk + r) : a.len0 + kept_total;
  }
}

}  // namespace rh

using namespace rh;

extern "C" int rh_screen(rh_ctx* ctx, const rh_screen_params* params, int64_t series_len,
                         const double* hist, int64_t n, const double* observed,
                         const uint8_t* it_status, const uint8_t* reset, uint8_t* outcome,
                         int64_t* series_len_out, void* stream) {
  if (!ctx || !params || n < 0 || series_len < 0 || params->window < 1 ||
      params->window > kMaxWindow || (n && (!observed || !it_status || !outcome)) ||
      (series_len > 0 && !hist)) {
    set_error("rh_screen: invalid arguments (window must be 1..%d)", kMaxWindow);
    return RH_E_INVALID;
  }
  if (n >= 0x7fffffff) {
    set_error("rh_screen: batch too large");
    return RH_E_SHAPE;
  }
  cudaStream_t st = as_stream(stream);
  if (n == 0) {
    if (series_len_out)
      RH_CUDA(cudaMemcpyAsync(series_len_out, &series_len, sizeof(int64_t),
                              cudaMemcpyHostToDevice, st));
    return RH_OK;
  }
  const bool w20 = params->window == 20;
  void* coop = w20 ? (void*)screen_kernel<20> : (void*)screen_kernel<0>;
  static int occ[2] = {-1, -1};  // cached occupancy of the two instantiations
  int& max_blocks_per_sm = occ[w20 ? 1 : 0];
  if (max_blocks_per_sm < 0)
    RH_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&max_blocks_per_sm, coop,
                                                          kScreenThreads, 0));
  if (max_blocks_per_sm < 1) {
    set_error("rh_screen: kernel does not fit on an SM");
    return RH_E_SHAPE;
  }
  int blocks = ctx->num_sms;  // one co-resident CTA per SM (cooperative launch)
  const int64_t grid0 = (n + kScreenThreads - 1) / kScreenThreads;
  if (grid0 < blocks) blocks = (int)std::max<int64_t>(1, grid0);
  size_t bytes = 0;
  auto take = [&](size_t n_bytes) {
    const size_t o = bytes;
    bytes = (bytes + n_bytes + 255) & ~size_t(255);
    return o;
  };
  const size_t oR = take(sizeof(int32_t) * n), oP = take(sizeof(int32_t) * (n + 1));
  const size_t oC = take(sizeof(int32_t) * (n + 1)), oK = take(sizeof(int32_t) * n);
  const size_t oV = take(sizeof(double) * n), oPop = take(n), oChg = take(n);
  const size_t oB = take(sizeof(int32_t) * blocks * 2);
  const size_t oRes = take(sizeof(int32_t) * grid0), oBar = take(sizeof(unsigned) * 2);
  void* ws = nullptr;
  int rc = workspace(ctx, bytes, &ws, 1);
  if (rc) return rc;
  char* base = static_cast<char*>(ws);
  ScreenArgs a;
  a.w = params->window;
  a.fe = params->filter_enabled != 0;
  a.kappa = params->kappa;
  a.len0 = series_len;
  a.h = (int)std::min<int64_t>(series_len, params->window);
  a.hist = hist;
  a.n = n;
  a.obs = observed;
  a.st = it_status;
  a.reset = reset;
  a.outcome = outcome;
  a.len_out = series_len_out;
  a.R = reinterpret_cast<int32_t*>(base + oR);
  a.Pk = reinterpret_cast<int32_t*>(base + oP);
  a.Cc = reinterpret_cast<int32_t*>(base + oC);
  a.Kidx = reinterpret_cast<int32_t*>(base + oK);
  a.Vk = reinterpret_cast<double*>(base + oV);
  a.pop = reinterpret_cast<uint8_t*>(base + oPop);
  a.chg = reinterpret_cast<uint8_t*>(base + oChg);
  a.bsum = reinterpret_cast<int32_t*>(base + oB);
  a.bres = reinterpret_cast<int32_t*>(base + oRes);
  a.bar = reinterpret_cast<unsigned*>(base + oBar);
  RH_CUDA(cudaMemsetAsync(a.bar, 0, sizeof(unsigned) * 2, st));
  reset_scan_kernel<<<(unsigned)grid0, kScreenThreads, 0, st>>>(a);
  RH_CHECK_LAUNCH(ctx);
  if (w20)
    round0_kernel<20><<<(unsigned)grid0, kScreenThreads, 0, st>>>(a);
  else
    round0_kernel<0><<<(unsigned)grid0, kScreenThreads, 0, st>>>(a);
  RH_CHECK_LAUNCH(ctx);
  void* kargs[] = {&a};
  RH_CUDA(cudaLaunchCooperativeKernel(coop, dim3(blocks), dim3(kScreenThreads), kargs, 0, st));
  RH_CHECK_LAUNCH(ctx);
  return RH_OK;
}
