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

constexpr int kScreenThreads = 256;
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
  double* Vk;        // [n] compacted kept observations
  uint8_t* pop;      // [n] current pop decisions
  int32_t* bsum;     // [blocks]
  int32_t* bres;     // [blocks] last reset in block chunk
  unsigned* bar;     // [2] barrier count, generation
  int32_t* changed;  // [2]
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

// exclusive block scan of one int per thread; returns the block total
__device__ int block_exclusive_scan(int v, int* out_excl, int* smem) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int x = v;
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) smem[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int t = lane < (int)(blockDim.x >> 5) ? smem[lane] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    smem[lane] = t;  // inclusive warp totals
  }
  __syncthreads();
  const int warp_off = wid ? smem[wid - 1] : 0;
  *out_excl = warp_off + x - v;
  const int total = smem[(blockDim.x >> 5) - 1];
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

// pop decision + outcome bits of iteration i under the current kept-set
__device__ uint8_t decide(const ScreenArgs& a, int64_t i, bool& pop) {
  const int w = a.w;
  const int32_t r = a.R[i];
  const int64_t pb = __ldcg(a.Pk + i);
  const int64_t base = r >= 0 ? __ldcg(a.Pk + r) : 0;
  const int64_t nk = pb - base;
  const int64_t len_before = r >= 0 ? nk : a.len0 + nk;
  const int64_t len = len_before + 1;
  const double x = a.obs[i];
  bool cand = false;
  if (len >= w + 1) {
    double win[kMaxWindow], dev[kMaxWindow];
    int c = 0;
    if (nk < w) {  // only without a reset: the window starts in the history
      for (int q = a.h - (w - (int)nk); q < a.h; ++q) win[c++] = a.hist[q];
      for (int64_t q = base; q < pb; ++q) win[c++] = __ldcg(a.Vk + q);
    } else {
      for (int64_t q = pb - w; q < pb; ++q) win[c++] = __ldcg(a.Vk + q);
    }
    for (int q = 0; q < w; ++q) dev[q] = win[q];
    sort_small(dev, w);
    const double med = median_sorted(dev, w);
    for (int q = 0; q < w; ++q) dev[q] = fabs(__dsub_rn(win[q], med));
    sort_small(dev, w);
    const double mad = median_sorted(dev, w);
    cand = fabs(__dsub_rn(x, med)) > __dmul_rn(a.kappa, mad);
  }
  const bool refill = !cand && a.fe && len <= w;
  pop = false;
  if (!cand && !refill) return 0;
  uint8_t oc = cand ? RH_SC_CANDIDATE : 0;
  const uint8_t st = a.st[i];
  if (a.fe) {
    oc |= RH_SC_FILTERED;
    if (!(st & RH_IT_ESCALATE)) {
      if (cand) {
        pop = true;
        oc |= RH_SC_POPPED;
      }
      return oc;
    }
  }
  oc |= RH_SC_ESCALATED;
  if (!(st & (RH_IT_STAGE_FLAG | RH_IT_LINK_FLAG))) {
    pop = true;
    oc |= RH_SC_POPPED;
  } else {
    oc |= RH_SC_CONFIRMED;
  }
  return oc;
}

__global__ void __launch_bounds__(kScreenThreads) screen_kernel(const ScreenArgs a) {
  __shared__ int sm[32];
  __shared__ int s_pref, s_res, s_changed;
  const unsigned nb = gridDim.x;
  const int64_t per_block = (a.n + nb - 1) / nb;
  const int64_t b0 = (int64_t)blockIdx.x * per_block;
  const int64_t b1 = min(a.n, b0 + per_block);
  const int64_t per_thread = (per_block + blockDim.x - 1) / blockDim.x;
  const int64_t t0 = min(b1, b0 + (int64_t)threadIdx.x * per_thread);
  const int64_t t1 = min(b1, t0 + per_thread);

  // ---- last reset index <= i (once)
  {
    int last = -1;
    if (a.reset)
      for (int64_t i = t0; i < t1; ++i)
        if (a.reset[i]) last = (int)i;
    // block max-scan (inclusive) via warp shuffles + smem
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int x = last;
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x = max(x, y);
    }
    if (lane == 31) sm[wid] = x;
    __syncthreads();
    if (wid == 0) {
      int t = lane < (int)(blockDim.x >> 5) ? sm[lane] : -1;
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, t, o);
        if (lane >= o) t = max(t, y);
      }
      sm[lane] = t;
    }
    __syncthreads();
    int excl = __shfl_up_sync(0xffffffffu, x, 1);
    if (lane == 0) excl = wid ? sm[wid - 1] : -1;
    else excl = max(excl, wid ? sm[wid - 1] : -1);
    if (threadIdx.x == 0) a.bres[blockIdx.x] = sm[(blockDim.x >> 5) - 1];
    for (int64_t i = t0; i < t1; ++i) {
      if (a.reset && a.reset[i]) excl = (int)i;
      a.R[i] = excl;  // block-local; fixed up below
    }
    for (int64_t i = t0; i < t1; ++i) a.pop[i] = 0;
    grid_barrier(a.bar, nb);
    if (threadIdx.x == 0) {
      int m = -1;
      for (unsigned b = 0; b < blockIdx.x; ++b) m = max(m, __ldcg(a.bres + b));
      s_res = m;
    }
    __syncthreads();
    for (int64_t i = t0; i < t1; ++i)
      if (a.R[i] < 0) a.R[i] = s_res;
  }

  for (int64_t round = 0; round <= a.n + 1; ++round) {
    // ---- phase A: kept counts
    int cnt = 0;
    for (int64_t i = t0; i < t1; ++i) cnt += a.pop[i] ? 0 : 1;
    int excl;
    const int tot = block_exclusive_scan(cnt, &excl, sm);
    if (threadIdx.x == 0) a.bsum[blockIdx.x] = tot;
    grid_barrier(a.bar, nb);
    // ---- phase B: global prefix + compaction
    if (threadIdx.x == 0) {
      int acc = 0;
      for (unsigned b = 0; b < blockIdx.x; ++b) acc += __ldcg(a.bsum + b);
      s_pref = acc;
      if (blockIdx.x == 0) a.changed[(round + 1) & 1] = 0;
    }
    __syncthreads();
    {
      int64_t pos = (int64_t)s_pref + excl;
      for (int64_t i = t0; i < t1; ++i) {
        a.Pk[i] = (int32_t)pos;
        if (!a.pop[i]) a.Vk[pos++] = a.obs[i];
      }
      if (t1 == a.n && t1 > t0) a.Pk[a.n] = (int32_t)pos;
    }
    grid_barrier(a.bar, nb);
    // ---- phase C: decisions
    int ch = 0;
    for (int64_t i = t0; i < t1; ++i) {
      bool p;
      const uint8_t oc = decide(a, i, p);
      a.outcome[i] = oc;
      if ((uint8_t)p != a.pop[i]) {
        a.pop[i] = p;
        ch = 1;
      }
    }
    if (__syncthreads_or(ch) && threadIdx.x == 0) atomicExch(a.changed + (round & 1), 1);
    grid_barrier(a.bar, nb);
    if (threadIdx.x == 0) s_changed = __ldcg(a.changed + (round & 1));
    __syncthreads();
    if (!s_changed) break;
  }
  // final series length (the decisions are the fixpoint now)
  if (blockIdx.x == nb - 1 && threadIdx.x == 0 && a.len_out) {
    // recount kept after the last reset
    const int64_t last = a.n - 1;
    const int32_t r = __ldcg(a.R + last);
    int64_t kept_total = __ldcg(a.Pk + last) + (__ldcg(a.pop + last) ? 0 : 1);
    int64_t len = r >= 0 ? kept_total - __ldcg(a.Pk + r) : a.len0 + kept_total;
    *a.len_out = len;
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
  int max_blocks_per_sm = 0;
  RH_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&max_blocks_per_sm, screen_kernel,
                                                        kScreenThreads, 0));
  int blocks = ctx->num_sms * std::max(1, std::min(max_blocks_per_sm, 1));
  const int64_t want = (n + kScreenThreads - 1) / kScreenThreads;
  if (want < blocks) blocks = (int)std::max<int64_t>(1, want);
  size_t bytes = 0;
  auto align = [](size_t x) { return (x + 255) & ~size_t(255); };
  const size_t oR = 0;
  bytes = align(oR + sizeof(int32_t) * n);
  const size_t oP = bytes;
  bytes = align(oP + sizeof(int32_t) * (n + 1));
  const size_t oV = bytes;
  bytes = align(oV + sizeof(double) * n);
  const size_t oPop = bytes;
  bytes = align(oPop + n);
  const size_t oB = bytes;
  bytes = align(oB + sizeof(int32_t) * blocks * 2);
  const size_t oBar = bytes;
  bytes = align(oBar + sizeof(unsigned) * 2 + sizeof(int32_t) * 2);
  void* ws = nullptr;
  int rc = workspace(ctx, bytes, &ws);
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
  a.Vk = reinterpret_cast<double*>(base + oV);
  a.pop = reinterpret_cast<uint8_t*>(base + oPop);
  a.bsum = reinterpret_cast<int32_t*>(base + oB);
  a.bres = a.bsum + blocks;
  a.bar = reinterpret_cast<unsigned*>(base + oBar);
  a.changed = reinterpret_cast<int32_t*>(a.bar + 2);
  RH_CUDA(cudaMemsetAsync(a.bar, 0, sizeof(unsigned) * 2 + sizeof(int32_t) * 2, st));
  void* kargs[] = {&a};
  RH_CUDA(cudaLaunchCooperativeKernel((const void*)screen_kernel, dim3(blocks),
                                      dim3(kScreenThreads), kargs, 0, st));
  RH_CHECK_LAUNCH(ctx);
  return RH_OK;
}
