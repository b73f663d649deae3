// The canonical 1F1B / ZBH chunk-DAG recurrence of one replica pipeline,
// shared by the Detector pass (pipeline.cu) and the candidate search
// (search.cu).
//
// Lane s of a pw-lane group (pw = next_pow2(P), lanes >= P idle) walks the
// chunk chain of stage s (pipeline.py:92-126) and computes, for each chunk v,
//   c(v)     = ((ratio(kind)*L_s) * base_j) / p_s        (workload.py:88-98)
//   start(v) = max(finish(previous chunk of s), finish(data pred) + hop)
//   finish(v)= start(v) + c(v)                           (pipeline.py:275-291)
// returning the last finish (the stage's contribution to the makespan), the
// chain-order cost sum (pipeline.py:446-453) and the activation check
// (pipeline.py:516-539: on one resource the chain order is the time order).
//
// Static wavefront.  Every chunk is processed at its DAG level (longest path
// from a source, in chunks), which has a closed form for the canonical
// schedules (w = min(P-1-s, M), M = micro-batches of the replica):
//   F_j           : s + j               if j <= w, else 2j + s
//   B_j / BW_j    : 2P - 1 - s + 2j
//   W_j (ZBH)     : 2P - s + 2(M - w + j)                 if j < w (drain)
//                   last drain/B level + (j - w + 1)      otherwise (tail)
// (checked against the exact DAG levels for P <= 32, M <= 64, both
// schedules — tests/test_wavefront_property.py).  Along a chain these levels
// strictly increase, so a lane only compares the step t with the level of its
// next F, next B and next W.  At the start of step t the neighbours publish,
// by warp shuffle, the finish of the last F / B they completed; a B
// dependency is always exactly one level old and a producer never leads its
// consumer by more than one F, so those are exactly the needed values.  No
// readiness checks, no shared memory.
//
// Every lane of the warp must call this (full-mask shuffles / reductions).
// All fp64 ops are explicit _rn intrinsics (no FMA contraction).
#pragma once

#include <climits>

#include "common.cuh"

namespace rh {

// Exact fp64 division, out of line so the common unit-speed path is a branch
// over it rather than an always-executed predicated sequence.
__device__ __noinline__ inline double div_slow(double a, double b) { return __ddiv_rn(a, b); }

// Correctly rounded a / b with a hoisted reciprocal y = __drcp_rn(b)
// (Markstein): q = RN(a*y), r = a - b*q exactly (FMA), RN(q + r*y) = RN(a/b)
// whenever nothing under- or overflows.  Outside a conservative range it
// defers to __ddiv_rn, so the result always equals __ddiv_rn(a, b)
// (rh_selftest_division checks this on the device).  With b == 1, y == 1:
// q = a, r = 0 and the result is a -- unit speeds cost 3 flops, no branch.
// Safe range: a == 0 or |a| in [2^-900, 2^900], b in [2^-100, 2^100] -- then
// a/b, the residual and r*y are all normal.  recip_of returns 0 for an
// out-of-range b, which sends every division by it to __ddiv_rn.
__device__ __forceinline__ double div_recip(double a, double b, double y) {
  const double q = __dmul_rn(a, y);
  const double r = __fma_rn(-b, q, a);
  const double res = __fma_rn(r, y, q);
  const double aa = fabs(a);
  if (!((aa >= 0x1p-900 && aa <= 0x1p900) || a == 0.0) || y == 0.0) return div_slow(a, b);
  return res;
}

// div_recip without the per-call range test, for callers that checked the
// operand ranges once for a whole walk (see div_range_ok).
__device__ __forceinline__ double div_fast(double a, double b, double y) {
  const double q = __dmul_rn(a, y);
  return __fma_rn(__fma_rn(-b, q, a), y, q);
}

// every numerator of a walk lies in [lo, hi] (lo = smallest non-zero one):
// div_fast is then exact for divisors with recip_of(b) != 0
__device__ __forceinline__ bool div_range_ok(double lo, double hi) {
  return !(hi > 0x1p900) && (hi == 0.0 || lo >= 0x1p-900);
}

__device__ __forceinline__ double recip_of(double b) {
  if (!(b >= 0x1p-100 && b <= 0x1p100)) return 0.0;
  return b == 1.0 ? 1.0 : __drcp_rn(b);
}

struct ChainLevels {
  int s, P, m, w;
  __host__ __device__ __forceinline__ constexpr int F(int j) const {
    return j >= m ? INT_MAX : (j <= w ? s + j : 2 * j + s);
  }
  __host__ __device__ __forceinline__ constexpr int B(int j) const { return j >= m ? INT_MAX : 2 * P - 1 - s + 2 * j; }
  __host__ __device__ __forceinline__ constexpr int W(int j) const {
    if (j >= m) return INT_MAX;
    if (j < w) return 2 * P - s + 2 * (m - w + j);
    return (w > 0 ? 2 * P - s + 2 * m - 2 : 2 * P - 1 - s + 2 * (m - 1)) + (j - w + 1);
  }
  // Inverse: the chunk of this chain at level t -- kind 1 F, 2 B/BW, 3 W (ZBH),
  // 0 none -- and its micro-batch j.  A chain holds at most one chunk per level.
  __host__ __device__ __forceinline__ constexpr int at(int t, bool zbh, int& j) const {
    const int k = t - s;
    if (k >= 0 && k <= w && k < m) {
      j = k;
      return 1;
    }
    if (k > 2 * w && (k & 1) == 0 && k / 2 < m) {
      j = k / 2;
      return 1;
    }
    const int kb = t - (2 * P - 1 - s);
    if (kb >= 0 && (kb & 1) == 0 && kb / 2 < m) {
      j = kb / 2;
      return 2;
    }
    if (zbh) {
      const int kw = t - (2 * P - s) - 2 * (m - w);
      if (kw >= 0 && (kw & 1) == 0 && kw / 2 < w) {
        j = kw / 2;
        return 3;
      }
      const int tail = w > 0 ? 2 * P - s + 2 * m - 2 : 2 * P - 1 - s + 2 * (m - 1);
      const int jt = t - tail + w - 1;
      if (jt >= w && jt < m) {
        j = jt;
        return 3;
      }
    }
    j = 0;
    return 0;
  }
  // one past the last level of the chain
  __host__ __device__ __forceinline__ constexpr int end(bool zbh) const {
    return m == 0 ? 0 : 1 + (zbh ? W(m - 1) : B(m - 1));
  }
};

template <int ZBH>
__device__ __forceinline__ void chain_walk(int s, int P, int pw, int md, int w, int n_chain,
                                           const double* base, double rlF, double rlB,
                                           double rlW, double sp, double hopf, double hopb,
                                           int cap, int /*mmax*/, double& fin, double& ssum,
                                           bool& over, bool& /*hung*/) {
  const double inv = recip_of(sp);  // exact division by div_recip
  const ChainLevels lv{s, P, n_chain > 0 ? md : 0, w};
  int jf = 0, jb = 0, jw = 0, live = 0;
  int LF = lv.F(0), LB = lv.B(0), LW = ZBH ? lv.W(0) : INT_MAX;
  const int last = lv.m == 0 ? 0 : 1 + (ZBH ? lv.W(lv.m - 1) : lv.B(lv.m - 1));
  const int T = __reduce_max_sync(0xffffffffu, last);
  const double hF = s > 0 ? hopf : 0.0, hB = s < P - 1 ? hopb : 0.0;
  const bool getF = s > 0, getB = s < P - 1;
  double lastF = 0.0, lastB = 0.0;
  // Branch-free step: F-, B- and idle lanes of a warp execute the same
  // instruction stream (selects instead of divergent paths; division by the
  // stage speed is the branch-free div_recip).
  const int jmax = lv.m > 0 ? lv.m - 1 : 0;
  for (int t = 0; t < T; ++t) {
    const double nF = __shfl_up_sync(0xffffffffu, lastF, 1, pw);
    const double nB = __shfl_down_sync(0xffffffffu, lastB, 1, pw);
    const bool doF = t == LF, doB = t == LB, doW = ZBH && t == LW;
    const bool act = doF || doB || doW;
    const double dF = getF ? __dadd_rn(nF, hF) : 0.0;
    const double dB = getB ? __dadd_rn(nB, hB) : 0.0;
    const double dep = doF ? dF : (doB ? dB : 0.0);
    const double rl = doF ? rlF : (doB ? rlB : rlW);
    const int j = min(doF ? jf : (doB ? jb : jw), jmax);
    const double c = div_recip(__dmul_rn(rl, base[j]), sp, inv);
    const double st = fin > dep ? fin : dep;  // max (no NaNs on this path)
    const double nf = __dadd_rn(st, c);
    fin = act ? nf : fin;
    ssum = act ? __dadd_rn(ssum, c) : ssum;
    lastF = doF ? nf : lastF;
    lastB = doB ? nf : lastB;
    jf += doF;
    jb += doB;
    if (ZBH) jw += doW;
    LF = doF ? lv.F(jf) : LF;
    LB = doB ? lv.B(jb) : LB;
    if (ZBH) LW = doW ? lv.W(jw) : LW;
    live += (int)doF - (int)doB;
    over = over || (cap > 0 && doF && live > cap);
  }
}

}  // namespace rh
