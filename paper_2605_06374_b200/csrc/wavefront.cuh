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
// Data predecessors live on the neighbouring lanes and travel by warp
// shuffle: each lane publishes (index, finish) of the last F and the last
// B/BW it completed.  In the canonical DAG a B dependency is produced exactly
// one step before it is consumed and a producer never runs more than one F
// ahead of its consumer (verified exhaustively for P <= 32, M <= 64, both
// schedules — DESIGN.md §3), so the published value is exactly the needed
// one; an index skip is detected and reported through `hung`.
//
// Every lane of the warp must call this (warp-synchronous: __any_sync and
// full-mask shuffles).  All fp64 ops are explicit _rn intrinsics.
#pragma once

#include "common.cuh"

namespace rh {

// Exact fp64 division, out of line so the common unit-speed path is a branch
// over it rather than an always-executed predicated sequence.
__device__ __noinline__ inline double div_slow(double a, double b) { return __ddiv_rn(a, b); }

template <int ZBH>
__device__ __forceinline__ void chain_walk(int s, int P, int pw, int md, int w, int n_chain,
                                           const double* base, double rlF, double rlB,
                                           double rlW, double sp, double hopf, double hopb,
                                           int cap, int mmax, double& fin, double& ssum,
                                           bool& over, bool& hung) {
  const bool unit = sp == 1.0;  // x / 1.0 == x exactly: skip the division
  const int lim = 2 * md - w;   // end of the steady F/B pairs
  int k = 0, jf = 0, jb = 0, jw = 0, live = 0;
  double lastF = 0.0, lastB = 0.0;
  int lastFi = -1, lastBi = -1;
  bool pending = n_chain > 0;
  // every step retires >= 1 chunk of each unfinished pipeline (acyclic DAG)
  const int max_steps = (ZBH ? 3 : 2) * mmax * P + 2;
  int steps = 0;
  while (__any_sync(0xffffffffu, pending)) {
    if (++steps > max_steps) {  // defensive: never spin on a malformed input
      hung = hung || pending;
      break;
    }
    const double nF = __shfl_up_sync(0xffffffffu, lastF, 1, pw);
    const int nFi = __shfl_up_sync(0xffffffffu, lastFi, 1, pw);
    const double nB = __shfl_down_sync(0xffffffffu, lastB, 1, pw);
    const int nBi = __shfl_down_sync(0xffffffffu, lastBi, 1, pw);
    if (pending) {
      // kind at chain position k (pipeline.py:92-118): 0=F 1=B/BW 2=W
      int kind;
      if (k < w) {
        kind = 0;
      } else if (k < lim) {
        kind = (k - w) & 1;
      } else if (!ZBH) {
        kind = 1;
      } else if (k < 2 * md + w) {
        kind = ((k - lim) & 1) ? 2 : 1;
      } else {
        kind = 2;
      }
      const int j = kind == 0 ? jf : (kind == 1 ? jb : jw);
      bool ready = true;
      double dep = 0.0;
      if (kind == 0 && s > 0) {
        ready = nFi == j;
        if (nFi > j) hung = true;  // lead bound violated: never guess
        dep = __dadd_rn(nF, hopf);
      } else if (kind == 1 && s < P - 1) {
        ready = nBi == j;
        if (nBi > j) hung = true;
        dep = __dadd_rn(nB, hopb);
      }
      if (hung) {
        pending = false;
      } else if (ready) {
        double c = __dmul_rn(kind == 0 ? rlF : (kind == 1 ? rlB : rlW), base[j]);
        if (!unit) c = div_slow(c, sp);
        fin = __dadd_rn(fmax(fin, dep), c);
        ssum = __dadd_rn(ssum, c);
        if (kind == 0) {
          lastF = fin;
          lastFi = jf++;
          if (cap > 0 && ++live > cap) over = true;
        } else if (kind == 1) {
          lastB = fin;
          lastBi = jb++;
          --live;
        } else {
          ++jw;
        }
        ++k;
        pending = k < n_chain;
      }
    }
  }
}

}  // namespace rh
