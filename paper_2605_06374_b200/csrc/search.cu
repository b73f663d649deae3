// Scheduler re-plan search (rh_search_*): DESIGN.md §5.
//
// Candidate space (index order defines the (score, index) tie-break):
//   layouts (T, D, P), T a power of two dividing devices_per_node, ordered by
//   T, then P, then D; a layout is enumerated when D*P TP blocks of T
//   executable devices exist, T*D*P >= min_utilization * executable and
//   D <= min(max_dp, M), P <= min(max_pp, L / min_layers)
//   x partition variants  v: 0 even split, 1 repartition_layers(stage
//     speeds) (scheduler.py:146-207), 2.. one layer moved src->dst from it
//   x count variants      u: 0 even split (cluster.py:318-321), 1
//     proportional_split(M, replica speeds) (policies.py:138-162), 2.. one
//     micro-batch moved src->dst from it
// Placement of a layout: every node's executable devices sorted by (speed
// desc, id) form blocks of T (the fastest-k rule of select_tp_subgroup,
// scheduler.py:114-137); the D*P fastest blocks (ties: node, position) are
// taken in node order and assigned replica-major, which is build_cluster's
// layout (cluster.py:175-208) on a healthy cluster.
//
// GPU work: one warp per layout prepares group speeds/nodes, hop weights,
// all-reduce ring bandwidths, repartition and proportional split
// (prep_kernel); one thread per (layout, partition variant, range case,
// replica) walks that replica pipeline's op list (pipe_kernel, the replica
// table); one thread per candidate combines the table exactly, adds the
// amortised reconfiguration surcharge and keeps a lexicographic (score,
// index) min (combine_kernel, minloc_kernel).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <limits>
#include <mutex>
#include <utility>
#include <vector>

#include <math_constants.h>

#include "common.cuh"
#include "wavefront.cuh"

struct rh_search {
  rh_search_desc d{};
  int n_nodes = 0;
  // host copies
  std::vector<double> speed;
  std::vector<int32_t> link_nodes;
  std::vector<double> link_factor;
  std::vector<int32_t> cur_groups, cur_partition;
  // prep results read back once (rh_search_decode is then host-only)
  std::vector<int32_t> h_gblk, h_repart, h_pstart;
  std::mutex host_mu;       // guards the lazy fetch of the three above
  bool host_ready = false;
  // layouts
  std::vector<int32_t> lT, lD, lP, lgoff, lpoff, ldoff, lboff, lnb;
  std::vector<long long> lbase, lnv, lnu, lpair, lrt;
  int64_t total = 0, n_pairs = 0, n_rt = 0;
  // blocks (concatenated over the distinct T values)
  std::vector<int32_t> blk_node, blk_rank, blk_members, blk_moff;
  std::vector<double> blk_speed;
  // device memory (one allocation)
  void* dmem = nullptr;
  size_t dbytes = 0;
  cudaStream_t last_stream = nullptr;  // stream of the latest create / eval
  // recorded after the latest create / eval: a later eval on another stream
  // waits for it (the task list and block results are per search)
  cudaEvent_t done_ev = nullptr;
  int div_safe = 0;  // see SearchArgs::div_safe
  bool div_dens = true;            // divisor range part of div_safe
  double div_r_lo = 0.0, div_r_hi = 0.0;  // (ratio * L) range
  bool workload_ready = false;     // quad loads uploaded and base costs built
  struct Dev {
    int32_t *lT, *lD, *lP, *lgoff, *lpoff, *ldoff, *lboff, *lnb;
    long long *lbase, *lnv, *lnu, *lpair, *lrt;
    double* rtab;   // replica table [sum over layouts nv*8*D]
    double* pinfo;  // per (layout, v): all-reduce cost (-1: none), surcharge (inf: infeasible)
    void* tasks;    // PipeTask[n_layouts]
    int32_t *blk_node, *blk_rank, *blk_members, *blk_moff;
    double* blk_speed;
    int32_t *gblk, *gnode;
    double *gspeed, *ghop;
    // per-group tables of the pipe kernel, TRANSPOSED to [s][d] so the lanes
    // of a warp (consecutive replicas) read consecutive addresses
    double *tspeed, *tinv, *thop;
    double *ring, *sspeed;
    int32_t* repart;
    double* rspeed;
    int32_t* pstart;
    int32_t* same;
    double* base;
    int64_t* quad;
    int32_t *link_nodes, *cur_groups, *cur_partition;
    double* link_factor;
    double* blk_best;
    long long* blk_idx;
    double* rl;  // [n_pairs][3][32] ratio * layers (rl_kernel)
    // op lists of the pipe kernel (separate pooled allocation)
    const uint32_t* ops;
    const int32_t *tab_off, *tab_cnt, *tab_peak;  // [33][M+2]
  } dv{};
  void* dops = nullptr;
  int eval_blocks = 0;
  size_t n_groups = 0, n_stage = 0, n_rep = 0;
};

namespace rh {

constexpr int kEvalThreads = 256;

struct SearchArgs {
  rh_cost_model m;
  int sched, N, M, L, min_layers, cap, has_comm, p2p_opt, n_layouts, n_links;
  double intra, inter, nbytes, lb, worst_inter, rebuild_s;
  int amort;
  int cur_T, cur_D, cur_P, T0;
  double r_bw;     // ratio_b + ratio_w (1F1B's fused BW chunk)
  int div_safe;    // every chunk's (numerator, speed) is in div_fast's exact range
  int tab_stride;  // op-list index: slot = P * tab_stride + md
  rh_search::Dev v;
};

// comm.py:32-36 — inter-node bandwidth of a node pair
__device__ __forceinline__ double link_inter(const SearchArgs& a, int x, int y) {
  const int lo = min(x, y), hi = max(x, y);
  double f = 1.0;
  for (int q = 0; q < a.n_links; ++q)
    if (a.v.link_nodes[2 * q] == lo && a.v.link_nodes[2 * q + 1] == hi) {
      f = a.v.link_factor[q];
      break;
    }
  return __dmul_rn(a.inter, f);
}

// edge_cost_fn (pipeline.py:336-353) between two T-wide groups
__device__ __forceinline__ double hop_cost(const SearchArgs& a, int na, int nb, int T) {
  if (!a.has_comm) return 0.0;
  if (na == nb) return __ddiv_rn(a.nbytes, a.intra);
  const double inter = link_inter(a, na, nb);
  if (!a.p2p_opt) {  // comm.py:73-75
    const double cross = __dmul_rn((double)T, a.nbytes);
    return __ddiv_rn(cross, inter);
  }
  const double gather = __ddiv_rn(__dmul_rn(a.nbytes, (double)(T - 1)), __dmul_rn((double)T, a.intra));
  return __dadd_rn(__ddiv_rn(a.nbytes, inter), gather);  // comm.py:76-78
}

// repartition_layers (scheduler.py:146-207), executed by a whole warp
// (n <= 32 stages, lane i owns stage i).  The largest-remainder split and
// the min_layers fix-up are tiny and run on lane 0; the greedy improvement
// loop is lane-parallel: lane src scans every dst.  A move changes only two
// stages, so its stage max is max(top value among the other stages,
// (lay[src]-1)/sp[src], (lay[dst]+1)/sp[dst]) -- the same set of quotients
// the reference maximises, hence the same double.  The reference's scan
// order (src outer, dst inner, strict <) is reproduced by a lexicographic
// (c, src, dst) warp argmin.
__device__ void repartition_warp(const double* sp_in, int n, int L, int ml, int32_t* out) {
  const int lane = threadIdx.x & 31;
  const unsigned full = 0xffffffffu;
  if (lane == 0) {
    double tot = 0.0;
    for (int i = 0; i < n; ++i) tot = __dadd_rn(tot, sp_in[i]);
    double frac[32];
    int lay[32];
    int sum = 0;
    for (int i = 0; i < n; ++i) {
      const double share = __ddiv_rn(__dmul_rn((double)L, sp_in[i]), tot);
      lay[i] = (int)floor(share);
      frac[i] = __dsub_rn(share, (double)lay[i]);
      sum += lay[i];
    }
    // largest remainder, ties to the earlier stage
    unsigned used = 0u;
    for (int r = 0; r < L - sum; ++r) {
      int bi = -1;
      for (int i = 0; i < n; ++i)
        if (!(used >> i & 1u) && (bi < 0 || frac[i] > frac[bi])) bi = i;
      used |= 1u << bi;
      lay[bi] += 1;
    }
    // starved stages up to the floor, taking from the largest (ties: lowest)
    for (;;) {
      int rec = -1;
      for (int i = 0; i < n; ++i)
        if (lay[i] < ml) {
          rec = i;
          break;
        }
      if (rec < 0) break;
      int don = -1;
      for (int i = 0; i < n; ++i)
        if (lay[i] > ml && (don < 0 || lay[i] > lay[don])) don = i;
      if (don < 0) break;
      lay[don] -= 1;
      lay[rec] += 1;
    }
    for (int i = 0; i < n; ++i) out[i] = lay[i];
  }
  __syncwarp();
  const bool mine = lane < n;
  int lay = mine ? out[lane] : 0;
  const double sp = mine ? sp_in[lane] : 1.0;
  const double min_gain = __ddiv_rn(1.0, __dmul_rn(2.0, (double)L));
  const double NEG = -CUDART_INF;
  for (;;) {
    const double t = mine ? __ddiv_rn((double)lay, sp) : NEG;
    const double dec = mine ? __ddiv_rn((double)(lay - 1), sp) : NEG;
    const double inc = mine ? __ddiv_rn((double)(lay + 1), sp) : NEG;
    // top three quotients (distinct stages, ties in any order)
    double v1 = t;
    for (int o = 16; o > 0; o >>= 1) v1 = fmax(v1, __shfl_xor_sync(full, v1, o));
    const int i1 = __ffs(__ballot_sync(full, t == v1)) - 1;
    const double t2 = lane == i1 ? NEG : t;
    double v2 = t2;
    for (int o = 16; o > 0; o >>= 1) v2 = fmax(v2, __shfl_xor_sync(full, v2, o));
    const int i2 = __ffs(__ballot_sync(full, t2 == v2 && lane != i1)) - 1;
    const double t3 = (lane == i1 || lane == i2) ? NEG : t;
    double v3 = t3;
    for (int o = 16; o > 0; o >>= 1) v3 = fmax(v3, __shfl_xor_sync(full, v3, o));
    const int i3 = __ffs(__ballot_sync(full, t3 == v3 && lane != i1 && lane != i2)) - 1;
    const double cur = v1;  // stage max of the current partition
    const double bar = __dmul_rn(cur, __dsub_rn(1.0, min_gain));
    // lane = src: the first dst (ascending) with the smallest c < bar
    double best = CUDART_INF;
    int bd = -1;
    const bool can = mine && lay > ml;
    for (int dst = 0; dst < n; ++dst) {
      const double inc_d = __shfl_sync(full, inc, dst);
      if (!can || dst == lane) continue;
      const double rest = (i1 != lane && i1 != dst) ? v1 : (i2 != lane && i2 != dst) ? v2
                                                        : (i3 >= 0 ? v3 : NEG);
      double c = rest > dec ? rest : dec;
      c = c > inc_d ? c : inc_d;
      if (c < bar && (bd < 0 || c < best)) {
        best = c;
        bd = dst;
      }
    }
    // lexicographic (c, src) argmin over lanes: ties keep the smaller src
    double wb = bd >= 0 ? best : CUDART_INF;
    int ws = bd >= 0 ? lane : 64;
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(full, wb, o);
      const int os = __shfl_xor_sync(full, ws, o);
      if (ob < wb || (ob == wb && os < ws)) {
        wb = ob;
        ws = os;
      }
    }
    if (ws == 64) break;  // no improving move
    const int wd = __shfl_sync(full, bd, ws);
    if (lane == ws) lay -= 1;
    if (lane == wd) lay += 1;
  }
  if (mine) out[lane] = lay;
  __syncwarp();
}

// proportional_split (policies.py:151-162) -> prefix starts[n+1]
__device__ void proportional_dev(int total, const double* w, int n, int32_t* start) {
  double wsum = 0.0;
  for (int i = 0; i < n; ++i) wsum = __dadd_rn(wsum, w[i]);
  int cnt[64];
  double frac[64];
  bool used[64];
  int sum = 0;
  for (int i = 0; i < n; ++i) {
    const double share = __ddiv_rn(__dmul_rn((double)total, w[i]), wsum);
    cnt[i] = (int)share;  // int() truncation, share >= 0
    frac[i] = __dsub_rn(share, (double)cnt[i]);
    sum += cnt[i];
    used[i] = false;
  }
  for (int r = 0; r < total - sum; ++r) {
    int bi = -1;
    for (int i = 0; i < n; ++i)
      if (!used[i] && (bi < 0 || frac[i] > frac[bi])) bi = i;
    used[bi] = true;
    cnt[bi] += 1;
  }
  start[0] = 0;
  for (int i = 0; i < n; ++i) start[i + 1] = start[i] + cnt[i];
}

__global__ void base_kernel(SearchArgs a) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= a.M) return;
  a.v.base[j] = __dadd_rn(__dmul_rn(a.m.alpha, (double)a.N),
                          __dmul_rn(a.m.beta, (double)a.v.quad[j]));
}

// one warp per layout
__global__ void prep_kernel(SearchArgs a) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= a.n_layouts) return;
  const int T = a.v.lT[warp], D = a.v.lD[warp], P = a.v.lP[warp];
  const int K = D * P, goff = a.v.lgoff[warp], poff = a.v.lpoff[warp];
  const int doff = a.v.ldoff[warp], boff = a.v.lboff[warp], nb = a.v.lnb[warp];
  // placement: the K fastest blocks, kept in node order
  int taken = 0;
  for (int c0 = 0; c0 < nb; c0 += 32) {
    const int b = c0 + lane;
    const bool sel = b < nb && a.v.blk_rank[boff + b] < K;
    const unsigned m = __ballot_sync(0xffffffffu, sel);
    if (sel) {
      const int g = taken + __popc(m & ((1u << lane) - 1u));
      a.v.gblk[goff + g] = boff + b;
      // slowest * |group| / nominal_tp (cluster.py:155-169)
      const double gsp = __ddiv_rn(__dmul_rn(a.v.blk_speed[boff + b], (double)T),
                                   (double)a.T0);
      a.v.gspeed[goff + g] = gsp;
      a.v.gnode[goff + g] = a.v.blk_node[boff + b];
    }
    taken += __popc(m);
  }
  __syncwarp();
  // hop weights on stage boundaries (same in both directions: T == T);
  // transposed copies for the pipe kernel
  for (int g = lane; g < K; g += 32) {
    const int s = g % P, d = g / P;
    const double h = s < P - 1 ? hop_cost(a, a.v.gnode[goff + g], a.v.gnode[goff + g + 1], T)
                               : 0.0;
    a.v.ghop[goff + g] = h;
    a.v.thop[goff + s * D + d] = h;
    const double gsp = a.v.gspeed[goff + g];
    a.v.tspeed[goff + s * D + d] = gsp;
    a.v.tinv[goff + s * D + d] = recip_of(gsp);
  }
  // per stage: all-reduce ring bandwidth (comm.py:87-107), min speed
  for (int s = lane; s < P; s += 32) {
    bool same_node = true;
    const int n0 = a.v.gnode[goff + s];
    double mn = a.v.gspeed[goff + s];
    for (int d = 1; d < D; ++d) {
      same_node &= a.v.gnode[goff + d * P + s] == n0;
      mn = fmin(mn, a.v.gspeed[goff + d * P + s]);
    }
    double bw;
    if (same_node) {
      bw = a.intra;
    } else {
      bw = a.inter;
      for (int d = 0; d < D; ++d) {
        const int x = a.v.gnode[goff + d * P + s];
        const int y = a.v.gnode[goff + ((d + 1) % D) * P + s];
        if (x != y) bw = fmin(bw, link_inter(a, x, y));
      }
    }
    a.v.ring[poff + s] = bw;
    a.v.sspeed[poff + s] = mn;
  }
  // per replica: min speed over stages (_replica_speeds, policies.py:138-148)
  for (int d = lane; d < D; d += 32) {
    double mn = a.v.gspeed[goff + d * P];
    for (int s = 1; s < P; ++s) mn = fmin(mn, a.v.gspeed[goff + d * P + s]);
    a.v.rspeed[doff + d] = mn;
  }
  // same groups as the current plan?
  int same = a.cur_T == T && a.cur_D == D && a.cur_P == P;
  if (same) {
    for (int g = lane; g < K; g += 32) {
      const int b = a.v.gblk[goff + g];
      for (int t = 0; t < T; ++t)
        if (a.v.blk_members[a.v.blk_moff[b] + t] != a.v.cur_groups[g * T + t]) same = 0;
    }
    same = __all_sync(0xffffffffu, same);
  }
  __syncwarp();
  repartition_warp(a.v.sspeed + poff, P, a.L, a.min_layers, a.v.repart + poff);
  if (lane == 0) {
    a.v.same[warp] = same;
    proportional_dev(a.M, a.v.rspeed + doff, D, a.v.pstart + doff + warp);
  }
}

__device__ __forceinline__ bool lex_less(double a, long long ia, double b, long long ib) {
  return a < b || (a == b && ia < ib);
}

// ---- phase 1: replica pipeline table --------------------------------------
// For every (layout, partition variant v) in the evaluated range and every
// replica d, the makespan contribution of d's pipeline is computed for the 8
// micro-batch ranges that count variants can give it:
//   case 0 even split, 1 proportional, then proportional shifted by
//   (start, end) = 2 (0,-1)  3 (-1,-1)  4 (-1,0)  5 (0,+1)  6 (+1,+1)  7 (+1,0)
// (moving one micro-batch src->dst shifts every replica between them by one).
// Infeasible ranges / capacity overflow are stored as +inf.
//
// One THREAD per (layout, v, case, replica) pipeline.  It walks the
// replica's chunks in the order of the op list for (P, md) -- DAG level
// ascending, stage descending (wavefront.cuh closed forms), built on the
// host for the (P, md) pairs that can occur -- so every dependency is final
// when read (see pipeline.cu's small kernel for the argument) and no lane
// idles.  Per-stage state lives in shared memory laid out [field][stage]
// [thread] (conflict-free):  for 1F1B the finish of the last F and of the
// last BW -- the chain's own finish is their max, finishes being monotone
// along a chain -- and for ZBH also the chain finish (W feeds nothing).
__constant__ int kDs[8] = {0, 0, 0, -1, -1, 0, 1, 1};
__constant__ int kDe[8] = {0, 0, -1, -1, 0, 1, 1, 0};

struct PipeTask {
  int layout;
  int v_lo;
  long long pipe_base;  // first pipeline id of this task
  long long row_base;   // first (layout, v) row of this task (rl_kernel)
};

// op list entry: stage (bits 0-5) | kind << 6 (1 F, 2 B or BW, 3 W)
//                | dependency << 8 (0 none, 1 F of stage-1, 2 B of stage+1) | j << 10
enum : unsigned { kOpF = 1, kOpB = 2, kOpW = 3 };

// per (layout, v) pair: rl[kind-1][s] = ratio(kind) * L_s  (workload.py:88-98)
__global__ void rl_kernel(SearchArgs a, const PipeTask* tk, int n_tk, int P, long long n_rows) {
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n_rows * P) return;
  const long long row = g / P;
  const int s = (int)(g % P);
  int lo = 0, hi = n_tk - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (tk[mid].row_base <= row) lo = mid;
    else hi = mid - 1;
  }
  const int li = tk[lo].layout;
  const int vv = tk[lo].v_lo + (int)(row - tk[lo].row_base);
  const int32_t* rep = a.v.repart + a.v.lpoff[li];
  int psrc = -1, pdst = -1;
  if (vv >= 2) {
    const int m = vv - 2, r = m % (P - 1);
    psrc = m / (P - 1);
    pdst = r < psrc ? r : r + 1;
  }
  const int Ls = vv == 0 ? a.L / P + (s < a.L % P ? 1 : 0)
                         : rep[s] + (s == pdst ? 1 : 0) - (s == psrc ? 1 : 0);
  const double L = (double)Ls;
  double* out = a.v.rl + (a.v.lpair[li] + vv) * 3LL * 32;
  out[s] = __dmul_rn(a.m.ratio_f, L);
  out[32 + s] = __dmul_rn(a.sched == RH_SCHED_ZBH ? a.m.ratio_b : a.r_bw, L);
  out[64 + s] = __dmul_rn(a.m.ratio_w, L);
}

__device__ __forceinline__ int layer_of(const SearchArgs& a, const int32_t* rep, int P, int vv,
                                        int psrc, int pdst, int s) {
  return vv == 0 ? a.L / P + (s < a.L % P ? 1 : 0)
                 : rep[s] + (s == pdst ? 1 : 0) - (s == psrc ? 1 : 0);
}

constexpr int kPipeThreads = 128;

// One replica pipeline of the search, identified by its id g within a P
// group: its layout, partition variant, range case and replica, its
// micro-batch range, and whether it is evaluated at all.  With `info` set the
// caller also writes the per-(layout, v) all-reduce vertex and amortised
// reconfiguration surcharge.
struct PipeId {
  int li, D, vv, cs, d, goff, start, md;
  long long pair;
  bool feas_v, valid;
};

__device__ __forceinline__ PipeId pipe_id(const SearchArgs& a, const PipeTask* tk, int n_tk,
                                          int P, long long g, bool info) {
  int lo = 0, hi = n_tk - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (tk[mid].pipe_base <= g) lo = mid;
    else hi = mid - 1;
  }
  const int li = tk[lo].layout;
  const int D = a.v.lD[li];
  const long long local = g - tk[lo].pipe_base;
  const int vv = tk[lo].v_lo + (int)(local / (8 * D));
  const int rr = (int)(local % (8 * D));
  const int cs = rr / D, d = rr % D;
  const int goff = a.v.lgoff[li], poff = a.v.lpoff[li];
  const int32_t* rep = a.v.repart + poff;
  const int32_t* pst = a.v.pstart + a.v.ldoff[li] + li;
  int psrc = -1, pdst = -1;
  if (vv >= 2) {
    const int m = vv - 2, r = m % (P - 1);
    psrc = m / (P - 1);
    pdst = r < psrc ? r : r + 1;
  }
  const bool feas_v = !(psrc >= 0 && rep[psrc] - 1 < a.min_layers);
  const long long pair = a.v.lpair[li] + vv;
  if (info && cs == 0 && d == 0) {
    // per (layout, v): all-reduce vertex (pipeline.py:356-372) and the
    // amortised reconfiguration surcharge (scheduler.py:562-593)
    const bool has_ar = a.has_comm && D > 1;
    double ar = 0.0;
    if (has_ar)
      for (int q = 0; q < P; ++q) {
        const double nbytes = __dmul_rn((double)layer_of(a, rep, P, vv, psrc, pdst, q), a.lb);
        ar = fmax(ar, __ddiv_rn(__dmul_rn(__dmul_rn(2.0, nbytes), (double)(D - 1)),
                                __dmul_rn((double)D, a.v.ring[poff + q])));
      }
    const bool same_layout = a.v.same[li] != 0;
    const bool sameP = P == a.cur_P;
    bool changed = false;
    long long moved = 0;
    for (int q = 0; q < P && sameP; ++q) {
      const int lq = layer_of(a, rep, P, vv, psrc, pdst, q);
      const int old = a.v.cur_partition[q];
      if (lq != old) changed = true;
      if (lq > old) moved += lq - old;
    }
    double reshard = 0.0;
    if (!same_layout)
      for (int dd = 0; dd < D; ++dd)
        for (int q = 0; q < P; ++q)
          reshard = __dadd_rn(reshard,
                              __dmul_rn((double)layer_of(a, rep, P, vv, psrc, pdst, q), a.lb));
    double sur = 0.0;
    if (!same_layout || changed) {
      const double transfer = __ddiv_rn(__dadd_rn(__dmul_rn((double)moved, a.lb), reshard),
                                        a.worst_inter);
      sur = __ddiv_rn(__dadd_rn(a.rebuild_s, transfer), (double)max(1, a.amort));
    }
    a.v.pinfo[2 * pair] = has_ar ? ar : -1.0;  // -1: no all-reduce vertex
    a.v.pinfo[2 * pair + 1] = feas_v ? sur : CUDART_INF;
  }
  int start = 0, md = 0;
  bool valid = true;
  if (cs == 0) {
    const int base = a.M / D, extra = a.M % D;
    start = d * base + min(d, extra);
    md = base + (d < extra ? 1 : 0);
  } else {
    start = pst[d] + kDs[cs];
    md = pst[d + 1] + kDe[cs] - start;
    valid = start >= 0 && md >= 0 && start + md <= a.M;
  }
  PipeId id;
  id.li = li;
  id.D = D;
  id.vv = vv;
  id.cs = cs;
  id.d = d;
  id.goff = goff;
  id.start = start;
  id.md = md;
  id.pair = pair;
  id.feas_v = feas_v;
  id.valid = valid;
  return id;
}

template <int ZBH, bool SAFE>
__global__ void __launch_bounds__(kPipeThreads) pipe_kernel(SearchArgs a, const PipeTask* tk,
                                                           int n_tk, long long n_pipes, int P) {
  extern __shared__ double pipe_smem[];
  const int tid = threadIdx.x, nt = blockDim.x;
  for (long long g = (long long)blockIdx.x * nt + tid; g < n_pipes;
       g += (long long)gridDim.x * nt) {
    const PipeId id = pipe_id(a, tk, n_tk, P, g, true);
    const int li = id.li, D = id.D, vv = id.vv, cs = id.cs, d = id.d, goff = id.goff;
    const int start = id.start, md = id.md;
    const long long pair = id.pair;
    const bool feas_v = id.feas_v, valid = id.valid;
    double res = CUDART_INF;
    if (feas_v && valid) {
      const int slot = P * a.tab_stride + md;
      const int e0 = __ldg(a.v.tab_off + slot), ne = __ldg(a.v.tab_cnt + slot);
      const bool over = a.cap > 0 && __ldg(a.v.tab_peak + slot) > a.cap;
      // state index: ((field * P) + stage) * kPipeThreads + tid; fields 0 LF, 1 LB, 2 FN
      const int fB = P * kPipeThreads, fN = 2 * P * kPipeThreads;
      for (int q = 0; q < P; ++q) {
        pipe_smem[q * kPipeThreads + tid] = 0.0;
        pipe_smem[fB + q * kPipeThreads + tid] = 0.0;
        if (ZBH) pipe_smem[fN + q * kPipeThreads + tid] = 0.0;
      }
      const double* bs = a.v.base + start;
      // [s][d] tables: element (d, s) at s * D
      const double* sp_d = a.v.tspeed + goff + d;
      const double* inv_d = a.v.tinv + goff + d;
      const double* hop_d = a.v.thop + goff + d;
      const double* rlt = a.v.rl + pair * 3LL * 32 - 32;  // indexed by kind * 32 + s
      const uint32_t* opp = a.v.ops + e0;
      // software pipeline: op codes two ahead, their global operands one ahead,
      // so only the shared-memory state chain is serial.  The loop body is
      // branch-free: the prefetch indices clamp to the last op (a harmless
      // re-fetch), an op without a data predecessor reads a valid dummy slot
      // and selects 0, and the division is always the exact hoisted-reciprocal
      // form (unit speeds: inv == 1 gives c unchanged) when the host proved the
      // search's operand ranges safe.
      struct Operands {
        unsigned op;
        double rl, b, sp, inv, hop;
      };
      auto fetch = [&](unsigned op) {
        Operands o;
        o.op = op;
        const int st = op & 63u;
        const unsigned kind = (op >> 6) & 3u, dk = (op >> 8) & 3u;
        const int so = st * D;  // [s][d] tables: element (d, s) at s * D
        o.rl = __ldg(rlt + (int)(kind * 32 + st));
        o.b = __ldg(bs + (int)(op >> 10));
        o.sp = __ldg(sp_d + so);
        o.inv = __ldg(inv_d + so);
        o.hop = __ldg(hop_d + (dk == 1 ? so - D : so));
        return o;
      };
      const int last = ne - 1;
      unsigned op2 = 0u;
      Operands nx{};
      if (ne > 0) {  // real op codes only (kind >= 1): every fetch stays in its tables
        op2 = __ldg(opp + min(1, last));
        nx = fetch(__ldg(opp));
      }
      for (int e = 0; e < ne; ++e) {
        const Operands o = nx;
        const unsigned op3 = __ldg(opp + min(e + 2, last));
        nx = fetch(op2);
        op2 = op3;
        const int st = o.op & 63u;
        const unsigned kind = (o.op >> 6) & 3u, dk = (o.op >> 8) & 3u;
        double c = __dmul_rn(o.rl, o.b);
        if (SAFE) c = div_fast(c, o.sp, o.inv);
        else if (o.sp != 1.0) c = div_slow(c, o.sp);
        const int self = st * kPipeThreads + tid;
        // F: last F of stage-1 (+ hop s-1 -> s); B: last B of stage+1 (+ hop s)
        const int src = dk == 1 ? self - kPipeThreads : (dk ? fB + self + kPipeThreads : self);
        const double dep = dk ? __dadd_rn(pipe_smem[src], o.hop) : 0.0;
        double fin;
        if (ZBH) {
          fin = pipe_smem[fN + self];
        } else {
          const double x = pipe_smem[self], y = pipe_smem[fB + self];
          fin = x > y ? x : y;
        }
        const double nf = __dadd_rn(fin > dep ? fin : dep, c);
        if (ZBH) {
          pipe_smem[fN + self] = nf;
          if (kind != kOpW) pipe_smem[(kind == kOpF ? 0 : fB) + self] = nf;
        } else {
          pipe_smem[(kind == kOpF ? 0 : fB) + self] = nf;  // 1F1B: F or BW only
        }
      }
      double gm = 0.0;
      for (int q = 0; q < P; ++q) {
        const int self = q * kPipeThreads + tid;
        const double f = ZBH ? pipe_smem[fN + self] : fmax(pipe_smem[self], pipe_smem[fB + self]);
        gm = fmax(gm, f);
      }
      res = over ? CUDART_INF : gm;
    }
    a.v.rtab[a.v.lrt[li] + (long long)vv * 8 * D + cs * D + d] = res;
  }
}

// ---- phase 1 for 1F1B, P <= 32: register-resident replica walks ----------
// One thread per replica pipeline, as in pipe_kernel, but the chain state
// (each stage's last finish) lives in registers and the
// chunks are visited in the loop-form topological order of the Detector's
// pass_wide_kernel (pass_wide.cu): a warm-up triangle (F_j on stages
// ascending) and a main loop of (B_i, F_{P-s+i}) pairs on stages descending,
// with the stage index unrolled at compile time.  Per chunk: one base-cost
// load, a broadcast ratio * layers load, a coalesced hop load ([s][d] tables),
// and the division only on stages some replica of the warp runs slow.  The
// per-stage constants are reloaded per use (ld.global.nc through asm
// volatile) instead of pinning 4P registers.
__device__ __forceinline__ double ldg_nc(const double* p) {
  double v;
  asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

template <int P, bool SAFE>
struct SearchWalk {
  const double* bs;   // base costs of the replica's first micro-batch on
  const double* rl;   // [rlF: 32][rlB: 32] of the (layout, partition) pair
  const double* sp;   // [s][d] tables at this replica: element s at s * D
  const double* inv;
  const double* hop;  // hop s -> s+1 at s * D
  int D;
  unsigned slow;      // warp-uniform: bit s = some replica of the warp runs stage s slow
  // A stage's last F finish is never kept apart from its chain finish: when
  // F(s+1) reads it, that F is stage s's latest chunk (the warm-up walks
  // stages ascending, the main loop descending; pass_wide.cu).  With P
  // doubles of chain state instead of 2P, C5 eval 4.62 -> 3.88 ms.
  double fin[P];

  template <int S>
  __device__ __forceinline__ double cost(double rl_, double b) const {
    const double x = __dmul_rn(rl_, b);
    if (slow & (1u << S)) {  // warp-uniform branch; x / 1.0 == x otherwise
      const double v = __ldg(sp + S * D);
      if (SAFE) return div_fast(x, v, __ldg(inv + S * D));
      return v != 1.0 ? div_slow(x, v) : x;
    }
    return x;
  }
  // NODEP: no data dependency (dep == 0.0): start = chain finish (a finish
  // is a sum of non-negative costs from +0.0; see walks.cuh chunk())
  template <int S, bool NODEP = false>
  __device__ __forceinline__ double step(double c, double dep) {
    const double st = (NODEP || fin[S] > dep) ? fin[S] : dep;
    fin[S] = __dadd_rn(st, c);
    return fin[S];
  }
  template <int S>
  __device__ __forceinline__ void tri(int j, int m, double bj) {
    if (j <= P - 1 - S && j < m) {
      const double dep = S > 0 ? __dadd_rn(fin[S > 0 ? S - 1 : 0], ldg_nc(hop + (S - 1) * D)) : 0.0;
      step<S, S == 0>(cost<S>(ldg_nc(rl + S), bj), dep);
    }
  }
  template <int S>
  __device__ __forceinline__ void pair(int i, int m, double bi, double& nB) {
    const double depB = S < P - 1 ? __dadd_rn(nB, ldg_nc(hop + S * D)) : 0.0;
    nB = step<S, S == P - 1>(cost<S>(ldg_nc(rl + 32 + S), bi), depB);
    if (i < m - P + S) {
      const double bF = __ldg(bs + (P - S + i));
      const double dep = S > 0 ? __dadd_rn(fin[S > 0 ? S - 1 : 0], ldg_nc(hop + (S - 1) * D)) : 0.0;
      step<S, S == 0>(cost<S>(ldg_nc(rl + S), bF), dep);
    }
  }
  template <int... I>
  __device__ __forceinline__ void tri_all(int j, int m, double bj, std::integer_sequence<int, I...>) {
    (tri<I>(j, m, bj), ...);
  }
  template <int... I>
  __device__ __forceinline__ void pair_all(int i, int m, double bi, std::integer_sequence<int, I...>) {
    double nB = 0.0;
    (pair<P - 1 - I>(i, m, bi, nB), ...);
  }
  __device__ __forceinline__ double walk(int m) {
#pragma unroll
    for (int s = 0; s < P; ++s) fin[s] = 0.0;
#pragma unroll 1
    for (int j = 0; j < P; ++j)
      tri_all(j, m, __ldg(bs + (j < m ? j : 0)), std::make_integer_sequence<int, P>());
    // (two steps at once, skewed as in pass_wide.cu: spills at these register
    // budgets, C5 eval 3.88 -> 6.19 ms)
#pragma unroll 1
    for (int i = 0; i < m; ++i)
      pair_all(i, m, __ldg(bs + i), std::make_integer_sequence<int, P>());
    double g = 0.0;
#pragma unroll
    for (int s = 0; s < P; ++s) g = fin[s] > g ? fin[s] : g;
    return g;
  }
};

// (one more CTA per SM at every length, spending the registers the last-F
// array freed: spills, C5 eval 3.88 -> 4.34 ms)
constexpr int search_reg_min_blocks(int P) { return P <= 12 ? 4 : (P <= 24 ? 3 : 2); }

template <int P, bool SAFE>
__global__ void __launch_bounds__(kPipeThreads, search_reg_min_blocks(P))
    pipe_reg_kernel(SearchArgs a, const PipeTask* tk, int n_tk, long long n_pipes) {
  const int nt = blockDim.x;
  // every lane of a warp runs the same trip count (the slow mask is a warp vote)
  const long long stride = (long long)gridDim.x * nt;
  const long long g0 = (long long)blockIdx.x * nt + threadIdx.x;
  const long long trips = (n_pipes + stride - 1 - ((long long)blockIdx.x * nt)) / stride + 1;
  for (long long t = 0, g = g0; t < trips; ++t, g += stride) {
    const bool live = g < n_pipes;
    PipeId id{};
    bool run = false;
    const double *sp_d = nullptr, *inv_d = nullptr, *hop_d = nullptr;
    unsigned slow = 0;
    int md = 0;
    bool over = false;
    if (live) {
      id = pipe_id(a, tk, n_tk, P, g, true);
      md = id.md;
      run = id.feas_v && id.valid && md > 0;
      sp_d = a.v.tspeed + id.goff + id.d;
      inv_d = a.v.tinv + id.goff + id.d;
      hop_d = a.v.thop + id.goff + id.d;
      // 1F1B activation peak (the op lists' in-flight count): stage 0 holds
      // min(P, md) forward chunks before its first backward
      if (id.feas_v && id.valid) over = a.cap > 0 && min(P, md) > a.cap;
      if (run)
#pragma unroll 4
        for (int s = 0; s < P; ++s)
          if (__ldg(sp_d + s * id.D) != 1.0) slow |= 1u << s;
    }
    const unsigned wslow = __reduce_or_sync(0xffffffffu, slow);
    if (!live) continue;
    double res = CUDART_INF;
    if (id.feas_v && id.valid) {
      double gm = 0.0;
      if (run) {
        SearchWalk<P, SAFE> w{a.v.base + id.start, a.v.rl + id.pair * 3LL * 32, sp_d, inv_d,
                              hop_d, id.D, wslow, {}};
        gm = w.walk(md);
      }
      res = over ? CUDART_INF : gm;
    }
    a.v.rtab[a.v.lrt[id.li] + (long long)id.vv * 8 * id.D + id.cs * id.D + id.d] = res;
  }
}

template <bool SAFE>
static void* pipe_reg_kernel_for(int P) {
  switch (P) {
#define RH_REG_CASE(n) \
  case n:              \
    return (void*)pipe_reg_kernel<n, SAFE>;
    RH_REG_CASE(1) RH_REG_CASE(2) RH_REG_CASE(3) RH_REG_CASE(4) RH_REG_CASE(5) RH_REG_CASE(6)
    RH_REG_CASE(7) RH_REG_CASE(8) RH_REG_CASE(9) RH_REG_CASE(10) RH_REG_CASE(11)
    RH_REG_CASE(12) RH_REG_CASE(13) RH_REG_CASE(14) RH_REG_CASE(15) RH_REG_CASE(16)
    RH_REG_CASE(17) RH_REG_CASE(18) RH_REG_CASE(19) RH_REG_CASE(20) RH_REG_CASE(21)
    RH_REG_CASE(22) RH_REG_CASE(23) RH_REG_CASE(24) RH_REG_CASE(25) RH_REG_CASE(26)
    RH_REG_CASE(27) RH_REG_CASE(28) RH_REG_CASE(29) RH_REG_CASE(30) RH_REG_CASE(31)
    RH_REG_CASE(32)
#undef RH_REG_CASE
    default: return nullptr;
  }
}

// ---- phase 2: every candidate from the table (thread per candidate) -------
__global__ void __launch_bounds__(kEvalThreads) combine_kernel(SearchArgs a, long long begin,
                                                              long long end, long long sbegin,
                                                              double* scores, double* out_best,
                                                              long long* out_idx) {
  __shared__ double s_best[kEvalThreads / 32];
  __shared__ long long s_idx[kEvalThreads / 32];
  double best = CUDART_INF;
  long long best_i = -1;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long idx = begin + (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < end;
       idx += stride) {
    int lo = 0, hi = a.n_layouts - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (a.v.lbase[mid] <= idx) lo = mid;
      else hi = mid - 1;
    }
    const int li = lo;
    const int D = a.v.lD[li];
    const long long local = idx - a.v.lbase[li];
    const long long nu = a.v.lnu[li];
    const int vv = (int)(local / nu), uu = (int)(local % nu);
    const long long pair = a.v.lpair[li] + vv;
    const double ar = a.v.pinfo[2 * pair], sur = a.v.pinfo[2 * pair + 1];
    const double* Rp = a.v.rtab + a.v.lrt[li] + (long long)vv * 8 * D;
    double ms = 0.0;
    bool feasible = sur < CUDART_INF;
    if (uu <= 1) {
      for (int d = 0; d < D; ++d) ms = fmax(ms, Rp[uu * D + d]);
    } else {
      const int m = uu - 2, r = m % (D - 1);
      const int src = m / (D - 1), dst = r < src ? r : r + 1;
      const int32_t* pst = a.v.pstart + a.v.ldoff[li] + li;
      if (pst[src + 1] - pst[src] == 0) feasible = false;
      for (int d = 0; d < D && feasible; ++d) {
        int cs = 1;
        if (src < dst) cs = d == src ? 2 : (d == dst ? 4 : ((d > src && d < dst) ? 3 : 1));
        else cs = d == dst ? 5 : (d == src ? 7 : ((d > dst && d < src) ? 6 : 1));
        ms = fmax(ms, Rp[cs * D + d]);
      }
    }
    double score = CUDART_INF;
    if (feasible && ms < CUDART_INF) {
      // max_d(g_d + AR) == max_d(g_d) + AR: rounding is monotone
      if (ar >= 0.0) ms = __dadd_rn(ms, ar);
      score = __dadd_rn(ms, sur);
    }
    if (scores) scores[idx - sbegin] = score;
    if (lex_less(score, idx, best, best_i)) {
      best = score;
      best_i = idx;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const long long oi = __shfl_xor_sync(0xffffffffu, best_i, o);
    if (oi >= 0 && (best_i < 0 || lex_less(ob, oi, best, best_i))) {
      best = ob;
      best_i = oi;
    }
  }
  if ((threadIdx.x & 31) == 0) {
    s_best[threadIdx.x >> 5] = best;
    s_idx[threadIdx.x >> 5] = best_i;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = s_best[0];
    long long bi = s_idx[0];
    for (int q = 1; q < (int)(blockDim.x >> 5); ++q)
      if (s_idx[q] >= 0 && (bi < 0 || lex_less(s_best[q], s_idx[q], b, bi))) {
        b = s_best[q];
        bi = s_idx[q];
      }
    out_best[blockIdx.x] = b;
    out_idx[blockIdx.x] = bi;
  }
}

// ---- phase 2, one CTA per (layout, partition) pair: O(1) per candidate ----
// A count variant u >= 2 moves one micro-batch src -> dst; the replicas
// between them shift by one position.  Its makespan is the max of the
// case-1 row outside [min, max], the two moved replicas' cases and the
// case-3 (src < dst) or case-6 (dst < src) row strictly inside: prefix /
// suffix maxima of the case-1 row and a sparse table (range max) of rows 3
// and 6, built once per pair in shared memory, make every candidate O(1)
// instead of O(D) (max is exact and order-free, so the value is unchanged).
constexpr int kComb2Threads = 256;
constexpr int kComb2MaxD = 64;
constexpr int kComb2Levels = 7;  // 2^6 = 64

__global__ void __launch_bounds__(kComb2Threads) combine2_kernel(SearchArgs a, int li,
                                                                long long begin, long long end,
                                                                long long sbegin, int v_lo,
                                                                double* scores, double* out_best,
                                                                long long* out_idx) {
  __shared__ double rows[8][kComb2MaxD];
  __shared__ double pre1[kComb2MaxD + 1], suf1[kComb2MaxD + 1];
  __shared__ double sp3[kComb2Levels][kComb2MaxD], sp6[kComb2Levels][kComb2MaxD];
  __shared__ double s_best[kComb2Threads / 32];
  __shared__ long long s_idx[kComb2Threads / 32];
  const int vv = v_lo + blockIdx.x;
  const int D = a.v.lD[li];
  const long long nu = a.v.lnu[li];
  const long long pbase = a.v.lbase[li] + (long long)vv * nu;
  const long long u_lo = max(0LL, begin - pbase), u_hi = min(nu, end - pbase);
  const long long pair = a.v.lpair[li] + vv;
  const double ar = a.v.pinfo[2 * pair], sur = a.v.pinfo[2 * pair + 1];
  const double* Rp = a.v.rtab + a.v.lrt[li] + (long long)vv * 8 * D;
  for (int k = threadIdx.x; k < 8 * D; k += blockDim.x) rows[k / D][k % D] = Rp[k];
  __syncthreads();
  if (threadIdx.x == 0) {  // D <= 64: one thread each
    double m = 0.0;
    pre1[0] = 0.0;
    for (int d = 0; d < D; ++d) pre1[d + 1] = m = fmax(m, rows[1][d]);
    m = 0.0;
    suf1[D] = 0.0;
    for (int d = D - 1; d >= 0; --d) suf1[d] = m = fmax(m, rows[1][d]);
  }
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    sp3[0][d] = rows[3][d];
    sp6[0][d] = rows[6][d];
  }
  __syncthreads();
  for (int k = 1; k < kComb2Levels && (1 << k) <= D; ++k) {
    for (int d = threadIdx.x; d + (1 << k) <= D; d += blockDim.x) {
      sp3[k][d] = fmax(sp3[k - 1][d], sp3[k - 1][d + (1 << (k - 1))]);
      sp6[k][d] = fmax(sp6[k - 1][d], sp6[k - 1][d + (1 << (k - 1))]);
    }
    __syncthreads();
  }
  const int32_t* pst = a.v.pstart + a.v.ldoff[li] + li;
  double best = CUDART_INF;
  long long best_i = -1;
  for (long long u = u_lo + threadIdx.x; u < u_hi; u += blockDim.x) {
    double ms = 0.0;
    bool feasible = sur < CUDART_INF;
    if (u <= 1) {
      for (int d = 0; d < D; ++d) ms = fmax(ms, rows[u][d]);
    } else {
      const int m = (int)(u - 2), r = m % (D - 1);
      const int src = m / (D - 1), dst = r < src ? r : r + 1;
      if (pst[src + 1] - pst[src] == 0) feasible = false;
      const int lo = min(src, dst), hi = max(src, dst);
      ms = fmax(pre1[lo], suf1[hi + 1]);  // case-1 replicas outside [lo, hi]
      if (src < dst) ms = fmax(ms, fmax(rows[2][src], rows[4][dst]));
      else ms = fmax(ms, fmax(rows[5][dst], rows[7][src]));
      if (hi - lo >= 2) {  // strictly inside: case 3 (src < dst) or 6
        const int l = lo + 1, len = hi - lo - 1;
        const int k = 31 - __clz(len);
        const double(*sp)[kComb2MaxD] = src < dst ? sp3 : sp6;
        ms = fmax(ms, fmax(sp[k][l], sp[k][hi - (1 << k)]));
      }
    }
    double score = CUDART_INF;
    if (feasible && ms < CUDART_INF) {
      if (ar >= 0.0) ms = __dadd_rn(ms, ar);  // max_d(g_d + AR) == max_d(g_d) + AR
      score = __dadd_rn(ms, sur);
    }
    const long long idx = pbase + u;
    if (scores) scores[idx - sbegin] = score;
    if (lex_less(score, idx, best, best_i)) {
      best = score;
      best_i = idx;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const long long oi = __shfl_xor_sync(0xffffffffu, best_i, o);
    if (oi >= 0 && (best_i < 0 || lex_less(ob, oi, best, best_i))) {
      best = ob;
      best_i = oi;
    }
  }
  if ((threadIdx.x & 31) == 0) {
    s_best[threadIdx.x >> 5] = best;
    s_idx[threadIdx.x >> 5] = best_i;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = s_best[0];
    long long bi = s_idx[0];
    for (int q = 1; q < (int)(blockDim.x >> 5); ++q)
      if (s_idx[q] >= 0 && (bi < 0 || lex_less(s_best[q], s_idx[q], b, bi))) {
        b = s_best[q];
        bi = s_idx[q];
      }
    out_best[blockIdx.x] = b;
    out_idx[blockIdx.x] = bi;
  }
}

__global__ void minloc_kernel(const double* sc, const long long* ix, int n, double* out_s,
                              int64_t* out_i) {
  __shared__ double sb[32];
  __shared__ long long si[32];
  double b = CUDART_INF;
  long long bi = -1;
  for (int q = threadIdx.x; q < n; q += blockDim.x)
    if (ix[q] >= 0 && (bi < 0 || lex_less(sc[q], ix[q], b, bi))) {
      b = sc[q];
      bi = ix[q];
    }
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, b, o);
    const long long oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (oi >= 0 && (bi < 0 || lex_less(ob, oi, b, bi))) {
      b = ob;
      bi = oi;
    }
  }
  if ((threadIdx.x & 31) == 0) {
    sb[threadIdx.x >> 5] = b;
    si[threadIdx.x >> 5] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    b = sb[0];
    bi = si[0];
    for (int q = 1; q < (int)(blockDim.x >> 5); ++q)
      if (si[q] >= 0 && (bi < 0 || lex_less(sb[q], si[q], b, bi))) {
        b = sb[q];
        bi = si[q];
      }
    // nothing feasible -> (+inf, -1)
    if (!(b < CUDART_INF)) bi = -1;
    *out_s = b;
    *out_i = bi;
  }
}

static SearchArgs make_args(const rh_search* S) {
  SearchArgs a{};
  const rh_search_desc& d = S->d;
  a.m = d.model;
  a.sched = d.schedule;
  a.N = d.token_budget;
  a.M = d.n_micro_batches;
  a.L = d.total_layers;
  a.min_layers = d.min_layers;
  a.cap = d.capacity;
  a.has_comm = d.has_comm;
  a.p2p_opt = d.p2p_optimized;
  a.n_layouts = (int)S->lT.size();
  a.n_links = d.n_links;
  a.intra = d.intra_bw;
  a.inter = d.inter_bw;
  a.nbytes = d.hidden_bytes_per_token * (double)d.token_budget;  // comm.py:57-58
  a.lb = d.layer_bytes;
  double f = 1.0;
  bool any = false;
  for (double x : S->link_factor) {
    f = any ? std::min(f, x) : x;
    any = true;
  }
  a.worst_inter = d.inter_bw * (any ? f : 1.0);  // comm.py:38-40
  a.rebuild_s = d.group_rebuild_s;
  a.amort = d.amortize_iterations;
  a.cur_T = d.cur_tp;
  a.cur_D = d.cur_dp;
  a.cur_P = d.cur_pp;
  a.T0 = d.nominal_tp > 0 ? d.nominal_tp : 1;
  a.r_bw = d.model.ratio_b + d.model.ratio_w;
  a.div_safe = S->div_safe;
  a.tab_stride = d.n_micro_batches + 2;
  a.v = S->dv;
  return a;
}

}  // namespace rh

namespace rh {

// Op lists of the pipe kernel for every (P, md) a pipeline of this search can
// have: the even split (M/D, M/D+1) and the proportional counts +-1 of every
// layout (read back after prep_kernel).  Entry order: DAG level ascending,
// stage descending; peak = most forward chunks in flight on any stage.
// The prep kernel's per-layout results the host needs (decode, op lists):
// group blocks, repartitions, proportional splits.  Fetched once, after the
// create's kernels (a sync on the search's last stream).
static int fetch_host_tables(rh_search* S, cudaStream_t st) {
  std::lock_guard<std::mutex> lock(S->host_mu);
  if (S->host_ready) return RH_OK;
  const int NL = (int)S->lT.size();
  std::vector<int32_t>& pst = S->h_pstart;
  pst.resize(S->n_rep + NL);
  S->h_gblk.resize(S->n_groups);
  S->h_repart.resize(S->n_stage);
  RH_CUDA(cudaMemcpyAsync(pst.data(), S->dv.pstart, 4 * pst.size(), cudaMemcpyDeviceToHost, st));
  RH_CUDA(cudaMemcpyAsync(S->h_gblk.data(), S->dv.gblk, 4 * S->n_groups, cudaMemcpyDeviceToHost,
                          st));
  RH_CUDA(cudaMemcpyAsync(S->h_repart.data(), S->dv.repart, 4 * S->n_stage,
                          cudaMemcpyDeviceToHost, st));
  RH_CUDA(cudaStreamSynchronize(st));
  S->host_ready = true;
  return RH_OK;
}

// Op lists and capacity peaks of the op-list pipe kernel (ZBH, P > 32, or
// the RH_SEARCH_SMEM_WALK A/B build); the 1F1B register walk needs neither.
static int build_op_lists(rh_ctx* ctx, rh_search* S, cudaStream_t st) {
  const int NL = (int)S->lT.size(), M = S->d.n_micro_batches;
  const int stride = M + 2;
  const bool zbh = S->d.schedule == RH_SCHED_ZBH;
  bool want_ops = zbh || getenv("RH_SEARCH_SMEM_WALK") != nullptr;
  for (int li = 0; li < NL && !want_ops; ++li) want_ops = S->lP[li] > 32;
  if (!want_ops) {
    S->dv.tab_off = S->dv.tab_cnt = S->dv.tab_peak = nullptr;
    S->dv.ops = nullptr;
    return RH_OK;
  }
  if (int rc = fetch_host_tables(S, st)) return rc;
  const std::vector<int32_t>& pst = S->h_pstart;
  std::vector<char> need(33 * (size_t)stride, 0);
  for (int li = 0; li < NL; ++li) {
    const int D = S->lD[li], P = S->lP[li];
    char* row = need.data() + (size_t)P * stride;
    row[M / D] = 1;
    row[std::min(M, M / D + 1)] = 1;
    const int32_t* ps = pst.data() + S->ldoff[li] + li;
    for (int dd = 0; dd < D; ++dd) {
      const int c = ps[dd + 1] - ps[dd];
      for (int x = c - 1; x <= c + 1; ++x)
        if (x >= 0 && x <= M) row[x] = 1;
    }
  }
  std::vector<int32_t> off(33 * (size_t)stride, 0), cnt(33 * (size_t)stride, 0),
      peak(33 * (size_t)stride, 0);
  std::vector<uint32_t> ops;
  for (int P = 1; P <= 32; ++P)
    for (int md = 0; md <= M; ++md) {
      const size_t slot = (size_t)P * stride + md;
      if (!need[slot]) continue;
      // counting sort by DAG level of the forward closed forms; stages are
      // visited in descending order, so each level lists them descending
      off[slot] = (int32_t)ops.size();
      int t_end = 0;
      for (int s2 = 0; s2 < P; ++s2)
        t_end = std::max(t_end, ChainLevels{s2, P, md, std::min(P - 1 - s2, md)}.end(zbh));
      std::vector<int32_t> lvl_start(t_end + 1, 0);
      const int kinds = zbh ? 3 : 2;
      for (int s2 = 0; s2 < P; ++s2) {
        const ChainLevels lv{s2, P, md, std::min(P - 1 - s2, md)};
        for (int j = 0; j < md; ++j) {
          ++lvl_start[lv.F(j) + 1];
          ++lvl_start[lv.B(j) + 1];
          if (zbh) ++lvl_start[lv.W(j) + 1];
        }
      }
      for (int t = 0; t < t_end; ++t) lvl_start[t + 1] += lvl_start[t];
      const size_t base_op = ops.size();
      ops.resize(base_op + (size_t)kinds * P * md);
      for (int s2 = P - 1; s2 >= 0; --s2) {
        const ChainLevels lv{s2, P, md, std::min(P - 1 - s2, md)};
        const uint32_t depF = s2 > 0 ? 1u : 0u, depB = s2 < P - 1 ? 2u : 0u;
        for (int j = 0; j < md; ++j) {
          ops[base_op + lvl_start[lv.F(j)]++] =
              (uint32_t)s2 | (kOpF << 6) | (depF << 8) | ((uint32_t)j << 10);
          ops[base_op + lvl_start[lv.B(j)]++] =
              (uint32_t)s2 | (kOpB << 6) | (depB << 8) | ((uint32_t)j << 10);
          if (zbh)
            ops[base_op + lvl_start[lv.W(j)]++] =
                (uint32_t)s2 | (kOpW << 6) | ((uint32_t)j << 10);
        }
      }
      // capacity peak: forward chunks in flight on any stage
      std::vector<int> live(P, 0);
      int pk = 0;
      for (size_t e = base_op; e < ops.size(); ++e) {
        const int s2 = ops[e] & 63u;
        const unsigned kind = (ops[e] >> 6) & 3u;
        if (kind == kOpF) pk = std::max(pk, ++live[s2]);
        if (kind == kOpB) --live[s2];
      }
      cnt[slot] = (int32_t)ops.size() - off[slot];
      peak[slot] = pk;
    }
  const size_t tab_bytes = 3 * off.size() * 4;
  const size_t bytes = tab_bytes + 4 * std::max<size_t>(1, ops.size());
  RH_CUDA(cudaMallocFromPoolAsync(&S->dops, bytes, ctx->pool, st));
  std::vector<char> stage(bytes, 0);
  memcpy(stage.data(), off.data(), off.size() * 4);
  memcpy(stage.data() + off.size() * 4, cnt.data(), cnt.size() * 4);
  memcpy(stage.data() + 2 * off.size() * 4, peak.data(), peak.size() * 4);
  if (!ops.empty()) memcpy(stage.data() + tab_bytes, ops.data(), ops.size() * 4);
  RH_CUDA(cudaMemcpyAsync(S->dops, stage.data(), bytes, cudaMemcpyHostToDevice, st));
  RH_CUDA(cudaStreamSynchronize(st));  // the staging buffer dies here
  char* B = static_cast<char*>(S->dops);
  S->dv.tab_off = reinterpret_cast<const int32_t*>(B);
  S->dv.tab_cnt = reinterpret_cast<const int32_t*>(B + off.size() * 4);
  S->dv.tab_peak = reinterpret_cast<const int32_t*>(B + 2 * off.size() * 4);
  S->dv.ops = reinterpret_cast<const uint32_t*>(B + tab_bytes);
  (void)ctx;
  return RH_OK;
}

}  // namespace rh

namespace rh {
// div_fast is exact for every chunk of the search when every numerator
// (ratio * L) * base and every divisor (group speed) is in range
static void set_div_safe(rh_search* S, const int64_t* quad) {
  const rh_search_desc& d = S->d;
  double q_lo = HUGE_VAL, q_hi = 0.0;
  for (int j = 0; j < d.n_micro_batches; ++j) {
    const double b = d.model.alpha * d.token_budget + d.model.beta * (double)quad[j];
    q_hi = std::max(q_hi, b);
    if (b > 0.0) q_lo = std::min(q_lo, b);
  }
  const double r_lo = S->div_r_lo, r_hi = S->div_r_hi;
  const bool nums = q_hi * r_hi <= 0x1p890 && (q_hi * r_hi == 0.0 || q_lo * r_lo >= 0x1p-890);
  S->div_safe = nums && S->div_dens ? 1 : 0;
}
}  // namespace rh

using namespace rh;

extern "C" {

int rh_search_create(rh_ctx* ctx, const rh_search_desc* desc, rh_search** out, void* stream) {
  if (!ctx || !desc || !out || desc->n_devices <= 0 || desc->devices_per_node <= 0 ||
      !desc->device_speed || desc->n_micro_batches <= 0 ||
      desc->total_layers <= 0 || desc->min_layers < 0 || desc->token_budget <= 0 ||
      (desc->schedule != RH_SCHED_1F1B && desc->schedule != RH_SCHED_ZBH) ||
      desc->intra_bw <= 0 || desc->inter_bw <= 0 || (desc->n_links && !desc->link_nodes)) {
    set_error("rh_search_create: invalid descriptor");
    return RH_E_INVALID;
  }
  cudaStream_t st = as_stream(stream);
  DeviceGuard guard(ctx);
  // RH_SEARCH_TRACE=1: host wall time of the create's phases on stderr (debug aid)
  static const bool trace = getenv("RH_SEARCH_TRACE") != nullptr;
  const auto tc0 = std::chrono::steady_clock::now();
  auto tmark = [&](const char* what) {
    if (trace)
      fprintf(stderr, "rh_search_create %-10s %8.1f us\n", what,
              std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - tc0)
                  .count());
  };
  rh_search* S = new rh_search();
  S->d = *desc;
  const rh_search_desc& d = *desc;
  const int dpn = d.devices_per_node;
  S->n_nodes = (d.n_devices + dpn - 1) / dpn;
  S->speed.assign(d.device_speed, d.device_speed + d.n_devices);
  S->link_nodes.assign(d.link_nodes, d.link_nodes + 2 * d.n_links);
  S->link_factor.assign(d.link_factor, d.link_factor + d.n_links);
  const int cur_groups_n = d.cur_tp * d.cur_dp * d.cur_pp;
  if (d.cur_groups && cur_groups_n > 0)
    S->cur_groups.assign(d.cur_groups, d.cur_groups + cur_groups_n);
  else
    S->cur_groups.assign(1, -1);
  if (d.cur_partition && d.cur_pp > 0)
    S->cur_partition.assign(d.cur_partition, d.cur_partition + d.cur_pp);
  else
    S->cur_partition.assign(1, 0);
  S->d.device_speed = nullptr;
  S->d.link_nodes = nullptr;
  S->d.link_factor = nullptr;
  S->d.quad = nullptr;
  S->d.cur_groups = nullptr;
  S->d.cur_partition = nullptr;
  int executable = 0;
  for (double x : S->speed) executable += x > 0.0;

  // ---- blocks per TP degree: node-local fastest-first chunks of T
  std::vector<int> degrees;
  for (int T = 1; T <= dpn && T <= std::max(1, d.max_tp); T <<= 1)
    if (dpn % T == 0) degrees.push_back(T);
  std::vector<int> t_off(degrees.size()), t_nb(degrees.size());
  for (size_t ti = 0; ti < degrees.size(); ++ti) {
    const int T = degrees[ti];
    t_off[ti] = (int)S->blk_node.size();
    std::vector<int> order;
    for (int n = 0; n < S->n_nodes; ++n) {
      order.clear();
      for (int q = n * dpn; q < std::min(d.n_devices, (n + 1) * dpn); ++q)
        if (S->speed[q] > 0.0) order.push_back(q);
      std::stable_sort(order.begin(), order.end(), [&](int x, int y) {
        return S->speed[x] > S->speed[y];
      });
      for (size_t b = 0; b + T <= order.size(); b += T) {
        std::vector<int> mem(order.begin() + b, order.begin() + b + T);
        double mn = S->speed[mem[0]];
        for (int q : mem) mn = std::min(mn, S->speed[q]);
        std::sort(mem.begin(), mem.end());
        S->blk_moff.push_back((int)S->blk_members.size());
        S->blk_members.insert(S->blk_members.end(), mem.begin(), mem.end());
        S->blk_node.push_back(n);
        S->blk_speed.push_back(mn);
      }
    }
    const int nb = (int)S->blk_node.size() - t_off[ti];
    t_nb[ti] = nb;
    std::vector<int> idx(nb);
    for (int q = 0; q < nb; ++q) idx[q] = q;
    std::stable_sort(idx.begin(), idx.end(), [&](int x, int y) {
      return S->blk_speed[t_off[ti] + x] > S->blk_speed[t_off[ti] + y];
    });
    S->blk_rank.resize(S->blk_node.size());
    for (int r = 0; r < nb; ++r) S->blk_rank[t_off[ti] + idx[r]] = r;
  }
  // ---- layouts
  const int max_pp = std::min(32, d.max_pp > 0 ? d.max_pp : 32);
  const int max_dp = std::min(64, d.max_dp > 0 ? d.max_dp : 64);
  const int ml = std::max(1, d.min_layers);
  long long base = 0;
  int goff = 0, poff = 0, doff = 0;
  for (size_t ti = 0; ti < degrees.size(); ++ti) {
    const int T = degrees[ti];
    for (int P = 1; P <= max_pp && P * ml <= d.total_layers; ++P) {
      for (int D = 1; D <= max_dp && D <= d.n_micro_batches; ++D) {
        if (D * P > t_nb[ti]) break;
        if ((double)T * D * P < d.min_utilization * executable) continue;
        const long long nv = 2 + (long long)P * (P - 1);
        const long long nu = 2 + (long long)D * (D - 1);
        S->lT.push_back(T);
        S->lD.push_back(D);
        S->lP.push_back(P);
        S->lgoff.push_back(goff);
        S->lpoff.push_back(poff);
        S->ldoff.push_back(doff);
        S->lboff.push_back(t_off[ti]);
        S->lnb.push_back(t_nb[ti]);
        S->lbase.push_back(base);
        S->lnv.push_back(nv);
        S->lnu.push_back(nu);
        S->lpair.push_back(S->n_pairs);
        S->lrt.push_back(S->n_rt);
        S->n_pairs += nv;
        S->n_rt += nv * 8 * D;
        base += nv * nu;
        goff += D * P;
        poff += P;
        doff += D;
      }
    }
  }
  tmark("layouts");
  S->total = base;
  S->n_groups = goff;
  S->n_stage = poff;
  S->n_rep = doff;
  const int NL = (int)S->lT.size();
  if (NL == 0) {
    S->workload_ready = true;  // nothing to score
    *out = S;
    return RH_OK;
  }
  {  // ranges of every numerator ((ratio * L) * base) and divisor (group speed);
     // the base-cost part waits for the workload when it is deferred
    const double ratios[4] = {d.model.ratio_f, d.model.ratio_b, d.model.ratio_w,
                              d.model.ratio_b + d.model.ratio_w};
    double r_lo = HUGE_VAL, r_hi = 0.0;
    for (double r : ratios) {
      r_hi = std::max(r_hi, r * d.total_layers);
      if (r > 0.0) r_lo = std::min(r_lo, r);  // times at least one layer
    }
    double s_lo = HUGE_VAL, s_hi = 0.0;
    const double T0 = d.nominal_tp > 0 ? d.nominal_tp : 1;
    for (double v : S->blk_speed) {
      s_lo = std::min(s_lo, v * 1.0 / T0);
      s_hi = std::max(s_hi, v * 32.0 / T0);
    }
    // margins of 2^10 absorb the rounding of these host estimates
    S->div_dens = S->blk_speed.empty() || (s_lo >= 0x1p-90 && s_hi <= 0x1p90);
    S->div_r_lo = r_lo;
    S->div_r_hi = r_hi;
    if (desc->quad) set_div_safe(S, desc->quad);
  }
  // ---- device memory
  int& max_blocks_per_sm = ctx->combine_occ;  // cached occupancy of the combine kernel
  if (max_blocks_per_sm < 0)
    RH_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&max_blocks_per_sm, combine_kernel,
                                                          kEvalThreads, 0));
  S->eval_blocks = ctx->num_sms * std::max(1, max_blocks_per_sm);
  size_t bytes = 0;
  auto take = [&](size_t n) {
    const size_t o = bytes;
    bytes = (bytes + std::max<size_t>(n, 8) + 255) & ~size_t(255);
    return o;
  };
  const size_t nblk = S->blk_node.size(), nmem = S->blk_members.size();
  struct Up {
    size_t off;
    const void* src;
    size_t n;
  };
  std::vector<Up> ups;
  auto up = [&](const void* src, size_t n) {
    const size_t o = take(n);
    ups.push_back({o, src, n});
    return o;
  };
  const size_t o_lT = up(S->lT.data(), 4 * NL), o_lD = up(S->lD.data(), 4 * NL),
               o_lP = up(S->lP.data(), 4 * NL), o_lgoff = up(S->lgoff.data(), 4 * NL),
               o_lpoff = up(S->lpoff.data(), 4 * NL), o_ldoff = up(S->ldoff.data(), 4 * NL),
               o_lboff = up(S->lboff.data(), 4 * NL), o_lnb = up(S->lnb.data(), 4 * NL),
               o_lbase = up(S->lbase.data(), 8 * NL), o_lnv = up(S->lnv.data(), 8 * NL),
               o_lnu = up(S->lnu.data(), 8 * NL), o_lpair = up(S->lpair.data(), 8 * NL),
               o_lrt = up(S->lrt.data(), 8 * NL);
  const size_t o_bnode = up(S->blk_node.data(), 4 * nblk),
               o_brank = up(S->blk_rank.data(), 4 * nblk),
               o_bmem = up(S->blk_members.data(), 4 * nmem),
               o_bmoff = up(S->blk_moff.data(), 4 * nblk),
               o_bspeed = up(S->blk_speed.data(), 8 * nblk);
  const size_t o_quad = up(desc->quad, 8 * (size_t)d.n_micro_batches);
  const size_t o_ln = up(S->link_nodes.data(), 4 * S->link_nodes.size()),
               o_lf = up(S->link_factor.data(), 8 * S->link_factor.size()),
               o_cg = up(S->cur_groups.data(), 4 * S->cur_groups.size()),
               o_cp = up(S->cur_partition.data(), 4 * S->cur_partition.size());
  const size_t up_bytes = bytes;  // everything uploaded sits in front
  const size_t o_gblk = take(4 * S->n_groups), o_gnode = take(4 * S->n_groups),
               o_gspeed = take(8 * S->n_groups), o_ghop = take(8 * S->n_groups),
               o_tspeed = take(8 * S->n_groups), o_tinv = take(8 * S->n_groups),
               o_thop = take(8 * S->n_groups),
               o_ring = take(8 * S->n_stage), o_sspeed = take(8 * S->n_stage),
               o_repart = take(4 * S->n_stage), o_rspeed = take(8 * S->n_rep),
               o_pstart = take(4 * (S->n_rep + NL)), o_same = take(4 * NL),
               o_base = take(8 * (size_t)d.n_micro_batches),
               // block results: the old combine's grid per layout, or one per
               // (layout, partition) pair (combine2)
               o_bb = take(8 * std::max<size_t>((size_t)S->eval_blocks * NL, S->n_pairs + NL)),
               o_bi = take(8 * std::max<size_t>((size_t)S->eval_blocks * NL, S->n_pairs + NL)),
               o_rtab = take(8 * (size_t)S->n_rt), o_pinfo = take(16 * (size_t)S->n_pairs),
               o_rl = take(8 * 96 * (size_t)S->n_pairs),
               o_tasks = take(sizeof(PipeTask) * (size_t)NL);
  // private stream-ordered pool: after the first re-plan the memory is
  // reused, not mapped again (the device's default pool is not touched)
  if (!ctx->pool) {
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = ctx->device;
    RH_CUDA(cudaMemPoolCreate(&ctx->pool, &props));
    uint64_t keep = ~0ull;
    RH_CUDA(cudaMemPoolSetAttribute(ctx->pool, cudaMemPoolAttrReleaseThreshold, &keep));
  }
  cudaError_t e = cudaMallocFromPoolAsync(&S->dmem, bytes, ctx->pool, st);
  if (e != cudaSuccess) {
    delete S;
    set_error("rh_search_create: %zu bytes: %s", bytes, cudaGetErrorString(e));
    return RH_E_NOMEM;
  }
  S->dbytes = bytes;
  S->last_stream = st;
  char* B = static_cast<char*>(S->dmem);
  {  // one host staging buffer, one copy
    std::vector<char> stage(up_bytes, 0);
    for (const Up& u : ups)
      if (u.n && u.src) memcpy(stage.data() + u.off, u.src, u.n);
    RH_CUDA(cudaMemcpyAsync(B, stage.data(), up_bytes, cudaMemcpyHostToDevice, st));
    RH_CUDA(cudaStreamSynchronize(st));  // the staging buffer dies here
  }
  tmark("upload");
  auto I = [&](size_t o) { return reinterpret_cast<int32_t*>(B + o); };
  auto Dp = [&](size_t o) { return reinterpret_cast<double*>(B + o); };
  auto LL = [&](size_t o) { return reinterpret_cast<long long*>(B + o); };
  rh_search::Dev& v = S->dv;
  v.lT = I(o_lT); v.lD = I(o_lD); v.lP = I(o_lP); v.lgoff = I(o_lgoff); v.lpoff = I(o_lpoff);
  v.ldoff = I(o_ldoff); v.lboff = I(o_lboff); v.lnb = I(o_lnb);
  v.lbase = LL(o_lbase); v.lnv = LL(o_lnv); v.lnu = LL(o_lnu);
  v.lpair = LL(o_lpair); v.lrt = LL(o_lrt);
  v.rtab = Dp(o_rtab); v.pinfo = Dp(o_pinfo); v.tasks = B + o_tasks; v.rl = Dp(o_rl);
  v.blk_node = I(o_bnode); v.blk_rank = I(o_brank); v.blk_members = I(o_bmem);
  v.blk_moff = I(o_bmoff); v.blk_speed = Dp(o_bspeed);
  v.quad = reinterpret_cast<int64_t*>(B + o_quad);
  v.link_nodes = I(o_ln); v.link_factor = Dp(o_lf); v.cur_groups = I(o_cg);
  v.cur_partition = I(o_cp);
  v.gblk = I(o_gblk); v.gnode = I(o_gnode); v.gspeed = Dp(o_gspeed); v.ghop = Dp(o_ghop);
  v.tspeed = Dp(o_tspeed); v.tinv = Dp(o_tinv); v.thop = Dp(o_thop);
  v.ring = Dp(o_ring); v.sspeed = Dp(o_sspeed); v.repart = I(o_repart);
  v.rspeed = Dp(o_rspeed); v.pstart = I(o_pstart); v.same = I(o_same); v.base = Dp(o_base);
  v.blk_best = Dp(o_bb); v.blk_idx = LL(o_bi);
  SearchArgs a = make_args(S);
  if (desc->quad) {
    base_kernel<<<(d.n_micro_batches + 255) / 256, 256, 0, st>>>(a);
    RH_CHECK_LAUNCH(ctx);
    S->workload_ready = true;
  }
  prep_kernel<<<(NL * 32 + 127) / 128, 128, 0, st>>>(a);
  RH_CHECK_LAUNCH(ctx);
  if (int rc = build_op_lists(ctx, S, st)) {
    rh_search_destroy(S);
    return rc;
  }
  tmark("op lists");
  // the preparation kernels stay queued: set_workload, eval and decode order
  // after them (done_ev / the stream)
  RH_CUDA(cudaEventCreateWithFlags(&S->done_ev, cudaEventDisableTiming));
  RH_CUDA(cudaEventRecord(S->done_ev, st));
  tmark("done");
  *out = S;
  return RH_OK;
}

int rh_search_destroy(rh_search* S) {
  if (!S) return RH_OK;
  // back to the pool, ordered after the latest work issued on the search
  if (S->dmem) cudaFreeAsync(S->dmem, S->last_stream);
  if (S->dops) cudaFreeAsync(S->dops, S->last_stream);
  if (S->done_ev) cudaEventDestroy(S->done_ev);
  delete S;
  return RH_OK;
}

int rh_search_set_workload(rh_ctx* ctx, rh_search* S, const int64_t* quad, void* stream) {
  if (!ctx || !S || !quad) {
    set_error("rh_search_set_workload: invalid arguments");
    return RH_E_INVALID;
  }
  DeviceGuard guard(ctx);
  std::lock_guard<std::mutex> lock(ctx->search_mu);
  cudaStream_t st = as_stream(stream);
  if (S->done_ev) RH_CUDA(cudaStreamWaitEvent(st, S->done_ev, 0));
  set_div_safe(S, quad);
  if (S->dmem && S->d.n_micro_batches > 0) {
    RH_CUDA(cudaMemcpyAsync(S->dv.quad, quad, 8 * (size_t)S->d.n_micro_batches,
                            cudaMemcpyHostToDevice, st));
    SearchArgs a = make_args(S);
    base_kernel<<<(S->d.n_micro_batches + 255) / 256, 256, 0, st>>>(a);
    RH_CHECK_LAUNCH(ctx);
    if (S->done_ev) RH_CUDA(cudaEventRecord(S->done_ev, st));
    // the host copy source may be released when this returns
    RH_CUDA(cudaStreamSynchronize(st));
  }
  S->workload_ready = true;
  return RH_OK;
}

int64_t rh_search_size(const rh_search* S) { return S ? S->total : 0; }

int rh_search_shard(const rh_search* S, int32_t rank, int32_t world, int64_t* begin,
                    int64_t* end) {
  if (!S || world < 1 || rank < 0 || rank >= world || !begin || !end) {
    set_error("rh_search_shard: invalid arguments");
    return RH_E_INVALID;
  }
  // work of one (layout, v) block: 8*D pipelines of ~c*P*(M/D) chunks each
  // (~c*P*M*8 chunk steps) plus nu candidates combining D table entries
  // (one combination step ~ 1/8 of a chunk step, measured on B200)
  const int c = S->d.schedule == RH_SCHED_ZBH ? 3 : 2;
  const double M = (double)S->d.n_micro_batches;
  double total = 0.0;
  for (size_t li = 0; li < S->lT.size(); ++li)
    total += (double)S->lnv[li] *
             (8.0 * c * S->lP[li] * M + 0.125 * (double)S->lnu[li] * S->lD[li]);
  const double lo = total * rank / world, hi = total * (rank + 1) / world;
  // block k belongs to the rank whose cost interval holds its cumulative midpoint
  int64_t b = -1, e = -1;
  double acc = 0.0;
  for (size_t li = 0; li < S->lT.size(); ++li) {
    const double w = 8.0 * c * S->lP[li] * M + 0.125 * (double)S->lnu[li] * S->lD[li];
    for (long long v = 0; v < S->lnv[li]; ++v) {
      const double mid = acc + 0.5 * w;
      acc += w;
      if (mid < lo) continue;
      if (mid >= hi && rank < world - 1) break;
      const int64_t first = S->lbase[li] + v * S->lnu[li];
      if (b < 0) b = first;
      e = first + S->lnu[li];
    }
  }
  if (b < 0) {  // an empty shard: place it where the cost boundary falls
    b = e = 0;
    double acc2 = 0.0;
    for (size_t li = 0; li < S->lT.size() && acc2 < lo; ++li) {
      const double w = 8.0 * c * S->lP[li] * M + 0.125 * (double)S->lnu[li] * S->lD[li];
      for (long long v = 0; v < S->lnv[li] && acc2 + 0.5 * w < lo; ++v) {
        acc2 += w;
        b = e = S->lbase[li] + (v + 1) * S->lnu[li];
      }
    }
  }
  *begin = b;
  *end = e;
  return RH_OK;
}
int32_t rh_search_layouts(const rh_search* S) { return S ? (int32_t)S->lT.size() : 0; }

int rh_search_eval(rh_ctx* ctx, rh_search* S, int64_t begin, int64_t end, double* best_score,
                   int64_t* best_index, double* scores, void* stream) {
  if (!ctx || !S || !best_score || !best_index || begin < 0 || end < begin ||
      end > S->total) {
    set_error("rh_search_eval: invalid range [%lld, %lld) of %lld", (long long)begin,
              (long long)end, (long long)(S ? S->total : 0));
    return RH_E_INVALID;
  }
  if (!S->workload_ready) {
    set_error("rh_search_eval: the workload (quad loads) was deferred and not yet set");
    return RH_E_INVALID;
  }
  cudaStream_t st = as_stream(stream);
  DeviceGuard guard(ctx);
  // the context's auxiliary streams and fork / join events are shared
  std::lock_guard<std::mutex> lock(ctx->search_mu);
  // the previous eval (maybe on another stream) still reads this search's
  // task list and block results
  if (S->done_ev) RH_CUDA(cudaStreamWaitEvent(st, S->done_ev, 0));
  if (begin == end) {
    const double inf = std::numeric_limits<double>::infinity();
    const int64_t none = -1;
    RH_CUDA(cudaMemcpyAsync(best_score, &inf, 8, cudaMemcpyHostToDevice, st));
    RH_CUDA(cudaMemcpyAsync(best_index, &none, 8, cudaMemcpyHostToDevice, st));
    return RH_OK;
  }
  S->last_stream = st;
  SearchArgs a = make_args(S);
  const long long n = end - begin;
  // phase 1 tasks: (layout, partition variant range) overlapping [begin, end),
  // grouped by P (one pipe_kernel launch per stage count: its shared memory
  // holds P stage slots per thread)
  std::vector<PipeTask> tk;
  struct Group {
    int P;
    size_t first, count;
    long long n_pipes, n_rows;
  };
  std::vector<Group> groups;
  for (int P = 1; P <= 32; ++P) {
    Group g{P, tk.size(), 0, 0, 0};
    for (int li = 0; li < (int)S->lT.size(); ++li) {
      if (S->lP[li] != P) continue;
      const long long lb = S->lbase[li], le = lb + S->lnv[li] * S->lnu[li];
      if (le <= begin || lb >= end) continue;
      const int v_lo = (int)((std::max<long long>(begin, lb) - lb) / S->lnu[li]);
      const int v_hi = (int)((std::min<long long>(end, le) - 1 - lb) / S->lnu[li]);
      tk.push_back({li, v_lo, g.n_pipes, g.n_rows});
      g.n_pipes += (long long)(v_hi - v_lo + 1) * 8 * S->lD[li];
      g.n_rows += v_hi - v_lo + 1;
    }
    g.count = tk.size() - g.first;
    if (g.count) groups.push_back(g);
  }
  RH_CUDA(cudaMemcpyAsync(S->dv.tasks, tk.data(), sizeof(PipeTask) * tk.size(),
                          cudaMemcpyHostToDevice, st));
  const bool zbh = S->d.schedule == RH_SCHED_ZBH;
  void* kern = zbh ? (S->div_safe ? (void*)pipe_kernel<1, true> : (void*)pipe_kernel<1, false>)
                  : (S->div_safe ? (void*)pipe_kernel<0, true> : (void*)pipe_kernel<0, false>);
  // the per-P launches write disjoint table rows: run them concurrently on the
  // context's auxiliary streams (fork / join by events on `st`) so one
  // launch's last wave overlaps the next launch instead of idling SMs
  constexpr int kAux = rh_ctx::kAuxStreams;
  for (int q = 0; q < kAux; ++q) {
    if (!ctx->aux_stream[q])
      RH_CUDA(cudaStreamCreateWithFlags(&ctx->aux_stream[q], cudaStreamNonBlocking));
    if (!ctx->aux_ev[q]) RH_CUDA(cudaEventCreateWithFlags(&ctx->aux_ev[q], cudaEventDisableTiming));
  }
  if (!ctx->aux_fork) RH_CUDA(cudaEventCreateWithFlags(&ctx->aux_fork, cudaEventDisableTiming));
  RH_CUDA(cudaEventRecord(ctx->aux_fork, st));
  const int n_used = std::min<int>(kAux, (int)groups.size());
  for (int q = 0; q < n_used; ++q) RH_CUDA(cudaStreamWaitEvent(ctx->aux_stream[q], ctx->aux_fork, 0));
  int gi = 0;
  long long n_blk = 0;  // block results written so far (contiguous)
  for (const Group& g : groups) {
    cudaStream_t gs = ctx->aux_stream[gi++ % kAux];
    const size_t smem = (size_t)(zbh ? 3 : 2) * g.P * kPipeThreads * sizeof(double);
    // (the pipe kernel strides its state by kPipeThreads)
    if (int e = ensure_smem(ctx, kern, smem)) return e;
    int occ = 0;
    RH_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kPipeThreads, smem));
    const long long want = (g.n_pipes + kPipeThreads - 1) / kPipeThreads;
    const int blocks = (int)std::max<long long>(
        1, std::min<long long>(want, (long long)ctx->num_sms * std::max(1, occ) * 8));
    const PipeTask* tp = reinterpret_cast<const PipeTask*>(S->dv.tasks) + g.first;
    int n_tk = (int)g.count;
    {
      const long long n_rl = g.n_rows * g.P;
      rl_kernel<<<(unsigned)((n_rl + 255) / 256), 256, 0, gs>>>(a, tp, n_tk, g.P, g.n_rows);
      RH_CHECK_LAUNCH(ctx);
    }
    long long n_pipes = g.n_pipes;
    int P = g.P;
    void* reg = (!zbh && !getenv("RH_SEARCH_SMEM_WALK"))
                    ? (S->div_safe ? pipe_reg_kernel_for<true>(P) : pipe_reg_kernel_for<false>(P))
                    : nullptr;
    if (reg) {  // register-resident walk (1F1B)
      int rocc = 0;
      RH_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&rocc, reg, kPipeThreads, 0));
      const int rblocks = (int)std::max<long long>(
          1, std::min<long long>(want, (long long)ctx->num_sms * std::max(1, rocc) * 8));
      void* rargs[] = {&a, &tp, &n_tk, &n_pipes};
      RH_CUDA(cudaLaunchKernel(reg, dim3(rblocks), dim3(kPipeThreads), rargs, 0, gs));
    } else {
      void* args[] = {&a, &tp, &n_tk, &n_pipes, &P};
      RH_CUDA(cudaLaunchKernel(kern, dim3(blocks), dim3(kPipeThreads), args, smem, gs));
    }
    RH_CHECK_LAUNCH(ctx);
    // this group's candidates, layout by layout, right behind its table rows
    for (size_t q = g.first; q < g.first + g.count; ++q) {
      const int li = tk[q].layout;
      const long long lo = std::max<long long>(begin, S->lbase[li]);
      const long long hi = std::min<long long>(end, S->lbase[li] + S->lnv[li] * S->lnu[li]);
      if (lo >= hi) continue;
      if (S->lD[li] <= kComb2MaxD && !getenv("RH_SEARCH_OLD_COMBINE")) {
        // one CTA per (layout, partition) pair overlapping [lo, hi)
        const int vlo = (int)((lo - S->lbase[li]) / S->lnu[li]);
        const int vhi = (int)((hi - 1 - S->lbase[li]) / S->lnu[li]);
        const int cb = vhi - vlo + 1;
        combine2_kernel<<<cb, kComb2Threads, 0, gs>>>(a, li, lo, hi, begin, vlo, scores,
                                                     S->dv.blk_best + n_blk,
                                                     S->dv.blk_idx + n_blk);
        RH_CHECK_LAUNCH(ctx);
        n_blk += cb;
      } else {
        const int cb = (int)std::min<long long>(S->eval_blocks, (hi - lo + kEvalThreads - 1) / kEvalThreads);
        combine_kernel<<<cb, kEvalThreads, 0, gs>>>(a, lo, hi, begin, scores, S->dv.blk_best + n_blk,
                                                   S->dv.blk_idx + n_blk);
        RH_CHECK_LAUNCH(ctx);
        n_blk += cb;
      }
    }
  }
  for (int q = 0; q < n_used; ++q) {
    RH_CUDA(cudaEventRecord(ctx->aux_ev[q], ctx->aux_stream[q]));
    RH_CUDA(cudaStreamWaitEvent(st, ctx->aux_ev[q], 0));
  }
  (void)n;
  minloc_kernel<<<1, 1024, 0, st>>>(S->dv.blk_best, S->dv.blk_idx, (int)n_blk, best_score,
                                    best_index);
  RH_CHECK_LAUNCH(ctx);
  RH_CUDA(cudaEventRecord(S->done_ev, st));
  return RH_OK;
}

int rh_search_decode(rh_ctx* ctx, rh_search* S, int64_t index, rh_candidate* out,
                     int32_t* groups, int32_t* partition, int32_t* counts) {
  if (!ctx || !S || !out || index < 0 || index >= S->total) {
    set_error("rh_search_decode: index out of range");
    return RH_E_INVALID;
  }
  DeviceGuard guard(ctx);
  if (!S->host_ready) {
    if (S->done_ev) RH_CUDA(cudaEventSynchronize(S->done_ev));
    if (int rc = fetch_host_tables(S, S->last_stream)) return rc;
  }
  const int NL = (int)S->lT.size();
  int li = (int)(std::upper_bound(S->lbase.begin(), S->lbase.end(), (long long)index) -
                 S->lbase.begin()) - 1;
  li = std::max(0, std::min(li, NL - 1));
  const int T = S->lT[li], D = S->lD[li], P = S->lP[li];
  const long long local = index - S->lbase[li];
  const int vv = (int)(local / S->lnu[li]), uu = (int)(local % S->lnu[li]);
  out->index = index;
  out->tp = T;
  out->dp = D;
  out->pp = P;
  out->layout = li;
  out->partition_variant = vv;
  out->count_variant = uu;
  const int32_t* gblk = S->h_gblk.data() + S->lgoff[li];
  const int32_t* rep = S->h_repart.data() + S->lpoff[li];
  const int32_t* pst = S->h_pstart.data() + S->ldoff[li] + li;
  const rh_search_desc& d = S->d;
  std::vector<int> part(P), cnt(D);
  int psrc = -1, pdst = -1, csrc = -1, cdst = -1;
  if (vv >= 2) {
    const int m = vv - 2, r = m % (P - 1);
    psrc = m / (P - 1);
    pdst = r < psrc ? r : r + 1;
  }
  if (uu >= 2) {
    const int m = uu - 2, r = m % (D - 1);
    csrc = m / (D - 1);
    cdst = r < csrc ? r : r + 1;
  }
  for (int s = 0; s < P; ++s)
    part[s] = vv == 0 ? d.total_layers / P + (s < d.total_layers % P ? 1 : 0)
                      : rep[s] + (s == pdst) - (s == psrc);
  for (int q = 0; q < D; ++q) {
    if (uu == 0) cnt[q] = d.n_micro_batches / D + (q < d.n_micro_batches % D ? 1 : 0);
    else cnt[q] = pst[q + 1] - pst[q] + (q == cdst) - (q == csrc);
  }
  bool feas = true;
  for (int s = 0; s < P; ++s) feas &= part[s] >= d.min_layers;
  for (int q = 0; q < D; ++q) feas &= cnt[q] >= 0;
  out->feasible = feas;
  if (groups)
    for (int g = 0; g < D * P; ++g)
      for (int t = 0; t < T; ++t) groups[g * T + t] = S->blk_members[S->blk_moff[gblk[g]] + t];
  if (partition)
    for (int s = 0; s < P; ++s) partition[s] = part[s];
  if (counts)
    for (int q = 0; q < D; ++q) counts[q] = cnt[q];
  return RH_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Batched scalar Scheduler rows (one thread per problem): the same device
// functions the search prep uses, exposed for the drop-in resihp_adapt.
namespace rh {

// one warp per problem
__global__ void repartition_batch_kernel(int n, const int32_t* off, const double* sp,
                                         const int32_t* L, const int32_t* ml, int32_t* out,
                                         int32_t* err) {
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (i >= n) return;
  const int a = off[i], P = off[i + 1] - a;
  int e = 0;
  if (P > 32) e = 3;
  for (int s = 0; s < P && !e; ++s)
    if (!(sp[a + s] > 0.0)) e = 1;  // "all stage speeds must be positive"
  if (!e && L[i] < P * ml[i]) e = 2;  // "cannot give n stages ..."
  if ((threadIdx.x & 31) == 0) err[i] = e;
  if (!e) repartition_warp(sp + a, P, L[i], ml[i], out + a);
}

__global__ void proportional_batch_kernel(int n, const int32_t* off, const double* w,
                                          const int32_t* total, int32_t* counts, int32_t* err) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int a = off[i], D = off[i + 1] - a;
  double wsum = 0.0;
  for (int q = 0; q < D; ++q) wsum = __dadd_rn(wsum, w[a + q]);
  int e = D > 64 ? 3 : (wsum <= 0.0 ? 1 : 0);  // "no capacity left to assign work to"
  err[i] = e;
  if (e) return;
  int32_t start[65];
  proportional_dev(total[i], w + a, D, start);
  for (int q = 0; q < D; ++q) counts[a + q] = start[q + 1] - start[q];
}

// select_tp_subgroup (scheduler.py:114-137): rank by (-speed, id); for each
// allowed power-of-two degree k (ascending) keep the first strictly better
// k * speed_k; ties go to the smaller group.
__global__ void subgroup_batch_kernel(int n, const int32_t* off, const double* sp,
                                      const int32_t* ids, const uint32_t* degree_mask,
                                      int32_t* ranked, int32_t* best_k) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int a = off[i], m = off[i + 1] - a;
  int32_t* r = ranked + a;
  for (int q = 0; q < m; ++q) r[q] = q;
  for (int q = 1; q < m; ++q) {  // insertion sort by (-speed, id)
    const int v = r[q];
    int k = q - 1;
    while (k >= 0 && (sp[a + r[k]] < sp[a + v] ||
                      (sp[a + r[k]] == sp[a + v] && ids[a + r[k]] > ids[a + v]))) {
      r[k + 1] = r[k];
      --k;
    }
    r[k + 1] = v;
  }
  int bk = 0;
  double bs = -1.0;
  for (int e = 0; e < 31; ++e) {
    if (!(degree_mask[i] >> e & 1u)) continue;
    const int k = 1 << e;
    if (k > m) continue;
    const double score = __dmul_rn((double)k, sp[a + r[k - 1]]);
    if (score > bs) {
      bs = score;
      bk = k;
    }
  }
  for (int q = 0; q < m; ++q) r[q] = ids[a + r[q]];
  best_k[i] = bk;  // 0: GroupUnrecoverable
}

}  // namespace rh

extern "C" {

int rh_repartition_batch(rh_ctx* ctx, int32_t n, const int32_t* off, const double* speeds,
                         const int32_t* total_layers, const int32_t* min_layers, int32_t* out,
                         int32_t* err, void* stream) {
  if (!ctx || n < 0 || (n && (!off || !speeds || !total_layers || !min_layers || !out || !err))) {
    set_error("rh_repartition_batch: invalid arguments");
    return RH_E_INVALID;
  }
  if (!n) return RH_OK;
  DeviceGuard guard(ctx);
  repartition_batch_kernel<<<(n * 32 + 127) / 128, 128, 0, as_stream(stream)>>>(
      n, off, speeds, total_layers, min_layers, out, err);
  RH_CHECK_LAUNCH(ctx);
  return RH_OK;
}

int rh_proportional_split_batch(rh_ctx* ctx, int32_t n, const int32_t* off,
                                const double* weights, const int32_t* totals, int32_t* counts,
                                int32_t* err, void* stream) {
  if (!ctx || n < 0 || (n && (!off || !weights || !totals || !counts || !err))) {
    set_error("rh_proportional_split_batch: invalid arguments");
    return RH_E_INVALID;
  }
  if (!n) return RH_OK;
  DeviceGuard guard(ctx);
  proportional_batch_kernel<<<(n + 127) / 128, 128, 0, as_stream(stream)>>>(n, off, weights,
                                                                           totals, counts, err);
  RH_CHECK_LAUNCH(ctx);
  return RH_OK;
}

int rh_select_subgroup_batch(rh_ctx* ctx, int32_t n, const int32_t* off, const double* speeds,
                             const int32_t* ids, const uint32_t* degree_mask, int32_t* ranked,
                             int32_t* best_k, void* stream) {
  if (!ctx || n < 0 || (n && (!off || !speeds || !ids || !degree_mask || !ranked || !best_k))) {
    set_error("rh_select_subgroup_batch: invalid arguments");
    return RH_E_INVALID;
  }
  if (!n) return RH_OK;
  DeviceGuard guard(ctx);
  subgroup_batch_kernel<<<(n + 127) / 128, 128, 0, as_stream(stream)>>>(n, off, speeds, ids,
                                                                       degree_mask, ranked, best_k);
  RH_CHECK_LAUNCH(ctx);
  return RH_OK;
}

}  // extern "C"
