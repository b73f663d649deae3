// General chunk-DAG critical path (rh_dag_critical_path): pipeline.py:259-292
// for DAGs that are not canonical 1F1B/ZBH chains (migrated chunks,
// planner-realised stage orders, user-built DAGs).
//
// Level-synchronous Kahn relaxation in one CTA: every vertex of the current
// frontier pushes finish+w into its successors with a 64-bit atomicMax on
// the (non-negative) double bit pattern, and decrements their in-degree; a
// successor whose in-degree hits zero joins the next frontier.  max() is
// order-independent, so starts[] equals the reference's bit for bit.
#include "common.cuh"

namespace rh {

constexpr int kDagThreads = 1024;

__global__ void __launch_bounds__(kDagThreads)
dag_kernel(int32_t nv, const double* __restrict__ cost, const int32_t* __restrict__ off,
           const int32_t* __restrict__ dst, const double* __restrict__ w,
           int32_t n_chains, const int32_t* __restrict__ chain_off,
           const uint8_t* __restrict__ kind, int32_t capacity,
           double* __restrict__ starts, double* __restrict__ makespan,
           double* __restrict__ chain_sum, int32_t* __restrict__ flags,
           int32_t* indeg, int32_t* fa, int32_t* fb) {
  __shared__ int32_t s_n_next;
  __shared__ int32_t s_processed;
  __shared__ double s_red[32];
  for (int32_t v = threadIdx.x; v < nv; v += blockDim.x) {
    starts[v] = 0.0;
    indeg[v] = 0;
  }
  if (threadIdx.x == 0) {
    s_n_next = 0;
    s_processed = 0;
  }
  __syncthreads();
  const int32_t ne = off[nv];
  for (int32_t e = threadIdx.x; e < ne; e += blockDim.x) atomicAdd(indeg + dst[e], 1);
  __syncthreads();
  for (int32_t v = threadIdx.x; v < nv; v += blockDim.x)
    if (indeg[v] == 0) fa[atomicAdd(&s_n_next, 1)] = v;
  __syncthreads();
  int32_t n_cur = s_n_next;
  int32_t *cur = fa, *nxt = fb;
  while (n_cur > 0) {
    __syncthreads();
    if (threadIdx.x == 0) {
      s_n_next = 0;
      s_processed += n_cur;
    }
    __syncthreads();
    for (int32_t q = threadIdx.x; q < n_cur; q += blockDim.x) {
      const int32_t u = cur[q];
      const double finish = __dadd_rn(starts[u], cost[u]);
      for (int32_t e = off[u]; e < off[u + 1]; ++e) {
        const int32_t v = dst[e];
        atomic_max_nonneg(starts + v, __dadd_rn(finish, w[e]));
        if (atomicSub(indeg + v, 1) == 1) nxt[atomicAdd(&s_n_next, 1)] = v;
      }
    }
    __syncthreads();
    n_cur = s_n_next;
    int32_t* t = cur;
    cur = nxt;
    nxt = t;
  }
  __syncthreads();
  double m = 0.0;
  for (int32_t v = threadIdx.x; v < nv; v += blockDim.x)
    m = fmax(m, __dadd_rn(starts[v], cost[v]));
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double r = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) r = fmax(r, s_red[k]);
    *makespan = r;
    flags[0] = s_processed < nv ? 1 : 0;
    flags[1] = 0;
  }
  __syncthreads();
  // resource chains: sequential sum in creation order; on one resource the
  // start times are monotone along the chain, so chain order is time order
  // and the sorted event sweep of pipeline.py:522-539 is a linear scan
  for (int32_t k = threadIdx.x; k < n_chains; k += blockDim.x) {
    double acc = 0.0;
    int live = 0;
    bool over = false;
    for (int32_t v = chain_off[k]; v < chain_off[k + 1]; ++v) {
      acc = __dadd_rn(acc, cost[v]);
      if (kind) {
        if (kind[v] == 0) {
          if (capacity > 0 && ++live > capacity) over = true;
        } else if (kind[v] == 1 || kind[v] == 3) {
          --live;
        }
      }
    }
    if (chain_sum) chain_sum[k] = acc;
    if (over) atomicExch(flags + 1, 1);
  }
}

}  // namespace rh

using namespace rh;

extern "C" int rh_dag_critical_path(rh_ctx* ctx, int32_t n_vertices, const double* cost,
                                    const int32_t* succ_off, const int32_t* succ_dst,
                                    const double* succ_w, int32_t n_chains,
                                    const int32_t* chain_off, const uint8_t* kind,
                                    int32_t capacity, double* starts, double* makespan,
                                    double* chain_sum, int32_t* flags, void* stream) {
  if (!ctx || n_vertices < 0 || !makespan || !flags || !succ_off || n_chains < 0 ||
      (n_vertices && (!cost || !starts)) || (n_chains && !chain_off)) {
    set_error("rh_dag_critical_path: invalid arguments");
    return RH_E_INVALID;
  }
  DeviceGuard guard(ctx);
  void* ws = nullptr;
  const size_t per = ((size_t)n_vertices * sizeof(int32_t) + 255) & ~size_t(255);
  int rc = workspace(ctx, 3 * per + 256, &ws, 1, as_stream(stream));
  if (rc) return rc;
  int32_t* indeg = static_cast<int32_t*>(ws);
  int32_t* fa = reinterpret_cast<int32_t*>(static_cast<char*>(ws) + per);
  int32_t* fb = reinterpret_cast<int32_t*>(static_cast<char*>(ws) + 2 * per);
  dag_kernel<<<1, kDagThreads, 0, as_stream(stream)>>>(n_vertices, cost, succ_off, succ_dst,
                                                      succ_w, n_chains, chain_off, kind,
                                                      capacity, starts, makespan, chain_sum,
                                                      flags, indeg, fa, fb);
  RH_CHECK_LAUNCH(ctx);
  return RH_OK;
}
