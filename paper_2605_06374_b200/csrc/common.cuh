// Shared plumbing for the ResiHP B200 library: error state, context, launch
// accounting.  Every translation unit of libresihp_b200.so includes this.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <atomic>
#include <cstring>
#include <mutex>
#include <vector>
#include <string>

#include "../../include/resihp_b200.h"

struct rh_ctx {
  int device = 0;
  int num_sms = 148;
  size_t smem_optin = 0;
  std::atomic<int64_t> launches{0};
  // grow-only device workspaces, one per (slot, stream) so calls on distinct
  // streams never share scratch: slot 0 = host-buffer staging, slot 1 =
  // kernel scratch (screen kept-state, general DAG), slot 2 = rh_screen_prepare
  // results (reset indices, round-0 verdicts), slot 3 = the screen's
  // cooperative-kernel control words (zeroed on allocation; kernels leave
  // them zero).  A grown buffer is retired, never freed on the call path
  // (work still queued or a captured graph may reference it); retired
  // buffers are freed by rh_ctx_destroy.  ws_epoch counts reallocations and
  // is part of the host-pass graph key.
  struct Workspace {
    int slot;
    cudaStream_t stream;
    void* p;
    size_t bytes;
  };
  std::vector<Workspace> ws;
  std::vector<void*> ws_retired;
  uint64_t ws_epoch = 0;
  std::mutex ws_mu;
  // cached occupancies (per context, hence per device)
  int screen_occ = -1;
  int combine_occ = -1;
  // host-buffer entry points: copy stream + per-chunk events (lazily made)
  static constexpr int kChunkEvents = 8;
  cudaStream_t copy_stream = nullptr;
  // pinned staging of the host pass's small inputs (fill_small_stage)
  void* host_stage = nullptr;
  size_t host_stage_bytes = 0;
  std::vector<void*> host_stage_retired;
  cudaEvent_t chunk_ev[kChunkEvents] = {};
  // read-back stream of the host pass: chunk k's results cross PCIe while
  // later chunks (and the screen) run; done_ev[k] = chunk k's kernels finished
  cudaStream_t d2h_stream = nullptr;
  // per-call host entry points (rh_*_host): pinned in / out staging and the
  // stream they run on, one call at a time per context
  std::mutex call_mu;
  void* call_stage = nullptr;
  size_t call_stage_bytes = 0;
  cudaStream_t call_stream = nullptr;
  cudaEvent_t done_ev[kChunkEvents] = {};
  cudaEvent_t d2h_ev = nullptr;
  // side stream of the host pass (rh_screen_prepare while the trace streams in)
  cudaStream_t side_stream = nullptr;
  cudaEvent_t side_ev = nullptr;
  // per-(pp, schedule, max micro-batches) op-order tables of the
  // thread-per-replica pass kernel, built and uploaded on first use
  struct SchedTable {
    int pp, zbh, mmax;
    void* dev;
  };
  std::vector<SchedTable> sched;
  std::mutex sched_mu;
  // concurrent per-P launches of the search's table stage (fork / join)
  static constexpr int kAuxStreams = 4;
  cudaStream_t aux_stream[kAuxStreams] = {};
  cudaEvent_t aux_ev[kAuxStreams] = {};
  cudaEvent_t aux_fork = nullptr;
  std::mutex search_mu;  // serialises the enqueue of search evals (shared aux streams)
  // private stream-ordered pool of the re-plan searches (keeps what it has,
  // so a re-plan reuses memory instead of mapping it; the device's default
  // pool is left untouched)
  cudaMemPool_t pool = nullptr;
  // rh_detector_pass_host*: the captured pass for the last argument key
  struct HostGraph {
    std::vector<uint64_t> key;
    cudaGraphExec_t exec = nullptr;
    bool failed = false;
  } host_graph;
  // the last rh_screen_prepare: its arguments and completion event
  struct ScreenPrep {
    bool valid = false;
    int32_t window = 0, filter_enabled = 0;
    double kappa = 0.0;
    int64_t series_len = 0, n = 0;
    const void *hist = nullptr, *observed = nullptr, *reset = nullptr;
    void* buf = nullptr;  // the slot-2 buffer holding the results
    cudaEvent_t done = nullptr;
    // recorded after each rh_screen: the slot-2 results are free again
    cudaEvent_t consumed = nullptr;
    bool consumed_recorded = false;
  } prep;
  std::mutex prep_mu;  // guards prep (one pending prepare per context)
};

namespace rh {

void set_error(const char* fmt, ...);

inline int cuda_fail(cudaError_t e, const char* what) {
  set_error("%s: %s", what, cudaGetErrorString(e));
  return RH_E_CUDA;
}

#define RH_CUDA(call)                                   \
  do {                                                  \
    cudaError_t _e = (call);                            \
    if (_e != cudaSuccess) return rh::cuda_fail(_e, #call); \
  } while (0)

#define RH_CHECK_LAUNCH(ctx)                                        \
  do {                                                              \
    cudaError_t _e = cudaGetLastError();                            \
    if (_e != cudaSuccess) return rh::cuda_fail(_e, "kernel launch"); \
    (ctx)->launches.fetch_add(1, std::memory_order_relaxed);        \
  } while (0)

// The (slot, stream) workspace of at least `bytes` (see rh_ctx::ws).  Growth
// inside a stream capture is refused (a captured graph must not depend on a
// reallocation); zero = memset a newly allocated buffer on `stream`.
int workspace(rh_ctx* ctx, size_t bytes, void** out, int slot, cudaStream_t stream,
              bool zero = false);

// Makes ctx's device current for the lifetime of the guard and restores the
// caller's device afterwards (every entry point that touches the device).
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(const rh_ctx* ctx) {
    if (ctx && cudaGetDevice(&prev) == cudaSuccess && prev != ctx->device)
      cudaSetDevice(ctx->device);
    else
      prev = -1;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;
};

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) only when a kernel needs
// more than it was last granted on the context's device (the attribute is per
// device; the call costs microseconds per launch)
int ensure_smem(const rh_ctx* ctx, const void* kernel, size_t bytes);

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Doubles that are >= 0 order like their bit patterns (used by atomicMax).
__device__ __forceinline__ void atomic_max_nonneg(double* addr, double v) {
  atomicMax(reinterpret_cast<unsigned long long*>(addr),
            static_cast<unsigned long long>(__double_as_longlong(v)));
}


// The per-call host entry points (rh_*_host): the caller's host arrays are
// gathered into the context's pinned staging buffer, cross PCIe in ONE copy,
// the device entry point runs on the staged copies, and every output comes
// back in ONE copy -- instead of a synchronous copy per array (the drop-in
// API's scalar calls: quad_load, predict_chunk_time, validate, the screen of
// one DetectorState.observe).
struct HostCall {
  struct In {
    const void* src;
    size_t bytes, off;
  };
  struct Out {
    void* dst;
    size_t bytes, off;
  };
  std::vector<In> ins;
  std::vector<Out> outs;
  size_t in_bytes = 0, out_bytes = 0;
  static size_t up(size_t x) { return (x + 15) & ~size_t(15); }
  size_t in(const void* p, size_t b) {
    ins.push_back({p, b, in_bytes});
    in_bytes = up(in_bytes + b);
    return ins.back().off;
  }
  size_t out(void* p, size_t b) {
    outs.push_back({p, b, out_bytes});
    out_bytes = up(out_bytes + b);
    return outs.back().off;
  }
  // stage, copy in, launch(dev_in, dev_out, stream), copy out, wait, scatter
  template <class F>
  int run(rh_ctx* ctx, F&& launch) {
    std::lock_guard<std::mutex> lock(ctx->call_mu);
    const size_t total = in_bytes + out_bytes + 16;
    if (total > ctx->call_stage_bytes) {
      if (ctx->call_stage) RH_CUDA(cudaFreeHost(ctx->call_stage));
      ctx->call_stage = nullptr;
      ctx->call_stage_bytes = 0;
      const size_t want = total + total / 2 + 4096;
      RH_CUDA(cudaMallocHost(&ctx->call_stage, want));
      ctx->call_stage_bytes = want;
    }
    if (!ctx->call_stream)
      RH_CUDA(cudaStreamCreateWithFlags(&ctx->call_stream, cudaStreamNonBlocking));
    cudaStream_t st = ctx->call_stream;
    void* dev = nullptr;
    if (int rc = workspace(ctx, total, &dev, 5, st)) return rc;
    char* h = static_cast<char*>(ctx->call_stage);
    for (const In& a : ins)
      if (a.src && a.bytes) memcpy(h + a.off, a.src, a.bytes);
    char* d_in = static_cast<char*>(dev);
    char* d_out = d_in + in_bytes;
    if (in_bytes) RH_CUDA(cudaMemcpyAsync(d_in, h, in_bytes, cudaMemcpyHostToDevice, st));
    if (int rc = launch(d_in, d_out, st)) return rc;
    if (out_bytes)
      RH_CUDA(cudaMemcpyAsync(h + in_bytes, d_out, out_bytes, cudaMemcpyDeviceToHost, st));
    RH_CUDA(cudaStreamSynchronize(st));
    for (const Out& o : outs)
      if (o.dst && o.bytes) memcpy(o.dst, h + in_bytes + o.off, o.bytes);
    return RH_OK;
  }
};

}  // namespace rh
