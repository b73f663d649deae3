// Context, error reporting and the small batch kernels of the C ABI:
// quad_load (workload.py:83-85), predict_chunk_time (workload.py:88-98) and
// validate (detector.py:127-158).
#include <stdarg.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "common.cuh"
#include "wavefront.cuh"

namespace {
thread_local char g_err[1024] = "";
}

namespace rh {

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int workspace(rh_ctx* ctx, size_t bytes, void** out, int slot, cudaStream_t stream, bool zero) {
  std::lock_guard<std::mutex> lock(ctx->ws_mu);
  rh_ctx::Workspace* w = nullptr;
  for (auto& x : ctx->ws)
    if (x.slot == slot && x.stream == stream) w = &x;
  if (w && w->bytes >= bytes) {
    *out = w->p;
    return RH_OK;
  }
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  RH_CUDA(cudaStreamIsCapturing(stream, &cap));
  if (cap != cudaStreamCaptureStatusNone) {
    set_error("workspace growth to %zu bytes inside a stream capture: run the call once "
              "outside the capture first", bytes);
    return RH_E_INVALID;
  }
  const size_t want = bytes + bytes / 4 + (1u << 20);
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, want);
  if (e != cudaSuccess) {
    set_error("workspace of %zu bytes: %s", want, cudaGetErrorString(e));
    return RH_E_NOMEM;
  }
  if (zero) RH_CUDA(cudaMemsetAsync(p, 0, want, stream));
  if (w) {  // queued work or a captured graph may still use the old buffer
    ctx->ws_retired.push_back(w->p);
    w->p = p;
    w->bytes = want;
  } else {
    ctx->ws.push_back({slot, stream, p, want});
  }
  ++ctx->ws_epoch;
  *out = p;
  return RH_OK;
}

int ensure_smem(const rh_ctx* ctx, const void* kernel, size_t bytes) {
  static std::mutex mu;
  static std::unordered_map<const void*, size_t> granted[64];  // per device ordinal
  if (bytes <= 48 * 1024) return RH_OK;  // the default limit
  std::lock_guard<std::mutex> lock(mu);
  auto& g = granted[ctx->device & 63];
  auto it = g.find(kernel);
  if (it != g.end() && it->second >= bytes) return RH_OK;
  RH_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  g[kernel] = bytes;
  return RH_OK;
}

// ---------------------------------------------------------------- kernels

// One thread per micro-batch: Q_j = sum l^2 in int64 (exact; Python bigint).
__global__ void quad_load_kernel(int64_t n, const int32_t* __restrict__ off,
                                 const int32_t* __restrict__ len,
                                 int64_t* __restrict__ out) {
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  int32_t a = off[j], b = off[j + 1];
  int64_t q = 0;
  for (int32_t k = a; k < b; ++k) {
    int64_t l = len[k];
    q += l * l;
  }
  out[j] = q;
}

__global__ void chunk_time_kernel(rh_cost_model m, int64_t n,
                                  const int64_t* __restrict__ quad,
                                  const int64_t* __restrict__ mb_idx,  // nullable: quad[mb_idx[i]]
                                  const int32_t* __restrict__ budget,
                                  const uint8_t* __restrict__ kind,
                                  const int32_t* __restrict__ layers,
                                  const double* __restrict__ speed,
                                  double* __restrict__ t, uint8_t* __restrict__ bad) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double sp = speed[i];
  if (sp <= 0.0) {  // workload.py:95-96
    t[i] = 0.0;
    if (bad) bad[i] = 1;
    return;
  }
  int k = kind[i];
  double ratio = k == 0 ? m.ratio_f : k == 1 ? m.ratio_b : k == 2 ? m.ratio_w
                                                          : m.ratio_b + m.ratio_w;
  // ((ratio * L) * (alpha*N + beta*Q)) / speed, two roundings per a*b+c
  const int64_t q = mb_idx ? quad[mb_idx[i]] : quad[i];
  double base = __dadd_rn(__dmul_rn(m.alpha, (double)budget[i]), __dmul_rn(m.beta, (double)q));
  double num = __dmul_rn(__dmul_rn(ratio, (double)layers[i]), base);
  t[i] = sp == 1.0 ? num : __ddiv_rn(num, sp);
  if (bad) bad[i] = 0;
}

__global__ void validate_kernel(int64_t n, const double* __restrict__ meas,
                                const double* __restrict__ expd, double thr,
                                uint8_t* __restrict__ flag, double* __restrict__ sev) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double m = meas[i];
  uint8_t f = 0;
  double s = 0.0;
  if (expd) {
    double e = expd[i];
    if (!(e <= 0.0 || m <= 0.0) && m > __dmul_rn(thr, e)) {
      f = 1;
      s = __ddiv_rn(e, m);
    }
  } else if (m > thr) {
    f = 1;
    s = __ddiv_rn(1.0, m);
  }
  flag[i] = f;
  sev[i] = s;
}

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

// div_recip (hoisted-reciprocal division) against __ddiv_rn over regimes of
// divisors: random in (0, 1], k / 2^m fractions (TP-subgroup speeds), random
// severities, all-ones mantissas, 1 - ulp, and wide exponents for both.
__global__ void selftest_div_kernel(int64_t n, uint64_t seed, unsigned long long* bad) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t h1 = splitmix64(seed ^ (uint64_t)i), h2 = splitmix64(h1 ^ 0x5bd1e995ull);
    const uint64_t mant_a = h1 & 0xfffffffffffffull, mant_b = h2 & 0xfffffffffffffull;
    const int ea = (int)((h1 >> 52) % 200) - 120;  // a in [2^-120, 2^80)
    double a = __longlong_as_double((long long)(((uint64_t)(1023 + ea) << 52) | mant_a));
    double b;
    switch ((h2 >> 52) & 7) {
      case 0: b = __longlong_as_double((long long)((1022ull << 52) | mant_b)); break;  // [0.5,1)
      case 1: b = (double)(1 + (h2 >> 56) % 8) / 8.0; break;                          // k/8
      case 2: b = 0.3 + 0.4 * (double)(mant_b >> 20) / (double)(1ull << 32); break;     // severity
      case 3: b = __longlong_as_double((long long)(((uint64_t)(1023 - (int)((h2 >> 56) % 30)) << 52) |
                                                   0xfffffffffffffull)); break;     // all-ones
      case 4: b = 1.0 - 0x1p-53 * (double)(1 + (h2 >> 60)); break;                   // 1 - k ulp
      case 5: b = __longlong_as_double((long long)(((uint64_t)(1023 - (int)((h2 >> 56) % 90)) << 52) |
                                                   mant_b)); break;  // [2^-89, 2)
      case 6: b = 1.0; break;
      default: b = (double)(1 + (h2 >> 56) % 7) / 7.0; a = b * (double)(1 + (h1 >> 60)); break;
    }
    const double q1 = div_recip(a, b, recip_of(b));
    const double q2 = __ddiv_rn(a, b);
    if (__double_as_longlong(q1) != __double_as_longlong(q2)) atomicAdd(bad, 1ull);
  }
}

}  // namespace rh

using namespace rh;

extern "C" {

int rh_selftest_division(rh_ctx* ctx, int64_t n, uint64_t seed, int64_t* mismatches) {
  if (!ctx || n < 0 || !mismatches) {
    set_error("rh_selftest_division: invalid arguments");
    return RH_E_INVALID;
  }
  DeviceGuard guard(ctx);
  unsigned long long* d = nullptr;
  RH_CUDA(cudaMalloc(&d, sizeof(unsigned long long)));
  RH_CUDA(cudaMemset(d, 0, sizeof(unsigned long long)));
  selftest_div_kernel<<<ctx->num_sms * 8, 256>>>(n, seed, d);
  cudaError_t e = cudaGetLastError();
  unsigned long long h = 0;
  if (e == cudaSuccess) e = cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) return cuda_fail(e, "rh_selftest_division");
  *mismatches = (int64_t)h;
  return RH_OK;
}

// FP64 pipe peak: 8 independent DFMA chains per thread, 4 x 256-thread CTAs
// per SM -- enough independent work to saturate the pipe.  The roofline
// denominator of the search kernels (bench.py); one fp64 instruction (add,
// mul, compare, fma) per slot.
__global__ void __launch_bounds__(256) fp64_peak_kernel(int iters, double seed, double* sink) {
  double a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = seed + threadIdx.x * 1e-9 + k;
  const double m = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = __fma_rn(a[k], m, c);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 12345.678) *sink = s;  // keeps the chains live
}

int rh_fp64_peak(rh_ctx* ctx, double* instr_per_s) {
  if (!ctx || !instr_per_s) {
    set_error("rh_fp64_peak: invalid arguments");
    return RH_E_INVALID;
  }
  DeviceGuard guard(ctx);
  double* sink = nullptr;
  RH_CUDA(cudaMalloc(&sink, sizeof(double)));
  cudaEvent_t e0, e1;
  RH_CUDA(cudaEventCreate(&e0));
  RH_CUDA(cudaEventCreate(&e1));
  const int blocks = ctx->num_sms * 4, iters = 1 << 14;
  fp64_peak_kernel<<<blocks, 256>>>(iters / 8, 1.0, sink);  // warm-up
  RH_CUDA(cudaEventRecord(e0));
  fp64_peak_kernel<<<blocks, 256>>>(iters, 1.0, sink);
  RH_CUDA(cudaEventRecord(e1));
  cudaError_t e = cudaEventSynchronize(e1);
  float ms = 0.f;
  if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(sink);
  if (e != cudaSuccess) return cuda_fail(e, "rh_fp64_peak");
  *instr_per_s = (double)blocks * 256.0 * 8.0 * iters / (ms * 1e-3);
  return RH_OK;
}

int rh_abi_version(void) { return RH_ABI_VERSION; }

const char* rh_last_error(void) { return g_err; }

int rh_ctx_create(int device, rh_ctx** out) {
  if (!out) {
    set_error("rh_ctx_create: out is NULL");
    return RH_E_INVALID;
  }
  int n = 0;
  RH_CUDA(cudaGetDeviceCount(&n));
  if (device < 0 || device >= n) {
    set_error("rh_ctx_create: device %d out of range (%d devices)", device, n);
    return RH_E_INVALID;
  }
  // the caller's current device is left as it was
  cudaDeviceProp prop;
  RH_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10) {
    set_error("rh_ctx_create: device %d is sm_%d%d; this library is built for sm_100a",
              device, prop.major, prop.minor);
    return RH_E_INVALID;
  }
  rh_ctx* c = new rh_ctx();
  c->device = device;
  c->num_sms = prop.multiProcessorCount;
  c->smem_optin = prop.sharedMemPerBlockOptin;
  *out = c;
  return RH_OK;
}

int rh_ctx_destroy(rh_ctx* ctx) {
  if (!ctx) return RH_OK;
  DeviceGuard guard(ctx);
  cudaDeviceSynchronize();  // nothing queued may still use the context's memory
  for (auto& w : ctx->ws)
    if (w.p) cudaFree(w.p);
  for (void* p : ctx->ws_retired) cudaFree(p);
  for (cudaEvent_t e : ctx->chunk_ev)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : ctx->done_ev)
    if (e) cudaEventDestroy(e);
  if (ctx->d2h_ev) cudaEventDestroy(ctx->d2h_ev);
  if (ctx->d2h_stream) cudaStreamDestroy(ctx->d2h_stream);
  if (ctx->call_stream) cudaStreamDestroy(ctx->call_stream);
  if (ctx->call_stage) cudaFreeHost(ctx->call_stage);
  if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
  if (ctx->side_stream) cudaStreamDestroy(ctx->side_stream);
  if (ctx->side_ev) cudaEventDestroy(ctx->side_ev);
  for (auto& t : ctx->sched) cudaFree(t.dev);
  if (ctx->prep.done) cudaEventDestroy(ctx->prep.done);
  if (ctx->prep.consumed) cudaEventDestroy(ctx->prep.consumed);
  if (ctx->host_graph.exec) cudaGraphExecDestroy(ctx->host_graph.exec);
  for (int q = 0; q < rh_ctx::kAuxStreams; ++q) {
    if (ctx->aux_stream[q]) cudaStreamDestroy(ctx->aux_stream[q]);
    if (ctx->aux_ev[q]) cudaEventDestroy(ctx->aux_ev[q]);
  }
  if (ctx->aux_fork) cudaEventDestroy(ctx->aux_fork);
  if (ctx->pool) cudaMemPoolDestroy(ctx->pool);
  if (ctx->host_stage) cudaFreeHost(ctx->host_stage);
  for (void* p : ctx->host_stage_retired) cudaFreeHost(p);
  delete ctx;
  return RH_OK;
}

int64_t rh_ctx_launches(const rh_ctx* ctx) { return ctx ? ctx->launches.load() : 0; }

int rh_quad_load(rh_ctx* ctx, int64_t n_mb, const int32_t* mb_off,
                 const int32_t* doc_len, int64_t* quad_out, void* stream) {
  if (!ctx || n_mb < 0 || (n_mb && (!mb_off || !doc_len || !quad_out))) {
    set_error("rh_quad_load: invalid arguments");
    return RH_E_INVALID;
  }
  if (n_mb == 0) return RH_OK;
  DeviceGuard guard(ctx);
  int th = 256;
  quad_load_kernel<<<(unsigned)((n_mb + th - 1) / th), th, 0, as_stream(stream)>>>(
      n_mb, mb_off, doc_len, quad_out);
  RH_CHECK_LAUNCH(ctx);
  return RH_OK;
}

int rh_chunk_time(rh_ctx* ctx, const rh_cost_model* model, int64_t n,
                  const int64_t* quad, const int32_t* budget, const uint8_t* kind,
                  const int32_t* layers, const double* speed, double* t_out,
                  uint8_t* bad_out, void* stream) {
  if (!ctx || !model || n < 0) {
    set_error("rh_chunk_time: invalid arguments");
    return RH_E_INVALID;
  }
  if (n == 0) return RH_OK;
  DeviceGuard guard(ctx);
  int th = 256;
  chunk_time_kernel<<<(unsigned)((n + th - 1) / th), th, 0, as_stream(stream)>>>(
      *model, n, quad, nullptr, budget, kind, layers, speed, t_out, bad_out);
  RH_CHECK_LAUNCH(ctx);
  return RH_OK;
}

int rh_validate(rh_ctx* ctx, int64_t n, const double* measured, const double* expected,
                double threshold, uint8_t* flag, double* severity, void* stream) {
  if (!ctx || n < 0 || (n && (!measured || !flag || !severity))) {
    set_error("rh_validate: invalid arguments");
    return RH_E_INVALID;
  }
  if (n == 0) return RH_OK;
  DeviceGuard guard(ctx);
  int th = 256;
  validate_kernel<<<(unsigned)((n + th - 1) / th), th, 0, as_stream(stream)>>>(
      n, measured, expected, threshold, flag, severity);
  RH_CHECK_LAUNCH(ctx);
  return RH_OK;
}


}  // extern "C"

extern "C" {

int rh_quad_load_host(rh_ctx* ctx, int64_t n_mb, const int32_t* mb_off, const int32_t* doc_len,
                      int64_t* quad_out) {
  if (!ctx || n_mb < 0 || (n_mb && (!mb_off || !quad_out))) {
    set_error("rh_quad_load_host: invalid arguments");
    return RH_E_INVALID;
  }
  if (n_mb == 0) return RH_OK;
  const int64_t n_doc = mb_off[n_mb];
  if (n_doc < 0 || (n_doc && !doc_len)) {
    set_error("rh_quad_load_host: invalid offsets / documents");
    return RH_E_INVALID;
  }
  DeviceGuard guard(ctx);
  HostCall c;
  const size_t o_off = c.in(mb_off, 4 * (size_t)(n_mb + 1));
  const size_t o_doc = c.in(doc_len, 4 * (size_t)n_doc);
  const size_t o_q = c.out(quad_out, 8 * (size_t)n_mb);
  return c.run(ctx, [&](char* din, char* dout, cudaStream_t st) {
    return rh_quad_load(ctx, n_mb, reinterpret_cast<const int32_t*>(din + o_off),
                        reinterpret_cast<const int32_t*>(din + o_doc),
                        reinterpret_cast<int64_t*>(dout + o_q), st);
  });
}

int rh_chunk_time_host(rh_ctx* ctx, const rh_cost_model* model, int64_t n, const int64_t* quad,
                       const int32_t* budget, const uint8_t* kind, const int32_t* layers,
                       const double* speed, double* t_out, uint8_t* bad_out) {
  if (!ctx || !model || n < 0 ||
      (n && (!quad || !budget || !kind || !layers || !speed || !t_out))) {
    set_error("rh_chunk_time_host: invalid arguments");
    return RH_E_INVALID;
  }
  if (n == 0) return RH_OK;
  DeviceGuard guard(ctx);
  HostCall c;
  const size_t oq = c.in(quad, 8 * (size_t)n), ob = c.in(budget, 4 * (size_t)n),
               ok = c.in(kind, (size_t)n), ol = c.in(layers, 4 * (size_t)n),
               os = c.in(speed, 8 * (size_t)n);
  const size_t ot = c.out(t_out, 8 * (size_t)n);
  // bad flags start zero: they travel in with the inputs' zeroed tail
  std::vector<uint8_t> zeros(bad_out ? (size_t)n : 0, 0);
  const size_t oz = c.in(zeros.data(), zeros.size());
  const size_t obad = c.out(bad_out, bad_out ? (size_t)n : 0);
  return c.run(ctx, [&](char* din, char* dout, cudaStream_t st) {
    uint8_t* bad = bad_out ? reinterpret_cast<uint8_t*>(dout + obad) : nullptr;
    if (bad) RH_CUDA(cudaMemcpyAsync(bad, din + oz, (size_t)n, cudaMemcpyDeviceToDevice, st));
    return rh_chunk_time(ctx, model, n, reinterpret_cast<const int64_t*>(din + oq),
                         reinterpret_cast<const int32_t*>(din + ob),
                         reinterpret_cast<const uint8_t*>(din + ok),
                         reinterpret_cast<const int32_t*>(din + ol),
                         reinterpret_cast<const double*>(din + os),
                         reinterpret_cast<double*>(dout + ot), bad, st);
  });
}

int rh_validate_host(rh_ctx* ctx, int64_t n, const double* measured, const double* expected,
                     double threshold, uint8_t* flag, double* severity) {
  if (!ctx || n < 0 || (n && (!measured || !flag || !severity))) {
    set_error("rh_validate_host: invalid arguments");
    return RH_E_INVALID;
  }
  if (n == 0) return RH_OK;
  DeviceGuard guard(ctx);
  HostCall c;
  const size_t om = c.in(measured, 8 * (size_t)n);
  const size_t oe = c.in(expected, expected ? 8 * (size_t)n : 0);
  const size_t of = c.out(flag, (size_t)n), os = c.out(severity, 8 * (size_t)n);
  return c.run(ctx, [&](char* din, char* dout, cudaStream_t st) {
    return rh_validate(ctx, n, reinterpret_cast<const double*>(din + om),
                       expected ? reinterpret_cast<const double*>(din + oe) : nullptr, threshold,
                       reinterpret_cast<uint8_t*>(dout + of),
                       reinterpret_cast<double*>(dout + os), st);
  });
}

int rh_screen_host(rh_ctx* ctx, const rh_screen_params* params, int64_t series_len,
                   const double* hist, int64_t n, const double* observed,
                   const uint8_t* it_status, const uint8_t* reset, uint8_t* outcome,
                   int64_t* series_len_out) {
  if (!ctx || !params || n < 0 || series_len < 0 || (n && (!observed || !it_status || !outcome)) ||
      (series_len > 0 && !hist)) {
    set_error("rh_screen_host: invalid arguments");
    return RH_E_INVALID;
  }
  DeviceGuard guard(ctx);
  const int64_t h = std::min<int64_t>(series_len, params->window > 0 ? params->window : 0);
  HostCall c;
  // hist holds the last min(series_len, window) series values
  const size_t oh = c.in(h ? hist : nullptr, 8 * (size_t)h);
  const size_t oo = c.in(observed, 8 * (size_t)n), os = c.in(it_status, (size_t)n);
  const size_t orr = c.in(reset, reset ? (size_t)n : 0);
  const size_t ooc = c.out(outcome, (size_t)n);
  const size_t olen = c.out(series_len_out, series_len_out ? 8 : 0);
  return c.run(ctx, [&](char* din, char* dout, cudaStream_t st) {
    const double* dh = reinterpret_cast<const double*>(din + oh);
    return rh_screen(ctx, params, series_len, h ? dh : nullptr, n,
                     reinterpret_cast<const double*>(din + oo),
                     reinterpret_cast<const uint8_t*>(din + os),
                     reset ? reinterpret_cast<const uint8_t*>(din + orr) : nullptr,
                     reinterpret_cast<uint8_t*>(dout + ooc),
                     series_len_out ? reinterpret_cast<int64_t*>(dout + olen) : nullptr, st);
  });
}

int rh_dag_critical_path_host(rh_ctx* ctx, int32_t n_vertices, const double* cost,
                              const int32_t* succ_off, const int32_t* succ_dst,
                              const double* succ_w, int32_t n_chains, const int32_t* chain_off,
                              const uint8_t* kind, int32_t capacity, double* starts,
                              double* makespan, double* chain_sum, int32_t* flags) {
  if (!ctx || n_vertices < 0 || !makespan || !flags || !succ_off || n_chains < 0 ||
      (n_vertices && (!cost || !starts)) || (n_chains && (!chain_off || !chain_sum))) {
    set_error("rh_dag_critical_path_host: invalid arguments");
    return RH_E_INVALID;
  }
  const int64_t ne = succ_off[n_vertices];
  if (ne < 0 || (ne && (!succ_dst || !succ_w))) {
    set_error("rh_dag_critical_path_host: invalid successor lists");
    return RH_E_INVALID;
  }
  DeviceGuard guard(ctx);
  HostCall c;
  const size_t oc = c.in(cost, 8 * (size_t)n_vertices);
  const size_t oo = c.in(succ_off, 4 * ((size_t)n_vertices + 1));
  const size_t od = c.in(succ_dst, 4 * (size_t)ne), ow = c.in(succ_w, 8 * (size_t)ne);
  const size_t och = c.in(chain_off, n_chains ? 4 * ((size_t)n_chains + 1) : 0);
  const size_t ok = c.in(kind, kind ? (size_t)n_vertices : 0);
  const size_t os = c.out(starts, 8 * (size_t)n_vertices), om = c.out(makespan, 8);
  const size_t osum = c.out(chain_sum, 8 * (size_t)n_chains), of = c.out(flags, 8);
  return c.run(ctx, [&](char* din, char* dout, cudaStream_t st) {
    RH_CUDA(cudaMemsetAsync(dout + of, 0, 8, st));
    return rh_dag_critical_path(
        ctx, n_vertices, reinterpret_cast<const double*>(din + oc),
        reinterpret_cast<const int32_t*>(din + oo), reinterpret_cast<const int32_t*>(din + od),
        reinterpret_cast<const double*>(din + ow), n_chains,
        n_chains ? reinterpret_cast<const int32_t*>(din + och) : nullptr,
        kind ? reinterpret_cast<const uint8_t*>(din + ok) : nullptr, capacity,
        reinterpret_cast<double*>(dout + os), reinterpret_cast<double*>(dout + om),
        n_chains ? reinterpret_cast<double*>(dout + osum) : nullptr,
        reinterpret_cast<int32_t*>(dout + of), st);
  });
}

int rh_pipeline_batch_host(rh_ctx* ctx, const rh_pipe_shape* shape, const rh_cost_model* model,
                           const rh_segments* segs, const rh_trace* trace,
                           const rh_pass_out* out) {
  if (!ctx || !shape || !model || !segs || !trace || !out || !out->makespan || !out->status ||
      !trace->mb_off || segs->n_seg < 1 || trace->n_iter < 0) {
    set_error("rh_pipeline_batch_host: invalid arguments");
    return RH_E_INVALID;
  }
  const int64_t n = trace->n_iter, S = segs->n_seg;
  if (n == 0) return RH_OK;
  const int64_t P = shape->pp, D = shape->dp, M = shape->micro_batches, G = D * P;
  if (P < 1 || D < 1 || M < 1) {
    set_error("rh_pipeline_batch_host: invalid shape");
    return RH_E_INVALID;
  }
  const int64_t n_docs = trace->mb_off[n * M];
  const int64_t n_links = segs->link_off ? segs->link_off[S] : 0;
  DeviceGuard guard(ctx);
  HostCall c;
  const size_t o_lay = c.in(segs->layers, 4 * S * P), o_mbs = c.in(segs->mb_start, 4 * S * (D + 1)),
               o_sp = c.in(segs->speed, 8 * S * G), o_hf = c.in(segs->hop_fwd, 8 * S * G),
               o_hb = c.in(segs->hop_bwd, 8 * S * G),
               o_ar = c.in(segs->allreduce, segs->allreduce ? 8 * S * D : 0),
               o_lo = c.in(segs->link_off, segs->link_off ? 4 * (S + 1) : 0),
               o_lr = c.in(segs->link_ratio, segs->link_off ? 8 * n_links : 0),
               o_lm = c.in(segs->link_max, segs->link_off && segs->link_max ? 8 * S : 0);
  const size_t o_seg = c.in(trace->seg, trace->seg ? 4 * n : 0),
               o_off = c.in(trace->mb_off, 4 * (n * M + 1)), o_doc = c.in(trace->doc_len, 4 * n_docs);
  const size_t o_ms = c.out(out->makespan, 8 * n), o_st = c.out(out->status, n),
               o_sc = c.out(out->stage_cost, out->stage_cost ? 8 * n * G : 0);
  return c.run(ctx, [&](char* din, char* dout, cudaStream_t st) {
    rh_segments ds = *segs;
    ds.layers = reinterpret_cast<const int32_t*>(din + o_lay);
    ds.mb_start = reinterpret_cast<const int32_t*>(din + o_mbs);
    ds.speed = reinterpret_cast<const double*>(din + o_sp);
    ds.hop_fwd = reinterpret_cast<const double*>(din + o_hf);
    ds.hop_bwd = reinterpret_cast<const double*>(din + o_hb);
    ds.allreduce = segs->allreduce ? reinterpret_cast<const double*>(din + o_ar) : nullptr;
    ds.link_off = segs->link_off ? reinterpret_cast<const int32_t*>(din + o_lo) : nullptr;
    ds.link_ratio = segs->link_off ? reinterpret_cast<const double*>(din + o_lr) : nullptr;
    ds.link_max = segs->link_off && segs->link_max ? reinterpret_cast<const double*>(din + o_lm)
                                                   : nullptr;
    rh_trace dt = *trace;
    dt.seg = trace->seg ? reinterpret_cast<const int32_t*>(din + o_seg) : nullptr;
    dt.mb_off = reinterpret_cast<const int32_t*>(din + o_off);
    dt.doc_len = reinterpret_cast<const int32_t*>(din + o_doc);
    dt.device_time = nullptr;
    dt.observed = nullptr;
    rh_pass_out dout_ = {};
    dout_.makespan = reinterpret_cast<double*>(dout + o_ms);
    dout_.status = reinterpret_cast<uint8_t*>(dout + o_st);
    dout_.stage_cost = out->stage_cost ? reinterpret_cast<double*>(dout + o_sc) : nullptr;
    return rh_pipeline_batch(ctx, shape, model, &ds, &dt, &dout_, st);
  });
}

int rh_chunk_time_docs_host(rh_ctx* ctx, const rh_cost_model* model, int64_t n_mb,
                            const int32_t* mb_off, const int32_t* doc_len, int64_t n,
                            const int64_t* mb_idx, const int32_t* budget, const uint8_t* kind,
                            const int32_t* layers, const double* speed, double* t_out,
                            uint8_t* bad_out) {
  if (!ctx || !model || n_mb < 1 || n < 0 || !mb_off ||
      (n && (!mb_idx || !budget || !kind || !layers || !speed || !t_out || !bad_out))) {
    set_error("rh_chunk_time_docs_host: invalid arguments");
    return RH_E_INVALID;
  }
  if (n == 0) return RH_OK;
  const int64_t n_doc = mb_off[n_mb];
  if (n_doc < 0 || (n_doc && !doc_len)) {
    set_error("rh_chunk_time_docs_host: invalid offsets / documents");
    return RH_E_INVALID;
  }
  for (int64_t i = 0; i < n; ++i)
    if (mb_idx[i] < 0 || mb_idx[i] >= n_mb) {
      set_error("rh_chunk_time_docs_host: micro-batch index out of range");
      return RH_E_INVALID;
    }
  DeviceGuard guard(ctx);
  HostCall c;
  const size_t o_off = c.in(mb_off, 4 * (size_t)(n_mb + 1)), o_doc = c.in(doc_len, 4 * (size_t)n_doc),
               o_idx = c.in(mb_idx, 8 * (size_t)n), o_b = c.in(budget, 4 * (size_t)n),
               o_k = c.in(kind, (size_t)n), o_l = c.in(layers, 4 * (size_t)n),
               o_s = c.in(speed, 8 * (size_t)n);
  const size_t o_t = c.out(t_out, 8 * (size_t)n), o_bad = c.out(bad_out, (size_t)n);
  const size_t o_q = c.out(nullptr, 8 * (size_t)n_mb);  // device scratch: the quad loads
  return c.run(ctx, [&](char* din, char* dout, cudaStream_t st) -> int {
    int64_t* q = reinterpret_cast<int64_t*>(dout + o_q);
    if (int rc = rh_quad_load(ctx, n_mb, reinterpret_cast<const int32_t*>(din + o_off),
                              reinterpret_cast<const int32_t*>(din + o_doc), q, st))
      return rc;
    const int th = 256;
    chunk_time_kernel<<<(unsigned)((n + th - 1) / th), th, 0, st>>>(
        *model, n, q, reinterpret_cast<const int64_t*>(din + o_idx),
        reinterpret_cast<const int32_t*>(din + o_b), reinterpret_cast<const uint8_t*>(din + o_k),
        reinterpret_cast<const int32_t*>(din + o_l), reinterpret_cast<const double*>(din + o_s),
        reinterpret_cast<double*>(dout + o_t), reinterpret_cast<uint8_t*>(dout + o_bad));
    RH_CHECK_LAUNCH(ctx);
    return RH_OK;
  });
}

}  // extern "C"
