// Context, error reporting and the small batch kernels of the C ABI:
// quad_load (workload.py:83-85), predict_chunk_time (workload.py:88-98) and
// validate (detector.py:127-158).
#include <stdarg.h>

#include <mutex>
#include <unordered_map>

#include "common.cuh"

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

int workspace(rh_ctx* ctx, size_t bytes, void** out, int slot) {
  if (bytes > ctx->ws_bytes[slot]) {
    if (ctx->ws[slot]) {
      RH_CUDA(cudaDeviceSynchronize());
      RH_CUDA(cudaFree(ctx->ws[slot]));
      ctx->ws[slot] = nullptr;
      ctx->ws_bytes[slot] = 0;
    }
    size_t want = bytes + bytes / 4 + (1u << 20);
    cudaError_t e = cudaMalloc(&ctx->ws[slot], want);
    if (e != cudaSuccess) {
      set_error("workspace of %zu bytes: %s", want, cudaGetErrorString(e));
      return RH_E_NOMEM;
    }
    ctx->ws_bytes[slot] = want;
  }
  *out = ctx->ws[slot];
  return RH_OK;
}

int ensure_smem(const void* kernel, size_t bytes) {
  static std::mutex mu;
  static std::unordered_map<const void*, size_t> granted;
  std::lock_guard<std::mutex> lock(mu);
  auto it = granted.find(kernel);
  if (it != granted.end() && it->second >= bytes) return RH_OK;
  RH_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  granted[kernel] = bytes;
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
  double base = __dadd_rn(__dmul_rn(m.alpha, (double)budget[i]),
                          __dmul_rn(m.beta, (double)quad[i]));
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

}  // namespace rh

using namespace rh;

extern "C" {

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
  RH_CUDA(cudaSetDevice(device));
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
  for (void* w : ctx->ws)
    if (w) cudaFree(w);
  for (cudaEvent_t e : ctx->chunk_ev)
    if (e) cudaEventDestroy(e);
  if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
  if (ctx->side_stream) cudaStreamDestroy(ctx->side_stream);
  if (ctx->side_ev) cudaEventDestroy(ctx->side_ev);
  for (auto& t : ctx->sched) cudaFree(t.dev);
  if (ctx->prep.done) cudaEventDestroy(ctx->prep.done);
  if (ctx->prep.consumed) cudaEventDestroy(ctx->prep.consumed);
  if (ctx->host_graph.exec) cudaGraphExecDestroy(ctx->host_graph.exec);
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
  int th = 256;
  chunk_time_kernel<<<(unsigned)((n + th - 1) / th), th, 0, as_stream(stream)>>>(
      *model, n, quad, budget, kind, layers, speed, t_out, bad_out);
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
  int th = 256;
  validate_kernel<<<(unsigned)((n + th - 1) / th), th, 0, as_stream(stream)>>>(
      n, measured, expected, threshold, flag, severity);
  RH_CHECK_LAUNCH(ctx);
  return RH_OK;
}

}  // extern "C"
