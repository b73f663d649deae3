// Fused pipeline predictor + Detector residual pass (rh_pipeline_batch,
// rh_detect_batch, rh_detect_batch_host).
//
// What it computes, per iteration i of the batch:
//   Q_j   = sum of squared doc lengths of micro-batch j      (workload.py:83-85)
//   c(v)  = ((ratio(kind)*L_s) * (alpha*N + beta*Q_j)) / p   (workload.py:88-98)
//   start(v) = max(finish(chain predecessor), finish(data predecessor) + hop)
//   makespan = max_d ( max_s finish(last chunk of (d,s)) + AR_d )
//              — the critical path of build_dag's canonical DAG
//              (pipeline.py:129-292), evaluated as a wavefront
//   stage_cost[d][s] = sum of c(v) over the (d,s) chain, in chain order
//              (pipeline.py:446-453)
//   detect: filter verdict observed > thr*makespan (detector.py:111-116) and
//           per-(d,s) flag measured > thr*stage_cost, severity
//           stage_cost/measured (detector.py:127-158), measured = max over
//           the group's member device times (float4 loads).
//
// Mapping (B200): one replica pipeline = `pw` lanes (pw = next_pow2(P) <= 32,
// lane s = stage s), so a warp runs 32/pw pipelines; all D pipelines of an
// iteration sit in one CTA and reduce the makespan through shared memory.
// Each lane walks its stage's 1F1B/ZBH chain in order; a chunk whose data
// predecessor lives on a neighbouring stage waits until that lane has
// published the finish time in shared memory (dynamic wavefront, one
// __syncwarp per step).  The canonical DAG is acyclic, so the chain head of
// the earliest unprocessed vertex is always ready and the loop terminates.
// All fp64 ops use explicit _rn intrinsics: no FMA contraction anywhere.
#include <algorithm>

#include "common.cuh"
#include "wavefront.cuh"

namespace rh {

struct PassParams {
  rh_pipe_shape sh;
  rh_cost_model m;
  rh_segments sg;
  rh_trace tr;
  rh_pass_out out;
  double thr;
  int pw, log_pw;  // lanes per pipeline
  int lpi;         // lanes per iteration = D * pw
  int ipb;         // iterations per CTA
  int mmax;        // micro-batches per replica (smem row length)
  int vec4;        // device_time rows are float4-aligned
};

template <int ZBH, int DETECT>
__global__ void __launch_bounds__(1024) pass_kernel(const PassParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tid = threadIdx.x;
  const int P = p.sh.pp, D = p.sh.dp, M = p.sh.micro_batches, T = p.sh.tp;
  const int li = tid / p.lpi;
  const int within = tid - li * p.lpi;
  const int d = within >> p.log_pw;
  const int s = within & (p.pw - 1);
  const int64_t it = (int64_t)blockIdx.x * p.ipb + li;
  const bool iter_ok = li < p.ipb && it < p.tr.n_iter;
  const bool lane_on = iter_ok && s < P;
  const unsigned gmask = p.pw == 32 ? 0xffffffffu
                                    : (((1u << p.pw) - 1u) << (tid & 31 & ~(p.pw - 1)));

  double* it_ms = reinterpret_cast<double*>(smem_raw);
  unsigned* it_st = reinterpret_cast<unsigned*>(it_ms + p.ipb);
  const int it_bytes = ((p.ipb * 12 + 15) / 16) * 16;
  // per pipeline: base cost alpha*N + beta*Q_j of its micro-batches
  double* gbase = reinterpret_cast<double*>(smem_raw + it_bytes) +
                  (size_t)(tid >> p.log_pw) * p.mmax;

  if (tid < p.ipb) {
    it_ms[tid] = 0.0;
    it_st[tid] = 0u;
  }

  int seg = 0, m0 = 0, md = 0;
  if (iter_ok) {
    seg = p.tr.seg ? p.tr.seg[it] : 0;
    const int32_t* ms = p.sg.mb_start + (int64_t)seg * (D + 1);
    m0 = ms[d];
    md = ms[d + 1] - m0;
    if (md > p.mmax) md = -1;  // overflow: flagged below
  }
  // base cost alpha*N + beta*Q_j of the replica's micro-batches; the pw lanes
  // of the pipeline split the micro-batches between them
  if (iter_ok && md > 0) {
    const int64_t mb0 = it * M + m0;
    const double lin = __dmul_rn(p.m.alpha, (double)p.sh.token_budget);
    for (int jj = s; jj < md; jj += p.pw) {
      const int32_t a = __ldg(p.tr.mb_off + mb0 + jj);
      const int32_t b = __ldg(p.tr.mb_off + mb0 + jj + 1);
      long long q = 0;
      for (int32_t k = a; k < b; ++k) {
        const long long l = __ldg(p.tr.doc_len + k);
        q += l * l;
      }
      gbase[jj] = __dadd_rn(lin, __dmul_rn(p.m.beta, (double)q));
    }
  }

  double sp = 1.0, rlF = 0.0, rlB = 0.0, rlW = 0.0, hopf = 0.0, hopb = 0.0;
  int n_chain = 0, w = 0;
  bool stopped = false;
  if (lane_on && md > 0) {
    const int64_t gs = ((int64_t)seg * D + d) * P + s;
    sp = __ldg(p.sg.speed + gs);
    const double L = (double)__ldg(p.sg.layers + (int64_t)seg * P + s);
    rlF = __dmul_rn(p.m.ratio_f, L);
    rlB = __dmul_rn(ZBH ? p.m.ratio_b : __dadd_rn(p.m.ratio_b, p.m.ratio_w), L);
    rlW = __dmul_rn(p.m.ratio_w, L);
    if (s > 0) hopf = __ldg(p.sg.hop_fwd + gs - 1);
    if (s < P - 1) hopb = __ldg(p.sg.hop_bwd + gs);
    w = min(P - 1 - s, md);
    n_chain = (ZBH ? 3 : 2) * md;
    if (sp <= 0.0) {  // completeness violated (pipeline.py:408-415)
      stopped = true;
      n_chain = 0;
    }
  }
  __syncthreads();  // base costs visible; iteration slots initialised
  // a stopped stage invalidates the whole iteration (the reference raises
  // before building any DAG); its pipeline neighbours must not wait on it
  const unsigned bad = __ballot_sync(0xffffffffu, stopped) & gmask;
  if (bad) n_chain = 0;

  // ---------------------------------------------------------- wavefront
  double fin = 0.0, ssum = 0.0;
  bool over = false, hung = false;
  chain_walk<ZBH>(s, P, p.pw, md, w, n_chain, gbase, rlF, rlB, rlW, sp, hopf, hopb,
                  p.sh.capacity, p.mmax, fin, ssum, over, hung);

  // ------------------------------------------------------ reductions
  double gmax = fin;
  for (int off = p.pw >> 1; off > 0; off >>= 1)
    gmax = fmax(gmax, __shfl_xor_sync(0xffffffffu, gmax, off));
  const unsigned ovf = __ballot_sync(0xffffffffu, over) & gmask;
  const unsigned hang = __ballot_sync(0xffffffffu, hung) & gmask;

  uint8_t flag = 0;
  float sev = 0.0f;
  if (DETECT && lane_on && md >= 0) {
    const float* dt = p.tr.device_time + ((it * D + d) * P + s) * (int64_t)T;
    float mx = 0.0f;
    if (p.vec4) {
      for (int t = 0; t < T; t += 4) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(dt + t));
        mx = fmaxf(mx, fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w)));
      }
    } else {
      for (int t = 0; t < T; ++t) mx = fmaxf(mx, __ldg(dt + t));
    }
    const double meas = (double)mx;
    if (!(ssum <= 0.0 || meas <= 0.0) && meas > __dmul_rn(p.thr, ssum)) {
      flag = 1;
      sev = (float)__ddiv_rn(ssum, meas);
    }
  }
  if (iter_ok) {
    unsigned bits = 0;
    if (s == 0) {
      if (md < 0 || hang) bits |= RH_IT_OVERFLOW;
      if (bad) bits |= RH_IT_STOPPED;
      if (ovf) bits |= RH_IT_CAPACITY;
      double msd = gmax;
      if (p.sh.has_allreduce && D > 1)
        msd = __dadd_rn(gmax, __ldg(p.sg.allreduce + (int64_t)seg * D + d));
      atomic_max_nonneg(it_ms + li, msd);
    }
    if (flag) bits |= RH_IT_STAGE_FLAG;
    if (bits) atomicOr(it_st + li, bits);
  }
  __syncthreads();

  if (!iter_ok) return;
  const unsigned st_bits = it_st[li];
  const bool dead = (st_bits & (RH_IT_STOPPED | RH_IT_OVERFLOW)) != 0;
  if (lane_on) {
    const int64_t o = (it * D + d) * P + s;
    if (p.out.stage_cost) p.out.stage_cost[o] = dead ? 0.0 : ssum;
    if (DETECT) {
      if (p.out.stage_flag) p.out.stage_flag[o] = dead ? 0 : flag;
      if (p.out.severity) p.out.severity[o] = dead ? 0.0f : sev;
    }
  }
  if (within == 0) {
    unsigned st = st_bits;
    double ms = dead ? 0.0 : it_ms[li];
    if (dead) st &= (RH_IT_STOPPED | RH_IT_OVERFLOW);
    if (DETECT && !dead) {
      const double obs = __ldg(p.tr.observed + it);
      if (ms <= 0.0 || obs > __dmul_rn(p.thr, ms)) st |= RH_IT_ESCALATE;
      if (p.sg.link_off) {
        for (int32_t q = p.sg.link_off[seg]; q < p.sg.link_off[seg + 1]; ++q)
          if (__ldg(p.sg.link_ratio + q) > p.thr) st |= RH_IT_LINK_FLAG;
      }
    }
    p.out.makespan[it] = ms;
    p.out.status[it] = (uint8_t)st;
  }
}

static int next_pow2(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}

int launch_pass(rh_ctx* ctx, const rh_pipe_shape* sh, const rh_cost_model* m,
                const rh_segments* sg, const rh_trace* tr, double thr, int detect,
                const rh_pass_out* out, cudaStream_t stream) {
  if (!ctx || !sh || !m || !sg || !tr || !out || !out->makespan || !out->status) {
    set_error("pass: NULL argument");
    return RH_E_INVALID;
  }
  const int P = sh->pp, D = sh->dp, M = sh->micro_batches;
  if (P < 1 || D < 1 || M < 1 || sh->tp < 1 || sh->token_budget < 1 ||
      (sh->schedule != RH_SCHED_1F1B && sh->schedule != RH_SCHED_ZBH)) {
    set_error("pass: invalid shape pp=%d dp=%d tp=%d M=%d N=%d schedule=%d", P, D,
              sh->tp, M, sh->token_budget, sh->schedule);
    return RH_E_INVALID;
  }
  if (tr->n_iter == 0) return RH_OK;
  if (!tr->mb_off || !tr->doc_len || !sg->layers || !sg->mb_start || !sg->speed ||
      !sg->hop_fwd || !sg->hop_bwd || (sh->has_allreduce && D > 1 && !sg->allreduce) ||
      (detect && (!tr->device_time || !tr->observed))) {
    set_error("pass: missing trace/segment array");
    return RH_E_INVALID;
  }
  if (P > 32) {
    set_error("pass: pp=%d exceeds the 32-stage envelope", P);
    return RH_E_SHAPE;
  }
  PassParams p;
  p.sh = *sh;
  p.m = *m;
  p.sg = *sg;
  p.tr = *tr;
  p.out = *out;
  p.thr = thr;
  p.pw = next_pow2(P);
  p.log_pw = 0;
  while ((1 << p.log_pw) < p.pw) ++p.log_pw;
  p.lpi = D * p.pw;
  if (p.lpi > 1024) {
    set_error("pass: dp*next_pow2(pp) = %d exceeds 1024 lanes per CTA", p.lpi);
    return RH_E_SHAPE;
  }
  p.mmax = sh->max_mb_per_replica > 0 ? sh->max_mb_per_replica : M;
  p.ipb = std::max(1, 256 / p.lpi);
  p.vec4 = (sh->tp % 4 == 0) && ((reinterpret_cast<uintptr_t>(tr->device_time) & 15) == 0);
  const int threads = ((p.ipb * p.lpi + 31) / 32) * 32;
  const int it_bytes = ((p.ipb * 12 + 15) / 16) * 16;
  const size_t smem = it_bytes + (size_t)(threads / p.pw) * p.mmax * 8;
  if (smem > ctx->smem_optin) {
    set_error("pass: %zu bytes of shared memory needed (max_mb_per_replica=%d, pp=%d); "
              "limit %zu", smem, p.mmax, P, ctx->smem_optin);
    return RH_E_SHAPE;
  }
  const int64_t blocks = (tr->n_iter + p.ipb - 1) / p.ipb;
  if (blocks > 0x7fffffff) {
    set_error("pass: too many iterations");
    return RH_E_SHAPE;
  }
  void (*kern)(const PassParams);
  if (sh->schedule == RH_SCHED_ZBH)
    kern = detect ? pass_kernel<1, 1> : pass_kernel<1, 0>;
  else
    kern = detect ? pass_kernel<0, 1> : pass_kernel<0, 0>;
  RH_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kern<<<(unsigned)blocks, threads, smem, stream>>>(p);
  RH_CHECK_LAUNCH(ctx);
  return RH_OK;
}

// ------------------------------------------------------------------ host I/O
namespace {
struct Carver {
  char* base;
  size_t off = 0;
  template <class T>
  T* take(size_t n) {
    off = (off + 255) & ~size_t(255);
    T* r = reinterpret_cast<T*>(base + off);
    off += n * sizeof(T);
    return r;
  }
};
}  // namespace

int detect_host(rh_ctx* ctx, const rh_pipe_shape* sh, const rh_cost_model* m,
                const rh_segments* sg, const rh_trace* tr, double thr,
                const rh_screen_params* screen, int64_t series_len, const double* hist,
                const uint8_t* reset, const rh_pass_out* out, uint8_t* outcome,
                int64_t* series_len_out, cudaStream_t stream) {
  if (!ctx || !sh || !sg || !tr || !out || !tr->mb_off) {
    set_error("detect_host: NULL argument");
    return RH_E_INVALID;
  }
  const int P = sh->pp, D = sh->dp, T = sh->tp, M = sh->micro_batches;
  const int64_t n = tr->n_iter, G = (int64_t)D * P, S = sg->n_seg;
  if (n == 0) return RH_OK;
  const int64_t n_docs = tr->mb_off[n * M];
  const int64_t n_links = sg->link_off ? sg->link_off[S] : 0;
  size_t need = 0;
  {
    Carver c{nullptr};
    c.take<int32_t>(n);
    c.take<int32_t>(n * M + 1);
    c.take<int32_t>(n_docs);
    c.take<float>(n * G * T);
    c.take<double>(n);
    c.take<int32_t>(S * P);
    c.take<int32_t>(S * (D + 1));
    c.take<double>(S * G * 3);
    c.take<double>(S * D);
    c.take<int32_t>(S + 1);
    c.take<double>(n_links + 1);
    c.take<double>(n);
    c.take<uint8_t>(n);
    c.take<double>(n * G);
    c.take<uint8_t>(n * G);
    c.take<float>(n * G);
    c.take<double>(64);
    c.take<uint8_t>(n);
    c.take<uint8_t>(n);
    c.take<int64_t>(1);
    need = c.off + 256;
  }
  void* ws = nullptr;
  int rc = workspace(ctx, need, &ws, 0);
  if (rc) return rc;
  Carver c{static_cast<char*>(ws)};
  rh_trace dtr = *tr;
  rh_segments dsg = *sg;
  rh_pass_out dout = {};
  auto h2d = [&](auto* dst, const auto* src, size_t count) -> int {
    if (!src || !count) return RH_OK;
    RH_CUDA(cudaMemcpyAsync(dst, src, count * sizeof(*src), cudaMemcpyHostToDevice, stream));
    return RH_OK;
  };
#define RH_H2D(field_dst, src, count, T_)                \
  do {                                                   \
    T_* _d = c.take<T_>(count);                          \
    if ((rc = h2d(_d, src, count))) return rc;           \
    field_dst = src ? _d : nullptr;                      \
  } while (0)
  RH_H2D(dtr.seg, tr->seg, (size_t)n, int32_t);
  RH_H2D(dtr.mb_off, tr->mb_off, (size_t)(n * M + 1), int32_t);
  RH_H2D(dtr.doc_len, tr->doc_len, (size_t)n_docs, int32_t);
  RH_H2D(dtr.device_time, tr->device_time, (size_t)(n * G * T), float);
  RH_H2D(dtr.observed, tr->observed, (size_t)n, double);
  RH_H2D(dsg.layers, sg->layers, (size_t)(S * P), int32_t);
  RH_H2D(dsg.mb_start, sg->mb_start, (size_t)(S * (D + 1)), int32_t);
  RH_H2D(dsg.speed, sg->speed, (size_t)(S * G), double);
  RH_H2D(dsg.hop_fwd, sg->hop_fwd, (size_t)(S * G), double);
  RH_H2D(dsg.hop_bwd, sg->hop_bwd, (size_t)(S * G), double);
  RH_H2D(dsg.allreduce, sg->allreduce, (size_t)(S * D), double);
  RH_H2D(dsg.link_off, sg->link_off, (size_t)(S + 1), int32_t);
  RH_H2D(dsg.link_ratio, sg->link_ratio, (size_t)n_links, double);
#undef RH_H2D
  dout.makespan = c.take<double>(n);
  dout.status = c.take<uint8_t>(n);
  dout.stage_cost = out->stage_cost ? c.take<double>(n * G) : nullptr;
  dout.stage_flag = out->stage_flag ? c.take<uint8_t>(n * G) : nullptr;
  dout.severity = out->severity ? c.take<float>(n * G) : nullptr;
  double* d_hist = c.take<double>(64);
  uint8_t* d_reset = c.take<uint8_t>(n);
  uint8_t* d_outcome = c.take<uint8_t>(n);
  int64_t* d_len = c.take<int64_t>(1);
  const int64_t h = screen ? std::min<int64_t>(series_len, screen->window) : 0;
  if (screen && h > 64) {
    set_error("detector_pass_host: window > 64");
    return RH_E_INVALID;
  }
  if (h) RH_CUDA(cudaMemcpyAsync(d_hist, hist, h * sizeof(double), cudaMemcpyHostToDevice, stream));
  if (screen && reset)
    RH_CUDA(cudaMemcpyAsync(d_reset, reset, n, cudaMemcpyHostToDevice, stream));
  rc = launch_pass(ctx, sh, m, &dsg, &dtr, thr, 1, &dout, stream);
  if (rc) return rc;
  if (screen) {
    rc = rh_screen(ctx, screen, series_len, d_hist, n, dtr.observed, dout.status,
                   reset ? d_reset : nullptr, d_outcome, d_len, stream);
    if (rc) return rc;
    if (outcome)
      RH_CUDA(cudaMemcpyAsync(outcome, d_outcome, n, cudaMemcpyDeviceToHost, stream));
    if (series_len_out)
      RH_CUDA(cudaMemcpyAsync(series_len_out, d_len, sizeof(int64_t), cudaMemcpyDeviceToHost,
                              stream));
  }
  RH_CUDA(cudaMemcpyAsync(out->makespan, dout.makespan, n * sizeof(double),
                          cudaMemcpyDeviceToHost, stream));
  RH_CUDA(cudaMemcpyAsync(out->status, dout.status, n, cudaMemcpyDeviceToHost, stream));
  if (out->stage_cost)
    RH_CUDA(cudaMemcpyAsync(out->stage_cost, dout.stage_cost, n * G * sizeof(double),
                            cudaMemcpyDeviceToHost, stream));
  if (out->stage_flag)
    RH_CUDA(cudaMemcpyAsync(out->stage_flag, dout.stage_flag, n * G,
                            cudaMemcpyDeviceToHost, stream));
  if (out->severity)
    RH_CUDA(cudaMemcpyAsync(out->severity, dout.severity, n * G * sizeof(float),
                            cudaMemcpyDeviceToHost, stream));
  RH_CUDA(cudaStreamSynchronize(stream));
  return RH_OK;
}

}  // namespace rh

extern "C" {

int rh_pipeline_batch(rh_ctx* ctx, const rh_pipe_shape* shape, const rh_cost_model* model,
                      const rh_segments* segs, const rh_trace* trace,
                      const rh_pass_out* out, void* stream) {
  return rh::launch_pass(ctx, shape, model, segs, trace, 0.0, 0, out, rh::as_stream(stream));
}

int rh_detect_batch(rh_ctx* ctx, const rh_pipe_shape* shape, const rh_cost_model* model,
                    const rh_segments* segs, const rh_trace* trace, double threshold,
                    const rh_pass_out* out, void* stream) {
  return rh::launch_pass(ctx, shape, model, segs, trace, threshold, 1, out,
                         rh::as_stream(stream));
}

int rh_detector_pass_host(rh_ctx* ctx, const rh_pipe_shape* shape, const rh_cost_model* model,
                          const rh_segments* segs, const rh_trace* trace, double threshold,
                          const rh_screen_params* screen, int64_t series_len,
                          const double* hist, const uint8_t* reset, const rh_pass_out* out,
                          uint8_t* outcome, int64_t* series_len_out, void* stream) {
  return rh::detect_host(ctx, shape, model, segs, trace, threshold, screen, series_len, hist,
                         reset, out, outcome, series_len_out, rh::as_stream(stream));
}

}  // extern "C"
