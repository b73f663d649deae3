/*
 * resihp_b200.h — C ABI of the B200-native ResiHP data-parallel core.
 *
 * The reference (arxiv 2605.06374, `resilsim`, /root/reference/pkg/src) is a
 * pure-Python package with no FFI; its "interface" for this path is the set
 * of Python functions exported from resilsim/__init__.py:5-60.  Every entry
 * point below replaces one of those functions (cited per declaration) for a
 * BATCH of inputs; the Python package paper_2605_06374_b200 binds them with
 * ctypes and keeps the reference's Python signatures.
 *
 * Conventions
 *   - plain C types only; all array pointers are DEVICE pointers unless the
 *     function name ends in _host;
 *   - every function returns RH_OK (0) or a negative RH_E_* code, with a
 *     message in rh_last_error() (thread-local);
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default);
 *     functions are asynchronous on that stream unless documented otherwise;
 *   - arithmetic on every decision-carrying quantity is IEEE fp64 with the
 *     reference's evaluation order and no FMA contraction.
 *
 * Threading contract
 *   - An rh_ctx belongs to one device; every entry point makes that device
 *     current for the call and restores the caller's current device.
 *   - A context may be used from several host threads.  Scratch memory is
 *     per (context, stream): calls on distinct streams never share scratch,
 *     so they may run concurrently; calls on one stream are stream-ordered.
 *     Scratch only grows; a grown buffer is retired (not freed) until
 *     rh_ctx_destroy, so work already queued never sees freed memory, and
 *     growth is refused (RH_E_INVALID) inside a stream capture — run a call
 *     once outside the capture before capturing it.
 *   - rh_screen_prepare / rh_screen: one pending prepare per context (the
 *     next rh_screen with the same arguments consumes it).
 *   - An rh_search handle may be evaluated from several streams: each eval
 *     waits for the handle's previous create / eval.  No call ever
 *     synchronises the device, and the device's default memory pool is not
 *     modified (searches allocate from a private pool).
 *   - rh_detector_pass_host*: synchronous; the context replays one captured
 *     graph per argument key (serialise calls that share a context).
 */
#ifndef RESIHP_B200_H
#define RESIHP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RH_ABI_VERSION 1

enum {
  RH_OK = 0,
  RH_E_INVALID = -1,   /* bad argument: Python shim raises ValueError        */
  RH_E_CUDA = -2,      /* CUDA runtime failure                               */
  RH_E_NOMEM = -3,     /* workspace allocation failed                        */
  RH_E_SHAPE = -4      /* shape outside this kernel's envelope (documented)  */
};

/* Per-iteration status bits (rh_pipeline_batch / rh_detect_batch). */
enum {
  RH_IT_ESCALATE = 1,   /* filter_candidate(...) == ESCALATE  (detector.py:111-116) */
  RH_IT_STAGE_FLAG = 2, /* validate: >=1 (replica,stage) flagged (detector.py:141-147) */
  RH_IT_LINK_FLAG = 4,  /* validate: >=1 link flagged (detector.py:148-152)          */
  RH_IT_STOPPED = 8,    /* chunk mapped to a stopped stage (pipeline.py:408-415)      */
  RH_IT_CAPACITY = 16,  /* activation footprint > capacity (pipeline.py:516-539)      */
  RH_IT_OVERFLOW = 32   /* a replica owns more than max_mb_per_replica micro-batches  */
};

enum { RH_SCHED_1F1B = 0, RH_SCHED_ZBH = 1 };  /* cluster.py SCHEDULES */

/* CostModel (workload.py:29-49).  ratio(BW) = ratio_b + ratio_w. */
typedef struct rh_cost_model {
  double alpha;   /* seconds per token    */
  double beta;    /* seconds per token^2  */
  double ratio_f;
  double ratio_b;
  double ratio_w;
} rh_cost_model;

/* Fixed pipeline shape of a batch (ParallelismConfig, cluster.py:37-50). */
typedef struct rh_pipe_shape {
  int32_t pp;             /* P stages                                        */
  int32_t dp;             /* D replicas                                      */
  int32_t tp;             /* nominal TP degree T = device slots per group    */
  int32_t schedule;       /* RH_SCHED_*                                      */
  int32_t micro_batches;  /* M micro-batches per iteration                   */
  int32_t token_budget;   /* N tokens per micro-batch                        */
  int32_t capacity;       /* activation capacity; <= 0 = unchecked           */
  int32_t has_allreduce;  /* terminal AR vertex per replica (pipeline.py:242) */
  int32_t max_mb_per_replica; /* upper bound on dp_counts over all segments;
                                 sizes shared memory (<= 0: use M)          */
} rh_pipe_shape;

/*
 * Segment tables: a segment is a span of iterations with one layout / one
 * view of device speeds.  All tables are per segment, row-major.
 *   speed[d][s]   effective stage speed (ClusterState.effective_stage_speed,
 *                 cluster.py:155-169); <= 0 marks a stopped stage
 *   hop_fwd[d][s] seconds on the data edge F(j,s) -> F(j,s+1), s < P-1
 *   hop_bwd[d][s] seconds on the data edge B(j,s+1) -> B(j,s), s < P-1
 *                 (edge_cost_fn, pipeline.py:336-353)
 *   allreduce[d]  terminal AR vertex cost (_allreduce_map, pipeline.py:356-372)
 *   mb_start[d]   first micro-batch (index within the iteration) owned by
 *                 replica d; mb_start[D] = M (split_micro_batches,
 *                 cluster.py:309-328)
 *   link_ratio    measured/expected ratios of the exercised inter-node links
 *                 (_used_link_ratios, pipeline.py:491-513), CSR by link_off.
 */
typedef struct rh_segments {
  int32_t n_seg;
  const int32_t* layers;      /* [n_seg][P]                    */
  const int32_t* mb_start;    /* [n_seg][D+1]                  */
  const double* speed;        /* [n_seg][D][P]                 */
  const double* hop_fwd;      /* [n_seg][D][P]                 */
  const double* hop_bwd;      /* [n_seg][D][P]                 */
  const double* allreduce;    /* [n_seg][D]; read iff has_allreduce */
  const int32_t* link_off;    /* [n_seg+1] or NULL (no links)  */
  const double* link_ratio;   /* [link_off[n_seg]]             */
  /* Optional [n_seg]: the largest link_ratio of each segment (0 for none).
   * When given, the exercised-link test of an iteration is one compare
   * (any ratio > thr  <=>  max > thr) instead of a scan; it must match
   * link_ratio.  NULL: the kernels scan link_ratio. */
  const double* link_max;
} rh_segments;

/*
 * A batch of iterations (the device x iteration trace).
 *   mb_off[i*M + j] .. mb_off[i*M + j + 1] index the packed documents of
 *   micro-batch j of iteration i in doc_len (padding document included,
 *   workload.py:52-80).  Offsets are int32: a batch holds < 2^31 documents.
 *   device_time[i][d][s][t]: measured stage seconds of member t of group
 *   (d,s); 0 for an empty slot.  The group's measured stage time is the max
 *   over its members (a TP group runs at its slowest member, cluster.py:155).
 */
typedef struct rh_trace {
  int64_t n_iter;
  const int32_t* seg;          /* [n_iter] segment id; NULL = segment 0 */
  const int32_t* mb_off;       /* [n_iter*M + 1]                       */
  const int32_t* doc_len;      /* [mb_off[n_iter*M]]                   */
  const float* device_time;    /* [n_iter][D][P][T]  (detect only)     */
  const double* observed;      /* [n_iter]           (detect only)     */
} rh_trace;

/* Outputs.  Optional arrays may be NULL. */
typedef struct rh_pass_out {
  double* makespan;     /* [n_iter] critical path (pipeline.py:259-292)     required */
  uint8_t* status;      /* [n_iter] RH_IT_* bits                            required */
  double* stage_cost;   /* [n_iter][D][P] sum of chunk costs (pipeline.py:446-453) */
  uint8_t* stage_flag;  /* [n_iter][D][P] validate flag            (detect only)    */
  float* severity;      /* [n_iter][D][P] expected/measured if flagged else 0       */
} rh_pass_out;

typedef struct rh_ctx rh_ctx;

/* ---------------------------------------------------------------- context */
int rh_abi_version(void);
const char* rh_last_error(void);
int rh_ctx_create(int device, rh_ctx** out);
int rh_ctx_destroy(rh_ctx* ctx);
/* number of kernel launches issued through this context (for bench.py) */
int64_t rh_ctx_launches(const rh_ctx* ctx);

/* Device self-test of the exact division used on the hot path (a hoisted
 * correctly rounded reciprocal + Markstein correction, with __ddiv_rn outside
 * a safe range): counts the bit mismatches against __ddiv_rn over n seeded
 * random (a, b) pairs.  Synchronous; 0 is the only acceptable result. */
int rh_selftest_division(rh_ctx* ctx, int64_t n, uint64_t seed, int64_t* mismatches);
/* Measured FP64 pipe peak of the context's device (fp64 instructions per
 * second, thread-level: independent DFMA chains on every SM).  The roofline
 * denominator bench.py reports the re-plan search against. */
int rh_fp64_peak(rh_ctx* ctx, double* instr_per_s);

/* ------------------------------------------------------- cost model rows */
/* quad_load (workload.py:83-85) for n micro-batches given a CSR of docs. */
int rh_quad_load(rh_ctx* ctx, int64_t n_mb, const int32_t* mb_off,
                 const int32_t* doc_len, int64_t* quad_out, void* stream);

/* predict_chunk_time (workload.py:88-98) for n chunks:
 *   t[i] = ((ratio(kind[i]) * layers[i]) * (alpha*budget[i] + beta*quad[i])) / speed[i]
 * kind: 0=F 1=B 2=W 3=BW.  speed <= 0 sets bad[i]=1 and t[i]=0 (ValueError). */
int rh_chunk_time(rh_ctx* ctx, const rh_cost_model* model, int64_t n,
                  const int64_t* quad, const int32_t* budget, const uint8_t* kind,
                  const int32_t* layers, const double* speed, double* t_out,
                  uint8_t* bad_out, void* stream);

/* --------------------------------------------- pipeline predictor (Eq. 2) */
/*
 * Canonical (migration-free) chunk-DAG critical path for a batch of
 * iterations: per iteration i, the makespan of build_dag(...) +
 * critical_path(...) (pipeline.py:129-292) under the segment's speeds, the
 * per-(replica,stage) stage cost sums and the activation check.  Replaces
 * the two build_dag/critical_path calls inside simulate_iteration
 * (pipeline.py:432-441) for every iteration of the batch at once.
 * Envelope: 1 <= P <= 32, D*next_pow2(P) <= 1024.
 */
int rh_pipeline_batch(rh_ctx* ctx, const rh_pipe_shape* shape,
                      const rh_cost_model* model, const rh_segments* segs,
                      const rh_trace* trace, const rh_pass_out* out,
                      void* stream);
/* Host-buffer twin of rh_pipeline_batch (segments, trace and outputs in
 * HOST memory): one staged copy in, one copy out, synchronous -- the drop-in
 * simulate_iteration's per-call path. */
int rh_pipeline_batch_host(rh_ctx* ctx, const rh_pipe_shape* shape, const rh_cost_model* model,
                           const rh_segments* segs, const rh_trace* trace,
                           const rh_pass_out* out);

/*
 * Fused Detector pass: rh_pipeline_batch on the KNOWN view (the predictor,
 * harness.py:406-410) fused with filter_candidate (detector.py:111-116) and
 * validate (detector.py:127-158) against the measured device trace.
 * threshold = DetectorState.escalation_factor (1.25).
 */
int rh_detect_batch(rh_ctx* ctx, const rh_pipe_shape* shape,
                    const rh_cost_model* model, const rh_segments* segs,
                    const rh_trace* trace, double threshold,
                    const rh_pass_out* out, void* stream);

/* ------------------------------------------------------ validate (batch) */
/* validate (detector.py:127-158) on explicit arrays: flag[i] = measured[i] >
 * thr*expected[i] (skipping non-positive entries), sev[i] = expected/measured
 * when flagged else 0.  Used for standalone validate() and link ratios
 * (pass expected=NULL to test ratio[i] > thr with sev = 1/ratio). */
int rh_validate(rh_ctx* ctx, int64_t n, const double* measured,
                const double* expected, double threshold, uint8_t* flag,
                double* severity, void* stream);

/* ------------------------------------------------ change-point screen */
enum {
  RH_SC_CANDIDATE = 1,  /* detect_change_point fired (detector.py:94-108)  */
  RH_SC_FILTERED = 2,   /* filter ran (candidate or refill, detector.py:221) */
  RH_SC_ESCALATED = 4,  /* escalated to validation                         */
  RH_SC_CONFIRMED = 8,  /* validation confirmed                            */
  RH_SC_POPPED = 16     /* observation removed from the series             */
};

typedef struct rh_screen_params {
  int32_t window;          /* DetectorState.window (20)             */
  int32_t filter_enabled;  /* DetectorState.filter_enabled          */
  double kappa;            /* DetectorState.kappa (3.0)             */
} rh_screen_params;

/*
 * DetectorState.observe state machine (detector.py:198-271) over n
 * iterations.  The carried series state is (series_len, the last
 * min(series_len, window) values in hist).  it_status are the RH_IT_* bits
 * of rh_detect_batch; reset[i] != 0 clears the series before iteration i
 * (harness.py:398); reset may be NULL.  outcome[i] gets RH_SC_* bits.
 * series_len_out (device int64) receives the final series length.
 */
int rh_screen(rh_ctx* ctx, const rh_screen_params* params, int64_t series_len,
              const double* hist, int64_t n, const double* observed,
              const uint8_t* it_status, const uint8_t* reset, uint8_t* outcome,
              int64_t* series_len_out, void* stream);

/* ------------------------------------------- per-call host entry points */
/* One DetectorState.observe (detector.py:198-271) in one round trip: when
 * do_validate, validate the n_stage (measured, expected) pairs and the n_link
 * exercised-link ratios (detector.py:127-158) into the flag / severity arrays;
 * fold the flags and `escalate` (the host's filter verdict) into the status
 * bits; screen `observed` against the carried series (series_len, hist = its
 * last min(series_len, window) values) -> outcome (RH_SC_* bits) and the new
 * series length.  Host pointers, synchronous. */
int rh_observe_host(rh_ctx* ctx, const rh_screen_params* params, int64_t series_len,
                    const double* hist, double observed, int32_t escalate, int32_t do_validate,
                    int32_t n_stage, const double* measured, const double* expected,
                    int32_t n_link, const double* link_ratio, double threshold,
                    uint8_t* stage_flag, double* stage_sev, uint8_t* link_flag, double* link_sev,
                    uint8_t* outcome, int64_t* series_len_out);

/* Host-buffer twins of rh_quad_load, rh_chunk_time, rh_validate and rh_screen
 * for the drop-in API's per-call functions (workload.quad_load /
 * predict_chunk_time, detector.validate, one DetectorState.observe): every
 * pointer is HOST memory (any, not necessarily pinned); the inputs are
 * gathered into the context's pinned staging and cross PCIe in one copy,
 * the outputs come back in one copy, and the call returns when they are in
 * the caller's arrays.  Synchronous; calls on one context are serialised. */
int rh_quad_load_host(rh_ctx* ctx, int64_t n_mb, const int32_t* mb_off,
                      const int32_t* doc_len, int64_t* quad_out);
int rh_chunk_time_host(rh_ctx* ctx, const rh_cost_model* model, int64_t n,
                       const int64_t* quad, const int32_t* budget, const uint8_t* kind,
                       const int32_t* layers, const double* speed, double* t_out,
                       uint8_t* bad_out);
/* predict_chunk_time from the documents in one round trip: quad loads of the
 * n_mb micro-batches (CSR mb_off / doc_len), then t[i] for chunk i of
 * micro-batch mb_idx[i] (host arrays; bad_out required). */
int rh_chunk_time_docs_host(rh_ctx* ctx, const rh_cost_model* model, int64_t n_mb,
                            const int32_t* mb_off, const int32_t* doc_len, int64_t n,
                            const int64_t* mb_idx, const int32_t* budget, const uint8_t* kind,
                            const int32_t* layers, const double* speed, double* t_out,
                            uint8_t* bad_out);
int rh_validate_host(rh_ctx* ctx, int64_t n, const double* measured,
                     const double* expected, double threshold, uint8_t* flag,
                     double* severity);
int rh_screen_host(rh_ctx* ctx, const rh_screen_params* params, int64_t series_len,
                   const double* hist, int64_t n, const double* observed,
                   const uint8_t* it_status, const uint8_t* reset, uint8_t* outcome,
                   int64_t* series_len_out);

/*
 * Optional early half of rh_screen: the parts that depend only on the inputs
 * (reset indices and the round-0 median/MAD verdicts, which read observed,
 * hist and reset but not it_status).  Launch it on a side stream as soon as
 * those inputs are ready -- typically before rh_detect_batch, so it overlaps
 * the detect kernel.  The next rh_screen on the same context with the same
 * (params, series_len, hist, n, observed, reset) waits on it instead of
 * recomputing; inputs must not change in between.  Any other rh_screen call
 * recomputes as usual.
 */
int rh_screen_prepare(rh_ctx* ctx, const rh_screen_params* params, int64_t series_len,
                      const double* hist, int64_t n, const double* observed,
                      const uint8_t* reset, void* stream);

/* ---------------------------------------------------- workload ingest */
/*
 * pack_sequences (workload.py:52-80), HOST function: first-fit-decreasing
 * packing of n_docs lengths into bins of exactly `budget` tokens (residual
 * appended as a padding document).  Keeps the first max_bins bins
 * (max_bins < 0: all; harness.py:251-252 keeps packed[:M]).  With mb_off or
 * doc_len NULL only *n_bins_out / *n_entries_out are computed (size query);
 * otherwise mb_off[n_bins+1] and doc_len[n_entries] are filled (host memory).
 */
int rh_pack_sequences(int64_t n_docs, const int32_t* lengths, int32_t budget,
                      int64_t max_bins, int32_t* mb_off, int32_t* doc_len,
                      int64_t* n_bins_out, int64_t* n_entries_out);
/* rh_pack_sequences plus quad[b] = quad_load of kept bin b (int64, padding
 * included; workload.py:83-85) -- what a re-plan needs of its workload. */
int rh_pack_sequences_quad(int64_t n_docs, const int32_t* lengths, int32_t budget,
                           int64_t max_bins, int32_t* mb_off, int32_t* doc_len, int64_t* quad,
                           int64_t* n_bins_out, int64_t* n_entries_out);

/* ------------------------------------------- end-to-end Detector pass */
/*
 * The whole Detector for a trace, HOST buffers in and out: copies segs and
 * trace (and hist/reset) to the device, runs rh_detect_batch then rh_screen
 * (when screen != NULL), copies `out`, outcome[n] and *series_len_out back
 * and synchronises `stream`.  This is the reference-facing call: one
 * DetectorState.observe(...) per iteration of resilsim (harness.py:402-431)
 * becomes one call per trace.  Pinned host memory gives full PCIe/C2C rate.
 */
int rh_detector_pass_host(rh_ctx* ctx, const rh_pipe_shape* shape,
                          const rh_cost_model* model, const rh_segments* segs,
                          const rh_trace* trace, double threshold,
                          const rh_screen_params* screen, int64_t series_len,
                          const double* hist, const uint8_t* reset,
                          const rh_pass_out* out, uint8_t* outcome,
                          int64_t* series_len_out, void* stream);

/*
 * Packed wire form of a trace for the host-buffer pass (the same data as
 * rh_trace, ~40 % fewer bytes over PCIe).  pack_sequences bins hold at most
 * `token_budget` tokens (workload.py:52-80), so a document length fits 16 bits
 * whenever token_budget <= 65535; a micro-batch holds at most 255 documents.
 *   iter_doc[i] .. iter_doc[i+1]   documents of iteration i (int32, < 2^31)
 *   mb_docs[i*M + j]               documents in micro-batch j of iteration i
 *   doc_len[k]                     length of document k
 * The device rebuilds the int32 CSR chunk by chunk while later chunks cross
 * PCIe, then runs exactly the rh_detector_pass_host pipeline.
 */
typedef struct rh_trace_packed {
  int64_t n_iter;
  const int32_t* seg;          /* [n_iter] segment id; NULL = segment 0 */
  const int32_t* iter_doc;     /* [n_iter + 1]                          */
  const uint8_t* mb_docs;      /* [n_iter * M]                          */
  const uint16_t* doc_len;     /* [iter_doc[n_iter]]                    */
  const float* device_time;    /* [n_iter][D][P][T]                     */
  const double* observed;      /* [n_iter]                              */
} rh_trace_packed;

int rh_detector_pass_host_packed(rh_ctx* ctx, const rh_pipe_shape* shape,
                                 const rh_cost_model* model, const rh_segments* segs,
                                 const rh_trace_packed* trace, double threshold,
                                 const rh_screen_params* screen, int64_t series_len,
                                 const double* hist, const uint8_t* reset,
                                 const rh_pass_out* out, uint8_t* outcome,
                                 int64_t* series_len_out, void* stream);

/* -------------------------------------------- general DAG critical path */
/*
 * critical_path (pipeline.py:259-292) on an arbitrary DAG given in CSR by
 * source (succ_off[V+1], succ_dst[E], succ_w[E]); writes starts[V] and
 * makespan[0].  Optionally (n_chains > 0) reduces resource chains — vertex
 * ranges [chain_off[k], chain_off[k+1]) in creation order, as build_dag
 * emits them per (replica, stage) — to chain_sum[k] (sequential sum,
 * pipeline.py:446-453) and runs the activation check along each chain with
 * kind[v] (0=F +1 at start, 1=B/3=BW -1 at finish; pipeline.py:516-539).
 * flags[0] = 1 on a cycle (CycleError), flags[1] = 1 if capacity > 0 was
 * exceeded.  flags is a device int32[2].  Level-synchronous, one CTA.
 */
int rh_dag_critical_path(rh_ctx* ctx, int32_t n_vertices, const double* cost,
                         const int32_t* succ_off, const int32_t* succ_dst,
                         const double* succ_w, int32_t n_chains,
                         const int32_t* chain_off, const uint8_t* kind,
                         int32_t capacity, double* starts, double* makespan,
                         double* chain_sum, int32_t* flags, void* stream);
/* Host-buffer twin of rh_dag_critical_path (every pointer HOST memory; flags
 * are zeroed by the call): one staged copy in, one copy out, synchronous. */
int rh_dag_critical_path_host(rh_ctx* ctx, int32_t n_vertices, const double* cost,
                              const int32_t* succ_off, const int32_t* succ_dst,
                              const double* succ_w, int32_t n_chains, const int32_t* chain_off,
                              const uint8_t* kind, int32_t capacity, double* starts,
                              double* makespan, double* chain_sum, int32_t* flags);

/* ------------------------------------------- batched scalar Scheduler rows */
/* One thread per problem; problems are CSR slices off[i]..off[i+1] (device).
 * repartition_layers (scheduler.py:146-207), <= 32 stages per problem;
 *   err[i]: 0 ok, 1 non-positive speed, 2 too few layers, 3 too many stages. */
int rh_repartition_batch(rh_ctx* ctx, int32_t n, const int32_t* off, const double* speeds,
                         const int32_t* total_layers, const int32_t* min_layers, int32_t* out,
                         int32_t* err, void* stream);
/* proportional_split (policies.py:151-162), <= 64 weights per problem;
 *   err[i]: 0 ok, 1 sum(weights) <= 0, 3 too many weights. */
int rh_proportional_split_batch(rh_ctx* ctx, int32_t n, const int32_t* off,
                                const double* weights, const int32_t* totals, int32_t* counts,
                                int32_t* err, void* stream);
/* select_tp_subgroup (scheduler.py:114-137): ranked[] = member ids by
 * (-speed, id); best_k[i] = chosen degree (0 = GroupUnrecoverable).
 * degree_mask bit e allows degree 2^e (candidate_tp_degrees, :101-111). */
int rh_select_subgroup_batch(rh_ctx* ctx, int32_t n, const int32_t* off, const double* speeds,
                             const int32_t* ids, const uint32_t* degree_mask, int32_t* ranked,
                             int32_t* best_k, void* stream);

/* ---------------------------------------- progress-aware migration (Alg. 1) */
/*
 * plan_migration (scheduler.py:272-513), HOST function: the work-conserving
 * co-simulation of one iteration with progress-aware stage-level migration
 * (migration_decision, scheduler.py:210-251).  Micro-batch ids are 0..n_mb-1
 * in order.  Hop weights are tables (edge_seconds evaluated by the caller):
 *   hop_next[s][a][b] = edge(s, a, s+1, b)   hop_prev[s][a][b] = edge(s, a, s-1, b)
 *   hop_same[s][a][b] = edge(s, a, s,   b)   ([P][D][D]; NULL = no comm)
 * Outputs (host): migrations[k] = (mb, stage, source, executor) in decision
 * order; start_log[c] = (replica, stage, kind 0=F 1=B/BW 2=W, mb) in start
 * order (stage_orders); *makespan.  Returns RH_E_STRANDED with the
 * reference's message when work is unexecutable.
 */
enum { RH_E_STRANDED = -5 };

typedef struct rh_migration_desc {
  int32_t pp, dp, schedule, n_mb;
  int32_t token_budget;
  rh_cost_model model;
  const int32_t* mb_off;      /* [n_mb+1] CSR of packed documents   */
  const int32_t* doc_len;
  const int32_t* layers;      /* [pp]                               */
  const double* speed;        /* [dp][pp]; <= 0 = stopped stage     */
  const int32_t* dp_counts;   /* [dp] or NULL (even split)          */
  int32_t delta, capacity, migrate;
  const int32_t* preset;      /* [n_mb][pp] executor or -1; or NULL */
  const double* hop_next;     /* [pp][dp][dp] or NULL               */
  const double* hop_prev;
  const double* hop_same;
} rh_migration_desc;

int rh_plan_migration(const rh_migration_desc* desc, int32_t* migrations, int32_t* n_migrations,
                      int32_t* start_log, int32_t* n_started, double* makespan);

/* ------------------------------------------------ Scheduler re-plan search */
/*
 * Exhaustive re-plan search over (DP, TP, PP) layouts x layer partitions x
 * workload-to-replica assignments (BASELINE.json north star; DESIGN.md §5
 * defines the space).  Every candidate is scored exactly like
 * resihp_adapt scores its variants (policies.py:329-347):
 *   score = evaluate_plan(...)          (scheduler.py:543-559: canonical
 *                                        chunk-DAG makespan incl. terminal
 *                                        all-reduce, activation capacity)
 *         + reconfig_cost(...) / max(1, amortize_iterations)
 * and the best candidate is the lexicographic (score, index) minimum.
 * Building blocks on the path: candidate_tp_degrees-style power-of-two
 * degrees (scheduler.py:101-111), fastest-k member selection
 * (select_tp_subgroup, :114-137), repartition_layers (:146-207),
 * _replica_speeds + proportional_split (policies.py:138-162).
 * All pointers in rh_search_desc are HOST pointers (copied at create).
 */
typedef struct rh_search_desc {
  /* cluster: known speed per device (<= 0: not executable, e.g. fail-stop) */
  int32_t n_devices;
  int32_t devices_per_node;
  const double* device_speed;      /* [n_devices]                          */
  double intra_bw, inter_bw;       /* bytes/s                              */
  int32_t n_links;                 /* degraded inter-node links            */
  const int32_t* link_nodes;       /* [n_links][2], a < b                  */
  const double* link_factor;       /* [n_links]                            */
  /* workload + cost model */
  rh_cost_model model;
  int32_t schedule;                /* RH_SCHED_*                           */
  int32_t token_budget;
  int32_t n_micro_batches;
  const int64_t* quad;             /* [n_micro_batches] sum of l^2         */
  int32_t total_layers;
  int32_t min_layers;
  int32_t capacity;                /* activation capacity (<= 0: none)     */
  /* communication (CommSpec, comm.py:49-58) */
  int32_t has_comm;
  double hidden_bytes_per_token;
  double layer_bytes;
  int32_t p2p_optimized;
  /* candidate space */
  int32_t nominal_tp;              /* cfg.tp: a T-wide group of slowest speed v runs at
                                      v*T/nominal_tp (effective_stage_speed, cluster.py:155) */
  int32_t max_tp;                  /* TP degrees: powers of two dividing devices_per_node */
  int32_t max_pp;                  /* <= 32                                */
  int32_t max_dp;
  double min_utilization;          /* layouts use >= this share of executable devices */
  /* current plan (reconfiguration surcharge) */
  int32_t cur_tp, cur_dp, cur_pp;  /* 0 = none                             */
  const int32_t* cur_groups;       /* [cur_dp*cur_pp][cur_tp] members, replica-major */
  const int32_t* cur_partition;    /* [cur_pp]                             */
  double group_rebuild_s;
  int32_t amortize_iterations;
} rh_search_desc;

typedef struct rh_search rh_search;

/* One decoded candidate (host memory). */
typedef struct rh_candidate {
  int64_t index;
  int32_t tp, dp, pp;
  int32_t layout;                  /* layout ordinal                       */
  int32_t partition_variant;       /* 0 even, 1 repartition, >=2 one move  */
  int32_t count_variant;           /* 0 even, 1 proportional, >=2 one move */
  int32_t feasible;
} rh_candidate;

/* Enumerate layouts, upload inputs and queue the per-layout preparation
 * (placement, hop/ring tables, repartition_layers, proportional_split) on
 * the GPU.  Returns once the inputs are on the device; the preparation
 * kernels stay queued on `stream` (rh_search_set_workload, rh_search_eval
 * and rh_search_decode order after them, on any stream). */
int rh_search_create(rh_ctx* ctx, const rh_search_desc* desc, rh_search** out, void* stream);
/* Returns the search's device memory to the stream-ordered pool on the stream
 * of its latest create / eval call (so pending work on that stream finishes
 * first); that stream must still exist. */
/*
 * Deferred workload: rh_search_create accepts desc->quad == NULL (layouts,
 * placement, repartition, proportional splits and op lists do not depend on
 * the micro-batches' quad loads), and rh_search_set_workload supplies the
 * quad loads (host, n_micro_batches int64) before the first eval -- so a
 * re-plan can pack its sequences (rh_pack_sequences) on a host thread while
 * the search is being created.  Synchronous on `stream`.
 */
int rh_search_set_workload(rh_ctx* ctx, rh_search* search, const int64_t* quad, void* stream);
int rh_search_destroy(rh_search* search);
/* total number of candidates / layouts */
int64_t rh_search_size(const rh_search* search);
int32_t rh_search_layouts(const rh_search* search);
/* Cost-balanced contiguous shard of [0, size) for `rank` of `world` (HOST):
 * boundaries fall between (layout, partition variant) blocks of candidates,
 * weighted by each block's evaluation work (its replica-pipeline table plus
 * the per-candidate combination), so that no table row is computed twice and
 * ranks finish together.  The union over ranks is [0, size). */
int rh_search_shard(const rh_search* search, int32_t rank, int32_t world, int64_t* begin,
                    int64_t* end);
/* Score candidates [begin, end) and min-loc them.  best_score/best_index are
 * DEVICE scalars (+inf / -1 when nothing is feasible); scores (optional,
 * device, [end-begin]) receives every candidate's score (+inf infeasible). */
int rh_search_eval(rh_ctx* ctx, rh_search* search, int64_t begin, int64_t end,
                   double* best_score, int64_t* best_index, double* scores,
                   void* stream);
/* Decode a candidate index: layout, variants, and (host arrays, optional)
 * groups[dp*pp][tp] member ids, partition[pp], counts[dp]. */
int rh_search_decode(rh_ctx* ctx, rh_search* search, int64_t index, rh_candidate* out,
                     int32_t* groups, int32_t* partition, int32_t* counts);

/* ------------------------------------------- multi-GPU search collective */
/*
 * The one collective of the sharded re-plan search (search.py
 * distributed_best), for callers without torch: every rank
 * holds its shard's (score, index) winner on the device (rh_search_eval
 * outputs); rh_minloc_allreduce all-gathers the 16-byte pairs over NCCL and
 * reduces them on the device with the lexicographic (score, index) rule, in
 * place, identically on every rank.  Asynchronous on `stream`.  NCCL is
 * resolved at run time (the process's, else libnccl.so.2).
 */
int rh_nccl_unique_id(uint8_t* id_out /* 128 bytes */);
int rh_nccl_comm_create(rh_ctx* ctx, int32_t world, int32_t rank, const uint8_t* id,
                        void** comm_out);
int rh_nccl_comm_destroy(void* comm);
int rh_minloc_allreduce(rh_ctx* ctx, void* comm, int32_t world, double* score,
                        int64_t* index, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* RESIHP_B200_H */
