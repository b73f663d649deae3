/*
 * TEST INFRASTRUCTURE — NOT PRODUCT CODE.
 *
 * CPU restatement of the reference algorithm (arxiv 2605.06374 `resilsim`,
 * /root/reference/pkg/src/resilsim) for the ResiHP data-parallel hot path.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load liboracle.so, and only as the checker or
 * the timed CPU baseline.  The product (paper_2605_06374_b200) never links it.
 *
 * Parity is PINNED: tests/test_oracle_golden.py checks every function here
 * against golden vectors produced by importing the reference itself
 * (tests/golden/make_golden.py, committed with its fixtures).
 *
 * The entry points take the same descriptor structs as the product ABI
 * (include/resihp_b200.h) but HOST pointers.
 */
#ifndef RESIHP_ORACLE_H
#define RESIHP_ORACLE_H

#include <stdint.h>
#include "../include/resihp_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* workload.py:83-85 */
int64_t orc_quad_load(int32_t n_docs, const int32_t* docs);
/* workload.py:52-80 pack_sequences, literally (sort descending, first fit by
 * scanning the bins in creation order, residual appended as padding), keeping
 * the first max_bins bins (harness.py:251-252; max_bins < 0 = all).  Same
 * contract as rh_pack_sequences: mb_off / doc_len may be NULL to size the
 * output.  Returns -1 for a length <= 0 or > budget. */
int orc_pack_sequences(int64_t n_docs, const int32_t* lengths, int32_t budget, int64_t max_bins,
                       int32_t* mb_off, int32_t* doc_len, int64_t* n_bins, int64_t* n_entries);
/* workload.py:88-98; kind 0=F 1=B 2=W 3=BW.  Returns 0 and sets *bad when
 * speed <= 0 (the reference raises ValueError). */
double orc_chunk_time(const rh_cost_model* m, int kind, int64_t quad,
                      int32_t budget, int32_t layers, double speed, int* bad);

/* pipeline.py:92-118: writes kinds/ids of the stage sequence, returns length */
int orc_stage_sequence(int schedule, int pp, int stage, int m, int first_id,
                       int* kinds, int* ids);

/* pipeline.py:259-292 on an edge list; returns 1 on a cycle (CycleError). */
int orc_critical_path(int32_t nv, const double* cost, int32_t ne,
                      const int32_t* src, const int32_t* dst, const double* w,
                      double* starts, double* makespan);

/* Canonical build_dag + critical_path + stage sums + activation check for a
 * batch (pipeline.py:129-292,446-453,516-539).  n_threads <= 0: all cores. */
int orc_pipeline_batch(const rh_pipe_shape* shape, const rh_cost_model* model,
                       const rh_segments* segs, const rh_trace* trace,
                       const rh_pass_out* out, int n_threads);

/* Predictor on the known view fused with filter_candidate + validate
 * (detector.py:111-158), same contract as rh_detect_batch. */
int orc_detect_batch(const rh_pipe_shape* shape, const rh_cost_model* model,
                     const rh_segments* segs, const rh_trace* trace,
                     double threshold, const rh_pass_out* out, int n_threads);

/* detector.py:127-158 on arrays (expected == NULL: link-ratio mode). */
int orc_validate(int64_t n, const double* measured, const double* expected,
                 double threshold, uint8_t* flag, double* severity);

/* detector.py:94-108 */
int orc_change_point(int64_t len, const double* series, int window, double kappa);

/* DetectorState.observe state machine, detector.py:198-271 */
int orc_screen(const rh_screen_params* params, int64_t series_len,
               const double* hist, int64_t n, const double* observed,
               const uint8_t* it_status, const uint8_t* reset, uint8_t* outcome,
               int64_t* series_len_out);

/* scratch for one canonical DAG evaluation (sized by `sh`) */
void* orc_scratch_new(const rh_pipe_shape* sh);
void orc_scratch_delete(void* s);
int64_t* orc_scratch_quad(void* s);  /* [M] quad loads consumed by orc_dag_iteration */
struct scratch_s;
uint8_t orc_dag_iteration(struct scratch_s* S, const rh_pipe_shape* sh,
                          const rh_cost_model* model, const rh_segments* sg, int seg,
                          double* makespan, double* stage_cost);

/* ---- re-plan search, restated on the CPU (search_oracle.c) */
typedef struct orc_search orc_search;
orc_search* orc_search_create(const rh_search_desc* desc);
void orc_search_destroy(orc_search* s);
int64_t orc_search_size(const orc_search* s);
/* score of one candidate: evaluate_plan makespan (canonical DAG + Kahn,
 * capacity) + amortised reconfiguration surcharge; +inf when infeasible */
double orc_search_score(orc_search* s, int64_t index);
/* lexicographic (score, index) min over [begin, end) on n_threads */
/* the same scores and (score, index) winner, with each replica pipeline's
 * critical path computed once per (layout, partition, replica, first
 * micro-batch, count) and reused across assignment variants (max is exact):
 * full-space argmin at 10^6-10^7 candidates in seconds */
int orc_search_eval_memo(orc_search* s, int64_t begin, int64_t end, int n_threads,
                         double* best_score, int64_t* best_index, double* scores);
int orc_search_eval(orc_search* s, int64_t begin, int64_t end, int n_threads,
                    double* best_score, int64_t* best_index, double* scores);
int orc_search_decode(orc_search* s, int64_t index, rh_candidate* out, int32_t* groups,
                      int32_t* partition, int32_t* counts);

#ifdef __cplusplus
}
#endif
#endif
