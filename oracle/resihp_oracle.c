/*
 * TEST INFRASTRUCTURE — NOT PRODUCT CODE.  See resihp_oracle.h.
 *
 * A deliberately literal restatement of the reference: it materialises the
 * chunk DAG exactly as build_dag does (same vertex creation order, same edge
 * list) and runs the same Kahn relaxation as critical_path, instead of the
 * product's wavefront recurrence.  Compiled with -ffp-contract=off so every
 * a*b+c rounds twice, as CPython's float arithmetic does.
 */
#include "resihp_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

enum { K_F = 0, K_B = 1, K_W = 2, K_BW = 3, K_AR = 4 };

/* workload.py:83-85  quad_load = sum(l*l for l in mb.doc_lengths) */
int64_t orc_quad_load(int32_t n_docs, const int32_t* docs) {
  int64_t q = 0;
  for (int32_t i = 0; i < n_docs; ++i) q += (int64_t)docs[i] * (int64_t)docs[i];
  return q;
}

static int cmp_desc_i32(const void* a, const void* b) {
  const int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return (x < y) - (x > y);
}

/* workload.py:52-80
 *   for l in sorted(lengths, reverse=True):
 *       for i, space in enumerate(remaining):
 *           if l <= space: bins[i].append(l); remaining[i] -= l; break
 *       else: bins.append([l]); remaining.append(token_budget - l)
 *   padding document = residual space, when > 0                            */
int orc_pack_sequences(int64_t n_docs, const int32_t* lengths, int32_t budget, int64_t max_bins,
                       int32_t* mb_off, int32_t* doc_len, int64_t* n_bins, int64_t* n_entries) {
  int32_t* v = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n_docs > 0 ? n_docs : 1));
  int64_t* rem = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_docs > 0 ? n_docs : 1));
  int64_t* bin_of = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_docs > 0 ? n_docs : 1));
  int64_t nb = 0, i, b;
  for (i = 0; i < n_docs; ++i) {
    if (lengths[i] <= 0 || lengths[i] > budget) {
      free(v);
      free(rem);
      free(bin_of);
      return -1;
    }
    v[i] = lengths[i];
  }
  qsort(v, (size_t)n_docs, sizeof(int32_t), cmp_desc_i32);
  for (i = 0; i < n_docs; ++i) {
    for (b = 0; b < nb; ++b)
      if (v[i] <= rem[b]) break;
    if (b == nb) rem[nb++] = budget;
    rem[b] -= v[i];
    bin_of[i] = b;
  }
  const int64_t keep = (max_bins >= 0 && max_bins < nb) ? max_bins : nb;
  /* documents of bin b in insertion order (= the sorted order), then padding */
  int64_t* start = (int64_t*)calloc((size_t)(nb + 1), sizeof(int64_t));
  for (i = 0; i < n_docs; ++i) ++start[bin_of[i] + 1];
  for (b = 0; b < nb; ++b) start[b + 1] += start[b] + (rem[b] > 0 ? 1 : 0);
  if (doc_len) {
    int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nb > 0 ? nb : 1));
    for (b = 0; b < nb; ++b) fill[b] = start[b];
    for (i = 0; i < n_docs; ++i)
      if (bin_of[i] < keep) doc_len[fill[bin_of[i]]++] = v[i];
    for (b = 0; b < keep; ++b)
      if (rem[b] > 0) doc_len[fill[b]] = (int32_t)rem[b];
    free(fill);
  }
  if (mb_off)
    for (b = 0; b <= keep; ++b) mb_off[b] = (int32_t)start[b];
  const int64_t e = start[keep];
  free(start);
  *n_bins = keep;
  *n_entries = e;
  free(v);
  free(rem);
  free(bin_of);
  return 0;
}

/* workload.py:46-49  ratio(BW) = B + W */
static double ratio_of(const rh_cost_model* m, int kind) {
  switch (kind) {
    case K_F: return m->ratio_f;
    case K_B: return m->ratio_b;
    case K_W: return m->ratio_w;
    default: return m->ratio_b + m->ratio_w;
  }
}

/* workload.py:88-98
 *   base = model.alpha * mb.token_budget + model.beta * quad_load(mb)
 *   return model.ratio(kind) * layers_on_stage * base / device_speed      */
double orc_chunk_time(const rh_cost_model* m, int kind, int64_t quad,
                      int32_t budget, int32_t layers, double speed, int* bad) {
  if (speed <= 0.0) {
    if (bad) *bad = 1;
    return 0.0;
  }
  double lin = m->alpha * (double)budget;
  double qd = m->beta * (double)quad;
  double base = lin + qd;
  double rl = ratio_of(m, kind) * (double)layers;
  double num = rl * base;
  return num / speed;
}

/* pipeline.py:92-101 (1F1B) and 104-118 (ZBH). mb ids are first_id.. */
int orc_stage_sequence(int schedule, int pp, int stage, int m, int first_id,
                       int* kinds, int* ids) {
  int w = pp - 1 - stage;
  if (m < w) w = m;
  int n = 0;
  for (int k = 0; k < w; ++k) { kinds[n] = K_F; ids[n++] = first_id + k; }
  if (schedule == RH_SCHED_1F1B) {
    for (int k = 0; k < m - w; ++k) {
      kinds[n] = K_F; ids[n++] = first_id + w + k;
      kinds[n] = K_BW; ids[n++] = first_id + k;
    }
    for (int k = m - w; k < m; ++k) { kinds[n] = K_BW; ids[n++] = first_id + k; }
  } else {
    for (int k = 0; k < m - w; ++k) {
      kinds[n] = K_F; ids[n++] = first_id + w + k;
      kinds[n] = K_B; ids[n++] = first_id + k;
    }
    int next_w = 0;
    for (int k = m - w; k < m; ++k) {
      kinds[n] = K_B; ids[n++] = first_id + k;
      kinds[n] = K_W; ids[n++] = first_id + next_w;
      ++next_w;
    }
    for (int k = next_w; k < m; ++k) { kinds[n] = K_W; ids[n++] = first_id + k; }
  }
  return n;
}

/* pipeline.py:259-292 — Kahn order, starts init 0.0, strict '>' relaxation,
 * makespan = max(0.0, max(starts[i] + cost[i])). */
int orc_critical_path(int32_t nv, const double* cost, int32_t ne,
                      const int32_t* src, const int32_t* dst, const double* w,
                      double* starts, double* makespan) {
  int32_t* indeg = (int32_t*)calloc((size_t)nv + 1, sizeof(int32_t));
  int32_t* off = (int32_t*)calloc((size_t)nv + 2, sizeof(int32_t));
  int32_t* adj = (int32_t*)malloc(sizeof(int32_t) * ((size_t)ne + 1));
  int32_t* fill = (int32_t*)calloc((size_t)nv + 1, sizeof(int32_t));
  int32_t* queue = (int32_t*)malloc(sizeof(int32_t) * ((size_t)nv + 1));
  /* succ[u] keeps edges in edge-list order (pipeline.py:268-271) */
  for (int32_t e = 0; e < ne; ++e) { off[src[e] + 1]++; indeg[dst[e]]++; }
  for (int32_t v = 0; v < nv; ++v) off[v + 1] += off[v];
  for (int32_t e = 0; e < ne; ++e) adj[off[src[e]] + fill[src[e]]++] = e;
  int32_t qn = 0, head = 0, processed = 0;
  for (int32_t v = 0; v < nv; ++v) {
    starts[v] = 0.0;
    if (indeg[v] == 0) queue[qn++] = v;
  }
  while (head < qn) {
    int32_t u = queue[head++];
    processed++;
    double finish = starts[u] + cost[u];
    for (int32_t k = off[u]; k < off[u + 1]; ++k) {
      int32_t e = adj[k];
      int32_t v = dst[e];
      double cand = finish + w[e];
      if (cand > starts[v]) starts[v] = cand;
      if (--indeg[v] == 0) queue[qn++] = v;
    }
  }
  int cyc = processed < nv;
  double ms = 0.0;
  for (int32_t v = 0; v < nv; ++v) {
    double f = starts[v] + cost[v];
    if (f > ms) ms = f; /* Python max(makespan, x): keeps first on ties */
  }
  *makespan = ms;
  free(indeg); free(off); free(adj); free(fill); free(queue);
  return cyc;
}

/* --------------------------------------------------------------- batch DAG */

typedef struct scratch_s {
  /* scratch sized for the largest iteration of a batch */
  int cap_v, cap_e;
  int* kind; int* mb; int* stage; int* rep;
  double* cost; double* starts;
  int32_t* src; int32_t* dst; double* w;
  int* vid_f; int* vid_b; int* vid_w; /* [M][P] vertex ids */
  int* chain_first; int* chain_last;  /* [D][P] */
  int* seq_kind; int* seq_id;
  int64_t* quad;
  double* ev_t; int* ev_d;
} scratch_t;

void orc_scratch_init(scratch_t* s, const rh_pipe_shape* sh);
void orc_scratch_free(scratch_t* s);
static uint8_t dag_iteration(scratch_t* S, const rh_pipe_shape* sh,
                             const rh_cost_model* model, const rh_segments* sg, int seg,
                             double* makespan, double* stage_cost);
uint8_t orc_dag_iteration(scratch_t* S, const rh_pipe_shape* sh, const rh_cost_model* model,
                          const rh_segments* sg, int seg, double* makespan,
                          double* stage_cost) {
  return dag_iteration(S, sh, model, sg, seg, makespan, stage_cost);
}
static void scratch_init(scratch_t* s, const rh_pipe_shape* sh) {
  int c = sh->schedule == RH_SCHED_1F1B ? 2 : 3;
  int M = sh->micro_batches, P = sh->pp, D = sh->dp;
  s->cap_v = c * M * P + D + 1;
  s->cap_e = 3 * c * M * P + D * P + 1;
  s->kind = malloc(sizeof(int) * s->cap_v);
  s->mb = malloc(sizeof(int) * s->cap_v);
  s->stage = malloc(sizeof(int) * s->cap_v);
  s->rep = malloc(sizeof(int) * s->cap_v);
  s->cost = malloc(sizeof(double) * s->cap_v);
  s->starts = malloc(sizeof(double) * s->cap_v);
  s->src = malloc(sizeof(int32_t) * s->cap_e);
  s->dst = malloc(sizeof(int32_t) * s->cap_e);
  s->w = malloc(sizeof(double) * s->cap_e);
  s->vid_f = malloc(sizeof(int) * (M * P + 1));
  s->vid_b = malloc(sizeof(int) * (M * P + 1));
  s->vid_w = malloc(sizeof(int) * (M * P + 1));
  s->chain_first = malloc(sizeof(int) * (D * P + 1));
  s->chain_last = malloc(sizeof(int) * (D * P + 1));
  s->seq_kind = malloc(sizeof(int) * (3 * M + 1));
  s->seq_id = malloc(sizeof(int) * (3 * M + 1));
  s->quad = malloc(sizeof(int64_t) * (M + 1));
  s->ev_t = malloc(sizeof(double) * (2 * M + 2));
  s->ev_d = malloc(sizeof(int) * (2 * M + 2));
}

void orc_scratch_init(scratch_t* s, const rh_pipe_shape* sh) { scratch_init(s, sh); }
void* orc_scratch_new(const rh_pipe_shape* sh) {
  scratch_t* s = (scratch_t*)malloc(sizeof(scratch_t));
  scratch_init(s, sh);
  return s;
}
int64_t* orc_scratch_quad(void* s) { return ((scratch_t*)s)->quad; }
static void scratch_free(scratch_t* s);
void orc_scratch_free(scratch_t* s) { scratch_free(s); }
void orc_scratch_delete(void* s) {
  scratch_free((scratch_t*)s);
  free(s);
}
static void scratch_free(scratch_t* s) {
  free(s->kind); free(s->mb); free(s->stage); free(s->rep); free(s->cost);
  free(s->starts); free(s->src); free(s->dst); free(s->w); free(s->vid_f);
  free(s->vid_b); free(s->vid_w); free(s->chain_first); free(s->chain_last);
  free(s->seq_kind); free(s->seq_id); free(s->quad); free(s->ev_t); free(s->ev_d);
}

typedef struct { double t; int d; } ev_t;
static int ev_cmp(const void* a, const void* b) {
  const ev_t* x = (const ev_t*)a; const ev_t* y = (const ev_t*)b;
  if (x->t < y->t) return -1;
  if (x->t > y->t) return 1;
  return (x->d > y->d) - (x->d < y->d);
}

/*
 * One iteration: build_dag (pipeline.py:129-256) with the segment's speeds,
 * hop weights and AR costs, critical_path, stage sums (pipeline.py:446-453)
 * and _check_activation_memory (pipeline.py:516-539).
 */
static uint8_t dag_iteration(scratch_t* S, const rh_pipe_shape* sh,
                             const rh_cost_model* model, const rh_segments* sg, int seg,
                             double* makespan, double* stage_cost);

static uint8_t run_iteration(scratch_t* S, const rh_pipe_shape* sh,
                             const rh_cost_model* model, const rh_segments* sg,
                             const rh_trace* tr, int64_t it, double* makespan,
                             double* stage_cost /* [D][P] or NULL */) {
  const int M = sh->micro_batches;
  for (int j = 0; j < M; ++j) {
    int64_t a = tr->mb_off[it * M + j], b = tr->mb_off[it * M + j + 1];
    S->quad[j] = orc_quad_load((int32_t)(b - a), tr->doc_len + a);
  }
  return dag_iteration(S, sh, model, sg, tr->seg ? tr->seg[it] : 0, makespan, stage_cost);
}

/* One iteration given S->quad[]: build_dag + critical_path + stage sums +
 * activation check for segment `seg`. */
static uint8_t dag_iteration(scratch_t* S, const rh_pipe_shape* sh,
                             const rh_cost_model* model, const rh_segments* sg, int seg,
                             double* makespan, double* stage_cost) {
  const int P = sh->pp, D = sh->dp, M = sh->micro_batches;
  const int zbh = sh->schedule == RH_SCHED_ZBH;
  const int32_t* layers = sg->layers + (int64_t)seg * P;
  const int32_t* mb_start = sg->mb_start + (int64_t)seg * (D + 1);
  const double* speed = sg->speed + (int64_t)seg * D * P;
  const double* hf = sg->hop_fwd + (int64_t)seg * D * P;
  const double* hb = sg->hop_bwd + (int64_t)seg * D * P;
  uint8_t status = 0;
  (void)M;
  /* completeness check (pipeline.py:408-415): every chunk's stage alive */
  for (int d = 0; d < D; ++d)
    if (mb_start[d + 1] > mb_start[d])
      for (int s = 0; s < P; ++s)
        if (speed[d * P + s] <= 0.0) status |= RH_IT_STOPPED;
  if (status) {
    *makespan = 0.0;
    if (stage_cost) for (int k = 0; k < D * P; ++k) stage_cost[k] = 0.0;
    return status;
  }

  int nv = 0, ne = 0;
  for (int d = 0; d < D; ++d) {
    int first = mb_start[d], m = mb_start[d + 1] - mb_start[d];
    for (int s = 0; s < P; ++s) {
      S->chain_first[d * P + s] = -1;
      S->chain_last[d * P + s] = -1;
      if (m == 0) continue;
      int n = orc_stage_sequence(sh->schedule, P, s, m, first, S->seq_kind, S->seq_id);
      double sp = speed[d * P + s];
      int prev = -1;
      for (int k = 0; k < n; ++k) {
        int kind = S->seq_kind[k], j = S->seq_id[k];
        int bad = 0;
        double c = orc_chunk_time(model, kind, S->quad[j], sh->token_budget,
                                  layers[s], sp, &bad);
        int v = nv++;
        S->kind[v] = kind; S->mb[v] = j; S->stage[v] = s; S->rep[v] = d;
        S->cost[v] = c;
        if (kind == K_F) S->vid_f[j * P + s] = v;
        else if (kind == K_W) S->vid_w[j * P + s] = v;
        else S->vid_b[j * P + s] = v;
        if (prev >= 0) { S->src[ne] = prev; S->dst[ne] = v; S->w[ne] = 0.0; ne++; }
        if (S->chain_first[d * P + s] < 0) S->chain_first[d * P + s] = v;
        prev = v;
      }
      S->chain_last[d * P + s] = prev;
    }
  }
  /* data edges in micro-batch order (pipeline.py:224-240) */
  for (int d = 0; d < D; ++d) {
    for (int j = mb_start[d]; j < mb_start[d + 1]; ++j) {
      for (int s = 1; s < P; ++s) {
        S->src[ne] = S->vid_f[j * P + s - 1]; S->dst[ne] = S->vid_f[j * P + s];
        S->w[ne] = hf[d * P + s - 1]; ne++;
      }
      for (int s = 0; s < P - 1; ++s) {
        S->src[ne] = S->vid_b[j * P + s + 1]; S->dst[ne] = S->vid_b[j * P + s];
        S->w[ne] = hb[d * P + s]; ne++;
      }
      if (zbh)
        for (int s = 0; s < P; ++s) {
          S->src[ne] = S->vid_b[j * P + s]; S->dst[ne] = S->vid_w[j * P + s];
          S->w[ne] = 0.0; ne++;
        }
    }
  }
  int n_chunk = nv;
  /* terminal all-reduce vertices (pipeline.py:242-254) */
  if (D > 1 && sh->has_allreduce) {
    const double* ar = sg->allreduce + (int64_t)seg * D;
    for (int d = 0; d < D; ++d) {
      int v = nv++;
      S->kind[v] = K_AR; S->mb[v] = -1; S->stage[v] = -1; S->rep[v] = d;
      S->cost[v] = ar[d];
      for (int s = 0; s < P; ++s) {
        int last = S->chain_last[d * P + s];
        if (last >= 0) { S->src[ne] = last; S->dst[ne] = v; S->w[ne] = 0.0; ne++; }
      }
    }
  }
  double ms;
  orc_critical_path(nv, S->cost, ne, S->src, S->dst, S->w, S->starts, &ms);
  *makespan = ms;

  if (stage_cost) {
    for (int k = 0; k < D * P; ++k) stage_cost[k] = 0.0;
    for (int v = 0; v < n_chunk; ++v)
      stage_cost[S->rep[v] * P + S->stage[v]] += S->cost[v];
  }
  /* _check_activation_memory (pipeline.py:516-539), per (replica, stage) */
  if (sh->capacity > 0) {
    ev_t* evs = (ev_t*)malloc(sizeof(ev_t) * (2 * (size_t)M + 2));
    for (int d = 0; d < D && !(status & RH_IT_CAPACITY); ++d)
      for (int s = 0; s < P; ++s) {
        int first = S->chain_first[d * P + s];
        if (first < 0) continue;
        int ne2 = 0;
        for (int v = first; v <= S->chain_last[d * P + s]; ++v) {
          if (S->kind[v] == K_F) { evs[ne2].t = S->starts[v]; evs[ne2++].d = 1; }
          else if (S->kind[v] == K_B || S->kind[v] == K_BW) {
            evs[ne2].t = S->starts[v] + S->cost[v]; evs[ne2++].d = -1;
          }
        }
        qsort(evs, ne2, sizeof(ev_t), ev_cmp);
        int live = 0;
        for (int k = 0; k < ne2; ++k) {
          live += evs[k].d;
          if (live > sh->capacity) { status |= RH_IT_CAPACITY; break; }
        }
        if (status & RH_IT_CAPACITY) break;
      }
    free(evs);
  }
  return status;
}

/* detector.py:111-116 and 127-158 on one iteration */
static uint8_t detect_tail(const rh_pipe_shape* sh, const rh_segments* sg,
                           const rh_trace* tr, int64_t it, double threshold,
                           double predicted, const double* expected,
                           uint8_t* flags, float* sev) {
  const int P = sh->pp, D = sh->dp, T = sh->tp;
  uint8_t st = 0;
  /* filter_candidate */
  double observed = tr->observed[it];
  if (predicted <= 0.0 || observed > threshold * predicted) st |= RH_IT_ESCALATE;
  /* validate: per (replica, stage) */
  for (int g = 0; g < D * P; ++g) {
    const float* dt = tr->device_time + (it * D * P + g) * (int64_t)T;
    float mx = 0.0f;
    for (int t = 0; t < T; ++t) if (dt[t] > mx) mx = dt[t];
    double measured = (double)mx;
    double exp_ = expected[g];
    uint8_t f = 0;
    float sv = 0.0f;
    if (!(exp_ <= 0.0 || measured <= 0.0) && measured > threshold * exp_) {
      f = 1;
      sv = (float)(exp_ / measured);
      st |= RH_IT_STAGE_FLAG;
    }
    if (flags) flags[it * D * P + g] = f;
    if (sev) sev[it * D * P + g] = sv;
  }
  /* link ratios (detector.py:148-152) */
  if (sg->link_off) {
    int seg = tr->seg ? tr->seg[it] : 0;
    for (int32_t k = sg->link_off[seg]; k < sg->link_off[seg + 1]; ++k)
      if (sg->link_ratio[k] > threshold) st |= RH_IT_LINK_FLAG;
  }
  return st;
}

typedef struct {
  const rh_pipe_shape* sh; const rh_cost_model* model; const rh_segments* sg;
  const rh_trace* tr; const rh_pass_out* out; double threshold; int detect;
  int64_t begin, end;
} job_t;

static void* worker(void* arg) {
  job_t* J = (job_t*)arg;
  scratch_t S;
  scratch_init(&S, J->sh);
  const int DP = J->sh->dp * J->sh->pp;
  double* sc = malloc(sizeof(double) * (DP + 1));
  for (int64_t it = J->begin; it < J->end; ++it) {
    double ms = 0.0;
    uint8_t st = run_iteration(&S, J->sh, J->model, J->sg, J->tr, it, &ms, sc);
    J->out->makespan[it] = ms;
    if (J->out->stage_cost)
      memcpy(J->out->stage_cost + it * DP, sc, sizeof(double) * DP);
    if (J->detect && !(st & RH_IT_STOPPED)) {
      st |= detect_tail(J->sh, J->sg, J->tr, it, J->threshold, ms, sc,
                        J->out->stage_flag, J->out->severity);
    } else if (J->detect) {
      if (J->out->stage_flag) memset(J->out->stage_flag + it * DP, 0, DP);
      if (J->out->severity) memset(J->out->severity + it * DP, 0, sizeof(float) * DP);
    }
    J->out->status[it] = st;
  }
  free(sc);
  scratch_free(&S);
  return NULL;
}

static int run_batch(const rh_pipe_shape* sh, const rh_cost_model* model,
                     const rh_segments* sg, const rh_trace* tr,
                     const rh_pass_out* out, double thr, int detect, int n_threads) {
  if (n_threads <= 0) n_threads = (int)sysconf(_SC_NPROCESSORS_ONLN);
  if (n_threads < 1) n_threads = 1;
  int64_t n = tr->n_iter;
  if (n_threads > n) n_threads = (int)(n > 0 ? n : 1);
  pthread_t* th = malloc(sizeof(pthread_t) * n_threads);
  job_t* jobs = malloc(sizeof(job_t) * n_threads);
  for (int k = 0; k < n_threads; ++k) {
    jobs[k] = (job_t){sh, model, sg, tr, out, thr, detect,
                      n * k / n_threads, n * (k + 1) / n_threads};
    if (n_threads == 1) worker(&jobs[k]);
    else pthread_create(&th[k], NULL, worker, &jobs[k]);
  }
  if (n_threads > 1)
    for (int k = 0; k < n_threads; ++k) pthread_join(th[k], NULL);
  free(th); free(jobs);
  return 0;
}

int orc_pipeline_batch(const rh_pipe_shape* shape, const rh_cost_model* model,
                       const rh_segments* segs, const rh_trace* trace,
                       const rh_pass_out* out, int n_threads) {
  return run_batch(shape, model, segs, trace, out, 0.0, 0, n_threads);
}

int orc_detect_batch(const rh_pipe_shape* shape, const rh_cost_model* model,
                     const rh_segments* segs, const rh_trace* trace,
                     double threshold, const rh_pass_out* out, int n_threads) {
  return run_batch(shape, model, segs, trace, out, threshold, 1, n_threads);
}

/* detector.py:141-152 */
int orc_validate(int64_t n, const double* measured, const double* expected,
                 double threshold, uint8_t* flag, double* severity) {
  for (int64_t i = 0; i < n; ++i) {
    flag[i] = 0;
    severity[i] = 0.0;
    if (expected) {
      if (expected[i] <= 0.0 || measured[i] <= 0.0) continue;
      if (measured[i] > threshold * expected[i]) {
        flag[i] = 1;
        severity[i] = expected[i] / measured[i];
      }
    } else if (measured[i] > threshold) {
      flag[i] = 1;
      severity[i] = 1.0 / measured[i];
    }
  }
  return 0;
}

/* ----------------------------------------------------------- the screen */

static int dbl_cmp(const void* a, const void* b) {
  double x = *(const double*)a, y = *(const double*)b;
  return (x > y) - (x < y);
}

/* statistics.median: sorted; odd -> middle, even -> (a + b) / 2 */
static double median_sorted(const double* v, int n) {
  if (n % 2 == 1) return v[n / 2];
  return (v[n / 2 - 1] + v[n / 2]) / 2.0;
}

/* detector.py:94-108 */
int orc_change_point(int64_t len, const double* series, int window, double kappa) {
  if (len < window + 1) return 0;
  double* win = malloc(sizeof(double) * (window + 1));
  memcpy(win, series + len - window - 1, sizeof(double) * window);
  qsort(win, window, sizeof(double), dbl_cmp);
  double med = median_sorted(win, window);
  for (int k = 0; k < window; ++k) win[k] = fabs(series[len - window - 1 + k] - med);
  qsort(win, window, sizeof(double), dbl_cmp);
  double mad = median_sorted(win, window);
  double x = series[len - 1];
  free(win);
  return fabs(x - med) > kappa * mad;
}

/* DetectorState.observe, detector.py:198-271 (+ reset_series, :195-196) */
int orc_screen(const rh_screen_params* p, int64_t series_len, const double* hist,
               int64_t n, const double* observed, const uint8_t* it_status,
               const uint8_t* reset, uint8_t* outcome, int64_t* series_len_out) {
  const int w = p->window;
  int64_t h = series_len < w ? series_len : w;
  /* buffer holds the visible tail of the series; len is the full length */
  double* buf = malloc(sizeof(double) * (size_t)(h + n + 1));
  memcpy(buf, hist, sizeof(double) * (size_t)h);
  int64_t nb = h, len = series_len;
  for (int64_t i = 0; i < n; ++i) {
    if (reset && reset[i]) { nb = 0; len = 0; }
    buf[nb++] = observed[i];
    len++;
    uint8_t oc = 0;
    int cand = (len >= w + 1) && orc_change_point(nb, buf, w, p->kappa);
    int refill = !cand && p->filter_enabled && len <= w;
    if (!cand && !refill) { outcome[i] = 0; continue; }
    if (cand) oc |= RH_SC_CANDIDATE;
    if (p->filter_enabled) {
      oc |= RH_SC_FILTERED;
      if (!(it_status[i] & RH_IT_ESCALATE)) {
        if (cand) { nb--; len--; oc |= RH_SC_POPPED; }
        outcome[i] = oc;
        continue;
      }
    }
    oc |= RH_SC_ESCALATED;
    if (!(it_status[i] & (RH_IT_STAGE_FLAG | RH_IT_LINK_FLAG))) {
      nb--; len--;
      oc |= RH_SC_POPPED;
    } else {
      oc |= RH_SC_CONFIRMED;
    }
    outcome[i] = oc;
  }
  if (series_len_out) *series_len_out = len;
  free(buf);
  return 0;
}
