/*
 * TEST INFRASTRUCTURE — NOT PRODUCT CODE.  See resihp_oracle.h.
 *
 * CPU restatement of the re-plan search.  Each candidate is
 * scored the way resihp_adapt scores a variant (policies.py:329-347):
 * evaluate_plan (scheduler.py:543-559) — here: the canonical chunk DAG built
 * literally (build_dag, pipeline.py:129-256) and Kahn's relaxation
 * (critical_path, pipeline.py:259-292) with the activation check
 * (pipeline.py:516-539) — plus reconfig_cost (scheduler.py:562-593) divided
 * by the amortisation horizon (policies.py:341-345).  Layout placement,
 * repartition_layers (scheduler.py:146-207) and proportional_split
 * (policies.py:151-162) are restated here independently of the CUDA code.
 * Candidate makespans are pinned to the reference's own evaluate_plan on
 * sampled candidates (tests/golden/search.json).
 */
#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#include "resihp_oracle.h"

typedef struct {
  int T, D, P;
  int64_t base, nv, nu;
  int* gblk;      /* [D*P] block index (global) */
  double* gspeed; /* [D*P] effective group speed */
  double* hop;    /* [D*P] boundary hop (s < P-1) */
  double* ring;   /* [P] all-reduce ring bandwidth */
  int* repart;    /* [P] */
  int* prop;      /* [D] proportional counts */
  int same;       /* same groups as the current plan */
} layout_t;

struct orc_search {
  rh_search_desc d;
  double* speed;
  int* link_nodes;
  double* link_factor;
  int64_t* quad;
  int* cur_groups;
  int* cur_part;
  int n_nodes;
  /* blocks */
  int nblk;
  int* blk_node;
  double* blk_speed;
  int* blk_rank;
  int* blk_moff;
  int* blk_mem;
  int blk_T[8], blk_off[8], blk_n[8], n_deg;
  /* layouts */
  int nl;
  layout_t* L;
  int64_t total;
  int maxD, maxP, T0;
  double worst_inter;
};

static double inter_bw(const orc_search* s, int a, int b) {
  int lo = a < b ? a : b, hi = a < b ? b : a;
  double f = 1.0;
  for (int q = 0; q < s->d.n_links; ++q)
    if (s->link_nodes[2 * q] == lo && s->link_nodes[2 * q + 1] == hi) { f = s->link_factor[q]; break; }
  return s->d.inter_bw * f;
}

/* edge_cost_fn (pipeline.py:336-353) + p2p_cost (comm.py:61-84) */
static double edge_cost(const orc_search* s, int na, int nb, int T) {
  if (!s->d.has_comm) return 0.0;
  double nbytes = s->d.hidden_bytes_per_token * (double)s->d.token_budget;
  if (na == nb) return nbytes / s->d.intra_bw;
  double inter = inter_bw(s, na, nb);
  if (!s->d.p2p_optimized) {
    double cross = (double)T * nbytes;
    return cross / inter;
  }
  int n = T;
  double gather = nbytes * (double)(n - 1) / ((double)n * s->d.intra_bw);
  return nbytes / inter + gather;
}

/* repartition_layers, scheduler.py:146-207 */
static void repartition(const double* sp, int n, int L, int ml, int* out) {
  double tot = 0.0;
  for (int i = 0; i < n; ++i) tot += sp[i];
  double share[64];
  int lay[64], chosen[64];
  int sum = 0;
  for (int i = 0; i < n; ++i) {
    share[i] = (double)L * sp[i] / tot;
    lay[i] = (int)floor(share[i]);
    sum += lay[i];
    chosen[i] = 0;
  }
  for (int r = 0; r < L - sum; ++r) { /* sorted by (-(share-layers), i) */
    int bi = -1;
    for (int i = 0; i < n; ++i) {
      if (chosen[i]) continue;
      if (bi < 0 || (share[i] - lay[i]) > (share[bi] - lay[bi])) bi = i;
    }
    chosen[bi] = 1;
  }
  for (int i = 0; i < n; ++i) lay[i] += chosen[i];
  for (;;) {
    int rec = -1, don = -1;
    for (int i = 0; i < n && rec < 0; ++i) if (lay[i] < ml) rec = i;
    if (rec < 0) break;
    for (int i = 0; i < n; ++i)
      if (lay[i] > ml && (don < 0 || lay[i] > lay[don])) don = i;
    if (don < 0) break;
    lay[don]--; lay[rec]++;
  }
  double min_gain = 1.0 / (2.0 * L);
  for (;;) {
    double cur = 0.0;
    for (int i = 0; i < n; ++i) { double x = lay[i] / sp[i]; if (i == 0 || x > cur) cur = x; }
    int bs = -1, bd = -1;
    double best = 0.0;
    for (int src = 0; src < n; ++src) {
      if (lay[src] <= ml) continue;
      for (int dst = 0; dst < n; ++dst) {
        if (dst == src) continue;
        lay[src]--; lay[dst]++;
        double c = 0.0;
        for (int i = 0; i < n; ++i) { double x = lay[i] / sp[i]; if (i == 0 || x > c) c = x; }
        lay[src]++; lay[dst]--;
        if (c < cur * (1.0 - min_gain) && (bs < 0 || c < best)) { best = c; bs = src; bd = dst; }
      }
    }
    if (bs < 0) break;
    lay[bs]--; lay[bd]++;
  }
  for (int i = 0; i < n; ++i) out[i] = lay[i];
}

/* proportional_split, policies.py:151-162 */
static void proportional(int total, const double* w, int n, int* out) {
  double wsum = 0.0;
  for (int i = 0; i < n; ++i) wsum += w[i];
  double share[64];
  int chosen[64], sum = 0;
  for (int i = 0; i < n; ++i) {
    share[i] = (double)total * w[i] / wsum;
    out[i] = (int)share[i];
    sum += out[i];
    chosen[i] = 0;
  }
  for (int r = 0; r < total - sum; ++r) {
    int bi = -1;
    for (int i = 0; i < n; ++i) {
      if (chosen[i]) continue;
      if (bi < 0 || (share[i] - out[i]) > (share[bi] - out[bi])) bi = i;
    }
    chosen[bi] = 1;
  }
  for (int i = 0; i < n; ++i) out[i] += chosen[i];
}

typedef struct { double v; int id; } sid_t;
static int by_speed_desc(const void* a, const void* b) {
  const sid_t* x = a; const sid_t* y = b;
  if (x->v > y->v) return -1;
  if (x->v < y->v) return 1;
  return (x->id > y->id) - (x->id < y->id);
}
static int int_cmp(const void* a, const void* b) {
  int x = *(const int*)a, y = *(const int*)b;
  return (x > y) - (x < y);
}

orc_search* orc_search_create(const rh_search_desc* desc) {
  orc_search* s = calloc(1, sizeof(orc_search));
  s->d = *desc;
  const rh_search_desc* d = desc;
  int n = d->n_devices, dpn = d->devices_per_node;
  s->speed = malloc(sizeof(double) * n);
  memcpy(s->speed, d->device_speed, sizeof(double) * n);
  s->link_nodes = malloc(sizeof(int) * (2 * d->n_links + 1));
  s->link_factor = malloc(sizeof(double) * (d->n_links + 1));
  if (d->n_links) {
    memcpy(s->link_nodes, d->link_nodes, sizeof(int) * 2 * d->n_links);
    memcpy(s->link_factor, d->link_factor, sizeof(double) * d->n_links);
  }
  s->quad = malloc(sizeof(int64_t) * d->n_micro_batches);
  memcpy(s->quad, d->quad, sizeof(int64_t) * d->n_micro_batches);
  int ncg = d->cur_tp * d->cur_dp * d->cur_pp;
  s->cur_groups = malloc(sizeof(int) * (ncg + 1));
  if (d->cur_groups && ncg) memcpy(s->cur_groups, d->cur_groups, sizeof(int) * ncg);
  s->cur_part = malloc(sizeof(int) * (d->cur_pp + 1));
  if (d->cur_partition && d->cur_pp) memcpy(s->cur_part, d->cur_partition, sizeof(int) * d->cur_pp);
  s->n_nodes = (n + dpn - 1) / dpn;
  s->T0 = d->nominal_tp > 0 ? d->nominal_tp : 1;
  double wf = 1.0;
  for (int q = 0; q < d->n_links; ++q) if (q == 0 || s->link_factor[q] < wf) wf = s->link_factor[q];
  s->worst_inter = d->inter_bw * wf; /* comm.py:38-40 (min(..., default=1.0)) */
  int executable = 0;
  for (int q = 0; q < n; ++q) executable += s->speed[q] > 0.0;
  /* blocks per TP degree */
  s->blk_node = malloc(sizeof(int) * (8 * n + 8));
  s->blk_speed = malloc(sizeof(double) * (8 * n + 8));
  s->blk_rank = malloc(sizeof(int) * (8 * n + 8));
  s->blk_moff = malloc(sizeof(int) * (8 * n + 8));
  s->blk_mem = malloc(sizeof(int) * (8 * n + 8));
  int nmem = 0;
  sid_t* tmp = malloc(sizeof(sid_t) * (dpn + n + 1));
  for (int T = 1; T <= dpn && T <= (d->max_tp > 0 ? d->max_tp : 1); T <<= 1) {
    if (dpn % T) continue;
    int di = s->n_deg++;
    s->blk_T[di] = T;
    s->blk_off[di] = s->nblk;
    for (int nd = 0; nd < s->n_nodes; ++nd) {
      int c = 0;
      for (int q = nd * dpn; q < (nd + 1) * dpn && q < n; ++q)
        if (s->speed[q] > 0.0) { tmp[c].v = s->speed[q]; tmp[c].id = q; c++; }
      qsort(tmp, c, sizeof(sid_t), by_speed_desc);
      for (int b = 0; b + T <= c; b += T) {
        int k = s->nblk++;
        s->blk_node[k] = nd;
        double mn = tmp[b].v;
        for (int t = 0; t < T; ++t) if (tmp[b + t].v < mn) mn = tmp[b + t].v;
        s->blk_speed[k] = mn;
        s->blk_moff[k] = nmem;
        for (int t = 0; t < T; ++t) s->blk_mem[nmem + t] = tmp[b + t].id;
        qsort(s->blk_mem + nmem, T, sizeof(int), int_cmp);
        nmem += T;
      }
    }
    s->blk_n[di] = s->nblk - s->blk_off[di];
    /* rank: speed desc, ties by position */
    int nb = s->blk_n[di];
    for (int b = 0; b < nb; ++b) {
      int r = 0;
      double v = s->blk_speed[s->blk_off[di] + b];
      for (int o = 0; o < nb; ++o) {
        double w = s->blk_speed[s->blk_off[di] + o];
        if (w > v || (w == v && o < b)) r++;
      }
      s->blk_rank[s->blk_off[di] + b] = r;
    }
  }
  free(tmp);
  /* layouts: T, then P, then D */
  int max_pp = d->max_pp > 0 && d->max_pp < 32 ? d->max_pp : 32;
  int max_dp = d->max_dp > 0 && d->max_dp < 64 ? d->max_dp : 64;
  int ml = d->min_layers > 1 ? d->min_layers : 1;
  int cap_l = 1024;
  s->L = malloc(sizeof(layout_t) * cap_l);
  for (int di = 0; di < s->n_deg; ++di) {
    int T = s->blk_T[di];
    for (int P = 1; P <= max_pp && P * ml <= d->total_layers; ++P)
      for (int D = 1; D <= max_dp && D <= d->n_micro_batches; ++D) {
        if (D * P > s->blk_n[di]) break;
        if ((double)T * D * P < d->min_utilization * executable) continue;
        if (s->nl == cap_l) { cap_l *= 2; s->L = realloc(s->L, sizeof(layout_t) * cap_l); }
        layout_t* l = &s->L[s->nl++];
        l->T = T; l->D = D; l->P = P;
        l->nv = 2 + (int64_t)P * (P - 1);
        l->nu = 2 + (int64_t)D * (D - 1);
        l->base = s->total;
        s->total += l->nv * l->nu;
        if (D > s->maxD) s->maxD = D;
        if (P > s->maxP) s->maxP = P;
        /* placement */
        int K = D * P, g = 0;
        l->gblk = malloc(sizeof(int) * K);
        for (int b = 0; b < s->blk_n[di]; ++b)
          if (s->blk_rank[s->blk_off[di] + b] < K) l->gblk[g++] = s->blk_off[di] + b;
        l->hop = calloc(K, sizeof(double));
        for (int q = 0; q < K; ++q)
          if (q % P < P - 1)
            l->hop[q] = edge_cost(s, s->blk_node[l->gblk[q]], s->blk_node[l->gblk[q + 1]], T);
        l->ring = malloc(sizeof(double) * P);
        /* effective_stage_speed: slowest * |group| / nominal_tp */
        l->gspeed = malloc(sizeof(double) * K);
        for (int q = 0; q < K; ++q)
          l->gspeed[q] = s->blk_speed[l->gblk[q]] * (double)T / (double)s->T0;
        double sspeed[64], rspeed[64];
        for (int st = 0; st < P; ++st) {
          int same = 1, n0 = s->blk_node[l->gblk[st]];
          sspeed[st] = l->gspeed[st];
          for (int r = 1; r < D; ++r) {
            same &= s->blk_node[l->gblk[r * P + st]] == n0;
            double v = l->gspeed[r * P + st];
            if (v < sspeed[st]) sspeed[st] = v;
          }
          double bw;
          if (same) bw = d->intra_bw;
          else {
            bw = d->inter_bw;
            for (int r = 0; r < D; ++r) {
              int a = s->blk_node[l->gblk[r * P + st]];
              int b = s->blk_node[l->gblk[((r + 1) % D) * P + st]];
              if (a != b) { double x = inter_bw(s, a, b); if (x < bw) bw = x; }
            }
          }
          l->ring[st] = bw;
        }
        for (int r = 0; r < D; ++r) {
          rspeed[r] = l->gspeed[r * P];
          for (int st = 1; st < P; ++st) {
            double v = l->gspeed[r * P + st];
            if (v < rspeed[r]) rspeed[r] = v;
          }
        }
        l->repart = malloc(sizeof(int) * P);
        repartition(sspeed, P, d->total_layers, d->min_layers, l->repart);
        l->prop = malloc(sizeof(int) * D);
        proportional(d->n_micro_batches, rspeed, D, l->prop);
        l->same = d->cur_tp == T && d->cur_dp == D && d->cur_pp == P && d->cur_groups;
        for (int q = 0; l->same && q < K; ++q)
          for (int t = 0; t < T; ++t)
            if (s->blk_mem[s->blk_moff[l->gblk[q]] + t] != s->cur_groups[q * T + t]) l->same = 0;
      }
  }
  return s;
}

void orc_search_destroy(orc_search* s) {
  if (!s) return;
  for (int i = 0; i < s->nl; ++i) {
    free(s->L[i].gblk); free(s->L[i].gspeed); free(s->L[i].hop); free(s->L[i].ring); free(s->L[i].repart);
    free(s->L[i].prop);
  }
  free(s->L); free(s->speed); free(s->link_nodes); free(s->link_factor); free(s->quad);
  free(s->cur_groups); free(s->cur_part); free(s->blk_node); free(s->blk_speed);
  free(s->blk_rank); free(s->blk_moff); free(s->blk_mem);
  free(s);
}

int64_t orc_search_size(const orc_search* s) { return s->total; }

static int find_layout(const orc_search* s, int64_t idx) {
  int lo = 0, hi = s->nl - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) / 2;
    if (s->L[mid].base <= idx) lo = mid; else hi = mid - 1;
  }
  return lo;
}

/* partition / counts of a candidate; returns feasibility */
static int decode(const orc_search* s, int64_t idx, int* li_out, int* part, int* cnt) {
  int li = find_layout(s, idx);
  const layout_t* l = &s->L[li];
  int64_t local = idx - l->base;
  int v = (int)(local / l->nu), u = (int)(local % l->nu);
  int P = l->P, D = l->D, Ltot = s->d.total_layers, M = s->d.n_micro_batches;
  for (int st = 0; st < P; ++st)
    part[st] = v == 0 ? Ltot / P + (st < Ltot % P ? 1 : 0) : l->repart[st];
  if (v >= 2) {
    int m = v - 2, r = m % (P - 1), src = m / (P - 1), dst = r < src ? r : r + 1;
    part[src]--; part[dst]++;
  }
  for (int r = 0; r < D; ++r) cnt[r] = u == 0 ? M / D + (r < M % D ? 1 : 0) : l->prop[r];
  if (u >= 2) {
    int m = u - 2, r = m % (D - 1), src = m / (D - 1), dst = r < src ? r : r + 1;
    cnt[src]--; cnt[dst]++;
  }
  *li_out = li;
  int ok = 1;
  for (int st = 0; st < P; ++st) ok &= part[st] >= s->d.min_layers;
  for (int r = 0; r < D; ++r) ok &= cnt[r] >= 0;
  return ok;
}

static double score_with(orc_search* s, int64_t idx, void* scratch) {
  int part[64], cnt[64], li;
  if (!decode(s, idx, &li, part, cnt)) return INFINITY;
  const layout_t* l = &s->L[li];
  int T = l->T, D = l->D, P = l->P, K = D * P;
  const rh_search_desc* d = &s->d;
  rh_pipe_shape sh = {P, D, T, d->schedule, d->n_micro_batches, d->token_budget, d->capacity,
                      d->has_comm, 0};
  int mb_start[65];
  mb_start[0] = 0;
  for (int r = 0; r < D; ++r) mb_start[r + 1] = mb_start[r] + cnt[r];
  double* speed = malloc(sizeof(double) * K);
  for (int q = 0; q < K; ++q) speed[q] = l->gspeed[q];
  /* _allreduce_map: worst ring over stages, same for every replica */
  double ar_v = 0.0;
  if (d->has_comm && D > 1)
    for (int st = 0; st < P; ++st) {
      double nbytes = (double)part[st] * d->layer_bytes;
      double x = 2.0 * nbytes * (double)(D - 1) / ((double)D * l->ring[st]);
      if (x > ar_v) ar_v = x;
    }
  double ar[64];
  for (int r = 0; r < D; ++r) ar[r] = ar_v;
  rh_segments sg = {1, part, mb_start, speed, l->hop, l->hop, ar, NULL, NULL};
  memcpy(orc_scratch_quad(scratch), s->quad, sizeof(int64_t) * d->n_micro_batches);
  double ms = 0.0;
  uint8_t st = orc_dag_iteration((struct scratch_s*)scratch, &sh, &d->model, &sg, 0, &ms, NULL);
  free(speed);
  if (st) return INFINITY;
  /* reconfig_cost (scheduler.py:562-593) generalised to layout changes */
  int same_P = P == d->cur_pp, changed = 0;
  long long moved = 0;
  if (same_P)
    for (int q = 0; q < P; ++q) {
      if (part[q] != s->cur_part[q]) changed = 1;
      if (part[q] > s->cur_part[q]) moved += part[q] - s->cur_part[q];
    }
  double reshard = 0.0;
  if (!l->same)
    for (int r = 0; r < D; ++r)
      for (int q = 0; q < P; ++q) reshard += (double)part[q] * d->layer_bytes;
  double sur = 0.0;
  if (!l->same || changed) {
    double transfer = ((double)moved * d->layer_bytes + reshard) / s->worst_inter;
    int am = d->amortize_iterations > 1 ? d->amortize_iterations : 1;
    sur = (d->group_rebuild_s + transfer) / (double)am;
  }
  return ms + sur;
}

static void* new_scratch(const orc_search* s) {
  rh_pipe_shape sh = {s->maxP, s->maxD, 1, s->d.schedule, s->d.n_micro_batches,
                      s->d.token_budget, 0, 1, 0};
  return orc_scratch_new(&sh);
}

double orc_search_score(orc_search* s, int64_t index) {
  void* scr = new_scratch(s);
  double v = score_with(s, index, scr);
  orc_scratch_delete(scr);
  return v;
}

typedef struct {
  orc_search* s;
  int64_t begin, end;
  double best;
  int64_t best_i;
  double* scores;
  int64_t base;
} sjob_t;

static void* sworker(void* arg) {
  sjob_t* J = arg;
  void* scr = new_scratch(J->s);
  J->best = INFINITY;
  J->best_i = -1;
  for (int64_t i = J->begin; i < J->end; ++i) {
    double v = score_with(J->s, i, scr);
    if (J->scores) J->scores[i - J->base] = v;
    if (v < J->best) { J->best = v; J->best_i = i; } /* index order: first wins ties */
  }
  orc_scratch_delete(scr);
  return NULL;
}

int orc_search_eval(orc_search* s, int64_t begin, int64_t end, int n_threads,
                    double* best_score, int64_t* best_index, double* scores) {
  if (n_threads <= 0) n_threads = (int)sysconf(_SC_NPROCESSORS_ONLN);
  int64_t n = end - begin;
  if (n_threads > n) n_threads = n > 0 ? (int)n : 1;
  pthread_t* th = malloc(sizeof(pthread_t) * n_threads);
  sjob_t* jobs = malloc(sizeof(sjob_t) * n_threads);
  for (int k = 0; k < n_threads; ++k) {
    jobs[k] = (sjob_t){s, begin + n * k / n_threads, begin + n * (k + 1) / n_threads,
                       INFINITY, -1, scores, begin};
    if (n_threads == 1) sworker(&jobs[0]);
    else pthread_create(&th[k], NULL, sworker, &jobs[k]);
  }
  if (n_threads > 1) for (int k = 0; k < n_threads; ++k) pthread_join(th[k], NULL);
  double b = INFINITY;
  int64_t bi = -1;
  for (int k = 0; k < n_threads; ++k) /* chunks are in index order */
    if (jobs[k].best_i >= 0 && (bi < 0 || jobs[k].best < b)) { b = jobs[k].best; bi = jobs[k].best_i; }
  *best_score = b;
  *best_index = bi;
  free(th); free(jobs);
  return 0;
}

int orc_search_decode(orc_search* s, int64_t index, rh_candidate* out, int32_t* groups,
                      int32_t* partition, int32_t* counts) {
  int part[64], cnt[64], li;
  int ok = decode(s, index, &li, part, cnt);
  const layout_t* l = &s->L[li];
  int64_t local = index - l->base;
  out->index = index; out->tp = l->T; out->dp = l->D; out->pp = l->P; out->layout = li;
  out->partition_variant = (int)(local / l->nu);
  out->count_variant = (int)(local % l->nu);
  out->feasible = ok;
  if (groups)
    for (int q = 0; q < l->D * l->P; ++q)
      for (int t = 0; t < l->T; ++t) groups[q * l->T + t] = s->blk_mem[s->blk_moff[l->gblk[q]] + t];
  if (partition) for (int q = 0; q < l->P; ++q) partition[q] = part[q];
  if (counts) for (int q = 0; q < l->D; ++q) counts[q] = cnt[q];
  return 0;
}

/*
 * Full-space argmin at the benchmarked sizes (10^6-10^7 candidates).  The
 * canonical DAG of a candidate is D disconnected replica pipelines plus one
 * terminal all-reduce vertex per replica (pipeline.py:242-254), so Kahn's
 * relaxation gives makespan = max_d RN(fin_d + AR) with fin_d the replica's
 * own critical path (AR >= 0; an empty replica contributes RN(0 + AR)), and
 * the candidate is infeasible when any replica is (a stopped stage with
 * work, or the activation check).  fin_d depends only on (layout, partition
 * variant, replica, first micro-batch, count): it is computed ONCE per such
 * key -- by the same literal build_dag + critical_path (dag_iteration on the
 * replica alone, D = 1) -- and reused across the assignment variants, which
 * only shift replica boundaries.  The max is exact, so scores equal
 * score_with() bit for bit (tests/test_search_oracle.py checks it).
 */
typedef struct {
  int32_t r, start, cnt, used;
  double fin;
  int bad;
} memo_e;

typedef struct {
  memo_e* tab;
  int cap;
} memo_t;

static memo_e* memo_get(memo_t* m, int r, int start, int cnt) {
  uint32_t h = (uint32_t)r * 2654435761u ^ (uint32_t)start * 40503u ^ (uint32_t)cnt * 97u;
  for (int k = 0;; ++k) {
    memo_e* e = &m->tab[(h + (uint32_t)k) & (uint32_t)(m->cap - 1)];
    if (!e->used) {
      e->used = 1; e->r = r; e->start = start; e->cnt = cnt; e->bad = -1;
      return e;
    }
    if (e->r == r && e->start == start && e->cnt == cnt) return e;
  }
}

typedef struct {
  orc_search* s;
  int64_t begin, end;
  int64_t* next_block; /* shared work counter over (layout, partition) blocks */
  pthread_mutex_t* mu;
  double best;
  int64_t best_i;
  double* scores;
} mjob_t;

static void memo_block(mjob_t* J, void* scr, memo_t* memo, int li, int v) {
  orc_search* s = J->s;
  const rh_search_desc* d = &s->d;
  const layout_t* l = &s->L[li];
  const int T = l->T, D = l->D, P = l->P, M = d->n_micro_batches;
  const int64_t b0 = l->base + (int64_t)v * l->nu;
  const int64_t lo = b0 > J->begin ? b0 : J->begin;
  const int64_t hi = b0 + l->nu < J->end ? b0 + l->nu : J->end;
  if (lo >= hi) return;
  int part[64], cnt[64], li2;
  /* the block's partition (decode of its first candidate; u only moves counts) */
  int part_ok = decode(s, b0, &li2, part, cnt);
  for (int q = 0; q < P; ++q) part_ok &= part[q] >= d->min_layers;
  double ar_v = 0.0;
  if (d->has_comm && D > 1)
    for (int st = 0; st < P; ++st) {
      double nbytes = (double)part[st] * d->layer_bytes;
      double x = 2.0 * nbytes * (double)(D - 1) / ((double)D * l->ring[st]);
      if (x > ar_v) ar_v = x;
    }
  const int use_ar = d->has_comm && D > 1;
  /* surcharge (as in score_with) */
  int changed = 0;
  long long moved = 0;
  if (P == d->cur_pp)
    for (int q = 0; q < P; ++q) {
      if (part[q] != s->cur_part[q]) changed = 1;
      if (part[q] > s->cur_part[q]) moved += part[q] - s->cur_part[q];
    }
  double reshard = 0.0;
  if (!l->same)
    for (int r = 0; r < D; ++r)
      for (int q = 0; q < P; ++q) reshard += (double)part[q] * d->layer_bytes;
  double sur = 0.0;
  if (!l->same || changed) {
    double transfer = ((double)moved * d->layer_bytes + reshard) / s->worst_inter;
    int am = d->amortize_iterations > 1 ? d->amortize_iterations : 1;
    sur = (d->group_rebuild_s + transfer) / (double)am;
  }
  memset(memo->tab, 0, sizeof(memo_e) * (size_t)memo->cap);
  rh_pipe_shape sh = {P, 1, T, d->schedule, M, d->token_budget, d->capacity, 0, 0};
  for (int64_t idx = lo; idx < hi; ++idx) {
    double score = INFINITY;
    if (part_ok && decode(s, idx, &li2, part, cnt)) {
      int start = 0, bad = 0;
      double ms = 0.0;
      for (int r = 0; r < D && !bad; ++r) {
        memo_e* e = memo_get(memo, r, start, cnt[r]);
        if (e->bad < 0) {
          int mbs[2] = {start, start + cnt[r]};
          rh_segments sg = {1, part, mbs, l->gspeed + (size_t)r * P, l->hop + (size_t)r * P,
                            l->hop + (size_t)r * P, NULL, NULL, NULL};
          double f = 0.0;
          uint8_t stt = orc_dag_iteration((struct scratch_s*)scr, &sh, &d->model, &sg, 0, &f,
                                          NULL);
          e->bad = stt != 0;
          e->fin = cnt[r] > 0 ? f : 0.0;
        }
        bad |= e->bad;
        double c = use_ar ? e->fin + ar_v : e->fin;
        if (c > ms) ms = c;
        start += cnt[r];
      }
      if (!bad) score = ms + sur;
    }
    if (J->scores) J->scores[idx - J->begin] = score;
    /* lexicographic (score, index) over feasible candidates */
    if (score < INFINITY &&
        (J->best_i < 0 || score < J->best || (score == J->best && idx < J->best_i))) {
      J->best = score;
      J->best_i = idx;
    }
  }
}

static void* mworker(void* arg) {
  mjob_t* J = arg;
  orc_search* s = J->s;
  void* scr = new_scratch(s);
  memcpy(orc_scratch_quad(scr), s->quad, sizeof(int64_t) * s->d.n_micro_batches);
  memo_t memo;
  memo.cap = 1;
  while (memo.cap < 64 * (s->maxD > 0 ? s->maxD : 1)) memo.cap <<= 1;
  memo.tab = malloc(sizeof(memo_e) * (size_t)memo.cap);
  J->best = INFINITY;
  J->best_i = -1;
  /* blocks enumerated in index order: (layout, partition variant) */
  int64_t nblocks = 0;
  for (int li = 0; li < s->nl; ++li) nblocks += s->L[li].nv;
  for (;;) {
    pthread_mutex_lock(J->mu);
    int64_t k = (*J->next_block)++;
    pthread_mutex_unlock(J->mu);
    if (k >= nblocks) break;
    int li = 0;
    int64_t kk = k;
    while (kk >= s->L[li].nv) kk -= s->L[li++].nv;
    memo_block(J, scr, &memo, li, (int)kk);
  }
  free(memo.tab);
  orc_scratch_delete(scr);
  return NULL;
}

int orc_search_eval_memo(orc_search* s, int64_t begin, int64_t end, int n_threads,
                         double* best_score, int64_t* best_index, double* scores) {
  if (n_threads <= 0) n_threads = (int)sysconf(_SC_NPROCESSORS_ONLN);
  if (n_threads < 1) n_threads = 1;
  pthread_t* th = malloc(sizeof(pthread_t) * n_threads);
  mjob_t* jobs = malloc(sizeof(mjob_t) * n_threads);
  int64_t next = 0;
  pthread_mutex_t mu = PTHREAD_MUTEX_INITIALIZER;
  for (int k = 0; k < n_threads; ++k) {
    jobs[k] = (mjob_t){s, begin, end, &next, &mu, INFINITY, -1, scores};
    if (n_threads == 1) mworker(&jobs[0]);
    else pthread_create(&th[k], NULL, mworker, &jobs[k]);
  }
  if (n_threads > 1) for (int k = 0; k < n_threads; ++k) pthread_join(th[k], NULL);
  double b = INFINITY;
  int64_t bi = -1;
  for (int k = 0; k < n_threads; ++k) {
    if (jobs[k].best_i < 0) continue;
    if (bi < 0 || jobs[k].best < b || (jobs[k].best == b && jobs[k].best_i < bi)) {
      b = jobs[k].best;
      bi = jobs[k].best_i;
    }
  }
  *best_score = b;
  *best_index = bi;
  free(th); free(jobs);
  return 0;
}
