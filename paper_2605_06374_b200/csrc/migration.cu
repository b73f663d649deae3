// Progress-aware workload migration (rh_plan_migration): the host-side
// co-simulation of plan_migration (scheduler.py:272-513) with
// migration_decision (scheduler.py:210-251), restated in C++.
//
// Semantics kept exactly: one global event heap ordered by (time, sequence
// number) with "finish"/"ready" events, per-(replica, stage, kind) ready heaps
// ordered by (ready time, micro-batch), the back > F > W pick order of
// try_start, activation capacity on F starts, scheduling slots that group
// every completion sharing a timestamp, one sweep of migration decisions per
// slot in stage order, owner credit at migration time, and the trailing
// try_start over sorted (replica, stage) keys.
//
// Complexity: the reference rescans all micro-batches for unstarted_f and
// next_pending on every decision (O(M), 95% of a 256-GPU re-plan, SURVEY
// §0.1); here both are O(1) amortised (counters + a monotone cursor).
// Arithmetic: chunk costs are predict_chunk_time (workload.py:88-98) in fp64
// with the reference's operation order; the host compiler runs with
// -ffp-contract=off.
#include <algorithm>
#include <cstdio>
#include <queue>
#include <string>
#include <vector>

#include "common.cuh"

namespace {

enum { KF = 0, KB = 1, KW = 2 };

struct Ev {
  double t;
  long long seq;
  int tag;  // 0 = ready, 1 = finish
  int a, b, c, d;
  bool operator>(const Ev& o) const { return t > o.t || (t == o.t && seq > o.seq); }
};

struct Ready {
  double t;
  int j;
  bool operator>(const Ready& o) const { return t > o.t || (t == o.t && j > o.j); }
};

template <class T>
using MinHeap = std::priority_queue<T, std::vector<T>, std::greater<T>>;

struct Sim {
  const rh_migration_desc& d;
  int P, D, M, back;
  bool merged;
  std::vector<int> owner, exec;  // exec[j*P+s]
  std::vector<char> dead, migrated_in, started;  // started[(kind*M + j)*P + s]
  std::vector<double> done_f;                    // finish time of F(j,s), <0 if not done
  std::vector<double> grad_arrival, f_ready;     // <0: unset
  std::vector<char> running;
  std::vector<int> in_flight, unstarted;         // per (d,s)
  std::vector<int> cursor;                       // next_pending cursor per (d,s)
  std::vector<int> own_lo, own_hi;               // owner ranges
  std::vector<std::vector<MinHeap<Ready>>> queues;  // [(d,s)][kind]
  std::vector<std::vector<int>> progress;        // [d][s]
  MinHeap<Ev> events;
  long long seq = 0;
  std::vector<int32_t> migrations, log;
  std::vector<double> base;

  explicit Sim(const rh_migration_desc& desc) : d(desc) {}

  double hop(const double* tab, int s, int a, int b) const {
    return tab ? tab[((size_t)s * D + a) * D + b] : 0.0;
  }
  double cost(int kind, int j, int r, int s) const {
    const rh_cost_model& m = d.model;
    double ratio = kind == KF ? m.ratio_f : (merged ? m.ratio_b + m.ratio_w
                                                    : (kind == KB ? m.ratio_b : m.ratio_w));
    double rl = ratio * (double)d.layers[s];
    double num = rl * base[j];
    return num / d.speed[r * P + s];
  }
  void push(double t, int tag, int a, int b, int c, int e) {
    events.push(Ev{t, seq++, tag, a, b, c, e});
  }
  void enqueue(int kind, int j, int s, double t) {
    const int r = exec[j * P + s];
    queues[r * P + s][kind].push(Ready{t, j});
    if (kind == KF) f_ready[j * P + s] = t;
  }
  bool is_started(int kind, int j, int s) const { return started[((size_t)kind * M + j) * P + s]; }
  int next_pending(int r, int s) {
    int& c = cursor[r * P + s];
    while (c < own_hi[r]) {
      const int j = c;
      if (exec[j * P + s] == r && !migrated_in[j * P + s] && !is_started(KF, j, s)) return j;
      ++c;  // j left the candidate set for good
    }
    return -1;
  }
  bool memory_feasible(int s, int r) const {
    return in_flight[r * P + s] + unstarted[r * P + s] < d.capacity;
  }
  void try_start(int r, int s, double now) {
    const int key = r * P + s;
    if (running[key] || dead[key]) return;
    int pick_kind = -1, pick_j = -1;
    const int order[3] = {back, KF, KW};
    for (int oi = 0; oi < 3 && pick_kind < 0; ++oi) {
      const int kind = order[oi];
      if (merged && kind == KW) continue;
      auto& heap = queues[key][kind];
      while (!heap.empty()) {
        const Ready top = heap.top();
        if (top.t > now) break;
        if (exec[top.j * P + s] != r || is_started(kind, top.j, s)) {
          heap.pop();
          continue;
        }
        if (kind == KF && in_flight[key] >= d.capacity) break;
        pick_kind = kind;
        pick_j = top.j;
        heap.pop();
        break;
      }
    }
    if (pick_kind < 0) return;
    started[((size_t)pick_kind * M + pick_j) * P + s] = 1;
    if (pick_kind == KF) unstarted[key]--;
    log.insert(log.end(), {r, s, pick_kind == back ? 1 : pick_kind, pick_j});
    running[key] = 1;
    if (pick_kind == KF) in_flight[key]++;
    push(now + cost(pick_kind, pick_j, r, s), 1, r, s, pick_kind, pick_j);
  }
  // migration_decision (scheduler.py:210-251)
  bool decide(int s, int& j, int& dmin, int& dmax) {
    dmin = -1;
    for (int r = 0; r < D; ++r) {
      if (dmin < 0) {
        dmin = r;
        continue;
      }
      const int cr = progress[r][s], cm = progress[dmin][s];
      const int kr = dead[r * P + s] ? 0 : 1, km = dead[dmin * P + s] ? 0 : 1;
      if (cr < cm || (cr == cm && kr < km)) dmin = r;  // ties on d keep the lower index
    }
    int best = -1;
    bool any = false;
    for (int r = 0; r < D; ++r)
      if (!dead[r * P + s]) {
        best = any ? std::max(best, progress[r][s]) : progress[r][s];
        any = true;
      }
    if (!any) return false;
    dmax = -1;
    for (int r = 0; r < D; ++r) {
      if (dead[r * P + s] || progress[r][s] != best) continue;
      const int lr = in_flight[r * P + s] + unstarted[r * P + s];
      if (dmax < 0 || lr < in_flight[dmax * P + s] + unstarted[dmax * P + s]) dmax = r;
    }
    if (dmax == dmin) return false;
    const int gap = progress[dmax][s] - progress[dmin][s];
    if (!dead[dmin * P + s] && gap <= d.delta) return false;
    j = next_pending(dmin, s);
    if (j < 0) return false;
    if (!memory_feasible(s, dmax)) return false;
    return true;
  }
  void sweep(double now) {
    if (!d.migrate) return;
    for (int s = 0; s < P; ++s) {
      int j, dmin, dmax;
      if (!decide(s, j, dmin, dmax)) continue;
      exec[j * P + s] = dmax;
      migrated_in[j * P + s] = 1;
      unstarted[dmin * P + s]--;
      unstarted[dmax * P + s]++;
      progress[dmin][s] += 1;  // owner credit: backlog shrank
      migrations.insert(migrations.end(), {j, s, dmin, dmax});
      if (f_ready[j * P + s] >= 0.0) {
        const double t = std::max(now, f_ready[j * P + s]) + hop(d.hop_same, s, dmin, dmax);
        push(t, 0, KF, j, s, 0);
      }
      try_start(dmax, s, now);
    }
  }
};

}  // namespace

extern "C" int rh_plan_migration(const rh_migration_desc* desc, int32_t* migrations,
                                 int32_t* n_migrations, int32_t* start_log, int32_t* n_started,
                                 double* makespan) {
  if (!desc || desc->pp < 1 || desc->dp < 1 || desc->n_mb < 1 || !desc->mb_off ||
      !desc->doc_len ||
      !desc->layers || !desc->speed || !makespan || !n_migrations || !n_started) {
    rh::set_error("rh_plan_migration: invalid arguments");
    return RH_E_INVALID;
  }
  Sim S(*desc);
  const int P = desc->pp, D = desc->dp, M = desc->n_mb;
  S.P = P;
  S.D = D;
  S.M = M;
  S.merged = desc->schedule == RH_SCHED_1F1B;
  S.back = KB;
  // ownership (split_micro_batches, cluster.py:309-328)
  std::vector<int> counts(D);
  if (desc->dp_counts) {
    long long tot = 0;
    for (int r = 0; r < D; ++r) {
      counts[r] = desc->dp_counts[r];
      tot += counts[r];
      if (counts[r] < 0) tot = -1 << 30;
    }
    if (tot != M) {
      rh::set_error("bad ownership counts for %d micro-batches", M);
      return RH_E_INVALID;
    }
  } else {
    for (int r = 0; r < D; ++r) counts[r] = M / D + (r < M % D ? 1 : 0);
  }
  S.owner.resize(M);
  S.own_lo.resize(D);
  S.own_hi.resize(D);
  for (int r = 0, c = 0; r < D; ++r) {
    S.own_lo[r] = c;
    for (int q = 0; q < counts[r]; ++q) S.owner[c++] = r;
    S.own_hi[r] = c;
  }
  S.base.resize(M);
  for (int j = 0; j < M; ++j) {
    const double lin = desc->model.alpha * (double)desc->token_budget;
    long long q = 0;  // quad_load, workload.py:83-85
    for (int k = desc->mb_off[j]; k < desc->mb_off[j + 1]; ++k)
      q += (long long)desc->doc_len[k] * desc->doc_len[k];
    const double qd = desc->model.beta * (double)q;
    S.base[j] = lin + qd;
  }
  S.dead.assign(D * P, 0);
  for (int k = 0; k < D * P; ++k) S.dead[k] = desc->speed[k] <= 0.0;
  S.exec.resize((size_t)M * P);
  S.migrated_in.assign((size_t)M * P, 0);
  for (int j = 0; j < M; ++j)
    for (int s = 0; s < P; ++s) {
      int e = S.owner[j];
      if (desc->preset && desc->preset[j * P + s] >= 0) e = desc->preset[j * P + s];
      if (e < 0 || e >= D) {
        rh::set_error("preset executor %d out of range", e);
        return RH_E_INVALID;
      }
      S.exec[j * P + s] = e;
      S.migrated_in[j * P + s] = e != S.owner[j];
    }
  // stranded check (scheduler.py:315-323), in sorted (mb, stage) order
  for (int j = 0; j < M; ++j)
    for (int s = 0; s < P; ++s) {
      if (!S.dead[S.exec[j * P + s] * P + s]) continue;
      bool rescuable = false;
      if (desc->migrate)
        for (int r = 0; r < D; ++r) rescuable |= !S.dead[r * P + s];
      if (!rescuable) {
        rh::set_error("stranded workload: chunk (mb %d, stage %d) assigned to a stopped stage "
                      "with no executable replica", j, s);
        return RH_E_STRANDED;
      }
    }
  const int c = S.merged ? 2 : 3;
  S.started.assign((size_t)3 * M * P, 0);
  S.done_f.assign((size_t)M * P, -1.0);
  S.grad_arrival.assign((size_t)M * P, -1.0);
  S.f_ready.assign((size_t)M * P, -1.0);
  S.running.assign(D * P, 0);
  S.in_flight.assign(D * P, 0);
  S.unstarted.assign(D * P, 0);
  for (int j = 0; j < M; ++j)
    for (int s = 0; s < P; ++s) S.unstarted[S.exec[j * P + s] * P + s]++;
  S.cursor.resize(D * P);
  for (int r = 0; r < D; ++r)
    for (int s = 0; s < P; ++s) S.cursor[r * P + s] = S.own_lo[r];
  S.queues.assign(D * P, std::vector<MinHeap<Ready>>(3));
  S.progress.assign(D, std::vector<int>(P, 0));
  long long remaining = (long long)M * P * c;

  for (int j = 0; j < M; ++j) S.enqueue(KF, j, 0, 0.0);
  for (int r = 0; r < D; ++r)
    for (int s = 0; s < P; ++s) S.try_start(r, s, 0.0);
  double end = 0.0;
  while (!S.events.empty()) {
    const double t = S.events.top().t;
    end = std::max(end, t);
    bool finished = false;
    while (!S.events.empty() && S.events.top().t == t) {
      const Ev e = S.events.top();
      S.events.pop();
      if (e.tag == 0) {  // ready: (kind, j, s)
        S.enqueue(e.a, e.b, e.c, t);
        continue;
      }
      finished = true;
      const int r = e.a, s = e.b, kind = e.c, j = e.d;
      S.running[r * P + s] = 0;
      remaining--;
      if (kind == KF) {
        S.done_f[j * P + s] = t;
        if (!S.migrated_in[j * P + s]) S.progress[r][s] += 1;
        if (s + 1 < P) {
          const int nxt = S.exec[j * P + s + 1];
          S.push(t + S.hop(desc->hop_next, s, r, nxt), 0, KF, j, s + 1, 0);
        }
        if (s == P - 1) {
          S.push(t, 0, KB, j, s, 0);
        } else if (S.grad_arrival[j * P + s] >= 0.0) {
          S.push(std::max(t, S.grad_arrival[j * P + s]), 0, KB, j, s, 0);
        }
      } else if (kind == KB) {
        S.in_flight[r * P + s]--;
        if (s > 0) {
          const int prev = S.exec[j * P + s - 1];
          const double arrival = t + S.hop(desc->hop_prev, s, r, prev);
          S.grad_arrival[j * P + s - 1] = arrival;
          if (S.done_f[j * P + s - 1] >= 0.0)
            S.push(std::max(arrival, S.done_f[j * P + s - 1]), 0, KB, j, s - 1, 0);
        }
        if (!S.merged) S.push(t, 0, KW, j, s, 0);
      }
    }
    if (finished) S.sweep(t);
    for (int r = 0; r < D; ++r)
      for (int s = 0; s < P; ++s) S.try_start(r, s, t);
  }
  if (remaining > 0) {
    int n = 0;
    for (int j = 0; j < M; ++j)
      for (int s = 0; s < P; ++s)
        if (S.done_f[j * P + s] < 0.0 && S.dead[S.exec[j * P + s] * P + s]) ++n;
    rh::set_error("stranded workload: %d chunks unexecutable", n);
    return RH_E_STRANDED;
  }
  *makespan = end;
  *n_migrations = (int32_t)(S.migrations.size() / 4);
  *n_started = (int32_t)(S.log.size() / 4);
  if (migrations) std::copy(S.migrations.begin(), S.migrations.end(), migrations);
  if (start_log) std::copy(S.log.begin(), S.log.end(), start_log);
  return RH_OK;
}
