// Workload ingest (host-side, native): first-fit-decreasing packing of
// document lengths into token-budget micro-batches — pack_sequences,
// workload.py:52-80 — in O(n log n) with a max-segment-tree over bin
// residuals ("leftmost bin with room >= l" is a tree descent) instead of the
// reference's O(n * bins) scan.  Output is identical: bins in creation
// order, documents in insertion (descending) order, the residual appended as
// a padding document when non-zero.
#include <algorithm>
#include <functional>
#include <vector>

#include "common.cuh"

static int pack_sequences(int64_t n_docs, const int32_t* lengths, int32_t budget,
                          int64_t max_bins, int32_t* mb_off, int32_t* doc_len,
                          int64_t* n_bins_out, int64_t* n_entries_out, int64_t* quad_out) {
  if (n_docs < 0 || budget <= 0 || !n_bins_out || !n_entries_out ||
      (n_docs && !lengths)) {
    rh::set_error("rh_pack_sequences: invalid arguments");
    return RH_E_INVALID;
  }
  std::vector<int32_t> v(lengths, lengths + n_docs);
  for (int32_t l : v) {
    if (l <= 0) {
      rh::set_error("document length must be positive, got %d", l);
      return RH_E_INVALID;
    }
    if (l > budget) {
      rh::set_error("document of %d tokens exceeds budget %d", l, budget);
      return RH_E_INVALID;
    }
  }
  // descending order: counting sort over [1, budget] when the histogram is
  // small next to the input (10^5 documents: ~0.3 ms instead of ~8 ms)
  if ((int64_t)budget <= 8 * std::max<int64_t>(n_docs, 1) + (1 << 16)) {
    std::vector<int32_t> hist((size_t)budget + 1, 0);
    for (int32_t l : v) ++hist[l];
    int64_t k = 0;
    for (int32_t l = budget; l >= 1; --l)
      for (int32_t c = hist[l]; c > 0; --c) v[k++] = l;
  } else {
    std::sort(v.begin(), v.end(), std::greater<int32_t>());
  }
  // The segment tree covers `cap` bin slots (unopened slots hold `budget`),
  // so a descent is log2(cap) levels.  Start from ~11/9 of the volume bound
  // (FFD <= 11/9 OPT + 6/9, OPT >= ceil(total / budget)); if the documents
  // need more bins than that (OPT above the volume bound), double and redo.
  //
  // Equal lengths are placed in bulk: the leftmost bin with room >= l takes
  // floor(room / l) of them (one by one, first fit would put each of them
  // there: no earlier bin gains room), so a run of equal documents costs one
  // descent per bin it touches rather than one per document -- the same
  // bins, in the same insertion order.
  int64_t total = 0;
  for (int32_t l : v) total += l;
  const int64_t vol = (total + budget - 1) / budget;
  int64_t cap = 1;
  while (cap < std::min<int64_t>(std::max<int64_t>(n_docs, 1), (11 * vol) / 9 + 2)) cap <<= 1;
  std::vector<int32_t> tree;
  std::vector<int64_t> bin_of(n_docs);
  std::vector<int64_t> bin_count;
  int64_t opened = 0;
  for (;;) {
    tree.assign(2 * cap, budget);
    bin_count.assign(cap + 1, 0);
    opened = 0;
    bool overflow = false;
    for (int64_t i = 0; i < n_docs && !overflow;) {
      const int32_t l = v[i];
      int64_t run = i + 1;
      while (run < n_docs && v[run] == l) ++run;
      while (i < run) {
        if (tree[1] < l) {  // no slot left with room: more bins than slots
          overflow = true;
          break;
        }
        // leftmost slot with residual >= l: first-fit over opened bins, else
        // the next fresh slot (index == opened, residual == budget >= l)
        int64_t node = 1;
        while (node < cap) node = 2 * node + (tree[2 * node] < l);  // branch-free descent
        const int64_t b = node - cap;
        if (b == opened) ++opened;
        const int64_t k = std::min<int64_t>(run - i, tree[node] / l);
        for (int64_t q = 0; q < k; ++q) bin_of[i + q] = b;
        i += k;
        bin_count[b] += k;
        tree[node] -= (int32_t)(k * l);
        // propagate the new maximum upward while it changes
        for (node >>= 1; node; node >>= 1) {
          const int32_t m = std::max(tree[2 * node], tree[2 * node + 1]);
          if (tree[node] == m) break;
          tree[node] = m;
        }
      }
    }
    if (!overflow) break;
    cap <<= 1;
  }
  const int64_t keep = max_bins >= 0 ? std::min(opened, max_bins) : opened;
  // CSR: docs of bin b in insertion order, then padding if residual > 0
  std::vector<int64_t> start(keep + 1, 0);
  for (int64_t b = 0; b < keep; ++b)
    start[b + 1] = start[b] + bin_count[b] + (tree[cap + b] > 0 ? 1 : 0);
  if (start[keep] >= INT32_MAX) {
    rh::set_error("rh_pack_sequences: too many entries for int32 offsets");
    return RH_E_SHAPE;
  }
  *n_bins_out = keep;
  *n_entries_out = start[keep];
  if (!mb_off || !doc_len) return RH_OK;  // size query
  std::vector<int64_t> fill(start.begin(), start.end() - 1);
  for (int64_t i = 0; i < n_docs; ++i)
    if (bin_of[i] < keep) doc_len[fill[bin_of[i]]++] = v[i];
  for (int64_t b = 0; b < keep; ++b) {
    if (tree[cap + b] > 0) doc_len[fill[b]++] = tree[cap + b];
    mb_off[b] = (int32_t)start[b];
  }
  mb_off[keep] = (int32_t)start[keep];
  if (quad_out) {  // quad_load of every kept bin, padding included (workload.py:83-85)
    for (int64_t b = 0; b < keep; ++b) {
      int64_t q = 0;
      for (int64_t e = start[b]; e < start[b + 1]; ++e) q += (int64_t)doc_len[e] * doc_len[e];
      quad_out[b] = q;
    }
  }
  return RH_OK;
}

extern "C" int rh_pack_sequences(int64_t n_docs, const int32_t* lengths, int32_t budget,
                                 int64_t max_bins, int32_t* mb_off, int32_t* doc_len,
                                 int64_t* n_bins_out, int64_t* n_entries_out) {
  return pack_sequences(n_docs, lengths, budget, max_bins, mb_off, doc_len, n_bins_out,
                        n_entries_out, nullptr);
}

extern "C" int rh_pack_sequences_quad(int64_t n_docs, const int32_t* lengths, int32_t budget,
                                      int64_t max_bins, int32_t* mb_off, int32_t* doc_len,
                                      int64_t* quad, int64_t* n_bins_out,
                                      int64_t* n_entries_out) {
  return pack_sequences(n_docs, lengths, budget, max_bins, mb_off, doc_len, n_bins_out,
                        n_entries_out, quad);
}
