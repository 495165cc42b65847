// Native, bit-exact restatement of the reference's chunk generation (PGC,
// weighted label propagation): dynpart.partition.propagate's label
// computation (partition.py:200-270) with _propagation_edges (:138-152),
// _greedy_coloring (:155-168) and _class_argmax (:171-197).
//
// The Python version spends O(n) interpreter work per colouring and per
// adoption (377 s at 1M instances). Here:
//   * messages are held once as an in-CSR by destination (src, weight);
//   * colouring: vertex v (ascending) takes the smallest colour not used by an
//     already-coloured in-neighbour -- the same greedy order as the reference;
//   * per colour class, phase 1 decides every member against the labels and
//     chunk counts as they stand at the start of the class (the reference's
//     `admissible = counts[lab] < size_cap` snapshot and its per-(dst, label)
//     integer sums; max weight, ties to the smallest label; switch iff the best
//     weight strictly beats the weight of the current label among ADMISSIBLE
//     messages), phase 2 applies the switches in ascending vertex order with
//     live cap accounting, exactly like the reference's adoption loop.
// Integer weights => results are exact; the labels equal the reference's
// (tests/test_propagate_native.py, golden labels from the unmodified reference).
#include <algorithm>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/dgc_b200.h"

namespace dgc {
void set_error(const std::string& msg);
}

namespace {
using i64 = int64_t;
}

extern "C" int dgc_propagate_labels(int64_t n, int64_t n_spatial, const int64_t* spatial_edges,
                                    int64_t n_temporal, const int64_t* temporal_links,
                                    int64_t spatial_weight, const int64_t* temporal_weights,
                                    int64_t size_cap, int32_t max_rounds, int64_t* labels,
                                    int32_t* rounds_run, int32_t* n_colors) {
  if (size_cap < 1) {
    dgc::set_error("propagate: size_cap must be >= 1");
    return DGC_ERR_ARG;
  }
  if (max_rounds < 1) {
    dgc::set_error("propagate: max_rounds must be >= 1");
    return DGC_ERR_ARG;
  }
  if (n < 0 || n_spatial < 0 || n_temporal < 0 || (n_temporal > 0 && !temporal_weights)) {
    dgc::set_error("propagate: bad sizes");
    return DGC_ERR_ARG;
  }
  for (i64 i = 0; i < n; ++i) labels[i] = i;  // init_labels (partition.py:104-108)
  if (rounds_run) *rounds_run = 0;
  if (n_colors) *n_colors = 0;
  if (n == 0 || n_spatial + n_temporal == 0) return DGC_OK;
  // messages (partition.py:138-152): spatial both ways, temporal both ways
  std::vector<i64> indeg(n + 1, 0);
  auto check = [&](i64 v) { return v >= 0 && v < n; };
  for (i64 e = 0; e < n_spatial; ++e) {
    const i64 a = spatial_edges[2 * e], b = spatial_edges[2 * e + 1];
    if (!check(a) || !check(b)) {
      dgc::set_error("propagate: spatial edge endpoint out of range");
      return DGC_ERR_ARG;
    }
    ++indeg[a];
    ++indeg[b];
  }
  for (i64 e = 0; e < n_temporal; ++e) {
    const i64 a = temporal_links[2 * e], b = temporal_links[2 * e + 1];
    if (!check(a) || !check(b)) {
      dgc::set_error("propagate: temporal link endpoint out of range");
      return DGC_ERR_ARG;
    }
    ++indeg[a];
    ++indeg[b];
  }
  std::vector<i64> ptr(n + 1, 0);
  for (i64 v = 0; v < n; ++v) ptr[v + 1] = ptr[v] + indeg[v];
  const i64 m = ptr[n];
  std::vector<i64> in_src(m), in_w(m);
  {
    std::vector<i64> fill(ptr.begin(), ptr.end() - 1);
    auto add = [&](i64 s, i64 d, i64 w) {
      in_src[fill[d]] = s;
      in_w[fill[d]] = w;
      ++fill[d];
    };
    for (i64 e = 0; e < n_spatial; ++e) {
      add(spatial_edges[2 * e], spatial_edges[2 * e + 1], spatial_weight);
      add(spatial_edges[2 * e + 1], spatial_edges[2 * e], spatial_weight);
    }
    for (i64 e = 0; e < n_temporal; ++e) {
      add(temporal_links[2 * e], temporal_links[2 * e + 1], temporal_weights[e]);
      add(temporal_links[2 * e + 1], temporal_links[2 * e], temporal_weights[e]);
    }
  }
  // greedy colouring (partition.py:155-168)
  std::vector<i64> color(n, -1);
  std::vector<i64> stamp;  // stamp[c] == v + 1  <=>  colour c used by v's in-neighbours
  i64 max_color = -1;
  for (i64 v = 0; v < n; ++v) {
    for (i64 k = ptr[v]; k < ptr[v + 1]; ++k) {
      const i64 c = color[in_src[k]];
      if (c < 0) continue;
      if ((i64)stamp.size() <= c) stamp.resize(c + 1, 0);
      stamp[c] = v + 1;
    }
    i64 c = 0;
    while (c < (i64)stamp.size() && stamp[c] == v + 1) ++c;
    color[v] = c;
    if (c > max_color) max_color = c;
  }
  const i64 n_cls = max_color + 1;
  if (n_colors) *n_colors = (int32_t)n_cls;
  std::vector<i64> cls_ptr(n_cls + 1, 0), cls_v(n);
  for (i64 v = 0; v < n; ++v) ++cls_ptr[color[v] + 1];
  for (i64 c = 0; c < n_cls; ++c) cls_ptr[c + 1] += cls_ptr[c];
  {
    std::vector<i64> fill(cls_ptr.begin(), cls_ptr.end() - 1);
    for (i64 v = 0; v < n; ++v) cls_v[fill[color[v]]++] = v;  // ascending within a class
  }
  std::vector<i64> counts(n, 1);  // bincount of the unique initial labels
  // per-vertex label aggregation scratch (labels of one vertex's in-messages)
  std::vector<std::pair<i64, i64>> agg;
  std::vector<std::pair<i64, i64>> switches;
  for (int32_t round = 0; round < max_rounds; ++round) {
    i64 changed = 0;
    for (i64 c = 0; c < n_cls; ++c) {
      // phase 1: decisions against the class-start labels and counts
      switches.clear();
      for (i64 q = cls_ptr[c]; q < cls_ptr[c + 1]; ++q) {
        const i64 v = cls_v[q];
        agg.clear();
        for (i64 k = ptr[v]; k < ptr[v + 1]; ++k) {
          const i64 lab = labels[in_src[k]];
          if (counts[lab] < size_cap) agg.emplace_back(lab, in_w[k]);
        }
        if (agg.empty()) continue;  // no admissible message: v is not a candidate
        std::sort(agg.begin(), agg.end(),
                  [](const std::pair<i64, i64>& x, const std::pair<i64, i64>& y) {
                    return x.first < y.first;
                  });
        const i64 cur = labels[v];
        i64 best_lab = -1, best_w = 0, cur_w = 0;
        for (size_t i = 0; i < agg.size();) {
          const i64 lab = agg[i].first;
          i64 sum = 0;
          for (; i < agg.size() && agg[i].first == lab; ++i) sum += agg[i].second;
          if (best_lab < 0 || sum > best_w) {  // labels ascending: ties keep the smallest
            best_lab = lab;
            best_w = sum;
          }
          if (lab == cur) cur_w = sum;
        }
        if (best_w > cur_w && best_lab != cur) switches.emplace_back(v, best_lab);
      }
      // phase 2: adoption in ascending vertex order, live cap accounting
      for (const auto& sw : switches) {
        const i64 v = sw.first, c_new = sw.second;
        if (counts[c_new] >= size_cap) continue;
        --counts[labels[v]];
        ++counts[c_new];
        labels[v] = c_new;
        ++changed;
      }
    }
    if (rounds_run) *rounds_run = round + 1;
    if (changed == 0) break;
  }
  return DGC_OK;
}
