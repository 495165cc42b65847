// Native, bit-exact restatement of the reference's spatial chunk-fusion
// planner (fusion.py:108-220 plan_spatial_fusion / plan_fusion) and of the
// chunk statistics it consumes (partition.py:273-359 _build_chunk_graph:
// per-chunk degree sums, halos over spatial edges + consecutive temporal
// links, inter-chunk message bytes).
//
// The Python planner copies member/halo sets on every merge (quadratic; > 1
// CPU-hour and > 46 GB at 200k instances). Here every group
// keeps only |members|, its EXTERNAL halo set and an owner map, merged
// small-into-large, so the memory estimate 256*|members U halo| + 64*edges
// (fusion.py:119-121) costs O(smaller side) per candidate merge. The heap
// pops the largest saving first, ties to the smallest (a, b) -- exactly
// Python's heapq order on (-w, (a, b)) -- with the same lazy invalidation,
// dead-pair and re-keying rules, so the output groups, memory_bytes and
// saved_bytes equal the reference's (tests/test_fusion_native.py).
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cstdint>
#include <queue>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "../../include/dgc_b200.h"

namespace dgc {
void set_error(const std::string& msg);
}

namespace {

using i64 = int64_t;

struct Group {
  std::vector<i64> chunk_ids;          // sorted at the end
  std::vector<i64> member_list;        // instances (for owner updates)
  std::unordered_set<i64> ext_halo;    // halo \ members
  i64 edges = 0;
  i64 saved = 0;
  i64 rep = 0;
};

struct HeapItem {
  i64 w, a, b;
  bool operator<(const HeapItem& o) const {  // priority_queue: top = largest
    if (w != o.w) return w < o.w;
    if (a != o.a) return a > o.a;
    return b > o.b;
  }
};

}  // namespace

extern "C" int dgc_plan_spatial_fusion(
    int64_t n_instances, const int32_t* spatial_edges, int64_t n_spatial_edges,
    const int32_t* temporal_links, int64_t n_temporal_links, const int32_t* chunk_of,
    int64_t n_chunks, const int32_t* device_chunks, int64_t n_device_chunks,
    int64_t spatial_msg_bytes, int64_t temporal_msg_bytes, int64_t memory_budget,
    int64_t bytes_per_vertex, int64_t bytes_per_edge, int32_t* out_group_of_chunk,
    int64_t* out_group_memory, int64_t* out_group_saved, int64_t* n_groups_out) {
  // chunk stats restricted to this device's chunks
  std::vector<int> local(n_chunks, -1);
  for (i64 i = 0; i < n_device_chunks; ++i) local[device_chunks[i]] = (int)i;
  const i64 C = n_device_chunks;
  std::vector<Group> g(C);
  for (i64 i = 0; i < C; ++i) {
    g[i].chunk_ids = {device_chunks[i]};
    g[i].rep = device_chunks[i];
  }
  for (i64 v = 0; v < n_instances; ++v) {
    const int c = local[chunk_of[v]];
    if (c >= 0) g[c].member_list.push_back(v);
  }
  // degree sums, halos, inter-chunk bytes (partition.py:307-346)
  std::unordered_map<i64, i64> inter;  // key lo*n_chunks+hi
  auto add_pair = [&](i64 u, i64 v, i64 bytes, bool spatial) {
    const i64 cu = chunk_of[u], cv = chunk_of[v];
    if (spatial) {
      if (local[cu] >= 0) g[local[cu]].edges++;
      if (local[cv] >= 0) g[local[cv]].edges++;
    }
    if (cu == cv) return;
    if (local[cu] >= 0) g[local[cu]].ext_halo.insert(v);
    if (local[cv] >= 0) g[local[cv]].ext_halo.insert(u);
    const i64 lo = std::min(cu, cv), hi = std::max(cu, cv);
    inter[lo * n_chunks + hi] += bytes;
  };
  for (i64 e = 0; e < n_spatial_edges; ++e)
    add_pair(spatial_edges[2 * e], spatial_edges[2 * e + 1], 2 * spatial_msg_bytes, true);
  for (i64 l = 0; l < n_temporal_links; ++l)
    add_pair(temporal_links[2 * l], temporal_links[2 * l + 1], temporal_msg_bytes, false);
  auto memory_of = [&](i64 n_members, i64 n_ext, i64 edges) {
    return bytes_per_vertex * (n_members + n_ext) + bytes_per_edge * edges;
  };
  for (i64 i = 0; i < C; ++i) {
    const i64 mem = memory_of((i64)g[i].member_list.size(), (i64)g[i].ext_halo.size(), g[i].edges);
    if (mem > memory_budget) {
      dgc::set_error("BudgetExceededError: chunk " + std::to_string(g[i].rep) + " needs " +
                     std::to_string(mem) + " bytes, budget is " + std::to_string(memory_budget));
      return DGC_ERR_PLAN;
    }
  }
  // Fast exact path. If even the union of ALL this device's chunks fits the
  // budget, no merge can ever be rejected (a group's estimate only grows with
  // its member set), so the greedy loop merges every pair with positive saving
  // until none is left: the result is the connected components of the
  // positive-inter_cost chunk graph, saved = the inter_cost inside each
  // component, independent of merge order. Equal to the heap path on every
  // non-binding golden case (tests/test_fusion_native.py).
  {
    std::unordered_set<i64> all_members;
    i64 all_edges = 0, n_mem = 0;
    for (i64 i = 0; i < C; ++i) {
      n_mem += (i64)g[i].member_list.size();
      all_edges += g[i].edges;
      for (i64 v : g[i].member_list) all_members.insert(v);
    }
    std::unordered_set<i64> all_ext;
    for (i64 i = 0; i < C; ++i)
      for (i64 x : g[i].ext_halo)
        if (!all_members.count(x)) all_ext.insert(x);
    if (memory_of(n_mem, (i64)all_ext.size(), all_edges) <= memory_budget &&
        !std::getenv("DGC_FUSION_FORCE_HEAP")) {
      std::vector<i64> parent(C);
      for (i64 i = 0; i < C; ++i) parent[i] = i;
      auto find = [&](i64 x) {
        while (parent[x] != x) x = parent[x] = parent[parent[x]];
        return x;
      };
      std::vector<std::pair<i64, i64>> pos_pairs;
      for (auto& kv : inter) {
        if (kv.second <= 0) continue;
        const i64 a = kv.first / n_chunks, b = kv.first % n_chunks;
        if (local[a] < 0 || local[b] < 0) continue;
        pos_pairs.emplace_back(kv.first, kv.second);
        const i64 ra = find(local[a]), rb = find(local[b]);
        if (ra != rb) parent[std::max(ra, rb)] = std::min(ra, rb);
      }
      std::unordered_map<i64, std::vector<i64>> comp;  // root -> device chunk indices
      for (i64 i = 0; i < C; ++i) comp[find(i)].push_back(i);
      std::unordered_map<i64, i64> comp_saved;
      for (auto& pw : pos_pairs) comp_saved[find(local[pw.first / n_chunks])] += pw.second;
      std::vector<std::pair<i64, i64>> reps;  // (min chunk id, root)
      for (auto& kv : comp) {
        i64 mn = INT64_MAX;
        for (i64 i : kv.second) mn = std::min<i64>(mn, device_chunks[i]);
        reps.emplace_back(mn, kv.first);
      }
      std::sort(reps.begin(), reps.end());
      i64 ng = 0;
      std::vector<int> in_comp(0);
      for (auto& rv : reps) {
        const auto& idx = comp[rv.second];
        std::unordered_set<i64> mem_set;
        i64 nm = 0, ed = 0;
        for (i64 i : idx) {
          out_group_of_chunk[i] = (int32_t)ng;
          nm += (i64)g[i].member_list.size();
          ed += g[i].edges;
          for (i64 v : g[i].member_list) mem_set.insert(v);
        }
        std::unordered_set<i64> ext;
        for (i64 i : idx)
          for (i64 x : g[i].ext_halo)
            if (!mem_set.count(x)) ext.insert(x);
        out_group_memory[ng] = memory_of(nm, (i64)ext.size(), ed);
        auto cs = comp_saved.find(rv.second);
        out_group_saved[ng] = cs == comp_saved.end() ? 0 : cs->second;
        ++ng;
      }
      *n_groups_out = ng;
      return DGC_OK;
    }
  }
  // owner: instance -> live group index; rep -> group index
  std::unordered_map<i64, i64> owner;
  owner.reserve((size_t)n_instances / 2 + 16);
  std::unordered_map<i64, i64> gi_of_rep;
  for (i64 i = 0; i < C; ++i) {
    gi_of_rep[g[i].rep] = i;
    for (i64 v : g[i].member_list) owner[v] = i;
  }
  auto key = [&](i64 a, i64 b) { return a < b ? a * n_chunks + b : b * n_chunks + a; };
  std::unordered_map<i64, i64> saving;
  std::unordered_set<i64> dead;
  std::unordered_map<i64, std::unordered_set<i64>> pairs_of;
  std::priority_queue<HeapItem> heap;
  for (auto& kv : inter) {
    if (kv.second <= 0) continue;
    const i64 a = kv.first / n_chunks, b = kv.first % n_chunks;
    if (local[a] < 0 || local[b] < 0) continue;
    saving[kv.first] = kv.second;
    pairs_of[a].insert(kv.first);
    pairs_of[b].insert(kv.first);
    heap.push({kv.second, a, b});
  }
  auto owner_of = [&](i64 v) {
    auto it = owner.find(v);
    return it == owner.end() ? (i64)-1 : it->second;
  };
  while (!heap.empty()) {
    const HeapItem top = heap.top();
    heap.pop();
    const i64 k = key(top.a, top.b);
    auto sit = saving.find(k);
    if (sit == saving.end() || sit->second != top.w || dead.count(k)) continue;
    const i64 ia = gi_of_rep[top.a], ib = gi_of_rep[top.b];
    Group& A = g[ia];
    Group& B = g[ib];
    // small-into-large estimate of |members U halo| after the merge
    const i64 sa = (i64)A.member_list.size() + (i64)A.ext_halo.size();
    const i64 sb = (i64)B.member_list.size() + (i64)B.ext_halo.size();
    const i64 is = sa <= sb ? ia : ib, il = sa <= sb ? ib : ia;
    Group& S = g[is];
    Group& Lg = g[il];
    i64 ms_in_xl = 0;
    for (i64 m : S.member_list) ms_in_xl += Lg.ext_halo.count(m);
    i64 new_from_xs = 0;
    for (i64 x : S.ext_halo)
      if (owner_of(x) != il && !Lg.ext_halo.count(x)) ++new_from_xs;
    const i64 n_ext = (i64)Lg.ext_halo.size() - ms_in_xl + new_from_xs;
    const i64 n_mem = (i64)S.member_list.size() + (i64)Lg.member_list.size();
    if (memory_of(n_mem, n_ext, A.edges + B.edges) > memory_budget) {
      dead.insert(k);
      continue;
    }
    // apply the merge into the larger group
    const i64 w = top.w;
    const i64 new_saved = A.saved + B.saved + w;
    const i64 rep = std::min(top.a, top.b);
    for (i64 m : S.member_list) {
      Lg.ext_halo.erase(m);
      owner[m] = il;
    }
    for (i64 x : S.ext_halo)
      if (owner_of(x) != il) Lg.ext_halo.insert(x);
    Lg.member_list.insert(Lg.member_list.end(), S.member_list.begin(), S.member_list.end());
    Lg.chunk_ids.insert(Lg.chunk_ids.end(), S.chunk_ids.begin(), S.chunk_ids.end());
    Lg.edges = A.edges + B.edges;
    Lg.saved = new_saved;
    Lg.rep = rep;
    S.member_list.clear();
    S.member_list.shrink_to_fit();
    S.ext_halo.clear();
    S.chunk_ids.clear();
    gi_of_rep.erase(top.a);
    gi_of_rep.erase(top.b);
    gi_of_rep[rep] = il;
    // re-key the pair savings (fusion.py:182-198)
    std::unordered_set<i64> touched;
    for (i64 kk : pairs_of[top.a]) touched.insert(kk);
    for (i64 kk : pairs_of[top.b]) touched.insert(kk);
    pairs_of.erase(top.a);
    pairs_of.erase(top.b);
    pairs_of[rep];
    for (i64 kk : touched) {
      const i64 k0 = kk / n_chunks, k1 = kk % n_chunks;
      const i64 other = (k1 == top.a || k1 == top.b) ? k0 : k1;
      i64 w_old = 0;
      auto it = saving.find(kk);
      if (it != saving.end()) {
        w_old = it->second;
        saving.erase(it);
      }
      dead.erase(kk);
      if (other == top.a || other == top.b || w_old == 0) continue;
      pairs_of[other].erase(kk);
      const i64 nk = key(rep, other);
      auto it2 = saving.find(nk);
      const i64 new_w = (it2 == saving.end() ? 0 : it2->second) + w_old;
      saving[nk] = new_w;
      pairs_of[other].insert(nk);
      pairs_of[rep].insert(nk);
      heap.push({new_w, std::min(rep, other), std::max(rep, other)});
    }
  }
  // output: groups sorted by representative chunk id (fusion.py:200-203)
  std::vector<std::pair<i64, i64>> reps(gi_of_rep.begin(), gi_of_rep.end());
  std::sort(reps.begin(), reps.end());
  i64 ng = 0;
  for (auto& rv : reps) {
    Group& G = g[rv.second];
    for (i64 c : G.chunk_ids) out_group_of_chunk[local[c]] = (int32_t)ng;
    out_group_memory[ng] = memory_of((i64)G.member_list.size(), (i64)G.ext_halo.size(), G.edges);
    out_group_saved[ng] = G.saved;
    ++ng;
  }
  *n_groups_out = ng;
  return DGC_OK;
}
