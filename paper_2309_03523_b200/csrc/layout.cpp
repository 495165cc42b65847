// Host-side plan -> per-device layout builder.
//
// Consumes the reference plan unchanged (Plan.structure_device sim.py:120,
// chunk membership partition.py:49-56, FusionPlan groups fusion.py:78-105)
// and derives, for one device, every index array the GPU step needs:
//   * own rows in fusion-group order (groups sorted by representative chunk,
//     fusion.py:200-203), ascending global index inside a group
//     (partition.py:303-304) -> one batched CSR per device;
//   * halo = remote spatial neighbours, ascending global index; CSR with the
//     self loop, columns sorted by neighbour global index (fixed reduction
//     order); its transpose for the backward;
//   * boundary keys and per-peer send/recv lists (cut spatial messages,
//     costmodel.py:106-165);
//   * time-encoder runs enumerated exactly as _device_sequences
//     (sim.py:401-420), keyed by run index, FFD-packed as pack_sequences
//     (fusion.py:249-313), plus the cross-device carry lists;
//   * loaded rows per execution unit as _pgc_units counts them (sim.py:339-360).
// Native because the reference planner's Python loops do not scale to the
// 1M-10M instance configurations.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/dgc_b200.h"

namespace dgc {
void set_error(const std::string& msg);
}

struct dgc_layout {
  std::vector<int64_t> f[DGC_F_COUNT];
};

namespace {

using i64 = int64_t;

// fusion.py:249-275 -- exact first-fit-decreasing; the scan restarts only when
// the length value drops.
void ffd_place(const std::vector<i64>& lengths, i64 row_length, std::vector<i64>& row_of,
               std::vector<i64>& used) {
  const i64 n = (i64)lengths.size();
  std::vector<i64> order(n);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(),
                   [&](i64 a, i64 b) { return lengths[a] > lengths[b]; });
  row_of.assign(n, 0);
  used.clear();
  i64 start = 0, prev = -1;
  for (i64 i : order) {
    const i64 len = lengths[i];
    if (len != prev) {
      start = 0;
      prev = len;
    }
    i64 r = start;
    while (r < (i64)used.size() && used[r] + len > row_length) ++r;
    start = r;
    if (r == (i64)used.size()) used.push_back(0);
    used[r] += len;
    row_of[i] = r;
  }
}

// fusion.py:278-313 pack_sequences keyed by sequence index.
void pack(const std::vector<i64>& lengths, i64& R, i64& L, std::vector<i64>& slot_seq,
          std::vector<i64>& slot_pos, std::vector<i64>& mask, i64& padding) {
  const i64 n = (i64)lengths.size();
  if (n == 0) {
    R = L = padding = 0;
    slot_seq.clear();
    slot_pos.clear();
    mask.clear();
    return;
  }
  L = *std::max_element(lengths.begin(), lengths.end());
  std::vector<i64> row_of, used;
  ffd_place(lengths, L, row_of, used);
  R = (i64)used.size();
  slot_seq.assign(R * L, -1);
  slot_pos.assign(R * L, -1);
  std::vector<i64> fill(R, 0), order(n);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(),
                   [&](i64 a, i64 b) { return lengths[a] > lengths[b]; });
  for (i64 i : order) {
    const i64 r = row_of[i];
    for (i64 p = 0; p < lengths[i]; ++p) {
      slot_seq[r * L + fill[r] + p] = i;
      slot_pos[r * L + fill[r] + p] = p;
    }
    fill[r] += lengths[i];
  }
  mask.assign(R * L, 0);
  for (i64 r = 0; r < R; ++r)
    for (i64 p = 1; p < L; ++p) {
      const i64 a = r * L + p - 1, b = r * L + p;
      if (slot_seq[a] >= 0 && slot_seq[b] == slot_seq[a] && slot_pos[b] == slot_pos[a] + 1)
        mask[b] = 1;
    }
  padding = 0;
  for (i64 u : used) padding += L - u;
}

void build(const dgc_plan_view& pv, int d, dgc_layout& out) {
  const i64 N = pv.n_instances;
  const int D = pv.n_devices;
  const int32_t* sdev = pv.structure_device;
  auto& F = out.f;
  // own rows: (segment, gid)
  std::vector<i64> seg_of_chunk;
  if (pv.n_groups > 0) {
    i64 max_chunk = 0;
    for (i64 i = 0; i < N; ++i) max_chunk = std::max<i64>(max_chunk, pv.chunk_of[i]);
    seg_of_chunk.assign(max_chunk + 1, -1);
    i64 seg = 0;
    for (i64 g = 0; g < pv.n_groups; ++g) {
      if (pv.group_device[g] != d) continue;
      for (i64 k = pv.group_ptr[g]; k < pv.group_ptr[g + 1]; ++k) seg_of_chunk[pv.group_chunks[k]] = seg;
      ++seg;
    }
  }
  std::vector<std::pair<i64, i64>> own_key;
  for (i64 i = 0; i < N; ++i) {
    if (sdev[i] != d) continue;
    const i64 seg = pv.n_groups > 0 ? seg_of_chunk[pv.chunk_of[i]] : pv.chunk_of[i];
    if (seg < 0) throw std::runtime_error("instance's chunk is not in any fusion group of its device");
    own_key.emplace_back(seg, i);
  }
  std::sort(own_key.begin(), own_key.end());
  auto& own = F[DGC_F_OWN_GID];
  auto& gptr = F[DGC_F_GROUP_PTR];
  auto& segp = F[DGC_F_SEG_PTR];
  gptr.clear();
  segp.clear();
  own.clear();
  if (pv.segment_rows > 0) {
    // EvolveGCN (per-snapshot weights): rows grouped by snapshot, each snapshot
    // block padded with -1 rows to a multiple of segment_rows so every GEMM
    // M-tile lies in one snapshot. Fusion groups of such plans are
    // snapshot-local, so a group stays one contiguous segment.
    i64 T = 0;
    for (i64 i = 0; i < N; ++i) T = std::max<i64>(T, pv.inst_t[i]);
    std::stable_sort(own_key.begin(), own_key.end(), [&](const std::pair<i64, i64>& a,
                                                         const std::pair<i64, i64>& b) {
      return pv.inst_t[a.second] < pv.inst_t[b.second];
    });
    size_t k = 0;
    for (i64 t = 1; t <= T; ++t) {
      segp.push_back((i64)own.size());
      i64 prev_seg = -1;
      while (k < own_key.size() && pv.inst_t[own_key[k].second] == t) {
        if (own_key[k].first != prev_seg) gptr.push_back((i64)own.size());
        prev_seg = own_key[k].first;
        own.push_back(own_key[k].second);
        ++k;
      }
      while (own.size() % (size_t)pv.segment_rows) own.push_back(-1);
    }
    segp.push_back((i64)own.size());
  } else {
    for (size_t k = 0; k < own_key.size(); ++k) {
      own.push_back(own_key[k].second);
      if (k == 0 || own_key[k].first != own_key[k - 1].first) gptr.push_back((i64)k);
    }
  }
  const i64 n_own = (i64)own.size();
  gptr.push_back(n_own);
  // global adjacency (neighbours sorted by gid) and degrees
  const i64 E = pv.n_spatial_edges;
  std::vector<i64> adj_ptr(N + 1, 0), adj;
  for (i64 e = 0; e < E; ++e) {
    adj_ptr[pv.spatial_edges[2 * e] + 1]++;
    adj_ptr[pv.spatial_edges[2 * e + 1] + 1]++;
  }
  for (i64 i = 0; i < N; ++i) adj_ptr[i + 1] += adj_ptr[i];
  adj.resize(adj_ptr[N]);
  {
    std::vector<i64> fill(adj_ptr.begin(), adj_ptr.end() - 1);
    for (i64 e = 0; e < E; ++e) {
      const i64 u = pv.spatial_edges[2 * e], v = pv.spatial_edges[2 * e + 1];
      adj[fill[u]++] = v;
      adj[fill[v]++] = u;
    }
    for (i64 i = 0; i < N; ++i) std::sort(adj.begin() + adj_ptr[i], adj.begin() + adj_ptr[i + 1]);
  }
  // local ids: own then halo (ascending gid)
  std::vector<i64> local(N, -1);
  for (i64 k = 0; k < n_own; ++k)
    if (own[k] >= 0) local[own[k]] = k;
  auto& halo = F[DGC_F_HALO_GID];
  halo.clear();
  for (i64 k = 0; k < n_own; ++k) {
    if (own[k] < 0) continue;
    for (i64 e = adj_ptr[own[k]]; e < adj_ptr[own[k] + 1]; ++e)
      if (sdev[adj[e]] != d) halo.push_back(adj[e]);
  }
  std::sort(halo.begin(), halo.end());
  halo.erase(std::unique(halo.begin(), halo.end()), halo.end());
  const i64 n_halo = (i64)halo.size();
  for (i64 h = 0; h < n_halo; ++h) local[halo[h]] = n_own + h;
  const i64 n_loc = n_own + n_halo;
  // degrees of every local column (full snapshot graph, Appendix B.1)
  auto& deg = F[DGC_F_DEG];
  deg.resize(n_loc);
  for (i64 c = 0; c < n_loc; ++c) {
    const i64 g = c < n_own ? own[c] : halo[c - n_own];
    deg[c] = g >= 0 ? adj_ptr[g + 1] - adj_ptr[g] : 0;  // padding rows: no entries
  }
  // forward CSR with self loop, columns by neighbour gid
  auto& rp = F[DGC_F_ROW_PTR];
  auto& col = F[DGC_F_COL];
  rp.assign(1, 0);
  col.clear();
  for (i64 k = 0; k < n_own; ++k) {
    const i64 u = own[k];
    if (u < 0) {  // padding row: empty
      rp.push_back((i64)col.size());
      continue;
    }
    bool self_done = false;
    for (i64 e = adj_ptr[u]; e < adj_ptr[u + 1]; ++e) {
      if (!self_done && adj[e] > u) {
        col.push_back(k);
        self_done = true;
      }
      col.push_back(local[adj[e]]);
    }
    if (!self_done) col.push_back(k);
    rp.push_back((i64)col.size());
  }
  // transposed CSR: per local column, own rows in ascending gid
  auto& trp = F[DGC_F_T_ROW_PTR];
  auto& tcol = F[DGC_F_T_COL];
  trp.assign(n_loc + 1, 0);
  for (i64 e = 0; e < (i64)col.size(); ++e) trp[col[e] + 1]++;
  for (i64 c = 0; c < n_loc; ++c) trp[c + 1] += trp[c];
  tcol.assign(col.size(), 0);
  {
    std::vector<i64> by_gid(n_own);
    std::iota(by_gid.begin(), by_gid.end(), 0);
    std::sort(by_gid.begin(), by_gid.end(), [&](i64 a, i64 b) { return own[a] < own[b]; });
    std::vector<i64> fill(trp.begin(), trp.end() - 1);
    for (i64 k : by_gid)
      for (i64 e = rp[k]; e < rp[k + 1]; ++e) tcol[fill[col[e]]++] = k;
  }
  // boundary keys (ascending gid) and per-peer lists
  std::vector<i64> own_sorted;
  for (i64 g : own)
    if (g >= 0) own_sorted.push_back(g);
  std::sort(own_sorted.begin(), own_sorted.end());
  auto& keys = F[DGC_F_KEY_ROWS];
  keys.clear();
  std::vector<i64> key_pos(n_own, -1);
  for (i64 g : own_sorted) {
    bool b = false;
    for (i64 e = adj_ptr[g]; e < adj_ptr[g + 1] && !b; ++e) b = sdev[adj[e]] != d;
    if (b) {
      key_pos[local[g]] = (i64)keys.size();
      keys.push_back(local[g]);
    }
  }
  auto& kncut = F[DGC_F_KEY_NCUT];
  kncut.assign(keys.size(), 0);
  for (size_t kk = 0; kk < keys.size(); ++kk) {
    const i64 g = own[keys[kk]];
    for (i64 e = adj_ptr[g]; e < adj_ptr[g + 1]; ++e) kncut[kk] += sdev[adj[e]] != d;
  }
  auto& sptr = F[DGC_F_SEND_PTR];
  auto& spos = F[DGC_F_SEND_POS];
  auto& rptr = F[DGC_F_RECV_PTR];
  auto& rslot = F[DGC_F_RECV_SLOT];
  sptr.assign(1, 0);
  rptr.assign(1, 0);
  spos.clear();
  rslot.clear();
  for (int p = 0; p < D; ++p) {
    if (p != d) {
      for (i64 kk = 0; kk < (i64)keys.size(); ++kk) {
        const i64 g = own[keys[kk]];
        bool b = false;
        for (i64 e = adj_ptr[g]; e < adj_ptr[g + 1] && !b; ++e) b = sdev[adj[e]] == p;
        if (b) spos.push_back(kk);
      }
      for (i64 h = 0; h < n_halo; ++h)
        if (sdev[halo[h]] == p) rslot.push_back(n_own + h);
    }
    sptr.push_back((i64)spos.size());
    rptr.push_back((i64)rslot.size());
  }
  // temporal links: pred/succ
  std::vector<i64> pred(N, -1), succ(N, -1);
  for (i64 l = 0; l < pv.n_temporal_links; ++l) {
    const i64 a = pv.temporal_links[2 * l], b = pv.temporal_links[2 * l + 1];
    succ[a] = b;
    pred[b] = a;
  }
  // runs: entities ascending, presences ascending, split at device changes
  std::vector<i64> order(N);
  std::iota(order.begin(), order.end(), 0);
  std::sort(order.begin(), order.end(), [&](i64 a, i64 b) {
    if (pv.inst_entity[a] != pv.inst_entity[b]) return pv.inst_entity[a] < pv.inst_entity[b];
    return pv.inst_t[a] < pv.inst_t[b];
  });
  auto& run_ptr = F[DGC_F_RUN_PTR];
  auto& run_rows = F[DGC_F_RUN_ROWS];
  auto& run_pred = F[DGC_F_RUN_PRED_GID];
  auto& run_carry = F[DGC_F_RUN_CARRY];
  run_ptr.assign(1, 0);
  run_rows.clear();
  run_pred.clear();
  run_carry.clear();
  i64 n_carry = 0;
  for (i64 k = 0; k < N;) {
    const i64 e0 = pv.inst_entity[order[k]];
    const int dd = sdev[order[k]];
    i64 k2 = k;
    while (k2 < N && pv.inst_entity[order[k2]] == e0 && sdev[order[k2]] == dd) ++k2;
    if (dd == d) {
      for (i64 q = k; q < k2; ++q) run_rows.push_back(local[order[q]]);
      run_ptr.push_back((i64)run_rows.size());
      const i64 pg = pred[order[k]];
      const bool remote = pg >= 0 && sdev[pg] != d;
      run_pred.push_back(remote ? pg : -1);
      run_carry.push_back(remote ? n_carry++ : -1);
    }
    k = k2;
  }
  const i64 n_runs = (i64)run_pred.size();
  std::vector<i64> lengths(n_runs);
  for (i64 r = 0; r < n_runs; ++r) lengths[r] = run_ptr[r + 1] - run_ptr[r];
  i64 R = 0, L = 0, padding = 0;
  std::vector<i64> sseq, spos2, mask;
  pack(lengths, R, L, sseq, spos2, mask, padding);
  auto& srow = F[DGC_F_SLOT_ROW];
  auto& smask = F[DGC_F_SLOT_MASK];
  auto& scarry = F[DGC_F_SLOT_CARRY];
  srow.assign(R * L, -1);
  scarry.assign(R * L, -1);
  smask = mask;
  for (i64 s = 0; s < R * L; ++s) {
    if (sseq[s] < 0) continue;
    srow[s] = run_rows[run_ptr[sseq[s]] + spos2[s]];
    if (spos2[s] == 0) scarry[s] = run_carry[sseq[s]];
  }
  i64 naive = 0;
  for (i64 len : lengths) naive += L - len;
  // temporal carry keys and lists
  auto& tkeys = F[DGC_F_TKEY_ROWS];
  tkeys.clear();
  for (i64 g : own_sorted)
    if (succ[g] >= 0 && sdev[succ[g]] != d) tkeys.push_back(local[g]);
  auto& tsp = F[DGC_F_TSEND_PTR];
  auto& tspos = F[DGC_F_TSEND_POS];
  auto& trp2 = F[DGC_F_TRECV_PTR];
  auto& trc = F[DGC_F_TRECV_CARRY];
  tsp.assign(1, 0);
  trp2.assign(1, 0);
  tspos.clear();
  trc.clear();
  std::vector<std::pair<i64, i64>> pred_carry;  // (pred gid, carry slot)
  for (i64 r = 0; r < n_runs; ++r)
    if (run_pred[r] >= 0) pred_carry.emplace_back(run_pred[r], run_carry[r]);
  std::sort(pred_carry.begin(), pred_carry.end());
  for (int p = 0; p < D; ++p) {
    if (p != d) {
      for (i64 kk = 0; kk < (i64)tkeys.size(); ++kk)
        if (sdev[succ[own[tkeys[kk]]]] == p) tspos.push_back(kk);
      for (auto& pc : pred_carry)
        if (sdev[pc.first] == p) trc.push_back(pc.second);
    }
    tsp.push_back((i64)tspos.size());
    trp2.push_back((i64)trc.size());
  }
  // loaded rows per execution unit (members U chunk halos), sim.py:339-360
  i64 loaded = 0;
  {
    std::vector<i64> stamp(N, -1);
    for (size_t gi = 0; gi + 1 < gptr.size(); ++gi) {
      i64 cnt = 0;
      auto mark = [&](i64 g) {
        if (stamp[g] != (i64)gi) {
          stamp[g] = (i64)gi;
          ++cnt;
        }
      };
      for (i64 k = gptr[gi]; k < gptr[gi + 1]; ++k) {
        const i64 g = own[k];
        if (g < 0) continue;
        mark(g);
        for (i64 e = adj_ptr[g]; e < adj_ptr[g + 1]; ++e) mark(adj[e]);
        if (pred[g] >= 0) mark(pred[g]);
        if (succ[g] >= 0) mark(succ[g]);
      }
      loaded += cnt;
    }
  }
  F[DGC_F_SCALARS] = {n_own, n_halo, R, L, padding, naive, n_carry, loaded};
}

}  // namespace

extern "C" int dgc_layout_build(const dgc_plan_view* plan, int32_t device, dgc_layout** out) {
  if (!plan || !out) {
    dgc::set_error("layout_build: null argument");
    return DGC_ERR_ARG;
  }
  if (device < 0 || device >= plan->n_devices) {
    dgc::set_error("layout_build: device out of range");
    return DGC_ERR_ARG;
  }
  for (int64_t i = 0; i < plan->n_instances; ++i) {
    if (plan->structure_device[i] < 0 || plan->structure_device[i] >= plan->n_devices) {
      dgc::set_error("layout_build: structure_device entry out of range (PlanGraphMismatch)");
      return DGC_ERR_PLAN;
    }
  }
  auto* lay = new dgc_layout();
  try {
    build(*plan, device, *lay);
  } catch (const std::exception& e) {
    delete lay;
    dgc::set_error(std::string("layout_build: ") + e.what());
    return DGC_ERR_PLAN;
  }
  *out = lay;
  return DGC_OK;
}

extern "C" int64_t dgc_layout_field(const dgc_layout* lay, int32_t field, const int64_t** data) {
  if (!lay || field < 0 || field >= DGC_F_COUNT) return -1;
  *data = lay->f[field].data();
  return (int64_t)lay->f[field].size();
}

extern "C" void dgc_layout_free(dgc_layout* lay) { delete lay; }

extern "C" int dgc_pack_sequences(const int32_t* lengths, int64_t n, int32_t row_len,
                                  int64_t capacity_rows, int32_t* slot_seq, int32_t* slot_pos,
                                  uint8_t* mask, int64_t* n_rows, int64_t* padding) {
  std::vector<int64_t> len(n);
  int64_t mx = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (lengths[i] < 1) {
      dgc::set_error("pack_sequences: sequence length must be >= 1");
      return DGC_ERR_ARG;
    }
    len[i] = lengths[i];
    mx = std::max<int64_t>(mx, lengths[i]);
  }
  if (n > 0 && row_len != mx) {
    dgc::set_error("pack_sequences: row_len must equal max(lengths)");
    return DGC_ERR_ARG;
  }
  int64_t R, L, pad;
  std::vector<int64_t> sseq, spos, m;
  pack(len, R, L, sseq, spos, m, pad);
  if (R > capacity_rows) {
    dgc::set_error("pack_sequences: capacity_rows too small");
    return DGC_ERR_ARG;
  }
  for (int64_t s = 0; s < R * L; ++s) {
    slot_seq[s] = (int32_t)sseq[s];
    slot_pos[s] = (int32_t)spos[s];
    mask[s] = (uint8_t)m[s];
  }
  *n_rows = R;
  *padding = pad;
  return DGC_OK;
}
