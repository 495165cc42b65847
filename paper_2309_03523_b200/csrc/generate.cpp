// Native synthetic dynamic-graph generator.
//
// Restates the contract of the reference generator dynpart.graphstore.generate
// (graphstore.py:525-579) -- not its random stream (bit-exact RNG is not
// required; the plan built from the graph is what the training step consumes
// unchanged):
//   * entities draw a presence length from the LengthDistribution
//     (graphstore.py:367-382: constant / uniform / bimodal / geometric, clipped
//     to [1, T]) until the lengths sum to total_vertices (the last one
//     truncated), and are placed at a uniform start so the run of consecutive
//     presences fits in [1, T] (graphstore.py:537-553);
//   * per-snapshot edge counts are normal(mean, stddev) draws clipped at 0 and
//     renormalised to total_edges by largest remainder (graphstore.py:555-557,
//     _largest_remainder :440-451);
//   * each snapshot samples its count of distinct unordered vertex pairs:
//     uniformly (_sample_distinct_pairs :454-478) or preferentially
//     (_sample_preferential_pairs :481-522: batched rounds of 2*(k-chosen)+8
//     endpoint draws proportional to within-snapshot degree + 1, the weights
//     fixed within a round, rejecting self pairs and duplicates; after four
//     rounds without progress the remainder is filled uniformly from the unused
//     pairs); a snapshot that cannot host its quota is an error
//     (InfeasibleSpecError).
// Output in the reference's orders: presences grouped by entity (ascending
// entity id, ascending t), edges by snapshot with each snapshot's pairs sorted
// (u < v, entity ids). Snapshots are sampled in parallel from per-snapshot
// streams (splitmix64-seeded xoshiro256**), so the result depends only on the
// seed, never on the thread count. C5 (10M instances, 40M edges, 128
// snapshots) takes seconds instead of the reference's ~25 minutes.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <string>
#include <thread>
#include <unordered_set>
#include <vector>

#include "../../include/dgc_b200.h"

namespace dgc {
int fail(int code, const std::string& msg);
}

namespace {

struct Rng {  // xoshiro256**, seeded by splitmix64
  uint64_t s[4];
  explicit Rng(uint64_t seed) {
    for (int i = 0; i < 4; ++i) {
      seed += 0x9e3779b97f4a7c15ull;
      uint64_t z = seed;
      z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
      z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
      s[i] = z ^ (z >> 31);
    }
  }
  static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
  uint64_t next() {
    const uint64_t r = rotl(s[1] * 5, 7) * 9, t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return r;
  }
  double uniform() { return (next() >> 11) * 0x1.0p-53; }          // [0, 1)
  int64_t integer(int64_t lo, int64_t hi) {                          // [lo, hi]
    const uint64_t span = (uint64_t)(hi - lo) + 1;
    return lo + (int64_t)(((unsigned __int128)next() * span) >> 64);
  }
  double normal() {  // Box-Muller
    double u1 = uniform();
    while (u1 <= 0.0) u1 = uniform();
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * uniform());
  }
  int64_t geometric(double p) {  // trials to first success, >= 1
    if (p >= 1.0) return 1;
    double u = uniform();
    while (u <= 0.0) u = uniform();
    return 1 + (int64_t)std::floor(std::log(u) / std::log1p(-p));
  }
};

int64_t sample_length(Rng& rng, const dgc_length_dist& d, int T) {
  int64_t v;
  switch (d.kind) {
    case DGC_LEN_CONSTANT: v = d.value; break;
    case DGC_LEN_UNIFORM: v = rng.integer(d.low, d.high); break;
    case DGC_LEN_BIMODAL:
      v = rng.integer(d.low, d.high);
      if (rng.uniform() < d.long_fraction) v = rng.integer(d.long_low, d.long_high);
      break;
    default: v = rng.geometric(1.0 / d.mean); break;
  }
  return std::min<int64_t>(std::max<int64_t>(v, 1), T);
}

// k distinct sorted pairs (i < j) of range(n): uniform or preferential.
// Returns false when k exceeds n(n-1)/2.
bool sample_pairs(Rng& rng, int64_t n, int64_t k, bool preferential,
                  std::vector<std::pair<int32_t, int32_t>>& out) {
  out.clear();
  const int64_t max_pairs = n * (n - 1) / 2;
  if (k > max_pairs) return false;
  if (k == 0) return true;
  auto key = [n](int64_t u, int64_t v) { return (uint64_t)u * (uint64_t)n + (uint64_t)v; };
  std::unordered_set<uint64_t> chosen;
  chosen.reserve((size_t)k * 2);
  auto fill_uniform_from_pool = [&](int64_t remaining) {
    // dense corner: every unused pair, then a uniform choice without replacement
    std::vector<uint64_t> pool;
    pool.reserve((size_t)(max_pairs - (int64_t)chosen.size()));
    for (int64_t i = 0; i < n; ++i)
      for (int64_t j = i + 1; j < n; ++j)
        if (!chosen.count(key(i, j))) pool.push_back(key(i, j));
    for (int64_t r = 0; r < remaining; ++r) {  // partial Fisher-Yates
      const int64_t pick = rng.integer(r, (int64_t)pool.size() - 1);
      std::swap(pool[r], pool[pick]);
      chosen.insert(pool[r]);
    }
  };
  if (!preferential) {
    if (2 * k >= max_pairs) {
      fill_uniform_from_pool(k);
    } else {
      while ((int64_t)chosen.size() < k) {
        const int64_t u = rng.integer(0, n - 1), v = rng.integer(0, n - 1);
        if (u == v) continue;
        chosen.insert(key(std::min(u, v), std::max(u, v)));
      }
    }
  } else {
    std::vector<double> deg((size_t)n, 1.0), cdf((size_t)n);
    int stall = 0;
    while ((int64_t)chosen.size() < k) {
      const int64_t m = 2 * (k - (int64_t)chosen.size()) + 8;
      std::partial_sum(deg.begin(), deg.end(), cdf.begin());
      const double total = cdf.back();
      auto draw = [&]() {
        const double x = rng.uniform() * total;
        const int64_t i = std::upper_bound(cdf.begin(), cdf.end(), x) - cdf.begin();
        return std::min<int64_t>(i, n - 1);
      };
      std::vector<int64_t> a((size_t)m), b((size_t)m);
      for (int64_t i = 0; i < m; ++i) a[i] = draw();
      for (int64_t i = 0; i < m; ++i) b[i] = draw();
      int64_t added = 0;
      for (int64_t i = 0; i < m && (int64_t)chosen.size() < k; ++i) {
        const int64_t u = a[i], v = b[i];
        if (u == v) continue;
        if (!chosen.insert(key(std::min(u, v), std::max(u, v))).second) continue;
        deg[u] += 1.0;
        deg[v] += 1.0;
        ++added;
      }
      stall = added == 0 ? stall + 1 : 0;
      if (stall >= 4) fill_uniform_from_pool(k - (int64_t)chosen.size());
    }
  }
  std::vector<uint64_t> keys(chosen.begin(), chosen.end());
  std::sort(keys.begin(), keys.end());
  out.reserve(keys.size());
  for (uint64_t kk : keys) out.emplace_back((int32_t)(kk / (uint64_t)n), (int32_t)(kk % (uint64_t)n));
  return true;
}

}  // namespace

extern "C" int dgc_generate_graph(const dgc_synthetic_spec* spec, int32_t* presences,
                                  int32_t* edges, int64_t* n_entities, int32_t n_threads) {
  if (!spec || !presences || !edges || !n_entities) return dgc::fail(DGC_ERR_ARG, "generate: null argument");
  const int T = spec->T;
  if (T < 1) return dgc::fail(DGC_ERR_ARG, "T must be >= 1");
  if (spec->total_vertices < 1) return dgc::fail(DGC_ERR_ARG, "total_vertices must be >= 1");
  if (spec->total_edges < 0) return dgc::fail(DGC_ERR_ARG, "total_edges must be >= 0");
  if (!(spec->edges_per_snapshot_mean > 0)) return dgc::fail(DGC_ERR_ARG, "edges_per_snapshot_mean must be > 0");
  if (!(spec->edges_per_snapshot_stddev >= 0)) return dgc::fail(DGC_ERR_ARG, "edges_per_snapshot_stddev must be >= 0");
  const dgc_length_dist& d = spec->length;
  if ((d.kind == DGC_LEN_UNIFORM || d.kind == DGC_LEN_BIMODAL) && !(1 <= d.low && d.low <= d.high))
    return dgc::fail(DGC_ERR_ARG, "uniform length bounds need 1 <= low <= high");
  if (d.kind == DGC_LEN_CONSTANT && d.value < 1) return dgc::fail(DGC_ERR_ARG, "constant length must be >= 1");
  if (d.kind == DGC_LEN_GEOMETRIC && !(d.mean >= 1.0)) return dgc::fail(DGC_ERR_ARG, "geometric mean length must be >= 1");
  if (d.kind == DGC_LEN_BIMODAL &&
      (!(1 <= d.long_low && d.long_low <= d.long_high) || !(0.0 <= d.long_fraction && d.long_fraction <= 1.0)))
    return dgc::fail(DGC_ERR_ARG, "bimodal long bounds need 1 <= long_low <= long_high, 0 <= long_fraction <= 1");

  Rng rng(spec->rng_seed);
  // presence lengths and starts
  std::vector<int32_t> lengths, starts;
  int64_t remaining = spec->total_vertices;
  while (remaining > 0) {
    const int64_t len = std::min(sample_length(rng, d, T), remaining);
    lengths.push_back((int32_t)len);
    remaining -= len;
  }
  const int64_t n_ent = (int64_t)lengths.size();
  starts.resize((size_t)n_ent);
  for (int64_t e = 0; e < n_ent; ++e) starts[e] = (int32_t)rng.integer(1, T - lengths[e] + 1);
  std::vector<std::vector<int32_t>> verts((size_t)T);
  int64_t w = 0;
  for (int64_t e = 0; e < n_ent; ++e)
    for (int t = starts[e]; t < starts[e] + lengths[e]; ++t) {
      presences[2 * w] = (int32_t)e;
      presences[2 * w + 1] = t;
      ++w;
      verts[(size_t)t - 1].push_back((int32_t)e);  // ascending entity order
    }
  // per-snapshot edge counts: clipped normal draws, largest remainder
  std::vector<double> quota((size_t)T);
  double wsum = 0.0;
  for (int t = 0; t < T; ++t) {
    quota[t] = std::max(0.0, spec->edges_per_snapshot_mean + spec->edges_per_snapshot_stddev * rng.normal());
    wsum += quota[t];
  }
  if (wsum <= 0.0) {
    std::fill(quota.begin(), quota.end(), 1.0);
    wsum = T;
  }
  std::vector<int64_t> counts((size_t)T);
  int64_t assigned = 0;
  for (int t = 0; t < T; ++t) {
    quota[t] *= (double)spec->total_edges / wsum;
    counts[t] = (int64_t)std::floor(quota[t]);
    assigned += counts[t];
  }
  if (assigned < spec->total_edges) {
    std::vector<int> order((size_t)T);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
      return quota[a] - counts[a] > quota[b] - counts[b];
    });
    for (int64_t i = 0; i < spec->total_edges - assigned; ++i) counts[order[(size_t)i]] += 1;
  }
  std::vector<int64_t> eoff((size_t)T + 1, 0);
  for (int t = 0; t < T; ++t) eoff[t + 1] = eoff[t] + counts[t];
  // snapshots in parallel, one stream per snapshot
  std::atomic<int> next{0}, bad{-1};
  auto worker = [&]() {
    std::vector<std::pair<int32_t, int32_t>> pairs;
    for (int t = next++; t < T; t = next++) {
      Rng r(spec->rng_seed ^ (0xd1b54a32d192ed03ull * (uint64_t)(t + 1)));
      const auto& vs = verts[(size_t)t];
      if (!sample_pairs(r, (int64_t)vs.size(), counts[t], spec->preferential != 0, pairs)) {
        int expect = -1;
        bad.compare_exchange_strong(expect, t);
        continue;
      }
      int32_t* o = edges + 3 * eoff[t];
      for (size_t i = 0; i < pairs.size(); ++i) {
        o[3 * i] = t + 1;
        o[3 * i + 1] = vs[(size_t)pairs[i].first];
        o[3 * i + 2] = vs[(size_t)pairs[i].second];
      }
    }
  };
  int nt = n_threads > 0 ? n_threads : (int)std::max(1u, std::thread::hardware_concurrency());
  nt = std::min(nt, T);
  std::vector<std::thread> pool;
  for (int i = 1; i < nt; ++i) pool.emplace_back(worker);
  worker();
  for (auto& th : pool) th.join();
  if (bad.load() >= 0) {
    const int t = bad.load();
    const int64_t n = (int64_t)verts[(size_t)t].size();
    return dgc::fail(DGC_ERR_ARG, "snapshot " + std::to_string(t + 1) + ": " + std::to_string(counts[t]) +
                                      " edges requested but only " + std::to_string(n * (n - 1) / 2) +
                                      " possible");
  }
  *n_entities = n_ent;
  return DGC_OK;
}
