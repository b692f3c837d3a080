// Host side of libshapflow_b200: the C-ABI (include/shapflow_b200.h), the
// size plan, graph construction / SFG1 I/O / computational-graph
// extraction, model construction, and the explain_node orchestration that
// drives the sm_100a kernels. Written from the reference's documented
// behaviour (citations per function); no compute falls back to the CPU.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <cinttypes>
#include <charconv>
#include <fstream>
#include <numeric>
#include <sstream>
#include <atomic>
#include <exception>
#include <mutex>
#include <thread>

#include "../../include/shapflow_b200.h"
#include "sf_internal.hpp"

namespace sfb {

// ---------------------------------------------------------------- Philox (host)
// philox.hpp:13-73, for model generation and seeds on the host.
namespace {
struct HostPhilox {
  uint32_t key[2], stream[2];
  uint64_t counter = 0;
  uint32_t block[4] = {};
  int have = 0;
  HostPhilox(uint64_t seed, uint64_t s)
      : key{uint32_t(seed), uint32_t(seed >> 32)}, stream{uint32_t(s), uint32_t(s >> 32)} {}
  uint64_t next_u64() {
    if (have == 0) {
      uint32_t c[4] = {uint32_t(counter), uint32_t(counter >> 32), stream[0], stream[1]};
      uint32_t k0 = key[0], k1 = key[1];
      for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = uint64_t(0xD2511F53u) * c[0];
        const uint64_t p1 = uint64_t(0xCD9E8D57u) * c[2];
        const uint32_t n0 = uint32_t(p1 >> 32) ^ c[1] ^ k0;
        const uint32_t n2 = uint32_t(p0 >> 32) ^ c[3] ^ k1;
        c[0] = n0;
        c[1] = uint32_t(p1);
        c[2] = n2;
        c[3] = uint32_t(p0);
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
      }
      std::memcpy(block, c, sizeof c);
      ++counter;
      have = 2;
    }
    --have;
    return (uint64_t(block[2 * have + 1]) << 32) | block[2 * have];
  }
  double next_double() { return double(next_u64() >> 11) * 0x1.0p-53; }
};
}  // namespace

// ---------------------------------------------------------------- plan
uint64_t binomial_or_max(uint32_t n, uint32_t s) {  // sampler.cpp:67-77
  if (s > n) return 0;
  s = std::min(s, n - s);
  unsigned __int128 r = 1;
  for (uint32_t i = 1; i <= s; ++i) {
    r = r * (n - s + i) / i;
    if (r > UINT64_MAX) return UINT64_MAX;
  }
  return static_cast<uint64_t>(r);
}

SizePlan plan_sizes(uint32_t n, uint64_t k, bool allow_exhaustive) {
  // sampler.cpp:93-151: pairs split by per-size mass (n-1)/(s(n-s)) (x2 for
  // a pair covering sizes s and n-s), floor quotas then largest remainder
  // with ties to the smaller size; classes contiguous in the pair index.
  if (n < 2)
    throw DataError("plan_sizes: need at least 2 players, got " + std::to_string(n));
  if (k == 0) throw DataError("plan_sizes: sample budget must be positive");
  SizePlan plan;
  plan.n = n;
  if (k & 1) ++k;
  plan.requested = k;
  if (allow_exhaustive && n <= 62 && ((uint64_t{1} << n) - 2) <= k) {
    plan.exhaustive = true;
    uint64_t next = 0;
    for (uint32_t s = 1; 2 * s <= n; ++s) {
      uint64_t pairs = binomial_or_max(n, s);
      if (2 * s == n) pairs /= 2;  // keep the half containing player 0
      plan.classes.push_back({s, pairs, next});
      next += pairs;
    }
    return plan;
  }
  const uint64_t total_pairs = k / 2;
  const uint32_t half = n / 2;
  std::vector<double> mass(half + 1, 0.0);
  double mass_sum = 0.0;
  for (uint32_t s = 1; s <= half; ++s) {
    const double rho = (n - 1.0) / (double(s) * double(n - s));
    mass[s] = (2 * s == n) ? rho : 2.0 * rho;
    mass_sum += mass[s];
  }
  std::vector<uint64_t> quota(half + 1, 0);
  std::vector<std::pair<double, uint32_t>> order;
  order.reserve(half);
  uint64_t assigned = 0;
  for (uint32_t s = 1; s <= half; ++s) {
    const double ideal = double(total_pairs) * (mass[s] / mass_sum);
    const uint64_t q = static_cast<uint64_t>(std::floor(ideal));
    quota[s] = q;
    assigned += q;
    order.emplace_back(-(ideal - double(q)), s);
  }
  // the reference sorts and hands one extra pair to the first R entries,
  // cycling; only the SET of the first R % size entries matters, so a
  // selection (same comparator, ties to the smaller size) replaces the sort
  const uint64_t R = total_pairs - assigned;
  const uint64_t rounds = R / order.size(), rest = R % order.size();
  if (rounds)
    for (uint32_t s = 1; s <= half; ++s) quota[s] += rounds;
  if (rest) {
    std::nth_element(order.begin(), order.begin() + (rest - 1), order.end());
    for (uint64_t i = 0; i < rest; ++i) ++quota[order[i].second];
  }
  assigned = total_pairs;
  uint64_t next = 0;
  for (uint32_t s = 1; s <= half; ++s) {
    if (quota[s] == 0) continue;
    plan.classes.push_back({s, quota[s], next});
    next += quota[s];
  }
  return plan;
}

std::vector<uint64_t> global_rows_of_size(const SizePlan& plan) {
  // sampler.cpp:168-176
  std::vector<uint64_t> c(size_t(plan.n) + 1, 0);
  for (const SizeClass& cls : plan.classes) {
    if (2 * cls.size == plan.n) {
      c[cls.size] += 2 * cls.pairs;
    } else {
      c[cls.size] += cls.pairs;
      c[plan.n - cls.size] += cls.pairs;
    }
  }
  return c;
}

uint64_t local_pair_count(uint64_t global_pairs, int rank, int world) {
  // pairs g = rank, rank + world, ... (sampler.cpp:177-178)
  if (uint64_t(rank) >= global_pairs) return 0;
  return (global_pairs - rank + world - 1) / world;
}

// per-size weights normalized by the first populated size (solver.cpp:125-138)
static std::vector<double> weight_of_size(uint32_t n, const std::vector<uint64_t>& counts) {
  std::vector<double> w(size_t(n) + 1, 0.0);
  double scale = 0.0;
  for (uint32_t s = 1; s < n; ++s) {
    if (counts[s] == 0) continue;
    const double rho = (n - 1.0) / (double(s) * double(n - s));
    const double ws = rho / static_cast<double>(counts[s]);
    if (scale == 0.0) scale = ws;
    w[s] = ws / scale;
  }
  return w;
}

// ---------------------------------------------------------------- graphs
static Graph build_graph(uint32_t num_nodes, const uint64_t* edges, uint64_t num_edges,
                         std::vector<float> features, uint64_t dim,
                         std::vector<uint32_t> labels) {
  // graph.cpp:127-163: symmetrize, drop self-loops, dedupe, sorted rows
  if (features.size() != uint64_t(num_nodes) * dim)
    throw DataError("feature buffer size does not match num_nodes x dim");
  if (labels.empty()) labels.assign(num_nodes, 0xFFFFFFFFu);
  if (labels.size() != num_nodes) throw DataError("label buffer size does not match num_nodes");
  std::vector<uint64_t> dir;
  dir.reserve(num_edges * 2);
  for (uint64_t i = 0; i < num_edges; ++i) {
    const uint64_t u = edges[2 * i], v = edges[2 * i + 1];
    if (u >= num_nodes || v >= num_nodes)
      throw DataError("edge endpoint out of range: (" + std::to_string(u) + ", " +
                      std::to_string(v) + ") with " + std::to_string(num_nodes) + " nodes");
    if (u == v) continue;
    dir.push_back((u << 32) | v);
    dir.push_back((v << 32) | u);
  }
  std::sort(dir.begin(), dir.end());
  dir.erase(std::unique(dir.begin(), dir.end()), dir.end());
  Graph g;
  g.num_nodes = num_nodes;
  g.feature_dim = dim;
  g.features = std::move(features);
  g.labels = std::move(labels);
  g.row_ptr.assign(size_t(num_nodes) + 1, 0);
  for (uint64_t x : dir) g.row_ptr[(x >> 32) + 1]++;
  for (size_t i = 1; i <= num_nodes; ++i) g.row_ptr[i] += g.row_ptr[i - 1];
  g.col.resize(dir.size());
  for (size_t i = 0; i < dir.size(); ++i) g.col[i] = uint32_t(dir[i]);
  return g;
}

template <typename T>
static void read_raw(std::istream& in, T* dst, size_t count, const char* what) {
  in.read(reinterpret_cast<char*>(dst), std::streamsize(sizeof(T) * count));
  if (!in) throw DataError(std::string("graph file truncated while reading ") + what);
}

static Graph load_sfg(const std::string& path) {
  // SFG1 (graph.cpp:35-64): magic, u64 nodes, u64 edges, u64 dim,
  // edges as u64 pairs, f32 features, u32 labels
  std::ifstream in(path, std::ios::binary);
  if (!in) throw DataError("cannot open graph file: " + path);
  char magic[4];
  read_raw(in, magic, 4, "magic");
  if (std::memcmp(magic, "SFG1", 4) != 0) throw DataError("bad magic in " + path + " (expected SFG1)");
  uint64_t nodes = 0, edges = 0, dim = 0;
  read_raw(in, &nodes, 1, "node count");
  read_raw(in, &edges, 1, "edge count");
  read_raw(in, &dim, 1, "feature dim");
  if (nodes > 0xFFFFFFFFull) throw DataError("node count too large: " + std::to_string(nodes));
  std::vector<uint64_t> flat(edges * 2);
  read_raw(in, flat.data(), flat.size(), "edges");
  std::vector<float> f(nodes * dim);
  read_raw(in, f.data(), f.size(), "features");
  std::vector<uint32_t> labels(nodes);
  read_raw(in, labels.data(), labels.size(), "labels");
  return build_graph(uint32_t(nodes), flat.data(), edges, std::move(f), dim, std::move(labels));
}

static void save_sfg(const Graph& g, const std::string& path) {
  std::ofstream out(path, std::ios::binary | std::ios::trunc);
  if (!out) throw DataError("cannot write graph file: " + path);
  out.write("SFG1", 4);
  const uint64_t nodes = g.num_nodes, edges = g.col.size() / 2, dim = g.feature_dim;
  out.write(reinterpret_cast<const char*>(&nodes), 8);
  out.write(reinterpret_cast<const char*>(&edges), 8);
  out.write(reinterpret_cast<const char*>(&dim), 8);
  for (uint32_t u = 0; u < g.num_nodes; ++u)
    for (uint64_t i = g.row_ptr[u]; i < g.row_ptr[u + 1]; ++i)
      if (u < g.col[i]) {
        const uint64_t pr[2] = {u, g.col[i]};
        out.write(reinterpret_cast<const char*>(pr), 16);
      }
  out.write(reinterpret_cast<const char*>(g.features.data()), std::streamsize(g.features.size() * 4));
  out.write(reinterpret_cast<const char*>(g.labels.data()), std::streamsize(g.labels.size() * 4));
  if (!out) throw DataError("write failed: " + path);
}

// graphs with at least this many CSR entries are extracted on the device
// (SF_EXTRACT=host|device|auto)
constexpr uint64_t kDeviceExtractNnz = 1u << 20;

static Subgraph extract(const Graph& g, uint32_t target, int hops, bool with_features = true) {
  // graph.cpp:195-261: BFS ball (discovery order = local ids, target 0),
  // induced undirected edges sorted lexicographically, symmetric local CSR
  // with edge_player, feature slice.
  if (target >= g.num_nodes) throw DataError("target node " + std::to_string(target) + " out of range");
  if (hops < 0) throw DataError("hop count must be nonnegative");
  DebugTimer dt("extract");
  std::vector<uint32_t> local_of(g.num_nodes, 0xFFFFFFFFu);
  Subgraph sg;
  sg.target_global = target;
  sg.feature_dim = g.feature_dim;
  sg.local_to_global.push_back(target);
  local_of[target] = 0;
  size_t fb = 0;
  for (int hop = 0; hop < hops; ++hop) {
    const size_t fe = sg.local_to_global.size();
    if (fb == fe) break;
    for (size_t i = fb; i < fe; ++i) {
      const uint32_t u = sg.local_to_global[i];
      for (uint64_t k = g.row_ptr[u]; k < g.row_ptr[u + 1]; ++k) {
        const uint32_t nb = g.col[k];
        if (local_of[nb] == 0xFFFFFFFFu) {
          local_of[nb] = uint32_t(sg.local_to_global.size());
          sg.local_to_global.push_back(nb);
        }
      }
    }
    fb = fe;
  }
  dt.lap("bfs");
  const uint32_t V = sg.num_nodes();
  // lexicographic (lu, lv) order without a sort: walking the larger
  // endpoint lv in ascending order and appending it to bucket lu fills every
  // bucket in ascending lv; buckets laid out in lu order (counting pass
  // first). Multi-edges stay adjacent, as after a sort.
  // (branch-free: the lu < lv test is a coin flip per entry; rejected
  // entries go to a dummy bucket V whose cursor never moves)
  std::vector<uint64_t> bstart(size_t(V) + 2, 0);
  for (uint32_t lv = 0; lv < V; ++lv) {
    const uint32_t v = sg.local_to_global[lv];
    for (uint64_t k = g.row_ptr[v]; k < g.row_ptr[v + 1]; ++k) {
      const uint32_t lu = local_of[g.col[k]];  // unmapped ids are 0xFFFFFFFF > lv
      const bool keep = lu < lv;
      bstart[(keep ? lu : V) + 1] += keep;
    }
  }
  for (uint32_t u = 0; u < V; ++u) bstart[u + 1] += bstart[u];
  const uint64_t total = bstart[V];
  bstart[V] = total;  // the dummy bucket's cursor: one scratch slot past the end
  sg.players.resize(total + 1);
  for (uint32_t lv = 0; lv < V; ++lv) {
    const uint32_t v = sg.local_to_global[lv];
    for (uint64_t k = g.row_ptr[v]; k < g.row_ptr[v + 1]; ++k) {
      const uint32_t lu = local_of[g.col[k]];
      const bool keep = lu < lv;
      uint64_t& cur = bstart[keep ? lu : V];
      sg.players[cur] = {lu, lv};
      cur += keep;
    }
  }
  sg.players.pop_back();
  dt.lap("edges");
  std::vector<uint64_t> deg(V, 0);
  for (const auto& [u, v] : sg.players) {
    deg[u]++;
    deg[v]++;
  }
  sg.row_ptr.assign(size_t(V) + 1, 0);
  for (uint32_t u = 0; u < V; ++u) sg.row_ptr[u + 1] = sg.row_ptr[u] + deg[u];
  sg.col.resize(sg.row_ptr.back());
  sg.edge_player.resize(sg.row_ptr.back());
  std::vector<uint64_t> cursor(sg.row_ptr.begin(), sg.row_ptr.end() - 1);
  for (uint32_t e = 0; e < sg.players.size(); ++e) {
    const auto [u, v] = sg.players[e];
    sg.col[cursor[u]] = v;
    sg.edge_player[cursor[u]++] = e;
    sg.col[cursor[v]] = u;
    sg.edge_player[cursor[v]++] = e;
  }
  dt.lap("csr");
  if (!with_features) {  // the engine gathers the rows from a device copy of the graph's features
    sg.source = &g;
    return sg;
  }
  sg.features.resize(uint64_t(V) * g.feature_dim);
  for (uint32_t lu = 0; lu < V; ++lu)
    std::memcpy(sg.features.data() + uint64_t(lu) * g.feature_dim,
                g.features.data() + uint64_t(sg.local_to_global[lu]) * g.feature_dim,
                g.feature_dim * 4);
  return sg;
}

std::vector<uint64_t> Subgraph::ball_sizes(int hops) const {
  const uint32_t V = num_nodes();
  std::vector<int> dist(V, -1);
  std::vector<uint32_t> q;
  q.reserve(V);
  if (V) {
    dist[0] = 0;
    q.push_back(0);
  }
  for (size_t h = 0; h < q.size(); ++h) {
    const uint32_t u = q[h];
    for (uint64_t k = row_ptr[u]; k < row_ptr[u + 1]; ++k)
      if (dist[col[k]] < 0) {
        dist[col[k]] = dist[u] + 1;
        q.push_back(col[k]);
      }
  }
  std::vector<uint64_t> out(size_t(hops) + 1, 0);
  for (int h = 0; h <= hops; ++h) {
    uint64_t c = 0;
    while (c < V && dist[c] >= 0 && dist[c] <= h) ++c;
    for (uint64_t x = c; x < V; ++x)
      if (dist[x] >= 0 && dist[x] <= h)
        throw DataError("subgraph local ids are not in breadth-first order");
    out[h] = c;
  }
  return out;
}

// ---------------------------------------------------------------- model
static void validate_model(const Model& m) {  // gcn.cpp:14-33
  if (m.layers.empty()) throw DataError("model has no layers");
  for (size_t l = 0; l < m.layers.size(); ++l) {
    const Layer& lay = m.layers[l];
    if (lay.in == 0 || lay.out == 0)
      throw DataError("layer " + std::to_string(l) + " has a zero dimension");
    if (l > 0 && m.layers[l - 1].out != lay.in)
      throw DataError("dimension chain broken between layers " + std::to_string(l - 1) +
                      " and " + std::to_string(l));
  }
}

static Model random_model(uint64_t input_dim, const uint64_t* hidden, int nh, uint32_t classes,
                          uint64_t seed) {
  // synthetic.cpp:88-118: Glorot uniform from Philox(seed, 16 + l), zero bias
  if (input_dim == 0 || classes == 0)
    throw DataError("model needs at least one input feature and one class");
  std::vector<uint64_t> dims{input_dim};
  for (int i = 0; i < nh; ++i) dims.push_back(hidden[i]);
  dims.push_back(classes);
  Model m;
  for (size_t l = 0; l + 1 < dims.size(); ++l) {
    Layer lay;
    lay.in = dims[l];
    lay.out = dims[l + 1];
    if (lay.in == 0 || lay.out == 0) throw DataError("hidden layer widths must be positive");
    HostPhilox rng(seed, 16 + l);
    const double limit = std::sqrt(6.0 / double(lay.in + lay.out));
    lay.weight.resize(lay.in * lay.out);
    for (float& w : lay.weight) w = static_cast<float>(limit * (2.0 * rng.next_double() - 1.0));
    lay.bias.assign(lay.out, 0.0f);
    m.layers.push_back(std::move(lay));
  }
  return m;
}

// ---------------------------------------------------------------- engine I/O
static void upload_rows(Ctx& ctx, const uint64_t* bits, uint64_t rows, uint64_t words,
                        uint32_t W) {
  // rows may be wider than words_for_bits(n); keep the first W words
  ctx.masks.reserve(std::max<uint64_t>(rows * W, 1));
  if (rows == 0) return;
  ctx.h2d_bytes += rows * W * 8;
  if (words == W) {
    SF_CUDA(cudaMemcpyAsync(ctx.masks.p, bits, rows * W * 8, cudaMemcpyHostToDevice, ctx.stream));
  } else {
    SF_CUDA(cudaMemcpy2DAsync(ctx.masks.p, W * 8, bits, words * 8, W * 8, rows,
                              cudaMemcpyHostToDevice, ctx.stream));
  }
}

static void predict_rows(Ctx& ctx, const Subgraph& sg, const Model& m, const uint64_t* dev_rows,
                         uint64_t rows, uint32_t cls, float* host_out, float* host_probs) {
  engine_prepare(ctx, sg, m);
  const uint32_t C = uint32_t(m.layers.back().out);
  ctx.preds.reserve(std::max<uint64_t>(rows * (host_probs ? C + 1 : 1), 1));
  float* d_out = ctx.preds.p;
  float* d_probs = host_probs ? ctx.preds.p + rows : nullptr;
  engine_predict(ctx, dev_rows, rows, cls, d_out, d_probs, nullptr);
  ctx.d2h_bytes += (host_out ? rows * 4 : 0) + (host_probs ? rows * C * 4 : 0);
  if (host_out)
    SF_CUDA(cudaMemcpyAsync(host_out, d_out, rows * 4, cudaMemcpyDeviceToHost, ctx.stream));
  if (host_probs)
    SF_CUDA(cudaMemcpyAsync(host_probs, d_probs, rows * C * 4, cudaMemcpyDeviceToHost, ctx.stream));
  SF_CUDA(cudaStreamSynchronize(ctx.stream));
}

// ---------------------------------------------------------------- fidelity
static uint32_t kept_at_sparsity(uint32_t n, double sparsity) {  // fidelity.cpp:42-49
  if (!(sparsity >= 0.0 && sparsity <= 1.0))
    throw DataError("sparsity must lie in [0, 1], got " + std::to_string(sparsity));
  const auto kept = static_cast<uint32_t>(std::ceil((1.0 - sparsity) * double(n)));
  return std::min(kept, n);
}

// solver.cpp:430-440: players by phi descending, ties by index ascending.
// LSD radix sort (8 stable byte passes) on an order-preserving key of phi
// (+0 and -0 share a key, as they compare equal): input in index order, so
// stability gives the index tie-break. NaN never reaches here (the solver
// rejects non-finite values).
static std::vector<uint32_t> ranking(const std::vector<double>& phi) {
  const size_t n = phi.size();
  if (n == 0) return {};
  std::vector<uint64_t> key(n), key2(n);
  std::vector<uint32_t> o(n), o2(n);
  for (size_t i = 0; i < n; ++i) {
    const double v = phi[i] == 0.0 ? 0.0 : phi[i];
    uint64_t b;
    std::memcpy(&b, &v, 8);
    b = (b >> 63) ? ~b : (b | (uint64_t{1} << 63));  // ascending in v
    key[i] = ~b;                                     // descending
    o[i] = uint32_t(i);
  }
  for (int pass = 0; pass < 8; ++pass) {
    const int sh = pass * 8;
    size_t cnt[257] = {0};
    for (size_t i = 0; i < n; ++i) ++cnt[((key[i] >> sh) & 255) + 1];
    if (cnt[((key[0] >> sh) & 255) + 1] == n) continue;  // all equal: nothing to do
    for (int b = 0; b < 256; ++b) cnt[b + 1] += cnt[b];
    for (size_t i = 0; i < n; ++i) {
      const size_t d = cnt[(key[i] >> sh) & 255]++;
      key2[d] = key[i];
      o2[d] = o[i];
    }
    key.swap(key2);
    o.swap(o2);
  }
  return o;
}

struct FidelityOut {
  std::vector<uint32_t> counts;
  std::vector<double> plus, plus_random, sparsities, minus, minus_random;
};

// fidelity.cpp:126-162, every mask scored in one batch on the device engine.
// Row layout: [full] [plus_c for each count] [plus_random trials per count]
// [minus_s per sparsity] [minus_random trials per sparsity]; the random
// baselines are Floyd draws on the device with the reference's streams.
static FidelityOut fidelity(Ctx& ctx, const Subgraph& sg, const Model& m, uint32_t cls,
                            const std::vector<double>& phi, const std::vector<uint32_t>& counts,
                            const std::vector<double>& sparsities, uint64_t seed,
                            uint32_t trials, const std::vector<uint32_t>* ranked_in = nullptr) {
  const uint32_t n = uint32_t(sg.num_players());
  if (phi.size() != n)
    throw DataError("attribution vector has " + std::to_string(phi.size()) + " entries for " +
                    std::to_string(n) + " players");
  DebugTimer dt("fidelity");
  const uint32_t W = std::max<uint32_t>(1, (n + 63) / 64);
  const std::vector<uint32_t> ranked = ranked_in ? *ranked_in : ranking(phi);
  dt.lap("ranking");
  const uint64_t tail = (n % 64) ? ((uint64_t{1} << (n % 64)) - 1) : ~uint64_t{0};
  std::vector<uint64_t> full(W, ~uint64_t{0});
  if (n == 0) full.assign(W, 0);
  else full[W - 1] = tail;
  const size_t nc = counts.size(), ns = sparsities.size();
  const uint64_t rows = 1 + nc + nc * trials + ns + ns * trials;
  std::vector<uint64_t> host(rows * W, 0);
  auto row = [&](uint64_t r) { return host.data() + r * W; };
  std::copy(full.begin(), full.end(), row(0));
  FidelityOut out;
  std::vector<uint64_t> streams;
  std::vector<uint32_t> sizes;
  std::vector<uint8_t> invert;
  std::vector<uint64_t> job_rows;
  for (size_t i = 0; i < nc; ++i) {
    const uint32_t c = std::min(counts[i], n);
    out.counts.push_back(c);
    uint64_t* r = row(1 + i);
    std::copy(full.begin(), full.end(), r);
    for (uint32_t k = 0; k < c; ++k) r[ranked[k] >> 6] &= ~(uint64_t{1} << (ranked[k] & 63));
    for (uint32_t t = 0; t < trials; ++t) {
      streams.push_back((uint64_t(c) << 32) | t);  // fidelity.cpp:99-100
      sizes.push_back(c);
      invert.push_back(1);
      job_rows.push_back(1 + nc + i * trials + t);
    }
  }
  const uint64_t mbase = 1 + nc + nc * trials;
  for (size_t i = 0; i < ns; ++i) {
    const uint32_t keep = kept_at_sparsity(n, sparsities[i]);
    out.sparsities.push_back(sparsities[i]);
    uint64_t* r = row(mbase + i);
    for (uint32_t k = 0; k < keep; ++k) r[ranked[k] >> 6] |= uint64_t{1} << (ranked[k] & 63);
    for (uint32_t t = 0; t < trials; ++t) {
      streams.push_back((uint64_t(keep) << 32) | (uint64_t{1} << 63) | t);  // 117-118
      sizes.push_back(keep);
      invert.push_back(0);
      job_rows.push_back(mbase + ns + i * trials + t);
    }
  }
  dt.lap("host rows");
  // device: deterministic rows, then the Floyd jobs written in place
  ctx.masks.reserve(rows * W);
  SF_CUDA(cudaMemcpyAsync(ctx.masks.p, host.data(), rows * W * 8, cudaMemcpyHostToDevice, ctx.stream));
  ctx.h2d_bytes += rows * W * 8;
  const uint64_t jobs = streams.size();
  if (jobs) {
    DevBuf<uint64_t>& d_streams = ctx.fid_streams;
    DevBuf<uint64_t>& d_rows = ctx.fid_rows;
    DevBuf<uint32_t>& d_sizes = ctx.fid_sizes;
    DevBuf<uint8_t>& d_inv = ctx.fid_inv;
    d_streams.upload(streams.data(), jobs, ctx.stream);
    d_sizes.upload(sizes.data(), jobs, ctx.stream);
    d_inv.upload(invert.data(), jobs, ctx.stream);
    d_rows.reserve(jobs * W);
    launch_floyd_jobs(ctx, n, seed, d_streams.p, d_sizes.p, d_inv.p, jobs, d_rows.p);
    // trial rows are contiguous per block: copy the job rows into place
    for (uint64_t j = 0; j < jobs;) {
      uint64_t k = j;
      while (k + 1 < jobs && job_rows[k + 1] == job_rows[k] + 1) ++k;
      SF_CUDA(cudaMemcpyAsync(ctx.masks.p + job_rows[j] * W, d_rows.p + j * W,
                              (k - j + 1) * W * 8, cudaMemcpyDeviceToDevice, ctx.stream));
      j = k + 1;
    }
    SF_CUDA(cudaStreamSynchronize(ctx.stream));
  }
  dt.lap("random baselines");
  std::vector<float> score(rows);
  predict_rows(ctx, sg, m, ctx.masks.p, rows, cls, score.data(), nullptr);
  dt.lap("predict");
  const double f0 = double(score[0]);
  for (size_t i = 0; i < nc; ++i) {
    out.plus.push_back(std::abs(f0 - double(score[1 + i])));
    double acc = 0.0;
    for (uint32_t t = 0; t < trials; ++t) acc += std::abs(f0 - double(score[1 + nc + i * trials + t]));
    out.plus_random.push_back(trials ? acc / double(trials) : 0.0);
  }
  for (size_t i = 0; i < ns; ++i) {
    out.minus.push_back(std::abs(f0 - double(score[mbase + i])));
    double acc = 0.0;
    for (uint32_t t = 0; t < trials; ++t)
      acc += std::abs(f0 - double(score[mbase + ns + i * trials + t]));
    out.minus_random.push_back(trials ? acc / double(trials) : 0.0);
  }
  return out;
}

// ---------------------------------------------------------------- explain
using Clock = std::chrono::steady_clock;
static double ms_since(Clock::time_point t) {
  return std::chrono::duration<double, std::milli>(Clock::now() - t).count();
}

template <typename T>
static T* dup_array(const std::vector<T>& v) {
  T* p = static_cast<T*>(std::malloc(sizeof(T) * std::max<size_t>(v.size(), 1)));
  if (!p) throw std::bad_alloc();
  if (!v.empty()) std::memcpy(p, v.data(), sizeof(T) * v.size());
  return p;
}

static void explain_node(Ctx& ctx, const Graph& g, const Model& m, uint32_t node,
                         const sf_explain_options& o, sf_explanation* out) {
  // explain.cpp:42-143
  const auto t_start = Clock::now();
  std::memset(out, 0, sizeof(*out));
  out->node = node;
  out->converged = 1;
  if (o.batch_size == 0) throw DataError("batch_size must be positive");
  if (o.solver_mode < SF_SOLVER_CGLS || o.solver_mode > SF_SOLVER_AUTO)
    throw DataError("unknown solver mode " + std::to_string(o.solver_mode));
  if (m.layers.front().in != g.feature_dim)
    throw DataError("model expects " + std::to_string(m.layers.front().in) +
                    " input features but the graph has " + std::to_string(g.feature_dim));
  DebugTimer("explain").lap("start");
  // large graphs: the BFS ball and local CSR on the device (byte-identical)
  static const char* ex_env = std::getenv("SF_EXTRACT");
  static const std::string ex_mode = ex_env ? ex_env : "auto";
  const bool on_device = ex_mode == "device" || (ex_mode == "auto" && g.col.size() >= kDeviceExtractNnz);
  const Subgraph sg = on_device ? extract_device(ctx, g, node, int(m.depth())) : extract(g, node, m.depth(), false);
  out->extract_ms = ms_since(t_start);
  DebugTimer("explain").lap("extracted");
  const uint64_t n_raw = sg.num_players();
  if (o.player_cap != 0 && n_raw > o.player_cap) {
    out->skipped = 1;
    std::snprintf(out->warning, sizeof(out->warning),
                  "node %u skipped: %llu players exceed the cap of %llu", node,
                  (unsigned long long)n_raw, (unsigned long long)o.player_cap);
    out->total_ms = ms_since(t_start);
    return;
  }
  const uint32_t n = uint32_t(n_raw);
  const uint64_t seed = sf_node_sampling_seed(o.seed, node);
  const uint32_t W = std::max<uint32_t>(1, (n + 63) / 64);
  const uint32_t C = uint32_t(m.layers.back().out);

  // full-mask probabilities -> class (first argmax), empty-mask base score
  {
    const auto t_setup = Clock::now();
    std::vector<uint64_t> two(2 * W, 0);
    for (uint32_t w = 0; w < W; ++w) two[w] = ~uint64_t{0};
    if (n % 64) two[W - 1] = (uint64_t{1} << (n % 64)) - 1;
    if (n == 0) two[0] = 0;
    upload_rows(ctx, two.data(), 2, W, W);
    std::vector<float> probs(2 * C);
    predict_rows(ctx, sg, m, ctx.masks.p, 2, 0, nullptr, probs.data());
    const uint32_t cls = uint32_t(std::max_element(probs.begin(), probs.begin() + C) - probs.begin());
    DebugTimer("explain").lap("full/empty scores done");
    out->predicted_class = cls;
    out->full_score = double(probs[cls]);
    out->base_score = double(probs[C + cls]);
    out->setup_ms = ms_since(t_setup);
  }
  std::vector<uint32_t> players_global;
  players_global.reserve(2 * n);
  for (const auto& [u, v] : sg.players) {
    uint32_t gu = sg.local_to_global[u], gv = sg.local_to_global[v];
    if (gu > gv) std::swap(gu, gv);
    players_global.push_back(gu);
    players_global.push_back(gv);
  }
  out->num_players = n;
  out->players_global = dup_array(players_global);
  std::vector<double> phi;
  if (n == 0) {
    out->exhaustive = 1;
  } else if (n == 1) {
    phi = {out->full_score - out->base_score};
    out->exhaustive = 1;
  } else {
    const uint64_t k = o.samples ? o.samples : sf_auto_samples(n);
    comm_barrier(ctx);
    auto t_stage = Clock::now();
    DebugTimer sdt("sampling");
    const SizePlan plan = plan_sizes(n, k, o.allow_exhaustive != 0);
    sdt.lap("plan");
    const uint64_t pairs = local_pair_count(plan.total_pairs(), ctx.rank, ctx.world);
    const uint64_t rows = 2 * pairs;
    // kept-set rows only (the complement of every pair is derived where it
    // is read): half the mask bytes in HBM and half the sampler writes
    ctx.masks.reserve(std::max<uint64_t>(pairs * W, 1));
    launch_generate_masks(ctx, plan, seed, ctx.rank, ctx.world, ctx.masks.p, /*kept_only=*/true);
    sdt.lap("launch");
    comm_barrier(ctx);
    sdt.lap("masks");
    out->sampling_ms = ms_since(t_stage);
    out->exhaustive = plan.exhaustive ? 1 : 0;
    out->rows = plan.total_pairs() * 2;

    t_stage = Clock::now();
    engine_prepare(ctx, sg, m);
    ctx.preds.reserve(std::max<uint64_t>(rows, 1));
    engine_predict(ctx, ctx.masks.p, rows, out->predicted_class, ctx.preds.p, nullptr, nullptr, /*kept_only=*/true);
    comm_barrier(ctx);
    out->prediction_ms = ms_since(t_stage);
    if (ctx.keep_stages) {
      ctx.kept_preds.resize(rows);
      SF_CUDA(cudaMemcpyAsync(ctx.kept_preds.data(), ctx.preds.p, rows * 4, cudaMemcpyDeviceToHost, ctx.stream));
      SF_CUDA(cudaStreamSynchronize(ctx.stream));
    }

    t_stage = Clock::now();
    const std::vector<double> wsize = weight_of_size(n, global_rows_of_size(plan));
    DevBuf<double>& d_wsize = ctx.wsize_dev;
    DevBuf<double>& d_sw = ctx.sw_dev;
    DevBuf<double>& d_tgt = ctx.tgt_dev;
    DevBuf<int>& d_bad = ctx.bad_dev;
    d_wsize.upload(wsize.data(), wsize.size(), ctx.stream);
    d_sw.reserve(std::max<uint64_t>(rows, 1));
    d_tgt.reserve(std::max<uint64_t>(rows, 1));
    const int big = 0x7fffffff;
    d_bad.upload(&big, 1, ctx.stream);
    ctx.pop_dev.reserve(std::max<uint64_t>(rows, 1));
    ctx.comp_dev.reserve(std::max<uint64_t>(rows / 2, 1));
    launch_assemble_pairs(ctx, ctx.masks.p, rows, W, n, d_wsize.p, ctx.preds.p, out->base_score, d_sw.p,
                          d_tgt.p, d_bad.p, ctx.pop_dev.p, ctx.comp_dev.p, /*kept_only=*/true);
    ctx.h2d_bytes += wsize.size() * 8 + 4;
    ctx.d2h_bytes += 4;
    int bad = big;
    SF_CUDA(cudaMemcpyAsync(&bad, d_bad.p, sizeof(int), cudaMemcpyDeviceToHost, ctx.stream));
    SF_CUDA(cudaStreamSynchronize(ctx.stream));
    if (bad != big)
      throw DataError("coalition row " + std::to_string(bad) + " keeps all or no players");
    CglsInput in;
    in.n = n;
    in.rows = rows;
    in.W = W;
    in.dev_rows = ctx.masks.p;
    in.dev_sw = d_sw.p;
    in.dev_targets = d_tgt.p;
    in.constraint_target = out->full_score - out->base_score;
    in.constraint_weight = o.constraint_scale;
    in.global_pair_count = plan.total_pairs();
    in.dev_pop = ctx.pop_dev.p;
    in.dev_is_comp = ctx.comp_dev.p;
    in.kept_only = true;
    in.rows_scratch_words = ctx.masks.n;  // the masks are not read after the solve
    DebugTimer("explain").lap("assemble done");
    // Solver dispatch: the direct (tcgen05 Gram + device Cholesky) path
    // for small player counts on one worker, CGLS otherwise. Crossover
    // measured at k = 100K (profiles/round2/solver_crossover.jsonl): direct
    // 0.53-0.99 ms vs CGLS 0.83-1.08 ms up to n = 250, slower from n = 500.
    static const uint64_t direct_max =
        std::getenv("SF_DIRECT_MAX") ? std::strtoull(std::getenv("SF_DIRECT_MAX"), nullptr, 10) : 256;
    const bool direct = o.solver_mode == SF_SOLVER_DIRECT ||
                        (o.solver_mode == SF_SOLVER_AUTO && ctx.world == 1 && n <= direct_max);
    if (o.solver_mode == SF_SOLVER_DIRECT && ctx.world != 1)
      throw DataError("direct solve needs the full system on a single worker");
    CglsResult res;
    if (direct) {
      // one weight run per size class (w_s == w_{n-s}: both rows of a pair)
      std::vector<GramRun> runs;
      for (const SizeClass& c : plan.classes) {
        const double we = wsize[c.size], wo = wsize[n - c.size];
        const uint64_t r0 = 2 * c.first_pair, r1 = 2 * (c.first_pair + c.pairs);
        if (we == wo) {
          runs.push_back(GramRun{r0, r1, we});
        } else {
          for (uint64_t r = r0; r < r1; ++r) runs.push_back(GramRun{r, r + 1, (r & 1) ? wo : we});
        }
      }
      res.phi = gram_solve(ctx, in, runs);
      res.converged = true;
    } else {
      in.fixed_order = o.fixed_order != 0 && o.solver_mode != SF_SOLVER_FUSED;
      res = cgls_solve(ctx, in, o.tol, o.max_iter, o.solver_mode == SF_SOLVER_FUSED ? 1 : 0, false);
    }
    comm_barrier(ctx);
    out->solve_ms = ms_since(t_stage);
    phi = std::move(res.phi);
    out->iterations = uint32_t(res.iterations);
    out->residual = res.relative_residual;
    out->converged = res.converged ? 1 : 0;
    if (!res.converged) {
      std::ostringstream msg;
      msg << "node " << node << ": solver stopped after " << res.iterations
          << " iterations at relative residual " << res.relative_residual << " (tol " << o.tol
          << ")";
      std::snprintf(out->warning, sizeof(out->warning), "%s", msg.str().c_str());
    }
  }
  DebugTimer tail("explain tail");
  out->phi = dup_array(phi);
  const std::vector<uint32_t> ranked = rank_players(ctx, phi);
  tail.lap("ranking");
  const size_t keep = std::min<size_t>(o.top_k, ranked.size());
  std::vector<uint32_t> tp(ranked.begin(), ranked.begin() + keep);
  std::vector<double> tv(keep);
  for (size_t i = 0; i < keep; ++i) tv[i] = phi[tp[i]];
  out->num_top = uint32_t(keep);
  out->top_player = dup_array(tp);
  out->top_phi = dup_array(tv);
  if (o.fidelity) {
    const auto t_fid = Clock::now();
    std::vector<uint32_t> counts = o.top_counts ? std::vector<uint32_t>(o.top_counts, o.top_counts + o.num_top_counts)
                                                : std::vector<uint32_t>{5, 10, 20};
    std::vector<double> sp = o.sparsities ? std::vector<double>(o.sparsities, o.sparsities + o.num_sparsities)
                                          : std::vector<double>{0.1, 0.3, 0.5, 0.7, 0.9};
    FidelityOut f = fidelity(ctx, sg, m, out->predicted_class, phi, counts, sp, seed, o.baseline_trials, &ranked);
    out->has_fidelity = 1;
    out->num_counts = uint32_t(f.counts.size());
    out->fid_counts = dup_array(f.counts);
    out->fid_plus = dup_array(f.plus);
    out->fid_plus_random = dup_array(f.plus_random);
    out->num_sparsities = uint32_t(f.sparsities.size());
    out->fid_sparsities = dup_array(f.sparsities);
    out->fid_minus = dup_array(f.minus);
    out->fid_minus_random = dup_array(f.minus_random);
    out->fidelity_ms = ms_since(t_fid);
  }
  out->total_ms = ms_since(t_start);
  DebugTimer("explain").lap("end");
}

}  // namespace sfb

// ================================================================ C-ABI
using namespace sfb;

struct sf_ctx {
  Ctx c;
  // explain_nodes on one device: extra contexts (own stream and buffers)
  // run other targets concurrently from worker threads (sf_ctx_set_workers)
  int workers = 1;
  std::vector<std::unique_ptr<sf_ctx>> helpers;
};
struct sf_graph {
  Graph g;
};
struct sf_model {
  Model m;
};
struct sf_subgraph {
  Subgraph s;
};
// device-resident MaskBlock (sampler.hpp:55-78): kept-set rows only
struct sf_dmasks {
  int device = 0;
  SizePlan plan;
  int rank = 0, world = 1;
  uint64_t pairs = 0;  // local pairs
  uint32_t W = 1;
  DevBuf<uint64_t> rows;
};

namespace {
thread_local std::string g_last_error;

template <typename F>
int guard(F&& f) {
  try {
    f();
    return SF_OK;
  } catch (const DataError& e) {
    g_last_error = e.what();
    return SF_ERR_DATA;
  } catch (const NumericalError& e) {
    g_last_error = e.what();
    return SF_ERR_NUMERICAL;
  } catch (const ProtocolError& e) {
    g_last_error = e.what();
    return SF_ERR_PROTOCOL;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return SF_ERR_INTERNAL;
  } catch (...) {
    g_last_error = "unknown error";
    return SF_ERR_INTERNAL;
  }
}

void need(const void* p, const char* what) {
  if (!p) throw DataError(std::string("null ") + what);
}

SizePlan plan_from_arrays(uint32_t n, const uint32_t* sizes, const uint64_t* pairs,
                          const uint64_t* first, uint64_t nclasses, int exhaustive) {
  SizePlan p;
  p.n = n;
  p.exhaustive = exhaustive != 0;
  for (uint64_t i = 0; i < nclasses; ++i) {
    if (sizes[i] == 0 || 2 * uint64_t(sizes[i]) > n)
      throw DataError("size class " + std::to_string(sizes[i]) + " invalid for " +
                      std::to_string(n) + " players");
    if (i > 0 && first[i] != first[i - 1] + pairs[i - 1])
      throw DataError("size classes must be contiguous in the pair index");
    p.classes.push_back({sizes[i], pairs[i], first[i]});
  }
  return p;
}
}  // namespace

extern "C" {

const char* sf_last_error(void) { return g_last_error.c_str(); }
const char* sf_version(void) { return "shapflow_b200 0.1 (sm_100a)"; }

int sf_ctx_create(int device, sf_ctx** out) {
  return guard([&] {
    need(out, "output");
    int count = 0;
    SF_CUDA(cudaGetDeviceCount(&count));
    if (device < 0 || device >= count)
      throw DataError("CUDA device " + std::to_string(device) + " not present (" +
                      std::to_string(count) + " visible)");
    auto* c = new sf_ctx;
    c->c.device = device;
    try {
      // Host wait policy for stream syncs (the CGLS loop syncs twice per
      // iteration): spin by default (blocking/yield waits measured +1 to
      // +25 ms per C2 solve); SF_SCHED=auto|yield|blocking overrides. Only
      // takes effect if the device's context is not active yet.
      {
        const char* sch = std::getenv("SF_SCHED");
        const std::string p = sch ? sch : "spin";
        if (p != "auto") {
          const unsigned f = p == "yield"      ? cudaDeviceScheduleYield
                             : p == "blocking" ? cudaDeviceScheduleBlockingSync
                                               : cudaDeviceScheduleSpin;
          cudaSetDevice(device);
          if (cudaSetDeviceFlags(f) != cudaSuccess) cudaGetLastError();
        }
      }
      SF_CUDA(cudaSetDevice(device));
      SF_CUDA(cudaStreamCreateWithFlags(&c->c.stream, cudaStreamNonBlocking));
    } catch (...) {
      delete c;
      throw;
    }
    *out = c;
  });
}

int sf_ctx_destroy(sf_ctx* ctx) {
  return guard([&] {
    if (ctx) {
      cudaSetDevice(ctx->c.device);
      delete ctx;
    }
  });
}

int sf_ctx_rank(const sf_ctx* ctx) { return ctx ? ctx->c.rank : -1; }
int sf_ctx_world(const sf_ctx* ctx) { return ctx ? ctx->c.world : -1; }
uint64_t sf_ctx_launches(const sf_ctx* ctx) { return ctx ? ctx->c.launches : 0; }

int sf_ctx_set_fused_kernel(sf_ctx* ctx, int kind) {
  return guard([&] {
    need(ctx, "context");
    if (kind < 0 || kind > 3)
      throw DataError("fused kernel kind must be 0 (auto), 1 (simt), 2 (tc) or 3 (tc16)");
    ctx->c.fused_kind = kind;
  });
}

int sf_ctx_fused_plan(const sf_ctx* ctx, uint64_t* entries, uint64_t* padded_entries,
                      uint32_t* items, uint32_t* width) {
  return guard([&] {
    need(ctx, "context");
    const Engine& e = ctx->c.engine;
    if (entries) *entries = e.fused ? e.entries : 0;
    if (padded_entries) *padded_entries = e.tc ? e.tc_entries : 0;
    if (items) *items = e.fused ? (e.tc ? e.tc_items : e.items) : 0;
    if (width) *width = e.fused ? uint32_t(e.dims[1]) : 0;
  });
}

int sf_ctx_fused_kernel_used(const sf_ctx* ctx) {
  if (!ctx) return -1;
  const Engine& e = ctx->c.engine;
  return e.fused ? (e.tc16 ? 3 : e.tc ? 2 : 1) : 0;
}

int sf_ctx_io_bytes(const sf_ctx* ctx, uint64_t* h2d, uint64_t* d2h) {
  return guard([&] {
    need(ctx, "context");
    if (h2d) *h2d = ctx->c.h2d_bytes;
    if (d2h) *d2h = ctx->c.d2h_bytes;
  });
}

int sf_ctx_event_record(sf_ctx* ctx, int slot) {
  return guard([&] {
    need(ctx, "context");
    if (slot < 0 || slot >= 8) throw DataError("event slot out of range");
    SF_CUDA(cudaSetDevice(ctx->c.device));
    if (!ctx->c.events[slot]) SF_CUDA(cudaEventCreate(&ctx->c.events[slot]));
    SF_CUDA(cudaEventRecord(ctx->c.events[slot], ctx->c.stream));
  });
}

int sf_ctx_event_elapsed(sf_ctx* ctx, int a, int b, float* ms) {
  return guard([&] {
    need(ctx, "context");
    need(ms, "output");
    if (a < 0 || a >= 8 || b < 0 || b >= 8 || !ctx->c.events[a] || !ctx->c.events[b])
      throw DataError("event slot not recorded");
    SF_CUDA(cudaEventSynchronize(ctx->c.events[b]));
    SF_CUDA(cudaEventElapsedTime(ms, ctx->c.events[a], ctx->c.events[b]));
  });
}

int sf_ctx_synchronize(sf_ctx* ctx) {
  return guard([&] {
    need(ctx, "context");
    SF_CUDA(cudaStreamSynchronize(ctx->c.stream));
  });
}

int sf_ctx_keep_stages(sf_ctx* ctx, int enable) {
  return guard([&] {
    need(ctx, "context");
    ctx->c.keep_stages = enable != 0;
    if (!enable) std::vector<float>().swap(ctx->c.kept_preds);
  });
}

int sf_ctx_stage_predictions(const sf_ctx* ctx, float* out, uint64_t cap, uint64_t* rows) {
  return guard([&] {
    need(ctx, "context");
    const auto& k = ctx->c.kept_preds;
    if (rows) *rows = k.size();
    if (out) {
      if (cap < k.size()) throw DataError("prediction buffer too small");
      std::memcpy(out, k.data(), k.size() * 4);
    }
  });
}

int sf_ctx_time_dominant(sf_ctx* ctx, int enable) {
  return guard([&] {
    need(ctx, "context");
    SF_CUDA(cudaStreamSynchronize(ctx->c.stream));
    ctx->c.time_dominant = enable != 0;
    ctx->c.dom_used = 0;
    ctx->c.dom_pairs = 0;
  });
}

int sf_ctx_dominant_stats(sf_ctx* ctx, double* total_ms, uint64_t* launches, uint64_t* pairs) {
  return guard([&] {
    need(ctx, "context");
    SF_CUDA(cudaStreamSynchronize(ctx->c.stream));
    double tot = 0.0;
    for (size_t i = 0; i < ctx->c.dom_used; ++i) {
      float ms = 0.f;
      SF_CUDA(cudaEventElapsedTime(&ms, ctx->c.dom_events[i].first, ctx->c.dom_events[i].second));
      tot += ms;
    }
    if (total_ms) *total_ms = tot;
    if (launches) *launches = ctx->c.dom_used;
    if (pairs) *pairs = ctx->c.dom_pairs;
  });
}

int sf_spmm_bytes_per_pair(const sf_model* m, const sf_subgraph* sgp, double* bytes, double* flops) {
  return guard([&] {
    need(m, "model");
    need(sgp, "subgraph");
    const Subgraph& sg = sgp->s;
    const int L = m->m.depth();
    const auto ball = sg.ball_sizes(L);
    // layer 0 produces rows R = B_{L-1} (the target row alone when L == 1)
    const uint64_t R = ball[L - 1];
    const double d = double(m->m.layers.front().out);
    uint64_t deg = 0;
    for (uint64_t u = 0; u < R; ++u) deg += sg.row_ptr[u + 1] - sg.row_ptr[u];
    const double W = double((sg.num_players() + 63) / 64);
    if (bytes) *bytes = (double(deg) + 2.0 * R) * d * 4.0 + 2.0 * R * d * 4.0 + 2.0 * W * 8.0;
    if (flops) *flops = 2.0 * (double(deg) + 2.0 * R) * d;
  });
}

int sf_nccl_unique_id(void* out) {
  return guard([&] {
    need(out, "output");
    nccl_unique_id(out);
  });
}

int sf_ctx_join_nccl(sf_ctx* ctx, const void* id, int rank, int world) {
  return guard([&] {
    need(ctx, "context");
    if (world > 1) need(id, "unique id");
    SF_CUDA(cudaSetDevice(ctx->c.device));
    ctx->c.host_comm = HostComm{};
    nccl_join(ctx->c, id, rank, world);
  });
}

int sf_ctx_set_host_comm(sf_ctx* ctx, int rank, int world, void* user,
                         int (*all_reduce)(void*, double*, uint64_t), int (*barrier)(void*)) {
  return guard([&] {
    need(ctx, "context");
    if (world < 1 || rank < 0 || rank >= world)
      throw DataError("invalid worker rank " + std::to_string(rank) + " of " + std::to_string(world));
    if ((all_reduce == nullptr) != (barrier == nullptr))
      throw DataError("host communicator needs both all_reduce and barrier");
    if (world > 1 && !all_reduce) throw DataError("host communicator needs all_reduce and barrier");
    comm_drop_nccl(ctx->c);
    ctx->c.rank = rank;
    ctx->c.world = world;
    ctx->c.host_comm = HostComm{user, all_reduce, barrier};
  });
}

int sf_ctx_allreduce_host(sf_ctx* ctx, double* buf, uint64_t count) {
  return guard([&] {
    need(ctx, "context");
    if (count) need(buf, "buffer");
    SF_CUDA(cudaSetDevice(ctx->c.device));
    DevBuf<double>& d = ctx->c.barrier_buf;
    d.reserve(std::max<uint64_t>(count, 1));
    SF_CUDA(cudaMemcpyAsync(d.p, buf, count * 8, cudaMemcpyHostToDevice, ctx->c.stream));
    comm_allreduce_sum(ctx->c, d.p, count);
    SF_CUDA(cudaMemcpyAsync(buf, d.p, count * 8, cudaMemcpyDeviceToHost, ctx->c.stream));
    comm_sync(ctx->c);
  });
}

int sf_ctx_device_memory(const sf_ctx* ctx, uint64_t* used, uint64_t* total) {
  return guard([&] {
    need(ctx, "context");
    SF_CUDA(cudaSetDevice(ctx->c.device));
    size_t f = 0, t = 0;
    SF_CUDA(cudaMemGetInfo(&f, &t));
    if (used) *used = t - f;
    if (total) *total = t;
  });
}

int sf_ctx_set_workers(sf_ctx* ctx, int workers) {
  return guard([&] {
    need(ctx, "context");
    if (workers < 1 || workers > 16) throw DataError("workers must be in [1, 16]");
    ctx->workers = workers;
  });
}

int sf_ctx_set_comm_timeout(sf_ctx* ctx, int timeout_ms) {
  return guard([&] {
    need(ctx, "context");
    if (timeout_ms <= 0) throw DataError("communicator timeout must be positive");
    ctx->c.comm_timeout_ms = timeout_ms;
  });
}

int sf_ctx_stats(const sf_ctx* ctx, uint64_t* s, uint64_t* v, uint64_t* b, uint64_t* d) {
  return guard([&] {
    need(ctx, "context");
    if (s) *s = ctx->c.stats.scalar_allreduce;
    if (v) *v = ctx->c.stats.vector_allreduce;
    if (b) *b = ctx->c.stats.barriers;
    if (d) *d = ctx->c.stats.doubles_reduced;
  });
}

int sf_ctx_barrier(sf_ctx* ctx) {
  return guard([&] {
    need(ctx, "context");
    SF_CUDA(cudaSetDevice(ctx->c.device));
    comm_barrier(ctx->c);
  });
}

uint64_t sf_node_sampling_seed(uint64_t seed, uint32_t node) {
  return seed ^ (0x9E3779B97F4A7C15ull * (uint64_t(node) + 1));  // explain.cpp:37-40
}

uint64_t sf_auto_samples(uint64_t n) { return n < 5000 ? 60000 : 600000; }

uint64_t sf_binomial_or_max(uint32_t n, uint32_t s) { return binomial_or_max(n, s); }

int sf_kernel_weight(uint32_t n, uint32_t s, double* out) {
  return guard([&] {  // sampler.cpp:79-91
    need(out, "output");
    if (n < 2 || s == 0 || s >= n)
      throw DataError("coalition weight undefined for size " + std::to_string(s) + " of " +
                      std::to_string(n) + " players");
    if (n <= 60) {
      const double c = double(binomial_or_max(n, s));
      *out = (n - 1.0) / (c * s * (n - s));
      return;
    }
    const double log_c = std::lgamma(n + 1.0) - std::lgamma(s + 1.0) - std::lgamma(n - s + 1.0);
    *out = std::exp(std::log(n - 1.0) - log_c - std::log(double(s)) - std::log(double(n - s)));
  });
}

int sf_philox_u64(sf_ctx* ctx, uint64_t seed, uint64_t stream, uint64_t count, uint64_t* out) {
  return guard([&] {
    need(ctx, "context");
    need(out, "output");
    SF_CUDA(cudaSetDevice(ctx->c.device));
    DevBuf<uint64_t> d;
    d.reserve(std::max<uint64_t>(count, 1));
    launch_philox_stream(ctx->c, seed, stream, count, d.p);
    SF_CUDA(cudaMemcpyAsync(out, d.p, count * 8, cudaMemcpyDeviceToHost, ctx->c.stream));
    SF_CUDA(cudaStreamSynchronize(ctx->c.stream));
  });
}

int sf_plan_sizes(uint32_t n, uint64_t k, int allow, uint32_t* sizes, uint64_t* pairs,
                  uint64_t* first, uint64_t cap, uint64_t* nclasses, int* exhaustive,
                  uint64_t* requested) {
  return guard([&] {
    const SizePlan p = plan_sizes(n, k, allow != 0);
    if (nclasses) *nclasses = p.classes.size();
    if (exhaustive) *exhaustive = p.exhaustive ? 1 : 0;
    if (requested) *requested = p.requested;
    if (sizes && pairs && first) {
      if (p.classes.size() > cap) throw DataError("plan arrays too small");
      for (size_t i = 0; i < p.classes.size(); ++i) {
        sizes[i] = p.classes[i].size;
        pairs[i] = p.classes[i].pairs;
        first[i] = p.classes[i].first_pair;
      }
    }
  });
}

int sf_generate_masks(sf_ctx* ctx, uint32_t n, const uint32_t* sizes, const uint64_t* pairs,
                      const uint64_t* first, uint64_t nclasses, int exhaustive, uint64_t seed,
                      int rank, int world, uint64_t* out, uint64_t cap_words, uint64_t* rows,
                      uint64_t* rows_of_size) {
  return guard([&] {
    need(ctx, "context");
    if (world < 1 || rank < 0 || rank >= world)
      throw DataError("invalid worker rank " + std::to_string(rank) + " of " + std::to_string(world));
    const SizePlan p = plan_from_arrays(n, sizes, pairs, first, nclasses, exhaustive);
    const uint64_t lp = local_pair_count(p.total_pairs(), rank, world);
    const uint64_t W = (n + 63) / 64;
    if (rows) *rows = 2 * lp;
    if (rows_of_size) {
      const auto c = global_rows_of_size(p);
      std::memcpy(rows_of_size, c.data(), c.size() * 8);
    }
    if (!out) return;
    if (2 * lp * W > cap_words) throw DataError("mask output buffer too small");
    SF_CUDA(cudaSetDevice(ctx->c.device));
    ctx->c.masks.reserve(std::max<uint64_t>(2 * lp * W, 1));
    launch_generate_masks(ctx->c, p, seed, rank, world, ctx->c.masks.p);
    SF_CUDA(cudaMemcpyAsync(out, ctx->c.masks.p, 2 * lp * W * 8, cudaMemcpyDeviceToHost, ctx->c.stream));
    SF_CUDA(cudaStreamSynchronize(ctx->c.stream));
  });
}

int sf_masks_device(sf_ctx* ctx, uint32_t n, const uint32_t* sizes, const uint64_t* pairs,
                    const uint64_t* first, uint64_t nclasses, int exhaustive, uint64_t seed, int rank,
                    int world, sf_dmasks** out) {
  return guard([&] {
    need(ctx, "context");
    need(out, "output");
    if (world < 1 || rank < 0 || rank >= world)
      throw DataError("invalid worker rank " + std::to_string(rank) + " of " + std::to_string(world));
    SF_CUDA(cudaSetDevice(ctx->c.device));
    auto d = std::make_unique<sf_dmasks>();
    d->device = ctx->c.device;
    d->plan = plan_from_arrays(n, sizes, pairs, first, nclasses, exhaustive);
    d->rank = rank;
    d->world = world;
    d->pairs = local_pair_count(d->plan.total_pairs(), rank, world);
    d->W = std::max<uint32_t>(1, (n + 63) / 64);
    d->rows.reserve(std::max<uint64_t>(d->pairs * d->W, 1));
    launch_generate_masks(ctx->c, d->plan, seed, rank, world, d->rows.p, /*kept_only=*/true);
    SF_CUDA(cudaStreamSynchronize(ctx->c.stream));
    *out = d.release();
  });
}

int sf_dmasks_info(const sf_dmasks* m, uint64_t* rows, uint32_t* num_players, uint64_t* rows_of_size) {
  return guard([&] {
    need(m, "masks");
    if (rows) *rows = 2 * m->pairs;
    if (num_players) *num_players = m->plan.n;
    if (rows_of_size) {
      const auto c = global_rows_of_size(m->plan);
      std::memcpy(rows_of_size, c.data(), c.size() * 8);
    }
  });
}

int sf_dmasks_download(sf_ctx* ctx, const sf_dmasks* m, uint64_t* out, uint64_t cap_words) {
  return guard([&] {
    need(ctx, "context");
    need(m, "masks");
    const uint64_t W = m->W, total = 2 * m->pairs * W;
    if (total == 0) return;
    need(out, "output");
    if (cap_words < total) throw DataError("mask output buffer too small");
    SF_CUDA(cudaSetDevice(m->device));
    std::vector<uint64_t> kept(m->pairs * W);
    SF_CUDA(cudaMemcpyAsync(kept.data(), m->rows.p, kept.size() * 8, cudaMemcpyDeviceToHost, ctx->c.stream));
    SF_CUDA(cudaStreamSynchronize(ctx->c.stream));
    ctx->c.d2h_bytes += kept.size() * 8;
    const uint32_t n = m->plan.n;
    const uint64_t tail = (n % 64) ? ((uint64_t{1} << (n % 64)) - 1) : ~uint64_t{0};
    for (uint64_t j = 0; j < m->pairs; ++j) {  // rows 2j (kept), 2j+1 (complement, sampler.cpp:205-207)
      std::memcpy(out + 2 * j * W, kept.data() + j * W, W * 8);
      for (uint64_t w = 0; w < W; ++w) out[(2 * j + 1) * W + w] = (w + 1 == W) ? (~kept[j * W + w] & tail) : ~kept[j * W + w];
      if (n == 0) out[(2 * j + 1) * W] = 0;
    }
  });
}

int sf_dmasks_free(sf_dmasks* m) {
  delete m;
  return SF_OK;
}

int sf_predict_dmasks(sf_ctx* ctx, const sf_model* m, const sf_subgraph* sg, const sf_dmasks* masks,
                      uint32_t class_index, uint64_t batch_size, float* out) {
  return guard([&] {  // gcn.cpp:259-270 on device-resident rows
    need(ctx, "context");
    need(m, "model");
    need(sg, "subgraph");
    need(masks, "masks");
    if (batch_size == 0) throw DataError("batch_size must be positive");
    if (class_index >= m->m.layers.back().out) throw DataError("class index out of range");
    if (masks->device != ctx->c.device) throw DataError("masks live on another device");
    if (masks->plan.n != sg->s.num_players()) throw DataError("masks do not match the subgraph's player count");
    const uint64_t rows = 2 * masks->pairs;
    if (rows == 0) return;
    need(out, "output");
    Ctx& c = ctx->c;
    SF_CUDA(cudaSetDevice(c.device));
    engine_prepare(c, sg->s, m->m);
    c.preds.reserve(rows);
    engine_predict(c, masks->rows.p, rows, class_index, c.preds.p, nullptr, nullptr, /*kept_only=*/true);
    SF_CUDA(cudaMemcpyAsync(out, c.preds.p, rows * 4, cudaMemcpyDeviceToHost, c.stream));
    SF_CUDA(cudaStreamSynchronize(c.stream));
    c.d2h_bytes += rows * 4;
  });
}

int sf_solve_dmasks(sf_ctx* ctx, const sf_dmasks* masks, const float* values, double base, double full,
                    double constraint_scale, double tol, uint64_t max_iter, int mode, double* phi,
                    uint64_t* iterations, double* rel, int* converged) {
  return guard([&] {  // assemble_problem (solver.cpp:95-156) + solve_cgls (158-362) on device rows
    need(ctx, "context");
    need(masks, "masks");
    const uint32_t n = masks->plan.n;
    if (iterations) *iterations = 0;
    if (rel) *rel = 0.0;
    if (converged) *converged = 1;
    if (n == 0) return;
    need(phi, "output");
    if (masks->rank != ctx->c.rank || masks->world != ctx->c.world)
      throw DataError("system slice does not match the communicator layout");
    if (mode < 0 || mode > 2) throw DataError("solver mode must be 0, 1 or 2");
    const uint64_t rows = 2 * masks->pairs;
    if (rows) need(values, "values");
    Ctx& c = ctx->c;
    SF_CUDA(cudaSetDevice(c.device));
    const std::vector<double> wsize = weight_of_size(n, global_rows_of_size(masks->plan));
    c.wsize_dev.upload(wsize.data(), wsize.size(), c.stream);
    c.preds.reserve(std::max<uint64_t>(rows, 1));
    if (rows) SF_CUDA(cudaMemcpyAsync(c.preds.p, values, rows * 4, cudaMemcpyHostToDevice, c.stream));
    c.sw_dev.reserve(std::max<uint64_t>(rows, 1));
    c.tgt_dev.reserve(std::max<uint64_t>(rows, 1));
    c.pop_dev.reserve(std::max<uint64_t>(rows, 1));
    c.comp_dev.reserve(std::max<uint64_t>(rows / 2, 1));
    const int big = 0x7fffffff;
    c.bad_dev.upload(&big, 1, c.stream);
    c.h2d_bytes += wsize.size() * 8 + rows * 4 + 4;
    launch_assemble_pairs(c, masks->rows.p, rows, masks->W, n, c.wsize_dev.p, c.preds.p, base, c.sw_dev.p, c.tgt_dev.p,
                          c.bad_dev.p, c.pop_dev.p, c.comp_dev.p, /*kept_only=*/true);
    int bad = big;
    SF_CUDA(cudaMemcpyAsync(&bad, c.bad_dev.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    SF_CUDA(cudaStreamSynchronize(c.stream));
    if (bad != big) throw DataError("coalition row " + std::to_string(bad) + " keeps all or no players");
    CglsInput in;
    in.n = n;
    in.rows = rows;
    in.W = masks->W;
    in.dev_rows = masks->rows.p;
    in.dev_sw = c.sw_dev.p;
    in.dev_targets = c.tgt_dev.p;
    in.constraint_target = full - base;
    in.constraint_weight = constraint_scale;
    in.global_pair_count = masks->plan.total_pairs();
    in.dev_pop = c.pop_dev.p;
    in.dev_is_comp = c.comp_dev.p;
    in.kept_only = true;
    in.fixed_order = mode == 2;
    const CglsResult r = cgls_solve(c, in, tol, max_iter, mode == 1 ? 1 : 0, false);
    std::memcpy(phi, r.phi.data(), uint64_t(n) * 8);
    if (iterations) *iterations = r.iterations;
    if (rel) *rel = r.relative_residual;
    if (converged) *converged = r.converged ? 1 : 0;
  });
}

int sf_graph_build(uint32_t num_nodes, const uint64_t* edges, uint64_t num_edges,
                   const float* features, uint64_t dim, const uint32_t* labels, sf_graph** out) {
  return guard([&] {
    need(out, "output");
    if (num_edges) need(edges, "edges");
    if (uint64_t(num_nodes) * dim != 0) need(features, "features");
    std::vector<float> f(features, features + uint64_t(num_nodes) * dim);
    std::vector<uint32_t> lab;
    if (labels) lab.assign(labels, labels + num_nodes);
    auto* g = new sf_graph{build_graph(num_nodes, edges, num_edges, std::move(f), dim, std::move(lab))};
    *out = g;
  });
}

int sf_graph_from_csr(uint32_t num_nodes, const uint64_t* row_ptr, const uint32_t* col, const float* features,
                      uint64_t dim, const uint32_t* labels, sf_graph** out) {
  return guard([&] {
    need(out, "output");
    need(row_ptr, "row_ptr");
    const uint64_t nnz = row_ptr[num_nodes];
    if (nnz) need(col, "col");
    if (uint64_t(num_nodes) * dim != 0) need(features, "features");
    Graph g;
    g.num_nodes = num_nodes;
    g.feature_dim = dim;
    g.row_ptr.assign(row_ptr, row_ptr + num_nodes + 1);
    g.col.assign(col, col + nnz);
    for (uint32_t u = 0; u < num_nodes; ++u) {
      if (g.row_ptr[u] > g.row_ptr[u + 1]) throw DataError("row_ptr is not monotone");
      for (uint64_t i = g.row_ptr[u]; i < g.row_ptr[u + 1]; ++i) {
        if (g.col[i] >= num_nodes) throw DataError("edge endpoint out of range");
        if (i > g.row_ptr[u] && g.col[i] <= g.col[i - 1]) throw DataError("CSR rows must be sorted and unique");
      }
    }
    g.features.assign(features, features + uint64_t(num_nodes) * dim);
    g.labels.assign(num_nodes, 0xFFFFFFFFu);
    if (labels) g.labels.assign(labels, labels + num_nodes);
    *out = new sf_graph{std::move(g)};
  });
}

int sf_graph_load(const char* path, sf_graph** out) {
  return guard([&] {
    need(path, "path");
    need(out, "output");
    const std::string p(path);
    if (p.size() < 4 || p.substr(p.size() - 4) != ".sfg")
      throw DataError("only binary SFG1 graphs (.sfg) are supported: " + p);
    *out = new sf_graph{load_sfg(p)};
  });
}

int sf_graph_save(const sf_graph* g, const char* path) {
  return guard([&] {
    need(g, "graph");
    need(path, "path");
    save_sfg(g->g, path);
  });
}

int sf_graph_free(sf_graph* g) {
  delete g;
  return SF_OK;
}

int sf_graph_dims(const sf_graph* g, uint32_t* nodes, uint64_t* nnz, uint64_t* dim) {
  return guard([&] {
    need(g, "graph");
    if (nodes) *nodes = g->g.num_nodes;
    if (nnz) *nnz = g->g.col.size();
    if (dim) *dim = g->g.feature_dim;
  });
}

int sf_graph_csr(const sf_graph* g, uint64_t* row_ptr, uint32_t* col) {
  return guard([&] {
    need(g, "graph");
    if (row_ptr) std::memcpy(row_ptr, g->g.row_ptr.data(), g->g.row_ptr.size() * 8);
    if (col) std::memcpy(col, g->g.col.data(), g->g.col.size() * 4);
  });
}

int sf_model_create(int L, const uint64_t* dims, const float* weights, const float* biases,
                    sf_model** out) {
  return guard([&] {
    need(out, "output");
    need(dims, "dims");
    if (L < 1) throw DataError("model has no layers");
    Model m;
    for (int l = 0; l < L; ++l) {
      Layer lay;
      lay.in = dims[l];
      lay.out = dims[l + 1];
      lay.weight.assign(weights, weights + lay.in * lay.out);
      lay.bias.assign(biases, biases + lay.out);
      weights += lay.in * lay.out;
      biases += lay.out;
      m.layers.push_back(std::move(lay));
    }
    validate_model(m);
    *out = new sf_model{std::move(m)};
  });
}

int sf_model_random(uint64_t input_dim, const uint64_t* hidden, int nh, uint32_t classes,
                    uint64_t seed, sf_model** out) {
  return guard([&] {
    need(out, "output");
    *out = new sf_model{random_model(input_dim, hidden, nh, classes, seed)};
  });
}

int sf_model_free(sf_model* m) {
  delete m;
  return SF_OK;
}

int sf_model_dims(const sf_model* m, int* L, uint64_t* dims) {
  return guard([&] {
    need(m, "model");
    if (L) *L = m->m.depth();
    if (dims) {
      dims[0] = m->m.layers.front().in;
      for (int l = 0; l < m->m.depth(); ++l) dims[l + 1] = m->m.layers[l].out;
    }
  });
}

int sf_model_layer(const sf_model* m, int l, float* w, float* b) {
  return guard([&] {
    need(m, "model");
    if (l < 0 || l >= m->m.depth()) throw DataError("layer index out of range");
    const Layer& lay = m->m.layers[l];
    if (w) std::memcpy(w, lay.weight.data(), lay.weight.size() * 4);
    if (b) std::memcpy(b, lay.bias.data(), lay.bias.size() * 4);
  });
}

int sf_extract(const sf_graph* g, uint32_t target, int hops, sf_subgraph** out) {
  return guard([&] {
    need(g, "graph");
    need(out, "output");
    *out = new sf_subgraph{extract(g->g, target, hops)};
  });
}

int sf_subgraph_create(uint32_t target_global, uint32_t V, uint64_t n, const uint64_t* row_ptr, const uint32_t* col,
                       const uint32_t* edge_player, const uint32_t* players_uv, const uint32_t* local_to_global,
                       const float* features, uint64_t dim, sf_subgraph** out) {
  return guard([&] {
    need(out, "output");
    need(row_ptr, "row_ptr");
    const uint64_t nnz = row_ptr[V];
    if (nnz) {
      need(col, "col");
      need(edge_player, "edge_player");
    }
    if (n) need(players_uv, "players");
    if (V) need(local_to_global, "local_to_global");
    if (uint64_t(V) * dim != 0) need(features, "features");
    Subgraph sg;
    sg.target_global = target_global;
    sg.feature_dim = dim;
    sg.local_to_global.assign(local_to_global, local_to_global + V);
    sg.players.resize(n);
    for (uint64_t e = 0; e < n; ++e) {
      sg.players[e] = {players_uv[2 * e], players_uv[2 * e + 1]};
      if (sg.players[e].first >= V || sg.players[e].second >= V) throw DataError("player endpoint out of range");
    }
    sg.row_ptr.assign(row_ptr, row_ptr + V + 1);
    sg.col.assign(col, col + nnz);
    sg.edge_player.assign(edge_player, edge_player + nnz);
    for (uint64_t i = 0; i < nnz; ++i)
      if (sg.col[i] >= V || sg.edge_player[i] >= n) throw DataError("subgraph CSR entry out of range");
    sg.features.assign(features, features + uint64_t(V) * dim);
    *out = new sf_subgraph{std::move(sg)};
  });
}

int sf_extract_device(sf_ctx* ctx, const sf_graph* g, uint32_t target, int hops, sf_subgraph** out) {
  return guard([&] {
    need(ctx, "context");
    need(g, "graph");
    need(out, "output");
    SF_CUDA(cudaSetDevice(ctx->c.device));
    Subgraph sg = extract_device(ctx->c, g->g, target, hops);
    sg.source = nullptr;  // a standalone subgraph carries its feature slice
    const uint64_t d = g->g.feature_dim;
    sg.features.resize(uint64_t(sg.num_nodes()) * d);
    for (uint32_t lu = 0; lu < sg.num_nodes(); ++lu)
      std::memcpy(sg.features.data() + uint64_t(lu) * d, g->g.features.data() + uint64_t(sg.local_to_global[lu]) * d,
                  d * 4);
    *out = new sf_subgraph{std::move(sg)};
  });
}

int sf_subgraph_free(sf_subgraph* sg) {
  delete sg;
  return SF_OK;
}

int sf_subgraph_dims(const sf_subgraph* sg, uint32_t* V, uint64_t* n, uint64_t* nnz, uint64_t* dim) {
  return guard([&] {
    need(sg, "subgraph");
    if (V) *V = sg->s.num_nodes();
    if (n) *n = sg->s.num_players();
    if (nnz) *nnz = sg->s.col.size();
    if (dim) *dim = sg->s.feature_dim;
  });
}

int sf_subgraph_copy(const sf_subgraph* sgp, uint64_t* row_ptr, uint32_t* col, uint32_t* ep,
                     uint32_t* players_uv, uint32_t* l2g, float* features) {
  return guard([&] {
    need(sgp, "subgraph");
    const Subgraph& sg = sgp->s;
    if (row_ptr) std::memcpy(row_ptr, sg.row_ptr.data(), sg.row_ptr.size() * 8);
    if (col) std::memcpy(col, sg.col.data(), sg.col.size() * 4);
    if (ep) std::memcpy(ep, sg.edge_player.data(), sg.edge_player.size() * 4);
    if (players_uv)
      for (size_t e = 0; e < sg.players.size(); ++e) {
        players_uv[2 * e] = sg.players[e].first;
        players_uv[2 * e + 1] = sg.players[e].second;
      }
    if (l2g) std::memcpy(l2g, sg.local_to_global.data(), sg.local_to_global.size() * 4);
    if (features) std::memcpy(features, sg.features.data(), sg.features.size() * 4);
  });
}

int sf_subgraph_ball_sizes(const sf_subgraph* sg, int hops, uint64_t* sizes) {
  return guard([&] {
    need(sg, "subgraph");
    need(sizes, "output");
    const auto b = sg->s.ball_sizes(hops);
    std::memcpy(sizes, b.data(), b.size() * 8);
  });
}

int sf_predict_batched(sf_ctx* ctx, const sf_model* m, const sf_subgraph* sg, const uint64_t* bits,
                       uint64_t rows, uint64_t words, uint32_t cls, uint64_t batch_size, float* out) {
  return guard([&] {  // gcn.cpp:259-270 + validation 43-49
    need(ctx, "context");
    need(m, "model");
    need(sg, "subgraph");
    if (cls >= m->m.layers.back().out) throw DataError("class index out of range");
    if (m->m.layers.front().in != sg->s.feature_dim)
      throw DataError("model input dim " + std::to_string(m->m.layers.front().in) +
                      " does not match feature dim " + std::to_string(sg->s.feature_dim));
    if (batch_size == 0) throw DataError("batch_size must be positive");
    const uint32_t W = uint32_t((sg->s.num_players() + 63) / 64);
    if (rows > 0 && words < W) throw DataError("mask rows narrower than the player count");
    if (rows == 0) return;
    need(bits, "mask rows");
    need(out, "output");
    SF_CUDA(cudaSetDevice(ctx->c.device));
    const uint32_t Wd = std::max<uint32_t>(W, 1);
    if (W == 0) {
      // no players: every mask is the empty one
      std::vector<uint64_t> z(rows, 0);
      upload_rows(ctx->c, z.data(), rows, 1, 1);
    } else {
      upload_rows(ctx->c, bits, rows, words, Wd);
    }
    predict_rows(ctx->c, sg->s, m->m, ctx->c.masks.p, rows, cls, out, nullptr);
  });
}

int sf_predict_probs(sf_ctx* ctx, const sf_model* m, const sf_subgraph* sg, const uint64_t* mask,
                     uint64_t words, float* probs) {
  return guard([&] {  // gcn.cpp:239-248
    need(ctx, "context");
    need(m, "model");
    need(sg, "subgraph");
    need(probs, "output");
    const uint32_t W = uint32_t((sg->s.num_players() + 63) / 64);
    if (words < W) throw DataError("mask shorter than the player count");
    if (m->m.layers.front().in != sg->s.feature_dim)
      throw DataError("model input dim does not match feature dim");
    SF_CUDA(cudaSetDevice(ctx->c.device));
    if (W == 0) {
      uint64_t z = 0;
      upload_rows(ctx->c, &z, 1, 1, 1);
    } else {
      need(mask, "mask");
      upload_rows(ctx->c, mask, 1, words, W);
    }
    predict_rows(ctx->c, sg->s, m->m, ctx->c.masks.p, 1, 0, nullptr, probs);
  });
}

int sf_assemble_weights(uint32_t n, const uint64_t* bits, uint64_t rows, uint64_t words,
                        const uint64_t* rows_of_size, double* weights) {
  return guard([&] {  // solver.cpp:116-151 (weights part)
    need(weights, "output");
    std::vector<uint64_t> counts;
    if (rows_of_size) {
      counts.assign(rows_of_size, rows_of_size + n + 1);
    } else {
      counts.assign(size_t(n) + 1, 0);
      for (uint64_t i = 0; i < rows; ++i) {
        uint64_t c = 0;
        for (uint64_t w = 0; w < words; ++w) c += __builtin_popcountll(bits[i * words + w]);
        if (c <= n) ++counts[c];
      }
    }
    const auto ws = weight_of_size(n, counts);
    for (uint64_t i = 0; i < rows; ++i) {
      uint64_t c = 0;
      for (uint64_t w = 0; w < words; ++w) c += __builtin_popcountll(bits[i * words + w]);
      if (c == 0 || c >= n)
        throw DataError("coalition row " + std::to_string(i) + " keeps all or no players");
      weights[i] = ws[c];
    }
  });
}

static void solve_common(sf_ctx* ctx, uint32_t n, const uint64_t* bits, uint64_t rows,
                         uint64_t words, const double* weights, const double* targets,
                         DevBuf<double>& d_sw, DevBuf<double>& d_tgt, CglsInput& in, bool pairs = true) {
  need(ctx, "context");
  if (pairs && rows % 2) throw DataError("local rows must come in adjacent pairs");
  const uint32_t W = uint32_t((n + 63) / 64);
  if (rows && words < W) throw DataError("rows narrower than the player count");
  SF_CUDA(cudaSetDevice(ctx->c.device));
  std::vector<double> sw(rows);
  // non-finite weights/targets are passed through: like the reference they
  // surface as a non-finite step norm (NumericalError) inside the solve
  for (uint64_t i = 0; i < rows; ++i) sw[i] = std::sqrt(weights[i]);
  upload_rows(ctx->c, bits, rows, words, std::max<uint32_t>(W, 1));
  d_sw.upload(sw.data(), rows, ctx->c.stream);
  d_tgt.upload(targets, rows, ctx->c.stream);
  in.n = n;
  in.rows = rows;
  in.W = std::max<uint32_t>(W, 1);
  in.dev_rows = ctx->c.masks.p;
  in.dev_sw = d_sw.p;
  in.dev_targets = d_tgt.p;
}

static void solve_cgls_impl(sf_ctx* ctx, uint32_t n, const uint64_t* bits, uint64_t rows, uint64_t words,
                            const double* weights, const double* targets, double ct, double cw, double tol,
                            uint64_t max_iter, int mode, uint64_t global_pairs, double* phi, uint64_t* iterations,
                            double* rel, int* converged, double* trace, double* row_trace, uint64_t trace_cap) {
  // solver.cpp:158-362
  if (n == 0) {
    if (iterations) *iterations = 0;
    if (converged) *converged = 1;
    if (rel) *rel = 0.0;
    return;
  }
  need(phi, "output");
  DevBuf<double> d_sw, d_tgt;
  CglsInput in;
  solve_common(ctx, n, bits, rows, words, weights, targets, d_sw, d_tgt, in);
  in.constraint_target = ct;
  in.constraint_weight = cw;
  in.global_pair_count = global_pairs;
  if (mode < 0 || mode > 2) throw DataError("solver mode must be 0 (reference protocol), 1 (fused) or 2 (fixed order)");
  in.fixed_order = mode == 2;
  CglsResult r = cgls_solve(ctx->c, in, tol, max_iter, mode == 2 ? 0 : mode, trace || row_trace);
  std::memcpy(phi, r.phi.data(), uint64_t(n) * 8);
  if (iterations) *iterations = r.iterations;
  if (rel) *rel = r.relative_residual;
  if (converged) *converged = r.converged ? 1 : 0;
  for (uint64_t i = 0; i < trace_cap; ++i) {
    if (trace && i < r.trace.size()) trace[i] = r.trace[i];
    if (row_trace && i < r.row_residual_trace.size()) row_trace[i] = r.row_residual_trace[i];
  }
}

int sf_solve_cgls(sf_ctx* ctx, uint32_t n, const uint64_t* bits, uint64_t rows, uint64_t words,
                  const double* weights, const double* targets, double ct, double cw, double tol,
                  uint64_t max_iter, int mode, double* phi, uint64_t* iterations, double* rel,
                  int* converged, double* trace, double* row_trace, uint64_t trace_cap) {
  return guard([&] {
    solve_cgls_impl(ctx, n, bits, rows, words, weights, targets, ct, cw, tol, max_iter, mode, rows / 2, phi,
                    iterations, rel, converged, trace, row_trace, trace_cap);
  });
}

int sf_solve_cgls_ex(sf_ctx* ctx, uint32_t n, const uint64_t* bits, uint64_t rows, uint64_t words,
                     const double* weights, const double* targets, double ct, double cw, double tol,
                     uint64_t max_iter, int mode, uint64_t global_pair_count, double* phi, uint64_t* iterations,
                     double* rel, int* converged, double* trace, double* row_trace, uint64_t trace_cap) {
  return guard([&] {
    solve_cgls_impl(ctx, n, bits, rows, words, weights, targets, ct, cw, tol, max_iter, mode, global_pair_count,
                    phi, iterations, rel, converged, trace, row_trace, trace_cap);
  });
}

int sf_solve_direct(sf_ctx* ctx, uint32_t n, const uint64_t* bits, uint64_t rows, uint64_t words,
                    const double* weights, const double* targets, double ct, double cw,
                    double* phi) {
  return guard([&] {  // solver.cpp:364-428
    if (ctx && ctx->c.world != 1)
      throw DataError("direct solve needs the full system on a single worker");
    if (n > 20000) throw DataError("direct solve limited to 20000 players, got " + std::to_string(n));
    if (n == 0) return;
    need(phi, "output");
    if (rows) {
      need(bits, "rows");
      need(weights, "weights");
      need(targets, "targets");
    }
    // runs of equal weight; rows in many short runs are first ordered by
    // weight (G and rhs are sums over rows, so row order is free)
    auto count_runs = [&](const double* w) {
      uint64_t c = 0;
      for (uint64_t i = 0; i < rows; ++i) c += (i == 0 || w[i] != w[i - 1]);
      return c;
    };
    std::vector<uint64_t> pb;
    std::vector<double> pw, pt;
    const uint64_t* ub = bits;
    const double *uw = weights, *ut = targets;
    if (count_runs(weights) > std::max<uint64_t>(64, rows / 16)) {
      std::vector<uint64_t> order(rows);
      for (uint64_t i = 0; i < rows; ++i) order[i] = i;
      std::stable_sort(order.begin(), order.end(), [&](uint64_t a, uint64_t b) { return weights[a] < weights[b]; });
      pb.resize(rows * words);
      pw.resize(rows);
      pt.resize(rows);
      for (uint64_t i = 0; i < rows; ++i) {
        std::memcpy(pb.data() + i * words, bits + order[i] * words, words * 8);
        pw[i] = weights[order[i]];
        pt[i] = targets[order[i]];
      }
      ub = pb.data();
      uw = pw.data();
      ut = pt.data();
    }
    std::vector<GramRun> runs;
    for (uint64_t i = 0; i < rows; ++i) {
      if (i == 0 || uw[i] != uw[i - 1]) runs.push_back(GramRun{i, i, uw[i]});
      runs.back().end = i + 1;
    }
    DevBuf<double> d_sw, d_tgt;
    CglsInput in;
    solve_common(ctx, n, ub, rows, words, uw, ut, d_sw, d_tgt, in, /*pairs=*/false);
    in.constraint_target = ct;
    in.constraint_weight = cw;
    const auto r = gram_solve(ctx->c, in, runs);
    std::memcpy(phi, r.data(), uint64_t(n) * 8);
  });
}

int sf_rank_edges(const double* phi, uint64_t n, uint32_t* order) {
  return guard([&] {
    need(order, "output");
    const auto o = ranking(std::vector<double>(phi, phi + n));
    std::memcpy(order, o.data(), n * 4);
  });
}

void sf_explain_options_default(sf_explain_options* o) {
  std::memset(o, 0, sizeof(*o));
  o->batch_size = 50;
  o->top_k = 10;
  o->tol = 1.0e-6;
  o->allow_exhaustive = 1;
  o->constraint_scale = 1.0e6;
  o->fidelity = 1;
  o->baseline_trials = 8;
  o->solver_mode = SF_SOLVER_AUTO;
}

int sf_explain_node(sf_ctx* ctx, const sf_graph* g, const sf_model* m, uint32_t node,
                    const sf_explain_options* opts, sf_explanation* out) {
  return guard([&] {
    need(ctx, "context");
    need(g, "graph");
    need(m, "model");
    need(out, "output");
    sf_explain_options o;
    if (opts)
      o = *opts;
    else
      sf_explain_options_default(&o);
    SF_CUDA(cudaSetDevice(ctx->c.device));
    explain_node(ctx->c, g->g, m->m, node, o, out);
  });
}

int sf_explain_nodes(sf_ctx* ctx, const sf_graph* g, const sf_model* m, const uint32_t* nodes,
                     uint64_t count, const sf_explain_options* opts, sf_explanation* out) {
  return guard([&] {
    need(ctx, "context");
    need(g, "graph");
    need(m, "model");
    if (count) {
      need(nodes, "nodes");
      need(out, "output");
    }
    if (m->m.layers.front().in != g->g.feature_dim)  // explain.cpp:149-153
      throw DataError("model expects " + std::to_string(m->m.layers.front().in) +
                      " input features but the graph has " + std::to_string(g->g.feature_dim));
    sf_explain_options o;
    if (opts)
      o = *opts;
    else
      sf_explain_options_default(&o);
    SF_CUDA(cudaSetDevice(ctx->c.device));
    const int workers = ctx->c.world == 1 ? int(std::min<uint64_t>(uint64_t(ctx->workers), count)) : 1;
    if (workers > 1) {
      // Targets are independent on one worker: pull them from a shared
      // counter on `workers` contexts of this device (one host thread each),
      // so one target's solve overlaps another's sampling and inference.
      // Each target's result is what explain_node gives on its own.
      while (int(ctx->helpers.size()) < workers - 1) {
        sf_ctx* h = nullptr;
        const int rc = sf_ctx_create(ctx->c.device, &h);
        if (rc != SF_OK) throw CudaError(std::string("helper context: ") + sf_last_error());
        h->c.fused_kind = ctx->c.fused_kind;
        ctx->helpers.emplace_back(h);
      }
      std::atomic<uint64_t> next{0};
      std::mutex mu;
      uint64_t bad = count;
      std::exception_ptr err;
      std::vector<char> filled(count, 0);
      auto run = [&](Ctx& c) {
        cudaSetDevice(c.device);
        c.concurrent = true;
        struct Reset {
          Ctx& c;
          ~Reset() { c.concurrent = false; }
        } reset{c};
        for (;;) {
          const uint64_t i = next++;
          if (i >= count) return;
          {
            std::lock_guard<std::mutex> g(mu);
            if (bad < i) return;  // an earlier target failed: stop
          }
          try {
            explain_node(c, g->g, m->m, nodes[i], o, &out[i]);
            filled[i] = 1;
          } catch (...) {
            std::lock_guard<std::mutex> g(mu);
            if (i < bad) {
              bad = i;
              err = std::current_exception();
            }
          }
        }
      };
      std::vector<std::thread> pool;
      for (int w = 1; w < workers; ++w) pool.emplace_back(run, std::ref(ctx->helpers[w - 1]->c));
      run(ctx->c);
      for (auto& t : pool) t.join();
      if (err) {
        for (uint64_t i = 0; i < count; ++i)
          if (filled[i]) sf_explanation_free(&out[i]);
        const uint32_t node = nodes[bad];
        try {
          std::rethrow_exception(err);
        } catch (const DataError& e) {  // explain.cpp:171-175
          throw DataError("node " + std::to_string(node) + ": " + e.what());
        } catch (const NumericalError& e) {
          throw NumericalError("node " + std::to_string(node) + ": " + e.what());
        }
      }
      return;
    }
    uint64_t done = 0;
    try {
      for (; done < count; ++done) {
        const uint32_t node = nodes[done];
        try {
          explain_node(ctx->c, g->g, m->m, node, o, &out[done]);
        } catch (const DataError& e) {  // explain.cpp:171-175
          throw DataError("node " + std::to_string(node) + ": " + e.what());
        } catch (const NumericalError& e) {
          throw NumericalError("node " + std::to_string(node) + ": " + e.what());
        }
      }
    } catch (...) {
      for (uint64_t i = 0; i <= done && i < count; ++i) sf_explanation_free(&out[i]);
      throw;
    }
  });
}

// explain.cpp:183-230: "degree-range:[lo,hi]:count" or a comma-separated id list
int sf_select_nodes(const sf_graph* g, const char* rule, uint32_t* out, uint64_t cap,
                    uint64_t* count) {
  return guard([&] {
    need(g, "graph");
    need(rule, "rule");
    need(count, "count");
    const Graph& gr = g->g;
    const std::string r(rule);
    std::vector<uint32_t> sel;
    const std::string pre = "degree-range:[";
    if (r.rfind("degree-range", 0) == 0) {
      uint64_t lo = 0, hi = 0, want = 0;
      char tail = 0;
      const bool ok = r.rfind(pre, 0) == 0 &&
                      std::sscanf(r.c_str() + pre.size(), "%20" SCNu64 ",%20" SCNu64 "]:%20" SCNu64 "%c", &lo, &hi,
                                  &want, &tail) == 3 &&
                      r.find_first_not_of("0123456789,]:", pre.size()) == std::string::npos;
      if (!ok)
        throw DataError("malformed selection rule '" + r + "' (expected degree-range:[lo,hi]:count)");
      if (lo > hi)
        throw DataError("degree range [" + std::to_string(lo) + "," + std::to_string(hi) + "] is empty");
      for (uint32_t u = 0; u < gr.num_nodes && sel.size() < want; ++u) {
        const uint64_t deg = gr.row_ptr[u + 1] - gr.row_ptr[u];
        if (deg >= lo && deg <= hi) sel.push_back(u);
      }
    } else {
      size_t pos = 0;
      while (pos <= r.size()) {
        size_t comma = r.find(',', pos);
        if (comma == std::string::npos) comma = r.size();
        size_t b = pos, e = comma;
        while (b < e && r[b] == ' ') ++b;
        while (e > b && r[e - 1] == ' ') --e;
        uint64_t id = 0;
        const auto [ptr, ec] = std::from_chars(r.data() + b, r.data() + e, id);
        if (ec != std::errc{} || ptr != r.data() + e || b == e)
          throw DataError("cannot parse node id '" + r.substr(pos, comma - pos) + "' in selection '" + r + "'");
        if (id >= gr.num_nodes)
          throw DataError("node id " + std::to_string(id) + " out of range for a graph with " +
                          std::to_string(gr.num_nodes) + " nodes");
        sel.push_back(uint32_t(id));
        pos = comma + 1;
      }
    }
    *count = sel.size();
    if (out) std::memcpy(out, sel.data(), std::min<uint64_t>(cap, sel.size()) * 4);
  });
}

int sf_explanation_free(sf_explanation* e) {
  if (!e) return SF_OK;
  for (void* p : {static_cast<void*>(e->phi), static_cast<void*>(e->players_global),
                  static_cast<void*>(e->top_player), static_cast<void*>(e->top_phi),
                  static_cast<void*>(e->fid_counts), static_cast<void*>(e->fid_plus),
                  static_cast<void*>(e->fid_plus_random), static_cast<void*>(e->fid_sparsities),
                  static_cast<void*>(e->fid_minus), static_cast<void*>(e->fid_minus_random)})
    std::free(p);
  std::memset(e, 0, sizeof(*e));
  return SF_OK;
}

int sf_evaluate_fidelity(sf_ctx* ctx, const sf_model* m, const sf_subgraph* sg, uint32_t cls,
                         const double* phi, const uint32_t* counts, uint32_t nc, const double* sp,
                         uint32_t ns, uint64_t seed, uint32_t trials, uint32_t* counts_out,
                         double* plus, double* plus_random, double* minus, double* minus_random) {
  return guard([&] {
    need(ctx, "context");
    need(m, "model");
    need(sg, "subgraph");
    SF_CUDA(cudaSetDevice(ctx->c.device));
    const uint64_t n = sg->s.num_players();
    FidelityOut f = fidelity(ctx->c, sg->s, m->m, cls, std::vector<double>(phi, phi + n),
                             std::vector<uint32_t>(counts, counts + nc),
                             std::vector<double>(sp, sp + ns), seed, trials);
    for (uint32_t i = 0; i < nc; ++i) {
      if (counts_out) counts_out[i] = f.counts[i];
      plus[i] = f.plus[i];
      plus_random[i] = f.plus_random[i];
    }
    for (uint32_t i = 0; i < ns; ++i) {
      minus[i] = f.minus[i];
      minus_random[i] = f.minus_random[i];
    }
  });
}

int sf_sample_and_predict(sf_ctx* ctx, const sf_model* m, const sf_subgraph* sg, uint32_t cls,
                          uint64_t k, uint64_t seed, int allow_exhaustive, double* stage_ms,
                          uint64_t* rows_local) {
  return guard([&] {
    need(ctx, "context");
    need(m, "model");
    need(sg, "subgraph");
    Ctx& c = ctx->c;
    SF_CUDA(cudaSetDevice(c.device));
    const uint32_t n = uint32_t(sg->s.num_players());
    const SizePlan plan = plan_sizes(n, k, allow_exhaustive != 0);
    const uint64_t rows = 2 * local_pair_count(plan.total_pairs(), c.rank, c.world);
    const uint32_t W = std::max<uint32_t>(1, (n + 63) / 64);
    c.masks.reserve(std::max<uint64_t>(rows / 2 * W, 1));  // kept-set rows only
    c.preds.reserve(std::max<uint64_t>(rows, 1));
    engine_prepare(c, sg->s, m->m);
    cudaEvent_t e0, e1, e2;
    SF_CUDA(cudaEventCreate(&e0));
    SF_CUDA(cudaEventCreate(&e1));
    SF_CUDA(cudaEventCreate(&e2));
    SF_CUDA(cudaEventRecord(e0, c.stream));
    launch_generate_masks(c, plan, seed, c.rank, c.world, c.masks.p, /*kept_only=*/true);
    SF_CUDA(cudaEventRecord(e1, c.stream));
    float dom = 0.f;
    engine_predict(c, c.masks.p, rows, cls, c.preds.p, nullptr, stage_ms ? &dom : nullptr, /*kept_only=*/true);
    SF_CUDA(cudaEventRecord(e2, c.stream));
    SF_CUDA(cudaEventSynchronize(e2));
    float a = 0.f, b = 0.f;
    SF_CUDA(cudaEventElapsedTime(&a, e0, e1));
    SF_CUDA(cudaEventElapsedTime(&b, e1, e2));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaEventDestroy(e2);
    if (stage_ms) {
      stage_ms[0] = a;
      stage_ms[1] = b;
      stage_ms[2] = dom;
    }
    if (rows_local) *rows_local = rows;
  });
}

}  // extern "C"
