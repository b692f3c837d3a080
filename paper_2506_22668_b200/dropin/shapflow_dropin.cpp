// C++ drop-in for the shapflow hot path (include/shapflow_b200.hpp): the
// reference declarations, defined over the libshapflow_b200 C-ABI.
//
// Compiled against the reference's unchanged public headers
// (proj/core/include/shapflow/*.hpp); see INTEGRATION.md for the build
// recipe and tests/test_gpu_conformance.py for the reference's own doctest
// suites run against it. Each definition cites the declaration it provides.
//
// Ownership and layout follow the reference: results are value types, mask
// rows are u64 words with bit e = player e. Graphs, models and computational
// graphs are converted to library handles once per object (cached per host
// thread by address and a content fingerprint), so repeated calls on the same
// Graph / GcnModel do not re-upload them.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "shapflow/bits.hpp"
#include "shapflow/comm.hpp"
#include "shapflow/document.hpp"
#include "shapflow/error.hpp"
#include "shapflow/explain.hpp"
#include "shapflow/fidelity.hpp"
#include "shapflow/gcn.hpp"
#include "shapflow/graph.hpp"
#include "shapflow/sampler.hpp"
#include "shapflow/solver.hpp"
#include "shapflow_b200.hpp"

namespace shapflow {
namespace {

// ----------------------------------------------------------------- errors
// C-ABI status -> the reference exception types (error.hpp:10-27)
[[noreturn]] void raise(int rc) {
  const std::string msg = sf_last_error();
  switch (rc) {
    case SF_ERR_DATA: throw DataError(msg);
    case SF_ERR_NUMERICAL: throw NumericalError(msg);
    case SF_ERR_PROTOCOL: throw ProtocolError(msg);
    default: throw std::runtime_error("shapflow_b200: " + msg);
  }
}
inline void check(int rc) {
  if (rc != SF_OK) raise(rc);
}

// ----------------------------------------------------------------- context
int g_default_device = -1;

int pick_device() {
  if (g_default_device >= 0) return g_default_device;
  const char* e = std::getenv("SHAPFLOW_B200_DEVICE");
  return e ? std::atoi(e) : 0;
}

struct ThreadCtx {
  sf_ctx* ctx = nullptr;
  int device = -1;
  ~ThreadCtx() {
    if (ctx) sf_ctx_destroy(ctx);
  }
};

sf_ctx* thread_context() {
  thread_local ThreadCtx t;
  const int dev = pick_device();
  if (!t.ctx || t.device != dev) {
    if (t.ctx) sf_ctx_destroy(t.ctx);
    t.ctx = nullptr;
    check(sf_ctx_create(dev, &t.ctx));
    t.device = dev;
  }
  return t.ctx;
}

// The communicator a call runs under. NcclCommunicator: its own context and
// device-side collectives. Anything else: this thread's context with the
// Communicator's all_reduce_sum / barrier behind the host-comm hooks (world 1
// needs no collective at all).
class Binding {
 public:
  explicit Binding(Communicator& comm) : comm_(comm) {
    nccl_ = dynamic_cast<b200::NcclCommunicator*>(&comm);
    if (nccl_) {
      ctx_ = nccl_->context();
      return;
    }
    ctx_ = thread_context();
    // every collective goes through `comm` (for one worker the sums are
    // identities, but its CollectiveStats still count them)
    check(sf_ctx_set_host_comm(ctx_, comm.rank(), comm.world_size(), this, &Binding::all_reduce, &Binding::barrier));
  }
  ~Binding() {
    if (nccl_) {
      nccl_->absorb_device_stats();
    } else {  // no hooks outlive this call (they point at *this)
      sf_ctx_set_host_comm(ctx_, 0, 1, nullptr, nullptr, nullptr);
    }
  }
  sf_ctx* ctx() const { return ctx_; }
  // a failure inside the Communicator (e.g. a ProtocolError) is rethrown as is
  void check_call(int rc) {
    if (rc != SF_OK && pending_) {
      auto e = pending_;
      pending_ = nullptr;
      std::rethrow_exception(e);
    }
    check(rc);
  }

 private:
  static int all_reduce(void* user, double* buf, std::uint64_t count) {
    auto* self = static_cast<Binding*>(user);
    try {
      if (buf == nullptr) {  // one worker: count the call, the sum is the identity
        thread_local std::vector<double> scratch;
        scratch.assign(count, 0.0);
        self->comm_.all_reduce_sum(std::span<double>(scratch.data(), count));
        return 0;
      }
      self->comm_.all_reduce_sum(std::span<double>(buf, count));
      return 0;
    } catch (...) {
      self->pending_ = std::current_exception();
      return 1;
    }
  }
  static int barrier(void* user) {
    auto* self = static_cast<Binding*>(user);
    try {
      self->comm_.barrier();
      return 0;
    } catch (...) {
      self->pending_ = std::current_exception();
      return 1;
    }
  }
  Communicator& comm_;
  b200::NcclCommunicator* nccl_ = nullptr;
  sf_ctx* ctx_ = nullptr;
  std::exception_ptr pending_;
};

// ----------------------------------------------------------------- handles
// FNV-1a over a bounded sample of a buffer: cheap content fingerprint that
// catches a different object reusing an address.
template <typename T>
std::uint64_t sample_hash(const std::vector<T>& v) {
  std::uint64_t h = 1469598103934665603ull ^ v.size();
  const std::size_t n = v.size(), step = std::max<std::size_t>(1, n / 4096);
  for (std::size_t i = 0; i < n; i += step) {
    std::uint64_t x = 0;
    std::memcpy(&x, &v[i], std::min(sizeof(T), sizeof(x)));
    h = (h ^ x) * 1099511628211ull;
  }
  if (n) {
    std::uint64_t x = 0;
    std::memcpy(&x, &v[n - 1], std::min(sizeof(T), sizeof(x)));
    h = (h ^ x) * 1099511628211ull;
  }
  return h;
}

template <typename H, int (*Free)(H*)>
struct Handle {
  H* h = nullptr;
  Handle() = default;
  explicit Handle(H* p) : h(p) {}
  Handle(const Handle&) = delete;
  Handle& operator=(const Handle&) = delete;
  ~Handle() {
    if (h) Free(h);
  }
};
using GraphH = Handle<sf_graph, sf_graph_free>;
using ModelH = Handle<sf_model, sf_model_free>;
using SubH = Handle<sf_subgraph, sf_subgraph_free>;

template <typename Key, typename H>
struct Cache {  // small per-thread LRU of converted objects
  std::vector<std::pair<Key, std::shared_ptr<H>>> items;
  std::shared_ptr<H> find(const Key& k) {
    for (size_t i = 0; i < items.size(); ++i)
      if (items[i].first == k) {
        auto v = items[i].second;
        if (i) std::rotate(items.begin(), items.begin() + i, items.begin() + i + 1);
        return v;
      }
    return nullptr;
  }
  void put(const Key& k, std::shared_ptr<H> v) {
    items.insert(items.begin(), {k, std::move(v)});
    if (items.size() > 8) items.pop_back();
  }
};

using GraphKey = std::tuple<const void*, std::uint32_t, std::size_t, std::size_t, std::uint64_t, std::uint64_t>;
using ModelKey = std::tuple<const void*, std::size_t, std::uint64_t>;
using SubKey = std::tuple<const void*, std::uint32_t, std::size_t, std::size_t, std::uint64_t, std::uint64_t>;

std::shared_ptr<GraphH> graph_handle(const Graph& g) {  // graph.hpp:16-31
  thread_local Cache<GraphKey, GraphH> cache;
  const GraphKey key{&g, g.num_nodes, g.col.size(), g.feature_dim, sample_hash(g.col), sample_hash(g.features)};
  if (auto h = cache.find(key)) return h;
  if (g.row_ptr.size() != std::size_t{g.num_nodes} + 1) throw DataError("graph CSR is malformed");
  if (g.features.size() != std::size_t{g.num_nodes} * g.feature_dim)
    throw DataError("graph feature buffer does not match its dimensions");
  std::vector<std::uint64_t> rp(g.row_ptr.begin(), g.row_ptr.end());
  sf_graph* out = nullptr;
  check(sf_graph_from_csr(g.num_nodes, rp.data(), g.col.data(), g.features.data(), g.feature_dim,
                          g.labels.size() == g.num_nodes ? g.labels.data() : nullptr, &out));
  auto h = std::make_shared<GraphH>(out);
  cache.put(key, h);
  return h;
}

std::shared_ptr<ModelH> model_handle(const GcnModel& m) {  // gcn.hpp:13-30
  thread_local Cache<ModelKey, ModelH> cache;
  std::uint64_t fp = m.layers.size();
  for (const auto& l : m.layers) fp = fp * 31 + sample_hash(l.weight) + 7 * sample_hash(l.bias) + l.in * 131 + l.out;
  const ModelKey key{&m, m.layers.size(), fp};
  if (auto h = cache.find(key)) return h;
  if (m.layers.empty()) throw DataError("model has no layers");
  std::vector<std::uint64_t> dims{m.layers.front().in};
  std::vector<float> w, b;
  for (const auto& l : m.layers) {
    if (l.in != dims.back()) throw DataError("model layer widths do not chain");
    if (l.weight.size() != l.in * l.out || l.bias.size() != l.out)
      throw DataError("model layer buffers do not match its widths");
    dims.push_back(l.out);
    w.insert(w.end(), l.weight.begin(), l.weight.end());
    b.insert(b.end(), l.bias.begin(), l.bias.end());
  }
  sf_model* out = nullptr;
  check(sf_model_create(int(m.layers.size()), dims.data(), w.data(), b.data(), &out));
  auto h = std::make_shared<ModelH>(out);
  cache.put(key, h);
  return h;
}

std::shared_ptr<SubH> subgraph_handle(const ComputationalGraph& cg) {  // graph.hpp:36-53
  thread_local Cache<SubKey, SubH> cache;
  const SubKey key{&cg, cg.num_nodes(), cg.players.size(), cg.feature_dim, sample_hash(cg.col),
                   sample_hash(cg.features)};
  if (auto h = cache.find(key)) return h;
  const std::uint32_t V = cg.num_nodes();
  if (cg.row_ptr.size() != std::size_t{V} + 1 || cg.edge_player.size() != cg.col.size())
    throw DataError("computational graph CSR is malformed");
  if (cg.features.size() != std::size_t{V} * cg.feature_dim)
    throw DataError("computational graph features do not match its dimensions");
  std::vector<std::uint64_t> rp(cg.row_ptr.begin(), cg.row_ptr.end());
  std::vector<std::uint32_t> pl(2 * cg.players.size());
  for (std::size_t e = 0; e < cg.players.size(); ++e) {
    pl[2 * e] = cg.players[e].first;
    pl[2 * e + 1] = cg.players[e].second;
  }
  sf_subgraph* out = nullptr;
  check(sf_subgraph_create(cg.target_global, V, cg.players.size(), rp.data(), cg.col.data(), cg.edge_player.data(),
                           pl.data(), cg.local_to_global.data(), cg.features.data(), cg.feature_dim, &out));
  auto h = std::make_shared<SubH>(out);
  cache.put(key, h);
  return h;
}

}  // namespace

// ================================================================ sampler
// sampler.hpp:49-50
SizePlan plan_sizes(std::uint32_t n, std::uint64_t k, bool allow_exhaustive) {
  std::uint64_t ncls = 0, requested = 0;
  int exhaustive = 0;
  check(sf_plan_sizes(n, k, allow_exhaustive ? 1 : 0, nullptr, nullptr, nullptr, 0, &ncls, &exhaustive, &requested));
  std::vector<std::uint32_t> sizes(ncls);
  std::vector<std::uint64_t> pairs(ncls), first(ncls);
  check(sf_plan_sizes(n, k, allow_exhaustive ? 1 : 0, sizes.data(), pairs.data(), first.data(), ncls, &ncls,
                      &exhaustive, &requested));
  SizePlan p;
  p.num_players = n;
  p.requested = requested;
  p.exhaustive = exhaustive != 0;
  p.classes.resize(ncls);
  for (std::uint64_t c = 0; c < ncls; ++c) p.classes[c] = SizeClass{sizes[c], pairs[c], first[c]};
  return p;
}

// sampler.hpp:84-85 — generated on the GPU (Philox-4x32-10 + Floyd, bit-exact)
MaskBlock generate_masks(const SizePlan& plan, std::uint64_t seed, int rank, int world) {
  if (world < 1 || rank < 0 || rank >= world)
    throw DataError("invalid worker rank " + std::to_string(rank) + " of " + std::to_string(world));
  const std::uint64_t nc = plan.classes.size();
  std::vector<std::uint32_t> sizes(nc);
  std::vector<std::uint64_t> pairs(nc), first(nc);
  for (std::uint64_t c = 0; c < nc; ++c) {
    sizes[c] = plan.classes[c].size;
    pairs[c] = plan.classes[c].pairs;
    first[c] = plan.classes[c].first_pair;
  }
  sf_ctx* ctx = thread_context();
  std::uint64_t rows = 0;
  check(sf_generate_masks(ctx, plan.num_players, sizes.data(), pairs.data(), first.data(), nc,
                          plan.exhaustive ? 1 : 0, seed, rank, world, nullptr, 0, &rows, nullptr));
  MaskBlock mb;
  mb.num_players = plan.num_players;
  mb.num_rows = rows;
  mb.words_per_row = words_for_bits(plan.num_players);
  mb.rank = rank;
  mb.world = world;
  mb.seed = seed;
  mb.global_pair_count = plan.total_pairs();
  mb.global_pairs.resize(rows / 2);
  for (std::uint64_t j = 0; j < rows / 2; ++j) mb.global_pairs[j] = std::uint64_t(rank) + j * std::uint64_t(world);
  mb.global_rows_of_size.assign(std::size_t{plan.num_players} + 1, 0);
  mb.bits.assign(rows * mb.words_per_row, 0);
  check(sf_generate_masks(ctx, plan.num_players, sizes.data(), pairs.data(), first.data(), nc,
                          plan.exhaustive ? 1 : 0, seed, rank, world, mb.bits.data(), mb.bits.size(), &rows,
                          mb.global_rows_of_size.data()));
  return mb;
}

// ================================================================ inference
// gcn.hpp:50-51
std::vector<float> predict_probs(const GcnModel& m, const ComputationalGraph& cg,
                                 std::span<const std::uint64_t> mask) {
  auto mh = model_handle(m);
  auto sh = subgraph_handle(cg);
  std::vector<float> probs(m.num_classes());
  check(sf_predict_probs(thread_context(), mh->h, sh->h, mask.data(), mask.size(), probs.data()));
  return probs;
}

// gcn.hpp:53-55
float predict(const GcnModel& m, const ComputationalGraph& cg, std::span<const std::uint64_t> mask,
              std::uint32_t class_index) {
  if (class_index >= m.num_classes()) throw DataError("class index out of range");
  return predict_probs(m, cg, mask)[class_index];
}

// gcn.hpp:60-62 — the batched masked-GCN engine (tcgen05 3xTF32 layer 0)
std::vector<float> predict_batched(const GcnModel& m, const ComputationalGraph& cg, const BitRows& masks,
                                   std::uint32_t class_index, std::size_t batch_size) {
  auto mh = model_handle(m);
  auto sh = subgraph_handle(cg);
  std::vector<float> out(masks.rows);
  check(sf_predict_batched(thread_context(), mh->h, sh->h, masks.data, masks.rows, masks.words_per_row, class_index,
                           batch_size, out.data()));
  return out;
}

// ================================================================ solver
namespace {
// WlsProblem rows are dense 0/1 floats (assemble_problem, solver.cpp:140-147);
// the device solver takes them as bit rows.
std::vector<std::uint64_t> pack_rows(const WlsProblem& p) {
  const std::uint32_t n = p.num_players;
  const std::size_t W = std::max<std::size_t>(1, words_for_bits(n));
  std::vector<std::uint64_t> bits(p.num_rows * W, 0);
  for (std::uint64_t i = 0; i < p.num_rows; ++i) {
    const float* r = p.row(i);
    for (std::uint32_t e = 0; e < n; ++e) {
      if (r[e] == 1.0f)
        bits[i * W + (e >> 6)] |= std::uint64_t{1} << (e & 63);
      else if (r[e] != 0.0f)
        throw DataError("row " + std::to_string(i) + " holds a value other than 0 or 1");
    }
  }
  return bits;
}

void validate_slice(const WlsProblem& p, const Communicator& comm) {  // solver.cpp:165-172
  if (p.rank != comm.rank() || p.world != comm.world_size())
    throw DataError("system slice does not match the communicator layout");
  if (p.num_rows % 2 != 0) throw DataError("local rows must come in adjacent pairs");
  if (p.weights.size() != p.num_rows || p.targets.size() != p.num_rows ||
      p.rows.size() != p.num_rows * std::size_t{p.num_players})
    throw DataError("inconsistent system slice");
}
}  // namespace

// solver.hpp:94-95 — distributed CGLS on the bit rows (FP64); one vector + one
// scalar all-reduce per iteration through `comm` (+1 scalar with trace)
CglsResult solve_cgls(const WlsProblem& p, Communicator& comm, const CglsOptions& opts) {
  CglsResult res;
  if (p.num_players == 0) {
    res.converged = true;
    return res;
  }
  validate_slice(p, comm);
  const std::vector<std::uint64_t> bits = pack_rows(p);
  const std::size_t W = std::max<std::size_t>(1, words_for_bits(p.num_players));
  Binding bind(comm);
  res.phi.assign(p.num_players, 0.0);
  const std::uint64_t cap = opts.trace ? (opts.max_iter ? opts.max_iter : std::min<std::uint64_t>(p.num_players, 5000)) : 0;
  std::vector<double> trace(cap), row_trace(cap);
  std::uint64_t it = 0;
  double rel = 0.0;
  int conv = 0;
  bind.check_call(sf_solve_cgls_ex(bind.ctx(), p.num_players, bits.data(), p.num_rows, W, p.weights.data(),
                                   p.targets.data(), p.constraint_target, p.constraint_weight, opts.tol,
                                   opts.max_iter, /*mode=*/opts.fixed_order ? 2 : 0,
                                   std::max<std::uint64_t>(p.global_pair_count, p.num_rows / 2), res.phi.data(), &it,
                                   &rel, &conv, opts.trace ? trace.data() : nullptr,
                                opts.trace ? row_trace.data() : nullptr, cap));
  res.iterations = it;
  res.relative_residual = rel;
  res.converged = conv != 0;
  if (opts.trace) {
    trace.resize(std::min<std::uint64_t>(it, cap));
    row_trace.resize(std::min<std::uint64_t>(it, cap));
    res.trace = std::move(trace);
    res.row_residual_trace = std::move(row_trace);
  }
  return res;
}

// solver.hpp:100 — Gram + Cholesky on the device, world 1, n <= 20000
std::vector<double> solve_direct(const WlsProblem& p) {
  const std::uint32_t n = p.num_players;
  if (p.world != 1) throw DataError("direct solve needs the full system on a single worker");
  if (n > 20000) throw DataError("direct solve limited to 20000 players, got " + std::to_string(n));
  if (p.weights.size() != p.num_rows || p.targets.size() != p.num_rows ||
      p.rows.size() != p.num_rows * std::size_t{n})
    throw DataError("inconsistent system slice");
  std::vector<double> phi(n, 0.0);
  if (n == 0) return phi;
  const std::vector<std::uint64_t> bits = pack_rows(p);
  sf_ctx* ctx = thread_context();
  check(sf_ctx_set_host_comm(ctx, 0, 1, nullptr, nullptr, nullptr));
  check(sf_solve_direct(ctx, n, bits.data(), p.num_rows, std::max<std::size_t>(1, words_for_bits(n)),
                        p.weights.data(), p.targets.data(), p.constraint_target, p.constraint_weight, phi.data()));
  return phi;
}

// solver.hpp:109
std::vector<RankedEdge> rank_edges(std::span<const double> phi) {
  std::vector<std::uint32_t> order(phi.size());
  check(sf_rank_edges(phi.data(), phi.size(), order.data()));
  std::vector<RankedEdge> out(phi.size());
  for (std::size_t i = 0; i < phi.size(); ++i) out[i] = RankedEdge{order[i], phi[order[i]]};
  return out;
}

// ================================================================ pipeline
// explain.hpp:35
std::uint64_t auto_samples(std::size_t num_players) { return sf_auto_samples(num_players); }

// explain.hpp:39
std::uint64_t node_sampling_seed(std::uint64_t seed, std::uint32_t node) { return sf_node_sampling_seed(seed, node); }

// explain.hpp:47-49 — extraction, sampling, masked inference, CGLS, ranking
// and Fidelity on the device, collective over `comm`
NodeExplanation explain_node(const Graph& g, const GcnModel& m, std::uint32_t node, const ExplainOptions& opts,
                             Communicator& comm) {
  if (node >= g.num_nodes) throw DataError("node " + std::to_string(node) + " out of range");
  auto gh = graph_handle(g);
  auto mh = model_handle(m);
  Binding bind(comm);
  sf_explain_options o;
  sf_explain_options_default(&o);
  o.samples = opts.samples;
  o.batch_size = opts.batch_size;
  o.top_k = opts.top_k;
  o.seed = opts.seed;
  o.tol = opts.tol;
  o.max_iter = opts.max_iter;
  o.player_cap = opts.player_cap;
  o.allow_exhaustive = opts.allow_exhaustive ? 1 : 0;
  o.constraint_scale = opts.constraint_scale;
  o.fidelity = opts.fidelity ? 1 : 0;
  o.baseline_trials = opts.baseline_trials;
  o.solver_mode = SF_SOLVER_CGLS;  // the reference's solver and protocol
  o.fixed_order = opts.fixed_order ? 1 : 0;
  o.top_counts = opts.top_counts.data();
  o.num_top_counts = std::uint32_t(opts.top_counts.size());
  o.sparsities = opts.sparsities.data();
  o.num_sparsities = std::uint32_t(opts.sparsities.size());
  sf_explanation e;
  std::memset(&e, 0, sizeof(e));
  bind.check_call(sf_explain_node(bind.ctx(), gh->h, mh->h, node, &o, &e));
  struct Free {
    sf_explanation* e;
    ~Free() { sf_explanation_free(e); }
  } guard{&e};
  NodeExplanation out;
  out.node = e.node;
  out.skipped = e.skipped != 0;
  out.warning = e.warning;
  out.timings.sampling_ms = e.sampling_ms;
  out.timings.prediction_ms = e.prediction_ms;
  out.timings.solve_ms = e.solve_ms;
  out.timings.total_ms = e.total_ms;
  if (out.skipped) return out;
  out.predicted_class = e.predicted_class;
  out.base_score = e.base_score;
  out.full_score = e.full_score;
  out.players.resize(e.num_players);
  for (std::uint64_t i = 0; i < e.num_players; ++i)
    out.players[i] = {e.players_global[2 * i], e.players_global[2 * i + 1]};
  out.phi.assign(e.phi, e.phi + e.num_players);
  out.exhaustive = e.exhaustive != 0;
  out.rows = e.rows;
  out.iterations = e.iterations;
  out.residual = e.residual;
  out.converged = e.converged != 0;
  out.top.resize(e.num_top);
  for (std::uint32_t i = 0; i < e.num_top; ++i) out.top[i] = RankedEdge{e.top_player[i], e.top_phi[i]};
  if (e.has_fidelity) {
    FidelityReport f;
    f.node = node;
    f.predicted_class = e.predicted_class;
    f.full_score = e.full_score;
    f.top_counts.assign(e.fid_counts, e.fid_counts + e.num_counts);
    f.plus.assign(e.fid_plus, e.fid_plus + e.num_counts);
    f.plus_random.assign(e.fid_plus_random, e.fid_plus_random + e.num_counts);
    f.sparsities.assign(e.fid_sparsities, e.fid_sparsities + e.num_sparsities);
    f.minus.assign(e.fid_minus, e.fid_minus + e.num_sparsities);
    f.minus_random.assign(e.fid_minus_random, e.fid_minus_random + e.num_sparsities);
    f.baseline_seed = node_sampling_seed(opts.seed, node);
    f.baseline_trials = opts.baseline_trials;
    out.fidelity = std::move(f);
  }
  return out;
}

// ================================================================ NCCL communicator
namespace b200 {

std::array<char, 128> nccl_unique_id() {
  std::array<char, 128> id{};
  check(sf_nccl_unique_id(id.data()));
  return id;
}

void set_default_device(int device) { g_default_device = device; }
int default_device() { return pick_device(); }

NcclCommunicator::NcclCommunicator(int device, int rank, int world, const std::array<char, 128>& unique_id)
    : rank_(rank), world_(world) {
  if (world < 1 || rank < 0 || rank >= world)
    throw DataError("invalid worker rank " + std::to_string(rank) + " of " + std::to_string(world));
  check(sf_ctx_create(device, &ctx_));
  const int rc = sf_ctx_join_nccl(ctx_, unique_id.data(), rank, world);
  if (rc != SF_OK) {
    const std::string msg = sf_last_error();
    sf_ctx_destroy(ctx_);
    ctx_ = nullptr;
    throw ProtocolError(msg);
  }
}

NcclCommunicator::~NcclCommunicator() {
  if (ctx_) sf_ctx_destroy(ctx_);
}

void NcclCommunicator::absorb_device_stats() {
  std::uint64_t now[4] = {0, 0, 0, 0};
  check(sf_ctx_stats(ctx_, &now[0], &now[1], &now[2], &now[3]));
  stats_.scalar_allreduce += now[0] - seen_[0];
  stats_.vector_allreduce += now[1] - seen_[1];
  stats_.barriers += now[2] - seen_[2];
  stats_.doubles_reduced += now[3] - seen_[3];
  next_seq_ += (now[0] - seen_[0]) + (now[1] - seen_[1]) + (now[2] - seen_[2]);
  std::copy(now, now + 4, seen_);
}

// Communicator::all_reduce_sum has already counted this call; the context's
// own counters are absorbed here so absorb_device_stats does not recount it.
void NcclCommunicator::all_reduce_impl(std::uint64_t, std::span<double> buf) {
  check(sf_ctx_allreduce_host(ctx_, buf.data(), buf.size()));
  check(sf_ctx_stats(ctx_, &seen_[0], &seen_[1], &seen_[2], &seen_[3]));
}

void NcclCommunicator::barrier_impl(std::uint64_t) {
  check(sf_ctx_barrier(ctx_));
  check(sf_ctx_stats(ctx_, &seen_[0], &seen_[1], &seen_[2], &seen_[3]));
}

// root receives the concatenation in rank order (comm.hpp:38-39): segment
// lengths, then the zero-padded segments, summed across ranks
std::vector<double> NcclCommunicator::gather_impl(std::uint64_t, std::span<const double> buf) {
  std::vector<double> lens(world_, 0.0);
  lens[rank_] = double(buf.size());
  check(sf_ctx_allreduce_host(ctx_, lens.data(), lens.size()));
  std::vector<std::uint64_t> off(world_ + 1, 0);
  for (int r = 0; r < world_; ++r) off[r + 1] = off[r] + std::uint64_t(lens[r]);
  std::vector<double> all(off[world_], 0.0);
  std::copy(buf.begin(), buf.end(), all.begin() + off[rank_]);
  check(sf_ctx_allreduce_host(ctx_, all.data(), all.size()));
  check(sf_ctx_stats(ctx_, &seen_[0], &seen_[1], &seen_[2], &seen_[3]));
  if (rank_ != 0) return {};
  return all;
}

}  // namespace b200
}  // namespace shapflow
