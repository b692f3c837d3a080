// TEST INFRASTRUCTURE ONLY — the checker, never the product.
//
// A thin extern "C" driver over the UNMODIFIED reference core
// (/root/reference/proj/core/src/*.cpp, compiled by oracle/Makefile into
// oracle/_ref/libshapflow_ref.so). Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference leg may load it. Nothing in
// paper_2506_22668_b200/ links or calls it.
//
// Every entry point forwards to the reference API named in its comment;
// exceptions are mapped to status codes exactly like the reference CLI maps
// them to exit codes (tools/shapflow.cpp:496-505): DataError -> 2,
// NumericalError -> 3, ProtocolError -> 4, anything else -> 1.

#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "shapflow/bits.hpp"
#include "shapflow/comm.hpp"
#include "shapflow/error.hpp"
#include "shapflow/explain.hpp"
#include "shapflow/fidelity.hpp"
#include "shapflow/gcn.hpp"
#include "shapflow/graph.hpp"
#include "shapflow/oracle.hpp"
#include "shapflow/philox.hpp"
#include "shapflow/sampler.hpp"
#include "shapflow/solver.hpp"
#include "shapflow/synthetic.hpp"

using namespace shapflow;

namespace {

thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const DataError& e) {
    g_err = e.what();
    return 2;
  } catch (const NumericalError& e) {
    g_err = e.what();
    return 3;
  } catch (const ProtocolError& e) {
    g_err = e.what();
    return 4;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

using Clock = std::chrono::steady_clock;
double ms_since(Clock::time_point t) {
  return std::chrono::duration<double, std::milli>(Clock::now() - t).count();
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---------------------------------------------------------------- philox
// philox.hpp:13-73
void ref_philox_u64(uint64_t seed, uint64_t stream, uint64_t count,
                    uint64_t* out) {
  Philox p(seed, stream);
  for (uint64_t i = 0; i < count; ++i) out[i] = p.next_u64();
}

// explain.cpp:37-40
uint64_t ref_node_sampling_seed(uint64_t seed, uint32_t node) {
  return node_sampling_seed(seed, node);
}

// sampler.cpp:79-91
int ref_kernel_weight(uint32_t n, uint32_t s, double* out) {
  return guard([&] { *out = kernel_weight(n, s); });
}

uint64_t ref_binomial_or_max(uint32_t n, uint32_t s) {
  return binomial_or_max(n, s);
}

// ---------------------------------------------------------------- plan
// sampler.cpp:93-151. Returns class count via *nclasses; arrays may be
// null to query the count first.
int ref_plan_sizes(uint32_t n, uint64_t k, int allow_exhaustive,
                   uint32_t* sizes, uint64_t* pairs, uint64_t* first_pair,
                   uint64_t cap, uint64_t* nclasses, int* exhaustive,
                   uint64_t* requested) {
  return guard([&] {
    SizePlan p = plan_sizes(n, k, allow_exhaustive != 0);
    *nclasses = p.classes.size();
    *exhaustive = p.exhaustive ? 1 : 0;
    *requested = p.requested;
    if (sizes && p.classes.size() <= cap) {
      for (size_t i = 0; i < p.classes.size(); ++i) {
        sizes[i] = p.classes[i].size;
        pairs[i] = p.classes[i].pairs;
        first_pair[i] = p.classes[i].first_pair;
      }
    }
  });
}

// sampler.cpp:153-210. out (rows x words) may be null to query rows.
// rows_of_size (n+1 entries) receives global_rows_of_size when non-null.
int ref_generate_masks(uint32_t n, uint64_t k, int allow_exhaustive,
                       uint64_t seed, int rank, int world, uint64_t* out,
                       uint64_t cap_words, uint64_t* rows, uint64_t* words,
                       uint64_t* rows_of_size) {
  return guard([&] {
    SizePlan p = plan_sizes(n, k, allow_exhaustive != 0);
    MaskBlock mb = generate_masks(p, seed, rank, world);
    *rows = mb.num_rows;
    *words = mb.words_per_row;
    if (out) {
      if (mb.bits.size() > cap_words) throw DataError("output too small");
      std::memcpy(out, mb.bits.data(), mb.bits.size() * 8);
    }
    if (rows_of_size)
      std::memcpy(rows_of_size, mb.global_rows_of_size.data(),
                  mb.global_rows_of_size.size() * 8);
  });
}

// ---------------------------------------------------------------- graphs
// graph.cpp:165-193 (load_graph) / synthetic.cpp:56-86
void* ref_graph_load(const char* path) {
  Graph* g = nullptr;
  int rc = guard([&] { g = new Graph(load_graph(path)); });
  return rc == 0 ? g : nullptr;
}

void* ref_graph_random(uint32_t nodes, uint64_t edges, uint64_t dim,
                       uint32_t classes, uint64_t seed) {
  Graph* g = nullptr;
  int rc = guard([&] {
    g = new Graph(gen_random_graph(nodes, edges, dim, classes, seed));
  });
  return rc == 0 ? g : nullptr;
}

void* ref_graph_build(uint32_t num_nodes, const uint64_t* edges_uv,
                      uint64_t num_edges, const float* features,
                      uint64_t dim) {
  Graph* g = nullptr;
  int rc = guard([&] {
    std::vector<std::pair<uint64_t, uint64_t>> e(num_edges);
    for (uint64_t i = 0; i < num_edges; ++i)
      e[i] = {edges_uv[2 * i], edges_uv[2 * i + 1]};
    std::vector<float> f(features, features + uint64_t(num_nodes) * dim);
    g = new Graph(build_graph(num_nodes, e, std::move(f), dim, {}));
  });
  return rc == 0 ? g : nullptr;
}

int ref_graph_save(void* g, const char* path) {
  return guard([&] { save_graph(*static_cast<Graph*>(g), path); });
}

void ref_graph_free(void* g) { delete static_cast<Graph*>(g); }

void ref_graph_dims(void* gp, uint32_t* nodes, uint64_t* nnz, uint64_t* dim) {
  const Graph& g = *static_cast<Graph*>(gp);
  *nodes = g.num_nodes;
  *nnz = g.col.size();
  *dim = g.feature_dim;
}

void ref_graph_copy(void* gp, uint64_t* row_ptr, uint32_t* col) {
  const Graph& g = *static_cast<Graph*>(gp);
  for (size_t i = 0; i < g.row_ptr.size(); ++i) row_ptr[i] = g.row_ptr[i];
  std::memcpy(col, g.col.data(), g.col.size() * 4);
}

// ---------------------------------------------------------------- models
// synthetic.cpp:88-118
void* ref_model_random(uint64_t input_dim, const uint64_t* hidden, int nh,
                       uint32_t classes, uint64_t seed) {
  GcnModel* m = nullptr;
  int rc = guard([&] {
    std::vector<size_t> h(hidden, hidden + nh);
    m = new GcnModel(gen_random_model(input_dim, h, classes, seed));
  });
  return rc == 0 ? m : nullptr;
}

// layers given as dims[0..L] and concatenated weights / biases
void* ref_model_from_arrays(int L, const uint64_t* dims, const float* weights,
                            const float* biases) {
  auto* m = new GcnModel;
  for (int l = 0; l < L; ++l) {
    GcnLayer lay;
    lay.in = dims[l];
    lay.out = dims[l + 1];
    lay.weight.assign(weights, weights + lay.in * lay.out);
    lay.bias.assign(biases, biases + lay.out);
    weights += lay.in * lay.out;
    biases += lay.out;
    m->layers.push_back(std::move(lay));
  }
  return m;
}

void* ref_model_load(const char* path) {
  GcnModel* m = nullptr;
  int rc = guard([&] { m = new GcnModel(load_model(path)); });
  return rc == 0 ? m : nullptr;
}

int ref_model_save(void* m, const char* path) {
  return guard([&] { save_model(*static_cast<GcnModel*>(m), path); });
}

void ref_model_free(void* m) { delete static_cast<GcnModel*>(m); }

int ref_model_depth(void* m) {
  return static_cast<int>(static_cast<GcnModel*>(m)->depth());
}

void ref_model_layer(void* mp, int l, uint64_t* in, uint64_t* out, float* w,
                     float* b) {
  const GcnLayer& lay = static_cast<GcnModel*>(mp)->layers[l];
  *in = lay.in;
  *out = lay.out;
  if (w) std::memcpy(w, lay.weight.data(), lay.weight.size() * 4);
  if (b) std::memcpy(b, lay.bias.data(), lay.bias.size() * 4);
}

// ---------------------------------------------------------------- subgraph
// graph.cpp:195-261
void* ref_extract(void* g, uint32_t target, int hops) {
  ComputationalGraph* cg = nullptr;
  int rc = guard([&] {
    cg = new ComputationalGraph(
        extract_computational_graph(*static_cast<Graph*>(g), target, hops));
  });
  return rc == 0 ? cg : nullptr;
}

void ref_cg_free(void* cg) { delete static_cast<ComputationalGraph*>(cg); }

void ref_cg_dims(void* cgp, uint32_t* V, uint64_t* n, uint64_t* nnz,
                 uint64_t* dim) {
  const ComputationalGraph& cg = *static_cast<ComputationalGraph*>(cgp);
  *V = cg.num_nodes();
  *n = cg.num_players();
  *nnz = cg.col.size();
  *dim = cg.feature_dim;
}

void ref_cg_copy(void* cgp, uint64_t* row_ptr, uint32_t* col,
                 uint32_t* edge_player, uint32_t* players_uv,
                 uint32_t* local_to_global, float* features) {
  const ComputationalGraph& cg = *static_cast<ComputationalGraph*>(cgp);
  for (size_t i = 0; i < cg.row_ptr.size(); ++i) row_ptr[i] = cg.row_ptr[i];
  std::memcpy(col, cg.col.data(), cg.col.size() * 4);
  std::memcpy(edge_player, cg.edge_player.data(), cg.edge_player.size() * 4);
  for (size_t e = 0; e < cg.players.size(); ++e) {
    players_uv[2 * e] = cg.players[e].first;
    players_uv[2 * e + 1] = cg.players[e].second;
  }
  std::memcpy(local_to_global, cg.local_to_global.data(),
              cg.local_to_global.size() * 4);
  if (features)
    std::memcpy(features, cg.features.data(), cg.features.size() * 4);
}

// ---------------------------------------------------------------- predict
// gcn.cpp:259-270
int ref_predict_batched(void* m, void* cg, const uint64_t* bits, uint64_t rows,
                        uint64_t words, uint32_t cls, uint64_t batch,
                        float* out) {
  return guard([&] {
    std::vector<float> r =
        predict_batched(*static_cast<GcnModel*>(m),
                        *static_cast<ComputationalGraph*>(cg),
                        BitRows{bits, rows, words}, cls, batch);
    std::memcpy(out, r.data(), r.size() * 4);
  });
}

// gcn.cpp:239-248
int ref_predict_probs(void* m, void* cg, const uint64_t* mask, uint64_t words,
                      float* out) {
  return guard([&] {
    std::vector<float> r = predict_probs(*static_cast<GcnModel*>(m),
                                         *static_cast<ComputationalGraph*>(cg),
                                         {mask, words});
    std::memcpy(out, r.data(), r.size() * 4);
  });
}

// ---------------------------------------------------------------- solve
// solver.cpp:95-156 + 158-362 on one worker: masks are the caller's rows,
// per-size counts are taken from the rows themselves (world == 1 path of
// assemble_problem).
int ref_solve_cgls(uint32_t n, const uint64_t* bits, uint64_t rows,
                   uint64_t words, const double* values, double base,
                   double full, double cscale, double tol, uint64_t max_iter,
                   int fixed_order, double* phi, uint64_t* iters,
                   double* resid, int* converged) {
  return guard([&] {
    MaskBlock mb;
    mb.num_players = n;
    mb.num_rows = rows;
    mb.words_per_row = words;
    mb.global_pair_count = rows / 2;
    for (uint64_t j = 0; j < rows / 2; ++j) mb.global_pairs.push_back(j);
    mb.bits.assign(bits, bits + rows * words);
    WlsProblem p = assemble_problem(mb, {values, rows}, base, full, cscale);
    auto comm = make_local_communicator();
    CglsOptions o;
    o.tol = tol;
    o.max_iter = max_iter;
    o.fixed_order = fixed_order != 0;
    CglsResult r = solve_cgls(p, *comm, o);
    std::memcpy(phi, r.phi.data(), n * 8);
    *iters = r.iterations;
    *resid = r.relative_residual;
    *converged = r.converged ? 1 : 0;
  });
}

// solver.cpp:364-428
int ref_solve_direct(uint32_t n, const uint64_t* bits, uint64_t rows,
                     uint64_t words, const double* values, double base,
                     double full, double cscale, double* phi) {
  return guard([&] {
    MaskBlock mb;
    mb.num_players = n;
    mb.num_rows = rows;
    mb.words_per_row = words;
    mb.global_pair_count = rows / 2;
    mb.bits.assign(bits, bits + rows * words);
    WlsProblem p = assemble_problem(mb, {values, rows}, base, full, cscale);
    std::vector<double> r = solve_direct(p);
    std::memcpy(phi, r.data(), n * 8);
  });
}

// oracle.cpp:41-60
int ref_exact_shapley_gnn(void* m, void* cg, uint32_t cls, double* phi) {
  return guard([&] {
    std::vector<double> r =
        exact_shapley_gnn(*static_cast<GcnModel*>(m),
                          *static_cast<ComputationalGraph*>(cg), cls);
    std::memcpy(phi, r.data(), r.size() * 8);
  });
}

// fidelity.cpp:51-65
int ref_fidelity_plus(void* m, void* cg, uint32_t cls, const uint32_t* sel,
                      uint64_t nsel, double* out) {
  return guard([&] {
    *out = fidelity_plus(*static_cast<GcnModel*>(m),
                         *static_cast<ComputationalGraph*>(cg), cls,
                         {sel, nsel});
  });
}

// fidelity.cpp:126-162; outputs sized by the counts/sparsities given
int ref_evaluate_fidelity(void* m, void* cg, uint32_t cls, const double* phi,
                          uint64_t n, const uint32_t* counts, uint64_t ncounts,
                          const double* sparsities, uint64_t nsp, uint64_t seed,
                          uint32_t trials, double* plus, double* plus_random,
                          double* minus, double* minus_random) {
  return guard([&] {
    FidelityReport r = evaluate_fidelity(
        *static_cast<GcnModel*>(m), *static_cast<ComputationalGraph*>(cg), cls,
        {phi, n}, {counts, ncounts}, {sparsities, nsp}, seed, trials);
    for (uint64_t i = 0; i < ncounts; ++i) {
      plus[i] = r.plus[i];
      plus_random[i] = r.plus_random[i];
    }
    for (uint64_t i = 0; i < nsp; ++i) {
      minus[i] = r.minus[i];
      minus_random[i] = r.minus_random[i];
    }
  });
}

// ---------------------------------------------------------------- explain
// explain.cpp:42-143 under run_on_thread_workers(world) (comm.cpp:448-455).
// meta[]: 0 class, 1 base, 2 full, 3 iterations, 4 residual, 5 converged,
// 6 rows, 7 exhaustive, 8 sampling_ms, 9 prediction_ms, 10 solve_ms,
// 11 total_ms, 12 n, 13.. fidelity plus for top_counts {5,10,20} (3 values)
int ref_explain_node(void* g, void* m, uint32_t node, uint64_t samples,
                     uint64_t batch, uint64_t seed, double tol,
                     uint64_t max_iter, int allow_exhaustive, int fidelity,
                     uint32_t trials, int world, double* phi, uint64_t phi_cap,
                     double* meta) {
  return guard([&] {
    ExplainOptions o;
    o.samples = samples;
    o.batch_size = batch;
    o.seed = seed;
    o.tol = tol;
    o.max_iter = max_iter;
    o.allow_exhaustive = allow_exhaustive != 0;
    o.fidelity = fidelity != 0;
    o.baseline_trials = trials;
    NodeExplanation out;
    std::mutex mu;
    run_on_thread_workers(world, [&](Communicator& comm) {
      NodeExplanation ex = explain_node(*static_cast<Graph*>(g),
                                        *static_cast<GcnModel*>(m), node, o,
                                        comm);
      if (comm.rank() == 0) {
        std::lock_guard<std::mutex> lock(mu);
        out = std::move(ex);
      }
    });
    if (out.phi.size() > phi_cap) throw DataError("phi buffer too small");
    std::memcpy(phi, out.phi.data(), out.phi.size() * 8);
    meta[0] = out.predicted_class;
    meta[1] = out.base_score;
    meta[2] = out.full_score;
    meta[3] = double(out.iterations);
    meta[4] = out.residual;
    meta[5] = out.converged ? 1.0 : 0.0;
    meta[6] = double(out.rows);
    meta[7] = out.exhaustive ? 1.0 : 0.0;
    meta[8] = out.timings.sampling_ms;
    meta[9] = out.timings.prediction_ms;
    meta[10] = out.timings.solve_ms;
    meta[11] = out.timings.total_ms;
    meta[12] = double(out.phi.size());
    for (int i = 0; i < 3; ++i) meta[13 + i] = -1.0;
    if (out.fidelity) {
      for (size_t i = 0; i < out.fidelity->plus.size() && i < 3; ++i)
        meta[13 + i] = out.fidelity->plus[i];
    }
  });
}

// CPU baseline for the sample + masked-inference metric on a bounded
// sample: `world` reference ranks on `world` host
// threads each run generate_masks for their full shard of the plan
// (sampler.cpp:153-210) and then predict_batched (gcn.cpp:259-270) on the
// first `infer_rows` rows of that shard. Times are wall clock between the
// barriers of run_on_thread_workers. out[]: 0 sampling_ms, 1 predict_ms,
// 2 rows predicted in total, 3 rows sampled in total.
int ref_sample_predict(void* m, void* cg, uint32_t cls, uint64_t k,
                       uint64_t seed, int world, uint64_t infer_rows,
                       uint64_t batch, int allow_exhaustive, double* out) {
  return guard([&] {
    const auto& model = *static_cast<GcnModel*>(m);
    const auto& sub = *static_cast<ComputationalGraph*>(cg);
    const auto n = static_cast<uint32_t>(sub.num_players());
    SizePlan plan = plan_sizes(n, k, allow_exhaustive != 0);
    double t_sample = 0, t_pred = 0;
    uint64_t predicted = 0, sampled = 0;
    std::mutex mu;
    run_on_thread_workers(world, [&](Communicator& comm) {
      comm.barrier();
      auto t0 = Clock::now();
      MaskBlock mb = generate_masks(plan, seed, comm.rank(), comm.world_size());
      comm.barrier();
      double ts = ms_since(t0);
      uint64_t r = std::min<uint64_t>(infer_rows, mb.num_rows);
      auto t1 = Clock::now();
      std::vector<float> p = predict_batched(
          model, sub, BitRows{mb.bits.data(), r, mb.words_per_row}, cls, batch);
      comm.barrier();
      double tp = ms_since(t1);
      std::lock_guard<std::mutex> lock(mu);
      predicted += r;
      sampled += mb.num_rows;
      if (comm.rank() == 0) {
        t_sample = ts;
        t_pred = tp;
      }
    });
    out[0] = t_sample;
    out[1] = t_pred;
    out[2] = double(predicted);
    out[3] = double(sampled);
  });
}

// explain.cpp:183-230 select_nodes
int ref_select_nodes(void* g, const char* rule, uint32_t* out, uint64_t cap, uint64_t* count) {
  return guard([&] {
    const std::vector<uint32_t> sel = select_nodes(*static_cast<Graph*>(g), std::string(rule));
    *count = sel.size();
    for (uint64_t i = 0; i < sel.size() && i < cap; ++i) out[i] = sel[i];
  });
}

}  // extern "C"
