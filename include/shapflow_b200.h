/*
 * shapflow_b200 — C-ABI of the B200-native DistShap explanation hot path
 * (coalition sampler -> masked GCN inference -> weighted least squares).
 *
 * Plain pointers and sizes only. Every entry point returns an int status
 * that maps onto the reference's exception types (error.hpp:10-27):
 *   SF_OK 0, SF_ERR_INTERNAL 1 (CUDA / allocation), SF_ERR_DATA 2
 *   (DataError), SF_ERR_NUMERICAL 3 (NumericalError), SF_ERR_PROTOCOL 4
 *   (ProtocolError). sf_last_error() returns the thread-local message.
 * The C++ drop-in (include/shapflow_b200.hpp) rethrows the matching type.
 *
 * Each declaration cites the reference interface it replaces
 * (paths relative to /root/reference/proj/core).
 */
#ifndef SHAPFLOW_B200_H
#define SHAPFLOW_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  SF_OK = 0,
  SF_ERR_INTERNAL = 1,
  SF_ERR_DATA = 2,
  SF_ERR_NUMERICAL = 3,
  SF_ERR_PROTOCOL = 4
};

typedef struct sf_ctx sf_ctx;           /* one rank = one GPU + stream + comm */
typedef struct sf_graph sf_graph;       /* graph.hpp:16-31  Graph */
typedef struct sf_model sf_model;       /* gcn.hpp:13-30    GcnModel */
typedef struct sf_subgraph sf_subgraph; /* graph.hpp:36-53  ComputationalGraph */
typedef struct sf_dmasks sf_dmasks;     /* sampler.hpp:55-78 MaskBlock, in HBM */

const char* sf_last_error(void);
const char* sf_version(void);

/* ------------------------------------------------------------ context
 * A context owns one CUDA device, one stream and (optionally) one NCCL
 * communicator; it replaces the reference's per-rank Communicator
 * (comm.hpp:28-52) for the hot path. */
int sf_ctx_create(int device, sf_ctx** out);
int sf_ctx_destroy(sf_ctx* ctx);
int sf_ctx_rank(const sf_ctx* ctx);
int sf_ctx_world(const sf_ctx* ctx);
/* NCCL over NVLink: 128-byte ncclUniqueId from rank 0, shared by the caller
 * (e.g. through torch.distributed), then every rank joins. */
int sf_nccl_unique_id(void* out_128_bytes);
int sf_ctx_join_nccl(sf_ctx* ctx, const void* unique_id_128, int rank,
                     int world);
/* A caller-provided communicator instead of NCCL (the reference's
 * Communicator behind the ABI: thread or socket workers, comm.hpp:28-52).
 * all_reduce sums `count` doubles in place across ranks, barrier waits for
 * every rank; both return 0 on success. The library stages device buffers
 * through pinned host memory for each call. Replaces any NCCL communicator.
 * With world == 1 the hooks are still called (buf == NULL for all_reduce:
 * the sum is the identity) so the caller's collective accounting matches. */
int sf_ctx_set_host_comm(sf_ctx* ctx, int rank, int world, void* user,
                         int (*all_reduce)(void* user, double* buf,
                                           uint64_t count),
                         int (*barrier)(void* user));
/* Communicator::all_reduce_sum on a host span through the context's
 * communicator (NCCL or host); counted in the context stats. */
int sf_ctx_allreduce_host(sf_ctx* ctx, double* buf, uint64_t count);
/* Bound on a collective's wait (default 60000 ms, the reference's
 * kDefaultCommTimeout, comm.hpp:54). A rank that never joins aborts the NCCL
 * communicator and the call fails with SF_ERR_PROTOCOL. */
int sf_ctx_set_comm_timeout(sf_ctx* ctx, int timeout_ms);
/* CollectiveStats (comm.hpp:13-19) */
int sf_ctx_stats(const sf_ctx* ctx, uint64_t* scalar_allreduce,
                 uint64_t* vector_allreduce, uint64_t* barriers,
                 uint64_t* doubles_reduced);
int sf_ctx_barrier(sf_ctx* ctx); /* Communicator::barrier (comm.hpp:37) */
/* kernel launches issued by this context so far (for bench accounting) */
uint64_t sf_ctx_launches(const sf_ctx* ctx);
/* host<->device bytes copied by this context so far */
int sf_ctx_io_bytes(const sf_ctx* ctx, uint64_t* h2d, uint64_t* d2h);
/* CUDA-event timers on the context stream (slots 0..7) */
int sf_ctx_event_record(sf_ctx* ctx, int slot);
int sf_ctx_event_elapsed(sf_ctx* ctx, int from_slot, int to_slot, float* ms);
int sf_ctx_synchronize(sf_ctx* ctx);
/* Fused layer-0/1 kernel selection for this context (no reference
 * counterpart; the reference has one CPU kernel, gcn.cpp:96-160):
 * SF_KERNEL_AUTO = tcgen05 3xTF32 where the hidden width allows (env
 * SF_FUSED_TC=0 forces SIMT), SF_KERNEL_SIMT = FP32 SIMT kernel,
 * SF_KERNEL_TC = tcgen05 where possible. Takes effect on the next call. */
enum { SF_KERNEL_AUTO = 0, SF_KERNEL_SIMT = 1, SF_KERNEL_TC = 2, SF_KERNEL_TC16 = 3 };
int sf_ctx_set_fused_kernel(sf_ctx* ctx, int kind);
/* which fused kernel the last prediction used: 0 none, 1 SIMT, 2 tcgen05
 * 3xTF32, 3 tcgen05 fp16x2 (SF_KERNEL_TC16: opt-in variant, widths 64/128) */
int sf_ctx_fused_kernel_used(const sf_ctx* ctx);
/* Plan of the fused kernel prepared by the last prediction: layer-0 entries
 * gathered per coalition (with the fused recompute), the same padded to the
 * tcgen05 K granularity (0 on the SIMT kernel), work items, hidden width. */
int sf_ctx_fused_plan(const sf_ctx* ctx, uint64_t* entries,
                      uint64_t* padded_entries, uint32_t* items,
                      uint32_t* width);
/* Per-launch timing of the dominant kernel (layer-0 masked SpMM): enable,
 * run work, then read the summed duration (ms), launch count and the
 * complement pairs those launches covered. */
int sf_ctx_time_dominant(sf_ctx* ctx, int enable);
int sf_ctx_dominant_stats(sf_ctx* ctx, double* total_ms, uint64_t* launches,
                          uint64_t* pairs);
/* Stage outputs for stage-wise parity checks (no reference counterpart;
 * the reference's explain.cpp:100-102 keeps its predictions in a local):
 * with keep on, sf_explain_node retains this rank's predictions of the node
 * (rank-local row order, rows 2j / 2j+1 of local pair j) on the host;
 * sf_ctx_stage_predictions copies them out (NULL `out` to query *rows). */
int sf_ctx_keep_stages(sf_ctx* ctx, int enable);
int sf_ctx_stage_predictions(const sf_ctx* ctx, float* out, uint64_t cap,
                             uint64_t* rows);
/* Algorithmic bytes of the masked SpMM per complement pair for a
 * (subgraph, model): (sum_{u in R} deg(u) + 2|R|) d 4
 * gathered + 2|R| d 4 written + 2 W 8 mask, R = rows layer 0 produces. */
int sf_spmm_bytes_per_pair(const sf_model* m, const sf_subgraph* sg,
                           double* bytes, double* flops);

/* ------------------------------------------------------------ primitives */
/* explain.cpp:37-40 */
uint64_t sf_node_sampling_seed(uint64_t seed, uint32_t node);
/* explain.cpp:33-35 */
uint64_t sf_auto_samples(uint64_t num_players);
/* sampler.cpp:67-77 */
uint64_t sf_binomial_or_max(uint32_t n, uint32_t s);
/* sampler.cpp:79-91 */
int sf_kernel_weight(uint32_t n, uint32_t s, double* out);
/* Philox-4x32-10 stream (philox.hpp:13-73) generated ON THE DEVICE; used to
 * pin the device generator bit-for-bit. */
int sf_philox_u64(sf_ctx* ctx, uint64_t seed, uint64_t stream, uint64_t count,
                  uint64_t* out_host);

/* sampler.hpp:49-50 plan_sizes. Arrays of capacity `cap` (n/2 suffices);
 * pass NULL arrays to query *nclasses. */
int sf_plan_sizes(uint32_t n, uint64_t k, int allow_exhaustive,
                  uint32_t* sizes, uint64_t* pairs, uint64_t* first_pair,
                  uint64_t cap, uint64_t* nclasses, int* exhaustive,
                  uint64_t* requested);

/* sampler.hpp:84-85 generate_masks for the plan (sizes/pairs/first_pair as
 * returned by sf_plan_sizes): this rank's pairs g = rank, rank+world, ...,
 * row 2j kept-set of local pair j, row 2j+1 its complement; u64 words, bit e
 * = player e, words_for_bits(n) words per row, row-major. Generated on the
 * GPU and copied into out_host (capacity cap_words; NULL to query *rows).
 * rows_of_size (n+1 entries, may be NULL) receives global_rows_of_size. */
int sf_generate_masks(sf_ctx* ctx, uint32_t n, const uint32_t* sizes,
                      const uint64_t* pairs, const uint64_t* first_pair,
                      uint64_t nclasses, int exhaustive, uint64_t seed,
                      int rank, int world, uint64_t* out_host,
                      uint64_t cap_words, uint64_t* rows,
                      uint64_t* rows_of_size);

/* Device-resident stages (the reference's explain.cpp:91-114 sequence
 * generate_masks -> predict_batched -> assemble_problem -> solve_cgls without
 * moving the mask block across PCIe). sf_masks_device samples this rank's
 * pairs into HBM, one kept-set row per pair (the complement rows are derived
 * by every consumer); sf_dmasks_download expands them into the reference's
 * MaskBlock.bits layout (rows 2j, 2j+1) on the host. */
int sf_masks_device(sf_ctx* ctx, uint32_t n, const uint32_t* sizes,
                    const uint64_t* pairs, const uint64_t* first_pair,
                    uint64_t nclasses, int exhaustive, uint64_t seed, int rank,
                    int world, sf_dmasks** out);
/* rows (2 per local pair), player count, global rows per size (n+1, may be NULL) */
int sf_dmasks_info(const sf_dmasks* m, uint64_t* rows, uint32_t* num_players,
                   uint64_t* rows_of_size);
int sf_dmasks_download(sf_ctx* ctx, const sf_dmasks* m, uint64_t* out_host,
                       uint64_t cap_words);
int sf_dmasks_free(sf_dmasks* m);
/* gcn.hpp:60-62 predict_batched over device masks: p[class] per row to the host */
int sf_predict_dmasks(sf_ctx* ctx, const sf_model* m, const sf_subgraph* sg,
                      const sf_dmasks* masks, uint32_t class_index,
                      uint64_t batch_size, float* out);
/* solver.hpp:46-49 assemble_problem + 94-95 solve_cgls over device masks:
 * values[row] the model outputs (float, as predict_batched returns them),
 * base / full the empty / full outputs; mode as sf_solve_cgls. Collective
 * over the context's ranks. */
int sf_solve_dmasks(sf_ctx* ctx, const sf_dmasks* masks, const float* values,
                    double base, double full, double constraint_scale,
                    double tol, uint64_t max_iter, int mode, double* phi,
                    uint64_t* iterations, double* relative_residual,
                    int* converged);

/* ------------------------------------------------------------ graph + model */
/* graph.hpp:57-60 build_graph: symmetrize, dedupe, drop self-loops.
 * edges_uv: num_edges (u, v) pairs; labels may be NULL (kNoLabel). */
int sf_graph_build(uint32_t num_nodes, const uint64_t* edges_uv,
                   uint64_t num_edges, const float* features,
                   uint64_t feature_dim, const uint32_t* labels,
                   sf_graph** out);
/* graph.hpp:64 load_graph, binary SFG1 (graph.cpp:35-64) */
int sf_graph_load(const char* path, sf_graph** out);
/* An already-built symmetric CSR (Graph, graph.hpp:16-31: rows sorted, no
 * duplicates, both directions stored) taken as-is; labels may be NULL. */
int sf_graph_from_csr(uint32_t num_nodes, const uint64_t* row_ptr,
                      const uint32_t* col, const float* features,
                      uint64_t feature_dim, const uint32_t* labels,
                      sf_graph** out);
/* graph.hpp:65 save_graph (graph.cpp:171-193) */
int sf_graph_save(const sf_graph* g, const char* path);
int sf_graph_free(sf_graph* g);
int sf_graph_dims(const sf_graph* g, uint32_t* num_nodes, uint64_t* nnz,
                  uint64_t* feature_dim);
int sf_graph_csr(const sf_graph* g, uint64_t* row_ptr, uint32_t* col);

/* gcn.hpp:13-30: L layers, dims[0..L], weights concatenated per layer
 * (in x out row-major), biases concatenated. */
int sf_model_create(int L, const uint64_t* dims, const float* weights,
                    const float* biases, sf_model** out);
/* synthetic.hpp:25-27 gen_random_model (Glorot, Philox stream 16+l) */
int sf_model_random(uint64_t input_dim, const uint64_t* hidden, int nh,
                    uint32_t classes, uint64_t seed, sf_model** out);
int sf_model_free(sf_model* m);
int sf_model_dims(const sf_model* m, int* L, uint64_t* dims /* L+1 */);
int sf_model_layer(const sf_model* m, int l, float* weight, float* bias);

/* graph.hpp:69-70 extract_computational_graph (BFS ball, local ids in
 * discovery order, players sorted, symmetric local CSR with edge_player) */
int sf_extract(const sf_graph* g, uint32_t target, int hops,
               sf_subgraph** out);
/* graph.hpp:69-70 extract_computational_graph on the device (level-
 * synchronous BFS with the reference's discovery order, segmented sorts for
 * the local CSR): byte-identical to sf_extract; explain_node uses it for
 * graphs with >= 2^20 CSR entries (env SF_EXTRACT=host|device|auto). */
int sf_extract_device(sf_ctx* ctx, const sf_graph* g, uint32_t target,
                      int hops, sf_subgraph** out);
int sf_subgraph_free(sf_subgraph* sg);
/* A ComputationalGraph built by the caller (graph.hpp:36-53 layout: local
 * ids BFS order, players_uv 2n local endpoints u < v sorted, symmetric CSR
 * with edge_player, V x dim features). */
int sf_subgraph_create(uint32_t target_global, uint32_t V, uint64_t n,
                       const uint64_t* row_ptr, const uint32_t* col,
                       const uint32_t* edge_player, const uint32_t* players_uv,
                       const uint32_t* local_to_global, const float* features,
                       uint64_t feature_dim, sf_subgraph** out);
int sf_subgraph_dims(const sf_subgraph* sg, uint32_t* V, uint64_t* n,
                     uint64_t* nnz, uint64_t* feature_dim);
int sf_subgraph_copy(const sf_subgraph* sg, uint64_t* row_ptr, uint32_t* col,
                     uint32_t* edge_player, uint32_t* players_uv,
                     uint32_t* local_to_global, float* features);
/* |B_h| for h = 0..hops (local ids are BFS order, so each ball is a prefix) */
int sf_subgraph_ball_sizes(const sf_subgraph* sg, int hops, uint64_t* sizes);

/* ------------------------------------------------------------ inference */
/* gcn.hpp:60-62 predict_batched: p[class_index] per mask row (host rows in,
 * host floats out). batch_size is validated like the reference (> 0) but
 * does not change results: the device engine tiles coalitions itself. */
int sf_predict_batched(sf_ctx* ctx, const sf_model* m, const sf_subgraph* sg,
                       const uint64_t* bits, uint64_t rows,
                       uint64_t words_per_row, uint32_t class_index,
                       uint64_t batch_size, float* out);
/* gcn.hpp:50-51 predict_probs: all class probabilities for one mask */
int sf_predict_probs(sf_ctx* ctx, const sf_model* m, const sf_subgraph* sg,
                     const uint64_t* mask, uint64_t words, float* probs);

/* ------------------------------------------------------------ solver */
/* solver.hpp:82-95 solve_cgls on an assembled system whose rows are 0/1
 * bit rows (WlsProblem.rows packed; row i = bits[i*words ...]).
 * weights (per row, normalized) and targets (per row, value - base) as in
 * WlsProblem (solver.hpp:22-38). Collective across the context's ranks.
 * mode: 0 = reference protocol (1 vector + 1 scalar all-reduce per
 * iteration, solver.hpp:82-85), 1 = fused (one (n+1)-double all-reduce per
 * iteration), 2 = reference protocol with fixed-order (exact, layout-
 * independent) sums: CglsOptions::fixed_order (solver.hpp:62-65), phi
 * bitwise identical for any worker count; it adds one all-reduce at init and
 * sends delta as 3 doubles. trace != 0 records per-iteration residuals (out arrays of
 * capacity trace_cap, may be NULL). */
int sf_solve_cgls(sf_ctx* ctx, uint32_t n, const uint64_t* bits,
                  uint64_t rows, uint64_t words, const double* weights,
                  const double* targets, double constraint_target,
                  double constraint_weight, double tol, uint64_t max_iter,
                  int mode, double* phi, uint64_t* iterations,
                  double* relative_residual, int* converged,
                  double* trace, double* row_residual_trace,
                  uint64_t trace_cap);
/* sf_solve_cgls for one rank's slice of a multi-rank system: the global
 * pair count (WlsProblem::global_pair_count, solver.hpp:17-18) sizes the
 * fixed-order tree identically on every rank (mode 2). sf_solve_cgls
 * assumes the rows are the whole system. */
int sf_solve_cgls_ex(sf_ctx* ctx, uint32_t n, const uint64_t* bits,
                     uint64_t rows, uint64_t words, const double* weights,
                     const double* targets, double constraint_target,
                     double constraint_weight, double tol, uint64_t max_iter,
                     int mode, uint64_t global_pair_count, double* phi,
                     uint64_t* iterations, double* relative_residual,
                     int* converged, double* trace, double* row_residual_trace,
                     uint64_t trace_cap);
/* solver.hpp:46-49 assemble_problem weights: per-row normalized weight
 * from the global per-size row counts (solver.cpp:125-138). */
int sf_assemble_weights(uint32_t n, const uint64_t* bits, uint64_t rows,
                        uint64_t words, const uint64_t* rows_of_size,
                        double* weights);
/* solver.hpp:100 solve_direct: dense normal equations (Gram built on the
 * GPU from the bit rows, Cholesky), n <= 20000, world 1. */
int sf_solve_direct(sf_ctx* ctx, uint32_t n, const uint64_t* bits,
                    uint64_t rows, uint64_t words, const double* weights,
                    const double* targets, double constraint_target,
                    double constraint_weight, double* phi);
/* solver.hpp:109 rank_edges: descending phi, ties to the smaller index */
int sf_rank_edges(const double* phi, uint64_t n, uint32_t* order);

/* ------------------------------------------------------------ pipeline */
/* Solver of explain_node: SF_SOLVER_CGLS = reference CGLS protocol
 * (solver.hpp:82-95: 1 vector + 1 scalar all-reduce per iteration),
 * SF_SOLVER_FUSED = CGLS with one (n+1)-double all-reduce per iteration,
 * SF_SOLVER_DIRECT = normal equations (tcgen05 Gram + device Cholesky,
 * solve_direct semantics, one worker), SF_SOLVER_AUTO (default) = DIRECT
 * when one worker holds the system and n <= 256 (env SF_DIRECT_MAX), else
 * CGLS. DIRECT reports iterations 0 and residual 0. */
enum { SF_SOLVER_CGLS = 0, SF_SOLVER_FUSED = 1, SF_SOLVER_DIRECT = 2, SF_SOLVER_AUTO = 3 };

/* explain.hpp:15-32 ExplainOptions */
typedef struct sf_explain_options {
  uint64_t samples;         /* 0: sf_auto_samples(n) */
  uint64_t batch_size;      /* validated, > 0 */
  uint32_t top_k;
  uint64_t seed;
  double tol;
  uint64_t max_iter;        /* 0: min(n, 5000) */
  uint64_t player_cap;      /* 0: no cap */
  int allow_exhaustive;
  double constraint_scale;
  int fidelity;
  uint32_t baseline_trials;
  int solver_mode;          /* SF_SOLVER_* below */
  const uint32_t* top_counts; /* default {5,10,20} when NULL */
  uint32_t num_top_counts;
  const double* sparsities;   /* default {.1,.3,.5,.7,.9} when NULL */
  uint32_t num_sparsities;
  /* ExplainOptions::fixed_order (explain.hpp:31): CGLS sums in a
   * layout-independent (exact) order, phi bitwise identical for any worker
   * count; costs 3 passes per transpose/forward product. Default 0. */
  int fixed_order;
} sf_explain_options;

void sf_explain_options_default(sf_explain_options* o);

/* document.hpp:22-44 NodeExplanation (+ fidelity.hpp:36-51). Arrays are
 * owned by the library and released by sf_explanation_free. */
typedef struct sf_explanation {
  uint32_t node;
  int skipped;
  uint32_t predicted_class;
  double base_score, full_score;
  uint64_t num_players;
  double* phi;              /* num_players */
  uint32_t* players_global; /* 2 * num_players, smaller id first */
  int exhaustive;
  uint64_t rows;
  uint32_t iterations;
  double residual;
  int converged;
  uint32_t num_top;
  uint32_t* top_player;
  double* top_phi;
  int has_fidelity;
  uint32_t num_counts;
  uint32_t* fid_counts;
  double* fid_plus;
  double* fid_plus_random;
  uint32_t num_sparsities;
  double* fid_sparsities;
  double* fid_minus;
  double* fid_minus_random;
  double sampling_ms, prediction_ms, solve_ms, total_ms;
  /* host-side stage timings: subgraph extraction, full/empty scores (engine
   * preparation included), Fidelity+ evaluation */
  double extract_ms, setup_ms, fidelity_ms;
  char warning[512];
} sf_explanation;

/* explain.hpp:47-49 explain_node, collective over the context's ranks */
int sf_explain_node(sf_ctx* ctx, const sf_graph* g, const sf_model* m,
                    uint32_t node, const sf_explain_options* opts,
                    sf_explanation* out);
int sf_explanation_free(sf_explanation* e);

/* explain.hpp:54-57 explain_nodes: explain_node per node in order (each
 * collective over the context's ranks); errors are prefixed "node N: "
 * (explain.cpp:168-180) and every filled entry is freed on error. `out`
 * holds `count` entries, each released with sf_explanation_free. */
int sf_explain_nodes(sf_ctx* ctx, const sf_graph* g, const sf_model* m,
                     const uint32_t* nodes, uint64_t count,
                     const sf_explain_options* opts, sf_explanation* out);

/* Device memory in use on the context's GPU (all allocations of the
 * process, cudaMemGetInfo) and its capacity, in bytes. */
int sf_ctx_device_memory(const sf_ctx* ctx, uint64_t* used, uint64_t* total);

/* Concurrent targets for sf_explain_nodes on a one-worker context (no
 * reference counterpart; the reference loops over nodes, explain.cpp:145-181):
 * `workers` contexts on this device (own stream and buffers, created on
 * first use) each take the next target from a shared counter, so one
 * target's CGLS overlaps another's sampling and inference. Results per
 * target are unchanged; errors report the lowest failing node. 1..16,
 * default 1. Ignored for multi-rank contexts (every rank must run the same
 * collective sequence). */
int sf_ctx_set_workers(sf_ctx* ctx, int workers);

/* explain.hpp:59-64 select_nodes: "degree-range:[lo,hi]:count" (first
 * `count` ids in ascending order with degree in [lo, hi]) or a comma
 * separated id list. Writes up to `cap` ids, *count = number selected. */
int sf_select_nodes(const sf_graph* g, const char* rule, uint32_t* out,
                    uint64_t cap, uint64_t* count);

/* fidelity.hpp:45-51 evaluate_fidelity on the device engine */
int sf_evaluate_fidelity(sf_ctx* ctx, const sf_model* m, const sf_subgraph* sg,
                         uint32_t class_index, const double* phi,
                         const uint32_t* top_counts, uint32_t num_counts,
                         const double* sparsities, uint32_t num_sparsities,
                         uint64_t seed, uint32_t trials, uint32_t* counts_out,
                         double* plus, double* plus_random, double* minus,
                         double* minus_random);

/* ------------------------------------------------------------ bench hooks
 * Device-resident sample + masked inference for one target (the
 * coalitions/s metric): samples this rank's shard on the GPU and scores it,
 * leaving masks and predictions in HBM. Times (ms, CUDA events on the
 * context stream) are written to stage_ms[0..1] = {sampling, prediction}
 * and the dominant kernel's summed duration to stage_ms[2] (may be NULL). */
int sf_sample_and_predict(sf_ctx* ctx, const sf_model* m, const sf_subgraph* sg,
                          uint32_t class_index, uint64_t k, uint64_t seed,
                          int allow_exhaustive, double* stage_ms,
                          uint64_t* rows_local);

#ifdef __cplusplus
}
#endif
#endif /* SHAPFLOW_B200_H */
