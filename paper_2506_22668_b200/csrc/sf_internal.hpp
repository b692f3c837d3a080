// Internal declarations shared by the host C++ and the CUDA translation
// units of libshapflow_b200. Not part of the public ABI.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>
#include <cstdlib>
#include <chrono>

namespace sfb {

// ---------------------------------------------------------------- errors
// Mirror of the reference exception types (error.hpp:10-27); the C-ABI maps
// them to status codes 2/3/4 and CUDA failures to 1.
struct DataError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NumericalError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ProtocolError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void cuda_check(cudaError_t e, const char* what, const char* file,
                       int line) {
  if (e != cudaSuccess)
    throw CudaError(std::string(what) + " failed at " + file + ":" +
                    std::to_string(line) + ": " + cudaGetErrorString(e));
}
#define SF_CUDA(x) ::sfb::cuda_check((x), #x, __FILE__, __LINE__)
#define SF_LAUNCHED(ctx)                                                  \
  do {                                                                    \
    ::sfb::cuda_check(cudaGetLastError(), "kernel launch", __FILE__,      \
                      __LINE__);                                          \
    (ctx).launches++;                                                     \
  } while (0)

// cudaFuncSetAttribute applies to the current device only; remember which
// (kernel, device, bytes) combinations are set so one process can drive
// several devices (thread-per-GPU ranks).
void set_max_dynamic_smem(const void* kernel, int bytes);
template <class K>
inline void set_max_dynamic_smem(K* kernel, int bytes) {
  set_max_dynamic_smem(reinterpret_cast<const void*>(kernel), bytes);
}

inline uint64_t next_object_id() {
  static std::atomic<uint64_t> id{1};
  return id++;
}

// ---------------------------------------------------------------- host data
struct Graph {  // graph.hpp:16-31
  uint64_t id = next_object_id();
  uint32_t num_nodes = 0;
  uint64_t feature_dim = 0;
  std::vector<uint64_t> row_ptr;
  std::vector<uint32_t> col;
  std::vector<float> features;
  std::vector<uint32_t> labels;
};

struct Layer {
  uint64_t in = 0, out = 0;
  std::vector<float> weight;  // in x out
  std::vector<float> bias;
};

struct Model {  // gcn.hpp:13-30
  uint64_t id = next_object_id();
  std::vector<Layer> layers;
  int depth() const { return static_cast<int>(layers.size()); }
};

struct Subgraph {  // graph.hpp:36-53
  uint64_t id = next_object_id();
  uint32_t target_global = 0;
  uint64_t feature_dim = 0;
  std::vector<uint32_t> local_to_global;
  std::vector<std::pair<uint32_t, uint32_t>> players;
  std::vector<uint64_t> row_ptr;
  std::vector<uint32_t> col;
  std::vector<uint32_t> edge_player;
  std::vector<float> features;  // empty when `source` is set (explain path)
  const Graph* source = nullptr;  // features gathered on the device from this graph
  uint32_t num_nodes() const {
    return static_cast<uint32_t>(local_to_global.size());
  }
  uint64_t num_players() const { return players.size(); }
  // |B_h|, h = 0..H: local ids are BFS discovery order, so balls are prefixes
  std::vector<uint64_t> ball_sizes(int hops) const;
};

// ---------------------------------------------------------------- device mem
template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;  // capacity in elements
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  void reserve(size_t count) {
    if (count <= n) return;
    release();
    SF_CUDA(cudaMalloc(&p, sizeof(T) * (count ? count : 1)));
    n = count;
  }
  void upload(const T* src, size_t count, cudaStream_t s) {
    reserve(count);
    if (count)
      SF_CUDA(cudaMemcpyAsync(p, src, sizeof(T) * count,
                              cudaMemcpyHostToDevice, s));
  }
};

template <typename T>
struct PinnedBuf {  // page-locked host staging
  T* p = nullptr;
  size_t n = 0;
  PinnedBuf() = default;
  PinnedBuf(const PinnedBuf&) = delete;
  PinnedBuf& operator=(const PinnedBuf&) = delete;
  ~PinnedBuf() {
    if (p) cudaFreeHost(p);
  }
  void reserve(size_t count) {
    if (count <= n) return;
    if (p) cudaFreeHost(p);
    p = nullptr;
    SF_CUDA(cudaMallocHost(&p, sizeof(T) * (count ? count : 1)));
    n = count;
  }
};

// Device-resident copy of one (subgraph, model) pair: the inputs of the
// masked-inference engine.
struct Engine {
  uint64_t sg_id = 0, model_id = 0;
  int kind = 0;  // Ctx::fused_kind the engine was prepared for
  uint32_t V = 0;
  uint64_t n = 0;
  uint32_t W = 0;  // u64 words per mask row
  int L = 0;
  std::vector<uint64_t> dims;       // d_0..d_L
  std::vector<uint64_t> ball;       // |B_h|, h = 0..L
  DevBuf<uint32_t> row_ptr, col, edge_player;
  DevBuf<uint32_t> isd_order;  // nodes by descending degree (isd_kernel)
  uint32_t isd_nbig = 0;       // nodes with more than 32 incidences
  DevBuf<float> isd_tab;       // inv_sqrt_deg(d), d = 0..maxdeg+1
  uint32_t isd_tab_n = 0;      // entries in isd_tab
  DevBuf<float> p0;                 // X W_0, V x d_1 (layer-0 transform-first)
  std::vector<std::unique_ptr<DevBuf<float>>> w, b;  // per layer (w[0] unused)
  // Fused layer-0 + layer-1 aggregation plan:
  // rows U = B_{L-2} (prefix of local ids); for each u in U the segments
  // v in {u} u N(u) (self first, CSR order), each segment the entries
  // {v} u N(v) whose P0 rows layer 0 gathers. Work items are contiguous
  // segment ranges of one u, balanced by entry count.
  bool fused = false;
  uint32_t U = 0, items = 0;
  uint64_t entries = 0;
  DevBuf<uint32_t> ent;  // 4 words per entry: x, e, e_uv, flags
  DevBuf<uint32_t> item_ent, item_order, u_items;
  // tensor-core (tcgen05) plan: segments padded to 8 entries (sf_fused_tc.cu)
  bool tc = false;
  uint32_t tc_items = 0;
  uint64_t tc_entries = 0;  // padded entries (K of the per-tile MMA chain)
  uint32_t tc_kstep = 8;    // entries per MMA k-step: 8 (tf32 kernel), 16 (fp16 kernel)
  DevBuf<float> tc_bbank;          // per chunk: K-major tf32 hi | lo B tile (3xTF32 kernel)
  DevBuf<uint32_t> tc_item_chunk;  // first B-bank chunk of each item
  DevBuf<uint32_t> tc_chunk_ent;   // per chunk: first entry, entry count
  bool tc16 = false;        // fp16x2 kernel (sf_fused_f16.cu) instead of 3xTF32
  DevBuf<uint16_t> p16;     // P0 split into fp16 hi | lo planes per row, scaled (fp16 kernel)
  DevBuf<float> p16_scale;  // [0] P0 scale (power of two), [1] its inverse
  DevBuf<uint32_t> tc_ent, tc_seg, tc_item_ent, tc_item_seg, tc_item_order, tc_u_items, tc_const;
  DevBuf<uint8_t> tc_kflags;
  // tensor-core tail (sf_tail_tc.cu): 3-layer, hidden 128/128
  bool tail_tc = false;         // tcgen05 tail available (W1 image built)
  bool tail_tc_always = false;  // SF_TAIL_TC=1: for every batch, not only >= 64 tile pairs
  // degrees as u16 rows + a 1/sqrt table instead of f32 isd rows for the
  // fused kernel (decided per predict call, engine_predict)
  bool deg_capable = false;  // tcgen05 3-layer path with the table in shared memory
  int deg_mode = 2;           // SF_ISD_U16: 0 never, 1 always, 2 with the mma.sync tail
  DevBuf<float> tail_w1img;  // W1 as a K-major tf32 hi | lo image
};

// SF_TIMING=1: host-side stage timings to stderr (debug aid, off by default)
struct DebugTimer {
  bool on;
  std::chrono::steady_clock::time_point t;
  const char* scope;
  explicit DebugTimer(const char* sc) : on(std::getenv("SF_TIMING") != nullptr), t(std::chrono::steady_clock::now()), scope(sc) {}
  void lap(const char* what) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    static const auto epoch = now;
    std::fprintf(stderr, "[timing] %10.3f %s %s %.3f ms\n",
                 std::chrono::duration<double, std::milli>(now - epoch).count(), scope, what,
                 std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

struct CommStats {  // comm.hpp:13-19
  uint64_t scalar_allreduce = 0, vector_allreduce = 0, barriers = 0,
           doubles_reduced = 0;
};

struct Nccl;  // dlopen'ed NCCL (sf_comm.cpp)

// A caller-provided host communicator (the reference's Communicator behind
// the C-ABI, e.g. thread or socket workers, comm.hpp:28-52): all-reduces of
// device buffers are staged through pinned host memory and handed to it.
struct HostComm {
  void* user = nullptr;
  int (*all_reduce)(void* user, double* buf, uint64_t count) = nullptr;
  int (*barrier)(void* user) = nullptr;
};

// device extraction state (sf_extract.cu): the graph CSR once per graph and
// scratch reused across targets
struct ExtractState {
  uint64_t graph_id = 0;
  DevBuf<uint64_t> rp, off, deg, lrp, cnt, ufirst, pstart, first;
  DevBuf<uint32_t> col, local_of, l2g, flag, pos, lcol_raw, lcol, ep, players;
  DevBuf<unsigned char> tmp;
};

// A second stream on the same device for work that overlaps the main
// stream's kernels (fork/join through the two events).
struct SideStream {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  SideStream() = default;
  SideStream(const SideStream&) = delete;
  SideStream& operator=(const SideStream&) = delete;
  ~SideStream() {
    if (fork) cudaEventDestroy(fork);
    if (join) cudaEventDestroy(join);
    if (s) cudaStreamDestroy(s);
  }
};

struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  SideStream side;  // CGLS: the sparse-pair list passes beside the dense-pair passes
  bool concurrent = false;  // one of several explain_nodes worker contexts right now
  int rank = 0, world = 1;
  std::unique_ptr<Nccl> nccl;
  HostComm host_comm;
  PinnedBuf<double> comm_stage;  // host staging for host_comm all-reduces
  int comm_timeout_ms = 60000;   // kDefaultCommTimeout (comm.hpp:54)
  CommStats stats;
  uint64_t launches = 0;
  int fused_kind = 0;  // SF_KERNEL_AUTO / SIMT / TC
  uint64_t h2d_bytes = 0, d2h_bytes = 0;  // host<->device traffic issued
  cudaEvent_t events[8] = {};             // bench timers on `stream`
  // dominant-kernel (layer-0 masked SpMM) timing: event pairs per launch,
  // read back after the work is done (no per-batch synchronization)
  bool time_dominant = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> dom_events;
  size_t dom_used = 0;
  uint64_t dom_pairs = 0;  // complement pairs covered by the timed launches
  Engine engine;
  // scratch reused across calls
  DevBuf<uint64_t> masks;      // row-major mask rows
  DevBuf<uint32_t> maskt;      // tile-transposed kept-set bits
  DevBuf<float> preds;
  DevBuf<unsigned char> work;  // engine workspace
  DevBuf<unsigned char> solver_work;
  DevBuf<unsigned char> solver_lists;  // CGLS kept-set lists of the sparse pairs
  DevBuf<uint64_t> solver_dense;       // CGLS dense pairs' even rows, word-major
  DevBuf<unsigned char> rank_work;     // rank_players scratch
  // sampler class table (pinned staging + device copy, reused per call)
  PinnedBuf<uint64_t> plan_host;
  PinnedBuf<uint32_t> plan_host32;
  DevBuf<uint64_t> plan_dev64;
  DevBuf<uint32_t> plan_dev32;
  cudaEvent_t plan_ready = nullptr;
  DevBuf<double> barrier_buf;
  // per-call scratch kept across calls (no allocation on the explain path)
  DevBuf<double> wsize_dev, sw_dev, tgt_dev;
  DevBuf<int> bad_dev;
  DevBuf<uint32_t> pop_dev;     // set bits per row (assemble_pairs)
  DevBuf<uint8_t> comp_dev;     // complement flag per pair
  PinnedBuf<double> solver_host;  // CGLS scalars fetched by the host loop
  PinnedBuf<uint32_t> cgls_hpop;  // CGLS setup: set bits per row, complement flags
  PinnedBuf<uint8_t> cgls_hcomp;
  DevBuf<float> feat_dev, w0_dev; // engine_prepare temporaries (X, W0 for P0 = X W0)
  DevBuf<float> graph_feat;       // device copy of a graph's features (explain path)
  uint64_t graph_feat_id = 0;     // Graph::id it holds
  DevBuf<uint32_t> ball_rows;     // local -> global node ids of the prepared subgraph
  DevBuf<uint64_t> fid_streams, fid_rows;  // fidelity random-baseline jobs
  DevBuf<uint32_t> fid_sizes;
  DevBuf<uint8_t> fid_inv;
  ExtractState extract;             // device extraction (large balls)
  DevBuf<float> tail_part;          // tcgen05 tail: per-u-range partial layer-2 aggregations
  DevBuf<uint32_t> tail_count;      // tcgen05 tail: arrivals per tile pair (last CTA finishes)
  DevBuf<uint64_t> gram_maskt;      // direct solve: tile-transposed rows
  DevBuf<unsigned char> gram_work;  // direct solve: plan, run weights, targets
  DevBuf<double> gram_g;            // direct solve: Gram partials, factor, copy, rhs
  // stage outputs retained for stage-wise parity checks (sf_ctx_keep_stages)
  bool keep_stages = false;
  std::vector<float> kept_preds;  // this rank's predictions of the last explain_node
  Ctx();
  ~Ctx();
};

// ---------------------------------------------------------------- comm
void nccl_unique_id(void* out128);
void nccl_join(Ctx& ctx, const void* id128, int rank, int world);
void comm_allreduce_sum(Ctx& ctx, double* dev_buf, size_t count);
void comm_barrier(Ctx& ctx);
void comm_drop_nccl(Ctx& ctx);
// Waits for the context stream; with a multi-rank NCCL communicator the wait
// is bounded by ctx.comm_timeout_ms (a rank that never joins a collective
// aborts the communicator and raises ProtocolError instead of hanging).
void comm_sync(Ctx& ctx);

// ---------------------------------------------------------------- plan
struct SizeClass {
  uint32_t size = 0;
  uint64_t pairs = 0, first_pair = 0;
};
struct SizePlan {
  uint32_t n = 0;
  uint64_t requested = 0;
  bool exhaustive = false;
  std::vector<SizeClass> classes;
  uint64_t total_pairs() const {
    return classes.empty() ? 0 : classes.back().first_pair + classes.back().pairs;
  }
};
SizePlan plan_sizes(uint32_t n, uint64_t k, bool allow_exhaustive);
uint64_t binomial_or_max(uint32_t n, uint32_t s);
std::vector<uint64_t> global_rows_of_size(const SizePlan& plan);
uint64_t local_pair_count(uint64_t global_pairs, int rank, int world);

// ---------------------------------------------------------------- kernels
// sf_sampler.cu
void launch_philox_stream(Ctx& ctx, uint64_t seed, uint64_t stream,
                          uint64_t count, uint64_t* dev_out);
// Generates this rank's rows (row-major, 2 rows per local pair) into
// dev_rows; also writes the tile-transposed kept-set layout when dev_maskt
// is non-null.
// kept_only: row j holds local pair j's kept-set only (W words per pair;
// the complement row is derived by every consumer) — half the mask bytes
void launch_generate_masks(Ctx& ctx, const SizePlan& plan, uint64_t seed,
                           int rank, int world, uint64_t* dev_rows, bool kept_only = false);
// kept-only pair rows -> tile layout with the complement rows interleaved
// (bit 2i = pair i kept, bit 2i+1 = its complement, players < n)
void launch_transpose_pairs(Ctx& ctx, const uint64_t* dev_kept, uint64_t pairs, uint32_t W, uint32_t n,
                            uint64_t tiles, uint64_t* dev_maskt);
// Independent Floyd draws (fidelity baselines, fidelity.cpp:25-33): row j
// is the size-sizes[j] subset drawn from Philox(seed, streams[j]), or the
// full row minus that subset when invert[j] != 0.
void launch_floyd_jobs(Ctx& ctx, uint32_t n, uint64_t seed,
                       const uint64_t* dev_streams, const uint32_t* dev_sizes,
                       const uint8_t* dev_invert, uint64_t jobs,
                       uint64_t* dev_rows);
// Row-major rows -> tile layout: maskt[t][e] bit i = row (row0+t*64+i)
// bit e, for all 64 rows of the tile (u32 pairs: low = rows 0..31).
void launch_transpose_tiles(Ctx& ctx, const uint64_t* dev_rows, uint64_t rows,
                            uint32_t W, uint64_t tiles, uint64_t* dev_maskt,
                            uint64_t stride = 0);  // words between rows (0: W)

// sf_gcn.cu
void engine_prepare(Ctx& ctx, const Subgraph& sg, const Model& m);
// Scores `rows` mask rows (row-major on device) into dev_probs (class
// `cls`) and, when dev_allprobs is non-null, every class probability.
void engine_predict(Ctx& ctx, const uint64_t* dev_rows, uint64_t rows,
                    uint32_t cls, float* dev_out, float* dev_allprobs,
                    float* dominant_ms, bool kept_only = false);

// sf_fused_tc.cu
bool tc_width(uint64_t d);

// sf_fused_f16.cu
bool tc16_width(uint64_t d);
uint32_t tc16_max_table();  // largest 1/sqrt(deg) table the fp16 kernel stages
void prepare_tc16(Ctx& ctx, Engine& e);  // P0 -> scaled fp16 hi/lo planes
bool launch_fused_tc16(Ctx& ctx, const Engine& e, const uint64_t* maskt, uint64_t Wp,
                       const float* isd, const uint16_t* deg16, uint64_t ntp, float* apart);
void build_tc_plan(Ctx& ctx, Engine& e, const Subgraph& sg);
bool launch_fused_tc(Ctx& ctx, const Engine& e, const uint64_t* maskt, uint64_t Wp,
                     const float* isd, const uint16_t* deg16, uint64_t ntp, float* apart);

// sf_cgls.cu
struct CglsResult {
  std::vector<double> phi;
  uint64_t iterations = 0;
  double relative_residual = 0.0;
  bool converged = false;
  std::vector<double> trace, row_residual_trace;
};
struct CglsInput {
  uint32_t n = 0;
  uint64_t rows = 0;  // local rows (even)
  uint32_t W = 0;
  const uint64_t* dev_rows = nullptr;  // row-major bits on device
  const double* dev_sw = nullptr;      // sqrt(weight) per local row
  const double* dev_targets = nullptr; // value - base per local row
  double constraint_target = 0.0, constraint_weight = 0.0;
  uint64_t global_pair_count = 0;
  // optional, from launch_assemble_pairs: set bits per row, complement flags
  const uint32_t* dev_pop = nullptr;
  const uint8_t* dev_is_comp = nullptr;
  // fixed-order mode (CglsOptions::fixed_order, solver.hpp:62-65): every
  // cross-row sum exact, so phi is bitwise identical for any worker layout
  bool fixed_order = false;
  // dev_rows holds kept-set rows only (one per pair, W words each; every
  // pair a complement pair)
  bool kept_only = false;
  // > 0: dev_rows is the caller's scratch (capacity in words) and may be
  // overwritten once the solver's own layouts are built — the dense pairs'
  // word-major rows then live there instead of in a separate buffer
  uint64_t rows_scratch_words = 0;
};
CglsResult cgls_solve(Ctx& ctx, const CglsInput& in, double tol,
                      uint64_t max_iter, int mode, bool trace);
// tensor-core tail (sf_tail_tc.cu)
// Tensor-core (tcgen05 kind::i8, exact integer) passes of the bit-row CGLS
// over the dense pairs (sf_cgls_i8.cu). SF_CGLS_I8=0 keeps the nibble tables.
bool cgls_i8_enabled();
uint64_t cgls_i8_digit_bytes(uint64_t elements);
uint64_t cgls_i8_scratch_doubles();
// digit groups of x over [beg, len) (groups aligned down from beg); the grid
// exponent goes to *exp_slot
void launch_cgls_digits(const double* x, uint64_t beg, uint64_t len, double* partial, uint8_t* digits, int* exp_slot,
                        cudaStream_t st);
// out[p][lane] = sum over the words of part p of the lane's bits x the digit groups
void launch_bitmat_i8(const uint64_t* words, uint64_t stride, uint64_t lanes, uint64_t out_lanes, uint32_t nparts,
                      const uint32_t* split_start, uint32_t part_words, uint32_t total_words, const uint8_t* digits,
                      const int* exp_slot, double* out, uint64_t out_stride, int sms, cudaStream_t st);

bool tail_tc_supported(const Engine& e);
uint32_t tc_deg_table_cap();
void build_tail_tc(Ctx& ctx, Engine& e);
void launch_tail_tc(Ctx& ctx, const Engine& e, const float* apart, const uint64_t* maskt, uint64_t Wp,
                    const float* isd, const uint16_t* deg16, uint64_t ntp, uint32_t cls, uint64_t row0,
                    uint64_t rows, float* out, float* allprobs);
// extract_computational_graph (graph.cpp:195-261) on the device, byte-
// identical to the host version; features are not copied (sg.source = &g)
Subgraph extract_device(Ctx& ctx, const Graph& g, uint32_t target, int hops);
// Runs of rows with one weight (explain_node: a size class; solve_direct:
// equal caller weights), rows [begin, end)
struct GramRun {
  uint64_t begin = 0, end = 0;
  double weight = 0.0;
};
// solve_direct (solver.cpp:364-428) on the device: tcgen05 Gram, blocked
// FP64 Cholesky with the reference's jitter retry, triangular solves
std::vector<double> gram_solve(Ctx& ctx, const CglsInput& in, const std::vector<GramRun>& runs);
// players by phi descending, ties by index (solver.cpp:430-440), on the device
std::vector<uint32_t> rank_players(Ctx& ctx, const std::vector<double>& phi);

// sf_assemble (sf_cgls.cu): per-row sqrt(weight) and targets on device from
// per-size weights and float predictions.
void launch_assemble(Ctx& ctx, const uint64_t* dev_rows, uint64_t rows,
                     uint32_t W, uint32_t n, const double* dev_wsize,
                     const float* dev_values, double base, double* dev_sw,
                     double* dev_targets, int* dev_bad_row);
// the same for adjacent row pairs in one read of both rows, also writing the
// set bits per row and the complement flags the solver needs
void launch_assemble_pairs(Ctx& ctx, const uint64_t* dev_rows, uint64_t rows,
                           uint32_t W, uint32_t n, const double* dev_wsize,
                           const float* dev_values, double base, double* dev_sw,
                           double* dev_targets, int* dev_bad_row, uint32_t* dev_pop,
                           uint8_t* dev_is_comp, bool kept_only = false);

}  // namespace sfb
