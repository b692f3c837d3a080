// shapflow_b200.hpp — C++ drop-in for the shapflow hot path on B200.
//
// The reference explainer's own headers stay unchanged (they are the API
// contract): a maintainer compiles paper_2506_22668_b200/dropin/
// shapflow_dropin.cpp against them in place of the hot-path definitions of
// sampler.cpp / gcn.cpp / solver.cpp / explain.cpp and links
// libshapflow_b200.so. The drop-in defines, in namespace shapflow and with
// the reference declarations verbatim:
//   plan_sizes, generate_masks            (sampler.hpp:49-50, 84-85)
//   predict_probs, predict, predict_batched (gcn.hpp:50-62)
//   solve_cgls, solve_direct, rank_edges  (solver.hpp:94-109)
//   explain_node, auto_samples, node_sampling_seed (explain.hpp:35-49)
// Everything else (graph/model I/O, assemble_problem, explain_nodes,
// select_nodes, fidelity, documents, the thread/socket communicators) keeps
// the reference's code; explain_nodes and the fidelity/oracle helpers reach
// the GPU through the functions above.
//
// This header adds what the reference has no counterpart for:
//   * NcclCommunicator — a shapflow::Communicator over NCCL/NVLink, one rank
//     per GPU (comm.hpp:28-52). Passed to explain_node / solve_cgls, the
//     per-iteration all-reduces run on device buffers in stream order; with
//     any other Communicator (thread or socket workers) they are staged
//     through host memory and go through that Communicator, so its
//     CollectiveStats count exactly what the reference would.
//   * device selection and the per-thread B200 context used by the drop-in.
#pragma once

#include <array>
#include <cstdint>
#include <span>
#include <vector>

#include "shapflow/comm.hpp"
#include "shapflow_b200.h"

namespace shapflow::b200 {

// NCCL unique id (128 bytes) created on rank 0 and shared with the other
// ranks by the caller (file, socket, MPI, torch.distributed ...).
std::array<char, 128> nccl_unique_id();

class NcclCommunicator : public Communicator {
 public:
  // One rank on one GPU. world == 1 needs no unique id.
  NcclCommunicator(int device, int rank, int world, const std::array<char, 128>& unique_id);
  ~NcclCommunicator() override;
  NcclCommunicator(const NcclCommunicator&) = delete;
  NcclCommunicator& operator=(const NcclCommunicator&) = delete;

  int rank() const override { return rank_; }
  int world_size() const override { return world_; }
  sf_ctx* context() const { return ctx_; }
  // Folds the collectives a library call issued on the device into stats_.
  void absorb_device_stats();

 protected:
  void all_reduce_impl(std::uint64_t seq, std::span<double> buf) override;
  void barrier_impl(std::uint64_t seq) override;
  std::vector<double> gather_impl(std::uint64_t seq, std::span<const double> buf) override;

 private:
  sf_ctx* ctx_ = nullptr;
  int rank_ = 0, world_ = 1;
  std::uint64_t seen_[4] = {0, 0, 0, 0};  // device stats already absorbed
};

// GPU used by the drop-in for callers that pass a non-NCCL Communicator:
// SHAPFLOW_B200_DEVICE if set, else 0. Each host thread gets its own
// context (stream, buffers) on that device.
void set_default_device(int device);
int default_device();

}  // namespace shapflow::b200
