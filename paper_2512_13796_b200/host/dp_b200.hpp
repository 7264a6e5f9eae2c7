// Data-parallel training over views for the C++ nexel::train drop-in (SURVEY.md §8(f)-4,
// around the reference loop trainer.cpp:262-344): one process per GPU, each with a
// replica of the scene and the optimizer state; every iteration each rank renders its own
// view, the ranks average their gradients in place on the device, and every rank applies
// the same Adam step, so the replicas stay bit-identical.
//
// Configured from the environment (the reference's train() has no parallel arguments):
//   NEXEL_DP_WORLD   number of ranks (absent or 1: single process, no communicator)
//   NEXEL_DP_RANK    this rank, 0 .. world-1
//   NEXEL_DP_DIR     a fresh, node-local directory for the rendezvous files
//   NEXEL_DP_BACKEND "nccl" (default: NCCL all-reduce on the run's stream, NVLink /
//                    NVSwitch between the GPUs; libnccl is loaded on first use) or "host"
//                    (device -> pinned host -> a shared-memory segment in NEXEL_DP_DIR,
//                    summed in rank order; for ranks sharing one GPU, e.g. the tests)
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <memory>

namespace nexel {

class DpComm {
   public:
    virtual ~DpComm() = default;
    int world = 1, rank = 0;
    // In-place all-reduce of n doubles on the device, ordered on `stream`: the sum, or the
    // sum divided by the world size. Every rank ends with identical values.
    virtual void all_reduce(double* dev, size_t n, bool average, cudaStream_t stream) = 0;
    // The communicator the environment asks for, or nullptr for one process. `device` is
    // the CUDA device of this rank.
    static std::unique_ptr<DpComm> from_env(int device);
};

// NEXEL_DP_RANK / NEXEL_DP_WORLD as configured (0 / 1 without data parallelism).
int dp_env_rank();
int dp_env_world();

}  // namespace nexel
