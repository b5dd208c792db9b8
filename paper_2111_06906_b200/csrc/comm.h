// comm.h -- collective backends behind prx_collectives (comm.cpp): NCCL and in-process local.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <vector>

#include "prx.h"

namespace prx {

constexpr int kMaxLocalRanks = 16;

struct Comm {
    int rank = 0, world = 1;
    virtual ~Comm() = default;
    virtual void table(prx_collectives* out) = 0;
};

void nccl_unique_id(uint8_t out[128]);
std::unique_ptr<Comm> nccl_comm(const uint8_t id[128], int rank, int world, int device);
std::vector<std::unique_ptr<Comm>> local_comms(int world);

// dst[i] = sum over r < n_src of src[r][i]; kind 0 = u32, 1 = f32, 2 = u64 (comm_kernels.cu)
void launch_local_reduce(const void* const* src, int n_src, void* dst, size_t n, int kind, cudaStream_t st);

}  // namespace prx
