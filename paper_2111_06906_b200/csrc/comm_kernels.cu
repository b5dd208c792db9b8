// comm_kernels.cu -- the local collective backend's reduction (comm.cpp): sums of the ranks'
// published buffers (peer pointers, any device with peer access) into this rank's staging.
#include <cuda_runtime.h>

#include <cstdint>

#include "comm.h"
#include "kernels.h"

namespace prx {

namespace {

struct Peers {
    const void* p[kMaxLocalRanks];
};

template <typename T>
__global__ void k_local_reduce(Peers src, int n_src, T* __restrict__ dst, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        T acc = static_cast<const T*>(src.p[0])[i];
        for (int r = 1; r < n_src; ++r) acc += static_cast<const T*>(src.p[r])[i];  // rank order: deterministic
        dst[i] = acc;
    }
}

}  // namespace

void launch_local_reduce(const void* const* src, int n_src, void* dst, size_t n, int kind, cudaStream_t st) {
    if (n == 0) return;
    Peers P{};
    for (int r = 0; r < n_src; ++r) P.p[r] = src[r];
    const unsigned grid = launch_grid(n, 256);
    if (kind == 0) k_local_reduce<uint32_t><<<grid, 256, 0, st>>>(P, n_src, static_cast<uint32_t*>(dst), n);
    else if (kind == 1) k_local_reduce<float><<<grid, 256, 0, st>>>(P, n_src, static_cast<float*>(dst), n);
    else k_local_reduce<unsigned long long><<<grid, 256, 0, st>>>(P, n_src, static_cast<unsigned long long*>(dst), n);
    ++g_launches;
}

}  // namespace prx
