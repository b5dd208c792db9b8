// prims.h -- device-wide primitives of the B200 engine (hand-written, no CUB/Thrust):
// tile scan, stable stream compaction and stable LSD radix sort.  Element counts may live
// in device memory (`n_dev`) so whole frames run without host round trips; grids are
// sized from a host-side upper bound `n_max`.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace prx {

constexpr int kPrimThreads = 256;
constexpr int kPrimItems = 8;
constexpr uint32_t kPrimTile = kPrimThreads * kPrimItems;  // 2048 elements per tile

inline uint32_t prim_tiles(uint64_t n) { return static_cast<uint32_t>((n + kPrimTile - 1) / kPrimTile); }

// Scratch sized for n_max elements (bytes for prim_scratch_bytes).
size_t prim_scratch_bytes(uint64_t n_max);

// out[i] = sum_{j<i} in[j] for i < n (n = *n_dev if n_dev else n_max); *total_dev = sum.
// in and out may alias.
void scan_exclusive_u32(const uint32_t* in, uint32_t* out, uint32_t n_max, const uint32_t* n_dev,
                        uint32_t* total_dev, void* scratch, cudaStream_t st);

// Stable compaction: out[k] = base + i for the k-th i (ascending) with flags[i] != 0.
void compact_u8(const uint8_t* flags, uint32_t n_max, const uint32_t* n_dev, uint32_t base,
                uint32_t* out, uint32_t* count_dev, void* scratch, cudaStream_t st);
// Stable compaction into pairs: for the k-th flagged i, vals[k] = i and keys[k] = key_of[i].
void compact_u8_pairs(const uint8_t* flags, const uint32_t* key_of, uint32_t n_max, uint32_t* keys,
                      uint32_t* vals, uint32_t* count_dev, void* scratch, cudaStream_t st);
// Same with a u32 flag array (nonzero = keep).
void compact_u32(const uint32_t* flags, uint32_t n_max, const uint32_t* n_dev, uint32_t base,
                 uint32_t* out, uint32_t* count_dev, void* scratch, cudaStream_t st);

// Stable LSD radix sort of `bits` low key bits; results land back in keys/vals
// (keys_tmp/vals_tmp are ping-pong buffers of the same size).
// as radix_sort_pairs without the final copy: returns true when the sorted pairs are in
// keys_tmp / vals_tmp (odd number of passes), false when in keys / vals
bool radix_sort_pairs_nocopy(uint32_t* keys, uint32_t* vals, uint32_t* keys_tmp, uint32_t* vals_tmp,
                             uint32_t n_max, const uint32_t* n_dev, int bits, void* scratch, cudaStream_t st);
// Payload gathered by the last pass of radix_sort_gather: out_a[k] = a[stride * v_k],
// out_b[k] = b[stride * v_k] for the k-th sorted value v_k.
struct SortGather {
    const float4* a = nullptr;
    const float4* b = nullptr;
    uint32_t stride = 1;
    float4* out_a = nullptr;
    float4* out_b = nullptr;
};
// Stable sort by `bits` low key bits whose result is the payload records of the sorted
// values (keys/vals and the tmp buffers are clobbered).  With `ragged`, the input is tiled:
// tile t (of rs tiles over n_max) holds ragged[t] pairs at keys/vals[t * kSortTile...], in
// order, and *n_dev is their total.
constexpr uint32_t kSortTile = 4096;
void radix_sort_gather(uint32_t* keys, uint32_t* vals, uint32_t* keys_tmp, uint32_t* vals_tmp, uint32_t n_max,
                       const uint32_t* n_dev, int bits, const SortGather& pg, void* scratch, cudaStream_t st,
                       const uint32_t* ragged = nullptr);
void radix_sort_pairs(uint32_t* keys, uint32_t* vals, uint32_t* keys_tmp, uint32_t* vals_tmp,
                      uint32_t n_max, const uint32_t* n_dev, int bits, void* scratch,
                      cudaStream_t st);

}  // namespace prx
