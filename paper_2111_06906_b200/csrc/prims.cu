// prims.cu -- tile scan, stable compaction and stable LSD radix sort (see prims.h).
//
// Layout of every tiled kernel: a tile is 2048 consecutive elements handled by 256
// threads in 8 rounds; in round k thread t owns element tile_base + k*256 + t, so a
// round is one coalesced 1 KiB access and element order within a tile is preserved.
#include "prims.h"

#include <algorithm>
#include <atomic>

#include <cstdio>

namespace prx {

extern std::atomic<uint64_t> g_launches;  // kernels.cu: launches by this library (bench evidence)

namespace {

__device__ __forceinline__ uint32_t n_of(uint32_t n_max, const uint32_t* n_dev) {
    return n_dev ? min(*n_dev, n_max) : n_max;
}

__device__ __forceinline__ uint32_t rs_tiles_dev(uint32_t n) { return (n + 4095u) / 4096u; }

// Exclusive scan across the 256 threads of a block; returns the block total.
__device__ __forceinline__ uint32_t block_exclusive(uint32_t v, uint32_t& total, uint32_t* sh_warp) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sh_warp[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = lane < (kPrimThreads / 32) ? sh_warp[lane] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        if (lane < (kPrimThreads / 32)) sh_warp[lane] = w;  // inclusive warp prefix
    }
    __syncthreads();
    total = sh_warp[kPrimThreads / 32 - 1];
    const uint32_t before = warp > 0 ? sh_warp[warp - 1] : 0u;
    __syncthreads();
    return before + x - v;
}

// ----------------------------------------------------------------------------- scan
__global__ void k_tile_sum(const uint32_t* __restrict__ in, uint32_t n_max, const uint32_t* n_dev,
                           uint32_t* __restrict__ sums) {
    __shared__ uint32_t sh[kPrimThreads / 32];
    const uint32_t n = n_of(n_max, n_dev);
    const uint64_t base = (uint64_t)blockIdx.x * kPrimTile;
    uint32_t acc = 0;
    if (base < n) {
#pragma unroll
        for (int k = 0; k < kPrimItems; ++k) {
            const uint64_t i = base + (uint64_t)k * kPrimThreads + threadIdx.x;
            if (i < n) acc += in[i];
        }
    }
    uint32_t total;
    block_exclusive(acc, total, sh);
    if (threadIdx.x == 0) sums[blockIdx.x] = total;
}

// Single-CTA exclusive scan of m values (in place), chunked with a running carry.
constexpr int kScanItems = 16;  // values per thread per chunk of the single-CTA scan

__global__ void k_scan_small(uint32_t* __restrict__ v, uint32_t m, uint32_t* total_dev) {
    __shared__ uint32_t sh[kPrimThreads / 32];
    uint32_t carry = 0;
    for (uint32_t base = 0; base < m; base += kPrimThreads * kScanItems) {
        uint32_t x[kScanItems];
        uint32_t s = 0;
#pragma unroll
        for (int k = 0; k < kScanItems; ++k) {
            const uint32_t i = base + threadIdx.x * kScanItems + k;
            x[k] = i < m ? v[i] : 0u;
            s += x[k];
        }
        uint32_t total;
        const uint32_t ex = block_exclusive(s, total, sh);
        uint32_t run = carry + ex;
#pragma unroll
        for (int k = 0; k < kScanItems; ++k) {
            const uint32_t i = base + threadIdx.x * kScanItems + k;
            if (i < m) v[i] = run;
            run += x[k];
        }
        carry += total;
    }
    if (threadIdx.x == 0 && total_dev) *total_dev = carry;
}

__global__ void k_tile_scan(const uint32_t* __restrict__ in, uint32_t* __restrict__ out, uint32_t n_max,
                            const uint32_t* n_dev, const uint32_t* __restrict__ offs) {
    __shared__ uint32_t sh[kPrimThreads / 32];
    const uint32_t n = n_of(n_max, n_dev);
    const uint64_t base = (uint64_t)blockIdx.x * kPrimTile;
    if (base >= n) return;
    uint32_t run = offs[blockIdx.x];
#pragma unroll
    for (int k = 0; k < kPrimItems; ++k) {
        const uint64_t i = base + (uint64_t)k * kPrimThreads + threadIdx.x;
        const uint32_t x = i < n ? in[i] : 0u;
        uint32_t total;
        const uint32_t ex = block_exclusive(x, total, sh);
        if (i < n) out[i] = run + ex;
        run += total;
    }
}

// ----------------------------------------------------------------------------- compaction
template <typename T>
__global__ void k_flag_count(const T* __restrict__ flags, uint32_t n_max, const uint32_t* n_dev,
                             uint32_t* __restrict__ counts) {
    const uint32_t n = n_of(n_max, n_dev);
    const uint64_t base = (uint64_t)blockIdx.x * kPrimTile;
    uint32_t c = 0;
    if (base < n) {
#pragma unroll
        for (int k = 0; k < kPrimItems; ++k) {
            const uint64_t i = base + (uint64_t)k * kPrimThreads + threadIdx.x;
            c += (i < n && flags[i] != 0) ? 1u : 0u;
        }
    }
    c = __reduce_add_sync(0xffffffffu, c);
    __shared__ uint32_t sh[kPrimThreads / 32];
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
        for (int w = 0; w < kPrimThreads / 32; ++w) t += sh[w];
        counts[blockIdx.x] = t;
    }
}

template <typename T>
__global__ void k_flag_scatter(const T* __restrict__ flags, uint32_t n_max, const uint32_t* n_dev,
                               uint32_t base_id, const uint32_t* __restrict__ offs,
                               uint32_t* __restrict__ out) {
    __shared__ uint32_t sh[kPrimThreads / 32];
    const uint32_t n = n_of(n_max, n_dev);
    const uint64_t base = (uint64_t)blockIdx.x * kPrimTile;
    if (base >= n) return;
    uint32_t run = offs[blockIdx.x];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < kPrimItems; ++k) {
        const uint64_t i = base + (uint64_t)k * kPrimThreads + threadIdx.x;
        const bool f = i < n && flags[i] != 0;
        const uint32_t ball = __ballot_sync(0xffffffffu, f);
        if (lane == 0) sh[warp] = __popc(ball);
        __syncthreads();
        uint32_t before = 0, total = 0;
#pragma unroll
        for (int w = 0; w < kPrimThreads / 32; ++w) {
            const uint32_t c = sh[w];
            before += w < warp ? c : 0u;
            total += c;
        }
        if (f) out[run + before + __popc(ball & ((1u << lane) - 1u))] = base_id + (uint32_t)i;
        run += total;
        __syncthreads();
    }
}

// ----------------------------------------------------------------------------- radix sort
// One LSD pass = histogram + per-digit row scan + rank-and-scatter, over tiles of 4096 keys
// (256 threads x 16).  Histograms are digit-major (hist[d * tiles_max + t]); the row scan
// and the scatter only touch the tiles the device count reaches, so a sort sized for a
// large n_max costs what its live elements cost.  The scatter ranks a tile in shared memory
// (warp w owns tile elements [512 w, 512 w + 512), warp-private digit counters with
// match_any leaders), stages it digit-sorted, and writes each digit's run contiguously.
constexpr int kRadixBits = 8;
constexpr int kRadix = 1 << kRadixBits;
constexpr int kRsItems = 16;
constexpr uint32_t kRsTile = kPrimThreads * kRsItems;  // 4096
constexpr int kRsWarps = kPrimThreads / 32;
static_assert(kRadix == kPrimThreads, "one digit per thread in the per-digit loops");

inline uint32_t rs_tiles(uint64_t n) { return static_cast<uint32_t>((n + kRsTile - 1) / kRsTile); }

__global__ void __launch_bounds__(kPrimThreads) k_rs_hist(const uint32_t* __restrict__ keys, uint32_t n_max,
                                                          const uint32_t* n_dev, int shift, uint32_t mask,
                                                          uint32_t tiles, uint32_t* __restrict__ hist) {
    __shared__ uint32_t h[kRadix];
    const uint32_t n = n_of(n_max, n_dev);
    const uint64_t base = (uint64_t)blockIdx.x * kRsTile;
    if (base >= n) return;  // beyond the live tiles: never read
    h[threadIdx.x] = 0;
    __syncthreads();
#pragma unroll 4
    for (int k = 0; k < kRsItems; ++k) {
        const uint64_t i = base + (uint64_t)k * kPrimThreads + threadIdx.x;
        if (i < n) atomicAdd(&h[(keys[i] >> shift) & mask], 1u);
    }
    __syncthreads();
    hist[(uint64_t)threadIdx.x * tiles + blockIdx.x] = h[threadIdx.x];
}

// one CTA per digit: exclusive scan of the digit's row over the live tiles, row total out
__global__ void __launch_bounds__(kPrimThreads) k_rs_rowscan(uint32_t* __restrict__ hist, uint32_t tiles,
                                                             uint32_t n_max, const uint32_t* n_dev,
                                                             uint32_t* __restrict__ rowtot) {
    __shared__ uint32_t sh[kPrimThreads / 32];
    const uint32_t live = rs_tiles_dev(n_of(n_max, n_dev));
    uint32_t* row = hist + (uint64_t)blockIdx.x * tiles;
    uint32_t carry = 0;
    for (uint32_t b = 0; b < live; b += kPrimThreads * 4) {
        uint32_t x[4], sum = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t t = b + threadIdx.x * 4 + k;
            x[k] = t < live ? row[t] : 0u;
            sum += x[k];
        }
        uint32_t total;
        uint32_t run = carry + block_exclusive(sum, total, sh);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t t = b + threadIdx.x * 4 + k;
            if (t < live) row[t] = run;
            run += x[k];
        }
        carry += total;
    }
    if (threadIdx.x == 0) rowtot[blockIdx.x] = carry;
}

__global__ void __launch_bounds__(kPrimThreads, 3) k_rs_scatter(const uint32_t* __restrict__ kin,
                                                             const uint32_t* __restrict__ vin,
                                                             uint32_t* __restrict__ kout, uint32_t* __restrict__ vout,
                                                             uint32_t n_max, const uint32_t* n_dev, int shift,
                                                             uint32_t mask, uint32_t tiles,
                                                             const uint32_t* __restrict__ hist,
                                                             const uint32_t* __restrict__ rowtot) {
    __shared__ uint32_t gbase[kRadix];           // global start of the tile's run of digit d
    __shared__ uint32_t tstart[kRadix];          // tile-local start of digit d
    __shared__ uint32_t wc[kRsWarps][kRadix];    // warp digit counters -> warp digit starts
    __shared__ uint32_t sk[kRsTile], sv[kRsTile];  // staged keys, their tile indices
    __shared__ uint32_t sh[kPrimThreads / 32];
    const uint32_t n = n_of(n_max, n_dev);
    const uint64_t base = (uint64_t)blockIdx.x * kRsTile;
    if (base >= n) return;
    const uint32_t cnt = n - base < kRsTile ? (uint32_t)(n - base) : kRsTile;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    {
        uint32_t total;
        const uint32_t d0 = block_exclusive(rowtot[threadIdx.x], total, sh);  // digits below d
        gbase[threadIdx.x] = d0 + hist[(uint64_t)threadIdx.x * tiles + blockIdx.x];
    }
#pragma unroll
    for (int w = 0; w < kRsWarps; ++w) wc[w][threadIdx.x] = 0;
    __syncthreads();
    // rank: warp `warp` walks its 512 elements in order, 32 per round
    uint32_t key[kRsItems], rk[kRsItems];  // (values follow through their tile index)
    const uint32_t wbase = warp * (kRsTile / kRsWarps);
#pragma unroll
    for (int k = 0; k < kRsItems; ++k) {
        const uint32_t j = wbase + k * 32 + lane;
        key[k] = j < cnt ? kin[base + j] : 0u;
    }
#pragma unroll
    for (int k = 0; k < kRsItems; ++k) {
        const uint32_t j = wbase + k * 32 + lane;
        const uint32_t d = j < cnt ? ((key[k] >> shift) & mask) : (uint32_t)kRadix;  // sentinel
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        const uint32_t below = __popc(peers & ((1u << lane) - 1u));
        const uint32_t prior = d < kRadix ? wc[warp][d] : 0u;
        __syncwarp();
        if (d < kRadix && below == 0) wc[warp][d] = prior + __popc(peers);
        __syncwarp();
        rk[k] = prior + below;
    }
    __syncthreads();
    {  // digit-major offsets: (digit, warp) order == (digit, element) order
        const uint32_t d = threadIdx.x;
        uint32_t s = 0;
#pragma unroll
        for (int w = 0; w < kRsWarps; ++w) {
            const uint32_t c = wc[w][d];
            wc[w][d] = s;
            s += c;
        }
        uint32_t total;
        const uint32_t t0 = block_exclusive(s, total, sh);
        tstart[d] = t0;
#pragma unroll
        for (int w = 0; w < kRsWarps; ++w) wc[w][d] += t0;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kRsItems; ++k) {
        const uint32_t j = wbase + k * 32 + lane;
        if (j < cnt) {
            const uint32_t d = (key[k] >> shift) & mask;
            const uint32_t pos = wc[warp][d] + rk[k];
            sk[pos] = key[k];
            sv[pos] = j;
        }
    }
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < cnt; j += kPrimThreads) {
        const uint32_t k = sk[j];
        const uint32_t d = (k >> shift) & mask;
        const uint32_t g = gbase[d] + (j - tstart[d]);
        kout[g] = k;
        vout[g] = __ldg(&vin[base + sv[j]]);
    }
}

struct Scratch {
    uint32_t* tile;    // per-tile values (counts / sums), tiles entries
    uint32_t* tile2;   // second-level sums for large scans
    uint32_t* rowtot;  // radix: per-digit totals
    uint32_t* hist;    // radix histograms, 256 * radix tiles entries
};

Scratch carve(void* p, uint64_t n_max) {
    const uint64_t tiles = prim_tiles(n_max ? n_max : 1);
    Scratch s;
    s.tile = static_cast<uint32_t*>(p);
    s.tile2 = s.tile + tiles + 64;
    s.rowtot = s.tile2 + prim_tiles(tiles) + 64;
    s.hist = s.rowtot + kRadix + 64;
    return s;
}

// Exclusive scan of m device values in place (any m): tile sums + single-CTA scan.
void scan_inplace(uint32_t* v, uint32_t m, uint32_t* total_dev, uint32_t* tmp, cudaStream_t st) {
    if (m <= 64u * 1024u) {
        k_scan_small<<<1, kPrimThreads, 0, st>>>(v, m, total_dev);
        ++g_launches;
        return;
    }
    const uint32_t tiles = prim_tiles(m);
    k_tile_sum<<<tiles, kPrimThreads, 0, st>>>(v, m, nullptr, tmp);
    k_scan_small<<<1, kPrimThreads, 0, st>>>(tmp, tiles, total_dev);
    k_tile_scan<<<tiles, kPrimThreads, 0, st>>>(v, v, m, nullptr, tmp);
    g_launches += 3;
}

}  // namespace

size_t prim_scratch_bytes(uint64_t n_max) {
    const uint64_t tiles = prim_tiles(n_max ? n_max : 1);
    return 4ull * (tiles + 64 + prim_tiles(tiles) + 64 + kRadix + 64 + (uint64_t)rs_tiles(n_max ? n_max : 1) * kRadix + 64);
}

void scan_exclusive_u32(const uint32_t* in, uint32_t* out, uint32_t n_max, const uint32_t* n_dev,
                        uint32_t* total_dev, void* scratch, cudaStream_t st) {
    if (n_max == 0) return;
    Scratch s = carve(scratch, n_max);
    const uint32_t tiles = prim_tiles(n_max);
    k_tile_sum<<<tiles, kPrimThreads, 0, st>>>(in, n_max, n_dev, s.tile);
    scan_inplace(s.tile, tiles, total_dev, s.tile2, st);
    k_tile_scan<<<tiles, kPrimThreads, 0, st>>>(in, out, n_max, n_dev, s.tile);
    g_launches += 2;
}

void compact_u8(const uint8_t* flags, uint32_t n_max, const uint32_t* n_dev, uint32_t base,
                uint32_t* out, uint32_t* count_dev, void* scratch, cudaStream_t st) {
    if (n_max == 0) {
        cudaMemsetAsync(count_dev, 0, 4, st);
        return;
    }
    Scratch s = carve(scratch, n_max);
    const uint32_t tiles = prim_tiles(n_max);
    k_flag_count<uint8_t><<<tiles, kPrimThreads, 0, st>>>(flags, n_max, n_dev, s.tile);
    scan_inplace(s.tile, tiles, count_dev, s.tile2, st);
    k_flag_scatter<uint8_t><<<tiles, kPrimThreads, 0, st>>>(flags, n_max, n_dev, base, s.tile, out);
    g_launches += 2;
}

void compact_u32(const uint32_t* flags, uint32_t n_max, const uint32_t* n_dev, uint32_t base,
                 uint32_t* out, uint32_t* count_dev, void* scratch, cudaStream_t st) {
    if (n_max == 0) {
        cudaMemsetAsync(count_dev, 0, 4, st);
        return;
    }
    Scratch s = carve(scratch, n_max);
    const uint32_t tiles = prim_tiles(n_max);
    k_flag_count<uint32_t><<<tiles, kPrimThreads, 0, st>>>(flags, n_max, n_dev, s.tile);
    scan_inplace(s.tile, tiles, count_dev, s.tile2, st);
    k_flag_scatter<uint32_t><<<tiles, kPrimThreads, 0, st>>>(flags, n_max, n_dev, base, s.tile, out);
    g_launches += 2;
}

bool radix_sort_pairs_nocopy(uint32_t* keys, uint32_t* vals, uint32_t* keys_tmp, uint32_t* vals_tmp,
                             uint32_t n_max, const uint32_t* n_dev, int bits, void* scratch, cudaStream_t st) {
    if (n_max == 0 || bits <= 0) return false;
    Scratch s = carve(scratch, n_max);
    const uint32_t tiles = rs_tiles(n_max);
    uint32_t *ki = keys, *vi = vals, *ko = keys_tmp, *vo = vals_tmp;
    int passes = 0;
    for (int shift = 0; shift < bits; shift += kRadixBits, ++passes) {
        const int w = bits - shift < kRadixBits ? bits - shift : kRadixBits;
        const uint32_t mask = (1u << w) - 1u;
        k_rs_hist<<<tiles, kPrimThreads, 0, st>>>(ki, n_max, n_dev, shift, mask, tiles, s.hist);
        k_rs_rowscan<<<kRadix, kPrimThreads, 0, st>>>(s.hist, tiles, n_max, n_dev, s.rowtot);
        k_rs_scatter<<<tiles, kPrimThreads, 0, st>>>(ki, vi, ko, vo, n_max, n_dev, shift, mask, tiles, s.hist,
                                                     s.rowtot);
        g_launches += 3;
        uint32_t* t = ki;
        ki = ko;
        ko = t;
        t = vi;
        vi = vo;
        vo = t;
    }
    return (passes & 1) != 0;
}

namespace {
__global__ void k_copy_pairs(const uint32_t* __restrict__ ks, const uint32_t* __restrict__ vs, uint32_t* kd,
                             uint32_t* vd, uint32_t n_max, const uint32_t* n_dev) {
    const uint32_t n = n_of(n_max, n_dev);
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        kd[i] = ks[i];
        vd[i] = vs[i];
    }
}
}  // namespace

void radix_sort_pairs(uint32_t* keys, uint32_t* vals, uint32_t* keys_tmp, uint32_t* vals_tmp,
                      uint32_t n_max, const uint32_t* n_dev, int bits, void* scratch,
                      cudaStream_t st) {
    if (radix_sort_pairs_nocopy(keys, vals, keys_tmp, vals_tmp, n_max, n_dev, bits, scratch, st)) {
        // result in the tmp buffers: copy back the live elements only (n_dev, not n_max)
        const uint32_t grid = (uint32_t)std::min<uint64_t>((n_max + 255) / 256, 148u * 16u);
        k_copy_pairs<<<grid, 256, 0, st>>>(keys_tmp, vals_tmp, keys, vals, n_max, n_dev);
        ++g_launches;
    }
}

}  // namespace prx
