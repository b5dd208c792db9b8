// prims.cu -- tile scan, stable compaction and stable LSD radix sort (see prims.h).
//
// Layout of every tiled kernel: a tile is 2048 consecutive elements handled by 256
// threads in 8 rounds; in round k thread t owns element tile_base + k*256 + t, so a
// round is one coalesced 1 KiB access and element order within a tile is preserved.
#include "prims.h"

#include <algorithm>
#include <atomic>
#include <cstdlib>

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

// out[k] = base_id + i for the k-th flagged i; with key_of, also keys[k] = key_of[i]
template <typename T>
__global__ void k_flag_scatter(const T* __restrict__ flags, uint32_t n_max, const uint32_t* n_dev,
                               uint32_t base_id, const uint32_t* __restrict__ offs,
                               uint32_t* __restrict__ out, const uint32_t* __restrict__ key_of = nullptr,
                               uint32_t* __restrict__ keys = nullptr) {
    __shared__ uint32_t sh[kPrimItems][kPrimThreads / 32];
    const uint32_t n = n_of(n_max, n_dev);
    const uint64_t base = (uint64_t)blockIdx.x * kPrimTile;
    if (base >= n) return;
    uint32_t run = offs[blockIdx.x];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // every load of the tile in flight before the ordered rounds
    bool fl[kPrimItems];
    uint32_t kv[kPrimItems];
#pragma unroll
    for (int k = 0; k < kPrimItems; ++k) {
        const uint64_t i = base + (uint64_t)k * kPrimThreads + threadIdx.x;
        fl[k] = i < n && flags[i] != 0;
    }
    if (key_of) {
#pragma unroll
        for (int k = 0; k < kPrimItems; ++k)
            kv[k] = fl[k] ? __ldg(&key_of[base + (uint64_t)k * kPrimThreads + threadIdx.x]) : 0u;
    }
    // one exchange for the whole tile: every warp publishes its per-round counts; a flagged
    // element's slot = run + earlier rounds (all warps) + earlier warps + lane rank
    uint32_t ball[kPrimItems];
#pragma unroll
    for (int k = 0; k < kPrimItems; ++k) {
        ball[k] = __ballot_sync(0xffffffffu, fl[k]);
        if (lane == 0) sh[k][warp] = __popc(ball[k]);
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kPrimItems; ++k) {
        const uint64_t i = base + (uint64_t)k * kPrimThreads + threadIdx.x;
        uint32_t before = 0, total = 0;
#pragma unroll
        for (int w = 0; w < kPrimThreads / 32; ++w) {
            const uint32_t c = sh[k][w];
            before += w < warp ? c : 0u;
            total += c;
        }
        if (fl[k]) {
            const uint32_t o = run + before + __popc(ball[k] & ((1u << lane) - 1u));
            out[o] = base_id + (uint32_t)i;
            if (key_of) keys[o] = kv[k];
        }
        run += total;
    }
}

// ----------------------------------------------------------------------------- radix sort
// One LSD pass = histogram + per-digit row scan + rank-and-scatter, over tiles of 4096 keys
// (256 threads x 16).  Histograms are digit-major (hist[d * tiles_max + t]); the row scan
// and the scatter only touch the tiles the device count reaches, so a sort sized for a
// large n_max costs what its live elements cost.  The scatter ranks a tile in shared memory
// (warp w owns the w-th contiguous eighth of the tile's elements, warp-private digit counters
// with match_any leaders), stages it digit-sorted, and writes each digit's run contiguously.
// Digits are 8 bits (10-bit digits as an opt-in knob, see digit_bits); the final pass can
// write two gathered float4 payload streams instead of the pairs.
constexpr int kRsItems = 16;
constexpr uint32_t kRsTile = kPrimThreads * kRsItems;  // 4096
static_assert(kRsTile == kSortTile, "ragged tiles are sort tiles");
constexpr int kRsWarps = kPrimThreads / 32;
constexpr int kRadixMax = 1024;                        // widest digit: 10 bits

inline uint32_t rs_tiles(uint64_t n) { return static_cast<uint32_t>((n + kRsTile - 1) / kRsTile); }
template <int B>
constexpr size_t rs_scatter_smem() {
    return sizeof(uint32_t) * ((size_t)(2 + kRsWarps) * (1u << B) + 2 * kRsTile);
}

// the pairs of tile t: [t * kRsTile, t * kRsTile + count); count from the device total, or
// per tile (`ragged`: tile t holds ragged[t] pairs at its start, every tile live)
__device__ __forceinline__ uint32_t rs_tile_count(uint32_t n_max, const uint32_t* n_dev, const uint32_t* ragged) {
    if (ragged) return ragged[blockIdx.x];
    const uint32_t n = n_of(n_max, n_dev);
    const uint64_t base = (uint64_t)blockIdx.x * kRsTile;
    return base >= n ? 0u : (n - base < kRsTile ? (uint32_t)(n - base) : kRsTile);
}

template <int B>
__global__ void __launch_bounds__(kPrimThreads) k_rs_hist(const uint32_t* __restrict__ keys, uint32_t n_max,
                                                          const uint32_t* n_dev, const uint32_t* ragged, int shift,
                                                          uint32_t mask, uint32_t tiles, uint32_t* __restrict__ hist) {
    constexpr int D = 1 << B;
    __shared__ uint32_t h[D];
    const uint64_t base = (uint64_t)blockIdx.x * kRsTile;
    if (!ragged && base >= n_of(n_max, n_dev)) return;  // beyond the live tiles: never read
    const uint32_t cnt = rs_tile_count(n_max, n_dev, ragged);
    for (int d = threadIdx.x; d < D; d += kPrimThreads) h[d] = 0;
    __syncthreads();
#pragma unroll 4
    for (int k = 0; k < kRsItems; ++k) {
        const uint32_t j = (uint32_t)k * kPrimThreads + threadIdx.x;
        if (j < cnt) atomicAdd(&h[(keys[base + j] >> shift) & mask], 1u);
    }
    __syncthreads();
    for (int d = threadIdx.x; d < D; d += kPrimThreads) hist[(uint64_t)d * tiles + blockIdx.x] = h[d];
}

// one CTA per digit: exclusive scan of the digit's row over the live tiles, row total out
__global__ void __launch_bounds__(kPrimThreads) k_rs_rowscan(uint32_t* __restrict__ hist, uint32_t tiles,
                                                             uint32_t n_max, const uint32_t* n_dev, bool ragged,
                                                             uint32_t* __restrict__ rowtot) {
    __shared__ uint32_t sh[kPrimThreads / 32];
    const uint32_t live = ragged ? tiles : rs_tiles_dev(n_of(n_max, n_dev));
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

template <int B, bool GATHER>
__global__ void __launch_bounds__(kPrimThreads, 3) k_rs_scatter(const uint32_t* __restrict__ kin,
                                                                const uint32_t* __restrict__ vin,
                                                                uint32_t* __restrict__ kout,
                                                                uint32_t* __restrict__ vout, uint32_t n_max,
                                                                const uint32_t* n_dev, const uint32_t* ragged,
                                                                int shift, uint32_t mask,
                                                                uint32_t tiles, const uint32_t* __restrict__ hist,
                                                                const uint32_t* __restrict__ rowtot, SortGather pg) {
    constexpr int D = 1 << B, DPT = D / kPrimThreads;  // digits per thread in the per-digit loops
    static_assert(DPT >= 1 && D % kPrimThreads == 0, "digit count");
    extern __shared__ uint32_t smem[];
    uint32_t* gbase = smem;                  // [D] global start of the tile's run of digit d
    uint32_t* tstart = gbase + D;            // [D] tile-local start of digit d
    uint32_t* wc = tstart + D;               // [kRsWarps][D] warp digit counters -> starts
    uint32_t* sk = wc + kRsWarps * D;        // [kRsTile] staged keys
    uint32_t* sv = sk + kRsTile;             // [kRsTile] their tile indices
    __shared__ uint32_t sh[kPrimThreads / 32];
    const uint64_t base = (uint64_t)blockIdx.x * kRsTile;
    if (!ragged && base >= n_of(n_max, n_dev)) return;
    const uint32_t cnt = rs_tile_count(n_max, n_dev, ragged);
    if (cnt == 0) return;  // (an empty ragged tile)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t d0 = threadIdx.x * DPT;  // this thread's digits in the per-digit loops
    {
        uint32_t r[DPT], sum = 0;
#pragma unroll
        for (int q = 0; q < DPT; ++q) {
            r[q] = rowtot[d0 + q];
            sum += r[q];
        }
        uint32_t total;
        uint32_t below = block_exclusive(sum, total, sh);  // all digits < d0
#pragma unroll
        for (int q = 0; q < DPT; ++q) {
            gbase[d0 + q] = below + hist[(uint64_t)(d0 + q) * tiles + blockIdx.x];
            below += r[q];
        }
    }
    {
        uint4* wz = reinterpret_cast<uint4*>(wc);
        for (int e = threadIdx.x; e < kRsWarps * D / 4; e += kPrimThreads) wz[e] = make_uint4(0, 0, 0, 0);
    }
    __syncthreads();
    // rank: the tile's cnt elements split into kRsWarps contiguous blocks of `per` (a multiple
    // of 32); warp `warp` walks its block in order, 32 per round (sparse ragged tiles run few
    // rounds instead of 16 mostly idle ones)
    const uint32_t per = ((cnt + kPrimThreads - 1) / kPrimThreads) * 32;
    const uint32_t wbase = warp * per;
    const uint32_t rounds = (per + 31) / 32;  // same for every warp; elements past cnt idle
    uint32_t key[kRsItems], rk[kRsItems];  // (values follow through their tile index)
#pragma unroll
    for (int k = 0; k < kRsItems; ++k) {
        const uint32_t j = wbase + k * 32 + lane;
        key[k] = (k < (int)rounds && j < cnt) ? kin[base + j] : 0u;
    }
    __syncwarp();
    uint32_t* mine = wc + warp * D;
#pragma unroll
    for (int k = 0; k < kRsItems; ++k) {
        if (k >= (int)rounds) break;
        const uint32_t j = wbase + k * 32 + lane;
        const uint32_t d = j < cnt ? ((key[k] >> shift) & mask) : (uint32_t)D;  // sentinel
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        const uint32_t below = __popc(peers & ((1u << lane) - 1u));
        const uint32_t prior = d < D ? mine[d] : 0u;
        __syncwarp();
        if (d < D && below == 0) mine[d] = prior + __popc(peers);
        __syncwarp();
        rk[k] = prior + below;
    }
    __syncthreads();
    {  // digit-major offsets: (digit, warp) order == (digit, element) order
        uint32_t cnt_d[DPT], sum = 0;
#pragma unroll
        for (int q = 0; q < DPT; ++q) {
            uint32_t s = 0;
#pragma unroll
            for (int w = 0; w < kRsWarps; ++w) {
                const uint32_t c = wc[w * D + d0 + q];
                wc[w * D + d0 + q] = s;
                s += c;
            }
            cnt_d[q] = s;
            sum += s;
        }
        uint32_t total;
        uint32_t t0 = block_exclusive(sum, total, sh);
#pragma unroll
        for (int q = 0; q < DPT; ++q) {
            tstart[d0 + q] = t0;
#pragma unroll
            for (int w = 0; w < kRsWarps; ++w) wc[w * D + d0 + q] += t0;
            t0 += cnt_d[q];
        }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kRsItems; ++k) {
        if (k >= (int)rounds) break;
        const uint32_t j = wbase + k * 32 + lane;
        if (j < cnt) {
            const uint32_t d = (key[k] >> shift) & mask;
            const uint32_t pos = mine[d] + rk[k];
            sk[pos] = key[k];
            sv[pos] = j;
        }
    }
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < cnt; j += kPrimThreads) {
        const uint32_t k = sk[j];
        const uint32_t d = (k >> shift) & mask;
        const uint32_t g = gbase[d] + (j - tstart[d]);
        const uint32_t v = __ldg(&vin[base + sv[j]]);
        if (GATHER) {
            pg.out_a[g] = __ldg(&pg.a[(size_t)pg.stride * v]);
            pg.out_b[g] = __ldg(&pg.b[(size_t)pg.stride * v]);
        } else {
            kout[g] = k;
            vout[g] = v;
        }
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
    s.hist = s.rowtot + kRadixMax + 64;
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
    return 4ull * (tiles + 64 + prim_tiles(tiles) + 64 + kRadixMax + 64 + (uint64_t)rs_tiles(n_max ? n_max : 1) * kRadixMax + 64);
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

void compact_u8_pairs(const uint8_t* flags, const uint32_t* key_of, uint32_t n_max, uint32_t* keys,
                      uint32_t* vals, uint32_t* count_dev, void* scratch, cudaStream_t st) {
    if (n_max == 0) {
        cudaMemsetAsync(count_dev, 0, 4, st);
        return;
    }
    Scratch s = carve(scratch, n_max);
    const uint32_t tiles = prim_tiles(n_max);
    k_flag_count<uint8_t><<<tiles, kPrimThreads, 0, st>>>(flags, n_max, nullptr, s.tile);
    scan_inplace(s.tile, tiles, count_dev, s.tile2, st);
    k_flag_scatter<uint8_t><<<tiles, kPrimThreads, 0, st>>>(flags, n_max, nullptr, 0, s.tile, vals, key_of, keys);
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

namespace {
// digit width per sort: 8 bits; PRX_RADIX10=1: 10-bit digits where they save a pass (measured
// slower on the splat's 20-bit slots: 0.62 vs 0.50 ms, the wider scatter holds 72 KB of shared memory)
int digit_bits(int bits) {
    static const bool wide = [] {
        const char* e = std::getenv("PRX_RADIX10");
        return e && e[0] == '1';
    }();
    const int p8 = (bits + 7) / 8, p10 = (bits + 9) / 10;
    return wide && p10 < p8 ? 10 : 8;
}

template <int B, bool GATHER>
void rs_pass(const uint32_t* ki, const uint32_t* vi, uint32_t* ko, uint32_t* vo, uint32_t n_max,
             const uint32_t* n_dev, const uint32_t* ragged, int shift, int w, uint32_t tiles, const Scratch& s,
             const SortGather& pg, cudaStream_t st) {
    constexpr size_t smem = rs_scatter_smem<B>();
    if (smem > 48 * 1024) {  // opt-in shared memory, once per device (an uncaptured first use)
        static std::atomic<uint64_t> set_on{0};
        int dev = 0;
        cudaGetDevice(&dev);
        const uint64_t bit = 1ull << (dev & 63);
        if (!(set_on.load() & bit)) {
            cudaFuncSetAttribute(k_rs_scatter<B, GATHER>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            set_on.fetch_or(bit);
        }
    }
    const uint32_t mask = (1u << w) - 1u;
    k_rs_hist<B><<<tiles, kPrimThreads, 0, st>>>(ki, n_max, n_dev, ragged, shift, mask, tiles, s.hist);
    k_rs_rowscan<<<1u << B, kPrimThreads, 0, st>>>(s.hist, tiles, n_max, n_dev, ragged != nullptr, s.rowtot);
    k_rs_scatter<B, GATHER><<<tiles, kPrimThreads, smem, st>>>(ki, vi, ko, vo, n_max, n_dev, ragged, shift, mask,
                                                                tiles, s.hist, s.rowtot, pg);
    g_launches += 3;
}

// the passes; with pg set the last pass writes the gathered payloads.  Returns the number of
// passes that wrote pairs (their parity says where the pairs are).
int rs_run(uint32_t* keys, uint32_t* vals, uint32_t* keys_tmp, uint32_t* vals_tmp, uint32_t n_max,
           const uint32_t* n_dev, int bits, void* scratch, const SortGather* pg, const uint32_t* ragged,
           cudaStream_t st) {
    Scratch s = carve(scratch, n_max);
    const uint32_t tiles = rs_tiles(n_max);
    const int db = digit_bits(bits);
    const int passes = (bits + db - 1) / db;
    uint32_t *ki = keys, *vi = vals, *ko = keys_tmp, *vo = vals_tmp;
    int shift = 0, written = 0;
    const SortGather none{};
    for (int p = 0; p < passes; ++p) {
        const int w = (bits - shift + (passes - p) - 1) / (passes - p);  // even split of the rest
        const bool gather = pg && p == passes - 1;
        const uint32_t* rg = p == 0 ? ragged : nullptr;  // the first pass reads the ragged tiles
        if (db == 10) {
            if (gather) rs_pass<10, true>(ki, vi, ko, vo, n_max, n_dev, rg, shift, w, tiles, s, *pg, st);
            else rs_pass<10, false>(ki, vi, ko, vo, n_max, n_dev, rg, shift, w, tiles, s, none, st);
        } else {
            if (gather) rs_pass<8, true>(ki, vi, ko, vo, n_max, n_dev, rg, shift, w, tiles, s, *pg, st);
            else rs_pass<8, false>(ki, vi, ko, vo, n_max, n_dev, rg, shift, w, tiles, s, none, st);
        }
        shift += w;
        if (!gather) {
            ++written;
            std::swap(ki, ko);
            std::swap(vi, vo);
        }
    }
    return written;
}
}  // namespace

bool radix_sort_pairs_nocopy(uint32_t* keys, uint32_t* vals, uint32_t* keys_tmp, uint32_t* vals_tmp,
                             uint32_t n_max, const uint32_t* n_dev, int bits, void* scratch, cudaStream_t st) {
    if (n_max == 0 || bits <= 0) return false;
    return (rs_run(keys, vals, keys_tmp, vals_tmp, n_max, n_dev, bits, scratch, nullptr, nullptr, st) & 1) != 0;
}

void radix_sort_gather(uint32_t* keys, uint32_t* vals, uint32_t* keys_tmp, uint32_t* vals_tmp, uint32_t n_max,
                       const uint32_t* n_dev, int bits, const SortGather& pg, void* scratch, cudaStream_t st,
                       const uint32_t* ragged) {
    if (n_max == 0 || bits <= 0) return;
    rs_run(keys, vals, keys_tmp, vals_tmp, n_max, n_dev, bits, scratch, &pg, ragged, st);
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
