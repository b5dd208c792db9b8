// splat.cu -- gather_image (gather.cpp:35-75) on the GPU (north_star subsystem 6).
//
// The reference, per pixel: primary hit x (camera_ray + intersect_scene), then every live
// photon in the 27 grid cells around cell(x) (cell edge = r, 21-bit wrapped keys,
// gather.hpp:38-74) with the same object and |x_ph - x|^2 <= r^2 adds its energy, in cell
// order (dz, dy, dx) and photon insertion order.
//   k_gbuffer   primary hits (same float ops as camera_ray / intersect_scene);
//   k_pixcells  each hit pixel inserts its 27 neighbour-cell keys into an open-addressing
//               table (the cells any pixel can read);
//   mode 1 (default, bit-exact): photons of those cells are compacted and stably sorted by
//               cell slot (= the reference's insertion order per cell), copied contiguous, and
//               summed per pixel in the reference's order -- one warp per pixel with staged
//               in-order accumulation (k_gather_staged), or, for large images, one warp per 32
//               pixels that share a home cell walking the shared candidates (k_gather_groups);
//   mode 0 (atomic splat, fp32 atomics): the same candidate photons binned per cell without
//               order -- block-aggregated append + per-cell atomic counts (k_bin_filter), atomic
//               cursors (k_bin_scatter): no stable sort, no candidate compaction pass -- then
//               accumulated in any order: one warp per pixel with lane partial sums and a warp
//               reduction (k_splat_pixels); for large images 32-pixel groups sharing a home cell
//               with register accumulators over shared photon slabs (k_gather_groups), or
//               (PRX_SPLAT_TILES=1) photon-parallel tiles adding into shared-memory pixel
//               accumulators with shared-memory atomics (k_splat_tiles, measured slower).  Same
//               contributing set as gather_image, different fp32 summation order;
//   both        L = sum(E) * albedo / pi / (pi r^2) (gather.cpp:71).
#include <cstdlib>

#include "device_scene.cuh"
#include "kernels.h"
#include "prims.h"

namespace prx {

namespace {

constexpr int kT = 256;
constexpr unsigned long long kEmptyKey = ~0ull;
#ifndef PRX_GATHER_UNROLL
#define PRX_GATHER_UNROLL 8
#endif

__device__ __forceinline__ long long cell_coord(float v, float r) { return (long long)floorf(v / r); }

// GatherGrid::key (gather.hpp:64-69): three 21-bit wrapped coordinates
__device__ __forceinline__ unsigned long long grid_key(long long x, long long y, long long z) {
    return (((unsigned long long)x & 0x1FFFFFull) << 42) | (((unsigned long long)y & 0x1FFFFFull) << 21) |
           ((unsigned long long)z & 0x1FFFFFull);
}

__device__ __forceinline__ uint32_t slot_of(unsigned long long key, int bits) {
    return (uint32_t)((key * 0x9E3779B97F4A7C15ull) >> (64 - bits));
}

// |p - x|^2 of the gather test (gather.hpp:54): dot(d, d) = ((dx dx) + (dy dy)) + dz dz, with
// the x and y lanes on packed fp32 pairs (same per-lane rounding)
__device__ __forceinline__ float gather_d2(const float4& p, V3 x) {
#if PRX_F32X2
    float qx, qy;
    const unsigned long long d = f2_sub(f2_pack(p.x, p.y), f2_pack(x.x, x.y));
    f2_unpack(f2_mul(d, d), qx, qy);
    const float dz = p.z - x.z;
    return (qx + qy) + dz * dz;
#else
    const V3 d = sub(V3{p.x, p.y, p.z}, x);
    return dot(d, d);
#endif
}

__global__ void k_gbuffer(SceneDev S, CamDev C, float4* gbuf) {
    const uint32_t n = C.w * C.h;
    for (uint32_t pix = blockIdx.x * blockDim.x + threadIdx.x; pix < n; pix += gridDim.x * blockDim.x) {
        const uint32_t px = pix % C.w, py = pix / C.w;
        // camera_ray (gather.cpp:22-33)
        const float sx = (2.0f * ((float)px + 0.5f) / (float)C.w - 1.0f) * C.tan_half * C.aspect;
        const float sy = (1.0f - 2.0f * ((float)py + 0.5f) / (float)C.h) * C.tan_half;
        const V3 dir = normalized(add(add(C.fwd, mul(C.right, sx)), mul(C.up, sy)));
        Hit h;
        if (intersect_scene(S, C.pos, dir, 0.0f, h))
            gbuf[pix] = make_float4(h.pos.x, h.pos.y, h.pos.z, __uint_as_float(h.obj));
        else
            gbuf[pix] = make_float4(0.f, 0.f, 0.f, __uint_as_float(kInvalidObj));
    }
}

// every hit pixel registers its 27 neighbour-cell keys in an open-addressing table (the
// cells any pixel can read: the photons of other cells never contribute).  Pixels of a warp
// that share a home cell register its neighbours once, split over those pixels.
__device__ __forceinline__ void insert_key(unsigned long long* keys, unsigned long long key, int bits) {
    const uint32_t mask = (1u << bits) - 1u;
    uint32_t s = slot_of(key, bits);
    // (bounded: a full table drops the key; the occupied-slot count then equals the table
    // size, which the host reads as an overflow and rebuilds at full size)
    for (uint32_t probe = 0; probe <= mask; ++probe) {
        const unsigned long long prev = atomicCAS(&keys[s], kEmptyKey, key);
        if (prev == kEmptyKey || prev == key) break;
        s = (s + 1) & mask;
    }
}

// small images: one thread per (pixel, neighbour) -- enough threads to hide the CAS latency
__global__ void k_pixcells_each(const float4* __restrict__ gbuf, uint32_t npx, float r, unsigned long long* keys,
                                int bits) {
    for (uint32_t w = blockIdx.x * blockDim.x + threadIdx.x; w < 27u * npx; w += gridDim.x * blockDim.x) {
        const uint32_t pix = w / 27u, o = w % 27u;
        const float4 g = gbuf[pix];
        if (__float_as_uint(g.w) == kInvalidObj) continue;
        insert_key(keys,
                   grid_key(cell_coord(g.x, r) + (long long)(o % 3) - 1, cell_coord(g.y, r) + (long long)((o / 3) % 3) - 1,
                            cell_coord(g.z, r) + (long long)(o / 9) - 1),
                   bits);
    }
}

__global__ void k_pixcells(const float4* __restrict__ gbuf, uint32_t npx, float r, unsigned long long* keys,
                           int bits) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t base = blockIdx.x * blockDim.x; base < npx; base += stride) {  // warp-uniform trips
        const uint32_t pix = base + threadIdx.x;
        bool hit = false;
        long long cx = 0, cy = 0, cz = 0;
        if (pix < npx) {
            const float4 g = gbuf[pix];
            hit = __float_as_uint(g.w) != kInvalidObj;
            cx = cell_coord(g.x, r), cy = cell_coord(g.y, r), cz = cell_coord(g.z, r);
        }
        const unsigned long long home = hit ? grid_key(cx, cy, cz) : kEmptyKey;
        const uint32_t peers = __match_any_sync(0xffffffffu, home);
        if (!hit) continue;
        const uint32_t n = __popc(peers), rank = __popc(peers & ((1u << lane) - 1u));
        for (uint32_t o = rank; o < 27u; o += n)
            insert_key(keys, grid_key(cx + (long long)(o % 3) - 1, cy + (long long)((o / 3) % 3) - 1,
                                      cz + (long long)(o / 9) - 1),
                       bits);
    }
}

__global__ void k_slot_used(const unsigned long long* __restrict__ keys, uint32_t slots, uint32_t* used) {
    for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < slots; s += gridDim.x * blockDim.x)
        used[s] = keys[s] != kEmptyKey ? 1u : 0u;
}

// ---------------------------------------------------------------- mode 0: atomic splat
// Binning without order: every live photon whose grid cell some pixel registered is appended
// to a candidate list (block-aggregated: one global atomic per 256 photons) and counted per
// cell (global atomics spread over the cells); the candidates are then scattered into per-cell
// runs by atomic cursors (counting sort, any order inside a cell).
__global__ void __launch_bounds__(kT) k_bin_filter(PathDev P, float radius, const unsigned long long* __restrict__ keys,
                                                   int bits, uint2* __restrict__ cand, uint32_t* __restrict__ n_cand,
                                                   uint32_t* __restrict__ pcnt) {
    __shared__ uint32_t warp_n[kT / 32];
    __shared__ uint32_t block_base;
    const uint32_t mask = (1u << bits) - 1u;
    const size_t total = (size_t)P.n * P.B;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (size_t t0 = (size_t)blockIdx.x * kT; t0 < total; t0 += (size_t)gridDim.x * kT) {  // block-uniform
        const size_t v = t0 + threadIdx.x;
        uint32_t s = 0;
        bool hit = false;
        if (v < total) {
            const float4 po = __ldcs(&P.pos_obj[kVS * (v)]);
            if (__float_as_uint(po.w) != kInvalidObj) {
                const unsigned long long key =
                    grid_key(cell_coord(po.x, radius), cell_coord(po.y, radius), cell_coord(po.z, radius));
                s = slot_of(key, bits);
                unsigned long long k;
                while ((k = __ldg(&keys[s])) != key && k != kEmptyKey) s = (s + 1) & mask;
                hit = k == key;
            }
        }
        const unsigned b = __ballot_sync(0xffffffffu, hit);
        if (lane == 0) warp_n[warp] = __popc(b);
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t sum = 0;
            for (int w = 0; w < kT / 32; ++w) {
                const uint32_t c = warp_n[w];
                warp_n[w] = sum;
                sum += c;
            }
            block_base = sum ? atomicAdd(n_cand, sum) : 0u;
        }
        __syncthreads();
        if (hit) {
            cand[block_base + warp_n[warp] + __popc(b & ((1u << lane) - 1u))] = make_uint2((uint32_t)v, s);
            atomicAdd(&pcnt[s], 1u);
        }
        __syncthreads();
    }
}

__global__ void k_bin_scatter(PathDev P, const uint2* __restrict__ cand, const uint32_t* __restrict__ n_cand,
                              const uint32_t* __restrict__ pstart, uint32_t* __restrict__ cursor, float4* __restrict__ spo,
                              float4* __restrict__ sen) {
    const uint32_t n = *n_cand;
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        const uint2 vs = cand[j];
        const uint32_t at = __ldg(&pstart[vs.y]) + atomicAdd(&cursor[vs.y], 1u);
        spo[at] = __ldg(&P.pos_obj[kVS * (vs.x)]);
        sen[at] = __ldg(&P.energy[kVS * (vs.x)]);
    }
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Per-pixel accumulation, any order: one warp per pixel (work counter), lanes test 32
// candidates at a time and keep per-lane partial sums, one warp reduction per pixel.
__global__ void __launch_bounds__(kT) k_splat_pixels(const float4* __restrict__ gbuf, uint32_t npx, float radius,
                                                     const unsigned long long* __restrict__ keys, int bits,
                                                     const uint32_t* __restrict__ pstart,
                                                     const uint32_t* __restrict__ pcnt, const float4* __restrict__ spo,
                                                     const float4* __restrict__ sen, const float4* __restrict__ mat,
                                                     float inv_pi, float inv_area, uint32_t* work,
                                                     float* __restrict__ img, const uint32_t* __restrict__ pix_list,
                                                     const uint32_t* pix_count) {
    const uint32_t n_items = pix_list ? *pix_count : npx;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t mask = (1u << bits) - 1u;
    const float r2 = radius * radius;
    while (true) {
        uint32_t item = 0;
        if (lane == 0) item = atomicAdd(work, 1u);
        item = __shfl_sync(0xffffffffu, item, 0);
        if (item >= n_items) break;
        const uint32_t pix = pix_list ? pix_list[item] : item;
        const float4 g = gbuf[pix];
        const uint32_t obj = __float_as_uint(g.w);
        if (obj == kInvalidObj) {
            if (lane < 3) img[3 * pix + lane] = 0.0f;
            continue;
        }
        const V3 x{g.x, g.y, g.z};
        const long long cx = cell_coord(g.x, radius), cy = cell_coord(g.y, radius), cz = cell_coord(g.z, radius);
        float ax = 0.0f, ay = 0.0f, az = 0.0f;
        for (int o = 0; o < 27; ++o) {
            const int dx = o % 3 - 1, dy = (o / 3) % 3 - 1, dz = o / 9 - 1;
            const unsigned long long key = grid_key(cx + dx, cy + dy, cz + dz);
            uint32_t s = slot_of(key, bits);
            unsigned long long k;
            while ((k = __ldg(&keys[s])) != key && k != kEmptyKey) s = (s + 1) & mask;
            if (k != key) continue;
            const uint32_t b0 = __ldg(&pstart[s]), n = __ldg(&pcnt[s]);
            // kU candidate loads in flight per lane before the tests, then the contributors'
            // energy loads of the whole step in flight before the adds (latency overlap)
            constexpr int kU = PRX_GATHER_UNROLL;
            for (uint32_t base = 0; base < n; base += 32 * kU) {
                float4 po[kU];
#pragma unroll
                for (int u = 0; u < kU; ++u) {
                    const uint32_t j = base + 32 * u + lane;
                    po[u] = j < n ? __ldg(&spo[b0 + j]) : make_float4(0.f, 0.f, 0.f, __uint_as_float(kInvalidObj));
                }
                float4 en[kU];
#pragma unroll
                for (int u = 0; u < kU; ++u) {
                    const V3 d = sub(V3{po[u].x, po[u].y, po[u].z}, x);  // gather.hpp:54
                    const bool hit = dot(d, d) <= r2 && __float_as_uint(po[u].w) == obj;
                    en[u] = hit ? __ldg(&sen[b0 + base + 32 * u + lane]) : make_float4(0.f, 0.f, 0.f, 0.f);
                }
#pragma unroll
                for (int u = 0; u < kU; ++u) {
                    ax += en[u].x;
                    ay += en[u].y;
                    az += en[u].z;
                }
            }
        }
        ax = warp_sum(ax);
        ay = warp_sum(ay);
        az = warp_sum(az);
        if (lane == 0) {
            const float4 a = mat[obj];
            img[3 * pix] = ((ax * a.x) * inv_pi) * inv_area;  // gather.cpp:71
            img[3 * pix + 1] = ((ay * a.y) * inv_pi) * inv_area;
            img[3 * pix + 2] = ((az * a.z) * inv_pi) * inv_area;
        }
    }
}

// Tiled splat for pixel groups (large images): one warp per chunk of <= 32 pixels sharing a
// home cell (so the same 27 cells).  The chunk's hit points and fp32 accumulators live in
// shared memory; each lane takes one candidate photon of a 32-photon slab and splats it onto
// the chunk's pixels it reaches (same object, |x_ph - x_px|^2 <= r^2) with shared-memory
// atomics, walking the pixels from a lane-rotated start so concurrent adds hit different
// addresses.
__global__ void __launch_bounds__(kT) k_splat_tiles(const float4* __restrict__ gbuf, float radius,
                                                    const unsigned long long* __restrict__ keys, int bits,
                                                    const uint32_t* __restrict__ pstart,
                                                    const uint32_t* __restrict__ pcnt, const float4* __restrict__ spo,
                                                    const float4* __restrict__ sen, const float4* __restrict__ mat,
                                                    float inv_pi, float inv_area, const uint2* __restrict__ chunks,
                                                    const uint32_t* n_chunks, const uint32_t* __restrict__ pv,
                                                    uint32_t* work, float* __restrict__ img) {
    __shared__ float4 s_px[kT];       // per warp: its pixels' hit points {x, obj}
    __shared__ float s_acc[kT * 3];   // per warp: 32 pixels x 3 channels
    const uint32_t lane = threadIdx.x & 31;
    float4* const wpx = s_px + (threadIdx.x & ~31u);
    float* const wacc = s_acc + 3 * (threadIdx.x & ~31u);
    const uint32_t mask = (1u << bits) - 1u;
    const float r2 = radius * radius;
    const uint32_t nch = *n_chunks;
    while (true) {
        uint32_t c = 0;
        if (lane == 0) c = atomicAdd(work, 1u);
        c = __shfl_sync(0xffffffffu, c, 0);
        if (c >= nch) break;
        const uint2 ch = chunks[c];
        const uint32_t m = ch.y;
        __syncwarp();
        if (lane < m) wpx[lane] = gbuf[pv[ch.x + lane]];
        wacc[lane] = 0.0f;
        wacc[32 + lane] = 0.0f;
        wacc[64 + lane] = 0.0f;
        __syncwarp();
        const float4 g0 = wpx[0];
        const uint32_t lane0 = lane % m;
        const long long cx = cell_coord(g0.x, radius), cy = cell_coord(g0.y, radius), cz = cell_coord(g0.z, radius);
        for (int o = 0; o < 27; ++o) {
            const int dx = o % 3 - 1, dy = (o / 3) % 3 - 1, dz = o / 9 - 1;
            const unsigned long long key = grid_key(cx + dx, cy + dy, cz + dz);
            uint32_t s = slot_of(key, bits);
            unsigned long long k;
            while ((k = __ldg(&keys[s])) != key && k != kEmptyKey) s = (s + 1) & mask;
            if (k != key) continue;
            const uint32_t b0 = __ldg(&pstart[s]), n = __ldg(&pcnt[s]);
            for (uint32_t j = lane; j < n; j += 32) {
                const float4 po = __ldg(&spo[b0 + j]);
                const uint32_t obj = __float_as_uint(po.w);
                float4 e;
                bool have = false;
                uint32_t t = lane0;  // lane-rotated pixel walk (no per-step modulo)
                for (uint32_t q = 0; q < m; ++q, t = t + 1 == m ? 0u : t + 1) {
                    const float4 px = wpx[t];
                    const V3 d = sub(V3{po.x, po.y, po.z}, V3{px.x, px.y, px.z});  // gather.hpp:54
                    if (__float_as_uint(px.w) != obj || dot(d, d) > r2) continue;
                    if (!have) {
                        e = __ldg(&sen[b0 + j]);
                        have = true;
                    }
                    atomicAdd(&wacc[3 * t], e.x);
                    atomicAdd(&wacc[3 * t + 1], e.y);
                    atomicAdd(&wacc[3 * t + 2], e.z);
                }
            }
        }
        __syncwarp();
        if (lane < m) {
            const float4 px = wpx[lane];
            const uint32_t pix = pv[ch.x + lane];
            const float4 a = mat[__float_as_uint(px.w)];
            img[3 * pix] = ((wacc[3 * lane] * a.x) * inv_pi) * inv_area;  // gather.cpp:71
            img[3 * pix + 1] = ((wacc[3 * lane + 1] * a.y) * inv_pi) * inv_area;
            img[3 * pix + 2] = ((wacc[3 * lane + 2] * a.z) * inv_pi) * inv_area;
        }
    }
}

// ---------------------------------------------------------------- mode 1: ordered gather
// Bit-exact image: photons are binned by grid cell in ascending flat record order (the
// insertion order of the reference's GatherGrid, gather.cpp:13-20,42-52), and one warp per
// pixel (k_gather_staged) visits its 27 cells in the reference's (dz, dy, dx) order, summing
// contributors strictly in that order -- the same fp32 additions as gather_image's
// per-pixel loop.
// One CTA per sort tile of kSortTile records (record order): finds the candidates (live
// photons whose grid cell some pixel registered, gather.cpp:42-52), counts them per cell, and
// compacts the tile's candidates in record order as (dense cell id, record) pairs at the
// tile's start -- the ragged input of the sort's first pass (no flag array, no separate
// compaction pass).
constexpr int kBinItems = kSortTile / kT;  // 16
__global__ void __launch_bounds__(kT) k_gather_bin(PathDev P, float radius, const unsigned long long* __restrict__ keys,
                                                   int bits, const uint32_t* __restrict__ dense,
                                                   uint32_t* __restrict__ ck, uint32_t* __restrict__ cv,
                                                   uint32_t* __restrict__ tile_cnt, uint32_t* __restrict__ total,
                                                   uint32_t* __restrict__ pcnt) {
    constexpr int kHalf = kBinItems / 2;  // two halves: loads of a half in flight together
    __shared__ uint32_t wsum[kHalf][kT / 32];
    const uint32_t mask = (1u << bits) - 1u;
    const uint64_t nvv = (uint64_t)P.n * P.B;
    const uint64_t base = (uint64_t)blockIdx.x * kSortTile;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t run = 0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        uint32_t cell[kHalf];
        uint32_t fm = 0;
#pragma unroll
        for (int q = 0; q < kHalf; ++q) {
            const uint64_t v = base + (uint64_t)(h * kHalf + q) * kT + threadIdx.x;
            cell[q] = 0;
            if (v < nvv) {
                const float4 po = __ldcs(&P.pos_obj[kVS * (v)]);
                if (__float_as_uint(po.w) != kInvalidObj) {
                    const unsigned long long key =
                        grid_key(cell_coord(po.x, radius), cell_coord(po.y, radius), cell_coord(po.z, radius));
                    uint32_t s = slot_of(key, bits);
                    unsigned long long k;
                    while ((k = __ldg(&keys[s])) != key && k != kEmptyKey) s = (s + 1) & mask;
                    if (k == key) {
                        fm |= 1u << q;
                        cell[q] = __ldg(&dense[s]);  // sort key: dense cell id (slot order)
                        atomicAdd(&pcnt[s], 1u);
                    }
                }
            }
        }
        // one exchange per half: every warp publishes its per-round counts, then each
        // candidate's offset = run + earlier rounds (all warps) + earlier warps + lane rank
        uint32_t ball[kHalf];
#pragma unroll
        for (int q = 0; q < kHalf; ++q) {
            ball[q] = __ballot_sync(0xffffffffu, (fm >> q) & 1u);
            if (lane == 0) wsum[q][warp] = __popc(ball[q]);
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < kHalf; ++q) {
            uint32_t before = 0, tot = 0;
#pragma unroll
            for (int w = 0; w < kT / 32; ++w) {
                const uint32_t c = wsum[q][w];
                before += w < (int)warp ? c : 0u;
                tot += c;
            }
            if ((fm >> q) & 1u) {
                const uint32_t o = run + before + __popc(ball[q] & ((1u << lane) - 1u));
                ck[base + o] = cell[q];
                cv[base + o] = (uint32_t)(base + (uint64_t)(h * kHalf + q) * kT + threadIdx.x);
            }
            run += tot;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        tile_cnt[blockIdx.x] = run;
        if (run) atomicAdd(total, run);
    }
}

// Fused ordered gather, staged: one warp per pixel taken from a work counter (heavy pixels
// cluster in the image, so static striding would pile them onto a few SMs); per 32-photon
// chunk the warp tests the candidates in parallel, compacts the contributors' energies into
// a shared-memory stage in insertion order (ballot prefix), and lanes 0..2 add them
// sequentially, one channel each.  Cells that cannot reach the hit point are skipped.
__device__ __forceinline__ bool cell_reaches(long long ix, long long iy, long long iz, const float4& g, float radius,
                                             float r2) {
    const double rd = radius;
    auto gap = [&](long long i, float x) {  // box widened for the rounding of floor(p / r)
        const double m = 1e-5 * rd * (double)(llabs(i) + 2);
        const double lo = (double)i * rd - m, hi = (double)(i + 1) * rd + m;
        return x < lo ? lo - x : (x > hi ? x - hi : 0.0);
    };
    const double gx = gap(ix, g.x), gy = gap(iy, g.y), gz = gap(iz, g.z);
    return gx * gx + gy * gy + gz * gz <= (double)r2 * (1.0 + 1e-4) + 1e-30;
}

// Conservative reach tests against a box of hit points (pixel groups): false only when every
// point of the box is farther than r from the cell / point even after rounding.
__device__ __forceinline__ bool cell_reaches_box(long long ix, long long iy, long long iz, const float4& bmin,
                                                 const float4& bmax, float radius) {
    const double rd = radius;
    auto gap = [&](long long i, float l, float h) {  // cell widened for the rounding of floor(p / r)
        const double m = 1e-5 * rd * (double)(llabs(i) + 2);
        const double lo = (double)i * rd - m, hi = (double)(i + 1) * rd + m;
        return h < lo ? lo - h : (l > hi ? l - hi : 0.0);
    };
    const double gx = gap(ix, bmin.x, bmax.x), gy = gap(iy, bmin.y, bmax.y), gz = gap(iz, bmin.z, bmax.z);
    return gx * gx + gy * gy + gz * gz <= rd * rd * (1.0 + 1e-4) + 1e-30;
}

__device__ __forceinline__ bool point_reaches_box(const float4& p, const float4& bmin, const float4& bmax,
                                                  float radius) {
    // per-axis gap to the box with an absolute slack for the rounding of p - x in the pixel test
    auto gap = [](float v, float l, float h) {
        const float slack = 1e-5f * (fabsf(v) + fabsf(l) + fabsf(h)) + 1e-30f;
        const float g = v < l ? l - v : (v > h ? v - h : 0.0f);
        return fmaxf(g - slack, 0.0f);
    };
    const float gx = gap(p.x, bmin.x, bmax.x), gy = gap(p.y, bmin.y, bmax.y), gz = gap(p.z, bmin.z, bmax.z);
    return gx * gx + gy * gy + gz * gz <= radius * radius * 1.0001f;
}

__global__ void __launch_bounds__(kT) k_gather_staged(const float4* __restrict__ gbuf, uint32_t npx, float radius,
                                                      const unsigned long long* __restrict__ keys, int bits,
                                                      const uint32_t* __restrict__ pstart,
                                                      const uint32_t* __restrict__ pcnt,
                                                      const float4* __restrict__ spo, const float4* __restrict__ sen,
                                                      const float4* __restrict__ mat, float inv_pi, float inv_area,
                                                      uint32_t* work, float* __restrict__ img,
                                                      const uint32_t* __restrict__ pix_list, const uint32_t* pix_count) {
    __shared__ float4 stage[kT];
    const uint32_t n_items = pix_list ? *pix_count : npx;
    const uint32_t lane = threadIdx.x & 31;
    float4* const my = stage + (threadIdx.x & ~31u);
    const uint32_t mask = (1u << bits) - 1u;
    const float r2 = radius * radius;
    while (true) {
        uint32_t item = 0;
        if (lane == 0) item = atomicAdd(work, 1u);
        item = __shfl_sync(0xffffffffu, item, 0);
        if (item >= n_items) break;
        const uint32_t pix = pix_list ? pix_list[item] : item;
        const float4 g = gbuf[pix];
        const uint32_t obj = __float_as_uint(g.w);
        if (obj == kInvalidObj) {  // no primary hit: pixel stays 0 (gather.cpp:66)
            if (lane < 3) img[3 * pix + lane] = 0.0f;
            continue;
        }
        const V3 x{g.x, g.y, g.z};
        const long long cx = cell_coord(g.x, radius), cy = cell_coord(g.y, radius), cz = cell_coord(g.z, radius);
        float acc = 0.0f;  // radiance += E (gather.cpp:68), channel `lane` for lanes 0..2
        for (int dz = -1; dz <= 1; ++dz)
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {  // gather.hpp:48-50 visiting order
                    if (!cell_reaches(cx + dx, cy + dy, cz + dz, g, radius, r2)) continue;
                    const unsigned long long key = grid_key(cx + dx, cy + dy, cz + dz);
                    uint32_t s = slot_of(key, bits);
                    unsigned long long k;
                    while ((k = __ldg(&keys[s])) != key && k != kEmptyKey) s = (s + 1) & mask;
                    if (k != key) continue;
                    const uint32_t b0 = __ldg(&pstart[s]), n = __ldg(&pcnt[s]);
                    // kU chunks per step: all candidate loads and contributor loads of the step
                    // are issued before the ordered adds, so L2 latency overlaps kU-fold
                    constexpr int kU = PRX_GATHER_UNROLL;
                    for (uint32_t base = 0; base < n; base += 32 * kU) {
                        float4 po[kU];
#pragma unroll
                        for (int u = 0; u < kU; ++u) {
                            const uint32_t j = base + 32 * u + lane;
                            po[u] = j < n ? __ldg(&spo[b0 + j]) : make_float4(0.f, 0.f, 0.f, __uint_as_float(kInvalidObj));
                        }
                        uint32_t ball[kU];
                        float4 en[kU];
#pragma unroll
                        for (int u = 0; u < kU; ++u) {
                            const V3 d = sub(V3{po[u].x, po[u].y, po[u].z}, x);  // gather.hpp:54
                            const bool hit = dot(d, d) <= r2 && __float_as_uint(po[u].w) == obj;
                            ball[u] = __ballot_sync(0xffffffffu, hit);
                            en[u] = hit ? __ldg(&sen[b0 + base + 32 * u + lane]) : make_float4(0.f, 0.f, 0.f, 0.f);
                        }
#pragma unroll
                        for (int u = 0; u < kU; ++u) {
                            if (!ball[u]) continue;
                            if ((ball[u] >> lane) & 1u) my[__popc(ball[u] & ((1u << lane) - 1u))] = en[u];
                            __syncwarp();
                            if (lane < 3) {
                                const float* col = reinterpret_cast<const float*>(my) + lane;
                                const uint32_t m = __popc(ball[u]);
                                for (uint32_t i = 0; i < m; ++i) acc = acc + col[4 * i];
                            }
                            __syncwarp();
                        }
                    }
                }
        if (lane < 3) {
            const float4 a = mat[obj];
            const float alb = lane == 0 ? a.x : (lane == 1 ? a.y : a.z);
            img[3 * pix + lane] = ((acc * alb) * inv_pi) * inv_area;  // gather.cpp:71
        }
    }
}

// ---- pixel groups: pixels whose hit points share a grid cell share the 27 neighbour cells
// and their visiting order, so one warp can serve up to 32 of them: the warp stages each
// chunk of 32 candidate photons in shared memory and every lane walks the chunk in order for
// its own pixel (same tests, same per-pixel addition order as gather_image).  Pays off when
// many pixels fall in one cell (high resolutions); small groups keep the per-pixel path.
constexpr uint32_t kGroupMin = 12;

__global__ void k_pixel_home(const float4* __restrict__ gbuf, uint32_t npx, float radius,
                             const unsigned long long* __restrict__ keys, int bits, uint32_t* hk, uint32_t* pv) {
    const uint32_t mask = (1u << bits) - 1u;
    for (uint32_t pix = blockIdx.x * blockDim.x + threadIdx.x; pix < npx; pix += gridDim.x * blockDim.x) {
        const float4 g = gbuf[pix];
        uint32_t slot = 1u << bits;  // no hit: sorts last
        if (__float_as_uint(g.w) != kInvalidObj) {
            const unsigned long long key =
                grid_key(cell_coord(g.x, radius), cell_coord(g.y, radius), cell_coord(g.z, radius));
            uint32_t s = slot_of(key, bits);
            while (__ldg(&keys[s]) != key) s = (s + 1) & mask;  // inserted by k_pixcells
            slot = s;
        }
        hk[pix] = slot;
        pv[pix] = pix;
    }
}

__global__ void k_group_heads(const uint32_t* __restrict__ hk, uint32_t npx, uint8_t* head) {
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < npx; j += gridDim.x * blockDim.x)
        head[j] = (j == 0 || hk[j] != hk[j - 1]) ? 1 : 0;
}

// groups of >= kGroupMin hit pixels -> 32-pixel chunks; the rest -> the per-pixel list
__global__ void k_group_split(const uint32_t* __restrict__ starts, const uint32_t* n_groups, uint32_t npx,
                              const uint32_t* __restrict__ hk, const uint32_t* __restrict__ pv, int bits,
                              uint2* chunks, uint32_t* n_chunks, uint32_t* small, uint32_t* n_small) {
    const uint32_t G = *n_groups;
    for (uint32_t g = blockIdx.x * blockDim.x + threadIdx.x; g < G; g += gridDim.x * blockDim.x) {
        const uint32_t b = starts[g], e = g + 1 < G ? starts[g + 1] : npx;
        const uint32_t len = e - b;
        if (hk[b] != (1u << bits) && len >= kGroupMin) {
            const uint32_t nc = (len + 31) / 32;
            const uint32_t c0 = atomicAdd(n_chunks, nc);
            for (uint32_t c = 0; c < nc; ++c) chunks[c0 + c] = make_uint2(b + 32 * c, min(32u, len - 32 * c));
        } else {
            const uint32_t s0 = atomicAdd(n_small, len);
            for (uint32_t k = 0; k < len; ++k) small[s0 + k] = pv[b + k];
        }
    }
}

__global__ void __launch_bounds__(kT) k_gather_groups(const float4* __restrict__ gbuf, float radius,
                                                      const unsigned long long* __restrict__ keys, int bits,
                                                      const uint32_t* __restrict__ pstart,
                                                      const uint32_t* __restrict__ pcnt,
                                                      const float4* __restrict__ spo, const float4* __restrict__ sen,
                                                      const float4* __restrict__ mat, float inv_pi, float inv_area,
                                                      const uint2* __restrict__ chunks, const uint32_t* n_chunks,
                                                      const uint32_t* __restrict__ pv, uint32_t* work,
                                                      float* __restrict__ img) {
    __shared__ float4 s_pos[kT];
    __shared__ float4 s_en[kT];
    const uint32_t lane = threadIdx.x & 31;
    float4* const wpos = s_pos + (threadIdx.x & ~31u);
    float4* const wen = s_en + (threadIdx.x & ~31u);
    const uint32_t mask = (1u << bits) - 1u;
    const float r2 = radius * radius;
    const uint32_t nch = *n_chunks;
    while (true) {
        uint32_t c = 0;
        if (lane == 0) c = atomicAdd(work, 1u);
        c = __shfl_sync(0xffffffffu, c, 0);
        if (c >= nch) break;
        const uint2 ch = chunks[c];
        const bool mine = lane < ch.y;
        const uint32_t pix = mine ? pv[ch.x + lane] : pv[ch.x];
        const float4 g = gbuf[pix];
        const uint32_t obj = __float_as_uint(g.w);
        const V3 x{g.x, g.y, g.z};
        // every pixel of the chunk has this home cell (grouped by it)
        const float4 g0 = gbuf[pv[ch.x]];
        const long long cx = cell_coord(g0.x, radius), cy = cell_coord(g0.y, radius), cz = cell_coord(g0.z, radius);
        // the chunk's hit points' box: candidate photons (and whole cells) farther than r from
        // it reach none of its pixels and are dropped before the per-pixel loop (in order, so
        // each pixel's additions are unchanged); the reach test is conservative (float slack)
        float lo[3] = {x.x, x.y, x.z}, hi[3] = {x.x, x.y, x.z};
        if (!mine) lo[0] = lo[1] = lo[2] = INFINITY, hi[0] = hi[1] = hi[2] = -INFINITY;
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                lo[a] = fminf(lo[a], __shfl_xor_sync(0xffffffffu, lo[a], o));
                hi[a] = fmaxf(hi[a], __shfl_xor_sync(0xffffffffu, hi[a], o));
            }
        const float4 gmin = make_float4(lo[0], lo[1], lo[2], 0.f), gmax = make_float4(hi[0], hi[1], hi[2], 0.f);
        float ax = 0.0f, ay = 0.0f, az = 0.0f;  // radiance += E (gather.cpp:68), per lane
        for (int dz = -1; dz <= 1; ++dz)
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {  // gather.hpp:48-50 visiting order
                    if (!cell_reaches_box(cx + dx, cy + dy, cz + dz, gmin, gmax, radius)) continue;
                    const unsigned long long key = grid_key(cx + dx, cy + dy, cz + dz);
                    uint32_t s = slot_of(key, bits);
                    unsigned long long k;
                    while ((k = __ldg(&keys[s])) != key && k != kEmptyKey) s = (s + 1) & mask;
                    if (k != key) continue;
                    const uint32_t b0 = __ldg(&pstart[s]), n = __ldg(&pcnt[s]);
                    for (uint32_t base = 0; base < n; base += 32) {
                        const uint32_t j = base + lane;
                        float4 cp = make_float4(0.f, 0.f, 0.f, 0.f), ce = cp;
                        bool keep = false;
                        if (j < n) {
                            cp = __ldg(&spo[b0 + j]);
                            keep = point_reaches_box(cp, gmin, gmax, radius);
                            if (keep) ce = __ldg(&sen[b0 + j]);
                        }
                        const uint32_t kb = __ballot_sync(0xffffffffu, keep);
                        __syncwarp();
                        if (keep) {
                            const uint32_t at = __popc(kb & ((1u << lane) - 1u));
                            wpos[at] = cp;
                            wen[at] = ce;
                        }
                        __syncwarp();
                        const uint32_t m = __popc(kb);
                        if (mine) {
                            for (uint32_t q = 0; q < m; ++q) {
                                const float4 po = wpos[q];
                                if (gather_d2(po, x) <= r2 && __float_as_uint(po.w) == obj) {  // gather.hpp:54
                                    const float4 e = wen[q];
                                    ax = ax + e.x;
                                    ay = ay + e.y;
                                    az = az + e.z;
                                }
                            }
                        }
                    }
                }
        if (mine) {
            const float4 a = mat[obj];
            img[3 * pix] = ((ax * a.x) * inv_pi) * inv_area;  // gather.cpp:71
            img[3 * pix + 1] = ((ay * a.y) * inv_pi) * inv_area;
            img[3 * pix + 2] = ((az * a.z) * inv_pi) * inv_area;
        }
    }
}

}  // namespace

// Cell-key table sizes: the worst case is 27 distinct cells per pixel (load <= 1/2); large
// images register far fewer (neighbouring pixels share cells), so they start from a table of
// at most 2^kTableCapBits slots and fall back to the worst-case size when its load passes 3/4.
constexpr int kTableCapBits = 22;
int splat_table_bits(uint32_t npx) {
    uint64_t want = 2ull * 27ull * npx;
    int bits = 10;
    while ((1ull << bits) < want && bits < 30) ++bits;
    return bits;
}
int splat_table_bits_capped(uint32_t npx) {
    int cap = kTableCapBits;
    if (const char* e = std::getenv("PRX_SPLAT_TABLE_CAP")) cap = std::atoi(e) >= 10 ? std::atoi(e) : 10;  // (tests)
    const int b = splat_table_bits(npx);
    return b < cap ? b : cap;
}
bool splat_table_overflow(uint32_t n_cells, int bits) { return 4ull * n_cells > (3ull << bits); }

// the prefix's work buffer: cell-key table (8 B/slot) | dense cell ids (4 B/slot) | the
// registered-cell count | scan scratch
size_t splat_ncell_offset(int bits) { return (1ull << bits) * 12; }
size_t splat_work_bytes(int bits) {
    const uint64_t slots = 1ull << bits;
    return slots * 12 + 256 + prim_scratch_bytes(slots) + 256;
}

size_t gather_work_bytes(uint64_t n_vertices, uint32_t npx, int bits) {
    const uint64_t slots = 1ull << bits;
    const uint64_t nv = n_vertices;
    uint64_t scan_n = nv > slots ? nv : slots;
    if (npx > scan_n) scan_n = npx;
    return 64 + nv * (1 + 4 + 4 + 16 + 32) + slots * 12 + 41ull * npx + 2 * prim_scratch_bytes(scan_n) + 64 * 256;
}

// The photon-independent part of a splat: the G-buffer and the key table of the cells the
// pixels' gather spheres touch. It depends only on the placed scene, the camera and the radius,
// so the engine can run it on a side stream during verify/retrace (Engine::splat_prefix_fork).
void launch_splat_prefix(SceneDev S, const CamDev& C, float radius, float4* gbuf, void* work, int bits,
                         cudaStream_t st) {
    const uint32_t npx = C.w * C.h;
    const uint64_t slots = 1ull << bits;
    auto* keys = static_cast<unsigned long long*>(work);
    auto* dense = reinterpret_cast<uint32_t*>(keys + slots);
    auto* ncell = reinterpret_cast<uint32_t*>(static_cast<char*>(work) + splat_ncell_offset(bits));
    k_gbuffer<<<launch_grid(npx, kT), kT, 0, st>>>(S, C, gbuf);
    cudaMemsetAsync(keys, 0xFF, 8 * slots, st);
    if (npx < (1u << 16))
        k_pixcells_each<<<launch_grid(27ull * npx, kT), kT, 0, st>>>(gbuf, npx, radius, keys, bits);
    else
        k_pixcells<<<launch_grid(npx, kT), kT, 0, st>>>(gbuf, npx, radius, keys, bits);
    // dense cell ids in slot order (the ordered gather sorts by these: fewer key bits)
    k_slot_used<<<launch_grid(slots, kT), kT, 0, st>>>(keys, (uint32_t)slots, dense);
    scan_exclusive_u32(dense, dense, (uint32_t)slots, nullptr, ncell, ncell + 64, st);
    g_launches += 3;  // gbuffer, pixcells, slot flags (the scan counts its own)
}

int splat_cell_bits(uint32_t n_cells) {
    int b = 1;
    while ((1ull << b) < n_cells) ++b;
    return b;
}

void launch_splat(SceneDev S, PathDev P, const CamDev& C, float radius, float4* gbuf, float* img, float inv_pi,
                  float inv_area, void* work, void* cand_buf, int mode, void* gather_buf, int bits,
                  bool prefix_done, int cell_bits, cudaStream_t st, cudaEvent_t photons_read) {
    const uint32_t npx = C.w * C.h;
    const uint64_t slots = 1ull << bits;
    auto* keys = static_cast<unsigned long long*>(work);
    (void)cand_buf;

    if (!prefix_done) launch_splat_prefix(S, C, radius, gbuf, work, bits, st);
    const uint64_t nv = (uint64_t)P.n * P.B;
    // carve the work buffer in 256-byte aligned pieces (float4 / u32 views of any n)
    char* w = static_cast<char*>(gather_buf);
    auto take = [&](size_t bytes) {
        char* p = w;
        w += (bytes + 255) & ~size_t(255);
        return p;
    };
    uint32_t* m_count = reinterpret_cast<uint32_t*>(take(64));
    // Large images: pixels grouped by home cell (sorted), groups of >= kGroupMin pixels cut in
    // 32-pixel chunks, the rest walked per pixel.  Small images go straight to the per-pixel walk.
    const char* genv = std::getenv("PRX_GATHER_GROUPS");
    const bool groups = genv ? genv[0] == '1' : npx >= (1u << 18);
    struct Groups {
        uint32_t *pv, *small, *ctl;
        uint2* chunks;
    };
    auto group_pixels = [&](void* gscratch_unused) {
        (void)gscratch_unused;
        Groups G{};
        uint32_t* hk = reinterpret_cast<uint32_t*>(take(4ull * npx));
        G.pv = reinterpret_cast<uint32_t*>(take(4ull * npx));
        uint32_t* hk2 = reinterpret_cast<uint32_t*>(take(4ull * npx));
        uint32_t* pv2 = reinterpret_cast<uint32_t*>(take(4ull * npx));
        uint8_t* head = reinterpret_cast<uint8_t*>(take(npx));
        uint32_t* starts = reinterpret_cast<uint32_t*>(take(4ull * npx));
        G.chunks = reinterpret_cast<uint2*>(take(8ull * npx));
        G.small = reinterpret_cast<uint32_t*>(take(4ull * npx));
        void* gscratch2 = take(0);
        G.ctl = m_count + 4;  // [0] group count, [1] chunks, [2] small, [3] / [4] work counters
        cudaMemsetAsync(G.ctl, 0, 5 * 4, st);
        k_pixel_home<<<launch_grid(npx, kT), kT, 0, st>>>(gbuf, npx, radius, keys, bits, hk, G.pv);
        radix_sort_pairs(hk, G.pv, hk2, pv2, npx, nullptr, bits + 1, gscratch2, st);
        k_group_heads<<<launch_grid(npx, kT), kT, 0, st>>>(hk, npx, head);
        compact_u8(head, npx, nullptr, 0, starts, G.ctl + 0, gscratch2, st);
        k_group_split<<<launch_grid(npx, kT), kT, 0, st>>>(starts, G.ctl + 0, npx, hk, G.pv, bits, G.chunks, G.ctl + 1,
                                                         G.small, G.ctl + 2);
        g_launches += 3;  // home, heads, split (the prims count their own)
        return G;
    };
    if (mode == 0) {  // atomic splat: unordered binning + tiled shared-memory atomics
        uint2* cand = reinterpret_cast<uint2*>(take(8 * nv));
        float4* spo = reinterpret_cast<float4*>(take(16 * nv));
        float4* sen = reinterpret_cast<float4*>(take(16 * nv));
        uint32_t* pcnt = reinterpret_cast<uint32_t*>(take(4 * slots));
        uint32_t* pstart = reinterpret_cast<uint32_t*>(take(4 * slots));
        uint32_t* pcur = reinterpret_cast<uint32_t*>(take(4 * slots));
        void* gscratch = take(0);
        cudaMemsetAsync(m_count, 0, 64, st);
        cudaMemsetAsync(pcnt, 0, 4 * slots, st);
        cudaMemsetAsync(pcur, 0, 4 * slots, st);
        k_bin_filter<<<launch_grid(nv, kT), kT, 0, st>>>(P, radius, keys, bits, cand, m_count, pcnt);
        scan_exclusive_u32(pcnt, pstart, (uint32_t)slots, nullptr, nullptr, gscratch, st);
        k_bin_scatter<<<launch_grid(nv, kT), kT, 0, st>>>(P, cand, m_count, pstart, pcur, spo, sen);
        g_launches += 2;  // filter, scatter
        if (photons_read) cudaEventRecord(photons_read, st);  // (the photon map is not read past here)
        if (!groups) {
            uint32_t* wq = m_count + 4;  // zeroed above
            k_splat_pixels<<<launch_grid(32ull * npx, kT), kT, 0, st>>>(gbuf, npx, radius, keys, bits, pstart, pcnt,
                                                                        spo, sen, S.mat, inv_pi, inv_area, wq, img,
                                                                        nullptr, nullptr);
            ++g_launches;
            return;
        }
        const Groups G = group_pixels(gscratch);
        // 32-pixel groups: lanes own pixels and accumulate in registers over the shared photon
        // slabs (k_gather_groups) -- measured 3x faster at 1920x1080 than the photon-parallel
        // shared-memory-atomic tiles (k_splat_tiles, PRX_SPLAT_TILES=1; profiles/r02_sweeps.md)
        const char* tenv = std::getenv("PRX_SPLAT_TILES");
        if (tenv && tenv[0] == '1')
            k_splat_tiles<<<launch_grid(32ull * npx / 8 + 32, kT), kT, 0, st>>>(gbuf, radius, keys, bits, pstart, pcnt,
                                                                               spo, sen, S.mat, inv_pi, inv_area,
                                                                               G.chunks, G.ctl + 1, G.pv, G.ctl + 3, img);
        else
            k_gather_groups<<<launch_grid(32ull * npx / 8 + 32, kT), kT, 0, st>>>(
                gbuf, radius, keys, bits, pstart, pcnt, spo, sen, S.mat, inv_pi, inv_area, G.chunks, G.ctl + 1, G.pv,
                G.ctl + 3, img);
        k_splat_pixels<<<launch_grid(32ull * npx, kT), kT, 0, st>>>(gbuf, npx, radius, keys, bits, pstart, pcnt, spo,
                                                                    sen, S.mat, inv_pi, inv_area, G.ctl + 4, img,
                                                                    G.small, G.ctl + 2);
        g_launches += 2;
        return;
    }
    {  // mode 1: ordered, bit-exact gather
        uint32_t* sk = reinterpret_cast<uint32_t*>(take(4 * nv));
        uint32_t* sv = reinterpret_cast<uint32_t*>(take(4 * nv));
        uint32_t* sk2 = reinterpret_cast<uint32_t*>(take(4 * nv));
        uint32_t* sv2 = reinterpret_cast<uint32_t*>(take(4 * nv));
        float4* spo = reinterpret_cast<float4*>(take(16 * nv));
        float4* sen = reinterpret_cast<float4*>(take(16 * nv));
        uint32_t* pcnt = reinterpret_cast<uint32_t*>(take(4 * slots));
        uint32_t* pstart = reinterpret_cast<uint32_t*>(take(4 * slots));
        const uint32_t tiles = (uint32_t)((nv + kSortTile - 1) / kSortTile);
        uint32_t* tile_cnt = reinterpret_cast<uint32_t*>(take(4ull * tiles + 4));
        void* gscratch = take(0);
        cudaMemsetAsync(pcnt, 0, 4 * slots, st);
        cudaMemsetAsync(m_count, 0, 4, st);
        const uint32_t* dense = reinterpret_cast<const uint32_t*>(keys + slots);
        // candidates as (cell, record) pairs in record order per tile, stably sorted by cell;
        // the sort's last pass writes the candidates' {position, object} and energy contiguous
        k_gather_bin<<<tiles, kT, 0, st>>>(P, radius, keys, bits, dense, sk, sv, tile_cnt, m_count, pcnt);
        SortGather pg;
        pg.a = P.pos_obj;
        pg.b = P.energy;
        pg.stride = kVS;
        pg.out_a = spo;
        pg.out_b = sen;
        radix_sort_gather(sk, sv, sk2, sv2, (uint32_t)nv, m_count, cell_bits > 0 ? cell_bits : bits, pg, gscratch,
                          st, tile_cnt);
        if (photons_read) cudaEventRecord(photons_read, st);  // (the photon map is not read past here)
        scan_exclusive_u32(pcnt, pstart, (uint32_t)slots, nullptr, nullptr, gscratch, st);
        g_launches += 1;  // bin (the prims count their own)
        if (!groups) {
            uint32_t* wq = m_count + 4;
            cudaMemsetAsync(wq, 0, 4, st);
            k_gather_staged<<<launch_grid(32ull * npx, kT), kT, 0, st>>>(gbuf, npx, radius, keys, bits, pstart, pcnt,
                                                                         spo, sen, S.mat, inv_pi, inv_area, wq, img,
                                                                         nullptr, nullptr);
            ++g_launches;
            return;
        }
        const Groups G = group_pixels(gscratch);
        k_gather_groups<<<launch_grid(32ull * npx / 8 + 32, kT), kT, 0, st>>>(
            gbuf, radius, keys, bits, pstart, pcnt, spo, sen, S.mat, inv_pi, inv_area, G.chunks, G.ctl + 1, G.pv,
            G.ctl + 3, img);
        k_gather_staged<<<launch_grid(32ull * npx, kT), kT, 0, st>>>(gbuf, npx, radius, keys, bits, pstart, pcnt, spo,
                                                                     sen, S.mat, inv_pi, inv_area, G.ctl + 4, img,
                                                                     G.small, G.ctl + 2);
        g_launches += 2;  // groups, staged
    }
}

}  // namespace prx
