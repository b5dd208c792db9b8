// lbvh.cu -- per-frame LBVH over every dynamic object (north_star subsystem 2).
//
// The reference brute-forces dynamic meshes behind an AABB gate (scene.cpp:153-165,
// bvh.cpp:108-117) -- its dominant CPU cost.  Here each dynamic object
// with more than 32 triangles gets a fresh binary radix tree every frame it moves:
//   1. 24-bit Morton code of each triangle centroid inside the object's current bounds,
//      keyed (object << 24 | morton), value = object-local triangle index;
//   2. one stable LSD radix sort over all dynamic triangles (prims.cu);
//   3. Karras 2012 hierarchy per object (ties broken by sorted position);
//   4. bottom-up refit with arrival counters; child boxes are stored in the parent and
//      inflated so the float culling of dyn_closest/dyn_any stays conservative.
// The query result is the (t, index)-lexicographic minimum over the object's triangles,
// identical to the reference's linear scan (device_scene.cuh: dyn_closest).
#include "device_scene.cuh"
#include "kernels.h"
#include "prims.h"

namespace prx {

namespace {

constexpr int kT = 256;

__device__ __forceinline__ uint32_t spread8(uint32_t x) {  // 8 bits -> every 3rd bit
    x &= 0xFFu;
    x = (x | (x << 8)) & 0x0300F00Fu;
    x = (x | (x << 4)) & 0x030C30C3u;
    x = (x | (x << 2)) & 0x09249249u;
    return x;
}

__global__ void k_morton(const float4* __restrict__ tris, const uint32_t* __restrict__ tri_obj, uint32_t n,
                         const DynObj* __restrict__ dyn, uint32_t* keys, uint32_t* vals) {
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
        const uint32_t j = tri_obj[t];
        const DynObj D = dyn[j];
        const float4 a = tris[3 * t], e1 = tris[3 * t + 1], e2 = tris[3 * t + 2];
        const float cx = a.x + (e1.x + e2.x) * (1.0f / 3.0f);
        const float cy = a.y + (e1.y + e2.y) * (1.0f / 3.0f);
        const float cz = a.z + (e1.z + e2.z) * (1.0f / 3.0f);
        auto q = [](float v, float lo, float hi) {
            const float ext = hi - lo;
            float u = ext > 0.0f ? (v - lo) / ext : 0.5f;
            u = fminf(fmaxf(u, 0.0f), 1.0f);
            return (uint32_t)fminf(u * 256.0f, 255.0f);
        };
        const uint32_t m = (spread8(q(cx, D.cur.lo.x, D.cur.hi.x)) << 2) |
                           (spread8(q(cy, D.cur.lo.y, D.cur.hi.y)) << 1) | spread8(q(cz, D.cur.lo.z, D.cur.hi.z));
        keys[t] = (j << 24) | m;
        vals[t] = t - D.tri_begin;
    }
}

__device__ __forceinline__ int delta(const uint32_t* __restrict__ k, int n, int i, int j, uint32_t mask) {
    if (j < 0 || j >= n) return -1;
    const uint32_t a = k[i] & mask, b = k[j] & mask;
    if (a == b) return 32 + __clz((uint32_t)(i ^ j));
    return __clz(a ^ b);
}

// Karras 2012: range [lo, hi] of internal node i over sorted keys k[0, n) and its split g
// (left child covers [lo, g], right child [g + 1, hi]).
__device__ __forceinline__ void karras_node(const uint32_t* __restrict__ k, int n, int i, uint32_t mask, int& g,
                                            int& lo, int& hi) {
    const int d = (delta(k, n, i, i + 1, mask) - delta(k, n, i, i - 1, mask)) >= 0 ? 1 : -1;
    const int dmin = delta(k, n, i, i - d, mask);
    int lmax = 2;
    while (delta(k, n, i, i + lmax * d, mask) > dmin) lmax <<= 1;
    int l = 0;
    for (int s = lmax >> 1; s >= 1; s >>= 1)
        if (delta(k, n, i, i + (l + s) * d, mask) > dmin) l += s;
    const int jj = i + l * d;
    const int dnode = delta(k, n, i, jj, mask);
    int s = 0;
    int div = 2;
    int step = (l + div - 1) / div;
    while (true) {
        if (delta(k, n, i, i + (s + step) * d, mask) > dnode) s += step;
        if (step <= 1) break;
        div <<= 1;
        step = (l + div - 1) / div;
    }
    g = i + s * d + (d < 0 ? -1 : 0);
    lo = i < jj ? i : jj;
    hi = i < jj ? jj : i;
}

// Karras 2012, one thread per internal node of every object; `keys` sorted.
__global__ void k_karras(const uint32_t* __restrict__ keys, uint32_t n_all, const DynObj* __restrict__ dyn,
                         float4* nodes, uint32_t* parent, uint32_t n_leaf_total) {
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < n_all; t += gridDim.x * blockDim.x) {
        const uint32_t j = keys[t] >> 24;
        const DynObj D = dyn[j];
        if (D.node_begin == kLbvhBrute) continue;
        const int n = (int)D.tri_count;
        const int i = (int)(t - D.tri_begin);
        if (i >= n - 1) continue;
        int g, lo, hi;
        karras_node(keys + D.tri_begin, n, i, 0xFFFFFFu, g, lo, hi);
        const uint32_t left = (lo == g) ? (kLeafBit | (uint32_t)g) : (uint32_t)g;
        const uint32_t right = (hi == g + 1) ? (kLeafBit | (uint32_t)(g + 1)) : (uint32_t)(g + 1);
        float4* N = nodes + 4ull * (D.node_begin + i);
        N[0].w = __uint_as_float(left);
        N[2].w = __uint_as_float(right);
        // parents: leaves by sorted position, internals after n_leaf_total
        const uint32_t me = D.node_begin + (uint32_t)i;
        if (left & kLeafBit) parent[D.tri_begin + g] = me;
        else parent[n_leaf_total + D.node_begin + g] = me;
        if (right & kLeafBit) parent[D.tri_begin + g + 1] = me;
        else parent[n_leaf_total + D.node_begin + g + 1] = me;
        if (i == 0) parent[n_leaf_total + D.node_begin] = 0xFFFFFFFFu;
    }
}

// Bottom-up refit: each leaf walks up; the second arrival at a node unions its children.
__global__ void k_refit(const float4* __restrict__ tris, const uint32_t* __restrict__ keys,
                        const uint32_t* __restrict__ leaf, uint32_t n_all, const DynObj* __restrict__ dyn,
                        float4* nodes, const uint32_t* __restrict__ parent, uint32_t* flags,
                        uint32_t n_leaf_total) {
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < n_all; t += gridDim.x * blockDim.x) {
        const uint32_t j = keys[t] >> 24;
        const DynObj D = dyn[j];
        if (D.node_begin == kLbvhBrute) continue;
        const uint32_t pos = t - D.tri_begin;
        const uint32_t tri = D.tri_begin + leaf[t];
        const float4 a = tris[3 * tri], e1 = tris[3 * tri + 1], e2 = tris[3 * tri + 2];
        const float ext = fmaxf(fmaxf(D.cur.hi.x - D.cur.lo.x, D.cur.hi.y - D.cur.lo.y), D.cur.hi.z - D.cur.lo.z);
        const float bx = a.x + e1.x, by = a.y + e1.y, bz = a.z + e1.z;
        const float cx = a.x + e2.x, cy = a.y + e2.y, cz = a.z + e2.z;
        float lox = fminf(a.x, fminf(bx, cx)), hix = fmaxf(a.x, fmaxf(bx, cx));
        float loy = fminf(a.y, fminf(by, cy)), hiy = fmaxf(a.y, fmaxf(by, cy));
        float loz = fminf(a.z, fminf(bz, cz)), hiz = fmaxf(a.z, fmaxf(bz, cz));
        const float mag = fmaxf(fmaxf(fabsf(lox), fabsf(hix)), fmaxf(fmaxf(fabsf(loy), fabsf(hiy)),
                                                                      fmaxf(fabsf(loz), fabsf(hiz))));
        const float m = 1e-5f * ext + 4e-6f * mag + 1e-30f;
        lox -= m, loy -= m, loz -= m, hix += m, hiy += m, hiz += m;
        uint32_t child = kLeafBit | pos;
        uint32_t p = parent[D.tri_begin + pos];
        while (p != 0xFFFFFFFFu) {
            float4* N = nodes + 4ull * p;
            const bool is_left = __float_as_uint(__ldcg(&N[0].w)) == child;
            const int o = is_left ? 0 : 2;
            N[o].x = lox, N[o].y = loy, N[o].z = loz;
            N[o + 1] = make_float4(hix, hiy, hiz, 0.f);
            __threadfence();
            if (atomicAdd(&flags[p], 1u) == 0) break;  // sibling not done yet
            __threadfence();
            const int q = is_left ? 2 : 0;
            const float4 smin = __ldcg(&N[q]), smax = __ldcg(&N[q + 1]);
            lox = fminf(lox, smin.x), loy = fminf(loy, smin.y), loz = fminf(loz, smin.z);
            hix = fmaxf(hix, smax.x), hiy = fmaxf(hiy, smax.y), hiz = fmaxf(hiz, smax.z);
            child = p - D.node_begin;
            p = parent[n_leaf_total + p];
        }
    }
}

__global__ void k_copy_leaf(const uint32_t* __restrict__ vals, uint32_t n, uint32_t* leaf) {
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) leaf[t] = vals[t];
}

// ---------------------------------------------------------------- combined tree
// One Karras tree over ALL dynamic triangles (full 32-bit key: object, then Morton), in the
// fast-tree layout of fast_bvh.h ({lo0, c0} {hi0, c1} {lo1, -} {hi1, -}, leaf code
// kLeafBit | position << 3), walked by fast_closest for the certified dynamic phase
// (device_scene.cuh: dyn_closest_exact).  Leaves are the triangles themselves, copied in
// sorted order with their global index (== (object, index) order) in a.w.
__global__ void k_karras_all(const uint32_t* __restrict__ keys, uint32_t n, float4* nodes, uint32_t* parent,
                             uint2* range) {
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t + 1 < n; t += gridDim.x * blockDim.x) {
        int g, lo, hi;
        karras_node(keys, (int)n, (int)t, 0xFFFFFFFFu, g, lo, hi);
        range[t] = make_uint2((uint32_t)lo, (uint32_t)hi);
        const uint32_t left = (lo == g) ? (kLeafBit | ((uint32_t)g << 3)) : (uint32_t)g;
        const uint32_t right = (hi == g + 1) ? (kLeafBit | ((uint32_t)(g + 1) << 3)) : (uint32_t)(g + 1);
        float4* N = nodes + 4ull * t;
        N[0].w = __uint_as_float(left);
        N[1].w = __uint_as_float(right);
        if (left & kLeafBit) parent[g] = t;
        else parent[n + g] = t;
        if (right & kLeafBit) parent[g + 1] = t;
        else parent[n + g + 1] = t;
        if (t == 0) parent[n] = 0xFFFFFFFFu;
    }
}

// Leaf collapse: a child subtree spanning <= kCollapse sorted triangles becomes one leaf
// (Karras ranges are contiguous in sorted order, and the triangles are stored that way), so
// the walk tests a few triangles instead of descending the last levels one box at a time.
// Runs after the refit, which still needs the binary child codes.
#ifndef PRX_COLLAPSE
#define PRX_COLLAPSE 4
#endif
constexpr uint32_t kCollapse = PRX_COLLAPSE;
__global__ void k_collapse_all(uint32_t n, float4* nodes, const uint2* __restrict__ range) {
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t + 1 < n; t += gridDim.x * blockDim.x) {
        float4* N = nodes + 4ull * t;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const uint32_t code = __float_as_uint(N[c].w);
            if (code & kLeafBit) continue;
            const uint2 r = range[code];
            const uint32_t cnt = r.y - r.x + 1;
            if (cnt <= kCollapse) N[c].w = __uint_as_float(kLeafBit | (r.x << 3) | (cnt - 1));
        }
    }
}

__global__ void k_sorted_tris(const float4* __restrict__ tris, const uint32_t* __restrict__ keys,
                              const uint32_t* __restrict__ vals, uint32_t n, const DynObj* __restrict__ dyn,
                              float4* out) {
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
        const uint32_t j = keys[t] >> 24;
        const uint32_t g = dyn[j].tri_begin + vals[t];
        float4 a = tris[3 * g], e1 = tris[3 * g + 1], e2 = tris[3 * g + 2];
        a.w = __uint_as_float(g);
        e1.w = __uint_as_float(j);
        e2.w = 0.0f;
        out[kFT * t] = a;
        out[kFT * t + 1] = e1;
        out[kFT * t + 2] = e2;
    }
}

// internal child codes of the combined tree -> indices into the static tree's node array
__global__ void k_offset_codes(uint32_t n_nodes, float4* nodes, uint32_t off) {
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < n_nodes; t += gridDim.x * blockDim.x) {
        float4* N = nodes + 4ull * t;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const uint32_t code = __float_as_uint(N[c].w);
            if (code != 0xFFFFFFFFu && !(code & kLeafBit)) N[c].w = __uint_as_float(code + off);
        }
    }
}

__global__ void k_refit_all(const float4* __restrict__ stris, uint32_t n, const DynObj* __restrict__ dyn,
                            float4* nodes, const uint32_t* __restrict__ parent, uint32_t* flags) {
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
        const float4 a = stris[kFT * t], e1 = stris[kFT * t + 1], e2 = stris[kFT * t + 2];
        const DynObj D = dyn[__float_as_uint(e1.w)];
        const float ext = fmaxf(fmaxf(D.cur.hi.x - D.cur.lo.x, D.cur.hi.y - D.cur.lo.y), D.cur.hi.z - D.cur.lo.z);
        const float bx = a.x + e1.x, by = a.y + e1.y, bz = a.z + e1.z;
        const float cx = a.x + e2.x, cy = a.y + e2.y, cz = a.z + e2.z;
        float lox = fminf(a.x, fminf(bx, cx)), hix = fmaxf(a.x, fmaxf(bx, cx));
        float loy = fminf(a.y, fminf(by, cy)), hiy = fmaxf(a.y, fmaxf(by, cy));
        float loz = fminf(a.z, fminf(bz, cz)), hiz = fmaxf(a.z, fmaxf(bz, cz));
        const float mag = fmaxf(fmaxf(fabsf(lox), fabsf(hix)), fmaxf(fmaxf(fabsf(loy), fabsf(hiy)),
                                                                      fmaxf(fabsf(loz), fabsf(hiz))));
        const float m = 1e-5f * ext + 4e-6f * mag + 1e-30f;
        lox -= m, loy -= m, loz -= m, hix += m, hiy += m, hiz += m;
        uint32_t child = kLeafBit | (t << 3);
        uint32_t p = parent[t];
        while (p != 0xFFFFFFFFu) {
            float4* N = nodes + 4ull * p;
            const bool is_left = __float_as_uint(__ldcg(&N[0].w)) == child;
            const int o = is_left ? 0 : 2;
            N[o].x = lox, N[o].y = loy, N[o].z = loz;
            N[o + 1].x = hix, N[o + 1].y = hiy, N[o + 1].z = hiz;
            __threadfence();
            if (atomicAdd(&flags[p], 1u) == 0) break;  // sibling not done yet
            __threadfence();
            const int q = is_left ? 2 : 0;
            const float4 smin = __ldcg(&N[q]), smax = __ldcg(&N[q + 1]);
            lox = fminf(lox, smin.x), loy = fminf(loy, smin.y), loz = fminf(loz, smin.z);
            hix = fmaxf(hix, smax.x), hiy = fmaxf(hiy, smax.y), hiz = fmaxf(hiz, smax.z);
            child = p;
            p = parent[n + p];
        }
    }
}

// ---------------------------------------------------------------- fixed SAH topology
// The movers are rigid, so a per-object SAH tree built once over the local triangles stays
// a good tree under the frame's transform: each frame only the leaves (triangles copied into
// slot order) and the boxes (bottom-up refit) change.
__global__ void k_dsah_tris(const float4* __restrict__ tris, const uint32_t* __restrict__ tri_obj,
                            const uint32_t* __restrict__ perm, uint32_t n, float4* out) {
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
        const uint32_t g = perm[t];
        float4 a = tris[3 * g], e1 = tris[3 * g + 1], e2 = tris[3 * g + 2];
        a.w = __uint_as_float(g);
        e1.w = __uint_as_float(tri_obj[g]);
        e2.w = 0.0f;
        out[kFT * t] = a;
        out[kFT * t + 1] = e1;
        out[kFT * t + 2] = e2;
    }
}

// one thread per leaf: the union of its (padded, as k_refit_all) triangle boxes goes into
// the parent's child slot; the second arrival at a node carries the union upwards.
__global__ void k_dsah_refit(const float4* __restrict__ stris, const uint4* __restrict__ leaves, uint32_t n_leaves,
                             const DynObj* __restrict__ dyn, float4* nodes, const uint32_t* __restrict__ parent,
                             uint32_t* flags) {
    for (uint32_t l = blockIdx.x * blockDim.x + threadIdx.x; l < n_leaves; l += gridDim.x * blockDim.x) {
        const uint4 L = leaves[l];
        float lox = INFINITY, loy = INFINITY, loz = INFINITY, hix = -INFINITY, hiy = -INFINITY, hiz = -INFINITY;
        for (uint32_t t = L.x; t < L.x + L.y; ++t) {
            const float4 a = stris[kFT * t], e1 = stris[kFT * t + 1], e2 = stris[kFT * t + 2];
            const DynObj D = dyn[__float_as_uint(e1.w)];
            const float ext = fmaxf(fmaxf(D.cur.hi.x - D.cur.lo.x, D.cur.hi.y - D.cur.lo.y), D.cur.hi.z - D.cur.lo.z);
            const float bx = a.x + e1.x, by = a.y + e1.y, bz = a.z + e1.z;
            const float cx = a.x + e2.x, cy = a.y + e2.y, cz = a.z + e2.z;
            float tlx = fminf(a.x, fminf(bx, cx)), thx = fmaxf(a.x, fmaxf(bx, cx));
            float tly = fminf(a.y, fminf(by, cy)), thy = fmaxf(a.y, fmaxf(by, cy));
            float tlz = fminf(a.z, fminf(bz, cz)), thz = fmaxf(a.z, fmaxf(bz, cz));
            const float mag = fmaxf(fmaxf(fmaxf(fabsf(tlx), fabsf(thx)), fmaxf(fabsf(tly), fabsf(thy))),
                                    fmaxf(fabsf(tlz), fabsf(thz)));
            const float m = 1e-5f * ext + 4e-6f * mag + 1e-30f;
            lox = fminf(lox, tlx - m), loy = fminf(loy, tly - m), loz = fminf(loz, tlz - m);
            hix = fmaxf(hix, thx + m), hiy = fmaxf(hiy, thy + m), hiz = fmaxf(hiz, thz + m);
        }
        uint32_t p = L.z, side = L.w;
        while (true) {
            float4* N = nodes + 4ull * p;
            const int o = side ? 2 : 0;
            N[o].x = lox, N[o].y = loy, N[o].z = loz;
            N[o + 1].x = hix, N[o + 1].y = hiy, N[o + 1].z = hiz;
            const uint32_t sib = __float_as_uint(__ldcg(&N[side ? 0 : 1].w));
            if (sib != 0xFFFFFFFFu) {  // two children: the second arrival continues
                __threadfence();
                if (atomicAdd(&flags[p], 1u) == 0) break;
                __threadfence();
                const int q = side ? 0 : 2;
                const float4 smin = __ldcg(&N[q]), smax = __ldcg(&N[q + 1]);
                lox = fminf(lox, smin.x), loy = fminf(loy, smin.y), loz = fminf(loz, smin.z);
                hix = fmaxf(hix, smax.x), hiy = fmaxf(hiy, smax.y), hiz = fmaxf(hiz, smax.z);
            }
            const uint32_t pp = parent[p];
            if (pp == 0xFFFFFFFFu) break;
            p = pp >> 1;
            side = pp & 1u;
        }
    }
}

}  // namespace

void build_dynamic_lbvh(const float4* world_tris, const uint32_t* tri_obj, uint32_t n_tris,
                        const DynObj* dyn_host, uint32_t n_dyn, const DynObj* dyn_dev, float4* nodes,
                        uint32_t* leaf, const LbvhBuffers& buf, cudaStream_t st) {
    (void)dyn_host;
    (void)n_dyn;
    if (n_tris < 2) return;
    const int g = launch_grid(n_tris, kT);
    const bool sah = buf.all_nodes && buf.sah_perm;
    if (sah) {  // combined tree: fixed SAH topology, refit
        k_dsah_tris<<<g, kT, 0, st>>>(world_tris, tri_obj, buf.sah_perm, n_tris, buf.all_tris);
        cudaMemsetAsync(buf.flags, 0, 4ull * buf.n_sah_nodes, st);
        k_dsah_refit<<<launch_grid(buf.n_sah_leaves, kT), kT, 0, st>>>(buf.all_tris, buf.sah_leaf, buf.n_sah_leaves,
                                                                      dyn_dev, buf.all_nodes, buf.sah_parent,
                                                                      buf.flags);
        g_launches += 2;
        if (!nodes) return;
    }
    k_morton<<<g, kT, 0, st>>>(world_tris, tri_obj, n_tris, dyn_dev, buf.keys, buf.vals);
    radix_sort_pairs(buf.keys, buf.vals, buf.keys_tmp, buf.vals_tmp, n_tris, nullptr, 31, buf.scratch, st);
    ++g_launches;  // (the sort counts its own)
    if (nodes) {  // per-object trees (sequential fallback and DFS mode)
        k_copy_leaf<<<g, kT, 0, st>>>(buf.vals, n_tris, leaf);
        k_karras<<<g, kT, 0, st>>>(buf.keys, n_tris, dyn_dev, nodes, buf.parent, n_tris);
        cudaMemsetAsync(buf.flags, 0, 4ull * n_tris, st);
        k_refit<<<g, kT, 0, st>>>(world_tris, buf.keys, leaf, n_tris, dyn_dev, nodes, buf.parent, buf.flags, n_tris);
        g_launches += 3;
    }
    if (buf.all_nodes && !sah) {  // combined tree (fast dynamic phase), Karras
        k_sorted_tris<<<g, kT, 0, st>>>(world_tris, buf.keys, buf.vals, n_tris, dyn_dev, buf.all_tris);
        uint2* range = reinterpret_cast<uint2*>(buf.keys_tmp);  // free after the sort (2n words)
        k_karras_all<<<g, kT, 0, st>>>(buf.keys, n_tris, buf.all_nodes, buf.parent, range);
        cudaMemsetAsync(buf.flags, 0, 4ull * n_tris, st);
        k_refit_all<<<g, kT, 0, st>>>(buf.all_tris, n_tris, dyn_dev, buf.all_nodes, buf.parent, buf.flags);
        k_collapse_all<<<g, kT, 0, st>>>(n_tris, buf.all_nodes, range);
        g_launches += 4;
        if (buf.code_off) {
            k_offset_codes<<<g, kT, 0, st>>>(n_tris - 1, buf.all_nodes, buf.code_off);
            ++g_launches;
        }
    }
}

}  // namespace prx
