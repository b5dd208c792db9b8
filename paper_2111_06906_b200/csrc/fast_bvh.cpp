// fast_bvh.cpp -- binned-SAH BVH2 over the static triangles for the fast traversal.
//
// The certified fast traversal (device_scene.cuh: static_fast) returns the (t, reference
// permutation position)-minimum over all static triangles, which is independent of the
// tree it walks; exactness w.r.t. the reference's own median-split tree is established
// afterwards by the certificate.  So this tree is free to be built for speed: binned SAH
// (Wald 2007), leaves of <= 8 triangles, child boxes stored in the parent (one 64-byte node
// fetch per traversal step) and inflated by `pad` so that float culling stays conservative.
#include "fast_bvh.h"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <stdexcept>

namespace prx {

namespace {

constexpr int kMaxBins = 64;
// The traversal kernels keep a 64-entry stack (device_scene.cuh: fast_closest /
// joint_closest push at most one entry per level).  The binned SAH has no depth bound on
// adversarial inputs (clustered or log-spaced centroids peel off a few triangles per
// level), so a subtree that could not finish within g_max_depth levels is split at its
// centroid median instead, which needs at most ceil(log2(n / 2)) more levels.
int g_max_depth = 48;  // PRX_SAH_MAXDEPTH overrides (tests: measure the uncapped depth)

int ceil_log2(uint32_t n) {
    int d = 0;
    while ((1ull << d) < n) ++d;
    return d;
}
// build knobs (PRX_SAH_BINS / PRX_SAH_TRAV / PRX_SAH_MAXLEAF override, for tuning runs)
int g_bins = 16;
float g_trav = 1.0f;
uint32_t g_max_leaf = 8;

struct Prim {
    Box box;
    V3 c;
};

float area(const Box& b) {
    const V3 e = sub(b.hi, b.lo);
    if (e.x < 0.0f || e.y < 0.0f || e.z < 0.0f) return 0.0f;
    return 2.0f * (e.x * e.y + e.y * e.z + e.z * e.x);
}

struct Builder {
    const std::vector<Prim>& prims;
    std::vector<uint32_t>& idx;
    std::vector<FastNode>& nodes;

    // Returns the child code for the range [b, e) (leaf code or internal node index).
    int max_depth = 0;  // internal-node levels of the finished tree (root = 1)

    uint32_t build(uint32_t b, uint32_t e, const Box& bounds, int depth = 1) {
        const uint32_t n = e - b;
        if (n <= 2) return leaf(b, n);
        Box cb = empty_box();
        for (uint32_t i = b; i < e; ++i) expand(cb, prims[idx[i]].c);
        if (depth + ceil_log2(n) >= g_max_depth) return median(b, e, cb, depth);
        int best_axis = -1;
        int best_split = 0;
        float best_cost = INFINITY;
        for (int axis = 0; axis < 3; ++axis) {
            const float lo = comp(cb.lo, axis), hi = comp(cb.hi, axis);
            if (!(hi > lo)) continue;
            const int kBins = g_bins;
            Box bb[kMaxBins];
            uint32_t cnt[kMaxBins] = {};
            for (int k = 0; k < kBins; ++k) bb[k] = empty_box();
            const float scale = kBins / (hi - lo);
            for (uint32_t i = b; i < e; ++i) {
                const Prim& p = prims[idx[i]];
                int k = static_cast<int>((comp(p.c, axis) - lo) * scale);
                k = std::min(std::max(k, 0), kBins - 1);
                ++cnt[k];
                expand(bb[k], p.box);
            }
            float right_area[kMaxBins];
            uint32_t right_cnt[kMaxBins];
            Box acc = empty_box();
            uint32_t c = 0;
            for (int k = kBins - 1; k > 0; --k) {
                expand(acc, bb[k]);
                c += cnt[k];
                right_area[k] = area(acc);
                right_cnt[k] = c;
            }
            acc = empty_box();
            c = 0;
            for (int k = 0; k < kBins - 1; ++k) {
                expand(acc, bb[k]);
                c += cnt[k];
                if (c == 0 || right_cnt[k + 1] == 0) continue;
                const float cost = area(acc) * c + right_area[k + 1] * right_cnt[k + 1];
                if (cost < best_cost) {
                    best_cost = cost;
                    best_axis = axis;
                    best_split = k + 1;
                }
            }
        }
        const float leaf_cost = area(bounds) * n;
        if (n <= g_max_leaf && (best_axis < 0 || leaf_cost <= best_cost + area(bounds) * g_trav)) return leaf(b, n);
        uint32_t mid;
        if (best_axis < 0) {  // all centroids coincide: split in the middle
            mid = b + n / 2;
        } else {
            const float lo = comp(cb.lo, best_axis), hi = comp(cb.hi, best_axis);
            const int kBins = g_bins;
            const float scale = kBins / (hi - lo);
            auto it = std::partition(idx.begin() + b, idx.begin() + e, [&](uint32_t i) {
                int k = static_cast<int>((comp(prims[i].c, best_axis) - lo) * scale);
                k = std::min(std::max(k, 0), kBins - 1);
                return k < best_split;
            });
            mid = static_cast<uint32_t>(it - idx.begin());
            if (mid == b || mid == e) mid = b + n / 2;
        }
        return internal(b, mid, e, depth);
    }

    // centroid-median split on the widest centroid axis (the depth-bounded fallback)
    uint32_t median(uint32_t b, uint32_t e, const Box& cb, int depth) {
        const V3 ext = sub(cb.hi, cb.lo);
        const int axis = ext.x >= ext.y && ext.x >= ext.z ? 0 : (ext.y >= ext.z ? 1 : 2);
        const uint32_t mid = b + (e - b) / 2;
        std::nth_element(idx.begin() + b, idx.begin() + mid, idx.begin() + e, [&](uint32_t i, uint32_t j) {
            const float ci = comp(prims[i].c, axis), cj = comp(prims[j].c, axis);
            return ci < cj || (ci == cj && i < j);
        });
        return internal(b, mid, e, depth);
    }

    uint32_t internal(uint32_t b, uint32_t mid, uint32_t e, int depth) {
        max_depth = std::max(max_depth, depth);
        Box lb = empty_box(), rb = empty_box();
        for (uint32_t i = b; i < mid; ++i) expand(lb, prims[idx[i]].box);
        for (uint32_t i = mid; i < e; ++i) expand(rb, prims[idx[i]].box);
        const uint32_t me = static_cast<uint32_t>(nodes.size());
        nodes.emplace_back();
        const uint32_t l = build(b, mid, lb, depth + 1);
        const uint32_t r = build(mid, e, rb, depth + 1);
        FastNode& nd = nodes[me];
        nd.box[0] = lb;
        nd.box[1] = rb;
        nd.child[0] = l;
        nd.child[1] = r;
        return me;
    }

    uint32_t leaf(uint32_t b, uint32_t n) {
        if (n > 8) {  // leaf codes hold <= 8 triangles: split evenly
            Box lb = empty_box(), rb = empty_box();
            const uint32_t mid = b + n / 2;
            for (uint32_t i = b; i < mid; ++i) expand(lb, prims[idx[i]].box);
            for (uint32_t i = mid; i < b + n; ++i) expand(rb, prims[idx[i]].box);
            const uint32_t me = static_cast<uint32_t>(nodes.size());
            nodes.emplace_back();
            const uint32_t l = leaf(b, mid - b), r = leaf(mid, b + n - mid);
            nodes[me].box[0] = lb;
            nodes[me].box[1] = rb;
            nodes[me].child[0] = l;
            nodes[me].child[1] = r;
            return me;
        }
        return kFastLeaf | (b << 3) | (n - 1);
    }
};

}  // namespace

FastBvh build_fast_bvh(const std::vector<Tri>& tris_ref_order, float pad) {
    if (const char* e = std::getenv("PRX_SAH_BINS")) g_bins = std::min(std::max(std::atoi(e), 4), kMaxBins);
    if (const char* e = std::getenv("PRX_SAH_TRAV")) g_trav = static_cast<float>(std::atof(e));
    if (const char* e = std::getenv("PRX_SAH_MAXLEAF"))
        g_max_leaf = static_cast<uint32_t>(std::min(std::max(std::atoi(e), 1), 8));
    if (const char* e = std::getenv("PRX_SAH_MAXDEPTH")) g_max_depth = std::max(std::atoi(e), 8);
    FastBvh out;
    if (tris_ref_order.size() >= kMaxTreeTris)  // leaf codes hold first << 3 below kTreeBit
        throw std::length_error("fast BVH: more than 2^27 - 1 triangles in one tree");
    const uint32_t n = static_cast<uint32_t>(tris_ref_order.size());
    if (n == 0) return out;
    std::vector<Prim> prims(n);
    Box all = empty_box();
    for (uint32_t i = 0; i < n; ++i) {
        prims[i].box = tri_bounds(tris_ref_order[i]);
        prims[i].c = mul(add(prims[i].box.lo, prims[i].box.hi), 0.5f);
        expand(all, prims[i].box);
    }
    out.order.resize(n);
    std::iota(out.order.begin(), out.order.end(), 0u);
    out.nodes.reserve(n);
    out.nodes.emplace_back();  // root placeholder: the root is always an internal node
    Builder B{prims, out.order, out.nodes};
    uint32_t root_child[2];
    Box root_box[2];
    if (n == 1) {
        root_child[0] = kFastLeaf | 0u;
        root_child[1] = kFastEmpty;
        root_box[0] = prims[0].box;
        root_box[1] = empty_box();
    } else {
        // split the top like any other internal node, then move it into slot 0
        const uint32_t code = B.build(0, n, all);
        out.depth = std::max(1, B.max_depth);
        if (code & kFastLeaf) {
            root_child[0] = code;
            root_child[1] = kFastEmpty;
            root_box[0] = all;
            root_box[1] = empty_box();
        } else {
            root_child[0] = out.nodes[code].child[0];
            root_child[1] = out.nodes[code].child[1];
            root_box[0] = out.nodes[code].box[0];
            root_box[1] = out.nodes[code].box[1];
        }
    }
    out.nodes[0].child[0] = root_child[0];
    out.nodes[0].child[1] = root_child[1];
    out.nodes[0].box[0] = root_box[0];
    out.nodes[0].box[1] = root_box[1];
    for (FastNode& nd : out.nodes)
        for (int c = 0; c < 2; ++c)
            if (nd.child[c] != kFastEmpty) inflate(nd.box[c], pad);
    return out;
}

namespace {

float f_of(uint32_t u) {
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}

// top tree over objects: median split on the widest centroid axis; returns the child code
// (object root / internal top node) of the subtree over objs[lo, hi)
uint32_t build_top(std::vector<uint32_t>& objs, uint32_t lo, uint32_t hi, const std::vector<Box>& boxes,
                   const std::vector<uint32_t>& obj_root, std::vector<FastNode>& top) {
    if (hi - lo == 1) return obj_root[objs[lo]];
    Box cb = empty_box();
    for (uint32_t i = lo; i < hi; ++i) {
        const V3 c = mul(add(boxes[objs[i]].lo, boxes[objs[i]].hi), 0.5f);
        expand(cb, Box{c, c});
    }
    const V3 e = sub(cb.hi, cb.lo);
    const int axis = e.x >= e.y && e.x >= e.z ? 0 : (e.y >= e.z ? 1 : 2);
    auto key = [&](uint32_t j) {
        const V3 c = add(boxes[j].lo, boxes[j].hi);
        return axis == 0 ? c.x : (axis == 1 ? c.y : c.z);
    };
    const uint32_t mid = lo + (hi - lo) / 2;
    std::nth_element(objs.begin() + lo, objs.begin() + mid, objs.begin() + hi,
                     [&](uint32_t a, uint32_t b) { return key(a) < key(b) || (key(a) == key(b) && a < b); });
    const uint32_t me = static_cast<uint32_t>(top.size());
    top.emplace_back();
    const uint32_t l = build_top(objs, lo, mid, boxes, obj_root, top);
    const uint32_t r = build_top(objs, mid, hi, boxes, obj_root, top);
    top[me].child[0] = l;
    top[me].child[1] = r;
    return me;
}

}  // namespace

DynSahTopology build_dyn_sah(const std::vector<std::vector<Tri>>& objects, const std::vector<uint32_t>& tri_begin,
                             const std::vector<Box>& boxes) {
    DynSahTopology out;
    const uint32_t n_obj = static_cast<uint32_t>(objects.size());
    if (n_obj == 0) return out;
    std::vector<FastBvh> trees(n_obj);
    for (uint32_t j = 0; j < n_obj; ++j) trees[j] = build_fast_bvh(objects[j], 0.0f);
    // node numbering: top nodes [0, n_top), then each object's nodes at obj_off[j]
    const uint32_t n_top = std::max<uint32_t>(1, n_obj - 1);
    std::vector<uint32_t> obj_off(n_obj), obj_root(n_obj);
    uint32_t total = n_top;
    for (uint32_t j = 0; j < n_obj; ++j) {
        obj_off[j] = total;
        obj_root[j] = total;  // build_fast_bvh's root (node 0) is always internal
        total += static_cast<uint32_t>(trees[j].nodes.size());
    }
    std::vector<FastNode> top;
    top.reserve(n_top);
    std::vector<uint32_t> objs;  // objects with triangles (an empty mesh has no tree)
    for (uint32_t j = 0; j < n_obj; ++j)
        if (!objects[j].empty()) objs.push_back(j);
    if (objs.size() <= 1) {
        top.emplace_back();
        if (!objs.empty()) top[0].child[0] = obj_root[objs[0]];
    } else {  // the first node made (0) is the root
        build_top(objs, 0, static_cast<uint32_t>(objs.size()), boxes, obj_root, top);
    }
    if (top.size() > n_top) throw std::logic_error("build_dyn_sah: top tree overflow");
    // stack bound of the joint walk: the static root is parked while the dynamic tree is
    // walked, so the combined depth (top median tree + deepest object tree) must stay < 63
    int obj_depth = 0;
    for (uint32_t j = 0; j < n_obj; ++j) obj_depth = std::max(obj_depth, trees[j].depth);
    out.depth = (objs.size() > 1 ? ceil_log2(static_cast<uint32_t>(objs.size())) : 0) + obj_depth;
    if (out.depth + 1 > kMaxTraversalDepth)
        throw std::length_error("dynamic BVH deeper than the traversal stack (too many dynamic objects)");
    out.obj_root.assign(n_obj, ~0u);
    for (uint32_t j : objs) out.obj_root[j] = obj_root[j];
    size_t n_tris_all = 0;
    for (uint32_t j = 0; j < n_obj; ++j) n_tris_all += objects[j].size();
    if (n_tris_all >= kMaxTreeTris) throw std::length_error("dynamic BVH: more than 2^27 - 1 triangles");
    const uint32_t n_tris = static_cast<uint32_t>(n_tris_all);
    out.nodes.assign(4ull * total, float4{0.f, 0.f, 0.f, 0.f});
    out.parent.assign(total, ~0u);
    out.perm.resize(n_tris);
    auto emit = [&](uint32_t node, const FastNode& nd, uint32_t code_off_node, int32_t obj) {
        for (int c = 0; c < 2; ++c) {
            uint32_t code = nd.child[c];
            if (code == kFastEmpty) {
                out.nodes[4ull * node + c].w = f_of(kFastEmpty);
                continue;
            }
            if (code & kFastLeaf) {
                const uint32_t first = ((code & ~kFastLeaf) >> 3) + tri_begin[obj];
                const uint32_t count = (code & 7u) + 1u;
                code = kFastLeaf | (first << 3) | (count - 1u);
                out.leaves.insert(out.leaves.end(), {first, count, node, static_cast<uint32_t>(c)});
            } else {
                code += code_off_node;
                out.parent[code] = node << 1 | static_cast<uint32_t>(c);
            }
            out.nodes[4ull * node + c].w = f_of(code);
        }
    };
    for (uint32_t k = 0; k < top.size(); ++k) emit(k, top[k], 0, -1);
    for (uint32_t j = 0; j < n_obj; ++j) {
        const FastBvh& t = trees[j];
        // only the nodes reachable from the root (build_fast_bvh leaves the node it moved into
        // slot 0 orphaned); unreachable slots keep empty codes and are never refit
        for (uint32_t k = 0; k < t.nodes.size(); ++k) {
            out.nodes[4ull * (obj_off[j] + k)].w = f_of(kFastEmpty);
            out.nodes[4ull * (obj_off[j] + k) + 1].w = f_of(kFastEmpty);
        }
        std::vector<uint32_t> stack{0u};
        while (!stack.empty()) {
            const uint32_t k = stack.back();
            stack.pop_back();
            emit(obj_off[j] + k, t.nodes[k], obj_off[j], static_cast<int32_t>(j));
            for (int c = 0; c < 2; ++c)
                if (t.nodes[k].child[c] != kFastEmpty && !(t.nodes[k].child[c] & kFastLeaf))
                    stack.push_back(t.nodes[k].child[c]);
        }
        for (uint32_t s = 0; s < t.order.size(); ++s) out.perm[tri_begin[j] + s] = tri_begin[j] + t.order[s];
    }
    return out;
}

}  // namespace prx
