// fast_bvh.h -- the fast traversal's own BVH (see fast_bvh.cpp).
#pragma once

#include <cstdint>
#include <vector>

#include <vector_types.h>

#include "host_scene.h"

namespace prx {

constexpr uint32_t kFastLeaf = 0x80000000u;   // child code: leaf | first << 3 | (count - 1)
constexpr uint32_t kFastEmpty = 0xFFFFFFFFu;  // absent child
constexpr size_t kMaxTreeTris = size_t(1) << 27;  // leaf code `first << 3` stays below bit 30
constexpr int kMaxTraversalDepth = 63;            // device traversal stacks hold 64 entries

struct FastNode {
    Box box[2];
    uint32_t child[2] = {kFastEmpty, kFastEmpty};
};

struct FastBvh {
    std::vector<FastNode> nodes;   // nodes[0] is the root (always internal)
    std::vector<uint32_t> order;   // leaf slot -> reference permutation position
    int depth = 1;                 // internal-node levels (<= 48 by construction)
};

// `tris_ref_order[k]` is the static triangle at reference permutation position k.
FastBvh build_fast_bvh(const std::vector<Tri>& tris_ref_order, float pad);

// The combined dynamic tree's fixed topology (lbvh.cu: refit every frame the movers move):
// one SAH tree per rigid dynamic object, built once over its object-local triangles, under
// a top tree over the objects.  Nodes are in the fast layout with child codes in .w and
// boxes left for the refit; internal node 0 is the root.
struct DynSahTopology {
    std::vector<float4> nodes;      // 4 per internal node: {lo0, c0} {hi0, c1} {lo1, -} {hi1, -}
    std::vector<uint32_t> perm;     // leaf slot -> global dynamic triangle index
    std::vector<uint32_t> leaves;   // 4 per leaf: first slot, count, parent node, side
    std::vector<uint32_t> parent;   // per internal node: parent << 1 | side (root: ~0u)
    std::vector<uint32_t> obj_root; // per object: its root node (~0u: no triangles)
    int depth = 0;                  // internal-node levels of the combined tree
};
// `objects[j]` holds object j's local triangles (global indices tri_begin[j] + i);
// `boxes[j]` is a representative world box (frame 0) that orders the top tree.
DynSahTopology build_dyn_sah(const std::vector<std::vector<Tri>>& objects, const std::vector<uint32_t>& tri_begin,
                             const std::vector<Box>& boxes);

}  // namespace prx
