// fast_bvh.h -- the fast traversal's own BVH (see fast_bvh.cpp).
#pragma once

#include <cstdint>
#include <vector>

#include "host_scene.h"

namespace prx {

constexpr uint32_t kFastLeaf = 0x80000000u;   // child code: leaf | first << 3 | (count - 1)
constexpr uint32_t kFastEmpty = 0xFFFFFFFFu;  // absent child

struct FastNode {
    Box box[2];
    uint32_t child[2] = {kFastEmpty, kFastEmpty};
};

struct FastBvh {
    std::vector<FastNode> nodes;   // nodes[0] is the root (always internal)
    std::vector<uint32_t> order;   // leaf slot -> reference permutation position
};

// `tris_ref_order[k]` is the static triangle at reference permutation position k.
FastBvh build_fast_bvh(const std::vector<Tri>& tris_ref_order, float pad);

}  // namespace prx
