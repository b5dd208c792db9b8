// Depth of the fast traversal's SAH trees on adversarial inputs: three chains of
// equal small triangles with centroids at ratio^k along x, y and z (log-spaced centroids
// make the binned SAH peel off a few triangles per level).
// usage: bvh_depth <n per chain> <ratio> <size>; prints "<static depth> <dynamic depth> <tris>"
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <vector>

#include "fast_bvh.h"

using namespace prx;

int main(int argc, char** argv) {
    const int n = argc > 1 ? std::atoi(argv[1]) : 200;
    const float ratio = argc > 2 ? static_cast<float>(std::atof(argv[2])) : 1.5f;
    const float s = argc > 3 ? static_cast<float>(std::atof(argv[3])) : 1e-3f;
    std::vector<Tri> tris;
    for (int axis = 0; axis < 3; ++axis)
        for (int k = 0; k < n; ++k) {
            const float c = std::pow(ratio, static_cast<float>(k - n / 2));
            const float du[3] = {-s, s, 0.0f}, dv[3] = {-s, -s, s};
            V3 p[3];
            for (int v = 0; v < 3; ++v) {
                float q[3] = {0.0f, 0.0f, 0.0f};
                q[axis] = c;
                q[(axis + 1) % 3] += du[v];
                q[(axis + 2) % 3] += dv[v];
                p[v] = V3{q[0], q[1], q[2]};
            }
            tris.push_back(Tri{p[0], p[1], p[2]});
        }
    const FastBvh fb = build_fast_bvh(tris, 0.0f);
    // the same chains as 4 dynamic objects under the top tree
    std::vector<std::vector<Tri>> objs(4, tris);
    std::vector<uint32_t> begin(4);
    std::vector<Box> boxes(4);
    for (int j = 0; j < 4; ++j) {
        begin[j] = j * static_cast<uint32_t>(tris.size());
        boxes[j] = Box{V3{float(j), 0, 0}, V3{float(j) + 1, 1, 1}};
    }
    int dyn_depth = -1;  // -1: rejected as deeper than the traversal stack
    try {
        dyn_depth = build_dyn_sah(objs, begin, boxes).depth;
    } catch (const std::length_error&) {
    }
    std::printf("%d %d %zu\n", fb.depth, dyn_depth, tris.size());
    return 0;
}
