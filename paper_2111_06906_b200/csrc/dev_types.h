// dev_types.h -- plain structs shared by the host engine and the device kernels.
#pragma once

#include <stdint.h>

#include "exact_math.h"
#include "prx.h"

#include <cuda_runtime.h>

namespace prx {

constexpr uint32_t kInvalidObj = 0xFFFFFFFFu;
constexpr uint32_t kLeafBit = 0x80000000u;
constexpr int kMaxDyn = 128;
// float4s per triangle record of the fast trees (ftris / datris): {a, .} {e1, .} {e2, .} and a
// pad, so a record is two aligned 32-byte halves (two 256-bit loads, whole sectors)
constexpr int kFT = 4;
constexpr uint8_t kDead = 0, kLive = 1, kReplace = 2;  // engine.cpp:17-19
constexpr uint8_t kNoRetrace = 0xFF;                    // engine.hpp:56
constexpr double kTwoPiD = 6.283185307179586476925286766559;  // 2 * std::numbers::pi
constexpr uint32_t kLbvhBrute = 0xFFFFFFFFu;

struct DynObj {
    uint32_t obj;         // scene object id
    uint32_t tri_begin;   // first triangle in the dynamic triangle arrays
    uint32_t tri_count;
    uint32_t node_begin;  // first LBVH node, kLbvhBrute = linear scan
    Box cur;              // bounds_current (scene.cpp:129)
    uint32_t sah_root;    // its subtree in the combined SAH tree (kLbvhBrute: none)
};

struct LightDev {
    int32_t kind;
    uint32_t begin, end;  // global path block (engine.cpp:76-101)
    int32_t moved;        // engine.cpp:208
    V3 position, normal, tangent, bitangent;
    float scale;
    float radius, half_x, half_y;
    double cos_half;      // light.cpp:36-38 (host libm)
    V3 flux_pp;           // engine.cpp:95-96
    uint32_t ndims, cells;
    uint32_t dims[4];
    uint32_t* dm_t;
    uint32_t* dm_c;
    int32_t xt_force;     // PRX_XT_FORCE=1: every light transcendental takes the exact path (tests)
};

struct FrameParams {
    int32_t frame;
    uint32_t n_lights;
    uint32_t n_dyn;
    uint32_t n_boxes;
    LightDev lights[PRX_MAX_LIGHTS];
    DynObj dyn[kMaxDyn];
    Box boxes[kMaxDyn];  // occlusion boxes (engine.cpp:211-218)
};

struct SceneDev {
    const float4* nodes;       // static BVH: 2 float4 per node {lo, a} {hi, b}
    uint32_t n_nodes;
    const uint32_t* leaf_of;   // permutation position -> reference leaf node
    float cull_pad;            // fast traversal: box inflation for conservative culling
    int32_t fast;              // 1: near-first traversal + exactness certificate
    int32_t cert_off;          // 1: every certificate fails (tests: exercises the exact fallbacks)
    const float4* fnodes;      // fast SAH BVH2: 4 float4 per node {lo0,c0} {hi0,c1} {lo1,-} {hi1,-}
    const float4* ftris;       // its triangles in leaf order: {a, ref position} {e1, obj} {e2, -}
    const float4* stris;       // static tris, BVH order: {a, orig idx} {e1, obj} {e2, -}
    const float4* dtris;       // dynamic tris, world space, object-local index order
    const float4* dnodes;      // LBVH nodes: 4 float4 per internal node
    const uint32_t* dleaf;     // LBVH leaf -> object-local triangle index
    int32_t dfast;             // 1: combined LBVH over all dynamic triangles is built
    const float4* danodes;     // combined LBVH, fast-tree layout (4 float4 per node), at fnodes + 4 dnode_off
    uint32_t dnode_off;        // index of its first node in the fnodes array: its internal child codes
                               // (and per-object roots) are fnodes indices, so one base serves both trees
    const float4* datris;      // dynamic tris in combined-leaf order: {a, global idx} {e1, obj j} {e2, -}
    const uint32_t* dtri_obj;  // global dynamic triangle -> dynamic object j
    const float4* mat;         // per object {albedo, glossy exponent}
    const uint32_t* oflags;    // per object: bit0 dynamic, bit1 glossy, bit2 exact pow table, bits8+ its slot
    const FrameParams* fp;
    float eps;                 // engine.cpp:74
    float two_diag;            // engine.cpp:138
    uint64_t seed_mix;         // mix64(seed) (rng.hpp:36)
    float gather_radius;
    const float2* trig;        // exact cos/sin of 2*pi*k/2^24 from the host libm (or null)
    const float* const* pow_tabs;  // exact powf(k*2^-24, 1/(e+1)) per glossy exponent slot
};

// Per-path and per-vertex device state of one engine (one shard).  Vertex arrays are
// bounce-major [B][n] like the reference PhotonMap (photon_store.cpp:32-36), split into
// 16-byte streams so the verify kernels read exactly {position, object} per vertex.
// Vertex streams (PRX_VERTEX_SOA, build knob): 0 (default) = two interleaved 32-byte record
// streams {pos_obj, energy} {in_dir, out_dir}, each [B][n]; 1 = four 16-byte streams pos_obj |
// energy | in_dir | out_dir.  Measured end to end on C4 (profiles/r02_sweeps.md): the SoA
// streams speed up the sequential pos_obj readers but slow the verify walk and the splat's
// candidate copy (one vertex then touches 4 sectors instead of 2): 10.92 vs 10.63 ms/frame.
// Kernels index vertex v of a stream as stream[kVS * v].
#ifndef PRX_VERTEX_SOA
#define PRX_VERTEX_SOA 0
#endif
constexpr uint32_t kVS = PRX_VERTEX_SOA ? 1u : 2u;

struct PathDev {
    uint32_t n;      // paths held by this engine
    uint32_t base;   // global id of local path 0
    uint32_t B;      // max_bounces
    float4* pos_obj; // {aux.position, photon.object_id}
    float4* energy;  // {photon.energy, photon.radius}
    float4* in_dir;  // {photon.incoming_dir, 0}
    float4* out_dir; // {aux.outgoing, 0}
    float4* origin;
    float4* emis;
    float4* canon;
    uint32_t* cell;
    uint32_t* epoch;
    uint32_t* path_info;
    uint32_t* seg_flags;
    uchar4* meta;    // {photon_count, escaped, status, filled_this_frame}
    uint8_t* rstart; // retrace_start (0xFF = none)
};

// camera_ray (gather.cpp:22-33) constants, computed on the host libm
struct CamDev {
    V3 pos, fwd, right, up;
    float tan_half, aspect;
    uint32_t w, h;
};

struct Counters {
    unsigned long long traced, segments, replaced, pruned, filled, vis, flagged, retrace,
        live_segments, fill_overflow, scratch0, scratch1;
};

}  // namespace prx
