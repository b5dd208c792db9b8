// engine.cpp -- host orchestration of the B200 path-reuse engine (see engine.h).
//
// Compiled by the host compiler without -march/fast-math: the keyframe, light-pose and
// box arithmetic done here matches the reference's host arithmetic bit for bit.
#include "engine.h"

#include "comm.h"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <numbers>
#include <thread>

#include "fast_bvh.h"
#include "prims.h"

#ifndef PRX_TRACE_LONGEST_FIRST
#define PRX_TRACE_LONGEST_FIRST 1  // trace queue ordered by retrace start (most bounces left first)
#endif
#ifndef PRX_WALK_ORDER
#define PRX_WALK_ORDER 1  // verify-walk queue: 0 append order, 1 most flagged segments first, 2 earliest flag first, 3 = 1 then 2
#endif

namespace prx {

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw CudaError(std::string("CUDA error ") + cudaGetErrorName(e) + " (" +
                        cudaGetErrorString(e) + ") at " + what);
}

void DevBuf::alloc(size_t bytes) {
    reset();
    if (bytes == 0) return;
    PRX_CUDA(cudaMalloc(&p_, bytes));
    n_ = bytes;
}

void DevBuf::reset() {
    if (p_) cudaFree(p_);
    p_ = nullptr;
    n_ = 0;
}

namespace {

enum { kCntTrim = 0, kCntPruned = 1, kCntRetrace = 2, kCntWalk = 3, kCntDead0 = 8, kCntNeed0 = 24, kCntN = 40 };
enum {
    kEvFrame0 = 0,
    kEvVerify0 = 1,
    kEvOccl0 = 2,
    kEvDm0 = 3,
    kEvPrune0 = 4,
    kEvFill0 = 5,
    kEvTrace0 = 6,
    kEvEnd = 7,
    kEvSplat0 = 8,
    kEvSplat1 = 9
};

float4 f4(V3 v, float w) { return float4{v.x, v.y, v.z, w}; }
float f_of_u(uint32_t u) {
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}

}  // namespace

// ----------------------------------------------------------------------- exact pow tables
// phong_lobe_sample (engine.cpp:34-42) raises the 24-bit uniform u1 = k * 2^-24 to
// 1 / (exponent + 1) with the host libm's powf (std::pow(float, float)).  One table of all
// 2^24 results per distinct glossy exponent (64 MB each) makes glossy bounces bit-identical
// to the reference on the same host libm, like the trig table does for cosine_sample.
const float* exact_pow_table(int device, float exponent) {
    static std::mutex mu;
    static std::map<std::pair<int, uint32_t>, float*> dev;
    uint32_t bits;
    std::memcpy(&bits, &exponent, 4);
    std::lock_guard<std::mutex> lock(mu);
    auto it = dev.find({device, bits});
    if (it != dev.end()) return it->second;
    constexpr uint32_t kN = 1u << 24;
    std::vector<float> host(kN);
    const float inv = 1.0f / (exponent + 1.0f);
    const unsigned nt = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    std::vector<std::thread> th;
    for (unsigned t = 0; t < nt; ++t) {
        th.emplace_back([t, nt, inv, &host] {
            const uint32_t lo = static_cast<uint32_t>((uint64_t)kN * t / nt);
            const uint32_t hi = static_cast<uint32_t>((uint64_t)kN * (t + 1) / nt);
            for (uint32_t k = lo; k < hi; ++k) {
                const float u1 = static_cast<float>(k) * 0x1.0p-24f;
                host[k] = std::pow(u1, inv);
            }
        });
    }
    for (auto& x : th) x.join();
    int prev = 0;
    PRX_CUDA(cudaGetDevice(&prev));
    PRX_CUDA(cudaSetDevice(device));
    float* d = nullptr;
    PRX_CUDA(cudaMalloc(&d, sizeof(float) * kN));
    PRX_CUDA(cudaMemcpy(d, host.data(), sizeof(float) * kN, cudaMemcpyHostToDevice));
    PRX_CUDA(cudaSetDevice(prev));
    dev[{device, bits}] = d;
    return d;
}

// ----------------------------------------------------------------------- exact trig table
// cosine_sample draws phi = fl(2*pi_f) * (k * 2^-24) and evaluates cos/sin with the host
// libm (sincosf after GCC's sin/cos CSE).  The device looks the pair up by k, so bounce
// directions are bit-identical to the reference on the same host libm.
const float2* exact_trig_table(int device) {
    static std::mutex mu;
    static std::vector<float2> host;
    static std::map<int, float2*> dev;
    std::lock_guard<std::mutex> lock(mu);
    auto it = dev.find(device);
    if (it != dev.end()) return it->second;
    constexpr uint32_t kN = 1u << 24;
    if (host.empty()) {
        host.resize(kN);
        const unsigned nt = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
        std::vector<std::thread> th;
        for (unsigned t = 0; t < nt; ++t) {
            th.emplace_back([t, nt] {
                const uint32_t lo = static_cast<uint32_t>((uint64_t)kN * t / nt);
                const uint32_t hi = static_cast<uint32_t>((uint64_t)kN * (t + 1) / nt);
                for (uint32_t k = lo; k < hi; ++k) {
                    const float u2 = static_cast<float>(k) * 0x1.0p-24f;
                    const float phi = 2.0f * std::numbers::pi_v<float> * u2;
                    float s, c;
                    ::sincosf(phi, &s, &c);
                    host[k] = float2{c, s};
                }
            });
        }
        for (auto& x : th) x.join();
    }
    int prev = 0;
    PRX_CUDA(cudaGetDevice(&prev));
    PRX_CUDA(cudaSetDevice(device));
    float2* d = nullptr;
    PRX_CUDA(cudaMalloc(&d, sizeof(float2) * kN));
    PRX_CUDA(cudaMemcpy(d, host.data(), sizeof(float2) * kN, cudaMemcpyHostToDevice));
    PRX_CUDA(cudaSetDevice(prev));
    dev[device] = d;
    return d;
}

// ----------------------------------------------------------------------- construction
Engine::Engine(std::shared_ptr<const Scene> scene, const prx_config& cfg)
    : scene_(std::move(scene)), cfg_(cfg) {
    // engine.cpp:64-72
    if (cfg_.n_paths == 0) throw std::invalid_argument("engine: n_paths must be positive");
    if (cfg_.max_bounces < 1 || cfg_.max_bounces > 16)
        throw std::invalid_argument("engine: max_bounces must be in 1..16");
    if (scene_->lights.empty()) throw std::invalid_argument("engine: scene has no lights");
    if (cfg_.mode < PRX_MODE_BASELINE || cfg_.mode > PRX_MODE_ERROR)
        throw std::invalid_argument("engine: unknown mode");
    n_total_ = cfg_.n_paths;
    sb_ = cfg_.shard_begin;
    se_ = cfg_.shard_end;
    if (sb_ == 0 && se_ == 0) se_ = n_total_;
    if (sb_ >= se_ || se_ > n_total_) throw std::invalid_argument("engine: bad shard range");
    n_ = se_ - sb_;
    B_ = cfg_.max_bounces;
    device_ = cfg_.device;
    eps_ = 1e-4f * scene_->diagonal();
    diag_ = scene_->diagonal();
    seed_mix_ = mix64(cfg_.seed);
    if (const char* e = std::getenv("PRX_XT_FORCE")) xt_force_ = e[0] == '1' ? 1 : 0;

    PRX_CUDA(cudaSetDevice(device_));
    PRX_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
    for (auto& e : ev_) PRX_CUDA(cudaEventCreate(&e));
    PRX_CUDA(cudaStreamCreateWithFlags(&side_stream_, cudaStreamNonBlocking));
    PRX_CUDA(cudaEventCreateWithFlags(&ev_fork_, cudaEventDisableTiming));
    PRX_CUDA(cudaEventCreateWithFlags(&ev_join_, cudaEventDisableTiming));
    PRX_CUDA(cudaEventCreateWithFlags(&ev_splat_, cudaEventDisableTiming));
    PRX_CUDA(cudaEventCreateWithFlags(&ev_splat_read_, cudaEventDisableTiming));
    if (const char* e = std::getenv("PRX_SPLAT_PREFIX")) pre_on_ = e[0] != '0';
    PRX_CUDA(cudaHostAlloc(&h_ncell_, 8, cudaHostAllocDefault));
    h_ncell_[0] = h_ncell_[1] = 0;
    launch_base_ = g_launches;

    // light blocks (engine.cpp:76-101)
    const uint32_t nl = static_cast<uint32_t>(scene_->lights.size());
    const uint32_t base = n_total_ / nl, extra = n_total_ % nl;
    uint32_t next = 0;
    lights_.resize(nl);
    for (uint32_t li = 0; li < nl; ++li) {
        LightBlock& b = lights_[li];
        b.light = &scene_->lights[li];
        const uint32_t count = base + (li < extra ? 1u : 0u);
        if (count == 0) throw std::invalid_argument("engine: fewer paths than lights");
        b.begin = next;
        b.end = next + count;
        next = b.end;
        if (b.light->param_dims() == 4) {
            b.ndims = 4;
            for (int a = 0; a < 4; ++a) b.dims[a] = cfg_.dm_dims[a];
        } else {
            b.ndims = 2;
            b.dims[0] = cfg_.dm_dims[2];
            b.dims[1] = cfg_.dm_dims[3];
        }
        uint64_t cells = 1;
        for (uint32_t a = 0; a < b.ndims; ++a) {
            if (b.dims[a] == 0) throw std::invalid_argument("init_dm_target: zero-sized DM axis");
            cells *= b.dims[a];
        }
        if (cells > (1u << 22)) throw std::invalid_argument("init_dm_target: more than 2^22 DM cells");
        b.cells = static_cast<uint32_t>(cells);
        max_cells_ = std::max(max_cells_, b.cells);
        // flux_per_path = flux / sum(DM_T); every draw lands in a cell so the sum is `count`
        const float binned = static_cast<float>(static_cast<double>(count));
        b.flux_pp = divs(b.light->flux, binned);
        b.cos_half = std::cos(static_cast<double>(b.light->cone_angle_deg) * std::numbers::pi / 360.0);
        b.pose_now = light_pose_at(*b.light, 0);
        b.pose_prev = b.pose_now;
        b.dm_t.alloc(4ull * b.cells);
        b.dm_c.alloc(4ull * b.cells);
        b.unm.alloc(4ull * b.cells);
        b.seg_start.alloc(4ull * b.cells);
        PRX_CUDA(cudaMemsetAsync(b.dm_t.get(), 0, 4ull * b.cells, stream_));
        PRX_CUDA(cudaMemsetAsync(b.dm_c.get(), 0, 4ull * b.cells, stream_));
    }

    PRX_CUDA(cudaMallocHost(&h_fp_, sizeof(FrameParams)));
    std::memset(h_fp_, 0, sizeof(FrameParams));
    d_fp_.alloc(sizeof(FrameParams));
    PRX_CUDA(cudaMallocHost(&h_ctr_, sizeof(Counters)));
    PRX_CUDA(cudaMallocHost(&h_cnt32_, 4 * kCntN));
    PRX_CUDA(cudaMallocHost(&h_prune_frame_, 4));
    *h_prune_frame_ = 0;
    d_prune_frame_.alloc(4);
    if (const char* e = std::getenv("PRX_GRAPHS")) graphs_on_ = std::atoi(e) != 0;
    d_ctr_.alloc(sizeof(Counters));
    d_cnt32_.alloc(4 * kCntN);
    d_work_.alloc(64);
    PRX_CUDA(cudaMemsetAsync(d_ctr_.get(), 0, sizeof(Counters), stream_));
    PRX_CUDA(cudaMemsetAsync(d_cnt32_.get(), 0, 4 * kCntN, stream_));

    if (const char* e = std::getenv("PRX_CERT_OFF")) cert_off_ = std::atoi(e) != 0 ? 1 : 0;
    upload_scene();
    apply_l2_policy();
    alloc_state();
    place_frame(0);
    if (cfg_.exact_trig >= 0) d_trig_ = exact_trig_table(device_);

    // DM_T (init_dm_target, light.cpp:230-252), keyed by the sample index within the block
    fill_frame_params();
    for (uint32_t li = 0; li < nl; ++li)
        launch_init_dm_target(&h_fp_->lights[li], lights_[li].end - lights_[li].begin, seed_mix_,
                              lights_[li].dm_t.as<uint32_t>(), stream_);
    PRX_CUDA(cudaStreamSynchronize(stream_));
}

// Forget the captured frame graphs (they are re-captured on the next repeated frame signature).
void Engine::drop_graphs() {
    if (stream_) PRX_CUDA(cudaStreamSynchronize(stream_));
    for (auto& kv : graphs_)
        if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
    graphs_.clear();
    last_sig_ = ~0u;
}

Engine::~Engine() {
    if (stream_) cudaStreamSynchronize(stream_);
    for (auto& e : ev_)
        if (e) cudaEventDestroy(e);
    if (h_fp_) cudaFreeHost(h_fp_);
    if (h_ctr_) cudaFreeHost(h_ctr_);
    if (h_cnt32_) cudaFreeHost(h_cnt32_);
    if (h_xf_) cudaFreeHost(h_xf_);
    if (h_prune_frame_) cudaFreeHost(h_prune_frame_);
    if (h_ncell_) cudaFreeHost(h_ncell_);
    if (h_img_stage_) cudaFreeHost(h_img_stage_);
    for (auto& kv : graphs_)
        if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
    if (capture_stream_) cudaStreamDestroy(capture_stream_);
    if (side_stream_) {
        cudaStreamSynchronize(side_stream_);
        cudaStreamDestroy(side_stream_);
    }
    if (ev_fork_) cudaEventDestroy(ev_fork_);
    if (ev_join_) cudaEventDestroy(ev_join_);
    if (ev_splat_) cudaEventDestroy(ev_splat_);
    if (ev_splat_read_) cudaEventDestroy(ev_splat_read_);
    if (stream_ && own_stream_) cudaStreamDestroy(stream_);
}

// Keep the traversal's static working set (C4: ~85 MB of nodes and triangles, read at random
// by every ray) resident in L2 against the path store's streaming traffic: one persisting
// access-policy window on the engine stream over the hot arena's prefix, sized to the
// device's persisting-L2 limit. Opt-in (PRX_L2_PERSIST=1, or =N for an N MB cap): measured on
// C4 it does not pay -- 8-16 MB windows are neutral, 32-85 MB slow every stage by 1-18% by
// shrinking the normal L2 (profiles/r01_sweeps.md); traversal is issue-bound, not DRAM-bound.
void Engine::apply_l2_policy() {
    const char* env = std::getenv("PRX_L2_PERSIST");
    if (!d_hot_.get() || !env || std::atoi(env) <= 0) return;
    int max_persist = 0, max_window = 0;
    PRX_CUDA(cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, device_));
    PRX_CUDA(cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, device_));
    if (max_persist <= 0 || max_window <= 0) return;
    size_t limit = static_cast<size_t>(max_persist);
    if (env && std::atoi(env) > 1) limit = std::min(limit, static_cast<size_t>(std::atoi(env)) << 20);
    const size_t window = std::min({d_hot_.size(), static_cast<size_t>(max_window), limit});
    PRX_CUDA(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, limit));
    cudaStreamAttrValue attr{};
    attr.accessPolicyWindow.base_ptr = d_hot_.get();
    attr.accessPolicyWindow.num_bytes = window;
    attr.accessPolicyWindow.hitRatio = 1.0f;
    attr.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    attr.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    PRX_CUDA(cudaStreamSetAttribute(stream_, cudaStreamAttributeAccessPolicyWindow, &attr));
    l2_window_ = window;
}

void Engine::upload_scene() {
    const Scene& s = *scene_;
    // static BVH nodes: {lo, a} {hi, b}; leaf: a = first | leaf bit, b = count
    const size_t nn = s.bvh_nodes.size();
    if (nn) {
        std::vector<float4> nodes(2 * nn);
        for (size_t i = 0; i < nn; ++i) {
            const BvhNode& n = s.bvh_nodes[i];
            const uint32_t a = n.count ? (n.first | kLeafBit) : n.left;
            const uint32_t b = n.count ? n.count : n.first;
            nodes[2 * i] = f4(n.bounds.lo, f_of_u(a));
            nodes[2 * i + 1] = f4(n.bounds.hi, f_of_u(b));
        }
        std::vector<float4> tris(3 * s.bvh_perm.size());
        for (size_t k = 0; k < s.bvh_perm.size(); ++k) {
            const uint32_t orig = s.bvh_perm[k];
            const Tri& t = s.static_tris[orig];
            tris[3 * k] = f4(t.a, f_of_u(orig));
            tris[3 * k + 1] = f4(sub(t.b, t.a), f_of_u(s.static_tri_obj[orig]));
            tris[3 * k + 2] = f4(sub(t.c, t.a), 0.0f);
        }
        d_stris_.alloc(sizeof(float4) * tris.size());
        PRX_CUDA(cudaMemcpy(d_stris_.get(), tris.data(), d_stris_.size(), cudaMemcpyHostToDevice));
        // leaf_of[k]: reference leaf holding permutation position k (the fast traversal's
        // certificate tests that leaf's box; ancestors contain it, see device_scene.cuh)
        std::vector<uint32_t> leaf_of(s.bvh_perm.size(), 0);
        for (size_t k = 0; k < nn; ++k) {
            const BvhNode& n = s.bvh_nodes[k];
            for (uint32_t i = 0; i < n.count; ++i) leaf_of[n.first + i] = static_cast<uint32_t>(k);
        }
        // the fast traversal's own SAH tree over the triangles in reference order
        std::vector<Tri> ref_order(s.bvh_perm.size());
        for (size_t k = 0; k < ref_order.size(); ++k) ref_order[k] = s.static_tris[s.bvh_perm[k]];
        const FastBvh fb = build_fast_bvh(ref_order, 1e-5f * diag_ + 1e-6f);
        if (fb.depth + 1 > kMaxTraversalDepth)  // only with a PRX_SAH_MAXDEPTH override
            throw std::length_error("static fast BVH deeper than the traversal stack");
        std::vector<float4> fn(4 * fb.nodes.size());
        for (size_t k = 0; k < fb.nodes.size(); ++k) {
            const FastNode& nd = fb.nodes[k];
            fn[4 * k] = f4(nd.box[0].lo, f_of_u(nd.child[0]));
            fn[4 * k + 1] = f4(nd.box[0].hi, f_of_u(nd.child[1]));
            fn[4 * k + 2] = f4(nd.box[1].lo, 0.0f);
            fn[4 * k + 3] = f4(nd.box[1].hi, 0.0f);
        }
        std::vector<float4> ft(kFT * fb.order.size(), float4{0.f, 0.f, 0.f, 0.f});
        for (size_t k = 0; k < fb.order.size(); ++k) {
            const uint32_t pos = fb.order[k];
            ft[kFT * k] = float4{tris[3 * pos].x, tris[3 * pos].y, tris[3 * pos].z, f_of_u(pos)};
            ft[kFT * k + 1] = tris[3 * pos + 1];
            ft[kFT * k + 2] = tris[3 * pos + 2];
            ft[kFT * k + 2].w = f_of_u(leaf_of[pos]);  // the certificate's reference leaf (static_cert_slot)
        }
        // hot arena, hottest first: a window over its prefix keeps what fits persisting in L2.
        // The combined dynamic tree's nodes follow the static tree's in the same array (room
        // for its largest form: <= 2 n + kMaxDyn nodes), so the joint walk reads both trees
        // from one base: dynamic internal child codes are offset by the static node count.
        size_t n_dyn_tris = 0;
        for (const Object& o : s.objects)
            if (o.dynamic) n_dyn_tris += o.mesh.size();
        const size_t dyn_node_cap = n_dyn_tris >= 2 ? 2 * n_dyn_tris + kMaxDyn : 0;
        const auto up = [](size_t b) { return (b + 255) & ~size_t(255); };
        const size_t b_fn = sizeof(float4) * (fn.size() + 4 * dyn_node_cap), b_ft = sizeof(float4) * ft.size();
        const size_t b_lo = 4 * leaf_of.size(), b_nd = sizeof(float4) * nodes.size();
        d_hot_.alloc(up(b_fn) + up(b_ft) + up(b_lo) + up(b_nd));
        char* base = static_cast<char*>(d_hot_.get());
        p_fnodes_ = reinterpret_cast<float4*>(base);
        dnode_off_ = static_cast<uint32_t>(fb.nodes.size());
        p_dnodes_ = dyn_node_cap ? p_fnodes_ + fn.size() : nullptr;
        dnode_cap_ = dyn_node_cap;
        p_ftris_ = reinterpret_cast<float4*>(base + up(b_fn));
        p_leaf_of_ = reinterpret_cast<uint32_t*>(base + up(b_fn) + up(b_ft));
        p_nodes_ = reinterpret_cast<float4*>(base + up(b_fn) + up(b_ft) + up(b_lo));
        PRX_CUDA(cudaMemcpy(p_fnodes_, fn.data(), sizeof(float4) * fn.size(), cudaMemcpyHostToDevice));
        PRX_CUDA(cudaMemcpy(p_ftris_, ft.data(), b_ft, cudaMemcpyHostToDevice));
        PRX_CUDA(cudaMemcpy(p_leaf_of_, leaf_of.data(), b_lo, cudaMemcpyHostToDevice));
        PRX_CUDA(cudaMemcpy(p_nodes_, nodes.data(), b_nd, cudaMemcpyHostToDevice));
    }
    // materials / flags
    std::vector<float4> mat(s.objects.size());
    std::vector<uint32_t> flags(s.objects.size());
    std::vector<const float*> pow_tabs;  // one exact pow table per distinct glossy exponent
    std::vector<float> pow_exps;
    for (size_t i = 0; i < s.objects.size(); ++i) {
        const Object& o = s.objects[i];
        mat[i] = f4(o.material.albedo, o.material.glossy_exponent);
        flags[i] = (o.dynamic ? 1u : 0u) | (o.material.kind == PRX_MATERIAL_GLOSSY ? 2u : 0u);
        if (o.material.kind == PRX_MATERIAL_GLOSSY && cfg_.exact_trig >= 0) {
            const float e = o.material.glossy_exponent;
            size_t slot = 0;
            while (slot < pow_exps.size() && std::memcmp(&pow_exps[slot], &e, 4) != 0) ++slot;
            if (slot == pow_exps.size()) {
                pow_exps.push_back(e);
                pow_tabs.push_back(exact_pow_table(device_, e));
            }
            flags[i] |= 4u | (static_cast<uint32_t>(slot) << 8);  // bit2: exact pow table at slot
        }
    }
    if (!pow_tabs.empty()) {
        d_pow_tabs_.alloc(sizeof(const float*) * pow_tabs.size());
        PRX_CUDA(cudaMemcpy(d_pow_tabs_.get(), pow_tabs.data(), d_pow_tabs_.size(), cudaMemcpyHostToDevice));
    }
    d_mat_.alloc(sizeof(float4) * mat.size());
    d_oflags_.alloc(4 * flags.size());
    PRX_CUDA(cudaMemcpy(d_mat_.get(), mat.data(), d_mat_.size(), cudaMemcpyHostToDevice));
    PRX_CUDA(cudaMemcpy(d_oflags_.get(), flags.data(), d_oflags_.size(), cudaMemcpyHostToDevice));
    // dynamic meshes (object-local), per-triangle transform slot
    std::vector<float4> local;
    std::vector<uint32_t> tri_xf;
    uint32_t tri = 0, nodes_total = 0;
    // the combined dynamic tree: per-object SAH topologies refit per frame (default), or a
    // per-frame Karras rebuild (PRX_DYN_TREE=karras, A/B runs).  With the SAH topology the
    // fast mode answers per-object queries from the object's subtree, so the per-object
    // Karras trees are only built for the DFS traversal mode or the Karras variant.
    const char* tree_kind = std::getenv("PRX_DYN_TREE");
    const bool karras_all = tree_kind && std::strcmp(tree_kind, "karras") == 0;
    const bool per_object = cfg_.dfs_traversal || karras_all;
    for (const Object& o : s.objects) {
        if (!o.dynamic) continue;
        if (dyn_.size() >= static_cast<size_t>(kMaxDyn))
            throw std::invalid_argument("engine: more than 128 dynamic objects");
        DynInfo d;
        d.obj = o.id;
        d.tri_begin = tri;
        d.tri_count = static_cast<uint32_t>(o.mesh.size());
        if (per_object && d.tri_count > 32) {  // LBVH for anything beyond a few boxes
            d.node_begin = nodes_total;
            nodes_total += d.tri_count - 1;
        }
        for (const Tri& t : o.mesh) {
            local.push_back(f4(t.a, 0));
            local.push_back(f4(t.b, 0));
            local.push_back(f4(t.c, 0));
            tri_xf.push_back(static_cast<uint32_t>(dyn_.size()));
        }
        tri += d.tri_count;
        dyn_.push_back(d);
    }
    n_dyn_tris_ = tri;
    n_lbvh_nodes_ = nodes_total;
    if (tri) {
        d_dyn_local_.alloc(sizeof(float4) * local.size());
        d_dyn_world_.alloc(sizeof(float4) * local.size());
        d_dyn_tri_xf_.alloc(4 * tri_xf.size());
        d_dyn_xf_.alloc(sizeof(float4) * 2 * dyn_.size());
        PRX_CUDA(cudaMallocHost(&h_xf_, sizeof(float4) * 2 * kMaxDyn));
        PRX_CUDA(cudaMemcpy(d_dyn_local_.get(), local.data(), d_dyn_local_.size(), cudaMemcpyHostToDevice));
        PRX_CUDA(cudaMemcpy(d_dyn_tri_xf_.get(), tri_xf.data(), d_dyn_tri_xf_.size(), cudaMemcpyHostToDevice));
        d_lbvh_leaf_.alloc(4ull * tri);
        if (nodes_total) d_lbvh_nodes_.alloc(sizeof(float4) * 4ull * nodes_total);
        if (tri >= 2) {
            const size_t n = tri;
            const size_t scratch = prim_scratch_bytes(n);
            d_lbvh_work_.alloc(4 * n * 4 + 4 * (2 * n + 2) * 2 + scratch);
            uint32_t* w = d_lbvh_work_.as<uint32_t>();
            lbvh_.keys = w;
            lbvh_.vals = w + n;
            lbvh_.keys_tmp = w + 2 * n;
            lbvh_.vals_tmp = w + 3 * n;
            lbvh_.parent = w + 4 * n;
            lbvh_.flags = w + 4 * n + (2 * n + 2);
            lbvh_.scratch = w + 4 * n + 2 * (2 * n + 2);
            d_dall_tris_.alloc(sizeof(float4) * kFT * n);
            PRX_CUDA(cudaMemset(d_dall_tris_.get(), 0, d_dall_tris_.size()));  // (pads stay zero)
            lbvh_.all_tris = d_dall_tris_.as<float4>();
            // the combined tree's nodes: in the hot arena after the static tree's (codes offset
            // by dnode_off_), or alone when the scene has no static tree (offset 0)
            float4* dnodes = nullptr;
            auto place_dnodes = [&](size_t n_nodes) {
                if (p_dnodes_) {  // (the joint walk addresses both trees from the arena base)
                    if (n_nodes > dnode_cap_) throw std::logic_error("dynamic tree larger than its arena room");
                    dnodes = p_dnodes_;
                } else {
                    d_dall_nodes_.alloc(sizeof(float4) * 4 * n_nodes);
                    dnodes = d_dall_nodes_.as<float4>();
                    dnode_off_ = 0;
                }
            };
            if (karras_all) {
                place_dnodes(n - 1);
                lbvh_.code_off = p_dnodes_ ? dnode_off_ : 0;
            } else {  // per-object SAH topologies, built once, refit per frame
                std::vector<std::vector<Tri>> objs;
                std::vector<uint32_t> begins;
                std::vector<Box> boxes;
                for (const DynInfo& d : dyn_) {
                    const Object& o = s.objects[d.obj];
                    objs.push_back(o.mesh);
                    begins.push_back(d.tri_begin);
                    boxes.push_back(transform_box(o.local_bounds, transform_at(o.kfs, 0)));
                }
                DynSahTopology topo = build_dyn_sah(objs, begins, boxes);
                place_dnodes(topo.nodes.size() / 4);
                const uint32_t off = p_dnodes_ ? dnode_off_ : 0;
                for (size_t k = 0; k < topo.nodes.size(); ++k) {  // internal child codes -> arena indices
                    if ((k & 3) > 1) continue;  // codes live in the .w of a node's first two float4
                    uint32_t code;
                    std::memcpy(&code, &topo.nodes[k].w, 4);
                    if (code != 0xFFFFFFFFu && !(code & kLeafBit)) code += off;
                    std::memcpy(&topo.nodes[k].w, &code, 4);
                }
                PRX_CUDA(cudaMemcpy(dnodes, topo.nodes.data(), sizeof(float4) * topo.nodes.size(),
                                    cudaMemcpyHostToDevice));
                const size_t b_perm = 4 * topo.perm.size(), b_leaf = 4 * topo.leaves.size();
                d_dsah_.alloc(b_perm + b_leaf + 4 * topo.parent.size());
                char* base = d_dsah_.as<char>();
                PRX_CUDA(cudaMemcpy(base, topo.perm.data(), b_perm, cudaMemcpyHostToDevice));
                PRX_CUDA(cudaMemcpy(base + b_perm, topo.leaves.data(), b_leaf, cudaMemcpyHostToDevice));
                PRX_CUDA(cudaMemcpy(base + b_perm + b_leaf, topo.parent.data(), 4 * topo.parent.size(),
                                    cudaMemcpyHostToDevice));
                lbvh_.sah_perm = reinterpret_cast<const uint32_t*>(base);
                lbvh_.sah_leaf = reinterpret_cast<const uint4*>(base + b_perm);
                lbvh_.sah_parent = reinterpret_cast<const uint32_t*>(base + b_perm + b_leaf);
                lbvh_.n_sah_leaves = static_cast<uint32_t>(topo.leaves.size() / 4);
                lbvh_.n_sah_nodes = static_cast<uint32_t>(topo.parent.size());
                if (!cfg_.dfs_traversal)
                    for (size_t j = 0; j < dyn_.size(); ++j)
                        dyn_[j].sah_root = topo.obj_root[j] == kLbvhBrute ? kLbvhBrute : topo.obj_root[j] + off;
            }
            lbvh_.all_nodes = dnodes;
        }
    }
}

void Engine::alloc_state() {
    const size_t nv = static_cast<size_t>(n_) * B_;
    // vertex streams, interleaved per vertex so that every vertex write of the trace is a
    // whole 32-byte sector (no read-modify-write): [B][n] x {pos_obj, energy} and
    // [B][n] x {in_dir, out_dir}
    d_pos_obj_.alloc(32 * nv);
    d_in_dir_.alloc(32 * nv);
    d_origin_.alloc(16ull * n_);
    d_emis_.alloc(16ull * n_);
    d_canon_.alloc(16ull * n_);
    d_cell_.alloc(4ull * n_);
    d_epoch_.alloc(4ull * n_);
    d_path_info_.alloc(4ull * n_);
    d_seg_flags_.alloc(4ull * n_);
    d_meta_.alloc(4ull * n_);
    d_rstart_.alloc(n_);
    // reference initial state (engine.cpp:104-116): empty photons, emission dir (0,0,1),
    // everything else zero, status dead, retrace 0xFF
    PRX_CUDA(cudaMemsetAsync(d_pos_obj_.get(), 0, d_pos_obj_.size(), stream_));
    PRX_CUDA(cudaMemsetAsync(d_in_dir_.get(), 0, d_in_dir_.size(), stream_));
    PRX_CUDA(cudaMemsetAsync(d_origin_.get(), 0, d_origin_.size(), stream_));
    PRX_CUDA(cudaMemsetAsync(d_canon_.get(), 0, d_canon_.size(), stream_));
    PRX_CUDA(cudaMemsetAsync(d_cell_.get(), 0, d_cell_.size(), stream_));
    PRX_CUDA(cudaMemsetAsync(d_epoch_.get(), 0, d_epoch_.size(), stream_));
    PRX_CUDA(cudaMemsetAsync(d_path_info_.get(), 0, d_path_info_.size(), stream_));
    PRX_CUDA(cudaMemsetAsync(d_seg_flags_.get(), 0, d_seg_flags_.size(), stream_));
    PRX_CUDA(cudaMemsetAsync(d_meta_.get(), 0, d_meta_.size(), stream_));
    PRX_CUDA(cudaMemsetAsync(d_rstart_.get(), 0xFF, d_rstart_.size(), stream_));
    {
        std::vector<float4> emis(n_, float4{0, 0, 1, 0});
        PRX_CUDA(cudaMemcpy(d_emis_.get(), emis.data(), d_emis_.size(), cudaMemcpyHostToDevice));
        // empty photon records: object id 0xFFFFFFFF (photon_store.hpp:15)
        std::vector<float4> po(std::min<size_t>(nv, 1 << 20), float4{0, 0, 0, f_of_u(kInvalidObj)});
        for (size_t off = 0; off < nv; off += po.size()) {
            const size_t cnt = std::min(po.size(), nv - off);
            PRX_CUDA(cudaMemcpy2DAsync(path_dev().pos_obj + kVS * off, 16 * kVS, po.data(), 16, 16, cnt,
                                       cudaMemcpyHostToDevice, stream_));
            PRX_CUDA(cudaStreamSynchronize(stream_));
        }
    }
    // work arrays
    d_list_.alloc(4ull * n_);
    d_masks_.alloc(4ull * n_);
    d_flags8_.alloc(n_);
    d_flags8b_.alloc(n_);
    d_keys_.alloc(4ull * n_);
    d_vals_.alloc(4ull * n_);
    d_keys_tmp_.alloc(4ull * n_);
    d_vals_tmp_.alloc(4ull * n_);
    d_pruned_list_.alloc(4ull * n_);
    d_need_.alloc(4ull * max_cells_ + 16);
    d_scratch_.alloc(prim_scratch_bytes(std::max<uint64_t>(n_, max_cells_)));
    // per-light pointer tables: [0] unm, [1] seg_start, [2] prefix, [3] total (prx_prune_apply),
    // [4] prefix, [5] total (in-engine sharded prune, set by set_collectives)
    std::vector<uint32_t*> ptrs(6 * PRX_MAX_LIGHTS, nullptr);
    for (size_t li = 0; li < lights_.size(); ++li) {
        ptrs[li] = lights_[li].unm.as<uint32_t>();
        ptrs[PRX_MAX_LIGHTS + li] = lights_[li].seg_start.as<uint32_t>();
    }
    d_light_ptrs_.alloc(sizeof(uint32_t*) * ptrs.size());
    PRX_CUDA(cudaMemcpy(d_light_ptrs_.get(), ptrs.data(), d_light_ptrs_.size(), cudaMemcpyHostToDevice));
    PRX_CUDA(cudaStreamSynchronize(stream_));
}

SceneDev Engine::scene_dev() const {
    SceneDev S{};
    S.nodes = p_nodes_;
    S.n_nodes = static_cast<uint32_t>(scene_->bvh_nodes.size());
    S.leaf_of = p_leaf_of_;
    S.cull_pad = 1e-5f * diag_ + 1e-6f;
    S.fast = cfg_.dfs_traversal ? 0 : 1;
    S.cert_off = cert_off_;
    S.fnodes = p_fnodes_ ? p_fnodes_ : lbvh_.all_nodes;  // (no static tree: the dynamic tree's own array)
    S.ftris = p_ftris_;
    S.stris = d_stris_.as<float4>();
    S.dtris = d_dyn_world_.as<float4>();
    S.dnodes = d_lbvh_nodes_.as<float4>();
    S.dleaf = d_lbvh_leaf_.as<uint32_t>();
    S.dfast = lbvh_.all_nodes ? 1 : 0;
    S.danodes = lbvh_.all_nodes;
    S.dnode_off = p_dnodes_ ? dnode_off_ : 0;
    S.datris = d_dall_tris_.as<float4>();
    S.dtri_obj = d_dyn_tri_xf_.as<uint32_t>();
    S.mat = d_mat_.as<float4>();
    S.oflags = d_oflags_.as<uint32_t>();
    S.fp = d_fp_.as<FrameParams>();
    S.eps = eps_;
    S.two_diag = 2.0f * diag_;
    S.seed_mix = seed_mix_;
    S.gather_radius = cfg_.gather_radius;
    S.trig = d_trig_;
    S.pow_tabs = d_pow_tabs_.as<const float*>();
    return S;
}

PathDev Engine::path_dev() const {
    PathDev P{};
    P.n = n_;
    P.base = sb_;
    P.B = B_;
    // vertex v of a stream at [kVS * v] (dev_types.h): four SoA streams or two interleaved
    const size_t second = PRX_VERTEX_SOA ? static_cast<size_t>(n_) * B_ : 1;
    P.pos_obj = d_pos_obj_.as<float4>();
    P.energy = d_pos_obj_.as<float4>() + second;
    P.in_dir = d_in_dir_.as<float4>();
    P.out_dir = d_in_dir_.as<float4>() + second;
    P.origin = d_origin_.as<float4>();
    P.emis = d_emis_.as<float4>();
    P.canon = d_canon_.as<float4>();
    P.cell = d_cell_.as<uint32_t>();
    P.epoch = d_epoch_.as<uint32_t>();
    P.path_info = d_path_info_.as<uint32_t>();
    P.seg_flags = d_seg_flags_.as<uint32_t>();
    P.meta = d_meta_.as<uchar4>();
    P.rstart = d_rstart_.as<uint8_t>();
    return P;
}

uint32_t Engine::local_lb(const LightBlock& b) const { return std::max(b.begin, sb_) - sb_; }
uint32_t Engine::local_le(const LightBlock& b) const {
    const uint32_t e = std::min(b.end, se_);
    const uint32_t s = std::max(b.begin, sb_);
    return e > s ? e - sb_ : local_lb(b);
}

void Engine::record(int idx) {
    if (capturing_)  // an event-record node of the frame graph (timed like a stream event)
        PRX_CUDA(cudaEventRecordWithFlags(ev_[idx], stream_, cudaEventRecordExternal));
    else
        PRX_CUDA(cudaEventRecord(ev_[idx], stream_));
    ev_recorded_[idx] = true;
}

double Engine::elapsed_ms(int a, int b) {
    if (!ev_recorded_[a] || !ev_recorded_[b]) return 0.0;
    float ms = 0.0f;
    if (cudaEventElapsedTime(&ms, ev_[a], ev_[b]) != cudaSuccess) return 0.0;
    return ms;
}

// ----------------------------------------------------------------------- frame params
void Engine::fill_frame_params_host() {
    FrameParams& fp = *h_fp_;
    fp.frame = cur_frame_;
    fp.n_lights = static_cast<uint32_t>(lights_.size());
    for (size_t li = 0; li < lights_.size(); ++li) {
        const LightBlock& b = lights_[li];
        LightDev& L = fp.lights[li];
        L.kind = b.light->kind;
        L.begin = b.begin;
        L.end = b.end;
        L.moved = b.moved ? 1 : 0;
        L.position = b.pose_now.position;
        L.normal = b.pose_now.normal;
        L.tangent = b.pose_now.tangent;
        L.bitangent = b.pose_now.bitangent;
        L.scale = b.pose_now.scale;
        L.radius = b.light->radius;
        L.half_x = b.light->half_x;
        L.half_y = b.light->half_y;
        L.cos_half = b.cos_half;
        L.flux_pp = b.flux_pp;
        L.ndims = b.ndims;
        L.cells = b.cells;
        for (int a = 0; a < 4; ++a) L.dims[a] = b.dims[a];
        L.dm_t = b.dm_t.as<uint32_t>();
        L.dm_c = b.dm_c.as<uint32_t>();
        L.xt_force = xt_force_;
    }
    fp.n_dyn = static_cast<uint32_t>(dyn_.size());
}

void Engine::fill_frame_params() {
    fill_frame_params_host();
    copy_async(d_fp_.get(), h_fp_, sizeof(FrameParams), cudaMemcpyHostToDevice);
}

// state_at (scene.cpp:115-134) on the host: every dynamic object's descriptor and current
// bounds, and the occlusion boxes united(prev, cur).inflate(eps) (engine.cpp:211-218).
void Engine::place_frame(int frame) {
    FrameParams& fp = *h_fp_;
    fp.n_boxes = 0;
    for (size_t j = 0; j < dyn_.size(); ++j) {
        const Object& o = scene_->objects[dyn_[j].obj];
        const Xform now = transform_at(o.kfs, frame);
        const Xform prev = transform_at(o.kfs, frame > 0 ? frame - 1 : 0);
        const Box cur = transform_box(o.local_bounds, now);
        const Box prv = transform_box(o.local_bounds, prev);
        DynObj& D = fp.dyn[j];
        D.obj = dyn_[j].obj;
        D.tri_begin = dyn_[j].tri_begin;
        D.tri_count = dyn_[j].tri_count;
        D.node_begin = dyn_[j].node_begin;
        D.sah_root = dyn_[j].sah_root;
        D.cur = cur;
        if (frame > 0) {
            Box box = prv;
            expand(box, cur);
            inflate(box, eps_);
            fp.boxes[fp.n_boxes++] = box;
        }
    }
}

// device placement of the dynamics (+ LBVH) for the transforms of cur_frame_
void Engine::place_dynamics(bool force) {
    if (place_dynamics_host(force)) place_dynamics_enqueue();
}

// transforms of cur_frame_ into pinned host memory; true when the device copy must change
bool Engine::place_dynamics_host(bool force) {
    if (dyn_.empty()) return false;
    bool changed = force;
    for (size_t j = 0; j < dyn_.size(); ++j) {
        const Object& o = scene_->objects[dyn_[j].obj];
        const Xform now = transform_at(o.kfs, cur_frame_);
        if (!dyn_[j].placed || !(now == dyn_[j].last_xf)) changed = true;
        dyn_[j].last_xf = now;
        dyn_[j].placed = true;
        h_xf_[2 * j] = float4{now.rot.x, now.rot.y, now.rot.z, now.rot.w};
        h_xf_[2 * j + 1] = float4{now.trans.x, now.trans.y, now.trans.z, now.scale};
    }
    return changed;
}

void Engine::place_dynamics_enqueue() {
    pre_ok_ = false;  // the splat prefix saw the previous placement
    copy_async(d_dyn_xf_.get(), h_xf_, sizeof(float4) * 2 * dyn_.size(), cudaMemcpyHostToDevice);
    launch_transform_dynamic(d_dyn_local_.as<float4>(), d_dyn_tri_xf_.as<uint32_t>(),
                             d_dyn_xf_.as<float4>(), n_dyn_tris_, d_dyn_world_.as<float4>(), stream_);
    if (n_dyn_tris_ >= 2)
        build_dynamic_lbvh(d_dyn_world_.as<float4>(), d_dyn_tri_xf_.as<uint32_t>(), n_dyn_tris_,
                           h_fp_->dyn, static_cast<uint32_t>(dyn_.size()),
                           reinterpret_cast<const DynObj*>(d_fp_.as<char>() + offsetof(FrameParams, dyn)),
                           n_lbvh_nodes_ ? d_lbvh_nodes_.as<float4>() : nullptr, d_lbvh_leaf_.as<uint32_t>(), lbvh_, stream_);
}

void Engine::copy_async(void* dst, const void* src, size_t bytes, cudaMemcpyKind kind) {
    PRX_CUDA(cudaMemcpyAsync(dst, src, bytes, kind, stream_));
    if (kind == cudaMemcpyHostToDevice) h2d_bytes_ += bytes;
    if (kind == cudaMemcpyDeviceToHost) d2h_bytes_ += bytes;
}

// ----------------------------------------------------------------------- stages
// frame_update = its host part (frame counter, light poses, frame parameters and transforms in
// pinned host memory) + its device part (uploads and kernels), split so that run_frame can
// replay the device parts of a whole frame as one CUDA graph.
void Engine::frame_update(prx_frame_stats* st) {
    PRX_CUDA(cudaSetDevice(device_));
    frame_update_host();
    frame_update_enqueue();
    if (st) {
        st->frame = cur_frame_;
        st->mode = cfg_.mode;
    }
}

void Engine::frame_update_host() {
    PRX_CUDA(cudaSetDevice(device_));
    for (bool& r : ev_recorded_) r = false;
    const int frame = frames_run_++;
    cur_frame_ = frame;
    n_pruned_ = 0;
    // light poses (engine.cpp:205-209)
    for (LightBlock& b : lights_) {
        b.pose_prev = b.pose_now;
        b.pose_now = light_pose_at(*b.light, frame);
        b.moved = frame > 0 && !(b.pose_now == b.pose_prev);
    }
    place_frame(frame);
    fill_frame_params_host();
    dyn_changed_ = place_dynamics_host(false);
    *h_prune_frame_ = static_cast<uint32_t>(cur_frame_);
}

void Engine::frame_update_enqueue() {
    record(kEvFrame0);
    PRX_CUDA(cudaMemsetAsync(d_ctr_.get(), 0, sizeof(Counters), stream_));
    PRX_CUDA(cudaMemsetAsync(d_cnt32_.get(), 0, 4 * kCntN, stream_));
    copy_async(d_fp_.get(), h_fp_, sizeof(FrameParams), cudaMemcpyHostToDevice);
    copy_async(d_prune_frame_.get(), h_prune_frame_, 4, cudaMemcpyHostToDevice);
    if (dyn_changed_) place_dynamics_enqueue();
    launch_frame_reset(path_dev(), cfg_.record_flags, d_ctr_.as<Counters>(), stream_);
    if (cfg_.mode == PRX_MODE_BASELINE) {  // engine.cpp:228-232
        wait_splat(stream_, false);  // (truncates every path: a photon-map write)
        launch_release_all(path_dev(), stream_);
        for (LightBlock& b : lights_) PRX_CUDA(cudaMemsetAsync(b.dm_c.get(), 0, 4ull * b.cells, stream_));
    }
    record(kEvVerify0);
}

void Engine::stage_update_origins() {
    bool any = false;
    for (const LightBlock& b : lights_) any = any || b.moved;
    if (any) launch_update_origins(scene_dev(), path_dev(), d_ctr_.as<Counters>(), stream_);
}

void Engine::stage_occlusions() {
    if (h_fp_->n_boxes == 0) return;  // engine.cpp:308-312
    launch_occlusion_flags(scene_dev(), path_dev(), cfg_.mode, cfg_.record_flags, d_list_.as<uint32_t>(),
                           d_masks_.as<uint32_t>(), d_ctr_.as<Counters>(), stream_);
    if (cfg_.mode == PRX_MODE_ERROR) {
        wait_splat(stream_, false);  // the walk rewrites vertices an overlapped splat may still read
        const uint32_t* list = d_list_.as<uint32_t>();
        const uint32_t* masks = d_masks_.as<uint32_t>();
#if PRX_WALK_ORDER
        // the flagged list (atomic append order) sorted by expected walk length, longest first
        uint32_t* n32 = d_cnt32_.as<uint32_t>() + kCntWalk;
        const uint32_t top = B_ + 1;  // segments per path <= B + 1
        int bits = 1;
        while ((1u << bits) <= top) ++bits;
        if (PRX_WALK_ORDER == 3) bits += 4;
        launch_walk_keys(masks, d_ctr_.as<Counters>(), n32, top, PRX_WALK_ORDER, n_, d_keys_.as<uint32_t>(),
                         d_vals_.as<uint32_t>(), stream_);
        const bool in_tmp = radix_sort_pairs_nocopy(d_keys_.as<uint32_t>(), d_vals_.as<uint32_t>(),
                                                    d_keys_tmp_.as<uint32_t>(), d_vals_tmp_.as<uint32_t>(), n_, n32,
                                                    bits, d_scratch_.get(), stream_);
        uint32_t* l2 = in_tmp ? d_keys_.as<uint32_t>() : d_keys_tmp_.as<uint32_t>();
        uint32_t* m2 = in_tmp ? d_vals_.as<uint32_t>() : d_vals_tmp_.as<uint32_t>();
        launch_walk_permute(list, masks, in_tmp ? d_vals_tmp_.as<uint32_t>() : d_vals_.as<uint32_t>(), n32, n_, l2,
                            m2, stream_);
        list = l2;
        masks = m2;
#endif
        launch_verify_error(scene_dev(), path_dev(), cfg_.threshold, list, masks, d_ctr_.as<Counters>(),
                            d_work_.as<uint32_t>(), d_ctr_.as<Counters>(), stream_);
    }
}

void Engine::stage_compute_dm() {
    for (LightBlock& b : lights_) PRX_CUDA(cudaMemsetAsync(b.dm_c.get(), 0, 4ull * b.cells, stream_));
    launch_compute_dm(scene_dev(), path_dev(), d_ctr_.as<Counters>(), stream_);
}

void Engine::verify_paths(prx_frame_stats* st) {
    (void)st;
    PRX_CUDA(cudaSetDevice(device_));
    record(kEvVerify0);
    if (cfg_.mode != PRX_MODE_BASELINE && cur_frame_ > 0) {
        stage_update_origins();
        record(kEvOccl0);
        stage_occlusions();
    } else {
        record(kEvOccl0);
    }
    wait_splat(stream_, false);  // (compute_dm truncates paths: the first photon-map write otherwise)
    record(kEvDm0);
    stage_compute_dm();
    if (sharded()) exchange_dm();
    record(kEvPrune0);
}

// stage_prune (engine.cpp:473-497), split at the cross-shard exchange point.
// Marks (Eq. 1 Bernoulli, keyed by (path, frame)) and per-cell unmarked counts.
void Engine::prune_mark_all() {
    if (!capturing_) {  // (a frame graph uploads the frame number itself, from frame_update_host)
        *h_prune_frame_ = static_cast<uint32_t>(cur_frame_);
        copy_async(d_prune_frame_.get(), h_prune_frame_, 4, cudaMemcpyHostToDevice);
    }
    for (LightBlock& b : lights_) PRX_CUDA(cudaMemsetAsync(b.unm.get(), 0, 4ull * b.cells, stream_));
    launch_prune_mark(scene_dev(), path_dev(), d_prune_frame_.as<uint32_t>(), d_light_ptrs_.as<uint32_t*>(),
                      d_flags8_.as<uint8_t>(), d_flags8b_.as<uint8_t>(), stream_);
}

// Trim to exactly dm_t survivors per overfull cell, keeping the lowest path ids; `prefix`
// (device table, may be null) holds the unmarked counts of lower shards, `total` those of
// all shards; total_host[li] is the device address of light li's total counts.
void Engine::prune_trim_all(uint32_t* const* prefix_tab, uint32_t* const* total_tab,
                            const uint32_t* const* total_host) {
    const PathDev P = path_dev();
    uint32_t* cnt = d_cnt32_.as<uint32_t>();
    uint8_t* trim = reinterpret_cast<uint8_t*>(d_keys_tmp_.as<uint32_t>());  // n bytes of scratch
    launch_prune_trim_flags(P, d_fp_.as<FrameParams>(), total_tab, d_flags8b_.as<uint8_t>(), trim, stream_);
    compact_u8(trim, n_, nullptr, 0, d_list_.as<uint32_t>(), cnt + kCntTrim, d_scratch_.get(), stream_);
    launch_prune_keys(P, d_fp_.as<FrameParams>(), d_list_.as<uint32_t>(), cnt + kCntTrim, d_keys_.as<uint32_t>(),
                      d_vals_.as<uint32_t>(), n_, stream_);
    int light_bits = 0;
    while ((1u << light_bits) < lights_.size()) ++light_bits;
    const bool in_tmp = radix_sort_pairs_nocopy(d_keys_.as<uint32_t>(), d_vals_.as<uint32_t>(),
                                                d_keys_tmp_.as<uint32_t>(), d_vals_tmp_.as<uint32_t>(), n_,
                                                cnt + kCntTrim, 22 + light_bits, d_scratch_.get(), stream_);
    const uint32_t* sk = in_tmp ? d_keys_tmp_.as<uint32_t>() : d_keys_.as<uint32_t>();
    const uint32_t* sv = in_tmp ? d_vals_tmp_.as<uint32_t>() : d_vals_.as<uint32_t>();
    launch_prune_trim(P, d_fp_.as<FrameParams>(), sk, sv, cnt + kCntTrim,
                      n_, d_light_ptrs_.as<uint32_t*>() + PRX_MAX_LIGHTS, prefix_tab, d_flags8_.as<uint8_t>(),
                      stream_);
    launch_prune_apply(P, d_flags8_.as<uint8_t>(), in_full_frame_ ? 0 : 1, stream_);
    for (size_t li = 0; li < lights_.size(); ++li)
        launch_dm_after_prune(lights_[li].dm_c.as<uint32_t>(), lights_[li].dm_t.as<uint32_t>(), total_host[li],
                              lights_[li].cells, stream_);
    compact_u8(d_flags8_.as<uint8_t>(), n_, nullptr, sb_, d_pruned_list_.as<uint32_t>(), cnt + kCntPruned,
               d_scratch_.get(), stream_);
}

void Engine::stage_prune_local() {
    prune_mark_all();
    std::vector<const uint32_t*> totals(lights_.size());
    for (size_t li = 0; li < lights_.size(); ++li) totals[li] = lights_[li].unm.as<uint32_t>();
    prune_trim_all(nullptr, d_light_ptrs_.as<uint32_t*>(), totals.data());
}

// stage_fill (engine.cpp:499-546), split at the exchange point: the dead slots of this
// shard, ascending, per light (written at d_list_ + local block begin).
void Engine::fill_collect_dead() {
    const PathDev P = path_dev();
    uint32_t* cnt = d_cnt32_.as<uint32_t>();
    for (uint32_t li = 0; li < lights_.size(); ++li) {
        const uint32_t lb = local_lb(lights_[li]), le = local_le(lights_[li]);
        launch_dead_flags(P, lb, le, d_flags8_.as<uint8_t>() + lb, stream_);
        compact_u8(d_flags8_.as<uint8_t>() + lb, le - lb, nullptr, lb, d_list_.as<uint32_t>() + lb,
                   cnt + kCntDead0 + li, d_scratch_.get(), stream_);
    }
}

// Deficit cells ascending <-> dead slots ascending over the whole path range: this shard
// owns global dead-slot ranks [prefix, prefix + local count).  Without prefix/total the
// shard is the whole range.
void Engine::fill_assign_all(const uint64_t* prefix, const uint64_t* total, const uint64_t* prefix_dev,
                             const uint64_t* total_dev) {
    const PathDev P = path_dev();
    uint32_t* cnt = d_cnt32_.as<uint32_t>();
    for (uint32_t li = 0; li < lights_.size(); ++li) {
        LightBlock& b = lights_[li];
        const uint32_t lb = local_lb(b), le = local_le(b);
        uint32_t* need_total = cnt + kCntNeed0 + li;
        launch_fill_need(b.dm_t.as<uint32_t>(), b.dm_c.as<uint32_t>(), d_need_.as<uint32_t>(), b.cells, stream_);
        scan_exclusive_u32(d_need_.as<uint32_t>(), d_need_.as<uint32_t>(), b.cells, nullptr, need_total,
                           d_scratch_.get(), stream_);
        const bool all_ranks = total || total_dev;
        launch_fill_check(all_ranks ? nullptr : cnt + kCntDead0 + li, total ? total[li] : 0, total_dev, li,
                          need_total, d_ctr_.as<Counters>(), stream_);
        launch_fill_assign(scene_dev(), P, li, d_list_.as<uint32_t>() + lb, cnt + kCntDead0 + li,
                           std::max(1u, le - lb), prefix ? prefix[li] : 0, prefix_dev, d_need_.as<uint32_t>(), need_total,
                           b.cells, d_ctr_.as<Counters>(), stream_);
        launch_dm_after_fill(b.dm_c.as<uint32_t>(), b.dm_t.as<uint32_t>(), b.cells, stream_);
    }
}

void Engine::stage_fill_local() {
    fill_collect_dead();
    fill_assign_all(nullptr, nullptr);
}

// ---- in-engine sharded frame: the exchanges enqueued between the kernels
void Engine::coll_ok(int rc, const char* what) const {
    if (rc != 0) throw CudaError(std::string("collective failed: ") + what);
}

// DM_C per light, summed over the ranks (stage_compute_dm counts this shard's live paths)
void Engine::exchange_dm() {
    for (LightBlock& b : lights_)
        coll_ok(coll_.all_reduce_sum_u32(coll_.ctx, b.dm_c.as<uint32_t>(), b.cells, stream_), "DM_C all-reduce");
}

// stage_prune over shards: Bernoulli marks are per path (key (path, frame)); the trim keeps the
// lowest path ids, so a rank offsets its survivors' ranks by the unmarked counts of the lower
// ranks (gathered, prefix on the device) and every rank sets DM_C from the all-rank totals
void Engine::stage_prune_sharded() {
    prune_mark_all();
    const uint32_t W = static_cast<uint32_t>(coll_.world), R = static_cast<uint32_t>(coll_.rank);
    std::vector<const uint32_t*> totals(lights_.size());
    for (size_t li = 0; li < lights_.size(); ++li) {
        LightBlock& b = lights_[li];
        coll_ok(coll_.all_gather_u32(coll_.ctx, b.unm.as<uint32_t>(), d_gath_.as<uint32_t>(), b.cells, stream_),
                "unmarked-count all-gather");
        launch_rank_prefix_u32(d_gath_.as<uint32_t>(), b.cells, W, R, b.pref.as<uint32_t>(), b.tot.as<uint32_t>(),
                               stream_);
        totals[li] = b.tot.as<uint32_t>();
    }
    uint32_t** tab = d_light_ptrs_.as<uint32_t*>() + 4 * PRX_MAX_LIGHTS;
    prune_trim_all(tab, tab + PRX_MAX_LIGHTS, totals.data());
}

// stage_fill over shards: deficit cells ascending <-> dead slots ascending over all ranks;
// this rank owns dead-slot ranks [prefix, prefix + local count) of each light
void Engine::stage_fill_sharded() {
    fill_collect_dead();
    const uint32_t nl = static_cast<uint32_t>(lights_.size());
    coll_ok(coll_.all_gather_u32(coll_.ctx, d_cnt32_.as<uint32_t>() + kCntDead0, d_dead_g_.as<uint32_t>(), nl,
                                 stream_),
            "dead-slot all-gather");
    uint64_t* pt = d_dead_pt_.as<uint64_t>();
    launch_rank_prefix_u64(d_dead_g_.as<uint32_t>(), nl, static_cast<uint32_t>(coll_.world),
                           static_cast<uint32_t>(coll_.rank), pt, pt + PRX_MAX_LIGHTS, stream_);
    fill_assign_all(nullptr, nullptr, pt, pt + PRX_MAX_LIGHTS);
}

// the frame's counters summed over the ranks (read back instead of the local ones)
void Engine::exchange_counters() {
    PRX_CUDA(cudaMemcpyAsync(d_ctr_sum_.get(), d_ctr_.get(), sizeof(Counters), cudaMemcpyDeviceToDevice, stream_));
    coll_ok(coll_.all_reduce_sum_u64(coll_.ctx, d_ctr_sum_.as<uint64_t>(), sizeof(Counters) / 8, stream_),
            "counter all-reduce");
    PRX_CUDA(cudaMemcpyAsync(d_cnt32_sum_.get(), d_cnt32_.get(), 4 * kCntN, cudaMemcpyDeviceToDevice, stream_));
    coll_ok(coll_.all_reduce_sum_u32(coll_.ctx, d_cnt32_sum_.as<uint32_t>(), kCntN, stream_), "count all-reduce");
}

void Engine::set_collectives(const prx_collectives* c) {
    PRX_CUDA(cudaSetDevice(device_));
    PRX_CUDA(cudaStreamSynchronize(stream_));
    if (!c) {
        coll_ = prx_collectives{};
        return;
    }
    if (c->world < 1 || c->rank < 0 || c->rank >= c->world)
        throw std::invalid_argument("collectives: rank must be in [0, world)");
    if (c->world > 1 &&
        (!c->all_reduce_sum_u32 || !c->all_reduce_sum_u64 || !c->all_reduce_sum_f32 || !c->all_gather_u32))
        throw std::invalid_argument("collectives: missing entry point");
    if (c->world > 1 && sb_ == 0 && se_ == n_total_ && c->rank > 0)
        throw std::invalid_argument("collectives: a sharded engine needs its rank's path range (shard_begin/end)");
    coll_ = *c;
    if (!sharded()) return;
    const uint32_t W = static_cast<uint32_t>(coll_.world);
    d_gath_.alloc(4ull * W * max_cells_);
    std::vector<uint32_t*> tab(2 * PRX_MAX_LIGHTS, nullptr);
    for (size_t li = 0; li < lights_.size(); ++li) {
        LightBlock& b = lights_[li];
        b.pref.alloc(4ull * b.cells);
        b.tot.alloc(4ull * b.cells);
        tab[li] = b.pref.as<uint32_t>();
        tab[PRX_MAX_LIGHTS + li] = b.tot.as<uint32_t>();
    }
    PRX_CUDA(cudaMemcpy(d_light_ptrs_.as<uint32_t*>() + 4 * PRX_MAX_LIGHTS, tab.data(), sizeof(uint32_t*) * tab.size(),
                        cudaMemcpyHostToDevice));
    d_dead_g_.alloc(4ull * W * PRX_MAX_LIGHTS);
    d_dead_pt_.alloc(8ull * 2 * PRX_MAX_LIGHTS);
    d_ctr_sum_.alloc(sizeof(Counters));
    d_cnt32_sum_.alloc(4 * kCntN);
    if (!h_ctr_sum_) PRX_CUDA(cudaMallocHost(&h_ctr_sum_, sizeof(Counters)));
    if (!h_cnt32_sum_) PRX_CUDA(cudaMallocHost(&h_cnt32_sum_, 4 * kCntN));
}

void Engine::stage_trace() {
    const PathDev P = path_dev();
    uint32_t* cnt = d_cnt32_.as<uint32_t>();
    const uint32_t* list = d_list_.as<uint32_t>();
#if PRX_TRACE_LONGEST_FIRST
    // queue order = retrace start ascending (most bounces left first, stable within a start):
    // the persistent trace's tail is then made of the shortest paths.  Each path's result
    // depends on its own data only, so the order changes timing, not bits.
    int bits = 1;
    while ((1u << bits) <= B_) ++bits;
    launch_retrace_flags(P, d_flags8_.as<uint8_t>(), d_masks_.as<uint32_t>(), stream_);
    compact_u8_pairs(d_flags8_.as<uint8_t>(), d_masks_.as<uint32_t>(), n_, d_keys_.as<uint32_t>(),
                     d_vals_.as<uint32_t>(), cnt + kCntRetrace, d_scratch_.get(), stream_);
    list = radix_sort_pairs_nocopy(d_keys_.as<uint32_t>(), d_vals_.as<uint32_t>(), d_keys_tmp_.as<uint32_t>(),
                                   d_vals_tmp_.as<uint32_t>(), n_, cnt + kCntRetrace, bits, d_scratch_.get(), stream_)
               ? d_vals_tmp_.as<uint32_t>()
               : d_vals_.as<uint32_t>();
#else
    launch_retrace_flags(P, d_flags8_.as<uint8_t>(), nullptr, stream_);
    compact_u8(d_flags8_.as<uint8_t>(), n_, nullptr, 0, d_list_.as<uint32_t>(), cnt + kCntRetrace,
               d_scratch_.get(), stream_);
#endif
    launch_trace(scene_dev(), P, list, cnt + kCntRetrace, d_work_.as<uint32_t>(), d_ctr_.as<Counters>(), stream_);
    launch_finalize(P, d_ctr_.as<Counters>(), stream_);
}

void Engine::read_back(prx_frame_stats* st, bool with_times) {
    copy_async(h_ctr_, d_ctr_.get(), sizeof(Counters), cudaMemcpyDeviceToHost);
    copy_async(h_cnt32_, d_cnt32_.get(), 4 * kCntN, cudaMemcpyDeviceToHost);
    const bool summed = sharded() && in_sharded_frame_;
    in_sharded_frame_ = false;
    if (summed) {  // all-rank sums (exchange_counters) for the frame statistics
        copy_async(h_ctr_sum_, d_ctr_sum_.get(), sizeof(Counters), cudaMemcpyDeviceToHost);
        copy_async(h_cnt32_sum_, d_cnt32_sum_.get(), 4 * kCntN, cudaMemcpyDeviceToHost);
    }
    PRX_CUDA(cudaStreamSynchronize(stream_));
    PRX_CUDA(cudaGetLastError());
    n_pruned_ = h_cnt32_[kCntPruned];
    launches_ = g_launches - launch_base_;
    const Counters& C = summed ? *h_ctr_sum_ : *h_ctr_;
    const uint32_t* c32 = summed ? h_cnt32_sum_ : h_cnt32_;
    if (C.fill_overflow) throw std::logic_error("fill: ran out of free path slots");
    if (!st) return;
    st->frame = cur_frame_;
    st->mode = cfg_.mode;
    st->rays_traced = C.traced;
    st->rays_reused = C.segments - C.traced;
    st->paths_replaced = C.replaced;
    st->paths_pruned = c32[kCntPruned];
    st->paths_filled = C.filled;
    st->visibility_rays = C.vis;
    st->live_segments_before = C.live_segments;
    st->paths_retraced = c32[kCntRetrace];
    if (with_times) {
        st->t_update = elapsed_ms(kEvVerify0, kEvOccl0) * 1e-3;
        st->t_occlusion = elapsed_ms(kEvOccl0, kEvDm0) * 1e-3;
        st->t_dm = elapsed_ms(kEvDm0, kEvPrune0) * 1e-3;
        st->t_prune = elapsed_ms(kEvPrune0, kEvFill0) * 1e-3;
        st->t_fill = elapsed_ms(kEvFill0, kEvTrace0) * 1e-3;
        st->t_trace = elapsed_ms(kEvTrace0, kEvEnd) * 1e-3;
        st->ms_frame_update = elapsed_ms(kEvFrame0, kEvVerify0);
        st->ms_verify = elapsed_ms(kEvVerify0, kEvPrune0);
        st->ms_retrace = elapsed_ms(kEvPrune0, kEvEnd);
    }
}

void Engine::retrace_invalid(prx_frame_stats* st) {
    retrace_enqueue();
    read_back(st, true);
}

void Engine::retrace_enqueue() {
    PRX_CUDA(cudaSetDevice(device_));
    record(kEvPrune0);
    in_full_frame_ = true;  // prune -> fill -> trace run back to back: skip the prune clears
    in_sharded_frame_ = sharded();
    if (cfg_.mode != PRX_MODE_BASELINE) {
        if (sharded()) stage_prune_sharded();
        else stage_prune_local();
    }
    in_full_frame_ = false;
    record(kEvFill0);
    if (sharded()) stage_fill_sharded();
    else stage_fill_local();
    record(kEvTrace0);
    stage_trace();
    if (sharded()) exchange_counters();
    record(kEvEnd);
}

// One frame. The device work of a frame depends on the host only through a few decisions
// (first frame, lights moved, occlusion boxes present, dynamics moved, mode); a frame whose
// decisions repeat the previous frame's is captured once as a CUDA graph and replayed
// (its uploads read the pinned frame parameters at execution time), removing the per-launch
// gaps of ~120 small launches. PRX_GRAPHS=0 keeps plain stream launches.
void Engine::run_frame(prx_frame_stats* st) {
    PRX_CUDA(cudaSetDevice(device_));
    if (st) std::memset(st, 0, sizeof(*st));
    frame_update_host();
    bool any_moved = false;
    for (const LightBlock& b : lights_) any_moved = any_moved || b.moved;
    const uint32_t sig = (cur_frame_ > 0 ? 1u : 0u) | (any_moved ? 2u : 0u) | (h_fp_->n_boxes > 0 ? 4u : 0u) |
                         (dyn_changed_ ? 8u : 0u) | (static_cast<uint32_t>(cfg_.mode) << 4);
    auto plain = [&] {
        frame_update_enqueue();
        const bool pre = splat_prefix_fork();
        verify_paths(nullptr);
        retrace_enqueue();
        if (pre) splat_prefix_join();
    };
    // (sharded frames run plain launches: their exchanges call back into the collectives)
    const bool graphs = graphs_on_ && !sharded();
    auto it = graphs ? graphs_.find(sig) : graphs_.end();
    if (it != graphs_.end()) {
        launch_graph(it->second);
    } else if (graphs && sig == last_sig_) {
        FrameGraph g;
        if (capture_graph(plain, g)) graphs_[sig] = g;
    } else {
        plain();
    }
    last_sig_ = sig;
    if (splat_pending_) {  // (the frame waited for it: its prefix branch joined after the splat's end)
        splat_pending_ = false;
        finish_splat();
    }
    pre_ok_ = pre_on_ && pre_radius_ > 0.0f;  // (graphs are dropped when the prefix radius changes)
    if (st) {
        st->frame = cur_frame_;
        st->mode = cfg_.mode;
    }
    read_back(st, true);
}

// Capture `enqueue` into a graph and launch it once; on any capture failure run it on the
// stream as usual and stay on plain launches from then on.
template <typename F>
bool Engine::capture_graph(F&& enqueue, FrameGraph& out) {
    if (!capture_stream_) PRX_CUDA(cudaStreamCreateWithFlags(&capture_stream_, cudaStreamNonBlocking));
    const cudaStream_t saved = stream_;
    const uint64_t h2d0 = h2d_bytes_, d2h0 = d2h_bytes_, l0 = g_launches;
    cudaGraph_t graph = nullptr;
    stream_ = capture_stream_;
    capturing_ = true;
    cudaError_t err = cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal);
    if (err == cudaSuccess) {
        try {
            enqueue();
        } catch (...) {
            err = cudaErrorStreamCaptureInvalidated;
        }
        const cudaError_t end = cudaStreamEndCapture(stream_, &graph);
        if (err == cudaSuccess) err = end;
    }
    capturing_ = false;
    stream_ = saved;
    cudaGraphExec_t exec = nullptr;
    if (err == cudaSuccess && graph) err = cudaGraphInstantiate(&exec, graph, 0);
    if (graph) cudaGraphDestroy(graph);
    if (err != cudaSuccess || !exec) {  // stay on plain launches; the frame was not executed
        cudaGetLastError();
        graphs_on_ = false;
        h2d_bytes_ = h2d0;
        d2h_bytes_ = d2h0;
        g_launches = l0;
        enqueue();
        return false;
    }
    out.exec = exec;
    out.h2d = h2d_bytes_ - h2d0;
    out.d2h = d2h_bytes_ - d2h0;
    out.launches = g_launches - l0;
    for (int k = 0; k < 12; ++k) out.ev[k] = ev_recorded_[k];
    PRX_CUDA(cudaGraphLaunch(exec, stream_));
    return true;
}

void Engine::launch_graph(const FrameGraph& g) {
    PRX_CUDA(cudaGraphLaunch(g.exec, stream_));
    h2d_bytes_ += g.h2d;
    d2h_bytes_ += g.d2h;
    g_launches += g.launches;
    for (int k = 0; k < 12; ++k)
        if (g.ev[k]) ev_recorded_[k] = true;
}

void Engine::run_stage(int stage, prx_frame_stats* st) {
    PRX_CUDA(cudaSetDevice(device_));
    const bool active = cfg_.mode != PRX_MODE_BASELINE && cur_frame_ > 0;
    if (sharded() && (stage == PRX_STAGE_PRUNE || stage == PRX_STAGE_FILL))
        throw std::logic_error("run_stage: prune/fill of a sharded engine run inside retrace_invalid / run_frame");
    prx_frame_stats tmp{};
    switch (stage) {
        case PRX_STAGE_UPDATE_ORIGINS:
            if (active) stage_update_origins();
            break;
        case PRX_STAGE_OCCLUSIONS:
            if (active) stage_occlusions();
            break;
        case PRX_STAGE_COMPUTE_DM: stage_compute_dm(); break;
        case PRX_STAGE_PRUNE:
            if (cfg_.mode != PRX_MODE_BASELINE) stage_prune_local();
            break;
        case PRX_STAGE_FILL: stage_fill_local(); break;
        case PRX_STAGE_TRACE: stage_trace(); break;
        case PRX_STAGE_RELEASE_ALL:
            launch_release_all(path_dev(), stream_);
            for (LightBlock& b : lights_) PRX_CUDA(cudaMemsetAsync(b.dm_c.get(), 0, 4ull * b.cells, stream_));
            break;
        default: throw std::invalid_argument("unknown stage");
    }
    read_back(&tmp, false);
    if (st) {  // counters accumulate over the frame; report the running totals
        st->frame = tmp.frame;
        st->mode = tmp.mode;
        st->rays_traced = tmp.rays_traced;
        st->rays_reused = stage == PRX_STAGE_TRACE ? tmp.rays_reused : 0;
        st->paths_replaced = tmp.paths_replaced;
        st->paths_pruned = tmp.paths_pruned;
        st->paths_filled = tmp.paths_filled;
        st->visibility_rays = tmp.visibility_rays;
        st->paths_retraced = tmp.paths_retraced;
        st->live_segments_before = tmp.live_segments_before;
    }
}

// ----------------------------------------------------------------------- sharded exchange
void Engine::dm_current_ptr(uint32_t light, void** ptr, uint32_t* cells) {
    if (light >= lights_.size()) throw std::out_of_range("light index");
    *ptr = lights_[light].dm_c.get();
    *cells = lights_[light].cells;
}

void Engine::prune_count(uint32_t* const* unmarked_dev) {
    PRX_CUDA(cudaSetDevice(device_));
    prune_mark_all();
    for (size_t li = 0; li < lights_.size(); ++li)
        PRX_CUDA(cudaMemcpyAsync(unmarked_dev[li], lights_[li].unm.get(), 4ull * lights_[li].cells,
                                 cudaMemcpyDeviceToDevice, stream_));
}

void Engine::prune_apply(const uint32_t* const* prefix_dev, const uint32_t* const* total_dev,
                         prx_frame_stats* st) {
    PRX_CUDA(cudaSetDevice(device_));
    // device pointer tables [2] prefix, [3] total
    std::vector<const uint32_t*> tab(2 * PRX_MAX_LIGHTS, nullptr);
    for (size_t li = 0; li < lights_.size(); ++li) {
        tab[li] = prefix_dev[li];
        tab[PRX_MAX_LIGHTS + li] = total_dev[li];
    }
    uint32_t** dtab = d_light_ptrs_.as<uint32_t*>() + 2 * PRX_MAX_LIGHTS;
    copy_async(dtab, tab.data(), sizeof(uint32_t*) * tab.size(), cudaMemcpyHostToDevice);
    prune_trim_all(dtab, dtab + PRX_MAX_LIGHTS, total_dev);
    read_back(st, false);
}

void Engine::fill_count(uint32_t* dead_out) {
    PRX_CUDA(cudaSetDevice(device_));
    fill_collect_dead();
    read_back(nullptr, false);
    for (size_t li = 0; li < lights_.size(); ++li) dead_out[li] = h_cnt32_[kCntDead0 + li];
}

void Engine::fill_apply(const uint64_t* dead_prefix, const uint64_t* dead_total, prx_frame_stats* st) {
    PRX_CUDA(cudaSetDevice(device_));
    fill_assign_all(dead_prefix, dead_total);
    read_back(st, false);
}

// ----------------------------------------------------------------------- splat
void Engine::splat(const prx_camera* cam, float radius, int mode, float* rgb_host, float* rgb_dev,
                   prx_frame_stats* st) {
    splat_store(path_dev(), cam, radius, mode, rgb_host, rgb_dev, st, sharded());
}

// gather_image(state, photons, aux, ...) over a host photon map (gather.hpp:81-83): the
// records are converted to the engine's 32-byte {pos_obj, energy} vertex layout, uploaded
// to scratch and splatted against the scene as placed for the engine's current frame.
void Engine::gather_photons(const void* photons, const void* aux, uint32_t n_paths, uint32_t max_bounces,
                            int frame, const prx_camera* cam, float radius, int mode, float* rgb_host) {
    PRX_CUDA(cudaSetDevice(device_));
    if (frame != cur_frame_)
        throw std::invalid_argument("gather_image: the scene state is not the engine's current frame");
    if ((n_paths && max_bounces && (!photons || !aux)) || !rgb_host)
        throw std::invalid_argument("gather_image: NULL photon, aux or image buffer");
    const size_t nv = static_cast<size_t>(n_paths) * max_bounces;
    struct RefPhoton { float dir[3]; uint32_t obj; float e[3]; float radius; };
    struct RefAux { float pos[3]; float out[3]; };
    static_assert(sizeof(RefPhoton) == 32 && sizeof(RefAux) == 24, "reference record sizes");
    // the engine's vertex layout (kVS, dev_types.h): {pos_obj, energy} streams
    const size_t second = PRX_VERTEX_SOA ? nv : 1;
    std::vector<float4> rec(2 * std::max<size_t>(nv, 1));
    const auto* ph = static_cast<const RefPhoton*>(photons);
    const auto* ax = static_cast<const RefAux*>(aux);
    for (size_t v = 0; v < nv; ++v) {
        float w;
        std::memcpy(&w, &ph[v].obj, 4);
        rec[kVS * v] = float4{ax[v].pos[0], ax[v].pos[1], ax[v].pos[2], w};
        rec[kVS * v + second] = float4{ph[v].e[0], ph[v].e[1], ph[v].e[2], ph[v].radius};
    }
    DevBuf store(sizeof(float4) * rec.size());
    copy_async(store.get(), rec.data(), sizeof(float4) * 2 * nv, cudaMemcpyHostToDevice);
    PathDev P{};
    P.n = n_paths;
    P.B = max_bounces;
    P.pos_obj = store.as<float4>();
    P.energy = store.as<float4>() + second;
    d_gather_.reset();  // sized for this store
    splat_store(P, cam, radius, mode, rgb_host, nullptr, nullptr, false);
    d_gather_.reset();
}

// camera_ray (gather.cpp:22-33): per-image constants on the host libm
CamDev Engine::camera_dev(const Camera& c) const {
    CamDev C{};
    C.pos = c.position;
    C.fwd = normalized(sub(c.look_at, c.position));
    V3 up{0, 1, 0};
    if (std::abs(dot(C.fwd, up)) > 0.999f) up = V3{1, 0, 0};
    C.right = normalized(cross(C.fwd, up));
    C.up = cross(C.right, C.fwd);
    C.tan_half = std::tan(c.fov_deg * static_cast<float>(M_PI) / 360.0f);
    C.aspect = static_cast<float>(c.width) / static_cast<float>(c.height);
    C.w = c.width;
    C.h = c.height;
    return C;
}

// Fork the splat prefix of the scene camera onto the side stream once the frame has placed the
// dynamics; it overlaps verify/retrace (it reads only the scene). false: no prefix this frame.
bool Engine::splat_prefix_fork() {
    if (!pre_on_ || !(pre_radius_ > 0.0f)) return false;
    const Camera& c = scene_->camera;
    if (c.width == 0 || c.height == 0) return false;
    const uint32_t npx = c.width * c.height;
    if (d_pre_gbuf_.size() == 0) {
        pre_bits_ = splat_table_bits_capped(npx);
        d_pre_gbuf_.alloc(16ull * npx);
        d_pre_work_.alloc(splat_work_bytes(pre_bits_));
    }
    PRX_CUDA(cudaEventRecord(ev_fork_, stream_));
    PRX_CUDA(cudaStreamWaitEvent(side_stream_, ev_fork_, 0));
    wait_splat(side_stream_, true);  // (the prefix rewrites the tables an overlapped splat reads)
    launch_splat_prefix(scene_dev(), camera_dev(c), pre_radius_, d_pre_gbuf_.as<float4>(), d_pre_work_.get(),
                        pre_bits_, side_stream_);
    // the registered-cell count sizes the splat's sort keys and shows a table overflow (read
    // after the frame's sync)
    PRX_CUDA(cudaMemcpyAsync(h_ncell_, d_pre_work_.as<char>() + splat_ncell_offset(pre_bits_), 4,
                             cudaMemcpyDeviceToHost, side_stream_));
    d2h_bytes_ += 4;
    return true;
}

void Engine::splat_prefix_join() {
    PRX_CUDA(cudaEventRecord(ev_join_, side_stream_));
    PRX_CUDA(cudaStreamWaitEvent(stream_, ev_join_, 0));
}

void Engine::splat_store(const PathDev& P, const prx_camera* cam, float radius, int mode, float* rgb_host,
                         float* rgb_dev, prx_frame_stats* st, bool reduce_ranks) {
    PRX_CUDA(cudaSetDevice(device_));
    if (!(radius > 0.0f)) throw std::invalid_argument("gather: radius must be positive");
    if (mode != 0 && mode != 1) throw std::invalid_argument("splat: mode must be 0 (atomic splat) or 1 (ordered gather)");
    Camera c = scene_->camera;
    bool scene_cam = true;
    if (cam) {
        c.position = V3{cam->position.x, cam->position.y, cam->position.z};
        c.look_at = V3{cam->look_at.x, cam->look_at.y, cam->look_at.z};
        c.fov_deg = cam->fov_deg;
        c.width = cam->width;
        c.height = cam->height;
        const Camera& s = scene_->camera;
        auto eq = [](const V3& a, const V3& b) { return a.x == b.x && a.y == b.y && a.z == b.z; };
        scene_cam = eq(c.position, s.position) && eq(c.look_at, s.look_at) && c.fov_deg == s.fov_deg &&
                    c.width == s.width && c.height == s.height;
    }
    if (c.width == 0 || c.height == 0) throw std::invalid_argument("splat: empty image");
    const CamDev C = camera_dev(c);
    const uint32_t npx = c.width * c.height;
    // a scene-camera splat at the radius the frame's side stream used skips the G-buffer and
    // the cell keys; a new radius becomes the prefix radius of the following frames
    bool use_pre = false;
    if (scene_cam && pre_on_) {
        if (radius == pre_radius_) {
            use_pre = pre_ok_;
        } else {
            pre_radius_ = radius;
            pre_ok_ = false;
            drop_graphs();  // their side branch bakes the old radius in
        }
    }
    if (use_pre && splat_table_overflow(h_ncell_[0], pre_bits_)) use_pre = false;  // (rebuilt below)
    const bool overlap = splat_overlap_ && use_pre && !st && !reduce_ranks && !capturing_;
    if (!overlap) join_splat();
    if (c.width != img_w_ || c.height != img_h_) {
        d_gbuf_.alloc(16ull * npx);
        d_img_.alloc(12ull * npx);
        d_splat_work_.reset();
        splat_work_bits_ = 0;
        d_gather_.reset();
        img_w_ = c.width;
        img_h_ = c.height;
    }
    const uint64_t nv = static_cast<uint64_t>(P.n) * P.B;
    const float inv_area = 1.0f / (static_cast<float>(M_PI) * radius * radius);
    const float inv_pi = 1.0f / static_cast<float>(M_PI);
    float* out = rgb_dev ? rgb_dev : d_img_.as<float>();
    const SceneDev S = scene_dev();
    // (plain launches: a captured graph of these ~25 launches measured slower, 1.93 vs 1.89 ms)
    record(kEvSplat0);
    int bits = pre_bits_, cell_bits = 0;
    float4* gbuf = d_pre_gbuf_.as<float4>();
    void* work = d_pre_work_.get();
    if (use_pre) {
        cell_bits = splat_cell_bits(h_ncell_[0]);
    } else {
        // the prefix inline: a capped table first; when capped, one read-back of its load (a
        // rebuild at the worst-case size on overflow) that also sizes the sort keys
        bits = splat_table_bits_capped(npx);
        auto run_prefix = [&](int b) {
            if (splat_work_bits_ < b) {
                d_splat_work_.alloc(splat_work_bytes(b));
                splat_work_bits_ = b;
            }
            launch_splat_prefix(S, C, radius, d_gbuf_.as<float4>(), d_splat_work_.get(), b, stream_);
        };
        run_prefix(bits);
        if (bits < splat_table_bits(npx)) {
            copy_async(h_ncell_ + 1, d_splat_work_.as<char>() + splat_ncell_offset(bits), 4, cudaMemcpyDeviceToHost);
            PRX_CUDA(cudaStreamSynchronize(stream_));
            if (splat_table_overflow(h_ncell_[1], bits)) {
                bits = splat_table_bits(npx);
                run_prefix(bits);
            } else {
                cell_bits = splat_cell_bits(h_ncell_[1]);
            }
        }
        gbuf = d_gbuf_.as<float4>();
        work = d_splat_work_.get();
    }
    if (d_gather_.size() == 0 || gather_bits_ < bits) {  // both modes
        d_gather_.alloc(gather_work_bytes(nv, npx, bits));
        gather_bits_ = bits;
    }
    if (overlap) {  // on the side stream after the frame; no host wait (see prx_engine_set_splat_overlap)
        PRX_CUDA(cudaEventRecord(ev_fork_, stream_));
        PRX_CUDA(cudaStreamWaitEvent(side_stream_, ev_fork_, 0));
        launch_splat(S, P, C, radius, gbuf, out, inv_pi, inv_area, work, d_splat_cand_.get(), mode, d_gather_.get(),
                     bits, true, cell_bits, side_stream_, ev_splat_read_);
        if (rgb_host) {  // -> pinned staging now, -> rgb_host in finish_splat
            const size_t bytes = 12ull * npx;
            if (h_img_stage_bytes_ < bytes) {
                if (h_img_stage_) PRX_CUDA(cudaFreeHost(h_img_stage_));
                PRX_CUDA(cudaHostAlloc(&h_img_stage_, bytes, cudaHostAllocDefault));
                h_img_stage_bytes_ = bytes;
            }
            PRX_CUDA(cudaMemcpyAsync(h_img_stage_, out, bytes, cudaMemcpyDeviceToHost, side_stream_));
            d2h_bytes_ += bytes;
            pending_host_out_ = rgb_host;
            pending_host_bytes_ = bytes;
        }
        PRX_CUDA(cudaEventRecord(ev_splat_, side_stream_));
        PRX_CUDA(cudaGetLastError());
        splat_pending_ = true;
        launches_ = g_launches - launch_base_;
        return;
    }
    launch_splat(S, P, C, radius, gbuf, out, inv_pi, inv_area, work, d_splat_cand_.get(), mode, d_gather_.get(), bits,
                 true, cell_bits, stream_);
    if (reduce_ranks)  // every rank splats its own photons; the image is their sum
        coll_ok(coll_.all_reduce_sum_f32(coll_.ctx, out, 3ull * npx, stream_), "image all-reduce");
    record(kEvSplat1);
    if (rgb_host)
        copy_async(rgb_host, out, 12ull * npx, cudaMemcpyDeviceToHost);
    PRX_CUDA(cudaStreamSynchronize(stream_));
    PRX_CUDA(cudaGetLastError());
    launches_ = g_launches - launch_base_;
    if (st) {
        st->ms_splat = elapsed_ms(kEvSplat0, kEvSplat1);
        st->t_gather = st->ms_splat * 1e-3;
    }
}

// ----------------------------------------------------------------------- scene queries
void Engine::intersect_batch(const float* rays, size_t n, int any_hit, float* hits) {
    PRX_CUDA(cudaSetDevice(device_));
    if (n == 0) return;
    if (n > 0xFFFFFFFFull / 9) throw std::invalid_argument("intersect_batch: too many rays");
    const size_t out_floats = any_hit ? n : 9 * n;
    DevBuf d_rays, d_out;
    d_rays.alloc(sizeof(float) * 8 * n);
    d_out.alloc(sizeof(float) * out_floats);
    copy_async(d_rays.get(), rays, sizeof(float) * 8 * n, cudaMemcpyHostToDevice);
    launch_intersect_batch(scene_dev(), d_rays.as<float>(), static_cast<uint32_t>(n), any_hit, d_out.as<float>(),
                           stream_);
    copy_async(hits, d_out.get(), sizeof(float) * out_floats, cudaMemcpyDeviceToHost);
    PRX_CUDA(cudaStreamSynchronize(stream_));
    PRX_CUDA(cudaGetLastError());
}

// ----------------------------------------------------------------------- field I/O
size_t Engine::field_bytes(int field, uint32_t index) const {
    const size_t nv = static_cast<size_t>(n_) * B_;
    switch (field) {
        case PRX_FIELD_PHOTONS: return nv * 32;
        case PRX_FIELD_AUX: return nv * 24;
        case PRX_FIELD_POS_OBJ:
        case PRX_FIELD_ENERGY:
        case PRX_FIELD_IN_DIR:
        case PRX_FIELD_OUT_DIR: return nv * 16;
        case PRX_FIELD_ORIGIN:
        case PRX_FIELD_EMISSION_DIR:
        case PRX_FIELD_CANONICAL: return 16ull * n_;
        case PRX_FIELD_CELL:
        case PRX_FIELD_EPOCH:
        case PRX_FIELD_PATH_INFO:
        case PRX_FIELD_META:
        case PRX_FIELD_SEGMENT_FLAGS: return 4ull * n_;
        case PRX_FIELD_RETRACE_START: return n_;
        case PRX_FIELD_DM_TARGET:
        case PRX_FIELD_DM_CURRENT:
            if (index >= lights_.size()) throw std::out_of_range("light index out of range");
            return 4ull * lights_[index].cells;
        case PRX_FIELD_PRUNED: return 4ull * n_pruned_;
    }
    throw std::invalid_argument("unknown field");
}

namespace {
struct FieldPtr {
    void* p;
    bool convert;
};
}  // namespace

void Engine::download(int field, uint32_t index, void* dst, size_t bytes) {
    PRX_CUDA(cudaSetDevice(device_));
    if (bytes != field_bytes(field, index)) throw std::invalid_argument("download: size mismatch");
    if (bytes == 0) return;
    void* src = nullptr;
    DevBuf tmp;
    switch (field) {
        case PRX_FIELD_PHOTONS:
            tmp.alloc(bytes);
            launch_pack_photons(path_dev(), tmp.get(), nullptr, stream_);
            src = tmp.get();
            break;
        case PRX_FIELD_AUX:
            tmp.alloc(bytes);
            launch_pack_photons(path_dev(), nullptr, tmp.get(), stream_);
            src = tmp.get();
            break;
        case PRX_FIELD_POS_OBJ:
        case PRX_FIELD_ENERGY:
        case PRX_FIELD_IN_DIR:
        case PRX_FIELD_OUT_DIR: {  // one float4 per vertex of that stream (stride kVS)
            const PathDev P = path_dev();
            const float4* base = field == PRX_FIELD_POS_OBJ ? P.pos_obj
                                 : field == PRX_FIELD_ENERGY ? P.energy
                                 : field == PRX_FIELD_IN_DIR ? P.in_dir : P.out_dir;
            PRX_CUDA(cudaMemcpy2DAsync(dst, 16, base, 16 * kVS, 16, bytes / 16, cudaMemcpyDeviceToHost, stream_));
            d2h_bytes_ += bytes;
            PRX_CUDA(cudaStreamSynchronize(stream_));
            return;
        }
        case PRX_FIELD_ORIGIN: src = d_origin_.get(); break;
        case PRX_FIELD_EMISSION_DIR: src = d_emis_.get(); break;
        case PRX_FIELD_CANONICAL: src = d_canon_.get(); break;
        case PRX_FIELD_CELL: src = d_cell_.get(); break;
        case PRX_FIELD_EPOCH: src = d_epoch_.get(); break;
        case PRX_FIELD_PATH_INFO: src = d_path_info_.get(); break;
        case PRX_FIELD_META: src = d_meta_.get(); break;
        case PRX_FIELD_RETRACE_START: src = d_rstart_.get(); break;
        case PRX_FIELD_SEGMENT_FLAGS: src = d_seg_flags_.get(); break;
        case PRX_FIELD_DM_TARGET: src = lights_[index].dm_t.get(); break;
        case PRX_FIELD_DM_CURRENT: src = lights_[index].dm_c.get(); break;
        case PRX_FIELD_PRUNED: src = d_pruned_list_.get(); break;
        default: throw std::invalid_argument("unknown field");
    }
    copy_async(dst, src, bytes, cudaMemcpyDeviceToHost);
    PRX_CUDA(cudaStreamSynchronize(stream_));
}

void Engine::upload(int field, uint32_t index, const void* src, size_t bytes) {
    PRX_CUDA(cudaSetDevice(device_));
    if (bytes != field_bytes(field, index)) throw std::invalid_argument("upload: size mismatch");
    if (bytes == 0) return;
    void* dst = nullptr;
    DevBuf tmp;
    switch (field) {
        case PRX_FIELD_PHOTONS:
        case PRX_FIELD_AUX: {
            tmp.alloc(bytes);
            copy_async(tmp.get(), src, bytes, cudaMemcpyHostToDevice);
            if (field == PRX_FIELD_PHOTONS) launch_unpack_photons(path_dev(), tmp.get(), nullptr, stream_);
            else launch_unpack_photons(path_dev(), nullptr, tmp.get(), stream_);
            PRX_CUDA(cudaStreamSynchronize(stream_));
            return;
        }
        case PRX_FIELD_POS_OBJ:
        case PRX_FIELD_ENERGY:
        case PRX_FIELD_IN_DIR:
        case PRX_FIELD_OUT_DIR: {
            const PathDev P = path_dev();
            float4* base = field == PRX_FIELD_POS_OBJ ? P.pos_obj
                           : field == PRX_FIELD_ENERGY ? P.energy
                           : field == PRX_FIELD_IN_DIR ? P.in_dir : P.out_dir;
            PRX_CUDA(cudaMemcpy2DAsync(base, 16 * kVS, src, 16, 16, bytes / 16, cudaMemcpyHostToDevice, stream_));
            h2d_bytes_ += bytes;
            PRX_CUDA(cudaStreamSynchronize(stream_));
            return;
        }
        case PRX_FIELD_ORIGIN: dst = d_origin_.get(); break;
        case PRX_FIELD_EMISSION_DIR: dst = d_emis_.get(); break;
        case PRX_FIELD_CANONICAL: dst = d_canon_.get(); break;
        case PRX_FIELD_CELL: dst = d_cell_.get(); break;
        case PRX_FIELD_EPOCH: dst = d_epoch_.get(); break;
        case PRX_FIELD_PATH_INFO: dst = d_path_info_.get(); break;
        case PRX_FIELD_META: dst = d_meta_.get(); break;
        case PRX_FIELD_RETRACE_START: dst = d_rstart_.get(); break;
        case PRX_FIELD_SEGMENT_FLAGS: dst = d_seg_flags_.get(); break;
        case PRX_FIELD_DM_TARGET: dst = lights_[index].dm_t.get(); break;
        case PRX_FIELD_DM_CURRENT: dst = lights_[index].dm_c.get(); break;
        case PRX_FIELD_PRUNED: throw std::invalid_argument("upload: the pruned list is read-only");
        default: throw std::invalid_argument("unknown field");
    }
    copy_async(dst, src, bytes, cudaMemcpyHostToDevice);
    PRX_CUDA(cudaStreamSynchronize(stream_));
}

void Engine::set_frame_counter(int frames_run) {
    if (frames_run < 0) throw std::invalid_argument("frames_run must be >= 0");
    PRX_CUDA(cudaSetDevice(device_));
    frames_run_ = frames_run;
    cur_frame_ = frames_run > 0 ? frames_run - 1 : 0;
    for (LightBlock& b : lights_) {
        b.pose_now = light_pose_at(*b.light, cur_frame_);
        b.pose_prev = b.pose_now;
        b.moved = false;
    }
    place_frame(cur_frame_);
    fill_frame_params();
    place_dynamics(true);
    PRX_CUDA(cudaStreamSynchronize(stream_));
}

void Engine::set_stream(cudaStream_t s) {
    PRX_CUDA(cudaStreamSynchronize(stream_));
    if (own_stream_ && stream_) cudaStreamDestroy(stream_);
    if (s) {
        stream_ = s;
        own_stream_ = false;
    } else {
        PRX_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
        own_stream_ = true;
    }
}

void Engine::synchronize() {
    join_splat();
    PRX_CUDA(cudaStreamSynchronize(stream_));
}

void Engine::set_splat_overlap(bool on) {
    if (on == splat_overlap_) return;
    join_splat();
    splat_overlap_ = on;
    drop_graphs();  // (captured frames carry the overlap waits or not)
}

void Engine::join_splat() {
    if (!splat_pending_) return;
    PRX_CUDA(cudaStreamWaitEvent(stream_, ev_splat_, 0));
    splat_pending_ = false;
    finish_splat();
}

// the host part of an overlapped splat with a host output: wait for it, copy out of staging
void Engine::finish_splat() {
    if (!pending_host_out_) return;
    PRX_CUDA(cudaEventSynchronize(ev_splat_));
    std::memcpy(pending_host_out_, h_img_stage_, pending_host_bytes_);
    pending_host_out_ = nullptr;
}

// a frame's wait for an overlapped splat: a plain stream wait, or inside a frame-graph capture an
// external event-wait node (it waits for the splat enqueued before each replay; when none is,
// the event's last record has long completed)
// (whole: the splat's end; else its last read of the photon map -- the sort's gather pass)
void Engine::wait_splat(cudaStream_t s, bool whole) {
    if (!splat_overlap_) return;
    cudaEvent_t e = whole ? ev_splat_ : ev_splat_read_;
    if (capturing_)
        PRX_CUDA(cudaStreamWaitEvent(s, e, cudaEventWaitExternal));
    else if (splat_pending_)
        PRX_CUDA(cudaStreamWaitEvent(s, e, 0));
}

void Engine::info(prx_engine_info* out) const {
    std::memset(out, 0, sizeof(*out));
    out->n_paths = n_total_;
    out->max_bounces = B_;
    out->n_lights = static_cast<uint32_t>(lights_.size());
    out->shard_begin = sb_;
    out->shard_end = se_;
    out->eps_world = eps_;
    out->diagonal = diag_;
    out->frames_run = frames_run_;
    out->n_pruned = n_pruned_;
    for (size_t li = 0; li < lights_.size(); ++li) {
        const LightBlock& b = lights_[li];
        out->light_path_begin[li] = b.begin;
        out->light_path_end[li] = b.end;
        out->dm_ndims[li] = b.ndims;
        for (int a = 0; a < 4; ++a) out->dm_dims[li][a] = b.dims[a];
        out->dm_cells[li] = b.cells;
        out->flux_per_path[li][0] = b.flux_pp.x;
        out->flux_per_path[li][1] = b.flux_pp.y;
        out->flux_per_path[li][2] = b.flux_pp.z;
    }
    uint64_t bytes = 0;
    for (const DevBuf* b : {&d_hot_, &d_stris_, &d_dyn_local_, &d_dyn_world_, &d_lbvh_nodes_, &d_pos_obj_,
                            &d_in_dir_, &d_origin_, &d_emis_, &d_canon_, &d_cell_,
                            &d_epoch_, &d_path_info_, &d_seg_flags_, &d_meta_, &d_rstart_, &d_list_, &d_masks_,
                            &d_keys_, &d_vals_, &d_keys_tmp_, &d_vals_tmp_, &d_pruned_list_})
        bytes += b->size();
    out->device_bytes = bytes;
}

}  // namespace prx
