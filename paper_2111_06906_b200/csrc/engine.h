// engine.h -- host side of one B200 path-reuse engine (one GPU, one path shard).
//
// Mirrors pathreuse::Engine (engine.hpp:69-179): owns the device path store, the scene's
// device copy, per-light distribution maps, and orchestrates the frame as the north_star
// stages frame_update / verify_paths / retrace_invalid, all enqueued on
// one CUDA stream with no host round trip until the frame's statistics are read back.
#pragma once

#include <cuda_runtime.h>

#include <memory>
#include <stdexcept>
#include <string>
#include <map>
#include <vector>

#include "dev_types.h"
#include "host_scene.h"
#include "kernels.h"
#include "prx.h"

namespace prx {

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

void cuda_check(cudaError_t e, const char* what);
#define PRX_CUDA(x) ::prx::cuda_check((x), #x)

// RAII device allocation
class DevBuf {
public:
    DevBuf() = default;
    explicit DevBuf(size_t bytes) { alloc(bytes); }
    ~DevBuf() { reset(); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr, o.n_ = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        reset();
        p_ = o.p_;
        n_ = o.n_;
        o.p_ = nullptr;
        o.n_ = 0;
        return *this;
    }
    void alloc(size_t bytes);
    void reset();
    template <typename T>
    T* as() const { return static_cast<T*>(p_); }
    void* get() const { return p_; }
    size_t size() const { return n_; }

private:
    void* p_ = nullptr;
    size_t n_ = 0;
};

class Engine {
public:
    Engine(std::shared_ptr<const Scene> scene, const prx_config& cfg);
    ~Engine();
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;

    void frame_update(prx_frame_stats* st);
    void verify_paths(prx_frame_stats* st);
    void retrace_invalid(prx_frame_stats* st);
    void run_frame(prx_frame_stats* st);
    void run_stage(int stage, prx_frame_stats* st);

    // sharded exchange points
    void dm_current_ptr(uint32_t light, void** ptr, uint32_t* cells);
    void prune_count(uint32_t* const* unmarked_dev);
    void prune_apply(const uint32_t* const* prefix_dev, const uint32_t* const* total_dev, prx_frame_stats* st);
    void fill_count(uint32_t* dead_out);
    void fill_apply(const uint64_t* dead_prefix, const uint64_t* dead_total, prx_frame_stats* st);

    void splat(const prx_camera* cam, float radius, int mode, float* rgb_host, float* rgb_dev,
               prx_frame_stats* st);
    void gather_photons(const void* photons, const void* aux, uint32_t n_paths, uint32_t max_bounces, int frame,
                        const prx_camera* cam, float radius, int mode, float* rgb_host);

    size_t field_bytes(int field, uint32_t index) const;
    void download(int field, uint32_t index, void* dst, size_t bytes);
    void upload(int field, uint32_t index, const void* src, size_t bytes);
    void set_frame_counter(int frames_run);
    void intersect_batch(const float* rays, size_t n, int any_hit, float* hits);
    void set_stream(cudaStream_t s);
    void set_collectives(const prx_collectives* c);  // in-engine sharded frames (comm.cpp)
    void synchronize();
    // overlapped splat (prx_engine_set_splat_overlap): join_splat orders the engine stream
    // after a pending one (every C-ABI entry but run_frame / splat calls it)
    void set_splat_overlap(bool on);
    void join_splat();
    void info(prx_engine_info* out) const;
    uint64_t launches() const { return launches_; }
    // bytes moved host->device / device->host by this engine since creation
    void transfer_bytes(uint64_t* h2d, uint64_t* d2h) const {
        if (h2d) *h2d = h2d_bytes_;
        if (d2h) *d2h = d2h_bytes_;
    }

private:
    // every host<->device copy of the frame/splat/field paths goes through here (counted)
    void copy_async(void* dst, const void* src, size_t bytes, cudaMemcpyKind kind);
    uint64_t h2d_bytes_ = 0, d2h_bytes_ = 0;
    bool in_full_frame_ = false;  // retrace_invalid: prune/fill/trace back to back
    bool in_sharded_frame_ = false;  // the counters of this read-back were summed over ranks

    struct LightBlock {
        const Light* light = nullptr;
        uint32_t begin = 0, end = 0;  // global path range
        uint32_t ndims = 0, dims[4] = {0, 0, 0, 0}, cells = 0;
        V3 flux_pp{0, 0, 0};
        double cos_half = 0.0;
        LightPose pose_prev, pose_now;
        bool moved = false;
        DevBuf dm_t, dm_c, unm, seg_start;
        DevBuf pref, tot;  // sharded prune: unmarked counts of the lower ranks / of all ranks
    };
    struct DynInfo {
        uint32_t obj = 0, tri_begin = 0, tri_count = 0, node_begin = kLbvhBrute, sah_root = kLbvhBrute;
        Xform last_xf;
        bool placed = false;
    };

    void upload_scene();
    void apply_l2_policy();
    void alloc_state();
    void fill_frame_params();
    void fill_frame_params_host();
    void frame_update_host();
    void frame_update_enqueue();
    void retrace_enqueue();
    bool place_dynamics_host(bool force);
    void place_dynamics_enqueue();
    struct FrameGraph;
    template <typename F>
    bool capture_graph(F&& enqueue, FrameGraph& out);
    void launch_graph(const FrameGraph& g);
    void place_frame(int frame);
    void place_dynamics(bool force);
    void stage_update_origins();
    void stage_occlusions();
    void stage_compute_dm();
    void stage_prune_local();
    void stage_fill_local();
    void prune_mark_all();
    void prune_trim_all(uint32_t* const* prefix_tab, uint32_t* const* total_tab, const uint32_t* const* total_host);
    void fill_collect_dead();
    void fill_assign_all(const uint64_t* prefix, const uint64_t* total, const uint64_t* prefix_dev = nullptr,
                         const uint64_t* total_dev = nullptr);
    // in-engine sharded frame (prx_collectives attached, world > 1)
    // a collectives table is attached: the exchanges run (world 1 included: identity exchanges,
    // which is how a one-GPU box exercises the NCCL backend end to end)
    bool sharded() const { return coll_.world >= 1; }
    void coll_ok(int rc, const char* what) const;
    void exchange_dm();
    void stage_prune_sharded();
    void stage_fill_sharded();
    void exchange_counters();
    void stage_trace();
    void read_back(prx_frame_stats* st, bool with_times);
    void splat_store(const PathDev& P, const prx_camera* cam, float radius, int mode, float* rgb_host,
                     float* rgb_dev, prx_frame_stats* st, bool reduce_ranks);
    void record(int idx);
    double elapsed_ms(int a, int b);
    SceneDev scene_dev() const;
    PathDev path_dev() const;
    uint32_t local_lb(const LightBlock& b) const;
    uint32_t local_le(const LightBlock& b) const;

    std::shared_ptr<const Scene> scene_;
    prx_config cfg_;
    int device_ = 0;
    cudaStream_t stream_ = nullptr;
    bool own_stream_ = true;
    uint32_t n_total_ = 0, sb_ = 0, se_ = 0, n_ = 0, B_ = 0;
    float eps_ = 0.0f, diag_ = 0.0f;
    uint64_t seed_mix_ = 0;
    int frames_run_ = 0;
    int cur_frame_ = 0;
    uint64_t launches_ = 0;
    uint64_t launch_base_ = 0;

    std::vector<LightBlock> lights_;
    std::vector<DynInfo> dyn_;
    uint32_t n_dyn_tris_ = 0, n_lbvh_nodes_ = 0;

    // scene device data
    DevBuf d_pow_tabs_, d_stris_, d_mat_, d_oflags_, d_dyn_local_, d_dyn_world_, d_dyn_xf_, d_dyn_tri_xf_,
        d_lbvh_nodes_, d_lbvh_leaf_, d_lbvh_work_, d_dall_nodes_, d_dall_tris_, d_dsah_;
    LbvhBuffers lbvh_{};
    // the traversal's hot static data in one arena (fast SAH nodes | their triangles |
    // leaf_of | reference nodes) so one L2 access-policy window can cover it (apply_l2_policy)
    DevBuf d_hot_;
    float4 *p_fnodes_ = nullptr, *p_ftris_ = nullptr, *p_nodes_ = nullptr;
    float4* p_dnodes_ = nullptr;  // the combined dynamic tree's nodes inside the arena (after fnodes)
    uint32_t dnode_off_ = 0;      // their index offset in fnodes (SceneDev::dnode_off)
    size_t dnode_cap_ = 0;        // room reserved for them (nodes)
    uint32_t* p_leaf_of_ = nullptr;
    size_t l2_window_ = 0;
    int32_t cert_off_ = 0;
    int32_t xt_force_ = 0;  // PRX_XT_FORCE=1: exact light transcendentals everywhere (tests)  // PRX_CERT_OFF=1: every query takes its exact fallback (tests)
    const float2* d_trig_ = nullptr;

    // frame params (pinned host + device)
    FrameParams* h_fp_ = nullptr;
    DevBuf d_fp_;
    float4* h_xf_ = nullptr;
    DevBuf d_light_ptrs_;  // uint32_t*[3][PRX_MAX_LIGHTS]: unm, seg_start, prefix

    // path state
    DevBuf d_pos_obj_, d_in_dir_, d_origin_, d_emis_, d_canon_, d_cell_,
        d_epoch_, d_path_info_, d_seg_flags_, d_meta_, d_rstart_;
    // work arrays
    DevBuf d_list_, d_masks_, d_flags8_, d_flags8b_, d_keys_, d_vals_, d_keys_tmp_, d_vals_tmp_,
        d_pruned_list_, d_need_, d_scratch_;
    DevBuf d_ctr_, d_cnt32_, d_work_;
    Counters* h_ctr_ = nullptr;
    uint32_t* h_cnt32_ = nullptr;
    uint32_t n_pruned_ = 0;
    prx_collectives coll_{};                        // world 0: no table attached
    DevBuf d_gath_, d_dead_g_, d_dead_pt_, d_ctr_sum_, d_cnt32_sum_;
    Counters* h_ctr_sum_ = nullptr;                 // pinned: the all-rank sums read back
    uint32_t* h_cnt32_sum_ = nullptr;
    uint32_t max_cells_ = 1;

    // splat buffers
    DevBuf d_gbuf_, d_img_, d_splat_work_, d_splat_cand_, d_gather_;
    uint32_t img_w_ = 0, img_h_ = 0;
    // the splat's photon-independent prefix (G-buffer + cell keys) for the scene camera at the
    // radius of the last scene-camera splat, run on a side stream during verify/retrace
    cudaStream_t side_stream_ = nullptr;
    cudaEvent_t ev_fork_ = nullptr, ev_join_ = nullptr;
    // overlapped splat: enqueued on the side stream, ev_splat_ marks its end; the next frame
    // waits for it before its first photon-map write and before its own prefix
    cudaEvent_t ev_splat_ = nullptr, ev_splat_read_ = nullptr;  // its end / its last photon-map read
    bool splat_overlap_ = false, splat_pending_ = false;
    // a host output of the overlapped splat: copied to pinned staging on the side stream, then
    // to the caller's buffer once the splat is known complete (finish_splat)
    float* h_img_stage_ = nullptr;
    size_t h_img_stage_bytes_ = 0;
    float* pending_host_out_ = nullptr;
    size_t pending_host_bytes_ = 0;
    void wait_splat(cudaStream_t s, bool whole);
    void finish_splat();
    DevBuf d_pre_gbuf_, d_pre_work_;
    float pre_radius_ = 0.0f;  // 0: no scene-camera splat yet, no prefix
    bool pre_ok_ = false;      // d_pre_* match the current placement of the scene
    bool pre_on_ = true;       // PRX_SPLAT_PREFIX=0: always compute the prefix in the splat
    uint32_t* h_ncell_ = nullptr;  // pinned: registered cells of the prefix [side stream, inline]
    int pre_bits_ = 0;             // the side-stream prefix's cell-table bits
    int splat_work_bits_ = 0;      // d_splat_work_ is sized for a table of this many bits
    int gather_bits_ = 0;          // d_gather_ is sized for a table of this many bits
    bool splat_prefix_fork();
    void splat_prefix_join();
    void drop_graphs();
    CamDev camera_dev(const Camera& c) const;

    cudaEvent_t ev_[12] = {};
    bool ev_recorded_[12] = {};

    // whole-frame CUDA graphs (run_frame), keyed by the frame's host decisions
    struct FrameGraph {
        cudaGraphExec_t exec = nullptr;
        uint64_t h2d = 0, d2h = 0, launches = 0;
        bool ev[12] = {};
    };
    std::map<uint32_t, FrameGraph> graphs_;
    uint32_t last_sig_ = ~0u;
    bool graphs_on_ = true, capturing_ = false, dyn_changed_ = false;
    cudaStream_t capture_stream_ = nullptr;
    uint32_t* h_prune_frame_ = nullptr;  // pinned: the frame number the prune marks are keyed by
    DevBuf d_prune_frame_;
};

// host-libm cos/sin table for cosine_sample's 2^24 possible angles (device copy, cached)
const float2* exact_trig_table(int device);

}  // namespace prx
