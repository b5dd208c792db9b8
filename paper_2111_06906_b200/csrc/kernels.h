// kernels.h -- host-callable launchers of the engine's stage kernels (kernels.cu,
// lbvh.cu, splat.cu).  Each launcher cites the reference function its kernel replaces.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

#include "dev_types.h"

namespace prx {

int launch_grid(uint64_t n, int threads);
extern std::atomic<uint64_t> g_launches;  // kernels launched by this library (bench evidence, all engines of the process)

// dm_t histogram of init_dm_target (light.cpp:230-252)
void launch_init_dm_target(const LightDev* light_host, uint32_t n_samples, uint64_t seed_mix,
                           uint32_t* dm_t, cudaStream_t st);
// per-dynamic-triangle placement: transform_triangle (transform.hpp:98-100) for the frame
void launch_transform_dynamic(const float4* local_tris, const uint32_t* tri_xf, const float4* xf,
                              uint32_t n_tris, float4* world_tris, cudaStream_t st);
// run_frame prelude resets (engine.cpp:223-226) + live-segment count
void launch_frame_reset(PathDev P, int record_flags, Counters* ctr, cudaStream_t st);
// release_all_paths (engine.cpp:149-157)
void launch_release_all(PathDev P, cudaStream_t st);
// stage_update_origins (engine.cpp:244-304)
void launch_update_origins(SceneDev S, PathDev P, Counters* ctr, cudaStream_t st);
// stage_occlusions naive / flag pass (engine.cpp:306-337 + compute_flag_mask :172-199)
void launch_occlusion_flags(SceneDev S, PathDev P, int mode, int record, uint32_t* list,
                            uint32_t* masks, Counters* ctr, cudaStream_t st);
// verify_path_error_based (engine.cpp:339-403) over the flagged list
void launch_verify_error(SceneDev S, PathDev P, float threshold, const uint32_t* list,
                         const uint32_t* masks, const Counters* ctr_count, uint32_t* work,
                         Counters* ctr, cudaStream_t st);
// stage_compute_dm (engine.cpp:405-441)
void launch_compute_dm(SceneDev S, PathDev P, Counters* ctr, cudaStream_t st);
// stage_prune (engine.cpp:443-497): marks + per-cell unmarked counts
void launch_prune_mark(SceneDev S, PathDev P, const uint32_t* frame, uint32_t* const* unmarked,
                       uint8_t* pruned, uint8_t* cand, cudaStream_t st);
void launch_prune_trim_flags(PathDev P, const FrameParams* fp, uint32_t* const* unm_total,
                             const uint8_t* cand, uint8_t* trim, cudaStream_t st);
void launch_prune_keys(PathDev P, const FrameParams* fp, const uint32_t* list, const uint32_t* count,
                       uint32_t* keys, uint32_t* vals, uint32_t n_max, cudaStream_t st);
void launch_prune_trim(PathDev P, const FrameParams* fp, const uint32_t* keys, const uint32_t* vals,
                       const uint32_t* count, uint32_t n_max, uint32_t* const* seg_start,
                       uint32_t* const* prefix, uint8_t* pruned, cudaStream_t st);
void launch_prune_apply(PathDev P, const uint8_t* pruned, int clear_records, cudaStream_t st);
void launch_dm_after_prune(uint32_t* dm_c, const uint32_t* dm_t, const uint32_t* unm_total,
                           uint32_t cells, cudaStream_t st);
// stage_fill (engine.cpp:499-546)
void launch_fill_need(const uint32_t* dm_t, const uint32_t* dm_c, uint32_t* need, uint32_t cells,
                      cudaStream_t st);
void launch_dead_flags(PathDev P, uint32_t lb, uint32_t le, uint8_t* flags, cudaStream_t st);
// the dead-slot rank offset of this shard: dead_prefix_dev[light] when non-null, else dead_prefix
void launch_fill_assign(SceneDev S, PathDev P, uint32_t light, const uint32_t* dead,
                        const uint32_t* dead_count, uint32_t n_max, uint64_t dead_prefix,
                        const uint64_t* dead_prefix_dev, const uint32_t* need_off,
                        const uint32_t* need_total, uint32_t cells, Counters* ctr, cudaStream_t st);
void launch_fill_check(const uint32_t* dead_count, uint64_t dead_total, const uint64_t* dead_total_dev,
                       uint32_t light, const uint32_t* need_total, Counters* ctr, cudaStream_t st);
// sharded exchange: prefix over lower ranks / total over all ranks of gathered counts
void launch_rank_prefix_u32(const uint32_t* gathered, uint32_t n, uint32_t world, uint32_t rank,
                            uint32_t* prefix, uint32_t* total, cudaStream_t st);
void launch_rank_prefix_u64(const uint32_t* gathered, uint32_t n, uint32_t world, uint32_t rank,
                            uint64_t* prefix, uint64_t* total, cudaStream_t st);
void launch_dm_after_fill(uint32_t* dm_c, const uint32_t* dm_t, uint32_t cells, cudaStream_t st);
// stage_trace (engine.cpp:548-598)
// verify-walk queue order: keys of the flagged list (cnt->flagged entries, copied to *n32) and
// the permutation of list / masks by the sorted slots
void launch_walk_keys(const uint32_t* masks, const Counters* cnt, uint32_t* n32, uint32_t top, int how,
                      uint32_t n_max, uint32_t* keys, uint32_t* vals, cudaStream_t st);
void launch_walk_permute(const uint32_t* list, const uint32_t* masks, const uint32_t* order, const uint32_t* n32,
                         uint32_t n_max, uint32_t* list2, uint32_t* masks2, cudaStream_t st);
// flags[i] = path i is retraced; with start_of, start_of[i] = its retrace start (flagged i only)
void launch_retrace_flags(PathDev P, uint8_t* flags, uint32_t* start_of, cudaStream_t st);
void launch_trace(SceneDev S, PathDev P, const uint32_t* list, const uint32_t* count,
                  uint32_t* work, Counters* ctr, cudaStream_t st);
void launch_finalize(PathDev P, Counters* ctr, cudaStream_t st);
// intersect_scene / occluded for a ray batch (scene.cpp:136-177)
void launch_intersect_batch(SceneDev S, const float* rays, uint32_t n, int any_hit, float* out, cudaStream_t st);
// layout conversion for drop-in accessors
void launch_pack_photons(PathDev P, void* photons, void* aux, cudaStream_t st);
void launch_unpack_photons(PathDev P, const void* photons, const void* aux, cudaStream_t st);

// G-buffer + splat + resolve (splat.cu), replacing gather_image (gather.cpp:35-75)
int splat_table_bits(uint32_t npx);         // worst-case cell-table bits (27 cells per pixel)
int splat_table_bits_capped(uint32_t npx);  // the first try: at most 2^22 slots
bool splat_table_overflow(uint32_t n_cells, int bits);  // load above 3/4: rebuild at full size
size_t splat_work_bytes(int bits);
size_t gather_work_bytes(uint64_t n_vertices, uint32_t npx, int bits);
size_t splat_ncell_offset(int bits);       // byte offset of the registered-cell count in `work`
int splat_cell_bits(uint32_t n_cells);     // key bits of n_cells dense cell ids
// mode 0: tiled shared-memory atomic splat; mode 1: ordered gather (bit-exact vs gather_image)
// `bits`: the cell table's size; prefix_done: the G-buffer, the cell-key table and the dense
// cell ids (launch_splat_prefix) are already in gbuf/work; cell_bits > 0: the dense ids fit
// that many bits (else the table's)
void launch_splat(SceneDev S, PathDev P, const CamDev& C, float radius, float4* gbuf, float* img,
                  float inv_pi, float inv_area, void* work, void* cand_buf, int mode, void* gather_buf, int bits,
                  bool prefix_done, int cell_bits, cudaStream_t st, cudaEvent_t photons_read = nullptr);
void launch_splat_prefix(SceneDev S, const CamDev& C, float radius, float4* gbuf, void* work, int bits,
                         cudaStream_t st);

// Dynamic LBVH (lbvh.cu)
struct LbvhBuffers {
    uint32_t* keys;
    uint32_t* vals;
    uint32_t* keys_tmp;
    uint32_t* vals_tmp;
    uint32_t* parent;     // per node/leaf parent index
    uint32_t* flags;      // refit arrival counters
    void* scratch;
    float4* all_nodes;    // combined tree over all dynamic triangles (null: not built)
    float4* all_tris;     // its leaves: dynamic triangles in sorted order
    // fixed-topology variant of the combined tree (fast_bvh.h: DynSahTopology), refit only;
    // null sah_perm: rebuild it as a Karras tree every frame
    const uint32_t* sah_perm;    // leaf slot -> global dynamic triangle
    const uint4* sah_leaf;       // {first slot, count, parent, side}
    const uint32_t* sah_parent;  // per internal node: parent << 1 | side
    uint32_t n_sah_leaves, n_sah_nodes;
    uint32_t code_off;           // added to the combined tree's internal child codes (SceneDev::dnode_off)
};
void build_dynamic_lbvh(const float4* world_tris, const uint32_t* tri_obj, uint32_t n_tris,
                        const DynObj* dyn_host, uint32_t n_dyn, const DynObj* dyn_dev,
                        float4* nodes, uint32_t* leaf, const LbvhBuffers& buf, cudaStream_t st);

}  // namespace prx
