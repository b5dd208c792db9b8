/*
 * ORACLE / TEST INFRASTRUCTURE ONLY -- never linked into or called by the product.
 *
 * pathreuse_oracle: a plain-C, single-threaded restatement of the reference's hot path
 * (/root/reference/proj: scene.cpp, bvh.cpp, light.cpp, engine.cpp, gather.cpp) used by
 * tests/ as an independent checker.  State is held in the product's C-ABI field layouts
 * (include/prx.h: prx_field) so any stage can be fed exactly the state the GPU engine saw.
 * Pinned against the compiled reference (oracle/_ref) by tests/test_oracle.py:
 * builtin/synthetic scenes, BVH permutations, per-frame counters and full state.
 */
#ifndef PATHREUSE_ORACLE_H_
#define PATHREUSE_ORACLE_H_

#include <stddef.h>
#include <stdint.h>

#include "../include/prx.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct po_scene po_scene;
typedef struct po_engine po_engine;

const char* po_last_error(void);

double po_prune_probability(uint32_t dm_c, uint32_t dm_t);
int po_energies_close(const float e_old[3], const float e_new[3], float threshold);
int po_encode_path_info(uint32_t cell, uint32_t seg_count, uint32_t retrace_start, int replace,
                        int reuse_light, uint32_t* word);
void po_decode_path_info(uint32_t word, uint32_t out[5]);
void po_memory_footprint(uint64_t n_paths, uint32_t max_bounces, const uint32_t* dims, uint32_t n_dims,
                         int area_light, double out[7]);
int po_select_paths_to_prune(const uint32_t* paths, size_t n, uint32_t dm_c, uint32_t dm_t, uint64_t seed,
                             uint32_t frame, uint32_t* out, size_t* count);

int po_scene_create(const prx_scene_desc* desc, po_scene** out);
void po_scene_destroy(po_scene* s);
float po_scene_diagonal(const po_scene* s);
int po_scene_bvh_permutation(const po_scene* s, uint32_t* out, size_t cap, size_t* count);

int po_engine_create(const po_scene* s, const prx_config* cfg, po_engine** out);
void po_engine_destroy(po_engine* e);
int po_run_frame(po_engine* e, prx_frame_stats* st);
int po_frame_update(po_engine* e, prx_frame_stats* st);
int po_run_stage(po_engine* e, int stage, prx_frame_stats* st);
size_t po_field_bytes(const po_engine* e, int field, uint32_t index);
int po_download(const po_engine* e, int field, uint32_t index, void* dst, size_t bytes);
int po_upload(po_engine* e, int field, uint32_t index, const void* src, size_t bytes);
int po_set_frame_counter(po_engine* e, int frames_run);
int po_gather(po_engine* e, const prx_camera* cam, float radius, float* rgb_out);
/* sharded prune/fill exchange points (cfg.shard_begin/end select the shard) */
int po_prune_count(po_engine* e, uint32_t** unmarked);
int po_prune_apply(po_engine* e, const uint32_t** prefix, const uint32_t** total, prx_frame_stats* st);
int po_fill_count(po_engine* e, uint32_t* dead);
int po_fill_apply(po_engine* e, const uint64_t* prefix, const uint64_t* total, prx_frame_stats* st);
/* closest hit at `frame`: rays [n][8] {o, d, t_min, t_max} -> hits [n][9] as prxref_intersect_batch */
int po_intersect_batch(const po_scene* s, int frame, const float* rays, size_t n, float* hits);

#ifdef __cplusplus
}
#endif
#endif
