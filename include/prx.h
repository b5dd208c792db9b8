/*
 * prx.h -- C ABI of the B200-native photon-path verification and reuse engine.
 *
 * This is the drop-in boundary for the hot path of arXiv 2111.06906 as implemented by
 * the reference `pathreuse` C++ library (/root/reference/proj).  The reference exposes
 * no plugin/FFI layer; its public surface is the C++ `pathreuse::Engine`
 * and the pybind11 module `_pathreuse`.  Every entry point below replaces one of those
 * calls; the reference interface it replaces is cited beside it (paths relative to
 * /root/reference/proj).  Plain pointers and sizes only -- no C++ or torch types.
 *
 * Error behaviour mirrors the reference's exception types (SURVEY.md s8b "Errors"):
 * every fallible call returns a prx_status; the message of the last failure on the
 * calling thread is available from prx_last_error().  Language bindings map
 *   PRX_E_INVALID_ARGUMENT -> std::invalid_argument / ValueError
 *   PRX_E_OUT_OF_RANGE     -> std::out_of_range     / IndexError
 *   PRX_E_LOGIC            -> std::logic_error      / RuntimeError
 *   PRX_E_SCENE            -> pathreuse::SceneError / RuntimeError
 *   PRX_E_CUDA, PRX_E_RUNTIME -> std::runtime_error / RuntimeError
 */
#ifndef PRX_H_
#define PRX_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PRX_ABI_VERSION 1
#define PRX_MAX_LIGHTS 16

typedef enum prx_status {
    PRX_OK = 0,
    PRX_E_INVALID_ARGUMENT = 1,
    PRX_E_OUT_OF_RANGE = 2,
    PRX_E_LOGIC = 3,
    PRX_E_SCENE = 4,
    PRX_E_RUNTIME = 5,
    PRX_E_CUDA = 6
} prx_status;

/* ---- scene description (POD mirror of pathreuse::Scene, scene.hpp:16-60) ---------- */

typedef struct prx_vec3 { float x, y, z; } prx_vec3;
typedef struct prx_quat { float x, y, z, w; } prx_quat;            /* transform.hpp:10 */
typedef struct prx_triangle { prx_vec3 a, b, c; } prx_triangle;    /* geometry.hpp:61  */

typedef struct prx_keyframe {                                      /* scene.hpp:24, light.hpp:15 */
    int32_t frame;
    prx_quat rotation;
    prx_vec3 translation;
    float scale;
} prx_keyframe;

enum { PRX_MATERIAL_DIFFUSE = 0, PRX_MATERIAL_GLOSSY = 1 };        /* scene.hpp:16 */

typedef struct prx_material {                                      /* scene.hpp:18-22 */
    int32_t kind;
    prx_vec3 albedo;
    float glossy_exponent;
} prx_material;

typedef struct prx_object_desc {                                   /* scene.hpp:29-37 */
    const char* name;
    const prx_triangle* mesh;       /* object-local space */
    uint32_t n_triangles;
    prx_material material;
    const prx_keyframe* keyframes;  /* may be NULL/0: identity at frame 0 */
    uint32_t n_keyframes;
} prx_object_desc;

enum {                                                             /* light.hpp:13 */
    PRX_LIGHT_POINT = 0,
    PRX_LIGHT_SPOT = 1,
    PRX_LIGHT_DISC_AREA = 2,
    PRX_LIGHT_RECT_AREA = 3
};

typedef struct prx_light_desc {                                    /* light.hpp:24-37 */
    int32_t kind;
    prx_vec3 flux;
    float cone_angle_deg;
    float radius;
    float half_x, half_y;
    const prx_keyframe* keyframes;
    uint32_t n_keyframes;
} prx_light_desc;

typedef struct prx_camera {                                        /* scene.hpp:39-45 */
    prx_vec3 position;
    prx_vec3 look_at;
    float fov_deg;
    uint32_t width, height;
} prx_camera;

typedef struct prx_scene_desc {                                    /* scene.hpp:47-60 */
    const prx_object_desc* objects;
    uint32_t n_objects;
    const prx_light_desc* lights;
    uint32_t n_lights;
    prx_camera camera;
    int32_t frames;
} prx_scene_desc;

typedef struct prx_scene prx_scene;     /* finalized scene: validated, static BVH built */
typedef struct prx_engine prx_engine;   /* per-GPU engine over a path range           */

/* ---- engine configuration / statistics ------------------------------------------ */

enum { PRX_MODE_BASELINE = 0, PRX_MODE_NAIVE = 1, PRX_MODE_ERROR = 2 }; /* engine.hpp:14 */

typedef struct prx_config {                                        /* engine.hpp:43-53 */
    int32_t mode;
    uint32_t n_paths;
    uint32_t max_bounces;       /* 1..16 */
    uint32_t dm_dims[4];
    float threshold;
    uint64_t seed;
    float gather_radius;
    uint32_t workers;           /* accepted for API parity; the GPU ignores it */
    int32_t record_flags;
    /* B200 extensions (0 = defaults) */
    int32_t device;             /* CUDA device ordinal                              */
    uint32_t shard_begin;       /* path range owned by this engine; [0,0) = all     */
    uint32_t shard_end;
    int32_t exact_trig;         /* >= 0 (default): host-libm cosf/sinf table for bounces */
    int32_t dfs_traversal;      /* 1: reference-order DFS for every ray; 0 (default): near-
                                   first traversal + exactness certificate (same results) */
} prx_config;

typedef struct prx_frame_stats {                                   /* engine.hpp:19-30 */
    int32_t frame;
    int32_t mode;
    uint64_t rays_traced;
    uint64_t rays_reused;
    uint64_t paths_replaced;
    uint64_t paths_pruned;
    uint64_t paths_filled;
    uint64_t visibility_rays;
    double t_update, t_occlusion, t_dm, t_prune, t_fill, t_trace, t_gather;
    /* B200 extensions: device time (ms, CUDA events) of the named north_star stages */
    double ms_frame_update, ms_verify, ms_retrace, ms_splat;
    uint64_t live_segments_before;  /* segments verified this frame (paths live at entry) */
    uint64_t paths_retraced;        /* paths with retrace_start != 0xFF after verify    */
} prx_frame_stats;

typedef struct prx_engine_info {
    uint32_t n_paths;           /* total paths of the (unsharded) problem */
    uint32_t max_bounces;
    uint32_t n_lights;
    uint32_t shard_begin, shard_end;
    float eps_world;            /* engine.cpp:74 */
    float diagonal;
    int32_t frames_run;
    uint32_t n_pruned;          /* length of the last frame's pruned list */
    uint32_t light_path_begin[PRX_MAX_LIGHTS];
    uint32_t light_path_end[PRX_MAX_LIGHTS];
    uint32_t dm_ndims[PRX_MAX_LIGHTS];
    uint32_t dm_dims[PRX_MAX_LIGHTS][4];
    uint32_t dm_cells[PRX_MAX_LIGHTS];
    float flux_per_path[PRX_MAX_LIGHTS][3];
    uint64_t device_bytes;      /* device memory held by the engine */
} prx_engine_info;

/* State fields for prx_engine_download / prx_engine_upload.  Vertex fields are
 * bounce-major [max_bounces][n_paths] (photon_store.cpp:32-36); path fields are
 * [n_paths] (shard-local when sharded).                                          */
typedef enum prx_field {
    PRX_FIELD_PHOTONS = 0,     /* 32-byte pathreuse::Photon records (photon_store.hpp:13) */
    PRX_FIELD_AUX = 1,         /* 24-byte PathVertexAux records (photon_store.hpp:75)     */
    PRX_FIELD_POS_OBJ = 2,     /* float4 {position, object id bits}                       */
    PRX_FIELD_ENERGY = 3,      /* float4 {energy rgb, radius}                             */
    PRX_FIELD_IN_DIR = 4,      /* float4 {incoming dir, 0}                                */
    PRX_FIELD_OUT_DIR = 5,     /* float4 {outgoing dir, 0}                                */
    PRX_FIELD_ORIGIN = 6,      /* float4 per path                                         */
    PRX_FIELD_EMISSION_DIR = 7,/* float4 per path                                         */
    PRX_FIELD_CANONICAL = 8,   /* float4 per path (canonical coords c[0..3])              */
    PRX_FIELD_CELL = 9,        /* u32 per path                                            */
    PRX_FIELD_EPOCH = 10,      /* u32 per path                                            */
    PRX_FIELD_PATH_INFO = 11,  /* u32 per path (photon_store.hpp:23-40)                   */
    PRX_FIELD_META = 12,       /* u8x4 per path {photon_count, escaped, status, filled}   */
    PRX_FIELD_RETRACE_START = 13, /* u8 per path (0xFF = no retrace)                      */
    PRX_FIELD_SEGMENT_FLAGS = 14, /* u32 per path (record_flags)                          */
    PRX_FIELD_DM_TARGET = 15,  /* u32 [cells] of light `index`                            */
    PRX_FIELD_DM_CURRENT = 16, /* u32 [cells] of light `index`                            */
    PRX_FIELD_PRUNED = 17      /* u32 [n_pruned], ascending path ids                      */
} prx_field;

/* ---- pure functions (pybind module.cpp:47-82) ------------------------------------ */

/* select_paths_to_prune (engine.hpp:62-63, engine.cpp:443-471): the prune selection of one
 * DM cell (Eq. 1 Bernoulli marks keyed (path, frame, PruneMark), then the trim from the
 * highest path id down to exactly dm_t); `out` (capacity n) receives the pruned ids in
 * ascending order.  The engine itself selects on the GPU (k_prune_mark / k_prune_trim). */
prx_status prx_select_paths_to_prune(const uint32_t* cell_paths, size_t n, uint32_t dm_c, uint32_t dm_t,
                                     uint64_t seed, uint32_t frame, uint32_t* out, size_t* n_out);

/* light.hpp:132-135 */
double prx_prune_probability(uint32_t dm_current, uint32_t dm_target);
/* engine.hpp:34-41 */
int prx_energies_close(const float e_old[3], const float e_new[3], float threshold);
/* photon_store.cpp:9-20 (PRX_E_OUT_OF_RANGE on a field overflow) */
prx_status prx_encode_path_info(uint32_t cell, uint32_t seg_count, uint32_t retrace_start,
                                int replace, int reuse_light, uint32_t* word_out);
/* photon_store.cpp:22-30 */
void prx_decode_path_info(uint32_t word, uint32_t* cell, uint32_t* seg_count,
                          uint32_t* retrace_start, int* replace, int* reuse_light);
/* photon_store.cpp:38-54; out[7] = {path_info, origin_positions, distribution_maps,
 * pruned_array, photon_map, subtotal_reuse, total} in MiB */
void prx_memory_footprint(uint64_t n_paths, uint32_t max_bounces, const uint32_t* dm_dims,
                          uint32_t n_dims, int area_light, double out[7]);

/* ---- scenes ----------------------------------------------------------------------- */

/* finalize_scene (scene.cpp:63-113): validates, assigns dense ids, builds the static BVH. */
prx_status prx_scene_create(const prx_scene_desc* desc, prx_scene** out);
/* make_builtin_scene (scene.cpp:603-611); names as in builtin_scenes() (module.cpp:57-61). */
prx_status prx_scene_builtin(const char* name, prx_scene** out);
/* Scene documents, scene.cpp:272-398 (load_scene_text / load_scene / load_scene_source):
 * JSON with inline meshes or OBJ files (relative to the document's directory);
 * `source` is "builtin:NAME", a builtin name, or a path.  PRX_E_SCENE on bad input. */
prx_status prx_scene_load(const char* source, prx_scene** out);
prx_status prx_scene_load_text(const char* json_text, const char* base_dir, prx_scene** out);
/* Procedural BASELINE configurations: "C1".."C5" plus parameters
 * (0 = default): C5 uses n_dynamic objects; tri_scale scales static tessellation.   */
prx_status prx_scene_synthetic(const char* name, uint32_t n_dynamic, float tri_scale,
                               prx_scene** out);
/* Borrowed view of the finalized scene's description (valid until destroy). */
prx_status prx_scene_describe(const prx_scene* scene, prx_scene_desc* out);
/* Static BVH permutation (Bvh::permutation, bvh.hpp:36) -- parity harness. */
prx_status prx_scene_bvh_permutation(const prx_scene* scene, uint32_t* out, size_t capacity,
                                     size_t* count);
/* counts: {static triangles, dynamic triangles, bvh nodes, objects} */
prx_status prx_scene_counts(const prx_scene* scene, uint64_t counts[4]);
float prx_scene_diagonal(const prx_scene* scene);
/* state_at (scene.cpp:115-134) on the host: every dynamic object placed at `frame` --
 * world-space triangles (transform_triangle) and bounds_current / bounds_previous -- for
 * Engine::scene_state() of the C++ drop-in.  Pass NULL buffers to query the counts. */
typedef struct prx_placed_dynamic {
    uint32_t object_id;
    uint32_t tri_begin;   /* first triangle of this object in the `tris` array */
    uint32_t tri_count;
    uint32_t reserved;
    prx_vec3 cur_lo, cur_hi, prev_lo, prev_hi;
} prx_placed_dynamic;
prx_status prx_scene_state_at(const prx_scene* scene, int32_t frame, prx_placed_dynamic* dyn,
                              size_t dyn_capacity, size_t* n_dyn, prx_triangle* tris,
                              size_t tri_capacity, size_t* n_tris);
void prx_scene_destroy(prx_scene* scene);

/* ---- engine (engine.hpp:69-179) --------------------------------------------------- */

/* Engine::Engine(Scene, EngineConfig) -- engine.cpp:63-117 */
prx_status prx_engine_create(const prx_scene* scene, const prx_config* cfg, prx_engine** out);
void prx_engine_destroy(prx_engine* engine);
prx_status prx_engine_get_info(const prx_engine* engine, prx_engine_info* out);

/* Engine::run_frame() -- engine.cpp:201-242.  Equivalent to frame_update, verify_paths,
 * retrace_invalid in order; synchronous, fills stats on return. */
prx_status prx_run_frame(prx_engine* engine, prx_frame_stats* stats);

/* north_star stage split of run_frame (SURVEY.md s8b "New named entry points"):
 *   frame_update   = state_at + run_frame prelude (scene.cpp:115-134, engine.cpp:202-226)
 *   verify_paths   = stage_update_origins + stage_occlusions + stage_compute_dm
 *   retrace_invalid= stage_prune + stage_fill + stage_trace
 * Stats accumulate into the struct passed to each call (zero it before frame_update). */
prx_status prx_frame_update(prx_engine* engine, prx_frame_stats* stats);
prx_status prx_verify_paths(prx_engine* engine, prx_frame_stats* stats);
prx_status prx_retrace_invalid(prx_engine* engine, prx_frame_stats* stats);

/* Sub-stages of the above for multi-GPU orchestration and stage-level parity tests.
 * stage ids: */
typedef enum prx_stage {
    PRX_STAGE_UPDATE_ORIGINS = 0,   /* engine.cpp:244-304 */
    PRX_STAGE_OCCLUSIONS = 1,       /* engine.cpp:306-337 */
    PRX_STAGE_COMPUTE_DM = 2,       /* engine.cpp:405-441 (local histogram only)      */
    PRX_STAGE_PRUNE = 3,            /* engine.cpp:473-497 (single shard)              */
    PRX_STAGE_FILL = 4,             /* engine.cpp:499-546 (single shard)              */
    PRX_STAGE_TRACE = 5,            /* engine.cpp:548-598 (+ refresh_path_info)       */
    PRX_STAGE_RELEASE_ALL = 6       /* baseline prelude engine.cpp:228-232            */
} prx_stage;
prx_status prx_run_stage(prx_engine* engine, int stage, prx_frame_stats* stats);

/* Sharded prune/fill exchange points.  Per-light arrays are indexed by
 * light; every `*_dev` buffer is a DEVICE pointer on the engine's device, ordered on the
 * engine stream.  A sharded frame is:
 *   frame_update; verify_paths (local DM_C histogram);
 *   all-reduce(sum) DM_C of every light (prx_engine_dm_current gives its address);
 *   prx_prune_count -> per-cell unmarked counts of this shard; all-gather them; pass the
 *     exclusive prefix over lower shards and the total over all shards to prx_prune_apply
 *     (survivors are the dm_t lowest path ids of a cell, engine.cpp:459-466);
 *   prx_fill_count -> dead slots of this shard per light (host); all-gather; pass the
 *     exclusive prefix and the total to prx_fill_apply (deficit cells ascending <-> dead
 *     slots ascending over the whole path range, engine.cpp:503-519);
 *   prx_run_stage(PRX_STAGE_TRACE); all-reduce the counters.
 * With one shard, prefix = 0 and total = local reproduce run_frame exactly. */
prx_status prx_engine_dm_current(prx_engine* engine, uint32_t light, void** dev_ptr,
                                 uint32_t* cells);
prx_status prx_prune_count(prx_engine* engine, uint32_t* const* unmarked_dev);
prx_status prx_prune_apply(prx_engine* engine, const uint32_t* const* prefix_dev,
                           const uint32_t* const* total_dev, prx_frame_stats* stats);
prx_status prx_fill_count(prx_engine* engine, uint32_t* dead_out);
prx_status prx_fill_apply(prx_engine* engine, const uint64_t* dead_prefix,
                          const uint64_t* dead_total, prx_frame_stats* stats);
/* Stream the engine orders its work on (cudaStream_t as void*); NULL = engine-owned. */
/* ---- in-engine multi-GPU ------------------------------------------
 * A path-sharded engine (prx_config.shard_begin/end = rank r's contiguous path range, ranks
 * in ascending path order) with a collectives table attached runs the whole sharded frame
 * itself: prx_run_frame enqueues the DM_C all-reduce, the per-cell unmarked-count and
 * dead-slot all-gathers (prefix over lower ranks + totals, computed on the device), and the
 * counter all-reduce on its stream between its kernels, with one host read-back per frame,
 * and prx_splat all-reduces the image.  Every rank calls the same entry points in the same
 * order (collective semantics).  Tables come from prx_comm_* (NCCL, or the in-process local
 * backend for several engines driven by several host threads) or from the caller. */
typedef struct prx_collectives {
    void* ctx;
    int32_t rank, world;
    /* each returns 0 on success; enqueued on `stream` (a cudaStream_t); sums in place */
    int (*all_reduce_sum_u32)(void* ctx, uint32_t* buf, size_t count, void* stream);
    int (*all_reduce_sum_u64)(void* ctx, uint64_t* buf, size_t count, void* stream);
    int (*all_reduce_sum_f32)(void* ctx, float* buf, size_t count, void* stream);
    /* recv[r * count + i] = rank r's send[i] */
    int (*all_gather_u32)(void* ctx, const uint32_t* send, uint32_t* recv, size_t count, void* stream);
} prx_collectives;
/* attach (copied) / detach (NULL); world 1 behaves as an unsharded engine */
prx_status prx_engine_set_collectives(prx_engine* engine, const prx_collectives* coll);

/* One process over several GPUs (several shards may share a device): `n_devices` engines on
 * contiguous path shards of cfg->n_paths, attached to in-process local collectives, driven
 * by one persistent host thread each.  prx_group_run_frame runs every shard's frame
 * concurrently (stats: the all-shard counters); prx_group_splat returns the summed image;
 * prx_group_engine gives a shard's engine (owned by the group) for downloads. */
typedef struct prx_group prx_group;
prx_status prx_group_create(const prx_scene* scene, const prx_config* cfg, const int32_t* devices,
                            int32_t n_devices, prx_group** out);
prx_status prx_group_run_frame(prx_group* group, prx_frame_stats* stats);
prx_status prx_group_splat(prx_group* group, const prx_camera* camera, float radius, int mode,
                           float* rgb_out);
prx_engine* prx_group_engine(prx_group* group, int32_t rank);
int32_t prx_group_size(const prx_group* group);
void prx_group_destroy(prx_group* group);

typedef struct prx_comm prx_comm;
/* NCCL (loaded at run time, PRX_NCCL_LIB overrides "libnccl.so.2"): rank 0 makes the id,
 * the caller ships it to the other ranks, every rank creates its communicator */
prx_status prx_comm_nccl_unique_id(uint8_t id_out[128]);
prx_status prx_comm_nccl_create(const uint8_t id[128], int32_t rank, int32_t world, int32_t device,
                                prx_comm** out);
/* in-process: `world` communicators (comms_out[world]), each used by one host thread */
prx_status prx_comm_local_create(int32_t world, prx_comm** comms_out);
prx_status prx_comm_collectives(prx_comm* comm, prx_collectives* out);
void prx_comm_destroy(prx_comm* comm);

prx_status prx_engine_set_stream(prx_engine* engine, void* cuda_stream);
prx_status prx_engine_synchronize(prx_engine* engine);
/* Overlapped splat (no reference counterpart; default off).  When on, a prx_splat of the scene
 * camera at the frame's prefix radius with a device output only (rgb_out NULL, stats NULL,
 * unsharded) is enqueued on the engine's side stream and returns at once: it runs while the
 * next prx_run_frame updates the scene and computes the occlusion flags, and that frame waits
 * for it before its first write to the photon map.  rgb_dev is complete after the next
 * engine call that touches engine state, or after prx_engine_synchronize. */
prx_status prx_engine_set_splat_overlap(prx_engine* engine, int32_t on);

/* gather_image (gather.cpp:35-75) as a GPU splat over the engine's live photons.
 * rgb_out: host float[3*w*h] (may be NULL) -- top-left origin, RGB rows;
 * rgb_dev: optional device float[3*w*h] written on the engine stream.
 * mode: 0 = tiled shared-memory atomic splat, 1 = ordered gather (bit-exact vs the
 * reference's 27-cell insertion order). */
prx_status prx_splat(prx_engine* engine, const prx_camera* camera, float radius, int mode,
                     float* rgb_out, float* rgb_dev, prx_frame_stats* stats);
/* gather_image(state, photons, aux, camera, radius, workers) (gather.hpp:81-83) over a HOST
 * photon map that need not be the engine's own: the records (32-byte Photon + 24-byte
 * PathVertexAux, [max_bounces][n_paths]) are uploaded to engine scratch and splatted against
 * the scene placed at frame `frame` (the engine's state is not modified).  mode as prx_splat. */
prx_status prx_gather_photons(prx_engine* engine, const void* photons, const void* aux, uint32_t n_paths,
                              uint32_t max_bounces, int32_t frame, const prx_camera* camera, float radius,
                              int mode, float* rgb_out);

/* Lazy host mirrors for the introspection accessors (engine.hpp:76-122) and the
 * state-injection parity harness.  `index` selects the light for DM fields.
 * bytes must equal the field size (prx_field_bytes). */
size_t prx_field_bytes(const prx_engine* engine, int field, uint32_t index);
prx_status prx_engine_download(prx_engine* engine, int field, uint32_t index, void* dst,
                               size_t bytes);
prx_status prx_engine_upload(prx_engine* engine, int field, uint32_t index, const void* src,
                             size_t bytes);
/* Sets frames_run and the previous light poses as if frame (frames_run-1) had run --
 * used after uploading a full state captured from another implementation. */
prx_status prx_engine_set_frame_counter(prx_engine* engine, int32_t frames_run);

/* intersect_scene / occluded (scene.cpp:136-177) on the engine's current frame state (the
 * static BVH + the dynamic objects as placed by the last frame_update), as one GPU batch.
 * rays: n x 8 floats {origin xyz, dir xyz (unit), t_min, t_max}.  any_hit == 0: hits n x 9
 * floats {t, object id (u32 bits, 0xFFFFFFFF = miss), Hit::triangle (u32 bits), position
 * xyz, normal xyz}; any_hit != 0: hits n floats, 1 = occluded.  Host buffers. */
prx_status prx_intersect_batch(prx_engine* engine, const float* rays, size_t n, int any_hit, float* hits);

/* ---- offline artefacts (byte-compatible with the reference's files) ---- */
/* PHM1 photon dump, photon_store.cpp:55-102: "PHM1", u32 n_paths, u32 max_bounces, u32 0,
 * then n_paths*max_bounces 32-byte Photon records in b*N+p order.  PRX_E_RUNTIME on I/O
 * errors.  _read with records == NULL only reports the sizes. */
prx_status prx_photon_dump_write(const char* path, uint32_t n_paths, uint32_t max_bounces,
                                 const void* records, size_t bytes);
prx_status prx_photon_dump_read(const char* path, uint32_t* n_paths, uint32_t* max_bounces,
                                void* records, size_t capacity);
/* write_photon_dump(engine.photon_map(), path) of an unsharded engine */
prx_status prx_engine_write_photon_dump(prx_engine* engine, const char* path);
/* write_image, gather.cpp:77-92 (P6, gamma 1/2.2, lround) and frame_image_name :94-98;
 * the latter returns the name length and writes a NUL-terminated copy into buf. */
prx_status prx_image_write_ppm(const char* path, const float* rgb, uint32_t width, uint32_t height);
size_t prx_frame_image_name(int32_t frame, char* buf, size_t capacity);
/* stats.cpp:10-70 (write_stats_csv / read_stats_csv) and :72-107 (reuse_report).  Only
 * frame, mode, the six counters and the t_* fields are written / read. */
prx_status prx_stats_csv_write(const char* path, const prx_frame_stats* rows, size_t n);
prx_status prx_stats_csv_read(const char* path, prx_frame_stats* rows, size_t capacity, size_t* n_out);
prx_status prx_reuse_report(const prx_frame_stats* rows, size_t n, char* buf, size_t capacity,
                            size_t* len_out);

/* Number of kernel launches issued by this engine since creation (bench evidence). */
uint64_t prx_engine_launch_count(const prx_engine* engine);

/* Bytes this engine copied host->device and device->host since creation (every frame,
 * splat and field transfer is counted; scene upload at creation is included). */
prx_status prx_engine_transfer_bytes(const prx_engine* engine, uint64_t* h2d, uint64_t* d2h);

const char* prx_last_error(void);
int prx_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PRX_H_ */
