// capi.cpp -- the extern "C" boundary declared in include/prx.h.
//
// Every entry point catches the C++ exception its reference counterpart would throw and
// returns the matching prx_status (SURVEY.md s8b "Errors"); prx_last_error() returns the
// message on the calling thread.
#include <algorithm>
#include <cstring>
#include <memory>
#include <string>

#include "comm.h"
#include "engine.h"
#include "group.h"
#include "host_scene.h"
#include "prx.h"
#include "wire.h"

struct prx_scene {
    std::shared_ptr<prx::Scene> scene;
};

struct prx_engine {
    std::unique_ptr<prx::Engine> engine;
};

namespace {

thread_local std::string g_error;

prx_status fail(const std::exception& e) {
    g_error = e.what();
    if (dynamic_cast<const prx::SceneError*>(&e)) return PRX_E_SCENE;
    if (dynamic_cast<const prx::CudaError*>(&e)) return PRX_E_CUDA;
    if (dynamic_cast<const std::invalid_argument*>(&e)) return PRX_E_INVALID_ARGUMENT;
    if (dynamic_cast<const std::out_of_range*>(&e)) return PRX_E_OUT_OF_RANGE;
    if (dynamic_cast<const std::logic_error*>(&e)) return PRX_E_LOGIC;
    return PRX_E_RUNTIME;
}

template <typename F>
prx_status guarded(F&& f) {
    try {
        f();
        return PRX_OK;
    } catch (const std::exception& e) {
        return fail(e);
    } catch (...) {
        g_error = "unknown error";
        return PRX_E_RUNTIME;
    }
}

void need(const void* p, const char* what) {
    if (!p) throw std::invalid_argument(std::string(what) + " is NULL");
}

// (every entry but run_frame / splat first orders the engine stream after an overlapped splat)
prx::Engine& eng_raw(prx_engine* e) {
    need(e, "engine");
    return *e->engine;
}
prx::Engine& eng(prx_engine* e) {
    prx::Engine& E = eng_raw(e);
    E.join_splat();
    return E;
}

}  // namespace

extern "C" {

const char* prx_last_error(void) { return g_error.c_str(); }
int prx_abi_version(void) { return PRX_ABI_VERSION; }

// select_paths_to_prune (engine.cpp:443-471), host restatement for the C++ drop-in
prx_status prx_select_paths_to_prune(const uint32_t* cell_paths, size_t n, uint32_t dm_c, uint32_t dm_t,
                                     uint64_t seed, uint32_t frame, uint32_t* out, size_t* n_out) {
    return guarded([&] {
        if (n && (!cell_paths || !out)) throw std::invalid_argument("select_paths_to_prune: NULL buffer");
        need(n_out, "n_out");
        std::vector<uint32_t> sorted(cell_paths, cell_paths + n);
        std::sort(sorted.begin(), sorted.end());
        const double prob = prx::prune_probability(dm_c, dm_t);
        const uint64_t mix = prx::mix64(seed);
        std::vector<uint8_t> marks(n, 0);
        uint32_t survivors = 0;
        for (size_t i = 0; i < n; ++i) {
            const float u = prx::rng_uniform_m(mix, sorted[i], frame, 0, prx::kPruneMark, 0);
            if (prob > 0.0 && u < prob) marks[i] = 1;
            else ++survivors;
        }
        for (size_t i = n; survivors > dm_t && i-- > 0;)  // trim from the top path id down
            if (!marks[i]) {
                marks[i] = 1;
                --survivors;
            }
        size_t k = 0;
        for (size_t i = 0; i < n; ++i)
            if (marks[i]) out[k++] = sorted[i];
        *n_out = k;
    });
}

// state_at (scene.cpp:115-134): dynamic objects placed at `frame`, on the host
prx_status prx_scene_state_at(const prx_scene* scene, int32_t frame, prx_placed_dynamic* dyn,
                              size_t dyn_capacity, size_t* n_dyn, prx_triangle* tris, size_t tri_capacity,
                              size_t* n_tris) {
    return guarded([&] {
        need(scene, "scene");
        const prx::Scene& s = *scene->scene;
        size_t nd = 0, nt = 0;
        for (const prx::Object& o : s.objects) {
            if (!o.dynamic) continue;
            if (dyn && nd < dyn_capacity) {
                const prx::Xform now = prx::transform_at(o.kfs, frame);
                const prx::Xform prev = prx::transform_at(o.kfs, frame > 0 ? frame - 1 : 0);
                const prx::Box cur = prx::transform_box(o.local_bounds, now);
                const prx::Box prv = prx::transform_box(o.local_bounds, prev);
                prx_placed_dynamic& d = dyn[nd];
                d.object_id = o.id;
                d.tri_begin = static_cast<uint32_t>(nt);
                d.tri_count = static_cast<uint32_t>(o.mesh.size());
                d.reserved = 0;
                d.cur_lo = {cur.lo.x, cur.lo.y, cur.lo.z};
                d.cur_hi = {cur.hi.x, cur.hi.y, cur.hi.z};
                d.prev_lo = {prv.lo.x, prv.lo.y, prv.lo.z};
                d.prev_hi = {prv.hi.x, prv.hi.y, prv.hi.z};
                if (tris && nt + o.mesh.size() <= tri_capacity)
                    for (size_t t = 0; t < o.mesh.size(); ++t) {
                        const prx::Tri& m = o.mesh[t];
                        const prx::V3 a = prx::apply_point(now, m.a), b = prx::apply_point(now, m.b),
                                      c = prx::apply_point(now, m.c);
                        tris[nt + t] = {{a.x, a.y, a.z}, {b.x, b.y, b.z}, {c.x, c.y, c.z}};
                    }
            }
            ++nd;
            nt += o.mesh.size();
        }
        if (n_dyn) *n_dyn = nd;
        if (n_tris) *n_tris = nt;
    });
}

double prx_prune_probability(uint32_t dm_current, uint32_t dm_target) {
    return prx::prune_probability(dm_current, dm_target);
}

int prx_energies_close(const float e_old[3], const float e_new[3], float threshold) {
    return prx::energies_close(prx::V3{e_old[0], e_old[1], e_old[2]}, prx::V3{e_new[0], e_new[1], e_new[2]},
                               threshold)
               ? 1
               : 0;
}

// photon_store.cpp:9-20
prx_status prx_encode_path_info(uint32_t cell, uint32_t seg_count, uint32_t retrace_start, int replace,
                                int reuse_light, uint32_t* word_out) {
    return guarded([&] {
        need(word_out, "word_out");
        if (cell >= (1u << 22)) throw std::out_of_range("path info: cell id needs 22 bits");
        if (seg_count < 1 || seg_count > 16) throw std::out_of_range("path info: segment count must be in 1..16");
        if (retrace_start > 15) throw std::out_of_range("path info: retrace start must be in 0..15");
        *word_out = prx::pack_path_info(cell, seg_count, retrace_start, replace != 0, reuse_light != 0);
    });
}

void prx_decode_path_info(uint32_t word, uint32_t* cell, uint32_t* seg_count, uint32_t* retrace_start,
                          int* replace, int* reuse_light) {
    if (cell) *cell = word & ((1u << 22) - 1);
    if (seg_count) *seg_count = ((word >> 22) & 0xF) + 1;
    if (retrace_start) *retrace_start = (word >> 26) & 0xF;
    if (replace) *replace = (word >> 30) & 1;
    if (reuse_light) *reuse_light = (word >> 31) & 1;
}

// photon_store.cpp:38-54 (Table 1 of the paper)
void prx_memory_footprint(uint64_t n_paths, uint32_t max_bounces, const uint32_t* dm_dims, uint32_t n_dims,
                          int area_light, double out[7]) {
    constexpr double kMiB = 1024.0 * 1024.0;
    uint64_t cells = 1;
    for (uint32_t i = 0; i < n_dims; ++i) cells *= dm_dims[i];
    const double n = static_cast<double>(n_paths);
    out[0] = 4.0 * n / kMiB;
    out[1] = area_light ? 12.0 * n / kMiB : 0.0;
    out[2] = 2.0 * 4.0 * static_cast<double>(cells) / kMiB;
    out[3] = 4.0 * n / kMiB;
    out[4] = 32.0 * n * max_bounces / kMiB;
    out[5] = out[0] + out[1] + out[2] + out[3];
    out[6] = out[5] + out[4];
}

prx_status prx_scene_create(const prx_scene_desc* desc, prx_scene** out) {
    return guarded([&] {
        need(desc, "desc");
        need(out, "out");
        auto s = std::make_unique<prx_scene>();
        s->scene = std::make_shared<prx::Scene>(prx::scene_from_desc(*desc));
        *out = s.release();
    });
}

prx_status prx_scene_builtin(const char* name, prx_scene** out) {
    return guarded([&] {
        need(name, "name");
        need(out, "out");
        auto s = std::make_unique<prx_scene>();
        s->scene = std::make_shared<prx::Scene>(prx::make_builtin_scene(name));
        *out = s.release();
    });
}

// scene.cpp:272-398
prx_status prx_scene_load(const char* source, prx_scene** out) {
    return guarded([&] {
        need(source, "source");
        need(out, "out");
        auto s = std::make_unique<prx_scene>();
        s->scene = std::make_shared<prx::Scene>(prx::load_scene_source(source));
        *out = s.release();
    });
}

prx_status prx_scene_load_text(const char* json_text, const char* base_dir, prx_scene** out) {
    return guarded([&] {
        need(json_text, "json_text");
        need(out, "out");
        auto s = std::make_unique<prx_scene>();
        s->scene = std::make_shared<prx::Scene>(prx::load_scene_text(json_text, base_dir ? base_dir : ""));
        *out = s.release();
    });
}

prx_status prx_scene_synthetic(const char* name, uint32_t n_dynamic, float tri_scale, prx_scene** out) {
    return guarded([&] {
        need(name, "name");
        need(out, "out");
        auto s = std::make_unique<prx_scene>();
        s->scene = std::make_shared<prx::Scene>(prx::make_synthetic_scene(name, n_dynamic, tri_scale));
        *out = s.release();
    });
}

prx_status prx_scene_describe(const prx_scene* scene, prx_scene_desc* out) {
    return guarded([&] {
        need(scene, "scene");
        need(out, "out");
        const prx::Scene& s = *scene->scene;
        out->objects = s.desc_objects.data();
        out->n_objects = static_cast<uint32_t>(s.desc_objects.size());
        out->lights = s.desc_lights.data();
        out->n_lights = static_cast<uint32_t>(s.desc_lights.size());
        out->camera.position = {s.camera.position.x, s.camera.position.y, s.camera.position.z};
        out->camera.look_at = {s.camera.look_at.x, s.camera.look_at.y, s.camera.look_at.z};
        out->camera.fov_deg = s.camera.fov_deg;
        out->camera.width = s.camera.width;
        out->camera.height = s.camera.height;
        out->frames = s.frames;
    });
}

prx_status prx_scene_bvh_permutation(const prx_scene* scene, uint32_t* out, size_t capacity, size_t* count) {
    return guarded([&] {
        need(scene, "scene");
        need(count, "count");
        const auto& perm = scene->scene->bvh_perm;
        *count = perm.size();
        if (out) std::memcpy(out, perm.data(), std::min(capacity, perm.size()) * 4);
    });
}

prx_status prx_scene_counts(const prx_scene* scene, uint64_t counts[4]) {
    return guarded([&] {
        need(scene, "scene");
        const prx::Scene& s = *scene->scene;
        uint64_t dyn = 0;
        for (const auto& o : s.objects)
            if (o.dynamic) dyn += o.mesh.size();
        counts[0] = s.static_tris.size();
        counts[1] = dyn;
        counts[2] = s.bvh_nodes.size();
        counts[3] = s.objects.size();
    });
}

float prx_scene_diagonal(const prx_scene* scene) { return scene ? scene->scene->diagonal() : 0.0f; }

void prx_scene_destroy(prx_scene* scene) { delete scene; }

prx_status prx_engine_create(const prx_scene* scene, const prx_config* cfg, prx_engine** out) {
    return guarded([&] {
        need(scene, "scene");
        need(cfg, "cfg");
        need(out, "out");
        auto e = std::make_unique<prx_engine>();
        e->engine = std::make_unique<prx::Engine>(scene->scene, *cfg);
        *out = e.release();
    });
}

void prx_engine_destroy(prx_engine* engine) { delete engine; }

prx_status prx_engine_get_info(const prx_engine* engine, prx_engine_info* out) {
    return guarded([&] {
        need(engine, "engine");
        need(out, "out");
        engine->engine->info(out);
    });
}

prx_status prx_run_frame(prx_engine* engine, prx_frame_stats* stats) {
    return guarded([&] { eng_raw(engine).run_frame(stats); });
}
prx_status prx_frame_update(prx_engine* engine, prx_frame_stats* stats) {
    return guarded([&] { eng(engine).frame_update(stats); });
}
prx_status prx_verify_paths(prx_engine* engine, prx_frame_stats* stats) {
    return guarded([&] { eng(engine).verify_paths(stats); });
}
prx_status prx_retrace_invalid(prx_engine* engine, prx_frame_stats* stats) {
    return guarded([&] { eng(engine).retrace_invalid(stats); });
}
prx_status prx_run_stage(prx_engine* engine, int stage, prx_frame_stats* stats) {
    return guarded([&] { eng(engine).run_stage(stage, stats); });
}

prx_status prx_engine_dm_current(prx_engine* engine, uint32_t light, void** dev_ptr, uint32_t* cells) {
    return guarded([&] { eng(engine).dm_current_ptr(light, dev_ptr, cells); });
}
prx_status prx_prune_count(prx_engine* engine, uint32_t* const* unmarked_dev) {
    return guarded([&] {
        need(unmarked_dev, "unmarked_dev");
        eng(engine).prune_count(unmarked_dev);
    });
}
prx_status prx_prune_apply(prx_engine* engine, const uint32_t* const* prefix_dev, const uint32_t* const* total_dev,
                           prx_frame_stats* stats) {
    return guarded([&] {
        need(prefix_dev, "prefix_dev");
        need(total_dev, "total_dev");
        eng(engine).prune_apply(prefix_dev, total_dev, stats);
    });
}
prx_status prx_fill_count(prx_engine* engine, uint32_t* dead_out) {
    return guarded([&] {
        need(dead_out, "dead_out");
        eng(engine).fill_count(dead_out);
    });
}
prx_status prx_fill_apply(prx_engine* engine, const uint64_t* dead_prefix, const uint64_t* dead_total,
                          prx_frame_stats* stats) {
    return guarded([&] {
        need(dead_prefix, "dead_prefix");
        need(dead_total, "dead_total");
        eng(engine).fill_apply(dead_prefix, dead_total, stats);
    });
}
prx_status prx_engine_set_collectives(prx_engine* engine, const prx_collectives* coll) {
    return guarded([&] { eng(engine).set_collectives(coll); });
}

struct prx_comm {
    std::unique_ptr<prx::Comm> comm;
};

struct prx_group {
    std::vector<std::unique_ptr<prx_engine>> engines;
    std::unique_ptr<prx::EngineGroup> group;
};

prx_status prx_group_create(const prx_scene* scene, const prx_config* cfg, const int32_t* devices,
                            int32_t n_devices, prx_group** out) {
    return guarded([&] {
        need(scene, "scene");
        need(cfg, "cfg");
        need(devices, "devices");
        need(out, "out");
        if (n_devices < 1 || n_devices > prx::kMaxLocalRanks)
            throw std::invalid_argument("group: n_devices must be 1..16");
        auto g = std::make_unique<prx_group>();
        std::vector<prx::Engine*> raw;
        const uint64_t n = cfg->n_paths;
        for (int32_t r = 0; r < n_devices; ++r) {
            prx_config c = *cfg;
            c.device = devices[r];
            c.shard_begin = static_cast<uint32_t>(n * r / n_devices);
            c.shard_end = static_cast<uint32_t>(n * (r + 1) / n_devices);
            auto e = std::make_unique<prx_engine>();
            e->engine = std::make_unique<prx::Engine>(scene->scene, c);
            raw.push_back(e->engine.get());
            g->engines.push_back(std::move(e));
        }
        g->group = std::make_unique<prx::EngineGroup>(raw, prx::local_comms(n_devices));
        *out = g.release();
    });
}

prx_status prx_group_run_frame(prx_group* group, prx_frame_stats* stats) {
    return guarded([&] {
        need(group, "group");
        std::vector<prx_frame_stats> st(group->engines.size());
        group->group->run_all([&](int r, prx::Engine& e) { e.run_frame(&st[r]); });
        if (stats) *stats = st[0];  // the counters are all-shard sums on every shard
    });
}

prx_status prx_group_splat(prx_group* group, const prx_camera* camera, float radius, int mode, float* rgb_out) {
    return guarded([&] {
        need(group, "group");
        group->group->run_all([&](int r, prx::Engine& e) {
            e.splat(camera, radius, mode, r == 0 ? rgb_out : nullptr, nullptr, nullptr);
        });
    });
}

prx_engine* prx_group_engine(prx_group* group, int32_t rank) {
    if (!group || rank < 0 || rank >= static_cast<int32_t>(group->engines.size())) return nullptr;
    return group->engines[rank].get();
}

int32_t prx_group_size(const prx_group* group) {
    return group ? static_cast<int32_t>(group->engines.size()) : 0;
}

void prx_group_destroy(prx_group* group) {
    if (!group) return;
    group->group.reset();  // joins the shard threads before the engines go
    delete group;
}

prx_status prx_comm_nccl_unique_id(uint8_t id_out[128]) {
    return guarded([&] {
        need(id_out, "id_out");
        prx::nccl_unique_id(id_out);
    });
}
prx_status prx_comm_nccl_create(const uint8_t id[128], int32_t rank, int32_t world, int32_t device, prx_comm** out) {
    return guarded([&] {
        need(id, "id");
        need(out, "out");
        auto c = std::make_unique<prx_comm>();
        c->comm = prx::nccl_comm(id, rank, world, device);
        *out = c.release();
    });
}
prx_status prx_comm_local_create(int32_t world, prx_comm** comms_out) {
    return guarded([&] {
        need(comms_out, "comms_out");
        auto v = prx::local_comms(world);
        for (int r = 0; r < world; ++r) {
            comms_out[r] = new prx_comm;
            comms_out[r]->comm = std::move(v[r]);
        }
    });
}
prx_status prx_comm_collectives(prx_comm* comm, prx_collectives* out) {
    return guarded([&] {
        need(comm, "comm");
        need(out, "out");
        comm->comm->table(out);
    });
}
void prx_comm_destroy(prx_comm* comm) { delete comm; }

prx_status prx_engine_set_stream(prx_engine* engine, void* cuda_stream) {
    return guarded([&] { eng(engine).set_stream(static_cast<cudaStream_t>(cuda_stream)); });
}
prx_status prx_engine_synchronize(prx_engine* engine) {
    return guarded([&] { eng(engine).synchronize(); });
}

prx_status prx_engine_set_splat_overlap(prx_engine* engine, int32_t on) {
    return guarded([&] { eng(engine).set_splat_overlap(on != 0); });
}

prx_status prx_splat(prx_engine* engine, const prx_camera* camera, float radius, int mode, float* rgb_out,
                     float* rgb_dev, prx_frame_stats* stats) {
    return guarded([&] { eng_raw(engine).splat(camera, radius, mode, rgb_out, rgb_dev, stats); });
}

prx_status prx_gather_photons(prx_engine* engine, const void* photons, const void* aux, uint32_t n_paths,
                              uint32_t max_bounces, int32_t frame, const prx_camera* camera, float radius,
                              int mode, float* rgb_out) {
    return guarded([&] {
        eng(engine).gather_photons(photons, aux, n_paths, max_bounces, frame, camera, radius, mode, rgb_out);
    });
}

size_t prx_field_bytes(const prx_engine* engine, int field, uint32_t index) {
    try {
        if (!engine) return 0;
        return engine->engine->field_bytes(field, index);
    } catch (const std::exception& e) {
        fail(e);
        return 0;
    }
}

prx_status prx_engine_download(prx_engine* engine, int field, uint32_t index, void* dst, size_t bytes) {
    return guarded([&] {
        if (bytes) need(dst, "dst");
        eng(engine).download(field, index, dst, bytes);
    });
}

prx_status prx_engine_upload(prx_engine* engine, int field, uint32_t index, const void* src, size_t bytes) {
    return guarded([&] {
        if (bytes) need(src, "src");
        eng(engine).upload(field, index, src, bytes);
    });
}

prx_status prx_engine_set_frame_counter(prx_engine* engine, int32_t frames_run) {
    return guarded([&] { eng(engine).set_frame_counter(frames_run); });
}

prx_status prx_intersect_batch(prx_engine* engine, const float* rays, size_t n, int any_hit, float* hits) {
    return guarded([&] {
        if (n) {
            need(rays, "rays");
            need(hits, "hits");
        }
        eng(engine).intersect_batch(rays, n, any_hit, hits);
    });
}

// ------------------------------------------------------------------ offline artefacts
prx_status prx_photon_dump_write(const char* path, uint32_t n_paths, uint32_t max_bounces, const void* records,
                                 size_t bytes) {
    return guarded([&] {
        need(path, "path");
        if (bytes) need(records, "records");
        prx::write_photon_dump(path, n_paths, max_bounces, records, bytes);
    });
}

prx_status prx_photon_dump_read(const char* path, uint32_t* n_paths, uint32_t* max_bounces, void* records,
                                size_t capacity) {
    return guarded([&] {
        need(path, "path");
        std::vector<char> buf;
        uint32_t n = 0, b = 0;
        prx::read_photon_dump(path, &n, &b, records ? &buf : nullptr);
        if (records) {
            if (capacity < buf.size()) throw std::invalid_argument("photon dump: records buffer too small");
            std::memcpy(records, buf.data(), buf.size());
        }
        if (n_paths) *n_paths = n;
        if (max_bounces) *max_bounces = b;
    });
}

prx_status prx_engine_write_photon_dump(prx_engine* engine, const char* path) {
    return guarded([&] {
        need(path, "path");
        prx_engine_info info{};
        eng(engine).info(&info);
        if (info.shard_begin != 0 || info.shard_end != info.n_paths)
            throw std::invalid_argument("photon dump: engine holds a path shard, dump the gathered map");
        const size_t bytes = eng(engine).field_bytes(PRX_FIELD_PHOTONS, 0);
        std::vector<char> buf(bytes);
        eng(engine).download(PRX_FIELD_PHOTONS, 0, buf.data(), bytes);
        prx::write_photon_dump(path, info.n_paths, info.max_bounces, buf.data(), bytes);
    });
}

prx_status prx_image_write_ppm(const char* path, const float* rgb, uint32_t width, uint32_t height) {
    return guarded([&] {
        need(path, "path");
        if (width && height) need(rgb, "rgb");
        prx::write_image_ppm(path, rgb, width, height);
    });
}

size_t prx_frame_image_name(int32_t frame, char* buf, size_t capacity) {
    const std::string name = prx::frame_image_name(frame);
    if (buf && capacity) {
        const size_t n = std::min(capacity - 1, name.size());
        std::memcpy(buf, name.data(), n);
        buf[n] = 0;
    }
    return name.size();
}

prx_status prx_stats_csv_write(const char* path, const prx_frame_stats* rows, size_t n) {
    return guarded([&] {
        need(path, "path");
        if (n) need(rows, "rows");
        prx::write_stats_csv(path, rows, n);
    });
}

prx_status prx_stats_csv_read(const char* path, prx_frame_stats* rows, size_t capacity, size_t* n_out) {
    return guarded([&] {
        need(path, "path");
        const std::vector<prx_frame_stats> r = prx::read_stats_csv(path);
        if (n_out) *n_out = r.size();
        if (rows) {
            if (capacity < r.size()) throw std::invalid_argument("stats CSV: rows buffer too small");
            std::copy(r.begin(), r.end(), rows);
        }
    });
}

prx_status prx_reuse_report(const prx_frame_stats* rows, size_t n, char* buf, size_t capacity, size_t* len_out) {
    return guarded([&] {
        if (n) need(rows, "rows");
        const std::string text = prx::reuse_report(rows, n);
        if (len_out) *len_out = text.size();
        if (buf && capacity) {
            const size_t k = std::min(capacity - 1, text.size());
            std::memcpy(buf, text.data(), k);
            buf[k] = 0;
        }
    });
}

uint64_t prx_engine_launch_count(const prx_engine* engine) {
    return engine ? engine->engine->launches() : 0;
}

prx_status prx_engine_transfer_bytes(const prx_engine* engine, uint64_t* h2d, uint64_t* d2h) {
    return guarded([&] { eng(const_cast<prx_engine*>(engine)).transfer_bytes(h2d, d2h); });
}

}  // extern "C"
