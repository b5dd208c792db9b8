// ORACLE / TEST INFRASTRUCTURE ONLY -- never linked into the product.
//
// C ABI over the UNMODIFIED reference engine compiled from /root/reference/proj/src
// (see oracle/Makefile).  Gives the parity tests, smoke() and bench.py's reference arm
// access to:
//   * scenes built through the reference's own Scene + finalize_scene (scene.cpp:63-113)
//     and builtins (scene.cpp:603-611);
//   * Engine::run_frame (engine.cpp:201-242) and each stage of it (engine.cpp:244-598),
//     with the frame prelude (engine.cpp:202-226) restated here because run_frame does
//     not expose it separately;
//   * state download/upload in the product's prx_field layouts (include/prx.h), so any
//     stage can be fed identical inputs on both sides;
//   * gather_image (gather.cpp:35-75).
// The private engine members are reached with the usual test-only access trick.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>
#include <functional>
#include <map>
#include <unordered_map>
#include <atomic>
#include <thread>
#include <mutex>

#define private public
#include "pathreuse/engine.hpp"
#include "pathreuse/gather.hpp"
#include "pathreuse/light.hpp"
#include "pathreuse/parallel.hpp"
#include "pathreuse/scene.hpp"
#include "pathreuse/stats.hpp"
#include "pathreuse/photon_store.hpp"
#undef private

#include "prx.h"

using namespace pathreuse;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
    g_err = e.what();
    if (dynamic_cast<const SceneError*>(&e)) return PRX_E_SCENE;
    if (dynamic_cast<const std::invalid_argument*>(&e)) return PRX_E_INVALID_ARGUMENT;
    if (dynamic_cast<const std::out_of_range*>(&e)) return PRX_E_OUT_OF_RANGE;
    if (dynamic_cast<const std::logic_error*>(&e)) return PRX_E_LOGIC;
    return PRX_E_RUNTIME;
}

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return PRX_OK;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

Vec3 V(const prx_vec3& v) { return {v.x, v.y, v.z}; }
prx_vec3 P(const Vec3& v) { return {v.x, v.y, v.z}; }

RigidTransform xf_of(const prx_keyframe& k) {
    RigidTransform xf;
    xf.rotation = {k.rotation.x, k.rotation.y, k.rotation.z, k.rotation.w};
    xf.translation = V(k.translation);
    xf.scale = k.scale;
    return xf;
}

prx_keyframe kf_of(int frame, const RigidTransform& xf) {
    prx_keyframe k;
    k.frame = frame;
    k.rotation = {xf.rotation.x, xf.rotation.y, xf.rotation.z, xf.rotation.w};
    k.translation = P(xf.translation);
    k.scale = xf.scale;
    return k;
}

// Scene wrapper holding flattened description arrays for prxref_scene_describe.
struct RefScene {
    Scene scene;
    std::vector<std::vector<prx_triangle>> meshes;
    std::vector<std::vector<prx_keyframe>> obj_kfs, light_kfs;
    std::vector<prx_object_desc> objs;
    std::vector<prx_light_desc> lights;
    std::vector<std::string> names;
};

struct RefEngine {
    std::unique_ptr<Engine> engine;
};

void flatten(RefScene& rs) {
    const Scene& s = rs.scene;
    rs.meshes.clear();
    rs.obj_kfs.clear();
    rs.light_kfs.clear();
    rs.objs.clear();
    rs.lights.clear();
    rs.names.clear();
    for (const auto& o : s.objects) {
        std::vector<prx_triangle> m;
        for (const auto& t : o.mesh) m.push_back({P(t.a), P(t.b), P(t.c)});
        rs.meshes.push_back(std::move(m));
        std::vector<prx_keyframe> k;
        for (const auto& kf : o.keyframes) k.push_back(kf_of(kf.frame, kf.xf));
        rs.obj_kfs.push_back(std::move(k));
        rs.names.push_back(o.name);
    }
    for (const auto& l : s.lights) {
        std::vector<prx_keyframe> k;
        for (const auto& kf : l.keyframes) k.push_back(kf_of(kf.frame, kf.xf));
        rs.light_kfs.push_back(std::move(k));
    }
    for (size_t i = 0; i < s.objects.size(); ++i) {
        const auto& o = s.objects[i];
        prx_object_desc d{};
        d.name = rs.names[i].c_str();
        d.mesh = rs.meshes[i].data();
        d.n_triangles = static_cast<uint32_t>(rs.meshes[i].size());
        d.material.kind = o.material.kind == MaterialKind::Glossy ? PRX_MATERIAL_GLOSSY
                                                                  : PRX_MATERIAL_DIFFUSE;
        d.material.albedo = P(o.material.albedo);
        d.material.glossy_exponent = o.material.glossy_exponent;
        d.keyframes = rs.obj_kfs[i].data();
        d.n_keyframes = static_cast<uint32_t>(rs.obj_kfs[i].size());
        rs.objs.push_back(d);
    }
    for (size_t i = 0; i < s.lights.size(); ++i) {
        const auto& l = s.lights[i];
        prx_light_desc d{};
        d.kind = static_cast<int32_t>(l.kind);
        d.flux = P(l.flux);
        d.cone_angle_deg = l.cone_angle_deg;
        d.radius = l.radius;
        d.half_x = l.half_x;
        d.half_y = l.half_y;
        d.keyframes = rs.light_kfs[i].data();
        d.n_keyframes = static_cast<uint32_t>(rs.light_kfs[i].size());
        rs.lights.push_back(d);
    }
}

EngineConfig cfg_of(const prx_config& c) {
    EngineConfig cfg;
    cfg.mode = c.mode == PRX_MODE_BASELINE ? EngineMode::Baseline
               : c.mode == PRX_MODE_NAIVE  ? EngineMode::Naive
                                           : EngineMode::ErrorBased;
    cfg.n_paths = c.n_paths;
    cfg.max_bounces = c.max_bounces;
    cfg.dm_dims.assign(c.dm_dims, c.dm_dims + 4);
    cfg.threshold = c.threshold;
    cfg.seed = c.seed;
    cfg.gather_radius = c.gather_radius;
    cfg.workers = c.workers;
    cfg.record_flags = c.record_flags != 0;
    return cfg;
}

void fill_stats(const FrameStats& s, prx_frame_stats* out) {
    if (!out) return;
    out->frame = s.frame;
    out->mode = s.mode == EngineMode::Baseline ? PRX_MODE_BASELINE
                : s.mode == EngineMode::Naive  ? PRX_MODE_NAIVE
                                               : PRX_MODE_ERROR;
    out->rays_traced = s.rays_traced;
    out->rays_reused = s.rays_reused;
    out->paths_replaced = s.paths_replaced;
    out->paths_pruned = s.paths_pruned;
    out->paths_filled = s.paths_filled;
    out->visibility_rays = s.visibility_rays;
    out->t_update = s.t_update;
    out->t_occlusion = s.t_occlusion;
    out->t_dm = s.t_dm;
    out->t_prune = s.t_prune;
    out->t_fill = s.t_fill;
    out->t_trace = s.t_trace;
    out->t_gather = s.t_gather;
}

void to_stats(const prx_frame_stats* in, FrameStats& s) {
    if (!in) return;
    s.frame = in->frame;
    s.rays_traced = in->rays_traced;
    s.rays_reused = in->rays_reused;
    s.paths_replaced = in->paths_replaced;
    s.paths_pruned = in->paths_pruned;
    s.paths_filled = in->paths_filled;
    s.visibility_rays = in->visibility_rays;
    s.t_update = in->t_update;
    s.t_occlusion = in->t_occlusion;
    s.t_dm = in->t_dm;
    s.t_prune = in->t_prune;
    s.t_fill = in->t_fill;
    s.t_trace = in->t_trace;
}

struct F4 {
    float x, y, z, w;
};

float bits_f(uint32_t u) {
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}
uint32_t f_bits(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    return u;
}

size_t field_bytes(const Engine& e, int field, uint32_t index) {
    const size_t n = e.total_paths_;
    const size_t v = e.photons_.records().size();
    switch (field) {
        case PRX_FIELD_PHOTONS: return v * sizeof(Photon);
        case PRX_FIELD_AUX: return v * sizeof(PathVertexAux);
        case PRX_FIELD_POS_OBJ:
        case PRX_FIELD_ENERGY:
        case PRX_FIELD_IN_DIR:
        case PRX_FIELD_OUT_DIR: return v * 16;
        case PRX_FIELD_ORIGIN:
        case PRX_FIELD_EMISSION_DIR:
        case PRX_FIELD_CANONICAL: return n * 16;
        case PRX_FIELD_CELL:
        case PRX_FIELD_EPOCH:
        case PRX_FIELD_PATH_INFO:
        case PRX_FIELD_META:
        case PRX_FIELD_SEGMENT_FLAGS: return n * 4;
        case PRX_FIELD_RETRACE_START: return n;
        case PRX_FIELD_DM_TARGET:
        case PRX_FIELD_DM_CURRENT:
            if (index >= e.lights_.size()) throw std::out_of_range("light index");
            return e.lights_[index].dm_t.counts.size() * 4;
        case PRX_FIELD_PRUNED: return e.pruned_.size() * 4;
    }
    throw std::invalid_argument("unknown field");
}

// The frame prelude of Engine::run_frame (engine.cpp:202-232), restated so the stages
// can be driven one by one.  Returns the frame number.
int prelude(Engine& e, FrameStats& stats) {
    const int frame = e.frame_counter_++;
    e.state_cur_ = state_at(e.scene_, frame);
    for (auto& block : e.lights_) {
        block.pose_prev = block.pose_now;
        block.pose_now = light_pose_at(*block.light, frame);
        block.moved = frame > 0 && !(block.pose_now == block.pose_prev);
    }
    e.occlusion_boxes_.clear();
    if (frame > 0) {
        for (const PlacedDynamic& pd : e.state_cur_.placed_dynamics) {
            Aabb box = Aabb::united(pd.bounds_previous, pd.bounds_current);
            box.inflate(e.eps_world_);
            e.occlusion_boxes_.push_back(box);
        }
    }
    stats.frame = frame;
    stats.mode = e.cfg_.mode;
    e.pruned_.clear();
    std::fill(e.filled_this_frame_.begin(), e.filled_this_frame_.end(), uint8_t{0});
    std::fill(e.retrace_start_.begin(), e.retrace_start_.end(), kNoRetrace);
    if (e.cfg_.record_flags) e.segment_flags_.assign(e.total_paths_, 0);
    return frame;
}

}  // namespace

extern "C" {

const char* prxref_last_error(void) { return g_err.c_str(); }

int prxref_scene_create(const prx_scene_desc* d, void** out) {
    return guarded([&] {
        auto rs = std::make_unique<RefScene>();
        Scene& s = rs->scene;
        for (uint32_t i = 0; i < d->n_objects; ++i) {
            const prx_object_desc& od = d->objects[i];
            SceneObject obj;
            obj.name = od.name ? od.name : "";
            for (uint32_t t = 0; t < od.n_triangles; ++t)
                obj.mesh.push_back({V(od.mesh[t].a), V(od.mesh[t].b), V(od.mesh[t].c)});
            obj.material.kind = od.material.kind == PRX_MATERIAL_GLOSSY ? MaterialKind::Glossy
                                                                        : MaterialKind::Diffuse;
            obj.material.albedo = V(od.material.albedo);
            obj.material.glossy_exponent = od.material.glossy_exponent;
            for (uint32_t k = 0; k < od.n_keyframes; ++k)
                obj.keyframes.push_back({od.keyframes[k].frame, xf_of(od.keyframes[k])});
            s.objects.push_back(std::move(obj));
        }
        for (uint32_t i = 0; i < d->n_lights; ++i) {
            const prx_light_desc& ld = d->lights[i];
            Light l;
            l.kind = static_cast<LightKind>(ld.kind);
            l.flux = V(ld.flux);
            l.cone_angle_deg = ld.cone_angle_deg;
            l.radius = ld.radius;
            l.half_x = ld.half_x;
            l.half_y = ld.half_y;
            for (uint32_t k = 0; k < ld.n_keyframes; ++k)
                l.keyframes.push_back({ld.keyframes[k].frame, xf_of(ld.keyframes[k])});
            s.lights.push_back(std::move(l));
        }
        s.camera.position = V(d->camera.position);
        s.camera.look_at = V(d->camera.look_at);
        s.camera.fov_deg = d->camera.fov_deg;
        s.camera.width = d->camera.width;
        s.camera.height = d->camera.height;
        s.frames = d->frames;
        finalize_scene(s);
        flatten(*rs);
        *out = rs.release();
    });
}

int prxref_scene_builtin(const char* name, void** out) {
    return guarded([&] {
        auto rs = std::make_unique<RefScene>();
        rs->scene = make_builtin_scene(name);
        flatten(*rs);
        *out = rs.release();
    });
}

int prxref_scene_describe(void* sp, prx_scene_desc* out) {
    auto* rs = static_cast<RefScene*>(sp);
    const Scene& s = rs->scene;
    out->objects = rs->objs.data();
    out->n_objects = static_cast<uint32_t>(rs->objs.size());
    out->lights = rs->lights.data();
    out->n_lights = static_cast<uint32_t>(rs->lights.size());
    out->camera.position = P(s.camera.position);
    out->camera.look_at = P(s.camera.look_at);
    out->camera.fov_deg = s.camera.fov_deg;
    out->camera.width = s.camera.width;
    out->camera.height = s.camera.height;
    out->frames = s.frames;
    return PRX_OK;
}

float prxref_scene_diagonal(void* sp) { return static_cast<RefScene*>(sp)->scene.diagonal(); }

int prxref_scene_bvh_permutation(void* sp, uint32_t* out, size_t cap, size_t* count) {
    const Scene& s = static_cast<RefScene*>(sp)->scene;
    if (!s.static_bvh) {
        *count = 0;
        return PRX_OK;
    }
    const auto& perm = s.static_bvh->permutation();
    *count = perm.size();
    if (out) std::memcpy(out, perm.data(), std::min(cap, perm.size()) * 4);
    return PRX_OK;
}

// Dynamic flags per object (finalize_scene, scene.cpp:189).
int prxref_scene_dynamic_flags(void* sp, uint8_t* out, size_t cap) {
    const Scene& s = static_cast<RefScene*>(sp)->scene;
    for (size_t i = 0; i < s.objects.size() && i < cap; ++i) out[i] = s.objects[i].dynamic;
    return PRX_OK;
}

void prxref_scene_destroy(void* sp) { delete static_cast<RefScene*>(sp); }

int prxref_engine_create(void* sp, const prx_config* c, void** out) {
    return guarded([&] {
        auto re = std::make_unique<RefEngine>();
        re->engine = std::make_unique<Engine>(static_cast<RefScene*>(sp)->scene, cfg_of(*c));
        *out = re.release();
    });
}

void prxref_engine_destroy(void* ep) { delete static_cast<RefEngine*>(ep); }

void prxref_engine_set_workers(void* ep, unsigned workers) {
    auto& e = *static_cast<RefEngine*>(ep)->engine;
    e.cfg_.workers = workers == 0 ? default_worker_count() : workers;
}

int prxref_engine_get_info(void* ep, prx_engine_info* info) {
    const Engine& e = *static_cast<RefEngine*>(ep)->engine;
    std::memset(info, 0, sizeof(*info));
    info->n_paths = e.total_paths_;
    info->max_bounces = e.cfg_.max_bounces;
    info->n_lights = static_cast<uint32_t>(e.lights_.size());
    info->shard_begin = 0;
    info->shard_end = e.total_paths_;
    info->eps_world = e.eps_world_;
    info->diagonal = e.scene_.diagonal();
    info->frames_run = e.frame_counter_;
    info->n_pruned = static_cast<uint32_t>(e.pruned_.size());
    for (size_t li = 0; li < e.lights_.size() && li < PRX_MAX_LIGHTS; ++li) {
        const auto& b = e.lights_[li];
        info->light_path_begin[li] = b.path_begin;
        info->light_path_end[li] = b.path_end;
        info->dm_ndims[li] = static_cast<uint32_t>(b.layout.dims.size());
        for (size_t a = 0; a < b.layout.dims.size(); ++a) info->dm_dims[li][a] = b.layout.dims[a];
        info->dm_cells[li] = b.layout.total_cells();
        info->flux_per_path[li][0] = b.flux_per_path.x;
        info->flux_per_path[li][1] = b.flux_per_path.y;
        info->flux_per_path[li][2] = b.flux_per_path.z;
    }
    return PRX_OK;
}

int prxref_run_frame(void* ep, prx_frame_stats* out) {
    return guarded([&] {
        const FrameStats s = static_cast<RefEngine*>(ep)->engine->run_frame();
        if (out) std::memset(out, 0, sizeof(*out));
        fill_stats(s, out);
    });
}

// Frame prelude (+ the baseline release, engine.cpp:228-232).
int prxref_frame_update(void* ep, prx_frame_stats* out) {
    return guarded([&] {
        Engine& e = *static_cast<RefEngine*>(ep)->engine;
        FrameStats s;
        prelude(e, s);
        if (e.cfg_.mode == EngineMode::Baseline) {
            e.release_all_paths();
            for (auto& block : e.lights_)
                std::fill(block.dm_c.counts.begin(), block.dm_c.counts.end(), 0u);
        }
        if (out) std::memset(out, 0, sizeof(*out));
        fill_stats(s, out);
    });
}

// One stage of run_frame, with run_frame's own guards (engine.cpp:233-240).
int prxref_run_stage(void* ep, int stage, prx_frame_stats* io) {
    return guarded([&] {
        Engine& e = *static_cast<RefEngine*>(ep)->engine;
        FrameStats s;
        to_stats(io, s);
        s.mode = e.cfg_.mode;
        const int frame = e.frame_counter_ - 1;
        switch (stage) {
            case PRX_STAGE_UPDATE_ORIGINS:
                if (e.cfg_.mode != EngineMode::Baseline && frame > 0) e.stage_update_origins(s);
                break;
            case PRX_STAGE_OCCLUSIONS:
                if (e.cfg_.mode != EngineMode::Baseline && frame > 0) e.stage_occlusions(s);
                break;
            case PRX_STAGE_COMPUTE_DM: e.stage_compute_dm(s); break;
            case PRX_STAGE_PRUNE:
                if (e.cfg_.mode != EngineMode::Baseline) e.stage_prune(s);
                break;
            case PRX_STAGE_FILL: e.stage_fill(s); break;
            case PRX_STAGE_TRACE: e.stage_trace(s); break;
            default: throw std::invalid_argument("unknown stage");
        }
        fill_stats(s, io);
    });
}

size_t prxref_field_bytes(void* ep, int field, uint32_t index) {
    try {
        return field_bytes(*static_cast<RefEngine*>(ep)->engine, field, index);
    } catch (const std::exception& ex) {
        fail(ex);
        return 0;
    }
}

int prxref_download(void* ep, int field, uint32_t index, void* dst, size_t bytes) {
    return guarded([&] {
        const Engine& e = *static_cast<RefEngine*>(ep)->engine;
        if (bytes != field_bytes(e, field, index)) throw std::invalid_argument("size mismatch");
        const auto& ph = e.photons_.records();
        const auto& aux = e.aux_;
        const size_t n = e.total_paths_;
        F4* f4 = static_cast<F4*>(dst);
        uint32_t* u32 = static_cast<uint32_t*>(dst);
        uint8_t* u8 = static_cast<uint8_t*>(dst);
        switch (field) {
            case PRX_FIELD_PHOTONS: std::memcpy(dst, ph.data(), bytes); break;
            case PRX_FIELD_AUX: std::memcpy(dst, aux.data(), bytes); break;
            case PRX_FIELD_POS_OBJ:
                for (size_t i = 0; i < ph.size(); ++i)
                    f4[i] = {aux[i].position.x, aux[i].position.y, aux[i].position.z,
                             bits_f(ph[i].object_id)};
                break;
            case PRX_FIELD_ENERGY:
                for (size_t i = 0; i < ph.size(); ++i)
                    f4[i] = {ph[i].energy.x, ph[i].energy.y, ph[i].energy.z, ph[i].radius};
                break;
            case PRX_FIELD_IN_DIR:
                for (size_t i = 0; i < ph.size(); ++i)
                    f4[i] = {ph[i].incoming_dir.x, ph[i].incoming_dir.y, ph[i].incoming_dir.z, 0};
                break;
            case PRX_FIELD_OUT_DIR:
                for (size_t i = 0; i < ph.size(); ++i)
                    f4[i] = {aux[i].outgoing.x, aux[i].outgoing.y, aux[i].outgoing.z, 0};
                break;
            case PRX_FIELD_ORIGIN:
                for (size_t p = 0; p < n; ++p)
                    f4[p] = {e.origin_[p].x, e.origin_[p].y, e.origin_[p].z, 0};
                break;
            case PRX_FIELD_EMISSION_DIR:
                for (size_t p = 0; p < n; ++p)
                    f4[p] = {e.emission_dir_[p].x, e.emission_dir_[p].y, e.emission_dir_[p].z, 0};
                break;
            case PRX_FIELD_CANONICAL:
                for (size_t p = 0; p < n; ++p)
                    f4[p] = {e.canonical_[p].c[0], e.canonical_[p].c[1], e.canonical_[p].c[2],
                             e.canonical_[p].c[3]};
                break;
            case PRX_FIELD_CELL: std::memcpy(dst, e.cell_.data(), bytes); break;
            case PRX_FIELD_EPOCH: std::memcpy(dst, e.epoch_.data(), bytes); break;
            case PRX_FIELD_PATH_INFO: std::memcpy(dst, e.path_info_.data(), bytes); break;
            case PRX_FIELD_META:
                for (size_t p = 0; p < n; ++p) {
                    u8[4 * p + 0] = e.photon_count_[p];
                    u8[4 * p + 1] = e.escaped_[p];
                    u8[4 * p + 2] = e.status_[p];
                    u8[4 * p + 3] = e.filled_this_frame_[p];
                }
                break;
            case PRX_FIELD_RETRACE_START: std::memcpy(dst, e.retrace_start_.data(), bytes); break;
            case PRX_FIELD_SEGMENT_FLAGS:
                if (e.segment_flags_.size() == n)
                    std::memcpy(dst, e.segment_flags_.data(), bytes);
                else
                    std::memset(dst, 0, bytes);
                break;
            case PRX_FIELD_DM_TARGET:
                std::memcpy(dst, e.lights_[index].dm_t.counts.data(), bytes);
                break;
            case PRX_FIELD_DM_CURRENT:
                std::memcpy(dst, e.lights_[index].dm_c.counts.data(), bytes);
                break;
            case PRX_FIELD_PRUNED:
                for (size_t i = 0; i < e.pruned_.size(); ++i) u32[i] = e.pruned_[i];
                break;
        }
    });
}

int prxref_upload(void* ep, int field, uint32_t index, const void* src, size_t bytes) {
    return guarded([&] {
        Engine& e = *static_cast<RefEngine*>(ep)->engine;
        if (bytes != field_bytes(e, field, index)) throw std::invalid_argument("size mismatch");
        auto& ph = e.photons_.records();
        auto& aux = e.aux_;
        const size_t n = e.total_paths_;
        const F4* f4 = static_cast<const F4*>(src);
        const uint8_t* u8 = static_cast<const uint8_t*>(src);
        switch (field) {
            case PRX_FIELD_PHOTONS: std::memcpy(ph.data(), src, bytes); break;
            case PRX_FIELD_AUX: std::memcpy(aux.data(), src, bytes); break;
            case PRX_FIELD_POS_OBJ:
                for (size_t i = 0; i < ph.size(); ++i) {
                    aux[i].position = {f4[i].x, f4[i].y, f4[i].z};
                    ph[i].object_id = f_bits(f4[i].w);
                }
                break;
            case PRX_FIELD_ENERGY:
                for (size_t i = 0; i < ph.size(); ++i) {
                    ph[i].energy = {f4[i].x, f4[i].y, f4[i].z};
                    ph[i].radius = f4[i].w;
                }
                break;
            case PRX_FIELD_IN_DIR:
                for (size_t i = 0; i < ph.size(); ++i) ph[i].incoming_dir = {f4[i].x, f4[i].y, f4[i].z};
                break;
            case PRX_FIELD_OUT_DIR:
                for (size_t i = 0; i < ph.size(); ++i) aux[i].outgoing = {f4[i].x, f4[i].y, f4[i].z};
                break;
            case PRX_FIELD_ORIGIN:
                for (size_t p = 0; p < n; ++p) e.origin_[p] = {f4[p].x, f4[p].y, f4[p].z};
                break;
            case PRX_FIELD_EMISSION_DIR:
                for (size_t p = 0; p < n; ++p) e.emission_dir_[p] = {f4[p].x, f4[p].y, f4[p].z};
                break;
            case PRX_FIELD_CANONICAL:
                for (size_t p = 0; p < n; ++p) {
                    const int li = static_cast<int>(e.light_of_path(static_cast<uint32_t>(p)));
                    e.canonical_[p].dims = e.lights_[li].light->param_dims();
                    e.canonical_[p].c[0] = f4[p].x;
                    e.canonical_[p].c[1] = f4[p].y;
                    e.canonical_[p].c[2] = f4[p].z;
                    e.canonical_[p].c[3] = f4[p].w;
                }
                break;
            case PRX_FIELD_CELL: std::memcpy(e.cell_.data(), src, bytes); break;
            case PRX_FIELD_EPOCH: std::memcpy(e.epoch_.data(), src, bytes); break;
            case PRX_FIELD_PATH_INFO: std::memcpy(e.path_info_.data(), src, bytes); break;
            case PRX_FIELD_META:
                for (size_t p = 0; p < n; ++p) {
                    e.photon_count_[p] = u8[4 * p + 0];
                    e.escaped_[p] = u8[4 * p + 1];
                    e.status_[p] = u8[4 * p + 2];
                    e.filled_this_frame_[p] = u8[4 * p + 3];
                }
                break;
            case PRX_FIELD_RETRACE_START: std::memcpy(e.retrace_start_.data(), src, bytes); break;
            case PRX_FIELD_SEGMENT_FLAGS:
                e.segment_flags_.assign(static_cast<const uint32_t*>(src),
                                        static_cast<const uint32_t*>(src) + n);
                break;
            case PRX_FIELD_DM_TARGET:
                std::memcpy(e.lights_[index].dm_t.counts.data(), src, bytes);
                break;
            case PRX_FIELD_DM_CURRENT:
                std::memcpy(e.lights_[index].dm_c.counts.data(), src, bytes);
                break;
            case PRX_FIELD_PRUNED: throw std::invalid_argument("pruned list is read-only");
        }
    });
}

// Pretend frames [0, frames_run) have run: light poses of frame frames_run-1 become
// pose_now (engine.cpp:205-209 reads pose_now as the previous pose of the next frame).
int prxref_set_frame_counter(void* ep, int frames_run) {
    return guarded([&] {
        Engine& e = *static_cast<RefEngine*>(ep)->engine;
        e.frame_counter_ = frames_run;
        const int last = frames_run > 0 ? frames_run - 1 : 0;
        for (auto& block : e.lights_) {
            block.pose_now = light_pose_at(*block.light, last);
            block.pose_prev = block.pose_now;
        }
        e.state_cur_ = state_at(e.scene_, last);
    });
}

// gather_image (gather.cpp:35-75) over the engine's current state.
int prxref_gather(void* ep, const prx_camera* cam, float radius, unsigned workers,
                  float* out, double* seconds) {
    return guarded([&] {
        const Engine& e = *static_cast<RefEngine*>(ep)->engine;
        Camera c = e.scene_.camera;
        if (cam) {
            c.position = V(cam->position);
            c.look_at = V(cam->look_at);
            c.fov_deg = cam->fov_deg;
            c.width = cam->width;
            c.height = cam->height;
        }
        const auto t0 = std::chrono::steady_clock::now();
        const Image img = gather_image(e.state_cur_, e.photons_, e.aux_, c, radius,
                                       workers == 0 ? default_worker_count() : workers);
        if (seconds)
            *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        std::memcpy(out, img.pixels.data(), img.pixels.size() * sizeof(float));
    });
}

// select_paths_to_prune (engine.cpp:443-471) -- pure function KAT access.
int prxref_select_paths_to_prune(const uint32_t* paths, size_t n, uint32_t dm_c, uint32_t dm_t,
                                 uint64_t seed, uint32_t frame, uint32_t* out, size_t* count) {
    return guarded([&] {
        const auto pruned = select_paths_to_prune(std::span<const uint32_t>(paths, n), dm_c, dm_t,
                                                  seed, frame);
        *count = pruned.size();
        if (out) std::memcpy(out, pruned.data(), pruned.size() * 4);
    });
}

// Closest hit of intersect_scene (scene.cpp:136-168) for a batch of rays at `frame`;
// hit = {t, object, triangle, px, py, pz, nx, ny, nz} (object = 0xFFFFFFFF on miss).
int prxref_intersect_batch(void* sp, int frame, const float* rays, size_t n, float* hits) {
    return guarded([&] {
        const Scene& s = static_cast<RefScene*>(sp)->scene;
        const SceneState st = state_at(s, frame);
        for (size_t i = 0; i < n; ++i) {
            const float* r = rays + 8 * i;
            const Ray ray{{r[0], r[1], r[2]}, {r[3], r[4], r[5]}, r[6], r[7]};
            float* h = hits + 9 * i;
            const auto hit = intersect_scene(ray, st);
            if (!hit) {
                h[0] = 0;
                h[1] = bits_f(kInvalidObjectId);
                h[2] = 0;
                for (int k = 3; k < 9; ++k) h[k] = 0;
                continue;
            }
            h[0] = hit->t;
            h[1] = bits_f(hit->object_id);
            h[2] = bits_f(hit->triangle);
            h[3] = hit->position.x;
            h[4] = hit->position.y;
            h[5] = hit->position.z;
            h[6] = hit->normal.x;
            h[7] = hit->normal.y;
            h[8] = hit->normal.z;
        }
    });
}

// occluded (scene.cpp:170-177) for a ray batch {o, d, t_min, t_max} -> 1/0 floats
int prxref_occluded_batch(void* sp, int frame, const float* rays, size_t n, float* out) {
    return guarded([&] {
        const Scene& s = static_cast<RefScene*>(sp)->scene;
        const SceneState st = state_at(s, frame);
        for (size_t i = 0; i < n; ++i) {
            const float* r = rays + 8 * i;
            const Ray ray{{r[0], r[1], r[2]}, {r[3], r[4], r[5]}, r[6], r[7]};
            out[i] = occluded(ray, st) ? 1.0f : 0.0f;
        }
    });
}

// ---- offline artefacts through the reference's own writers ----
// load_scene_text (scene.cpp:272-379)
int prxref_scene_load_text(const char* text, const char* base_dir, void** out) {
    return guarded([&] {
        auto rs = std::make_unique<RefScene>();
        rs->scene = load_scene_text(text, base_dir ? base_dir : "");
        flatten(*rs);
        *out = rs.release();
    });
}

// write_photon_dump(engine.photon_map(), path) (photon_store.cpp:76-86)
int prxref_write_photon_dump(void* ep, const char* path) {
    return guarded([&] { write_photon_dump(static_cast<RefEngine*>(ep)->engine->photon_map(), path); });
}

// write_image (gather.cpp:77-92) of a caller-provided float RGB buffer
int prxref_write_image(const char* path, const float* rgb, uint32_t w, uint32_t h) {
    return guarded([&] {
        Image img;
        img.width = w;
        img.height = h;
        img.pixels.assign(rgb, rgb + static_cast<size_t>(w) * h * 3);
        write_image(img, path);
    });
}

static FrameStats stats_of(const prx_frame_stats& r) {
    FrameStats s;
    s.frame = r.frame;
    s.mode = static_cast<EngineMode>(r.mode);
    s.rays_traced = r.rays_traced;
    s.rays_reused = r.rays_reused;
    s.paths_replaced = r.paths_replaced;
    s.paths_pruned = r.paths_pruned;
    s.paths_filled = r.paths_filled;
    s.visibility_rays = r.visibility_rays;
    s.t_update = r.t_update;
    s.t_occlusion = r.t_occlusion;
    s.t_dm = r.t_dm;
    s.t_prune = r.t_prune;
    s.t_fill = r.t_fill;
    s.t_trace = r.t_trace;
    s.t_gather = r.t_gather;
    return s;
}

// write_stats_csv (stats.cpp:14-33)
int prxref_write_stats_csv(const char* path, const prx_frame_stats* rows, size_t n) {
    return guarded([&] {
        std::vector<FrameStats> v;
        for (size_t i = 0; i < n; ++i) v.push_back(stats_of(rows[i]));
        write_stats_csv(v, std::string(path));
    });
}

// reuse_report (stats.cpp:72-107) into a caller buffer
int prxref_reuse_report(const prx_frame_stats* rows, size_t n, char* buf, size_t cap, size_t* len) {
    return guarded([&] {
        std::vector<FrameStats> v;
        for (size_t i = 0; i < n; ++i) v.push_back(stats_of(rows[i]));
        const std::string t = reuse_report(v);
        *len = t.size();
        if (buf && cap) {
            const size_t k = std::min(cap - 1, t.size());
            std::memcpy(buf, t.data(), k);
            buf[k] = 0;
        }
    });
}

}  // extern "C"
