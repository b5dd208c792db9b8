// pathreuse_b200.hpp -- source-compatible C++ surface of the reference `pathreuse` library
// (proj/include/pathreuse/*.hpp) backed by the B200 engine through the C ABI (prx.h).
//
// A reference user swaps `#include "pathreuse/engine.hpp"` (+ gather.hpp) for this header and
// links paper_2111_06906_b200/_prx.so.  Types keep the reference's names and fields; Engine
// keeps its constructor, run_frame() and the introspection accessors of engine.hpp:76-122
// (served from lazily refreshed host mirrors of the device state); gather_image keeps the
// reference's meaning.  Errors surface as the reference's exception types.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "prx.h"

namespace pathreuse {

// ---------------------------------------------------------------- errors (scene.hpp:76)
struct SceneError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

namespace detail {
inline void check(prx_status s) {
    if (s == PRX_OK) return;
    const std::string msg = prx_last_error();
    switch (s) {
        case PRX_E_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case PRX_E_OUT_OF_RANGE: throw std::out_of_range(msg);
        case PRX_E_LOGIC: throw std::logic_error(msg);
        case PRX_E_SCENE: throw SceneError(msg);
        default: throw std::runtime_error(msg);
    }
}
}  // namespace detail

// ---------------------------------------------------------------- math (vec3.hpp, geometry.hpp)
struct Vec3 {
    float x = 0.0f, y = 0.0f, z = 0.0f;
    constexpr Vec3() = default;
    constexpr Vec3(float x_, float y_, float z_) : x(x_), y(y_), z(z_) {}
    explicit constexpr Vec3(float s) : x(s), y(s), z(s) {}
    float operator[](int i) const { return i == 0 ? x : (i == 1 ? y : z); }
    Vec3 operator+(const Vec3& o) const { return {x + o.x, y + o.y, z + o.z}; }
    Vec3 operator-(const Vec3& o) const { return {x - o.x, y - o.y, z - o.z}; }
    Vec3 operator*(float s) const { return {x * s, y * s, z * s}; }
    Vec3 operator*(const Vec3& o) const { return {x * o.x, y * o.y, z * o.z}; }
    bool operator==(const Vec3& o) const { return x == o.x && y == o.y && z == o.z; }
};
inline constexpr uint32_t kInvalidObjectId = 0xFFFFFFFFu;
struct Triangle {
    Vec3 a, b, c;
};
struct Aabb {  // geometry.hpp:20-39
    Vec3 lo{3.402823466e+38f, 3.402823466e+38f, 3.402823466e+38f};
    Vec3 hi{-3.402823466e+38f, -3.402823466e+38f, -3.402823466e+38f};
    bool valid() const { return lo.x <= hi.x && lo.y <= hi.y && lo.z <= hi.z; }
};
struct Quat {
    float x = 0.0f, y = 0.0f, z = 0.0f, w = 1.0f;
};
struct RigidTransform {
    Quat rotation;
    Vec3 translation;
    float scale = 1.0f;
};

// ---------------------------------------------------------------- scene (scene.hpp, light.hpp)
enum class MaterialKind { Diffuse, Glossy };
struct Material {
    MaterialKind kind = MaterialKind::Diffuse;
    Vec3 albedo{0.5f, 0.5f, 0.5f};
    float glossy_exponent = 1.0f;
};
struct ObjectKeyframe {
    int frame = 0;
    RigidTransform xf;
};
struct SceneObject {
    uint32_t id = 0;
    std::string name;
    std::vector<Triangle> mesh;
    Material material;
    std::vector<ObjectKeyframe> keyframes;
    bool dynamic = false;
};
enum class LightKind { Point, Spot, DiscArea, RectArea };
struct LightKeyframe {
    int frame = 0;
    RigidTransform xf;
};
struct Light {
    LightKind kind = LightKind::Point;
    Vec3 flux;
    float cone_angle_deg = 60.0f;
    float radius = 1.0f;
    float half_x = 1.0f, half_y = 1.0f;
    std::vector<LightKeyframe> keyframes;
};
struct Camera {
    Vec3 position{0, 1, 4};
    Vec3 look_at{0, 1, 0};
    float fov_deg = 60.0f;
    uint32_t width = 120, height = 90;
};

// A finalized scene: plain data plus the finalized device-ready handle.
struct Scene {
    std::vector<SceneObject> objects;
    std::vector<Light> lights;
    Camera camera;
    int frames = 1;
    std::shared_ptr<prx_scene> handle;  // set by finalize_scene / make_builtin_scene
    float diagonal() const { return handle ? prx_scene_diagonal(handle.get()) : 0.0f; }
};

namespace detail {
inline prx_vec3 v(const Vec3& a) { return {a.x, a.y, a.z}; }
inline Vec3 v(const prx_vec3& a) { return {a.x, a.y, a.z}; }
inline prx_keyframe kf(int frame, const RigidTransform& x) {
    return {frame, {x.rotation.x, x.rotation.y, x.rotation.z, x.rotation.w}, v(x.translation), x.scale};
}
inline RigidTransform xf(const prx_keyframe& k) {
    return {{k.rotation.x, k.rotation.y, k.rotation.z, k.rotation.w}, v(k.translation), k.scale};
}
inline std::shared_ptr<prx_scene> own(prx_scene* s) { return {s, prx_scene_destroy}; }

// Fill the plain-data view of `s` from its finalized handle.
inline void load_view(Scene& s) {
    prx_scene_desc d{};
    check(prx_scene_describe(s.handle.get(), &d));
    s.objects.clear();
    s.lights.clear();
    for (uint32_t i = 0; i < d.n_objects; ++i) {
        const prx_object_desc& o = d.objects[i];
        SceneObject obj;
        obj.id = i;
        obj.name = o.name ? o.name : "";
        for (uint32_t t = 0; t < o.n_triangles; ++t) obj.mesh.push_back({v(o.mesh[t].a), v(o.mesh[t].b), v(o.mesh[t].c)});
        obj.material.kind = o.material.kind == PRX_MATERIAL_GLOSSY ? MaterialKind::Glossy : MaterialKind::Diffuse;
        obj.material.albedo = v(o.material.albedo);
        obj.material.glossy_exponent = o.material.glossy_exponent;
        for (uint32_t k = 0; k < o.n_keyframes; ++k) obj.keyframes.push_back({o.keyframes[k].frame, xf(o.keyframes[k])});
        for (size_t k = 1; k < obj.keyframes.size(); ++k) {
            const RigidTransform& a = obj.keyframes[k].xf;
            const RigidTransform& b = obj.keyframes[0].xf;
            if (!(a.rotation.x == b.rotation.x && a.rotation.y == b.rotation.y && a.rotation.z == b.rotation.z &&
                  a.rotation.w == b.rotation.w && a.translation == b.translation && a.scale == b.scale))
                obj.dynamic = true;
        }
        s.objects.push_back(std::move(obj));
    }
    for (uint32_t i = 0; i < d.n_lights; ++i) {
        const prx_light_desc& l = d.lights[i];
        Light light;
        light.kind = static_cast<LightKind>(l.kind);
        light.flux = v(l.flux);
        light.cone_angle_deg = l.cone_angle_deg;
        light.radius = l.radius;
        light.half_x = l.half_x;
        light.half_y = l.half_y;
        for (uint32_t k = 0; k < l.n_keyframes; ++k) light.keyframes.push_back({l.keyframes[k].frame, xf(l.keyframes[k])});
        s.lights.push_back(std::move(light));
    }
    s.camera = {v(d.camera.position), v(d.camera.look_at), d.camera.fov_deg, d.camera.width, d.camera.height};
    s.frames = d.frames;
}
}  // namespace detail

// finalize_scene (scene.cpp:63-113): validates and builds the static BVH (on the C side).
inline void finalize_scene(Scene& s) {
    std::vector<std::vector<prx_triangle>> meshes;
    std::vector<std::vector<prx_keyframe>> okf, lkf;
    std::vector<prx_object_desc> objs;
    std::vector<prx_light_desc> lights;
    for (const SceneObject& o : s.objects) {
        std::vector<prx_triangle> m;
        for (const Triangle& t : o.mesh) m.push_back({detail::v(t.a), detail::v(t.b), detail::v(t.c)});
        meshes.push_back(std::move(m));
        std::vector<prx_keyframe> k;
        for (const ObjectKeyframe& x : o.keyframes) k.push_back(detail::kf(x.frame, x.xf));
        okf.push_back(std::move(k));
    }
    for (const Light& l : s.lights) {
        std::vector<prx_keyframe> k;
        for (const LightKeyframe& x : l.keyframes) k.push_back(detail::kf(x.frame, x.xf));
        lkf.push_back(std::move(k));
    }
    for (size_t i = 0; i < s.objects.size(); ++i) {
        const SceneObject& o = s.objects[i];
        objs.push_back({o.name.c_str(), meshes[i].data(), static_cast<uint32_t>(meshes[i].size()),
                        {o.material.kind == MaterialKind::Glossy ? PRX_MATERIAL_GLOSSY : PRX_MATERIAL_DIFFUSE,
                         detail::v(o.material.albedo), o.material.glossy_exponent},
                        okf[i].data(), static_cast<uint32_t>(okf[i].size())});
    }
    for (size_t i = 0; i < s.lights.size(); ++i) {
        const Light& l = s.lights[i];
        lights.push_back({static_cast<int32_t>(l.kind), detail::v(l.flux), l.cone_angle_deg, l.radius, l.half_x,
                          l.half_y, lkf[i].data(), static_cast<uint32_t>(lkf[i].size())});
    }
    prx_scene_desc d{objs.data(), static_cast<uint32_t>(objs.size()), lights.data(),
                     static_cast<uint32_t>(lights.size()),
                     {detail::v(s.camera.position), detail::v(s.camera.look_at), s.camera.fov_deg, s.camera.width,
                      s.camera.height},
                     s.frames};
    prx_scene* h = nullptr;
    detail::check(prx_scene_create(&d, &h));
    s.handle = detail::own(h);
    detail::load_view(s);
}

// make_builtin_scene (scene.cpp:603-611)
inline Scene make_builtin_scene(const std::string& name) {
    prx_scene* h = nullptr;
    detail::check(prx_scene_builtin(name.c_str(), &h));
    Scene s;
    s.handle = detail::own(h);
    detail::load_view(s);
    return s;
}

// state_at (scene.hpp:62-74): the dynamic objects placed at one frame.  The static BVH lives
// on the device (the reference's `static_bvh` member has no host counterpart here); `engine`
// (B200 extension) names the engine whose device scene this state describes, which is what
// gather_image(state, ...) splats against.
struct PlacedDynamic {
    uint32_t object_id = 0;
    std::vector<Triangle> triangles;  // world space at the current frame
    Aabb bounds_current;
    Aabb bounds_previous;  // equals bounds_current of frame-1 (frame 0: identical)
};
class Engine;
struct SceneState {
    int frame = 0;
    const Scene* scene = nullptr;
    std::vector<PlacedDynamic> placed_dynamics;
    const Engine* engine = nullptr;
};

// state_at (scene.cpp:115-134), evaluated on the host in the reference's float order
inline SceneState state_at(const Scene& scene, int frame) {
    SceneState st;
    st.frame = frame;
    st.scene = &scene;
    size_t nd = 0, nt = 0;
    detail::check(prx_scene_state_at(scene.handle.get(), frame, nullptr, 0, &nd, nullptr, 0, &nt));
    std::vector<prx_placed_dynamic> dyn(nd);
    std::vector<prx_triangle> tris(nt);
    detail::check(prx_scene_state_at(scene.handle.get(), frame, dyn.data(), nd, &nd, tris.data(), nt, &nt));
    for (const prx_placed_dynamic& d : dyn) {
        PlacedDynamic pd;
        pd.object_id = d.object_id;
        for (uint32_t t = 0; t < d.tri_count; ++t) {
            const prx_triangle& x = tris[d.tri_begin + t];
            pd.triangles.push_back({detail::v(x.a), detail::v(x.b), detail::v(x.c)});
        }
        pd.bounds_current = {detail::v(d.cur_lo), detail::v(d.cur_hi)};
        pd.bounds_previous = {detail::v(d.prev_lo), detail::v(d.prev_hi)};
        st.placed_dynamics.push_back(std::move(pd));
    }
    return st;
}

// ---------------------------------------------------------------- photon store (photon_store.hpp)
struct Photon {
    Vec3 incoming_dir;
    uint32_t object_id = kInvalidObjectId;
    Vec3 energy;
    float radius = 0.0f;
    bool live() const { return object_id != kInvalidObjectId; }
};
static_assert(sizeof(Photon) == 32, "photon record must serialize to 32 bytes");
struct PathVertexAux {
    Vec3 position;
    Vec3 outgoing;
};
struct PathInfoFields {
    uint32_t cell = 0, seg_count = 1, retrace_start = 0;
    bool replace = false, reuse_light = false;
    bool operator==(const PathInfoFields&) const = default;
};
inline uint32_t encode_path_info(const PathInfoFields& f) {
    uint32_t w = 0;
    detail::check(prx_encode_path_info(f.cell, f.seg_count, f.retrace_start, f.replace, f.reuse_light, &w));
    return w;
}
inline PathInfoFields decode_path_info(uint32_t word) {
    PathInfoFields f;
    int rep = 0, reuse = 0;
    prx_decode_path_info(word, &f.cell, &f.seg_count, &f.retrace_start, &rep, &reuse);
    f.replace = rep != 0;
    f.reuse_light = reuse != 0;
    return f;
}
class PhotonMap {
public:
    PhotonMap() = default;
    PhotonMap(uint32_t n_paths, uint32_t max_bounces)
        : n_paths_(n_paths), max_bounces_(max_bounces), photons_(static_cast<size_t>(n_paths) * max_bounces) {}
    uint32_t n_paths() const { return n_paths_; }
    uint32_t max_bounces() const { return max_bounces_; }
    size_t flat_index(uint32_t bounce, uint32_t path) const {  // photon_store.cpp:32-36
        if (bounce >= max_bounces_ || path >= n_paths_) throw std::out_of_range("PhotonMap: bounce/path out of range");
        return static_cast<size_t>(bounce) * n_paths_ + path;
    }
    const Photon& at(uint32_t bounce, uint32_t path) const { return photons_[flat_index(bounce, path)]; }
    const std::vector<Photon>& records() const { return photons_; }
    std::vector<Photon>& records() { return photons_; }

private:
    uint32_t n_paths_ = 0, max_bounces_ = 0;
    std::vector<Photon> photons_;
};
struct MemoryFootprint {
    double path_info = 0, origin_positions = 0, distribution_maps = 0, pruned_array = 0, photon_map = 0,
           subtotal_reuse = 0, total = 0;
};
inline MemoryFootprint memory_footprint(uint64_t n_paths, uint32_t max_bounces, const std::vector<uint32_t>& dm_dims,
                                        bool area_light) {
    double o[7];
    prx_memory_footprint(n_paths, max_bounces, dm_dims.data(), static_cast<uint32_t>(dm_dims.size()), area_light, o);
    return {o[0], o[1], o[2], o[3], o[4], o[5], o[6]};
}

// ---------------------------------------------------------------- engine (engine.hpp)
enum class EngineMode { Baseline, Naive, ErrorBased };
inline const char* to_string(EngineMode m) {
    return m == EngineMode::Baseline ? "baseline" : (m == EngineMode::Naive ? "naive" : "error");
}
inline EngineMode engine_mode_from_string(const std::string& n) {
    if (n == "baseline") return EngineMode::Baseline;
    if (n == "naive") return EngineMode::Naive;
    if (n == "error" || n == "error_based" || n == "error-based") return EngineMode::ErrorBased;
    throw std::invalid_argument("unknown engine mode: " + n);
}
struct FrameStats {
    int frame = 0;
    EngineMode mode = EngineMode::Baseline;
    uint64_t rays_traced = 0, rays_reused = 0, paths_replaced = 0, paths_pruned = 0, paths_filled = 0,
             visibility_rays = 0;
    double t_update = 0, t_occlusion = 0, t_dm = 0, t_prune = 0, t_fill = 0, t_trace = 0, t_gather = 0;
};
inline bool energies_close(const Vec3& a, const Vec3& b, float threshold) {
    const float x[3] = {a.x, a.y, a.z}, y[3] = {b.x, b.y, b.z};
    return prx_energies_close(x, y, threshold) != 0;
}
inline double prune_probability(uint32_t dm_c, uint32_t dm_t) { return prx_prune_probability(dm_c, dm_t); }
struct EngineConfig {
    EngineMode mode = EngineMode::Naive;
    uint32_t n_paths = 100000;
    uint32_t max_bounces = 7;
    std::vector<uint32_t> dm_dims = {8, 8, 64, 64};
    float threshold = 0.001f;
    uint64_t seed = 1;
    float gather_radius = 0.25f;
    unsigned workers = 1;
    bool record_flags = false;
    int device = 0;  // B200 extension
};
constexpr uint8_t kNoRetrace = 0xFF;
struct DmLayout {  // light.hpp:62-70
    std::vector<uint32_t> dims;
    uint32_t total_cells() const {
        uint32_t n = 1;
        for (uint32_t d : dims) n *= d;
        return n;
    }
};
struct DistributionMap {  // light.hpp:72-84
    DmLayout layout;
    std::vector<uint32_t> counts;
    explicit DistributionMap(DmLayout l = {})
        : layout(std::move(l)), counts(layout.dims.empty() ? 0 : layout.total_cells(), 0u) {}
    uint64_t total() const {
        uint64_t s = 0;
        for (uint32_t c : counts) s += c;
        return s;
    }
};

// select_paths_to_prune (engine.hpp:62-63, engine.cpp:443-471)
inline std::vector<uint32_t> select_paths_to_prune(std::span<const uint32_t> cell_paths, uint32_t dm_c,
                                                   uint32_t dm_t, uint64_t seed, uint32_t frame) {
    std::vector<uint32_t> out(cell_paths.size());
    size_t n = 0;
    detail::check(prx_select_paths_to_prune(cell_paths.data(), cell_paths.size(), dm_c, dm_t, seed, frame,
                                            out.data(), &n));
    out.resize(n);
    return out;
}
struct Image {
    uint32_t width = 0, height = 0;
    std::vector<float> pixels;  // RGB rows, top-left origin
};

class Engine {
public:
    Engine(Scene scene, EngineConfig cfg) : scene_(std::move(scene)), cfg_(std::move(cfg)) {
        if (cfg_.dm_dims.size() != 4) throw std::invalid_argument("engine: dm_dims needs 4 axis counts");
        if (!scene_.handle) finalize_scene(scene_);
        prx_config c{};
        c.mode = static_cast<int32_t>(cfg_.mode);
        c.n_paths = cfg_.n_paths;
        c.max_bounces = cfg_.max_bounces;
        for (int i = 0; i < 4; ++i) c.dm_dims[i] = cfg_.dm_dims[i];
        c.threshold = cfg_.threshold;
        c.seed = cfg_.seed;
        c.gather_radius = cfg_.gather_radius;
        c.workers = cfg_.workers;
        c.record_flags = cfg_.record_flags;
        c.device = cfg_.device;
        prx_engine* e = nullptr;
        detail::check(prx_engine_create(scene_.handle.get(), &c, &e));
        engine_.reset(e, prx_engine_destroy);
        refresh_info();
    }

    FrameStats run_frame() {
        prx_frame_stats s{};
        detail::check(prx_run_frame(engine_.get(), &s));
        invalidate();
        return convert(s);
    }
    // north_star stage split
    void frame_update(prx_frame_stats& s) { detail::check(prx_frame_update(engine_.get(), &s)); invalidate(); }
    void verify_paths(prx_frame_stats& s) { detail::check(prx_verify_paths(engine_.get(), &s)); invalidate(); }
    void retrace_invalid(prx_frame_stats& s) { detail::check(prx_retrace_invalid(engine_.get(), &s)); invalidate(); }

    const Scene& scene() const { return scene_; }
    const EngineConfig& config() const { return cfg_; }
    int frames_run() const { return info_.frames_run; }
    uint32_t total_paths() const { return info_.n_paths; }
    size_t light_count() const { return info_.n_lights; }
    size_t light_of_path(uint32_t path) const {
        for (uint32_t li = 0; li < info_.n_lights; ++li)
            if (path >= info_.light_path_begin[li] && path < info_.light_path_end[li]) return li;
        throw std::out_of_range("light_of_path: path out of range");
    }
    Vec3 flux_per_path(size_t li) const {
        return {info_.flux_per_path[li][0], info_.flux_per_path[li][1], info_.flux_per_path[li][2]};
    }
    float position_epsilon() const { return info_.eps_world; }

    const PhotonMap& photon_map() const {
        if (!photons_) {
            photons_ = std::make_unique<PhotonMap>(info_.n_paths, info_.max_bounces);
            fetch(PRX_FIELD_PHOTONS, 0, photons_->records().data());
        }
        return *photons_;
    }
    const std::vector<PathVertexAux>& vertex_aux() const {
        if (!aux_) {
            aux_ = std::make_unique<std::vector<PathVertexAux>>(static_cast<size_t>(info_.n_paths) * info_.max_bounces);
            fetch(PRX_FIELD_AUX, 0, aux_->data());
        }
        return *aux_;
    }
    const PathVertexAux& aux_at(uint32_t bounce, uint32_t path) const {
        return vertex_aux()[photon_map().flat_index(bounce, path)];
    }
    const std::vector<uint32_t>& path_info_words() const { return u32(PRX_FIELD_PATH_INFO, path_info_); }
    uint8_t photon_count(uint32_t p) const { return meta()[4 * p]; }
    bool path_escaped(uint32_t p) const { return meta()[4 * p + 1] != 0; }
    bool path_alive(uint32_t p) const { return meta()[4 * p + 2] == 1; }
    uint8_t last_retrace_start(uint32_t p) const {
        if (!rstart_) {
            rstart_ = std::make_unique<std::vector<uint8_t>>(info_.n_paths);
            fetch(PRX_FIELD_RETRACE_START, 0, rstart_->data());
        }
        return (*rstart_)[p];
    }
    Vec3 path_origin(uint32_t p) const { return vec4(PRX_FIELD_ORIGIN, origin_, p); }
    Vec3 path_emission_dir(uint32_t p) const { return vec4(PRX_FIELD_EMISSION_DIR, emis_, p); }
    uint32_t path_cell(uint32_t p) const { return u32(PRX_FIELD_CELL, cell_)[p]; }
    uint32_t path_epoch(uint32_t p) const { return u32(PRX_FIELD_EPOCH, epoch_)[p]; }
    uint32_t segment_count(uint32_t p) const { return photon_count(p) + (path_escaped(p) ? 1u : 0u); }
    const SceneState& scene_state() const {  // engine.hpp:79 (state_at of the last frame run)
        if (!state_) {
            state_ = std::make_unique<SceneState>();
            if (info_.frames_run > 0) *state_ = state_at(scene_, info_.frames_run - 1);
            state_->engine = this;
        }
        return *state_;
    }
    const DmLayout& dm_layout(size_t li) const { return layouts().at(li); }  // engine.hpp:102
    const DistributionMap& dm_target(size_t li) const { return dm(PRX_FIELD_DM_TARGET, li, dm_t_); }
    const DistributionMap& dm_current(size_t li) const { return dm(PRX_FIELD_DM_CURRENT, li, dm_c_); }
    // engine.cpp:125-139: segment i runs from vertex i-1 (or the light) toward vertex i
    Vec3 segment_origin(uint32_t p, uint32_t i) const {
        if (i == 0) return path_origin(p);
        return aux_at(i - 1, p).position;
    }
    Vec3 segment_dir(uint32_t p, uint32_t i) const {
        if (i == 0) return path_emission_dir(p);
        return aux_at(i - 1, p).outgoing;
    }
    Vec3 segment_end(uint32_t p, uint32_t i) const {  // escape segments clipped at 2 x diagonal
        if (i < photon_count(p)) return aux_at(i, p).position;
        return segment_origin(p, i) + segment_dir(p, i) * (2.0f * scene_.diagonal());
    }
    const std::vector<uint32_t>& pruned_paths() const { return u32(PRX_FIELD_PRUNED, pruned_); }
    const std::vector<uint32_t>& segment_flags() const { return u32(PRX_FIELD_SEGMENT_FLAGS, flags_); }
    prx_engine* native() const { return engine_.get(); }

    // prx_frame_stats -> FrameStats (also used by read_stats_csv)
    static FrameStats convert(const prx_frame_stats& s) {
        FrameStats f;
        f.frame = s.frame;
        f.mode = static_cast<EngineMode>(s.mode);
        f.rays_traced = s.rays_traced;
        f.rays_reused = s.rays_reused;
        f.paths_replaced = s.paths_replaced;
        f.paths_pruned = s.paths_pruned;
        f.paths_filled = s.paths_filled;
        f.visibility_rays = s.visibility_rays;
        f.t_update = s.t_update;
        f.t_occlusion = s.t_occlusion;
        f.t_dm = s.t_dm;
        f.t_prune = s.t_prune;
        f.t_fill = s.t_fill;
        f.t_trace = s.t_trace;
        f.t_gather = s.t_gather;
        return f;
    }

private:
    void refresh_info() { detail::check(prx_engine_get_info(engine_.get(), &info_)); }
    void invalidate() {
        refresh_info();
        state_.reset();
        dm_t_.clear();
        dm_c_.clear();
        photons_.reset();
        aux_.reset();
        meta_.reset();
        rstart_.reset();
        for (auto* v : {&path_info_, &cell_, &epoch_, &pruned_, &flags_}) v->reset();
        origin_.reset();
        emis_.reset();
    }
    void fetch(int field, uint32_t index, void* dst) const {
        const size_t n = prx_field_bytes(engine_.get(), field, index);
        detail::check(prx_engine_download(engine_.get(), field, index, dst, n));
    }
    const std::vector<uint32_t>& u32(int field, std::unique_ptr<std::vector<uint32_t>>& cache) const {
        if (!cache) {
            cache = std::make_unique<std::vector<uint32_t>>(prx_field_bytes(engine_.get(), field, 0) / 4);
            if (!cache->empty()) fetch(field, 0, cache->data());
        }
        return *cache;
    }
    const std::vector<uint8_t>& meta() const {
        if (!meta_) {
            meta_ = std::make_unique<std::vector<uint8_t>>(4ull * info_.n_paths);
            fetch(PRX_FIELD_META, 0, meta_->data());
        }
        return *meta_;
    }
    Vec3 vec4(int field, std::unique_ptr<std::vector<float>>& cache, uint32_t p) const {
        if (!cache) {
            cache = std::make_unique<std::vector<float>>(4ull * info_.n_paths);
            fetch(field, 0, cache->data());
        }
        return {(*cache)[4 * p], (*cache)[4 * p + 1], (*cache)[4 * p + 2]};
    }
    const std::vector<DmLayout>& layouts() const {
        if (layouts_.empty())
            for (uint32_t li = 0; li < info_.n_lights; ++li) {
                DmLayout l;
                for (uint32_t a = 0; a < info_.dm_ndims[li]; ++a) l.dims.push_back(info_.dm_dims[li][a]);
                layouts_.push_back(std::move(l));
            }
        return layouts_;
    }
    const DistributionMap& dm(int field, size_t li, std::vector<std::unique_ptr<DistributionMap>>& cache) const {
        if (li >= info_.n_lights) throw std::out_of_range("light index out of range");
        if (cache.size() < info_.n_lights) cache.resize(info_.n_lights);
        if (!cache[li]) {
            cache[li] = std::make_unique<DistributionMap>(layouts()[li]);
            fetch(field, static_cast<uint32_t>(li), cache[li]->counts.data());
        }
        return *cache[li];
    }

    Scene scene_;
    EngineConfig cfg_;
    std::shared_ptr<prx_engine> engine_;
    prx_engine_info info_{};
    mutable std::unique_ptr<PhotonMap> photons_;
    mutable std::unique_ptr<std::vector<PathVertexAux>> aux_;
    mutable std::unique_ptr<std::vector<uint8_t>> meta_, rstart_;
    mutable std::unique_ptr<std::vector<uint32_t>> path_info_, cell_, epoch_, pruned_, flags_;
    mutable std::unique_ptr<std::vector<float>> origin_, emis_;
    mutable std::unique_ptr<SceneState> state_;
    mutable std::vector<DmLayout> layouts_;
    mutable std::vector<std::unique_ptr<DistributionMap>> dm_t_, dm_c_;
};

// gather_image (gather.hpp:81-83) with the reference's signature.  The state must come from
// engine.scene_state() (it names the engine whose device scene the splat runs against).  When
// `photons`/`aux` are that engine's own mirrors the splat reads the device path store directly;
// any other host photon map is uploaded and splatted (prx_gather_photons).  The image is the
// ordered GPU gather: byte-identical to the reference's.  `workers` is ignored.
inline Image gather_image(const SceneState& state, const PhotonMap& photons, std::span<const PathVertexAux> aux,
                          const Camera& cam, float radius, unsigned workers);
// B200 convenience: the engine's current photons
inline Image gather_image(const Engine& engine, const Camera& cam, float radius, unsigned /*workers*/ = 1) {
    Image img;
    img.width = cam.width;
    img.height = cam.height;
    img.pixels.assign(3ull * cam.width * cam.height, 0.0f);
    const prx_camera c{detail::v(cam.position), detail::v(cam.look_at), cam.fov_deg, cam.width, cam.height};
    detail::check(prx_splat(engine.native(), &c, radius, 1, img.pixels.data(), nullptr, nullptr));
    return img;
}

inline Image gather_image(const SceneState& state, const PhotonMap& photons, std::span<const PathVertexAux> aux,
                          const Camera& cam, float radius, unsigned workers) {
    if (!state.engine)
        throw std::invalid_argument("gather_image: the SceneState does not come from an Engine (scene_state())");
    const Engine& engine = *state.engine;
    if (&photons == &engine.photon_map() && aux.data() == engine.vertex_aux().data())
        return gather_image(engine, cam, radius, workers);
    if (aux.size() != photons.records().size())
        throw std::invalid_argument("gather_image: photon map and aux sizes differ");
    Image img;
    img.width = cam.width;
    img.height = cam.height;
    img.pixels.assign(3ull * cam.width * cam.height, 0.0f);
    const prx_camera c{detail::v(cam.position), detail::v(cam.look_at), cam.fov_deg, cam.width, cam.height};
    detail::check(prx_gather_photons(engine.native(), photons.records().data(), aux.data(), photons.n_paths(),
                                     photons.max_bounces(), state.frame, &c, radius, 1, img.pixels.data()));
    return img;
}

// ---------------------------------------------------------------- multi-GPU (B200 extension)
// One Engine over several GPUs (devices may repeat): contiguous path shards, the exchanges
// inside the engines (prx_group_*).  Frames are bit-identical to one Engine; the image is
// the sum of the shards' splats (fp32 order differs).
class MultiGpuEngine {
public:
    MultiGpuEngine(Scene scene, EngineConfig cfg, const std::vector<int>& devices)
        : scene_(std::move(scene)), cfg_(std::move(cfg)) {
        if (!scene_.handle) finalize_scene(scene_);
        prx_config c{};
        c.mode = static_cast<int32_t>(cfg_.mode);
        c.n_paths = cfg_.n_paths;
        c.max_bounces = cfg_.max_bounces;
        for (int i = 0; i < 4; ++i) c.dm_dims[i] = cfg_.dm_dims.at(i);
        c.threshold = cfg_.threshold;
        c.seed = cfg_.seed;
        c.gather_radius = cfg_.gather_radius;
        c.workers = cfg_.workers;
        c.record_flags = cfg_.record_flags;
        std::vector<int32_t> devs(devices.begin(), devices.end());
        prx_group* g = nullptr;
        detail::check(prx_group_create(scene_.handle.get(), &c, devs.data(), static_cast<int32_t>(devs.size()), &g));
        group_.reset(g, prx_group_destroy);
    }
    FrameStats run_frame() {
        prx_frame_stats s{};
        detail::check(prx_group_run_frame(group_.get(), &s));
        return Engine::convert(s);
    }
    Image splat(const Camera& cam, float radius, int mode = 1) {
        Image img;
        img.width = cam.width;
        img.height = cam.height;
        img.pixels.assign(3ull * cam.width * cam.height, 0.0f);
        const prx_camera c{detail::v(cam.position), detail::v(cam.look_at), cam.fov_deg, cam.width, cam.height};
        detail::check(prx_group_splat(group_.get(), &c, radius, mode, img.pixels.data()));
        return img;
    }
    int size() const { return prx_group_size(group_.get()); }
    const Scene& scene() const { return scene_; }

private:
    Scene scene_;
    EngineConfig cfg_;
    std::shared_ptr<prx_group> group_;
};

// ---------------------------------------------------------------- scene documents (scene.hpp)
namespace detail {
inline Scene adopt(prx_scene* h) {
    Scene s;
    s.handle = own(h);
    load_view(s);
    return s;
}
inline prx_frame_stats to_prx(const FrameStats& f) {
    prx_frame_stats s{};
    s.frame = f.frame;
    s.mode = static_cast<int32_t>(f.mode);
    s.rays_traced = f.rays_traced;
    s.rays_reused = f.rays_reused;
    s.paths_replaced = f.paths_replaced;
    s.paths_pruned = f.paths_pruned;
    s.paths_filled = f.paths_filled;
    s.visibility_rays = f.visibility_rays;
    s.t_update = f.t_update;
    s.t_occlusion = f.t_occlusion;
    s.t_dm = f.t_dm;
    s.t_prune = f.t_prune;
    s.t_fill = f.t_fill;
    s.t_trace = f.t_trace;
    s.t_gather = f.t_gather;
    return s;
}
inline std::vector<prx_frame_stats> to_prx(const std::vector<FrameStats>& rows) {
    std::vector<prx_frame_stats> v;
    for (const FrameStats& r : rows) v.push_back(to_prx(r));
    return v;
}
}  // namespace detail

// load_scene_text / load_scene / load_scene_source (scene.cpp:272-398)
inline Scene load_scene_text(const std::string& json_text, const std::string& base_dir = "") {
    prx_scene* h = nullptr;
    detail::check(prx_scene_load_text(json_text.c_str(), base_dir.c_str(), &h));
    return detail::adopt(h);
}
inline Scene load_scene_source(const std::string& source) {
    prx_scene* h = nullptr;
    detail::check(prx_scene_load(source.c_str(), &h));
    return detail::adopt(h);
}
inline Scene load_scene(const std::string& path) { return load_scene_source(path); }

// ---------------------------------------------------------------- offline artefacts
// write_image / frame_image_name (gather.hpp)
inline void write_image(const Image& image, const std::string& path) {
    detail::check(prx_image_write_ppm(path.c_str(), image.pixels.data(), image.width, image.height));
}
inline std::string frame_image_name(int frame) {
    char buf[64];
    prx_frame_image_name(frame, buf, sizeof(buf));
    return buf;
}
// write_photon_dump / read_photon_dump (photon_store.hpp)
inline void write_photon_dump(const PhotonMap& map, const std::string& path) {
    detail::check(prx_photon_dump_write(path.c_str(), map.n_paths(), map.max_bounces(), map.records().data(),
                                        map.records().size() * sizeof(Photon)));
}
inline PhotonMap read_photon_dump(const std::string& path) {
    uint32_t n = 0, b = 0;
    detail::check(prx_photon_dump_read(path.c_str(), &n, &b, nullptr, 0));
    PhotonMap map(n, b);
    detail::check(prx_photon_dump_read(path.c_str(), &n, &b, map.records().data(),
                                       map.records().size() * sizeof(Photon)));
    return map;
}
// write_stats_csv / read_stats_csv / reuse_report (stats.hpp)
inline void write_stats_csv(const std::vector<FrameStats>& rows, const std::string& path) {
    const std::vector<prx_frame_stats> v = detail::to_prx(rows);
    detail::check(prx_stats_csv_write(path.c_str(), v.data(), v.size()));
}
inline std::vector<FrameStats> read_stats_csv(const std::string& path) {
    size_t n = 0;
    detail::check(prx_stats_csv_read(path.c_str(), nullptr, 0, &n));
    std::vector<prx_frame_stats> v(n);
    detail::check(prx_stats_csv_read(path.c_str(), v.data(), v.size(), &n));
    std::vector<FrameStats> out;
    for (const prx_frame_stats& s : v) out.push_back(Engine::convert(s));
    return out;
}
inline std::string reuse_report(const std::vector<FrameStats>& rows) {
    const std::vector<prx_frame_stats> v = detail::to_prx(rows);
    size_t n = 0;
    detail::check(prx_reuse_report(v.data(), v.size(), nullptr, 0, &n));
    std::string text(n + 1, '\0');
    detail::check(prx_reuse_report(v.data(), v.size(), text.data(), text.size(), &n));
    text.resize(n);
    return text;
}

}  // namespace pathreuse
