// host_scene.cpp -- host half of the scene model (see host_scene.h).
//
// Compiled WITHOUT -march / fast-math (like the reference, proj/CMakeLists.txt), so
// float expressions evaluate with the same rounding as the reference's host code.
#include "host_scene.h"

#include <algorithm>
#include <cmath>
#include <numbers>
#include <numeric>

namespace prx {

// ------------------------------------------------------------------ quaternions / xforms
bool operator==(const Quat& a, const Quat& b) {
    return a.x == b.x && a.y == b.y && a.z == b.z && a.w == b.w;
}

float quat_norm(const Quat& q) { return std::sqrt(q.x * q.x + q.y * q.y + q.z * q.z + q.w * q.w); }

Quat quat_normalized(const Quat& q) {
    const float n = quat_norm(q);
    return {q.x / n, q.y / n, q.z / n, q.w / n};
}

Quat quat_axis_angle(V3 axis, float radians) {
    const V3 u = normalized(axis);
    const float s = std::sin(radians * 0.5f);
    return {u.x * s, u.y * s, u.z * s, std::cos(radians * 0.5f)};
}

V3 rotate(const Quat& q, V3 v) {
    const V3 u{q.x, q.y, q.z};
    const V3 t = mul(cross(u, v), 2.0f);
    return add(add(v, mul(t, q.w)), cross(u, t));
}

static float quat_dot(const Quat& a, const Quat& b) {
    return a.x * b.x + a.y * b.y + a.z * b.z + a.w * b.w;
}

Quat slerp(const Quat& a, Quat b, float t) {
    float cos_omega = quat_dot(a, b);
    if (cos_omega < 0.0f) {
        b = {-b.x, -b.y, -b.z, -b.w};
        cos_omega = -cos_omega;
    }
    float ka, kb;
    if (cos_omega > 0.9995f) {
        ka = 1.0f - t;
        kb = t;
    } else {
        const float omega = std::acos(fmin_std(cos_omega, 1.0f));
        const float inv_sin = 1.0f / std::sin(omega);
        ka = std::sin((1.0f - t) * omega) * inv_sin;
        kb = std::sin(t * omega) * inv_sin;
    }
    const Quat r{ka * a.x + kb * b.x, ka * a.y + kb * b.y, ka * a.z + kb * b.z,
                 ka * a.w + kb * b.w};
    return quat_normalized(r);
}

bool operator==(const Xform& a, const Xform& b) {
    return a.rot == b.rot && eq(a.trans, b.trans) && a.scale == b.scale;
}

V3 apply_point(const Xform& xf, V3 p) { return add(rotate(xf.rot, mul(p, xf.scale)), xf.trans); }

Xform interpolate(const Xform& a, const Xform& b, float t) {
    Xform r;
    r.rot = slerp(a.rot, b.rot, t);
    r.trans = add(a.trans, mul(sub(b.trans, a.trans), t));
    r.scale = a.scale + (b.scale - a.scale) * t;
    return r;
}

Box transform_box(const Box& box, const Xform& xf) {
    Box out = empty_box();
    for (int i = 0; i < 8; ++i) {
        const V3 corner{(i & 1) ? box.hi.x : box.lo.x, (i & 2) ? box.hi.y : box.lo.y,
                        (i & 4) ? box.hi.z : box.lo.z};
        expand(out, apply_point(xf, corner));
    }
    return out;
}

Xform transform_at(const std::vector<Keyframe>& kfs, int frame) {
    if (kfs.empty()) return Xform{};
    if (frame <= kfs.front().frame) return kfs.front().xf;
    if (frame >= kfs.back().frame) return kfs.back().xf;
    for (size_t i = 1; i < kfs.size(); ++i) {
        if (frame > kfs[i].frame) continue;
        if (frame == kfs[i].frame) return kfs[i].xf;
        const Keyframe& k0 = kfs[i - 1];
        const float t = static_cast<float>(frame - k0.frame) /
                        static_cast<float>(kfs[i].frame - k0.frame);
        return interpolate(k0.xf, kfs[i].xf, t);
    }
    return kfs.back().xf;
}

bool has_distinct(const std::vector<Keyframe>& kfs) {
    for (size_t i = 1; i < kfs.size(); ++i)
        if (!(kfs[i].xf == kfs[0].xf)) return true;
    return false;
}

// ------------------------------------------------------------------ triangles
Box tri_bounds(const Tri& t) {
    Box b = empty_box();
    expand(b, t.a);
    expand(b, t.b);
    expand(b, t.c);
    return b;
}
V3 tri_centroid(const Tri& t) { return divs(add(add(t.a, t.b), t.c), 3.0f); }
float tri_area(const Tri& t) { return 0.5f * length(cross(sub(t.b, t.a), sub(t.c, t.a))); }

// ------------------------------------------------------------------ lights
bool operator==(const LightPose& a, const LightPose& b) {
    return eq(a.position, b.position) && eq(a.normal, b.normal) && eq(a.tangent, b.tangent) &&
           eq(a.bitangent, b.bitangent) && a.scale == b.scale;
}

LightPose light_pose_at(const Light& light, int frame) {
    const Xform xf = transform_at(light.kfs, frame);
    LightPose p;
    p.position = xf.trans;
    p.normal = rotate(xf.rot, V3{0, 0, 1});
    p.tangent = rotate(xf.rot, V3{1, 0, 0});
    p.bitangent = rotate(xf.rot, V3{0, 1, 0});
    p.scale = xf.scale;
    return p;
}

void validate_light(const Light& light) {
    if (light.flux.x < 0 || light.flux.y < 0 || light.flux.z < 0)
        throw std::invalid_argument("light: flux must be non-negative");
    if (light.kind == PRX_LIGHT_SPOT &&
        (light.cone_angle_deg <= 0.0f || light.cone_angle_deg >= 180.0f))
        throw std::invalid_argument("light: spot cone angle must be in (0, 180)");
    if (light.kind == PRX_LIGHT_DISC_AREA && light.radius <= 0.0f)
        throw std::invalid_argument("light: disc radius must be positive");
    if (light.kind == PRX_LIGHT_RECT_AREA && (light.half_x <= 0.0f || light.half_y <= 0.0f))
        throw std::invalid_argument("light: rect half extents must be positive");
    if (light.kind < PRX_LIGHT_POINT || light.kind > PRX_LIGHT_RECT_AREA)
        throw std::invalid_argument("light: unknown kind");
    for (const auto& kf : light.kfs) {
        if (std::fabs(quat_norm(kf.xf.rot) - 1.0f) > 1e-5f)
            throw std::invalid_argument("light: keyframe rotation is not a unit quaternion");
        if (kf.xf.scale <= 0.0f) throw std::invalid_argument("light: keyframe scale must be > 0");
    }
}

// ------------------------------------------------------------------ static BVH
// Median split on the longest centroid axis, leaves of <= 4 triangles, nodes numbered in
// creation (pre-)order with the left subtree first -- the tree of Bvh::build
// (bvh.cpp:13-77).  std::nth_element with the same strict total order yields the same
// partition and leaf order, which fixes the closest-hit tie rule (first hit in left-first
// DFS order wins, bvh.cpp:94-97) on the GPU as well.
namespace {
constexpr uint32_t kLeafSize = 4;

struct BvhBuilder {
    std::vector<BvhNode>& nodes;
    std::vector<uint32_t>& order;
    const std::vector<Box>& tb;
    const std::vector<V3>& cent;

    uint32_t build(uint32_t begin, uint32_t end) {
        const uint32_t idx = static_cast<uint32_t>(nodes.size());
        nodes.emplace_back();
        Box bounds = empty_box();
        for (uint32_t i = begin; i < end; ++i) expand(bounds, tb[order[i]]);
        nodes[idx].bounds = bounds;
        const uint32_t count = end - begin;
        if (count <= kLeafSize) {
            nodes[idx].first = begin;
            nodes[idx].count = static_cast<uint16_t>(count);
            return idx;
        }
        Box cb = empty_box();
        for (uint32_t i = begin; i < end; ++i) expand(cb, cent[order[i]]);
        const V3 ext = sub(cb.hi, cb.lo);
        int axis = 0;
        if (ext.y > ext.x) axis = 1;
        if (ext.z > comp(ext, axis)) axis = 2;
        const uint32_t mid = begin + count / 2;
        std::nth_element(order.begin() + begin, order.begin() + mid, order.begin() + end,
                         [&](uint32_t a, uint32_t b) {
                             const float ca = comp(cent[a], axis), cbv = comp(cent[b], axis);
                             if (ca != cbv) return ca < cbv;
                             return a < b;
                         });
        nodes[idx].axis = static_cast<uint16_t>(axis);
        const uint32_t left = build(begin, mid);
        const uint32_t right = build(mid, end);
        nodes[idx].left = left;
        nodes[idx].first = right;
        nodes[idx].count = 0;
        return idx;
    }
};
}  // namespace

void build_static_bvh(Scene& scene) {
    scene.bvh_nodes.clear();
    scene.bvh_perm.clear();
    const size_t n = scene.static_tris.size();
    if (n == 0) return;
    scene.bvh_perm.resize(n);
    std::iota(scene.bvh_perm.begin(), scene.bvh_perm.end(), 0u);
    std::vector<Box> tb(n);
    std::vector<V3> cent(n);
    for (size_t i = 0; i < n; ++i) {
        tb[i] = tri_bounds(scene.static_tris[i]);
        cent[i] = tri_centroid(scene.static_tris[i]);
    }
    scene.bvh_nodes.reserve(2 * n);
    BvhBuilder b{scene.bvh_nodes, scene.bvh_perm, tb, cent};
    b.build(0, static_cast<uint32_t>(n));
}

// ------------------------------------------------------------------ finalize
namespace {
void validate_material(const Material& m, const std::string& where) {
    for (int ch = 0; ch < 3; ++ch) {
        const float a = comp(m.albedo, ch);
        if (!(a >= 0.0f && a <= 1.0f))
            throw SceneError(where + ": albedo channels must lie in [0, 1]");
    }
    if (m.kind == PRX_MATERIAL_GLOSSY && m.glossy_exponent < 1.0f)
        throw SceneError(where + ": glossy_exponent must be >= 1");
}

void validate_keyframes(const std::vector<Keyframe>& kfs, const std::string& where) {
    for (size_t i = 0; i < kfs.size(); ++i) {
        if (std::fabs(quat_norm(kfs[i].xf.rot) - 1.0f) > 1e-5f)
            throw SceneError(where + ": keyframe rotation is not a unit quaternion");
        if (kfs[i].xf.scale <= 0.0f) throw SceneError(where + ": keyframe scale must be > 0");
        if (i > 0 && kfs[i].frame <= kfs[i - 1].frame)
            throw SceneError(where + ": keyframe frames must be strictly increasing");
    }
}
}  // namespace

void finalize_scene(Scene& scene) {
    if (scene.objects.empty()) throw SceneError("scene: needs at least one object");
    if (scene.lights.empty()) throw SceneError("scene: needs at least one light");
    if (scene.lights.size() > PRX_MAX_LIGHTS)
        throw SceneError("scene: at most " + std::to_string(PRX_MAX_LIGHTS) + " lights");
    if (scene.camera.width < 1 || scene.camera.height < 1)
        throw SceneError("scene: camera resolution must be >= 1");
    if (!(scene.camera.fov_deg > 0.0f && scene.camera.fov_deg < 180.0f))
        throw SceneError("scene: camera fov must be in (0, 180)");
    for (size_t i = 0; i < scene.objects.size(); ++i) {
        Object& obj = scene.objects[i];
        obj.id = static_cast<uint32_t>(i);
        const std::string where = "object '" + obj.name + "'";
        if (obj.mesh.empty()) throw SceneError(where + ": empty mesh");
        validate_material(obj.material, where);
        if (obj.kfs.empty()) obj.kfs.push_back({0, Xform{}});
        validate_keyframes(obj.kfs, where);
        obj.dynamic = has_distinct(obj.kfs);
        obj.local_bounds = empty_box();
        for (const Tri& t : obj.mesh) {
            if (tri_area(t) < 1e-10f) throw SceneError(where + ": degenerate triangle in mesh");
            expand(obj.local_bounds, tri_bounds(t));
        }
    }
    for (Light& light : scene.lights) {
        if (light.kfs.empty()) light.kfs.push_back({0, Xform{}});
        validate_light(light);
    }
    scene.static_tris.clear();
    scene.static_tri_obj.clear();
    scene.world_bounds = empty_box();
    for (const Object& obj : scene.objects) {
        const Xform xf0 = transform_at(obj.kfs, 0);
        if (obj.dynamic) {
            expand(scene.world_bounds, transform_box(obj.local_bounds, xf0));
            continue;
        }
        for (const Tri& t : obj.mesh) {
            const Tri w{apply_point(xf0, t.a), apply_point(xf0, t.b), apply_point(xf0, t.c)};
            scene.static_tris.push_back(w);
            scene.static_tri_obj.push_back(obj.id);
            expand(scene.world_bounds, tri_bounds(w));
        }
    }
    build_static_bvh(scene);
    for (const Light& light : scene.lights) expand(scene.world_bounds, light_pose_at(light, 0).position);
    fill_desc_views(scene);
}

// ------------------------------------------------------------------ C-ABI description
namespace {
V3 from(const prx_vec3& v) { return {v.x, v.y, v.z}; }
prx_vec3 to(V3 v) { return {v.x, v.y, v.z}; }
Xform xf_from(const prx_keyframe& k) {
    Xform xf;
    xf.rot = {k.rotation.x, k.rotation.y, k.rotation.z, k.rotation.w};
    xf.trans = from(k.translation);
    xf.scale = k.scale;
    return xf;
}
prx_keyframe kf_to(const Keyframe& k) {
    prx_keyframe o;
    o.frame = k.frame;
    o.rotation = {k.xf.rot.x, k.xf.rot.y, k.xf.rot.z, k.xf.rot.w};
    o.translation = to(k.xf.trans);
    o.scale = k.xf.scale;
    return o;
}
}  // namespace

Scene scene_from_desc(const prx_scene_desc& d) {
    if (d.n_objects && !d.objects) throw std::invalid_argument("scene desc: objects is NULL");
    if (d.n_lights && !d.lights) throw std::invalid_argument("scene desc: lights is NULL");
    Scene s;
    for (uint32_t i = 0; i < d.n_objects; ++i) {
        const prx_object_desc& od = d.objects[i];
        Object o;
        o.name = od.name ? od.name : "";
        if (od.n_triangles && !od.mesh) throw std::invalid_argument("scene desc: mesh is NULL");
        o.mesh.reserve(od.n_triangles);
        for (uint32_t t = 0; t < od.n_triangles; ++t)
            o.mesh.push_back({from(od.mesh[t].a), from(od.mesh[t].b), from(od.mesh[t].c)});
        o.material.kind = od.material.kind;
        o.material.albedo = from(od.material.albedo);
        o.material.glossy_exponent = od.material.glossy_exponent;
        for (uint32_t k = 0; k < od.n_keyframes; ++k)
            o.kfs.push_back({od.keyframes[k].frame, xf_from(od.keyframes[k])});
        s.objects.push_back(std::move(o));
    }
    for (uint32_t i = 0; i < d.n_lights; ++i) {
        const prx_light_desc& ld = d.lights[i];
        Light l;
        l.kind = ld.kind;
        l.flux = from(ld.flux);
        l.cone_angle_deg = ld.cone_angle_deg;
        l.radius = ld.radius;
        l.half_x = ld.half_x;
        l.half_y = ld.half_y;
        for (uint32_t k = 0; k < ld.n_keyframes; ++k)
            l.kfs.push_back({ld.keyframes[k].frame, xf_from(ld.keyframes[k])});
        s.lights.push_back(std::move(l));
    }
    s.camera.position = from(d.camera.position);
    s.camera.look_at = from(d.camera.look_at);
    s.camera.fov_deg = d.camera.fov_deg;
    s.camera.width = d.camera.width;
    s.camera.height = d.camera.height;
    s.frames = d.frames;
    finalize_scene(s);
    return s;
}

void fill_desc_views(Scene& s) {
    s.desc_meshes.clear();
    s.desc_obj_kfs.clear();
    s.desc_light_kfs.clear();
    s.desc_objects.clear();
    s.desc_lights.clear();
    for (const Object& o : s.objects) {
        std::vector<prx_triangle> m;
        m.reserve(o.mesh.size());
        for (const Tri& t : o.mesh) m.push_back({to(t.a), to(t.b), to(t.c)});
        s.desc_meshes.push_back(std::move(m));
        std::vector<prx_keyframe> k;
        for (const Keyframe& kf : o.kfs) k.push_back(kf_to(kf));
        s.desc_obj_kfs.push_back(std::move(k));
    }
    for (const Light& l : s.lights) {
        std::vector<prx_keyframe> k;
        for (const Keyframe& kf : l.kfs) k.push_back(kf_to(kf));
        s.desc_light_kfs.push_back(std::move(k));
    }
    for (size_t i = 0; i < s.objects.size(); ++i) {
        const Object& o = s.objects[i];
        prx_object_desc d{};
        d.name = o.name.c_str();
        d.mesh = s.desc_meshes[i].data();
        d.n_triangles = static_cast<uint32_t>(s.desc_meshes[i].size());
        d.material.kind = o.material.kind;
        d.material.albedo = to(o.material.albedo);
        d.material.glossy_exponent = o.material.glossy_exponent;
        d.keyframes = s.desc_obj_kfs[i].data();
        d.n_keyframes = static_cast<uint32_t>(s.desc_obj_kfs[i].size());
        s.desc_objects.push_back(d);
    }
    for (size_t i = 0; i < s.lights.size(); ++i) {
        const Light& l = s.lights[i];
        prx_light_desc d{};
        d.kind = l.kind;
        d.flux = to(l.flux);
        d.cone_angle_deg = l.cone_angle_deg;
        d.radius = l.radius;
        d.half_x = l.half_x;
        d.half_y = l.half_y;
        d.keyframes = s.desc_light_kfs[i].data();
        d.n_keyframes = static_cast<uint32_t>(s.desc_light_kfs[i].size());
        s.desc_lights.push_back(d);
    }
}

// ------------------------------------------------------------------ meshes
std::vector<Tri> make_box_mesh(V3 h) {
    // Corners indexed by (x<0?0:1, y, z) bits; two triangles per face with outward winding.
    auto P = [&](int ix, int iy, int iz) {
        return V3{ix ? h.x : -h.x, iy ? h.y : -h.y, iz ? h.z : -h.z};
    };
    const V3 c000 = P(0, 0, 0), c001 = P(0, 0, 1), c010 = P(0, 1, 0), c011 = P(0, 1, 1);
    const V3 c100 = P(1, 0, 0), c101 = P(1, 0, 1), c110 = P(1, 1, 0), c111 = P(1, 1, 1);
    return {
        {c000, c100, c101}, {c000, c101, c001},  // y-
        {c010, c111, c110}, {c010, c011, c111},  // y+
        {c000, c010, c110}, {c000, c110, c100},  // z-
        {c001, c101, c111}, {c001, c111, c011},  // z+
        {c000, c001, c011}, {c000, c011, c010},  // x-
        {c100, c110, c111}, {c100, c111, c101},  // x+
    };
}

}  // namespace prx
