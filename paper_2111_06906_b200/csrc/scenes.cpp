// scenes.cpp -- scene generators.
//
// 1. The reference builtins (scene.cpp:404-611): same names, geometry, keyframes, lights
//    and cameras, so `run_builtin`/`render_builtin` are drop-ins.  Parity is checked by
//    tests/test_abi.py::test_builtin_scene_bvh_matches_reference and tests/test_io.py::
//    test_builtin_sources against the reference's own make_builtin_scene.
// 2. Procedural BASELINE configurations C1..C5: Cornell box (~1K tris),
//    Sponza-scale (~300K static + 4 x 20K dynamic), Villa-scale (~1M static + 8 x 20K
//    dynamic + 2 moving lights) and the dynamic-object stress sweep.  Both the GPU engine
//    and the CPU oracles consume the exact same triangles via prx_scene_describe.
#include <cmath>
#include <numbers>

#include "host_scene.h"

namespace prx {

namespace {

constexpr float kPi = std::numbers::pi_v<float>;
constexpr float kTau = 2.0f * std::numbers::pi_v<float>;

Keyframe kf_at(int frame, V3 pos, Quat rot = Quat{}, float scale = 1.0f) {
    Keyframe k;
    k.frame = frame;
    k.xf.rot = rot;
    k.xf.trans = pos;
    k.xf.scale = scale;
    return k;
}

Object box_obj(const std::string& name, V3 half, V3 albedo, std::vector<Keyframe> kfs) {
    Object o;
    o.name = name;
    o.mesh = make_box_mesh(half);
    o.material.albedo = albedo;
    o.kfs = std::move(kfs);
    return o;
}

Quat down_facing() { return quat_axis_angle(V3{1, 0, 0}, kPi / 2.0f); }

// scene.cpp:32-39
Quat rotation_z_to(V3 target) {
    const V3 z{0, 0, 1};
    const V3 t = normalized(target);
    const float c = dot(z, t);
    if (c > 1.0f - 1e-6f) return Quat{};
    if (c < -1.0f + 1e-6f) return quat_axis_angle(V3{1, 0, 0}, kPi);
    return quat_normalized(quat_axis_angle(cross(z, t), std::acos(c)));
}

void room(Scene& s, V3 half, V3 center, V3 albedo) {
    s.objects.push_back(box_obj("room", half, albedo, {kf_at(0, center)}));
}

Light make_light(int kind, V3 flux, std::vector<Keyframe> kfs) {
    Light l;
    l.kind = kind;
    l.flux = flux;
    l.kfs = std::move(kfs);
    return l;
}

Camera cam(V3 pos, V3 at, float fov) {
    Camera c;
    c.position = pos;
    c.look_at = at;
    c.fov_deg = fov;
    c.width = 120;
    c.height = 90;
    return c;
}

// ---------------------------------------------------------------- reference builtins
Scene static_box() {
    Scene s;
    s.frames = 10;
    room(s, {5, 3, 5}, {0, 3, 0}, {0.6f, 0.6f, 0.6f});
    s.objects.push_back(box_obj("block-a", {0.5f, 0.5f, 0.5f}, {0.7f, 0.3f, 0.3f},
                                {kf_at(0, {-1.5f, 0.5f, -1})}));
    s.objects.push_back(box_obj("block-b", {0.4f, 0.8f, 0.4f}, {0.3f, 0.3f, 0.7f},
                                {kf_at(0, {1.5f, 0.8f, 0.5f})}));
    s.lights.push_back(make_light(PRX_LIGHT_POINT, {50, 50, 50}, {kf_at(0, {0, 5, 0}, down_facing())}));
    s.camera = cam({0, 2.5f, 4.5f}, {0, 1, 0}, 60.0f);
    return s;
}

Scene moving_cube() {
    Scene s;
    s.frames = 100;
    room(s, {5, 3, 5}, {0, 3, 0}, {0.6f, 0.6f, 0.6f});
    s.objects.push_back(box_obj("block", {0.6f, 0.6f, 0.6f}, {0.3f, 0.5f, 0.7f},
                                {kf_at(0, {1.8f, 0.6f, -1.2f})}));
    std::vector<Keyframe> path;
    for (int i = 0; i <= 8; ++i)
        path.push_back(kf_at(i * 25, {(i % 2 == 0) ? -2.5f : 2.5f, 1.0f, 0.5f}));
    s.objects.push_back(box_obj("cube", {0.3f, 0.3f, 0.3f}, {0.8f, 0.4f, 0.3f}, path));
    Light l = make_light(PRX_LIGHT_RECT_AREA, {80, 80, 80}, {kf_at(0, {0, 5.9f, 0}, down_facing())});
    l.half_x = 0.8f;
    l.half_y = 0.8f;
    s.lights.push_back(l);
    s.camera = cam({0, 2.5f, 4.5f}, {0, 1, 0}, 60.0f);
    return s;
}

Scene parallel_spot() {
    Scene s;
    s.frames = 30;
    s.objects.push_back(box_obj("ground", {8, 0.1f, 8}, {0.6f, 0.6f, 0.6f}, {kf_at(0, {0, -0.1f, 0})}));
    s.objects.push_back(box_obj("block", {0.5f, 0.5f, 0.5f}, {0.5f, 0.4f, 0.3f}, {kf_at(0, {0, 0.5f, -2})}));
    Light l = make_light(PRX_LIGHT_SPOT, {60, 60, 60},
                         {kf_at(0, {-2, 4, 0}, down_facing()), kf_at(20, {2, 4, 0}, down_facing()),
                          kf_at(2000, {2, 4, 0}, down_facing())});
    l.cone_angle_deg = 70.0f;
    s.lights.push_back(l);
    s.camera = cam({0, 3, 7}, {0, 0.5f, 0}, 60.0f);
    return s;
}

Scene armadillo_analog() {
    Scene s;
    s.frames = 200;
    room(s, {6, 2, 4}, {0, 2, 0}, {0.6f, 0.6f, 0.6f});
    s.objects.push_back(box_obj("table", {1.5f, 0.45f, 0.8f}, {0.55f, 0.4f, 0.3f}, {kf_at(0, {0, 0.45f, 0})}));
    s.objects.push_back(box_obj("stand", {0.4f, 0.5f, 0.4f}, {0.45f, 0.45f, 0.5f}, {kf_at(0, {4, 0.5f, 2})}));
    std::vector<Keyframe> walk = {
        kf_at(0, {-5, 0.6f, -3}),   kf_at(40, {0, 0.6f, 2.5f}),  kf_at(60, {0, 0.6f, 2.5f}),
        kf_at(100, {5, 0.6f, -3}),  kf_at(140, {0, 0.6f, 2.5f}), kf_at(160, {0, 0.6f, 2.5f}),
        kf_at(200, {-5, 0.6f, -3}),
    };
    s.objects.push_back(box_obj("walker", {0.25f, 0.6f, 0.25f}, {0.4f, 0.45f, 0.5f}, walk));
    Light l = make_light(PRX_LIGHT_DISC_AREA, {100, 100, 100}, {kf_at(0, {0, 3.95f, 0}, down_facing())});
    l.radius = 0.7f;
    s.lights.push_back(l);
    s.camera = cam({0, 2, 3.8f}, {0, 1, 0}, 70.0f);
    return s;
}

Scene merry_go_round() {
    Scene s;
    s.frames = 200;
    room(s, {5, 2.5f, 5}, {0, 2.5f, 0}, {0.6f, 0.6f, 0.6f});
    s.objects.push_back(box_obj("table", {1.8f, 0.4f, 1.8f}, {0.5f, 0.35f, 0.25f}, {kf_at(0, {0, 0.4f, 0})}));
    for (int i = 0; i < 3; ++i) {
        std::vector<Keyframe> kfs;
        const float base = kTau * static_cast<float>(i) / 3.0f;
        for (int k = 0; k <= 10; ++k) {
            const float spin = kTau * static_cast<float>(k) / 4.0f;
            const float scale = (k % 2 == 0) ? 1.0f : 1.3f;
            const V3 pos{0.9f * std::cos(base), 1.05f, 0.9f * std::sin(base)};
            kfs.push_back(kf_at(k * 20, pos, quat_axis_angle({0, 1, 0}, spin), scale));
        }
        s.objects.push_back(box_obj("teapot-" + std::to_string(i), {0.25f, 0.25f, 0.25f},
                                    {0.7f, 0.7f, 0.75f}, kfs));
    }
    for (int i = 0; i < 8; ++i) {
        std::vector<Keyframe> kfs;
        const float base = kTau * static_cast<float>(i) / 8.0f;
        for (int k = 0; k <= 20; ++k) {
            const int frame = k * 10;
            const float angle = base + kTau * static_cast<float>(frame) / 200.0f;
            kfs.push_back(kf_at(frame, {3.0f * std::cos(angle), 0.3f, 3.0f * std::sin(angle)}));
        }
        s.objects.push_back(box_obj("bunny-" + std::to_string(i), {0.2f, 0.3f, 0.2f},
                                    {0.75f, 0.7f, 0.65f}, kfs));
    }
    Light l = make_light(PRX_LIGHT_DISC_AREA, {120, 120, 120}, {kf_at(0, {0, 4.9f, 0}, down_facing())});
    l.radius = 0.6f;
    s.lights.push_back(l);
    s.camera = cam({0, 2.8f, 4.6f}, {0, 0.8f, 0}, 65.0f);
    return s;
}

Scene villa_analog() {
    Scene s;
    s.frames = 200;
    room(s, {8, 2, 4}, {0, 2, 0}, {0.65f, 0.62f, 0.58f});
    const V3 wall{0.6f, 0.6f, 0.6f};
    s.objects.push_back(box_obj("wall-a", {0.15f, 2, 1.7f}, wall, {kf_at(0, {0, 2, -2.3f})}));
    s.objects.push_back(box_obj("wall-b", {0.15f, 2, 1.7f}, wall, {kf_at(0, {0, 2, 2.3f})}));
    s.objects.push_back(box_obj("lintel", {0.15f, 0.75f, 0.6f}, wall, {kf_at(0, {0, 3.25f, 0})}));
    s.objects.push_back(box_obj("kitchen-table", {1, 0.4f, 0.6f}, {0.5f, 0.35f, 0.25f}, {kf_at(0, {-4, 0.4f, 0})}));
    s.objects.push_back(box_obj("cabinet", {0.5f, 0.75f, 0.5f}, {0.45f, 0.3f, 0.2f}, {kf_at(0, {-7, 0.75f, -2.5f})}));
    s.objects.push_back(box_obj("sofa", {1.2f, 0.4f, 0.5f}, {0.3f, 0.4f, 0.5f}, {kf_at(0, {4, 0.4f, 2})}));
    s.objects.push_back(box_obj("coffee-table", {0.6f, 0.3f, 0.6f}, {0.5f, 0.4f, 0.3f}, {kf_at(0, {5, 0.3f, -1})}));
    Light torch;
    torch.kind = PRX_LIGHT_DISC_AREA;
    torch.flux = {90, 90, 90};
    torch.radius = 0.25f;
    const Quat aim = rotation_z_to({1.0f, -1.0f, 0.0f});
    for (int k = 0; k <= 8; ++k) {
        const float angle = kTau * static_cast<float>(k) / 8.0f;
        const V3 pos{-4.0f + 1.5f * std::cos(angle), 1.8f, 1.2f * std::sin(angle)};
        torch.kfs.push_back(kf_at(k * 25, pos, aim));
    }
    s.lights.push_back(torch);
    s.camera = cam({5.5f, 1.8f, 3}, {0, 1.2f, 0}, 70.0f);
    return s;
}

// ---------------------------------------------------------------- procedural meshes
// A planar quad grid spanning origin + u*[0,1] + v*[0,1], nu x nv cells, 2 tris per cell.
void add_grid(std::vector<Tri>& out, V3 origin, V3 u, V3 v, int nu, int nv) {
    for (int j = 0; j < nv; ++j)
        for (int i = 0; i < nu; ++i) {
            const float u0 = static_cast<float>(i) / nu, u1 = static_cast<float>(i + 1) / nu;
            const float v0 = static_cast<float>(j) / nv, v1 = static_cast<float>(j + 1) / nv;
            const V3 p00 = add(origin, add(mul(u, u0), mul(v, v0)));
            const V3 p10 = add(origin, add(mul(u, u1), mul(v, v0)));
            const V3 p11 = add(origin, add(mul(u, u1), mul(v, v1)));
            const V3 p01 = add(origin, add(mul(u, u0), mul(v, v1)));
            out.push_back({p00, p10, p11});
            out.push_back({p00, p11, p01});
        }
}

// UV sphere: `slices` around, `stacks` from pole to pole; 2*slices*(stacks-1) triangles.
std::vector<Tri> uv_sphere(float r, int slices, int stacks) {
    std::vector<Tri> out;
    auto P = [&](int i, int j) {
        const float th = kPi * static_cast<float>(j) / stacks;
        const float ph = kTau * static_cast<float>(i % slices) / slices;
        return V3{r * std::sin(th) * std::cos(ph), r * std::cos(th), r * std::sin(th) * std::sin(ph)};
    };
    for (int j = 0; j < stacks; ++j)
        for (int i = 0; i < slices; ++i) {
            const V3 a = P(i, j), b = P(i + 1, j), c = P(i + 1, j + 1), d = P(i, j + 1);
            if (j != 0) out.push_back({a, b, c});
            if (j != stacks - 1) out.push_back({a, c, d});
        }
    return out;
}

// Open cylinder along +y (base at y=0) with end caps as fans.
void add_cylinder(std::vector<Tri>& out, V3 base, float r, float h, int seg, int rings) {
    auto P = [&](int i, float y) {
        const float ph = kTau * static_cast<float>(i % seg) / seg;
        return V3{base.x + r * std::cos(ph), base.y + y, base.z + r * std::sin(ph)};
    };
    for (int j = 0; j < rings; ++j) {
        const float y0 = h * static_cast<float>(j) / rings, y1 = h * static_cast<float>(j + 1) / rings;
        for (int i = 0; i < seg; ++i) {
            out.push_back({P(i, y0), P(i + 1, y0), P(i + 1, y1)});
            out.push_back({P(i, y0), P(i + 1, y1), P(i, y1)});
        }
    }
    const V3 top{base.x, base.y + h, base.z};
    for (int i = 0; i < seg; ++i) out.push_back({top, P(i + 1, h), P(i, h)});
}

// Half torus (an arch) in the plane spanned by x and y, centred at c.
void add_arch(std::vector<Tri>& out, V3 c, float R, float r, int seg, int tube) {
    auto P = [&](int i, int j) {
        const float a = kPi * static_cast<float>(i) / seg;          // 0..pi (half)
        const float b = kTau * static_cast<float>(j % tube) / tube;
        const float rr = R + r * std::cos(b);
        return V3{c.x + rr * std::cos(a), c.y + rr * std::sin(a), c.z + r * std::sin(b)};
    };
    for (int i = 0; i < seg; ++i)
        for (int j = 0; j < tube; ++j) {
            out.push_back({P(i, j), P(i + 1, j), P(i + 1, j + 1)});
            out.push_back({P(i, j), P(i + 1, j + 1), P(i, j + 1)});
        }
}

// Torus knot-ish blob for dynamic objects: a torus with given tessellation.
std::vector<Tri> torus(float R, float r, int seg, int tube) {
    std::vector<Tri> out;
    auto P = [&](int i, int j) {
        const float a = kTau * static_cast<float>(i % seg) / seg;
        const float b = kTau * static_cast<float>(j % tube) / tube;
        const float rr = R + r * std::cos(b);
        return V3{rr * std::cos(a), r * std::sin(b), rr * std::sin(a)};
    };
    for (int i = 0; i < seg; ++i)
        for (int j = 0; j < tube; ++j) {
            out.push_back({P(i, j), P(i + 1, j), P(i + 1, j + 1)});
            out.push_back({P(i, j), P(i + 1, j + 1), P(i, j + 1)});
        }
    return out;
}

Object mesh_obj(const std::string& name, std::vector<Tri> mesh, V3 albedo,
                std::vector<Keyframe> kfs = {}) {
    Object o;
    o.name = name;
    o.mesh = std::move(mesh);
    o.material.albedo = albedo;
    o.kfs = kfs.empty() ? std::vector<Keyframe>{kf_at(0, {0, 0, 0})} : std::move(kfs);
    return o;
}

int scaled(int n, float s) { return std::max(1, static_cast<int>(std::lround(n * s))); }

// Tessellated axis-aligned room shell [lo, hi]; `open_front` drops the +z wall.
void add_room_shell(Scene& s, V3 lo, V3 hi, int cells_per_unit, bool open_front, float ts) {
    const V3 e = sub(hi, lo);
    auto n = [&](float len) { return scaled(std::max(1, static_cast<int>(len * cells_per_unit)), ts); };
    const V3 white{0.75f, 0.75f, 0.75f};
    std::vector<Tri> floor_, ceil_, back, left, right, front;
    add_grid(floor_, lo, {e.x, 0, 0}, {0, 0, e.z}, n(e.x), n(e.z));
    add_grid(ceil_, {lo.x, hi.y, lo.z}, {e.x, 0, 0}, {0, 0, e.z}, n(e.x), n(e.z));
    add_grid(back, lo, {e.x, 0, 0}, {0, e.y, 0}, n(e.x), n(e.y));
    add_grid(left, lo, {0, 0, e.z}, {0, e.y, 0}, n(e.z), n(e.y));
    add_grid(right, {hi.x, lo.y, lo.z}, {0, 0, e.z}, {0, e.y, 0}, n(e.z), n(e.y));
    s.objects.push_back(mesh_obj("floor", floor_, white));
    s.objects.push_back(mesh_obj("ceiling", ceil_, white));
    s.objects.push_back(mesh_obj("back-wall", back, white));
    s.objects.push_back(mesh_obj("left-wall", left, {0.75f, 0.25f, 0.25f}));
    s.objects.push_back(mesh_obj("right-wall", right, {0.25f, 0.75f, 0.25f}));
    if (!open_front) {
        add_grid(front, {lo.x, lo.y, hi.z}, {e.x, 0, 0}, {0, e.y, 0}, n(e.x), n(e.y));
        s.objects.push_back(mesh_obj("front-wall", front, white));
    }
}

// Dynamic object tour: `n_keys` keyframes over `frames`, on an ellipse with spin.
std::vector<Keyframe> tour(V3 center, float rx, float rz, float phase, int frames, int n_keys,
                           float y_amp) {
    std::vector<Keyframe> k;
    for (int i = 0; i <= n_keys; ++i) {
        const int f = frames * i / n_keys;
        const float a = phase + kTau * static_cast<float>(i) / n_keys;
        const V3 p{center.x + rx * std::cos(a), center.y + y_amp * std::sin(2.0f * a),
                   center.z + rz * std::sin(a)};
        k.push_back(kf_at(f, p, quat_axis_angle({0.3f, 1.0f, 0.2f}, 0.5f * kTau * i / n_keys)));
    }
    return k;
}

// ---------------------------------------------------------------- C1 / C2: Cornell box
void cornell_base(Scene& s, float ts) {
    add_room_shell(s, {-1, 0, -1}, {1, 2, 1}, 5, /*open_front=*/true, ts);  // 5 walls x 200
    s.objects.push_back(box_obj("tall-block", {0.3f, 0.6f, 0.3f}, {0.75f, 0.75f, 0.75f},
                                {kf_at(0, {-0.35f, 0.6f, -0.3f}, quat_axis_angle({0, 1, 0}, 0.35f))}));
    s.objects.push_back(box_obj("short-block", {0.3f, 0.3f, 0.3f}, {0.75f, 0.75f, 0.75f},
                                {kf_at(0, {0.4f, 0.3f, 0.3f}, quat_axis_angle({0, 1, 0}, -0.3f))}));
    s.camera = cam({0, 1, 3.6f}, {0, 1, 0}, 40.0f);
    s.frames = 200;
}

Scene synth_c1(float ts) {
    Scene s;
    cornell_base(s, ts);
    // one UV sphere (31 x 17 -> 992 triangles) translating linearly
    s.objects.push_back(mesh_obj("sphere", uv_sphere(0.25f, 31, 17), {0.8f, 0.8f, 0.8f},
                                 {kf_at(0, {-0.55f, 1.2f, 0.2f}), kf_at(200, {0.55f, 1.2f, 0.2f})}));
    s.lights.push_back(make_light(PRX_LIGHT_POINT, {40, 40, 40}, {kf_at(0, {0, 1.95f, 0}, down_facing())}));
    return s;
}

Scene synth_c2(float ts) {
    Scene s;
    cornell_base(s, ts);
    s.objects.push_back(mesh_obj("sphere", uv_sphere(0.25f, 31, 17), {0.8f, 0.8f, 0.8f},
                                 {kf_at(0, {0.0f, 1.2f, 0.2f})}));
    Light l = make_light(PRX_LIGHT_RECT_AREA, {40, 40, 40},
                         {kf_at(0, {-0.4f, 1.98f, -0.2f}, down_facing()),
                          kf_at(200, {0.4f, 1.98f, 0.2f}, down_facing())});
    l.half_x = 0.25f;
    l.half_y = 0.25f;
    s.lights.push_back(l);
    return s;
}

// ---------------------------------------------------------------- C3 / C4 / C5: halls
// A colonnade hall: tessellated shell + two rows of columns joined by arches.
void hall(Scene& s, V3 lo, V3 hi, int cols_per_row, int col_seg, int col_rings, int arch_seg,
          int arch_tube, int shell_cells, float ts) {
    add_room_shell(s, lo, hi, shell_cells, /*open_front=*/false, ts);
    const float col_h = (hi.y - lo.y) * 0.75f;
    const float span = (hi.x - lo.x) * 0.8f;
    const float step = span / (cols_per_row - 1);
    std::vector<Tri> cols, arches;
    for (int row = 0; row < 2; ++row) {
        const float z = (row == 0 ? lo.z : hi.z) * 0.55f;
        for (int i = 0; i < cols_per_row; ++i) {
            const float x = -span / 2 + step * i;
            add_cylinder(cols, {x, lo.y, z}, 0.35f, col_h, scaled(col_seg, ts), scaled(col_rings, ts));
            if (i + 1 < cols_per_row)
                add_arch(arches, {x + step / 2, lo.y + col_h, z}, step / 2, 0.2f,
                         scaled(arch_seg, ts), scaled(arch_tube, ts));
        }
    }
    s.objects.push_back(mesh_obj("columns", cols, {0.7f, 0.68f, 0.62f}));
    s.objects.push_back(mesh_obj("arches", arches, {0.65f, 0.6f, 0.55f}));
}

void add_movers(Scene& s, int n, V3 lo, V3 hi, int frames) {
    const V3 c = mul(add(lo, hi), 0.5f);
    const V3 e = sub(hi, lo);
    for (int i = 0; i < n; ++i) {
        // ~20K triangles each: alternate spheres (100 x 101 -> 20,000) and tori (100 x 100)
        std::vector<Tri> mesh = (i % 2 == 0) ? uv_sphere(0.6f, 100, 101) : torus(0.6f, 0.22f, 100, 100);
        const float phase = kTau * static_cast<float>(i) / std::max(1, n);
        const float ring = 0.22f + 0.18f * static_cast<float>(i % 3);
        s.objects.push_back(mesh_obj("mover-" + std::to_string(i), std::move(mesh),
                                     {0.8f, 0.55f + 0.05f * (i % 4), 0.4f},
                                     tour({c.x, lo.y + 0.3f * e.y, c.z}, 0.5f * ring * e.x, 0.5f * ring * e.z, phase,
                                          frames, 8, 0.1f * e.y)));
    }
}

Scene synth_c3(float ts) {
    Scene s;
    s.frames = 200;
    const V3 lo{-10, 0, -5}, hi{10, 8, 5};
    // ~300K static triangles: shell (~60K) + 16 columns (~12.4K) + 14 arches (~1.5K)
    hall(s, lo, hi, 8, 64, 96, 48, 16, 6, ts);
    add_movers(s, 4, lo, hi, s.frames);
    Light l = make_light(PRX_LIGHT_DISC_AREA, {600, 600, 600}, {kf_at(0, {0, 7.9f, 0}, down_facing())});
    l.radius = 1.0f;
    s.lights.push_back(l);
    s.camera = cam({0, 3, 4.8f}, {0, 2.5f, 0}, 70.0f);
    return s;
}

Scene synth_c4_like(float ts, int n_dyn, const char* /*tag*/) {
    Scene s;
    s.frames = 200;
    const V3 lo{-20, 0, -10}, hi{20, 10, 10};
    // ~1M static triangles: shell (~330K) + 32 columns (~18.6K) + 30 arches (~2.3K)
    hall(s, lo, hi, 16, 96, 96, 72, 16, 8, ts);
    add_movers(s, n_dyn, lo, hi, s.frames);
    // two moving lights: a disc torch sweeping the hall and a rect panel sliding
    Light torch;
    torch.kind = PRX_LIGHT_DISC_AREA;
    torch.flux = {800, 760, 700};
    torch.radius = 0.35f;
    const Quat aim = rotation_z_to({0.4f, -1.0f, 0.2f});
    for (int k = 0; k <= 8; ++k) {
        const float a = kTau * static_cast<float>(k) / 8.0f;
        torch.kfs.push_back(kf_at(k * 25, {-8.0f + 4.0f * std::cos(a), 6.0f, 3.0f * std::sin(a)}, aim));
    }
    s.lights.push_back(torch);
    Light panel = make_light(PRX_LIGHT_RECT_AREA, {1200, 1200, 1200},
                             {kf_at(0, {-12.0f, 9.9f, 0}, down_facing()),
                              kf_at(200, {12.0f, 9.9f, 0}, down_facing())});
    panel.half_x = 1.5f;
    panel.half_y = 1.0f;
    s.lights.push_back(panel);
    s.camera = cam({0, 4, 9.5f}, {0, 3, 0}, 70.0f);
    return s;
}

}  // namespace

bool is_builtin_scene(const std::string& name) {
    return name == "static-box" || name == "moving-cube" || name == "parallel-spot" ||
           name == "merry-go-round-analog" || name == "armadillo-analog" ||
           name == "villa-analog" || name == "villa-torch";
}

Scene make_builtin_scene(const std::string& name) {
    Scene s;
    if (name == "static-box") s = static_box();
    else if (name == "moving-cube") s = moving_cube();
    else if (name == "parallel-spot") s = parallel_spot();
    else if (name == "merry-go-round-analog") s = merry_go_round();
    else if (name == "armadillo-analog") s = armadillo_analog();
    else if (name == "villa-analog" || name == "villa-torch") s = villa_analog();
    else throw SceneError("unknown builtin scene: " + name);
    finalize_scene(s);
    return s;
}

Scene make_synthetic_scene(const std::string& name, uint32_t n_dynamic, float tri_scale) {
    const float ts = tri_scale > 0.0f ? tri_scale : 1.0f;
    Scene s;
    if (name == "C1") s = synth_c1(ts);
    else if (name == "C2") s = synth_c2(ts);
    else if (name == "C3") s = synth_c3(ts);
    else if (name == "C4") s = synth_c4_like(ts, n_dynamic ? static_cast<int>(n_dynamic) : 8, "C4");
    else if (name == "C5") s = synth_c4_like(ts, n_dynamic ? static_cast<int>(n_dynamic) : 16, "C5");
    else throw SceneError("unknown synthetic scene: " + name);
    finalize_scene(s);
    return s;
}

}  // namespace prx
