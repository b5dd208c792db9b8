// host_scene.h -- host-side scene model of the B200 engine.
//
// Holds what the reference keeps in pathreuse::Scene (scene.hpp:47-60) and the host-only
// math that produces per-frame placements (transform.hpp, animation.hpp, light.cpp:58-68).
// The per-frame triangle placement itself runs on the GPU (engine kernels); this file
// only evaluates keyframes (a handful of slerps per frame) and builds the static BVH once
// at scene load.  All arithmetic follows the reference's operation order so the values
// fed to the device are bit-identical to the reference's.
#pragma once

#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "exact_math.h"
#include "prx.h"

namespace prx {

struct SceneError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

struct Quat {
    float x = 0.0f, y = 0.0f, z = 0.0f, w = 1.0f;
};
bool operator==(const Quat& a, const Quat& b);
float quat_norm(const Quat& q);                       // transform.hpp:17
Quat quat_normalized(const Quat& q);                  // transform.hpp:19-22
Quat quat_axis_angle(V3 axis, float radians);         // transform.hpp:26-30
V3 rotate(const Quat& q, V3 v);                       // transform.hpp:33-37
Quat slerp(const Quat& a, Quat b, float t);           // transform.hpp:43-61

struct Xform {
    Quat rot;
    V3 trans{0.0f, 0.0f, 0.0f};
    float scale = 1.0f;
};
bool operator==(const Xform& a, const Xform& b);
V3 apply_point(const Xform& xf, V3 p);                // transform.hpp:72
Xform interpolate(const Xform& a, const Xform& b, float t);  // transform.hpp:79-85
Box transform_box(const Box& box, const Xform& xf);   // transform.hpp:88-96

struct Keyframe {
    int frame = 0;
    Xform xf;
};
Xform transform_at(const std::vector<Keyframe>& kfs, int frame);  // animation.hpp:13-28
bool has_distinct(const std::vector<Keyframe>& kfs);               // animation.hpp:31-36

struct Tri {
    V3 a, b, c;
};
Box tri_bounds(const Tri& t);
V3 tri_centroid(const Tri& t);
float tri_area(const Tri& t);

struct Material {
    int kind = PRX_MATERIAL_DIFFUSE;
    V3 albedo{0.5f, 0.5f, 0.5f};
    float glossy_exponent = 1.0f;
};

struct Object {
    uint32_t id = 0;
    std::string name;
    std::vector<Tri> mesh;  // object-local
    Material material;
    std::vector<Keyframe> kfs;
    bool dynamic = false;
    Box local_bounds = empty_box();
};

struct Light {
    int kind = PRX_LIGHT_POINT;
    V3 flux{0.0f, 0.0f, 0.0f};
    float cone_angle_deg = 60.0f;
    float radius = 1.0f;
    float half_x = 1.0f, half_y = 1.0f;
    std::vector<Keyframe> kfs;
    bool is_area() const { return kind == PRX_LIGHT_DISC_AREA || kind == PRX_LIGHT_RECT_AREA; }
    int param_dims() const { return is_area() ? 4 : 2; }
};

struct LightPose {
    V3 position{0, 0, 0}, normal{0, 0, 0}, tangent{0, 0, 0}, bitangent{0, 0, 0};
    float scale = 1.0f;
};
bool operator==(const LightPose& a, const LightPose& b);
LightPose light_pose_at(const Light& light, int frame);  // light.cpp:58-68

struct Camera {
    V3 position{0, 1, 4};
    V3 look_at{0, 1, 0};
    float fov_deg = 60.0f;
    uint32_t width = 120, height = 90;
};

// Median-split static BVH node, identical in layout semantics to Bvh::Node (bvh.hpp:15-21):
// internal nodes: left child `left`, right child `first`; leaves: `count` triangles
// starting at `first` in the permutation.
struct BvhNode {
    Box bounds;
    uint32_t left = 0;
    uint32_t first = 0;
    uint16_t count = 0;
    uint16_t axis = 0;
};

struct Scene {
    std::vector<Object> objects;
    std::vector<Light> lights;
    Camera camera;
    int frames = 1;

    // finalize products (scene.cpp:90-112)
    std::vector<Tri> static_tris;           // world space, original order
    std::vector<uint32_t> static_tri_obj;   // object id per static triangle
    Box world_bounds = empty_box();
    std::vector<BvhNode> bvh_nodes;
    std::vector<uint32_t> bvh_perm;          // permutation of static triangle indices
    float diagonal() const { return length(sub(world_bounds.hi, world_bounds.lo)); }

    // C-ABI description view (prx_scene_describe)
    std::vector<std::vector<prx_triangle>> desc_meshes;
    std::vector<std::vector<prx_keyframe>> desc_obj_kfs, desc_light_kfs;
    std::vector<prx_object_desc> desc_objects;
    std::vector<prx_light_desc> desc_lights;
};

void validate_light(const Light& light);   // light.cpp:254-269 (std::invalid_argument)
void finalize_scene(Scene& scene);         // scene.cpp:63-113 (SceneError)
void build_static_bvh(Scene& scene);       // bvh.cpp:13-77
Scene scene_from_desc(const prx_scene_desc& d);
void fill_desc_views(Scene& scene);
std::vector<Tri> make_box_mesh(V3 half);   // scene.cpp:16-28
Scene make_builtin_scene(const std::string& name);  // scene.cpp:603-611
bool is_builtin_scene(const std::string& name);
Scene make_synthetic_scene(const std::string& name, uint32_t n_dynamic, float tri_scale);

// scene documents (scene_io.cpp; scene.cpp:179-398)
std::vector<Tri> load_obj_mesh(const std::string& path);
Scene load_scene_text(const std::string& json_text, const std::string& base_dir);
Scene load_scene_file(const std::string& path);
Scene load_scene_source(const std::string& source);  // "builtin:NAME", a builtin name, or a file

}  // namespace prx
