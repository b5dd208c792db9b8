// scene_io.cpp -- scene documents (JSON + OBJ meshes) for the GPU scene build.
//
// Behaviour follows the reference loader, scene.cpp:179-398:
//   * document keys {objects, lights, camera, frames}; unknown keys are a SceneError;
//   * numbers are read as double (strtod) and narrowed like nlohmann::json::get<T>()
//     (static_cast), so every float lands on the same bits as in the reference;
//   * OBJ: `v x y z` via stream extraction (the reference's `ls >> p.x`), `f` with
//     "i", "i/..", "i//.." tokens (std::stoi of the part before '/'), negative indices
//     relative to the end, fan triangulation (0, i-1, i); any other statement is an error;
//   * `builtin:NAME` or a bare builtin name selects a builtin (scene.cpp:392-398).
// The parsed scene then goes through finalize_scene like every other source.
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <utility>
#include <vector>

#include "host_scene.h"

namespace prx {

namespace {

// ------------------------------------------------------------------ minimal JSON DOM
struct JVal {
    enum Kind { Null, Bool, Num, Str, Arr, Obj } kind = Null;
    bool b = false;
    double num = 0.0;
    bool integral = false;   // written without fraction/exponent
    long long ival = 0;      // exact value when integral
    std::string str;
    std::vector<JVal> arr;
    std::vector<std::pair<std::string, JVal>> obj;  // document order

    const JVal* find(const std::string& key) const {
        const JVal* hit = nullptr;
        for (const auto& kv : obj)
            if (kv.first == key) hit = &kv.second;  // a repeated key keeps the last value
        return hit;
    }
};

class Parser {
public:
    explicit Parser(const std::string& text) : s_(text) {}

    JVal document() {
        JVal v = value();
        ws();
        if (p_ != s_.size()) error("trailing characters");
        return v;
    }

private:
    const std::string& s_;
    size_t p_ = 0;

    [[noreturn]] void error(const std::string& what) const {
        throw SceneError("scene parse error: " + what + " at byte " + std::to_string(p_));
    }
    void ws() {
        while (p_ < s_.size() && (s_[p_] == ' ' || s_[p_] == '\t' || s_[p_] == '\n' || s_[p_] == '\r')) ++p_;
    }
    bool lit(const char* w) {
        const size_t n = std::strlen(w);
        if (s_.compare(p_, n, w) == 0) {
            p_ += n;
            return true;
        }
        return false;
    }
    JVal value() {
        ws();
        if (p_ >= s_.size()) error("unexpected end of input");
        const char c = s_[p_];
        JVal v;
        if (c == '{') {
            v.kind = JVal::Obj;
            ++p_;
            ws();
            if (p_ < s_.size() && s_[p_] == '}') {
                ++p_;
                return v;
            }
            while (true) {
                ws();
                if (p_ >= s_.size() || s_[p_] != '"') error("expected a key string");
                std::string key = string();
                ws();
                if (p_ >= s_.size() || s_[p_] != ':') error("expected ':'");
                ++p_;
                v.obj.emplace_back(std::move(key), value());
                ws();
                if (p_ < s_.size() && s_[p_] == ',') {
                    ++p_;
                    continue;
                }
                if (p_ < s_.size() && s_[p_] == '}') {
                    ++p_;
                    return v;
                }
                error("expected ',' or '}'");
            }
        }
        if (c == '[') {
            v.kind = JVal::Arr;
            ++p_;
            ws();
            if (p_ < s_.size() && s_[p_] == ']') {
                ++p_;
                return v;
            }
            while (true) {
                v.arr.push_back(value());
                ws();
                if (p_ < s_.size() && s_[p_] == ',') {
                    ++p_;
                    continue;
                }
                if (p_ < s_.size() && s_[p_] == ']') {
                    ++p_;
                    return v;
                }
                error("expected ',' or ']'");
            }
        }
        if (c == '"') {
            v.kind = JVal::Str;
            v.str = string();
            return v;
        }
        if (lit("true")) {
            v.kind = JVal::Bool;
            v.b = true;
            return v;
        }
        if (lit("false")) {
            v.kind = JVal::Bool;
            return v;
        }
        if (lit("null")) return v;
        return number();
    }
    unsigned hex4(size_t at) const {
        if (at + 4 > s_.size()) error("bad \\u escape");
        unsigned v = 0;
        for (size_t k = at; k < at + 4; ++k) {
            const char c = s_[k];
            const int d = (c >= '0' && c <= '9') ? c - '0' : (c >= 'a' && c <= 'f') ? c - 'a' + 10
                        : (c >= 'A' && c <= 'F') ? c - 'A' + 10 : -1;
            if (d < 0) error("bad \\u escape");
            v = v * 16 + static_cast<unsigned>(d);
        }
        return v;
    }
    std::string string() {
        ++p_;  // opening quote
        std::string out;
        while (true) {
            if (p_ >= s_.size()) error("unterminated string");
            const char c = s_[p_++];
            if (c == '"') return out;
            if (static_cast<unsigned char>(c) < 0x20) error("control character in string");
            if (c != '\\') {
                out.push_back(c);
                continue;
            }
            if (p_ >= s_.size()) error("unterminated escape");
            const char e = s_[p_++];
            switch (e) {
                case '"': out.push_back('"'); break;
                case '\\': out.push_back('\\'); break;
                case '/': out.push_back('/'); break;
                case 'b': out.push_back('\b'); break;
                case 'f': out.push_back('\f'); break;
                case 'n': out.push_back('\n'); break;
                case 'r': out.push_back('\r'); break;
                case 't': out.push_back('\t'); break;
                case 'u': {
                    unsigned cp = hex4(p_);
                    p_ += 4;
                    if (cp >= 0xD800 && cp < 0xDC00 && p_ + 6 <= s_.size() && s_[p_] == '\\' && s_[p_ + 1] == 'u') {
                        const unsigned lo = hex4(p_ + 2);
                        p_ += 6;
                        cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
                    }
                    if (cp < 0x80) {
                        out.push_back(static_cast<char>(cp));
                    } else if (cp < 0x800) {
                        out.push_back(static_cast<char>(0xC0 | (cp >> 6)));
                        out.push_back(static_cast<char>(0x80 | (cp & 0x3F)));
                    } else if (cp < 0x10000) {
                        out.push_back(static_cast<char>(0xE0 | (cp >> 12)));
                        out.push_back(static_cast<char>(0x80 | ((cp >> 6) & 0x3F)));
                        out.push_back(static_cast<char>(0x80 | (cp & 0x3F)));
                    } else {
                        out.push_back(static_cast<char>(0xF0 | (cp >> 18)));
                        out.push_back(static_cast<char>(0x80 | ((cp >> 12) & 0x3F)));
                        out.push_back(static_cast<char>(0x80 | ((cp >> 6) & 0x3F)));
                        out.push_back(static_cast<char>(0x80 | (cp & 0x3F)));
                    }
                    break;
                }
                default: error("bad escape");
            }
        }
    }
    JVal number() {
        const size_t b = p_;
        if (p_ < s_.size() && s_[p_] == '-') ++p_;
        auto digits = [&] {
            const size_t d = p_;
            while (p_ < s_.size() && s_[p_] >= '0' && s_[p_] <= '9') ++p_;
            return p_ - d;
        };
        if (digits() == 0) error("invalid literal");
        bool integral = true;
        if (p_ < s_.size() && s_[p_] == '.') {
            ++p_;
            if (digits() == 0) error("invalid number");
            integral = false;
        }
        if (p_ < s_.size() && (s_[p_] == 'e' || s_[p_] == 'E')) {
            ++p_;
            if (p_ < s_.size() && (s_[p_] == '+' || s_[p_] == '-')) ++p_;
            if (digits() == 0) error("invalid exponent");
            integral = false;
        }
        JVal v;
        v.kind = JVal::Num;
        const std::string tok = s_.substr(b, p_ - b);
        v.num = std::strtod(tok.c_str(), nullptr);
        v.integral = integral;
        if (integral) v.ival = std::strtoll(tok.c_str(), nullptr, 10);
        return v;
    }
};

// nlohmann get<T>() narrowing: integers convert from their exact value, floats by static_cast
float as_float(const JVal& v, const std::string& where) {
    if (v.kind != JVal::Num) throw SceneError(where + ": expected a number");
    return v.integral ? static_cast<float>(v.ival) : static_cast<float>(v.num);
}
long long as_int(const JVal& v, const std::string& where) {
    if (v.kind != JVal::Num) throw SceneError(where + ": expected a number");
    return v.integral ? v.ival : static_cast<long long>(v.num);
}
const std::string& as_string(const JVal& v, const std::string& where) {
    if (v.kind != JVal::Str) throw SceneError(where + ": expected a string");
    return v.str;
}
const JVal& at(const JVal& node, const char* key, const std::string& where) {
    const JVal* v = node.kind == JVal::Obj ? node.find(key) : nullptr;
    if (!v) throw SceneError(where + ": missing key '" + key + "'");
    return *v;
}
const JVal& as_array(const JVal& v, const std::string& where) {
    if (v.kind != JVal::Arr) throw SceneError(where + ": expected an array");
    return v;
}

void allow_keys(const JVal& node, std::initializer_list<const char*> keys, const std::string& where) {
    if (node.kind != JVal::Obj) throw SceneError(where + ": expected an object");
    for (const auto& kv : node.obj) {
        bool ok = false;
        for (const char* k : keys) ok = ok || kv.first == k;
        if (!ok) throw SceneError(where + ": unknown key '" + kv.first + "'");
    }
}

V3 vec3(const JVal& v, const std::string& where) {
    if (v.kind != JVal::Arr || v.arr.size() != 3) throw SceneError(where + ": expected an array of 3 numbers");
    return {as_float(v.arr[0], where), as_float(v.arr[1], where), as_float(v.arr[2], where)};
}

std::vector<Keyframe> keyframes(const JVal& node, const std::string& where) {
    std::vector<Keyframe> out;
    for (size_t i = 0; i < as_array(node, where + ".keyframes").arr.size(); ++i) {
        const JVal& kf = node.arr[i];
        const std::string kw = where + ".keyframes[" + std::to_string(i) + "]";
        allow_keys(kf, {"frame", "translation", "rotation", "scale"}, kw);
        Keyframe k;
        k.frame = static_cast<int>(as_int(at(kf, "frame", kw), kw));
        if (const JVal* t = kf.find("translation")) k.xf.trans = vec3(*t, kw);
        if (const JVal* q = kf.find("rotation")) {
            if (q->kind != JVal::Arr || q->arr.size() != 4) throw SceneError(kw + ": rotation expects [x, y, z, w]");
            k.xf.rot = {as_float(q->arr[0], kw), as_float(q->arr[1], kw), as_float(q->arr[2], kw),
                        as_float(q->arr[3], kw)};
        }
        if (const JVal* s = kf.find("scale")) k.xf.scale = as_float(*s, kw);
        out.push_back(k);
    }
    return out;
}

Material material(const JVal& node, const std::string& where) {
    allow_keys(node, {"kind", "albedo", "glossy_exponent"}, where);
    Material m;
    const std::string& kind = as_string(at(node, "kind", where), where);
    if (kind == "diffuse") m.kind = PRX_MATERIAL_DIFFUSE;
    else if (kind == "glossy") m.kind = PRX_MATERIAL_GLOSSY;
    else throw SceneError(where + ": material kind must be 'diffuse' or 'glossy'");
    m.albedo = vec3(at(node, "albedo", where), where + ".albedo");
    if (const JVal* e = node.find("glossy_exponent")) m.glossy_exponent = as_float(*e, where);
    return m;
}

}  // namespace

// OBJ subset of scene.cpp:225-265 (positions and faces only).
std::vector<Tri> load_obj_mesh(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw SceneError("missing mesh file: " + path);
    std::vector<V3> pos;
    std::vector<Tri> tris;
    std::string line;
    int line_no = 0;
    while (std::getline(in, line)) {
        ++line_no;
        const std::string at_line = path + ":" + std::to_string(line_no);
        std::istringstream ls(line);
        std::string tag;
        if (!(ls >> tag) || tag == "#") continue;
        if (tag == "v") {
            V3 p;
            if (!(ls >> p.x >> p.y >> p.z)) throw SceneError(at_line + ": bad vertex");
            pos.push_back(p);
            continue;
        }
        if (tag != "f") throw SceneError(at_line + ": unsupported OBJ statement '" + tag + "'");
        std::vector<int> idx;
        for (std::string tok; ls >> tok;) idx.push_back(std::stoi(tok.substr(0, tok.find('/'))));
        if (idx.size() < 3) throw SceneError(at_line + ": face needs 3+ vertices");
        auto vtx = [&](int i) -> V3 {
            const long long v = i > 0 ? i - 1 : static_cast<long long>(pos.size()) + i;
            if (v < 0 || v >= static_cast<long long>(pos.size()))
                throw SceneError(at_line + ": face index out of range");
            return pos[static_cast<size_t>(v)];
        };
        for (size_t k = 2; k < idx.size(); ++k) tris.push_back({vtx(idx[0]), vtx(idx[k - 1]), vtx(idx[k])});
    }
    if (tris.empty()) throw SceneError(path + ": no faces");
    return tris;
}

// scene.cpp:272-379
Scene load_scene_text(const std::string& text, const std::string& base_dir) {
    const JVal doc = Parser(text).document();
    allow_keys(doc, {"objects", "lights", "camera", "frames"}, "document");
    Scene scene;
    if (const JVal* f = doc.find("frames")) scene.frames = static_cast<int>(as_int(*f, "frames"));

    const JVal& cam = at(doc, "camera", "document");
    allow_keys(cam, {"position", "look_at", "fov", "resolution"}, "camera");
    scene.camera.position = vec3(at(cam, "position", "camera"), "camera.position");
    scene.camera.look_at = vec3(at(cam, "look_at", "camera"), "camera.look_at");
    scene.camera.fov_deg = as_float(at(cam, "fov", "camera"), "camera.fov");
    const JVal& res = at(cam, "resolution", "camera");
    if (res.kind != JVal::Arr || res.arr.size() != 2) throw SceneError("camera.resolution: expected [width, height]");
    scene.camera.width = static_cast<uint32_t>(as_int(res.arr[0], "camera.resolution"));
    scene.camera.height = static_cast<uint32_t>(as_int(res.arr[1], "camera.resolution"));

    const JVal& objects = as_array(at(doc, "objects", "document"), "objects");
    for (size_t i = 0; i < objects.arr.size(); ++i) {
        const JVal& node = objects.arr[i];
        const std::string where = "objects[" + std::to_string(i) + "]";
        allow_keys(node, {"name", "material", "mesh", "keyframes"}, where);
        Object obj;
        const JVal* name = node.find("name");
        obj.name = name ? as_string(*name, where + ".name") : where;
        obj.material = material(at(node, "material", where), where + ".material");
        const JVal& mesh = at(node, "mesh", where);
        if (mesh.kind == JVal::Obj && mesh.find("obj")) {
            allow_keys(mesh, {"obj"}, where + ".mesh");
            std::string path = as_string(*mesh.find("obj"), where + ".mesh.obj");
            if (!base_dir.empty() && !path.empty() && path[0] != '/') path = base_dir + "/" + path;
            obj.mesh = load_obj_mesh(path);
        } else {
            allow_keys(mesh, {"vertices", "faces"}, where + ".mesh");
            std::vector<V3> verts;
            for (const JVal& v : as_array(at(mesh, "vertices", where + ".mesh"), where + ".mesh.vertices").arr)
                verts.push_back(vec3(v, where + ".mesh.vertices"));
            for (const JVal& f : as_array(at(mesh, "faces", where + ".mesh"), where + ".mesh.faces").arr) {
                if (f.kind != JVal::Arr || f.arr.size() != 3)
                    throw SceneError(where + ".mesh.faces: expected index triples");
                V3 c[3];
                for (int k = 0; k < 3; ++k) {
                    const size_t idx = static_cast<size_t>(as_int(f.arr[k], where + ".mesh.faces"));
                    if (idx >= verts.size()) throw SceneError(where + ".mesh.faces: index out of range");
                    c[k] = verts[idx];
                }
                obj.mesh.push_back({c[0], c[1], c[2]});
            }
        }
        if (const JVal* kf = node.find("keyframes")) obj.kfs = keyframes(*kf, where);
        scene.objects.push_back(std::move(obj));
    }

    const JVal& lights = as_array(at(doc, "lights", "document"), "lights");
    for (size_t i = 0; i < lights.arr.size(); ++i) {
        const JVal& node = lights.arr[i];
        const std::string where = "lights[" + std::to_string(i) + "]";
        allow_keys(node, {"kind", "flux", "cone_angle", "radius", "half_extents", "keyframes"}, where);
        Light light;
        const std::string& kind = as_string(at(node, "kind", where), where + ".kind");
        if (kind == "point") light.kind = PRX_LIGHT_POINT;
        else if (kind == "spot") light.kind = PRX_LIGHT_SPOT;
        else if (kind == "disc_area") light.kind = PRX_LIGHT_DISC_AREA;
        else if (kind == "rect_area") light.kind = PRX_LIGHT_RECT_AREA;
        else throw SceneError(where + ": unknown light kind '" + kind + "'");
        light.flux = vec3(at(node, "flux", where), where + ".flux");
        if (const JVal* c = node.find("cone_angle")) light.cone_angle_deg = as_float(*c, where);
        if (const JVal* r = node.find("radius")) light.radius = as_float(*r, where);
        if (const JVal* he = node.find("half_extents")) {
            if (he->kind != JVal::Arr || he->arr.size() != 2)
                throw SceneError(where + ".half_extents: expected [hx, hy]");
            light.half_x = as_float(he->arr[0], where);
            light.half_y = as_float(he->arr[1], where);
        }
        if (const JVal* kf = node.find("keyframes")) light.kfs = keyframes(*kf, where);
        scene.lights.push_back(std::move(light));
    }
    finalize_scene(scene);
    return scene;
}

// scene.cpp:381-390
Scene load_scene_file(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw SceneError("cannot open scene file: " + path);
    std::stringstream buf;
    buf << in.rdbuf();
    const size_t slash = path.find_last_of('/');
    return load_scene_text(buf.str(), slash == std::string::npos ? "" : path.substr(0, slash));
}

// scene.cpp:392-398
Scene load_scene_source(const std::string& source) {
    const std::string prefix = "builtin:";
    if (source.rfind(prefix, 0) == 0) return make_builtin_scene(source.substr(prefix.size()));
    if (is_builtin_scene(source)) return make_builtin_scene(source);
    return load_scene_file(source);
}

}  // namespace prx
