// The reference's own call patterns against the C++ drop-in (include/pathreuse_b200.hpp):
//   gather_image(engine.scene_state(), engine.photon_map(), engine.vertex_aux(), cam, r, w)
//     (tools/pathreuse_cli.cpp:93, tests/acceptance/acceptance.cpp:58, test_gather.cpp:68)
//   segment_origin / segment_end / segment_count (test_engine.cpp:101-120, acceptance.cpp:206-208)
//   scene_state().placed_dynamics, dm_layout(li), dm_target/dm_current by const&
//   select_paths_to_prune(span, dm_c, dm_t, seed, frame) (test_light_dm.cpp:194-201)
// usage: dropin_reference_calls <scene> <mode> <frames>; prints one "key value..." per line.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>

#include "pathreuse_b200.hpp"

using namespace pathreuse;

static uint64_t fnv(const void* p, size_t n) {
    uint64_t h = 1469598103934665603ull;
    const unsigned char* b = static_cast<const unsigned char*>(p);
    for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
    return h;
}

int main(int argc, char** argv) {
    const char* scene_name = argc > 1 ? argv[1] : "moving-cube";
    EngineConfig cfg;
    cfg.mode = engine_mode_from_string(argc > 2 ? argv[2] : "error");
    const int frames = argc > 3 ? std::atoi(argv[3]) : 3;
    cfg.n_paths = 6000;
    cfg.max_bounces = 5;
    cfg.dm_dims = {1, 1, 8, 8};
    cfg.seed = 7;
    Engine engine(make_builtin_scene(scene_name), cfg);
    for (int f = 0; f < frames; ++f) engine.run_frame();

    // gather_image with the reference signature: the engine's own mirrors ...
    const Camera& cam = engine.scene().camera;
    const Image a = gather_image(engine.scene_state(), engine.photon_map(), engine.vertex_aux(), cam,
                                 cfg.gather_radius, 4);
    std::printf("image %llu\n", (unsigned long long)fnv(a.pixels.data(), a.pixels.size() * 4));
    // ... and a host copy of them (uploaded and splatted through prx_gather_photons)
    const PhotonMap copy = engine.photon_map();
    const std::vector<PathVertexAux> aux_copy = engine.vertex_aux();
    const Image b = gather_image(engine.scene_state(), copy, aux_copy, cam, cfg.gather_radius, 4);
    std::printf("image_host %llu\n", (unsigned long long)fnv(b.pixels.data(), b.pixels.size() * 4));

    // segments (test_engine.cpp:101-120): the incoming direction matches the chord
    uint64_t segs = 0, bad_chord = 0, bad_end = 0;
    for (uint32_t p = 0; p < engine.total_paths(); ++p) {
        if (!engine.path_alive(p)) continue;
        const uint32_t k = engine.photon_count(p);
        for (uint32_t i = 0; i < engine.segment_count(p); ++i) {
            const Vec3 from = engine.segment_origin(p, i), to = engine.segment_end(p, i);
            ++segs;
            if (i < k) {
                const Vec3 d = to - from;
                const float len = std::sqrt(d.x * d.x + d.y * d.y + d.z * d.z);
                const Vec3 s = engine.photon_map().at(i, p).incoming_dir;
                const float c = (d.x * s.x + d.y * s.y + d.z * s.z) / len;
                if (!(std::fabs(c - 1.0f) <= 1e-3f)) ++bad_chord;
                if (!(to == engine.aux_at(i, p).position)) ++bad_end;
            }
            if (i + 1 < engine.segment_count(p) && !(engine.segment_origin(p, i + 1) == to)) ++bad_end;
        }
    }
    std::printf("segments %llu %llu %llu\n", (unsigned long long)segs, (unsigned long long)bad_chord,
                (unsigned long long)bad_end);

    // scene state: frame, dynamic objects, their triangles, bounds containing the triangles
    const SceneState& st = engine.scene_state();
    size_t tris = 0, outside = 0;
    for (const PlacedDynamic& pd : st.placed_dynamics) {
        tris += pd.triangles.size();
        for (const Triangle& t : pd.triangles)
            for (const Vec3& v : {t.a, t.b, t.c})
                if (v.x < pd.bounds_current.lo.x || v.y < pd.bounds_current.lo.y || v.z < pd.bounds_current.lo.z ||
                    v.x > pd.bounds_current.hi.x || v.y > pd.bounds_current.hi.y || v.z > pd.bounds_current.hi.z)
                    ++outside;
    }
    std::printf("state %d %zu %zu %zu\n", st.frame, st.placed_dynamics.size(), tris, outside);

    // distribution maps by const reference, with their layouts
    for (size_t li = 0; li < engine.light_count(); ++li) {
        const DmLayout& lay = engine.dm_layout(li);
        const DistributionMap& t = engine.dm_target(li);
        const DistributionMap& c = engine.dm_current(li);
        std::printf("dm %zu %u %zu %llu %llu\n", li, lay.total_cells(), t.counts.size(),
                    (unsigned long long)t.total(), (unsigned long long)c.total());
    }

    // select_paths_to_prune (test_light_dm.cpp:194-201)
    std::vector<uint32_t> paths(1000);
    std::iota(paths.begin(), paths.end(), 100u);
    const std::vector<uint32_t> pr = select_paths_to_prune(paths, 1000, 600, 5, 3);
    std::printf("prune %zu", pr.size());
    for (uint32_t v : pr) std::printf(" %u", v);
    std::printf("\n");
    std::vector<uint32_t> exact(600);
    std::iota(exact.begin(), exact.end(), 0u);
    std::printf("prune_exact %zu\n", select_paths_to_prune(exact, 600, 600, 5, 3).size());

    // the same frames on a 2-shard MultiGpuEngine (both shards on device 0)
    MultiGpuEngine multi(make_builtin_scene(scene_name), cfg, {0, 0});
    for (int f = 0; f < frames; ++f) {
        const FrameStats s = multi.run_frame();
        std::printf("group %d %llu %llu %llu %llu %llu\n", s.frame, (unsigned long long)s.rays_traced,
                    (unsigned long long)s.rays_reused, (unsigned long long)s.paths_pruned,
                    (unsigned long long)s.paths_filled, (unsigned long long)s.visibility_rays);
    }
    return 0;
}
