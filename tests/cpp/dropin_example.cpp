// A reference-style program against the drop-in C++ surface (include/pathreuse_b200.hpp):
// the same calls a proj/tools or proj/tests user makes on pathreuse::Engine.
// Prints one line per frame: "frame traced reused replaced pruned filled vis"
// and, with --check, exits non-zero if the reference's invariants do not hold.
#include <cstdio>
#include <cstring>

#include "pathreuse_b200.hpp"

using namespace pathreuse;

int main(int argc, char** argv) {
    const char* scene_name = argc > 1 ? argv[1] : "moving-cube";
    EngineConfig cfg;
    cfg.mode = engine_mode_from_string(argc > 2 ? argv[2] : "error");
    cfg.n_paths = 5000;
    cfg.dm_dims = {1, 1, 8, 8};
    cfg.seed = 11;
    Engine engine(make_builtin_scene(scene_name), cfg);
    int bad = 0;
    for (int f = 0; f < 5; ++f) {
        const FrameStats s = engine.run_frame();
        std::printf("%d %llu %llu %llu %llu %llu %llu\n", s.frame, (unsigned long long)s.rays_traced,
                    (unsigned long long)s.rays_reused, (unsigned long long)s.paths_replaced,
                    (unsigned long long)s.paths_pruned, (unsigned long long)s.paths_filled,
                    (unsigned long long)s.visibility_rays);
        // test_engine.cpp:143-153: traced + reused == stored segments
        uint64_t segs = 0;
        for (uint32_t p = 0; p < engine.total_paths(); ++p)
            if (engine.path_alive(p)) segs += engine.segment_count(p);
        if (segs != s.rays_traced + s.rays_reused) ++bad;
        // test_engine.cpp:228-238: path info mirrors the state
        for (uint32_t p = 0; p < engine.total_paths(); ++p) {
            if (!engine.path_alive(p)) continue;
            const PathInfoFields fi = decode_path_info(engine.path_info_words()[p]);
            if (fi.cell != engine.path_cell(p) || fi.replace) ++bad;
        }
        // test_engine.cpp:101-120: live records exactly below the photon count
        for (uint32_t p = 0; p < engine.total_paths(); ++p) {
            if (!engine.path_alive(p)) continue;
            for (uint32_t b = 0; b < cfg.max_bounces; ++b)
                if (engine.photon_map().at(b, p).live() != (b < engine.photon_count(p))) ++bad;
        }
    }
    const Image img = gather_image(engine, engine.scene().camera, cfg.gather_radius);
    bool lit = false;
    for (float v : img.pixels) lit = lit || v > 0.0f;
    if (!lit) ++bad;
    if (argc > 3 && std::strcmp(argv[3], "--check") == 0 && bad) {
        std::fprintf(stderr, "%d invariant violations\n", bad);
        return 1;
    }
    return 0;
}
