// pathreuse_cli -- the reference's command line (tools/pathreuse_cli.cpp:120-171) over the
// B200 engine, written against the C++ drop-in header (include/pathreuse_b200.hpp).
//
//   pathreuse_cli [--scene S] [--mode baseline|naive|error] [--paths N] [--bounces B]
//                 [--dm AxBxCxD] [--threshold T] [--frames F] [--seed S] [--radius R]
//                 [--out DIR] [--images on|off] [--workers W] [--dump-photons FILE]
//   pathreuse_cli report STATS.csv...
//
// Same flags, defaults, outputs (DIR/config.json, DIR/frame_NNNN.ppm, DIR/stats.csv, the
// optional PHM1 dump, one progress line per frame) and exit codes: 0 ok, 1 scene/run
// error, 2 command-line error (the reference's CLI11 parse errors).  `--workers` and
// PHOTON_REUSE_THREADS are accepted for compatibility; the GPU engine ignores them.
#include <charconv>
#include <chrono>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "pathreuse_b200.hpp"

namespace fs = std::filesystem;
using namespace pathreuse;

namespace {

struct Usage : std::runtime_error {
    using std::runtime_error::runtime_error;
};

struct RunConfig {  // pathreuse_cli.cpp:35-49 defaults
    std::string scene = "builtin:static-box";
    std::string mode = "naive";
    uint32_t paths = 100000;
    uint32_t bounces = 7;
    std::string dm = "8x8x64x64";
    float threshold = 0.001f;
    int frames = 1;
    uint64_t seed = 1;
    float radius = 0.25f;
    std::string out = "out";
    std::string images = "on";
    unsigned workers = 0;
    std::string dump_photons;
};

const char* kHelp =
    "photon path-reuse renderer (B200 engine)\n"
    "Usage: pathreuse_cli [OPTIONS] [SUBCOMMAND]\n\n"
    "Options:\n"
    "  -h,--help              Print this help message and exit\n"
    "  --scene TEXT           scene file or builtin:NAME\n"
    "  --mode TEXT            baseline | naive | error\n"
    "  --paths UINT           light paths per frame\n"
    "  --bounces UINT         max photons per path (1..16)\n"
    "  --dm TEXT              distribution map dims AxBxCxD\n"
    "  --threshold FLOAT      error-based energy threshold\n"
    "  --frames INT           frames to run\n"
    "  --seed UINT            RNG seed\n"
    "  --radius FLOAT         gather radius, world units\n"
    "  --out TEXT             output directory\n"
    "  --images TEXT          write per-frame PPM images (on | off)\n"
    "  --workers UINT         worker threads (0 = logical cores; ignored on the GPU)\n"
    "  --dump-photons TEXT    write final photon map dump here\n\n"
    "Subcommands:\n"
    "  report                 summarize stats CSVs against the baseline\n";

template <typename T>
T number(const std::string& flag, const std::string& text) {
    T v{};
    const char* b = text.data();
    const char* e = b + text.size();
    auto [p, ec] = std::from_chars(b, e, v);
    if (ec != std::errc() || p != e) throw Usage(flag + ": " + text + " is not a valid number");
    return v;
}

std::vector<uint32_t> parse_dm_dims(const std::string& text) {  // pathreuse_cli.cpp:23-33
    std::vector<uint32_t> dims;
    std::stringstream ss(text);
    std::string part;
    while (std::getline(ss, part, 'x')) {
        if (part.empty()) throw Usage("--dm: expected AxBxCxD");
        dims.push_back(number<uint32_t>("--dm", part));
    }
    if (dims.size() != 4) throw Usage("--dm: expected exactly 4 axis counts");
    return dims;
}

std::string config_json(const RunConfig& rc) {  // pathreuse_cli.cpp:51-59 (keys sorted)
    auto num = [](double v) {
        char buf[64];
        auto r = std::to_chars(buf, buf + sizeof(buf), v);
        return std::string(buf, r.ptr);
    };
    auto str = [](const std::string& s) {
        std::string o = "\"";
        for (char c : s) {
            if (c == '"' || c == '\\') o.push_back('\\');
            o.push_back(c);
        }
        return o + "\"";
    };
    std::ostringstream o;
    o << "{\n  \"bounces\": " << rc.bounces << ",\n  \"dm\": " << str(rc.dm) << ",\n  \"frames\": " << rc.frames
      << ",\n  \"images\": " << str(rc.images) << ",\n  \"mode\": " << str(rc.mode) << ",\n  \"out\": " << str(rc.out)
      << ",\n  \"paths\": " << rc.paths << ",\n  \"radius\": " << num(rc.radius) << ",\n  \"scene\": " << str(rc.scene)
      << ",\n  \"seed\": " << rc.seed << ",\n  \"threshold\": " << num(rc.threshold) << ",\n  \"workers\": "
      << rc.workers << "\n}";
    return o.str();
}

int run(const RunConfig& rc) {  // pathreuse_cli.cpp:61-116
    Scene scene;
    try {
        scene = load_scene_source(rc.scene);
    } catch (const std::exception& e) {
        std::cerr << "scene error: " << e.what() << "\n";
        return 1;
    }
    EngineConfig cfg;
    cfg.mode = engine_mode_from_string(rc.mode);
    cfg.n_paths = rc.paths;
    cfg.max_bounces = rc.bounces;
    cfg.dm_dims = parse_dm_dims(rc.dm);
    cfg.threshold = rc.threshold;
    cfg.seed = rc.seed;
    cfg.gather_radius = rc.radius;
    cfg.workers = rc.workers;
    try {
        fs::create_directories(rc.out);
        {
            std::ofstream echo(fs::path(rc.out) / "config.json");
            echo << config_json(rc) << "\n";
        }
        const Camera camera = scene.camera;
        Engine engine(std::move(scene), cfg);
        std::vector<FrameStats> rows;
        for (int f = 0; f < rc.frames; ++f) {
            FrameStats stats = engine.run_frame();
            if (rc.images == "on") {
                const auto t0 = std::chrono::steady_clock::now();
                const Image img = gather_image(engine, camera, cfg.gather_radius, cfg.workers);
                write_image(img, (fs::path(rc.out) / frame_image_name(f)).string());
                stats.t_gather = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            }
            rows.push_back(stats);
            std::cout << "frame " << f << " traced " << stats.rays_traced << " reused " << stats.rays_reused
                      << " pruned " << stats.paths_pruned << " filled " << stats.paths_filled << "\n";
        }
        write_stats_csv(rows, (fs::path(rc.out) / "stats.csv").string());
        if (!rc.dump_photons.empty()) write_photon_dump(engine.photon_map(), rc.dump_photons);
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
    return 0;
}

int report(const std::vector<std::string>& csvs) {  // pathreuse_cli.cpp:118-131
    try {
        std::vector<FrameStats> rows;
        for (const std::string& path : csvs) {
            auto part = read_stats_csv(path);
            rows.insert(rows.end(), part.begin(), part.end());
        }
        std::cout << reuse_report(rows);
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    RunConfig rc;
    std::vector<std::string> csvs;
    bool is_report = false;
    try {
        std::vector<std::string> args(argv + 1, argv + argc);
        for (size_t i = 0; i < args.size(); ++i) {
            std::string a = args[i];
            if (a == "-h" || a == "--help") {
                std::cout << kHelp;
                return 0;
            }
            if (!is_report && a == "report") {
                is_report = true;
                continue;
            }
            if (is_report && a.rfind("--", 0) != 0) {
                csvs.push_back(a);
                continue;
            }
            std::string value;
            const size_t eq = a.find('=');
            if (a.rfind("--", 0) == 0 && eq != std::string::npos) {
                value = a.substr(eq + 1);
                a = a.substr(0, eq);
            } else if (a.rfind("--", 0) == 0) {
                if (i + 1 >= args.size()) throw Usage(a + ": requires an argument");
                value = args[++i];
            } else {
                throw Usage("The following argument was not expected: " + a);
            }
            if (is_report) throw Usage("report: unexpected option " + a);
            if (a == "--scene") rc.scene = value;
            else if (a == "--mode") {
                if (value != "baseline" && value != "naive" && value != "error")
                    throw Usage("--mode: " + value + " not in {baseline,naive,error}");
                rc.mode = value;
            } else if (a == "--paths") rc.paths = number<uint32_t>(a, value);
            else if (a == "--bounces") rc.bounces = number<uint32_t>(a, value);
            else if (a == "--dm") rc.dm = value;
            else if (a == "--threshold") rc.threshold = number<float>(a, value);
            else if (a == "--frames") rc.frames = number<int>(a, value);
            else if (a == "--seed") rc.seed = number<uint64_t>(a, value);
            else if (a == "--radius") rc.radius = number<float>(a, value);
            else if (a == "--out") rc.out = value;
            else if (a == "--images") {
                if (value != "on" && value != "off") throw Usage("--images: " + value + " not in {on,off}");
                rc.images = value;
            } else if (a == "--workers") rc.workers = number<unsigned>(a, value);
            else if (a == "--dump-photons") rc.dump_photons = value;
            else throw Usage("The following argument was not expected: " + a);
        }
        if (is_report && csvs.empty()) throw Usage("csv is required");
        if (!is_report) parse_dm_dims(rc.dm);  // validate before any work
    } catch (const Usage& e) {
        std::cerr << e.what() << "\nRun with --help for more information.\n";
        return 2;
    }
    if (is_report) return report(csvs);
    if (const char* env = std::getenv("PHOTON_REUSE_THREADS"))
        rc.workers = static_cast<unsigned>(std::strtoul(env, nullptr, 10));
    return run(rc);
}
