// wire.cpp -- the reference's offline artefacts: PHM1 photon dumps, the
// per-frame stats CSV and reuse report, PPM images.  Byte formats follow
// photon_store.cpp:55-102, stats.cpp:10-107 and gather.cpp:77-98, so files written here
// and by the reference are interchangeable (tests compare them byte for byte).
#include "wire.h"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <sstream>
#include <stdexcept>

namespace prx {

namespace {

constexpr char kPhotonMagic[4] = {'P', 'H', 'M', '1'};

void le32(std::ostream& out, uint32_t v) {
    const unsigned char b[4] = {static_cast<unsigned char>(v), static_cast<unsigned char>(v >> 8),
                                static_cast<unsigned char>(v >> 16), static_cast<unsigned char>(v >> 24)};
    out.write(reinterpret_cast<const char*>(b), 4);
}

uint32_t le32(std::istream& in) {
    unsigned char b[4] = {0, 0, 0, 0};
    in.read(reinterpret_cast<char*>(b), 4);
    return uint32_t(b[0]) | uint32_t(b[1]) << 8 | uint32_t(b[2]) << 16 | uint32_t(b[3]) << 24;
}

const char* mode_name(int mode) {
    switch (mode) {
        case PRX_MODE_BASELINE: return "baseline";
        case PRX_MODE_NAIVE: return "naive";
        case PRX_MODE_ERROR: return "error";
        default: throw std::invalid_argument("unknown engine mode");
    }
}

int mode_of(const std::string& s) {  // engine_mode_from_string (engine.cpp:52-61)
    if (s == "baseline") return PRX_MODE_BASELINE;
    if (s == "naive") return PRX_MODE_NAIVE;
    if (s == "error") return PRX_MODE_ERROR;
    throw std::invalid_argument("unknown engine mode: " + s);
}

}  // namespace

const char* const kStatsCsvHeader =
    "frame,mode,rays_traced,rays_reused,paths_replaced,paths_pruned,paths_filled,"
    "visibility_rays,t_update,t_occlusion,t_dm,t_prune,t_fill,t_trace,t_gather";

// ------------------------------------------------------------------ PHM1 (photon_store.cpp:55-102)
void write_photon_dump(const std::string& path, uint32_t n_paths, uint32_t max_bounces, const void* records,
                       size_t bytes) {
    if (bytes != static_cast<size_t>(n_paths) * max_bounces * kPhotonRecordBytes)
        throw std::invalid_argument("photon dump: record bytes do not match n_paths * max_bounces * 32");
    std::ofstream out(path, std::ios::binary);
    if (!out) throw std::runtime_error("cannot open photon dump for writing: " + path);
    out.write(kPhotonMagic, 4);
    le32(out, n_paths);
    le32(out, max_bounces);
    le32(out, 0);  // reserved
    out.write(static_cast<const char*>(records), static_cast<std::streamsize>(bytes));
    if (!out) throw std::runtime_error("failed writing photon dump: " + path);
}

void read_photon_dump(const std::string& path, uint32_t* n_paths, uint32_t* max_bounces, std::vector<char>* records) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw std::runtime_error("cannot open photon dump: " + path);
    char magic[4];
    in.read(magic, 4);
    if (!in || std::memcmp(magic, kPhotonMagic, 4) != 0) throw std::runtime_error("bad photon dump magic: " + path);
    const uint32_t n = le32(in), b = le32(in);
    le32(in);  // reserved
    if (n_paths) *n_paths = n;
    if (max_bounces) *max_bounces = b;
    if (records) {
        records->resize(static_cast<size_t>(n) * b * kPhotonRecordBytes);
        in.read(records->data(), static_cast<std::streamsize>(records->size()));
        if (!in) throw std::runtime_error("truncated photon dump: " + path);
    }
}

// ------------------------------------------------------------------ PPM (gather.cpp:77-98)
void write_image_ppm(const std::string& path, const float* rgb, uint32_t width, uint32_t height) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw std::runtime_error("cannot open image for writing: " + path);
    out << "P6\n" << width << " " << height << "\n255\n";
    const float inv_gamma = 1.0f / 2.2f;
    std::vector<unsigned char> row(static_cast<size_t>(width) * 3);
    size_t i = 0;
    for (uint32_t y = 0; y < height; ++y) {
        for (size_t x = 0; x < row.size(); ++x) {
            const float v = std::clamp(rgb[i++], 0.0f, 1.0f);  // tone curve of write_image
            row[x] = static_cast<unsigned char>(std::lround(std::pow(v, inv_gamma) * 255.0f));
        }
        out.write(reinterpret_cast<const char*>(row.data()), static_cast<std::streamsize>(row.size()));
    }
    if (!out) throw std::runtime_error("failed writing image: " + path);
}

std::string frame_image_name(int frame) {
    char buf[32];
    std::snprintf(buf, sizeof(buf), "frame_%04d.ppm", frame);
    return buf;
}

// ------------------------------------------------------------------ stats CSV (stats.cpp:10-70)
void write_stats_csv(std::ostream& out, const prx_frame_stats* rows, size_t n) {
    out << kStatsCsvHeader << "\n";
    for (size_t i = 0; i < n; ++i) {
        const prx_frame_stats& s = rows[i];
        out << s.frame << ',' << mode_name(s.mode) << ',' << s.rays_traced << ',' << s.rays_reused << ','
            << s.paths_replaced << ',' << s.paths_pruned << ',' << s.paths_filled << ',' << s.visibility_rays
            << ',' << s.t_update << ',' << s.t_occlusion << ',' << s.t_dm << ',' << s.t_prune << ',' << s.t_fill
            << ',' << s.t_trace << ',' << s.t_gather << "\n";
    }
}

void write_stats_csv(const std::string& path, const prx_frame_stats* rows, size_t n) {
    std::ofstream out(path);
    if (!out) throw std::runtime_error("cannot open stats CSV for writing: " + path);
    write_stats_csv(out, rows, n);
    if (!out) throw std::runtime_error("failed writing stats CSV: " + path);
}

std::vector<prx_frame_stats> read_stats_csv(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw std::runtime_error("cannot open stats CSV: " + path);
    std::string line;
    if (!std::getline(in, line) || line != kStatsCsvHeader)
        throw std::runtime_error("bad stats CSV header in " + path);
    std::vector<prx_frame_stats> rows;
    while (std::getline(in, line)) {
        if (line.empty()) continue;
        std::vector<std::string> f;
        std::istringstream ls(line);
        for (std::string cell; std::getline(ls, cell, ',');) f.push_back(cell);
        const std::string bad = "bad stats CSV row in " + path + ": " + line;
        if (f.size() != 15) throw std::runtime_error(bad);
        prx_frame_stats s{};
        try {
            s.frame = std::stoi(f[0]);
            s.mode = mode_of(f[1]);
            uint64_t* counters[6] = {&s.rays_traced, &s.rays_reused, &s.paths_replaced,
                                     &s.paths_pruned, &s.paths_filled, &s.visibility_rays};
            for (int k = 0; k < 6; ++k) *counters[k] = std::stoull(f[2 + k]);
            double* times[7] = {&s.t_update, &s.t_occlusion, &s.t_dm, &s.t_prune, &s.t_fill, &s.t_trace, &s.t_gather};
            for (int k = 0; k < 7; ++k) *times[k] = std::stod(f[8 + k]);
        } catch (const std::exception&) {
            throw std::runtime_error(bad);
        }
        rows.push_back(s);
    }
    return rows;
}

// stats.cpp:72-107: per-frame traced-ray ratio of every mode against the baseline rows
std::string reuse_report(const prx_frame_stats* rows, size_t n) {
    std::map<std::string, std::vector<prx_frame_stats>> by_mode;  // sorted by mode name
    for (size_t i = 0; i < n; ++i) by_mode[mode_name(rows[i].mode)].push_back(rows[i]);
    const auto base = by_mode.find("baseline");
    if (base == by_mode.end()) throw std::runtime_error("report: no baseline rows to compare against");
    for (const auto& [mode, r] : by_mode)
        if (r.size() != base->second.size())
            throw std::runtime_error("report: mode '" + mode + "' has " + std::to_string(r.size()) +
                                     " frames but baseline has " + std::to_string(base->second.size()));
    std::ostringstream out;
    out << "frames: " << base->second.size() << "\n";
    for (const auto& [mode, r] : by_mode) {
        double ratio_sum = 0.0, reuse_sum = 0.0;
        out << "mode " << mode << "\n";
        for (size_t i = 0; i < r.size(); ++i) {
            const double b = static_cast<double>(base->second[i].rays_traced);
            const double ratio = b > 0 ? static_cast<double>(r[i].rays_traced) / b : 1.0;
            const double segs = static_cast<double>(r[i].rays_traced + r[i].rays_reused);
            const double reuse = segs > 0 ? static_cast<double>(r[i].rays_reused) / segs : 0.0;
            ratio_sum += ratio;
            reuse_sum += reuse;
            out << "  frame " << r[i].frame << " traced " << r[i].rays_traced << " ratio_vs_baseline " << ratio
                << " reuse_fraction " << reuse << "\n";
        }
        out << "  mean ratio_vs_baseline " << ratio_sum / r.size() << " mean reuse_fraction " << reuse_sum / r.size()
            << "\n";
    }
    return out.str();
}

}  // namespace prx
