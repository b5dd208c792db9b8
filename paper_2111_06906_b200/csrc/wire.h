// wire.h -- offline artefacts of the reference (see wire.cpp).
#pragma once

#include <cstddef>
#include <cstdint>
#include <iosfwd>
#include <string>
#include <vector>

#include "prx.h"

namespace prx {

constexpr size_t kPhotonRecordBytes = 32;  // sizeof(Photon), photon_store.hpp:13-21
extern const char* const kStatsCsvHeader;   // stats.cpp:10-12

void write_photon_dump(const std::string& path, uint32_t n_paths, uint32_t max_bounces, const void* records,
                       size_t bytes);
void read_photon_dump(const std::string& path, uint32_t* n_paths, uint32_t* max_bounces, std::vector<char>* records);

void write_image_ppm(const std::string& path, const float* rgb, uint32_t width, uint32_t height);
std::string frame_image_name(int frame);

void write_stats_csv(std::ostream& out, const prx_frame_stats* rows, size_t n);
void write_stats_csv(const std::string& path, const prx_frame_stats* rows, size_t n);
std::vector<prx_frame_stats> read_stats_csv(const std::string& path);
std::string reuse_report(const prx_frame_stats* rows, size_t n);

}  // namespace prx
