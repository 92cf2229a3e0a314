// archive_meta.h -- archive metadata (proj/include/spid/archive.hpp:15-31) and
// its JSON codec, compiled by g++ in archive_meta.cpp against nlohmann/json
// (the library the reference serialises with) so the metadata section is
// byte-identical to the reference's meta_to_json(...).dump().
#pragma once

#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

namespace spidgpu {

struct ArchiveMetaHost {
    bool structured = true;
    std::vector<std::size_t> dims;  // structured
    std::vector<bool> periodic;     // structured
    std::size_t points = 0;         // unstructured
    std::vector<std::size_t> blocks_per_axis;
    std::size_t time_chunk = 0;
    std::vector<std::size_t> strides;
    bool include_boundary = true;
    std::string mode;
    std::string rank_rule_mode;
    std::size_t rank_k = 0;
    double rank_tol = 0.0;
    double stage2_tol = 0.0;
    std::string interp_recipe;
    std::string qoi;
    std::size_t m = 0;
    std::size_t n = 0;
    std::string provenance;
};

// meta_to_json(meta).dump() (proj/src/archive.cpp:119-136, json_io.cpp:5-17).
std::string meta_to_json_string(const ArchiveMetaHost& meta);

// nlohmann::json::parse + meta_from_json (archive.cpp:138-157, json_io.cpp:
// 19-29). Returns a spidgpu status (SPID_TRUNCATED_PAYLOAD for invalid JSON,
// SPID_BAD_GRID_GEOM for an unknown grid kind or invalid dims) and a message.
int meta_from_json_bytes(const uint8_t* data, std::size_t len, ArchiveMetaHost* out,
                         std::string* msg);

// archive_info_json (archive.cpp:260-268): metadata plus block_count,
// block_ranks, stored_entries and compression_factor, dump(2).
std::string archive_info_string(const ArchiveMetaHost& meta, const std::vector<std::size_t>& ranks,
                                std::size_t stored_entries, double compression_factor);

}  // namespace spidgpu
