// archive_meta.cpp -- JSON metadata of the archive container.
//
// Key set, value types and nesting follow meta_to_json / grid_to_json
// (proj/src/archive.cpp:119-136, proj/src/json_io.cpp:5-17); nlohmann::json's
// default object is key-sorted and dump() without indent is compact, so the
// emitted bytes equal the reference's for the same metadata.
#include "archive_meta.h"

#include "../../include/spidgpu_status.h"
#include "json.hpp"

namespace spidgpu {

namespace {

nlohmann::json meta_json(const ArchiveMetaHost& meta) {
    nlohmann::json grid;
    if (meta.structured) {
        grid["kind"] = "structured";
        grid["dims"] = meta.dims;
        grid["periodic"] = meta.periodic;
    } else {
        grid["kind"] = "unstructured";
        grid["points"] = meta.points;
    }
    nlohmann::json j;
    j["grid"] = grid;
    j["blocks_per_axis"] = meta.blocks_per_axis;
    j["time_chunk"] = meta.time_chunk;
    j["strides"] = meta.strides;
    j["include_boundary"] = meta.include_boundary;
    j["mode"] = meta.mode;
    j["rank_rule"] = {{"mode", meta.rank_rule_mode}, {"k", meta.rank_k}, {"tol", meta.rank_tol}};
    j["stage2_tol"] = meta.stage2_tol;
    j["interp"] = meta.interp_recipe;
    j["qoi"] = meta.qoi;
    j["m"] = meta.m;
    j["n"] = meta.n;
    j["provenance"] = meta.provenance;
    return j;
}

}  // namespace

std::string meta_to_json_string(const ArchiveMetaHost& meta) { return meta_json(meta).dump(); }

int meta_from_json_bytes(const uint8_t* data, std::size_t len, ArchiveMetaHost* out,
                         std::string* msg) {
    nlohmann::json j;
    try {
        j = nlohmann::json::parse(data, data + len);
    } catch (const nlohmann::json::exception& e) {
        *msg = std::string("metadata is not valid JSON: ") + e.what();
        return SPID_TRUNCATED_PAYLOAD;
    }
    try {
        ArchiveMetaHost m;
        const nlohmann::json& g = j.at("grid");
        const std::string kind = g.at("kind").get<std::string>();
        if (kind == "structured") {
            m.structured = true;
            m.dims = g.at("dims").get<std::vector<std::size_t>>();
            if (g.contains("periodic")) m.periodic = g.at("periodic").get<std::vector<bool>>();
            // GridGeom::structured (grid.cpp:7-20)
            if (m.dims.empty() || m.dims.size() > 3) {
                *msg = "structured grids have 1 to 3 axes";
                return SPID_BAD_GRID_GEOM;
            }
            for (std::size_t d : m.dims)
                if (d < 2) {
                    *msg = "each structured axis needs at least 2 points";
                    return SPID_BAD_GRID_GEOM;
                }
            if (m.periodic.empty()) m.periodic.assign(m.dims.size(), false);
            if (m.periodic.size() != m.dims.size()) {
                *msg = "periodic flag count must match axis count";
                return SPID_BAD_GRID_GEOM;
            }
        } else if (kind == "unstructured") {
            m.structured = false;
            m.points = g.at("points").get<std::size_t>();
            if (m.points < 1) {
                *msg = "need at least one point";
                return SPID_BAD_GRID_GEOM;
            }
        } else {
            *msg = "unknown grid kind in metadata: " + kind;
            return SPID_BAD_GRID_GEOM;
        }
        m.blocks_per_axis = j.at("blocks_per_axis").get<std::vector<std::size_t>>();
        m.time_chunk = j.at("time_chunk").get<std::size_t>();
        m.strides = j.at("strides").get<std::vector<std::size_t>>();
        m.include_boundary = j.at("include_boundary").get<bool>();
        m.mode = j.at("mode").get<std::string>();
        m.rank_rule_mode = j.at("rank_rule").at("mode").get<std::string>();
        m.rank_k = j.at("rank_rule").at("k").get<std::size_t>();
        m.rank_tol = j.at("rank_rule").at("tol").get<double>();
        m.stage2_tol = j.at("stage2_tol").get<double>();
        m.interp_recipe = j.at("interp").get<std::string>();
        m.qoi = j.at("qoi").get<std::string>();
        m.m = j.at("m").get<std::size_t>();
        m.n = j.at("n").get<std::size_t>();
        m.provenance = j.at("provenance").get<std::string>();
        *out = std::move(m);
        return SPID_OK;
    } catch (const nlohmann::json::exception& e) {
        // the reference lets json::out_of_range / type_error escape decode();
        // a C ABI reports them as a malformed payload
        *msg = std::string("metadata field: ") + e.what();
        return SPID_TRUNCATED_PAYLOAD;
    }
}

std::string archive_info_string(const ArchiveMetaHost& meta, const std::vector<std::size_t>& ranks,
                                std::size_t stored_entries, double compression_factor) {
    nlohmann::json j = meta_json(meta);
    j["block_count"] = ranks.size();
    j["block_ranks"] = ranks;
    j["stored_entries"] = stored_entries;
    j["compression_factor"] = compression_factor;
    return j.dump(2);
}

}  // namespace spidgpu
