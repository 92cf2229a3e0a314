// archive_internal.h -- block layout and archive emission shared by the
// batch archive ABI (archive_api.cu) and the streaming pipeline
// (stream_api.cu). Internal; not part of include/spidgpu.h.
#pragma once

#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "archive_meta.h"
#include "context.h"

namespace spidgpu {

constexpr uint32_t kArchiveVersion = 1;
constexpr size_t kArenaAlign = 256;

// ---- make_block_domains (proj/src/blocking.cpp:12-104) ------------------------
struct Seg {
    int64_t start, len;
};

struct Domain {
    int64_t base;    // global flat index of the block's first point
    int64_t l[3];    // local dims (unstructured: l[0] = points)
    int32_t per[3];  // local periodic flags
};

struct Layout {
    bool structured = true;
    int naxes = 1;
    int64_t dims[3] = {1, 1, 1};
    int64_t points = 0;
    std::vector<Domain> doms;
    std::vector<Seg> segs[3];
};

int axis_segments(spidgpu_handle h, int64_t dim, int64_t count, std::vector<Seg>* out);
int make_domains(spidgpu_handle h, bool structured, int naxes, const int64_t* dims,
                 const int32_t* periodic, int64_t points, const std::vector<int64_t>& blocks,
                 Layout* L);

// Blocks of one local geometry (and, for decompress, one coarse flag) share
// their row maps and run as one batch.
struct Group {
    Domain proto;
    int32_t coarse = 0;
    std::vector<int64_t> members;  // block ids, ascending
};
std::vector<Group> group_blocks(const Layout& L, const std::vector<int32_t>* coarse);

// global offset (relative to the block base) of local flat index l
inline int64_t globalize(const Layout& L, const Domain& d, int64_t l) {
    const int64_t i0 = l % d.l[0], i1 = (l / d.l[0]) % d.l[1], i2 = l / (d.l[0] * d.l[1]);
    return i0 + L.dims[0] * i1 + L.dims[0] * L.dims[1] * i2;
}

// local SubsampleSpec::strided(local, strides, include_boundary)
int local_spec(spidgpu_handle h, const Layout& L, const Domain& d, const int64_t* strides, int incl,
               GridSpecDev* g, int64_t* P, int64_t* Pc, bool lift = true);

// Byte arena carved out of one device buffer.
struct Carve {
    size_t off = 0;
    template <class T>
    size_t take(size_t count) {
        off = (off + kArenaAlign - 1) / kArenaAlign * kArenaAlign;
        const size_t o = off;
        off += sizeof(T) * std::max<size_t>(count, 1);
        return o;
    }
};

template <class T>
T* at(DevBuf& buf, size_t off) {
    return reinterpret_cast<T*>(static_cast<uint8_t*>(buf.ptr) + off);
}

// SPIDGPU_TRACE=1: per-phase device times of the archive calls on stderr.
struct Trace {
    bool on = std::getenv("SPIDGPU_TRACE") != nullptr;
    cudaStream_t st;
    std::vector<std::pair<std::string, cudaEvent_t>> marks;
    explicit Trace(cudaStream_t s) : st(s) { mark("start"); }
    void mark(const char* name) {
        if (!on) return;
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, st);
        marks.emplace_back(name, e);
    }
    ~Trace() {
        if (!on) return;
        cudaEventSynchronize(marks.back().second);
        std::string line = "[spidgpu trace]";
        for (size_t i = 1; i < marks.size(); ++i) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, marks[i - 1].second, marks[i].second);
            line += " " + marks[i].first + "=" + std::to_string(ms) + "ms";
        }
        std::fprintf(stderr, "%s\n", line.c_str());
        for (auto& m : marks) cudaEventDestroy(m.second);
    }
};

inline void put_u32(std::vector<uint8_t>& o, uint32_t v) {
    for (int i = 0; i < 4; ++i) o.push_back(static_cast<uint8_t>(v >> (8 * i)));
}
inline void put_u64(std::vector<uint8_t>& o, uint64_t v) {
    for (int i = 0; i < 8; ++i) o.push_back(static_cast<uint8_t>(v >> (8 * i)));
}

// encode() (archive.cpp:193-212) of blocks whose factors are in device memory:
// host formats the header + metadata, fills each PackBlock's sec_off, the
// device packs every block section, checksums all sections and the finished
// archive lands in the handle's pinned buffer (spidgpu_archive_view/fetch).
// Uses ws.blocks / ws.crc / ws.bytes of `ws`.
int emit_archive(spidgpu_handle h, Workspace& ws, const ArchiveMetaHost& meta,
                 std::vector<PackBlock>& pack, cudaStream_t st, Trace* tr, int64_t* nbytes);

}  // namespace spidgpu
