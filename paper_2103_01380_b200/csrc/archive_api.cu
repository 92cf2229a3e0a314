// archive_api.cu -- spidgpu archive ABI: whole-field batch compression into
// the reference's archive container, decode checks, and decompress.
//
// Host code here only walks the container framing, lays out byte offsets and
// sequences launches; gathers, column IDs, packing, checksums, unpacking,
// lifting and the reconstruct/assemble run in the kernels of archive.cu,
// cpqr*.cu, sketch.cu, gather.cu and interp.cu.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <algorithm>
#include <thread>
#include <vector>

#include "archive_internal.h"

using namespace spidgpu;

namespace spidgpu {

// ---- make_block_domains (proj/src/blocking.cpp:12-104) ------------------------
int axis_segments(spidgpu_handle h, int64_t dim, int64_t count, std::vector<Seg>* out) {
    if (count < 1 || count > dim)
        return fail(h, SPID_BLOCK_TOO_SMALL, "blocks per axis must lie in [1, axis dim]");
    const int64_t base = dim / count;
    int64_t at = 0;
    out->clear();
    for (int64_t b = 0; b < count; ++b) {
        const int64_t len = (b + 1 == count) ? dim - at : base;
        if (len < 1) return fail(h, SPID_BLOCK_TOO_SMALL, "a block would hold no points");
        out->push_back({at, len});
        at += len;
    }
    return SPID_OK;
}

int make_domains(spidgpu_handle h, bool structured, int naxes, const int64_t* dims,
                 const int32_t* periodic, int64_t points, const std::vector<int64_t>& blocks,
                 Layout* L) {
    L->structured = structured;
    L->doms.clear();
    if (!structured) {
        if (blocks.size() != 1)
            return fail(h, SPID_BAD_GRID_GEOM, "unstructured grids are blocked along the single row axis");
        int rc = axis_segments(h, points, blocks[0], &L->segs[0]);
        if (rc) return rc;
        L->naxes = 1;
        L->dims[0] = points;
        L->points = points;
        for (const Seg& s : L->segs[0]) L->doms.push_back({s.start, {s.len, 1, 1}, {0, 0, 0}});
        return SPID_OK;
    }
    if (static_cast<int>(blocks.size()) != naxes)
        return fail(h, SPID_BAD_GRID_GEOM, "blocks_per_axis arity must match axis count");
    L->naxes = naxes;
    L->points = 1;
    for (int ax = 0; ax < 3; ++ax) {
        L->dims[ax] = ax < naxes ? dims[ax] : 1;
        if (ax < naxes) {
            int rc = axis_segments(h, dims[ax], blocks[ax], &L->segs[ax]);
            if (rc) return rc;
            L->points *= dims[ax];
        } else {
            L->segs[ax] = {{0, 1}};
        }
    }
    const int64_t d0 = L->dims[0], d1 = L->dims[1];
    for (const Seg& s2 : L->segs[2])
        for (const Seg& s1 : L->segs[1])
            for (const Seg& s0 : L->segs[0]) {
                Domain d;
                d.base = s0.start + d0 * s1.start + d0 * d1 * s2.start;
                d.l[0] = s0.len;
                d.l[1] = s1.len;
                d.l[2] = s2.len;
                for (int ax = 0; ax < 3; ++ax)
                    d.per[ax] = ax < naxes && periodic[ax] && d.l[ax] == L->dims[ax] ? 1 : 0;
                L->doms.push_back(d);
            }
    return SPID_OK;
}

std::vector<Group> group_blocks(const Layout& L, const std::vector<int32_t>* coarse) {
    std::vector<Group> groups;
    for (int64_t b = 0; b < static_cast<int64_t>(L.doms.size()); ++b) {
        const Domain& d = L.doms[b];
        const int32_t c = coarse ? (*coarse)[b] : 0;
        Group* hit = nullptr;
        for (Group& g : groups)
            if (g.coarse == c && !std::memcmp(g.proto.l, d.l, sizeof(d.l)) &&
                !std::memcmp(g.proto.per, d.per, sizeof(d.per)))
                hit = &g;
        if (!hit) {
            groups.push_back(Group{d, c, {}});
            hit = &groups.back();
        }
        hit->members.push_back(b);
    }
    return groups;
}

int local_spec(spidgpu_handle h, const Layout& L, const Domain& d, const int64_t* strides,
               int incl, GridSpecDev* g, int64_t* P, int64_t* Pc, bool lift) {
    spidgpu_grid_spec sp{};
    sp.naxes = L.naxes;
    sp.include_boundary = incl;
    sp.nqoi = 1;
    for (int ax = 0; ax < 3; ++ax) {
        sp.dims[ax] = d.l[ax];
        sp.strides[ax] = ax < L.naxes ? strides[ax] : 1;
        sp.periodic[ax] = d.per[ax];
    }
    return spec_to_dev(h, &sp, g, P, Pc, /*min_dim=*/1, lift);
}

namespace {

constexpr uint32_t kVersion = kArchiveVersion;

// ---- decode() framing (archive.cpp:37-98, 214-249) --------------------------------
struct Reader {
    const uint8_t* p;
    int64_t size, at = 0;
    bool need(int64_t count) const { return count >= 0 && at <= size && count <= size - at; }
    uint64_t u64() {
        uint64_t v = 0;
        for (int i = 0; i < 8; ++i) v |= static_cast<uint64_t>(p[at + i]) << (8 * i);
        at += 8;
        return v;
    }
    uint32_t u32() {
        uint32_t v = 0;
        for (int i = 0; i < 4; ++i) v |= static_cast<uint32_t>(p[at + i]) << (8 * i);
        at += 4;
        return v;
    }
};

struct SecRef {
    int64_t begin, len;
    uint32_t stored;
};
struct BlockRef {
    int32_t coarse;
    int64_t sr, sc, cr, cc;       // skeleton rows/cols, coeff rows/cols
    int64_t skel_off, coef_off;   // absolute offsets of the first f64
};
struct Framing {
    int status = SPID_OK;         // first framing failure (Truncated/BadMagic/Version)
    std::string msg;
    int fail_stage = 0;           // 0 header, 1 meta section, 2 block count, 3 + b block b
    std::vector<SecRef> secs;     // meta + blocks framed so far
    uint64_t block_count = 0;
};

void frame_archive(const uint8_t* bytes, int64_t nbytes, Framing* F) {
    Reader r{bytes, nbytes};
    auto section = [&](int stage) -> bool {
        if (!r.need(8)) {
            F->status = SPID_TRUNCATED_PAYLOAD;
            F->fail_stage = stage;
            F->msg = "archive ends before the promised payload";
            return false;
        }
        const uint64_t len = r.u64();
        if (len > static_cast<uint64_t>(INT64_MAX) || !r.need(static_cast<int64_t>(len)) ||
            !r.need(static_cast<int64_t>(len) + 4)) {
            F->status = SPID_TRUNCATED_PAYLOAD;
            F->fail_stage = stage;
            F->msg = "archive ends before the promised payload";
            return false;
        }
        SecRef s{r.at, static_cast<int64_t>(len), 0};
        r.at += static_cast<int64_t>(len);
        s.stored = r.u32();
        F->secs.push_back(s);
        return true;
    };
    if (!r.need(4)) {
        F->status = SPID_TRUNCATED_PAYLOAD;
        F->msg = "archive ends before the promised payload";
        return;
    }
    if (std::memcmp(bytes, "SPID", 4) != 0) {
        F->status = SPID_BAD_MAGIC;
        F->msg = "not a SPID archive";
        return;
    }
    r.at = 4;
    if (!r.need(4)) {
        F->status = SPID_TRUNCATED_PAYLOAD;
        F->msg = "archive ends before the promised payload";
        return;
    }
    const uint32_t version = r.u32();
    if (version != kVersion) {
        F->status = SPID_VERSION_UNSUPPORTED;
        F->msg = "archive version " + std::to_string(version);
        return;
    }
    if (!section(1)) return;
    if (!r.need(8)) {
        F->status = SPID_TRUNCATED_PAYLOAD;
        F->fail_stage = 2;
        F->msg = "archive ends before the promised payload";
        return;
    }
    F->block_count = r.u64();
    for (uint64_t b = 0; b < F->block_count; ++b)
        if (!section(3 + static_cast<int>(std::min<uint64_t>(b, 1u << 30)))) return;
    if (r.at != nbytes) {
        F->status = SPID_TRUNCATED_PAYLOAD;
        F->fail_stage = -1;  // after the last section
        F->msg = "trailing bytes after the last section";
    }
}

// Block payload (archive.cpp:230-243): coarse | index array x2 | matrix x2.
int parse_block(const uint8_t* bytes, const SecRef& s, BlockRef* b, std::string* msg) {
    Reader r{bytes + s.begin, s.len};
    auto trunc = [&](const char* m) {
        *msg = m;
        return SPID_TRUNCATED_PAYLOAD;
    };
    if (!r.need(1)) return trunc("archive ends before the promised payload");
    b->coarse = bytes[s.begin] != 0;
    r.at = 1;
    for (int arr = 0; arr < 2; ++arr) {
        if (!r.need(8)) return trunc("archive ends before the promised payload");
        const uint64_t count = r.u64();
        if (count > static_cast<uint64_t>((r.size - r.at) / 8)) return trunc("archive ends before the promised payload");
        r.at += static_cast<int64_t>(count) * 8;
    }
    int64_t dims[2][2], offs[2];
    for (int mat = 0; mat < 2; ++mat) {
        if (!r.need(16)) return trunc("archive ends before the promised payload");
        const uint64_t rows = r.u64(), cols = r.u64();
        if (rows == 0 || cols == 0) return trunc("matrix section has empty dimensions");
        // division, not rows * cols: the product of two section-sized
        // values can wrap uint64 and pass a multiplied check
        const uint64_t avail = static_cast<uint64_t>((r.size - r.at) / 8);
        if (rows > avail || cols > avail || cols > avail / rows)
            return trunc("archive ends before the promised payload");
        dims[mat][0] = static_cast<int64_t>(rows);
        dims[mat][1] = static_cast<int64_t>(cols);
        offs[mat] = s.begin + r.at;
        r.at += static_cast<int64_t>(rows * cols) * 8;
    }
    if (r.at != r.size) return trunc("trailing bytes in block section");
    b->sr = dims[0][0];
    b->sc = dims[0][1];
    b->cr = dims[1][0];
    b->cc = dims[1][1];
    b->skel_off = offs[0];
    b->coef_off = offs[1];
    return SPID_OK;
}

struct Decoded {
    ArchiveMetaHost meta;
    std::vector<BlockRef> blocks;
};

// decode() with the checksums already computed on the device (crcs[i] for
// F.secs[i]); errors are reported in the reference's order.
int decode_checked(spidgpu_handle h, const uint8_t* bytes, const Framing& F,
                   const std::vector<uint32_t>& crcs, Decoded* out) {
    if (F.secs.empty()) return fail(h, F.status ? F.status : SPID_TRUNCATED_PAYLOAD, F.msg);
    // metadata section
    if (crcs[0] != F.secs[0].stored)
        return fail(h, SPID_CHECKSUM_MISMATCH, "section checksum does not match payload");
    std::string msg;
    int rc = meta_from_json_bytes(bytes + F.secs[0].begin, static_cast<size_t>(F.secs[0].len),
                                  &out->meta, &msg);
    if (rc) return fail(h, rc, msg);
    if (F.status && F.fail_stage == 2) return fail(h, F.status, F.msg);
    out->blocks.clear();
    for (size_t i = 1; i < F.secs.size(); ++i) {
        if (crcs[i] != F.secs[i].stored)
            return fail(h, SPID_CHECKSUM_MISMATCH, "section checksum does not match payload");
        BlockRef b;
        rc = parse_block(bytes, F.secs[i], &b, &msg);
        if (rc) return fail(h, rc, msg);
        out->blocks.push_back(b);
    }
    if (F.status) return fail(h, F.status, F.msg);  // framing stopped early / trailing bytes
    return SPID_OK;
}

// Host bytes -> device. Page-locked sources (spidgpu_archive_view, pinned
// buffers) go straight to the copy engine; pageable ones (an archive read
// from a file) would crawl through the driver's bounce buffer at ~10 GB/s,
// so T host threads copy 4 MB chunks into their own two pinned slots while
// the copy engine drains the previous ones.
int upload_host_bytes(spidgpu_handle h, uint8_t* dst, const uint8_t* src, int64_t n, cudaStream_t st) {
    constexpr int64_t kChunk = int64_t(4) << 20;
    cudaPointerAttributes pa{};
    const bool pinned = cudaPointerGetAttributes(&pa, src) == cudaSuccess && pa.type == cudaMemoryTypeHost;
    cudaGetLastError();
    if (pinned || n < 2 * kChunk) {
        CK(h, cudaMemcpyAsync(dst, src, static_cast<size_t>(n), cudaMemcpyHostToDevice, st));
        return SPID_OK;
    }
    const int64_t nchunks = (n + kChunk - 1) / kChunk;
    const unsigned hc = std::thread::hardware_concurrency();
    const int T = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>({8, hc ? hc / 2 : 4, (nchunks + 1) / 2})));
    const size_t want = static_cast<size_t>(2 * T * kChunk);
    for (cudaEvent_t e : h->upload_ev)  // slots of a previous call may still be draining
        if (e) CK(h, cudaEventSynchronize(e));
    if (h->upload_cap < want) {
        if (h->upload_pinned) cudaFreeHost(h->upload_pinned);
        h->upload_pinned = nullptr;
        h->upload_cap = 0;
        CK(h, cudaHostAlloc(reinterpret_cast<void**>(&h->upload_pinned), want, cudaHostAllocDefault));
        h->upload_cap = want;
    }
    for (int i = 0; i < 2 * T; ++i)
        if (!h->upload_ev[i]) CK(h, cudaEventCreateWithFlags(&h->upload_ev[i], cudaEventDisableTiming));
    std::vector<cudaError_t> errs(T, cudaSuccess);
    std::vector<std::thread> workers;
    for (int w = 0; w < T; ++w)
        workers.emplace_back([&, w] {
            cudaError_t e = cudaSetDevice(h->device);
            for (int64_t c = w, j = 0; c < nchunks && e == cudaSuccess; c += T, ++j) {
                const int slot = 2 * w + static_cast<int>(j & 1);
                uint8_t* buf = h->upload_pinned + slot * kChunk;
                if (j >= 2) e = cudaEventSynchronize(h->upload_ev[slot]);
                if (e != cudaSuccess) break;
                const int64_t len = std::min(kChunk, n - c * kChunk);
                std::memcpy(buf, src + c * kChunk, static_cast<size_t>(len));
                e = cudaMemcpyAsync(dst + c * kChunk, buf, static_cast<size_t>(len), cudaMemcpyHostToDevice, st);
                if (e == cudaSuccess) e = cudaEventRecord(h->upload_ev[slot], st);
            }
            errs[w] = e;
        });
    for (auto& t : workers) t.join();
    for (cudaError_t e : errs) CK(h, e);
    return SPID_OK;
}

int decode_archive(spidgpu_handle h, const uint8_t* bytes, int64_t nbytes, Decoded* out,
                   cudaStream_t st) {
    Framing F;
    frame_archive(bytes, nbytes, &F);
    if (F.secs.empty()) return fail(h, F.status, F.msg);
    Workspace& ws = h->ws[0];
    std::vector<CrcSection> secs;
    for (const SecRef& s : F.secs) secs.push_back({s.begin, s.len});
    std::vector<CrcPart> parts;
    std::vector<int64_t> first_part;
    crc_plan_parts(secs.data(), static_cast<int64_t>(secs.size()), &parts, &first_part);
    Carve cv;
    const size_t o_bytes = cv.take<uint8_t>(static_cast<size_t>(nbytes));
    const size_t o_secs = cv.take<CrcSection>(secs.size());
    const size_t o_crc = cv.take<uint32_t>(secs.size());
    const size_t o_parts = cv.take<CrcPart>(parts.size());
    const size_t o_first = cv.take<int64_t>(first_part.size());
    const size_t o_pcrc = cv.take<uint32_t>(parts.size());
    CK(h, ws.bytes.ensure(cv.off, st));
    int rc = upload_host_bytes(h, at<uint8_t>(ws.bytes, o_bytes), bytes, nbytes, st);
    if (rc) return rc;
    CK(h, cudaMemcpyAsync(at<CrcSection>(ws.bytes, o_secs), secs.data(),
                          sizeof(CrcSection) * secs.size(), cudaMemcpyHostToDevice, st));
    CK(h, cudaMemcpyAsync(at<CrcPart>(ws.bytes, o_parts), parts.data(), sizeof(CrcPart) * parts.size(),
                          cudaMemcpyHostToDevice, st));
    CK(h, cudaMemcpyAsync(at<int64_t>(ws.bytes, o_first), first_part.data(),
                          sizeof(int64_t) * first_part.size(), cudaMemcpyHostToDevice, st));
    CK(h, launch_crc_sections(at<uint8_t>(ws.bytes, o_bytes), at<CrcSection>(ws.bytes, o_secs),
                              static_cast<int64_t>(secs.size()), at<CrcPart>(ws.bytes, o_parts),
                              static_cast<int64_t>(parts.size()), at<int64_t>(ws.bytes, o_first),
                              at<uint32_t>(ws.bytes, o_pcrc), at<uint32_t>(ws.bytes, o_crc), nullptr, st));
    h->launches += 2;
    std::vector<uint32_t> crcs(secs.size());
    CK(h, cudaMemcpyAsync(crcs.data(), at<uint32_t>(ws.bytes, o_crc), sizeof(uint32_t) * crcs.size(),
                          cudaMemcpyDeviceToHost, st));
    CK(h, cudaStreamSynchronize(st));
    return decode_checked(h, bytes, F, crcs, out);
}

int layout_from_meta(spidgpu_handle h, const ArchiveMetaHost& m, Layout* L) {
    int64_t dims[3] = {1, 1, 1};
    int32_t per[3] = {0, 0, 0};
    for (size_t ax = 0; ax < m.dims.size() && ax < 3; ++ax) {
        dims[ax] = static_cast<int64_t>(m.dims[ax]);
        per[ax] = m.periodic[ax] ? 1 : 0;
    }
    std::vector<int64_t> blocks(m.blocks_per_axis.begin(), m.blocks_per_axis.end());
    return make_domains(h, m.structured, static_cast<int>(m.dims.size()), dims, per,
                        static_cast<int64_t>(m.points), blocks, L);
}

}  // namespace

int emit_archive(spidgpu_handle h, Workspace& ws, const ArchiveMetaHost& meta,
                 std::vector<PackBlock>& pack, cudaStream_t st, Trace* tr, int64_t* nbytes) {
    // container layout: magic | u32 version | meta section | u64 count | blocks
    const int64_t nblocks = static_cast<int64_t>(pack.size());
    const std::string mj = meta_to_json_string(meta);
    std::vector<uint8_t> head;
    head.insert(head.end(), {'S', 'P', 'I', 'D'});
    put_u32(head, kArchiveVersion);
    put_u64(head, mj.size());
    head.insert(head.end(), mj.begin(), mj.end());
    put_u32(head, 0);  // CRC, written on the device
    put_u64(head, static_cast<uint64_t>(nblocks));

    std::vector<CrcSection> secs(nblocks + 1);
    secs[0] = {16, static_cast<int64_t>(mj.size())};
    int64_t off = static_cast<int64_t>(head.size()), max_items = 1;
    for (int64_t b = 0; b < nblocks; ++b) {
        PackBlock& d = pack[b];
        d.sec_off = off;
        const int64_t payload = 49 + 8 * d.nu + 8 * d.k + 8 * d.mc * d.k + 8 * d.k * d.n;
        max_items = std::max(max_items, 8 + d.nu + d.k + d.mc * d.k + d.k * d.n);
        secs[b + 1] = {off + 8, payload};
        off += 8 + payload + 4;
    }
    const int64_t total = off;
    std::vector<CrcPart> parts;
    std::vector<int64_t> first_part;
    crc_plan_parts(secs.data(), static_cast<int64_t>(secs.size()), &parts, &first_part);
    Carve cc;
    const size_t o_pack = cc.take<PackBlock>(pack.size());
    const size_t o_secs = cc.take<CrcSection>(secs.size());
    const size_t o_crc = cc.take<uint32_t>(secs.size());
    const size_t o_parts = cc.take<CrcPart>(parts.size());
    const size_t o_first = cc.take<int64_t>(first_part.size());
    const size_t o_pcrc = cc.take<uint32_t>(parts.size());
    CK(h, ws.crc.ensure(cc.off, st));
    CK(h, ws.bytes.ensure(static_cast<size_t>(total), st));
    uint8_t* dev = ws.bytes.as<uint8_t>();
    CK(h, cudaMemcpyAsync(dev, head.data(), head.size(), cudaMemcpyHostToDevice, st));
    CK(h, cudaMemcpyAsync(at<PackBlock>(ws.crc, o_pack), pack.data(), sizeof(PackBlock) * pack.size(),
                          cudaMemcpyHostToDevice, st));
    CK(h, cudaMemcpyAsync(at<CrcSection>(ws.crc, o_secs), secs.data(), sizeof(CrcSection) * secs.size(),
                          cudaMemcpyHostToDevice, st));
    CK(h, cudaMemcpyAsync(at<CrcPart>(ws.crc, o_parts), parts.data(), sizeof(CrcPart) * parts.size(),
                          cudaMemcpyHostToDevice, st));
    CK(h, cudaMemcpyAsync(at<int64_t>(ws.crc, o_first), first_part.data(), sizeof(int64_t) * first_part.size(),
                          cudaMemcpyHostToDevice, st));
    if (tr) tr->mark("host-layout");
    if (nblocks) {
        CK(h, launch_pack_blocks(at<PackBlock>(ws.crc, o_pack), nblocks, max_items, dev, st));
        h->launches += 1;
    }
    if (tr) tr->mark("pack");
    CK(h, launch_crc_sections(dev, at<CrcSection>(ws.crc, o_secs), nblocks + 1, at<CrcPart>(ws.crc, o_parts),
                              static_cast<int64_t>(parts.size()), at<int64_t>(ws.crc, o_first),
                              at<uint32_t>(ws.crc, o_pcrc), at<uint32_t>(ws.crc, o_crc), dev, st));
    h->launches += 2;
    if (tr) tr->mark("crc");
    // one device-to-host copy of the finished archive into pinned memory
    if (h->archive_cap < static_cast<size_t>(total)) {
        CK(h, cudaStreamSynchronize(st));
        const size_t want = std::max(static_cast<size_t>(total), h->archive_cap * 3 / 2);
        if (h->archive_pinned) cudaFreeHost(h->archive_pinned);
        h->archive_pinned = nullptr;
        h->archive_cap = 0;
        h->archive_size = 0;
        CK(h, cudaHostAlloc(reinterpret_cast<void**>(&h->archive_pinned), want, cudaHostAllocDefault));
        h->archive_cap = want;
    }
    CK(h, cudaMemcpyAsync(h->archive_pinned, dev, static_cast<size_t>(total), cudaMemcpyDeviceToHost, st));
    if (tr) tr->mark("d2h");
    CK(h, cudaStreamSynchronize(st));
    h->archive_size = static_cast<size_t>(total);
    *nbytes = total;
    return SPID_OK;
}

}  // namespace spidgpu

extern "C" {

int spidgpu_crc32(spidgpu_handle h, const void* data, int64_t nbytes, int32_t on_device,
                  uint32_t* out) {
    if (!h) return SPID_INVALID_ARGUMENT;
    if (!out || (nbytes > 0 && !data) || nbytes < 0)
        return fail(h, SPID_INVALID_ARGUMENT, "null buffer / negative length");
    cudaSetDevice(h->device);
    Workspace& ws = h->ws[0];
    cudaStream_t st = h->lanes[0];
    const uint8_t* src = static_cast<const uint8_t*>(data);
    Carve cv;
    const size_t o_data = on_device ? 0 : cv.take<uint8_t>(static_cast<size_t>(nbytes));
    const size_t o_scr = cv.take<uint32_t>(static_cast<size_t>(crc32_scratch_words(nbytes)));
    const size_t o_out = cv.take<uint32_t>(1);
    CK(h, ws.crc.ensure(cv.off, st));
    if (!on_device) {
        if (nbytes) {
            const int rc = upload_host_bytes(h, at<uint8_t>(ws.crc, o_data), src, nbytes, st);
            if (rc) return rc;
        }
        src = at<uint8_t>(ws.crc, o_data);
    }
    CK(h, launch_crc32(src, nbytes, at<uint32_t>(ws.crc, o_scr), at<uint32_t>(ws.crc, o_out), st));
    h->launches += 2;
    CK(h, cudaMemcpyAsync(out, at<uint32_t>(ws.crc, o_out), sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    CK(h, cudaStreamSynchronize(st));
    return SPID_OK;
}

int spidgpu_archive_compress(spidgpu_handle h, const double* a, int64_t m, int64_t n, int64_t lda,
                             int32_t a_on_device, const spidgpu_archive_spec* spec,
                             const spidgpu_rank_rule* rule, int64_t* nbytes) {
    NvtxRange nvtx_range("spidgpu.archive_compress");
    if (!h) return SPID_INVALID_ARGUMENT;
    if (!a || !spec || !rule || !nbytes) return fail(h, SPID_INVALID_ARGUMENT, "null argument");
    if (spec->mode != SPIDGPU_ARCHIVE_EXACT && spec->mode != SPIDGPU_ARCHIVE_SKETCH)
        return fail(h, SPID_INVALID_ARGUMENT, "unknown archive mode");
    // GridGeom::structured (grid.cpp:7-20), as the frame sidecar constructs it
    if (spec->naxes < 1 || spec->naxes > 3)
        return fail(h, SPID_BAD_GRID_GEOM, "structured grids have 1 to 3 axes");
    for (int ax = 0; ax < spec->naxes; ++ax)
        if (spec->dims[ax] < 2 || spec->dims[ax] > (1 << 20))
            return fail(h, SPID_BAD_GRID_GEOM, "each structured axis needs at least 2 points");
    const int naxes = spec->naxes;
    Layout L;
    std::vector<int64_t> blocks(spec->blocks_per_axis, spec->blocks_per_axis + naxes);
    int rc = make_domains(h, true, naxes, spec->dims, spec->periodic, 0, blocks, &L);
    if (rc) return rc;
    // RankRule::fixed / tolerance (qr.hpp:16-24), constructed after the domains
    if (rule->at_most) return fail(h, SPID_INVALID_ARGUMENT, "batch archives take a strict rank rule");
    if (rule->mode == SPIDGPU_RULE_FIXED) {
        if (rule->k < 1) return fail(h, SPID_BAD_RANK_RULE, "rank must be >= 1");
    } else if (rule->mode == SPIDGPU_RULE_TOL) {
        if (!(rule->tol > 0.0 && rule->tol < 1.0)) return fail(h, SPID_BAD_RANK_RULE, "tolerance must lie in (0, 1)");
    } else {
        return fail(h, SPID_BAD_RANK_RULE, "batch archives take a fixed or tolerance rule");
    }
    if (m < 1 || n < 1) return fail(h, SPID_EMPTY_MATRIX, "matrix dimensions must be at least 1x1");
    if (lda < m) return fail(h, SPID_INVALID_ARGUMENT, "lda < m");
    for (int ax = 0; ax < naxes; ++ax)
        if (spec->strides[ax] < 1) return fail(h, SPID_BAD_SUBSAMPLE_SPEC, "strides must be >= 1");
    if (m < L.points) return fail(h, SPID_INDEX_OUT_OF_RANGE, "row index out of range");  // select_rows
    const bool sketch = spec->mode == SPIDGPU_ARCHIVE_SKETCH;
    if (sketch && spec->ell < 1) return fail(h, SPID_EMPTY_SKETCH, "sketch needs ell >= 1");

    cudaSetDevice(h->device);
    Workspace& ws = h->ws[0];
    cudaStream_t st = h->lanes[0];
    const int64_t nblocks = static_cast<int64_t>(L.doms.size());

    // groups of equal local geometry, their coarse row maps and buffer plan
    std::vector<Group> groups = group_blocks(L, nullptr);
    struct GPlan {
        GridSpecDev g;
        int64_t P, Pc, nb, ldb, rows, kcap;
        std::vector<int64_t> rel;
        size_t o_rel, o_bases, o_B, o_Y, o_idx, o_uni, o_C, o_skel, o_rank, o_resid, o_status;
    };
    std::vector<GPlan> plans(groups.size());
    Carve cv;
    const size_t o_A = a_on_device ? 0 : cv.take<double>(static_cast<size_t>(m) * n);
    const size_t o_flags = cv.take<int32_t>(nblocks);
    int64_t max_items = 0;
    for (size_t gi = 0; gi < groups.size(); ++gi) {
        GPlan& p = plans[gi];
        const Group& G = groups[gi];
        rc = local_spec(h, L, G.proto, spec->strides, 1, &p.g, &p.P, &p.Pc);
        if (rc) return rc;
        const std::vector<int64_t> J = spec_rows(p.g, p.P);
        p.rel.resize(J.size());
        for (size_t i = 0; i < J.size(); ++i) p.rel[i] = globalize(L, G.proto, J[i]);
        p.nb = static_cast<int64_t>(G.members.size());
        p.ldb = (p.Pc + 1) & ~int64_t(1);  // even: TMA row pitch for the sketch
        p.rows = sketch ? spec->ell : p.Pc;
        const int64_t mn = std::min(p.rows, n);
        p.kcap = rule->mode == SPIDGPU_RULE_FIXED ? std::max<int64_t>(rule->k, 1) : std::max<int64_t>(mn, 1);
        if (p.Pc * p.kcap >= (int64_t(1) << 31) || p.kcap * n >= (int64_t(1) << 31))
            return fail(h, SPID_SHAPE_UNSUPPORTED, "block too large for the archive packer");
        p.o_rel = cv.take<int64_t>(p.rel.size());
        p.o_bases = cv.take<int64_t>(p.nb);
        p.o_B = cv.take<double>(static_cast<size_t>(p.nb * p.ldb * n));
        p.o_Y = sketch ? cv.take<double>(static_cast<size_t>(p.nb * spec->ell * n)) : 0;
        p.o_idx = cv.take<int64_t>(p.nb * p.kcap);
        p.o_uni = cv.take<int64_t>(p.nb * p.kcap);
        p.o_C = cv.take<double>(static_cast<size_t>(p.nb * p.kcap * n));
        p.o_skel = cv.take<double>(static_cast<size_t>(p.nb * p.Pc * p.kcap));
        p.o_rank = cv.take<int64_t>(p.nb);
        p.o_resid = cv.take<double>(p.nb);
        p.o_status = cv.take<int32_t>(p.nb);
        max_items = std::max(max_items, 8 + 2 * p.kcap + p.Pc * p.kcap + p.kcap * n);
    }
    CK(h, ws.bsk.ensure(cv.off, st));
    Trace tr(st);

    const double* A = a;
    int64_t ldA = lda;
    if (!a_on_device) {
        CK(h, cudaMemcpy2DAsync(at<double>(ws.bsk, o_A), sizeof(double) * m, a, sizeof(double) * lda,
                                sizeof(double) * m, n, cudaMemcpyHostToDevice, st));
        A = at<double>(ws.bsk, o_A);
        ldA = m;
    }
    // spid(): NonFiniteInput over each block's fine rows (id.cpp:68-69)
    BlockGridDev bg{};
    bg.naxes = naxes;
    for (int ax = 0; ax < 3; ++ax) {
        bg.dims[ax] = L.dims[ax];
        bg.seg_count[ax] = static_cast<int64_t>(L.segs[ax].size());
        bg.seg_base[ax] = std::max<int64_t>(1, L.dims[ax] / bg.seg_count[ax]);
    }
    CK(h, cudaMemsetAsync(at<int32_t>(ws.bsk, o_flags), 0, sizeof(int32_t) * nblocks, st));
    CK(h, launch_nonfinite_blocks(A, ldA, L.points, n, bg, at<int32_t>(ws.bsk, o_flags), st));
    h->launches += 1;
    tr.mark("h2d+scan");

    spidgpu_rank_rule r = *rule;
    for (size_t gi = 0; gi < groups.size(); ++gi) {
        GPlan& p = plans[gi];
        std::vector<int64_t> bases;
        for (int64_t b : groups[gi].members) bases.push_back(L.doms[b].base);
        CK(h, cudaMemcpyAsync(at<int64_t>(ws.bsk, p.o_rel), p.rel.data(), sizeof(int64_t) * p.rel.size(),
                              cudaMemcpyHostToDevice, st));
        CK(h, cudaMemcpyAsync(at<int64_t>(ws.bsk, p.o_bases), bases.data(), sizeof(int64_t) * bases.size(),
                              cudaMemcpyHostToDevice, st));
        double* B = at<double>(ws.bsk, p.o_B);
        // select_rows(a, domain.rows) then subsample(spec): B_b = A(base_b + rel, :)
        CK(h, launch_gather_block_rows(A, ldA, at<int64_t>(ws.bsk, p.o_rel), p.Pc,
                                       at<int64_t>(ws.bsk, p.o_bases), p.nb, n, B, p.ldb, p.ldb * n, st));
        h->launches += 1;
        tr.mark("gather");
        const double* Ycp = B;
        int64_t ldy = p.ldb, rows = p.Pc;
        if (sketch) {
            spidgpu_omega om{};
            om.mode = SPIDGPU_OMEGA_PHILOX;
            om.seed = spec->seed;
            om.subdomain_base = groups[gi].members[0];
            double* Y = at<double>(ws.bsk, p.o_Y);
            rc = do_sketch(h, ws, B, p.Pc, n, p.ldb, p.ldb * n, p.nb, spec->ell, &om, Y, spec->ell,
                           spec->ell * n, st);
            if (rc) return rc;
            Ycp = Y;
            ldy = spec->ell;
            rows = spec->ell;
            tr.mark("sketch");
        }
        CK(h, cudaMemsetAsync(at<double>(ws.bsk, p.o_C), 0, sizeof(double) * p.nb * p.kcap * n, st));
        rc = do_cpqr(h, ws, Ycp, rows, n, ldy, ldy * n, p.nb, &r, p.kcap, at<int64_t>(ws.bsk, p.o_idx),
                     at<double>(ws.bsk, p.o_C), p.kcap * n, at<int64_t>(ws.bsk, p.o_rank),
                     at<double>(ws.bsk, p.o_resid), at<int32_t>(ws.bsk, p.o_status), nullptr, nullptr,
                     nullptr, st);
        if (rc) return rc;
        tr.mark("cpqr");
        // f.base.skeleton = B(:, I) (id.cpp:82): coarse rows of the block
        rc = do_gather(h, B, p.Pc, n, p.ldb, p.ldb * n, p.nb, at<int64_t>(ws.bsk, p.o_idx), p.kcap,
                       at<int64_t>(ws.bsk, p.o_rank), at<double>(ws.bsk, p.o_skel), p.Pc, p.Pc * p.kcap, st);
        if (rc) return rc;
        CK(h, launch_sort_union(at<int64_t>(ws.bsk, p.o_idx), p.kcap, at<int64_t>(ws.bsk, p.o_rank), p.nb,
                                at<int64_t>(ws.bsk, p.o_uni), st));
        h->launches += 1;
        tr.mark("skel+sort");
    }
    // per-block ranks / statuses back to the host (one small copy per group)
    std::vector<int32_t> flags(nblocks);
    std::vector<int64_t> rank(nblocks);
    std::vector<int32_t> status(nblocks);
    std::vector<std::vector<int64_t>> grank(groups.size());
    std::vector<std::vector<int32_t>> gstat(groups.size());
    CK(h, cudaMemcpyAsync(flags.data(), at<int32_t>(ws.bsk, o_flags), sizeof(int32_t) * nblocks,
                          cudaMemcpyDeviceToHost, st));
    for (size_t gi = 0; gi < groups.size(); ++gi) {
        grank[gi].resize(plans[gi].nb);
        gstat[gi].resize(plans[gi].nb);
        CK(h, cudaMemcpyAsync(grank[gi].data(), at<int64_t>(ws.bsk, plans[gi].o_rank),
                              sizeof(int64_t) * plans[gi].nb, cudaMemcpyDeviceToHost, st));
        CK(h, cudaMemcpyAsync(gstat[gi].data(), at<int32_t>(ws.bsk, plans[gi].o_status),
                              sizeof(int32_t) * plans[gi].nb, cudaMemcpyDeviceToHost, st));
    }
    CK(h, cudaStreamSynchronize(st));
    std::vector<int64_t> gid(nblocks), pos(nblocks);
    for (size_t gi = 0; gi < groups.size(); ++gi)
        for (size_t t = 0; t < groups[gi].members.size(); ++t) {
            const int64_t b = groups[gi].members[t];
            gid[b] = static_cast<int64_t>(gi);
            pos[b] = static_cast<int64_t>(t);
            rank[b] = grank[gi][t];
            status[b] = gstat[gi][t];
        }
    for (int64_t b = 0; b < nblocks; ++b) {  // the reference stops at the first failing block
        if (flags[b]) return fail(h, SPID_NON_FINITE_INPUT, "input matrix contains NaN or infinity");
        if (status[b]) return fail(h, status[b], "column ID failed for block " + std::to_string(b));
    }

    // container layout: magic | u32 version | meta section | u64 count | blocks
    ArchiveMetaHost meta;
    meta.structured = true;
    for (int ax = 0; ax < naxes; ++ax) {
        meta.dims.push_back(static_cast<size_t>(spec->dims[ax]));
        meta.periodic.push_back(spec->periodic[ax] != 0);
        meta.blocks_per_axis.push_back(static_cast<size_t>(spec->blocks_per_axis[ax]));
        meta.strides.push_back(static_cast<size_t>(spec->strides[ax]));
    }
    meta.time_chunk = 0;
    meta.include_boundary = true;
    meta.mode = "batch";
    const bool fixed = rule->mode == SPIDGPU_RULE_FIXED;
    meta.rank_rule_mode = fixed ? "fixed" : "tolerance";
    meta.rank_k = fixed ? static_cast<size_t>(rule->k) : 0;
    meta.rank_tol = fixed ? 0.0 : rule->tol;
    meta.interp_recipe = "strided-multilinear";
    meta.qoi = spec->qoi ? spec->qoi : "";
    meta.m = static_cast<size_t>(m);
    meta.n = static_cast<size_t>(n);
    meta.provenance = spec->provenance ? spec->provenance : "";
    std::vector<PackBlock> pack(nblocks);
    for (int64_t b = 0; b < nblocks; ++b) {
        const GPlan& p = plans[gid[b]];
        const int64_t k = rank[b], t = pos[b];
        PackBlock& d = pack[b];
        d.k = k;
        d.nu = k;
        d.mc = p.Pc;
        d.n = n;
        d.coarse = p.Pc < L.doms[b].l[0] * L.doms[b].l[1] * L.doms[b].l[2] ? 1 : 0;
        d.uni = at<int64_t>(ws.bsk, p.o_uni) + t * p.kcap;
        d.sel = at<int64_t>(ws.bsk, p.o_idx) + t * p.kcap;
        d.skel = at<double>(ws.bsk, p.o_skel) + t * p.Pc * p.kcap;
        d.ld_s = p.Pc;
        d.coeffs = at<double>(ws.bsk, p.o_C) + t * p.kcap * n;
        d.ld_c = p.kcap;
    }
    return emit_archive(h, ws, meta, pack, st, &tr, nbytes);
}

int spidgpu_archive_fetch(spidgpu_handle h, uint8_t* dst, int64_t cap) {
    if (!h) return SPID_INVALID_ARGUMENT;
    if (!dst || cap < static_cast<int64_t>(h->archive_size))
        return fail(h, SPID_INVALID_ARGUMENT, "destination smaller than the archive");
    if (h->archive_size) std::memcpy(dst, h->archive_pinned, h->archive_size);
    return SPID_OK;
}

int spidgpu_archive_view(spidgpu_handle h, const uint8_t** data, int64_t* nbytes) {
    if (!h) return SPID_INVALID_ARGUMENT;
    if (!data || !nbytes) return fail(h, SPID_INVALID_ARGUMENT, "null output");
    *data = h->archive_pinned;
    *nbytes = static_cast<int64_t>(h->archive_size);
    return SPID_OK;
}

int spidgpu_archive_shape(const uint8_t* bytes, int64_t nbytes, int64_t* rows, int64_t* cols,
                          int64_t* blocks) {
    if (!bytes || nbytes < 0) return SPID_INVALID_ARGUMENT;
    Framing F;
    frame_archive(bytes, nbytes, &F);
    if (F.status) return F.status;
    ArchiveMetaHost meta;
    std::string msg;
    int rc = meta_from_json_bytes(bytes + F.secs[0].begin, static_cast<size_t>(F.secs[0].len), &meta, &msg);
    if (rc) return rc;
    Layout L;
    rc = layout_from_meta(nullptr, meta, &L);
    if (rc) return rc;
    int64_t c = 0;
    if (F.secs.size() > 1) {
        BlockRef b;
        rc = parse_block(bytes, F.secs[1], &b, &msg);
        if (rc) return rc;
        c = b.cc;
    }
    if (rows) *rows = L.points;
    if (cols) *cols = c;
    if (blocks) *blocks = static_cast<int64_t>(F.block_count);
    return SPID_OK;
}

int spidgpu_archive_info(spidgpu_handle h, const uint8_t* bytes, int64_t nbytes, char* out,
                         int64_t cap, int64_t* len) {
    if (!h) return SPID_INVALID_ARGUMENT;
    if (!bytes || nbytes < 0) return fail(h, SPID_INVALID_ARGUMENT, "null archive");
    cudaSetDevice(h->device);
    Decoded D;
    int rc = decode_archive(h, bytes, nbytes, &D, h->lanes[0]);
    if (rc) return rc;
    std::vector<size_t> ranks;
    size_t stored = 0;
    for (const BlockRef& b : D.blocks) {
        ranks.push_back(static_cast<size_t>(b.cr));
        stored += static_cast<size_t>(b.sr * b.sc + b.cr * b.cc);
    }
    // compression_factor (metrics.cpp:5-12)
    if (D.meta.m == 0 || D.meta.n == 0 || stored == 0)
        return fail(h, SPID_ZERO_DENOMINATOR, "matrix dimensions / stored entries must be positive");
    const double cf = static_cast<double>(D.meta.m) * static_cast<double>(D.meta.n) / static_cast<double>(stored);
    const std::string s = archive_info_string(D.meta, ranks, stored, cf);
    if (len) *len = static_cast<int64_t>(s.size());
    if (out) {
        if (cap < static_cast<int64_t>(s.size()) + 1) return fail(h, SPID_INVALID_ARGUMENT, "cap too small");
        std::memcpy(out, s.c_str(), s.size() + 1);
    }
    return SPID_OK;
}

int spidgpu_archive_decompress(spidgpu_handle h, const uint8_t* bytes, int64_t nbytes, double* out,
                               int64_t ldo, int32_t out_on_device) {
    NvtxRange nvtx_range("spidgpu.archive_decompress");
    if (!h) return SPID_INVALID_ARGUMENT;
    if (!bytes || !out || nbytes < 0) return fail(h, SPID_INVALID_ARGUMENT, "null argument");
    cudaSetDevice(h->device);
    Workspace& ws = h->ws[0];
    cudaStream_t st = h->lanes[0];
    Decoded D;
    Trace tr(st);
    int rc = decode_archive(h, bytes, nbytes, &D, st);  // leaves the archive bytes in ws.bytes
    tr.mark("h2d+crc");
    if (rc) return rc;
    const uint8_t* dev_bytes = ws.bytes.as<uint8_t>();
    Layout L;
    rc = layout_from_meta(h, D.meta, &L);
    if (rc) return rc;
    const int64_t nblocks = static_cast<int64_t>(L.doms.size());
    if (nblocks != static_cast<int64_t>(D.blocks.size()))
        return fail(h, SPID_COVERAGE_GAP, "block count does not match the partition plan");

    // per-block recipe checks in block order (archive.cpp:287-299)
    std::vector<int32_t> coarse(nblocks);
    std::vector<int64_t> lifted_rows(nblocks);
    const int64_t strides3[3] = {
        D.meta.strides.size() > 0 ? static_cast<int64_t>(D.meta.strides[0]) : 1,
        D.meta.strides.size() > 1 ? static_cast<int64_t>(D.meta.strides[1]) : 1,
        D.meta.strides.size() > 2 ? static_cast<int64_t>(D.meta.strides[2]) : 1};
    for (int64_t b = 0; b < nblocks; ++b) {
        const BlockRef& B = D.blocks[b];
        const Domain& d = L.doms[b];
        const int64_t drows = d.l[0] * d.l[1] * d.l[2];
        coarse[b] = B.coarse;
        if (B.coarse) {
            if (D.meta.interp_recipe != "strided-multilinear")
                return fail(h, SPID_UNSTRUCTURED_NO_INTERP, "coarse skeleton without an interpolation recipe");
            if (!L.structured) return fail(h, SPID_BAD_SUBSAMPLE_SPEC, "strided subsampling needs a structured grid");
            if (static_cast<int>(D.meta.strides.size()) != L.naxes)
                return fail(h, SPID_BAD_SUBSAMPLE_SPEC, "stride count must match axis count");
            for (size_t ax = 0; ax < D.meta.strides.size(); ++ax)
                if (D.meta.strides[ax] < 1) return fail(h, SPID_BAD_SUBSAMPLE_SPEC, "strides must be >= 1");
            GridSpecDev g;
            int64_t P = 0, Pc = 0;
            rc = local_spec(h, L, d, strides3, D.meta.include_boundary ? 1 : 0, &g, &P, &Pc);
            if (rc) return rc;
            if (B.sr != Pc) return fail(h, SPID_DIMENSION_MISMATCH, "coarse row count does not match operator");
        }
        if (B.sc != B.cr) return fail(h, SPID_DIMENSION_MISMATCH, "matmul inner dimensions disagree");
        lifted_rows[b] = B.coarse ? drows : B.sr;
    }
    // assemble (blocking.cpp:219-241)
    const int64_t ncols = D.blocks[0].cc;
    for (int64_t b = 0; b < nblocks; ++b) {
        const Domain& d = L.doms[b];
        if (D.blocks[b].cc != ncols) return fail(h, SPID_DIMENSION_MISMATCH, "blocks disagree on column count");
        if (lifted_rows[b] != d.l[0] * d.l[1] * d.l[2])
            return fail(h, SPID_DIMENSION_MISMATCH, "row set size does not match block rows");
    }
    const int64_t mout = L.points;
    if (ldo < mout) return fail(h, SPID_INVALID_ARGUMENT, "ldo < rows");
    if (ncols > (int64_t(1) << 31)) return fail(h, SPID_SHAPE_UNSUPPORTED, "too many columns");

    std::vector<Group> groups = group_blocks(L, &coarse);
    struct GPlan {
        GridSpecDev g;
        int64_t P, Pc, nb, mb, rows_s, kcap;
        std::vector<int64_t> rel;
        size_t o_rel, o_bases, o_S, o_F, o_C, o_rank, o_unpack;
    };
    std::vector<GPlan> plans(groups.size());
    Carve cv;
    const size_t o_out = out_on_device ? 0 : cv.take<double>(static_cast<size_t>(mout) * ncols);
    for (size_t gi = 0; gi < groups.size(); ++gi) {
        GPlan& p = plans[gi];
        const Group& G = groups[gi];
        p.nb = static_cast<int64_t>(G.members.size());
        p.mb = G.proto.l[0] * G.proto.l[1] * G.proto.l[2];
        p.kcap = 1;
        for (int64_t b : G.members) p.kcap = std::max(p.kcap, D.blocks[b].cr);
        if (p.kcap > 200 * 1024 / (8 * 65)) return fail(h, SPID_SHAPE_UNSUPPORTED, "rank too large for decompress");
        if (G.coarse) {
            rc = local_spec(h, L, G.proto, strides3, D.meta.include_boundary ? 1 : 0, &p.g, &p.P, &p.Pc);
            if (rc) return rc;
            p.rows_s = p.Pc;
        } else {
            p.rows_s = p.mb;
        }
        p.rel.resize(p.mb);
        for (int64_t l = 0; l < p.mb; ++l) p.rel[l] = L.structured ? globalize(L, G.proto, l) : l;
        p.o_rel = cv.take<int64_t>(p.rel.size());
        p.o_bases = cv.take<int64_t>(p.nb);
        p.o_S = cv.take<double>(static_cast<size_t>(p.nb * p.rows_s * p.kcap));
        p.o_F = G.coarse ? cv.take<double>(static_cast<size_t>(p.nb * p.mb * p.kcap)) : 0;
        p.o_C = cv.take<double>(static_cast<size_t>(p.nb * p.kcap * ncols));
        p.o_rank = cv.take<int64_t>(p.nb);
        p.o_unpack = cv.take<UnpackBlock>(p.nb);
    }
    CK(h, ws.bsk.ensure(cv.off, st));
    double* outd = out_on_device ? out : at<double>(ws.bsk, o_out);
    const int64_t ldd = out_on_device ? ldo : mout;
    for (size_t gi = 0; gi < groups.size(); ++gi) {
        GPlan& p = plans[gi];
        const Group& G = groups[gi];
        std::vector<int64_t> bases, ranks;
        std::vector<UnpackBlock> ub;
        int64_t max_items = 0;
        for (size_t t = 0; t < G.members.size(); ++t) {
            const int64_t b = G.members[t];
            const BlockRef& B = D.blocks[b];
            bases.push_back(L.doms[b].base);
            ranks.push_back(B.cr);
            UnpackBlock u;
            u.skel_off = B.skel_off;
            u.coef_off = B.coef_off;
            u.mc = B.sr;
            u.k = B.sc;
            u.n = B.cc;
            u.skel = at<double>(ws.bsk, p.o_S) + t * p.rows_s * p.kcap;
            u.ld_s = p.rows_s;
            u.coeffs = at<double>(ws.bsk, p.o_C) + t * p.kcap * ncols;
            u.ld_c = p.kcap;
            ub.push_back(u);
            max_items = std::max(max_items, B.sr * B.sc + B.cr * B.cc);
        }
        CK(h, cudaMemcpyAsync(at<int64_t>(ws.bsk, p.o_rel), p.rel.data(), sizeof(int64_t) * p.rel.size(),
                              cudaMemcpyHostToDevice, st));
        CK(h, cudaMemcpyAsync(at<int64_t>(ws.bsk, p.o_bases), bases.data(), sizeof(int64_t) * p.nb,
                              cudaMemcpyHostToDevice, st));
        CK(h, cudaMemcpyAsync(at<int64_t>(ws.bsk, p.o_rank), ranks.data(), sizeof(int64_t) * p.nb,
                              cudaMemcpyHostToDevice, st));
        CK(h, cudaMemcpyAsync(at<UnpackBlock>(ws.bsk, p.o_unpack), ub.data(), sizeof(UnpackBlock) * p.nb,
                              cudaMemcpyHostToDevice, st));
        CK(h, launch_unpack_blocks(dev_bytes, at<UnpackBlock>(ws.bsk, p.o_unpack), p.nb, max_items, st));
        tr.mark("unpack");
        h->launches += 1;
        const double* Fm = at<double>(ws.bsk, p.o_S);
        if (G.coarse) {  // lift.apply(skeleton) (interp.cpp:168-186)
            CK(h, launch_interp_apply(p.g, at<double>(ws.bsk, p.o_S), p.rows_s, p.rows_s * p.kcap, p.kcap,
                                      at<int64_t>(ws.bsk, p.o_rank), p.nb, at<double>(ws.bsk, p.o_F), p.mb,
                                      p.mb * p.kcap, nullptr, st));
            h->launches += 1;
            Fm = at<double>(ws.bsk, p.o_F);
            tr.mark("lift");
        }
        CK(h, launch_recon_scatter(Fm, p.mb, p.mb * p.kcap, at<double>(ws.bsk, p.o_C), p.kcap,
                                   p.kcap * ncols, at<int64_t>(ws.bsk, p.o_rank), p.nb, p.mb, ncols,
                                   at<int64_t>(ws.bsk, p.o_rel), at<int64_t>(ws.bsk, p.o_bases), outd, ldd,
                                   st));
        h->launches += 1;
        tr.mark("recon");
    }
    if (!out_on_device)
        CK(h, cudaMemcpy2DAsync(out, sizeof(double) * ldo, outd, sizeof(double) * mout, sizeof(double) * mout,
                                ncols, cudaMemcpyDeviceToHost, st));
    CK(h, cudaStreamSynchronize(st));
    return SPID_OK;
}

}  // extern "C"
