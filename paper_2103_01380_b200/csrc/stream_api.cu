// stream_api.cu -- spidgpu streaming two-stage compressor (run_pipeline,
// proj/src/pipeline.cpp:104-294) on the GPU.
//
// Ingestion runs on one CUDA stream (frame staging + coarse-row gather into
// the open chunk of every block), stage 1 on a second (batched
// column_id_at_most of all blocks' closed chunk + sorted skeleton columns),
// with two chunk buffers per block so ingestion of chunk c+1 overlaps stage 1
// of chunk c and waits only when two chunks are in flight -- the reference's
// backpressure bound (pipeline.cpp:184-189). Stage 2 and the archive run at
// finish. The host never touches snapshot data.
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "archive_internal.h"

using namespace spidgpu;

namespace spidgpu {
namespace stream_detail {

// stage-1 lanes: chunks in flight at once (each a chunk buffer, a stream and
// a column-ID workspace). Four lanes, with a narrow column-ID variant capped
// at 96 registers and a 96 KB ring so that two CTAs share an SM, measured
// -7% device-frame time at best but +1.5% with host frames and a wider
// spread (more buffers to allocate per stream); two it is.
constexpr int kLanes = 2;

struct ChunkArena {  // one closed chunk of one geometry group
    void* mem = nullptr;
    int64_t cols = 0, col0 = 0, kcap = 0;
    size_t o_idx = 0, o_rank = 0, o_resid = 0, o_status = 0, o_C0 = 0, o_sidx = 0, o_spos = 0, o_skel = 0;
    template <class T>
    T* p(size_t off) const {
        return reinterpret_cast<T*>(static_cast<uint8_t*>(mem) + off);
    }
};

struct SGroup {
    Group G;
    GridSpecDev g{};
    int64_t P = 0, Pc = 0, nb = 0;
    std::vector<int64_t> rel, bases;
    DevBuf rel_d, bases_d, chunkbuf[kLanes], fin;
    bool used[kLanes] = {};
    std::vector<ChunkArena> chunks;
};

}  // namespace stream_detail
}  // namespace spidgpu

using spidgpu::stream_detail::ChunkArena;
using spidgpu::stream_detail::kLanes;
using spidgpu::stream_detail::SGroup;

struct spidgpu_stream {
    spidgpu_handle h = nullptr;
    spidgpu_stream_config cfg{};
    std::string qoi, provenance;
    Layout L;
    std::vector<SGroup> groups;
    // chunk c's stage 1 runs on lane c % kLanes (its own chunk buffer,
    // stream and workspace), so several chunks' column IDs (64 CTAs each for
    // 64 blocks) share the GPU instead of queueing behind each other; lane
    // 0's stream (s_cmp) then runs stage 2 and the archive
    cudaStream_t s_in = nullptr, s_lane[kLanes] = {};
    cudaStream_t& s_cmp = s_lane[0];
    cudaEvent_t ready = nullptr, free_ev[kLanes] = {};
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> s1_events;
    // event log (spid::TaskEvent): device-timeline events
    cudaEvent_t t0 = nullptr, f0 = nullptr, f1 = nullptr;  // open; stage 2 start / end
    struct Push {
        cudaEvent_t b, e;  // ingestion of frames [first, first + count) on s_in
        int64_t first, count;
    };
    std::vector<Push> pushes;
    std::vector<cudaEvent_t> closes;  // chunk c ingested (recorded before its stage 1)
    Workspace ws_lane[kLanes], ws_fin;
    // host frames land in alternating staging buffers: the gather of one push
    // (same stream, so ordered before the buffer's next copy) overlaps the
    // next push's copy; a push returns once its own copy has read the host data
    DevBuf staging[2];
    int64_t staged[2] = {0, 0};  // entries each staging buffer holds
    cudaEvent_t copied = nullptr;
    cudaStream_t s_copy = nullptr;           // host frames' copies into staging
    cudaEvent_t stg_free[2] = {nullptr, nullptr};  // the gather that last read staging[i] is done
    bool stg_used[2] = {false, false};
    int stg = 0;
    int64_t filled = 0, snapshots = 0, nchunks = 0, stage1_tasks = 0, stage2_tasks = 0;
    int64_t fine_peak = 0, coarse_peak = 0;
    double stage2_ms = 0.0;
    int cur = 0;
    bool finished = false;
    std::string last_error;
};

namespace {

int sfail(spidgpu_stream* s, int code, const std::string& msg) {
    fail(s->h, code, msg);
    s->last_error = std::string(spidgpu_status_name(code)) + ": " + msg;
    return code;
}

#define SCK(s, expr)                                                                   \
    do {                                                                               \
        cudaError_t _e = (expr);                                                       \
        if (_e != cudaSuccess)                                                         \
            return sfail((s), SPID_CUDA_ERROR, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
    } while (0)

#define SRC(s, expr)                                                   \
    do {                                                               \
        int _rc = (expr);                                              \
        if (_rc) {                                                     \
            (s)->last_error = (s)->h->last_error;                      \
            return _rc;                                                \
        }                                                              \
    } while (0)

// Stage 1 of every block's closed chunk (pipeline.cpp:192-215 ->
// stage1_compress_coarse, blocking.cpp:112-115).
int close_chunk(spidgpu_stream* s) {
    NvtxRange nvtx_range("spidgpu.stream.stage1");
    const int64_t cols = s->filled;
    if (cols == 0) return SPID_OK;
    const int64_t T = s->cfg.time_chunk;
    const int64_t kcap = std::min<int64_t>(s->cfg.stage1_rank, cols);
    cudaStream_t sc = s->s_lane[s->cur];  // chunk buffer cur's stage-1 stream
    Workspace& wsc = s->ws_lane[s->cur];
    SCK(s, cudaEventRecord(s->ready, s->s_in));
    SCK(s, cudaStreamWaitEvent(sc, s->ready, 0));
    cudaEvent_t ce;
    SCK(s, cudaEventCreate(&ce));
    SCK(s, cudaEventRecord(ce, s->s_in));
    s->closes.push_back(ce);
    cudaEvent_t e0, e1;
    SCK(s, cudaEventCreate(&e0));
    SCK(s, cudaEventCreate(&e1));
    SCK(s, cudaEventRecord(e0, sc));
    spidgpu_rank_rule rule{SPIDGPU_RULE_FIXED, 1, kcap, 0, 0.0};  // column_id_at_most(chunk, min(k, cols))
    for (SGroup& g : s->groups) {
        ChunkArena c;
        c.cols = cols;
        c.col0 = s->snapshots - cols;
        c.kcap = kcap;
        Carve cv;
        c.o_idx = cv.take<int64_t>(g.nb * kcap);
        c.o_rank = cv.take<int64_t>(g.nb);
        c.o_resid = cv.take<double>(g.nb);
        c.o_status = cv.take<int32_t>(g.nb);
        c.o_C0 = cv.take<double>(g.nb * kcap * cols);
        c.o_sidx = cv.take<int64_t>(g.nb * kcap);
        c.o_spos = cv.take<int32_t>(g.nb * kcap);
        c.o_skel = cv.take<double>(g.nb * kcap * g.Pc);
        SCK(s, cudaMallocAsync(&c.mem, cv.off, sc));
        const double* chunk = g.chunkbuf[s->cur].as<double>();
        SRC(s, do_cpqr(s->h, wsc, chunk, g.Pc, cols, g.Pc, g.Pc * T, g.nb, &rule, kcap,
                       c.p<int64_t>(c.o_idx), c.p<double>(c.o_C0), kcap * cols, c.p<int64_t>(c.o_rank),
                       c.p<double>(c.o_resid), c.p<int32_t>(c.o_status), nullptr, nullptr, nullptr, sc));
        // skeleton = the chunk's coarse columns, kept in sorted (union) order
        SCK(s, launch_sort_pairs(c.p<int64_t>(c.o_idx), c.p<int64_t>(c.o_rank), kcap, g.nb,
                                 c.p<int64_t>(c.o_sidx), c.p<int32_t>(c.o_spos), sc));
        SCK(s, launch_gather_cols(chunk, g.Pc, g.Pc, g.Pc * T, g.nb, c.p<int64_t>(c.o_sidx), kcap,
                                  c.p<int64_t>(c.o_rank), cols, c.p<double>(c.o_skel), g.Pc, g.Pc * kcap,
                                  nullptr, sc));
        s->h->launches += 2;
        g.used[s->cur] = true;
        g.chunks.push_back(c);
        s->stage1_tasks += g.nb;
    }
    SCK(s, cudaEventRecord(e1, sc));
    SCK(s, cudaEventRecord(s->free_ev[s->cur], sc));
    s->s1_events.emplace_back(e0, e1);
    s->cur = (s->cur + 1) % kLanes;
    s->filled = 0;
    s->nchunks += 1;
    return SPID_OK;
}

// the begin / end events of one push on the ingestion stream (event log)
struct Stream_push_log {
    spidgpu_stream* s;
    spidgpu_stream::Push p{};
    Stream_push_log(spidgpu_stream* st, int64_t count) : s(st) {
        p.first = s->snapshots;
        p.count = count;
        if (count > 0 && cudaEventCreate(&p.b) == cudaSuccess) cudaEventRecord(p.b, s->s_in);
    }
    ~Stream_push_log() {
        if (!p.b) return;
        if (cudaEventCreate(&p.e) == cudaSuccess && cudaEventRecord(p.e, s->s_in) == cudaSuccess)
            s->pushes.push_back(p);
        else
            cudaEventDestroy(p.b);
    }
};

void destroy(spidgpu_stream* s) {
    for (cudaStream_t st : s->s_lane)
        if (st) cudaStreamSynchronize(st);
    if (s->s_in) cudaStreamSynchronize(s->s_in);
    if (s->s_copy) cudaStreamSynchronize(s->s_copy);
    for (SGroup& g : s->groups) {
        for (ChunkArena& c : g.chunks)
            if (c.mem) cudaFree(c.mem);
        g.rel_d.release();
        g.bases_d.release();
        for (DevBuf& cb : g.chunkbuf) cb.release();
        g.fin.release();
    }
    for (Workspace& w : s->ws_lane) w.release();
    s->ws_fin.release();
    s->staging[0].release();
    s->staging[1].release();
    if (s->copied) cudaEventDestroy(s->copied);
    for (cudaEvent_t e : s->stg_free)
        if (e) cudaEventDestroy(e);
    for (auto& e : s->s1_events) {
        cudaEventDestroy(e.first);
        cudaEventDestroy(e.second);
    }
    for (auto& p : s->pushes) {
        cudaEventDestroy(p.b);
        cudaEventDestroy(p.e);
    }
    for (cudaEvent_t e : s->closes) cudaEventDestroy(e);
    for (cudaEvent_t e : {s->t0, s->f0, s->f1})
        if (e) cudaEventDestroy(e);
    if (s->ready) cudaEventDestroy(s->ready);
    for (cudaEvent_t e : s->free_ev)
        if (e) cudaEventDestroy(e);
    if (s->s_in) cudaStreamDestroy(s->s_in);
    if (s->s_copy) cudaStreamDestroy(s->s_copy);
    for (cudaStream_t st : s->s_lane)
        if (st) cudaStreamDestroy(st);
}

}  // namespace

extern "C" {

int spidgpu_stream_open(spidgpu_handle h, const spidgpu_stream_config* cfg, spidgpu_stream_handle* out) {
    if (!h) return SPID_INVALID_ARGUMENT;
    if (!cfg || !out) return fail(h, SPID_INVALID_ARGUMENT, "null argument");
    *out = nullptr;
    // GridGeom::structured (grid.cpp:7-20), then run_pipeline's checks in order
    if (cfg->naxes < 1 || cfg->naxes > 3) return fail(h, SPID_BAD_GRID_GEOM, "structured grids have 1 to 3 axes");
    for (int ax = 0; ax < cfg->naxes; ++ax)
        if (cfg->dims[ax] < 2 || cfg->dims[ax] > (1 << 20))
            return fail(h, SPID_BAD_GRID_GEOM, "each structured axis needs at least 2 points");
    if (cfg->time_chunk < 1) return fail(h, SPID_BAD_STREAM_CONFIG, "time_chunk must be >= 1");
    if (cfg->stage1_rank < 1) return fail(h, SPID_BAD_STREAM_CONFIG, "stage-1 rank must be >= 1");
    cudaSetDevice(h->device);
    auto* s = new spidgpu_stream();
    s->h = h;
    s->cfg = *cfg;
    s->qoi = cfg->qoi ? cfg->qoi : "";
    s->provenance = cfg->provenance ? cfg->provenance : "";
    s->cfg.qoi = nullptr;
    s->cfg.provenance = nullptr;
    std::vector<int64_t> blocks(cfg->blocks_per_axis, cfg->blocks_per_axis + cfg->naxes);
    int rc = make_domains(h, true, cfg->naxes, cfg->dims, cfg->periodic, 0, blocks, &s->L);
    if (rc) {
        delete s;
        return rc;
    }
    for (int ax = 0; ax < cfg->naxes; ++ax)
        if (cfg->strides[ax] < 1) {
            delete s;
            return fail(h, SPID_BAD_SUBSAMPLE_SPEC, "strides must be >= 1");
        }
    auto bail = [&](int code) {
        destroy(s);
        delete s;
        return code;
    };
    bool lanes_ok = true;
    for (int l = 0; l < kLanes; ++l)
        lanes_ok = lanes_ok && cudaStreamCreateWithFlags(&s->s_lane[l], cudaStreamNonBlocking) == cudaSuccess &&
                   cudaEventCreateWithFlags(&s->free_ev[l], cudaEventDisableTiming) == cudaSuccess;
    if (!lanes_ok || cudaStreamCreateWithFlags(&s->s_in, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&s->s_copy, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&s->stg_free[0], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&s->stg_free[1], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&s->ready, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&s->copied, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreate(&s->t0) != cudaSuccess || cudaEventRecord(s->t0, s->s_in) != cudaSuccess)
        return bail(fail(h, SPID_CUDA_ERROR, "stream/event creation failed"));
    for (const Group& G : group_blocks(s->L, nullptr)) {
        SGroup g;
        g.G = G;
        // SubsampleSpec::strided(domain.local, strides, include_boundary).row_indices()
        rc = local_spec(h, s->L, G.proto, cfg->strides, cfg->include_boundary ? 1 : 0, &g.g, &g.P, &g.Pc,
                        /*lift=*/false);
        if (rc) return bail(rc);
        const std::vector<int64_t> J = spec_rows(g.g, g.P);
        g.rel.resize(J.size());
        for (size_t i = 0; i < J.size(); ++i) g.rel[i] = globalize(s->L, G.proto, J[i]);
        for (int64_t b : G.members) g.bases.push_back(s->L.doms[b].base);
        g.nb = static_cast<int64_t>(G.members.size());
        s->groups.push_back(std::move(g));
    }
    for (SGroup& g : s->groups) {
        if (to_dev(h, g.rel_d, g.rel.data(), g.rel.size(), s->s_in) ||
            to_dev(h, g.bases_d, g.bases.data(), g.bases.size(), s->s_in))
            return bail(SPID_CUDA_ERROR);
        const size_t cb = sizeof(double) * g.nb * g.Pc * cfg->time_chunk;
        for (DevBuf& buf : g.chunkbuf)
            if (buf.ensure(cb, s->s_in) != cudaSuccess)
                return bail(fail(h, SPID_CUDA_ERROR, "chunk buffer allocation failed"));
        s->coarse_peak += kLanes * g.nb * g.Pc * cfg->time_chunk;
    }
    *out = s;
    return SPID_OK;
}

int spidgpu_stream_push(spidgpu_stream_handle s, const double* frames, int64_t m, int64_t count, int64_t ld,
                        int32_t on_device) {
    if (!s) return SPID_INVALID_ARGUMENT;
    if (s->finished) return sfail(s, SPID_INVALID_ARGUMENT, "stream already finished");
    if (count < 0 || (count > 0 && !frames)) return sfail(s, SPID_INVALID_ARGUMENT, "bad frames");
    if (m != s->L.points)  // pipeline.cpp:116-117
        return sfail(s, SPID_GEOMETRY_MISMATCH, "producer frame size does not match grid");
    if (count > 0 && ld < m) return sfail(s, SPID_INVALID_ARGUMENT, "ld < m");
    if (on_device < 0 || on_device > 2) return sfail(s, SPID_INVALID_ARGUMENT, "on_device must be 0, 1 or 2");
    // 0: host frames, read before the call returns; 1: device frames, 2: host
    // frames, both read asynchronously (the caller keeps them unmodified
    // until finish)
    const bool dev = on_device == 1, async = on_device != 0;
    cudaSetDevice(s->h->device);
    const int64_t T = s->cfg.time_chunk;
    Stream_push_log log(s, count);
    for (int64_t j = 0; j < count;) {
        const int64_t c = std::min(count - j, T - s->filled);
        const double* src = frames + j * ld;
        int64_t lds = ld;
        const int bi = s->stg;
        if (!dev) {  // stage the frames (the only fine-grid data the stream holds)
            DevBuf& sb = s->staging[bi];
            const size_t need = sizeof(double) * m * c;
            s->staged[bi] = m * c;
            s->stg ^= 1;
            if (sb.bytes < need) {  // reallocation: no reader or writer left
                SCK(s, cudaStreamSynchronize(s->s_copy));
                SCK(s, cudaStreamSynchronize(s->s_in));
            }
            SCK(s, sb.ensure(need, s->s_in));
            if (async) {
                // on their own copy stream, so that a frame's copy does not
                // queue behind the previous frame's gather; a staging buffer
                // is rewritten only after the gather that read it
                if (s->stg_used[bi]) SCK(s, cudaStreamWaitEvent(s->s_copy, s->stg_free[bi], 0));
                SCK(s, cudaMemcpy2DAsync(sb.ptr, sizeof(double) * m, src, sizeof(double) * ld,
                                         sizeof(double) * m, c, cudaMemcpyHostToDevice, s->s_copy));
                SCK(s, cudaEventRecord(s->copied, s->s_copy));
                SCK(s, cudaStreamWaitEvent(s->s_in, s->copied, 0));
            } else {
                // the host waits for this copy anyway: in stream order on s_in
                // (measured faster than the cross-stream hand-off per frame)
                SCK(s, cudaMemcpy2DAsync(sb.ptr, sizeof(double) * m, src, sizeof(double) * ld,
                                         sizeof(double) * m, c, cudaMemcpyHostToDevice, s->s_in));
                SCK(s, cudaEventRecord(s->copied, s->s_in));
            }
            src = sb.as<double>();
            lds = m;
            s->fine_peak = std::max(s->fine_peak, s->staged[0] + s->staged[1]);
        }
        if (s->filled == 0 && s->groups[0].used[s->cur])  // <= kLanes chunks in flight
            SCK(s, cudaStreamWaitEvent(s->s_in, s->free_ev[s->cur], 0));
        for (SGroup& g : s->groups) {
            double* B = g.chunkbuf[s->cur].as<double>() + s->filled * g.Pc;
            SCK(s, launch_gather_block_rows(src, lds, g.rel_d.as<int64_t>(), g.Pc, g.bases_d.as<int64_t>(), g.nb, c,
                                            B, g.Pc, g.Pc * T, s->s_in));
            s->h->launches += 1;
        }
        if (!dev) {
            SCK(s, cudaEventRecord(s->stg_free[bi], s->s_in));
            s->stg_used[bi] = true;
        }
        s->filled += c;
        s->snapshots += c;
        j += c;
        if (s->filled == T) {
            const int rc = close_chunk(s);
            if (rc) return rc;
        }
    }
    if (!async) SCK(s, cudaEventSynchronize(s->copied));  // the host frames have been read
    return SPID_OK;
}

int spidgpu_stream_finish(spidgpu_stream_handle s, int64_t* nbytes) {
    NvtxRange nvtx_range("spidgpu.stream.finish");
    if (!s) return SPID_INVALID_ARGUMENT;
    if (!nbytes) return sfail(s, SPID_INVALID_ARGUMENT, "null nbytes");
    if (s->finished) return sfail(s, SPID_INVALID_ARGUMENT, "stream already finished");
    cudaSetDevice(s->h->device);
    int rc = close_chunk(s);  // final short chunks (pipeline.cpp:249)
    if (rc) return rc;
    if (s->snapshots == 0) return sfail(s, SPID_SHORT_STREAM, "producer yielded no snapshots");
    for (cudaStream_t st : s->s_lane) SCK(s, cudaStreamSynchronize(st));
    s->finished = true;
    const int64_t nblocks = static_cast<int64_t>(s->L.doms.size());
    const int64_t n_total = s->snapshots, T = s->cfg.time_chunk;

    // ---- stage-1 failures: first (chunk, block) in ingestion order (pipeline.cpp:159-171, 252-255)
    std::vector<std::vector<std::vector<int64_t>>> ranks(s->groups.size());  // [group][chunk][member]
    {
        std::vector<int32_t> st_all(static_cast<size_t>(s->nchunks * nblocks), 0);
        for (size_t gi = 0; gi < s->groups.size(); ++gi) {
            SGroup& g = s->groups[gi];
            ranks[gi].resize(g.chunks.size());
            for (size_t c = 0; c < g.chunks.size(); ++c) {
                std::vector<int32_t> st(g.nb);
                ranks[gi][c].resize(g.nb);
                SCK(s, cudaMemcpy(st.data(), g.chunks[c].p<int32_t>(g.chunks[c].o_status), sizeof(int32_t) * g.nb,
                                  cudaMemcpyDeviceToHost));
                SCK(s, cudaMemcpy(ranks[gi][c].data(), g.chunks[c].p<int64_t>(g.chunks[c].o_rank),
                                  sizeof(int64_t) * g.nb, cudaMemcpyDeviceToHost));
                for (int64_t t = 0; t < g.nb; ++t) st_all[c * nblocks + g.G.members[t]] = st[t];
            }
        }
        for (int64_t c = 0; c < s->nchunks; ++c)
            for (int64_t b = 0; b < nblocks; ++b)
                if (const int32_t code = st_all[c * nblocks + b])
                    return sfail(s, code, "stage-1 failed on block " + std::to_string(b) + ", chunk " +
                                              std::to_string(c) + ": " + spidgpu_status_name(code));
    }

    // ---- stage 2 per geometry group (blocking.cpp:128-204) ---------------------------------
    SCK(s, cudaEventCreate(&s->f0));
    SCK(s, cudaEventCreate(&s->f1));
    cudaEvent_t f0 = s->f0, f1 = s->f1;
    SCK(s, cudaEventRecord(f0, s->s_cmp));
    spidgpu_rank_rule rule2{SPIDGPU_RULE_TOL, 0, 0, 0, s->cfg.stage2_tol};
    struct Fin {
        int64_t rmax, kcap2, nch;
        size_t o_tab, o_concat, o_uglob, o_upos, o_uoff, o_R, o_idx2, o_C1, o_rank2, o_resid2, o_st2, o_C, o_bad,
            o_fskel, o_fglob;
    };
    std::vector<Fin> fins(s->groups.size());
    for (size_t gi = 0; gi < s->groups.size(); ++gi) {
        SGroup& g = s->groups[gi];
        Fin& f = fins[gi];
        f.nch = static_cast<int64_t>(g.chunks.size());
        f.rmax = 1;
        for (int64_t t = 0; t < g.nb; ++t) {
            int64_t R = 0;
            for (int64_t c = 0; c < f.nch; ++c) R += ranks[gi][c][t];
            f.rmax = std::max(f.rmax, R);
        }
        f.kcap2 = std::max<int64_t>(1, std::min(g.Pc, f.rmax));
        Carve cv;
        f.o_tab = cv.take<StreamChunkDev>(f.nch);
        f.o_concat = cv.take<double>(g.nb * f.rmax * g.Pc);
        f.o_uglob = cv.take<int64_t>(g.nb * f.rmax);
        f.o_upos = cv.take<int32_t>(g.nb * f.rmax);
        f.o_uoff = cv.take<int64_t>(g.nb * (f.nch + 1));
        f.o_R = cv.take<int64_t>(g.nb);
        f.o_idx2 = cv.take<int64_t>(g.nb * f.kcap2);
        f.o_C1 = cv.take<double>(g.nb * f.kcap2 * f.rmax);
        f.o_rank2 = cv.take<int64_t>(g.nb);
        f.o_resid2 = cv.take<double>(g.nb);
        f.o_st2 = cv.take<int32_t>(g.nb);
        f.o_C = cv.take<double>(g.nb * f.kcap2 * n_total);
        f.o_bad = cv.take<int32_t>(g.nb);
        f.o_fskel = cv.take<double>(g.nb * f.kcap2 * g.Pc);
        f.o_fglob = cv.take<int64_t>(g.nb * f.kcap2);
        SCK(s, g.fin.ensure(cv.off, s->s_cmp));
        std::vector<StreamChunkDev> tab(f.nch);
        for (int64_t c = 0; c < f.nch; ++c) {
            const ChunkArena& a = g.chunks[c];
            tab[c] = {a.p<double>(a.o_skel), a.p<int64_t>(a.o_sidx), a.p<int32_t>(a.o_spos),
                      a.p<int64_t>(a.o_rank), a.p<double>(a.o_C0), a.kcap, a.cols, a.col0};
        }
        SCK(s, cudaMemcpyAsync(at<StreamChunkDev>(g.fin, f.o_tab), tab.data(), sizeof(StreamChunkDev) * f.nch,
                               cudaMemcpyHostToDevice, s->s_cmp));
        SCK(s, cudaMemsetAsync(at<double>(g.fin, f.o_concat), 0, sizeof(double) * g.nb * f.rmax * g.Pc, s->s_cmp));
        SCK(s, cudaMemsetAsync(at<int32_t>(g.fin, f.o_bad), 0, sizeof(int32_t) * g.nb, s->s_cmp));
        SCK(s, launch_concat_union(at<StreamChunkDev>(g.fin, f.o_tab), f.nch, g.nb, g.Pc, f.rmax,
                                   at<double>(g.fin, f.o_concat), at<int64_t>(g.fin, f.o_uglob),
                                   at<int32_t>(g.fin, f.o_upos), at<int64_t>(g.fin, f.o_uoff),
                                   at<int64_t>(g.fin, f.o_R), s->s_cmp));
        // column_id(concat, RankRule::tolerance(stage2_tol)) (blocking.cpp:178)
        SRC(s, do_cpqr(s->h, s->ws_fin, at<double>(g.fin, f.o_concat), g.Pc, f.rmax, g.Pc, g.Pc * f.rmax, g.nb,
                       &rule2, f.kcap2, at<int64_t>(g.fin, f.o_idx2), at<double>(g.fin, f.o_C1), f.kcap2 * f.rmax,
                       at<int64_t>(g.fin, f.o_rank2), at<double>(g.fin, f.o_resid2), at<int32_t>(g.fin, f.o_st2),
                       nullptr, nullptr, nullptr, s->s_cmp));
        SCK(s, launch_compose(at<StreamChunkDev>(g.fin, f.o_tab), f.nch, T, n_total, at<double>(g.fin, f.o_C1),
                              f.kcap2, f.rmax, at<int64_t>(g.fin, f.o_rank2), at<int32_t>(g.fin, f.o_upos),
                              at<int64_t>(g.fin, f.o_uoff), g.nb, at<double>(g.fin, f.o_C),
                              at<int32_t>(g.fin, f.o_bad), s->s_cmp));
        SCK(s, launch_gather_cols(at<double>(g.fin, f.o_concat), g.Pc, g.Pc, g.Pc * f.rmax, g.nb,
                                  at<int64_t>(g.fin, f.o_idx2), f.kcap2, at<int64_t>(g.fin, f.o_rank2), f.rmax,
                                  at<double>(g.fin, f.o_fskel), g.Pc, g.Pc * f.kcap2, nullptr, s->s_cmp));
        SCK(s, launch_final_global(at<int64_t>(g.fin, f.o_idx2), at<int64_t>(g.fin, f.o_rank2), f.kcap2,
                                   at<int64_t>(g.fin, f.o_uglob), f.rmax, g.nb, at<int64_t>(g.fin, f.o_fglob),
                                   s->s_cmp));
        s->h->launches += 5;
        s->stage2_tasks += g.nb;
    }
    // stage-2 outcomes, reported in block order (pipeline.cpp:277-289)
    std::vector<int64_t> rank2(nblocks), R(nblocks);
    std::vector<int32_t> st2(nblocks), bad(nblocks);
    std::vector<int64_t> gid(nblocks), pos(nblocks);
    for (size_t gi = 0; gi < s->groups.size(); ++gi) {
        SGroup& g = s->groups[gi];
        const Fin& f = fins[gi];
        std::vector<int64_t> r2(g.nb), rr(g.nb);
        std::vector<int32_t> s2(g.nb), bd(g.nb);
        SCK(s, cudaMemcpyAsync(r2.data(), at<int64_t>(g.fin, f.o_rank2), sizeof(int64_t) * g.nb,
                               cudaMemcpyDeviceToHost, s->s_cmp));
        SCK(s, cudaMemcpyAsync(rr.data(), at<int64_t>(g.fin, f.o_R), sizeof(int64_t) * g.nb, cudaMemcpyDeviceToHost,
                               s->s_cmp));
        SCK(s, cudaMemcpyAsync(s2.data(), at<int32_t>(g.fin, f.o_st2), sizeof(int32_t) * g.nb,
                               cudaMemcpyDeviceToHost, s->s_cmp));
        SCK(s, cudaMemcpyAsync(bd.data(), at<int32_t>(g.fin, f.o_bad), sizeof(int32_t) * g.nb,
                               cudaMemcpyDeviceToHost, s->s_cmp));
        SCK(s, cudaStreamSynchronize(s->s_cmp));
        for (int64_t t = 0; t < g.nb; ++t) {
            const int64_t b = g.G.members[t];
            rank2[b] = r2[t];
            R[b] = rr[t];
            st2[b] = s2[t];
            bad[b] = bd[t];
            gid[b] = static_cast<int64_t>(gi);
            pos[b] = t;
        }
    }
    for (int64_t b = 0; b < nblocks; ++b) {
        if (st2[b]) return sfail(s, st2[b], "stage 2 failed on block " + std::to_string(b));
        if (bad[b]) return sfail(s, SPID_NON_FINITE_COEFFS, "composed coefficients contain NaN or infinity");
    }

    // ---- the "two-stage" archive (pipeline.cpp:259-291) -------------------------------------
    ArchiveMetaHost meta;
    meta.structured = true;
    for (int ax = 0; ax < s->cfg.naxes; ++ax) {
        meta.dims.push_back(static_cast<size_t>(s->cfg.dims[ax]));
        meta.periodic.push_back(s->cfg.periodic[ax] != 0);
        meta.blocks_per_axis.push_back(static_cast<size_t>(s->cfg.blocks_per_axis[ax]));
        meta.strides.push_back(static_cast<size_t>(s->cfg.strides[ax]));
    }
    meta.time_chunk = static_cast<size_t>(T);
    meta.include_boundary = s->cfg.include_boundary != 0;
    meta.mode = "two-stage";
    meta.rank_rule_mode = "fixed";
    meta.rank_k = static_cast<size_t>(s->cfg.stage1_rank);
    meta.rank_tol = 0.0;
    meta.stage2_tol = s->cfg.stage2_tol;
    meta.interp_recipe = "strided-multilinear";
    meta.qoi = s->qoi;
    meta.m = static_cast<size_t>(s->L.points);
    meta.n = static_cast<size_t>(n_total);
    meta.provenance = s->provenance;
    std::vector<PackBlock> pack(nblocks);
    for (int64_t b = 0; b < nblocks; ++b) {
        SGroup& g = s->groups[gid[b]];
        const Fin& f = fins[gid[b]];
        const int64_t t = pos[b];
        const Domain& d = s->L.doms[b];
        PackBlock& pb = pack[b];
        pb.k = rank2[b];
        pb.nu = R[b];
        pb.mc = g.Pc;
        pb.n = n_total;
        pb.coarse = g.Pc < d.l[0] * d.l[1] * d.l[2] ? 1 : 0;
        pb.uni = at<int64_t>(g.fin, f.o_uglob) + t * f.rmax;
        pb.sel = at<int64_t>(g.fin, f.o_fglob) + t * f.kcap2;
        pb.skel = at<double>(g.fin, f.o_fskel) + t * f.kcap2 * g.Pc;
        pb.ld_s = g.Pc;
        pb.coeffs = at<double>(g.fin, f.o_C) + t * f.kcap2 * n_total;
        pb.ld_c = f.kcap2;
    }
    rc = emit_archive(s->h, s->ws_fin, meta, pack, s->s_cmp, nullptr, nbytes);
    if (rc) {
        s->last_error = s->h->last_error;
        return rc;
    }
    SCK(s, cudaEventRecord(f1, s->s_cmp));
    SCK(s, cudaEventSynchronize(f1));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, f0, f1);
    s->stage2_ms = ms;
    return SPID_OK;
}

int spidgpu_stream_events(spidgpu_stream_handle s, spidgpu_task_event* out, int64_t cap, int64_t* count) {
    if (!s || !count || (cap > 0 && !out)) return SPID_INVALID_ARGUMENT;
    if (!s->finished || !s->f1) return sfail(s, SPID_INVALID_ARGUMENT, "the event log is complete after finish");
    cudaSetDevice(s->h->device);
    SCK(s, cudaEventSynchronize(s->f1));
    auto at = [&](cudaEvent_t e) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, s->t0, e);
        return 1e-3 * ms;
    };
    auto span = [&](cudaEvent_t a, cudaEvent_t b) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        return 1e-3 * ms;
    };
    const int64_t nblocks = static_cast<int64_t>(s->L.doms.size());
    std::vector<spidgpu_task_event> ev;
    for (const auto& p : s->pushes)
        for (int64_t j = 0; j < p.count; ++j)
            ev.push_back({SPIDGPU_EVENT_SNAPSHOT_INGESTED, -1, p.first + j, at(p.e), span(p.b, p.e)});
    for (size_t c = 0; c < s->closes.size(); ++c)
        for (int64_t b = 0; b < nblocks; ++b)
            ev.push_back({SPIDGPU_EVENT_CHUNK_CLOSED, b, static_cast<int64_t>(c), at(s->closes[c]), 0.0});
    for (size_t c = 0; c < s->s1_events.size(); ++c)
        for (int64_t b = 0; b < nblocks; ++b)
            ev.push_back({SPIDGPU_EVENT_STAGE1_DONE, b, static_cast<int64_t>(c), at(s->s1_events[c].second),
                          span(s->s1_events[c].first, s->s1_events[c].second)});
    for (int64_t b = 0; b < nblocks; ++b)
        ev.push_back({SPIDGPU_EVENT_STAGE2_DONE, b, -1, at(s->f1), span(s->f0, s->f1)});
    *count = static_cast<int64_t>(ev.size());
    for (int64_t i = 0; i < cap && i < *count; ++i) out[i] = ev[static_cast<size_t>(i)];
    return SPID_OK;
}

// Merged producer (ingestion) intervals, then the stage-1 time inside them,
// in the reference's order of operations (pipeline.cpp:296-332).
int spidgpu_overlap_report(const spidgpu_task_event* events, int64_t count, spidgpu_overlap* out) {
    if (!out || (count > 0 && !events)) return SPID_INVALID_ARGUMENT;
    if (count <= 0) return SPID_EMPTY_LOG;
    std::vector<std::pair<double, double>> producer, stage1, merged;
    for (int64_t i = 0; i < count; ++i) {
        const spidgpu_task_event& e = events[i];
        if (e.kind == SPIDGPU_EVENT_SNAPSHOT_INGESTED)
            producer.emplace_back(e.wall_time - e.duration, e.wall_time);
        else if (e.kind == SPIDGPU_EVENT_STAGE1_DONE)
            stage1.emplace_back(e.wall_time - e.duration, e.wall_time);
    }
    std::sort(producer.begin(), producer.end());
    for (const auto& iv : producer) {
        if (!merged.empty() && iv.first <= merged.back().second)
            merged.back().second = std::max(merged.back().second, iv.second);
        else
            merged.push_back(iv);
    }
    spidgpu_overlap r{0.0, 0.0, 0.0};
    for (const auto& iv : merged) r.producer_busy_seconds += iv.second - iv.first;
    double overlap = 0.0;
    for (const auto& iv : stage1) {
        r.stage1_busy_seconds += iv.second - iv.first;
        for (const auto& pv : merged) {
            const double lo = std::max(iv.first, pv.first), hi = std::min(iv.second, pv.second);
            if (hi > lo) overlap += hi - lo;
        }
    }
    r.overlap_fraction = r.stage1_busy_seconds > 0.0 ? overlap / r.stage1_busy_seconds : 0.0;
    *out = r;
    return SPID_OK;
}

int spidgpu_stream_get_stats(spidgpu_stream_handle s, spidgpu_stream_stats* out) {
    if (!s || !out) return SPID_INVALID_ARGUMENT;
    cudaSetDevice(s->h->device);
    std::memset(out, 0, sizeof(*out));
    out->snapshots = s->snapshots;
    out->stage1_tasks = s->stage1_tasks;
    out->stage2_tasks = s->stage2_tasks;
    out->fine_entries_peak = s->fine_peak;
    out->coarse_entries_peak = s->coarse_peak;
    double ms1 = 0.0;
    for (auto& e : s->s1_events) {
        if (cudaEventSynchronize(e.second) != cudaSuccess) break;
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, e.first, e.second) == cudaSuccess) ms1 += ms;
    }
    out->stage1_ms = ms1;
    out->stage2_ms = s->stage2_ms;
    return SPID_OK;
}

const char* spidgpu_stream_last_error(spidgpu_stream_handle s) { return s ? s->last_error.c_str() : ""; }

int spidgpu_stream_close(spidgpu_stream_handle s) {
    if (!s) return SPID_INVALID_ARGUMENT;
    cudaSetDevice(s->h->device);
    destroy(s);
    delete s;
    return SPID_OK;
}

}  // extern "C"
