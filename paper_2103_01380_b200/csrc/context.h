// context.h -- internal state of a spidgpu handle and the launch sequences
// shared by the ABI translation units (api.cu, archive_api.cu). Not part of
// the public interface (include/spidgpu.h).
#pragma once

#include <nvtx3/nvToolsExt.h>

#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/spidgpu.h"
#include "kernels.h"

namespace spidgpu {

// ---- device buffers --------------------------------------------------------
struct DevBuf {
    void* ptr = nullptr;
    size_t bytes = 0;
    cudaError_t ensure(size_t need, cudaStream_t stream) {
        if (need <= bytes) return cudaSuccess;
        if (ptr) {
            cudaError_t e = cudaStreamSynchronize(stream);
            if (e != cudaSuccess) return e;
            cudaFree(ptr);
            ptr = nullptr;
            bytes = 0;
        }
        size_t want = std::max(need, bytes * 3 / 2);
        cudaError_t e = cudaMalloc(&ptr, want);
        if (e != cudaSuccess) {
            ptr = nullptr;
            return e;
        }
        bytes = want;
        return cudaSuccess;
    }
    template <class T>
    T* as() const {
        return static_cast<T*>(ptr);
    }
    void release() {
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        bytes = 0;
    }
};

// One workspace set per concurrently used stream.
struct Workspace {
    DevBuf partial, rws, wws, r11ws, ybuf, vpart, flag;
    // host-API / compress_host staging
    DevBuf a, omega, idx, coeffs, skel, rank, resid, status, err2, ref2, rows, out, pivots, r, q;
    // archive codec: gathered coarse rows, block tables, the archive image
    DevBuf bsk, rel, bases, uni, blocks, bytes, crc;
    void release() {
        for (DevBuf* b : {&partial, &rws, &wws, &r11ws, &ybuf, &vpart, &flag, &a, &omega, &idx,
                          &coeffs, &skel, &rank, &resid, &status, &err2, &ref2, &rows, &out,
                          &pivots, &r, &q, &bsk, &rel, &bases, &uni, &blocks, &bytes, &crc})
            b->release();
    }
};

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

}  // namespace spidgpu

struct spidgpu_context {
    int device = 0;
    int num_sms = 148;
    spidgpu::Workspace ws[3];
    cudaStream_t lanes[2] = {nullptr, nullptr};
    cudaEvent_t ev[2] = {nullptr, nullptr};
    spidgpu::EncodeTiledFn encode = nullptr;
    int64_t launches = 0;
    std::string last_error;
    bool force_generic_cpqr = false;  // tests: exercise the shared/global-W kernel too
    bool force_dmma_sketch = false;   // Philox sketches on the FP64 DMMA kernel
    int sketch_sms = 0;               // SMs the persistent sketch grid may occupy (0 = all)
    int sketch_pairs = 1;             // tcgen05 sketch CTA pairs: 0/1 off (ell <= 64), 2 always, 3 split (80)
    bool tall_pairs = true;           // tall column IDs with 64 < n <= 256 over a cluster of two
    bool reg_pairs = true;            // sketch-sized column IDs with 128 < n <= 256 over a cluster of two
    int64_t sketch_seg_rows = 0;      // tcgen05 sketch segment rows (0 = kSketchSegRows; experiments)
    uint8_t* archive_pinned = nullptr;  // last archive built by spidgpu_archive_compress
    size_t archive_cap = 0, archive_size = 0;
    // pinned staging slots for pageable host uploads (upload_host_bytes)
    uint8_t* upload_pinned = nullptr;
    size_t upload_cap = 0;
    cudaEvent_t upload_ev[16] = {};
    // deferred status of asynchronous batched calls (first error wins; read
    // and cleared by spidgpu_stream_status): out-of-range gather indices
    int32_t* dev_status = nullptr;
};

namespace spidgpu {

// NVTX phase ranges (header-only NVTX3: free unless a tool -- nsys, ncu
// --nvtx -- injects a handler): every C-ABI phase of the compress path shows
// up by name on a timeline, e.g. "spidgpu.sketch", "spidgpu.cpqr".
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

int fail(spidgpu_handle h, int code, const std::string& msg);
int cuda_fail(spidgpu_handle h, cudaError_t e, const char* where);

#define CK(h, expr)                                              \
    do {                                                         \
        cudaError_t _e = (expr);                                 \
        if (_e != cudaSuccess) return cuda_fail((h), _e, #expr); \
    } while (0)

struct RuleInfo {
    int status = SPID_OK;       // immediate (BadRankRule, InvalidArgument)
    int pre_status = SPID_OK;   // batch-uniform kernel-reported (RankUnreachable)
    int64_t step_limit = 0;
};
RuleInfo resolve_rule(const spidgpu_rank_rule* rule, int64_t rows, int64_t n, int64_t kcap);

int do_sketch(spidgpu_handle h, Workspace& ws, const double* A, int64_t m, int64_t n, int64_t lda,
              int64_t strideA, int64_t batch, int64_t ell, const spidgpu_omega* om, double* Y,
              int64_t ldy, int64_t strideY, cudaStream_t st);
int do_cpqr(spidgpu_handle h, Workspace& ws, const double* Y, int64_t rows, int64_t n, int64_t ldy,
            int64_t strideY, int64_t batch, const spidgpu_rank_rule* rule, int64_t kcap,
            int64_t* indices, double* C, int64_t strideC, int64_t* rank, double* resid,
            int32_t* status, int64_t* pivots, double* R, double* Q, cudaStream_t st);
int do_gather(spidgpu_handle h, const double* A, int64_t m, int64_t n, int64_t lda, int64_t strideA,
              int64_t batch, const int64_t* indices, int64_t kcap, const int64_t* rank,
              double* skel, int64_t ldskel, int64_t strideS, cudaStream_t st);

template <class T>
int to_dev(spidgpu_handle h, DevBuf& buf, const T* src, size_t count, cudaStream_t st) {
    CK(h, buf.ensure(sizeof(T) * std::max<size_t>(count, 1), st));
    if (count) CK(h, cudaMemcpyAsync(buf.ptr, src, sizeof(T) * count, cudaMemcpyHostToDevice, st));
    return SPID_OK;
}

// Structured grid + strided subsample validation (grid.cpp:7-33, 62-75);
// min_dim = 2 for GridGeom::structured, 1 for structured_block.
int spec_to_dev(spidgpu_handle h, const spidgpu_grid_spec* sp, GridSpecDev* g, int64_t* P,
                int64_t* Pc, int min_dim = 2, bool lift = true);
std::vector<int64_t> spec_rows(const GridSpecDev& g, int64_t P);

}  // namespace spidgpu
