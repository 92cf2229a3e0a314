// kernels.h -- launch interfaces of the spidgpu kernels (host side).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include <vector>

namespace spidgpu {

enum RuleMode { RULE_FIXED = 0, RULE_TOL = 1, RULE_BLOCKED = 2 };

// ---- CPQR / column ID (cpqr.cu) ------------------------------------------
struct CpqrParams {
    const double* Y;
    int64_t rows, n, ldy, strideY, batch;
    int mode, strict;
    int64_t kstep;
    double tol;
    int64_t step_limit;  // steps the loop may take (k, min(rows,n), ...)
    int64_t step_cap;    // rows of the R workspace
    int64_t kcap;
    int pre_status;      // batch-uniform failure decided on the host
    int npad;
    double* w_ws;        // rows*npad per subdomain when W does not fit smem
    double* r_ws;        // step_cap*n per subdomain
    double* r11_ws;      // step_cap^2 per subdomain when R11 does not fit smem
    int64_t* indices;
    double* C;
    int64_t strideC;
    int64_t* rank;
    double* resid;
    int32_t* status;
    int64_t* pivots;
    double* Rout;
    double* Qout;
};
size_t cpqr_smem_bytes(int64_t rows, int64_t n, int64_t step_cap, bool w_in_shared);
size_t cpqr_max_dyn_smem();
cudaError_t launch_cpqr(const CpqrParams& p, bool w_in_shared, cudaStream_t stream);
// tall inputs (rows >= 256, n <= 256): W in global memory, streamed through a
// TMA ring; wmap = 3D map {npad, rows, batch} of w_ws, box {npad, ring_rows, 1}
bool cpqr_tall_supported(int64_t rows, int64_t n);
int cpqr_tall_npad(int64_t n);
int cpqr_tall_ring_rows(int64_t n);
cudaError_t launch_cpqr_tall(const CpqrParams& p, const CUtensorMap* wmap, cudaStream_t stream);
// tall inputs with 64 < n <= 256 and the fixed / tolerance rules: each
// subdomain's columns split over a cluster of two CTAs (cpqr_pair.cu); W rows
// are 2 * cpqr_pair_half(n) long, the TMA box is {half, ring_rows, 1} (pmap: the
// same map with box {2, ring_rows, 1}, the pivot column pair) and the
// r11 workspace holds two step_cap^2 blocks per subdomain
size_t cpqr_pair_smem_bytes(int64_t rows, int64_t n, int64_t step_cap);
bool cpqr_pair_supported(int64_t rows, int64_t n, int mode, int64_t step_cap);
int cpqr_pair_half(int64_t n);
int cpqr_pair_ring_rows(int64_t n);
cudaError_t launch_cpqr_pair(const CpqrParams& p, const CUtensorMap* wmap, const CUtensorMap* pmap,
                             cudaStream_t stream);
// the register-resident column ID with each subdomain's columns split over a
// cluster of two CTAs (cpqr_reg_pair.cu): 32 < rows <= 48, 128 < n <= 256,
// fixed / tolerance rules; R in r_ws as for cpqr_reg
bool cpqr_regpair_supported(int64_t rows, int64_t n, int mode, int64_t step_cap);
cudaError_t launch_cpqr_regpair(const CpqrParams& p, cudaStream_t stream);
// register-resident variant for sketch-sized inputs (rows <= 80, n <= 512)
bool cpqr_reg_supported(int64_t rows, int64_t n, int64_t step_cap);
cudaError_t launch_cpqr_reg(const CpqrParams& p, cudaStream_t stream);

// ---- sketch Y = Omega * A (sketch.cu) -------------------------------------
// Work decomposition shared by both sketch kernels. A subdomain's column tile
// is cut into SEGMENTS of kSketchSegRows rows at fixed absolute row offsets
// (they depend on m only). A work unit is one (subdomain, column tile,
// segment); each persistent CTA (or CTA pair) takes a contiguous range of
// whole units, accumulates every segment on its own and writes it to the
// segment's own partial slot; the reduction sums a tile's slots in segment
// order. So Y_s is bitwise the same whatever the batch, the grouping, the
// grid size (SM cap) or the GPU count -- the reference's "bitwise identical
// regardless of scheduling" contract (
// proj/tests/test_pipeline.cpp:104-125).
constexpr int64_t kSketchSegRows = 4096;
struct SketchPlan {
    int ell_pad;     // Omega rows computed (8..80)
    int mt;          // M tiles of 8 rows (ell_pad = 8*mt)
    int nw;          // N tiles of 8 columns per warp
    int nt;          // columns per CTA tile
    int64_t ntiles_col;   // column tiles per subdomain
    int64_t nchunk;       // row chunks (stages) per subdomain
    int kc_rows;          // rows per chunk (16 DMMA, 32 integer-sliced)
    int64_t seg_len;      // chunks per segment (kSketchSegRows / kc_rows)
    int64_t nseg;         // segments per column tile
    int64_t total_units;  // batch * (ntiles_col / (1 + pair)) * nseg
    int grid;             // CTAs (persistent, contiguous ranges of whole units)
    int halves = 1;       // partial tiles per slot (2: slice halves of a split CTA pair)
    int pair = 0;         // sketch_tc.cu cluster mode: 0 none, 1 column-tile pairs, 2 slice-split pairs
    size_t smem;
    size_t partial_elems; // doubles of the partial workspace: batch*ntiles_col*nseg*halves*ell_pad*nt
};
// first chunk (in the flat (subdomain, column tile, chunk) order) of unit u
__host__ __device__ inline int64_t sketch_unit_chunk(int64_t u, int64_t nseg, int64_t seg_len, int64_t nchunk) {
    return (u / nseg) * nchunk + (u % nseg) * seg_len;
}
struct SketchParams {
    const double* A;
    int64_t m, n, lda, strideA, batch;
    int64_t ell;          // rows produced by this launch (<= 8*mt)
    int64_t row0;         // first Omega row of this launch (ell > 80 is sliced)
    int omega_mode;       // 0 explicit, 1 philox
    const double* omega;  // explicit: Omega_s(r, k) at omega + s*stride + k*ldo + r
    int64_t ldo, stride_o;
    uint64_t seed;
    int64_t sub_base;
    double* partial;      // [subdomain][column tile][segment][half][ell_pad][nt]
    double* Y;            // final: Y_s(r, j) at Y + s*strideY + j*ldy + (row0 + r)
    int64_t ldy, strideY;
};
bool sketch_make_plan(int64_t m, int64_t n, int64_t batch, int64_t ell, int num_sms,
                      SketchPlan* plan);
cudaError_t launch_sketch(const SketchParams& p, const SketchPlan& plan, const CUtensorMap* tmap,
                          cudaStream_t stream);
// fixed-order reduction of the segment partials into Y (both sketch kernels)
cudaError_t launch_sketch_reduce(const SketchParams& p, const SketchPlan& plan, cudaStream_t stream);
// the exact integer-sliced sketch on tcgen05.mma kind::i8 with TMEM accumulators (sketch_tc.cu)
constexpr int64_t kSketchTcMaxEll = 80;
// seg_rows: rows per segment (0 = kSketchSegRows; a multiple of 512, <= 65536)
bool sketch_tc_make_plan(int64_t m, int64_t n, int64_t batch, int64_t ell, int num_sms, int pair_mode,
                         int64_t seg_rows, SketchPlan* plan);
int sketch_tc_flush_counters(int64_t* out, bool reset);
cudaError_t launch_sketch_tc(const SketchParams& p, const SketchPlan& plan, const CUtensorMap* tmap,
                             cudaStream_t stream);
cudaError_t launch_philox_omega(uint64_t seed, int64_t s, int64_t ell, int64_t m, double* out,
                                int64_t ldo, cudaStream_t stream);

// ---- gathers (gather.cu) --------------------------------------------------
cudaError_t launch_gather_cols(const double* A, int64_t m, int64_t lda, int64_t strideA,
                               int64_t batch, const int64_t* indices, int64_t kcap,
                               const int64_t* rank, int64_t n, double* skel, int64_t ldskel,
                               int64_t strideS, int32_t* err_flag, cudaStream_t stream);
cudaError_t launch_gather_rows(const double* A, int64_t m, int64_t n, int64_t lda,
                               int64_t strideA, int64_t batch, const int64_t* rows,
                               int64_t nrows, double* B, int64_t ldb, int64_t strideB, int32_t* err_flag,
                               cudaStream_t stream);

// ---- verify / reconstruct (verify.cu) ------------------------------------
struct VerifyParams {
    const double* A;
    int64_t m, n, lda, strideA, batch;
    const double* skel;
    int64_t ldskel, strideS;
    const double* C;
    int64_t kcap, strideC;
    const int64_t* rank;
    double* part;      // [batch][nblk][2] partial sums
    int64_t nblk;      // row blocks per subdomain
    double* err2;
    double* ref2;
};
int64_t verify_row_blocks(int64_t m);
struct VerifyPlan {  // same segment units as the sketch (SketchPlan)
    int nwv, ks, nt;
    int64_t ntiles_col, nchunk, seg_len, nseg, total_units;
    int grid;
    size_t part_elems;
};
bool verify_make_plan(int64_t m, int64_t n, int64_t batch, int64_t kcap, int num_sms,
                      VerifyPlan* plan);
cudaError_t launch_verify_tma(const VerifyParams& p, const VerifyPlan& plan, const CUtensorMap* tA,
                              const CUtensorMap* tS, double* part, cudaStream_t stream);
cudaError_t launch_verify(const VerifyParams& p, int num_sms, cudaStream_t stream);
cudaError_t launch_reconstruct(const double* skel, int64_t m, int64_t ldskel, int64_t strideS,
                               const double* C, int64_t kcap, int64_t strideC,
                               const int64_t* rank, int64_t n, int64_t batch, double* out,
                               int64_t ldo, int64_t strideO, cudaStream_t stream);
cudaError_t launch_sqdiff(const double* a, const double* b, int64_t count, double* part,
                          int64_t nparts, cudaStream_t stream);

// ---- SPID coarse skeleton + multilinear lift (interp.cu) -------------------
struct GridSpecDev {
    int naxes;
    int dims[3];
    int strides[3];
    bool periodic[3];
    bool incl;  // SubsampleSpec::include_boundary
    int nqoi;   // QoI blocks stacked along the rows
};
cudaError_t launch_interp_apply(const GridSpecDev& g, const double* coarse, int64_t ldc,
                                int64_t strideC, int64_t k, const int64_t* rank, int64_t batch,
                                double* fine, int64_t ldf, int64_t strideF, int32_t* err_flag,
                                cudaStream_t stream);
cudaError_t launch_gather_coarse(const double* A, int64_t lda, int64_t strideA, const int64_t* rows,
                                 int64_t nrows, const int64_t* idx, int64_t kcap,
                                 const int64_t* rank, int64_t batch, double* skel, int64_t ldskel,
                                 int64_t strideS, cudaStream_t stream);

// ---- CRC-32 (crc.cu) -------------------------------------------------------
cudaError_t launch_crc32(const uint8_t* data, int64_t nbytes, uint32_t* block_scratch,
                         uint32_t* out, cudaStream_t stream);
int64_t crc32_scratch_words(int64_t nbytes);

// ---- archive codec (archive.cu) --------------------------------------------
struct PackBlock {          // one block section of the archive
    int64_t sec_off;        // archive offset of the section's u64 length field
    int64_t k, mc, n;       // rank, skeleton rows, snapshot columns
    int64_t nu;             // union index count (== k for batch archives)
    int32_t coarse;
    const int64_t* uni;     // union_indices (sorted)
    const int64_t* sel;     // skeleton indices in selection order
    const double* skel;     // mc x k, ld ld_s
    int64_t ld_s;
    const double* coeffs;   // k x n, ld ld_c
    int64_t ld_c;
};
struct CrcSection {
    int64_t begin, len;     // payload byte range; the CRC follows it
};
constexpr int64_t kCrcPart = 65536;  // bytes per CTA work unit of the section CRC
struct CrcPart {
    int64_t begin, end;     // <= kCrcPart bytes, end-aligned inside a section
};
struct UnpackBlock {
    int64_t skel_off, coef_off;  // archive offsets of the first f64 of each matrix
    int64_t mc, k, n;
    double* skel;                // destination mc x k, ld ld_s
    int64_t ld_s;
    double* coeffs;              // destination k x n, ld ld_c
    int64_t ld_c;
};
struct BlockGridDev {       // make_block_domains segments per axis
    int naxes;
    int64_t dims[3], seg_base[3], seg_count[3];
};
cudaError_t launch_gather_block_rows(const double* A, int64_t lda, const int64_t* rel,
                                     int64_t nrows, const int64_t* bases, int64_t nb, int64_t n,
                                     double* B, int64_t ldb, int64_t strideB, cudaStream_t st);
cudaError_t launch_sort_union(const int64_t* idx, int64_t kcap, const int64_t* rank, int64_t nb,
                              int64_t* uni, cudaStream_t st);
cudaError_t launch_pack_blocks(const PackBlock* blocks, int64_t nblocks, int64_t max_items,
                               uint8_t* out, cudaStream_t st);
// host: split sections into parts (first_part has nsec + 1 entries)
void crc_plan_parts(const CrcSection* secs, int64_t nsec, std::vector<CrcPart>* parts,
                    std::vector<int64_t>* first_part);
cudaError_t launch_crc_sections(const uint8_t* data, const CrcSection* secs, int64_t nsec,
                                const CrcPart* parts, int64_t nparts, const int64_t* first_part,
                                uint32_t* part_crc, uint32_t* crc_out, uint8_t* write_back,
                                cudaStream_t st);
cudaError_t launch_unpack_blocks(const uint8_t* bytes, const UnpackBlock* blocks, int64_t nblocks,
                                 int64_t max_items, cudaStream_t st);
cudaError_t launch_recon_scatter(const double* F, int64_t ldf, int64_t strideF, const double* C,
                                 int64_t kcap, int64_t strideC, const int64_t* rank, int64_t nb,
                                 int64_t mb, int64_t n, const int64_t* rel, const int64_t* bases,
                                 double* out, int64_t ldo, cudaStream_t st);
cudaError_t launch_nonfinite_blocks(const double* A, int64_t lda, int64_t m, int64_t n,
                                    const BlockGridDev& g, int32_t* flags, cudaStream_t st);

// ---- streaming two-stage compressor (stream.cu) -----------------------------
struct StreamChunkDev {        // one closed chunk of one geometry group
    const double* skel;        // nb x kcap x mc: skeleton columns in sorted order
    const int64_t* sorted_idx; // nb x kcap: chunk-local skeleton indices, ascending
    const int32_t* sorted_pos; // nb x kcap: their stage-1 selection positions
    const int64_t* rank;       // nb
    const double* C0;          // nb x kcap x cols (ld kcap): stage-1 coefficients
    int64_t kcap, cols, col0;
};
cudaError_t launch_sort_pairs(const int64_t* idx, const int64_t* rank, int64_t kcap, int64_t nb,
                              int64_t* out_idx, int32_t* out_pos, cudaStream_t st);
cudaError_t launch_concat_union(const StreamChunkDev* chunks, int64_t nchunks, int64_t nb, int64_t mc,
                                int64_t rmax, double* concat, int64_t* uglob, int32_t* upos,
                                int64_t* uoff, int64_t* R, cudaStream_t st);
cudaError_t launch_compose(const StreamChunkDev* chunks, int64_t nchunks, int64_t time_chunk,
                           int64_t n_total, const double* C1, int64_t kcap2, int64_t rmax,
                           const int64_t* rank2, const int32_t* upos, const int64_t* uoff, int64_t nb,
                           double* out, int32_t* bad, cudaStream_t st);
cudaError_t launch_final_global(const int64_t* idx2, const int64_t* rank2, int64_t kcap2,
                                const int64_t* uglob, int64_t rmax, int64_t nb, int64_t* out,
                                cudaStream_t st);

// ---- synthetic fields (fields.cu) ----------------------------------------
struct FieldParams {
    int kind;
    int64_t grid, block, snapshots;
    double t_end, nu, sigma;
    uint64_t seed;
    int64_t first, batch;
    double* A;
    int64_t lda, strideA;
    // modes: per mode (kx, ky, kz, amp, phase, ax, ay, az) in device memory
    const double* modes;
    int n_modes;
    const double* heavy_modes;
    int n_heavy;
    const uint8_t* is_heavy;  // device, batch entries (may be null)
};
cudaError_t launch_field(const FieldParams& p, cudaStream_t stream);

}  // namespace spidgpu
