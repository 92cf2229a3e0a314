// interop_check.cpp -- the reference's own C++ callers, switched to the GPU.
//
// Compiled against the reference's headers (proj/include) and library
// (oracle/_ref/libspidref.so, built from the reference's sources), the
// oracle (test infrastructure: the CPU Omega) and libspidgpu.so by
// oracle/Makefile (target interop); run on a B200 by
// tests/test_gpu_interop.py. Every check computes the same thing twice --
// with namespace spid (the reference, CPU) and with namespace spid::gpu
// (include/spidgpu_spid.hpp, the B200) -- on the reference's own types and
// data generators, and feeds the GPU's factors to the reference's own
// downstream code (reconstruct, encode, quality_report, compression_factor):
//   1. analytic Taylor-Green reproduction, as acceptance criterion 1 states it
//      (rank 1, k(m+n) stored entries, CF exactly 80, error <= 1e-12,
//      proj/tests/acceptance.cpp:77-114), structured and unstructured;
//   2. the residual identity of acceptance criterion 6 (proj/tests/
//      acceptance.cpp:325-344) on SplitMix64 matrices;
//   3. the CLI's structured batch loop (proj/tools/spid_cli.cpp:195-232) into
//      an archive whose spid::encode bytes equal the CPU loop's, one handle
//      and two handles on worker threads (the multi-device pattern);
//   4. the two-stage compressor's stages (proj/src/blocking.cpp:107-196);
//   5. batched Gaussian-sketch column IDs (the north star) vs column_id of
//      the reference's matmul on the same Omega.
// Output: one "PASS name" / "FAIL name: why" line per check; exit 1 on any FAIL.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

#include "spid/archive.hpp"
#include "spid/datagen.hpp"
#include "spid/rng.hpp"
#include "spidgpu_spid.hpp"

extern "C" void orc_philox_omega(uint64_t seed, uint64_t s, size_t row0, size_t ell, size_t m, double* out);

namespace {

int failures = 0;

void check(const std::string& name, const std::function<void()>& body) {
    try {
        body();
        std::printf("PASS %s\n", name.c_str());
    } catch (const std::exception& e) {
        ++failures;
        std::printf("FAIL %s: %s\n", name.c_str(), e.what());
    }
    std::fflush(stdout);
}

void need(bool ok, const std::string& what) {
    if (!ok) throw std::runtime_error(what);
}

bool same(const spid::DenseMatrix& a, const spid::DenseMatrix& b) {
    return a.same_shape(b) && std::memcmp(a.data(), b.data(), sizeof(double) * a.entry_count()) == 0;
}

void same_factors(const spid::IdFactors& cpu, const spid::IdFactors& gpu, const std::string& what) {
    need(cpu.skeleton_indices == gpu.skeleton_indices, what + ": skeleton indices differ");
    need(cpu.achieved_rank == gpu.achieved_rank, what + ": rank differs");
    need(same(cpu.coeffs, gpu.coeffs), what + ": coefficients differ");
    need(same(cpu.skeleton, gpu.skeleton), what + ": skeleton differs");
    need(cpu.qr_residual_fro == gpu.qr_residual_fro, what + ": residual_fro differs");
}

spid::TaylorGreenParams tgv(spid::TaylorGreenQoi qoi) {
    spid::TaylorGreenParams p;
    p.grid = spid::GridGeom::structured({20, 20}, {true, true});
    p.qoi = qoi;
    return p;
}

}  // namespace

int main() {
    using spid::DenseMatrix;

    // 1. analytic Taylor-Green: rank 1, CF exactly 80, error <= 1e-12
    check("criterion1_structured", [] {
        for (auto qoi : {spid::TaylorGreenQoi::U1, spid::TaylorGreenQoi::U2, spid::TaylorGreenQoi::P}) {
            const DenseMatrix a = spid::taylor_green_matrix(tgv(qoi));
            const spid::IdFactors g = spid::gpu::column_id(a, spid::RankRule::fixed(1));
            same_factors(spid::column_id(a, spid::RankRule::fixed(1)), g, spid::qoi_name(qoi));
            const std::size_t stored = g.skeleton.entry_count() + g.coeffs.entry_count();
            need(g.achieved_rank == 1 && stored == 500, "rank 1 and k(m+n) = 500 stored entries");
            need(spid::compression_factor(400, 100, stored) == 80.0, "CF must be exactly 80");
            need(spid::rel_frob_error(a, spid::gpu::reconstruct(g)) <= 1e-12, "error above 1e-12");
            need(same(spid::gpu::reconstruct(g), spid::reconstruct(g)), "GPU reconstruct != reference matmul");
        }
    });
    check("criterion1_unstructured_sub_id", [] {
        spid::TaylorGreenParams p = tgv(spid::TaylorGreenQoi::U1);
        p.grid = spid::gen_unstructured_grid(400, 7, {{0.0, 2 * M_PI}, {0.0, 2 * M_PI}});
        const DenseMatrix a = spid::taylor_green_matrix(p);
        std::vector<std::size_t> rows;
        for (std::size_t r = 0; r < 400; r += 2) rows.push_back(r);
        const auto spec = spid::SubsampleSpec::explicit_list(p.grid, rows);
        const spid::IdFactors g = spid::gpu::sub_id(a, spec, spid::RankRule::fixed(1));
        same_factors(spid::sub_id(a, spec, spid::RankRule::fixed(1)), g, "sub_id");
        need(spid::compression_factor(400, 100, g.skeleton.entry_count() + g.coeffs.entry_count()) == 80.0, "CF");
        need(spid::rel_frob_error(a, spid::reconstruct(g)) <= 1e-12, "error above 1e-12");
    });

    // 2. residual identity: ||A - reconstruct||_F == qr_residual_fro (rel 1e-10)
    check("criterion6_residual_identity", [] {
        spid::SplitMix64 rng(777);
        for (int rep = 0; rep < 50; ++rep) {
            const std::size_t m = 8 + rng.next_u64() % 20, n = 6 + rng.next_u64() % 16;
            DenseMatrix a(m, n);
            for (std::size_t i = 0; i < a.entry_count(); ++i) a.data()[i] = rng.next_sym();
            for (std::size_t k : {std::size_t{1}, std::size_t{3}, std::min(m, n)}) {
                const spid::IdFactors g = spid::gpu::column_id(a, spid::RankRule::fixed(k));
                same_factors(spid::column_id(a, spid::RankRule::fixed(k)), g, "rep " + std::to_string(rep));
                const double err = spid::frobenius_norm(spid::subtract(a, spid::gpu::reconstruct(g)));
                const double res = g.qr_residual_fro;
                if (std::max(err, res) <= 1e-13 * spid::frobenius_norm(a)) continue;
                need(std::abs(err - res) / res <= 1e-10, "residual identity off");
            }
        }
    });

    // 3. the CLI batch loop -> archive bytes identical to the reference's
    spid::SmoothField3dParams fp;
    fp.grid = spid::GridGeom::structured({16, 12, 10}, {true, false, false});
    fp.steps = 40;
    DenseMatrix field = spid::smooth_field3d_matrix(fp);
    spid::SplitMix64 noise(5);
    for (std::size_t i = 0; i < field.entry_count(); ++i) field.data()[i] += 1e-3 * noise.next_sym();
    const std::vector<std::size_t> bpa{2, 2, 1}, strides{2, 2, 3};
    auto archive_of = [&](std::vector<spid::ArchiveBlock> blocks) {
        spid::Archive ar;
        ar.meta.grid = fp.grid;
        ar.meta.blocks_per_axis = bpa;
        ar.meta.strides = strides;
        ar.meta.mode = "batch";
        ar.meta.rank_rule_mode = "fixed";
        ar.meta.rank_k = 3;
        ar.meta.interp_recipe = "strided-multilinear";
        ar.meta.qoi = "u";
        ar.meta.m = field.rows();
        ar.meta.n = field.cols();
        ar.meta.provenance = "interop_check";
        ar.blocks = std::move(blocks);
        return ar;
    };
    const auto rule3 = spid::RankRule::fixed(3);
    std::vector<spid::ArchiveBlock> cpu_blocks;
    for (const auto& d : spid::make_block_domains(fp.grid, bpa)) {
        const DenseMatrix block = spid::select_rows(field, d.rows);
        const auto spec = spid::SubsampleSpec::strided(d.local, strides, true);
        cpu_blocks.push_back(spid::gpu::to_archive_block(spid::spid(block, spec, rule3), spec, d.rows.size()));
    }
    const spid::Archive cpu_ar = archive_of(cpu_blocks);
    const std::vector<std::uint8_t> cpu_bytes = spid::encode(cpu_ar);
    check("cli_batch_loop_archive_bytes", [&] {
        const spid::Archive gpu_ar = archive_of(spid::gpu::spid_blocks(field, fp.grid, bpa, strides, rule3));
        need(spid::encode(gpu_ar) == cpu_bytes, "encode() bytes differ from the reference loop's");
        const spid::QualityReport qc = spid::quality_report(field, cpu_ar), qg = spid::quality_report(field, gpu_ar);
        need(qc.cf == qg.cf && qc.rel_frob_error == qg.rel_frob_error && qc.block_ranks == qg.block_ranks,
             "quality_report differs");
        need(same(spid::decompress(gpu_ar), spid::decompress(cpu_ar)), "decompress differs");
    });
    check("cli_batch_loop_two_handles_on_threads", [&] {
        const spid::Archive gpu_ar =
            archive_of(spid::gpu::spid_blocks_multi(field, fp.grid, bpa, strides, rule3, {0, 0}));
        need(spid::encode(gpu_ar) == cpu_bytes, "multi-handle archive differs");
    });
    check("spid_lift_on_gpu", [&] {
        const auto d = spid::make_block_domains(fp.grid, bpa)[1];
        const DenseMatrix block = spid::select_rows(field, d.rows);
        const auto spec = spid::SubsampleSpec::strided(d.local, strides, true);
        const spid::SpidFactors g = spid::gpu::spid(block, spec, rule3);
        same_factors(spid::spid(block, spec, rule3).base, g.base, "spid");
        const DenseMatrix lifted_ref = g.interp.apply(g.base.skeleton);
        DenseMatrix lifted(lifted_ref.rows(), lifted_ref.cols());
        const spidgpu_grid_spec gs = spid::gpu::to_gpu(spec);
        spid::gpu::default_context().check(spidgpu_interp_apply(spid::gpu::default_context().get(), &gs,
                                                                g.base.skeleton.data(), g.base.skeleton.rows(),
                                                                g.base.skeleton.cols(), lifted.data()));
        double dl = 0.0;
        for (std::size_t i = 0; i < lifted.entry_count(); ++i)
            dl = std::max(dl, std::abs(lifted.data()[i] - lifted_ref.data()[i]));
        const DenseMatrix r_gpu = spid::gpu::reconstruct(g, spec), r_ref = spid::reconstruct(g);
        double dr = 0.0;
        for (std::size_t i = 0; i < r_ref.entry_count(); ++i)
            dr = std::max(dr, std::abs(r_gpu.data()[i] - r_ref.data()[i]));
        need(dl == 0.0, "GPU lift != InterpOperator::apply (max diff " + std::to_string(dl) + ")");
        need(same(r_gpu, r_ref), "GPU lift + product != reference (max diff " + std::to_string(dr) + ")");
    });

    // 4. the two-stage compressor: stage 1 per time chunk, stage 2 merge
    check("stage1_stage2", [&] {
        const auto spec = spid::SubsampleSpec::strided(fp.grid, {2, 2, 2}, true);
        std::vector<spid::IdFactors> s1c, s1g;
        for (std::size_t c0 = 0; c0 < field.cols(); c0 += 16) {
            const std::size_t w = std::min<std::size_t>(16, field.cols() - c0);
            DenseMatrix chunk(field.rows(), w);
            std::memcpy(chunk.data(), field.col(c0), sizeof(double) * field.rows() * w);
            s1c.push_back(spid::stage1_compress(chunk, spec, 4));
            s1g.push_back(spid::gpu::stage1_compress(chunk, spec, 4));
            same_factors(s1c.back(), s1g.back(), "stage1 chunk " + std::to_string(c0));
        }
        const spid::TwoStageFactors c = spid::stage2_compress(s1c, 1e-6);
        const spid::TwoStageFactors g = spid::gpu::stage2_compress(s1g, 1e-6);
        need(c.union_indices == g.union_indices, "union indices differ");
        need(c.final_skeleton_union_pos == g.final_skeleton_union_pos, "stage-2 selection differs");
        need(same(c.final_skeleton, g.final_skeleton) && same(c.stage2_coeffs, g.stage2_coeffs), "stage-2 factors");
        need(same(c.final_coeffs, g.final_coeffs), "composed coefficients C1 C0' differ");
    });

    // 5. batched Gaussian-sketch column IDs vs column_id(matmul(Omega, A))
    check("column_id_batched_vs_reference_matmul", [] {
        std::vector<DenseMatrix> blocks;
        for (int s = 0; s < 5; ++s) blocks.push_back(spid::gen_exact_rank(2048, 64, 8, 100 + s));
        const auto g = spid::gpu::column_id_batched(blocks, spid::RankRule::fixed(8), 24, 99, 10);
        for (int s = 0; s < 5; ++s) {
            // the exact Omega_s the kernel contracts (ell x m), from the
            // oracle's CPU restatement of its definition (oracle/workload.c)
            DenseMatrix O(24, 2048);
            orc_philox_omega(99, 10 + s, 0, 24, 2048, O.data());
            const spid::IdFactors c = spid::column_id(spid::matmul(O, blocks[s]), spid::RankRule::fixed(8));
            need(c.skeleton_indices == g[s].skeleton_indices, "pivots differ (block " + std::to_string(s) + ")");
            double worst = 0.0, cmax = 0.0;
            for (std::size_t i = 0; i < c.coeffs.entry_count(); ++i) {
                worst = std::max(worst, std::abs(c.coeffs.data()[i] - g[s].coeffs.data()[i]));
                cmax = std::max(cmax, std::abs(c.coeffs.data()[i]));
            }
            need(worst <= 1e-10 * cmax, "coefficients beyond 1e-10 relative");
            need(same(g[s].skeleton, spid::select_columns(blocks[s], g[s].skeleton_indices)), "skeleton gather");
            need(spid::rel_frob_error(blocks[s], spid::reconstruct(g[s])) <= 1e-10, "rank-8 data not reproduced");
        }
    });

    std::printf("%s (%d failure%s)\n", failures ? "FAILED" : "OK", failures, failures == 1 ? "" : "s");
    return failures ? 1 : 0;
}
