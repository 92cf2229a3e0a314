// shim_check.cpp -- the C++ host shim compiled against libspidgpu.so.
// With a GPU: runs the reference's TGV rank-1 KAT (acceptance.cpp:77-114)
// through spidgpu::column_id / reconstruct / rel_frob_error.
// Without one (--no-device-ok): checks that creation fails with NoDevice.
#include <cmath>
#include <cstdio>
#include <cstring>

#include "spidgpu.hpp"

int main(int argc, char** argv) {
    const bool no_device_ok = argc > 1 && std::strcmp(argv[1], "--no-device-ok") == 0;
    if (spidgpu::compression_factor(400, 100, 500) != 80.0) return 1;
    try {
        spidgpu::RankRule::tolerance(1.5);
        return 2;
    } catch (const spidgpu::Error& e) {
        if (e.name() != "BadRankRule") return 3;
    }
    spidgpu_handle h = nullptr;
    const int rc = spidgpu_create(0, &h);
    if (rc) {
        std::printf("no device: %s\n", spidgpu_status_name(rc));
        return (no_device_ok && rc == SPID_NO_DEVICE) ? 0 : 4;
    }
    spidgpu_destroy(h);
    // 2D Taylor-Green u1 on 20x20, 100 snapshots (proj/src/datagen.cpp:47-69)
    spidgpu::Matrix a(400, 100);
    for (std::size_t j = 0; j < 100; ++j)
        for (std::size_t i = 0; i < 400; ++i) {
            const double x = 2 * M_PI * (i % 20) / 20.0, y = 2 * M_PI * (i / 20) / 20.0;
            a(i, j) = std::sin(x) * std::cos(y) * std::exp(-2 * 0.1 * 0.1 * j);
        }
    const auto f = spidgpu::column_id(a, spidgpu::RankRule::fixed(1));
    const std::size_t stored = f.skeleton.entry_count() + f.coeffs.entry_count();
    const double cf = spidgpu::compression_factor(400, 100, stored);
    const double err = spidgpu::rel_frob_error(a, spidgpu::reconstruct(f));
    std::printf("rank %zu cf %.1f err %.3e\n", f.achieved_rank, cf, err);
    return (f.achieved_rank == 1 && cf == 80.0 && err <= 1e-12) ? 0 : 5;
}
