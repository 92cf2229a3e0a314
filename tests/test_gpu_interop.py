"""The reference's own C++ callers on the GPU (include/spidgpu_spid.hpp).

oracle/_ref/interop_check (tests/interop_check.cpp, built by oracle/Makefile
against the reference's headers and library, which are not on the GPU box --
the binary travels prebuilt) runs each check twice, with namespace spid (the
reference, CPU) and namespace spid::gpu (the B200), on the reference's own
types, generators and downstream code: acceptance criteria 1 and 6, the CLI's
structured batch loop into an archive whose spid::encode bytes equal the
reference's (one handle, and two handles on worker threads), the two-stage
compressor, and batched Gaussian-sketch column IDs."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "interop_check")


def test_interop_header_compiles_against_reference():
    """CPU-side: the shim compiles against the reference headers (when they
    are present, i.e. in the build container)."""
    inc = "/root/reference/proj/include"
    if not os.path.isdir(inc):
        pytest.skip("reference headers not present")
    src = os.path.join(ROOT, "tests", "interop_check.cpp")
    r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-include", "cstdint", f"-I{inc}",
                        f"-I{ROOT}/include", src], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]


@pytest.mark.gpu
def test_reference_callers_on_gpu():
    if not os.path.exists(BIN):
        pytest.fail("oracle/_ref/interop_check was not built (make -C oracle interop)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    lines = r.stdout.strip().splitlines()
    fails = [ln for ln in lines if ln.startswith("FAIL")]
    assert r.returncode == 0 and not fails, "\n".join(fails) + r.stderr[-2000:]
    names = {ln.split()[1] for ln in lines if ln.startswith("PASS")}
    assert {"criterion1_structured", "criterion6_residual_identity", "cli_batch_loop_archive_bytes",
            "cli_batch_loop_two_handles_on_threads", "stage1_stage2",
            "column_id_batched_vs_reference_matmul"} <= names
