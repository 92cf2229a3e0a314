"""CPU: the C-ABI library is built for sm_100a, loads, and exports every symbol
the headers declare; error-name mapping and argument validation work without
a GPU (no compute call is made here)."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    from paper_2103_01380_b200 import _native as N

    declared = N.header_symbols()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(N.lib, name), name
    # and the Python binding declares a signature for each of them
    assert set(declared) <= set(N._SIGS)


def test_status_names_match_reference_errors():
    from paper_2103_01380_b200 import _native as N

    hdr = open(os.path.join(ROOT, "include", "spidgpu_status.h")).read()
    pairs = re.findall(r"SPID_\w+ = (\d+),?\s*/\* \"(\w+)\"", hdr)
    assert len(pairs) >= 19
    for code, name in pairs:
        assert N.status_name(int(code)) == name
    assert N.status_name(0) == "Ok"


def test_abi_version_and_pure_functions():
    from paper_2103_01380_b200 import _native as N
    from paper_2103_01380_b200 import spid

    assert N.lib.spidgpu_abi_version() == 1
    assert spid.compression_factor(400, 100, 500) == 80.0
    with pytest.raises(N.SpidError) as e:
        spid.compression_factor(4, 4, 0)
    assert e.value.name == "ZeroDenominator"


def test_no_device_fails_loudly():
    """Without a GPU the product refuses to run (no CPU fallback)."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2103_01380_b200 import _native as N
    from paper_2103_01380_b200 import spid

    with pytest.raises(N.SpidError) as e:
        N.Handle(0)
    assert e.value.name == "NoDevice"
    with pytest.raises(N.SpidError):
        spid.column_id([[1.0, 2.0], [3.0, 4.0]], rank=1)


def test_null_handle_rejected():
    from paper_2103_01380_b200 import _native as N

    assert N.lib.spidgpu_destroy(None) == 101
    assert N.lib.spidgpu_launch_count(None) == 0
    assert N.lib.spidgpu_last_error(None) == b""


@pytest.mark.parametrize("obj,mnemonics", [
    # the shipped Philox sketch: tcgen05 integer MMAs, TMEM loads/stores, TMA,
    # multicast MMA commits (CTA pairs) and st.async (DSMEM) of the split pair
    ("sketch_tc.o", ["UTCIMMA", "LDTM", "STTM", "UTMALDG", "UTCBAR.MULTICAST", "STAS"]),
    # the explicit-Omega (oracle-mode) sketch and the verify kernel: FP64 tensor cores + TMA
    ("sketch.o", ["DMMA.8x8x4", "UTMALDG"]),
    ("verify_tma.o", ["DMMA.8x8x4", "UTMALDG"]),
])
def test_sass_is_sm100a_with_tensor_cores_and_tma(obj, mnemonics):
    """The kernel objects hold sm_100a SASS with the instructions their design
    relies on -- checked with cuobjdump, no GPU needed."""
    path = os.path.join(ROOT, "paper_2103_01380_b200", "lib", "obj", obj)
    if not os.path.exists(path):
        pytest.skip("objects not built")
    out = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    for mn in mnemonics:
        assert mn in out, mn


def test_rank_rule_validation():
    from paper_2103_01380_b200 import spid

    for bad in (lambda: spid.RankRule.fixed(0), lambda: spid.RankRule.tolerance(0.0),
                lambda: spid.RankRule.tolerance(1.0), lambda: spid.RankRule.blocked(64, 0, 1e-3)):
        with pytest.raises(spid.SpidError) as e:
            bad()
        assert e.value.name == "BadRankRule"


def test_cpp_shim_compiles():
    """include/spidgpu.hpp (the C++ host shim mirroring namespace spid) compiles
    and links against the C ABI."""
    shim = os.path.join(ROOT, "include", "spidgpu.hpp")
    if not os.path.exists(shim):
        pytest.skip("no C++ shim")
    src = os.path.join(ROOT, "tools", "shim_check.cpp")
    out = "/tmp/spidgpu_shim_check"
    lib = os.path.join(ROOT, "paper_2103_01380_b200", "lib")
    r = subprocess.run(["g++", "-std=c++17", "-O1", f"-I{ROOT}/include", src, "-o", out,
                        f"-L{lib}", "-lspidgpu", f"-Wl,-rpath,{lib}"], capture_output=True,
                       text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([out, "--no-device-ok"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_cpp_shim_runs_on_device():
    """The same shim program with a device: the reference's TGV rank-1 known
    answer (proj/tests/acceptance.cpp:77-114) through spidgpu::column_id,
    reconstruct and rel_frob_error on the B200."""
    src = os.path.join(ROOT, "tools", "shim_check.cpp")
    out = "/tmp/spidgpu_shim_check_dev"
    lib = os.path.join(ROOT, "paper_2103_01380_b200", "lib")
    r = subprocess.run(["g++", "-std=c++17", "-O1", f"-I{ROOT}/include", src, "-o", out,
                        f"-L{lib}", "-lspidgpu", f"-Wl,-rpath,{lib}"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([out], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
