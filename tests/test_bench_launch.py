"""bench.py's launch contract: `python bench.py --gpus N` starts N ranks
itself (torchrun, 127.0.0.1), a rank count that differs from --gpus is
rejected, and the reference arm runs the reference's CPU code with inputs
built on the CPU -- its process loads no product library."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BENCH = os.path.join(ROOT, "bench.py")


def _run(args, env=None, timeout=600):
    e = dict(os.environ)
    e.pop("WORLD_SIZE", None)
    e.update(env or {})
    r = subprocess.run([sys.executable, BENCH] + args, capture_output=True, text=True, env=e, timeout=timeout,
                       cwd=ROOT)
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    return r, [json.loads(ln) for ln in lines]


def test_reference_arm_two_ranks_cpu_only():
    r, out = _run(["--impl", "reference", "--gpus", "2", "--config", "cfg1", "--steps", "1", "--warmup", "0"])
    assert r.returncode == 0, r.stderr[-2000:]
    assert len(out) == 1  # rank 0 alone prints
    line = out[0]
    assert line["impl"] == "reference" and line["n_gpus"] == 2
    assert line["reference_class"] == "cpu" and line["cpu_baseline"]["ranks_ok"]
    assert line["cpu_baseline"]["t1"]["cores"] == 1 and line["cpu_baseline"]["cpu_model"]
    assert not any("libspidgpu" in lib for lib in line["libraries_loaded"]), line["libraries_loaded"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0


def test_world_size_mismatch_is_rejected():
    r, out = _run(["--impl", "reference", "--gpus", "1"], env={"WORLD_SIZE": "2"}, timeout=60)
    assert r.returncode == 2 and not out
    assert "WORLD_SIZE=2" in r.stderr


@pytest.mark.gpu
def test_two_ranks_same_report_as_one():
    """BENCH_BACKEND=gloo: two ranks on the one GPU this pool exposes split
    config 1's 8 subdomains; the reduced CF and error equal one rank's (the
    4-double report). Functional check only: no numbers."""
    base = ["--config", "cfg1", "--steps", "2", "--warmup", "3", "--no-e2e", "--no-quality", "--no-archive",
            "--no-cpu-baseline"]
    r1, o1 = _run(["--gpus", "1"] + base)
    assert r1.returncode == 0, r1.stderr[-2000:]
    r2, o2 = _run(["--gpus", "2"] + base, env={"BENCH_BACKEND": "gloo"})
    assert r2.returncode == 0, r2.stderr[-2000:]
    a, b = o1[0], o2[0]
    assert a["n_gpus"] == 1 and b["n_gpus"] == 2
    assert a["config"]["subdomains"] == b["config"]["subdomains"] == 8
    assert a["cf"] == b["cf"] and a["stored_entries"] == b["stored_entries"]
    assert abs(a["rel_frob_error"] - b["rel_frob_error"]) <= 1e-12 * a["rel_frob_error"]
