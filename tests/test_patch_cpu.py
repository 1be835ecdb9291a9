"""The reference-side integration patch (oracle/reference_gpu.patch) applies cleanly
to the reference sources, and the patched library built from it (oracle/Makefile target `patched`)
exists with the GPU hook compiled in. CPU-only: running it needs the GPU (tests/test_dropin_gpu.py)."""
import shutil
import subprocess
import tempfile
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF = Path("/root/reference/proj")


@pytest.mark.skipif(not REF.exists(), reason="reference sources not mounted")
def test_patch_applies_to_reference():
    with tempfile.TemporaryDirectory() as d:
        for sub in ("include", "src"):
            shutil.copytree(REF / sub, Path(d) / sub)
        res = subprocess.run(["patch", "-p1", "--dry-run", "-i", str(ROOT / "oracle" / "reference_gpu.patch")],
                             cwd=d, capture_output=True, text=True)
        assert res.returncode == 0, res.stdout + res.stderr
        assert "FAILED" not in res.stdout and "offset" not in res.stdout


def test_patch_touches_only_the_runtime_seam():
    text = (ROOT / "oracle" / "reference_gpu.patch").read_text()
    files = sorted(l.split()[1] for l in text.splitlines() if l.startswith("+++ "))
    assert files == ["b/include/iolm/runtime.hpp", "b/src/CMakeLists.txt", "b/src/calib.cpp", "b/src/runtime.cpp"]


@pytest.mark.skipif(not (ROOT / "oracle" / "_ref" / "patched" / "libiolm_ref_gpu.so").exists(),
                    reason="patched reference not built")
def test_patched_library_links_the_engine():
    res = subprocess.run(["nm", "-D", "-C", str(ROOT / "oracle" / "_ref" / "patched" / "libiolm_ref_gpu.so")],
                         capture_output=True, text=True, check=True)
    assert "U iolm_cuda_create" in res.stdout and "U iolm_cuda_decode" in res.stdout
    assert "iolm::ModelRuntime::batch_decode" in res.stdout
