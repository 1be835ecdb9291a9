"""The reference's own C++ ModelBundle through the C++ shim (include/iolm_cuda_runtime.hpp), side by
side with iolm::ModelRuntime in one process (tests/cpp/dropin_test.cpp, built by oracle/Makefile)."""
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
BIN = Path(__file__).resolve().parents[1] / "oracle" / "_ref" / "dropin_test"


@pytest.mark.skipif(not BIN.exists(), reason="drop-in binary not built (needs /root/reference at build time)")
def test_cpp_dropin_against_reference_runtime():
    res = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=600)
    assert res.returncode == 0 and "DROPIN OK" in res.stdout, res.stdout + res.stderr


def test_smoke_entry():
    import __graft_entry__
    __graft_entry__.smoke()


PATCHED = Path(__file__).resolve().parents[1] / "oracle" / "_ref" / "patched" / "patched_ref_test"


@pytest.mark.skipif(not PATCHED.exists(), reason="patched reference not built (needs /root/reference at build time)")
def test_patched_reference_through_unchanged_callers():
    """oracle/reference_gpu.patch applied to the reference (3 files) and rebuilt against the B200
    runtime: iolm::execute (prompt() + SEMANTIC JOIN), capture_calibration, validate and specialize
    run unchanged on the GPU and agree with the same library's CPU path (tests/cpp/patched_ref_test.cpp)."""
    res = subprocess.run([str(PATCHED)], capture_output=True, text=True, timeout=1200)
    print(res.stdout)
    assert res.returncode == 0 and "PATCHED REFERENCE OK" in res.stdout, res.stdout + res.stderr
