"""Streaming prompt() resolver (include/iolm_cuda_resolver.hpp) vs the reference executor.

tests/cpp/resolver_test.cpp, built by oracle/Makefile against the unmodified reference:
* CPU build: the resolver drives the reference's own iolm::ModelRuntime and must reproduce
  iolm::execute (PromptResolver, proj/src/exec.cpp:84-159) exactly - outputs, row order, cache hits /
  misses and the invocation-count law - for batch sizes 1/4/16/64, cache capacities 0/3/1024 and
  device batches 1/7/100000, streaming take_ready(), cache reuse and the SequenceTooLong row suffix
  (the scenarios of proj/tests/test_query.cpp:375-431).
* GPU build: the same with iolm::cuda::ModelRuntime (B200) as the model.
"""
import subprocess
from pathlib import Path

import pytest

REF = Path(__file__).resolve().parents[1] / "oracle" / "_ref"


@pytest.mark.skipif(not (REF / "resolver_test").exists(), reason="resolver test not built (needs /root/reference)")
def test_resolver_matches_reference_executor_cpu():
    res = subprocess.run([str(REF / "resolver_test")], capture_output=True, text=True, timeout=600)
    assert res.returncode == 0 and "RESOLVER OK" in res.stdout, res.stdout + res.stderr


@pytest.mark.gpu
@pytest.mark.skipif(not (REF / "resolver_test_gpu").exists(), reason="resolver GPU test not built")
def test_resolver_on_gpu_runtime():
    res = subprocess.run([str(REF / "resolver_test_gpu")], capture_output=True, text=True, timeout=600)
    assert res.returncode == 0 and "RESOLVER OK" in res.stdout, res.stdout + res.stderr
