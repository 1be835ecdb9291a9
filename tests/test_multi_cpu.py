"""Multi-device row split (iolm_cuda_create_multi's partition, engine.cu partition_rows) - host only.

The table is range-partitioned over full per-GPU replicas: contiguous, non-empty ranges
in row order covering every row once, with near-equal token counts (prefill dominates a row's
cost). The GPU side (bit-identical outputs to one device, error mapping) is tests/test_multi_gpu.py."""
import ctypes as C

import numpy as np
import pytest

from paper_2507_04967_b200 import _lib


def split(offs, shards):
    lib = _lib.load()
    offs = np.ascontiguousarray(offs, dtype=np.int64)
    cut = np.zeros(shards + 1, np.int64)
    n = C.c_int32()
    st = lib.iolm_cuda_debug_partition(offs.ctypes.data, len(offs) - 1, shards, cut.ctypes.data, C.byref(n))
    assert st == 0, _lib.last_error()
    return cut[:n.value]


@pytest.mark.parametrize("shards", [1, 2, 3, 8])
@pytest.mark.parametrize("seed", range(5))
def test_ranges_cover_rows_in_order_with_balanced_tokens(shards, seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 3000))
    lens = rng.integers(1, 600, size=n)
    offs = np.concatenate([[int(rng.integers(0, 50))], lens]).cumsum()
    cut = split(offs, shards)
    used = min(shards, n)
    assert len(cut) == used + 1 and cut[0] == 0 and cut[-1] == n
    assert np.all(np.diff(cut) >= 1)  # non-empty, ascending, contiguous
    tok = [offs[cut[i + 1]] - offs[cut[i]] for i in range(used)]
    if used > 1:
        assert max(tok) - min(tok) <= 2 * lens.max() + 1, (tok, lens.max())


def test_fewer_rows_than_devices():
    assert list(split(np.array([0, 5, 9]), 8)) == [0, 1, 2]
    assert list(split(np.array([0, 5]), 4)) == [0, 1]


def test_uniform_rows_split_evenly():
    offs = np.arange(0, 97 * 1000 + 1, 97)
    cut = split(offs, 8)
    assert list(np.diff(cut)) == [125] * 8


def test_bad_arguments():
    lib = _lib.load()
    offs = np.array([0, 4], np.int64)
    cut = np.zeros(4, np.int64)
    n = C.c_int32()
    assert lib.iolm_cuda_debug_partition(offs.ctypes.data, 1, 0, cut.ctypes.data, C.byref(n)) == _lib.IOLM_E_CONTRACT
    assert lib.iolm_cuda_debug_partition(offs.ctypes.data, 0, 2, cut.ctypes.data, C.byref(n)) == _lib.IOLM_E_CONTRACT
