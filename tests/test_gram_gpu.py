"""Calibration Gram matrix on the GPU (iolm_cuda_gram): h = scale * X^T X in f64,
BIT-identical to the reference's fastmath::gram_accumulate (proj/src/fastmath.cpp:79-100): the same
sequential f64 sum over samples of exact f32 x f32 products. The restatement here is that sum in numpy
(elementwise adds in sample order). The reference itself is compared in tests/cpp/patched_ref_test.cpp
(build_hessian with and without IOLM_CUDA_DEVICE, and the GPTQ bundle built on it)."""
import ctypes as C

import numpy as np
import pytest

from paper_2507_04967_b200 import _lib

pytestmark = pytest.mark.gpu


def gram_gpu(x, scale=2.0):
    x = np.ascontiguousarray(x, np.float32)
    h = np.empty((x.shape[1], x.shape[1]), np.float64)
    st = _lib.load().iolm_cuda_gram(0, x.ctypes.data, x.shape[0], x.shape[1], C.c_double(scale), h.ctypes.data)
    assert st == 0, _lib.last_error()
    return h


def gram_ref(x, scale=2.0):
    acc = np.zeros((x.shape[1], x.shape[1]), np.float64)
    for s in range(x.shape[0]):  # ascending sample order; each product exact in f64
        r = x[s].astype(np.float64)
        acc = acc + np.outer(r, r)
    return scale * np.triu(acc) + scale * np.triu(acc, 1).T


@pytest.mark.parametrize("rows,cols", [(1, 1), (7, 63), (300, 128), (97, 200), (1000, 64)])
def test_gram_bit_exact(rows, cols):
    rng = np.random.default_rng(rows * 1000 + cols)
    x = rng.standard_normal((rows, cols)).astype(np.float32) * rng.uniform(0.01, 30, cols).astype(np.float32)
    x[rng.random((rows, cols)) < 0.1] = 0.0  # the reference skips x_si == 0 terms
    g, r = gram_gpu(x), gram_ref(x)
    assert np.array_equal(g, r)
    assert np.array_equal(g, g.T)


def test_gram_rejects_bad_arguments():
    lib = _lib.load()
    h = np.empty(4, np.float64)
    x = np.ones((2, 2), np.float32)
    assert lib.iolm_cuda_gram(0, x.ctypes.data, 0, 2, C.c_double(2.0), h.ctypes.data) == _lib.IOLM_E_CONTRACT
