"""A/B of the GEMM epilogue store path at the C1 engine shapes (run with IOLM_GEMM_TMA_EPI=0 / 1)."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2507_04967_b200 import _lib  # noqa: E402

lib = _lib.load()
T = 18944
for name, (N, K, epi) in {"o resid": (1280, 1280, 3), "out resid": (1280, 5120, 3), "in gelu": (5120, 1280, 2)}.items():
    ms = C.c_float()
    assert lib.iolm_cuda_debug_gemm_time(T, N, K, epi, 1, 0, 20, C.byref(ms)) == 0
    print(f"{name:10s} {ms.value * 1000:7.1f} us {2.0 * T * N * K / ms.value / 1e9:6.0f} TFLOP/s", flush=True)
