"""One sparse and one dense kind::i8 GEMM launch at a C3 shape (for ncu captures)."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2507_04967_b200 import _lib  # noqa: E402

lib = _lib.load()
T, N, K, epi = (int(a) for a in (sys.argv[1:5] if len(sys.argv) >= 5 else (18944, 2560, 1280, 2)))
ms = C.c_float()
assert lib.iolm_cuda_debug_gemm_sp24_time(T, N, K, epi, 2, C.byref(ms)) == 0, _lib.last_error()
assert lib.iolm_cuda_debug_gemm_time(T, N, K, epi, 1, 1, 2, C.byref(ms)) == 0, _lib.last_error()
