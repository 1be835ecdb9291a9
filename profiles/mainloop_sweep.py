"""Mainloop-only GEMM rates (EPI_NONE: accumulators drained, not read): dense kind::i8 vs 2:4 sparse
kind::i8 vs dense bf16, dense-equivalent TOP/s. Kernel tuning aid; never a bench number."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2507_04967_b200 import _lib  # noqa: E402

lib = _lib.load()
T = 18944
for N, K in [(2560, 1280), (1280, 5120), (2048, 16384), (4096, 4096)]:
    for name in ("sparse-i8", "dense-i8", "dense-bf16"):
        ms = C.c_float()
        if name == "sparse-i8":
            st = lib.iolm_cuda_debug_gemm_sp24_time(T, N, K, 6, 10, C.byref(ms))
        else:
            st = lib.iolm_cuda_debug_gemm_time(T, N, K, 6, 1, 1 if name == "dense-i8" else 0, 10, C.byref(ms))
        if st:
            print(N, K, name, "failed", _lib.last_error())
            continue
        print(f"N={N:5d} K={K:5d} {name:10s} {ms.value*1000:8.1f} us {2.0*T*N*K/(ms.value*1e-3)/1e12:6.0f} TOP/s", flush=True)
