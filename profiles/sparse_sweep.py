"""Sparse (tcgen05.mma.sp kind::i8) vs dense kind::i8 GEMM micro-benchmark at the C3 / C4 shapes
(kernel tuning aid; never a bench number). Dense-equivalent TOP/s = 2*T*N*K / time."""
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2507_04967_b200 import _lib  # noqa: E402

lib = _lib.load()
T = int(sys.argv[1]) if len(sys.argv) > 1 else 18944
shapes = {"c3 qkv": (T, 1920, 1280), "c3 o": (T, 1280, 640), "c3 in": (T, 2560, 1280), "c3 out": (T, 1280, 2560),
          "c1 in": (T, 5120, 1280), "c1 out": (T, 1280, 5120),
          "c4 qkv": (T, 3072, 2048), "c4 in": (T, 4096, 2048), "c4 out": (T, 2048, 4096)}
res = {}
for name, (M, N, K) in shapes.items():
    for epi, en in [(2, "gelu"), (3, "resid")]:
        for sp in (1, 0):
            ms = C.c_float()
            if sp:
                st = lib.iolm_cuda_debug_gemm_sp24_time(M, N, K, epi, 20, C.byref(ms))
            else:
                st = lib.iolm_cuda_debug_gemm_time(M, N, K, epi, 1, 1, 20, C.byref(ms))
            if st:
                print(name, en, sp, "failed", _lib.last_error())
                continue
            tops = 2.0 * M * N * K / (ms.value * 1e-3) / 1e12
            key = f"{name} {en} {'sparse' if sp else 'dense'}"
            res[key] = (round(ms.value * 1000, 1), round(tops))
            print(f"{key:24s} {ms.value*1000:8.1f} us  {tops:6.0f} TOP/s (dense-equivalent)", flush=True)
Path("gpurun_out").mkdir(exist_ok=True)
Path("gpurun_out/sparse_sweep.json").write_text(json.dumps(res, indent=1))
