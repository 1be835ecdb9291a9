"""GEMM micro-benchmark sweep (kernel tuning aid; never a bench number): C1 shapes x epilogues."""
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2507_04967_b200 import _lib  # noqa: E402

lib = _lib.load()
T = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
shapes = {"qkv": (T, 3840, 1280), "o": (T, 1280, 1280), "in": (T, 5120, 1280), "out": (T, 1280, 5120)}
res = {}
for name, (M, N, K) in shapes.items():
    for epi, en in [(0, "f32"), (1, "bf16"), (2, "gelu"), (3, "resid")]:
        for pair in (1, 0):
            for i8 in (0, 1, 2):
                ms = C.c_float()
                st = lib.iolm_cuda_debug_gemm_time(M, N, K, epi, pair, i8, 20, C.byref(ms))
                if st:
                    continue
                tf = 2.0 * M * N * K / (ms.value * 1e-3) / 1e12
                key = f"{name} {en} {'pair' if pair else 'single'} {['bf16', 'i8', 'w4a16'][i8]}"
                res[key] = (round(ms.value * 1000, 1), round(tf))
                print(f"{key:28s} {ms.value*1000:8.1f} us  {tf:6.0f} TFLOP/s", flush=True)
Path("gpurun_out/gemm_sweep.json").write_text(json.dumps(res, indent=1))
