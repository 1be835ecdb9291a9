"""W4A16 (int4 expanded in smem) vs bf16 GEMM rates at C1 shapes; epi 6 = mainloop only (tuning aid)."""
import ctypes as C, sys
sys.path.insert(0, '.')
from paper_2507_04967_b200 import _lib
lib = _lib.load()
T = 18944
for N, K in [(3840, 1280), (5120, 1280), (1280, 5120)]:
    for epi in (6, 2):
        for i8 in (0, 2):
            ms = C.c_float()
            st = lib.iolm_cuda_debug_gemm_time(T, N, K, epi, 1, i8, 10, C.byref(ms))
            print(N, K, 'epi', epi, ['bf16', 'i8', 'w4'][i8], 'fail' if st else f"{ms.value*1000:.1f} us {2*T*N*K/ms.value/1e9:.0f} TF", flush=True)
for N, K in [(5120, 1280)]:
    for epi in (6, 2):
        for i8 in (0, 2):
            ms = C.c_float()
            st = lib.iolm_cuda_debug_gemm_time(T, N, K, epi, 0, i8, 10, C.byref(ms))
            print('single', N, K, 'epi', epi, ['bf16', 'i8', 'w4'][i8], 'fail' if st else f"{ms.value*1000:.1f} us {2*T*N*K/ms.value/1e9:.0f} TF", flush=True)
