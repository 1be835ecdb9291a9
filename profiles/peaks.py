"""Measured tensor-core peaks for the roofline denominators of the int8 configs (C2-W8A8, C3, C4).

VERDICT r01 #4: the kind::i8 and 2:4 .sp kind::i8 peaks were datasheet ratios (2x / 4x of the bf16
figure). This measures them, with the SM clocks and throttle reasons sampled by nvidia-smi during
every timed loop:

  * library references: cuBLAS bf16 (torch.matmul) and cuBLASLt int8 (torch._int_mm, s8 x s8 -> s32)
    at a large square shape;
  * the engine's own tcgen05 mainloops with the epilogue disabled (EPI_NONE: accumulators drained,
    not read; iolm_cuda_debug_gemm_time / _sp24_time), dense bf16, dense kind::i8 and 2:4 sparse
    kind::i8 (dense-equivalent ops: 2*M*N*K), at a large shape (T = 16384 tokens, N = K = 8192).

Each is run as a burst (~0.2 s) and sustained (a loop of >= 4 s, the regime of a kernel inside a
long bench step under the 1000 W cap). Output: one JSON object (gpurun_out/r02_peaks.json, copied to
profiles/r02_peaks.json). bench.py takes the int8 denominators from the larger of the library and
mainloop figures of the same kind (sustained), so a fraction never exceeds what the hardware was
measured to do. Never a bench number.
"""
from __future__ import annotations

import ctypes as C
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from bench import ClockSampler  # noqa: E402
from paper_2507_04967_b200 import _lib  # noqa: E402

lib = _lib.load()


def timed(fn, ops_per_call: float, seconds: float) -> dict:
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    n = 0
    while time.perf_counter() - t0 < 0.05:
        fn()
        n += 1
    torch.cuda.synchronize()
    per = (time.perf_counter() - t0) / max(n, 1)
    iters = max(3, int(seconds / max(per, 1e-6)))
    clk = ClockSampler(torch.cuda.current_device())
    clk.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    c = clk.stop()
    ms = e0.elapsed_time(e1) / iters
    return {"tops": ops_per_call / (ms * 1e-3) / 1e12, "ms_per_call": ms, "iters": iters,
            "sm_mhz": c["sm_mhz"], "reasons": c["reasons"]}


def engine_timed(kind: str, T: int, N: int, K: int, seconds: float) -> dict:
    """The debug entry point times `iters` back-to-back launches itself (CUDA events)."""
    def call(iters):
        ms = C.c_float()
        if kind == "sp24_i8":
            st = lib.iolm_cuda_debug_gemm_sp24_time(T, N, K, 6, iters, C.byref(ms))
        elif kind == "sp24_bf16":
            st = lib.iolm_cuda_debug_gemm_sp24_f16_time(T, N, K, 6, iters, C.byref(ms))
        else:
            st = lib.iolm_cuda_debug_gemm_time(T, N, K, 6, 1, 1 if kind == "i8" else 0, iters, C.byref(ms))
        if st:
            raise RuntimeError(_lib.last_error())
        return ms.value
    per = call(3)
    iters = max(3, int(seconds / (per * 1e-3)))
    clk = ClockSampler(torch.cuda.current_device())
    clk.start()
    ms = call(iters)
    c = clk.stop()
    return {"tops": 2.0 * T * N * K / (ms * 1e-3) / 1e12, "ms_per_call": ms, "iters": iters,
            "sm_mhz": c["sm_mhz"], "reasons": c["reasons"]}


def main():
    out = {"gpu": torch.cuda.get_device_name(0), "note": __doc__.split("\n\n")[0]}
    S = 8192
    a = torch.randn(S, S, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(S, S, device="cuda", dtype=torch.bfloat16)
    ai = torch.randint(-127, 128, (S, S), device="cuda", dtype=torch.int8)
    bi = torch.randint(-127, 128, (S, S), device="cuda", dtype=torch.int8)
    ops = 2.0 * S * S * S
    res = {}
    res["cublas_bf16"] = {m: timed(lambda: torch.matmul(a, b), ops, s) for m, s in (("burst", 0.2), ("sustained", 4.0))}
    try:
        res["cublaslt_i8"] = {m: timed(lambda: torch._int_mm(ai, bi.t()), ops, s)
                              for m, s in (("burst", 0.2), ("sustained", 4.0))}
    except Exception as e:  # noqa: BLE001
        res["cublaslt_i8"] = {"error": str(e)[:200]}
    del a, b, ai, bi
    torch.cuda.empty_cache()
    T, N, K = 16384, 8192, 8192
    for kind in ("bf16", "i8", "sp24_i8", "sp24_bf16"):
        res[f"engine_mainloop_{kind}"] = {m: engine_timed(kind, T, N, K, s) for m, s in (("burst", 0.2), ("sustained", 4.0))}
        res[f"engine_mainloop_{kind}"]["shape"] = [T, N, K]
    src = torch.empty(1 << 30, device="cuda", dtype=torch.float32)
    dst = torch.empty_like(src)
    hb = timed(lambda: dst.copy_(src), 2.0 * src.numel() * 4 * 1e3, 2.0)  # "tops" slot holds GB/s here
    res["hbm_copy"] = {"gbs": hb["tops"], "ms_per_call": hb["ms_per_call"], "sm_mhz": hb["sm_mhz"],
                       "reasons": hb["reasons"], "bytes_per_call": 2 * src.numel() * 4}
    del src, dst
    out["results"] = res

    def best(keys):
        vals = [res[k]["sustained"]["tops"] for k in keys if "sustained" in res.get(k, {})]
        return max(vals) if vals else None

    out["peaks_tops_sustained"] = {
        "bf16": best(["cublas_bf16", "engine_mainloop_bf16"]),
        "i8": best(["cublaslt_i8", "engine_mainloop_i8"]),
        "sp24_i8": best(["engine_mainloop_sp24_i8"]),
        "sp24_bf16": best(["engine_mainloop_sp24_bf16"]),
    }
    out["hbm_gbs"] = res["hbm_copy"]["gbs"]
    out["peaks_tops_burst"] = {
        k: max(res[x]["burst"]["tops"] for x in xs if "burst" in res.get(x, {}))
        for k, xs in (("bf16", ["cublas_bf16", "engine_mainloop_bf16"]), ("i8", ["cublaslt_i8", "engine_mainloop_i8"]),
                      ("sp24_i8", ["engine_mainloop_sp24_i8"]), ("sp24_bf16", ["engine_mainloop_sp24_bf16"]))}
    text = json.dumps(out, indent=1)
    print(text)
    (ROOT / "gpurun_out").mkdir(exist_ok=True)
    (ROOT / "gpurun_out" / "r02_peaks.json").write_text(text)


if __name__ == "__main__":
    main()
