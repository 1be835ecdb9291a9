#!/usr/bin/env python
"""Throughput benchmark of the B200 prompt() hot path (IOLM-DB, arXiv 2507.04967).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c1] [--rows-per-step B]
    python bench.py --impl reference ...        # the reference's own CPU path on the host cores

Metric (BASELINE.json): rows/sec for the whole box. A "step" is one pass of the hot path over one
batch of B synthetic table rows (BOS + 31-char instruction + R random printable
chars, 8 greedy new tokens) on every GPU; rows are distinct across steps and ranks (weak scaling:
rank r of N processes rows [(k*N + r)*B, (k*N + r + 1)*B) in step k).

  value : rows/s with the token ids already resident in HBM (iolm_cuda_decode_device_ids)
  e2e   : rows/s through the public C ABI with HOST buffers (iolm_cuda_decode): pinned host ids
          -> H2D -> prefill/decode -> generated ids back on the host, all inside the timed region
Each step's activations (~GBs) exceed the 126 MB L2, so no explicit flush is needed between steps.
Timing: torch CUDA events around the K steps after a barrier + synchronize, max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    # name: dims (d, L, H, F, S), row chars, quant, description
    "c0": dict(dims=(128, 4, 4, 512, 160), row_chars=64, quant="dense",
               desc="C0: toy decoder (128,4,4,512,160) dense, 32-token prefix + 64-token row, 8 new tokens"),
    "c1": dict(dims=(1280, 24, 20, 5120, 128), row_chars=64, quant="dense",
               desc="C1: 0.5B-class decoder (1280,24,20,5120,128) fp16 dense, 32-token prefix + 64-token row, "
                    "8 new tokens"),
    "c2-w8a8": dict(dims=(1280, 24, 20, 5120, 128), row_chars=64, quant="q8", act_quant=True,
                    desc="C2: C1 model, q8_perchannel RTN weights + per-token int8 activations (W8A8, "
                         "tcgen05 kind::i8), 32+64 tokens, 8 new tokens"),
    "c2-w4a16": dict(dims=(1280, 24, 20, 5120, 128), row_chars=64, quant="q4",
                     desc="C2: C1 model, q4_perchannel RTN weights, fp16 activations (W4A16), 32+64, 8 new"),
    "c3": dict(dims=(1280, 24, 20, 5120, 128), row_chars=64, quant="sparse24", act_quant=True,
               heads=[10] * 24, ffn=[2560] * 24,
               desc="C3: C1 model pruned 50% (10 of 20 heads, FFN 2560) + 2:4 magnitude + q8 (sparse24_q8), "
                    "W8A8, 32+64, 8 new"),
    "c3-f16": dict(dims=(1280, 24, 20, 5120, 128), row_chars=64, quant="sparse24",
                    heads=[10] * 24, ffn=[2560] * 24,
                    desc="C3 model (pruned 50% + 2:4 + q8 codes, sparse24_q8) with fp16 activations - the drop-in "
                         "default without act_quant: 2:4 sparse tensor cores kind::f16, 32+64, 8 new"),
    "c3b": dict(dims=(1280, 24, 20, 5120, 128), row_chars=64, quant="sparse24", act_quant=True,
                heads=[7 + l % 6 for l in range(24)], ffn=[2500 + 12 * l for l in range(24)],
                desc="C3b: C1 model with irregular per-layer pruning (7-12 of 20 heads, FFN 2500 + 12 l) + 2:4 + q8 "
                     "(sparse24_q8), W8A8, 32+64, 8 new"),
    "c4": dict(dims=(2048, 28, 16, 8192, 576), row_chars=512, quant="sparse24", act_quant=True,
               heads=[8] * 28, ffn=[4096] * 28,
               desc="C4: 1.5B-class (2048,28,16,8192,576) pruned 50% + 2:4 + q8, W8A8, 32-token prefix + "
                    "512-token row, 8 new"),
}
MAX_NEW = 8
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def load_peaks() -> tuple[dict, str]:
    """hbm / 16-bit tensor denominators (fp16 and bf16 run at the same tcgen05 kind::f16 rate): the driver's MEASURED_PEAKS.json; else this repo's own measurement
    on the pool (profiles/r02_peaks.json, profiles/peaks.py); else the guide's fallback."""
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return json.loads(p.read_text()), "measured (MEASURED_PEAKS.json)"
    own = int8_peaks()
    if own and "cublas_bf16" in own["results"]:
        # the driver's method: a copy and cuBLAS bf16 (not the engine's own, faster mainloop)
        r = own["results"]
        return ({"hbm_gbs": own["hbm_gbs"], "bf16_tflops": r["cublas_bf16"]["burst"]["tops"],
                 "bf16_tflops_sustained": r["cublas_bf16"]["sustained"]["tops"]},
                "measured on this pool: copy + cuBLAS bf16 (profiles/r02_peaks.json; MEASURED_PEAKS.json absent)")
    return PEAKS_FALLBACK, "fallback (B200_PROFILING.md)"


def int8_peaks() -> dict | None:
    """Measured kind::i8 and 2:4 sparse kind::i8 rates (profiles/peaks.py -> profiles/r02_peaks.json):
    the larger of cuBLASLt int8 and the engine's own mainloop-only kernel, sustained (>= 4 s loops)."""
    p = ROOT / "profiles" / "r02_peaks.json"
    return json.loads(p.read_text()) if p.exists() else None


def cpu_model() -> str:
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampling of SM clocks and throttle reasons during the timed region."""

    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.sw_power_cap",
              "clocks_event_reasons.hw_slowdown", "clocks_event_reasons.hw_thermal_slowdown",
              "clocks_event_reasons.sw_thermal_slowdown"]

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={','.join(self.FIELDS)}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------------------- distributed plumbing
def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
        if backend == "nccl":
            import torch
            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend)
        _cpu_group()  # collective: created by every rank up front
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def allreduce_max(world, value: float, device=None) -> float:
    if world == 1:
        return value
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def allreduce_sum(world, value: float, device=None) -> float:
    if world == 1:
        return value
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def step_rows(step: int, world: int, rank: int, B: int) -> int:
    """First global table row of (step, rank): weak scaling, no row reused."""
    return (step * world + rank) * B


_CPU_GROUP = None


def _cpu_group():
    global _CPU_GROUP
    import torch.distributed as dist
    if _CPU_GROUP is None:
        _CPU_GROUP = dist.new_group(backend="gloo") if dist.get_backend() != "gloo" else dist.group.WORLD
    return _CPU_GROUP


# --------------------------------------------------------------------------- CPU reference
def cpu_reference_sample(bundle: bytes, cfg: dict, n_rows: int, first_row: int, threads: int):
    """Times the reference's CPU batch_decode on n_rows synthetic rows with `threads` host threads.
    Returns (rows/s, kind, seconds, outputs)."""
    from oracle import oracle as O
    from paper_2507_04967_b200 import synth
    prompts = synth.row_strings(first_row, n_rows, cfg["row_chars"])
    if O.ref_available():
        rt = O.RefRuntime(bundle)
        t0 = time.perf_counter()
        outs, _ = rt.batch_decode(prompts, MAX_NEW, threads=threads, batch_size=1)
        dt = time.perf_counter() - t0
        return n_rows / dt, "reference", dt, outs
    om = O.OracleModel(bundle)
    ids, offs = synth.rows(first_row, n_rows, cfg["row_chars"])
    t0 = time.perf_counter()
    oi, ol, _ = om.decode_ids(ids, offs, MAX_NEW, threads=threads)
    dt = time.perf_counter() - t0
    return n_rows / dt, "port", dt, [O.render(oi[i], ol[i]) for i in range(n_rows)]


def divergence_gaps(bundle: bytes, cfg: dict, first_row: int, cpu_outs, gpu_outs) -> list:
    """Each row where the GPU's greedy output differs from the CPU reference's: the first differing
    character and the CPU top-1/top-2 logit gap there (the C restatement, bit-exact with the
    reference, replays prompt + common prefix), against the near-tie bound 0.05 + 4e-3 max|logit|
    of tests/parity.py. Checker only: runs after the timed regions."""
    bad = [i for i, (a, b) in enumerate(zip(cpu_outs, gpu_outs)) if a != b]
    if not bad:
        return []
    from oracle import oracle as O
    from paper_2507_04967_b200 import synth
    om = O.OracleModel(bundle)
    prompts = synth.row_strings(first_row, len(cpu_outs), cfg["row_chars"])
    res = []
    for i in bad:
        a, b = cpu_outs[i], gpu_outs[i]
        k = 0
        while k < min(len(a), len(b)) and a[k] == b[k]:
            k += 1
        ids = np.array([129] + [ord(c) for c in prompts[i] + a[:k]], np.int32)
        lg = om.forward(ids)[0][-1]
        top = np.sort(lg)
        gap = float(top[-1] - top[-2])
        tol = 0.05 + 4e-3 * float(np.abs(lg).max())
        res.append({"row": i, "char": k, "cpu_top2_gap": gap, "tie_bound": tol, "tie": gap < tol})
    return res


def cpu_sample_rows(name: str, cores: int) -> int:
    # ~10-30 s of CPU work: C1 costs ~25 s per row per core, C0 ~36 ms per row per core
    return cores if name != "c0" else 256 * cores


def run_reference_arm(args, cfg: dict, world: int, rank: int) -> None:
    if rank != 0:
        return
    from oracle import oracle as O
    cores = os.cpu_count() or 1
    if O.ref_available() and cfg["quant"] == "dense" and "heads" not in cfg:
        bundle = O.ref_toy_bundle(*cfg["dims"], seed=42)
    else:
        from paper_2507_04967_b200 import synth
        bundle = synth.toy_bundle(*cfg["dims"], seed=42, quant=cfg["quant"], heads=cfg.get("heads"),
                                  ffn=cfg.get("ffn"))
    n = cpu_sample_rows(args.config, cores)
    # untimed warm-up: W rows of the same workload, one per thread, run concurrently
    if args.warmup > 0:
        cpu_reference_sample(bundle, cfg, args.warmup, 10_000_000, args.warmup)
    rates, kinds, secs = [], [], 0.0
    for k in range(args.steps):
        r, kind, dt, _ = cpu_reference_sample(bundle, cfg, n, step_rows(k, 1, 0, n), cores)
        rates.append(r)
        kinds.append(kind)
        secs += dt
    value = args.steps * n / secs
    line = {
        "impl": "reference", "metric": "rows/sec", "value": value, "unit": "rows/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * secs / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": {"workload": cfg["desc"], "rows_per_step": n, "max_new_tokens": MAX_NEW,
                                        "sample": f"{n} rows per step, one reference batch_decode per row"},
        "cpu_baseline": {"value": value, "unit": "rows/s", "cores": cores, "cpu_model": cpu_model(), "kind": kinds[0],
                         "sample": f"{n} rows x {args.steps} steps on {cores} host threads"},
        "e2e": {"value": value, "unit": "rows/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- GPU arm
def multi_device_e2e(args, cfg: dict, bundle: bytes, world: int, B: int, W: int, K: int, rank0_outs):
    """Rank 0 of an N-rank run: e2e rows/s through one multi-device context over GPUs 0..N-1."""
    import torch
    from paper_2507_04967_b200 import runtime as R
    from paper_2507_04967_b200 import synth
    devs = [0] * world if os.environ.get("BENCH_SHARE_GPUS") else list(range(world))
    mrt = R.ModelRuntime(bundle, device=devs, max_tokens_per_step=args.tokens_per_step,
                         prefill_tc={"auto": None, "on": True, "off": False}[args.prefill_tc],
                         act_quant=cfg.get("act_quant", False))
    host = []
    for k in range(W + K):  # step k's rows of all ranks: [k*N*B, (k+1)*N*B) (step_rows is rank-major)
        ids, offs = synth.rows(step_rows(k, world, 0, B), world * B, cfg["row_chars"])
        host.append((torch.from_numpy(ids).pin_memory(), offs))
    mrt.decode_token_rows(host[0][0].numpy(), host[0][1], MAX_NEW)  # warm-up
    torch.cuda.synchronize()
    # CUDA events on device 0 around synchronous calls: each returns with every device's ids on the host
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = None
    for k in range(W, W + K):
        out = mrt.decode_token_rows(host[k][0].numpy(), host[k][1], MAX_NEW)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    o, ln, _ = out
    o0, ln0 = rank0_outs[-1]
    if not (np.array_equal(ln[:B], ln0) and np.array_equal(o[:B], o0)):
        raise SystemExit("bench: multi-device e2e disagrees with rank 0's device-resident run")
    mrt.close()
    return ms, world * B * K


def run_gpu_arm(args, cfg: dict, world: int, rank: int, local: int) -> None:
    import torch
    from paper_2507_04967_b200 import runtime as R
    from paper_2507_04967_b200 import synth
    if os.environ.get("BENCH_SHARE_GPUS"):  # plumbing test only: N ranks on fewer GPUs
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    B, K, W = args.rows_per_step, args.steps, args.warmup
    t_setup = time.perf_counter()
    bundle = synth.toy_bundle(*cfg["dims"], seed=42, quant=cfg["quant"], heads=cfg.get("heads"),
                              ffn=cfg.get("ffn"))
    rt = R.ModelRuntime(bundle, device=local, kernel_timing=True, max_tokens_per_step=args.tokens_per_step,
                        prefill_tc={"auto": None, "on": True, "off": False}[args.prefill_tc],
                        act_quant=cfg.get("act_quant", False), sparse_mma=args.sparse_mma == "on")
    # this rank's rows for every warmup + timed step, host (pinned) and device copies
    host_ids, dev_ids, offsets = [], [], []
    for k in range(W + K):
        ids, offs = synth.rows(step_rows(k, world, rank, B), B, cfg["row_chars"])
        pinned = torch.from_numpy(ids).pin_memory()
        host_ids.append(pinned)
        dev_ids.append(pinned.to(dev))
        offsets.append(offs)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t_setup

    def run(k: int, device_inputs: bool):
        if device_inputs:
            return rt.decode_token_rows(None, offsets[k], MAX_NEW, device_ids=dev_ids[k].data_ptr())
        return rt.decode_token_rows(host_ids[k].numpy(), offsets[k], MAX_NEW)

    # per-kernel CUDA events cost ~3% of a step: off for the timed regions, on for a separate
    # roofline pass afterwards
    rt.set_kernel_timing(False)
    for w in range(W):
        run(w, True)
    # ---- timed region 1: inputs resident in HBM
    clocks = ClockSampler(local)
    barrier(world)
    torch.cuda.synchronize()
    clocks.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    launches, emitted, kt = 0, 0, {}
    eng_ms = 0.0
    outs = []
    for k in range(W, W + K):
        o, ln, _ = run(k, True)
        st = rt.last_stats()
        launches += st["kernel_launches"]
        eng_ms += st["device_ms"]
        emitted += int(ln.sum())
        outs.append((o, ln))
    ev1.record()
    torch.cuda.synchronize()
    barrier(world)
    clk = clocks.stop()
    ms = ev0.elapsed_time(ev1)
    ms_max = allreduce_max(world, ms, dev)

    # ---- timed region 2 (e2e), one GPU: host buffers through the public ABI
    gathered_rows = 0
    if world == 1:
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for k in range(W, W + K):
            o2, ln2, _ = run(k, False)
            gathered_rows += len(ln2)
        e1.record()
        torch.cuda.synchronize()
        e2e_ms = e0.elapsed_time(e1)
        # both regions must produce the same tokens (last step spot check)
        o_last, ln_last = outs[-1]
        if not (np.array_equal(ln2, ln_last) and np.array_equal(o2, o_last)):
            raise SystemExit("bench: device-input and host-input runs disagree")

    # ---- roofline pass (untimed for `value`): the same step inputs with per-kernel CUDA events
    kt_steps = 0
    if not args.no_kernel_timing:
        rt.set_kernel_timing(True)
        kt_steps = min(K, 2)
        for k in range(W, W + kt_steps):
            run(k, True)
            for name, (kms_, work_, cnt_) in rt.kernel_times().items():
                a = kt.setdefault(name, [0.0, 0.0, 0])
                a[0] += kms_
                a[1] += work_
                a[2] += cnt_
        rt.set_kernel_timing(False)

    if world > 1:
        # ---- timed region 2 (e2e), N GPUs: the product's multi-GPU API. Every rank releases its
        # context; rank 0 opens ONE context over all N GPUs (iolm_cuda_create_multi) and pushes each
        # step's N*B rows (exactly the rows the N ranks processed in that step) through it with host
        # buffers: H2D, range-partitioned decode on every GPU, ids written back into one host output
        # column in row order (the gather). The other ranks wait at the barrier.
        rt.close()
        barrier(world)
        e2e_ms, gathered_rows = 0.0, 0
        if rank == 0:
            e2e_ms, gathered_rows = multi_device_e2e(args, cfg, bundle, world, B, W, K, outs)
        e2e_ms = allreduce_max(world, e2e_ms, dev)
        barrier(world)

    rows_total = world * B * K
    value = rows_total / (ms_max / 1000.0)
    e2e = rows_total / (e2e_ms / 1000.0)
    peaks, peak_src = load_peaks()
    if not kt or max(v[0] for v in kt.values()) <= 0:  # --no-kernel-timing: no per-class times
        kt = {"none": [1e-9, 0.0, 0]}
    # dominant kernel class by device time
    dom = max(kt.items(), key=lambda kv: kv[1][0])
    name, (kms, work, cnt) = dom
    hbm_classes = {"attn_decode", "ln", "embed_ln", "head", "quant"}
    if name in hbm_classes:
        achieved = work / (kms / 1000.0) / 1e9
        peak = peaks["hbm_gbs"]
        unit, bound = "GB/s", "hbm"
    else:
        achieved = work / (kms / 1000.0) / 1e12
        peak = peaks["bf16_tflops_sustained"]
        unit, bound = "TFLOP/s", "tensor"
        if cfg["quant"] == "sparse24" and not cfg.get("act_quant"):
            ip = int8_peaks()
            if ip and ip["peaks_tops_sustained"].get("sp24_bf16"):
                peak = ip["peaks_tops_sustained"]["sp24_bf16"]
                peak_src = "measured sustained 2:4 sparse kind::f16 (engine mainloop-only), profiles/r02_peaks.json"
        if cfg.get("act_quant"):
            # int8 GEMMs (ops counted dense-equivalent): the MEASURED sustained kind::i8 / 2:4 sparse
            # kind::i8 rate (profiles/r02_peaks.json); the datasheet ratios (2x / 4x bf16) only if absent
            sparse = cfg["quant"] == "sparse24"
            ip = int8_peaks()
            if ip and ip["peaks_tops_sustained"].get("sp24_i8" if sparse else "i8"):
                peak = ip["peaks_tops_sustained"]["sp24_i8" if sparse else "i8"]
                peak_src = ("measured sustained " + ("2:4 sparse kind::i8 (engine mainloop-only, N=K=8192)" if sparse
                            else "kind::i8 (max of cuBLASLt int8 and engine mainloop-only, 8192^3)") +
                            ", profiles/r02_peaks.json")
            else:
                mult = 4.0 if sparse else 2.0
                peak *= mult
                peak_src = f"{peak_src} x {mult:g} (int8{' 2:4 sparse' if mult == 4 else ''} datasheet ratio)"
    traffic = None
    prof = ROOT / "profiles" / "traffic.json"
    if prof.exists():
        try:
            traffic = json.loads(prof.read_text()).get(args.config, {}).get(name)
        except Exception:
            traffic = None
    kernels = {}
    for n_, (kms_, work_, cnt_) in kt.items():
        if cnt_ == 0:
            continue
        is_bytes = n_ in hbm_classes
        rate = work_ / (kms_ / 1000.0) / (1e9 if is_bytes else 1e12) if kms_ > 0 else None
        kernels[n_] = {"ms": round(kms_, 3), "launches": cnt_, "share": round(kms_ / max(1e-9, sum(v[0] for v in kt.values())), 4),
                       ("GB/s" if is_bytes else "TFLOP/s"): None if rate is None else round(rate, 2)}
    gemm_ms = sum(kt[c][0] for c in ("gemm_qkv", "gemm_o", "gemm_in", "gemm_out") if c in kt)
    gemm_fl = sum(kt[c][1] for c in ("gemm_qkv", "gemm_o", "gemm_in", "gemm_out") if c in kt)

    cpu = None
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        cores = os.cpu_count() or 1
        n = cpu_sample_rows(args.config, cores)
        rate, kind, dt, cpu_outs = cpu_reference_sample(bundle, cfg, n, step_rows(W, 1, 0, B), cores)
        gpu_outs = [R.decode_ids(outs[0][0][i, :outs[0][1][i]]) for i in range(n)]
        agree = sum(a == b for a, b in zip(cpu_outs, gpu_outs)) / n
        cpu = {"value": rate, "unit": "rows/s", "cores": cores, "cpu_model": cpu_model(), "kind": kind,
               "sample": f"first {n} rows of timed step 0, one batch_decode per row, {cores} threads, {dt:.1f} s",
               "greedy_agreement_with_gpu": agree,
               "divergences": divergence_gaps(bundle, cfg, step_rows(W, 1, 0, B), cpu_outs, gpu_outs)}
    if rank != 0:
        return
    h2d = sum(int(h.numel()) * 4 for h in host_ids[W:]) // K + (B + 1) * 8
    d2h = B * MAX_NEW * 4 + B * 4
    line = {
        "metric": "rows/sec", "value": value, "unit": "rows/s", "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": ms_max / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "s8 x s8 -> s32 (W8A8)" if cfg.get("act_quant") else "f16", "data": "synthetic (seeded rows, random-init weights: ToyModelParams::init seed 42)",
        "config": {"workload": cfg["desc"], "rows_per_step_per_gpu": B, "max_new_tokens": MAX_NEW,
                   "tokens_per_engine_step": args.tokens_per_step or (
                       "SMs/2 x 224 (16576 on B200: whole waves of the 2:4 sparse kernel's 224-token tiles)"
                       if cfg["quant"] == "sparse24" and cfg.get("act_quant") else "SMs/2 x 256 (18944 on B200)"),
                   "l2": "inputs larger than L2 (GB-scale activations per step)",
                   "parallelism": f"rows range-partitioned over {world} GPU(s), full replica each"},
        "e2e": {"value": e2e, "unit": "rows/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": launches,
        "roofline": {"bound": bound, "kernel": name, "achieved": achieved, "peak": peak, "unit": unit,
                     "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src},
        "gemm_all": {"tflops": gemm_fl / (gemm_ms / 1000.0) / 1e12 if gemm_ms else None,
                     "share_of_step": gemm_ms / max(sum(v[0] for v in kt.values()), 1e-9)},
        "kernels": kernels,
        "kernel_timing": {"steps": kt_steps, "note": "per-kernel CUDA events on the engine stream in a separate "
                          "pass over the first timed steps' inputs; the timed regions run without them"},
        "clocks": clk,
        "cpu_baseline": cpu,
        "mean_new_tokens_per_row": emitted / (B * K),
        "rows_gathered_on_rank0": gathered_rows,
        "engine_device_ms": eng_ms,
        "setup_s": setup_s,
    }
    print(json.dumps(line), flush=True)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c1")
    ap.add_argument("--rows-per-step", type=int, default=16384)
    ap.add_argument("--tokens-per-step", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--prefill-tc", choices=["auto", "on", "off"], default="auto",
                    help="prefill attention kernel: engine default = O-in-TMEM tcgen05 kernel (auto), round-1 128-query tcgen05 kernel (on), mma.sync (off)")
    ap.add_argument("--sparse-mma", choices=["on", "off"], default="on",
                    help="2:4 bundles: sparse tensor cores (on) or weights expanded to dense codes (off), A/B")
    ap.add_argument("--no-kernel-timing", action="store_true",
                    help="no per-kernel CUDA events (A/B check of their overhead; no roofline)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    cfg = CONFIGS[args.config]
    world, rank, local = dist_setup()
    if args.impl == "reference":
        run_reference_arm(args, cfg, world, rank)
    else:
        run_gpu_arm(args, cfg, world, rank, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
