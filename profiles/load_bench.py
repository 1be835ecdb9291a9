"""Model load time: bundle (iolm_cuda_create: parse, FNV-1a over the serialized bundle, decode /
repack every weight on load) vs device-layout image (iolm_cuda_create_from_image: streamed read +
H2D of the pre-tiled HBM layout), for the bench configs. Both through the C ABI, CUDA context
already initialised. "cold" evicts the image from the page cache first (posix_fadvise DONTNEED).
Checks that the image-loaded runtime decodes bit-identically. Writes gpurun_out/load_times.json.

usage: python profiles/load_bench.py [config ...]"""
import ctypes as C
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402  (CONFIGS)
from paper_2507_04967_b200 import _lib  # noqa: E402
from paper_2507_04967_b200 import runtime as R  # noqa: E402
from paper_2507_04967_b200 import synth  # noqa: E402


def opts_for(cfg):
    return R.ModelRuntime._opts(act_quant=cfg.get("act_quant", False))


def timed_create(lib, fn):
    h = C.c_void_p()
    t = time.perf_counter()
    st = fn(h)
    dt = time.perf_counter() - t
    if st:
        raise RuntimeError(_lib.last_error())
    return h, dt


def evict(path):
    fd = os.open(path, os.O_RDONLY)
    try:
        os.fsync(fd)
        os.posix_fadvise(fd, 0, 0, os.POSIX_FADV_DONTNEED)
    finally:
        os.close(fd)


def decode(lib, h, ids, offs):
    n = len(offs) - 1
    oi = np.zeros((n, 8), np.int32)
    ol = np.zeros(n, np.int32)
    m, bad = C.c_uint64(), C.c_int64()
    st = lib.iolm_cuda_decode(h, ids.ctypes.data, offs.ctypes.data, n, 8, oi.ctypes.data, ol.ctypes.data,
                              C.byref(m), C.byref(bad))
    if st:
        raise RuntimeError(_lib.last_error())
    return oi, ol, m.value


def free_bytes(d):
    st = os.statvfs(d)
    return st.f_bavail * st.f_frsize


def main():
    names = sys.argv[1:] or ["c1", "c2-w4a16", "c3", "c4"]
    lib = _lib.load()
    warm = synth.toy_bundle(128, 2, 4, 512, 160, seed=1)
    h0, _ = timed_create(lib, lambda h: lib.iolm_cuda_create(C.c_char_p(warm), len(warm), 0, None, C.byref(h)))
    lib.iolm_cuda_destroy(h0)
    out = {}
    for name in names:
        cfg = bench.CONFIGS[name]
        bundle = synth.toy_bundle(*cfg["dims"], seed=42, quant=cfg["quant"], heads=cfg.get("heads"),
                                  ffn=cfg.get("ffn"))
        o = opts_for(cfg)
        ids, offs = synth.rows(0, 64, cfg["row_chars"])
        bhash = synth.fnv1a(bundle)  # the registry index entry's hash (known before loading)
        hb, t_mem = timed_create(
            lib, lambda h: lib.iolm_cuda_create(C.c_char_p(bundle), len(bundle), 0, C.byref(o), C.byref(h)))
        ref = decode(lib, hb, ids, offs)
        r = {"bundle_bytes": len(bundle), "create_from_bundle_in_memory_s": round(t_mem, 3)}
        for d in ["/dev/shm", "/tmp"]:
            if free_bytes(d) < 3 * len(bundle) + (1 << 30):
                r[d] = "skipped: not enough space"
                continue
            bpath, ipath = f"{d}/iolm_lb.iolm", f"{d}/iolm_lb.iolmdev"
            Path(bpath).write_bytes(bundle)
            t = time.perf_counter()
            if lib.iolm_cuda_save_image(hb, ipath.encode()):
                raise RuntimeError(_lib.last_error())
            t_save = time.perf_counter() - t
            res = {"image_bytes": os.path.getsize(ipath), "save_image_s": round(t_save, 3)}
            for mode in (["warm", "cold"] if d == "/tmp" else ["warm"]):
                if mode == "cold":
                    evict(bpath)
                t = time.perf_counter()
                data = Path(bpath).read_bytes()  # the registry's load_bundle(entry.path) reads the file
                h1, t_c = timed_create(
                    lib, lambda h: lib.iolm_cuda_create(C.c_char_p(data), len(data), 0, C.byref(o), C.byref(h)))
                res[f"bundle_file_{mode}_s"] = round(time.perf_counter() - t, 3)
                lib.iolm_cuda_destroy(h1)
                del data
                if mode == "cold":
                    evict(ipath)
                hi, t_i = timed_create(lib, lambda h: lib.iolm_cuda_create_from_image(
                    ipath.encode(), bhash, 0, C.byref(o), C.byref(h)))
                res[f"image_file_{mode}_s"] = round(t_i, 3)
                if mode == "warm":
                    t = time.perf_counter()
                    Path(ipath).read_bytes()
                    res["image_plain_read_warm_s"] = round(time.perf_counter() - t, 3)
                res[f"decode_bit_identical_{mode}"] = all(
                    np.array_equal(x, y) for x, y in zip(ref, decode(lib, hi, ids, offs)))
                lib.iolm_cuda_destroy(hi)
            os.remove(bpath)
            os.remove(ipath)
            r[d] = res
        lib.iolm_cuda_destroy(hb)
        out[name] = r
        print(name, json.dumps(r), flush=True)
    Path("gpurun_out").mkdir(exist_ok=True)
    Path("gpurun_out/load_times.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
