"""Build recipe for the sm_100a engine library (libiolm_cuda.so) and the harness library
(libiolm_synth.so). Both are built in-tree so they travel with the repo snapshot to the GPU box.

    python -m paper_2507_04967_b200.build          # incremental
    python -m paper_2507_04967_b200.build --force  # rebuild everything
"""
from __future__ import annotations

import hashlib
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
ENGINE_SO = PKG / "libiolm_cuda.so"
SYNTH_SO = PKG / "libiolm_synth.so"
OBJ_DIR = PKG / "_build"

NVCC = os.environ.get("NVCC", shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + [
    "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
    "--expt-relaxed-constexpr", "-Xptxas", "-v", f"-I{ROOT / 'include'}",
]


def _run(cmd: list[str], log: Path | None = None) -> None:
    res = subprocess.run(cmd, capture_output=True, text=True)
    if log is not None:
        log.write_text(res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"build step failed: {' '.join(cmd[:3])} ...")


def _digest(paths: list[Path], extra: str) -> str:
    h = hashlib.sha256(extra.encode())
    for p in sorted(paths):
        h.update(p.name.encode())
        h.update(p.read_bytes())
    return h.hexdigest()


def build_engine(force: bool = False) -> Path:
    headers = list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.hpp")) + list((ROOT / "include").glob("*.h"))
    sources = sorted(CSRC.glob("*.cu"))
    OBJ_DIR.mkdir(exist_ok=True)
    hdr_digest = _digest(headers, " ".join(NVCC_FLAGS))
    objs = []
    for src in sources:
        obj = OBJ_DIR / (src.stem + ".o")
        stamp = OBJ_DIR / (src.stem + ".stamp")
        d = _digest([src], hdr_digest)
        if force or not obj.exists() or not stamp.exists() or stamp.read_text() != d:
            _run([NVCC, *NVCC_FLAGS, "-c", str(src), "-o", str(obj)], OBJ_DIR / (src.stem + ".ptxas.log"))
            stamp.write_text(d)
        objs.append(obj)
    link_stamp = OBJ_DIR / "link.stamp"
    ld = _digest(objs, "link")
    if force or not ENGINE_SO.exists() or not link_stamp.exists() or link_stamp.read_text() != ld:
        _run([NVCC, *ARCH, "-shared", "-o", str(ENGINE_SO), *map(str, objs), "-lcudart_static", "-lpthread", "-ldl", "-lrt"])
        link_stamp.write_text(ld)
    return ENGINE_SO


def build_synth(force: bool = False) -> Path:
    src = CSRC / "synth.cpp"
    stamp = OBJ_DIR / "synth.stamp"
    OBJ_DIR.mkdir(exist_ok=True)
    d = _digest([src], "synth")
    if force or not SYNTH_SO.exists() or not stamp.exists() or stamp.read_text() != d:
        _run(["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-ffp-contract=off", "-pthread",
              "-o", str(SYNTH_SO), str(src)])
        stamp.write_text(d)
    return SYNTH_SO


def build_all(force: bool = False) -> None:
    build_synth(force)
    build_engine(force)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
    print(f"built {ENGINE_SO.name} and {SYNTH_SO.name}")
