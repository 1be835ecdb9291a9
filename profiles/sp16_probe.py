"""Probe of the kind::f16 sparse MMA metadata layout (debug only): X = identity rows, so output column n
of token t is the effective dense weight W_hw[n, t]; the positions of its two nonzeros per group of 4
give the nibble the hardware applied. Saves intended and observed nibbles to gpurun_out/sp16_probe.npz."""
import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2507_04967_b200 import _lib
lib = _lib.load()
N, K = 256, 256
G = K // 4
PAIRS = [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)]
rng = np.random.default_rng(7)
sel = rng.integers(0, 6, size=(N, G))
pos = np.array(PAIRS, np.uint8)[sel]
codes = np.ones((N, G, 2), np.int8)
codes[..., 1] = 2
nib = (pos[..., 0] | (pos[..., 1] << 2)).astype(np.uint8)
idx = (nib[:, 0::2] | (nib[:, 1::2] << 4)).astype(np.uint8)
scales = np.ones(N, np.float32)
payload = np.frombuffer(codes.tobytes() + idx.tobytes() + scales.tobytes(), np.uint8).copy()
T = K
X = np.eye(T, K, dtype=np.float32)
xb = (X.view(np.uint32) >> 16).astype(np.uint16)
out = np.zeros((T, N), np.float32)
st = lib.iolm_cuda_debug_gemm_sp24_bf16(xb.ctypes.data, payload.ctypes.data, T, N, K, out.ctypes.data)
print("status", st, _lib.last_error())
W = out.T.reshape(N, G, 4)
hw = np.full((N, G), 255, np.uint8)
for r in range(N):
    for g in range(G):
        p0 = np.where(W[r, g] == 1)[0]
        p1 = np.where(W[r, g] == 2)[0]
        if len(p0) == 1 and len(p1) == 1:
            hw[r, g] = p0[0] | (p1[0] << 2)
print("match", float((hw == nib).mean()), "decodable", float((hw != 255).mean()))
Path("gpurun_out").mkdir(exist_ok=True)
np.savez("gpurun_out/sp16_probe.npz", nib=nib, hw=hw, W=W)
