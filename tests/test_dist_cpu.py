"""Multi-process host logic of the N-GPU bench on CPU (gloo, world size 2): row-range sharding is a
partition with no overlap whose rank blocks of one step are contiguous (so rank 0's multi-device e2e
call over all GPUs, bench.multi_device_e2e, pushes exactly the rows the ranks processed), and
max-over-ranks timing. The output-column gather itself is the multi-device context writing every
device's ids into one host column (tests/test_multi_gpu.py, tests/test_multi_cpu.py)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import bench


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank), BENCH_DIST_BACKEND="gloo")
    w, r, _ = bench.dist_setup()
    B = 5
    first = [bench.step_rows(k, w, r, B) for k in range(3)]
    t = bench.allreduce_max(w, float(10 + r))
    s = bench.allreduce_sum(w, 1.0)
    q.put((f"rank{r}", first, t, s, [bench.step_rows(k, w, 0, B) for k in range(3)]))
    import torch.distributed as dist
    dist.destroy_process_group()


def test_two_rank_sharding_and_gather():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((x[0], x[1:]) for x in [q.get(timeout=120) for _ in range(2)])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    f0, t0, s0, blk = res["rank0"]
    f1, t1, s1, _ = res["rank1"]
    rows = sorted(r + i for r in f0 + f1 for i in range(5))
    assert rows == list(range(30))  # 3 steps x 2 ranks x 5 rows: a partition
    assert t0 == t1 == 11.0 and s0 == s1 == 2.0
    # step k's rows of all ranks are one contiguous block starting at rank 0's first row
    for k in range(3):
        assert sorted(list(range(f0[k], f0[k] + 5)) + list(range(f1[k], f1[k] + 5))) == list(range(blk[k], blk[k] + 10))
