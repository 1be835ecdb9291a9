"""Multi-process host logic of the N-GPU path on CPU (gloo, world size 2): row-range sharding is a
partition with no overlap, max-over-ranks timing, and the final output-column gather - the only
cross-rank exchange of the job."""
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
    ids = np.full((B, 8), r, np.int32)
    ln = np.full(B, 8 - r, np.int32)
    g = bench.gather_token_column(w, r, ids, ln)
    if r == 0:
        q.put(("rank0", first, t, s, g[0].tolist(), g[1].tolist()))
    else:
        q.put(("rank1", first, t, s, None, None))
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
    f0, t0, s0, ids, lens = res["rank0"]
    f1, t1, s1, _, _ = res["rank1"]
    rows = sorted(r + i for r in f0 + f1 for i in range(5))
    assert rows == list(range(30))  # 3 steps x 2 ranks x 5 rows: a partition
    assert t0 == t1 == 11.0 and s0 == s1 == 2.0
    assert ids == [[0] * 8] * 5 + [[1] * 8] * 5 and lens == [8] * 5 + [7] * 5
