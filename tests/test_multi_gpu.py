"""One context over several devices (iolm_cuda_create_multi): the multi-GPU deployment of SURVEY §8e
behind the same batch_decode surface. On this 1-GPU box the device list repeats device 0 (two or
three engines with their own replicas and KV pools on one GPU), which exercises the partition, the
concurrent per-device host threads and the direct writes into the caller's output column.

Outputs must equal a one-device context's BIT FOR BIT (batch invariance, runtime.hpp:57-60), madds
must be the one-device sum, SequenceTooLong must name the batch's first offending row, and a bad
token id anywhere must raise ContractViolation."""
import numpy as np
import pytest

from paper_2507_04967_b200 import runtime as R
from paper_2507_04967_b200 import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rts():
    b = synth.toy_bundle(128, 4, 4, 512, 160, seed=42)
    one = R.ModelRuntime(b)
    two = R.ModelRuntime(b, device=[0, 0])
    three = R.ModelRuntime(b, device=[0, 0, 0], max_tokens_per_step=512, max_slots=16)
    yield b, one, two, three
    for r in (one, two, three):
        r.close()


def test_device_count(rts):
    _, one, two, three = rts
    assert (one.device_count(), two.device_count(), three.device_count()) == (1, 2, 3)


@pytest.mark.parametrize("n_rows,budget", [(1, 8), (2, 3), (5, 8), (333, 8), (2000, 4)])
def test_multi_device_bit_identical(rts, n_rows, budget):
    _, one, two, three = rts
    ids, offs = synth.rows(7, n_rows, 64)
    # ragged rows: cut every third row short
    lens = np.diff(offs)
    lens[::3] = np.maximum(1, lens[::3] // 3)
    rows = [ids[offs[i]:offs[i] + lens[i]] for i in range(n_rows)]
    ids = np.concatenate(rows).astype(np.int32)
    offs = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    a, la, ma = one.decode_token_rows(ids, offs, budget)
    for rt in (two, three):
        b_, lb, mb = rt.decode_token_rows(ids, offs, budget)
        assert np.array_equal(la, lb) and ma == mb
        for i in range(n_rows):
            assert np.array_equal(a[i, :la[i]], b_[i, :lb[i]]), i
        st = rt.last_stats()
        assert st["kernel_launches"] > 0 and st["decode_tokens"] + st["prefill_tokens"] + st["prefix_tokens"] > 0


def test_multi_device_batch_decode_strings(rts):
    _, one, two, _ = rts
    prompts = synth.row_strings(100, 64, 64) + ["", "x", "PAD and BOS render nothing"]
    c1, c2 = R.FlopCounter(), R.FlopCounter()
    assert one.batch_decode(prompts, 8, c1) == two.batch_decode(prompts, 8, c2)
    assert c1.total() == c2.total()


def test_multi_device_errors(rts):
    _, one, two, three = rts
    ids, offs = synth.rows(0, 40, 64)
    # a too-long row late in the batch: the first offending row is reported whichever device owns it
    rows = [ids[offs[i]:offs[i + 1]] for i in range(40)]
    rows[29] = np.concatenate([rows[29], np.full(200, 65, np.int32)])
    rows[35] = np.concatenate([rows[35], np.full(300, 65, np.int32)])
    big = np.concatenate(rows).astype(np.int32)
    boffs = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.int64)
    for rt in (one, two, three):
        with pytest.raises(R.SequenceTooLong, match="prompt 29 "):
            rt.decode_token_rows(big, boffs, 8)
    bad = ids.copy()
    bad[offs[33] + 5] = 131  # out-of-range id on the last device's range
    for rt in (one, two, three):
        with pytest.raises(R.ContractViolation):
            rt.decode_token_rows(bad, offs, 8)
    # the context still works after a failed call on one of its devices
    a, la, _ = one.decode_token_rows(ids, offs, 8)
    b_, lb, _ = three.decode_token_rows(ids, offs, 8)
    assert np.array_equal(la, lb) and all(np.array_equal(a[i, :la[i]], b_[i, :lb[i]]) for i in range(40))


def test_multi_device_forward_on_first_device(rts):
    _, one, two, _ = rts
    ids, offs = synth.rows(3, 1, 64)
    assert np.array_equal(one.forward(ids), two.forward(ids))


def test_device_resident_ids_single_device_only(rts):
    import torch
    _, _, two, _ = rts
    ids, offs = synth.rows(0, 4, 64)
    d = torch.from_numpy(ids).cuda()
    with pytest.raises(R.UnsupportedOnGpu):
        two.decode_token_rows(None, offs, 8, device_ids=d.data_ptr())
