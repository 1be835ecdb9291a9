"""Device-layout images (iolm_cuda_save_image / iolm_cuda_create_from_image).

An image is the pre-tiled cache a registry keeps next to a bundle (ModelRegistry::store/lookup,
proj/src/optimize.cpp:139-160): the weights in this engine's HBM layout, the config and the bundle
hash. The bar is bit-identity: a runtime loaded from an image must produce exactly the ids, lengths,
FlopCounter totals and logits of the runtime built from the bundle, in every weight form the engine
has (fp16 values, W8A16 codes, W8A8 int8, 2:4 sparse int8, packed int4), on pruned shapes. The
failure modes map to the reference's: bad magic / checksum -> CorruptHeader, short file ->
TruncatedBlob; another bundle or other weight options -> StaleImage (rebuild from the bundle)."""
import numpy as np
import pytest

from paper_2507_04967_b200 import runtime as R
from paper_2507_04967_b200 import synth

pytestmark = pytest.mark.gpu

# (quant, runtime options, expected weight forms)
CASES = [
    ("dense", {}, {"values"}),
    ("q8", {}, {"codes"}),
    ("q8", {"act_quant": True}, {"int8"}),
    ("sparse24", {"act_quant": True}, {"sp24"}),
    ("sparse24", {"act_quant": True, "sparse_mma": False}, {"int8"}),
    ("q4", {}, {"int4"}),
    ("q4", {"int4_mma": False}, {"codes"}),
]


def _same_outputs(a, b, n=24, max_new=8):
    ids, offs = synth.rows(300, n, 64)
    ai, al, am = a.decode_token_rows(ids, offs, max_new)
    bi, bl, bm = b.decode_token_rows(ids, offs, max_new)
    assert am == bm
    assert np.array_equal(al, bl)
    assert np.array_equal(ai, bi)
    seq = ids[offs[0]:offs[1]]
    assert np.array_equal(a.forward(seq), b.forward(seq))


@pytest.mark.parametrize("quant,opts,forms", CASES, ids=[f"{q}-{'-'.join(o) or 'default'}" for q, o, _ in CASES])
def test_image_roundtrip_bit_identical(tmp_path, quant, opts, forms):
    b = synth.toy_bundle(128, 3, 4, 512, 160, seed=7, quant=quant, heads=[4, 2, 3], ffn=[512, 256, 384])
    path = tmp_path / "m.iolmdev"
    with R.ModelRuntime(b, **opts) as rt:
        rt.save_image(path)
        hdr = R.image_header(path)
        assert hdr["bundle_hash"] == rt.bundle_hash() == synth.fnv1a(b)
        assert set(hdr["weight_forms"]) == forms
        assert hdr["config"] == R.bundle_config(b)
        with R.ModelRuntime.from_image(path, expected_hash=synth.fnv1a(b), **opts) as im:
            assert im.bundle_hash() == rt.bundle_hash()
            assert im.config() == rt.config()
            _same_outputs(rt, im)


def test_image_engine_options_may_differ(tmp_path):
    """Token budget / prefix sharing are engine-only options: outputs stay bit-identical (batch
    invariance, test_model.cpp:240-267)."""
    b = synth.toy_bundle(128, 2, 4, 512, 160, seed=9, quant="dense")
    path = tmp_path / "m.iolmdev"
    with R.ModelRuntime(b) as rt:
        rt.save_image(path)
        with R.ModelRuntime.from_image(path, max_tokens_per_step=256, prefix_sharing=False) as im:
            _same_outputs(rt, im)


def test_image_errors(tmp_path):
    b = synth.toy_bundle(128, 2, 4, 512, 160, seed=11, quant="q8")
    path = tmp_path / "m.iolmdev"
    with R.ModelRuntime(b) as rt:
        rt.save_image(path)
    h = synth.fnv1a(b)
    with pytest.raises(R.StaleImage):
        R.ModelRuntime.from_image(path, expected_hash=h ^ 1)
    with pytest.raises(R.StaleImage):
        R.ModelRuntime.from_image(path, expected_hash=h, act_quant=True)
    with pytest.raises(R.StaleImage):
        R.ModelRuntime.from_image(path, expected_hash=h, int4_mma=False)  # q8 codes: int4 flag still recorded
    data = path.read_bytes()
    short = tmp_path / "short.iolmdev"
    short.write_bytes(data[:len(data) // 2])
    with pytest.raises(R.TruncatedBlob):
        R.ModelRuntime.from_image(short, expected_hash=h)
    flipped = bytearray(data)
    flipped[len(data) // 2] ^= 0x10
    bad = tmp_path / "bad.iolmdev"
    bad.write_bytes(bytes(flipped))
    with pytest.raises(R.CorruptHeader, match="checksum"):
        R.ModelRuntime.from_image(bad, expected_hash=h)
    with pytest.raises(R.ContractViolation):
        R.ModelRuntime.from_image(tmp_path / "missing.iolmdev")
    # a good image still loads after the failures (no leaked state)
    with R.ModelRuntime.from_image(path, expected_hash=h) as im:
        assert im.bundle_hash() == h
