"""ZOPK checkpoints (src/zosim/model.py:375-425).

The golden fixtures hold the bytes the REAL reference's ``save_checkpoint``
wrote for each case's trained store (tests/golden/make_golden.py).  CPU tests
pin the host-side reader / writer to those bytes; GPU tests round-trip the
device and pinned-host masters through the same files.
"""

import os

import numpy as np
import pytest

from paper_2507_03211_b200 import checkpoint as CK
from paper_2507_03211_b200.errors import ConfigurationError, ProtocolError
from paper_2507_03211_b200.model import ModelConfig

CASES = ["tiny32", "tiny64", "ragged32", "mid32", "wide32"]


def _case(golden, name):
    return next(c for c in golden["_meta"]["cases"] if c["name"] == name)


def _cfg(c):
    return ModelConfig(c["vocab"], c["d"], c["heads"], c["n_blocks"], c["seq"], c["dtype"])


def _final(golden, c):
    return [golden[f"{c['name']}/final/{b}"] for b in range(c["n_blocks"] + 2)]


@pytest.mark.parametrize("name", CASES)
def test_reader_matches_reference_file(golden, name, tmp_path):
    c = _case(golden, name)
    p = tmp_path / "ref.zopk"
    p.write_bytes(golden[f"{name}/ckpt"].tobytes())
    cfg, seed, blocks = CK.read_zopk_blocks(p)
    assert cfg == _cfg(c) and seed == 7
    for got, want in zip(blocks, _final(golden, c)):
        assert got.dtype == want.dtype and np.array_equal(got, want)


@pytest.mark.parametrize("name", ["tiny32", "ragged32", "mid32", "wide32"])
def test_writer_is_byte_identical_f32(golden, name, tmp_path):
    c = _case(golden, name)
    flat = np.concatenate(_final(golden, c))
    p = tmp_path / "ours.zopk"
    CK.write_zopk(p, _cfg(c), 7, lambda k, n: flat[k:k + n])
    assert p.read_bytes() == golden[f"{name}/ckpt"].tobytes()


def test_writer_f64_header_identical_values_widened(golden, tmp_path):
    """An f64 config: our master is fp32, so the header is identical and the
    values are the fp32 master widened exactly."""
    c = _case(golden, "tiny64")
    ref = golden["tiny64/ckpt"].tobytes()
    flat = np.concatenate(_final(golden, c)).astype(np.float32)
    p = tmp_path / "ours.zopk"
    CK.write_zopk(p, _cfg(c), 7, lambda k, n: flat[k:k + n])
    got = p.read_bytes()
    hlen = 8 + int.from_bytes(ref[4:8], "little")
    assert got[:hlen] == ref[:hlen] and len(got) == len(ref)
    assert np.array_equal(np.frombuffer(got[hlen:], "<f8"), flat.astype(np.float64))


def test_read_chunked_to_f32(golden, tmp_path):
    p = tmp_path / "ref.zopk"
    p.write_bytes(golden["tiny64/ckpt"].tobytes())
    got = {}
    cfg, _ = CK.read_zopk(p, lambda k, v: got.__setitem__(k, v))
    flat = np.concatenate([got[k] for k in sorted(got)])
    want = np.concatenate(_final(golden, _case(golden, "tiny64"))).astype(np.float32)
    assert cfg.dtype == "f64" and flat.dtype == np.float32 and np.array_equal(flat, want)


def test_bad_magic_and_mismatch(golden, tmp_path):
    p = tmp_path / "bad.zopk"
    p.write_bytes(b"NOPE" + b"\0" * 16)
    with pytest.raises(ConfigurationError, match="magic"):
        CK.read_zopk_blocks(p)
    raw = bytearray(golden["tiny32/ckpt"].tobytes())
    hlen = int.from_bytes(raw[4:8], "little")
    import json

    hdr = json.loads(raw[8:8 + hlen].decode())
    hdr["blocks"][1]["elem_count"] += 1
    hb = json.dumps(hdr).encode()
    bad = b"ZOPK" + len(hb).to_bytes(4, "little") + hb + bytes(raw[8 + hlen:])
    p.write_bytes(bad)
    with pytest.raises(ConfigurationError, match="elements"):
        CK.read_zopk_blocks(p)
    p.write_bytes(bytes(raw[:-4]))     # truncated value stream
    with pytest.raises(ConfigurationError, match="truncated"):
        CK.read_zopk(p, lambda k, v: None)


def test_refuses_unflushed_master(tmp_path):
    class Deferred:
        unflushed = True

    with pytest.raises(ProtocolError, match="flush"):
        CK.save_checkpoint(Deferred(), os.path.join(tmp_path, "x.zopk"))


# ---------------------------------------------------------------------------- GPU
@pytest.mark.gpu
def test_device_store_roundtrip(golden, tmp_path):
    import torch

    from paper_2507_03211_b200 import zo
    from paper_2507_03211_b200.engine import DeviceStore
    from paper_2507_03211_b200.model import make_batch
    from paper_2507_03211_b200.rng import iteration_seeds

    c = _case(golden, "mid32")
    # the reference's file loads into a device master bit-exactly
    ref = tmp_path / "ref.zopk"
    ref.write_bytes(golden["mid32/ckpt"].tobytes())
    st = CK.load_checkpoint(ref, device="cuda:0")
    assert np.array_equal(st.theta.cpu().numpy(), np.concatenate(_final(golden, c)))
    # ... and writes back byte-identically
    out = tmp_path / "out.zopk"
    CK.save_checkpoint(st, out)
    assert out.read_bytes() == ref.read_bytes()
    # a lazy runner must flush before checkpointing; after flush the file
    # holds exactly the device master
    store = DeviceStore(_cfg(c), init_seed=7, device="cuda:0")
    sz = zo.StreamingZo(store, zo.ZoHyper(1e-3, 1e-2))
    for j, s in enumerate(iteration_seeds(3, 2), 1):
        sz.step(make_batch(store.config, 2, 50 + j), s)
    with pytest.raises(ProtocolError):
        CK.save_checkpoint(store, out)
    sz.flush()
    CK.save_checkpoint(store, out)
    _, _, blocks = CK.read_zopk_blocks(out)
    assert np.array_equal(np.concatenate(blocks), store.theta.cpu().numpy())
    back = CK.load_checkpoint(out, device="cuda:0")
    assert torch.equal(back.theta, store.theta) and back.checksum() == store.checksum()


@pytest.mark.gpu
def test_host_store_roundtrip(golden, tmp_path):
    c = _case(golden, "wide32")
    ref = tmp_path / "ref.zopk"
    ref.write_bytes(golden["wide32/ckpt"].tobytes())
    hs = CK.load_checkpoint(ref, host=True)
    assert hs.theta.is_pinned()
    assert np.array_equal(hs.theta.numpy(), np.concatenate(_final(golden, c)))
    out = tmp_path / "out.zopk"
    CK.save_checkpoint(hs, out)
    assert out.read_bytes() == ref.read_bytes()
