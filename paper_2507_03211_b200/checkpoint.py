"""ZOPK parameter checkpoints (src/zosim/model.py:375-425).

Wire format, byte-compatible with the reference's ``save_checkpoint`` /
``load_checkpoint``:

    b"ZOPK" | u32 LE header length | UTF-8 JSON header | block values

The header is ``{"config": ModelConfig.to_dict(), "init_seed": int,
"blocks": [{"block_id", "kind", "elem_count", "tensors": [{"name",
"shape"}]}]}`` (model.py:381-393) and the values follow in block order as
little-endian f32 (config dtype "f32") or f64 ("f64") (model.py:376-378).

The B200 build keeps an fp32 master, so an "f64" checkpoint written here holds
the fp32 values widened exactly; reading an "f64" checkpoint narrows each value
to fp32 with round-to-nearest (the only lossy direction, and only for files the
reference wrote in f64).

Checkpoints are taken on a flushed master ("checkpoints always
flush first"): a runner whose last update is still deferred marks its store,
and ``save_checkpoint`` raises ProtocolError until ``flush()`` is called.

The device / pinned-host stores are read and written in 64 Mi-element chunks
through one pinned staging buffer, so a 13B-shape master (52 GB) never needs a
second full host copy.
"""

from __future__ import annotations

import json

import numpy as np

from .errors import ConfigurationError, ProtocolError
from .model import ModelConfig, model_layout

CHECKPOINT_MAGIC = b"ZOPK"          # model.py:31
_CHUNK = 1 << 26


def _wire_dtype(config: ModelConfig) -> np.dtype:
    """model.py:376-378."""
    return np.dtype("<f4" if config.dtype == "f32" else "<f8")


def checkpoint_header(config: ModelConfig, init_seed: int) -> bytes:
    """The JSON header exactly as model.py:381-393 serialises it."""
    header = {
        "config": config.to_dict(),
        "init_seed": init_seed,
        "blocks": [
            {
                "block_id": bl.block_id,
                "kind": bl.kind,
                "elem_count": bl.elem_count,
                "tensors": [{"name": n, "shape": list(bl.shapes[n])} for n in bl.names],
            }
            for bl in model_layout(config)
        ],
    }
    return json.dumps(header).encode("utf-8")


def write_zopk(path, config: ModelConfig, init_seed: int, read_chunk) -> None:
    """Write a checkpoint; ``read_chunk(key, n)`` returns the fp32 master
    values [key, key+n) as a numpy array (keys are the global element order,
    which is the block order of the file)."""
    raw = checkpoint_header(config, init_seed)
    wire = _wire_dtype(config)
    total = sum(bl.elem_count for bl in model_layout(config))
    with open(path, "wb") as f:
        f.write(CHECKPOINT_MAGIC)
        f.write(len(raw).to_bytes(4, "little"))
        f.write(raw)
        for k in range(0, total, _CHUNK):
            n = min(_CHUNK, total - k)
            f.write(np.ascontiguousarray(read_chunk(k, n), dtype=wire).tobytes())


def read_zopk_header(f):
    """Parse magic + header from an open binary file (model.py:407-414)."""
    magic = f.read(4)
    if magic != CHECKPOINT_MAGIC:
        raise ConfigurationError(f"not a checkpoint file: bad magic {magic!r}")
    hlen = int.from_bytes(f.read(4), "little")
    header = json.loads(f.read(hlen).decode("utf-8"))
    config = ModelConfig.from_dict(header["config"])
    layouts = model_layout(config)
    metas = header["blocks"]
    if len(metas) != len(layouts):
        raise ConfigurationError(f"checkpoint has {len(metas)} blocks, model expects {len(layouts)}")
    for bl, meta in zip(layouts, metas):
        if meta["elem_count"] != bl.elem_count:        # model.py:418-422
            raise ConfigurationError(f"block {bl.block_id}: checkpoint has {meta['elem_count']} elements, "
                                     f"model expects {bl.elem_count}")
    return config, header.get("init_seed", 0), layouts


def read_zopk(path, write_chunk) -> tuple[ModelConfig, int]:
    """Read a checkpoint; ``write_chunk(key, values_f32)`` receives the
    master values in key order.  Returns (config, init_seed)."""
    with open(path, "rb") as f:
        config, init_seed, layouts = read_zopk_header(f)
        wire = _wire_dtype(config)
        total = sum(bl.elem_count for bl in layouts)
        for k in range(0, total, _CHUNK):
            n = min(_CHUNK, total - k)
            data = f.read(n * wire.itemsize)
            if len(data) != n * wire.itemsize:
                raise ConfigurationError(f"checkpoint truncated at element {k}")
            write_chunk(k, np.frombuffer(data, dtype=wire).astype(np.float32))
    return config, init_seed


def read_zopk_blocks(path) -> tuple[ModelConfig, int, list]:
    """Host-only reader: (config, init_seed, [block values in the file's
    wire dtype]) -- the reference's ParamStore contents, for tests/tools."""
    with open(path, "rb") as f:
        config, init_seed, layouts = read_zopk_header(f)
        wire = _wire_dtype(config)
        blocks = [np.frombuffer(f.read(bl.elem_count * wire.itemsize), dtype=wire).copy() for bl in layouts]
    return config, init_seed, blocks


def _check_flushed(store) -> None:
    if getattr(store, "unflushed", False):
        raise ProtocolError("checkpoint of a master with a deferred update: call flush() first (SPEC.md:192)")


def save_checkpoint(store, path) -> None:
    """Write a DeviceStore / HostStore (or anything with ``config``,
    ``init_seed`` and an fp32 ``theta`` tensor in key order) as ZOPK."""
    import torch

    _check_flushed(store)
    theta = store.theta
    if theta.is_cuda:
        stage = torch.empty(min(_CHUNK, theta.numel()), dtype=torch.float32, pin_memory=True)

        def read_chunk(k, n):
            stage[:n].copy_(theta[k:k + n])       # synchronous D2H into the pinned stage
            return stage[:n].numpy()
    else:
        def read_chunk(k, n):
            return theta[k:k + n].numpy()
    write_zopk(path, store.config, int(store.init_seed), read_chunk)


def load_checkpoint(path, device=None, host: bool = False, directions=None):
    """Read a ZOPK file into a new DeviceStore on ``device`` (or, with
    ``host=True``, a pinned HostStore for the offload runtime).  The
    reference re-runs init_model before overwriting (model.py:415); here the
    master is allocated uninitialised and filled from the file."""
    import torch

    with open(path, "rb") as f:
        config, init_seed, _ = read_zopk_header(f)
    if host:
        from .scheduler import HostStore

        store = HostStore(config, init_seed=init_seed, init="none")
    else:
        from .engine import MINUS, PLUS, DeviceStore

        store = DeviceStore(config, init_seed=init_seed, device=device, init="none",
                            directions=directions or (PLUS, MINUS))
    theta = store.theta
    stage = torch.empty(min(_CHUNK, theta.numel()), dtype=torch.float32, pin_memory=theta.is_cuda)

    def write_chunk(k, vals):
        stage[:len(vals)].copy_(torch.from_numpy(vals))
        theta[k:k + len(vals)].copy_(stage[:len(vals)])

    read_zopk(path, write_chunk)
    if theta.is_cuda:
        torch.cuda.current_stream().synchronize()
    return store
