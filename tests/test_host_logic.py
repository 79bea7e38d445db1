"""CPU tests of the drop-in's host-side logic (no GPU): configuration and
batch validation (model.py:43-274), the RNG manager protocol (rng.py:45-108),
the seed schedule, the status-code -> exception mapping (errors.py), the
T_comm model (comm.py:250-256).  Mirrors pkg/tests/test_model.py,
test_rng.py and test_comm.py where they do not need a device."""

import numpy as np
import pytest

from oracle import zo_oracle as O
from paper_2507_03211_b200 import errors as E
from paper_2507_03211_b200.model import Batch, ModelConfig, block_tensor_spec, make_batch, model_layout, opt_config
from paper_2507_03211_b200.rng import PhiloxKey, RngStateManager, iteration_seeds
from paper_2507_03211_b200.scheduler import sliced_upload_time


def test_config_validation_and_param_count(golden):
    with pytest.raises(E.ConfigurationError):
        ModelConfig(16, 15, 2, 1, 8).validate()          # d % heads
    with pytest.raises(E.ConfigurationError):
        ModelConfig(0, 16, 2, 1, 8).validate()
    with pytest.raises(E.ConfigurationError):
        ModelConfig(16, 16, 2, 1, 8, "bf16").validate()
    for c in golden["_meta"]["cases"]:
        cfg = ModelConfig(c["vocab"], c["d"], c["heads"], c["n_blocks"], c["seq"], c["dtype"])
        assert cfg.param_count() == O.param_count(c["vocab"], c["d"], c["n_blocks"], c["seq"])
        lays = model_layout(cfg)
        assert sum(b.elem_count for b in lays) == cfg.param_count()
        assert [b.key0 for b in lays] == list(np.cumsum([0] + [b.elem_count for b in lays[:-1]]))
    # the shape sheet of SURVEY section 8
    assert opt_config("opt-125m", 64).param_count() == 162_373_216
    assert opt_config("opt-1.3b", 512).param_count() == 1_415_615_584
    assert opt_config("opt-175b", 2048).param_count() == 175_222_236_256


def test_tensor_spec_matches_oracle():
    cfg = ModelConfig(50, 24, 4, 2, 12)
    for kind in ("embedding", "transformer", "head"):
        assert block_tensor_spec(cfg, kind) == O.tensor_spec(50, 24, 12, kind)


def test_batches_match_reference_and_validate(golden):
    cfg = ModelConfig(16, 16, 2, 2, 8, "f32")
    b = make_batch(cfg, 4, 101)
    assert np.array_equal(b.token_ids, golden["tiny32/ids/1"])
    assert np.array_equal(b.targets, golden["tiny32/tgt/1"])
    with pytest.raises(E.DimensionError):
        Batch(np.zeros((2, 3), dtype=np.int64), np.zeros((2, 4), dtype=np.int64))
    with pytest.raises(E.ConfigurationError):
        Batch(np.full((2, 8), 99), np.zeros((2, 8), dtype=np.int64)).validate(cfg)
    shards = [b.shard(2, r) for r in range(2)]
    assert np.array_equal(np.concatenate([s.token_ids for s in shards]), b.token_ids)
    with pytest.raises(E.ConfigurationError):
        b.shard(3, 0)


def test_iteration_seeds_match_reference(golden):
    assert iteration_seeds(1234, 8) == [int(s) for s in golden["kat/iteration_seeds_1234"]]
    s = iteration_seeds(7, 50)
    assert len(set(s)) == 50 and all(0 <= x < 2**63 for x in s)


def test_rng_manager_oracle_protocol_matches_reference_semantics():
    m = RngStateManager("oracle")
    m.reset(3)
    a = m.normal(3, 10)
    m.reset(3)
    st = m.capture(3)
    b = m.normal(3, 10)
    m.restore(3, st)
    c = m.normal(3, 10)
    assert np.array_equal(a, b) and np.array_equal(b, c)
    # chunked draws == one draw (rng.py:29-36)
    m.reset(5)
    whole = m.normal(5, 100)
    m.reset(5)
    parts = np.concatenate([m.normal(5, 30), m.normal(5, 70)])
    assert np.array_equal(whole, parts)
    # FIFO depth 2 and underflow
    m.push_state(1)
    m.push_state(2)
    with pytest.raises(E.ProtocolError):
        m.push_state(3)
    assert m.pop_state() == 1 and m.pop_state() == 2
    with pytest.raises(E.ProtocolError):
        m.pop_state()


def test_rng_manager_philox_keys_install_like_states():
    m = RngStateManager()
    assert isinstance(m.generator(11), PhiloxKey) and m.generator(11).seed == 11
    st = m.capture(11)
    m.restore(99, st)                 # a state captured under one seed installed under another
    assert m.generator(99).seed == 11
    m.reset(99)
    assert m.generator(99).seed == 99
    with pytest.raises(E.ProtocolError):
        m.normal(11, 3)


def test_status_codes_map_to_reference_exceptions():
    for code, cls in ((1, E.ProtocolError), (2, E.ConfigurationError), (3, E.NumericError),
                      (4, E.FabricFault), (5, E.CudaError)):
        with pytest.raises(cls):
            E.raise_for(code, "x")
    E.raise_for(0, "ok")
    assert E.ConfigurationError.exit_code == 2 and E.NumericError.exit_code == 3
    assert issubclass(E.ConsistencyError, E.FabricFault) and issubclass(E.DimensionError, E.ConfigurationError)


def test_tcomm_model_matches_reference(golden):
    for m, n, t in golden["comm/tcomm"]:
        assert sliced_upload_time(int(m), int(n), 4e8, 2.4e9) == t
