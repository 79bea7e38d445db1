"""Multi-process (gloo, CPU) tests of the distributed host logic: ordered
collectives (fabric.py:90-113) and the loss-gather layout every strategy's
device reduction reads (strategies.py:145-147, 197-216)."""

import pytest

from oracle import zo_oracle as O
from tests import dist_helpers as H


@pytest.mark.parametrize("world", [2, 4])
def test_fabric_ordered_collectives_and_mesh_layout(world):
    res = H.run(H.fabric_worker, world)
    outs = [r[1] for r in res]
    vals = [0.1, 0.2, 0.3, 1e16, -1e16, 0.7, 0.9, 1.1][:world]
    for o in outs:
        assert o["gather"] == [10.0 + r for r in range(world)]
        assert o["bcast"] == 42
        assert o["mean"] == O.ordered_mean(vals)            # ascending-rank order, bit-exact
    # every rank derives the same g, equal to the oracle's ordered reduction
    eps = 1e-3
    ddp = [O.zo_grad(2.0 + 0.01 * r, 2.0 - 0.013 * r, eps) for r in range(world)]
    twod = [O.zo_grad(2.0 + 0.01 * i, 2.0 - 0.013 * i, eps) for i in range(world // 2)]
    for o in outs:
        assert o["ddp"] == O.ordered_mean(ddp)
        assert o["2d"] == O.ordered_mean(twod)
        if world == 2:
            assert o["pertp"] == O.zo_grad(2.0, 2.0, eps) or o["pertp"] == twod[0]
    # only scalar traffic crosses the fabric (strategies.py docstring, test_strategies.py:99-111)
    assert set(outs[0]["bytes"]) <= {"seed", "loss", "grad", "checksum"}


@pytest.mark.parametrize("world", [2, 4])
def test_direction_aware_slice_exchange(world):
    """rank q holds slice k of its own direction's buffer from
    every rank k after the exchange; each rank contributes one bf16 slice."""
    import torch

    w = 5
    res = H.run(H.exchange_worker, world, w)
    for r, out, nbytes in res:
        d = r % 2
        want = [float(torch.tensor(100 * d + k + i / 64).bfloat16()) for k in range(world) for i in range(w)]
        assert out == want
        assert nbytes == {"param": w * 2}


def test_mesh_layout_rejects_bad_meshes():
    from paper_2507_03211_b200.errors import ConfigurationError
    from paper_2507_03211_b200.strategies import MeshLayout, mesh_assignments

    with pytest.raises(ConfigurationError):
        MeshLayout("pertp", 3, 0)
    with pytest.raises(ConfigurationError):
        MeshLayout("2d", 3, 0)
    a = mesh_assignments(2)
    assert [(x.rank, x.group, x.direction) for x in a] == [(0, 0, 1), (1, 0, -1), (2, 1, 1), (3, 1, -1)]
    assert a[3].pair_ranks == (2, 3)
