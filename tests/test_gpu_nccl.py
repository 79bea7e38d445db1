"""The NCCL branches of the fabric on the GPU box's one GPU (world_size 1):
the rank-ordered loss all-gather (all_gather_into_tensor) inside a captured
CUDA graph of the lazy mesh step, and the sliced offload runtime over an NCCL
fabric, both against the single-GPU paths bit for bit.  (Two NCCL ranks need
two GPUs -- NCCL refuses a duplicate device -- so the point-to-point exchange
is covered by the gloo tests with the same bookkeeping.)"""

import pytest

pytestmark = pytest.mark.gpu


def test_nccl_world1_mesh_graph_and_sliced_offload():
    from tests import dist_helpers as H

    res = H.run(H.nccl_world1_worker, 1)
    out = res[0][1]
    assert out["backend"] == "nccl"
    assert out["mesh_graph"] and out["mesh_same"]
    assert out["offload_same"]
    assert {"h2d", "d2h", "compute"} <= set(out["phases"])
