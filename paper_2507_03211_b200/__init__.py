"""paper_2507_03211_b200: the DistZO2 zeroth-order training step, B200-native.

Drop-in for the hot path of the reference package ``zosim``: the same
function names and error classes, with parameters resident on a B200 and
every op running in hand-written sm_100a kernels (libzo_b200.so, C ABI in
include/zo_b200.h).  See DESIGN.md.
"""

from .errors import (ConfigurationError, ConsistencyError, CudaError, DimensionError, FabricFault,  # noqa: F401
                     MemoryCapacityError, NumericError, ProtocolError, SimulationError, ZosimError)
from .model import (Batch, ModelConfig, block_tensor_spec, make_batch, model_layout, opt_config,  # noqa: F401
                    OPT_SHAPES)
from .rng import PhiloxKey, RngStateManager, iteration_seeds  # noqa: F401

__version__ = "0.1.0"


_LAZY = {"ZoHyper": "zo", "ZoStep": "zo", "zo_grad": "zo", "mezo_step": "zo", "StreamingZo": "zo",
         "dual_forward": "zo", "flush_pending_update": "zo", "perturb_block": "zo", "perturb_params": "zo",
         "update_block": "zo", "update_params": "zo", "forward_block": "zo", "forward": "zo", "loss": "zo",
         "DeviceStore": "engine", "init_model": "engine"}


def __getattr__(name):
    # GPU-side symbols load lazily so the package imports on a CPU-only host
    mod = _LAZY.get(name)
    if mod is None:
        raise AttributeError(name)
    import importlib

    return getattr(importlib.import_module(f".{mod}", __name__), name)
