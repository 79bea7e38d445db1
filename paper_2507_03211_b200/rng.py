"""Direction sources and the seed schedule (mirror of src/zosim/rng.py).

Production: the direction z of iteration j is Philox4x32-10(seed_j, key)
+ Box-Muller, generated in registers by every kernel that needs it
(csrc/common.cuh).  It is a pure function of (seed, global element key):
no generator state, no capture/restore, bit-identical on every rank and
for every slicing of a block -- the properties zosim obtains by
capturing/restoring PCG64 states (rng.py:1-13, 45-108).

Oracle mode: ``RngStateManager(mode="oracle")`` draws the reference's own
stream, ``numpy.random.Generator(PCG64(seed)).standard_normal``, in the
reference's (block, tensor, element) order and injects it into the same
kernels (ZO_Z_ORACLE) -- this is how parity with the CPU reference is
proven bit-for-bit on the perturb/update arithmetic.
"""

from __future__ import annotations

from collections import deque

import numpy as np

from .errors import ProtocolError

FIFO_MAX_DEPTH = 2   # rng.py:27


def iteration_seeds(base_seed: int, steps: int) -> list:
    """Per-iteration seed schedule, identical to rng.py:35-42, so every rank
    derives it locally from the base seed."""
    gen = np.random.Generator(np.random.PCG64(np.random.SeedSequence([int(base_seed), 0x5EED])))
    return [int(s) for s in gen.integers(0, 2**63 - 1, size=steps)]


class PhiloxKey:
    """Stateless direction key: z(e) = philox_normal(seed, e)."""

    __slots__ = ("seed",)

    def __init__(self, seed: int):
        self.seed = int(seed)

    def __repr__(self):
        return f"PhiloxKey({self.seed})"


class RngStateManager:
    """API-compatible stand-in for zosim's RngStateManager (rng.py:45-108).

    mode="philox": ``generator(seed)`` returns a PhiloxKey; capture/restore
    are identities (the stream has no position).  mode="oracle": the numpy
    PCG64 generators of the reference, with exact capture/restore.
    """

    def __init__(self, mode: str = "philox"):
        if mode not in ("philox", "oracle"):
            raise ProtocolError(f"unknown rng mode {mode!r}")
        self.mode = mode
        self._gens: dict = {}
        self._installed: dict = {}   # philox: key -> seed of a restored state
        self.state_fifo: deque = deque()
        self.prev_state = None

    @property
    def oracle(self) -> bool:
        return self.mode == "oracle"

    def reset(self, seed: int) -> None:
        if self.oracle:
            self._gens[seed] = np.random.Generator(np.random.PCG64(seed))
        else:
            self._installed.pop(seed, None)

    def generator(self, seed: int):
        if not self.oracle:
            return PhiloxKey(self._installed.get(seed, seed))
        if seed not in self._gens:
            self.reset(seed)
        return self._gens[seed]

    def capture(self, seed: int):
        if not self.oracle:
            return ("philox", int(self._installed.get(seed, seed)))
        import copy

        return copy.deepcopy(self.generator(seed).bit_generator.state)

    def restore(self, seed: int, state) -> None:
        """A state captured under one seed may be installed under another
        (rng.py:70-77); for Philox the 'state' is just the key."""
        if not self.oracle:
            self._installed[seed] = int(state[1])
            return
        if self.oracle:
            import copy

            self.generator(seed).bit_generator.state = copy.deepcopy(state)

    def normal(self, seed: int, n: int) -> np.ndarray:
        if not self.oracle:
            raise ProtocolError("normal() draws host z; only available in oracle mode")
        return self.generator(seed).standard_normal(n)

    def push_state(self, state) -> None:
        if len(self.state_fifo) >= FIFO_MAX_DEPTH:
            raise ProtocolError(f"state FIFO is full (depth {len(self.state_fifo)})")
        self.state_fifo.append(state)

    def pop_state(self):
        if not self.state_fifo:
            raise ProtocolError("state FIFO is empty; no pending iteration state to consume")
        self.prev_state = self.state_fifo.popleft()
        return self.prev_state

    @property
    def fifo_depth(self) -> int:
        return len(self.state_fifo)
