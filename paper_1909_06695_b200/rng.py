"""Host side of the counter-based splitmix64 stream.

The stream itself (seed, position) -> 53-bit uniform is evaluated on the
device (csrc/common.cuh `rng_bits53`, used by dropout epilogues and
`rp_init_uniform`).  The host only folds integers into seeds
(reference tensor.py:28-38: layer seeds mix64(dropout_seed, step, layer),
model.py:218-219, and the init stream seed mix64(init_seed), model.py:54) and
provides a small numpy `SeededRng` for callers that build batches the
reference way (tests/test_engine.py:26-33).
"""

import math

import numpy as np

_MASK = (1 << 64) - 1
_PHI = 0x9E3779B97F4A7C15


def _fmix(z):
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK
    return z ^ (z >> 31)


def mix64(*parts):
    """Fold integers into one well-mixed 64-bit value."""
    h = 0
    for part in parts:
        h = _fmix((h + (int(part) & _MASK) * _PHI) & _MASK)
    return h


def keep_threshold(p):
    """Dropout keeps an element iff bits53 >= ceil(p * 2^53), exactly the
    reference's float test u >= p with u = bits53 * 2^-53."""
    return int(math.ceil(float(p) * 9007199254740992.0))


class SeededRng:
    """Host uniform stream with the reference's (seed, position) surface."""

    def __init__(self, seed, position=0):
        self.seed = int(seed)
        self.position = int(position)

    def uniform(self, shape):
        count = int(np.prod(shape, dtype=np.int64)) if shape else 1
        ctr = np.arange(self.position + 1, self.position + 1 + count, dtype=np.uint64)
        with np.errstate(over="ignore"):
            z = np.uint64(self.seed & _MASK) + ctr * np.uint64(_PHI)
            z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
            z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
            z = z ^ (z >> np.uint64(31))
        self.position += count
        return ((z >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)).reshape(shape)

    def uniform_signed(self, shape, scale):
        return (self.uniform(shape) * 2.0 - 1.0) * scale

    def at(self, position):
        return SeededRng(self.seed, position)

    def derive(self, *tags):
        return SeededRng(mix64(self.seed, *tags))
