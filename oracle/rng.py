"""Counter-based splitmix64 stream (TEST INFRASTRUCTURE ONLY).

Restates reference tensor.py:28-82: `mix64` (tensor.py:28-38), the vectorised
finalizer (tensor.py:41-48) and `SeededRng.uniform` (tensor.py:63-70), i.e.
u(seed, pos) = (fmix(seed + (pos+1)*GOLDEN) >> 11) * 2^-53.
"""

import numpy as np

M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
C1 = 0xBF58476D1CE4E5B9
C2 = 0x94D049BB133111EB


def fmix(h):
    """splitmix64 finalizer on a python int (tensor.py:33-37)."""
    h ^= h >> 30
    h = (h * C1) & M64
    h ^= h >> 27
    h = (h * C2) & M64
    h ^= h >> 31
    return h


def hash64(*words):
    """Fold integers into one 64-bit value (tensor.py:28-38)."""
    acc = 0
    for w in words:
        acc = fmix((acc + (int(w) & M64) * GOLDEN) & M64)
    return acc


def bits53(seed, start, count):
    """The 53-bit integers behind positions [start, start+count)."""
    pos = np.arange(start, start + count, dtype=np.uint64) + np.uint64(1)
    with np.errstate(over="ignore"):
        x = np.uint64(seed & M64) + pos * np.uint64(GOLDEN)
        x ^= x >> np.uint64(30)
        x *= np.uint64(C1)
        x ^= x >> np.uint64(27)
        x *= np.uint64(C2)
        x ^= x >> np.uint64(31)
    return x >> np.uint64(11)


def uniform(seed, start, shape):
    """Uniform [0,1) draws of a stream window (tensor.py:63-70)."""
    n = int(np.prod(shape, dtype=np.int64)) if shape else 1
    return (bits53(seed, start, n) * (1.0 / (1 << 53))).reshape(shape)


def keep_threshold(p):
    """Integer form of `u >= p`: bits53 >= ceil(p * 2^53) (exact)."""
    import math

    return int(math.ceil(p * float(1 << 53)))


def dropout_scale_mask(seed, start, shape, p):
    """The reference's dropout multiplier (layers.py:57-59)."""
    u = uniform(seed, start, shape)
    return (u >= p).astype(np.float64) * (1.0 / (1.0 - p))


class Stream:
    """Positioned stream object with the reference SeededRng surface
    (tensor.py:51-82): uniform / uniform_signed / at / derive."""

    def __init__(self, seed, position=0):
        self.seed = seed
        self.position = position

    def uniform(self, shape):
        out = uniform(self.seed, self.position, shape)
        self.position += int(np.prod(shape, dtype=np.int64)) if shape else 1
        return out

    def uniform_signed(self, shape, scale):
        return (self.uniform(shape) * 2.0 - 1.0) * scale

    def at(self, position):
        return Stream(self.seed, position)

    def derive(self, *tags):
        return Stream(hash64(self.seed, *tags))
