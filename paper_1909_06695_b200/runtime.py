"""Per-device runtime: library load, device check and the status word.

Kernels OR status bits (RP_FLAG_*) into one device int32 instead of raising
at every layer output like the reference's check_finite (tensor.py:93-96);
the host reads it once per step (the loss read-back is the step's sync
point anyway) and raises the reference's exception class.
"""

import torch

from . import _native as N
from .errors import DimensionError, NonFiniteError


class Runtime:
    _by_device = {}

    def __init__(self, device):
        if device.type != "cuda":
            raise RuntimeError("ringpipe-b200 runs on CUDA devices only (no CPU fallback)")
        N.lib()  # raises ImportError when the extension is missing
        if not torch.cuda.is_available():
            raise RuntimeError("CUDA is not available: the B200 path has no CPU fallback")
        major, minor = torch.cuda.get_device_capability(device)
        if major != 10:
            raise RuntimeError(f"libringpipe_b200 is built for sm_100a; device is sm_{major}{minor}")
        self.device = device
        self.flag = torch.zeros(1, dtype=torch.int32, device=device)
        self._host = torch.zeros(1, dtype=torch.int32).pin_memory()

    @classmethod
    def get(cls, device=None):
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device())
        device = torch.device(device)
        if device.type == "cuda" and device.index is None:
            device = torch.device("cuda", torch.cuda.current_device())
        rt = cls._by_device.get(device)
        if rt is None:
            rt = cls(device)
            cls._by_device[device] = rt
        return rt

    def check(self, context="step", modules=()):
        """Synchronously read and clear the status words (the optimizer's and
        each module's); raise the reference exception naming the culprit."""
        words = [m.flag for m in modules] + [self.flag]
        host = torch.cat([w.view(1) for w in words]).cpu()
        bad = [(i, int(b)) for i, b in enumerate(host.tolist()) if b]
        if not bad:
            return
        for w in words:
            w.zero_()
        i, bits = bad[0]
        where = f"module {modules[i].index}" if i < len(modules) else "optimizer update"
        if bits & N.FLAG_DIMENSION:
            raise DimensionError(f"token or target id out of range in {where} ({context})")
        raise NonFiniteError(f"non-finite values in {where} ({context})")
