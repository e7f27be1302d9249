"""RPCK checkpoint container: named arrays plus a JSON sidecar.

Byte-compatible with the reference container (checkpoint.py:1-70).  The
reference's checkpoints load here (runner.load_training_state re-derives the
pending slots from the reference's ring, including its snapshots of V).  The
other direction is one-way by design: this package keeps no snapshots of the
tied matrix (module 1's slots carry their embedding output instead, entry
`m1.slot{j}.embedded`), so its checkpoints lack the reference's
`m{k}.ring.{s}.L{i}.tied` entries and the reference loader, which requires
them (reference runner.py:186-195), cannot read them.  The container layout:

    "RPCK" | u32 version=1 | u32 count |
    count x ( u16 name_len | name utf-8 | u8 dtype tag | u8 ndim |
              ndim x i64 shape | little-endian data )

dtype tags 0 = f8, 1 = i8, 2 = u8.  The sidecar `<path>.json` carries the
run config and scalar state.  Device tensors are accepted on save (copied to
the host once); fp32 / bf16 tensors are widened to f8, which is exact, so a
save -> load round trip is bit-exact for every dtype this package keeps.
"""

import json
import struct

import numpy as np

MAGIC = b"RPCK"
VERSION = 1

_TAG_OF = {np.dtype("<f8"): 0, np.dtype("<i8"): 1, np.dtype("<u8"): 2}
_DTYPE_OF = {tag: dt for dt, tag in _TAG_OF.items()}
_WIDEN = {"f": np.dtype("<f8"), "i": np.dtype("<i8"), "u": np.dtype("<u8")}


class CheckpointError(RuntimeError):
    pass


def _host_array(value, name):
    try:
        import torch

        if isinstance(value, torch.Tensor):
            t = value.detach()
            if t.dtype in (torch.bfloat16, torch.float16, torch.float32):
                t = t.double()
            value = t.cpu().numpy()
    except ImportError:  # pragma: no cover - torch is always present here
        pass
    arr = np.asarray(value)
    target = _WIDEN.get(arr.dtype.kind)
    if target is None:
        raise CheckpointError(f"unsupported dtype {arr.dtype} for {name!r}")
    if arr.dtype.kind == "f" and arr.dtype.itemsize > 8:
        raise CheckpointError(f"unsupported dtype {arr.dtype} for {name!r}")
    return arr.astype(target, order="C", copy=False)  # keeps 0-d shapes


def save_arrays(path, arrays):
    with open(path, "wb") as fh:
        fh.write(MAGIC + struct.pack("<II", VERSION, len(arrays)))
        for name, value in arrays.items():
            arr = _host_array(value, name)
            key = name.encode("utf-8")
            header = struct.pack(f"<H{len(key)}sBB{arr.ndim}q", len(key), key, _TAG_OF[arr.dtype], arr.ndim,
                                 *arr.shape)
            fh.write(header)
            fh.write(arr.tobytes())


def load_arrays(path):
    out = {}
    with open(path, "rb") as fh:
        blob = fh.read()
    if blob[:4] != MAGIC:
        raise CheckpointError(f"{path} is not a checkpoint container")
    if len(blob) < 12:
        raise CheckpointError(f"truncated header in {path}")
    version, count = struct.unpack_from("<II", blob, 4)
    if version != VERSION:
        raise CheckpointError(f"unsupported container version {version}")
    pos = 12
    try:
        for _ in range(count):
            (name_len,) = struct.unpack_from("<H", blob, pos)
            pos += 2
            name = blob[pos: pos + name_len].decode("utf-8")
            pos += name_len
            tag, ndim = struct.unpack_from("<BB", blob, pos)
            pos += 2
            shape = struct.unpack_from(f"<{ndim}q", blob, pos)
            pos += 8 * ndim
            nbytes = 8 * int(np.prod(shape, dtype=np.int64))
            if pos + nbytes > len(blob):
                raise CheckpointError(f"truncated entry {name!r}")
            out[name] = np.frombuffer(blob, dtype=_DTYPE_OF[tag], count=nbytes // 8, offset=pos).reshape(shape).copy()
            pos += nbytes
    except struct.error as exc:
        raise CheckpointError(f"truncated container {path}: {exc}") from None
    except KeyError as exc:
        raise CheckpointError(f"unknown dtype tag {exc} in {path}") from None
    return out


def save_sidecar(path, payload):
    with open(f"{path}.json", "w") as fh:
        json.dump(payload, fh, indent=2, sort_keys=True)


def load_sidecar(path):
    with open(f"{path}.json") as fh:
        return json.load(fh)
