"""C-ABI state export/import (rp_export_state / rp_import_state,
include/ringpipe_b200.h) on host buffers: the container it writes is the
reference's RPCK checkpoint format (checkpoint.py:1-70) -- our Python loader
reads it -- and it imports what the Python saver writes.  No GPU needed."""

import os
import tempfile

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_1909_06695_b200 import checkpoint as ckpt  # noqa: E402
from paper_1909_06695_b200 import comm_abi  # noqa: E402
from paper_1909_06695_b200.errors import DimensionError  # noqa: E402


def _arrays():
    rng = np.random.default_rng(0)
    f32 = rng.standard_normal((3, 5)).astype(np.float32)
    bf = torch.from_numpy(rng.standard_normal((4, 8)).astype(np.float32)).to(torch.bfloat16)
    return {
        "stack.L1.wq": f32,
        "m1.slot0.meta": np.array([7, 7], dtype=np.int64),
        "m1.slot0.seeds": np.array([2 ** 63 + 5, 11], dtype=np.uint64),
        "m2.ring.3.L2.w1": bf,
        "boundary.1": np.zeros((2, 3, 4), dtype=np.float32) + 0.25,
    }


def _as_numpy(v):
    return v.double().numpy() if torch.is_tensor(v) else v


def test_export_writes_the_rpck_container():
    arrs = _arrays()
    blob = comm_abi.export_state(arrs)
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "state.bin")
        with open(path, "wb") as fh:
            fh.write(blob)
        back = ckpt.load_arrays(path)
    assert list(back) == list(arrs)
    for k, v in arrs.items():
        want = _as_numpy(v)
        assert back[k].shape == want.shape
        np.testing.assert_array_equal(back[k], want.astype(back[k].dtype))


def test_import_reads_the_python_saver_and_round_trips_bitwise():
    arrs = _arrays()
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "state.bin")
        ckpt.save_arrays(path, arrs)
        with open(path, "rb") as fh:
            blob = fh.read()
    dst = {k: (torch.zeros_like(v) if torch.is_tensor(v) else np.zeros_like(v)) for k, v in arrs.items()}
    comm_abi.import_state(list(dst.items())[::-1], blob)  # by name, any order
    for k, v in arrs.items():
        if torch.is_tensor(v):
            assert torch.equal(dst[k], v)
        else:
            np.testing.assert_array_equal(dst[k], v)
    # export -> import is the identity
    dst2 = {k: (torch.zeros_like(v) if torch.is_tensor(v) else np.zeros_like(v)) for k, v in arrs.items()}
    comm_abi.import_state(dst2, comm_abi.export_state(arrs))
    for k, v in arrs.items():
        assert (torch.equal(dst2[k], v) if torch.is_tensor(v) else np.array_equal(dst2[k], v))


def test_import_errors_name_the_entry():
    blob = comm_abi.export_state({"a": np.zeros(4, dtype=np.float32)})
    with pytest.raises(ValueError, match="lacks b"):
        comm_abi.import_state({"b": np.zeros(4, dtype=np.float32)}, blob)
    with pytest.raises(DimensionError, match="elements"):
        comm_abi.import_state({"a": np.zeros(5, dtype=np.float32)}, blob)
    with pytest.raises(ValueError, match="RPCK"):
        comm_abi.import_state({"a": np.zeros(4, dtype=np.float32)}, b"nope" + bytes(20))
