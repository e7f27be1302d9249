"""C-ABI distributed context (rp_ctx_create / rp_send / rp_recv /
rp_group_*) and device-state export/import, called the way a C host binds
them (ctypes, include/ringpipe_b200.h).  One GPU: a 1-rank communicator
moves a boundary-gradient-sized buffer to itself inside a group."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def test_nccl_context_self_send_recv(dev):
    from paper_1909_06695_b200.comm_abi import NcclContext

    uid = NcclContext.unique_id()
    assert len(uid) == 128
    ctx = NcclContext(0, uid, 0, 1)
    assert (ctx.rank, ctx.nranks) == (0, 1)
    # a C2 boundary gradient [B*T, d] fp32 and a bf16 relay activation
    for t in (torch.randn(16 * 512, 512, device=dev), torch.randn(22 * 512, 512, device=dev).to(torch.bfloat16)):
        u = torch.empty_like(t)
        NcclContext.group_start()
        ctx.send(t, 0)
        ctx.recv(u, 0)
        NcclContext.group_end()
        torch.cuda.synchronize()
        assert torch.equal(u, t)
    ctx.close()


def test_device_state_export_import_bitwise(dev):
    from paper_1909_06695_b200 import comm_abi

    g = torch.Generator(device="cuda").manual_seed(3)
    state = {
        "stack.L1.w1": torch.randn(128, 512, device=dev, generator=g),
        "m1.ring.4.L1.w1": torch.randn(128, 512, device=dev, generator=g).to(torch.bfloat16),
        "m1.slot0.inputs": torch.randint(0, 1000, (16, 64), device=dev, generator=g),
        "optim.adam.v.L1.w1": torch.rand(128, 512, device=dev, generator=g),
    }
    blob = comm_abi.export_state(state)
    back = {k: torch.zeros_like(v) for k, v in state.items()}
    comm_abi.import_state(back, blob)
    for k in state:
        assert torch.equal(back[k], state[k]), k
