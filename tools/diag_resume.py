"""Diagnose resume fidelity: run N steps, checkpoint, reload into a fresh
runtime, diff every piece of device state and the next step's packet."""
import os, sys, tempfile
import torch
from paper_1909_06695_b200 import runner as R
from paper_1909_06695_b200.config import parse_config_file

gold = os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "runner")
os.chdir(gold)
cfg = parse_config_file("run.cfg")
cfg.dtype = sys.argv[1] if len(sys.argv) > 1 else "fp32"
N = 5
a = R.build_runtime(cfg)
for t in range(N):
    a.engine.step(t, a.source.batch_at(t), a.optimizer)
path = os.path.join(tempfile.mkdtemp(), "ck.bin")
R.save_training_state(path, a, N)
b = R.build_runtime(cfg)
R.load_training_state(path, b)
def cmp(name, x, y):
    if not torch.equal(x, y):
        print("DIFF", name, float((x.float() - y.float()).abs().max()))
for i, (sa, sb) in enumerate(zip(a.stack.storage, b.stack.storage)):
    cmp(f"master{i}", sa.master, sb.master)
    if sa.m is not None: cmp(f"m{i}", sa.m, sb.m); cmp(f"v{i}", sa.v, sb.v)
    print(i, "ring", sa.ring_step, sb.ring_step)
    for j, s in enumerate(sa.ring_step):
        if s is None: continue
        if s not in sb.ring_step: print("ring missing", i, s); continue
        jb = sb.ring_step.index(s)
        cmp(f"ring{i}.{s}.vec", sa.ring[j][0], sb.ring[jb][0]); cmp(f"ring{i}.{s}.mat", sa.ring[j][1], sb.ring[jb][1])
cmp("tied", a.stack.tied, b.stack.tied)
cmp("tied_m", a.stack.tied_store.m, b.stack.tied_store.m)
for ma, mb in zip(a.engine.modules, b.engine.modules):
    print("module", ma.index, [s.step for s in ma.slots], [s.step for s in mb.slots])
    for sa, sb in zip(ma.slots, mb.slots):
        A, B = sa.arena, sb.arena
        if A.tokens is not None: cmp(f"m{ma.index}.s{sa.step}.tokens", A.tokens, B.tokens)
        for j, (x, y) in enumerate(zip(A.acts, B.acts)): cmp(f"m{ma.index}.s{sa.step}.act{j}", x, y)
        for j, (x, y) in enumerate(zip(A.tapes, B.tapes)):
            for f in ("a", "qkv", "probs_buf", "ctx", "x1", "m", "h1", "mean1", "rstd1", "mean2", "rstd2"):
                cmp(f"m{ma.index}.s{sa.step}.tape{j}.{f}", getattr(x, f), getattr(y, f))
for k in a.engine.boundary:
    cmp(f"boundary{k}", a.engine.boundary[k], b.engine.boundary[k])
pa, la = a.engine.step(N, a.source.batch_at(N), a.optimizer)
pb, lb = b.engine.step(N, b.source.batch_at(N), b.optimizer)
print("loss", la, lb)
for k, (ga, gb) in enumerate(zip(pa.module_grads, pb.module_grads)):
    for key in ga: cmp(f"grad m{k+1} {key}", ga[key], gb[key])
cmp("emb_grad", pa.emb_grad, pb.emb_grad)
print("done")
