"""The training harness on the device: train / resume / verify / bench, and
checkpoints exchanged with the reference (fixtures written by the live
reference, tests/golden/make_runner_golden.py)."""

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_1909_06695_b200 import checkpoint as ckpt  # noqa: E402
from paper_1909_06695_b200 import runner as R  # noqa: E402
from paper_1909_06695_b200.config import parse_config_file  # noqa: E402
from paper_1909_06695_b200.metrics import read_metrics  # noqa: E402

GOLD = os.path.join(os.path.dirname(__file__), "golden", "runner")
# fp32 check mode vs the reference's fp64 run of the same 12 Adam steps
LOSS_RTOL = 5e-4


@pytest.fixture
def in_gold(monkeypatch):
    monkeypatch.chdir(GOLD)  # the fixture config names data = corpus.txt


def cfg_for(tmp_path, name="run", **kw):
    cfg = parse_config_file(os.path.join(GOLD, "run.cfg"))
    cfg.out_dir = str(tmp_path / name)
    cfg.dtype = "fp32"
    for k, v in kw.items():
        setattr(cfg, k, v)
    return cfg


def test_train_tracks_reference_run(in_gold, tmp_path):
    summary = R.train(cfg_for(tmp_path))
    assert summary["steps_run"] == 12 and not summary["diverged"]
    ours = read_metrics(summary["metrics_path"])
    ref = read_metrics(os.path.join(GOLD, "metrics_full.csv"))
    for a, b in zip(ours, ref):
        assert a.step == b.step and a.lr == b.lr and a.logical == b.logical
        assert abs(a.loss - b.loss) <= LOSS_RTOL * abs(b.loss)
        assert abs(a.grad_sq_norm - b.grad_sq_norm) <= 2e-3 * max(b.grad_sq_norm, 1e-3)
    assert os.path.getsize(summary["trace_path"]) > 0
    assert os.path.isfile(summary["checkpoint_path"]) and os.path.isfile(summary["checkpoint_path"] + ".json")


@pytest.mark.parametrize("mode,dtype", [("ouroboros-ref", "fp32"), ("ouroboros-concurrent", "bf16"),
                                        ("sequential", "bf16")])
def test_halt_and_resume_is_bit_exact(in_gold, tmp_path, mode, dtype):
    full = R.train(cfg_for(tmp_path, "full", mode=mode, dtype=dtype))
    R.train(cfg_for(tmp_path, "halt", mode=mode, dtype=dtype, halt_at=5))
    resumed = R.train(cfg_for(tmp_path, "resumed", mode=mode, dtype=dtype,
                              resume=str(tmp_path / "halt" / "checkpoint.bin")))
    assert resumed["start_step"] == 5 and resumed["steps_run"] == 7
    a = read_metrics(full["metrics_path"])[5:]
    b = read_metrics(resumed["metrics_path"])
    assert [(r.step, r.loss, r.grad_sq_norm, r.logical) for r in a] == \
           [(r.step, r.loss, r.grad_sq_norm, r.logical) for r in b]
    x = ckpt.load_arrays(full["checkpoint_path"])
    y = ckpt.load_arrays(resumed["checkpoint_path"])
    assert sorted(x) == sorted(y)
    for k in x:
        np.testing.assert_array_equal(x[k], y[k], err_msg=k)


def test_resume_from_reference_checkpoint(in_gold, tmp_path):
    """The reference's own halt-at-6 checkpoint (fp64) resumes on the device
    and continues along the reference's resumed trajectory."""
    cfg = cfg_for(tmp_path, "from_ref", resume="halt6.bin")
    summary = R.train(cfg)
    assert summary["start_step"] == 6 and summary["steps_run"] == 6
    ours = read_metrics(summary["metrics_path"])
    ref = read_metrics(os.path.join(GOLD, "metrics_resumed.csv"))
    assert [r.step for r in ours] == [r.step for r in ref]
    for a, b in zip(ours, ref):
        assert abs(a.loss - b.loss) <= LOSS_RTOL * abs(b.loss)
        assert a.logical == b.logical


def test_checkpoint_config_mismatch_is_rejected(in_gold, tmp_path):
    cfg = cfg_for(tmp_path, "bad", resume="halt6.bin", lr=0.003)
    with pytest.raises(ckpt.CheckpointError):
        R.train(cfg)


@pytest.mark.parametrize("dtype,k", [("fp32", 3), ("bf16", 4)])
def test_verify_passes_exactly(in_gold, tmp_path, dtype, k):
    report = R.verify(cfg_for(tmp_path, dtype=dtype, k=k), steps=10)
    assert report["passed"], report
    assert report["oracle_max_abs"] == 0.0 and report["emb_max_abs"] == 0.0
    assert report["dropout_replay_mismatches"] == 0 and report["k1_bitwise_ok"]


def test_verify_current_mode_is_informational(in_gold, tmp_path):
    report = R.verify(cfg_for(tmp_path, stale_weights="current"), steps=6)
    assert report["oracle_informational"] and report["passed"]
    assert report["oracle_max_abs"] > 0.0  # live weights differ from the snapshots


def test_bench_table(in_gold, tmp_path):
    rows = R.bench(cfg_for(tmp_path, dtype="bf16"), [1, 2, 4], steps=8)
    assert [r["k"] for r in rows] == [1, 2, 4]
    # equal synthetic module costs: the logical speed-up grows with K
    assert rows[0]["speedup_logical"] == pytest.approx(1.0, rel=0.05)
    assert rows[2]["speedup_logical"] > rows[1]["speedup_logical"] > 1.0
    assert all(r["device_ms_per_step"] > 0 and r["tokens_per_sec"] > 0 for r in rows)


def test_by_cost_partition_from_device_costs(in_gold, tmp_path):
    from paper_1909_06695_b200.model import measure_layer_costs

    rt = R.build_runtime(cfg_for(tmp_path, balance="by_cost", k=2, dtype="bf16"))
    costs = measure_layer_costs(rt.stack, rt.source.batch_at(0).x)
    assert len(costs) == rt.stack.num_layers and all(c > 0 for c in costs)
    groups = rt.part.groups
    assert groups[0][0] == 0 and groups[-1][1] == rt.stack.num_layers and len(groups) == 2


@pytest.mark.parametrize("mode", ["ouroboros-ref", "ouroboros-concurrent"])
def test_xl_train_halt_and_resume_is_bit_exact(in_gold, tmp_path, mode):
    """Transformer-XL runs carry the segment memory (per module and per
    pending slot) through the checkpoint."""
    kw = dict(mode=mode, n_heads=2, mem_len=16, k=3)
    full = R.train(cfg_for(tmp_path, "full", **kw))
    R.train(cfg_for(tmp_path, "halt", halt_at=5, **kw))
    resumed = R.train(cfg_for(tmp_path, "resumed", resume=str(tmp_path / "halt" / "checkpoint.bin"), **kw))
    a = read_metrics(full["metrics_path"])[5:]
    b = read_metrics(resumed["metrics_path"])
    assert [(r.loss, r.grad_sq_norm) for r in a] == [(r.loss, r.grad_sq_norm) for r in b]
    x = ckpt.load_arrays(full["checkpoint_path"])
    y = ckpt.load_arrays(resumed["checkpoint_path"])
    assert any(k.startswith("m1.mem.") for k in x) and sorted(x) == sorted(y)
    for k in x:
        np.testing.assert_array_equal(x[k], y[k], err_msg=k)


def test_xl_adaptive_train_resume_and_verify(in_gold, tmp_path):
    """A Transformer-XL run with the adaptive tied softmax through the
    harness: halt + resume bit-exact (cluster weights in the checkpoint) and
    verify's delayed gradients equal K=1 backprop exactly."""
    kw = dict(mode="ouroboros-concurrent", n_heads=2, mem_len=16, k=3, adaptive_cutoffs="16,40")
    full = R.train(cfg_for(tmp_path, "full", **kw))
    R.train(cfg_for(tmp_path, "halt", halt_at=4, **kw))
    resumed = R.train(cfg_for(tmp_path, "resumed", resume=str(tmp_path / "halt" / "checkpoint.bin"), **kw))
    a = read_metrics(full["metrics_path"])[4:]
    b = read_metrics(resumed["metrics_path"])
    assert [(r.loss, r.grad_sq_norm) for r in a] == [(r.loss, r.grad_sq_norm) for r in b]
    x = ckpt.load_arrays(full["checkpoint_path"])
    assert any(k.endswith("cluster_weight") for k in x)
    report = R.verify(cfg_for(tmp_path, "verify", **kw), steps=6)
    assert report["passed"], report
    assert report["oracle_max_abs"] == 0.0


def test_verify_xl_passes_exactly(in_gold, tmp_path):
    """verify on a Transformer-XL run: the twin K=1 replay carries the segment
    memory, so every delayed gradient still matches exactly."""
    report = R.verify(cfg_for(tmp_path, n_heads=2, mem_len=16, k=3), steps=8)
    assert report["passed"], report
    assert report["oracle_max_abs"] == 0.0 and report["emb_max_abs"] == 0.0


def test_timed_trace_rows_follow_the_device(tmp_path):
    """with timed_trace the engine writes trace_device.jsonl, one
    row per (step, module, phase) timed by CUDA events on the module's own
    stream: forwards of a step are ordered along the relay, every span has
    positive length, and the logical trace is unchanged."""
    import json

    from paper_1909_06695_b200.config import RunConfig
    from paper_1909_06695_b200.runner import train

    data = tmp_path / "corpus.txt"
    data.write_text("the quick brown fox jumps over the lazy dog " * 200)
    cfg = RunConfig(data=str(data), seq_len=16, batch_size=4, n_blocks=4, model_dim=32, ffn_dim=64, k=3,
                    mode="ouroboros-concurrent", steps=6, warmup_steps=1, dtype="fp32", out_dir=str(tmp_path / "o"),
                    timed_trace=True)
    train(cfg)
    rows = [json.loads(line) for line in open(tmp_path / "o" / "trace_device.jsonl")]
    logical = [json.loads(line) for line in open(tmp_path / "o" / "trace.jsonl")]
    assert len(rows) == 6 * 3 + sum(1 for r in logical if r["phase"] == "backward")
    for r in rows:
        assert r["end"] > r["start"] >= 0.0
    for t in range(6):
        fwd = sorted((r for r in rows if r["step"] == t and r["phase"] == "forward"), key=lambda r: r["module"])
        assert [r["module"] for r in fwd] == [1, 2, 3]
        for a, b in zip(fwd, fwd[1:]):
            assert b["start"] >= a["end"] - 1e-3  # the relay: module k+1 starts after module k


def test_checkpoint_compatibility_is_one_way(in_gold, tmp_path):
    """ADVICE r1 (checkpoint.py docstring): our checkpoints carry module 1's
    embedding outputs (m1.slot{j}.embedded) instead of snapshots of the tied
    matrix, so the reference's `m{k}.ring.{s}.L{i}.tied` entries -- which the
    reference loader pops for every ring parameter (reference runner.py:186-195)
    -- are absent; the reference's own checkpoint has them and loads here
    (test_resume_from_reference_checkpoint)."""
    R.train(cfg_for(tmp_path, "halt", halt_at=5))
    ours = ckpt.load_arrays(str(tmp_path / "halt" / "checkpoint.bin"))
    ring = [n for n in ours if ".ring." in n]
    assert ring and not any(n.endswith(".tied") for n in ring)
    assert any(n.startswith("m1.slot") and n.endswith(".embedded") for n in ours)
    theirs = ckpt.load_arrays(os.path.join(GOLD, "halt6.bin"))
    assert any(".ring." in n and n.endswith(".tied") for n in theirs)
