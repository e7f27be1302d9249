"""Host side of the training harness against fixtures written by the live
reference (tests/golden/make_runner_golden.py): config files, the batch
stream, the RPCK checkpoint container and the metrics log / trend report."""

import json
import os

import numpy as np
import pytest

from paper_1909_06695_b200 import checkpoint as ckpt
from paper_1909_06695_b200 import config as C
from paper_1909_06695_b200.data import BatchSource, DataError, encode_chars, load_corpus, seeded_permutation
from paper_1909_06695_b200.metrics import MetricsWriter, gradient_norm_report, read_metrics
from paper_1909_06695_b200.rng import mix64

GOLD = os.path.join(os.path.dirname(__file__), "golden", "runner")


def test_config_file_round_trip():
    cfg = C.parse_config_file(os.path.join(GOLD, "run.cfg"))
    assert (cfg.k, cfg.model_dim, cfg.ffn_dim, cfg.n_blocks, cfg.seq_len) == (3, 16, 32, 2, 16)
    assert cfg.adam_eps == 1e-8 and cfg.lr == 0.002 and cfg.data == "corpus.txt"
    assert cfg.dtype == "bf16"  # the one added field keeps its default
    cfg.validate(check_paths=False)
    assert cfg.n_layers == 4


def test_config_validation_and_overrides(tmp_path):
    cfg = C.RunConfig()
    C.apply_overrides(cfg, {"seed": 5, "k": "4", "lr": "0.1", "mode": None})
    assert (cfg.seed_init, cfg.seed_data, cfg.seed_dropout) == (mix64(5, 1), mix64(5, 2), mix64(5, 3))
    assert cfg.k == 4 and cfg.lr == 0.1
    with pytest.raises(C.ConfigError):
        C.apply_overrides(cfg, {"nope": 1})
    bad = [dict(mode="x"), dict(k=0), dict(k=11), dict(mode="ouroboros-concurrent", k=1), dict(steps=0),
           dict(dropout_p=1.0), dict(warmup_steps=1000), dict(seq_len=1), dict(dtype="fp16")]
    for kw in bad:
        with pytest.raises(C.ConfigError):
            C.RunConfig(**kw).validate(check_paths=False)
    with pytest.raises(C.ConfigError):
        C.RunConfig().validate()  # data file missing
    p = tmp_path / "c.cfg"
    p.write_text("k = 2  # comment\n\n mode=ouroboros-concurrent\n")
    got = C.parse_config_file(str(p))
    assert got.k == 2 and got.mode == "ouroboros-concurrent"
    p.write_text("garbage\n")
    with pytest.raises(C.ConfigError):
        C.parse_config_file(str(p))
    C.write_config_file(got, str(p))
    assert C.parse_config_file(str(p)) == got


def test_batch_stream_matches_reference():
    gold = np.load(os.path.join(GOLD, "batches.npz"))
    for mode in ("byte", "char"):
        tokens, vocab = load_corpus(os.path.join(GOLD, "corpus.txt"), mode)
        assert vocab == int(gold[f"{mode}_vocab"])
        src = BatchSource(tokens, 16, 4, 2)
        assert src.n_windows == int(gold[f"{mode}_n_windows"])
        for t in gold[f"{mode}_steps"]:
            b = src.batch_at(int(t))
            np.testing.assert_array_equal(b.x, gold[f"{mode}_x{t}"])
            np.testing.assert_array_equal(b.y, gold[f"{mode}_y{t}"])
            assert b.sample_id == t


def test_data_edge_cases(tmp_path):
    assert sorted(seeded_permutation(17, 3)) == list(range(17))
    assert list(seeded_permutation(1, 3)) == [0]
    assert list(encode_chars(b"Ab, z!")) == [1, 2, 0, 26]
    with pytest.raises(DataError):
        BatchSource(np.arange(10), 1, 2, 0)
    with pytest.raises(DataError):
        BatchSource(np.arange(4), 4, 2, 0)
    empty = tmp_path / "e.txt"
    empty.write_bytes(b"")
    with pytest.raises(DataError):
        load_corpus(str(empty), "byte")
    digits = tmp_path / "d.txt"
    digits.write_bytes(b"1234")
    with pytest.raises(DataError):
        load_corpus(str(digits), "char")
    with pytest.raises(DataError):
        load_corpus(str(digits), "word")


def test_checkpoint_container_is_byte_compatible(tmp_path):
    src = os.path.join(GOLD, "halt6.bin")
    arrays = ckpt.load_arrays(src)
    assert arrays["stack.tied"].shape == (256, 16) and arrays["stack.tied"].dtype == np.float64
    assert arrays["m1.slot0.seeds"].dtype == np.uint64
    assert arrays["m1.slot0.inputs"].dtype == np.int64
    assert sorted(k for k in arrays if k.startswith("boundary.")) == ["boundary.1", "boundary.2"]
    out = tmp_path / "re.bin"
    ckpt.save_arrays(str(out), arrays)
    with open(src, "rb") as a, open(out, "rb") as b:
        assert a.read() == b.read()  # our writer reproduces the reference file byte for byte


def test_checkpoint_errors_and_widening(tmp_path):
    p = str(tmp_path / "x.bin")
    ckpt.save_arrays(p, {"f": np.arange(3, dtype=np.float32), "i": np.array(7), "u": np.array([1], np.uint32)})
    got = ckpt.load_arrays(p)
    assert got["f"].dtype == np.float64 and got["i"].shape == () and got["u"].dtype == np.uint64
    with pytest.raises(ckpt.CheckpointError):
        ckpt.save_arrays(p, {"b": np.array(["s"])})
    blob = open(p, "rb").read()
    open(p, "wb").write(blob[:-4])
    with pytest.raises(ckpt.CheckpointError):
        ckpt.load_arrays(p)
    open(p, "wb").write(b"NOPE" + blob[4:])
    with pytest.raises(ckpt.CheckpointError):
        ckpt.load_arrays(p)
    ckpt.save_sidecar(p, {"next_step": 3})
    assert ckpt.load_sidecar(p) == {"next_step": 3}


def test_metrics_log_round_trip_and_report(tmp_path):
    src = os.path.join(GOLD, "metrics_full.csv")
    rows = read_metrics(src)
    assert [r.step for r in rows] == list(range(12))
    out = tmp_path / "m.csv"
    with MetricsWriter(str(out)) as w:
        for r in rows:
            w.write(r)
    assert out.read_text() == open(src).read()
    with open(os.path.join(GOLD, "metrics_report.json")) as fh:
        want = json.load(fh)
    assert gradient_norm_report(rows) == want
    with pytest.raises(ValueError):
        gradient_norm_report([])
    (tmp_path / "bad.csv").write_text("a,b\n1,2\n")
    with pytest.raises(ValueError):
        read_metrics(str(tmp_path / "bad.csv"))
