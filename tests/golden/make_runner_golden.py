"""Generates tests/golden/runner/* by running the live reference harness
(`ringpipe.runner`, `ringpipe.data`, `ringpipe.config`, `ringpipe.metrics`).

Run in the build container only (the reference tree is not shipped to the GPU
box):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_runner_golden.py

Fixtures:
  corpus.txt                 a deterministic synthetic text corpus
  batches.npz                BatchSource.batch_at(t) for t across two epochs
                             (byte and char vocabularies)
  run.cfg                    the reference's write_config_file of the run config
  metrics_full.csv           reference train() for 12 steps (K=3, Adam, dropout)
  metrics_report.json        reference gradient_norm_report of that log
  halt6.bin / halt6.bin.json reference checkpoint after halting at step 6
  metrics_resumed.csv        reference train() resumed from halt6.bin
"""

import json
import os
import shutil
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "runner")

from ringpipe import runner  # noqa: E402
from ringpipe.config import RunConfig, write_config_file  # noqa: E402
from ringpipe.data import BatchSource, load_corpus  # noqa: E402
from ringpipe.metrics import gradient_norm_report, read_metrics  # noqa: E402
from ringpipe.tensor import SeededRng  # noqa: E402

WORDS = ("the ring of modules passes activations forward while each module computes a stale "
         "gradient for an older sample so no module waits for the backward of its successors "
         "tied embedding weights live on the first device").split()


def make_corpus(path, n_words=3000, seed=5):
    rng = SeededRng(seed)
    picks = (rng.uniform((n_words,)) * len(WORDS)).astype(np.int64)
    caps = rng.uniform((n_words,)) < 0.1
    words = [w.capitalize() if c else w for w, c in zip((WORDS[i] for i in picks), caps)]
    text = " ".join(words)
    text = text.replace(" the ", ". The ", 40)  # a little punctuation for the char vocab filter
    with open(path, "w") as fh:
        fh.write(text + "\n")


def run_config(corpus, out_dir, **kw):
    base = dict(data=corpus, vocab_mode="byte", seq_len=16, batch_size=4, n_blocks=2, model_dim=16,
                ffn_dim=32, dropout_p=0.1, k=3, mode="ouroboros-ref", optimizer="adam", lr=0.002,
                lr_mode="warmup-cosine", warmup_steps=3, steps=12, seed_init=1, seed_data=2,
                seed_dropout=3, out_dir=out_dir)
    base.update(kw)
    return RunConfig(**base)


def main():
    os.makedirs(OUT, exist_ok=True)
    corpus = os.path.join(OUT, "corpus.txt")
    make_corpus(corpus)

    batches = {}
    for mode in ("byte", "char"):
        tokens, vocab = load_corpus(corpus, mode)
        src = BatchSource(tokens, 16, 4, 2)
        batches[f"{mode}_vocab"] = np.array(vocab)
        batches[f"{mode}_n_windows"] = np.array(src.n_windows)
        steps = [0, 1, 2, src.n_windows // 4 - 1, src.n_windows // 4, src.n_windows // 2 + 1]
        batches[f"{mode}_steps"] = np.array(steps)
        for t in steps:
            b = src.batch_at(t)
            batches[f"{mode}_x{t}"] = b.x
            batches[f"{mode}_y{t}"] = b.y
    np.savez_compressed(os.path.join(OUT, "batches.npz"), **batches)

    tmp = tempfile.mkdtemp()
    try:
        # paths inside the fixture are relative to tests/golden/runner
        full = run_config(corpus, os.path.join(tmp, "full"))
        write_config_file(run_config("corpus.txt", "run_out"), os.path.join(OUT, "run.cfg"))
        runner.train(full)
        shutil.copy(os.path.join(tmp, "full", "metrics.csv"), os.path.join(OUT, "metrics_full.csv"))
        report = gradient_norm_report(read_metrics(os.path.join(OUT, "metrics_full.csv")))
        with open(os.path.join(OUT, "metrics_report.json"), "w") as fh:
            json.dump(report, fh, indent=1, sort_keys=True)

        halted = run_config(corpus, os.path.join(tmp, "halt"), halt_at=6)
        runner.train(halted)
        ck = os.path.join(tmp, "halt", "checkpoint.bin")
        shutil.copy(ck, os.path.join(OUT, "halt6.bin"))
        with open(ck + ".json") as fh:
            side = json.load(fh)
        side["config"]["data"] = "corpus.txt"
        side["config"]["out_dir"] = "run_out"
        with open(os.path.join(OUT, "halt6.bin.json"), "w") as fh:
            json.dump(side, fh, indent=2, sort_keys=True)

        resumed = run_config(corpus, os.path.join(tmp, "resumed"), resume=ck)
        runner.train(resumed)
        shutil.copy(os.path.join(tmp, "resumed", "metrics.csv"), os.path.join(OUT, "metrics_resumed.csv"))
    finally:
        shutil.rmtree(tmp)
    print("wrote", sorted(os.listdir(OUT)), file=sys.stderr)


if __name__ == "__main__":
    main()
