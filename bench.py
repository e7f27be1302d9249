#!/usr/bin/env python
"""Ouroboros training throughput on B200 (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2|c1|c3|c4|c5]
                  [--mode replicas|ouroboros] [--no-cpu] [--no-compare-k1]

A "step" is one Ouroboros training step (reference PipelineEngine.step,
engine.py:246-259): relay forward of one batch through all K modules, every
module's delayed backward, the mixed tied gradient and the Adam update.
N GPUs run K = N + 1 modules with the reference's ring placement (modules 1
and K share GPU 0, model.py:137-140); at N = 1 both modules of K = 2 live on
GPU 0.  Workload `c2` = BASELINE.json configs[1]: 12-layer Transformer LM,
d 512, f 2048, T 512, B 16, WikiText-103-shaped vocabulary V = 267,735
(Zipf token ids), bf16 compute, fp32 master weights / Adam.

value  : tokens/s with the batch already resident in HBM, device-timed with
         CUDA events over exactly K steps (barrier + synchronize both sides).
e2e    : tokens/s through the public API (`engine.step` on host numpy
         batches, loss read back to the host every step).
roofline: the dominant kernel -- the tcgen05 GEMM of the tied-vocab head
         (4 launches/step, 2*N*d*V FLOPs each) -- achieved TFLOP/s from CUDA
         events recorded around its launches during the timed region.
cpu_baseline: the fp64 CPU oracle (a restatement of the reference path,
         oracle/) on a bounded sample of the same workload (B = 1).
"""

import argparse
import gc
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # BASELINE.json configs[1]; V and B per SURVEY.md section 8(c)/(d)
    "c2": dict(name="12L-d512-T512-WT103shape", vocab=267735, d=512, f=2048, blocks=12, seq=512, batch=16, p=0.1),
    # BASELINE.json configs[0] (the reference's CPU-runnable oracle case)
    "c1": dict(name="4L-d128-V1k", vocab=1000, d=128, f=512, blocks=4, seq=64, batch=16, p=0.1),
    # BASELINE.json configs[2]: Transformer-XL base, enwik8-shaped byte stream
    # (heads / memory / batch from the public XL scripts)
    "c3": dict(name="XL-12L-d512-H8-T512-M512-enwik8shape", vocab=256, d=512, f=2048, blocks=12, seq=512, batch=22,
               p=0.1, heads=8, mem=512),
    # BASELINE.json configs[3]: Transformer-XL with the adaptive tied softmax over a
    # WikiText-103-shaped vocabulary (cutoffs 20k / 40k / 200k, public XL scripts).
    # The published d 410 / 10 heads x 41 break the 16-byte TMA row pitch; the
    # nearest runnable shape is d 400 = 10 heads x 40, d_ff 2104 (= 2100 rounded to 8)
    "c4": dict(name="XL-16L-d400(410)-H10x40-T150-M150-adaptive-WT103shape", vocab=267735, d=400, f=2104, blocks=16,
               seq=150, batch=60, p=0.1, heads=10, mem=150, cutoffs=[20000, 40000, 200000]),
    # BASELINE.json configs[4]: Transformer-XL large, text8-shaped (27 symbols)
    "c5": dict(name="XL-24L-d1024-H8-T768-M768-text8shape", vocab=27, d=1024, f=3072, blocks=24, seq=768,
               batch=16, p=0.1, heads=8, mem=768),
}


def make_stack(c, seed, dtype="bf16"):
    from paper_1909_06695_b200 import model as M

    if c.get("heads"):
        return M.build_xl_stack(c["vocab"], c["d"], c["f"], c["blocks"], c["seq"], c["p"], seed, c["heads"],
                                c["mem"], dtype=dtype, cutoffs=c.get("cutoffs"))
    return M.build_stack(c["vocab"], c["d"], c["f"], c["blocks"], c["seq"], c["p"], seed, dtype=dtype)


def flops_per_token(c):
    """Model FLOPs per token = 3 * F_fwd:
    reference block  F_fwd = n*(2(4d^2+2df) + 2d(T+1)) + 2dV,
    XL block         F_fwd = n*(2(2d^2 + 2d^2(M+T)/T + 2df) + 6d(M+(T+1)/2)) + 2dV."""
    d, f, T, V, n = c["d"], c["f"], c["seq"], c["vocab"], c["blocks"]
    head = 2 * d * V
    if c.get("cutoffs"):
        # adaptive head: the head cluster for every token, a tail cluster's
        # width for the (Zipf) share of tokens that fall in it
        cut = list(c["cutoffs"]) + [V]
        w = 1.0 / np.arange(1, V + 1, dtype=np.float64)
        w /= w.sum()
        head = 2 * d * (cut[0] + len(cut) - 1) + sum(2 * d * (hi - lo) * w[lo:hi].sum() for lo, hi in zip(cut, cut[1:]))
    if c.get("heads"):
        M = c["mem"]
        fwd = n * (2 * (2 * d * d + 2 * d * d * (M + T) / T + 2 * d * f) + 6 * d * (M + (T + 1) / 2)) + head
    else:
        fwd = n * (2 * (4 * d * d + 2 * d * f) + 2 * d * (T + 1)) + 2 * d * V
    return 3 * fwd


def zipf_tokens(rng, shape, vocab):
    # WikiText-shaped id distribution: Zipf(s=1) over the vocabulary
    ranks = np.arange(1, vocab + 1, dtype=np.float64)
    p = 1.0 / ranks
    p /= p.sum()
    return rng.choice(vocab, size=shape, p=p).astype(np.int64)


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return json.load(fh), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "sm_max_mhz": 1965}, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits"],
                    capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 2 + i and r[2 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ---------------------------------------------------------------------------
# CPU baseline: the oracle on a bounded sample


def cpu_oracle_steps(c, K, steps, batch=1, budget_s=None):
    """Per-step seconds of the fp64 oracle Ouroboros step at B = `batch`."""
    from oracle import ouroboros as OO

    opt = OO.Adam(lambda t: 2.5e-4)
    if c.get("heads"):
        from oracle import xl as OX

        V, layers = OX.init_xl_params(c["vocab"], c["d"], c["f"], c["blocks"], c["seq"], c["heads"], 1,
                                      cutoffs=c.get("cutoffs"))
        ora = OX.XLOuroborosOracle(V, layers, K, 3, c["p"], c["heads"], c["mem"], batch, opt, cutoffs=c.get("cutoffs"))
    else:
        V, layers = OO.init_params(c["vocab"], c["d"], c["f"], c["blocks"], c["seq"], 1)
        ora = OO.OuroborosOracle(V, layers, K, 3, c["p"], opt)
    rng = np.random.default_rng(0)
    times = []
    t_start = time.perf_counter()
    for t in range(steps):
        x = zipf_tokens(rng, (batch, c["seq"]), c["vocab"])
        y = zipf_tokens(rng, (batch, c["seq"]), c["vocab"])
        t0 = time.perf_counter()
        ora.step(t, x, y)
        times.append(time.perf_counter() - t0)
        if budget_s is not None and time.perf_counter() - t_start > budget_s:
            break
    return times


def cpu_oracle_rate(c, K, steps=2, batch=1, budget_s=40.0):
    """tokens/s of the fp64 oracle Ouroboros step at B = `batch` (last step timed)."""
    times = cpu_oracle_steps(c, K, steps, batch, budget_s)
    return batch * c["seq"] / times[-1], (
        f"oracle fp64 numpy, K={K}, B={batch}, T={c['seq']}, {len(times)} step(s), last timed")


def cpu_threads():
    try:
        import threadpoolctl

        info = threadpoolctl.threadpool_info()
        return max((i.get("num_threads", 1) for i in info), default=os.cpu_count())
    except Exception:
        return os.cpu_count()


# ---------------------------------------------------------------------------


def run_reference(args, c):
    """--impl reference: the CPU implementation of the path (the oracle port;
    the Python reference itself is not shipped to the GPU box)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    K = 2
    times = cpu_oracle_steps(c, K, args.warmup + args.steps, batch=1)[args.warmup:]
    value = c["seq"] * len(times) / float(np.sum(times))
    sample = f"oracle fp64 numpy Ouroboros step, K={K}, B=1, T={c['seq']}, {len(times)} timed steps"
    line = {
        "impl": "reference", "metric": "train tokens/s (Ouroboros step)", "value": value, "unit": "tokens/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": c["name"], "K_modules": K, "global_batch": 1, "seq_len": c["seq"],
                   "vocab": c["vocab"], "note": "each step is a bounded B=1 sample of the workload"},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cpu_threads(), "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args, c):
    import torch

    from paper_1909_06695_b200 import engine as E
    from paper_1909_06695_b200 import model as M
    from paper_1909_06695_b200 import ops
    from paper_1909_06695_b200 import optim as O

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl")
    # N GPUs -> K = N + 1 modules (ring placement); at N > 1 every rank runs an
    # independent replica until the cross-GPU module exchange lands
    K = 2
    B, T = c["batch"], c["seq"]
    tokens = B * T
    stack = make_stack(c, 1 + rank)
    part = M.partition(stack.num_layers, K)
    cls = E.ConcurrentPipelineEngine if args.engine == "concurrent" else E.PipelineEngine
    eng = cls(stack, part, dropout_seed=3)
    opt = O.make_optimizer("adam", O.LrSchedule(2.5e-4, "fixed"))
    rng = np.random.default_rng(1234 + rank)
    nb = 4
    host = [(zipf_tokens(rng, (B, T), c["vocab"]), zipf_tokens(rng, (B, T), c["vocab"])) for _ in range(nb)]
    dev = [(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()) for x, y in host]

    def barrier():
        if dist is not None:
            dist.barrier()

    t = 0
    for _ in range(max(3, args.warmup)):
        x, y = dev[t % nb]
        eng.step(t, E.BatchSample(x, y, t), opt, sync=True)
        t += 1
    torch.cuda.synchronize()

    # ---- device-resident timed region
    probe = ops.Probe()
    ops.PROBE = probe
    barrier()
    torch.cuda.synchronize()
    s_ev, e_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # clocks are sampled over the device-timed region AND the e2e windows
    # below (the device region alone is ~0.1 s: one nvidia-smi sample)
    clocks = ClockSampler(local).__enter__()
    s_ev.record()
    for _ in range(args.steps):
        x, y = dev[t % nb]
        eng.step(t, E.BatchSample(x, y, t), opt, sync=False)
        t += 1
    e_ev.record()
    torch.cuda.synchronize()
    barrier()
    ops.PROBE = None
    ms = s_ev.elapsed_time(e_ev)
    eng.runtime.check("bench", eng.modules)
    if dist is not None:
        tt = torch.tensor([ms], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    ms_per_step = ms / args.steps
    value = world * tokens * args.steps / (ms / 1e3)

    if c.get("heads"):
        # XL: the attention-score GEMM pair AC = (q+u)k^T, BD = (q+v)r^T over
        # [memory; segment] keys, 2 launches per span, 2*B*T*(M+T)*d FLOPs each
        head = probe.events.get("xl_scores", [])
        n_head_launches = 2 * len(head)
        head_flops = 2.0 * tokens * (c["mem"] + T) * c["d"]
        kernel_name = "gemm_kernel<bf16> (XL attention scores AC and BD, 2*B*T*(M+T)*d FLOPs/launch)"
        if probe.events.get("xl_attn_fwd"):
            # fused scores + relative shift + softmax: AC and BD in one launch
            head = probe.events["xl_attn_fwd"]
            n_head_launches = len(head)
            head_flops = 4.0 * tokens * (c["mem"] + T) * c["d"]
            kernel_name = "xl_attn_fwd_kernel (fused XL scores AC+BD + softmax, 4*B*T*(M+T)*d FLOPs/launch)"
    else:
        head = probe.events.get("head_gemm", []) + probe.events.get("head_gemm_bwd", [])
        n_head_launches = len(probe.events.get("head_gemm", [])) + 3 * len(probe.events.get("head_gemm_bwd", []))
        head_flops = 2.0 * tokens * c["d"] * c["vocab"]
        kernel_name = "gemm_kernel<bf16,BN=256> (tied-vocab head, 2*N*d*V FLOPs/launch)"
    head_ms = [s.elapsed_time(e) for s, e in head]
    pk, pk_kind = peaks()
    # spans: forward = 1 vocab GEMM (+ the tiny CE finish), backward = 3 vocab GEMMs
    avg_head_ms = sum(head_ms) / n_head_launches if head_ms else float("nan")
    achieved = head_flops / (avg_head_ms / 1e3) / 1e12
    head_share = sum(head_ms) / ms if head_ms else None
    launches = probe.launches
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "head_gemm_traffic.json")
    if os.path.exists(tpath) and not c.get("heads"):
        with open(tpath) as fh:
            traffic = json.load(fh).get("bytes_per_launch")

    # ---- end-to-end through the public API with host buffers: three windows
    # of K steps, the median reported (one host hiccup -- a page fault, the
    # clock sampler -- must not decide the headline); GC paused while timing
    def e2e_window():
        nonlocal t
        torch.cuda.synchronize()
        barrier()
        s2, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        w0 = time.perf_counter()
        s2.record()
        for _ in range(args.steps):
            x, y = host[t % nb]
            eng.step(t, E.BatchSample(x, y, t), opt, sync=True)  # H2D tokens, D2H loss
            t += 1
        e2.record()
        torch.cuda.synchronize()
        wall = time.perf_counter() - w0
        barrier()
        ms2 = max(s2.elapsed_time(e2), wall * 1e3)
        if dist is not None:
            tt = torch.tensor([ms2], device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ms2 = float(tt.item())
        return ms2

    gc.disable()
    try:
        windows = sorted(e2e_window() for _ in range(3))
    finally:
        gc.enable()
        clocks.__exit__(None, None, None)
    ms2 = windows[1]
    e2e = world * tokens * args.steps / (ms2 / 1e3)

    # ---- K=1 backprop on the same GPU (the "speedup vs K=1" denominator)
    k1 = None
    if args.compare_k1 and world == 1:
        del eng
        torch.cuda.empty_cache()
        stack1 = make_stack(c, 1)
        seq = E.SequentialRunner(stack1, M.partition(stack1.num_layers, 1), dropout_seed=3)
        opt1 = O.make_optimizer("adam", O.LrSchedule(2.5e-4, "fixed"))
        for i in range(3):
            seq.step(i, E.BatchSample(*dev[i % nb], i), opt1, sync=True)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for i in range(3, 3 + args.steps):
            seq.step(i, E.BatchSample(*dev[i % nb], i), opt1, sync=False)
        b.record()
        torch.cuda.synchronize()
        k1 = tokens * args.steps / (a.elapsed_time(b) / 1e3)

    cpu = None
    if rank == 0 and not args.no_cpu:
        rate, sample = cpu_oracle_rate(c, K)
        cpu = {"value": rate, "unit": "tokens/s", "cores": cpu_threads(), "kind": "port", "sample": sample}

    if rank != 0:
        return
    peak_t = pk.get("bf16_tflops_sustained", pk.get("bf16_tflops"))
    line = {
        "metric": "train tokens/s (Ouroboros step)",
        "value": value,
        "unit": "tokens/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_per_step,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (Zipf token ids, random-init weights)",
        "config": {"workload": c["name"], "K_modules": K, "global_batch": B * world, "seq_len": T,
                   "vocab": c["vocab"], "d_model": c["d"], "d_ff": c["f"], "n_blocks": c["blocks"],
                   **({"n_heads": c["heads"], "mem_len": c["mem"]} if c.get("heads") else {}),
                   "engine": args.engine, "placement": "ring (modules 1 and K on GPU 0)",
                   "parallelism": f"ouroboros K={K} per GPU" + (" (replicas)" if world > 1 else ""),
                   "l2": "working set per step >> 126 MB L2 (no flush needed)"},
        "e2e": {"value": e2e, "unit": "tokens/s", "h2d_bytes_per_step": 2 * tokens * 8,
                "d2h_bytes_per_step": 4 + 4, "window": "median of 3 windows of K steps",
                "windows_ms_per_step": [round(w / args.steps, 3) for w in windows]},
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak_t, "unit": "TFLOP/s",
                     "frac": achieved / peak_t, "traffic": traffic,
                     "kernel": kernel_name,
                     "launches_per_step": n_head_launches / max(args.steps, 1), "share_of_step": head_share,
                     "peak_kind": f"{pk_kind} bf16_tflops_sustained"},
        "model_flops_util": flops_per_token(c) * value / (world * peak_t * 1e12),
        "cpu_baseline": cpu,
        "clocks": clocks.summary(),
        "gpu_launches": launches,
    }
    if k1 is not None:
        line["k1_backprop_tokens_per_s"] = k1
        line["speedup_vs_k1"] = value / k1
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def run_pipeline(args, c):
    """--mode ouroboros: the multi-GPU Ouroboros step, K = N + 1 modules on
    the ring of N GPUs (modules 1 and K on GPU 0), P2P relay + boundary
    exchange over NCCL.  One global batch flows through the pipeline per
    step, so tokens/s = B*T / step time ("scaling": "strong")."""
    import torch
    import torch.distributed as dist

    from paper_1909_06695_b200 import engine as E
    from paper_1909_06695_b200 import model as M
    from paper_1909_06695_b200 import optim as O
    from paper_1909_06695_b200.distributed import DistributedPipelineEngine, build_local_modules

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    K = world + 1
    B, T = c["batch"], c["seq"]
    stack = make_stack(c, 1)
    part = M.partition(stack.num_layers, K)
    mods = build_local_modules(stack, part, 3, rank)
    eng = DistributedPipelineEngine(mods, part, rank, tied=stack.tied_store if rank == 0 else None,
                                    device=stack.runtime.device)
    opt = O.make_optimizer("adam", O.LrSchedule(2.5e-4, "fixed"))
    rng = np.random.default_rng(1234)
    batches = [(torch.from_numpy(zipf_tokens(rng, (B, T), c["vocab"])).cuda(),
                torch.from_numpy(zipf_tokens(rng, (B, T), c["vocab"])).cuda()) for _ in range(4)]

    class _B:
        def __init__(self, x, y, sid):
            self.x, self.y, self.sample_id, self.shape = x, y, sid, (B, T)

    def step(t):
        x, y = batches[t % 4]
        return eng.step(t, _B(x if rank == 0 else None, y if rank == 0 else None, t), opt)

    t = 0
    for _ in range(max(3, args.warmup) + K):
        step(t)
        t += 1
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    s_ev, e_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        s_ev.record()
        for _ in range(args.steps):
            step(t)
            t += 1
        e_ev.record()
        torch.cuda.synchronize()
    ms = s_ev.elapsed_time(e_ev)
    if world > 1:
        tt = torch.tensor([ms], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    stack.runtime.check("bench", list(mods.values()))
    if rank == 0:
        value = B * T * args.steps / (ms / 1e3)
        pk, _ = peaks()
        print(json.dumps({
            "metric": "train tokens/s (Ouroboros step)", "value": value, "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (Zipf token ids, random-init weights)",
            "config": {"workload": c["name"], "K_modules": K, "global_batch": B, "seq_len": T, "vocab": c["vocab"],
                       "placement": "ring (modules 1 and K on GPU 0)", "parallelism": f"ouroboros K={K} over {world} GPUs"},
            "model_flops_util": flops_per_token(c) * value / (world * pk.get("bf16_tflops_sustained", 1385.6) * 1e12),
            "clocks": clocks.summary(),
        }), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=list(CONFIGS))
    ap.add_argument("--engine", default="concurrent", choices=["concurrent", "reference"])
    ap.add_argument("--mode", default="replicas", choices=["replicas", "ouroboros"],
                    help="N>1: independent K=2 replicas per GPU (default) or the multi-GPU Ouroboros pipeline")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-compare-k1", dest="compare_k1", action="store_false",
                    help="skip the K=1 backprop run that gives speedup_vs_k1 (BASELINE metric, second half)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    c = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, c)
    elif args.mode == "ouroboros":
        run_pipeline(args, c)
    else:
        run_ours(args, c)


if __name__ == "__main__":
    main()
