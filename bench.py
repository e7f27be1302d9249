#!/usr/bin/env python
"""Ouroboros training throughput on B200 (BASELINE.json metric:
"train tokens/s at K=1/2/4/8 B200 (Transformer-XL); speedup vs K=1 backprop").

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config c3|c1|c2|c4|c5] [--mode pipeline|replicas]
                  [--micro M] [--no-cpu] [--no-compare-k1] [--no-fp32]

A "step" is one Ouroboros training step (reference PipelineEngine.step,
engine.py:246-259): relay forward of one batch through all K modules, every
module's delayed backward, the mixed tied gradient and the Adam update.

Default workload `c3` = BASELINE.json configs[2], the configuration the
metric is quoted on: Transformer-XL base, 12 layers, d 512, 8 heads x 64,
d_ff 2048, segment T = 512 with memory M = 512, enwik8-shaped byte stream
(vocabulary 256), B 22; bf16 compute, fp32 master weights and Adam.

N GPUs run the Ouroboros pipeline with K = N + 1 modules on the reference's
ring placement (modules 1 and K share GPU 0, model.py:137-140); at N = 1 both
modules of K = 2 live on GPU 0.  One global batch per step, so "scaling" is
"strong".  `--mode replicas` instead runs independent K=2 replicas per GPU
(weak scaling; opt-in, not the metric).

value   : tokens/s with the batches resident in HBM, device-timed with CUDA
          events over exactly K steps (barrier + synchronize on both sides,
          max over ranks).
e2e     : tokens/s through the public API (`engine.step` on host numpy
          batches: H2D tokens + targets, D2H loss + status word every step).
roofline: the dominant kernel family, timed live with CUDA events in a second
          K-step window: at XL configs the block's dense tcgen05 GEMMs (QKV, R,
          out-projection, FFN and their gradients; 2*M*N*K FLOPs per launch),
          at c2 the tied-vocab head GEMM (2*N*d*V per launch).
check_mode_fp32: the same step in the fp32 check mode (3xTF32 GEMMs), the
          precision class the parity tests run in.
cpu_baseline: the fp64 CPU oracle port (oracle/, a restatement of the
          reference path) on a bounded B = 1 sample of the same workload.
--impl reference: the live reference (baseline/_ref, numba kernels) on the
          box's host cores when installed, else the oracle port.
"""

import argparse
import contextlib
import gc
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # BASELINE.json configs[2]: Transformer-XL base, enwik8-shaped byte stream
    # (heads / memory / batch from the public XL scripts)
    "c3": dict(name="XL-12L-d512-H8-T512-M512-enwik8shape", vocab=256, d=512, f=2048, blocks=12, seq=512, batch=22,
               p=0.1, heads=8, mem=512),
    # BASELINE.json configs[1]; V and B per SURVEY.md section 8(c)/(d)
    "c2": dict(name="12L-d512-T512-WT103shape", vocab=267735, d=512, f=2048, blocks=12, seq=512, batch=16, p=0.1),
    # BASELINE.json configs[0] (the reference's CPU-runnable oracle case)
    "c1": dict(name="4L-d128-V1k", vocab=1000, d=128, f=512, blocks=4, seq=64, batch=16, p=0.1),
    # BASELINE.json configs[3]: Transformer-XL with the adaptive tied softmax over a
    # WikiText-103-shaped vocabulary (cutoffs 20k / 40k / 200k, public XL scripts);
    # the published d 410 = 10 heads x 41 and d_ff 2100: bf16 rows at 16-byte pitches
    "c4": dict(name="XL-16L-d410-H10x41-T150-M150-adaptive-WT103shape", vocab=267735, d=410, f=2100, blocks=16,
               seq=150, batch=60, p=0.1, heads=10, mem=150, cutoffs=[20000, 40000, 200000]),
    # BASELINE.json configs[4]: Transformer-XL large, text8-shaped (27 symbols)
    "c5": dict(name="XL-24L-d1024-H8-T768-M768-text8shape", vocab=27, d=1024, f=3072, blocks=24, seq=768,
               batch=16, p=0.1, heads=8, mem=768),
}

METRIC = "train tokens/s (Ouroboros step)"


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


def cpu_info():
    """Host CPU model, physical cores and the CPUs this process may use."""
    model = None
    phys = set()
    cur = {}
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if ":" not in line:
                    if cur:
                        phys.add((cur.get("physical id", "0"), cur.get("core id", cur.get("processor"))))
                    cur = {}
                    continue
                k, v = (s.strip() for s in line.split(":", 1))
                cur[k] = v
                if k == "model name" and model is None:
                    model = v
        if cur:
            phys.add((cur.get("physical id", "0"), cur.get("core id", cur.get("processor"))))
    except OSError:
        pass
    try:
        usable = len(os.sched_getaffinity(0))
    except AttributeError:
        usable = os.cpu_count()
    return {"model": model, "physical_cores": len(phys) or None, "logical_cpus": os.cpu_count(),
            "usable_cpus": usable}


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
# CPU baselines


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


def blas_threads():
    try:
        import threadpoolctl

        info = threadpoolctl.threadpool_info()
        return max((i.get("num_threads", 1) for i in info), default=os.cpu_count())
    except Exception:
        return os.cpu_count()


def cpu_port_baseline(c, K=2):
    """The oracle port timed on one B = 1 step of the workload (~10-30 s)."""
    times = cpu_oracle_steps(c, K, 1, batch=1)
    arch = "Transformer-XL restatement (oracle/xl.py)" if c.get("heads") else "reference architecture"
    return {"value": c["seq"] / times[-1], "unit": "tokens/s", "cores": blas_threads(), "kind": "port",
            "sample": f"oracle fp64 numpy Ouroboros step ({arch}), K={K}, B=1, T={c['seq']}, 1 step timed",
            "cpu": cpu_info()}


def _live_reference():
    """The installed reference package (baseline/_ref), or None."""
    path = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(path, "ringpipe")):
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/rp_numba_cache")
    if path not in sys.path:
        sys.path.insert(0, path)
    try:
        import ringpipe  # noqa: F401
        from ringpipe import engine, kernels, model, optim
    except Exception:
        return None
    return model, engine, optim, kernels


def run_reference(args, c):
    """--impl reference: the reference's own CPU implementation of the path on
    the box's host cores.  The live reference (baseline/_ref: numba fp64
    kernels, ConcurrentPipelineEngine with one worker thread per module) runs
    the reference architecture at the workload's shapes -- it has no
    Transformer-XL attention, so at XL configs it runs the reference block at
    the same d, d_ff, depth, T and vocabulary (labelled).  Without the install
    the oracle port stands in.  Each step is a bounded B = 1 sample."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    K = world + 1
    ref = _live_reference()
    budget = float(os.environ.get("RP_REF_BUDGET_S", "150"))
    if ref is not None:
        RM, RE, RO, RK = ref
        RK.warmup()
        stack = RM.build_stack(c["vocab"], c["d"], c["f"], c["blocks"], c["seq"], c["p"], 1)
        part = RM.partition(len(stack.layers), K)
        eng = RE.ConcurrentPipelineEngine(stack, part, 3)
        opt = RO.make_optimizer("adam", RO.LrSchedule(2.5e-4, "fixed"))
        rng = np.random.default_rng(0)
        times = []
        t0 = time.perf_counter()
        n_warm = 1
        for t in range(n_warm + args.steps):
            x = zipf_tokens(rng, (1, c["seq"]), c["vocab"])
            y = zipf_tokens(rng, (1, c["seq"]), c["vocab"])
            s = time.perf_counter()
            eng.step(t, RE.BatchSample(x, y, t), opt)
            if t >= n_warm:
                times.append(time.perf_counter() - s)
            if time.perf_counter() - t0 > budget and times:
                break
        eng.close()
        kind, cores = "reference", K + 1
        arch = ("reference block (no XL memory / relative positions) at the XL shapes" if c.get("heads")
                else "reference architecture")
        sample = (f"live reference ringpipe (baseline/_ref, numba fp64), ConcurrentPipelineEngine K={K} "
                  f"({K} worker threads + coordinator), {arch}, B=1, T={c['seq']}, {n_warm} warm-up step, "
                  f"{len(times)} timed step(s) (wall budget {budget:.0f} s)")
    else:
        times = cpu_oracle_steps(c, K, 1 + args.steps, batch=1, budget_s=budget)[1:] or cpu_oracle_steps(c, K, 1)
        kind, cores = "port", blas_threads()
        sample = f"oracle fp64 numpy port, K={K}, B=1, T={c['seq']}, {len(times)} timed step(s)"
    value = c["seq"] * len(times) / float(np.sum(times))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s",
        "n_gpus": args.gpus, "steps": len(times), "warmup": 1, "ms_per_step": 1e3 * float(np.mean(times)),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": c["name"], "K_modules": K, "global_batch": 1, "seq_len": c["seq"],
                   "vocab": c["vocab"], "d_model": c["d"], "d_ff": c["f"], "n_blocks": c["blocks"],
                   "note": "each step is a bounded B=1 sample of the workload"},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": kind, "sample": sample,
                         "cpu": cpu_info()},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm


class _Job:
    """One bench configuration on this rank: a step function over resident
    device batches or host batches, plus the engine's status check."""

    def __init__(self, args, c, world, rank, dtype="bf16"):
        import torch

        from paper_1909_06695_b200 import engine as E
        from paper_1909_06695_b200 import model as M
        from paper_1909_06695_b200 import optim as O

        self.E = E
        self.B, self.T = c["batch"], c["seq"]
        self.world, self.rank = world, rank
        # --engine distributed at N = 1 runs the multi-GPU engine itself (K = 2
        # on one rank, no transfers): the pipeline code path of this bench on a
        # single GPU (its micro-batched relay included)
        self.pipeline = (world > 1 and args.mode == "pipeline") or args.engine == "distributed"
        self.K = world + 1 if self.pipeline else 2
        B, T = self.B, self.T
        stack = make_stack(c, 1 if self.pipeline else 1 + rank, dtype)
        self.stack = stack
        part = M.partition(stack.num_layers, self.K)
        self.opt = O.make_optimizer("adam", O.LrSchedule(2.5e-4, "fixed"))
        if self.pipeline:
            from paper_1909_06695_b200.distributed import DistributedPipelineEngine, build_local_modules

            mods = build_local_modules(stack, part, 3, rank)
            self.eng = DistributedPipelineEngine(mods, part, rank, tied=stack.tied_store if rank == 0 else None,
                                                 device=stack.runtime.device, micro_batches=args.micro)
            self.mods = [mods[k] for k in sorted(mods)]
        else:
            self.eng = E.ConcurrentPipelineEngine(stack, part, dropout_seed=3)
            self.mods = self.eng.modules
        seed = 1234 if self.pipeline else 1234 + rank
        rng = np.random.default_rng(seed)
        nb = 4
        self.host = [(zipf_tokens(rng, (B, T), c["vocab"]), zipf_tokens(rng, (B, T), c["vocab"])) for _ in range(nb)]
        self.dev = [(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()) for x, y in self.host]
        self.t = 0

    def step(self, host=False, sync=False):
        x, y = (self.host if host else self.dev)[self.t % len(self.dev)]
        if self.pipeline and self.rank != 0:
            x = y = None  # tokens and targets live on the Ouroboros rank only
        b = self.E.BatchSample(x, y, self.t)
        if self.pipeline:
            self.eng.step(self.t, b, self.opt, sync=sync, shape=(self.B, self.T))
        else:
            self.eng.step(self.t, b, self.opt, sync=sync)
        self.t += 1

    def flush(self):
        """Read the last step's result (sync="lagged" leaves one in flight)."""
        self.eng.flush_lagged()

    def check(self):
        self.stack.runtime.check("bench", self.mods)

    @contextlib.contextmanager
    def serial(self):
        """Issue every module's work on the current stream (the concurrent
        engine's issue order is a topological order of its event graph, so
        the step is unchanged): per-launch CUDA-event times then measure each
        kernel alone, as the serialized ncu launch list does, instead of
        kernels sharing the GPU with the other module's stream."""
        import torch

        eng = self.eng
        if self.pipeline or not hasattr(eng, "_fs"):
            yield False
            return
        main = torch.cuda.current_stream()
        saved = (eng._fs, eng._bs, eng._ts)
        eng._fs, eng._bs, eng._ts = [main] * len(saved[0]), [main] * len(saved[1]), main
        try:
            yield True
        finally:
            eng._fs, eng._bs, eng._ts = saved


def _timed(job, steps, barrier, host=False, sync=False):
    """Device ms over `steps` steps (max over ranks), barrier + sync both sides."""
    import torch

    torch.cuda.synchronize()
    barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    s.record()
    for _ in range(steps):
        job.step(host=host, sync=sync)
    if sync == "lagged":
        job.flush()
    e.record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - w0
    barrier()
    ms = s.elapsed_time(e)
    if host:
        ms = max(ms, wall * 1e3)  # host-side work between launches counts end to end
    return ms


def _max_over_ranks(ms, dist):
    if dist is None:
        return ms
    import torch

    tt = torch.tensor([ms], device="cuda")
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    return float(tt.item())


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

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if dist is not None:
            dist.barrier()

    job = _Job(args, c, world, rank)
    K, B, T = job.K, job.B, job.T
    pipeline = job.pipeline
    tokens_step = B * T * (1 if pipeline else world)
    for _ in range(K):  # fill the stale slots, checking every step
        job.step(sync=True)
    # the host issues each step while the device runs the previous one and
    # reads that step's loss one step later (engine.step(sync="lagged")); it
    # never queues further ahead: with several steps queued, a full launch
    # queue on one stream blocks the host from feeding the others and the
    # modules' streams lose their overlap (measured: sync=False windows
    # 13.7-14.9 ms/step against 13.5 at C3)
    step_sync = "lagged"
    for _ in range(max(3, args.warmup)):  # warm-up steps issued exactly like the timed ones
        job.step(sync=step_sync)
    if step_sync == "lagged":
        job.flush()
    torch.cuda.synchronize()
    job.check()

    clocks = ClockSampler(local).__enter__()
    # ---- 1. device-resident timed window (the headline `value`)
    ms = _max_over_ranks(_timed(job, args.steps, barrier, sync=step_sync), dist)
    job.check()
    ms_per_step = ms / args.steps
    value = tokens_step * args.steps / (ms / 1e3)

    # ---- 2. instrumented window: CUDA events around the dominant kernel
    # family's launches (on the streams they run on) + launch count
    probe = ops.Probe()
    ops.PROBE = probe
    with job.serial() as serialized:
        ms_probe = _max_over_ranks(_timed(job, args.steps, barrier), dist)
    ops.PROBE = None
    pk, pk_kind = peaks()
    peak_t = pk.get("bf16_tflops_sustained", pk.get("bf16_tflops"))
    if c.get("heads"):
        fl, kms, nl = probe.achieved("block_gemm")
        kernel_name = ("rp::gemm_kernel (tcgen05, TMA, 2-CTA) over the block's dense contractions: QKV, R, "
                       "out-projection, FFN fwd + their gradient GEMMs; 2*M*N*K FLOPs per launch")
    else:
        head = probe.events.get("head_gemm", []) + probe.events.get("head_gemm_bwd", [])
        n_head = len(probe.events.get("head_gemm", [])) + 3 * len(probe.events.get("head_gemm_bwd", []))
        kms = sum(s.elapsed_time(e) for s, e in head)
        fl = 2.0 * B * T * c["d"] * c["vocab"] * n_head
        nl = n_head
        kernel_name = "rp::gemm_kernel<bf16,BN=256,2-CTA> (tied-vocab head, 2*N*d*V FLOPs per launch)"
    achieved = fl / (kms / 1e3) / 1e12 if kms > 0 else float("nan")
    roofline = {"bound": "tensor", "achieved": achieved, "peak": peak_t, "unit": "TFLOP/s",
                "frac": achieved / peak_t, "traffic": None, "kernel": kernel_name,
                "flops_per_launch": fl / max(nl, 1), "avg_launch_ms": kms / max(nl, 1),
                "launches_per_step": nl / args.steps, "share_of_step": kms / ms_probe if ms_probe else None,
                "peak_kind": f"{pk_kind} bf16_tflops_sustained",
                "window": ("second K-step window, every launch on one stream (kernels timed alone, as in the "
                           "serialized ncu launch list), CUDA events around each launch"
                           if serialized else "second K-step window with CUDA events (ms_per_step_instrumented)"),
                "ms_per_step_instrumented": ms_probe / args.steps}
    if c.get("heads"):
        for tag in ("xl_attn_fwd", "xl_attn_bwd"):
            ev = probe.events.get(tag, [])
            if ev:
                roofline[f"{tag}_ms_per_step"] = sum(s.elapsed_time(e) for s, e in ev) / args.steps
    tpath = os.path.join(ROOT, "profiles", "dominant_kernel_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as fh:
            tr = json.load(fh).get(args.config)
        if tr:
            roofline["traffic"] = tr.get("bytes_per_launch")
            roofline["traffic_source"] = tr.get("source")
    launches = probe.launches

    # ---- 3. end to end through the public API with host batches: three
    # windows of K steps, the median reported; GC paused while timing
    gc.disable()
    try:
        # the public step API with host batches; the host reads every step's
        # loss (and status words) from pinned memory one step behind, so it
        # never idles the GPU between steps (engine.step(sync="lagged"))
        windows = sorted(_max_over_ranks(_timed(job, args.steps, barrier, host=True, sync="lagged"), dist)
                         for _ in range(3))
    finally:
        gc.enable()
        clocks.__exit__(None, None, None)
    ms2 = windows[1]
    e2e = tokens_step * args.steps / (ms2 / 1e3)
    job_mods = list(job.mods)
    del job
    gc.collect()
    torch.cuda.empty_cache()

    # ---- 4. fp32 check mode (3xTF32 GEMMs, fp32 row kernels): same step
    fp32 = None
    if args.fp32:
        barrier()
        job32 = _Job(args, c, world, rank, dtype="fp32")
        for _ in range(3 + job32.K):
            job32.step(sync=True)
        n32 = max(3, args.steps // 2)
        ms32 = _max_over_ranks(_timed(job32, n32, barrier), dist)
        job32.check()
        fp32 = {"value": tokens_step * n32 / (ms32 / 1e3), "unit": "tokens/s", "ms_per_step": ms32 / n32,
                "steps": n32, "dtype": "fp32 (3xTF32 tensor-core GEMMs, fp32 activations)"}
        del job32
        gc.collect()
        torch.cuda.empty_cache()

    barrier()
    # ---- 5. K=1 backprop on one GPU, same global batch (the "speedup vs K=1" denominator)
    k1 = None
    if args.compare_k1 and rank == 0:
        stack1 = make_stack(c, 1)
        seq = E.SequentialRunner(stack1, M.partition(stack1.num_layers, 1), dropout_seed=3)
        opt1 = O.make_optimizer("adam", O.LrSchedule(2.5e-4, "fixed"))
        rng = np.random.default_rng(1234)
        dev = [(torch.from_numpy(zipf_tokens(rng, (B, T), c["vocab"])).cuda(),
                torch.from_numpy(zipf_tokens(rng, (B, T), c["vocab"])).cuda()) for _ in range(4)]
        for i in range(3):
            seq.step(i, E.BatchSample(*dev[i % 4], i), opt1, sync=True)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for i in range(3, 3 + args.steps):
            seq.step(i, E.BatchSample(*dev[i % 4], i), opt1, sync=False)
        b.record()
        torch.cuda.synchronize()
        k1 = B * T * args.steps / (a.elapsed_time(b) / 1e3)
        del seq, stack1

    cpu = None
    if rank == 0 and args.cpu:
        cpu = cpu_port_baseline(c)

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": value,
            "unit": "tokens/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": max(3, args.warmup),
            "ms_per_step": ms_per_step,
            "higher_is_better": True,
            "scaling": "weak" if world > 1 and not pipeline else "strong",
            "vs_baseline": None,
            "dtype": "bf16",
            "data": "synthetic (Zipf token ids, random-init weights)",
            "config": {"workload": c["name"], "K_modules": K, "global_batch": B * (1 if pipeline else world),
                       "seq_len": T, "vocab": c["vocab"], "d_model": c["d"], "d_ff": c["f"], "n_blocks": c["blocks"],
                       **({"n_heads": c["heads"], "mem_len": c["mem"]} if c.get("heads") else {}),
                       "placement": "ring (modules 1 and K on GPU 0)",
                       "engine": "DistributedPipelineEngine" if pipeline else "ConcurrentPipelineEngine",
                       "parallelism": (f"ouroboros pipeline K={K} over {world} GPUs"
                                       + (f", {args.micro} micro-batches" if args.micro > 1 else "")
                                       if pipeline else
                                       f"ouroboros K={K} per GPU" + (" (replicas)" if world > 1 else "")),
                       "l2": "working set per step >> 126 MB L2 (no flush needed)",
                       "issue": "engine.step(sync='lagged'): the host stays one step ahead of the device"},
            "e2e": {"value": e2e, "unit": "tokens/s", "h2d_bytes_per_step": 2 * B * T * 8,
                    "d2h_bytes_per_step": 4 + 4 * (len(job_mods) + 1), "window": "median of 3 windows of K steps",
                    "api": ("engine.step(t, host batch, optimizer, sync='lagged'): pinned H2D of the step's tokens "
                            "and targets, D2H of its loss + status words, each read on the host one step later; "
                            "the window ends after the last step's loss is read"),
                    "windows_ms_per_step": [round(w / args.steps, 3) for w in windows]},
            "roofline": roofline,
            "model_flops_util": flops_per_token(c) * value / (world * peak_t * 1e12),
            "check_mode_fp32": fp32,
            "cpu_baseline": cpu,
            "clocks": clocks.summary(),
            "gpu_launches": launches,
        }
        if k1 is not None:
            line["k1_backprop_tokens_per_s"] = k1
            line["speedup_vs_k1"] = value / k1
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=list(CONFIGS))
    ap.add_argument("--mode", default="pipeline", choices=["pipeline", "replicas"],
                    help="N>1: the Ouroboros pipeline K=N+1 (default) or independent K=2 replicas per GPU")
    # Default 1: on one B200 a C3 step with 2 micro-batches through the same
    # engine measured 21.4 vs 13.6 ms -- at 11 x 512 rows the N = 512 block
    # GEMMs fill 0.6 waves of CTA pairs, so halving the rows nearly doubles
    # their time per token; the micro-batched relay pays off only when the
    # pipeline bubble it removes exceeds that (many GPUs, large batches)
    ap.add_argument("--micro", type=int, default=int(os.environ.get("RP_MICRO", "1")),
                    help="micro-batches per relay in the multi-GPU pipeline")
    ap.add_argument("--engine", default="auto", choices=["auto", "distributed"],
                    help="distributed: the multi-GPU engine even at N = 1 (K = 2 on one rank)")
    ap.add_argument("--no-cpu", dest="cpu", action="store_false")
    ap.add_argument("--no-fp32", dest="fp32", action="store_false", help="skip the fp32 check-mode line")
    ap.add_argument("--no-compare-k1", dest="compare_k1", action="store_false",
                    help="skip the K=1 backprop run that gives speedup_vs_k1 (BASELINE metric, second half)")
    ap.add_argument("--dropout", type=float, default=None,
                    help="override the config's dropout probability (A/B of the mask cost; not a bench line)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    c = dict(CONFIGS[args.config])
    if args.dropout is not None:
        c["p"] = args.dropout
        c["name"] += f"-dropout{args.dropout:g}"
    if args.impl == "reference":
        run_reference(args, c)
    else:
        run_ours(args, c)


if __name__ == "__main__":
    main()
