#!/usr/bin/env python
"""Decode-throughput benchmark of the B200 XQuant hot path (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl xquant|reference]
                    [--config c2|c3|c4|c1]

Default workload (BASELINE.json configs[1]): XQuant 3-bit (layers 0-2 at
4-bit, LayerPolicy.for_bits), Llama-2-7B shape (32 layers, d=4096, 32 MHA
heads), batch 8 per GPU, 32K context, random-init weights, synthetic
activations. A step = one decode token for every sequence through all 32
layers' attention block (q projection, quantize+append, fused remat +
attention). Under torchrun every rank runs its own batch of 8 (weak scaling,
no data-path collective); the timing is the max over ranks.

Besides the headline line it reports, in the same JSON: the fp16-KV decode
baseline on the same GPU, the roofline of the dominant kernel (fused remat +
attention), the memory-compression factor, the end-to-end number through the
public API with host buffers, and the reference CPU path timed on this box's
host cores.
"""

from __future__ import annotations

import argparse
import gc
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decode tokens/s at 32K ctx vs fp16 KV-cache; remat roofline %; memory compression"

# model shapes (d, heads, kv group, layers) -- the same table as
# paper_2508_10395_b200.decode.SHAPES, inlined so the reference arm never imports
# the package (its process must load no library of ours)
REF_SHAPES = {
    "llama2-7b": dict(hidden_dim=4096, n_heads=32, kv_group=1, n_layers=32),
    "llama3.1-8b": dict(hidden_dim=4096, n_heads=32, kv_group=4, n_layers=32),
    "llama2-13b": dict(hidden_dim=5120, n_heads=40, kv_group=1, n_layers=40),
}

CONFIGS = {
    "c2": dict(workload="XQuant 3-bit, Llama-2-7B shape (32 layers), batch 8, 32K context",
               shape="llama2-7b", variant="xq-mha", bits=3, batch=8, ctx=32768),
    # configs[2]: one global batch of 16 split by sequence over the ranks (16/n per GPU)
    "c3": dict(workload="XQuant-CL 2-bit, Llama-2-7B shape, batch 16, 32K context",
               shape="llama2-7b", variant="xq-cl-mha", bits=2, batch=16, ctx=32768,
               parallel="batch"),
    "c4": dict(workload="xq-gqa 3-bit latent, Llama-3.1-8B shape, batch 32, 16K context",
               shape="llama3.1-8b", variant="xq-gqa", bits=3, batch=32, ctx=16384,
               parallel="heads"),
    # XQuant-CL on the GQA shape (shared K|V latent subspace)
    "c6": dict(workload="xq-cl-gqa 3-bit, Llama-3.1-8B shape, batch 8, 16K context",
               shape="llama3.1-8b", variant="xq-cl-gqa", bits=3, batch=8, ctx=16384),
    "c1": dict(workload="XQuant 4-bit, one Llama-2-7B layer, batch 1, 2K context",
               shape="llama2-7b", variant="xq-mha", bits=4, batch=1, ctx=2048, layers=1),
    # C5 long-context sweep (8K-128K, batch 1-64 over 8 GPUs): one point per run, the
    # per-GPU shard of a batch-sharded deployment; tools/sweep_c5.py drives --ctx/--batch
    "c5": dict(workload="XQuant-CL 3-bit, Llama-2-13B shape (40 layers), batch 8 per GPU, 32K context",
               shape="llama2-13b", variant="xq-cl-mha", bits=3, batch=8, ctx=32768),
}


def _split(cfg, world: int, rank: int) -> tuple[int, int, int]:
    """(sequences on this rank, sequences per step over all ranks, first sequence).

    "batch": configs[2]'s one global batch split by sequence (16/n per GPU, strong
    scaling); "heads": every rank serves the whole batch for its KV heads; else
    every rank decodes its own batch (weak scaling)."""
    B, mode = cfg["batch"], cfg.get("parallel")
    if mode == "batch" and world > 1:
        per, extra = divmod(B, world)
        start = rank * per + min(rank, extra)
        return per + (1 if rank < extra else 0), B, start
    if mode == "heads" and world > 1:
        return B, B, 0
    return B, world * B, rank * B


def _config_dict(cfg, world: int, gather: str = "nccl") -> dict:
    """The workload description both arms print (identical keys and values)."""
    sh = REF_SHAPES[cfg["shape"]]
    n_layers = cfg.get("layers", sh["n_layers"])
    bits = cfg["bits"]
    policy = [max(bits, 4) if i < 3 else bits for i in range(n_layers)]  # LayerPolicy.for_bits
    mode = cfg.get("parallel")
    if world == 1:
        par = "single GPU"
    elif mode == "heads":
        par = f"kv-head-group x{world} (" + (
            "peer-store gather from the projection kernel into symmetric memory" if gather == "peer"
            else "NCCL all-gather of attention outputs") + ")"
    elif mode == "batch":
        par = f"batch-split x{world} ({cfg['batch']} sequences over {world} GPUs, no data-path collective)"
    else:
        par = f"batch-sharded x{world} ({cfg['batch']} sequences per GPU, no data-path collective)"
    return {"workload": cfg["workload"], "shape": cfg["shape"], "variant": cfg["variant"],
            "bits": bits, "policy_bits": policy[:4] + ["..."], "global_batch": _split(cfg, world, 0)[1],
            "batch_per_gpu": _split(cfg, world, 0)[0],
            "context": cfg["ctx"] + 1, "layers": n_layers, "parallelism": par,
            "l2": "no flush: per-step inputs (packed caches, GBs) exceed the 126 MB L2"}


def _peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            p = json.load(f)
        return p, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.lines, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi's start-up (a fork/exec, ~100 ms of CPU) stays outside the timed
            # region: wait for its first sample, then mark where the region's samples begin
            t_end = time.perf_counter() + 3.0
            while not self.lines and time.perf_counter() < t_end and self.proc.poll() is None:
                time.sleep(0.01)
        except OSError:
            self.proc = None
        self.mark = len(self.lines)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        mark = getattr(self, "mark", 0)
        lines = self.lines[mark:]
        note = None
        if not lines and mark > 0:  # region shorter than the 200 ms sampling period
            lines = self.lines[mark - 1:mark]
            note = "timed region shorter than the 200 ms sampling period: nearest sample before it"
        for ln in lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        out = {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
               "reasons": sorted(reasons), "samples": 0 if note else len(sm)}
        if note:
            out["note"] = note
        return out


# ---------------------------------------------------------------------------
# reference CPU path (oracle/_ref = the unmodified reference, else the port)
# ---------------------------------------------------------------------------


def _import_reference():
    ref = os.path.join(ROOT, "oracle", "_ref")
    if os.path.isdir(os.path.join(ref, "xcache")):
        sys.path.insert(0, ref)
        import xcache  # noqa: F401

        return "reference"
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    return "port"


class CpuReferenceStep:
    """One layer x one sequence of the reference decode step at full context:
    decode_append -> rematerialize -> _attention (model.py:232-235)."""

    def __init__(self, cfg, seed=0):
        import numpy as np

        self.kind = _import_reference()
        sh = REF_SHAPES[cfg["shape"]]
        self.d, self.H, self.g = sh["hidden_dim"], sh["n_heads"], sh["kv_group"]
        self.L = sh["n_layers"] if "layers" not in cfg else cfg["layers"]
        self.variant, self.bits, self.ctx, self.batch = cfg["variant"], cfg["bits"], cfg["ctx"], cfg["batch"]
        rng = np.random.default_rng(seed)
        d, kvw = self.d, self.d // self.g
        self.w_k = rng.normal(size=(d, kvw)) / math.sqrt(d)
        self.w_v = rng.normal(size=(d, kvw)) / math.sqrt(d)
        x = rng.normal(size=(self.ctx, d))
        self.rng = rng
        if self.kind == "reference":
            from xcache.cache import LayerPolicy, LayerWeights, make_cache
            from xcache.linalg import SvdFactors

            z = np.zeros((1, 1))
            kw = {}
            if self.variant == "xq-gqa":
                kw = self._svd(SvdFactors)
            if self.variant == "xq-cl-gqa":
                u, sg, vt = np.linalg.svd(np.hstack([self.w_k, self.w_v]), full_matrices=False)
                kw = {"svd_kv": SvdFactors(u=u, sigma=sg, b_t=vt)}
            self.lw = LayerWeights(gamma_attn=None, gamma_mlp=None, w_q=z, w_k=self.w_k,
                                   w_v=self.w_v, w_o=z, w_up=z, w_down=z, **kw)
            # a delta layer is the CL steady state; the accumulator is seeded
            # from a synthetic base reconstruction (cache.py:463-467)
            variant = "xq-mha" if self.variant == "xq-mha" else self.variant
            pol = LayerPolicy([self.bits] * 2, base_layers=1, high_precision_prefix=1)
            self.cache = make_cache(variant, 1 if variant in ("xq-cl-mha", "xq-cl-gqa") else 0, pol, 128)
            self.acc = None
            if variant in ("xq-cl-mha", "xq-cl-gqa"):
                from xcache.cache import Accumulator

                self.acc = Accumulator()
                self.acc.seed(x + 0.01 * rng.normal(size=x.shape))
            self.cache.prefill(x, self.lw, self.acc)
        else:
            import xq_oracle as O

            self.O = O
            self.x_rows = x
            self.cache = O.XqMhaCache(self.bits, 128, 128)
            self.cache.append(x)

    def _svd(self, SvdFactors):
        import numpy as np

        out = {}
        for name, w in (("svd_k", self.w_k), ("svd_v", self.w_v)):
            u, s, vt = np.linalg.svd(w, full_matrices=False)
            out[name] = SvdFactors(u=u, sigma=s, b_t=vt)
        return out

    def step(self) -> float:
        import numpy as np

        row = self.rng.normal(size=(self.d,))
        q = self.rng.normal(size=(1, self.H * 128))
        t0 = time.perf_counter()
        if self.kind == "reference":
            from xcache.linalg import apply_rope
            from xcache.model import _attention

            if self.acc is not None:  # extend the seed accumulator by the new row
                self.acc.x_hat = np.vstack([self.acc.x_hat, row[None]])
            self.cache.decode_append(row, self.lw, self.acc)
            n = self.cache.n_tokens
            k, v = self.cache.rematerialize(self.lw, np.arange(n), self.acc)
            qr = apply_rope(q, np.array([n - 1]), 128)
            _attention(qr, k, v, self.H, self.g)
        else:
            O = self.O
            self.cache.append(row)
            k, v = self.cache.remat(self.w_k, self.w_v)
            n = k.shape[0]
            O.attention(O.apply_rope(q, [n - 1], 128), k, v, self.H, self.g)
        return time.perf_counter() - t0

    def tokens_per_s(self, seconds_per_layer_seq: float) -> float:
        # a full step = L layers x B sequences of this work and yields B tokens
        return 1.0 / (seconds_per_layer_seq * self.L)

    def sample_desc(self):
        return (f"{'reference xcache (oracle/_ref, native Cython lane + OpenBLAS fp64)' if self.kind == 'reference' else 'numpy port (oracle/xq_oracle.py)'}: "
                f"1 layer x 1 sequence of the {self.variant} {self.bits}-bit decode step at "
                f"l={self.ctx + 1} (decode_append + rematerialize + _attention), "
                f"extrapolated x{self.L} layers (x{self.batch} sequences per {self.batch} tokens)")


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    t_build = time.perf_counter()
    ref = CpuReferenceStep(cfg)
    build_s = time.perf_counter() - t_build
    for _ in range(args.warmup):
        ref.step()
    times = [ref.step() for _ in range(args.steps)]
    per = statistics.mean(times)
    val = ref.tokens_per_s(per)
    # a reference "step" is the bounded sample: one layer x one sequence of the
    # full-context decode step; value extrapolates it to tokens/s of the workload
    # (L layer-samples per token of a sequence; sequences run one after another)
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "tokens/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": per * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": _config_dict(cfg, args.gpus, args.gather),
        "cpu_baseline": {"value": val, "unit": "tokens/s", "cores": os.cpu_count(),
                         "kind": ref.kind, "sample": ref.sample_desc(),
                         "seconds_per_layer_seq": per, "setup_s": build_s,
                         "ms_per_full_step_extrapolated": per * 1e3 * ref.L * cfg["batch"]},
        "e2e": {"value": val, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------


def _dist():
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        # communicator-init lines on stderr: the rank count is checkable from the log
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def _barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def _max_over_ranks(world, v: float) -> float:
    if world == 1:
        return v
    import torch
    import torch.distributed as dist

    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _time_steps(dec, xs, steps, world, timers=None, sampler=None):
    import torch

    _barrier(world)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ctx = sampler if sampler is not None else _Null()
    with ctx:
        torch.cuda.nvtx.range_push("bench_timed")  # ncu launch lists filter on this range
        e0.record()
        for k in range(steps):
            dec.step(xs[k], timers=timers)
        e1.record()
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_pop()
    _barrier(world)
    return e0.elapsed_time(e1) / 1e3


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def _prefill_leg(cfg, shape, n_layers, weights, w_q, dev, n_max: int = 8192):
    """One sequence's prompt through every layer's prefill_attend (model.py:205-221):
    bulk quantize, K/V rebuilt by the tcgen05 remat GEMM (RoPE in its epilogue),
    causal flash attention. Inputs device-resident; CUDA events around the layers."""
    import torch

    from paper_2508_10395_b200 import decode as D

    n = min(cfg["ctx"], n_max)
    try:
        dec = D.Decoder(shape, cfg["variant"], cfg["bits"], 1, -(-n // 128) * 128, weights, w_q,
                        device=dev)
        g = torch.Generator(device=dev).manual_seed(7)
        xs = [torch.randn(n, shape.hidden_dim, generator=g, device=dev).to(torch.bfloat16)
              for _ in range(n_layers)]
        qs = [torch.matmul(x, w) for x, w in zip(xs, w_q)]

        def run():
            for i, c in enumerate(dec.caches):
                c.n_tokens[:] = 0
                c.prefill_attend(xs[i], qs[i], dec.weights[i], dec.acc)

        run()  # warm-up (weight layouts, workspaces)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run()
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 1e3
        d, kvw, H = shape.hidden_dim, shape.kv_width, shape.n_heads
        kdim = kvw if cfg["variant"] == "xq-gqa" else d
        flops = n_layers * (2.0 * n * kdim * 2 * kvw + 2.0 * n * n * H * 128)  # remat + causal attn
        out = {"value": n / t, "unit": "prompt tokens/s", "prompt_tokens": n, "layers": n_layers,
               "ms": t * 1e3, "tflops_achieved": flops / t / 1e12,
               "kernels": "xq_quantize_rows (+ CL / latent variants), k_dequant_rows_f16, "
                          "k_gemm_f16 (tcgen05 remat, RoPE epilogue), k_rope_rows, k_prefill_attend"}
        del dec, xs, qs
        return out
    except torch.OutOfMemoryError as e:
        return {"value": None, "note": f"prefill leg out of memory: {str(e)[:100]}"}


def run_xquant(args, cfg):
    import torch

    from paper_2508_10395_b200 import decode as D
    from paper_2508_10395_b200 import sysmodel as S

    world, rank, local = _dist()
    dev = torch.device("cuda", local)
    shape = D.SHAPES[cfg["shape"]]
    n_layers = cfg.get("layers", shape.n_layers)
    B, tokens_per_step, _ = _split(cfg, world, rank)
    ctx = cfg["ctx"]
    total_steps = args.warmup + 2 * args.steps + 2
    L_max = -(-(ctx + total_steps) // 128) * 128
    # "heads": KV-head-group sharding of one global batch (strong scaling, one
    # all-gather of attention outputs per layer); "batch": the global batch split
    # by sequence (strong scaling, no collective); otherwise every rank decodes
    # its own batch (weak scaling, no collective)
    heads = cfg.get("parallel") == "heads" and world > 1
    strong = heads or (cfg.get("parallel") == "batch" and world > 1)
    wseed = 0 if strong else rank  # one model; batch-split ranks fill their own sequences
    weights, w_q = D.synthetic_weights(shape, cfg["variant"], dev, seed=wseed, layers=n_layers)
    shard = (world, rank) if heads else None

    def make(variant):
        dec = D.Decoder(shape, variant, cfg["bits"], B, L_max, weights, w_q, device=dev,
                        head_shard=shard, gather=args.gather)
        t0 = time.perf_counter()
        dec.fill_synthetic(ctx, seed=1 + (rank if not heads else 0))
        return dec, time.perf_counter() - t0

    g = torch.Generator(device=dev).manual_seed(100 + (rank if not heads else 0))
    d = shape.hidden_dim
    n_in = args.warmup + args.steps
    xs = [torch.randn(n_layers, B, d, generator=g, device=dev).to(torch.bfloat16) for _ in range(n_in)]

    # ---------------- XQuant arm (device-resident inputs) ----------------
    dec, fill_s = make(cfg["variant"])
    for k in range(args.warmup):
        dec.step(xs[k])
    dec.check_finite()
    timers = []
    sampler = ClockSampler(local)
    launches0 = dec.launches
    ctx_before = int(dec.n_tokens[0])
    t = _time_steps(dec, xs[args.warmup:], args.steps, world, timers=timers, sampler=sampler)
    launches = dec.launches - launches0
    t = _max_over_ranks(world, t)
    kern_s = sum(a.elapsed_time(b) for a, b in timers) / 1e3
    kern_s = _max_over_ranks(world, kern_s)
    value = tokens_per_step * args.steps / t
    ms_per_step = t / args.steps * 1e3
    l_avg = ctx_before + (args.steps + 1) / 2.0

    # ---------------- end to end through the public API ----------------
    x_host = [x.cpu().pin_memory() for x in xs[:args.steps]]
    out_host = torch.empty((B, shape.n_heads, 128), dtype=torch.float32).pin_memory()  # gathered
    x_dev = torch.empty_like(xs[0])
    _barrier(world)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for k in range(args.steps):
        x_dev.copy_(x_host[k], non_blocking=True)
        out = dec.step(x_dev)
        out_host.copy_(out, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    t_e2e = _max_over_ranks(world, e0.elapsed_time(e1) / 1e3)
    e2e_value = tokens_per_step * args.steps / t_e2e
    mem = dec.memory_bytes()
    last = dec.caches[-1]
    dec_absorbed = (cfg["variant"] != "fp16"
                    and last._use_absorbed(D.cache_kdim(last), int(last.n_tokens.max())))
    bits_per_layer = dec.policy.bits
    del dec
    for w in weights:
        w._cache.clear()
    gc.collect()
    torch.cuda.empty_cache()

    # ---------------- fp16-KV baseline on the same GPU ----------------
    fp16 = None
    if not args.no_fp16:
        try:
            fdec, _ = make("fp16")
            for k in range(args.warmup):
                fdec.step(xs[k])
            t16 = _time_steps(fdec, xs[args.warmup:], args.steps, world)
            t16 = _max_over_ranks(world, t16)
            kv_bytes = S.cache_bytes("fp16", l_avg, d, 16, shape.kv_group) * n_layers * B
            fp16 = {"value": tokens_per_step * args.steps / t16, "unit": "tokens/s",
                    "ms_per_step": t16 / args.steps * 1e3,
                    "kv_cache_bytes": fdec.memory_bytes().get("kv_cache"),
                    "hbm_gbs_achieved": kv_bytes / (t16 / args.steps) / 1e9,
                    "kernel": "xq_kv_decode_attend (split-K flash-decode, bf16 K/V)"}
            del fdec
            gc.collect()
            torch.cuda.empty_cache()
        except torch.OutOfMemoryError as e:
            fp16 = {"value": None, "note": f"fp16 KV cache does not fit one B200: {str(e)[:120]}"}

    # ------- quantized-KV baseline at equal bits (kvq, cache.py:326-360; opt-in) -------
    kvq = None
    if args.kvq:
        try:
            qdec, _ = make("kvq")
            for k in range(args.warmup):
                qdec.step(xs[k])
            tq = _time_steps(qdec, xs[args.warmup:], args.steps, world)
            tq = _max_over_ranks(world, tq)
            qbytes = sum(S.cache_bytes("kvq", l_avg, d, b, shape.kv_group) for b in qdec.policy.bits) * B
            kvq = {"value": tokens_per_step * args.steps / tq, "unit": "tokens/s",
                   "ms_per_step": tq / args.steps * 1e3,
                   "hbm_gbs_achieved": qbytes / (tq / args.steps) / 1e9,
                   "compression": S.compression_factor("kvq", qdec.policy.bits, shape.kv_group),
                   "kernel": "xq_kvq_decode_attend (cp.async-staged codes, register dequant + RoPE flash-decode)"}
            del qdec
            gc.collect()
            torch.cuda.empty_cache()
        except torch.OutOfMemoryError as e:
            kvq = {"value": None, "note": f"kvq cache does not fit one B200: {str(e)[:120]}"}

    # ---------------- prefill (the attention block of _Session.prefill) ----------------
    prefill = None
    if world == 1 and not args.no_prefill:
        prefill = _prefill_leg(cfg, shape, n_layers, weights, w_q, dev)

    if rank != 0:
        return
    # ---------------- roofline of the dominant kernel ----------------
    peaks, peak_src = _peaks()
    absorbed = dec_absorbed
    flops_unabsorbed = B * (S.remat_flops(cfg["variant"], l_avg, d, shape.kv_group)
                            + S.attention_flops(l_avg, shape.n_heads)) / (world if heads else 1)
    if absorbed:
        flops_launch = B * S.absorbed_flops(cfg["variant"], l_avg, d, shape.kv_group,
                                            shape.n_heads) / (world if heads else 1)
    else:
        flops_launch = flops_unabsorbed
    per_launch = kern_s / (args.steps * n_layers)
    achieved = flops_launch / per_launch / 1e12
    peak = peaks["bf16_tflops_sustained"]
    traffic = None
    prof = os.path.join(ROOT, "profiles", "decode_kernel_ncu.json")
    if os.path.exists(prof):
        with open(prof) as f:
            traffic = json.load(f).get(cfg["variant"] + f"_{cfg['bits']}", {}).get("dram_bytes_per_launch")
    step_flops = n_layers * flops_launch
    step_bytes = sum(S.cache_bytes(cfg["variant"], l_avg, d, b, shape.kv_group) for b in bits_per_layer) * B
    t_roof = max(step_flops / (peak * 1e12), step_bytes / (peaks["hbm_gbs"] * 1e9))
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            ref = CpuReferenceStep(cfg)
            ref.step()
            per = statistics.mean(ref.step() for _ in range(2))
            cpu = {"value": ref.tokens_per_s(per), "unit": "tokens/s", "cores": os.cpu_count(),
                   "kind": ref.kind, "sample": ref.sample_desc(), "seconds_per_layer_seq": per}
        except Exception as e:  # pragma: no cover - reported, not fatal
            cpu = {"value": None, "error": repr(e)[:200]}
    comp = S.compression_factor(cfg["variant"], bits_per_layer, shape.kv_group)
    fp16_arena = S.cache_bytes("fp16", 1, d, 16, shape.kv_group) * B * L_max * n_layers
    xq_arena = mem.get("codes", 0) + mem.get("params", 0) + mem.get("k_codes", 0) + mem.get("k_params", 0) \
        + mem.get("v_codes", 0) + mem.get("v_params", 0) + mem.get("x16", 0)
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "strong" if strong else "weak", "vs_baseline": None,
        "dtype": "f16",
        "data": "synthetic (random-init weights, N(0,1) activations)",
        "config": _config_dict(cfg, world, args.gather),
        "fp16_kv": fp16,
        "speedup_vs_fp16_kv": (value / fp16["value"]) if fp16 and fp16.get("value") else None,
        "kvq": kvq,
        "prefill": prefill,
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": ("k_decode_absorbed (+k_absorb_finish: tile merge + W_v projection)" if absorbed
                                else "k_decode_attend (+k_combine)"),
                     "flops_per_launch": flops_launch, "launch_us": per_launch * 1e6,
                     "flops_note": ("algorithmic FLOPs of the V-absorbed path (sysmodel.absorbed_flops); "
                                    "the unabsorbed remat+attention count is flops_unabsorbed"
                                    if absorbed else "sysmodel.remat_flops + attention_flops"),
                     "flops_unabsorbed": flops_unabsorbed,
                     "peak_source": f"{peak_src} bf16_tflops_sustained (fp16 MMA, same rate)"},
        "remat_roofline_frac_step": t_roof / (ms_per_step / 1e3),
        "compression": {"factor": comp, "formula": "1/sysmodel.normalized_kv_size",
                        "arena_bytes_measured": xq_arena,
                        "fp16_kv_bytes_same_capacity": fp16_arena,
                        "measured_factor": fp16_arena / xq_arena if xq_arena else None,
                        "extra_bytes": {k: v for k, v in mem.items() if k not in ("codes", "params")}},
        "e2e": {"value": e2e_value, "unit": "tokens/s",
                "h2d_bytes_per_step": x_host[0].numel() * x_host[0].element_size(),
                "d2h_bytes_per_step": out_host.numel() * 4,
                "api": "paper_2508_10395_b200.decode.Decoder.step (pinned host in/out)"},
        "gpu_launches": launches,
        "clocks": sampler.summary(),
        "cpu_baseline": cpu,
        "setup": {"fill_s": fill_s},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["xquant", "reference"], default="xquant")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c2")
    ap.add_argument("--no-fp16", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--kvq", action="store_true", help="also time the kvq baseline at equal bits")
    ap.add_argument("--no-prefill", action="store_true", help="skip the prefill leg")
    ap.add_argument("--gather", choices=["nccl", "peer"], default="nccl",
                    help="KV-head-group sharding (c4 under torchrun): NCCL all-gather, or the "
                         "fused kernel's peer stores into torch symmetric memory")
    ap.add_argument("--ctx", type=int, default=None, help="override the config's context")
    ap.add_argument("--batch", type=int, default=None, help="override the per-GPU batch")
    args = ap.parse_args()
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    world = int(os.environ.get("WORLD_SIZE", "0"))
    if world == 0 and args.gpus > 1:
        # not under torchrun: start one rank per GPU ourselves (same launch as the driver's)
        import socket

        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
               f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))
    if world and world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(2)
    cfg = dict(CONFIGS[args.config])
    if args.ctx or args.batch:
        cfg["ctx"] = args.ctx or cfg["ctx"]
        cfg["batch"] = args.batch or cfg["batch"]
        cfg["workload"] = (cfg["workload"].split(", batch")[0] +
                           f", batch {cfg['batch']} per GPU, {cfg['ctx'] // 1024}K context")
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_xquant(args, cfg)


if __name__ == "__main__":
    main()
