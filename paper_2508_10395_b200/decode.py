"""Multi-layer decode-step driver on B200 (the attention block of
``model._Session.decode``, model.py:223-240).

Per layer, in strict order (model.py:230-235):
  q = x @ W_q                       (cuBLAS GEMV; RoPE at pos is applied in-kernel)
  cache.decode_append(x)            (quantize-and-pack kernel; CL: delta vs acc,
                                     then acc += deq(all deltas); GQA: latents)
  ctx = fused remat + attention     (tcgen05 kernel + split combine)
The per-layer input ``x`` is a synthetic post-norm activation supplied by the
caller (layer >= 1 inputs depend on upstream math the hot path does not own),
so W_o / MLP are outside the step, identically for XQuant and the fp16-KV
baseline.

Shapes: ``SHAPES`` mirrors BASELINE.json configs (Llama-2-7B, Llama-3.1-8B,
Llama-2-13B). Batch slots share one length vector; a step appends one token
to every slot.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import cache as C
from .errors import ConfigError


@dataclass(frozen=True)
class ModelShape:
    name: str
    hidden_dim: int
    n_layers: int
    n_heads: int
    kv_group: int = 1
    head_dim: int = 128

    @property
    def kv_width(self) -> int:
        return self.hidden_dim // self.kv_group


SHAPES = {
    "llama2-7b": ModelShape("llama2-7b", 4096, 32, 32, 1),
    "llama3.1-8b": ModelShape("llama3.1-8b", 4096, 32, 32, 4),
    "llama2-13b": ModelShape("llama2-13b", 5120, 40, 40, 1),
}


def synthetic_weights(shape: ModelShape, variant: str, device, seed: int = 0,
                      layers: int | None = None):
    """Random-init bf16 weights, N(0, 1/d) like gen_weights (linalg.py:231-236).

    For xq-gqa the offline SVD factors (linalg.py:103-126) are computed in
    float32 on the device with the reference sign rule (linalg.py:171-176)."""
    g = torch.Generator(device=device).manual_seed(seed)
    d, kvw = shape.hidden_dim, shape.kv_width
    n = shape.n_layers if layers is None else layers
    out, wq = [], []
    std = 1.0 / math.sqrt(d)
    for _ in range(n):
        w_k = (torch.randn(d, kvw, generator=g, device=device) * std).to(torch.bfloat16)
        w_v = (torch.randn(d, kvw, generator=g, device=device) * std).to(torch.bfloat16)
        wq.append((torch.randn(d, d, generator=g, device=device) * std).to(torch.bfloat16))
        lw = C.LayerWeights(w_k=w_k, w_v=w_v)
        if variant == "xq-gqa":
            lw.u_k, lw.fused_k = _svd_factors(w_k)
            lw.u_v, lw.fused_v = _svd_factors(w_v)
        if variant == "xq-cl-gqa":  # shared subspace of [W_k | W_v] (model.py:135-142)
            lw.u_kv, lw.fused_kv = _svd_factors(torch.cat([w_k, w_v], dim=1), u_dtype=torch.float32)
        out.append(lw)
    return out, wq


def _svd_factors(w: torch.Tensor, u_dtype=torch.bfloat16):
    u, s, vt = torch.linalg.svd(w.float(), full_matrices=False)
    idx = torch.argmax(u.abs(), dim=0)
    sign = torch.sign(u[idx, torch.arange(u.shape[1], device=u.device)])
    sign[sign == 0] = 1
    u = u * sign[None, :]
    vt = vt * sign[:, None]
    fused = s[:, None] * vt
    return u.to(u_dtype), fused.to(torch.bfloat16)


def cache_kdim(cache) -> int:
    """Channel count of the fused kernel's A operand (d, or the GQA latent rank)."""
    return cache.latent if cache.variant == "xq-gqa" else cache.d


class Decoder:
    """Per-layer caches of one model shape for ``n_slots`` sequences."""

    def __init__(self, shape: ModelShape, variant: str, bits: int, n_slots: int, max_len: int,
                 weights, w_q, device="cuda", policy: C.LayerPolicy | None = None,
                 tiles_per_chunk: int | None = None, head_shard: tuple[int, int] | None = None,
                 group=None, gather: str = "nccl", acc_precision: str | None = None):
        """``head_shard=(world, rank)``: KV-head-group sharding (parallel.py).
        This rank serves KV heads parallel.head_shard(...) with column-sliced
        weights; step() all-gathers the attention outputs of all ranks, by
        ``all_gather_into_tensor`` (``gather="nccl"``) or by the fused kernel's
        peer stores into symmetric memory (``gather="peer"``)."""
        from . import parallel as P

        if variant not in C.SUPPORTED:
            raise ConfigError(f"variant {variant!r} not supported by the decoder")
        self.shape, self.variant = shape, variant
        self.device = torch.device(device)
        self.n_slots, self.L = n_slots, max_len
        self.policy = policy or (C.LayerPolicy.uniform(16, shape.n_layers) if variant == "fp16"
                                 else C.LayerPolicy.for_bits(bits, shape.n_layers))
        n_heads = shape.n_heads
        self.gather = None
        if head_shard is not None and head_shard[0] > 1:
            if variant == "xq-cl-gqa":
                raise ConfigError("xq-cl-gqa runs batch-sharded (no KV-head-group sharding)")
            world, rank = head_shard
            kv = P.head_shard(shape.n_heads // shape.kv_group, world, rank)
            weights = [P.shard_layer_weights(lw, variant, kv) for lw in weights]
            w_q = [P.shard_wq(w, kv, shape.kv_group) for w in w_q]
            n_heads = len(kv) * shape.kv_group
            if gather == "peer":
                self.gather = P.PeerHeadGather(n_slots, n_heads, world, rank, self.device, group)
            elif gather == "nccl":
                self.gather = P.HeadGather(n_slots, n_heads, world, self.device, group)
            else:
                raise ConfigError(f"gather must be 'nccl' or 'peer', got {gather!r}")
        self.n_heads_local = n_heads
        self.weights, self.w_q = weights, w_q
        kw = dict(n_slots=n_slots, max_len=max_len, hidden_dim=shape.hidden_dim,
                  n_heads=n_heads, n_heads_total=shape.n_heads, kv_group=shape.kv_group,
                  device=self.device)
        self.caches = [C.make_cache(variant, i, self.policy, shape.head_dim, **kw)
                       for i in range(len(weights))]
        # fp16-storage remat accumulator by default (the deltas themselves are formed
        # against float64 accumulator rows in either precision)
        if acc_precision is None:
            acc_precision = "fp16"
        self.acc = (C.Accumulator(n_slots, max_len, shape.hidden_dim, self.device,
                                  precision=acc_precision)
                    if variant in C.CL_VARIANTS else None)
        # one shared length vector (host + device) for all layers
        self.n_tokens = np.zeros(n_slots, dtype=np.int64)
        self.lens_dev = torch.zeros(n_slots, dtype=torch.int32, device=self.device)
        for c in self.caches:
            c.n_tokens = self.n_tokens
            c.lens_dev = self.lens_dev
        self.tpc = tiles_per_chunk
        self.launches = 0  # kernels of this library launched by step()

    # ------------------------------------------------------------------ fill
    def fill_synthetic(self, n_tokens: int, seed: int = 1, rows_per_chunk: int = 8192,
                       mlp_scale: float = 0.03):
        """Cache a synthetic prefix of ``n_tokens`` per slot with the GPU quantizer.

        X rows ~ N(0,1) (unit-RMS post-norm activations); for XQuant-CL the
        per-layer inputs drift like the residual stream, X_i = X_{i-1} +
        mlp_scale * N(0,1) (tests/test_acceptance.py:31-33 uses 0.03)."""
        if n_tokens > self.L:
            raise ConfigError("prefix longer than max_len")
        g = torch.Generator(device=self.device).manual_seed(seed)
        d = self.shape.hidden_dim
        for s in range(self.n_slots):
            x_prev = None
            for i, (cache, lw) in enumerate(zip(self.caches, self.weights)):
                if self.variant in C.CL_VARIANTS:
                    noise = torch.randn(n_tokens, d, generator=g, device=self.device)
                    x_prev = noise if x_prev is None else x_prev + mlp_scale * noise
                    x = x_prev.to(torch.bfloat16)
                else:
                    x = torch.randn(n_tokens, d, generator=g, device=self.device).to(torch.bfloat16)
                cache._prefill(s, x, lw, self.acc)
            if self.acc is not None:
                self.acc.release_prefill(s)
        self.n_tokens[:] = n_tokens
        self.lens_dev.fill_(n_tokens)
        torch.cuda.synchronize(self.device)

    # ------------------------------------------------------------------ step
    def step(self, x_layers: torch.Tensor, attn_out: torch.Tensor | None = None,
             timers: list | None = None) -> torch.Tensor:
        """One decode step: x_layers [n_layers, n_slots, d] (bf16/fp32, device).

        Returns the last layer's attention output [n_slots, n_heads, 128]
        (all layers' outputs when ``attn_out`` [n_layers, n_slots, H, 128]
        is given). With head sharding the gathered output is a copy: the
        gather buffers are rewritten by every rank at the next step. ``timers``: optional list that receives (start, end) CUDA
        event pairs around every fused attention launch."""
        if np.any(self.n_tokens >= self.L):
            raise ConfigError("cache full")
        self.n_tokens += 1
        self.lens_dev.add_(1)
        max_len = int(self.n_tokens.max())
        H = self.n_heads_local
        out = None
        for i, (cache, lw) in enumerate(zip(self.caches, self.weights)):
            x = x_layers[i]
            q = torch.matmul(x, self.w_q[i]).float().view(self.n_slots, H, 128)
            cache._decode(x, lw, self.acc, self.lens_dev)
            out = attn_out[i] if attn_out is not None else torch.empty_like(q)
            if timers is not None:
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
            peer = self.gather is not None and getattr(self.gather, "peer", False)
            if peer:  # the absorbed kernel stores into every rank's gather slot
                cache.peer_outs = self.gather.out_ptrs(i) + [out.data_ptr()]  # + the local copy
                cache.peer_stored = False
            try:
                cache._attend(q, lw, self.acc, self.lens_dev, max_len, out, self.tpc)
            finally:
                if peer:
                    cache.peer_outs = None
            if timers is not None:
                e1.record()
                timers.append((e0, e1))
            self.launches += self._launches_per_layer(cache)
            if peer:  # [B, H_local, 128] -> [B, H, 128]
                out = self.gather.finish(i) if cache.peer_stored else self.gather(out, i)
            elif self.gather is not None:
                out = self.gather(out)
        if self.gather is not None:
            out = out.clone()
        return out

    def _launches_per_layer(self, cache) -> int:
        if self.variant == "fp16":
            return 3  # kv_append, kv_decode, combine
        if self.variant == "kvq":
            return 2  # kvq decode, combine (+ quantizer launches on flushes)
        # fused decode + merge: absorbed = fused, then k_absorb_finish (combine + project
        # in one launch when kdim % 32 == 0, else the two kernels) (+ the q fragments of
        # the grouped-query score mma); unabsorbed = fused, combine
        kdim = cache_kdim(cache)
        absorbed = cache._use_absorbed(kdim, int(cache.n_tokens.max()))
        merge = 1 if kdim % 32 == 0 else 2
        attend = (1 + merge + (1 if self.shape.kv_group == 4 else 0)) if absorbed else 2
        if self.variant == "xq-gqa":
            return 1 + attend  # v-latent quantize (+ a K-latent flush every 128 steps)
        if self.variant == "xq-cl-gqa":  # latent64 (+ flush), fused + merge; the seed /
            # delta layers add the row update, per slot a dequant and the remat GEMM(s)
            upd = cache.layer_index >= self.policy.base_layers - 1
            return 1 + attend + (1 + getattr(cache, "acc16_launches", 2 * self.n_slots) if upd else 0)
        if self.variant == "xq-cl-mha":
            base = cache.layer_index < self.policy.base_layers
            seed = cache.layer_index == self.policy.base_layers - 1
            if getattr(cache, "fused_accumulate", False):
                return 1 + attend  # the delta accumulate ran inside the fused launch
            return 1 + attend + (0 if base and not seed else 1)
        return 1 + attend  # quantize

    # ------------------------------------------------------------- accounting
    def memory_bytes(self) -> dict:
        tot: dict = {}
        for c in self.caches:
            for k, v in c.memory_bytes().items():
                tot[k] = tot.get(k, 0) + v
        if self.acc is not None:
            if self.acc.x_hat is not None:
                tot["cl_accumulator_f32"] = self.acc.x_hat.numel() * 4
            tot["cl_accumulator_f16"] = self.acc.x16.numel() * 2
        return tot

    def check_finite(self):
        for c in self.caches:
            for s in ("stream", "k_stream", "v_stream"):
                st = getattr(c, s, None)
                if st is not None:
                    st.check_finite()
