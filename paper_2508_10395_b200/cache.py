"""Per-layer cache backends on B200 -- batched, device-resident mirror of the
reference's ``xcache.cache`` (/root/reference/pkg/src/xcache/cache.py).

Same variant tags (``cache.py:41``), ``LayerPolicy`` (``cache.py:70-121``),
``make_cache`` factory (``cache.py:620-630``) and backend interface
``prefill / decode_append / rematerialize`` (``cache.py:255-281``). The
differences are the ones the hot path needs:

* a backend holds ``n_slots`` sequences (the reference holds one,
  ``SPEC.md:311``); inputs carry a leading slot dimension;
* payloads live in packed HBM arenas (codes byte-identical to the reference's
  ``pack_codes`` per row, fp16 scale/zero-point per group) filled by the
  sm_100a quantizer;
* ``decode_attend(q, weights, acc)`` runs the fused dequant -> tcgen05
  rematerialise -> RoPE -> flash-decode kernel and returns the attention
  output without materialising K/V; ``rematerialize`` stays for parity and
  returns float32 K/V (SIMT debug kernel).

All six variants (``cache.py:41``) have a GPU backend: ``fp16`` (baseline
semantics), ``xq-mha``, ``xq-gqa``, ``xq-cl-mha`` on the hot path, and the
"next" rows ``kvq`` and ``xq-cl-gqa``.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from .errors import ConfigError, DataError, ShapeError, UsageError

VARIANTS = ("fp16", "kvq", "xq-mha", "xq-gqa", "xq-cl-mha", "xq-cl-gqa")  # cache.py:41
CL_VARIANTS = ("xq-cl-mha", "xq-cl-gqa")
SUPPORTED = ("fp16", "kvq", "xq-mha", "xq-gqa", "xq-cl-mha", "xq-cl-gqa")
DEFAULT_GROUP_SIZE = 128
DEFAULT_ACCUMULATOR_BITS = 4  # cache.py:45 (accounting only)
# arena rows of a backend built by the reference-signature make_cache (which
# does not name a capacity): a desk-scale session; pass max_len= for more
DEFAULT_MAX_LEN = 8192
HEAD_DIM = 128
ROPE_THETA = 10000.0
TOKEN, CHANNEL = 0, 1
# fused decode kernel: "auto" (the V-absorbed kernel when the workload has enough
# 256-token tiles, else the unabsorbed one), "absorbed" or "unabsorbed"; read
# when a backend is constructed
FUSED_KERNEL = "auto"


# ---------------------------------------------------------------------------
# Policy (cache.py:70-121)
# ---------------------------------------------------------------------------


@dataclass
class LayerPolicy:
    """Per-layer bit widths plus the cross-layer base/prefix structure."""

    bits: list[int]
    base_layers: int = 3
    high_precision_prefix: int = 3

    def __post_init__(self):
        if self.base_layers > self.high_precision_prefix:
            raise ConfigError("base_layers must not exceed high_precision_prefix")

    @classmethod
    def for_bits(cls, bits: int, n_layers: int, prefix: int = 3, prefix_bits: int = 4):
        """Uniform ``bits`` with the leading layers kept at 4-bit (cache.py:89-112)."""
        if bits == 16:
            return cls([16] * n_layers, base_layers=min(prefix, n_layers))
        per_layer = [max(bits, prefix_bits) if i < prefix else bits for i in range(n_layers)]
        return cls(per_layer, base_layers=min(prefix, n_layers),
                   high_precision_prefix=min(prefix, n_layers))

    @classmethod
    def uniform(cls, bits: int, n_layers: int):
        n = min(3, n_layers)  # cache.py:114-118
        return cls([bits] * n_layers, base_layers=n, high_precision_prefix=n)

    def bits_for(self, layer: int) -> int:
        return self.bits[layer]


# ---------------------------------------------------------------------------
# Weights and shared device tables
# ---------------------------------------------------------------------------


@dataclass
class LayerWeights:
    """K/V projections of one layer on the device (x @ W convention).

    ``w_k``/``w_v``: [d, kv_width]. For ``xq-gqa`` the offline SVD factors
    (linalg.py:103-126): ``u_k``/``u_v`` [d, r] and ``fused_k``/``fused_v``
    [r, r] (= diag(sigma) B^T). Arranged fp16 copies for the fused kernel are
    built lazily and cached.
    """

    w_k: torch.Tensor | None = None
    w_v: torch.Tensor | None = None
    u_k: torch.Tensor | None = None
    u_v: torch.Tensor | None = None
    fused_k: torch.Tensor | None = None
    fused_v: torch.Tensor | None = None
    u_kv: torch.Tensor | None = None      # xq-cl-gqa: shared K|V subspace, d x 2*kv_width
    fused_kv: torch.Tensor | None = None  # xq-cl-gqa: diag(sigma) B^T, 2*kv_width x 2*kv_width
    _cache: dict = field(default_factory=dict, repr=False)

    def arranged(self, key, a_mode_k, bits_k, a_mode_v, bits_v, wk, wv) -> torch.Tensor:
        if key not in self._cache:
            kdim, width = wk.shape
            if width % HEAD_DIM:
                raise ShapeError(f"kv width {width} not a multiple of {HEAD_DIM}")
            n_kv = width // HEAD_DIM
            out = torch.empty((n_kv, 256, kdim), dtype=torch.float16, device=wk.device)
            wk_c, wv_c = wk.contiguous(), wv.contiguous()
            N.call("xq_arrange_weights", N.ptr(wk_c), N.ptr(wv_c), _dtype_code(wk_c), kdim, n_kv,
                   a_mode_k, bits_k, a_mode_v, bits_v, N.ptr(out), N.stream_of(wk.device))
            self._cache[key] = out
        return self._cache[key]

    def arranged_absorbed(self, key, a_mode_k, bits_k, a_mode_v, bits_v, wk, wv):
        """(W_k rows for the K passes, W_v [n_kv, kdim, 128]) of the V-absorbed kernel."""
        key = ("absorbed",) + tuple(key)
        if key not in self._cache:
            kdim, width = wk.shape
            if width % HEAD_DIM:
                raise ShapeError(f"kv width {width} not a multiple of {HEAD_DIM}")
            n_kv = width // HEAD_DIM
            wk_out = torch.empty(((n_kv + 3) // 4 * 512, kdim), dtype=torch.float16,
                                 device=wk.device)
            wv_out = torch.empty((n_kv, kdim, HEAD_DIM), dtype=torch.float16, device=wk.device)
            wk_c, wv_c = wk.contiguous(), wv.contiguous()
            N.call("xq_arrange_weights_absorbed", N.ptr(wk_c), N.ptr(wv_c), _dtype_code(wk_c), kdim,
                   n_kv, a_mode_k, bits_k, a_mode_v, bits_v, N.ptr(wk_out), N.ptr(wv_out),
                   N.stream_of(wk.device))
            self._cache[key] = (wk_out, wv_out)
        return self._cache[key]

    def f32(self, name: str) -> torch.Tensor:
        key = ("f32", name)
        if key not in self._cache:
            self._cache[key] = getattr(self, name).float().contiguous()
        return self._cache[key]


_T16: dict = {}


def _t16(w: torch.Tensor) -> torch.Tensor:
    """fp16 W^T (K-major [N, K] rows) of a [K, N] projection, the remat GEMM's B
    operand; built once per weight tensor (keyed by storage, dropped with it)."""
    import weakref

    key = (w.data_ptr(), tuple(w.shape), w.dtype)
    hit = _T16.get(key)
    if hit is not None and hit[0]() is not None:
        return hit[1]
    t = w.t().to(torch.float16).contiguous()
    try:
        ref = weakref.ref(w, lambda _r, k=key: _T16.pop(k, None))
    except TypeError:
        return t
    _T16[key] = (ref, t)
    return t


def _dtype_code(t: torch.Tensor) -> int:
    return {torch.float32: N.F32, torch.bfloat16: N.BF16, torch.float16: N.F16,
            torch.float64: N.F64}[t.dtype]


_ROPE: dict = {}
_SCRATCH: dict = {}
_REC: dict = {}


def _rec_rows(device, rows: int, width: int) -> torch.Tensor:
    """Per-device fp16 staging rows [rows, width] of the xq-cl-gqa accumulator GEMM
    (zero-initialised, so rows never written hold finite values; shared by the layers)."""
    device = torch.device(device)
    key = (device.index if device.index is not None else torch.cuda.current_device(), width)
    cur = _REC.get(key)
    if cur is None or cur.shape[0] < rows:
        _REC[key] = cur = torch.zeros((rows, width), dtype=torch.float16, device=device)
    return cur[:rows]


def _scratch(device, nbytes: int) -> torch.Tensor:
    """Per-device reusable workspace of the fused kernels' split partials
    (launches on one stream are ordered, so every layer can share it)."""
    device = torch.device(device)
    key = device.index if device.index is not None else torch.cuda.current_device()
    cur = _SCRATCH.get(key)
    if cur is None or cur.numel() * 4 < nbytes:
        _SCRATCH[key] = cur = torch.empty(nbytes // 4 + 1, dtype=torch.float32, device=device)
    return cur


def _rope(n_pos: int, device, j_major: int) -> torch.Tensor:
    device = torch.device(device)
    key = (device.index if device.index is not None else torch.cuda.current_device(), j_major)
    cur = _ROPE.get(key)
    have = (cur.shape[1] // 2 if j_major else cur.shape[0]) if cur is not None else 0
    if have < n_pos:
        n = max(1024, 1 << math.ceil(math.log2(max(n_pos, 1))))
        shape = (HEAD_DIM // 2, 2 * n) if j_major else (n, HEAD_DIM)
        t = torch.empty(shape, dtype=torch.float32, device=device)
        N.call("xq_rope_table", N.ptr(t), n, HEAD_DIM, ROPE_THETA, j_major, N.stream_of(device))
        _ROPE[key] = cur = t
    return cur


def _rope_rows(m: torch.Tensor, pos0: int, device) -> torch.Tensor:
    """RoPE (linalg.py:58-95) of rows m [n, heads*128] at positions pos0..pos0+n-1."""
    n = m.shape[0]
    rope = rope_table(pos0 + n, device)
    cos, sin = rope[pos0:pos0 + n, 0::2], rope[pos0:pos0 + n, 1::2]
    mm = m.view(n, -1, HEAD_DIM // 2, 2)
    e, o = mm[..., 0], mm[..., 1]
    c, s = cos[:, None, :], sin[:, None, :]
    return torch.stack([e * c - o * s, e * s + o * c], dim=-1).view(n, -1)


def rope_table(n_pos: int, device) -> torch.Tensor:
    """cos/sin table [n_pos, 64] float2 (angle formed in float64, linalg.py:84-88)."""
    return _rope(n_pos, device, 0)


def rope_table_t(n_pos: int, device) -> torch.Tensor:
    """Frequency-major cos/sin table [64, n] float2 (n >= n_pos) for the fused kernel."""
    return _rope(n_pos, device, 1)


class Accumulator:
    """XQuant-CL running reconstruction (cache.py:124-146) on the device.

    Two parts with two jobs:

    * the remat operand of the delta layers, for every cached token: ``x16``
      (fp16 [n_slots, L_max, d]) and, with precision "fp32", ``x_hat`` (float32).
      It is rebuilt every step from the arenas (the base layer re-seeds it,
      model.py:228) by the accumulate kernel;
    * the accumulator at the tokens being appended, in float64 like the
      reference's: ``row64`` [n_slots, d] at decode, and per prefilled slot a
      [n, d] block (``prefill_rows``). The quantize kernel forms each delta
      against it and adds the float64 reconstruction of the codes it just wrote
      (``xq_quantize_rows_cl``), so delta codes are bit-exact with the
      reference's whatever precision the remat operand is stored in.
    """

    def __init__(self, n_slots: int | None = None, max_len: int | None = None,
                 width: int | None = None, device="cuda", precision="fp32", *,
                 accounting_bits: int = DEFAULT_ACCUMULATOR_BITS):
        """precision "fp16": the fp16 copy is the accumulator (``x_hat`` is None),
        which halves the per-layer accumulate traffic twice over (xq-cl-mha
        only; the reference charges the accumulator 4 bits, cache.py:45).

        ``Accumulator()`` (the reference's call, cache.py:124-133) defers the
        device arrays to the first backend that uses it, which sizes them."""
        if precision not in ("fp32", "fp16"):
            raise ConfigError(f"accumulator precision {precision!r}")
        self.precision = precision
        self.accounting_bits = accounting_bits
        self.width = width
        self.x_hat = self.x16 = self.row64 = None
        self._prefill64: dict = {}
        self.seeded = False
        # an xq-cl-mha delta layer's accumulate deferred to its fused decode launch
        # (xq_decode_attend_absorbed_cl): (backend, lens, max_len); settle() runs it
        # standalone when anything else needs the remat operand first
        self.pending = None
        if n_slots is not None:
            if max_len is None or width is None:
                raise ConfigError("Accumulator needs n_slots, max_len and width together")
            self._allocate(n_slots, max_len, width, torch.device(device))

    def _allocate(self, n_slots, max_len, width, device):
        self.n_slots, self.L, self.width = n_slots, max_len, width
        self.x_hat = (torch.zeros((n_slots, max_len, width), dtype=torch.float32, device=device)
                      if self.precision == "fp32" else None)
        self.x16 = torch.zeros((n_slots, max_len, width), dtype=torch.float16, device=device)
        self.row64 = torch.zeros((n_slots, width), dtype=torch.float64, device=device)

    def ensure(self, n_slots: int, max_len: int, width: int, device) -> "Accumulator":
        """Size a deferred accumulator for a backend (or check an allocated one)."""
        if self.x16 is None:
            self._allocate(n_slots, max_len, width, torch.device(device))
        elif (self.x16.shape[0] < n_slots or self.x16.shape[1] < max_len
              or self.x16.shape[2] != width):
            raise ShapeError(f"accumulator {tuple(self.x16.shape)} too small for "
                             f"{n_slots} slots x {max_len} rows x {width}")
        return self

    # -- the reference's direct API (cache.py:135-146), one sequence ----------
    def seed(self, x) -> None:
        """acc = x (rows 0..n-1 of slot 0; float64 at the rows, fp16/fp32 operand)."""
        x = torch.as_tensor(x, dtype=torch.float64)
        x = x.reshape(-1, x.shape[-1])
        if self.x16 is None:
            self._allocate(1, max(x.shape[0], DEFAULT_MAX_LEN), x.shape[1],
                           torch.device("cuda", torch.cuda.current_device()))
        x = x.to(self.x16.device)
        n = x.shape[0]
        self._prefill64[0] = x.clone()
        self.row64[0] = x[-1]
        self.x16[0, :n] = x.to(torch.float16)
        if self.x_hat is not None:
            self.x_hat[0, :n] = x.float()
        self._n_direct = n
        self.seeded = True

    def add(self, delta) -> None:
        """acc += delta (same shape as the seed, cache.py:139-146)."""
        if not self.seeded:
            raise UsageError("accumulator used before the base layer seeded it")
        delta = torch.as_tensor(delta, dtype=torch.float64).to(self.x16.device)
        delta = delta.reshape(-1, delta.shape[-1])
        n = getattr(self, "_n_direct", None)
        if n is None or delta.shape[0] != n or delta.shape[1] != self.width:
            raise ShapeError(f"accumulator shape {(n, self.width)} vs update {tuple(delta.shape)}")
        rows = self._prefill64[0] + delta
        self.seed(rows)

    def assign_rows(self, rows16: torch.Tensor, n: int, slot: int | None = None) -> None:
        """acc = the rows themselves (a 16-bit layer: delta = x - acc is kept exactly,
        so acc + delta = x): rows16 [n_slots, >= n, d] fp16 (or [>= n, d] for ``slot``)."""
        self.settle()  # a deferred update of the previous layer would land on top
        if slot is None:
            self.x16[:, :n] = rows16[:, :n]
            if self.x_hat is not None:
                self.x_hat[:, :n] = rows16[:, :n]
        else:
            self.x16[slot, :n] = rows16[:n]
            if self.x_hat is not None:
                self.x_hat[slot, :n] = rows16[:n]
        self.seeded = True

    def settle(self) -> None:
        """Apply a deferred delta-layer accumulate (the remat operand is then current)."""
        if self.pending is not None:
            backend, lens, max_len = self.pending
            self.pending = None
            backend._accumulate(self, False, max_len, lens)

    def rows(self, slot, n) -> torch.Tensor:
        """float32 view/copy of the accumulator rows 0..n-1 of a slot."""
        self.settle()
        return self.x_hat[slot, :n] if self.x_hat is not None else self.x16[slot, :n].float()

    def prefill_rows(self, slot: int, n: int, seed: bool) -> torch.Tensor:
        """The float64 accumulator of a slot's n prefilled tokens (allocated by the
        seeding base layer, reused by the delta layers of the same prefill)."""
        cur = self._prefill64.get(slot)
        if seed or cur is None or cur.shape[0] != n:
            if not seed:
                raise UsageError("accumulator used before the base layer seeded it")
            cur = torch.empty((n, self.width), dtype=torch.float64, device=self.x16.device)
            self._prefill64[slot] = cur
            self._n_direct = None
        return cur

    def release_prefill(self, slot: int | None = None) -> None:
        """Drop the float64 prefill blocks (all slots, or one)."""
        if slot is None:
            self._prefill64.clear()
        else:
            self._prefill64.pop(slot, None)


# ---------------------------------------------------------------------------
# Packed payload stream (cache.py:154-230 on the device)
# ---------------------------------------------------------------------------


class PackedStream:
    """Quantized payload arena of one layer for ``n_slots`` sequences.

    Per-token: codes [n_slots*L_max, row_bytes] + half2 params per group.
    Per-channel (always buffered, cache.py:173): codes + planar params per
    128-token group, plus an fp32 residual buffer [n_slots, G, width] holding
    the rows of the current incomplete group (cache.py:203-208, 218-221).
    """

    def __init__(self, bits, axis, width, group_size, n_slots, max_len, device, resid_f64=False,
                 buffered=False, keep_first=False):
        """``resid_f64``: per-channel only -- keep the residual rows in float64 as
        well (quantized from float64, like the reference); ``resid`` is then
        their float32 mirror read by the fused kernel."""
        if bits not in (2, 3, 4, 8):
            raise ConfigError(f"packed stream bits must be 2/3/4/8, got {bits}")
        if axis == CHANNEL and max_len % group_size:
            raise ConfigError("per-channel arena needs max_len % group_size == 0")
        self.bits, self.axis, self.width, self.g = bits, axis, width, group_size
        self.n_slots, self.L = n_slots, max_len
        self.row_bytes = (width * bits + 63) // 64 * 8
        self.codes = torch.zeros((n_slots * max_len, self.row_bytes), dtype=torch.uint8, device=device)
        if axis == TOKEN:
            ng = -(-width // group_size)
            ngp = -(-ng // 4) * 4  # row stride padded to 16-byte quads (include/xquant.h)
            self.params = torch.zeros((n_slots * max_len, ngp, 2), dtype=torch.float16, device=device)
            if buffered:  # per-token with a residual buffer (kvq V, cache.py:340-341)
                self.resid = torch.zeros((n_slots, group_size, width), dtype=torch.float32,
                                         device=device)
                self.n_flushed = np.zeros(n_slots, dtype=np.int64)
                self.nflushed_dev = torch.zeros(n_slots, dtype=torch.int32, device=device)
        else:
            self.params = torch.zeros((n_slots * max_len // group_size, 2, width),
                                      dtype=torch.float16, device=device)
            self.resid = torch.zeros((n_slots, group_size, width), dtype=torch.float32, device=device)
            self.resid64 = (torch.zeros((n_slots, group_size, width), dtype=torch.float64, device=device)
                            if resid_f64 else None)
            # fp16 outlier channel (cache.py:406-411): channel 0 of the flushed rows
            # kept in full precision (float32 per arena row) beside the codes
            self.first = (torch.zeros(n_slots * max_len, dtype=torch.float32, device=device)
                          if keep_first else None)
            self.n_flushed = np.zeros(n_slots, dtype=np.int64)
            self.nflushed_dev = torch.zeros(n_slots, dtype=torch.int32, device=device)
        self.flag = torch.zeros(1, dtype=torch.int32, device=device)

    def nbytes(self) -> dict:
        out = {"codes": self.codes.numel(), "params": self.params.numel() * 2}
        if self.axis == TOKEN and hasattr(self, "resid"):
            out["residual"] = self.resid.numel() * 4
        if self.axis == CHANNEL:
            out["residual"] = self.resid.numel() * 4
            if self.resid64 is not None:
                out["residual_f64"] = self.resid64.numel() * 8
            if self.first is not None:
                out["first_channel_f32"] = self.first.numel() * 4
        return out

    # -- per-token ---------------------------------------------------------
    def append_token_rows_cl(self, x: torch.Tensor, lens_dev: torch.Tensor, acc64: torch.Tensor,
                             seed: bool):
        """XQuant-CL append of one row per slot against / into the float64
        accumulator rows ``acc64`` [n_slots, width] (xq_quantize_rows_cl)."""
        N.call("xq_quantize_rows_cl", N.ptr(x), _dtype_code(x), x.stride(0), x.shape[0], self.width,
               self.bits, self.g, N.ptr(lens_dev), 0, self.L, N.ptr(acc64), 2 if seed else 1,
               N.ptr(self.codes), self.row_bytes, N.ptr(self.params), N.ptr(self.flag),
               N.stream_of(x.device))

    def fill_rows_cl(self, x: torch.Tensor, slot: int, pos0: int, acc64: torch.Tensor, seed: bool):
        """Bulk XQuant-CL quantization of x [n, width] into slot rows pos0.. against /
        into the float64 accumulator block ``acc64`` [n, width]."""
        if x.shape[0] == 0:
            return
        N.call("xq_quantize_rows_cl", N.ptr(x), _dtype_code(x), x.stride(0), x.shape[0], self.width,
               self.bits, self.g, None, slot * self.L + pos0, self.L, N.ptr(acc64),
               2 if seed else 1, N.ptr(self.codes), self.row_bytes, N.ptr(self.params),
               N.ptr(self.flag), N.stream_of(x.device))

    def append_token_rows(self, x: torch.Tensor, lens_dev: torch.Tensor, sub=None, x_eff=None):
        """Quantize one row per slot and store it at position lens[b]-1."""
        N.call("xq_quantize_rows", N.ptr(x), _dtype_code(x), x.stride(0), x.shape[0], self.width,
               self.bits, self.g, N.ptr(lens_dev), 0, self.L, N.ptr(sub), N.ptr(self.codes),
               self.row_bytes, N.ptr(self.params), N.ptr(x_eff), N.ptr(self.flag),
               N.stream_of(x.device))

    def fill_rows(self, x: torch.Tensor, slot: int, pos0: int, sub=None, x_eff=None):
        """Bulk per-token quantization of x [n, width] into slot rows pos0.."""
        if x.shape[0] == 0:
            return
        N.call("xq_quantize_rows", N.ptr(x), _dtype_code(x), x.stride(0), x.shape[0], self.width,
               self.bits, self.g, None, slot * self.L + pos0, self.L, N.ptr(sub),
               N.ptr(self.codes), self.row_bytes, N.ptr(self.params), N.ptr(x_eff),
               N.ptr(self.flag), N.stream_of(x.device))

    def token_bulk(self, slot: int, x: torch.Tensor):
        """Buffered per-token bulk (cache.py:191-201): every row is quantized."""
        self.fill_rows(x.contiguous(), slot, 0)
        self.n_flushed[slot] = x.shape[0]
        self.nflushed_dev[slot] = x.shape[0]

    def token_push(self, x: torch.Tensor, n_tokens: np.ndarray):
        """Buffered per-token push (cache.py:210-221): the row waits in the
        residual buffer; a full buffer of G rows is quantized at once."""
        dev = x.device
        buf_pos = torch.as_tensor(n_tokens - 1 - self.n_flushed, device=dev)
        self.resid[torch.arange(self.n_slots, device=dev), buf_pos] = x.float()
        full = np.nonzero(n_tokens - self.n_flushed >= self.g)[0]
        for s in full:
            self.fill_rows(self.resid[int(s)], int(s), int(self.n_flushed[s]))
            self.n_flushed[s] += self.g
        if len(full):
            self.nflushed_dev.copy_(torch.from_numpy(self.n_flushed.astype(np.int32)))

    # -- per-channel -------------------------------------------------------
    def flush_blocks(self, blocks: torch.Tensor, dst_row0: list[int]):
        dst = torch.tensor(dst_row0, dtype=torch.int64, device=blocks.device)
        if getattr(self, "first", None) is not None:
            rows = dst[:, None] + torch.arange(self.g, device=blocks.device)[None, :]
            self.first[rows.reshape(-1)] = blocks.reshape(-1, self.width)[:, 0].float()
        fn = ("xq_quantize_blocks_per_channel_f64" if blocks.dtype == torch.float64
              else "xq_quantize_blocks_per_channel")
        N.call(fn, N.ptr(blocks), len(dst_row0), self.width,
               self.bits, self.g, N.ptr(dst), N.ptr(self.codes), self.row_bytes,
               N.ptr(self.params), N.ptr(self.flag), N.stream_of(blocks.device))

    def channel_bulk(self, slot: int, lat: torch.Tensor):
        """Per-channel bulk (cache.py:191-208) into an empty slot: whole G-row
        groups are quantized, the tail waits in the residual buffer."""
        g, n = self.g, lat.shape[0]
        n_full = n // g * g
        if self.resid64 is not None:
            lat = lat.double()
        if n_full:
            self.flush_blocks(lat[:n_full].contiguous(), [slot * self.L + i for i in range(0, n_full, g)])
        self.resid[slot, :n - n_full] = lat[n_full:]
        if self.resid64 is not None:
            self.resid64[slot, :n - n_full] = lat[n_full:]
        self.n_flushed[slot] = n_full
        self.nflushed_dev[slot] = n_full

    def channel_push(self, lat: torch.Tensor, n_tokens: np.ndarray):
        """Per-channel push of one row per slot (cache.py:210-221); ``n_tokens``
        counts the rows including this one. Full groups are flushed."""
        dev = lat.device
        buf_pos = torch.as_tensor(n_tokens - 1 - self.n_flushed, device=dev)
        rows = torch.arange(self.n_slots, device=dev)
        self.resid[rows, buf_pos] = lat.float()
        if self.resid64 is not None:
            self.resid64[rows, buf_pos] = lat.double()
        self.flush_full(n_tokens)

    def flush_full(self, n_tokens: np.ndarray):
        """Quantize the residual buffers that hold a whole group (cache.py:218-221)."""
        dev = self.resid.device
        full = np.nonzero(n_tokens - self.n_flushed >= self.g)[0]
        if len(full):
            src = self.resid64 if self.resid64 is not None else self.resid
            blocks = src[torch.as_tensor(full, device=dev)].contiguous()
            self.flush_blocks(blocks, [int(s) * self.L + int(self.n_flushed[s]) for s in full])
            self.n_flushed[full] += self.g
            self.nflushed_dev.copy_(torch.from_numpy(self.n_flushed.astype(np.int32)))

    def channel_reconstruct(self, slot: int, n: int) -> torch.Tensor:
        """float32 [n, width]: dequantized flushed rows + residual rows (cache.py:223-230)."""
        out = torch.empty((n, self.width), dtype=torch.float32, device=self.codes.device)
        nfl = int(self.n_flushed[slot])
        if nfl:
            N.call("xq_dequant_rows", N.ptr(self.codes), self.row_bytes, N.ptr(self.params), CHANNEL,
                   self.bits, self.g, self.width, slot * self.L, nfl, N.ptr(out),
                   N.stream_of(out.device))
        if nfl and self.first is not None:
            out[:nfl, 0] = self.first[slot * self.L:slot * self.L + nfl]
        out[nfl:] = self.resid[slot, :n - nfl]
        return out

    # -- XQT1 on-disk format (quant.py:232-291) ----------------------------
    def _channel_perm(self) -> torch.Tensor:
        """Storage position of each natural channel in the per-channel params
        (the producer order of csrc/xq_layout.cuh)."""
        bs = {2: 16, 3: 32, 4: 8, 8: 4}[self.bits]
        h = bs // 2
        c = np.arange(self.width)
        j = c % bs
        pos = (c // bs) * bs + np.where(j < h, 2 * j, 2 * (j - h) + 1)
        return torch.as_tensor(pos, device=self.codes.device)

    def _packed_rows(self, r0: int, n: int) -> bytes:
        """One LSB-first bit stream over rows r0..r0+n (row-major elements)."""
        rows = self.codes[r0:r0 + n]
        if (self.width * self.bits) % 64 == 0:  # arena rows are u64-aligned: the bytes concatenate
            return rows.contiguous().cpu().numpy().tobytes()
        dev = self.codes.device
        flat = torch.empty((n, self.width), dtype=torch.uint8, device=dev)
        for i in range(n):
            N.call("xq_unpack_codes", N.ptr(rows[i]), self.bits, self.width, N.ptr(flat[i]),
                   N.stream_of(dev))
        words = torch.empty(((n * self.width * self.bits + 63) // 64,), dtype=torch.int64, device=dev)
        N.call("xq_pack_codes", N.ptr(flat), n * self.width, self.bits, N.ptr(words), N.stream_of(dev))
        return words.cpu().numpy().tobytes()

    def export_xqt1(self, slot: int, n_rows: int) -> bytes:
        """XQT1 dump (quant.py:232-254) of one slot's quantized rows: the header,
        the scale and zero-point grids (float64 of the stored fp16 values) and the
        packed codes, which are byte-identical to the reference's for the same
        codes. Per-token: rows 0..n_rows-1. Per-channel: the flushed rows (whole
        groups; the residual buffer is not part of the quantized tensor)."""
        import struct

        r0 = slot * self.L
        if self.axis == TOKEN:
            n = int(n_rows)
            ng = -(-self.width // self.g)
            p = self.params[r0:r0 + n, :ng].double()
            sc, zp = p[..., 0], p[..., 1]
        else:
            n = int(self.n_flushed[slot])
            perm = self._channel_perm()
            p = self.params[r0 // self.g:(r0 + n) // self.g].double()  # [groups, 2, width]
            sc, zp = p[:, 0][:, perm], p[:, 1][:, perm]
        head = b"XQT1" + struct.pack("<5i", n, self.width, self.bits, self.axis, self.g)
        body = sc.contiguous().cpu().numpy().astype("<f8").tobytes() + \
            zp.contiguous().cpu().numpy().astype("<f8").tobytes()
        return head + body + self._packed_rows(r0, n)

    def check_finite(self):
        """Raise DataError if any quantized input was NaN/Inf (quant.py:114-115).

        Synchronises; the decode engine calls it once per step, not per layer."""
        if int(self.flag.item()):
            self.flag.zero_()
            raise DataError("input contains NaN or Inf")


class RawRows:
    """16-bit pass-through payload (quant.py:117-118: a bits=16 QuantizedTensor keeps
    the raw rows; ``_Stream`` never buffers or quantizes them): fp16 rows
    [n_slots * L_max, width], row ``slot * L_max + t`` = token t. The fused kernels
    read them as their fp16-row A operand (XQ_A_F16_ROWS)."""

    bits = 16

    def __init__(self, width: int, n_slots: int, max_len: int, device):
        self.width, self.n_slots, self.L = width, n_slots, max_len
        self.rows = torch.zeros((n_slots * max_len, width), dtype=torch.float16, device=device)

    def fill(self, x: torch.Tensor, slot: int, pos0: int = 0):
        r0 = slot * self.L + pos0
        self.rows[r0:r0 + x.shape[0]] = x.to(torch.float16)

    def append(self, x: torch.Tensor, lens_dev: torch.Tensor):
        """One row per slot at position lens[b]-1."""
        idx = torch.arange(self.n_slots, device=x.device) * self.L + lens_dev.long() - 1
        self.rows[idx] = x.to(torch.float16)

    def slot_rows(self, slot: int, n: int) -> torch.Tensor:
        return self.rows[slot * self.L:slot * self.L + n]

    def slots_view(self) -> torch.Tensor:
        return self.rows.view(self.n_slots, self.L, self.width)

    def nbytes(self) -> dict:
        return {"rows_f16": self.rows.numel() * 2}


# ---------------------------------------------------------------------------
# Backends
# ---------------------------------------------------------------------------


class CacheBackend:
    """Common interface (cache.py:238-299) with a slot dimension."""

    variant = ""
    needs_accumulator = False

    def __init__(self, layer_index: int, policy: LayerPolicy, head_dim: int,
                 group_size: int = DEFAULT_GROUP_SIZE, *, n_slots: int = 1, max_len: int = 4096,
                 hidden_dim: int | None = None, n_heads: int | None = None, kv_group: int = 1,
                 n_heads_total: int | None = None, device="cuda", exact: bool = False):
        """``n_heads`` is the number of query heads this backend serves; with
        KV-head-group sharding (parallel.py) it is a slice of
        ``n_heads_total`` and the weights passed in are column-sliced.
        ``exact``: float64 inputs keep float64 arithmetic up to quantization
        where the variant allows it (xq-gqa latents as float64 GEMMs with a
        float64 residual buffer), as the reference-signature make_cache sets."""
        if head_dim != HEAD_DIM:
            raise ConfigError(f"the B200 kernels are specialised for head_dim {HEAD_DIM}, got {head_dim}")
        if hidden_dim is None or n_heads is None:
            raise ConfigError("hidden_dim and n_heads are required (device arenas are preallocated)")
        total = n_heads_total or n_heads
        if hidden_dim != total * head_dim or n_heads % kv_group or total % kv_group:
            raise ConfigError("hidden_dim must equal n_heads*head_dim and n_heads % kv_group == 0")
        self.layer_index = layer_index
        self.policy = policy
        self.exact = exact
        self.head_dim = head_dim
        self.group_size = group_size
        self.bits = policy.bits_for(layer_index)
        self.n_slots, self.L = n_slots, max_len
        self.d, self.n_heads, self.g = hidden_dim, n_heads, kv_group
        self.latent = hidden_dim // kv_group  # full K/V width = SVD latent rank r (xq-gqa)
        self.n_kv = n_heads // kv_group       # KV heads served here
        self.kvw = self.n_kv * head_dim       # K/V width served here
        self.device = torch.device(device)
        self.n_tokens = np.zeros(n_slots, dtype=np.int64)
        self.lens_dev = torch.zeros(n_slots, dtype=torch.int32, device=self.device)
        # V absorption (xq_absorb.cu): exact reassociation p.(x W_v) = (p.x) W_v.
        # FUSED_KERNEL "auto" picks by workload size; the tests pin both kernels
        self.absorb = {"auto": "auto", "absorbed": True, "unabsorbed": False}[FUSED_KERNEL]
        # KV-head-group sharding (decode.Decoder with parallel.PeerHeadGather): device
        # addresses the absorbed kernel's projection stores to, set around one _attend
        # call; peer_stored tells the decoder whether that launch did the gather
        self.peer_outs: list[int] | None = None
        self.peer_stored = False

    # -- interface ---------------------------------------------------------
    def _adopt(self, weights, acc):
        """Accept the reference's LayerWeights / Accumulator (cache.py:49-67,
        124-146) as well as this module's, and check the accumulator rule."""
        weights = as_layer_weights(weights, self.device)
        if acc is not None:
            acc = device_accumulator(acc).ensure(self.n_slots, self.L, self.d, self.device)
        self._check_acc(acc)
        return weights, acc

    def prefill(self, x, weights: LayerWeights, acc: Accumulator | None = None, slot=None):
        """Bulk-cache a prefix: x [n_slots, n, d] (all slots) or [n, d] for ``slot``."""
        weights, acc = self._adopt(weights, acc)
        slots, xs = self._split_slots(x, slot)
        for s, xx in zip(slots, xs):
            if self.n_tokens[s]:
                raise UsageError("prefill on a non-empty cache")  # cache.py:258-259
            if xx.shape[0] > self.L:
                raise ShapeError(f"prefill of {xx.shape[0]} tokens exceeds max_len {self.L}")
            self._prefill(s, xx, weights, acc)
            self.n_tokens[s] = xx.shape[0]
        self._sync_lens()

    def decode_append(self, x_token, weights: LayerWeights, acc: Accumulator | None = None):
        """Append one token per slot: x_token [n_slots, d] (cache.py:264-269)."""
        weights, acc = self._adopt(weights, acc)
        x_token = self._as_rows(x_token)
        if x_token.shape[0] != self.n_slots:
            raise ShapeError(f"expected {self.n_slots} rows, got {x_token.shape[0]}")
        if np.any(self.n_tokens >= self.L):
            raise ShapeError("cache full")
        self.n_tokens += 1
        self._sync_lens()
        self._decode(x_token, weights, acc, self.lens_dev)

    def rematerialize(self, weights: LayerWeights, positions, acc: Accumulator | None = None,
                      slot: int = 0):
        """(K, V) float32 of one slot (cache.py:271-281), SIMT parity path."""
        n = int(self.n_tokens[slot])
        if n == 0:
            raise UsageError("rematerialize on an empty cache")
        positions = np.asarray(positions).reshape(-1)
        if positions.shape[0] != n:
            raise ShapeError(f"got {positions.shape[0]} positions for {n} tokens")
        if not np.array_equal(positions, np.arange(n)):
            raise ShapeError("positions must be 0..n-1 (the cache's own timeline)")
        weights, acc = self._adopt(weights, acc)
        return self._rematerialize(weights, acc, slot, n)

    def decode_attend(self, q_pre, weights: LayerWeights, acc: Accumulator | None = None,
                      tiles_per_chunk: int | None = None):
        """Fused remat + attention for the newest token of every slot.

        q_pre: [n_slots, n_heads, 128] (or [n_slots, n_heads*128]) float32,
        before RoPE; it is rotated to position n_tokens-1 in the kernel
        (model.py:234). Returns float32 [n_slots, n_heads, 128].
        """
        weights, acc = self._adopt(weights, acc)
        if np.any(self.n_tokens == 0):
            raise UsageError("decode_attend on an empty cache")
        q = q_pre.reshape(self.n_slots, self.n_heads, self.head_dim).float().contiguous()
        out = torch.empty_like(q)
        self._attend(q, weights, acc, self.lens_dev, int(self.n_tokens.max()), out, tiles_per_chunk)
        return out

    def prefill_attend(self, x, q_pre, weights: LayerWeights, acc: Accumulator | None = None,
                       slot: int = 0):
        """Prefill of one slot and its causal attention (the attention block of
        ``_Session.prefill``, model.py:205-221): cache the prompt x [n, d]
        (``prefill``), rebuild K/V of all n positions from the cache just written
        (``rematerialize``, cache.py:271-281), rotate q_pre [n, n_heads*128] to
        positions 0..n-1 and attend causally (model.py:150-182).

        Prefill is GEMM-shaped: K/V of all n positions are materialized in fp16 by
        the tcgen05 remat GEMM (xq_gemm_f16, RoPE fused into the K epilogue) from
        fp16 rows of the cache, and a flash-attention kernel (xq_prefill_attend)
        attends causally. Returns float32 [n, n_heads, 128]."""
        weights, acc = self._adopt(weights, acc)
        x = torch.as_tensor(x, device=self.device)
        n = x.shape[0]
        self.prefill(x, weights, acc, slot=slot)
        k, v = self._prefill_kv(weights, acc, slot, n)  # fp16 (bf16 baseline), K rotated, [n, kvw]
        qf = q_pre.reshape(n, self.n_heads * self.head_dim).float().contiguous()
        q = torch.empty((n, self.n_heads * self.head_dim), dtype=k.dtype, device=self.device)
        rope = rope_table(n, self.device)
        dt = _dtype_code(k)
        N.call("xq_rope_rows", N.ptr(qf), N.F32, qf.stride(0), n, qf.shape[1], N.ptr(rope),
               rope.shape[0], 0, N.ptr(q), dt, q.stride(0), N.stream_of(self.device))
        out = torch.empty((n, self.n_heads, self.head_dim), dtype=torch.float32, device=self.device)
        N.call("xq_prefill_attend", N.ptr(q), N.ptr(k), N.ptr(v), dt, n, self.n_heads, self.g,
               q.stride(0), k.stride(0), 1.0 / math.sqrt(self.head_dim), N.ptr(out),
               self.n_heads * self.head_dim, N.stream_of(self.device))
        return out

    def _prefill_kv(self, weights, acc, slot, n):  # pragma: no cover
        raise NotImplementedError

    def _dequant_rows(self, stream, slot, n):
        """float32 [n, width] of a per-token stream's rows of one slot."""
        out = torch.empty((n, stream.width), dtype=torch.float32, device=self.device)
        N.call("xq_dequant_rows", N.ptr(stream.codes), stream.row_bytes, N.ptr(stream.params), TOKEN,
               stream.bits, stream.g, stream.width, slot * self.L, n, N.ptr(out),
               N.stream_of(self.device))
        return out

    def _rows16(self, stream, slot, n, out=None):
        """fp16 [n, width] operand rows of one slot: dequantized codes, then (buffered
        streams) the residual rows (cache.py:223-230); into ``out`` when given."""
        if out is None:
            out = torch.empty((n, stream.width), dtype=torch.float16, device=self.device)
        buffered = getattr(stream, "n_flushed", None) is not None
        nfl = min(int(stream.n_flushed[slot]), n) if buffered else n
        resid = stream.resid[slot] if nfl < n else None
        N.call("xq_dequant_rows_f16", N.ptr(stream.codes), stream.row_bytes, N.ptr(stream.params),
               stream.axis, stream.bits, stream.g, stream.width, slot * self.L, nfl, N.ptr(resid),
               n, N.ptr(out), out.stride(0), N.stream_of(self.device))
        if stream.axis == CHANNEL and stream.first is not None and nfl:
            out[:nfl, 0] = stream.first[slot * self.L:slot * self.L + nfl].half()
        return out

    def _gemm(self, a, w_t, epi, n):
        """fp16 [n, N] = a [n, K] @ w_t[N, K]^T on tcgen05; epi 1 rotates the rows."""
        out = torch.empty((n, w_t.shape[0]), dtype=torch.float16, device=self.device)
        rope = rope_table(n, self.device) if epi == 1 else None
        N.call("xq_gemm_f16", N.ptr(a), a.stride(0), N.ptr(w_t), w_t.stride(0), N.ptr(out),
               out.stride(0), n, w_t.shape[0], a.shape[1], epi, N.ptr(rope),
               rope.shape[0] if rope is not None else 0, 0, N.stream_of(self.device))
        return out

    def _kv_from(self, a_k, a_v, wk, wv, n):
        """K (rotated to 0..n-1) and V in fp16 from fp16 operand rows and [K, N] weights."""
        return self._gemm(a_k, _t16(wk), 1, n), self._gemm(a_v, _t16(wv), 0, n)

    # -- helpers -------------------------------------------------------------
    def _sync_lens(self):
        self.lens_dev.copy_(torch.from_numpy(self.n_tokens.astype(np.int32)), non_blocking=False)

    def _as_rows(self, x):
        x = torch.as_tensor(x, device=self.device)
        if x.dim() == 1:
            x = x[None]
        if x.dtype == torch.float64:
            x = x.contiguous()
        return x

    def _split_slots(self, x, slot):
        x = torch.as_tensor(x, device=self.device)
        if slot is not None:
            if x.dim() != 2:
                raise ShapeError("prefill with slot= expects [n, d]")
            return [slot], [x]
        if x.dim() == 2 and self.n_slots == 1:
            return [0], [x]
        if x.dim() != 3 or x.shape[0] != self.n_slots:
            raise ShapeError(f"prefill expects [{self.n_slots}, n, d]")
        return list(range(self.n_slots)), [x[s] for s in range(self.n_slots)]

    def _check_acc(self, acc):
        if self.needs_accumulator and acc is None:
            raise UsageError(f"{self.variant} requires an accumulator")  # cache.py:294-296

    def _workspace(self, max_len, group, tpc):
        nbytes = N.lib.xq_decode_workspace_bytes(self.n_slots, max_len, self.n_kv, group, tpc)
        return torch.empty(nbytes // 4 + 1, dtype=torch.float32, device=self.device), nbytes

    def _fused(self, ak_mode, ak_src, ak_params, ak_resid, ak_nfl, ak_bits, ak_rb, av_mode,
               av_src, av_params, av_bits, av_rb, kdim, w_spec, weights, group, q, lens, max_len,
               out, tpc, force_absorbed=False, ak_first=None):
        """One fused decode launch. ``w_spec`` = (key, a_mode_k, bits_k, a_mode_v, bits_v,
        W_k, W_v) names the projection pair and the A operands that feed it."""
        key, mk, bk, mv, bv, wk, wv = w_spec
        rope = rope_table_t(max_len, self.device)
        if force_absorbed or self._use_absorbed(kdim, max_len):
            wk_arr, wv_arr = weights.arranged_absorbed(key, mk, bk, mv, bv, wk, wv)
            nbytes = N.lib.xq_absorbed_workspace_bytes(self.n_slots, max_len, self.n_kv * group, kdim)
            ws = _scratch(self.device, nbytes)
            args = (ak_mode, N.ptr(ak_src), N.ptr(ak_params), N.ptr(ak_resid), N.ptr(ak_nfl),
                    N.ptr(ak_first), ak_bits, ak_rb, av_mode, N.ptr(av_src), N.ptr(av_params), av_bits,
                    av_rb, self.group_size, self.L, kdim, N.ptr(lens), self.n_slots, max_len,
                    N.ptr(wk_arr), N.ptr(wv_arr), self.n_kv, group, N.ptr(q), N.ptr(rope),
                    rope.shape[1] // 2, 1.0 / math.sqrt(HEAD_DIM), N.ptr(ws), nbytes)
            peers = self.peer_outs
            if peers:  # head-sharded engine: the projection stores into every rank's gather slot
                arr = (ctypes.c_void_p * len(peers))(*peers)
                N.call("xq_decode_attend_absorbed_peers", *args, ctypes.cast(arr, ctypes.c_void_p),
                       len(peers), N.stream_of(self.device))
                self.peer_stored = True
                return
            N.call("xq_decode_attend_absorbed", *args, N.ptr(out), N.stream_of(self.device))
            return
        w_arr = weights.arranged(key, mk, bk, mv, bv, wk, wv)
        tpc = tpc or default_tiles_per_chunk(self.n_slots, max_len, self.n_kv)
        ws, nbytes = self._workspace(max_len, group, tpc)
        N.call("xq_decode_attend", ak_mode, N.ptr(ak_src), N.ptr(ak_params), N.ptr(ak_resid),
               N.ptr(ak_nfl), ak_bits, ak_rb, av_mode, N.ptr(av_src), N.ptr(av_params), av_bits,
               av_rb, self.group_size, self.L, kdim, N.ptr(lens), self.n_slots, max_len,
               N.ptr(w_arr), self.n_kv, group, N.ptr(q), N.ptr(rope), rope.shape[1] // 2,
               1.0 / math.sqrt(HEAD_DIM), tpc, N.ptr(ws), nbytes, N.ptr(out),
               N.stream_of(self.device))

    def _use_absorbed(self, kdim: int, max_len: int) -> bool:
        if self.group_size != DEFAULT_GROUP_SIZE:
            return kdim % 256 == 0  # the unabsorbed kernel takes 128-channel groups only
        if kdim % 256 or self.absorb is False:
            return False
        return self.absorb is True or self._absorb_pays(max_len)

    def _absorb_pays(self, max_len: int) -> bool:
        """The absorbed kernel's work unit is a whole 256-token tile with all heads;
        with fewer units than half the CTA pairs (e.g. one short sequence) the
        unabsorbed kernel, which also splits by KV head, keeps more SMs busy."""
        units = self.n_slots * max(1, -(-max_len // 256))
        return units >= 37

    def _remat_f32(self, ak_mode, ak_src, ak_params, ak_resid, ak_nfl, ak_bits, ak_rb, av_mode,
                   av_src, av_params, av_bits, av_rb, kdim, wk, wv, slot, n):
        n_out = wk.shape[1]
        k = torch.empty((n, n_out), dtype=torch.float32, device=self.device)
        v = torch.empty((n, n_out), dtype=torch.float32, device=self.device)
        rope = rope_table(n, self.device)
        N.call("xq_remat_f32", ak_mode, N.ptr(ak_src), N.ptr(ak_params), N.ptr(ak_resid), ak_nfl,
               ak_bits, ak_rb, av_mode, N.ptr(av_src), N.ptr(av_params), av_bits, av_rb,
               self.group_size, self.L, kdim, slot, n, N.ptr(wk), N.ptr(wv), n_out, N.ptr(rope),
               N.ptr(k), N.ptr(v), N.stream_of(self.device))
        return k, v

    def memory_bytes(self) -> dict:
        return {}

    # hooks
    def _prefill(self, slot, x, weights, acc):  # pragma: no cover
        raise NotImplementedError

    def _decode(self, x, weights, acc, lens):  # pragma: no cover
        raise NotImplementedError

    def _rematerialize(self, weights, acc, slot, n):  # pragma: no cover
        raise NotImplementedError

    def _attend(self, q, weights, acc, lens, max_len, out, tpc):  # pragma: no cover
        raise NotImplementedError


def default_tiles_per_chunk(n_slots: int, max_len: int, n_kv: int, n_sm: int = 148,
                            max_tiles: int = 2) -> int:
    """Tiles (of 256 tokens, one per CTA pair) per work unit.

    Enough units for >= ~4 waves of CTA pairs, and at most ``max_tiles`` tiles
    per unit: units are ordered KV-head-fastest, so the pairs in flight cover
    only a few token ranges and every head re-reads those codes from L2."""
    n_tiles = max(1, -(-max_len // 256))
    target_units = 2 * n_sm
    per_seq_head = max(1, n_slots * n_kv)
    chunks = max(1, min(n_tiles, -(-target_units // per_seq_head)))
    return max(1, min(max_tiles, -(-n_tiles // chunks)))


class FullPrecisionCache(CacheBackend):
    """``fp16`` baseline (cache.py:302-323): bf16 post-RoPE K/V in HBM."""

    variant = "fp16"

    def __init__(self, *a, **kw):
        super().__init__(*a, **kw)
        shape = (self.n_slots * self.L, self.kvw)
        self.k = torch.zeros(shape, dtype=torch.bfloat16, device=self.device)
        self.v = torch.zeros(shape, dtype=torch.bfloat16, device=self.device)

    def _project(self, x, weights):
        # bf16 GEMM with fp32 accumulation (cuBLAS); K/V are stored in bf16 anyway
        xb = x.to(weights.w_k.dtype)
        return (xb @ weights.w_k).float(), (xb @ weights.w_v).float()

    def _prefill(self, slot, x, weights, acc):
        k, v = self._project(x, weights)
        self._append_rows(k, v, slot, 0)

    def _append_rows(self, k, v, slot, pos0):
        """Bulk append with RoPE at positions pos0.. (torch ops; prefill only)."""
        n = k.shape[0]
        rope = rope_table(pos0 + n, self.device)
        cos = rope[pos0:pos0 + n, 0::2]
        sin = rope[pos0:pos0 + n, 1::2]
        kk = k.view(n, self.n_kv, 64, 2)
        e, o = kk[..., 0], kk[..., 1]
        c, s = cos[:, None, :], sin[:, None, :]
        rot = torch.stack([e * c - o * s, e * s + o * c], dim=-1).view(n, self.kvw)
        base = slot * self.L + pos0
        self.k[base:base + n] = rot.to(torch.bfloat16)
        self.v[base:base + n] = v.to(torch.bfloat16)

    def _decode(self, x, weights, acc, lens):
        k, v = self._project(x, weights)
        rope = rope_table(int(self.n_tokens.max()), self.device)
        N.call("xq_kv_append", N.ptr(k.contiguous()), N.ptr(v.contiguous()), N.ptr(lens),
               self.n_slots, self.n_kv, self.L, N.ptr(rope), N.ptr(self.k), N.ptr(self.v),
               N.stream_of(self.device))

    def _rematerialize(self, weights, acc, slot, n):
        base = slot * self.L
        return self.k[base:base + n].float(), self.v[base:base + n].float()

    def _prefill_kv(self, weights, acc, slot, n):
        base = slot * self.L  # the stored bf16 rows themselves (K already rotated)
        return self.k[base:base + n], self.v[base:base + n]

    def _attend(self, q, weights, acc, lens, max_len, out, tpc):
        chunk = tpc * 128 if tpc else kv_chunk_tokens(self.n_slots, max_len, self.n_kv,
                                                       ctas_per_sm=4 if self.g == 1 else 24)
        nbytes = N.lib.xq_kv_decode_workspace_bytes(self.n_slots, max_len, self.n_kv, self.g, chunk)
        ws = torch.empty(nbytes // 4 + 1, dtype=torch.float32, device=self.device)
        rope = rope_table(max_len, self.device)
        N.call("xq_kv_decode_attend", N.ptr(self.k), N.ptr(self.v), self.L, N.ptr(lens),
               self.n_slots, max_len, self.n_kv, self.g, N.ptr(q), N.ptr(rope),
               1.0 / math.sqrt(HEAD_DIM), chunk, N.ptr(ws), nbytes, N.ptr(out),
               N.stream_of(self.device))

    def memory_bytes(self):
        return {"kv_cache": 2 * self.k.numel() * 2}


def kv_chunk_tokens(n_slots, max_len, n_kv, n_sm=148, ctas_per_sm=4):
    """Tokens per CTA of the fp16-KV flash-decode: >= ~ctas_per_sm CTAs per SM in total.

    The grouped-query kernel keeps 3 CTAs resident per SM; 24 per SM (8 waves) keeps its
    tail short."""
    units_per_chunk = max(1, n_slots * n_kv)
    chunks = max(1, -(-ctas_per_sm * n_sm // units_per_chunk))
    return max(512, -(-max_len // chunks))


class QuantizedKvCache(CacheBackend):
    """``kvq`` (cache.py:326-360): the quantized K/V baseline at equal bits.
    Pre-RoPE K quantized per channel, V per token, both buffered while decoding
    (prefill quantizes V whole and K by whole groups); K/V from one bf16 GEMM
    per token as in the fp16 baseline. Decode attention dequantizes the K/V
    tiles in shared memory (csrc/xq_kvq.cu)."""

    variant = "kvq"

    def __init__(self, *a, **kw):
        super().__init__(*a, **kw)
        if self.bits == 16:
            raise ConfigError("kvq at 16 bits is QuantizedKvPassthrough (make_cache picks it)")
        if self.group_size != DEFAULT_GROUP_SIZE:
            raise ConfigError(f"the kvq decode kernel takes 128-wide groups, got {self.group_size}")
        self.k_stream = PackedStream(self.bits, CHANNEL, self.kvw, self.group_size, self.n_slots,
                                     self.L, self.device)
        self.v_stream = PackedStream(self.bits, TOKEN, self.kvw, self.group_size, self.n_slots,
                                     self.L, self.device, buffered=True)

    def _project(self, x, weights):
        # float32 GEMMs: K/V are quantized here, so their rounding picks codes
        xf = x.float()
        return xf @ weights.f32("w_k"), xf @ weights.f32("w_v")

    def _prefill(self, slot, x, weights, acc):
        k, v = self._project(x, weights)  # cache.py:344-349
        self.k_stream.channel_bulk(slot, k)
        self.v_stream.token_bulk(slot, v)

    def _decode(self, x, weights, acc, lens):
        k, v = self._project(x, weights)  # cache.py:351-354
        self.k_stream.channel_push(k, self.n_tokens)
        self.v_stream.token_push(v, self.n_tokens)

    def _kv_rows(self, slot, n):
        k = self.k_stream.channel_reconstruct(slot, n)
        vs = self.v_stream
        nfl = int(vs.n_flushed[slot])
        v = torch.empty((n, self.kvw), dtype=torch.float32, device=self.device)
        if nfl:
            v[:nfl] = self._dequant_rows(vs, slot, nfl)
        v[nfl:] = vs.resid[slot, :n - nfl]
        return k, v

    def _rematerialize(self, weights, acc, slot, n):  # cache.py:356-360
        k, v = self._kv_rows(slot, n)
        return _rope_rows(k, 0, self.device), v

    def _prefill_kv(self, weights, acc, slot, n):
        k = self._rows16(self.k_stream, slot, n)  # pre-RoPE K (cache.py:356-360)
        rope = rope_table(n, self.device)
        N.call("xq_rope_rows", N.ptr(k), N.F16, k.stride(0), n, k.shape[1], N.ptr(rope),
               rope.shape[0], 0, N.ptr(k), N.F16, k.stride(0), N.stream_of(self.device))
        return k, self._rows16(self.v_stream, slot, n)

    def _attend(self, q, weights, acc, lens, max_len, out, tpc):
        ks, vs = self.k_stream, self.v_stream
        # one CTA per (sequence, KV head, chunk of whole 128-token groups)
        chunk = tpc * 128 if tpc else -(-kv_chunk_tokens(self.n_slots, max_len, self.n_kv) // 128) * 128
        nbytes = N.lib.xq_kvq_workspace_bytes(self.n_slots, max_len, self.n_heads, chunk)
        ws = _scratch(self.device, nbytes)
        rope = rope_table(max_len, self.device)
        N.call("xq_kvq_decode_attend", N.ptr(ks.codes), N.ptr(ks.params), N.ptr(ks.resid),
               N.ptr(vs.codes), N.ptr(vs.params), N.ptr(vs.resid), N.ptr(ks.nflushed_dev),
               N.ptr(vs.nflushed_dev), self.bits, self.group_size, ks.row_bytes, self.L,
               N.ptr(lens), self.n_slots, max_len, self.n_kv, self.g, N.ptr(q), N.ptr(rope),
               1.0 / math.sqrt(HEAD_DIM), chunk, N.ptr(ws), nbytes, N.ptr(out),
               N.stream_of(self.device))

    def memory_bytes(self):
        out = {f"k_{k}": v for k, v in self.k_stream.nbytes().items()}
        out.update({f"v_{k}": v for k, v in self.v_stream.nbytes().items()})
        return out


class InputCacheMHA(CacheBackend):
    """``xq-mha`` (cache.py:363-387): per-token X codes; K/V rebuilt from X."""

    variant = "xq-mha"

    def __init__(self, *a, **kw):
        super().__init__(*a, **kw)
        self.passthrough = self.bits == 16
        if self.passthrough:  # bits=16 -> fp16 rows (quant.py:117-118 keeps raw data)
            self.raw = RawRows(self.d, self.n_slots, self.L, self.device)
        else:
            self.stream = PackedStream(self.bits, TOKEN, self.d, self.group_size, self.n_slots,
                                       self.L, self.device)

    def _prefill(self, slot, x, weights, acc):
        if self.passthrough:
            self.raw.fill(x, slot)
        else:
            self.stream.fill_rows(x.contiguous(), slot, 0)

    def _decode(self, x, weights, acc, lens):
        if self.passthrough:
            self.raw.append(x, lens)
        else:
            self.stream.append_token_rows(x.contiguous(), lens)

    def _a_operand(self):
        if self.passthrough:
            return N.A_F16_ROWS, self.raw.rows, None, 16, 0
        s = self.stream
        return N.A_CODES_TOKEN, s.codes, s.params, s.bits, s.row_bytes

    def _prefill_kv(self, weights, acc, slot, n):
        a = (self.raw.slot_rows(slot, n) if self.passthrough
             else self._rows16(self.stream, slot, n))
        return self._kv_from(a, a, weights.w_k, weights.w_v, n)

    def _rematerialize(self, weights, acc, slot, n):
        mode, src, params, bits, rb = self._a_operand()
        return self._remat_f32(mode, src, params, None, 0, bits, rb, N.A_SAME, None, None, 0, 0,
                               self.d, weights.f32("w_k"), weights.f32("w_v"), slot, n)

    def _attend(self, q, weights, acc, lens, max_len, out, tpc):
        mode, src, params, bits, rb = self._a_operand()
        spec = (("mha", mode, bits), mode, bits, N.A_SAME, bits, weights.w_k, weights.w_v)
        self._fused(mode, src, params, None, None, bits, rb, N.A_SAME, None, None, 0, 0, self.d,
                    spec, weights, 1, q, lens, max_len, out, tpc)

    def memory_bytes(self):
        if self.passthrough:
            return {"x16": self.raw.rows.numel() * 2}
        return self.stream.nbytes()


class LatentInputCacheGQA(CacheBackend):
    """``xq-gqa`` (cache.py:390-437): K latent per-channel (buffered) + V latent
    per-token; K/V rebuilt through fused = diag(sigma) B^T."""

    variant = "xq-gqa"

    def __init__(self, *a, **kw):
        super().__init__(*a, **kw)
        r = self.latent  # the latent cache is whole even when heads are sharded
        if self.group_size != DEFAULT_GROUP_SIZE and self.bits != 16:
            raise ConfigError("the per-channel K latent needs 128-token groups (one per CTA tile) "
                              f"on the B200 path, got group_size {self.group_size}")
        self.fp16_first_channel = False
        self.passthrough = self.bits == 16
        if self.passthrough:  # 16-bit latents kept raw (quant.py:117-118), no flush
            self.k_raw = RawRows(r, self.n_slots, self.L, self.device)
            self.v_raw = RawRows(r, self.n_slots, self.L, self.device)
            return
        self.k_stream = PackedStream(self.bits, CHANNEL, r, self.group_size, self.n_slots, self.L,
                                     self.device, resid_f64=self.exact)
        self.v_stream = PackedStream(self.bits, TOKEN, r, self.group_size, self.n_slots, self.L,
                                     self.device)

    def set_fp16_first_channel(self, enable: bool) -> None:
        """Pin channel 0 of the K latent to full precision (cache.py:403-409)."""
        if np.any(self.n_tokens):
            raise UsageError("toggle the full-precision channel before caching")
        self.fp16_first_channel = bool(enable)
        if self.passthrough:  # every channel is already raw (cache.py:174: bits != 16)
            return
        self.k_stream = PackedStream(self.bits, CHANNEL, self.latent, self.group_size, self.n_slots,
                                     self.L, self.device, keep_first=self.fp16_first_channel,
                                     resid_f64=self.exact)

    def _latents(self, x, weights):
        if self.exact and x.dtype == torch.float64:  # the reference's float64 GEMMs
            key = ("f64", "u_kv_cat")
            if key not in weights._cache:
                weights._cache[key] = torch.cat([weights.u_k.double(), weights.u_v.double()],
                                                dim=1).contiguous()
            lat = x @ weights._cache[key]
            return lat[:, :self.latent], lat[:, self.latent:]
        # one float32 GEMM against [U_k | U_v] (cache.py:429-432)
        key = ("f32", "u_kv_cat")
        if key not in weights._cache:
            weights._cache[key] = torch.cat([weights.f32("u_k"), weights.f32("u_v")], dim=1).contiguous()
        lat = x.float() @ weights._cache[key]
        r = self.latent
        return lat[:, :r], lat[:, r:]

    def _prefill(self, slot, x, weights, acc):
        lat_k, lat_v = self._latents(x, weights)
        if self.passthrough:
            self.k_raw.fill(lat_k, slot)
            self.v_raw.fill(lat_v, slot)
            return
        self.v_stream.fill_rows(lat_v.contiguous(), slot, 0)
        self.k_stream.channel_bulk(slot, lat_k)  # cache.py:203-208

    def _decode(self, x, weights, acc, lens):
        if self.passthrough:
            lat_k, lat_v = self._latents(x, weights)
            self.k_raw.append(lat_k, lens)
            self.v_raw.append(lat_v, lens)
            return
        if self.exact and x.dtype == torch.float64:  # the reference's float64 latents
            lat_k, lat_v = self._latents(x, weights)
            self.v_stream.append_token_rows(lat_v.contiguous(), lens)
            self.k_stream.channel_push(lat_k, self.n_tokens)  # cache.py:218-221
            return
        # one tcgen05 launch: x @ [U_k | U_v] (bf16 operands, fp32 accumulation), the V
        # latent quantized into its arena, the K latent into the residual buffer
        xb = x if x.dtype == torch.bfloat16 else x.to(torch.bfloat16)
        xb = xb.contiguous()
        ks, vs = self.k_stream, self.v_stream
        N.call("xq_latent_project_append", N.ptr(xb), xb.stride(0), xb.shape[0], self.d,
               N.ptr(self._u_cat_bf16(weights)), self.latent, self.bits, self.group_size,
               N.ptr(lens), N.ptr(ks.nflushed_dev), self.L, N.ptr(ks.resid), N.ptr(vs.codes),
               vs.row_bytes, N.ptr(vs.params), None, N.ptr(vs.flag), N.stream_of(self.device))
        ks.flush_full(self.n_tokens)

    @staticmethod
    def _u_cat_bf16(weights):
        """[U_k | U_v] in bf16, the tcgen05 operand of the latent projection."""
        key = ("bf16", "u_kv_cat")
        if key not in weights._cache:
            weights._cache[key] = torch.cat([weights.u_k, weights.u_v], dim=1).to(
                torch.bfloat16).contiguous()
        return weights._cache[key]

    def _prefill_kv(self, weights, acc, slot, n):
        if self.passthrough:
            lat_k, lat_v = self.k_raw.slot_rows(slot, n), self.v_raw.slot_rows(slot, n)
        else:
            lat_k = self._rows16(self.k_stream, slot, n)
            lat_v = self._rows16(self.v_stream, slot, n)
        return self._kv_from(lat_k, lat_v, weights.fused_k, weights.fused_v, n)

    def _rematerialize(self, weights, acc, slot, n):
        if self.passthrough:
            return self._remat_f32(N.A_F16_ROWS, self.k_raw.rows, None, None, 0, 16, 0,
                                   N.A_F16_ROWS, self.v_raw.rows, None, 16, 0, self.latent,
                                   weights.f32("fused_k"), weights.f32("fused_v"), slot, n)
        ks, vs = self.k_stream, self.v_stream
        if ks.first is not None:  # float32 torch path (the SIMT debug kernel has no outlier channel)
            k = ks.channel_reconstruct(slot, n) @ weights.f32("fused_k")
            v = self._dequant_rows(vs, slot, n) @ weights.f32("fused_v")
            return _rope_rows(k, 0, self.device), v
        return self._remat_f32(N.A_CODES_CHANNEL, ks.codes, ks.params, ks.resid,
                               int(ks.n_flushed[slot]), ks.bits, ks.row_bytes, N.A_CODES_TOKEN,
                               vs.codes, vs.params, vs.bits, vs.row_bytes, self.latent,
                               weights.f32("fused_k"), weights.f32("fused_v"), slot, n)

    def _attend(self, q, weights, acc, lens, max_len, out, tpc):
        if self.passthrough:  # fp16 latent rows: K side and V side from their own arenas
            spec = (("gqa", 16), N.A_F16_ROWS, 16, N.A_F16_ROWS, 16, weights.fused_k,
                    weights.fused_v)
            self._fused(N.A_F16_ROWS, self.k_raw.rows, None, None, None, 16, 0, N.A_F16_ROWS,
                        self.v_raw.rows, None, 16, 0, self.latent, spec, weights, self.g, q, lens,
                        max_len, out, tpc, force_absorbed=True)
            return
        ks, vs = self.k_stream, self.v_stream
        spec = (("gqa", self.bits), N.A_CODES_CHANNEL, ks.bits, N.A_CODES_TOKEN, vs.bits,
                weights.fused_k, weights.fused_v)
        self._fused(N.A_CODES_CHANNEL, ks.codes, ks.params, ks.resid, ks.nflushed_dev, ks.bits,
                    ks.row_bytes, N.A_CODES_TOKEN, vs.codes, vs.params, vs.bits, vs.row_bytes,
                    self.latent, spec, weights, self.g, q, lens, max_len, out, tpc,
                    force_absorbed=ks.first is not None, ak_first=ks.first)

    def memory_bytes(self):
        ks, vs = (self.k_raw, self.v_raw) if self.passthrough else (self.k_stream, self.v_stream)
        out = {f"k_{k}": v for k, v in ks.nbytes().items()}
        out.update({f"v_{k}": v for k, v in vs.nbytes().items()})
        return out


class DeltaInputCacheMHA(CacheBackend):
    """``xq-cl-mha`` (cache.py:440-535): base layers cache X; the last base
    layer seeds the accumulator; delta layers cache x - acc[pos] and add the
    reconstruction of all their deltas to the accumulator; delta-layer K/V are
    rebuilt from the accumulator."""

    variant = "xq-cl-mha"
    needs_accumulator = True

    def __init__(self, *a, **kw):
        super().__init__(*a, **kw)
        if self.policy.base_layers < 1:
            raise ConfigError("cross-layer variants need at least one base layer")
        # 16 bits: the payload (x, or the delta x - acc) is kept exactly, so after the
        # layer acc = x (cache.py:463-481 with a pass-through QuantizedTensor). The
        # arena keeps x itself as fp16 rows, which carries the same information as
        # the delta given acc, and is the layer's remat operand directly.
        self.passthrough = self.bits == 16
        if self.passthrough:
            self.raw = RawRows(self.d, self.n_slots, self.L, self.device)
        else:
            self.stream = PackedStream(self.bits, TOKEN, self.d, self.group_size, self.n_slots,
                                       self.L, self.device)

    @property
    def is_base(self):
        return self.layer_index < self.policy.base_layers

    @property
    def seeds_accumulator(self):
        return self.layer_index == self.policy.base_layers - 1

    def _accumulate(self, acc, seed, max_len, lens):
        if acc.pending is not None and acc.pending[0] is not self:
            acc.settle()  # the previous delta layer's update comes first
        s = self.stream
        x16 = acc.x16 if (acc.x_hat is None or not seed) else None
        N.call("xq_cl_accumulate", 1 if seed else 0, N.ptr(s.codes), s.row_bytes, N.ptr(s.params),
               s.bits, self.group_size, self.d, N.ptr(lens), self.n_slots, max_len, self.L,
               N.ptr(acc.x_hat), N.ptr(x16), N.stream_of(self.device))
        acc.seeded = True

    def _prefill(self, slot, x, weights, acc):
        n = x.shape[0]
        if self.passthrough:
            self.raw.fill(x, slot)
            if self.is_base and not self.seeds_accumulator:
                return
            if not self.is_base and not acc.seeded:
                raise UsageError("accumulator used before the base layer seeded it")
            acc.prefill_rows(slot, n, seed=self.is_base).copy_(x.double())
            acc.assign_rows(self.raw.slot_rows(slot, n), n, slot=slot)
            return
        lens = torch.zeros(self.n_slots, dtype=torch.int32, device=self.device)
        lens[slot] = n
        x = x.contiguous()
        if self.is_base and not self.seeds_accumulator:
            self.stream.fill_rows(x, slot, 0)
            return
        if not self.is_base and not acc.seeded:
            raise UsageError("accumulator used before the base layer seeded it")
        # codes against the float64 accumulator (cache.py:463-470), then the
        # remat operand of all n rows from the arena (cache.py:139-146)
        acc64 = acc.prefill_rows(slot, n, seed=self.is_base)
        self.stream.fill_rows_cl(x, slot, 0, acc64, seed=self.is_base)
        self._accumulate(acc, self.is_base, n, lens)

    def _decode(self, x, weights, acc, lens):
        max_len = int(self.n_tokens.max())
        x = x.contiguous()
        if self.passthrough:
            self.raw.append(x, lens)
            if self.is_base and not self.seeds_accumulator:
                return
            if not self.is_base and not acc.seeded:
                raise UsageError("accumulator used before the base layer seeded it")
            if self.is_base:
                acc.release_prefill()
            acc.row64.copy_(x.double())  # acc at the new token = x
            acc.assign_rows(self.raw.slots_view(), max_len)
            return
        if self.is_base and not self.seeds_accumulator:
            self.stream.append_token_rows(x, lens)
            return
        if not self.is_base and not acc.seeded:
            raise UsageError("accumulator used before the base layer seeded it")
        if self.is_base:
            acc.release_prefill()
        # the new token's delta against the float64 accumulator row (cache.py:473-481)
        self.stream.append_token_rows_cl(x, lens, acc.row64, seed=self.is_base)
        if not self.is_base and acc.x_hat is None:
            # acc += deq(deltas) waits for this layer's fused decode launch, which
            # does it in its first K pass (settle() otherwise)
            acc.settle()
            acc.pending = (self, lens.clone(), max_len)
            return
        self._accumulate(acc, self.is_base, max_len, lens)

    def _prefill_kv(self, weights, acc, slot, n):
        acc.settle()
        if self.passthrough:
            a = self.raw.slot_rows(slot, n)
        else:
            a = self._rows16(self.stream, slot, n) if self.is_base else acc.x16[slot, :n]
        return self._kv_from(a, a, weights.w_k, weights.w_v, n)

    def _rematerialize(self, weights, acc, slot, n):
        wk, wv = weights.f32("w_k"), weights.f32("w_v")
        if self.passthrough:
            return self._remat_f32(N.A_F16_ROWS, self.raw.rows, None, None, 0, 16, 0, N.A_SAME,
                                   None, None, 0, 0, self.d, wk, wv, slot, n)
        if self.is_base:
            s = self.stream
            return self._remat_f32(N.A_CODES_TOKEN, s.codes, s.params, None, 0, s.bits,
                                   s.row_bytes, N.A_SAME, None, None, 0, 0, self.d, wk, wv, slot, n)
        return self._remat_acc(acc, wk, wv, slot, n)

    def _remat_acc(self, acc, wk, wv, slot, n):
        # parity path from the float32 accumulator itself (cache.py:531-535)
        xh = acc.rows(slot, n)
        k = xh @ wk
        v = xh @ wv
        rope = rope_table(n, self.device)
        cos, sin = rope[:n, 0::2], rope[:n, 1::2]
        kk = k.view(n, -1, 64, 2)
        e, o = kk[..., 0], kk[..., 1]
        c, s = cos[:, None, :], sin[:, None, :]
        return torch.stack([e * c - o * s, e * s + o * c], dim=-1).view(n, -1), v

    def _attend(self, q, weights, acc, lens, max_len, out, tpc):
        self.fused_accumulate = False
        if (acc is not None and acc.pending is not None and acc.pending[0] is self
                and not self.peer_outs and self._use_absorbed(self.d, max_len)):
            acc.pending = None
            self._attend_cl(q, weights, acc, lens, max_len, out)
            self.fused_accumulate = True
            return
        if acc is not None:
            acc.settle()
        if self.passthrough:
            spec = (("mha", N.A_F16_ROWS, 16), N.A_F16_ROWS, 16, N.A_SAME, 16, weights.w_k,
                    weights.w_v)
            self._fused(N.A_F16_ROWS, self.raw.rows, None, None, None, 16, 0, N.A_SAME, None, None,
                        0, 0, self.d, spec, weights, 1, q, lens, max_len, out, tpc)
        elif self.is_base:
            s = self.stream
            spec = (("mha", N.A_CODES_TOKEN, s.bits), N.A_CODES_TOKEN, s.bits, N.A_SAME, s.bits,
                    weights.w_k, weights.w_v)
            self._fused(N.A_CODES_TOKEN, s.codes, s.params, None, None, s.bits, s.row_bytes,
                        N.A_SAME, None, None, 0, 0, self.d, spec, weights, 1, q, lens, max_len,
                        out, tpc)
        else:
            spec = (("mha", N.A_F16_ROWS, 16), N.A_F16_ROWS, 16, N.A_SAME, 16, weights.w_k,
                    weights.w_v)
            self._fused(N.A_F16_ROWS, acc.x16, None, None, None, 16, 0, N.A_SAME, None, None, 0,
                        0, self.d, spec, weights, 1, q, lens, max_len, out, tpc)

    def _attend_cl(self, q, weights, acc, lens, max_len, out):
        """Delta layer: the accumulate (acc += deq(this layer's deltas), cache.py:472-481,
        139-146) fused into the first K pass of the decode kernel, which then
        rematerialises from the updated rows (cache.py:527-535)."""
        s = self.stream
        spec = (("mha", N.A_F16_ROWS, 16), N.A_F16_ROWS, 16, N.A_SAME, 16, weights.w_k, weights.w_v)
        key, mk, bk, mv, bv, wk, wv = spec
        wk_arr, wv_arr = weights.arranged_absorbed(key, mk, bk, mv, bv, wk, wv)
        rope = rope_table_t(max_len, self.device)
        nbytes = N.lib.xq_absorbed_workspace_bytes(self.n_slots, max_len, self.n_kv, self.d)
        ws = _scratch(self.device, nbytes)
        N.call("xq_decode_attend_absorbed_cl", N.ptr(acc.x16), N.ptr(s.codes), N.ptr(s.params), s.bits,
               s.row_bytes, self.group_size, self.L, self.d, N.ptr(lens), self.n_slots, max_len,
               N.ptr(wk_arr), N.ptr(wv_arr), self.n_kv, N.ptr(q), N.ptr(rope), rope.shape[1] // 2,
               1.0 / math.sqrt(HEAD_DIM), N.ptr(ws), nbytes, N.ptr(out), N.stream_of(self.device))

    def memory_bytes(self):
        return (self.raw if self.passthrough else self.stream).nbytes()


class DeltaLatentCacheGQA(CacheBackend):
    """``xq-cl-gqa`` (cache.py:538-604): cross-layer deltas in the shared latent
    subspace U_kv of svd([W_k | W_v]) (model.py:135-142), quantized per-channel
    (buffered); the accumulator is d-wide (cache.py:124-146).

    Base layers cache x @ U; layer base-1 seeds acc = reconstruct() @ U^T.
    Delta layers cache (x - acc[pos]) @ U and add reconstruct() @ U^T to acc
    (cache.py:574-589). Remat (cache.py:591-604): base kv = reconstruct() @ fused;
    delta kv = (acc @ U) @ fused, run here as acc @ (U @ fused) -- the same
    product reassociated, so the fused kernel reads the fp16 accumulator rows
    like xq-cl-mha with W' = U @ fused_{k|v} (d x kv_width) precomputed once.

    Decode, per layer: the new token's latent in float64 against the float64
    accumulator row (``xq_clgqa_latent64``), the per-channel flush of a full
    group with its float64 reconstruction written back (so the accumulator row
    follows the reference's reconstruct() exactly), the row update
    acc_row (+)= rec @ U^T (``xq_clgqa_row_update``), and the fp16 remat operand
    of every cached row, acc16 (+)= rec16 @ U^T, on the tcgen05 remat GEMM.
    """

    variant = "xq-cl-gqa"
    needs_accumulator = True

    def __init__(self, *a, **kw):
        super().__init__(*a, **kw)
        if self.policy.base_layers < 1:
            raise ConfigError("cross-layer variants need at least one base layer")
        if self.group_size != DEFAULT_GROUP_SIZE and self.bits != 16:
            raise ConfigError("the per-channel latent needs 128-token groups (one per CTA tile) "
                              f"on the B200 path, got group_size {self.group_size}")
        kv_width = self.d // self.g
        if 2 * kv_width > self.d:  # model.py:135-142: the shared subspace only when 2*kvw <= d
            raise ConfigError("xq-cl-gqa needs a shared K/V subspace (2*kv_width <= hidden_dim)")
        self.rank = 2 * kv_width
        self.kv_width = kv_width
        self.rec_pos = torch.zeros(self.n_slots, dtype=torch.int32, device=self.device)
        self.passthrough = self.bits == 16
        if self.passthrough:
            # 16 bits: the latent rows are kept raw (quant.py:117-118) as fp16, the
            # remat operand; the new token's float64 latent lives in a one-row
            # buffer per slot (row 0), which the accumulator row update reads
            self.raw = RawRows(self.rank, self.n_slots, self.L, self.device)
            self.lat64 = torch.zeros((self.n_slots, 1, self.rank), dtype=torch.float64,
                                     device=self.device)
            self.lat32 = torch.zeros((self.n_slots, 1, self.rank), dtype=torch.float32,
                                     device=self.device)
            self.pos_m1 = torch.zeros(self.n_slots, dtype=torch.int32, device=self.device)
            self.flag = torch.zeros(1, dtype=torch.int32, device=self.device)
            return
        # latents formed and quantized in float64 like the reference's (a base-layer
        # code flip is a full quantization step, large against later deltas)
        self.stream = PackedStream(self.bits, CHANNEL, self.rank, self.group_size, self.n_slots,
                                   self.L, self.device, resid_f64=True)

    @property
    def is_base(self):
        return self.layer_index < self.policy.base_layers

    @property
    def seeds_accumulator(self):
        return self.layer_index == self.policy.base_layers - 1

    @staticmethod
    def _sub(weights):
        if weights.u_kv is None or weights.fused_kv is None:
            raise ConfigError("xq-cl-gqa needs the shared K/V subspace (u_kv, fused_kv)")
        return weights.f32("u_kv"), weights.f32("fused_kv")

    @staticmethod
    def _u(weights):
        """U as stored (float32 or float64), the float64 GEMVs' operand."""
        u = weights.u_kv
        if u.dtype not in (torch.float32, torch.float64):
            u = weights.f32("u_kv")
        return u.contiguous(), _dtype_code(u)

    @staticmethod
    def _u64(weights):
        key = ("f64", "u_kv")
        if key not in weights._cache:
            weights._cache[key] = weights.u_kv.double().contiguous()
        return weights._cache[key]

    @staticmethod
    def _u16(weights):
        """fp16 U [d, r]: the remat GEMM's B operand for acc (+)= rec @ U^T (N=d, K=r)."""
        key = ("f16", "u_kv")
        if key not in weights._cache:
            weights._cache[key] = weights.u_kv.to(torch.float16).contiguous()
        return weights._cache[key]

    def _acc16(self, acc, weights, slots, seed):
        """acc16[s, :n] (+)= rec16 @ U^T for every slot (cache.py:571-572, 588-589).

        When every slot is in use and filled to at least 3/4 of the accumulator rows, the
        slots' reconstructions are staged in one shared buffer and multiplied in one GEMM
        over all rows (rows past a slot's length hold finite stale values and are never
        attended to; the seeding layer rewrites them every step)."""
        u16 = self._u16(weights)
        slots = [s for s in slots if self.n_tokens[s] > 0]
        la = acc.x16.shape[1]
        if (len(slots) == self.n_slots > 1 and not self.passthrough
                and 4 * int(self.n_tokens.max()) >= 3 * la):
            buf = _rec_rows(self.device, self.n_slots * la, self.rank)
            for s in slots:
                n = int(self.n_tokens[s])
                self._rows16(self.stream, s, n, out=buf[s * la:s * la + n])
            c = acc.x16
            N.call("xq_gemm_f16", N.ptr(buf), buf.stride(0), N.ptr(u16), u16.stride(0), N.ptr(c),
                   c.stride(1), self.n_slots * la, self.d, self.rank, 0 if seed else 2, None, 0, 0,
                   N.stream_of(self.device))
            acc.seeded = True
            self.acc16_launches = len(slots) + 1
            return
        self.acc16_launches = 2 * len(slots)
        for s in slots:
            n = int(self.n_tokens[s])
            if n == 0:
                continue
            rec = self.raw.slot_rows(s, n) if self.passthrough else self._rows16(self.stream, s, n)
            c = acc.x16[s]
            N.call("xq_gemm_f16", N.ptr(rec), rec.stride(0), N.ptr(u16), u16.stride(0), N.ptr(c),
                   c.stride(0), n, self.d, self.rank, 0 if seed else 2, None, 0, 0,
                   N.stream_of(self.device))
        acc.seeded = True

    def _flush(self, n_tokens):
        """Flush full residual groups with the float64 reconstruction written back
        over their rows (the new token's reconstruction stays at its row)."""
        st = self.stream
        full = np.nonzero(n_tokens - st.n_flushed >= st.g)[0]
        if not len(full):
            return
        dst = torch.tensor([int(s) * st.L + int(st.n_flushed[s]) for s in full], dtype=torch.int64,
                           device=self.device)
        blocks = st.resid64 if len(full) == st.n_slots else st.resid64[torch.as_tensor(full, device=self.device)].contiguous()
        N.call("xq_quantize_blocks_per_channel_f64_recon", N.ptr(blocks), len(full), st.width,
               st.bits, st.g, N.ptr(dst), N.ptr(st.codes), st.row_bytes, N.ptr(st.params),
               N.ptr(blocks), N.ptr(st.flag), N.stream_of(self.device))
        if blocks is not st.resid64:
            st.resid64[torch.as_tensor(full, device=self.device)] = blocks
        st.n_flushed[full] += st.g
        st.nflushed_dev.copy_(torch.from_numpy(st.n_flushed.astype(np.int32)))

    def _prefill(self, slot, x, weights, acc):
        self._sub(weights)
        n = x.shape[0]
        xf = x.double()
        if not self.is_base:
            if not acc.seeded:
                raise UsageError("accumulator used before the base layer seeded it")
            xf = xf - acc.prefill_rows(slot, n, seed=False)  # cache.py:574-577 (delta = x - acc)
        u64 = self._u64(weights)
        lat = (xf @ u64).contiguous()
        if self.passthrough:
            self.raw.fill(lat, slot)
            self.n_tokens[slot] = n
            if self.is_base and not self.seeds_accumulator:
                return
            rows = acc.prefill_rows(slot, n, seed=self.is_base)
            upd = lat @ u64.t()
            if self.is_base:
                rows.copy_(upd)
            else:
                rows += upd
            self._acc16(acc, weights, [slot], seed=self.is_base)
            return
        st = self.stream
        g = st.g
        n_full = n // g * g
        if n_full:  # whole groups: codes + their float64 reconstruction in place of lat
            dst = torch.tensor([slot * st.L + i for i in range(0, n_full, g)], dtype=torch.int64,
                               device=self.device)
            N.call("xq_quantize_blocks_per_channel_f64_recon", N.ptr(lat), n_full // g, st.width,
                   st.bits, g, N.ptr(dst), N.ptr(st.codes), st.row_bytes, N.ptr(st.params),
                   N.ptr(lat), N.ptr(st.flag), N.stream_of(self.device))
        st.resid64[slot, :n - n_full] = lat[n_full:]
        st.resid[slot, :n - n_full] = lat[n_full:].float()
        st.n_flushed[slot] = n_full
        st.nflushed_dev[slot] = n_full
        self.n_tokens[slot] = n  # the accumulator update reads the new length
        if self.is_base and not self.seeds_accumulator:
            return
        rows = acc.prefill_rows(slot, n, seed=self.is_base)
        upd = lat @ u64.t()  # float64 reconstruction @ U^T (prefill only)
        if self.is_base:
            rows.copy_(upd)
        else:
            rows += upd
        self._acc16(acc, weights, [slot], seed=self.is_base)

    def _decode(self, x, weights, acc, lens):
        self._sub(weights)
        if not self.is_base and not acc.seeded:
            raise UsageError("accumulator used before the base layer seeded it")
        if self.is_base:
            acc.release_prefill()
        u, udt = self._u(weights)
        x = x.contiguous()
        if self.passthrough:
            self._decode16(x, u, udt, acc, lens, weights)
            return
        st = self.stream
        pos = (self.n_tokens - 1 - st.n_flushed).astype(np.int32)  # before this step's flush
        N.call("xq_clgqa_latent64", N.ptr(x), _dtype_code(x), x.stride(0), x.shape[0], self.d,
               None if self.is_base else N.ptr(acc.row64), N.ptr(u), udt, self.rank, N.ptr(lens),
               N.ptr(st.nflushed_dev), st.g, N.ptr(st.resid64), N.ptr(st.resid), N.ptr(st.flag),
               N.stream_of(self.device))
        self._flush(self.n_tokens)
        if self.is_base and not self.seeds_accumulator:
            return
        self.rec_pos.copy_(torch.from_numpy(pos))
        N.call("xq_clgqa_row_update", N.ptr(st.resid64), N.ptr(self.rec_pos), self.n_slots, st.g,
               N.ptr(u), udt, self.d, self.rank, 1 if self.is_base else 0, N.ptr(acc.row64),
               N.stream_of(self.device))
        self._acc16(acc, weights, range(self.n_slots), seed=self.is_base)

    def _decode16(self, x, u, udt, acc, lens, weights):
        """16-bit decode: the float64 latent (x - acc_row) @ U of the new token into
        row 0 of the one-row buffers (nflushed = len-1 puts it there), stored raw as
        fp16; the accumulator row and the fp16 remat operand as for coded layers."""
        torch.sub(lens, 1, out=self.pos_m1)
        N.call("xq_clgqa_latent64", N.ptr(x), _dtype_code(x), x.stride(0), x.shape[0], self.d,
               None if self.is_base else N.ptr(acc.row64), N.ptr(u), udt, self.rank, N.ptr(lens),
               N.ptr(self.pos_m1), 1, N.ptr(self.lat64), N.ptr(self.lat32), N.ptr(self.flag),
               N.stream_of(self.device))
        self.raw.append(self.lat32[:, 0], lens)
        if self.is_base and not self.seeds_accumulator:
            return
        self.rec_pos.zero_()
        N.call("xq_clgqa_row_update", N.ptr(self.lat64), N.ptr(self.rec_pos), self.n_slots, 1,
               N.ptr(u), udt, self.d, self.rank, 1 if self.is_base else 0, N.ptr(acc.row64),
               N.stream_of(self.device))
        self._acc16(acc, weights, range(self.n_slots), seed=self.is_base)

    def _w_delta(self, weights):
        key = ("clgqa_w", id(weights))
        if key not in weights._cache:
            u, fused = self._sub(weights)
            w = u @ fused  # (acc @ U) @ fused == acc @ (U @ fused)
            weights._cache[key] = (w[:, :self.kv_width].contiguous(), w[:, self.kv_width:].contiguous())
        return weights._cache[key]

    def _prefill_kv(self, weights, acc, slot, n):
        _, fused = self._sub(weights)
        if self.is_base:
            a = self.raw.slot_rows(slot, n) if self.passthrough else self._rows16(self.stream, slot, n)
            return self._kv_from(a, a, fused[:, :self.kv_width], fused[:, self.kv_width:], n)
        wk, wv = self._w_delta(weights)
        a = acc.x16[slot, :n]
        return self._kv_from(a, a, wk, wv, n)

    def _rematerialize(self, weights, acc, slot, n):
        _, fused = self._sub(weights)
        if self.is_base and self.passthrough:
            return self._remat_f32(N.A_F16_ROWS, self.raw.rows, None, None, 0, 16, 0, N.A_SAME, None,
                                   None, 0, 0, self.rank, fused[:, :self.kv_width].contiguous(),
                                   fused[:, self.kv_width:].contiguous(), slot, n)
        if self.is_base:
            s = self.stream
            return self._remat_f32(N.A_CODES_CHANNEL, s.codes, s.params, s.resid,
                                   int(s.n_flushed[slot]), s.bits, s.row_bytes, N.A_SAME, None,
                                   None, 0, 0, self.rank, fused[:, :self.kv_width].contiguous(),
                                   fused[:, self.kv_width:].contiguous(), slot, n)
        wk, wv = self._w_delta(weights)
        # parity path from the fp16 remat operand itself (cache.py:595-604)
        xh = acc.x16[slot, :n].float()
        k = _rope_rows(xh @ wk, 0, self.device)
        return k, xh @ wv

    def _attend(self, q, weights, acc, lens, max_len, out, tpc):
        _, fused = self._sub(weights)
        if self.is_base:
            fk = weights._cache.setdefault(("clgqa_fk", id(weights)), fused[:, :self.kv_width].contiguous())
            fv = weights._cache.setdefault(("clgqa_fv", id(weights)), fused[:, self.kv_width:].contiguous())
            if self.passthrough:
                spec = (("clgqa-base", 16), N.A_F16_ROWS, 16, N.A_SAME, 16, fk, fv)
                self._fused(N.A_F16_ROWS, self.raw.rows, None, None, None, 16, 0, N.A_SAME, None, None,
                            0, 0, self.rank, spec, weights, self.g, q, lens, max_len, out, tpc,
                            force_absorbed=True)
                return
            s = self.stream
            spec = (("clgqa-base", s.bits), N.A_CODES_CHANNEL, s.bits, N.A_SAME, s.bits, fk, fv)
            self._fused(N.A_CODES_CHANNEL, s.codes, s.params, s.resid, s.nflushed_dev, s.bits,
                        s.row_bytes, N.A_SAME, None, None, 0, 0, self.rank, spec, weights, self.g,
                        q, lens, max_len, out, tpc, force_absorbed=True)
        else:
            wk, wv = self._w_delta(weights)
            spec = (("clgqa-delta",), N.A_F16_ROWS, 16, N.A_SAME, 16, wk, wv)
            self._fused(N.A_F16_ROWS, acc.x16, None, None, None, 16, 0, N.A_SAME, None, None, 0, 0,
                        self.d, spec, weights, self.g, q, lens, max_len, out, tpc,
                        force_absorbed=True)

    def memory_bytes(self):
        return (self.raw if self.passthrough else self.stream).nbytes()


class QuantizedKvPassthrough(FullPrecisionCache):
    """``kvq`` at 16 bits: K and V are kept raw (quant.py:117-118), which is the
    fp16 baseline's cache (cache.py:326-360 with pass-through tensors)."""

    variant = "kvq"


_BACKENDS = {
    cls.variant: cls
    for cls in (FullPrecisionCache, QuantizedKvCache, InputCacheMHA, LatentInputCacheGQA, DeltaInputCacheMHA,
                DeltaLatentCacheGQA)
}


def fp16_outlier_channel_variant(state, enable: bool):
    """Pin channel 0 of the K latent to full precision (cache.py:653-658; xq-gqa only)."""
    if isinstance(state, ReferenceCache):
        state.set_fp16_first_channel(enable)
        return state
    if not isinstance(state, LatentInputCacheGQA):
        raise UsageError("full-precision outlier channel applies to xq-gqa only")
    state.set_fp16_first_channel(enable)
    return state


def make_cache(variant: str, layer_index: int, policy: LayerPolicy, head_dim: int,
               group_size: int = DEFAULT_GROUP_SIZE, **kw):
    """Instantiate the backend for one layer (cache.py:620-630).

    With ``hidden_dim`` / ``n_heads`` (and ``n_slots``, ``max_len``) the device
    arenas are allocated here. Called with the reference's signature alone, it
    returns a :class:`ReferenceCache` for one sequence that sizes its arenas from
    the first ``prefill`` / ``decode_append`` and speaks NumPy like the
    reference's backends."""
    if variant not in VARIANTS:
        raise ConfigError(f"unknown variant {variant!r}; expected one of {VARIANTS}")
    if variant not in _BACKENDS:
        raise ConfigError(f"variant {variant!r} is not on the B200 hot path (next row)")
    if kw.get("hidden_dim") is None or kw.get("n_heads") is None:
        return ReferenceCache(variant, layer_index, policy, head_dim, group_size, **kw)
    return backend_class(variant, policy.bits_for(layer_index))(layer_index, policy, head_dim,
                                                                group_size, **kw)


def backend_class(variant: str, bits: int):
    """The backend of a variant at a layer's bit width (kvq at 16 bits keeps K/V raw)."""
    if variant == "kvq" and bits == 16:
        return QuantizedKvPassthrough
    return _BACKENDS[variant]


# ---------------------------------------------------------------------------
# The reference's objects at the boundary (cache.py:49-67, 124-146, 620-650)
# ---------------------------------------------------------------------------

_ADOPTED_W: dict = {}    # id(reference LayerWeights) -> (weakref, device LayerWeights)
_ADOPTED_ACC: dict = {}  # id(reference Accumulator) -> (weakref, device Accumulator)


def _adopt_cached(table: dict, obj, build):
    import weakref

    key = id(obj)
    hit = table.get(key)
    if hit is not None and hit[0]() is obj:
        return hit[1]
    val = build()
    try:
        ref = weakref.ref(obj, lambda _r, k=key: table.pop(k, None))
    except TypeError:  # not weak-referenceable: adopt afresh every call
        return val
    table[key] = (ref, val)
    return val


def as_layer_weights(weights, device=None) -> LayerWeights:
    """This module's LayerWeights, or the reference's (NumPy float64 w_k / w_v and
    SvdFactors svd_k / svd_v / svd_kv, cache.py:49-67) copied once to the device.
    The projections stay float64 on the device; every kernel path converts them
    (fp16 tensor-core operands, float32 SIMT remat, float64 latent GEMMs)."""
    if isinstance(weights, LayerWeights) or weights is None:
        return weights
    if not hasattr(weights, "w_k"):
        raise UsageError(f"expected LayerWeights, got {type(weights).__name__}")
    dev = torch.device(device) if device is not None else torch.device(
        "cuda", torch.cuda.current_device())

    def t(a):
        return None if a is None else torch.as_tensor(np.asarray(a, np.float64), device=dev)

    def build():
        lw = LayerWeights(w_k=t(weights.w_k), w_v=t(weights.w_v))
        for name, (u, f) in (("svd_k", ("u_k", "fused_k")), ("svd_v", ("u_v", "fused_v")),
                             ("svd_kv", ("u_kv", "fused_kv"))):
            fac = getattr(weights, name, None)
            if fac is not None:
                setattr(lw, u, t(fac.u))
                setattr(lw, f, t(fac.fused))
        return lw

    return _adopt_cached(_ADOPTED_W, weights, build)


def device_accumulator(acc) -> Accumulator:
    """This module's Accumulator, or a device accumulator standing in for the
    reference's (``Accumulator()``, cache.py:124-146). The reference creates one
    per forward pass (model.py:202, :227) and threads it through the layers in
    order; the stand-in follows the same object through that pass."""
    if isinstance(acc, Accumulator):
        return acc
    if not (hasattr(acc, "seed") and hasattr(acc, "add")):
        raise UsageError(f"expected an Accumulator, got {type(acc).__name__}")
    bits = getattr(acc, "accounting_bits", DEFAULT_ACCUMULATOR_BITS)
    return _adopt_cached(_ADOPTED_ACC, acc, lambda: Accumulator(accounting_bits=bits))


class ReferenceCache:
    """One sequence's cache behind the reference's backend interface
    (``cache.py:238-281``): ``prefill(x, weights, acc)``, ``decode_append(x_token,
    weights, acc)``, ``rematerialize(weights, positions, acc) -> (K, V)``, with
    NumPy in and NumPy float64 out (torch in -> torch out), the reference's
    LayerWeights / Accumulator objects accepted as they are.

    It is what ``make_cache(variant, layer_index, policy, head_dim, group_size)``
    returns, so ``model._Session`` (model.py:185-240) runs unchanged on the
    device backends. The arenas are sized from the first call: d from x, the
    KV width from the weights (hidden = n_heads * head_dim), ``max_len`` rows
    (``DEFAULT_MAX_LEN`` unless given). Inputs given in float64 keep the
    reference's float64 arithmetic up to quantization: CL deltas against a
    float64 accumulator row, xq-gqa latents as float64 GEMMs.
    """

    def __init__(self, variant, layer_index, policy, head_dim, group_size=DEFAULT_GROUP_SIZE,
                 **kw):
        if head_dim != HEAD_DIM:
            raise ConfigError(f"the B200 kernels are specialised for head_dim {HEAD_DIM}, got {head_dim}")
        self.variant, self.layer_index, self.policy = variant, layer_index, policy
        self.head_dim, self.group_size = head_dim, group_size
        self.bits = policy.bits_for(layer_index)
        self.needs_accumulator = _BACKENDS[variant].needs_accumulator
        self._kw = dict(kw)
        self._inner: CacheBackend | None = None
        self._first_channel = False

    # the reference's attributes
    @property
    def n_tokens(self) -> int:
        return 0 if self._inner is None else int(self._inner.n_tokens[0])

    @property
    def backend(self) -> CacheBackend | None:
        """The device backend (None before the first call)."""
        return self._inner

    def __getattr__(self, name):
        inner = self.__dict__.get("_inner")
        if inner is None:
            raise AttributeError(name)
        return getattr(inner, name)

    def set_fp16_first_channel(self, enable: bool) -> None:
        if self.n_tokens:
            raise UsageError("toggle the full-precision channel before caching")
        if self.variant != "xq-gqa":
            raise UsageError("full-precision outlier channel applies to xq-gqa only")
        self._first_channel = bool(enable)
        if self._inner is not None:
            self._inner.set_fp16_first_channel(enable)

    def _build(self, d: int, weights: LayerWeights):
        if weights.w_k is not None:
            kvw = weights.w_k.shape[1]
        elif weights.fused_k is not None:
            kvw = weights.fused_k.shape[1]
        else:
            raise ConfigError("weights carry no K projection to size the cache from")
        if d % HEAD_DIM or kvw % HEAD_DIM or d % kvw:
            raise ShapeError(f"hidden {d} / kv width {kvw} must be multiples of {HEAD_DIM}")
        kw = dict(self._kw)
        kw.setdefault("n_slots", 1)
        kw.setdefault("max_len", DEFAULT_MAX_LEN)
        kw.setdefault("device", torch.device("cuda", torch.cuda.current_device()))
        kw.setdefault("exact", True)
        self._inner = backend_class(self.variant, self.bits)(self.layer_index, self.policy, self.head_dim,
                                              self.group_size, hidden_dim=d,
                                              n_heads=d // HEAD_DIM, kv_group=d // kvw, **kw)
        if self._first_channel:
            self._inner.set_fp16_first_channel(True)

    def _rows(self, x, weights):
        is_np = not isinstance(x, torch.Tensor)
        x = torch.as_tensor(np.asarray(x, np.float64) if is_np else x)
        lw = as_layer_weights(weights, self._kw.get("device"))
        if self._inner is None:
            self._build(x.shape[-1], lw)
        return x.to(self._inner.device), lw, is_np

    def prefill(self, x, weights, acc=None):
        x, lw, is_np = self._rows(x, weights)
        if x.dim() != 2:
            raise ShapeError("prefill expects [n, d]")
        self._np = is_np
        self._inner.prefill(x, lw, acc, slot=0)

    def decode_append(self, x_token, weights, acc=None):
        x, lw, is_np = self._rows(x_token, weights)
        self._np = getattr(self, "_np", is_np) and is_np
        self._inner.decode_append(x.reshape(1, -1), lw, acc)

    def rematerialize(self, weights, positions, acc=None):
        if self._inner is None:
            raise UsageError("rematerialize on an empty cache")
        k, v = self._inner.rematerialize(as_layer_weights(weights, self._inner.device), positions,
                                         acc, slot=0)
        if getattr(self, "_np", True):
            return k.double().cpu().numpy(), v.double().cpu().numpy()
        return k, v

    def memory_bytes(self) -> dict:
        return {} if self._inner is None else self._inner.memory_bytes()


# Free-function surface mirroring the backend methods (cache.py:633-650).


def prefill(state, x_postnorm, weights, acc=None):
    state.prefill(x_postnorm, weights, acc)
    return state


def decode_append(state, x_token, weights, acc=None):
    state.decode_append(x_token, weights, acc)
    return state


def rematerialize(state, weights, positions, acc=None):
    return state.rematerialize(weights, positions, acc)
