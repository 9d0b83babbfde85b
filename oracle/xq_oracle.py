"""CPU oracle for the XQuant decode hot path -- TEST INFRASTRUCTURE ONLY.

This module is a float64 NumPy restatement of the reference's algorithm
(package ``xcache``, /root/reference/pkg/src/xcache). Only ``tests/``,
``__graft_entry__.smoke()`` and the ``cpu_baseline`` / ``--impl reference``
legs of ``bench.py`` may import it, and only as the checker or as the timed
CPU baseline -- never as the product path. The product path
(``paper_2508_10395_b200``) runs on sm_100a CUDA and fails loudly when its
extension is missing.

Pinning: every function here is checked against golden vectors produced by
the reference itself (``tests/golden/make_golden.py`` imports the reference
from ``oracle/_ref`` or ``/root/reference``), see ``tests/test_oracle.py``.

Each function cites the reference file:line it restates.
"""

from __future__ import annotations

import math

import numpy as np

ROPE_THETA = 10000.0  # linalg.py:18
VALID_BITS = (2, 3, 4, 8, 16)  # quant.py:25
PASSTHROUGH_BITS = 16  # quant.py:26
PER_TOKEN, PER_CHANNEL = 0, 1  # quant.py:32-34
DEFAULT_GROUP_SIZE = 128  # cache.py:44


# ---------------------------------------------------------------------------
# Bit packing: _kernels/fallback.py:58-94 (_native.pyx:64-108)
# ---------------------------------------------------------------------------


def pack_codes(codes: np.ndarray, bits: int) -> np.ndarray:
    """LSB-first little-endian u64 bit stream; element i at bits [i*e,(i+1)*e).

    Restates fallback.py:58-79: bit k of the stream lives at position
    ``k & 63`` of word ``k >> 6``.
    """
    codes = np.ascontiguousarray(codes, dtype=np.uint8).reshape(-1)
    n = codes.shape[0]
    if n == 0:
        return np.zeros(0, dtype=np.uint64)
    n_words = (n * bits + 63) // 64
    words = np.zeros(n_words, dtype=np.uint64)
    off = np.arange(n, dtype=np.uint64) * np.uint64(bits)
    w = (off >> np.uint64(6)).astype(np.int64)
    s = off & np.uint64(63)
    c = codes.astype(np.uint64)
    np.bitwise_or.at(words, w, c << s)
    spill = (s.astype(np.int64) + bits) > 64
    if spill.any():
        np.bitwise_or.at(words, w[spill] + 1, c[spill] >> (np.uint64(64) - s[spill]))
    return words


def unpack_codes(words: np.ndarray, bits: int, n: int) -> np.ndarray:
    """Inverse of :func:`pack_codes` (fallback.py:82-94)."""
    if n == 0:
        return np.zeros(0, dtype=np.uint8)
    words = np.ascontiguousarray(words, dtype=np.uint64)
    off = np.arange(n, dtype=np.uint64) * np.uint64(bits)
    w = (off >> np.uint64(6)).astype(np.int64)
    s = off & np.uint64(63)
    vals = words[w] >> s
    spill = (s.astype(np.int64) + bits) > 64
    if spill.any():
        vals[spill] |= words[w[spill] + 1] << (np.uint64(64) - s[spill])
    return (vals & np.uint64((1 << bits) - 1)).astype(np.uint8)


def pack_rows(codes: np.ndarray, bits: int) -> np.ndarray:
    """Pack every row of a [rows, cols] code matrix independently.

    The GPU arena stores each token row as ``pack_codes(row)`` (bytes); this
    helper produces the same bytes for comparison. Returns uint8
    [rows, ceil(cols*bits/64)*8].
    """
    rows = codes.shape[0]
    out = [pack_codes(codes[r], bits).view(np.uint8) for r in range(rows)]
    return np.stack(out) if rows else np.zeros((0, 0), np.uint8)


# ---------------------------------------------------------------------------
# Grouped asymmetric quantization: fallback.py:102-146 (_native.pyx:111-177)
# ---------------------------------------------------------------------------


def _group_edges(length: int, group_size: int):
    starts = np.arange(0, length, group_size)  # fallback.py:102-105
    reps = np.diff(np.append(starts, length))
    return starts, reps


def quantize_groups(x: np.ndarray, group_size: int, bits: int):
    """Per row, contiguous groups of ``group_size`` (fallback.py:108-131).

    scale = (max-min)/(2^e-1) or 1 for a degenerate group; zp = min;
    code = clamp(floor((x-min)/scale + 0.5), 0, 2^e-1), all in float64.
    """
    x = np.ascontiguousarray(x, dtype=np.float64)
    rows, cols = x.shape
    starts, reps = _group_edges(cols, group_size)
    mins = np.minimum.reduceat(x, starts, axis=1)
    maxs = np.maximum.reduceat(x, starts, axis=1)
    qmax = float(2**bits - 1)
    spans = maxs - mins
    with np.errstate(invalid="ignore"):
        scales = np.where(spans == 0.0, 1.0, spans / qmax)
    v = (x - np.repeat(mins, reps, axis=1)) / np.repeat(scales, reps, axis=1)
    q = np.floor(v + 0.5)
    np.clip(q, 0.0, qmax, out=q)
    return q.astype(np.uint8), scales, mins.copy()


def dequantize_groups(codes, scales, zero_points, group_size: int) -> np.ndarray:
    """``code * scale + zero_point`` in float64 (fallback.py:134-146)."""
    _, cols = codes.shape
    _, reps = _group_edges(cols, group_size)
    return codes.astype(np.float64) * np.repeat(scales, reps, axis=1) + np.repeat(
        zero_points, reps, axis=1
    )


def quantize(t: np.ndarray, bits: int, axis: int = PER_TOKEN, group_size: int = 128):
    """quant.quantize (quant.py:104-134): per-channel = transposed per-token.

    Returns ``(codes, scales, zps)``; for bits=16 returns ``(data, None, None)``.
    """
    t = np.ascontiguousarray(t, dtype=np.float64)
    if not np.all(np.isfinite(t)):
        raise ValueError("input contains NaN or Inf")  # quant.py:114-115
    if bits == PASSTHROUGH_BITS:
        return t.copy(), None, None
    if axis == PER_TOKEN:
        return quantize_groups(t, group_size, bits)
    c, s, z = quantize_groups(np.ascontiguousarray(t.T), group_size, bits)
    return (np.ascontiguousarray(c.T), np.ascontiguousarray(s.T), np.ascontiguousarray(z.T))


def dequantize(codes, scales, zps, bits: int, axis: int = PER_TOKEN, group_size: int = 128):
    """quant.dequantize (quant.py:137-153)."""
    if bits == PASSTHROUGH_BITS:
        return np.array(codes, dtype=np.float64)
    if codes.shape[0] == 0:
        return np.zeros((0, codes.shape[1]))
    if axis == PER_TOKEN:
        return dequantize_groups(codes, scales, zps, group_size)
    out = dequantize_groups(
        np.ascontiguousarray(codes.T), np.ascontiguousarray(scales.T),
        np.ascontiguousarray(zps.T), group_size,
    )
    return np.ascontiguousarray(out.T)


# ---------------------------------------------------------------------------
# RoPE (linalg.py:58-95) and decode attention (model.py:150-182)
# ---------------------------------------------------------------------------


def apply_rope(m: np.ndarray, positions, head_dim: int, theta_base: float = ROPE_THETA):
    """Interleaved-pair rotary embedding (linalg.py:58-95).

    Pair (2j, 2j+1) of every head is rotated by pos * theta^(-2j/head_dim).
    """
    m = np.asarray(m, dtype=np.float64)
    positions = np.asarray(positions, dtype=np.float64).reshape(-1)
    n_rows, n_cols = m.shape
    n_heads = n_cols // head_dim
    half = head_dim // 2
    freqs = theta_base ** (-2.0 * np.arange(half) / head_dim)
    angles = positions[:, None] * freqs[None, :]
    cos = np.cos(angles)[:, None, :]
    sin = np.sin(angles)[:, None, :]
    pairs = m.reshape(n_rows, n_heads, half, 2)
    even, odd = pairs[..., 0], pairs[..., 1]
    out = np.empty_like(pairs)
    out[..., 0] = even * cos - odd * sin
    out[..., 1] = even * sin + odd * cos
    return out.reshape(n_rows, n_cols)


def rope_tables(n_pos: int, head_dim: int, theta_base: float = ROPE_THETA):
    """cos/sin tables [n_pos, head_dim/2] in float64, as linalg.py:84-88 forms them."""
    half = head_dim // 2
    freqs = theta_base ** (-2.0 * np.arange(half) / head_dim)
    ang = np.arange(n_pos, dtype=np.float64)[:, None] * freqs[None, :]
    return np.cos(ang), np.sin(ang)


def attention(q, k, v, n_heads: int, kv_group: int) -> np.ndarray:
    """Causal grouped softmax attention (model.py:150-182).

    Query rows are the trailing rows of the key timeline; at decode the
    single query row sees every key (no mask).
    """
    q = np.asarray(q, np.float64)
    k = np.asarray(k, np.float64)
    v = np.asarray(v, np.float64)
    l_q, d = q.shape
    l_k = k.shape[0]
    head_dim = d // n_heads
    offset = l_k - l_q
    scale = 1.0 / np.sqrt(head_dim)
    blocked = np.arange(l_k)[None, :] > np.arange(l_q)[:, None] + offset
    out = np.empty((l_q, d))
    for h in range(n_heads):
        kv_h = h // kv_group
        qh = q[:, h * head_dim:(h + 1) * head_dim]
        kh = k[:, kv_h * head_dim:(kv_h + 1) * head_dim]
        vh = v[:, kv_h * head_dim:(kv_h + 1) * head_dim]
        scores = (qh @ kh.T) * scale
        scores[blocked] = -np.inf
        scores -= scores.max(axis=1, keepdims=True)
        w = np.exp(scores)
        w /= w.sum(axis=1, keepdims=True)
        out[:, h * head_dim:(h + 1) * head_dim] = w @ vh
    return out


# ---------------------------------------------------------------------------
# Layer policy (cache.py:70-121)
# ---------------------------------------------------------------------------


def policy_for_bits(bits: int, n_layers: int, prefix: int = 3, prefix_bits: int = 4):
    """LayerPolicy.for_bits (cache.py:89-112): returns (per-layer bits, base_layers)."""
    if bits == 16:
        return [16] * n_layers, min(prefix, n_layers)
    per_layer = [max(bits, prefix_bits) if i < prefix else bits for i in range(n_layers)]
    return per_layer, min(prefix, n_layers)


# ---------------------------------------------------------------------------
# Payload stream (cache.py:154-230)
# ---------------------------------------------------------------------------


class Stream:
    """A quantized payload fed row by row (cache.py:154-230).

    Per-channel payloads always buffer (groups span tokens, cache.py:173);
    per-token payloads of xq-mha / xq-cl-mha / xq-gqa-V are unbuffered.
    """

    def __init__(self, bits: int, axis: int, width: int, group_size: int, buffered: bool,
                 params_f16: bool = False, keep_first_channel: bool = False):
        """``params_f16``: dequantize with the scale / zero point rounded to fp16,
        the storage format of the B200 arena (the reference charges 16+16 bits per
        group, quant.py:44-45, but keeps float64 in memory)."""
        self.params_f16 = params_f16
        # channel 0 verbatim, the rest quantized (cache.py:174-177, 184-189, 223-230)
        self.keep_first = keep_first_channel and bits != 16
        self.first = np.zeros(0)
        self.bits, self.axis, self.width, self.g = bits, axis, width, group_size
        stored = width - 1 if self.keep_first else width
        self.buffered = buffered or axis == PER_CHANNEL  # cache.py:173
        self.codes = np.zeros((0, stored), np.uint8) if bits != 16 else np.zeros((0, stored))
        ngrid = (0, -(-stored // group_size)) if axis == PER_TOKEN else (0, stored)
        self.scales = np.zeros(ngrid)
        self.zps = np.zeros(ngrid)
        self.buf = np.zeros((0, width))

    def __len__(self):
        return self.codes.shape[0] + self.buf.shape[0]

    def _flush(self, block):  # cache.py:184-189 -> quant.append_rows (quant.py:210-228)
        if self.keep_first:
            self.first = np.concatenate([self.first, block[:, 0]])
            block = np.ascontiguousarray(block[:, 1:])
        c, s, z = quantize(block, self.bits, self.axis, self.g)
        self.codes = np.vstack([self.codes, c])
        if s is not None:
            self.scales = np.vstack([self.scales, s])
            self.zps = np.vstack([self.zps, z])

    def bulk(self, mat):  # cache.py:191-208
        mat = np.asarray(mat, np.float64)
        if self.axis == PER_TOKEN:
            self._flush(mat)
            return
        g = self.g
        block = np.vstack([self.buf, mat]) if len(self.buf) else mat
        n_full = block.shape[0] // g * g
        for i in range(0, n_full, g):
            self._flush(block[i:i + g])
        self.buf = np.array(block[n_full:], dtype=np.float64)

    def push(self, row):  # cache.py:210-221
        row = np.asarray(row, np.float64).reshape(1, -1)
        if not self.buffered:
            self._flush(row)
            return
        self.buf = np.vstack([self.buf, row])
        if self.buf.shape[0] >= self.g:
            self._flush(self.buf)
            self.buf = np.zeros((0, self.width))

    def reconstruct(self):  # cache.py:223-230
        sc, zp = self.scales, self.zps
        if self.params_f16 and self.bits != 16:
            sc, zp = sc.astype(np.float16).astype(np.float64), zp.astype(np.float16).astype(np.float64)
        flushed = dequantize(self.codes, sc, zp, self.bits, self.axis, self.g)
        if self.keep_first:
            flushed = np.hstack([self.first[:, None], flushed])
        if len(self.buf):
            return np.vstack([flushed, self.buf])
        return flushed


# ---------------------------------------------------------------------------
# Cache backends on the hot path (cache.py:302-535)
# ---------------------------------------------------------------------------


class Fp16Cache:
    """FullPrecisionCache "fp16" (cache.py:302-323): pre-RoPE K and V verbatim."""

    def __init__(self, head_dim):
        self.hd = head_dim
        self.k_pre = None
        self.v = None

    def append(self, x, w_k, w_v):
        x = np.atleast_2d(np.asarray(x, np.float64))
        k, v = x @ w_k, x @ w_v
        self.k_pre = k if self.k_pre is None else np.vstack([self.k_pre, k])
        self.v = v if self.v is None else np.vstack([self.v, v])

    def remat(self):
        n = self.k_pre.shape[0]
        return apply_rope(self.k_pre, np.arange(n), self.hd), self.v.copy()


class KvqCache:
    """QuantizedKvCache "kvq" (cache.py:326-360): pre-RoPE K per-channel and V
    per-token, both buffered (cache.py:336-342); K/V given pre-projected."""

    def __init__(self, bits, head_dim, group_size=128):
        self.hd = head_dim
        self.bits, self.g = bits, group_size
        self.k = None
        self.v = None

    def _ensure(self, width):
        if self.k is None:
            self.k = Stream(self.bits, PER_CHANNEL, width, self.g, buffered=True)
            self.v = Stream(self.bits, PER_TOKEN, width, self.g, buffered=True)

    def prefill(self, k, v):  # cache.py:344-349
        self._ensure(k.shape[1])
        self.k.bulk(k)
        self.v.bulk(v)

    def push(self, k_row, v_row):  # cache.py:351-354
        self._ensure(np.asarray(k_row).reshape(-1).shape[0])
        self.k.push(k_row)
        self.v.push(v_row)

    def remat(self):  # cache.py:356-360
        k = self.k.reconstruct()
        return apply_rope(k, np.arange(k.shape[0]), self.hd), self.v.reconstruct()


class XqMhaCache:
    """InputCacheMHA "xq-mha" (cache.py:363-387): per-token X, unbuffered."""

    def __init__(self, bits, head_dim, group_size=128):
        self.hd = head_dim
        self.bits, self.g = bits, group_size
        self.stream = None

    def append(self, x):  # prefill (bulk) and decode (push) give identical codes
        x = np.atleast_2d(np.asarray(x, np.float64))
        if self.stream is None:
            self.stream = Stream(self.bits, PER_TOKEN, x.shape[1], self.g, buffered=False)
        self.stream.bulk(x)

    def remat(self, w_k, w_v):  # cache.py:385-387
        x_hat = self.stream.reconstruct()
        n = x_hat.shape[0]
        return apply_rope(x_hat @ w_k, np.arange(n), self.hd), x_hat @ w_v


class XqGqaCache:
    """LatentInputCacheGQA "xq-gqa" (cache.py:390-437).

    K latent = x @ U_k quantized per-channel (buffered, flush every G rows);
    V latent = x @ U_v per-token. Remat through fused = diag(sigma) B^T.
    """

    def __init__(self, bits, head_dim, group_size=128, fp16_first_channel=False, params_f16=False):
        self.hd = head_dim
        self.bits, self.g = bits, group_size
        self.first = fp16_first_channel  # cache.py:403-409
        self.params_f16 = params_f16
        self.k_stream = None
        self.v_stream = None

    def _ensure(self, r):
        if self.k_stream is None:
            self.k_stream = Stream(self.bits, PER_CHANNEL, r, self.g, buffered=True,
                                   keep_first_channel=self.first, params_f16=self.params_f16)
            self.v_stream = Stream(self.bits, PER_TOKEN, r, self.g, buffered=False,
                                   params_f16=self.params_f16)

    def prefill(self, lat_k, lat_v):  # cache.py:422-427 (latents precomputed)
        self._ensure(lat_k.shape[1])
        self.k_stream.bulk(lat_k)
        self.v_stream.bulk(lat_v)

    def push(self, lat_k_row, lat_v_row):  # cache.py:429-432
        self._ensure(np.asarray(lat_k_row).reshape(-1).shape[0])
        self.k_stream.push(lat_k_row)
        self.v_stream.push(lat_v_row)

    def remat(self, fused_k, fused_v):  # cache.py:434-437
        k_pre = self.k_stream.reconstruct() @ fused_k
        v = self.v_stream.reconstruct() @ fused_v
        n = k_pre.shape[0]
        return apply_rope(k_pre, np.arange(n), self.hd), v


def svd_factors(w: np.ndarray):
    """Thin SVD w = U diag(sigma) B^T with the reference sign convention.

    The reference uses one-sided Jacobi (linalg.py:129-178); we use LAPACK and
    apply the same determinism rule: each column of U is signed so its
    largest-magnitude entry (lowest index on ties) is positive
    (linalg.py:171-176). Returns (u, sigma, b_t, fused = diag(sigma) b_t)
    (linalg.py:103-126).
    """
    u, s, vt = np.linalg.svd(np.asarray(w, np.float64), full_matrices=False)
    for j in range(u.shape[1]):
        i = int(np.argmax(np.abs(u[:, j])))
        if u[i, j] < 0:
            u[:, j] = -u[:, j]
            vt[j] = -vt[j]
    return u, s, vt, s[:, None] * vt


class XqClMhaStack:
    """DeltaInputCacheMHA "xq-cl-mha" over a whole layer stack (cache.py:440-535).

    Layers < base_layers cache X directly (per-token); layer base-1 seeds the
    accumulator with its full reconstruction; delta layer i caches
    delta = x - acc[pos] and then acc += reconstruct(all deltas of layer i)
    (cache.py:460-481). Remat of a delta layer reads the accumulator
    (cache.py:531-535). The accumulator is transient per forward pass
    (model.py:228).
    """

    def __init__(self, bits_per_layer, base_layers, head_dim, group_size=128, params_f16=False):
        self.bits = list(bits_per_layer)
        self.base = base_layers
        self.hd = head_dim
        self.g = group_size
        self.params_f16 = params_f16
        self.streams = [None] * len(self.bits)
        self.n_tokens = 0

    def _stream(self, i, width):
        if self.streams[i] is None:
            self.streams[i] = Stream(self.bits[i], PER_TOKEN, width, self.g, buffered=False,
                                     params_f16=self.params_f16)
        return self.streams[i]

    def step(self, xs, weights=None, on_layer=None, keep=True):
        """Append rows ``xs[i]`` ([n_new, d]) to every layer in order.

        Returns the per-layer accumulator snapshots (None for base layers
        before the seed) and, when ``weights`` (list of (w_k, w_v)) is
        given, the per-layer remat (K, V). ``xs`` may be an iterable that
        produces the layers one at a time; ``on_layer(i, src)`` receives each
        layer's remat source (x_hat or the accumulator) as it is formed, and
        ``keep=False`` skips the snapshots (full-size runs).
        """
        acc = None
        accs, kvs = [], []
        n_new = None
        for i, x in enumerate(xs):
            x = np.atleast_2d(np.asarray(x, np.float64))
            st = self._stream(i, x.shape[1])
            if i < self.base:
                st.bulk(x)
                x_hat = st.reconstruct()
                if i == self.base - 1:
                    acc = x_hat.copy()  # cache.py:463-467 / 473-477
                if keep:
                    accs.append(acc.copy() if acc is not None else None)
                src = x_hat
            else:
                pos = self.n_tokens
                delta = x - acc[pos:pos + x.shape[0]]  # cache.py:468, 478-479
                st.bulk(delta)
                acc = acc + st.reconstruct()  # cache.py:470, 481
                if keep:
                    accs.append(acc.copy())
                src = acc
            n_new = x.shape[0]
            if on_layer is not None:
                on_layer(i, src)
            if weights is not None:
                w_k, w_v = weights[i]
                n = src.shape[0]
                kvs.append((apply_rope(src @ w_k, np.arange(n), self.hd), src @ w_v))
        self.n_tokens += n_new
        return accs, kvs


class XqClGqaStack:
    """DeltaLatentCacheGQA "xq-cl-gqa" over a layer stack (cache.py:538-604).

    Every layer caches a per-channel (buffered) latent in the shared K|V
    subspace U_kv of svd([W_k | W_v]) (model.py:135-142). Base layers cache
    x @ U (cache.py:562-569); layer base-1 seeds the d-wide accumulator with
    reconstruct() @ U^T (cache.py:571-572 via _DeltaBackend, :463-467). A
    delta layer caches (x - acc[pos]) @ U (cache.py:574-586) and then adds
    reconstruct() @ U^T to the accumulator (cache.py:588-589). Remat: base
    kv = reconstruct() @ fused (cache.py:591-593); delta kv = (acc @ U) @ fused
    (cache.py:595-598); K = RoPE(kv[:, :kvw]), V = kv[:, kvw:] (cache.py:600-604).
    """

    def __init__(self, bits_per_layer, base_layers, head_dim, group_size=128, params_f16=False):
        self.bits = list(bits_per_layer)
        self.base = base_layers
        self.hd = head_dim
        self.g = group_size
        self.params_f16 = params_f16
        self.streams = [None] * len(self.bits)
        self.n_tokens = 0

    def _stream(self, i, width):
        if self.streams[i] is None:
            self.streams[i] = Stream(self.bits[i], PER_CHANNEL, width, self.g, buffered=True,
                                     params_f16=self.params_f16)
        return self.streams[i]

    def step(self, xs, subspaces):
        """Append rows ``xs[i]`` ([n_new, d]) to every layer in order.

        ``subspaces[i]`` = (u, fused) of layer i (u: d x r, fused: r x 2*kvw).
        Returns per-layer (latent rows quantized by this call, K, V, acc)."""
        acc = None
        out = []
        for i, x in enumerate(xs):
            x = np.atleast_2d(np.asarray(x, np.float64))
            u, fused = subspaces[i]
            st = self._stream(i, u.shape[1])
            n_new = x.shape[0]
            if i < self.base:
                lat = x @ u
                st.bulk(lat)
                if i == self.base - 1:
                    acc = st.reconstruct() @ u.T
                kv = st.reconstruct() @ fused
            else:
                pos = self.n_tokens
                lat = (x - acc[pos:pos + n_new]) @ u
                st.bulk(lat)
                acc = acc + st.reconstruct() @ u.T
                kv = (acc @ u) @ fused
            kvw = fused.shape[1] // 2
            n = kv.shape[0]
            out.append((lat, apply_rope(kv[:, :kvw], np.arange(n), self.hd), kv[:, kvw:],
                        None if acc is None else acc.copy()))
        self.n_tokens += np.atleast_2d(xs[0]).shape[0]
        return out


# ---------------------------------------------------------------------------
# Performance / footprint model (sysmodel.py:85-196) -- metric definitions
# ---------------------------------------------------------------------------


def remat_flops(variant: str, seq_len: int, hidden_dim: int, kv_group: int = 1) -> float:
    """Per-layer remat FLOPs (sysmodel.py:85-102)."""
    d = hidden_dim
    kvw = d / kv_group
    if variant in ("fp16", "kvq"):
        return 0.0
    if variant == "xq-mha":
        return 4.0 * seq_len * d**2
    if variant == "xq-gqa":
        return 4.0 * seq_len * kvw**2
    if variant == "xq-cl-mha":
        return 4.0 * seq_len * d**2 + 2.0 * seq_len * d
    if variant == "xq-cl-gqa":
        return 8.0 * seq_len * kvw * d
    raise ValueError(variant)


def cache_bytes(variant: str, seq_len: int, hidden_dim: int, bits: int,
                kv_group: int = 1, accum_bits: int = 4) -> float:
    """Per-layer cache traffic per decode step (sysmodel.py:105-124)."""
    d = hidden_dim
    kvw = d / kv_group
    e = bits
    if variant == "fp16":
        return 2.0 * 2.0 * seq_len * kvw
    if variant == "kvq":
        return 2.0 * (e / 8.0) * seq_len * kvw
    if variant == "xq-mha":
        return (e / 8.0) * seq_len * d
    if variant == "xq-gqa":
        return 2.0 * (e / 8.0) * seq_len * kvw
    if variant == "xq-cl-mha":
        return (e / 8.0) * seq_len * d + (accum_bits / 8.0) * seq_len * d
    if variant == "xq-cl-gqa":
        return 2.0 * (e / 8.0) * seq_len * kvw + (accum_bits / 8.0) * seq_len * d
    raise ValueError(variant)


def bits_per_element(bits: int, group_size: int = 128) -> float:
    """quant.bits_per_element (quant.py:58-62): 16-bit scale + 16-bit zp per group."""
    if bits == 16:
        return 16.0
    return bits + 32.0 / group_size


def normalized_kv_size(variant: str, bits_per_layer, kv_group: int = 1,
                       group_size: int = 128) -> float:
    """Footprint per token relative to fp16 K/V (sysmodel.py:161-196)."""
    denom = 32.0
    total = 0.0
    for e in bits_per_layer:
        pe = bits_per_element(e, group_size)
        if variant == "fp16":
            ratio = 1.0
        elif variant in ("kvq", "xq-gqa", "xq-cl-gqa"):
            ratio = 2.0 * pe / denom
        else:
            ratio = kv_group * pe / denom
        total += ratio
    return total / len(bits_per_layer)


def breakeven_length(variant: str, hidden_dim: int, kv_group: int, bits: int,
                     peak_flops: float, mem_bw: float, weight_bytes: float = 0.0,
                     accum_bits: int = 4) -> float:
    """sysmodel.breakeven_length (sysmodel.py:127-158), one-latent convention."""
    p = peak_flops / mem_bw
    a = remat_flops(variant, 1, hidden_dim, kv_group)
    if variant in ("xq-gqa", "xq-cl-gqa"):
        b = (bits / 8.0) * hidden_dim / kv_group
        if variant == "xq-cl-gqa":
            b += (accum_bits / 8.0) * hidden_dim
    else:
        b = cache_bytes(variant, 1, hidden_dim, bits, kv_group, accum_bits)
    slack = a - p * b
    if slack <= 0:
        return math.inf
    return p * weight_bytes / slack
