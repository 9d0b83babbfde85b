"""Metric definitions of the hot path (the reference's analytical model,
/root/reference/pkg/src/xcache/sysmodel.py), used by bench.py for the
roofline denominators and the compression factor.

* remat FLOPs per layer per sequence (sysmodel.py:85-102), a MAC = 2 FLOPs;
* cache bytes streamed per layer per step (sysmodel.py:105-124);
* normalized K/V footprint (sysmodel.py:161-196) -> compression = 1/size.
"""

from __future__ import annotations


def bits_per_element(bits: int, group_size: int = 128) -> float:
    """quant.bits_per_element (quant.py:58-62): 16-bit scale + 16-bit zp per group."""
    return 16.0 if bits == 16 else bits + 32.0 / group_size


def remat_flops(variant: str, seq_len: int, hidden_dim: int, kv_group: int = 1) -> float:
    d = hidden_dim
    kvw = d / kv_group
    if variant in ("fp16", "kvq"):
        return 0.0
    if variant == "xq-mha":
        return 4.0 * seq_len * d * d
    if variant == "xq-gqa":
        return 4.0 * seq_len * kvw * kvw
    if variant == "xq-cl-mha":
        return 4.0 * seq_len * d * d + 2.0 * seq_len * d
    if variant == "xq-cl-gqa":
        return 8.0 * seq_len * kvw * d
    raise ValueError(variant)


def absorbed_flops(variant: str, seq_len: int, hidden_dim: int, kv_group: int, n_heads: int,
                   head_dim: int = 128) -> float:
    """Tensor-core FLOPs per layer per sequence of the V-absorbed fused kernel
    (csrc/xq_absorb.cu): K remat 2*l*kdim*d_kv, the V-side GEMM
    sum_t p_t x_t 2*l*kdim*H, q.k 2*l*H*hd; the final per-head projection
    through W_v (2*H*kdim*hd, independent of l) is included. kdim = d for the
    X / CL caches, r = d_kv for the GQA latents; xq-cl-gqa counts its delta
    layers (the d-wide accumulator rows, W' = U @ fused)."""
    d = hidden_dim
    kvw = d / kv_group
    if variant in ("xq-mha", "xq-cl-mha", "xq-cl-gqa"):
        kdim = d
    elif variant == "xq-gqa":
        kdim = kvw
    else:
        raise ValueError(variant)
    return (2.0 * seq_len * kdim * kvw + 2.0 * seq_len * kdim * n_heads
            + 2.0 * seq_len * n_heads * head_dim + 2.0 * n_heads * kdim * head_dim)


def attention_flops(seq_len: int, n_heads: int, head_dim: int = 128) -> float:
    """q.K^T and p.V for one decode token: 4 * l * H * hd."""
    return 4.0 * seq_len * n_heads * head_dim


def cache_bytes(variant: str, seq_len: int, hidden_dim: int, bits: int, kv_group: int = 1,
                group_size: int = 128) -> float:
    """Bytes of cache streamed per layer per step incl. the fp16 scale/zp the
    arena stores (the reference's sysmodel charges codes only, :105-124)."""
    d = hidden_dim
    kvw = d / kv_group
    pe = bits_per_element(bits, group_size) / 8.0
    if variant == "fp16":
        return 2.0 * 2.0 * seq_len * kvw
    if variant in ("xq-mha", "xq-cl-mha"):
        return pe * seq_len * d
    if variant in ("xq-gqa", "kvq", "xq-cl-gqa"):  # two kvw-wide latents / the shared r = 2 kvw
        return 2.0 * pe * seq_len * kvw
    raise ValueError(variant)


def normalized_kv_size(variant: str, bits_per_layer, kv_group: int = 1,
                       group_size: int = 128) -> float:
    total = 0.0
    for e in bits_per_layer:
        pe = bits_per_element(e, group_size)
        if variant == "fp16":
            ratio = 1.0
        elif variant in ("kvq", "xq-gqa", "xq-cl-gqa"):
            ratio = 2.0 * pe / 32.0
        else:
            ratio = kv_group * pe / 32.0
        total += ratio
    return total / len(bits_per_layer)


def compression_factor(variant: str, bits_per_layer, kv_group: int = 1) -> float:
    return 1.0 / normalized_kv_size(variant, bits_per_layer, kv_group)
