"""Multi-GPU decomposition of the decode step.

* Batch sharding (C2, C3): rank r decodes its own contiguous slice of the
  sequences with a full weight replica; sequences are independent
  (SPEC.md:305), so there is no collective in the decode loop.
* KV-head-group sharding (C4): rank r owns a contiguous block of KV heads.
  It holds W_k / W_v columns for those heads (xq-mha) or fused_k / fused_v
  columns (xq-gqa, linalg.py:118-126), and the W_q columns of their query
  heads. The X / latent cache is replicated: every KV head's K uses all
  channels of X (cache.py:385-387, 434-437), so every rank quantizes the same
  row. After the fused attention each rank holds [B, H/world, 128]; one
  all-gather per layer assembles [B, H, 128] for the replicated W_o.
  * ``HeadGather``: ``all_gather_into_tensor`` (NCCL on GPUs, gloo in tests).
  * ``PeerHeadGather``: torch symmetric memory. The fused kernel's projection
    stores this rank's [B, H/world, 128] straight into its slot of every rank's
    buffer through peer pointers (NVLink), then one device-side barrier. There is
    no separate collective launch. The buffers alternate per layer, so the next
    layer's stores never land in a buffer a slower rank is still reading.

One process per GPU, torch.distributed (NCCL on GPUs, gloo on CPU in tests).
"""

from __future__ import annotations

from dataclasses import replace

import torch

from .cache import HEAD_DIM, LayerWeights
from .errors import ConfigError


def batch_shard(n_seqs: int, world: int, rank: int) -> range:
    """Contiguous block of sequence indices owned by ``rank``."""
    if not 0 <= rank < world:
        raise ConfigError(f"rank {rank} outside world {world}")
    per, extra = divmod(n_seqs, world)
    start = rank * per + min(rank, extra)
    return range(start, start + per + (1 if rank < extra else 0))


def head_shard(n_kv_heads: int, world: int, rank: int) -> range:
    """Contiguous block of KV heads owned by ``rank`` (equal split required)."""
    if n_kv_heads % world:
        raise ConfigError(f"{n_kv_heads} KV heads do not split over {world} ranks")
    per = n_kv_heads // world
    return range(rank * per, (rank + 1) * per)


def _cols(kv_heads: range, head_dim: int = HEAD_DIM) -> slice:
    return slice(kv_heads.start * head_dim, kv_heads.stop * head_dim)


def shard_layer_weights(lw: LayerWeights, variant: str, kv_heads: range) -> LayerWeights:
    """Column slice of one layer's K/V projections for ``kv_heads``.

    xq-mha / xq-cl-mha / fp16: W_k, W_v columns. xq-gqa: fused_k / fused_v
    columns; the latent projections U_k / U_v stay whole (replicated cache)."""
    c = _cols(kv_heads)
    out = replace(lw, _cache={})
    if lw.w_k is not None:
        out.w_k = lw.w_k[:, c].contiguous()
        out.w_v = lw.w_v[:, c].contiguous()
    if variant == "xq-gqa":
        out.fused_k = lw.fused_k[:, c].contiguous()
        out.fused_v = lw.fused_v[:, c].contiguous()
    return out


def shard_wq(w_q: torch.Tensor, kv_heads: range, kv_group: int) -> torch.Tensor:
    """W_q columns of the query heads served by ``kv_heads`` (head h -> kv h // g)."""
    q = range(kv_heads.start * kv_group, kv_heads.stop * kv_group)
    return w_q[:, _cols(q)].contiguous()


class HeadGather:
    """All-gather of per-rank attention outputs [B, H_local, 128] -> [B, H, 128].

    Uses one preallocated flat buffer and ``all_gather_into_tensor`` (NCCL or
    gloo); rank r's heads land at [r*H_local, (r+1)*H_local)."""

    def __init__(self, n_seqs: int, n_heads_local: int, world: int, device, group=None):
        self.world, self.group = world, group
        self.h = n_heads_local
        self.buf = torch.empty((world, n_seqs, n_heads_local, HEAD_DIM), dtype=torch.float32,
                               device=device)

    def __call__(self, local: torch.Tensor) -> torch.Tensor:
        import torch.distributed as dist

        local = local.contiguous()
        if self.world == 1:
            return local
        dist.all_gather_into_tensor(self.buf.view(-1), local.view(-1), group=self.group)
        # [world, B, H_local, 128] -> [B, world*H_local, 128]
        return self.buf.permute(1, 0, 2, 3).reshape(local.shape[0], self.world * self.h, HEAD_DIM)


class PeerHeadGather:
    """KV-head-group gather by peer stores (torch symmetric memory over NVLink).

    ``out_ptrs(i)`` are the device addresses of this rank's slot in every rank's
    buffer for layer i. The decoder hands them to the fused kernel
    (``xq_decode_attend_absorbed_peers``), and ``finish(i)`` is the barrier plus
    the [B, H, 128] view. ``__call__`` covers the unabsorbed kernel: the local
    output is copied into the peers' slots and then the same barrier runs.
    """

    peer = True

    def __init__(self, n_seqs: int, n_heads_local: int, world: int, rank: int, device,
                 group=None):
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm

        self.world, self.rank, self.h, self.n_seqs = world, rank, n_heads_local, n_seqs
        self.shape = (world, n_seqs, n_heads_local, HEAD_DIM)
        torch.cuda.set_device(device)  # symmetric allocations land on the current device
        name = (group or dist.group.WORLD).group_name
        self.bufs = [symm.empty(self.shape, dtype=torch.float32, device=device) for _ in range(2)]
        self.hdls = [symm.rendezvous(b, name) for b in self.bufs]
        slot = n_seqs * n_heads_local * HEAD_DIM * 4
        self._ptrs, self._offs = [], []
        for b, hdl in zip(self.bufs, self.hdls):
            off = b.data_ptr() - hdl.buffer_ptrs[rank]  # the tensor inside its allocation
            self._offs.append(off // 4)
            self._ptrs.append([hdl.buffer_ptrs[p] + off + rank * slot for p in range(world)])

    def out_ptrs(self, layer: int) -> list[int]:
        return self._ptrs[layer % 2]

    def finish(self, layer: int) -> torch.Tensor:
        self.hdls[layer % 2].barrier(channel=0)
        return gathered_view(self.bufs[layer % 2])

    def __call__(self, local: torch.Tensor, layer: int = 0) -> torch.Tensor:
        hdl, off = self.hdls[layer % 2], self._offs[layer % 2]
        for p in range(self.world):  # the same addresses out_ptrs() hands the kernel
            hdl.get_buffer(p, self.shape, torch.float32, storage_offset=off)[self.rank].copy_(local)
        return self.finish(layer)


def gathered_view(buf: torch.Tensor) -> torch.Tensor:
    """[world, B, H_local, 128] -> [B, world*H_local, 128] (rank r's heads at r*H_local)."""
    world, n, h, d = buf.shape
    return buf.permute(1, 0, 2, 3).reshape(n, world * h, d)
