"""Multi-GPU sharding of the KV codec (one process per GPU).

The KV cache shards naturally by layer (or KV head): every rank compresses
its own (L/N, H, T, C) shard with no data-path collective.  The only
exchange is an all-gather of one int64 per rank — the rank's compressed
byte count — from which every rank derives the global wire offsets
(exclusive scan), so the per-rank payloads can be laid out back to back in
a sender buffer or NIC queue.  Mixed-head labels come from one global
classify_heads on the host (importance is L*H scalars) and are sliced per
rank, so sharded encodes equal the whole-tensor encode.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

__all__ = ["shard_range", "global_offsets", "ShardedCodec"]


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """[start, end) of rank's contiguous share of n units (layers or heads)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def global_offsets(local_bytes: int, group=None, device=None) -> tuple[list[int], int]:
    """All-gather per-rank byte counts; returns (offsets per rank, total)."""
    if not dist.is_available() or not dist.is_initialized():
        return [0], int(local_bytes)
    world = dist.get_world_size(group)
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else torch.device("cpu")
    mine = torch.tensor([int(local_bytes)], dtype=torch.int64, device=device)
    allv = torch.empty(world, dtype=torch.int64, device=device)
    dist.all_gather_into_tensor(allv, mine, group=group)
    sizes = allv.cpu().tolist()
    offs = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64).tolist()
    return offs, int(sum(sizes))


class ShardedCodec:
    """Layer-sharded encode/decode: rank r owns layers [l0, l1) of an
    (L, H, T, C) cache."""

    def __init__(self, strategy_id: str, shape, rank: int | None = None, world: int | None = None, **kw) -> None:
        from paper_2605_13734_b200.codec import KVCodec

        L, H, T, C = shape
        self.rank = dist.get_rank() if rank is None and dist.is_initialized() else (rank or 0)
        self.world = dist.get_world_size() if world is None and dist.is_initialized() else (world or 1)
        self.l0, self.l1 = shard_range(L, self.world, self.rank)
        self.local_shape = (self.l1 - self.l0, H, T, C)
        self.codec = KVCodec(strategy_id, self.local_shape, **kw)

    def local_classes(self, global_classes):
        if global_classes is None:
            return None
        return np.asarray(global_classes, dtype=bool)[self.l0 : self.l1]

    def encode(self, local_kv, global_classes=None, out=None):
        return self.codec.encode(local_kv, head_classes=self.local_classes(global_classes), out=out)

    def wire_layout(self, blob) -> tuple[int, int]:
        """(this rank's offset in the global wire buffer, global total bytes)."""
        local = blob.payload_nbytes() + blob.metadata.numel() + blob.framing_nbytes
        offs, total = global_offsets(local)
        return offs[self.rank if len(offs) > 1 else 0], total
