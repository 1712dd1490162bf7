"""Multi-GPU sharding of the KV codec (one process per GPU).

The KV cache shards naturally by layer or by KV head: every
rank compresses its own shard with no data-path collective.  The only
exchange is an all-gather of one int64 per rank -- the rank's compressed
byte count -- from which every rank derives the global wire offsets
(exclusive scan), so the per-rank payloads can be laid out back to back in
a sender buffer or NIC queue.  Mixed-head labels come from one global
classify_heads on the host (importance is L*H scalars) and are sliced per
rank, so every rank quantizes exactly as the whole-tensor encode would
(quantize.py:126 with head_classes; compress.py:124 classifies per call,
which per-shard calls must not do).

  by="layer": rank r owns layers [l0, l1) of all heads -- with codec none
              the rank payloads, in rank order, ARE the whole-tensor payload;
  by="head":  rank r owns KV heads [h0, h1) of all layers -- the TP layout of
              a serving engine (a GPU holds its heads' cache for every layer);
              each (layer, head) slab's bytes equal the whole-tensor encode's.
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
    """Layer- or head-sharded encode / decode of an (L, H, T, C) cache.

    `codec_factory(strategy_id, local_shape, **kw)` builds the rank's codec
    (default KVCodec); a rank whose share is empty (more ranks than heads)
    has no codec and contributes 0 bytes to the wire.
    """

    def __init__(self, strategy_id: str, shape, rank: int | None = None, world: int | None = None,
                 by: str = "layer", codec_factory=None, **kw) -> None:
        L, H, T, C = (int(v) for v in shape)
        if by not in ("layer", "head"):
            raise ValueError(f"by must be 'layer' or 'head', got {by!r}")
        self.shape = (L, H, T, C)
        self.by = by
        initialized = dist.is_available() and dist.is_initialized()
        self.rank = dist.get_rank() if rank is None and initialized else (rank or 0)
        self.world = dist.get_world_size() if world is None and initialized else (world or 1)
        if by == "layer":
            (self.l0, self.l1), (self.h0, self.h1) = shard_range(L, self.world, self.rank), (0, H)
        else:
            (self.l0, self.l1), (self.h0, self.h1) = (0, L), shard_range(H, self.world, self.rank)
        self.local_shape = (self.l1 - self.l0, self.h1 - self.h0, T, C)
        self.empty = min(self.local_shape) == 0
        if codec_factory is None:
            from paper_2605_13734_b200.codec import KVCodec

            codec_factory = KVCodec
        self.codec = None if self.empty else codec_factory(strategy_id, self.local_shape, **kw)

    def local_slice(self, kv_global):
        """This rank's shard of a global (L, H, T, C) tensor, contiguous."""
        v = kv_global[self.l0:self.l1, self.h0:self.h1]
        return v.contiguous() if isinstance(v, torch.Tensor) else np.ascontiguousarray(v)

    def local_classes(self, global_classes):
        """The rank's slice of the GLOBAL head labels (classify_heads over all L*H)."""
        if global_classes is None:
            return None
        return np.ascontiguousarray(np.asarray(global_classes, dtype=bool)[self.l0:self.l1, self.h0:self.h1])

    def encode(self, local_kv, global_classes=None, out=None, stream=None):
        if self.codec is None:
            return None
        return self.codec.encode(local_kv, head_classes=self.local_classes(global_classes), out=out, stream=stream)

    def decode(self, blob, out=None, stream=None, device_length: bool = False):
        if self.codec is None:
            return None
        return self.codec.decode(blob, out=out, stream=stream, device_length=device_length)

    @staticmethod
    def wire_bytes(blob) -> int:
        """Bytes this rank puts on the wire: payload + metadata + block table."""
        if blob is None:
            return 0
        return int(blob.payload_nbytes() + blob.metadata.numel() + blob.framing_nbytes)

    def wire_layout(self, blob, group=None, device=None) -> tuple[int, int]:
        """(this rank's offset in the global wire buffer, global total bytes):
        the one collective of the sharded path (an int64 all-gather)."""
        offs, total = global_offsets(self.wire_bytes(blob), group=group, device=device)
        return offs[self.rank if len(offs) > 1 else 0], total
