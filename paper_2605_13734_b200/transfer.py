"""Pipelined compress -> transfer -> decompress between two GPUs
(SURVEY.md §8f rank 3).

The reference's simulator models KV movement as three serial stages
(`engine.py:143-157`: compress, send, decompress; Eq. 1 of the paper charges
V/s_p for the codec).  Here the KV tensor is cut into layer chunks and the
three stages run concurrently on different engines:

    src GPU, stream e:  encode chunk i                  (KVCodec.encode)
    src GPU, stream c:  copy chunk i's wire bytes -> dst (peer stores over
                        NVLink; the payload length stays on the device,
                        kvc_copy_device_length, so nothing syncs to the host)
    dst GPU, stream d:  decode chunk i into the output  (KVCodec.decode with
                        the device-side length)

chained by CUDA events, so chunk i's transfer and decode overlap chunk i+1's
encode.  Each chunk is an independent blob of its (l, H, T, C) slab — the same
per-layer sharding as distributed.py — so the decoded KV equals a whole-tensor
decode bit for bit.
"""

from __future__ import annotations

import torch

from paper_2605_13734_b200 import _native as N
from paper_2605_13734_b200.codec import DeviceBlob, KVCodec, _stream_handle

__all__ = ["PipelinedKVTransfer", "enable_peer_access"]


def enable_peer_access(a: int, b: int) -> None:
    """Let each device read / write the other's memory (no-op for a == b)."""
    if a == b:
        return
    lib = N.lib()
    N.check(lib.kvc_enable_peer_access(int(a), int(b)))
    N.check(lib.kvc_enable_peer_access(int(b), int(a)))


class PipelinedKVTransfer:
    """Move one (L, H, T, C) KV tensor from `src` to `dst` compressed.

    The layer dimension is cut into chunks of `chunk_layers`; plans, wire
    buffers and streams are built once and reused by every `run`.  For
    mixed-head strategies pass the global labels (classify_heads) to `run`.
    """

    def __init__(self, strategy_id: str, shape, src, dst, chunk_layers: int = 8, block_symbols: int = 2048,
                 in_dtype: torch.dtype = torch.bfloat16, out_dtype: torch.dtype = torch.bfloat16) -> None:
        L, H, T, C = (int(v) for v in shape)
        self.shape = (L, H, T, C)
        self.src = torch.device("cuda", torch.device(src).index if torch.device(src).index is not None else 0)
        self.dst = torch.device("cuda", torch.device(dst).index if torch.device(dst).index is not None else 0)
        enable_peer_access(self.src.index, self.dst.index)
        self.out_dtype = out_dtype
        self.chunks = [(l0, min(L, l0 + chunk_layers)) for l0 in range(0, L, chunk_layers)]
        self.enc, self.dec, self.tx_src, self.tx_dst = [], [], [], []
        plans: dict[int, tuple[KVCodec, KVCodec]] = {}
        for l0, l1 in self.chunks:
            n = l1 - l0
            if n not in plans:
                plans[n] = (
                    KVCodec(strategy_id, (n, H, T, C), in_dtype=in_dtype, block_symbols=block_symbols, device=self.src),
                    KVCodec(strategy_id, (n, H, T, C), out_dtype=out_dtype, block_symbols=block_symbols,
                            device=self.dst),
                )
            e, d = plans[n]
            self.enc.append(e)
            self.dec.append(d)
            with torch.cuda.device(self.src):
                self.tx_src.append(e.alloc_blob())
            with torch.cuda.device(self.dst):
                self.tx_dst.append(d.alloc_blob())
        with torch.cuda.device(self.src):
            self.s_enc = torch.cuda.Stream(self.src)
            self.s_copy = torch.cuda.Stream(self.src)
            self.ev_enc = [torch.cuda.Event() for _ in self.chunks]
            self.ev_copy = [torch.cuda.Event() for _ in self.chunks]
        with torch.cuda.device(self.dst):
            self.s_dec = torch.cuda.Stream(self.dst)
            self.ev_dec = [torch.cuda.Event() for _ in self.chunks]
        # a device "length" larger than any buffer: fixed-size copies go
        # through the same kernel, ordered on the copy stream
        self._big = torch.full((1,), 1 << 62, dtype=torch.int64, device=self.src)
        torch.cuda.synchronize(self.src)

    def _copy(self, dst: torch.Tensor, src: torch.Tensor, len_ptr: int, max_bytes: int) -> None:
        if max_bytes > 0:
            N.check(N.lib().kvc_copy_device_length(dst.data_ptr(), src.data_ptr(), len_ptr, int(max_bytes),
                                                   _stream_handle(self.s_copy)))

    def run(self, kv: torch.Tensor, out: torch.Tensor | None = None, head_classes=None) -> torch.Tensor:
        """Start the pipelined transfer; returns the dst tensor (ordered on
        the dst decode stream, which the caller's current dst stream joins)."""
        if tuple(kv.shape) != self.shape or kv.device != self.src:
            raise ValueError("kv must be the transfer's shape on the source device")
        if out is None:
            out = torch.empty(self.shape, dtype=self.out_dtype, device=self.dst)
        cur_src = torch.cuda.current_stream(self.src)
        cur_dst = torch.cuda.current_stream(self.dst)
        # work already queued by the caller: kv's producer on the source, and
        # any pending use of `out` (a reused KV slot) on the destination
        self.s_enc.wait_stream(cur_src)
        self.s_copy.wait_stream(cur_dst)
        self.s_dec.wait_stream(cur_dst)
        kv.record_stream(self.s_enc)
        out.record_stream(self.s_dec)
        for i, (l0, l1) in enumerate(self.chunks):
            cls = None if head_classes is None else head_classes[l0:l1]
            src_blob, dst_blob = self.tx_src[i], self.tx_dst[i]
            with torch.cuda.device(self.src):
                # the previous run's copy of this chunk has read its wire buffer
                self.s_enc.wait_event(self.ev_copy[i])
                self.enc[i].encode(kv[l0:l1], head_classes=cls, out=src_blob, stream=self.s_enc)
                self.ev_enc[i].record(self.s_enc)
                self.s_copy.wait_event(self.ev_enc[i])
                self.s_copy.wait_event(self.ev_dec[i])  # ... and its decode is done with the dst buffer
                big = self._big.data_ptr()
                self._copy(dst_blob.metadata, src_blob.metadata, big, src_blob.metadata.numel())
                if src_blob.offsets is not None:
                    self._copy(dst_blob.offsets, src_blob.offsets, big, 8 * (src_blob.nblocks + 1))
                    # payload length = offsets[nblocks], read on the device
                    self._copy(dst_blob.payload, src_blob.payload, src_blob.offsets[src_blob.nblocks:].data_ptr(),
                               src_blob.payload.numel())
                else:  # codec none: static length
                    self._copy(dst_blob.payload, src_blob.payload, big, src_blob.payload_nbytes())
                self.ev_copy[i].record(self.s_copy)
            dst_blob.nblocks = src_blob.nblocks
            dst_blob._nbytes = src_blob._nbytes
            with torch.cuda.device(self.dst):
                self.s_dec.wait_event(self.ev_copy[i])
                self.dec[i].decode(dst_blob, out=out[l0:l1], stream=self.s_dec,
                                   device_length=dst_blob.offsets is not None)
                self.ev_dec[i].record(self.s_dec)
        cur_dst.wait_stream(self.s_dec)
        # the caller may free or overwrite kv once its own stream moves on
        cur_src.wait_stream(self.s_enc)
        cur_src.wait_stream(self.s_copy)
        return out

    def check(self) -> None:
        """Synchronise both ends and raise for device-side errors."""
        for codec in {id(c): c for c in self.enc}.values():
            codec.check(stream=self.s_enc)
        for codec in {id(c): c for c in self.dec}.values():
            codec.check(stream=self.s_dec, decoding=True)

    def wire_bytes(self) -> int:
        """Bytes that crossed the link in the last run (syncs)."""
        return sum(b.payload_nbytes() + b.metadata.numel() + (0 if b.offsets is None else 8 * (b.nblocks + 1))
                   for b in self.tx_src)
