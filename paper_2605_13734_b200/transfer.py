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
encode.  `run_paged` is the KV-connector form: source and destination are
paged caches (vLLM layout), read by kvc_encode_paged and written by
kvc_decode_paged, so no gather or scatter pass touches the KV.  Each chunk is an independent blob of its (l, H, T, C) slab — the same
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
        torch.cuda.synchronize(self.src)

    def _copy(self, dst: torch.Tensor, src: torch.Tensor, len_ptr: int, max_bytes: int) -> None:
        """Length known on the device only (entropy / rle payloads): the
        copy kernel reads it there, so nothing syncs to the host."""
        if max_bytes > 0:
            N.check(N.lib().kvc_copy_device_length(dst.data_ptr(), src.data_ptr(), len_ptr, int(max_bytes),
                                                   _stream_handle(self.s_copy)))

    def _dma(self, dst: torch.Tensor, src: torch.Tensor, nbytes: int) -> None:
        """Length known on the host: a copy-engine peer copy, which leaves the
        source GPU's SMs to the encoder of the next chunk."""
        if nbytes > 0:
            with torch.cuda.stream(self.s_copy):
                dst[:nbytes].copy_(src[:nbytes], non_blocking=True)

    def run(self, kv: torch.Tensor, out: torch.Tensor | None = None, head_classes=None) -> torch.Tensor:
        """Start the pipelined transfer; returns the dst tensor (ordered on
        the dst decode stream, which the caller's current dst stream joins)."""
        if tuple(kv.shape) != self.shape or kv.device != self.src:
            raise ValueError("kv must be the transfer's shape on the source device")
        if out is None:
            out = torch.empty(self.shape, dtype=self.out_dtype, device=self.dst)

        def enc(i, l0, l1, cls, blob):
            self.enc[i].encode(kv[l0:l1], head_classes=cls, out=blob, stream=self.s_enc)

        def dec(i, l0, l1, blob):
            self.dec[i].decode(blob, out=out[l0:l1], stream=self.s_dec, device_length=blob.offsets is not None)

        self._pipeline(kv, out, enc, dec, head_classes)
        return out

    def run_paged(self, src_pages: torch.Tensor, src_table: torch.Tensor, dst_pages: torch.Tensor,
                  dst_table: torch.Tensor, page_tokens: int, src_layer_stride: int, dst_layer_stride: int,
                  head_classes=None) -> torch.Tensor:
        """The KV-connector form: compress straight from the source GPU's
        paged cache (kvc_encode_paged) and decompress straight into the
        destination's (kvc_decode_paged), both vLLM layout [pages,
        page_tokens, H, C] per layer with their own block tables; layer
        chunk [l0, l1) of a pool starts l0 * layer_stride elements in."""
        if src_pages.device != self.src or dst_pages.device != self.dst:
            raise ValueError("page pools must live on the transfer's source / destination devices")
        if not (src_pages.is_contiguous() and dst_pages.is_contiguous()):
            raise ValueError("page pools must be contiguous")
        L = self.shape[0]
        if src_pages.numel() < L * src_layer_stride or dst_pages.numel() < L * dst_layer_stride:
            raise ValueError("page pool smaller than layers x layer_stride")
        sflat, dflat = src_pages.view(-1), dst_pages.view(-1)
        st = src_table.to(device=self.src, dtype=torch.int32).contiguous()
        dt = dst_table.to(device=self.dst, dtype=torch.int32).contiguous()

        def enc(i, l0, l1, cls, blob):
            self.enc[i].encode_paged(sflat[l0 * src_layer_stride:], st, page_tokens, src_layer_stride,
                                     head_classes=cls, out=blob, stream=self.s_enc)

        def dec(i, l0, l1, blob):
            self.dec[i].decode_paged(blob, dflat[l0 * dst_layer_stride:], dt, page_tokens, dst_layer_stride,
                                     stream=self.s_dec, device_length=blob.offsets is not None)

        self._pipeline(src_pages, dst_pages, enc, dec, head_classes, keep=(st, dt))
        return dst_pages

    def _pipeline(self, src_t: torch.Tensor, dst_t: torch.Tensor, enc, dec, head_classes, keep=()) -> None:
        cur_src = torch.cuda.current_stream(self.src)
        cur_dst = torch.cuda.current_stream(self.dst)
        # work already queued by the caller: the source's producer, and any
        # pending use of the destination (a reused KV slot or page)
        self.s_enc.wait_stream(cur_src)
        self.s_copy.wait_stream(cur_dst)
        self.s_dec.wait_stream(cur_dst)
        src_t.record_stream(self.s_enc)
        dst_t.record_stream(self.s_dec)
        for t in keep:  # block tables built here: alive until their kernels ran
            t.record_stream(self.s_enc if t.device == self.src else self.s_dec)
        for i, (l0, l1) in enumerate(self.chunks):
            cls = None if head_classes is None else head_classes[l0:l1]
            src_blob, dst_blob = self.tx_src[i], self.tx_dst[i]
            with torch.cuda.device(self.src):
                # the previous run's copy of this chunk has read its wire buffer
                self.s_enc.wait_event(self.ev_copy[i])
                enc(i, l0, l1, cls, src_blob)
                self.ev_enc[i].record(self.s_enc)
                self.s_copy.wait_event(self.ev_enc[i])
                self.s_copy.wait_event(self.ev_dec[i])  # ... and its decode is done with the dst buffer
                self._dma(dst_blob.metadata, src_blob.metadata, src_blob.metadata.numel())
                if src_blob.offsets is not None:
                    self._dma(dst_blob.offsets, src_blob.offsets, src_blob.nblocks + 1)
                    # payload length = offsets[nblocks], read on the device
                    self._copy(dst_blob.payload, src_blob.payload, src_blob.offsets[src_blob.nblocks:].data_ptr(),
                               src_blob.payload.numel())
                else:  # codec none: static length
                    self._dma(dst_blob.payload, src_blob.payload, src_blob.payload_nbytes())
                self.ev_copy[i].record(self.s_copy)
            dst_blob.nblocks = src_blob.nblocks
            dst_blob._nbytes = src_blob._nbytes
            with torch.cuda.device(self.dst):
                self.s_dec.wait_event(self.ev_copy[i])
                dec(i, l0, l1, dst_blob)
                self.ev_dec[i].record(self.s_dec)
        cur_dst.wait_stream(self.s_dec)
        # the caller may free or overwrite the source once its own stream moves on
        cur_src.wait_stream(self.s_enc)
        cur_src.wait_stream(self.s_copy)

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
