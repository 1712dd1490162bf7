"""Host-memory round trip, pipelined: the end-to-end path a serving engine
takes when the compressed KV leaves the GPU (to a NIC, another host, disk).

    pinned host KV --H2D--> encode --D2H--> host wire --H2D--> decode --> HBM

Per layer chunk, on five streams chained by events, so copy engines, PCIe
and SMs work concurrently:

    s_in   H2D of the chunk's bf16 KV (copy engine)
    s_enc  KVCodec.encode
    s_out  wire -> pinned host memory; the payload's length stays in device
           memory and the copy kernel writes straight into the mapped pinned
           buffer (kvc_copy_device_length), so nothing waits on the host
    s_back host wire -> HBM, same kernel reading the mapped pinned buffer and
           the length from the host copy of the block table
    s_dec  KVCodec.decode + the squared-error scalar (kvc_sq_error)

Chunks are whole layers; with 2048-symbol blocks aligned to chunk boundaries
(H*T*C a multiple of the block for per-token groups, T a multiple of it for
per-channel groups) the chunk payloads concatenate to the whole-tensor
payload byte for byte.
"""

from __future__ import annotations

import torch

from paper_2605_13734_b200 import _native as N
from paper_2605_13734_b200.codec import KVCodec, _stream_handle

__all__ = ["HostRoundTrip"]


class HostRoundTrip:
    def __init__(self, strategy_id: str, shape, chunk_layers: int = 4, block_symbols: int = 2048, device=None,
                 paged=None, wire_via_host: bool = True) -> None:
        """paged = (block_table int32 cuda, page_tokens, layer_stride): decode
        into a paged cache (kvc_decode_paged; one table shared by every
        layer, `out` the page pool of all layers) instead of a contiguous
        (L, H, T, C) tensor.  wire_via_host=False: the blob stays in HBM
        between encode and decode, as in the reference's compress()
        (compress.py:122-130) -- only the KV crosses PCIe."""
        L, H, T, C = (int(v) for v in shape)
        self.shape = (L, H, T, C)
        self.paged = paged
        self.wire_via_host = wire_via_host
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.chunks = [(l0, min(L, l0 + chunk_layers)) for l0 in range(0, L, chunk_layers)]
        enc_plans: dict[int, KVCodec] = {}
        dec_plans: dict[int, KVCodec] = {}
        self.enc, self.dec, self.blob, self.rx = [], [], [], []
        self.h_pay, self.h_meta, self.h_off = [], [], []
        with torch.cuda.device(self.device):
            for l0, l1 in self.chunks:
                n = l1 - l0
                if n not in enc_plans:  # separate plans (workspaces) for the two ends
                    enc_plans[n] = KVCodec(strategy_id, (n, H, T, C), block_symbols=block_symbols, device=self.device)
                    dec_plans[n] = KVCodec(strategy_id, (n, H, T, C), block_symbols=block_symbols, device=self.device)
                e, d = enc_plans[n], dec_plans[n]
                self.enc.append(e)
                self.dec.append(d)
                self.blob.append(e.alloc_blob())
                self.rx.append(d.alloc_blob() if wire_via_host else self.blob[-1])
                if not wire_via_host:
                    continue
                # the full payload capacity: the device-length copy can never
                # truncate a chunk (a shorter buffer would drop bytes silently)
                self.h_pay.append(torch.empty(max(e.payload_capacity, 16), dtype=torch.uint8, pin_memory=True))
                self.h_meta.append(torch.empty(max(e.metadata_bytes, 1), dtype=torch.uint8, pin_memory=True))
                self.h_off.append(None if e.codec_kind == "none" else
                                  torch.zeros(e.max_blocks + 1, dtype=torch.int64, pin_memory=True))
            mk = lambda: torch.cuda.Stream(self.device)  # noqa: E731
            self.s_in, self.s_enc, self.s_out, self.s_back, self.s_dec = mk(), mk(), mk(), mk(), mk()
            ev = lambda: [torch.cuda.Event() for _ in self.chunks]  # noqa: E731
            self.e_in, self.e_enc, self.e_out, self.e_back, self.e_dec = ev(), ev(), ev(), ev(), ev()
            torch.cuda.synchronize(self.device)

    def _copy(self, dst_ptr: int, src_ptr: int, len_ptr: int, max_bytes: int, stream) -> None:
        if max_bytes > 0:
            N.check(N.lib().kvc_copy_device_length(dst_ptr, src_ptr, len_ptr, int(max_bytes), _stream_handle(stream)))

    def run(self, host_kv: torch.Tensor, dev_in: torch.Tensor, out: torch.Tensor,
            err_sum: torch.Tensor | None = None) -> torch.Tensor | None:
        """Enqueue one round trip of `host_kv` (pinned, bf16) through `dev_in`
        into `out`; adds the squared reconstruction error to `err_sum`
        (device float64 scalar) if given.  Ordered before the device's
        current stream afterwards."""
        cur = torch.cuda.current_stream(self.device)
        with torch.cuda.device(self.device):
            for s in (self.s_in, self.s_enc, self.s_out, self.s_back, self.s_dec):
                s.wait_stream(cur)
            for i, (l0, l1) in enumerate(self.chunks):
                blob, rx = self.blob[i], self.rx[i]
                enc, dec = self.enc[i], self.dec[i]
                # H2D of the chunk (after the previous run's encode and error pass read dev_in)
                self.s_in.wait_event(self.e_dec[i])
                with torch.cuda.stream(self.s_in):
                    dev_in[l0:l1].copy_(host_kv[l0:l1], non_blocking=True)
                self.e_in[i].record(self.s_in)
                # encode (after the previous run's D2H -- or decode -- read this chunk's blob)
                self.s_enc.wait_event(self.e_in[i])
                self.s_enc.wait_event(self.e_out[i] if self.wire_via_host else self.e_dec[i])
                enc.encode(dev_in[l0:l1], out=blob, stream=self.s_enc)
                self.e_enc[i].record(self.s_enc)
                if not self.wire_via_host:
                    self.s_dec.wait_event(self.e_enc[i])
                    self._decode(i, rx, blob, dec, out, dev_in, err_sum, device_length=blob.offsets is not None)
                    continue
                # wire -> pinned host (after the previous run's H2D of the wire)
                self.s_out.wait_event(self.e_enc[i])
                self.s_out.wait_event(self.e_back[i])
                hp, hm, ho = self.h_pay[i], self.h_meta[i], self.h_off[i]
                with torch.cuda.stream(self.s_out):
                    if blob.metadata.numel():
                        hm[: blob.metadata.numel()].copy_(blob.metadata, non_blocking=True)
                    if ho is not None:
                        ho[: blob.nblocks + 1].copy_(blob.offsets[: blob.nblocks + 1], non_blocking=True)
                if ho is not None:
                    self._copy(hp.data_ptr(), blob.payload.data_ptr(), blob.offsets[blob.nblocks:].data_ptr(),
                               hp.numel(), self.s_out)
                else:  # static length: the copy engine, no SMs taken from the codec
                    n = blob.payload_nbytes()
                    with torch.cuda.stream(self.s_out):
                        hp[:n].copy_(blob.payload[:n], non_blocking=True)
                self.e_out[i].record(self.s_out)
                # host wire -> HBM (after the previous run's decode read rx)
                self.s_back.wait_event(self.e_out[i])
                self.s_back.wait_event(self.e_dec[i])
                with torch.cuda.stream(self.s_back):
                    if blob.metadata.numel():
                        rx.metadata.copy_(hm[: blob.metadata.numel()], non_blocking=True)
                    if ho is not None:
                        rx.offsets[: blob.nblocks + 1].copy_(ho[: blob.nblocks + 1], non_blocking=True)
                if ho is not None:
                    # the length comes from the pinned host block table (mapped)
                    self._copy(rx.payload.data_ptr(), hp.data_ptr(), ho.data_ptr() + 8 * blob.nblocks, hp.numel(),
                               self.s_back)
                else:
                    n = blob.payload_nbytes()
                    with torch.cuda.stream(self.s_back):
                        rx.payload[:n].copy_(hp[:n], non_blocking=True)
                self.e_back[i].record(self.s_back)
                rx.nblocks, rx._nbytes = blob.nblocks, blob._nbytes
                self.s_dec.wait_event(self.e_back[i])
                self._decode(i, rx, blob, dec, out, dev_in, err_sum, device_length=ho is not None)
            cur.wait_stream(self.s_dec)
        return err_sum

    def _decode(self, i, rx, blob, dec, out, dev_in, err_sum, device_length: bool) -> None:
        """Decode chunk i on s_dec and add the step's scalar result: the squared
        reconstruction error (contiguous) or the compressed bytes (paged)."""
        l0, l1 = self.chunks[i]
        if self.paged is not None:
            table, page_tokens, stride = self.paged
            dec.decode_paged(rx, out[l0 * stride:l1 * stride], table, page_tokens, stride, stream=self.s_dec,
                             device_length=device_length)
            if err_sum is not None and rx.offsets is not None:
                with torch.cuda.stream(self.s_dec):
                    err_sum.add_(rx.offsets[rx.nblocks].to(torch.float64))
        else:
            dec.decode(rx, out=out[l0:l1], stream=self.s_dec, device_length=device_length)
            if err_sum is not None:
                n = (l1 - l0) * self.shape[1] * self.shape[2] * self.shape[3]
                dt = N.DTYPE_BF16 if out.dtype == torch.bfloat16 else N.DTYPE_F32
                N.check(N.lib().kvc_sq_error(out[l0:l1].data_ptr(), dev_in[l0:l1].data_ptr(), n, dt,
                                             err_sum.data_ptr(), _stream_handle(self.s_dec)))
        self.e_dec[i].record(self.s_dec)

    def check(self) -> None:
        for c in {id(c): c for c in self.enc}.values():
            c.check(stream=self.s_enc)
        for c in {id(c): c for c in self.dec}.values():
            c.check(stream=self.s_dec, decoding=True)

    def wire_bytes(self) -> int:
        """Compressed bytes of the last run (payload + metadata + block table)."""
        return sum(b.payload_nbytes() + b.metadata.numel() + (0 if b.offsets is None else 8 * (b.nblocks + 1))
                   for b in self.blob)
