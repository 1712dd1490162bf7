"""Block-framed wire / disk container for compressed KV.

The reference's blob (codecs.py:41-59) is not self-describing: decoding needs
the strategy id and shape from elsewhere (compress.py:143-166), and nothing
detects corruption short of a CodecError from the range decoder.  This
container carries everything decode needs plus a CRC-32 per codec block
(computed and verified on the GPU, `kvc_block_crc32`), so a damaged block is
reported by index before any decode runs.

Layout (little-endian):

    magic "KVW1" | u16 version | u16 flags | u32 header_len
    u64 L, H, T, C | u64 block_symbols | u64 nblocks
    u64 metadata_len | u64 payload_len | u16 id_len | id (utf-8)
    u32 crc32(header bytes before this field)
    metadata bytes                              (codecs.py:348-352 + extensions)
    u64 block_offsets[nblocks + 1]              (entropy / rle; absent for none)
    u32 crc[max(nblocks, 1)]                    (per block; one for the whole payload of codec none)
    u32 crc32(metadata)
    payload bytes

`pack` reads the blob back to the host once; `unpack` uploads it, verifies
every CRC on the device and returns a (KVCodec, DeviceBlob) pair ready for
`KVCodec.decode`.
"""

from __future__ import annotations

import struct
import zlib

import numpy as np
import torch

from paper_2605_13734_b200 import _native as N
from paper_2605_13734_b200.codec import DeviceBlob, KVCodec

__all__ = ["pack", "unpack", "block_crc32"]

MAGIC = b"KVW1"
VERSION = 1
_FIXED = struct.Struct("<4sHHI4QQQQQH")


def block_crc32(payload: torch.Tensor, offsets: torch.Tensor, nblocks: int,
                stream: torch.cuda.Stream | None = None) -> torch.Tensor:
    """CRC-32 of each block [offsets[b], offsets[b+1]) of a device payload."""
    out = torch.empty(max(nblocks, 1), dtype=torch.int32, device=payload.device)
    if nblocks == 0:
        return out[:0]
    s = stream if stream is not None else torch.cuda.current_stream(payload.device)
    N.check(N.lib().kvc_block_crc32(payload.data_ptr(), offsets.data_ptr(), int(nblocks), out.data_ptr(),
                                    s.cuda_stream or None))
    return out


def _crc_table(blob: DeviceBlob) -> tuple[np.ndarray, np.ndarray | None]:
    nb = blob.nblocks
    if nb == 0:  # codec none: one block over the whole payload
        offs = torch.tensor([0, blob.payload_nbytes()], dtype=torch.int64, device=blob.payload.device)
        return block_crc32(blob.payload, offs, 1).cpu().numpy().view(np.uint32), None
    crc = block_crc32(blob.payload, blob.offsets, nb).cpu().numpy().view(np.uint32)
    return crc, blob.offsets_array()


def pack(codec: KVCodec, blob: DeviceBlob) -> bytes:
    """Serialize an encoded blob (device) into a self-describing byte string."""
    crc, offsets = _crc_table(blob)
    meta = blob.metadata_bytes()
    payload = blob.payload_bytes()
    sid = blob.strategy_id.encode()
    L, H, T, C = blob.shape
    head = _FIXED.pack(MAGIC, VERSION, 0, 0, L, H, T, C, codec.block_symbols, blob.nblocks, len(meta), len(payload),
                       len(sid)) + sid
    head = head[:8] + struct.pack("<I", len(head) + 4) + head[12:]
    parts = [head, struct.pack("<I", zlib.crc32(head)), meta]
    if offsets is not None:
        parts.append(offsets.astype("<u8").tobytes())
    parts.append(crc.astype("<u4").tobytes())
    parts.append(struct.pack("<I", zlib.crc32(meta)))
    parts.append(payload)
    return b"".join(parts)


def unpack(data: bytes, device=None, out_dtype: torch.dtype = torch.bfloat16) -> tuple[KVCodec, DeviceBlob]:
    """Parse and verify a container; CodecError on any mismatch (header,
    metadata or a block's CRC, reported by block index)."""
    mv = memoryview(data)
    if len(data) < _FIXED.size + 4 or bytes(mv[:4]) != MAGIC:
        raise N.CodecError("not a KVW1 container")
    (_, version, _flags, header_len, L, H, T, C, block_symbols, nblocks, meta_len, payload_len,
     id_len) = _FIXED.unpack_from(mv, 0)
    if version != VERSION:
        raise N.CodecError(f"unsupported container version {version}")
    hend = _FIXED.size + id_len
    if header_len != hend + 4 or len(data) < hend + 4:
        raise N.CodecError("truncated container header")
    if zlib.crc32(mv[:hend]) != struct.unpack_from("<I", mv, hend)[0]:
        raise N.CodecError("container header checksum mismatch")
    sid = bytes(mv[_FIXED.size:hend]).decode()
    pos = hend + 4
    meta = bytes(mv[pos:pos + meta_len])
    pos += meta_len
    offsets = None
    if nblocks:
        offsets = np.frombuffer(mv[pos:pos + 8 * (nblocks + 1)], dtype="<u8").astype(np.int64)
        pos += 8 * (nblocks + 1)
    ncrc = max(nblocks, 1)
    crc = np.frombuffer(mv[pos:pos + 4 * ncrc], dtype="<u4").copy()
    pos += 4 * ncrc
    meta_crc = struct.unpack_from("<I", mv, pos)[0]
    pos += 4
    if len(data) != pos + payload_len:
        raise N.CodecError(f"container has {len(data) - pos} payload bytes, header says {payload_len}")
    if zlib.crc32(meta) != meta_crc:
        raise N.CodecError("metadata checksum mismatch")

    codec = KVCodec(sid, (L, H, T, C), out_dtype=out_dtype, block_symbols=int(block_symbols), device=device)
    if len(meta) != codec.metadata_bytes:
        raise N.CodecError(f"metadata is {len(meta)} bytes, expected {codec.metadata_bytes}")
    dev = codec.device
    payload = torch.empty(max(codec.payload_capacity, payload_len, 1), dtype=torch.uint8, device=dev)
    if payload_len:
        payload[:payload_len].copy_(torch.frombuffer(bytearray(mv[pos:pos + payload_len]), dtype=torch.uint8))
    meta_t = torch.frombuffer(bytearray(meta), dtype=torch.uint8).to(dev) if meta else torch.empty(0, dtype=torch.uint8,
                                                                                                     device=dev)
    offs_t = None
    if nblocks:
        if offsets[0] != 0 or offsets[-1] != payload_len or np.any(np.diff(offsets) < 0):
            raise N.CodecError("malformed block table")
        offs_t = torch.zeros(codec.max_blocks + 1, dtype=torch.int64, device=dev)
        offs_t[: nblocks + 1] = torch.from_numpy(offsets).to(dev)
        got = block_crc32(payload, offs_t, nblocks).cpu().numpy().view(np.uint32)
    else:
        got = block_crc32(payload, torch.tensor([0, payload_len], dtype=torch.int64, device=dev), 1).cpu().numpy().view(
            np.uint32)
    bad = np.nonzero(got != crc)[0]
    if bad.size:
        raise N.CodecError(f"{bad.size} block(s) fail their CRC-32, first at block {int(bad[0])}")
    blob = DeviceBlob(payload, meta_t, offs_t, codec.strategy_id, (L, H, T, C), None, int(nblocks), payload_len)
    return codec, blob
