"""Block-framed wire container: self-describing
header, per-block CRC-32 computed on the GPU (checked against zlib.crc32),
corruption reported by block index before decode."""

import struct
import zlib

import numpy as np
import pytest

import oracle


def test_rejects_foreign_and_truncated_bytes():
    from paper_2605_13734_b200 import _native as N
    from paper_2605_13734_b200 import wire

    with pytest.raises(N.CodecError):
        wire.unpack(b"not a container at all, clearly" * 4)
    head = wire._FIXED.pack(wire.MAGIC, wire.VERSION, 0, 0, 1, 1, 8, 64, 2048, 0, 0, 0, 3) + b"t=x"
    with pytest.raises(N.CodecError):  # header_len field left at 0
        wire.unpack(head + struct.pack("<I", zlib.crc32(head)))
    head = head[:8] + struct.pack("<I", len(head) + 4) + head[12:]
    with pytest.raises(N.CodecError):  # checksum of a different header
        wire.unpack(head + struct.pack("<I", zlib.crc32(head) ^ 1))


@pytest.mark.gpu
@pytest.mark.parametrize("sid", ["t=identity;q=uniform,b=2,g=32;c=entropy", "t=hadamard;q=uniform,b=4,g=32;c=none",
                                 "t=identity;q=uchan,b=2,g=32;c=entropy", "t=delta;q=uniform,b=4,g=32;c=rle",
                                 "t=affine;q=uniform,b=8,g=32;c=entropy"])
def test_roundtrip_and_block_crc(sid):
    torch = pytest.importorskip("torch")
    from paper_2605_13734_b200 import KVCodec, wire

    shape = (2, 2, 1024, 128)
    v, _ = oracle.generate_kv(*shape, seed=11)
    kv = torch.from_numpy(v).to(torch.bfloat16).cuda()
    codec = KVCodec(sid, shape, block_symbols=1024)
    blob = codec.encode(kv)
    codec.check()
    ref_out = codec.decode(blob)
    data = wire.pack(codec, blob)
    # the GPU CRC equals zlib's on every block
    pay = blob.payload_bytes()
    if blob.nblocks:
        offs = blob.offsets_array()
        want = [zlib.crc32(pay[offs[b]:offs[b + 1]]) for b in range(blob.nblocks)]
        got = wire.block_crc32(blob.payload, blob.offsets, blob.nblocks).cpu().numpy().view(np.uint32)
        assert list(got) == want
    codec2, blob2 = wire.unpack(data)
    assert codec2.strategy_id == codec.strategy_id and blob2.shape == shape
    out = codec2.decode(blob2)
    codec2.check(decoding=True)
    assert torch.equal(out, ref_out)


@pytest.mark.gpu
def test_corruption_is_reported_by_block():
    torch = pytest.importorskip("torch")
    from paper_2605_13734_b200 import KVCodec, _native, wire

    shape = (1, 2, 1024, 128)
    v, _ = oracle.generate_kv(*shape, seed=12)
    codec = KVCodec("t=identity;q=uniform,b=2,g=32;c=entropy", shape, block_symbols=1024)
    blob = codec.encode(torch.from_numpy(v).to(torch.bfloat16).cuda())
    codec.check()
    data = bytearray(wire.pack(codec, blob))
    offs = blob.offsets_array()
    victim = 100
    pos = len(data) - blob.payload_nbytes() + int(offs[victim]) + 7
    data[pos] ^= 0x40
    with pytest.raises(_native.CodecError, match=f"first at block {victim}"):
        wire.unpack(bytes(data))
    data[pos] ^= 0x40
    data[60] ^= 1  # inside the header
    with pytest.raises(_native.CodecError):
        wire.unpack(bytes(data))
