"""Corrupted blobs never fault the device.

The reference decoder raises CodecError on malformed streams
(codecs.py:283-288, :155-174); the GPU decoders must do the same from any
payload bytes and any block-offset table, given the true payload length
(the C-ABI's trust boundary: `payload_bytes` bounds every read, kvc.h).
Each case decodes a randomly corrupted copy, accepts success or CodecError,
and then proves the context is still healthy with a clean round trip.
"""

import os
import zlib

import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

IDS = [
    ("t=identity;q=uniform,b=2,g=32;c=entropy", (2, 4, 256, 128)),  # fused per-token coder
    ("t=identity;q=uchan,b=2,g=32;c=entropy", (2, 2, 2048, 128)),  # fused per-channel coder
    ("t=hadamard;q=mixed,hi=8,lo=2,g=32,rho=0.25;c=entropy", (2, 4, 128, 128)),  # rc_large + rc_small
    ("t=delta;q=uniform,b=4,g=64;c=entropy", (1, 3, 200, 64)),  # generic + rc_small
    ("t=identity;q=uniform,b=4,g=32;c=rle", (2, 4, 128, 128)),
    ("t=hadamard;q=mixed,hi=4,lo=2,g=32,rho=0.25;c=rle", (2, 4, 96, 128)),
    ("t=affine;q=uniform,b=8,g=32;c=entropy", (2, 2, 256, 128)),
    ("t=hadamard;q=mixed,hi=8,lo=2,g=32,rho=0.25;c=none", (2, 4, 128, 128)),  # fast128, payload read in place
    ("t=delta;q=uniform,b=4,g=32;c=none", (1, 2, 4096, 128)),  # chunked delta decode
    ("t=identity;q=uchan,b=2,g=32;c=none", (1, 2, 256, 128)),
    ("t=identity;q=uniform,b=3,g=4;c=none", (1, 2, 40, 20)),  # generic
]


def _blob(sid, shape, seed):
    from paper_2605_13734_b200 import KVCodec

    v, imp = oracle.generate_kv(*shape, seed=seed)
    s = oracle.parse_id(sid)
    cls = oracle.classify_heads(imp, s.rho) if s.quant == "mixed" else None
    kv = torch.from_numpy(v).to(torch.bfloat16).cuda()
    codec = KVCodec(sid, shape, out_dtype=torch.float32)
    blob = codec.encode(kv, head_classes=cls)
    codec.check()
    return codec, blob, kv


def _clone(blob):
    from dataclasses import replace

    b = replace(blob, payload=blob.payload.clone(), metadata=blob.metadata.clone(),
                offsets=None if blob.offsets is None else blob.offsets.clone())
    b._nbytes = blob.payload_nbytes()
    return b


def _try_decode(codec, blob):
    from paper_2605_13734_b200 import _native

    try:
        codec.decode(blob)
        codec.check(decoding=True)
    except (_native.CodecError, ValueError):
        pass
    torch.cuda.synchronize()  # a device fault would surface here


@pytest.mark.parametrize("sid,shape", IDS)
def test_corrupted_blobs_do_not_fault(sid, shape):
    codec, blob, kv = _blob(sid, shape, seed=11)
    ref = codec.decode(blob).clone()
    n = blob.payload_nbytes()
    rng = np.random.default_rng(zlib.crc32(sid.encode()))
    for trial in range(int(os.environ.get("KVC_CORRUPT_TRIALS", "40"))):
        b = _clone(blob)
        kind = trial % 4
        if kind == 0:  # random byte overwrites
            k = int(rng.integers(1, 16))
            pos = torch.from_numpy(rng.integers(0, n, size=k)).cuda()
            b.payload[pos] = torch.from_numpy(rng.integers(0, 256, size=k).astype(np.uint8)).cuda()
        elif kind == 1:  # a zeroed or 0xff-filled span
            a = int(rng.integers(0, n))
            b.payload[a:min(n, a + int(rng.integers(1, 512)))] = int(rng.choice([0, 255]))
        elif kind == 2 and b.offsets is not None:  # offset table: random values, some out of range
            k = int(rng.integers(1, 4))
            idx = torch.from_numpy(rng.integers(0, b.nblocks + 1, size=k)).cuda()
            vals = rng.choice([0, n, n + 1, -1, 1 << 40, int(rng.integers(0, n + 1))], size=k)
            b.offsets[idx] = torch.from_numpy(np.asarray(vals, dtype=np.int64)).cuda()
        else:  # truncated payload length
            b._nbytes = int(rng.integers(0, n))
        _try_decode(codec, b)
    # the context is healthy and the pristine blob still decodes identically
    assert torch.equal(codec.decode(blob), ref)
    codec.check(decoding=True)
