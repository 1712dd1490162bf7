"""ShardedCodec with the real CUDA codec (ranks simulated one after another on
one GPU; the multi-process NCCL run is tools/run_sharded_nccl.py): layer
shards of a codec-none profile concatenate to the whole-tensor payload, and
every shard -- by layer or by KV head, any codec, mixed labels sliced from
the global classify_heads -- decodes to the whole-tensor decode's slice."""

import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

SIDS = [
    "t=hadamard;q=uniform,b=4,g=32;c=none",
    "t=identity;q=uniform,b=2,g=32;c=entropy",
    "t=identity;q=uchan,b=2,g=32;c=entropy",
    "t=hadamard;q=mixed,hi=8,lo=2,g=32,rho=0.25;c=rle",
]


@pytest.mark.parametrize("sid", SIDS)
@pytest.mark.parametrize("by,world", [("layer", 2), ("layer", 3), ("head", 2), ("head", 8)])
def test_shards_decode_to_the_whole_tensor(sid, by, world):
    from paper_2605_13734_b200 import KVCodec
    from paper_2605_13734_b200.distributed import ShardedCodec
    from paper_2605_13734_b200.pipeline import classify_heads

    shape = (5, 8, 2048, 128)
    v, imp = oracle.generate_kv(*shape, seed=3)
    kv = torch.from_numpy(v).to(torch.bfloat16).cuda()
    cls = classify_heads(imp, 0.25) if "mixed" in sid else None
    whole = KVCodec(sid, shape)
    wblob = whole.encode(kv, head_classes=cls)
    want = whole.decode(wblob)
    whole.check(decoding=True)
    pays = []
    for r in range(world):
        sc = ShardedCodec(sid, shape, rank=r, world=world, by=by)
        blob = sc.encode(sc.local_slice(kv), global_classes=cls)
        got = sc.decode(blob)
        sc.codec.check(decoding=True)
        assert torch.equal(got, want[sc.l0:sc.l1, sc.h0:sc.h1]), (sid, by, world, r)
        pays.append(blob.payload_bytes())
    if by == "layer" and sid.endswith("c=none") and "mixed" not in sid:
        assert b"".join(pays) == wblob.payload_bytes()
