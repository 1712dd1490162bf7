"""kvc_encode_paged: encode straight from a paged KV cache.

The pages hold the same KV as a contiguous (L,H,T,C) tensor, scattered over
a pool in the vLLM layout [pages, page_tokens, H, C] per layer (the layout
kvc_decode_paged writes).  The blob must be byte-identical to kvc_encode of
the contiguous tensor: payload, metadata and block offsets, on every kernel
family (fused TMA encoder with 5D page-run boxes, fused range coders, the
generic kernels and their fallbacks).
"""

import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _scatter(kv, P, rng, spare=3):
    """Pages of P tokens holding kv (L,H,T,C) under a random block table."""
    L, H, T, C = kv.shape
    need = -(-T // P)
    npages = need + spare
    table = torch.from_numpy(rng.permutation(npages)[:need].astype(np.int32)).cuda()
    pool = torch.full((L, npages * P, H, C), float("nan"), dtype=kv.dtype, device="cuda")
    rows = (table.long()[:, None] * P + torch.arange(P, device="cuda")[None, :]).reshape(-1)[:T]
    pool[:, rows] = kv.permute(0, 2, 1, 3)
    return pool.contiguous(), table, npages * P * H * C


def _classes(sid, imp):
    s = oracle.parse_id(sid)
    if s.quant == "mixed":
        return oracle.classify_heads(imp, s.rho)
    if s.quant == "mixlayer":
        return oracle.layer_classes(imp, s.rho)
    return None


def _check(sid, shape, P, seed, dtype=torch.bfloat16, block=2048, zeros=False):
    from paper_2605_13734_b200 import KVCodec

    v, imp = oracle.generate_kv(*shape, seed=seed)
    if zeros:  # rows the fused Hadamard encode leaves to the exact fixup pass
        v[0, 0, 1] = 0.0
        v[0, 0, 2, ::3] = 0.0
    kv = torch.from_numpy(v).to(dtype).cuda().contiguous()
    cls = _classes(sid, imp)
    codec = KVCodec(sid, shape, in_dtype=dtype, block_symbols=block)
    ref = codec.encode(kv, head_classes=cls)
    codec.check()
    want = (ref.payload_bytes(), ref.metadata_bytes(), ref.offsets_array())
    pool, table, stride = _scatter(kv, P, np.random.default_rng(seed))
    got = codec.encode_paged(pool, table, P, stride, head_classes=cls)
    codec.check()
    assert got.payload_bytes() == want[0], ("payload", sid, shape, P)
    assert got.metadata_bytes() == want[1], ("metadata", sid, shape, P)
    if want[2] is not None:
        assert np.array_equal(got.offsets_array(), want[2]), ("offsets", sid, shape, P)


@pytest.mark.parametrize("P", [4, 16, 64, 128, 1, 24])
@pytest.mark.parametrize("sid", [
    "t=identity;q=uniform,b=4,g=32;c=none",
    "t=delta;q=uniform,b=8,g=32;c=none",
    "t=hadamard;q=uniform,b=4,g=32;c=none",
    "t=affine;q=uniform,b=8,g=32;c=entropy",
    "t=hadamard;q=mixed,hi=8,lo=2,g=32,rho=0.25;c=entropy",
    "t=identity;q=mixtok,hi=8,lo=2,g=64,rho=0.25;c=rle",
    "t=identity;q=uniform,b=2,g=32;c=entropy",
    "t=identity;q=uchan,b=2,g=32;c=entropy",
    "t=identity;q=uchan,b=4,g=32;c=none",
])
def test_paged_encode_matches_contiguous(sid, P):
    """P = 4 .. 128 tile the 64-token tiles (5D TMA page runs on the fused
    encoder); P = 1 and 24 do not and take the generic kernels."""
    _check(sid, (2, 3, 256, 128), P, seed=P, zeros="hadamard" in sid)


@pytest.mark.parametrize("sid,shape,P", [
    ("t=identity;q=uniform,b=2,g=32;c=entropy", (2, 2, 200, 128), 16),  # ragged last block, rows across heads
    ("t=hadamard;q=uniform,b=4,g=32;c=none", (1, 2, 100, 128), 32),      # T not a multiple of 64
    ("t=delta;q=uniform,b=4,g=16;c=rle", (2, 2, 70, 64), 8),              # generic, head_dim 64
    ("t=identity;q=uniform,b=3,g=4;c=entropy", (1, 3, 33, 20), 5),        # generic, odd shapes
])
def test_paged_encode_ragged(sid, shape, P):
    _check(sid, shape, P, seed=7, block=256 if shape[3] != 128 else 2048)


def test_paged_encode_fp32_input():
    _check("t=hadamard;q=uniform,b=4,g=32;c=entropy", (1, 2, 128, 128), 16, seed=3, dtype=torch.float32)


@pytest.mark.parametrize("k", range(40))
def test_paged_encode_fuzz(k):
    from test_gpu_parity import _fuzz_case, _fuzz_case_fast

    sid, shape, block, in_f32 = (_fuzz_case_fast if k % 2 else _fuzz_case)(2000 + k)
    P = int(np.random.default_rng(k).choice([1, 4, 8, 16, 64, 100]))
    _check(sid, shape, P, seed=k, dtype=torch.float32 if in_f32 else torch.bfloat16, block=block)


def test_paged_roundtrip_through_the_cache():
    """Connector round trip: paged cache -> encode_paged -> decode_paged into a
    second pool equals the contiguous decode."""
    from paper_2605_13734_b200 import KVCodec

    shape = (2, 4, 512, 128)
    v, _ = oracle.generate_kv(*shape, seed=5)
    kv = torch.from_numpy(v).to(torch.bfloat16).cuda()
    for sid in ("t=hadamard;q=uniform,b=4,g=32;c=none", "t=identity;q=uchan,b=2,g=32;c=entropy"):
        codec = KVCodec(sid, shape)
        flat = codec.decode(codec.encode(kv))
        pool, table, stride = _scatter(kv, 16, np.random.default_rng(1))
        blob = codec.encode_paged(pool, table, 16, stride)
        dst = torch.zeros_like(pool)
        codec.decode_paged(blob, dst, table, 16, stride)
        codec.check(decoding=True)
        L, H, T, C = shape
        rows = (table.long()[:, None] * 16 + torch.arange(16, device="cuda")[None, :]).reshape(-1)[:T]
        assert torch.equal(dst[:, rows].permute(0, 2, 1, 3), flat), sid
