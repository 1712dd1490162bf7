"""Pipelined compress -> transfer -> decompress: the
chunked, event-chained transfer reproduces a direct whole-tensor decode bit
for bit, on one GPU (loopback) and across two when present."""

import pytest

import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _kv(shape, seed):
    v, _ = oracle.generate_kv(*shape, seed=seed)
    return torch.from_numpy(v).to(torch.bfloat16)


@pytest.mark.parametrize("sid", ["t=identity;q=uniform,b=2,g=32;c=entropy", "t=hadamard;q=uniform,b=4,g=32;c=none",
                                 "t=identity;q=uchan,b=2,g=32;c=entropy", "t=delta;q=uniform,b=4,g=32;c=rle"])
def test_loopback_matches_direct_decode(sid):
    from paper_2605_13734_b200 import KVCodec
    from paper_2605_13734_b200.transfer import PipelinedKVTransfer

    shape = (5, 2, 1024, 128)  # 5 layers in chunks of 2: a short last chunk
    kv = _kv(shape, 3).cuda()
    ref = KVCodec(sid, shape, block_symbols=1024)
    want = ref.decode(ref.encode(kv))
    tx = PipelinedKVTransfer(sid, shape, 0, 0, chunk_layers=2, block_symbols=1024)
    for _ in range(2):  # buffers are reused across runs
        got = tx.run(kv)
        tx.check()
        torch.cuda.synchronize()
        assert torch.equal(got, want)
    assert 0 < tx.wire_bytes() < kv.numel() * 2


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs")
def test_two_gpus():
    from paper_2605_13734_b200 import KVCodec
    from paper_2605_13734_b200.transfer import PipelinedKVTransfer

    sid = "t=identity;q=uniform,b=2,g=32;c=entropy"
    shape = (4, 2, 2048, 128)
    kv = _kv(shape, 4).cuda(0)
    ref = KVCodec(sid, shape)
    want = ref.decode(ref.encode(kv))
    tx = PipelinedKVTransfer(sid, shape, 0, 1, chunk_layers=1)
    got = tx.run(kv)
    tx.check()
    torch.cuda.synchronize(1)
    assert got.device.index == 1 and torch.equal(got.cpu(), want.cpu())


def _pool(kv, P, seed, device):
    """Scatter kv (L,H,T,C) into a paged pool [L, pages*P, H, C] (random table)."""
    import numpy as np

    L, H, T, C = kv.shape
    need = -(-T // P)
    npages = need + 2
    table = torch.from_numpy(np.random.default_rng(seed).permutation(npages)[:need].astype(np.int32)).to(device)
    pool = torch.zeros((L, npages * P, H, C), dtype=kv.dtype, device=device)
    rows = (table.long()[:, None] * P + torch.arange(P, device=device)[None, :]).reshape(-1)[:T]
    pool[:, rows] = kv.to(device).permute(0, 2, 1, 3)
    return pool, table, rows, npages * P * H * C


@pytest.mark.parametrize("sid", ["t=hadamard;q=uniform,b=4,g=32;c=none", "t=identity;q=uniform,b=2,g=32;c=entropy",
                                 "t=affine;q=uniform,b=8,g=32;c=entropy"])
def test_loopback_paged_connector(sid):
    """Paged source cache -> encode_paged -> copy -> decode_paged into a
    differently paged destination equals the direct contiguous decode."""
    from paper_2605_13734_b200 import KVCodec
    from paper_2605_13734_b200.transfer import PipelinedKVTransfer

    shape = (5, 2, 1024, 128)
    kv = _kv(shape, 8).cuda()
    ref = KVCodec(sid, shape)
    want = ref.decode(ref.encode(kv))
    src, st, _, sstride = _pool(kv, 16, 1, "cuda:0")
    dst, dt, drows, dstride = _pool(torch.zeros_like(kv), 16, 2, "cuda:0")
    tx = PipelinedKVTransfer(sid, shape, 0, 0, chunk_layers=2)
    for _ in range(2):
        tx.run_paged(src, st, dst, dt, 16, sstride, dstride)
        tx.check()
        torch.cuda.synchronize()
        assert torch.equal(dst[:, drows].permute(0, 2, 1, 3), want), sid


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs")
def test_two_gpus_paged_connector():
    from paper_2605_13734_b200 import KVCodec
    from paper_2605_13734_b200.transfer import PipelinedKVTransfer

    sid = "t=hadamard;q=uniform,b=4,g=32;c=none"
    shape = (4, 2, 2048, 128)
    kv = _kv(shape, 9).cuda(0)
    ref = KVCodec(sid, shape)
    want = ref.decode(ref.encode(kv)).cpu()
    src, st, _, sstride = _pool(kv, 16, 3, "cuda:0")
    dst, dt, drows, dstride = _pool(torch.zeros_like(kv), 16, 4, "cuda:1")
    tx = PipelinedKVTransfer(sid, shape, 0, 1, chunk_layers=1)
    tx.run_paged(src, st, dst, dt, 16, sstride, dstride)
    tx.check()
    torch.cuda.synchronize(1)
    assert torch.equal(dst[:, drows].permute(0, 2, 1, 3).cpu(), want)


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs")
def test_codec_on_another_device_than_current():
    """A KVCodec on cuda:1 used while cuda:0 is the current device: its calls
    run on its own device and stream, and give cuda:0's results."""
    from paper_2605_13734_b200 import KVCodec

    shape = (2, 4, 512, 128)
    kv0 = _kv(shape, 12).cuda(0)
    for sid in ("t=hadamard;q=uniform,b=4,g=32;c=none", "t=identity;q=uniform,b=2,g=32;c=entropy"):
        c0 = KVCodec(sid, shape, device="cuda:0")
        c1 = KVCodec(sid, shape, device="cuda:1")
        torch.cuda.set_device(0)
        want = c0.decode(c0.encode(kv0)).cpu()
        kv1 = kv0.to("cuda:1")
        b1 = c1.encode(kv1)
        got = c1.decode(b1)
        c1.check(decoding=True)
        assert got.device.index == 1 and torch.equal(got.cpu(), want), sid
