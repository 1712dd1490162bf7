"""Pipelined host round trip (hostpath.HostRoundTrip, the e2e path of
bench.py): pinned host KV -> encode -> (wire through pinned host memory, or
the blob kept in HBM) -> decode reproduces a direct decode bit for bit, and
the fused squared-error scalar equals the fp64 reference."""

import pytest

import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("via_host", [True, False])
@pytest.mark.parametrize("sid", ["t=identity;q=uniform,b=2,g=32;c=entropy", "t=identity;q=uchan,b=2,g=32;c=entropy",
                                 "t=hadamard;q=uniform,b=4,g=32;c=none", "t=delta;q=uniform,b=4,g=32;c=rle"])
def test_host_round_trip(sid, via_host):
    from paper_2605_13734_b200 import KVCodec
    from paper_2605_13734_b200.hostpath import HostRoundTrip

    shape = (6, 2, 2048, 128)
    v, _ = oracle.generate_kv(*shape, seed=5)
    kv = torch.from_numpy(v).to(torch.bfloat16)
    ref = KVCodec(sid, shape)
    want = ref.decode(ref.encode(kv.cuda()))
    rt = HostRoundTrip(sid, shape, chunk_layers=4, wire_via_host=via_host)  # a short last chunk
    host = kv.pin_memory()
    dev_in = torch.empty(shape, dtype=torch.bfloat16, device="cuda")
    out = torch.empty_like(dev_in)
    for _ in range(2):
        err = torch.zeros((), dtype=torch.float64, device="cuda")
        rt.run(host, dev_in, out, err)
        rt.check()
        assert torch.equal(out, want)
        e_ref = ((want.double() - kv.cuda().double()) ** 2).sum().item()
        assert err.item() == pytest.approx(e_ref, rel=1e-12)
    assert 0 < rt.wire_bytes() < kv.numel() * 2


@pytest.mark.parametrize("via_host", [True, False])
def test_host_round_trip_paged(via_host):
    """The c5 e2e path: decode into a paged cache (one block table for every
    layer), equal to a direct paged decode; the scalar is the compressed size."""
    from paper_2605_13734_b200 import KVCodec
    from paper_2605_13734_b200.hostpath import HostRoundTrip

    sid = "t=affine;q=uniform,b=8,g=32;c=entropy"
    shape = (5, 2, 1024, 128)
    L, H, T, C = shape
    v, _ = oracle.generate_kv(*shape, seed=6)
    kv = torch.from_numpy(v).to(torch.bfloat16)
    pt, n_pages = 16, T // 16
    table = torch.randperm(n_pages, device="cuda").to(torch.int32)
    stride = n_pages * pt * H * C
    ref = KVCodec(sid, shape)
    blob = ref.encode(kv.cuda())
    want = torch.empty(L * stride, dtype=torch.bfloat16, device="cuda")
    ref.decode_paged(blob, want, table, pt, stride)
    ref.check(decoding=True)
    rt = HostRoundTrip(sid, shape, chunk_layers=2, paged=(table, pt, stride), wire_via_host=via_host)
    host = kv.pin_memory()
    dev_in = torch.empty(shape, dtype=torch.bfloat16, device="cuda")
    out = torch.empty_like(want)
    res = torch.zeros((), dtype=torch.float64, device="cuda")
    rt.run(host, dev_in, out, res)
    rt.check()
    assert torch.equal(out, want)
    assert 0 < res.item() < kv.numel() * 2
