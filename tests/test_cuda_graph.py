"""The codec inside CUDA graphs: encode and decode (contiguous and paged)
enqueue no host synchronisation and no allocation, so a serving loop can
capture a fixed-shape round trip once and replay it with one launch.
Replays must produce exactly the eager results, with fresh inputs copied into
the captured input buffer between replays."""

import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

IDS = [
    "t=hadamard;q=uniform,b=4,g=32;c=none",          # fused TMA encoder + exact fixup pass
    "t=identity;q=uniform,b=2,g=32;c=entropy",       # fused range coder + look-back scan + gather
    "t=identity;q=uchan,b=2,g=32;c=entropy",
    "t=affine;q=uniform,b=8,g=32;c=entropy",         # calibrate + rc_large
    "t=hadamard;q=mixed,hi=8,lo=2,g=32,rho=0.25;c=rle",
    "t=delta;q=uniform,b=4,g=16;c=none",              # generic path
]


@pytest.mark.parametrize("sid", IDS)
def test_graph_replay_matches_eager(sid):
    from paper_2605_13734_b200 import KVCodec

    shape = (2, 4, 512, 128)
    s = oracle.parse_id(sid)
    codec = KVCodec(sid, shape)
    cls = None
    inputs = []
    for seed in range(3):
        v, imp = oracle.generate_kv(*shape, seed=seed)
        if s.quant == "mixed":
            cls = oracle.classify_heads(imp, s.rho)
        inputs.append(torch.from_numpy(v).to(torch.bfloat16).cuda())
    # eager references
    want = []
    for x in inputs:
        b = codec.encode(x, head_classes=cls)
        want.append((b.payload_bytes(), codec.decode(b).clone()))
    codec.check(decoding=True)

    kv = torch.empty_like(inputs[0])
    kv.copy_(inputs[0])
    blob = codec.alloc_blob(cls)
    out = torch.empty(shape, dtype=torch.bfloat16, device="cuda")
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):  # warm up on the capture stream (torch's recipe)
        codec.encode(kv, head_classes=cls, out=blob, stream=side)
        codec.decode(blob, out=out, device_length=True, stream=side)
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        cur = torch.cuda.current_stream()
        codec.encode(kv, head_classes=cls, out=blob, stream=cur)
        codec.decode(blob, out=out, device_length=True, stream=cur)
    for k in (1, 2, 0, 1):
        kv.copy_(inputs[k])
        g.replay()
        torch.cuda.synchronize()
        codec.check(decoding=True)
        blob.refresh()  # the replay re-filled the blob behind encode()'s back
        assert blob.payload_bytes() == want[k][0], (sid, k)
        assert torch.equal(out, want[k][1]), (sid, k)


def test_graph_paged_connector():
    """Paged encode + paged decode captured together (the connector step)."""
    from paper_2605_13734_b200 import KVCodec

    sid = "t=hadamard;q=uniform,b=4,g=32;c=none"
    L, H, T, C, P = 2, 4, 512, 128, 16
    codec = KVCodec(sid, (L, H, T, C))
    rng = np.random.default_rng(0)
    n_pages = T // P + 2
    table = torch.from_numpy(rng.permutation(n_pages)[: T // P].astype(np.int32)).cuda()
    rows = (table.long()[:, None] * P + torch.arange(P, device="cuda")[None, :]).reshape(-1)
    stride = n_pages * P * H * C
    src = torch.zeros((L, n_pages * P, H, C), dtype=torch.bfloat16, device="cuda")
    dst = torch.zeros_like(src)
    blob = codec.alloc_blob()

    def fill(seed):
        v, _ = oracle.generate_kv(L, H, T, C, seed=seed)
        x = torch.from_numpy(v).to(torch.bfloat16).cuda()
        src[:, rows] = x.permute(0, 2, 1, 3)
        return codec.decode(codec.encode(x))

    fill(9)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        codec.encode_paged(src, table, P, stride, out=blob, stream=side)
        codec.decode_paged(blob, dst, table, P, stride, stream=side, device_length=True)
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        cur = torch.cuda.current_stream()
        codec.encode_paged(src, table, P, stride, out=blob, stream=cur)
        codec.decode_paged(blob, dst, table, P, stride, stream=cur, device_length=True)
    for seed in (3, 4):
        want = fill(seed)
        g.replay()
        torch.cuda.synchronize()
        codec.check(decoding=True)
        assert torch.equal(dst[:, rows].permute(0, 2, 1, 3), want)
