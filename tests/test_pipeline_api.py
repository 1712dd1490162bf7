"""Reference-facing API on the GPU: compress / decompress / timers /
evaluator behave like kvpilot.pipeline (tests mirror test_compress.py)."""

import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _tensor(shape=(2, 4, 64, 64), seed=0, bf16=False):
    from paper_2605_13734_b200 import KVTensor

    rng = np.random.default_rng(seed)
    vals = rng.normal(0, 1.0, shape).astype(np.float32)
    if bf16:
        vals = torch.from_numpy(vals).to(torch.bfloat16).float().numpy()
    return KVTensor(values=vals, head_importance=rng.uniform(0.0, 1.0, shape[:2]))


def test_measured_cr_equals_analytic_for_bitpack_codec():  # test_compress.py:18-25
    from paper_2605_13734_b200 import CostModelTimer, analytic_cr, compress, parse_strategy_id

    t = _tensor()
    for sid in ("t=identity;q=uniform,b=4,g=32;c=none", "t=identity;q=uniform,b=2,g=32;c=none"):
        s = parse_strategy_id(sid)
        blob, m = compress(t, s, timer=CostModelTimer())
        assert m.cr == pytest.approx(analytic_cr(s), rel=1e-12)


def test_fp32_inputs_match_oracle_and_roundtrip():
    """Arbitrary fp32 (not bf16-exact) inputs take the fp32 plan: blobs equal
    the oracle's; reconstruction equals the reference's bit for bit."""
    from paper_2605_13734_b200 import compress, decompress

    t = _tensor(seed=3)
    for sid in ("t=hadamard;q=uniform,b=4,g=32;c=none", "t=delta;q=mixed,hi=8,lo=2,g=32,rho=0.25;c=entropy"):
        blob, m = compress(t, sid)
        ref = oracle.encode_blob(t.values, t.head_importance, sid, block=2048)
        assert blob.payload == ref["payload"] and blob.metadata == ref["metadata"]
        rec, s_dec = decompress(blob, sid)
        want = oracle.decode_blob(ref["payload"], ref["metadata"], ref["offsets"], sid, t.shape, block=2048)
        assert np.array_equal(rec.values.cpu().numpy(), want)
        assert m.quality == pytest.approx(oracle.quality_score(t.values, want), abs=1e-12)
        assert s_dec > 0 and m.s_enc > 0 and m.s_dec > 0


def test_codec_choice_does_not_change_reconstruction():  # test_compress.py:55-64
    from paper_2605_13734_b200 import compress, decompress

    t = _tensor(seed=4, bf16=True)
    recs = []
    for codec in ("none", "rle", "entropy"):
        sid = f"t=identity;q=uniform,b=4,g=32;c={codec}"
        blob, _ = compress(t, sid)
        back, _ = decompress(blob, sid)
        recs.append(back.values.cpu().numpy())
    assert np.array_equal(recs[0], recs[1]) and np.array_equal(recs[0], recs[2])


def test_host_blob_decodes_without_device_copy():
    import dataclasses

    from paper_2605_13734_b200 import compress, decompress

    t = _tensor(seed=5, bf16=True)
    sid = "t=identity;q=uchan,b=2,g=32;c=entropy"
    blob, _ = compress(t, sid)
    host_only = dataclasses.replace(blob, device=None)
    a, _ = decompress(blob, sid)
    b, _ = decompress(host_only, sid)
    assert torch.equal(a.values, b.values)


def test_decompress_rejects_mismatched_strategy():  # test_compress.py:82-95
    from paper_2605_13734_b200 import CodecError, compress, decompress

    t = _tensor(seed=7)
    blob, _ = compress(t, "t=identity;q=uniform,b=4,g=32;c=none")
    for bad in ("t=identity;q=uniform,b=4,g=16;c=none", "t=identity;q=uniform,b=3,g=32;c=none",
                "t=identity;q=mixed,hi=8,lo=2,g=32,rho=0.25;c=none"):
        with pytest.raises(CodecError):
            decompress(blob, bad)


def test_nonfinite_input_raises_value_error():  # tensors.py:41-42
    from paper_2605_13734_b200 import KVTensor, compress

    for sid in ("t=identity;q=uniform,b=4,g=32;c=none", "t=hadamard;q=uniform,b=4,g=32;c=none",
                "t=delta;q=uniform,b=2,g=64;c=entropy", "t=affine;q=uniform,b=8,g=32;c=none",
                "t=identity;q=uchan,b=2,g=32;c=none", "t=hadamard;q=mixed,hi=8,lo=2,g=128,rho=0.25;c=rle"):
        for bad in (float("nan"), float("inf"), float("-inf")):
            v = torch.randn(1, 2, 128, 128, device="cuda", dtype=torch.bfloat16)
            v[0, 1, 37, 7] = bad
            with pytest.raises(ValueError):
                compress(KVTensor(v), sid)
    v = torch.randn(1, 2, 8, 64, device="cuda", dtype=torch.bfloat16)  # generic path
    v[0, 0, 2, 5] = float("nan")
    with pytest.raises(ValueError):
        compress(KVTensor(v), "t=hadamard;q=uniform,b=4,g=32;c=none")
    with pytest.raises(ValueError):
        KVTensor(np.full((1, 1, 2, 4), np.inf, np.float32))


def test_quality_improves_with_bits():  # test_compress.py:73-79
    from paper_2605_13734_b200 import CostModelTimer, compress

    t = _tensor(seed=6)
    q = [compress(t, f"t=identity;q=uniform,b={b},g=32;c=none", timer=CostModelTimer())[1].quality for b in (2, 4, 8)]
    assert q[0] < q[1] < q[2]


def test_cuda_event_timer_and_evaluator():
    from paper_2605_13734_b200 import CudaEventTimer, GpuCorpusEvaluator, KVTensor, parse_strategy_id

    corpus = []
    for i in range(6):
        v, imp = oracle.generate_kv(2, 4, 256, 128, seed=i)
        corpus.append(KVTensor(torch.from_numpy(v).to(torch.bfloat16).cuda(), imp))
    ev = GpuCorpusEvaluator(corpus, sample_size=3, timer=CudaEventTimer(repeats=2))
    s = parse_strategy_id("t=hadamard;q=uniform,b=4,g=32;c=none")
    acc, cr, lat = ev(s)
    assert 0.8 < acc < 1.0, acc
    assert cr == pytest.approx(3.2) and lat > 0, (cr, lat)
    s_enc, s_dec = ev.throughputs[s.id]
    # small (0.5 MB) tensors are launch-bound; still far above the CPU reference (~1e7 B/s)
    assert s_enc > 1e8 and s_dec > 1e8, (s_enc, s_dec)
    assert ev(s)[:2] == (acc, cr)  # sampling is a function of (seed, id)


@pytest.mark.parametrize("P", [4, 16, 64, 128, 24])
def test_paged_decode_matches_contiguous(P):
    """Paged decode (staged tensor stores for page runs of 4..128 tokens; 24
    does not tile 64 and takes the direct kernel) equals the contiguous one."""
    from paper_2605_13734_b200 import KVCodec

    L, H, T, C = 2, 4, 256, 128
    T = T if 256 % P == 0 else 192
    v, _ = oracle.generate_kv(L, H, T, C, seed=9)
    kv = torch.from_numpy(v).to(torch.bfloat16).cuda()
    for sid in ("t=hadamard;q=uniform,b=4,g=32;c=none", "t=identity;q=uchan,b=2,g=32;c=entropy",
                "t=affine;q=uniform,b=8,g=32;c=entropy", "t=delta;q=uniform,b=8,g=32;c=none"):
        codec = KVCodec(sid, (L, H, T, C))
        blob = codec.encode(kv)
        flat = codec.decode(blob)
        npages = T // P + 3
        table = torch.randperm(npages, device="cuda")[: T // P].to(torch.int32)
        pages = torch.zeros(L * npages * P * H * C, dtype=torch.bfloat16, device="cuda")
        codec.decode_paged(blob, pages, table, P, npages * P * H * C)
        codec.check(decoding=True)
        pv = pages.view(L, npages, P, H, C)[:, table.long()].reshape(L, T, H, C).permute(0, 2, 1, 3)
        assert torch.equal(pv, flat), sid


def test_paged_delta_long_sequence_chunked():
    """The chunked delta decode (long T) writes the same values into a paged
    cache as into a contiguous tensor."""
    from paper_2605_13734_b200 import KVCodec

    L, H, T, C = 2, 2, 2048, 128
    v, _ = oracle.generate_kv(L, H, T, C, seed=19)
    kv = torch.from_numpy(v).to(torch.bfloat16).cuda()
    for sid in ("t=delta;q=uniform,b=4,g=32;c=none", "t=delta;q=uniform,b=3,g=64;c=entropy"):
        codec = KVCodec(sid, (L, H, T, C))
        blob = codec.encode(kv)
        flat = codec.decode(blob)
        P = 32
        npages = T // P + 2
        table = torch.randperm(npages, device="cuda")[: T // P].to(torch.int32)
        pages = torch.zeros(L * npages * P * H * C, dtype=torch.bfloat16, device="cuda")
        codec.decode_paged(blob, pages, table, P, npages * P * H * C)
        codec.check(decoding=True)
        pv = pages.view(L, npages, P, H, C)[:, table.long()].reshape(L, T, H, C).permute(0, 2, 1, 3)
        assert torch.equal(pv, flat), sid


@pytest.mark.parametrize("T,P", [(200, 8), (240, 16), (256, 32)])
def test_paged_decode_ragged_tokens(T, P):
    """Token counts that do not tile 64-row (T = 200, 240: the direct paged
    kernel) and a page run of 32 (the staged kernel) give the contiguous
    decode's values in the paged cache."""
    from paper_2605_13734_b200 import KVCodec

    L, H, C = 2, 3, 128
    v, _ = oracle.generate_kv(L, H, T, C, seed=T + P)
    kv = torch.from_numpy(v).to(torch.bfloat16).cuda()
    for sid in ("t=hadamard;q=uniform,b=4,g=32;c=none", "t=affine;q=uniform,b=8,g=32;c=entropy",
                "t=identity;q=uniform,b=2,g=64;c=none"):
        codec = KVCodec(sid, (L, H, T, C))
        blob = codec.encode(kv)
        flat = codec.decode(blob)
        npages = -(-T // P) + 2
        table = torch.randperm(npages, device="cuda")[: -(-T // P)].to(torch.int32)
        pages = torch.zeros(L * npages * P * H * C, dtype=torch.bfloat16, device="cuda")
        codec.decode_paged(blob, pages, table, P, npages * P * H * C)
        codec.check(decoding=True)
        pv = pages.view(L, npages * P, H, C)
        rows = (table.long()[:, None] * P + torch.arange(P, device="cuda")[None, :]).reshape(-1)[:T]
        got = pv[:, rows].permute(0, 2, 1, 3)
        assert torch.equal(got, flat), sid


def _reference_blob(g, k, sid):
    """A CompressedBlob as the reference's compress() builds it
    (codecs.py:41-71): whole-tensor payload and metadata, no block table,
    no device copy -- from the golden fixtures the unmodified reference wrote."""
    from dataclasses import dataclass, field

    from golden_io import items

    @dataclass(frozen=True, eq=False)
    class RefBlob:
        payload: bytes
        metadata: bytes
        original_bytes: int
        shape: tuple
        group_size: int
        bits_per_head: np.ndarray
        mixed: bool
        head_importance: np.ndarray = field(repr=False, default=None)

    vals, imp = g["values"], g["importance"]
    s = oracle.parse_id(sid)
    L, H = vals.shape[:2]
    if s.quant == "mixed":
        cls = oracle.classify_heads(imp, s.rho)
        bits = np.where(cls, s.hi, s.lo).astype(np.int64)
    else:
        bits = np.full((L, H), s.bits, dtype=np.int64)
    pay = items(g["payload"], g["payload_off"])[k]
    meta = items(g["metadata"], g["metadata_off"])[k]
    return RefBlob(pay, meta, vals.size * 2, tuple(vals.shape), s.group, bits, s.quant == "mixed", imp)


def test_decompress_consumes_reference_written_blobs():
    """Drop-in in the other direction: blobs the reference CPU pipeline wrote
    (all 180 ids, none / rle / entropy, mixed included) decompress on the GPU
    to the reference's own reconstruction, bit for bit (block_symbols=None:
    the whole-tensor format; the entropy block table is walked from the
    BE32 stream headers)."""
    from golden_io import load

    from paper_2605_13734_b200 import decompress

    g = load("pipeline_180.npz")
    for k, sid in enumerate(g["ids"]):
        sid = str(sid)
        blob = _reference_blob(g, k, sid)
        rec, _ = decompress(blob, sid, block_symbols=None)
        got = rec.values.float().cpu().numpy() if hasattr(rec.values, "cpu") else np.asarray(rec.values)
        assert np.array_equal(got.view(np.uint32), g["recon"][k].view(np.uint32)), sid


def test_reference_written_blob_errors_are_codec_errors():
    import dataclasses

    from golden_io import load

    from paper_2605_13734_b200 import CodecError, decompress

    g = load("pipeline_180.npz")
    ids = [str(x) for x in g["ids"]]
    for sid in ("t=identity;q=uniform,b=2,g=32;c=entropy", "t=delta;q=mixed,hi=8,lo=2,g=32,rho=0.25;c=entropy",
                "t=identity;q=uniform,b=4,g=64;c=rle"):
        blob = _reference_blob(g, ids.index(sid), sid)
        for bad in (blob.payload + b"\x00", blob.payload[:-1], blob.payload[:3]):
            with pytest.raises(CodecError):
                decompress(dataclasses.replace(blob, payload=bad), sid, block_symbols=None)
