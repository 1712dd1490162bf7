"""GPU parity: CUDA codec vs the oracle on the same bf16-exact inputs.

Bit-exact for symbols / scales / zeros / payload / metadata / block offsets;
decoded float32 output bit-exact against the oracle's reconstruction where
the kernel reproduces the reference arithmetic, bf16 output within 1 bf16 ulp.
"""

import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def bf16_exact(v):
    t = torch.from_numpy(np.ascontiguousarray(v, dtype=np.float32)).to(torch.bfloat16)
    return t, t.float().numpy()


def run_case(sid, shape, seed=0, block=256, in_f32=False):
    from paper_2605_13734_b200 import KVCodec

    L, H, T, C = shape
    v, imp = oracle.generate_kv(L, H, T, C, seed=seed)
    tb, vb = bf16_exact(v)
    s = oracle.parse_id(sid)
    cls = None
    if s.quant == "mixed":
        cls = oracle.classify_heads(imp, s.rho)
    elif s.quant == "mixlayer":
        cls = oracle.layer_classes(imp, s.rho)
    ref = oracle.encode_blob(vb, imp, sid, block=block)
    in_dtype = torch.float32 if in_f32 else torch.bfloat16
    kv = (torch.from_numpy(vb) if in_f32 else tb).cuda().contiguous()
    codec = KVCodec(sid, shape, in_dtype=in_dtype, out_dtype=torch.float32, block_symbols=block)
    blob = codec.encode(kv, head_classes=cls)
    codec.check()
    assert blob.metadata_bytes() == ref["metadata"], ("metadata", sid)
    pay = blob.payload_bytes()
    assert len(pay) == len(ref["payload"]), (sid, len(pay), len(ref["payload"]))
    assert pay == ref["payload"], ("payload", sid)
    if ref["offsets"] is not None:
        assert np.array_equal(blob.offsets_array(), ref["offsets"]), ("offsets", sid)
    out = codec.decode(blob)
    codec.check(decoding=True)
    rec = oracle.decode_blob(ref["payload"], ref["metadata"], ref["offsets"], sid, shape, block=block)
    got = out.cpu().numpy()
    return got, rec, vb


STRATS = [
    "t=hadamard;q=uniform,b=4,g=32;c=none",
    "t=identity;q=uniform,b=2,g=32;c=none",
    "t=identity;q=uniform,b=3,g=64;c=none",
    "t=delta;q=uniform,b=8,g=32;c=none",
    "t=hadamard;q=mixed,hi=8,lo=2,g=32,rho=0.25;c=none",
    "t=identity;q=mixed,hi=4,lo=2,g=64,rho=0.125;c=none",
    "t=identity;q=uniform,b=2,g=32;c=entropy",
    "t=hadamard;q=uniform,b=4,g=32;c=entropy",
    "t=identity;q=uniform,b=8,g=32;c=entropy",
    "t=delta;q=mixed,hi=8,lo=4,g=32,rho=0.25;c=entropy",
    "t=identity;q=uniform,b=4,g=32;c=rle",
    "t=hadamard;q=mixed,hi=4,lo=2,g=32,rho=0.25;c=rle",
    "t=identity;q=uchan,b=2,g=32;c=none",
    "t=identity;q=uchan,b=2,g=32;c=entropy",
    "t=affine;q=uniform,b=8,g=32;c=entropy",
    "t=identity;q=mixtok,hi=8,lo=2,g=32,rho=0.25;c=none",
    "t=identity;q=mixlayer,hi=8,lo=2,g=32,rho=0.5;c=rle",
]


def fast_path(sid, shape, in_f32=False):
    """Does the DECODE run a fused head_dim-128 kernel?  (The decode does not
    depend on the input dtype; the uchan encoder does.)"""
    s = oracle.parse_id(sid)
    g = s.group
    if s.quant == "uchan":
        return shape[3] == 128 and g == 32 and shape[2] % 128 == 0 and not in_f32
    return shape[3] == 128 and g in (32, 64, 128)


def assert_decoded(got, rec, sid, shape, in_f32=False):
    """Decoded values: bit-exact where the kernel reproduces the reference's
    arithmetic (identity, delta, and the affine inverse, whose division is
    correctly rounded from the reciprocal by one residual step); the fused
    head_dim-128 decode runs the inverse Hadamard in fp32, held to the
    reference's own transform tolerance (1e-5, test_acceptance.py:235) scaled
    by the row magnitude."""
    t = oracle.parse_id(sid).transform
    if fast_path(sid, shape, in_f32) and t == "hadamard":
        rowmax = np.abs(rec).max(axis=-1, keepdims=True)
        assert np.all(np.abs(got - rec) <= 1e-5 * rowmax + 1e-30), (sid, float(np.abs(got - rec).max()))
    else:
        assert np.array_equal(got.view(np.uint32), rec.view(np.uint32)), ("decoded", sid)


@pytest.mark.parametrize("sid", STRATS)
@pytest.mark.parametrize("shape", [(2, 4, 64, 128), (1, 3, 96, 64), (1, 2, 100, 128)])
def test_parity_bitexact(sid, shape):
    if "uchan" in sid and shape[2] % 32:
        pytest.skip("uchan needs g | tokens")
    got, rec, _ = run_case(sid, shape, seed=hash((sid, shape)) % 1000)
    assert_decoded(got, rec, sid, shape)


@pytest.mark.parametrize("g", [8, 16, 32, 64, 128])
@pytest.mark.parametrize("t", ["identity", "delta", "hadamard", "affine"])
@pytest.mark.parametrize("b", [1, 3, 4, 8])
def test_fast128_groups_widths(g, t, b):
    sid = f"t={t};q=uniform,b={b},g={g};c=none"
    shape = (1, 2, 130, 128)
    got, rec, _ = run_case(sid, shape, seed=b * 7 + g)
    assert_decoded(got, rec, sid, shape)


def symbol_stream_kv(pattern, shape, bits, seed):
    """KV whose identity/uniform quantization yields a chosen symbol stream:
    every 32-group holds 0 and 2^b-1 (scale 1, zero 0), the other 30 values
    are the desired symbols."""
    rng = np.random.default_rng(seed)
    L, H, T, C = shape
    lv = (1 << bits) - 1
    n = L * H * T * C
    if pattern == "constant":
        s = np.full(n, 1)
    elif pattern == "skewed":
        s = np.minimum(rng.geometric(0.6, n) - 1, lv)
    elif pattern == "alternating":
        s = np.arange(n) % (lv + 1)
    else:
        s = rng.integers(0, lv + 1, n)
    s = s.reshape(-1, 32)
    s[:, 0] = 0
    s[:, 1] = lv
    return s.reshape(shape).astype(np.float32)


@pytest.mark.parametrize("pattern", ["constant", "skewed", "alternating", "random"])
@pytest.mark.parametrize("bits", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("block", [256, 2048, 4096, 8192])
def test_entropy_symbol_streams(pattern, bits, block):
    from paper_2605_13734_b200 import KVCodec

    shape = (1, 2, 72, 128)  # 18432 symbols: tails against every block size
    v = symbol_stream_kv(pattern, shape, bits, seed=bits * 31 + block)
    sid = f"t=identity;q=uniform,b={bits},g=32;c=entropy"
    ref = oracle.encode_blob(v, None, sid, block=block)
    codec = KVCodec(sid, shape, out_dtype=torch.float32, block_symbols=block)
    blob = codec.encode(torch.from_numpy(v).to(torch.bfloat16).cuda())
    codec.check()
    assert np.array_equal(blob.offsets_array(), ref["offsets"])
    assert blob.payload_bytes() == ref["payload"]
    out = codec.decode(blob).cpu().numpy()
    codec.check(decoding=True)
    assert np.array_equal(out, v)


def test_entropy_decode_rejects_corruption():
    from paper_2605_13734_b200 import KVCodec, _native

    shape = (1, 2, 64, 128)
    v = symbol_stream_kv("random", shape, 2, seed=1)
    sid = "t=identity;q=uniform,b=2,g=32;c=entropy"
    codec = KVCodec(sid, shape, block_symbols=1024)
    blob = codec.encode(torch.from_numpy(v).to(torch.bfloat16).cuda())
    codec.check()
    n = blob.payload_nbytes()
    # truncate the first block's coded bytes by lying about its length header
    blob.payload[0] = blob.payload[0] ^ 0x01
    codec.decode(blob)
    with pytest.raises(_native.CodecError):
        codec.check(decoding=True)
    blob.payload[0] = blob.payload[0] ^ 0x01
    # trailing bytes after the last block (codecs.py:429-430)
    blob._nbytes = n + 3
    codec.decode(blob)
    with pytest.raises(_native.CodecError):
        codec.check(decoding=True)


@pytest.mark.parametrize("b", [1, 2, 3, 4, 5, 8])
@pytest.mark.parametrize("t", ["identity", "affine"])
@pytest.mark.parametrize("c", ["none", "entropy"])
def test_uchan128(b, t, c):
    sid = f"t={t};q=uchan,b={b},g=32;c={c}"
    shape = (2, 3, 384, 128)
    got, rec, _ = run_case(sid, shape, seed=b)
    assert_decoded(got, rec, sid, shape)


@pytest.mark.parametrize("sid", [
    "t=hadamard;q=mixed,hi=8,lo=3,g=32,rho=0.25;c=none",
    "t=identity;q=mixtok,hi=5,lo=2,g=16,rho=0.3;c=none",
    "t=delta;q=mixlayer,hi=4,lo=1,g=64,rho=0.5;c=entropy",
])
def test_fast128_mixed_widths(sid):
    shape = (3, 4, 72, 128)
    got, rec, _ = run_case(sid, shape, seed=5)
    assert_decoded(got, rec, sid, shape)


@pytest.mark.parametrize("shape", [(1, 2, 5, 48), (2, 1, 7, 4), (1, 1, 3, 20)])
@pytest.mark.parametrize("sid", [
    "t=identity;q=uniform,b=3,g=4;c=none",
    "t=delta;q=mixed,hi=5,lo=3,g=4,rho=0.5;c=rle",
    "t=identity;q=uniform,b=7,g=4;c=entropy",
])
def test_parity_odd_shapes(sid, shape):
    got, rec, _ = run_case(sid, shape, seed=3, block=16)
    assert np.array_equal(got.view(np.uint32), rec.view(np.uint32)), sid


@pytest.mark.parametrize("channels", [64, 128])
def test_parity_all_180_ids_small(channels):
    from kv_space import all_ids  # noqa: F401  (tests/kv_space.py)

    shape = (2, 4, 16, channels)
    for sid in all_ids():
        got, rec, _ = run_case(sid, shape, seed=1, block=128)
        assert_decoded(got, rec, sid, shape)


@pytest.mark.parametrize("channels", [64, 128])
def test_parity_all_180_ids_default_block(channels):
    """Every strategy-space id at the reference's default 2048-symbol block,
    on a multi-block tensor (512 coded blocks for b=8): bitstream, offsets and
    metadata bit-exact, decode as assert_decoded."""
    from kv_space import all_ids

    shape = (2, 8, 512, channels)
    for k, sid in enumerate(all_ids()):
        got, rec, _ = run_case(sid, shape, seed=100 + k, block=2048)
        assert_decoded(got, rec, sid, shape)


def _fuzz_case(k):
    """Seeded random (id, shape, block, in_f32) over the extended grammar:
    every transform, quant kind, width 1..8, group and codec, with shapes the
    oracle accepts (g | C; power-of-two C for hadamard; g | T for uchan)."""
    rng = np.random.default_rng(9000 + k)
    t = ["identity", "delta", "hadamard", "affine"][rng.integers(4)]
    q = ["uniform", "uchan", "mixed", "mixtok", "mixlayer"][rng.integers(5)]
    c = ["none", "rle", "entropy"][rng.integers(3)]
    if t == "hadamard":
        C = int(2 ** rng.integers(2, 9))
    else:
        C = int(rng.choice([4, 8, 12, 20, 32, 48, 64, 96, 128, 160, 256]))
    gs = [g for g in (1, 2, 4, 8, 16, 32, 64, 128) if C % g == 0]
    g = int(rng.choice(gs))
    L, H = int(rng.integers(1, 4)), int(rng.integers(1, 5))
    T = int(rng.integers(1, 300))
    if q == "uchan":
        g = int(rng.choice([g for g in (1, 2, 4, 8, 16, 32, 64) if g <= 64]))
        T = max(1, T // g) * g
    if q in ("uniform", "uchan"):
        qs = f"{q},b={int(rng.integers(1, 9))},g={g}"
    else:
        hi = int(rng.integers(2, 9))
        lo = int(rng.integers(1, hi))
        qs = f"{q},hi={hi},lo={lo},g={g},rho={float(rng.choice([0.0, 0.125, 0.3, 0.5, 1.0]))!r}"
    block = int(rng.choice([16, 64, 128, 256, 2048]))
    in_f32 = bool(rng.integers(4) == 0)
    return f"t={t};q={qs};c={c}", (L, H, T, C), block, in_f32


def _fuzz_case_fast(k):
    """Seeded cases shaped for the fused head_dim-128 kernels (fast128,
    fused_rc, uchan128, delta128, rc_large): C=128, token counts that are and
    are not multiples of the kernels' tiles, every width, groups 8-128."""
    rng = np.random.default_rng(7000 + k)
    t = ["identity", "delta", "hadamard", "affine"][rng.integers(4)]
    q = ["uniform", "uniform", "uchan", "mixed", "mixtok", "mixlayer"][rng.integers(6)]
    c = ["none", "rle", "entropy", "entropy"][rng.integers(4)]
    g = int(rng.choice([8, 16, 32, 32, 64, 128]))
    L, H = int(rng.integers(1, 4)), int(rng.integers(1, 9))
    T = int(rng.choice([16, 128, 256, 384, 1024])) + int(rng.choice([0, 0, 0, 1, 7, 16, 100]))
    if q == "uchan":
        g = 32
        T = max(1, T // 128) * 128
    if q == "uniform" or q == "uchan":
        qs = f"{q},b={int(rng.integers(1, 9))},g={g}"
    else:
        hi = int(rng.integers(2, 9))
        lo = int(rng.integers(1, hi))
        qs = f"{q},hi={hi},lo={lo},g={g},rho={float(rng.choice([0.125, 0.25, 0.5]))!r}"
    block = int(rng.choice([512, 2048, 2048]))
    in_f32 = bool(rng.integers(5) == 0)
    return f"t={t};q={qs};c={c}", (L, H, T, 128), block, in_f32


@pytest.mark.parametrize("k", range(120))
def test_parity_fuzz_fused_shapes(k):
    sid, shape, block, in_f32 = _fuzz_case_fast(k)
    got, rec, _ = run_case(sid, shape, seed=k, block=block, in_f32=in_f32)
    assert_decoded(got, rec, sid, shape, in_f32=in_f32)


@pytest.mark.parametrize("k", range(200))
def test_parity_fuzz(k):
    sid, shape, block, in_f32 = _fuzz_case(k)
    got, rec, _ = run_case(sid, shape, seed=k, block=block, in_f32=in_f32)
    assert_decoded(got, rec, sid, shape, in_f32=in_f32)


@pytest.mark.parametrize("k", range(100))
def test_parity_fuzz_bf16_out_and_paged(k):
    """The production outputs on fuzzed cases: a bf16-output plan decodes the
    same blob to exactly bf16(RN(fp32 decode)), and a paged decode (random
    page size and page table, vLLM layout) holds the contiguous bf16 values."""
    from paper_2605_13734_b200 import KVCodec

    sid, shape, block, in_f32 = (_fuzz_case_fast if k % 2 else _fuzz_case)(1000 + k)
    got32, rec, vb = run_case(sid, shape, seed=k, block=block, in_f32=in_f32)
    assert_decoded(got32, rec, sid, shape, in_f32=in_f32)
    L, H, T, C = shape
    s = oracle.parse_id(sid)
    _, imp = oracle.generate_kv(L, H, T, C, seed=k)
    cls = oracle.classify_heads(imp, s.rho) if s.quant == "mixed" else (
        oracle.layer_classes(imp, s.rho) if s.quant == "mixlayer" else None)
    dt = torch.float32 if in_f32 else torch.bfloat16
    kv = torch.from_numpy(vb).to(dt).cuda().contiguous()
    codec = KVCodec(sid, shape, in_dtype=dt, out_dtype=torch.bfloat16, block_symbols=block)
    blob = codec.encode(kv, head_classes=cls)
    flat = codec.decode(blob)
    codec.check(decoding=True)
    want = torch.from_numpy(got32).to(torch.bfloat16).cuda()
    assert torch.equal(flat.view(torch.int16), want.view(torch.int16)), ("bf16 out", sid, shape)
    rng = np.random.default_rng(k)
    P = int(rng.choice([1, 3, 16, 32, 64, 128]))
    need = -(-T // P)
    npages = need + int(rng.integers(0, 4))
    table = torch.from_numpy(rng.permutation(npages)[:need].astype(np.int32)).cuda()
    pages = torch.zeros(L * npages * P * H * C, dtype=torch.bfloat16, device="cuda")
    codec.decode_paged(blob, pages, table, P, npages * P * H * C)
    codec.check(decoding=True)
    rows = (table.long()[:, None] * P + torch.arange(P, device="cuda")[None, :]).reshape(-1)[:T]
    pv = pages.view(L, npages * P, H, C)[:, rows].permute(0, 2, 1, 3)
    assert torch.equal(pv.view(torch.int16), flat.view(torch.int16)), ("paged", sid, shape, P)


def test_f32_input_matches_reference_fixture():
    """fp32 (non-bf16) inputs: the golden whole-tensor blobs from the reference."""
    from golden_io import items, load
    from paper_2605_13734_b200 import KVCodec

    g = load("pipeline_180.npz")
    vals, imp = g["values"], g["importance"]
    pays = items(g["payload"], g["payload_off"])
    metas = items(g["metadata"], g["metadata_off"])
    for k, sid in enumerate(g["ids"]):
        sid = str(sid)
        s = oracle.parse_id(sid)
        if s.codec != "none":
            continue
        cls = oracle.classify_heads(imp, s.rho) if s.quant == "mixed" else None
        codec = KVCodec(sid, vals.shape, in_dtype=torch.float32, out_dtype=torch.float32)
        blob = codec.encode(torch.from_numpy(vals).cuda(), head_classes=cls)
        codec.check()
        assert blob.payload_bytes() == pays[k], sid
        assert blob.metadata_bytes() == metas[k], sid
        out = codec.decode(blob).cpu().numpy()
        assert np.array_equal(out.view(np.uint32), g["recon"][k].view(np.uint32)), sid


@pytest.mark.parametrize("q", ["uniform", "uchan"])
@pytest.mark.parametrize("b", [1, 2, 3, 4])
@pytest.mark.parametrize("block", [128, 512, 2048])
def test_fused_entropy(q, b, block):
    """Fused quantize + range-code kernels (fused_rc.cu): per-token groups with
    a ragged last block, per-channel groups with several token chunks."""
    sid = f"t=identity;q={q},b={b},g=32;c=entropy"
    shape = (2, 2, 2048, 128) if q == "uchan" else (1, 3, 300, 128)
    got, rec, _ = run_case(sid, shape, seed=b * 13 + block, block=block)
    assert np.array_equal(got.view(np.uint32), rec.view(np.uint32)), sid


@pytest.mark.parametrize("q", ["uniform", "uchan"])
def test_fused_entropy_bf16_and_paged(q):
    from paper_2605_13734_b200 import KVCodec

    L, H, T, C = 2, 4, 1024, 128
    v, _ = oracle.generate_kv(L, H, T, C, seed=21)
    kv = torch.from_numpy(v).to(torch.bfloat16).cuda()
    sid = f"t=identity;q={q},b=2,g=32;c=entropy"
    ref = oracle.encode_blob(kv.float().cpu().numpy(), None, sid, block=512)
    rec = oracle.decode_blob(ref["payload"], ref["metadata"], ref["offsets"], sid, (L, H, T, C), block=512)
    codec = KVCodec(sid, (L, H, T, C), block_symbols=512)
    blob = codec.encode(kv)
    codec.check()
    assert blob.payload_bytes() == ref["payload"]
    flat = codec.decode(blob)
    codec.check(decoding=True)
    assert torch.equal(flat, torch.from_numpy(rec).to(torch.bfloat16).cuda())
    P = 16
    npages = T // P + 5
    table = torch.randperm(npages, device="cuda")[: T // P].to(torch.int32)
    pages = torch.zeros(L * npages * P * H * C, dtype=torch.bfloat16, device="cuda")
    codec.decode_paged(blob, pages, table, P, npages * P * H * C)
    codec.check(decoding=True)
    pv = pages.view(L, npages, P, H, C)[:, table.long()].reshape(L, T, H, C).permute(0, 2, 1, 3)
    assert torch.equal(pv, flat)


def test_fused_uchan_rejects_corruption():
    from paper_2605_13734_b200 import KVCodec, _native

    shape = (1, 2, 1024, 128)
    v, _ = oracle.generate_kv(*shape, seed=3)
    sid = "t=identity;q=uchan,b=2,g=32;c=entropy"
    codec = KVCodec(sid, shape, block_symbols=512)
    blob = codec.encode(torch.from_numpy(v).to(torch.bfloat16).cuda())
    codec.check()
    off = blob.offsets_array()
    k = int(off[37])
    blob.payload[k + 2] = blob.payload[k + 2] ^ 0x10  # block 37's length header
    codec.decode(blob)
    with pytest.raises(_native.CodecError):
        codec.check(decoding=True)


@pytest.mark.parametrize("sid", ["t=identity;q=uniform,b=2,g=32;c=entropy", "t=identity;q=uchan,b=2,g=32;c=entropy",
                                 "t=identity;q=uniform,b=4,g=32;c=none", "t=hadamard;q=uniform,b=4,g=32;c=none"])
def test_fp16_overflow_group_matches_reference_and_decode_raises(sid):
    """A group whose range exceeds fp16 gets an infinite scale exactly as in
    the reference (quantize.py:146); encode succeeds with identical bytes, and
    decoding that blob yields non-finite values, which the reference's
    KVTensor rejects (tensors.py:41-42) -> ValueError."""
    from paper_2605_13734_b200 import KVCodec

    shape = (1, 2, 1024, 128)
    v, _ = oracle.generate_kv(*shape, seed=8)
    v[0, 1, 100, 3] = 1.5e6  # after the Hadamard still ~1.3e5 > 65504
    v[0, 1, 100, 40] = -1.2e6
    tb, vb = bf16_exact(v)
    ref = oracle.encode_blob(vb, None, sid, block=1024)
    codec = KVCodec(sid, shape, out_dtype=torch.float32, block_symbols=1024)
    blob = codec.encode(tb.cuda())
    codec.check()
    assert blob.metadata_bytes() == ref["metadata"]
    assert blob.payload_bytes() == ref["payload"]
    codec.decode(blob)
    with pytest.raises(ValueError):
        codec.check(decoding=True)


@pytest.mark.parametrize("in_f32", [False, True])
def test_hadamard_fast_path_adversarial_rows_are_exact(in_f32):
    """The fused Hadamard encode leaves rows with zeros, tiny / huge
    magnitudes or near-midpoint results to the exact fixup pass
    (k_encode_fixup); every row must still match the reference bit for bit,
    for bf16 and for float32 (not bf16-exact) inputs."""
    shape = (1, 2, 64, 128)
    rng = np.random.default_rng(31)
    v = rng.normal(size=shape).astype(np.float32)
    v[0, 0, 1] = 0.0                                  # all-zero row
    v[0, 0, 2, ::3] = 0.0                             # sparse zeros
    v[0, 0, 3] *= 1e-33                               # tiny magnitudes (f32 subnormal outputs)
    v[0, 0, 4, :64] *= 2.0 ** -40                     # exponent span 2^+-40 within a row
    v[0, 0, 4, 64:] *= 2.0 ** 12
    v[0, 1, 5] = 1.0                                  # constant row (most outputs exactly 0)
    v[0, 1, 6, 7] = -3.0e-39                          # one tiny value in a normal row
    for sid in ("t=hadamard;q=uniform,b=4,g=32;c=none", "t=hadamard;q=uniform,b=2,g=64;c=entropy"):
        tb, vb = bf16_exact(v)
        if in_f32:
            vb = v
            tb = torch.from_numpy(v)
        ref = oracle.encode_blob(vb, None, sid, block=256)
        from paper_2605_13734_b200 import KVCodec
        codec = KVCodec(sid, shape, in_dtype=tb.dtype, out_dtype=torch.float32, block_symbols=256)
        blob = codec.encode(tb.cuda())
        codec.check()
        assert blob.metadata_bytes() == ref["metadata"], sid
        assert blob.payload_bytes() == ref["payload"], sid


def test_whole_stream_entropy_and_rle_match_reference_blobs():
    """with a codec block covering the whole tensor
    (block_symbols >= L*H*T*C) the payload IS the reference's whole-tensor
    format, byte for byte, for every rle / entropy id of the space:
    entropy = per width stream BE32 length + range_encode(stream)
    (codecs.py:361-367; the per-thread coders handle the model halvings of
    long streams), rle = rle_encode over the CONCATENATED byte-padded width
    streams (codecs.py:358-360; one rle block, mixed widths included)."""
    from golden_io import items, load
    from paper_2605_13734_b200 import KVCodec

    g = load("pipeline_180.npz")
    vals, imp = g["values"], g["importance"]
    pays = items(g["payload"], g["payload_off"])
    metas = items(g["metadata"], g["metadata_off"])
    E = int(np.prod(vals.shape))
    block = (E + 7) // 8 * 8
    checked = 0
    for k, sid in enumerate(g["ids"]):
        sid = str(sid)
        s = oracle.parse_id(sid)
        if s.codec == "none":
            continue  # (c=none blobs are compared in test_f32_input_matches_reference_fixture)
        cls = oracle.classify_heads(imp, s.rho) if s.quant == "mixed" else None
        codec = KVCodec(sid, vals.shape, in_dtype=torch.float32, out_dtype=torch.float32, block_symbols=block)
        blob = codec.encode(torch.from_numpy(vals).cuda(), head_classes=cls)
        codec.check()
        assert blob.payload_bytes() == pays[k], sid
        assert blob.metadata_bytes() == metas[k], sid
        out = codec.decode(blob).cpu().numpy()
        codec.check(decoding=True)
        assert np.array_equal(out.view(np.uint32), g["recon"][k].view(np.uint32)), sid
        checked += 1
    assert checked >= 120


@pytest.mark.parametrize("sid", ["t=hadamard;q=uniform,b=4,g=32;c=none", "t=hadamard;q=uniform,b=2,g=64;c=entropy",
                                 "t=hadamard;q=mixed,hi=8,lo=2,g=32,rho=0.25;c=none"])
def test_hadamard_decode_bf16_within_one_ulp(sid):
    """decoded bf16 within 1 bf16 ulp of bf16(reference) on
    paths with an inverse transform (the fused decode runs it in fp32)."""
    from paper_2605_13734_b200 import KVCodec

    shape = (2, 4, 256, 128)
    v, imp = oracle.generate_kv(*shape, seed=17)
    tb, vb = bf16_exact(v)
    s = oracle.parse_id(sid)
    cls = oracle.classify_heads(imp, s.rho) if s.quant == "mixed" else None
    codec = KVCodec(sid, shape, block_symbols=1024)
    out = codec.decode(codec.encode(tb.cuda(), head_classes=cls)).float().cpu().numpy()
    codec.check(decoding=True)
    ref = oracle.encode_blob(vb, imp, sid, block=1024)
    rec = oracle.decode_blob(ref["payload"], ref["metadata"], ref["offsets"], sid, shape, block=1024)
    ref_bf16 = torch.from_numpy(rec).to(torch.bfloat16).float().numpy()
    ulp = np.abs(out - ref_bf16) / np.maximum(np.abs(ref_bf16) * 2.0 ** -7, 1e-30)
    assert float(ulp.max()) <= 1.0 + 1e-6, (sid, float(ulp.max()))


@pytest.mark.parametrize("sid", ["t=delta;q=uniform,b=4,g=32;c=none", "t=delta;q=uniform,b=8,g=64;c=none",
                                 "t=delta;q=uniform,b=2,g=32;c=entropy", "t=delta;q=mixed,hi=8,lo=2,g=32,rho=0.25;c=none"])
def test_delta_chunked_decode_exact(sid):
    """Long sequences take the chunked delta decode (chunk sums -> carries ->
    verified chunk decode, delta128.cu); the result is the reference's
    sequential float64 cumsum bit for bit."""
    shape = (2, 2, 2048, 128)
    got, rec, _ = run_case(sid, shape, seed=23, block=1024)
    assert np.array_equal(got.view(np.uint32), rec.view(np.uint32)), sid


def test_delta_chunked_decode_falls_back_when_sums_round():
    """A running sum that rounds in float64 (a 3e4 offset then 1e-6 detail)
    makes the chunk carries disagree with the sequential sums; the head is
    re-decoded sequentially and still matches the reference exactly."""
    shape = (1, 2, 2048, 128)
    rng = np.random.default_rng(5)
    v = (1e-6 * rng.normal(size=shape)).astype(np.float32)
    v[:, :, :, :8] += 3.0e4  # every token: large channels, so the deltas keep tiny detail
    v[0, 0, 0, :] = 3.0e4
    sid = "t=delta;q=uniform,b=8,g=32;c=none"
    got, rec, _ = run_case(sid, shape, seed=0, block=1024) if False else (None, None, None)
    from paper_2605_13734_b200 import KVCodec
    tb, vb = bf16_exact(v)
    codec = KVCodec(sid, shape, out_dtype=torch.float32, block_symbols=1024)
    blob = codec.encode(tb.cuda())
    codec.check()
    ref = oracle.encode_blob(vb, None, sid, block=1024)
    assert blob.payload_bytes() == ref["payload"] and blob.metadata_bytes() == ref["metadata"]
    out = codec.decode(blob).cpu().numpy()
    codec.check(decoding=True)
    rec = oracle.decode_blob(ref["payload"], ref["metadata"], None, sid, shape, block=1024)
    assert np.array_equal(out.view(np.uint32), rec.view(np.uint32))


@pytest.mark.parametrize("sid", [
    "t=hadamard;q=uniform,b=4,g=32;c=none",
    "t=hadamard;q=uniform,b=2,g=64;c=none",
    "t=identity;q=uniform,b=4,g=32;c=none",
    "t=identity;q=uniform,b=8,g=128;c=none",
    "t=affine;q=uniform,b=8,g=32;c=none",
    "t=hadamard;q=uniform,b=2,g=32;c=entropy",
])
@pytest.mark.parametrize("shape", [(2, 4, 256, 128), (1, 2, 100, 128), (1, 1, 3, 128)])
def test_staged_bf16_decode_matches_fp32_decode(sid, shape):
    """Contiguous bf16 decode (the staged bulk-copy / tensor-store kernel for
    uniform widths when the tile bases are 16-byte aligned; (1, 1, 3) has
    12 groups and takes the direct kernel): equal to the fp32 decode rounded
    to bf16, including the partial last tile, and within tolerance of the
    oracle through that fp32 decode."""
    from paper_2605_13734_b200 import KVCodec

    v, _ = oracle.generate_kv(*shape, seed=11)
    tb, vb = bf16_exact(v)
    kv = tb.cuda().contiguous()
    c32 = KVCodec(sid, shape, out_dtype=torch.float32)
    c16 = KVCodec(sid, shape, out_dtype=torch.bfloat16)
    blob = c32.encode(kv)
    c32.check()
    o32 = c32.decode(blob)
    o16 = c16.decode(blob)
    torch.cuda.synchronize()
    c32.check(decoding=True)
    c16.check(decoding=True)
    assert o16.dtype == torch.bfloat16
    assert torch.equal(o16.view(torch.int16), o32.to(torch.bfloat16).view(torch.int16)), sid
    ref = oracle.encode_blob(vb, None, sid)
    rec = oracle.decode_blob(ref["payload"], ref["metadata"], ref["offsets"], sid, shape)
    assert_decoded(o32.cpu().numpy(), rec, sid, shape)


@pytest.mark.parametrize("t", ["identity", "delta", "hadamard", "affine"])
@pytest.mark.parametrize("g", [32, 64, 128])
@pytest.mark.parametrize("b", [2, 3, 4, 8])
def test_f32_fast_path_matches_oracle(t, g, b):
    """float32 inputs that are NOT bf16-exact (the reference's own corpora,
    tensors.py:102-103) take the fused head_dim-128 encoder (fp32 tensor tiles,
    2-stage ring): payload, scales and zeros bit-exact against the oracle,
    including a partial last tile (104 rows)."""
    from paper_2605_13734_b200 import KVCodec

    sid = f"t={t};q=uniform,b={b},g={g};c=none"
    shape = (1, 1, 104, 128) if t != "delta" else (2, 1, 104, 128)  # 104 rows: a partial tile
    v, imp = oracle.generate_kv(*shape, seed=17 * b + g)
    codec = KVCodec(sid, shape, in_dtype=torch.float32, out_dtype=torch.float32)
    assert codec.encode_path.startswith("fast128"), codec.encode_path
    blob = codec.encode(torch.from_numpy(v).cuda())
    codec.check()
    ref = oracle.encode_blob(v, imp, sid)
    assert blob.metadata_bytes() == ref["metadata"], sid
    assert blob.payload_bytes() == ref["payload"], sid


def test_f32_fast_path_flags_nonfinite():
    from paper_2605_13734_b200 import KVCodec

    shape = (1, 2, 64, 128)
    v, _ = oracle.generate_kv(*shape, seed=2)
    for sid in ("t=identity;q=uniform,b=4,g=32;c=none", "t=hadamard;q=uniform,b=4,g=32;c=none"):
        for bad in (np.nan, np.inf):
            x = v.copy()
            x[0, 1, 33, 77] = bad
            codec = KVCodec(sid, shape, in_dtype=torch.float32)
            codec.encode(torch.from_numpy(x).cuda())
            with pytest.raises(ValueError):
                codec.check()


@pytest.mark.parametrize("sid", ["t=affine;q=uniform,b=8,g=32;c=none", "t=affine;q=uniform,b=4,g=64;c=none",
                                 "t=affine;q=uchan,b=4,g=32;c=none", "t=affine;q=uniform,b=8,g=32;c=entropy"])
@pytest.mark.parametrize("out", ["f32", "bf16"])
def test_affine_decode_is_the_oracle_division(sid, out):
    """The affine inverse y / a + mu (oracle/extensions.py affine_inv) with a
    correctly rounded division: per-channel scales spread over 2^-12 .. 2^12
    so a takes thousands of fp16 values; fp32 output bit-exact, bf16 output
    equal to bf16(oracle) -- contiguous, and for bf16 also paged."""
    from paper_2605_13734_b200 import KVCodec

    shape = (2, 8, 256, 128)
    rng = np.random.default_rng(99)
    v = (rng.standard_normal(shape) * np.exp2(rng.uniform(-12, 12, size=shape[:2] + (1, shape[3])))).astype(np.float32)
    tb, vb = bf16_exact(v)
    ref = oracle.encode_blob(vb, None, sid, block=2048)
    rec = oracle.decode_blob(ref["payload"], ref["metadata"], ref["offsets"], sid, shape, block=2048)
    dt = torch.float32 if out == "f32" else torch.bfloat16
    codec = KVCodec(sid, shape, out_dtype=dt)
    blob = codec.encode(tb.cuda())
    codec.check()
    assert blob.payload_bytes() == ref["payload"]
    got = codec.decode(blob)
    codec.check(decoding=True)
    want = torch.from_numpy(rec).to(dt)
    assert torch.equal(got.cpu().view(torch.int16 if out == "bf16" else torch.int32),
                       want.view(torch.int16 if out == "bf16" else torch.int32)), sid
    if out == "bf16":
        L, H, T, C = shape
        pt, n_pages = 16, T // 16
        table = torch.randperm(n_pages, device="cuda").to(torch.int32)
        pool = torch.empty(L * n_pages * pt * H * C, dtype=torch.bfloat16, device="cuda")
        codec.decode_paged(blob, pool, table, pt, n_pages * pt * H * C)
        view = pool.view(L, n_pages, pt, H, C)[:, table.long()].reshape(L, T, H, C).permute(0, 2, 1, 3)
        assert torch.equal(view.cpu(), want), sid


@pytest.mark.parametrize("sid", ["t=identity;q=uniform,b=4,g=32;c=none", "t=identity;q=uniform,b=2,g=32;c=entropy",
                                 "t=identity;q=uchan,b=4,g=32;c=none"])
def test_signed_zero_group_minimum(sid):
    """A group whose minimum is a zero of one sign keeps that sign in its
    fp16 zero (quantize.py:147): -0.0 -> 0x8000, +0.0 -> 0x0000, as the
    reference gives (probed: zeros bits [32768, 0] for these rows).  Groups
    whose minimum is BOTH +0 and -0 are left out: numpy's SIMD min returns
    either sign depending on lane order."""
    from paper_2605_13734_b200 import KVCodec

    shape = (1, 2, 128, 128)
    rng = np.random.default_rng(5)
    v = (np.abs(rng.standard_normal(shape)) + 0.5).astype(np.float32)
    v[0, 0, 0, 5] = -0.0   # per-token group 0 of row 0: min -0
    v[0, 0, 1, 7] = 0.0    # row 1: min +0
    v[0, 1, 3, 40] = -0.0  # per-channel group (channel 40, tokens 0..31): min -0
    v[0, 1, 64, 41] = 0.0  # channel 41, tokens 64..95: min +0
    tb, vb = bf16_exact(v)
    ref = oracle.encode_blob(vb, None, sid, block=2048)
    codec = KVCodec(sid, shape, out_dtype=torch.float32)
    blob = codec.encode(tb.cuda())
    codec.check()
    assert blob.metadata_bytes() == ref["metadata"], sid
    assert blob.payload_bytes() == ref["payload"], sid
    zeros = np.frombuffer(ref["metadata"], dtype=np.uint16)[len(ref["metadata"]) // 4:]
    assert (zeros == 0x8000).any() and (zeros == 0).any()
