"""Pin the oracle (CPU restatement) against the reference's own outputs.

Two independent pins: (1) the golden fixtures generated from the unmodified
reference (tests/golden/make_golden.py) — these also run on the GPU box;
(2) live comparison against the reference package when it is mounted.
"""

import numpy as np
import pytest

import oracle
from golden_io import items, load


@pytest.fixture(scope="module")
def g180():
    return load("pipeline_180.npz")


def test_golden_180_whole_tensor_blobs(g180):
    vals, imp = g180["values"], g180["importance"]
    pays = items(g180["payload"], g180["payload_off"])
    metas = items(g180["metadata"], g180["metadata_off"])
    assert len(g180["ids"]) == 180
    for k, sid in enumerate(g180["ids"]):
        sid = str(sid)
        ob = oracle.encode_blob(vals, imp, sid, block=1 << 40)
        assert ob["metadata"] == metas[k], sid
        s = oracle.parse_id(sid)
        whole = oracle.pipeline.whole_payload(ob["streams"], s.codec)
        assert whole == pays[k], sid
        if s.codec in ("none", "rle"):
            # rle with a block covering the tensor is framed as ONE block over
            # the concatenated width streams: the reference payload itself
            assert ob["payload"] == pays[k], sid


def test_golden_180_reconstruction_through_block_framing(g180):
    vals, imp = g180["values"], g180["importance"]
    for k, sid in enumerate(g180["ids"]):
        sid = str(sid)
        for block in (64, 1 << 40):
            ob = oracle.encode_blob(vals, imp, sid, block=block)
            rec = oracle.decode_blob(ob["payload"], ob["metadata"], ob["offsets"], sid, vals.shape, block=block)
            assert np.array_equal(rec, g180["recon"][k]), (sid, block)


def test_golden_numerics_hd128():
    g = load("numerics_hd128.npz")
    v = g["values"]
    for tk, kind in (("identity", "identity"), ("delta_over_tokens", "delta"), ("hadamard_over_channels", "hadamard")):
        y = oracle.transform_fwd(v, kind)
        assert np.array_equal(y.view(np.uint32), g[f"y_{tk}"].view(np.uint32)), tk
        for b in (1, 2, 3, 4, 5, 8):
            for grp in (16, 32, 64, 128):
                bits = np.full(y.shape[:3], b, dtype=np.uint8)
                sym, sc, ze = oracle.quantize_any(y, bits, grp)
                key = f"{tk}_b{b}_g{grp}"
                assert np.array_equal(sym, g[f"sym_{key}"]), key
                assert sc.tobytes() == g[f"sc_{key}"].tobytes(), key
                assert ze.tobytes() == g[f"ze_{key}"].tobytes(), key
                if grp == 32:
                    deq = oracle.dequantize_rows(sym, sc, ze, grp)
                    ref = g[f"deq_{key}"]
                    if not np.isnan(ref).any():
                        assert np.array_equal(deq.view(np.uint32), ref.view(np.uint32)), key


def test_golden_codec_kats():
    g = load("codec_kats.npz")
    syms = items(g["rc_sym"], g["rc_sym_off"])
    outs = items(g["rc_out"], g["rc_out_off"])
    for s, a, o in zip(syms, g["rc_alpha"], outs):
        arr = np.frombuffer(s, dtype="<u2")
        assert oracle.range_encode(arr, int(a)) == o
        assert np.array_equal(oracle.range_decode(o, int(a), arr.size).astype(np.uint16), arr)
    for i, o in zip(items(g["rle_in"], g["rle_in_off"]), items(g["rle_out"], g["rle_out_off"])):
        assert oracle.rle_encode(i) == o
        assert oracle.rle_decode(o) == i
    for s, w, o in zip(items(g["pk_sym"], g["pk_sym_off"]), g["pk_w"], items(g["pk_out"], g["pk_out_off"])):
        arr = np.frombuffer(s, dtype=np.uint8)
        assert oracle.pack_bits(arr, int(w)) == o
        assert np.array_equal(oracle.unpack_bits(o, int(w), arr.size), arr)


def test_reference_test_vectors():
    """Known answers quoted in the reference's own tests."""
    assert oracle.pack_bits(np.array([1, 5, 2], np.uint8), 3) == bytes([0b00110101, 0])  # test_codecs.py:39-42
    assert oracle.rle_encode(b"AAAAB") == bytes([129, 65, 0, 66])  # test_codecs.py:74-79
    assert oracle.rle_encode(b"ABC") == bytes([2]) + b"ABC"
    assert oracle.rle_encode(b"") == b""
    assert oracle.rle_encode(b"\x07" * 300) == bytes([255, 7, 255, 7, 165, 7])  # :82-87
    assert oracle.rle_encode(b"\x07" * 131 + b"Z") == bytes([255, 7, 1]) + b"\x07Z"  # :90-94
    data = bytes(range(200))
    assert oracle.rle_encode(data) == bytes([127]) + data[:128] + bytes([71]) + data[128:]  # :97-101
    assert len(oracle.rle_encode(b"\x00" * 4096)) == 64  # :117-120
    with pytest.raises(oracle.OracleError):
        oracle.rle_decode(b"\x05ab")
    with pytest.raises(oracle.OracleError):
        oracle.rle_decode(b"\x81")
    coded = oracle.range_encode(np.arange(16, dtype=np.uint8) % 4, 4)
    with pytest.raises(oracle.OracleError):
        oracle.range_decode(coded[: max(1, len(coded) - 4)], 4, 64)  # test_codecs.py:153-157
    assert oracle.range_encode(np.zeros(0, np.uint8), 4) == b"\x00" * 4
    # SPEC example: group [0,1,2,3] at 2 bits -> symbols 0..3, scale 1, zero 0
    sym, sc, ze = oracle.quantize_any(np.arange(4, dtype=np.float32).reshape(1, 1, 1, 4), np.full((1, 1, 1), 2, np.uint8), 4)
    assert sym.reshape(-1).tolist() == [0, 1, 2, 3] and float(sc.reshape(-1)[0]) == 1.0 and float(ze.reshape(-1)[0]) == 0.0
    # degenerate group dequantizes to its anchor exactly (test_quantize.py:40-46)
    sym, sc, ze = oracle.quantize_any(np.full((1, 1, 2, 4), 5.0, np.float32), np.full((1, 1, 2), 2, np.uint8), 4)
    assert np.all(sc == 0) and np.all(sym == 0)
    assert np.all(oracle.dequantize_rows(sym, sc, ze, 4) == 5.0)


@pytest.mark.parametrize("shape", [(2, 3, 8, 32), (1, 2, 5, 48), (3, 1, 7, 16), (1, 1, 3, 4)])
def test_live_reference_pipeline(reference, shape):
    kp = reference
    from kvpilot.profiling.space import SpaceDef, enumerate_space

    L, H, T, C = shape
    x = kp.generate_kv_tensor(layers=L, heads=H, tokens=T, channels=C, seed=sum(shape))
    v, imp = oracle.generate_kv(L, H, T, C, seed=sum(shape))
    assert np.array_equal(v, x.values) and np.array_equal(imp, x.head_importance)
    for s in enumerate_space(SpaceDef(group_sizes=(C // 2 if C % 2 == 0 else C, C))).candidates:
        if s.transform.kind == "hadamard_over_channels" and C & (C - 1):
            continue
        tr = kp.apply_transform(x, s.transform)
        labels = kp.classify_heads(x, s.quant.retrieval_fraction) if s.quant.kind == "mixed_head" else None
        qt = kp.quantize(tr, s.quant, labels)
        blob = kp.encode_lossless(qt, s.codec)
        ob = oracle.encode_blob(x.values, x.head_importance, s.id, block=1 << 40)
        assert np.array_equal(ob["symbols"], qt.symbols), s.id
        assert ob["metadata"] == blob.metadata, s.id
        assert oracle.pipeline.whole_payload(ob["streams"], oracle.parse_id(s.id).codec) == blob.payload, s.id


def test_live_reference_uchan_is_transpose(reference):
    """The per-channel extension is the reference quantizer on the transpose."""
    kp = reference
    x = kp.generate_kv_tensor(layers=2, heads=2, tokens=64, channels=32, seed=4)
    xt = kp.KVTensor(values=x.values.transpose(0, 1, 3, 2).copy())
    qt = kp.quantize(xt, kp.QuantConfig(kind="uniform_group", bits=2, group_size=32))
    blob = kp.encode_lossless(qt, kp.CodecConfig(kind="none"))
    ob = oracle.encode_blob(x.values, None, "t=identity;q=uchan,b=2,g=32;c=none")
    assert ob["payload"] == blob.payload and ob["metadata"] == blob.metadata


def test_live_reference_mixlayer_is_mixed_head(reference):
    kp = reference
    x = kp.generate_kv_tensor(layers=4, heads=2, tokens=8, channels=32, seed=9)
    cls = oracle.layer_classes(x.head_importance, 0.5)
    q = kp.QuantConfig(kind="mixed_head", high_bits=8, low_bits=2, group_size=32, retrieval_fraction=0.5)
    blob = kp.encode_lossless(kp.quantize(x, q, cls), kp.CodecConfig(kind="none"))
    ob = oracle.encode_blob(x.values, x.head_importance, "t=identity;q=mixlayer,hi=8,lo=2,g=32,rho=0.5;c=none")
    assert ob["payload"] == blob.payload and ob["metadata"] == blob.metadata


@pytest.mark.parametrize("sid", [
    "t=affine;q=uniform,b=8,g=32;c=entropy",
    "t=identity;q=mixtok,hi=8,lo=2,g=32,rho=0.25;c=rle",
    "t=hadamard;q=uchan,b=2,g=16;c=entropy",
    "t=delta;q=mixlayer,hi=4,lo=2,g=64,rho=0.5;c=none",
])
def test_extension_roundtrip_and_error_bound(sid):
    v, imp = oracle.generate_kv(2, 4, 64, 64, seed=3)
    ob = oracle.encode_blob(v, imp, sid, block=256)
    rec = oracle.decode_blob(ob["payload"], ob["metadata"], ob["offsets"], sid, v.shape, block=256)
    assert rec.shape == v.shape and np.all(np.isfinite(rec))
    if not sid.startswith("t=delta"):  # delta integrates quantization error (test_compress.py:108-114)
        assert oracle.quality_score(v, rec) > 0.5
    with pytest.raises(oracle.OracleError):
        oracle.decode_blob(ob["payload"] + b"\x00", ob["metadata"], ob["offsets"], sid, v.shape, block=256) \
            if ob["offsets"] is None else oracle.decode_blob(ob["payload"], ob["metadata"] + b"\x00", ob["offsets"], sid, v.shape, block=256)
