"""Generate the golden fixtures in tests/golden/ from the UNMODIFIED reference.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

It imports kvpilot from /root/reference/pkg/src and records, for seeded
bf16-exact inputs, the reference's own outputs: transformed values, symbols,
scales/zeros, whole-tensor blobs (payload + metadata) for all 180 ids of
enumerate_space(SpaceDef()), reconstructions, and codec known-answer vectors
(range coder, RLE, bit packing).  These fixtures pin the oracle
(tests/test_oracle_pins.py) and the CUDA path on the GPU box, where the
reference is absent.
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round float32 to the nearest bf16 (RNE), returned as float32."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    r = ((u + 0x7FFF + lsb) >> 16) << 16
    return r.astype(np.uint32).view(np.float32)


def _pack_list(items):
    """list[bytes] -> (concatenated uint8, int64 offsets)."""
    off = np.zeros(len(items) + 1, dtype=np.int64)
    off[1:] = np.cumsum([len(b) for b in items])
    buf = np.frombuffer(b"".join(items), dtype=np.uint8) if off[-1] else np.zeros(0, dtype=np.uint8)
    return buf, off


def edge_rows(C: int, rng) -> np.ndarray:
    """Adversarial rows for the transform/quantizer numerics."""
    rows = []
    rows.append(np.zeros(C, np.float32))                              # all zeros
    rows.append(np.full(C, 5.0, np.float32))                          # constant (degenerate groups)
    r = rng.normal(0, 1, C).astype(np.float32)
    r[::7] = 0.0
    rows.append(r)                                                    # sprinkled zeros
    r = rng.normal(0, 1, C).astype(np.float32) * np.float32(2.0) ** rng.integers(-40, 40, C).astype(np.float32)
    rows.append(r)                                                    # huge exponent span
    r = (rng.normal(0, 1, C) * 1e-39).astype(np.float32)
    rows.append(r)                                                    # bf16/fp32 subnormals
    r = rng.normal(0, 1, C).astype(np.float32)
    r[3] = 70000.0
    r[5] = -70000.0
    rows.append(r)                                                    # beyond fp16 range
    r = (rng.integers(-8, 8, C) * 0.25).astype(np.float32)
    rows.append(r)                                                    # quantizer ties
    r = np.linspace(-1, 1, C).astype(np.float32)
    rows.append(r)
    return bf16_round(np.stack(rows))


def main() -> None:
    sys.path.insert(0, REF)
    from kvpilot.pipeline import (
        KVTensor,
        apply_transform,
        classify_heads,
        decode_lossless,
        dequantize,
        encode_lossless,
        generate_kv_tensor,
        invert_transform,
        quantize,
    )
    from kvpilot.pipeline.codecs import pack_bits, range_encode, rle_encode
    from kvpilot.profiling.space import SpaceDef, enumerate_space

    # ---------------- whole pipeline, all 180 strategy ids -----------------
    base = generate_kv_tensor(layers=2, heads=4, tokens=16, channels=64, seed=11)
    vals = bf16_round(base.values)
    x = KVTensor(values=vals, head_importance=base.head_importance)
    ids, payloads, metas, recons = [], [], [], []
    for s in enumerate_space(SpaceDef()).candidates:
        tr = apply_transform(x, s.transform)
        labels = classify_heads(x, s.quant.retrieval_fraction) if s.quant.kind == "mixed_head" else None
        qt = quantize(tr, s.quant, labels)
        blob = encode_lossless(qt, s.codec)
        rec = invert_transform(dequantize(decode_lossless(blob, s.codec), s.quant), s.transform)
        ids.append(s.id)
        payloads.append(blob.payload)
        metas.append(blob.metadata)
        recons.append(rec.values)
    pbuf, poff = _pack_list(payloads)
    mbuf, moff = _pack_list(metas)
    np.savez_compressed(
        os.path.join(HERE, "pipeline_180.npz"),
        values=vals,
        importance=base.head_importance,
        ids=np.array(ids),
        payload=pbuf,
        payload_off=poff,
        metadata=mbuf,
        metadata_off=moff,
        recon=np.stack(recons),
        numpy_version=np.array(np.__version__),
    )

    # ------------- transform + quantizer numerics at head_dim 128 ------------
    rng = np.random.default_rng(5)
    kv = generate_kv_tensor(layers=1, heads=2, tokens=96, channels=128, seed=7)
    v = bf16_round(kv.values)
    edges = edge_rows(128, rng)
    v[0, 1, : edges.shape[0]] = edges
    xt = KVTensor(values=v)
    out = {"values": v}
    from kvpilot.pipeline.quantize import QuantConfig
    from kvpilot.pipeline.transforms import TransformConfig

    for tk in ("identity", "delta_over_tokens", "hadamard_over_channels"):
        tr = apply_transform(xt, TransformConfig(kind=tk))
        out[f"y_{tk}"] = tr.values
        for b in (1, 2, 3, 4, 5, 8):
            for g in (16, 32, 64, 128):
                qt = quantize(tr, QuantConfig(kind="uniform_group", bits=b, group_size=g))
                out[f"sym_{tk}_b{b}_g{g}"] = qt.symbols
                out[f"sc_{tk}_b{b}_g{g}"] = qt.scales
                out[f"ze_{tk}_b{b}_g{g}"] = qt.zeros
                if g == 32:
                    try:
                        deq = dequantize(qt, QuantConfig(kind="uniform_group", bits=b, group_size=g)).values
                    except ValueError:  # the fp16-overflow edge row reconstructs to +-inf
                        deq = np.full(v.shape, np.nan, np.float32)
                    out[f"deq_{tk}_b{b}_g{g}"] = deq
    np.savez_compressed(os.path.join(HERE, "numerics_hd128.npz"), **out)

    # ----------------------------- codec KATs ---------------------------------
    rng = np.random.default_rng(2024)
    rc_sym, rc_alpha, rc_out = [], [], []
    for k in range(120):
        alpha = [2, 4, 8, 16, 256, int(rng.integers(2, 257))][k % 6]
        n = int(rng.integers(0, 5000)) if k % 10 else int(rng.integers(2000, 70000))
        if k % 3 == 0:
            s = rng.integers(0, alpha, n)
        elif k % 3 == 1:
            s = np.minimum(rng.geometric(0.35, n) - 1, alpha - 1)
        else:
            s = np.full(n, alpha - 1)
        s = s.astype(np.uint16)
        rc_sym.append(s.astype("<u2").tobytes())
        rc_alpha.append(alpha)
        rc_out.append(range_encode(s, alpha))
    rle_in, rle_out = [], []
    for k in range(200):
        n = int(rng.integers(0, 3000))
        if k % 3 == 0:
            d = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
        elif k % 3 == 1:
            a = np.zeros(n, dtype=np.uint8)
            if n:
                hot = rng.integers(0, n, max(1, n // 50))
                a[hot] = rng.integers(1, 256, hot.size, dtype=np.uint8)
            d = a.tobytes()
        else:
            reps = rng.integers(1, 300, max(1, n // 8))
            d = np.repeat(rng.integers(0, 4, reps.size).astype(np.uint8), reps)[:n].tobytes()
        rle_in.append(d)
        rle_out.append(rle_encode(d))
    pk_sym, pk_w, pk_out = [], [], []
    for k in range(64):
        w = 1 + k % 8
        n = int(rng.integers(0, 700))
        s = rng.integers(0, 1 << w, n).astype(np.uint8)
        pk_sym.append(s.tobytes())
        pk_w.append(w)
        pk_out.append(pack_bits(s, w))
    a, ao = _pack_list(rc_sym)
    b, bo = _pack_list(rc_out)
    c, co = _pack_list(rle_in)
    d, do = _pack_list(rle_out)
    e, eo = _pack_list(pk_sym)
    f, fo = _pack_list(pk_out)
    np.savez_compressed(
        os.path.join(HERE, "codec_kats.npz"),
        rc_sym=a, rc_sym_off=ao, rc_alpha=np.array(rc_alpha), rc_out=b, rc_out_off=bo,
        rle_in=c, rle_in_off=co, rle_out=d, rle_out_off=do,
        pk_sym=e, pk_sym_off=eo, pk_w=np.array(pk_w), pk_out=f, pk_out_off=fo,
    )
    for name in ("pipeline_180.npz", "numerics_hd128.npz", "codec_kats.npz"):
        p = os.path.join(HERE, name)
        print(name, os.path.getsize(p), hashlib.sha256(open(p, "rb").read()).hexdigest()[:16])


if __name__ == "__main__":
    main()
