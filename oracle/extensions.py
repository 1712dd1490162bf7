"""ORACLE (test infrastructure only): the full wire format of the GPU codec,
restated on top of the pinned primitives in ``oracle.pipeline``.

For the reference's own strategy kinds (t in identity/delta/hadamard,
q in uniform/mixed) the transform, quantizer, metadata and width-stream
layout are exactly the reference's whole-tensor ones
(compress.py:122-125 -> transforms.py, quantize.py, codecs.py:339-352).
The GPU codec differs from the reference blob only in the codec *framing*
for ``rle`` and ``entropy``: each width stream is cut into blocks of
``block`` symbols and every block is coded independently with the
reference's own codec function (so decoding is parallel):

    entropy block = BE32(len) || range_encode(chunk, 1 << w)  (codecs.py:364-366)
    rle block     = rle_encode(pack_bits(chunk, w))           (codecs.py:359-360)

plus a table of block byte offsets.  ``none`` is byte-identical to the
reference whole-tensor payload.

Extension kinds (absent from the reference — parity unpinned):
  * q=uchan,b,g    per-channel (KIVI-K) groups of g tokens: the reference
                   quantizer applied to the (L,H,C,T) transpose.
  * q=mixlayer     mixed_head with head classes = top ceil(rho*L) layers by
                   mean head importance (ties to the lower layer).
  * q=mixtok       per-token widths: the most recent ceil(rho*T) tokens of
                   every (layer, head) get hi bits, the rest lo bits.
  * t=affine       per-(layer, head, channel) shift/scale calibrated on the
                   first min(T, 128) tokens (midrange / half-range, fp16
                   parameters carried in the metadata).
"""

from __future__ import annotations

import math
import struct

import numpy as np

from oracle.pipeline import (
    OracleError,
    classify_heads,
    dequantize_rows,
    pack_bits,
    parse_id,
    range_decode,
    range_encode,
    rle_decode,
    rle_encode,
    transform_fwd,
    transform_inv,
    unpack_bits,
)

__all__ = [
    "AFFINE_PREFIX",
    "affine_calibrate",
    "affine_fwd",
    "affine_inv",
    "layer_classes",
    "row_bits",
    "quantize_any",
    "encode_blob",
    "decode_blob",
    "blob_streams",
]

AFFINE_PREFIX = 128


# --------------------------------------------------------------------------
# affine transform (extension)
# --------------------------------------------------------------------------


def affine_calibrate(values: np.ndarray):
    """(mu16, a16), each (L,H,C) float16, from the first min(T,128) tokens.

    mu = f16(0.5 * (max + min)), a = f16(2 / (max - min)) (fp32 ops, a = 1
    for a flat channel); a is clamped to the finite fp16 range.
    """
    v = np.asarray(values, dtype=np.float32)
    p = v[:, :, : min(v.shape[2], AFFINE_PREFIX), :]
    mx = p.max(axis=2)
    mn = p.min(axis=2)
    mu = (np.float32(0.5) * (mx + mn)).astype(np.float16)
    rng = mx - mn
    with np.errstate(divide="ignore", over="ignore"):
        a32 = np.where(rng > 0, np.float32(2.0) / np.where(rng > 0, rng, np.float32(1.0)), np.float32(1.0))
    a32 = np.minimum(a32.astype(np.float32), np.float32(65504.0))
    return mu, a32.astype(np.float16)


def affine_fwd(values: np.ndarray, params) -> np.ndarray:
    mu, a = params
    v = np.asarray(values, dtype=np.float32)
    return ((v - mu.astype(np.float32)[:, :, None, :]) * a.astype(np.float32)[:, :, None, :]).astype(np.float32)


def affine_inv(values: np.ndarray, params) -> np.ndarray:
    mu, a = params
    v = np.asarray(values, dtype=np.float32)
    return ((v / a.astype(np.float32)[:, :, None, :]) + mu.astype(np.float32)[:, :, None, :]).astype(np.float32)


# --------------------------------------------------------------------------
# width assignment
# --------------------------------------------------------------------------


def layer_classes(importance: np.ndarray, rho: float) -> np.ndarray:
    """mixlayer head classes: top ceil(rho*L) layers by mean importance."""
    imp = np.asarray(importance, dtype=np.float64)
    L, H = imp.shape
    per_layer = imp.mean(axis=1)
    k = math.ceil(rho * L)
    cls = np.zeros(L, dtype=bool)
    if k > 0:
        cls[np.argsort(-per_layer, kind="stable")[:k]] = True
    return np.repeat(cls[:, None], H, axis=1)


def row_bits(s, shape, importance):
    """(bits (L,H,T) uint8, head_classes or None) for strategy `s`."""
    L, H, T, _ = shape
    if s.quant in ("uniform", "uchan"):
        return np.full((L, H, T), s.bits, dtype=np.uint8), None
    if s.quant == "mixed":
        cls = classify_heads(importance, s.rho)
    elif s.quant == "mixlayer":
        cls = layer_classes(importance, s.rho)
    else:  # mixtok
        k = math.ceil(s.rho * T)
        tok = np.zeros(T, dtype=bool)
        if k:
            tok[T - k :] = True
        bits = np.where(tok, s.hi, s.lo).astype(np.uint8)
        return np.broadcast_to(bits[None, None, :], (L, H, T)).copy(), None
    bits = np.where(cls, s.hi, s.lo).astype(np.uint8)
    return np.broadcast_to(bits[:, :, None], (L, H, T)).copy(), cls


def quantize_any(y: np.ndarray, bits: np.ndarray, group: int):
    """quantize.py:126-164 with per-row widths (bits shaped (L,H,T))."""
    L, H, T, C = y.shape
    if C % group:
        raise ValueError(f"group_size {group} does not divide {C}")
    levels = (2.0 ** bits.astype(np.float64) - 1.0)[..., None]  # (L,H,T,1)
    grp = y.reshape(L, H, T, C // group, group)
    lo = grp.min(axis=-1)
    hi = grp.max(axis=-1)
    scales = ((hi - lo) / levels).astype(np.float16)
    zeros = lo.astype(np.float16)
    s32 = scales.astype(np.float32)
    z32 = zeros.astype(np.float32)
    div = np.where(s32 > 0.0, s32, np.float32(1.0))
    with np.errstate(invalid="ignore", over="ignore"):
        q = np.rint((grp - z32[..., None]) / div[..., None])
        q = np.clip(q, 0.0, levels[..., None])
        q = np.where(s32[..., None] > 0.0, q, 0.0)
        q = np.nan_to_num(q, nan=0.0)
    return q.astype(np.uint8).reshape(L, H, T, C), scales, zeros


# --------------------------------------------------------------------------
# full GPU wire format
# --------------------------------------------------------------------------


def _layout(s, values):
    """Quant-layout view: (L,H,rows,cols) with groups along cols."""
    return values.transpose(0, 1, 3, 2) if s.quant == "uchan" else values


def blob_streams(sym_l: np.ndarray, bits: np.ndarray):
    """[(w, flat symbols)] widths descending, rows in C order (codecs.py:339-345)."""
    out = []
    for w in sorted({int(b) for b in bits.reshape(-1)}, reverse=True):
        out.append((w, sym_l[bits == w].reshape(-1)))
    return out


def rle_whole(s, n_symbols: int, block: int) -> bool:
    """A block covering every symbol frames rle as ONE block over the
    concatenated byte-padded width streams: the reference's whole-tensor rle
    payload (codecs.py:358-360), mixed widths included (api.cu Geo::rle_whole)."""
    return s.codec == "rle" and block >= n_symbols and n_symbols * 8 < (1 << 31)


def encode_blob(values, importance, sid: str, block: int = 4096):
    """Returns dict(payload, metadata, offsets, streams, symbols, scales, zeros, y).

    `offsets` is None for codec none, else int64 array (nblocks+1).
    """
    s = parse_id(sid)
    v = np.asarray(values, dtype=np.float32)
    if not np.all(np.isfinite(v)):
        raise ValueError("values must be finite")
    if importance is None:
        importance = np.zeros(v.shape[:2])
    aff = affine_calibrate(v) if s.transform == "affine" else None
    y = transform_fwd(v, s.transform, aff)
    yl = np.ascontiguousarray(_layout(s, y))
    if s.quant == "uchan":
        bits = np.full(yl.shape[:3], s.bits, dtype=np.uint8)
        cls = None
    else:
        bits, cls = row_bits(s, v.shape, importance)
    sym, scales, zeros = quantize_any(yl, bits, s.group)
    streams = blob_streams(sym, bits)
    meta = [scales.tobytes(), zeros.tobytes()]
    if cls is not None:
        meta.append(np.packbits(cls.reshape(-1)).tobytes())
    if aff is not None:
        meta += [aff[0].tobytes(), aff[1].tobytes()]
    offsets = None
    if s.codec == "none":
        payload = b"".join(pack_bits(st, w) for w, st in streams)
    elif rle_whole(s, v.size, block):
        payload = rle_encode(b"".join(pack_bits(st, w) for w, st in streams))
        offsets = np.array([0, len(payload)] if payload else [0], dtype=np.int64)
    else:
        if block <= 0 or block % 8:
            raise ValueError("block must be a positive multiple of 8")
        parts = []
        for w, st in streams:
            for b0 in range(0, st.size, block):
                chunk = st[b0 : b0 + block]
                if s.codec == "entropy":
                    coded = range_encode(chunk, 1 << w)
                    parts.append(struct.pack(">I", len(coded)) + coded)
                else:
                    parts.append(rle_encode(pack_bits(chunk, w)))
        offsets = np.zeros(len(parts) + 1, dtype=np.int64)
        offsets[1:] = np.cumsum([len(p) for p in parts])
        payload = b"".join(parts)
    return dict(
        payload=payload,
        metadata=b"".join(meta),
        offsets=offsets,
        streams=streams,
        symbols=sym,
        scales=scales,
        zeros=zeros,
        bits=bits,
        classes=cls,
        affine=aff,
        y=y,
    )


def decode_blob(payload: bytes, metadata: bytes, offsets, sid: str, shape, block: int = 4096):
    """Inverse of encode_blob; returns float32 (L,H,T,C)."""
    s = parse_id(sid)
    L, H, T, C = shape
    lshape = (L, H, C, T) if s.quant == "uchan" else (L, H, T, C)
    G = lshape[3] // s.group
    ng = L * H * lshape[2] * G
    pos = 0
    scales = np.frombuffer(metadata[pos : pos + 2 * ng], dtype=np.float16).reshape(L, H, lshape[2], G)
    pos += 2 * ng
    zeros = np.frombuffer(metadata[pos : pos + 2 * ng], dtype=np.float16).reshape(scales.shape)
    pos += 2 * ng
    cls = None
    if s.quant in ("mixed", "mixlayer"):
        nb = (L * H + 7) // 8
        cls = np.unpackbits(np.frombuffer(metadata[pos : pos + nb], dtype=np.uint8), count=L * H).astype(bool).reshape(L, H)
        pos += nb
    aff = None
    if s.transform == "affine":
        n = L * H * C
        mu = np.frombuffer(metadata[pos : pos + 2 * n], dtype=np.float16).reshape(L, H, C)
        pos += 2 * n
        a = np.frombuffer(metadata[pos : pos + 2 * n], dtype=np.float16).reshape(L, H, C)
        pos += 2 * n
        aff = (mu, a)
    if pos != len(metadata):
        raise OracleError(f"metadata is {len(metadata)} bytes, expected {pos}")
    if s.quant == "uchan":
        bits = np.full(lshape[:3], s.bits, dtype=np.uint8)
    elif s.quant in ("mixed", "mixlayer"):
        bits = np.broadcast_to(np.where(cls, s.hi, s.lo).astype(np.uint8)[:, :, None], (L, H, T)).copy()
    elif s.quant == "mixtok":
        bits, _ = row_bits(s, shape, None)
    else:
        bits = np.full((L, H, T), s.bits, dtype=np.uint8)
    sym = np.zeros(lshape, dtype=np.uint8)
    off = 0
    blk = 0
    whole = None
    if rle_whole(s, L * H * T * C, block):
        nbytes = sum((int((bits == w).sum()) * lshape[3] * w + 7) // 8 for w in {int(b) for b in bits.reshape(-1)})
        seg = payload[offsets[0] : offsets[-1]] if offsets is not None and len(offsets) > 1 else b""
        whole = rle_decode(seg, cap=nbytes + 130) if seg else b""
        if len(whole) != nbytes:
            raise OracleError("rle payload decodes to the wrong length")
    for w in sorted({int(b) for b in bits.reshape(-1)}, reverse=True):
        mask = bits == w
        count = int(mask.sum()) * lshape[3]
        if s.codec == "none" or whole is not None:
            nbytes = (count * w + 7) // 8
            st = unpack_bits((whole if whole is not None else payload)[off : off + nbytes], w, count)
            off += nbytes
        else:
            pieces = []
            for b0 in range(0, count, block):
                n = min(block, count - b0)
                seg = payload[offsets[blk] : offsets[blk + 1]]
                blk += 1
                if s.codec == "entropy":
                    if len(seg) < 4:
                        raise OracleError("entropy payload truncated at stream header")
                    (ln,) = struct.unpack_from(">I", seg, 0)
                    if ln + 4 != len(seg):
                        raise OracleError("entropy block length mismatch")
                    pieces.append(range_decode(seg[4:], 1 << w, n))
                else:
                    raw = rle_decode(seg, cap=(n * w + 7) // 8 + 130)
                    pieces.append(unpack_bits(raw, w, n))
            st = np.concatenate(pieces) if pieces else np.zeros(0, dtype=np.uint8)
            off = int(offsets[blk]) if offsets is not None and len(offsets) else off
        sym[mask] = st.reshape(-1, lshape[3])
    if whole is not None:
        off = int(offsets[-1]) if offsets is not None and len(offsets) else 0
    if off != len(payload):
        raise OracleError(f"{len(payload) - off} trailing bytes in payload")
    deq = dequantize_rows(sym, scales, zeros, s.group)
    if s.quant == "uchan":
        deq = np.ascontiguousarray(deq.transpose(0, 1, 3, 2))
    return transform_inv(deq, s.transform, aff)
