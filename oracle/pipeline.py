"""ORACLE (test infrastructure only): numpy restatement of the reference
pipeline stages.  Every function cites the reference file:line it follows;
paths are relative to /root/reference/pkg/src/kvpilot/pipeline/.

Arithmetic contract (what makes the CUDA path bit-exact against this):
  * Hadamard: float64 natural-order butterfly, stage h = 1, 2, ..., n/2,
    then a float64 division by sqrt(n) and a float32 cast
    (transforms.py:33-47, :58-63).
  * Delta: float32 differences along tokens, token 0 kept (transforms.py:56);
    inverse is a float64 cumulative sum cast to float32 (transforms.py:72).
  * Group scale = float16(float64(fp32(max - min)) / (2^b - 1)), zero =
    float16(min) (quantize.py:142-147); symbols from an IEEE fp32 division,
    rint half-to-even, clip, forced 0 where the scale is 0
    (quantize.py:149-154); dequantize is an unfused fp32 multiply then add
    (quantize.py:175-178).
  * Bit packing is MSB-first per width stream, streams by descending width,
    heads in (layer, head) order (codecs.py:79-100, :339-345).
"""

from __future__ import annotations

import ctypes
import math
import os
import struct
from dataclasses import dataclass

import numpy as np

__all__ = [
    "OracleError",
    "Strategy",
    "parse_id",
    "generate_kv",
    "fwht64",
    "transform_fwd",
    "transform_inv",
    "classify_heads",
    "quantize_rows",
    "dequantize_rows",
    "pack_bits",
    "unpack_bits",
    "rle_encode",
    "rle_decode",
    "range_encode",
    "range_decode",
    "width_streams",
    "metadata_bytes",
    "quality_score",
    "clib",
]


class OracleError(ValueError):
    """Mirrors the reference's CodecError(ValueError) (codecs.py:28)."""


# --------------------------------------------------------------------------
# strategy ids (strategy.py:8-19 grammar, plus the extension kinds of
# t=affine, q=uchan / mixlayer / mixtok)
# --------------------------------------------------------------------------

_T = {"identity": "identity", "delta": "delta", "hadamard": "hadamard", "affine": "affine"}
_C = {"none": "none", "rle": "rle", "entropy": "entropy"}
_Q_MIXED = ("mixed", "mixlayer", "mixtok")


@dataclass(frozen=True)
class Strategy:
    transform: str
    quant: str  # uniform | uchan | mixed | mixlayer | mixtok
    bits: int
    group: int
    hi: int
    lo: int
    rho: float
    codec: str

    @property
    def mixed(self) -> bool:
        return self.quant in _Q_MIXED


def parse_id(text: str) -> Strategy:
    """Parse a strategy id (strategy.py:68-109 grammar + extension kinds)."""
    seg = text.strip().split(";")
    if len(seg) != 3 or not seg[0].startswith("t=") or not seg[1].startswith("q=") or not seg[2].startswith("c="):
        raise ValueError(f"bad strategy id {text!r}")
    t = _T.get(seg[0][2:])
    c = _C.get(seg[2][2:])
    if t is None or c is None:
        raise ValueError(f"bad strategy id {text!r}")
    parts = seg[1][2:].split(",")
    kind, kv = parts[0], {}
    for p in parts[1:]:
        if "=" not in p:
            raise ValueError(f"bad token {p!r}")
        k, v = p.split("=", 1)
        kv[k] = v
    if kind in ("uniform", "uchan"):
        if set(kv) != {"b", "g"}:
            raise ValueError(f"bad quant segment {seg[1]!r}")
        b, g = int(kv["b"]), int(kv["g"])
        if not 1 <= b <= 8 or g < 1:
            raise ValueError(f"bad quant segment {seg[1]!r}")
        return Strategy(t, kind, b, g, 8, 2, 0.25, c)
    if kind in _Q_MIXED:
        if set(kv) != {"hi", "lo", "g", "rho"}:
            raise ValueError(f"bad quant segment {seg[1]!r}")
        hi, lo, g, rho = int(kv["hi"]), int(kv["lo"]), int(kv["g"]), float(kv["rho"])
        if not (1 <= lo < hi <= 8) or g < 1 or not 0.0 <= rho <= 1.0:
            raise ValueError(f"bad quant segment {seg[1]!r}")
        return Strategy(t, kind, 4, g, hi, lo, rho, c)
    raise ValueError(f"unknown quant kind {kind!r}")


# --------------------------------------------------------------------------
# synthetic KV (tensors.py:79-105) — same generator call sequence
# --------------------------------------------------------------------------


def generate_kv(layers=4, heads=8, tokens=64, channels=64, seed=0, outlier_fraction=0.01, outlier_scale=10.0):
    """Returns (values fp32 (L,H,T,C), importance fp64 (L,H)).

    Same draws, in the same order, as generate_kv_tensor (tensors.py:95-105).
    """
    rng = np.random.default_rng(seed)
    ch_scale = rng.lognormal(mean=0.0, sigma=0.5, size=(layers, heads, channels))
    n_hot = max(1, round(outlier_fraction * channels))
    for li in range(layers):
        for hi in range(heads):
            idx = rng.choice(channels, size=n_hot, replace=False)
            ch_scale[li, hi, idx] *= outlier_scale
    z = rng.standard_normal(size=(layers, heads, tokens, channels))
    vals = (z * ch_scale[:, :, None, :]).astype(np.float32)
    imp = rng.uniform(0.0, 1.0, size=(layers, heads))
    return vals, imp


# --------------------------------------------------------------------------
# transforms (transforms.py)
# --------------------------------------------------------------------------


def fwht64(x: np.ndarray) -> np.ndarray:
    """Unnormalised natural-order WHT in float64 (transforms.py:33-47).

    Stage h pairs element j*2h+i with j*2h+h+i -> (a+b, a-b); h = 1, 2, ...
    """
    n = x.shape[-1]
    y = np.array(x, dtype=np.float64)
    lead = y.shape[:-1]
    h = 1
    while h < n:
        v = y.reshape(*lead, n // (2 * h), 2, h)
        a = v[..., 0, :]
        b = v[..., 1, :]
        y = np.concatenate([(a + b)[..., None, :], (a - b)[..., None, :]], axis=-2).reshape(*lead, n)
        h <<= 1
    return y


def transform_fwd(values: np.ndarray, kind: str, affine=None) -> np.ndarray:
    """apply_transform (transforms.py:50-64); `affine` is the extension."""
    v = np.asarray(values, dtype=np.float32)
    if kind == "identity":
        return v
    if kind == "delta":
        out = np.empty_like(v)
        out[:, :, :1] = v[:, :, :1]
        out[:, :, 1:] = v[:, :, 1:] - v[:, :, :-1]
        return out
    if kind == "hadamard":
        n = v.shape[-1]
        if n & (n - 1):
            raise ValueError(f"hadamard needs power-of-two channels, got {n}")
        out = (fwht64(v) / np.sqrt(n)).astype(np.float32)
        if not np.all(np.isfinite(out)):
            raise ValueError("values must be finite")  # KVTensor re-validation, tensors.py:41-42
        return out
    if kind == "affine":
        from oracle.extensions import affine_fwd

        return affine_fwd(v, affine)
    raise ValueError(kind)


def transform_inv(values: np.ndarray, kind: str, affine=None) -> np.ndarray:
    """invert_transform (transforms.py:67-76)."""
    v = np.asarray(values, dtype=np.float32)
    if kind == "identity":
        return v
    if kind == "delta":
        return np.cumsum(v, axis=2, dtype=np.float64).astype(np.float32)
    if kind == "hadamard":
        return transform_fwd(v, "hadamard")
    if kind == "affine":
        from oracle.extensions import affine_inv

        return affine_inv(v, affine)
    raise ValueError(kind)


# --------------------------------------------------------------------------
# quantizer (quantize.py)
# --------------------------------------------------------------------------


def classify_heads(importance: np.ndarray, rho: float) -> np.ndarray:
    """Top ceil(rho*L*H) heads by importance, ties to lower index (quantize.py:97-112)."""
    imp = np.asarray(importance, dtype=np.float64)
    flat = imp.reshape(-1)
    k = math.ceil(rho * flat.size)
    out = np.zeros(flat.size, dtype=bool)
    if k > 0:
        out[np.argsort(-flat, kind="stable")[:k]] = True
    return out.reshape(imp.shape)


def quantize_rows(values: np.ndarray, bits_per_head: np.ndarray, group: int):
    """quantize (quantize.py:126-164) for given per-head widths.

    Groups are `group` consecutive entries of the last axis.
    Returns (symbols u8 same shape, scales f16 (..., C/g), zeros f16).
    """
    v = np.asarray(values, dtype=np.float32)
    L, H, T, C = v.shape
    if C % group:
        raise ValueError(f"group_size {group} does not divide channels {C}")
    levels = (2.0 ** np.asarray(bits_per_head, dtype=np.float64) - 1.0).reshape(L, H, 1, 1)
    grp = v.reshape(L, H, T, C // group, group)
    lo = grp.min(axis=-1)
    hi = grp.max(axis=-1)
    scales = ((hi - lo) / levels).astype(np.float16)  # fp32 diff, fp64 divide, one fp16 rounding
    zeros = lo.astype(np.float16)
    s32 = scales.astype(np.float32)
    z32 = zeros.astype(np.float32)
    div = np.where(s32 > 0.0, s32, np.float32(1.0))
    with np.errstate(invalid="ignore", over="ignore"):
        q = np.rint((grp - z32[..., None]) / div[..., None])
        q = np.clip(q, 0.0, levels[..., None])
        q = np.where(s32[..., None] > 0.0, q, 0.0)
        q = np.nan_to_num(q, nan=0.0)  # numpy's NaN->uint8 cast yields 0 on x86
    sym = q.astype(np.uint8).reshape(L, H, T, C)
    return sym, scales, zeros


def dequantize_rows(symbols: np.ndarray, scales: np.ndarray, zeros: np.ndarray, group: int) -> np.ndarray:
    """dequantize (quantize.py:175-178): zero + symbol*scale, unfused fp32."""
    L, H, T, C = symbols.shape
    s = scales.astype(np.float32)[..., None]
    z = zeros.astype(np.float32)[..., None]
    g = symbols.reshape(L, H, T, C // group, group).astype(np.float32)
    with np.errstate(invalid="ignore", over="ignore"):
        prod = g * s
        out = z + prod
    return out.reshape(L, H, T, C)


# --------------------------------------------------------------------------
# bit packing (codecs.py:79-100)
# --------------------------------------------------------------------------


def pack_bits(symbols: np.ndarray, width: int) -> bytes:
    """MSB-first packing of `width`-bit symbols, zero padded to a byte."""
    s = np.ascontiguousarray(symbols, dtype=np.uint8).reshape(-1)
    if s.size and int(s.max()) >= (1 << width):
        raise ValueError(f"symbol exceeds {width}-bit range")
    bits = (s[:, None] >> np.arange(width - 1, -1, -1, dtype=np.uint8)) & 1
    return np.packbits(bits.reshape(-1)).tobytes()


def unpack_bits(data: bytes, width: int, count: int) -> np.ndarray:
    need = (count * width + 7) // 8
    if len(data) != need:
        raise OracleError(f"bit-packed stream is {len(data)} bytes, expected {need}")
    if count == 0:
        return np.zeros(0, dtype=np.uint8)
    bits = np.unpackbits(np.frombuffer(data, dtype=np.uint8), count=count * width).reshape(count, width)
    weights = (1 << np.arange(width - 1, -1, -1)).astype(np.uint16)
    return (bits.astype(np.uint16) @ weights).astype(np.uint8)


# --------------------------------------------------------------------------
# serial codecs via the C restatement (oracle/codec.c)
# --------------------------------------------------------------------------

_LIB = None


def clib():
    """Load oracle/_build/liboracle.so, building it with make if needed."""
    global _LIB
    if _LIB is not None:
        return _LIB
    here = os.path.dirname(os.path.abspath(__file__))
    path = os.path.join(here, "_build", "liboracle.so")
    if not os.path.exists(path):
        import subprocess

        subprocess.run(["make", "-s", "-C", here], check=True)
    lib = ctypes.CDLL(path)
    P, S, U32, L = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint32, ctypes.c_long
    lib.oc_range_encode.argtypes = [P, S, U32, P, S]
    lib.oc_range_encode.restype = L
    lib.oc_range_decode.argtypes = [P, S, U32, S, P]
    lib.oc_range_decode.restype = ctypes.c_int
    lib.oc_rle_encode.argtypes = [P, S, P, S]
    lib.oc_rle_encode.restype = L
    lib.oc_rle_decode.argtypes = [P, S, P, S]
    lib.oc_rle_decode.restype = L
    lib.oc_entropy_encode_blocks.argtypes = [P, S, U32, S, P, S, P, ctypes.c_int]
    lib.oc_entropy_encode_blocks.restype = L
    lib.oc_entropy_decode_blocks.argtypes = [P, P, S, U32, S, P, ctypes.c_int]
    lib.oc_entropy_decode_blocks.restype = L
    _LIB = lib
    return lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def range_encode(symbols, alphabet: int) -> bytes:
    """range_encode (codecs.py:310-317)."""
    s = np.ascontiguousarray(np.asarray(symbols).reshape(-1), dtype=np.uint16)
    cap = 4 * s.size + 64
    out = np.empty(cap, dtype=np.uint8)
    n = clib().oc_range_encode(_ptr(s), s.size, alphabet, _ptr(out), cap)
    if n < 0:
        raise ValueError("range_encode failed (symbol out of range)")
    return out[:n].tobytes()


def range_decode(data: bytes, alphabet: int, count: int) -> np.ndarray:
    """range_decode (codecs.py:320-331); truncation raises OracleError."""
    buf = np.frombuffer(data, dtype=np.uint8).copy() if len(data) else np.zeros(1, dtype=np.uint8)
    out = np.empty(max(count, 1), dtype=np.uint16)
    rc = clib().oc_range_decode(_ptr(buf), len(data), alphabet, count, _ptr(out))
    if rc != 0:
        raise OracleError("range-coded stream truncated")
    return out[:count].astype(np.uint8 if alphabet <= 256 else np.uint16)


def rle_encode(data: bytes) -> bytes:
    """rle_encode (codecs.py:112-152)."""
    src = np.frombuffer(data, dtype=np.uint8).copy() if len(data) else np.zeros(1, dtype=np.uint8)
    cap = len(data) + len(data) // 128 + 16
    out = np.empty(cap, dtype=np.uint8)
    n = clib().oc_rle_encode(_ptr(src), len(data), _ptr(out), cap)
    if n < 0:
        raise ValueError("rle_encode capacity")
    return out[:n].tobytes()


def rle_decode(data: bytes, cap: int | None = None) -> bytes:
    """rle_decode (codecs.py:155-174); truncation raises OracleError."""
    src = np.frombuffer(data, dtype=np.uint8).copy() if len(data) else np.zeros(1, dtype=np.uint8)
    cap = cap if cap is not None else 130 * len(data) + 16
    out = np.empty(max(cap, 1), dtype=np.uint8)
    n = clib().oc_rle_decode(_ptr(src), len(data), _ptr(out), cap)
    if n == -1:
        raise OracleError("truncated literal run")
    if n == -2:
        raise OracleError("truncated repeat run")
    if n < 0:
        raise OracleError("rle output exceeds capacity")
    return out[:n].tobytes()


# --------------------------------------------------------------------------
# blob assembly (codecs.py:339-440)
# --------------------------------------------------------------------------


def width_streams(symbols: np.ndarray, bits_per_head: np.ndarray):
    """[(width, flat symbols)] for each distinct width, descending (codecs.py:339-345)."""
    out = []
    for w in sorted({int(b) for b in np.asarray(bits_per_head).reshape(-1)}, reverse=True):
        mask = np.asarray(bits_per_head) == w
        out.append((w, symbols[mask].reshape(-1)))
    return out


def metadata_bytes(scales: np.ndarray, zeros: np.ndarray, head_classes=None) -> bytes:
    """scales || zeros (fp16, C order) || packbits(class map) (codecs.py:348-352)."""
    parts = [np.ascontiguousarray(scales, dtype=np.float16).tobytes(), np.ascontiguousarray(zeros, dtype=np.float16).tobytes()]
    if head_classes is not None:
        parts.append(np.packbits(np.asarray(head_classes, dtype=bool).reshape(-1)).tobytes())
    return b"".join(parts)


def whole_payload(streams, codec: str) -> bytes:
    """encode_lossless payload over whole width streams (codecs.py:357-367)."""
    if codec in ("none", "rle"):
        packed = b"".join(pack_bits(s, w) for w, s in streams)
        return packed if codec == "none" else rle_encode(packed)
    parts = []
    for w, s in streams:
        coded = range_encode(s, 1 << w)
        parts.append(struct.pack(">I", len(coded)) + coded)
    return b"".join(parts)


def quality_score(original: np.ndarray, reconstructed: np.ndarray) -> float:
    """quality_score (tensors.py:115-134)."""
    a = np.asarray(original, dtype=np.float64)
    b = np.asarray(reconstructed, dtype=np.float64)
    if a.shape != b.shape:
        raise ValueError("shape mismatch")
    d = a - b
    rmse = math.sqrt(float(np.mean(d * d)))
    if rmse <= 1e-9:
        return 1.0
    rms = math.sqrt(float(np.mean(a * a)))
    if rms == 0.0:
        return 0.0
    return max(0.0, 1.0 - rmse / rms)
