"""Reference-facing pipeline API (kvpilot.pipeline), backed by the GPU codec.

Same entry points and signatures as the reference so the Bayesian profiling
engine and the online controller swap the codec in per profile with no
call-site change:

    compress(x, s, timer=None) -> (CompressedBlob, PipelineMetrics)   compress.py:111-140
    decompress(blob, s, timer=None) -> (KVTensor, s_dec)              compress.py:143-154
    StageTimer protocol; WallClockTimer / CostModelTimer              compress.py:43-108
    CudaEventTimer   (new) device-time StageTimer for GPU throughput
    GpuCorpusEvaluator (new) the Evaluator of profiling/search.py:318-368
    classify_heads, quality_score                                     quantize.py:97-112, tensors.py:115-134

`x` may be the reference's KVTensor (numpy float32 values), this module's
KVTensor, or anything with `.values` / `.head_importance`; values may be a
CUDA tensor (bf16 serving cache or fp32).  Strategies may be the reference's
StrategyConfig, ours, or an id string: the plan is keyed by `s.id`.
The CUDA path is the only path: without libkvc.so these functions raise.
"""

from __future__ import annotations

import hashlib
import math
import statistics
import time
from dataclasses import dataclass, field
from typing import Callable, Protocol, TypeVar

import numpy as np
import torch

from paper_2605_13734_b200 import _native as N
from paper_2605_13734_b200.codec import DeviceBlob, KVCodec
from paper_2605_13734_b200.strategy import StrategyConfig, as_strategy

__all__ = [
    "KVTensor",
    "CompressedBlob",
    "PipelineMetrics",
    "StageTimer",
    "WallClockTimer",
    "CostModelTimer",
    "CudaEventTimer",
    "CodecError",
    "classify_heads",
    "layer_classes",
    "quality_score",
    "compress",
    "decompress",
    "GpuCorpusEvaluator",
]

T = TypeVar("T")
CodecError = N.CodecError
SOURCE_WIDTH_BYTES = 2  # tensors.py:16


# --------------------------------------------------------------------------
# containers
# --------------------------------------------------------------------------


class KVTensor:
    """One KV block (tensors.py:22-76): values (L,H,T,C), importance (L,H).

    Values stay where they are: numpy (float32, like the reference) or a CUDA
    tensor (bf16 / fp32).  Validation follows tensors.py:35-51; the finite
    check of device values happens in the encode kernel (status word).
    """

    def __init__(self, values, head_importance=None) -> None:
        if isinstance(values, torch.Tensor):
            if values.dim() != 4:
                raise ValueError(f"values must be 4-D (layers, heads, tokens, channels), got shape {tuple(values.shape)}")
            shape = tuple(values.shape)
        else:
            values = np.asarray(values, dtype=np.float32)
            if values.ndim != 4:
                raise ValueError(f"values must be 4-D (layers, heads, tokens, channels), got shape {values.shape}")
            if not np.all(np.isfinite(values)):
                raise ValueError("values must be finite")
            shape = values.shape
        if min(shape) < 1:
            raise ValueError(f"all dims must be >= 1, got shape {shape}")
        if head_importance is None:
            imp = np.zeros(shape[:2], dtype=np.float64)
        else:
            imp = np.asarray(head_importance, dtype=np.float64).reshape(shape[:2])
            if imp.min() < 0.0 or imp.max() > 1.0:
                raise ValueError("head_importance must lie in [0, 1]")
        self.values = values
        self.head_importance = imp

    @property
    def shape(self):
        return tuple(self.values.shape)

    @property
    def nbytes_source(self) -> int:
        return int(np.prod(self.shape)) * SOURCE_WIDTH_BYTES

    def numpy(self) -> np.ndarray:
        v = self.values
        return v.float().cpu().numpy() if isinstance(v, torch.Tensor) else v


@dataclass(frozen=True, eq=False)
class CompressedBlob:
    """Encoded KV (codecs.py:41-71) in the GPU wire format.

    payload/metadata are host bytes; `block_offsets` frames rle/entropy
    blocks for parallel decode; `device` keeps the HBM copy for zero-copy
    decompress on the same GPU.
    """

    payload: bytes
    metadata: bytes
    original_bytes: int
    shape: tuple
    group_size: int
    bits_per_head: np.ndarray
    mixed: bool
    head_importance: np.ndarray = field(repr=False, default=None)
    block_offsets: np.ndarray | None = field(repr=False, default=None)
    strategy_id: str = ""
    device: DeviceBlob | None = field(repr=False, default=None)

    @property
    def metadata_nbytes(self) -> int:
        return len(self.metadata)

    @property
    def framing_nbytes(self) -> int:
        return 0 if self.block_offsets is None else 4 * (len(self.block_offsets) - 1)

    @property
    def compressed_nbytes(self) -> int:
        return len(self.payload) + len(self.metadata)

    @property
    def cr(self) -> float:
        """Reference accounting: original / (payload + metadata) (codecs.py:69-71)."""
        return self.original_bytes / self.compressed_nbytes

    @property
    def cr_wire(self) -> float:
        """Wire ratio including the block table needed for parallel decode."""
        return self.original_bytes / (self.compressed_nbytes + self.framing_nbytes)


@dataclass(frozen=True)
class PipelineMetrics:
    """(cr, s_enc, s_dec, quality) of one run (compress.py:25-40)."""

    cr: float
    s_enc: float
    s_dec: float
    quality: float

    @property
    def s_p(self) -> float:
        return self.s_enc * self.s_dec / (self.s_enc + self.s_dec)


# --------------------------------------------------------------------------
# timers (StageTimer protocol, compress.py:43-48)
# --------------------------------------------------------------------------


class StageTimer(Protocol):
    def measure(self, fn: Callable[[], T], nbytes: int, stage: str, strategy) -> tuple[T, float]: ...


class WallClockTimer:
    """Median-of-n host wall clock (compress.py:51-73); syncs the device."""

    def __init__(self, repeats: int = 3) -> None:
        if repeats < 1:
            raise ValueError("repeats must be >= 1")
        self.repeats = repeats

    def measure(self, fn, nbytes, stage, strategy):
        durations = []
        result = None
        for _ in range(self.repeats):
            result = None
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            result = fn()
            torch.cuda.synchronize()
            durations.append(time.perf_counter() - t0)
        return result, max(statistics.median(durations), 1e-12)


# per-byte stage costs (ns) of the reference's deterministic timer (compress.py:76-88)
_COST_TRANSFORM_NS = {"identity": 0.0, "delta_over_tokens": 0.05, "hadamard_over_channels": 0.45,
                      "affine_per_channel": 0.05}
_COST_QUANT_NS = {"uniform_group": 0.30, "mixed_head": 0.36, "uniform_channel": 0.30, "mixed_layer": 0.36,
                  "mixed_token": 0.36}
_COST_CODEC_ENC_NS = {"none": 0.10, "rle_bitpack": 0.90, "entropy": 55.0}
_COST_CODEC_DEC_NS = {"none": 0.08, "rle_bitpack": 0.55, "entropy": 60.0}


class CostModelTimer:
    """Deterministic seconds = bytes * per-byte cost (compress.py:91-108)."""

    def __init__(self, scale: float = 1.0) -> None:
        if scale <= 0.0:
            raise ValueError("scale must be positive")
        self.scale = scale

    def measure(self, fn, nbytes, stage, strategy):
        s = as_strategy(strategy)
        codec = _COST_CODEC_ENC_NS if stage == "encode" else _COST_CODEC_DEC_NS
        ns = _COST_TRANSFORM_NS[s.transform.kind] + _COST_QUANT_NS[s.quant.kind] + codec[s.codec.kind]
        return fn(), self.scale * nbytes * ns * 1e-9


class CudaEventTimer:
    """Device time of `fn` with CUDA events on the current stream, median of
    `repeats` — GPU throughput for the controller's latency model."""

    def __init__(self, repeats: int = 3, warmup: int = 1) -> None:
        if repeats < 1:
            raise ValueError("repeats must be >= 1")
        self.repeats = repeats
        self.warmup = warmup

    def measure(self, fn, nbytes, stage, strategy):
        result = None
        for _ in range(self.warmup):
            result = fn()
        times = []
        for _ in range(self.repeats):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            result = None  # free the previous result first: its allocation is reused, not grown
            a.record()
            result = fn()
            b.record()
            b.synchronize()
            times.append(a.elapsed_time(b) * 1e-3)
        return result, max(statistics.median(times), 1e-12)


# --------------------------------------------------------------------------
# head classes and quality
# --------------------------------------------------------------------------


def classify_heads(x, retrieval_fraction: float) -> np.ndarray:
    """Top ceil(rho*L*H) heads by importance, ties to lower (l,h) (quantize.py:97-112)."""
    if not 0.0 <= retrieval_fraction <= 1.0:
        raise ValueError(f"retrieval_fraction must be in [0, 1], got {retrieval_fraction}")
    imp = np.asarray(getattr(x, "head_importance", x), dtype=np.float64)
    flat = imp.reshape(-1)
    k = math.ceil(retrieval_fraction * flat.size)
    labels = np.zeros(flat.size, dtype=bool)
    if k > 0:
        labels[np.argsort(-flat, kind="stable")[:k]] = True
    return labels.reshape(imp.shape)


def layer_classes(x, retrieval_fraction: float) -> np.ndarray:
    """q=mixlayer head classes: the top ceil(rho*L) layers by mean importance."""
    imp = np.asarray(getattr(x, "head_importance", x), dtype=np.float64)
    L, H = imp.shape
    k = math.ceil(retrieval_fraction * L)
    cls = np.zeros(L, dtype=bool)
    if k > 0:
        cls[np.argsort(-imp.mean(axis=1), kind="stable")[:k]] = True
    return np.repeat(cls[:, None], H, axis=1)


def _as_device_values(x, device) -> torch.Tensor:
    v = x if isinstance(x, (torch.Tensor, np.ndarray)) else x.values
    if isinstance(v, torch.Tensor):
        return v.to(device) if v.device != device else v
    return torch.from_numpy(np.ascontiguousarray(v, dtype=np.float32)).to(device)


_SQ_PARTIALS = 592  # CTAs of the deterministic squared-sum kernel (4 per SM)


def _sum_sq(a: torch.Tensor, b: torch.Tensor | None) -> float:
    """sum((a - b)^2) (b None: sum(a^2)) in fp64 through kvc_sq_error_partials:
    one HBM-bound pass, no full-size fp64 temporaries, and the same bits on
    every call (fixed work split and reduction order)."""
    a = a.contiguous()
    b = None if b is None else b.contiguous()
    part = torch.zeros(_SQ_PARTIALS, dtype=torch.float64, device=a.device)
    dt = N.DTYPE_BF16 if a.dtype == torch.bfloat16 else N.DTYPE_F32
    N.check(N.lib().kvc_sq_error_partials(a.data_ptr(), None if b is None else b.data_ptr(), a.numel(), dt,
                                          part.data_ptr(), _SQ_PARTIALS,
                                          torch.cuda.current_stream(a.device).cuda_stream or None))
    return float(np.sum(part.cpu().numpy()))


def quality_score(original, reconstructed) -> float:
    """max(0, 1 - RMSE/RMS) in float64 (tensors.py:115-134), on the device:
    the squared error and the squared norm are fp64 sums from the fused
    kvc_sq_error kernel (per-element differences are exact in fp32 for
    bf16/fp32 inputs of one dtype)."""
    dev = torch.device("cuda", torch.cuda.current_device())
    a = _as_device_values(original, dev)
    b = _as_device_values(reconstructed, dev)
    if a.shape != b.shape:
        raise ValueError(f"shape mismatch: {tuple(a.shape)} vs {tuple(b.shape)}")
    if a.dtype != b.dtype or a.dtype not in (torch.bfloat16, torch.float32):
        a, b = a.float(), b.float()
    n = a.numel()
    rmse = math.sqrt(_sum_sq(a, b) / n)
    if rmse <= 1e-9:
        return 1.0
    rms = math.sqrt(_sum_sq(a, None) / n)
    if rms == 0.0:
        return 0.0
    return max(0.0, 1.0 - rmse / rms)


# --------------------------------------------------------------------------
# plans
# --------------------------------------------------------------------------

_PLANS: dict = {}


def _plan(sid: str, shape, in_dtype, block_symbols: int) -> KVCodec:
    key = (sid, tuple(shape), in_dtype, block_symbols, torch.cuda.current_device())
    p = _PLANS.get(key)
    if p is None:
        if len(_PLANS) > 64:
            _PLANS.clear()
        p = KVCodec(sid, shape, in_dtype=in_dtype, out_dtype=torch.float32, block_symbols=block_symbols)
        _PLANS[key] = p
    return p


def _bf16_exact(v: torch.Tensor) -> bool:
    """fp32 values that are all bf16-representable run through the bf16 fast
    path with identical results (the kernels see the same numbers)."""
    return bool(((v.view(torch.int32) & 0xFFFF) == 0).all())


def _classes_for(s: StrategyConfig, x) -> np.ndarray | None:
    if s.quant.kind == "mixed_head":
        return classify_heads(x, s.quant.retrieval_fraction)
    if s.quant.kind == "mixed_layer":
        return layer_classes(x, s.quant.retrieval_fraction)
    return None


def _bits_per_head(s: StrategyConfig, shape, classes) -> np.ndarray:
    L, H = shape[:2]
    q = s.quant
    if classes is not None:
        return np.where(classes, q.high_bits, q.low_bits).astype(np.uint8)
    if q.kind == "mixed_token":
        return np.full((L, H), q.high_bits, dtype=np.uint8)
    return np.full((L, H), q.bits, dtype=np.uint8)


# --------------------------------------------------------------------------
# compress / decompress (compress.py:111-166)
# --------------------------------------------------------------------------


def reference_block_symbols(shape) -> int:
    """A codec block covering the whole tensor: rle / entropy payloads then
    take the reference's whole-tensor format byte for byte (codecs.py:355-367;
    one range-coded stream per width, rle over the concatenated streams), so
    `cr` is the reference's own.  Decoding is then serial per width stream."""
    E = int(np.prod(shape))
    return max(8, (E + 7) // 8 * 8)


def compress(x, s, timer: StageTimer | None = None, block_symbols: int | None = 2048):
    """Encode + decode on the GPU and measure both sides (compress.py:111-140).
    block_symbols=None: the reference's whole-tensor payload format."""
    s = as_strategy(s)
    if not isinstance(x, KVTensor):
        vals = x if isinstance(x, (torch.Tensor, np.ndarray)) else x.values
        x = KVTensor(vals, getattr(x, "head_importance", None))
    timer = timer if timer is not None else CudaEventTimer()
    dev = torch.device("cuda", torch.cuda.current_device())
    v = _as_device_values(x, dev).contiguous()
    if v.dtype == torch.float32 and _bf16_exact(v):
        v = v.to(torch.bfloat16)
    if v.dtype not in (torch.bfloat16, torch.float32):
        v = v.float()
    nbytes = x.nbytes_source
    if block_symbols is None:
        block_symbols = reference_block_symbols(v.shape)
    codec = _plan(s.id, v.shape, v.dtype, block_symbols)
    classes = _classes_for(s, x)
    dblob, enc_s = timer.measure(lambda: codec.encode(v, head_classes=classes), nbytes, "encode", s)
    codec.check()
    rec, dec_s = timer.measure(lambda: codec.decode(dblob), nbytes, "decode", s)
    codec.check(decoding=True)
    blob = CompressedBlob(
        payload=dblob.payload_bytes(),
        metadata=dblob.metadata_bytes(),
        original_bytes=nbytes,
        shape=tuple(v.shape),
        group_size=s.quant.group_size,
        bits_per_head=_bits_per_head(s, v.shape, classes),
        mixed=s.quant.kind in ("mixed_head", "mixed_layer"),
        head_importance=x.head_importance,
        block_offsets=dblob.offsets_array(),
        strategy_id=s.id,
        device=_trimmed(dblob),
    )
    metrics = PipelineMetrics(cr=blob.cr, s_enc=nbytes / enc_s, s_dec=nbytes / dec_s, quality=quality_score(v, rec))
    return blob, metrics


def _trimmed(d: DeviceBlob) -> DeviceBlob:
    """The blob with its payload cut to the bytes actually written (the
    encode buffer is capacity-sized: ~4 B per symbol for entropy)."""
    n = d.payload_nbytes()
    offs = None if d.offsets is None else d.offsets[: d.nblocks + 1].clone()
    t = DeviceBlob(d.payload[: max(n, 1)].clone(), d.metadata.clone(), offs, d.strategy_id, d.shape, d.head_classes,
                   d.nblocks)
    t._nbytes = n
    return t


def _check_blob_matches(blob, s: StrategyConfig) -> None:
    """compress.py:157-166."""
    q = s.quant
    if blob.group_size != q.group_size:
        raise CodecError(f"blob group_size {blob.group_size} != strategy group_size {q.group_size}")
    if blob.mixed != (q.kind in ("mixed_head", "mixed_layer")):
        raise CodecError(f"blob quantizer layout does not match strategy {s.id!r}")
    widths = {int(w) for w in np.asarray(blob.bits_per_head).reshape(-1)}
    allowed = {q.high_bits, q.low_bits} if q.kind in ("mixed_head", "mixed_layer", "mixed_token") else {q.bits}
    if not widths <= allowed:
        raise CodecError(f"blob symbol widths {sorted(widths)} incompatible with strategy {s.id!r}")
    sid = getattr(blob, "strategy_id", "")
    if sid and sid != s.id:
        raise CodecError(f"blob was encoded with {sid!r}, not {s.id!r}")


def _checked_offsets(offsets, payload_len: int, nblocks: int) -> np.ndarray:
    """Validate a host block table before it reaches the device: starts at 0,
    ends at the payload length, never decreases, one entry per block + 1."""
    o = np.asarray(offsets)
    if o.ndim != 1 or o.dtype.kind not in "iu":
        raise CodecError("block offsets must be a 1-D integer array")
    o = o.astype(np.int64)
    if o.size != nblocks + 1:
        raise CodecError(f"block table has {o.size - 1} blocks, expected {nblocks}")
    if o[0] != 0 or o[-1] != payload_len:
        raise CodecError(f"block offsets span [{o[0]}, {o[-1]}], payload is {payload_len} bytes")
    if np.any(np.diff(o) < 0):
        raise CodecError("block offsets decrease")
    return np.ascontiguousarray(o)


def _whole_format_offsets(payload: np.ndarray, codec_kind: str, nblocks: int) -> np.ndarray:
    """Block table of a reference whole-tensor payload (codecs.py:355-367),
    which carries none: rle is one block; entropy is one BE32-length-prefixed
    stream per width (codecs.py:364-366), walked here with the reference's
    truncation / trailing-byte rules (codecs.py:412-413, :429-430)."""
    n = payload.size
    if codec_kind == "rle":
        return np.array([0, n] if nblocks else [0], dtype=np.int64)
    offs = [0]
    for _ in range(nblocks):
        o = offs[-1]
        if o + 4 > n:
            raise CodecError("entropy payload truncated at a stream header")
        ln = int.from_bytes(payload[o:o + 4].tobytes(), "big")
        if o + 4 + ln > n:
            raise CodecError("entropy payload truncated inside a stream")
        offs.append(o + 4 + ln)
    if offs[-1] != n:
        raise CodecError(f"{n - offs[-1]} trailing bytes in entropy payload")
    return np.array(offs, dtype=np.int64)


def decompress(blob: CompressedBlob, s, timer: StageTimer | None = None, block_symbols: int | None = 2048):
    """Full inverse pipeline on the GPU; returns (KVTensor fp32 on device, s_dec).
    block_symbols=None: the blob is in the reference's whole-tensor format --
    including a CompressedBlob the reference's own compress() produced
    (no block table, no device copy: both are derived here)."""
    s = as_strategy(s)
    whole = block_symbols is None
    if block_symbols is None:
        block_symbols = reference_block_symbols(blob.shape)
    timer = timer if timer is not None else CudaEventTimer()
    _check_blob_matches(blob, s)
    dev = torch.device("cuda", torch.cuda.current_device())
    dblob = getattr(blob, "device", None)
    in_dtype = torch.bfloat16
    if dblob is None or dblob.payload.device != dev:
        codec = _plan(s.id, blob.shape, in_dtype, block_symbols)
        dblob = codec.alloc_blob(None)
        pay = np.frombuffer(blob.payload, dtype=np.uint8)
        meta = np.frombuffer(blob.metadata, dtype=np.uint8)
        if meta.size != codec.metadata_bytes:
            raise CodecError(f"metadata is {meta.size} bytes, expected {codec.metadata_bytes}")
        if pay.size > dblob.payload.numel():
            raise CodecError("payload exceeds the plan's capacity")
        dblob.payload[: pay.size].copy_(torch.from_numpy(pay.copy()))
        dblob.metadata.copy_(torch.from_numpy(meta.copy()))
        block_offsets = getattr(blob, "block_offsets", None)
        if codec.codec_kind != "none":
            cls = (np.asarray(blob.bits_per_head) == s.quant.high_bits) if blob.mixed else None
            nblocks = codec.num_blocks(head_classes=cls)
            if block_offsets is None:
                if not whole:
                    raise CodecError("rle/entropy blob without a block offset table")
                block_offsets = _whole_format_offsets(pay, codec.codec_kind, nblocks)
            offs_np = _checked_offsets(block_offsets, pay.size, nblocks)
            offs = torch.from_numpy(offs_np)
            dblob.offsets[: offs.numel()].copy_(offs)
            dblob.nblocks = offs.numel() - 1
        dblob._nbytes = pay.size
    else:
        codec = _plan(s.id, blob.shape, torch.bfloat16, block_symbols)
    rec, dec_s = timer.measure(lambda: codec.decode(dblob), blob.original_bytes, "decode", s)
    codec.check(decoding=True)
    return KVTensor(rec, blob.head_importance), blob.original_bytes / dec_s


# --------------------------------------------------------------------------
# profiling-engine evaluator (profiling/search.py:318-368)
# --------------------------------------------------------------------------


def _stable_hash(text: str) -> int:
    return int.from_bytes(hashlib.sha256(text.encode()).digest()[:8], "big")


class GpuCorpusEvaluator:
    """Drop-in for CorpusEvaluator: same sampling, same (acc, cr, lat) return,
    same `.throughputs[strategy.id] = (s_enc, s_dec)` — measured on the GPU.

    Pass it as `evaluate` to run_search (search.py:174-188); `kvpilot profile`
    then stores GPU s_enc/s_dec in each Profile (cli.py:111-121).
    """

    def __init__(self, corpus, sample_size: int = 8, v_ref: float = float(2**30), timer=None, seed: int = 0,
                 reference_format: bool = False) -> None:
        """reference_format=True codes rle / entropy profiles in the reference's
        whole-tensor payload format (one block per tensor), so `cr` equals the
        reference CorpusEvaluator's; the default block-framed format (2048-symbol
        blocks, parallel decode) costs ~1% of cr at 2 bits."""
        if sample_size < 1:
            raise ValueError("sample_size must be >= 1")
        if len(corpus) < sample_size:
            raise ValueError(f"corpus has {len(corpus)} tensors, need >= {sample_size}")
        self.corpus = corpus
        self.sample_size = sample_size
        self.v_ref = v_ref
        self.timer = timer if timer is not None else CudaEventTimer()
        self.seed = seed
        self.reference_format = reference_format
        self.throughputs: dict[str, tuple[float, float]] = {}
        self.picks: dict[str, list[int]] = {}
        self._dev: dict[int, KVTensor] = {}

    def _device_tensor(self, i: int) -> KVTensor:
        t = self._dev.get(i)
        if t is None:
            src = self.corpus[i]
            dev = torch.device("cuda", torch.cuda.current_device())
            t = KVTensor(_as_device_values(src, dev), getattr(src, "head_importance", None))
            self._dev[i] = t
        return t

    def __call__(self, strategy) -> tuple[float, float, float]:
        s = as_strategy(strategy)
        sid = getattr(strategy, "id", s.id)
        rng = np.random.default_rng([self.seed, _stable_hash(sid)])
        picks = rng.choice(len(self.corpus), size=self.sample_size, replace=False)
        self.picks[sid] = [int(i) for i in picks]
        total = enc = dec = 0.0
        accs, crs = [], []
        block = None if self.reference_format else 2048
        for i in picks:
            x = self._device_tensor(int(i))
            _, m = compress(x, s, self.timer, block_symbols=block)
            accs.append(m.quality)
            crs.append(m.cr)
            total += x.nbytes_source
            enc += x.nbytes_source / m.s_enc
            dec += x.nbytes_source / m.s_dec
        s_enc, s_dec = total / enc, total / dec
        s_p = s_enc * s_dec / (s_enc + s_dec)
        self.throughputs[sid] = (s_enc, s_dec)
        return float(np.mean(accs)), float(np.mean(crs)), float(self.v_ref / s_p)
