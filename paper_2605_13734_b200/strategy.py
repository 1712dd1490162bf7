"""Strategy identity: the reference's strategy/profile API, unchanged.

Mirrors kvpilot.pipeline.strategy / transforms / quantize / codecs configs
(strategy.py:8-127, transforms.py:25-30, quantize.py:26-62, codecs.py:32-38):
same class names, fields, canonical ids, validation and ValueError messages,
so strategy ids from a profile store select a GPU plan with no call-site
change.  Extension kinds use new tokens and never change the
meaning of a reference id:

    t=affine                         per-channel shift/scale transform
    q=uchan,b=B,g=G                  per-channel (KIVI-K) groups of G tokens
    q=mixlayer,hi,lo,g,rho           mixed precision by layer
    q=mixtok,hi,lo,g,rho             mixed precision by token (recent window)
"""

from __future__ import annotations

from dataclasses import dataclass

__all__ = [
    "TransformConfig",
    "QuantConfig",
    "CodecConfig",
    "StrategyConfig",
    "parse_strategy_id",
    "analytic_cr",
    "as_strategy",
]

TRANSFORM_KINDS = ("identity", "delta_over_tokens", "hadamard_over_channels", "affine_per_channel")
QUANT_KINDS = ("uniform_group", "mixed_head", "uniform_channel", "mixed_layer", "mixed_token")
CODEC_KINDS = ("none", "rle_bitpack", "entropy")

_T_TOK = {
    "identity": "identity",
    "delta_over_tokens": "delta",
    "hadamard_over_channels": "hadamard",
    "affine_per_channel": "affine",
}
_C_TOK = {"none": "none", "rle_bitpack": "rle", "entropy": "entropy"}
_Q_TOK = {"uniform_group": "uniform", "mixed_head": "mixed", "uniform_channel": "uchan",
          "mixed_layer": "mixlayer", "mixed_token": "mixtok"}
_T_KIND = {v: k for k, v in _T_TOK.items()}
_C_KIND = {v: k for k, v in _C_TOK.items()}
_Q_KIND = {v: k for k, v in _Q_TOK.items()}
_MIXED = ("mixed_head", "mixed_layer", "mixed_token")


@dataclass(frozen=True)
class TransformConfig:
    kind: str = "identity"

    def __post_init__(self) -> None:
        if self.kind not in TRANSFORM_KINDS:
            raise ValueError(f"unknown transform kind {self.kind!r}; expected one of {TRANSFORM_KINDS}")


@dataclass(frozen=True)
class QuantConfig:
    """Quantizer knobs; unused knobs are pinned so equality is semantic."""

    kind: str = "uniform_group"
    bits: int = 4
    group_size: int = 32
    high_bits: int = 8
    low_bits: int = 2
    retrieval_fraction: float = 0.25

    def __post_init__(self) -> None:
        if self.kind not in QUANT_KINDS:
            raise ValueError(f"unknown quant kind {self.kind!r}; expected one of {QUANT_KINDS}")
        if self.group_size < 1:
            raise ValueError(f"group_size must be >= 1, got {self.group_size}")
        if self.kind in ("uniform_group", "uniform_channel"):
            if not 1 <= self.bits <= 8:
                raise ValueError(f"bits must be in 1..8, got {self.bits}")
            object.__setattr__(self, "high_bits", 8)
            object.__setattr__(self, "low_bits", 2)
            object.__setattr__(self, "retrieval_fraction", 0.25)
        else:
            for name in ("high_bits", "low_bits"):
                value = getattr(self, name)
                if not 1 <= value <= 8:
                    raise ValueError(f"{name} must be in 1..8, got {value}")
            if self.high_bits <= self.low_bits:
                raise ValueError(f"high_bits must exceed low_bits, got {self.high_bits} <= {self.low_bits}")
            if not 0.0 <= self.retrieval_fraction <= 1.0:
                raise ValueError(f"retrieval_fraction must be in [0, 1], got {self.retrieval_fraction}")
            object.__setattr__(self, "bits", 4)


@dataclass(frozen=True)
class CodecConfig:
    kind: str = "none"

    def __post_init__(self) -> None:
        if self.kind not in CODEC_KINDS:
            raise ValueError(f"unknown codec kind {self.kind!r}; expected one of {CODEC_KINDS}")


@dataclass(frozen=True)
class StrategyConfig:
    transform: TransformConfig
    quant: QuantConfig
    codec: CodecConfig

    @property
    def id(self) -> str:
        q = self.quant
        tok = _Q_TOK[q.kind]
        if q.kind in _MIXED:
            quant = f"{tok},hi={q.high_bits},lo={q.low_bits},g={q.group_size},rho={q.retrieval_fraction!r}"
        else:
            quant = f"{tok},b={q.bits},g={q.group_size}"
        return f"t={_T_TOK[self.transform.kind]};q={quant};c={_C_TOK[self.codec.kind]}"

    def __str__(self) -> str:
        return self.id


def _kv(token: str, segment: str):
    if "=" not in token:
        raise ValueError(f"malformed token {token!r} in strategy id segment {segment!r}")
    k, _, v = token.partition("=")
    return k, v


def parse_strategy_id(text: str) -> StrategyConfig:
    """Parse an id; raises ValueError on any deviation from the grammar."""
    segs = text.strip().split(";")
    if len(segs) != 3:
        raise ValueError(f"strategy id must have 3 ';'-separated segments, got {len(segs)}: {text!r}")
    k, v = _kv(segs[0], segs[0])
    if k != "t" or v not in _T_KIND:
        raise ValueError(f"bad transform segment {segs[0]!r}")
    transform = TransformConfig(kind=_T_KIND[v])
    k, v = _kv(segs[1], segs[1])
    if k != "q":
        raise ValueError(f"bad quant segment {segs[1]!r}")
    parts = v.split(",")
    kind_tok = parts[0]
    params = dict(_kv(p, segs[1]) for p in parts[1:])
    if kind_tok not in _Q_KIND:
        raise ValueError(f"unknown quant kind {kind_tok!r} in {segs[1]!r}")
    kind = _Q_KIND[kind_tok]
    if kind in _MIXED:
        if set(params) != {"hi", "lo", "g", "rho"}:
            raise ValueError(f"{kind_tok} quant needs exactly hi, lo, g, rho, got {sorted(params)} in {segs[1]!r}")
        quant = QuantConfig(kind=kind, high_bits=int(params["hi"]), low_bits=int(params["lo"]),
                            group_size=int(params["g"]), retrieval_fraction=float(params["rho"]))
    else:
        if set(params) != {"b", "g"}:
            raise ValueError(f"{kind_tok} quant needs exactly b and g, got {sorted(params)} in {segs[1]!r}")
        quant = QuantConfig(kind=kind, bits=int(params["b"]), group_size=int(params["g"]))
    k, v = _kv(segs[2], segs[2])
    if k != "c" or v not in _C_KIND:
        raise ValueError(f"bad codec segment {segs[2]!r}")
    return StrategyConfig(transform=transform, quant=quant, codec=CodecConfig(kind=_C_KIND[v]))


def analytic_cr(strategy) -> float:
    """16 / (b_eff + 32 / g) (strategy.py:112-127), codec-agnostic."""
    q = as_strategy(strategy).quant
    if q.kind in _MIXED:
        b_eff = q.retrieval_fraction * q.high_bits + (1.0 - q.retrieval_fraction) * q.low_bits
    else:
        b_eff = float(q.bits)
    return 16.0 / (b_eff + 32.0 / q.group_size)


def as_strategy(s) -> StrategyConfig:
    """Accept our StrategyConfig, the reference's (duck-typed via .id), or an id string."""
    if isinstance(s, StrategyConfig):
        return s
    if isinstance(s, str):
        return parse_strategy_id(s)
    sid = getattr(s, "id", None)
    if isinstance(sid, str):
        return parse_strategy_id(sid)
    raise TypeError(f"not a strategy: {s!r}")
