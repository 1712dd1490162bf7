"""B200-native KV-cache compression codec (KVServe's codec hot path).

Host-side mirror of the reference pipeline API (kvpilot.pipeline) backed by
hand-written sm_100a CUDA kernels in libkvc.so (include/kvc.h).  There is no
CPU fallback: without the built library the codec raises on first use.

    from paper_2605_13734_b200 import compress, decompress, parse_strategy_id
    blob, metrics = compress(kv, parse_strategy_id("t=hadamard;q=uniform,b=4,g=32;c=none"))
"""

__version__ = "0.1.0"

from paper_2605_13734_b200.strategy import (  # noqa: E402
    CodecConfig,
    QuantConfig,
    StrategyConfig,
    TransformConfig,
    analytic_cr,
    parse_strategy_id,
)
from paper_2605_13734_b200.codec import DeviceBlob, KVCodec  # noqa: E402

__all__ = [
    "CodecConfig",
    "QuantConfig",
    "StrategyConfig",
    "TransformConfig",
    "analytic_cr",
    "parse_strategy_id",
    "KVCodec",
    "DeviceBlob",
    # pipeline API (lazy: needs torch + CUDA)
    "KVTensor",
    "CompressedBlob",
    "PipelineMetrics",
    "WallClockTimer",
    "CostModelTimer",
    "CudaEventTimer",
    "CodecError",
    "classify_heads",
    "quality_score",
    "compress",
    "decompress",
    "GpuCorpusEvaluator",
]


def __getattr__(name):
    if name in __all__:
        from paper_2605_13734_b200 import pipeline

        return getattr(pipeline, name)
    raise AttributeError(name)
