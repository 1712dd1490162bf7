"""B200-native KV-cache compression codec (KVServe's codec hot path).

Host-side mirror of the reference pipeline API (kvpilot.pipeline) backed by
hand-written sm_100a CUDA kernels in libkvc.so (include/kvc.h).  There is no
CPU fallback: without the built library the codec raises on first use.
"""

__version__ = "0.1.0"

from paper_2605_13734_b200.codec import DeviceBlob, KVCodec  # noqa: E402

__all__ = ["KVCodec", "DeviceBlob"]
