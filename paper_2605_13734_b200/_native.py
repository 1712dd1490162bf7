"""ctypes binding of libkvc.so (the C ABI declared in include/kvc.h).

The product path has no CPU fallback: if the library is missing or fails to
load, importing the codec raises immediately.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libkvc.so")

KVC_OK, KVC_ERR_CONFIG, KVC_ERR_CODEC, KVC_ERR_CUDA, KVC_ERR_VALUE = 0, 1, 2, 3, 4
DTYPE_BF16, DTYPE_F32 = 0, 1
FLAG_NONFINITE_INPUT = 1
FLAG_NONFINITE_TRANSFORM = 2
FLAG_CODEC = 4
FLAG_CAPACITY = 8
FLAG_FP16_RANGE = 16

# every symbol include/kvc.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "kvc_plan_create",
    "kvc_plan_destroy",
    "kvc_plan_strategy_id",
    "kvc_plan_encode_path",
    "kvc_plan_decode_path",
    "kvc_metadata_bytes",
    "kvc_payload_capacity",
    "kvc_workspace_bytes",
    "kvc_max_blocks",
    "kvc_static_payload_bytes",
    "kvc_num_blocks",
    "kvc_encode",
    "kvc_encode_paged",
    "kvc_decode",
    "kvc_decode_paged",
    "kvc_read_status",
    "kvc_last_error",
    "kvc_version",
    "kvc_profile_enable",
    "kvc_profile_collect",
    "kvc_block_crc32",
    "kvc_copy_device_length",
    "kvc_enable_peer_access",
    "kvc_sq_error",
    "kvc_sq_error_partials",
)


class GenericKernelWarning(UserWarning):
    """A plan runs the generic per-element CUDA kernels (still on the GPU, but
    several times slower than the fused head_dim-128 kernels), e.g. for
    float32 input that is not bf16-exact."""


class CodecError(ValueError):
    """Malformed or mismatched payload (mirrors kvpilot's CodecError, codecs.py:28)."""


class KvcOptions(ctypes.Structure):
    _fields_ = [
        ("block_symbols", ctypes.c_int64),
        ("in_dtype", ctypes.c_int32),
        ("out_dtype", ctypes.c_int32),
        ("reserved", ctypes.c_int32 * 8),
    ]


_lib = None


def lib() -> ctypes.CDLL:
    """Load libkvc.so once; raise loudly when it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} not found: build it with `python -m paper_2605_13734_b200._build` "
            "(there is deliberately no CPU fallback)"
        )
    L = ctypes.CDLL(LIB_PATH)
    P, I64, I32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
    L.kvc_plan_create.argtypes = [ctypes.POINTER(P), ctypes.c_char_p, I64, I64, I64, I64, ctypes.POINTER(KvcOptions)]
    L.kvc_plan_create.restype = I32
    L.kvc_plan_destroy.argtypes = [P]
    L.kvc_plan_destroy.restype = I32
    L.kvc_plan_strategy_id.argtypes = [P]
    L.kvc_plan_strategy_id.restype = ctypes.c_char_p
    for name in ("kvc_plan_encode_path", "kvc_plan_decode_path"):
        getattr(L, name).argtypes = [P]
        getattr(L, name).restype = ctypes.c_char_p
    for name in ("kvc_metadata_bytes", "kvc_payload_capacity", "kvc_workspace_bytes", "kvc_max_blocks"):
        getattr(L, name).argtypes = [P]
        getattr(L, name).restype = I64
    L.kvc_static_payload_bytes.argtypes = [P, P]
    L.kvc_static_payload_bytes.restype = I64
    L.kvc_num_blocks.argtypes = [P, P]
    L.kvc_num_blocks.restype = I64
    L.kvc_encode.argtypes = [P, P, P, P, P, P, P, P]
    L.kvc_encode.restype = I32
    L.kvc_encode_paged.argtypes = [P, P, P, I64, I64, P, P, P, P, P, P]
    L.kvc_encode_paged.restype = I32
    L.kvc_decode.argtypes = [P, P, I64, P, P, P, P, P]
    L.kvc_decode.restype = I32
    L.kvc_decode_paged.argtypes = [P, P, I64, P, P, P, P, I64, I64, P, P]
    L.kvc_decode_paged.restype = I32
    L.kvc_read_status.argtypes = [P, P, P, ctypes.POINTER(ctypes.c_uint32)]
    L.kvc_read_status.restype = I32
    L.kvc_last_error.argtypes = []
    L.kvc_last_error.restype = ctypes.c_char_p
    L.kvc_version.argtypes = []
    L.kvc_version.restype = ctypes.c_char_p
    L.kvc_profile_enable.argtypes = [I32]
    L.kvc_profile_enable.restype = I32
    L.kvc_profile_collect.argtypes = [ctypes.c_char_p, I64, P, P, I32]
    L.kvc_profile_collect.restype = I32
    L.kvc_block_crc32.argtypes = [P, P, I64, P, P]
    L.kvc_block_crc32.restype = I32
    L.kvc_copy_device_length.argtypes = [P, P, P, I64, P]
    L.kvc_copy_device_length.restype = I32
    L.kvc_enable_peer_access.argtypes = [I32, I32]
    L.kvc_enable_peer_access.restype = I32
    L.kvc_sq_error.argtypes = [P, P, I64, I32, P, P]
    L.kvc_sq_error.restype = I32
    L.kvc_sq_error_partials.argtypes = [P, P, I64, I32, P, I64, P]
    L.kvc_sq_error_partials.restype = I32
    _lib = L
    return L


def check(rc: int) -> None:
    """Map a kvc_status to the reference's exception types."""
    if rc == KVC_OK:
        return
    msg = lib().kvc_last_error().decode(errors="replace")
    if rc == KVC_ERR_CODEC:
        raise CodecError(msg)
    if rc in (KVC_ERR_CONFIG, KVC_ERR_VALUE):
        raise ValueError(msg)
    raise RuntimeError(f"CUDA error: {msg}")


def raise_for_flags(flags: int, decoding: bool) -> None:
    """Device status word -> the reference's exceptions."""
    if flags & (FLAG_CODEC | FLAG_CAPACITY):
        raise CodecError(f"malformed payload (device status 0x{flags:x})")
    if flags & FLAG_NONFINITE_INPUT:
        raise ValueError("values must be finite")
    if flags & FLAG_NONFINITE_TRANSFORM:
        raise ValueError("values must be finite")


def profile_enable(on: bool) -> None:
    lib().kvc_profile_enable(1 if on else 0)


def profile_collect() -> dict:
    """{kernel name: (total ms, launches)} since the last collect (syncs)."""
    import numpy as np

    cap = 64
    names = ctypes.create_string_buffer(4096)
    ms = np.zeros(cap, dtype=np.float64)
    cnt = np.zeros(cap, dtype=np.int64)
    n = lib().kvc_profile_collect(names, 4096, ms.ctypes.data_as(ctypes.c_void_p), cnt.ctypes.data_as(ctypes.c_void_p), cap)
    keys = names.raw.split(b"\0")[:n]
    return {k.decode(): (float(ms[i]), int(cnt[i])) for i, k in enumerate(keys)}
