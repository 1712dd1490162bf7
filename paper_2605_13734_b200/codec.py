"""Device-resident codec: one plan per (strategy id, KV shape).

This is the batched / serving-side API.  Inputs and outputs stay in HBM;
nothing synchronises except ``DeviceBlob.payload_nbytes`` for the
data-dependent codecs and ``KVCodec.check``.

    codec = KVCodec("t=hadamard;q=uniform,b=4,g=32;c=none", (32, 8, 4096, 128))
    blob = codec.encode(kv_bf16_cuda)           # (L,H,T,C) bf16 on cuda
    kv2 = codec.decode(blob)                    # bf16 (L,H,T,C)
"""

from __future__ import annotations

import ctypes
import warnings
from dataclasses import dataclass, field

import numpy as np
import torch

from paper_2605_13734_b200 import _native as N

__all__ = ["KVCodec", "DeviceBlob"]


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _stream_handle(stream: torch.cuda.Stream | None, device: torch.device | None = None) -> int | None:
    s = stream if stream is not None else torch.cuda.current_stream(device)
    return s.cuda_stream or None


@dataclass
class DeviceBlob:
    """Compressed KV in device memory (GPU counterpart of the reference's
    CompressedBlob, codecs.py:41-71)."""

    payload: torch.Tensor  # uint8, capacity-sized; valid prefix = payload_nbytes
    metadata: torch.Tensor  # uint8, exactly the metadata bytes
    offsets: torch.Tensor | None  # int64 (max_blocks + 1); block_offsets for rle/entropy
    strategy_id: str
    shape: tuple
    head_classes: np.ndarray | None = None
    nblocks: int = 0
    _nbytes: int | None = field(default=None, repr=False)

    @property
    def original_bytes(self) -> int:
        L, H, T, C = self.shape
        return L * H * T * C * 2  # declared 16-bit source width (tensors.py:16, :69-72)

    def refresh(self) -> None:
        """Forget the cached payload length: call after a CUDA-graph replay
        (or any encode enqueued outside encode()) re-filled this blob."""
        if self.offsets is not None:
            self._nbytes = None

    def payload_nbytes(self) -> int:
        """Payload length; syncs once for data-dependent codecs."""
        if self._nbytes is None:
            self._nbytes = int(self.offsets[self.nblocks].item())
        return self._nbytes

    @property
    def framing_nbytes(self) -> int:
        """Block table bytes on the wire (u32 per block; 0 for codec none)."""
        return 4 * self.nblocks

    @property
    def compressed_nbytes(self) -> int:
        return self.payload_nbytes() + self.metadata.numel()

    @property
    def cr(self) -> float:
        """Reference accounting: original / (payload + metadata) (codecs.py:69-71)."""
        return self.original_bytes / self.compressed_nbytes

    @property
    def cr_wire(self) -> float:
        """Including the block offset table needed for parallel decode."""
        return self.original_bytes / (self.compressed_nbytes + self.framing_nbytes)

    def payload_bytes(self) -> bytes:
        return bytes(self.payload[: self.payload_nbytes()].cpu().numpy().tobytes())

    def metadata_bytes(self) -> bytes:
        return bytes(self.metadata.cpu().numpy().tobytes())

    def offsets_array(self) -> np.ndarray | None:
        if self.offsets is None:
            return None
        return self.offsets[: self.nblocks + 1].cpu().numpy().astype(np.int64)


_WARNED: set = set()


def _warn_generic(sid: str, side: str, path: str) -> None:
    key = (sid, side, path)
    if key not in _WARNED:
        _WARNED.add(key)
        warnings.warn(f"{sid}: {side} runs the {path}", N.GenericKernelWarning, stacklevel=3)


class KVCodec:
    """A compiled plan (kvc_plan) plus its device workspace.

    The workspace holds one operation's scratch and status word: calls on
    one KVCodec are ordered on their streams, and operations that must run
    concurrently (K and V on two streams) use one KVCodec each."""

    def __init__(
        self,
        strategy_id: str,
        shape,
        in_dtype: torch.dtype = torch.bfloat16,
        out_dtype: torch.dtype = torch.bfloat16,
        block_symbols: int = 2048,
        device: torch.device | str | int | None = None,
    ) -> None:
        L, H, T, C = (int(v) for v in shape)
        self.shape = (L, H, T, C)
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.in_dtype = in_dtype
        self.out_dtype = out_dtype
        self.block_symbols = int(block_symbols)
        opts = N.KvcOptions()
        opts.block_symbols = int(block_symbols)
        opts.in_dtype = N.DTYPE_BF16 if in_dtype == torch.bfloat16 else N.DTYPE_F32
        opts.out_dtype = N.DTYPE_BF16 if out_dtype == torch.bfloat16 else N.DTYPE_F32
        if in_dtype not in (torch.bfloat16, torch.float32) or out_dtype not in (torch.bfloat16, torch.float32):
            raise ValueError("dtypes must be bfloat16 or float32")
        lib = N.lib()
        handle = ctypes.c_void_p()
        sid = strategy_id.strip() if isinstance(strategy_id, str) else str(strategy_id)
        # the plan (SM count, range-coder tables) belongs to self.device
        with torch.cuda.device(self.device):
            N.check(lib.kvc_plan_create(ctypes.byref(handle), sid.encode(), L, H, T, C, ctypes.byref(opts)))
        self._h = handle
        self._lib = lib
        self.strategy_id = lib.kvc_plan_strategy_id(handle).decode()
        self.encode_path = lib.kvc_plan_encode_path(handle).decode()
        self.decode_path = lib.kvc_plan_decode_path(handle).decode()
        for side, path in (("encode", self.encode_path), ("decode", self.decode_path)):
            if path.startswith("generic") and C == 128:
                _warn_generic(self.strategy_id, side, path)
        self.metadata_bytes = int(lib.kvc_metadata_bytes(handle))
        self.payload_capacity = int(lib.kvc_payload_capacity(handle))
        self.max_blocks = int(lib.kvc_max_blocks(handle))
        self.codec_kind = sid.split(";")[2].split("=")[1].strip()
        self.quant_kind = sid.split(";")[1].split("=", 1)[1].split(",")[0]
        with torch.cuda.device(self.device):
            self.workspace = torch.zeros(int(lib.kvc_workspace_bytes(handle)), dtype=torch.uint8, device=self.device)

    def __del__(self) -> None:
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._lib.kvc_plan_destroy(h)
            self._h = None

    # ------------------------------------------------------------ helpers
    @property
    def needs_classes(self) -> bool:
        return self.quant_kind in ("mixed", "mixlayer")

    def _classes_arg(self, head_classes):
        if not self.needs_classes:
            return None, None
        if head_classes is None:
            raise ValueError("mixed_head quantization needs head labels from classify_heads")
        arr = np.ascontiguousarray(np.asarray(head_classes, dtype=bool).reshape(-1).astype(np.uint8))
        L, H = self.shape[:2]
        if arr.size != L * H:
            raise ValueError(f"head labels shape does not match heads {(L, H)}")
        return arr, arr.ctypes.data_as(ctypes.c_void_p)

    def alloc_blob(self, head_classes=None) -> DeviceBlob:
        """Pre-allocate output buffers (reuse across encode calls)."""
        dev = self.device
        payload = torch.empty(max(self.payload_capacity, 1), dtype=torch.uint8, device=dev)
        meta = torch.empty(max(self.metadata_bytes, 1), dtype=torch.uint8, device=dev)[: self.metadata_bytes]
        offsets = None
        if self.codec_kind != "none":
            offsets = torch.zeros(self.max_blocks + 1, dtype=torch.int64, device=dev)
        cls = None if head_classes is None else np.asarray(head_classes, dtype=bool).reshape(self.shape[:2])
        return DeviceBlob(payload, meta, offsets, self.strategy_id, self.shape, cls)

    def num_blocks(self, blob: DeviceBlob | None = None, head_classes=None) -> int:
        """Codec blocks of an encode with these head labels (0 for c=none)."""
        cls = head_classes if head_classes is not None else (None if blob is None else blob.head_classes)
        if self.needs_classes and cls is None:
            raise ValueError("mixed_head quantization needs head labels to count blocks")
        arr, cptr = self._classes_arg(cls) if self.needs_classes else (None, None)
        n = int(self._lib.kvc_num_blocks(self._h, cptr))
        del arr
        return n

    # ------------------------------------------------------------- encode
    def encode(self, kv: torch.Tensor, head_classes=None, out: DeviceBlob | None = None,
               stream: torch.cuda.Stream | None = None) -> DeviceBlob:
        if tuple(kv.shape) != self.shape:
            raise ValueError(f"kv shape {tuple(kv.shape)} != plan shape {self.shape}")
        if kv.dtype != self.in_dtype or not kv.is_cuda or not kv.is_contiguous():
            raise ValueError(f"kv must be a contiguous {self.in_dtype} CUDA tensor")
        arr, cptr = self._classes_arg(head_classes)
        blob = out if out is not None else self.alloc_blob(arr)
        if arr is not None:
            blob.head_classes = arr.astype(bool).reshape(self.shape[:2])
        with torch.cuda.device(self.device):
            N.check(
                self._lib.kvc_encode(
                    self._h, kv.data_ptr(), cptr, blob.payload.data_ptr(), blob.metadata.data_ptr() if self.metadata_bytes else blob.payload.data_ptr(),
                    _ptr(blob.offsets), self.workspace.data_ptr(), _stream_handle(stream, self.device),
                )
            )
        if self.codec_kind == "none":
            blob._nbytes = int(self._lib.kvc_static_payload_bytes(self._h, cptr))
            blob.nblocks = 0
        else:
            blob._nbytes = None
            blob.nblocks = int(self._lib.kvc_num_blocks(self._h, cptr))
        return blob

    def encode_paged(self, pages: torch.Tensor, block_table: torch.Tensor, page_tokens: int, layer_stride: int,
                     head_classes=None, out: DeviceBlob | None = None,
                     stream: torch.cuda.Stream | None = None) -> DeviceBlob:
        """Encode straight from a paged cache (vLLM layout [pages, page_tokens,
        H, C] per layer, the layout decode_paged writes): the blob is
        byte-identical to encode() of the gathered (L,H,T,C) tensor."""
        if pages.dtype != self.in_dtype or not pages.is_cuda or not pages.is_contiguous():
            raise ValueError(f"pages must be a contiguous {self.in_dtype} CUDA tensor")
        L, H, T, C = self.shape
        if page_tokens < 1 or layer_stride < 0:
            raise ValueError("page_tokens must be >= 1 and layer_stride >= 0")
        if pages.numel() < L * layer_stride or layer_stride < page_tokens * H * C:
            raise ValueError("page pool smaller than layers x layer_stride, or layer_stride below one page")
        need = -(-T // page_tokens)
        bt = block_table
        if bt.device != self.device or bt.dtype != torch.int32 or not bt.is_contiguous():
            bt = block_table.to(device=self.device, dtype=torch.int32).contiguous()
            if stream is not None:  # the copy was made on the current stream: order and keep it
                stream.wait_stream(torch.cuda.current_stream(self.device))
                bt.record_stream(stream)
        if bt.numel() < need:
            raise ValueError(f"block_table has {bt.numel()} entries, {need} needed for {T} tokens")
        # the fused kernels' paged-input conditions (fast128.cu paged_input_ok;
        # the per-channel TMA kernel reads contiguous input only)
        why = None
        if self.encode_path.startswith("fast128"):
            P = int(page_tokens)
            tiles = P >= 4 and (64 % P == 0 if P < 64 else P % 64 == 0)
            if not (self.in_dtype == torch.bfloat16 and T % 64 == 0 and tiles and layer_stride % (H * 128) == 0
                    and pages.data_ptr() % 16 == 0):
                why = "generic: paged input needs bf16, whole 64-token tiles and page runs that tile 64 tokens"
        elif self.encode_path == "uchan128":
            why = "generic: the per-channel kernel reads contiguous input"
        if why:
            _warn_generic(self.strategy_id, "paged encode", why)
        arr, cptr = self._classes_arg(head_classes)
        blob = out if out is not None else self.alloc_blob(arr)
        if arr is not None:
            blob.head_classes = arr.astype(bool).reshape(self.shape[:2])
        with torch.cuda.device(self.device):
            N.check(
                self._lib.kvc_encode_paged(
                    self._h, pages.data_ptr(), bt.data_ptr(), int(page_tokens), int(layer_stride), cptr,
                    blob.payload.data_ptr(), blob.metadata.data_ptr() if self.metadata_bytes else blob.payload.data_ptr(),
                    _ptr(blob.offsets), self.workspace.data_ptr(), _stream_handle(stream, self.device),
                )
            )
        if self.codec_kind == "none":
            blob._nbytes = int(self._lib.kvc_static_payload_bytes(self._h, cptr))
            blob.nblocks = 0
        else:
            blob._nbytes = None
            blob.nblocks = int(self._lib.kvc_num_blocks(self._h, cptr))
        return blob

    # ------------------------------------------------------------- decode
    def decode(self, blob: DeviceBlob, out: torch.Tensor | None = None,
               stream: torch.cuda.Stream | None = None, device_length: bool = False) -> torch.Tensor:
        """Decode a blob.  device_length=True takes the payload length from the
        device offset table (no host sync; for device-resident blobs)."""
        if out is None:
            out = torch.empty(self.shape, dtype=self.out_dtype, device=self.device)
        if out.dtype != self.out_dtype or tuple(out.shape) != self.shape or not out.is_contiguous():
            raise ValueError("bad output tensor")
        if blob.metadata.numel() != self.metadata_bytes:
            raise N.CodecError(f"metadata is {blob.metadata.numel()} bytes, expected {self.metadata_bytes}")
        nbytes = -1 if (device_length and blob.offsets is not None) else blob.payload_nbytes()
        with torch.cuda.device(self.device):
            N.check(
                self._lib.kvc_decode(
                    self._h, blob.payload.data_ptr(), nbytes, blob.metadata.data_ptr(), _ptr(blob.offsets),
                    out.data_ptr(), self.workspace.data_ptr(), _stream_handle(stream, self.device),
                )
            )
        return out

    def decode_paged(self, blob: DeviceBlob, pages: torch.Tensor, block_table: torch.Tensor, page_tokens: int,
                     layer_stride: int, stream: torch.cuda.Stream | None = None,
                     device_length: bool = False) -> torch.Tensor:
        """Decode into a paged cache (vLLM layout [pages, page_tokens, H, C] per
        layer).  device_length=True: payload length from the device offset
        table (no host sync)."""
        if pages.dtype != self.out_dtype:
            raise ValueError("page dtype must match the plan's out_dtype")
        L, H, T, C = self.shape
        if page_tokens < 1 or layer_stride < page_tokens * H * C or pages.numel() < L * layer_stride:
            raise ValueError("page pool smaller than layers x layer_stride, or layer_stride below one page")
        if not pages.is_cuda or not pages.is_contiguous():
            raise ValueError("pages must be a contiguous CUDA tensor")
        if block_table.numel() < -(-T // page_tokens):
            raise ValueError(f"block_table has {block_table.numel()} entries, {-(-T // page_tokens)} needed")
        if blob.metadata.numel() != self.metadata_bytes:
            raise N.CodecError(f"metadata is {blob.metadata.numel()} bytes, expected {self.metadata_bytes}")
        bt = block_table
        if bt.device != self.device or bt.dtype != torch.int32 or not bt.is_contiguous():
            bt = block_table.to(device=self.device, dtype=torch.int32).contiguous()
            if stream is not None:  # the copy was made on the current stream: order and keep it
                stream.wait_stream(torch.cuda.current_stream(self.device))
                bt.record_stream(stream)
        nbytes = -1 if (device_length and blob.offsets is not None) else blob.payload_nbytes()
        with torch.cuda.device(self.device):
            N.check(
                self._lib.kvc_decode_paged(
                    self._h, blob.payload.data_ptr(), nbytes, blob.metadata.data_ptr(), _ptr(blob.offsets),
                    pages.data_ptr(), bt.data_ptr(), int(page_tokens), int(layer_stride), self.workspace.data_ptr(),
                    _stream_handle(stream, self.device),
                )
            )
        return pages

    def check(self, stream: torch.cuda.Stream | None = None, decoding: bool = False) -> int:
        """Synchronise and raise ValueError / CodecError for device-side errors."""
        flags = ctypes.c_uint32(0)
        with torch.cuda.device(self.device):
            N.check(self._lib.kvc_read_status(self._h, self.workspace.data_ptr(), _stream_handle(stream, self.device), ctypes.byref(flags)))
        N.raise_for_flags(int(flags.value), decoding)
        return int(flags.value)
