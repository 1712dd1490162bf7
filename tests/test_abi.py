"""CPU-side checks of the C ABI: the library loads, exports every symbol
include/kvc.h declares, and plan creation validates like the reference."""

import ctypes
import os
import re

import pytest

from paper_2605_13734_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2605_13734_b200._build import build

    build()
    return N.lib()


def header_symbols():
    text = open(os.path.join(ROOT, "include", "kvc.h")).read()
    return sorted(set(re.findall(r"\b(kvc_[a-z0-9_]+)\s*\(", text)))


def test_exports_every_declared_symbol(lib):
    syms = header_symbols()
    assert set(syms) == set(N.EXPORTS)
    for s in syms:
        assert hasattr(lib, s), s


def _plan(lib, sid, shape=(2, 4, 64, 128), block=4096):
    h = ctypes.c_void_p()
    o = N.KvcOptions()
    o.block_symbols = block
    rc = lib.kvc_plan_create(ctypes.byref(h), sid.encode(), *shape, ctypes.byref(o))
    return rc, h


def test_plan_sizes(lib):
    rc, h = _plan(lib, "t=hadamard;q=uniform,b=4,g=32;c=none")
    assert rc == 0
    L, H, T, C = 2, 4, 64, 128
    assert lib.kvc_metadata_bytes(h) == 4 * L * H * T * C // 32
    assert lib.kvc_static_payload_bytes(h, None) == L * H * T * C * 4 // 8
    assert lib.kvc_plan_strategy_id(h).decode() == "t=hadamard;q=uniform,b=4,g=32;c=none"
    lib.kvc_plan_destroy(h)
    rc, h = _plan(lib, " t=identity;q=mixed,hi=8,lo=2,g=32,rho=0.25;c=entropy\n", block=512)
    assert rc == 0
    assert lib.kvc_metadata_bytes(h) == 4 * L * H * T * C // 32 + 1
    cls = (ctypes.c_uint8 * 8)(1, 0, 0, 0, 0, 0, 0, 1)
    assert lib.kvc_num_blocks(h, cls) == (2 * T * C + 511) // 512 + (6 * T * C + 511) // 512
    lib.kvc_plan_destroy(h)


@pytest.mark.parametrize("text", [
    "t=identity;q=uniform,b=4,g=32",
    "t=identity;q=uniform,b=4,g=32;c=none;extra=1",
    "t=fourier;q=uniform,b=4,g=32;c=none",
    "x=identity;q=uniform,b=4,g=32;c=none",
    "t=identity;q=uniform,b=4,g=32;c=zstd",
    "t=identity;q=vector,b=4,g=32;c=none",
    "t=identity;q=uniform,b=4;c=none",
    "t=identity;q=uniform,b=4,g=32,rho=0.5;c=none",
    "t=identity;q=mixed,hi=8,lo=2,g=32;c=none",
    "t=identity;q=uniform,b4,g=32;c=none",
    "t=identity;q=uniform,b=four,g=32;c=none",
    "t=identity;q=uniform,b=9,g=32;c=none",
    "t=identity;q=mixed,hi=2,lo=4,g=32,rho=0.25;c=none",
    "t=identity;q=mixed,hi=8,lo=2,g=32,rho=1.5;c=none",
    "t=identity;q=uniform,b=4,g=48;c=none",
])
def test_rejects_like_reference(lib, text):
    """Malformed ids from test_strategy.py:179-197 plus config validation."""
    rc, h = _plan(lib, text)
    assert rc == N.KVC_ERR_CONFIG, text
    with pytest.raises(ValueError):
        N.check(rc)


def test_hadamard_needs_power_of_two(lib):
    rc, _ = _plan(lib, "t=hadamard;q=uniform,b=4,g=16;c=none", shape=(1, 1, 2, 48))
    assert rc == N.KVC_ERR_CONFIG
    assert "power-of-two" in lib.kvc_last_error().decode()


def test_canonical_rho_repr(lib):
    rc, h = _plan(lib, "t=delta;q=mixed,hi=4,lo=3,g=64,rho=0.1250;c=rle", shape=(1, 1, 4, 64))
    assert rc == 0
    assert lib.kvc_plan_strategy_id(h).decode() == "t=delta;q=mixed,hi=4,lo=3,g=64,rho=0.125;c=rle"


def _plan_dtype(lib, sid, in_dtype, shape=(2, 4, 64, 128), block=2048):
    h = ctypes.c_void_p()
    o = N.KvcOptions()
    o.block_symbols = block
    o.in_dtype = in_dtype
    assert lib.kvc_plan_create(ctypes.byref(h), sid.encode(), *shape, ctypes.byref(o)) == N.KVC_OK
    return h


@pytest.mark.parametrize("sid,bf16_path,f32_path", [
    ("t=hadamard;q=uniform,b=4,g=32;c=none", "fast128-cert+fp64+fixup", "fast128-cert+fp64+fixup"),
    ("t=hadamard;q=uniform,b=4,g=64;c=none", "fast128-cert+fp64+fixup", "fast128-cert+fp64+fixup"),
    ("t=identity;q=uniform,b=2,g=32;c=entropy", "fused_rc", "fast128"),
    ("t=identity;q=uchan,b=2,g=32;c=entropy", "fused_rc", "generic"),
    ("t=identity;q=uchan,b=2,g=32;c=none", "uchan128", "generic"),
    ("t=delta;q=uniform,b=4,g=16;c=none", "generic: no fused kernel for this group / layout", "generic"),
])
def test_plan_reports_its_kernel_path(lib, sid, bf16_path, f32_path):
    """kvc_plan_encode_path names the kernel family (the generic fallbacks
    are visible, and KVCodec warns about them)."""
    shape = (1, 2, 2048, 128)  # per-channel groups tile 128 tokens, fused blocks 2048
    h = _plan_dtype(lib, sid, N.DTYPE_BF16, shape)
    assert lib.kvc_plan_encode_path(h).decode() == bf16_path
    lib.kvc_plan_destroy(h)
    h = _plan_dtype(lib, sid, N.DTYPE_F32, shape)
    assert lib.kvc_plan_encode_path(h).decode().startswith(f32_path)
    lib.kvc_plan_destroy(h)


def test_rle_block_covering_the_tensor_is_one_block(lib):
    """block_symbols >= L*H*T*C with rle: one block over the concatenated
    width streams (the reference's whole-tensor rle, codecs.py:358-360)."""
    shape = (2, 4, 64, 128)
    E = 2 * 4 * 64 * 128
    h = _plan_dtype(lib, "t=identity;q=mixed,hi=8,lo=2,g=32,rho=0.25;c=rle", N.DTYPE_BF16, shape, block=E)
    cls = (ctypes.c_uint8 * 8)(1, 0, 0, 1, 0, 0, 0, 0)
    assert lib.kvc_num_blocks(h, cls) == 1
    lib.kvc_plan_destroy(h)
    h = _plan_dtype(lib, "t=identity;q=mixed,hi=8,lo=2,g=32,rho=0.25;c=rle", N.DTYPE_BF16, shape, block=E // 2)
    assert lib.kvc_num_blocks(h, cls) > 1
    lib.kvc_plan_destroy(h)
