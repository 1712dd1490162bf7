"""The certified float32 Hadamard encoder (fast128.cu: had32_row / cert_group).

The hot path of the reference default profile (transforms.py:62 then
quantize.py:142-154 at 32-channel groups) runs the butterfly in float32 and
accepts a row only when every quantizer decision is provably the one the
reference's float64 butterfly leads to; other rows go to the float64 pass.

CPU part: a numpy restatement of the certificate (same float32 butterfly,
same bound D, same interval tests) over 131,072 reference-generator rows --
every certified row must quantize exactly like the reference, and rows where
plain float32 would give different bytes must all be rejected.
GPU part: those rows (plus the certificate's near-miss rows) through the C
ABI, bit-exact against the oracle.
"""

from __future__ import annotations

import numpy as np
import pytest

import oracle

U = 2.0 ** -24
C = np.sqrt(128.0)
R32 = np.float32(1.0 / C)


def _bf16(a):
    b = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)
    b = ((b + 0x7FFF + ((b >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)
    return b.view(np.float32)


def _fwht32(x):
    """float32 butterfly in the kernel's stage order (h = 1, 2, .., 64)."""
    y = np.array(x, dtype=np.float32)
    n = y.shape[-1]
    lead = y.shape[:-1]
    h = 1
    while h < n:
        v = y.reshape(*lead, n // (2 * h), 2, h)
        a, b = v[..., 0, :], v[..., 1, :]
        y = np.concatenate([(a + b)[..., None, :], (a - b)[..., None, :]], axis=-2).reshape(*lead, n)
        h <<= 1
    return y


def _f16bits(v):
    return np.asarray(v, dtype=np.float32).astype(np.float16).view(np.uint16)


def certify(x):
    """(y_hat, certified) per row of bf16-exact x (N, 128), as cert_group."""
    N = x.shape[0]
    yh = (_fwht32(x) * R32).astype(np.float32)
    ax = np.abs(x).astype(np.float64)
    e = np.frexp(np.where(ax > 0, ax, 0.0))[1] - 1
    e = np.where(ax > 0, e, -127)
    emin = e.min(1)
    s1 = ax.sum(1)
    es1 = np.frexp(s1 * (1 + 2.0 ** -16))[1] - 1
    # every stage exact when all partial sums (< 2^(es1+1)) fit 24 bits above
    # the inputs' 2^(emin-7) grid; other rows take the gamma_7 bound
    exact = es1 <= emin + 16
    g = yh.reshape(N, 4, 32).astype(np.float64)
    mn, mx = g.min(-1), g.max(-1)
    d_sum = (9.3 * U * s1 / C * 1.002 + 2.0 ** -140)[:, None]
    ex = exact[:, None]
    dz = np.where(ex, 2.3 * U * np.abs(mn) + 2.0 ** -140, d_sum)
    dx = np.where(ex, 2.3 * U * np.abs(mx) + 2.0 ** -140, d_sum)
    D = np.maximum(dz, dx)
    dn = lambda v: np.nextafter(v.astype(np.float32), np.float32(-np.inf))  # noqa: E731
    up = lambda v: np.nextafter(v.astype(np.float32), np.float32(np.inf))  # noqa: E731
    zl, zh = _f16bits(dn(mn - dz)), _f16bits(up(mn + dz))
    dl, dh = dn(mx - mn - (dz + dx)).astype(np.float64), up(mx - mn + (dz + dx)).astype(np.float64)
    sl, sh = _f16bits(dl / 15 * (1 - 2.0 ** -22)), _f16bits(dh / 15 * (1 + 2.0 ** -22))
    ok = (zl == zh) & (sl == sh) & (dl > 0)
    s = sl.view(np.float16).astype(np.float32)
    z = zl.view(np.float16).astype(np.float32)
    with np.errstate(divide="ignore", invalid="ignore"):
        t = (g.astype(np.float32) - z[..., None]) / np.where(s > 0, s, 1)[..., None]
        tmax = np.maximum(np.abs((mn - z) / np.where(s > 0, s, 1)), np.abs((mx - z) / np.where(s > 0, s, 1)))
        tau = D / np.where(s > 0, s, np.inf) * 1.0001 + 2.0 ** -21 * (tmax + 1)
    rho = np.abs(t - np.rint(t)).max(-1)
    ok &= (rho < 0.5 - tau) | (s == 0)
    return yh, ok.all(1)


def _rows(n_layers=4):
    vals, _ = oracle.generate_kv(n_layers, 8, 4096, 128, seed=1)
    return _bf16(vals).reshape(-1, 128)


def _quant(y):
    sym, sc, zr = oracle.quantize_rows(y.reshape(1, 1, -1, 128), np.array([[4]]), 32)
    n = y.shape[0]
    return sym.reshape(n, -1), sc.reshape(n, -1).view(np.uint16), zr.reshape(n, -1).view(np.uint16)


def test_certificate_is_sound_on_reference_rows():
    x = _rows()
    yref = (oracle.fwht64(x) / C).astype(np.float32)
    yh, cert = certify(x)
    a, b = _quant(yref), _quant(yh)
    same = np.ones(x.shape[0], bool)
    for p, q in zip(a, b):
        same &= (p == q).all(1)
    # float32 alone is wrong on some rows; the certificate rejects every one
    assert (~same).sum() > 0
    assert not (cert & ~same).any()
    # and keeps the float64 pass small (2 % of rows on this distribution)
    assert cert.mean() > 0.975


def _hard_rows():
    """Rows where plain float32 bytes differ from the reference, plus the
    rejected rows closest to certification (64 rows in all)."""
    x = _rows()
    yref = (oracle.fwht64(x) / C).astype(np.float32)
    yh, cert = certify(x)
    a, b = _quant(yref), _quant(yh)
    same = np.ones(x.shape[0], bool)
    for p, q in zip(a, b):
        same &= (p == q).all(1)
    wrong = np.flatnonzero(~same)
    rejected = np.flatnonzero(~cert & same)
    take = np.concatenate([wrong, rejected[: 64 - len(wrong)], np.flatnonzero(cert)[:64]])[:128]
    return x[take], len(wrong)


@pytest.mark.gpu
@pytest.mark.parametrize("sid", ["t=hadamard;q=uniform,b=4,g=32;c=none", "t=hadamard;q=uniform,b=2,g=32;c=entropy",
                                 "t=hadamard;q=mixed,hi=8,lo=2,g=32,rho=0.5;c=none"])
def test_gpu_certified_encoder_on_hard_rows(sid):
    import torch

    from paper_2605_13734_b200 import KVCodec

    rows, nwrong = _hard_rows()
    assert nwrong > 0
    shape = (2, 1, rows.shape[0] // 2, 128)
    vb = rows.reshape(shape)
    imp = np.array([[0.9], [0.1]])
    s = oracle.parse_id(sid)
    cls = oracle.classify_heads(imp, s.rho) if s.quant == "mixed" else None
    ref = oracle.encode_blob(vb, imp, sid, block=256)
    codec = KVCodec(sid, shape, block_symbols=256)
    blob = codec.encode(torch.from_numpy(vb).to(torch.bfloat16).cuda(), head_classes=cls)
    codec.check()
    assert blob.metadata_bytes() == ref["metadata"]
    assert blob.payload_bytes() == ref["payload"]


def _stress_rows(seed, n=8192):
    """bf16 rows from distributions unlike the reference generator: heavy
    tails, integer grids (exact zero outputs, ties, degenerate groups), wide
    exponent spans, tiny / subnormal magnitudes, near-constant rows."""
    rng = np.random.default_rng(seed)
    k = n // 8
    parts = [
        rng.standard_cauchy((k, 128)).clip(-1e3, 1e3),                      # heavy tails
        rng.integers(-8, 9, (k, 128)).astype(np.float64),                   # integer grid
        rng.normal(size=(k, 128)) * 2.0 ** rng.integers(-30, 30, (k, 1)),   # row scales
        rng.normal(size=(k, 128)) * 2.0 ** rng.integers(-40, 20, (k, 128)),  # per-value exponent spread
        rng.normal(size=(k, 128)) * 1e-38,                                  # float32 subnormal range
        1.0 + rng.normal(size=(k, 128)) * 2.0 ** -9,                        # near-constant rows
        rng.uniform(-1, 1, (k, 128)) * (rng.uniform(size=(k, 128)) < 0.1),   # sparse
        rng.lognormal(0, 2, (k, 128)) * rng.choice([-1.0, 1.0], (k, 128)),  # log-normal magnitudes
    ]
    x = np.concatenate(parts).astype(np.float32)
    return _bf16(x)[rng.permutation(len(x))]


def test_certificate_is_sound_on_stress_rows():
    x = _stress_rows(7)
    yref = (oracle.fwht64(x) / C).astype(np.float32)
    yh, cert = certify(x)
    with np.errstate(all="ignore"):
        a, b = _quant(yref), _quant(yh)
    same = np.ones(x.shape[0], bool)
    for p, q in zip(a, b):
        same &= (p == q).all(1)
    assert not (cert & ~same).any()


@pytest.mark.gpu
@pytest.mark.parametrize("seed,sid", [(1, "t=hadamard;q=uniform,b=4,g=32;c=none"),
                                      (2, "t=hadamard;q=uniform,b=4,g=32;c=none"),
                                      (3, "t=hadamard;q=uniform,b=2,g=64;c=none"),
                                      (4, "t=hadamard;q=uniform,b=8,g=128;c=none"),
                                      (5, "t=hadamard;q=uniform,b=3,g=64;c=entropy")])
def test_gpu_certified_encoder_on_stress_rows(seed, sid):
    import torch

    from paper_2605_13734_b200 import KVCodec

    rows = _stress_rows(seed)
    shape = (4, 2, rows.shape[0] // 8, 128)
    vb = rows.reshape(shape)
    with np.errstate(all="ignore"):
        ref = oracle.encode_blob(vb, None, sid, block=256)
    codec = KVCodec(sid, shape, block_symbols=256)
    blob = codec.encode(torch.from_numpy(vb).to(torch.bfloat16).cuda())
    codec.check()
    assert blob.metadata_bytes() == ref["metadata"]
    assert blob.payload_bytes() == ref["payload"]


@pytest.mark.gpu
@pytest.mark.parametrize("sid", ["t=hadamard;q=uniform,b=4,g=32;c=none", "t=hadamard;q=uniform,b=2,g=128;c=entropy"])
def test_gpu_certified_encoder_float32_input(sid):
    """float32 inputs (the reference's own corpora, tensors.py:79-112): no
    exact-butterfly shortcut, every row on the gamma_7 bound; reference
    generator rows plus the stress rows, bit-exact against the oracle."""
    import torch

    from paper_2605_13734_b200 import KVCodec

    vals, _ = oracle.generate_kv(2, 4, 1024, 128, seed=11)
    rows = np.concatenate([vals.reshape(-1, 128), _stress_rows(12, 4096) * np.float32(1.0 + 2.0 ** -12)])
    shape = (4, 2, rows.shape[0] // 8, 128)
    vb = np.ascontiguousarray(rows.reshape(shape), dtype=np.float32)
    with np.errstate(all="ignore"):
        ref = oracle.encode_blob(vb, None, sid, block=256)
    codec = KVCodec(sid, shape, in_dtype=torch.float32, block_symbols=256)
    blob = codec.encode(torch.from_numpy(vb).cuda())
    codec.check()
    assert codec.encode_path == "fast128-cert+fp64+fixup"
    assert blob.metadata_bytes() == ref["metadata"]
    assert blob.payload_bytes() == ref["payload"]
