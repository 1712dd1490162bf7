"""Byte parity at the benchmarked sizes (BASELINE.json configs c2, c3, c5).

The parity suite (test_gpu_parity.py) pins every strategy on small tensors;
this file encodes the FULL benchmark tensors on the GPU -- c2 (1.07 G
elements per tensor), c3 (10.5 G elements, a 5.2 GB payload whose byte
offsets cross 2^32) and c5 -- and checks sampled (layer, head) slabs byte for
byte against the oracle (the CPU restatement of the reference) run on the
same slab:

  * c=none: slab payload = bytes [(l*H+h)*T*C*w/8, +T*C*w/8) of the packed
    stream (codecs.py:79-87, :339-345), scales / zeros = the slab's groups of
    the global arrays (quantize.py:142-147, codecs.py:348-352);
  * c=entropy: T*C is a multiple of the 2048-symbol block, so the slab's
    blocks start at block (l*H+h)*T*C/2048; their bytes and lengths must equal
    the oracle's blocks of the slab (codecs.py:310-317, :361-366 per block);
  * per-channel (uchan) K: the slab is the head's (C, T) transpose, groups
    and blocks along tokens;
  * affine (c5): the slab's mu / a rows of the appended metadata.

Then the decoded bf16 slab equals bf16(oracle decode) -- exactly for
identity and affine; for the fp32 inverse Hadamard within the reference's
transform tolerance (1e-5 of the row magnitude) plus one bf16 rounding -- and
c5's paged decode equals its contiguous decode.  Slabs include (0, 0) and the
last (l, h) (for c3 its payload starts beyond 2^32 bytes).
"""

from __future__ import annotations

import concurrent.futures as cf
import multiprocessing as mp
import os

import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

BLOCK = 2048
C1 = "t=hadamard;q=uniform,b=4,g=32;c=none"
CASES = {
    "c2-K-uchan-entropy": ((32, 8, 32768, 128), "t=identity;q=uchan,b=2,g=32;c=entropy"),
    "c2-V-uniform-entropy": ((32, 8, 32768, 128), "t=identity;q=uniform,b=2,g=32;c=entropy"),
    "c3-hadamard-none": ((80, 8, 128000, 128), C1),
    "c5-affine-b8-entropy": ((36, 8, 16384, 128), "t=affine;q=uniform,b=8,g=32;c=entropy"),
}
N_SLABS = 16

_JOBS: list = []


def _oracle_job(i):
    sid, v = _JOBS[i]
    ob = oracle.encode_blob(v, None, sid, block=BLOCK)
    rec = oracle.decode_blob(ob["payload"], ob["metadata"], ob["offsets"], sid, v.shape, block=BLOCK)
    return ob["payload"], ob["metadata"], ob["offsets"], rec


def _run_oracle(jobs):
    """Oracle encode + decode of each (sid, slab) on the host cores (the
    slabs are handed to forked workers through a module global)."""
    _JOBS[:] = jobs
    try:
        procs = max(1, min(len(jobs), len(os.sched_getaffinity(0))))
        with cf.ProcessPoolExecutor(procs, mp_context=mp.get_context("fork")) as ex:
            return list(ex.map(_oracle_job, range(len(jobs))))
    finally:
        _JOBS.clear()


def _slabs(L, H, seed):
    rng = np.random.default_rng(seed)
    picks = {(0, 0), (L - 1, H - 1)}
    while len(picks) < N_SLABS:
        picks.add((int(rng.integers(L)), int(rng.integers(H))))
    return sorted(picks)


def _bf16_of(a: np.ndarray) -> np.ndarray:
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(torch.bfloat16).float().numpy()


@pytest.mark.parametrize("case", sorted(CASES))
def test_config_scale_slab_parity(case):
    from paper_2605_13734_b200 import KVCodec
    from paper_2605_13734_b200.synth import synthetic_kv

    shape, sid = CASES[case]
    L, H, T, C = shape
    s = oracle.parse_id(sid)
    w, g = s.bits, s.group
    dev = torch.device("cuda", 0)
    free, _ = torch.cuda.mem_get_info(dev)
    need = 3 * L * H * T * C * 2 * 1.4  # kv, a decoded copy / the page pool, blobs
    if free < need:
        pytest.skip(f"needs {need / 1e9:.0f} GB of free HBM, {free / 1e9:.0f} GB available")
    kv, _ = synthetic_kv(L, H, T, C, seed=7, device=dev)
    codec = KVCodec(sid, shape, block_symbols=BLOCK, device=dev)
    blob = codec.encode(kv)
    codec.check()
    picks = _slabs(L, H, seed=11)
    jobs = [(sid, kv[l, h].float().cpu().numpy().reshape(1, 1, T, C)) for l, h in picks]
    results = _run_oracle(jobs)

    ng_slab = T * C // g
    ngroups = L * H * ng_slab
    meta = blob.metadata
    nblk = T * C // BLOCK
    if s.codec != "none":
        offs_all = blob.offsets[: blob.nblocks + 1].cpu().numpy().astype(np.int64)
    crossed_2_32 = False
    for (l, h), (pay_ref, meta_ref, offs_ref, _) in zip(picks, results):
        lh = l * H + h
        # metadata: the slab's scales, zeros (and affine mu, a)
        parts = [meta[2 * lh * ng_slab: 2 * (lh + 1) * ng_slab],
                 meta[2 * (ngroups + lh * ng_slab): 2 * (ngroups + (lh + 1) * ng_slab)]]
        if s.transform == "affine":
            base = 4 * ngroups
            parts += [meta[base + 2 * lh * C: base + 2 * (lh + 1) * C],
                      meta[base + 2 * L * H * C + 2 * lh * C: base + 2 * L * H * C + 2 * (lh + 1) * C]]
        got_meta = b"".join(bytes(p.cpu().numpy().tobytes()) for p in parts)
        assert got_meta == meta_ref, f"{case}: metadata of slab {(l, h)} differs"
        # payload
        if s.codec == "none":
            p0 = lh * T * C * w // 8
            p1 = p0 + T * C * w // 8
            crossed_2_32 |= p0 >= (1 << 32)
        else:
            b0 = lh * nblk
            p0, p1 = int(offs_all[b0]), int(offs_all[b0 + nblk])
            assert np.array_equal(offs_all[b0: b0 + nblk + 1] - p0, offs_ref), f"{case}: block sizes of slab {(l, h)}"
        got = bytes(blob.payload[p0:p1].cpu().numpy().tobytes())
        assert len(got) == len(pay_ref), f"{case}: slab {(l, h)} payload length {len(got)} != {len(pay_ref)}"
        assert got == pay_ref, f"{case}: payload bytes of slab {(l, h)} differ"
    if case.startswith("c3"):
        assert crossed_2_32, "no sampled c3 slab starts beyond 2^32 payload bytes"

    # decode (contiguous bf16) against the oracle's reconstruction of each slab
    out = codec.decode(blob, device_length=True)
    codec.check(decoding=True)
    for (l, h), (_, _, _, rec) in zip(picks, results):
        ref = _bf16_of(rec.reshape(T, C))
        got = out[l, h].float().cpu().numpy()
        if s.transform in ("identity", "affine"):  # the affine division is correctly rounded
            assert np.array_equal(got, ref), f"{case}: decoded slab {(l, h)} differs"
        else:
            # the fp32 inverse transform is held to the reference's transform
            # tolerance (1e-5 of the row magnitude, test_acceptance.py:235),
            # then rounded to bf16: at most one bf16 ulp more
            rec32 = rec.reshape(T, C)
            tol = 1e-5 * np.abs(rec32).max(axis=-1, keepdims=True) + 2.0 ** -7 * np.abs(ref) + 2.0 ** -133
            err = np.abs(got - ref)
            assert np.all(err <= tol), f"{case}: decoded slab {(l, h)} off by {float((err / tol).max())}x tolerance"

    if s.transform == "affine":
        # paged decode (the c5 serving layout) == contiguous decode
        pt = 16
        n_pages = T // pt
        table = torch.randperm(n_pages, device=dev).to(torch.int32)
        pool = torch.empty(L * n_pages * pt * H * C, dtype=torch.bfloat16, device=dev)
        codec.decode_paged(blob, pool, table, pt, n_pages * pt * H * C, device_length=True)
        codec.check(decoding=True)
        view = pool.view(L, n_pages, pt, H, C)[:, table.long()].reshape(L, T, H, C).permute(0, 2, 1, 3)
        assert torch.equal(view, out), f"{case}: paged decode differs from the contiguous decode"
        del pool, view

    # the whole tensor encoded again straight from a paged cache
    # (kvc_encode_paged, 16-token pages, random table): the same blob
    del out
    torch.cuda.empty_cache()
    pt = 16
    n_pages = T // pt
    table = torch.randperm(n_pages, device=dev).to(torch.int32)
    pool = torch.empty((L, n_pages * pt, H, C), dtype=torch.bfloat16, device=dev)
    rows = (table.long()[:, None] * pt + torch.arange(pt, device=dev)[None, :]).reshape(-1)
    for li in range(L):
        pool[li, rows] = kv[li].permute(1, 0, 2)
    blob2 = codec.encode_paged(pool, table, pt, n_pages * pt * H * C)
    codec.check()
    n = blob.payload_nbytes()
    assert blob2.payload_nbytes() == n, f"{case}: paged encode payload length differs"
    assert torch.equal(blob2.payload[:n], blob.payload[:n]), f"{case}: paged encode payload differs"
    assert torch.equal(blob2.metadata, blob.metadata), f"{case}: paged encode metadata differs"
    if blob.offsets is not None:
        nb = blob.nblocks + 1
        assert torch.equal(blob2.offsets[:nb], blob.offsets[:nb]), f"{case}: paged encode offsets differ"
