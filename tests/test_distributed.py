"""Multi-process host logic on CPU (gloo, world size 2): layer sharding,
global class slicing and the compressed-size all-gather -> wire offsets.
Sharded oracle blobs equal the whole-tensor blob (codec none), so the only
cross-rank exchange needed is the sizes."""

import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2605_13734_b200.distributed import global_offsets, shard_range


def test_shard_range_covers_exactly():
    for n in (1, 7, 32, 80):
        for world in (1, 2, 3, 8):
            spans = [shard_range(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(e - s for s, e in spans) - min(e - s for s, e in spans) <= 1


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    L, H, T, C = 5, 4, 16, 64
    v, imp = oracle.generate_kv(L, H, T, C, seed=42)
    sid = "t=hadamard;q=mixed,hi=8,lo=2,g=32,rho=0.25;c=none"
    cls = oracle.classify_heads(imp, 0.25)  # global labels, sliced per rank
    l0, l1 = shard_range(L, world, rank)
    from oracle.extensions import quantize_any

    y = oracle.transform_fwd(v[l0:l1], "hadamard")
    bits = np.broadcast_to(np.where(cls[l0:l1], 8, 2).astype(np.uint8)[:, :, None], y.shape[:3]).copy()
    sym, sc, ze = quantize_any(y, bits, 32)
    local_bytes = sym.size  # any per-rank size
    offs, total = global_offsets(local_bytes, device=torch.device("cpu"))
    out[rank] = (offs, total, sym.tobytes(), sc.tobytes())
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_two_ranks_offsets_and_equivalence():
    world = 2
    port = 29500 + os.getpid() % 1000
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    sizes = [len(res[r][2]) for r in range(world)]
    for r in range(world):
        offs, total = res[r][0], res[r][1]
        assert offs == [0, sizes[0]] and total == sum(sizes)
    # sharded quantization == whole-tensor quantization (global class labels)
    L, H, T, C = 5, 4, 16, 64
    v, imp = oracle.generate_kv(L, H, T, C, seed=42)
    whole = oracle.encode_blob(v, imp, "t=hadamard;q=mixed,hi=8,lo=2,g=32,rho=0.25;c=none")
    assert b"".join(res[r][2] for r in range(world)) == whole["symbols"].tobytes()
    assert b"".join(res[r][3] for r in range(world)) == whole["scales"].tobytes()


class _OracleBlob:
    """What ShardedCodec.wire_bytes reads from a DeviceBlob, host-side."""

    def __init__(self, payload: bytes, metadata: bytes, symbols, scales):
        self.payload, self._meta = payload, metadata
        self.metadata = torch.zeros(len(metadata), dtype=torch.uint8)
        self.framing_nbytes = 0
        self.symbols, self.scales = symbols, scales

    def payload_nbytes(self):
        return len(self.payload)


class _OracleCodec:
    """Stands in for KVCodec (the CUDA part) on CPU: the oracle's transform ->
    quantize (with the GIVEN head classes) -> width streams -> packing."""

    def __init__(self, sid, shape, **kw):
        self.s = oracle.parse_id(sid)
        self.shape = shape

    def encode(self, kv, head_classes=None, out=None, stream=None):
        from oracle.extensions import blob_streams, quantize_any

        s = self.s
        y = oracle.transform_fwd(np.asarray(kv, dtype=np.float32), s.transform)
        if head_classes is not None:
            w = np.where(head_classes, s.hi, s.lo).astype(np.uint8)
        else:
            w = np.full(y.shape[:2], s.bits, dtype=np.uint8)
        bits = np.broadcast_to(w[:, :, None], y.shape[:3]).copy()
        sym, sc, ze = quantize_any(y, bits, s.group)
        payload = b"".join(oracle.pack_bits(st, bw) for bw, st in blob_streams(sym, bits))
        meta = sc.tobytes() + ze.tobytes()
        if head_classes is not None:
            meta += np.packbits(np.asarray(head_classes).reshape(-1)).tobytes()
        return _OracleBlob(payload, meta, sym, sc)


def _sharded_worker(rank, world, port, out):
    from paper_2605_13734_b200.distributed import ShardedCodec

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    shape = (5, 4, 16, 128)
    v, imp = oracle.generate_kv(*shape, seed=43)
    res = {}
    for by in ("layer", "head"):
        for sid in ("t=hadamard;q=uniform,b=4,g=32;c=none", "t=identity;q=mixed,hi=8,lo=2,g=32,rho=0.25;c=none"):
            sc = ShardedCodec(sid, shape, by=by, codec_factory=_OracleCodec)  # rank / world from the process group
            cls = oracle.classify_heads(imp, 0.25) if "mixed" in sid else None  # global labels
            blob = sc.encode(sc.local_slice(v), global_classes=cls)
            off, total = sc.wire_layout(blob, device=torch.device("cpu"))
            res[(by, sid)] = (sc.l0, sc.l1, sc.h0, sc.h1, off, total, sc.wire_bytes(blob), blob.payload,
                              blob.symbols.tobytes(), blob.symbols.shape)
    out[rank] = res
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_sharded_codec_wire_layout_layer_and_head():
    """The product's ShardedCodec on two gloo ranks (its CUDA codec replaced
    by the oracle): shard ranges, global class slicing and wire_layout's
    all-gather -> exclusive offsets; layer shards of a uniform profile
    concatenate to the whole-tensor payload, and head shards reproduce the
    whole-tensor symbols of their heads (mixed labels sliced, not re-derived)."""
    world = 2
    port = 29500 + (os.getpid() + 7) % 1000
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_sharded_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    shape = (5, 4, 16, 128)
    v, imp = oracle.generate_kv(*shape, seed=43)
    for key in res[0]:
        by, sid = key
        sizes = [res[r][key][6] for r in range(world)]
        for r in range(world):
            off, total = res[r][key][4], res[r][key][5]
            assert off == sum(sizes[:r]) and total == sum(sizes), key
        whole = oracle.encode_blob(v, imp, sid)
        wsym = whole["symbols"]
        for r in range(world):
            l0, l1, h0, h1 = res[r][key][:4]
            sym = np.frombuffer(res[r][key][8], dtype=wsym.dtype).reshape(res[r][key][9])
            assert np.array_equal(sym, wsym[l0:l1, h0:h1]), (key, r)
        if by == "layer" and "uniform" in sid:
            assert b"".join(res[r][key][7] for r in range(world)) == whole["payload"], key
    # the head split covers all heads once
    spans = sorted(res[r][("head", "t=hadamard;q=uniform,b=4,g=32;c=none")][2:4] for r in range(world))
    assert spans[0][0] == 0 and spans[-1][1] == 4 and spans[0][1] == spans[1][0]
