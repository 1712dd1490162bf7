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
