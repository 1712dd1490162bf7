"""Multi-process check of the sharded codec over NCCL (one process per GPU):

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/run_sharded_nccl.py

Every rank builds the same global (L, H, T, C) cache on its GPU (seeded),
encodes its layer- or head-shard with ShardedCodec, and the one collective
of the sharded path -- the int64 all-gather of compressed sizes
(wire_layout) -- lays the rank payloads out back to back.  Each rank then
checks its shard's decode against the whole-tensor decode's slice, the
offsets against the gathered sizes, and rank 0 prints one JSON line.
"""

from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main() -> None:
    import torch
    import torch.distributed as dist

    from paper_2605_13734_b200 import KVCodec
    from paper_2605_13734_b200.distributed import ShardedCodec
    from paper_2605_13734_b200.pipeline import classify_heads
    from paper_2605_13734_b200.synth import synthetic_kv

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    rank, world = dist.get_rank(), dist.get_world_size()
    shape = (8, 8, 4096, 128)
    kv, imp = synthetic_kv(*shape, seed=5, device=dev)
    results = []
    for sid in ("t=hadamard;q=uniform,b=4,g=32;c=none", "t=identity;q=uniform,b=2,g=32;c=entropy",
                "t=hadamard;q=mixed,hi=8,lo=2,g=32,rho=0.25;c=entropy"):
        cls = classify_heads(imp, 0.25) if "mixed" in sid else None
        whole = KVCodec(sid, shape, device=dev)
        want = whole.decode(whole.encode(kv, head_classes=cls))
        for by in ("layer", "head"):
            sc = ShardedCodec(sid, shape, by=by, device=dev)
            blob = sc.encode(sc.local_slice(kv), global_classes=cls)
            got = sc.decode(blob)
            sc.codec.check(decoding=True)
            ok = bool(torch.equal(got, want[sc.l0:sc.l1, sc.h0:sc.h1]))
            off, total = sc.wire_layout(blob)
            sizes = [None] * world
            dist.all_gather_object(sizes, sc.wire_bytes(blob))
            ok_layout = off == sum(sizes[:rank]) and total == sum(sizes)
            flags = torch.tensor([int(ok and ok_layout)], device=dev)
            dist.all_reduce(flags, op=dist.ReduceOp.MIN)
            results.append({"sid": sid, "by": by, "ok": bool(flags.item()), "rank_wire_bytes": sizes})
    if rank == 0:
        print(json.dumps({"world": world, "nccl": torch.cuda.nccl.version(), "cases": results,
                          "all_ok": all(r["ok"] for r in results)}))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
