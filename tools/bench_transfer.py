"""KV transfer GPU0 -> GPU1: raw bf16 peer copy vs the pipelined compressed
transfer (contiguous and paged-connector forms).  Needs two GPUs.

    python tools/bench_transfer.py [--layers 80] [--tokens 32768] [--steps 5]

Timed on the destination device: an event on GPU1's stream starts the
window, GPU0's streams wait on it, and a second GPU1 event closes it after
the last chunk's decode.  Prints one JSON line.
"""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=80)
    ap.add_argument("--tokens", type=int, default=32768)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--chunk-layers", type=int, default=8)
    args = ap.parse_args()
    import torch

    from paper_2605_13734_b200.synth import synthetic_kv
    from paper_2605_13734_b200.transfer import PipelinedKVTransfer, enable_peer_access

    d0, d1 = torch.device("cuda:0"), torch.device("cuda:1")
    L, H, T, C = args.layers, 8, args.tokens, 128
    with torch.cuda.device(d0):
        kv, _ = synthetic_kv(L, H, T, C, seed=11, device=d0)
    V = kv.numel() * 2
    enable_peer_access(0, 1)

    def timed(fn):
        fn()
        torch.cuda.synchronize(d0)
        torch.cuda.synchronize(d1)
        ms = []
        for _ in range(args.steps):
            s1 = torch.cuda.current_stream(d1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.device(d1):
                e0.record(s1)
            torch.cuda.current_stream(d0).wait_event(e0)
            fn()
            with torch.cuda.device(d1):
                e1.record(s1)
            torch.cuda.synchronize(d1)
            torch.cuda.synchronize(d0)
            ms.append(e0.elapsed_time(e1))
        return sorted(ms)[len(ms) // 2]

    out = {"shape": [L, H, T, C], "bytes": V, "chunk_layers": args.chunk_layers, "results": []}
    dst_raw = torch.empty_like(kv, device=d1)

    def raw():
        with torch.cuda.device(d1):
            torch.cuda.current_stream(d1).wait_stream(torch.cuda.current_stream(d0))
            dst_raw.copy_(kv, non_blocking=True)

    ms = timed(raw)
    out["results"].append({"path": "raw bf16 peer copy (torch copy_)", "ms": round(ms, 3), "kv_gbs": round(V / ms / 1e6, 1),
                           "wire_bytes": V})
    P = 16
    n_pages = T // P
    g = torch.Generator().manual_seed(5)
    st = torch.randperm(n_pages, generator=g).to(torch.int32).to(d0)
    dt = torch.randperm(n_pages, generator=g).to(torch.int32).to(d1)
    stride = n_pages * P * H * C
    src_pool = torch.empty((L, n_pages * P, H, C), dtype=torch.bfloat16, device=d0)
    rows = (st.long()[:, None] * P + torch.arange(P, device=d0)[None, :]).reshape(-1)
    for li in range(L):
        src_pool[li, rows] = kv[li].permute(1, 0, 2)
    dst_pool = torch.empty((L, n_pages * P, H, C), dtype=torch.bfloat16, device=d1)
    for sid in ("t=hadamard;q=uniform,b=4,g=32;c=none", "t=identity;q=uniform,b=2,g=32;c=entropy"):
        tx = PipelinedKVTransfer(sid, (L, H, T, C), 0, 1, chunk_layers=args.chunk_layers)
        dst = torch.empty_like(kv, device=d1)
        ms = timed(lambda: tx.run(kv, out=dst))
        tx.check()
        wb = tx.wire_bytes()
        out["results"].append({"path": "pipelined compressed, contiguous", "id": sid, "ms": round(ms, 3),
                               "kv_gbs": round(V / ms / 1e6, 1), "wire_bytes": wb})
        ms = timed(lambda: tx.run_paged(src_pool, st, dst_pool, dt, P, stride, stride))
        tx.check()
        out["results"].append({"path": f"pipelined compressed, paged connector (page {P})", "id": sid,
                               "ms": round(ms, 3), "kv_gbs": round(V / ms / 1e6, 1), "wire_bytes": tx.wire_bytes()})
        del tx, dst
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
