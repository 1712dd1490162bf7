"""Compress from a paged KV cache vs from a contiguous tensor (one B200).

    python tools/bench_paged_encode.py [--layers 80] [--tokens 131072] [--steps 5]

One c3-shaped tensor (Llama-3.1-70B 128K: 80 x 8 x 131072 x 128 bf16, 21 GB)
with the c3 profile (Hadamard, 4-bit, g=32, c=none), and the c2 V profile
(identity 2-bit + entropy, fused coder).  The same KV is scattered into a
paged pool (vLLM layout [pages, page_tokens, H, C] per layer, random block
table) and compressed with kvc_encode_paged; the blob is checked
byte-identical to the contiguous encode.  Prints one JSON line.
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
    ap.add_argument("--tokens", type=int, default=131072)
    ap.add_argument("--steps", type=int, default=5)
    args = ap.parse_args()
    import torch

    from paper_2605_13734_b200 import KVCodec
    from paper_2605_13734_b200.synth import synthetic_kv

    dev = torch.device("cuda:0")
    L, H, T, C = args.layers, 8, args.tokens, 128
    kv, _ = synthetic_kv(L, H, T, C, seed=7, device=dev)
    out = {"shape": [L, H, T, C], "bytes_in": kv.numel() * 2, "results": []}

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(args.steps):
            fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / args.steps

    for sid in ("t=hadamard;q=uniform,b=4,g=32;c=none", "t=identity;q=uniform,b=2,g=32;c=entropy"):
        codec = KVCodec(sid, (L, H, T, C), device=dev)
        blob = codec.alloc_blob()
        ms_c = timed(lambda: codec.encode(kv, out=blob))
        codec.check()
        ref = (blob.payload_bytes(), blob.metadata_bytes())
        for P in (16, 64):
            n_pages = T // P
            table = torch.randperm(n_pages, device=dev).to(torch.int32)
            pool = torch.empty((L, n_pages * P, H, C), dtype=torch.bfloat16, device=dev)
            rows = (table.long()[:, None] * P + torch.arange(P, device=dev)[None, :]).reshape(-1)
            for li in range(L):
                pool[li, rows] = kv[li].permute(1, 0, 2)
            stride = n_pages * P * H * C
            ms_p = timed(lambda: codec.encode_paged(pool, table, P, stride, out=blob))
            codec.check()
            same = (blob.payload_bytes(), blob.metadata_bytes()) == ref
            out["results"].append({"id": sid, "page_tokens": P, "contiguous_ms": round(ms_c, 3),
                                   "paged_ms": round(ms_p, 3),
                                   "contiguous_gbs": round(kv.numel() * 2 / ms_c / 1e6, 1),
                                   "paged_gbs": round(kv.numel() * 2 / ms_p / 1e6, 1), "identical_blob": same})
            del pool
            torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
