"""Round-trip latency of small KV tensors: eager launches vs one CUDA-graph
replay (serving-sized requests, where launch overhead matters).

    python tools/bench_graph_latency.py [--iters 200]

For each (profile, shape): the mean wall time per encode + decode of a
device-resident tensor over `iters` back-to-back round trips (synchronised
once at the end), eager through KVCodec, and as a captured graph replayed.
Prints one JSON line.
"""

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=200)
    args = ap.parse_args()
    import torch

    from paper_2605_13734_b200 import KVCodec
    from paper_2605_13734_b200.synth import synthetic_kv

    dev = torch.device("cuda:0")
    res = []
    cases = [(sid, shape, 2048) for sid in ("t=hadamard;q=uniform,b=4,g=32;c=none",
                                            "t=identity;q=uniform,b=2,g=32;c=entropy")
             for shape in ((1, 8, 1024, 128), (1, 8, 8192, 128), (8, 8, 8192, 128))]
    # entropy latency is one thread's serial pass over its block: shorter blocks
    cases += [("t=identity;q=uniform,b=2,g=32;c=entropy", (1, 8, 1024, 128), b) for b in (1024, 512, 256)]
    for sid, shape, block in cases:
        kv, _ = synthetic_kv(*shape, seed=3, device=dev)
        codec = KVCodec(sid, shape, block_symbols=block, device=dev)
        blob = codec.alloc_blob()
        out = torch.empty_like(kv)

        def step(stream=None):
            codec.encode(kv, out=blob, stream=stream)
            codec.decode(blob, out=out, device_length=True, stream=stream)

        for _ in range(5):
            step()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.iters):
            step()
        torch.cuda.synchronize()
        eager_us = (time.perf_counter() - t0) / args.iters * 1e6

        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            step(side)
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            step(torch.cuda.current_stream())
        for _ in range(5):
            g.replay()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.iters):
            g.replay()
        torch.cuda.synchronize()
        graph_us = (time.perf_counter() - t0) / args.iters * 1e6
        codec.check(decoding=True)
        nbytes = kv.numel() * 2
        res.append({"id": sid, "shape": list(shape), "block_symbols": block, "cr_wire": round(blob.cr_wire, 4),
                    "bytes": nbytes, "eager_us": round(eager_us, 1),
                    "graph_us": round(graph_us, 1), "eager_gbs": round(nbytes / eager_us / 1e3, 1),
                    "graph_gbs": round(nbytes / graph_us / 1e3, 1)})
        del g, kv, out, blob, codec
        torch.cuda.empty_cache()
    print(json.dumps({"iters": args.iters, "results": res}))


if __name__ == "__main__":
    main()
