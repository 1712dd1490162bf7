"""BASELINE config 4: profile sweep over the strategy space on Llama-3.1-8B
KV at 16K tokens (32 layers x 8 KV heads x 16384 x 128, K and V).

For every candidate — the 180 ids of the reference's enumerate_space(SpaceDef())
(profiling/space.py:24-35, restated in tests/kv_space.py) plus per-layer
(q=mixlayer) and per-token (q=mixtok) mixed-precision variants — measure
the reference's profile tuple through the reference-facing API
(pipeline.compress with CudaEventTimer): cr (wire), s_enc, s_dec (bf16-in
B/s, compress.py:134-137) and quality (tensors.py:115-134), i.e. exactly what
`kvpilot profile` stores per Profile (cli.py:111-121).  Prints one JSON line
per strategy and a summary (Pareto front on (cr, s_p, quality)).

    python tools/sweep_c4.py [--tokens 16384] [--layers 32] [--limit N] [--out gpurun_out/sweep_c4.jsonl]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def candidates():
    from kv_space import all_ids

    ids = list(all_ids())
    for t in ("identity", "hadamard"):
        for hi, lo in ((8, 2), (4, 2), (8, 4)):
            for rho in (0.125, 0.25):
                for c in ("none", "entropy"):
                    ids.append(f"t={t};q=mixlayer,hi={hi},lo={lo},g=32,rho={rho!r};c={c}")
                    ids.append(f"t={t};q=mixtok,hi={hi},lo={lo},g=32,rho={rho!r};c={c}")
    return ids


def pareto(rows):
    front = []
    for r in rows:
        dominated = any(
            o["cr"] >= r["cr"] and o["s_p"] >= r["s_p"] and o["quality"] >= r["quality"]
            and (o["cr"] > r["cr"] or o["s_p"] > r["s_p"] or o["quality"] > r["quality"])
            for o in rows
        )
        if not dominated:
            front.append(r["id"])
    return front


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=16384)
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--limit", type=int, default=0)
    ap.add_argument("--out", default="")
    ap.add_argument("--match", default="", help="only ids containing all of these comma-separated substrings")
    args = ap.parse_args()

    import torch

    from paper_2605_13734_b200 import CudaEventTimer, KVTensor, compress
    from paper_2605_13734_b200.synth import synthetic_kv

    shape = (args.layers, 8, args.tokens, 128)
    kvs = []
    for seed in (0, 1):  # K and V
        kv, imp = synthetic_kv(*shape, seed=seed)
        kvs.append(KVTensor(kv, imp))
    timer = CudaEventTimer(repeats=3, warmup=1)
    ids = candidates()
    if args.match:
        ids = [i for i in ids if all(m in i for m in args.match.split(","))]
    if args.limit:
        ids = ids[: args.limit]
    out = open(args.out, "w") if args.out else None
    rows = []
    t0 = time.time()
    for sid in ids:
        tot = enc = dec = 0.0
        crs, qs = [], []
        for x in kvs:
            blob, m = compress(x, sid, timer)
            tot += x.nbytes_source
            enc += x.nbytes_source / m.s_enc
            dec += x.nbytes_source / m.s_dec
            crs.append(m.cr)
            qs.append(m.quality)
            del blob
        s_enc, s_dec = tot / enc, tot / dec
        row = {"id": sid, "cr": sum(crs) / len(crs), "s_enc": s_enc, "s_dec": s_dec,
               "s_p": s_enc * s_dec / (s_enc + s_dec), "quality": sum(qs) / len(qs)}
        rows.append(row)
        line = json.dumps(row)
        print(line, flush=True)
        if out:
            out.write(line + "\n")
        torch.cuda.empty_cache()
    front = pareto(rows)
    summary = {"summary": True, "n": len(rows), "shape": list(shape), "seconds": round(time.time() - t0, 1),
               "pareto": front,
               "s_p_GBps_min_median_max": [round(sorted(r["s_p"] for r in rows)[k] / 1e9, 2)
                                            for k in (0, len(rows) // 2, len(rows) - 1)]}
    print(json.dumps(summary), flush=True)
    if out:
        out.write(json.dumps(summary) + "\n")


if __name__ == "__main__":
    main()
