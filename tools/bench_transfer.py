"""KV transfer between two GPUs: raw bf16 copy vs compressed + pipelined
(paper_2605_13734_b200.transfer), and the serial compress -> copy ->
decompress the reference's simulator assumes (engine.py:143-157).

    python tools/bench_transfer.py [--workload c1|c2] [--chunk-layers 4] [--reps 10]

Prints one JSON line per mode: delivered bf16 GB/s (2 * elements / time),
wire bytes, CUDA-event time on the destination stream after a full sync.
Needs two visible GPUs (gpurun --gpus 2); src = cuda:0, dst = cuda:1.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2605_13734_b200 import KVCodec  # noqa: E402
from paper_2605_13734_b200.synth import synthetic_kv  # noqa: E402
from paper_2605_13734_b200.transfer import PipelinedKVTransfer, enable_peer_access  # noqa: E402

WORKLOADS = {
    "c1": ((32, 8, 4096, 128), "t=hadamard;q=uniform,b=4,g=32;c=none"),
    "c2": ((32, 8, 32768, 128), "t=identity;q=uniform,b=2,g=32;c=entropy"),
}


def timed(fn, reps, src, dst):
    """Median device time: both events on the destination device; the source
    stream waits for the start event, so the span covers every stage."""
    for _ in range(2):
        fn()
    torch.cuda.synchronize(src)
    torch.cuda.synchronize(dst)
    ts = []
    for _ in range(reps):
        with torch.cuda.device(dst):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(torch.cuda.current_stream(dst))
        torch.cuda.current_stream(src).wait_event(a)
        fn()
        with torch.cuda.device(dst):
            b.record(torch.cuda.current_stream(dst))
        torch.cuda.synchronize(src)
        torch.cuda.synchronize(dst)
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--workload", default="c1", choices=sorted(WORKLOADS))
    p.add_argument("--chunk-layers", type=int, nargs="+", default=[8])
    p.add_argument("--reps", type=int, default=10)
    args = p.parse_args()
    if torch.cuda.device_count() < 2:
        print(json.dumps({"unavailable": "needs two GPUs"}))
        return
    shape, sid = WORKLOADS[args.workload]
    src, dst = torch.device("cuda", 0), torch.device("cuda", 1)
    enable_peer_access(0, 1)
    kv, _ = synthetic_kv(*shape, seed=0, device=src)
    nbytes = kv.numel() * 2
    out = torch.empty(shape, dtype=torch.bfloat16, device=dst)

    def raw():
        with torch.cuda.device(dst):
            out.copy_(kv, non_blocking=True)

    ms = timed(raw, args.reps, src, dst)
    print(json.dumps({"mode": "raw_bf16_copy", "workload": args.workload, "ms": round(ms, 4),
                      "delivered_gbs": round(nbytes / ms / 1e6, 1), "wire_bytes": nbytes}))

    for cl in args.chunk_layers:
        tx = PipelinedKVTransfer(sid, shape, src, dst, chunk_layers=cl)

        def piped():
            tx.run(kv, out=out)

        ms = timed(piped, args.reps, src, dst)
        tx.check()
        print(json.dumps({"mode": "pipelined_compressed", "workload": args.workload, "strategy": sid,
                          "chunk_layers": cl, "ms": round(ms, 4),
                          "delivered_gbs": round(nbytes / ms / 1e6, 1), "wire_bytes": tx.wire_bytes()}))
        # the source side alone (encode + copy of every chunk), for the stage split
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t2 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.device(src):
            torch.cuda.synchronize(src)
            t0.record(tx.s_enc)
            for i, (l0, l1) in enumerate(tx.chunks):
                tx.enc[i].encode(kv[l0:l1], out=tx.tx_src[i], stream=tx.s_enc)
            t1.record(tx.s_enc)
            torch.cuda.synchronize(src)
        with torch.cuda.device(dst):
            torch.cuda.synchronize(dst)
            a = torch.cuda.Event(enable_timing=True)
            a.record(tx.s_dec)
            for i, (l0, l1) in enumerate(tx.chunks):
                tx.dec[i].decode(tx.tx_dst[i], out=out[l0:l1], stream=tx.s_dec,
                                 device_length=tx.tx_dst[i].offsets is not None)
            t2.record(tx.s_dec)
            torch.cuda.synchronize(dst)
        print(json.dumps({"mode": "stage_split", "chunk_layers": cl, "encode_ms": round(t0.elapsed_time(t1), 4),
                          "decode_ms": round(a.elapsed_time(t2), 4)}))

    enc = KVCodec(sid, shape, device=src)
    dec = KVCodec(sid, shape, device=dst)
    blob = enc.encode(kv)
    with torch.cuda.device(dst):
        dblob = dec.alloc_blob()

    def serial():
        b = enc.encode(kv, out=blob)
        n = b.payload_nbytes()  # the serial model: wait for compress, then send
        with torch.cuda.device(dst):
            dblob.payload[:n].copy_(b.payload[:n], non_blocking=True)
            dblob.metadata.copy_(b.metadata, non_blocking=True)
            if b.offsets is not None:
                dblob.offsets.copy_(b.offsets, non_blocking=True)
            dblob.nblocks, dblob._nbytes = b.nblocks, n
            dec.decode(dblob, out=out)

    ms = timed(serial, args.reps, src, dst)
    print(json.dumps({"mode": "serial_compressed", "workload": args.workload, "ms": round(ms, 4),
                      "delivered_gbs": round(nbytes / ms / 1e6, 1)}))


if __name__ == "__main__":
    main()
