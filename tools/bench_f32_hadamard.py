"""Encode time of the reference default profile on float32 input (the
reference's own corpora, tensors.py:79-112): certified float32 encoder vs the
float64 encoder (run once plain and once with KVC_HADAMARD_FP64=1).

    python tools/bench_f32_hadamard.py [L H T]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2605_13734_b200 import KVCodec  # noqa: E402
from paper_2605_13734_b200.synth import synthetic_kv  # noqa: E402


def main():
    L, H, T = (int(v) for v in sys.argv[1:4]) if len(sys.argv) > 3 else (32, 8, 4096)
    sid = "t=hadamard;q=uniform,b=4,g=32;c=none"
    kv, _ = synthetic_kv(L, H, T, 128, seed=0, dtype=torch.float32)
    codec = KVCodec(sid, (L, H, T, 128), in_dtype=torch.float32)
    for _ in range(3):
        codec.encode(kv)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 10
    a.record()
    for _ in range(n):
        codec.encode(kv)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / n
    print(json.dumps({"path": codec.encode_path, "shape": [L, H, T, 128], "encode_ms": round(ms, 4),
                      "f32_in_gbs": round(kv.numel() * 4 / ms / 1e6, 1)}))


if __name__ == "__main__":
    main()
