"""Run tests/test_gpu_parity.py's seeded fuzz cases one by one and report each
failure; a CUDA error poisons the context, so the process exits and the
caller restarts it after the failing index.

    python tools/fuzz_parity.py START END [fused]  -> prints 'FAIL k sid shape block f32 : msg' / 'DONE k'

`fused` draws from _fuzz_case_fast (head_dim-128 shapes for the fused kernels).
"""
import os
import sys
import traceback

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import test_gpu_parity as T  # noqa: E402


def main():
    a, b = int(sys.argv[1]), int(sys.argv[2])
    gen = T._fuzz_case_fast if len(sys.argv) > 3 and sys.argv[3] == "fused" else T._fuzz_case
    for k in range(a, b):
        sid, shape, block, f32 = gen(k)
        try:
            got, rec, _ = T.run_case(sid, shape, seed=k, block=block, in_f32=f32)
            T.assert_decoded(got, rec, sid, shape, in_f32=f32)
        except Exception as e:  # noqa: BLE001
            msg = str(e).splitlines()[0][:160]
            print(f"FAIL {k} {sid} {shape} {block} {f32} : {type(e).__name__}: {msg}", flush=True)
            if "CUDA" in msg or "Accelerator" in type(e).__name__ or "misaligned" in msg or "illegal" in msg:
                print(f"RESTART {k + 1}", flush=True)
                sys.exit(3)
    print(f"DONE {b}", flush=True)


if __name__ == "__main__":
    main()
