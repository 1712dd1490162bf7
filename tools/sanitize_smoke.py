"""Small workload touching every kernel family once, for compute-sanitizer
(memcheck / racecheck / synccheck, one tool per run):

    compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_smoke.py

Each strategy is encoded and decoded on a tiny tensor (contiguous and paged),
plus the wire CRC, the device-length copy and the squared-error kernels, and
the results are checked against the oracle so a sanitizer-clean run is also a
correct one.
"""

from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SIDS = [
    "t=hadamard;q=uniform,b=4,g=32;c=none",        # k_enc128 hadamard + fixup, staged decode
    "t=identity;q=uniform,b=2,g=32;c=entropy",     # fused per-token range coder
    "t=identity;q=uchan,b=2,g=32;c=entropy",       # fused per-channel range coder
    "t=identity;q=uchan,b=2,g=32;c=none",          # uchan128
    "t=affine;q=uniform,b=8,g=32;c=entropy",       # affine calibrate, rc_large, gather
    "t=delta;q=uniform,b=4,g=32;c=rle",            # delta128 decode, rle
    "t=hadamard;q=mixed,hi=8,lo=2,g=32,rho=0.25;c=entropy",  # mixed widths, rc_small + rc_large
    "t=identity;q=uniform,b=3,g=16;c=none",        # generic kernels
]


def main() -> None:
    import numpy as np
    import torch

    import oracle
    from paper_2605_13734_b200 import KVCodec
    from paper_2605_13734_b200 import _native as N
    from paper_2605_13734_b200.pipeline import classify_heads

    shape = (2, 2, 2048, 128)
    L, H, T, C = shape
    v, imp = oracle.generate_kv(*shape, seed=1)
    kv = torch.from_numpy(v).to(torch.bfloat16)
    vb = kv.float().numpy()
    kvd = kv.cuda()
    for sid in SIDS:
        cls = classify_heads(imp, 0.25) if "mixed" in sid else None
        codec = KVCodec(sid, shape, out_dtype=torch.float32)
        blob = codec.encode(kvd, head_classes=cls)
        out = codec.decode(blob)
        codec.check(decoding=True)
        ref = oracle.encode_blob(vb, imp, sid, block=2048)
        assert blob.payload_bytes() == ref["payload"], sid
        rec = oracle.decode_blob(ref["payload"], ref["metadata"], ref["offsets"], sid, shape, block=2048)
        assert np.allclose(out.cpu().numpy(), rec, rtol=0, atol=1e-4 * max(1.0, float(np.abs(rec).max()))), sid
        # paged bf16 decode
        c16 = KVCodec(sid, shape)
        pt, n_pages = 16, T // 16
        table = torch.randperm(n_pages, device="cuda").to(torch.int32)
        pool = torch.empty(L * n_pages * pt * H * C, dtype=torch.bfloat16, device="cuda")
        c16.decode_paged(blob, pool, table, pt, n_pages * pt * H * C, device_length=True)
        c16.check(decoding=True)
        print("ok", sid, flush=True)
    # wire container kernels
    codec = KVCodec(SIDS[1], shape)
    blob = codec.encode(kvd)
    crc = torch.zeros(blob.nblocks, dtype=torch.int32, device="cuda")
    N.check(N.lib().kvc_block_crc32(blob.payload.data_ptr(), blob.offsets.data_ptr(), blob.nblocks, crc.data_ptr(),
                                    None))
    dst = torch.empty_like(blob.payload)
    N.check(N.lib().kvc_copy_device_length(dst.data_ptr(), blob.payload.data_ptr(),
                                           blob.offsets[blob.nblocks:].data_ptr(), dst.numel(), None))
    acc = torch.zeros(8, dtype=torch.float64, device="cuda")
    N.check(N.lib().kvc_sq_error(kvd.data_ptr(), kvd.data_ptr(), kvd.numel(), N.DTYPE_BF16, acc.data_ptr(), None))
    N.check(N.lib().kvc_sq_error_partials(kvd.data_ptr(), None, kvd.numel(), N.DTYPE_BF16, acc.data_ptr(), 8, None))
    torch.cuda.synchronize()
    n = blob.payload_nbytes()
    assert torch.equal(dst[:n], blob.payload[:n])
    print("ok wire kernels", flush=True)


if __name__ == "__main__":
    main()
