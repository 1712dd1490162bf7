"""Benchmark of the KV compress/decompress hot path (BASELINE.json metric:
"KV compress/decompress GB/s (bf16-in) per B200 & 8-GPU, at compression ratio").

One step = the reference's compress() round trip (compress.py:111-140) for
every KV tensor of the workload: encode (transform -> quantize -> lossless
codec) then decode (codec -> dequantize -> inverse transform) back to bf16,
inputs and outputs resident in HBM.  `value` is bf16-in GB/s of that round
trip, V / (t_enc + t_dec) -- the reference's s_p (compress.py:32-40) --
summed over ranks; compress and decompress GB/s are reported separately.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c3|c1|c2|c5]
                    [--impl ours|reference] [--no-extras]

Workloads (BASELINE.json configs; c3 = the north-star scaling config, the
largest single-GPU config, is the headline):
  c3  Llama-3.1-70B 128K (80,8,128000,128) K,V: t=hadamard;q=uniform,b=4,g=32;c=none,
                                           layers sharded over ranks (strong scaling)
  c1  Llama-3.1-8B 4K   (32,8,4096,128)   K,V: the same reference default profile
  c2  Llama-3.1-8B 32K  (32,8,32768,128)  K: t=identity;q=uchan,b=2,g=32;c=entropy (KIVI per-channel)
                                           V: t=identity;q=uniform,b=2,g=32;c=entropy (per-token)
  c5  Qwen3-8B 16K      (36,8,16384,128)  K,V: t=affine;q=uniform,b=8,g=32;c=entropy, decoded into paged KV
  c4  Llama-3.1-8B 16K   (32,8,16384,128)  the mixed-precision profiles (per-layer mixlayer,
                                           per-token mixtok, per-head mixed; 36 ids), swept
At N=1 the default run also measures c1, c2, c4 and c5 and nests them under
"extra" (same fields, fewer steps; c4 as an aggregate + per-profile list).
Multi-GPU: torchrun, one process per
GPU; no collective on the data path -- only the per-rank compressed sizes
are all-gathered (offsets for the wire).

--impl reference: the reference pipeline's CPU implementation -- the oracle
port (oracle/, the reference is Python and cannot travel to the GPU box) --
on all host cores, same metric / config / unit as this arm.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "KV compress+decompress round-trip GB/s (bf16-in)"
C1_PROFILE = "t=hadamard;q=uniform,b=4,g=32;c=none"
WORKLOADS = {
    "c3": dict(name="Llama-3.1-70B KV 128K tokens, reference default profile, layer-sharded", shape=(80, 8, 128000, 128),
               tensors=[("K", C1_PROFILE), ("V", C1_PROFILE)], shard=True, paged=False),
    "c1": dict(name="Llama-3.1-8B KV 4K tokens, reference default profile", shape=(32, 8, 4096, 128),
               tensors=[("K", C1_PROFILE), ("V", C1_PROFILE)], shard=False, paged=False),
    "c2": dict(name="Llama-3.1-8B KV 32K tokens, KIVI 2-bit per-channel K / per-token V + entropy",
               shape=(32, 8, 32768, 128),
               tensors=[("K", "t=identity;q=uchan,b=2,g=32;c=entropy"), ("V", "t=identity;q=uniform,b=2,g=32;c=entropy")],
               shard=False, paged=False),
    "c5": dict(name="Qwen3-8B GQA KV 16K tokens, affine + 8-bit + entropy, paged decode", shape=(36, 8, 16384, 128),
               tensors=[("K", "t=affine;q=uniform,b=8,g=32;c=entropy"), ("V", "t=affine;q=uniform,b=8,g=32;c=entropy")],
               shard=False, paged=True),
}
EXTRAS = ("c1", "c2", "c4", "c5")
# BASELINE configs[3]: the mixed-precision profiles of the strategy space --
# per-layer (q=mixlayer) and per-token (q=mixtok) mixed precision, plus the
# reference's per-head mixed_head -- on Llama-3.1-8B KV at 16K tokens
C4_SHAPE = (32, 8, 16384, 128)


def c4_ids() -> list[str]:
    ids = []
    for t in ("identity", "hadamard"):
        for kind in ("mixlayer", "mixtok", "mixed"):
            for hi, lo in ((8, 2), (4, 2), (8, 4)):
                for c in ("none", "entropy"):
                    ids.append(f"t={t};q={kind},hi={hi},lo={lo},g=32,rho=0.25;c={c}")
    return ids
EXTRA_STEPS = 5
BLOCK = 2048
PAGE_TOKENS = 16
CPU_TOKENS = 8192  # tokens per head slab in the CPU samples


def _args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--workload", default="c3", choices=sorted(WORKLOADS))
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--no-extras", action="store_true", help="headline workload only")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--block", type=int, default=None, help="codec block symbols (default 2048)")
    p.add_argument("--serial", action="store_true", help="K and V on one stream (default: one stream each)")
    args = p.parse_args()
    global BLOCK
    if args.block:
        BLOCK = args.block
    return args


def config_of(workload: str, world: int) -> dict:
    """The `config` object, identical in both arms."""
    wl = WORKLOADS[workload]
    return {"workload": workload, "name": wl["name"], "shape": list(wl["shape"]), "tensors": dict(wl["tensors"]),
            "block_symbols": BLOCK, "paged": wl["paged"], "l2": "inputs larger than L2 (no flush needed)",
            "parallelism": (f"layer-sharded x{world} (strong)" if wl["shard"] else f"dp{world} independent caches (weak)")}


def _shard_shape(wl, rank, world):
    L, H, T, C = wl["shape"]
    if not wl["shard"]:
        return (L, H, T, C), (0, L)
    per = [L // world + (1 if r < L % world else 0) for r in range(world)]
    l0 = sum(per[:rank])
    return (per[rank], H, T, C), (l0, l0 + per[rank])


# ----------------------------------------------------------------------------
# CPU side: the reference pipeline's CPU implementation (the oracle port) on
# the host cores.  Inputs are generated in the parent BEFORE the worker pool
# forks; only encode + decode run inside the timed region.
# ----------------------------------------------------------------------------
_CPU_SLABS: list = []


def _cpu_slab(i):
    """Round trip of pre-generated head slab i through the oracle; runs in a
    pool worker; returns (bf16 bytes, seconds)."""
    import oracle

    sid, v, imp = _CPU_SLABS[i]
    t0 = time.perf_counter()
    ob = oracle.encode_blob(v, imp, sid, block=BLOCK)
    oracle.decode_blob(ob["payload"], ob["metadata"], ob["offsets"], sid, v.shape, block=BLOCK)
    return v.size * 2, time.perf_counter() - t0


def _cpu_ping(_):
    return os.getpid()


class CpuBaseline:
    """The oracle round trip of `slabs_per_step` head slabs per step, one
    slab per worker process (all host cores); value = bytes / wall seconds
    of the codec work only (pool started and inputs generated beforehand)."""

    def __init__(self, workload: str, slabs_per_step: int, steps: int, seed0: int = 1000):
        import multiprocessing as mp

        import numpy as np

        import oracle

        wl = WORKLOADS[workload]
        _, _, T, C = wl["shape"]
        self.tok = min(T, CPU_TOKENS)
        self.procs = len(os.sched_getaffinity(0))
        self.per_step = slabs_per_step
        self.steps = steps
        _CPU_SLABS.clear()
        for i in range(slabs_per_step * steps):
            sid = wl["tensors"][i % len(wl["tensors"])][1]
            v, imp = oracle.generate_kv(1, 1, self.tok, C, seed=seed0 + i)
            u = v.view(np.uint32).astype(np.uint64)
            v = ((((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16).astype(np.uint32)).view(np.float32)  # bf16-exact
            _CPU_SLABS.append((sid, v, imp))
        self.pool = mp.get_context("fork").Pool(self.procs)
        self.pool.map(_cpu_ping, range(self.procs), chunksize=1)  # workers up before any timing

    def run_step(self, k: int) -> tuple[int, float]:
        idx = list(range(k * self.per_step, (k + 1) * self.per_step))
        t0 = time.perf_counter()
        res = self.pool.map(_cpu_slab, idx, chunksize=1)
        return sum(r[0] for r in res), time.perf_counter() - t0

    def close(self):
        self.pool.close()
        self.pool.join()
        _CPU_SLABS.clear()

    def sample(self, C: int) -> str:
        return (f"{self.per_step} head slabs per step x {self.tok} tokens x {C} ch of this workload's strategies "
                f"(bf16-exact reference-generator data), oracle encode+decode on {self.procs} worker processes")


def cpu_measure(workload: str, steps: int, warmup: int) -> dict:
    """cpu_baseline object for `workload` (the same figure the reference arm reports)."""
    procs = len(os.sched_getaffinity(0))
    cb = CpuBaseline(workload, procs, warmup + steps)
    try:
        for k in range(warmup):
            cb.run_step(k)
        nb = wall = 0.0
        for k in range(warmup, warmup + steps):
            b, w = cb.run_step(k)
            nb += b
            wall += w
    finally:
        cb.close()
    return {"value": round(nb / wall / 1e9, 6), "unit": "GB/s", "cores": procs, "kind": "port",
            "sample": cb.sample(WORKLOADS[workload]["shape"][3]), "ms_per_step": round(1e3 * wall / steps, 3)}


def reference_arm(args, rank, world):
    """--impl reference: the oracle port of the reference pipeline on all host cores."""
    if rank != 0:
        return
    cpu = cpu_measure(args.workload, args.steps, max(1, min(args.warmup, 1)))
    line = {
        "impl": "reference", "metric": METRIC, "value": cpu["value"], "unit": "GB/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": cpu["ms_per_step"], "higher_is_better": True,
        "scaling": "strong" if WORKLOADS[args.workload]["shard"] else "weak", "vs_baseline": None,
        "dtype": "bf16 in/out; f32/f64 numpy transform+quantizer, u32 C range coder", "data": "synthetic",
        "config": config_of(args.workload, args.gpus),
        "cpu_baseline": {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": cpu["value"], "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)


# ----------------------------------------------------------------------------
# ncu evidence for the dominant kernel (committed captures under profiles/)
# ----------------------------------------------------------------------------
_NCU_KERNELS = {
    "fused_encode": ("k_fused_tok_encode", "k_fused_chan_encode"),
    "fused_decode": ("k_fused_tok_decode", "k_fused_chan_decode"),
    "encode_fast128": ("k_enc128",), "decode_fast128": ("k_dec128",),
    "rc_encode": ("k_rc_large_encode", "k_rc_small_encode"), "rc_decode": ("k_rc_large_decode", "k_rc_small_decode"),
    "gather": ("k_gather",),
}


def _ncu_evidence(workload: str, scope: str):
    """Per-launch DRAM bytes, warp instructions and issue-active % of the
    kernels behind `scope`, averaged over the launches in the newest
    profiles/r*/ncu_full_<workload>_raw.csv (tools/prof_one.sh), or None."""
    import csv
    import glob

    names = _NCU_KERNELS.get(scope)
    paths = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", f"ncu_full_{workload}_raw.csv")))
    if not names or not paths:
        return None
    unit = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "inst": 1.0, "%": 1.0}
    try:
        rows = list(csv.reader(open(paths[-1])))
        h, u = rows[0], rows[1]
        col = {n: h.index(n) for n in ("Kernel Name", "dram__bytes_read.sum", "dram__bytes_write.sum",
                                        "smsp__inst_executed.sum",
                                        "smsp__issue_active.avg.pct_of_peak_sustained_active")}
        acc, n = [0.0, 0.0, 0.0], 0
        for r in rows[2:]:
            if not any(k in r[col["Kernel Name"]] for k in names):
                continue
            v = lambda key: float(r[col[key]].replace(",", "")) * unit.get(u[col[key]], 1.0)  # noqa: E731
            acc[0] += v("dram__bytes_read.sum") + v("dram__bytes_write.sum")
            acc[1] += v("smsp__inst_executed.sum")
            acc[2] += v("smsp__issue_active.avg.pct_of_peak_sustained_active")
            n += 1
        if n == 0:
            return None
        return {"dram_bytes": acc[0] / n, "inst": acc[1] / n, "issue_pct": acc[2] / n,
                "source": os.path.relpath(paths[-1], ROOT)}
    except Exception:
        return None


# ----------------------------------------------------------------------------
# clocks during the timed region
# ----------------------------------------------------------------------------

class ClockSampler:
    def __init__(self, index):
        self.proc = None
        self.path = None
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(index), "--query-gpu=clocks.sm,clocks.max.sm,power.draw,"
                 "clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 8:
                try:
                    rows.append((float(parts[0]), float(parts[1]), parts[4:8]))
                except ValueError:
                    pass
        os.unlink(self.path)
        if not rows:
            return None
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for _, _, r in rows for i, v in enumerate(r) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(r[0] for r in rows), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows)}


# ----------------------------------------------------------------------------
# GPU side
# ----------------------------------------------------------------------------

def _bits_group(sid: str):
    w = int(sid.split("b=")[1].split(",")[0]) if "b=" in sid else 4
    g = int(sid.split("g=")[1].split(",")[0].split(";")[0])
    return w, g


def run_workload(workload: str, args, steps: int, rank: int, world: int, dev, do_e2e: bool,
                 cpu: dict | None, hbm_peak: float, peak_src: str) -> dict:
    """Measure one workload on this rank; returns the fields of its JSON line
    (collectives inside are executed by every rank)."""
    import torch
    import torch.distributed as dist

    from paper_2605_13734_b200 import KVCodec
    from paper_2605_13734_b200 import _native as N
    from paper_2605_13734_b200.synth import synthetic_kv

    wl = WORKLOADS[workload]
    shape, (l0, l1) = _shard_shape(wl, rank, world)
    L, H, T, C = shape
    E = L * H * T * C
    tensors = []
    for ti, (name, sid) in enumerate(wl["tensors"]):
        kv, _ = synthetic_kv(L, H, T, C, seed=1000 * rank + 17 * ti + l0, device=dev)
        codec = KVCodec(sid, shape, block_symbols=BLOCK, device=dev)
        tensors.append(dict(name=name, sid=sid, kv=kv, codec=codec, blob=codec.alloc_blob(), out=None))
    torch.cuda.synchronize()
    V_rank = 2 * E * len(tensors)  # bf16-in bytes per step on this rank

    paged = None
    if wl["paged"]:
        n_pages = T // PAGE_TOKENS
        perm = torch.randperm(n_pages, device=dev).to(torch.int32)
        paged = dict(page_tokens=PAGE_TOKENS, table=perm, layer_stride=n_pages * PAGE_TOKENS * H * C)
        for t in tensors:
            t["out"] = torch.empty(L * n_pages * PAGE_TOKENS * H * C, dtype=torch.bfloat16, device=dev)
    else:
        for t in tensors:
            t["out"] = torch.empty_like(t["kv"])

    # K and V are independent: each runs on its own stream
    main = torch.cuda.current_stream()
    for t in tensors:
        t["stream"] = main if args.serial else torch.cuda.Stream(device=dev)

    def _fork():
        e = torch.cuda.Event()
        e.record(main)
        for t in tensors:
            t["stream"].wait_event(e)

    def _join():
        for t in tensors:
            e = torch.cuda.Event()
            e.record(t["stream"])
            main.wait_event(e)

    def encode_all():
        _fork()
        for t in tensors:
            t["codec"].encode(t["kv"], out=t["blob"], stream=t["stream"])
        _join()

    def decode_all():
        _fork()
        for t in tensors:
            if paged:
                t["codec"].decode_paged(t["blob"], t["out"], paged["table"], paged["page_tokens"], paged["layer_stride"],
                                        stream=t["stream"], device_length=True)
            else:
                t["codec"].decode(t["blob"], out=t["out"], device_length=True, stream=t["stream"])
        _join()

    for _ in range(args.warmup):
        encode_all()
        decode_all()
    for t in tensors:
        t["codec"].check()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    # ---------------- timed region
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(steps)]
    clocks = ClockSampler(dev.index)
    time.sleep(0.3)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    wall0 = time.perf_counter()
    for k in range(steps):
        ev[k][0].record()
        encode_all()
        ev[k][1].record()
        decode_all()
        ev[k][2].record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - wall0
    clk = clocks.stop()
    total_ms = ev[0][0].elapsed_time(ev[-1][2])
    enc_ms = sum(e[0].elapsed_time(e[1]) for e in ev)
    dec_ms = sum(e[1].elapsed_time(e[2]) for e in ev)
    if world > 1:
        tt = torch.tensor([total_ms, enc_ms, dec_ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms, enc_ms, dec_ms = (float(x) for x in tt.tolist())
    for t in tensors:
        t["codec"].check(decoding=True)

    # compressed sizes: the only cross-rank exchange (wire offsets per rank)
    comp_rank = sum(t["blob"].payload_nbytes() + t["blob"].metadata.numel() + t["blob"].framing_nbytes for t in tensors)
    if world > 1:
        sizes = torch.zeros(world, dtype=torch.int64, device=dev)
        dist.all_gather_into_tensor(sizes, torch.tensor([comp_rank], dtype=torch.int64, device=dev))
        all_sizes = sizes.tolist()
    else:
        all_sizes = [comp_rank]
    cr = V_rank / sum(t["blob"].compressed_nbytes for t in tensors)
    cr_wire = V_rank / comp_rank

    # quality of the round trip (reference quality_score, tensors.py:115-134),
    # squared sums from the fused kvc_sq_error kernel, per layer
    qual = []
    for t in tensors:
        se = torch.zeros((), dtype=torch.float64, device=dev)
        sx = torch.zeros((), dtype=torch.float64, device=dev)
        for li in range(L):
            if paged:
                pg = t["out"].view(L, -1, paged["page_tokens"], H, C)[li, paged["table"].long()]
                rec = pg.reshape(T, H, C).permute(1, 0, 2).contiguous()
            else:
                rec = t["out"][li]
            x = t["kv"][li]
            N.check(N.lib().kvc_sq_error(x.data_ptr(), rec.data_ptr(), x.numel(), N.DTYPE_BF16, se.data_ptr(), None))
            N.check(N.lib().kvc_sq_error(x.data_ptr(), None, x.numel(), N.DTYPE_BF16, sx.data_ptr(), None))
        rmse, rms = math.sqrt(float(se) / E), math.sqrt(float(sx) / E)
        qual.append(max(0.0, 1.0 - rmse / rms) if rmse > 1e-9 else 1.0)

    step_ms = total_ms / steps
    V_all = world * V_rank if not wl["shard"] else 2 * math.prod(wl["shape"]) * len(tensors)

    # paged workloads: compress straight from the paged cache too (the
    # connector's prefill side, kvc_encode_paged), timed like encode_all
    paged_enc = None
    if paged:
        def encode_paged_all():
            _fork()
            for t in tensors:
                t["codec"].encode_paged(t["out"], paged["table"], paged["page_tokens"], paged["layer_stride"],
                                        out=t["blob"], stream=t["stream"])
            _join()

        encode_paged_all()
        torch.cuda.synchronize()
        pe = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        for k in range(steps):
            pe[k][0].record()
            encode_paged_all()
            pe[k][1].record()
        torch.cuda.synchronize()
        pms = sum(a_.elapsed_time(b_) for a_, b_ in pe) / steps
        if world > 1:
            tt = torch.tensor([pms], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            pms = float(tt.item())
        for t in tensors:
            t["codec"].check()
        paged_enc = {"compress_gbs": round(V_all / (pms * 1e-3) / 1e9, 3), "ms_per_step": round(pms, 4),
                     "contiguous_compress_ms_per_step": round(enc_ms / steps, 4),
                     "page_tokens": paged["page_tokens"],
                     "source": "the decoded paged cache (random page table), kvc_encode_paged"}
    value = V_all / (step_ms * 1e-3) / 1e9
    enc_gbs = V_all / (enc_ms / steps * 1e-3) / 1e9
    dec_gbs = V_all / (dec_ms / steps * 1e-3) / 1e9

    # ---------------- per-kernel times (dominant kernel roofline)
    N.profile_enable(True)
    prof_steps = 2
    saved = [t["stream"] for t in tensors]
    for t in tensors:  # per-kernel event times are only meaningful serialised
        t["stream"] = main
    for _ in range(prof_steps):
        encode_all()
        decode_all()
    prof = N.profile_collect()
    for t, s_ in zip(tensors, saved):
        t["stream"] = s_
    N.profile_enable(False)
    launches_per_step = sum(c for _, c in prof.values()) / prof_steps
    alg = {}  # algorithmic bytes per launch for each kernel family
    for t in tensors:
        w, g = _bits_group(t["sid"])
        packed = E * w // 8
        meta = t["blob"].metadata.numel()
        coded = t["blob"].payload_nbytes()
        for k in ("encode_generic", "encode_fast128", "encode_uchan", "decode_generic", "decode_fast128",
                  "decode_uchan", "decode_delta"):
            alg.setdefault(k, []).append(2 * E + packed + meta)
        for k in ("rc_encode", "rc_decode", "rle_encode", "rle_decode"):
            alg.setdefault(k, []).append(packed + coded)
        alg.setdefault("gather", []).append(2 * coded)
        alg.setdefault("fused_encode", []).append(2 * E + coded + meta)
        alg.setdefault("fused_decode", []).append(2 * E + coded + meta)
    dom_name, (dom_ms, dom_n) = max(prof.items(), key=lambda kv: kv[1][0])
    per_launch_ms = dom_ms / dom_n
    roofline = None
    if alg.get(dom_name):
        per_launch_bytes = sum(alg[dom_name]) / len(alg[dom_name])
        achieved = per_launch_bytes / (per_launch_ms * 1e-3) / 1e9
        evd = _ncu_evidence(workload, dom_name)
        roofline = {"bound": "hbm", "kernel": dom_name, "achieved": round(achieved, 2), "peak": hbm_peak,
                    "unit": "GB/s", "frac": round(achieved / hbm_peak, 4),
                    "traffic": round(evd["dram_bytes"]) if evd else None,
                    "peak_source": peak_src, "launch_ms": round(per_launch_ms, 4),
                    "algorithmic_bytes_per_launch": int(per_launch_bytes),
                    "share_of_step": round(dom_ms / prof_steps / step_ms, 3)}
        if evd:
            # instruction roofline: warp-instructions per launch (same capture)
            # over this run's launch time, against 4 issue slots per SM per cycle
            roofline["traffic_source"] = evd["source"]
            roofline["issue"] = {"warp_inst_per_launch": round(evd["inst"]),
                                 "achieved_tinst_s": round(evd["inst"] / (per_launch_ms * 1e-3) / 1e12, 3),
                                 "ncu_issue_active_pct": round(evd["issue_pct"], 1)}
            mhz = (clk or {}).get("sm_mhz") or (clk or {}).get("sm_max_mhz")
            if mhz:
                sms = torch.cuda.get_device_properties(dev).multi_processor_count
                peak_i = sms * 4 * mhz * 1e6
                roofline["issue"]["peak_tinst_s"] = round(peak_i / 1e12, 3)
                roofline["issue"]["frac"] = round(evd["inst"] / (per_launch_ms * 1e-3) / peak_i, 4)
    step_alg = 2 * sum(2 * E + t["blob"].compressed_nbytes for t in tensors)
    kernels = {k: {"ms_per_step": round(v[0] / prof_steps, 4), "launches_per_step": v[1] / prof_steps}
               for k, v in prof.items()}

    # ---------------- end-to-end through the public API with host buffers
    e2e = None
    if do_e2e:
        for t in tensors:  # free the device-resident blobs first (a c3 rank holds 13 GB of them)
            t["blob"] = None
        torch.cuda.empty_cache()
        e2e = measure_e2e(tensors, paged, steps, world, dev, V_all)

    res = {
        "value": round(value, 3), "unit": "GB/s", "ms_per_step": round(step_ms, 4), "steps": steps,
        "config": config_of(workload, world),
        "shape_per_rank": list(shape),
        "compress_gbs": round(enc_gbs, 3), "decompress_gbs": round(dec_gbs, 3),
        "compress_hbm_frac": round(enc_gbs * (1 + 1 / cr) / world / hbm_peak, 4),  # per GPU
        "decompress_hbm_frac": round(dec_gbs * (1 + 1 / cr) / world / hbm_peak, 4),
        "cr": round(cr, 4), "cr_wire": round(cr_wire, 4), "quality": [round(q, 6) for q in qual],
        "step_hbm_frac": round(step_alg / (step_ms * 1e-3) / 1e9 / hbm_peak, 4),
        "roofline": roofline, "kernels": kernels, "gpu_launches": int(round(launches_per_step * steps)),
        "cpu_baseline": cpu, "e2e": e2e, "clocks": clk, "rank_compressed_bytes": all_sizes,
        "paged_encode": paged_enc,
        "wall_s": round(wall, 3),
    }
    del tensors
    torch.cuda.empty_cache()
    return res


def run_sweep(args, steps: int, rank: int, world: int, dev, hbm_peak: float) -> dict:
    """c4: the round trip of every mixed-precision profile (K and V, one
    stream each) on the same synthetic 8B 16K cache; value = all profiles'
    bf16-in bytes / their summed step time (per-profile numbers alongside)."""
    import torch

    from paper_2605_13734_b200 import KVCodec
    from paper_2605_13734_b200 import _native as N
    from paper_2605_13734_b200.pipeline import classify_heads, layer_classes
    from paper_2605_13734_b200.synth import synthetic_kv

    L, H, T, C = C4_SHAPE
    E = L * H * T * C
    kvs = []
    for ti in range(2):
        kv, imp = synthetic_kv(L, H, T, C, seed=4000 + 1000 * rank + ti, device=dev)
        kvs.append((kv, imp, torch.empty_like(kv)))
    main = torch.cuda.current_stream()
    streams = [torch.cuda.Stream(device=dev) for _ in kvs]
    rows, tot_bytes, tot_ms = [], 0, 0.0
    for sid in c4_ids():
        codecs, blobs, cls = [], [], []
        for kv, imp, _ in kvs:
            c = KVCodec(sid, C4_SHAPE, block_symbols=BLOCK, device=dev)
            q = sid.split(";")[1]
            k = classify_heads(imp, 0.25) if q.startswith("q=mixed") else (
                layer_classes(imp, 0.25) if q.startswith("q=mixlayer") else None)
            codecs.append(c)
            cls.append(k)
            blobs.append(c.alloc_blob(k))

        def step():
            e = torch.cuda.Event()
            e.record(main)
            for st, c, (kv, _, out), b, k in zip(streams, codecs, kvs, blobs, cls):
                st.wait_event(e)
                c.encode(kv, head_classes=k, out=b, stream=st)
                c.decode(b, out=out, device_length=True, stream=st)
            for st in streams:
                f = torch.cuda.Event()
                f.record(st)
                main.wait_event(f)

        step()
        for c in codecs:
            c.check(decoding=True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            step()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        comp = sum(b.compressed_nbytes for b in blobs)
        qual = []
        for (kv, _, out) in kvs:
            se = torch.zeros((), dtype=torch.float64, device=dev)
            sx = torch.zeros((), dtype=torch.float64, device=dev)
            N.check(N.lib().kvc_sq_error(kv.data_ptr(), out.data_ptr(), E, N.DTYPE_BF16, se.data_ptr(), None))
            N.check(N.lib().kvc_sq_error(kv.data_ptr(), None, E, N.DTYPE_BF16, sx.data_ptr(), None))
            rmse, rms = math.sqrt(float(se) / E), math.sqrt(float(sx) / E)
            qual.append(max(0.0, 1.0 - rmse / rms) if rmse > 1e-9 else 1.0)
        V = 2 * E * len(kvs)
        rows.append({"id": sid, "gbs": round(V / (ms * 1e-3) / 1e9, 1), "cr": round(V / comp, 4),
                     "quality": round(sum(qual) / len(qual), 6)})
        tot_bytes += V
        tot_ms += ms
        del codecs, blobs
    gbs = sorted(r["gbs"] for r in rows)
    return {"value": round(tot_bytes / (tot_ms * 1e-3) / 1e9, 3), "unit": "GB/s", "steps": steps,
            "ms_per_step": round(tot_ms, 4), "config": {"workload": "c4", "shape": list(C4_SHAPE),
                                                        "profiles": len(rows), "rho": 0.25},
            "median_profile_gbs": gbs[len(gbs) // 2], "min_profile_gbs": gbs[0], "max_profile_gbs": gbs[-1],
            "profiles": rows}


def measure_e2e(tensors, paged, steps, world, dev, V_all) -> dict:
    """Same metric end to end through the public API (hostpath.HostRoundTrip):
    pinned host KV -> H2D -> encode -> decode (contiguous or paged) -> D2H of
    the step's scalar result, pipelined by layer chunks across copy engines,
    PCIe and SMs; the blob stays in HBM as in the reference's compress().
    "wire_via_host" repeats it with the compressed wire shipped to pinned host
    memory and back between encode and decode (a network hop's PCIe cost)."""
    import torch
    import torch.distributed as dist

    from paper_2605_13734_b200.hostpath import HostRoundTrip

    host_in = []
    for t in tensors:
        h = torch.empty(t["kv"].shape, dtype=t["kv"].dtype, pin_memory=True)
        h.copy_(t["kv"])
        host_in.append(h)
    L_rank = tensors[0]["kv"].shape[0]
    chunk = max(1, min(8, L_rank // 4)) if L_rank >= 4 else L_rank
    pg = None if paged is None else (paged["table"], paged["page_tokens"], paged["layer_stride"])
    out = {}
    for via_host in (False, True):
        rts = [HostRoundTrip(t["sid"], tuple(t["kv"].shape), chunk_layers=chunk, block_symbols=BLOCK, device=dev,
                             paged=pg, wire_via_host=via_host) for t in tensors]
        ms = _time_e2e(rts, host_in, tensors, steps, world, dev)
        wire = sum(rt.wire_bytes() for rt in rts)
        h2d = sum(h.numel() * 2 for h in host_in) + (wire if via_host else 0)
        d2h = (wire if via_host else 0) + 8
        res_kind = "squared reconstruction error (fp64 scalar)" if paged is None else "compressed bytes (paged decode)"
        path = ("pinned host KV -> H2D -> encode -> wire to pinned host -> H2D -> decode" if via_host else
                "pinned host KV -> H2D -> encode -> decode (blob stays in HBM, as in compress())")
        r = {"value": round(V_all / (ms * 1e-3) / 1e9, 3), "unit": "GB/s", "h2d_bytes_per_step": int(h2d),
             "d2h_bytes_per_step": int(d2h), "ms_per_step": round(ms, 3), "steps": max(1, min(3, steps)),
             "chunk_layers": chunk,
             "path": f"{path} -> D2H of the {res_kind} (hostpath.HostRoundTrip, layer-chunk pipeline)"}
        if via_host:
            out["wire_via_host"] = r
        else:
            out.update(r)
        del rts
    del host_in
    return out


def _time_e2e(rts, host_in, tensors, steps, world, dev) -> float:
    import torch
    import torch.distributed as dist

    result = torch.zeros((), dtype=torch.float64, device=dev)

    def e2e_step():
        result.zero_()
        # the H2D lands in the kv buffers themselves (identical values): no second 42 GB device copy
        for rt, h, t in zip(rts, host_in, tensors):
            rt.run(h, t["kv"], t["out"], result)
        return result.item()  # D2H of the step's result (syncs)

    e2e_step()  # warm-up (plans, pinned buffers)
    for rt in rts:
        rt.check()
    n = max(1, min(3, steps))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    s0 = torch.cuda.Event(enable_timing=True)
    s1 = torch.cuda.Event(enable_timing=True)
    s0.record()
    for _ in range(n):
        e2e_step()
    s1.record()
    torch.cuda.synchronize()
    ms = s0.elapsed_time(s1) / n
    if world > 1:
        tt = torch.tensor([ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    return ms


def main():
    args = _args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return reference_arm(args, rank, world)

    extras = [] if (args.no_extras or world > 1 or args.workload != "c3") else list(EXTRAS)
    # CPU baselines first (the worker pools fork before any CUDA context exists)
    cpus = {}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpus[args.workload] = cpu_measure(args.workload, 2, 1)
        for w in extras:
            if w == "c5":
                cpus[w] = cpu_measure(w, 1, 0)

    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)" if "hbm_gbs" in peaks else "fallback (B200_PROFILING.md)"

    def strip(c):
        return None if c is None else {k: c[k] for k in ("value", "unit", "cores", "kind", "sample")}

    head = run_workload(args.workload, args, args.steps, rank, world, dev, not args.no_e2e,
                        strip(cpus.get(args.workload)), hbm_peak, peak_src)
    extra = {}
    for w in extras:
        if w == "c4":
            extra[w] = run_sweep(args, 3, rank, world, dev, hbm_peak)
            continue
        extra[w] = run_workload(w, args, EXTRA_STEPS, rank, world, dev, (w == "c5") and not args.no_e2e,
                                strip(cpus.get(w)), hbm_peak, peak_src)

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": head["value"],
            "unit": "GB/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": head["ms_per_step"],
            "higher_is_better": True,
            "scaling": "strong" if WORKLOADS[args.workload]["shard"] else "weak",
            "vs_baseline": None,
            "dtype": "bf16 in/out; fp64 Hadamard butterfly, fp32 quantizer, u32 range coder",
            "data": "synthetic (reference generator distribution, rounded to bf16), generated on the device",
            "config": head["config"],
        }
        for k in ("shape_per_rank", "compress_gbs", "decompress_gbs", "compress_hbm_frac", "decompress_hbm_frac", "cr",
                  "cr_wire", "quality", "step_hbm_frac", "roofline", "kernels", "gpu_launches", "cpu_baseline", "e2e",
                  "clocks", "rank_compressed_bytes", "wall_s"):
            line[k] = head[k]
        if head.get("paged_encode"):
            line["paged_encode"] = head["paged_encode"]
        if extra:
            line["extra"] = {w: {k: v for k, v in r.items()} for w, r in extra.items()}
        emit(line)
    if world > 1:
        dist.destroy_process_group()


# stdout carries exactly the one JSON line: every other write to fd 1 (NCCL's
# version banner, library chatter from C code) is sent to stderr
_JSON_OUT = None


def emit(line: dict) -> None:
    out = _JSON_OUT if _JSON_OUT is not None else sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


if __name__ == "__main__":
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    main()
