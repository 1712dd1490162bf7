"""Benchmark of the KV compress/decompress hot path (BASELINE.json metric:
"KV compress/decompress GB/s (bf16-in) per B200 & 8-GPU, at compression ratio").

One step = the reference's compress() round trip (compress.py:111-140) for
every KV tensor of the workload: encode (transform -> quantize -> lossless
codec) then decode (codec -> dequantize -> inverse transform) back to bf16,
inputs and outputs resident in HBM.  `value` is bf16-in GB/s of that round
trip, V / (t_enc + t_dec) — the reference's s_p (compress.py:32-40) — summed
over ranks; compress and decompress GB/s are reported separately.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2|c1|c3|c5] [--impl ours|reference]

Workloads (BASELINE.json configs; c2 = configs[1] is the default headline):
  c1  Llama-3.1-8B 4K   (32,8,4096,128)   K,V: t=hadamard;q=uniform,b=4,g=32;c=none
  c2  Llama-3.1-8B 32K  (32,8,32768,128)  K: t=identity;q=uchan,b=2,g=32;c=entropy (KIVI per-channel)
                                           V: t=identity;q=uniform,b=2,g=32;c=entropy (per-token)
  c3  Llama-3.1-70B 128K (80,8,128000,128) K,V: C1 profile, layers sharded over ranks (strong scaling)
  c5  Qwen3-8B 16K      (36,8,16384,128)  K,V: t=affine;q=uniform,b=8,g=32;c=entropy, decoded into paged KV
Multi-GPU: torchrun, one process per GPU; no collective on the data path —
only the per-rank compressed sizes are all-gathered (offsets for the wire).
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

C1_PROFILE = "t=hadamard;q=uniform,b=4,g=32;c=none"
WORKLOADS = {
    "c1": dict(name="Llama-3.1-8B KV 4K tokens, reference default profile", shape=(32, 8, 4096, 128),
               tensors=[("K", C1_PROFILE), ("V", C1_PROFILE)], shard=False, paged=False),
    "c2": dict(name="Llama-3.1-8B KV 32K tokens, KIVI 2-bit per-channel K / per-token V + entropy",
               shape=(32, 8, 32768, 128),
               tensors=[("K", "t=identity;q=uchan,b=2,g=32;c=entropy"), ("V", "t=identity;q=uniform,b=2,g=32;c=entropy")],
               shard=False, paged=False),
    "c3": dict(name="Llama-3.1-70B KV 128K tokens, layer-sharded", shape=(80, 8, 128000, 128),
               tensors=[("K", C1_PROFILE), ("V", C1_PROFILE)], shard=True, paged=False),
    "c5": dict(name="Qwen3-8B GQA KV 16K tokens, affine + 8-bit + entropy, paged decode", shape=(36, 8, 16384, 128),
               tensors=[("K", "t=affine;q=uniform,b=8,g=32;c=entropy"), ("V", "t=affine;q=uniform,b=8,g=32;c=entropy")],
               shard=False, paged=True),
}
BLOCK = 2048


def _args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--block", type=int, default=None, help="codec block symbols (default 2048)")
    p.add_argument("--streams", type=int, default=1, help="1: one CUDA stream per KV tensor (default); 0: serial")
    args = p.parse_args()
    global BLOCK
    if args.block:
        BLOCK = args.block
    return args


def _shard_shape(wl, rank, world):
    L, H, T, C = wl["shape"]
    if not wl["shard"]:
        return (L, H, T, C), (0, L)
    per = [L // world + (1 if r < L % world else 0) for r in range(world)]
    l0 = sum(per[:rank])
    return (per[rank], H, T, C), (l0, l0 + per[rank])


# ----------------------------------------------------------------------------
# CPU side: the oracle (CPU restatement of the reference) on host cores
# ----------------------------------------------------------------------------

def _oracle_slab(job):
    """Round trip of one (1 layer, 1 head) slab through the oracle; returns
    (bf16 bytes, seconds).  Runs in a worker process."""
    import numpy as np

    import oracle

    sid, tokens, channels, seed = job
    v, imp = oracle.generate_kv(1, 1, tokens, channels, seed=seed)
    u = v.view(np.uint32).astype(np.uint64)
    v = ((((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16).astype(np.uint32)).view(np.float32)  # bf16-exact
    t0 = time.perf_counter()
    ob = oracle.encode_blob(v, imp, sid, block=BLOCK)
    oracle.decode_blob(ob["payload"], ob["metadata"], ob["offsets"], sid, v.shape, block=BLOCK)
    return v.size * 2, time.perf_counter() - t0


def cpu_roundtrip(wl, n_slabs, procs, seed0=1000):
    """bf16-in GB/s of the oracle round trip over `n_slabs` head slabs."""
    import multiprocessing as mp

    _, H, T, C = wl["shape"]
    tok = min(T, 8192)
    jobs = [(wl["tensors"][i % len(wl["tensors"])][1], tok, C, seed0 + i) for i in range(n_slabs)]
    ctx = mp.get_context("fork")
    t0 = time.perf_counter()
    with ctx.Pool(procs) as pool:
        res = pool.map(_oracle_slab, jobs, chunksize=1)
    wall = time.perf_counter() - t0
    nbytes = sum(r[0] for r in res)
    return nbytes / wall / 1e9, nbytes, wall, tok


def reference_arm(args, wl, rank):
    """--impl reference: the oracle port of the reference pipeline on all host cores."""
    if rank != 0:
        return
    procs = len(os.sched_getaffinity(0))
    for _ in range(max(args.warmup, 0) and 1):
        cpu_roundtrip(wl, procs, procs, seed0=1)
    vals, total_bytes, total_wall = [], 0, 0.0
    tok = None
    for k in range(args.steps):
        gbs, nb, wall, tok = cpu_roundtrip(wl, procs, procs, seed0=100 + k * procs)
        vals.append(gbs)
        total_bytes += nb
        total_wall += wall
    value = total_bytes / total_wall / 1e9
    sample = f"{procs} head slabs x {tok} tokens x {wl['shape'][3]} ch per step ({procs} processes), bf16-exact synthetic"
    line = {
        "impl": "reference", "metric": "KV compress+decompress round-trip GB/s (bf16-in)", "value": round(value, 6),
        "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * total_wall / args.steps, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32/f64 (numpy) + u32 (C range coder)", "data": "synthetic",
        "config": {"workload": args.workload, "name": wl["name"], "tensors": dict(wl["tensors"]),
                   "shape": list(wl["shape"]), "block_symbols": BLOCK},
        "cpu_baseline": {"value": round(value, 6), "unit": "GB/s", "cores": procs, "kind": "port", "sample": sample},
        "e2e": {"value": round(value, 6), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
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

def main():
    args = _args()
    wl = WORKLOADS[args.workload]
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return reference_arm(args, wl, rank)

    # CPU baseline first (fork before any CUDA context exists)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        procs = len(os.sched_getaffinity(0))
        gbs, nb, wall, tok = cpu_roundtrip(wl, 4 * procs, procs)
        cpu = {"value": round(gbs, 6), "unit": "GB/s", "cores": procs, "kind": "port",
               "sample": f"{4 * procs} head slabs x {tok} tokens x {wl['shape'][3]} ch of this workload's strategies, "
                         f"oracle round trip on {procs} processes ({wall:.1f} s wall)"}

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2605_13734_b200 import KVCodec
    from paper_2605_13734_b200 import _native as N
    from paper_2605_13734_b200.synth import synthetic_kv

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        # keep stdout to the one JSON line (NCCL prints a version banner at VERSION level)
        if os.environ.get("NCCL_DEBUG", "VERSION").upper() == "VERSION":
            os.environ["NCCL_DEBUG"] = "WARN"
        dist.init_process_group("nccl", device_id=dev)
    shape, (l0, l1) = _shard_shape(wl, rank, world)
    L, H, T, C = shape
    E = L * H * T * C

    tensors = []
    for ti, (name, sid) in enumerate(wl["tensors"]):
        kv, imp = synthetic_kv(L, H, T, C, seed=1000 * rank + 17 * ti + l0, device=dev)
        codec = KVCodec(sid, shape, block_symbols=BLOCK, device=dev)
        blob = codec.alloc_blob()
        # a 70B 128K cache on one GPU: K, V (2 x 39 GiB) + payloads leave room
        # for one decode target only -> the tensors share it (serial streams)
        share = wl["shard"] and world == 1
        out = tensors[0]["out"] if (share and tensors) else torch.empty_like(kv)
        tensors.append(dict(name=name, sid=sid, kv=kv, codec=codec, blob=blob, out=out))
    if wl["shard"] and world == 1:
        args.streams = 0
    torch.cuda.synchronize()
    V_rank = 2 * E * len(tensors)  # bf16-in bytes per step on this rank

    paged = None
    if wl["paged"]:
        page_tokens = 16
        n_pages = T // page_tokens
        perm = torch.randperm(n_pages, device=dev).to(torch.int32)
        paged = dict(page_tokens=page_tokens, table=perm, layer_stride=n_pages * page_tokens * H * C)
        for t in tensors:
            t["out"] = torch.empty(L * n_pages * page_tokens * H * C, dtype=torch.bfloat16, device=dev)

    # K and V are independent: each runs on its own stream so the HBM-bound
    # quantize kernels of one overlap the issue-bound range coder of the other
    main = torch.cuda.current_stream()
    for t in tensors:
        t["stream"] = torch.cuda.Stream(device=dev) if args.streams else main

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
                                        stream=t["stream"])
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
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    clocks = ClockSampler(local)
    time.sleep(0.3)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    wall0 = time.perf_counter()
    for k in range(args.steps):
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
    comp = []
    for t in tensors:
        b = t["blob"]
        comp.append(b.payload_nbytes() + b.metadata.numel() + b.framing_nbytes)
    comp_rank = sum(comp)
    if world > 1:
        sizes = torch.zeros(world, dtype=torch.int64, device=dev)
        dist.all_gather_into_tensor(sizes, torch.tensor([comp_rank], dtype=torch.int64, device=dev))
        all_sizes = sizes.tolist()
    else:
        all_sizes = [comp_rank]
    cr = sum(2 * E for _ in tensors) / sum(t["blob"].compressed_nbytes for t in tensors)
    cr_wire = V_rank / comp_rank

    # quality of the round trip (reference quality_score, tensors.py:115-134)
    qual = []
    for t in tensors:
        if t["out"] is tensors[0]["out"] and t is not tensors[0]:
            t["codec"].decode(t["blob"], out=t["out"], device_length=True)  # shared decode target
        elif t is tensors[0] and len(tensors) > 1 and tensors[1]["out"] is t["out"]:
            t["codec"].decode(t["blob"], out=t["out"], device_length=True)
        se = sx = 0.0
        for li in range(L):  # per layer: no full-size fp32 temporaries
            if paged:
                pg = t["out"].view(L, -1, paged["page_tokens"], H, C)[li, paged["table"].long()]
                rec = pg.reshape(T, H, C).permute(1, 0, 2).double()
            else:
                rec = t["out"][li].double()
            x = t["kv"][li].double()
            se += float(((x - rec) ** 2).sum())
            sx += float((x * x).sum())
        rmse, rms = math.sqrt(se / E), math.sqrt(sx / E)
        qual.append(max(0.0, 1.0 - rmse / rms) if rmse > 1e-9 else 1.0)

    step_ms = total_ms / args.steps
    value = world * V_rank / (step_ms * 1e-3) / 1e9 if not wl["shard"] else 2 * math.prod(wl["shape"]) * len(tensors) / (step_ms * 1e-3) / 1e9
    enc_gbs = world * V_rank / (enc_ms / args.steps * 1e-3) / 1e9
    dec_gbs = world * V_rank / (dec_ms / args.steps * 1e-3) / 1e9

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
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "measured" if "hbm_gbs" in peaks else "fallback"
    # algorithmic bytes per launch for each kernel family
    alg = {}
    for t in tensors:
        s = t["sid"]
        w = int(s.split("b=")[1].split(",")[0]) if "b=" in s else 4
        g = int(s.split("g=")[1].split(",")[0].split(";")[0])
        packed = E * w // 8
        meta = t["blob"].metadata.numel()
        coded = t["blob"].payload_nbytes()
        for k in ("encode_generic", "encode_fast128", "encode_uchan"):
            alg.setdefault(k, []).append(2 * E + packed + meta)
        for k in ("decode_generic", "decode_fast128", "decode_uchan", "decode_delta"):
            alg.setdefault(k, []).append(2 * E + packed + meta)
        alg.setdefault("rc_encode", []).append(packed + coded)
        alg.setdefault("rc_decode", []).append(packed + coded)
        alg.setdefault("rle_encode", []).append(packed + coded)
        alg.setdefault("rle_decode", []).append(packed + coded)
        alg.setdefault("gather", []).append(2 * coded)
        # fused quantize + range code: bf16 in, coded blocks + metadata out (and the reverse)
        alg.setdefault("fused_encode", []).append(2 * E + coded + meta)
        alg.setdefault("fused_decode", []).append(2 * E + coded + meta)
    dom = max(prof.items(), key=lambda kv: kv[1][0])
    dom_name, (dom_ms, dom_n) = dom
    per_launch_ms = dom_ms / dom_n
    bytes_list = alg.get(dom_name)
    roofline = None
    if bytes_list:
        per_launch_bytes = sum(bytes_list) / len(bytes_list)
        achieved = per_launch_bytes / (per_launch_ms * 1e-3) / 1e9
        ev = _ncu_evidence(args.workload, dom_name)
        roofline = {"bound": "hbm", "kernel": dom_name, "achieved": round(achieved, 2), "peak": hbm_peak,
                    "unit": "GB/s", "frac": round(achieved / hbm_peak, 4),
                    "traffic": round(ev["dram_bytes"]) if ev else None,
                    "peak_source": peak_src, "launch_ms": round(per_launch_ms, 4),
                    "share_of_step": round(dom_ms / prof_steps / step_ms, 3)}
        if ev:
            # the serial range coders are instruction-bound: warp-instructions
            # per launch (same capture) over this run's launch time, against
            # 4 issue slots per SM per cycle at the measured SM clock
            roofline["traffic_source"] = ev["source"]
            roofline["issue"] = {"warp_inst_per_launch": round(ev["inst"]),
                                 "achieved_tinst_s": round(ev["inst"] / (per_launch_ms * 1e-3) / 1e12, 3),
                                 "ncu_issue_active_pct": round(ev["issue_pct"], 1)}
            mhz = (clk or {}).get("sm_mhz") or (clk or {}).get("sm_max_mhz")
            if mhz:
                sms = torch.cuda.get_device_properties(dev).multi_processor_count
                peak_i = sms * 4 * mhz * 1e6
                roofline["issue"]["peak_tinst_s"] = round(peak_i / 1e12, 3)
                roofline["issue"]["frac"] = round(ev["inst"] / (per_launch_ms * 1e-3) / peak_i, 4)
    step_alg = 2 * sum(2 * E + t["blob"].compressed_nbytes for t in tensors)
    kernels = {k: {"ms_per_step": round(v[0] / prof_steps, 4), "launches_per_step": v[1] / prof_steps} for k, v in prof.items()}

    # ---------------- end-to-end through the public API with host buffers
    # paper_2605_13734_b200.hostpath.HostRoundTrip: pinned host KV -> H2D ->
    # encode -> wire into pinned host memory -> H2D -> decode, pipelined by
    # layer chunks across copy engines / PCIe / SMs; the step's result is the
    # reconstruction squared error, read back to the host.
    e2e = None
    if not args.no_e2e and not paged:
        from paper_2605_13734_b200.hostpath import HostRoundTrip

        host_in = [t["kv"].cpu().pin_memory() for t in tensors]
        dev_in = [torch.empty_like(t["kv"]) for t in tensors]
        L_rank = tensors[0]["kv"].shape[0]
        chunk = max(1, min(8, L_rank // 4)) if L_rank >= 4 else L_rank
        rts = [HostRoundTrip(t["sid"], tuple(t["kv"].shape), chunk_layers=chunk, block_symbols=BLOCK, device=dev,
                             wire_bytes_hint=t["blob"].payload_nbytes()) for t in tensors]
        outs = [t["out"] for t in tensors]
        err = torch.zeros((), dtype=torch.float64, device=dev)

        def e2e_step():
            err.zero_()
            for rt, h, d_in, o in zip(rts, host_in, dev_in, outs):
                rt.run(h, d_in, o, err)
            return err.item()  # D2H of the step's result (syncs)

        e2e_step()  # warm-up (plans, pinned buffers)
        for rt in rts:
            rt.check()
        e2e_steps = max(1, min(3, args.steps))
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        s0.record()
        for _ in range(e2e_steps):
            e2e_step()
        s1.record()
        torch.cuda.synchronize()
        e2e_ms = s0.elapsed_time(s1) / e2e_steps
        wire = sum(rt.wire_bytes() for rt in rts)
        h2d = sum(h.numel() * 2 for h in host_in) + wire
        d2h = wire + 8
        if world > 1:
            tt = torch.tensor([e2e_ms], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e2e_ms = float(tt.item())
        e2e = {"value": round(world * V_rank / (e2e_ms * 1e-3) / 1e9, 3), "unit": "GB/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "ms_per_step": round(e2e_ms, 3),
               "chunk_layers": chunk,
               "path": "pinned host KV -> H2D -> encode -> wire to pinned host -> H2D -> decode -> D2H squared-error "
                       "scalar (hostpath.HostRoundTrip, layer-chunk pipeline)"}

    if rank == 0:
        line = {
            "metric": "KV compress+decompress round-trip GB/s (bf16-in), s_p = V/(t_enc+t_dec)",
            "value": round(value, 3),
            "unit": "GB/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(step_ms, 4),
            "higher_is_better": True,
            "scaling": "strong" if wl["shard"] else "weak",
            "vs_baseline": None,
            "dtype": "bf16 in/out; fp32/fp64 transform+quantizer, u32 range coder",
            "data": "synthetic (reference generator distribution, rounded to bf16)",
            "config": {"workload": args.workload, "name": wl["name"], "shape_per_rank": list(shape),
                       "tensors": dict(wl["tensors"]), "block_symbols": BLOCK,
                       "l2": "inputs larger than L2 (no flush needed)", "parallelism": f"dp{world} (independent shards)"},
            "compress_gbs": round(enc_gbs, 3),
            "decompress_gbs": round(dec_gbs, 3),
            "cr": round(cr, 4),
            "cr_wire": round(cr_wire, 4),
            "quality": [round(q, 6) for q in qual],
            "step_hbm_frac": round(step_alg / (step_ms * 1e-3) / 1e9 / hbm_peak, 4),
            "roofline": roofline,
            "kernels": kernels,
            "gpu_launches": int(round(launches_per_step * args.steps)),
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": clk,
            "rank_compressed_bytes": all_sizes,
            "wall_s": round(wall, 3),
        }
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
