"""Per-kernel opcode mix from an ncu --page source CSV (gzip ok), normalised
to instructions per coded symbol when --per N (warp-level units) is given.

    python tools/ncu_ops.py gpurun_out/p_x_source.csv.gz [--per 33554432]
"""
import collections
import csv
import gzip
import sys

path = sys.argv[1]
per = float(sys.argv[sys.argv.index("--per") + 1]) if "--per" in sys.argv else None
op = gzip.open if path.endswith(".gz") else open
data = op(path, "rt").read().splitlines()
secs = [i for i, l in enumerate(data) if l.startswith('"Kernel Name"')] + [len(data)]
seen = set()
for a, b in zip(secs[:-1], secs[1:]):
    name = data[a].split(",", 1)[1][:70]
    if name in seen:
        continue
    seen.add(name)
    rows = list(csv.reader(data[a + 1:b]))
    hdr = rows[0]
    ie, src = hdr.index("Instructions Executed"), hdr.index("Source")
    st = hdr.index("Warp Stall Sampling (All Samples)")
    ops, stall = collections.Counter(), collections.Counter()
    tot = 0.0
    for r in rows[1:]:
        try:
            n = float(r[ie])
        except ValueError:
            continue
        t = r[src].split()
        if not t:
            continue
        o = ("@" + t[1]) if t[0].startswith("@") else t[0]
        ops[o] += n
        tot += n
        try:
            stall[o] += float(r[st])
        except ValueError:
            pass
    scale = (1.0 / per) if per else (100.0 / tot)
    print(f"{name}  total {tot:.4g}" + (f"  per unit {tot / per:.1f}" if per else ""))
    print("   " + ", ".join(f"{k}:{v * scale:.2f}" for k, v in ops.most_common(30)))
    st_tot = sum(stall.values()) or 1
    print("   stall samples by opcode: " + ", ".join(f"{k}:{v / st_tot * 100:.0f}%" for k, v in stall.most_common(8)))
