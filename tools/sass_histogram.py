"""Static SASS opcode histogram per kernel of libkvc.so (cuobjdump -sass):

    python tools/sass_histogram.py [regex ...] > profiles/r2/sass_histograms.md

For each kernel whose mangled name matches a regex: instruction count and
the opcodes that prove the Blackwell data paths -- UTMALDG / UTMASTG (TMA
tensor load / store), UBLKCP (cp.async.bulk), SYNCS (mbarrier), UTC*MMA /
LDTM (tcgen05) -- followed by the top opcodes.
"""

from __future__ import annotations

import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2605_13734_b200", "libkvc.so")
MARK = ("UTMALDG", "UTMASTG", "UBLKCP", "SYNCS", "UTCHMMA", "UTCQMMA", "UTCIMMA", "LDTM", "STTM", "FFMA2", "FADD2",
        "FMUL2", "DADD", "DFMA", "SHFL")


def demangle(names):
    r = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True)
    return r.stdout.splitlines() if r.returncode == 0 else names


def main() -> None:
    pats = [re.compile(p) for p in (sys.argv[1:] or ["k_enc128", "k_dec128r", "k_fused_", "k_enc_uchan", "k_rc_"])]
    txt = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    funcs = {}
    cur = None
    for line in txt.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = collections.Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
        if cur and m:
            funcs[cur][m.group(2).split(".")[0]] += 1
    names = [n for n in funcs if any(p.search(n) for p in pats)]
    print("# Static SASS opcode histograms (cuobjdump -sass of libkvc.so, sm_100a)\n")
    print("Counts are static instructions in the kernel body (not executed counts).\n")
    for raw, pretty in zip(names, demangle(names)):
        c = funcs[raw]
        marks = ", ".join(f"{k} {c[k]}" for k in MARK if c[k])
        top = ", ".join(f"{k} {v}" for k, v in c.most_common(12))
        print(f"## `{pretty}`\n\n- instructions: {sum(c.values())}\n- data-path opcodes: {marks or '-'}\n- top: {top}\n")


if __name__ == "__main__":
    main()
