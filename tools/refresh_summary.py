"""Install a run_round_measure.sh output directory into profiles/r1/ and
regenerate the bench and ncu tables of profiles/r1_summary.md.

    python tools/refresh_summary.py gpurun_out
"""

from __future__ import annotations

import json
import shutil
import subprocess
import sys

SUMMARY = "profiles/r1_summary.md"
HBM_PEAK = 6372.5


def install(src: str) -> None:
    for w in ("c1", "c2", "c3", "c5", "ref_c2"):
        shutil.copy(f"{src}/bench_{w}.json", f"profiles/r1/bench_{w}.json")
    shutil.copy(f"{src}/launches_c2.csv", "profiles/r1/launches_c2.csv")
    for w in ("c1", "c2", "c5"):
        shutil.copy(f"{src}/prof_{w}_raw.csv", f"profiles/r1/ncu_full_{w}_raw.csv")


def _table(kind: str, path: str) -> str:
    return subprocess.run([sys.executable, "tools/summarize_ncu.py", kind, path],
                          capture_output=True, text=True, check=True).stdout.strip()


def _section(s: str, head: str, body: str) -> str:
    i = s.index(head)
    j = s.index("\n## ", i + len(head))
    return s[:i] + head + "\n\n" + body + "\n" + s[j:]


def _f(x: float) -> str:
    return f"{x:.1f}" if x >= 10 else f"{x:.3f}"


def regenerate() -> None:
    s = open(SUMMARY).read()
    s = _section(s, "## C2 — launch list (serialised cold-cache, `--streams 0`)",
                 _table("launches", "profiles/r1/launches_c2.csv"))
    s = _section(s, "## C2 — full captures", _table("raw", "profiles/r1/ncu_full_c2_raw.csv"))
    s = _section(s, "## C1 — Hadamard encode + decode", _table("raw", "profiles/r1/ncu_full_c1_raw.csv"))
    s = _section(s, "## C5 — 8-bit entropy path", _table("raw", "profiles/r1/ncu_full_c5_raw.csv"))
    b = {w: json.load(open(f"profiles/r1/bench_{w}.json")) for w in ("c1", "c2", "c3", "c5", "ref_c2")}
    c1, c2, c3, c5 = b["c1"], b["c2"], b["c3"], b["c5"]
    rows = [
        f"| c2 (headline) | {_f(c2['value'])} | {c2['compress_gbs']:.0f} / {c2['decompress_gbs']:.0f} | {c2['cr']:.2f} "
        f"| fused_encode {c2['roofline']['frac']:.2f}; issue {c2['roofline']['issue']['frac']:.2f} "
        f"| {c2['cpu_baseline']['value']:.3f} GB/s; `--impl reference` {b['ref_c2']['value']:.3f} GB/s "
        f"| {c2['e2e']['value']:.1f} GB/s |",
        f"| c1 | {_f(c1['value'])} | {c1['compress_gbs']:.0f} / {c1['decompress_gbs']:.0f} | {c1['cr']:.2f} "
        f"| encode_fast128 (Hadamard) {c1['roofline']['frac']:.2f}; issue {c1['roofline']['issue']['frac']:.2f} "
        f"| {c1['cpu_baseline']['value']:.3f} GB/s | {c1['e2e']['value']:.1f} GB/s |",
        f"| c3 (1 GPU, 70B 128K) | {_f(c3['value'])} | {c3['compress_gbs']:.0f} / {c3['decompress_gbs']:.0f} "
        f"| {c3['cr']:.2f} | encode_fast128 {c3['roofline']['frac']:.2f} "
        f"(decode: {c3['decompress_gbs'] * (1 + 1 / c3['cr']) / HBM_PEAK:.2f}) | — | — |",
        f"| c5 (paged) | {_f(c5['value'])} | {c5['compress_gbs']:.0f} / {c5['decompress_gbs']:.0f} | {c5['cr']:.2f} "
        f"| rc_decode {c5['roofline']['frac']:.3f}; issue {c5['roofline']['issue']['frac']:.2f} | — | — |",
    ]
    i = s.index("| c2 (headline) |")
    j = s.index("\n\n", i)
    s = s[:i] + "\n".join(rows) + s[j:]
    open(SUMMARY, "w").write(s)
    print("\n".join(rows))


if __name__ == "__main__":
    if len(sys.argv) > 1:
        install(sys.argv[1])
    regenerate()
