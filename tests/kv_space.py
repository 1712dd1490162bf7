"""The reference's default strategy space (profiling/space.py:24-35, :120-160),
restated so GPU tests can enumerate all 180 ids without the reference."""

TRANSFORMS = ("identity", "delta", "hadamard")
BITS = (2, 3, 4, 8)
GROUPS = (32, 64)
HIGH = (4, 8)
LOW = (2, 4)
RHOS = (0.125, 0.25)
CODECS = ("none", "rle", "entropy")


def all_ids():
    out = []
    for t in TRANSFORMS:
        quants = [f"uniform,b={b},g={g}" for b in BITS for g in GROUPS]
        quants += [f"mixed,hi={hi},lo={lo},g={g},rho={rho!r}" for hi in HIGH for lo in LOW if hi > lo for g in GROUPS for rho in RHOS]
        for q in quants:
            for c in CODECS:
                out.append(f"t={t};q={q};c={c}")
    return out
