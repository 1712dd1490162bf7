"""Golden values of the reference's profiling evaluator (CorpusEvaluator,
profiling/search.py:318-368), generated from the UNMODIFIED reference:

    python tests/golden/make_evaluator_golden.py

For a seeded corpus (generate_corpus, tensors.py:108-112; reproducible
without the reference through oracle.generate_kv and the same child seeds)
and a fixed list of strategy ids from enumerate_space(SpaceDef()), it records
what CorpusEvaluator(corpus, sample_size=3, timer=CostModelTimer(), seed=0)
returns: the sampled tensor indices, (acc, cr, lat) and the pooled
(s_enc, s_dec).  Two corpora: the reference's float32 values as generated,
and the same values rounded to bf16 (the serving dtype).  The GPU evaluator
test (tests/test_evaluator_parity.py) checks GpuCorpusEvaluator against
these on the GPU box, where the reference is absent.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "evaluator.json")

CORPUS = dict(count=6, seed=11, layers=2, heads=4, tokens=64, channels=128)
SAMPLE = 3


def bf16_round(x: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32)


def main() -> None:
    sys.path.insert(0, REF)
    from kvpilot.pipeline.compress import CostModelTimer
    from kvpilot.pipeline.tensors import KVTensor, generate_corpus
    from kvpilot.profiling.search import CorpusEvaluator, _stable_hash
    from kvpilot.profiling.space import SpaceDef, enumerate_space

    shape = {k: CORPUS[k] for k in ("layers", "heads", "tokens", "channels")}
    corpus32 = generate_corpus(CORPUS["count"], seed=CORPUS["seed"], **shape)
    corpus16 = [KVTensor(values=bf16_round(t.values), head_importance=t.head_importance) for t in corpus32]
    space = enumerate_space(SpaceDef())
    ids = [space.candidates[i].id for i in range(0, len(space), 8)]
    if "t=hadamard;q=uniform,b=4,g=32;c=none" not in ids:
        ids.append("t=hadamard;q=uniform,b=4,g=32;c=none")
    cands = {c.id: c for c in space.candidates}
    out = {"corpus": CORPUS, "sample_size": SAMPLE, "seed": 0, "timer": "CostModelTimer(scale=1.0)",
           "numpy": np.__version__, "cases": {}}
    for name, corpus in (("f32", corpus32), ("bf16", corpus16)):
        ev = CorpusEvaluator(corpus, sample_size=SAMPLE, timer=CostModelTimer(), seed=0)
        rows = []
        for sid in ids:
            s = cands[sid]
            picks = np.random.default_rng([0, _stable_hash(sid)]).choice(len(corpus), size=SAMPLE, replace=False)
            acc, cr, lat = ev(s)
            s_enc, s_dec = ev.throughputs[sid]
            rows.append({"id": sid, "picks": [int(p) for p in picks], "acc": acc, "cr": cr, "lat": lat,
                         "s_enc": s_enc, "s_dec": s_dec})
        out["cases"][name] = rows
    with open(OUT, "w") as f:
        json.dump(out, f, indent=1)
    print(f"wrote {OUT}: {len(ids)} strategies x 2 corpora")


if __name__ == "__main__":
    main()
