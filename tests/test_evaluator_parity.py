"""GpuCorpusEvaluator vs the reference CorpusEvaluator (profiling/search.py:318-368).

tests/golden/evaluator.json holds what the UNMODIFIED reference evaluator
returned (tests/golden/make_evaluator_golden.py) for 24 strategy ids of
enumerate_space(SpaceDef()) on a seeded corpus -- the reference's own float32
values, and the same values rounded to bf16 -- with the deterministic
CostModelTimer.  The GPU evaluator (reference_format=True: whole-tensor
rle / entropy payloads) must sample the same tensors and return the same
(acc, cr, lat) and pooled (s_enc, s_dec): cr, lat and throughputs exactly,
acc to the summation order of quality_score (identity / delta decode is the
reference arithmetic bit for bit) or, for Hadamard ids, within the fused
decode's fp32 inverse-transform tolerance.
"""

from __future__ import annotations

import json
import os

import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "evaluator.json")))


def _corpus(rounded: bool):
    """generate_corpus (tensors.py:108-112) through the oracle's generator
    (pinned equal to tensors.py:79-105): the same child seeds."""
    c = GOLD["corpus"]
    seeds = np.random.default_rng(c["seed"]).integers(0, 2**31 - 1, size=c["count"])
    out = []
    for s in seeds:
        v, imp = oracle.generate_kv(c["layers"], c["heads"], c["tokens"], c["channels"], seed=int(s))
        if rounded:
            u = v.view(np.uint32).astype(np.uint64)
            v = ((((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16).astype(np.uint32)).view(np.float32)
        out.append((v, imp))
    return out


def test_golden_picks_follow_the_reference_sampler():
    """The sampled indices in the fixture are rng([seed, sha256(id)]) draws
    (search.py:348-349); the GPU evaluator uses the same rule (CPU check)."""
    from paper_2605_13734_b200.pipeline import _stable_hash

    for row in GOLD["cases"]["f32"]:
        picks = np.random.default_rng([GOLD["seed"], _stable_hash(row["id"])]).choice(
            GOLD["corpus"]["count"], size=GOLD["sample_size"], replace=False)
        assert [int(p) for p in picks] == row["picks"], row["id"]


@pytest.mark.gpu
@pytest.mark.parametrize("corpus", ["f32", "bf16"])
def test_gpu_evaluator_matches_reference_evaluator(corpus):
    from paper_2605_13734_b200 import CostModelTimer, GpuCorpusEvaluator, KVTensor, parse_strategy_id

    data = [KVTensor(v, imp) for v, imp in _corpus(corpus == "bf16")]
    ev = GpuCorpusEvaluator(data, sample_size=GOLD["sample_size"], timer=CostModelTimer(), seed=GOLD["seed"],
                            reference_format=True)
    for row in GOLD["cases"][corpus]:
        s = parse_strategy_id(row["id"])
        acc, cr, lat = ev(s)
        assert ev.picks[s.id] == row["picks"], row["id"]
        assert cr == row["cr"], (row["id"], cr, row["cr"])
        assert lat == row["lat"], (row["id"], lat, row["lat"])
        assert ev.throughputs[s.id] == (row["s_enc"], row["s_dec"]), row["id"]
        # identity / delta decode reproduces the reference arithmetic bit for
        # bit, so only quality_score's summation order differs; the fused
        # head_dim-128 decode runs the inverse Hadamard in fp32 (held to 1e-5 of
        # the row magnitude, test_acceptance.py:235)
        tol = 1e-5 if "hadamard" in row["id"] else 1e-9
        assert abs(acc - row["acc"]) <= tol, (row["id"], acc, row["acc"])
