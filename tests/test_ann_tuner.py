"""The auto-tuner's performance model and two-phase search (§4 lines
249-256; R23), host code in libicl.so, run on
CPU through icl_ann_fit / icl_ann_search.

Pins: exhaustive evaluation of the whole space (the brute-force optimum) and
a noiseless log-linear cost the network can represent."""
import itertools
import math
import random

import pytest

import paper_1605_06399_b200 as icl

SPACE = list(itertools.product(range(8), range(8), range(6)))  # 384 configurations


def cost(c):  # separable synthetic cost with one optimum at (5, 2, 3)
    return 1.0 + (c[0] - 5) ** 2 + 0.5 * (c[1] - 2) ** 2 + 2.0 * abs(c[2] - 3)


def test_fit_noiseless_log_linear():
    for s in range(5):
        rnd = random.Random(s)
        X = [[rnd.random(), rnd.random(), rnd.random()] for _ in range(30)]
        y = [math.exp(0.5 * a - 1.2 * b + 0.3 * c) for a, b, c in X]
        r = icl.ann_fit(X, y, seed=s)
        assert r["final_loss"] < 5e-3
        assert max(abs(p / v - 1.0) for p, v in zip(r["pred"], y)) < 0.05


def test_fit_duplicates_converge():
    X = [[1.0, 2.0]] * 6 + [[3.0, 1.0]] * 6
    y = [2.0] * 6 + [5.0] * 6
    r = icl.ann_fit(X, y, seed=1)
    assert all(abs(p / v - 1.0) < 0.05 for p, v in zip(r["pred"], y))


def test_fit_needs_ten_samples():
    with pytest.raises(icl.IclError):
        icl.ann_fit([[float(i)] for i in range(9)], [1.0 + i for i in range(9)])
    with pytest.raises(icl.IclError):
        icl.ann_fit([[float(i)] for i in range(10)], [0.0] + [1.0] * 9)  # values must be > 0


def test_search_finds_near_optimum_over_seeds():
    costs = sorted(cost(c) for c in SPACE)
    top5 = costs[int(0.05 * len(costs))]
    hits = 0
    for seed in range(50):
        r = icl.ann_search(SPACE, lambda i: cost(SPACE[i]), n1=30, topk=10, seed=seed)
        assert len(r["evaluated"]) == 40 and len(set(r["evaluated"])) == 40
        assert r["value"] == min(cost(SPACE[i]) for i in r["evaluated"])
        hits += r["value"] <= top5
    assert hits >= 45  # >= 90% of seeds within the best 5% of the exhaustive ranking


def test_search_deterministic_and_phase2_never_worse():
    a = icl.ann_search(SPACE, lambda i: cost(SPACE[i]), n1=20, topk=8, seed=11)
    b = icl.ann_search(SPACE, lambda i: cost(SPACE[i]), n1=20, topk=8, seed=11)
    assert a == b
    phase1 = min(cost(SPACE[i]) for i in a["evaluated"][:20])
    assert a["value"] <= phase1


def test_search_full_budget_is_exhaustive():
    small = SPACE[:40]
    r = icl.ann_search(small, lambda i: cost(small[i]), n1=40, topk=5, seed=3)
    assert sorted(r["evaluated"]) == list(range(40))
    assert r["value"] == min(cost(c) for c in small)


def test_search_single_and_failing():
    r = icl.ann_search([[0.0]], lambda i: 3.0, n1=10, topk=5)
    assert r["best"] == 0 and r["evaluated"] == [0]
    with pytest.raises(icl.IclError):
        icl.ann_search(SPACE[:20], lambda i: None, n1=10, topk=5)


def test_search_skips_failed_configurations():
    bad = {i for i, c in enumerate(SPACE) if c[0] == 5}  # the optimum's column fails
    r = icl.ann_search(SPACE, lambda i: None if i in bad else cost(SPACE[i]), n1=40, topk=20, seed=2)
    assert r["best"] not in bad
    assert r["value"] == min(cost(SPACE[i]) for i in r["evaluated"] if i not in bad)


def test_search_too_few_ok_samples_finishes_exhaustively():
    n = 30
    r = icl.ann_search([[float(i)] for i in range(n)], lambda i: None if i % 4 else 1.0 + i, n1=12, topk=2, seed=5)
    assert sorted(r["evaluated"]) == list(range(n))  # < 10 ok in phase 1 -> every configuration runs
    assert r["best"] == 0
