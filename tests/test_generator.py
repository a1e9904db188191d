"""Pins of the oracle's Pipeline Generator (oracle/generator.py, reading R28 of
P:334-372) against properties that do not come from the generator itself:

* the result re-simulates to the reported makespan (oracle.simulate);
* the trajectory starts at the best seed and falls strictly (rollback rule,
  P:351 "If a tuning step degrades pipeline performance, it is rolled back");
* the result is a local optimum of all three phases, checked by brute-force
  enumeration of the L1 ball (oracle.enumerate_space + eval_indices, not the
  search the generator uses) and of the placement / schedule alternatives;
* when the ball covers every partition, the partition phase reaches the
  exhaustive optimum of the final combo (FULL-space search);
* the seeds are the P:346 baselines: equal-layer cuts and the min-max split.
"""
import random

import pytest

from oracle import generator as G
from oracle import oracle as O
from paper_2509_23722_b200 import workloads as W


def small_problem(seed, L=7, p=2, m=4, cap=None):
    rng = random.Random(seed)
    t_f = [rng.randint(1, 9) for _ in range(L)]
    t_b = [rng.randint(1, 9) for _ in range(L)]
    t_w = [rng.randint(1, 9) for _ in range(L)]
    act = [rng.randint(0, 5) for _ in range(L)]
    stash = [rng.randint(0, 3) for _ in range(L)]
    weight = [rng.randint(0, 4) for _ in range(L)]
    grad = [rng.randint(0, 4) for _ in range(L)]
    comm = [rng.randint(0, 3) for _ in range(L - 1)] + [0]
    return W.Problem(t_f=t_f, t_b=t_b, t_w=t_w, act=act, stash=stash, weight=weight, grad=grad,
                     comm=comm, p=p, m=m, cap=cap if cap is not None else W.INT64_MAX,
                     name="gen-small-%d" % seed)


def ball(cuts, R, L):
    """Every strictly increasing interior cut vector within L1 distance R (brute force)."""
    out = []
    n = len(cuts)

    def rec(i, left, acc):
        if i == n:
            if all(0 < a < b for a, b in zip([0] + acc, acc + [L])):
                out.append(list(acc))
            return
        for d in range(-left, left + 1):
            rec(i + 1, left - abs(d), acc + [cuts[i] + d])
    rec(0, R, [])
    return out


def mk(pr, v, pl, po, cuts):
    r = O.simulate(pr, v, pl, po, cuts)
    return r["makespan"] if r["status"] == 0 else None


CASES = [(small_problem(s), 0x3, 2) for s in range(4)] + [(small_problem(11, L=9, p=3, m=6), 0x3, 1)]


@pytest.mark.parametrize("pr,vs_mask,R", CASES, ids=lambda x: getattr(x, "name", str(x)))
def test_result_resimulates_and_trajectory_falls(pr, vs_mask, R):
    r = G.generate(pr, vs_mask=vs_mask, radius=R)
    assert r["status"] == "ok"
    pl = r["plan"]
    assert mk(pr, pl["v"], pl["placement"], pl["policy"], pl["cuts"][1:-1]) == r["makespan"]
    ms = [x[1] for x in r["steps"]]
    assert r["steps"][0][0] == "seed"
    assert all(a > b for a, b in zip(ms, ms[1:]))
    assert ms[-1] == r["makespan"]


@pytest.mark.parametrize("pr,vs_mask,R", CASES, ids=lambda x: getattr(x, "name", str(x)))
def test_result_is_local_optimum(pr, vs_mask, R):
    r = G.generate(pr, vs_mask=vs_mask, radius=R)
    pl = r["plan"]
    v, place, pol, cuts = pl["v"], pl["placement"], pl["policy"], pl["cuts"][1:-1]
    L = len(pr.t_f)
    best = r["makespan"]
    # partition neighbourhood, enumerated by brute force
    for c in ball(cuts, R, L):
        x = mk(pr, v, place, pol, c)
        assert x is None or x >= best, (c, x, best)
    # schedule alternatives (R12)
    for po2 in range(4):
        if G.admitted(v, place, po2):
            x = mk(pr, v, place, po2, cuts)
            assert x is None or x >= best
    # placement alternatives with the same v (grouped permutation INT <-> WAVE)
    if v >= 2:
        for pl2 in (G.INT, G.WAVE):
            po2 = pol if G.admitted(v, pl2, pol) else G.GREEDY
            x = mk(pr, v, pl2, po2, cuts)
            assert x is None or x >= best


def test_seed_is_best_of_p346_baselines():
    """Seeds: equal layers and min-max, S-1F1B / ZB / I-1F1B / Hanayo."""
    pr = small_problem(3)
    L, p = len(pr.t_f), pr.p
    assert G.equal_layers(8, 4) == [2, 4, 6]
    assert G.equal_layers(7, 2) == [3]
    plans = []
    for v in (1, 2):
        S = p * v
        for cuts in (G.equal_layers(L, S), G.mist(pr, S)):
            for pl, po in ([(0, 1), (0, 2)] if v == 1 else [(1, 1), (1, 2), (2, 3)]):
                plans.append(mk(pr, v, pl, po, cuts))
    r = G.generate(pr, max_rounds=1)
    assert r["steps"][0][1] == min(x for x in plans if x is not None)


def test_covering_ball_reaches_exhaustive_optimum_of_final_combo():
    pr = small_problem(5, L=6, p=2, m=4)
    r = G.generate(pr, vs_mask=0x1, radius=6)  # R >= L: the ball holds every partition
    pl = r["plan"]
    k = G.combo_index(pl["v"], pl["placement"], pl["policy"])
    full = O.search(pr, W.Space([W.Group(pl["v"], W.FULL, combo_mask=1 << k)]), prune=False)
    assert r["makespan"] == full["makespan"]


def test_infeasible_seeds():
    pr = small_problem(2, cap=0)
    pr.weight = [1] * len(pr.t_f)
    r = G.generate(pr)
    assert r["status"] == "infeasible"


@pytest.mark.parametrize("cid", [1, 2])
def test_generator_on_configs(cid):
    pr, _ = W.config(cid)
    r = G.generate(pr)
    assert r["status"] == "ok"
    pl = r["plan"]
    assert mk(pr, pl["v"], pl["placement"], pl["policy"], pl["cuts"][1:-1]) == r["makespan"]


def test_transfer_moves_one_layer_and_keeps_stages_contiguous():
    """R28' partition move ("transferring layers from the stage with the
    lowest bubble ratio to the stage with the highest"): worked by hand."""
    # stages [0,2) [2,4) [4,6) [6,8): stage 0 gives its last layer to stage 2,
    # stage 1 shifts left by one and keeps two layers
    assert G.transfer([2, 4, 6], 8, 0, 2) == [1, 3, 6]
    # stage 3 gives its first layer to stage 1, stage 2 shifts right by one
    assert G.transfer([2, 4, 6], 8, 3, 1) == [2, 5, 7]
    assert G.transfer([2, 4, 6], 8, 1, 2) == [2, 3, 6]
    assert G.transfer([1, 4, 6], 8, 0, 1) is None  # stage 0 would be empty
    sizes = lambda c: [b - a for a, b in zip([0] + c, c + [8])]  # noqa: E731
    for src in range(4):
        for dst in range(4):
            if src != dst:
                c = G.transfer([2, 4, 6], 8, src, dst)
                want = [2, 2, 2, 2]
                want[src] -= 1
                want[dst] += 1
                assert sizes(c) == want, (src, dst)


@pytest.mark.parametrize("pr,vs_mask,R", CASES, ids=lambda x: getattr(x, "name", str(x)))
def test_bottleneck_mode_phase_order_and_round_robin_mode(pr, vs_mask, R):
    """R28' (default): every round starts with the bottleneck phase: the
    partition when the BubbleTime spread is >= the largest stage cost;
    the trajectory falls strictly; the round-1 reading R28 still runs."""
    r = G.generate(pr, vs_mask=vs_mask, radius=R)
    ms = [x[1] for x in r["steps"]]
    assert all(a > b for a, b in zip(ms, ms[1:]))
    rr = G.generate(pr, vs_mask=vs_mask, radius=R, mode="round-robin")
    assert rr["status"] == "ok" and rr["steps"][0] == r["steps"][0]  # same seeds


def test_bottleneck_transfer_fires_on_an_unbalanced_seed():
    """A heavy last layer leaves the device of stage 0 idle; with the spread of
    BubbleTime(d) above the largest stage cost, the first tuning round moves
    a layer (a partition step right after the seed), and that step is a
    single-layer transfer or the ball's best, both within the L1 ball."""
    L, p, m = 8, 2, 4
    z = [0] * L
    pr = W.Problem(t_f=[1, 1, 1, 1, 1, 1, 1, 9], t_b=[1, 1, 1, 1, 1, 1, 1, 9],
                   t_w=[1, 1, 1, 1, 1, 1, 1, 9], act=z, stash=z, weight=z, grad=z,
                   comm=[1] * (L - 1) + [0], p=p, m=m)
    r = G.generate(pr, vs_mask=0x1)
    assert r["status"] == "ok"
    # the equal-layer seed [4] is unbalanced (4 vs 12 per micro-batch); Mist's seed is better
    bub, T, maxcs = G.bottleneck(pr, (1, G.SEQ, G.ONEF1B, [4]))
    assert max(bub) - min(bub) >= maxcs
    assert r["makespan"] <= G.score(pr, 1, G.SEQ, G.ONEF1B, G.mist(pr, 2))
