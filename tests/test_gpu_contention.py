"""GPU parity of communication-engine contention on explicit lists
(adaptis_eval_lists_contended, reading R34; SPEC S:206 (a)/(c)) against
the event-driven oracle (oracle/contention.py): realised orders of every
policy and placement, perturbed and micro-batch-shuffled orders (new
schedules and cyclic waits), caps, the R29 report rows, and the reduction to
adaptis_eval_lists when every latency is 0."""
import random

import numpy as np
import pytest

from oracle import oracle as O
from oracle.contention import simulate_lists_contended as SC
from paper_2509_23722_b200 import workloads as W

from test_gpu_lists import combos, perturb, realised, swap_mbs

pytestmark = pytest.mark.gpu

LIST, LIST_FUSED = 4, 5


@pytest.fixture(scope="module")
def ctx():
    from paper_2509_23722_b200 import adaptis as A
    c = A.Context(0)
    yield c
    c.close()


def plan_of(pr, v, pl, fused, cuts):
    return {"v": v, "placement": pl, "policy": LIST_FUSED if fused else LIST, "S": pr.p * v,
            "cuts": [0] + list(cuts) + [len(pr.t_f)]}


def check(prep, pr, items):
    plans = [plan_of(pr, v, pl, f, c) for (v, pl, f, c, _l) in items]
    got = prep.eval_lists_contended(plans, [x[4] for x in items], report=True)
    n_ok = n_stuck = n_slower = 0
    for i, (v, pl, f, c, lists) in enumerate(items):
        want = SC(pr, v, pl, f, c, lists)
        assert got["status"][i] == want["status"], (i, got["status"][i], want["status"])
        if want["status"] == 0:
            n_ok += 1
            assert got["makespan"][i] == want["makespan"], (i, got["makespan"][i], want["makespan"])
            busy = sum(want["busy_d"])
            assert abs(got["bubble"][i] - (1 - busy / (pr.p * want["makespan"]))) < 1e-6
            lp = O.longest_path(pr, v, pl, c, f, lists)
            n_slower += want["makespan"] > lp[0]
        if want["status"] in (0, 2):
            assert got["peak_mem"][i] == want["peak_mem"], i
            for key in ("T_d", "busy_d", "M_d", "comm_d", "exposed_d"):
                assert list(got[key][i]) == want[key], (i, key, list(got[key][i]), want[key])
            # R29's derived rows come from the ABI report, checked against the definition
            assert list(got["overlap_d"][i]) == [c - e for c, e in zip(want["comm_d"], want["exposed_d"])]
            assert list(got["bubble_d"][i]) == [t - b - e for t, b, e in
                                                zip(want["T_d"], want["busy_d"], want["exposed_d"])]
        n_stuck += want["status"] == 3
    return n_ok, n_stuck, n_slower


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_contended_realised_and_perturbed_small(ctx, seed):
    rng = W.SplitMix64(700 + seed)
    prng = random.Random(seed)
    tot = np.zeros(3, int)
    for t in range(10):
        p = [1, 2, 3, 4, 5][t % 5]
        L = 2 * p + 4
        cap = W.INT64_MAX if t % 3 else 50 + 11 * t
        pr = W.random_problem(rng, L, p, 2 * p, tmax=6, cmax=7, bytes_max=5, cap=cap)
        prep = ctx.prepare(pr, W.Space([W.Group(1, W.FULL, combo_mask=0xF)]))
        items = []
        for v in (1, 2):
            cuts = sorted(prng.sample(range(1, L), p * v - 1))
            for pl, po in combos(v):
                fused, lists = realised(pr, v, pl, po, cuts)
                if lists is None:
                    continue
                items.append((v, pl, fused, cuts, lists))
                for noise in (1.5, 4.0):
                    items.append((v, pl, fused, cuts, perturb(lists, prng, noise)))
                if v == 1:
                    items.append((v, pl, fused, cuts, swap_mbs(lists, prng)))
        tot += check(prep, pr, items)
    assert tot[0] > 50 and tot[1] > 0 and tot[2] > 20  # ok, stuck and contended regimes


def test_contended_zero_latency_equals_eval_lists(ctx):
    rng = W.SplitMix64(77)
    prng = random.Random(77)
    for t in range(4):
        p = 2 + t
        L = 3 * p
        pr = W.random_problem(rng, L, p, 2 * p, tmax=9, cmax=0)
        pr.comm[:] = 0
        prep = ctx.prepare(pr, W.Space([W.Group(1, W.FULL, combo_mask=0xF)]))
        items = []
        for v in (1, 2):
            cuts = sorted(prng.sample(range(1, L), p * v - 1))
            for pl, po in combos(v):
                fused, lists = realised(pr, v, pl, po, cuts)
                if lists is not None:
                    items.append((plan_of(pr, v, pl, fused, cuts), lists))
        a = prep.eval_lists_contended([x[0] for x in items], [x[1] for x in items], report=True)
        b = prep.eval_lists([x[0] for x in items], [x[1] for x in items], report=True)
        for key in ("status", "makespan", "peak_mem", "T_d", "busy_d", "M_d"):
            assert np.array_equal(np.asarray(a[key]), np.asarray(b[key])), key


def test_contended_wide_pipelines(ctx):
    """p = 16 and 32 (every lane of the warp a device), v up to 4."""
    rng = W.SplitMix64(99)
    prng = random.Random(99)
    for p, vs in ((16, (1, 2)), (32, (1,)), (8, (3, 4))):
        L = 4 * p + 3
        pr = W.random_problem(rng, L, p, p, tmax=3, cmax=40, bytes_max=3)
        # any valid space: explicit plans only reuse the prepared tables
        prep = ctx.prepare(pr, W.Space([W.Group(1, W.BALL, radius=1, combo_mask=0xF)]))
        items = []
        for v in vs:
            cuts = sorted(prng.sample(range(1, L), p * v - 1))
            for pl, po in combos(v)[:3]:
                fused, lists = realised(pr, v, pl, po, cuts)
                if lists is not None:
                    items.append((v, pl, fused, cuts, lists))
        ok, _stuck, slower = check(prep, pr, items)
        assert ok >= 2 and slower >= 1


def test_contended_cfg3_shapes(ctx):
    """cfg3's tables (61+2 rows, p = 8, m = 32): realised 1F1B / ZB / GREEDY
    orders of random partitions, and a perturbed copy of each."""
    pr, sp = W.config(3)
    prep = ctx.prepare(pr, sp)
    prng = random.Random(3)
    items = []
    for i in range(4):
        v = 1 + i % 2
        cuts = sorted(prng.sample(range(1, len(pr.t_f)), pr.p * v - 1))
        for pl, po in combos(v)[1:4]:
            fused, lists = realised(pr, v, pl, po, cuts)
            if lists is None:
                continue
            items.append((v, pl, fused, cuts, lists))
            items.append((v, pl, fused, cuts, perturb(lists, prng, 2.0)))
    ok, _stuck, _slower = check(prep, pr, items)
    assert ok >= 6


def test_contended_validation(ctx):
    from paper_2509_23722_b200 import adaptis as A
    z = [0, 0]
    pr = W.Problem(t_f=[1, 1], t_b=[1, 1], t_w=[1, 1], act=z, stash=z, weight=z, grad=z,
                   comm=[2, 0], p=2, m=2)
    prep = ctx.prepare(pr, W.Space([W.Group(1, W.FULL, combo_mask=0xF)]))
    plan = {"v": 1, "placement": 0, "policy": LIST_FUSED, "S": 2, "cuts": [0, 1, 2]}
    d0 = [(0, 0, 0), (1, 0, 0), (0, 0, 1), (1, 0, 1)]
    r = prep.eval_lists_contended([plan, plan], [[d0, [(0, 1, 0), (1, 1, 0), (0, 1, 1), (1, 1, 1)]],
                                                 [d0, [(0, 1, 0), (0, 1, 1), (1, 1, 0), (1, 1, 1)]]])
    assert list(r["status"]) == [0, 3] and r["makespan"][0] == 20
    with pytest.raises(A.AdaptisError) as e:
        prep.eval_lists_contended([plan], [[d0[:3], d0]])
    assert e.value.status == A.EINVAL
