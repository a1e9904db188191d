"""GPU parity of the memory timeline (adaptis_memory_timeline, reading R35:
Eq. 2, "identifies potential OOM time") against the
oracle's timeline (oracle.memory_timeline): every breakpoint (time, bytes) and
the first violation time, on policy plans of every policy and placement and
on explicit schedules (R30), with binding caps."""
import random

import pytest

from oracle import oracle as O
from paper_2509_23722_b200 import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_2509_23722_b200 import adaptis as A
    c = A.Context(0)
    yield c
    c.close()


def _plans(pr, rng, n):
    L, p = len(pr.t_f), pr.p
    combos = [(1, W.SEQ, po) for po in range(4)]
    if pr.m % p == 0 and 2 * p <= L:
        combos += [(2, W.INTERLEAVED, po) for po in range(4)] + [(2, W.WAVE, 0), (2, W.WAVE, 3)]
    for _ in range(n):
        v, pl, po = combos[rng.randrange(len(combos))]
        S = p * v
        yield {"v": v, "placement": pl, "policy": po, "S": S,
               "cuts": [0] + sorted(rng.sample(range(1, L), S - 1)) + [L]}


@pytest.mark.parametrize("seed", [1, 2, 3, 4])
def test_memory_timeline_policy_plans(ctx, seed):
    rng = random.Random(seed)
    srng = W.SplitMix64(seed)
    checked = 0
    for t in range(6):
        p = [1, 2, 4, 3][t % 4]
        m = p * (1 + t % 2)
        L = 2 * p + 3
        cap = W.INT64_MAX if t % 2 else 40
        pr = W.random_problem(srng, L, p, m, tmax=9, cmax=5, bytes_max=9, cap=cap)
        prep = ctx.prepare(pr, W.Space([W.Group(1, W.FULL, combo_mask=0xF)]))
        for plan in _plans(pr, rng, 12):
            sim = O.simulate(pr, plan["v"], plan["placement"], plan["policy"], plan["cuts"][1:-1])
            if sim["status"] not in (0, 2):
                continue
            want = O.memory_timeline(pr, plan["v"], plan["placement"], plan["policy"], plan["cuts"][1:-1])
            got = prep.memory_timeline(plan)
            assert got["points"] == [list(map(tuple, x)) for x in want["points"]], plan
            assert got["first_violation"] == want["first_violation"], plan
            checked += 1
    assert checked > 20


def test_memory_timeline_config_plans(ctx):
    """cfg3 tables at the 180 GB cap: violations happen (ZB / GREEDY plans of
    unbalanced partitions) and are located at the same tick."""
    pr, sp = W.config(3)
    prep = ctx.prepare(pr, sp)
    rng = random.Random(33)
    viol = 0
    for plan in _plans(pr, rng, 40):
        sim = O.simulate(pr, plan["v"], plan["placement"], plan["policy"], plan["cuts"][1:-1])
        if sim["status"] not in (0, 2):
            continue
        want = O.memory_timeline(pr, plan["v"], plan["placement"], plan["policy"], plan["cuts"][1:-1])
        got = prep.memory_timeline(plan)
        assert got["points"] == [list(map(tuple, x)) for x in want["points"]]
        assert got["first_violation"] == want["first_violation"]
        viol += any(x >= 0 for x in want["first_violation"])
    assert viol > 0


def test_memory_timeline_explicit_lists(ctx):
    """Explicit schedules (R30): the event loop's realised orders, split and fused."""
    srng = W.SplitMix64(99)
    n = 0
    for t in range(8):
        p = [2, 3, 4][t % 3]
        m = p * 2
        pr = W.random_problem(srng, 2 * p + 2, p, m, tmax=9, cmax=5, bytes_max=9,
                              cap=W.INT64_MAX if t % 2 else 45)
        prep = ctx.prepare(pr, W.Space([W.Group(1, W.FULL, combo_mask=0xF)]))
        cuts = list(range(1, 2 * p))
        for po in range(4):
            r = O.simulate(pr, 2, W.INTERLEAVED, po, cuts, trace=True)
            if r["status"] not in (0, 2):
                continue
            fused = po in (0, 1)
            lists = [[(k, s, j) for (k, s, j, _t) in lst if not (fused and k == 2)] for lst in r["trace"]]
            pol = 5 if fused else 4
            plan = {"v": 2, "placement": W.INTERLEAVED, "policy": pol, "S": 2 * p,
                    "cuts": [0] + cuts + [len(pr.t_f)]}
            want = O.memory_timeline(pr, 2, W.INTERLEAVED, pol, cuts, lists=lists)
            got = prep.memory_timeline(plan, lists=lists)
            assert got["points"] == [list(map(tuple, x)) for x in want["points"]]
            assert got["first_violation"] == want["first_violation"]
            # the list's timeline is the policy's (same realised order)
            assert want == O.memory_timeline(pr, 2, W.INTERLEAVED, po, cuts)
            n += 1
    assert n > 10


def test_realized_lists_equal_the_event_loop_order(ctx):
    """adaptis_realize_lists: the policy's realised per-device order equals the
    oracle event loop's trace order, and evaluating it as an explicit schedule
    (R30, LIST / LIST_FUSED) reproduces the plan's result."""
    srng = W.SplitMix64(123)
    rng = random.Random(123)
    n = 0
    for t in range(6):
        p = [2, 3, 4][t % 3]
        pr = W.random_problem(srng, 2 * p + 3, p, 2 * p, tmax=9, cmax=5, bytes_max=9,
                              cap=W.INT64_MAX if t % 2 else 45)
        prep = ctx.prepare(pr, W.Space([W.Group(1, W.FULL, combo_mask=0xF)]))
        for plan in _plans(pr, rng, 10):
            cuts = plan["cuts"][1:-1]
            r = O.simulate(pr, plan["v"], plan["placement"], plan["policy"], cuts, trace=True)
            if r["status"] not in (0, 2):
                continue
            fused = plan["policy"] in (W.GPIPE, W.ONEF1B)
            want = [[(k, s, j) for (k, s, j, _t) in lst if not (fused and k == 2)] for lst in r["trace"]]
            got = prep.realize_lists(plan)
            assert got == want, plan
            lp = dict(plan, policy=5 if fused else 4)
            ev = prep.eval_lists([lp], [got])
            assert int(ev["status"][0]) == r["status"]
            if r["status"] == 0:
                assert int(ev["makespan"][0]) == r["makespan"]
            n += 1
    assert n > 20
