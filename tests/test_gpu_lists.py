"""GPU parity of explicit per-device task orders (adaptis_eval_lists, reading
R30: Alg. 1 Step 3 on given workload scheduling results) against the
oracle's `simulate_lists` (longest path over DAG + list edges, memory walked
along the lists): the event loop's realised orders of every policy, and
randomly perturbed orders (new schedules, cyclic waits, caps)."""
import random

import numpy as np
import pytest

from oracle import oracle as O
from paper_2509_23722_b200 import workloads as W

pytestmark = pytest.mark.gpu

LIST, LIST_FUSED = 4, 5


@pytest.fixture(scope="module")
def ctx():
    from paper_2509_23722_b200 import adaptis as A
    c = A.Context(0)
    yield c
    c.close()


def combos(v):
    return [(0, k) for k in range(4)] if v == 1 else [(1, k) for k in range(4)] + [(2, 0), (2, 3)]


def realised(pr, v, pl, po, cuts):
    """The event loop's realised order, or None when it got stuck (incomplete)."""
    r = O.simulate(pr, v, pl, po, cuts, trace=True)
    if r["status"] == 3:
        return po in (0, 1), None
    fused = po in (0, 1)
    return fused, [[(k, s, j) for (k, s, j, _t) in lst if not (fused and k == 2)] for lst in r["trace"]]


def perturb(lists, rng, noise):
    """A random linear extension near the given order: per device, tasks keyed by
    position + noise, emitted greedily while keeping F < B < W per (stage, mb)."""
    out = []
    for lst in lists:
        key = {t: i + rng.uniform(0, noise) for i, t in enumerate(lst)}
        done, res, pend = set(), [], sorted(lst, key=lambda t: key[t])
        while pend:
            for i, (k, s, j) in enumerate(pend):
                if k == 0 or (k - 1, s, j) in done:
                    res.append((k, s, j)); done.add((k, s, j)); pend.pop(i)
                    break
        out.append(res)
    return out


def check(prep, pr, items):
    plans = [{"v": v, "placement": pl, "policy": LIST_FUSED if f else LIST, "S": pr.p * v,
              "cuts": [0] + list(c) + [len(pr.t_f)]} for (v, pl, f, c, _l) in items]
    got = prep.eval_lists(plans, [x[4] for x in items], report=True)
    n_ok = n_stuck = 0
    for i, (v, pl, f, c, lists) in enumerate(items):
        want = O.simulate_lists(pr, v, pl, f, c, lists)
        assert got["status"][i] == want["status"], (i, got["status"][i], want["status"])
        if want["status"] == 0:
            n_ok += 1
            assert got["makespan"][i] == want["makespan"], i
            assert list(got["T_d"][i]) == want["T_d"], i
        if want["status"] in (0, 2):
            assert got["peak_mem"][i] == want["peak_mem"], i
            assert list(got["M_d"][i]) == want["M_d"] and list(got["busy_d"][i]) == want["busy_d"], i
        n_stuck += want["status"] == 3
    return n_ok, n_stuck


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_realised_and_perturbed_orders_small(ctx, seed):
    rng = W.SplitMix64(300 + seed)
    prng = random.Random(seed)
    tot_ok = tot_stuck = 0
    for t in range(10):
        p = [1, 2, 3, 4, 5][t % 5]
        L = 2 * p + 4
        cap = W.INT64_MAX if t % 3 else 50 + 11 * t
        pr = W.random_problem(rng, L, p, 2 * p, tmax=8, cmax=4, bytes_max=5, cap=cap)
        prep = ctx.prepare(pr, W.Space([W.Group(1, W.FULL, combo_mask=0xF)]))
        items = []
        for v in (1, 2):
            S = p * v
            cuts = sorted(prng.sample(range(1, L), S - 1))
            for pl, po in combos(v):
                fused, lists = realised(pr, v, pl, po, cuts)
                if lists is None:
                    continue
                items.append((v, pl, fused, cuts, lists))
                for noise in (1.5, 4.0):
                    items.append((v, pl, fused, cuts, perturb(lists, prng, noise)))
        ok, stuck = check(prep, pr, items)
        tot_ok += ok
        tot_stuck += stuck
    assert tot_ok > 50 and tot_stuck > 0  # both regimes exercised


def test_realised_orders_cfg3(ctx):
    pr, sp = W.config(3)
    prep = ctx.prepare(pr, sp)
    prng = random.Random(33)
    items = []
    for i in range(12):
        v = 1 + i % 2
        S = pr.p * v
        cuts = sorted(prng.sample(range(1, len(pr.t_f)), S - 1))
        for pl, po in combos(v)[i % 3::3]:
            fused, lists = realised(pr, v, pl, po, cuts)
            if lists is None:
                continue
            items.append((v, pl, fused, cuts, lists))
            items.append((v, pl, fused, cuts, perturb(lists, prng, 2.0)))
    ok, _ = check(prep, pr, items)
    assert ok > 5


def test_lists_validation(ctx):
    from paper_2509_23722_b200 import adaptis as A
    z = [0, 0]
    pr = W.Problem(t_f=[1, 1], t_b=[1, 1], t_w=[1, 1], act=z, stash=z, weight=z, grad=z,
                   comm=[1, 0], p=2, m=2)
    prep = ctx.prepare(pr, W.Space([W.Group(1, W.FULL, combo_mask=0xF)]))
    plan = {"v": 1, "placement": 0, "policy": LIST_FUSED, "S": 2, "cuts": [0, 1, 2]}
    good = [[(0, 0, 0), (0, 0, 1), (1, 0, 0), (1, 0, 1)], [(0, 1, 0), (1, 1, 0), (0, 1, 1), (1, 1, 1)]]
    r = prep.eval_lists([plan], [good])
    assert r["status"][0] == 0 and r["makespan"][0] == O.simulate(pr, 1, 0, 1, [1])["makespan"]
    bad = {
        "duplicate": [[(0, 0, 0), (0, 0, 0), (1, 0, 0), (1, 0, 1)], good[1]],
        "wrong device": [[(0, 1, 0), (0, 0, 1), (1, 0, 0), (1, 0, 1)], good[1]],
        "B before F": [[(1, 0, 0), (0, 0, 0), (0, 0, 1), (1, 0, 1)], good[1]],
        "missing": [[(0, 0, 0), (0, 0, 1), (1, 0, 0)], good[1]],
    }
    for why, lists in bad.items():
        with pytest.raises(A.AdaptisError) as e:
            prep.eval_lists([plan], [lists])
        assert e.value.status == A.EINVAL, why
    with pytest.raises(A.AdaptisError):  # W listed in a fused plan
        prep.eval_lists([plan], [[good[0] + [(2, 0, 0)], good[1]]])
