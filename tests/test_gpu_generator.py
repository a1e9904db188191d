"""GPU parity of the explicit-plan evaluator (adaptis_eval_plans, including the
R29 communication accounting of its per-device report) and of the
Pipeline Generator (adaptis_generate, readings R28' and R28) against the
oracle: per-plan results and per-device reports bit-exact against
oracle.simulate; the generator's whole trajectory (every accepted step, the
rounds, the plans evaluated) and its final plan identical to
oracle/generator.py's."""
import random

import numpy as np
import pytest

from oracle import generator as G
from oracle import oracle as O
from paper_2509_23722_b200 import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_2509_23722_b200 import adaptis as A
    c = A.Context(0)
    yield c
    c.close()


def small_problem(seed, L=9, p=2, m=4, cap=None):
    rng = random.Random(seed)
    r = lambda a, b: [rng.randint(a, b) for _ in range(L)]  # noqa: E731
    return W.Problem(t_f=r(1, 9), t_b=r(1, 9), t_w=r(1, 9), act=r(0, 5), stash=r(0, 3),
                     weight=r(0, 4), grad=r(0, 4), comm=r(0, 3)[:-1] + [0], p=p, m=m,
                     cap=cap if cap is not None else W.INT64_MAX, name="gpu-gen-%d" % seed)


def random_plans(pr, n, seed, invalid_every=7):
    """Plans over every admitted combo and v, with a share of non-increasing cuts."""
    rng = random.Random(seed)
    L, p = len(pr.t_f), pr.p
    combos = [(1, 0, po) for po in range(4)]
    if pr.m % p == 0:
        for v in (2, 4):
            if p * v <= min(64, L):
                combos += [(v, 1, po) for po in range(4)] + [(v, 2, 0), (v, 2, 3)]
    out = []
    for i in range(n):
        v, pl, po = combos[rng.randrange(len(combos))]
        S = p * v
        cuts = sorted(rng.sample(range(1, L), S - 1))
        if invalid_every and i % invalid_every == 3 and S > 2:
            cuts[1] = cuts[0]  # not strictly increasing: status 1
        out.append({"v": v, "placement": pl, "policy": po, "S": S, "cuts": [0] + cuts + [L]})
    return out


def check_plans(prep, pr, plans):
    got = prep.eval_plans(plans, report=True)
    for i, d in enumerate(plans):
        S = d["S"]
        if any(a >= b for a, b in zip(d["cuts"], d["cuts"][1:])):
            assert got["status"][i] == 1, (i, d)
            continue
        want = O.comm_accounting(pr, d["v"], d["placement"], d["policy"], d["cuts"][1:S])
        assert got["status"][i] == want["status"], (i, d, got["status"][i], want)
        if want["status"] == 0:
            assert got["makespan"][i] == want["makespan"], (i, d)
        if want["status"] in (0, 2):
            assert got["peak_mem"][i] == want["peak_mem"], (i, d)
            assert list(got["M_d"][i]) == want["M_d"], (i, d)
            assert list(got["busy_d"][i]) == want["busy_d"], (i, d)
        if want["status"] == 0:
            assert list(got["T_d"][i]) == want["T_d"], (i, d)
            for k in ("comm_d", "exposed_d", "overlap_d", "bubble_d"):  # R29
                assert list(got[k][i]) == want[k], (i, d, k, list(got[k][i]), want[k])


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_eval_plans_random_small(ctx, seed):
    pr = small_problem(seed, L=11, p=2, m=4, cap=60 if seed == 2 else None)
    prep = ctx.prepare(pr, W.Space([W.Group(1, W.FULL, combo_mask=0xF)]))
    check_plans(prep, pr, random_plans(pr, 300, seed))


@pytest.mark.parametrize("cid,n", [(3, 400), (4, 200)])
def test_eval_plans_configs(ctx, cid, n):
    pr, sp = W.config(cid)
    prep = ctx.prepare(pr, sp)
    check_plans(prep, pr, random_plans(pr, n, cid))


def test_eval_plans_rejects_bad_combo(ctx):
    from paper_2509_23722_b200 import adaptis as A
    pr, sp = W.config(2)
    prep = ctx.prepare(pr, sp)
    bad = {"v": 2, "placement": 2, "policy": 1, "S": 8, "cuts": [0, 4, 8, 12, 16, 20, 24, 28, 34]}
    with pytest.raises(A.AdaptisError) as e:
        prep.eval_plans([bad])
    assert e.value.status == A.EINVAL and "R12" in str(e.value)


def same_trajectory(got, want):
    assert got["status"] == 0 and want["status"] == "ok"
    assert got["steps"] == want["steps"]
    assert got["makespan"] == want["makespan"]
    assert got["plan"] == want["plan"]
    assert got["rounds"] == want["rounds"]
    assert got["n_seeds"] == want["n_seeds"]
    assert got["n_evaluated"] == want["n_evaluated"]


@pytest.mark.parametrize("mode", ["bottleneck", "round-robin"])
@pytest.mark.parametrize("seed", [1, 2, 3, 4, 5, 6])
def test_generate_random_small(ctx, seed, mode):
    pr = small_problem(seed, L=10 + seed % 3, p=2 + (seed % 2) * 2, m=4)
    same_trajectory(ctx.generate(pr, radius=2, mode=mode), G.generate(pr, radius=2, mode=mode))


@pytest.mark.parametrize("mode", ["bottleneck", "round-robin"])
@pytest.mark.parametrize("cid", [1, 2, 3, 4])
def test_generate_configs(ctx, cid, mode):
    pr, _ = W.config(cid)
    got = ctx.generate(pr, mode=mode)
    same_trajectory(got, G.generate(pr, mode=mode))
    want = O.simulate(pr, got["plan"]["v"], got["plan"]["placement"], got["plan"]["policy"],
                      got["plan"]["cuts"][1:-1])
    assert got["T_d"] == want["T_d"] and got["M_d"] == want["M_d"]


def test_generate_infeasible(ctx):
    pr = small_problem(9, cap=0)
    pr.weight = np.ones(len(pr.t_f), np.int64)
    got = ctx.generate(pr)
    assert got["status"] == 2 and got["steps"] == []
