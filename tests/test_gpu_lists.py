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


def swap_mbs(lists, rng):
    """Per device, emit the micro-batches of every (kind, stage) in a random order
    (far from Lemma 4's micro-batch order) while keeping F < B < W per (stage, mb)."""
    out = []
    for lst in lists:
        perm = {}
        for (k, s, j) in lst:
            perm.setdefault(s, None)
        order = list(range(max(j for (_k, _s, j) in lst) + 1))
        rng.shuffle(order)
        rank = {j: i for i, j in enumerate(order)}
        out.append(sorted(lst, key=lambda t: (t[0], rank[t[2]], t[1])))
    return out


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


def test_orders_out_of_microbatch_order(ctx):
    """Orders whose producers emit micro-batches far out of order (GPipe-like
    lists with shuffled micro-batches): every micro-batch has its own ring slot."""
    prng = random.Random(5)
    rng = W.SplitMix64(505)
    for t in range(6):
        p = [1, 2, 3][t % 3]
        L = 2 * p + 3
        pr = W.random_problem(rng, L, p, 12, tmax=6, cmax=3, bytes_max=4)
        prep = ctx.prepare(pr, W.Space([W.Group(1, W.FULL, combo_mask=0xF)]))
        cuts = sorted(prng.sample(range(1, L), p - 1))
        items = []
        for po in (0, 2):
            fused, lists = realised(pr, 1, 0, po, cuts)
            items.append((1, 0, fused, cuts, swap_mbs(lists, prng)))
        ok, _ = check(prep, pr, items)
        assert ok >= 1


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


# ----------------------------------------------------------------- R31 OOM repair
def test_repair_oom_worked_example_gpu(ctx):
    # the oracle pin's single-device case with L = 2 rows (the library needs L >= 2):
    # stage sums t_F 2, t_B + t_W 4, 10 B per activation, cap 25
    pr = W.Problem(t_f=[1, 1], t_b=[1, 1], t_w=[1, 1], act=[5, 5], stash=[0, 0], weight=[0, 0],
                   grad=[0, 0], comm=[0, 0], p=1, m=4, cap=25)
    prep = ctx.prepare(pr, W.Space([W.Group(1, W.FULL, combo_mask=0xF)]))
    plan = {"v": 1, "placement": 0, "policy": LIST_FUSED, "S": 1, "cuts": [0, 2]}
    gp = [[(0, 0, j) for j in range(4)] + [(1, 0, j) for j in range(4)]]
    r = prep.repair_oom(plan, gp)
    assert r["moves"] == 2 and r["status"] == 0 and r["makespan"] == 24
    assert r["lists"] == [[(0, 0, 0), (0, 0, 1), (1, 0, 1), (0, 0, 2), (1, 0, 2), (0, 0, 3), (1, 0, 0), (1, 0, 3)]]


@pytest.mark.parametrize("seed", [1, 2, 3, 4])
def test_repair_oom_matches_oracle(ctx, seed):
    """Over-cap realised orders of GPipe / 1F1B / ZB repaired on the GPU and by the
    oracle: same final lists, number of moves, status and makespan."""
    rng = W.SplitMix64(700 + seed)
    prng = random.Random(seed)
    n_cases = n_fixed = 0
    for t in range(12):
        p = [1, 2, 3, 4][t % 4]
        L = 2 * p + 3
        pr = W.random_problem(rng, L, p, 2 * p + 2, tmax=6, cmax=3, bytes_max=8)
        v = 1 + (t % 2) if (2 * p + 2) % p == 0 else 1
        S = p * v
        cuts = sorted(prng.sample(range(1, L), S - 1))
        pl = 0 if v == 1 else 1
        for po in (0, 1, 2):
            r0 = O.simulate(pr, v, pl, po, cuts, trace=True)
            # a cap between the static memory and the schedule's peak makes it over the cap
            stat = max(m_ - 0 for m_ in r0["M_d"])
            pr.cap = max(1, stat - 1 - prng.randrange(0, 6))
            r = O.simulate(pr, v, pl, po, cuts, trace=True)
            if r["status"] != 2:
                continue
            fused = po in (0, 1)
            lists = [[(k, s, j) for (k, s, j, _t) in lst if not (fused and k == 2)] for lst in r["trace"]]
            prep = ctx.prepare(pr, W.Space([W.Group(1, W.FULL, combo_mask=0xF)]))
            plan = {"v": v, "placement": pl, "policy": LIST_FUSED if fused else LIST, "S": S,
                    "cuts": [0] + cuts + [L]}
            got = prep.repair_oom(plan, lists)
            wl, wm, wr = O.repair_oom(pr, v, pl, fused, cuts, lists)
            assert got["moves"] == wm and got["lists"] == wl, (t, po)
            assert got["status"] == wr["status"], (t, po)
            if wr["status"] == 0:
                assert got["makespan"] == wr["makespan"]
                n_fixed += 1
            n_cases += 1
            pr.cap = W.INT64_MAX
    assert n_cases > 10 and n_fixed > 0


def test_repair_oom_cfg3_order(ctx):
    """A cfg3 1F1B plan whose cap is tightened below its peak, repaired on the GPU
    and by the oracle."""
    pr, sp = W.config(3)
    cuts = W.config(3)[1].groups[0].seed_cuts or O.seed_minmax(
        [pr.t_f[i] + pr.t_b[i] + pr.t_w[i] for i in range(len(pr.t_f))], pr.p)[1]
    r0 = O.simulate(pr, 1, 0, 1, cuts, trace=True)
    pr.cap = int(max(r0["M_d"]) - 1)
    r = O.simulate(pr, 1, 0, 1, cuts, trace=True)
    assert r["status"] == 2
    lists = [[(k, s, j) for (k, s, j, _t) in lst if k != 2] for lst in r["trace"]]
    prep = ctx.prepare(pr, sp)
    plan = {"v": 1, "placement": 0, "policy": LIST_FUSED, "S": pr.p, "cuts": [0] + list(cuts) + [len(pr.t_f)]}
    got = prep.repair_oom(plan, lists)
    wl, wm, wr = O.repair_oom(pr, 1, 0, True, cuts, lists)
    assert (got["moves"], got["status"], got["lists"]) == (wm, wr["status"], wl)


# ----------------------------------------------------------------- R32 overlap-aware reordering
@pytest.mark.parametrize("seed", [1, 2])
def test_tune_overlap_matches_oracle(ctx, seed):
    rng = W.SplitMix64(3200 + seed)
    prng = random.Random(seed)
    moved = 0
    for t in range(8):
        p = [2, 3, 4][t % 3]
        L = 2 * p + 3
        pr = W.random_problem(rng, L, p, 2 * p, tmax=6, cmax=8, bytes_max=3)
        prep = ctx.prepare(pr, W.Space([W.Group(1, W.FULL, combo_mask=0xF)]))
        cuts = sorted(prng.sample(range(1, L), p - 1))
        for po in (1, 2):
            fused, lists = realised(pr, 1, 0, po, cuts)
            if lists is None:
                continue
            plan = {"v": 1, "placement": 0, "policy": LIST_FUSED if fused else LIST, "S": p,
                    "cuts": [0] + cuts + [L]}
            got = prep.tune_overlap(plan, lists)
            wl, ws, wa = O.tune_overlap(pr, 1, 0, fused, cuts, lists)
            assert got["swaps"] == ws and got["lists"] == wl, (t, po)
            assert got["makespan"] == wa["makespan"] and got["overlap_after"] == sum(wa["overlap_d"])
            moved += ws
    assert moved > 0


def test_tune_overlap_cfg3_plan(ctx):
    pr, sp = W.config(3)
    prep = ctx.prepare(pr, sp)
    cuts = O.seed_minmax([pr.t_f[i] + pr.t_b[i] + pr.t_w[i] for i in range(len(pr.t_f))], pr.p)[1]
    fused, lists = realised(pr, 1, 0, 2, cuts)
    plan = {"v": 1, "placement": 0, "policy": LIST, "S": pr.p, "cuts": [0] + list(cuts) + [len(pr.t_f)]}
    got = prep.tune_overlap(plan, lists, max_swaps=6)
    wl, ws, wa = O.tune_overlap(pr, 1, 0, False, cuts, lists, max_rounds=6)
    assert (got["swaps"], got["makespan"], got["lists"]) == (ws, wa["makespan"], wl)


def test_int64_kernels_for_lists_plans_and_reports(ctx, monkeypatch):
    """The int64-tick instantiations of the explicit-plan, LIST and TRACE /
    accounting kernels (selected when the makespan bound exceeds 2^31; forced
    here) against the oracle, plus an OOM repair through them."""
    monkeypatch.setenv("ADAPTIS_FORCE_INT64", "1")
    rng = W.SplitMix64(6464)
    prng = random.Random(64)
    for t in range(4):
        p = [2, 3][t % 2]
        L = 2 * p + 4
        pr = W.random_problem(rng, L, p, 2 * p, tmax=8, cmax=4, bytes_max=5)
        prep = ctx.prepare(pr, W.Space([W.Group(1, W.FULL, combo_mask=0xF)]))
        items = []
        for v in (1, 2):
            cuts = sorted(prng.sample(range(1, L), p * v - 1))
            for pl, po in combos(v):
                fused, lists = realised(pr, v, pl, po, cuts)
                if lists is not None:
                    items.append((v, pl, fused, cuts, lists))
                    items.append((v, pl, fused, cuts, perturb(lists, prng, 3.0)))
        ok, _ = check(prep, pr, items)
        assert ok > 4
        plans = [{"v": v, "placement": pl, "policy": po, "S": p * v, "cuts": [0] + c + [L]}
                 for (v, c) in ((1, sorted(prng.sample(range(1, L), p - 1))),) for pl, po in combos(1)]
        got = prep.eval_plans(plans, report=True)
        for i, d in enumerate(plans):
            want = O.comm_accounting(pr, d["v"], d["placement"], d["policy"], d["cuts"][1:-1])
            assert got["status"][i] == want["status"]
            if want["status"] == 0:
                assert got["makespan"][i] == want["makespan"]
                for k in ("exposed_d", "overlap_d", "bubble_d"):  # R29 rows of the ABI report
                    assert list(got[k][i]) == want[k], k
    pr = W.Problem(t_f=[1, 1], t_b=[1, 1], t_w=[1, 1], act=[5, 5], stash=[0, 0], weight=[0, 0],
                   grad=[0, 0], comm=[0, 0], p=1, m=4, cap=25)
    prep = ctx.prepare(pr, W.Space([W.Group(1, W.FULL, combo_mask=0xF)]))
    r = prep.repair_oom({"v": 1, "placement": 0, "policy": LIST_FUSED, "S": 1, "cuts": [0, 2]},
                        [[(0, 0, j) for j in range(4)] + [(1, 0, j) for j in range(4)]])
    assert r["moves"] == 2 and r["status"] == 0 and r["makespan"] == 24


def test_eval_lists_shared_and_reordered_task_ranges(ctx):
    """Plans may share one task range or list their ranges out of order (ADVICE
    r1: the device copy is sized by the largest range end, not by the last
    plan's): results equal each plan evaluated alone."""
    from paper_2509_23722_b200 import adaptis as A
    import ctypes as C
    pr, sp = W.config(1)
    prep = ctx.prepare(pr, sp)
    L, p = len(pr.t_f), pr.p
    plans = [{"v": 1, "placement": 0, "policy": 4, "S": 2, "cuts": [0, c, L]} for c in (2, 4, 6)]
    fused, lists = realised(pr, 1, 0, 2, [4])
    tasks, one = A.Prepared._task_arrays([lists], p)
    n = len(plans)
    for offs in (np.tile(one, n),                                   # one shared range
                 np.concatenate([one + len(tasks), one, one])):      # first plan points past the others
        big = np.concatenate([tasks, tasks]) if offs[0] > 0 else tasks
        out = A._host_results(n)
        soa = A._soa_from_numpy(out)
        A._check(A.lib().adaptis_eval_lists(ctx.ptr, prep.ptr, A.make_plans(plans), big.ctypes.data,
                                            offs.astype(np.uint64).ctypes.data_as(C.POINTER(C.c_uint64)),
                                            n, C.byref(soa), None), ctx.ptr)
        for i, pl in enumerate(plans):
            alone = prep.eval_lists([pl], [lists])
            assert int(out["status"][i]) == int(alone["status"][0])
            assert int(out["makespan"][i]) == int(alone["makespan"][0])
