"""Oracle self-consistency (T2 of SURVEY §4.2): the event loop against the
independent longest-path checker, exact pruning against the plain search,
and invariants that hold for any correct simulator."""
import pytest

from oracle import oracle as O
from paper_2509_23722_b200 import workloads as W


def _random_case(rng, allow_wave=True):
    p = [1, 2, 3, 4][rng.next() % 4]
    v = 1 + rng.next() % 3
    m = p * (1 + rng.next() % 3) if v > 1 else 1 + rng.next() % 5
    S = p * v
    L = S + rng.next() % 4
    cap = W.INT64_MAX if rng.next() % 2 else 20 + rng.next() % 200
    pr = W.random_problem(rng, L, p, m, cmax=4, bytes_max=6, cap=cap)
    cuts = sorted(int(x) for x in _choose(rng, list(range(1, L)), S - 1))
    if v == 1:
        placement, policies = W.SEQ, [0, 1, 2, 3]
    elif allow_wave and rng.next() % 3 == 0:
        placement, policies = W.WAVE, [0, 3]
    else:
        placement, policies = W.INTERLEAVED, [0, 1, 2, 3]
    return pr, v, placement, policies, cuts


def _choose(rng, items, k):
    items = list(items)
    out = []
    for _ in range(k):
        out.append(items.pop(rng.next() % len(items)))
    return out


def test_event_loop_equals_longest_path_fixed_lists():
    """SURVEY T2 / S:224: >=200 random fixed-order plans with comm; the
    event loop equals the longest path over DAG + list edges."""
    rng = W.SplitMix64(2024)
    n = 0
    while n < 240:
        pr, v, placement, policies, cuts = _random_case(rng)
        for pol in (W.GPIPE, W.ONEF1B):
            if pol not in policies:
                continue
            r = O.simulate(pr, v, placement, pol, cuts)
            lists = [O.fixed_order(pr, v, placement, pol, cuts, d) for d in range(pr.p)]
            lp = O.longest_path(pr, v, placement, cuts, True, lists)
            if r["status"] == 3:
                assert lp is None
                continue
            assert lp is not None
            mk, Td, _ = lp
            assert r["T_d"] == Td
            if r["status"] == 0:
                assert r["makespan"] == mk
            n += 1


def test_event_loop_start_times_equal_longest_path_of_realised_order():
    """For every policy (incl. the dynamic ZB / GREEDY decisions) the realised
    per-device order, fed to the checker, reproduces every start time: the
    event loop never idles a device voluntarily."""
    rng = W.SplitMix64(77)
    n = 0
    while n < 300:
        pr, v, placement, policies, cuts = _random_case(rng)
        pol = policies[rng.next() % len(policies)]
        r = O.simulate(pr, v, placement, pol, cuts, trace=True)
        if r["status"] == 3:
            continue
        lists = [[(k, s, j) for (k, s, j, _) in dev] for dev in r["trace"]]
        fused = pol in (W.GPIPE, W.ONEF1B)
        lp = O.longest_path(pr, v, placement, cuts, fused, lists)
        assert lp is not None
        mk, Td, starts = lp
        assert starts == [[t[3] for t in dev] for dev in r["trace"]]
        assert Td == r["T_d"]
        n += 1


def test_lemma4_per_stage_mb_order():
    """DESIGN.md Lemma 4: on every stage, F, B and W each run in micro-batch order."""
    rng = W.SplitMix64(4)
    for _ in range(200):
        pr, v, placement, policies, cuts = _random_case(rng)
        for pol in (W.ZB, W.GREEDY):
            if pol not in policies:
                continue
            r = O.simulate(pr, v, placement, pol, cuts, trace=True)
            if r["status"] == 3:
                continue
            seen = {}
            for dev in r["trace"]:
                for (k, s, j, st) in sorted(dev, key=lambda t: t[3]):
                    last = seen.get((k, s), -1)
                    assert j == last + 1
                    seen[(k, s)] = j


def test_lower_bound_and_busy():
    rng = W.SplitMix64(11)
    for _ in range(150):
        pr, v, placement, policies, cuts = _random_case(rng)
        for pol in policies:
            r = O.simulate(pr, v, placement, pol, cuts)
            if r["status"] != 0:
                continue
            assert max(r["busy_d"]) <= r["makespan"]
            assert sum(r["busy_d"]) == pr.m * int(sum(pr.t_f) + sum(pr.t_b) + sum(pr.t_w))
            assert 0.0 <= r["bubble"] < 1.0


def test_fixed_order_monotone():
    """Fixed orders are longest paths, hence monotone in every duration."""
    rng = W.SplitMix64(12)
    for _ in range(100):
        pr, v, placement, policies, cuts = _random_case(rng)
        pr.cap = W.INT64_MAX
        for pol in (W.GPIPE, W.ONEF1B):
            if pol not in policies:
                continue
            base = O.simulate(pr, v, placement, pol, cuts)
            if base["status"] != 0:
                continue
            col = ["t_f", "t_b", "t_w"][rng.next() % 3]
            row = rng.next() % pr.L
            getattr(pr, col)[row] += 1 + rng.next() % 5
            bigger = O.simulate(pr, v, placement, pol, cuts)
            assert bigger["makespan"] >= base["makespan"]


def test_pruned_search_equals_plain_search():
    rng = W.SplitMix64(31)
    for trial in range(12):
        p = 2 + rng.next() % 2
        m = p * (1 + rng.next() % 2)
        L = 2 * p + 2 + rng.next() % 3
        cap = W.INT64_MAX if trial % 2 else 60 + rng.next() % 60
        pr = W.random_problem(rng, L, p, m, bytes_max=8, cap=cap)
        sp = W.Space([W.Group(1, W.FULL, combo_mask=0xF), W.Group(2, W.BALL, 2, combo_mask=0x3F)])
        a = O.search(pr, sp, prune=False, nthreads=2)
        b = O.search(pr, sp, prune=True, nthreads=3)
        assert (a["index"], a["makespan"]) == (b["index"], b["makespan"])
        assert a["n_total"] == b["n_total"] == O.space_size(pr, sp)
        # brute force over eval_indices
        N = O.space_size(pr, sp)
        ev = O.eval_indices(pr, sp, range(N))
        feas = [(int(ev["makespan"][i]), i) for i in range(N) if ev["status"][i] == 0]
        if feas:
            assert min(feas) == (a["makespan"], a["index"])
        else:
            assert a["index"] == O.UINT64_MAX


def test_stuck_greedy_reports_status_3():
    """GREEDY with a cap that admits no forward stalls (status 3, R14)."""
    pr = W.Problem(t_f=[1, 1], t_b=[1, 1], t_w=[1, 1], act=[5, 5], stash=[0, 0], weight=[1, 1],
                   grad=[0, 0], comm=[0, 0], p=2, m=2, cap=5)
    r = O.simulate(pr, 1, W.SEQ, W.GREEDY, [1])
    assert r["status"] == 3 and r["makespan"] == O.INT64_MAX
