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


def test_greedy_trace_satisfies_r14_rule():
    """An independent checker of R14 ("advances the F first, followed by the
    B, and finally the W within the memory constraints") on the event loop's
    GREEDY traces: at every decision of every device, the candidates are the next
    unissued F of each own stage (only if static + dyn + act + stash fits the
    cap), every B whose F is done, every pending W; the task started is at
    max(device free, earliest candidate ready time) and has the smallest (kind,
    mb, stage) key among the candidates ready by then. Ready times come from the
    final trace (anything scheduled later is ready strictly later, R17)."""
    import random as _r
    rng = W.SplitMix64(1414)
    checked = 0
    for t in range(60):
        p = [1, 2, 3, 4][t % 4]
        L = 2 * p + 3
        m = 2 * p
        cap = W.INT64_MAX if t % 3 else 60 + 9 * t
        pr = W.random_problem(rng, L, p, m, tmax=7, cmax=4, bytes_max=6, cap=cap)
        v = 1 + (t % 2)
        S = p * v
        cuts = sorted(_r.Random(t).sample(range(1, L), S - 1))
        for pl in ([0] if v == 1 else [1, 2]):
            r = O.simulate(pr, v, pl, 3, cuts, trace=True)
            if r["status"] == 3:
                continue
            full = [0] + cuts + [L]
            ssum = lambda col, s: int(sum(col[full[s]:full[s + 1]]))  # noqa: E731
            dur = {0: [ssum(pr.t_f, s) for s in range(S)], 1: [ssum(pr.t_b, s) for s in range(S)],
                   2: [ssum(pr.t_w, s) for s in range(S)]}
            act = [ssum(pr.act, s) for s in range(S)]
            sta = [ssum(pr.stash, s) for s in range(S)]
            wg = [ssum(pr.weight, s) + ssum(pr.grad, s) for s in range(S)]
            dev = [O.device_of_stage(pl, p, v, s) for s in range(S)]
            lat = [int(pr.comm[full[s + 1] - 1]) if s + 1 < S and dev[s + 1] != dev[s] else 0 for s in range(S)]
            fin = {}
            for lst in r["trace"]:
                for (k, s, j, st) in lst:
                    fin[(k, s, j)] = st + dur[k][s]

            def ready(k, s, j):
                if k == 0:
                    return 0 if s == 0 else fin[(0, s - 1, j)] + lat[s - 1]
                if k == 1:
                    x = fin[(0, s, j)]
                    return max(x, fin[(1, s + 1, j)] + lat[s]) if s + 1 < S else x
                return fin[(1, s, j)]
            for d, lst in enumerate(r["trace"]):
                own = [s for s in range(S) if dev[s] == d]
                stat = sum(wg[s] for s in own)
                done, dyn, free = set(), 0, 0
                for (k, s, j, st) in lst:
                    cand = []
                    for s2 in own:
                        nf = min([j2 for j2 in range(m) if (0, s2, j2) not in done], default=None)
                        if nf is not None and stat + dyn + act[s2] + sta[s2] <= pr.cap:
                            cand.append((0, s2, nf))
                        for j2 in range(m):
                            if (0, s2, j2) in done and (1, s2, j2) not in done:
                                cand.append((1, s2, j2))
                            if (1, s2, j2) in done and (2, s2, j2) not in done:
                                cand.append((2, s2, j2))
                    at = max(free, min(ready(*c) for c in cand))
                    assert st == at, (t, d, (k, s, j))
                    best = min((c for c in cand if ready(*c) <= at), key=lambda c: (c[0], c[2], c[1]))
                    assert best == (k, s, j), (t, d, best, (k, s, j))
                    done.add((k, s, j))
                    free = st + dur[k][s]
                    dyn += act[s] + sta[s] if k == 0 else (-act[s] if k == 1 else -sta[s])
                    checked += 1
    assert checked > 3000


def test_zb_trace_satisfies_r13_rule():
    """An independent checker of R13 ("only reschedules W to fill bubbles")
    on the event loop's ZB traces: the F/B tasks follow the R9/R10 list; before
    each of them (ready time r) the oldest pending Ws (B-completion order) run
    while the F would not fit under the cap, then while free < r; the F/B then
    starts at max(free, r); leftover Ws run in order at the end."""
    import random as _r
    rng = W.SplitMix64(1313)
    checked = 0
    for t in range(60):
        p = [1, 2, 3, 4][t % 4]
        L = 2 * p + 3
        m = 2 * p
        cap = W.INT64_MAX if t % 3 else 60 + 9 * t
        pr = W.random_problem(rng, L, p, m, tmax=7, cmax=4, bytes_max=6, cap=cap)
        v = 1 + (t % 2)
        S = p * v
        pl = 0 if v == 1 else 1
        cuts = sorted(_r.Random(t).sample(range(1, L), S - 1))
        r = O.simulate(pr, v, pl, 2, cuts, trace=True)
        if r["status"] == 3:
            continue
        full = [0] + cuts + [L]
        ssum = lambda col, s: int(sum(col[full[s]:full[s + 1]]))  # noqa: E731
        dur = {0: [ssum(pr.t_f, s) for s in range(S)], 1: [ssum(pr.t_b, s) for s in range(S)],
               2: [ssum(pr.t_w, s) for s in range(S)]}
        act = [ssum(pr.act, s) for s in range(S)]
        sta = [ssum(pr.stash, s) for s in range(S)]
        wg = [ssum(pr.weight, s) + ssum(pr.grad, s) for s in range(S)]
        dev = [O.device_of_stage(pl, p, v, s) for s in range(S)]
        lat = [int(pr.comm[full[s + 1] - 1]) if s + 1 < S and dev[s + 1] != dev[s] else 0 for s in range(S)]
        fin = {(k, s, j): st + dur[k][s] for lst in r["trace"] for (k, s, j, st) in lst}

        def ready(k, s, j):
            if k == 0:
                return 0 if s == 0 else fin[(0, s - 1, j)] + lat[s - 1]
            x = fin[(0, s, j)]
            return max(x, fin[(1, s + 1, j)] + lat[s]) if s + 1 < S else x
        for d, lst in enumerate(r["trace"]):
            fb = [(k, s, j) for (k, s, j, _st) in lst if k < 2]
            assert fb == [tuple(x) for x in O.fixed_order(pr, v, pl, 2, cuts, d)]
            stat = sum(wg[s] for s in range(S) if dev[s] == d)
            pend, free, dyn, i = [], 0, 0, 0
            for task in fb + [None]:
                k, s, j = task if task is not None else (None, None, None)
                # the Ws the rule runs before this F/B (or all leftovers at the end)
                want = []
                q = list(pend)
                f2, dy2 = free, dyn
                rr = ready(k, s, j) if task is not None else None
                while q:
                    if k is None or (k == 0 and stat + dy2 + act[s] + sta[s] > pr.cap) or f2 < rr:
                        w = q.pop(0)
                        want.append(w)
                        f2 += dur[2][w[1]]
                        dy2 -= sta[w[1]]
                    else:
                        break
                for w in want:
                    kk, ss, jj, st = lst[i]
                    assert (kk, ss, jj) == w and st == free, (t, d, w, lst[i])
                    free = st + dur[2][ss]
                    dyn -= sta[ss]
                    pend.remove(w)
                    i += 1
                    checked += 1
                if k is None:
                    break
                kk, ss, jj, st = lst[i]
                assert (kk, ss, jj) == (k, s, j) and st == max(free, rr), (t, d, (k, s, j), lst[i])
                free = st + dur[k][s]
                dyn += act[s] + sta[s] if k == 0 else -act[s]
                if k == 1:
                    pend.append((2, s, j))
                i += 1
                checked += 1
            assert i == len(lst)
    assert checked > 3000
