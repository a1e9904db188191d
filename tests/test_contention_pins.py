"""Pins of the engine-contention oracle (oracle/contention.py, reading R34;
SPEC S:206 (a)-(c)) against things other than itself:
  * special case with no transfer (all latencies 0, or p = 1): it reduces to
    the uncontended longest path of R30 (oracle.simulate_lists);
  * special case with no conflict: when the uncontended schedule never has
    two transfers on one engine at once, contention changes nothing;
  * closed form: GPipe with uniform stages is two permutation flow shops of
    identical jobs, machines compute / link / compute / ..., whose makespan is
    sum of the machine times + (m - 1) * the largest (textbook flow-shop
    bound for identical jobs);
  * the defining equations, checked on the trace by an independent checker:
    per engine, transfers in (eligible, mb, stage, F<B) order and each starting
    at max(eligible, previous arrival on its send engine, on its receive
    engine); per device, tasks in list order starting at max(previous finish,
    inputs ready);
  * invariant: contention never shortens the makespan."""
import random

import pytest

from oracle import oracle as O
from oracle.contention import simulate_lists_contended as SC
from paper_2509_23722_b200 import workloads as W


def realised(pr, v, pl, po, cuts):
    r = O.simulate(pr, v, pl, po, cuts, trace=True)
    if r["status"] == 3:
        return po in (0, 1), None
    fused = po in (0, 1)
    return fused, [[(k, s, j) for (k, s, j, _t) in lst if not (fused and k == 2)] for lst in r["trace"]]


def combos(v):
    return [(0, k) for k in range(4)] if v == 1 else [(1, k) for k in range(4)] + [(2, 0), (2, 3)]


def cases(seed, n, cmax=4, zero_comm=False):
    rng = W.SplitMix64(900 + seed)
    prng = random.Random(seed)
    for t in range(n):
        p = [1, 2, 3, 4][t % 4]
        L = 2 * p + 3
        pr = W.random_problem(rng, L, p, 2 * p, tmax=6, cmax=cmax, bytes_max=4,
                              cap=W.INT64_MAX if t % 3 else 40 + 7 * t)
        if zero_comm:
            pr.comm[:] = 0
        for v in (1, 2):
            cuts = sorted(prng.sample(range(1, L), p * v - 1))
            for pl, po in combos(v):
                fused, lists = realised(pr, v, pl, po, cuts)
                if lists is not None:
                    yield pr, v, pl, fused, cuts, lists


def test_zero_latency_reduces_to_longest_path():
    n = 0
    for pr, v, pl, fused, cuts, lists in cases(1, 8, zero_comm=True):
        a = SC(pr, v, pl, fused, cuts, lists)
        b = O.simulate_lists(pr, v, pl, fused, cuts, lists)
        for key in ("status", "makespan", "peak_mem", "T_d", "busy_d", "M_d"):
            assert a[key] == b[key], key
        n += 1
    assert n > 30


def _uncontended_engine_conflict(pr, v, pl, fused, cuts, lists):
    """True if two transfers of the R30 (latency-only) schedule overlap on one engine."""
    L, p = len(pr.t_f), pr.p
    full = [0] + list(cuts) + [L]
    S = len(full) - 1
    lp = O.longest_path(pr, v, pl, cuts, fused, lists)
    dur_f = [sum(pr.t_f[full[s]:full[s + 1]]) for s in range(S)]
    dur_b = [sum(pr.t_b[full[s]:full[s + 1]]) + (sum(pr.t_w[full[s]:full[s + 1]]) if fused else 0)
             for s in range(S)]
    dev = [O.device_of_stage(pl, p, v, s) for s in range(S)]
    eng = {}
    for d in range(p):
        for (k, s, j), st in zip(lists[d], lp[2][d]):
            if k == 0 and s + 1 < S and dev[s + 1] != d:
                lat, tgt, fin = int(pr.comm[full[s + 1] - 1]), dev[s + 1], st + dur_f[s]
            elif k == 1 and s > 0 and dev[s - 1] != d:
                lat, tgt, fin = int(pr.comm[full[s] - 1]), dev[s - 1], st + dur_b[s]
            else:
                continue
            if lat == 0:
                continue
            eng.setdefault(("s", d), []).append((fin, fin + lat))
            eng.setdefault(("r", tgt), []).append((fin, fin + lat))
    for ivs in eng.values():
        ivs.sort()
        if any(b[0] < a[1] for a, b in zip(ivs, ivs[1:])):
            return True
    return False


def test_no_conflict_means_no_change_and_contention_never_helps():
    n_same = n_diff = 0
    for pr, v, pl, fused, cuts, lists in cases(2, 16, cmax=6):
        a = SC(pr, v, pl, fused, cuts, lists)
        b = O.simulate_lists(pr, v, pl, fused, cuts, lists)
        assert a["status"] == b["status"] and a["M_d"] == b["M_d"]
        if b["status"] == 3:
            continue
        lp = O.longest_path(pr, v, pl, cuts, fused, lists)
        assert max(a["T_d"]) >= lp[0]
        if not _uncontended_engine_conflict(pr, v, pl, fused, cuts, lists):
            assert a["T_d"] == lp[1]
            n_same += 1
        elif max(a["T_d"]) > lp[0]:
            n_diff += 1
    assert n_same > 10 and n_diff > 10  # both regimes exercised


@pytest.mark.parametrize("p,m,f,tb,tw,c", [(2, 4, 1, 1, 1, 3), (3, 5, 2, 1, 1, 4), (4, 6, 3, 2, 3, 2),
                                           (4, 3, 1, 1, 1, 7), (5, 8, 2, 2, 1, 2), (2, 1, 4, 3, 1, 9)])
def test_gpipe_flow_shop_closed_form(p, m, f, tb, tw, c):
    """GPipe (F0..F(m-1) then B0..B(m-1) on every device), one row per stage of
    costs f / b = tb + tw (fused B+W) and latency c: the forward phase is the
    flow shop f, c, f, ..., f (2p - 1 machines) of m identical jobs; the
    backward phase starts when the last device ends its forwards and is the
    flow shop b, c, ..., b. Makespan = p*f + (p-1)*c + (m-1)*max(f, c) + p*b +
    (p-1)*c + (m-1)*max(b, c)."""
    z = [0] * p
    pr = W.Problem(t_f=[f] * p, t_b=[tb] * p, t_w=[tw] * p, act=z, stash=z, weight=z, grad=z,
                   comm=[c] * p, p=p, m=m)
    b = tb + tw
    lists = [[(0, d, j) for j in range(m)] + [(1, d, j) for j in range(m)] for d in range(p)]
    r = SC(pr, 1, 0, True, list(range(1, p)), lists)
    want = p * f + (p - 1) * c + (m - 1) * max(f, c) + p * b + (p - 1) * c + (m - 1) * max(b, c)
    assert r["status"] == 0 and r["makespan"] == want
    if c <= min(f, b):  # the uncontended GPipe closed form (m+p-1)(f+b) + 2(p-1)c
        assert want == (m + p - 1) * (f + b) + 2 * (p - 1) * c


def _check_equations(pr, v, pl, fused, cuts, lists, r):
    L, p = len(pr.t_f), pr.p
    full = [0] + list(cuts) + [L]
    S = len(full) - 1
    dev = [O.device_of_stage(pl, p, v, s) for s in range(S)]
    fin = {}
    for d in range(p):
        assert [x[2] for x in r["tasks"][d]] == list(lists[d])
        for (a, b_, t) in r["tasks"][d]:
            fin[t] = b_
    arr = {x[4]: x[3] for x in r["transfers"]}
    elig = {x[4]: fin[x[4]] for x in r["transfers"]}
    # per engine: order by (eligible, mb, stage, kind), start = max(eligible, both engines free)
    order = sorted(r["transfers"], key=lambda x: (elig[x[4]], x[4][2], x[4][1], x[4][0]))
    sf, rf = [0] * p, [0] * p
    for (src, dst, st, ar, t) in order:
        k, s, j = t
        assert st == max(elig[t], sf[src], rf[dst])
        lat = int(pr.comm[full[s + 1] - 1]) if k == 0 else int(pr.comm[full[s] - 1])
        assert ar == st + lat and lat > 0 and src == dev[s] and src != dst
        sf[src] = rf[dst] = ar

    def over_edge(q):  # a stage edge's output: its arrival if it travelled
        return arr.get(q, fin[q])
    for d in range(p):
        prev = 0
        for (a, b_, (k, s, j)) in r["tasks"][d]:
            if k == 0:
                ins = [over_edge((0, s - 1, j))] if s > 0 else []
            elif k == 1:
                ins = [fin[(0, s, j)]] + ([over_edge((1, s + 1, j))] if s + 1 < S else [])
            else:
                ins = [fin[(1, s, j)]]
            assert a == max([prev] + ins)
            prev = b_


def test_trace_satisfies_the_defining_equations():
    n = 0
    for pr, v, pl, fused, cuts, lists in cases(3, 12, cmax=7):
        r = SC(pr, v, pl, fused, cuts, lists, trace=True)
        if r["status"] == 3:
            continue
        _check_equations(pr, v, pl, fused, cuts, lists, r)
        for d in range(pr.p):  # R29 identity with the contended transfers
            # exposed_d by brute force on the tick grid
            busy_t, xt = set(), set()
            for (a, b_, _x) in r["tasks"][d]:
                busy_t.update(range(a, b_))
            for (src, dst, a, b_, _x) in r["transfers"]:
                if d in (src, dst):
                    xt.update(range(a, min(b_, r["T_d"][d])))
            assert r["exposed_d"][d] == len(xt - busy_t)
            assert 0 <= r["exposed_d"][d] <= r["comm_d"][d]
            assert r["T_d"][d] - r["busy_d"][d] - r["exposed_d"][d] >= 0
        n += 1
    assert n > 40


def test_cyclic_wait_is_stuck():
    z = [0, 0]
    pr = W.Problem(t_f=[1, 1], t_b=[1, 1], t_w=[1, 1], act=z, stash=z, weight=z, grad=z,
                   comm=[2, 0], p=2, m=2)
    d0 = [(0, 0, 0), (1, 0, 0), (0, 0, 1), (1, 0, 1)]
    r = SC(pr, 1, 0, True, [1], [d0, [(0, 1, 0), (1, 1, 0), (0, 1, 1), (1, 1, 1)]])
    # per micro-batch, serially: F(0) 1, link 2, F(1) 1, B(1) 2, link 2, B(0) 2
    assert r["status"] == 0 and r["makespan"] == 20
    # device 1 wants F(1, 1) before B(1, 0); device 0 sends F(0, 1) only after B(0, 0)
    r = SC(pr, 1, 0, True, [1], [d0, [(0, 1, 0), (0, 1, 1), (1, 1, 0), (1, 1, 1)]])
    assert r["status"] == 3 and r["makespan"] == INT64_MAX and r["peak_mem"] == 0


INT64_MAX = (1 << 63) - 1
