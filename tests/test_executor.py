"""Executor lowering (reading R33, CPU only):
the library's adaptis_lower against oracle/executor.py, SPEC's worked
examples, and the equivalence properties of the emitted programs."""
import random

import pytest

from oracle import executor as X
from oracle import oracle as O
from paper_2509_23722_b200 import adaptis as A
from paper_2509_23722_b200 import workloads as W

C_F, C_B, C_W, S_F, S_B, R_F, R_B, W_F, W_B = range(9)


def _plan(p, v, placement, fused):
    return {"v": v, "placement": placement, "policy": 5 if fused else 4, "S": p * v,
            "cuts": [0] * (p * v + 1)}


def test_spec_two_device_layout():
    """S:452 example: 2 devices, S = 2, one micro-batch, fused:
    d0 = [C_F, S_F, R_B, W_B, C_B]; d1 = [R_F, W_F, C_F, C_B, S_B]."""
    lists = [[(0, 0, 0), (1, 0, 0)], [(0, 1, 0), (1, 1, 0)]]
    want = [[(C_F, 0, 0, -1), (S_F, 0, 0, 1), (R_B, 0, 0, 1), (W_B, 0, 0, 1), (C_B, 0, 0, -1)],
            [(R_F, 0, 0, 0), (W_F, 0, 0, 0), (C_F, 1, 0, -1), (C_B, 1, 0, -1), (S_B, 0, 0, 0)]]
    assert X.emit(2, 2, [0, 1], lists) == want
    got = A.lower(2, _plan(2, 1, 0, True), lists, repair=False, hoist=False)
    assert got["programs"] == want
    assert X.check(want) is None


def test_spec_cross_case_repair():
    """crossing sends deadlock (frontier d0@S_F(a), d1@S_B(b)); the
    repair hoists d0's R_B(b) in front of its S_F(a) and the run completes."""
    prog = [[(C_F, 0, 1, -1), (S_F, 0, 1, 1), (R_B, 0, 0, 1), (W_B, 0, 0, 1), (C_B, 0, 0, -1)],
            [(C_B, 1, 0, -1), (S_B, 0, 0, 0), (R_F, 0, 1, 0), (W_F, 0, 1, 0), (C_F, 1, 1, -1)]]
    assert X.check(prog) == [1, 1]
    fixed, n = X.repair(prog)
    assert n == 1 and fixed[0][:3] == [(C_F, 0, 1, -1), (R_B, 0, 0, 1), (S_F, 0, 1, 1)]
    assert X.check(fixed) is None


def _cases():
    rng = W.SplitMix64(33)
    prng = random.Random(33)
    for t in range(24):
        p = [2, 3, 4][t % 3]
        L = 2 * p + 3
        pr = W.random_problem(rng, L, p, 2 * p, tmax=6, cmax=3, bytes_max=0)
        v = 1 + (t % 2)
        S = p * v
        cuts = sorted(prng.sample(range(1, L), S - 1))
        combos = [(0, 1), (0, 2), (0, 3)] if v == 1 else [(1, 1), (1, 2), (2, 3)]
        pl, po = combos[t % 3]
        r = O.simulate(pr, v, pl, po, cuts, trace=True)
        if r["status"] == 3:
            continue
        fused = po in (0, 1)
        lists = [[(k, s, j) for (k, s, j, _) in lst if not (fused and k == 2)] for lst in r["trace"]]
        dev = [O.device_of_stage(pl, p, v, s) for s in range(S)]
        yield p, v, S, pl, fused, dev, lists


def test_library_equals_oracle():
    n = 0
    for p, v, S, pl, fused, dev, lists in _cases():
        want, wr, wh = X.lower(p, S, dev, lists)
        got = A.lower(p, _plan(p, v, pl, fused), lists)
        assert got["programs"] == want and (got["repairs"], got["hoists"]) == (wr, wh)
        n += 1
    assert n > 15


def test_lowered_programs_are_equivalent_and_complete():
    """SPEC verify_equivalence: per device the compute order is the schedule's;
    every cross-device edge has exactly one S, R and W with consistent peers; the
    repaired + hoisted programs complete under rendezvous semantics."""
    hoisted = 0
    for p, v, S, pl, fused, dev, lists in _cases():
        got = A.lower(p, _plan(p, v, pl, fused), lists)
        prog = got["programs"]
        hoisted += got["hoists"]
        assert X.check(prog) is None
        for d in range(p):
            comp = [(op, s, j) for (op, s, j, _) in prog[d] if op <= C_W]
            assert comp == lists[d]
        sends = {(op, b, j, d, e) for d in range(p) for (op, b, j, e) in prog[d] if op in (S_F, S_B)}
        recvs = {(op - 2, b, j, e, d) for d in range(p) for (op, b, j, e) in prog[d] if op in (R_F, R_B)}
        waits = {(op - 4, b, j, e, d) for d in range(p) for (op, b, j, e) in prog[d] if op in (W_F, W_B)}
        assert sends == recvs == waits
        edges = sum(1 for d in range(p) for (k, s, j) in lists[d]
                    if (k == 0 and s + 1 < S and dev[s + 1] != d) or (k == 1 and s > 0 and dev[s - 1] != d))
        assert len(sends) == edges
    assert hoisted > 0


def test_unrepairable_and_bad_input():
    with pytest.raises(A.AdaptisError):
        A.lower(2, _plan(2, 1, 0, True), [[(0, 1, 0), (1, 1, 0)], [(0, 0, 0), (1, 0, 0)]])  # wrong devices


def test_s1f1b_naive_lowering_deadlocks_and_is_repaired():
    """S-1F1B, p = 2, m = 2 (S:288 lists): the naive emission deadlocks exactly as
    Fig. 9's cross case (d0 sends F(0,1) while d1 sends B(1,0)); one repair hoists
    d0's R_B(0,0) in front of its S_F(0,1)."""
    lists = [[(0, 0, 0), (0, 0, 1), (1, 0, 0), (1, 0, 1)], [(0, 1, 0), (1, 1, 0), (0, 1, 1), (1, 1, 1)]]
    naive = X.emit(2, 2, [0, 1], lists)
    assert X.check(naive) is not None
    got = A.lower(2, _plan(2, 1, 0, True), lists, hoist=False)
    assert got["repairs"] == 1
    assert got["programs"][0][:5] == [(C_F, 0, 0, -1), (S_F, 0, 0, 1), (C_F, 0, 1, -1), (R_B, 0, 0, 1),
                                      (S_F, 0, 1, 1)]
    assert X.check(got["programs"]) is None
