"""Pins of the CPU oracle against what the paper and the mathematics fix
(closed forms, SPEC/paper worked examples, brute force on tiny inputs).

None of these re-types the oracle's formulas: each expected value comes from a
closed form, a cited worked example (tests/golden/), or an exhaustive
brute force written here in plain Python.
"""
import itertools
import json
import math
import os
import random
from fractions import Fraction

import numpy as np
import pytest

from oracle import oracle as O
from paper_2509_23722_b200 import workloads as W

GOLD = os.path.join(os.path.dirname(__file__), "golden")
SPEC = json.load(open(os.path.join(GOLD, "spec_examples.json")))
CFG1 = json.load(open(os.path.join(GOLD, "cfg1_unit.json")))


def homo(L, p, m, tf, tb, tw, comm=0, act=0, stash=0, weight=0, cap=W.INT64_MAX):
    return W.Problem(t_f=[tf] * L, t_b=[tb] * L, t_w=[tw] * L, act=[act] * L, stash=[stash] * L,
                     weight=[weight] * L, grad=[0] * L, comm=[comm] * L, p=p, m=m, cap=cap)


def seq_cuts(S):
    return list(range(1, S))


# ---------------------------------------------------------------- Alg. 1 Step 1
def test_stage_sums_whole_model_equals_column_sums():
    """with S = 1 the stage cost is the column sum; busy = m * sum (Alg.1 Step 1-2)."""
    pr = W.random_problem(W.SplitMix64(7), 9, 1, 3)
    for pol in range(4):
        r = O.simulate(pr, 1, W.SEQ, pol, [])
        total = sum(int(pr.t_f[i] + pr.t_b[i] + pr.t_w[i]) for i in range(9))
        assert r["busy_d"] == [3 * total]
        assert r["makespan"] == 3 * total  # serial device: no bubbles
        assert r["static_d"] == [int(pr.weight.sum() + pr.grad.sum())]


def test_stage_sum_pair_spec_example():
    ex = SPEC["stage_sum_pair"]
    pr = W.Problem(t_f=ex["t_f"] + [1], t_b=[1] * 3, t_w=[1] * 3, act=[0] * 3, stash=[0] * 3,
                   weight=[0] * 3, grad=[0] * 3, comm=[0] * 3, p=2, m=1)
    # stage 0 = rows {0,1}: with m=1 GPIPE on 2 devices the F of stage 1 starts at c_F(0)
    r = O.simulate(pr, 1, W.SEQ, W.GPIPE, [2], trace=True)
    f1 = [t for t in r["trace"][1] if t[0] == 0][0]
    assert f1[3] == ex["c_F"]


def test_serial_example():
    ex = SPEC["serial"]
    tf, tb, tw = ex["t"]
    pr = homo(1, 1, ex["m"], tf, tb, tw)
    for pol in range(4):
        r = O.simulate(pr, 1, W.SEQ, pol, [])
        assert r["makespan"] == ex["makespan"]
        assert r["bubble"] == 0.0


# ---------------------------------------------------------------- placements (R12)
@pytest.mark.parametrize("key,placement", [("interleaved_4_2", W.INTERLEAVED),
                                           ("wave_4_2", W.WAVE), ("wave_8_4", W.WAVE)])
def test_placement_examples(key, placement):
    ex = SPEC[key]
    v = ex["S"] // ex["p"]
    assert [O.device_of_stage(placement, ex["p"], v, s) for s in range(ex["S"])] == ex["dev"]


def test_combo_table():
    assert [O.combo(1, k) for k in range(5)] == [(0, 0), (0, 1), (0, 2), (0, 3), None]
    assert [O.combo(2, k) for k in range(7)] == [(1, 0), (1, 1), (1, 2), (1, 3), (2, 0), (2, 3), None]


# ---------------------------------------------------------------- orders (R9-R11)
def _fmt(lst):
    return [("F" if k == 0 else "B") + str(j + 1) for (k, s, j) in lst]


def test_s1f1b_lists_spec_example():
    ex = SPEC["s1f1b_lists"]
    pr = homo(2, 2, 3, 1, 1, 1)
    assert _fmt(O.fixed_order(pr, 1, W.SEQ, W.ONEF1B, [1], 0)) == ex["dev0"]
    assert _fmt(O.fixed_order(pr, 1, W.SEQ, W.ONEF1B, [1], 1)) == ex["dev1"]


def test_interleaved_order_megatron_structure():
    """R10: warm-up length, chunk pattern and completeness of each list."""
    p, v, m = 4, 2, 8
    pr = homo(p * v, p, m, 1, 1, 1)
    for d in range(p):
        lst = O.fixed_order(pr, v, W.INTERLEAVED, W.ONEF1B, seq_cuts(p * v), d)
        w = min(m * v, 2 * (p - d - 1) + (v - 1) * p)
        kinds = [k for k, _, _ in lst]
        assert kinds[:w] == [0] * w and kinds[w] == 0 and kinds[w + 1] == 1
        assert sorted((k, s, j) for k, s, j in lst) == sorted(
            (k, c * p + d, j) for k in (0, 1) for c in range(v) for j in range(m))
        fw = [(s, j) for k, s, j in lst if k == 0]
        # the first p forwards are chunk 0, micro-batches 0..p-1; then chunk 1
        assert fw[:p] == [(d, j) for j in range(p)]
        assert fw[p:2 * p] == [(p + d, j) for j in range(p)]


# ---------------------------------------------------------------- closed forms
@pytest.mark.parametrize("p", [2, 4, 8])
@pytest.mark.parametrize("mult", [0, 1, 2, 4])
@pytest.mark.parametrize("c", [0, 1, 2, 7])
def test_gpipe_makespan_closed_form(p, mult, c):
    """GPipe: (m+p-1)(t_f+t_b) + 2(p-1)c with uniform comm c (north_star closed form)."""
    m = 1 if mult == 0 else mult * p
    tf, tb, tw = 3, 4, 2
    pr = homo(p, p, m, tf, tb, tw, comm=c)
    r = O.simulate(pr, 1, W.SEQ, W.GPIPE, seq_cuts(p))
    assert r["makespan"] == (m + p - 1) * (tf + tb + tw) + 2 * (p - 1) * c


@pytest.mark.parametrize("p", [2, 3, 4, 8])
@pytest.mark.parametrize("m", [1, 2, 3, 4, 8, 16, 32])
def test_s1f1b_makespan_and_bubble_closed_form(p, m):
    """S-1F1B at zero comm: (m+p-1)(t_f+t_b) for any m; bubble = (p-1)/(m+p-1)."""
    tf, tb, tw = 5, 7, 3
    pr = homo(p, p, m, tf, tb, tw)
    r = O.simulate(pr, 1, W.SEQ, W.ONEF1B, seq_cuts(p))
    assert r["makespan"] == (m + p - 1) * (tf + tb + tw)
    busy = sum(r["busy_d"])
    assert Fraction(p * r["makespan"] - busy, p * r["makespan"]) == Fraction(p - 1, m + p - 1)
    assert abs(r["bubble"] - (p - 1) / (m + p - 1)) < 1e-12


@pytest.mark.parametrize("p", [2, 4, 8])
@pytest.mark.parametrize("v", [2, 3, 4])
@pytest.mark.parametrize("q", [1, 2, 4])
def test_interleaved_1f1b_closed_form(p, v, q):
    """I-1F1B: makespan (vm+p-1)(f+b) in per-chunk costs, bubble (p-1)/(vm+p-1) (1/v of S-1F1B's)."""
    m = q * p
    tf, tb, tw = 2, 3, 1
    pr = homo(p * v, p, m, tf, tb, tw)
    r = O.simulate(pr, v, W.INTERLEAVED, W.ONEF1B, seq_cuts(p * v))
    assert r["makespan"] == (v * m + p - 1) * (tf + tb + tw)
    assert abs(r["bubble"] - (p - 1) / (v * m + p - 1)) < 1e-12
    r1 = O.simulate(homo(p, p, m, v * tf, v * tb, v * tw), 1, W.SEQ, W.ONEF1B, seq_cuts(p))
    # the same model on v-times coarser stages (S-1F1B): bubble (p-1)/(m+p-1)
    assert abs(r1["bubble"] - (p - 1) / (m + p - 1)) < 1e-12 and r["bubble"] < r1["bubble"]


def test_s1f1b_worked_example_scaled():
    """S:209 (t_F = t_B = 1, t_W = 0, fused) in units of 2 ticks (t_W >= 1 by R17)."""
    ex = SPEC["s1f1b_p2_m2"]
    pr = homo(2, 2, 2, 2, 1, 1)
    r = O.simulate(pr, 1, W.SEQ, W.ONEF1B, [1])
    assert r["makespan"] == ex["scale"] * ex["makespan"]
    assert r["T_d"] == [ex["scale"] * t for t in ex["T_d"]]


def test_zb_wfill_7_vs_immediate_w_8():
    ex = SPEC["zb_p2_m2"]
    pr = homo(2, 2, 2, 1, 1, 1)
    assert O.simulate(pr, 1, W.SEQ, W.ZB, [1])["makespan"] == ex["makespan_wfill"]
    # immediate W: the 1F1B list with each W right after its B (independent checker)
    lists = []
    for d in range(2):
        lst = []
        for (k, s, j) in O.fixed_order(pr, 1, W.SEQ, W.ONEF1B, [1], d):
            lst.append((k, s, j))
            if k == 1:
                lst.append((2, s, j))
        lists.append(lst)
    mk, _, _ = O.longest_path(pr, 1, W.SEQ, [1], False, lists)
    assert mk == ex["makespan_immediate_w"]


@pytest.mark.parametrize("p", [2, 4, 8])
@pytest.mark.parametrize("q", [1, 2, 4])
def test_zb_equal_costs_closed_form(p, q):
    """ZB W-fill with t_F = t_B = t_W = t and m >= p: (3m+p-1) t (R13)."""
    m, t = q * p, 3
    pr = homo(p, p, m, t, t, t)
    assert O.simulate(pr, 1, W.SEQ, W.ZB, seq_cuts(p))["makespan"] == (3 * m + p - 1) * t


@pytest.mark.parametrize("p", [2, 4, 8])
@pytest.mark.parametrize("m", [1, 2, 4, 8, 16])
def test_greedy_closed_form(p, m):
    """GREEDY, cap = inf, zero comm, homogeneous: (m+p-1)(t_f+t_b) + m t_w (R14)."""
    tf, tb, tw = 4, 6, 3
    pr = homo(p, p, m, tf, tb, tw)
    assert O.simulate(pr, 1, W.SEQ, W.GREEDY, seq_cuts(p))["makespan"] == \
        (m + p - 1) * (tf + tb) + m * tw


# ---------------------------------------------------------------- memory (R16, Eq. 2)
@pytest.mark.parametrize("p", [2, 4])
@pytest.mark.parametrize("m", [2, 4, 8])
def test_peak_memory_closed_forms_v1(p, m):
    pr = homo(p, p, m, 1, 1, 1, act=3, stash=2)  # one unit = 5 bytes per stage per mb
    g = O.simulate(pr, 1, W.SEQ, W.GPIPE, seq_cuts(p))
    assert g["M_d"] == [5 * m] * p
    o = O.simulate(pr, 1, W.SEQ, W.ONEF1B, seq_cuts(p))
    assert o["M_d"] == [5 * min(p - d, m) for d in range(p)]


@pytest.mark.parametrize("p,v", [(2, 2), (4, 2), (4, 3), (2, 4)])
def test_peak_memory_closed_forms_interleaved(p, v):
    m = 2 * p
    pr = homo(p * v, p, m, 1, 1, 1, act=1)
    o = O.simulate(pr, v, W.INTERLEAVED, W.ONEF1B, seq_cuts(p * v))
    assert o["M_d"] == [min(m * v, 2 * (p - d - 1) + (v - 1) * p + 1) for d in range(p)]
    g = O.simulate(pr, v, W.INTERLEAVED, W.GPIPE, seq_cuts(p * v))
    assert g["M_d"] == [m * v] * p


def test_gpipe_memory_cap_example():
    """GPipe with nmb=4 holds 4 units; capacity 3 units is violated, 4 is not."""
    ex = SPEC["gpipe_mem"]
    u = 7
    pr = homo(2, 2, ex["m"], 1, 1, 1, act=u, weight=100, cap=100 + ex["cap_units"] * u)
    r = O.simulate(pr, 1, W.SEQ, W.GPIPE, [1])
    assert r["status"] == 2 and r["makespan"] == O.INT64_MAX
    assert r["peak_mem"] == 100 + 4 * u  # static (weight of one row) + 4 units
    pr.cap = 100 + 4 * u
    assert O.simulate(pr, 1, W.SEQ, W.GPIPE, [1])["status"] == 0


def test_greedy_and_zb_respect_or_report_cap():
    rng = W.SplitMix64(99)
    for _ in range(60):
        p = 2 + rng.next() % 3
        m = p * (1 + rng.next() % 2)
        pr = W.random_problem(rng, 2 * p + 1, p, m, bytes_max=9, cap=60 + rng.next() % 80)
        cuts = sorted(set(range(1, 2 * p + 1)) - {int(1 + rng.next() % (2 * p))})
        cuts = cuts[:2 * p - 1]
        for pol in (W.ZB, W.GREEDY):
            r = O.simulate(pr, 2, W.INTERLEAVED, pol, cuts)
            if r["status"] == 0:
                assert max(r["M_d"]) <= pr.cap
            if pol == W.GREEDY and r["status"] != 3:
                assert max(r["M_d"]) <= pr.cap


# ---------------------------------------------------------------- seed (R20)
@pytest.mark.parametrize("key", ["balanced_1", "balanced_2"])
def test_seed_spec_examples(key):
    ex = SPEC[key]
    val, cuts = O.seed_minmax(ex["w"], ex["S"])
    assert (val, cuts) == (ex["max"], ex["cuts"])


def test_seed_brute_force():
    rng = W.SplitMix64(3)
    for _ in range(150):
        L = 2 + rng.next() % 11
        S = 1 + rng.next() % min(4, L)
        w = [1 + rng.next() % 9 for _ in range(L)]
        best = None
        for cuts in itertools.combinations(range(1, L), S - 1):
            b = [0, *cuts, L]
            val = max(sum(w[b[i]:b[i + 1]]) for i in range(S))
            if best is None or (val, cuts) < best:
                best = (val, cuts)
        assert O.seed_minmax(w, S) == (best[0], list(best[1]))


# ---------------------------------------------------------------- space (R19)
def test_full_count_and_colex_order():
    pr = homo(9, 2, 2, 1, 1, 1)
    sp = W.Space([W.Group(2, W.FULL, combo_mask=0x1)])  # S = 4 -> C(8, 3)
    out = O.enumerate_space(pr, sp)
    assert len(out) == math.comb(8, 3) == O.space_size(pr, sp)
    inner = [tuple(pl["cuts"][1:-1]) for _, pl in out]
    assert inner == sorted(itertools.combinations(range(1, 9), 3), key=lambda t: t[::-1])
    assert [i for i, _ in out] == list(range(len(out)))


def _ball_key(delta):
    return tuple(2 * abs(x) - (1 if x < 0 else 0) for x in delta)  # 0,-1,+1,-2,+2 -> 0,1,2,3,4


@pytest.mark.parametrize("n,R", [(1, 3), (3, 2), (4, 3), (2, 5)])
def test_ball_count_bijection_and_order(n, R):
    L = 40
    seed = [5 * (i + 1) for i in range(n)]
    p = n + 1
    pr = homo(L, p, 2, 1, 1, 1)
    sp = W.Space([W.Group(1, W.BALL, R, seed_cuts=seed, combo_mask=0x1)])
    out = O.enumerate_space(pr, sp)
    closed = sum(2 ** k * math.comb(n, k) * math.comb(R, k) for k in range(0, min(n, R) + 1))
    assert len(out) == closed == O.space_size(pr, sp)
    deltas = [tuple(c - s for c, s in zip(pl["cuts"][1:-1], seed)) for _, pl in out]
    brute = [d for d in itertools.product(range(-R, R + 1), repeat=n) if sum(map(abs, d)) <= R]
    assert sorted(deltas) == sorted(brute)
    assert deltas == sorted(deltas, key=_ball_key)


def test_decode_matches_enumeration():
    pr = W.random_problem(W.SplitMix64(5), 10, 2, 4)
    sp = W.Space([W.Group(1, W.FULL, combo_mask=0xF), W.Group(2, W.BALL, 3, combo_mask=0x35),
                  W.Group(4, W.FULL, combo_mask=0x3F)])
    out = O.enumerate_space(pr, sp)
    assert len(out) == O.space_size(pr, sp)
    for idx, pl in out:
        assert O.decode(pr, sp, idx) == pl


def test_config_space_sizes():
    """|space| of the five configs; closed forms computed here."""
    def ball(n, R):
        return sum(2 ** k * math.comb(n, k) * math.comb(R, k) for k in range(min(n, R) + 1))
    exp = {1: 7 * 4 + 35 * 6 + 1 * 6, 2: math.comb(33, 7),
           3: 4 * ball(7, 16) + 6 * ball(15, 8), 4: 6 * ball(15, 8),
           5: 4 * ball(15, 9) + 6 * ball(31, 6) + 6 * ball(63, 4)}
    for cid in range(1, 6):
        pr, sp = W.config(cid)
        assert O.space_size(pr, sp) == exp[cid]
    assert exp[2] == 4_272_048 and 9.4e8 < exp[5] < 9.6e8


# ---------------------------------------------------------------- cfg1 anchors
def test_cfg1_unit_advisory_golden():
    g = CFG1
    pr = W.cfg1_unit()
    sp = W.Space([W.Group(1, W.FULL, combo_mask=0xF), W.Group(2, W.FULL), W.Group(4, W.FULL)])
    assert O.space_size(pr, sp) == g["full"]["N"]
    b = O.search(pr, sp, prune=False)
    assert (b["index"], b["makespan"]) == (g["full"]["argmin_index"], g["full"]["makespan"])
    assert b["plan"]["cuts"] == g["full"]["plan"]["cuts"]
    ev = O.eval_indices(pr, sp, range(g["full"]["N"]))
    assert int(ev["makespan"].max()) == g["full"]["worst_makespan"] == int(ev["makespan"][0])
    for name, pol in (("GPIPE", 0), ("ONEF1B", 1), ("ZB", 2), ("GREEDY", 3)):
        assert O.simulate(pr, 1, W.SEQ, pol, [4])["makespan"] == g["uniform_v1_cut4"][name]
    lit = W.Space([W.Group(1, W.FULL, combo_mask=0x7), W.Group(2, W.FULL, combo_mask=0x17),
                   W.Group(4, W.FULL, combo_mask=0x17)])
    assert O.space_size(pr, lit) == g["literal_three_policy"]["N"]
    bl = O.search(pr, lit, prune=False)
    assert (bl["index"], bl["makespan"]) == (g["literal_three_policy"]["argmin_index"],
                                             g["literal_three_policy"]["makespan"])
    evl = O.eval_indices(pr, lit, range(165))
    ties = [i for i in range(165) if evl["makespan"][i] == 218]
    assert ties == g["literal_three_policy"]["tied_indices"]
    # per-combo optima: the only cross-implementation anchors on WAVE placement
    # and on the v = 4 ZB / GREEDY combos (SURVEY §8(c) cfg1 golden values)
    names = {(W.SEQ, 0): "GPIPE", (W.SEQ, 1): "ONEF1B", (W.SEQ, 2): "ZB", (W.SEQ, 3): "GREEDY"}
    for plc, pn in ((W.INTERLEAVED, "INT"), (W.WAVE, "WAVE")):
        for pol, qn in ((0, "GPIPE"), (1, "ONEF1B"), (2, "ZB"), (3, "GREEDY")):
            names[(plc, pol)] = pn + "_" + qn
    seen = 0
    for v in (1, 2, 4):
        for k in range(6):
            c = O.combo(v, k)
            if c is None:
                continue
            one = W.Space([W.Group(v, W.FULL, combo_mask=1 << k)])
            bc = O.search(pr, one, prune=False)
            assert bc["makespan"] == g["per_combo_best"]["v%d" % v][names[c]], (v, c)
            seen += 1
    assert seen == 16


# ---------------------------------------------------------------- fp64 reference of the fp32 variant
def test_f64_event_loop_equals_int64_on_integer_costs():
    """The fp64 simulator on integer-valued costs reproduces the exact int64 one."""
    rng = W.SplitMix64(555)
    for _ in range(120):
        p = 1 + rng.next() % 4
        m = p * (1 + rng.next() % 2)
        L = 2 * p + 1 + rng.next() % 3
        pr = W.random_problem(rng, L, p, m, bytes_max=6, cap=W.INT64_MAX if rng.next() % 2 else 80)
        prf = W.Problem(**{c: getattr(pr, c) for c in W.COLUMNS}, p=p, m=m, cap=pr.cap, cost_type=1,
                        costs_f32=np.stack([pr.t_f, pr.t_b, pr.t_w, pr.comm]).astype(np.float32))
        cuts = sorted(set(range(1, L)) - {int(1 + rng.next() % (L - 1))})[: 2 * p - 1]
        v, placement = (2, W.INTERLEAVED) if len(cuts) == 2 * p - 1 else (1, W.SEQ)
        if v == 1:
            cuts = list(range(1, p))
        for pol in range(4):
            a = O.simulate(pr, v, placement, pol, cuts)
            b = O.simulate(prf, v, placement, pol, cuts)
            assert (a["status"], a["makespan"], a["peak_mem"]) == (b["status"], b["makespan"], b["peak_mem"])
            if a["status"] == 0:
                assert b["makespan_f"] == float(a["makespan"])


def test_f32_event_loop_equals_int64_on_integer_costs():
    """R27: the fp32-time event loop on integer costs (exact in fp32 below 2^24)
    reproduces the exact int64 one, decisions included, for every policy."""
    rng = W.SplitMix64(556)
    for _ in range(120):
        p = 1 + rng.next() % 4
        m = p * (1 + rng.next() % 2)
        L = 2 * p + 1 + rng.next() % 3
        pr = W.random_problem(rng, L, p, m, bytes_max=6, cap=W.INT64_MAX if rng.next() % 2 else 80)
        prf = W.Problem(**{c: getattr(pr, c) for c in W.COLUMNS}, p=p, m=m, cap=pr.cap, cost_type=1,
                        costs_f32=np.stack([pr.t_f, pr.t_b, pr.t_w, pr.comm]).astype(np.float32))
        v, placement = (2, W.INTERLEAVED) if L >= 2 * p else (1, W.SEQ)
        cuts = list(range(1, p * v))
        for pol in range(4):
            a = O.simulate(pr, v, placement, pol, cuts)
            b = O.simulate(prf, v, placement, pol, cuts, precision="f32")
            assert (a["status"], a["makespan"], a["peak_mem"]) == (b["status"], b["makespan"], b["peak_mem"])
            if a["status"] == 0:
                assert b["makespan_f"] == float(a["makespan"])


@pytest.mark.parametrize("policy", [W.GPIPE, W.ONEF1B, W.ZB, W.GREEDY])
def test_f32_serial_device_rounds_every_addition(policy):
    """R27 fp32 arithmetic on one device (p = 1, no latency): the makespan is
    the fp32 running sum of the task durations in execution order, each stage
    duration the fp32 rounding of its exact row sum (fused B: of t_B + t_W).
    On one device every task is ready when the device is free, so the order is
    the policy's priority order alone; it is taken from the int64 oracle's trace
    (pinned by the closed forms above) and the sum is done here with numpy
    float32 additions. Costs near 1e7 make fp32 rounding differ from fp64."""
    m = 5
    t = np.array([[1e7 + 0.375, 3.25], [2e7 + 0.125, 1.5], [1.0e7 + 0.625, 0.75], [0, 0]], np.float64)
    t32 = t.astype(np.float32).astype(np.float64)
    z = [0, 0]
    pri = W.Problem(t_f=[3, 1], t_b=[3, 1], t_w=[3, 1], act=z, stash=z, weight=z, grad=z, comm=z, p=1, m=m)
    prf = W.Problem(t_f=[3, 1], t_b=[3, 1], t_w=[3, 1], act=z, stash=z, weight=z, grad=z, comm=z,
                    p=1, m=m, cost_type=1, costs_f32=t.astype(np.float32))
    fused = policy in (W.GPIPE, W.ONEF1B)
    dur = {0: np.float32(t32[0].sum()),
           1: np.float32(t32[1].sum() + (t32[2].sum() if fused else 0.0)),
           2: np.float32(t32[2].sum())}
    order = O.simulate(pri, 1, W.SEQ, policy, [], trace=True)["trace"][0]
    assert len(order) == m * (2 if fused else 3)
    acc = np.float32(0)
    for (k, _s, _j, _st) in order:
        acc = np.float32(acc + dur[k])
    r = O.simulate(prf, 1, W.SEQ, policy, [], precision="f32")
    assert r["status"] == 0 and r["makespan_f"] == float(acc)
    exact = O.simulate(prf, 1, W.SEQ, policy, [])["makespan_f"]
    assert r["makespan_f"] != exact  # fp32 rounding is visible here
    assert abs(r["makespan_f"] - exact) <= 1e-5 * exact


@pytest.mark.parametrize("p,m", [(2, 4), (4, 8)])
def test_f64_closed_forms_with_fractional_costs(p, m):
    """GPipe and S-1F1B closed forms hold for real costs (dyadic, exact in fp64)."""
    tf, tb, tw = 1.25, 2.5, 1.125
    pr = homo(p, p, m, 1, 1, 1)
    prf = W.Problem(**{c: getattr(pr, c) for c in W.COLUMNS}, p=p, m=m, cost_type=1,
                    costs_f32=np.array([[tf] * p, [tb] * p, [tw] * p, [0.0] * p], np.float32))
    g = O.simulate(prf, 1, W.SEQ, W.GPIPE, seq_cuts(p))
    o = O.simulate(prf, 1, W.SEQ, W.ONEF1B, seq_cuts(p))
    assert g["makespan_f"] == (m + p - 1) * (tf + tb + tw) == o["makespan_f"]


# ----------------------------------------------------------------- R29 comm accounting
def _acct_problem(L, p, m, tf, tb, tw, comm):
    z = [0] * L
    return W.Problem(t_f=tf, t_b=tb, t_w=tw, act=z, stash=z, weight=z, grad=z, comm=comm, p=p, m=m)


def test_comm_accounting_hand_example():
    """GPipe, p = 2, m = 1, t_F = 1, fused B = t_B + t_W = 2, latency 3 (worked by hand):
    d0 computes [0,1] and [10,12], its transfers are [1,4] and [7,10] -> exposed 6,
    bubble 3 (idle [4,7]); d1 computes [4,7], transfers [1,4] and [7,10] (the latter
    after T_1 = 7) -> exposed 3, overlap 3, bubble 1."""
    pr = _acct_problem(2, 2, 1, [1, 1], [1, 1], [1, 1], [3, 0])
    r = O.comm_accounting(pr, 1, 0, 0, [1])
    assert r["T_d"] == [12, 7] and r["busy_d"] == [3, 3]
    assert r["comm_d"] == [6, 6] and r["exposed_d"] == [6, 3]
    assert r["overlap_d"] == [0, 3] and r["bubble_d"] == [3, 1]


@pytest.mark.parametrize("policy", [0, 1, 2, 3])
def test_comm_accounting_spec_device_comm_total(policy):
    """S:198 example: S = 2, P = 2, nmb = 3, one boundary of 10 ticks -> each
    device sends 3 and receives 3 transfers: comm total 2 x 3 x 10 = 60."""
    pr = _acct_problem(2, 2, 3, [5, 5], [5, 5], [2, 2], [10, 0])
    r = O.comm_accounting(pr, 1, 0, policy, [1])
    assert r["comm_d"] == [60, 60]


@pytest.mark.parametrize("p,m", [(2, 2), (3, 4), (4, 4), (4, 7)])
def test_comm_accounting_zero_comm_1f1b(p, m):
    """Zero comm: no exposed or overlapped transfer time, and device 0 of a
    homogeneous S-1F1B pipeline idles (p-1)(t_F+t_B) (S:210 closed form)."""
    f, b, w = 3, 4, 2
    pr = _acct_problem(p, p, m, [f] * p, [b] * p, [w] * p, [0] * p)
    r = O.comm_accounting(pr, 1, 0, 1, list(range(1, p)))
    assert r["comm_d"] == [0] * p and r["exposed_d"] == [0] * p
    assert r["bubble_d"][0] == (p - 1) * (f + b + w)  # fused B runs t_B + t_W (R2)


def test_comm_accounting_identity_and_bounds():
    """Alg. 1 Step 3 identity T_d = (busy_d + comm_d) + bubble_d - overlap_d, and
    0 <= exposed_d <= min(comm_d, T_d - busy_d), on random plans of every policy."""
    rng = W.SplitMix64(29)
    n = 0
    for t in range(60):
        p = [2, 3, 4][t % 3]
        L = 2 * p + 2
        pr = W.random_problem(rng, L, p, 2 * p, tmax=7, cmax=6, bytes_max=0)
        v = 1 + (t % 2)
        S = p * v
        cuts = sorted(random.Random(t).sample(range(1, L), S - 1))
        for pl, po in ([(0, k) for k in range(4)] if v == 1 else [(1, k) for k in range(4)] + [(2, 0), (2, 3)]):
            r = O.comm_accounting(pr, v, pl, po, cuts)
            if r["status"] != 0:
                continue
            n += 1
            for d in range(p):
                assert r["T_d"][d] == r["busy_d"][d] + r["comm_d"][d] + r["bubble_d"][d] - r["overlap_d"][d]
                assert 0 <= r["exposed_d"][d] <= min(r["comm_d"][d], r["T_d"][d] - r["busy_d"][d])
    assert n > 200


# ----------------------------------------------------------------- R30 explicit orders
def _realised_lists(r, fused):
    """The event loop's realised per-device order as (kind, stage, mb) lists."""
    return [[(k, s, j) for (k, s, j, _st) in lst if not (fused and k == 2)] for lst in r["trace"]]


def test_simulate_lists_reproduces_event_loop():
    """Feeding the event loop's own realised order back as an explicit schedule
    reproduces its status, makespan, T_d, busy_d and M_d, for every policy and
    placement (fused for GPIPE / 1F1B, split for ZB / GREEDY), with binding caps."""
    rng = W.SplitMix64(30)
    n = 0
    for t in range(80):
        p = [1, 2, 3, 4][t % 4]
        L = 2 * p + 3
        cap = W.INT64_MAX if t % 3 else 40 + (t * 7) % 60
        pr = W.random_problem(rng, L, p, 2 * p, tmax=7, cmax=4, bytes_max=5, cap=cap)
        v = 1 + (t % 2)
        S = p * v
        cuts = sorted(random.Random(t).sample(range(1, L), S - 1))
        combos = [(0, k) for k in range(4)] if v == 1 else [(1, k) for k in range(4)] + [(2, 0), (2, 3)]
        for pl, po in combos:
            r = O.simulate(pr, v, pl, po, cuts, trace=True)
            if r["status"] == 3:
                continue
            fused = po in (0, 1)
            q = O.simulate_lists(pr, v, pl, fused, cuts, _realised_lists(r, fused))
            assert q["status"] == r["status"], (t, pl, po)
            assert q["busy_d"] == r["busy_d"] and q["M_d"] == r["M_d"]
            if r["status"] == 0:
                assert q["makespan"] == r["makespan"] and q["T_d"] == r["T_d"]
            n += 1
    assert n > 300


def test_simulate_lists_cyclic_wait_is_stuck():
    """The S-1F1B lists evaluate like the policy; two devices whose orders cross
    (d0 runs B(0,0) before sending F(0,1), d1 runs F(1,1) before sending
    B(1,0)) wait on each other: status 3."""
    z = [0, 0]
    pr = W.Problem(t_f=[1, 1], t_b=[1, 1], t_w=[1, 1], act=z, stash=z, weight=z, grad=z,
                   comm=[1, 0], p=2, m=2)
    s1f1b = [[(0, 0, 0), (0, 0, 1), (1, 0, 0), (1, 0, 1)],   # d0: warm-up 1, then F B F B
             [(0, 1, 0), (1, 1, 0), (0, 1, 1), (1, 1, 1)]]   # d1: F B F B (S:288 lists)
    r = O.simulate_lists(pr, 1, 0, True, [1], s1f1b)
    assert r["status"] == 0 and r["makespan"] == O.simulate(pr, 1, 0, 1, [1])["makespan"]
    crossed = [[(0, 0, 0), (1, 0, 0), (0, 0, 1), (1, 0, 1)],  # d0 waits for B(1,0) before F(0,1)
               [(0, 1, 0), (0, 1, 1), (1, 1, 0), (1, 1, 1)]]  # d1 waits for F(0,1) before B(1,0)
    assert O.simulate_lists(pr, 1, 0, True, [1], crossed)["status"] == 3


# ----------------------------------------------------------------- R31 OOM repair
def _one_device(cap, weight=0):
    return W.Problem(t_f=[2], t_b=[2], t_w=[1], act=[10], stash=[0], weight=[weight], grad=[0],
                     comm=[0], p=1, m=4, cap=cap)


def test_repair_oom_worked_example():
    """One device, GPipe order F0 F1 F2 F3 B0 B1 B2 B3, 10 B per activation, cap 25
    (two in flight). By hand: F2 overflows (30); the latest B whose F precedes it
    is B1 -> F0 F1 B1 F2 F3 B0 B2 B3; now F3 overflows; the latest eligible B is
    B2 -> F0 F1 B1 F2 B2 F3 B0 B3, which fits. Two moves, makespan unchanged (20)."""
    pr = _one_device(25)
    gp = [[(0, 0, j) for j in range(4)] + [(1, 0, j) for j in range(4)]]
    lists, moves, r = O.repair_oom(pr, 1, 0, True, [], gp)
    assert moves == 2 and r["status"] == 0 and r["makespan"] == 20
    assert lists == [[(0, 0, 0), (0, 0, 1), (1, 0, 1), (0, 0, 2), (1, 0, 2), (0, 0, 3), (1, 0, 0), (1, 0, 3)]]
    assert max(r["M_d"]) <= 25


def test_repair_oom_identity_and_unrepairable():
    gp = [[(0, 0, j) for j in range(4)] + [(1, 0, j) for j in range(4)]]
    lists, moves, r = O.repair_oom(_one_device(40), 1, 0, True, [], gp)   # fits: identity
    assert moves == 0 and r["status"] == 0 and lists == gp
    lists, moves, r = O.repair_oom(_one_device(5, weight=6), 1, 0, True, [], gp)  # static > cap
    assert moves == 0 and r["status"] == 2 and lists == gp


def test_repair_oom_split_moves_w_with_b():
    """Split B/W: the advanced B takes its W right behind it; stash frees at W."""
    pr = W.Problem(t_f=[2], t_b=[2], t_w=[1], act=[6], stash=[4], weight=[0], grad=[0],
                   comm=[0], p=1, m=3, cap=25)
    order = [[(0, 0, 0), (0, 0, 1), (0, 0, 2), (1, 0, 0), (2, 0, 0), (1, 0, 1), (2, 0, 1),
              (1, 0, 2), (2, 0, 2)]]
    lists, moves, r = O.repair_oom(pr, 1, 0, False, [], order)
    assert r["status"] == 0 and moves == 1
    assert lists == [[(0, 0, 0), (0, 0, 1), (1, 0, 1), (2, 0, 1), (0, 0, 2), (1, 0, 0), (2, 0, 0),
                      (1, 0, 2), (2, 0, 2)]]


# ----------------------------------------------------------------- R32 overlap-aware reordering
def _r32_cases():
    rng = W.SplitMix64(32)
    for t in range(12):
        p = [2, 3, 4][t % 3]
        L = 2 * p + 3
        pr = W.random_problem(rng, L, p, 2 * p, tmax=6, cmax=8, bytes_max=0)
        cuts = sorted(random.Random(t).sample(range(1, L), p - 1))
        for po in (1, 2):
            r = O.simulate(pr, 1, 0, po, cuts, trace=True)
            fused = po == 1
            yield pr, cuts, po, fused, [[(k, s, j) for (k, s, j, _t) in lst if not (fused and k == 2)]
                                        for lst in r["trace"]]


def test_list_accounting_equals_policy_accounting():
    """R29 on explicit lists (longest-path schedule) equals R29 on the event loop
    when the lists are the event loop's own realised order."""
    for pr, cuts, po, fused, lists in _r32_cases():
        a = O.comm_accounting_lists(pr, 1, 0, fused, cuts, lists)
        b = O.comm_accounting(pr, 1, 0, po, cuts)
        for k in ("comm_d", "exposed_d", "overlap_d", "bubble_d", "T_d"):
            assert a[k] == b[k], k


def test_tune_overlap_invariants():
    """Every accepted move keeps the makespan and raises the total OverlapTime; the
    result re-simulates; zero latency gives nothing to overlap, hence no move."""
    moved = 0
    for pr, cuts, po, fused, lists in _r32_cases():
        a0 = O.comm_accounting_lists(pr, 1, 0, fused, cuts, lists)
        nl, swaps, acc = O.tune_overlap(pr, 1, 0, fused, cuts, lists)
        assert acc["status"] == 0 and acc["makespan"] <= a0["makespan"]
        assert (swaps == 0) == (sum(acc["overlap_d"]) == sum(a0["overlap_d"]))
        assert sum(acc["overlap_d"]) >= sum(a0["overlap_d"]) + swaps
        re = O.comm_accounting_lists(pr, 1, 0, fused, cuts, nl)
        assert re["makespan"] == acc["makespan"] and re["overlap_d"] == acc["overlap_d"]
        moved += swaps
        pr0 = W.Problem(t_f=pr.t_f, t_b=pr.t_b, t_w=pr.t_w, act=pr.act, stash=pr.stash, weight=pr.weight,
                        grad=pr.grad, comm=[0] * len(pr.t_f), p=pr.p, m=pr.m)
        assert O.tune_overlap(pr0, 1, 0, fused, cuts, lists)[1] == 0
    assert moved > 20


def test_tune_overlap_spec_two_device_example():
    """SPEC S:374 (tune_overlap examples, R32): a two-device instance with
    comm_time = t_F where a consumer waits right after its producer's transfer.
    Worked by hand (unit costs, one layer per stage, latency 1, split B/W):
      dev0 [F00 F01 B00 B01 W00 W01]: F00 [0,1] F01 [1,2] B00 [5,6] (waits for
        B10's arrival 4+1) B01 [7,8] (waits for B11's arrival 6+1) W00 [8,9] W01 [9,10]
      dev1 [F10 B10 F11 B11 W10 W11]: [2,3] [3,4] [4,5] [5,6] [6,7] [7,8]
    makespan 10; exposed (union of incident transfers outside compute, R29)
    dev0 [2,3] [4,5] [6,7] = 3 of comm 4, dev1 [1,2] = 1 of comm 4: overlap 1 + 3.
    The R32 neighbours are: B01 before B00 (makespan 11), F11 before F10 (11),
    and W00 before the waiting B01 (W00 [6,7] hides B11's transfer, makespan 9),
    so exactly one swap is accepted and the overlap rises by comm_time = 1; in
    the new schedule the remaining neighbours are both 11 (no further swap).
    The fully dependent chain (m = 1) has no neighbour at all: no-op."""
    z = [0, 0]
    pr = W.Problem(t_f=[1, 1], t_b=[1, 1], t_w=[1, 1], act=z, stash=z, weight=z, grad=z,
                   comm=[1, 0], p=2, m=2)
    F, B, Wk = 0, 1, 2
    lists = [[(F, 0, 0), (F, 0, 1), (B, 0, 0), (B, 0, 1), (Wk, 0, 0), (Wk, 0, 1)],
             [(F, 1, 0), (B, 1, 0), (F, 1, 1), (B, 1, 1), (Wk, 1, 0), (Wk, 1, 1)]]
    a0 = O.comm_accounting_lists(pr, 1, W.SEQ, False, [1], lists)
    assert a0["makespan"] == 10 and a0["T_d"] == [10, 8]
    assert a0["comm_d"] == [4, 4] and a0["exposed_d"] == [3, 1] and a0["overlap_d"] == [1, 3]
    nl, swaps, acc = O.tune_overlap(pr, 1, W.SEQ, False, [1], lists)
    assert swaps == 1
    assert [list(map(tuple, x)) for x in nl] == [
        [(F, 0, 0), (F, 0, 1), (B, 0, 0), (Wk, 0, 0), (B, 0, 1), (Wk, 0, 1)], lists[1]]
    assert acc["makespan"] == 9 and acc["T_d"] == [9, 8]
    assert acc["exposed_d"] == [2, 1] and acc["overlap_d"] == [2, 3]
    assert sum(acc["overlap_d"]) == sum(a0["overlap_d"]) + 1  # + comm_time
    pr1 = W.Problem(t_f=[1, 1], t_b=[1, 1], t_w=[1, 1], act=z, stash=z, weight=z, grad=z,
                    comm=[1, 0], p=2, m=1)
    chain = [[(F, 0, 0), (B, 0, 0), (Wk, 0, 0)], [(F, 1, 0), (B, 1, 0), (Wk, 1, 0)]]
    assert O.overlap_candidates(pr1, 1, W.SEQ, False, [1], chain) == []
    assert O.tune_overlap(pr1, 1, W.SEQ, False, [1], chain)[1] == 0


# ----------------------------------------------------------------- R35 memory timeline
def test_memory_timeline_spec_examples():
    """GPipe with nmb = 4 and 1 unit of activation per stage and
    micro-batch, capacity 3 units above static: the violation is at the start
    of the 4th F (worked by hand: one device, t_F = 2, F starts at 0, 2, 4, 6);
    capacity infinite: no violation; fused B frees act + stash at its end."""
    u = 1 << 20
    pr = W.Problem(t_f=[2], t_b=[3], t_w=[1], act=[u], stash=[0], weight=[5 * u], grad=[0], comm=[0],
                   p=1, m=4, cap=5 * u + 3 * u)
    r = O.memory_timeline(pr, 1, W.SEQ, W.GPIPE, [])
    pts = r["points"][0]
    assert pts[:5] == [(0, 5 * u), (0, 6 * u), (2, 7 * u), (4, 8 * u), (6, 9 * u)]
    assert r["first_violation"] == [6]
    # GPipe then runs the 4 fused backwards (t_B + t_W = 4 each) from t = 8
    assert pts[5:] == [(12, 8 * u), (16, 7 * u), (20, 6 * u), (24, 5 * u)]
    pr.cap = W.INT64_MAX
    assert O.memory_timeline(pr, 1, W.SEQ, W.GPIPE, [])["first_violation"] == [-1]
    # split (ZB): B frees act at its end, W frees stash at its end
    pr2 = W.Problem(t_f=[2], t_b=[3], t_w=[1], act=[2], stash=[1], weight=[0], grad=[0], comm=[0], p=1, m=1)
    assert O.memory_timeline(pr2, 1, W.SEQ, W.ZB, [])["points"][0] == [(0, 0), (0, 3), (5, 1), (6, 0)]


def test_memory_timeline_peak_equals_simulated_peak():
    """The timeline's maximum is the event loop's per-device M_d, every policy,
    placement and binding caps; breakpoint times never decrease; memory returns
    to the static bytes; the first violation is the first breakpoint above the
    cap."""
    rng = W.SplitMix64(707)
    n = 0
    for _ in range(60):
        p = 1 + rng.next() % 4
        m = p * (1 + rng.next() % 2)
        L = 2 * p + 1 + rng.next() % 3
        pr = W.random_problem(rng, L, p, m, bytes_max=6, cap=W.INT64_MAX if rng.next() % 2 else 30)
        v, placement = (2, W.INTERLEAVED) if L >= 2 * p else (1, W.SEQ)
        cuts = list(range(1, p * v))
        for pol in range(4):
            sim = O.simulate(pr, v, placement, pol, cuts)
            if sim["status"] not in (0, 2):
                continue
            r = O.memory_timeline(pr, v, placement, pol, cuts)
            for d in range(p):
                pts = r["points"][d]
                assert max(b for _, b in pts) == sim["M_d"][d]
                assert all(a[0] <= b[0] for a, b in zip(pts, pts[1:]))
                assert pts[-1][1] == pts[0][1] == sim["static_d"][d]
                over = [t for t, b in pts if b > pr.cap]
                assert r["first_violation"][d] == (over[0] if over else -1)
            n += 1
    assert n > 100
