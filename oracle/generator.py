"""oracle/generator.py — TEST INFRASTRUCTURE ONLY.

The Pipeline Generator of AdaPtis (arXiv 2509.23722 §4.3) written
out step by step as reading R28 of DESIGN.md fixes it, on top of the oracle's
event-loop simulator (`oracle.simulate`) and exhaustive search
(`oracle.search`). Only tests/ and bench.py's CPU legs may use it; it shares
no code with paper_2509_23722_b200/.

R28, in the paper's order:
  * Seeds ("For model partition, we adopt the policies from S-1F1B and
    Mist. For model placement, the baselines include S-1F1B, I-1F1B, and
    Hanayo. For workload scheduling, we consider S-1F1B and ZB"): for each
    admitted v (ascending), partitions [equal layers, Mist min-max (R20)] x
    combos v = 1: [(SEQ, 1F1B), (SEQ, ZB)]; v >= 2: [(INT, 1F1B), (INT, ZB),
    (WAVE, GREEDY)]. The baseline is the first seed of smallest makespan.
  * Rounds ("identifies the bottleneck phase ... tunes it ... If a
    tuning step degrades pipeline performance, it is rolled back ... repeats
    until no further improvement"): partition, then placement, then schedule;
    each phase proposes its best neighbour and is accepted only if it lowers
    the makespan strictly. A round without an accepted step ends the loop.
      - partition (layer transfers between stages): the best plan of
        the L1 ball of radius R around the current cuts, same combo, ties to
        the lowest canonical index (R19);
      - placement (grouped permutations of stage-device assignment):
        for each admitted v ascending, each placement (SEQ for v = 1; INT,
        WAVE for v >= 2) other than the current one; cuts kept when v is
        unchanged, else the Mist seed; policy kept when R12 admits it, else
        GREEDY; the first of smallest makespan;
      - schedule: every other policy R12 admits for the
        placement (GPIPE, 1F1B, ZB, GREEDY order); the first of smallest makespan.
Parity: pinned by tests/test_generator.py (monotone trajectory, local
optimality by brute force, global optimum when the ball covers the space).
"""
from paper_2509_23722_b200 import workloads as W

from . import oracle as O

SEQ, INT, WAVE = 0, 1, 2
GPIPE, ONEF1B, ZB, GREEDY = 0, 1, 2, 3
ADMITTED = {1: {SEQ: (GPIPE, ONEF1B, ZB, GREEDY)},
            2: {INT: (GPIPE, ONEF1B, ZB, GREEDY), WAVE: (GPIPE, GREEDY)}}


def admitted(v, placement, policy):
    """R12 combo table."""
    table = ADMITTED[1] if v == 1 else ADMITTED[2]
    return policy in table.get(placement, ())


def combo_index(v, placement, policy):
    for k in range(6):
        c = O.combo(v, k)
        if c == (placement, policy):
            return k
    raise ValueError((v, placement, policy))


def equal_layers(L, S):
    """S-1F1B partition: equal layer counts, cut i at floor(i L / S)."""
    return [i * L // S for i in range(1, S)]


def mist(pr, S):
    """Mist-style min-max partition of per-row t_F + t_B + t_W (R20)."""
    w = [pr.t_f[i] + pr.t_b[i] + pr.t_w[i] for i in range(len(pr.t_f))]
    return O.seed_minmax(w, S)[1]


def score(pr, v, placement, policy, cuts):
    r = O.simulate(pr, v, placement, policy, cuts)
    return r["makespan"] if r["status"] == 0 else None


def first_best(pr, plans):
    """(index, makespan) of the first plan with the smallest feasible makespan."""
    bi, bm = -1, None
    for i, (v, pl, po, cuts) in enumerate(plans):
        s = score(pr, v, pl, po, cuts)
        if s is not None and (bm is None or s < bm):
            bi, bm = i, s
    return bi, bm


def generate(pr, vs_mask=0x3, radius=2, max_rounds=32):
    L, p, m = len(pr.t_f), pr.p, pr.m
    vs = [v for v in range(1, 5) if (vs_mask >> (v - 1)) & 1 and p * v <= min(64, L)
          and (v == 1 or m % p == 0)]
    seeds = []
    for v in vs:
        S = p * v
        for part in (equal_layers(L, S), mist(pr, S)):
            combos = [(SEQ, ONEF1B), (SEQ, ZB)] if v == 1 else [(INT, ONEF1B), (INT, ZB), (WAVE, GREEDY)]
            for pl, po in combos:
                seeds.append((v, pl, po, list(part)))
    n_eval = len(seeds)
    bi, cur_mk = first_best(pr, seeds)
    if bi < 0:
        return {"status": "infeasible", "n_seeds": len(seeds), "steps": []}
    cur = seeds[bi]
    steps = [("seed", cur_mk)]
    rounds = 0
    while rounds < max_rounds:
        rounds += 1
        improved = False
        # partition phase: the L1 ball of radius R around the current cuts
        v, pl, po, cuts = cur
        sp = W.Space([W.Group(v, W.BALL, radius, seed_cuts=list(cuts),
                              combo_mask=1 << combo_index(v, pl, po))])
        n_eval += O.space_size(pr, sp)
        b = O.search(pr, sp, prune=True)
        if b["index"] != (1 << 64) - 1 and b["makespan"] < cur_mk:
            bc = b["plan"]["cuts"]
            cur = (v, pl, po, bc[1:-1])
            cur_mk = b["makespan"]
            steps.append(("partition", cur_mk))
            improved = True
        # placement phase
        v, pl, po, cuts = cur
        cand = []
        for v2 in vs:
            for pl2 in ([SEQ] if v2 == 1 else [INT, WAVE]):
                if (v2, pl2) == (v, pl):
                    continue
                po2 = po if admitted(v2, pl2, po) else GREEDY
                cuts2 = list(cuts) if v2 == v else mist(pr, p * v2)
                cand.append((v2, pl2, po2, cuts2))
        n_eval += len(cand)
        bi, bm = first_best(pr, cand)
        if bi >= 0 and bm < cur_mk:
            cur, cur_mk = cand[bi], bm
            steps.append(("placement", cur_mk))
            improved = True
        # schedule phase
        v, pl, po, cuts = cur
        cand = [(v, pl, po2, list(cuts)) for po2 in (GPIPE, ONEF1B, ZB, GREEDY)
                if po2 != po and admitted(v, pl, po2)]
        n_eval += len(cand)
        bi, bm = first_best(pr, cand)
        if bi >= 0 and bm < cur_mk:
            cur, cur_mk = cand[bi], bm
            steps.append(("schedule", cur_mk))
            improved = True
        if not improved:
            break
    v, pl, po, cuts = cur
    return {"status": "ok", "plan": {"v": v, "placement": pl, "policy": po, "S": p * v,
                                      "cuts": [0] + list(cuts) + [L]},
            "makespan": cur_mk, "steps": steps, "rounds": rounds, "n_seeds": len(seeds),
            "n_evaluated": n_eval}
