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

R28' (mode="bottleneck", the default; round 2), closer to P:349-358:
  * each round first identifies the bottleneck phase from the current plan's
    BubbleTime(d) (R29): when the spread max_d - min_d BubbleTime(d) is at
    least the largest stage cost C_s = t_F + t_B + t_W of a micro-batch
    (P:358's stopping threshold), the partition is the bottleneck and is
    tuned first, else placement, then schedule, then partition; the first
    phase that lowers the makespan is accepted and the next round
    re-identifies the bottleneck ("If a tuning step degrades pipeline
    performance, it is rolled back, and alternative adjustments are
    attempted");
  * partition: transfer one layer from the stage of the device with
    the lowest bubble ratio BubbleTime(d) / T_d to the stage of the device
    with the highest (the closest such pair of stages; intermediate stages
    shift by one layer, so stages stay contiguous), with the schedule re-tuned
    in tandem (every policy R12 admits, the best kept); repeated while
    it lowers the makespan and the spread stays >= max C_s. When the first
    transfer does not help, the alternative adjustment is R28's best of the
    L1 ball of radius R around the cuts (same combo);
  * placement: every admitted (v, placement) other than the
    current one, cuts kept for the same v (else the Mist seed), the schedule
    re-tuned in tandem (best admitted policy);
  * schedule: every other admitted policy.
Ties everywhere: the first in the stated order.
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


def stage_costs(pr, cuts):
    """C_s = t_F + t_B + t_W of each stage for one micro-batch (Alg. 1 Step 1)."""
    L = len(pr.t_f)
    full = [0] + list(cuts) + [L]
    return [sum(int(pr.t_f[l]) + int(pr.t_b[l]) + int(pr.t_w[l]) for l in range(a, b))
            for a, b in zip(full, full[1:])]


def transfer(cuts, L, src, dst):
    """Move one layer from stage src to stage dst; the stages between them each
    shift by one layer so that every stage stays contiguous. None if a stage
    would become empty."""
    full = [0] + list(cuts) + [L]
    if src < dst:      # src gives its last layer: cuts src+1 .. dst move left
        for i in range(src + 1, dst + 1):
            full[i] -= 1
    else:              # src gives its first layer: cuts dst+1 .. src move right
        for i in range(dst + 1, src + 1):
            full[i] += 1
    if any(b <= a for a, b in zip(full, full[1:])):
        return None
    return full[1:-1]


def best_policy(pr, v, placement, cuts):
    """The schedule re-tuned in tandem: the first admitted policy of
    smallest makespan for this partition and placement; (plan, makespan)."""
    cands = [(v, placement, po, list(cuts)) for po in (GPIPE, ONEF1B, ZB, GREEDY)
             if admitted(v, placement, po)]
    bi, bm = first_best(pr, cands)
    return (cands[bi], bm) if bi >= 0 else (None, None)


def bottleneck(pr, plan):
    """R29 BubbleTime(d) and T_d of a plan, and the largest stage cost."""
    v, pl, po, cuts = plan
    a = O.comm_accounting(pr, v, pl, po, cuts)
    return a["bubble_d"], a["T_d"], max(stage_costs(pr, cuts))


def generate(pr, vs_mask=0x3, radius=2, max_rounds=32, mode="bottleneck"):
    if mode == "round-robin":
        return _generate_r28(pr, vs_mask, radius, max_rounds)
    if mode != "bottleneck":
        raise ValueError(mode)
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
    state = {"cur": cur, "mk": cur_mk, "n": n_eval}

    def partition_phase():
        accepted = False
        while True:
            bub, T, maxcs = bottleneck(pr, state["cur"])
            if max(bub) - min(bub) < maxcs:
                break          # BubbleTime spread below the largest C_s
            v, pl, po, cuts = state["cur"]
            # bubble ratios compared exactly: bub[a] / T[a] vs bub[b] / T[b]
            lo = hi = 0
            for d in range(1, p):
                if bub[d] * T[lo] < bub[lo] * T[d]:
                    lo = d
                if bub[d] * T[hi] > bub[hi] * T[d]:
                    hi = d
            if lo == hi:
                break
            S = p * v
            src_st = [s for s in range(S) if O.device_of_stage(pl, p, v, s) == lo]
            dst_st = [s for s in range(S) if O.device_of_stage(pl, p, v, s) == hi]
            pair = min(((abs(a - b), a, b) for a in src_st for b in dst_st))
            nc = transfer(cuts, L, pair[1], pair[2])
            if nc is None:
                break
            plan, bm = best_policy(pr, v, pl, nc)
            state["n"] += sum(1 for po2 in range(4) if admitted(v, pl, po2))
            if bm is None or bm >= state["mk"]:
                break          # rolled back
            state["cur"], state["mk"] = plan, bm
            steps.append(("partition", bm))
            accepted = True
        if accepted:
            return True
        # alternative adjustment: the best partition of the L1 ball (R28)
        v, pl, po, cuts = state["cur"]
        sp = W.Space([W.Group(v, W.BALL, radius, seed_cuts=list(cuts),
                              combo_mask=1 << combo_index(v, pl, po))])
        state["n"] += O.space_size(pr, sp)
        b = O.search(pr, sp, prune=True)
        if b["index"] != (1 << 64) - 1 and b["makespan"] < state["mk"]:
            state["cur"], state["mk"] = (v, pl, po, b["plan"]["cuts"][1:-1]), b["makespan"]
            steps.append(("partition", state["mk"]))
            return True
        return False

    def placement_phase():
        v, pl, po, cuts = state["cur"]
        best = None
        for v2 in vs:
            for pl2 in ([SEQ] if v2 == 1 else [INT, WAVE]):
                if (v2, pl2) == (v, pl):
                    continue
                cuts2 = list(cuts) if v2 == v else mist(pr, p * v2)
                plan, bm = best_policy(pr, v2, pl2, cuts2)
                state["n"] += sum(1 for po2 in range(4) if admitted(v2, pl2, po2))
                if bm is not None and (best is None or bm < best[1]):
                    best = (plan, bm)
        if best is not None and best[1] < state["mk"]:
            state["cur"], state["mk"] = best
            steps.append(("placement", best[1]))
            return True
        return False

    def schedule_phase():
        v, pl, po, cuts = state["cur"]
        cand = [(v, pl, po2, list(cuts)) for po2 in (GPIPE, ONEF1B, ZB, GREEDY)
                if po2 != po and admitted(v, pl, po2)]
        state["n"] += len(cand)
        bi, bm = first_best(pr, cand)
        if bi >= 0 and bm < state["mk"]:
            state["cur"], state["mk"] = cand[bi], bm
            steps.append(("schedule", bm))
            return True
        return False

    rounds = 0
    while rounds < max_rounds:
        rounds += 1
        bub, T, maxcs = bottleneck(pr, state["cur"])
        order = ([partition_phase, placement_phase, schedule_phase] if max(bub) - min(bub) >= maxcs
                 else [placement_phase, schedule_phase, partition_phase])
        if not any(ph() for ph in order):   # any() stops at the first accepted phase
            break
    v, pl, po, cuts = state["cur"]
    return {"status": "ok", "plan": {"v": v, "placement": pl, "policy": po, "S": p * v,
                                      "cuts": [0] + list(cuts) + [L]},
            "makespan": state["mk"], "steps": steps, "rounds": rounds, "n_seeds": len(seeds),
            "n_evaluated": state["n"]}


def _generate_r28(pr, vs_mask=0x3, radius=2, max_rounds=32):
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
