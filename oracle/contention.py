"""Engine-contention oracle (reading R34). TEST INFRASTRUCTURE ONLY.

Only tests/ (and smoke / bench's cpu legs) may import this module. It shares
no code with the CUDA path: plain Python, one discrete-event loop written
from the rules it cites, slow and small-case only.

What it computes: Alg. 1 Step 3 on explicit per-device task lists
(reading R30) when transfers compete for the devices' communication
engines, as SPEC S:206 (a)-(c) and S:232 state:
  (a) each device owns one compute engine, one send engine and one receive
      engine (S:206 (a); full duplex);
  (b) a device runs its list strictly in order; a task starts when the
      previous task of the device has finished and every DAG predecessor
      (S:141 edges) has finished or, across devices, its transfer has arrived;
  (c) a cross-device transfer becomes eligible when its producing task ends,
      then occupies the sender's send engine and the receiver's receive
      engine, FIFO by eligibility time with ties broken by the smaller
      (mb, stage, kind-order F < B) of the producing task, for comm_time
      ticks (the boundary's comm_ticks entry, R3-R5).
Readings (R34): a transfer holds both engines for its whole
duration, so it starts at max(eligible, send engine free, receive engine
free); an edge between stages on one device, or with latency 0, is not a
transfer (it arrives at the producer's finish, as in R29); memory follows R16
at task starts, so M_d depends on the lists alone.
"""
from __future__ import annotations

import heapq

INT64_MAX = (1 << 63) - 1


def _device_of_stage(placement, p, s):
    """Placement families of P:177-178 (R12), written out."""
    if placement == 0:          # SEQ (S-1F1B)
        return s
    if placement == 1:          # INTERLEAVED (I-1F1B): stage s on device s mod p
        return s % p
    c, j = divmod(s, p)         # WAVE (Hanayo): direction flips every p stages
    return p - 1 - j if c % 2 else j


def simulate_lists_contended(pr, v, placement, fused, cuts, lists, trace=False):
    """Event-driven simulation under R34. Returns a dict with status
    (0 ok, 2 over cap, 3 stuck; stuck wins, R26/R30), makespan (INT64_MAX unless
    ok), peak_mem (0 when stuck), T_d, busy_d, M_d, comm_d, exposed_d and, with
    trace=True, the task intervals and the transfer intervals."""
    L, p, m = len(pr.t_f), pr.p, pr.m
    cuts = list(cuts)
    full = cuts if (cuts and cuts[0] == 0 and cuts[-1] == L) else [0] + cuts + [L]
    S = len(full) - 1

    def ssum(col, s):
        return int(sum(int(x) for x in col[full[s]:full[s + 1]]))

    tf = [ssum(pr.t_f, s) for s in range(S)]
    tb = [ssum(pr.t_b, s) for s in range(S)]
    tw = [ssum(pr.t_w, s) for s in range(S)]
    act = [ssum(pr.act, s) for s in range(S)]
    sta = [ssum(pr.stash, s) for s in range(S)]
    wg = [ssum(pr.weight, s) + ssum(pr.grad, s) for s in range(S)]
    dev = [_device_of_stage(placement, p, s) for s in range(S)]
    dur = {0: tf, 1: [b + w for b, w in zip(tb, tw)] if fused else tb, 2: tw}

    def out_edge(k, s):
        """(consumer device, latency, consumer stage) of task (k, s)'s output
        edge, or None. F(s) feeds F(s+1); B(s) feeds B(s-1)."""
        if k == 0 and s + 1 < S:
            return dev[s + 1], int(pr.comm[full[s + 1] - 1]), s + 1
        if k == 1 and s > 0:
            return dev[s - 1], int(pr.comm[full[s] - 1]), s - 1
        return None

    def inputs(k, s, j):
        """DAG predecessors of (k, s, j) as (task, over an edge?): F(s-1)
        -> F(s) and B(s+1) -> B(s) are stage edges (their output may travel);
        F(s) -> B(s) and B(s) -> W(s) stay on the stage's device."""
        if k == 0:
            return [((0, s - 1, j), True)] if s > 0 else []
        if k == 1:
            return [((0, s, j), False)] + ([((1, s + 1, j), True)] if s + 1 < S else [])
        return [((1, s, j), False)]

    # memory along each list (R16): order only
    busy = [0] * p
    Md = [0] * p
    for d in range(p):
        stat = sum(wg[s] for s in range(S) if dev[s] == d)
        dyn = peak = 0
        for (k, s, j) in lists[d]:
            busy[d] += dur[k][s]
            if k == 0:
                dyn += act[s] + sta[s]
                peak = max(peak, dyn)
            elif k == 1:
                dyn -= act[s] + (sta[s] if fused else 0)
            else:
                dyn -= sta[s]
        Md[d] = stat + peak

    fin = {}        # task -> finish time
    ready = {}      # task -> time its output reaches the next (F) / previous (B) stage
    ptr = [0] * p
    free = [0] * p
    send_free = [0] * p
    recv_free = [0] * p
    pending = []    # heap of (eligible, mb, stage, kind, src, dst, latency)
    task_iv = [[] for _ in range(p)]
    xfer_iv = []    # (src, dst, start, arrival, (kind, stage, mb))

    def startable(d):
        if ptr[d] >= len(lists[d]):
            return None
        k, s, j = lists[d][ptr[d]]
        t = free[d]
        for q, edge in inputs(k, s, j):
            have = ready if edge else fin
            if q not in have:
                return None
            t = max(t, have[q])
        return t

    while True:
        # (b): run every task whose inputs are all there, one device at a time
        progressed = True
        while progressed:
            progressed = False
            for d in range(p):
                t = startable(d)
                if t is None:
                    continue
                k, s, j = lists[d][ptr[d]]
                f = t + dur[k][s]
                fin[(k, s, j)] = f
                task_iv[d].append((t, f, (k, s, j)))
                free[d] = f
                ptr[d] += 1
                e = out_edge(k, s)
                if k == 2 or e is None or e[0] == d or e[1] == 0:
                    ready[(k, s, j)] = f   # local edge, zero latency, or no consumer
                else:
                    heapq.heappush(pending, (f, j, s, k, d, e[0], e[1]))
                progressed = True
        # (c): no compute engine can start anything, so every transfer still to
        # be created will be eligible strictly later than the earliest pending
        # one: that one is next on both of its engines
        if not pending:
            break
        f, j, s, k, src, dst, lat = heapq.heappop(pending)
        start = max(f, send_free[src], recv_free[dst])
        arr = start + lat
        send_free[src] = arr
        recv_free[dst] = arr
        ready[(k, s, j)] = arr
        xfer_iv.append((src, dst, start, arr, (k, s, j)))

    if any(ptr[d] < len(lists[d]) for d in range(p)):
        res = {"status": 3, "makespan": INT64_MAX, "peak_mem": 0, "T_d": [0] * p,
               "busy_d": busy, "M_d": Md, "comm_d": [0] * p, "exposed_d": [0] * p}
        return res
    Td = [max((iv[1] for iv in task_iv[d]), default=0) for d in range(p)]
    # R29 on the contended schedule: transfers occupy [start, arrival) on both
    # devices; exposed = ticks t < T_d inside some transfer and outside compute
    comm = [0] * p
    exposed = [0] * p
    for d in range(p):
        # sweep over the interval endpoints: count open transfers and open
        # compute intervals, add the length where a transfer and no compute is open
        ev = []
        for (a, b, _x) in task_iv[d]:
            ev += [(a, 0, 1), (b, 0, -1)]
        for (src, dst, a, b, _x) in xfer_iv:
            if d in (src, dst):
                comm[d] += b - a
                ev += [(a, 1, 1), (b, 1, -1)]
        ev.sort()
        open_c = open_x = 0
        prev = 0
        for (x, kind, delta) in ev:
            x = min(x, Td[d])
            if open_x > 0 and open_c == 0 and x > prev:
                exposed[d] += x - prev
            prev = max(prev, x)
            if kind == 0:
                open_c += delta
            else:
                open_x += delta
    status = 2 if max(Md) > pr.cap else 0
    res = {"status": status, "makespan": max(Td) if status == 0 else INT64_MAX,
           "peak_mem": max(Md), "T_d": Td, "busy_d": busy, "M_d": Md,
           "comm_d": comm, "exposed_d": exposed}
    if trace:
        res["tasks"] = task_iv
        res["transfers"] = xfer_iv
    return res


def simulate_realised_contended(pr, v, placement, policy, cuts):
    """Reading R36 (contention on realised orders): the policy decides each
    device's order with pure-latency communication (the event loop, R9-R14);
    that order is then executed as an explicit schedule (R30) under the R34
    send/receive engines. Candidates without a complete order (invalid cuts,
    stuck GREEDY) keep the event loop's status. `cuts` is the full list
    [0, c_1, ..., L] (unambiguous also for invalid decodes)."""
    from . import oracle as O
    r = O.simulate(pr, v, placement, policy, cuts, trace=True)
    if r["status"] not in (0, 2):
        return {"status": r["status"], "makespan": O.INT64_MAX, "peak_mem": 0}
    fused = policy in (0, 1)
    lists = [[(k, s, j) for (k, s, j, _t) in lst if not (fused and k == 2)] for lst in r["trace"]]
    return simulate_lists_contended(pr, v, placement, fused, cuts, lists)
