"""ctypes wrapper of the C oracle (oracle.c). TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this module. It never imports the CUDA
package; inputs arrive as plain numpy arrays (workloads.Problem/Space objects
are duck-typed: only their attributes are read).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")
SRC = os.path.join(HERE, "oracle.c")
HDR = os.path.join(HERE, "oracle.h")
INC = os.path.join(HERE, "oracle_sim.inc")
MAXS, MAXP = 64, 32
INT64_MAX = (1 << 63) - 1
UINT64_MAX = (1 << 64) - 1

_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (plain C11 + pthreads)."""
    stale = (not os.path.exists(LIB) or
             max(os.path.getmtime(f) for f in (SRC, HDR, INC)) > os.path.getmtime(LIB))
    if force or stale:
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-Wall", "-fPIC", "-shared", "-pthread",
                               SRC, "-o", LIB + ".tmp", "-lm"])
        os.replace(LIB + ".tmp", LIB)
    return LIB


class _Problem(C.Structure):
    _fields_ = [("L", C.c_int)] + [(n, C.POINTER(C.c_int64)) for n in
                                   ("t_f", "t_b", "t_w", "act", "stash", "weight", "grad", "comm")] + \
               [("p", C.c_int), ("m", C.c_int), ("cap", C.c_int64),
                ("costs_f64", C.POINTER(C.c_double)), ("time_f32", C.c_int)]


class _Plan(C.Structure):
    _fields_ = [("v", C.c_int), ("placement", C.c_int), ("policy", C.c_int), ("S", C.c_int),
                ("cuts", C.c_int * (MAXS + 1))]


class _Result(C.Structure):
    _fields_ = [("status", C.c_int), ("makespan", C.c_int64), ("peak_mem", C.c_int64),
                ("bubble", C.c_double)] + [(n, C.c_int64 * MAXP) for n in
                                           ("T_d", "busy_d", "M_d", "static_d")] + \
               [("makespan_f", C.c_double), ("T_f", C.c_double * MAXP)]


class _Trace(C.Structure):
    _fields_ = [("cap_per_dev", C.c_int), ("n", C.c_int * MAXP),
                ("kind", C.POINTER(C.c_int)), ("stage", C.POINTER(C.c_int)),
                ("mb", C.POINTER(C.c_int)), ("start", C.POINTER(C.c_int64))]


class _Group(C.Structure):
    _fields_ = [("v", C.c_int), ("part_mode", C.c_int), ("radius", C.c_int),
                ("seed_cuts", C.POINTER(C.c_int)), ("combo_mask", C.c_uint)]


class _Space(C.Structure):
    _fields_ = [("n_groups", C.c_int), ("group", _Group * 4)]


class _Best(C.Structure):
    _fields_ = [("index", C.c_uint64), ("makespan", C.c_int64), ("plan", _Plan),
                ("n_total", C.c_uint64), ("n_invalid", C.c_uint64), ("n_simulated", C.c_uint64),
                ("n_feasible", C.c_uint64)]


CB = C.CFUNCTYPE(None, C.c_uint64, C.POINTER(_Plan), C.c_void_p)


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = C.CDLL(LIB)
            L.orc_simulate.argtypes = [C.POINTER(_Problem), C.POINTER(_Plan), C.POINTER(_Result),
                                       C.POINTER(_Trace)]
            L.orc_longest_path.argtypes = [C.POINTER(_Problem), C.POINTER(_Plan), C.c_int,
                                           C.POINTER(_Trace), C.POINTER(C.c_int64),
                                           C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
            L.orc_fixed_order.argtypes = [C.POINTER(_Problem), C.POINTER(_Plan), C.c_int,
                                          C.POINTER(C.c_int), C.POINTER(C.c_int),
                                          C.POINTER(C.c_int), C.c_int]
            L.orc_seed_minmax.restype = C.c_int64
            L.orc_seed_minmax.argtypes = [C.c_int, C.POINTER(C.c_int64), C.c_int, C.POINTER(C.c_int)]
            L.orc_device_of_stage.argtypes = [C.c_int] * 4
            L.orc_combo.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]
            L.orc_space_size.restype = C.c_uint64
            L.orc_space_size.argtypes = [C.POINTER(_Problem), C.POINTER(_Space), C.POINTER(C.c_int)]
            L.orc_enumerate.argtypes = [C.POINTER(_Problem), C.POINTER(_Space), CB, C.c_void_p]
            L.orc_decode.argtypes = [C.POINTER(_Problem), C.POINTER(_Space), C.c_uint64,
                                     C.POINTER(_Plan)]
            L.orc_eval_indices.argtypes = [C.POINTER(_Problem), C.POINTER(_Space),
                                           C.POINTER(C.c_uint64), C.c_uint64, C.c_int,
                                           C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                           C.POINTER(C.c_double), C.POINTER(C.c_uint8),
                                           C.POINTER(C.c_double)]
            L.orc_simulate_f64.argtypes = L.orc_simulate.argtypes
            L.orc_simulate_f32.argtypes = L.orc_simulate.argtypes
            L.orc_search.argtypes = [C.POINTER(_Problem), C.POINTER(_Space), C.c_int, C.c_int,
                                     C.POINTER(_Best)]
            _lib = L
    return _lib


def _i64p(a):
    return a.ctypes.data_as(C.POINTER(C.c_int64))


class _Ctx:
    """Keeps numpy arrays alive while C structs point into them."""

    def __init__(self, pr, sp=None, precision="f64"):
        self.keep = []
        cols = {}
        for n in ("t_f", "t_b", "t_w", "act", "stash", "weight", "grad", "comm"):
            a = np.ascontiguousarray(np.asarray(getattr(pr, n), dtype=np.int64))
            self.keep.append(a)
            cols[n] = _i64p(a)
        cf = None
        if getattr(pr, "costs_f32", None) is not None and getattr(pr, "cost_type", 0) == 1:
            # the fp64 reference of the fp32-cost variant reads the same fp32 values
            a = np.ascontiguousarray(np.asarray(pr.costs_f32, dtype=np.float64))
            self.keep.append(a)
            cf = a.ctypes.data_as(C.POINTER(C.c_double))
        if precision not in ("f64", "f32"):
            raise ValueError(precision)
        # fp32-cost variant: "f64" = real-arithmetic reference, "f32" = every time
        # value and decision in fp32, as the kernel computes them (reading R27)
        self.pr = _Problem(L=len(pr.t_f), p=pr.p, m=pr.m, cap=int(pr.cap), costs_f64=cf,
                           time_f32=int(precision == "f32"), **cols)
        self.sp = None
        if sp is not None:
            s = _Space()
            s.n_groups = len(sp.groups)
            for i, g in enumerate(sp.groups):
                seed = None
                if g.seed_cuts is not None:
                    arr = (C.c_int * len(g.seed_cuts))(*g.seed_cuts)
                    self.keep.append(arr)
                    seed = C.cast(arr, C.POINTER(C.c_int))
                s.group[i] = _Group(v=g.v, part_mode=g.part_mode, radius=g.radius,
                                    seed_cuts=seed, combo_mask=g.combo_mask)
            self.sp = s


def make_plan(v, placement, policy, cuts, L=None):
    """cuts: interior cuts (S-1 values) or the full list [0, ..., L]."""
    cuts = list(cuts)
    if L is not None and (not cuts or cuts[0] != 0 or cuts[-1] != L):
        cuts = [0] + cuts + [L]
    pl = _Plan(v=v, placement=placement, policy=policy, S=len(cuts) - 1)
    for i, c in enumerate(cuts):
        pl.cuts[i] = c
    return pl


def plan_dict(pl):
    return {"v": pl.v, "placement": pl.placement, "policy": pl.policy, "S": pl.S,
            "cuts": [pl.cuts[i] for i in range(pl.S + 1)]}


def simulate(pr, v, placement, policy, cuts, trace=False, precision="f64"):
    """Alg. 1 for one candidate. cuts = interior cuts. Returns a dict."""
    ctx = _Ctx(pr, precision=precision)
    pl = make_plan(v, placement, policy, cuts, L=len(pr.t_f))
    res = _Result()
    tr_p = None
    if trace:
        capd = 3 * pl.S * pr.m
        arrs = [np.zeros(capd * pr.p, np.int32) for _ in range(3)] + [np.zeros(capd * pr.p, np.int64)]
        tr = _Trace(cap_per_dev=capd, kind=arrs[0].ctypes.data_as(C.POINTER(C.c_int)),
                    stage=arrs[1].ctypes.data_as(C.POINTER(C.c_int)),
                    mb=arrs[2].ctypes.data_as(C.POINTER(C.c_int)), start=_i64p(arrs[3]))
        tr_p = C.pointer(tr)
    sim = (lib().orc_simulate if not ctx.pr.costs_f64 else
           lib().orc_simulate_f32 if ctx.pr.time_f32 else lib().orc_simulate_f64)
    rc = sim(C.byref(ctx.pr), C.byref(pl), C.byref(res), tr_p)
    if rc != 0:
        raise RuntimeError("oracle internal inconsistency")
    p = pr.p
    out = {"status": res.status, "makespan": res.makespan, "peak_mem": res.peak_mem,
           "makespan_f": res.makespan_f,
           "bubble": res.bubble, "T_d": list(res.T_d[:p]), "busy_d": list(res.busy_d[:p]),
           "M_d": list(res.M_d[:p]), "static_d": list(res.static_d[:p])}
    if trace:
        lists = []
        for d in range(p):
            n = tr.n[d]
            o = d * capd
            lists.append([(int(arrs[0][o + i]), int(arrs[1][o + i]), int(arrs[2][o + i]),
                           int(arrs[3][o + i])) for i in range(n)])
        out["trace"] = lists
    return out


def longest_path(pr, v, placement, cuts, fused, lists):
    """Independent longest-path checker over explicit per-device lists of
    (kind, stage, mb). Returns (makespan, T_d, starts) or None on a cycle."""
    ctx = _Ctx(pr)
    pl = make_plan(v, placement, 0, cuts, L=len(pr.t_f))
    capd = max(1, max(len(x) for x in lists))
    p = pr.p
    kind = np.zeros(capd * p, np.int32)
    stage = np.zeros(capd * p, np.int32)
    mb = np.zeros(capd * p, np.int32)
    start = np.zeros(capd * p, np.int64)
    tr = _Trace(cap_per_dev=capd, kind=kind.ctypes.data_as(C.POINTER(C.c_int)),
                stage=stage.ctypes.data_as(C.POINTER(C.c_int)),
                mb=mb.ctypes.data_as(C.POINTER(C.c_int)), start=_i64p(start))
    for d, lst in enumerate(lists):
        tr.n[d] = len(lst)
        for i, t in enumerate(lst):
            kind[d * capd + i], stage[d * capd + i], mb[d * capd + i] = t[0], t[1], t[2]
    st = np.zeros(capd * p, np.int64)
    mk = C.c_int64()
    Td = (C.c_int64 * MAXP)()
    cyc = lib().orc_longest_path(C.byref(ctx.pr), C.byref(pl), int(fused), C.byref(tr), _i64p(st),
                                 C.byref(mk), Td)
    if cyc:
        return None
    starts = [[int(st[d * capd + i]) for i in range(len(lists[d]))] for d in range(p)]
    return mk.value, list(Td[:p]), starts


def fixed_order(pr, v, placement, policy, cuts, d):
    ctx = _Ctx(pr)
    pl = make_plan(v, placement, policy, cuts, L=len(pr.t_f))
    cap = 2 * pr.m * v
    k = (C.c_int * cap)(); s = (C.c_int * cap)(); j = (C.c_int * cap)()
    n = lib().orc_fixed_order(C.byref(ctx.pr), C.byref(pl), d, k, s, j, cap)
    return [(k[i], s[i], j[i]) for i in range(n)]


def seed_minmax(w, S):
    w = np.ascontiguousarray(np.asarray(w, dtype=np.int64))
    cuts = (C.c_int * max(1, S))()
    val = lib().orc_seed_minmax(len(w), _i64p(w), S, cuts)
    return val, [cuts[i] for i in range(S - 1)]


def device_of_stage(placement, p, v, s):
    return lib().orc_device_of_stage(placement, p, v, s)


def combo(v, k):
    a, b = C.c_int(), C.c_int()
    ok = lib().orc_combo(v, k, C.byref(a), C.byref(b))
    return (a.value, b.value) if ok else None


def space_size(pr, sp):
    ctx = _Ctx(pr, sp)
    of = C.c_int()
    n = lib().orc_space_size(C.byref(ctx.pr), C.byref(ctx.sp), C.byref(of))
    if of.value:
        raise OverflowError("space size does not fit in 63 bits")
    return int(n)


def enumerate_space(pr, sp, limit=10_000_000):
    """Every candidate in canonical order (small spaces only)."""
    ctx = _Ctx(pr, sp)
    out = []

    def cb(idx, plp, _):
        if len(out) < limit:
            out.append((int(idx), plan_dict(plp.contents)))
    f = CB(cb)
    lib().orc_enumerate(C.byref(ctx.pr), C.byref(ctx.sp), f, None)
    return out


def decode(pr, sp, index):
    ctx = _Ctx(pr, sp)
    pl = _Plan()
    if lib().orc_decode(C.byref(ctx.pr), C.byref(ctx.sp), index, C.byref(pl)) != 0:
        raise IndexError(index)
    return plan_dict(pl)


def eval_indices(pr, sp, indices, nthreads=None, precision="f64"):
    ctx = _Ctx(pr, sp, precision=precision)
    idx = np.ascontiguousarray(np.asarray(indices, dtype=np.uint64))
    n = idx.shape[0]
    ms = np.zeros(n, np.int64); pk = np.zeros(n, np.int64)
    bub = np.zeros(n, np.float64); st = np.zeros(n, np.uint8)
    msf = np.zeros(n, np.float64)
    nth = nthreads or os.cpu_count() or 1
    rc = lib().orc_eval_indices(C.byref(ctx.pr), C.byref(ctx.sp),
                                idx.ctypes.data_as(C.POINTER(C.c_uint64)), n, nth, _i64p(ms),
                                _i64p(pk), bub.ctypes.data_as(C.POINTER(C.c_double)),
                                st.ctypes.data_as(C.POINTER(C.c_uint8)),
                                msf.ctypes.data_as(C.POINTER(C.c_double)))
    if rc != 0:
        raise RuntimeError("oracle internal inconsistency")
    return {"makespan": ms, "peak_mem": pk, "bubble": bub, "status": st, "makespan_f": msf}


def search(pr, sp, prune=True, nthreads=None):
    ctx = _Ctx(pr, sp)
    b = _Best()
    nth = nthreads or os.cpu_count() or 1
    rc = lib().orc_search(C.byref(ctx.pr), C.byref(ctx.sp), int(prune), nth, C.byref(b))
    if rc != 0:
        raise RuntimeError("oracle internal inconsistency")
    return {"index": int(b.index), "makespan": int(b.makespan), "plan": plan_dict(b.plan),
            "n_total": int(b.n_total), "n_invalid": int(b.n_invalid),
            "n_simulated": int(b.n_simulated), "n_feasible": int(b.n_feasible)}


def comm_accounting(pr, v, placement, policy, cuts):
    """Reading R29 (Alg. 1 Step 3: T_d = C_d + BubbleTime(d) -
    OverlapTime(d), with C_d = busy_d + ProfiledCommCost), by brute force on the
    integer tick grid of the event loop's trace:
      * every cross-device dependency edge (F(s) -> F(s+1), B(s) -> B(s-1);
        R3-R6) is a transfer occupying [producer finish, + latency) on both
        the sending and the receiving device;
      * comm_d = sum of the latencies of the transfers incident to d;
      * exposed_d = ticks t < T_d with some incident transfer and no compute
        on d; overlap_d = comm_d - exposed_d; bubble_d = T_d - busy_d - exposed_d.
    Returns the simulate() dict extended with those four per-device lists."""
    r = simulate(pr, v, placement, policy, cuts, trace=True)
    L, p = len(pr.t_f), pr.p
    cuts = list(cuts)
    full = cuts if (cuts and cuts[0] == 0 and cuts[-1] == L) else [0] + cuts + [L]
    S = len(full) - 1
    fused = policy in (0, 1)  # GPIPE, ONEF1B run B and W fused (R2)
    dev = [device_of_stage(placement, p, v, s) for s in range(S)]
    tf = [int(sum(pr.t_f[full[s]:full[s + 1]])) for s in range(S)]
    tb = [int(sum(pr.t_b[full[s]:full[s + 1]])) for s in range(S)]
    tw = [int(sum(pr.t_w[full[s]:full[s + 1]])) for s in range(S)]
    dur = {0: tf, 1: [b + w for b, w in zip(tb, tw)] if fused else tb, 2: tw}
    out = {k: [0] * p for k in ("comm_d", "exposed_d", "overlap_d", "bubble_d")}
    if r["status"] not in (0, 2) or "trace" not in r:
        return {**r, **out}
    T = r["T_d"]
    busy = [np.zeros(max(T[d], 1), bool) for d in range(p)]
    xfer = [np.zeros(max(T[d], 1), bool) for d in range(p)]
    for d, lst in enumerate(r["trace"]):
        for (k, s, j, st) in lst:
            fin = st + dur[k][s]
            busy[d][st:fin] = True
            tgt = None
            if k == 0 and s + 1 < S and dev[s + 1] != d:
                tgt, lat = dev[s + 1], int(pr.comm[full[s + 1] - 1])
            elif k == 1 and s > 0 and dev[s - 1] != d:
                tgt, lat = dev[s - 1], int(pr.comm[full[s] - 1])
            if tgt is None or lat == 0:
                continue
            for e in (d, tgt):
                out["comm_d"][e] += lat
                xfer[e][fin:fin + lat] = True  # numpy clips at T_e
    for d in range(p):
        n = T[d]
        out["exposed_d"][d] = int(np.count_nonzero(xfer[d][:n] & ~busy[d][:n]))
        out["overlap_d"][d] = out["comm_d"][d] - out["exposed_d"][d]
        out["bubble_d"][d] = T[d] - r["busy_d"][d] - out["exposed_d"][d]
    return {**r, **out}


def simulate_lists(pr, v, placement, fused, cuts, lists):
    """Reading R30 (Alg. 1 Step 3 on explicit workload scheduling results):
    device d executes lists[d] = [(kind, stage, mb), ...] in order; times are the
    longest path over the task DAG plus the list edges (the independent checker
    `longest_path`); memory is walked along each list with the R16 rules. A
    cyclic wait gives status 3 (stuck), a device above the cap status 2."""
    L, p, m = len(pr.t_f), pr.p, pr.m
    cuts = list(cuts)
    full = cuts if (cuts and cuts[0] == 0 and cuts[-1] == L) else [0] + cuts + [L]
    S = len(full) - 1

    def ssum(col, s):
        return int(sum(col[full[s]:full[s + 1]]))
    tf = [ssum(pr.t_f, s) for s in range(S)]
    tb = [ssum(pr.t_b, s) for s in range(S)]
    tw = [ssum(pr.t_w, s) for s in range(S)]
    act = [ssum(pr.act, s) for s in range(S)]
    sta = [ssum(pr.stash, s) for s in range(S)]
    wg = [ssum(pr.weight, s) + ssum(pr.grad, s) for s in range(S)]
    dev = [device_of_stage(placement, p, v, s) for s in range(S)]
    dur = {0: tf, 1: [b + w for b, w in zip(tb, tw)] if fused else tb, 2: tw}
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
    lp = longest_path(pr, v, placement, full[1:-1], fused, lists)
    out = {"busy_d": busy, "M_d": Md}
    if lp is None:
        return {**out, "status": 3, "makespan": INT64_MAX, "peak_mem": 0, "T_d": [0] * p}
    mk, Td, _ = lp
    status = 2 if max(Md) > pr.cap else 0
    return {**out, "status": status, "makespan": mk if status == 0 else INT64_MAX,
            "peak_mem": max(Md), "T_d": Td}


def repair_oom(pr, v, placement, fused, cuts, lists, max_moves=0):
    """Reading R31 ("identifies potential OOM time ... advances the
    execution of the latest B and W to ahead of this time to free up memory,
    continuing this process until all potential OOM errors are resolved"),
    written out on top of simulate_lists / longest_path:
      1. simulate the lists; stop unless the status is 2 (over the cap);
      2. per device, walk the list's memory (R16) to the first F whose
         allocation exceeds the cap; visit these violations by start time
         (ties: lower device) and take the first with a movable B:
      3. on that device, among the B listed after that F whose own F is
         listed before it and whose input B(s+1, j) (same device: listed
         before it; other device: finish + latency <= that time) is there,
         take the latest listed; move it just before the F (its W right after
         it when split);
      4. repeat (at most max_moves moves; <= 0: the number of tasks).
    Returns (lists, moves, simulate_lists result)."""
    L, p = len(pr.t_f), pr.p
    cuts = list(cuts)
    full = cuts if (cuts and cuts[0] == 0 and cuts[-1] == L) else [0] + cuts + [L]
    S = len(full) - 1

    def ssum(col, s):
        return int(sum(col[full[s]:full[s + 1]]))
    act = [ssum(pr.act, s) for s in range(S)]
    sta = [ssum(pr.stash, s) for s in range(S)]
    wg = [ssum(pr.weight, s) + ssum(pr.grad, s) for s in range(S)]
    dur_f = [ssum(pr.t_f, s) for s in range(S)]
    dur_b = [ssum(pr.t_b, s) + (ssum(pr.t_w, s) if fused else 0) for s in range(S)]
    dur_w = [ssum(pr.t_w, s) for s in range(S)]
    dev = [device_of_stage(placement, p, v, s) for s in range(S)]
    lists = [list(x) for x in lists]
    total = sum(len(x) for x in lists)
    if max_moves <= 0:
        max_moves = total
    moves = 0
    while True:
        r = simulate_lists(pr, v, placement, fused, full, lists)
        if r["status"] != 2 or moves >= max_moves:
            return lists, moves, r
        lp = longest_path(pr, v, placement, full[1:-1], fused, lists)
        starts = lp[2]
        where = {}
        for d in range(p):
            for i, t in enumerate(lists[d]):
                where[t] = (d, i)
        viols = []
        for d in range(p):
            stat = sum(wg[s] for s in range(S) if dev[s] == d)
            dyn = 0
            for i, (k, s, j) in enumerate(lists[d]):
                if k == 0:
                    dyn += act[s] + sta[s]
                    if stat + dyn > pr.cap:
                        viols.append((starts[d][i], d, i))
                        break
                elif k == 1:
                    dyn -= act[s] + (sta[s] if fused else 0)
                else:
                    dyn -= sta[s]
        chosen = None
        for tv, d, q in sorted(viols):  # earliest violation with a movable B
            for i in range(len(lists[d]) - 1, q, -1):
                k, s, j = lists[d][i]
                if k != 1 or where[(0, s, j)][1] >= q:
                    continue
                if s + 1 < S:
                    d2, i2 = where[(1, s + 1, j)]
                    if d2 == d:
                        if i2 >= q:
                            continue
                    else:
                        lat = int(pr.comm[full[s + 1] - 1])
                        if starts[d2][i2] + dur_b[s + 1] + lat > tv:
                            continue
                chosen = i
                break
            if chosen is not None:
                break
        if chosen is None:
            return lists, moves, r
        b = lists[d].pop(chosen)
        lists[d].insert(q, b)
        if not fused:
            wi = lists[d].index((2, b[1], b[2]))
            if wi > q + 1:
                lists[d].insert(q + 1, lists[d].pop(wi))
        moves += 1


def _list_schedule(pr, v, placement, fused, cuts, lists):
    """Stage data, durations and the longest-path starts of explicit lists."""
    L, p = len(pr.t_f), pr.p
    full = list(cuts) if (cuts and cuts[0] == 0 and cuts[-1] == L) else [0] + list(cuts) + [L]
    S = len(full) - 1

    def ssum(col, s):
        return int(sum(col[full[s]:full[s + 1]]))
    dur = {0: [ssum(pr.t_f, s) for s in range(S)],
           1: [ssum(pr.t_b, s) + (ssum(pr.t_w, s) if fused else 0) for s in range(S)],
           2: [ssum(pr.t_w, s) for s in range(S)]}
    dev = [device_of_stage(placement, p, v, s) for s in range(S)]
    lp = longest_path(pr, v, placement, full[1:-1], fused, lists)
    return full, S, dur, dev, lp


def comm_accounting_lists(pr, v, placement, fused, cuts, lists):
    """R29 for explicit lists (R30), by brute force on the tick grid of the
    longest-path schedule: comm_d, exposed_d, overlap_d, bubble_d per device."""
    r = simulate_lists(pr, v, placement, fused, cuts, lists)
    p = pr.p
    out = {k: [0] * p for k in ("comm_d", "exposed_d", "overlap_d", "bubble_d")}
    if r["status"] not in (0, 2):
        return {**r, **out}
    full, S, dur, dev, lp = _list_schedule(pr, v, placement, fused, cuts, lists)
    T = r["T_d"]
    busy = [np.zeros(max(T[d], 1), bool) for d in range(p)]
    xfer = [np.zeros(max(T[d], 1), bool) for d in range(p)]
    for d in range(p):
        for (k, s, j), st in zip(lists[d], lp[2][d]):
            fin = st + dur[k][s]
            busy[d][st:fin] = True
            tgt = None
            if k == 0 and s + 1 < S and dev[s + 1] != d:
                tgt, lat = dev[s + 1], int(pr.comm[full[s + 1] - 1])
            elif k == 1 and s > 0 and dev[s - 1] != d:
                tgt, lat = dev[s - 1], int(pr.comm[full[s] - 1])
            if tgt is None or lat == 0:
                continue
            for e in (d, tgt):
                out["comm_d"][e] += lat
                xfer[e][fin:fin + lat] = True
    for d in range(p):
        n = T[d]
        out["exposed_d"][d] = int(np.count_nonzero(xfer[d][:n] & ~busy[d][:n]))
        out["overlap_d"][d] = out["comm_d"][d] - out["exposed_d"][d]
        out["bubble_d"][d] = T[d] - r["busy_d"][d] - out["exposed_d"][d]
    return {**r, **out}


def overlap_candidates(pr, v, placement, fused, cuts, lists):
    """R32 neighbourhood: for every task X with a cross-device input whose device
    idles before it, the schedule with the nearest later task Y independent of
    X (Y's own F / B listed before X) moved in front of X. Returns lists of lists."""
    full, S, dur, dev, lp = _list_schedule(pr, v, placement, fused, cuts, lists)
    if lp is None:
        return []
    starts = lp[2]
    out = []
    for d in range(pr.p):
        lst = lists[d]
        where = {t: i for i, t in enumerate(lst)}
        for i, (k, s, j) in enumerate(lst):
            cross = (k == 0 and s > 0 and dev[s - 1] != d) or (k == 1 and s + 1 < S and dev[s + 1] != d)
            if not cross:
                continue
            prev_fin = 0 if i == 0 else starts[d][i - 1] + dur[lst[i - 1][0]][lst[i - 1][1]]
            if starts[d][i] <= prev_fin:
                continue  # no idle gap before X: its input was not waited for
            for q in range(i + 1, len(lst)):
                ky, sy, jy = lst[q]
                if ky > 0 and where[(ky - 1, sy, jy)] >= i:
                    continue  # Y's own predecessor is not listed before X
                new = [list(x) for x in lists]
                y = new[d].pop(q)
                new[d].insert(i, y)
                out.append(new)
                break
    return out


def tune_overlap(pr, v, placement, fused, cuts, lists, max_rounds=0):
    """Reading R32 ("avoid scheduling dependent computation tasks
    consecutively and instead delay certain computations to enable communication
    overlap"): per round, evaluate every R32 neighbour and accept the one with
    the largest total OverlapTime among those that keep the makespan and raise
    the overlap (ties: smaller makespan, then first); stop when none does.
    Returns (lists, swaps, accounting of the result)."""
    lists = [list(x) for x in lists]
    cur = comm_accounting_lists(pr, v, placement, fused, cuts, lists)
    swaps = 0
    total = sum(len(x) for x in lists)
    max_rounds = max_rounds if max_rounds > 0 else total
    while swaps < max_rounds and cur["status"] == 0:
        best = None
        for c, cand in enumerate(overlap_candidates(pr, v, placement, fused, cuts, lists)):
            r = comm_accounting_lists(pr, v, placement, fused, cuts, cand)
            if r["status"] != 0 or r["makespan"] > cur["makespan"]:
                continue
            ov = sum(r["overlap_d"])
            if ov <= sum(cur["overlap_d"]):
                continue
            key = (-ov, r["makespan"], c)
            if best is None or key < best[0]:
                best = (key, cand, r)
        if best is None:
            break
        lists, cur = best[1], best[2]
        swaps += 1
    return lists, swaps, cur


def memory_timeline(pr, v, placement, policy, cuts, lists=None):
    """Reading R35 (Eq. 2; "identifies potential OOM time";
    SPEC memory_timeline S:213-221): per device, the breakpoints (time, bytes)
    of M_d(t) = static + dynamic bytes in event order, starting at (0,
    static), with the R16 rules: act + stash allocated at an F's start, act
    freed at its B's end, stash at its W's end (at the B's end when fused);
    and the first time M_d exceeds the cap (-1: never). Times come from the
    event loop's trace (policy plans) or the longest-path starts of explicit
    lists (R30, policy 4 = LIST, 5 = LIST_FUSED). Plans that do not complete
    (STUCK) are not covered."""
    L, p = len(pr.t_f), pr.p
    full = list(cuts) if (cuts and cuts[0] == 0 and cuts[-1] == L) else [0] + list(cuts) + [L]
    S = len(full) - 1

    def ssum(col, s):
        return int(sum(int(x) for x in col[full[s]:full[s + 1]]))
    fused = policy in (0, 1, 5)
    dur = {0: [ssum(pr.t_f, s) for s in range(S)],
           1: [ssum(pr.t_b, s) + (ssum(pr.t_w, s) if fused else 0) for s in range(S)],
           2: [ssum(pr.t_w, s) for s in range(S)]}
    act = [ssum(pr.act, s) for s in range(S)]
    sta = [ssum(pr.stash, s) for s in range(S)]
    wg = [ssum(pr.weight, s) + ssum(pr.grad, s) for s in range(S)]
    dev = [device_of_stage(placement, p, v, s) for s in range(S)]
    if lists is None:
        r = simulate(pr, v, placement, policy, full[1:-1], trace=True)
        if r["status"] not in (0, 2):
            raise ValueError("plan does not complete (status %d)" % r["status"])
        per_dev = [[(k, s, st) for (k, s, _j, st) in r["trace"][d]] for d in range(p)]
    else:
        lp = longest_path(pr, v, placement, full[1:-1], fused, lists)
        if lp is None:
            raise ValueError("cyclic wait (stuck)")
        per_dev = [[(k, s, st) for (k, s, _j), st in zip(lists[d], lp[2][d])] for d in range(p)]
    points, first = [], []
    for d in range(p):
        b = sum(wg[s] for s in range(S) if dev[s] == d)
        pts = [(0, b)]
        fv = 0 if b > pr.cap else -1
        for (k, s, st) in per_dev[d]:
            if k == 0:
                t, b = st, b + act[s] + sta[s]
            elif k == 1:
                t, b = st + dur[1][s], b - act[s] - (sta[s] if fused else 0)
            else:
                t, b = st + dur[2][s], b - sta[s]
            pts.append((t, b))
            if fv < 0 and b > pr.cap:
                fv = t
        points.append(pts)
        first.append(fv)
    return {"points": points, "first_violation": first}
