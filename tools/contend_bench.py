"""Throughput of adaptis_eval_lists_contended (R34) on cfg3-shaped explicit
schedules: n random partitions of cfg3 (p = 8, m = 32, v = 2, interleaved
placement, split B/W), each with the GPipe-style list F(chunk 0) F(chunk 1)
B+W(chunk 1) B+W(chunk 0) per device. All plans share one task array (their
offsets point into it).

usage: python tools/contend_bench.py [n_plans] [reps] [comm_scale]
Prints one JSON line: plans/s and simulated tasks/s of the kernel (CUDA
events, median of `reps` after one warm-up), the whole call's wall time, and
how many plans were slowed by contention (makespan vs latency-only lists).
"""
import ctypes as C
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_23722_b200 import adaptis as A, workloads as W  # noqa: E402


def workload(n, comm_scale=1):
    """The problem, n plans (random cfg3 partitions, seed 3) and the per-device
    lists they share."""
    pr, sp = W.config(3, cap=W.INT64_MAX)  # GPipe order keeps all m in flight
    pr.comm = pr.comm * comm_scale         # > 1: a slower link, so transfers queue
    p, m, v, L = pr.p, pr.m, 2, len(pr.t_f)
    S = p * v
    rng = np.random.default_rng(3)
    plans = []
    for _ in range(n):
        cuts = np.sort(rng.choice(np.arange(1, L), S - 1, replace=False)).tolist()
        plans.append({"v": v, "placement": 1, "policy": 4, "S": S, "cuts": [0] + cuts + [L]})
    per_dev = []
    for d in range(p):
        lst = [(0, d, j) for j in range(m)] + [(0, d + p, j) for j in range(m)]
        for s in (d + p, d):
            for j in range(m):
                lst += [(1, s, j), (2, s, j)]
        per_dev.append(lst)
    return pr, sp, plans, per_dev


def run(n=32768, reps=5, comm_scale=1, ctx=None):
    pr, sp, plans, per_dev = workload(n, comm_scale)
    ctx = ctx or A.Context(0)
    prep = ctx.prepare(pr, sp)
    arr = A.make_plans(plans)
    flat = [t for lst in per_dev for t in lst]
    tasks = np.zeros(len(flat), dtype=[("kind", "<i2"), ("stage", "<i2"), ("mb", "<i4")])
    tasks["kind"] = [t[0] for t in flat]
    tasks["stage"] = [t[1] for t in flat]
    tasks["mb"] = [t[2] for t in flat]
    one = np.cumsum([0] + [len(x) for x in per_dev]).astype(np.uint64)
    offs = np.tile(one, n)
    out = A._host_results(n)
    soa = A._soa_from_numpy(out)

    def call(fn):
        A._check(fn(ctx.ptr, prep.ptr, arr, tasks.ctypes.data,
                    offs.ctypes.data_as(C.POINTER(C.c_uint64)), n, C.byref(soa), None), ctx.ptr)
        return ctx.launch_info()[0]["ms"] if fn is A.lib().adaptis_eval_lists_contended else None

    fn = A.lib().adaptis_eval_lists_contended
    call(fn)
    ms, wall = [], []
    for _ in range(reps):
        t0 = time.perf_counter()
        ms.append(call(fn))
        wall.append(time.perf_counter() - t0)
    mk_c = out["makespan"].copy()
    st_c = out["status"].copy()
    call(A.lib().adaptis_eval_lists)
    mk_u = out["makespan"].copy()
    ms.sort()
    wall.sort()
    ntask = n * len(flat)
    k = ms[len(ms) // 2]
    return {
        "tool": "contend_bench", "makespans_first": [int(x) for x in mk_c[:4]], "config": "cfg3 p=8 m=32 v=2 INTERLEAVED LIST", "comm_scale": comm_scale, "plans": n,
        "tasks_per_plan": len(flat), "kernel_ms": round(k, 3),
        "plans_per_s": round(n / (k / 1e3), 1), "tasks_per_s": round(ntask / (k / 1e3), 1),
        "call_wall_ms": round(wall[len(wall) // 2] * 1e3, 2),
        "ok": int((st_c == 0).sum()), "slowed_by_contention": int(((mk_c > mk_u) & (st_c == 0)).sum()),
        "median_slowdown": float(np.median(mk_c[st_c == 0] / mk_u[st_c == 0])) if (st_c == 0).any() else None}


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    comm_scale = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    print(json.dumps(run(n, reps, comm_scale)))


if __name__ == "__main__":
    main()
