"""Pruned vs unpruned search on the configs: same winner, and how much the
exact lower-bound prune removes. usage: python tools/prune_check.py [cid ...]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_23722_b200 import adaptis as A, workloads as W  # noqa: E402

for cid in [int(a) for a in sys.argv[1:]] or [2, 3, 4]:
    pr, sp = W.config(cid)
    ctx = A.Context(0)
    t = time.perf_counter(); a = ctx.search(pr, sp); ta = time.perf_counter() - t
    ctx.set_prune(True)
    b = ctx.search(pr, sp)
    t = time.perf_counter(); b = ctx.search(pr, sp); tb = time.perf_counter() - t
    print(json.dumps({"config": cid, "same_winner": (a["index"], a["makespan"]) == (b["index"], b["makespan"]),
                      "index": a["index"], "makespan": a["makespan"], "unpruned_s": round(ta, 3),
                      "pruned_s": round(tb, 4), "n_candidates": b["n_candidates"], "n_pruned": b["n_pruned"],
                      "n_evaluated": b["n_evaluated"]}), flush=True)
    ctx.close()
