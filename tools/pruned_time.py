"""Time the exact-LB-pruned search (time to best plan) per config.

usage: python tools/pruned_time.py [cid ...]   (default 2 3 4 5)
Prints one JSON line per config: winner index/makespan, pruned and evaluated
counts, and the median of 3 timed searches after one warm-up (CUDA events on
the context stream).
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2509_23722_b200 import adaptis as A, workloads as W  # noqa: E402


def main():
    cids = [int(a) for a in sys.argv[1:]] or [2, 3, 4, 5]
    ctx = A.Context(0)
    ctx.set_prune(True)
    stream = torch.cuda.ExternalStream(ctx.stream)
    for cid in cids:
        pr, sp = W.config(cid)
        prep = ctx.prepare(pr, sp)
        best = prep.search()
        times = []
        for _ in range(3):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(stream)
            b = prep.search()
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1))
            assert b["index"] == best["index"]
        times.sort()
        print(json.dumps({"config": cid, "index": best["index"],
                          "makespan": best["makespan"],
                          "n_candidates": best["n_candidates"], "n_pruned": best["n_pruned"],
                          "n_evaluated": best["n_evaluated"], "ms": times[1]}), flush=True)


if __name__ == "__main__":
    main()
