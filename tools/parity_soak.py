"""Large-sample parity soak (evidence, not a test): seeded-uniform indices of
the BALL configs through adaptis_eval_indices (device decode + simulation)
compared element by element with the CPU oracle on the host's cores.

usage: python tools/parity_soak.py [--seed S] [cid:n ...]   (default 3:1000000 4:300000 5:100000;
n = all evaluates the whole space in index order)
Prints one JSON line per config."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2509_23722_b200 import adaptis as A, workloads as W  # noqa: E402


def main():
    argv = sys.argv[1:]
    seed = 12345
    if "--seed" in argv:
        i = argv.index("--seed")
        seed = int(argv[i + 1])
        argv = argv[:i] + argv[i + 2:]
    jobs = [a.split(":") for a in argv] or [["3", "1000000"], ["4", "300000"], ["5", "100000"]]
    ctx = A.Context(0)
    for cid, n in jobs:
        cid = int(cid)
        pr, sp = W.config(cid)
        N = O.space_size(pr, sp)
        if n == "all":
            n = N
            idx = np.arange(N, dtype=np.uint64)
        else:
            n = int(n)
            idx = np.random.default_rng(seed).integers(0, N, n).astype(np.uint64)
        prep = ctx.prepare(pr, sp)
        t = time.perf_counter()
        got = prep.eval_indices(idx)
        tg = time.perf_counter() - t
        t = time.perf_counter()
        want = O.eval_indices(pr, sp, idx)
        to = time.perf_counter() - t
        bad = {k: int(np.count_nonzero(np.asarray(got[k]) != np.asarray(want[k])))
               for k in ("status", "makespan", "peak_mem")}
        st = np.bincount(np.asarray(want["status"]), minlength=4).tolist()
        print(json.dumps({"config": cid, "indices": n, "seed": seed if n != N else None, "mismatches": bad,
                          "oracle_status_counts": st, "gpu_s": round(tg, 3), "oracle_s": round(to, 1),
                          "oracle_threads": os.cpu_count()}), flush=True)


if __name__ == "__main__":
    main()
