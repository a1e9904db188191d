"""List GPU-vs-oracle mismatches for a config range (debugging aid)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2509_23722_b200 import adaptis as A, workloads as W  # noqa: E402
cid = int(sys.argv[1]); first = int(sys.argv[2]); count = int(sys.argv[3])
pr, sp = W.config(cid)
ctx = A.Context(0)
got = ctx.eval_batch(pr, sp, first, count)
want = O.eval_indices(pr, sp, range(first, first + count))
bad = [i for i in range(count) if got["status"][i] != want["status"][i] or got["makespan"][i] != want["makespan"][i]]
print("mismatches", len(bad), "of", count)
for i in bad[:40]:
    pl = A.decode(pr, sp, first + i)
    print(first + i, pl["v"], pl["placement"], pl["policy"], pl["cuts"], "gpu", got["status"][i], got["makespan"][i],
          "oracle", want["status"][i], want["makespan"][i])
