"""Smallest GPU reproduction: cfg1 exhaustive eval through the C ABI."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_23722_b200 import adaptis as A, workloads as W  # noqa: E402
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 1
pr, sp = W.config(cid)
ctx = A.Context(0)
r = ctx.eval_batch(pr, sp, 0, min(A.space_size(pr, sp), 4096))
print("ok", r["status"][:16], r["makespan"][:4])
