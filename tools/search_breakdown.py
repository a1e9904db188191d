"""Per-launch breakdown of one full (unpruned) search.

usage: python tools/search_breakdown.py [cid] [--prune]
Runs one warm-up search and one measured search, then prints every segment
launch (group, v, placement, policy, candidates, tasks, device ms, Gtask/s)
and the totals per (v, placement, policy).
"""
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_23722_b200 import adaptis as A, workloads as W  # noqa: E402

PL = {0: "SEQ", 1: "INT", 2: "WAVE"}
PO = {0: "GPIPE", 1: "1F1B", 2: "ZB", 3: "GREEDY"}


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    cid = int(args[0]) if args else 3
    ctx = A.Context(0)
    ctx.set_prune("--prune" in sys.argv)
    pr, sp = W.config(cid)
    prep = ctx.prepare(pr, sp)
    prep.search()
    best = prep.search()
    info = ctx.launch_info()
    agg = defaultdict(lambda: [0, 0, 0.0, 0])
    total = 0.0
    for li in info:
        key = (li["v"], PL.get(li["placement"]), PO.get(li["policy"]))
        a = agg[key]
        a[0] += li["candidates"]
        a[1] += li["tasks"]
        a[2] += li["ms"]
        a[3] += li["fallback"]
        total += li["ms"]
    print("config %d: %d launches, %.1f ms summed, kernel_ms %.1f, winner %d"
          % (cid, len(info), total, best["kernel_ms"], best["index"]))
    for key, (n, t, ms, fb) in sorted(agg.items(), key=lambda kv: -kv[1][2]):
        print("  v=%d %-4s %-6s cand %11d tasks %14d  %9.2f ms  %5.1f%%  %7.1f Gtask/s  %8.1f Mcand/s fb %d"
              % (key[0], key[1], key[2], n, t, ms, 100 * ms / total, t / ms / 1e6 if ms else 0,
                 n / ms / 1e3 if ms else 0, fb))


if __name__ == "__main__":
    main()
