"""Oracle-only exhaustive argmin goldens (Eq. 1-2; reading R18).

Runs the C oracle's exact LB-pruned exhaustive search (`oracle.search`,
SURVEY §8(c) "Search / argmin: cfg3-5 exact LB-pruned exhaustive") on a
config's frozen tables and writes tests/golden/argmin_cfg<N>[_<tag>].json.
This script imports ONLY oracle/ and the seeded input generator
(workloads.py, which holds no arithmetic of the method): no value here comes
from the CUDA path.

usage: python tools/oracle_argmin.py CID [--threads T] [--group G --combo K]
  --group/--combo restrict the space to one (v-group, combo) segment: the
  other groups are dropped and the group's combo_mask keeps only bit K.  The
  golden then records the segment-local index and the offset of that segment
  in the full space (so the GPU's full-space index = offset + local index).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402
from paper_2509_23722_b200 import workloads as W  # noqa: E402  (input generator only)


def segment_space(sp, g, k):
    """The one-segment sub-space (group g, combo k) and its offset in sp."""
    import copy
    sub = copy.deepcopy(sp)
    grp = sub.groups[g]
    grp.combo_mask = 1 << k
    sub.groups = [grp]
    # offset: sizes of the earlier groups, plus the earlier enabled combos of g
    off = 0
    for gi in range(g):
        pre = copy.deepcopy(sp)
        pre.groups = [sp.groups[gi]]
        off += O.space_size(pr_global, pre)
    for kk in range(k):
        if (sp.groups[g].combo_mask >> kk) & 1 and O.combo(sp.groups[g].v, kk) is not None:
            one = copy.deepcopy(sp)
            one.groups = [copy.deepcopy(sp.groups[g])]
            one.groups[0].combo_mask = 1 << kk
            off += O.space_size(pr_global, one)
    return sub, off


def main():
    global pr_global
    ap = argparse.ArgumentParser()
    ap.add_argument("cid", type=int)
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--group", type=int, default=None)
    ap.add_argument("--combo", type=int, default=None)
    a = ap.parse_args()
    pr, sp = W.config(a.cid)
    pr_global = pr
    O.build()
    tag, off = "", 0
    if a.group is not None:
        sp, off = segment_space(sp, a.group, a.combo)
        tag = f"_g{a.group}k{a.combo}"
    t0 = time.time()
    b = O.search(pr, sp, prune=True, nthreads=a.threads)
    wall = time.time() - t0
    try:
        head = subprocess.check_output(["git", "-C", ROOT, "rev-parse", "--short=12", "HEAD"],
                                       text=True).strip()
    except Exception:  # noqa: BLE001
        head = "unknown"
    out = {
        "config": a.cid,
        "segment": None if a.group is None else {"group": a.group, "combo": a.combo,
                                                 "offset": off},
        "index": b["index"], "global_index": None if b["index"] == O.UINT64_MAX else off + b["index"],
        "makespan": b["makespan"], "plan": b["plan"],
        "n_total": b["n_total"], "n_invalid": b["n_invalid"],
        "n_valid": b["n_total"] - b["n_invalid"],
        "n_simulated": b["n_simulated"], "n_feasible_simulated": b["n_feasible"],
        "provenance": {
            "script": "tools/oracle_argmin.py", "oracle": "oracle/oracle.c orc_search(prune=1)",
            "inputs": f"workloads.config({a.cid}) (== tests/golden/tables_cfg{a.cid}.json)",
            "threads": a.threads, "wall_s": round(wall, 1), "git_head": head,
            "host_cores": os.cpu_count(),
            "note": "exact LB-pruned exhaustive search: a candidate is skipped only if its "
                    "busiest-device work exceeds the incumbent makespan (LB <= makespan) or "
                    "its fixed order exceeds the memory cap (R16); n_simulated depends on "
                    "thread timing, the winner does not",
        },
    }
    path = os.path.join(ROOT, "tests", "golden", f"argmin_cfg{a.cid}{tag}.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
