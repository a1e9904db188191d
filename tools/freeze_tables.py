"""Write tests/golden/tables_cfg{1..5}.json: the synthetic layer tables, caps and
search spaces of BASELINE.json's configs as produced by workloads.config().

Only the seeded input generator (paper_2509_23722_b200/workloads.py, which
holds none of the method's arithmetic) is called; tests/test_fixtures.py
checks that the generator still reproduces these files (SURVEY §8(d):
"freeze the generated tables as test fixtures").
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2509_23722_b200 import workloads as W  # noqa: E402

COLS = ("t_f", "t_b", "t_w", "act", "stash", "weight", "grad", "comm")


def table(cid):
    pr, sp = W.config(cid)
    return {"config": cid, "name": pr.name, "L": pr.L, "p": pr.p, "m": pr.m, "cap": pr.cap,
            "columns": {c: [int(x) for x in getattr(pr, c)] for c in COLS},
            "groups": [{"v": g.v, "part_mode": g.part_mode, "radius": g.radius,
                        "combo_mask": g.combo_mask} for g in sp.groups],
            "source": "tools/freeze_tables.py -> workloads.config(%d); jitter seed %d (SURVEY 8(d))"
                      % (cid, 1000 + cid)}


def main():
    for cid in range(1, 6):
        path = os.path.join(ROOT, "tests", "golden", "tables_cfg%d.json" % cid)
        with open(path, "w") as f:
            json.dump(table(cid), f, indent=1)
            f.write("\n")
        print(path)


if __name__ == "__main__":
    main()
