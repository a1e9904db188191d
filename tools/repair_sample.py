"""OOM repair (reading R31) as a policy variant on a sample of a
config's over-cap candidates: realise each candidate's policy order on the
GPU (adaptis_realize_lists), repair it (adaptis_repair_oom) and report how
many previously infeasible candidates become feasible, and whether a repaired
plan beats the config's exhaustive argmin (the oracle golden).

usage: python tools/repair_sample.py [cid ...] [--n N]
The sample: the first N over-cap candidates (status 2) of every ZB and ONEF1B
segment, in canonical order from the segment start, i.e. the L1-ball
neighbourhood of the Mist seed where the balanced, competitive partitions are.
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2509_23722_b200 import adaptis as A  # noqa: E402
from paper_2509_23722_b200 import workloads as W  # noqa: E402


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    n_per = int(sys.argv[sys.argv.index("--n") + 1]) if "--n" in sys.argv else 64
    cids = [int(a) for a in args if a.isdigit() and int(a) != n_per] or [3, 4]
    ctx = A.Context(0)
    for cid in cids:
        pr, sp = W.config(cid)
        prep = ctx.prepare(pr, sp)
        g = json.load(open(os.path.join(ROOT, "tests", "golden", "argmin_cfg%d.json" % cid)))
        base = 0
        sampled, fixed, moves, best = 0, 0, 0, None
        t0 = time.time()
        for grp in sp.groups:
            for k in range(6):
                if not (grp.combo_mask >> k) & 1:
                    continue
                one = W.Space([W.Group(grp.v, grp.part_mode, grp.radius, grp.seed_cuts, 1 << k)])
                try:
                    n_seg = A.space_size(pr, one)
                except A.AdaptisError:
                    continue
                plan0 = A.decode(pr, sp, base)
                if plan0["policy"] in (W.ZB, W.ONEF1B):
                    idx = np.arange(base, base + min(n_seg, 200_000), dtype=np.uint64)
                    ev = prep.eval_indices(idx)
                    over = idx[np.asarray(ev["status"]) == 2][:n_per]
                    for i in over:
                        plan = A.decode(pr, sp, int(i))
                        lists = prep.realize_lists(plan)
                        fused = plan["policy"] == W.ONEF1B
                        lp = dict(plan, policy=5 if fused else 4)
                        r = prep.repair_oom(lp, lists)
                        sampled += 1
                        moves += r["moves"]
                        if r["status"] == 0:
                            fixed += 1
                            if best is None or r["makespan"] < best[0]:
                                best = (r["makespan"], int(i))
                base += n_seg
        out = {"config": cid, "over_cap_sampled": sampled, "repaired_feasible": fixed,
               "moves": moves, "best_repaired": None if best is None else
               {"makespan": best[0], "index": best[1]},
               "exhaustive_argmin_makespan": g["makespan"],
               "argmin_moves": best is not None and best[0] < g["makespan"],
               "wall_s": round(time.time() - t0, 1)}
        print(json.dumps(out), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
