"""Per-segment throughput and fallback counts of the CUDA path (diagnostics)."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2509_23722_b200 import adaptis as A  # noqa: E402
from paper_2509_23722_b200 import workloads as W  # noqa: E402

NAMES = {(1, 0): "SEQ-GPIPE", (1, 1): "SEQ-1F1B", (1, 2): "SEQ-ZB", (1, 3): "SEQ-GREEDY",
         (2, 0): "INT-GPIPE", (2, 1): "INT-1F1B", (2, 2): "INT-ZB", (2, 3): "INT-GREEDY",
         (2, 4): "WAVE-GPIPE", (2, 5): "WAVE-GREEDY"}

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--count", type=int, default=2_000_000)
ap.add_argument("--only", type=int, default=-1)
a = ap.parse_args()
pr, sp = W.config(a.config)
ctx = A.Context(0)
prep = ctx.prepare(pr, sp)
prep.eval(0, min(prep.N, 4096), device_out=True)  # load kernels, allocate scratch
base = 0
seg = 0
for g in sp.groups:
    P = A.space_size(pr, W.Space([g]))
    ncomb = bin(g.combo_mask).count("1")
    per = P // ncomb
    k = 0
    for combo in range(6):
        if not (g.combo_mask >> combo) & 1:
            continue
        if a.only < 0 or a.only == seg:
            n = min(per, a.count)
            first = base + k * per
            prep.eval(first, min(n, 1024), device_out=True)  # warm this kernel
            fb0 = ctx.fallback_count
            c0 = ctx.counters
            stream = torch.cuda.ExternalStream(ctx.stream)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            dts = []
            for rep in range(2):  # best of two: the first launch of a kernel can be slow
                if rep == 1:
                    c0 = ctx.counters
                torch.cuda.synchronize()
                e0.record(stream)
                r = prep.eval(first, n, device_out=True)
                e1.record(stream)
                e1.synchronize()
                dts.append(e0.elapsed_time(e1) / 1e3)
            dt = min(dts)
            st = torch.bincount(r["status"].long(), minlength=4).tolist()
            c1 = ctx.counters
            tk = c1["tasks"] - c0["tasks"]
            rd = c1["rounds"] - c0["rounds"]
            lv = c1["live_lane_rounds"] - c0["live_lane_rounds"]
            print(json.dumps({"seg": seg, "v": g.v, "combo": NAMES[(min(g.v, 2), combo)], "n": n,
                              "ms": round(dt * 1e3, 2), "Mcand_s": round(n / dt / 1e6, 2),
                              "status": st, "fallback": ctx.fallback_count - fb0,
                              "Gtask_s": round(tk / dt / 1e9, 2), "tasks_per_round": round(tk / max(rd, 1), 2),
                              "lane_util": round(tk / max(lv, 1), 3)}), flush=True)
        k += 1
        seg += 1
    base += P
