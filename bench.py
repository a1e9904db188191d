#!/usr/bin/env python
"""Benchmark of the AdaPtis hot path: candidate pipeline strategies simulated
per second (and time-to-best-plan) for one full search over a BASELINE.json
config, on N GPUs of one node (one process per GPU, torchrun for N > 1).

  python bench.py --gpus N --steps K --warmup W [--config 5] [--impl adaptis|reference]

A step = one adaptis_search over the whole candidate space (all §8(a) rows:
decode, stage/device aggregation, memory check, simulation, argmin, the
cross-GPU allreduce-min and the winner report). `value` counts valid
candidates (status != invalid-decode) per second over the device-timed steps
with the tables already resident in HBM; `e2e` repeats the step through
adaptis_search with host inputs (validation, H2D of the tables, D2H of the
result). `--impl reference` times the CPU oracle (oracle/) on a bounded sample
of the same workload on this host's cores.
"""
import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "candidate pipeline strategies simulated/sec"
UNIT = "candidates/s"
ALG_INSTR_PER_TASK = 16      # ~16 SASS lane-instructions per simulated task (int64)
CONFIG_NAMES = {
    1: "cfg1: 8-layer heterogeneous toy, p=2, m=4, exhaustive",
    2: "cfg2: Llama-style 32 dense + heavy emb/head, p=4, m=16, I-1F1B v=2",
    3: "cfg3: DeepSeek-style 61 dense+MoE, p=8, m=32, joint search",
    4: "cfg4: Nemotron-H-style 52 Mamba/attn, p=8, v=2, m=64, cap 180 GB",
    5: "cfg5: 128-layer heterogeneous sweep, p=16, v<=4, m=128, ~1e9 candidates",
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--impl", default="adaptis", choices=["adaptis", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--cfg5-steps", type=int, default=1,
                    help="timed steps of the cfg5 leg (the 8-GPU target config); 0 disables it")
    return ap.parse_args()


def spawn_ranks(args):
    """`bench.py --gpus N` without a torchrun environment: re-launch this
    script under torch.distributed.run with N ranks (one process per GPU, NCCL,
    127.0.0.1 rendezvous); rank 0 prints the JSON line."""
    import socket
    import subprocess
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           "--nproc-per-node=%d" % args.gpus, "--master-addr", "127.0.0.1",
           "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    # exactly one line on stdout: rank 0's JSON; anything else the ranks print goes to stderr
    proc = subprocess.Popen(cmd, stdout=subprocess.PIPE, text=True)
    for line in proc.stdout:
        (sys.stdout if line.startswith("{") else sys.stderr).write(line)
        sys.stdout.flush()
    return proc.wait()


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi style clocks + throttle reasons sampled during the timed region (NVML)."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            self._stop.wait(0.1)

    def start(self):
        if self.nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join()
        import statistics
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ------------------------------------------------------------------ reference arm
def cpu_oracle_rate(pr, sp, seconds, seed=2025):
    """The oracle, as it stands, on a bounded random sample of the workload."""
    import numpy as np
    from oracle import oracle as O
    N = O.space_size(pr, sp)
    nth = os.cpu_count() or 1
    rng = np.random.default_rng(seed)
    # calibrate the sample size on a small probe, then run ~`seconds` of work
    probe = rng.integers(0, N, max(8, nth))
    t = time.perf_counter()
    O.eval_indices(pr, sp, probe, nthreads=nth)
    dt = max(time.perf_counter() - t, 1e-4)
    n = int(max(nth, min(2_000_000, len(probe) * seconds / dt)))
    idx = rng.integers(0, N, n)
    t = time.perf_counter()
    ev = O.eval_indices(pr, sp, idx, nthreads=nth)
    dt = time.perf_counter() - t
    valid = int((ev["status"] != 1).sum())
    # single-thread rate of the same oracle on a quarter-length prefix of the sample
    n1 = max(8, int(n / nth / 4))
    t = time.perf_counter()
    ev1 = O.eval_indices(pr, sp, idx[:n1], nthreads=1)
    dt1 = time.perf_counter() - t
    valid1 = int((ev1["status"] != 1).sum())
    return {"value": valid / dt, "unit": UNIT, "cores": nth, "kind": "oracle",
            "value_1thread": valid1 / dt1,
            "sample": "%d uniformly random candidates of %s (%d valid), event-loop oracle, %.1f s on "
                      "%d threads; 1-thread rate on the first %d of them (%.1f s)"
                      % (n, pr.name, valid, dt, nth, n1, dt1)}, n, dt


def contention_cpu_rate(contend_bench, gpu, seconds=5.0):
    """The R34 oracle (oracle/contention.py, pure Python, one core) on the first
    plans of the same contention workload: plans/s, and its makespans must equal
    the GPU's for those plans."""
    from oracle.contention import simulate_lists_contended
    pr, _sp, plans, per_dev = contend_bench.workload(64, gpu["comm_scale"])
    t0 = time.perf_counter()
    k = 0
    ms = []
    while k < len(plans) and (time.perf_counter() - t0 < seconds or k < 4):
        pl = plans[k]
        r = simulate_lists_contended(pr, pl["v"], pl["placement"], False, pl["cuts"][1:-1], per_dev)
        ms.append(r["makespan"])
        k += 1
    dt = time.perf_counter() - t0
    return {"value": k / dt, "unit": "plans/s", "cores": 1, "kind": "oracle",
            "sample": "first %d plans of the same workload" % k,
            "makespans_match_gpu": ms[:4] == gpu["makespans_first"][:4]}


def run_reference(args, rank, world):
    if rank != 0:
        return
    from paper_2509_23722_b200 import workloads as W
    pr, sp = W.config(args.config)
    per_step = max(2.0, min(20.0, 120.0 / max(1, args.steps + args.warmup)))
    for _ in range(args.warmup):
        cpu_oracle_rate(pr, sp, per_step / 4)
    vals, tot_t, tot_n = [], 0.0, 0
    info = None
    for _ in range(args.steps):
        info, n, dt = cpu_oracle_rate(pr, sp, per_step)
        vals.append(info["value"])
        tot_t += dt
        tot_n += n
    value = sum(vals) / len(vals)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000 * tot_t / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "config": {"workload": CONFIG_NAMES[args.config], "config_id": args.config,
                       "sample_per_step": "bounded random sample (see cpu_baseline)"},
            "cpu_baseline": info,
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm
def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    if world != args.gpus:
        raise SystemExit("bench.py: --gpus %d but WORLD_SIZE=%d" % (args.gpus, world))
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2509_23722_b200 import adaptis as A
    from paper_2509_23722_b200 import workloads as W

    torch.cuda.set_device(local)
    group = None
    # NCCL's own messages (e.g. the NCCL_DEBUG=VERSION banner) go to stderr, so that
    # rank 0's stdout carries exactly the one JSON line of the contract
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        group = dist.group.WORLD
    pr, sp = W.config(args.config)
    ctx = A.Context(local, rank=rank, world=world, group=group)
    prep = ctx.prepare(pr, sp)
    N = prep.N
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda:%d" % local)  # > 126 MB L2
    stream = torch.cuda.ExternalStream(ctx.stream, device=local)

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])
        torch.cuda.synchronize(local)

    for _ in range(args.warmup):
        best = prep.search()
    barrier()
    clocks = ClockSampler(local)
    clocks.start()
    step_ms, kern_ms = [], []
    launches0 = ctx.launch_count
    n_invalid = 0
    seg_ms, seg_tasks, seg_n = {}, {}, {}
    for _ in range(args.steps):
        flush.random_(0, 255)  # L2 flush between timed iterations (outside the timed region)
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        best = prep.search()
        e1.record(stream)
        e1.synchronize()
        step_ms.append(e0.elapsed_time(e1))
        kern_ms.append(best["kernel_ms"])
        n_invalid = best["n_invalid"]
        for li in ctx.launch_info():
            k = (li["v"], li["placement"], li["policy"], li["kernel"])
            seg_ms[k] = seg_ms.get(k, 0.0) + li["ms"]
            seg_tasks[k] = seg_tasks.get(k, 0) + li["tasks"]
            seg_n[k] = seg_n.get(k, 0) + 1
    barrier()
    clk = clocks.stop()
    launches = ctx.launch_count - launches0
    tot = torch.tensor([sum(step_ms), sum(kern_ms)], dtype=torch.float64, device="cuda:%d" % local)
    inv = torch.tensor([n_invalid], dtype=torch.int64, device="cuda:%d" % local)
    per_rank = tot.clone().reshape(1, 2)
    if world > 1:
        per_rank = torch.zeros(world, 2, dtype=torch.float64, device="cuda:%d" % local)
        dist.all_gather_into_tensor(per_rank, tot.reshape(1, 2))
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
        dist.all_reduce(inv, op=dist.ReduceOp.SUM)
    total_ms, total_kern_ms = float(tot[0]), float(tot[1])
    # per-rank device time of the timed steps (shard balance, §8e)
    rank_ms = [float(x) / args.steps for x in per_rank[:, 1].tolist()]
    valid = N - int(inv.item())

    # ---- time-to-best-plan with the exact lower-bound prune (same winner; the
    # simulated/s metric above keeps pruning off)
    ctx.set_prune(True)
    prep.search()
    pr_ms = []
    bp = None
    for _ in range(max(1, min(args.steps, 3))):
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        bp = prep.search()
        e1.record(stream)
        e1.synchronize()
        pr_ms.append(e0.elapsed_time(e1))
        assert bp["index"] == best["index"]
    ctx.set_prune(False)
    tp = torch.tensor([sum(pr_ms) / len(pr_ms)], dtype=torch.float64, device="cuda:%d" % local)
    if world > 1:
        dist.all_reduce(tp, op=dist.ReduceOp.MAX)
    pruned_ms = float(tp.item())

    # ---- e2e through the public call with host inputs (validation + H2D + D2H)
    e2e_ms = []
    for _ in range(max(1, min(args.steps, 3))):
        barrier()
        t = time.perf_counter()
        b2 = ctx.search(pr, sp)
        e2e_ms.append(1000 * (time.perf_counter() - t))
        assert b2["index"] == best["index"]
    e2 = torch.tensor([sum(e2e_ms) / len(e2e_ms)], dtype=torch.float64, device="cuda:%d" % local)
    if world > 1:
        dist.all_reduce(e2, op=dist.ReduceOp.MAX)
    e2e_ms_step = float(e2.item())
    h2d = 8 * (6 * pr.L + pr.L) + 8 * 160 * 65 + 8 * 4 * 64 * 257 + 2 * 4 * 64 + 8 * (2 + 4 * 16)
    d2h = 8 * (2 + 2 * 16) + 8 + 8 + 4 + 1 + 8 * 3 * pr.p

    # ---- cfg5 leg: the config BASELINE quotes the 8-GPU target on (949.9 M
    # candidates, p = 16, v <= 4, m = 128); same step definition, device-timed,
    # max over ranks, one warm-up step (a step is tens of seconds on one GPU)
    cfg5 = None
    if args.config != 5 and args.cfg5_steps > 0:
        pr5, sp5 = W.config(5)
        prep5 = ctx.prepare(pr5, sp5)
        b5 = prep5.search()  # warm-up
        ms5, k5 = [], []
        for _ in range(args.cfg5_steps):
            flush.random_(0, 255)
            barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            b5 = prep5.search()
            e1.record(stream)
            e1.synchronize()
            ms5.append(e0.elapsed_time(e1))
            k5.append(b5["kernel_ms"])
        t5 = torch.tensor([sum(ms5) / len(ms5), sum(k5) / len(k5)], dtype=torch.float64,
                          device="cuda:%d" % local)
        pr5_rank = t5.clone().reshape(1, 2)
        i5 = torch.tensor([b5["n_invalid"]], dtype=torch.int64, device="cuda:%d" % local)
        if world > 1:
            pr5_rank = torch.zeros(world, 2, dtype=torch.float64, device="cuda:%d" % local)
            dist.all_gather_into_tensor(pr5_rank, t5.reshape(1, 2))
            dist.all_reduce(t5, op=dist.ReduceOp.MAX)
            dist.all_reduce(i5, op=dist.ReduceOp.SUM)
        ctx.set_prune(True)
        prep5.search()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        bp5 = prep5.search()
        e1.record(stream)
        e1.synchronize()
        ctx.set_prune(False)
        tp5 = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda:%d" % local)
        if world > 1:
            dist.all_reduce(tp5, op=dist.ReduceOp.MAX)
        valid5 = prep5.N - int(i5.item())
        ms_step5 = float(t5[0])
        g5 = _golden(5)
        cfg5 = {"workload": CONFIG_NAMES[5], "steps": args.cfg5_steps, "warmup": 1,
                "candidates": prep5.N, "valid_candidates": valid5,
                "value": valid5 / (ms_step5 / 1000.0), "unit": UNIT, "ms_per_step": ms_step5,
                "time_to_best_plan_pruned_ms": float(tp5.item()),
                "per_rank_kernel_ms": [float(x) for x in pr5_rank[:, 1].tolist()],
                "best": {"index": b5["index"], "makespan_ticks": b5["makespan"], "plan": b5["plan"]},
                "same_winner_pruned": bp5["index"] == b5["index"],
                "matches_oracle_golden": None if g5 is None else
                (b5["index"], b5["makespan"]) == (g5["index"], g5["makespan"])}
        prep5.close()

    # ---- the paper's own search (Pipeline Generator, R28) on this GPU:
    # seeds + phase-by-phase tuning, every neighbourhood evaluated by the kernels
    gen = None
    if rank == 0:
        ctx.generate(pr)  # warm
        t = time.perf_counter()
        g = ctx.generate(pr)
        gen_ms = 1000 * (time.perf_counter() - t)
        gen = {"wall_ms": gen_ms, "kernel_ms": g["kernel_ms"], "makespan_ticks": g["makespan"],
               "plan": g["plan"], "plans_evaluated": g["n_evaluated"], "rounds": g["rounds"],
               "steps": g["steps"],
               "makespan_vs_exhaustive": g["makespan"] / best["makespan"] - 1.0,
               "note": "generator explores v in {1,2} x every R12 combo from the P:346 seeds; "
                       "the exhaustive search explores this config's enumerated space"}

    if rank == 0:
        ms_step = total_ms / args.steps
        value = valid / (ms_step / 1000.0)
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "int32" if not _int64(pr) else "int64", "data": "synthetic",
                "config": {"workload": CONFIG_NAMES[args.config], "config_id": args.config,
                           "candidates": N, "valid_candidates": valid,
                           "time_to_best_plan_ms": ms_step,
                           "time_to_best_plan_pruned_ms": pruned_ms,
                           "pruned_candidates": bp["n_pruned"],
                           "parallelism": "candidates%d" % world,
                           "l2": "flushed (256 MiB write) between timed steps"},
                "best": {"index": best["index"], "makespan_ticks": best["makespan"],
                         "plan": best["plan"], "bubble": best["bubble"],
                         "peak_mem_bytes": best["peak_mem"],
                         # Alg. 1 Step 3 per device (R29): T_d = busy + comm + bubble - overlap
                         "T_d": best["T_d"], "busy_d": best["busy_d"], "comm_d": best["comm_d"],
                         "overlap_d": best["overlap_d"], "bubble_d": best["bubble_d"]},
                "e2e": {"value": valid / (e2e_ms_step / 1000.0), "unit": UNIT,
                        "ms_per_step": e2e_ms_step, "h2d_bytes_per_step": h2d,
                        "d2h_bytes_per_step": d2h},
                "gpu_launches": launches,
                "kernel_ms_per_step": total_kern_ms / args.steps,
                "per_rank_kernel_ms": rank_ms,
                "rank_imbalance": (max(rank_ms) / (sum(rank_ms) / len(rank_ms)) - 1.0) if rank_ms else 0.0,
                "clocks": clk}
        line["roofline"] = roofline(seg_ms, seg_tasks, seg_n, args.config)
        g = _golden(args.config)
        line["best"]["matches_oracle_golden"] = None if g is None else \
            (best["index"], best["makespan"]) == (g["index"], g["makespan"])
        line["cfg5"] = cfg5
        line["generator"] = gen
        # §8(f) f1 / R36: the whole cfg2 space searched with every candidate's realised
        # order executed under send/receive-engine contention (one GPU)
        if world == 1:
            try:
                pr2, sp2 = W.config(2)
                prep2 = ctx.prepare(pr2, sp2)
                prep2.search_contended()  # warm
                t = time.perf_counter()
                bc = prep2.search_contended()
                wall = 1000 * (time.perf_counter() - t)
                bl = prep2.search()
                line["contended_search"] = {
                    "workload": CONFIG_NAMES[2], "candidates": prep2.N, "wall_ms": wall,
                    "kernel_ms": bc["kernel_ms"], "tasks": bc["n_tasks"],
                    "winner": {"index": bc["index"], "makespan_ticks": bc["makespan"], "plan": bc["plan"]},
                    "latency_only_winner": {"index": bl["index"], "makespan_ticks": bl["makespan"]},
                    "note": "R36: policy order realised with pure latency, then executed under FIFO "
                            "send/receive engines (R34); single GPU"}
                prep2.close()
            except Exception as e:  # reported, never silently replaced
                line["contended_search"] = {"error": repr(e)}
        # §8(f) f1 / R34: explicit cfg3-shaped schedules under send/receive-engine
        # contention (adaptis_eval_lists_contended), latencies x100 so transfers queue
        try:
            sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "tools"))
            import contend_bench
            line["contention"] = contend_bench.run(n=8192, reps=3, comm_scale=100, ctx=ctx)
            if not args.no_cpu_baseline and world == 1:
                line["contention"]["cpu_baseline"] = contention_cpu_rate(contend_bench, line["contention"])
        except Exception as e:  # reported, never silently replaced
            line["contention"] = {"error": repr(e)}
        if not args.no_cpu_baseline and world == 1:
            info, _, _ = cpu_oracle_rate(pr, sp, args.cpu_seconds)
            line["cpu_baseline"] = info
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier(device_ids=[local])
        dist.destroy_process_group()


def _golden(cid):
    """The oracle's exhaustive argmin of a config (tests/golden/argmin_cfgN.json,
    written by tools/oracle_argmin.py from oracle/ only), or None."""
    try:
        with open(os.path.join(ROOT, "tests", "golden", "argmin_cfg%d.json" % cid)) as f:
            return json.load(f)
    except Exception:  # noqa: BLE001
        return None


def _int64(pr):
    import numpy as np
    U = pr.m * (int(np.sum(pr.t_f + pr.t_b + pr.t_w)) + 2 * int(np.sum(pr.comm[:-1])))
    return U >= (1 << 31) - 1


POLICY = {0: "GPIPE", 1: "ONEF1B", 2: "ZB", 3: "GREEDY"}
PLACEMENT = {0: "SEQ", 1: "INT", 2: "WAVE"}


TRAFFIC_FILE = os.path.join(ROOT, "profiles", "r2_dominant_traffic.json")


def measured_traffic(config_id, kernel):
    """DRAM bytes per launch of the dominant kernel from the committed ncu --set
    full capture (profiles/r2_dominant_traffic.json), when it is this config's
    same kernel; None otherwise (the contract's null)."""
    try:
        t = json.load(open(TRAFFIC_FILE))
    except Exception:  # noqa: BLE001
        return None
    k = t.get("kernels", {}).get(kernel)
    if t.get("config_id") != config_id or k is None:
        return None
    return int(k["dram_read_bytes"]) + int(k["dram_write_bytes"])


def roofline(seg_ms, seg_tasks, seg_n, config_id=None):
    """Issue-rate roofline of the dominant kernel: ALU/issue
    bound, no tensor cores, HBM traffic negligible. achieved = algorithmic
    lane-instructions per launch (16 per simulated F/B/W task)
    / the launch's CUDA-event duration; peak = 148 SMs x 4 schedulers x 32
    lanes x the measured max SM clock (MEASURED_PEAKS.json sm_max_mhz)."""
    try:
        mhz = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["sm_max_mhz"])
        basis = "measured sm_max_mhz"
    except Exception:  # noqa: BLE001
        mhz, basis = 1965.0, "fallback 1965 MHz"
    peak = 148 * 4 * 32 * mhz * 1e6 / 1e12
    out = {"bound": "alu", "unit": "Tinstr/s", "peak": peak, "traffic": None,
           "peak_basis": "148 SM x 4 SMSP x 32 lanes x %.0f MHz (%s)" % (mhz, basis)}
    if not seg_ms:
        out.update(achieved=None, frac=None)
        return out
    k = max(seg_ms, key=seg_ms.get)
    per_launch_ms = seg_ms[k] / seg_n[k]
    tasks = seg_tasks[k] / seg_n[k]
    ach = ALG_INSTR_PER_TASK * tasks / (per_launch_ms / 1e3) / 1e12
    tot_ms, tot_tasks = sum(seg_ms.values()), sum(seg_tasks.values())
    allk = ALG_INSTR_PER_TASK * tot_tasks / (tot_ms / 1e3) / 1e12
    name = "seqg_kernel<v=%d, %s>" % (k[0], PLACEMENT[k[1]]) if k[3] == 1 else \
        "fixed_kernel<%s, v=%d> (%s placement)" % (POLICY[k[2]], k[0], PLACEMENT[k[1]]) if k[3] == 2 else \
        "seg_kernel<%s, v=%d> (%s placement)" % (POLICY[k[2]], k[0], PLACEMENT[k[1]])
    out.update(achieved=ach, frac=ach / peak, kernel=name,
               kernel_share_of_step=seg_ms[k] / tot_ms, tasks_per_launch=tasks,
               launch_ms=per_launch_ms, all_kernels_achieved=allk, all_kernels_frac=allk / peak,
               note="algorithmic work = 16 SASS lane-instr per simulated task (int64 form, SURVEY §8d)")
    out["traffic"] = measured_traffic(config_id, out["kernel"])
    if out["traffic"] is not None:
        out["traffic_note"] = ("dram read+write bytes per launch, ncu --set full "
                               "(profiles/r2_dominant_traffic.json); algorithmic bytes are ~0 "
                               "(ALU bound: inputs L2/smem-resident, search writes 8 B per warp)")
    return out


if __name__ == "__main__":
    main()
