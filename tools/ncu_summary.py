"""Summarise an ncu report: key metrics, stall reasons, and SASS hot spots."""
import csv
import subprocess
import sys
from collections import Counter

KEYS = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_issued.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio",
        "sm__warps_active.avg.per_cycle_active", "smsp__warps_eligible.avg.per_cycle_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "launch__grid_size",
        "launch__shared_mem_per_block_dynamic", "smsp__inst_executed.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]


def raw(rep, row=0):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u, v = rows[0], rows[1], rows[2 + row]
    return {h[i]: (v[i], u[i]) for i in range(len(h))}


def n_kernels(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    return max(0, len(list(csv.reader(out.splitlines()))) - 2)


def main(rep, row=0):
    m = raw(rep, row)
    for k in ("Kernel Name", "Block Size", "Grid Size"):
        if k in m:
            print("%-60s %s" % (k, m[k][0]))
    for k in KEYS:
        if k in m:
            print("%-60s %s %s" % (k, m[k][0], m[k][1]))
    stalls = sorted(((float(v[0]), k) for k, v in m.items()
                     if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("per_issue_active.ratio")
                     and v[0] not in ("", "n/a")), reverse=True)[:8]
    print("top stalls (warps per issue):", ", ".join("%s=%.2f" % (k.split("stalled_")[1].split("_per")[0], v)
                                                  for v, k in stalls))
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[1]
    ia, isrc = h.index("Instructions Executed"), h.index("Source")
    c = Counter()
    tot = 0
    for r in rows[2:]:
        try:
            n = int(r[ia])
        except (ValueError, IndexError):
            continue
        op = r[isrc].split()
        if not op:
            continue
        o = op[1] if op[0].startswith("@") and len(op) > 1 else op[0]
        c[o.split(".")[0]] += n
        tot += n
    print("opcode mix:", ", ".join("%s %.1f%%" % (k, 100 * v / tot) for k, v in c.most_common(14)))


if __name__ == "__main__":
    # one summary per captured kernel (the opcode mix is the report's, all kernels)
    for r in sys.argv[1:]:
        for k in range(max(1, n_kernels(r))):
            print("==", r, "kernel", k)
            main(r, k)
