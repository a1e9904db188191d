"""oracle/executor.py — TEST INFRASTRUCTURE ONLY.

Executor lowering of an explicit schedule (AdaPtis §5 "Pipeline Executor",
P:563-581, Table `tab:instruction_types`), written out as
reading R33 of DESIGN.md fixes it. Shares no code with the library's
adaptis_lower (paper_2509_23722_b200/csrc/adaptis_executor.cu).

Instructions are tuples (op, stage, mb, peer). Ops follow Table 5:
  0 C_F, 1 C_B, 2 C_W (compute; stage = the task's stage, peer = -1),
  3 S_F, 4 S_B (send start), 5 R_F, 6 R_B (receive start),
  7 W_F, 8 W_B (wait receive); for comm ops `stage` is the boundary b between
  stages b and b+1, `mb` the micro-batch and `peer` the other device.

emit: per device, for each compute in schedule order: if it needs
  a cross-device input, R then W before it; the compute; if it produces a
  cross-device output, S right after it.
check ("S and R must be executed synchronously on both the data sender
  and receiver sides"): abstract run, compute and W proceed, an S and its R
  (same tag) proceed together when both devices are at them. Returns the
  blocked frontier (device -> instruction index) or None when all finish.
repair ("reorders them to ensure deadlock-free execution"): while
  blocked, take the lowest blocked device d that some blocked S of another
  device targets (with d's matching R later in d's program; smallest sender);
  move that R to just before d's blocked instruction.
hoist ("identify an earlier insertion point for R_B"): for each
  device and each R in program order, move it one instruction earlier while
  the instruction before it is not a receive from the same peer and the
  program stays deadlock-free; stop at the first step that fails.
"""
C_F, C_B, C_W, S_F, S_B, R_F, R_B, W_F, W_B = range(9)


def emit(p, S, dev, lists):
    prog = []
    for d in range(p):
        out = []
        for (k, s, j) in lists[d]:
            if k == 0 and s > 0 and dev[s - 1] != d:
                out += [(R_F, s - 1, j, dev[s - 1]), (W_F, s - 1, j, dev[s - 1])]
            if k == 1 and s + 1 < S and dev[s + 1] != d:
                out += [(R_B, s, j, dev[s + 1]), (W_B, s, j, dev[s + 1])]
            out.append((k, s, j, -1))
            if k == 0 and s + 1 < S and dev[s + 1] != d:
                out.append((S_F, s, j, dev[s + 1]))
            if k == 1 and s > 0 and dev[s - 1] != d:
                out.append((S_B, s - 1, j, dev[s - 1]))
        prog.append(out)
    return prog


def _partner(ins, d):
    op, b, j, peer = ins
    if op in (S_F, S_B):
        return peer, (op + 2, b, j, d)   # the receive on the peer
    return peer, (op - 2, b, j, d)       # R_F -> S_F, R_B -> S_B


def check(prog):
    p = len(prog)
    pc = [0] * p
    while True:
        moved = False
        for d in range(p):
            while pc[d] < len(prog[d]):
                ins = prog[d][pc[d]]
                op = ins[0]
                if op in (S_F, S_B, R_F, R_B):
                    e, want = _partner(ins, d)
                    if pc[e] < len(prog[e]) and prog[e][pc[e]] == want:
                        pc[d] += 1
                        pc[e] += 1
                        moved = True
                        continue
                    break
                pc[d] += 1
                moved = True
        if all(pc[d] == len(prog[d]) for d in range(p)):
            return None
        if not moved:
            return pc


def repair(prog, cap=None):
    prog = [list(x) for x in prog]
    n = 0
    cap = cap if cap is not None else sum(len(x) for x in prog) ** 2
    while True:
        pc = check(prog)
        if pc is None:
            return prog, n
        if n >= cap:
            raise RuntimeError("repair failed")
        p = len(prog)
        fix = None
        for d in range(p):
            if pc[d] >= len(prog[d]):
                continue
            for c in range(p):
                if c == d or pc[c] >= len(prog[c]):
                    continue
                ins = prog[c][pc[c]]
                if ins[0] in (S_F, S_B) and ins[3] == d:
                    want = (ins[0] + 2, ins[1], ins[2], c)
                    if want in prog[d][pc[d] + 1:]:
                        fix = (d, want)
                        break
            if fix:
                break
        if fix is None:
            raise RuntimeError("repair failed: no blocked send to hoist against")
        d, want = fix
        i = prog[d].index(want)
        prog[d].insert(pc[d], prog[d].pop(i))
        n += 1


def hoist(prog):
    prog = [list(x) for x in prog]
    n = 0
    for d in range(len(prog)):
        for ins in [x for x in prog[d] if x[0] in (R_F, R_B)]:
            while True:
                i = prog[d].index(ins)
                if i == 0:
                    break
                prev = prog[d][i - 1]
                if prev[0] in (R_F, R_B) and prev[3] == ins[3]:
                    break
                prog[d][i - 1], prog[d][i] = prog[d][i], prog[d][i - 1]
                if check(prog) is not None:
                    prog[d][i - 1], prog[d][i] = prog[d][i], prog[d][i - 1]
                    break
                n += 1
    return prog, n


def lower(p, S, dev, lists, do_repair=True, do_hoist=True):
    prog = emit(p, S, dev, lists)
    nr = nh = 0
    if do_repair:
        prog, nr = repair(prog)
    if do_hoist:
        prog, nh = hoist(prog)
    return prog, nr, nh
