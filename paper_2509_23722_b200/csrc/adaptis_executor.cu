// adaptis_executor.cu — executor lowering of an explicit schedule (AdaPtis §5
// "Pipeline Executor", Table `tab:instruction_types`; reading R33):
// the per-device instruction programs of Table 5, the rendezvous deadlock
// check, deadlock repair by hoisting receives, and receive hoisting for
// overlap. Host code only ("not data-parallel, so CPU only").
#include <cstring>
#include <string>
#include <vector>

#include "adaptis_internal.h"

namespace {

thread_local std::string g_exec_error;

adaptis_status exec_fail(const std::string& msg) {
  g_exec_error = msg;
  return ADAPTIS_EINVAL;
}

int dev_of_stage(int placement, int p, int s) {  // R12
  if (placement == ADAPTIS_SEQ) return s;
  if (placement == ADAPTIS_INTERLEAVED) return s % p;
  const int c = s / p, j = s - c * p;
  return (c & 1) ? p - 1 - j : j;
}

bool is_comm(int op) { return op >= ADAPTIS_OP_S_F && op <= ADAPTIS_OP_R_B; }
bool same(const adaptis_instr& a, const adaptis_instr& b) {
  return a.op == b.op && a.stage == b.stage && a.mb == b.mb && a.peer == b.peer;
}
// the instruction the peer must be at for `x` (on device d) to rendezvous
adaptis_instr counterpart(const adaptis_instr& x, int d) {
  adaptis_instr y = x;
  y.op = (x.op == ADAPTIS_OP_S_F || x.op == ADAPTIS_OP_S_B) ? x.op + 2 : x.op - 2;
  y.peer = d;
  return y;
}

using Prog = std::vector<std::vector<adaptis_instr>>;

// abstract rendezvous run; returns true when every program completes, else
// fills pc with the blocked frontier
bool run_abstract(const Prog& prog, std::vector<size_t>& pc) {
  const int p = (int)prog.size();
  pc.assign(p, 0);
  for (;;) {
    bool any = false;
    for (int d = 0; d < p; ++d) {
      while (pc[d] < prog[d].size()) {
        const adaptis_instr& x = prog[d][pc[d]];
        if (!is_comm(x.op)) { ++pc[d]; any = true; continue; }
        const int e = x.peer;
        if (pc[e] < prog[e].size() && same(prog[e][pc[e]], counterpart(x, d))) {
          ++pc[d]; ++pc[e]; any = true;
          continue;
        }
        break;
      }
    }
    bool done = true;
    for (int d = 0; d < p; ++d) done = done && pc[d] == prog[d].size();
    if (done) return true;
    if (!any) return false;
  }
}

}  // namespace

extern "C" {

adaptis_status adaptis_lower(int32_t p, const adaptis_plan* plan, const adaptis_task* tasks,
                             const uint64_t* offsets, int32_t flags, adaptis_instr* out, uint64_t cap,
                             uint64_t* out_offsets, int32_t* n_repairs, int32_t* n_hoists) {
  if (!plan || !tasks || !offsets || !out || !out_offsets) return exec_fail("a pointer argument is NULL");
  if (p < 1 || p > ADAPTIS_MAX_P) return exec_fail("p out of range");
  if (plan->policy != ADAPTIS_LIST && plan->policy != ADAPTIS_LIST_FUSED)
    return exec_fail("plan.policy must be ADAPTIS_LIST or ADAPTIS_LIST_FUSED");
  const int S = plan->S;
  if (S != p * plan->v || S < 1 || S > ADAPTIS_MAX_S) return exec_fail("plan.S != p * v");
  std::vector<int> dev(S);
  for (int s = 0; s < S; ++s) dev[s] = dev_of_stage(plan->placement, p, s);
  // emit: R then W before a compute with a cross-device input, S after
  // a compute with a cross-device output; comm ops carry the boundary b (stages b, b+1)
  Prog prog(p);
  for (int d = 0; d < p; ++d) {
    for (uint64_t q = offsets[d]; q < offsets[d + 1]; ++q) {
      const adaptis_task& t = tasks[q];
      if (t.stage < 0 || t.stage >= S || dev[t.stage] != d || t.kind < 0 || t.kind > 2)
        return exec_fail("task " + std::to_string(q) + " is not a task of device " + std::to_string(d));
      const int s = t.stage, j = t.mb;
      auto push = [&](int op, int b, int peer) { prog[d].push_back(adaptis_instr{op, b, j, peer}); };
      if (t.kind == 0 && s > 0 && dev[s - 1] != d) {
        push(ADAPTIS_OP_R_F, s - 1, dev[s - 1]);
        push(ADAPTIS_OP_W_F, s - 1, dev[s - 1]);
      }
      if (t.kind == 1 && s + 1 < S && dev[s + 1] != d) {
        push(ADAPTIS_OP_R_B, s, dev[s + 1]);
        push(ADAPTIS_OP_W_B, s, dev[s + 1]);
      }
      push(t.kind, s, -1);  // C_F / C_B / C_W carry the task's stage
      if (t.kind == 0 && s + 1 < S && dev[s + 1] != d) push(ADAPTIS_OP_S_F, s, dev[s + 1]);
      if (t.kind == 1 && s > 0 && dev[s - 1] != d) push(ADAPTIS_OP_S_B, s - 1, dev[s - 1]);
    }
  }
  uint64_t total = 0;
  for (int d = 0; d < p; ++d) total += prog[d].size();
  int32_t nr = 0, nh = 0;
  std::vector<size_t> pc;
  // repair: hoist the receive a blocked send waits for
  if (flags & ADAPTIS_LOWER_REPAIR) {
    const uint64_t limit = total * total + 1;
    while (!run_abstract(prog, pc)) {
      if ((uint64_t)nr >= limit) return exec_fail("deadlock repair did not converge");
      int fd = -1;
      size_t fi = 0;
      for (int d = 0; d < p && fd < 0; ++d) {
        if (pc[d] >= prog[d].size()) continue;
        for (int c = 0; c < p && fd < 0; ++c) {
          if (c == d || pc[c] >= prog[c].size()) continue;
          const adaptis_instr& x = prog[c][pc[c]];
          if ((x.op != ADAPTIS_OP_S_F && x.op != ADAPTIS_OP_S_B) || x.peer != d) continue;
          const adaptis_instr want = counterpart(x, c);
          for (size_t i = pc[d] + 1; i < prog[d].size(); ++i)
            if (same(prog[d][i], want)) { fd = d; fi = i; break; }
        }
      }
      if (fd < 0) return exec_fail("deadlock cannot be repaired by hoisting a receive");
      const adaptis_instr r = prog[fd][fi];
      prog[fd].erase(prog[fd].begin() + fi);
      prog[fd].insert(prog[fd].begin() + pc[fd], r);
      ++nr;
    }
  }
  // hoist: each receive moves earlier while it passes no receive
  // from the same peer and the programs stay deadlock-free
  if (flags & ADAPTIS_LOWER_HOIST) {
    for (int d = 0; d < p; ++d) {
      std::vector<adaptis_instr> rs;
      for (const adaptis_instr& x : prog[d])
        if (x.op == ADAPTIS_OP_R_F || x.op == ADAPTIS_OP_R_B) rs.push_back(x);
      for (const adaptis_instr& r : rs) {
        size_t i = 0;
        while (!same(prog[d][i], r)) ++i;
        while (i > 0) {
          const adaptis_instr& prev = prog[d][i - 1];
          if ((prev.op == ADAPTIS_OP_R_F || prev.op == ADAPTIS_OP_R_B) && prev.peer == r.peer) break;
          std::swap(prog[d][i - 1], prog[d][i]);
          if (!run_abstract(prog, pc)) { std::swap(prog[d][i - 1], prog[d][i]); break; }
          --i;
          ++nh;
        }
      }
    }
  }
  if (cap < total) return exec_fail("out holds " + std::to_string(cap) + " instructions, " +
                                    std::to_string(total) + " needed");
  uint64_t o = 0;
  for (int d = 0; d < p; ++d) {
    out_offsets[d] = o;
    for (const adaptis_instr& x : prog[d]) out[o++] = x;
  }
  out_offsets[p] = o;
  if (n_repairs) *n_repairs = nr;
  if (n_hoists) *n_hoists = nh;
  return ADAPTIS_OK;
}

const char* adaptis_lower_error(void) { return g_exec_error.c_str(); }

}  // extern "C"
