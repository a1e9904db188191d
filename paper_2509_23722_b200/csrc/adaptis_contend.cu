// adaptis_contend.cu — Alg. 1 Step 3 on explicit per-device task
// lists (R30) with communication-engine contention (SPEC S:206 (a)/(c),
// S:232; reading R34 in DESIGN.md).
//
// One warp per plan, lane d = pipeline device d (p <= 32). Each device has a
// compute engine, a send engine and a receive engine. A transfer (a stage edge
// between devices with latency > 0) is eligible at its producer's finish and
// holds the sender's send engine and the receiver's receive engine together,
// starting at max(eligible, send free, receive free); every engine serves
// transfers in (eligible, mb, stage, F < B) order.
//
// Rounds (bounded lag, the contention analogue of Lemma 3): in one round
//   * every lane whose next listed task has all its inputs commits it (its
//     start is exact: device free time and arrival times are known);
//   * a lane's oldest unassigned transfer X (its sends are created in list
//     order, at strictly increasing finish times) is assigned when its packed
//     key (eligible << 23 | mb << 7 | stage << 1 | kind) is below every other
//     lane's lower bound on the key of any transfer it has not assigned yet:
//     its own oldest pending key; (t + 1) << 23 for a lane whose next task can
//     start at t; (F + 1) << 23 for a blocked lane, F = the round's minimum over
//     all lanes of those start times and pending eligibility times (every
//     uncommitted task starts at >= F, because it waits for a pending transfer
//     (eligible >= F), for a task not yet run, or for its device).
//   Then X is next on both of its engines: no transfer with a smaller key can
//   still appear. Two transfers into one receiver are never both assignable
//   (each would have to be below the other), so receive engines update without
//   conflicts. Each round commits a task or assigns the globally smallest
//   pending transfer, so a round without either means a cyclic wait (STUCK).
// Per-plan scratch in global memory (L2-resident at the sizes explicit lists
// have): finish times fin[3][S][m] and output-ready times rdy[2][S][m] (-1 =
// unknown); a stage edge's output is ready at its arrival when it travels, at
// the producer's finish otherwise.
#include <cstdint>

#include "adaptis_decode.cuh"
#include "adaptis_internal.h"

namespace adaptis {

namespace {

constexpr int kCWarps = 4;
constexpr int64_t kUnknown = -1;
constexpr unsigned long long kKeyInf = ~0ull;

struct ContendArgs {
  const int64_t* cols;          // [kNumCols][L]
  const int64_t* comm;          // [L]
  int L, p, m;
  int64_t cap;
  uint64_t n;
  const adaptis_plan* plans;    // device copies
  const adaptis_task* tasks;
  const uint64_t* offsets;      // [n][p + 1]
  int64_t* scratch;             // [n][stride]
  uint64_t stride;              // 5 * Smax * m
  int64_t* out_makespan;
  int64_t* out_peak;
  float* out_bubble;
  uint8_t* out_status;
  int64_t* report;              // optional [n][5][p]
  unsigned long long* n_tasks;  // simulated tasks (work counter)
};

// per-slot stage table in dynamic shared memory: kTabCols int64 arrays of Sm
// entries, then Sm device ids (int8)
constexpr int kTabCols = 9;
enum { kTF = 0, kTB, kTW, kAlloc, kFreeB, kFreeW, kWG, kLatF, kLatB };
struct Tab {
  int64_t* t;
  int Sm;
  __device__ __forceinline__ int64_t& at(int col, int s) const { return t[col * Sm + s]; }
  __device__ __forceinline__ int8_t& dev(int s) const { return ((int8_t*)(t + kTabCols * Sm))[s]; }
};
__host__ __device__ __forceinline__ int tab_bytes(int Sm) { return (kTabCols * Sm * 8 + Sm + 15) & ~15; }

__device__ __forceinline__ int place(int placement, int p, int s) {  // R12
  if (placement == ADAPTIS_SEQ) return s;
  if (placement == ADAPTIS_INTERLEAVED) return s % p;
  const int c = s / p, j = s - c * p;
  return (c & 1) ? p - 1 - j : j;
}

// reductions over aligned segments of p2 lanes (one candidate slot each)
__device__ __forceinline__ unsigned long long seg_min_u64(unsigned long long x, int p2) {
  for (int o = p2 >> 1; o > 0; o >>= 1) {
    const unsigned long long y = __shfl_xor_sync(0xffffffffu, x, o);
    x = y < x ? y : x;
  }
  return x;
}
__device__ __forceinline__ int64_t seg_min_i64(int64_t x, int p2) {
  for (int o = p2 >> 1; o > 0; o >>= 1) {
    const int64_t y = __shfl_xor_sync(0xffffffffu, x, o);
    x = y < x ? y : x;
  }
  return x;
}
__device__ __forceinline__ int64_t seg_max_i64(int64_t x, int p2) {
  for (int o = p2 >> 1; o > 0; o >>= 1) {
    const int64_t y = __shfl_xor_sync(0xffffffffu, x, o);
    x = y > x ? y : x;
  }
  return x;
}
__device__ __forceinline__ int64_t seg_sum_i64(int64_t x, int p2) {
  for (int o = p2 >> 1; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

__device__ __forceinline__ int64_t dur_of(const Tab& tb, const adaptis_task& t) {
  return t.kind == 0 ? tb.at(kTF, t.stage) : t.kind == 1 ? tb.at(kTB, t.stage) : tb.at(kTW, t.stage);
}
__device__ __forceinline__ int64_t out_lat(const Tab& tb, const adaptis_task& t) {
  return t.kind == 0 ? tb.at(kLatF, t.stage) : t.kind == 1 ? tb.at(kLatB, t.stage) : 0;
}

// length of [a, b) outside the device's compute intervals (its list, in order)
__device__ int64_t outside_compute(int64_t a, int64_t b, const adaptis_task* lst, int len,
                                   const int64_t* fin, const Tab& tb, int S, int m) {
  if (b <= a) return 0;
  // first listed task whose finish is > a (finish times increase along the list)
  int lo = 0, hi = len;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    const adaptis_task t = lst[mid];
    if (fin[((size_t)t.kind * S + t.stage) * m + t.mb] > a) hi = mid; else lo = mid + 1;
  }
  int64_t cov = 0;
  for (int i = lo; i < len; ++i) {
    const adaptis_task t = lst[i];
    const int64_t f = fin[((size_t)t.kind * S + t.stage) * m + t.mb];
    const int64_t s0 = f - dur_of(tb, t);
    if (s0 >= b) break;
    const int64_t x0 = s0 > a ? s0 : a, x1 = f < b ? f : b;
    if (x1 > x0) cov += x1 - x0;
  }
  return (b - a) - cov;
}

// G = 32 / p2 plans per warp (p2 = p rounded up to a power of two); lane
// slot * p2 + d is device d of the slot's plan
__global__ void __launch_bounds__(kCWarps * 32) contend_kernel(ContendArgs A, int p2, int Sm) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int64_t recv_val[kCWarps][32];
  __shared__ int32_t recv_round[kCWarps][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int G = 32 / p2, slot = lane / p2, d = lane - slot * p2, base = slot * p2;
  const unsigned smask = (p2 == 32 ? 0xffffffffu : ((1u << p2) - 1u)) << base;
  const uint64_t o = ((uint64_t)blockIdx.x * kCWarps + w) * G + slot;
  if (((uint64_t)blockIdx.x * kCWarps + w) * G >= A.n) return;  // warp-uniform
  const bool valid = o < A.n;
  const Tab tb{(int64_t*)(smem + (size_t)(w * G + slot) * tab_bytes(Sm)), Sm};
  const adaptis_plan& pl = A.plans[valid ? o : 0];
  const int p = A.p, m = A.m, L = A.L;
  const int S = valid ? pl.S : 0;
  const bool fused = pl.policy == ADAPTIS_LIST_FUSED;
  // ---- a2/a3: stage sums and edge latencies (R3-R6)
  for (int s = d; s < S; s += p2) {
    const int b0 = s == 0 ? 0 : pl.cuts[s], b1 = s == S - 1 ? L : pl.cuts[s + 1];
    int64_t c[kNumCols] = {0, 0, 0, 0, 0, 0};
    for (int r = b0; r < b1; ++r)
#pragma unroll
      for (int k = 0; k < kNumCols; ++k) c[k] += A.cols[(size_t)k * L + r];
    tb.at(kTF, s) = c[kColTF];
    tb.at(kTB, s) = c[kColTB] + (fused ? c[kColTW] : 0);
    tb.at(kTW, s) = c[kColTW];
    tb.at(kAlloc, s) = c[kColAct] + c[kColStash];
    tb.at(kFreeB, s) = c[kColAct] + (fused ? c[kColStash] : 0);
    tb.at(kFreeW, s) = fused ? 0 : c[kColStash];
    tb.at(kWG, s) = c[kColWG];
    tb.dev(s) = (int8_t)place(pl.placement, p, s);
  }
  __syncwarp();
  for (int s = d; s < S; s += p2) {
    const int b0 = s == 0 ? 0 : pl.cuts[s], b1 = s == S - 1 ? L : pl.cuts[s + 1];
    tb.at(kLatF, s) = (s + 1 < S && tb.dev(s + 1) != tb.dev(s)) ? A.comm[b1 - 1] : 0;
    tb.at(kLatB, s) = (s > 0 && tb.dev(s - 1) != tb.dev(s)) ? A.comm[b0 - 1] : 0;
  }
  recv_round[w][lane] = -1;
  int64_t* fin = A.scratch + (valid ? o : 0) * A.stride;  // [3][S][m]
  int64_t* rdy = fin + (size_t)3 * S * m;                  // [2][S][m]
  for (uint64_t q = d; q < (uint64_t)5 * S * m; q += p2) fin[q] = kUnknown;
  __syncwarp();
  const bool live = valid && d < p;
  const uint64_t* off = A.offsets + (valid ? o : 0) * (uint64_t)(p + 1);
  const uint64_t beg = live ? off[d] : 0, end = live ? off[d + 1] : 0;
  const adaptis_task* lst = A.tasks + beg;
  const int len = (int)(end - beg);
  int64_t stat = 0;
  for (int s = 0; s < S; ++s)
    if (tb.dev(s) == d) stat += tb.at(kWG, s);
  int ptr = 0, sq = 0;
  int64_t freet = 0, sfree = 0, rfree = 0, busy = 0, dyn = 0, peak = 0, Td = 0, commd = 0;
  uint64_t ntask = 0;
  bool stuck = false, done = !valid;
  for (int round = 0;; ++round) {
    // (1) can my next listed task start, and when?
    int64_t t = INT64_MAX;
    adaptis_task X{};
    if (!done && ptr < len) {
      X = lst[ptr];
      const size_t jm = (size_t)X.stage * m + X.mb;
      int64_t r0 = freet;
      bool ok = true;
      if (X.kind == 0) {
        if (X.stage > 0) {
          const int64_t a = ((volatile int64_t*)rdy)[jm - m];  // F(s-1, j), over the edge
          ok = a >= 0; r0 = a > r0 ? a : r0;
        }
      } else if (X.kind == 1) {
        const int64_t a = ((volatile int64_t*)fin)[jm];       // F(s, j), same device
        ok = a >= 0; r0 = a > r0 ? a : r0;
        if (X.stage + 1 < S) {
          const int64_t b = ((volatile int64_t*)rdy)[(size_t)S * m + jm + m];  // B(s+1, j)
          ok = ok && b >= 0; r0 = b > r0 ? b : r0;
        }
      } else {
        const int64_t a = ((volatile int64_t*)fin)[(size_t)S * m + jm];  // B(s, j), same device
        ok = a >= 0; r0 = a > r0 ? a : r0;
      }
      if (ok) t = r0;
    }
    // (2) my oldest unassigned transfer
    adaptis_task Y{};
    int64_t lat = 0;
    while (sq < ptr) {
      Y = lst[sq];
      lat = out_lat(tb, Y);
      if (lat > 0) break;
      ++sq;
    }
    unsigned long long hk = kKeyInf;
    int64_t he = INT64_MAX;
    if (sq < ptr) {
      he = ((volatile int64_t*)fin)[((size_t)Y.kind * S + Y.stage) * m + Y.mb];
      hk = ((unsigned long long)he << 23) | ((unsigned long long)Y.mb << 7) |
           ((unsigned long long)Y.stage << 1) | (unsigned long long)Y.kind;
    }
    // (3) F: earliest known start or pending eligibility over the slot
    const int64_t F = seg_min_i64(t < he ? t : he, p2);
    // (4) my lower bound on the key of any transfer I have not assigned
    unsigned long long lb;
    if (sq < ptr) lb = hk;
    else if (done || ptr >= len) lb = kKeyInf;
    else if (t != INT64_MAX) lb = (unsigned long long)(t + 1) << 23;
    else lb = F == INT64_MAX ? kKeyInf : (unsigned long long)(F + 1) << 23;
    // (5) minimum over the slot's other lanes: the min, its lane, the runner-up
    const unsigned long long m1 = seg_min_u64(lb, p2);
    const unsigned arg_mask = __ballot_sync(0xffffffffu, lb == m1) & smask;
    const int arg = __ffs(arg_mask) - 1;
    const unsigned long long m2 = seg_min_u64(lane == arg ? kKeyInf : lb, p2);
    const unsigned long long other = lane == arg ? m2 : m1;
    // equality can only be with another lane's bound (head keys are unique), and
    // no unassigned transfer of that lane can have exactly that key
    const bool safe = sq < ptr && hk <= other;
    // (6) assign the safe transfers
    const int dst = safe ? (int)tb.dev(Y.kind == 0 ? Y.stage + 1 : Y.stage - 1) : d;
    const int64_t rf = __shfl_sync(0xffffffffu, rfree, base + dst);
    if (safe) {
      const int64_t s0 = he > sfree ? he : sfree;
      const int64_t start = s0 > rf ? s0 : rf;
      const int64_t arr = start + lat;
      rdy[(size_t)(Y.kind == 0 ? 0 : 1) * S * m + (size_t)Y.stage * m + Y.mb] = arr;
      sfree = arr;
      commd += lat;
      recv_val[w][base + dst] = arr;
      recv_round[w][base + dst] = round;
      ++sq;
    }
    // (7) commit my task
    const bool commit = t != INT64_MAX;
    if (commit) {
      const int64_t du = dur_of(tb, X);
      const int64_t f = t + du;
      const size_t jm = (size_t)X.stage * m + X.mb;
      fin[(size_t)X.kind * S * m + jm] = f;
      freet = f;
      Td = f;
      busy += du;
      if (X.kind == 0) {
        dyn += tb.at(kAlloc, X.stage);
        peak = dyn > peak ? dyn : peak;
        if (tb.at(kLatF, X.stage) == 0) rdy[jm] = f;  // same device or zero latency: no transfer
      } else if (X.kind == 1) {
        dyn -= tb.at(kFreeB, X.stage);
        if (tb.at(kLatB, X.stage) == 0) rdy[(size_t)S * m + jm] = f;
      } else {
        dyn -= tb.at(kFreeW, X.stage);
      }
      ++ptr;
      ++ntask;
    }
    __syncwarp();
    if (live && recv_round[w][lane] == round) rfree = recv_val[w][lane];
    // a slot without a commit or an assignment is finished (or stuck)
    const unsigned prog = __ballot_sync(0xffffffffu, safe || commit);
    const unsigned left = __ballot_sync(0xffffffffu, !done && ptr < len);
    if (!done && (prog & smask) == 0) {
      done = true;
      stuck = (left & smask) != 0;
    }
    if (__all_sync(0xffffffffu, done)) break;
    __syncwarp();
  }
  // ---- a6: per-device report and per-plan metrics
  const int64_t Md = stat + peak;
  const int64_t makespan = seg_max_i64(live ? Td : 0, p2);
  const int64_t peak_all = seg_max_i64(live ? Md : 0, p2);
  const int64_t busy_all = seg_sum_i64(live ? busy : 0, p2);
  const unsigned long long nt = (unsigned long long)seg_sum_i64((int64_t)ntask, 32);
  if (lane == 0) atomicAdd(A.n_tasks, nt);
  if (!valid) return;
  const bool over = peak_all > A.cap;
  const uint8_t status = stuck ? ADAPTIS_CAND_STUCK : over ? ADAPTIS_CAND_OVER_CAP : ADAPTIS_CAND_OK;
  // R29 on the contended schedule: comm_d = latencies of the transfers d sends
  // or receives; exposed_d = |(sends U receives) within [0, T_d]| outside compute
  int64_t comm_in = 0, exposed = 0;
  if (A.report && live && !stuck) {
    // sends (disjoint, in list order) and receives (disjoint): inclusion-exclusion
    int64_t ex_s = 0, ex_r = 0, ex_sr = 0;
    for (int i = 0; i < len; ++i) {
      const adaptis_task U = lst[i];
      const size_t jm = (size_t)U.stage * m + U.mb;
      const int64_t ls = out_lat(tb, U);  // my send of U's output
      if (ls > 0) {
        const int64_t a1 = rdy[(size_t)(U.kind == 0 ? 0 : 1) * S * m + jm];
        ex_s += outside_compute(a1 - ls, a1 < Td ? a1 : Td, lst, len, fin, tb, S, m);
      }
      int64_t lr = 0, r1 = 0;             // my receive of U's cross-device input
      if (U.kind == 0 && U.stage > 0 && tb.at(kLatF, U.stage - 1) > 0) {
        lr = tb.at(kLatF, U.stage - 1); r1 = rdy[jm - m];
      } else if (U.kind == 1 && U.stage + 1 < S && tb.at(kLatB, U.stage + 1) > 0) {
        lr = tb.at(kLatB, U.stage + 1); r1 = rdy[(size_t)S * m + jm + m];
      }
      if (lr > 0) {
        comm_in += lr;
        const int64_t r0 = r1 - lr, rb = r1 < Td ? r1 : Td;
        ex_r += outside_compute(r0, rb, lst, len, fin, tb, S, m);
        for (int k2 = 0; k2 < len; ++k2) {  // overlap of this receive with my sends
          const adaptis_task V = lst[k2];
          const int64_t lv = out_lat(tb, V);
          if (lv <= 0) continue;
          const int64_t v1 = rdy[(size_t)(V.kind == 0 ? 0 : 1) * S * m + (size_t)V.stage * m + V.mb];
          const int64_t v0 = v1 - lv;
          const int64_t x0 = v0 > r0 ? v0 : r0, x1 = v1 < rb ? v1 : rb;
          if (x1 > x0) ex_sr += outside_compute(x0, x1, lst, len, fin, tb, S, m);
        }
      }
    }
    exposed = ex_s + ex_r - ex_sr;
  }
  if (A.report && live) {
    int64_t* rep = A.report + o * 5 * (uint64_t)p;
    rep[d] = stuck ? 0 : Td;
    rep[p + d] = busy;
    rep[2 * p + d] = Md;
    rep[3 * p + d] = stuck ? 0 : commd + comm_in;
    rep[4 * p + d] = stuck ? 0 : exposed;
  }
  if (d == 0) {
    A.out_status[o] = status;
    A.out_makespan[o] = status == ADAPTIS_CAND_OK ? makespan : INT64_MAX;
    A.out_peak[o] = stuck ? 0 : peak_all;
    A.out_bubble[o] = status == ADAPTIS_CAND_OK
                          ? (float)(1.0 - (double)busy_all / ((double)p * (double)makespan)) : 0.0f;
  }
}

}  // namespace

int launch_contend(const int64_t* cols, const int64_t* comm, int L, int p, int m, int64_t cap, uint64_t n,
                   const adaptis_plan* plans, const adaptis_task* tasks, const uint64_t* offsets,
                   int64_t* scratch, uint64_t stride, int64_t* makespan, int64_t* peak, float* bubble,
                   uint8_t* status, int64_t* report, unsigned long long* n_tasks, int Sm, void* stream) {
  if (n == 0) return 0;
  ContendArgs A{cols, comm, L, p, m, cap, n, plans, tasks, offsets, scratch, stride,
                makespan, peak, bubble, status, report, n_tasks};
  int p2 = 1;
  while (p2 < p) p2 <<= 1;
  const int G = 32 / p2;
  const size_t smem = (size_t)kCWarps * G * tab_bytes(Sm);
  const uint64_t warps = (n + G - 1) / G;
  const unsigned grid = (unsigned)((warps + kCWarps - 1) / kCWarps);
  if (smem > 48 * 1024) {
    const cudaError_t e = cudaFuncSetAttribute(contend_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return (int)e;
  }
  contend_kernel<<<grid, kCWarps * 32, smem, (cudaStream_t)stream>>>(A, p2, Sm);
  return (int)cudaGetLastError();
}

// ---- contention on realised orders (reading R36): candidates of one segment
// whose policy run (pure latency, R3-R6) was traced become explicit schedules
// (R30) for the contention kernel. One warp per candidate: the candidate's
// cuts are decoded (R19), its traced per-device orders are copied to a
// contiguous list, and kept candidates are compacted through an atomic slot.
__global__ void realised_lists_kernel(const TraceEntry* __restrict__ trace, const int* __restrict__ trace_n,
                                      int cap_t, int p, uint64_t n, uint64_t first,
                                      const uint8_t* __restrict__ status, RealisedSeg seg,
                                      adaptis_plan* __restrict__ plans, adaptis_task* __restrict__ tasks,
                                      uint64_t* __restrict__ offsets, uint64_t* __restrict__ slot_idx,
                                      unsigned int* __restrict__ n_kept) {
  const int lane = threadIdx.x & 31;
  const uint64_t o = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (o >= n) return;
  const uint8_t st = status[o];
  if (st != ADAPTIS_CAND_OK && st != ADAPTIS_CAND_OVER_CAP) return;  // invalid / stuck: no full order
  unsigned int k = 0;
  if (lane == 0) k = atomicAdd(n_kept, 1u);
  k = __shfl_sync(0xffffffffu, k, 0);
  const uint64_t tb = (uint64_t)k * p * cap_t;  // this candidate's task range
  if (lane == 0) {
    adaptis_plan pl;
    pl.v = seg.v; pl.placement = seg.placement; pl.S = seg.S;
    pl.policy = seg.fused ? ADAPTIS_LIST_FUSED : ADAPTIS_LIST;
    decode_cuts(seg.binom, seg.ball, seg.seeds, seg.group, seg.part_mode, seg.radius, seg.S, seg.L,
                first + o - seg.base, pl.cuts);
    plans[k] = pl;
    slot_idx[k] = o;
    uint64_t off = tb;
    for (int d = 0; d < p; ++d) {
      offsets[(uint64_t)k * (p + 1) + d] = off;
      off += (uint64_t)min(trace_n[o * p + d], cap_t);
    }
    offsets[(uint64_t)k * (p + 1) + p] = off;
  }
  __syncwarp();
  uint64_t off = tb;
  for (int d = 0; d < p; ++d) {
    const int nt = min(trace_n[o * p + d], cap_t);
    const TraceEntry* e = trace + (o * p + d) * (uint64_t)cap_t;
    for (int i = lane; i < nt; i += 32) {
      adaptis_task t;
      t.kind = e[i].kind; t.stage = e[i].stage; t.mb = e[i].mb;
      tasks[off + i] = t;
    }
    off += (uint64_t)nt;
  }
}

// packed argmin key of the contended results (R18: lowest index among equal
// makespans), folded into *key with one atomicMin per warp
__global__ void contended_key_kernel(const int64_t* __restrict__ makespan, const uint8_t* __restrict__ status,
                                     const uint64_t* __restrict__ slot_idx, uint64_t n, uint64_t first,
                                     int key_bits, unsigned long long* key) {
  const uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long v = ~0ull >> 1;
  if (k < n && status[k] == ADAPTIS_CAND_OK)
    v = ((unsigned long long)makespan[k] << key_bits) | (first + slot_idx[k]);
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long x = __shfl_xor_sync(0xffffffffu, v, o);
    v = x < v ? x : v;
  }
  if ((threadIdx.x & 31) == 0 && v != (~0ull >> 1)) atomicMin(key, v);
}

int launch_realised_lists(const TraceEntry* trace, const int* trace_n, int trace_cap, int p, uint64_t n,
                          uint64_t first, const uint8_t* status, const RealisedSeg& seg, adaptis_plan* plans,
                          adaptis_task* tasks, uint64_t* offsets, uint64_t* slot_idx, unsigned int* n_kept,
                          void* stream) {
  if (n == 0) return 0;
  const uint64_t threads = n * 32;
  realised_lists_kernel<<<(unsigned)((threads + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
      trace, trace_n, trace_cap, p, n, first, status, seg, plans, tasks, offsets, slot_idx, n_kept);
  return (int)cudaGetLastError();
}

int launch_contended_key(const int64_t* makespan, const uint8_t* status, const uint64_t* slot_idx, uint64_t n,
                         uint64_t first, int key_bits, unsigned long long* key, void* stream) {
  if (n == 0) return 0;
  contended_key_kernel<<<(unsigned)((n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(makespan, status, slot_idx,
                                                                                     n, first, key_bits, key);
  return (int)cudaGetLastError();
}

}  // namespace adaptis
