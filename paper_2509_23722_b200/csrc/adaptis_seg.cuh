#pragma once
// adaptis_seg.cuh — sm_100a kernels of the AdaPtis hot path (arXiv 2509.23722).
//
// One persistent kernel per (v-group, combo) segment of the candidate space.
// A warp holds G = 32 / p2 candidate slots (p2 = p rounded up to a power of
// two); inside a slot, lane d is pipeline device d. Slots are refilled
// independently from a warp-local queue of index positions, so invalid and
// over-capacity candidates never occupy simulation rounds. Per candidate
// (DESIGN.md §"Kernel"):
//   a1 decode        index -> cuts (colex / L1-ball unranking, lane 0 of the slot)
//   a2 stage sums    prefix differences of the CTA's shared-memory prefix table,
//                    built once per CTA by a warp-shuffle scan of coalesced loads
//   a3 device sums   static memory, busy time, edge latencies (R3-R6), folded
//                    into per-(kind, chunk) task records in shared memory
//   a4 memory check  fused fixed orders: exact peak from the order alone (R16,
//                    periodic closed form for the Megatron interleaved order)
//   a5 simulation    dataflow rounds (GPIPE / ONEF1B / ZB, Lemmas 1-2) or
//                    bounded-lag rounds (GREEDY, Lemma 3); cross-device arrival
//                    times travel through per-stage rings in shared memory
//   a6 metrics       segmented shuffle reductions (makespan, busy, peak)
//   a7 argmin        packed (makespan << bits | index) warp min -> atomicMin
// Ticks are int32 when the host proved the makespan bound fits, else int64.
#include <cuda_runtime.h>

#include <climits>
#include <cstdio>
#include <cstdint>
#include <type_traits>

#include "adaptis_decode.cuh"
#include "adaptis_internal.h"

namespace adaptis {

#ifdef ADAPTIS_DEBUG
#define DCHECK(cond, what, val)                                                          \
  do {                                                                                   \
    if (!(cond)) {                                                                       \
      printf("DCHECK %s failed: %s = %lld (block %d lane %d)\n", #cond, what,          \
             (long long)(val), blockIdx.x, threadIdx.x);                                 \
      __trap();                                                                          \
    }                                                                                    \
  } while (0)
#else
#define DCHECK(cond, what, val) do { } while (0)
#endif

constexpr unsigned FULLMASK = 0xffffffffu;
#ifndef ADAPTIS_KRUN
#define ADAPTIS_KRUN 32
#endif
constexpr int kRun = ADAPTIS_KRUN;  // consecutive positions a slot claims (incremental decode)
#ifndef ADAPTIS_TSTAR_REDUX
#define ADAPTIS_TSTAR_REDUX 0
#endif
#ifndef ADAPTIS_GREEDY_ALWAYS_DECIDE
#define ADAPTIS_GREEDY_ALWAYS_DECIDE 2  // from this V up, decide() always recomputes
#endif
#ifndef ADAPTIS_ZB_WFILL_ONE
#define ADAPTIS_ZB_WFILL_ONE 0
#endif
#ifndef ADAPTIS_GREEDY_COMMITS
#define ADAPTIS_GREEDY_COMMITS 1
#endif
constexpr int kGreedyCommits = ADAPTIS_GREEDY_COMMITS;  // GREEDY tasks a lane may commit per round
constexpr unsigned kTstarEvery = 1; // GREEDY t* refresh period (a stale t* costs more commits than it saves)

template <typename T> struct TT;
template <> struct TT<int32_t> { static constexpr int32_t INF = INT32_MAX; };
template <> struct TT<int64_t> { static constexpr int64_t INF = INT64_MAX; };
template <> struct TT<float> { static constexpr float INF = __builtin_huge_valf(); };
// busy-time accumulator and integer rounding per tick type
template <typename T> struct Acc { using type = int64_t; };
template <> struct Acc<float> { using type = double; };
__device__ __forceinline__ int64_t to_ticks(int32_t x) { return x; }
__device__ __forceinline__ int64_t to_ticks(int64_t x) { return x; }
__device__ __forceinline__ int64_t to_ticks(float x) { return llrintf(x); }
__device__ __forceinline__ int64_t to_ticks(double x) { return llrint(x); }

template <typename T>
struct __align__(16) Rec {  // one task kind of one own stage (chunk) of a lane
  T dur;        // duration (B includes c_W when fused, R2)
  T oc;         // latency added to the successor's arrival (R3-R6; 0 when co-located)
  int in_off;   // ring offset of the input slot row, -1 = no cross-stage input
  int out_off;  // ring offset of the output slot row, -1 = no successor
};

template <typename T>
struct GAux {      // GREEDY statics of one (lane, chunk); stored as SoA, this fixes the size
  int64_t gate;    // F of the chunk fits under Eq. 2 iff dyn <= gate (R14)
  int32_t tF, tB;  // consumer (lane << 3 | chunk) of the F / B output, -1: none
  T pF, pB;        // cost of the cross-device predecessor of an unknown F / B head
};
// fp32 ticks (R27): the predecessor's duration and its latency are kept apart so
// that a bound is rounded exactly like the arrival it bounds, fl(fl(t + dur) + lat)
// (monotone in t), never above it
template <>
struct GAux<float> {
  int64_t gate;
  int32_t tF, tB;
  float pF, pB;    // predecessor duration
  float lF, lB;    // predecessor edge latency
};

// per-lane state touched only at candidate setup / finalize and at kernel exit,
// kept in shared memory so that the round loop keeps its registers (48 bytes)
struct LaneCold {
  uint64_t idx;                   // global index of the slot's candidate
  int64_t busy;                   // busy time (int64, or double bits in the fp32 variant)
  unsigned long long key;         // running minimum of the packed argmin key
  unsigned long long invalid, tasks, live;  // counters flushed at kernel exit
  unsigned long long pruned;
  uint64_t slot;                  // eval: output slot of the candidate (idx - eval_first, or list_slot)
};
static_assert(sizeof(LaneCold) == 64, "LaneCold layout");

enum : int { F_INVALID = 1, F_PREOVER = 2, F_STUCK = 4, F_OVERFLOW = 8, F_PRUNED = 16 };

__device__ __forceinline__ int stage_of(int placement, int p, int c, int d) {
  if (placement == ADAPTIS_SEQ) return d;
  if (placement == ADAPTIS_INTERLEAVED) return c * p + d;
  return c * p + ((c & 1) ? p - 1 - d : d);  // WAVE (R12)
}
__device__ __forceinline__ int dev_of(int placement, int p, int s) {
  if (placement == ADAPTIS_SEQ) return s;
  if (placement == ADAPTIS_INTERLEAVED) return s % p;
  const int c = s / p, j = s - c * p;
  return (c & 1) ? p - 1 - j : j;
}

// segmented reductions over aligned groups of p2 lanes (p2 is warp-uniform, so
// the unrolled steps are uniform predicates, not a runtime loop)
template <typename X>
__device__ __forceinline__ X seg_max(X v, int p2) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1)
    if (o < p2) { X w = __shfl_xor_sync(FULLMASK, v, o); v = w > v ? w : v; }
  return v;
}
template <typename X>
__device__ __forceinline__ X seg_min(X v, int p2) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1)
    if (o < p2) { X w = __shfl_xor_sync(FULLMASK, v, o); v = w < v ? w : v; }
  return v;
}
// segment minimum over the slot's lanes `smask`: the shuffle ladder. REDUX with
// per-slot masks (ADAPTIS_TSTAR_REDUX) was measured 3.4 % slower on cfg3, where
// four 8-lane slots share a warp (11.8 % of GREEDY's stall samples on it)
template <typename X>
__device__ __forceinline__ X seg_min_m(X v, int p2, unsigned smask) {
#if ADAPTIS_TSTAR_REDUX
  if constexpr (std::is_same<X, int>::value) return __reduce_min_sync(smask, v);
  else return seg_min(v, p2);
#else
  (void)smask;
  return seg_min(v, p2);
#endif
}
template <typename X>
__device__ __forceinline__ X seg_sum(X v, int p2) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1)
    if (o < p2) v += __shfl_xor_sync(FULLMASK, v, o);
  return v;
}
template <typename T>
__device__ __forceinline__ T sat_add(T a, T b) {
  if constexpr (std::is_floating_point<T>::value) {
    return a + b;  // inf saturates
  } else {  // a, b in [0, INF]: the unsigned sum cannot wrap
    using U = typename std::make_unsigned<T>::type;
    const U x = (U)a + (U)b;
    return x < (U)TT<T>::INF ? (T)x : TT<T>::INF;
  }
}

// incremental position in Megatron's virtual order (R10): k -> (chunk, mb)
struct VPos {
  int q, c, mb0;  // k = (g * v + c) * p + q, mb = g * p + q = mb0 + q
  __device__ __forceinline__ void reset() { q = 0; c = 0; mb0 = 0; }
  __device__ __forceinline__ void next(int p, int v) {
    if (++q == p) { q = 0; if (++c == v) { c = 0; mb0 += p; } }
  }
  __device__ __forceinline__ int mb() const { return mb0 + q; }
};

// R16 for the Megatron order (R9/R10): the in-flight bytes right after the
// (w+i+1)-th forward and before the (i+1)-th backward are
// D(i) = Fsum(w+i+1) - Bsum(i), and D is periodic in i with period p*v, so the
// peak of the whole list is max(D(i), i < min(p*v, m*v - w)) (Fsum(m*v) when
// the warm-up covers everything).
template <int V>
__device__ __forceinline__ int64_t chunk_prefix(const int64_t (&a)[V], int p, int n, bool bwd) {
  const int P = p * V;
  const int q = n / P, r = n - q * P, cf = r / p;
  int64_t A = 0, s = 0;
#pragma unroll
  for (int c = 0; c < V; ++c) {
    const int64_t ac = bwd ? a[V - 1 - c] : a[c];
    A += ac;
    if (c < cf) s += (int64_t)p * ac;
    if (c == cf) s += (int64_t)(r - cf * p) * ac;
  }
  return (int64_t)q * p * A + s;
}
template <int V>
__device__ int64_t megatron_peak(const int64_t (&a)[V], int p, int m, int w) {
  const int tot = m * V;
  if (w >= tot) return chunk_prefix<V>(a, p, tot, false);
  const int lim = min(p * V, tot - w);
  int64_t best = 0;
  for (int i = 0; i < lim; ++i) {
    const int64_t x = chunk_prefix<V>(a, p, w + i + 1, false) - chunk_prefix<V>(a, p, i, true);
    best = x > best ? x : best;
  }
  return best;
}

// successors in the canonical order (R19), for consecutive indices of one slot:
// L1 ball: odometer over delta_n (fastest) .. delta_1 with digit order
// 0, -1, +1, -2, +2, ... and the remaining radius `rem`
__device__ __forceinline__ void ball_next(int16_t* cuts, const int16_t* seed, int n, int& rem) {
  for (int i = n; i >= 1; --i) {
    const int di = cuts[i] - seed[i - 1];
    const int ai = di < 0 ? -di : di;
    const int nd = di == 0 ? -1 : (di < 0 ? -di : -di - 1);
    const int cost = (nd < 0 ? -nd : nd) - ai;
    if (cost <= rem) { cuts[i] = (int16_t)(seed[i - 1] + nd); rem -= cost; return; }
    rem += ai;
    cuts[i] = seed[i - 1];  // digit back to 0, carry into delta_{i-1}
  }
}
// FULL: colex successor of c_1 < ... < c_{S-1} < cuts[S] = L
__device__ __forceinline__ void colex_next(int16_t* cuts, int S) {
  for (int i = 1; i <= S - 1; ++i) {
    if (cuts[i] + 1 < cuts[i + 1]) {
      cuts[i] = (int16_t)(cuts[i] + 1);
      for (int k = 1; k < i; ++k) cuts[k] = (int16_t)k;
      return;
    }
  }
}

__device__ __forceinline__ uint64_t pos_to_index(const SegLaunch& sl, uint64_t pos) {
  if (sl.list_slot) return sl.slot_idx[sl.list_slot[pos]];
  if (sl.list_idx) return sl.list_idx[pos];
  if (sl.list_out) return sl.list_out[pos];
  return shard_index(pos, sl.n0, sl.start0, sl.first_chunk, sl.world);
}

// register budget (measured on B200, DESIGN.md §4 "Occupancy"): every policy
// runs best at <= 102 registers (5 CTAs of 4 warps per SM); GREEDY with its
// rings in global memory so that shared memory does not cap occupancy
#ifndef ADAPTIS_GREEDY_MINB
#define ADAPTIS_GREEDY_MINB 4  // round 2: the lane kernel's GREEDY v <= 2 now runs mainly cfg5's p = 16 WAVE
#endif                         // segment: 4 CTAs 24.5 s, 5 CTAs 25.7 s, 3 CTAs 27.1 s
#ifndef ADAPTIS_GREEDY_V4_MINB
#define ADAPTIS_GREEDY_V4_MINB 3  // cfg5 p = 16 v = 4: 3 CTAs 4.32 / 3.58 s, 4 CTAs 4.45 / 3.69 s, 2 CTAs 5.43 / 4.51 s
#endif
#ifndef ADAPTIS_FIXED_V4_MINB
#define ADAPTIS_FIXED_V4_MINB 4
#endif
template <int POLICY, int V> struct MinBlocks {
  static constexpr int value = POLICY != ADAPTIS_GREEDY
                                   ? (V >= 3 ? ADAPTIS_FIXED_V4_MINB : 5)
                                   : (V >= 3 ? ADAPTIS_GREEDY_V4_MINB : ADAPTIS_GREEDY_MINB);
};

template <int POLICY, int V, typename T, bool GRING, bool TRACE = false>
__global__ void __launch_bounds__(kWarpsPerCta * 32, MinBlocks<POLICY, V>::value)
seg_kernel(const DevTables tab, const SegLaunch sl) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr bool FUSED = (POLICY == ADAPTIS_GPIPE || POLICY == ADAPTIS_ONEF1B);
  constexpr bool ZB = (POLICY == ADAPTIS_ZB);
  constexpr bool LISTP = (POLICY == ADAPTIS_LIST || POLICY == ADAPTIS_LIST_FUSED);
  constexpr bool BFUSED = FUSED || POLICY == ADAPTIS_LIST_FUSED;  // B runs t_B + t_W, frees act + stash
  constexpr bool GREEDY = (POLICY == ADAPTIS_GREEDY);
  constexpr bool kAlwaysDecide = V >= ADAPTIS_GREEDY_ALWAYS_DECIDE;
  constexpr T INF = TT<T>::INF;
  constexpr T EMPTY = (T)-1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int L = sl.L, p = sl.p, m = sl.m, S = sl.S, p2 = sl.p2, G = sl.G;

  constexpr bool FP = std::is_floating_point<T>::value;
  using BT = typename Acc<T>::type;
  // ---- a2 prologue: per-CTA prefix table of the layer columns (warp-shuffle scan);
  // in the fp32-cost variant the three duration columns are real-valued (double sums)
  int64_t* pre = reinterpret_cast<int64_t*>(smem);
  double* pref = reinterpret_cast<double*>(smem);
  for (int col = warp; col < kNumCols; col += kWarpsPerCta) {
    if (FP && col < 3) {
      double carry = 0;
      const double* src = tab.colsf + (size_t)col * L;
      double* dst = pref + (size_t)col * (L + 1);
      if (lane == 0) dst[0] = 0;
      for (int b = 0; b < L; b += 32) {
        double x = (b + lane < L) ? src[b + lane] : 0.0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const double y = __shfl_up_sync(FULLMASK, x, o);
          if (lane >= o) x += y;
        }
        if (b + lane < L) dst[b + lane + 1] = carry + x;
        carry += __shfl_sync(FULLMASK, x, 31);
      }
      continue;
    }
    int64_t carry = 0;
    const int64_t* src = tab.cols + (size_t)col * L;
    int64_t* dst = pre + (size_t)col * (L + 1);
    if (lane == 0) dst[0] = 0;
    for (int b = 0; b < L; b += 32) {
      int64_t x = (b + lane < L) ? src[b + lane] : 0;  // coalesced 8-byte loads
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(FULLMASK, x, o);
        if (lane >= o) x += y;
      }
      if (b + lane < L) dst[b + lane + 1] = carry + x;
      carry += __shfl_sync(FULLMASK, x, 31);
    }
  }
  __syncthreads();
  // stage sum of a duration column over rows [a, b) and an edge latency, per tick type
  auto dsum = [&](int col, int a, int b) -> BT {
    if constexpr (FP) return pref[col * (L + 1) + b] - pref[col * (L + 1) + a];
    else return pre[col * (L + 1) + b] - pre[col * (L + 1) + a];
  };
  auto lat = [&](int row) -> T {
    if constexpr (FP) return tab.commf[row];
    else return (T)tab.comm[row];
  };

  // ---- per-warp shared regions (layout mirrored by smem_bytes())
  const WarpLayout lay = warp_layout(S, G, V, sl.ring_k, (int)sizeof(T), (int)sizeof(Rec<T>), GRING,
                                     GREEDY ? (int)sizeof(GAux<T>) : 0);
  unsigned char* wbase = smem + lay.prefix_bytes(L) + (size_t)lay.per_warp * warp;
  Rec<T>* recs = reinterpret_cast<Rec<T>*>(wbase + lay.rec_off);
  int64_t* dmem = reinterpret_cast<int64_t*>(wbase + lay.dmem_off);
  int16_t* cuts_all = reinterpret_cast<int16_t*>(wbase + lay.cuts_off);
  unsigned* cntw = reinterpret_cast<unsigned*>(wbase + lay.cnt_off);  // [chunk][lane]
  // GREEDY statics, structure of arrays [field][chunk][lane] (conflict-free; the
  // GAux struct only fixes the region size)
  int64_t* ga_gate = reinterpret_cast<int64_t*>(wbase + lay.gaux_off);
  int32_t* ga_tF = reinterpret_cast<int32_t*>(ga_gate + V * 32);
  int32_t* ga_tB = ga_tF + V * 32;
  T* ga_pF = reinterpret_cast<T*>(ga_tB + V * 32);
  T* ga_pB = ga_pF + V * 32;
  T* ga_lF = ga_pB + V * 32;  // fp32 ticks only (GAux<float>)
  T* ga_lB = ga_lF + V * 32;
  LaneCold& cold = reinterpret_cast<LaneCold*>(wbase + lay.cold_off)[threadIdx.x & 31];
  cold.idx = 0; cold.slot = 0; cold.busy = 0; cold.key = ~0ull >> 1; cold.invalid = 0; cold.tasks = 0; cold.live = 0;
  cold.pruned = 0;
  T* ring;
  if constexpr (GRING) {
    const size_t gw = (size_t)blockIdx.x * kWarpsPerCta + warp;
    ring = reinterpret_cast<T*>(sl.gring) + gw * 2 * (size_t)sl.ring_k * G * S;
  } else {
    ring = reinterpret_cast<T*>(wbase + lay.ring_off);
  }

  const int g = lane >> sl.log2p2;
  const int d = lane & (p2 - 1);
  const bool dev_lane = d < p;
  const int leader = g * p2;
  const unsigned smask = (p2 == 32) ? FULLMASK : (((1u << p2) - 1u) << leader);
  int16_t* cuts = cuts_all + g * (S + 1);
  const int KM = sl.ring_k - 1;
  const int RS = G * S;             // ring row stride: [dir][slot][g*S + s]
  const int BOFF = sl.ring_k * RS;  // start of the backward direction
  const int tot = m * V;
  const int wup =
      dev_lane ? (V == 1 ? min(m, p - d - 1) : min(tot, 2 * (p - d - 1) + (V - 1) * p)) : 0;
  const int nleft = leader + (d == 0 ? p - 1 : d - 1);  // neighbour devices (wrap)
  const int nright = leader + (d + 1 >= p ? 0 : d + 1);
#define REC(kind, c) recs[((kind) * V + (c)) * 32 + lane]

#define DMEM(kind, c) dmem[((kind) * V + (c)) * 32 + lane]

  // ---- lane / slot state
  bool active = false;  // slot simulates a candidate (uniform within the slot)
  bool done = true;     // this lane has no task left
  int flags = 0;        // slot-uniform F_* bits
  T free_t = 0;
  int64_t dyn = 0, peak = 0, stat = 0;
  T window = INF;
  T w_dm = INF, w_cm = INF;  // fp32 ticks: the window's two terms, added in arrival order
  // fixed orders
  int nF = 0, nB = 0, nW = 0;
  VPos fp, bp, wp;
  fp.reset(); bp.reset(); wp.reset();
  int tk = 2, tc = 0, tj = 0;  // cached next F/B task (tk: 0 F, 1 B, 2 none)
  Rec<T> tr{};
  // GREEDY per-chunk counters and F-gate bytes
  int gF[V], gB[V], gW[V];
  unsigned pleft = 0; // bit c: F-pred of chunk c on the left neighbour; bit V+c: B-pred
  unsigned fitmask = 0, s0mask = 0, lastmask = 0;  // bit c: F fits / stage 0 / stage S-1
  T tstar = 0;        // t* of the slot (non-decreasing, refreshed every 4 rounds)
  bool ts_fresh = true, force_ts = false;  // warp-uniform
  T hF[V], hB[V];     // cached arrival of the F / B head (-1: not yet produced)
  unsigned seen[V];   // produced-count words seen at the last decision
  bool gdirty = true; // the lane's decision must be recomputed
  T g_at = INF;       // cached GREEDY decision: time, kind, chunk, mb, unknown heads
  int g_ak = -1, g_acx = 0, g_aj = 0;
  unsigned g_unk = 0;
#pragma unroll
  for (int c = 0; c < V; ++c) {
    gF[c] = gB[c] = gW[c] = 0;
    hF[c] = -1; hB[c] = -1; seen[c] = 0;
  }
  // work queue: every slot works through runs of consecutive positions
  uint64_t rpos = 0, rend = 0;  // slot-uniform current run
  uint64_t prev_idx = ~0ull - 1; // slot leader: index whose cuts are in smem (none yet)
  int brem = 0;                 // slot leader: remaining L1 radius of that decode
  bool exhausted = false;       // warp-uniform: the launch's positions are all claimed
  unsigned wrounds = 0;
  unsigned ctasks = 0, clive = 0;  // this lane's tasks / live rounds since the last flush
  int ntr = 0;                     // TRACE: tasks recorded for the slot's current candidate
  // TRACE (report mode, R29): append a committed task [start, fin) of (kind,
  // chunk) and its output transfer (latency oc to device tdev, -1: none) to this
  // candidate's device trace
  auto trace_task = [&](T start, T fin, T oc, int tdev, int kind, int chunk, int mb) {
    if constexpr (TRACE) {
      if (ntr < sl.trace_cap) {
        TraceEntry e;
        e.start = to_ticks(start);
        e.fin = to_ticks(fin);
        e.oc = (int32_t)to_ticks(oc);
        e.tgt = tdev;
        e.kind = (int16_t)kind;
        e.stage = (int16_t)stage_of(sl.placement, p, chunk, d);
        e.mb = mb;
        sl.trace[((size_t)cold.slot * p + d) * sl.trace_cap + ntr] = e;
      }
      ++ntr;
    }
  };

  auto next_task = [&]() {
    if constexpr (LISTP) {  // R30: the next task of this device's explicit order (nF = tasks done)
      const uint64_t* off = sl.list_task_off + cold.slot * (uint64_t)(p + 1);
      const uint64_t b = off[d], e = off[d + 1];
      if (b + (uint64_t)nF >= e) { tk = 3; return; }  // list finished
      const adaptis_task t = sl.list_tasks[b + nF];
      tk = t.kind; tc = t.stage / p; tj = t.mb;
      tr = REC(tk, tc);
      return;
    }
    if (nF < tot && (POLICY == ADAPTIS_GPIPE || nF - nB <= wup)) { tk = 0; tc = fp.c; tj = fp.mb(); }
    else if (nB < tot) { tk = 1; tc = V - 1 - bp.c; tj = bp.mb(); }
    else { tk = 2; return; }
    tr = REC(tk, tc);
  };

  // collective: write results of the slots with `fl` set (all lanes execute)
  auto finalize = [&](bool fl) {
    BT busy;
    if constexpr (FP) busy = __longlong_as_double(cold.busy); else busy = cold.busy;
    const uint64_t idx = cold.idx;
    const bool contrib = fl && dev_lane;
    const T mkT = seg_max(contrib ? free_t : (T)0, p2);
    const int64_t mk = to_ticks(mkT);
    const BT sb = seg_sum(contrib ? busy : (BT)0, p2);
    const int64_t Md = stat + peak;
    const int64_t Mmax = seg_max(contrib ? Md : (int64_t)0, p2);
    const bool anyover = (__ballot_sync(FULLMASK, contrib && Md > sl.cap) & smask) != 0;
    int status;
    if (flags & F_PRUNED) status = -3;  // search: cannot beat the incumbent key (exact LB prune)
    else if (flags & F_INVALID) status = ADAPTIS_CAND_INVALID;
    else if (flags & F_OVERFLOW) status = -2;
    else if (FUSED && ((flags & F_PREOVER) || anyover)) status = ADAPTIS_CAND_OVER_CAP;
    else if (flags & F_STUCK) status = ADAPTIS_CAND_STUCK;
    else if (anyover) status = ADAPTIS_CAND_OVER_CAP;
    else status = ADAPTIS_CAND_OK;
    // a candidate whose rings overflowed is re-run by the fallback: its partial
    // tasks are not counted (each candidate's tasks are counted once)
    if (fl) { if (status != -2) cold.tasks += ctasks; cold.live += clive; ctasks = 0; clive = 0; }
    if (fl && d == 0) {
      if (status == -2) {
        const unsigned k = atomicAdd(sl.overflow_count, 1u);
        if (k < sl.overflow_cap) sl.overflow_idx[k] = sl.list_slot ? cold.slot : idx;
      } else {
        if (status == ADAPTIS_CAND_INVALID) ++cold.invalid;
        if (status == -3) ++cold.pruned;
        if (sl.key) {
          if (status == ADAPTIS_CAND_OK) {
            unsigned long long kv;  // order-preserving: fp32 bits of a positive float
            if constexpr (FP) kv = (unsigned long long)__float_as_uint(mkT);
            else kv = (unsigned long long)mk;
            const unsigned long long key = (kv << sl.key_bits) | idx;
            if (key < cold.key) {
              cold.key = key;
              if (sl.prune) atomicMin(sl.key, key);  // share the incumbent at once
            }
          }
        } else {
          const uint64_t o = cold.slot;
          if (sl.out_status) sl.out_status[o] = (uint8_t)status;
          if (sl.out_makespan) sl.out_makespan[o] = status == 0 ? mk : INT64_MAX;
          if (sl.out_makespan_f32) sl.out_makespan_f32[o] = status == 0 ? (float)mkT : INFINITY;
          if (sl.out_peak)
            sl.out_peak[o] = (status == 0 || status == ADAPTIS_CAND_OVER_CAP) ? Mmax : 0;
          if (sl.out_bubble)
            sl.out_bubble[o] =
                status == 0 ? (float)(1.0 - (double)sb / ((double)p * (double)mkT)) : 0.0f;
        }
      }
    }
    if (sl.out_report && contrib && status >= 0) {
      int64_t* rep = sl.out_report + (size_t)cold.slot * 5 * p;
      rep[d] = to_ticks(free_t);
      rep[p + d] = to_ticks(busy);
      rep[2 * p + d] = Md;
      if constexpr (TRACE) sl.trace_n[(size_t)cold.slot * p + d] = ntr;
    }
  };

  bool maint = true;  // warp-uniform: some slot finished, or idle slots can be refilled
  for (;;) {
    // ================= maintenance: finalize finished slots, refill idle ones
    if (maint) {
      maint = false;
      const unsigned live_m = __ballot_sync(FULLMASK, active && !done);
      const bool fin = active && !(live_m & smask);
      const unsigned fin_m = __ballot_sync(FULLMASK, fin);
      if (fin_m) {
        finalize(fin);
        if (fin) active = false;
      }
      const unsigned idle_m = __ballot_sync(FULLMASK, !active);
      const bool runs_left = __any_sync(FULLMASK, rpos < rend);
      if (idle_m && (!exhausted || runs_left)) {
        for (int it = 0; it < 4; ++it) {
          // idle slots without positions claim runs of kRun consecutive positions
          const bool want = !active;
          const unsigned need_m = __ballot_sync(FULLMASK, want && rpos >= rend && d == 0);
          if (need_m && !exhausted) {
            const unsigned nw = __popc(need_m);
            const unsigned rank = __popc(need_m & ((1u << leader) - 1u));
            // run length: kRun, shortened near the end of the launch so that the
            // last runs spread over all slots (tail balance)
            unsigned long long b = 0, run = kRun;
            if (lane == 0) {
              const unsigned long long cur = *(volatile unsigned long long*)sl.cursor;
              const unsigned long long rem = cur < sl.n_pos ? sl.n_pos - cur : 0;
              const unsigned long long fair =
                  rem / ((unsigned long long)gridDim.x * kWarpsPerCta * G * 4);
              run = fair >= (unsigned long long)kRun ? kRun : (fair < 1 ? 1 : fair);
              b = atomicAdd(sl.cursor, (unsigned long long)nw * run);
            }
            b = __shfl_sync(FULLMASK, b, 0);
            run = __shfl_sync(FULLMASK, run, 0);
            if (b + (unsigned long long)nw * run >= sl.n_pos) exhausted = true;
            if (want && rpos >= rend) {
              const uint64_t st = b + (uint64_t)rank * run;
              rpos = st < sl.n_pos ? st : sl.n_pos;
              rend = st + run < sl.n_pos ? st + run : sl.n_pos;
            }
          }
          const bool take = want && rpos < rend;
          if (__ballot_sync(FULLMASK, take) == 0) break;
          const uint64_t mypos = rpos;
          if (take) ++rpos;
          DCHECK(!take || mypos < sl.n_pos, "mypos", mypos);

          // ---- a1 decode: the successor of the previous candidate when the slot
          // moves to the next index, else unranking from scratch
          uint64_t idx = 0;
          if (take) {
            idx = pos_to_index(sl, mypos);
            cold.idx = idx;
            cold.slot = sl.list_slot ? sl.list_slot[mypos] : idx - sl.eval_first;
          }
          DCHECK(!take || (idx >= sl.seg_base && idx < sl.hi), "idx", (long long)idx);
          if (take && d == 0) {
            const int16_t* seed = tab.seeds + sl.group * ADAPTIS_MAX_S;
            if (sl.list_cuts) {  // explicit plan: cuts as given (validity checked below)
              const int16_t* src = sl.list_cuts + (size_t)idx * (ADAPTIS_MAX_S + 1);
              for (int i = 0; i <= S; ++i) cuts[i] = src[i];
            } else if (idx == prev_idx + 1 && S > 1) {
              if (sl.part_mode == ADAPTIS_PART_FULL) colex_next(cuts, S);
              else ball_next(cuts, seed, S - 1, brem);
            } else {
              decode_cuts(tab.binom, tab.ball, tab.seeds, sl.group, sl.part_mode, sl.radius, S, L,
                          idx - sl.seg_base, cuts);
              if (sl.part_mode == ADAPTIS_PART_BALL) {
                int used = 0;
                for (int i = 1; i < S; ++i) {
                  const int di = cuts[i] - seed[i - 1];
                  used += di < 0 ? -di : di;
                }
                brem = sl.radius - used;
              }
            }
            prev_idx = idx;
          }
          __syncwarp();
          // validity (strictly increasing cuts, R19), checked by the slot's lanes.
          // The ballot runs on all lanes: a short-circuited collective diverges the warp.
          bool viol = false;
          if (take && dev_lane) {
#pragma unroll
            for (int c = 0; c < V; ++c) {
              const int s = stage_of(sl.placement, p, c, d);
              viol = viol || cuts[s] >= cuts[s + 1];
            }
          }
          const unsigned viol_m = __ballot_sync(FULLMASK, viol);
          const bool valid = take && !(viol_m & smask);
          __syncwarp();
          const bool lane_on = take && valid && dev_lane;
          if (take) {
            flags = valid ? 0 : F_INVALID;
            free_t = 0; dyn = 0; peak = 0; stat = 0;
            ntr = 0;
          }
          // ---- a2/a3 aggregation into task records
          T dmin = INF, cmin = INF;
          BT busy = 0, wsum = 0;  // wsum: t_W of the device's stages (prune bound)
          int64_t ac[V];
#pragma unroll
          for (int c = 0; c < V; ++c) ac[c] = 0;
          if (lane_on) {
#pragma unroll
            for (int c = 0; c < V; ++c) {
              const int s = stage_of(sl.placement, p, c, d);
              const int a = cuts[s], b = cuts[s + 1];
              DCHECK(s >= 0 && s < S, "stage", s);
              DCHECK(a >= 0 && b <= L && a < b, "cut", a * 100000 + b);
              const BT cF = dsum(kColTF, a, b);
              const BT cB = dsum(kColTB, a, b);
              const BT cW = dsum(kColTW, a, b);
              const int64_t act = pre[kColAct * (L + 1) + b] - pre[kColAct * (L + 1) + a];
              const int64_t sta = pre[kColStash * (L + 1) + b] - pre[kColStash * (L + 1) + a];
              stat += pre[kColWG * (L + 1) + b] - pre[kColWG * (L + 1) + a];
              busy += (BT)m * (cF + cB + cW);
              wsum += cW;
              T oF = 0, oB = 0;
              if (s < S - 1 && dev_of(sl.placement, p, s + 1) != d) {
                oF = lat(b - 1);
                cmin = oF < cmin ? oF : cmin;
              }
              if (s > 0 && dev_of(sl.placement, p, s - 1) != d) {
                oB = lat(a - 1);
                cmin = oB < cmin ? oB : cmin;
              }
              T mn = (T)cF < (T)cB ? (T)cF : (T)cB;
              mn = (T)cW < mn ? (T)cW : mn;
              dmin = mn < dmin ? mn : dmin;
              const int row = g * S + s;
              Rec<T> rf, rb, rw;
              rf.dur = (T)cF; rf.oc = oF;
              rf.in_off = s > 0 ? row : -1;
              rf.out_off = s < S - 1 ? row + 1 : -1;
              rb.dur = (T)(BFUSED ? cB + cW : cB); rb.oc = oB;
              rb.in_off = s < S - 1 ? BOFF + row : -1;
              rb.out_off = s > 0 ? BOFF + row - 1 : -1;
              rw.dur = (T)cW; rw.oc = 0; rw.in_off = -1; rw.out_off = -1;
              REC(0, c) = rf;
              REC(1, c) = rb;
              REC(2, c) = rw;
              if constexpr (!FUSED) {
                DMEM(0, c) = act + sta;
                DMEM(1, c) = BFUSED ? -(act + sta) : -act;
                DMEM(2, c) = -sta;
              }
              ac[c] = act + sta;
              if (c == V - 1) {
                if constexpr (FP) cold.busy = __double_as_longlong(busy); else cold.busy = busy;
              }
              if constexpr (GREEDY) {
                // Lemma 3 refinement: an unknown head F(s, j) waits for F(s-1, j) on the
                // device of stage s-1, which lasts c_F(s-1) and then travels oF(s-1)
                T pf = INF, pb = INF, lf = 0, lb = 0;
                bool fl = true, bl = false;
                if (s > 0 && dev_of(sl.placement, p, s - 1) != d) {
                  const int a0 = cuts[s - 1];
                  if constexpr (FP) { pf = (T)dsum(kColTF, a0, a); lf = lat(a - 1); }
                  else pf = (T)dsum(kColTF, a0, a) + lat(a - 1);
                  fl = dev_of(sl.placement, p, s - 1) == (d == 0 ? p - 1 : d - 1);
                }
                if (s < S - 1 && dev_of(sl.placement, p, s + 1) != d) {
                  const int b1 = cuts[s + 2];
                  if constexpr (FP) { pb = (T)dsum(kColTB, b, b1); lb = lat(b - 1); }
                  else pb = (T)dsum(kColTB, b, b1) + lat(b - 1);
                  bl = dev_of(sl.placement, p, s + 1) == (d == 0 ? p - 1 : d - 1);
                }
                if constexpr (FP) {
                  ga_lF[c * 32 + lane] = lf;
                  ga_lB[c * 32 + lane] = lb;
                }
                // gate is set below, once stat is complete
                ga_pF[c * 32 + lane] = pf;
                ga_pB[c * 32 + lane] = pb;
                ga_tF[c * 32 + lane] =
                    s < S - 1 ? (((leader + dev_of(sl.placement, p, s + 1)) << 3) | ((s + 1) / p)) : -1;
                ga_tB[c * 32 + lane] =
                    s > 0 ? (((leader + dev_of(sl.placement, p, s - 1)) << 3) | ((s - 1) / p)) : -1;
                s0mask = (s0mask & ~(1u << c)) | ((s == 0 ? 1u : 0u) << c);
                lastmask = (lastmask & ~(1u << c)) | ((s == S - 1 ? 1u : 0u) << c);
                hF[c] = s == 0 ? (T)0 : (T)-1;
                hB[c] = s == S - 1 ? (T)0 : (T)-1;
                cntw[c * 32 + lane] = 0;
                pleft = (pleft & ~((1u << c) | (1u << (V + c)))) | ((fl ? 1u : 0u) << c) |
                        ((bl ? 1u : 0u) << (V + c));
              }
            }
          }
          // ---- a4 memory precheck of the fused fixed orders (R16)
          if constexpr (FUSED) {
            if (lane_on) {
              if constexpr (POLICY == ADAPTIS_GPIPE) {
                int64_t A = 0;
#pragma unroll
                for (int c = 0; c < V; ++c) A += ac[c];
                peak = A * m;
              } else {
                peak = megatron_peak<V>(ac, p, m, wup);
              }
            }
            const bool ov = lane_on && stat + peak > sl.cap;
            const unsigned ov_m = __ballot_sync(FULLMASK, ov);
            if (take && valid && (ov_m & smask)) flags |= F_PREOVER;
          }
          if constexpr (GREEDY) {
            const T dm = seg_min_m(dmin, p2, smask), cm = seg_min_m(cmin, p2, smask);
            if (take) {
              window = (cm == INF) ? INF : dm + cm;
              w_dm = dm; w_cm = cm;
              gdirty = true;
#pragma unroll
              tstar = 0;
              fitmask = 0;
              for (int c = 0; c < V; ++c) {
                seen[c] = 0xffffffffu;
                if (lane_on) {
                  const int64_t gate = sl.cap - stat - ac[c];  // cap - stat cannot overflow
                  ga_gate[c * 32 + lane] = gate;
                  fitmask |= (0 <= gate ? 1u : 0u) << c;
                }
              }
            }
          }
          // ---- ring reset for the slots being set up
          if (!GREEDY && take && dev_lane) {
            for (int s = d; s < S; s += p)
              for (int k = 0; k < 2 * sl.ring_k; ++k) ring[(size_t)k * RS + g * S + s] = EMPTY;
          }
          __syncwarp();
          // exact lower-bound prune (search only). Device d's lowest stage is s0 = d
          // (chunk 0 of every placement, R12). Head: d starts no task before F(0..d-1)
          // of some micro-batch ran and travelled, t_F[0, cuts[d]) + the d edge
          // latencies. Tail: every F and B of d ends by the end E of its last B at
          // stage d (an F precedes its B; B(s', j) of a higher stage precedes B(d, j)),
          // and after E that micro-batch's B still runs down stages d-1..0 with the
          // same d latencies, then (split) its W at stage 0. So makespan >= max_d of
          //   fused: head + busy_d + (t_B + t_W)[0, cuts[d]) + lat_d
          //   split: max(head + busy_d, head + m (F + B)_d + t_B[0, cuts[d]) + lat_d
          //              + t_W(stage 0)).
          // A candidate whose (LB << bits | index) exceeds the incumbent key cannot win.
          if constexpr (!FP) {
            if (sl.prune) {
              const int s0 = stage_of(sl.placement, p, 0, d);
              int64_t lk = (lane_on && s0 >= 1) ? (int64_t)lat(cuts[s0] - 1) : (int64_t)0;
              for (int o = 1; o < p2; o <<= 1) {  // segmented inclusive scan: sum of edges 0..d
                const int64_t y = __shfl_up_sync(FULLMASK, lk, o);
                if (d >= o) lk += y;
              }
              int64_t lbd = 0;
              if (lane_on) {
                const int cs = cuts[s0];
                const int64_t head = (int64_t)pre[kColTF * (L + 1) + cs] + lk;
                const int64_t bpre = (int64_t)pre[kColTB * (L + 1) + cs];
                lbd = (int64_t)busy + head;
                if constexpr (BFUSED) {
                  lbd += bpre + (int64_t)pre[kColTW * (L + 1) + cs] + lk;
                } else {
                  const int64_t w0 = (int64_t)pre[kColTW * (L + 1) + cuts[1]];
                  const int64_t alt = (int64_t)busy - (int64_t)m * (int64_t)wsum + head + bpre + lk + w0;
                  lbd = alt > lbd ? alt : lbd;
                }
              }
              const int64_t lb = seg_max(lbd, p2);
              // one read of the incumbent per slot: lanes reading it separately could
              // straddle another warp's atomicMin and split the slot's prune decision
              unsigned long long inc = 0;
              if (d == 0) inc = *(volatile unsigned long long*)sl.key;
              inc = __shfl_sync(FULLMASK, inc, leader);
              if (take && valid && !(flags & F_PREOVER) &
                  ((((unsigned long long)lb << sl.key_bits) | idx) > inc))
                flags |= F_PRUNED;
            }
          }
          // a fused order over the cap is decided without simulating it, except in
          // report launches, whose traces (R29 accounting, the memory timeline,
          // realised lists) cover every plan of status 0 or 2
          const bool survivor = take && valid && !(flags & F_PRUNED) && (TRACE || !(flags & F_PREOVER));
          const unsigned nonsurv_m = __ballot_sync(FULLMASK, take && !survivor);
          if (nonsurv_m) finalize(take && !survivor);
          if (survivor) {
            active = true;
            done = !dev_lane;
            nF = nB = nW = 0;
            fp.reset(); bp.reset(); wp.reset();
#pragma unroll
            for (int c = 0; c < V; ++c) { gF[c] = gB[c] = gW[c] = 0; }
            if constexpr (!GREEDY) { if (dev_lane) next_task(); }
          }
          __syncwarp();
        }
      }
      const unsigned act_m = __ballot_sync(FULLMASK, active);
      const bool runs_any = __any_sync(FULLMASK, rpos < rend);
      const bool more = !exhausted || runs_any;
      if (act_m == 0) {
        if (!more) break;
        maint = true;
        continue;
      }
      maint = (act_m != FULLMASK) && more;  // some slot is still idle
    }

    // ================= a5: one simulation round
    bool progressed = false, blocked = false;
    const bool live = active && !done;
    ++wrounds;
    clive += live ? 1u : 0u;
    if constexpr (!GREEDY) {
      T r = 0;
      int iaddr = -1, oaddr = -1;
      bool ofree = true;
      if (live && tk < 2) {  // phase A: read the input arrival and the output slot
        iaddr = tr.in_off >= 0 ? tr.in_off + (tj & KM) * RS : -1;
        oaddr = tr.out_off >= 0 ? tr.out_off + (tj & KM) * RS : -1;
        DCHECK(iaddr < 2 * sl.ring_k * RS && oaddr < 2 * sl.ring_k * RS, "ring addr", iaddr * 100000 + oaddr);
        DCHECK(tc >= 0 && tc < V && tk >= 0 && tk < 2, "task", tk * 100 + tc);
        r = iaddr >= 0 ? ring[iaddr] : (T)0;
        ofree = oaddr < 0 || ring[oaddr] == EMPTY;
      }
      __syncwarp();
      if (LISTP && live) {  // phase B of an explicit order (R30): W at free_t, F/B when ready
        if (tk == 2) {
          trace_task(free_t, free_t + tr.dur, (T)0, -1, 2, tc, tj);
          free_t += tr.dur;
          dyn += DMEM(2, tc);
          ++nF; ++ctasks;
          progressed = true;
          next_task();
        } else if (tk < 2) {
          bool xgo = r >= 0;
          if (xgo && !ofree) { blocked = true; xgo = false; }
          if (xgo) {
            const T fin = (free_t > r ? free_t : r) + tr.dur;
            if constexpr (TRACE) {
              const int s0 = stage_of(sl.placement, p, tc, d);
              const int s1 = tk == 0 ? s0 + 1 : s0 - 1;
              int tdev = (oaddr >= 0 && s1 >= 0 && s1 < S) ? dev_of(sl.placement, p, s1) : -1;
              if (tdev == d) tdev = -1;
              trace_task(fin - tr.dur, fin, tdev >= 0 ? tr.oc : (T)0, tdev, tk, tc, tj);
            }
            free_t = fin;
            if (oaddr >= 0) ring[oaddr] = fin + tr.oc;
            if (iaddr >= 0) ring[iaddr] = EMPTY;
            dyn += DMEM(tk, tc);
            if (tk == 0) peak = dyn > peak ? dyn : peak;
            ++nF; ++ctasks;
            progressed = true;
            next_task();
          }
        }
        if (tk == 3) done = true;
      } else if (live) {  // phase B: execute
        if constexpr (ZB) {
          // R13: (i) memory-forced W before an F that does not fit, (ii) W fill while free < r.
          // ADAPTIS_ZB_WFILL_ONE: one W per lane and round (the rest in later rounds),
          // so that lanes with long W runs do not hold the warp in this loop
          for (int wi = 0; !ADAPTIS_ZB_WFILL_ONE || wi < 1; ++wi) {
            if (nW >= nB) break;
            bool runW;
            if (tk == 2) runW = true;
            else if (tk == 0 && stat + dyn + DMEM(0, tc) > sl.cap) runW = true;
            else runW = r >= 0 && free_t < r;
            if (!runW) break;
            const int c = V - 1 - wp.c;
            trace_task(free_t, free_t + REC(2, c).dur, (T)0, -1, 2, c, wp.mb());
            free_t += REC(2, c).dur;
            dyn += DMEM(2, c);
            ++nW; wp.next(p, V); ++ctasks;
            progressed = true;
          }
        }
        bool xgo = tk < 2 && r >= 0;
        if constexpr (ZB) {
          xgo = xgo && (nW >= nB || free_t >= r);
          // an F that does not fit waits while Ws remain to be drained (R13 (i))
          if (tk == 0 && nW < nB && stat + dyn + DMEM(0, tc) > sl.cap) xgo = false;
        }
        if (xgo && !ofree) { blocked = true; xgo = false; }
        if (xgo) {
          const T fin = (free_t > r ? free_t : r) + tr.dur;
          if constexpr (TRACE) {
            const int s0 = stage_of(sl.placement, p, tc, d);
            const int s1 = tk == 0 ? s0 + 1 : s0 - 1;
            int tdev = (oaddr >= 0 && s1 >= 0 && s1 < S) ? dev_of(sl.placement, p, s1) : -1;
            if (tdev == d) tdev = -1;
            trace_task(fin - tr.dur, fin, tdev >= 0 ? tr.oc : (T)0, tdev, tk, tc, tj);
          }
          free_t = fin;
          if (oaddr >= 0) ring[oaddr] = fin + tr.oc;
          if (iaddr >= 0) ring[iaddr] = EMPTY;
          if constexpr (ZB) {
            dyn += DMEM(tk, tc);
            if (tk == 0) {
              peak = dyn > peak ? dyn : peak;
              if (sl.key && stat + dyn > sl.cap) done = true;  // search: Eq. 2 already violated
            }
          }
          if (tk == 0) { ++nF; fp.next(p, V); } else { ++nB; bp.next(p, V); }
          ++ctasks;
          progressed = true;
          next_task();
        }
        if (tk == 2 && (!ZB || nW == tot)) done = true;
      }
    } else {
      // ---- GREEDY (R14) in bounded-lag rounds (Lemma 3 with per-head bounds).
      // Rings are >= m deep (every slot written once per candidate); producers
      // bump the consumer's produced-count word, consumers read a slot once it
      // exists and cache the head's arrival time. A lane's decision only changes
      // after its own commit or a new arrival, so it is cached otherwise.
      T& at = g_at;
      int& ak = g_ak;
      auto decide = [&](bool force) {
        unsigned cw[V];
        bool dirty = gdirty || force;
#pragma unroll
        for (int c = 0; c < V; ++c) {
          cw[c] = ((volatile unsigned*)cntw)[c * 32 + lane];
          dirty = dirty || cw[c] != seen[c];
        }
        // a lane-local early exit only saves warp instructions when every lane
        // takes it: measured worth it at V = 1 only (ADAPTIS_GREEDY_ALWAYS_DECIDE)
        if (!kAlwaysDecide && !dirty) return;
        gdirty = false;
        at = INF; ak = -1; g_unk = 0;
        unsigned okF = 0, okB = 0, okW = 0;
        T rmin = INF;
#pragma unroll
        for (int c = 0; c < V; ++c) {
          seen[c] = cw[c];
          if (hF[c] < 0 && gF[c] < (int)(cw[c] & 0xffffu))
            hF[c] = ring[REC(0, c).in_off + (gF[c] & KM) * RS];  // plain load: __syncwarp orders it
          if (hB[c] < 0 && gB[c] < (int)(cw[c] >> 16))
            hB[c] = ring[REC(1, c).in_off + (gB[c] & KM) * RS];
          if (gF[c] < m && ((fitmask >> c) & 1u)) {
            if (hF[c] >= 0) { okF |= 1u << c; rmin = hF[c] < rmin ? hF[c] : rmin; }
            else g_unk |= 1u << c;
          }
          if (gB[c] < gF[c]) {
            if (hB[c] >= 0) { okB |= 1u << c; rmin = hB[c] < rmin ? hB[c] : rmin; }
            else g_unk |= 1u << (V + c);
          }
          if (gW[c] < gB[c]) { okW |= 1u << c; rmin = 0; }
        }
        if (rmin != INF) {
          at = free_t > rmin ? free_t : rmin;
          // key (kind F < B < W, mb, stage); stage order == chunk order
          unsigned kF = 0xffffffffu, kB = 0xffffffffu, kW = 0xffffffffu;
#pragma unroll
          for (int c = 0; c < V; ++c) {
            const unsigned xf = ((unsigned)gF[c] << 2) | c, xb = ((unsigned)gB[c] << 2) | c,
                           xw = ((unsigned)gW[c] << 2) | c;
            if (((okF >> c) & 1u) && hF[c] <= at) kF = xf < kF ? xf : kF;
            if (((okB >> c) & 1u) && hB[c] <= at) kB = xb < kB ? xb : kB;
            if ((okW >> c) & 1u) kW = xw < kW ? xw : kW;
          }
          const unsigned k = kF != 0xffffffffu ? kF : (kB != 0xffffffffu ? kB : kW);
          ak = kF != 0xffffffffu ? 0 : (kB != 0xffffffffu ? 1 : 2);
          g_acx = (int)(k & 3u);
          g_aj = (int)(k >> 2);
        }
      };
      if (live) {
        decide(false);
      } else {
        at = INF; ak = -1;
      }
      // Every unscheduled task starts at >= t*, and a neighbour n starts every
      // further task at >= min(at_n, t* + window) for the rest of this round. An
      // unknown head therefore cannot become ready before that start plus its
      // predecessor's duration and latency; a decision below every such bound is
      // final (DESIGN.md Lemma 3').
      ts_fresh = kTstarEvery == 1 || (wrounds % kTstarEvery) == 0 || force_ts;
      if (ts_fresh) {  // t* is non-decreasing, so a stale value stays a valid (looser) bound
        const T ts = seg_min_m(at, p2, smask);
        if (active) tstar = ts > tstar ? ts : tstar;
        force_ts = false;
      }
      const T atl = __shfl_sync(FULLMASK, at, nleft);
      const T atr = __shfl_sync(FULLMASK, at, nright);
      T bound = INF;
      T tw;
      if constexpr (FP) tw = sat_add(sat_add(tstar, w_dm), w_cm);  // rounded as an arrival is
      else tw = sat_add(tstar, window);
      const T nl = atl < tw ? atl : tw;
      const T nr = atr < tw ? atr : tw;
      auto tighten = [&]() {
#pragma unroll
        for (int c = 0; c < V; ++c) {
          if (g_unk & (1u << c)) {
            T x = sat_add((pleft >> c) & 1u ? nl : nr, ga_pF[c * 32 + lane]);
            if constexpr (FP) x = sat_add(x, ga_lF[c * 32 + lane]);
            bound = x < bound ? x : bound;
          }
          if (g_unk & (1u << (V + c))) {
            T x = sat_add((pleft >> (V + c)) & 1u ? nl : nr, ga_pB[c * 32 + lane]);
            if constexpr (FP) x = sat_add(x, ga_lB[c * 32 + lane]);
            bound = x < bound ? x : bound;
          }
        }
      };
      if (g_unk) tighten();
      __syncwarp();
      // commit while the decision stays below the bound: the bound stays a lower
      // bound on every new arrival for the rest of the round once the terms of
      // newly unknown heads are added (DESIGN.md Lemma 3')
      for (int kc = 0; kc < kGreedyCommits && live && !done && ak >= 0 && at < bound; ++kc) {
        const int acx = g_acx, aj = g_aj;
        const Rec<T> rc = REC(ak, acx);
        const T fin = at + rc.dur;
        if constexpr (TRACE) {
          const int tg = ak == 0 ? ga_tF[acx * 32 + lane] : (ak == 1 ? ga_tB[acx * 32 + lane] : -1);
          const int tdev = tg >= 0 ? (tg >> 3) - leader : -1;
          trace_task(at, fin, (tdev >= 0 && tdev != d) ? rc.oc : (T)0, tdev == d ? -1 : tdev, ak, acx, aj);
        }
        free_t = fin;
        dyn += DMEM(ak, acx);
        if (ak == 0) peak = dyn > peak ? dyn : peak;
        int tgt = -1;
        const int dir = ak;
        if (ak == 0) tgt = ga_tF[acx * 32 + lane];
        else if (ak == 1) tgt = ga_tB[acx * 32 + lane];
#pragma unroll
        for (int c = 0; c < V; ++c) {
          if (c == acx) {
            if (ak == 0) {
              ++gF[c];
              hF[c] = gF[c] < m && ((s0mask >> c) & 1u) ? (T)0 : (T)-1;
            } else if (ak == 1) {
              ++gB[c];
              hB[c] = ((lastmask >> c) & 1u) ? (T)0 : (T)-1;
            } else {
              ++gW[c];
            }
          }
        }
        fitmask = 0;  // dyn changed: refresh the Eq. 2 gates
#pragma unroll
        for (int c = 0; c < V; ++c) fitmask |= (dyn <= ga_gate[c * 32 + lane] ? 1u : 0u) << c;
        if (tgt >= 0) {  // publish the arrival, then count it for the consumer
          ring[rc.out_off + (aj & KM) * RS] = fin + rc.oc;
          if (kGreedyCommits > 1) __threadfence_block();  // readers within this round
          atomicAdd(&cntw[(tgt & 7) * 32 + (tgt >> 3)], dir == 1 ? 0x10000u : 1u);
        }
        bool all = true;
#pragma unroll
        for (int c = 0; c < V; ++c) all = all && gW[c] == m;
        done = all;
        gdirty = true;
        ++ctasks;
        progressed = true;
        if (kGreedyCommits > 1 && !done && kc + 1 < kGreedyCommits) {
          decide(true);
          if (g_unk) tighten();
        }
      }
    }
    __syncwarp();
    // ---- per-slot bookkeeping: a slot whose lanes are all done finishes; a live
    // slot in which no lane progressed is deadlocked (stuck, or rings too shallow)
    {
      const unsigned prog_m = __ballot_sync(FULLMASK, progressed);
      const unsigned live_m = __ballot_sync(FULLMASK, active && !done);
      const bool slot_live = (live_m & smask) != 0;
      const bool stall = active && slot_live && !(prog_m & smask);
      if (__ballot_sync(FULLMASK, stall || (active && !slot_live))) {
        const unsigned blk_m = __ballot_sync(FULLMASK, blocked);
        if (GREEDY && !ts_fresh && __ballot_sync(FULLMASK, stall)) {
          force_ts = true;  // progress is only guaranteed with a fresh t*: retry once
        } else if (stall) {
          flags |= (blk_m & smask) ? F_OVERFLOW : F_STUCK;
          done = true;
        }
        maint = true;
      }
    }
  }
#undef REC
#undef DMEM

  // ---- a7 argmin: warp min -> one atomicMin per warp; counters
  unsigned long long wkey = cold.key, winvalid = cold.invalid, wtasks = cold.tasks + ctasks,
                     wlive = cold.live + clive, wpruned = cold.pruned;
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long x = __shfl_xor_sync(FULLMASK, wkey, o);
    wkey = x < wkey ? x : wkey;
    winvalid += __shfl_xor_sync(FULLMASK, winvalid, o);
    wtasks += __shfl_xor_sync(FULLMASK, wtasks, o);
    wlive += __shfl_xor_sync(FULLMASK, wlive, o);
    wpruned += __shfl_xor_sync(FULLMASK, wpruned, o);
  }
  if (lane == 0) {
    if (sl.key && wkey != (~0ull >> 1)) atomicMin(sl.key, wkey);
    if (winvalid) atomicAdd(sl.n_invalid, winvalid);
    if (wtasks) atomicAdd(sl.n_tasks, wtasks);
    if (wpruned) atomicAdd(sl.n_pruned, wpruned);
    if (wrounds) { atomicAdd(&sl.n_rounds[0], (unsigned long long)wrounds); atomicAdd(&sl.n_rounds[1], wlive); }
  }
}


using KFn = void (*)(const DevTables, const SegLaunch);
// per-policy kernel pickers (adaptis_inst_<policy>.cu)
KFn pick_policy_gpipe(int tick, int v, bool fb, bool tr);
KFn pick_policy_onef1b(int tick, int v, bool fb, bool tr);
KFn pick_policy_zb(int tick, int v, bool fb, bool tr);
KFn pick_policy_greedy(int tick, int v, bool fb, bool tr);
KFn pick_policy_list(int tick, int v, bool fb, bool tr, bool fused);

}  // namespace adaptis
