// adaptis_seqg.cu — the GREEDY policy (R14) as one exact event loop per
// thread: 32 candidates per warp, each simulated by the global event loop of
// Alg. 1 Step 3 in strict time order.
//
// Why a thread per candidate. The lane-per-device kernel (adaptis_seg.cuh)
// advances a candidate in bounded-lag rounds: every round all p lanes decide,
// reduce t*, exchange bounds and vote, and 55-67 % of them commit a task. That
// is ~16 warp-instructions per task. Here one thread commits exactly one task
// per step, with no shuffles, votes or bounds: a step is the argmin over the
// devices' cached decisions (at << 4 | d), the commit, and the re-decision of
// the two devices whose inputs changed (the committing device and the
// consumer of its output). All candidates of a segment have the same task
// count S * m * 3, so the 32 threads of a warp step in lockstep.
//
// Exact state compression (DESIGN.md §4 "Sequential GREEDY kernel"). In a
// time-ordered event loop every pending task starts at >= the current event
// time t. An item whose arrival A <= t is therefore interchangeable with t
// for its consumer's decision: at = max(free, min ready) and the set of tasks
// ready by `at` are unchanged when A is replaced by any X with A <= X <= at
// (if free >= t both give `free`; if free < t then at >= t >= A forces A = t).
// So an edge keeps the exact arrival times of its last K produced items only;
// an older unconsumed item is known to have arrived. A producer overwriting
// the slot of an unconsumed item whose arrival is still in the future marks
// the candidate OVERFLOW, and the exact global-ring kernel re-runs it. With
// the configs' tables (latency 40 ticks, stage tasks >= ~600 ticks) an edge has
// at most 2 future arrivals, so K = 2 never overflows there.
//
// Ties. Devices with the same decision time are independent (a commit at t
// produces arrivals > t, which change neither the other device's decision time
// nor the set of its tasks ready by t), so the order among them does not
// change the result; the key breaks them by device.
//
// Layout. All per-candidate state lives in shared memory as [field][lane]
// words (conflict-free for any per-lane index): per device the cached key
// (at << 4 | d), free << 4 | decision, room = cap - static - dynamic bytes
// (and its minimum, for M_d); per stage the counters gF | gB << 8 | gW << 16,
// the durations and the latency of its output edge (t_F | t_B << 16 and
// t_W | latency << 16; a stage with a duration >= 2^16 goes to the fallback),
// act + stash bytes, act bytes (40 bits: the low word and a byte beside the
// counters), and the K-slot arrival rings of its F and B inputs.
#include "adaptis_seg.cuh"

namespace adaptis {

#ifndef ADAPTIS_SEQG_K
#define ADAPTIS_SEQG_K 2
#endif
constexpr int kSeqK = ADAPTIS_SEQG_K;   // exact arrival slots per edge (power of two)
constexpr uint32_t kSeqInf = 0xffffffffu;

// shared-memory rows of one lane (a row is 32 lanes x 4 or 8 bytes)
struct SeqLayout {
  int key, fd, cnt, dur, actlo, rf, rb, n32;  // u32 rows
  int room, minroom, as, n64;                 // u64 rows
};
ADAPTIS_LAYOUT_HD constexpr SeqLayout seq_layout(int S, int P2, bool search) {
  SeqLayout l{};
  int r = 0;
  l.key = r; r += P2;
  l.fd = r; r += P2;
  l.cnt = r; r += S + 2;  // guard rows for stages -1 and S; bits 24-31: act bytes >> 32
  l.dur = r; r += 2 * S;  // t_F | t_B << 16, t_W | latency of edge (s, s+1) << 16
  l.actlo = r; r += S;    // act bytes, low 32 bits
  l.rf = r; r += kSeqK * S;
  l.rb = r; r += kSeqK * S;
  l.n32 = (r + 1) & ~1;  // keep the u64 rows 8-byte aligned
  r = 0;
  l.room = r; r += P2;      // cap - static - dynamic bytes
  l.minroom = r; r += search ? 0 : P2;  // its minimum (eval mode: M_d = cap - minroom)
  l.as = r; r += S;
  l.n64 = r;
  return l;
}
ADAPTIS_LAYOUT_HD constexpr size_t seqg_smem_bytes(int S, int p, bool search) {
  return (size_t)32 * (4 * seq_layout(S, p, search).n32 + 8 * seq_layout(S, p, search).n64);
}
// one-warp CTAs; the register cap follows the CTAs that shared memory admits
// per SM (228 KB, 1 KB reserved per CTA), rounded up to a multiple of 4: a
// warp's registers come from one of the 4 SM sub-partitions (16 K each), so n
// warps per SM need 16384 / ceil(n / 4) registers per warp (at most 20 warps)
template <int V, int P, bool SEARCH>
struct SeqOcc {
  static constexpr int by_smem = (int)((228 * 1024) / (seqg_smem_bytes(V * P, P, SEARCH) + 1024));
  static constexpr int r4 = (by_smem + 3) & ~3;
  static constexpr int value = r4 < 4 ? 4 : (r4 > 20 ? 20 : r4);
};

// placement of stage s = c * P + j (R12), compile-time P (a power of two)
template <int PLC, int P>
__device__ __forceinline__ int sq_stage(int c, int d) {
  if constexpr (PLC == ADAPTIS_SEQ) return d;
  else if constexpr (PLC == ADAPTIS_INTERLEAVED) return c * P + d;
  else return c * P + ((c & 1) ? P - 1 - d : d);
}
template <int PLC, int P>
__device__ __forceinline__ int sq_dev(int s) {
  if constexpr (PLC == ADAPTIS_SEQ) return s;
  else if constexpr (PLC == ADAPTIS_INTERLEAVED) return s & (P - 1);
  else { const int j = s & (P - 1); return ((s / P) & 1) ? P - 1 - j : j; }
}

template <int V, int P, int PLC, bool SEARCH>
__global__ void __launch_bounds__(32, (SeqOcc<V, P, SEARCH>::value))
seqg_kernel(const DevTables tab, const SegLaunch sl) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int S = V * P;
  const int lane = threadIdx.x & 31;
  const int L = sl.L, m = sl.m;
  const SeqLayout lay = seq_layout(S, P, SEARCH);
  // one pointer per field region (the regions are disjoint)
  uint32_t* __restrict__ w32 = reinterpret_cast<uint32_t*>(smem);
  int64_t* __restrict__ w64 = reinterpret_cast<int64_t*>(smem + (size_t)128 * lay.n32);
  uint32_t* __restrict__ rKEY = w32 + lay.key * 32 + lane;
  uint32_t* __restrict__ rFD = w32 + lay.fd * 32 + lane;
  uint32_t* __restrict__ rCNT = w32 + lay.cnt * 32 + lane;
  uint32_t* __restrict__ rDUR = w32 + lay.dur * 32 + lane;
  uint32_t* __restrict__ rRF = w32 + lay.rf * 32 + lane;
  uint32_t* __restrict__ rRB = w32 + lay.rb * 32 + lane;
  int64_t* __restrict__ rROOM = w64 + lay.room * 32 + lane;
  int64_t* __restrict__ rMINROOM = w64 + lay.minroom * 32 + lane;
  int64_t* __restrict__ rAS = w64 + lay.as * 32 + lane;
  uint32_t* __restrict__ rACTLO = w32 + lay.actlo * 32 + lane;
#define KEY(d) rKEY[(d) * 32]
#define FD(d) rFD[(d) * 32]
#define CNT(s) rCNT[((s) + 1) * 32]
#define DURFB(s) rDUR[(s) * 32]
#define DURWL(s) rDUR[(S + (s)) * 32]
#define RF(k, s) rRF[((k) * S + (s)) * 32]
#define RB(k, s) rRB[((k) * S + (s)) * 32]
#define ROOM(d) rROOM[(d) * 32]
#define MINROOM(d) rMINROOM[(d) * 32]
#define AS(s) rAS[(s) * 32]
#define ACTLO(s) rACTLO[(s) * 32]
  const int64_t* pre = tab.pre;  // [kNumCols][L + 1] prefix sums (global, read-only)
  auto PRE = [&](int col, int row) -> int64_t { return __ldg(pre + (size_t)col * (L + 1) + row); };

  // GREEDY decision of device d at event time tnow (R14): candidates are the
  // next F of each own stage if it fits under Eq. 2, the head B whose F is
  // done, the head W whose B is done; at = max(free, earliest ready); among
  // the tasks ready by `at` the smallest (kind F < B < W, mb, stage) wins.
  // Branch-free: every load is in bounds and selected afterwards. The guard
  // rows CNT(-1) (255 F items "produced" into stage 0) and CNT(S) (255 B items
  // into stage S-1) make the input-less heads F(0, j) and B(S-1, j) (ready by
  // the device's own free time) count as arrived: they take the current event
  // time, which the compression argument above admits for any X with
  // ready <= X <= the device's next action time.
  // The decision is split into its loads and its arithmetic so that the two
  // decisions of a step (the committing device and the consumer) issue their
  // shared-memory loads back to back and overlap their latencies; the free
  // time comes in a register (the committer's is its finish time).
  struct DecIn {
    uint32_t free_t, cnt[V], cp[V], cn[V], sF[V], sB[V];
    int64_t room, as[V];
  };
  auto dec_load = [&](int d, uint32_t free_t, DecIn& in) {
    in.free_t = free_t;
    in.room = ROOM(d);  // F of stage s fits iff act + stash <= room
#pragma unroll
    for (int c = 0; c < V; ++c) {
      const int s = sq_stage<PLC, P>(c, d);
      in.cnt[c] = CNT(s); in.cp[c] = CNT(s - 1); in.cn[c] = CNT(s + 1);
      in.as[c] = AS(s);
    }
#pragma unroll
    for (int c = 0; c < V; ++c) {
      const int s = sq_stage<PLC, P>(c, d);
      in.sF[c] = RF(in.cnt[c] & (kSeqK - 1), s);
      in.sB[c] = RB((in.cnt[c] >> 8) & (kSeqK - 1), s);
    }
  };
  auto dec_compute = [&](int d, const DecIn& in, uint32_t tnow) {
    uint32_t rf[V], rb[V], rw[V], gf[V], gb[V], gw[V];
    uint32_t rmin = kSeqInf;
#pragma unroll
    for (int c = 0; c < V; ++c) {
      const uint32_t cnt = in.cnt[c];
      const uint32_t gF = cnt & 255u, gB = (cnt >> 8) & 255u, gW = (cnt >> 16) & 255u;
      const uint32_t prodF = in.cp[c] & 255u;          // F items produced into s
      const uint32_t prodB = (in.cn[c] >> 8) & 255u;   // B items produced into s
      const uint32_t aF = gF + kSeqK >= prodF ? in.sF[c] : tnow;
      const uint32_t aB = gB + kSeqK >= prodB ? in.sB[c] : tnow;
      const bool okF = gF < (uint32_t)m && gF < prodF && in.as[c] <= in.room;
      const bool okB = gB < gF && gB < prodB;
      rf[c] = okF ? aF : kSeqInf;
      rb[c] = okB ? aB : kSeqInf;
      rw[c] = gW < gB ? 0u : kSeqInf;
      gf[c] = gF; gb[c] = gB; gw[c] = gW;
      rmin = min(rmin, min(rf[c], min(rb[c], rw[c])));
    }
    const uint32_t at = max(in.free_t, rmin);
    // the smallest (kind, mb, stage) among the tasks ready by `at`: kind << 10 | mb << 2 | chunk
    uint32_t best = kSeqInf;
#pragma unroll
    for (int c = 0; c < V; ++c) {
      best = min(best, rf[c] <= at ? ((gf[c] << 2) | (uint32_t)c) : kSeqInf);
      best = min(best, rb[c] <= at ? ((1u << 10) | (gb[c] << 2) | (uint32_t)c) : kSeqInf);
      best = min(best, rw[c] <= at ? ((2u << 10) | (gw[c] << 2) | (uint32_t)c) : kSeqInf);
    }
    KEY(d) = rmin == kSeqInf ? kSeqInf : ((at << 4) | (uint32_t)d);
    FD(d) = (in.free_t << 4) | ((best >> 10) & 3u) | ((best & 3u) << 2);
  };
  auto decide = [&](int d, uint32_t free_t, uint32_t tnow) {
    DecIn in;
    dec_load(d, free_t, in);
    dec_compute(d, in, tnow);
  };

  unsigned long long best_key = ~0ull >> 1, n_inv = 0, n_pr = 0, n_tasks = 0;
  int16_t cuts[ADAPTIS_MAX_S + 1];
  const int16_t* seed = tab.seeds + sl.group * ADAPTIS_MAX_S;
  uint64_t rpos = 0, rend = 0, prev_idx = ~0ull - 1;
  int brem = 0;
  bool exhausted = false;
  const int T = S * m * 3;  // tasks per candidate (split policy)

  for (;;) {
    // ---- setup: every lane looks for its next candidate to simulate (a1-a4);
    // invalid decodes and pruned candidates are finalised here
    bool have = false, wide = false;
    uint64_t idx = 0, slot = 0;
    for (;;) {
      const bool need = !have && !(exhausted && rpos >= rend);
      const unsigned need_m = __ballot_sync(FULLMASK, need);
      if (!need_m) break;
      // lanes whose runs are empty claim new runs with one atomicAdd
      const unsigned claim_m = __ballot_sync(FULLMASK, need && rpos >= rend);
      if (claim_m && !exhausted) {
        const unsigned nw = __popc(claim_m);
        const unsigned rank = __popc(claim_m & ((1u << lane) - 1u));
        unsigned long long b = 0, run = kRun;
        if (lane == 0) {
          const unsigned long long cur = *(volatile unsigned long long*)sl.cursor;
          const unsigned long long rem = cur < sl.n_pos ? sl.n_pos - cur : 0;
          const unsigned long long fair = rem / ((unsigned long long)gridDim.x * 32 * 4);
          run = fair >= (unsigned long long)kRun ? kRun : (fair < 1 ? 1 : fair);
          b = atomicAdd(sl.cursor, (unsigned long long)nw * run);
        }
        b = __shfl_sync(FULLMASK, b, 0);
        run = __shfl_sync(FULLMASK, run, 0);
        if (b + (unsigned long long)nw * run >= sl.n_pos) exhausted = true;
        if (need && rpos >= rend) {
          const uint64_t st = b + (uint64_t)rank * run;
          rpos = st < sl.n_pos ? st : sl.n_pos;
          rend = st + run < sl.n_pos ? st + run : sl.n_pos;
        }
      }
      if (!need || rpos >= rend) continue;
      const uint64_t pos = rpos++;
      idx = pos_to_index(sl, pos);
      slot = sl.list_slot ? sl.list_slot[pos] : idx - sl.eval_first;
      // a1: successor of the previous index of this lane's run, else unranking
      if (idx == prev_idx + 1 && S > 1) {
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
      bool valid = true;
      for (int s = 0; s < S; ++s) valid = valid && cuts[s] < cuts[s + 1];
      if (!valid) {
        ++n_inv;
        if (!SEARCH) {
          if (sl.out_status) sl.out_status[slot] = ADAPTIS_CAND_INVALID;
          if (sl.out_makespan_f32) sl.out_makespan_f32[slot] = INFINITY;
          if (sl.out_makespan) sl.out_makespan[slot] = INT64_MAX;
          if (sl.out_peak) sl.out_peak[slot] = 0;
          if (sl.out_bubble) sl.out_bubble[slot] = 0.0f;
        }
        continue;
      }
      // a2/a3: stage sums by prefix differences, device statics
#pragma unroll
      for (int d = 0; d < P; ++d) { ROOM(d) = sl.cap; FD(d) = 0; }
      wide = false;
      // prefix differences with the running prefix carried (one gather per column and stage)
      int64_t pv[kNumCols];
#pragma unroll
      for (int col = 0; col < kNumCols; ++col) pv[col] = PRE(col, cuts[0]);
      for (int s = 0; s < S; ++s) {
        const int a = cuts[s], b = cuts[s + 1];
        const int ds = sq_dev<PLC, P>(s);
        int64_t dv[kNumCols];
#pragma unroll
        for (int col = 0; col < kNumCols; ++col) {
          const int64_t x = PRE(col, b);
          dv[col] = x - pv[col];
          pv[col] = x;
        }
        const int64_t act = dv[kColAct];
        AS(s) = act + dv[kColStash];
        ROOM(ds) -= dv[kColWG];  // cap - static (cannot overflow: static >= 0)
        const int64_t tf = dv[kColTF], tb = dv[kColTB], tw = dv[kColTW];
        // 16-bit durations and 40-bit act bytes; a wider stage sends the candidate to the fallback
        wide = wide || tf >= 65536 || tb >= 65536 || tw >= 65536 || act >= (1ll << 40);
        // the latency of edge (s, s+1) (R3-R6: 0 between stages of one device)
        // serves F(s) -> F(s+1) and B(s+1) -> B(s)
        const uint32_t lf = (s < S - 1 && sq_dev<PLC, P>(s + 1) != ds) ? (uint32_t)tab.comm[b - 1] : 0u;
        DURFB(s) = (uint32_t)tf | ((uint32_t)tb << 16);
        DURWL(s) = (uint32_t)tw | (lf << 16);
        ACTLO(s) = (uint32_t)act;
        CNT(s) = (uint32_t)((uint64_t)act >> 32) << 24;  // 40-bit act: its high byte above the counters
      }
      if (!SEARCH) {
#pragma unroll
        for (int d = 0; d < P; ++d) MINROOM(d) = ROOM(d);  // M_d = static + peak dynamic = cap - min room
      }
      CNT(-1) = 255u;       // guard: stage 0's F input is always there
      CNT(S) = 255u << 8;   // guard: stage S-1's B input is always there
      // exact lower-bound prune (search): the bound of adaptis_seg.cuh, per
      // device d with lowest stage d: head = t_F[0, cuts[d]) + the d edge
      // latencies; split: max(head + busy_d, head + m (F + B)_d + t_B[0, cuts[d])
      // + latencies + t_W(stage 0)); a candidate whose (LB << bits | index)
      // exceeds the incumbent key cannot win
      if (SEARCH && sl.prune) {
        int64_t lk = 0, lb = 0;
        const int64_t w0 = PRE(kColTW, cuts[1]);
        for (int d = 0; d < P; ++d) {
          if (d >= 1) lk += (int64_t)tab.comm[cuts[d] - 1];
          int64_t busy = 0, wsum = 0;
#pragma unroll
          for (int c = 0; c < V; ++c) {
            const int s = sq_stage<PLC, P>(c, d);
            const int a = cuts[s], b = cuts[s + 1];
            const int64_t cw = PRE(kColTW, b) - PRE(kColTW, a);
            busy += (int64_t)m * ((PRE(kColTF, b) - PRE(kColTF, a)) + (PRE(kColTB, b) - PRE(kColTB, a)) + cw);
            wsum += cw;
          }
          const int64_t head = PRE(kColTF, cuts[d]) + lk;
          int64_t lbd = busy + head;
          const int64_t alt = busy - (int64_t)m * wsum + head + PRE(kColTB, cuts[d]) + lk + w0;
          lbd = alt > lbd ? alt : lbd;
          lb = lbd > lb ? lbd : lb;
        }
        const unsigned long long inc = *(volatile unsigned long long*)sl.key;
        if ((((unsigned long long)lb << sl.key_bits) | idx) > inc) { ++n_pr; continue; }
      }
#pragma unroll
      for (int d = 0; d < P; ++d) decide(d, 0u, 0u);
      have = true;
    }
    if (!__any_sync(FULLMASK, have)) break;

    // ---- a5: the event loop, one committed task per step (all lanes in lockstep)
    bool alive = have && !wide, stuck = false, overflow = have && wide;
    for (int t = 0; t < T; ++t) {
      if (alive) {
        uint32_t kmin = KEY(0);
#pragma unroll
        for (int d = 1; d < P; ++d) kmin = min(kmin, KEY(d));
        if (kmin == kSeqInf) {
          stuck = true;  // tasks remain but no device can ever act (R14: stuck)
          alive = false;
        } else {
          const int d = (int)(kmin & 15u);
          const uint32_t at = kmin >> 4;
          const uint32_t dec = FD(d) & 15u;
          const int kind = (int)(dec & 3u), c = (int)(dec >> 2);
          const int s = sq_stage<PLC, P>(c, d);
          const uint32_t cnt = CNT(s);
          const int sh = 8 * kind;
          const uint32_t j = (cnt >> sh) & 255u;
          const uint32_t fb = DURFB(s);
          const uint32_t wl = DURWL(s);
          const uint32_t dur = kind == 0 ? (fb & 0xffffu) : (kind == 1 ? (fb >> 16) : (wl & 0xffffu));
          const int64_t ac = (int64_t)(((uint64_t)(cnt >> 24) << 32) | ACTLO(s));
          const uint32_t fin = at + dur;
          // R16: act + stash at F start; act freed at B end, stash at W end
          const int64_t as = AS(s);
          const int64_t room = ROOM(d) - (kind == 0 ? as : (kind == 1 ? -ac : ac - as));
          // the output item: F(s, j) -> F(s+1, j), B(s, j) -> B(s-1, j)
          const bool out = kind == 0 ? s < S - 1 : (kind == 1 && s > 0);
          int tg = kind == 0 ? s + 1 : s - 1;
          tg = tg < 0 ? 0 : (tg > S - 1 ? S - 1 : tg);
          const uint32_t lat = (kind == 0 ? wl : DURWL(tg)) >> 16;  // edge (s, s+1) or (s-1, s)
          uint32_t* ring = (kind == 0 ? rRF : rRB) + (((int)(j & (kSeqK - 1)) * S + tg) * 32);
          const uint32_t old = *ring;
          const uint32_t consumed = (CNT(tg) >> sh) & 255u;
          // the slot's previous item j-K must be consumed or already arrived
          const bool ovf = out && j >= (uint32_t)kSeqK && consumed + kSeqK <= j && old > at;
          const int d2 = out ? sq_dev<PLC, P>(tg) : d;
          // the consumer's free time (read before this step's stores; the
          // committer's is its finish time, written with its next decision)
          const uint32_t free2 = d2 == d ? fin : (FD(d2) >> 4);
          CNT(s) = cnt + (1u << sh);
          ROOM(d) = room;
          if (!SEARCH && kind == 0 && room < MINROOM(d)) MINROOM(d) = room;
          if (out) *ring = fin + lat;
          if (ovf) { overflow = true; alive = false; }
          // re-decide the committer and the consumer (the committer itself
          // again when there is no output: same inputs, same result)
          DecIn A, B;
          dec_load(d, fin, A);
          dec_load(d2, free2, B);
          dec_compute(d, A, at);
          dec_compute(d2, B, at);
        }
      }
    }
    // ---- a6/a7: metrics, argmin key or SoA results
    if (have) {
      if (overflow) {
        const unsigned k = atomicAdd(sl.overflow_count, 1u);
        if (k < sl.overflow_cap) sl.overflow_idx[k] = sl.list_slot ? slot : idx;
      } else {
        n_tasks += stuck ? 0 : (unsigned long long)T;
        uint32_t mk = 0;
#pragma unroll
        for (int d = 0; d < P; ++d) mk = max(mk, FD(d) >> 4);
        if (SEARCH) {
          if (!stuck) {
            const unsigned long long key = ((unsigned long long)mk << sl.key_bits) | idx;
            if (key < best_key) {
              best_key = key;
              if (sl.prune) atomicMin(sl.key, key);  // share the incumbent at once
            }
          }
        } else {
          int64_t mmax = 0;
          double busy = 0;
          for (int d = 0; d < P; ++d) {
            const int64_t md = sl.cap - MINROOM(d);
            mmax = md > mmax ? md : mmax;
          }
          for (int s = 0; s < S; ++s) {
            const int a = cuts[s], b = cuts[s + 1];
            busy += (double)m * (double)((PRE(kColTF, b) - PRE(kColTF, a)) + (PRE(kColTB, b) - PRE(kColTB, a)) +
                                         (PRE(kColTW, b) - PRE(kColTW, a)));
          }
          if (sl.out_status) sl.out_status[slot] = stuck ? ADAPTIS_CAND_STUCK : ADAPTIS_CAND_OK;
          if (sl.out_makespan) sl.out_makespan[slot] = stuck ? INT64_MAX : (int64_t)mk;
          if (sl.out_makespan_f32) sl.out_makespan_f32[slot] = stuck ? INFINITY : (float)mk;
          if (sl.out_peak) sl.out_peak[slot] = stuck ? 0 : mmax;
          if (sl.out_bubble)
            sl.out_bubble[slot] = stuck ? 0.0f : (float)(1.0 - busy / ((double)P * (double)mk));
        }
      }
    }
  }
#undef KEY
#undef FD
#undef CNT
#undef DURFB
#undef DURWL
#undef RF
#undef RB
#undef ROOM
#undef MINROOM
#undef AS
#undef ACTLO
  // warp reductions of the key and the counters
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long x = __shfl_xor_sync(FULLMASK, best_key, o);
    best_key = x < best_key ? x : best_key;
    n_inv += __shfl_xor_sync(FULLMASK, n_inv, o);
    n_pr += __shfl_xor_sync(FULLMASK, n_pr, o);
    n_tasks += __shfl_xor_sync(FULLMASK, n_tasks, o);
  }
  if (lane == 0) {
    if (SEARCH && best_key != (~0ull >> 1)) atomicMin(sl.key, best_key);
    if (n_inv) atomicAdd(sl.n_invalid, n_inv);
    if (n_pr) atomicAdd(sl.n_pruned, n_pr);
    if (n_tasks) atomicAdd(sl.n_tasks, n_tasks);
  }
}

using SeqFn = void (*)(const DevTables, const SegLaunch);

template <int V, int P, bool SEARCH>
static SeqFn pick_plc(int plc) {
  if constexpr (V == 1) return seqg_kernel<1, P, ADAPTIS_SEQ, SEARCH>;
  else return plc == ADAPTIS_WAVE ? seqg_kernel<V, P, ADAPTIS_WAVE, SEARCH>
                                  : seqg_kernel<V, P, ADAPTIS_INTERLEAVED, SEARCH>;
}
template <int V, bool SEARCH>
static SeqFn pick_p(int p, int plc) {
  switch (p) {
    case 2: return pick_plc<V, 2, SEARCH>(plc);
    case 4: return pick_plc<V, 4, SEARCH>(plc);
    case 8: return pick_plc<V, 8, SEARCH>(plc);
    default: return pick_plc<V, 16, SEARCH>(plc);
  }
}
template <bool SEARCH>
static SeqFn pick_v(int v, int p, int plc) {
  switch (v) {
    case 1: return pick_p<1, SEARCH>(p, plc);
    case 2: return pick_p<2, SEARCH>(p, plc);
    case 3: return pick_p<3, SEARCH>(p, plc);
    default: return pick_p<4, SEARCH>(p, plc);
  }
}

// the sequential kernel needs int32 ticks with makespans < 2^28 (key at << 4 | d),
// m <= 255 (8-bit counters), latencies < 2^16, p in {2, 4, 8, 16} (compile-time
// placement arithmetic), and a plain position range (no explicit plans,
// lists or traces; the fallback re-run keeps the global-ring kernel), with
// `min_warps` warps of state per SM (0: 4, and 5 for the WAVE placement,
// measured on cfg5's p = 16 v = 2 segments against the lane kernel: INT 26.6 s
// against 29.3 s at 4 warps, WAVE 31.0 s against 25.6 s)
bool seqg_eligible(const SegLaunch& s, bool seq_ok, int max_smem, int min_warps) {
  if (min_warps <= 0) min_warps = s.placement == ADAPTIS_WAVE ? 5 : 4;
  if (!seq_ok || s.policy != ADAPTIS_GREEDY || s.tick != kTickI32 || s.trace || s.list_cuts ||
      s.list_tasks || s.out_report || s.m > 255 || s.v < 1 || s.v > 4 ||
      (s.p != 2 && s.p != 4 && s.p != 8 && s.p != 16))
    return false;
  const size_t per_warp = seqg_smem_bytes(s.S, s.p, s.key != nullptr);
  return per_warp <= (size_t)max_smem && (size_t)min_warps * per_warp <= (size_t)228 * 1024;
}

int launch_seqg(const DevTables& t, const SegLaunch& s, int num_sms, void* stream) {
  SeqFn f = s.key ? pick_v<true>(s.v, s.p, s.placement) : pick_v<false>(s.v, s.p, s.placement);
  const size_t sm = seqg_smem_bytes(s.S, s.p, s.key != nullptr);
  cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return (int)e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, f, 32, sm);
  if (e != cudaSuccess) return (int)e;
  if (per_sm < 1) return (int)cudaErrorInvalidConfiguration;
  static const int max_cta = getenv("ADAPTIS_SEQ_MAXCTA") ? atoi(getenv("ADAPTIS_SEQ_MAXCTA")) : 0;  // A/B hook
  if (max_cta > 0 && per_sm > max_cta) per_sm = max_cta;
  unsigned grid = (unsigned)num_sms * (unsigned)per_sm;
  const uint64_t warps_needed = (s.n_pos + 31) / 32;
  if (warps_needed < grid) grid = (unsigned)(warps_needed ? warps_needed : 1);
  f<<<grid, 32, sm, (cudaStream_t)stream>>>(t, s);
  return (int)cudaGetLastError();
}

}  // namespace adaptis
