// adaptis_fixed.cu — the fixed orders (GPIPE R11, ONEF1B R9/R10, ZB R13) as
// one static task order per segment, one thread per candidate.
//
// Why a static order. Under GPIPE / ONEF1B every device runs its Megatron list
// in order, so a candidate's times are the longest path over the DAG plus the
// list edges (Alg. 1 Step 3): any topological order of the tasks
// computes them, and which order is topological does not depend on the
// durations. ZB runs the same F/B lists with split B; its W-fill (R13) is a
// decision of one device from its own free time, its own memory and the ready
// time r of its next F/B, whose producer precedes it in a topological order of
// the F/B tasks. So all three run as one order of F/B entries, built once per
// segment on the host (fx_build_order) and shared by every candidate: per
// entry a thread reads its device's free time and its input's arrival, runs
// the ZB W-fill, writes the finish time and its output's arrival. No
// decisions, argmins, rings or overflow: arrivals live in the order's slots,
// assigned by liveness on the host (at most 32 on the configs).
//
// Exactness. The host sorts the entries by their start times under nominal
// durations (F = 1, B = 2): a consumer starts after its producer finishes and a
// device's tasks start in list order, so the sort is a topological order of
// DAG + list edges, and evaluating max(free, arrival) + duration in it gives
// the longest path for any durations >= 1 (R17). ZB: the oracle's rule (ii)
// runs the oldest pending W while free < r, where r = the arrival of the input
// (an F(s, j)'s own F precedes its B on the device, so it never binds); rule (i)
// runs it while the next F does not fit under Eq. 2; both only read the
// device's own state and r, which are final when the entry is reached.
//
// Layout: [field][lane] words (conflict-free for any per-lane index): per
// device free time (and ZB: B count | W count << 16, cap - static - dynamic
// bytes, its minimum); per stage t_F, t_B (fused: t_B + t_W), ZB t_W, both
// latencies, ZB act and stash bytes; the order's arrival slots.
#include <algorithm>
#include <vector>

#include "adaptis_seg.cuh"

namespace adaptis {

constexpr uint32_t kFxNone = 255u;  // entry field: no input / no output item

struct FxLayout {
  int free_, slot, df, db, dw, lat, nbwd, n32;  // u32 rows
  int as, act, room, minroom, n64;              // u64 rows
};
ADAPTIS_LAYOUT_HD FxLayout fx_layout(int S, int p, int R, bool zb, bool search) {
  FxLayout l{};
  int r = 0;
  l.free_ = r; r += p;
  l.slot = r; r += R;
  l.df = r; r += S;
  l.db = r; r += S;
  l.dw = r; r += zb ? S : 0;
  l.lat = r; r += S;
  l.nbwd = r; r += zb ? p : 0;
  l.n32 = (r + 1) & ~1;  // 8-byte alignment of the u64 rows
  r = 0;
  l.as = r; r += S;      // act + stash
  l.act = r; r += zb ? S : 0;
  l.room = r; r += p;    // cap - static (- dynamic, ZB)
  l.minroom = r; r += (zb && !search) ? p : 0;
  l.n64 = r;
  return l;
}
ADAPTIS_LAYOUT_HD size_t fx_smem_bytes(int S, int p, int R, bool zb, bool search) {
  const FxLayout l = fx_layout(S, p, R, zb, search);
  return (size_t)32 * (4 * l.n32 + 8 * l.n64);
}

// P: the device count when it is a power of two <= 16 (compile-time W-queue
// arithmetic), 0 for any other p
template <int V, int P, bool ZB, bool SEARCH>
__global__ void __launch_bounds__(32, 16)
fixed_kernel(const DevTables tab, const SegLaunch sl) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31;
  const int L = sl.L, m = sl.m, p = P > 0 ? P : sl.p, S = sl.S, plc = sl.placement;
  // ZB's k-th pending W of device d is the W of its k-th B: chunk v-1 - (k / p) mod v
  // (R10 backward order); ZB is enumerated on SEQ (v = 1) and INT placements only (R12)
  auto w_stage = [&](unsigned k, int d) -> int {
    if constexpr (V == 1) return d;
    else if constexpr (P > 0) return (V - 1 - (int)((k / (unsigned)P) % V)) * P + d;
    else return (V - 1 - (int)((k / (unsigned)p) % V)) * p + d;
  };
  const FxLayout lay = fx_layout(S, p, sl.fx_slots, ZB, SEARCH);
  uint32_t* __restrict__ w32 = reinterpret_cast<uint32_t*>(smem);
  int64_t* __restrict__ w64 = reinterpret_cast<int64_t*>(smem + (size_t)128 * lay.n32);
  uint32_t* __restrict__ rFREE = w32 + lay.free_ * 32 + lane;
  uint32_t* __restrict__ rSLOT = w32 + lay.slot * 32 + lane;
  uint32_t* __restrict__ rDF = w32 + lay.df * 32 + lane;
  uint32_t* __restrict__ rDB = w32 + lay.db * 32 + lane;
  uint32_t* __restrict__ rDW = w32 + lay.dw * 32 + lane;
  uint32_t* __restrict__ rLAT = w32 + lay.lat * 32 + lane;
  uint32_t* __restrict__ rNBWD = w32 + lay.nbwd * 32 + lane;
  int64_t* __restrict__ rAS = w64 + lay.as * 32 + lane;
  int64_t* __restrict__ rACT = w64 + lay.act * 32 + lane;
  int64_t* __restrict__ rROOM = w64 + lay.room * 32 + lane;
  int64_t* __restrict__ rMINROOM = w64 + lay.minroom * 32 + lane;
#define FREE(d) rFREE[(d) * 32]
#define SLOT(i) rSLOT[(i) * 32]
#define DF(s) rDF[(s) * 32]
#define DB(s) rDB[(s) * 32]
#define DW(s) rDW[(s) * 32]
#define LAT(s) rLAT[(s) * 32]
#define NBWD(d) rNBWD[(d) * 32]
#define AS(s) rAS[(s) * 32]
#define ACT(s) rACT[(s) * 32]
#define ROOM(d) rROOM[(d) * 32]
#define MINROOM(d) rMINROOM[(d) * 32]
  const int64_t* pre = tab.pre;  // [kNumCols][L + 1] prefix sums (global, read-only)
  auto PRE = [&](int col, int row) -> int64_t { return __ldg(pre + (size_t)col * (L + 1) + row); };
  const uint32_t* __restrict__ ent = sl.fx_ent;
  const int NE = sl.fx_n;
  const bool gpipe = sl.policy == ADAPTIS_GPIPE;
  // tasks per simulated candidate: the F/B entries, plus ZB's S * m W
  const unsigned long long T = (unsigned long long)NE + (ZB ? (unsigned long long)S * m : 0ull);

  unsigned long long best_key = ~0ull >> 1, n_inv = 0, n_pr = 0, n_tasks = 0;
  int16_t cuts[ADAPTIS_MAX_S + 1];
  const int16_t* seed = tab.seeds + sl.group * ADAPTIS_MAX_S;
  uint64_t rpos = 0, rend = 0, prev_idx = ~0ull - 1;
  int brem = 0;
  bool exhausted = false;

  for (;;) {
    // ---- setup: every lane looks for its next candidate (a1-a4); invalid
    // decodes, pruned candidates and fused orders over the cap end here
    bool have = false;
    uint64_t idx = 0, slot = 0;
    int64_t cand_peak = 0;  // fused orders: max_d M_d from the order (R16)
    for (;;) {
      const bool need = !have && !(exhausted && rpos >= rend);
      const unsigned need_m = __ballot_sync(FULLMASK, need);
      if (!need_m) break;
      unsigned long long inc = 0;  // the prune's incumbent, one read per warp
      if (SEARCH && sl.prune) {
        if (lane == 0) inc = *(volatile unsigned long long*)sl.key;
        inc = __shfl_sync(FULLMASK, inc, 0);
      }
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
      // a2/a3 statics: cap - weight/grad bytes per device, act + stash (and ZB:
      // act) bytes per stage; prefix differences with the running prefix carried
      for (int d = 0; d < p; ++d) { FREE(d) = 0; ROOM(d) = sl.cap; }
      {
        int64_t pwg = PRE(kColWG, cuts[0]), pact = PRE(kColAct, cuts[0]), pst = PRE(kColStash, cuts[0]);
        for (int s = 0; s < S; ++s) {
          const int b = cuts[s + 1];
          const int64_t wg = PRE(kColWG, b), act = PRE(kColAct, b), st = PRE(kColStash, b);
          ROOM(dev_of(plc, p, s)) -= wg - pwg;  // cap - static (cannot overflow: static >= 0)
          AS(s) = (act - pact) + (st - pst);
          if constexpr (ZB) ACT(s) = act - pact;
          pwg = wg; pact = act; pst = st;
        }
      }
      // a4 (R16): a fused order's peak is a function of the order (GPIPE: all
      // m forwards; Megatron: the periodic closed form), so over-cap fused
      // candidates are decided here. ZB: the first min(w + 1, m v) entries of a
      // device's list are forwards with no W pending, so if their act + stash
      // exceeds the room the candidate ends over the cap whatever follows
      // (search skips it; eval still simulates it for M_d)
      bool pre_over = false;
      int64_t fused_peak = 0;
      for (int d = 0; d < p; ++d) {
        int64_t ac[V];
        int64_t A = 0;
#pragma unroll
        for (int c = 0; c < V; ++c) {
          ac[c] = AS(stage_of(plc, p, c, d));
          A += ac[c];
        }
        const int tot = m * V;
        const int wup = V == 1 ? min(m, p - d - 1) : min(tot, 2 * (p - d - 1) + (V - 1) * p);
        if constexpr (!ZB) {
          const int64_t pk = gpipe ? A * m : megatron_peak<V>(ac, p, m, wup);
          const int64_t md = (sl.cap - ROOM(d)) + pk;
          pre_over = pre_over || pk > ROOM(d);
          fused_peak = md > fused_peak ? md : fused_peak;
        } else if constexpr (SEARCH) {
          pre_over = pre_over || chunk_prefix<V>(ac, p, min(wup + 1, tot), false) > ROOM(d);
        }
      }
      if (pre_over) {
        if (!SEARCH) {
          if (sl.out_status) sl.out_status[slot] = ADAPTIS_CAND_OVER_CAP;
          if (sl.out_makespan_f32) sl.out_makespan_f32[slot] = INFINITY;
          if (sl.out_makespan) sl.out_makespan[slot] = INT64_MAX;
          if (sl.out_peak) sl.out_peak[slot] = fused_peak;
          if (sl.out_bubble) sl.out_bubble[slot] = 0.0f;
        }
        continue;
      }
      // stage durations and output latencies (R3-R6: 0 between stages of one device)
      {
        int64_t pf = PRE(kColTF, cuts[0]), pb = PRE(kColTB, cuts[0]), pw = PRE(kColTW, cuts[0]);
        for (int s = 0; s < S; ++s) {
          const int a = cuts[s], b = cuts[s + 1];
          const int ds = dev_of(plc, p, s);
          const int64_t f = PRE(kColTF, b), bb = PRE(kColTB, b), w = PRE(kColTW, b);
          DF(s) = (uint32_t)(f - pf);
          DB(s) = (uint32_t)(ZB ? bb - pb : (bb - pb) + (w - pw));  // R2: GPIPE / ONEF1B fuse B and W
          if constexpr (ZB) DW(s) = (uint32_t)(w - pw);
          pf = f; pb = bb; pw = w;
          const uint32_t lf = (s < S - 1 && dev_of(plc, p, s + 1) != ds) ? (uint32_t)tab.comm[b - 1] : 0u;
          const uint32_t lb = (s > 0 && dev_of(plc, p, s - 1) != ds) ? (uint32_t)tab.comm[a - 1] : 0u;
          LAT(s) = lf | (lb << 16);
        }
      }
      if constexpr (ZB) {
        for (int d = 0; d < p; ++d) {
          NBWD(d) = 0;
          if (!SEARCH) MINROOM(d) = ROOM(d);
        }
      }
      // exact lower-bound prune (search; the bound of adaptis_seg.cuh) from the
      // stage rows: device d's lowest stage is d, head = t_F of stages < d + the
      // d edge latencies (their forward latencies);
      //   fused: head + busy_d + (t_B + t_W) of stages < d + latencies
      //   split: max(head + busy_d, head + m (F + B)_d + t_B of stages < d + latencies + t_W(stage 0))
      if (SEARCH && sl.prune) {
        int64_t hf = 0, hb = 0, lk = 0, lb = 0;  // sums over stages < d
        const int64_t w0 = ZB ? (int64_t)DW(0) : 0;
        for (int d = 0; d < p; ++d) {
          if (d >= 1) {
            hf += DF(d - 1);
            hb += DB(d - 1);  // fused: t_B + t_W
            lk += (int64_t)(LAT(d - 1) & 0xffffu);
          }
          int64_t busy = 0, wsum = 0;
#pragma unroll
          for (int c = 0; c < V; ++c) {
            const int s = stage_of(plc, p, c, d);
            const int64_t cw = ZB ? (int64_t)DW(s) : 0;
            busy += (int64_t)m * ((int64_t)DF(s) + (int64_t)DB(s) + cw);
            wsum += cw;
          }
          const int64_t head = hf + lk;
          int64_t lbd = busy + head;
          if constexpr (!ZB) {
            lbd += hb + lk;
          } else {
            const int64_t alt = busy - (int64_t)m * wsum + head + hb + lk + w0;
            lbd = alt > lbd ? alt : lbd;
          }
          lb = lbd > lb ? lbd : lb;
        }
        if ((((unsigned long long)lb << sl.key_bits) | idx) > inc) { ++n_pr; continue; }
      }
      cand_peak = fused_peak;
      have = true;
    }
    if (!__any_sync(FULLMASK, have)) break;

    // ---- a5: the static order, one F/B entry per step (all lanes in lockstep)
    bool over = false;
    int t_over = NE;  // search: entries simulated until the candidate went over the cap
    uint32_t e_next = __ldg(ent);
    for (int t = 0; t < NE; ++t) {
      // search: a ZB candidate over the cap cannot win; stop when none is left
      if (ZB && SEARCH && (t & 31) == 0 && !__any_sync(FULLMASK, have && !over)) break;
      const uint32_t e = e_next;
      if (t + 1 < NE) e_next = __ldg(ent + t + 1);
      if (have) {
        const int s = (int)(e & 63u), kind = (int)((e >> 6) & 1u);
        const uint32_t in = (e >> 8) & 255u, out = (e >> 16) & 255u;
        const int d = (int)((e >> 24) & 15u);
        uint32_t fr = FREE(d);
        const uint32_t r = in != kFxNone ? SLOT(in) : 0u;
        if constexpr (ZB) {
          // R13: the oldest pending W runs (i) while the next F does not fit
          // under Eq. 2, (ii) while the device would idle before r
          uint32_t nbwd = NBWD(d);
          int64_t room = ROOM(d);
          const int64_t need = kind == 0 ? AS(s) : INT64_MIN;
          while ((nbwd & 0xffffu) > (nbwd >> 16) && (fr < r || room < need)) {
            const int ws = w_stage(nbwd >> 16, d);  // the W of d's oldest pending B
            fr += DW(ws);
            room += AS(ws) - ACT(ws);  // R16: stash freed at W end
            nbwd += 1u << 16;
          }
          if (kind == 0) {
            room -= need;  // act + stash at F start (runs even when it does not fit: over cap)
            if (room < 0 && !over) { over = true; t_over = t + 1; }
            if (!SEARCH && room < MINROOM(d)) MINROOM(d) = room;
          } else {
            room += ACT(s);  // act freed at B end
            nbwd += 1u;
          }
          ROOM(d) = room;
          NBWD(d) = nbwd;
        }
        const uint32_t fin = max(fr, r) + (kind ? DB(s) : DF(s));
        FREE(d) = fin;
        if (out != kFxNone) SLOT(out) = fin + (kind ? (LAT(s) >> 16) : (LAT(s) & 0xffffu));
      }
    }
    // ---- a6/a7: metrics, argmin key or SoA results
    if (have) {
      uint32_t mk = 0;
      for (int d = 0; d < p; ++d) {
        uint32_t fr = FREE(d);
        if constexpr (ZB) {  // the Ws still pending after the last F/B run back to back
          const uint32_t nbwd = NBWD(d);
          for (int k = (int)(nbwd >> 16); k < (int)(nbwd & 0xffffu); ++k)
            fr += DW(w_stage((unsigned)k, d));
        }
        mk = max(mk, fr);
      }
      n_tasks += (SEARCH && over) ? (unsigned long long)t_over : T;
      if (SEARCH) {
        if (!over) {
          const unsigned long long key = ((unsigned long long)mk << sl.key_bits) | idx;
          if (key < best_key) {
            best_key = key;
            if (sl.prune) atomicMin(sl.key, key);  // share the incumbent at once
          }
        }
      } else {
        int64_t mmax = cand_peak;
        if constexpr (ZB) {
          mmax = 0;
          for (int d = 0; d < p; ++d) {
            const int64_t md = sl.cap - MINROOM(d);  // static + peak dynamic bytes
            mmax = md > mmax ? md : mmax;
          }
        }
        // busy time of all devices: m x every layer's t_F + t_B + t_W
        const double busy = (double)m * (double)(PRE(kColTF, L) + PRE(kColTB, L) + PRE(kColTW, L));
        if (sl.out_status) sl.out_status[slot] = over ? ADAPTIS_CAND_OVER_CAP : ADAPTIS_CAND_OK;
        if (sl.out_makespan) sl.out_makespan[slot] = over ? INT64_MAX : (int64_t)mk;
        if (sl.out_makespan_f32) sl.out_makespan_f32[slot] = over ? INFINITY : (float)mk;
        if (sl.out_peak) sl.out_peak[slot] = mmax;
        if (sl.out_bubble) sl.out_bubble[slot] = over ? 0.0f : (float)(1.0 - busy / ((double)p * (double)mk));
      }
    }
  }
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
#undef FREE
#undef SLOT
#undef DF
#undef DB
#undef DW
#undef LAT
#undef NBWD
#undef AS
#undef ACT
#undef ROOM
#undef MINROOM
}


// ---------------------------------------------------------------------------
// host: the static order of one segment

// R9-R11: device d's list of (kind, chunk, mb); forwards while GPIPE or while
// fewer than w + 1 forwards are ahead of the backwards (w = the warm-up), the
// k-th forward / backward at chunk (k / p) mod v (backwards: reversed) and
// micro-batch (k / (p v)) p + k mod p
static void fx_device_list(bool gpipe, int p, int v, int m, int d, std::vector<int>& kind,
                           std::vector<int>& chunk, std::vector<int>& mb) {
  const int tot = m * v;
  const int wup = v == 1 ? std::min(m, p - d - 1) : std::min(tot, 2 * (p - d - 1) + (v - 1) * p);
  int nF = 0, nB = 0;
  while (nF < tot || nB < tot) {
    const bool f = nF < tot && (gpipe || nF - nB <= wup);
    const int k = f ? nF++ : nB++;
    const int g = k / (p * v), r = k % (p * v), c = r / p;
    kind.push_back(f ? 0 : 1);
    chunk.push_back(f ? c : v - 1 - c);
    mb.push_back(g * p + r % p);
  }
}

static int fx_stage(int plc, int p, int c, int d) {
  if (plc == ADAPTIS_SEQ) return d;
  if (plc == ADAPTIS_INTERLEAVED) return c * p + d;
  return c * p + ((c & 1) ? p - 1 - d : d);
}

// The entries (s | kind << 6 | in << 8 | out << 16 | d << 24) in the order of
// their start times under nominal durations (F = 1, B = 2, no latency; ties by
// device), and the number of arrival slots. False when the lists deadlock or
// the order needs more than 254 slots (the lane kernels then run the segment).
bool fx_build_order(int policy, int placement, int p, int v, int m, std::vector<uint32_t>& ent, int& slots) {
  const int S = p * v;
  if (p > 16 || S > 64 || m < 1) return false;
  const bool gpipe = policy == ADAPTIS_GPIPE;
  std::vector<std::vector<int>> K(p), C(p), J(p);
  for (int d = 0; d < p; ++d) fx_device_list(gpipe, p, v, m, d, K[d], C[d], J[d]);
  // finish times under nominal durations; -1: not run yet
  std::vector<long> finF((size_t)S * m, -1), finB((size_t)S * m, -1);
  std::vector<long> fr(p, 0);
  std::vector<size_t> pos(p, 0);
  struct E { long start; int d, kind, s, j; };
  std::vector<E> es;
  es.reserve((size_t)2 * S * m);
  for (bool prog = true; prog;) {
    prog = false;
    for (int d = 0; d < p; ++d) {
      while (pos[d] < K[d].size()) {
        const int k = K[d][pos[d]], s = fx_stage(placement, p, C[d][pos[d]], d), j = J[d][pos[d]];
        long in = 0;
        if (k == 0) {
          if (s > 0) in = finF[(size_t)(s - 1) * m + j];
        } else {
          if (finF[(size_t)s * m + j] < 0) break;  // its F has not run
          if (s < S - 1) in = finB[(size_t)(s + 1) * m + j];
        }
        if (in < 0) break;
        const long st = std::max(fr[d], in);
        fr[d] = st + (k == 0 ? 1 : 2);
        (k == 0 ? finF : finB)[(size_t)s * m + j] = fr[d];
        es.push_back({st, d, k, s, j});
        ++pos[d];
        prog = true;
      }
    }
  }
  for (int d = 0; d < p; ++d)
    if (pos[d] < K[d].size()) return false;  // the lists deadlock
  std::stable_sort(es.begin(), es.end(),
                   [](const E& a, const E& b) { return a.start != b.start ? a.start < b.start : a.d < b.d; });
  // arrival slots by liveness: an item lives from its producer's entry to its consumer's
  std::vector<int> slotF((size_t)S * m, -1), slotB((size_t)S * m, -1), freel;
  slots = 0;
  ent.clear();
  for (const E& e : es) {
    uint32_t in = kFxNone, out = kFxNone;
    if (e.kind == 0 && e.s > 0) in = (uint32_t)slotF[(size_t)(e.s - 1) * m + e.j];
    if (e.kind == 1 && e.s < S - 1) in = (uint32_t)slotB[(size_t)(e.s + 1) * m + e.j];
    if (in != kFxNone) freel.push_back((int)in);
    const bool has_out = e.kind == 0 ? e.s < S - 1 : e.s > 0;
    if (has_out) {
      int sl;
      if (!freel.empty()) { sl = freel.back(); freel.pop_back(); }
      else sl = slots++;
      if (sl >= (int)kFxNone) return false;
      (e.kind == 0 ? slotF : slotB)[(size_t)e.s * m + e.j] = sl;
      out = (uint32_t)sl;
    }
    ent.push_back((uint32_t)e.s | ((uint32_t)e.kind << 6) | (in << 8) | (out << 16) | ((uint32_t)e.d << 24));
  }
  return true;
}

using FxFn = void (*)(const DevTables, const SegLaunch);
template <int V, bool ZB, bool SEARCH>
static FxFn fx_pick_p(int p) {
  switch (p) {
    case 1: return fixed_kernel<V, 1, ZB, SEARCH>;
    case 2: return fixed_kernel<V, 2, ZB, SEARCH>;
    case 4: return fixed_kernel<V, 4, ZB, SEARCH>;
    case 8: return fixed_kernel<V, 8, ZB, SEARCH>;
    case 16: return fixed_kernel<V, 16, ZB, SEARCH>;
    default: return fixed_kernel<V, 0, ZB, SEARCH>;
  }
}
template <bool ZB, bool SEARCH>
static FxFn fx_pick_v(int v, int p) {
  switch (v) {
    case 1: return fx_pick_p<1, ZB, SEARCH>(p);
    case 2: return fx_pick_p<2, ZB, SEARCH>(p);
    case 3: return fx_pick_p<3, ZB, SEARCH>(p);
    default: return fx_pick_p<4, ZB, SEARCH>(p);
  }
}

// the static-order kernel takes GPIPE / ONEF1B / ZB segments with int32 ticks
// (seq_ok: U < 2^28, latencies < 2^16), p <= 16, m <= 65535, a plain position
// range (no explicit plans, lists, traces or reports: the lane kernels keep
// those), and room for enough warps of state per SM (measured on cfg5's p = 16
// segments, where the lane kernel is faster below them): 4 for ONEF1B and ZB,
// 2 for GPIPE, which a4 decides at setup; ADAPTIS_FIXED_MINW overrides all three
bool fixed_eligible(const SegLaunch& s, bool seq_ok, int max_smem, int slots) {
  const char* me = getenv("ADAPTIS_FIXED_MINW");  // read per launch (tests set it)
  const int minw_env = me ? atoi(me) : 0;
  const int minw = minw_env > 0 ? minw_env : (s.policy == ADAPTIS_GPIPE ? 2 : 4);
  if (!seq_ok || (s.policy != ADAPTIS_GPIPE && s.policy != ADAPTIS_ONEF1B && s.policy != ADAPTIS_ZB) ||
      s.tick != kTickI32 || s.trace || s.list_cuts || s.list_tasks || s.out_report || s.p > 16 ||
      (s.policy == ADAPTIS_ZB && s.placement == ADAPTIS_WAVE) ||
      s.m > 65535 || s.v < 1 || s.v > 4 || s.S > 64)
    return false;
  const size_t per_warp = fx_smem_bytes(s.S, s.p, slots, s.policy == ADAPTIS_ZB, s.key != nullptr);
  return per_warp <= (size_t)max_smem && (size_t)minw * per_warp <= (size_t)228 * 1024;
}

int launch_fixed(const DevTables& t, const SegLaunch& s, int num_sms, void* stream) {
  const bool zb = s.policy == ADAPTIS_ZB;
  FxFn f = zb ? (s.key ? fx_pick_v<true, true>(s.v, s.p) : fx_pick_v<true, false>(s.v, s.p))
              : (s.key ? fx_pick_v<false, true>(s.v, s.p) : fx_pick_v<false, false>(s.v, s.p));
  const size_t sm = fx_smem_bytes(s.S, s.p, s.fx_slots, zb, s.key != nullptr);
  cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return (int)e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, f, 32, sm);
  if (e != cudaSuccess) return (int)e;
  if (per_sm < 1) return (int)cudaErrorInvalidConfiguration;
  unsigned grid = (unsigned)num_sms * (unsigned)per_sm;
  const uint64_t warps_needed = (s.n_pos + 31) / 32;
  if (warps_needed < grid) grid = (unsigned)(warps_needed ? warps_needed : 1);
  f<<<grid, 32, sm, (cudaStream_t)stream>>>(t, s);
  return (int)cudaGetLastError();
}

}  // namespace adaptis
