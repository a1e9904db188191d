// adaptis_kernels.cu — sm_100a kernels of the AdaPtis hot path (arXiv 2509.23722).
//
// One persistent kernel per (v-group, combo) segment of the candidate space.
// Each warp evaluates G = 32 / p2 candidates at a time (p2 = p rounded up to a
// power of two); within a candidate slot, lane d is pipeline device d. Per
// candidate the warp runs, in order (DESIGN.md §"Kernel"):
//   a1 decode        index -> cuts (colex / L1-ball unranking, one lane per slot)
//   a2 stage sums    prefix differences of the CTA's shared-memory prefix table,
//                    built once per CTA by a warp-shuffle scan of coalesced loads
//   a3 device sums   static memory, busy time, edge latencies (R3-R6)
//   a4 memory check  fused fixed orders: exact peak from the order alone (R16)
//   a5 simulation    dataflow rounds (GPIPE / ONEF1B / ZB, Lemmas 1-2) or
//                    bounded-lag rounds (GREEDY, Lemma 3); cross-device
//                    finish times travel through per-stage shared-memory rings
//   a6 metrics       segmented shuffle reductions (makespan, busy, peak)
//   a7 argmin        packed (makespan << bits | index) warp min -> atomicMin
// Timing is integer ticks: int32 when the host proved the makespan bound fits,
// int64 otherwise (bit-exact either way).
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>

#include "adaptis_decode.cuh"
#include "adaptis_internal.h"

namespace adaptis {

constexpr unsigned FULLMASK = 0xffffffffu;

template <typename T> struct TT;
template <> struct TT<int32_t> { static constexpr int32_t INF = INT32_MAX; };
template <> struct TT<int64_t> { static constexpr int64_t INF = INT64_MAX; };

template <typename T>
struct StageC {   // per (lane, own chunk) constants of one candidate
  T dF, dB, dW;   // task durations (dB includes c_W when fused, R2)
  T oF, oB;       // latency added to F(s) -> F(s+1) and B(s) -> B(s-1) (R3-R6)
  int64_t act, stash;
};

__device__ __forceinline__ int stage_of(int placement, int p, int c, int d) {
  if (placement == ADAPTIS_SEQ) return d;
  if (placement == ADAPTIS_INTERLEAVED) return c * p + d;
  return c * p + ((c & 1) ? p - 1 - d : d);  // WAVE (R12)
}
__device__ __forceinline__ int dev_of(int placement, int p, int s) {
  if (placement == ADAPTIS_SEQ) return s;
  if (placement == ADAPTIS_INTERLEAVED) return s % p;
  int c = s / p, j = s - c * p;
  return (c & 1) ? p - 1 - j : j;
}

template <typename X>
__device__ __forceinline__ X shfl_xor(X v, int o) { return __shfl_xor_sync(FULLMASK, v, o); }

// segmented reductions over aligned groups of p2 lanes
template <typename X>
__device__ __forceinline__ X seg_max(X v, int p2) {
  for (int o = 1; o < p2; o <<= 1) { X w = shfl_xor(v, o); v = w > v ? w : v; }
  return v;
}
template <typename X>
__device__ __forceinline__ X seg_min(X v, int p2) {
  for (int o = 1; o < p2; o <<= 1) { X w = shfl_xor(v, o); v = w < v ? w : v; }
  return v;
}
template <typename X>
__device__ __forceinline__ X seg_sum(X v, int p2) {
  for (int o = 1; o < p2; o <<= 1) v += shfl_xor(v, o);
  return v;
}

// incremental position in Megatron's virtual order (R10): k -> (chunk, mb)
struct VPos {
  int q, c, g;  // k = (g * v + c) * p + q
  __device__ __forceinline__ void reset() { q = 0; c = 0; g = 0; }
  __device__ __forceinline__ void next(int p, int v) {
    if (++q == p) { q = 0; if (++c == v) { c = 0; ++g; } }
  }
  __device__ __forceinline__ int mb(int p) const { return g * p + q; }
};

__device__ __forceinline__ uint64_t pos_to_index(const SegLaunch& sl, uint64_t pos) {
  if (sl.list_idx) return sl.list_idx[pos];
  if (pos < sl.n0) return sl.start0 + pos;
  uint64_t q = pos - sl.n0;
  uint64_t t = q >> kChunkBits;
  return ((sl.first_chunk + (t + 1) * (uint64_t)sl.world) << kChunkBits) +
         (q & ((1ull << kChunkBits) - 1));
}

// ------------------------------------------------------------------------------
// Ring addressing: ring[dir][slot j % K][cand g][stage s]
template <typename T>
struct Rings {
  T* base;
  int K, RS, gS;  // RS = G*S row stride, gS = g*S
  __device__ __forceinline__ T* at(int dir, int j, int s) const {
    return base + ((size_t)dir * K + (j & (K - 1))) * RS + gS + s;
  }
};

template <int POLICY, int V, typename T, bool FALLBACK>
__global__ void __launch_bounds__(kWarpsPerCta * 32)
seg_kernel(const DevTables tab, const SegLaunch sl) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int L = sl.L, p = sl.p, m = sl.m, S = sl.S, p2 = sl.p2, G = sl.G;
  constexpr bool FUSED = (POLICY == ADAPTIS_GPIPE || POLICY == ADAPTIS_ONEF1B);
  constexpr T INF = TT<T>::INF;
  constexpr T EMPTY = (T)-1;

  // ---- a2 prologue: per-CTA prefix table of the layer columns (warp-shuffle scan)
  int64_t* pre = reinterpret_cast<int64_t*>(smem);
  for (int col = warp; col < kNumCols; col += kWarpsPerCta) {
    int64_t carry = 0;
    const int64_t* src = tab.cols + (size_t)col * L;
    int64_t* dst = pre + (size_t)col * (L + 1);
    if (lane == 0) dst[0] = 0;
    for (int b = 0; b < L; b += 32) {
      int64_t x = (b + lane < L) ? src[b + lane] : 0;   // coalesced 8-byte loads
      for (int o = 1; o < 32; o <<= 1) {
        int64_t y = __shfl_up_sync(FULLMASK, x, o);
        if (lane >= o) x += y;
      }
      if (b + lane < L) dst[b + lane + 1] = carry + x;
      carry += __shfl_sync(FULLMASK, x, 31);
    }
  }
  __syncthreads();

  // ---- per-warp shared regions
  size_t off = ((size_t)kNumCols * (L + 1) * 8 + 15) & ~(size_t)15;
  const size_t cuts_bytes = (((size_t)G * (S + 1) * 2) + 15) & ~(size_t)15;
  const size_t sc_bytes = (size_t)(V > 1 ? V : 0) * 32 * sizeof(StageC<T>);
  const size_t ring_bytes = FALLBACK ? 0 : (size_t)2 * sl.ring_k * G * S * sizeof(T);
  const size_t per_warp = cuts_bytes + sc_bytes + ring_bytes;
  unsigned char* wbase = smem + off + per_warp * warp;
  int16_t* cuts_all = reinterpret_cast<int16_t*>(wbase);
  StageC<T>* scs = reinterpret_cast<StageC<T>*>(wbase + cuts_bytes);
  T* ring_base;
  if constexpr (FALLBACK) {
    const size_t gw = (size_t)blockIdx.x * kWarpsPerCta + warp;
    ring_base = reinterpret_cast<T*>(sl.gring) + gw * 2 * (size_t)sl.ring_k * G * S;
  } else {
    ring_base = reinterpret_cast<T*>(wbase + cuts_bytes + sc_bytes);
  }

  const int g = lane >> sl.log2p2;
  const int d = lane & (p2 - 1);
  const unsigned slot_mask = (p2 == 32) ? FULLMASK : (((1u << p2) - 1u) << (g * p2));
  int16_t* cuts = cuts_all + g * (S + 1);
  Rings<T> R{ring_base, sl.ring_k, G * S, g * S};

  unsigned long long wkey = ~0ull >> 1;  // running warp minimum (INT64_MAX)
  unsigned long long winvalid = 0;
  unsigned long long wtasks = 0;

  for (;;) {
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(sl.cursor, (unsigned long long)G);
    base = __shfl_sync(FULLMASK, base, 0);
    if (base >= sl.n_pos) break;
    const uint64_t pos = base + g;
    const bool slot_on = pos < sl.n_pos;
    const uint64_t idx = slot_on ? pos_to_index(sl, pos) : 0;

    // ---- a1 decode (lane 0 of each slot)
    bool valid = false;
    if (slot_on && d == 0)
      valid = decode_cuts(tab.binom, tab.ball, tab.seeds, sl.group, sl.part_mode, sl.radius, sl.S,
                          sl.L, idx - sl.seg_base, cuts);
    valid = __shfl_sync(FULLMASK, valid, g * p2);
    __syncwarp();
    const bool lane_on = slot_on && valid && d < p;

    // ---- a2/a3 aggregation for this lane's stages
    StageC<T> sc1{};  // V == 1 keeps the constants in registers
    int64_t busy = 0, stat = 0;
    T dmin = INF, cmin = INF;
    if (lane_on) {
#pragma unroll
      for (int c = 0; c < V; ++c) {
        const int s = stage_of(sl.placement, p, c, d);
        const int a = cuts[s], b = cuts[s + 1];
        StageC<T> x;
        const int64_t cF = pre[kColTF * (L + 1) + b] - pre[kColTF * (L + 1) + a];
        const int64_t cB = pre[kColTB * (L + 1) + b] - pre[kColTB * (L + 1) + a];
        const int64_t cW = pre[kColTW * (L + 1) + b] - pre[kColTW * (L + 1) + a];
        x.dF = (T)cF;
        x.dB = (T)(FUSED ? cB + cW : cB);
        x.dW = (T)cW;
        x.act = pre[kColAct * (L + 1) + b] - pre[kColAct * (L + 1) + a];
        x.stash = pre[kColStash * (L + 1) + b] - pre[kColStash * (L + 1) + a];
        stat += pre[kColWG * (L + 1) + b] - pre[kColWG * (L + 1) + a];
        busy += (int64_t)m * (cF + cB + cW);
        x.oF = 0;
        x.oB = 0;
        if (s < S - 1 && dev_of(sl.placement, p, s + 1) != d) {
          x.oF = (T)tab.comm[b - 1];
          cmin = x.oF < cmin ? x.oF : cmin;
        }
        if (s > 0 && dev_of(sl.placement, p, s - 1) != d) {
          x.oB = (T)tab.comm[a - 1];
          cmin = x.oB < cmin ? x.oB : cmin;
        }
        T mn = (T)cF < (T)cB ? (T)cF : (T)cB;
        mn = (T)cW < mn ? (T)cW : mn;
        dmin = mn < dmin ? mn : dmin;
        if constexpr (V == 1) sc1 = x; else scs[c * 32 + lane] = x;
      }
    }
    __syncwarp();
    auto SC = [&](int c) -> StageC<T> {
      if constexpr (V == 1) { (void)c; return sc1; } else { return scs[c * 32 + lane]; }
    };

    // ---- ring reset (this warp's slots)
    if constexpr (!FALLBACK) {
      const int n = 2 * sl.ring_k * G * S;
      for (int i = lane; i < n; i += 32) ring_base[i] = EMPTY;
    } else {
      const int n = 2 * sl.ring_k * G * S;
      for (int i = lane; i < n; i += 32) ring_base[i] = EMPTY;
    }
    __syncwarp();

    // ---- state
    const int tot = m * V;
    int w = 0;  // warm-up (R9, R10)
    if (V == 1) w = min(m, p - d - 1);
    else w = min(tot, 2 * (p - d - 1) + (V - 1) * p);
    T free_t = 0;
    int64_t dyn = 0, peak = 0;
    bool done = !lane_on;
    bool over = false;
    int status = 0;  // slot status, decided below

    // ---- a4: fused fixed orders: exact peak from the order alone (R16)
    if constexpr (FUSED) {
      if (lane_on) {
        if constexpr (POLICY == ADAPTIS_GPIPE) {
          int64_t sum = 0;
#pragma unroll
          for (int c = 0; c < V; ++c) { StageC<T> x = SC(c); sum += x.act + x.stash; }
          peak = sum * m;
        } else if constexpr (V == 1) {
          peak = (int64_t)min(m, w + 1) * (sc1.act + sc1.stash);
        } else {
          VPos fp, bp;
          fp.reset(); bp.reset();
          int nF = 0, nB = 0;
          int64_t dd = 0;
          while (nF < tot || nB < tot) {
            const bool isF = nF < tot && nF - nB <= w;
            if (isF) {
              StageC<T> x = SC(fp.c);
              dd += x.act + x.stash;
              peak = dd > peak ? dd : peak;
              fp.next(p, V); ++nF;
            } else {
              StageC<T> x = SC(V - 1 - bp.c);
              dd -= x.act + x.stash;
              bp.next(p, V); ++nB;
            }
          }
        }
        over = stat + peak > sl.cap;
      }
    }
    const bool pre_over = FUSED && (__ballot_sync(FULLMASK, over) & slot_mask);
    if (pre_over) done = true;  // fused fixed order infeasible by Eq. 2: no simulation

    // GREEDY window (Lemma 3): every unscheduled task starts at >= t* and no new
    // cross-device arrival can precede t* + dmin + cmin.
    T window = INF;
    if constexpr (POLICY == ADAPTIS_GREEDY) {
      const T dm = seg_min(dmin, p2);
      const T cm = seg_min(cmin, p2);
      window = (cm == INF) ? INF : dm + cm;
    }

    // ---- a5: simulation rounds
    int nF = 0, nB = 0, nW = 0;          // fixed orders: device-level counters
    VPos fp, bp, wp;
    fp.reset(); bp.reset(); wp.reset();
    int gF[V], gB[V], gW[V];             // GREEDY: per-chunk counters
#pragma unroll
    for (int c = 0; c < V; ++c) { gF[c] = 0; gB[c] = 0; gW[c] = 0; }
    bool slot_live = slot_on && valid && !pre_over;
    bool overflow = false;
    bool stuck = false;

    while (__any_sync(FULLMASK, slot_live)) {
      bool go = false, blocked = false;
      // action record
      int act_kind = -1, act_c = 0, act_j = 0, act_s = 0;
      T act_start = 0, r_in = 0;
      bool has_out = false, need_in = false;
      T tstar = INF;

      if constexpr (POLICY == ADAPTIS_GREEDY) {
        T at = INF;
        if (slot_live && !done) {
          T rFc[V], rBc[V];
          bool cF[V], cB[V], cW[V];
          T rmin = INF;
#pragma unroll
          for (int c = 0; c < V; ++c) {
            const int s = stage_of(sl.placement, p, c, d);
            StageC<T> x = SC(c);
            cF[c] = false; cB[c] = false; cW[c] = gW[c] < gB[c];
            rFc[c] = 0; rBc[c] = 0;
            if (gF[c] < m && stat + dyn + x.act + x.stash <= sl.cap) {
              T r = (s == 0) ? (T)0 : *R.at(0, gF[c], s);
              if (r >= 0) { cF[c] = true; rFc[c] = r; rmin = r < rmin ? r : rmin; }
            }
            if (gB[c] < gF[c]) {
              T r = (s == S - 1) ? (T)0 : *R.at(1, gB[c], s);
              if (r >= 0) { cB[c] = true; rBc[c] = r; rmin = r < rmin ? r : rmin; }
            }
            if (cW[c]) rmin = 0 < rmin ? 0 : rmin;
          }
          if (rmin != INF) {
            at = free_t > rmin ? free_t : rmin;
            // key (kind F < B < W, mb, stage); stage order == chunk order
            int bj = INT_MAX;
#pragma unroll
            for (int c = 0; c < V; ++c)
              if (cF[c] && rFc[c] <= at && gF[c] < bj) { bj = gF[c]; act_kind = 0; act_c = c; }
            if (act_kind < 0) {
#pragma unroll
              for (int c = 0; c < V; ++c)
                if (cB[c] && rBc[c] <= at && gB[c] < bj) { bj = gB[c]; act_kind = 1; act_c = c; }
            }
            if (act_kind < 0) {
#pragma unroll
              for (int c = 0; c < V; ++c)
                if (cW[c] && gW[c] < bj) { bj = gW[c]; act_kind = 2; act_c = c; }
            }
            act_j = bj;
          }
        }
        tstar = seg_min(at, p2);
        if (act_kind >= 0 && at - tstar < window) {
          act_s = stage_of(sl.placement, p, act_c, d);
          act_start = at;
          if (act_kind == 0) { need_in = act_s > 0; has_out = act_s < S - 1; }
          else if (act_kind == 1) { need_in = act_s < S - 1; has_out = act_s > 0; }
          bool out_ok = true;
          if (has_out)
            out_ok = *R.at(act_kind, act_j, act_kind == 0 ? act_s + 1 : act_s - 1) == EMPTY;
          go = out_ok;
          blocked = !out_ok;
        }
      } else {
        // fixed F/B lists (+ ZB's W fill)
        if (slot_live && !done) {
          const bool x_exists = nF < tot || nB < tot;
          const bool hasW = (POLICY == ADAPTIS_ZB) && nW < nB;
          bool doW = false;
          if (x_exists) {
            const bool isF = nF < tot && (POLICY == ADAPTIS_GPIPE || nF - nB <= w);
            const int c = isF ? fp.c : V - 1 - bp.c;
            const int j = isF ? fp.mb(p) : bp.mb(p);
            const int s = stage_of(sl.placement, p, c, d);
            StageC<T> x = SC(c);
            bool forced = false;
            if constexpr (POLICY == ADAPTIS_ZB)
              forced = isF && hasW && stat + dyn + x.act + x.stash > sl.cap;
            if (forced) {
              doW = true;
            } else {
              need_in = isF ? (s > 0) : (s < S - 1);
              T r = need_in ? *R.at(isF ? 0 : 1, j, s) : (T)0;
              if (r >= 0) {
                if (hasW && free_t < r) {
                  doW = true;  // R13 (ii): fill the bubble before r with the oldest W
                } else {
                  act_kind = isF ? 0 : 1; act_c = c; act_j = j; act_s = s; r_in = r;
                  act_start = free_t > r ? free_t : r;
                  has_out = isF ? (s < S - 1) : (s > 0);
                  bool out_ok = true;
                  if (has_out) out_ok = *R.at(act_kind, j, isF ? s + 1 : s - 1) == EMPTY;
                  go = out_ok;
                  blocked = !out_ok;
                }
              }
            }
          } else if (hasW) {
            doW = true;
          }
          if (doW) {
            act_kind = 2; act_c = V - 1 - wp.c; act_j = wp.mb(p);
            act_s = stage_of(sl.placement, p, act_c, d);
            act_start = free_t; need_in = false; has_out = false; go = true;
          }
        }
      }
      __syncwarp();
      // ---- execute (write phase)
      if (go) {
        ++wtasks;
        StageC<T> x = SC(act_c);
        const T dur = act_kind == 0 ? x.dF : (act_kind == 1 ? x.dB : x.dW);
        const T fin = act_start + dur;
        free_t = fin;
        if (act_kind == 0) {
          dyn += x.act + x.stash;
          peak = dyn > peak ? dyn : peak;
          if (has_out) *R.at(0, act_j, act_s + 1) = fin + x.oF;
          if (need_in) *R.at(0, act_j, act_s) = EMPTY;
          if constexpr (POLICY == ADAPTIS_GREEDY) {
#pragma unroll
            for (int c = 0; c < V; ++c) gF[c] += (c == act_c);
          } else {
            ++nF; fp.next(p, V);
          }
          if constexpr (POLICY == ADAPTIS_ZB)
            if (sl.key && stat + dyn > sl.cap) over = true;  // search: Eq. 2 already violated
        } else if (act_kind == 1) {
          dyn -= x.act + (FUSED ? x.stash : 0);
          if (has_out) *R.at(1, act_j, act_s - 1) = fin + x.oB;
          if (need_in) *R.at(1, act_j, act_s) = EMPTY;
          if constexpr (POLICY == ADAPTIS_GREEDY) {
#pragma unroll
            for (int c = 0; c < V; ++c) gB[c] += (c == act_c);
          } else {
            ++nB; bp.next(p, V);
          }
        } else {
          dyn -= x.stash;
          if constexpr (POLICY == ADAPTIS_GREEDY) {
#pragma unroll
            for (int c = 0; c < V; ++c) gW[c] += (c == act_c);
          } else {
            ++nW; wp.next(p, V);
          }
        }
        // lane completion
        if constexpr (POLICY == ADAPTIS_GREEDY) {
          bool all = true;
#pragma unroll
          for (int c = 0; c < V; ++c) all = all && gF[c] == m && gB[c] == m && gW[c] == m;
          done = all;
        } else if constexpr (POLICY == ADAPTIS_ZB) {
          done = nF == tot && nB == tot && nW == tot;
        } else {
          done = nF == tot && nB == tot;
        }
      }
      (void)r_in;
      __syncwarp();
      // ---- progress bookkeeping per slot
      const unsigned go_m = __ballot_sync(FULLMASK, go);
      const unsigned blk_m = __ballot_sync(FULLMASK, blocked);
      const unsigned done_m = __ballot_sync(FULLMASK, done || !(d < p));
      const unsigned over_m = __ballot_sync(FULLMASK, over);
      if (slot_live) {
        if ((done_m & slot_mask) == slot_mask) {
          slot_live = false;
        } else if (over_m & slot_mask) {
          slot_live = false;  // search mode ZB: already over the cap
        } else if (!(go_m & slot_mask)) {
          slot_live = false;
          if (blk_m & slot_mask) overflow = true; else stuck = true;
        }
      }
    }

    // ---- a6 metrics (all lanes participate in the shuffles)
    const bool contrib = slot_on && valid && d < p;
    const int64_t mk = seg_max(contrib ? (int64_t)free_t : (int64_t)0, p2);
    const int64_t sumbusy = seg_sum(contrib ? busy : (int64_t)0, p2);
    const int64_t Md = stat + peak;
    const int64_t Mmax = seg_max(contrib ? Md : (int64_t)0, p2);
    const bool any_over = (__ballot_sync(FULLMASK, contrib && Md > sl.cap) & slot_mask) != 0;
    if (!slot_on) status = -1;
    else if (!valid) status = ADAPTIS_CAND_INVALID;
    else if (overflow) status = -2;  // re-evaluated by the fallback kernel
    else if (FUSED && any_over) status = ADAPTIS_CAND_OVER_CAP;
    else if (stuck) status = ADAPTIS_CAND_STUCK;
    else if (any_over) status = ADAPTIS_CAND_OVER_CAP;
    else status = ADAPTIS_CAND_OK;

    if (d == 0 && slot_on) {
      if (status == -2) {
        unsigned int k = atomicAdd(sl.overflow_count, 1u);
        if (k < sl.overflow_cap) sl.overflow_idx[k] = idx;
      } else {
        if (status == ADAPTIS_CAND_INVALID) ++winvalid;
        if (sl.key) {
          if (status == ADAPTIS_CAND_OK) {
            unsigned long long key = ((unsigned long long)mk << sl.key_bits) | idx;
            wkey = key < wkey ? key : wkey;
          }
        } else {
          const uint64_t o = idx - sl.eval_first;
          if (sl.out_status) sl.out_status[o] = (uint8_t)status;
          if (sl.out_makespan) sl.out_makespan[o] = status == 0 ? mk : INT64_MAX;
          if (sl.out_peak)
            sl.out_peak[o] = (status == 0 || status == ADAPTIS_CAND_OVER_CAP) ? Mmax : 0;
          if (sl.out_bubble)
            sl.out_bubble[o] = status == 0
                ? (float)(1.0 - (double)sumbusy / ((double)p * (double)mk)) : 0.0f;
        }
      }
    }
    if (sl.out_report && contrib && status >= 0) {
      sl.out_report[d] = (int64_t)free_t;
      sl.out_report[p + d] = busy;
      sl.out_report[2 * p + d] = Md;
    }
    __syncwarp();
  }

  // ---- a7 argmin: warp min -> one atomicMin per warp
  if (sl.key) {
    for (int o = 16; o > 0; o >>= 1) {
      unsigned long long x = __shfl_xor_sync(FULLMASK, wkey, o);
      wkey = x < wkey ? x : wkey;
    }
    if (lane == 0 && wkey != (~0ull >> 1)) atomicMin(sl.key, wkey);
  }
  for (int o = 16; o > 0; o >>= 1) {
    winvalid += __shfl_xor_sync(FULLMASK, winvalid, o);
    wtasks += __shfl_xor_sync(FULLMASK, wtasks, o);
  }
  if (lane == 0 && winvalid) atomicAdd(sl.n_invalid, winvalid);
  if (lane == 0 && wtasks) atomicAdd(sl.n_tasks, wtasks);
}

// ------------------------------------------------------------------------------
size_t smem_bytes(const SegLaunch& s, bool fallback) {
  const size_t tsz = s.use_int64 ? 8 : 4;
  const size_t pre = ((size_t)kNumCols * (s.L + 1) * 8 + 15) & ~(size_t)15;
  const size_t cuts = (((size_t)s.G * (s.S + 1) * 2) + 15) & ~(size_t)15;
  const size_t scsz = s.use_int64 ? sizeof(StageC<int64_t>) : sizeof(StageC<int32_t>);
  const size_t sc = (size_t)(s.v > 1 ? s.v : 0) * 32 * scsz;
  const size_t ring = fallback ? 0 : (size_t)2 * s.ring_k * s.G * s.S * tsz;
  return pre + kWarpsPerCta * (cuts + sc + ring);
}

using KFn = void (*)(const DevTables, const SegLaunch);

template <int POLICY, int V, typename T>
static KFn pick_fb(bool fallback) {
  return fallback ? (KFn)seg_kernel<POLICY, V, T, true> : (KFn)seg_kernel<POLICY, V, T, false>;
}
template <int POLICY, typename T>
static KFn pick_v(int v, bool fb) {
  switch (v) {
    case 1: return pick_fb<POLICY, 1, T>(fb);
    case 2: return pick_fb<POLICY, 2, T>(fb);
    case 3: return pick_fb<POLICY, 3, T>(fb);
    default: return pick_fb<POLICY, 4, T>(fb);
  }
}
template <typename T>
static KFn pick_pol(int pol, int v, bool fb) {
  switch (pol) {
    case ADAPTIS_GPIPE: return pick_v<ADAPTIS_GPIPE, T>(v, fb);
    case ADAPTIS_ONEF1B: return pick_v<ADAPTIS_ONEF1B, T>(v, fb);
    case ADAPTIS_ZB: return pick_v<ADAPTIS_ZB, T>(v, fb);
    default: return pick_v<ADAPTIS_GREEDY, T>(v, fb);
  }
}
static KFn pick(const SegLaunch& s, bool fb) {
  return s.use_int64 ? pick_pol<int64_t>(s.policy, s.v, fb) : pick_pol<int32_t>(s.policy, s.v, fb);
}

int occupancy_ctas_per_sm(const SegLaunch& s, bool fallback) {
  KFn f = pick(s, fallback);
  size_t sm = smem_bytes(s, fallback);
  if (cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) != cudaSuccess)
    return 0;
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, f, kWarpsPerCta * 32, sm) != cudaSuccess)
    return 0;
  return n;
}

int launch_segment(const DevTables& t, const SegLaunch& s, int num_sms, void* stream,
                   bool fallback, unsigned grid_limit) {
  KFn f = pick(s, fallback);
  size_t sm = smem_bytes(s, fallback);
  cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return (int)e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, f, kWarpsPerCta * 32, sm);
  if (e != cudaSuccess) return (int)e;
  if (per_sm < 1) return (int)cudaErrorInvalidConfiguration;
  unsigned grid = (unsigned)num_sms * (unsigned)per_sm;
  // no more CTAs than there is work for
  const uint64_t warps_needed = (s.n_pos + s.G - 1) / s.G;
  const uint64_t ctas_needed = (warps_needed + kWarpsPerCta - 1) / kWarpsPerCta;
  if (ctas_needed < grid) grid = (unsigned)(ctas_needed ? ctas_needed : 1);
  if (grid_limit && grid > grid_limit) grid = grid_limit;
  f<<<grid, kWarpsPerCta * 32, sm, (cudaStream_t)stream>>>(t, s);
  e = cudaGetLastError();
  return (int)e;
}

}  // namespace adaptis
