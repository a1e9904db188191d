// adaptis_internal.h — private host/device contract of libadaptis.so (not part
// of the C ABI). Everything here belongs to the CUDA path; the CPU oracle
// (oracle/) shares none of it.
#pragma once
#include <cstdint>
#include <vector>

#include "../../include/adaptis.h"

namespace adaptis {

constexpr int kChunkBits = 16;  // block-cyclic shard chunk = 65536 indices
constexpr int kTickI32 = 0, kTickI64 = 1, kTickF32 = 2;
constexpr int kNumCols = 6;     // prefix columns: t_f, t_b, t_w, act, stash, weight+grad
constexpr int kColTF = 0, kColTB = 1, kColTW = 2, kColAct = 3, kColStash = 4, kColWG = 5;
constexpr int kRingK = 8;       // fast-path ring slots per stage and direction (power of two)
constexpr int kWarpsPerCta = 4;
constexpr int kMaxBinomN = 160; // FULL spaces: binomial table C(n, k), n < 160, k <= 64
constexpr int kMaxRadius = 256; // BALL spaces: count table N[n][r], r <= 256

// Device-resident tables of one prepared problem (uploaded once).
struct DevTables {
  const int64_t* cols;      // [kNumCols][L]   raw layer columns (weight+grad merged)
  const int64_t* comm;      // [L]
  const uint64_t* binom;    // [kMaxBinomN][ADAPTIS_MAX_S + 1], saturating
  const uint64_t* ball;     // [n_groups][ADAPTIS_MAX_S][kMaxRadius + 1]
  const int16_t* seeds;     // [n_groups][ADAPTIS_MAX_S]  (interior cuts of the BALL seed)
  const double* colsf;      // FP32 cost mode: [3][L] t_f, t_b, t_w as real ticks
  const float* commf;       // FP32 cost mode: [L] comm as real ticks
  const int64_t* pre;       // [kNumCols][L + 1] prefix sums of cols (sequential GREEDY setup)
};

// One launch = one (group, combo) segment of the canonical order (R19),
// intersected with a requested index range and this rank's shard.
struct SegLaunch {
  // problem
  int L, p, m, p2, log2p2, G;   // G = candidate slots per warp = 32 / p2
  int64_t cap;
  // candidate family
  int v, S, placement, policy, part_mode, radius, group;
  uint64_t seg_base;            // global index of the segment's first candidate
  // positions -> global indices (block-cyclic shard of [lo, hi))
  uint64_t lo, hi;              // global index range handled by this launch
  uint64_t n_pos;               // positions this rank processes
  uint64_t first_chunk;         // this rank's first chunk intersecting [lo, hi)
  uint64_t n0;                  // positions in that first (possibly partial) chunk
  uint64_t start0;              // global index of position 0
  int world;
  // outputs
  int key_bits;                 // index bits of the packed argmin key
  unsigned long long* key;      // search: atomicMin target (nullptr in eval mode)
  uint64_t eval_first;          // eval: results at [idx - eval_first]
  int64_t* out_makespan;
  int64_t* out_peak;
  float* out_bubble;
  uint8_t* out_status;
  float* out_makespan_f32;
  int64_t* out_report;          // optional [candidate][3][p]: T_d, busy_d, M_d, at idx - eval_first
  unsigned long long* cursor;   // work-claim counter (zeroed per launch)
  unsigned int* overflow_count; // candidates whose fast-path rings filled up
  uint64_t* overflow_idx;       // their global indices (capacity overflow_cap)
  unsigned int overflow_cap;
  unsigned long long* n_invalid;// invalid decodes counted by this launch
  unsigned long long* n_tasks;  // simulated tasks counted by this launch
  unsigned long long* n_rounds; // [0] warp rounds, [1] live device-lane rounds
  unsigned long long* n_pruned; // candidates skipped by the exact lower-bound prune
  int prune;                    // search: skip candidates whose LB key exceeds the incumbent
  // fallback mode: positions index overflow_idx_in[] instead of [lo, hi)
  const uint64_t* list_idx;
  // explicit-plan mode (adaptis_eval_plans): position q evaluates plan list_out[q]
  // (also its output slot); cuts come from list_cuts[plan][ADAPTIS_MAX_S + 1]
  const uint64_t* list_out;
  const int16_t* list_cuts;
  // explicit-index mode (adaptis_eval_indices): position q writes output slot
  // list_slot[q], which holds global index slot_idx[slot]; overflowed
  // candidates record their slot, so the fallback re-run lists slots too
  const uint64_t* list_slot;
  // LIST policies (R30): device d of candidate slot o runs
  // list_tasks[list_task_off[o * (p + 1) + d] .. list_task_off[o * (p + 1) + d + 1])
  const adaptis_task* list_tasks;
  const uint64_t* list_task_off;
  const uint64_t* slot_idx;
  // report mode with communication accounting (R29): every committed task of
  // candidate o on device d is appended to trace[(o * p + d) * trace_cap + k]
  // and the count stored in trace_n[o * p + d]
  struct TraceEntry* trace;
  int* trace_n;
  int trace_cap;
  int ring_k;                   // ring slots (fast path: kRingK; fallback: >= m)
  int64_t* gring;               // fallback: global ring scratch
  int tick;                     // kTickI32 (host-proved bound), kTickI64, kTickF32 (fp32 variant)
  // static-order kernel (adaptis_fixed.cu): the segment's F/B entries and arrival slots
  const uint32_t* fx_ent;
  int fx_n;
  int fx_slots;
};

// one committed task in report mode (R29): its compute interval and, when its
// output crosses devices, the transfer [fin, fin + oc] to device `tgt` (-1: none)
struct TraceEntry {
  int64_t start, fin;
  int32_t oc, tgt;
  int16_t kind, stage;  // the task (F 0, B 1, W 2; stage index, micro-batch), for the
  int32_t mb;           // memory timeline and the realised lists
};

#ifdef __CUDACC__
#define ADAPTIS_LAYOUT_HD __host__ __device__ __forceinline__
#else
#define ADAPTIS_LAYOUT_HD inline
#endif

// Shared-memory layout of one warp of the segment kernel (after the CTA's
// prefix table): task records [3 kinds][V chunks][32 lanes], memory deltas
// (split policies), the slots' cuts, and the fast-path rings
// [2 directions][K slots][G*S stages].
struct WarpLayout {
  int rec_off, dmem_off, cuts_off, cnt_off, gaux_off, cold_off, ring_off, per_warp;
  ADAPTIS_LAYOUT_HD size_t prefix_bytes(int L) const {
    return ((size_t)kNumCols * (L + 1) * 8 + 15) & ~(size_t)15;
  }
};
ADAPTIS_LAYOUT_HD int align16(int x) { return (x + 15) & ~15; }
ADAPTIS_LAYOUT_HD WarpLayout warp_layout(int S, int G, int V, int K, int tsz, int rsz, bool gring,
                                         int gaux_sz = 0) {
  WarpLayout l;
  int off = 0;
  l.rec_off = off;  off += 3 * V * 32 * rsz;
  l.dmem_off = off; off += 3 * V * 32 * 8;
  l.cuts_off = off; off += align16(G * (S + 1) * 2);
  l.cnt_off = off;  off += 32 * 4 * 4;  // GREEDY produced-count words [chunk][lane]
  l.gaux_off = off; off += align16(V * 32 * gaux_sz);  // GREEDY per-chunk statics
  l.cold_off = off; off += 32 * 64;                    // per-lane cold state (LaneCold)
  l.ring_off = off; if (!gring) off += 2 * K * G * S * tsz;
  l.per_warp = align16(off);
  return l;
}

// launchers implemented in adaptis_kernels.cu
// R29 communication accounting over the traces of n candidates: per device,
// comm = sum of incident transfer lengths, exposed = |union of incident
// transfers within [0, T_d], outside the device's compute intervals|; written
// to report rows 3 and 4 ([candidate][5][p]). Returns a cudaError_t.
int launch_comm_account(const TraceEntry* trace, const int* trace_n, int trace_cap, int p,
                        uint64_t n, int64_t* report, void* stream);
int launch_segment(const DevTables& t, const SegLaunch& s, int num_sms, void* stream,
                   bool fallback, unsigned grid_limit);
// Memory timeline (Eq. 2; SPEC memory_timeline, R35) of n traced plans:
// per (plan, device) the breakpoints (time, static + dynamic bytes) in event
// order, starting at (0, static), at [(o * p + d) * pcap], their count in
// npts[o * p + d], and the first time the bytes exceed cap (-1: none) in
// first[o * p + d]. plan_info[o] = v | placement << 4 | fused << 8. Returns a
// cudaError_t.
int launch_mem_timeline(const TraceEntry* trace, const int* trace_n, int trace_cap, int p, uint64_t n,
                        const int16_t* cuts, const int32_t* plan_info, const int64_t* pre, int L,
                        int64_t cap, adaptis_mem_point* points, int pcap, int* npts, int64_t* first,
                        void* stream);
// R34 engine contention on explicit lists (adaptis_contend.cu): one warp per
// plan slot (32 / p2 plans per warp); scratch [n][stride] int64 with stride >=
// 5 * S * m; Sm = the largest S of the batch. Returns a cudaError_t.
int launch_contend(const int64_t* cols, const int64_t* comm, int L, int p, int m, int64_t cap, uint64_t n,
                   const adaptis_plan* plans, const adaptis_task* tasks, const uint64_t* offsets,
                   int64_t* scratch, uint64_t stride, int64_t* makespan, int64_t* peak, float* bubble,
                   uint8_t* status, int64_t* report, unsigned long long* n_tasks, int Sm, void* stream);
// R36 (contention on realised orders): a segment's decode tables and shape
struct RealisedSeg {
  const uint64_t* binom;
  const uint64_t* ball;
  const int16_t* seeds;
  int group, part_mode, radius, S, L, v, placement, fused;
  uint64_t base;  // global index of the segment's first candidate
};
int launch_realised_lists(const TraceEntry* trace, const int* trace_n, int trace_cap, int p, uint64_t n,
                          uint64_t first, const uint8_t* status, const RealisedSeg& seg, adaptis_plan* plans,
                          adaptis_task* tasks, uint64_t* offsets, uint64_t* slot_idx, unsigned int* n_kept,
                          void* stream);
int launch_contended_key(const int64_t* makespan, const uint8_t* status, const uint64_t* slot_idx, uint64_t n,
                         uint64_t first, int key_bits, unsigned long long* key, void* stream);
int occupancy_ctas_per_sm(const SegLaunch& s, bool fallback);
// sequential GREEDY kernel (adaptis_seqg.cu): one thread per candidate
bool seqg_eligible(const SegLaunch& s, bool seq_ok, int max_smem, int min_warps);
int launch_seqg(const DevTables& t, const SegLaunch& s, int num_sms, void* stream);
// static-order kernel for GPIPE / ONEF1B / ZB (adaptis_fixed.cu): one thread per candidate
bool fx_build_order(int policy, int placement, int p, int v, int m, std::vector<uint32_t>& ent, int& slots);
bool fixed_eligible(const SegLaunch& s, bool seq_ok, int max_smem, int slots);
int launch_fixed(const DevTables& t, const SegLaunch& s, int num_sms, void* stream);
size_t smem_bytes(const SegLaunch& s, bool fallback);

}  // namespace adaptis
