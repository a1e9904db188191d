// adaptis_internal.h — private host/device contract of libadaptis.so (not part
// of the C ABI). Everything here belongs to the CUDA path; the CPU oracle
// (oracle/) shares none of it.
#pragma once
#include <cstdint>

#include "../../include/adaptis.h"

namespace adaptis {

constexpr int kChunkBits = 16;  // block-cyclic shard chunk = 65536 indices
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
  int64_t* out_report;          // optional [3][p]: T_d, busy_d, M_d (single candidate)
  unsigned long long* cursor;   // work-claim counter (zeroed per launch)
  unsigned int* overflow_count; // candidates whose fast-path rings filled up
  uint64_t* overflow_idx;       // their global indices (capacity overflow_cap)
  unsigned int overflow_cap;
  unsigned long long* n_invalid;// invalid decodes counted by this launch
  unsigned long long* n_tasks;  // simulated tasks counted by this launch
  // fallback mode: positions index overflow_idx_in[] instead of [lo, hi)
  const uint64_t* list_idx;
  int ring_k;                   // ring slots (fast path: kRingK; fallback: >= m)
  int64_t* gring;               // fallback: global ring scratch
  int use_int64;                // 0: int32 ticks (host-proved bound), 1: int64 ticks
};

// launchers implemented in adaptis_kernels.cu
int launch_segment(const DevTables& t, const SegLaunch& s, int num_sms, void* stream,
                   bool fallback, unsigned grid_limit);
int occupancy_ctas_per_sm(const SegLaunch& s, bool fallback);
size_t smem_bytes(const SegLaunch& s, bool fallback);

}  // namespace adaptis
