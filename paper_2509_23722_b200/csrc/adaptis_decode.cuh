// adaptis_decode.cuh — candidate index -> partition (R19), shared by the host
// entry point adaptis_decode and the device kernels (one implementation inside
// libadaptis; the CPU oracle has its own, independent one).
#pragma once
#include <cstdint>

#include "adaptis_internal.h"

#ifdef __CUDACC__
#define ADAPTIS_HD __host__ __device__ __forceinline__
#else
#define ADAPTIS_HD inline
#endif

namespace adaptis {

// binom[n * (MAX_S + 1) + k] = C(n, k) (saturating);
// ball[(group * MAX_S + n) * (kMaxRadius + 1) + r] = #{x in Z^n : |x|_1 <= r};
// seeds[group * MAX_S + i] = interior cut i+1 of the group's seed.
// Writes cuts[0..S]; returns whether they are strictly increasing (a valid
// partition). prank is the rank of the partition inside its group.
ADAPTIS_HD bool decode_cuts(const uint64_t* binom, const uint64_t* ball, const int16_t* seeds,
                            int group, int part_mode, int radius, int S, int L, uint64_t prank,
                            int16_t* cuts) {
  cuts[0] = 0;
  cuts[S] = (int16_t)L;
  if (part_mode == ADAPTIS_PART_FULL) {
    // colex unranking of the cut set {c_1 < ... < c_{S-1}} subset of {1..L-1}:
    // rank = sum_i C(c_i - 1, i); the largest c with C(c-1, i) <= rank is c_i
    int hi = L - 1;
    for (int i = S - 1; i >= 1; --i) {
      int c = hi;
      while (binom[(size_t)(c - 1) * (ADAPTIS_MAX_S + 1) + i] > prank) --c;
      prank -= binom[(size_t)(c - 1) * (ADAPTIS_MAX_S + 1) + i];
      cuts[i] = (int16_t)c;
      hi = c - 1;
    }
    return true;
  }
  // L1 ball: delta_1 most significant, digit order 0, -1, +1, -2, +2, ...
  const int n = S - 1;
  const uint64_t* cnt = ball + (size_t)group * ADAPTIS_MAX_S * (kMaxRadius + 1);
  const int16_t* seed = seeds + group * ADAPTIS_MAX_S;
  int rem = radius, prev = 0;
  bool ok = true;
  for (int i = 1; i <= n; ++i) {
    const uint64_t* row = cnt + (size_t)(n - i) * (kMaxRadius + 1);
    int dsel = 0;
    uint64_t sub = row[rem];
    if (prank >= sub) {
      prank -= sub;
      for (int a = 1; a <= rem; ++a) {
        sub = row[rem - a];
        if (prank < sub) { dsel = -a; break; }
        prank -= sub;
        if (prank < sub) { dsel = a; break; }
        prank -= sub;
      }
    }
    const int c = seed[i - 1] + dsel;
    rem -= dsel < 0 ? -dsel : dsel;
    ok = ok && (c > prev);
    prev = c;
    cuts[i] = (int16_t)(c < -32768 ? -32768 : (c > 32767 ? 32767 : c));
  }
  return ok && (L > prev);
}

// Block-cyclic shard map: the global index range [lo, hi) is cut
// into chunks of 2^kChunkBits indices, chunk k belonging to rank k mod world;
// position `pos` of this rank's share maps to a global index. first_chunk, n0
// and start0 describe the rank's first (possibly partial) chunk.
ADAPTIS_HD uint64_t shard_index(uint64_t pos, uint64_t n0, uint64_t start0, uint64_t first_chunk,
                                int world) {
  if (pos < n0) return start0 + pos;
  const uint64_t q = pos - n0;
  const uint64_t t = q >> kChunkBits;
  return ((first_chunk + (t + 1) * (uint64_t)world) << kChunkBits) + (q & ((1ull << kChunkBits) - 1));
}

}  // namespace adaptis
