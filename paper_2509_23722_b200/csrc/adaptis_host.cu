// adaptis_host.cu — the C ABI of libadaptis.so (include/adaptis.h): validation,
// host-derived tables (prefix columns, binomials, L1-ball counts, min-max seed),
// device residency, segment launches, the cross-GPU argmin and the winner report.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <tuple>
#include <vector>

#include "adaptis_decode.cuh"
#include "adaptis_internal.h"

using namespace adaptis;

namespace {

thread_local std::string g_tls_error;

struct Seg {               // one (group, combo) segment of the canonical order (R19)
  int group, combo, v, S, placement, policy, part_mode, radius;
  uint64_t base, count;
};

// fixed combo table (R12)
bool combo_of(int v, int k, int* placement, int* policy) {
  if (v == 1) {
    if (k < 0 || k > 3) return false;
    *placement = ADAPTIS_SEQ; *policy = k; return true;
  }
  if (k >= 0 && k <= 3) { *placement = ADAPTIS_INTERLEAVED; *policy = k; return true; }
  if (k == 4) { *placement = ADAPTIS_WAVE; *policy = ADAPTIS_GPIPE; return true; }
  if (k == 5) { *placement = ADAPTIS_WAVE; *policy = ADAPTIS_GREEDY; return true; }
  return false;
}

uint64_t sat_add(uint64_t a, uint64_t b) { return a > UINT64_MAX - b ? UINT64_MAX : a + b; }
uint64_t sat_mul(uint64_t a, uint64_t b) {
  if (a == 0 || b == 0) return 0;
  return a > UINT64_MAX / b ? UINT64_MAX : a * b;
}

}  // namespace

struct adaptis_prepared {
  // host copies
  int L = 0, p = 0, m = 0, n_groups = 0;
  int64_t cap = 0;
  double tick_seconds = 0;
  int64_t tokens_per_mb = 0;
  std::vector<Seg> segs;
  uint64_t N = 0;
  int key_bits = 1;
  int tick = kTickI32;
  bool seq_ok = false;  // sequential kernels admitted: U < 2^28, latencies < 2^16
  // static orders of the fixed-order segments (adaptis_fixed.cu), built on first use
  struct FxOrder { int policy, placement, v; bool ok; int n, slots; uint32_t* d_ent; };
  std::vector<FxOrder> fx_orders;
  std::vector<uint64_t> h_binom, h_ball;
  std::vector<int16_t> h_seeds;
  std::vector<int64_t> h_cols, h_comm;  // host copies of the layer columns (kNumCols x L) and comm
  int group_v[ADAPTIS_MAX_GROUPS] = {0};
  // device
  double* d_colsf = nullptr;
  float* d_commf = nullptr;
  int64_t* d_cols = nullptr;
  int64_t* d_pre = nullptr;
  int64_t* d_comm = nullptr;
  uint64_t* d_binom = nullptr;
  uint64_t* d_ball = nullptr;
  int16_t* d_seeds = nullptr;
  DevTables tabs{};
  adaptis_ctx* owner = nullptr;
};

struct adaptis_ctx {
  int device = 0, rank = 0, world = 1, num_sms = 148;
  int max_smem = 232448;  // cudaDevAttrMaxSharedMemoryPerBlockOptin (queried at create)
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  adaptis_allreduce_min_fn allreduce = nullptr;
  void* allreduce_user = nullptr;
  std::string err;
  uint64_t launches = 0;
  uint64_t fallback_cands = 0;
  int prune = 0;
  uint64_t counters[3] = {0, 0, 0};
  uint64_t last_tasks = 0, last_invalid = 0, last_pruned = 0;  // counts of the last run_jobs
  std::vector<cudaEvent_t> seg_events;
  std::vector<adaptis_launch_info> last_info;
  // scratch
  unsigned long long* d_scratch = nullptr;  // [0] key, [1] n_invalid, [2..] cursors/overflow counts
  size_t scratch_words = 0;
  uint64_t* d_overflow = nullptr;
  size_t overflow_cap = 0;
  int64_t* d_gring = nullptr;
  size_t gring_bytes = 0;
  int64_t* d_report = nullptr;  // winner report rows [5][MAX_P], then the winner's SoA block
  unsigned char* h_report = nullptr;  // pinned host copy of d_report (one D2H per search)
  TraceEntry* d_wtrace = nullptr;  // winner traces (R29), grown as needed
  int* d_wtrace_n = nullptr;
  size_t wtrace_entries = 0;
};

// winner report block behind the five report rows: makespan, peak, fp32
// makespan, bubble, status (one allocation and one D2H per search)
constexpr size_t kReportBytes = 5 * ADAPTIS_MAX_P * 8;
constexpr size_t kWinBytes = 40;  // + the contended search's key word at +32

namespace {

adaptis_status fail(adaptis_ctx* ctx, adaptis_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  if (ctx) ctx->err = buf; else g_tls_error = buf;
  return s;
}

#define CU(ctx, call)                                                                    \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return fail(ctx, ADAPTIS_ECUDA, "%s: %s", #call, cudaGetErrorString(e_));         \
  } while (0)

// -- validation (S:62-66 style: the message names the field) -------------------
adaptis_status validate(adaptis_ctx* ctx, const adaptis_problem* pr, const adaptis_space* sp) {
  if (!pr) return fail(ctx, ADAPTIS_EINVAL, "problem is NULL");
  if (!sp) return fail(ctx, ADAPTIS_EINVAL, "space is NULL");
  const adaptis_layers& Ly = pr->layers;
  if (Ly.L < 2 || Ly.L > 32767) return fail(ctx, ADAPTIS_EINVAL, "layers.L = %d not in [2, 32767]", Ly.L);
  const int64_t* cols[8] = {Ly.t_f, Ly.t_b, Ly.t_w, Ly.act_bytes, Ly.stash_bytes, Ly.weight_bytes,
                            Ly.grad_bytes, Ly.comm_ticks};
  const char* names[8] = {"t_f", "t_b", "t_w", "act_bytes", "stash_bytes", "weight_bytes",
                          "grad_bytes", "comm_ticks"};
  for (int c = 0; c < 8; ++c) {
    if (!cols[c]) return fail(ctx, ADAPTIS_EINVAL, "layers.%s is NULL", names[c]);
    const int n = (c == 7) ? Ly.L - 1 : Ly.L;
    for (int l = 0; l < n; ++l) {
      if (c < 3 && cols[c][l] < 1)  // R17: strictly positive durations
        return fail(ctx, ADAPTIS_EINVAL, "layers.%s[%d] < 1", names[c], l);
      if (cols[c][l] < 0) return fail(ctx, ADAPTIS_EINVAL, "layers.%s[%d] < 0", names[c], l);
      if (cols[c][l] > (int64_t)1 << 52)
        return fail(ctx, ADAPTIS_EINVAL, "layers.%s[%d] > 2^52", names[c], l);
    }
  }
  if (pr->cost_type != ADAPTIS_COST_TICKS && pr->cost_type != ADAPTIS_COST_FP32)
    return fail(ctx, ADAPTIS_EINVAL, "cost_type = %d", pr->cost_type);
  if (pr->cost_type == ADAPTIS_COST_FP32 && pr->costs_f32) {
    const char* fn[4] = {"t_f", "t_b", "t_w", "comm"};
    for (int c = 0; c < 4; ++c)
      for (int l = 0; l < (c == 3 ? Ly.L - 1 : Ly.L); ++l) {
        const float x = pr->costs_f32[(size_t)c * Ly.L + l];
        if (!(x == x) || x > 1e30f || (c < 3 && x < 1.0f) || (c == 3 && x < 0.0f))
          return fail(ctx, ADAPTIS_EINVAL, "costs_f32.%s[%d] = %g out of range", fn[c], l, (double)x);
      }
  }
  if (pr->p < 1 || pr->p > ADAPTIS_MAX_P) return fail(ctx, ADAPTIS_EINVAL, "p = %d not in [1, 32]", pr->p);
  if (pr->m < 1 || pr->m > 65535) return fail(ctx, ADAPTIS_EINVAL, "m = %d not in [1, 65535]", pr->m);
  if (pr->mem_cap_bytes < 0) return fail(ctx, ADAPTIS_EINVAL, "mem_cap_bytes < 0");
  if (sp->n_groups < 1 || sp->n_groups > ADAPTIS_MAX_GROUPS)
    return fail(ctx, ADAPTIS_EINVAL, "space.n_groups = %d not in [1, 4]", sp->n_groups);
  for (int g = 0; g < sp->n_groups; ++g) {
    const adaptis_group& G = sp->group[g];
    if (G.v < 1 || G.v > ADAPTIS_MAX_V)
      return fail(ctx, ADAPTIS_EINVAL, "space.group[%d].v = %d not in [1, 4]", g, G.v);
    const int S = pr->p * G.v;
    if (S > ADAPTIS_MAX_S) return fail(ctx, ADAPTIS_EINVAL, "space.group[%d]: S = p*v = %d > 64", g, S);
    if (S > Ly.L) return fail(ctx, ADAPTIS_EINVAL, "space.group[%d]: S = %d > layers.L = %d", g, S, Ly.L);
    if (G.v > 1 && pr->m % pr->p != 0)
      return fail(ctx, ADAPTIS_EINVAL, "space.group[%d]: v > 1 requires m %% p == 0 (R10)", g);
    if (G.part_mode != ADAPTIS_PART_FULL && G.part_mode != ADAPTIS_PART_BALL)
      return fail(ctx, ADAPTIS_EINVAL, "space.group[%d].part_mode = %d", g, G.part_mode);
    if (G.part_mode == ADAPTIS_PART_BALL && (G.radius < 0 || G.radius > kMaxRadius))
      return fail(ctx, ADAPTIS_EINVAL, "space.group[%d].radius = %d not in [0, %d]", g, G.radius, kMaxRadius);
    if (G.part_mode == ADAPTIS_PART_FULL && Ly.L > kMaxBinomN)
      return fail(ctx, ADAPTIS_EINVAL, "space.group[%d]: FULL partitions need L <= %d", g, kMaxBinomN);
    int nc = 0, a, b;
    for (int k = 0; k < 32; ++k)
      if ((G.combo_mask >> k) & 1u) {
        if (!combo_of(G.v, k, &a, &b))
          return fail(ctx, ADAPTIS_EINVAL, "space.group[%d].combo_mask bit %d is not a combo for v = %d", g, k, G.v);
        ++nc;
      }
    if (nc == 0) return fail(ctx, ADAPTIS_EINVAL, "space.group[%d].combo_mask is empty", g);
    if (G.part_mode == ADAPTIS_PART_BALL && G.seed_cuts) {
      int prev = 0;
      for (int i = 0; i < S - 1; ++i) {
        if (G.seed_cuts[i] <= prev || G.seed_cuts[i] >= Ly.L)
          return fail(ctx, ADAPTIS_EINVAL, "space.group[%d].seed_cuts[%d] = %d not increasing in [1, L-1]",
                      g, i, G.seed_cuts[i]);
        prev = G.seed_cuts[i];
      }
    }
  }
  return ADAPTIS_OK;
}

// -- R20 seed: min-max contiguous S-way split of w, lexicographically smallest cuts.
// Parametric search on the bound V with a greedy feasibility test (the
// oracle's exact DP is an independent implementation).
int min_parts(const std::vector<int64_t>& pre, int from, int L, int64_t V) {
  // fewest contiguous parts of rows [from, L) with every part sum <= V (greedy), or INT_MAX
  int parts = 0, i = from;
  while (i < L) {
    if (pre[i + 1] - pre[i] > V) return 1 << 30;
    int j = i + 1;
    while (j < L && pre[j + 1] - pre[i] <= V) ++j;
    ++parts;
    i = j;
  }
  return parts;
}

void seed_minmax(const adaptis_layers& Ly, int S, int16_t* cuts) {
  const int L = Ly.L;
  std::vector<int64_t> pre(L + 1, 0);
  for (int l = 0; l < L; ++l) pre[l + 1] = pre[l] + Ly.t_f[l] + Ly.t_b[l] + Ly.t_w[l];
  int64_t lo = 0, hi = pre[L];
  for (int l = 0; l < L; ++l) lo = std::max(lo, pre[l + 1] - pre[l]);
  while (lo < hi) {  // smallest V with a split into <= S parts (then exactly S: L >= S)
    int64_t mid = lo + (hi - lo) / 2;
    if (min_parts(pre, 0, L, mid) <= S) hi = mid; else lo = mid + 1;
  }
  const int64_t V = lo;
  int pos = 0;
  for (int t = 1; t <= S - 1; ++t) {
    for (int j = pos + 1; j <= L; ++j) {
      if (pre[j] - pre[pos] > V) break;
      const int rest = S - t;  // parts left for rows [j, L)
      if (L - j >= rest && min_parts(pre, j, L, V) <= rest) { cuts[t - 1] = (int16_t)j; pos = j; break; }
    }
  }
}

adaptis_status build_space(adaptis_ctx* ctx, const adaptis_problem* pr, const adaptis_space* sp,
                           adaptis_prepared* P) {
  adaptis_status st = validate(ctx, pr, sp);
  if (st != ADAPTIS_OK) return st;
  const adaptis_layers& Ly = pr->layers;
  P->L = Ly.L; P->p = pr->p; P->m = pr->m; P->cap = pr->mem_cap_bytes;
  P->tick_seconds = pr->tick_seconds; P->tokens_per_mb = pr->tokens_per_microbatch;
  P->n_groups = sp->n_groups;
  // binomials C(n, k) (saturating), n < kMaxBinomN, k <= MAX_S
  P->h_binom.assign((size_t)kMaxBinomN * (ADAPTIS_MAX_S + 1), 0);
  for (int n = 0; n < kMaxBinomN; ++n) {
    uint64_t c = 1;  // C(n, 0); C(n, k) = C(n, k-1) * (n-k+1) / k, exact while it fits
    for (int k = 0; k <= ADAPTIS_MAX_S && k <= n; ++k) {
      if (k > 0) {
        if (c == UINT64_MAX) { P->h_binom[(size_t)n * (ADAPTIS_MAX_S + 1) + k] = UINT64_MAX; continue; }
        unsigned __int128 x = (unsigned __int128)c * (uint64_t)(n - k + 1) / (uint64_t)k;
        c = x > (unsigned __int128)UINT64_MAX ? UINT64_MAX : (uint64_t)x;
      }
      P->h_binom[(size_t)n * (ADAPTIS_MAX_S + 1) + k] = c;
    }
  }
  // L1-ball counts by the closed form sum_k 2^k C(n,k) C(r,k)
  P->h_ball.assign((size_t)ADAPTIS_MAX_GROUPS * ADAPTIS_MAX_S * (kMaxRadius + 1), 0);
  P->h_seeds.assign((size_t)ADAPTIS_MAX_GROUPS * ADAPTIS_MAX_S, 0);
  auto C = [&](int n, int k) -> uint64_t {
    if (k < 0 || k > n) return 0;
    if (n < kMaxBinomN) return P->h_binom[(size_t)n * (ADAPTIS_MAX_S + 1) + std::min(k, n - k)];
    return UINT64_MAX;
  };
  uint64_t total = 0;
  P->segs.clear();
  for (int g = 0; g < sp->n_groups; ++g) {
    const adaptis_group& G = sp->group[g];
    const int S = pr->p * G.v;
    P->group_v[g] = G.v;
    uint64_t parts;
    if (G.part_mode == ADAPTIS_PART_FULL) {
      parts = C(Ly.L - 1, S - 1);
    } else {
      for (int n = 0; n < ADAPTIS_MAX_S; ++n)
        for (int r = 0; r <= G.radius; ++r) {
          uint64_t t = 0;
          for (int k = 0; k <= std::min(n, r); ++k)
            t = sat_add(t, sat_mul(sat_mul(1ull << std::min(k, 63), C(n, k)), C(r, k)));
          P->h_ball[((size_t)g * ADAPTIS_MAX_S + n) * (kMaxRadius + 1) + r] = t;
        }
      parts = P->h_ball[((size_t)g * ADAPTIS_MAX_S + (S - 1)) * (kMaxRadius + 1) + G.radius];
      int16_t* seed = &P->h_seeds[(size_t)g * ADAPTIS_MAX_S];
      if (G.seed_cuts) for (int i = 0; i < S - 1; ++i) seed[i] = G.seed_cuts[i];
      else seed_minmax(Ly, S, seed);
    }
    for (int k = 0; k < 32; ++k) {
      Seg s{};
      if (!((G.combo_mask >> k) & 1u) || !combo_of(G.v, k, &s.placement, &s.policy)) continue;
      s.group = g; s.combo = k; s.v = G.v; s.S = S; s.part_mode = G.part_mode; s.radius = G.radius;
      s.base = total; s.count = parts;
      if (parts == UINT64_MAX || total > ((1ull << 63) - 1) - parts)
        return fail(ctx, ADAPTIS_EOVERFLOW, "space size does not fit in 63 bits");
      total += parts;
      P->segs.push_back(s);
    }
  }
  P->N = total;
  // packed key: makespan << key_bits | index must fit in 63 bits
  int bits = 1;
  while (bits < 63 && (total - 1) >> bits) ++bits;
  P->key_bits = bits;
  // makespan bound U: every schedule's makespan is a path through the task DAG
  // plus list edges, so U = m * (sum of all durations + 2 * sum of boundary comms)
  unsigned __int128 U = 0;
  for (int l = 0; l < Ly.L; ++l) U += (unsigned __int128)(Ly.t_f[l] + Ly.t_b[l] + Ly.t_w[l]);
  for (int l = 0; l + 1 < Ly.L; ++l) U += 2 * (unsigned __int128)Ly.comm_ticks[l];
  U *= (unsigned __int128)pr->m;
  if (pr->cost_type == ADAPTIS_COST_FP32) {
    // fp32 makespans enter the key as their (order-preserving) 32-bit patterns
    if (bits > 31) return fail(ctx, ADAPTIS_EOVERFLOW, "fp32 keys need |space| < 2^31");
    P->tick = kTickF32;
    return ADAPTIS_OK;
  }
  if (bits >= 63 || U >= ((unsigned __int128)1 << (63 - bits)))
    return fail(ctx, ADAPTIS_EOVERFLOW, "makespan bound and %d index bits exceed the 63-bit key", bits);
  P->tick = U >= ((unsigned __int128)1 << 31) - 1 ? kTickI64 : kTickI32;
  if (getenv("ADAPTIS_FORCE_INT64")) P->tick = kTickI64;  // test hook: exercise the int64 path
  // the sequential kernels pack (at << 4 | device) into 32 bits and
  // both latencies of a stage into one word
  bool lat16 = true;
  for (int l = 0; l + 1 < Ly.L; ++l) lat16 = lat16 && Ly.comm_ticks[l] < (1 << 16);
  P->seq_ok = P->tick == kTickI32 && U < ((unsigned __int128)1 << 28) && lat16 &&
              !getenv("ADAPTIS_NO_SEQ");
  return ADAPTIS_OK;
}

adaptis_status upload(adaptis_ctx* ctx, const adaptis_problem* pr, adaptis_prepared* P) {
  const adaptis_layers& Ly = pr->layers;
  const int L = Ly.L;
  std::vector<int64_t> cols((size_t)kNumCols * L);
  for (int l = 0; l < L; ++l) {
    cols[(size_t)kColTF * L + l] = Ly.t_f[l];
    cols[(size_t)kColTB * L + l] = Ly.t_b[l];
    cols[(size_t)kColTW * L + l] = Ly.t_w[l];
    cols[(size_t)kColAct * L + l] = Ly.act_bytes[l];
    cols[(size_t)kColStash * L + l] = Ly.stash_bytes[l];
    cols[(size_t)kColWG * L + l] = Ly.weight_bytes[l] + Ly.grad_bytes[l];
  }
  std::vector<int64_t> comm(Ly.comm_ticks, Ly.comm_ticks + L);
  comm[L - 1] = 0;
  P->h_cols = cols;
  P->h_comm = comm;
  CU(ctx, cudaSetDevice(ctx->device));
  if (P->tick == kTickF32) {  // the fp32-cost variant's real-valued durations and latencies
    std::vector<double> cf((size_t)3 * L);
    std::vector<float> mf(L);
    for (int l = 0; l < L; ++l) {
      const float* c = pr->costs_f32;
      cf[l] = c ? (double)c[l] : (double)(float)Ly.t_f[l];
      cf[(size_t)L + l] = c ? (double)c[(size_t)L + l] : (double)(float)Ly.t_b[l];
      cf[(size_t)2 * L + l] = c ? (double)c[(size_t)2 * L + l] : (double)(float)Ly.t_w[l];
      mf[l] = l == L - 1 ? 0.0f : (c ? c[(size_t)3 * L + l] : (float)Ly.comm_ticks[l]);
    }
    CU(ctx, cudaMalloc(&P->d_colsf, cf.size() * 8));
    CU(ctx, cudaMalloc(&P->d_commf, mf.size() * 4));
    CU(ctx, cudaMemcpy(P->d_colsf, cf.data(), cf.size() * 8, cudaMemcpyHostToDevice));
    CU(ctx, cudaMemcpy(P->d_commf, mf.data(), mf.size() * 4, cudaMemcpyHostToDevice));
    P->tabs.colsf = P->d_colsf;
    P->tabs.commf = P->d_commf;
  }
  std::vector<int64_t> pre((size_t)kNumCols * (L + 1), 0);
  for (int c = 0; c < kNumCols; ++c)
    for (int l = 0; l < L; ++l)
      pre[(size_t)c * (L + 1) + l + 1] = pre[(size_t)c * (L + 1) + l] + cols[(size_t)c * L + l];
  CU(ctx, cudaMalloc(&P->d_cols, cols.size() * 8));
  CU(ctx, cudaMalloc(&P->d_pre, pre.size() * 8));
  CU(ctx, cudaMemcpyAsync(P->d_pre, pre.data(), pre.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
  CU(ctx, cudaMalloc(&P->d_comm, comm.size() * 8));
  CU(ctx, cudaMalloc(&P->d_binom, P->h_binom.size() * 8));
  CU(ctx, cudaMalloc(&P->d_ball, P->h_ball.size() * 8));
  CU(ctx, cudaMalloc(&P->d_seeds, P->h_seeds.size() * 2));
  CU(ctx, cudaMemcpyAsync(P->d_cols, cols.data(), cols.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
  CU(ctx, cudaMemcpyAsync(P->d_comm, comm.data(), comm.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
  CU(ctx, cudaMemcpyAsync(P->d_binom, P->h_binom.data(), P->h_binom.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
  CU(ctx, cudaMemcpyAsync(P->d_ball, P->h_ball.data(), P->h_ball.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
  CU(ctx, cudaMemcpyAsync(P->d_seeds, P->h_seeds.data(), P->h_seeds.size() * 2, cudaMemcpyHostToDevice, ctx->stream));
  CU(ctx, cudaStreamSynchronize(ctx->stream));  // host vectors die on return
  P->tabs.cols = P->d_cols; P->tabs.comm = P->d_comm; P->tabs.binom = P->d_binom;
  P->tabs.pre = P->d_pre;
  P->tabs.ball = P->d_ball; P->tabs.seeds = P->d_seeds;
  return ADAPTIS_OK;
}

adaptis_status ensure_scratch(adaptis_ctx* ctx, size_t words, size_t overflow_cap) {
  if (words > ctx->scratch_words) {
    // grow, keeping the words already there: a pass that continues from the
    // incumbent key of a previous pass (keep_key) reads word 0 after this
    unsigned long long* grown = nullptr;
    CU(ctx, cudaMalloc(&grown, words * 8));
    if (ctx->d_scratch) {
      CU(ctx, cudaMemcpyAsync(grown, ctx->d_scratch, ctx->scratch_words * 8, cudaMemcpyDeviceToDevice,
                              ctx->stream));
      CU(ctx, cudaStreamSynchronize(ctx->stream));
      cudaFree(ctx->d_scratch);
    }
    ctx->d_scratch = grown;
    ctx->scratch_words = words;
  }
  if (overflow_cap > ctx->overflow_cap) {
    if (ctx->d_overflow) cudaFree(ctx->d_overflow);
    ctx->d_overflow = nullptr;
    CU(ctx, cudaMalloc(&ctx->d_overflow, overflow_cap * 8));
    ctx->overflow_cap = overflow_cap;
  }
  if (!ctx->d_report) CU(ctx, cudaMalloc(&ctx->d_report, kReportBytes + kWinBytes));
  if (!ctx->h_report) CU(ctx, cudaMallocHost(&ctx->h_report, kReportBytes + kWinBytes));
  if (!ctx->d_wtrace_n) CU(ctx, cudaMalloc(&ctx->d_wtrace_n, ADAPTIS_MAX_P * sizeof(int)));
  return ADAPTIS_OK;
}

// The block-cyclic shard of [lo, hi): chunks of 2^16 indices, chunk k -> rank k mod world.
void shard(uint64_t lo, uint64_t hi, int rank, int world, SegLaunch* s) {
  s->n_pos = 0; s->n0 = 0; s->start0 = lo; s->first_chunk = 0; s->world = world;
  if (hi <= lo) return;
  const uint64_t CH = 1ull << kChunkBits;
  const uint64_t c_lo = lo >> kChunkBits, c_hi = (hi - 1) >> kChunkBits;
  const uint64_t w = (uint64_t)world;
  uint64_t c0 = c_lo + (((uint64_t)rank + w - (c_lo % w)) % w);
  if (c0 > c_hi) return;
  s->first_chunk = c0;
  s->start0 = std::max(lo, c0 * CH);
  const uint64_t end0 = std::min(hi, (c0 + 1) * CH);
  s->n0 = end0 - s->start0;
  uint64_t n = s->n0;
  for (uint64_t c = c0 + w; c <= c_hi; c += w) n += std::min(hi, (c + 1) * CH) - c * CH;
  s->n_pos = n;
}

constexpr size_t kOverflowPerSeg = 1u << 20;
// overflow list capacity of one job: the fixed orders' 8-slot shared rings can
// overflow on a large share of a segment (cfg5's v = 2 ZB: 38 %), so their lists
// hold up to 2^26 positions (512 MB) and only the overflowed candidates are
// re-run; beyond that (and for the other policies beyond 2^20) the whole shard
// is re-run in fallback mode
size_t overflow_cap_of(const SegLaunch& s) {
  if (const char* e = getenv("ADAPTIS_OVERFLOW_CAP"))  // test hook: exercise the whole-shard re-run
    return (size_t)std::min<uint64_t>(s.n_pos, (uint64_t)std::max(1, atoi(e)));
  const bool ringed = s.policy == ADAPTIS_ZB || s.policy == ADAPTIS_ONEF1B;
  return (size_t)std::min<uint64_t>(s.n_pos, ringed ? (1ull << 26) : kOverflowPerSeg);
}

// fast-path ring slots per stage and direction: GREEDY's F-first rule lets a
// producer run further ahead than the fixed orders do (DESIGN.md §"Rings")
int ring_slots(int policy, int m) {
  int mp = 1;
  while (mp < m) mp <<= 1;
  if (policy == ADAPTIS_GREEDY) return mp;  // GREEDY rings are never full: >= m slots
  // explicit orders (R30) need not produce an edge's items in micro-batch order,
  // so every micro-batch gets its own slot (Lemma 4 does not apply)
  if (policy == ADAPTIS_LIST || policy == ADAPTIS_LIST_FUSED) return mp;
  int k = kRingK;
  const char* e = getenv("ADAPTIS_RING_K");
  if (e && atoi(e) > 0) k = atoi(e);
  if (k > mp) k = mp;
  int pw = 1;
  while (pw < k) pw <<= 1;
  return pw;
}
// warps of sequential-kernel state an SM must hold for that kernel to be used
// (below, the lane-per-device kernel keeps more candidates in flight; measured
// on B200); ADAPTIS_SEQ_MINW overrides, ADAPTIS_NO_SEQ disables
int seq_min_warps() {
  const char* e = getenv("ADAPTIS_SEQ_MINW");
  return e ? atoi(e) : 0;  // 0: the kernel's per-placement default
}
// the static order of a GPIPE / ONEF1B / ZB segment for the static-order
// kernel, built and uploaded once per prepared problem; false when that kernel
// cannot take the segment (ADAPTIS_NO_FIXED=1 keeps the lane kernels)
bool fixed_order(adaptis_ctx* ctx, adaptis_prepared* P, SegLaunch& s) {
  if (s.policy != ADAPTIS_GPIPE && s.policy != ADAPTIS_ONEF1B && s.policy != ADAPTIS_ZB) return false;
  if (getenv("ADAPTIS_NO_FIXED") || !P->seq_ok) return false;
  const adaptis_prepared::FxOrder* fo = nullptr;
  for (const auto& o : P->fx_orders)
    if (o.policy == s.policy && o.placement == s.placement && o.v == s.v) fo = &o;
  if (!fo) {
    adaptis_prepared::FxOrder o{s.policy, s.placement, s.v, false, 0, 0, nullptr};
    std::vector<uint32_t> ent;
    if (fx_build_order(s.policy, s.placement, s.p, s.v, s.m, ent, o.slots) && !ent.empty() &&
        cudaMalloc(&o.d_ent, ent.size() * 4) == cudaSuccess) {
      if (cudaMemcpy(o.d_ent, ent.data(), ent.size() * 4, cudaMemcpyHostToDevice) == cudaSuccess) {
        o.ok = true;
        o.n = (int)ent.size();
      } else {
        cudaFree(o.d_ent);
        o.d_ent = nullptr;
      }
    }
    (void)ctx;
    P->fx_orders.push_back(o);
    fo = &P->fx_orders.back();
  }
  if (!fo->ok || !fixed_eligible(s, P->seq_ok, ctx->max_smem, fo->slots)) return false;
  s.fx_ent = fo->d_ent;
  s.fx_n = fo->n;
  s.fx_slots = fo->slots;
  return true;
}
constexpr uint64_t kSeedPass = 4096;  // indices per segment in the pruned search's seed pass
constexpr size_t kHdr = 8;  // [0] key [1] invalid [2] tasks [3] rounds [4] live lane-rounds [5] pruned
constexpr size_t kGreedySmemRing = 0;  // per warp: GREEDY rings live in global memory (L2)

// global-memory ring scratch for a launch with s.ring_k slots; bounds the grid
adaptis_status ensure_gring(adaptis_ctx* ctx, const adaptis_prepared* P, const SegLaunch& s,
                            unsigned* grid_limit) {
  const size_t tsz = P->tick == kTickI64 ? 8 : 4;
  const size_t per_warp = (size_t)2 * s.ring_k * s.G * s.S * tsz;
  const size_t budget = (size_t)1 << 30;
  unsigned gl = (unsigned)std::max<size_t>(1, budget / (per_warp * kWarpsPerCta));
  gl = std::min<unsigned>(gl, (unsigned)ctx->num_sms * 8);
  const size_t need = per_warp * kWarpsPerCta * gl;
  if (need > ctx->gring_bytes) {
    if (ctx->d_gring) cudaFree(ctx->d_gring);
    ctx->d_gring = nullptr;
    CU(ctx, cudaMalloc(&ctx->d_gring, need));
    ctx->gring_bytes = need;
  }
  *grid_limit = gl;
  return ADAPTIS_OK;
}

SegLaunch make_launch(const adaptis_prepared* P, const Seg& sg) {
  SegLaunch s{};
  s.L = P->L; s.p = P->p; s.m = P->m; s.cap = P->cap;
  int p2 = 1, lg = 0;
  while (p2 < P->p) { p2 <<= 1; ++lg; }
  s.p2 = p2; s.log2p2 = lg; s.G = 32 / p2;
  s.v = sg.v; s.S = sg.S; s.placement = sg.placement; s.policy = sg.policy;
  s.part_mode = sg.part_mode; s.radius = sg.radius; s.group = sg.group;
  s.seg_base = sg.base;
  s.key_bits = P->key_bits;
  s.ring_k = ring_slots(sg.policy, P->m);
  s.tick = P->tick;
  return s;
}

// One kernel launch of an evaluation: a segment of the canonical order (or a
// group of explicit plans) with its sharded position range, and the record
// reported through adaptis_ctx_launch_info.
struct Job {
  SegLaunch s;
  adaptis_launch_info info;
};

// Scratch words: [0] key [1] (unused) [2] (unused) [3] rounds [4] live
// lane-rounds [5] (unused), then per job i at kHdr + kSegWords*i: [0] cursor
// [1] overflow count [2] tasks [3] fallback cursor [4] fallback overflow count
// [5] invalid [6] pruned [7] fallback invalid [8] fallback pruned
// [9] fallback tasks. Counts are kept per job and per pass so that a fallback
// that re-runs a whole shard replaces that job's first-pass counts instead of
// adding to them (every candidate is counted once: invalid, pruned or simulated).
constexpr size_t kSegWords = 10;

// Launch every job on this context's stream; candidates whose fast-path rings
// filled up are re-run by the fallback kernel (exact, rings >= m).
// mode_search: pack keys into the key word; else write SoA results at
// idx - eval_first (and per-candidate reports when `report` is set).
struct TraceBuf {  // report mode with communication accounting (R29)
  TraceEntry* trace = nullptr;
  int* trace_n = nullptr;
  int cap = 0;
};

adaptis_status run_jobs(adaptis_ctx* ctx, adaptis_prepared* P, std::vector<Job>& jobs,
                        bool mode_search, const adaptis_results_soa* dout, uint64_t eval_first,
                        int64_t* report, float* kernel_ms, bool keep_key,
                        const TraceBuf* tb = nullptr) {
  const size_t nseg = jobs.size();
  const size_t nwords = kHdr + kSegWords * std::max<size_t>(nseg, 1);
  std::vector<size_t> ov_off(nseg + 1, 0);
  for (size_t i = 0; i < nseg; ++i) ov_off[i + 1] = ov_off[i] + overflow_cap_of(jobs[i].s);
  adaptis_status st = ensure_scratch(ctx, nwords, std::max<size_t>(ov_off[nseg], 1));
  if (st != ADAPTIS_OK) return st;
  while (ctx->seg_events.size() < 2 * nseg) {
    cudaEvent_t e;
    CU(ctx, cudaEventCreate(&e));
    ctx->seg_events.push_back(e);
  }
  unsigned long long* W = ctx->d_scratch;
  std::vector<unsigned long long> init(nwords, 0);
  init[0] = (~0ull) >> 1;
  if (keep_key)  // continue from the incumbent of a previous pass
    CU(ctx, cudaMemcpyAsync(W + 1, init.data() + 1, (nwords - 1) * 8, cudaMemcpyHostToDevice, ctx->stream));
  else
    CU(ctx, cudaMemcpyAsync(W, init.data(), nwords * 8, cudaMemcpyHostToDevice, ctx->stream));
  CU(ctx, cudaEventRecord(ctx->ev0, ctx->stream));
  std::vector<char> active(nseg, 0);
  for (size_t i = 0; i < nseg; ++i) {
    SegLaunch& s = jobs[i].s;
    if (s.n_pos == 0) continue;
    unsigned long long* sw = W + kHdr + kSegWords * i;
    s.key = mode_search ? W : nullptr;
    s.eval_first = eval_first;
    if (!mode_search && dout) {
      s.out_makespan = dout->makespan; s.out_peak = dout->peak_mem_bytes;
      s.out_bubble = dout->bubble_ratio; s.out_status = dout->status;
      s.out_makespan_f32 = dout->makespan_f32;
    }
    s.out_report = report;
    if (tb && P->tick != kTickF32) { s.trace = tb->trace; s.trace_n = tb->trace_n; s.trace_cap = tb->cap; }
    s.cursor = sw + 0;
    s.overflow_count = reinterpret_cast<unsigned int*>(sw + 1);
    s.overflow_idx = ctx->d_overflow + ov_off[i];
    s.overflow_cap = (unsigned)(ov_off[i + 1] - ov_off[i]);
    s.n_invalid = sw + 5;
    s.n_tasks = sw + 2;
    s.n_rounds = W + 3;
    s.n_pruned = sw + 6;
    s.prune = (mode_search && ctx->prune && P->tick != kTickF32) ? 1 : 0;
    // GREEDY rings hold all m items (its F-first rule can run m items ahead);
    // they live in global memory when they do not fit the shared-memory budget
    const size_t ring_bytes = (size_t)2 * s.ring_k * s.G * s.S * (P->tick == kTickI64 ? 8 : 4);
    static const size_t greedy_smem_ring =
        getenv("ADAPTIS_GREEDY_SMEM_RING") ? (size_t)atol(getenv("ADAPTIS_GREEDY_SMEM_RING")) : kGreedySmemRing;
    // the CTA's prefix table (6 x (L+1) int64) and the warps' state must fit in
    // shared memory; rings move to global memory when they do not fit beside them
    const bool direct_global = (s.policy == ADAPTIS_GREEDY && ring_bytes > greedy_smem_ring) ||
                               smem_bytes(s, false) > (size_t)ctx->max_smem || s.trace != nullptr ||
                               s.policy == ADAPTIS_LIST || s.policy == ADAPTIS_LIST_FUSED;
    if (smem_bytes(s, true) > (size_t)ctx->max_smem)
      return fail(ctx, ADAPTIS_EINVAL,
                  "layers.L = %d, S = %d: %zu B of shared memory per CTA needed, the device allows %d",
                  s.L, s.S, smem_bytes(s, true), ctx->max_smem);
    CU(ctx, cudaEventRecord(ctx->seg_events[2 * i], ctx->stream));
    int e;
    if (seqg_eligible(s, P->seq_ok, ctx->max_smem, seq_min_warps())) {
      // GREEDY as one exact event loop per thread (adaptis_seqg.cu); ring
      // overflows go to the global-ring fallback below like the fast path's
      jobs[i].info.kernel = 1;
      e = launch_seqg(P->tabs, s, ctx->num_sms, ctx->stream);
    } else if (fixed_order(ctx, P, s)) {
      // GPIPE / ONEF1B / ZB as one static task order, a thread per candidate
      jobs[i].info.kernel = 2;
      e = launch_fixed(P->tabs, s, ctx->num_sms, ctx->stream);
    } else if (direct_global) {
      unsigned grid_limit = 0;
      st = ensure_gring(ctx, P, s, &grid_limit);
      if (st != ADAPTIS_OK) return st;
      s.gring = ctx->d_gring;
      e = launch_segment(P->tabs, s, ctx->num_sms, ctx->stream, true, grid_limit);
    } else {
      e = launch_segment(P->tabs, s, ctx->num_sms, ctx->stream, false, 0);
    }
    if (e) return fail(ctx, ADAPTIS_ECUDA, "kernel launch (segment %zu): %s", i, cudaGetErrorString((cudaError_t)e));
    CU(ctx, cudaEventRecord(ctx->seg_events[2 * i + 1], ctx->stream));
    ctx->launches++;
    active[i] = 1;
  }
  // fallback for candidates whose fast-path rings filled up (exact re-run, rings >= m)
  std::vector<unsigned long long> words(nwords);
  CU(ctx, cudaMemcpyAsync(words.data(), W, nwords * 8, cudaMemcpyDeviceToHost, ctx->stream));
  CU(ctx, cudaStreamSynchronize(ctx->stream));
  std::vector<float> seg_ms(nseg, 0.0f);
  for (size_t i = 0; i < nseg; ++i)
    if (active[i]) CU(ctx, cudaEventElapsedTime(&seg_ms[i], ctx->seg_events[2 * i], ctx->seg_events[2 * i + 1]));
  for (size_t i = 0; i < nseg; ++i) {
    if (!active[i]) continue;
    const unsigned int cnt = (unsigned int)(words[kHdr + kSegWords * i + 1] & 0xffffffffu);
    if (cnt == 0) continue;
    ctx->fallback_cands += cnt;
    SegLaunch s = jobs[i].s;
    int K = 1;
    while (K < P->m) K <<= 1;
    s.ring_k = K;
    if (cnt <= jobs[i].s.overflow_cap) {
      if (s.list_slot) s.list_slot = s.overflow_idx;  // explicit-index mode records slots
      else s.list_idx = s.overflow_idx;
      s.n_pos = cnt;
    }  // else: re-run the whole segment shard in fallback mode
    unsigned long long* sw = W + kHdr + kSegWords * i;
    s.cursor = sw + 3;
    s.overflow_count = reinterpret_cast<unsigned int*>(sw + 4);
    s.overflow_cap = 0;
    s.n_invalid = sw + 7;
    s.n_pruned = sw + 8;
    s.n_tasks = sw + 9;
    unsigned grid_limit = 0;
    st = ensure_gring(ctx, P, s, &grid_limit);
    if (st != ADAPTIS_OK) return st;
    s.gring = ctx->d_gring;
    CU(ctx, cudaEventRecord(ctx->seg_events[2 * i], ctx->stream));
    int e = launch_segment(P->tabs, s, ctx->num_sms, ctx->stream, true, grid_limit);
    if (e) return fail(ctx, ADAPTIS_ECUDA, "fallback launch: %s", cudaGetErrorString((cudaError_t)e));
    CU(ctx, cudaEventRecord(ctx->seg_events[2 * i + 1], ctx->stream));
    ctx->launches++;
    active[i] = 2;
  }
  CU(ctx, cudaEventRecord(ctx->ev1, ctx->stream));
  CU(ctx, cudaStreamSynchronize(ctx->stream));
  if (kernel_ms) CU(ctx, cudaEventElapsedTime(kernel_ms, ctx->ev0, ctx->ev1));
  CU(ctx, cudaMemcpy(words.data(), W, nwords * 8, cudaMemcpyDeviceToHost));
  ctx->counters[1] += words[3];
  ctx->counters[2] += words[4];
  ctx->last_info.clear();
  uint64_t tasks = 0, invalid = 0, pruned = 0;
  for (size_t i = 0; i < nseg; ++i) {
    if (!active[i]) continue;
    float fb = 0.0f;
    if (active[i] == 2) CU(ctx, cudaEventElapsedTime(&fb, ctx->seg_events[2 * i], ctx->seg_events[2 * i + 1]));
    const unsigned long long* jw = words.data() + kHdr + kSegWords * i;
    // a whole-shard fallback re-counted every candidate of the job: its counts
    // replace the first pass's; a list fallback only saw the overflowed ones
    const bool whole = active[i] == 2 && (jw[1] & 0xffffffffu) > jobs[i].s.overflow_cap;
    const uint64_t jt = whole ? jw[9] : jw[2] + jw[9];
    invalid += whole ? jw[7] : jw[5] + jw[7];
    pruned += whole ? jw[8] : jw[6] + jw[8];
    adaptis_launch_info li = jobs[i].info;
    li.candidates = jobs[i].s.n_pos;
    li.tasks = jt;
    li.ms = seg_ms[i] + fb;
    li.fallback = active[i] == 2 ? (int32_t)(words[kHdr + kSegWords * i + 1] & 0xffffffffu) : 0;
    tasks += li.tasks;
    ctx->last_info.push_back(li);
  }
  ctx->counters[0] += tasks;
  ctx->last_tasks = tasks;
  ctx->last_invalid = invalid;
  ctx->last_pruned = pruned;
  return ADAPTIS_OK;
}

// Evaluate [lo, hi) (global indices) on this context's GPU: one job per
// segment the range touches, sharded block-cyclically over `world` ranks.
adaptis_status run_range(adaptis_ctx* ctx, adaptis_prepared* P, uint64_t lo, uint64_t hi,
                         bool mode_search, int rank, int world, const adaptis_results_soa* dout,
                         uint64_t eval_first, int64_t* report, float* kernel_ms,
                         bool keep_key = false, const TraceBuf* tb = nullptr) {
  std::vector<Job> jobs;
  for (const Seg& sg : P->segs) {
    const uint64_t a = std::max(lo, sg.base), b = std::min(hi, sg.base + sg.count);
    if (a >= b) continue;
    Job j{};
    j.s = make_launch(P, sg);
    shard(a, b, rank, world, &j.s);
    j.s.lo = a; j.s.hi = b;
    if (j.s.n_pos == 0) continue;
    j.info.group = sg.group; j.info.combo = sg.combo; j.info.v = sg.v;
    j.info.placement = sg.placement; j.info.policy = sg.policy;
    jobs.push_back(j);
  }
  return run_jobs(ctx, P, jobs, mode_search, dout, eval_first, report, kernel_ms, keep_key, tb);
}

void fill_plan(const adaptis_prepared& P, uint64_t index, adaptis_plan* out, bool* valid) {
  memset(out, 0, sizeof(*out));
  for (const Seg& s : P.segs) {
    if (index < s.base || index >= s.base + s.count) continue;
    out->v = s.v; out->placement = s.placement; out->policy = s.policy; out->S = s.S;
    bool ok = decode_cuts(P.h_binom.data(), P.h_ball.data(), P.h_seeds.data(), s.group, s.part_mode,
                          s.radius, s.S, P.L, index - s.base, out->cuts);
    if (valid) *valid = ok;
    return;
  }
}

// (placement, policy) admitted for v by the combo table (R12), and its combo bit
int combo_bit(int v, int placement, int policy) {
  for (int k = 0; k < 6; ++k) {
    int pl, po;
    if (combo_of(v, k, &pl, &po) && pl == placement && po == policy) return k;
  }
  return -1;
}

// Explicit plans on the device: one job per (v, placement, policy) group,
// positions mapped to plan (= output) indices in the caller's order.
int host_dev_of(int placement, int p, int s) {  // R12
  if (placement == ADAPTIS_SEQ) return s;
  if (placement == ADAPTIS_INTERLEAVED) return s % p;
  const int c = s / p, j = s - c * p;
  return (c & 1) ? p - 1 - j : j;
}

// R30: every (kind, own stage, mb) exactly once per device, F < B < W per (stage, mb)
// The public per-plan report (adaptis.h): the kernels' five rows T_d, busy_d,
// M_d, comm_d, exposed_d, completed by R29's derived terms OverlapTime(d) =
// comm_d - exposed_d and BubbleTime(d) = T_d - busy_d - exposed_d (Alg. 1
// Step 3), so that T_d = busy_d + comm_d + bubble_d - overlap_d.
constexpr int kReportRows = 7;
void expand_report(const int64_t* rep5, int64_t* out7, int p) {
  for (int r = 0; r < 5; ++r)
    for (int d = 0; d < p; ++d) out7[r * p + d] = rep5[r * p + d];
  for (int d = 0; d < p; ++d) {
    out7[5 * p + d] = rep5[3 * p + d] - rep5[4 * p + d];
    out7[6 * p + d] = rep5[d] - rep5[p + d] - rep5[4 * p + d];
  }
}

adaptis_status validate_lists(adaptis_ctx* ctx, const adaptis_prepared* P, const adaptis_plan* plans,
                              const adaptis_task* tasks, const uint64_t* offsets, uint64_t n) {
  const int p = P->p, m = P->m;
  for (uint64_t i = 0; i < n; ++i) {
    const adaptis_plan& pl = plans[i];
    const bool fused = pl.policy == ADAPTIS_LIST_FUSED;
    const int nk = fused ? 2 : 3, S = pl.S;
    std::vector<int64_t> pos((size_t)nk * S * m, -1);
    const uint64_t* off = offsets + i * (uint64_t)(p + 1);
    for (int d = 0; d < p; ++d) {
      if (off[d + 1] < off[d])
        return fail(ctx, ADAPTIS_EINVAL, "plans[%llu]: offsets of device %d decrease", (unsigned long long)i, d);
      for (uint64_t q = off[d]; q < off[d + 1]; ++q) {
        const adaptis_task& t = tasks[q];
        if (t.kind < 0 || t.kind >= nk || t.stage < 0 || t.stage >= S || t.mb < 0 || t.mb >= m ||
            host_dev_of(pl.placement, p, t.stage) != d)
          return fail(ctx, ADAPTIS_EINVAL, "plans[%llu] device %d task %llu (kind %d, stage %d, mb %d) is not a task of this device",
                      (unsigned long long)i, d, (unsigned long long)(q - off[d]), t.kind, t.stage, t.mb);
        int64_t& slot = pos[((size_t)t.kind * S + t.stage) * m + t.mb];
        if (slot >= 0)
          return fail(ctx, ADAPTIS_EINVAL, "plans[%llu] device %d lists (kind %d, stage %d, mb %d) twice",
                      (unsigned long long)i, d, t.kind, t.stage, t.mb);
        slot = (int64_t)q;
      }
    }
    for (int k = 0; k < nk; ++k)
      for (int s2 = 0; s2 < S; ++s2)
        for (int j = 0; j < m; ++j) {
          const int64_t x = pos[((size_t)k * S + s2) * m + j];
          if (x < 0)
            return fail(ctx, ADAPTIS_EINVAL, "plans[%llu]: (kind %d, stage %d, mb %d) is not listed",
                        (unsigned long long)i, k, s2, j);
          if (k > 0 && x < pos[((size_t)(k - 1) * S + s2) * m + j])
            return fail(ctx, ADAPTIS_EINVAL, "plans[%llu]: (kind %d, stage %d, mb %d) is listed before its %s",
                        (unsigned long long)i, k, s2, j, k == 1 ? "F" : "B");
        }
  }
  return ADAPTIS_OK;
}

// memory timeline request of run_plans (R35): per (plan, device) breakpoints
struct MemTimelineReq {
  int pcap = 0;                          // breakpoints per (plan, device)
  std::vector<adaptis_mem_point> points; // [n][p][pcap]
  std::vector<int> npts;                 // [n][p]
  std::vector<int64_t> first;            // [n][p], -1: no violation
};

adaptis_status run_plans(adaptis_ctx* ctx, adaptis_prepared* P, const adaptis_plan* plans,
                         uint64_t n, std::vector<int64_t>* mk, std::vector<int64_t>* peak,
                         std::vector<float>* bubble, std::vector<uint8_t>* status,
                         std::vector<int64_t>* report, float* kernel_ms,
                         const adaptis_task* tasks = nullptr, const uint64_t* offsets = nullptr,
                         std::vector<TraceEntry>* trace_out = nullptr, int* trace_cap_out = nullptr,
                         MemTimelineReq* mt = nullptr) {
  std::vector<int64_t> rep_local;
  if ((trace_out || mt) && !report) report = &rep_local;  // the trace rides on the report launch
  for (uint64_t i = 0; i < n; ++i) {
    const adaptis_plan& pl = plans[i];
    if (pl.policy == ADAPTIS_LIST || pl.policy == ADAPTIS_LIST_FUSED) {
      if (!tasks || !offsets)
        return fail(ctx, ADAPTIS_EINVAL, "plans[%llu]: LIST policies need task lists (adaptis_eval_lists)",
                    (unsigned long long)i);
      const bool ok_pl = pl.v == 1 ? pl.placement == ADAPTIS_SEQ
                                   : (pl.placement == ADAPTIS_INTERLEAVED || pl.placement == ADAPTIS_WAVE);
      if (pl.v < 1 || pl.v > ADAPTIS_MAX_V || pl.S != P->p * pl.v || pl.S > ADAPTIS_MAX_S || pl.S > P->L ||
          (pl.v > 1 && P->m % P->p != 0) || !ok_pl)
        return fail(ctx, ADAPTIS_EINVAL, "plans[%llu]: v = %d, S = %d, placement %d not admitted (R10, R12)",
                    (unsigned long long)i, pl.v, pl.S, pl.placement);
      continue;
    }
    if (pl.v < 1 || pl.v > ADAPTIS_MAX_V)
      return fail(ctx, ADAPTIS_EINVAL, "plans[%llu].v = %d not in [1, 4]", (unsigned long long)i, pl.v);
    if (pl.S != P->p * pl.v || pl.S > ADAPTIS_MAX_S || pl.S > P->L)
      return fail(ctx, ADAPTIS_EINVAL, "plans[%llu].S = %d (need p*v = %d <= min(64, L = %d))",
                  (unsigned long long)i, pl.S, P->p * pl.v, P->L);
    if (pl.v > 1 && P->m % P->p != 0)
      return fail(ctx, ADAPTIS_EINVAL, "plans[%llu]: v > 1 requires m %% p == 0 (R10)", (unsigned long long)i);
    if (combo_bit(pl.v, pl.placement, pl.policy) < 0)
      return fail(ctx, ADAPTIS_EINVAL, "plans[%llu]: (placement %d, policy %d) is not a combo for v = %d (R12)",
                  (unsigned long long)i, pl.placement, pl.policy, pl.v);
  }
  mk->assign(n, INT64_MAX);
  if (peak) peak->assign(n, 0);
  if (bubble) bubble->assign(n, 0.0f);
  status->assign(n, 0);
  if (report) report->assign((size_t)n * 5 * P->p, 0);
  if (n == 0) return ADAPTIS_OK;
  constexpr int CS = ADAPTIS_MAX_S + 1;
  std::vector<int16_t> hcuts((size_t)n * CS, 0);
  std::vector<std::vector<uint64_t>> groups(128);  // key (v-1)*32 + placement*8 + policy
  for (uint64_t i = 0; i < n; ++i) {
    const adaptis_plan& pl = plans[i];
    int16_t* c = &hcuts[(size_t)i * CS];
    for (int k = 1; k < pl.S; ++k) c[k] = pl.cuts[k];
    c[0] = 0;
    c[pl.S] = (int16_t)P->L;
    groups[(pl.v - 1) * 32 + pl.placement * 8 + pl.policy].push_back(i);
  }
  std::vector<uint64_t> order;
  order.reserve(n);
  for (auto& g : groups) order.insert(order.end(), g.begin(), g.end());
  CU(ctx, cudaSetDevice(ctx->device));
  int16_t* d_cuts = nullptr; uint64_t* d_order = nullptr;
  int64_t *d_mk = nullptr, *d_pk = nullptr, *d_rep = nullptr; float* d_bub = nullptr; uint8_t* d_st = nullptr;
  TraceBuf tb;
  adaptis_task* d_tasks = nullptr; uint64_t* d_toff = nullptr;
  adaptis_status st = ADAPTIS_OK;
  auto cleanup = [&]() {
    cudaFree(d_cuts); cudaFree(d_order); cudaFree(d_mk); cudaFree(d_pk); cudaFree(d_rep);
    cudaFree(d_bub); cudaFree(d_st); cudaFree(tb.trace); cudaFree(tb.trace_n);
    cudaFree(d_tasks); cudaFree(d_toff);
  };
#define CUP(call) do { cudaError_t e_ = (call); if (e_ != cudaSuccess) { cleanup(); \
    return fail(ctx, ADAPTIS_ECUDA, "%s: %s", #call, cudaGetErrorString(e_)); } } while (0)
  CUP(cudaMalloc(&d_cuts, hcuts.size() * 2));
  CUP(cudaMalloc(&d_order, n * 8));
  CUP(cudaMalloc(&d_mk, n * 8));
  CUP(cudaMalloc(&d_pk, n * 8));
  CUP(cudaMalloc(&d_bub, n * 4));
  CUP(cudaMalloc(&d_st, n));
  const bool account = report && P->tick != kTickF32;
  if (report) {
    CUP(cudaMalloc(&d_rep, (size_t)n * 5 * P->p * 8));
    CUP(cudaMemsetAsync(d_rep, 0, (size_t)n * 5 * P->p * 8, ctx->stream));
  }
  if (account) {  // one trace per (plan, device): at most 3 m v tasks (R29)
    int vmax = 1;
    for (uint64_t i = 0; i < n; ++i) vmax = std::max(vmax, (int)plans[i].v);
    tb.cap = 3 * P->m * vmax;
    const size_t bytes = (size_t)n * P->p * tb.cap * sizeof(TraceEntry);
    if (bytes > ((size_t)1 << 31)) {
      cleanup();
      return fail(ctx, ADAPTIS_EINVAL, "report for %llu plans needs %zu B of trace scratch (> 2 GiB): split the list",
                  (unsigned long long)n, bytes);
    }
    CUP(cudaMalloc(&tb.trace, bytes));
    CUP(cudaMalloc(&tb.trace_n, (size_t)n * P->p * sizeof(int)));
    CUP(cudaMemsetAsync(tb.trace_n, 0, (size_t)n * P->p * sizeof(int), ctx->stream));
  }
  if (tasks) {
    // plans may share or reorder task ranges: the device copy covers the largest end
    uint64_t ntask = 0;
    for (uint64_t i = 0; i < n; ++i) ntask = std::max(ntask, offsets[i * (uint64_t)(P->p + 1) + P->p]);
    CUP(cudaMalloc(&d_tasks, std::max<uint64_t>(ntask, 1) * sizeof(adaptis_task)));
    CUP(cudaMalloc(&d_toff, n * (P->p + 1) * 8));
    CUP(cudaMemcpyAsync(d_tasks, tasks, ntask * sizeof(adaptis_task), cudaMemcpyHostToDevice, ctx->stream));
    CUP(cudaMemcpyAsync(d_toff, offsets, n * (P->p + 1) * 8, cudaMemcpyHostToDevice, ctx->stream));
  }
  CUP(cudaMemcpyAsync(d_cuts, hcuts.data(), hcuts.size() * 2, cudaMemcpyHostToDevice, ctx->stream));
  CUP(cudaMemcpyAsync(d_order, order.data(), n * 8, cudaMemcpyHostToDevice, ctx->stream));
  std::vector<Job> jobs;
  uint64_t off = 0;
  for (int key = 0; key < 128; ++key) {
    const auto& g = groups[key];
    if (g.empty()) continue;
    const adaptis_plan& pl = plans[g[0]];
    Seg sg{};
    sg.group = 0; sg.combo = combo_bit(pl.v, pl.placement, pl.policy); sg.v = pl.v; sg.S = pl.S;
    sg.placement = pl.placement; sg.policy = pl.policy; sg.part_mode = ADAPTIS_PART_FULL;
    sg.base = 0; sg.count = n;
    Job j{};
    j.s = make_launch(P, sg);
    j.s.lo = 0; j.s.hi = n; j.s.seg_base = 0;
    j.s.n_pos = g.size(); j.s.n0 = g.size(); j.s.world = 1;
    j.s.list_out = d_order + off;
    j.s.list_cuts = d_cuts;
    if (pl.policy == ADAPTIS_LIST || pl.policy == ADAPTIS_LIST_FUSED) {
      j.s.list_tasks = d_tasks;
      j.s.list_task_off = d_toff;
    }
    j.info.group = -1; j.info.combo = sg.combo; j.info.v = pl.v;
    j.info.placement = pl.placement; j.info.policy = pl.policy;
    jobs.push_back(j);
    off += g.size();
  }
  adaptis_results_soa dout{d_mk, d_pk, d_bub, d_st, nullptr};
  st = run_jobs(ctx, P, jobs, false, &dout, 0, d_rep, kernel_ms, false, account ? &tb : nullptr);
  if (st != ADAPTIS_OK) { cleanup(); return st; }
  if (account) {
    const int e = launch_comm_account(tb.trace, tb.trace_n, tb.cap, P->p, n, d_rep, ctx->stream);
    if (e) { cleanup(); return fail(ctx, ADAPTIS_ECUDA, "comm accounting: %s", cudaGetErrorString((cudaError_t)e)); }
  }
  if (mt && account) {  // R35: the memory timeline from the same traces
    mt->pcap = 1 + tb.cap;
    std::vector<int32_t> info(n);
    for (uint64_t i = 0; i < n; ++i) {
      const int pol = plans[i].policy;
      const bool fused = pol == ADAPTIS_GPIPE || pol == ADAPTIS_ONEF1B || pol == ADAPTIS_LIST_FUSED;
      info[i] = plans[i].v | (plans[i].placement << 4) | ((fused ? 1 : 0) << 8);
    }
    const size_t np = (size_t)n * P->p;
    int32_t* d_info = nullptr; adaptis_mem_point* d_pts = nullptr; int* d_npts = nullptr; int64_t* d_first = nullptr;
    auto free_mt = [&]() { cudaFree(d_info); cudaFree(d_pts); cudaFree(d_npts); cudaFree(d_first); };
    cudaError_t ce = cudaMalloc(&d_info, n * 4);
    if (ce == cudaSuccess) ce = cudaMalloc(&d_pts, np * mt->pcap * sizeof(adaptis_mem_point));
    if (ce == cudaSuccess) ce = cudaMalloc(&d_npts, np * sizeof(int));
    if (ce == cudaSuccess) ce = cudaMalloc(&d_first, np * 8);
    if (ce == cudaSuccess) ce = cudaMemcpyAsync(d_info, info.data(), n * 4, cudaMemcpyHostToDevice, ctx->stream);
    if (ce == cudaSuccess)
      ce = (cudaError_t)launch_mem_timeline(tb.trace, tb.trace_n, tb.cap, P->p, n, d_cuts, d_info, P->d_pre, P->L,
                                            P->cap, d_pts, mt->pcap, d_npts, d_first, ctx->stream);
    mt->points.resize(np * mt->pcap);
    mt->npts.resize(np);
    mt->first.resize(np);
    if (ce == cudaSuccess)
      ce = cudaMemcpyAsync(mt->points.data(), d_pts, np * mt->pcap * sizeof(adaptis_mem_point),
                           cudaMemcpyDeviceToHost, ctx->stream);
    if (ce == cudaSuccess) ce = cudaMemcpyAsync(mt->npts.data(), d_npts, np * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream);
    if (ce == cudaSuccess) ce = cudaMemcpyAsync(mt->first.data(), d_first, np * 8, cudaMemcpyDeviceToHost, ctx->stream);
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(ctx->stream);
    free_mt();
    if (ce != cudaSuccess) { cleanup(); return fail(ctx, ADAPTIS_ECUDA, "memory timeline: %s", cudaGetErrorString(ce)); }
  }
  CUP(cudaMemcpyAsync(mk->data(), d_mk, n * 8, cudaMemcpyDeviceToHost, ctx->stream));
  if (peak) CUP(cudaMemcpyAsync(peak->data(), d_pk, n * 8, cudaMemcpyDeviceToHost, ctx->stream));
  if (bubble) CUP(cudaMemcpyAsync(bubble->data(), d_bub, n * 4, cudaMemcpyDeviceToHost, ctx->stream));
  CUP(cudaMemcpyAsync(status->data(), d_st, n, cudaMemcpyDeviceToHost, ctx->stream));
  if (report) CUP(cudaMemcpyAsync(report->data(), d_rep, (size_t)n * 5 * P->p * 8, cudaMemcpyDeviceToHost, ctx->stream));
  if (trace_out && account) {
    trace_out->resize((size_t)n * P->p * tb.cap);
    CUP(cudaMemcpyAsync(trace_out->data(), tb.trace, trace_out->size() * sizeof(TraceEntry),
                        cudaMemcpyDeviceToHost, ctx->stream));
    if (trace_cap_out) *trace_cap_out = tb.cap;
  }
  CUP(cudaStreamSynchronize(ctx->stream));
#undef CUP
  cleanup();
  return ADAPTIS_OK;
}

// Best (makespan, lowest index) of a prepared space on this GPU alone (no
// sharding, no allreduce): the generator's partition phase. Returns
// EINFEASIBLE when nothing is feasible.
adaptis_status best_of_space(adaptis_ctx* ctx, adaptis_prepared* P, adaptis_plan* plan,
                             int64_t* makespan, float* kernel_ms) {
  float t = 0;
  adaptis_status st = run_range(ctx, P, 0, P->N, true, 0, 1, nullptr, 0, nullptr, &t);
  if (kernel_ms) *kernel_ms += t;
  if (st != ADAPTIS_OK) return st;
  unsigned long long key = 0;
  CU(ctx, cudaMemcpyAsync(&key, ctx->d_scratch, 8, cudaMemcpyDeviceToHost, ctx->stream));
  CU(ctx, cudaStreamSynchronize(ctx->stream));
  if (key == (~0ull >> 1)) return ADAPTIS_EINFEASIBLE;
  const uint64_t idx = key & ((1ull << P->key_bits) - 1);
  fill_plan(*P, idx, plan, nullptr);
  *makespan = (int64_t)(key >> P->key_bits);
  return ADAPTIS_OK;
}

}  // namespace

// ================================================================================
extern "C" {

const char* adaptis_status_str(adaptis_status s) {
  switch (s) {
    case ADAPTIS_OK: return "ok";
    case ADAPTIS_EINVAL: return "invalid argument";
    case ADAPTIS_EINFEASIBLE: return "no feasible candidate";
    case ADAPTIS_EOVERFLOW: return "key overflow";
    case ADAPTIS_ECUDA: return "cuda error";
    case ADAPTIS_ECOLL: return "collective error";
  }
  return "unknown";
}

const char* adaptis_last_error(const adaptis_ctx* ctx) {
  return ctx ? ctx->err.c_str() : g_tls_error.c_str();
}

adaptis_status adaptis_ctx_create(int cuda_device, int rank, int world, adaptis_ctx** out) {
  if (!out) return fail(nullptr, ADAPTIS_EINVAL, "out is NULL");
  *out = nullptr;
  if (world < 1 || rank < 0 || rank >= world)
    return fail(nullptr, ADAPTIS_EINVAL, "rank = %d, world = %d", rank, world);
  adaptis_ctx* c = new adaptis_ctx();
  c->device = cuda_device; c->rank = rank; c->world = world;
  cudaError_t e = cudaSetDevice(cuda_device);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, cuda_device);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&c->max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, cuda_device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreate(&c->ev0);
  if (e == cudaSuccess) e = cudaEventCreate(&c->ev1);
  if (e != cudaSuccess) {
    fail(nullptr, ADAPTIS_ECUDA, "device %d: %s", cuda_device, cudaGetErrorString(e));
    delete c;
    return ADAPTIS_ECUDA;
  }
  *out = c;
  return ADAPTIS_OK;
}

void adaptis_ctx_destroy(adaptis_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  cudaFree(c->d_scratch); cudaFree(c->d_overflow); cudaFree(c->d_gring); cudaFree(c->d_report);
  cudaFreeHost(c->h_report); cudaFree(c->d_wtrace); cudaFree(c->d_wtrace_n);
  for (cudaEvent_t e : c->seg_events) cudaEventDestroy(e);
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

adaptis_status adaptis_ctx_set_prune(adaptis_ctx* ctx, int enable) {
  if (!ctx) return fail(nullptr, ADAPTIS_EINVAL, "ctx is NULL");
  ctx->prune = enable ? 1 : 0;
  return ADAPTIS_OK;
}

adaptis_status adaptis_ctx_set_allreduce(adaptis_ctx* ctx, adaptis_allreduce_min_fn fn, void* user) {
  if (!ctx) return fail(nullptr, ADAPTIS_EINVAL, "ctx is NULL");
  ctx->allreduce = fn; ctx->allreduce_user = user;
  return ADAPTIS_OK;
}

void* adaptis_ctx_stream(adaptis_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }
uint64_t adaptis_ctx_launch_count(const adaptis_ctx* ctx) { return ctx ? ctx->launches : 0; }
uint64_t adaptis_ctx_fallback_count(const adaptis_ctx* ctx) { return ctx ? ctx->fallback_cands : 0; }
int adaptis_ctx_launch_info(const adaptis_ctx* ctx, adaptis_launch_info* out, int max) {
  if (!ctx) return 0;
  const int n = (int)ctx->last_info.size();
  for (int i = 0; i < n && i < max && out; ++i) out[i] = ctx->last_info[i];
  return n;
}
void adaptis_ctx_counters(const adaptis_ctx* ctx, uint64_t out[3]) {
  for (int i = 0; i < 3; ++i) out[i] = ctx ? ctx->counters[i] : 0;
}

adaptis_status adaptis_static_order(int32_t policy, int32_t placement, int32_t p, int32_t v, int32_t m,
                                    uint32_t* entries, uint64_t cap, uint64_t* n_entries, int32_t* n_slots) {
  if (!n_entries || !n_slots || (!entries && cap)) return fail(nullptr, ADAPTIS_EINVAL, "a pointer argument is NULL");
  if (policy != ADAPTIS_GPIPE && policy != ADAPTIS_ONEF1B && policy != ADAPTIS_ZB)
    return fail(nullptr, ADAPTIS_EINVAL, "policy = %d is not GPIPE, ONEF1B or ZB", policy);
  if (placement < ADAPTIS_SEQ || placement > ADAPTIS_WAVE || p < 1 || v < 1 || m < 1 ||
      (placement == ADAPTIS_SEQ) != (v == 1) || (v > 1 && m % p != 0))
    return fail(nullptr, ADAPTIS_EINVAL, "placement %d, p %d, v %d, m %d is not an R12 combination", placement, p, v, m);
  std::vector<uint32_t> ent;
  int slots = 0;
  if (!fx_build_order(policy, placement, p, v, m, ent, slots))
    return fail(nullptr, ADAPTIS_EINVAL, "no static order (p > 16, S > 64, deadlocking lists or > 254 slots)");
  *n_entries = ent.size();
  *n_slots = slots;
  if (cap < ent.size()) return fail(nullptr, ADAPTIS_EOVERFLOW, "cap %llu < %zu entries", (unsigned long long)cap, ent.size());
  std::copy(ent.begin(), ent.end(), entries);
  return ADAPTIS_OK;
}

adaptis_status adaptis_space_size(const adaptis_problem* problem, const adaptis_space* space,
                                  uint64_t* n_out) {
  if (!n_out) return fail(nullptr, ADAPTIS_EINVAL, "n_out is NULL");
  adaptis_prepared P;
  adaptis_status st = build_space(nullptr, problem, space, &P);
  if (st != ADAPTIS_OK) return st;
  *n_out = P.N;
  return ADAPTIS_OK;
}

adaptis_status adaptis_decode(const adaptis_problem* problem, const adaptis_space* space,
                              uint64_t index, adaptis_plan* out) {
  if (!out) return fail(nullptr, ADAPTIS_EINVAL, "out is NULL");
  adaptis_prepared P;
  adaptis_status st = build_space(nullptr, problem, space, &P);
  if (st != ADAPTIS_OK) return st;
  if (index >= P.N) return fail(nullptr, ADAPTIS_EINVAL, "index %llu >= |space| = %llu",
                                (unsigned long long)index, (unsigned long long)P.N);
  fill_plan(P, index, out, nullptr);
  return ADAPTIS_OK;
}

adaptis_status adaptis_prepare(adaptis_ctx* ctx, const adaptis_problem* problem,
                               const adaptis_space* space, adaptis_prepared** out) {
  if (!ctx) return fail(nullptr, ADAPTIS_EINVAL, "ctx is NULL");
  if (!out) return fail(ctx, ADAPTIS_EINVAL, "out is NULL");
  *out = nullptr;
  adaptis_prepared* P = new adaptis_prepared();
  adaptis_status st = build_space(ctx, problem, space, P);
  if (st == ADAPTIS_OK) st = upload(ctx, problem, P);
  if (st != ADAPTIS_OK) { adaptis_prepared_free(P); return st; }
  P->owner = ctx;
  *out = P;
  return ADAPTIS_OK;
}

void adaptis_prepared_free(adaptis_prepared* P) {
  if (!P) return;
  cudaFree(P->d_cols); cudaFree(P->d_pre); cudaFree(P->d_comm); cudaFree(P->d_colsf); cudaFree(P->d_commf); cudaFree(P->d_binom); cudaFree(P->d_ball);
  cudaFree(P->d_seeds);
  for (auto& o : P->fx_orders) cudaFree(o.d_ent);
  delete P;
}

adaptis_status adaptis_eval_prepared(adaptis_ctx* ctx, adaptis_prepared* P, uint64_t first,
                                     uint64_t count, const adaptis_results_soa* out,
                                     int out_on_device) {
  if (!ctx || !P) return fail(ctx, ADAPTIS_EINVAL, "ctx or prepared is NULL");
  if (!out) return fail(ctx, ADAPTIS_EINVAL, "out is NULL");
  if (first > P->N || count > P->N - first)
    return fail(ctx, ADAPTIS_EINVAL, "range [%llu, +%llu) exceeds |space| = %llu",
                (unsigned long long)first, (unsigned long long)count, (unsigned long long)P->N);
  if (count == 0) return ADAPTIS_OK;
  CU(ctx, cudaSetDevice(ctx->device));
  adaptis_results_soa dout = *out;
  void* tmp[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  if (!out_on_device) {
    if (out->makespan) { CU(ctx, cudaMalloc(&tmp[0], count * 8)); dout.makespan = (int64_t*)tmp[0]; }
    if (out->peak_mem_bytes) { CU(ctx, cudaMalloc(&tmp[1], count * 8)); dout.peak_mem_bytes = (int64_t*)tmp[1]; }
    if (out->bubble_ratio) { CU(ctx, cudaMalloc(&tmp[2], count * 4)); dout.bubble_ratio = (float*)tmp[2]; }
    if (out->status) { CU(ctx, cudaMalloc(&tmp[3], count)); dout.status = (uint8_t*)tmp[3]; }
    if (out->makespan_f32) { CU(ctx, cudaMalloc(&tmp[4], count * 4)); dout.makespan_f32 = (float*)tmp[4]; }
  }
  adaptis_status st = run_range(ctx, P, first, first + count, false, 0, 1, &dout, first, nullptr, nullptr);
  if (st == ADAPTIS_OK && !out_on_device) {
    if (out->makespan) CU(ctx, cudaMemcpyAsync(out->makespan, tmp[0], count * 8, cudaMemcpyDeviceToHost, ctx->stream));
    if (out->peak_mem_bytes) CU(ctx, cudaMemcpyAsync(out->peak_mem_bytes, tmp[1], count * 8, cudaMemcpyDeviceToHost, ctx->stream));
    if (out->bubble_ratio) CU(ctx, cudaMemcpyAsync(out->bubble_ratio, tmp[2], count * 4, cudaMemcpyDeviceToHost, ctx->stream));
    if (out->status) CU(ctx, cudaMemcpyAsync(out->status, tmp[3], count, cudaMemcpyDeviceToHost, ctx->stream));
    if (out->makespan_f32) CU(ctx, cudaMemcpyAsync(out->makespan_f32, tmp[4], count * 4, cudaMemcpyDeviceToHost, ctx->stream));
    CU(ctx, cudaStreamSynchronize(ctx->stream));
  }
  for (void* t : tmp) if (t) cudaFree(t);
  return st;
}

adaptis_status adaptis_eval_batch(adaptis_ctx* ctx, const adaptis_problem* problem,
                                  const adaptis_space* space, uint64_t first, uint64_t count,
                                  const adaptis_results_soa* out, int out_on_device) {
  adaptis_prepared* P = nullptr;
  adaptis_status st = adaptis_prepare(ctx, problem, space, &P);
  if (st != ADAPTIS_OK) return st;
  st = adaptis_eval_prepared(ctx, P, first, count, out, out_on_device);
  adaptis_prepared_free(P);
  return st;
}

// ---- contention on realised orders (reading R36): every candidate's policy
// order is realised by its policy kernel with pure-latency communication
// (R3-R6, a traced report launch) and then executed as an explicit schedule
// (R30) under send/receive-engine contention (R34), in batches per segment.
// search: the packed argmin key of the contended makespans lands in *d_key;
// eval: host results at [idx - lo] (status 1 / 3 from the policy run for
// candidates without a complete order).
static adaptis_status run_contended(adaptis_ctx* ctx, adaptis_prepared* P, uint64_t lo, uint64_t hi, bool search,
                                    const adaptis_results_soa* hout, unsigned long long* d_key, float* kernel_ms,
                                    uint64_t* n_tasks, int64_t* report_one) {
  if (P->tick == kTickF32) return fail(ctx, ADAPTIS_EINVAL, "FP32 cost mode is not supported under contention");
  const int p = P->p, m = P->m, L = P->L;
  {
    long double bound = 0;  // the contention kernel's transfer keys hold eligibility times < 2^40
    for (int l = 0; l < L; ++l)
      bound += (long double)m * (P->h_cols[(size_t)kColTF * L + l] + P->h_cols[(size_t)kColTB * L + l] +
                                 P->h_cols[(size_t)kColTW * L + l]) + 2.0L * m * P->h_comm[l];
    if (bound >= (long double)(1ull << 40))
      return fail(ctx, ADAPTIS_EOVERFLOW, "serial bound %.0Lf ticks >= 2^40 (contention keys)", bound);
  }
  CU(ctx, cudaSetDevice(ctx->device));
  float ms_total = 0;
  uint64_t tasks_total = 0;
  for (const Seg& sg : P->segs) {
    const uint64_t a0 = std::max(lo, sg.base), b0 = std::min(hi, sg.base + sg.count);
    if (a0 >= b0) continue;
    const bool fused = sg.policy == ADAPTIS_GPIPE || sg.policy == ADAPTIS_ONEF1B;
    const int cap_t = 3 * m * sg.v;
    const uint64_t stride = (uint64_t)5 * sg.S * m;
    const uint64_t per = (uint64_t)p * cap_t * (sizeof(TraceEntry) + sizeof(adaptis_task)) + stride * 8 +
                         (uint64_t)p * 48 + 64;
    const uint64_t B = std::max<uint64_t>(256, std::min<uint64_t>(65536, ((uint64_t)1 << 32) / per));
    RealisedSeg rs{P->d_binom, P->d_ball, P->d_seeds, sg.group, sg.part_mode, sg.radius, sg.S, L,
                   sg.v, sg.placement, fused ? 1 : 0, sg.base};
    const uint64_t n = std::min(B, b0 - a0);  // buffers for the segment's largest batch, reused
    TraceEntry* d_tr = nullptr; int* d_trn = nullptr; uint8_t* d_pst = nullptr; int64_t* d_rep = nullptr;
    adaptis_plan* d_plans = nullptr; adaptis_task* d_tasks = nullptr; uint64_t *d_off = nullptr, *d_slot = nullptr;
    unsigned int* d_nk = nullptr; int64_t *d_scr = nullptr, *d_mk = nullptr, *d_pk = nullptr, *d_crep = nullptr;
    float* d_bub = nullptr; uint8_t* d_st = nullptr; unsigned long long* d_nt = nullptr;
    auto cleanup = [&]() {
      cudaFree(d_tr); cudaFree(d_trn); cudaFree(d_pst); cudaFree(d_rep); cudaFree(d_plans); cudaFree(d_tasks);
      cudaFree(d_off); cudaFree(d_slot); cudaFree(d_nk); cudaFree(d_scr); cudaFree(d_mk); cudaFree(d_pk);
      cudaFree(d_crep); cudaFree(d_bub); cudaFree(d_st); cudaFree(d_nt);
    };
#define CUR(call) do { cudaError_t e_ = (call); if (e_ != cudaSuccess) { cleanup(); \
    return fail(ctx, ADAPTIS_ECUDA, "%s: %s", #call, cudaGetErrorString(e_)); } } while (0)
    {
      CUR(cudaMalloc(&d_tr, n * p * cap_t * sizeof(TraceEntry)));
      CUR(cudaMalloc(&d_trn, n * p * sizeof(int)));
      CUR(cudaMalloc(&d_pst, n));
      CUR(cudaMalloc(&d_rep, n * 5 * p * 8));
      CUR(cudaMalloc(&d_plans, n * sizeof(adaptis_plan)));
      CUR(cudaMalloc(&d_tasks, n * p * cap_t * sizeof(adaptis_task)));
      CUR(cudaMalloc(&d_off, n * (p + 1) * 8));
      CUR(cudaMalloc(&d_slot, n * 8));
      CUR(cudaMalloc(&d_nk, 4));
      CUR(cudaMalloc(&d_scr, n * stride * 8));
      CUR(cudaMalloc(&d_mk, n * 8));
      CUR(cudaMalloc(&d_pk, n * 8));
      CUR(cudaMalloc(&d_bub, n * 4));
      CUR(cudaMalloc(&d_st, n));
      CUR(cudaMalloc(&d_nt, 8));
      if (report_one) CUR(cudaMalloc(&d_crep, n * 5 * p * 8));
    }
    for (uint64_t a = a0; a < b0; a += B) {
      const uint64_t n = std::min(B, b0 - a);
      CUR(cudaMemsetAsync(d_trn, 0, n * p * sizeof(int), ctx->stream));
      CUR(cudaMemsetAsync(d_rep, 0, n * 5 * p * 8, ctx->stream));
      CUR(cudaMemsetAsync(d_nk, 0, 4, ctx->stream));
      CUR(cudaMemsetAsync(d_nt, 0, 8, ctx->stream));
      // (1) the policy run with traces (pure latency): the realised orders
      TraceBuf tb;
      tb.trace = d_tr; tb.trace_n = d_trn; tb.cap = cap_t;
      adaptis_results_soa pso{nullptr, nullptr, nullptr, d_pst, nullptr};
      float t1 = 0;
      adaptis_status st = run_range(ctx, P, a, a + n, false, 0, 1, &pso, a, d_rep, &t1, false, &tb);
      if (st != ADAPTIS_OK) { cleanup(); return st; }
      tasks_total += ctx->last_tasks;
      CUR(cudaEventRecord(ctx->ev0, ctx->stream));
      // (2) the orders as explicit schedules, compacted
      int e = launch_realised_lists(d_tr, d_trn, cap_t, p, n, a, d_pst, rs, d_plans, d_tasks, d_off, d_slot,
                                    d_nk, ctx->stream);
      if (e) { cleanup(); return fail(ctx, ADAPTIS_ECUDA, "realised lists: %s", cudaGetErrorString((cudaError_t)e)); }
      unsigned int nk = 0;
      CUR(cudaMemcpyAsync(&nk, d_nk, 4, cudaMemcpyDeviceToHost, ctx->stream));
      CUR(cudaStreamSynchronize(ctx->stream));
      // (3) contention (R34) on them, (4) the argmin key or the results
      e = launch_contend(P->d_cols, P->d_comm, L, p, m, P->cap, nk, d_plans, d_tasks, d_off, d_scr, stride, d_mk,
                         d_pk, d_bub, d_st, d_crep, d_nt, sg.S, ctx->stream);
      if (e) { cleanup(); return fail(ctx, ADAPTIS_ECUDA, "contention kernel: %s", cudaGetErrorString((cudaError_t)e)); }
      if (search) {
        e = launch_contended_key(d_mk, d_st, d_slot, nk, a, P->key_bits, d_key, ctx->stream);
        if (e) { cleanup(); return fail(ctx, ADAPTIS_ECUDA, "contended key: %s", cudaGetErrorString((cudaError_t)e)); }
      }
      CUR(cudaEventRecord(ctx->ev1, ctx->stream));
      ctx->launches += 3;
      unsigned long long nt = 0;
      CUR(cudaMemcpyAsync(&nt, d_nt, 8, cudaMemcpyDeviceToHost, ctx->stream));
      if (!search && hout) {
        std::vector<uint8_t> pst(n), cst(nk);
        std::vector<int64_t> mk(nk), pk(nk);
        std::vector<float> bub(nk);
        std::vector<uint64_t> slot(nk);
        CUR(cudaMemcpyAsync(pst.data(), d_pst, n, cudaMemcpyDeviceToHost, ctx->stream));
        if (nk) {
          CUR(cudaMemcpyAsync(cst.data(), d_st, nk, cudaMemcpyDeviceToHost, ctx->stream));
          CUR(cudaMemcpyAsync(mk.data(), d_mk, nk * 8, cudaMemcpyDeviceToHost, ctx->stream));
          CUR(cudaMemcpyAsync(pk.data(), d_pk, nk * 8, cudaMemcpyDeviceToHost, ctx->stream));
          CUR(cudaMemcpyAsync(bub.data(), d_bub, nk * 4, cudaMemcpyDeviceToHost, ctx->stream));
          CUR(cudaMemcpyAsync(slot.data(), d_slot, nk * 8, cudaMemcpyDeviceToHost, ctx->stream));
        }
        if (report_one && nk) CUR(cudaMemcpyAsync(report_one, d_crep, 5 * p * 8, cudaMemcpyDeviceToHost, ctx->stream));
        CUR(cudaStreamSynchronize(ctx->stream));
        for (uint64_t i = 0; i < n; ++i) {  // no complete order: the policy run's status
          const uint64_t o = a + i - lo;
          if (hout->status) hout->status[o] = pst[i];
          if (hout->makespan) hout->makespan[o] = INT64_MAX;
          if (hout->peak_mem_bytes) hout->peak_mem_bytes[o] = 0;
          if (hout->bubble_ratio) hout->bubble_ratio[o] = 0.0f;
          if (hout->makespan_f32) hout->makespan_f32[o] = INFINITY;
        }
        for (unsigned int k = 0; k < nk; ++k) {
          const uint64_t o = a + slot[k] - lo;
          if (hout->status) hout->status[o] = cst[k];
          if (hout->makespan) hout->makespan[o] = mk[k];
          if (hout->peak_mem_bytes) hout->peak_mem_bytes[o] = pk[k];
          if (hout->bubble_ratio) hout->bubble_ratio[o] = bub[k];
          if (hout->makespan_f32) hout->makespan_f32[o] = cst[k] == 0 ? (float)mk[k] : INFINITY;
        }
      } else {
        CUR(cudaStreamSynchronize(ctx->stream));
      }
      float t2 = 0;
      cudaEventElapsedTime(&t2, ctx->ev0, ctx->ev1);
      ms_total += t1 + t2;
      tasks_total += nt;
    }
#undef CUR
    cleanup();
  }
  if (kernel_ms) *kernel_ms = ms_total;
  if (n_tasks) *n_tasks = tasks_total;
  return ADAPTIS_OK;
}

adaptis_status adaptis_eval_contended(adaptis_ctx* ctx, adaptis_prepared* P, uint64_t first, uint64_t count,
                                      const adaptis_results_soa* out) {
  if (!ctx || !P) return fail(ctx, ADAPTIS_EINVAL, "ctx or prepared is NULL");
  if (!out) return fail(ctx, ADAPTIS_EINVAL, "out is NULL");
  if (first > P->N || count > P->N - first)
    return fail(ctx, ADAPTIS_EINVAL, "range [%llu, +%llu) exceeds |space| = %llu", (unsigned long long)first,
                (unsigned long long)count, (unsigned long long)P->N);
  if (count == 0) return ADAPTIS_OK;
  float ms = 0; uint64_t nt = 0;
  adaptis_status st = run_contended(ctx, P, first, first + count, false, out, nullptr, &ms, &nt, nullptr);
  ctx->last_tasks = nt;
  return st;
}

adaptis_status adaptis_search_contended(adaptis_ctx* ctx, adaptis_prepared* P, adaptis_best* out) {
  if (!ctx || !P) return fail(ctx, ADAPTIS_EINVAL, "ctx or prepared is NULL");
  if (!out) return fail(ctx, ADAPTIS_EINVAL, "out is NULL");
  CU(ctx, cudaSetDevice(ctx->device));
  memset(out, 0, sizeof(*out));
  adaptis_status st = ensure_scratch(ctx, kHdr + kSegWords, kOverflowPerSeg);
  if (st != ADAPTIS_OK) return st;
  // the key lives apart from the scratch words, which every policy run resets
  unsigned long long* d_key = reinterpret_cast<unsigned long long*>(
      reinterpret_cast<unsigned char*>(ctx->d_report) + kReportBytes + 32);
  const unsigned long long inf = ~0ull >> 1;
  CU(ctx, cudaMemcpyAsync(d_key, &inf, 8, cudaMemcpyHostToDevice, ctx->stream));
  float ms = 0; uint64_t nt = 0;
  st = run_contended(ctx, P, 0, P->N, true, nullptr, d_key, &ms, &nt, nullptr);
  if (st != ADAPTIS_OK) return st;
  unsigned long long key = 0;
  CU(ctx, cudaMemcpyAsync(&key, d_key, 8, cudaMemcpyDeviceToHost, ctx->stream));
  CU(ctx, cudaStreamSynchronize(ctx->stream));
  out->kernel_ms = ms;
  out->n_tasks = nt;
  out->n_candidates = P->N;
  out->p = P->p;
  if (key == inf) {
    out->index = UINT64_MAX;
    out->result.makespan = INT64_MAX;
    return fail(ctx, ADAPTIS_EINFEASIBLE, "no candidate satisfies the memory constraint (Eq. 2)");
  }
  const uint64_t idx = key & ((1ull << P->key_bits) - 1);
  out->index = idx;
  fill_plan(*P, idx, &out->plan, nullptr);
  // the winner's contended result and per-device report
  int64_t mk = 0, pk = 0; float bub = 0, mkf = 0; uint8_t stt = 0;
  std::vector<int64_t> rep(5 * P->p, 0);
  adaptis_results_soa ho{&mk, &pk, &bub, &stt, &mkf};
  st = run_contended(ctx, P, idx, idx + 1, false, &ho, nullptr, nullptr, nullptr, rep.data());
  if (st != ADAPTIS_OK) return st;
  out->result.makespan = mk;
  out->result.peak_mem_bytes = pk;
  out->result.bubble_ratio = bub;
  out->result.status = stt;
  out->result.makespan_f32 = (float)mk;
  out->result.throughput = (mk > 0 && P->tick_seconds > 0)
      ? (double)P->m * (double)P->tokens_per_mb / ((double)mk * P->tick_seconds) : 0.0;
  for (int d = 0; d < P->p; ++d) {
    out->T_d[d] = rep[d]; out->busy_d[d] = rep[P->p + d]; out->M_d[d] = rep[2 * P->p + d];
  }
  if (stt != ADAPTIS_CAND_OK || mk != (int64_t)(key >> P->key_bits))
    return fail(ctx, ADAPTIS_ECUDA, "contended winner re-evaluation disagrees (index %llu: %llu vs %lld)",
                (unsigned long long)idx, (unsigned long long)(key >> P->key_bits), (long long)mk);
  return ADAPTIS_OK;
}

adaptis_status adaptis_search_prepared(adaptis_ctx* ctx, adaptis_prepared* P, adaptis_best* out) {
  if (!ctx || !P) return fail(ctx, ADAPTIS_EINVAL, "ctx or prepared is NULL");
  if (!out) return fail(ctx, ADAPTIS_EINVAL, "out is NULL");
  if (ctx->world > 1 && !ctx->allreduce)
    return fail(ctx, ADAPTIS_EINVAL, "world = %d needs adaptis_ctx_set_allreduce", ctx->world);
  CU(ctx, cudaSetDevice(ctx->device));
  memset(out, 0, sizeof(*out));
  float ms = 0;
  adaptis_status st;
  bool seeded = false;
  // scratch for every segment before the first pass, so the passes share one buffer
  st = ensure_scratch(ctx, kHdr + kSegWords * std::max<size_t>(P->segs.size(), 1),
                      kOverflowPerSeg * std::max<size_t>(P->segs.size(), 1));
  if (st != ADAPTIS_OK) return st;
  if (ctx->prune && P->tick != kTickF32) {
    // seed pass: the first indices of every segment (the seed neighbourhood of
    // BALL spaces) give the lower-bound prune a good incumbent early; every rank
    // runs it, duplicates do not change the minimum
    for (const Seg& sg : P->segs) {
      const uint64_t n = std::min<uint64_t>(sg.count, kSeedPass);
      float t = 0;
      st = run_range(ctx, P, sg.base, sg.base + n, true, 0, 1, nullptr, 0, nullptr, &t, seeded);
      if (st != ADAPTIS_OK) return st;
      ms += t;
      seeded = true;
    }
  }
  {
    float t = 0;
    st = run_range(ctx, P, 0, P->N, true, ctx->rank, ctx->world, nullptr, 0, nullptr, &t, seeded);
    ms += t;
  }
  if (st != ADAPTIS_OK) return st;
  unsigned long long words[6] = {0, 0, 0, 0, 0, 0};
  CU(ctx, cudaMemcpyAsync(words, ctx->d_scratch, 48, cudaMemcpyDeviceToHost, ctx->stream));
  CU(ctx, cudaStreamSynchronize(ctx->stream));
  out->n_invalid = ctx->last_invalid;
  out->n_tasks = ctx->last_tasks;
  out->n_pruned = ctx->last_pruned;
  const std::vector<adaptis_launch_info> search_info = ctx->last_info;
  out->kernel_ms = ms;
  out->n_candidates = P->N;
  {
    SegLaunch tmp{};
    uint64_t n = 0;
    for (const Seg& sg : P->segs) { shard(sg.base, sg.base + sg.count, ctx->rank, ctx->world, &tmp); n += tmp.n_pos; }
    out->n_evaluated = n;
  }
  if (ctx->world > 1) {  // one 8-byte allreduce(MIN) over the ranks
    if (ctx->allreduce(reinterpret_cast<int64_t*>(ctx->d_scratch), (void*)ctx->stream, ctx->allreduce_user) != 0)
      return fail(ctx, ADAPTIS_ECOLL, "allreduce callback failed");
    CU(ctx, cudaMemcpyAsync(words, ctx->d_scratch, 8, cudaMemcpyDeviceToHost, ctx->stream));
    CU(ctx, cudaStreamSynchronize(ctx->stream));
  }
  const unsigned long long key = words[0];
  out->p = P->p;
  if (key == (~0ull >> 1)) {
    out->index = UINT64_MAX;
    out->result.makespan = INT64_MAX;
    return fail(ctx, ADAPTIS_EINFEASIBLE, "no candidate satisfies the memory constraint (Eq. 2)");
  }
  const uint64_t idx = key & ((1ull << P->key_bits) - 1);
  out->index = idx;
  fill_plan(*P, idx, &out->plan, nullptr);
  // winner report: the same kernel on the single winning index; its buffers
  // are the context's (no allocation per search), read back with one D2H
  unsigned char* wb = reinterpret_cast<unsigned char*>(ctx->d_report) + kReportBytes;
  CU(ctx, cudaMemsetAsync(ctx->d_report, 0, kReportBytes + kWinBytes, ctx->stream));
  adaptis_results_soa so{reinterpret_cast<int64_t*>(wb), reinterpret_cast<int64_t*>(wb + 8),
                         reinterpret_cast<float*>(wb + 20), wb + 24, reinterpret_cast<float*>(wb + 16)};
  // with integer ticks the winner is re-run with its device traces for the
  // communication accounting of R29 (comm, exposed, overlap, bubble per device)
  TraceBuf tb;
  const bool account = P->tick != kTickF32;
  if (account) {
    tb.cap = 3 * P->m * out->plan.v;
    const size_t need = (size_t)P->p * tb.cap;
    if (need > ctx->wtrace_entries) {
      cudaFree(ctx->d_wtrace);
      ctx->d_wtrace = nullptr;
      CU(ctx, cudaMalloc(&ctx->d_wtrace, need * sizeof(TraceEntry)));
      ctx->wtrace_entries = need;
    }
    tb.trace = ctx->d_wtrace;
    tb.trace_n = ctx->d_wtrace_n;
    CU(ctx, cudaMemsetAsync(tb.trace_n, 0, (size_t)P->p * sizeof(int), ctx->stream));
  }
  st = run_range(ctx, P, idx, idx + 1, false, 0, 1, &so, idx, ctx->d_report, nullptr, false,
                 account ? &tb : nullptr);
  if (st == ADAPTIS_OK && account) {
    const int e = launch_comm_account(tb.trace, tb.trace_n, tb.cap, P->p, 1, ctx->d_report, ctx->stream);
    if (e) st = fail(ctx, ADAPTIS_ECUDA, "comm accounting: %s", cudaGetErrorString((cudaError_t)e));
  }
  if (st == ADAPTIS_OK) {
    CU(ctx, cudaMemcpyAsync(ctx->h_report, ctx->d_report, kReportBytes + kWinBytes, cudaMemcpyDeviceToHost,
                            ctx->stream));
    CU(ctx, cudaStreamSynchronize(ctx->stream));
  }
  ctx->last_info = search_info;  // report the search's launches, not the re-evaluation
  if (st != ADAPTIS_OK) return st;
  std::vector<int64_t> rep(5 * P->p, 0);
  for (int r = 0; r < 5; ++r)
    memcpy(rep.data() + (size_t)r * P->p, ctx->h_report + (size_t)r * P->p * 8, (size_t)P->p * 8);
  int64_t mk, pk; float bub, mkf; uint8_t stt;
  const unsigned char* hw = ctx->h_report + kReportBytes;
  memcpy(&mk, hw, 8); memcpy(&pk, hw + 8, 8); memcpy(&mkf, hw + 16, 4); memcpy(&bub, hw + 20, 4);
  stt = hw[24];
  out->result.makespan = mk;
  out->result.peak_mem_bytes = pk;
  out->result.bubble_ratio = bub;
  out->result.status = stt;
  out->result.makespan_f32 = P->tick == kTickF32 ? mkf : (float)mk;
  const double mkd = P->tick == kTickF32 ? (double)mkf : (double)mk;
  out->result.throughput = (mkd > 0 && P->tick_seconds > 0)
      ? (double)P->m * (double)P->tokens_per_mb / (mkd * P->tick_seconds) : 0.0;
  for (int d = 0; d < P->p; ++d) {
    out->T_d[d] = rep[d];
    out->busy_d[d] = rep[P->p + d];
    out->M_d[d] = rep[2 * P->p + d];
    out->comm_d[d] = rep[3 * P->p + d];
    out->exposed_d[d] = rep[4 * P->p + d];
    out->overlap_d[d] = out->comm_d[d] - out->exposed_d[d];
    out->bubble_d[d] = out->T_d[d] - out->busy_d[d] - out->exposed_d[d];
  }
  const unsigned long long kv = key >> P->key_bits;
  bool agree;
  if (P->tick == kTickF32) { float f; uint32_t u = (uint32_t)kv; memcpy(&f, &u, 4); agree = f == mkf; }
  else agree = mk == (int64_t)kv;
  if (!agree)
    return fail(ctx, ADAPTIS_ECUDA, "winner re-evaluation disagrees with its search key (index %llu: key makespan %llu, re-evaluated %lld, status %d)",
                (unsigned long long)idx, (unsigned long long)kv, (long long)mk, (int)stt);
  return ADAPTIS_OK;
}

// OOM repair (reading R31) on an explicit schedule: evaluate on the GPU
// (with per-task start times from the trace), find the earliest Eq. 2
// violation (the first F of a device whose allocation exceeds the cap, earliest
// start over devices, ties to the lower device), advance the latest-listed B
// of that device whose F is listed earlier and whose cross-device input has
// arrived by then (its W follows it when split) to just before that F, repeat.
adaptis_status adaptis_repair_oom(adaptis_ctx* ctx, adaptis_prepared* P, const adaptis_plan* plan,
                                  const adaptis_task* tasks, const uint64_t* offsets, int32_t max_moves,
                                  adaptis_task* tasks_out, adaptis_result* result, int32_t* n_moves) {
  if (!ctx || !P) return fail(ctx, ADAPTIS_EINVAL, "ctx or prepared is NULL");
  if (!plan || !tasks || !offsets || !tasks_out || !result || !n_moves)
    return fail(ctx, ADAPTIS_EINVAL, "a pointer argument is NULL");
  if (P->tick == kTickF32) return fail(ctx, ADAPTIS_EINVAL, "FP32 cost mode is not supported for explicit plans");
  if (plan->policy != ADAPTIS_LIST && plan->policy != ADAPTIS_LIST_FUSED)
    return fail(ctx, ADAPTIS_EINVAL, "plan.policy = %d is not ADAPTIS_LIST or ADAPTIS_LIST_FUSED", plan->policy);
  if (plan->S != P->p * plan->v || plan->S < 1 || plan->S > ADAPTIS_MAX_S)
    return fail(ctx, ADAPTIS_EINVAL, "plan.S = %d != p * v", plan->S);
  adaptis_status st = validate_lists(ctx, P, plan, tasks, offsets, 1);
  if (st != ADAPTIS_OK) return st;
  const int p = P->p, m = P->m, S = plan->S, L = P->L;
  const bool fused = plan->policy == ADAPTIS_LIST_FUSED;
  const uint64_t total = offsets[p];
  if (max_moves <= 0) max_moves = (int32_t)std::min<uint64_t>(total, INT32_MAX);
  std::vector<int> cuts(S + 1);
  for (int i = 1; i < S; ++i) cuts[i] = plan->cuts[i];
  cuts[0] = 0; cuts[S] = L;
  for (int i = 0; i < S; ++i)
    if (cuts[i] >= cuts[i + 1]) return fail(ctx, ADAPTIS_EINVAL, "plan.cuts not strictly increasing");
  auto csum = [&](int col, int s2) {
    int64_t x = 0;
    for (int l = cuts[s2]; l < cuts[s2 + 1]; ++l) x += P->h_cols[(size_t)col * L + l];
    return x;
  };
  std::vector<int64_t> act(S), sta(S), wg(S), xB(S, 0);
  std::vector<int> dev(S);
  for (int s2 = 0; s2 < S; ++s2) {
    act[s2] = csum(kColAct, s2); sta[s2] = csum(kColStash, s2); wg[s2] = csum(kColWG, s2);
    dev[s2] = host_dev_of(plan->placement, p, s2);
  }
  for (int s2 = 0; s2 + 1 < S; ++s2)  // latency of the B input of stage s2 (from stage s2 + 1)
    xB[s2] = dev[s2 + 1] != dev[s2] ? P->h_comm[cuts[s2 + 1] - 1] : 0;
  std::vector<adaptis_task> cur(tasks, tasks + total);
  int32_t moves = 0;
  std::vector<int64_t> mk, pk; std::vector<float> bub; std::vector<uint8_t> stt;
  std::vector<TraceEntry> trace;
  int cap = 0;
  const int nk = fused ? 2 : 3;
  std::vector<int> pos((size_t)nk * S * m);
  for (;;) {
    st = run_plans(ctx, P, plan, 1, &mk, &pk, &bub, &stt, nullptr, nullptr, cur.data(), offsets, &trace, &cap);
    if (st != ADAPTIS_OK) return st;
    if (stt[0] != ADAPTIS_CAND_OVER_CAP || moves >= max_moves) break;
    for (int d = 0; d < p; ++d)
      for (uint64_t q = offsets[d]; q < offsets[d + 1]; ++q) {
        const adaptis_task& t = cur[q];
        pos[((size_t)t.kind * S + t.stage) * m + t.mb] = (int)(q - offsets[d]);
      }
    // violations: the first F of each device over the cap; visited by start time
    // (ties: lower device), the first with a movable B is repaired
    std::vector<std::tuple<int64_t, int, int>> viols;
    for (int d = 0; d < p; ++d) {
      int64_t stat = 0, dyn = 0;
      for (int s2 = 0; s2 < S; ++s2) if (dev[s2] == d) stat += wg[s2];
      for (uint64_t q = offsets[d]; q < offsets[d + 1]; ++q) {
        const adaptis_task& t = cur[q];
        if (t.kind == 0) {
          dyn += act[t.stage] + sta[t.stage];
          if (stat + dyn > P->cap) {
            const int k = (int)(q - offsets[d]);
            viols.emplace_back(trace[(size_t)d * cap + k].start, d, k);
            break;
          }
        } else if (t.kind == 1) {
          dyn -= act[t.stage] + (fused ? sta[t.stage] : 0);
        } else {
          dyn -= sta[t.stage];
        }
      }
    }
    std::sort(viols.begin(), viols.end());
    int bd = -1, bq = 0, chosen = -1;
    uint64_t o = 0;
    int len = 0;
    for (const auto& vi : viols) {
      // the latest-listed B of that device that is DAG-feasible before the violation
      const int64_t bt = std::get<0>(vi);
      bd = std::get<1>(vi); bq = std::get<2>(vi);
      o = offsets[bd];
      len = (int)(offsets[bd + 1] - o);
      for (int r = len - 1; r > bq && chosen < 0; --r) {
        const adaptis_task& t = cur[o + r];
        if (t.kind != 1) continue;
        const int s2 = t.stage, j = t.mb;
        if (pos[((size_t)0 * S + s2) * m + j] >= bq) continue;  // its F is not yet listed
        if (s2 + 1 < S) {
          const int d2 = dev[s2 + 1];
          const int pb = pos[((size_t)1 * S + s2 + 1) * m + j];
          if (d2 == bd) {
            if (pb >= bq) continue;  // same-device input listed after the violation
          } else if (trace[(size_t)d2 * cap + pb].fin + xB[s2] > bt) {
            continue;  // the input has not arrived by the violation time
          }
        }
        chosen = r;
      }
      if (chosen >= 0) break;
    }
    if (chosen < 0) break;  // no violation can be repaired by advancing a B
    const adaptis_task b = cur[o + chosen];
    cur.erase(cur.begin() + o + chosen);
    cur.insert(cur.begin() + o + bq, b);
    if (!fused) {  // its W follows it
      for (int r = bq + 1; r < len; ++r) {
        const adaptis_task& w = cur[o + r];
        if (w.kind == 2 && w.stage == b.stage && w.mb == b.mb) {
          const adaptis_task wt = w;
          cur.erase(cur.begin() + o + r);
          cur.insert(cur.begin() + o + bq + 1, wt);
          break;
        }
      }
    }
    ++moves;
  }
  std::copy(cur.begin(), cur.end(), tasks_out);
  *n_moves = moves;
  memset(result, 0, sizeof(*result));
  result->makespan = mk[0];
  result->peak_mem_bytes = pk[0];
  result->bubble_ratio = bub[0];
  result->status = stt[0];
  result->makespan_f32 = stt[0] == 0 ? (float)mk[0] : INFINITY;
  result->throughput = (stt[0] == 0 && mk[0] > 0 && P->tick_seconds > 0)
      ? (double)m * (double)P->tokens_per_mb / ((double)mk[0] * P->tick_seconds) : 0.0;
  return ADAPTIS_OK;
}

// Overlap-aware reordering (reading R32) of an explicit schedule:
// every round evaluates, in one GPU batch, all schedules that move the nearest
// later independent task in front of a task whose device idled waiting for its
// cross-device input, and accepts the one with the largest total OverlapTime
// among those that keep the makespan and raise the overlap.
adaptis_status adaptis_tune_overlap(adaptis_ctx* ctx, adaptis_prepared* P, const adaptis_plan* plan,
                                    const adaptis_task* tasks, const uint64_t* offsets, int32_t max_swaps,
                                    adaptis_task* tasks_out, adaptis_result* result, int32_t* n_swaps,
                                    int64_t* overlap_before, int64_t* overlap_after) {
  if (!ctx || !P) return fail(ctx, ADAPTIS_EINVAL, "ctx or prepared is NULL");
  if (!plan || !tasks || !offsets || !tasks_out || !result || !n_swaps)
    return fail(ctx, ADAPTIS_EINVAL, "a pointer argument is NULL");
  if (P->tick == kTickF32) return fail(ctx, ADAPTIS_EINVAL, "FP32 cost mode is not supported for explicit plans");
  if (plan->policy != ADAPTIS_LIST && plan->policy != ADAPTIS_LIST_FUSED)
    return fail(ctx, ADAPTIS_EINVAL, "plan.policy = %d is not ADAPTIS_LIST or ADAPTIS_LIST_FUSED", plan->policy);
  if (plan->S != P->p * plan->v || plan->S < 1 || plan->S > ADAPTIS_MAX_S)
    return fail(ctx, ADAPTIS_EINVAL, "plan.S = %d != p * v", plan->S);
  adaptis_status st = validate_lists(ctx, P, plan, tasks, offsets, 1);
  if (st != ADAPTIS_OK) return st;
  const int p = P->p, m = P->m, S = plan->S;
  const bool fused = plan->policy == ADAPTIS_LIST_FUSED;
  const uint64_t total = offsets[p];
  if (max_swaps <= 0) max_swaps = (int32_t)std::min<uint64_t>(total, INT32_MAX);
  std::vector<int> dev(S);
  for (int s2 = 0; s2 < S; ++s2) dev[s2] = host_dev_of(plan->placement, p, s2);
  std::vector<adaptis_task> cur(tasks, tasks + total);
  std::vector<int64_t> mk, rep; std::vector<uint8_t> stt;
  std::vector<TraceEntry> trace;
  int cap = 0;
  auto overlap_of = [&](const std::vector<int64_t>& r, size_t i) {
    int64_t ov = 0;
    for (int d = 0; d < p; ++d) ov += r[(i * 5 + 3) * p + d] - r[(i * 5 + 4) * p + d];
    return ov;
  };
  st = run_plans(ctx, P, plan, 1, &mk, nullptr, nullptr, &stt, &rep, nullptr, cur.data(), offsets, &trace, &cap);
  if (st != ADAPTIS_OK) return st;
  int64_t cur_mk = mk[0], cur_ov = overlap_of(rep, 0);
  uint8_t cur_st = stt[0];
  if (overlap_before) *overlap_before = cur_st == 0 ? cur_ov : 0;
  const int nk = fused ? 2 : 3;
  std::vector<int> pos((size_t)nk * S * m);
  int32_t swaps = 0;
  while (cur_st == ADAPTIS_CAND_OK && swaps < max_swaps) {
    for (int d = 0; d < p; ++d)
      for (uint64_t q = offsets[d]; q < offsets[d + 1]; ++q) {
        const adaptis_task& t = cur[q];
        pos[((size_t)t.kind * S + t.stage) * m + t.mb] = (int)(q - offsets[d]);
      }
    // the R32 neighbourhood, all candidates concatenated
    std::vector<adaptis_task> cand;
    uint64_t nc = 0;
    for (int d = 0; d < p; ++d) {
      const uint64_t o = offsets[d];
      const int len = (int)(offsets[d + 1] - o);
      for (int i = 0; i < len; ++i) {
        const adaptis_task& x = cur[o + i];
        const bool cross = (x.kind == 0 && x.stage > 0 && dev[x.stage - 1] != d) ||
                           (x.kind == 1 && x.stage + 1 < S && dev[x.stage + 1] != d);
        if (!cross) continue;
        const int64_t prev_fin = i == 0 ? 0 : trace[(size_t)d * cap + i - 1].fin;
        if (trace[(size_t)d * cap + i].start <= prev_fin) continue;  // no idle gap before it
        for (int q = i + 1; q < len; ++q) {
          const adaptis_task& y = cur[o + q];
          if (y.kind > 0 && pos[((size_t)(y.kind - 1) * S + y.stage) * m + y.mb] >= i) continue;
          const size_t base = cand.size();
          cand.insert(cand.end(), cur.begin(), cur.end());
          adaptis_task* c = cand.data() + base + o;
          const adaptis_task yy = c[q];
          for (int r2 = q; r2 > i; --r2) c[r2] = c[r2 - 1];
          c[i] = yy;
          ++nc;
          break;
        }
      }
    }
    if (nc == 0) break;
    std::vector<adaptis_plan> cplans(nc, *plan);
    std::vector<uint64_t> coff(nc * (p + 1));
    for (uint64_t c = 0; c < nc; ++c)
      for (int d = 0; d <= p; ++d) coff[c * (p + 1) + d] = c * total + offsets[d];
    std::vector<int64_t> cmk, crep; std::vector<uint8_t> cst;
    st = run_plans(ctx, P, cplans.data(), nc, &cmk, nullptr, nullptr, &cst, &crep, nullptr, cand.data(),
                   coff.data());
    if (st != ADAPTIS_OK) return st;
    int64_t best = -1, bov = 0, bmk = 0;
    for (uint64_t c = 0; c < nc; ++c) {
      if (cst[c] != ADAPTIS_CAND_OK || cmk[c] > cur_mk) continue;
      const int64_t ov = overlap_of(crep, c);
      if (ov <= cur_ov) continue;
      if (best < 0 || ov > bov || (ov == bov && cmk[c] < bmk)) { best = (int64_t)c; bov = ov; bmk = cmk[c]; }
    }
    if (best < 0) break;
    std::copy(cand.begin() + best * total, cand.begin() + (best + 1) * total, cur.begin());
    ++swaps;
    st = run_plans(ctx, P, plan, 1, &mk, nullptr, nullptr, &stt, &rep, nullptr, cur.data(), offsets, &trace, &cap);
    if (st != ADAPTIS_OK) return st;
    cur_mk = mk[0]; cur_ov = overlap_of(rep, 0); cur_st = stt[0];
  }
  std::copy(cur.begin(), cur.end(), tasks_out);
  *n_swaps = swaps;
  if (overlap_after) *overlap_after = cur_st == 0 ? cur_ov : 0;
  memset(result, 0, sizeof(*result));
  result->makespan = cur_mk;
  result->status = cur_st;
  result->makespan_f32 = cur_st == 0 ? (float)cur_mk : INFINITY;
  result->throughput = (cur_st == 0 && cur_mk > 0 && P->tick_seconds > 0)
      ? (double)m * (double)P->tokens_per_mb / ((double)cur_mk * P->tick_seconds) : 0.0;
  return ADAPTIS_OK;
}

adaptis_status adaptis_eval_indices(adaptis_ctx* ctx, adaptis_prepared* P, const uint64_t* indices,
                                    uint64_t n, const adaptis_results_soa* out) {
  if (!ctx || !P) return fail(ctx, ADAPTIS_EINVAL, "ctx or prepared is NULL");
  if (!out) return fail(ctx, ADAPTIS_EINVAL, "out is NULL");
  if (n && !indices) return fail(ctx, ADAPTIS_EINVAL, "indices is NULL");
  if (n == 0) return ADAPTIS_OK;
  // slots grouped by segment (one launch each), in the caller's order within a segment
  std::vector<std::vector<uint64_t>> by_seg(P->segs.size());
  for (uint64_t q = 0; q < n; ++q) {
    const uint64_t i = indices[q];
    if (i >= P->N)
      return fail(ctx, ADAPTIS_EINVAL, "indices[%llu] = %llu >= |space| = %llu", (unsigned long long)q,
                  (unsigned long long)i, (unsigned long long)P->N);
    size_t lo = 0, hi = P->segs.size();
    while (hi - lo > 1) {  // last segment with base <= i
      const size_t mid = (lo + hi) / 2;
      if (P->segs[mid].base <= i) lo = mid; else hi = mid;
    }
    by_seg[lo].push_back(q);
  }
  std::vector<uint64_t> slots;
  slots.reserve(n);
  for (auto& v : by_seg) slots.insert(slots.end(), v.begin(), v.end());
  CU(ctx, cudaSetDevice(ctx->device));
  uint64_t *d_idx = nullptr, *d_slots = nullptr;
  void* tmp[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  adaptis_status st = ADAPTIS_OK;
  auto cleanup = [&]() { cudaFree(d_idx); cudaFree(d_slots); for (void* t : tmp) cudaFree(t); };
#define CUI(call) do { cudaError_t e_ = (call); if (e_ != cudaSuccess) { cleanup(); \
    return fail(ctx, ADAPTIS_ECUDA, "%s: %s", #call, cudaGetErrorString(e_)); } } while (0)
  CUI(cudaMalloc(&d_idx, n * 8));
  CUI(cudaMalloc(&d_slots, n * 8));
  CUI(cudaMemcpyAsync(d_idx, indices, n * 8, cudaMemcpyHostToDevice, ctx->stream));
  CUI(cudaMemcpyAsync(d_slots, slots.data(), n * 8, cudaMemcpyHostToDevice, ctx->stream));
  adaptis_results_soa dout{};
  if (out->makespan) { CUI(cudaMalloc(&tmp[0], n * 8)); dout.makespan = (int64_t*)tmp[0]; }
  if (out->peak_mem_bytes) { CUI(cudaMalloc(&tmp[1], n * 8)); dout.peak_mem_bytes = (int64_t*)tmp[1]; }
  if (out->bubble_ratio) { CUI(cudaMalloc(&tmp[2], n * 4)); dout.bubble_ratio = (float*)tmp[2]; }
  if (out->status) { CUI(cudaMalloc(&tmp[3], n)); dout.status = (uint8_t*)tmp[3]; }
  if (out->makespan_f32) { CUI(cudaMalloc(&tmp[4], n * 4)); dout.makespan_f32 = (float*)tmp[4]; }
  std::vector<Job> jobs;
  uint64_t off = 0;
  for (size_t i = 0; i < P->segs.size(); ++i) {
    const uint64_t k = by_seg[i].size();
    if (k == 0) continue;
    const Seg& sg = P->segs[i];
    Job j{};
    j.s = make_launch(P, sg);
    j.s.lo = sg.base; j.s.hi = sg.base + sg.count;
    j.s.n_pos = k; j.s.n0 = k; j.s.world = 1;
    j.s.list_slot = d_slots + off;
    j.s.slot_idx = d_idx;
    j.info.group = sg.group; j.info.combo = sg.combo; j.info.v = sg.v;
    j.info.placement = sg.placement; j.info.policy = sg.policy;
    jobs.push_back(j);
    off += k;
  }
  st = run_jobs(ctx, P, jobs, false, &dout, 0, nullptr, nullptr, false);
  if (st != ADAPTIS_OK) { cleanup(); return st; }
  if (out->makespan) CUI(cudaMemcpyAsync(out->makespan, tmp[0], n * 8, cudaMemcpyDeviceToHost, ctx->stream));
  if (out->peak_mem_bytes) CUI(cudaMemcpyAsync(out->peak_mem_bytes, tmp[1], n * 8, cudaMemcpyDeviceToHost, ctx->stream));
  if (out->bubble_ratio) CUI(cudaMemcpyAsync(out->bubble_ratio, tmp[2], n * 4, cudaMemcpyDeviceToHost, ctx->stream));
  if (out->status) CUI(cudaMemcpyAsync(out->status, tmp[3], n, cudaMemcpyDeviceToHost, ctx->stream));
  if (out->makespan_f32) CUI(cudaMemcpyAsync(out->makespan_f32, tmp[4], n * 4, cudaMemcpyDeviceToHost, ctx->stream));
  CUI(cudaStreamSynchronize(ctx->stream));
#undef CUI
  cleanup();
  return ADAPTIS_OK;
}

static adaptis_status eval_plans_common(adaptis_ctx* ctx, adaptis_prepared* P, const adaptis_plan* plans,
                                        uint64_t n, const adaptis_results_soa* out, int64_t* report,
                                        const adaptis_task* tasks, const uint64_t* offsets) {
  if (!ctx || !P) return fail(ctx, ADAPTIS_EINVAL, "ctx or prepared is NULL");
  if (!out) return fail(ctx, ADAPTIS_EINVAL, "out is NULL");
  if (n && !plans) return fail(ctx, ADAPTIS_EINVAL, "plans is NULL");
  if (P->tick == kTickF32) return fail(ctx, ADAPTIS_EINVAL, "FP32 cost mode is not supported for explicit plans");
  std::vector<int64_t> mk, pk, rep;
  std::vector<float> bub;
  std::vector<uint8_t> stt;
  adaptis_status st = run_plans(ctx, P, plans, n, &mk, &pk, &bub, &stt, report ? &rep : nullptr, nullptr,
                                tasks, offsets);
  if (st != ADAPTIS_OK) return st;
  for (uint64_t i = 0; i < n; ++i) {
    if (out->makespan) out->makespan[i] = mk[i];
    if (out->peak_mem_bytes) out->peak_mem_bytes[i] = pk[i];
    if (out->bubble_ratio) out->bubble_ratio[i] = bub[i];
    if (out->status) out->status[i] = stt[i];
    if (out->makespan_f32) out->makespan_f32[i] = stt[i] == 0 ? (float)mk[i] : INFINITY;
  }
  if (report)
    for (uint64_t i = 0; i < n; ++i)
      if (stt[i] == ADAPTIS_CAND_OK || stt[i] == ADAPTIS_CAND_OVER_CAP)
        expand_report(rep.data() + (size_t)i * 5 * P->p, report + (size_t)i * kReportRows * P->p, P->p);
  return ADAPTIS_OK;
}

adaptis_status adaptis_eval_plans(adaptis_ctx* ctx, adaptis_prepared* P, const adaptis_plan* plans,
                                  uint64_t n, const adaptis_results_soa* out, int64_t* report) {
  for (uint64_t i = 0; i < n && plans; ++i)
    if (plans[i].policy == ADAPTIS_LIST || plans[i].policy == ADAPTIS_LIST_FUSED)
      return fail(ctx, ADAPTIS_EINVAL, "plans[%llu]: LIST policies go through adaptis_eval_lists",
                  (unsigned long long)i);
  return eval_plans_common(ctx, P, plans, n, out, report, nullptr, nullptr);
}

adaptis_status adaptis_realize_lists(adaptis_ctx* ctx, adaptis_prepared* P, const adaptis_plan* plan,
                                     adaptis_task* tasks_out, uint64_t cap, uint64_t* offsets_out) {
  if (!ctx || !P) return fail(ctx, ADAPTIS_EINVAL, "ctx or prepared is NULL");
  if (!plan || !tasks_out || !offsets_out) return fail(ctx, ADAPTIS_EINVAL, "a pointer argument is NULL");
  if (P->tick == kTickF32) return fail(ctx, ADAPTIS_EINVAL, "FP32 cost mode is not supported for realised lists");
  if (plan->policy == ADAPTIS_LIST || plan->policy == ADAPTIS_LIST_FUSED)
    return fail(ctx, ADAPTIS_EINVAL, "plan.policy = %d: an explicit schedule is already realised", plan->policy);
  const uint64_t need = (uint64_t)P->p * 3 * (uint64_t)P->m * (plan->v > 0 ? plan->v : 1);
  if (cap < need)
    return fail(ctx, ADAPTIS_EINVAL, "cap = %llu < p * 3 * m * v = %llu", (unsigned long long)cap,
                (unsigned long long)need);
  std::vector<int64_t> mk; std::vector<uint8_t> stt; std::vector<TraceEntry> tr; int tcap = 0;
  adaptis_status st = run_plans(ctx, P, plan, 1, &mk, nullptr, nullptr, &stt, nullptr, nullptr, nullptr, nullptr,
                                &tr, &tcap);
  if (st != ADAPTIS_OK) return st;
  if (stt[0] == ADAPTIS_CAND_INVALID) return fail(ctx, ADAPTIS_EINVAL, "plan cuts are not strictly increasing");
  if (stt[0] == ADAPTIS_CAND_STUCK)
    return fail(ctx, ADAPTIS_EINFEASIBLE, "the plan's policy gets stuck (R14): no complete order");
  // status 0 or 2: every device executed all of its m v (2 or 3) tasks, in trace order
  const int per_dev = (plan->policy == ADAPTIS_GPIPE || plan->policy == ADAPTIS_ONEF1B ? 2 : 3) * P->m * plan->v;
  if (per_dev > tcap) return fail(ctx, ADAPTIS_ECUDA, "trace capacity %d < %d tasks per device", tcap, per_dev);
  uint64_t k = 0;
  for (int d = 0; d < P->p; ++d) {
    offsets_out[d] = k;
    for (int i = 0; i < per_dev; ++i) {
      const TraceEntry& e = tr[(size_t)d * tcap + i];
      tasks_out[k].kind = e.kind;
      tasks_out[k].stage = e.stage;
      tasks_out[k].mb = e.mb;
      ++k;
    }
  }
  offsets_out[P->p] = k;
  return ADAPTIS_OK;
}

adaptis_status adaptis_memory_timeline(adaptis_ctx* ctx, adaptis_prepared* P, const adaptis_plan* plan,
                                       const adaptis_task* tasks, const uint64_t* offsets, adaptis_mem_point* out,
                                       uint64_t cap_points, uint64_t* dev_offsets, int64_t* first_violation) {
  if (!ctx || !P) return fail(ctx, ADAPTIS_EINVAL, "ctx or prepared is NULL");
  if (!plan || !out || !dev_offsets || !first_violation) return fail(ctx, ADAPTIS_EINVAL, "a pointer argument is NULL");
  if (P->tick == kTickF32) return fail(ctx, ADAPTIS_EINVAL, "FP32 cost mode is not supported for the memory timeline");
  const bool lists = plan->policy == ADAPTIS_LIST || plan->policy == ADAPTIS_LIST_FUSED;
  if (lists != (tasks != nullptr && offsets != nullptr))
    return fail(ctx, ADAPTIS_EINVAL, "plan.policy = %d: task lists are %s", plan->policy,
                lists ? "required (LIST policies)" : "only for LIST policies");
  if (lists) {
    if (plan->S != P->p * plan->v || plan->S < 1 || plan->S > ADAPTIS_MAX_S)
      return fail(ctx, ADAPTIS_EINVAL, "plan.S = %d != p * v", plan->S);
    adaptis_status st = validate_lists(ctx, P, plan, tasks, offsets, 1);
    if (st != ADAPTIS_OK) return st;
  }
  const uint64_t need = (uint64_t)P->p * (1 + 3 * (uint64_t)P->m * plan->v);
  if (cap_points < need)
    return fail(ctx, ADAPTIS_EINVAL, "cap_points = %llu < p (1 + 3 m v) = %llu", (unsigned long long)cap_points,
                (unsigned long long)need);
  std::vector<int64_t> mk; std::vector<uint8_t> stt;
  MemTimelineReq mt;
  adaptis_status st = run_plans(ctx, P, plan, 1, &mk, nullptr, nullptr, &stt, nullptr, nullptr, tasks, offsets,
                                nullptr, nullptr, &mt);
  if (st != ADAPTIS_OK) return st;
  if (stt[0] == ADAPTIS_CAND_INVALID) return fail(ctx, ADAPTIS_EINVAL, "plan cuts are not strictly increasing");
  uint64_t k = 0;
  for (int d = 0; d < P->p; ++d) {
    dev_offsets[d] = k;
    const int np = mt.npts[d];
    for (int i = 0; i < np; ++i) out[k++] = mt.points[(size_t)d * mt.pcap + i];
    first_violation[d] = mt.first[d];
  }
  dev_offsets[P->p] = k;
  return ADAPTIS_OK;
}

adaptis_status adaptis_eval_lists(adaptis_ctx* ctx, adaptis_prepared* P, const adaptis_plan* plans,
                                  const adaptis_task* tasks, const uint64_t* offsets, uint64_t n,
                                  const adaptis_results_soa* out, int64_t* report) {
  if (!ctx || !P) return fail(ctx, ADAPTIS_EINVAL, "ctx or prepared is NULL");
  if (n && (!plans || !tasks || !offsets)) return fail(ctx, ADAPTIS_EINVAL, "plans, tasks or offsets is NULL");
  for (uint64_t i = 0; i < n; ++i) {
    const adaptis_plan& pl = plans[i];
    if (pl.policy != ADAPTIS_LIST && pl.policy != ADAPTIS_LIST_FUSED)
      return fail(ctx, ADAPTIS_EINVAL, "plans[%llu].policy = %d is not ADAPTIS_LIST or ADAPTIS_LIST_FUSED",
                  (unsigned long long)i, pl.policy);
    if (pl.S != P->p * pl.v || pl.S < 1 || pl.S > ADAPTIS_MAX_S)
      return fail(ctx, ADAPTIS_EINVAL, "plans[%llu].S = %d != p * v", (unsigned long long)i, pl.S);
  }
  adaptis_status st = validate_lists(ctx, P, plans, tasks, offsets, n);
  if (st != ADAPTIS_OK) return st;
  return eval_plans_common(ctx, P, plans, n, out, report, tasks, offsets);
}

// R34: explicit lists with communication-engine contention (adaptis_contend.cu)
adaptis_status adaptis_eval_lists_contended(adaptis_ctx* ctx, adaptis_prepared* P, const adaptis_plan* plans,
                                            const adaptis_task* tasks, const uint64_t* offsets, uint64_t n,
                                            const adaptis_results_soa* out, int64_t* report) {
  if (!ctx || !P) return fail(ctx, ADAPTIS_EINVAL, "ctx or prepared is NULL");
  if (!out) return fail(ctx, ADAPTIS_EINVAL, "out is NULL");
  if (n && (!plans || !tasks || !offsets)) return fail(ctx, ADAPTIS_EINVAL, "plans, tasks or offsets is NULL");
  if (P->tick == kTickF32) return fail(ctx, ADAPTIS_EINVAL, "FP32 cost mode is not supported for explicit plans");
  const int p = P->p, m = P->m, L = P->L;
  int Smax = 1;
  std::vector<adaptis_plan> hp(plans, plans + n);
  for (uint64_t i = 0; i < n; ++i) {
    adaptis_plan& pl = hp[i];
    if (pl.policy != ADAPTIS_LIST && pl.policy != ADAPTIS_LIST_FUSED)
      return fail(ctx, ADAPTIS_EINVAL, "plans[%llu].policy = %d is not ADAPTIS_LIST or ADAPTIS_LIST_FUSED",
                  (unsigned long long)i, pl.policy);
    const bool ok_pl = pl.v == 1 ? pl.placement == ADAPTIS_SEQ
                                 : (pl.placement == ADAPTIS_INTERLEAVED || pl.placement == ADAPTIS_WAVE);
    if (pl.v < 1 || pl.v > ADAPTIS_MAX_V || pl.S != p * pl.v || pl.S > ADAPTIS_MAX_S || pl.S > L ||
        (pl.v > 1 && m % p != 0) || !ok_pl)
      return fail(ctx, ADAPTIS_EINVAL, "plans[%llu]: v = %d, S = %d, placement %d not admitted (R10, R12)",
                  (unsigned long long)i, pl.v, pl.S, pl.placement);
    pl.cuts[0] = 0;
    pl.cuts[pl.S] = (int16_t)L;
    for (int k = 0; k < pl.S; ++k)
      if (pl.cuts[k + 1] <= pl.cuts[k])
        return fail(ctx, ADAPTIS_EINVAL, "plans[%llu]: cuts are not strictly increasing in [1, L-1]",
                    (unsigned long long)i);
    Smax = std::max(Smax, pl.S);
  }
  adaptis_status st = validate_lists(ctx, P, hp.data(), tasks, offsets, n);
  if (st != ADAPTIS_OK) return st;
  // packed transfer keys hold eligibility times < 2^40: bound the makespan by
  // every task and every transfer run back to back
  {
    long double bound = 0;
    for (int l = 0; l < L; ++l)
      bound += (long double)m * (P->h_cols[(size_t)kColTF * L + l] + P->h_cols[(size_t)kColTB * L + l] +
                                 P->h_cols[(size_t)kColTW * L + l]) +
               2.0L * m * P->h_comm[l];
    if (bound >= (long double)(1ull << 40))
      return fail(ctx, ADAPTIS_EOVERFLOW, "serial bound %.0Lf ticks >= 2^40 (contention keys)", bound);
  }
  const uint64_t stride = (uint64_t)5 * Smax * m;
  if ((long double)n * stride * 8 > (long double)(1ull << 31))
    return fail(ctx, ADAPTIS_EINVAL, "%llu plans need %.0Lf B of scratch (> 2 GiB): split the list",
                (unsigned long long)n, (long double)n * stride * 8);
  if (n == 0) return ADAPTIS_OK;
  CU(ctx, cudaSetDevice(ctx->device));
  uint64_t ntask = 0;  // plans may share or reorder task ranges: copy up to the largest end
  for (uint64_t i = 0; i < n; ++i) ntask = std::max(ntask, offsets[i * (uint64_t)(p + 1) + p]);
  adaptis_plan* d_plans = nullptr; adaptis_task* d_tasks = nullptr; uint64_t* d_off = nullptr;
  int64_t *d_scr = nullptr, *d_mk = nullptr, *d_pk = nullptr, *d_rep = nullptr;
  float* d_bub = nullptr; uint8_t* d_st = nullptr; unsigned long long* d_nt = nullptr;
  auto cleanup = [&]() {
    cudaFree(d_plans); cudaFree(d_tasks); cudaFree(d_off); cudaFree(d_scr); cudaFree(d_mk);
    cudaFree(d_pk); cudaFree(d_rep); cudaFree(d_bub); cudaFree(d_st); cudaFree(d_nt);
  };
#define CUC(call) do { cudaError_t e_ = (call); if (e_ != cudaSuccess) { cleanup(); \
    return fail(ctx, ADAPTIS_ECUDA, "%s: %s", #call, cudaGetErrorString(e_)); } } while (0)
  CUC(cudaMalloc(&d_plans, n * sizeof(adaptis_plan)));
  CUC(cudaMalloc(&d_tasks, std::max<uint64_t>(ntask, 1) * sizeof(adaptis_task)));
  CUC(cudaMalloc(&d_off, n * (p + 1) * 8));
  CUC(cudaMalloc(&d_scr, n * stride * 8));
  CUC(cudaMalloc(&d_mk, n * 8));
  CUC(cudaMalloc(&d_pk, n * 8));
  CUC(cudaMalloc(&d_bub, n * 4));
  CUC(cudaMalloc(&d_st, n));
  CUC(cudaMalloc(&d_nt, 8));
  if (report) CUC(cudaMalloc(&d_rep, n * 5 * p * 8));
  CUC(cudaMemcpyAsync(d_plans, hp.data(), n * sizeof(adaptis_plan), cudaMemcpyHostToDevice, ctx->stream));
  CUC(cudaMemcpyAsync(d_tasks, tasks, ntask * sizeof(adaptis_task), cudaMemcpyHostToDevice, ctx->stream));
  CUC(cudaMemcpyAsync(d_off, offsets, n * (p + 1) * 8, cudaMemcpyHostToDevice, ctx->stream));
  CUC(cudaMemsetAsync(d_nt, 0, 8, ctx->stream));
  CUC(cudaEventRecord(ctx->ev0, ctx->stream));
  const int e = launch_contend(P->d_cols, P->d_comm, L, p, m, P->cap, n, d_plans, d_tasks, d_off, d_scr, stride,
                               d_mk, d_pk, d_bub, d_st, d_rep, d_nt, Smax, ctx->stream);
  if (e) { cleanup(); return fail(ctx, ADAPTIS_ECUDA, "contention kernel: %s", cudaGetErrorString((cudaError_t)e)); }
  CUC(cudaEventRecord(ctx->ev1, ctx->stream));
  ctx->launches += 1;
  std::vector<int64_t> mk(n), pk(n), rep(report ? n * 5 * p : 0);
  std::vector<float> bub(n);
  std::vector<uint8_t> stt(n);
  unsigned long long nt = 0;
  CUC(cudaMemcpyAsync(mk.data(), d_mk, n * 8, cudaMemcpyDeviceToHost, ctx->stream));
  CUC(cudaMemcpyAsync(pk.data(), d_pk, n * 8, cudaMemcpyDeviceToHost, ctx->stream));
  CUC(cudaMemcpyAsync(bub.data(), d_bub, n * 4, cudaMemcpyDeviceToHost, ctx->stream));
  CUC(cudaMemcpyAsync(stt.data(), d_st, n, cudaMemcpyDeviceToHost, ctx->stream));
  CUC(cudaMemcpyAsync(&nt, d_nt, 8, cudaMemcpyDeviceToHost, ctx->stream));
  if (report) CUC(cudaMemcpyAsync(rep.data(), d_rep, n * 5 * p * 8, cudaMemcpyDeviceToHost, ctx->stream));
  CUC(cudaStreamSynchronize(ctx->stream));
  float ms = 0;
  cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
  ctx->counters[0] += nt;
  ctx->last_tasks = nt;
  ctx->last_info.clear();
  adaptis_launch_info li{};
  li.group = -1; li.combo = -1; li.v = hp[0].v; li.placement = hp[0].placement; li.policy = hp[0].policy;
  li.candidates = n; li.tasks = nt; li.ms = ms;
  ctx->last_info.push_back(li);
#undef CUC
  cleanup();
  for (uint64_t i = 0; i < n; ++i) {
    if (out->makespan) out->makespan[i] = mk[i];
    if (out->peak_mem_bytes) out->peak_mem_bytes[i] = pk[i];
    if (out->bubble_ratio) out->bubble_ratio[i] = bub[i];
    if (out->status) out->status[i] = stt[i];
    if (out->makespan_f32) out->makespan_f32[i] = stt[i] == 0 ? (float)mk[i] : INFINITY;
  }
  if (report)
    for (uint64_t i = 0; i < n; ++i)
      if (stt[i] == ADAPTIS_CAND_OK || stt[i] == ADAPTIS_CAND_OVER_CAP)
        expand_report(rep.data() + (size_t)i * 5 * p, report + (size_t)i * kReportRows * p, p);
  return ADAPTIS_OK;
}

// Pipeline Generator (reading R28): seeds, then rounds of
// partition / placement / schedule tuning, each accepted only if it strictly
// lowers the makespan (rollback otherwise), until a round changes nothing.
adaptis_status adaptis_generate(adaptis_ctx* ctx, const adaptis_problem* problem,
                                const adaptis_gen_options* options, adaptis_gen_result* out) {
  if (!ctx) return fail(nullptr, ADAPTIS_EINVAL, "ctx is NULL");
  if (!out) return fail(ctx, ADAPTIS_EINVAL, "out is NULL");
  memset(out, 0, sizeof(*out));
  adaptis_gen_options o{};
  if (options) o = *options;
  const uint32_t vs_mask = o.vs_mask ? o.vs_mask : 0x3u;
  const int R = o.radius ? o.radius : 2;
  const int max_rounds = o.max_rounds ? o.max_rounds : 32;
  if (o.mode != ADAPTIS_GEN_BOTTLENECK && o.mode != ADAPTIS_GEN_ROUND_ROBIN)
    return fail(ctx, ADAPTIS_EINVAL, "options.mode = %d is not ADAPTIS_GEN_BOTTLENECK or ADAPTIS_GEN_ROUND_ROBIN", o.mode);
  if (R < 1 || R > kMaxRadius) return fail(ctx, ADAPTIS_EINVAL, "options.radius = %d not in [1, %d]", R, kMaxRadius);
  if (max_rounds < 1) return fail(ctx, ADAPTIS_EINVAL, "options.max_rounds = %d < 1", max_rounds);
  if (vs_mask & ~0xFu) return fail(ctx, ADAPTIS_EINVAL, "options.vs_mask = 0x%x admits v > 4", vs_mask);
  if (!problem) return fail(ctx, ADAPTIS_EINVAL, "problem is NULL");
  if (problem->cost_type != ADAPTIS_COST_TICKS)
    return fail(ctx, ADAPTIS_EINVAL, "adaptis_generate: FP32 cost mode is not supported");
  const int L = problem->layers.L, p = problem->p, m = problem->m;
  // admitted v values (ascending): S = p*v <= min(64, L); v > 1 needs m % p == 0 (R10)
  std::vector<int> vs;
  for (int v = 1; v <= ADAPTIS_MAX_V; ++v)
    if (((vs_mask >> (v - 1)) & 1u) && p * v <= std::min(ADAPTIS_MAX_S, L) && (v == 1 || m % p == 0))
      vs.push_back(v);
  if (vs.empty()) return fail(ctx, ADAPTIS_EINVAL, "options.vs_mask admits no v with p*v <= min(64, L)");
  // tables: one prepared space (FULL v = vs[0], validated by build_space) for the plan lists
  adaptis_space base{};
  base.n_groups = 1;
  base.group[0].v = vs[0];
  base.group[0].part_mode = ADAPTIS_PART_BALL;  // any valid space: the tables only depend on the problem
  base.group[0].radius = 0;
  base.group[0].combo_mask = 1u << 1;
  adaptis_prepared* P = nullptr;
  adaptis_status st = adaptis_prepare(ctx, problem, &base, &P);
  if (st != ADAPTIS_OK) return st;
  float ms = 0;
  uint64_t n_eval = 0;
  auto mist = [&](int S, adaptis_plan* pl) {
    int16_t c[ADAPTIS_MAX_S];
    seed_minmax(problem->layers, S, c);
    for (int i = 1; i < S; ++i) pl->cuts[i] = c[i - 1];
    pl->cuts[0] = 0; pl->cuts[S] = (int16_t)L;
  };
  auto make = [&](int v, int placement, int policy) {
    adaptis_plan pl{};
    pl.v = v; pl.placement = placement; pl.policy = policy; pl.S = p * v;
    return pl;
  };
  // evaluate a list, pick the first plan with the smallest makespan among status 0
  auto eval_best = [&](const std::vector<adaptis_plan>& list, int* best, int64_t* best_mk) -> adaptis_status {
    std::vector<int64_t> mk; std::vector<uint8_t> stt;
    float t = 0;
    adaptis_status s2 = run_plans(ctx, P, list.data(), list.size(), &mk, nullptr, nullptr, &stt, nullptr, &t);
    ms += t;
    n_eval += list.size();
    *best = -1; *best_mk = INT64_MAX;
    if (s2 != ADAPTIS_OK) return s2;
    for (size_t i = 0; i < list.size(); ++i)
      if (stt[i] == ADAPTIS_CAND_OK && mk[i] < *best_mk) { *best = (int)i; *best_mk = mk[i]; }
    return ADAPTIS_OK;
  };
  auto push_step = [&](int phase, int64_t mk) {
    if (out->n_steps < ADAPTIS_GEN_MAX_STEPS) {
      out->step_phase[out->n_steps] = phase;
      out->step_makespan[out->n_steps] = mk;
      out->n_steps++;
    }
  };
  // ---- seeds: partitions {equal layers (S-1F1B), min-max (Mist, R20)} x
  // placement/schedule {S-1F1B, ZB} on SEQ (v = 1), {I-1F1B, ZB} on INTERLEAVED and
  // Hanayo WAVE with the dynamic schedule (v >= 2; R12 admits no fixed 1F1B/ZB order on WAVE)
  std::vector<adaptis_plan> seeds;
  for (int v : vs) {
    const int S = p * v;
    for (int part = 0; part < 2; ++part) {
      std::vector<std::pair<int, int>> combos;
      if (v == 1) combos = {{ADAPTIS_SEQ, ADAPTIS_ONEF1B}, {ADAPTIS_SEQ, ADAPTIS_ZB}};
      else combos = {{ADAPTIS_INTERLEAVED, ADAPTIS_ONEF1B}, {ADAPTIS_INTERLEAVED, ADAPTIS_ZB},
                     {ADAPTIS_WAVE, ADAPTIS_GREEDY}};
      for (auto& c : combos) {
        adaptis_plan pl = make(v, c.first, c.second);
        if (part == 0) {
          for (int i = 1; i < S; ++i) pl.cuts[i] = (int16_t)((int64_t)i * L / S);
          pl.cuts[0] = 0; pl.cuts[S] = (int16_t)L;
        } else {
          mist(S, &pl);
        }
        seeds.push_back(pl);
      }
    }
  }
  out->n_seeds = (int32_t)seeds.size();
  int bi; int64_t cur_mk;
  st = eval_best(seeds, &bi, &cur_mk);
  if (st != ADAPTIS_OK) { adaptis_prepared_free(P); return st; }
  if (bi < 0) {
    out->n_evaluated = n_eval; out->kernel_ms = ms; out->p = p;
    adaptis_prepared_free(P);
    return fail(ctx, ADAPTIS_EINFEASIBLE, "no seed pipeline satisfies the memory constraint (Eq. 2)");
  }
  adaptis_plan cur = seeds[bi];
  push_step(ADAPTIS_GEN_SEED, cur_mk);
  // ---- tuning rounds
  int rounds = 0;
  // phase (a) of R28: the exact best of the L1 ball of radius R around the cuts
  auto ball_phase = [&](bool* improved) -> adaptis_status {
    adaptis_space sp{};
    sp.n_groups = 1;
    int16_t seed[ADAPTIS_MAX_S];
    for (int i = 1; i < cur.S; ++i) seed[i - 1] = cur.cuts[i];
    sp.group[0].v = cur.v; sp.group[0].part_mode = ADAPTIS_PART_BALL; sp.group[0].radius = R;
    sp.group[0].seed_cuts = seed;
    sp.group[0].combo_mask = 1u << combo_bit(cur.v, cur.placement, cur.policy);
    adaptis_prepared* Q = nullptr;
    adaptis_status s2 = adaptis_prepare(ctx, problem, &sp, &Q);
    if (s2 != ADAPTIS_OK) return s2;
    adaptis_plan best{}; int64_t bmk = INT64_MAX;
    s2 = best_of_space(ctx, Q, &best, &bmk, &ms);
    n_eval += Q->N;
    adaptis_prepared_free(Q);
    if (s2 != ADAPTIS_OK && s2 != ADAPTIS_EINFEASIBLE) return s2;
    if (s2 == ADAPTIS_OK && bmk < cur_mk) {
      cur = best; cur_mk = bmk; *improved = true;
      push_step(ADAPTIS_GEN_PARTITION, cur_mk);
    }
    return ADAPTIS_OK;
  };
  // R28': the schedule re-tuned in tandem: the first admitted policy of
  // smallest makespan for a partition and placement
  auto best_policy = [&](adaptis_plan q, adaptis_plan* out_pl, int64_t* out_mk) -> adaptis_status {
    std::vector<adaptis_plan> list;
    for (int pol = ADAPTIS_GPIPE; pol <= ADAPTIS_GREEDY; ++pol)
      if (combo_bit(q.v, q.placement, pol) >= 0) { q.policy = pol; list.push_back(q); }
    int b; int64_t bm;
    adaptis_status s2 = eval_best(list, &b, &bm);
    if (s2 != ADAPTIS_OK) return s2;
    *out_mk = b >= 0 ? bm : INT64_MAX;
    if (b >= 0) *out_pl = list[b];
    return ADAPTIS_OK;
  };
  // R28': BubbleTime(d) = T_d - busy_d - exposed_d (R29) and T_d of the current
  // plan, and the largest stage cost C_s = t_F + t_B + t_W of one micro-batch
  std::vector<int64_t> bubt(p), Td(p);
  int64_t maxcs = 0;
  auto profile = [&]() -> adaptis_status {
    std::vector<int64_t> mk1, rep1; std::vector<uint8_t> st1;
    float t = 0;
    adaptis_status s2 = run_plans(ctx, P, &cur, 1, &mk1, nullptr, nullptr, &st1, &rep1, &t);
    ms += t;
    if (s2 != ADAPTIS_OK) return s2;
    for (int d = 0; d < p; ++d) {
      Td[d] = rep1[d];
      bubt[d] = rep1[d] - rep1[p + d] - rep1[4 * p + d];
    }
    maxcs = 0;
    for (int s2i = 0; s2i < cur.S; ++s2i) {
      int64_t c = 0;
      for (int l = cur.cuts[s2i]; l < cur.cuts[s2i + 1]; ++l)
        c += P->h_cols[(size_t)kColTF * L + l] + P->h_cols[(size_t)kColTB * L + l] + P->h_cols[(size_t)kColTW * L + l];
      maxcs = std::max(maxcs, c);
    }
    return ADAPTIS_OK;
  };
  auto spread = [&]() {
    return *std::max_element(bubt.begin(), bubt.end()) - *std::min_element(bubt.begin(), bubt.end());
  };
  // R28' partition: one-layer transfers from the stage of the device with
  // the lowest bubble ratio to that of the highest, while they help and the
  // BubbleTime spread is >= max C_s; else the ball as the alternative adjustment
  auto partition_phase = [&](bool* improved) -> adaptis_status {
    bool acc = false;
    for (;;) {
      adaptis_status s2 = profile();
      if (s2 != ADAPTIS_OK) return s2;
      if (spread() < maxcs) break;
      int lo = 0, hi = 0;  // bubble ratios compared exactly (cross products < 2^62)
      for (int d = 1; d < p; ++d) {
        if (bubt[d] * Td[lo] < bubt[lo] * Td[d]) lo = d;
        if (bubt[d] * Td[hi] > bubt[hi] * Td[d]) hi = d;
      }
      if (lo == hi) break;
      int bs = -1, bt = -1, bdist = 1 << 30;  // the closest (src, dst) stage pair, then the lowest
      for (int a = 0; a < cur.S; ++a) {
        if (host_dev_of(cur.placement, p, a) != lo) continue;
        for (int b = 0; b < cur.S; ++b) {
          if (host_dev_of(cur.placement, p, b) != hi) continue;
          const int dist = a > b ? a - b : b - a;
          if (dist < bdist) { bdist = dist; bs = a; bt = b; }
        }
      }
      adaptis_plan q = cur;
      if (bs < bt) for (int i = bs + 1; i <= bt; ++i) q.cuts[i] -= 1;
      else for (int i = bt + 1; i <= bs; ++i) q.cuts[i] += 1;
      bool ok = true;
      for (int i = 0; i < q.S; ++i) ok = ok && q.cuts[i] < q.cuts[i + 1];
      if (!ok) break;
      adaptis_plan bp{}; int64_t bm = INT64_MAX;
      s2 = best_policy(q, &bp, &bm);
      if (s2 != ADAPTIS_OK) return s2;
      if (bm >= cur_mk) break;  // rolled back
      cur = bp; cur_mk = bm; acc = true;
      push_step(ADAPTIS_GEN_PARTITION, cur_mk);
    }
    if (acc) { *improved = true; return ADAPTIS_OK; }
    return ball_phase(improved);
  };
  // R28' placement: every other admitted (v, placement), cuts kept for
  // the same v (else the Mist seed), the schedule re-tuned in tandem
  auto placement_phase = [&](bool* improved) -> adaptis_status {
    adaptis_plan best{}; int64_t bmk = INT64_MAX;
    for (int v : vs) {
      std::vector<int> pls = v == 1 ? std::vector<int>{ADAPTIS_SEQ}
                                    : std::vector<int>{ADAPTIS_INTERLEAVED, ADAPTIS_WAVE};
      for (int pl : pls) {
        if (v == cur.v && pl == cur.placement) continue;
        adaptis_plan q = make(v, pl, ADAPTIS_GREEDY);
        if (v == cur.v) memcpy(q.cuts, cur.cuts, sizeof(q.cuts));
        else mist(p * v, &q);
        adaptis_plan bp{}; int64_t bm = INT64_MAX;
        adaptis_status s2 = best_policy(q, &bp, &bm);
        if (s2 != ADAPTIS_OK) return s2;
        if (bm < bmk) { bmk = bm; best = bp; }
      }
    }
    if (bmk < cur_mk) {
      cur = best; cur_mk = bmk; *improved = true;
      push_step(ADAPTIS_GEN_PLACEMENT, cur_mk);
    }
    return ADAPTIS_OK;
  };
  auto schedule_phase = [&](bool* improved) -> adaptis_status {
    std::vector<adaptis_plan> list;
    for (int pol = ADAPTIS_GPIPE; pol <= ADAPTIS_GREEDY; ++pol) {
      if (pol == cur.policy || combo_bit(cur.v, cur.placement, pol) < 0) continue;
      adaptis_plan q = cur;
      q.policy = pol;
      list.push_back(q);
    }
    if (list.empty()) return ADAPTIS_OK;
    int b3; int64_t mk3;
    adaptis_status s2 = eval_best(list, &b3, &mk3);
    if (s2 != ADAPTIS_OK) return s2;
    if (b3 >= 0 && mk3 < cur_mk) {
      cur = list[b3]; cur_mk = mk3; *improved = true;
      push_step(ADAPTIS_GEN_SCHEDULE, cur_mk);
    }
    return ADAPTIS_OK;
  };
  for (; o.mode == ADAPTIS_GEN_BOTTLENECK && rounds < max_rounds;) {
    ++rounds;
    st = profile();
    if (st != ADAPTIS_OK) { adaptis_prepared_free(P); return st; }
    // the bottleneck phase first, then the alternatives; one accepted step per round
    const bool part_first = spread() >= maxcs;
    bool improved = false;
    for (int k = 0; k < 3 && !improved; ++k) {
      const int ph = part_first ? k : (k + 1) % 3;  // 0 partition, 1 placement, 2 schedule
      st = ph == 0 ? partition_phase(&improved) : ph == 1 ? placement_phase(&improved) : schedule_phase(&improved);
      if (st != ADAPTIS_OK) { adaptis_prepared_free(P); return st; }
    }
    if (!improved) break;
  }
  for (; o.mode == ADAPTIS_GEN_ROUND_ROBIN && rounds < max_rounds;) {
    ++rounds;
    bool improved = false;
    // (a) partition: exact best of the L1 ball of radius R around the cuts
    {
      adaptis_space sp{};
      sp.n_groups = 1;
      int16_t seed[ADAPTIS_MAX_S];
      for (int i = 1; i < cur.S; ++i) seed[i - 1] = cur.cuts[i];
      sp.group[0].v = cur.v; sp.group[0].part_mode = ADAPTIS_PART_BALL; sp.group[0].radius = R;
      sp.group[0].seed_cuts = seed;
      sp.group[0].combo_mask = 1u << combo_bit(cur.v, cur.placement, cur.policy);
      adaptis_prepared* Q = nullptr;
      st = adaptis_prepare(ctx, problem, &sp, &Q);
      if (st != ADAPTIS_OK) { adaptis_prepared_free(P); return st; }
      adaptis_plan best{}; int64_t bmk = INT64_MAX;
      st = best_of_space(ctx, Q, &best, &bmk, &ms);
      n_eval += Q->N;
      adaptis_prepared_free(Q);
      if (st != ADAPTIS_OK && st != ADAPTIS_EINFEASIBLE) { adaptis_prepared_free(P); return st; }
      if (st == ADAPTIS_OK && bmk < cur_mk) {
        cur = best; cur_mk = bmk; improved = true;
        push_step(ADAPTIS_GEN_PARTITION, cur_mk);
      }
    }
    // (b) placement: grouped stage-device permutations (INT <-> WAVE) and v changes
    {
      std::vector<adaptis_plan> list;
      for (int v : vs) {
        std::vector<int> pls = v == 1 ? std::vector<int>{ADAPTIS_SEQ}
                                      : std::vector<int>{ADAPTIS_INTERLEAVED, ADAPTIS_WAVE};
        for (int pl : pls) {
          if (v == cur.v && pl == cur.placement) continue;
          const int pol = combo_bit(v, pl, cur.policy) >= 0 ? cur.policy : ADAPTIS_GREEDY;
          adaptis_plan q = make(v, pl, pol);
          if (v == cur.v) memcpy(q.cuts, cur.cuts, sizeof(q.cuts));
          else mist(p * v, &q);
          list.push_back(q);
        }
      }
      if (!list.empty()) {
        int b2; int64_t mk2;
        st = eval_best(list, &b2, &mk2);
        if (st != ADAPTIS_OK) { adaptis_prepared_free(P); return st; }
        if (b2 >= 0 && mk2 < cur_mk) {
          cur = list[b2]; cur_mk = mk2; improved = true;
          push_step(ADAPTIS_GEN_PLACEMENT, cur_mk);
        }
      }
    }
    // (c) schedule: every policy R12 admits for the placement
    {
      std::vector<adaptis_plan> list;
      for (int pol = ADAPTIS_GPIPE; pol <= ADAPTIS_GREEDY; ++pol) {
        if (pol == cur.policy || combo_bit(cur.v, cur.placement, pol) < 0) continue;
        adaptis_plan q = cur;
        q.policy = pol;
        list.push_back(q);
      }
      if (!list.empty()) {
        int b3; int64_t mk3;
        st = eval_best(list, &b3, &mk3);
        if (st != ADAPTIS_OK) { adaptis_prepared_free(P); return st; }
        if (b3 >= 0 && mk3 < cur_mk) {
          cur = list[b3]; cur_mk = mk3; improved = true;
          push_step(ADAPTIS_GEN_SCHEDULE, cur_mk);
        }
      }
    }
    if (!improved) break;
  }
  // ---- report of the final plan
  std::vector<int64_t> mk, pk, rep; std::vector<float> bub; std::vector<uint8_t> stt;
  float t = 0;
  st = run_plans(ctx, P, &cur, 1, &mk, &pk, &bub, &stt, &rep, &t);  // not counted in n_evaluated
  ms += t;
  adaptis_prepared_free(P);
  if (st != ADAPTIS_OK) return st;
  if (stt[0] != ADAPTIS_CAND_OK || mk[0] != cur_mk)
    return fail(ctx, ADAPTIS_ECUDA, "generator: final re-evaluation disagrees (%lld vs %lld)",
                (long long)mk[0], (long long)cur_mk);
  out->plan = cur;
  out->result.makespan = mk[0];
  out->result.peak_mem_bytes = pk[0];
  out->result.bubble_ratio = bub[0];
  out->result.status = stt[0];
  out->result.makespan_f32 = (float)mk[0];
  out->result.throughput = (mk[0] > 0 && problem->tick_seconds > 0)
      ? (double)m * (double)problem->tokens_per_microbatch / ((double)mk[0] * problem->tick_seconds) : 0.0;
  out->p = p;
  for (int d = 0; d < p; ++d) {
    out->T_d[d] = rep[d]; out->busy_d[d] = rep[p + d]; out->M_d[d] = rep[2 * p + d];
    out->comm_d[d] = rep[3 * p + d]; out->exposed_d[d] = rep[4 * p + d];
    out->overlap_d[d] = out->comm_d[d] - out->exposed_d[d];
    out->bubble_d[d] = out->T_d[d] - out->busy_d[d] - out->exposed_d[d];
  }
  out->rounds = rounds;
  out->n_evaluated = n_eval;
  out->kernel_ms = ms;
  return ADAPTIS_OK;
}

adaptis_status adaptis_shard_indices(const adaptis_problem* problem, const adaptis_space* space,
                                     int rank, int world, uint64_t* out, uint64_t cap,
                                     uint64_t* n_out) {
  if (!n_out) return fail(nullptr, ADAPTIS_EINVAL, "n_out is NULL");
  if (world < 1 || rank < 0 || rank >= world)
    return fail(nullptr, ADAPTIS_EINVAL, "rank = %d, world = %d", rank, world);
  adaptis_prepared P;
  adaptis_status st = build_space(nullptr, problem, space, &P);
  if (st != ADAPTIS_OK) return st;
  uint64_t n = 0;
  for (const Seg& sg : P.segs) {
    SegLaunch s{};
    shard(sg.base, sg.base + sg.count, rank, world, &s);
    for (uint64_t q = 0; q < s.n_pos; ++q, ++n)
      if (out && n < cap) out[n] = shard_index(q, s.n0, s.start0, s.first_chunk, s.world);
  }
  *n_out = n;
  return ADAPTIS_OK;
}

adaptis_status adaptis_search(adaptis_ctx* ctx, const adaptis_problem* problem,
                              const adaptis_space* space, adaptis_best* out) {
  adaptis_prepared* P = nullptr;
  adaptis_status st = adaptis_prepare(ctx, problem, space, &P);
  if (st != ADAPTIS_OK) return st;
  st = adaptis_search_prepared(ctx, P, out);
  adaptis_prepared_free(P);
  return st;
}

}  // extern "C"
