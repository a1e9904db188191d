/*
 * adaptis.h — C ABI of libadaptis.so: batched evaluation of the AdaPtis
 * Pipeline Performance Model (arXiv 2509.23722, Alg. 1) over an enumerated
 * space of (model partition, model placement, workload schedule) candidates,
 * reduced to the best plan that satisfies the memory constraint (Eq. 1-2).
 *
 * Citation convention: "P:n" = line n of the paper text, with the
 * section / algorithm / equation it falls in; "R<k>" = reading k in DESIGN.md
 * (where the paper is silent or ambiguous).
 *
 * Conventions for every call
 *  - All integers are host-endian. Inputs are structure-of-arrays.
 *  - Ownership: every pointer is owned by the caller. Inputs are only read
 *    during the call (and copied to the device); the caller may free them on
 *    return. Outputs are caller-allocated (host memory, or device memory when
 *    `out_on_device` is non-zero).
 *  - Errors: every call returns an adaptis_status. No C++ exception crosses
 *    the ABI. After a failure on a call that takes a context,
 *    adaptis_last_error(ctx) names the offending field, e.g.
 *    "layers.t_f[3] < 1". Calls without a context write the message to a
 *    thread-local buffer readable through adaptis_last_error(NULL).
 *  - Threads: one context per thread at a time; distinct contexts may be used
 *    concurrently.
 *  - Determinism: results are pure functions of the inputs (integer ticks and
 *    bytes, total-order argmin key), identical for any number of GPUs.
 */
#ifndef ADAPTIS_H
#define ADAPTIS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define ADAPTIS_API __attribute__((visibility("default")))
#else
#define ADAPTIS_API
#endif

#define ADAPTIS_MAX_P 32      /* pipeline devices per candidate (lanes of one warp)   */
#define ADAPTIS_MAX_V 4       /* virtual stages per device                            */
#define ADAPTIS_MAX_S 64      /* stages S = p*v                                       */
#define ADAPTIS_MAX_GROUPS 4  /* v-groups per search space                            */

typedef enum {
  ADAPTIS_OK = 0,
  ADAPTIS_EINVAL = 1,      /* invalid argument; adaptis_last_error names the field            */
  ADAPTIS_EINFEASIBLE = 2, /* search: no candidate satisfies Eq. 2                */
  ADAPTIS_EOVERFLOW = 3,   /* makespan bound and index do not fit the 63-bit argmin key       */
  ADAPTIS_ECUDA = 4,       /* CUDA runtime error (message in adaptis_last_error)              */
  ADAPTIS_ECOLL = 5        /* the cross-GPU allreduce callback failed                         */
} adaptis_status;

/* Model placement families (§2.3): SEQ = S-1F1B sequential (v = 1),
 * INTERLEAVED = I-1F1B virtual stages (stage s -> device s mod p),
 * WAVE = Hanayo wave (stage c*p+j -> device j for even c, p-1-j for odd c). */
enum { ADAPTIS_SEQ = 0, ADAPTIS_INTERLEAVED = 1, ADAPTIS_WAVE = 2 };

/* Workload-scheduling policies (§2.4, §4.3, readings R9-R14):
 * GPIPE and ONEF1B run B and W fused; ZB and GREEDY split them. */
enum { ADAPTIS_GPIPE = 0, ADAPTIS_ONEF1B = 1, ADAPTIS_ZB = 2, ADAPTIS_GREEDY = 3 };
/* Explicit per-device task orders ("workload scheduling results"; reading
 * R30), for adaptis_eval_lists only: LIST splits B and W (W tasks are listed),
 * LIST_FUSED runs B and W fused (no W tasks). */
enum { ADAPTIS_LIST = 4, ADAPTIS_LIST_FUSED = 5 };

/* One task of an explicit per-device order: kind 0 = F, 1 = B, 2 = W. */
typedef struct {
  int16_t kind;
  int16_t stage;             /* 0 <= stage < S, a stage of the listing device        */
  int32_t mb;                /* micro-batch, 0 <= mb < m                              */
} adaptis_task;

/* Cost arithmetic (R1): exact int64 ticks, or the fp32-cost variant whose
 * makespans agree with an fp64 evaluation within 1e-5 relative. */
enum { ADAPTIS_COST_TICKS = 0, ADAPTIS_COST_FP32 = 1 };

/* Partition spaces (R19): FULL = every contiguous S-way split of the L rows;
 * BALL = cut vectors within L1 distance `radius` of a seed partition. */
enum { ADAPTIS_PART_FULL = 0, ADAPTIS_PART_BALL = 1 };

/* Per-candidate status codes (adaptis_results_soa.status, adaptis_result.status). */
enum {
  ADAPTIS_CAND_OK = 0,
  ADAPTIS_CAND_INVALID = 1,  /* BALL decode whose cuts are not strictly increasing in [1, L-1] */
  ADAPTIS_CAND_OVER_CAP = 2, /* some M_d > M_d^capacity (Eq. 2)                    */
  ADAPTIS_CAND_STUCK = 3     /* the schedule cannot complete (cyclic wait / memory gate)        */
};

/* Fixed combo table (R12). Bit k of adaptis_group.combo_mask enables combo k.
 *   v == 1 : 0 SEQ x GPIPE, 1 SEQ x ONEF1B, 2 SEQ x ZB, 3 SEQ x GREEDY
 *   v >= 2 : 0 INT x GPIPE, 1 INT x ONEF1B, 2 INT x ZB, 3 INT x GREEDY,
 *            4 WAVE x GPIPE, 5 WAVE x GREEDY                                       */

/* Profiled data per layer row: ProfiledCompCost(l) and ProfiledMemCost(l) of
 * Alg. 1 Step 1, split by computation type F / B / W (P:152-153,
 * P:181). Row 0 is the embedding, row L-1 the LM head (R24). Each pointer is a
 * host array of L int64 values. */
typedef struct {
  int32_t L;                 /* rows, 2 <= L <= 32767                                        */
  const int64_t* t_f;        /* forward ticks per micro-batch, >= 1 (R17)                    */
  const int64_t* t_b;        /* input-gradient ticks, >= 1                                   */
  const int64_t* t_w;        /* parameter-gradient ticks, >= 1                               */
  const int64_t* act_bytes;  /* held from F start to B end, per micro-batch, >= 0 (R16)      */
  const int64_t* stash_bytes;/* held from F start to W end (B end when fused), >= 0          */
  const int64_t* weight_bytes;/* static from t = 0, >= 0                                     */
  const int64_t* grad_bytes; /* static from t = 0, >= 0                                      */
  const int64_t* comm_ticks; /* p2p latency of the boundary after row l, >= 0 (R3-R5);
                                entry L-1 is ignored                                         */
} adaptis_layers;

typedef struct {
  adaptis_layers layers;
  int32_t p;                  /* pipeline devices P, 1 <= p <= 32                            */
  int32_t m;                  /* micro-batches nmb, 1 <= m <= 65535                          */
  int64_t mem_cap_bytes;      /* M_d^capacity (uniform); INT64_MAX = unconstrained           */
  double  tick_seconds;       /* seconds per tick, throughput only (R22)                     */
  int64_t tokens_per_microbatch; /* throughput only (TS)                              */
  int32_t cost_type;          /* ADAPTIS_COST_TICKS (exact integer ticks, default) or
                                 ADAPTIS_COST_FP32 (all time arithmetic in fp32, R1)          */
  const float* costs_f32;     /* FP32 only, optional: [4][L] real-valued t_f, t_b, t_w, comm
                                 (each t >= 1, comm >= 0); NULL = the int64 tables as floats  */
} adaptis_problem;

typedef struct {              /* one group of the space per virtual-stage count v            */
  int32_t v;                  /* 1..4; S = p*v <= min(64, L); v > 1 requires m % p == 0 (R10)*/
  int32_t part_mode;          /* ADAPTIS_PART_FULL or ADAPTIS_PART_BALL                       */
  int32_t radius;             /* BALL only: L1 radius R >= 0                                  */
  const int16_t* seed_cuts;   /* BALL only: S-1 interior cuts, or NULL = min-max seed (R20)   */
  uint32_t combo_mask;        /* non-empty subset of the combo table above                    */
} adaptis_group;

typedef struct {
  int32_t n_groups;           /* 1..4; index order follows group order (R19)                  */
  adaptis_group group[ADAPTIS_MAX_GROUPS];
} adaptis_space;

/* A decoded candidate: stage s owns rows [cuts[s], cuts[s+1]), cuts[0] = 0,
 * cuts[S] = L ("consecutive layers"; Layers(s) of Table `tab: notations`). */
typedef struct {
  int32_t v, placement, policy, S;
  int16_t cuts[ADAPTIS_MAX_S + 1];
} adaptis_plan;

/* Per-candidate outputs, structure of arrays, `count` entries each. Any
 * pointer may be NULL to skip that output. */
typedef struct {
  int64_t* makespan;         /* max_d T_d (Eq. 1) in ticks; INT64_MAX unless status == 0    */
  int64_t* peak_mem_bytes;   /* max_d M_d (Alg. 1 Step 3); 0 for status 1 and 3            */
  float*   bubble_ratio;     /* 1 - sum_d busy_d / (p * makespan) (R7); 0 unless status 0   */
  uint8_t* status;           /* ADAPTIS_CAND_*                                              */
  float*   makespan_f32;     /* FP32 cost mode: the fp32 makespan (makespan above is it
                                rounded to the nearest tick); NULL to skip                  */
} adaptis_results_soa;

typedef struct {             /* host-side result of one candidate                            */
  int64_t makespan, peak_mem_bytes;
  float   bubble_ratio;
  double  throughput;        /* tokens/s = m * tokens_per_microbatch / (makespan * tick_s)   */
  uint8_t status;
  float   makespan_f32;      /* FP32 cost mode: the unrounded makespan                       */
} adaptis_result;

typedef struct {             /* output of adaptis_search                                     */
  uint64_t index;            /* global index of the winner (lowest index among ties, R18)    */
  adaptis_plan plan;
  adaptis_result result;
  int32_t p;
  int64_t T_d[ADAPTIS_MAX_P];    /* per-device completion time (Alg. 1 Step 3 output)        */
  int64_t busy_d[ADAPTIS_MAX_P]; /* per-device compute ticks                                  */
  int64_t M_d[ADAPTIS_MAX_P];    /* per-device peak memory, static + dynamic (Eq. 2)          */
  /* Alg. 1 Step 3 accounting (reading R29; integer ticks only): with
   * C_d = busy_d + comm_d, T_d = C_d + bubble_d - overlap_d holds exactly.       */
  int64_t comm_d[ADAPTIS_MAX_P];    /* ProfiledCommCost: sum of transfers sent or received by d  */
  int64_t exposed_d[ADAPTIS_MAX_P]; /* transfer time on d, within [0, T_d], while d computes nothing */
  int64_t overlap_d[ADAPTIS_MAX_P]; /* OverlapTime(d) = comm_d - exposed_d                     */
  int64_t bubble_d[ADAPTIS_MAX_P];  /* BubbleTime(d) = T_d - busy_d - exposed_d (>= 0)         */
  uint64_t n_candidates;     /* |space| (all ranks)                                          */
  uint64_t n_evaluated;      /* candidates this rank evaluated                               */
  uint64_t n_invalid;        /* of those, invalid decodes (status 1)                         */
  uint64_t n_tasks;          /* F/B/W tasks this rank simulated (work counter for the roofline) */
  uint64_t n_pruned;         /* candidates skipped by the exact lower-bound prune (0 if off)  */
  float    kernel_ms;        /* device time of this rank's evaluation kernels                */
} adaptis_best;

typedef struct adaptis_ctx adaptis_ctx;
typedef struct adaptis_prepared adaptis_prepared;

/* Cross-GPU reduction hook for world > 1: must replace *dev_key (one int64 in
 * device memory of this rank's GPU) by its minimum over all ranks, ordered
 * after the work already queued on `cuda_stream`, and return 0 on success.
 * The Python binding installs torch.distributed.all_reduce(MIN) over an NCCL
 * process group (one 8-byte allreduce per search). */
typedef int (*adaptis_allreduce_min_fn)(int64_t* dev_key, void* cuda_stream, void* user);

/* Create a context bound to `cuda_device`. rank/world describe the candidate
 * sharding (block-cyclic chunks of 65536 indices, chunk k -> rank k mod world).
 * EINVAL if world < 1 or rank not in [0, world); ECUDA if the device is
 * unusable. */
ADAPTIS_API adaptis_status adaptis_ctx_create(int cuda_device, int rank, int world, adaptis_ctx** out);
ADAPTIS_API void           adaptis_ctx_destroy(adaptis_ctx* ctx);
ADAPTIS_API adaptis_status adaptis_ctx_set_allreduce(adaptis_ctx* ctx, adaptis_allreduce_min_fn fn, void* user);
/* Exact lower-bound pruning for adaptis_search (default off; SURVEY §8d
 * "time-to-best-plan with and without LB pruning"): a candidate is skipped when
 * (LB << bits | index) exceeds the best key found so far, with LB = max_d of
 * head_d + busy_d + tail_d. head_d = t_F of the stages before d's lowest
 * stage (= d) plus the d edge latencies between them. Fused B/W: tail_d =
 * (t_B + t_W) of those stages plus the same latencies. Split B/W: the max of
 * head_d + busy_d and head_d + m (t_F + t_B)_d + t_B of those stages + the
 * latencies + t_W of stage 0 (derivation in adaptis_seg.cuh). Since
 * makespan >= LB it cannot win, so the winner is unchanged. Skipped
 * candidates are counted in adaptis_best.n_pruned. Ignored in FP32 cost mode. */
ADAPTIS_API adaptis_status adaptis_ctx_set_prune(adaptis_ctx* ctx, int enable);
/* The CUDA stream (cudaStream_t) every kernel of this context is queued on. */
ADAPTIS_API void*          adaptis_ctx_stream(adaptis_ctx* ctx);
/* Number of kernel launches this context has issued since creation. */
ADAPTIS_API uint64_t       adaptis_ctx_launch_count(const adaptis_ctx* ctx);
/* Candidates re-evaluated by the exact fallback kernel (shared-memory rings
 * too small for their dependency lag) since creation. */
ADAPTIS_API uint64_t       adaptis_ctx_fallback_count(const adaptis_ctx* ctx);
/* Per-launch record of the most recent evaluation (search or eval) of a
 * context: one entry per (group, combo) segment launched. */
typedef struct {
  int32_t group, combo, v, placement, policy;
  int32_t fallback;          /* candidates re-run by the fallback kernel            */
  uint64_t candidates;       /* candidates this launch evaluated                    */
  uint64_t tasks;            /* F/B/W tasks it simulated                             */
  float ms;                  /* device time of the launch (+ its fallback), CUDA events */
  int32_t kernel;            /* 0 lane-per-device segment kernel, 1 sequential GREEDY,
                                 2 static-order kernel (GPIPE / ONEF1B / ZB)            */
} adaptis_launch_info;
/* Copies up to `max` records of the last evaluation into `out`; returns how
 * many there are. The winner re-evaluation of a search is not included. */
ADAPTIS_API int            adaptis_ctx_launch_info(const adaptis_ctx* ctx, adaptis_launch_info* out, int max);
/* Cumulative work counters of this context since creation: out[0] simulated
 * tasks, out[1] warp simulation rounds, out[2] live device-lane rounds (lane
 * utilisation = out[0] / out[2]; tasks per warp-round = out[0] / out[1]). */
ADAPTIS_API void           adaptis_ctx_counters(const adaptis_ctx* ctx, uint64_t out[3]);

/* The static task order the static-order kernel evaluates for a GPIPE /
 * ONEF1B / ZB segment (Alg. 1 Step 3, under the fixed lists of
 * readings R9-R11): every device's F/B list merged into one
 * topological order of the DAG plus list edges, shared by all candidates with
 * these (policy, placement, p, v, m). Host only, no GPU needed.
 * entries[i] = stage | kind << 6 (0 F, 1 B) | in_slot << 8 | out_slot << 16 |
 * device << 24, where a slot (< 255; 255 = none) holds the arrival time of
 * the item the entry consumes (its F or B input) or produces. *n_entries =
 * 2 S m; *n_slots = the slots used. Caller owns `entries` (capacity `cap`).
 * EINVAL: bad arguments, p > 16, S > 64, or the lists deadlock / need more
 * than 254 slots (the lane kernels then evaluate the segment); EOVERFLOW:
 * cap < 2 S m (n_entries still set). */
ADAPTIS_API adaptis_status adaptis_static_order(int32_t policy, int32_t placement, int32_t p, int32_t v,
                                                int32_t m, uint32_t* entries, uint64_t cap,
                                                uint64_t* n_entries, int32_t* n_slots);

/* |space| for this problem (the candidate space). EINVAL on an
 * invalid problem/space; EOVERFLOW if the count does not fit in 63 bits. */
ADAPTIS_API adaptis_status adaptis_space_size(const adaptis_problem* problem, const adaptis_space* space,
                                  uint64_t* n_out);

/* Decode a global index into its (v, placement, policy, cuts) candidate, in the
 * canonical order of R19. EINVAL if index >= |space|. An invalid BALL decode
 * is still returned (its cuts are not strictly increasing). */
ADAPTIS_API adaptis_status adaptis_decode(const adaptis_problem* problem, const adaptis_space* space,
                              uint64_t index, adaptis_plan* out);

/* Validate, derive host tables (prefix sums, seeds, counts) and upload them to
 * the device once, so repeated evaluations start with inputs resident in HBM. */
ADAPTIS_API adaptis_status adaptis_prepare(adaptis_ctx* ctx, const adaptis_problem* problem,
                               const adaptis_space* space, adaptis_prepared** out);
ADAPTIS_API void           adaptis_prepared_free(adaptis_prepared* prep);

/* Evaluate candidates [first, first+count) of the space (Alg. 1 Steps 1-3 per
 * candidate) and write per-candidate results. Unlike search this is not
 * sharded: the context's GPU evaluates the whole range. */
ADAPTIS_API adaptis_status adaptis_eval_batch(adaptis_ctx* ctx, const adaptis_problem* problem,
                                  const adaptis_space* space, uint64_t first, uint64_t count,
                                  const adaptis_results_soa* out, int out_on_device);
ADAPTIS_API adaptis_status adaptis_eval_prepared(adaptis_ctx* ctx, adaptis_prepared* prep,
                                     uint64_t first, uint64_t count,
                                     const adaptis_results_soa* out, int out_on_device);

/* Search the whole space for min (makespan, index) over candidates with
 * status 0 (Eq. 1-2, ties to the lowest index, R18). With world > 1 every
 * rank evaluates its shard and the allreduce hook combines the packed keys;
 * every rank returns the same `out`. EINFEASIBLE if no candidate is feasible
 * (out->index = UINT64_MAX). */
ADAPTIS_API adaptis_status adaptis_search(adaptis_ctx* ctx, const adaptis_problem* problem,
                              const adaptis_space* space, adaptis_best* out);
ADAPTIS_API adaptis_status adaptis_search_prepared(adaptis_ctx* ctx, adaptis_prepared* prep,
                                       adaptis_best* out);

/* The candidates rank `rank` of `world` evaluates in a sharded search
 * (block-cyclic chunks of 65536 global indices, chunk k -> rank k mod world,
 * within every (group, combo) segment), in the order the kernels visit them.
 * Writes up to `cap` indices to `out` (may be NULL) and their total count to
 * *n_out. Host-only; used to check that the shards partition [0, |space|). */
ADAPTIS_API adaptis_status adaptis_shard_indices(const adaptis_problem* problem,
                                                 const adaptis_space* space, int rank, int world,
                                                 uint64_t* out, uint64_t cap, uint64_t* n_out);

/* Evaluate an arbitrary list of global indices of the prepared space (decoded
 * on the device, canonical order R19; Alg. 1 Steps 1-3 per candidate) and
 * write results to host arrays `out` (n entries each) in list order.
 * Duplicates are allowed. EINVAL if some index >= |space| (the message names
 * it). The context's GPU evaluates the whole list (no sharding). */
ADAPTIS_API adaptis_status adaptis_eval_indices(adaptis_ctx* ctx, adaptis_prepared* prep,
                                                const uint64_t* indices, uint64_t n,
                                                const adaptis_results_soa* out);

/* Evaluate plans with explicit per-device task orders (Alg. 1 Step 3 on given
 * workload scheduling results; reading R30). Plan i has policy
 * ADAPTIS_LIST or ADAPTIS_LIST_FUSED, any placement of R12 for its v, and its
 * device d executes tasks[offsets[i*(p+1)+d] .. offsets[i*(p+1)+d+1]) in order:
 * every (F, B[, W]) x own stage x micro-batch exactly once, with F(s,j) before
 * B(s,j) before W(s,j) on the device (else EINVAL naming plan, device and
 * task). Each plan's offsets are non-decreasing (else EINVAL); plans may share
 * or reorder task ranges: tasks[0 .. max_i offsets[i*(p+1)+p]) is read.
 * Cross-device waits follow the DAG; a cyclic wait gives status
 * STUCK, a peak above the cap OVER_CAP (split precedence, R26). Outputs as
 * adaptis_eval_plans (report [n][7][p] optional). Not in FP32 cost mode. */
ADAPTIS_API adaptis_status adaptis_eval_lists(adaptis_ctx* ctx, adaptis_prepared* prep,
                                              const adaptis_plan* plans, const adaptis_task* tasks,
                                              const uint64_t* offsets, uint64_t n,
                                              const adaptis_results_soa* out, int64_t* report);

/* adaptis_eval_lists with communication-engine contention (Alg. 1 Step 3,
 * P:322-328, with SPEC S:206 (a)/(c) and S:232; reading R34 in DESIGN.md).
 * Same plans, lists, validation and outputs as adaptis_eval_lists, but every
 * stage edge between different devices with latency > 0 is a transfer that,
 * once its producer finishes, holds the sender's send engine and the
 * receiver's receive engine together for its latency; each engine serves
 * transfers FIFO by (eligible time, mb, stage, F before B). Memory and the
 * stuck / over-cap status are those of the lists (R16, R26, R30). `report`
 * rows 3-6 (comm_d, exposed_d, overlap_d, bubble_d) use the transfers' actual
 * [start, arrival) intervals. EOVERFLOW if the serial bound (m x all task ticks + 2m x all
 * latencies) reaches 2^40 ticks; EINVAL if the per-plan scratch
 * (n x 5 x max S x m x 8 B) exceeds 2 GiB. Not in FP32 cost mode. */
ADAPTIS_API adaptis_status adaptis_eval_lists_contended(adaptis_ctx* ctx, adaptis_prepared* prep,
                                                        const adaptis_plan* plans, const adaptis_task* tasks,
                                                        const uint64_t* offsets, uint64_t n,
                                                        const adaptis_results_soa* out, int64_t* report);

/* OOM repair ("advances the execution of the latest B and W to ahead of
 * this time to free up memory, continuing this process until all potential OOM
 * errors are resolved"; reading R31) of one explicit schedule (policy LIST or
 * LIST_FUSED, lists as in adaptis_eval_lists). Each step evaluates the
 * schedule on the GPU, finds the earliest Eq. 2 violation (the first F of a
 * device whose allocation exceeds the cap, earliest start over devices, ties
 * to the lower device) and moves the latest-listed B of that device whose F
 * is listed earlier and whose input has arrived by that time to just before
 * the F (its W right after it when split). It stops when the schedule fits
 * (result->status 0), nothing can move or it got stuck (status 2 / 3), or
 * after max_moves moves (<= 0: the number of tasks). tasks_out (same size and
 * offsets as the input) receives the repaired lists; *n_moves the moves made. */
ADAPTIS_API adaptis_status adaptis_repair_oom(adaptis_ctx* ctx, adaptis_prepared* prep,
                                              const adaptis_plan* plan, const adaptis_task* tasks,
                                              const uint64_t* offsets, int32_t max_moves,
                                              adaptis_task* tasks_out, adaptis_result* result,
                                              int32_t* n_moves);

/* Overlap-aware reordering ("avoid scheduling dependent computation
 * tasks consecutively and instead delay certain computations to enable
 * communication overlap"; reading R32) of one explicit schedule (LIST or
 * LIST_FUSED, status 0). Each round evaluates, in one GPU batch, every
 * schedule that moves the nearest later independent task (its own F / B
 * already listed) in front of a task whose device idled waiting for its
 * cross-device input, and accepts the one with the largest total OverlapTime
 * (R29) among those whose makespan does not grow and whose overlap grows
 * (ties: smaller makespan, then first). It stops when no candidate qualifies
 * or after max_swaps accepted moves (<= 0: the number of tasks). tasks_out
 * receives the tuned lists (offsets unchanged); overlap_* (may be NULL) the
 * total OverlapTime before and after. */
ADAPTIS_API adaptis_status adaptis_tune_overlap(adaptis_ctx* ctx, adaptis_prepared* prep,
                                                const adaptis_plan* plan, const adaptis_task* tasks,
                                                const uint64_t* offsets, int32_t max_swaps,
                                                adaptis_task* tasks_out, adaptis_result* result,
                                                int32_t* n_swaps, int64_t* overlap_before,
                                                int64_t* overlap_after);

/* Evaluate an explicit list of plans (Alg. 1 Steps 1-3 per plan),
 * e.g. the neighbourhood of one Pipeline Generator step. `prep`
 * must have been prepared from the same problem (any space; its tables are
 * reused). Plan i: S == p*v, 1 <= v <= 4, S <= min(64, L), v > 1 requires
 * m % p == 0, and (placement, policy) must be a combo of R12 (WAVE admits only
 * GPIPE and GREEDY); else EINVAL naming the plan. cuts[0] and cuts[S] are taken
 * as 0 and L; cuts that are not strictly increasing give status 1 (INVALID).
 * Results go to host arrays `out` (n entries each) in plan order; `report`,
 * when non-NULL, is a host array [n][7][p] receiving T_d, busy_d, M_d, comm_d,
 * exposed_d, overlap_d and bubble_d (R29, see adaptis_best: overlap_d =
 * comm_d - exposed_d is Alg. 1's OverlapTime(d), bubble_d = T_d - busy_d -
 * exposed_d its BubbleTime(d)) of every plan with status 0 or 2 (untouched
 * otherwise); its trace scratch (n * p * 3mv * 24 B) must stay
 * under 2 GiB (EINVAL). Not in FP32 cost mode (EINVAL). The context's GPU
 * evaluates the whole list. */
ADAPTIS_API adaptis_status adaptis_eval_plans(adaptis_ctx* ctx, adaptis_prepared* prep,
                                              const adaptis_plan* plans, uint64_t n,
                                              const adaptis_results_soa* out, int64_t* report);

/* Contention on realised orders (Alg. 1 Step 3 with SPEC S:206 (a)/(c) and
 * S:232; reading R36 in DESIGN.md): every candidate's policy decides its
 * per-device order with pure-latency communication (R3-R6); that order is
 * then executed as an explicit schedule (R30) under send/receive-engine
 * contention (R34), on the GPU in batches (the policy kernels with traces, a
 * conversion kernel and the contention kernel). adaptis_eval_contended writes
 * per-candidate results for [first, first + count) to host arrays `out`
 * (candidates without a complete order keep their policy status 1 or 3);
 * adaptis_search_contended is the argmin of Eq. 1-2 over the contended
 * makespans (lowest index among ties, R18) on this context's GPU, with the
 * winner's T_d / busy_d / M_d. EOVERFLOW if the serial bound reaches 2^40
 * ticks; not in FP32 cost mode. */
ADAPTIS_API adaptis_status adaptis_eval_contended(adaptis_ctx* ctx, adaptis_prepared* prep, uint64_t first,
                                                  uint64_t count, const adaptis_results_soa* out);
ADAPTIS_API adaptis_status adaptis_search_contended(adaptis_ctx* ctx, adaptis_prepared* prep, adaptis_best* out);

/* Realised workload scheduling results of one policy plan ("workload
 * scheduling results"; the Executor's compute-instruction lists): the
 * order in which each device executes its tasks under the plan's policy, as
 * explicit lists in the format of adaptis_eval_lists (reading R30): device d's
 * tasks are tasks_out[offsets_out[d] .. offsets_out[d+1]) (offsets_out has p + 1
 * entries; tasks_out holds `cap` entries, at most p * 3 * m * v are written,
 * EINVAL if too small). Fused policies (GPIPE, ONEF1B) give LIST_FUSED lists
 * (no W), split ones LIST lists; evaluating them with the matching LIST policy
 * reproduces the plan's result. EINFEASIBLE if the plan does not complete
 * (STUCK: no full order exists). Not in FP32 cost mode. */
ADAPTIS_API adaptis_status adaptis_realize_lists(adaptis_ctx* ctx, adaptis_prepared* prep,
                                                 const adaptis_plan* plan, adaptis_task* tasks_out,
                                                 uint64_t cap, uint64_t* offsets_out);

/* Memory timeline of one plan (Eq. 2; "identifies potential
 * OOM time"; SPEC memory_timeline S:213-221; reading R35 in DESIGN.md): per
 * device, the piecewise-constant memory M_d(t) = static + dynamic bytes as
 * breakpoints (time, bytes) in event order, starting with (0, static):
 * act + stash are allocated at an F's start, act freed at its B's end, stash
 * at its W's end (at the B's end when fused, R16); per-device events are
 * totally ordered on the device's engine (a free at t precedes an allocation
 * at t). `plan` is a policy plan (as adaptis_eval_plans) or, with `tasks` and
 * `offsets` (as adaptis_eval_lists, one plan), an explicit schedule. Device d's
 * breakpoints go to out[dev_offsets[d] .. dev_offsets[d+1]) (caller arrays:
 * dev_offsets has p + 1 entries; out holds `cap_points`, at most p (1 + 3 m v)
 * are written, EINVAL if too small); first_violation[d] is the first time
 * M_d exceeds the memory cap, -1 if never. A STUCK plan's timeline stops at
 * the stall. Not in FP32 cost mode. */
typedef struct { int64_t time, bytes; } adaptis_mem_point;
ADAPTIS_API adaptis_status adaptis_memory_timeline(adaptis_ctx* ctx, adaptis_prepared* prep,
                                                   const adaptis_plan* plan, const adaptis_task* tasks,
                                                   const uint64_t* offsets, adaptis_mem_point* out,
                                                   uint64_t cap_points, uint64_t* dev_offsets,
                                                   int64_t* first_violation);

/* Pipeline Generator (§4.3; readings R28 / R28' in DESIGN.md): seeds
 * from the baseline partitions (S-1F1B equal-layer and Mist min-max, R20),
 * placements (S-1F1B, I-1F1B, Hanayo) and schedules (S-1F1B, ZB) of P:346, then
 * rounds of phase-by-phase tuning with rollback, each step accepted
 * only if it strictly lowers the makespan, until a round changes nothing.
 * ADAPTIS_GEN_BOTTLENECK (R28', default): each round tunes the bottleneck phase
 * first (the partition when the spread of BubbleTime(d) is at least the
 * largest stage cost C_s; else placement, schedule, partition); the
 * partition phase transfers one layer at a time from the stage of the device
 * with the lowest bubble ratio to that of the highest while it helps,
 * else takes the best of the L1 ball of radius `radius` (one GPU search);
 * placement and partition changes re-tune the schedule in tandem (the
 * best policy R12 admits). ADAPTIS_GEN_ROUND_ROBIN (R28, round 1): partition
 * (ball), placement, schedule in every round. */
enum { ADAPTIS_GEN_BOTTLENECK = 0, ADAPTIS_GEN_ROUND_ROBIN = 1 };
typedef struct {
  uint32_t vs_mask;          /* bit v-1 admits v virtual stages per device; 0 = {1, 2}        */
  int32_t  radius;           /* partition-phase L1 radius, >= 1; 0 = 2                        */
  int32_t  max_rounds;       /* tuning rounds, >= 1; 0 = 32                                   */
  int32_t  mode;             /* ADAPTIS_GEN_BOTTLENECK (0) or ADAPTIS_GEN_ROUND_ROBIN         */
} adaptis_gen_options;

#define ADAPTIS_GEN_MAX_STEPS 128
enum { ADAPTIS_GEN_SEED = 0, ADAPTIS_GEN_PARTITION = 1, ADAPTIS_GEN_PLACEMENT = 2,
       ADAPTIS_GEN_SCHEDULE = 3 };

typedef struct {
  adaptis_plan plan;         /* the co-optimised pipeline                                     */
  adaptis_result result;
  int32_t p;
  int64_t T_d[ADAPTIS_MAX_P], busy_d[ADAPTIS_MAX_P], M_d[ADAPTIS_MAX_P];
  int64_t comm_d[ADAPTIS_MAX_P], exposed_d[ADAPTIS_MAX_P];   /* as in adaptis_best (R29)       */
  int64_t overlap_d[ADAPTIS_MAX_P], bubble_d[ADAPTIS_MAX_P];
  int32_t n_seeds;           /* seed plans evaluated                                          */
  int32_t rounds;            /* tuning rounds run (the last one changed nothing)              */
  uint64_t n_evaluated;      /* plans simulated in total (seeds + every neighbourhood)        */
  int32_t n_steps;           /* accepted steps: the chosen seed, then each accepted tuning    */
  int32_t step_phase[ADAPTIS_GEN_MAX_STEPS];     /* ADAPTIS_GEN_*                             */
  int64_t step_makespan[ADAPTIS_GEN_MAX_STEPS];  /* makespan after the step (strictly falling) */
  float   kernel_ms;         /* device time of all evaluation kernels                         */
} adaptis_gen_result;

/* EINVAL on an invalid problem/options (or FP32 cost mode); EINFEASIBLE if no
 * seed satisfies Eq. 2 (out->n_steps = 0). */
ADAPTIS_API adaptis_status adaptis_generate(adaptis_ctx* ctx, const adaptis_problem* problem,
                                            const adaptis_gen_options* options,
                                            adaptis_gen_result* out);

/* Executor lowering (AdaPtis §5 Pipeline Executor, Table
 * `tab:instruction_types`; reading R33; host only, no GPU needed). One
 * instruction of a device program; comm ops carry the boundary `stage` b
 * (between stages b and b+1), the micro-batch and the peer device; computes
 * carry their stage and peer -1. */
enum { ADAPTIS_OP_C_F = 0, ADAPTIS_OP_C_B = 1, ADAPTIS_OP_C_W = 2, ADAPTIS_OP_S_F = 3,
       ADAPTIS_OP_S_B = 4, ADAPTIS_OP_R_F = 5, ADAPTIS_OP_R_B = 6, ADAPTIS_OP_W_F = 7,
       ADAPTIS_OP_W_B = 8 };
typedef struct { int32_t op, stage, mb, peer; } adaptis_instr;
#define ADAPTIS_LOWER_REPAIR 1   /* hoist receives until the rendezvous run completes */
#define ADAPTIS_LOWER_HOIST 2    /* hoist every receive as early as stays deadlock-free */
/* Lower one explicit schedule (plan policy LIST / LIST_FUSED on p devices, lists
 * as in adaptis_eval_lists) to per-device instruction programs: R and W before
 * a compute with a cross-device input, S right after one with a cross-device
 * output; then, per `flags`, deadlock repair and receive hoisting
 * under rendezvous semantics (an S and its R proceed together). Writes
 * the programs to out (capacity `cap`; 4 x the number of tasks always
 * suffices) with device d at out[out_offsets[d] .. out_offsets[d+1]).
 * EINVAL (message: adaptis_lower_error()) on invalid input, a too small `out`,
 * or a deadlock that hoisting receives cannot repair. */
ADAPTIS_API adaptis_status adaptis_lower(int32_t p, const adaptis_plan* plan, const adaptis_task* tasks,
                                         const uint64_t* offsets, int32_t flags, adaptis_instr* out,
                                         uint64_t cap, uint64_t* out_offsets, int32_t* n_repairs,
                                         int32_t* n_hoists);
ADAPTIS_API const char*    adaptis_lower_error(void);

/* Message of the last failure on `ctx` (or of the calling thread when ctx is NULL). */
ADAPTIS_API const char*    adaptis_last_error(const adaptis_ctx* ctx);
ADAPTIS_API const char*    adaptis_status_str(adaptis_status s);

#ifdef __cplusplus
}
#endif
#endif /* ADAPTIS_H */
