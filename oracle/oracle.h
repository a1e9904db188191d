/*
 * oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of what the AdaPtis
 * hot path computes (arXiv 2509.23722): the Pipeline Performance Model of
 * Alg. 1 evaluated by a global event-loop simulation, the
 * canonical candidate enumeration (reading R19 in DESIGN.md) and
 * the exhaustive argmin of Eq. 1-2.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library. It shares no code, header,
 * table or constant with the CUDA path (paper_2509_23722_b200/) and neither
 * includes the other.
 *
 * Every function states the passage it follows. Parity status of each
 * function is listed in DESIGN.md §"Oracle pins".
 */
#ifndef ADAPTIS_ORACLE_H
#define ADAPTIS_ORACLE_H
#include <stdint.h>

#define ORC_MAXS 64
#define ORC_MAXP 32

/* policies / placements / partition modes, numbered as in DESIGN.md R9-R14, R12, R19 */
#define ORC_GPIPE 0
#define ORC_ONEF1B 1
#define ORC_ZB 2
#define ORC_GREEDY 3
#define ORC_SEQ 0
#define ORC_INTERLEAVED 1
#define ORC_WAVE 2
#define ORC_FULL 0
#define ORC_BALL 1

#define ORC_OK 0
#define ORC_INVALID 1
#define ORC_OVER_CAP 2
#define ORC_STUCK 3

typedef struct {
  int L;
  const int64_t *t_f, *t_b, *t_w;           /* ProfiledCompCost per computation type */
  const int64_t *act, *stash, *weight, *grad; /* ProfiledMemCost, R16              */
  const int64_t *comm;                      /* boundary after row l (R3-R5)               */
  int p, m;
  int64_t cap;                              /* M_d^capacity (Eq. 2)                       */
  const double* costs_f64;                  /* optional [4][L] real t_f, t_b, t_w, comm:
                                               selects the fp64 simulator                 */
  int time_f32;                             /* with costs_f64: time arithmetic in fp32
                                               (the fp32-cost variant, R27)               */
} orc_problem;

typedef struct {
  int v, placement, policy, S;
  int cuts[ORC_MAXS + 1];                   /* cuts[0]=0 < ... < cuts[S]=L (or invalid)   */
} orc_plan;

typedef struct {
  int status;
  int64_t makespan;                         /* max_d T_d, INT64_MAX unless status 0       */
  int64_t peak_mem;                         /* max_d M_d                                  */
  double bubble;                            /* 1 - sum busy / (p * makespan)              */
  int64_t T_d[ORC_MAXP], busy_d[ORC_MAXP], M_d[ORC_MAXP], static_d[ORC_MAXP];
  double makespan_f;                        /* the makespan as a real number             */
  double T_f[ORC_MAXP];
} orc_result;

/* realised per-device order of one simulation (optional output of orc_simulate) */
typedef struct {
  int cap_per_dev;                          /* capacity of each per-device array          */
  int n[ORC_MAXP];                          /* tasks recorded per device                  */
  int *kind, *stage, *mb;                   /* [d*cap_per_dev + i]; kind 0=F 1=B 2=W      */
  int64_t *start;
} orc_trace;

typedef struct {
  int v, part_mode, radius;
  const int* seed_cuts;                     /* S-1 cuts or NULL (then the R20 seed)       */
  unsigned combo_mask;
} orc_group;

typedef struct {
  int n_groups;
  orc_group group[4];
} orc_space;

typedef struct {
  uint64_t index;                           /* UINT64_MAX if nothing feasible             */
  int64_t makespan;
  orc_plan plan;
  uint64_t n_total, n_invalid, n_simulated, n_feasible;
} orc_best;

/* Alg. 1 Step 1: stage sums by direct loops; stage_dev by R12. */
int  orc_device_of_stage(int placement, int p, int v, int s);
/* fixed F/B order of device d for GPIPE / ONEF1B / ZB (R9-R11); returns length */
int  orc_fixed_order(const orc_problem* pr, const orc_plan* pl, int d,
                     int* kind, int* stage, int* mb, int cap);
/* Alg. 1 Steps 1-3 for one candidate (global event loop, R9-R16). Returns 0,
 * or -1 on an internal inconsistency (a test failure). */
int  orc_simulate(const orc_problem* pr, const orc_plan* pl, orc_result* out, orc_trace* tr);
/* the same event loop with real-valued times (fp64) on pr->costs_f64 */
int  orc_simulate_f64(const orc_problem* pr, const orc_plan* pl, orc_result* out, orc_trace* tr);
/* the same event loop with fp32 times on pr->costs_f64 (values exact in fp32) */
int  orc_simulate_f32(const orc_problem* pr, const orc_plan* pl, orc_result* out, orc_trace* tr);
/* Independent checker: longest path over the task DAG (S:141 edges) plus the
 * given per-device list-order edges, by relaxation to a fixpoint. Returns 0,
 * or 1 if the lists contain a cyclic wait. fused: B charged c_B + c_W, no W. */
int  orc_longest_path(const orc_problem* pr, const orc_plan* pl, int fused,
                      const orc_trace* lists, int64_t* start_out, int64_t* makespan,
                      int64_t* T_d);
/* R20 seed: min-max contiguous S-way split of w[0..L), ties -> lexicographically
 * smallest cuts. Writes S-1 interior cuts; returns the min-max value. */
int64_t orc_seed_minmax(int L, const int64_t* w, int S, int* cuts_out);
/* R19 canonical order */
int  orc_combo(int v, int k, int* placement, int* policy);   /* 0 if combo k does not exist */
uint64_t orc_space_size(const orc_problem* pr, const orc_space* sp, int* overflow);
/* enumeration by recursive generation, calling cb(index, plan, user) in order */
typedef void (*orc_cb)(uint64_t index, const orc_plan* plan, void* user);
void orc_enumerate(const orc_problem* pr, const orc_space* sp, orc_cb cb, void* user);
/* random access by recursive descent over subtree sizes */
int  orc_decode(const orc_problem* pr, const orc_space* sp, uint64_t index, orc_plan* out);
/* plain helpers for tests/bench */
int  orc_eval_indices(const orc_problem* pr, const orc_space* sp, const uint64_t* idx,
                      uint64_t n, int nthreads, int64_t* makespan, int64_t* peak,
                      double* bubble, uint8_t* status, double* makespan_f);
/* exhaustive argmin of Eq. 1-2 with lowest-index tie-break (R18). prune=1
 * enables the exact lower-bound prune (skip if max_d busy_d > best, or equal
 * with a larger index) and the fixed-order memory precheck. */
int  orc_search(const orc_problem* pr, const orc_space* sp, int prune, int nthreads,
                orc_best* out);

#endif
