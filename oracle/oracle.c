/*
 * oracle.c — TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * Plain CPU oracle of the AdaPtis Pipeline Performance Model (arXiv
 * 2509.23722). "P:n" = PAPER.md line n; "R<k>" = reading k in DESIGN.md.
 * Nothing here is blocked, fused or reordered beyond what the paper's
 * Alg. 1 / Eq. 1-2 and the readings state: stage sums are direct loops, the
 * schedule is a global event loop that executes, one at a time, the action
 * with the smallest (start time, device), and the search visits every
 * candidate of the canonical order produced by recursive generation.
 */
#include "oracle.h"

#include <limits.h>
#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#define UNK (-1) /* an unknown ready/finish time (times are >= 0) */

enum { KF = 0, KB = 1, KW = 2 };

static int64_t max64(int64_t a, int64_t b) { return a > b ? a : b; }
static int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }

/* Alg. 1 Step 1: C_s / M_s = sum over Layers(s) of the profiled cost. */
static int64_t rows_sum(const int64_t* col, int a, int b) {
  int64_t s = 0;
  for (int l = a; l < b; l++) s += col[l];
  return s;
}

/* R12: stage -> device for the three placement families. */
int orc_device_of_stage(int placement, int p, int v, int s) {
  (void)v;
  if (placement == ORC_SEQ) return s;              /* S = P, stage i -> device i           */
  if (placement == ORC_INTERLEAVED) return s % p;  /* I-1F1B virtual stages                */
  int c = s / p, j = s % p;                        /* Hanayo wave: boustrophedon           */
  return (c % 2 == 0) ? j : p - 1 - j;
}

/* the stage that device d holds in stage group ("chunk") c */
static int stage_of_chunk(int placement, int p, int c, int d) {
  if (placement == ORC_SEQ) return d;
  if (placement == ORC_INTERLEAVED) return c * p + d;
  return c * p + ((c % 2 == 0) ? d : p - 1 - d);
}

/* R10: the k-th forward / backward of a device in Megatron's interleaved order
 * (for v = 1 this is simply micro-batch k). */
static void virt_fwd(int k, int p, int v, int* chunk, int* mb) {
  *chunk = (k / p) % v;
  *mb = (k / (p * v)) * p + k % p;
}
static void virt_bwd(int k, int p, int v, int* chunk, int* mb) {
  *chunk = v - 1 - (k / p) % v;
  *mb = (k / (p * v)) * p + k % p;
}

/* R9-R11: the fixed F/B list of device d. GPIPE: every F (R10 forward order)
 * then every B (R10 backward order). ONEF1B and ZB: w warm-up forwards, then
 * (F, B) pairs, then w cool-down backwards, with w = min(m, p-d-1) for v = 1
 * (S-1F1B) and w = min(mv, 2(p-d-1) + (v-1)p) for v > 1 (Megatron I-1F1B). */
int orc_fixed_order(const orc_problem* pr, const orc_plan* pl, int d, int* kind, int* stage,
                    int* mb, int cap) {
  int p = pr->p, m = pr->m, v = pl->v, total = m * v, n = 0, c, j;
#define PUSH(K, C, J)                                                     \
  do {                                                                    \
    if (n < cap) {                                                        \
      kind[n] = (K);                                                      \
      stage[n] = stage_of_chunk(pl->placement, p, (C), d);                \
      mb[n] = (J);                                                        \
    }                                                                     \
    n++;                                                                  \
  } while (0)
  if (pl->policy == ORC_GPIPE) {
    for (int k = 0; k < total; k++) { virt_fwd(k, p, v, &c, &j); PUSH(KF, c, j); }
    for (int k = 0; k < total; k++) { virt_bwd(k, p, v, &c, &j); PUSH(KB, c, j); }
    return n;
  }
  int w;
  if (v == 1) w = (int)min64(m, p - d - 1);
  else w = (int)min64(total, 2 * (p - d - 1) + (v - 1) * p);
  for (int k = 0; k < w; k++) { virt_fwd(k, p, v, &c, &j); PUSH(KF, c, j); }
  for (int i = 0; i < total - w; i++) {
    virt_fwd(w + i, p, v, &c, &j); PUSH(KF, c, j);
    virt_bwd(i, p, v, &c, &j); PUSH(KB, c, j);
  }
  for (int i = total - w; i < total; i++) { virt_bwd(i, p, v, &c, &j); PUSH(KB, c, j); }
  return n;
#undef PUSH
}

static int cuts_valid(const orc_problem* pr, const orc_plan* pl) {
  if (pl->cuts[0] != 0 || pl->cuts[pl->S] != pr->L) return 0;
  for (int s = 0; s < pl->S; s++)
    if (pl->cuts[s + 1] <= pl->cuts[s]) return 0;
  return 1;
}

#define FIN(st, k, s, j) ((st)->fin[((size_t)(k) * (st)->c->S + (s)) * (st)->c->m + (j)])

static double rows_sum_f(const double* col, int a, int b) {
  double s = 0;
  for (int l = a; l < b; l++) s += col[l];
  return s;
}

/* exact integer ticks */
#define OT int64_t
#define OSUF(x) x
#define OTMAX INT64_MAX
#define OMAX max64
#define OMIN min64
#define ORND(x) (x)
#define ORC_F64 0
#define ORC_F32 0
#define COMM(row) (pr->comm[(row)])
#include "oracle_sim.inc"
#undef OT
#undef OSUF
#undef OTMAX
#undef OMAX
#undef OMIN
#undef ORND
#undef ORC_F64
#undef COMM

/* fp64 reference of the fp32-cost variant (costs from pr->costs_f64) */
#define OT double
#define OSUF(x) x##_f64
#define OTMAX HUGE_VAL
#define OMAX fmax
#define OMIN fmin
#define ORND(x) llround(x)
#define ORC_F64 1
#define COMM(row) (pr->costs_f64[3 * (size_t)pr->L + (row)])
#include "oracle_sim.inc"
#undef OT
#undef OSUF
#undef OTMAX
#undef OMAX
#undef OMIN
#undef ORND
#undef ORC_F32
#undef COMM

/* the fp32-cost variant in fp32 time arithmetic (reading R27): the same event
 * loop with every time value (finish, arrival, decision time) an fp32 number
 * produced by IEEE round-to-nearest additions, so that every scheduling
 * decision is taken in the precision the kernel takes it in */
static float fmaxf_(float a, float b) { return a > b ? a : b; }
static float fminf_(float a, float b) { return a < b ? a : b; }
#define OT float
#define OSUF(x) x##_f32
#define OTMAX HUGE_VALF
#define OMAX fmaxf_
#define OMIN fminf_
#define ORND(x) llroundf(x)
#define ORC_F32 1
#define COMM(row) ((float)pr->costs_f64[3 * (size_t)pr->L + (row)])
#include "oracle_sim.inc"
#undef OT
#undef OSUF
#undef OTMAX
#undef OMAX
#undef OMIN
#undef ORND
#undef ORC_F64
#undef ORC_F32
#undef COMM

/* ------------------------------------------------------------------------ */
/* Independent checker: longest path over DAG + list edges.          */
int orc_longest_path(const orc_problem* pr, const orc_plan* pl, int fused, const orc_trace* L_,
                     int64_t* start_out, int64_t* makespan, int64_t* T_d) {
  cand_t c;
  derive(pr, pl, &c);
  c.fused = fused;
  for (int s = 0; s < c.S; s++) {
    c.dur[KB][s] = fused ? c.cB[s] + c.cW[s] : c.cB[s];
  }
  const int S = c.S, m = pr->m, p = pr->p;
  size_t N = 3 * (size_t)S * m;
  int64_t* st = (int64_t*)calloc(N, sizeof(int64_t));
  int* listed = (int*)calloc(N, sizeof(int));
  int* prevnode = (int*)malloc(sizeof(int) * N);
  for (size_t i = 0; i < N; i++) prevnode[i] = -1;
#define NODE(k, s, j) (((k) * S + (s)) * m + (j))
  for (int d = 0; d < p; d++) {
    int prev = -1;
    for (int i = 0; i < L_->n[d]; i++) {
      int q = d * L_->cap_per_dev + i;
      int node = NODE(L_->kind[q], L_->stage[q], L_->mb[q]);
      listed[node] = 1;
      prevnode[node] = prev;
      prev = node;
    }
  }
  int cyc = 1;
  for (size_t it = 0; it <= N + 1; it++) {
    int changed = 0;
    for (int k = 0; k < 3; k++)
      for (int s = 0; s < S; s++)
        for (int j = 0; j < m; j++) {
          int node = NODE(k, s, j);
          if (!listed[node]) continue;
          int64_t t = 0;
          if (k == KF && s > 0) t = max64(t, st[NODE(KF, s - 1, j)] + c.dur[KF][s - 1] + c.xF[s]);
          if (k == KB) {
            t = max64(t, st[NODE(KF, s, j)] + c.dur[KF][s]);
            if (s < S - 1) t = max64(t, st[NODE(KB, s + 1, j)] + c.dur[KB][s + 1] + c.xB[s]);
          }
          if (k == KW) t = max64(t, st[NODE(KB, s, j)] + c.dur[KB][s]);
          int pv = prevnode[node];
          if (pv >= 0) {
            int pk = pv / (S * m), ps = (pv / m) % S;
            t = max64(t, st[pv] + c.dur[pk][ps]);
          }
          if (t != st[node]) { st[node] = t; changed = 1; }
        }
    if (!changed) { cyc = 0; break; }
  }
  int64_t mk = 0;
  for (int d = 0; d < p; d++) {
    int64_t td = 0;
    if (L_->n[d] > 0) {
      int q = d * L_->cap_per_dev + L_->n[d] - 1;
      int node = NODE(L_->kind[q], L_->stage[q], L_->mb[q]);
      td = st[node] + c.dur[L_->kind[q]][L_->stage[q]];
    }
    if (T_d) T_d[d] = td;
    mk = max64(mk, td);
    if (start_out)
      for (int i = 0; i < L_->n[d]; i++) {
        int q = d * L_->cap_per_dev + i;
        start_out[q] = st[NODE(L_->kind[q], L_->stage[q], L_->mb[q])];
      }
  }
#undef NODE
  *makespan = mk;
  free(st); free(listed); free(prevnode);
  return cyc;
}

/* ------------------------------------------------------------------------ */
/* R20 seed: Mist-style min-max contiguous partition, exact DP. */
int64_t orc_seed_minmax(int L, const int64_t* w, int S, int* cuts_out) {
  const int64_t INF = INT64_MAX;
  int64_t* pre = (int64_t*)malloc(sizeof(int64_t) * (L + 1));
  pre[0] = 0;
  for (int l = 0; l < L; l++) pre[l + 1] = pre[l] + w[l];
  /* best[k][i]: min over splits of rows [i, L) into k non-empty parts of the max part */
  int64_t* best = (int64_t*)malloc(sizeof(int64_t) * (size_t)(S + 1) * (L + 1));
#define BEST(k, i) best[(size_t)(k) * (L + 1) + (i)]
  for (int i = 0; i <= L; i++) BEST(0, i) = (i == L) ? 0 : INF;
  for (int k = 1; k <= S; k++)
    for (int i = 0; i <= L; i++) {
      int64_t b = INF;
      for (int j = i + 1; j <= L; j++) {
        if (BEST(k - 1, j) == INF) continue;
        int64_t val = max64(pre[j] - pre[i], BEST(k - 1, j));
        if (val < b) b = val;
      }
      BEST(k, i) = b;
    }
  int64_t V = BEST(S, 0);
  int pos = 0;
  for (int t = 1; t <= S - 1; t++) {      /* lexicographically smallest cuts */
    for (int j = pos + 1; j <= L; j++) {
      if (pre[j] - pre[pos] <= V && BEST(S - t, j) <= V) { cuts_out[t - 1] = j; pos = j; break; }
    }
  }
#undef BEST
  free(pre); free(best);
  return V;
}

/* ------------------------------------------------------------------------ */
/* R19: canonical candidate order.                                           */
int orc_combo(int v, int k, int* placement, int* policy) {
  if (v == 1) {
    if (k < 0 || k > 3) return 0;
    *placement = ORC_SEQ; *policy = k; return 1;
  }
  if (k >= 0 && k <= 3) { *placement = ORC_INTERLEAVED; *policy = k; return 1; }
  if (k == 4) { *placement = ORC_WAVE; *policy = ORC_GPIPE; return 1; }
  if (k == 5) { *placement = ORC_WAVE; *policy = ORC_GREEDY; return 1; }
  return 0;
}

static int n_combos(const orc_group* g) {
  int n = 0, a, b;
  for (int k = 0; k < 32; k++)
    if ((g->combo_mask >> k) & 1u) n += orc_combo(g->v, k, &a, &b);
  return n;
}

/* saturating binomial from Pascal's triangle, and the number of integer
 * vectors of length n with L1 norm <= r by recursion over the first digit
 * (value 0, or +-a for a = 1..r): cnt(n, r) = cnt(n-1, r) + 2 sum_a cnt(n-1, r-a). */
#define ORC_RMAX 512
static uint64_t pascal_tab[300][300];
static uint64_t ball_tab[ORC_MAXS + 1][ORC_RMAX];
static pthread_once_t tabs_once = PTHREAD_ONCE_INIT;

static uint64_t sat_add(uint64_t a, uint64_t b) { return (a > UINT64_MAX - b) ? UINT64_MAX : a + b; }

static void tabs_init(void) {
  for (int i = 0; i < 300; i++)
    for (int j = 0; j <= i; j++)
      pascal_tab[i][j] = (j == 0 || j == i) ? 1 : sat_add(pascal_tab[i - 1][j - 1], pascal_tab[i - 1][j]);
  for (int r = 0; r < ORC_RMAX; r++) ball_tab[0][r] = 1;
  for (int n = 1; n <= ORC_MAXS; n++)
    for (int r = 0; r < ORC_RMAX; r++) {
      uint64_t t = ball_tab[n - 1][r];
      for (int a = 1; a <= r; a++) t = sat_add(t, sat_add(ball_tab[n - 1][r - a], ball_tab[n - 1][r - a]));
      ball_tab[n][r] = t;
    }
}

static uint64_t binom(int n, int k) {
  pthread_once(&tabs_once, tabs_init);
  if (k < 0 || n < 0 || k > n) return 0;
  if (n >= 300) return UINT64_MAX;
  return pascal_tab[n][k];
}

static uint64_t ball_count(int n, int r) {
  pthread_once(&tabs_once, tabs_init);
  if (r < 0) return 0;
  if (n == 0) return 1;
  if (r >= ORC_RMAX) return UINT64_MAX;
  return ball_tab[n][r];
}

static uint64_t n_partitions(const orc_problem* pr, const orc_group* g) {
  int S = pr->p * g->v;
  if (g->part_mode == ORC_FULL) return binom(pr->L - 1, S - 1);
  return ball_count(S - 1, g->radius);
}

uint64_t orc_space_size(const orc_problem* pr, const orc_space* sp, int* overflow) {
  uint64_t n = 0;
  *overflow = 0;
  for (int gi = 0; gi < sp->n_groups; gi++) {
    uint64_t pg = n_partitions(pr, &sp->group[gi]);
    uint64_t nc = (uint64_t)n_combos(&sp->group[gi]);
    if (pg == UINT64_MAX || (nc && pg > (UINT64_MAX >> 1) / nc)) { *overflow = 1; return 0; }
    n += pg * nc;
    if (n >= (1ull << 63)) { *overflow = 1; return 0; }
  }
  return n;
}

static void group_seed(const orc_problem* pr, const orc_group* g, int* seed) {
  int S = pr->p * g->v;
  if (g->seed_cuts) { for (int i = 0; i < S - 1; i++) seed[i] = g->seed_cuts[i]; return; }
  int64_t* w = (int64_t*)malloc(sizeof(int64_t) * pr->L);
  for (int l = 0; l < pr->L; l++) w[l] = pr->t_f[l] + pr->t_b[l] + pr->t_w[l];
  orc_seed_minmax(pr->L, w, S, seed);
  free(w);
}

/* recursive generation of one group's partitions in canonical order */
typedef struct {
  const orc_problem* pr;
  orc_plan plan;
  int seed[ORC_MAXS];
  int delta[ORC_MAXS];
  uint64_t* idx;
  orc_cb cb;
  void* user;
} gen_t;

/* FULL: colex order = last cut most significant, each ascending */
static void gen_full(gen_t* g, int i, int hi) {
  if (i == 0) { g->cb((*g->idx)++, &g->plan, g->user); return; }
  for (int c = i; c <= hi; c++) { /* cut i takes values in [i, hi] */
    g->plan.cuts[i] = c;
    gen_full(g, i - 1, c - 1);
  }
}

/* BALL: delta_1 most significant, digit order 0, -1, +1, -2, +2, ... */
static void gen_ball(gen_t* g, int i, int rem) {
  int n = g->plan.S - 1;
  if (i > n) {
    for (int t = 1; t <= n; t++) g->plan.cuts[t] = g->seed[t - 1] + g->delta[t];
    g->cb((*g->idx)++, &g->plan, g->user);
    return;
  }
  g->delta[i] = 0;
  gen_ball(g, i + 1, rem);
  for (int a = 1; a <= rem; a++) {
    g->delta[i] = -a; gen_ball(g, i + 1, rem - a);
    g->delta[i] = +a; gen_ball(g, i + 1, rem - a);
  }
}

void orc_enumerate(const orc_problem* pr, const orc_space* sp, orc_cb cb, void* user) {
  uint64_t idx = 0;
  for (int gi = 0; gi < sp->n_groups; gi++) {
    const orc_group* G = &sp->group[gi];
    gen_t g;
    memset(&g, 0, sizeof(g));
    g.pr = pr; g.idx = &idx; g.cb = cb; g.user = user;
    g.plan.v = G->v; g.plan.S = pr->p * G->v;
    g.plan.cuts[0] = 0; g.plan.cuts[g.plan.S] = pr->L;
    if (G->part_mode == ORC_BALL) group_seed(pr, G, g.seed);
    for (int k = 0; k < 32; k++) {
      if (!((G->combo_mask >> k) & 1u)) continue;
      if (!orc_combo(G->v, k, &g.plan.placement, &g.plan.policy)) continue;
      if (G->part_mode == ORC_FULL) gen_full(&g, g.plan.S - 1, pr->L - 1);
      else gen_ball(&g, 1, G->radius);
    }
  }
}

/* random access: walk the same recursion, skipping whole subtrees by size */
int orc_decode(const orc_problem* pr, const orc_space* sp, uint64_t index, orc_plan* out) {
  uint64_t base = 0;
  for (int gi = 0; gi < sp->n_groups; gi++) {
    const orc_group* G = &sp->group[gi];
    uint64_t P = n_partitions(pr, G);
    uint64_t size = P * (uint64_t)n_combos(G);
    if (index >= base + size) { base += size; continue; }
    uint64_t r = index - base;
    uint64_t crank = r / P, prank = r % P;
    int S = pr->p * G->v, seen = 0;
    memset(out, 0, sizeof(*out));
    out->v = G->v; out->S = S; out->cuts[0] = 0; out->cuts[S] = pr->L;
    for (int k = 0; k < 32; k++) {
      int pl, po;
      if (!((G->combo_mask >> k) & 1u) || !orc_combo(G->v, k, &pl, &po)) continue;
      if ((uint64_t)seen == crank) { out->placement = pl; out->policy = po; break; }
      seen++;
    }
    if (G->part_mode == ORC_FULL) {
      int hi = pr->L - 1;
      for (int i = S - 1; i >= 1; i--) {
        for (int c = i; c <= hi; c++) {
          uint64_t sub = binom(c - 1, i - 1); /* ways to place cuts 1..i-1 below c */
          if (prank < sub) { out->cuts[i] = c; hi = c - 1; break; }
          prank -= sub;
        }
      }
    } else {
      int seed[ORC_MAXS];
      group_seed(pr, G, seed);
      int rem = G->radius, n = S - 1;
      for (int i = 1; i <= n; i++) {
        int dsel = 0;
        uint64_t sub = ball_count(n - i, rem);
        if (prank < sub) dsel = 0;
        else {
          prank -= sub;
          for (int a = 1; a <= rem; a++) {
            sub = ball_count(n - i, rem - a);
            if (prank < sub) { dsel = -a; break; }
            prank -= sub;
            if (prank < sub) { dsel = +a; break; }
            prank -= sub;
          }
        }
        out->cuts[i] = seed[i - 1] + dsel;
        rem -= dsel < 0 ? -dsel : dsel;
      }
    }
    return 0;
  }
  return -1;
}

/* ------------------------------------------------------------------------ */
/* Threaded drivers (plain work splitting; no change to the arithmetic).     */
typedef struct {
  const orc_problem* pr; const orc_space* sp; const uint64_t* idx; uint64_t n;
  int64_t* ms; int64_t* pk; double* bub; uint8_t* stt; double* msf;
  int tid, nth; int err;
} ev_arg;

static void* ev_worker(void* a_) {
  ev_arg* a = (ev_arg*)a_;
  for (uint64_t i = a->tid; i < a->n; i += a->nth) {
    orc_plan pl; orc_result r;
    if (orc_decode(a->pr, a->sp, a->idx[i], &pl) != 0) { a->err = 1; continue; }
    int rc = !a->pr->costs_f64 ? orc_simulate(a->pr, &pl, &r, NULL)
             : a->pr->time_f32 ? orc_simulate_f32(a->pr, &pl, &r, NULL)
                               : orc_simulate_f64(a->pr, &pl, &r, NULL);
    if (rc != 0) a->err = 1;
    if (a->msf) a->msf[i] = r.status == ORC_OK ? r.makespan_f : HUGE_VAL;
    if (a->ms) a->ms[i] = r.makespan;
    if (a->pk) a->pk[i] = r.peak_mem;
    if (a->bub) a->bub[i] = r.bubble;
    if (a->stt) a->stt[i] = (uint8_t)r.status;
  }
  return NULL;
}

int orc_eval_indices(const orc_problem* pr, const orc_space* sp, const uint64_t* idx, uint64_t n,
                     int nthreads, int64_t* makespan, int64_t* peak, double* bubble,
                     uint8_t* status, double* makespan_f) {
  if (nthreads < 1) nthreads = 1;
  pthread_t th[256];
  ev_arg args[256];
  if (nthreads > 256) nthreads = 256;
  for (int t = 0; t < nthreads; t++) {
    ev_arg a = {pr, sp, idx, n, makespan, peak, bubble, status, makespan_f, t, nthreads, 0};
    args[t] = a;
    pthread_create(&th[t], NULL, ev_worker, &args[t]);
  }
  int err = 0;
  for (int t = 0; t < nthreads; t++) { pthread_join(th[t], NULL); err |= args[t].err; }
  return err ? -1 : 0;
}

/* search: one producer runs the recursive enumerator and hands blocks of
 * candidates to worker threads; each worker keeps the lexicographic minimum
 * of (makespan, index) over feasible candidates (Eq. 1-2, R18). */
#define BLK 512
typedef struct { uint64_t idx[BLK]; orc_plan plan[BLK]; int n; } block_t;

typedef struct {
  const orc_problem* pr;
  int prune;
  pthread_mutex_t mu;
  pthread_cond_t cv_full, cv_empty;
  block_t** q; int qcap, qhead, qtail, qcount, done;
  block_t* cur;
  /* shared incumbent */
  int64_t best_ms; uint64_t best_idx; orc_plan best_plan;
  uint64_t n_total, n_invalid, n_sim, n_feas;
  int err;
} srch_t;

/* exact lower bound of the makespan: the busiest device (sum of its compute) */
static int64_t lower_bound(const orc_problem* pr, const orc_plan* pl, int64_t* fixed_peak_over) {
  cand_t c;
  derive(pr, pl, &c);
  int64_t busy[ORC_MAXP] = {0}, stat[ORC_MAXP] = {0}, lb = 0;
  for (int s = 0; s < c.S; s++) {
    busy[c.dev[s]] += (int64_t)pr->m * (c.cF[s] + c.cB[s] + c.cW[s]);
    stat[c.dev[s]] += c.wg[s];
  }
  for (int d = 0; d < pr->p; d++) lb = max64(lb, busy[d]);
  *fixed_peak_over = 0;
  if (c.fused) { /* R16: fused fixed-order peak from the list alone */
    int len = 2 * pr->m * pl->v;
    int* k = (int*)malloc(sizeof(int) * len * 3);
    for (int d = 0; d < pr->p && !*fixed_peak_over; d++) {
      int n = orc_fixed_order(pr, pl, d, k, k + len, k + 2 * len, len);
      int64_t dyn = 0;
      for (int i = 0; i < n; i++) {
        int s = k[len + i];
        if (k[i] == KF) dyn += c.act[s] + c.stash[s]; else dyn -= c.act[s] + c.stash[s];
        if (stat[d] + dyn > pr->cap) { *fixed_peak_over = 1; break; }
      }
    }
    free(k);
  }
  return lb;
}

static void consider(srch_t* S_, uint64_t idx, const orc_plan* pl) {
  if (!cuts_valid(S_->pr, pl)) {
    pthread_mutex_lock(&S_->mu); S_->n_invalid++; pthread_mutex_unlock(&S_->mu);
    return;
  }
  if (S_->prune) {
    int64_t over;
    int64_t lb = lower_bound(S_->pr, pl, &over);
    pthread_mutex_lock(&S_->mu);
    int skip = over || lb > S_->best_ms || (lb == S_->best_ms && idx > S_->best_idx);
    pthread_mutex_unlock(&S_->mu);
    if (skip) return;
  }
  orc_result r;
  int rc = orc_simulate(S_->pr, pl, &r, NULL);
  pthread_mutex_lock(&S_->mu);
  if (rc) S_->err = 1;
  S_->n_sim++;
  if (r.status == ORC_OK) {
    S_->n_feas++;
    if (r.makespan < S_->best_ms || (r.makespan == S_->best_ms && idx < S_->best_idx)) {
      S_->best_ms = r.makespan; S_->best_idx = idx; S_->best_plan = *pl;
    }
  }
  pthread_mutex_unlock(&S_->mu);
}

static void* srch_worker(void* a_) {
  srch_t* S_ = (srch_t*)a_;
  for (;;) {
    pthread_mutex_lock(&S_->mu);
    while (S_->qcount == 0 && !S_->done) pthread_cond_wait(&S_->cv_full, &S_->mu);
    if (S_->qcount == 0 && S_->done) { pthread_mutex_unlock(&S_->mu); return NULL; }
    block_t* b = S_->q[S_->qhead];
    S_->qhead = (S_->qhead + 1) % S_->qcap;
    S_->qcount--;
    pthread_cond_signal(&S_->cv_empty);
    pthread_mutex_unlock(&S_->mu);
    for (int i = 0; i < b->n; i++) consider(S_, b->idx[i], &b->plan[i]);
    free(b);
  }
}

static void push_block(srch_t* S_) {
  pthread_mutex_lock(&S_->mu);
  while (S_->qcount == S_->qcap) pthread_cond_wait(&S_->cv_empty, &S_->mu);
  S_->q[S_->qtail] = S_->cur;
  S_->qtail = (S_->qtail + 1) % S_->qcap;
  S_->qcount++;
  pthread_cond_signal(&S_->cv_full);
  pthread_mutex_unlock(&S_->mu);
  S_->cur = (block_t*)malloc(sizeof(block_t));
  S_->cur->n = 0;
}

static void srch_cb(uint64_t index, const orc_plan* plan, void* user) {
  srch_t* S_ = (srch_t*)user;
  S_->n_total++;
  S_->cur->idx[S_->cur->n] = index;
  S_->cur->plan[S_->cur->n] = *plan;
  if (++S_->cur->n == BLK) push_block(S_);
}

int orc_search(const orc_problem* pr, const orc_space* sp, int prune, int nthreads,
               orc_best* out) {
  srch_t S_;
  memset(&S_, 0, sizeof(S_));
  S_.pr = pr; S_.prune = prune;
  S_.best_ms = INT64_MAX; S_.best_idx = UINT64_MAX;
  pthread_mutex_init(&S_.mu, NULL);
  pthread_cond_init(&S_.cv_full, NULL);
  pthread_cond_init(&S_.cv_empty, NULL);
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  if (prune) {
    /* incumbent from a strided sample of the space; exactness does not depend on it */
    int of;
    uint64_t N = orc_space_size(pr, sp, &of);
    uint64_t stride = N / 4096 + 1;
    for (uint64_t i = 0; i < N; i += stride) {
      orc_plan pl;
      if (orc_decode(pr, sp, i, &pl) == 0) consider(&S_, i, &pl);
    }
    S_.n_sim = S_.n_feas = S_.n_invalid = 0;
  }
  S_.qcap = 4 * nthreads;
  S_.q = (block_t**)malloc(sizeof(block_t*) * S_.qcap);
  S_.cur = (block_t*)malloc(sizeof(block_t));
  S_.cur->n = 0;
  pthread_t th[256];
  for (int t = 0; t < nthreads; t++) pthread_create(&th[t], NULL, srch_worker, &S_);
  orc_enumerate(pr, sp, srch_cb, &S_);
  if (S_.cur->n > 0) push_block(&S_);
  free(S_.cur);
  pthread_mutex_lock(&S_.mu);
  S_.done = 1;
  pthread_cond_broadcast(&S_.cv_full);
  pthread_mutex_unlock(&S_.mu);
  for (int t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
  free(S_.q);
  memset(out, 0, sizeof(*out));
  out->index = S_.best_idx;
  out->makespan = S_.best_ms;
  out->plan = S_.best_plan;
  out->n_total = S_.n_total;
  out->n_invalid = S_.n_invalid;
  out->n_simulated = S_.n_sim;
  out->n_feasible = S_.n_feas;
  return S_.err ? -1 : 0;
}
