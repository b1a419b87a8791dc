/*
 * bnb.c -- CrossPipe CPU ORACLE, part 2: exact optimum by branch and bound.
 *          *** TEST INFRASTRUCTURE ONLY *** (see oracle.h)
 *
 * What it computes: min over all valid split plans with whole blocks (n_sub = 1) of the
 * makespan of the plan under the §3.5 performance model -- the schedule the paper's CO
 * formulation (§4.1) optimises: sets and decision variables :313-320, the
 * four constraint families :322-351 (dependencies with comm delays, one block at a time per
 * stage, memory capacity along the sequence, microbatch order per type), objective :356-360
 * with the DP extension :363.  It is the same optimum as or_enumerate_opt (exhaustive product
 * enumeration), reached by search instead of enumeration so that the paper's 4 x 8 E1 setup
 * (:486, :491) is within reach.
 *
 * Search ("DFS over placements ... B&B with incumbent = greedy + 1, plus
 * resource and path lower bounds"):
 *   node    = a partial schedule: per stage a prefix of its sequence, each block at a fixed start
 *   branch  = append one eligible block x (next F if its input arrived and memory fits; next D if
 *             its gradient arrived; next W if its D is done) to one stage s.  Its start is
 *             max(stage clock, input arrival [, ZeRO-1 AG end], floor), where the floor is the
 *             previous append's start t_last, plus one tick if s is below that append's stage.
 *             Appends in increasing (start, stage) order reproduce exactly the semi-active
 *             schedule of every plan (each plan once, no floor ever binds); other orders give
 *             the same plan delayed, which can only be longer (max-plus monotonicity).  So the
 *             minimum over all leaves is the minimum over plans.
 *   incumbent = the greedy's n_sub = 1 plan (or_greedy, a member of the plan set); a node is cut
 *             when its lower bound reaches the incumbent (only strictly better plans are sought).
 *   bound   = max of (a) the makespan so far and (b) per stage, Jackson's preemptive one-machine
 *             schedule of its remaining blocks with heads
 *             r (earliest starts from the dependency chains, link clocks and the floor) and tails
 *             q (longest dependency path from the block's end to the end of the schedule, DP
 *             allreduce included); the preemptive single-machine optimum of max(C + q) is a
 *             lower bound of any completion.
 *   dominance = a partial schedule's future depends only on its counts per (stage, type) and on
 *             its interface times: makespan so far, each stage's clock (raised to its floor),
 *             link clocks and the arrival times of messages not yet consumed (each raised to the
 *             consumer's clock, below which it cannot act).  If an explored node with the same
 *             counts has every interface time <= this node's, every completion of this node is
 *             matched by the same appends from that node, no later anywhere (monotonicity), so
 *             this node is cut.  Nodes are recorded on entry; a node at the same depth was
 *             finished before a later sibling subtree is entered, and equal vectors keep the
 *             first, so no cut relies on an unexplored node.
 * Result: the optimum (proven when the search finishes within max_nodes; otherwise the best plan
 * found with the root lower bound, a gap).  The returned plan is re-simulated by or_simulate and
 * its makespan reported from there.
 */
#include "oracle.h"
#include <stdlib.h>
#include <string.h>

#define BB_MAXP 8
#define BB_MAXM 16
#define BB_T_F 0
#define BB_T_D 1
#define BB_T_W 2

typedef struct {
  int8_t n[BB_MAXP][3];                    /* blocks done per (stage, type F/D/W) */
  int64_t clk[BB_MAXP], mem[BB_MAXP];
  int64_t endF[BB_MAXP][BB_MAXM], endD[BB_MAXP][BB_MAXM];
  int64_t arrF[BB_MAXP][BB_MAXM];          /* F_j input at stage s (from s-1), once F_j(s-1) ended */
  int64_t arrD[BB_MAXP][BB_MAXM];          /* D_j input at stage s (from s+1), once D_j(s+1) ended */
  int64_t linkF[BB_MAXP], linkB[BB_MAXP];  /* FIFO window clock of link s->s+1 / s->s-1 (App. X1) */
  int64_t t_last; int32_t s_last;
  int64_t M;                               /* makespan so far: max block end, DP tails of finished stages */
  int32_t depth;
  int8_t seq[BB_MAXP][3 * BB_MAXM];
} bb_state;

/* dominance table: count vector -> list of interface-time vectors (Pareto front) */
typedef struct { uint8_t key[BB_MAXP * 3]; int32_t nvec, cap; int32_t* vecs; } bb_bucket;
typedef struct {
  const or_inst* I;
  int p, m, L;
  int64_t qF[BB_MAXP][BB_MAXM], qD[BB_MAXP][BB_MAXM], qW[BB_MAXP][BB_MAXM];
  int64_t ub;
  int8_t best[BB_MAXP][3 * BB_MAXM];
  int64_t nodes, max_nodes;
  int aborted;
  bb_bucket* tab; int64_t tab_cap, tab_used; int vlen_max;
  int64_t stored_words, max_stored_words;
  int32_t flags;                           /* OR_BNB_NO_DOMINANCE, OR_BNB_NO_JPS (test cross-checks) */
} bb_ctx;

static int64_t mx(int64_t a, int64_t b) { return a > b ? a : b; }

static int64_t dur_of(const or_inst* I, int s, int ty) {
  return ty == BB_T_F ? I->t_f[s] : (ty == BB_T_D ? I->t_d[s] : I->t_w[s]);
}

/* tails: the longest dependency path from a block's end to the end of the schedule.  W_j(s) is
 * followed by W_{j+1}(s) and, after the stage's last block, the DP allreduce (:363); D_j(s) by
 * W_j(s), D_{j+1}(s) and, through link s->s-1, D_j(s-1); F_j(s) by F_{j+1}(s) and through the
 * link F_j(s+1), or on the last stage D_j(p-1) (loss turnaround, §3.3).                       */
static void bb_tails(bb_ctx* C) {
  const or_inst* I = C->I;
  const int p = C->p, m = C->m;
  for (int s = 0; s < p; ++s)
    for (int j = m - 1; j >= 0; --j)
      C->qW[s][j] = mx(I->t_dp[s], j + 1 < m ? I->t_w[s] + C->qW[s][j + 1] : 0);
  for (int j = m - 1; j >= 0; --j)
    for (int s = 0; s < p; ++s) {
      int64_t q = mx(I->t_dp[s], I->t_w[s] + C->qW[s][j]);
      if (j + 1 < m) q = mx(q, I->t_d[s] + C->qD[s][j + 1]);
      if (s > 0) q = mx(q, I->bw_b[s - 1] + I->lat_b[s - 1] + I->t_d[s - 1] + C->qD[s - 1][j]);
      C->qD[s][j] = q;
    }
  for (int j = m - 1; j >= 0; --j)
    for (int s = p - 1; s >= 0; --s) {
      int64_t q = I->t_dp[s];
      if (j + 1 < m) q = mx(q, I->t_f[s] + C->qF[s][j + 1]);
      if (s < p - 1) q = mx(q, I->bw_f[s] + I->lat_f[s] + I->t_f[s + 1] + C->qF[s + 1][j]);
      else q = mx(q, I->t_d[s] + C->qD[s][j]);
      C->qF[s][j] = q;
    }
}

static int64_t floor_of(const bb_state* S, int s) { return S->t_last + (s < S->s_last ? 1 : 0); }

/* Jackson's preemptive schedule: min over preemptive one-machine schedules of max(C_x + q_x). */
static int64_t jps(int n, const int64_t* r, const int64_t* d, const int64_t* q) {
  int64_t rem[3 * BB_MAXM];
  int left = 0;
  int64_t t = INT64_MAX, lb = 0;
  for (int i = 0; i < n; ++i) { rem[i] = d[i]; if (d[i] > 0) ++left; if (r[i] < t) t = r[i]; }
  while (left > 0) {
    int pick = -1;
    int64_t next_r = INT64_MAX;
    for (int i = 0; i < n; ++i) {
      if (rem[i] <= 0) continue;
      if (r[i] <= t) { if (pick < 0 || q[i] > q[pick]) pick = i; }
      else if (r[i] < next_r) next_r = r[i];
    }
    if (pick < 0) { t = next_r; continue; }
    int64_t run = rem[pick];
    if (next_r != INT64_MAX && t + run > next_r) run = next_r - t;
    t += run;
    rem[pick] -= run;
    if (rem[pick] == 0) { --left; lb = mx(lb, t + q[pick]); }
  }
  return lb;
}

/* lower bound of every completion of S */
static int64_t bb_bound(const bb_ctx* C, const bb_state* S) {
  const or_inst* I = C->I;
  const int p = C->p, m = C->m;
  int64_t lb = S->M;
  /* heads of the remaining blocks, in dependency order (F: s ascending; D: s descending) */
  int64_t rF[BB_MAXP][BB_MAXM], rD[BB_MAXP][BB_MAXM], rW[BB_MAXP][BB_MAXM];
  int64_t c[BB_MAXP];
  for (int s = 0; s < p; ++s) c[s] = mx(S->clk[s], floor_of(S, s));
  for (int s = 0; s < p; ++s) {
    int64_t prev = c[s];
    for (int j = S->n[s][BB_T_F]; j < m; ++j) {
      int64_t a;
      if (s == 0) a = 0;
      else if (j < S->n[s - 1][BB_T_F]) a = S->arrF[s][j];
      else {
        const int64_t e = rF[s - 1][j] + I->t_f[s - 1];
        a = (I->bw_f[s - 1] > 0 ? mx(e, S->linkF[s - 1]) : e) + I->bw_f[s - 1] + I->lat_f[s - 1];
      }
      if (I->zero1) a = mx(a, I->t_ag[s]);
      rF[s][j] = mx(a, prev);
      prev = rF[s][j] + I->t_f[s];
    }
  }
  for (int s = p - 1; s >= 0; --s) {
    int64_t prev = c[s];
    for (int j = S->n[s][BB_T_D]; j < m; ++j) {
      int64_t a = j < S->n[s][BB_T_F] ? S->endF[s][j] : rF[s][j] + I->t_f[s];
      if (s < p - 1) {
        int64_t g;
        if (j < S->n[s + 1][BB_T_D]) g = S->arrD[s][j];
        else {
          const int64_t e = rD[s + 1][j] + I->t_d[s + 1];
          g = (I->bw_b[s] > 0 ? mx(e, S->linkB[s + 1]) : e) + I->bw_b[s] + I->lat_b[s];
        }
        a = mx(a, g);
      }
      rD[s][j] = mx(a, prev);
      prev = rD[s][j] + I->t_d[s];
    }
  }
  for (int s = 0; s < p; ++s) {
    int64_t prev = c[s];
    for (int j = S->n[s][BB_T_W]; j < m; ++j) {
      const int64_t a = j < S->n[s][BB_T_D] ? S->endD[s][j] : rD[s][j] + I->t_d[s];
      rW[s][j] = mx(a, prev);
      prev = rW[s][j] + I->t_w[s];
    }
  }
  for (int s = 0; s < p; ++s) {
    int64_t r[3 * BB_MAXM], d[3 * BB_MAXM], q[3 * BB_MAXM];
    int n = 0;
    for (int j = S->n[s][BB_T_F]; j < m; ++j) { r[n] = rF[s][j]; d[n] = I->t_f[s]; q[n] = C->qF[s][j]; ++n; }
    for (int j = S->n[s][BB_T_D]; j < m; ++j) { r[n] = rD[s][j]; d[n] = I->t_d[s]; q[n] = C->qD[s][j]; ++n; }
    for (int j = S->n[s][BB_T_W]; j < m; ++j) { r[n] = rW[s][j]; d[n] = I->t_w[s]; q[n] = C->qW[s][j]; ++n; }
    if (!n) continue;
    if (C->flags & OR_BNB_NO_JPS) {            /* weaker bound: per block head + duration + tail */
      for (int i = 0; i < n; ++i) lb = mx(lb, r[i] + d[i] + q[i]);
    } else {
      lb = mx(lb, jps(n, r, d, q));
    }
  }
  return lb;
}

/* ---------------------------------------------------------------- dominance table */
static uint64_t bb_hash(const uint8_t* k, int n) {
  uint64_t h = 1469598103934665603ull;
  for (int i = 0; i < n; ++i) { h ^= k[i]; h *= 1099511628211ull; }
  return h;
}

/* interface vector of S (int32: tiny instances stay far below 2^31 ticks) */
static int bb_vector(const bb_ctx* C, const bb_state* S, int32_t* v) {
  const int p = C->p;
  int n = 0;
  int64_t c[BB_MAXP];
  for (int s = 0; s < p; ++s) c[s] = mx(S->clk[s], floor_of(S, s));
  v[n++] = (int32_t)S->M;
  for (int s = 0; s < p; ++s) v[n++] = (int32_t)c[s];
  for (int s = 0; s + 1 < p; ++s) v[n++] = (int32_t)mx(S->linkF[s], c[s]);
  for (int s = 1; s < p; ++s) v[n++] = (int32_t)mx(S->linkB[s], c[s]);
  for (int s = 1; s < p; ++s)
    for (int j = S->n[s][BB_T_F]; j < S->n[s - 1][BB_T_F]; ++j) v[n++] = (int32_t)mx(S->arrF[s][j], c[s]);
  for (int s = 0; s + 1 < p; ++s)
    for (int j = S->n[s][BB_T_D]; j < S->n[s + 1][BB_T_D]; ++j) v[n++] = (int32_t)mx(S->arrD[s][j], c[s]);
  return n;
}

static int leq(const int32_t* a, const int32_t* b, int n) {
  for (int i = 0; i < n; ++i) if (a[i] > b[i]) return 0;
  return 1;
}

/* returns 1 if S is dominated by a recorded node; else records S (dropping vectors it dominates) */
static int bb_dominated(bb_ctx* C, const bb_state* S) {
  uint8_t key[BB_MAXP * 3];
  memset(key, 0, sizeof(key));
  for (int s = 0; s < C->p; ++s) for (int t = 0; t < 3; ++t) key[3 * s + t] = (uint8_t)S->n[s][t];
  int32_t v[1 + 3 * BB_MAXP + 2 * BB_MAXP * BB_MAXM];
  const int n = bb_vector(C, S, v);
  if (C->tab_used * 2 >= C->tab_cap) {       /* grow (rehash) */
    const int64_t nc = C->tab_cap ? 2 * C->tab_cap : 1 << 16;
    bb_bucket* nt = (bb_bucket*)calloc((size_t)nc, sizeof(bb_bucket));
    for (int64_t i = 0; i < C->tab_cap; ++i) {
      if (!C->tab[i].vecs) continue;
      uint64_t h = bb_hash(C->tab[i].key, sizeof(key)) & (uint64_t)(nc - 1);
      while (nt[h].vecs) h = (h + 1) & (uint64_t)(nc - 1);
      nt[h] = C->tab[i];
    }
    free(C->tab);
    C->tab = nt; C->tab_cap = nc;
  }
  uint64_t h = bb_hash(key, sizeof(key)) & (uint64_t)(C->tab_cap - 1);
  while (C->tab[h].vecs && memcmp(C->tab[h].key, key, sizeof(key))) h = (h + 1) & (uint64_t)(C->tab_cap - 1);
  bb_bucket* b = &C->tab[h];
  if (b->vecs) {
    for (int i = 0; i < b->nvec; ++i) if (leq(b->vecs + (int64_t)i * n, v, n)) return 1;
    int k = 0;                                 /* drop recorded vectors S dominates */
    for (int i = 0; i < b->nvec; ++i)
      if (!leq(v, b->vecs + (int64_t)i * n, n)) {
        if (k != i) memcpy(b->vecs + (int64_t)k * n, b->vecs + (int64_t)i * n, sizeof(int32_t) * n);
        ++k;
      }
    C->stored_words -= (int64_t)(b->nvec - k) * n;
    b->nvec = k;
  }
  if (C->stored_words + n > C->max_stored_words) return 0;   /* table full: keep searching, record nothing */
  if (!b->vecs) { memcpy(b->key, key, sizeof(key)); b->cap = 4; b->vecs = (int32_t*)malloc(sizeof(int32_t) * 4 * n); b->nvec = 0; C->tab_used++; }
  if (b->nvec == b->cap) { b->cap *= 2; b->vecs = (int32_t*)realloc(b->vecs, sizeof(int32_t) * (size_t)b->cap * n); }
  memcpy(b->vecs + (int64_t)b->nvec * n, v, sizeof(int32_t) * n);
  b->nvec++;
  C->stored_words += n;
  return 0;
}

/* ---------------------------------------------------------------- search */
/* start of block (s, ty) appended to S, or -1 if it is not eligible */
static int64_t bb_start(const bb_ctx* C, const bb_state* S, int s, int ty) {
  const or_inst* I = C->I;
  const int m = C->m;
  const int j = S->n[s][ty];
  if (j >= m) return -1;
  int64_t a;
  if (ty == BB_T_F) {
    if (S->mem[s] + I->m_f[s] > I->m_lim[s]) return -1;
    if (s == 0) a = 0;
    else if (j < S->n[s - 1][BB_T_F]) a = S->arrF[s][j];
    else return -1;
    if (I->zero1) a = mx(a, I->t_ag[s]);
  } else if (ty == BB_T_D) {
    if (s == C->p - 1) { if (j >= S->n[s][BB_T_F]) return -1; a = S->endF[s][j]; }
    else if (j < S->n[s + 1][BB_T_D] && j < S->n[s][BB_T_F]) a = S->arrD[s][j];
    else return -1;
  } else {
    if (j >= S->n[s][BB_T_D]) return -1;
    a = S->endD[s][j];
  }
  return mx(mx(S->clk[s], a), floor_of(S, s));
}

static void bb_append(const bb_ctx* C, bb_state* S, int s, int ty, int64_t start) {
  const or_inst* I = C->I;
  const int p = C->p;
  const int j = S->n[s][ty];
  const int64_t end = start + dur_of(I, s, ty);
  S->seq[s][S->n[s][0] + S->n[s][1] + S->n[s][2]] = (int8_t)(ty == BB_T_F ? OR_F : (ty == BB_T_D ? OR_D : OR_W));
  S->n[s][ty]++;
  S->clk[s] = end;
  if (ty == BB_T_F) {
    S->mem[s] += I->m_f[s];
    S->endF[s][j] = end;
    if (s < p - 1) {     /* Alg. 1 :404-407 / §4.2.3: window at or after ready, then latency */
      int64_t ws = end;
      if (I->bw_f[s] > 0) { ws = mx(end, S->linkF[s]); S->linkF[s] = ws + I->bw_f[s]; }
      S->arrF[s + 1][j] = ws + I->bw_f[s] + I->lat_f[s];
    }
  } else if (ty == BB_T_D) {
    S->mem[s] += I->m_d[s];
    S->endD[s][j] = end;
    if (s > 0) {
      int64_t ws = end;
      if (I->bw_b[s - 1] > 0) { ws = mx(end, S->linkB[s]); S->linkB[s] = ws + I->bw_b[s - 1]; }
      S->arrD[s - 1][j] = ws + I->bw_b[s - 1] + I->lat_b[s - 1];
    }
  } else {
    S->mem[s] += I->m_w[s];
  }
  S->M = mx(S->M, end);
  if (S->n[s][BB_T_W] == C->m) S->M = mx(S->M, end + I->t_dp[s]);   /* DP allreduce after the last W */
  S->t_last = start;
  S->s_last = s;
  S->depth++;
}

static void bb_dfs(bb_ctx* C, const bb_state* S) {
  if (C->aborted) return;
  if (++C->nodes > C->max_nodes) { C->aborted = 1; return; }
  if (S->depth == C->L) {
    if (S->M < C->ub) { C->ub = S->M; memcpy(C->best, S->seq, sizeof(C->best)); }
    return;
  }
  if (bb_bound(C, S) >= C->ub) return;
  if (!(C->flags & OR_BNB_NO_DOMINANCE) && bb_dominated(C, S)) return;
  /* children in increasing start, then stage, then type D, F, W (the greedy's steady-state habit) */
  int cs[3 * BB_MAXP], ct[3 * BB_MAXP];
  int64_t cst[3 * BB_MAXP];
  int nc = 0;
  static const int order[3] = {BB_T_D, BB_T_F, BB_T_W};
  for (int s = 0; s < C->p; ++s)
    for (int k = 0; k < 3; ++k) {
      const int64_t st = bb_start(C, S, s, order[k]);
      if (st < 0) continue;
      int i = nc++;
      while (i > 0 && cst[i - 1] > st) { cs[i] = cs[i - 1]; ct[i] = ct[i - 1]; cst[i] = cst[i - 1]; --i; }
      cs[i] = s; ct[i] = order[k]; cst[i] = st;
    }
  for (int i = 0; i < nc; ++i) {
    bb_state T = *S;
    bb_append(C, &T, cs[i], ct[i], cst[i]);
    bb_dfs(C, &T);
    if (C->aborted) return;
  }
}

int32_t or_bnb_opt(const or_inst* I, int64_t max_nodes, int64_t max_table_bytes, int32_t flags, int8_t* best_codes,
                   int32_t* best_len, int32_t maxlen, or_result* best, or_bnb_info* info) {
  const int p = I->p, m = I->m, L = 3 * m;
  memset(info, 0, sizeof(*info));
  if (I->n_sub != 1 || p > BB_MAXP || m > BB_MAXM || L > maxlen || or_validate_instance(I)) return -1;
  bb_ctx* C = (bb_ctx*)calloc(1, sizeof(bb_ctx));
  C->I = I; C->p = p; C->m = m; C->L = L * p;
  C->max_nodes = max_nodes;
  C->max_stored_words = max_table_bytes / 4;
  C->flags = flags;
  bb_tails(C);
  /* incumbent: the greedy's n_sub = 1 plan (Alg. 1), a member of the plan set */
  int8_t* g = (int8_t*)calloc((size_t)p * L, 1);
  int32_t gl[OR_MAXP];
  or_result gr;
  if (or_greedy(I, g, gl, L, &gr, NULL) != 0) { free(g); free(C); return -1; }
  C->ub = gr.makespan;
  for (int s = 0; s < p; ++s) memcpy(C->best[s], g + (int64_t)s * L, (size_t)L);
  info->greedy = gr.makespan;
  bb_state* S = (bb_state*)calloc(1, sizeof(bb_state));
  S->s_last = 0;
  info->root_bound = bb_bound(C, S);
  if (info->root_bound < C->ub) bb_dfs(C, S);
  info->nodes = C->nodes;
  info->proven = !C->aborted;
  info->table_bytes = C->stored_words * 4;
  /* the plan, re-simulated by the §3.5 model */
  memset(best_codes, 0, (size_t)p * maxlen);
  for (int s = 0; s < p; ++s) { memcpy(best_codes + (int64_t)s * maxlen, C->best[s], (size_t)L); best_len[s] = L; }
  int32_t st = or_simulate(I, best_codes, best_len, maxlen, best, NULL);
  info->bound = info->proven ? best->makespan : info->root_bound;
  for (int64_t i = 0; i < C->tab_cap; ++i) free(C->tab[i].vecs);
  free(C->tab); free(S); free(g); free(C);
  return st ? -1 : info->proven;
}
