/*
 * oracle.c -- CrossPipe CPU ORACLE.  *** TEST INFRASTRUCTURE ONLY ***  (see oracle.h)
 *
 * Deliberately plain: explicit dependency DAG + Kahn topological order for the
 * performance model, explicit per-stage schedulable lists for Algorithm 1, an
 * interval list for the bandwidth-occupancy model.  int64 ticks throughout.
 * No blocking, fusion or reordering beyond what the cited passages state.
 */
#include "oracle.h"
#include <stdlib.h>
#include <string.h>
#include <math.h>

static int64_t max64(int64_t a, int64_t b) { return a > b ? a : b; }

/* ------------------------------------------------------------------------- */
/* §4.2.3: "determines the earliest available transmission
 * window of length T_bw, starting at or after T_ready, and returns its end time".
 * Range-based: sorted disjoint reserved intervals [s,e), first fit.
 * Reading Q4: a zero-width window does not occupy the link (returns t_ready).    */
void or_link_init(or_link* L) { L->s = L->e = NULL; L->n = L->cap = 0; }
void or_link_free(or_link* L) { free(L->s); free(L->e); or_link_init(L); }

int64_t or_reserve_window(or_link* L, int64_t t_ready, int64_t width) {
  if (width <= 0) return t_ready;
  int64_t t = t_ready;
  int32_t i, pos = L->n;
  for (i = 0; i < L->n; ++i) {
    if (L->e[i] <= t) continue;             /* interval entirely before candidate start */
    if (L->s[i] >= t + width) { pos = i; break; } /* gap [t, s_i) is long enough */
    t = L->e[i];                            /* overlap: move past this interval */
  }
  if (i == L->n) pos = L->n;
  if (L->n == L->cap) {
    L->cap = L->cap ? 2 * L->cap : 16;
    L->s = (int64_t*)realloc(L->s, sizeof(int64_t) * L->cap);
    L->e = (int64_t*)realloc(L->e, sizeof(int64_t) * L->cap);
  }
  memmove(L->s + pos + 1, L->s + pos, sizeof(int64_t) * (L->n - pos));
  memmove(L->e + pos + 1, L->e + pos, sizeof(int64_t) * (L->n - pos));
  L->s[pos] = t; L->e[pos] = t + width; L->n++;
  return t + width;
}

/* ------------------------------------------------------------------------- */
/* Instance invariants: SPEC.md:46-50 (durations > 0, delays >= 0, m_f > 0,
 * m_d,m_w <= 0, sum 0, m_lim >= m_f) and Q12 (every block >= n_sub ticks, so each of
 * its n_sub sub-blocks (Alg. 1 :398-403) lasts at least one tick).     */
int32_t or_validate_instance(const or_inst* I) {
  if (I->p < 1 || I->p > OR_MAXP || I->m < 1 || I->n_sub < 1) return OR_ST_BAD_INSTANCE;
  for (int s = 0; s < I->p; ++s) {
    if (I->t_f[s] <= 0 || I->t_d[s] <= 0 || I->t_w[s] <= 0) return OR_ST_BAD_INSTANCE;
    if (I->t_f[s] < I->n_sub || I->t_d[s] < I->n_sub || I->t_w[s] < I->n_sub) return OR_ST_BAD_INSTANCE;
    if (I->m_f[s] <= 0 || I->m_d[s] > 0 || I->m_w[s] > 0) return OR_ST_BAD_INSTANCE;
    if (I->m_f[s] + I->m_d[s] + I->m_w[s] != 0) return OR_ST_BAD_INSTANCE;
    if (I->m_lim[s] < I->m_f[s]) return OR_ST_BAD_INSTANCE;
    if (I->t_dp[s] < 0 || I->t_ag[s] < 0) return OR_ST_BAD_INSTANCE;
    if (s < I->p - 1 && (I->lat_f[s] < 0 || I->bw_f[s] < 0 || I->lat_b[s] < 0 || I->bw_b[s] < 0))
      return OR_ST_BAD_INSTANCE;
  }
  return 0;
}

/* ------------------------------------------------------------------------- */
/* Q29 static plan check (SPEC.md:268-276 validate_schedule):
 * per stage: #F == m; #D + #B == m; a stage is all-combined (B) or all-split (D/W);
 * #W == n_sub * #D; and no prefix holds more W entries than n_sub * (D entries so far). */
int32_t or_check_plan(const or_inst* I, const int8_t* codes, const int32_t* len, int32_t maxlen) {
  for (int s = 0; s < I->p; ++s) {
    if (len[s] < 0 || len[s] > maxlen) return OR_ST_BAD_PLAN;
    int64_t nF = 0, nB = 0, nD = 0, nW = 0;
    for (int k = 0; k < len[s]; ++k) {
      int c = codes[(int64_t)s * maxlen + k];
      if (c == OR_F) nF++;
      else if (c == OR_B) nB++;
      else if (c == OR_D) nD++;
      else if (c == OR_W) { nW++; if (nW > (int64_t)I->n_sub * nD) return OR_ST_BAD_PLAN; }
      else return OR_ST_BAD_PLAN;
    }
    if (nF != I->m || nB + nD != I->m) return OR_ST_BAD_PLAN;
    if (nB > 0 && (nD > 0 || nW > 0)) return OR_ST_BAD_PLAN;
    if (nW != (int64_t)I->n_sub * nD) return OR_ST_BAD_PLAN;
  }
  return 0;
}

/* Q12: integer sub-block k of a block of duration T split into n parts. */
static int64_t sub_dur(int64_t T, int32_t n, int32_t k) { return T / n + (k < (int32_t)(T % n) ? 1 : 0); }

/* ------------------------------------------------------------------------- */
/* §3.5 performance model: "The start time of each block is determined
 * by the maximum of two values: (1) the completion time of the preceding block on the
 * same stage, and (2) the completion time of the dependent block plus the communication
 * delay. The communication delay consists of a fixed latency component and a
 * bandwidth-related component, which depends on both link bandwidth and current
 * occupancy."  Dependency graph per §3.3 (:232-236): true dependencies (UD data flow)
 * + schedule dependencies (plan order), processed in topological (Kahn) order.
 * Comm: E_bw = BW_model(end, link, T_bw); avail = E_bw + T_lat (Alg. 1 :404-407).
 * DP overlap (:363, fig:wave_dependency :282): AR after the last W (or B) of the stage;
 * ZeRO-1 AG precedes the first F.  Runtime: App. A (:808), origin t = 0.            */
enum { EK_SCHED = 0, EK_LOCAL = 1, EK_LINK_F = 2, EK_LINK_B = 3 };
typedef struct { int32_t to, kind, link; } or_edge;

int32_t or_simulate(const or_inst* I, const int8_t* codes, const int32_t* len, int32_t maxlen,
                    or_result* R, int64_t* t_start) {
  const int p = I->p, m = I->m, ns = I->n_sub;
  memset(R, 0, sizeof(*R));
  R->makespan = -1; R->peak_mem = -1;
  int32_t st = or_validate_instance(I);
  if (st) { R->status = st; return st; }
  st = or_check_plan(I, codes, len, maxlen);
  if (st) { R->status = st; return st; }

  /* nodes: one per plan entry, plus per stage an AG node (ZeRO-1) and an AR node (DP). */
  int64_t off[OR_MAXP + 1]; off[0] = 0;
  for (int s = 0; s < p; ++s) off[s + 1] = off[s] + len[s];
  const int64_t NC = off[p];
  const int64_t N = NC + 2 * p;              /* AG(s) = NC + s, AR(s) = NC + p + s */
  int32_t* n_stage = (int32_t*)calloc(N, sizeof(int32_t));
  int32_t* n_type  = (int32_t*)calloc(N, sizeof(int32_t));
  int32_t* n_mb    = (int32_t*)calloc(N, sizeof(int32_t));
  int32_t* n_sub   = (int32_t*)calloc(N, sizeof(int32_t));
  int64_t* dur     = (int64_t*)calloc(N, sizeof(int64_t));
  int64_t* ready   = (int64_t*)calloc(N, sizeof(int64_t));
  int64_t* start   = (int64_t*)calloc(N, sizeof(int64_t));
  int64_t* end     = (int64_t*)calloc(N, sizeof(int64_t));
  int32_t* indeg   = (int32_t*)calloc(N, sizeof(int32_t));
  int32_t* ecount  = (int32_t*)calloc(N, sizeof(int32_t));
  or_edge** out    = (or_edge**)calloc(N, sizeof(or_edge*));
  int32_t* ecap    = (int32_t*)calloc(N, sizeof(int32_t));
  int64_t* idxF = (int64_t*)malloc(sizeof(int64_t) * p * m);
  int64_t* idxD = (int64_t*)malloc(sizeof(int64_t) * p * m);   /* D or B */
  int64_t* idxLastW = (int64_t*)malloc(sizeof(int64_t) * p * m);
  int64_t* wlist = (int64_t*)malloc(sizeof(int64_t) * (NC + 1)); /* W entries grouped by (s, mb) */
  int64_t* wfirst = (int64_t*)malloc(sizeof(int64_t) * p * m);
  int64_t* wcnt = (int64_t*)calloc((size_t)p * m, sizeof(int64_t));
  int64_t* queue = (int64_t*)malloc(sizeof(int64_t) * N);
  or_link* linkF = (or_link*)malloc(sizeof(or_link) * p);
  or_link* linkB = (or_link*)malloc(sizeof(or_link) * p);
  for (int s = 0; s < p; ++s) { or_link_init(&linkF[s]); or_link_init(&linkB[s]); }

#define ADD_EDGE(u, v, k, l) do { \
    if (ecount[u] == ecap[u]) { ecap[u] = ecap[u] ? 2 * ecap[u] : 4; \
      out[u] = (or_edge*)realloc(out[u], sizeof(or_edge) * ecap[u]); } \
    out[u][ecount[u]].to = (int32_t)(v); out[u][ecount[u]].kind = (k); out[u][ecount[u]].link = (l); \
    ecount[u]++; indeg[v]++; } while (0)

  /* label nodes: microbatch index from per-type counters (§4.1 :346-351, microbatch order) */
  for (int s = 0; s < p; ++s) {
    int32_t cF = 0, cD = 0, cW = 0;
    for (int k = 0; k < len[s]; ++k) {
      int64_t u = off[s] + k;
      int c = codes[(int64_t)s * maxlen + k];
      n_stage[u] = s; n_type[u] = c;
      if (c == OR_F) { n_mb[u] = cF; dur[u] = I->t_f[s]; idxF[s * m + cF] = u; cF++; }
      else if (c == OR_B) { n_mb[u] = cD; dur[u] = I->t_d[s] + I->t_w[s]; idxD[s * m + cD] = u; cD++; }
      else if (c == OR_D) { n_mb[u] = cD; dur[u] = I->t_d[s]; idxD[s * m + cD] = u; cD++; }
      else { n_mb[u] = cW / ns; n_sub[u] = cW % ns; dur[u] = sub_dur(I->t_w[s], ns, cW % ns); cW++; }
    }
  }
  /* W sub-block lists per (s, mb) */
  {
    int64_t w = 0;
    for (int s = 0; s < p; ++s)
      for (int j = 0; j < m; ++j) wfirst[s * m + j] = -1;
    for (int s = 0; s < p; ++s) {
      for (int k = 0; k < len[s]; ++k) {
        int64_t u = off[s] + k;
        if (n_type[u] != OR_W) continue;
        int64_t key = (int64_t)s * m + n_mb[u];
        if (wfirst[key] < 0) wfirst[key] = w;
        wlist[w++] = u; wcnt[key]++;
        if (n_sub[u] == ns - 1) idxLastW[key] = u;
      }
    }
  }
  for (int64_t s = 0; s < p; ++s) {
    n_stage[NC + s] = (int32_t)s; n_type[NC + s] = -1; dur[NC + s] = I->zero1 ? I->t_ag[s] : 0;
    n_stage[NC + p + s] = (int32_t)s; n_type[NC + p + s] = -2; dur[NC + p + s] = I->t_dp[s];
  }
  /* schedule dependencies: consecutive entries on a stage (§3.3 :236) */
  for (int s = 0; s < p; ++s)
    for (int k = 0; k + 1 < len[s]; ++k) ADD_EDGE(off[s] + k, off[s] + k + 1, EK_SCHED, -1);
  /* true dependencies, UD pattern (§3.3 :234, fig:pptravesal) */
  for (int s = 0; s < p; ++s) {
    for (int j = 0; j < m; ++j) {
      int64_t f = idxF[s * m + j], d = idxD[s * m + j];
      if (s < p - 1) ADD_EDGE(f, idxF[(s + 1) * m + j], EK_LINK_F, s);      /* activation s -> s+1 */
      else ADD_EDGE(f, d, EK_LOCAL, -1);                                   /* loss: F -> D on last stage */
      if (s > 0) ADD_EDGE(d, idxD[(s - 1) * m + j], EK_LINK_B, s - 1);     /* gradient s -> s-1 */
      if (wfirst[s * m + j] >= 0)
        for (int64_t q = 0; q < wcnt[s * m + j]; ++q)
          ADD_EDGE(d, wlist[wfirst[s * m + j] + q], EK_LOCAL, -1);          /* W depends on D */
    }
    /* ZeRO-1 allgather precedes the first F of the stage (:363) */
    ADD_EDGE(NC + s, idxF[s * m + 0], EK_LOCAL, -1);
    /* DP allreduce after the W (or B) of the final microbatch (:363) */
    int64_t last = (wfirst[s * m + (m - 1)] >= 0) ? idxLastW[s * m + (m - 1)] : idxD[s * m + (m - 1)];
    ADD_EDGE(last, NC + p + s, EK_LOCAL, -1);
  }
  /* Kahn topological order; each node starts at the max over its incoming edges. */
  int64_t qh = 0, qt = 0, done = 0;
  for (int64_t u = 0; u < N; ++u) if (indeg[u] == 0) queue[qt++] = u;
  while (qh < qt) {
    int64_t u = queue[qh++];
    start[u] = ready[u];
    end[u] = start[u] + dur[u];
    done++;
    for (int32_t e = 0; e < ecount[u]; ++e) {
      or_edge E = out[u][e];
      int64_t c;
      if (E.kind == EK_LINK_F)      c = or_reserve_window(&linkF[E.link], end[u], I->bw_f[E.link]) + I->lat_f[E.link];
      else if (E.kind == EK_LINK_B) c = or_reserve_window(&linkB[E.link], end[u], I->bw_b[E.link]) + I->lat_b[E.link];
      else                          c = end[u];
      ready[E.to] = max64(ready[E.to], c);
      if (--indeg[E.to] == 0) queue[qt++] = E.to;
    }
  }
  if (done < N) {
    R->status = OR_ST_DEADLOCK;
  } else {
    int64_t mk = 0, pk = 0;
    for (int s = 0; s < p; ++s) {
      /* memory: net change applied when a block completes (§4.1 Inputs :307);
       * W releases at its last sub-block (Q8). Running sum in stage order. */
      int64_t mem = 0, peak = 0, busy = 0;
      for (int k = 0; k < len[s]; ++k) {
        int64_t u = off[s] + k;
        int c = n_type[u];
        if (c == OR_F) mem += I->m_f[s];
        else if (c == OR_D) mem += I->m_d[s];
        else if (c == OR_B) mem += I->m_d[s] + I->m_w[s];
        else if (n_sub[u] == ns - 1) mem += I->m_w[s];
        peak = max64(peak, mem);
        busy += dur[u];
        if (t_start) t_start[(int64_t)s * maxlen + k] = start[u];
      }
      R->first_start[s] = start[off[s]];
      R->last_end[s] = end[off[s] + len[s] - 1];
      R->busy[s] = busy;
      R->peak[s] = peak;
      if (peak > I->m_lim[s]) R->status |= OR_ST_MEM_EXCEEDED;
      pk = max64(pk, peak);
    }
    for (int64_t u = 0; u < N; ++u) mk = max64(mk, end[u]);
    R->makespan = mk;
    R->peak_mem = pk;
  }
  for (int s = 0; s < p; ++s) { or_link_free(&linkF[s]); or_link_free(&linkB[s]); }
  for (int64_t u = 0; u < N; ++u) free(out[u]);
  free(n_stage); free(n_type); free(n_mb); free(n_sub); free(dur); free(ready); free(start); free(end);
  free(indeg); free(ecount); free(out); free(ecap); free(idxF); free(idxD); free(idxLastW);
  free(wlist); free(wfirst); free(wcnt); free(queue); free(linkF); free(linkB);
#undef ADD_EDGE
  return R->status;
}

/* ------------------------------------------------------------------------- */
/* Wave pattern (fig:pptravesal :226-234; SPEC patterns module; reading Q32).  Every stage holds
 * two model chunks.  Per microbatch j:
 *   F(0,s) -> F(0,s+1) over link s->s+1;  F(0,p-1) -> F(1,p-1) on the stage (turn-around);
 *   F(1,s) -> F(1,s-1) over link s->s-1;  F(1,0) -> D(1,0) on the stage (loss);
 *   D(1,s) -> D(1,s+1) over link s->s+1;  D(1,p-1) -> D(0,p-1) on the stage (turn-around);
 *   D(0,s) -> D(0,s-1) over link s->s-1;  D(c,s) -> W(c,s) sub-blocks.
 * Link s->s+1 carries F(0) and D(1) messages of stage s, link s->s-1 carries F(1) and D(0)
 * messages of stage s: one producer each, reserved in its execution order (App. X1 holds).
 * Costs and memory deltas of a chunk are the stage's per-block values; ZeRO-1 AG precedes the
 * stage's first F; DP AR follows the stage's last block (the final W or B of one of its chunks). */
#define WV_CODE(x) ((x) & 3)
#define WV_CHUNK(x) (((x) >> 2) & 1)
int32_t or_check_plan_wave(const or_inst* I, const int8_t* codes, const int32_t* len, int32_t maxlen) {
  for (int s = 0; s < I->p; ++s) {
    if (len[s] < 0 || len[s] > maxlen) return OR_ST_BAD_PLAN;
    int64_t nF[2] = {0, 0}, nB[2] = {0, 0}, nD[2] = {0, 0}, nW[2] = {0, 0};
    for (int k = 0; k < len[s]; ++k) {
      int x = codes[(int64_t)s * maxlen + k];
      if (x & ~7) return OR_ST_BAD_PLAN;
      int c = WV_CODE(x), ch = WV_CHUNK(x);
      if (c == OR_F) nF[ch]++;
      else if (c == OR_B) nB[ch]++;
      else if (c == OR_D) nD[ch]++;
      else { nW[ch]++; if (nW[ch] > (int64_t)I->n_sub * nD[ch]) return OR_ST_BAD_PLAN; }
    }
    for (int ch = 0; ch < 2; ++ch) {
      if (nF[ch] != I->m || nB[ch] + nD[ch] != I->m) return OR_ST_BAD_PLAN;
      if (nW[ch] != (int64_t)I->n_sub * nD[ch]) return OR_ST_BAD_PLAN;
    }
    if ((nB[0] + nB[1]) > 0 && (nD[0] + nD[1] + nW[0] + nW[1]) > 0) return OR_ST_BAD_PLAN;
  }
  return 0;
}

int32_t or_simulate_wave(const or_inst* I, const int8_t* codes, const int32_t* len, int32_t maxlen,
                         or_result* R, int64_t* t_start) {
  const int p = I->p, m = I->m, ns = I->n_sub;
  memset(R, 0, sizeof(*R));
  R->makespan = -1; R->peak_mem = -1;
  int32_t st = or_validate_instance(I);
  if (st) { R->status = st; return st; }
  st = or_check_plan_wave(I, codes, len, maxlen);
  if (st) { R->status = st; return st; }
  int64_t off[OR_MAXP + 1]; off[0] = 0;
  for (int s = 0; s < p; ++s) off[s + 1] = off[s] + len[s];
  const int64_t NC = off[p];
  const int64_t N = NC + 2 * p;              /* AG(s) = NC + s, AR(s) = NC + p + s */
  int32_t* n_type  = (int32_t*)calloc(N, sizeof(int32_t));
  int32_t* n_sub   = (int32_t*)calloc(N, sizeof(int32_t));
  int64_t* dur     = (int64_t*)calloc(N, sizeof(int64_t));
  int64_t* ready   = (int64_t*)calloc(N, sizeof(int64_t));
  int64_t* start   = (int64_t*)calloc(N, sizeof(int64_t));
  int64_t* end     = (int64_t*)calloc(N, sizeof(int64_t));
  int32_t* indeg   = (int32_t*)calloc(N, sizeof(int32_t));
  int32_t* ecount  = (int32_t*)calloc(N, sizeof(int32_t));
  or_edge** out    = (or_edge**)calloc(N, sizeof(or_edge*));
  int32_t* ecap    = (int32_t*)calloc(N, sizeof(int32_t));
  /* [chunk][stage][mb] node index of F, of D (or B); W sub-blocks listed per (chunk, stage, mb) */
  const int64_t PM = (int64_t)p * m;
  int64_t* idxF = (int64_t*)malloc(sizeof(int64_t) * 2 * PM);
  int64_t* idxD = (int64_t*)malloc(sizeof(int64_t) * 2 * PM);
  int64_t* wkey = (int64_t*)malloc(sizeof(int64_t) * (NC + 1));  /* W entry -> (chunk, stage, mb) key */
  int64_t* queue = (int64_t*)malloc(sizeof(int64_t) * N);
  or_link* linkR = (or_link*)malloc(sizeof(or_link) * p);   /* s -> s+1 */
  or_link* linkL = (or_link*)malloc(sizeof(or_link) * p);   /* s -> s-1 (index s-1, as bw_b/lat_b) */
  for (int s = 0; s < p; ++s) { or_link_init(&linkR[s]); or_link_init(&linkL[s]); }
#define ADD_EDGE(u, v, k, l) do { \
    if (ecount[u] == ecap[u]) { ecap[u] = ecap[u] ? 2 * ecap[u] : 4; \
      out[u] = (or_edge*)realloc(out[u], sizeof(or_edge) * ecap[u]); } \
    out[u][ecount[u]].to = (int32_t)(v); out[u][ecount[u]].kind = (k); out[u][ecount[u]].link = (l); \
    ecount[u]++; indeg[v]++; } while (0)
#define KEY(ch, s, j) ((int64_t)(ch) * PM + (int64_t)(s) * m + (j))
  {
    for (int s = 0; s < p; ++s) {
      int32_t cF[2] = {0, 0}, cD[2] = {0, 0}, cW[2] = {0, 0};
      for (int k = 0; k < len[s]; ++k) {
        int64_t u = off[s] + k;
        int x = codes[(int64_t)s * maxlen + k], c = WV_CODE(x), ch = WV_CHUNK(x);
        n_type[u] = x;
        if (c == OR_F) { dur[u] = I->t_f[s]; idxF[KEY(ch, s, cF[ch])] = u; cF[ch]++; }
        else if (c == OR_B) { dur[u] = I->t_d[s] + I->t_w[s]; idxD[KEY(ch, s, cD[ch])] = u; cD[ch]++; }
        else if (c == OR_D) { dur[u] = I->t_d[s]; idxD[KEY(ch, s, cD[ch])] = u; cD[ch]++; }
        else {
          int32_t j = cW[ch] / ns, q = cW[ch] % ns;
          n_sub[u] = q; dur[u] = sub_dur(I->t_w[s], ns, q); cW[ch]++;
          wkey[u] = KEY(ch, s, j);
        }
      }
    }
  }
  for (int64_t s = 0; s < p; ++s) {
    n_type[NC + s] = -1; dur[NC + s] = I->zero1 ? I->t_ag[s] : 0;
    n_type[NC + p + s] = -2; dur[NC + p + s] = I->t_dp[s];
  }
  for (int s = 0; s < p; ++s)                                   /* schedule dependencies */
    for (int k = 0; k + 1 < len[s]; ++k) ADD_EDGE(off[s] + k, off[s] + k + 1, EK_SCHED, -1);
  for (int s = 0; s < p; ++s) {
    for (int j = 0; j < m; ++j) {
      const int64_t f0 = idxF[KEY(0, s, j)], f1 = idxF[KEY(1, s, j)];
      const int64_t d0 = idxD[KEY(0, s, j)], d1 = idxD[KEY(1, s, j)];
      if (s < p - 1) ADD_EDGE(f0, idxF[KEY(0, s + 1, j)], EK_LINK_F, s);   /* chunk 0 forward */
      else ADD_EDGE(f0, f1, EK_LOCAL, -1);                              /* turn-around */
      if (s > 0) ADD_EDGE(f1, idxF[KEY(1, s - 1, j)], EK_LINK_B, s - 1); /* chunk 1 forward */
      else ADD_EDGE(f1, d1, EK_LOCAL, -1);                              /* loss */
      if (s < p - 1) ADD_EDGE(d1, idxD[KEY(1, s + 1, j)], EK_LINK_F, s); /* chunk 1 backward */
      else ADD_EDGE(d1, d0, EK_LOCAL, -1);                              /* turn-around */
      if (s > 0) ADD_EDGE(d0, idxD[KEY(0, s - 1, j)], EK_LINK_B, s - 1); /* chunk 0 backward */
    }
    for (int k = 0; k < len[s]; ++k)                                      /* W sub-block after its D */
      if (WV_CODE(n_type[off[s] + k]) == OR_W) ADD_EDGE(idxD[wkey[off[s] + k]], off[s] + k, EK_LOCAL, -1);
    ADD_EDGE(NC + s, idxF[KEY(0, s, 0)], EK_LOCAL, -1);        /* ZeRO-1 AG before chunk 0's first F */
    ADD_EDGE(NC + s, idxF[KEY(1, s, 0)], EK_LOCAL, -1);        /* ... and chunk 1's */
    ADD_EDGE(off[s] + len[s] - 1, NC + p + s, EK_LOCAL, -1);    /* DP AR after the stage's last block */
  }
  int64_t qh = 0, qt = 0, done = 0;
  for (int64_t u = 0; u < N; ++u) if (indeg[u] == 0) queue[qt++] = u;
  while (qh < qt) {
    int64_t u = queue[qh++];
    start[u] = ready[u];
    end[u] = start[u] + dur[u];
    done++;
    for (int32_t e = 0; e < ecount[u]; ++e) {
      or_edge E = out[u][e];
      int64_t c;
      if (E.kind == EK_LINK_F)      c = or_reserve_window(&linkR[E.link], end[u], I->bw_f[E.link]) + I->lat_f[E.link];
      else if (E.kind == EK_LINK_B) c = or_reserve_window(&linkL[E.link], end[u], I->bw_b[E.link]) + I->lat_b[E.link];
      else                          c = end[u];
      ready[E.to] = max64(ready[E.to], c);
      if (--indeg[E.to] == 0) queue[qt++] = E.to;
    }
  }
  if (done < N) {
    R->status = OR_ST_DEADLOCK;
  } else {
    int64_t mk = 0, pk = 0;
    for (int s = 0; s < p; ++s) {
      int64_t mem = 0, peak = 0, busy = 0;
      for (int k = 0; k < len[s]; ++k) {
        int64_t u = off[s] + k;
        int c = WV_CODE(n_type[u]);
        if (c == OR_F) mem += I->m_f[s];
        else if (c == OR_D) mem += I->m_d[s];
        else if (c == OR_B) mem += I->m_d[s] + I->m_w[s];
        else if (n_sub[u] == ns - 1) mem += I->m_w[s];
        peak = max64(peak, mem);
        busy += dur[u];
        if (t_start) t_start[(int64_t)s * maxlen + k] = start[u];
      }
      R->first_start[s] = start[off[s]];
      R->last_end[s] = end[off[s] + len[s] - 1];
      R->busy[s] = busy;
      R->peak[s] = peak;
      if (peak > I->m_lim[s]) R->status |= OR_ST_MEM_EXCEEDED;
      pk = max64(pk, peak);
    }
    for (int64_t u = 0; u < N; ++u) mk = max64(mk, end[u]);
    R->makespan = mk;
    R->peak_mem = pk;
  }
  for (int s = 0; s < p; ++s) { or_link_free(&linkR[s]); or_link_free(&linkL[s]); }
  for (int64_t u = 0; u < N; ++u) free(out[u]);
  free(n_type); free(n_sub); free(dur); free(ready); free(start); free(end); free(indeg); free(ecount);
  free(out); free(ecap); free(idxF); free(idxD); free(wkey); free(queue);
  free(linkR); free(linkL);
#undef KEY
#undef ADD_EDGE
  return R->status;
}

/* Loop pattern (fig:pptravesal :226-234; SPEC patterns module "Loop"; reading Q33), 2 chunks.
 * Per microbatch j:  F(0,s) -> F(0,s+1);  F(0,p-1) -> F(1,0) over the wrap link p-1 -> 0;
 *   F(1,s) -> F(1,s+1);  F(1,p-1) -> D(1,p-1) (loss);  D(1,s) -> D(1,s-1);
 *   D(1,0) -> D(0,p-1) over the wrap link 0 -> p-1;  D(0,s) -> D(0,s-1);  D(c,s) -> W(c,s).
 * Link s -> s+1 carries F(0), F(1) of stage s; link s+1 -> s carries D(0), D(1) of stage s+1; the
 * wrap links carry F(0) of stage p-1 and D(1) of stage 0: one producer per directed link (the
 * paper's alpha/beta are per device pair, :381), so App. X1's FIFO = first-fit still holds. */
int32_t or_simulate_loop(const or_inst* I, const int8_t* codes, const int32_t* len, int32_t maxlen,
                         or_result* R, int64_t* t_start) {
  const int p = I->p, m = I->m, ns = I->n_sub;
  memset(R, 0, sizeof(*R));
  R->makespan = -1; R->peak_mem = -1;
  int32_t st = or_validate_instance(I);
  if (st) { R->status = st; return st; }
  if (I->lat_f[p - 1] < 0 || I->bw_f[p - 1] < 0 || I->lat_b[p - 1] < 0 || I->bw_b[p - 1] < 0) {
    R->status = OR_ST_BAD_INSTANCE;                           /* wrap link delays */
    return R->status;
  }
  st = or_check_plan_wave(I, codes, len, maxlen);
  if (st) { R->status = st; return st; }
  int64_t off[OR_MAXP + 1]; off[0] = 0;
  for (int s = 0; s < p; ++s) off[s + 1] = off[s] + len[s];
  const int64_t NC = off[p];
  const int64_t N = NC + 2 * p;              /* AG(s) = NC + s, AR(s) = NC + p + s */
  int32_t* n_type  = (int32_t*)calloc(N, sizeof(int32_t));
  int32_t* n_sub   = (int32_t*)calloc(N, sizeof(int32_t));
  int64_t* dur     = (int64_t*)calloc(N, sizeof(int64_t));
  int64_t* ready   = (int64_t*)calloc(N, sizeof(int64_t));
  int64_t* start   = (int64_t*)calloc(N, sizeof(int64_t));
  int64_t* end     = (int64_t*)calloc(N, sizeof(int64_t));
  int32_t* indeg   = (int32_t*)calloc(N, sizeof(int32_t));
  int32_t* ecount  = (int32_t*)calloc(N, sizeof(int32_t));
  or_edge** out    = (or_edge**)calloc(N, sizeof(or_edge*));
  int32_t* ecap    = (int32_t*)calloc(N, sizeof(int32_t));
  /* [chunk][stage][mb] node index of F, of D (or B); W sub-blocks listed per (chunk, stage, mb) */
  const int64_t PM = (int64_t)p * m;
  int64_t* idxF = (int64_t*)malloc(sizeof(int64_t) * 2 * PM);
  int64_t* idxD = (int64_t*)malloc(sizeof(int64_t) * 2 * PM);
  int64_t* wkey = (int64_t*)malloc(sizeof(int64_t) * (NC + 1));  /* W entry -> (chunk, stage, mb) key */
  int64_t* queue = (int64_t*)malloc(sizeof(int64_t) * N);
  /* boundary s = link s -> (s+1) mod p (*_f) and its reverse (*_b); index p-1 is the wrap link */
  or_link* linkR = (or_link*)malloc(sizeof(or_link) * p);
  or_link* linkL = (or_link*)malloc(sizeof(or_link) * p);
  for (int s = 0; s < p; ++s) { or_link_init(&linkR[s]); or_link_init(&linkL[s]); }
#define ADD_EDGE(u, v, k, l) do { \
    if (ecount[u] == ecap[u]) { ecap[u] = ecap[u] ? 2 * ecap[u] : 4; \
      out[u] = (or_edge*)realloc(out[u], sizeof(or_edge) * ecap[u]); } \
    out[u][ecount[u]].to = (int32_t)(v); out[u][ecount[u]].kind = (k); out[u][ecount[u]].link = (l); \
    ecount[u]++; indeg[v]++; } while (0)
#define KEY(ch, s, j) ((int64_t)(ch) * PM + (int64_t)(s) * m + (j))
  {
    for (int s = 0; s < p; ++s) {
      int32_t cF[2] = {0, 0}, cD[2] = {0, 0}, cW[2] = {0, 0};
      for (int k = 0; k < len[s]; ++k) {
        int64_t u = off[s] + k;
        int x = codes[(int64_t)s * maxlen + k], c = WV_CODE(x), ch = WV_CHUNK(x);
        n_type[u] = x;
        if (c == OR_F) { dur[u] = I->t_f[s]; idxF[KEY(ch, s, cF[ch])] = u; cF[ch]++; }
        else if (c == OR_B) { dur[u] = I->t_d[s] + I->t_w[s]; idxD[KEY(ch, s, cD[ch])] = u; cD[ch]++; }
        else if (c == OR_D) { dur[u] = I->t_d[s]; idxD[KEY(ch, s, cD[ch])] = u; cD[ch]++; }
        else {
          int32_t j = cW[ch] / ns, q = cW[ch] % ns;
          n_sub[u] = q; dur[u] = sub_dur(I->t_w[s], ns, q); cW[ch]++;
          wkey[u] = KEY(ch, s, j);
        }
      }
    }
  }
  for (int64_t s = 0; s < p; ++s) {
    n_type[NC + s] = -1; dur[NC + s] = I->zero1 ? I->t_ag[s] : 0;
    n_type[NC + p + s] = -2; dur[NC + p + s] = I->t_dp[s];
  }
  for (int s = 0; s < p; ++s)                                   /* schedule dependencies */
    for (int k = 0; k + 1 < len[s]; ++k) ADD_EDGE(off[s] + k, off[s] + k + 1, EK_SCHED, -1);
  for (int s = 0; s < p; ++s) {
    for (int j = 0; j < m; ++j) {
      const int64_t f0 = idxF[KEY(0, s, j)], f1 = idxF[KEY(1, s, j)];
      const int64_t d0 = idxD[KEY(0, s, j)], d1 = idxD[KEY(1, s, j)];
      if (s < p - 1) ADD_EDGE(f0, idxF[KEY(0, s + 1, j)], EK_LINK_F, s);   /* chunk 0 forward */
      else ADD_EDGE(f0, idxF[KEY(1, 0, j)], EK_LINK_F, p - 1);            /* wrap p-1 -> 0 */
      if (s < p - 1) ADD_EDGE(f1, idxF[KEY(1, s + 1, j)], EK_LINK_F, s);   /* chunk 1 forward */
      else ADD_EDGE(f1, d1, EK_LOCAL, -1);                              /* loss */
      if (s > 0) ADD_EDGE(d1, idxD[KEY(1, s - 1, j)], EK_LINK_B, s - 1); /* chunk 1 backward */
      else ADD_EDGE(d1, idxD[KEY(0, p - 1, j)], EK_LINK_B, p - 1);       /* wrap 0 -> p-1 */
      if (s > 0) ADD_EDGE(d0, idxD[KEY(0, s - 1, j)], EK_LINK_B, s - 1); /* chunk 0 backward */
    }
    for (int k = 0; k < len[s]; ++k)                                      /* W sub-block after its D */
      if (WV_CODE(n_type[off[s] + k]) == OR_W) ADD_EDGE(idxD[wkey[off[s] + k]], off[s] + k, EK_LOCAL, -1);
    ADD_EDGE(NC + s, idxF[KEY(0, s, 0)], EK_LOCAL, -1);        /* ZeRO-1 AG before chunk 0's first F */
    ADD_EDGE(NC + s, idxF[KEY(1, s, 0)], EK_LOCAL, -1);        /* ... and chunk 1's */
    ADD_EDGE(off[s] + len[s] - 1, NC + p + s, EK_LOCAL, -1);    /* DP AR after the stage's last block */
  }
  int64_t qh = 0, qt = 0, done = 0;
  for (int64_t u = 0; u < N; ++u) if (indeg[u] == 0) queue[qt++] = u;
  while (qh < qt) {
    int64_t u = queue[qh++];
    start[u] = ready[u];
    end[u] = start[u] + dur[u];
    done++;
    for (int32_t e = 0; e < ecount[u]; ++e) {
      or_edge E = out[u][e];
      int64_t c;
      if (E.kind == EK_LINK_F)      c = or_reserve_window(&linkR[E.link], end[u], I->bw_f[E.link]) + I->lat_f[E.link];
      else if (E.kind == EK_LINK_B) c = or_reserve_window(&linkL[E.link], end[u], I->bw_b[E.link]) + I->lat_b[E.link];
      else                          c = end[u];
      ready[E.to] = max64(ready[E.to], c);
      if (--indeg[E.to] == 0) queue[qt++] = E.to;
    }
  }
  if (done < N) {
    R->status = OR_ST_DEADLOCK;
  } else {
    int64_t mk = 0, pk = 0;
    for (int s = 0; s < p; ++s) {
      int64_t mem = 0, peak = 0, busy = 0;
      for (int k = 0; k < len[s]; ++k) {
        int64_t u = off[s] + k;
        int c = WV_CODE(n_type[u]);
        if (c == OR_F) mem += I->m_f[s];
        else if (c == OR_D) mem += I->m_d[s];
        else if (c == OR_B) mem += I->m_d[s] + I->m_w[s];
        else if (n_sub[u] == ns - 1) mem += I->m_w[s];
        peak = max64(peak, mem);
        busy += dur[u];
        if (t_start) t_start[(int64_t)s * maxlen + k] = start[u];
      }
      R->first_start[s] = start[off[s]];
      R->last_end[s] = end[off[s] + len[s] - 1];
      R->busy[s] = busy;
      R->peak[s] = peak;
      if (peak > I->m_lim[s]) R->status |= OR_ST_MEM_EXCEEDED;
      pk = max64(pk, peak);
    }
    for (int64_t u = 0; u < N; ++u) mk = max64(mk, end[u]);
    R->makespan = mk;
    R->peak_mem = pk;
  }
  for (int s = 0; s < p; ++s) { or_link_free(&linkR[s]); or_link_free(&linkL[s]); }
  for (int64_t u = 0; u < N; ++u) free(out[u]);
  free(n_type); free(n_sub); free(dur); free(ready); free(start); free(end); free(indeg); free(ecount);
  free(out); free(ecap); free(idxF); free(idxD); free(wkey); free(queue);
  free(linkR); free(linkL);
#undef KEY
#undef ADD_EDGE
  return R->status;
}

/* ------------------------------------------------------------------------- */
/* Algorithm 1 with the §4.2.2 scheduling loop (:415-432).
 * Each stage keeps an explicit list of schedulable operations with T_avail.
 * Readings: Q11 F/D sub-blocks are contiguous (non-preemptive), W
 * sub-blocks are fillers; Q13 priority: prefer the opposite of the last full F/D
 * block (initially F), then the other, then a W sub-block; Q14/Q15 candidates are
 * eligible ops available at or before the stage's schedulable time; a memory-
 * infeasible F is not eligible; Q16 stage ties -> lowest index; Q18 seeding.   */
typedef struct { int32_t type, mb, subs_done; int64_t avail; } or_op;
typedef struct {
  or_op* ops; int32_t n, cap;
  int64_t last_end, mem, peak, busy, first_start;
  int32_t last_fd;            /* -1 none, OR_F, OR_D */
  int32_t in_prog;            /* index into ops of an F/D with sub-blocks left, or -1 */
  int32_t nemit;
} or_stage;

static void st_add(or_stage* S, int32_t type, int32_t mb, int64_t avail) {
  if (S->n == S->cap) { S->cap = S->cap ? 2 * S->cap : 16; S->ops = (or_op*)realloc(S->ops, sizeof(or_op) * S->cap); }
  S->ops[S->n].type = type; S->ops[S->n].mb = mb; S->ops[S->n].subs_done = 0; S->ops[S->n].avail = avail; S->n++;
}
static void st_del(or_stage* S, int32_t i) { memmove(S->ops + i, S->ops + i + 1, sizeof(or_op) * (S->n - i - 1)); S->n--; }

/* eligible op of a type: the lowest microbatch of that type in the list (microbatch
 * order within stage and type, :346-351); F additionally must fit in memory. */
static int32_t st_head(const or_inst* I, int s, const or_stage* S, int32_t type) {
  int32_t best = -1;
  for (int32_t i = 0; i < S->n; ++i)
    if (S->ops[i].type == type && (best < 0 || S->ops[i].mb < S->ops[best].mb)) best = i;
  if (best >= 0 && type == OR_F && S->mem + I->m_f[s] > I->m_lim[s]) return -1;
  return best;
}

int32_t or_greedy(const or_inst* I, int8_t* codes, int32_t* len, int32_t maxlen,
                  or_result* R, int64_t* t_start) {
  const int p = I->p, m = I->m, ns = I->n_sub;
  memset(R, 0, sizeof(*R));
  R->makespan = -1; R->peak_mem = -1;
  int32_t st = or_validate_instance(I);
  if (st) { R->status = st; return st; }
  if ((int64_t)(2 + ns) * m > maxlen) { R->status = OR_ST_BAD_PLAN; return R->status; }
  or_stage* S = (or_stage*)calloc(p, sizeof(or_stage));
  or_link* linkF = (or_link*)malloc(sizeof(or_link) * p);
  or_link* linkB = (or_link*)malloc(sizeof(or_link) * p);
  for (int s = 0; s < p; ++s) {
    or_link_init(&linkF[s]); or_link_init(&linkB[s]);
    S[s].last_fd = -1; S[s].in_prog = -1; S[s].first_start = -1; len[s] = 0;
  }
  /* lines 2-4: all F_i schedulable on stage 0 (ZeRO-1: after the stage's allgather) */
  for (int i = 0; i < m; ++i) st_add(&S[0], OR_F, i, I->zero1 ? I->t_ag[0] : 0);

  int64_t iters = 0;
  for (;;) {                                   /* line 5: scheduling loop */
    /* line 6: next_stage_to_schedule -- earliest max(last end, earliest avail of
     * schedulable ops) (§4.2.2 :419); ties -> lowest stage index. */
    int best = -1; int64_t best_t = 0;
    for (int s = 0; s < p; ++s) {
      int64_t t;
      if (S[s].in_prog >= 0) {
        t = S[s].last_end;                     /* continue the started F/D block */
      } else {
        int32_t hF = st_head(I, s, &S[s], OR_F), hD = st_head(I, s, &S[s], OR_D), hW = st_head(I, s, &S[s], OR_W);
        if (hF < 0 && hD < 0 && hW < 0) continue;
        int64_t mn = INT64_MAX;
        if (hF >= 0 && S[s].ops[hF].avail < mn) mn = S[s].ops[hF].avail;
        if (hD >= 0 && S[s].ops[hD].avail < mn) mn = S[s].ops[hD].avail;
        if (hW >= 0 && S[s].ops[hW].avail < mn) mn = S[s].ops[hW].avail;
        t = max64(S[s].last_end, mn);
      }
      if (best < 0 || t < best_t) { best = s; best_t = t; }
    }
    if (best < 0) break;                       /* lines 7-9 */
    const int s = best;
    or_stage* T = &S[s];
    int32_t i;
    if (T->in_prog >= 0) {
      i = T->in_prog;
    } else {
      /* line 10: schedulable operation of highest priority (§4.2.2 :421-429) */
      int32_t hF = st_head(I, s, T, OR_F), hD = st_head(I, s, T, OR_D), hW = st_head(I, s, T, OR_W);
      int cF = hF >= 0 && T->ops[hF].avail <= best_t;
      int cD = hD >= 0 && T->ops[hD].avail <= best_t;
      int cW = hW >= 0 && T->ops[hW].avail <= best_t;
      if (T->last_fd == OR_F) i = cD ? hD : (cF ? hF : (cW ? hW : -1));
      else                    i = cF ? hF : (cD ? hD : (cW ? hW : -1));
      if (i < 0) { R->status = OR_ST_DEADLOCK; break; }    /* unreachable by construction */
    }
    or_op* o = &T->ops[i];
    /* line 11: schedule next sub-block of p_cur */
    int64_t T_blk = o->type == OR_F ? I->t_f[s] : (o->type == OR_D ? I->t_d[s] : I->t_w[s]);
    int64_t d = sub_dur(T_blk, ns, o->subs_done);
    int64_t t0 = best_t, t1 = best_t + d;
    iters++;
    if (T->first_start < 0) T->first_start = t0;
    T->busy += d;
    T->last_end = t1;
    /* plan entry: F and D whole blocks at their first sub-block; W per sub-block */
    if (o->type == OR_W || o->subs_done == 0) {
      if (T->nemit < maxlen) {
        codes[(int64_t)s * maxlen + T->nemit] = (int8_t)o->type;
        if (t_start) t_start[(int64_t)s * maxlen + T->nemit] = t0;
      }
      T->nemit++;
    }
    o->subs_done++;
    if (o->subs_done < ns) {
      if (o->type != OR_W) T->in_prog = i;     /* F/D continue contiguously (Q11) */
      continue;
    }
    /* block complete */
    int32_t type = o->type, mb = o->mb;
    T->in_prog = -1;
    st_del(T, i);
    if (type == OR_F) {
      T->mem += I->m_f[s]; T->last_fd = OR_F;
      if (s < p - 1) {                         /* lines 15-21: hand off to the next stage */
        int64_t E = or_reserve_window(&linkF[s], t1, I->bw_f[s]);
        int64_t av = E + I->lat_f[s];
        if (I->zero1 && I->t_ag[s + 1] > av) av = I->t_ag[s + 1];
        st_add(&S[s + 1], OR_F, mb, av);
      } else {
        st_add(T, OR_D, mb, t1);               /* last stage: D depends on the local F */
      }
    } else if (type == OR_D) {
      T->mem += I->m_d[s]; T->last_fd = OR_D;
      st_add(T, OR_W, mb, t1);                 /* lines 12-14: W becomes schedulable */
      if (s > 0) {
        int64_t E = or_reserve_window(&linkB[s - 1], t1, I->bw_b[s - 1]);
        st_add(&S[s - 1], OR_D, mb, E + I->lat_b[s - 1]);
      }
    } else {
      T->mem += I->m_w[s];
    }
    if (T->mem > T->peak) T->peak = T->mem;
  }
  R->iterations = iters;
  int64_t mk = 0, pk = 0;
  int complete = 1;
  for (int s = 0; s < p; ++s) {
    len[s] = S[s].nemit;
    if (S[s].nemit != (2 + ns) * m) complete = 0;
  }
  if (!complete || R->status) {
    R->status |= OR_ST_DEADLOCK;
  } else {
    for (int s = 0; s < p; ++s) {
      R->first_start[s] = S[s].first_start;
      R->last_end[s] = S[s].last_end;
      R->busy[s] = S[s].busy;
      R->peak[s] = S[s].peak;
      if (S[s].peak > I->m_lim[s]) R->status |= OR_ST_MEM_EXCEEDED;
      int64_t e = S[s].last_end + I->t_dp[s];            /* DP allreduce after the last W */
      mk = max64(mk, max64(S[s].last_end, e));
      if (I->zero1) mk = max64(mk, I->t_ag[s]);
      pk = max64(pk, S[s].peak);
    }
    R->makespan = mk; R->peak_mem = pk;
  }
  for (int s = 0; s < p; ++s) { or_link_free(&linkF[s]); or_link_free(&linkB[s]); free(S[s].ops); }
  free(S); free(linkF); free(linkB);
  return R->status;
}

/* ------------------------------------------------------------------------- */
/* Static builders, Table tab:ppschedules (:470) and related work (:780).
 * 1F1B (PipeDream-Flush, combined backward): stage s runs w = min(p-s-1, m) warm-up
 * F, then (F, B) x (m-w), then B x w (reading Q23).
 * GPipe: F x m then B x m (reading Q22).                                         */
void or_build_1f1b(int32_t p, int32_t m, int8_t* codes, int32_t* len, int32_t maxlen) {
  for (int s = 0; s < p; ++s) {
    int w = p - s - 1; if (w > m) w = m;
    int k = 0;
    for (int i = 0; i < w; ++i) codes[(int64_t)s * maxlen + k++] = OR_F;
    for (int i = 0; i < m - w; ++i) { codes[(int64_t)s * maxlen + k++] = OR_F; codes[(int64_t)s * maxlen + k++] = OR_B; }
    for (int i = 0; i < w; ++i) codes[(int64_t)s * maxlen + k++] = OR_B;
    len[s] = k;
  }
}
/* ZB-H1 (Table tab:ppschedules :472; "1F1B ordering with D/W split and W blocks
 * deferred ... at unchanged peak activation memory"), reading Q31: stage s runs
 *   warm-up   F x w,  w = min(p - s, m)
 *   then for k = 0 .. m-1:  D_k,  W_{k-s} if k >= s,  F (the next one) if any remain
 *   then the W blocks still owed (the last min(s, m)).
 * Stage s defers its W blocks by s microbatches (stage 0 keeps W behind its D, the last stage
 * fills its tear-down with them).                                                      */
void or_build_zbh1(int32_t p, int32_t m, int8_t* codes, int32_t* len, int32_t maxlen) {
  for (int s = 0; s < p; ++s) {
    int8_t* row = codes + (int64_t)s * maxlen;
    int w = p - s; if (w > m) w = m;
    int k = 0, nF = 0, nW = 0;
    for (int i = 0; i < w; ++i) { row[k++] = OR_F; ++nF; }
    for (int j = 0; j < m; ++j) {
      row[k++] = OR_D;
      if (j >= s) { row[k++] = OR_W; ++nW; }
      if (nF < m) { row[k++] = OR_F; ++nF; }
    }
    while (nW < m) { row[k++] = OR_W; ++nW; }
    len[s] = k;
  }
}

/* Interleaved 1F1B (IV1F1B, Table tab:ppschedules :471, cited not restated; Megatron's interleaved
 * schedule), reading Q34, for the Loop pattern with 2 chunks and combined B.  Forward unit k
 * (k = 0 .. 2m-1) is chunk (k / p) % 2 of microbatch (k / 2p) p + k % p; backward unit k takes the
 * chunks in reverse, 1 - (k / p) % 2.  Stage s runs the first w = min(2 (p - s - 1) + p, 2m)
 * forward units, then (next forward, next backward) pairs, then the remaining backward units. */
int32_t or_build_iv1f1b(int32_t p, int32_t m, int8_t* codes, int32_t* len, int32_t maxlen) {
  if (p < 1 || m < 1 || m % p != 0 || maxlen < 4 * m) return -1;
  for (int s = 0; s < p; ++s) {
    int8_t* row = codes + (int64_t)s * maxlen;
    int w = 2 * (p - s - 1) + p; if (w > 2 * m) w = 2 * m;
    int k = 0;
#define FWD(u) ((int8_t)(OR_F | ((((u) / p) % 2) << 2)))
#define BWD(u) ((int8_t)(OR_B | ((1 - ((u) / p) % 2) << 2)))
    for (int u = 0; u < w; ++u) row[k++] = FWD(u);
    for (int i = 0; i < 2 * m - w; ++i) { row[k++] = FWD(w + i); row[k++] = BWD(i); }
    for (int u = 2 * m - w; u < 2 * m; ++u) row[k++] = BWD(u);
#undef FWD
#undef BWD
    len[s] = k;
  }
  return 0;
}

/* ZB-V (Table tab:ppschedules :473, cited not restated; the V-shaped Wave layout with split W),
 * reading Q35: the per-stage order of a unit-time list schedule of the Wave data flow (reading
 * Q32, 2 chunks) with every block one tick long and no delays.  At tick t every stage takes at
 * most one block whose inputs were produced at ticks < t:
 *   F0: from stage s-1 (stage 0: none)     F1: from stage s+1 (stage p-1: its own F0)
 *   D1: from stage s-1 (stage 0: its own F1)   D0: from stage s+1 (stage p-1: its own D1)
 *   W_c: after the stage's own D_c;  F only while the stage holds fewer than 2p chunk activations
 *   (F in, W out; 2p chunks = the p full-stage activations 1F1B holds on stage 0, Table :473
 *   "Medium").
 * Choice: a W (W0 before W1) when no other block is ready or the stage is at 2p, else the first
 * ready of F1, F0, D0, D1.  Rows have 6m entries.  Returns 0, or -1 (nothing defined) for p < 1,
 * m < 1 or maxlen < 6m.                                                                       */
int32_t or_build_zbv(int32_t p, int32_t m, int8_t* codes, int32_t* len, int32_t maxlen) {
  if (p < 1 || m < 1 || maxlen < 6 * m) return -1;
  /* n[s][0..5] = blocks done at stage s: F0, F1, D0, D1, W0, W1; prev = the same at tick start */
  int32_t (*n)[6] = (int32_t(*)[6])calloc((size_t)p, sizeof *n);
  int32_t (*prev)[6] = (int32_t(*)[6])calloc((size_t)p, sizeof *prev);
  for (int s = 0; s < p; ++s) len[s] = 0;
  int64_t left = (int64_t)p * 6 * m;
  while (left > 0) {
    memcpy(prev, n, (size_t)p * sizeof *n);
    for (int s = 0; s < p; ++s) {
      const int32_t* c = prev[s];
      const int f0 = c[0] < m && (s == 0 || prev[s - 1][0] > c[0]);
      const int f1 = c[1] < m && (s == p - 1 ? c[0] > c[1] : prev[s + 1][1] > c[1]);
      const int d1 = c[3] < m && (s == 0 ? c[1] > c[3] : prev[s - 1][3] > c[3]);
      const int d0 = c[2] < m && (s == p - 1 ? c[3] > c[2] : prev[s + 1][2] > c[2]);
      const int w0 = c[4] < c[2], w1 = c[5] < c[3];
      const int full = c[0] + c[1] - c[4] - c[5] >= 2 * p;
      const int fa = !full && f1, fb = !full && f0;
      int8_t e;
      if ((w0 || w1) && (full || !(fa || fb || d0 || d1))) e = w0 ? (int8_t)(OR_W | 0 << 2) : (int8_t)(OR_W | 1 << 2);
      else if (fa) e = (int8_t)(OR_F | 1 << 2);
      else if (fb) e = (int8_t)(OR_F | 0 << 2);
      else if (d0) e = (int8_t)(OR_D | 0 << 2);
      else if (d1) e = (int8_t)(OR_D | 1 << 2);
      else continue;                                      /* idle this tick */
      codes[(int64_t)s * maxlen + len[s]++] = e;
      const int ch = e >> 2, ty = e & 3;
      ++n[s][ty == OR_F ? ch : (ty == OR_D ? 2 + ch : 4 + ch)];
      --left;
    }
  }
  free(n); free(prev);
  return 0;
}

void or_build_gpipe(int32_t p, int32_t m, int8_t* codes, int32_t* len, int32_t maxlen) {
  for (int s = 0; s < p; ++s) {
    int k = 0;
    for (int i = 0; i < m; ++i) codes[(int64_t)s * maxlen + k++] = OR_F;
    for (int i = 0; i < m; ++i) codes[(int64_t)s * maxlen + k++] = OR_B;
    len[s] = k;
  }
}

/* ------------------------------------------------------------------------- */
/* Exhaustive optimum over the §4.1 validity set (:322-351) with whole blocks
 * (n_sub = 1, split D/W): every stage sequence respecting microbatch order per
 * type, D_j after F_j, W_j after D_j, and the memory capacity constraint; the
 * cartesian product over stages is simulated and deadlocked products skipped.  */
typedef struct { int8_t* seqs; int64_t n, cap; int32_t L; } or_seqset;

static void enum_stage(const or_inst* I, int s, int8_t* cur, int k, int nF, int nD, int nW, int64_t mem,
                       or_seqset* out, int64_t limit) {
  const int m = I->m, L = 3 * m;
  if (out->n > limit) return;
  if (k == L) {
    if (out->n == out->cap) { out->cap = out->cap ? 2 * out->cap : 64; out->seqs = (int8_t*)realloc(out->seqs, (size_t)out->cap * L); }
    memcpy(out->seqs + out->n * L, cur, L); out->n++;
    return;
  }
  if (nF < m && mem + I->m_f[s] <= I->m_lim[s]) { cur[k] = OR_F; enum_stage(I, s, cur, k + 1, nF + 1, nD, nW, mem + I->m_f[s], out, limit); }
  if (nD < nF) { cur[k] = OR_D; enum_stage(I, s, cur, k + 1, nF, nD + 1, nW, mem + I->m_d[s], out, limit); }
  if (nW < nD) { cur[k] = OR_W; enum_stage(I, s, cur, k + 1, nF, nD, nW + 1, mem + I->m_w[s], out, limit); }
}

int64_t or_enumerate_opt(const or_inst* I, int64_t max_plans, int8_t* best_codes, int32_t* best_len,
                         int32_t maxlen, or_result* best) {
  const int p = I->p, m = I->m, L = 3 * m;
  if (I->n_sub != 1 || L > maxlen || or_validate_instance(I)) return -1;
  or_seqset* sets = (or_seqset*)calloc(p, sizeof(or_seqset));
  int8_t* cur = (int8_t*)malloc(L);
  int64_t total = 1;
  for (int s = 0; s < p; ++s) {
    sets[s].L = L;
    enum_stage(I, s, cur, 0, 0, 0, 0, 0, &sets[s], max_plans);
    if (sets[s].n == 0) { total = 0; break; }
    if (total > max_plans / sets[s].n) total = max_plans + 1; else total *= sets[s].n;
  }
  int64_t evaluated = -1;
  if (total <= max_plans && total > 0) {
    int8_t* codes = (int8_t*)calloc((size_t)p * maxlen, 1);
    int32_t* len = (int32_t*)malloc(sizeof(int32_t) * p);
    int64_t* idx = (int64_t*)calloc(p, sizeof(int64_t));
    or_result r;
    evaluated = 0;
    best->makespan = -1;
    for (int64_t t = 0; t < total; ++t) {
      for (int s = 0; s < p; ++s) { memcpy(codes + (int64_t)s * maxlen, sets[s].seqs + idx[s] * L, L); len[s] = L; }
      if (or_simulate(I, codes, len, maxlen, &r, NULL) == 0) {
        evaluated++;
        if (best->makespan < 0 || r.makespan < best->makespan) {
          *best = r;
          memcpy(best_codes, codes, (size_t)p * maxlen); memcpy(best_len, len, sizeof(int32_t) * p);
        }
      }
      for (int s = p - 1; s >= 0; --s) { if (++idx[s] < sets[s].n) break; idx[s] = 0; }
    }
    free(codes); free(len); free(idx);
  }
  for (int s = 0; s < p; ++s) free(sets[s].seqs);
  free(sets); free(cur);
  (void)m;
  return evaluated;
}

/* ------------------------------------------------------------------------- */
/* Quantization SI -> integer ticks / memory units (Table tab:symbols :98-115;
 * Alg. 1 :404-405: T_lat = alpha[cur,next], T_bw = beta[cur,next] * Msg_Size).
 * One rounding per quantity, llround (half away from zero) in double; reading Q21.
 * m_lim is floored (a budget never grows by rounding).                            */
int32_t or_quantize(const or_spec_si* S, or_inst* o) {
  memset(o, 0, sizeof(*o));
  if (S->p < 1 || S->p > OR_MAXP || S->n_dc < 1 || S->n_dc > 4 || !(S->tick_s > 0) || !(S->mem_unit > 0))
    return OR_ST_BAD_INSTANCE;
  o->p = S->p; o->m = S->m; o->n_sub = S->n_sub; o->zero1 = S->zero1;
  for (int s = 0; s < S->p; ++s) {
    int dc = S->dc_of_stage[s];
    if (dc < 0 || dc >= S->n_dc) return OR_ST_BAD_INSTANCE;
    if (s > 0 && dc < S->dc_of_stage[s - 1]) return OR_ST_BAD_INSTANCE;   /* contiguous DCs */
    o->t_f[s] = llround(S->t_f[s] / S->tick_s);
    o->t_d[s] = llround(S->t_d[s] / S->tick_s);
    o->t_w[s] = llround(S->t_w[s] / S->tick_s);
    o->m_f[s] = llround(S->m_f[s] / S->mem_unit);
    o->m_d[s] = llround(S->m_d[s] / S->mem_unit);
    o->m_w[s] = llround(S->m_w[s] / S->mem_unit);
    o->m_lim[s] = (int64_t)floor(S->m_lim[s] / S->mem_unit);
    o->t_dp[s] = llround(S->t_dp[s] / S->tick_s);
    o->t_ag[s] = S->zero1 ? llround(S->t_ag[s] / S->tick_s) : 0;
    if (s < S->p - 1) {
      int a = S->dc_of_stage[s], b = S->dc_of_stage[s + 1];
      o->lat_f[s] = llround(S->alpha[a][b] / S->tick_s);
      o->bw_f[s]  = llround(S->beta[a][b] * S->msg_f[s] / S->tick_s);
      o->lat_b[s] = llround(S->alpha[b][a] / S->tick_s);
      o->bw_b[s]  = llround(S->beta[b][a] * S->msg_b[s] / S->tick_s);
    }
  }
  return or_validate_instance(o);
}

/* ------------------------------------------------------------------------- */
/* Sweep grid: point index is mixed radix
 * ((((i_pp*n_mb + i_mb)*n_lat + i_lat)*n_bw + i_bw)*n_mem + i_mem)*n_dp + i_dp.
 * Stages split contiguously over min(n_dc, p) DCs: dc(s) = s*n_dc/p; a boundary is
 * cross-DC iff dc(s) != dc(s+1) and then carries (lat, bw) in both directions,
 * intra-DC boundaries carry (0, 0).  m_lim[s] = (x*p*m_f[s] + 500) / 1000.       */
int64_t or_grid_points(const or_grid* G) {
  return (int64_t)G->n_pp_n * G->n_mb_n * G->n_lat * G->n_bw * G->n_mem * G->n_dp;
}

void or_grid_instance(const or_grid* G, int64_t k, or_inst* o) {
  int64_t i_dp = k % G->n_dp; k /= G->n_dp;
  int64_t i_mem = k % G->n_mem; k /= G->n_mem;
  int64_t i_bw = k % G->n_bw; k /= G->n_bw;
  int64_t i_lat = k % G->n_lat; k /= G->n_lat;
  int64_t i_mb = k % G->n_mb_n; k /= G->n_mb_n;
  int64_t i_pp = k;
  *o = G->base;
  const int p = G->n_pp_vals[i_pp];
  o->p = p; o->m = G->n_mb_vals[i_mb];
  int ndc = G->n_dc < p ? G->n_dc : p;
  for (int s = 0; s < OR_MAXP; ++s) {
    o->lat_f[s] = o->bw_f[s] = o->lat_b[s] = o->bw_b[s] = 0;
    if (s < p) {
      o->t_dp[s] = G->tdp[i_dp];
      o->m_lim[s] = (G->mlim_x1000[i_mem] * p * G->base.m_f[s] + 500) / 1000;
    }
    if (s < p - 1 && (int64_t)s * ndc / p != (int64_t)(s + 1) * ndc / p) {
      o->lat_f[s] = o->lat_b[s] = G->lat[i_lat];
      o->bw_f[s] = o->bw_b[s] = G->bw[i_bw];
    }
  }
}

uint64_t or_sweep_point(const or_grid* G, int64_t point, int64_t* cand_ms) {
  or_inst I;
  or_grid_instance(G, point, &I);
  const int p = I.p, m = I.m;
  const int32_t maxlen = 6 * m;
  int8_t* codes = (int8_t*)calloc((size_t)p * maxlen, 1);
  int32_t len[OR_MAXP];
  or_result r;
  uint64_t best = UINT64_MAX;
  static const int nsub_of[6] = {0, 0, 1, 2, 4, 0};
  for (int c = 0; c < 6; ++c) {
    if (cand_ms) cand_ms[c] = -1;
    if (!((G->cand_mask >> c) & 1u)) continue;
    int32_t st;
    if (c == 0) { or_build_gpipe(p, m, codes, len, maxlen); st = or_simulate(&I, codes, len, maxlen, &r, NULL); }
    else if (c == 1) { or_build_1f1b(p, m, codes, len, maxlen); st = or_simulate(&I, codes, len, maxlen, &r, NULL); }
    else if (c == 5) { or_build_zbh1(p, m, codes, len, maxlen); st = or_simulate(&I, codes, len, maxlen, &r, NULL); }
    else { or_inst J = I; J.n_sub = nsub_of[c]; st = or_greedy(&J, codes, len, maxlen, &r, NULL); }
    if (st != 0) continue;                       /* memory-infeasible (or invalid) candidate */
    if (cand_ms) cand_ms[c] = r.makespan;
    uint64_t key = ((uint64_t)r.makespan << 8) | (uint64_t)c;
    if (key < best) best = key;
  }
  free(codes);
  return best;
}
