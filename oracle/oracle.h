/*
 * oracle.h -- CrossPipe CPU ORACLE.  *** TEST INFRASTRUCTURE ONLY ***
 *
 * A plain, slow, single-threaded, int64 CPU implementation of what the CrossPipe
 * hot path computes (arXiv 2507.00217), written directly from PAPER.md.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load this library.  The product (paper_2507_00217_b200, libcrosspipe.so)
 * never includes, links or calls anything in oracle/, and this directory includes
 * nothing from the product (no shared headers, helpers, tables or constants).
 *
 * Citations are PAPER.md line numbers + section.
 *   simulate   : §3.5 "Pipeline Performance Model" PAPER.md:259, §3.3 :232-236,
 *                Alg. 1 comm rule :404-407, §4.2.3 BW model :436-437, App. A :808,
 *                §4.1 constraints :322-351, DP overlap :363
 *   greedy     : Alg. 1, §4.2.2 loop :415-432, §4.2.5 :449
 *   static     : Table tab:ppschedules :470 (1F1B), related work :780 (GPipe)
 *   enumerate  : §4.1 validity set :322-351 (exhaustive optimum, tiny instances)
 *   quantize   : Table tab:symbols :98-115, Alg. 1 inputs :381, :404-405
 *
 * Parity status: every function here is pinned by tests/test_oracle_*.py against
 * closed forms, worked examples (SPEC.md / PAPER.md), brute force or an independent
 * fixed-point formulation; see DESIGN.md §Oracle pins.  No function is "parity unpinned".
 *
 * Conventions (a documented FORMAT, re-declared independently by the product):
 *   op codes  F=0, B=1 (combined D+W), D=2, W=3 (one W entry = one W sub-block)
 *   status    bit0 DEADLOCK, bit1 MEM_EXCEEDED, bit2 BAD_PLAN, bit3 BAD_INSTANCE
 *   boundary s (0 <= s < p-1): forward link s->s+1 (lat_f[s], bw_f[s]),
 *                              backward link s+1->s (lat_b[s], bw_b[s])
 */
#ifndef CROSSPIPE_ORACLE_H
#define CROSSPIPE_ORACLE_H
#include <stdint.h>

#define OR_MAXP 32
#define OR_F 0
#define OR_B 1
#define OR_D 2
#define OR_W 3

#define OR_ST_DEADLOCK     1
#define OR_ST_MEM_EXCEEDED 2
#define OR_ST_BAD_PLAN     4
#define OR_ST_BAD_INSTANCE 8

typedef struct {
  int32_t p, m, n_sub, zero1;
  int64_t t_f[OR_MAXP], t_d[OR_MAXP], t_w[OR_MAXP];             /* ticks */
  int64_t m_f[OR_MAXP], m_d[OR_MAXP], m_w[OR_MAXP], m_lim[OR_MAXP]; /* memory units */
  int64_t t_dp[OR_MAXP], t_ag[OR_MAXP];                         /* ticks (DP allreduce, ZeRO-1 allgather) */
  int64_t lat_f[OR_MAXP], bw_f[OR_MAXP], lat_b[OR_MAXP], bw_b[OR_MAXP]; /* ticks, per boundary */
} or_inst;

typedef struct {
  int32_t status;
  int64_t makespan;                 /* App. A runtime, origin t=0; -1 if the plan cannot complete */
  int64_t peak_mem;                 /* max over stages; -1 if not completed */
  int64_t first_start[OR_MAXP], last_end[OR_MAXP], busy[OR_MAXP], peak[OR_MAXP];
  int64_t iterations;               /* greedy: sub-block scheduling iterations */
} or_result;

/* SI-unit problem description (Table tab:symbols) for the quantizer. */
typedef struct {
  int32_t p, m, n_sub, zero1, n_dc;
  int32_t dc_of_stage[OR_MAXP];
  double t_f[OR_MAXP], t_d[OR_MAXP], t_w[OR_MAXP];                 /* seconds */
  double m_f[OR_MAXP], m_d[OR_MAXP], m_w[OR_MAXP], m_lim[OR_MAXP]; /* bytes */
  double t_dp[OR_MAXP], t_ag[OR_MAXP];                             /* seconds */
  double alpha[4][4];                                              /* seconds */
  double beta[4][4];                                               /* seconds per byte */
  double msg_f[OR_MAXP], msg_b[OR_MAXP];                           /* bytes, per boundary */
  double tick_s, mem_unit;
} or_spec_si;

#ifdef __cplusplus
extern "C" {
#endif

/* §4.2.3 BW_model on one directed link: interval list of reserved windows. */
typedef struct { int64_t *s, *e; int32_t n, cap; } or_link;
void    or_link_init(or_link* L);
void    or_link_free(or_link* L);
int64_t or_reserve_window(or_link* L, int64_t t_ready, int64_t width); /* returns window END */

/* Q29 static plan check -> 0 or OR_ST_BAD_PLAN. codes: [p][maxlen], len: [p]. */
int32_t or_check_plan(const or_inst* I, const int8_t* codes, const int32_t* len, int32_t maxlen);

/* §3.5 performance model over an explicit dependency DAG (Kahn order). t_start nullable [p][maxlen]. */
int32_t or_simulate(const or_inst* I, const int8_t* codes, const int32_t* len, int32_t maxlen,
                    or_result* R, int64_t* t_start);

/* Wave traversal pattern (NEXT 1, reading Q32): 2 model chunks per stage in a V.  Plan entries
 * are type | (chunk << 2).  Static check and DAG simulation as or_check_plan / or_simulate.   */
int32_t or_check_plan_wave(const or_inst* I, const int8_t* codes, const int32_t* len, int32_t maxlen);
int32_t or_simulate_wave(const or_inst* I, const int8_t* codes, const int32_t* len, int32_t maxlen,
                         or_result* R, int64_t* t_start);

/* Loop traversal pattern (reading Q33): 2 model chunks, chunk 1 starts on stage 0 where chunk 0
 * left stage p-1, over the wrap-around link (boundary index p-1: lat_f/bw_f[p-1] is p-1 -> 0,
 * lat_b/bw_b[p-1] is 0 -> p-1).  Plan entries and checks as for Wave.                     */
int32_t or_simulate_loop(const or_inst* I, const int8_t* codes, const int32_t* len, int32_t maxlen,
                         or_result* R, int64_t* t_start);

/* Alg. 1 greedy CrossUD(Sub).  Writes plan (codes/len) and timeline; returns status. */
int32_t or_greedy(const or_inst* I, int8_t* codes, int32_t* len, int32_t maxlen,
                  or_result* R, int64_t* t_start);

/* Static builders (combined backward B). Return number of entries per stage written. */
void or_build_1f1b(int32_t p, int32_t m, int8_t* codes, int32_t* len, int32_t maxlen);
void or_build_gpipe(int32_t p, int32_t m, int8_t* codes, int32_t* len, int32_t maxlen);
/* Interleaved 1F1B for the Loop pattern with 2 chunks (reading Q34), combined B, entries type |
 * chunk << 2; needs m % p == 0 (returns 0) else writes nothing (returns -1); maxlen >= 4m. */
int32_t or_build_iv1f1b(int32_t p, int32_t m, int8_t* codes, int32_t* len, int32_t maxlen);
/* ZB-V for the Wave pattern with 2 chunks and split W (reading Q35): unit-time list schedule;
 * rows of 6m entries type | chunk << 2; returns 0, or -1 for p < 1, m < 1, maxlen < 6m. */
int32_t or_build_zbv(int32_t p, int32_t m, int8_t* codes, int32_t* len, int32_t maxlen);
/* ZB-H1 (split D/W), reading Q31: maxlen >= 3m. */
void or_build_zbh1(int32_t p, int32_t m, int8_t* codes, int32_t* len, int32_t maxlen);

/* Exhaustive optimum over all valid split plans with n_sub = 1 (tiny instances only).
 * Writes the best plan; returns number of complete (non-deadlocked) plans evaluated, -1 if too large. */
int64_t or_enumerate_opt(const or_inst* I, int64_t max_plans, int8_t* best_codes, int32_t* best_len,
                         int32_t maxlen, or_result* best);

/* Exact optimum over the same plan set by branch and bound (bnb.c): DFS over block appends with the
 * greedy's makespan as incumbent, Jackson-preemptive per-stage lower bounds and dominance on
 * interface times.  Tiny instances: p <= 8, m <= 16, n_sub = 1.  Returns 1 if proven optimal, 0 if
 * max_nodes ran out (best = best plan found, info->bound = root lower bound), -1 if not applicable.
 * max_table_bytes caps the dominance table (a full table only stops recording).  flags (tests):
 * OR_BNB_NO_DOMINANCE disables the dominance cut, OR_BNB_NO_JPS replaces the per-stage preemptive
 * bound by the per-block head + duration + tail bound -- independent cut logic, same optimum. */
#define OR_BNB_NO_DOMINANCE 1
#define OR_BNB_NO_JPS 2
typedef struct {
  int64_t greedy;        /* incumbent: or_greedy makespan (n_sub = 1) */
  int64_t root_bound;    /* lower bound at the root */
  int64_t bound;         /* proven lower bound: the optimum if proven, else root_bound */
  int64_t nodes;         /* search nodes visited */
  int64_t table_bytes;   /* dominance vectors recorded */
  int32_t proven;
} or_bnb_info;
int32_t or_bnb_opt(const or_inst* I, int64_t max_nodes, int64_t max_table_bytes, int32_t flags, int8_t* best_codes,
                   int32_t* best_len, int32_t maxlen, or_result* best, or_bnb_info* info);

/* SI -> ticks / units quantization; returns 0 or OR_ST_BAD_INSTANCE. */
int32_t or_quantize(const or_spec_si* S, or_inst* out);

/* Instance invariants (SPEC.md:46-50 + Q10/Q12); returns 0 or OR_ST_BAD_INSTANCE. */
int32_t or_validate_instance(const or_inst* I);

/* Grid sweep (§6.2 "schedule with the best simulation performance is selected").
 * Candidates: 0 GPipe, 1 1F1B, 2/3/4 greedy with n_sub = 1/2/4.  See DESIGN.md §Sweep. */
typedef struct {
  or_inst base;                   /* per-stage costs/memory deltas; p/m/lat/bw/m_lim/t_dp overridden */
  int32_t n_dc;
  int32_t n_pp_vals[8], n_pp_n, n_mb_vals[8], n_mb_n;
  const int64_t* lat; int32_t n_lat;      /* cross-DC latency ticks */
  const int64_t* bw;  int32_t n_bw;       /* cross-DC bandwidth window ticks (beta * msg) */
  const int64_t* mlim_x1000; int32_t n_mem; /* m_lim = round(x/1000 * p * m_f[s]) per stage */
  const int64_t* tdp; int32_t n_dp;       /* DP allreduce ticks */
  uint32_t cand_mask;
} or_grid;
int64_t or_grid_points(const or_grid* G);
void    or_grid_instance(const or_grid* G, int64_t point, or_inst* out);
/* best key = (makespan << 8) | cand, UINT64_MAX if none feasible; cand_ms[6] nullable (-1 = not run / infeasible) */
uint64_t or_sweep_point(const or_grid* G, int64_t point, int64_t* cand_ms);

#ifdef __cplusplus
}
#endif
#endif
