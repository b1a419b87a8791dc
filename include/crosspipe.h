/*
 * crosspipe.h -- C ABI (v3, CP_ABI_VERSION) of the B200-native CrossPipe hot path (arXiv 2507.00217).
 *
 * What the calls compute (citations are PAPER.md line numbers):
 *   cp_simulate    §3.5 pipeline performance model (:257-260): per-stage block order ->
 *                  timeline (start = max(previous block end on the stage, dependency end +
 *                  comm delay)), alpha-beta comm with link queuing (fig:comm_model :133,
 *                  Alg. 1 :404-407, §4.2.3 :436-437), memory accounting (§4.1 :307-308,
 *                  :341-345), DP-overlap tail and ZeRO-1 gate (:363), runtime App. A (:808).
 *   cp_greedy      Alg. 1 "Greedy Generation for CrossUDSub" (:383-412) with the §4.2.2
 *                  scheduling loop (:415-432); returns the schedule and its timeline.
 *   cp_sweep_shard schedule selection "with the best simulation performance" (:535, :543)
 *                  over a grid of instances; CP_N_CAND = 6 candidates: GPipe, 1F1B
 *                  (tab:ppschedules :470), greedy n_sub = 1, 2, 4, ZB-H1 (:472, Q31).
 *   cp_build_static  static plans of Table tab:ppschedules (:468-473).
 *   cp_exact       exact optimum of tiny instances (§4.1 validity set :322-351).
 *   cp_quantize    SI (seconds, bytes, s/byte) -> integer ticks / memory units (tab:symbols
 *                  :98-115, Alg. 1 inputs :381).
 * Every ambiguity is resolved by the readings Q1-Q37 listed in DESIGN.md §2.
 *
 * Conventions
 *   - Pointers are DEVICE pointers unless marked (host).  The caller owns every buffer;
 *     the library allocates nothing and keeps no global state (reentrant).
 *   - Compute calls enqueue on `stream` and return without synchronizing.  Return codes
 *     (cp_rc) are API-level and synchronous: bad descriptor, unsupported shape, workspace
 *     too small, CUDA launch error.  Per-item problems never fail a call: they set the
 *     item's cp_item status bits, visible once the stream has completed.
 *   - All device arithmetic is int32 on integer ticks; an item whose conservative horizon
 *     bound U (Q21) is >= 2^30, or whose sizes exceed the GPU limits below, gets
 *     CPI_OVERFLOW and is not evaluated.
 *   - Outputs are deterministic and bit-identical across runs, GPUs and world sizes.
 */
#ifndef CROSSPIPE_H
#define CROSSPIPE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CP_ABI_VERSION 3u      /* v2: ZB-H1 sweep candidate (6 candidates), cp_build_static;
                                  v3: cp_exact_bnb, CPI_INCOMPLETE, grid-sized sweep workspace */
#define CP_MAX_STAGES 32      /* lane-per-stage design: p <= 32 */
#define CP_MAX_MB 1024        /* microbatches per instance */
#define CP_MAX_SUB 16         /* n_sub limit of the GPU path */

/* op codes of a plan entry (2 bits) */
#define CP_OP_F 0u            /* forward block */
#define CP_OP_B 1u            /* combined backward block B = D + W (App. B :811-822) */
#define CP_OP_D 2u            /* input-gradient block (DGrad) */
#define CP_OP_W 3u            /* ONE weight-gradient sub-block (n_sub per W block) */

/* traversal patterns of cp_schedules.pattern */
#define CP_PATTERN_UD 0
#define CP_PATTERN_WAVE 1
#define CP_PATTERN_LOOP 2

/* static plan families (cp_build_static kind; equal to their sweep candidate ids) */
#define CP_PLAN_GPIPE 0       /* F x m, then B x m (reading Q22) */
#define CP_PLAN_1F1B 1        /* PipeDream-Flush, combined B, warm-up min(p-s-1, m) (Q23) */
#define CP_PLAN_ZBH1 5        /* ZB-H1, split D/W, W deferred by s microbatches on stage s (Q31) */
#define CP_PLAN_IV1F1B 6      /* interleaved 1F1B, Loop pattern plans (pattern CP_PATTERN_LOOP, 4-bit entries,
                                 2 chunks, combined B), needs n_mb % n_pp == 0 (Q34) */
#define CP_PLAN_ZBV 7         /* ZB-V, Wave pattern plans (pattern CP_PATTERN_WAVE, 4-bit entries, 2 chunks,
                                 split W): unit-time list schedule, 2p chunk-activation budget (Q35) */
#define CP_N_CAND 6           /* sweep candidates: 0 GPipe, 1 1F1B, 2/3/4 greedy n_sub 1/2/4, 5 ZB-H1 */

typedef enum { CP_OK = 0, CP_EINVAL = -1, CP_EUNSUPPORTED = -2, CP_ECUDA = -3, CP_EWORKSPACE = -4 } cp_rc;

typedef enum {                /* per-item status bitmask */
  CPI_OK = 0,
  CPI_DEADLOCK = 1,           /* plan cannot complete (cross-stage cycle / D_j before F_j) */
  CPI_MEM_EXCEEDED = 2,       /* completed, but a stage's peak > m_lim */
  CPI_BAD_PLAN = 4,           /* static plan check failed (reading Q29) */
  CPI_BAD_INSTANCE = 8,       /* instance invariant violated (Q10, Q12) */
  CPI_OVERFLOW = 16,          /* exceeds int32 horizon (U >= 2^30) or GPU size limits */
  CPI_INCOMPLETE = 64         /* cp_exact_bnb: a node / round / frontier limit stopped the search */
} cp_item;

/* Instance record v1: 1792 B, 128-B aligned, int32 ticks / memory units.
 * Per-stage arrays are indexed by stage s < n_pp.  Boundary arrays are indexed by
 * boundary s < n_pp-1: *_f = link s -> s+1 (activations), *_b = link s+1 -> s (gradients).
 * Invariants (else CPI_BAD_INSTANCE): 1 <= n_pp <= 32, n_mb >= 1, n_sub >= 1; t_f, t_d,
 * t_w > 0; every block >= n_sub ticks (t_f, t_d, t_w >= n_sub, Q12); m_f > 0, m_d <= 0, m_w <= 0, m_f + m_d + m_w == 0; m_lim >= m_f;
 * t_dp, t_ag >= 0; lat/bw >= 0.  flags bit0 = ZeRO-1 (t_ag gates the stage's F blocks). */
typedef struct {
  uint8_t n_pp, n_dc, n_sub, flags;
  uint16_t n_mb, version;                          /* version = 1 */
  int32_t tick_ns;                                 /* informational: tick length */
  uint8_t dc_first_stage[4];                       /* informational: contiguous DC split */
  uint8_t _pad0[16];
  int32_t t_f[32], t_d[32], t_w[32];               /* ticks */
  int32_t m_f[32], m_d[32], m_w[32], m_lim[32];    /* memory units */
  int32_t t_dp[32], t_ag[32];                      /* DP allreduce / ZeRO-1 allgather, ticks */
  int32_t lat_f[32], bw_f[32], lat_b[32], bw_b[32];/* per boundary, ticks (bw = beta * msg) */
  uint8_t _tail[96];
} cp_inst_v1;

typedef struct {
  int32_t n;                  /* number of instance records */
  int32_t max_pp;             /* upper bound of n_pp over the batch: selects the lane segment width */
  int32_t max_mb;             /* upper bound of n_mb: sizes the workspace of the overflow path */
  int32_t ring_hint;          /* upper bound of in-flight F blocks per stage, usually
                                 min(n_mb, floor(m_lim/m_f)); 0 -> max_mb.  Only a performance hint. */
  const cp_inst_v1* inst;     /* [n] */
} cp_instances;

/* Plan batch.  Entry k of stage s of schedule i is the 2-bit code
 *   (ops[(i*words + k/16)*stage_stride + s] >> (2*(k%16))) & 3        (LSB first)
 * i.e. word-major / stage-minor, so a warp reads word k of all its stages in one
 * coalesced transaction.  Microbatch indices are implied by per-type counters
 * (microbatch order within stage and type, §4.1 :346-351); W entries are sub-blocks. */
typedef struct {
  int32_t n;                  /* number of schedules */
  int32_t stage_stride;       /* >= max_pp */
  int32_t words;              /* words per stage row: capacity 16*words entries (8*words if pattern > 0) */
  int32_t pattern;            /* traversal pattern (fig:pptravesal) of the plans, cp_simulate only:
                                 CP_PATTERN_UD (0): 2-bit entries (above);
                                 CP_PATTERN_WAVE (1, reading Q32) and CP_PATTERN_LOOP (2, Q33): two model
                                 chunks per stage, 4-bit entries type | chunk << 2, 8 per word LSB-first,
                                 same [n][words][stage_stride] order; need max_pp <= 32, max_mb <= 256.
                                 Loop reads its wrap links at boundary index p-1 (Q33). */
  const int32_t* inst_of;     /* [n] instance of schedule i; NULL: instance i (or 0 if instances.n == 1) */
  uint32_t* ops;              /* [n][words][stage_stride]; input of cp_simulate, output of cp_greedy */
  uint16_t* len;              /* [n][stage_stride] entries per stage row */
} cp_schedules;

typedef struct {
  int64_t* makespan;          /* [n] App.-A runtime in ticks (origin t = 0); -1 if not completed */
  int32_t* peak_mem;          /* [n] max over stages, -1 if not completed (nullable) */
  int32_t* status;            /* [n] cp_item bitmask */
  int32_t* stage_stats;       /* [n][stage_stride][4] first_start, last_end, busy, peak (nullable) */
  int32_t* t_start;           /* [n][stage_stride][len_stride] start tick of every entry (nullable) */
  int32_t len_stride;
  int32_t index_base;         /* added to the item index in best_key (chunked calls report global ids) */
  uint64_t* best_key;         /* [1] nullable: atomic min of (makespan << 32 | (index_base + i)) over
                                 items with status 0; the caller initializes it to INT64_MAX */
} cp_results;

#define CP_GRID_MAX_AXIS 128
#define CP_GRID_MAX_SMALL 16
/* (host) Sweep grid.  Point k decodes mixed-radix as
 *   k = ((((i_pp*n_mb_n + i_mb)*n_lat + i_lat)*n_bw + i_bw)*n_mem + i_mem)*n_dp + i_dp.
 * Instance of a point: base per-stage costs / memory deltas / t_ag / flags, p = n_pp_vals[i_pp],
 * m = n_mb_vals[i_mb]; stages split contiguously over min(n_dc, p) DCs, dc(s) = s*n_dc/p;
 * a cross-DC boundary carries (lat[i_lat], bw[i_bw]) both ways, intra-DC boundaries (0, 0);
 * m_lim[s] = (mlim_x1000[i_mem]*p*m_f[s] + 500)/1000; t_dp[s] = tdp[i_dp].
 * Candidates (cand_mask bits, CP_N_CAND of them): 0 GPipe, 1 1F1B (combined B; n_sub ignored),
 * 2/3/4 greedy with n_sub = 1/2/4, 5 ZB-H1 (split D/W, whole W blocks; n_sub ignored).  key = (makespan << 8) | cand (int64 >= 0), INT64_MAX for a memory-infeasible
 * candidate; the point's key is the minimum (ties -> lower candidate id), INT64_MAX if no candidate
 * is feasible, INT64_MAX-1 if the point exceeds the GPU limits (CPI_OVERFLOW).  Signed keys let
 * an int64 all-reduce(MIN) across ranks act as allgather + argmin in one collective. */
typedef struct {
  cp_inst_v1 base;
  int32_t n_dc;
  int32_t n_pp_vals[8], n_pp_n;
  int32_t n_mb_vals[8], n_mb_n;
  int32_t lat[CP_GRID_MAX_AXIS], n_lat;
  int32_t bw[CP_GRID_MAX_AXIS], n_bw;
  int32_t mlim_x1000[CP_GRID_MAX_SMALL], n_mem;
  int32_t tdp[CP_GRID_MAX_SMALL], n_dp;
  uint32_t cand_mask;
} cp_grid;

uint32_t    cp_abi_version(void);
const char* cp_status_string(int32_t code);   /* cp_rc (<0) or cp_item bitmask (>=0) */

/* Workspace bytes (device memory, caller-allocated, need not be initialized) for a call
 * over n_items items: which = 0 cp_simulate (desc: cp_instances*, n_items = schedules),
 * 1 cp_greedy (desc: cp_instances*, n_items = instances), 2 cp_sweep_shard (desc: cp_grid*).
 * Holds the overflow list and the global arrival rings of the fix-up pass. */
size_t cp_workspace_bytes(int32_t which, const void* desc, int64_t n_items);

/* Evaluate sched->n fixed plans.  Errors: CP_EINVAL (NULL/inconsistent descriptors,
 * stage_stride < max_pp, words < 1, len_stride < 1 with t_start, unknown pattern, inst_of NULL
 * with 1 < inst->n < sched->n), CP_EUNSUPPORTED (max_pp > 32 or max_mb > 1024; Wave / Loop
 * plans with max_mb > 256, or whose staged rows do not fit one block's shared memory),
 * CP_EWORKSPACE, CP_ECUDA (launch failure).  A row longer than its capacity, or violating
 * Q29, is the item's CPI_BAD_PLAN, not an API error. */
int32_t cp_simulate(const cp_instances* inst, const cp_schedules* sched, const cp_results* res,
                    void* ws, size_t ws_bytes, void* stream /* cudaStream_t */);

/* Generate one greedy schedule per instance (out->n must equal inst->n, out->inst_of NULL,
 * stage_stride >= max_pp, words >= 1).  Writes out->ops / out->len and res (its timeline).  An
 * item whose schedule does not fit the rows (16*out->words < (2+n_sub)*n_mb) gets CPI_BAD_PLAN.
 * Errors as cp_simulate. */
int32_t cp_greedy(const cp_instances* inst, const cp_schedules* out, const cp_results* res,
                  void* ws, size_t ws_bytes, void* stream);

/* Evaluate grid points [point_lo, point_hi): initializes and writes keys[k] for k in range only
 * (the caller fills the rest with INT64_MAX; cp_sweep in python = fill + shard + all_reduce(MIN)).
 * Work is (point, candidate) tasks taken from a device counter (most expensive first) and combined
 * with a 64-bit atomicMin per point; p-classes run concurrently on streams forked from `stream`
 * and joined back to it (stream priorities: the largest-n_mb greedy tasks of a proper part of the
 * grid first, then greedy before static candidates across p-classes).  ws: cp_workspace_bytes(2,
 * grid, 0) bytes: 256 B of task counters; global-memory arrival rings for any p-class whose
 * in-flight bound min(m, M_L/m_f) does not fit one block's shared memory (about 900 microbatches);
 * for grids with static candidates and every n_mb <= 255, the per-call plan library (64 B of
 * counters + 3 x n_pp x n_mb plans of ceil(3 max_m / 16) words x 32 rows, 256-B aligned); and
 * 256 B of counters for the long-task launches.  Errors: CP_EINVAL for a malformed grid --
 * axis sizes, negative axis values, or any point whose synthesized instance violates the record
 * invariants (e.g. a p beyond the base record's stages, M_L < m_f or beyond int32) --,
 * CP_EUNSUPPORTED (p > 32, m > 1024), CP_EWORKSPACE, CP_ECUDA.
 * cand_makespan (nullable) [n_points][CP_N_CAND] int32: makespan of each candidate, -1 if not run
 * or memory-infeasible.  grid is a HOST pointer, passed to the kernel by value. */
int32_t cp_sweep_shard(const cp_grid* grid, int64_t point_lo, int64_t point_hi,
                       int64_t* keys, int32_t* cand_makespan, void* ws, size_t ws_bytes, void* stream);

/* Build static plans (PAPER.md Table tab:ppschedules :468-473; readings Q22, Q23, Q31, Q34, Q35)
 * for the out->n items of `out`: item i uses instance inst_of[i] (NULL: instance i, or 0 if
 * inst->n == 1) and gets its (p, m) plan in the packed layout cp_simulate reads.  kind:
 * CP_PLAN_GPIPE, CP_PLAN_1F1B, CP_PLAN_ZBH1 (2-bit UD entries), CP_PLAN_IV1F1B (4-bit Loop entries,
 * 8 per word; an item with n_mb % n_pp != 0 gets all-zero rows) or CP_PLAN_ZBV (4-bit Wave entries,
 * 6*n_mb per row; an item with n_pp > 32 gets all-zero rows).  Every word of out->ops and every row
 * of out->len is written (entries past a row's length and rows >= p are 0), so the result is fully
 * defined.
 * Errors: CP_EINVAL for an unknown kind, NULL / inconsistent descriptors, stage_stride < max_pp,
 * or the row capacity (16*words entries, 8*words for IV1F1B / ZB-V) < entries per row at max_mb
 * (2*max_mb; 3*max_mb for ZB-H1; 4*max_mb for IV1F1B; 6*max_mb for ZB-V).  An item whose own
 * (p, m) exceeds (stage_stride, words) gets all-zero rows.  Enqueued on `stream`, no sync. */
int32_t cp_build_static(int32_t kind, const cp_instances* inst, const cp_schedules* out, void* stream);

/* Exact optimum of tiny instances (the stand-in for the paper's CO solver,
 * PAPER.md §4.1 :322-360): for each of the inst->n instances, every plan of split blocks (F, D, W;
 * n_sub must be 1) whose stage sequences respect microbatch order per type, D_j after F_j, W_j after
 * D_j and the memory capacity m_lim along the sequence is enumerated and simulated (cp_simulate's
 * model), and the makespan-optimal plan is returned -- the first optimum in the order "stage sequences
 * in lexicographic order F < D < W, the last stage varying fastest".  Deadlocking plans are skipped.
 * Limits: n_pp <= 8, n_mb <= 8, at most `cap` valid sequences per stage and `max_plans` (< 2^52)
 * plans per instance, horizon < 2^30 ticks and < 2^(63 - ceil(log2 plans)) (the packed key); an
 * instance beyond them gets status CPI_OVERFLOW and makespan -1, one without any completing plan
 * CPI_DEADLOCK.
 * upper (nullable, device) [n] int32: a known feasible makespan per instance (e.g. cp_greedy's with
 * n_sub = 1), -1 for none; it only seeds the search's cut (plans longer than it are skipped early),
 * the result is the same.  An instance whose every plan is longer than its `upper` reports
 * CPI_DEADLOCK, so pass a makespan some valid plan reaches.
 * out: n == inst->n, inst_of NULL, stage_stride >= max_pp, 16*words >= 3*max_mb; every word and
 * row is written (2-bit entries, zero past 3m and for rows >= n_pp).  makespan, status: [n] int32.
 * ws: cp_exact_workspace_bytes(n, cap) bytes (n * 8 * cap * 8 B of sequences).  Errors: CP_EINVAL
 * for NULL / inconsistent arguments, cap < 1, max_plans outside [1, 2^52); CP_EWORKSPACE.
 * Enqueued on `stream`, no sync. */
size_t cp_exact_workspace_bytes(int32_t n, int32_t cap);
int32_t cp_exact(const cp_instances* inst, const cp_schedules* out, const int32_t* upper, int32_t* makespan,
                 int32_t* status, int32_t cap, int64_t max_plans, void* ws, size_t ws_bytes, void* stream);

/* Exact optimum of tiny instances by parallel branch and bound (exact_bnb.cu; SURVEY.md §8(f)
 * NEXT 3, §8(c) c5): the same optimum as cp_exact -- min over every plan of split blocks (F, D, W;
 * n_sub must be 1) in microbatch order per type, D_j after F_j, W_j after D_j, within m_lim along the
 * sequence, of its §3.5 makespan (§4.1 :313-363) -- found by search instead of
 * enumeration, which reaches the paper's 4 x 8 E1 setup (:486, :491).  Nodes are partial schedules
 * extended one block at a time; a node is cut by a lower bound (per-stage Jackson preemptive
 * schedule with dependency heads and tails) against the instance's incumbent, or by dominance (a
 * recorded node with the same block counts and no later interface times).  Warps search depth
 * first for at most `budget` nodes per work item and return the rest of their stack to a frontier;
 * the call repeats rounds until the frontier is empty, so it SYNCHRONIZES `stream` once per round.
 * Per instance: makespan [n] int32 and the plan in out (2-bit entries, 3m per row, rows >= n_pp
 * zero); status 0 = proven optimal; CPI_INCOMPLETE = stopped by max_nodes (nodes searched over all
 * instances), max_rounds or a full frontier: makespan / plan = best found, bound = lower bound
 * proven at the root; CPI_DEADLOCK = no plan reaches upper; CPI_OVERFLOW = outside the limits
 * (n_pp <= 8, n_mb <= 16, n_sub = 1, horizon < 2^29 ticks, record invariants).
 * upper (nullable, device) [n] int32: a feasible makespan per instance (e.g. cp_greedy's with
 * n_sub = 1), -1 for none; the search returns a plan of makespan <= upper, so pass one some plan
 * reaches.  bound (nullable) [n] int32: proven lower bound (= makespan when status 0).  nodes
 * (nullable) [n] int64: nodes searched.  front_cap: frontier items per round; table_entries: the
 * per-instance dominance table, a power of two.  ws: cp_exact_bnb_workspace_bytes(...) bytes.
 * out: n == inst->n, inst_of NULL, stage_stride >= max_pp, 16*words >= 3*max_mb.  Errors:
 * CP_EINVAL, CP_EWORKSPACE, CP_ECUDA. */
size_t cp_exact_bnb_workspace_bytes(const cp_instances* inst, int32_t front_cap, int64_t table_entries);
int32_t cp_exact_bnb(const cp_instances* inst, const cp_schedules* out, const int32_t* upper, int32_t* makespan,
                     int32_t* status, int32_t* bound, int64_t* nodes, int32_t budget, int64_t max_nodes,
                     int32_t max_rounds, int32_t front_cap, int64_t table_entries, void* ws, size_t ws_bytes,
                     void* stream);

/* Evaluate the points owned by `rank` of `world` under blocked ownership: every (n_pp, n_mb) block
 * of inner = n_lat*n_bw*n_mem*n_dp consecutive points is cut into `world` contiguous slices,
 * slice r = [inner*r/world, inner*(r+1)/world), and rank r owns slice r of every block.  Every
 * rank so gets the same mix of (p, m) work and all p-classes run concurrently on each GPU (the
 * contiguous ranges of cp_sweep_partition hold few classes per rank).  Initializes and writes
 * keys / cand_makespan of the owned points only; same ws and semantics as cp_sweep_shard. */
int32_t cp_sweep_shard_rank(const cp_grid* grid, int32_t rank, int32_t world, int64_t* keys,
                            int32_t* cand_makespan, void* ws, size_t ws_bytes, void* stream);

/* (host) Cost-balanced partition of the grid's points over `world` ranks: bounds[0..world]
 * with bounds[r]..bounds[r+1] owned by rank r; cuts at equal prefix sums of the estimated
 * cost p*m*sum_{cand}(2 + n_sub(cand)). */
int32_t cp_sweep_partition(const cp_grid* grid, int32_t world, int64_t* bounds);

/* (host) SI -> record quantization.  All arrays have n_pp entries (boundary arrays n_pp-1).
 * ticks = llround(x / tick_s) (half away from zero, double); bw = llround(beta*msg/tick_s);
 * memory = llround(bytes / mem_unit), m_lim = floor(m_lim / mem_unit).  Returns the item
 * status (0 or CPI_BAD_INSTANCE, CPI_OVERFLOW if a value does not fit int32). */
typedef struct {
  int32_t n_pp, n_mb, n_sub, zero1, n_dc;
  int32_t dc_of_stage[32];
  double t_f[32], t_d[32], t_w[32];                /* seconds */
  double m_f[32], m_d[32], m_w[32], m_lim[32];     /* bytes */
  double t_dp[32], t_ag[32];                       /* seconds */
  double alpha[4][4];                              /* seconds, [src dc][dst dc] */
  double beta[4][4];                               /* seconds per byte */
  double msg_f[32], msg_b[32];                     /* bytes per boundary */
  double tick_s, mem_unit;
} cp_spec_si;
int32_t cp_quantize(const cp_spec_si* spec /*host*/, cp_inst_v1* out /*host*/);

/* (host) Invariant check of one record; returns 0 or CPI_BAD_INSTANCE / CPI_OVERFLOW and,
 * if msg != NULL, a NUL-terminated message naming the violated invariant. */
int32_t cp_validate_instance(const cp_inst_v1* inst /*host*/, char* msg, size_t msg_len);

#ifdef __cplusplus
}
#endif
#endif /* CROSSPIPE_H */
