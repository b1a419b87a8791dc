// engine.h -- internal interface between the C-ABI host layer (abi.cpp) and the
// sm_100a kernels (engine.cu).  Not part of the public ABI (see include/crosspipe.h).
#pragma once
#include <stddef.h>
#include <stdint.h>

#include "crosspipe.h"

namespace cpk {

enum Mode : int32_t { MODE_SIM = 0, MODE_GREEDY = 1, MODE_SWEEP = 2 };

// Kernel arguments, passed by value (__grid_constant__) -- the sweep grid rides along
// in the kernel parameter space, so a sweep launch needs no host->device copy.
struct Args {
  // instances (SIM / GREEDY)
  const cp_inst_v1* inst;
  const int32_t* inst_of;
  int32_t n_inst;
  int32_t n_items;
  // lane geometry
  int32_t seg_lg;          // segment width W = 1 << seg_lg (>= p of every item)
  int32_t ring_slots;      // arrival-ring slots R (>= every producer->consumer lead)
  int32_t plan_words;      // plan words staged in shared memory per buffer (0: plans read from global)
  int32_t smem_words_per_warp;
  int32_t tma;             // plan rows fetched by TMA bulk copies, double-buffered (one item per warp)
  int32_t* ring_g;         // global rings (ring_global launches): [warps][2][R][32]
  // plans
  uint32_t* ops;
  uint16_t* len;
  int32_t stage_stride;
  int32_t words;
  // results
  int64_t* makespan;
  int32_t* peak_mem;
  int32_t* status;
  int32_t* stage_stats;
  int32_t* t_start;
  int32_t len_stride;
  int32_t from_list;       // items come from the overflow list (fix-up pass)
  int32_t index_base;      // added to item ids in best_key
  unsigned long long* best_key;
  // overflow list (items whose lead exceeded R in the fast pass)
  int32_t* ovf_count;
  int32_t* ovf_list;
  // sweep
  int64_t pt_lo, pt_hi;
  unsigned long long* keys;
  unsigned long long* sweep_counter;   // dynamic task counter of a sweep launch (workspace)
  int32_t* cand_ms;
  int32_t tier_lo, tier_hi;            // sweep greedy: only tasks whose ring lead bound is in [lo, hi]
  // sweep point set: contiguous [pt_lo, pt_hi) if own_hi == own_lo; otherwise blocked ownership:
  // blocks [pt_lo, pt_hi) of blk_inner points, slice [own_lo, own_hi) of each (cp_sweep_shard_rank)
  int64_t blk_inner;
  int32_t own_lo, own_hi;
  int32_t chunk_pattern;               // two-chunk plans: CP_PATTERN_WAVE or CP_PATTERN_LOOP
  int32_t shared_tab;                  // k_sim32: one cost / increment table per block (all items use instance 0)
  int32_t* work_counter;               // k_chunk32f: dynamic item counter (workspace; nullptr: static)
  cp_grid grid;
};

// launchers (return cudaError_t as int)
int launch_engine(Mode mode, bool ring_global, const Args& a, int blocks, int threads, size_t smem, void* stream);
// fast path of cp_simulate (sim32.cu): one item per warp, stage_stride 32, smem plans (TMA); with a
// timeline, start ticks are staged in shared memory and written 32 B per lane
int launch_sim32(bool timeline, const Args& a, int blocks, int threads, size_t smem, void* stream);
int sim32_blocks_per_sm(bool timeline, int threads, size_t smem);
int launch_wave32(const Args& a, int blocks, int threads, size_t smem, void* stream);
int wave32_blocks_per_sm(int threads, size_t smem);
// fast path of cp_greedy (greedy_fast.cu): compile-time segment width W in {8, 16, 32}, no timeline
// grid = false: cp_greedy; grid = true: the greedy candidates of cp_sweep_shard
int launch_greedy_fast(int W, bool grid, const Args& a, int blocks, int threads, size_t smem, void* stream);
int greedy_fast_blocks_per_sm(int W, bool grid, int threads, size_t smem);
int engine_blocks_per_sm(Mode mode, bool ring_global, int threads, size_t smem, bool timeline);
int device_sm_count();
int launch_build_static(int kind, const cp_inst_v1* inst, int n_inst, const int32_t* inst_of, long long n, int stride,
                        int words, uint32_t* ops, uint16_t* len, void* stream);
// cp_exact (exact.cu): batched exhaustive search for tiny instances
constexpr int kExactMaxP = 8;          // stages
constexpr int kExactMaxM = 8;          // microbatches (3m <= 24 entries: one uint64 per stage sequence)
int launch_exact(const cp_inst_v1* inst, int n, int cap, long long max_plans, const int32_t* upper, void* ws,
                 int stride, int words, uint32_t* ops, uint16_t* len, int32_t* makespan, int32_t* status,
                 void* stream);
size_t exact_ws_seq_bytes(int n, int cap);
size_t exact_ws_bytes(int n, int cap);
// cp_exact_bnb (exact_bnb.cu): batched parallel branch and bound for tiny instances
constexpr int kBnbMaxP = 8;            // stages
constexpr int kBnbMaxM = 16;           // microbatches
struct BnbLayout {
  size_t off_bi, off_ctl, off_plan, off_cnt, off_front0, off_front1, off_table, bytes;
  int front_stride, table_stride;
};
BnbLayout bnb_layout(int n, int lmax, int vlen_max, int front_cap, long long table_cap);
int launch_bnb(const cp_inst_v1* inst, int n, const int32_t* upper, int lmax, int vlen_max, int front_cap,
               long long table_cap, int budget, long long max_nodes, int max_rounds, void* ws, int stage_stride,
               int words, uint32_t* ops, uint16_t* len, int32_t* makespan, int32_t* status, int32_t* bound,
               long long* nodes_out, void* stream);
int launch_sweep_init(unsigned long long* keys, int32_t* cand_ms, long long lo, long long hi, long long inner, int own_lo,
                      int own_hi, void* stream);

constexpr int kThreads = 128;          // 4 warps per block
// fast-path kernels launch 2-warp blocks; their residency is set by shared memory (about 9 such
// blocks per SM), so the launch bound lets ptxas spend up to 113 registers instead of
// rematerializing addresses and flags inside the round (measured: greedy round 169 -> 154 SASS)
constexpr int kFastThreads = 64;
constexpr int kFastMinBlocks = 9;
constexpr int kFixWarps = 148 * 4;     // warps of a global-ring (fix-up) launch
constexpr int kGreedyTableWords = 256;   // k_greedy_fast per-warp parameter table: [F, D][32 lanes] int4
// k_greedy_fast: 12 two-warp blocks per SM (6 warps per scheduler) fit its 9 KB per warp; the bound
// caps registers at 85 (78 used)
constexpr int kGreedyMinBlocks = 12;

// k_sim32 shared-memory layout, in 32-bit words (host and device compute it the same way).
// Block header: the per-code uniform table U (8 int4) and -- when every item uses one instance --
// the cost table tabA [4 codes][32 lanes] int4.  Per warp: the F and D arrival rings [R][32] each,
// two plan buffers of (words + 1) rows, a store-sink row, the zero row, 2 mbarriers, 2 x 32 link
// clocks, tabA unless the block holds it, and with a timeline a [16][32] start-tick staging ring.
struct Sim32Layout {
  int uni, rings, plan, dum, zero, bars, link, tabA, stage, per_warp, hdr;
};
__host__ __device__ inline Sim32Layout sim32_layout(int R, int plan_words, bool shared_tab, bool timeline) {
  Sim32Layout L;
  L.uni = 0;                             // block-relative
  L.rings = 0;
  L.plan = 2 * R * 32;
  L.dum = L.plan + 2 * (plan_words + 1) * 32;
  L.zero = L.dum + 32;
  L.bars = L.zero + 32;                  // 8-B aligned: every region above is a multiple of 32 words
  L.link = L.bars + 4;
  int w = L.link + 64;
  if (shared_tab) {
    L.tabA = 32;                         // block-relative, after U
    L.hdr = 32 + 512;
  } else {
    L.tabA = w;
    w += 512;
    L.hdr = 32;
  }
  L.stage = w;
  if (timeline) w += 512;
  L.per_warp = (w + 3) & ~3;
  return L;
}

// k_chunk32f (chunk_fast.cu) shared-memory layout, in 32-bit words (host and device compute it the same
// way).  Block header (when every item uses instance 0): the per-lane tables T0 [8 entries][32 lanes]
// int4 {duration, memory delta, link bandwidth, latency}, T1 [8][32] int4 {input ring slot-0 address,
// message slot-0 address, link-clock address, count increment} (addresses relative to the warp region),
// U [8] int4 {W-deficit increment, -, -, -}.  Per warp: an mbarrier row; a block of zrows rows whose rows
// the arrival rings F0, F1, D0, D1 [R][32] each (UD: F, D); a block of zrows rows whose rows 0 and R-1
// stay zero (the input of W entries, whose ring slot is 0 or R-1) and which holds the two link-clock
// rows (rows 1 and 2 when R >= 4, else appended); the plan rows (words + 1, the last a padding row); the tables unless the block
// holds them.
constexpr int kChunkFTabWords = 2 * 8 * 32 * 4 + 8 * 4;
constexpr int kChunkFThreads = 128;
#ifndef CHUNKF_2C_THREADS
// Wave / Loop: 12-warp blocks, 2 per SM (the shared table amortized over 12 warps; 24 resident warps
// at <= 80 registers): +1.6% Wave, +0.7% Loop over 4-warp blocks; 6-warp blocks: -11%
#define CHUNKF_2C_THREADS 384
#endif
constexpr int kChunkF2CThreads = CHUNKF_2C_THREADS;
constexpr int kChunkFMinBlocks = 5;
struct ChunkFLayout {
  int hdr, bars, zero, zrows, lk, rings, plan, stage, tab, per_warp;
};
// timeline (UD): a [16][32] staging ring of start ticks after the plan rows
#ifndef CHUNKF_WBS
#define CHUNKF_WBS 1   // UD: 1 KB-aligned warp regions, ring slot offsets OR-ed into the warp base (R <= 8)
#endif
__host__ __device__ inline ChunkFLayout chunkf_layout(int R, int words, bool shared_tab, int rings, bool timeline = false) {
  ChunkFLayout L;
  L.hdr = shared_tab ? kChunkFTabWords : 0;
  L.bars = 0;
  L.rings = 32;
  L.zero = L.rings + rings * R * 32;
  L.zrows = R >= 4 ? R : R + 2;
  L.lk = R >= 4 ? L.zero + 32 : L.zero + R * 32;
  L.plan = L.zero + L.zrows * 32;
  int w = L.plan + (words + 1) * 32;
  L.stage = w;
  if (timeline) w += 16 * 32;
  L.tab = shared_tab ? -1 : w;
  if (!shared_tab) w += kChunkFTabWords;
  if (CHUNKF_WBS && rings == 2) {                 // UD (chunk_fast.cu: warp base | slot offset)
    L.hdr = (L.hdr + 255) & ~255;
    w = (w + 255) & ~255;
  }
  L.per_warp = w;
  return L;
}
int launch_chunkf(int pattern, bool timeline, const Args& a, int blocks, int threads, size_t smem, void* stream);
int chunkf_blocks_per_sm(int pattern, int threads, size_t smem, bool timeline = false);
// the sweep's static candidates (GPipe / 1F1B / ZB-H1) on k_chunk32f<UD, grid>: plans from a library
// of [3 kinds][n_pp][n_mb] plans of `words` words built per sweep call (k_plan_library)
struct PlanLibDims {
  int pp[8], mb[8], n_pp, n_mb, words;
};
int launch_plan_library(const PlanLibDims& d, uint32_t* lib, void* stream);
int launch_chunkf_grid(const Args& a, int blocks, int threads, size_t smem, void* stream);
int chunkf_grid_blocks_per_sm(int threads, size_t smem);

}  // namespace cpk
