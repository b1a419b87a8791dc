// abi.cpp -- host side of the C ABI declared in include/crosspipe.h.
// Descriptor validation, launch geometry (lane-segment width, arrival-ring size,
// occupancy-sized persistent grids), workspace layout, the overflow fix-up pass,
// cost-balanced sweep partition, SI -> tick quantization and the host validator.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cstdint>
#include <mutex>
#include <vector>

#include "crosspipe.h"
#include "engine.h"
#include "grid_synth.cuh"


namespace {

// experiments only: CP_NO_FAST=1 routes everything through the generic engine
bool getenv_nofast() { const char* v = std::getenv("CP_NO_FAST"); return v && v[0] == '1'; }

constexpr size_t kCtrlBytes = 256;
constexpr size_t kMaxSmemPerBlock = 227 * 1024;

int lg2_ceil(long long x) {
  int l = 0;
  while ((1LL << l) < x) ++l;
  return l;
}

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// Ring slots needed by items: min(n_mb, in-flight F bound); the memory argument
// bounds every producer->consumer lead by floor(m_lim/m_f).
int ring_slots_for(const cp_instances* in) {
  long long r = in->ring_hint > 0 ? in->ring_hint : in->max_mb;
  r = std::max(1LL, std::min<long long>(r, in->max_mb));
  return (int)r;
}

int big_ring_slots(const cp_instances* in) { return std::max(1, std::min(in->max_mb, CP_MAX_MB)); }

// fast paths use occupancy backpressure: the rings only need to absorb the producer->consumer skew
// of the round-synchronous evaluation (measured <= 10 on config 4), not the worst-case lead.  8
// slots: a block that finds its consumer's ring full just waits (exact), and the smaller per-warp
// shared memory keeps more warps resident (measured: config 4 +4%, Wave +8% over 16 slots)
int fast_ring_slots(const cp_instances* in) {
  int cap = 8;
  if (const char* v = std::getenv("CP_RING_CAP")) cap = std::max(1, std::atoi(v));   // experiments
  // a power of two: the n_sub == 1 rounds address ring slots as count & (R - 1)
  return 1 << lg2_ceil(std::min(ring_slots_for(in), cap));
}

constexpr int kPlanCapWords = 64;        // plans up to 1024 entries per stage row are staged in smem

size_t ring_bytes_per_warp(int slots) { return (size_t)2 * slots * 32 * 4; }

size_t ws_sim_greedy(const cp_instances* in, long long n_items) {
  return kCtrlBytes + align256(sizeof(int32_t) * (size_t)std::max(1LL, n_items)) +
         (size_t)cpk::kFixWarps * ring_bytes_per_warp(big_ring_slots(in));
}

// per-warp shared memory (32-bit words): rings + plan buffers + 2 mbarriers
int smem_words(bool ring_global, int slots, int plan_words, int nbuf, bool tma) {
  int w = ring_global ? 0 : 2 * slots * 32;
  w += nbuf * plan_words * 32;
  if (tma) w += 4;
  return (w + 3) & ~3;                       // 16-B aligned per warp
}

int check_instances(const cp_instances* in) {
  if (!in || !in->inst || in->n < 1) return CP_EINVAL;
  if (in->max_pp < 1 || in->max_mb < 1) return CP_EINVAL;
  if (in->max_pp > CP_MAX_STAGES) return CP_EUNSUPPORTED;
  if (in->max_mb > CP_MAX_MB) return CP_EUNSUPPORTED;
  return CP_OK;
}

// Blocks per SM such that the resident warps split evenly over the SM's four sub-partitions
// (warp schedulers).  The fast paths hand work out statically (grid stride), so with an uneven
// split the schedulers holding one warp more finish last and the others idle at the end
// (measured on k_sim32, 2-warp blocks: 11 per SM 50.8 M, 10 per SM 54.4 M evals/s).
int smsp_balanced(int bps, int wpb) {
  if (std::getenv("CP_NO_SMSP_BALANCE")) return bps;
  for (int b = bps; b >= 1; --b)
    if ((b * wpb) % 4 == 0) return b;
  return bps;
}

int launch_pass(cpk::Mode mode, bool ring_global, cpk::Args& a, long long n_tasks, int nseg, void* stream) {
  const int sms = cpk::device_sm_count();
  const int nbuf = a.tma ? 2 : 1;
  a.smem_words_per_warp = smem_words(ring_global, a.ring_slots, a.plan_words, nbuf, a.tma != 0);
  const size_t per_warp = (size_t)a.smem_words_per_warp * 4;
  if (ring_global) {
    const int wpb = 4;
    const size_t smem = per_warp * wpb;
    if (smem > kMaxSmemPerBlock) return CP_EUNSUPPORTED;
    return cpk::launch_engine(mode, true, a, cpk::kFixWarps / wpb, 32 * wpb, smem, stream) == cudaSuccess ? CP_OK
                                                                                                      : CP_ECUDA;
  }
  const int wpb = per_warp * 2 <= kMaxSmemPerBlock ? 2 : 1;
  const size_t smem = per_warp * wpb;
  if (smem > kMaxSmemPerBlock) return CP_EUNSUPPORTED;
  const int threads = 32 * wpb;
  const int bps = smsp_balanced(cpk::engine_blocks_per_sm(mode, false, threads, smem, a.t_start != nullptr), wpb);
  const long long need = (n_tasks + (long long)nseg * wpb - 1) / ((long long)nseg * wpb);
  const int blocks = (int)std::max(1LL, std::min<long long>(need, (long long)sms * bps));
  return cpk::launch_engine(mode, false, a, blocks, threads, smem, stream) == cudaSuccess ? CP_OK : CP_ECUDA;
}

int run_engine(cpk::Mode mode, const cp_instances* in, const cp_schedules* sc, const cp_results* res, void* ws,
               size_t ws_bytes, void* stream) {
  const long long n = sc->n;
  if (ws_bytes < ws_sim_greedy(in, n) || !ws) return CP_EWORKSPACE;
  cpk::Args a;
  std::memset(&a, 0, sizeof(a));
  a.inst = in->inst;
  a.inst_of = sc->inst_of;
  a.n_inst = in->n;
  a.n_items = (int32_t)n;
  a.seg_lg = lg2_ceil(in->max_pp);
  a.ops = sc->ops;
  a.len = sc->len;
  a.stage_stride = sc->stage_stride;
  a.words = sc->words;
  a.makespan = res->makespan;
  a.peak_mem = res->peak_mem;
  a.status = res->status;
  a.stage_stats = res->stage_stats;
  a.t_start = res->t_start;
  a.len_stride = res->len_stride;
  a.best_key = reinterpret_cast<unsigned long long*>(res->best_key);
  a.index_base = res->index_base;
  char* base = static_cast<char*>(ws);
  a.ovf_count = reinterpret_cast<int32_t*>(base);
  a.ovf_list = reinterpret_cast<int32_t*>(base + kCtrlBytes);
  int32_t* rings = reinterpret_cast<int32_t*>(base + kCtrlBytes + align256(sizeof(int32_t) * (size_t)std::max(1LL, n)));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (cudaMemsetAsync(a.ovf_count, 0, kCtrlBytes, st) != cudaSuccess) return CP_ECUDA;

  const int nseg = 32 >> a.seg_lg;
  a.plan_words = sc->words <= kPlanCapWords ? sc->words : 0;
#ifndef CP_DEBUG
  // k_sim32 with a timeline writes each lane's start ticks 8 at a time (two 16-B stores): rows must be
  // 32-B aligned and hold every entry a valid row can have
  const bool tl_vec = !res->t_start || (res->len_stride % 8 == 0 && res->len_stride >= 16 * sc->words &&
                                        (reinterpret_cast<uintptr_t>(res->t_start) & 31) == 0);
  if (mode == cpk::MODE_SIM && nseg == 1 && sc->stage_stride == 32 && a.plan_words > 0 && tl_vec &&
      !getenv_nofast()) {
    // fast path (sim32.cu): warp = one item, TMA double-buffered plan rows with a spare row.  When every
    // item uses instance 0, a 4-warp block shares one cost / increment table (24 resident warps).
    const bool tl = res->t_start != nullptr;
    // The first pass is k_chunk32f (chunk_fast.cu, byte-count readiness, dynamic item counter; with a
    // timeline its start ticks are staged in shared memory and written 32 B per lane); it lists the
    // items it does not finish for the exact second pass below (k_sim32).  CP_CHUNKF_OFF=1: k_sim32 for
    // both passes.
    bool first_done = false;
    if (!std::getenv("CP_CHUNKF_OFF")) {
      // W readiness needs R >= 2; the UD kernel's base | slot addressing needs R <= 8 (CHUNKF_WBS)
      a.ring_slots = std::max(2, CHUNKF_WBS ? std::min(8, fast_ring_slots(in)) : fast_ring_slots(in));
      a.shared_tab = (!sc->inst_of && in->n == 1) ? 1 : 0;
      const cpk::ChunkFLayout L = cpk::chunkf_layout(a.ring_slots, sc->words, a.shared_tab != 0, 2, tl);
      const int wpb = cpk::kChunkFThreads / 32, threads = cpk::kChunkFThreads;
      const size_t smem = ((size_t)L.hdr + (size_t)wpb * L.per_warp) * 4;
      if (smem <= kMaxSmemPerBlock) {
        int bps = smsp_balanced(cpk::chunkf_blocks_per_sm(CP_PATTERN_UD, threads, smem, tl), wpb);
        if (const char* v = std::getenv("CP_CHUNKF_BPS")) bps = std::max(1, std::min(bps, std::atoi(v)));   // experiments
        const long long need = (n + wpb - 1) / wpb;
        const int blocks = (int)std::max(1LL, std::min<long long>(need, (long long)cpk::device_sm_count() * bps));
        a.work_counter = std::getenv("CP_CHUNKF_STATIC") ? nullptr : reinterpret_cast<int32_t*>(base + 128);
        if (cpk::launch_chunkf(CP_PATTERN_UD, tl, a, blocks, threads, smem, stream) != cudaSuccess) return CP_ECUDA;
        a.work_counter = nullptr;
        first_done = true;
      }
    }
    a.ring_slots = fast_ring_slots(in);
    a.shared_tab = (!sc->inst_of && in->n == 1 && !std::getenv("CP_SIM32_NOSHARE")) ? 1 : 0;
    const cpk::Sim32Layout L1 = cpk::sim32_layout(a.ring_slots, a.plan_words, a.shared_tab != 0, tl);
    a.smem_words_per_warp = L1.per_warp;
    const int wpb = a.shared_tab ? 4 : 2, threads = 32 * wpb;
    const size_t smem = ((size_t)L1.hdr + (size_t)wpb * L1.per_warp) * 4;
    if (first_done || smem <= kMaxSmemPerBlock) {
      int bps = smsp_balanced(cpk::sim32_blocks_per_sm(tl, threads, smem), wpb);
      if (const char* v = std::getenv("CP_SIM32_BPS")) bps = std::max(1, std::min(bps, std::atoi(v)));   // experiments
      const long long need = (n + wpb - 1) / wpb;
      const int blocks = (int)std::max(1LL, std::min<long long>(need, (long long)cpk::device_sm_count() * bps));
      if (!first_done) {
        // the timeline first pass takes its items from the workspace counter (zeroed above)
        a.work_counter = std::getenv("CP_SIM32_STATIC") ? nullptr : reinterpret_cast<int32_t*>(base + 128);
        if (cpk::launch_sim32(tl, a, blocks, threads, smem, stream) != cudaSuccess) return CP_ECUDA;
        a.work_counter = nullptr;
      }
      // Items that stalled on a full 8-slot ring (cyclic backpressure) are re-run from the
      // overflow list by the same kernel with rings of R > n_mb slots, where no ring can fill (every
      // producer -> consumer lead is <= n_mb); only when such rings exceed shared memory does the
      // generic engine with global-memory rings take them.  An empty list costs one short launch.
      a.from_list = 1;
      a.ring_slots = 1 << lg2_ceil((long long)in->max_mb + 1);
      a.shared_tab = 0;
      const cpk::Sim32Layout L2 = cpk::sim32_layout(a.ring_slots, a.plan_words, false, tl);
      const size_t smem2 = ((size_t)L2.hdr + L2.per_warp) * 4;
      if (smem2 <= kMaxSmemPerBlock && !std::getenv("CP_SIM32_ENGINE_FIXUP")) {
        a.smem_words_per_warp = L2.per_warp;
        const int bps2 = cpk::sim32_blocks_per_sm(tl, 32, smem2);
        if (cpk::launch_sim32(tl, a, cpk::device_sm_count() * std::max(1, bps2), 32, smem2, stream) != cudaSuccess)
          return CP_ECUDA;
        return cudaGetLastError() == cudaSuccess ? CP_OK : CP_ECUDA;
      }
      a.tma = 0;
      a.ring_slots = big_ring_slots(in);
      a.ring_g = rings;
      const int rc = launch_pass(mode, true, a, n, nseg, stream);
      if (rc) return rc;
      return cudaGetLastError() == cudaSuccess ? CP_OK : CP_ECUDA;
    }
  }
  if (mode == cpk::MODE_GREEDY && !res->t_start && !getenv_nofast()) {
    // fast path (greedy_fast.cu): compile-time segment width, rings only in shared memory
    const int Wd = in->max_pp <= 8 ? 8 : (in->max_pp <= 16 ? 16 : 32);
    // lead bound (greedy gates on nF - nD, cheaper than occupancy); a power of two (count-addressed slots)
    a.ring_slots = 1 << lg2_ceil(ring_slots_for(in));
    a.smem_words_per_warp = (cpk::kGreedyTableWords + 2 * a.ring_slots * 32 + 3) & ~3;
    const size_t per_warp = (size_t)a.smem_words_per_warp * 4;
    if (per_warp * 2 <= kMaxSmemPerBlock) {
      const int wpb = 2, threads = 64;
      const size_t smem = per_warp * wpb;
      const int bps = smsp_balanced(cpk::greedy_fast_blocks_per_sm(Wd, false, threads, smem), wpb);
      const long long segs = (long long)(32 / Wd) * wpb;
      const long long need = (n + segs - 1) / segs;
      const int blocks = (int)std::max(1LL, std::min<long long>(need, (long long)cpk::device_sm_count() * bps));
      // instances from a counter in the workspace control block (zeroed above): segments that finish
      // early take more, instead of a static stride leaving a tail
      a.work_counter = std::getenv("CP_GREEDY_STATIC") ? nullptr : reinterpret_cast<int32_t*>(base + 128);
      if (cpk::launch_greedy_fast(Wd, false, a, blocks, threads, smem, stream) != cudaSuccess) return CP_ECUDA;
      a.work_counter = nullptr;
      a.from_list = 1;
      a.tma = 0;
      a.plan_words = sc->words <= kPlanCapWords ? sc->words : 0;
      a.ring_slots = big_ring_slots(in);
      a.ring_g = rings;
      const int rc = launch_pass(mode, true, a, n, nseg, stream);
      if (rc) return rc;
      return cudaGetLastError() == cudaSuccess ? CP_OK : CP_ECUDA;
    }
  }
#endif
  // fast pass: shared-memory rings sized to the in-flight bound, occupancy-sized persistent grid
  a.ring_slots = ring_slots_for(in);
  a.tma = (mode == cpk::MODE_SIM && nseg == 1 && sc->stage_stride == 32 && a.plan_words > 0) ? 1 : 0;
  int rc = launch_pass(mode, false, a, n, nseg, stream);
  if (rc == CP_EUNSUPPORTED) {
    // rings too large for shared memory: single global-ring pass over every item
    a.tma = 0;
    a.ring_slots = big_ring_slots(in);
    a.ring_g = rings;
    rc = launch_pass(mode, true, a, n, nseg, stream);
    if (rc) return rc;
    return cudaGetLastError() == cudaSuccess ? CP_OK : CP_ECUDA;
  }
  if (rc) return rc;
  // fix-up pass over the overflow list (items whose lead exceeded R) with n_mb-slot global rings
  a.from_list = 1;
  a.tma = 0;
  a.ring_slots = big_ring_slots(in);
  a.ring_g = rings;
  rc = launch_pass(mode, true, a, n, nseg, stream);
  if (rc) return rc;
  return cudaGetLastError() == cudaSuccess ? CP_OK : CP_ECUDA;
}

// grid helpers ---------------------------------------------------------------
long long grid_points(const cp_grid* g) {
  return (long long)g->n_pp_n * g->n_mb_n * g->n_lat * g->n_bw * g->n_mem * g->n_dp;
}

int check_grid(const cp_grid* g) {
  if (!g) return CP_EINVAL;
  if (g->n_pp_n < 1 || g->n_pp_n > 8 || g->n_mb_n < 1 || g->n_mb_n > 8) return CP_EINVAL;
  if (g->n_lat < 1 || g->n_lat > CP_GRID_MAX_AXIS || g->n_bw < 1 || g->n_bw > CP_GRID_MAX_AXIS) return CP_EINVAL;
  if (g->n_mem < 1 || g->n_mem > CP_GRID_MAX_SMALL || g->n_dp < 1 || g->n_dp > CP_GRID_MAX_SMALL) return CP_EINVAL;
  for (int i = 0; i < g->n_pp_n; ++i) {
    if (g->n_pp_vals[i] < 1) return CP_EINVAL;
    if (g->n_pp_vals[i] > CP_MAX_STAGES) return CP_EUNSUPPORTED;
  }
  for (int i = 0; i < g->n_mb_n; ++i) {
    if (g->n_mb_vals[i] < 1) return CP_EINVAL;
    if (g->n_mb_vals[i] > CP_MAX_MB) return CP_EUNSUPPORTED;
  }
  for (int i = 0; i < g->n_lat; ++i) if (g->lat[i] < 0) return CP_EINVAL;
  for (int i = 0; i < g->n_bw; ++i) if (g->bw[i] < 0) return CP_EINVAL;
  for (int i = 0; i < g->n_mem; ++i) if (g->mlim_x1000[i] < 0) return CP_EINVAL;
  for (int i = 0; i < g->n_dp; ++i) if (g->tdp[i] < 0) return CP_EINVAL;
  // Every point's synthesized instance must be valid: a malformed grid (a p beyond the base
  // record's stages, bad memory deltas, a budget below m_f or beyond int32) is an API error, not
  // "no feasible candidate".  Validity depends on (p, memory scale) only -- m, latency, bandwidth
  // and DP time enter through the checks above -- so one synthesized record per pair is checked
  // (grid_synth.cuh, the kernels' own synthesis).  The int32 horizon guard (CPI_OVERFLOW) stays
  // per point: such points get KEY_OVER.
  for (int ip = 0; ip < g->n_pp_n; ++ip)
    for (int ix = 0; ix < g->n_mem; ++ix) {
      const long long point = (((long long)ip * g->n_mb_n * g->n_lat * g->n_bw) * g->n_mem + ix) * g->n_dp;
      cp_inst_v1 r;
      std::memset(&r, 0, sizeof(r));
      const int p = g->n_pp_vals[ip];
      r.n_pp = (uint8_t)p;
      r.n_mb = (uint16_t)g->n_mb_vals[0];
      r.n_sub = 1;
      r.flags = g->base.flags & 1;
      r.version = 1;
      for (int s = 0; s < p; ++s) {
        if (((long long)g->mlim_x1000[ix] * p * g->base.m_f[s] + 500) / 1000 > INT32_MAX) return CP_EINVAL;
        const cpk::GridLane L = cpk::grid_lane(*g, point, s);
        r.t_f[s] = L.tf; r.t_d[s] = L.td; r.t_w[s] = L.tw;
        r.m_f[s] = L.mf; r.m_d[s] = L.md; r.m_w[s] = L.mw; r.m_lim[s] = L.mlim;
        r.t_dp[s] = L.tdp; r.t_ag[s] = L.tag;
      }
      if (cp_validate_instance(&r, nullptr, 0) == CPI_BAD_INSTANCE) return CP_EINVAL;
    }
  return CP_OK;
}

// ring slots needed by the points of one p-class: max over (m, M_L) of
// min(m, max_s floor(m_lim[s] / m_f[s])) -- greedy and feasible static plans never exceed it
int sweep_ring_slots(const cp_grid* g, int p) {
  long long r = 1;
  for (int im = 0; im < g->n_mb_n; ++im)
    for (int ix = 0; ix < g->n_mem; ++ix) {
      long long need = 1;
      for (int s = 0; s < p; ++s) {
        const long long mf = std::max(1, g->base.m_f[s]);
        const long long mlim = ((long long)g->mlim_x1000[ix] * p * mf + 500) / 1000;
        need = std::max(need, mlim / mf);
      }
      r = std::max(r, std::min<long long>(need, g->n_mb_vals[im]));
    }
  return (int)r;
}

// An engine sweep pass whose rings do not fit one block's shared memory (n_mb and M_L beyond ~900
// in-flight microbatches) runs with global-memory rings in the workspace instead: one region per
// p-class, since the classes run concurrently.  Returns that class's bytes (0 = shared memory).
size_t sweep_class_ring_bytes(const cp_grid* g, int ip) {
  const int slots = sweep_ring_slots(g, g->n_pp_vals[ip]);
  if ((size_t)smem_words(false, slots, 0, 1, false) * 4 <= kMaxSmemPerBlock) return 0;
  return align256((size_t)cpk::kFixWarps * ring_bytes_per_warp(slots));
}

// The static candidates (GPipe / 1F1B / ZB-H1) run on k_chunk32f<UD, grid> when every n_mb of the
// grid fits its count bytes; their plans come from a library built per call, after the ring regions.
constexpr unsigned kStaticCands = (1u << CP_PLAN_GPIPE) | (1u << CP_PLAN_1F1B) | (1u << CP_PLAN_ZBH1);
bool sweep_static_fast(const cp_grid* g) {
  if (!(g->cand_mask & kStaticCands) || getenv_nofast() || std::getenv("CP_SWEEP_STATIC_ENGINE")) return false;
  for (int i = 0; i < g->n_mb_n; ++i)
    if (g->n_mb_vals[i] > 255) return false;
  return true;
}
int plan_lib_words(const cp_grid* g) {
  int mx = 1;
  for (int i = 0; i < g->n_mb_n; ++i) mx = std::max(mx, g->n_mb_vals[i]);
  return (3 * mx + 15) / 16;                   // ZB-H1 rows (3m) are the longest
}
size_t plan_lib_bytes(const cp_grid* g) {
  // 8 task counters (one per p-class), then the plans
  return sweep_static_fast(g) ? align256(64 + (size_t)3 * g->n_pp_n * g->n_mb_n * plan_lib_words(g) * 32 * 4) : 0;
}

// Task counters of the long-task greedy launches (3 ring tiers per p-class), after the plan library.
constexpr size_t kLongCtrBytes = 256;
size_t sweep_ws_bytes(const cp_grid* g) {
  size_t b = kCtrlBytes;
  for (int ip = 0; ip < g->n_pp_n; ++ip) b += sweep_class_ring_bytes(g, ip);
  return b + plan_lib_bytes(g) + kLongCtrBytes;
}

long long point_cost(const cp_grid* g, int i_pp, int i_mb) {
  static const int units[CP_N_CAND] = {2, 2, 3, 4, 6, 3};   // entries per microbatch: 2m GPipe/1F1B, (2+n_sub)m greedy, 3m ZB-H1
  long long u = 0;
  for (int c = 0; c < CP_N_CAND; ++c)
    if ((g->cand_mask >> c) & 1u) u += units[c];
  return (long long)g->n_pp_vals[i_pp] * g->n_mb_vals[i_mb] * std::max(1LL, u);
}

}  // namespace

extern "C" {

uint32_t cp_abi_version(void) { return CP_ABI_VERSION; }

const char* cp_status_string(int32_t code) {
  switch (code) {
    case CP_OK: return "ok";
    case CP_EINVAL: return "invalid argument / descriptor";
    case CP_EUNSUPPORTED: return "unsupported shape (p > 32, n_mb > 1024, two-chunk n_mb > 256, rows beyond shared memory)";
    case CP_ECUDA: return "CUDA launch error";
    case CP_EWORKSPACE: return "workspace too small";
    case CPI_DEADLOCK: return "deadlock: plan cannot complete";
    case CPI_MEM_EXCEEDED: return "memory limit exceeded";
    case CPI_BAD_PLAN: return "bad plan";
    case CPI_BAD_INSTANCE: return "bad instance";
    case CPI_OVERFLOW: return "exceeds int32 horizon / GPU size limits";
    default: return code > 0 ? "multiple item status bits" : "unknown error";
  }
}

size_t cp_workspace_bytes(int32_t which, const void* desc, int64_t n_items) {
  if (which == 2) {
    const cp_grid* g = static_cast<const cp_grid*>(desc);
    return g && check_grid(g) == CP_OK ? sweep_ws_bytes(g) : kCtrlBytes;
  }
  if (which != 0 && which != 1) return 0;
  const cp_instances* in = static_cast<const cp_instances*>(desc);
  if (!in || n_items < 0) return 0;
  return ws_sim_greedy(in, n_items);
}

// Two-chunk plans, Wave (reading Q32) or Loop (Q33): k_chunk32, one item per warp.  A first pass with small occupancy-gated
// rings; items that stall on a full ring are re-run by a second pass with rings of n_mb slots.
int run_wave(const cp_instances* in, const cp_schedules* sc, const cp_results* res, void* ws, size_t ws_bytes,
             void* stream) {
  const long long n = sc->n;
  if (in->max_mb > 256 || sc->stage_stride < in->max_pp) return CP_EUNSUPPORTED;
  if (ws_bytes < ws_sim_greedy(in, n) || !ws) return CP_EWORKSPACE;
  cpk::Args a;
  std::memset(&a, 0, sizeof(a));
  a.chunk_pattern = sc->pattern;
  a.inst = in->inst;
  a.inst_of = sc->inst_of;
  a.n_inst = in->n;
  a.n_items = n;
  a.ops = sc->ops;
  a.len = sc->len;
  a.stage_stride = sc->stage_stride;
  a.words = sc->words;
  a.makespan = res->makespan;
  a.peak_mem = res->peak_mem;
  a.status = res->status;
  a.stage_stats = res->stage_stats;
  a.t_start = res->t_start;
  a.len_stride = res->len_stride;
  a.best_key = reinterpret_cast<unsigned long long*>(res->best_key);
  a.index_base = res->index_base;
  char* base = static_cast<char*>(ws);
  a.ovf_count = reinterpret_cast<int32_t*>(base);
  a.ovf_list = reinterpret_cast<int32_t*>(base + kCtrlBytes);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (cudaMemsetAsync(a.ovf_count, 0, kCtrlBytes, st) != cudaSuccess) return CP_ECUDA;
  const int sms = cpk::device_sm_count();
  int first_pass = 0;
#ifndef CP_DEBUG
  // First pass on k_chunk32f (chunk_fast.cu) for stage_stride-32 plans that fit shared memory: it
  // finishes every n_sub = 1, n_mb <= 127 item that does not stall on its small rings and lists the
  // rest; k_chunk32 then evaluates the listed items exactly (pass 1 below).
  if (sc->stage_stride == 32 && sc->words <= kPlanCapWords && !getenv_nofast() && !std::getenv("CP_CHUNKF_OFF")) {
    const bool tl = res->t_start != nullptr;
    a.from_list = 0;
    a.ring_slots = std::max(2, std::min(64, fast_ring_slots(in)));   // W readiness needs R >= 2; R << 24 fits
    a.plan_words = sc->words;
    a.shared_tab = (!sc->inst_of && in->n == 1) ? 1 : 0;
    const cpk::ChunkFLayout L = cpk::chunkf_layout(a.ring_slots, sc->words, a.shared_tab != 0, 4);
    const int wpb = cpk::kChunkF2CThreads / 32, threads = cpk::kChunkF2CThreads;
    const size_t smem = ((size_t)L.hdr + (size_t)wpb * L.per_warp) * 4;
    if (smem <= kMaxSmemPerBlock) {
      int bps = smsp_balanced(cpk::chunkf_blocks_per_sm(sc->pattern, threads, smem, tl), wpb);
      if (const char* v = std::getenv("CP_CHUNKF_BPS")) bps = std::max(1, std::min(bps, std::atoi(v)));   // experiments
      const long long need = (n + wpb - 1) / wpb;
      const int blocks = (int)std::max(1LL, std::min<long long>(need, (long long)sms * bps));
      // dynamic item counter in the workspace control block (zeroed with the overflow count above)
      a.work_counter = std::getenv("CP_CHUNKF_STATIC") ? nullptr : reinterpret_cast<int32_t*>(base + 128);
      if (cpk::launch_chunkf(sc->pattern, tl, a, blocks, threads, smem, stream) != cudaSuccess) return CP_ECUDA;
      a.work_counter = nullptr;
      first_pass = 1;
    }
    a.shared_tab = 0;
  }
#endif
  for (int pass = first_pass; pass < 2; ++pass) {
    a.from_list = pass;
    a.ring_slots = pass == 0 ? fast_ring_slots(in) : 1 << lg2_ceil(in->max_mb);
    a.plan_words = sc->words + 1;                       // one spare row: finished lanes read past their row
    a.smem_words_per_warp = (2048 + 4 * a.ring_slots * 32 + 32 + a.plan_words * 32 + 64 + 512 + 3) & ~3;   // tables, rings, zero row, plan, link clocks, increments
    const size_t per_warp = (size_t)a.smem_words_per_warp * 4;
    if (per_warp > kMaxSmemPerBlock) return CP_EUNSUPPORTED;
    const int wpb = per_warp * 2 <= kMaxSmemPerBlock ? 2 : 1, threads = 32 * wpb;
    const size_t smem = per_warp * wpb;
    const int bps = smsp_balanced(cpk::wave32_blocks_per_sm(threads, smem), wpb);
    const long long need = pass == 0 ? (n + wpb - 1) / wpb : (long long)cpk::kFixWarps / wpb;
    const int blocks = (int)std::max(1LL, std::min<long long>(need, (long long)sms * bps));
    if (cpk::launch_wave32(a, blocks, threads, smem, stream) != cudaSuccess) return CP_ECUDA;
  }
  return cudaGetLastError() == cudaSuccess ? CP_OK : CP_ECUDA;
}

int32_t cp_simulate(const cp_instances* in, const cp_schedules* sc, const cp_results* res, void* ws, size_t ws_bytes,
                    void* stream) {
  int rc = check_instances(in);
  if (rc) return rc;
  if (!sc || !res || sc->n < 0 || !sc->ops || !sc->len || !res->makespan || !res->status) return CP_EINVAL;
  if (sc->stage_stride < in->max_pp || sc->words < 1 || (res->t_start && res->len_stride < 1)) return CP_EINVAL;
  if (!sc->inst_of && in->n != 1 && in->n < sc->n) return CP_EINVAL;
  if (sc->pattern < CP_PATTERN_UD || sc->pattern > CP_PATTERN_LOOP) return CP_EINVAL;
  if (sc->n == 0) return CP_OK;
  if (sc->pattern != CP_PATTERN_UD) return run_wave(in, sc, res, ws, ws_bytes, stream);
  return run_engine(cpk::MODE_SIM, in, sc, res, ws, ws_bytes, stream);
}

int32_t cp_build_static(int32_t kind, const cp_instances* in, const cp_schedules* out, void* stream) {
  if (kind != CP_PLAN_GPIPE && kind != CP_PLAN_1F1B && kind != CP_PLAN_ZBH1 && kind != CP_PLAN_IV1F1B &&
      kind != CP_PLAN_ZBV)
    return CP_EINVAL;
  int rc = check_instances(in);
  if (rc) return rc;
  if (!out || out->n < 0 || !out->ops || !out->len || out->words < 1) return CP_EINVAL;
  if (out->stage_stride < in->max_pp) return CP_EINVAL;
  if (!out->inst_of && in->n != 1 && in->n < out->n) return CP_EINVAL;
  const long long per_mb = kind == CP_PLAN_ZBH1 ? 3 : (kind == CP_PLAN_IV1F1B ? 4 : (kind == CP_PLAN_ZBV ? 6 : 2));
  const bool nibbles = kind == CP_PLAN_IV1F1B || kind == CP_PLAN_ZBV;
  if ((nibbles ? 8LL : 16LL) * out->words < per_mb * in->max_mb) return CP_EINVAL;
  if (out->n == 0) return CP_OK;
  return cpk::launch_build_static(kind, in->inst, in->n, out->inst_of, out->n, out->stage_stride, out->words, out->ops,
                                  out->len, stream) == cudaSuccess ? CP_OK : CP_ECUDA;
}

size_t cp_exact_workspace_bytes(int32_t n, int32_t cap) {
  return n < 1 || cap < 1 ? 0 : cpk::exact_ws_bytes(n, cap);
}

int32_t cp_exact(const cp_instances* in, const cp_schedules* out, const int32_t* upper, int32_t* makespan,
                 int32_t* status, int32_t cap, int64_t max_plans, void* ws, size_t ws_bytes, void* stream) {
  int rc = check_instances(in);
  if (rc) return rc;
  if (!out || out->n != in->n || out->inst_of || !out->ops || !out->len || !makespan || !status) return CP_EINVAL;
  if (out->stage_stride < in->max_pp || out->words < 1 || 16LL * out->words < 3LL * std::min(in->max_mb, 8))
    return CP_EINVAL;
  if (cap < 1 || max_plans < 1 || max_plans >= (1LL << 52)) return CP_EINVAL;
  if (in->n == 0) return CP_OK;
  if (!ws || ws_bytes < cpk::exact_ws_bytes(in->n, cap)) return CP_EWORKSPACE;
  return cpk::launch_exact(in->inst, in->n, cap, max_plans, upper, ws, out->stage_stride, out->words, out->ops,
                           out->len, makespan, status, stream) == cudaSuccess ? CP_OK : CP_ECUDA;
}

static void bnb_dims(const cp_instances* in, int* lmax, int* vlen) {
  const int p = std::min(in->max_pp, cpk::kBnbMaxP), m = std::min(in->max_mb, cpk::kBnbMaxM);
  *lmax = 3 * p * m;
  *vlen = 3 * p - 1 + 2 * (p - 1) * m;
}

size_t cp_exact_bnb_workspace_bytes(const cp_instances* in, int32_t front_cap, int64_t table_entries) {
  if (!in || in->n < 1 || front_cap < 1 || table_entries < 1) return 0;
  int lmax, vlen;
  bnb_dims(in, &lmax, &vlen);
  return cpk::bnb_layout(in->n, lmax, vlen, front_cap, table_entries).bytes;
}

int32_t cp_exact_bnb(const cp_instances* in, const cp_schedules* out, const int32_t* upper, int32_t* makespan,
                     int32_t* status, int32_t* bound, int64_t* nodes, int32_t budget, int64_t max_nodes,
                     int32_t max_rounds, int32_t front_cap, int64_t table_entries, void* ws, size_t ws_bytes,
                     void* stream) {
  int rc = check_instances(in);
  if (rc) return rc;
  if (!out || out->n != in->n || out->inst_of || !out->ops || !out->len || !makespan || !status) return CP_EINVAL;
  if (out->stage_stride < in->max_pp || out->words < 1 || 16LL * out->words < 3LL * std::min(in->max_mb, cpk::kBnbMaxM))
    return CP_EINVAL;
  if (budget < 1 || max_nodes < 1 || max_rounds < 1 || front_cap < 1 || table_entries < 1 ||
      (table_entries & (table_entries - 1)))
    return CP_EINVAL;
  if (!ws || ws_bytes < cp_exact_bnb_workspace_bytes(in, front_cap, table_entries)) return CP_EWORKSPACE;
  int lmax, vlen;
  bnb_dims(in, &lmax, &vlen);
  return cpk::launch_bnb(in->inst, in->n, upper, lmax, vlen, front_cap, table_entries, budget, max_nodes, max_rounds,
                         ws, out->stage_stride, out->words, out->ops, out->len, makespan, status, bound,
                         reinterpret_cast<long long*>(nodes), stream) == cudaSuccess ? CP_OK : CP_ECUDA;
}

int32_t cp_greedy(const cp_instances* in, const cp_schedules* out, const cp_results* res, void* ws, size_t ws_bytes,
                  void* stream) {
  int rc = check_instances(in);
  if (rc) return rc;
  if (!out || !res || out->n != in->n || out->inst_of || !out->ops || !out->len || !res->makespan || !res->status)
    return CP_EINVAL;
  if (out->stage_stride < in->max_pp || out->words < 1 || (res->t_start && res->len_stride < 1)) return CP_EINVAL;
  return run_engine(cpk::MODE_GREEDY, in, out, res, ws, ws_bytes, stream);
}

// Evaluate a point set: contiguous points [lo, hi) (own_hi == own_lo), or the blocked ownership of
// cp_sweep_shard_rank: slice [own_lo, own_hi) of every (n_pp, n_mb) block of `inner` points.
// Launches go to streams forked from `parent` (one per launch) and joined back to it in join().
// The streams and events are created once per device and reused by later calls (a call that finds
// the pool in use by another host thread creates its own and destroys them at the join).
constexpr int kForkMax = 40;
// Launches take one of three stream-priority bands (0 = the device's greatest priority, 2 = the
// least): when SM resources free up, the block scheduler hands them to pending blocks of the
// higher band first.  The pool holds kForkBand streams per band.
constexpr int kForkBand = kForkMax / 3;
struct ForkPool {
  std::mutex mu;
  int dev = -1;
  cudaEvent_t fork = nullptr, joins[kForkMax] = {};
  cudaStream_t sub[kForkMax] = {};
};
ForkPool g_fork_pool;

inline int band_priority(int band) {
  int least = 0, greatest = 0;
  cudaDeviceGetStreamPriorityRange(&least, &greatest);
  return band == 0 ? greatest : (band == 1 ? (least + greatest) / 2 : least);
}

struct Forker {
  cudaStream_t parent;
  std::unique_lock<std::mutex> lk;
  bool pooled = false;
  cudaEvent_t fork = nullptr, joins[kForkMax] = {};
  cudaStream_t sub[kForkMax] = {};
  int used[3] = {0, 0, 0}, n = 0;                  // pooled: per band; own streams: n
  int own[kForkMax] = {};                          // own streams: indices in use
  bool used_parent = false, forked = false;
  explicit Forker(cudaStream_t p) : parent(p), lk(g_fork_pool.mu, std::try_to_lock) {
    int dev = -1;
    cudaGetDevice(&dev);
    if (lk.owns_lock() && (g_fork_pool.dev == dev || g_fork_pool.dev < 0)) {
      pooled = true;
      if (g_fork_pool.dev < 0) {                    // first call on this device: create the pool
        g_fork_pool.dev = dev;
        cudaEventCreateWithFlags(&g_fork_pool.fork, cudaEventDisableTiming);
        for (int i = 0; i < kForkMax; ++i) {
          cudaStreamCreateWithPriority(&g_fork_pool.sub[i], cudaStreamNonBlocking, band_priority(std::min(2, i / kForkBand)));
          cudaEventCreateWithFlags(&g_fork_pool.joins[i], cudaEventDisableTiming);
        }
      }
      fork = g_fork_pool.fork;
      for (int i = 0; i < kForkMax; ++i) { sub[i] = g_fork_pool.sub[i]; joins[i] = g_fork_pool.joins[i]; }
    }
  }
  ~Forker() { join(); }
  // The fork point is recorded before the first launch, so no launch waits for another.  The first
  // band-2 launch runs on the parent itself (a single-launch call forks nothing).
  bool record_fork() {
    if (forked) return true;
    if (!fork && cudaEventCreateWithFlags(&fork, cudaEventDisableTiming) != cudaSuccess) return false;
    cudaEventRecord(fork, parent);
    forked = true;
    return true;
  }
  cudaStream_t next(int band = 2) {
    if (!record_fork()) return parent;
    if (band == 2 && !used_parent) {
      used_parent = true;
      return parent;
    }
    int i;
    if (pooled) {
      const int lim = band == 2 ? kForkMax - 2 * kForkBand : kForkBand;
      if (used[band] == lim) return parent;
      i = band * kForkBand + used[band]++;
    } else {
      if (n == kForkMax) return parent;
      i = n;
      if (cudaStreamCreateWithPriority(&sub[i], cudaStreamNonBlocking, band_priority(band)) != cudaSuccess) return parent;
      if (cudaEventCreateWithFlags(&joins[i], cudaEventDisableTiming) != cudaSuccess) {
        cudaStreamDestroy(sub[i]);
        return parent;
      }
      own[n++] = i;
    }
    cudaStreamWaitEvent(sub[i], fork, 0);
    return sub[i];
  }
  void join() {
    auto join_one = [&](int i) {
      cudaEventRecord(joins[i], sub[i]);
      cudaStreamWaitEvent(parent, joins[i], 0);
      if (!pooled) {
        cudaEventDestroy(joins[i]);
        cudaStreamDestroy(sub[i]);
      }
    };
    if (pooled) {
      for (int b = 0; b < 3; ++b)
        for (int k = 0; k < used[b]; ++k) join_one(b * kForkBand + k);
    } else {
      for (int k = 0; k < n; ++k) join_one(own[k]);
    }
    if (!pooled && fork) cudaEventDestroy(fork);
    used[0] = used[1] = used[2] = n = 0;
    fork = pooled ? fork : nullptr;
    used_parent = forked = false;
  }
};

static int32_t sweep_run(const cp_grid* g, long long lo, long long hi, int own_lo, int own_hi, int64_t* keys,
                         int32_t* cand_ms, void* ws, void* stream) {
  int rc = CP_OK;
  const long long np = grid_points(g);
  const bool blocked = own_hi > own_lo;
  const long long inner = (long long)g->n_lat * g->n_bw * g->n_mem * g->n_dp;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  unsigned long long* ukeys = reinterpret_cast<unsigned long long*>(keys);
  unsigned long long* counters = static_cast<unsigned long long*>(ws);   // four task counters per p-class (kCtrlBytes = 32 counters)
  if (cpk::launch_sweep_init(ukeys, cand_ms, blocked ? 0 : lo, blocked ? (long long)g->n_pp_n * g->n_mb_n : hi, inner,
                             own_lo, own_hi, stream) != cudaSuccess)
    return CP_ECUDA;
  if (cudaMemsetAsync(counters, 0, sizeof(unsigned long long) * 32, st) != cudaSuccess) return CP_ECUDA;
  // static candidates on k_chunk32f: their plan library (every (kind, n_pp, n_mb) block of the grid)
  const bool static_fast = sweep_static_fast(g);
  uint32_t* plan_lib = nullptr;
  unsigned long long* static_counters = nullptr;
  if (static_fast) {
    size_t off = kCtrlBytes;
    for (int q = 0; q < g->n_pp_n; ++q) off += sweep_class_ring_bytes(g, q);
    static_counters = reinterpret_cast<unsigned long long*>(static_cast<char*>(ws) + off);
    plan_lib = reinterpret_cast<uint32_t*>(static_cast<char*>(ws) + off + 64);
    if (cudaMemsetAsync(static_counters, 0, 64, st) != cudaSuccess) return CP_ECUDA;
    cpk::PlanLibDims d;
    std::memset(&d, 0, sizeof(d));
    for (int i = 0; i < g->n_pp_n; ++i) d.pp[i] = g->n_pp_vals[i];
    for (int i = 0; i < g->n_mb_n; ++i) d.mb[i] = g->n_mb_vals[i];
    d.n_pp = g->n_pp_n;
    d.n_mb = g->n_mb_n;
    d.words = plan_lib_words(g);
    if (cpk::launch_plan_library(d, plan_lib, stream) != cudaSuccess) return CP_ECUDA;
  }
  // p is the slowest axis: one contiguous block of points per p-class; each class gets its own
  // segment width W and ring size, and the classes run concurrently on forked streams
  const long long per_pp = np / g->n_pp_n;
  int cls[8], ncls = 0;
  // largest p first: its launches hold the longest tasks (a launch ends on its longest task), so
  // they are enqueued first and take the SMs before the cheaper classes fill them
  for (int ip = g->n_pp_n - 1; ip >= 0; --ip)
    if (blocked || std::max<long long>(lo, ip * per_pp) < std::min<long long>(hi, (ip + 1) * per_pp)) cls[ncls++] = ip;
  // The longest tasks are the greedy candidates at the largest n_mb (up to ~2,700 rounds at p = 32,
  // m = 128, n_sub = 4): a rank shard cannot end before they do, so they must start at once.  In a
  // proper part of the grid (a shard of a multi-GPU sweep) the trailing mb blocks with
  // n_mb >= max / CP_SWEEP_LONG_DIV (default 1: the largest) go to launches of their own --
  // enqueued first on high-priority streams, the largest p first -- and the other points to the
  // launches below.  The whole grid on one GPU is throughput-bound: there the split costs ~3%.
  int mb_max = 0;
  for (int i = 0; i < g->n_mb_n; ++i) mb_max = std::max(mb_max, g->n_mb_vals[i]);
  int kcut = g->n_mb_n;                          // first mb block of the long part
  const char* ldv = std::getenv("CP_SWEEP_LONG_DIV");
  const int long_div = ldv ? std::max(1, std::atoi(ldv)) : 1;
  while (kcut > 0 && long_div * g->n_mb_vals[kcut - 1] >= mb_max) --kcut;
  const bool partial = blocked ? (long long)(own_hi - own_lo) < inner : hi - lo < np;
  const bool split_long = partial && kcut > 0 && kcut < g->n_mb_n && !getenv_nofast() && !std::getenv("CP_SWEEP_NO_LONG");
  unsigned long long* long_counters =
      reinterpret_cast<unsigned long long*>(static_cast<char*>(ws) + sweep_ws_bytes(g) - kLongCtrBytes);
  if (split_long && cudaMemsetAsync(long_counters, 0, kLongCtrBytes, st) != cudaSuccess) return CP_ECUDA;
  // every launch (greedy tier or static-candidate engine pass) gets its own stream forked from, and
  // joined back to, the caller's: a launch ends on its longest task, so launches that queue behind
  // each other would add those tails up
  Forker fk(st);
  // this class's point set [a0, a1) (points, or mb blocks with the owned slice when blocked) and
  // its size; part 0 = all, 1 = mb blocks [kcut, n_mb) only, 2 = blocks [0, kcut)
  auto class_set = [&](int ip, int part, long long& a0, long long& a1) -> long long {
    if (blocked) {
      a0 = (long long)ip * g->n_mb_n;
      a1 = (long long)(ip + 1) * g->n_mb_n;
      if (part == 1) a0 += kcut;
      if (part == 2) a1 = a0 + kcut;
      return (a1 - a0) * (long long)(own_hi - own_lo);
    }
    a0 = std::max<long long>(lo, ip * per_pp);
    a1 = std::min<long long>(hi, (ip + 1) * per_pp);
    const long long cut = std::min(a1, std::max(a0, ip * per_pp + (long long)kcut * inner));
    if (part == 1) a0 = cut;
    if (part == 2) a1 = cut;
    return std::max(0LL, a1 - a0);
  };
  auto base_args = [&](long long a0, long long a1) {
    cpk::Args a;
    std::memset(&a, 0, sizeof(a));
    a.grid = *g;
    a.pt_lo = a0;
    a.pt_hi = a1;
    a.blk_inner = inner;
    a.own_lo = own_lo;
    a.own_hi = own_hi;
    a.keys = ukeys;
    a.cand_ms = cand_ms;
    return a;
  };
  // greedy candidates (n_sub 1/2/4): k_greedy_fast on synthesized instances, rings sized to the
  // lead bound (rounded to a power of two) so they cannot fill.  Ring size sets residency, so
  // tasks whose own bound is <= 32 run in a launch with 32-slot rings and only the rest in one
  // sized to the class maximum.  Returns false if the class's rings do not fit shared memory.
  const unsigned greedy_mask = g->cand_mask & 0x1cu;
  // Stream priorities (Forker bands): the long-task launches first (band 0); then, across several
  // p-classes, the greedy tiers (band 1: the longer tasks) ahead of the static and engine passes
  // (band 2), which fill in around them (config 5 on one GPU: 5.35 -> 5.1 ms).  A single class
  // keeps one band: there the static pass would only queue behind the greedy grid and add its
  // tail (config 2: 0.25 -> 0.37 ms).
  const int greedy_band = ncls > 1 ? 1 : 2;
  const bool greedy_fast = greedy_mask && !getenv_nofast();
  auto greedy_launches = [&](int ip, long long a0, long long a1, long long npts, unsigned long long* ctr,
                             bool high) -> bool {
    const int p = g->n_pp_vals[ip];
    const int Wd = p <= 8 ? 8 : (p <= 16 ? 16 : 32);
    const int lead_max = sweep_ring_slots(g, p);
    // tiers of lead bound: [0, 32], (32, 64], (64, lead_max]
    const int edge[3] = {32, 64, CP_MAX_MB};
    int ntier = 1;
    while (ntier < 3 && lead_max > edge[ntier - 1]) ++ntier;
    const size_t big_warp = (size_t)((cpk::kGreedyTableWords + 2 * (1 << lg2_ceil(lead_max)) * 32 + 3) & ~3) * 4;
    if (big_warp > kMaxSmemPerBlock) return false;
    // the tier holding the largest leads (and the longest tasks: m up to 128 with large budgets) is
    // launched first, so its tasks start at once instead of queueing behind the persistent grids of
    // the short tiers (measured on one 1/8 rank shard of config 5: the last-enqueued long tier ended
    // the shard)
    for (int tier = ntier - 1; tier >= 0; --tier) {
      cpk::Args ag = base_args(a0, a1);
      ag.grid.cand_mask = greedy_mask;
      ag.sweep_counter = ctr + tier;
      ag.tier_lo = tier == 0 ? 0 : edge[tier - 1] + 1;
      ag.tier_hi = tier == ntier - 1 ? CP_MAX_MB : edge[tier];
      ag.ring_slots = 1 << lg2_ceil(std::min(lead_max, ag.tier_hi));
      ag.smem_words_per_warp = (cpk::kGreedyTableWords + 2 * ag.ring_slots * 32 + 3) & ~3;
      const size_t per_warp = (size_t)ag.smem_words_per_warp * 4;
      const int wpb = per_warp * 2 <= kMaxSmemPerBlock ? 2 : 1, threads = 32 * wpb;
      const size_t smem = per_warp * wpb;
      const int bps = cpk::greedy_fast_blocks_per_sm(Wd, true, threads, smem);
      const long long segs = (long long)(32 / Wd) * wpb;
      const long long need = (npts * __builtin_popcount(greedy_mask) + segs - 1) / segs;
      const int blocks = (int)std::max(1LL, std::min<long long>(need, (long long)cpk::device_sm_count() * bps));
      if (cpk::launch_greedy_fast(Wd, true, ag, blocks, threads, smem, fk.next(high ? 0 : greedy_band)) != cudaSuccess)
        rc = CP_ECUDA;
    }
    return true;
  };
  bool long_done[8] = {};
  if (split_long && greedy_fast)
    for (int c = 0; c < ncls && !rc; ++c) {
      long long a0, a1;
      const long long npts = class_set(cls[c], 1, a0, a1);
      if (npts > 0) long_done[c] = greedy_launches(cls[c], a0, a1, npts, long_counters + 3 * c, true);
    }
  for (int c = 0; c < ncls && !rc; ++c) {
    const int ip = cls[c];
    long long a0, a1;
    const long long npts = class_set(ip, 0, a0, a1);
    cpk::Args a = base_args(a0, a1);
    const int p = g->n_pp_vals[ip];
    // Static candidates (GPipe, 1F1B) and anything the fast path cannot hold in shared memory: the
    // generic engine.
    unsigned engine_mask = g->cand_mask & ((1u << CP_N_CAND) - 1u);
    if (greedy_fast) {
      bool ok = true;
      if (long_done[c]) {
        long long b0, b1;
        const long long nrest = class_set(ip, 2, b0, b1);
        if (nrest > 0) ok = greedy_launches(ip, b0, b1, nrest, counters + 4 * c + 1, false);
      } else {
        ok = greedy_launches(ip, a0, a1, npts, counters + 4 * c + 1, false);
      }
      if (ok) engine_mask &= ~greedy_mask;
    }
    if (!rc && static_fast && (engine_mask & kStaticCands)) {
      // GPipe / 1F1B / ZB-H1 of this class on k_chunk32f<UD, grid> (8-slot rings: the static families
      // never lead by more than two messages), plans from the library, one task per warp
      cpk::Args as = a;
      as.grid.cand_mask = engine_mask & kStaticCands;
      as.sweep_counter = static_counters + c;
      as.ops = plan_lib;
      as.words = plan_lib_words(g);
      as.ring_slots = 8;
      as.shared_tab = 0;
      const cpk::ChunkFLayout L = cpk::chunkf_layout(as.ring_slots, as.words, false, 2);
      const int wpb = cpk::kChunkFThreads / 32, threads = cpk::kChunkFThreads;
      const size_t smem = (size_t)wpb * L.per_warp * 4;
      const int bps = smsp_balanced(cpk::chunkf_grid_blocks_per_sm(threads, smem), wpb);
      const long long need = (npts * __builtin_popcount(as.grid.cand_mask) + wpb - 1) / wpb;
      const int blocks = (int)std::max(1LL, std::min<long long>(need, (long long)cpk::device_sm_count() * bps));
      if (cpk::launch_chunkf_grid(as, blocks, threads, smem, fk.next()) != cudaSuccess) rc = CP_ECUDA;
      engine_mask &= ~kStaticCands;
    }
    if (!rc && engine_mask) {
      a.grid.cand_mask = engine_mask;
      a.sweep_counter = counters + 4 * c;
      a.seg_lg = lg2_ceil(p);
      a.ring_slots = sweep_ring_slots(g, p);
      cudaStream_t es = fk.next();
      rc = launch_pass(cpk::MODE_SWEEP, false, a, npts * __builtin_popcount(engine_mask), 32 >> a.seg_lg, es);
      if (rc == CP_EUNSUPPORTED) {
        // rings beyond shared memory: this class's global-memory rings in the workspace
        size_t off = kCtrlBytes;
        for (int q = 0; q < ip; ++q) off += sweep_class_ring_bytes(g, q);
        a.ring_g = reinterpret_cast<int32_t*>(static_cast<char*>(ws) + off);
        rc = launch_pass(cpk::MODE_SWEEP, true, a, npts * __builtin_popcount(engine_mask), 32 >> a.seg_lg, es);
      }
    }
  }
  fk.join();
  if (rc) return rc;
  return cudaGetLastError() == cudaSuccess ? CP_OK : CP_ECUDA;
}

int32_t cp_sweep_shard(const cp_grid* g, int64_t lo, int64_t hi, int64_t* keys, int32_t* cand_ms, void* ws,
                       size_t ws_bytes, void* stream) {
  int rc = check_grid(g);
  if (rc) return rc;
  const long long np = grid_points(g);
  if (!keys || lo < 0 || hi < lo || hi > np) return CP_EINVAL;
  if (!ws || ws_bytes < sweep_ws_bytes(g)) return CP_EWORKSPACE;
  if (lo == hi) return CP_OK;
  return sweep_run(g, lo, hi, 0, 0, keys, cand_ms, ws, stream);
}

int32_t cp_sweep_shard_rank(const cp_grid* g, int32_t rank, int32_t world, int64_t* keys, int32_t* cand_ms, void* ws,
                            size_t ws_bytes, void* stream) {
  int rc = check_grid(g);
  if (rc) return rc;
  if (!keys || world < 1 || rank < 0 || rank >= world) return CP_EINVAL;
  if (!ws || ws_bytes < sweep_ws_bytes(g)) return CP_EWORKSPACE;
  const long long inner = (long long)g->n_lat * g->n_bw * g->n_mem * g->n_dp;
  const int own_lo = (int)(inner * rank / world), own_hi = (int)(inner * (rank + 1) / world);
  if (own_lo == own_hi) return CP_OK;
  return sweep_run(g, 0, 0, own_lo, own_hi, keys, cand_ms, ws, stream);
}

int32_t cp_sweep_partition(const cp_grid* g, int32_t world, int64_t* bounds) {
  int rc = check_grid(g);
  if (rc) return rc;
  if (world < 1 || !bounds) return CP_EINVAL;
  const long long inner = (long long)g->n_lat * g->n_bw * g->n_mem * g->n_dp;   // equal-cost run
  const int nblk = g->n_pp_n * g->n_mb_n;
  std::vector<long long> pre(nblk + 1, 0);
  for (int b = 0; b < nblk; ++b) pre[b + 1] = pre[b] + point_cost(g, b / g->n_mb_n, b % g->n_mb_n) * inner;
  const long long total = pre[nblk];
  bounds[0] = 0;
  for (int r = 1; r < world; ++r) {
    const long double target = (long double)total * r / world;
    int b = 0;
    while (b < nblk && pre[b + 1] <= target) ++b;
    long long pt;
    if (b >= nblk) pt = (long long)nblk * inner;
    else {
      const long long c = point_cost(g, b / g->n_mb_n, b % g->n_mb_n);
      long long k = (long long)std::llround((double)((target - pre[b]) / c));
      k = std::max(0LL, std::min(inner, k));
      pt = (long long)b * inner + k;
    }
    bounds[r] = std::max<long long>(pt, bounds[r - 1]);
  }
  bounds[world] = (long long)nblk * inner;
  return CP_OK;
}

int32_t cp_validate_instance(const cp_inst_v1* I, char* msg, size_t msg_len) {
  auto fail = [&](int code, const char* what, int s) {
    if (msg && msg_len) std::snprintf(msg, msg_len, "%s%s%d", what, s >= 0 ? " at stage/boundary " : "", s);
    return code;
  };
  if (!I) return fail(CPI_BAD_INSTANCE, "null record", -1);
  if (I->n_pp < 1 || I->n_pp > CP_MAX_STAGES) return fail(CPI_BAD_INSTANCE, "n_pp out of [1, 32]", -1);
  if (I->n_mb < 1) return fail(CPI_BAD_INSTANCE, "n_mb < 1", -1);
  if (I->n_sub < 1) return fail(CPI_BAD_INSTANCE, "n_sub < 1", -1);
  for (int s = 0; s < I->n_pp; ++s) {
    if (I->t_f[s] <= 0 || I->t_d[s] <= 0 || I->t_w[s] <= 0) return fail(CPI_BAD_INSTANCE, "durations must be > 0", s);
    if (I->t_f[s] < I->n_sub || I->t_d[s] < I->n_sub || I->t_w[s] < I->n_sub)
      return fail(CPI_BAD_INSTANCE, "a block shorter than n_sub ticks (every sub-block >= 1 tick, reading Q12)", s);
    if (I->m_f[s] <= 0 || I->m_d[s] > 0 || I->m_w[s] > 0) return fail(CPI_BAD_INSTANCE, "memory delta signs", s);
    if ((long long)I->m_f[s] + I->m_d[s] + I->m_w[s] != 0) return fail(CPI_BAD_INSTANCE, "memory deltas do not sum to zero", s);
    if (I->m_lim[s] < I->m_f[s]) return fail(CPI_BAD_INSTANCE, "m_lim < m_f", s);
    if (I->t_dp[s] < 0 || I->t_ag[s] < 0) return fail(CPI_BAD_INSTANCE, "negative DP time", s);
    if (s < I->n_pp - 1 && (I->lat_f[s] < 0 || I->bw_f[s] < 0 || I->lat_b[s] < 0 || I->bw_b[s] < 0))
      return fail(CPI_BAD_INSTANCE, "negative link delay", s);
  }
  if (I->n_mb > CP_MAX_MB || I->n_sub > CP_MAX_SUB) return fail(CPI_OVERFLOW, "n_mb/n_sub exceed GPU limits", -1);
  long long U = 0;
  for (int s = 0; s < I->n_pp; ++s) {
    U += (long long)I->n_mb * ((long long)I->t_f[s] + I->t_d[s] + I->t_w[s]) + I->t_dp[s] + ((I->flags & 1) ? I->t_ag[s] : 0);
    if (s < I->n_pp - 1) U += (long long)I->n_mb * ((long long)I->lat_f[s] + I->bw_f[s] + I->lat_b[s] + I->bw_b[s]);
  }
  if (U >= (1LL << 30)) return fail(CPI_OVERFLOW, "horizon bound U >= 2^30 ticks", -1);
  if (msg && msg_len) msg[0] = 0;
  return 0;
}

int32_t cp_quantize(const cp_spec_si* S, cp_inst_v1* o) {
  if (!S || !o) return CPI_BAD_INSTANCE;
  std::memset(o, 0, sizeof(*o));
  if (S->n_pp < 1 || S->n_pp > CP_MAX_STAGES || S->n_dc < 1 || S->n_dc > 4 || !(S->tick_s > 0) || !(S->mem_unit > 0))
    return CPI_BAD_INSTANCE;
  if (S->n_mb < 1 || S->n_mb > 65535 || S->n_sub < 1 || S->n_sub > 255) return CPI_BAD_INSTANCE;
  o->n_pp = (uint8_t)S->n_pp;
  o->n_mb = (uint16_t)S->n_mb;
  o->n_sub = (uint8_t)S->n_sub;
  o->n_dc = (uint8_t)S->n_dc;
  o->flags = S->zero1 ? 1 : 0;
  o->version = 1;
  o->tick_ns = (int32_t)std::llround(S->tick_s * 1e9);
  bool over = false;
  auto q = [&](double x, double unit) -> int32_t {
    const long long v = std::llround(x / unit);
    if (v > INT32_MAX || v < INT32_MIN) { over = true; return 0; }
    return (int32_t)v;
  };
  for (int s = 0; s < S->n_pp; ++s) {
    const int dc = S->dc_of_stage[s];
    if (dc < 0 || dc >= S->n_dc) return CPI_BAD_INSTANCE;
    if (s > 0 && dc < S->dc_of_stage[s - 1]) return CPI_BAD_INSTANCE;     // contiguous DC assignment
    if (s == 0 || dc != S->dc_of_stage[s - 1]) o->dc_first_stage[dc] = (uint8_t)s;
    o->t_f[s] = q(S->t_f[s], S->tick_s);
    o->t_d[s] = q(S->t_d[s], S->tick_s);
    o->t_w[s] = q(S->t_w[s], S->tick_s);
    o->m_f[s] = q(S->m_f[s], S->mem_unit);
    o->m_d[s] = q(S->m_d[s], S->mem_unit);
    o->m_w[s] = q(S->m_w[s], S->mem_unit);
    const double ml = std::floor(S->m_lim[s] / S->mem_unit);
    if (ml > INT32_MAX) over = true; else o->m_lim[s] = (int32_t)ml;
    o->t_dp[s] = q(S->t_dp[s], S->tick_s);
    o->t_ag[s] = S->zero1 ? q(S->t_ag[s], S->tick_s) : 0;
    if (s < S->n_pp - 1) {
      const int a = S->dc_of_stage[s], b = S->dc_of_stage[s + 1];
      o->lat_f[s] = q(S->alpha[a][b], S->tick_s);
      const double wf = S->beta[a][b] * S->msg_f[s];
      o->bw_f[s] = q(wf, S->tick_s);
      o->lat_b[s] = q(S->alpha[b][a], S->tick_s);
      const double wb = S->beta[b][a] * S->msg_b[s];
      o->bw_b[s] = q(wb, S->tick_s);
    }
  }
  const int32_t v = cp_validate_instance(o, nullptr, 0);
  if (v == CPI_BAD_INSTANCE) return v;
  return over ? CPI_OVERFLOW : 0;
}

}  // extern "C"
