// engine.cu -- sm_100a kernels of the CrossPipe hot path (arXiv 2507.00217).
//
// One warp evaluates 32/W items at a time: lane = pipeline stage, W = pow2 >= p is
// the lane-segment width (small-p items are packed several per warp; shuffles use
// the `width` argument so segments never talk to each other).  Evaluation is
// round-synchronous dataflow; each round every lane executes at most one block:
//   * the lane holds its stage's clock, memory, per-type counters and the FIFO clocks
//     of its two outgoing links in registers;
//   * a finished F (resp. D/B) block pushes its message through the link clock
//     (Alg. 1 :404-407: E_bw = BW_model(end), T_avail = E_bw + T_lat) and writes the
//     arrival time into the consumer's shared-memory arrival ring (slot-major [R][32]
//     layout: lane l always touches bank l or l+-1 -> conflict-free);
//   * producer counts are exchanged with one __shfl_up + one __shfl_down per round;
//   * block execution is branch-free (selects), so a warp walks one path per round
//     whatever mix of F / D / B / W its lanes execute;
//   * plan rows are staged in shared memory: one TMA bulk copy (cp.async.bulk,
//     double-buffered: the next item's plan lands while the current one runs) when a
//     warp holds one item, a cooperative copy when it holds several;
//   * one ballot per round detects "no progress"; completion, deadlock, bad plans and
//     ring overflow are resolved only on that rare path.
// MODE_SIM    : plan-driven (cp_simulate): a lane executes its next plan entry as soon
//               as the entry's input is known (the §3.5 max-plus recurrence).
// MODE_GREEDY : Alg. 1 + §4.2.2 (cp_greedy): every lane computes its schedulable time
//               t*_s; two min-plus warp scans give a causal horizon and every lane with
//               t*_s < horizon decides in the same round (DESIGN.md "Round-parallel
//               greedy"), which reproduces sequential Alg. 1 exactly.
// MODE_SWEEP  : (cp_sweep_shard) grid point -> instance synthesis in registers -> GPipe /
//               1F1B plans generated arithmetically + greedy n_sub = 1, 2, 4 -> packed
//               (makespan << 8 | cand) argmin per point.
// No tensor cores: nothing here is a dense contraction.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "engine.h"
#include "grid_synth.cuh"
#include "plan_codes.cuh"
#include "ptx.cuh"

namespace cpk {

constexpr int32_t INF = 1 << 30;        // > every valid tick value (guard U < 2^30)
constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ int imin(int a, int b) { return a < b ? a : b; }
__device__ __forceinline__ int imax(int a, int b) { return a > b ? a : b; }

#ifdef CP_DEBUG
// Debug build only: every shared / global access of the engine goes through a bounds check
// that records the first violation (tag, index, limit, item, lane) and skips the access.
__device__ int cp_dbg[8];
__device__ __noinline__ bool dbg_ok(long long idx, long long lim, int tag, long long item) {
  if (idx >= 0 && idx < lim) return true;
  if (atomicCAS(&cp_dbg[0], 0, tag) == 0) {
    cp_dbg[1] = (int)idx; cp_dbg[2] = (int)lim; cp_dbg[3] = (int)item; cp_dbg[4] = threadIdx.x;
    cp_dbg[5] = blockIdx.x; cp_dbg[6] = (int)(idx >> 32);
  }
  return false;
}
#define CHK(idx, lim, tag) dbg_ok((long long)(idx), (long long)(lim), (tag), item)
#else
#define CHK(idx, lim, tag) true
#endif


// Arithmetic static plans (Table tab:ppschedules :470; readings Q22/Q23).
// GPipe: F x m, B x m.  1F1B: w = min(p-s-1, m) F, (F,B) x (m-w), B x w.

struct LaneCfg {       // per-lane (stage) instance fields
  int p, m, nsub, tagate;
  int tf, td, tw, tB, wq, wr, mf, md, mw, mB, mlim, tdp;
  int latF, bwF, latB, bwB;
  int P, Q;            // greedy lookahead: exclusive prefix of (tf+bwF+latF), inclusive prefix of (td+bwB+latB)
};

// smem layout per warp (32-bit words, integer offsets from the warp base):
//   [ringF R*32][ringD R*32][plan 2*PW*32][2 mbarriers]   (rings live in global memory in
//   the fix-up pass, kRingGlobal)
template <int kMode, bool kRingGlobal, bool kTimeline>
__global__ void __launch_bounds__(kThreads) k_engine(const __grid_constant__ Args A) {
  extern __shared__ __align__(128) int32_t smem[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int lgW = A.seg_lg;
  const int W = 1 << lgW;
  const int s = lane & (W - 1);
  const int seg = lane >> lgW;
  const int nseg = 32 >> lgW;
  const unsigned segmask = (W == 32) ? FULL : (((1u << W) - 1u) << (seg * W));
  const int R = A.ring_slots;
  const long long gwarp = (long long)blockIdx.x * (blockDim.x >> 5) + wib;
  const long long nwarps = (long long)gridDim.x * (blockDim.x >> 5);
  const int wbase = wib * A.smem_words_per_warp;      // this warp's smem window (words)
  int32_t* const rg = kRingGlobal ? A.ring_g + gwarp * (2LL * R * 32) : nullptr;
  const int RW = R * 32;                               // D ring starts RW words after the F ring
  const int PW = A.plan_words;                         // plan words staged in smem (0: read from global)
  const int pbase = wbase + (kRingGlobal ? 0 : 2 * RW);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + pbase + 2 * PW * 32);
  uint32_t* const plan = reinterpret_cast<uint32_t*>(smem + pbase);
  const bool use_tma = (kMode == MODE_SIM) && A.tma && PW > 0;   // one item per warp, rows contiguous [words][32]
  const uint32_t plan_bytes = (uint32_t)A.words * 32u * 4u;
  // ring accessors: offsets are relative to the F ring of this warp
  auto ring_ld = [&](int off) -> int { return kRingGlobal ? rg[off] : smem[wbase + off]; };
  auto ring_st = [&](int off, int v) { if (kRingGlobal) rg[off] = v; else smem[wbase + off] = v; };

  long long task = gwarp * nseg + seg;
  const long long task_stride = nwarps * nseg;
#ifdef CP_DEBUG
  const long long s_lim = (long long)(blockDim.x >> 5) * A.smem_words_per_warp;
  long long item = -1;
  auto ROK = [&](int off, int tag) -> bool { return dbg_ok(kRingGlobal ? off : wbase + off, kRingGlobal ? 2LL * RW : s_lim, tag, item); };
  auto POK = [&](int off, int tag) -> bool { return dbg_ok(pbase + off, s_lim, tag, item); };
  const long long n_it = kMode == MODE_SWEEP ? (A.own_hi > A.own_lo ? A.pt_hi * A.blk_inner : A.pt_hi) : A.n_items;
#else
  long long item = -1;
#define ROK(off, tag) true
#define POK(off, tag) true
#endif

  // Output rows r = s, s + W, ... < stage_stride that this lane finishes for an item: zero stats
  // for rows no lane owns (r >= W); greedy: len and every plan word past the emitted entries zeroed
  // (the row's own words up to `used` are written by the caller), so outputs are fully defined.
  auto finish_rows = [&](long long it, int used) {
    if (kMode == MODE_SWEEP) return;
    for (int r = s; r < A.stage_stride; r += W) {
      const long long rb = it * A.stage_stride + r;
      if (A.stage_stats && r != s) *reinterpret_cast<int4*>(A.stage_stats + rb * 4) = make_int4(0, 0, 0, 0);
      if (kMode == MODE_GREEDY) {
        const int u = r == s ? used : 0;
        for (int k = (u + 15) >> 4; k < A.words; ++k) A.ops[(it * A.words + k) * A.stage_stride + r] = 0u;
        A.len[rb] = (uint16_t)u;
      }
    }
  };

  auto item_of = [&](long long t) -> long long {
    if (A.from_list) return (t < *(volatile int32_t*)A.ovf_count) ? (long long)A.ovf_list[t] : -1;
    return t < A.n_items ? t : -1;
  };

  uint32_t phase = 0;          // mbarrier parity of each plan buffer (bit b)
  int cur_buf = 0;
  int plan_off = lane;         // cur_buf * PW * 32 + lane
  if (use_tma) {
    if (lane == 0) { mbar_init(&bars[0]); mbar_init(&bars[1]); }
    __syncwarp();
    const long long it0 = item_of(task);
    if (lane == 0 && it0 >= 0) tma_load_1d(plan, A.ops + it0 * A.words * 32, plan_bytes, &bars[0]);
  }

  LaneCfg c = {};
  bool need_load = true, any_load = true, has_item = false;
  int load_status = 0;
  int zero1 = 0, valid_inst = 0;
  // dynamic state of this lane's stage
  int clk = 0, mem = 0, peak = 0, nF = 0, nD = 0, nW = 0, wsub = 0, linkF = 0, linkB = 0;
  int slF = 0, slD = 0;                   // ring slots = nF mod R, nD mod R
  int first = 0, busy = 0, pos = 0, plen = 0, comb = 0, last_fd = 0;
  uint32_t emitw = 0;
  int fmask = 0, dmask = 0;               // -1 where the lane consumes F (s > 0) / D (s < p-1) arrivals
  bool fmask_next = false;                // the lane sends F blocks (s < p-1)
  // sweep: candidate of the current (point, candidate) task
  int cand = 0;
  bool cand_greedy = (kMode == MODE_GREEDY);

  for (;;) {
    // ------------------------------------------------------------------ fetch + load (per segment)
    if (any_load) {
      bool just_loaded = false;
      if (need_load) {
        need_load = false;
        if (kMode == MODE_SWEEP) {
          // dynamic (point, candidate) tasks, most expensive first (grid_synth.cuh)
          long long t = 0;
          if (s == 0) t = atomicAdd(A.sweep_counter, 1ull);
          t = __shfl_sync(segmask, t, seg * W);
          item = sweep_task(A.grid.cand_mask & ((1u << CP_N_CAND) - 1u), SweepSet{A.pt_lo, A.pt_hi, A.blk_inner, A.own_lo, A.own_hi},
                        t, cand);
        } else {
          item = item_of(task);
          task += task_stride;
        }
        has_item = item >= 0;
        if (item >= 0) {
          just_loaded = true;
          int lat_b_s = 0, bw_b_s = 0;   // lane s validates boundary s in both directions
          c = LaneCfg{};
          if (kMode == MODE_SWEEP) {
            const GridLane g = grid_lane(A.grid, item, s);
            c.p = g.p;
            c.m = g.m;
            cand_greedy = cand >= 2 && cand <= 4;
            c.nsub = cand_greedy ? (1 << (cand - 2)) : 1;
            zero1 = g.zero1;
            c.tf = g.tf; c.td = g.td; c.tw = g.tw;
            c.mf = g.mf; c.md = g.md; c.mw = g.mw; c.mlim = g.mlim;
            c.tdp = g.tdp; c.tagate = g.tag;
            c.latF = g.latF; c.bwF = g.bwF; c.latB = g.latB; c.bwB = g.bwB;
            lat_b_s = c.latF; bw_b_s = c.bwF;
          } else {
            const long long ii = A.inst_of ? (long long)A.inst_of[item] : (A.n_inst == 1 ? 0 : item);
            const cp_inst_v1* I = A.inst + ii;
            c.p = I->n_pp; c.m = I->n_mb; c.nsub = I->n_sub;
            zero1 = I->flags & 1;
            if (s < c.p && s < CP_MAX_STAGES) {
              c.tf = I->t_f[s]; c.td = I->t_d[s]; c.tw = I->t_w[s];
              c.mf = I->m_f[s]; c.md = I->m_d[s]; c.mw = I->m_w[s]; c.mlim = I->m_lim[s];
              c.tdp = I->t_dp[s];
              c.tagate = I->t_ag[s];
              c.latF = (s < c.p - 1) ? I->lat_f[s] : 0; c.bwF = (s < c.p - 1) ? I->bw_f[s] : 0;
              c.latB = (s > 0) ? I->lat_b[s - 1] : 0; c.bwB = (s > 0) ? I->bw_b[s - 1] : 0;
              lat_b_s = (s < c.p - 1) ? I->lat_b[s] : 0; bw_b_s = (s < c.p - 1) ? I->bw_b[s] : 0;
            }
          }
          // instance invariants (readings Q10, Q12)
          bool bad = c.p < 1 || c.p > CP_MAX_STAGES || c.m < 1 || c.nsub < 1;
          if (!bad && s < c.p) {
            bad = !(c.tf >= c.nsub && c.td >= c.nsub && c.tw >= c.nsub && c.nsub >= 1 && c.mf > 0 && c.md <= 0 && c.mw <= 0 &&
                    (long long)c.mf + c.md + c.mw == 0 && c.mlim >= c.mf && c.tdp >= 0 && c.tagate >= 0 &&
                    c.latF >= 0 && c.bwF >= 0 && lat_b_s >= 0 && bw_b_s >= 0);
          }
          if (!zero1) c.tagate = 0;
          valid_inst = !bad;
          load_status = bad ? CPI_BAD_INSTANCE : 0;
          c.wq = c.tw / imax(c.nsub, 1);
          c.wr = c.tw % imax(c.nsub, 1);
          c.tB = c.td + c.tw;
          c.mB = c.md + c.mw;
          fmask = (s > 0) ? -1 : 0;
          dmask = (s < c.p - 1) ? -1 : 0;
          fmask_next = s < c.p - 1;
          plen = (kMode == MODE_SWEEP && s < c.p && !cand_greedy) ? plan_row_len(cand, c.m) : 0;
          if (kMode == MODE_SIM && s < c.p && s < A.stage_stride) {
            plen = A.len[item * A.stage_stride + s];
            if (plen > 16 * A.words && !bad) load_status = CPI_BAD_PLAN;     // row longer than its capacity
          }
          if (kMode == MODE_GREEDY && !bad && (long long)(2 + c.nsub) * c.m > 16LL * A.words)
            load_status = CPI_BAD_PLAN;                                      // output row capacity too small
          if (!load_status && (c.p > W || c.m > CP_MAX_MB || c.nsub > CP_MAX_SUB)) load_status = CPI_OVERFLOW;
          clk = mem = peak = nF = nD = nW = wsub = linkF = linkB = slF = slD = 0;
          first = busy = pos = comb = last_fd = 0;
          emitw = 0;
        }
      }
      if (__all_sync(FULL, item < 0)) break;

      // ---------------------------------------------------------------- warp-wide post-load
      if (__any_sync(FULL, just_loaded)) {
        const bool act = just_loaded && s < c.p && valid_inst;
        const int cf = act ? c.tf + c.bwF + c.latF : 0;      // hop s -> s+1 (F)
        const int cd = act ? c.td + c.bwB + c.latB : 0;      // hop s -> s-1 (D)
        long long u = 0;                                      // horizon bound U (reading Q21)
        if (act)
          u = (long long)c.m * ((long long)c.tf + c.td + c.tw) + c.tagate + c.tdp +
              (long long)c.m * ((long long)c.latF + c.bwF + c.latB + c.bwB);
        int pf = cf, qd = cd;
        for (int d = 1; d < W; d <<= 1) {
          const int a = __shfl_up_sync(FULL, pf, d, W);
          const int b = __shfl_up_sync(FULL, qd, d, W);
          if (s >= d) { pf += a; qd += b; }
        }
        for (int d = 1; d < W; d <<= 1) u += __shfl_xor_sync(FULL, u, d, W);
        // sweep: candidate statically infeasible (GPipe peak m*m_f, 1F1B peak min(p-s,m)*m_f (Z5),
        // greedy with a block shorter than n_sub ticks (Q12)) or masked out -> skipped (its cand_ms
        // stays -1, no key)
        bool skip_lane = false;
        if (kMode == MODE_SWEEP && just_loaded && s < c.p)
          skip_lane = cand == 0 ? (long long)c.m * c.mf > c.mlim
                                : (cand == 1 ? (long long)imin(c.p - s, c.m) * c.mf > c.mlim
                                             : (cand == 5 ? false      // ZB-H1: evaluated, excluded if over M_L
                                                          : (c.tf < c.nsub || c.td < c.nsub || c.tw < c.nsub)));
        const unsigned b_skip = __ballot_sync(FULL, skip_lane || (kMode == MODE_SWEEP && just_loaded &&
                                                                 !((A.grid.cand_mask >> cand) & 1u)));
        const unsigned b_inst = __ballot_sync(FULL, just_loaded && load_status == CPI_BAD_INSTANCE);
        const unsigned b_plan = __ballot_sync(FULL, just_loaded && load_status == CPI_BAD_PLAN);
        const unsigned b_over = __ballot_sync(FULL, just_loaded && load_status == CPI_OVERFLOW);
        if (just_loaded) {
          c.P = pf - cf;
          c.Q = qd;
          int st = (b_inst & segmask) ? CPI_BAD_INSTANCE
                   : (b_plan & segmask) ? CPI_BAD_PLAN
                   : (b_over & segmask) ? CPI_OVERFLOW : 0;
          if (!st && u >= (long long)INF) st = CPI_OVERFLOW;     // int32 horizon guard
          load_status = st;
          if (kMode == MODE_SWEEP) {
            if (st == CPI_OVERFLOW && s == 0) atomicMin(A.keys + item, KEY_OVER);
            if (st != 0 || (b_skip & segmask)) need_load = true;
          }
          if (kMode != MODE_SWEEP && st != 0) {
            // per-item failure: report now, no evaluation
            if (s == 0) {
              A.makespan[item] = -1;
              if (A.peak_mem) A.peak_mem[item] = -1;
              A.status[item] = st;
            }
            if (A.stage_stats && s < A.stage_stride)
              *reinterpret_cast<int4*>(A.stage_stats + (item * A.stage_stride + s) * 4) = make_int4(0, 0, 0, 0);
            finish_rows(item, 0);
            need_load = true;
          }
        }
        // stage the plan rows in shared memory
        if (kMode == MODE_SIM && PW > 0) {
          if (use_tma) {
            // this item's rows were prefetched into plan[cur_buf]: wait, then prefetch the next item
            if (just_loaded) {
              mbar_wait(&bars[cur_buf], (phase >> cur_buf) & 1u);
              phase ^= 1u << cur_buf;
              const long long nxt = item_of(task);
              if (lane == 0 && nxt >= 0)
                tma_load_1d(plan + (cur_buf ^ 1) * PW * 32, A.ops + nxt * A.words * 32, plan_bytes,
                            &bars[cur_buf ^ 1]);
              if (need_load) { cur_buf ^= 1; plan_off = cur_buf * PW * 32 + lane; }   // failed item
            }
          } else if (just_loaded && !need_load && s < c.p) {
            for (int k = 0; k < A.words && k * 16 < plen; ++k)
              if (POK(k * 32 + lane, 14) && CHK(item * A.words + k, n_it * A.words, 15))
                plan[k * 32 + lane] = A.ops[(item * A.words + k) * A.stage_stride + s];
          }
          __syncwarp();
        }
      }

      any_load = __any_sync(FULL, need_load);
      if (any_load) continue;     // warp-uniform: (re)load before running rounds
    }

    // ------------------------------------------------------------------ one round
    const bool in_round = has_item;                    // segment-uniform
    const bool is_greedy = (kMode == MODE_GREEDY) || (kMode == MODE_SWEEP && cand_greedy);
    // greedy: W_{m-1} is a stage's last block, so the stage is done iff nW == m
    const bool live = in_round && s < c.p && (is_greedy ? nW < c.m : pos < plen);

    const int leftF = __shfl_up_sync(FULL, nF, 1, W);
    const int rightD = __shfl_down_sync(FULL, nD, 1, W);
    // a lane's next F/D input is known once its producer has emitted it; an F additionally needs
    // room in the consumer's ring (lead <= R) -- a full ring stalls the lane and the
    // rare path hands the item to the global-ring fix-up pass
    const bool roomF = kRingGlobal || (nF - nD < R);
    const bool knowFg = nF < c.m && (fmask == 0 || leftF > nF);      // greedy: capacity not part of the decision
    const bool knowF = knowFg && roomF;
    const bool knowD = nD < c.m && (dmask == 0 ? nF > nD : rightD > nD);

    bool go = false, isF = false, isW = false, isB = false;
    int start = 0;
    if (kMode != MODE_GREEDY) {
      // ---- plan-driven selection: next entry of this stage's row.  Entries that violate the
      // static rules (Q29) are simply never ready; a stalled item is classified on the rare path.
      int code;
      if (kMode == MODE_SIM) {
        const int pq = live ? pos : 0;       // finished rows may sit at pos == 16*words: never index past them
        uint32_t wv;
        if (PW > 0) wv = POK(plan_off + ((pq >> 4) << 5), 1) ? plan[plan_off + ((pq >> 4) << 5)] : 0u;
        else wv = (live && CHK(item * A.words + (pq >> 4), n_it * A.words, 2)) ? A.ops[(item * A.words + (pq >> 4)) * A.stage_stride + s] : 0u;
        code = (int)((wv >> ((pq & 15) << 1)) & 3u);
      } else {
        code = plan_code(cand, s, c.p, c.m, pos);   // cand 0/1/5 = CP_PLAN_GPIPE/1F1B/ZBH1
      }
      const bool cF = code == (int)CP_OP_F, cW = code == (int)CP_OP_W, cB = code == (int)CP_OP_B;
      const int roff = cF ? lane + (slF << 5) : RW + lane + (slD << 5);
      const int arr = ROK(roff, 3) ? ring_ld(roff) : 0;
      const int avail = cF ? imax(arr & fmask, c.tagate) : (cW ? 0 : (arr & dmask));
      bool ready = cF ? knowF : (cW ? (nW * c.nsub + wsub < c.nsub * nD) : knowD);
      if (kMode == MODE_SIM) ready = ready && (cB ? comb != 2 : (cF || comb != 1));
      if (!is_greedy) {
        go = live && ready;
        isF = cF; isW = cW; isB = cB;
        start = imax(clk, avail);
      }
    }
    if (kMode != MODE_SIM) {
      // ---- greedy selection (Alg. 1 lines 6 and 10, §4.2.2)
      const int arrF = ROK(lane + (slF << 5), 4) ? ring_ld(lane + (slF << 5)) : 0;
      const int arrD = ROK(RW + lane + (slD << 5), 5) ? ring_ld(RW + lane + (slD << 5)) : 0;
      const int availF = imax(arrF & fmask, c.tagate);
      const int availD = arrD & dmask;
      const bool gl = live && is_greedy;
      const bool hasF = gl && knowFg && mem + c.mf <= c.mlim;     // Q15: memory-infeasible F is not eligible
      const bool hasD = gl && knowD;
      const bool hasW = gl && nW < nD;                             // W avail = its D end <= clk
      int mn = hasF ? availF : INF;
      mn = imin(mn, hasD ? availD : INF);
      mn = imin(mn, hasW ? clk : INF);
      const int tstar = (hasF || hasD || hasW) ? imax(clk, mn) : INF;   // §4.2.2 :419
      bool run_scan = true;
      if (kMode == MODE_SWEEP) run_scan = __any_sync(FULL, gl);
      if (run_scan) {
        // causal horizon: L_s = P_s + min_{k<s}(t*_k - P_k), R_s = min_{k>s}(t*_k + Q_k) - Q_s
        int x = tstar - c.P, y = tstar + c.Q;
        for (int d = 1; d < W; d <<= 1) {
          const int xu = __shfl_up_sync(FULL, x, d, W);
          const int yd = __shfl_down_sync(FULL, y, d, W);
          x = (s >= d) ? imin(x, xu) : x;
          y = (s + d < W) ? imin(y, yd) : y;
        }
        const int xe = __shfl_up_sync(FULL, x, 1, W);
        const int ye = __shfl_down_sync(FULL, y, 1, W);
        const int Lh = (s == 0) ? INF : c.P + xe;
        const int Rh = (s == W - 1) ? INF : ye - c.Q;
        const bool g_go = tstar < INF && tstar < imin(Lh, Rh);   // L, R may exceed INF: guard idle lanes
        // operation selection (reading Q13): opposite of the last full F/D block, then the
        // other, then a W sub-block
        const bool cF = hasF && availF <= tstar, cD = hasD && availD <= tstar;
        const bool pickD = (last_fd == 1) ? cD : (cD && !cF);
        const bool pickF = !pickD && cF;
        if (is_greedy) {
          // an F whose consumer ring is full is not executed (lane stalls -> fix-up pass); the
          // decision itself never depends on the ring capacity
          go = g_go && !(pickF && !roomF);
          isF = pickF; isW = !pickF && !pickD; isB = false;
          start = tstar;
        }
      }
    }

    // ------------------------------------------------------------------ execute (pure selects)
    {
      const bool isDB = !isF && !isW;
      const bool wfin = isW && (wsub + 1 == c.nsub);
      const int dur = isF ? c.tf : (isW ? c.wq + (wsub < c.wr ? 1 : 0) : (isB ? c.tB : c.td));
      const int end = start + dur;
      const int dmem = isF ? c.mf : (isW ? (wfin ? c.mw : 0) : (isB ? c.mB : c.md));
      // message through the FIFO link clock (= first fit under UD, App. X1)
      const int nl = imax(end, isF ? linkF : linkB) + (isF ? c.bwF : c.bwB);
      const int sl = isF ? slF : slD;
      const int woff = (isF ? lane + 1 : RW + lane - 1) + (sl << 5);
      const bool send = go && (isF ? fmask_next : (isDB && fmask != 0));
      if (send && ROK(woff, 6)) ring_st(woff, nl + (isF ? c.latF : c.latB));
      if (kTimeline && go && pos < A.len_stride && CHK(item * A.stage_stride + s, n_it * A.stage_stride, 7))
        A.t_start[(item * A.stage_stride + s) * (long long)A.len_stride + pos] = start;
      if (kMode == MODE_GREEDY && go) {
        const int code = isF ? (int)CP_OP_F : (isW ? (int)CP_OP_W : (int)CP_OP_D);
        emitw |= (uint32_t)code << ((pos & 15) << 1);
        if (PW > 0) { if (POK(((pos >> 4) << 5) + lane, 8)) plan[((pos >> 4) << 5) + lane] = emitw; }
        else if ((pos & 15) == 15 && CHK(item * A.words + (pos >> 4), n_it * A.words, 9))
          A.ops[(item * A.words + (pos >> 4)) * A.stage_stride + s] = emitw;
        emitw = ((pos & 15) == 15) ? 0u : emitw;
      }
      const bool gF = go && isF, gD = go && isDB, gW = go && isW;
      const int sl1 = (sl + 1 == R) ? 0 : sl + 1;
      first = (go && pos == 0) ? start : first;
      clk = go ? end : clk;
      busy += go ? dur : 0;
      mem += go ? dmem : 0;
      peak = imax(peak, mem);
      linkF = gF ? nl : linkF;
      linkB = gD ? nl : linkB;
      nF += gF ? 1 : 0;
      nD += gD ? 1 : 0;
      slF = gF ? sl1 : slF;
      slD = gD ? sl1 : slD;
      wsub = gW ? (wfin ? 0 : wsub + 1) : wsub;
      nW += (gW && wfin) ? 1 : 0;
      if (kMode == MODE_SIM) comb = (go && !isF) ? (isB ? 1 : 2) : comb;
      if (kMode != MODE_SIM) last_fd = gF ? 1 : (gD ? 2 : last_fd);
      pos += go ? 1 : 0;
    }
    __syncwarp();

    // ------------------------------------------------------------------ completion (rare path)
    const unsigned b_go = __ballot_sync(FULL, go);
    const bool seg_idle = in_round && !(b_go & segmask);      // no block executed in this segment
    if (__any_sync(FULL, seg_idle)) {
      const bool act = in_round && s < c.p;
      const unsigned b_unfin = __ballot_sync(FULL, live);
      const unsigned b_ring = __ballot_sync(FULL, act && !kRingGlobal && nF - nD >= R && nF < c.m);
      const bool seg_complete = seg_idle && !(b_unfin & segmask);
      const bool seg_stuck = seg_idle && !seg_complete;
      bool badc = false;
      if (kMode == MODE_SIM && seg_complete && act)          // Q29 counts at the end of the walk
        badc = nF != c.m || nD != c.m || (comb != 1 && nW * c.nsub + wsub != c.nsub * nD);
      if (kMode == MODE_SIM && seg_stuck && act) {
        // cannot continue: a statically bad plan reports BAD_PLAN (precedence) -> scan the rest
        int cF = nF, cD = nD, cW = nW * c.nsub + wsub, cb = comb;
        for (int k = pos; k < plen && !badc; ++k) {
          const uint32_t wv = A.ops[(item * A.words + (k >> 4)) * A.stage_stride + s];
          const uint32_t code = (wv >> ((k & 15) << 1)) & 3u;
          if (code == CP_OP_F) { badc = cF >= c.m; ++cF; }
          else if (code == CP_OP_W) { badc = cW >= c.nsub * cD || cb == 1; ++cW; cb = 2; }
          else { badc = cD >= c.m || (code == CP_OP_B ? cb == 2 : cb == 1); ++cD; cb = (code == CP_OP_B) ? 1 : 2; }
        }
        if (!badc) badc = cF != c.m || cD != c.m || (cb != 1 && cW != c.nsub * cD);
      }
      const unsigned b_badc = __ballot_sync(FULL, badc);
      const unsigned b_mem = __ballot_sync(FULL, act && peak > c.mlim);
      int ms = act ? imax(clk + c.tdp, c.tagate) : 0;   // App. A runtime incl. DP tail / AG
      int pk = act ? peak : 0;
      for (int d = 1; d < W; d <<= 1) {
        ms = imax(ms, __shfl_xor_sync(FULL, ms, d, W));
        pk = imax(pk, __shfl_xor_sync(FULL, pk, d, W));
      }
      if (seg_idle) {
        int st;
        bool completed = false;
        if (b_badc & segmask) st = CPI_BAD_PLAN;
        else if (seg_stuck && (b_ring & segmask)) st = -1;
        else if (seg_stuck) st = CPI_DEADLOCK;
        else { completed = true; st = (b_mem & segmask) ? CPI_MEM_EXCEEDED : 0; }
        if (st == -1) {
          // a stage's F lead reached the ring capacity: re-run the item in the global-ring pass
          if (kMode == MODE_SWEEP) {
            if (s == 0) atomicMin(A.keys + item, KEY_OVER);            // host sizes R so this never happens
          } else if (s == 0) {
            const int slot = atomicAdd(A.ovf_count, 1);
            A.ovf_list[slot] = (int32_t)item;
          }
          need_load = true;
        } else if (kMode == MODE_SWEEP) {
          // one (point, candidate) task: its makespan and the point's packed argmin key
          if (completed && st == 0 && s == 0) {
            if (A.cand_ms) A.cand_ms[item * CP_N_CAND + cand] = ms;
            atomicMin(A.keys + item, ((unsigned long long)ms << 8) | (unsigned)cand);
          }
          need_load = true;
        } else {
          if (s == 0 && CHK(item, n_it, 13)) {
            A.makespan[item] = completed ? (long long)ms : -1LL;
            if (A.peak_mem) A.peak_mem[item] = completed ? pk : -1;
            A.status[item] = st;
            if (A.best_key && st == 0)
              atomicMin(A.best_key, ((unsigned long long)ms << 32) | (unsigned long long)(uint32_t)(item + A.index_base));
          }
          if (A.stage_stats && s < A.stage_stride) {
            const int4 v = (completed && s < c.p) ? make_int4(first, clk, busy, peak) : make_int4(0, 0, 0, 0);
            *reinterpret_cast<int4*>(A.stage_stats + (item * A.stage_stride + s) * 4) = v;
          }
          if (kMode == MODE_GREEDY && s < A.stage_stride) {
            const bool own = s < c.p;
            if (PW > 0) {
              for (int k = 0; own && k * 16 < pos; ++k)
                if (POK((k << 5) + lane, 10) && CHK(item * A.words + k, n_it * A.words, 16))
                  A.ops[(item * A.words + k) * A.stage_stride + s] = plan[(k << 5) + lane];
            } else if (own && (pos & 15)) {
              A.ops[(item * A.words + (pos >> 4)) * A.stage_stride + s] = emitw;
            }
            emitw = 0;
          }
          finish_rows(item, (kMode == MODE_GREEDY && s < c.p) ? pos : 0);
          need_load = true;
        }
        if (use_tma && need_load) { cur_buf ^= 1; plan_off = cur_buf * PW * 32 + lane; }
      }
      any_load = __any_sync(FULL, need_load);
    }
  }
}

// sweep shard initialisation: keys of the launch's point set = INT64_MAX, candidate makespans = -1
__global__ void k_sweep_init(unsigned long long* keys, int32_t* cand_ms, SweepSet q) {
  const long long n = sweep_npts(q);
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n; j += (long long)gridDim.x * blockDim.x) {
    const long long k = sweep_point_of(q, j);
    keys[k] = KEY_NONE;
    if (cand_ms)
      for (int c = 0; c < CP_N_CAND; ++c) cand_ms[k * CP_N_CAND + c] = -1;
  }
}

int launch_sweep_init(unsigned long long* keys, int32_t* cand_ms, long long lo, long long hi, long long inner, int own_lo,
                      int own_hi, void* stream) {
  const SweepSet q{lo, hi, inner, own_lo, own_hi};
  const long long n = sweep_npts(q);
  const int blocks = (int)std::min<long long>(1024, (n + 255) / 256);
  k_sweep_init<<<blocks > 0 ? blocks : 1, 256, 0, (cudaStream_t)stream>>>(keys, cand_ms, q);
  return (int)cudaGetLastError();
}

template <int kMode, bool kRG, bool kTL>
static void* kernel_ptr() { return (void*)k_engine<kMode, kRG, kTL>; }

static void* pick(Mode mode, bool rg, bool tl) {
  switch (mode) {
    case MODE_SIM:
      return rg ? (tl ? kernel_ptr<MODE_SIM, true, true>() : kernel_ptr<MODE_SIM, true, false>())
                : (tl ? kernel_ptr<MODE_SIM, false, true>() : kernel_ptr<MODE_SIM, false, false>());
    case MODE_GREEDY:
      return rg ? (tl ? kernel_ptr<MODE_GREEDY, true, true>() : kernel_ptr<MODE_GREEDY, true, false>())
                : (tl ? kernel_ptr<MODE_GREEDY, false, true>() : kernel_ptr<MODE_GREEDY, false, false>());
    default: return rg ? kernel_ptr<MODE_SWEEP, true, false>() : kernel_ptr<MODE_SWEEP, false, false>();
  }
}

int launch_engine(Mode mode, bool ring_global, const Args& a, int blocks, int threads, size_t smem, void* stream) {
  void* fn = pick(mode, ring_global, a.t_start != nullptr);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return (int)e;
  }
  void* params[] = {(void*)&a};
  cudaError_t e = cudaLaunchKernel(fn, dim3(blocks), dim3(threads), params, smem, (cudaStream_t)stream);
  return (int)e;
}

int engine_blocks_per_sm(Mode mode, bool ring_global, int threads, size_t smem, bool timeline) {
  void* fn = pick(mode, ring_global, timeline);
  if (smem > 48 * 1024) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, threads, smem) != cudaSuccess) return 1;
  return n > 0 ? n : 1;
}

int device_sm_count() {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 148;
  return n;
}

}  // namespace cpk

#ifdef CP_DEBUG
extern "C" int cp_debug_read(int* out8) {
  cudaDeviceSynchronize();
  return (int)cudaMemcpyFromSymbol(out8, cpk::cp_dbg, 8 * sizeof(int));
}
#endif
