// greedy_fast.cu -- fast path of cp_greedy (Alg. 1 + §4.2.2, round-parallel) for
// batches without a per-entry timeline.  The segment width W (8, 16 or 32 lanes = stages) is a
// compile-time constant, so the two causal-horizon scans unroll to log2(W) shuffle steps, and
// 32/W instances share a warp.  Same semantics as k_engine<MODE_GREEDY> (engine.cu), which
// remains the GPU path for timelines and for the global-ring fix-up pass.
//
// Per round, every lane (stage) forms its eligible set from register state and the two heads
// of its shared-memory arrival rings, computes its schedulable time t*_s, and decides iff
// t*_s < min(L_s, R_s) (two min-plus warp scans).  Execution is branch-free; the emitted 2-bit
// plan word is stored straight to global memory (predicated) whenever it fills.  Loading a new
// instance and classifying a finished one happen on a rare, warp-uniform path.
#include <cuda_runtime.h>
#include <stdint.h>

#include "engine.h"
#include "grid_synth.cuh"

// Debug builds only (make variant V=... DEFS=-DGREEDY_DBG_ROUNDS=N; tools/greedy_rounds.py,
// greedy_task_times.py, greedy_task_starts.py): a sweep task's cand_ms gets, instead of its
// makespan, 1 = its round count, 2 = its duration (0.1 us), 3 = its start time (globaltimer / 100).
#ifndef GREEDY_DBG_ROUNDS
#define GREEDY_DBG_ROUNDS 0
#endif

namespace cpk {

namespace {
constexpr int32_t GINF = 1 << 30;
constexpr unsigned GFULL = 0xffffffffu;
__device__ __forceinline__ int gmin(int a, int b) { return a < b ? a : b; }
__device__ __forceinline__ int gmax(int a, int b) { return a > b ? a : b; }
// x + g * d as an integer multiply-add: conditional state updates issue on the FMA pipe (the
// round is ALU-pipe bound; a SEL would land on the ALU pipe)
__device__ __forceinline__ int gmadd(int g, int d, int x) {
  int r;
  asm("mad.lo.s32 %0, %1, %2, %3;" : "=r"(r) : "r"(g), "r"(d), "r"(x));
  return r;
}
}  // namespace

// kGrid = false: cp_greedy -- instances from memory, plans + metrics out.
// kGrid = true : cp_sweep_shard's greedy candidates -- (point, candidate) tasks from a device
//                counter, instances synthesized from the grid (grid_synth.cuh), no plan output;
//                the candidate's makespan and the point's packed argmin key out.
// Output rows r = s, s + W, ... < stage_stride of an item: len, every plan word past the emitted
// entries zeroed (outputs are fully defined, whatever the caller's buffer held) and, for rows no
// lane owns, zero stats.  The row's own partial last word is written by the caller.
__device__ __noinline__ void greedy_finish_rows(const Args& A, long long it, int s, int W, int used, bool stats_own) {
  for (int r = s; r < A.stage_stride; r += W) {
    const int u = r == s ? used : 0;
    const long long rb = it * A.stage_stride + r;
    for (int k = (u + 15) >> 4; k < A.words; ++k) A.ops[(it * A.words + k) * A.stage_stride + r] = 0u;
    A.len[rb] = (uint16_t)u;
    if (A.stage_stats && (r != s || stats_own)) *reinterpret_cast<int4*>(A.stage_stats + rb * 4) = make_int4(0, 0, 0, 0);
  }
}

template <int W, bool kGrid>
__global__ void __launch_bounds__(kFastThreads, kGreedyMinBlocks) k_greedy_fast(const __grid_constant__ Args A) {
  extern __shared__ __align__(128) int32_t smem[];
  constexpr int NSEG = 32 / W;
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int s = lane & (W - 1);
  const int seg = lane / W;
  const unsigned segmask = (W == 32) ? GFULL : (((1u << W) - 1u) << (seg * W));
  const int R = A.ring_slots;
  const int RW = R * 32;
  const long long gwarp = (long long)blockIdx.x * (blockDim.x >> 5) + wib;
  const long long nwarps = (long long)gridDim.x * (blockDim.x >> 5);
  const int Rm = R - 1;                              // R is a power of two: slot = count & Rm
  // per-warp smem (words): [params 6*32 int4][ringF R*32][ringD R*32]
  const int wbase = wib * A.smem_words_per_warp;
  const int iF = wbase + kGreedyTableWords + lane, iD = iF + RW;
  int* const ringF = smem + iF;                        // this lane's ring columns (slot k at [k << 5])
  int* const ringD = smem + iD;
  int4* const tab = reinterpret_cast<int4*>(smem + wbase) + lane;    // [entry][lane]
  // stage 0's F ring is never written by a producer: it must read 0 (cleared once)
  for (int k = lane; k < 2 * RW; k += 32) smem[wbase + kGreedyTableWords + k] = 0;
  __syncwarp();

  long long task = gwarp * NSEG + seg;
  const long long tstride = nwarps * NSEG;

  // per-lane instance constants
  int p = 0, m = 0, nsub = 1, tf = 0, td = 0, tw = 0, wq = 0, wr = 0, mf = 0, md = 0, mw = 0, mlim = 0;
  int tdp = 0, tag = 0, latF = 0, bwF = 0, latB = 0, bwB = 0, P = 0, Q = 0, lmF = 0;
  int PL = 0, QR = 0;                                  // horizon offsets (P, Q; +-GINF at the segment edges)
  bool lastS = false;
  int offF = 1, offD = -1;                             // F / D send target relative to the ring head
  // per-lane state
  int clk = 0, mem = 0, peak = 0, nF = 0, nD = 0, nW = 0, wsub = 0;
  int linkF = 0, linkB = 0, pos = 0, lastF = 0;       // lastF: the last full F/D block was an F
  uint32_t emitw = 0;
  // (out of line: inlined, this rare-path code changed the round's register allocation)
  auto finish_rows = [&](long long it, int used, bool stats_own) {
    if (!kGrid) greedy_finish_rows(A, it, s, W, used, stats_own);
  };
  long long item = -1;
  int cand = 0;                                        // sweep: candidate id (2/3/4 = greedy n_sub 1/2/4)
  bool need = true, done = false;
#if GREEDY_DBG_ROUNDS
  int dbg_rounds = 0;
  unsigned long long dbg_t0 = 0;
#endif

  for (;;) {
    // ------------------------------------------------------------------ rare: (re)load instances
    while (__any_sync(GFULL, need)) {
      bool fresh = false;
      int lat_b_s = 0, bw_b_s = 0, st0 = 0;
      if (need) {
        if (kGrid) {
          long long t = 0;
          if (s == 0) t = atomicAdd(A.sweep_counter, 1ull);
          t = __shfl_sync(segmask, t, seg * W);
          item = sweep_task(A.grid.cand_mask & ((1u << CP_N_CAND) - 1u), SweepSet{A.pt_lo, A.pt_hi, A.blk_inner, A.own_lo, A.own_hi},
                        t, cand);
        } else if (A.work_counter) {                     // dynamic: instances handed out by a counter
          long long t = 0;
          if (s == 0) t = atomicAdd(A.work_counter, 1);
          t = __shfl_sync(segmask, t, seg * W);
          item = t < A.n_items ? t : -1;
        } else {
          item = task < A.n_items ? task : -1;
          task += tstride;
        }
        need = false;
        fresh = item >= 0;
        p = m = 0;
        if (!fresh) { mlim = -1; nF = nD = nW = lmF = 0; }   // no instance: nothing eligible (see the round)
        if (fresh) {
          bool zero1;
          tf = td = tw = mf = md = mw = mlim = tdp = tag = latF = bwF = latB = bwB = 0;
          if (kGrid) {
            const GridLane g = grid_lane(A.grid, item, s);
            p = g.p; m = g.m; nsub = 1 << (cand - 2);
            zero1 = g.zero1;
            tf = g.tf; td = g.td; tw = g.tw; mf = g.mf; md = g.md; mw = g.mw; mlim = g.mlim;
            tdp = g.tdp; tag = g.tag;
            latF = g.latF; bwF = g.bwF; latB = g.latB; bwB = g.bwB;
            lat_b_s = latF; bw_b_s = bwF;
          } else {
            const cp_inst_v1* I = A.inst + (A.n_inst == 1 ? 0 : item);
            p = I->n_pp; m = I->n_mb; nsub = I->n_sub;
            zero1 = I->flags & 1;
            if (s < p) {
              tf = I->t_f[s]; td = I->t_d[s]; tw = I->t_w[s];
              mf = I->m_f[s]; md = I->m_d[s]; mw = I->m_w[s]; mlim = I->m_lim[s];
              tdp = I->t_dp[s]; tag = I->t_ag[s];
              if (s < p - 1) { latF = I->lat_f[s]; bwF = I->bw_f[s]; lat_b_s = I->lat_b[s]; bw_b_s = I->bw_b[s]; }
              if (s > 0) { latB = I->lat_b[s - 1]; bwB = I->bw_b[s - 1]; }
            }
          }
          bool bad = p < 1 || p > CP_MAX_STAGES || m < 1 || nsub < 1;
          if (!bad && s < p)
            bad = !(tf >= nsub && td >= nsub && tw >= nsub && nsub >= 1 && mf > 0 && md <= 0 && mw <= 0 &&
                    (long long)mf + md + mw == 0 && mlim >= mf && tdp >= 0 && tag >= 0 && latF >= 0 &&
                    bwF >= 0 && lat_b_s >= 0 && bw_b_s >= 0);
          if (!zero1) tag = 0;
          if (s >= p) mlim = -1;                // lanes past the last stage: no F can fit (see the round)
          st0 = bad ? CPI_BAD_INSTANCE : 0;
          if (!kGrid && !st0 && (long long)(2 + nsub) * m > 16LL * A.words) st0 = CPI_BAD_PLAN;
          if (!st0 && (p > W || m > CP_MAX_MB || nsub > CP_MAX_SUB)) st0 = CPI_OVERFLOW;
          wq = tw / (nsub > 0 ? nsub : 1);
          wr = tw % (nsub > 0 ? nsub : 1);
          lmF = s == 0 ? m : 0;                 // stage 0 has no F producer: all m available
          lastS = s == p - 1;
          // Sends without a consumer need no test: stage 0's D goes into the D slot it has just
          // consumed (message nD + R is sent only after this round: the ring bound nF - nD < R orders
          // it after this op), the last stage's F into its own D ring at slot nF -- its D follows its
          // own F, and the F's end (<= clk when that D is considered) reads like the cleared 0.
          offF = lastS ? RW : 1;
          offD = s == 0 ? 0 : -1;
          clk = mem = peak = nF = nD = nW = wsub = linkF = linkB = pos = lastF = 0;
          emitw = 0;
#if GREEDY_DBG_ROUNDS
          dbg_rounds = 0;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(dbg_t0));
#endif
          // the last stage's D ring may hold a larger instance's arrivals or an earlier instance's F
          // ends: it must read 0
          if (lastS)
            for (int k = 0; k < R; ++k) smem[iD + (k << 5)] = 0;
          // parameter table: 0 = F, 1 = D (W sub-blocks are computed from wq, wr, m_w in the round)
          tab[0 * 32] = make_int4(tf, mf, bwF, latF);
          tab[1 * 32] = make_int4(td, md, bwB, latB);
        }
      }
      // warp-wide: lookahead prefix sums (segment scans), horizon bound, status ballots
      const bool act = fresh && s < p && st0 == 0;
      const int cf = act ? tf + bwF + latF : 0;       // hop s -> s+1 (F)
      const int cd = act ? td + bwB + latB : 0;       // hop s -> s-1 (D)
      long long u = act ? (long long)m * ((long long)tf + td + tw) + tag + tdp +
                              (long long)m * ((long long)latF + bwF + latB + bwB) : 0;
      int pf = cf, qd = cd;
#pragma unroll
      for (int d = 1; d < W; d <<= 1) {
        const int a = __shfl_up_sync(GFULL, pf, d, W);
        const int b = __shfl_up_sync(GFULL, qd, d, W);
        if (s >= d) { pf += a; qd += b; }
      }
#pragma unroll
      for (int d = 1; d < W; d <<= 1) u += __shfl_xor_sync(GFULL, u, d, W);
      // sweep: a greedy candidate with a block shorter than n_sub ticks (reading Q12) is skipped --
      // no key, cand_ms -1;
      // a task whose ring lead bound min(m, max_s floor(M_L/m_f)) lies outside this
      // launch's tier is left to the launch sized for it
      unsigned b_skip = 0u;
      if (kGrid) {
        int lead = (fresh && s < p && mf > 0) ? mlim / mf : 0;
#pragma unroll
        for (int d = 1; d < W; d <<= 1) lead = gmax(lead, __shfl_xor_sync(GFULL, lead, d, W));
        lead = gmin(lead, m);
        b_skip = __ballot_sync(GFULL, fresh && ((s < p && (tf < nsub || td < nsub || tw < nsub)) ||
                                                 lead < A.tier_lo || lead > A.tier_hi));
      }
      const unsigned b_inst = __ballot_sync(GFULL, fresh && st0 == CPI_BAD_INSTANCE);
      const unsigned b_plan = __ballot_sync(GFULL, fresh && st0 == CPI_BAD_PLAN);
      const unsigned b_over = __ballot_sync(GFULL, fresh && st0 == CPI_OVERFLOW);
      if (fresh) {
        P = pf - cf;
        Q = qd;
        // At the segment edges the width-W shuffles return the lane's own scan value, so L_0 and
        // R_{W-1} would come out as t*; offsetting them by GINF makes them exceed any t* < GINF.
        PL = s == 0 ? P + GINF : P;
        QR = s == W - 1 ? Q - GINF : Q;
        int st = (b_inst & segmask) ? CPI_BAD_INSTANCE
                 : (b_plan & segmask) ? CPI_BAD_PLAN
                 : (b_over & segmask) ? CPI_OVERFLOW : 0;
        if (!st && u >= (long long)GINF) st = CPI_OVERFLOW;      // int32 horizon guard (Q21)
        if (kGrid) {
          if (st == CPI_OVERFLOW && s == 0) atomicMin(A.keys + item, KEY_OVER);
          if (st || (b_skip & segmask)) need = true;
        } else if (st) {
          if (s == 0) {
            A.makespan[item] = -1;
            if (A.peak_mem) A.peak_mem[item] = -1;
            A.status[item] = st;
          }
          finish_rows(item, 0, true);             // len 0, every word 0, stats 0
          need = true;
        }
      }
      if (__all_sync(GFULL, item < 0)) { done = true; break; }
    }                                                    // (failed items load again)
    if (done) break;
    const bool hasItem = item >= 0;                      // fixed until the next reload
    unsigned segmaskH = hasItem ? segmask : 0u;          // this segment's lanes if it holds an instance
    asm("mov.b32 %0, %0;" : "+r"(segmaskH));             // kept in a register (not re-derived per round)
    const bool onS = hasItem && s < p;
    for (;;) {
      __syncwarp();                                        // last round's ring stores -> these reads
#if GREEDY_DBG_ROUNDS
      ++dbg_rounds;
#endif

      // ------------------------------------------------------------------ one round
      // Eligibility without a liveness term: F needs leftF > nF, and leftF <= m (stage 0: leftF = m);
      // D needs rightD > nD with rightD <= m; W needs nW < nD <= m.  Lanes past the last stage (and
      // segments without an instance) hold m_lim = -1, so their F never fits, and no D / W counts.
      const int leftF = gmax(__shfl_up_sync(GFULL, nF, 1, W), lmF);
      const int rD0 = __shfl_down_sync(GFULL, nD, 1, W);
      const int rightD = lastS ? nF : rD0;                // the last stage's D follows its own F
      // ring heads (byte offsets: one mask and one multiply-add each)
      int* const hF = reinterpret_cast<int*>(reinterpret_cast<char*>(ringF) + ((nF & Rm) << 7));
      int* const hD = reinterpret_cast<int*>(reinterpret_cast<char*>(ringD) + ((nD & Rm) << 7));
      const int availF = gmax(*hF, tag);
      const int availD = *hD;
      const bool hasF = (leftF > nF) & (mem + mf <= mlim);   // Q15
      // D / W: rightD >= nD and nD >= nW always, so max(n - bound + 1, 0) is 1 exactly when the op is
      // not eligible, and a multiply-add lifts its time past GINF (times stay below 2^30)
      const int fD = gmadd(gmax(nD - rightD + 1, 0), GINF, availD);
      const int fW = gmadd(gmax(nW - nD + 1, 0), GINF, clk);
      const int mnv = gmin(gmin(hasF ? availF : GINF, fD), fW);
      const int tstar = gmax(clk, mnv);                   // §4.2.2 :419 (GINF when nothing is eligible)
      // causal horizon: L_s = P_s + min_{k<s}(t*_k - P_k), R_s = min_{k>s}(t*_k + Q_k) - Q_s.
      // Width-W shuffles return the lane's own value past the segment edge, so the scans need no
      // lane predicates (min with itself).
      // Radix-3 steps (two shuffles, one 3-input min each; ceil(log3 W) steps): fewer ALU-pipe mins
      // than log2 W min steps and a shorter dependency chain.
      int x = tstar - P, y = tstar + Q;
  #pragma unroll
      for (int d = 1; d < W; d *= 3) {
        const int a1 = __shfl_up_sync(GFULL, x, d, W), b1 = __shfl_down_sync(GFULL, y, d, W);
        if (2 * d < W) {                                   // (a shift of W or more returns x itself)
          const int a2 = __shfl_up_sync(GFULL, x, 2 * d, W), b2 = __shfl_down_sync(GFULL, y, 2 * d, W);
          x = gmin(gmin(x, a1), a2);
          y = gmin(gmin(y, b1), b2);
        } else {
          x = gmin(x, a1);
          y = gmin(y, b1);
        }
      }
      const int xe = __shfl_up_sync(GFULL, x, 1, W);
      const int ye = __shfl_down_sync(GFULL, y, 1, W);
      const int Lh = PL + xe;                              // (lanes with t* = GINF cannot go: overflow is harmless)
      const int Rh = ye - QR;
      // operation selection (Q13): opposite of the last full F/D block, then the other, then W
      const bool cF = hasF & (availF <= tstar), cD = fD <= tstar;
      const bool pD = cD & ((lastF != 0) | !cF);
      const bool pF = !pD & cF;
      // an F whose consumer ring is full (lead would exceed R: undersized ring hint) is not executed:
      // the lane stalls and the item is re-run by the global-ring fix-up pass (decisions unchanged)
      // (t* < GINF matters: an idle neighbour's horizon term can exceed GINF)
      // (sweep: rings hold the lead bound min(m, floor(M_L / m_f)), and memory caps nF - nD at it --
      // mem >= (nF - nD) m_f since m_d, m_w <= 0 and m_f + m_d + m_w = 0 -- so they cannot fill)
      const bool go = (tstar < GINF) & (tstar < gmin(Lh, Rh)) & (kGrid || !(pF & (nF - nD >= R)));
      const bool pW = !pD & !pF;
      const bool wfin = wsub + 1 == nsub;
      const int4 ta = tab[pF ? 0 : 32];                    // F or D row: {duration, memory delta, link bw, latency}
      // a W sub-block (Q12): duration wq + (sub-block index < t_w mod n_sub), memory delta m_w at the last
      int wdur;                                            // wq + (wsub < wr): the borrow bit of wsub - wr, by IMAD.HI
      asm("mad.hi.u32 %0, %1, 2, %2;" : "=r"(wdur) : "r"(wsub - wr), "r"(wq));
      const int dur = pW ? wdur : ta.x;
      const int dmv = pW ? (wfin ? mw : 0) : ta.y;
      const int end = tstar + dur;
      const int nl = gmax(end, pF ? linkF : linkB) + ta.z;   // FIFO link clock (App. X1)
      if (go & !pW) *(pF ? hF + offF : hD + offD) = nl + ta.w;
      // emit the 2-bit entry into a shift register (the newest entry enters at bits 30-31, so after
      // 16 entries entry k sits at bits 2k); a full word goes straight to global memory
      const int gi = go ? 1 : 0, gFi = (go & pF) ? 1 : 0, gDi = (go & pD) ? 1 : 0;
      if (!kGrid) {
        // (integer multiply-adds: the FMA pipe has room, the ALU pipe binds)
        // code << 30 = W - gFi (W - F) - gDi (W - D), valid when go
        static_assert(CP_OP_F == 0u && CP_OP_D == 2u && CP_OP_W == 3u, "op codes");
        const int code30 = gmadd(gFi, 0x40000000, gmadd(gDi, (int)0xC0000000u, (int)0xC0000000u));
        uint32_t w1;                                       // (emitw >> 2) + code30 in one IMAD.HI
        asm("mad.hi.u32 %0, %1, %2, %3;" : "=r"(w1) : "r"(emitw), "r"(0x40000000u), "r"(code30));
        const bool flush = go & ((pos & 15) == 15);
        if (flush) A.ops[(item * A.words + (pos >> 4)) * A.stage_stride + s] = w1;
        emitw = (uint32_t)gmadd(gi, (int)(w1 - emitw), (int)emitw);
      }
      const bool gW = go & pW;
      clk = gmadd(gi, end - clk, clk);
      mem = gmadd(gi, dmv, mem);
      if (!kGrid) peak = gmax(peak, mem);                 // (sweep: F's memory test keeps mem <= M_L)
      linkF = gmadd(gFi, nl - linkF, linkF);
      linkB = gmadd(gDi, nl - linkB, linkB);
      nF = gmadd(gFi, 1, nF);
      nD = gmadd(gDi, 1, nD);
      wsub = gW ? (wfin ? 0 : wsub + 1) : wsub;
      nW = gmadd((gW & wfin) ? 1 : 0, 1, nW);
      lastF = gmadd(lastF, gmadd(gFi, -1, gmadd(gDi, -1, 1)), gFi);   // F -> 1, D -> 0, else kept
      pos = gmadd(gi, 1, pos);

      // ------------------------------------------------------------------ rare: a segment went idle
      bool idle, any_idle;
      if constexpr (W == 32) {                             // one segment: idle is warp-uniform
        idle = (segmaskH != 0u) & !__any_sync(GFULL, go);
        any_idle = idle;
      } else {
        const unsigned bgo = __ballot_sync(GFULL, go);
        idle = (segmaskH != 0u) & ((bgo & segmaskH) == 0u);
        any_idle = __any_sync(GFULL, idle);
      }
      if (any_idle) {
        const unsigned b_unfin = __ballot_sync(GFULL, onS && nW < m);
        const unsigned b_ring = __ballot_sync(GFULL, item >= 0 && s < p && nF < m && nF - nD >= R);
        const unsigned b_mem = __ballot_sync(GFULL, item >= 0 && s < p && peak > mlim);
        const bool complete = idle && !(b_unfin & segmask);
        const bool on = item >= 0 && s < p;
        int ms = on ? gmax(clk + tdp, tag) : 0, pk = on ? peak : 0;
  #pragma unroll
        for (int d = 1; d < W; d <<= 1) {
          ms = gmax(ms, __shfl_xor_sync(GFULL, ms, d, W));
          pk = gmax(pk, __shfl_xor_sync(GFULL, pk, d, W));
        }
        // first_start = max-plus prefix over F_0's path (every row starts with F_0)
        const int cfw = on ? tf + bwF + latF : 0;
        int Pf = cfw;
  #pragma unroll
        for (int d = 1; d < W; d <<= 1) { const int t = __shfl_up_sync(GFULL, Pf, d, W); if (s >= d) Pf += t; }
        Pf -= cfw;
        int xf = (on ? tag : 0) - Pf;
  #pragma unroll
        for (int d = 1; d < W; d <<= 1) { const int t = __shfl_up_sync(GFULL, xf, d, W); if (s >= d) xf = gmax(xf, t); }
        if (idle) {
          if (kGrid) {
            // one (point, candidate) task: its makespan and the point's packed argmin key.  The
            // host sizes R to the lead bound, so a full ring cannot occur (it would mark the point
            // unevaluated rather than guess); the greedy never deadlocks or exceeds memory (Q15).
            if (s == 0) {
              if (!complete) atomicMin(A.keys + item, KEY_OVER);
              else if (!(b_mem & segmask)) {
#if GREEDY_DBG_ROUNDS
                unsigned long long t1;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
                if (A.cand_ms) A.cand_ms[item * CP_N_CAND + cand] = GREEDY_DBG_ROUNDS == 2 ? (int)((t1 - dbg_t0) / 100)
                                 : GREEDY_DBG_ROUNDS == 3 ? (int)((dbg_t0 / 100) & 0x3fffffff) : dbg_rounds;
#else
                if (A.cand_ms) A.cand_ms[item * CP_N_CAND + cand] = ms;
#endif
                atomicMin(A.keys + item, ((unsigned long long)ms << 8) | (unsigned)cand);
              }
            }
          } else if (!complete && (b_ring & segmask)) {
            // ring capacity reached (host under-sized R): re-run in the global-ring fix-up pass
            if (s == 0) { const int slot = atomicAdd(A.ovf_count, 1); A.ovf_list[slot] = (int32_t)item; }
          } else {
            const int st = !complete ? CPI_DEADLOCK : ((b_mem & segmask) ? CPI_MEM_EXCEEDED : 0);
            if (s == 0) {
              A.makespan[item] = complete ? (long long)ms : -1LL;
              if (A.peak_mem) A.peak_mem[item] = complete ? pk : -1;
              A.status[item] = st;
            }
            if (A.stage_stats && s < A.stage_stride) {
              const int4 v = (complete && on) ? make_int4(Pf + xf, clk, m * (tf + td + tw), peak) : make_int4(0, 0, 0, 0);
              *reinterpret_cast<int4*>(A.stage_stats + (item * A.stage_stride + s) * 4) = v;
            }
            if (on && (pos & 15) && s < A.stage_stride)         // the partial word, aligned to bit 0
              A.ops[(item * A.words + (pos >> 4)) * A.stage_stride + s] = emitw >> (32 - 2 * (pos & 15));
            finish_rows(item, on ? pos : 0, false);
          }
          need = true;
        }
        break;                                           // reload the finished segments
      }
    }
  }
}

template <int W, bool kGrid>
static int launch_w(const Args& a, int blocks, int threads, size_t smem, void* stream) {
  const void* fn = (const void*)k_greedy_fast<W, kGrid>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return (int)e;
  }
  void* params[] = {(void*)&a};
  return (int)cudaLaunchKernel(fn, dim3(blocks), dim3(threads), params, smem, (cudaStream_t)stream);
}

template <int W, bool kGrid>
static int bps_w(int threads, size_t smem) {
  const void* fn = (const void*)k_greedy_fast<W, kGrid>;
  if (smem > 48 * 1024) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, threads, smem) != cudaSuccess) return 1;
  return n > 0 ? n : 1;
}

int launch_greedy_fast(int W, bool grid, const Args& a, int blocks, int threads, size_t smem, void* stream) {
  if (grid)
    return W == 8 ? launch_w<8, true>(a, blocks, threads, smem, stream)
                  : (W == 16 ? launch_w<16, true>(a, blocks, threads, smem, stream)
                             : launch_w<32, true>(a, blocks, threads, smem, stream));
  return W == 8 ? launch_w<8, false>(a, blocks, threads, smem, stream)
                : (W == 16 ? launch_w<16, false>(a, blocks, threads, smem, stream)
                           : launch_w<32, false>(a, blocks, threads, smem, stream));
}

int greedy_fast_blocks_per_sm(int W, bool grid, int threads, size_t smem) {
  if (grid)
    return W == 8 ? bps_w<8, true>(threads, smem) : (W == 16 ? bps_w<16, true>(threads, smem) : bps_w<32, true>(threads, smem));
  return W == 8 ? bps_w<8, false>(threads, smem) : (W == 16 ? bps_w<16, false>(threads, smem) : bps_w<32, false>(threads, smem));
}

}  // namespace cpk
