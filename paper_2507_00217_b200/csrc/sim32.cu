// sim32.cu -- fast path of cp_simulate for the dominant shape: one item per warp (17..32
// stages, stage_stride 32), plan rows staged in shared memory by double-buffered TMA bulk
// copies, arrival rings in shared memory; optionally the per-entry timeline (kTL), staged in
// shared memory and written 8 start ticks (32 B) per lane at a time.
//
// Same semantics as k_engine<MODE_SIM> (engine.cu), which remains the reference GPU path for
// every other shape; both are parity-tested.  What makes this kernel fast is what
// it leaves out: the warp is one segment, so the "no block executed this round" test is a single
// ballot with a warp-uniform branch; the state is the minimum the §3.5 recurrence needs; entries
// past a row's end read as a never-ready D, so the round has no position test.  The round is
// bound by shared-memory wavefronts and issue together: per-code values that are
// the same for every lane come from broadcast rows, per-lane costs from one 128-bit row.
//
// Launches (abi.cpp): a first pass with 8-slot rings and occupancy backpressure over all items;
// items that stalled on a full ring (cyclic backpressure) are re-run by a second launch of this
// kernel over the overflow list with rings of R > n_mb slots, where no ring can fill.
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "engine.h"
#include "ptx.cuh"

#ifdef SIM32_MINB
#define SIM32_LB kFastThreads, SIM32_MINB
#else
#define SIM32_LB kThreads
#endif

namespace cpk {

namespace {
constexpr int32_t INF32 = 1 << 30;
constexpr unsigned FULLM = 0xffffffffu;
__device__ __forceinline__ int mn(int a, int b) { return a < b ? a : b; }
__device__ __forceinline__ int mx(int a, int b) { return a > b ? a : b; }
// x + g * d as an integer multiply-add: keeps conditional state updates on the FMA pipe
// (the kernel is ALU-pipe bound; a SEL would land on the ALU pipe)
__device__ __forceinline__ int madd(int g, int d, int x) {
  int r;
  asm("mad.lo.s32 %0, %1, %2, %3;" : "=r"(r) : "r"(g), "r"(d), "r"(x));
  return r;
}
// timeline staging: the 8 start ticks in the lane's slots [k][lane], k < 8, -> two 16-B global stores
__device__ __forceinline__ void tl_flush8(unsigned stg, int32_t* dst) {
  int v[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v[k]) : "r"(stg + 128u * k));
  __stcs(reinterpret_cast<int4*>(dst), make_int4(v[0], v[1], v[2], v[3]));
  __stcs(reinterpret_cast<int4*>(dst) + 1, make_int4(v[4], v[5], v[6], v[7]));
}
}  // namespace

template <bool kTL>   // kTL: per-entry start ticks requested (A.t_start; len_stride % 8 == 0, 32-B aligned rows)
__global__ void __launch_bounds__(SIM32_LB) k_sim32(const __grid_constant__ Args A) {
  extern __shared__ __align__(128) int32_t smem[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int R = A.ring_slots;
  const int RW = R * 32;
  const int PW = A.plan_words;                    // == words (host guarantees)
  const int PWr = PW + 1;                         // one spare row per buffer
  const long long gwarp = (long long)blockIdx.x * (blockDim.x >> 5) + wib;
  const long long nwarps = (long long)gridDim.x * (blockDim.x >> 5);
  const Sim32Layout Ly = sim32_layout(R, PW, A.shared_tab != 0, kTL);
  const int wbase = Ly.hdr + wib * Ly.per_warp;
  const int rbase = wbase + Ly.rings;
  const int pbase0 = wbase + Ly.plan;
  const int dum_row = Ly.dum;                     // relative to wbase
  const int zero_row = Ly.zero;
  const int tbase = A.shared_tab ? Ly.tabA : wbase + Ly.tabA;   // tabA (and tabC after it): block or warp
  uint32_t* const plan = reinterpret_cast<uint32_t*>(smem + pbase0);
  uint64_t* const bars = reinterpret_cast<uint64_t*>(smem + wbase + Ly.bars);
  int4* const tabA = reinterpret_cast<int4*>(smem + tbase) + lane;          // [code][lane]
  int4* const U = reinterpret_cast<int4*>(smem + Ly.uni);                  // [8] int4, block header
  const uint32_t plan_bytes = (uint32_t)A.words * 32u * 4u;
  // items: [0, n_items), or (fix-up pass) the overflow list of the first pass
  const long long n_items = A.from_list ? (long long)*(volatile int32_t*)A.ovf_count : (long long)A.n_items;
  auto item_of = [&](long long t) -> long long { return A.from_list ? (long long)A.ovf_list[t] : t; };

  // second pass over the overflow list: warps beyond the list leave before touching shared memory
  // (an empty list then costs one short launch)
  if (A.from_list && gwarp >= n_items) return;
  // items: a static stride, or (A.work_counter) handed out by a counter, fetched two items ahead
  // because the plan of the next item is prefetched while the current one runs
  const bool dyn = A.work_counter != nullptr && !A.from_list;
  const auto fetch = [&]() -> long long {
    int t = 0;
    if (lane == 0) t = atomicAdd(A.work_counter, 1);
    return (long long)__shfl_sync(FULLM, t, 0);
  };
  long long t_it = dyn ? fetch() : gwarp;
  long long t_nx = dyn ? fetch() : gwarp + nwarps;
  // the rings never written by a producer (stage 0's F ring) and the zero row read by W entries
  // must hold 0: clear both ring blocks and the zero row once
  for (int k = lane; k < 2 * RW; k += 32) smem[rbase + k] = 0;
  smem[wbase + zero_row + lane] = 0;
  if (lane == 0) { mbar_init(&bars[0]); mbar_init(&bars[1]); }
  __syncwarp();
  if (lane == 0 && t_it < n_items) tma_load_1d(plan, A.ops + item_of(t_it) * A.words * 32, plan_bytes, &bars[0]);
  uint32_t phase = 0;
  int buf = 0;

  int t_req = 0;                                   // the item after next (dynamic), in flight
  for (; t_it < n_items; t_it = t_nx, t_nx = dyn ? (long long)__shfl_sync(FULLM, t_req, 0) : t_nx + nwarps) {
    const long long item = item_of(t_it);
    if (dyn && lane == 0) t_req = atomicAdd(A.work_counter, 1);
    // ------------------------------------------------------------------ load (warp-uniform)
    const long long ii = A.inst_of ? (long long)A.inst_of[item] : (A.n_inst == 1 ? 0 : item);
    const cp_inst_v1* I = A.inst + ii;
    const int p = I->n_pp, m = I->n_mb, nsub = I->n_sub;
    const bool zero1 = I->flags & 1;
    const int s = lane;
    int tf = 0, td = 0, tw = 0, mf = 0, md = 0, mw = 0, mlim = 0, tdp = 0, tag = 0;
    int latF = 0, bwF = 0, latB = 0, bwB = 0, latbs = 0, bwbs = 0, plen = 0;
    if (s < p) {
      tf = I->t_f[s]; td = I->t_d[s]; tw = I->t_w[s];
      mf = I->m_f[s]; md = I->m_d[s]; mw = I->m_w[s]; mlim = I->m_lim[s];
      tdp = I->t_dp[s]; tag = I->t_ag[s];
      if (s < p - 1) { latF = I->lat_f[s]; bwF = I->bw_f[s]; latbs = I->lat_b[s]; bwbs = I->bw_b[s]; }
      if (s > 0) { latB = I->lat_b[s - 1]; bwB = I->bw_b[s - 1]; }
      plen = A.len[item * 32 + s];
    }
    bool bad = p < 1 || p > CP_MAX_STAGES || m < 1 || nsub < 1;
    if (!bad && s < p)
      bad = !(tf >= nsub && td >= nsub && tw >= nsub && nsub >= 1 && mf > 0 && md <= 0 && mw <= 0 &&
              (long long)mf + md + mw == 0 && mlim >= mf && tdp >= 0 && tag >= 0 && latF >= 0 && bwF >= 0 &&
              latbs >= 0 && bwbs >= 0);
    if (!zero1) tag = 0;
    long long u = (s < p && !bad) ? (long long)m * ((long long)tf + td + tw) + tag + tdp +
                                        (long long)m * ((long long)latF + bwF + latB + bwB)
                                  : 0;
    for (int d = 16; d > 0; d >>= 1) u += __shfl_xor_sync(FULLM, u, d);
    int st0 = 0;
    if (__any_sync(FULLM, bad)) st0 = CPI_BAD_INSTANCE;
    else if (__any_sync(FULLM, plen > 16 * A.words)) st0 = CPI_BAD_PLAN;
    else if (m > CP_MAX_MB || nsub > CP_MAX_SUB || u >= (long long)INF32) st0 = CPI_OVERFLOW;
    // this item's rows were prefetched into plan[buf]: wait, then prefetch the next item's
    mbar_wait(&bars[buf], (phase >> buf) & 1u);
    phase ^= 1u << buf;
    if (lane == 0 && t_nx < n_items)
      tma_load_1d(plan + (buf ^ 1) * PWr * 32, A.ops + item_of(t_nx) * A.words * 32, plan_bytes,
                  &bars[buf ^ 1]);
    buf ^= 1;
    if (st0) {
      if (lane == 0) {
        A.makespan[item] = -1;
        if (A.peak_mem) A.peak_mem[item] = -1;
        A.status[item] = st0;
      }
      if (A.stage_stats) *reinterpret_cast<int4*>(A.stage_stats + (item * 32 + s) * 4) = make_int4(0, 0, 0, 0);
      __syncwarp();
      continue;
    }
    const int wq = tw / nsub, wr = tw % nsub, tB = td + tw, mB = md + mw;
    const int fmask = s > 0 ? -1 : 0;             // lane consumes F arrivals
    const int dmask = s < p - 1 ? -1 : 0;         // lane consumes D arrivals
    const bool sendF = s < p - 1, sendD = s > 0 && s < p;
    // integer smem indices (shared window addressing, no generic pointers in the loop)
    const int iF = rbase + lane;                  // own F column
    const int iD = rbase + RW + lane;             // own D column
    const int iDum = wbase + dum_row + lane;      // store sink for lanes that send nothing
    const int iP = pbase0 + (buf ^ 1) * PWr * 32 + lane;   // this item's plan column (buf already flipped)

    // ---- Q29 count / mixing rules, once per row (popcounts over the staged words); the W-prefix
    // rule stays dynamic (a violating W entry stalls and the rare path classifies the item)
    bool bad_static = false;
    if (s < p) {
      int cF = 0, cB = 0, cD = 0, cW = 0;
      for (int k = 0; k * 16 < plen; ++k) {
        const uint32_t w = (uint32_t)smem[iP + (k << 5)];
        const int n = mn(16, plen - 16 * k);
        const uint32_t valid = (n == 16 ? 0xffffffffu : ((1u << (2 * n)) - 1u)) & 0x55555555u;
        const uint32_t lo = w & 0x55555555u, hi = (w >> 1) & 0x55555555u;
        cB += __popc(lo & ~hi & valid);
        cD += __popc(~lo & hi & valid);
        cW += __popc(lo & hi & valid);
      }
      cF = plen - cB - cD - cW;
      bad_static = cF != m || cB + cD != m || (cB > 0 && cD + cW > 0) || cW != nsub * cD;
    }
    if (__any_sync(FULLM, bad_static)) {
      if (lane == 0) {
        A.makespan[item] = -1;
        if (A.peak_mem) A.peak_mem[item] = -1;
        A.status[item] = CPI_BAD_PLAN;
      }
      if (A.stage_stats) *reinterpret_cast<int4*>(A.stage_stats + (item * 32 + s) * 4) = make_int4(0, 0, 0, 0);
      __syncwarp();
      continue;
    }

    // ------------------------------------------------------------------ rounds
    // ring heads are kept as pre-scaled word indices (own column + slot*32), wrapping at R slots
    const int iFend = iF + RW, iDend = iD + RW;
    int clk = 0, mem = 0, peak = 0, pos = 0;
    int nF = 0, nD = 0, went = 0, wcap = 0, wsub = 0, hF = iF, hD = iD, linkF = 0, linkB = 0;
    uint32_t wv = (uint32_t)smem[iP];             // plan word of entry `pos`, prefetched one round ahead
    auto rounds = [&](auto n1) {
      constexpr bool kN1 = decltype(n1)::value;   // n_sub == 1: a W entry is a whole W block
      for (;;) {
        // both neighbours' (nF, nD), 16 bits each, in one shuffle per direction
        const int cu = __shfl_up_sync(FULLM, nF | (nD << 16), 1);
        const int cd = __shfl_down_sync(FULLM, nF | (nD << 16), 1);
        const int leftF = cu & 0xffff, leftD = cu >> 16, rightF = cd & 0xffff, rightD = cd >> 16;
        const int aF = smem[hF];                  // both ring heads, independent of the entry type
        const int aD = smem[hD];
        const unsigned code = (wv >> ((pos & 15) << 1)) & 3u;
        const bool isF = code == CP_OP_F, isW = code == CP_OP_W, isB = code == CP_OP_B;
        const bool isDB = !isF & !isW;
        // readiness: input produced; room in the consumer's ring (occupancy < R: backpressure);
        // W sub-blocks only after their D
        const bool knowF = ((fmask == 0) | (leftF > nF)) & (!sendF | (nF - rightF < R));
        const bool knowD = ((dmask == 0) ? (nF > nD) : (rightD > nD)) & (!sendD | (nD - leftD < R));
        const bool wok = kN1 ? (went < nD) : (went < wcap);
        const bool go = (pos < plen) & (isF ? knowF : (isW ? wok : knowD));
        const int avail = isF ? mx(aF & fmask, tag) : (isW ? 0 : (aD & dmask));
        const int start = mx(clk, avail);
        const bool wfin = kN1 ? true : (wsub + 1 == nsub);
        const int wdur = kN1 ? tw : wq + (wsub < wr ? 1 : 0);
        const int dur = isF ? tf : (isW ? wdur : (isB ? tB : td));
        const int dm = isF ? mf : (isW ? (wfin ? mw : 0) : (isB ? mB : md));
        const int end = start + dur;
        const int nl = mx(end, isF ? linkF : linkB) + (isF ? bwF : bwB);   // FIFO link clock (App. X1)
        const bool send = go & (isF ? sendF : (isDB & sendD));
        smem[send ? (isF ? hF + 1 : hD - 1) : iDum] = nl + (isF ? latF : latB);
        if (kTL && go) A.t_start[(item * 32 + s) * (long long)A.len_stride + pos] = start;
        const int gi = go ? 1 : 0, gFi = (go & isF) ? 1 : 0, gDi = (go & isDB) ? 1 : 0;
        clk = madd(gi, end - clk, clk);
        mem = madd(gi, dm, mem);
        peak = mx(peak, mem);
        linkF = madd(gFi, nl - linkF, linkF);
        linkB = madd(gDi, nl - linkB, linkB);
        const int h1 = (isF ? hF : hD) + 32;
        hF = madd(gFi, (h1 == iFend ? iF : h1) - hF, hF);
        hD = madd(gDi, (h1 == iDend ? iD : h1) - hD, hD);
        nF = madd(gFi, 1, nF);
        nD = madd(gDi, 1, nD);
        went = madd((go & isW) ? 1 : 0, 1, went);
        if (!kN1) {
          wcap += gDi ? nsub : 0;
          wsub = (go & isW) ? (wfin ? 0 : wsub + 1) : wsub;
        }
        pos = madd(go ? 1 : 0, 1, pos);
        wv = (uint32_t)smem[iP + ((pos >> 4) << 5)];   // next round's word (spare row covers pos == 16*PW)
        __syncwarp();
        if (__ballot_sync(FULLM, go) == 0u) break;      // warp-uniform: nothing executed -> classify
      }
    };
    if (nsub == 1) {
      // ---- n_sub == 1: table-driven rounds. The per-entry-type parameters come from one
      // conflict-free 128-bit smem load per table instead of select chains; ring slots are
      // addressed by the block counters (slot = count mod R, R a power of two), so there are no
      // head registers; the ZeRO-1 gate max(arrival, t_ag) folds into the initial clock because
      // F_0 is the first block every completing row executes.
      const int Rm = R - 1;
      const bool last = s == p - 1;
      int lmF = s == 0 ? 0xffff : 0;                // stage 0 has no F producer: always available
      int rmF = last ? 0xffff : 0;                  // the last stage has no F consumer: always room
      asm("mov.b32 %0, %0;" : "+r"(lmF));           // opaque: keeps (x & 0xffff) | m one LOP3
      asm("mov.b32 %0, %0;" : "+r"(rmF));
      if (last && s < 31)                           // its D ring may hold a larger item's arrivals
        for (int k = 0; k < R; ++k) smem[iD + (k << 5)] = 0;
      {                                             // every lane: idle lanes get safe entries
        // per lane and entry code: {duration, memory delta, link bandwidth, latency of its message};
        // latency -1 marks an entry that sends nothing (W; F on the last stage; D/B on stage 0)
        tabA[0 * 32] = make_int4(tf, mf, bwF, sendF ? latF : -1);
        tabA[1 * 32] = make_int4(tB, mB, bwB, sendD ? latB : -1);
        tabA[2 * 32] = make_int4(td, md, bwB, sendD ? latB : -1);
        tabA[3 * 32] = make_int4(tw, mw, 0, -1);
        // per entry code, the same for every lane (a broadcast read: one smem wavefront), byte offsets
        // from the lane's own F ring column / F link clock: {input ring, slot mask on counts * 32,
        // send offset (the consumer's column: +1 lane for F, -1 for D/B), link clock (F: to s+1, D/B:
        // to s-1)}; then {increment of the packed (nF | nD << 16) counters, of the W count}
        if (lane < 4) {
          const int c = lane;
          const int ring = c == CP_OP_F ? 0 : (c == CP_OP_W ? 4 * (Ly.zero - Ly.rings) : 4 * RW);
          U[c] = make_int4(ring, c == CP_OP_W ? 0 : Rm << 5, c == CP_OP_F ? 4 : (c == CP_OP_W ? 0 : -4),
                           (c == CP_OP_F || c == CP_OP_W) ? 0 : 128);
          U[4 + c] = make_int4(c == CP_OP_F ? 32 : (c == CP_OP_W ? 0 : 32 << 16), c == CP_OP_W ? 32 : 0, 0, 0);
        }
        smem[wbase + Ly.link + lane] = 0;                  // both link clocks start at 0
        smem[wbase + Ly.link + 32 + lane] = 0;
        // entries past the row's end read as D, which is never ready once the row is done (its D count
        // is m, and no neighbour's D count -- nor, on the last stage, its own F count -- exceeds m), so
        // the round needs no position test; the rest of the staged row and the spare row are
        // overwritten (they are not part of the plan)
        for (int k = plen >> 4; k <= PW; ++k) {
          const int sh = 2 * (plen - 16 * k);
          const uint32_t pad = sh <= 0 ? 0xffffffffu : (0xffffffffu << sh);   // bits of entries >= plen
          smem[iP + (k << 5)] = (int)(((uint32_t)smem[iP + (k << 5)] & ~pad) | (0xaaaaaaaau & pad));
        }
      }
      __syncwarp();
      clk = tag;
      // Counters are kept scaled by 32 (one ring slot = 32 words) and the plan position doubled,
      // so that every address is one LEA off a shared-window base: the entry code comes from one
      // funnel shift of the staged word, the lane's cost row is tabA + code * 512 B, the code's
      // uniform row U + code * 16 B, the ring slot column + ((count & mask) << 2).  (A row holds at
      // most 1024 >= 2m entries, so 32 * m <= 16384 fits the 16-bit halves of the neighbour shuffle.)
      // Shared-memory wavefronts, not instructions, bound this loop (ncu: the LSU data pipe at 95% of
      // peak with per-lane address tables): per round one 4-wavefront cost row, two 1-wavefront
      // broadcast rows, three scalar loads, two predicated stores and the two shuffles.
      const unsigned sb = (unsigned)__cvta_generic_to_shared(smem);
      const unsigned tab0 = sb + 4u * (unsigned)(tbase + 4 * lane);        // tabA[0][lane]
      const unsigned ub = sb + 4u * (unsigned)Ly.uni;                      // U[0] (block header)
      unsigned colF = sb + 4u * (unsigned)iF;                              // own F ring column
      asm volatile("mov.b32 %0, %0;" : "+r"(colF));
      const unsigned lkF = sb + 4u * (unsigned)(wbase + Ly.link + lane);   // own F link clock
      const unsigned iPb = sb + 4u * (unsigned)iP;
      const int R32 = R << 5;
      const unsigned stg = sb + 4u * (unsigned)(wbase + Ly.stage + lane);  // timeline staging [16][32]
      int32_t* const trow = kTL ? A.t_start + (item * 32 + s) * (long long)A.len_stride : nullptr;
      int pos2 = 0, me = 0;                         // me: nF | nD << 16 (both scaled by 32)
      int rr = 0, fg = 0;                           // timeline: round counter, next group to write
      for (;;) {
        const int cu = __shfl_up_sync(FULLM, me, 1);
        const int cd = __shfl_down_sync(FULLM, me, 1);
        nF = me & 0xffff;
        nD = me >> 16;
        const int leftF = (cu & 0xffff) | lmF;
        const int leftD = cu >> 16;
        const int rightF = (cd & 0xffff) | rmF;
        const int rightD = last ? nF : (cd >> 16);
        unsigned code;
        asm("shf.r.wrap.b32 %0, %1, %1, %2;" : "=r"(code) : "r"(wv), "r"(pos2));
        code &= 3u;
        asm("mov.b32 %0, %0;" : "+r"(code));        // materialized once: LEA for the table rows
        const unsigned ta_addr = tab0 + (code << 9), u_addr = ub + (code << 4);
        int4 ta, tu;
        int2 tc;                                    // counter increments (off the critical path)
        asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(ta.x), "=r"(ta.y), "=r"(ta.z), "=r"(ta.w) : "r"(ta_addr));
        asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(tu.x), "=r"(tu.y), "=r"(tu.z), "=r"(tu.w) : "r"(u_addr));
        // one broadcast word (one wavefront) for the packed counter increment; the W count's
        // increment is a select
        asm volatile("ld.shared.b32 %0, [%1+64];" : "=r"(tc.x) : "r"(u_addr));
        const bool isF = code == CP_OP_F, isW = code == CP_OP_W;
        tc.y = isW ? 32 : 0;
        // readiness of the entry's own stream only: the producer count X and consumer count Y of F
        // (left, right) or D (right, left) are selected first, then one test
        const int n = isF ? nF : nD;
        const int X = isF ? leftF : rightD, Y = isF ? rightF : leftD;
        const bool go = isW ? (went < nD) : ((X > n) & (n - Y < R32));
        const unsigned raddr = colF + (unsigned)tu.x + ((unsigned)(n & tu.y) << 2);
        const unsigned laddr = lkF + (unsigned)tu.w;
        int arr, lk;
        asm volatile("ld.shared.b32 %0, [%1];" : "=r"(arr) : "r"(raddr));
        asm volatile("ld.shared.b32 %0, [%1];" : "=r"(lk) : "r"(laddr));     // the link's FIFO clock
        const int start = mx(clk, arr);
        const int end = start + ta.x;
        const int nl = mx(end, lk) + ta.z;                   // FIFO link clock (App. X1)
        if (go && ta.w >= 0) {
          asm volatile("st.shared.b32 [%0], %1;" :: "r"(raddr + tu.z), "r"(nl + ta.w) : "memory");
          asm volatile("st.shared.b32 [%0], %1;" :: "r"(laddr), "r"(nl) : "memory");
        }
        const int gi = go ? 1 : 0;
        if (kTL)   // start tick of entry pos into staging slot pos & 15 (predicated, no branch)
          asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.s32 q, %2, 0;\n\t@q st.shared.b32 [%0], %1;\n\t}"
                       :: "r"(stg + (((unsigned)pos2 & 30u) << 6)), "r"(start), "r"(gi) : "memory");
        clk = madd(gi, end - clk, clk);
        mem = madd(gi, ta.y, mem);
        peak = mx(peak, mem);
        pos2 = madd(gi, 2, pos2);
        me = madd(gi, tc.x, me);                    // the entry's counter(s), from the table
        went = madd(gi, tc.y, went);
        if (kTL && (++rr & 7) == 0) {               // warp-uniform: every 8th round
          // a lane advances <= 8 entries in 8 rounds, so at most one aligned group of 8 has completed
          // since the last flush, and the 16-slot staging ring still holds it: two 16-B stores, one
          // full 32-B sector of the lane's timeline row
          if ((pos2 >> 4) > fg) {
            tl_flush8(stg + ((unsigned)(fg & 1) << 10), trow + 8 * fg);
            ++fg;
          }
        }
        unsigned wa;                                // iPb + 4 * (pos2 & ~31): one LOP3 + one IMAD
        asm("mad.lo.u32 %0, %1, 4, %2;" : "=r"(wa) : "r"((unsigned)pos2 & ~31u), "r"(iPb));
        asm volatile("ld.shared.b32 %0, [%1];" : "=r"(wv) : "r"(wa));
        __syncwarp();                               // ring stores visible to the neighbours' next reads
        if (!__any_sync(FULLM, go)) break;
      }
      nF = (me & 0xffff) >> 5; nD = (me >> 16) >> 5; went >>= 5; pos = pos2 >> 1;
      if (kTL)                                      // entries not yet written (< 16)
        for (int k = 8 * fg; k < pos; ++k) trow[k] = smem[wbase + Ly.stage + ((k & 15) << 5) + lane];
    } else {
      rounds(std::false_type{});
    }

    // ------------------------------------------------------------------ no progress: classify
    {
      // a stall with a full consumer ring may be an artefact of the small ring (cyclic backpressure):
      // such items are re-run exactly by the global-ring fix-up pass
      const int cu = __shfl_up_sync(FULLM, nF | (nD << 16), 1);
      const int cd = __shfl_down_sync(FULLM, nF | (nD << 16), 1);
      const bool ring_full = (sendF && nF - (cd & 0xffff) >= R) || (sendD && nD - (cu >> 16) >= R);
      const bool unfin = pos < plen;
      const bool complete = !__any_sync(FULLM, unfin);
      bool badc = false;
      if (!complete && s < p) {
        // cannot continue: a W entry ahead of its D (prefix rule) reports BAD_PLAN -> scan the rest
        int cD = nD, cW = went;
        for (int k = pos; k < plen && !badc; ++k) {
          const uint32_t c2 = ((uint32_t)smem[iP + ((k >> 4) << 5)] >> ((k & 15) << 1)) & 3u;
          if (c2 == CP_OP_W) { badc = cW >= nsub * cD; ++cW; }
          else if (c2 != CP_OP_F) ++cD;
        }
      }
      int st;
      if (__any_sync(FULLM, badc)) st = CPI_BAD_PLAN;
      else if (!complete && !A.from_list && __any_sync(FULLM, ring_full)) st = -1;
      else if (!complete) st = CPI_DEADLOCK;
      else st = __any_sync(FULLM, s < p && peak > mlim) ? CPI_MEM_EXCEEDED : 0;
      if (st == -1) {                            // ring capacity reached: hand to the fix-up pass
        if (lane == 0) { const int slot = atomicAdd(A.ovf_count, 1); A.ovf_list[slot] = (int32_t)item; }
      } else {
        int ms = s < p ? mx(clk + tdp, tag) : 0, pk = s < p ? peak : 0;
        for (int d = 16; d > 0; d >>= 1) {
          ms = mx(ms, __shfl_xor_sync(FULLM, ms, d));
          pk = mx(pk, __shfl_xor_sync(FULLM, pk, d));
        }
        const bool done = complete && !(st & CPI_BAD_PLAN);
        if (lane == 0) {
          A.makespan[item] = done ? (long long)ms : -1LL;
          if (A.peak_mem) A.peak_mem[item] = done ? pk : -1;
          A.status[item] = st;
          if (A.best_key && st == 0)
            atomicMin(A.best_key, ((unsigned long long)ms << 32) | (unsigned long long)(uint32_t)(item + A.index_base));
        }
        if (A.stage_stats) {
          // a completed valid row executed every block exactly once: busy = m (t_f + t_d + t_w);
          // every row starts with F_0, whose message opens its link, so first_start is the max-plus
          // prefix first[s] = max(t_ag[s], first[s-1] + t_f + bw_f + lat_f of s-1) = P_s + max_{k<=s}(ag_k - P_k)
          const int busy = m * (tf + td + tw);
          const int cfw = s < p ? tf + bwF + latF : 0;
          int P = cfw;                              // inclusive prefix sum of hop costs
          for (int d = 1; d < 32; d <<= 1) { const int t = __shfl_up_sync(FULLM, P, d); if (s >= d) P += t; }
          P -= cfw;                                 // exclusive: P_s
          int x = (s < p ? tag : 0) - P;
          for (int d = 1; d < 32; d <<= 1) { const int t = __shfl_up_sync(FULLM, x, d); if (s >= d) x = mx(x, t); }
          const int first = P + x;
          const int4 v = (done && s < p) ? make_int4(first, clk, busy, peak) : make_int4(0, 0, 0, 0);
          *reinterpret_cast<int4*>(A.stage_stats + (item * 32 + s) * 4) = v;
        }
      }
    }
    __syncwarp();
  }
}

int launch_sim32(bool timeline, const Args& a, int blocks, int threads, size_t smem, void* stream) {
  const void* fn = timeline ? (const void*)k_sim32<true> : (const void*)k_sim32<false>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return (int)e;
  }
  void* params[] = {(void*)&a};
  return (int)cudaLaunchKernel(fn, dim3(blocks), dim3(threads), params, smem, (cudaStream_t)stream);
}

int sim32_blocks_per_sm(bool timeline, int threads, size_t smem) {
  const void* fn = timeline ? (const void*)k_sim32<true> : (const void*)k_sim32<false>;
  if (smem > 48 * 1024) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, threads, smem) != cudaSuccess) return 1;
  return n > 0 ? n : 1;
}

}  // namespace cpk
