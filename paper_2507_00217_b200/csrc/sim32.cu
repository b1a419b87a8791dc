// sim32.cu -- fast path of cp_simulate for the dominant shape: one item per warp (17..32
// stages, stage_stride 32), plan rows staged in shared memory by double-buffered TMA bulk
// copies, arrival rings in shared memory, no per-entry timeline.
//
// Same semantics as k_engine<MODE_SIM> (engine.cu), which remains the reference GPU path for
// every other shape and for the fix-up pass; both are parity-tested.
// What makes this kernel fast is what it leaves out: the warp is one segment, so the "no block
// executed this round" test is a single ballot with a warp-uniform branch; the state is the
// minimum the §3.5 recurrence needs; the plan buffers carry one spare row so finished lanes
// read without clamping.
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
}  // namespace

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
  // per-warp smem (words): [paramA 4*32 int4][paramB 4*32 int4][ringF R*32][ringD R*32]
  //                        [plan 2*(PW+1)*32][sink 32][zero 32][2 mbarriers][link clocks 2*32]
  //                        [counter increments 4*32 int2]
  const int wbase = wib * A.smem_words_per_warp;
  const int rbase = wbase + kSim32TableWords;
  const int pbase0 = rbase + 2 * RW;
  const int dum_row = kSim32TableWords + 2 * RW + 2 * PWr * 32;   // relative to wbase
  const int zero_row = dum_row + 32;
  uint32_t* const plan = reinterpret_cast<uint32_t*>(smem + pbase0);
  uint64_t* const bars = reinterpret_cast<uint64_t*>(smem + wbase + zero_row + 32);
  int4* const tabA = reinterpret_cast<int4*>(smem + wbase) + lane;          // [code][lane]
  int4* const tabB = reinterpret_cast<int4*>(smem + wbase + 512) + lane;
  const uint32_t plan_bytes = (uint32_t)A.words * 32u * 4u;

  long long item = gwarp;
  // the rings never written by a producer (stage 0's F ring) and the zero row read by W entries
  // must hold 0: clear both ring blocks and the zero row once
  for (int k = lane; k < 2 * RW; k += 32) smem[rbase + k] = 0;
  smem[wbase + zero_row + lane] = 0;
  if (lane == 0) { mbar_init(&bars[0]); mbar_init(&bars[1]); }
  __syncwarp();
  if (lane == 0 && item < A.n_items) tma_load_1d(plan, A.ops + item * A.words * 32, plan_bytes, &bars[0]);
  uint32_t phase = 0;
  int buf = 0;

  for (; item < A.n_items; item += nwarps) {
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
    if (lane == 0 && item + nwarps < A.n_items)
      tma_load_1d(plan + (buf ^ 1) * PWr * 32, A.ops + (item + nwarps) * A.words * 32, plan_bytes, &bars[buf ^ 1]);
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
        cF += __popc(~lo & ~hi & valid);
        cB += __popc(lo & ~hi & valid);
        cD += __popc(~lo & hi & valid);
        cW += __popc(lo & hi & valid);
      }
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
        tabA[0 * 32] = make_int4(tf, mf, bwF, latF);
        tabA[1 * 32] = make_int4(tB, mB, bwB, latB);
        tabA[2 * 32] = make_int4(td, md, bwB, latB);
        tabA[3 * 32] = make_int4(tw, mw, 0, 0);
        // shared-window byte addresses: {input ring column, slot mask on counts * 32, send offset,
        // the FIFO clock of the link the entry's message takes (F: to s+1, D/B: to s-1)}
        const unsigned sb = (unsigned)__cvta_generic_to_shared(smem);
        const int lkF = (int)(sb + 4u * (wbase + zero_row + 36 + lane)), lkB = lkF + 128;
        tabB[0 * 32] = make_int4((int)(sb + 4u * iF), Rm << 5, sendF ? 4 : 0, lkF);
        tabB[1 * 32] = make_int4((int)(sb + 4u * iD), Rm << 5, sendD ? -4 : 0, lkB);
        tabB[2 * 32] = make_int4((int)(sb + 4u * iD), Rm << 5, sendD ? -4 : 0, lkB);
        tabB[3 * 32] = make_int4((int)(sb + 4u * (wbase + zero_row + lane)), 0, 0, lkF);
        smem[wbase + zero_row + 36 + lane] = 0;            // both link clocks start at 0
        smem[wbase + zero_row + 68 + lane] = 0;
        // per code: the increments of the packed (nF | nD << 16) counters and of the W count
        int2* const tabC = reinterpret_cast<int2*>(smem + wbase + zero_row + 100) + lane;
        tabC[0 * 32] = make_int2(32, 0);
        tabC[1 * 32] = make_int2(32 << 16, 0);
        tabC[2 * 32] = make_int2(32 << 16, 0);
        tabC[3 * 32] = make_int2(0, 32);
      }
      __syncwarp();
      clk = tag;
      // Counters are kept scaled by 32 (one ring slot = 32 words) and the plan position doubled,
      // so that every address is one LEA off a shared-window base: the entry code comes from one
      // funnel shift of the staged word, the table row is tab + code * 512 B, the ring slot is
      // column + ((count & mask) << 2).  (A row holds at most 1024 >= 2m entries, so 32 * m <= 16384
      // fits the 16-bit halves of the neighbour shuffle.)
      const unsigned sb = (unsigned)__cvta_generic_to_shared(smem);
      const unsigned tab0 = sb + 4u * (unsigned)(wbase + 4 * lane);        // tabA[0][lane]; tabB at +2048 B
      const unsigned iPb = sb + 4u * (unsigned)iP;
      const int R32 = R << 5, plen2 = 2 * plen;
      const unsigned tc0 = sb + 4u * (unsigned)(wbase + zero_row + 100 + 2 * lane);   // tabC[0][lane]
      int pos2 = 0, me = 0;                         // me: nF | nD << 16 (both scaled by 32)
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
        asm("mov.b32 %0, %0;" : "+r"(code));        // materialized once: LEA for the table row
        const unsigned ta_addr = tab0 + (code << 9);
        int2 tc;                                    // counter increments (off the critical path)
        asm volatile("ld.shared.v2.s32 {%0, %1}, [%2];" : "=r"(tc.x), "=r"(tc.y) : "r"(tc0 + (code << 8)));
        int4 ta, tb;
        asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(ta.x), "=r"(ta.y), "=r"(ta.z), "=r"(ta.w) : "r"(ta_addr));
        asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4+2048];"
                     : "=r"(tb.x), "=r"(tb.y), "=r"(tb.z), "=r"(tb.w) : "r"(ta_addr));
        const bool isF = code == CP_OP_F, isW = code == CP_OP_W;
        const bool isDB = !isF & !isW;
        // readiness of the entry's own stream only: the producer count X and consumer count Y of F
        // (left, right) or D (right, left) are selected first, then one test
        const int n = isF ? nF : nD;
        const int X = isF ? leftF : rightD, Y = isF ? rightF : leftD;
        const bool go = (pos2 < plen2) & (isW ? (went < nD) : ((X > n) & (n - Y < R32)));
        const unsigned raddr = (unsigned)tb.x + ((unsigned)(n & tb.y) << 2);
        int arr, lk;
        asm volatile("ld.shared.b32 %0, [%1];" : "=r"(arr) : "r"(raddr));
        asm volatile("ld.shared.b32 %0, [%1];" : "=r"(lk) : "r"(tb.w));     // the link's FIFO clock
        const int start = mx(clk, arr);
        const int end = start + ta.x;
        const int nl = mx(end, lk) + ta.z;                   // FIFO link clock (App. X1)
        if (go && tb.z != 0) {
          asm volatile("st.shared.b32 [%0], %1;" :: "r"(raddr + tb.z), "r"(nl + ta.w) : "memory");
          asm volatile("st.shared.b32 [%0], %1;" :: "r"(tb.w), "r"(nl) : "memory");
        }
        const int gi = go ? 1 : 0;
        clk = madd(gi, end - clk, clk);
        mem = madd(gi, ta.y, mem);
        peak = mx(peak, mem);
        pos2 = madd(gi, 2, pos2);
        me = madd(gi, tc.x, me);                    // the entry's counter(s), from the table
        went = madd(gi, tc.y, went);
        unsigned wa;                                // iPb + 4 * (pos2 & ~31): one LOP3 + one IMAD
        asm("mad.lo.u32 %0, %1, 4, %2;" : "=r"(wa) : "r"((unsigned)pos2 & ~31u), "r"(iPb));
        asm volatile("ld.shared.b32 %0, [%1];" : "=r"(wv) : "r"(wa));
        __syncwarp();                               // ring stores visible to the neighbours' next reads
        if (!__any_sync(FULLM, go)) break;
      }
      nF = (me & 0xffff) >> 5; nD = (me >> 16) >> 5; went >>= 5; pos = pos2 >> 1;
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
      else if (!complete && __any_sync(FULLM, ring_full)) st = -1;
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

int launch_sim32(const Args& a, int blocks, int threads, size_t smem, void* stream) {
  const void* fn = (const void*)k_sim32;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return (int)e;
  }
  void* params[] = {(void*)&a};
  return (int)cudaLaunchKernel(fn, dim3(blocks), dim3(threads), params, smem, (cudaStream_t)stream);
}

int sim32_blocks_per_sm(int threads, size_t smem) {
  const void* fn = (const void*)k_sim32;
  if (smem > 48 * 1024) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, threads, smem) != cudaSuccess) return 1;
  return n > 0 ? n : 1;
}

}  // namespace cpk
