// wave32.cu -- cp_simulate for Wave-pattern plans (reading Q32, §8(f) NEXT 1): every stage holds
// two model chunks in a V.  One item per warp, lane = stage (p <= 32), round-synchronous like
// k_sim32: each round every lane runs its next plan entry if that entry's input has arrived, and
// one vote ends the item when no lane progressed.
//
// Per microbatch: F0 runs s -> s+1, turns to F1 on the last stage, F1 runs s -> s-1; the loss on
// stage 0 starts D1, D1 runs s -> s+1, turns to D0 on the last stage, D0 runs s -> s-1; W(c)
// follows D(c).  Lane s therefore hears four streams: F0 and D1 from the left, F1 and D0 from the
// right, each in microbatch order, through four shared-memory rings addressed by the consumer's
// count (slot = count mod R).  It sends F0 / D1 right through one FIFO link clock and F1 / D0 left
// through another: one producer per directed link (App. X1 holds for Wave).
//
// Rings: a block waits while its consumer's ring holds R unconsumed entries (occupancy
// backpressure).  An item stalled that way is re-run by a second pass with R >= n_mb slots.
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "engine.h"

namespace cpk {

namespace {
constexpr int32_t WINF = 1 << 30;
constexpr unsigned WFULL = 0xffffffffu;
__device__ __forceinline__ int wmx(int a, int b) { return a > b ? a : b; }
__device__ __forceinline__ int wmadd(int g, int d, int x) {   // x + g*d on the FMA pipe
  int r;
  asm("mad.lo.s32 %0, %1, %2, %3;" : "=r"(r) : "r"(g), "r"(d), "r"(x));
  return r;
}
}  // namespace

template <bool kLoop, bool kTL>   // kTL: per-entry start ticks requested (A.t_start)
__global__ void __launch_bounds__(kFastThreads, kFastMinBlocks) k_chunk32(const __grid_constant__ Args A) {
  extern __shared__ __align__(16) int32_t smem[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int R = A.ring_slots, Rm = R - 1, RW = R * 32;
  const int PW = A.plan_words;                         // staged words per row (>= A.words)
  const long long gwarp = (long long)blockIdx.x * (blockDim.x >> 5) + wib;
  const long long nwarps = (long long)gridDim.x * (blockDim.x >> 5);
  // per-warp smem (words): [tabA 8*32 int4][tabB 8*32 int4][rF0][rD1][rF1][rD0] (R*32 each)
  //                        [zero row 32][plan PW*32]
  const int wbase = wib * A.smem_words_per_warp;
  int4* const tabA = reinterpret_cast<int4*>(smem + wbase) + lane;          // [entry][lane]
  int4* const tabB = reinterpret_cast<int4*>(smem + wbase + 1024) + lane;
  const int rb0 = wbase + 2048;
  const int iF0 = rb0 + lane, iD1 = iF0 + RW, iF1 = iD1 + RW, iD0 = iF1 + RW;
  const int iZ = iD0 + RW;                             // zero row: inputs of W and of missing producers
  const int iP = iZ + 32;
  if (A.from_list && gwarp >= *(volatile int32_t*)A.ovf_count) return;   // beyond the overflow list
  for (int k = lane; k < 4 * RW + 32; k += 32) smem[rb0 + k] = 0;
  __syncwarp();

  for (long long t = gwarp; ; t += nwarps) {
    long long item;
    if (A.from_list) item = t < *(volatile int32_t*)A.ovf_count ? (long long)A.ovf_list[t] : -1;
    else item = t < A.n_items ? t : -1;
    if (item < 0) break;
    const long long ii = A.inst_of ? (long long)A.inst_of[item] : (A.n_inst == 1 ? 0 : item);
    const cp_inst_v1* I = A.inst + ii;
    const int p = I->n_pp, m = I->n_mb, ns = I->n_sub;
    const int s = lane;
    int tf = 0, td = 0, tw = 0, mf = 0, md = 0, mw = 0, mlim = 0, tdp = 0, tag = 0;
    int latR = 0, bwR = 0, latL = 0, bwL = 0, lat_b_s = 0, bw_b_s = 0, plen = 0;
    if (s < p && p <= CP_MAX_STAGES) {
      tf = I->t_f[s]; td = I->t_d[s]; tw = I->t_w[s];
      mf = I->m_f[s]; md = I->m_d[s]; mw = I->m_w[s]; mlim = I->m_lim[s];
      tdp = I->t_dp[s]; tag = (I->flags & 1) ? I->t_ag[s] : 0;
      // boundary s = link s -> s+1; Loop also uses index p-1, the wrap links p-1 -> 0 / 0 -> p-1 (Q33)
      if (s < p - 1 || kLoop) { latR = I->lat_f[s]; bwR = I->bw_f[s]; lat_b_s = I->lat_b[s]; bw_b_s = I->bw_b[s]; }
      if (s > 0) { latL = I->lat_b[s - 1]; bwL = I->bw_b[s - 1]; }
      else if (kLoop) { latL = I->lat_b[p - 1]; bwL = I->bw_b[p - 1]; }
      if (s < A.stage_stride) plen = A.len[item * A.stage_stride + s];
    }
    bool bad = p < 1 || p > CP_MAX_STAGES || p > A.stage_stride || m < 1 || ns < 1;
    if (!bad && s < p)
      bad = !(tf >= ns && td >= ns && tw >= ns && mf > 0 && md <= 0 && mw <= 0 && (long long)mf + md + mw == 0 &&
              mlim >= mf && tdp >= 0 && (I->t_ag[s] >= 0) && latR >= 0 && bwR >= 0 && lat_b_s >= 0 && bw_b_s >= 0);
    // int32 horizon guard (Q21, doubled for two chunks)
    long long u = (s < p && !bad) ? 2LL * m * ((long long)tf + td + tw) + tag + tdp +
                                        2LL * m * ((long long)latR + bwR + latL + bwL)
                                  : 0;
    for (int d = 16; d > 0; d >>= 1) u += __shfl_xor_sync(WFULL, u, d);
    int st = 0;
    if (__any_sync(WFULL, bad)) st = CPI_BAD_INSTANCE;
    else if (__any_sync(WFULL, plen > 8 * A.words)) st = CPI_BAD_PLAN;
    else if (m > CP_MAX_MB || ns > CP_MAX_SUB || u >= (long long)WINF) st = CPI_OVERFLOW;
    // stage this lane's row and check Q29's count and mixing rules per chunk, and codes < 8, with
    // nibble popcounts over the words; the W-prefix rule stays dynamic (a W ahead of its D stalls
    // and the non-completion path classifies the item)
    bool bplan = false;
    if (!st && s < p) {
      int cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0};          // per entry value type | chunk << 2
      for (int k = 0; k * 8 < plen; ++k) {
        const uint32_t w = A.ops[(item * A.words + k) * A.stage_stride + s];
        smem[iP + (k << 5)] = (int32_t)w;
        const int n = plen - 8 * k < 8 ? plen - 8 * k : 8;
        const uint32_t vm = (n == 8 ? 0xffffffffu : ((1u << (4 * n)) - 1u)) & 0x11111111u;
        if ((w >> 3) & vm) bplan = true;
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          const uint32_t t = w ^ (0x11111111u * (uint32_t)v);
          cnt[v] += __popc(~(t | (t >> 1) | (t >> 2) | (t >> 3)) & vm);
        }
      }
      for (int ch = 0; ch < 2; ++ch) {
        const int cF = cnt[4 * ch + CP_OP_F], cB = cnt[4 * ch + CP_OP_B], cD = cnt[4 * ch + CP_OP_D];
        const int cW = cnt[4 * ch + CP_OP_W];
        if (cF != m || cB + cD != m || cW != ns * cD) bplan = true;
      }
      if (cnt[CP_OP_B] + cnt[4 + CP_OP_B] > 0 &&
          cnt[CP_OP_D] + cnt[4 + CP_OP_D] + cnt[CP_OP_W] + cnt[4 + CP_OP_W] > 0)
        bplan = true;
    }
    if (!st && __any_sync(WFULL, bplan)) st = CPI_BAD_PLAN;
    if (st) {
      if (lane == 0) {
        A.makespan[item] = -1;
        if (A.peak_mem) A.peak_mem[item] = -1;
        A.status[item] = st;
      }
      if (A.stage_stats)
        for (int r = s; r < A.stage_stride; r += 32)
          *reinterpret_cast<int4*>(A.stage_stats + (item * A.stage_stride + r) * 4) = make_int4(0, 0, 0, 0);
      __syncwarp();
      continue;
    }
    const int wq = tw / ns, wr = tw % ns;
    const bool first_s = s == 0, last = s == p - 1;
    // streams F0, F1, D0, D1 (counts cF = nF0 | nF1 << 16, cD = nD0 | nD1 << 16).  Per stream: whether
    // it has a producer in another lane (else the zero row: stage 0's F0 and the own turn-arounds /
    // loss, all already behind the lane's clock), the consumer column of its messages (0: none), and
    // which link clock carries them (1: lkR, the right / forward link).
    //   Wave (Q32): F0, D1 go right, F1, D0 go left.
    //   Loop (Q33): F0, F1 go forward (right, the last stage's F0 over the wrap into stage 0's F1),
    //               D1, D0 go backward (left, stage 0's D1 over the wrap into the last stage's D0).
    const int inF0 = s > 0, inF1 = kLoop ? 1 : !last, inD1 = kLoop ? !last : s > 0, inD0 = kLoop ? 1 : !last;
    int oF0, oF1, oD0, oD1;
    if (kLoop) {
      oF0 = last ? iF1 - s : iF0 + 1;
      oF1 = last ? 0 : iF1 + 1;
      oD1 = first_s ? iD0 + (p - 1) : iD1 - 1;
      oD0 = first_s ? 0 : iD0 - 1;
    } else {
      oF0 = last ? 0 : iF0 + 1;
      oF1 = first_s ? 0 : iF1 - 1;
      oD1 = last ? 0 : iD1 + 1;
      oD0 = first_s ? 0 : iD0 - 1;
    }
    if (s >= p) oF0 = oF1 = oD0 = oD1 = 0;
    const unsigned sb = (unsigned)__cvta_generic_to_shared(smem);
    // parameter tables, entry x = type | chunk << 2:
    //   tabA[x] = {duration, memory delta, link bw, latency} (W: first sub-block / whole W if n_sub 1)
    //   tabB[x] = {input ring column (zero row without a producer), slot mask, consumer column (0: no
    //             message), the byte address of the message's link clock}
    {
      const int tW = ns == 1 ? tw : wq, mW = ns == 1 ? mw : 0;
      const int dF1 = kLoop ? 1 : 0, dD1 = kLoop ? 0 : 1;       // clock of F1 / D1 (F0: lkR, D0: lkL)
      tabA[0 * 32] = make_int4(tf, mf, bwR, latR);
      tabA[1 * 32] = make_int4(td + tw, md + mw, bwL, latL);
      tabA[2 * 32] = make_int4(td, md, bwL, latL);
      tabA[3 * 32] = make_int4(tW, mW, 0, 0);
      tabA[4 * 32] = make_int4(tf, mf, dF1 ? bwR : bwL, dF1 ? latR : latL);
      tabA[5 * 32] = make_int4(td + tw, md + mw, dD1 ? bwR : bwL, dD1 ? latR : latL);
      tabA[6 * 32] = make_int4(td, md, dD1 ? bwR : bwL, dD1 ? latR : latL);
      tabA[7 * 32] = make_int4(tW, mW, 0, 0);
      // columns as shared-window byte addresses (0: no consumer), masks on counts scaled by 32
      const auto B = [&](int col) { return col ? (int)(sb + 4u * (unsigned)col) : 0; };
      const int Rm32 = Rm << 5;
      // .w: byte address of the FIFO clock of the link the message takes (right / forward, left /
      // backward), two per-lane slots after the plan rows
      const int lkR = B(iP + A.plan_words * 32), lkL = lkR + 128;
      smem[iP + A.plan_words * 32] = 0;                // both link clocks start at 0
      smem[iP + A.plan_words * 32 + 32] = 0;
      // per entry x: the increments of the packed F counts (nF0 | nF1 << 16) and D counts
      int2* const tabC = reinterpret_cast<int2*>(smem + iP - lane + A.plan_words * 32 + 64) + lane;
      for (int e = 0; e < 8; ++e) {
        const int t = e & 3, inc = (e >> 2) ? (32 << 16) : 32;
        tabC[e * 32] = make_int2(t == (int)CP_OP_F ? inc : 0, (t == (int)CP_OP_B || t == (int)CP_OP_D) ? inc : 0);
      }
      tabB[0 * 32] = make_int4(B(inF0 ? iF0 : iZ), inF0 ? Rm32 : 0, B(oF0), lkR);
      tabB[1 * 32] = make_int4(B(inD0 ? iD0 : iZ), inD0 ? Rm32 : 0, B(oD0), lkL);
      tabB[2 * 32] = tabB[1 * 32];
      tabB[3 * 32] = make_int4(B(iZ), 0, 0, lkR);
      tabB[4 * 32] = make_int4(B(inF1 ? iF1 : iZ), inF1 ? Rm32 : 0, B(oF1), dF1 ? lkR : lkL);
      tabB[5 * 32] = make_int4(B(inD1 ? iD1 : iZ), inD1 ? Rm32 : 0, B(oD1), dD1 ? lkR : lkL);
      tabB[6 * 32] = tabB[5 * 32];
      tabB[7 * 32] = tabB[3 * 32];
    }
    int clk = tag, mem = 0, peak = 0, pos = 0;
    int cF = 0, cD = 0, wP = 0;                        // wP: W sub-blocks of chunk 0 | chunk 1 << 16
    int lm = first_s ? 0xffff : 0, rm = last ? 0xffff : 0;      // no producer / no consumer
    asm("mov.b32 %0, %0;" : "+r"(lm));
    asm("mov.b32 %0, %0;" : "+r"(rm));
    const int wsrc = first_s ? p - 1 : 0;              // Loop: the wrap partner lane
    // producer count X and consumer count Y of every stream, from the neighbours' packed counts
    struct XY { int xF0, yF0, xF1, yF1, xD0, yD0, xD1, yD1; };
    auto neighbours = [&]() -> XY {
      const int lF = __shfl_up_sync(WFULL, cF, 1), lD = __shfl_up_sync(WFULL, cD, 1);
      const int rF = __shfl_down_sync(WFULL, cF, 1), rD = __shfl_down_sync(WFULL, cD, 1);
      const int nF0 = cF & 0xffff, nF1 = cF >> 16, nD1 = cD >> 16;
      XY q;
      if (kLoop) {
        const int wF = __shfl_sync(WFULL, cF, wsrc), wD = __shfl_sync(WFULL, cD, wsrc);
        q.xF0 = (lF & 0xffff) | lm;               q.yF0 = last ? (wF >> 16) : (rF & 0xffff);
        q.xF1 = first_s ? (wF & 0xffff) : (lF >> 16); q.yF1 = (rF >> 16) | rm;
        q.xD1 = last ? nF1 : (rD >> 16);          q.yD1 = first_s ? (wD & 0xffff) : (lD >> 16);
        q.xD0 = last ? (wD >> 16) : (rD & 0xffff); q.yD0 = (lD & 0xffff) | lm;
      } else {
        q.xF0 = (lF & 0xffff) | lm;               q.yF0 = (rF & 0xffff) | rm;
        q.xF1 = last ? nF0 : (rF >> 16);          q.yF1 = (lF >> 16) | lm;
        q.xD1 = first_s ? nF1 : (lD >> 16);       q.yD1 = (rD >> 16) | rm;
        q.xD0 = last ? nD1 : (rD & 0xffff);       q.yD0 = (lD & 0xffff) | lm;
      }
      return q;
    };
    __syncwarp();
    auto rounds = [&](auto n1) {
      constexpr bool kN1 = decltype(n1)::value;       // n_sub == 1: a W entry is a whole W block
      // counts (and wP) are kept scaled by 32, one ring slot, and the plan position by 4 (one entry
      // nibble): the entry code is one funnel shift, the table row tab + x * 512 B and the ring slot
      // column + ((count & mask) << 2) are single LEAs off shared-window byte addresses
      const unsigned tab0 = sb + 4u * (unsigned)(wbase + 4 * lane), iPb = sb + 4u * (unsigned)iP;
      const unsigned tc0 = iPb + 4u * (unsigned)(A.plan_words * 32 + 64 + lane);   // tabC[0][lane]
      const int R32 = R << 5, Rm32 = Rm << 5, plen4 = 4 * plen;
      int pos4 = 0;
      for (;;) {
        const XY q = neighbours();
        const int nF0 = cF & 0xffff, nF1 = cF >> 16, nD0 = cD & 0xffff, nD1 = cD >> 16;
        unsigned wa, wv, x;
        asm("mad.lo.u32 %0, %1, 4, %2;" : "=r"(wa) : "r"((unsigned)pos4 & ~31u), "r"(iPb));
        asm volatile("ld.shared.b32 %0, [%1];" : "=r"(wv) : "r"(wa));
        asm("shf.r.wrap.b32 %0, %1, %1, %2;" : "=r"(x) : "r"(wv), "r"(pos4));
        x &= 7u;
        asm("mov.b32 %0, %0;" : "+r"(x));
        const unsigned ta_addr = tab0 + (x << 9);
        int2 tc;                                        // counter increments (off the critical path)
        asm volatile("ld.shared.v2.s32 {%0, %1}, [%2];" : "=r"(tc.x), "=r"(tc.y) : "r"(tc0 + (x << 8)));
        int4 ta, tb;
        asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(ta.x), "=r"(ta.y), "=r"(ta.z), "=r"(ta.w) : "r"(ta_addr));
        asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4+4096];"
                     : "=r"(tb.x), "=r"(tb.y), "=r"(tb.z), "=r"(tb.w) : "r"(ta_addr));
        const int ch = (int)(x >> 2);
        const bool isF = (x & 3u) == CP_OP_F, isW = (x & 3u) == CP_OP_W;
        // the entry's own count of its stream addresses both its input slot and its message slot
        const int cnt = ((isF ? cF : cD) >> (ch ? 16 : 0)) & 0xffff;
        // readiness of the entry's stream only: input produced (or the own turn-around / loss) and
        // room in the consumer's ring, from that stream's producer count X and consumer count Y
        const int X = isF ? (ch ? q.xF1 : q.xF0) : (ch ? q.xD1 : q.xD0);
        const int Y = isF ? (ch ? q.yF1 : q.yF0) : (ch ? q.yD1 : q.yD0);
        const int wc = ch ? (wP >> 16) : (wP & 0xffff), ndc = ch ? nD1 : nD0;
        const bool rW = kN1 ? wc < ndc : wc < ns * ndc;
        const bool rdy = isW ? rW : ((X > cnt) & (cnt - Y < R32));
        const bool go = (pos4 < plen4) & rdy;
        int arr, lk;
        asm volatile("ld.shared.b32 %0, [%1];" : "=r"(arr) : "r"((unsigned)tb.x + ((unsigned)(cnt & tb.y) << 2)));
        asm volatile("ld.shared.b32 %0, [%1];" : "=r"(lk) : "r"(tb.w));     // the message's link clock
        const int start = wmx(clk, arr);
        int dur = ta.x, dm = ta.y;
        if (!kN1) {                                     // W sub-block k of its W block (Q12)
          const int k = (wc >> 5) % ns;
          dur = isW ? wq + (k < wr ? 1 : 0) : dur;
          dm = isW ? (k == ns - 1 ? mw : 0) : dm;
        }
        const int end = start + dur;
        const int nl = wmx(end, lk) + ta.z;             // FIFO link clock (App. X1)
        // a link clock advances only with a message on it (Loop: stage 0's D0 and the last stage's F1
        // send nothing, while the same clocks carry their wrap-around D1 / F0 messages)
        if (go & (tb.z != 0)) {                         // (tb.z: consumer column, 0 = none)
          asm volatile("st.shared.b32 [%0], %1;" :: "r"((unsigned)tb.z + ((unsigned)(cnt & Rm32) << 2)), "r"(nl + ta.w)
                       : "memory");
          asm volatile("st.shared.b32 [%0], %1;" :: "r"(tb.w), "r"(nl) : "memory");
        }
        if (kTL && go && (pos4 >> 2) < A.len_stride)
          A.t_start[(item * A.stage_stride + s) * (long long)A.len_stride + (pos4 >> 2)] = start;
        const int gi = go ? 1 : 0;
        clk = wmadd(gi, end - clk, clk);
        mem = wmadd(gi, dm, mem);
        peak = wmx(peak, mem);
        cF = wmadd(gi, tc.x, cF);
        cD = wmadd(gi, tc.y, cD);
        wP = wmadd((go & isW) ? 1 : 0, ch ? (32 << 16) : 32, wP);
        pos4 = wmadd(gi, 4, pos4);
        __syncwarp();
        if (!__any_sync(WFULL, go)) break;
      }
      const auto unscale = [](int c) { return ((c & 0xffff) >> 5) | ((c >> 21) << 16); };
      cF = unscale(cF); cD = unscale(cD); wP = unscale(wP); pos = pos4 >> 2;
    };
    if (ns == 1) rounds(std::true_type{});
    else rounds(std::false_type{});
    const int nF0 = cF & 0xffff, nF1 = cF >> 16, nD0 = cD & 0xffff, nD1 = cD >> 16;
    // no lane progressed: complete, a cyclic wait on full rings (-> second pass), or deadlock
    const XY q = neighbours();
    const bool ring_full = (oF0 && nF0 - q.yF0 >= R) || (oF1 && nF1 - q.yF1 >= R) ||
                           (oD1 && nD1 - q.yD1 >= R) || (oD0 && nD0 - q.yD0 >= R);
    const bool complete = !__any_sync(WFULL, s < p && pos < plen);
    // cannot continue: a W ahead of its D (prefix rule) reports BAD_PLAN -> scan the rest of the row
    bool badc = false;
    if (!complete && s < p) {
      int cw[2] = {wP & 0xffff, wP >> 16}, cdd[2] = {nD0, nD1};
      for (int k = pos; k < plen && !badc; ++k) {
        const uint32_t x2 = ((uint32_t)smem[iP + ((k >> 3) << 5)] >> ((k & 7) << 2)) & 15u;
        const int t2 = x2 & 3, c2 = (x2 >> 2) & 1;
        if (t2 == CP_OP_W) { badc = cw[c2] >= ns * cdd[c2]; ++cw[c2]; }
        else if (t2 != CP_OP_F) ++cdd[c2];
      }
    }
    int st2;
    if (__any_sync(WFULL, badc)) st2 = CPI_BAD_PLAN;
    else if (!complete && __any_sync(WFULL, ring_full) && !A.from_list) st2 = -1;
    else if (!complete) st2 = CPI_DEADLOCK;
    else st2 = __any_sync(WFULL, s < p && peak > mlim) ? CPI_MEM_EXCEEDED : 0;
    if (st2 == -1) {
      if (lane == 0) { const int slot = atomicAdd(A.ovf_count, 1); A.ovf_list[slot] = (int32_t)item; }
    } else {
      int ms = s < p ? wmx(clk + tdp, tag) : 0, pk = s < p ? peak : 0;
      for (int d = 16; d > 0; d >>= 1) {
        ms = wmx(ms, __shfl_xor_sync(WFULL, ms, d));
        pk = wmx(pk, __shfl_xor_sync(WFULL, pk, d));
      }
      if (lane == 0) {
        const bool ok = complete && st2 != CPI_BAD_PLAN;
        A.makespan[item] = ok ? (long long)ms : -1LL;
        if (A.peak_mem) A.peak_mem[item] = ok ? pk : -1;
        A.status[item] = st2;
        if (A.best_key && st2 == 0)
          atomicMin(A.best_key, ((unsigned long long)ms << 32) | (unsigned long long)(uint32_t)(item + A.index_base));
      }
      if (A.stage_stats) {
        // a completed valid row ran every block once: busy = 2m (t_f + t_d + t_w); every row starts
        // with F0 of microbatch 0, whose path is chunk 0's forward: first[s] = max(t_ag[s], first[s-1]
        // + t_f + bw + lat of s-1), the max-plus prefix P_s + max_{k<=s}(ag_k - P_k)
        const int cfw = s < p ? tf + bwR + latR : 0;
        int Pp = cfw;
        for (int d = 1; d < 32; d <<= 1) { const int t2 = __shfl_up_sync(WFULL, Pp, d); if (s >= d) Pp += t2; }
        Pp -= cfw;
        int xq = (s < p ? tag : 0) - Pp;
        for (int d = 1; d < 32; d <<= 1) { const int t2 = __shfl_up_sync(WFULL, xq, d); if (s >= d) xq = wmx(xq, t2); }
        const int busy = 2 * m * (tf + td + tw);
        for (int r = s; r < A.stage_stride; r += 32) {
          const int4 v = (complete && r == s && s < p) ? make_int4(Pp + xq, clk, busy, peak) : make_int4(0, 0, 0, 0);
          *reinterpret_cast<int4*>(A.stage_stats + (item * A.stage_stride + r) * 4) = v;
        }
      }
    }
    __syncwarp();
  }
}

int launch_wave32(const Args& a, int blocks, int threads, size_t smem, void* stream) {
  const bool tl = a.t_start != nullptr;
  const void* fn = a.chunk_pattern == CP_PATTERN_LOOP ? (tl ? (const void*)k_chunk32<true, true> : (const void*)k_chunk32<true, false>)
                                                      : (tl ? (const void*)k_chunk32<false, true> : (const void*)k_chunk32<false, false>);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return (int)e;
  }
  void* params[] = {(void*)&a};
  return (int)cudaLaunchKernel(fn, dim3(blocks), dim3(threads), params, smem, (cudaStream_t)stream);
}

int wave32_blocks_per_sm(int threads, size_t smem) {
  const void* fn = (const void*)k_chunk32<false, false>;
  if (smem > 48 * 1024) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, threads, smem) != cudaSuccess) return 1;
  return n > 0 ? n : 1;
}

}  // namespace cpk
