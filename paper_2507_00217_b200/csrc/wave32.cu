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

__global__ void __launch_bounds__(kFastThreads, kFastMinBlocks) k_wave32(const __grid_constant__ Args A) {
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
      if (s < p - 1) { latR = I->lat_f[s]; bwR = I->bw_f[s]; lat_b_s = I->lat_b[s]; bw_b_s = I->bw_b[s]; }
      if (s > 0) { latL = I->lat_b[s - 1]; bwL = I->bw_b[s - 1]; }
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
    const bool sendR = s < p - 1, sendL = s > 0 && s < p;
    const int wq = tw / ns, wr = tw % ns;
    // parameter tables, entry x = type | chunk << 2:
    //   tabA[x] = {duration, memory delta, link bw, latency} (W: first sub-block / whole W if n_sub 1)
    //   tabB[x] = {input ring column (zero row without a producer), slot mask, output column at the
    //             consumer (0: no message), 1 if the message goes right}
    {
      const int hasL = s > 0, hasR = s < p - 1;
      const int tW = ns == 1 ? tw : wq, mW = ns == 1 ? mw : 0;
      tabA[0 * 32] = make_int4(tf, mf, bwR, latR);
      tabA[1 * 32] = make_int4(td + tw, md + mw, bwL, latL);
      tabA[2 * 32] = make_int4(td, md, bwL, latL);
      tabA[3 * 32] = make_int4(tW, mW, 0, 0);
      tabA[4 * 32] = make_int4(tf, mf, bwL, latL);
      tabA[5 * 32] = make_int4(td + tw, md + mw, bwR, latR);
      tabA[6 * 32] = make_int4(td, md, bwR, latR);
      tabA[7 * 32] = make_int4(tW, mW, 0, 0);
      tabB[0 * 32] = make_int4(hasL ? iF0 : iZ, hasL ? Rm : 0, sendR ? iF0 + 1 : 0, 1);
      tabB[1 * 32] = make_int4(hasR ? iD0 : iZ, hasR ? Rm : 0, sendL ? iD0 - 1 : 0, 0);
      tabB[2 * 32] = tabB[1 * 32];
      tabB[3 * 32] = make_int4(iZ, 0, 0, 0);
      tabB[4 * 32] = make_int4(hasR ? iF1 : iZ, hasR ? Rm : 0, sendL ? iF1 - 1 : 0, 0);
      tabB[5 * 32] = make_int4(hasL ? iD1 : iZ, hasL ? Rm : 0, sendR ? iD1 + 1 : 0, 1);
      tabB[6 * 32] = tabB[5 * 32];
      tabB[7 * 32] = tabB[3 * 32];
    }
    int clk = tag, mem = 0, peak = 0, pos = 0, lkR = 0, lkL = 0;
    // packed counts: aP = nF0 | nD1 << 16 (streams sent right), bP = nF1 | nD0 << 16 (sent left),
    // wP = W sub-blocks of chunk 0 | chunk 1 << 16
    int aP = 0, bP = 0, wP = 0;
    int lm = s == 0 ? 0xffff : 0, rm = s == p - 1 ? 0xffff : 0;      // no producer / no consumer
    asm("mov.b32 %0, %0;" : "+r"(lm));
    asm("mov.b32 %0, %0;" : "+r"(rm));
    const bool last = s == p - 1, first_s = s == 0;
    __syncwarp();
    auto rounds = [&](auto n1) {
      constexpr bool kN1 = decltype(n1)::value;       // n_sub == 1: a W entry is a whole W block
      for (;;) {
        const int la = __shfl_up_sync(WFULL, aP, 1), lb = __shfl_up_sync(WFULL, bP, 1);
        const int ra = __shfl_down_sync(WFULL, aP, 1), rb = __shfl_down_sync(WFULL, bP, 1);
        const int nF0 = aP & 0xffff, nD1 = aP >> 16, nF1 = bP & 0xffff, nD0 = bP >> 16;
        const uint32_t wv = (uint32_t)smem[iP + ((pos >> 3) << 5)];
        const uint32_t x = (wv >> ((pos & 7) << 2)) & 7u;
        const int4 ta = tabA[x << 5];
        const int4 tb = tabB[x << 5];
        const int ch = (int)(x >> 2);
        const bool isF = (x & 3u) == CP_OP_F, isW = (x & 3u) == CP_OP_W;
        // readiness: input produced (or the own turn-around / loss), room in the consumer's ring
        const bool rF0 = (((la & 0xffff) | lm) > nF0) & (nF0 - ((ra & 0xffff) | rm) < R);
        const bool rD1 = ((first_s ? nF1 : (la >> 16)) > nD1) & (nD1 - ((ra >> 16) | rm) < R);
        const bool rF1 = ((last ? nF0 : (rb & 0xffff)) > nF1) & (nF1 - ((lb & 0xffff) | lm) < R);
        const bool rD0 = ((last ? nD1 : (rb >> 16)) > nD0) & (nD0 - ((lb >> 16) | lm) < R);
        const int wc = ch ? (wP >> 16) : (wP & 0xffff), ndc = ch ? nD1 : nD0;
        const bool rW = kN1 ? wc < ndc : wc < ns * ndc;
        const bool rdy = isF ? (ch ? rF1 : rF0) : (isW ? rW : (ch ? rD1 : rD0));
        const bool go = (pos < plen) & rdy;
        const bool right = tb.w != 0;                   // F0, D1 go right; F1, D0 go left
        // the entry's own count of its stream addresses both its input slot and its message slot
        const int cnt = ((right ? aP : bP) >> (isF ? 0 : 16)) & 0xffff;
        const int start = wmx(clk, smem[tb.x + ((cnt & tb.y) << 5)]);
        int dur = ta.x, dm = ta.y;
        if (!kN1) {                                     // W sub-block k of its W block (Q12)
          const int k = wc % ns;
          dur = isW ? wq + (k < wr ? 1 : 0) : dur;
          dm = isW ? (k == ns - 1 ? mw : 0) : dm;
        }
        const int end = start + dur;
        const int nl = wmx(end, right ? lkR : lkL) + ta.z;   // FIFO link clock (App. X1)
        if (go & (tb.z != 0)) smem[tb.z + ((cnt & Rm) << 5)] = nl + ta.w;
        if (A.t_start && go && pos < A.len_stride)
          A.t_start[(item * A.stage_stride + s) * (long long)A.len_stride + pos] = start;
        const int gi = go ? 1 : 0;
        clk = wmadd(gi, end - clk, clk);
        mem = wmadd(gi, dm, mem);
        peak = wmx(peak, mem);
        const int gR = (go & !isW & right) ? 1 : 0, gL = (go & !isW & !right) ? 1 : 0;
        lkR = wmadd(gR, nl - lkR, lkR);
        lkL = wmadd(gL, nl - lkL, lkL);
        // count increments: F0 +1 / D1 +65536 into aP, F1 +1 / D0 +65536 into bP, W into wP
        const int inc = isF ? 1 : 65536;
        aP = wmadd(gR, inc, aP);
        bP = wmadd(gL, inc, bP);
        wP = wmadd((go & isW) ? 1 : 0, ch ? 65536 : 1, wP);
        pos = wmadd(gi, 1, pos);
        __syncwarp();
        if (!__any_sync(WFULL, go)) break;
      }
    };
    if (ns == 1) rounds(std::true_type{});
    else rounds(std::false_type{});
    const int nF0 = aP & 0xffff, nD1 = aP >> 16, nF1 = bP & 0xffff, nD0 = bP >> 16;
    // no lane progressed: complete, a cyclic wait on full rings (-> second pass), or deadlock
    const int lb = __shfl_up_sync(WFULL, bP, 1), ra = __shfl_down_sync(WFULL, aP, 1);
    const bool ring_full = (sendR && (nF0 - (ra & 0xffff) >= R || nD1 - (ra >> 16) >= R)) ||
                           (sendL && (nF1 - (lb & 0xffff) >= R || nD0 - (lb >> 16) >= R));
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
  const void* fn = (const void*)k_wave32;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return (int)e;
  }
  void* params[] = {(void*)&a};
  return (int)cudaLaunchKernel(fn, dim3(blocks), dim3(threads), params, smem, (cudaStream_t)stream);
}

int wave32_blocks_per_sm(int threads, size_t smem) {
  const void* fn = (const void*)k_wave32;
  if (smem > 48 * 1024) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, threads, smem) != cudaSuccess) return 1;
  return n > 0 ? n : 1;
}

}  // namespace cpk
