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

#include "engine.h"

namespace cpk {

namespace {
constexpr int32_t WINF = 1 << 30;
constexpr unsigned WFULL = 0xffffffffu;
__device__ __forceinline__ int wmx(int a, int b) { return a > b ? a : b; }
}  // namespace

__global__ void __launch_bounds__(kThreads) k_wave32(const __grid_constant__ Args A) {
  extern __shared__ __align__(16) int32_t smem[];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int R = A.ring_slots, Rm = R - 1, RW = R * 32;
  const int PW = A.plan_words;                         // staged words per row (>= A.words)
  const long long gwarp = (long long)blockIdx.x * (blockDim.x >> 5) + wib;
  const long long nwarps = (long long)gridDim.x * (blockDim.x >> 5);
  // per-warp smem (words): [rF0][rD1][rF1][rD0] (R*32 each) [plan PW*32]
  const int wbase = wib * A.smem_words_per_warp;
  const int iF0 = wbase + lane, iD1 = iF0 + RW, iF1 = iD1 + RW, iD0 = iF1 + RW;
  const int iP = iD0 + RW;
  for (int k = lane; k < 4 * RW; k += 32) smem[wbase + k] = 0;
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
    // stage this lane's row and check Q29 per chunk (counts, W prefix rule, codes < 8)
    bool bplan = false;
    if (!st && s < p) {
      int cF[2] = {0, 0}, cB[2] = {0, 0}, cD[2] = {0, 0}, cW[2] = {0, 0};
      for (int k = 0; k * 8 < plen; ++k) {
        const uint32_t w = A.ops[(item * A.words + k) * A.stage_stride + s];
        smem[iP + (k << 5)] = (int32_t)w;
        const int n = plen - 8 * k < 8 ? plen - 8 * k : 8;
        for (int e = 0; e < n; ++e) {
          const uint32_t x = (w >> (4 * e)) & 15u;
          const int ty = x & 3, ch = (x >> 2) & 1;
          if (x & 8u) bplan = true;
          if (ty == CP_OP_F) ++cF[ch];
          else if (ty == CP_OP_B) ++cB[ch];
          else if (ty == CP_OP_D) ++cD[ch];
          else { ++cW[ch]; if (cW[ch] > ns * cD[ch]) bplan = true; }
        }
      }
      for (int ch = 0; ch < 2; ++ch)
        if (cF[ch] != m || cB[ch] + cD[ch] != m || cW[ch] != ns * cD[ch]) bplan = true;
      if (cB[0] + cB[1] > 0 && cD[0] + cD[1] + cW[0] + cW[1] > 0) bplan = true;
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
    // the last stage's right rings and stage 0's left rings have no producer in this item: masks
    const int mL = s > 0 ? -1 : 0, mR = s < p - 1 ? -1 : 0;
    const bool sendR = s < p - 1, sendL = s > 0 && s < p;
    const int wq = tw / ns, wr = tw % ns;
    int clk = tag, mem = 0, peak = 0, busy = 0, first = 0, pos = 0;
    int nF0 = 0, nF1 = 0, nD0 = 0, nD1 = 0, w0 = 0, w1 = 0, lkR = 0, lkL = 0;
    __syncwarp();
    for (;;) {
      const int aP = nF0 | (nD1 << 16), bP = nF1 | (nD0 << 16);     // right-going / left-going counts
      const int la = __shfl_up_sync(WFULL, aP, 1), lb = __shfl_up_sync(WFULL, bP, 1);
      const int ra = __shfl_down_sync(WFULL, aP, 1), rb = __shfl_down_sync(WFULL, bP, 1);
      const uint32_t wv = (uint32_t)smem[iP + ((pos >> 3) << 5)];
      const uint32_t x = (wv >> ((pos & 7) << 2)) & 15u;
      const int ty = x & 3, ch = (x >> 2) & 1;
      const bool isF = ty == CP_OP_F, isW = ty == CP_OP_W, isB = ty == CP_OP_B, isDB = !isF && !isW;
      // readiness: input produced (or the own turn-around / loss), room in the consumer's ring
      const bool rF0 = (s == 0 || (la & 0xffff) > nF0) && (!sendR || nF0 - (ra & 0xffff) < R);
      const bool rD1 = (s == 0 ? nF1 > nD1 : (la >> 16) > nD1) && (!sendR || nD1 - (ra >> 16) < R);
      const bool rF1 = (s == p - 1 ? nF0 > nF1 : (rb & 0xffff) > nF1) && (!sendL || nF1 - (lb & 0xffff) < R);
      const bool rD0 = (s == p - 1 ? nD1 > nD0 : (rb >> 16) > nD0) && (!sendL || nD0 - (lb >> 16) < R);
      const int wc = ch ? w1 : w0, ndc = ch ? nD1 : nD0;
      const bool rW = wc < ns * ndc;
      const bool go = (pos < plen) && (isF ? (ch ? rF1 : rF0) : (isW ? rW : (ch ? rD1 : rD0)));
      // input arrival: F0 / D1 from the left rings, F1 / D0 from the right rings; W: none
      int avail = 0;
      if (isF && ch == 0) avail = smem[iF0 + ((nF0 & Rm) << 5)] & mL;
      else if (isF) avail = smem[iF1 + ((nF1 & Rm) << 5)] & mR;
      else if (isDB && ch == 1) avail = smem[iD1 + ((nD1 & Rm) << 5)] & mL;
      else if (isDB) avail = smem[iD0 + ((nD0 & Rm) << 5)] & mR;
      const int start = wmx(clk, avail);
      const int k = wc % ns;
      const int dur = isF ? tf : (isW ? wq + (k < wr ? 1 : 0) : (isB ? td + tw : td));
      const int dm = isF ? mf : (isW ? (k == ns - 1 ? mw : 0) : (isB ? md + mw : md));
      const int end = start + dur;
      const bool right = (isF && ch == 0) || (isDB && ch == 1);   // F0, D1 go right; F1, D0 go left
      const int nl = wmx(end, right ? lkR : lkL) + (right ? bwR : bwL);   // FIFO link clock (App. X1)
      if (go && !isW && (right ? sendR : sendL)) {
        const int col = (isF ? (ch ? iF1 : iF0) : (ch ? iD1 : iD0)) + (right ? 1 : -1);
        const int cnt = isF ? (ch ? nF1 : nF0) : (ch ? nD1 : nD0);
        smem[col + ((cnt & Rm) << 5)] = nl + (right ? latR : latL);
      }
      if (go) {
        if (A.t_start && pos < A.len_stride) A.t_start[(item * A.stage_stride + s) * (long long)A.len_stride + pos] = start;
        if (pos == 0) first = start;
        clk = end;
        busy += dur;
        mem += dm;
        peak = wmx(peak, mem);
        if (right && !isW) lkR = nl;
        else if (!isW) lkL = nl;
        if (isF) { if (ch) ++nF1; else ++nF0; }
        else if (isW) { if (ch) ++w1; else ++w0; }
        else { if (ch) ++nD1; else ++nD0; }
        ++pos;
      }
      __syncwarp();
      if (!__any_sync(WFULL, go)) break;
    }
    // no lane progressed: complete, a cyclic wait on full rings (-> second pass), or deadlock
    const int aP = nF0 | (nD1 << 16), bP = nF1 | (nD0 << 16);
    const int lb = __shfl_up_sync(WFULL, bP, 1), ra = __shfl_down_sync(WFULL, aP, 1);
    const bool ring_full = (sendR && (nF0 - (ra & 0xffff) >= R || nD1 - (ra >> 16) >= R)) ||
                           (sendL && (nF1 - (lb & 0xffff) >= R || nD0 - (lb >> 16) >= R));
    const bool complete = !__any_sync(WFULL, s < p && pos < plen);
    int st2;
    if (!complete && __any_sync(WFULL, ring_full) && !A.from_list) st2 = -1;
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
        A.makespan[item] = complete ? (long long)ms : -1LL;
        if (A.peak_mem) A.peak_mem[item] = complete ? pk : -1;
        A.status[item] = st2;
        if (A.best_key && st2 == 0)
          atomicMin(A.best_key, ((unsigned long long)ms << 32) | (unsigned long long)(uint32_t)(item + A.index_base));
      }
      if (A.stage_stats)
        for (int r = s; r < A.stage_stride; r += 32) {
          const int4 v = (complete && r == s && s < p) ? make_int4(first, clk, busy, peak) : make_int4(0, 0, 0, 0);
          *reinterpret_cast<int4*>(A.stage_stats + (item * A.stage_stride + r) * 4) = v;
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
