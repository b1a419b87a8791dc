// chunk_fast.cu -- first pass of cp_simulate for one-chunk UD plans (the config-4 bench shape) and
// two-chunk plans (Wave, reading Q32; Loop, Q33): one item per warp, lane = stage, round-synchronous.
// Items it does not finish (a stall, which may be an artefact of its 8-slot rings, n_sub > 1,
// n_mb > 127, anything invalid) go to the overflow list and are evaluated exactly by the second pass
// with rings of n_mb slots: k_sim32 (sim32.cu) for UD, k_chunk32 (wave32.cu) for Wave / Loop.
//
// What makes the round short:
//  * Block counts are bytes.  c = {F0, F1, D0, D1} counts + 128 (UD: {F, D, -, -}; every byte has its
//    top bit set), one register; one shuffle per direction hands a lane its neighbours' counts.
//  * Readiness of the entry's own stream in three PRMTs and three compares: the producer count X,
//    the consumer count Y and the own count n are byte-selected into the top byte (X from the left /
//    right neighbour, or the own count at a turn-around / the loss, or 0xFF = "no producer" by sign
//    replication of a biased byte), and the entry is ready iff X > n and n - Y < R.  The selectors
//    come from per-lane 8-entry byte tables held in registers, indexed by the entry code with one
//    more PRMT each.  W entries use the same test: their n is the sign of the chunk's W deficit byte
//    w = 128 - (#D - #W) (0x00 when a D is owed its W, else 0xFF) against X = Y = 0xFF.
//  * Costs, ring and link addresses and count increments come from two per-lane table rows (int4),
//    shared by the block when every item uses one instance.
//  * Ring slot = own count mod R, read from the top byte of n; a message goes to the consumer's ring
//    at the same slot (producer count = consumer's index of that message).
//  * Entries past a row's end read as D (D0), never ready once the row is done, so there is no
//    position test; the plan word is pre-rotated by 4 bits so the decode is one funnel shift and one
//    LOP3 (UD codes are 2 bits, 16 per word; two-chunk entries 4 bits, 8 per word).
#include <cuda_runtime.h>
#include <stdint.h>

#include "engine.h"
#include "ptx.cuh"

#ifndef CHUNKF_UD_LKREG
// UD: the two FIFO link clocks in registers (one select, two predicated updates) instead of a
// shared-memory load and store per round: measured +1.7% on config 4 (77.5 -> 78.8 M evals/s)
#define CHUNKF_UD_LKREG 1
#endif
#ifndef CHUNKF_2C_LKREG
#define CHUNKF_2C_LKREG 0   // the same for Wave / Loop (the link is the one the table's link address names)
#endif
#ifndef CHUNKF_2C_MINB
#define CHUNKF_2C_MINB 2   // Wave / Loop (with CHUNKF_2C_THREADS = 384)
#endif
#ifndef CHUNKF_UD_MINB
#define CHUNKF_UD_MINB 6   // UD: 24 resident warps at <= 80 registers (measured +0.6% over 20 warps; 28, 32: no further gain)
#endif

namespace cpk {

namespace {
constexpr unsigned FMASK = 0xffffffffu;
constexpr int32_t CINF = 1 << 30;
__device__ __forceinline__ int cmax(int a, int b) { return a > b ? a : b; }
__device__ __forceinline__ int cmadd(int g, int d, int x) {   // x + g*d on the FMA pipe
  int r;
  asm("mad.lo.s32 %0, %1, %2, %3;" : "=r"(r) : "r"(g), "r"(d), "r"(x));
  return r;
}
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
  return d;
}
// timeline staging: the 8 start ticks in the lane's slots [k][lane], k < 8, -> two 16-B global stores
__device__ __forceinline__ void tl_flush8(unsigned stg, int32_t* dst) {
  int v[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v[k]) : "r"(stg + 128u * k));
  __stcs(reinterpret_cast<int4*>(dst), make_int4(v[0], v[1], v[2], v[3]));
  __stcs(reinterpret_cast<int4*>(dst) + 1, make_int4(v[4], v[5], v[6], v[7]));
}
// 8 selector bytes (source byte index in the top nibble, 0xF below) -> two registers
__device__ __forceinline__ void pack_sel(const int (&ix)[8], uint32_t& lo, uint32_t& hi) {
  lo = hi = 0;
#pragma unroll
  for (int x = 0; x < 4; ++x) {
    lo |= (uint32_t)((ix[x] << 4) | 0xF) << (8 * x);
    hi |= (uint32_t)((ix[x + 4] << 4) | 0xF) << (8 * x);
  }
}

// Per-lane table rows of instance I (entry x = type | chunk << 2).  T0/T1 point at [x = 0][lane],
// rows 32 int4 apart; U at [0] (16-B rows).  Addresses are byte offsets from the warp region.
template <int kPat>   // CP_PATTERN_UD / _WAVE / _LOOP
__device__ void chunkf_tables(const cp_inst_v1* I, int s, int R, const ChunkFLayout& Ly, int4* T0, int4* T1, int* U) {
  constexpr bool kUD = kPat == CP_PATTERN_UD, kLoop = kPat == CP_PATTERN_LOOP;
  const int p = I->n_pp < 1 ? 1 : (I->n_pp > CP_MAX_STAGES ? CP_MAX_STAGES : I->n_pp);   // (other p: not run here)
  const bool live = s < p, first = s == 0, last = s == p - 1;
  int tf = 0, td = 0, tw = 0, mf = 0, md = 0, mw = 0, latR = 0, bwR = 0, latL = 0, bwL = 0;
  if (live) {
    tf = I->t_f[s]; td = I->t_d[s]; tw = I->t_w[s];
    mf = I->m_f[s]; md = I->m_d[s]; mw = I->m_w[s];
    // boundary s = link s -> s+1; Loop also uses index p-1, the wrap links p-1 -> 0 / 0 -> p-1 (Q33)
    if (s < p - 1 || kLoop) { latR = I->lat_f[s]; bwR = I->bw_f[s]; }
    if (s > 0) { latL = I->lat_b[s - 1]; bwL = I->bw_b[s - 1]; }
    else if (kLoop) { latL = I->lat_b[p - 1]; bwL = I->bw_b[p - 1]; }
  }
  const int RB = R * 128, col = 4 * s;
  const int rF0 = Ly.rings * 4 + col, rF1 = rF0 + RB, rD0 = rF0 + 2 * RB, rD1 = rF0 + 3 * RB;
  const int z = Ly.zero * 4 + col, lkR = Ly.lk * 4 + col, lkL = lkR + 128;
  const auto L = [&](int lat) { return live ? lat : -1; };   // latency -1: the entry sends nothing
  if (kUD) {
    // rings F (0) and D (1); F goes right, D / B left; entry x = code, rows 4..7 repeat 0..3.  One
    // count register c = {F, D, W deficit, #B} (+128 each): F +1; B: D +1, #B +1; D: D +1, deficit -1;
    // W: deficit +1
    for (int h = 0; h < 256; h += 128) {
      T0[h] = make_int4(tf, mf, bwR, L(last ? -1 : latR));
      T1[h] = make_int4(rF0, rF0 + 4, lkR, 1);
      T0[h + 32] = make_int4(td + tw, md + mw, bwL, L(first ? -1 : latL));
      T1[h + 32] = make_int4(rF1, rF1 - 4, lkL, (1 << 8) + (1 << 24));
      T0[h + 64] = make_int4(td, md, bwL, L(first ? -1 : latL));
      T1[h + 64] = make_int4(rF1, rF1 - 4, lkL, (1 << 8) - (1 << 16));
      T0[h + 96] = make_int4(tw, mw, 0, -1);
      T1[h + 96] = make_int4(z, z, lkR, 1 << 16);
    }
    return;
  }
  // chunk 0: F0 goes right (Loop: the last stage's F0 takes the wrap link into stage 0's F1 ring);
  // D0 / B0 go left (stage 0's have no consumer)
  T0[0] = make_int4(tf, mf, bwR, L(kLoop || !last ? latR : -1));
  T1[0] = make_int4(rF0, kLoop && last ? Ly.rings * 4 + RB : rF0 + 4, lkR, 1);
  T0[32] = make_int4(td + tw, md + mw, bwL, L(first ? -1 : latL));
  T1[32] = make_int4(rD0, rD0 - 4, lkL, 1 << 16);
  T0[64] = make_int4(td, md, bwL, L(first ? -1 : latL));
  T1[64] = T1[32];
  T0[96] = make_int4(tw, mw, 0, -1);
  T1[96] = make_int4(z, z, lkR, 0);
  // chunk 1.  Wave: F1 goes left (stage 0's F1 ends in the loss), D1 right (the last stage's turns
  // into its D0).  Loop: F1 goes right (the last stage's ends in the loss), D1 left (stage 0's takes
  // the wrap link into the last stage's D0 ring).
  if (kLoop) {
    T0[128] = make_int4(tf, mf, bwR, L(last ? -1 : latR));
    T1[128] = make_int4(rF1, rF1 + 4, lkR, 1 << 8);
    T0[160] = make_int4(td + tw, md + mw, bwL, L(latL));
    T1[160] = make_int4(rD1, first ? Ly.rings * 4 + 2 * RB + 4 * (p - 1) : rD1 - 4, lkL, 1 << 24);
    T0[192] = make_int4(td, md, bwL, L(latL));
  } else {
    T0[128] = make_int4(tf, mf, bwL, L(first ? -1 : latL));
    T1[128] = make_int4(rF1, rF1 - 4, lkL, 1 << 8);
    T0[160] = make_int4(td + tw, md + mw, bwR, L(last ? -1 : latR));
    T1[160] = make_int4(rD1, rD1 + 4, lkR, 1 << 24);
    T0[192] = make_int4(td, md, bwR, L(last ? -1 : latR));
  }
  T1[192] = T1[160];
  T0[224] = make_int4(tw, mw, 0, -1);
  T1[224] = make_int4(z, z, lkR, 0);
  // W-deficit increments (the byte of chunk c holds 128 - (#D - #W)): D -1, W +1
  // and B +1 << 16 (byte 2 counts B blocks: the mixing rule)
  if (s < 8) U[4 * s] = s == 2 ? -1 : s == 3 ? 1 : s == 6 ? -256 : s == 7 ? 256 : (s & 3) == 1 ? 1 << 16 : 0;
}
}  // namespace

template <int kPat, bool kTL>   // kPat: CP_PATTERN_UD / _WAVE / _LOOP; kTL: per-entry start ticks (A.t_start)
__global__ void __launch_bounds__(kPat == CP_PATTERN_UD ? kChunkFThreads : kChunkF2CThreads,
                                  kPat == CP_PATTERN_UD ? CHUNKF_UD_MINB : CHUNKF_2C_MINB) k_chunk32f(const __grid_constant__ Args A) {
  constexpr bool kUD = kPat == CP_PATTERN_UD, kLoop = kPat == CP_PATTERN_LOOP;
  constexpr int kRings = kUD ? 2 : 4, kEPW = kUD ? 16 : 8, kStep = 32 / kEPW;   // entries per word, bits per entry
  constexpr int kChunks = kUD ? 1 : 2;
  constexpr uint32_t kPad = kUD ? 0xaaaaaaaau : 0x22222222u;   // D (UD) / D0 entries: never ready at the end
  extern __shared__ __align__(1024) int32_t smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, s = lane;
  const int R = A.ring_slots, Rm = R - 1, PW = A.words;
  constexpr bool kStage = kTL && kUD;             // UD timelines: staged, written 8 ticks (32 B) per lane
  const ChunkFLayout Ly = chunkf_layout(R, PW, A.shared_tab != 0, kRings, kStage);
  const int wbase = Ly.hdr + wib * Ly.per_warp;
  const int tbase = A.shared_tab ? 0 : wbase + Ly.tab;
  const unsigned sb = smem_u32(smem), wb = sb + 4u * (unsigned)wbase;
  uint64_t* const bar = reinterpret_cast<uint64_t*>(smem + wbase + Ly.bars);
  int32_t* const plan = smem + wbase + Ly.plan;
  int4* const T0 = reinterpret_cast<int4*>(smem + tbase) + lane;
  int4* const T1 = T0 + 256;
  int* const U = smem + tbase + 2048;
  const long long gwarp = (long long)blockIdx.x * (blockDim.x >> 5) + wib;
  const long long nwarps = (long long)gridDim.x * (blockDim.x >> 5);

  // zero block (zero rows + link clocks) and rings start at 0; the zero rows are never written
  for (int k = lane; k < (kRings * R + Ly.zrows) * 32; k += 32) smem[wbase + Ly.rings + k] = 0;   // rings, zero block
  if (lane == 0) mbar_init(bar);
  if (A.shared_tab) {                               // every item uses instance 0 (host guarantees)
    if (wib == 0) chunkf_tables<kPat>(A.inst, lane, R, Ly, T0, T1, U);
    __syncthreads();
  }
  __syncwarp();
  long long tab_inst = -1;                          // instance of the warp's own tables
  uint32_t phase = 0;
  // 0 at run time, unknown to the compiler: keeps loop constants in registers ((r & 0x70) | 15 one
  // LOP3, the n-selector table not rematerialized every round)
  const uint32_t opq = (uint32_t)A.words >> 30;
  const uint32_t fifteen = 15u | (opq << 20);       // (bits >= 16 of a PRMT selector are ignored)

  // items are handed out by a counter (A.work_counter), the next index fetched one item ahead; without
  // a counter, warp w takes items w, w + warps, ...
  const bool dyn = A.work_counter != nullptr;
  long long item = gwarp, nxt = 0;
  if (dyn) {
    int t0 = 0;
    if (lane == 0) t0 = atomicAdd(A.work_counter, 1);
    item = __shfl_sync(FMASK, t0, 0);
  }
  for (; item < A.n_items; item = dyn ? (long long)__shfl_sync(FMASK, (int)nxt, 0) : item + nwarps) {
    if (dyn && lane == 0) nxt = atomicAdd(A.work_counter, 1);
    // the previous item's generic-proxy writes to the plan rows are ordered before the bulk copy
    if (lane == 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (lane == 0) tma_load_1d(plan, A.ops + item * PW * 32, (uint32_t)PW * 128u, bar);
    const long long ii = A.inst_of ? (long long)A.inst_of[item] : (A.n_inst == 1 ? 0 : item);
    const cp_inst_v1* I = A.inst + ii;
    const int p = I->n_pp, m = I->n_mb, ns = I->n_sub;
    int tf = 0, td = 0, tw = 0, mf = 0, md = 0, mw = 0, mlim = 0, tdp = 0, tag = 0;
    int latR = 0, bwR = 0, latL = 0, bwL = 0, lat_b_s = 0, bw_b_s = 0, plen = 0;
    if (s < p && p <= CP_MAX_STAGES) {
      tf = I->t_f[s]; td = I->t_d[s]; tw = I->t_w[s];
      mf = I->m_f[s]; md = I->m_d[s]; mw = I->m_w[s]; mlim = I->m_lim[s];
      tdp = I->t_dp[s]; tag = (I->flags & 1) ? I->t_ag[s] : 0;
      if (s < p - 1 || kLoop) { latR = I->lat_f[s]; bwR = I->bw_f[s]; lat_b_s = I->lat_b[s]; bw_b_s = I->bw_b[s]; }
      if (s > 0) { latL = I->lat_b[s - 1]; bwL = I->bw_b[s - 1]; }
      else if (kLoop) { latL = I->lat_b[p - 1]; bwL = I->bw_b[p - 1]; }
      plen = A.len[item * 32 + s];
    }
    // the shapes this pass takes; everything else is classified by the exact pass
    bool ok = p >= (kLoop ? 2 : 1) && p <= CP_MAX_STAGES && m >= 1 && m <= 127 && ns == 1;
    if (ok && s < p)
      ok = tf >= 1 && td >= 1 && tw >= 1 && mf > 0 && md <= 0 && mw <= 0 && (long long)mf + md + mw == 0 &&
           mlim >= mf && tdp >= 0 && I->t_ag[s] >= 0 && latR >= 0 && bwR >= 0 && lat_b_s >= 0 && bw_b_s >= 0 &&
           plen <= kEPW * PW;
    long long u = (s < p && ok) ? kChunks * (long long)m * ((long long)tf + td + tw) + tag + tdp +
                                      kChunks * (long long)m * ((long long)latR + bwR + latL + bwL)
                                : 0;
    for (int d = 16; d > 0; d >>= 1) u += __shfl_xor_sync(FMASK, u, d);
    ok = __all_sync(FMASK, ok) && u < (long long)CINF;
    mbar_wait(bar, phase);
    phase ^= 1u;
    // stage the row: codes < 8, pad past the end with D0, pre-rotate by one entry.  Q29's count and
    // mixing rules are checked on the final counts of a completed row (below); the W-prefix rule is
    // dynamic (a W ahead of its D never becomes ready).  No count can wrap its byte: an entry runs
    // only while its own count is below its producer's (<= 255), and a W only while a D is owed.
    if (ok) {
      bool bplan = false;
      for (int k = 0; k <= PW; ++k) {
        uint32_t w = (uint32_t)plan[(k << 5) + lane];
        const int n = s < p ? min(max(plen - kEPW * k, 0), kEPW) : 0;
        const uint32_t keep = n == kEPW ? 0xffffffffu : ((1u << (kStep * n)) - 1u);
        if (!kUD) bplan |= ((w & keep & 0x88888888u) != 0u);
        w = (w & keep) | (kPad & ~keep);
        plan[(k << 5) + lane] = (int32_t)((w << 4) | (w >> 28));
      }
      ok = !__any_sync(FMASK, bplan);
    }
    if (!ok) {                                      // the exact pass takes it
      if (lane == 0) { const int slot = atomicAdd(A.ovf_count, 1); A.ovf_list[slot] = (int32_t)item; }
      __syncwarp();
      continue;
    }
    if (!A.shared_tab && ii != tab_inst) {
      chunkf_tables<kPat>(I, lane, R, Ly, T0, T1, U);
      tab_inst = ii;
    }
    // ring columns read without a producer in this item but written by a larger previous one
    // (UD: the last stage's D input; Wave: the last stage's F1 / D0 inputs; Loop: its D1 input) must read 0
    if (p < 32)
      for (int k = lane; k < R; k += 32) {
        const int c0 = wbase + Ly.rings + (k << 5) + (p - 1);
        smem[c0 + R * 32] = 0;                      // UD: D; F1
        if (!kUD) {
          smem[c0 + 2 * R * 32] = 0;                // D0
          smem[c0 + 3 * R * 32] = 0;                // D1
        }
      }
    smem[wbase + Ly.lk + lane] = 0;                 // both link clocks start at 0
    smem[wbase + Ly.lk + 32 + lane] = 0;
    // selector tables (entry x -> source byte of X / Y in {R:L}, of n in {w:c}); 8 = no producer /
    // no consumer (sign of a biased byte = 0xFF)
    const bool first = s == 0, last = s == p - 1;
    uint32_t kxl, kxh, kyl, kyh, knl, knh;
    {
      int ix[8], iy[8];
      if (kUD) {
        const int tx[8] = {first ? 8 : 0, last ? 4 : 5, last ? 4 : 5, 8, first ? 8 : 0, last ? 4 : 5, last ? 4 : 5, 8};
        const int ty[8] = {last ? 8 : 4, first ? 8 : 1, first ? 8 : 1, 8, last ? 8 : 4, first ? 8 : 1, first ? 8 : 1, 8};
        for (int x = 0; x < 8; ++x) { ix[x] = tx[x]; iy[x] = ty[x]; }
      } else if (kLoop) {
        const int tx[8] = {first ? 8 : 0, 6, 6, 8, first ? 0 : 1, 7, 7, 8};
        const int ty[8] = {last ? 5 : 4, first ? 8 : 2, first ? 8 : 2, 8, last ? 8 : 5, first ? 2 : 3, first ? 2 : 3, 8};
        for (int x = 0; x < 8; ++x) { ix[x] = tx[x]; iy[x] = ty[x]; }
      } else {
        const int tx[8] = {first ? 8 : 0, last ? 7 : 6, last ? 7 : 6, 8, last ? 4 : 5, first ? 1 : 3, first ? 1 : 3, 8};
        const int ty[8] = {last ? 8 : 4, first ? 8 : 2, first ? 8 : 2, 8, first ? 8 : 1, last ? 8 : 7, last ? 8 : 7, 8};
        for (int x = 0; x < 8; ++x) { ix[x] = tx[x]; iy[x] = ty[x]; }
      }
      const int tn[8] = {0, kUD ? 1 : 2, kUD ? 1 : 2, kUD ? 10 : 12, kUD ? 0 : 1, kUD ? 1 : 3, kUD ? 1 : 3, kUD ? 10 : 13};
      pack_sel(ix, kxl, kxh);
      pack_sel(iy, kyl, kyh);
      pack_sel(tn, knl, knh);
      knl ^= opq;
      knh ^= opq;
    }
    // Loop: the left / right partner lanes (wrap at both ends); the last stage's right view carries
    // {-, stage 0's F1, stage 0's D1, own F1} (fix-up selector)
    const int srcL = first ? (kLoop ? p - 1 : s) : (s < p ? s - 1 : s);
    const int srcR = last ? (kLoop ? 0 : s) : (s < p ? s + 1 : s);
    const uint32_t fixR = (kLoop && last) ? 0x5310u : 0x3210u;
    __syncwarp();

    // counts + 128; two-chunk: W deficits (bytes 0, 1), #B (byte 2), sign byte 3 in w
    uint32_t c = 0x80808080u, w = 0x80008080u;
    int clk = tag, mem = 0, peak = 0, pos4 = 0, lkR = 0, lkL = 0;
    const unsigned tab0m = sb + 4u * (unsigned)tbase + 16u * (unsigned)lane - 480u;   // T0[x][lane] - 15*32
    const unsigned ubm = sb + 4u * (unsigned)(tbase + 2048) - 15u;                    // U[x] - 15
    const unsigned iPb = wb + 4u * (unsigned)(Ly.plan + lane);
    const int R24 = R << 24, Rm7 = Rm << 7, lk_off_r = 4 * (Ly.lk + lane);
    int32_t* const trow = kTL ? A.t_start + (item * A.stage_stride + s) * (long long)A.len_stride : nullptr;
    const unsigned stg = wb + 4u * (unsigned)(Ly.stage + lane);   // staging slot [0][lane]
    int rr = 0, fg = 0;                              // (staged timeline) round counter, next group to write
    uint32_t wv;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(wv) : "r"(iPb));
    for (;;) {
      uint32_t Lv, Rv;
      // both neighbours' counts (stage 0 / the last stage of Wave see their own; Loop wraps)
      asm volatile("shfl.sync.idx.b32 %0, %2, %3, 0x1f, 0xffffffff;\n\t"
                   "shfl.sync.idx.b32 %1, %2, %4, 0x1f, 0xffffffff;"
                   : "=r"(Lv), "=r"(Rv) : "r"(c), "r"(srcL), "r"(srcR));
      if (kLoop) Rv = prmt(Rv, c, fixR);
      uint32_t r, x4;
      asm("shf.r.wrap.b32 %0, %1, %1, %2;" : "=r"(r) : "r"(wv), "r"(pos4));
      asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(x4) : "r"(r), "n"(kUD ? 0x30 : 0x70), "r"(fifteen));   // entry << 4 | 15
      const unsigned ta = tab0m + (x4 << 5);
      int4 t0, t1;
      int iw;
      asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(t0.x), "=r"(t0.y), "=r"(t0.z), "=r"(t0.w) : "r"(ta));
      asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4+4096];" : "=r"(t1.x), "=r"(t1.y), "=r"(t1.z), "=r"(t1.w) : "r"(ta));
      if (!kUD) asm volatile("ld.shared.b32 %0, [%1];" : "=r"(iw) : "r"(ubm + x4));
      const uint32_t sX = prmt(kxl, kxh, x4), sY = prmt(kyl, kyh, x4), sN = prmt(knl, knh, x4);
      const uint32_t X = prmt(Lv, Rv, sX), Y = prmt(Lv, Rv, sY), n = prmt(c, kUD ? c : w, sN);
      const bool go = (X > n) & ((int)(n - Y) < R24);
      const bool isF = kUD ? (x4 & 0xF0u) == 0u : t1.z == lk_off_r;   // the message takes the right link
      unsigned ia, oa;
      const unsigned la = wb + (unsigned)t1.z;
      if (kUD && CHUNKF_WBS) {
        // UD warp regions are 1 KB-aligned (chunkf_layout, __align__(1024)) and a slot offset is below
        // 1 KB (R <= 8), so base | slot = base + slot: one LOP3, and the two adds become 2-input
        // (FMA-pipe) adds -- this loop is ALU-pipe bound (config 4: 79.4 -> 83.1 M evals/s)
        unsigned wbs;
        asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(wbs) : "r"(n >> 17), "r"((unsigned)Rm7), "r"(wb));
        ia = wbs + (unsigned)t1.x;
        oa = wbs + (unsigned)t1.y;
      } else {
        const unsigned slot = (n >> 17) & (unsigned)Rm7;
        ia = wb + (unsigned)t1.x + slot;
        oa = wb + (unsigned)t1.y + slot;
      }
      int arr, lk;
      asm volatile("ld.shared.b32 %0, [%1];" : "=r"(arr) : "r"(ia));
      constexpr bool kLkReg = kUD ? CHUNKF_UD_LKREG : CHUNKF_2C_LKREG;
      if (kLkReg) lk = isF ? lkR : lkL;
      else asm volatile("ld.shared.b32 %0, [%1];" : "=r"(lk) : "r"(la));
      const int start = cmax(clk, arr);
      const int end = start + t0.x;
      const int nl = cmax(end, lk) + t0.z;          // FIFO link clock (App. X1)
      const bool snd = go & (t0.w >= 0);
      if (snd) {
        asm volatile("st.shared.b32 [%0], %1;" :: "r"(oa), "r"(nl + t0.w) : "memory");
        if (!kLkReg) asm volatile("st.shared.b32 [%0], %1;" :: "r"(la), "r"(nl) : "memory");
      }
      if (kLkReg) {
        lkR = (snd & isF) ? nl : lkR;
        lkL = (snd & !isF) ? nl : lkL;
      }
      if (kStage)   // start tick of entry pos4 / 2 into staging slot (entry & 15), predicated, no branch
        asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.s32 q, %2, 0;\n\t@q st.shared.b32 [%0], %1;\n\t}"
                     :: "r"(stg + (((unsigned)pos4 & 30u) << 6)), "r"(start), "r"((int)go) : "memory");
      else if (kTL && go && pos4 / kStep < A.len_stride) trow[pos4 / kStep] = start;
      const int gi = go ? 1 : 0;
      clk = cmadd(gi, end - clk, clk);
      mem = cmadd(gi, t0.y, mem);
      peak = cmax(peak, mem);
      c = (uint32_t)cmadd(gi, t1.w, (int)c);
      if (!kUD) w = (uint32_t)cmadd(gi, iw, (int)w);
      pos4 = cmadd(gi, kStep, pos4);
      unsigned wa;
      asm("mad.lo.u32 %0, %1, 4, %2;" : "=r"(wa) : "r"((unsigned)pos4 & ~31u), "r"(iPb));
      asm volatile("ld.shared.b32 %0, [%1];" : "=r"(wv) : "r"(wa));
      if (kStage && (++rr & 7) == 0 && (pos4 >> 4) > fg) {
        // warp-uniform every 8th round: a lane advances <= 8 entries in 8 rounds, so at most one aligned
        // group of 8 has completed since the last flush and the 16-slot ring still holds it
        tl_flush8(stg + ((unsigned)(fg & 1) << 10), trow + 8 * fg);
        ++fg;
      }
      __syncwarp();
      if (!__any_sync(FMASK, go)) break;
    }
    if (kStage)                                     // entries not yet written (< 16)
      for (int k = 8 * fg; k < pos4 / kStep; ++k) trow[k] = smem[wbase + Ly.stage + ((k & 15) << 5) + lane];
    const int pos = pos4 / kStep;
    // completed, with Q29's counts: F, D + B of each chunk m (c), as many W as D per chunk (deficit
    // bytes back at 128), B and D not mixed on a stage (#B, byte 2 of w, is 0 or kChunks m)
    bool rowok;
    if (kUD) {   // c = {F, D, deficit, #B} + 128
      const uint32_t bcnt = c >> 24;
      rowok = s >= p || (pos == plen && (c & 0xffffffu) == 0x808080u + 0x0101u * (uint32_t)m &&
                         (bcnt == 128u || bcnt == 128u + (uint32_t)m));
    } else {
      const uint32_t bcnt = (w >> 16) & 0xffu;
      rowok = s >= p || (pos == plen && c == 0x01010101u * (uint32_t)(128 + m) && (w & 0xffffu) == 0x8080u &&
                         (bcnt == 0u || bcnt == (uint32_t)(2 * m)));
    }
    const bool complete = __all_sync(FMASK, rowok);
    if (!complete) {                                // stalled or invalid: the exact pass classifies it
      if (lane == 0) { const int slot = atomicAdd(A.ovf_count, 1); A.ovf_list[slot] = (int32_t)item; }
      __syncwarp();
      continue;
    }
    const int st = __any_sync(FMASK, s < p && peak > mlim) ? CPI_MEM_EXCEEDED : 0;
    int ms = s < p ? cmax(clk + tdp, tag) : 0, pk = s < p ? peak : 0;
    for (int d = 16; d > 0; d >>= 1) {
      ms = cmax(ms, __shfl_xor_sync(FMASK, ms, d));
      pk = cmax(pk, __shfl_xor_sync(FMASK, pk, d));
    }
    if (lane == 0) {
      A.makespan[item] = (long long)ms;
      if (A.peak_mem) A.peak_mem[item] = pk;
      A.status[item] = st;
      if (A.best_key && st == 0)
        atomicMin(A.best_key, ((unsigned long long)ms << 32) | (unsigned long long)(uint32_t)(item + A.index_base));
    }
    if (A.stage_stats) {
      // busy = chunks * m (t_f + t_d + t_w); first[s] = max(t_ag[s], first[s-1] + t_f + bw + lat of s-1): the
      // max-plus prefix P_s + max_{k<=s}(ag_k - P_k) along chunk 0's forward path (as k_chunk32)
      const int cfw = s < p ? tf + bwR + latR : 0;
      int Pp = cfw;
      for (int d = 1; d < 32; d <<= 1) { const int t2 = __shfl_up_sync(FMASK, Pp, d); if (s >= d) Pp += t2; }
      Pp -= cfw;
      int xq = (s < p ? tag : 0) - Pp;
      for (int d = 1; d < 32; d <<= 1) { const int t2 = __shfl_up_sync(FMASK, xq, d); if (s >= d) xq = cmax(xq, t2); }
      const int busy = kChunks * m * (tf + td + tw);
      for (int rr = s; rr < A.stage_stride; rr += 32) {
        const int4 v = (rr == s && s < p) ? make_int4(Pp + xq, clk, busy, peak) : make_int4(0, 0, 0, 0);
        *reinterpret_cast<int4*>(A.stage_stats + (item * A.stage_stride + rr) * 4) = v;
      }
    }
    __syncwarp();
  }
}

namespace {
const void* chunkf_fn(int pat, bool tl) {
  switch (pat) {
    case CP_PATTERN_UD: return tl ? (const void*)k_chunk32f<CP_PATTERN_UD, true> : (const void*)k_chunk32f<CP_PATTERN_UD, false>;
    case CP_PATTERN_WAVE: return tl ? (const void*)k_chunk32f<CP_PATTERN_WAVE, true> : (const void*)k_chunk32f<CP_PATTERN_WAVE, false>;
    default: return tl ? (const void*)k_chunk32f<CP_PATTERN_LOOP, true> : (const void*)k_chunk32f<CP_PATTERN_LOOP, false>;
  }
}
}  // namespace

int launch_chunkf(int pattern, bool timeline, const Args& a, int blocks, int threads, size_t smem, void* stream) {
  const void* fn = chunkf_fn(pattern, timeline);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return (int)e;
  }
  void* params[] = {(void*)&a};
  return (int)cudaLaunchKernel(fn, dim3(blocks), dim3(threads), params, smem, (cudaStream_t)stream);
}

int chunkf_blocks_per_sm(int pattern, int threads, size_t smem, bool timeline) {
  const void* fn = chunkf_fn(pattern, timeline);
  if (smem > 48 * 1024) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, threads, smem) != cudaSuccess) return 1;
  return n > 0 ? n : 1;
}

}  // namespace cpk
