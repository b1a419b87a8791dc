// chunk_grid.cu -- the sweep's static candidates (GPipe / 1F1B / ZB-H1 of cp_sweep_shard) on the
// k_chunk32f round (chunk_fast.cu): k_chunk32f_grid takes (point, candidate) tasks from
// a counter, synthesizes each lane's instance from the grid (grid_synth.cuh), fetches the candidate's
// plan by TMA from a per-call library of [kind][n_pp][n_mb] plans (k_plan_library, plan_code), and
// folds the makespan into the point's argmin key.
//
// It is the UD round of k_chunk32f with plain count bytes: c = {F, D, 128 - (#D - #W), 0x80}, so
// n_mb up to 255 fits (GPipe / 1F1B have no W and ZB-H1 owes at most s + 1 W blocks, so the deficit
// byte cannot wrap).  It is a separate kernel rather than a template branch of k_chunk32f because
// sharing the source changed the bench kernel's register allocation and instruction schedule
// (measured −5% on config 4).
#include <cuda_runtime.h>
#include <stdint.h>

#include "engine.h"
#include "grid_synth.cuh"
#include "plan_codes.cuh"
#include "ptx.cuh"

namespace cpk {

namespace {
constexpr unsigned GMASK = 0xffffffffu;
constexpr int32_t GRID_INF = 1 << 30;
__device__ __forceinline__ int gmax2(int a, int b) { return a > b ? a : b; }
__device__ __forceinline__ int gmadd2(int g, int d, int x) {   // x + g*d on the FMA pipe
  int r;
  asm("mad.lo.s32 %0, %1, %2, %3;" : "=r"(r) : "r"(g), "r"(d), "r"(x));
  return r;
}
__device__ __forceinline__ uint32_t gprmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
  return d;
}
// 8 selector bytes (source byte index in the top nibble, 0xF below) -> two registers
__device__ __forceinline__ void gpack_sel(const int (&ix)[8], uint32_t& lo, uint32_t& hi) {
  lo = hi = 0;
#pragma unroll
  for (int x = 0; x < 4; ++x) {
    lo |= (uint32_t)((ix[x] << 4) | 0xF) << (8 * x);
    hi |= (uint32_t)((ix[x + 4] << 4) | 0xF) << (8 * x);
  }
}
}  // namespace

// The static-candidate plans: one per (kind in GPipe / 1F1B / ZB-H1, n_pp, n_mb) block of the grid,
// in the simulate layout [words][32 stages]; lane = stage, entries from plan_code (plan_codes.cuh).
__global__ void k_plan_library(PlanLibDims d, uint32_t* lib) {
  const int b = blockIdx.x, s = threadIdx.x;
  const int nblk = d.n_pp * d.n_mb;
  const int kind = b / nblk == 0 ? CP_PLAN_GPIPE : (b / nblk == 1 ? CP_PLAN_1F1B : CP_PLAN_ZBH1);
  const int p = d.pp[(b % nblk) / d.n_mb], m = d.mb[(b % nblk) % d.n_mb];
  const int len = s < p ? plan_row_len(kind, m) : 0;
  uint32_t* out = lib + (long long)b * d.words * 32 + s;
  for (int k = 0; k < d.words; ++k) {
    uint32_t w = 0;
    for (int e = 0; e < 16 && 16 * k + e < len; ++e) w |= (uint32_t)plan_code(kind, s, p, m, 16 * k + e) << (2 * e);
    out[k * 32] = w;
  }
}

// Per-warp table rows of one task (rings F (0) and D (1); F goes right, D / B left; entry x = code,
// rows 4..7 repeat 0..3): T0 {duration, memory delta, link bw, latency (-1: sends nothing)}, T1 {input
// ring, message ring, link clock, count increment}; F +1; B: D +1; D: D +1 and byte 2 -1; W: byte 2 +1.
__device__ __forceinline__ void grid_tables(int s, int p, int R, const ChunkFLayout& Ly, int4* T0, int4* T1, int tf,
                                            int td, int tw, int mf, int md, int mw, int latR, int bwR, int latL,
                                            int bwL) {
  const bool live = s < p, first = s == 0, last = s == p - 1;
  const int RB = R * 128, col = 4 * s;
  const int rF = Ly.rings * 4 + col, rD = rF + RB;
  const int z = Ly.zero * 4 + col, lkR = Ly.lk * 4 + col, lkL = lkR + 128;
  const auto L = [&](int lat) { return live ? lat : -1; };
  for (int h = 0; h < 256; h += 128) {
    T0[h] = make_int4(tf, mf, bwR, L(last ? -1 : latR));
    T1[h] = make_int4(rF, rF + 4, lkR, 1);
    T0[h + 32] = make_int4(td + tw, md + mw, bwL, L(first ? -1 : latL));
    T1[h + 32] = make_int4(rD, rD - 4, lkL, 1 << 8);
    T0[h + 64] = make_int4(td, md, bwL, L(first ? -1 : latL));
    T1[h + 64] = make_int4(rD, rD - 4, lkL, (1 << 8) - (1 << 16));
    T0[h + 96] = make_int4(tw, mw, 0, -1);
    T1[h + 96] = make_int4(z, z, lkR, 1 << 16);
  }
}

__global__ void __launch_bounds__(kChunkFThreads, kChunkFMinBlocks) k_chunk32f_grid(const __grid_constant__ Args A) {
  extern __shared__ __align__(128) int32_t smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, s = lane;
  const int R = A.ring_slots, Rm = R - 1, PW = A.words;
  const ChunkFLayout Ly = chunkf_layout(R, PW, false, 2);
  const int wbase = wib * Ly.per_warp, tbase = wbase + Ly.tab;
  const unsigned sb = smem_u32(smem), wb = sb + 4u * (unsigned)wbase;
  uint64_t* const bar = reinterpret_cast<uint64_t*>(smem + wbase + Ly.bars);
  int32_t* const plan = smem + wbase + Ly.plan;
  int4* const T0 = reinterpret_cast<int4*>(smem + tbase) + lane;
  int4* const T1 = T0 + 256;

  for (int k = lane; k < (2 * R + Ly.zrows) * 32; k += 32) smem[wbase + Ly.rings + k] = 0;   // rings, zero block
  if (lane == 0) mbar_init(bar);
  __syncwarp();
  uint32_t phase = 0;
  const uint32_t opq = (uint32_t)A.words >> 30;    // 0 at run time, opaque to the compiler (chunk_fast.cu)
  const uint32_t fifteen = 15u | (opq << 20);

  const unsigned smask = A.grid.cand_mask & ((1u << CP_N_CAND) - 1u);
  const SweepSet sset{A.pt_lo, A.pt_hi, A.blk_inner, A.own_lo, A.own_hi};
  const long long inner = (long long)A.grid.n_lat * A.grid.n_bw * A.grid.n_mem * A.grid.n_dp;
  const long long nblk = (long long)A.grid.n_pp_n * A.grid.n_mb_n;
  int cand = 0;
  // tasks from the counter, the next index fetched one task ahead
  long long t0 = 0, tnx = 0;
  if (lane == 0) t0 = (long long)atomicAdd(A.sweep_counter, 1ull);
  for (long long item = sweep_task(smask, sset, __shfl_sync(GMASK, t0, 0), cand); item >= 0;
       item = sweep_task(smask, sset, __shfl_sync(GMASK, tnx, 0), cand)) {
    if (lane == 0) tnx = (long long)atomicAdd(A.sweep_counter, 1ull);
    if (lane == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // last task's plan writes -> the copy
      const long long pi = (cand == CP_PLAN_GPIPE ? 0 : (cand == CP_PLAN_1F1B ? 1 : 2)) * nblk + item / inner;
      tma_load_1d(plan, A.ops + pi * PW * 32, (uint32_t)PW * 128u, bar);
    }
    const GridLane g = grid_lane(A.grid, item, s);
    const int p = g.p, m = g.m;
    int tf = 0, td = 0, tw = 0, mf = 0, md = 0, mw = 0, mlim = 0, tdp = 0, tag = 0;
    int latR = 0, bwR = 0, latL = 0, bwL = 0, plen = 0;
    if (s < p) {
      tf = g.tf; td = g.td; tw = g.tw; mf = g.mf; md = g.md; mw = g.mw; mlim = g.mlim;
      tdp = g.tdp; tag = g.zero1 ? g.tag : 0;
      latR = g.latF; bwR = g.bwF; latL = g.latB; bwL = g.bwB;
      plen = plan_row_len(cand, m);
    }
    // statically infeasible candidates are skipped, as in the engine (GPipe peak m m_f, 1F1B peak
    // min(p - s, m) m_f over M_L, Z5; cand_ms stays -1, no key); ZB-H1 is evaluated and excluded if
    // over M_L; the int32 horizon guard (Q21) marks the point unevaluated (KEY_OVER)
    const bool skip = s < p && (cand == CP_PLAN_GPIPE ? (long long)m * mf > mlim
                                                        : (cand == CP_PLAN_1F1B ? (long long)min(p - s, m) * mf > mlim : false));
    long long u = s < p ? (long long)m * ((long long)tf + td + tw) + tag + tdp + (long long)m * ((long long)latR + bwR + latL + bwL) : 0;
    for (int d = 16; d > 0; d >>= 1) u += __shfl_xor_sync(GMASK, u, d);
    mbar_wait(bar, phase);
    phase ^= 1u;
    if (__any_sync(GMASK, skip) || m > 255) { __syncwarp(); continue; }
    if (u >= (long long)GRID_INF || p > CP_MAX_STAGES) {
      if (lane == 0) atomicMin(A.keys + item, KEY_OVER);
      __syncwarp();
      continue;
    }
    // stage the row: pad past the end with D (never ready at the end), pre-rotate by 4 bits
    for (int k = 0; k <= PW; ++k) {
      uint32_t w = (uint32_t)plan[(k << 5) + lane];
      const int n = s < p ? min(max(plen - 16 * k, 0), 16) : 0;
      const uint32_t keep = n == 16 ? 0xffffffffu : ((1u << (2 * n)) - 1u);
      w = (w & keep) | (0xaaaaaaaau & ~keep);
      plan[(k << 5) + lane] = (int32_t)((w << 4) | (w >> 28));
    }
    grid_tables(lane, p, R, Ly, T0, T1, tf, td, tw, mf, md, mw, latR, bwR, latL, bwL);
    if (p < 32)                                     // the last stage's D input column: no producer
      for (int k = lane; k < R; k += 32) smem[wbase + Ly.rings + (k << 5) + (p - 1) + R * 32] = 0;
    // selectors (plain count bytes): "no producer" and the W tests take the sign of byte 3 (0x80); a
    // block without a consumer compares with its own count (stage 0 / the last stage see their own
    // counts in the left / right view), so n - Y = 0
    const bool first = s == 0, last = s == p - 1;
    uint32_t kxl, kxh, kyl, kyh, knl, knh;
    {
      const int tx[8] = {first ? 11 : 0, last ? 4 : 5, last ? 4 : 5, 11, first ? 11 : 0, last ? 4 : 5, last ? 4 : 5, 11};
      const int ty[8] = {4, 1, 1, 11, 4, 1, 1, 11};
      const int tn[8] = {0, 1, 1, 10, 0, 1, 1, 10};
      gpack_sel(tx, kxl, kxh);
      gpack_sel(ty, kyl, kyh);
      gpack_sel(tn, knl, knh);
      kyl ^= opq; kyh ^= opq; knl ^= opq; knh ^= opq;
    }
    const int srcL = first ? s : (s < p ? s - 1 : s);
    const int srcR = last ? s : (s < p ? s + 1 : s);
    __syncwarp();

    uint32_t c = 0x80800000u;
    int clk = tag, mem = 0, peak = 0, pos2 = 0, lkR = 0, lkL = 0;
    const unsigned tab0m = sb + 4u * (unsigned)tbase + 16u * (unsigned)lane - 480u;   // T0[x][lane] - 15*32
    const unsigned iPb = wb + 4u * (unsigned)(Ly.plan + lane);
    const int R24 = R << 24, Rm7 = Rm << 7;
    uint32_t wv;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(wv) : "r"(iPb));
    for (;;) {
      uint32_t Lv, Rv;
      asm volatile("shfl.sync.idx.b32 %0, %2, %3, 0x1f, 0xffffffff;\n\t"
                   "shfl.sync.idx.b32 %1, %2, %4, 0x1f, 0xffffffff;"
                   : "=r"(Lv), "=r"(Rv) : "r"(c), "r"(srcL), "r"(srcR));
      uint32_t r, x4;
      asm("shf.r.wrap.b32 %0, %1, %1, %2;" : "=r"(r) : "r"(wv), "r"(pos2));
      asm("lop3.b32 %0, %1, 0x30, %2, 0xEA;" : "=r"(x4) : "r"(r), "r"(fifteen));   // code << 4 | 15
      const unsigned ta = tab0m + (x4 << 5);
      int4 t0, t1;
      asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(t0.x), "=r"(t0.y), "=r"(t0.z), "=r"(t0.w) : "r"(ta));
      asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4+4096];" : "=r"(t1.x), "=r"(t1.y), "=r"(t1.z), "=r"(t1.w) : "r"(ta));
      const uint32_t sX = gprmt(kxl, kxh, x4), sY = gprmt(kyl, kyh, x4), sN = gprmt(knl, knh, x4);
      const uint32_t X = gprmt(Lv, Rv, sX), Y = gprmt(Lv, Rv, sY), n = gprmt(c, c, sN);
      const bool go = (X > n) & ((int)(n - Y) < R24);
      const unsigned slot = (n >> 17) & (unsigned)Rm7;
      const bool isF = (x4 & 0xF0u) == 0u;
      const unsigned ia = wb + (unsigned)t1.x + slot, oa = wb + (unsigned)t1.y + slot;
      int arr;
      asm volatile("ld.shared.b32 %0, [%1];" : "=r"(arr) : "r"(ia));
      const int lk = isF ? lkR : lkL;
      const int start = gmax2(clk, arr);
      const int end = start + t0.x;
      const int nl = gmax2(end, lk) + t0.z;          // FIFO link clock (App. X1)
      const bool snd = go & (t0.w >= 0);
      if (snd) asm volatile("st.shared.b32 [%0], %1;" :: "r"(oa), "r"(nl + t0.w) : "memory");
      lkR = (snd & isF) ? nl : lkR;
      lkL = (snd & !isF) ? nl : lkL;
      const int gi = go ? 1 : 0;
      clk = gmadd2(gi, end - clk, clk);
      mem = gmadd2(gi, t0.y, mem);
      peak = gmax2(peak, mem);
      c = (uint32_t)gmadd2(gi, t1.w, (int)c);
      pos2 = gmadd2(gi, 2, pos2);
      unsigned wa;
      asm("mad.lo.u32 %0, %1, 4, %2;" : "=r"(wa) : "r"((unsigned)pos2 & ~31u), "r"(iPb));
      asm volatile("ld.shared.b32 %0, [%1];" : "=r"(wv) : "r"(wa));
      __syncwarp();
      if (!__any_sync(GMASK, go)) break;
    }
    // the static families cannot stall on 8-slot rings (a producer leads its consumer by at most two
    // messages): an incomplete row is the engine's "never happens" path, point unevaluated
    const bool rowok = s >= p || ((pos2 >> 1) == plen && c == 0x80800000u + 0x0101u * (uint32_t)m);
    if (!__all_sync(GMASK, rowok)) {
      if (lane == 0) atomicMin(A.keys + item, KEY_OVER);
      __syncwarp();
      continue;
    }
    const bool feasible = !__any_sync(GMASK, s < p && peak > mlim);
    int ms = s < p ? gmax2(clk + tdp, tag) : 0;
    for (int d = 16; d > 0; d >>= 1) ms = gmax2(ms, __shfl_xor_sync(GMASK, ms, d));
    if (lane == 0 && feasible) {
      if (A.cand_ms) A.cand_ms[item * CP_N_CAND + cand] = ms;
      atomicMin(A.keys + item, ((unsigned long long)ms << 8) | (unsigned)cand);
    }
    __syncwarp();
  }
}

int launch_plan_library(const PlanLibDims& d, uint32_t* lib, void* stream) {
  k_plan_library<<<3 * d.n_pp * d.n_mb, 32, 0, (cudaStream_t)stream>>>(d, lib);
  return (int)cudaGetLastError();
}

int launch_chunkf_grid(const Args& a, int blocks, int threads, size_t smem, void* stream) {
  const void* fn = (const void*)k_chunk32f_grid;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return (int)e;
  }
  void* params[] = {(void*)&a};
  return (int)cudaLaunchKernel(fn, dim3(blocks), dim3(threads), params, smem, (cudaStream_t)stream);
}

int chunkf_grid_blocks_per_sm(int threads, size_t smem) {
  const void* fn = (const void*)k_chunk32f_grid;
  if (smem > 48 * 1024) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, threads, smem) != cudaSuccess) return 1;
  return n > 0 ? n : 1;
}

}  // namespace cpk
