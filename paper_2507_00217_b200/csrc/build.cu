// build.cu -- cp_build_static: static plans (GPipe, 1F1B, ZB-H1 packed 2 bits per entry, 16 per
// word; IV1F1B and ZB-V 4 bits, 8 per word) in the [item][word][stage_stride] layout cp_simulate
// reads (include/crosspipe.h).
//
// One thread per (item, stage row): it walks its row with plan_code() (plan_codes.cuh), packs
// the words in a register and stores each as it fills, so consecutive threads (rows) of an item
// write consecutive addresses.  Every word and every row is written (zeros past the row's
// entries and for rows >= p), so the output is fully defined.
#include <cuda_runtime.h>
#include <stdint.h>

#include "engine.h"
#include "plan_codes.cuh"

namespace cpk {

__global__ void __launch_bounds__(256) k_build_static(int kind, const cp_inst_v1* __restrict__ inst, int n_inst,
                                                      const int32_t* __restrict__ inst_of, long long n,
                                                      int stride, int words, uint32_t* __restrict__ ops,
                                                      uint16_t* __restrict__ len) {
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long total = n * stride;
  for (long long t = tid; t < total; t += (long long)gridDim.x * blockDim.x) {
    const long long item = t / stride;
    const int r = (int)(t - item * stride);
    const long long ii = inst_of ? (long long)inst_of[item] : (n_inst == 1 ? 0 : item);
    const int p = inst[ii].n_pp, m = inst[ii].n_mb;
    const int eb = plan_entry_bits(kind), per = 32 / eb;          // 16 or 8 entries per word
    int L = (r < p && m >= 1 && p <= stride) ? plan_row_len(kind, m) : 0;
    if (L > per * words || (kind == CP_PLAN_IV1F1B && m % p != 0)) L = 0;   // does not fit: all-zero rows
    uint32_t* row = ops + item * (long long)words * stride + r;
    uint32_t wv = 0;
    int k = 0;
    for (int pos = 0; pos < L; ++pos) {
      wv |= (uint32_t)plan_code(kind, r, p, m, pos) << ((pos % per) * eb);
      if (pos % per == per - 1) { row[(long long)k * stride] = wv; wv = 0; ++k; }
    }
    if (L % per) { row[(long long)k * stride] = wv; ++k; }
    for (; k < words; ++k) row[(long long)k * stride] = 0u;
    len[item * stride + r] = (uint16_t)L;
  }
}

// ZB-V (reading Q35): the per-stage order of a unit-time list schedule of the Wave data flow
// (Q32).  One warp per item, lane = stage, one round per tick: the neighbours' counts at the start
// of the round arrive by shuffle (F0 and D1 flow down from lane s-1, F1 and D0 up from lane s+1),
// each lane takes at most one block, appends its 4-bit code (type | chunk << 2) to a register word
// and stores the word when 8 entries have filled it.  Items that do not fit (p > 32 or > stride,
// 6m > 8*words) get all-zero rows, as do rows >= p.
__global__ void __launch_bounds__(128) k_build_zbv(const cp_inst_v1* __restrict__ inst, int n_inst,
                                                   const int32_t* __restrict__ inst_of, long long n, int stride,
                                                   int words, uint32_t* __restrict__ ops, uint16_t* __restrict__ len) {
  constexpr unsigned FULL = 0xffffffffu;
  const int s = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long item = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); item < n; item += warps) {
    const long long ii = inst_of ? (long long)inst_of[item] : (n_inst == 1 ? 0 : item);
    const int p = inst[ii].n_pp, m = inst[ii].n_mb;
    const bool fits = p >= 1 && m >= 1 && p <= 32 && p <= stride && 6 * m <= 8 * words;
    const bool act = fits && s < p;
    uint32_t* row = ops + item * (long long)words * stride;
    int nF0 = 0, nF1 = 0, nD0 = 0, nD1 = 0, nW0 = 0, nW1 = 0, cnt = 0, k = 0;
    uint32_t wv = 0;
    const int L = act ? 6 * m : 0;
    while (__any_sync(FULL, cnt < L)) {
      const int upF0 = __shfl_up_sync(FULL, nF0, 1), upD1 = __shfl_up_sync(FULL, nD1, 1);
      const int dnF1 = __shfl_down_sync(FULL, nF1, 1), dnD0 = __shfl_down_sync(FULL, nD0, 1);
      const bool full = nF0 + nF1 - nW0 - nW1 >= 2 * p;
      const bool f0 = !full && nF0 < m && (s == 0 || upF0 > nF0);
      const bool f1 = !full && nF1 < m && (s == p - 1 ? nF0 > nF1 : dnF1 > nF1);
      const bool d1 = nD1 < m && (s == 0 ? nF1 > nD1 : upD1 > nD1);
      const bool d0 = nD0 < m && (s == p - 1 ? nD1 > nD0 : dnD0 > nD0);
      const bool w0 = nW0 < nD0, w1 = nW1 < nD1;
      int e = -1;
      if ((w0 || w1) && (full || !(f0 || f1 || d0 || d1))) e = w0 ? (int)CP_OP_W : ((int)CP_OP_W | 4);
      else if (f1) e = (int)CP_OP_F | 4;
      else if (f0) e = (int)CP_OP_F;
      else if (d0) e = (int)CP_OP_D;
      else if (d1) e = (int)CP_OP_D | 4;
      if (cnt < L && e >= 0) {
        nF0 += e == (int)CP_OP_F;       nF1 += e == ((int)CP_OP_F | 4);
        nD0 += e == (int)CP_OP_D;       nD1 += e == ((int)CP_OP_D | 4);
        nW0 += e == (int)CP_OP_W;       nW1 += e == ((int)CP_OP_W | 4);
        wv |= (uint32_t)e << (4 * (cnt & 7));
        if ((++cnt & 7) == 0) { row[(long long)k * stride + s] = wv; wv = 0; ++k; }
      }
    }
    for (int r = s; r < stride; r += 32) {
      int kk = r == s ? k : 0;
      if (r == s && (cnt & 7)) { row[(long long)kk * stride + r] = wv; ++kk; }
      for (; kk < words; ++kk) row[(long long)kk * stride + r] = 0u;
      len[item * stride + r] = (uint16_t)(r == s ? L : 0);
    }
  }
}

int launch_build_static(int kind, const cp_inst_v1* inst, int n_inst, const int32_t* inst_of, long long n, int stride,
                        int words, uint32_t* ops, uint16_t* len, void* stream) {
  const long long total = n * stride;
  if (total <= 0) return 0;
  if (kind == CP_PLAN_ZBV) {
    const long long want = (n + 3) / 4;
    const int blocks = (int)(want < 148LL * 16 ? want : 148LL * 16);
    k_build_zbv<<<blocks, 128, 0, (cudaStream_t)stream>>>(inst, n_inst, inst_of, n, stride, words, ops, len);
    return (int)cudaGetLastError();
  }
  const int threads = 256;
  const long long want = (total + threads - 1) / threads;
  const int blocks = (int)(want < 148LL * 32 ? want : 148LL * 32);
  k_build_static<<<blocks, threads, 0, (cudaStream_t)stream>>>(kind, inst, n_inst, inst_of, n, stride, words, ops, len);
  return (int)cudaGetLastError();
}

}  // namespace cpk
