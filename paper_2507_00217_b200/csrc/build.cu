// build.cu -- cp_build_static: static plans (GPipe, 1F1B, ZB-H1) packed 2 bits per entry, 16 per
// word, in the [item][word][stage_stride] layout cp_simulate reads (include/crosspipe.h).
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

int launch_build_static(int kind, const cp_inst_v1* inst, int n_inst, const int32_t* inst_of, long long n, int stride,
                        int words, uint32_t* ops, uint16_t* len, void* stream) {
  const long long total = n * stride;
  if (total <= 0) return 0;
  const int threads = 256;
  const long long want = (total + threads - 1) / threads;
  const int blocks = (int)(want < 148LL * 32 ? want : 148LL * 32);
  k_build_static<<<blocks, threads, 0, (cudaStream_t)stream>>>(kind, inst, n_inst, inst_of, n, stride, words, ops, len);
  return (int)cudaGetLastError();
}

}  // namespace cpk
