// int_peak.cu -- integer-pipe throughput microbenchmark for the ALU roofline (SURVEY.md §8(d):
// "measure the integer throughput per SM before quoting an ALU fraction").
//
// Each thread runs 8 independent dependency chains of one instruction class for `iters` steps,
// so issue is limited by the pipe, not by latency. Classes:
//   alu  : integer max / add / xor mix (VIMNMX, IADD3, LOP3 -- the ALU pipe)
//   fma  : integer multiply-add (IMAD -- the FMA pipe)
//   mix  : one alu and one fma chain step interleaved (both pipes)
// Output: one JSON line per class with lane-ops/s, warp-instr/clk/SM and the clock used.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o int_peak int_peak.cu
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdint.h>

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

template <int KIND>
__global__ void k_int(int iters, int seed, int* out, unsigned long long* clk) {
  // block 0 / thread 0 records (SM cycles, global ns) at entry and exit: the SM clock actually seen
  const bool rec = blockIdx.x == 0 && threadIdx.x == 0;
  if (rec) { clk[0] = clock64(); clk[1] = gtimer(); }
  int a0 = threadIdx.x ^ seed, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const int k = seed | 1, j = seed >> 3;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (KIND == 0) {        // ALU pipe: max, add, xor (3 ops per chain per step)
        asm volatile(
            "max.s32 %0, %0, %8;\n\tmax.s32 %1, %1, %8;\n\tmax.s32 %2, %2, %8;\n\tmax.s32 %3, %3, %8;\n\t"
            "max.s32 %4, %4, %8;\n\tmax.s32 %5, %5, %8;\n\tmax.s32 %6, %6, %8;\n\tmax.s32 %7, %7, %8;\n\t"
            "add.s32 %0, %0, %9;\n\tadd.s32 %1, %1, %9;\n\tadd.s32 %2, %2, %9;\n\tadd.s32 %3, %3, %9;\n\t"
            "add.s32 %4, %4, %9;\n\tadd.s32 %5, %5, %9;\n\tadd.s32 %6, %6, %9;\n\tadd.s32 %7, %7, %9;\n\t"
            "xor.b32 %0, %0, %8;\n\txor.b32 %1, %1, %8;\n\txor.b32 %2, %2, %8;\n\txor.b32 %3, %3, %8;\n\t"
            "xor.b32 %4, %4, %8;\n\txor.b32 %5, %5, %8;\n\txor.b32 %6, %6, %8;\n\txor.b32 %7, %7, %8;"
            : "+r"(a0), "+r"(a1), "+r"(a2), "+r"(a3), "+r"(a4), "+r"(a5), "+r"(a6), "+r"(a7)
            : "r"(k), "r"(j));
      } else if (KIND == 1) { // FMA pipe: integer multiply-add (3 per chain per step)
        asm volatile(
            "mad.lo.s32 %0, %0, %8, %9;\n\tmad.lo.s32 %1, %1, %8, %9;\n\tmad.lo.s32 %2, %2, %8, %9;\n\t"
            "mad.lo.s32 %3, %3, %8, %9;\n\tmad.lo.s32 %4, %4, %8, %9;\n\tmad.lo.s32 %5, %5, %8, %9;\n\t"
            "mad.lo.s32 %6, %6, %8, %9;\n\tmad.lo.s32 %7, %7, %8, %9;\n\t"
            "mad.lo.s32 %0, %0, %8, %9;\n\tmad.lo.s32 %1, %1, %8, %9;\n\tmad.lo.s32 %2, %2, %8, %9;\n\t"
            "mad.lo.s32 %3, %3, %8, %9;\n\tmad.lo.s32 %4, %4, %8, %9;\n\tmad.lo.s32 %5, %5, %8, %9;\n\t"
            "mad.lo.s32 %6, %6, %8, %9;\n\tmad.lo.s32 %7, %7, %8, %9;\n\t"
            "mad.lo.s32 %0, %0, %8, %9;\n\tmad.lo.s32 %1, %1, %8, %9;\n\tmad.lo.s32 %2, %2, %8, %9;\n\t"
            "mad.lo.s32 %3, %3, %8, %9;\n\tmad.lo.s32 %4, %4, %8, %9;\n\tmad.lo.s32 %5, %5, %8, %9;\n\t"
            "mad.lo.s32 %6, %6, %8, %9;\n\tmad.lo.s32 %7, %7, %8, %9;"
            : "+r"(a0), "+r"(a1), "+r"(a2), "+r"(a3), "+r"(a4), "+r"(a5), "+r"(a6), "+r"(a7)
            : "r"(k), "r"(j));
      } else {                // both pipes: chains 0-3 on ALU, 4-7 on FMA
        asm volatile(
            "max.s32 %0, %0, %8;\n\tmax.s32 %1, %1, %8;\n\tmax.s32 %2, %2, %8;\n\tmax.s32 %3, %3, %8;\n\t"
            "mad.lo.s32 %4, %4, %8, %9;\n\tmad.lo.s32 %5, %5, %8, %9;\n\tmad.lo.s32 %6, %6, %8, %9;\n\t"
            "mad.lo.s32 %7, %7, %8, %9;\n\t"
            "add.s32 %0, %0, %9;\n\tadd.s32 %1, %1, %9;\n\tadd.s32 %2, %2, %9;\n\tadd.s32 %3, %3, %9;\n\t"
            "mad.lo.s32 %4, %4, %8, %9;\n\tmad.lo.s32 %5, %5, %8, %9;\n\tmad.lo.s32 %6, %6, %8, %9;\n\t"
            "mad.lo.s32 %7, %7, %8, %9;\n\t"
            "xor.b32 %0, %0, %8;\n\txor.b32 %1, %1, %8;\n\txor.b32 %2, %2, %8;\n\txor.b32 %3, %3, %8;\n\t"
            "mad.lo.s32 %4, %4, %8, %9;\n\tmad.lo.s32 %5, %5, %8, %9;\n\tmad.lo.s32 %6, %6, %8, %9;\n\t"
            "mad.lo.s32 %7, %7, %8, %9;"
            : "+r"(a0), "+r"(a1), "+r"(a2), "+r"(a3), "+r"(a4), "+r"(a5), "+r"(a6), "+r"(a7)
            : "r"(k), "r"(j));
      }
    }
  }
  const int r = a0 ^ a1 ^ a2 ^ a3 ^ a4 ^ a5 ^ a6 ^ a7;
  if (r == 0x7fffffff) out[threadIdx.x] = r;   // keep the chains live
  if (rec) { clk[2] = clock64(); clk[3] = gtimer(); }
}

int main() {
  int dev = 0, sms = 0, clk_khz = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  int* out = nullptr;
  unsigned long long* clk = nullptr;
  cudaMalloc(&out, 1024 * sizeof(int));
  cudaMalloc(&clk, 4 * sizeof(unsigned long long));
  const int threads = 256, blocks = sms * 8, iters = 4096;
  const double ops_per_thread = (double)iters * 4 * 24;   // 24 instructions per asm block
  const char* names[3] = {"alu", "fma", "mix"};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int kind = 0; kind < 3; ++kind) {
    float best = 1e30f;
    double mhz_best = 0;
    // 200 launches (about 1 s per class, long enough for the nvidia-smi clock sampler of
    // tools/int_peak.sh); the best launch and the SM clock block 0 saw during it
    for (int rep = 0; rep < 200; ++rep) {
      cudaEventRecord(e0);
      if (kind == 0) k_int<0><<<blocks, threads>>>(iters, rep, out, clk);
      else if (kind == 1) k_int<1><<<blocks, threads>>>(iters, rep, out, clk);
      else k_int<2><<<blocks, threads>>>(iters, rep, out, clk);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      unsigned long long c[4];
      cudaMemcpy(c, clk, sizeof(c), cudaMemcpyDeviceToHost);
      if (rep > 0 && ms < best) {
        best = ms;
        mhz_best = (double)(c[2] - c[0]) / (double)(c[3] - c[1]) * 1e3;   // cycles per ns -> MHz
      }
    }
    const double lane_ops = ops_per_thread * threads * blocks;
    const double rate = lane_ops / (best / 1e3);                         // lane-ops/s
    const double warp_instr_per_clk_sm = rate / 32.0 / (sms * (clk_khz * 1e3));
    const double per_clk_observed = rate / 32.0 / (sms * mhz_best * 1e6);
    printf("{\"class\": \"%s\", \"lane_ops_per_s\": %.6e, \"warp_instr_per_clk_per_sm\": %.4f, "
           "\"sm_count\": %d, \"clock_mhz_attr\": %.1f, \"sm_mhz_observed\": %.1f, "
           "\"warp_instr_per_observed_clk_per_sm\": %.4f, \"ms\": %.4f}\n",
           names[kind], rate, warp_instr_per_clk_sm, sms, clk_khz / 1e3, mhz_best, per_clk_observed, best);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { fprintf(stderr, "cuda error %s\n", cudaGetErrorString(e)); return 1; }
  return 0;
}
