// exact.cu -- cp_exact: batched exhaustive search for the makespan-optimal split plan (n_sub = 1)
// of tiny instances (the stand-in for the paper's CO solver, §4.1
// :322-360: validity set = per-stage order of F/D/W respecting microbatch order per type, D_j after
// F_j, W_j after D_j, and the memory capacity; objective = makespan).
//
// 1. k_exact_sets: one thread per (instance, stage) enumerates the stage's valid sequences by DFS,
//    trying F, then D, then W at every position (lexicographic in that order), a sequence packed 2
//    bits per entry into a uint64 (3m <= 24 entries).
// 2. k_exact_prep: one thread per instance validates it, multiplies the set sizes into the product
//    size and lays out chunks of kExactChunk consecutive product indices; one thread then prefix-
//    sums the chunk counts over the batch.
// 3. k_exact_eval: persistent grid-stride over all chunks of all instances; a thread walks its
//    chunk's product indices as an odometer (last stage fastest) and simulates every plan
//    sequentially (§3.5 start-time rule, FIFO link windows = first fit under UD, App. X1; ZeRO-1
//    gate; DP tail).  Whenever the stages 0..p-2 change, the prefix is first simulated with the
//    last stage relaxed (instantaneous, order-free: a lower bound for every plan of the prefix) and
//    the prefix's whole run is skipped if that bound exceeds the incumbent.  A plan is abandoned
//    once a stage's clock + its remaining work + its DP tail exceeds the instance's best makespan
//    so far (strictly, so equal-makespan plans survive), and
//    the finished ones race on a 64-bit atomicMin of (makespan << b | product index), b = the bits of
//    the instance's product size: the result is the smallest-index optimum, independent of thread
//    timing.
// 4. k_exact_finish: decodes each instance's key into its plan (packed rows) and makespan.
#include <cuda_runtime.h>
#include <stdint.h>

#include "engine.h"

namespace cpk {

constexpr int kExactChunk = 64;
constexpr unsigned long long kExactNone = ~0ull;

__global__ void __launch_bounds__(128) k_exact_sets(const cp_inst_v1* __restrict__ inst, int n, int cap,
                                                    unsigned long long* __restrict__ seqs, int32_t* __restrict__ cnt) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)n * kExactMaxP) return;
  const int item = (int)(t / kExactMaxP), s = (int)(t % kExactMaxP);
  const cp_inst_v1* I = inst + item;
  const int p = I->n_pp, m = I->n_mb;
  if (s >= p || p > kExactMaxP || m < 1 || m > kExactMaxM) { cnt[t] = 0; return; }
  const int L = 3 * m;
  const long long mf = I->m_f[s], md = I->m_d[s], mw = I->m_w[s], mlim = I->m_lim[s];
  unsigned long long* out = seqs + t * (long long)cap;
  int ch[3 * kExactMaxM];
  int nF = 0, nD = 0, nW = 0, k = 0, count = 0;
  long long mem = 0;
  unsigned long long cur = 0;
  ch[0] = -1;
  while (true) {
    if (k == L) {
      if (count < cap) out[count] = cur;
      if (++count > cap) break;                                 // too many: reported as overflow
      --k;
    } else {
      int c = ch[k] + 1;
      for (; c < 3; ++c)
        if ((c == 0 && nF < m && mem + mf <= mlim) || (c == 1 && nD < nF) || (c == 2 && nW < nD)) break;
      if (c < 3) {
        ch[k] = c;
        if (c == 0) { ++nF; mem += mf; } else if (c == 1) { ++nD; mem += md; } else { ++nW; mem += mw; }
        cur |= (unsigned long long)(c == 0 ? CP_OP_F : (c == 1 ? CP_OP_D : CP_OP_W)) << (2 * k);
        if (++k < L) ch[k] = -1;
        continue;
      }
      --k;
    }
    if (k < 0) break;
    const int c = ch[k];                                        // undo level k, then try its next choice
    if (c == 0) { --nF; mem -= mf; } else if (c == 1) { --nD; mem -= md; } else { --nW; mem -= mw; }
    cur &= ~(3ull << (2 * k));
  }
  cnt[t] = count;
}

__global__ void k_exact_prep(const cp_inst_v1* __restrict__ inst, int n, int cap, long long max_plans,
                             const int32_t* __restrict__ upper, const int32_t* __restrict__ cnt,
                             int32_t* __restrict__ ibits, long long* __restrict__ total,
                             long long* __restrict__ chunks, int32_t* __restrict__ status,
                             unsigned long long* __restrict__ keys) {
  const int item = blockIdx.x * blockDim.x + threadIdx.x;
  if (item >= n) return;
  const cp_inst_v1* I = inst + item;
  const int p = I->n_pp, m = I->n_mb, ns = I->n_sub;
  int st = 0;
  bool bad = p < 1 || p > CP_MAX_STAGES || m < 1 || ns < 1;
  long long u = 0;
  for (int s = 0; !bad && s < p; ++s) {
    const long long tf = I->t_f[s], td = I->t_d[s], tw = I->t_w[s];
    bad = !(tf >= ns && td >= ns && tw >= ns && I->m_f[s] > 0 && I->m_d[s] <= 0 && I->m_w[s] <= 0 &&
            (long long)I->m_f[s] + I->m_d[s] + I->m_w[s] == 0 && I->m_lim[s] >= I->m_f[s] && I->t_dp[s] >= 0 &&
            I->t_ag[s] >= 0);
    if (s < p - 1)
      bad = bad || I->lat_f[s] < 0 || I->bw_f[s] < 0 || I->lat_b[s] < 0 || I->bw_b[s] < 0;
    u += m * (tf + td + tw) + ((I->flags & 1) ? I->t_ag[s] : 0) + I->t_dp[s];
    if (s < p - 1) u += m * ((long long)I->lat_f[s] + I->bw_f[s] + I->lat_b[s] + I->bw_b[s]);
  }
  long long tot = 1;
  if (bad) st = CPI_BAD_INSTANCE;
  else if (ns != 1 || p > kExactMaxP || m > kExactMaxM || u >= (1LL << 30)) st = CPI_OVERFLOW;
  else
    for (int s = 0; s < p; ++s) {
      const long long c = cnt[(long long)item * kExactMaxP + s];
      if (c > cap || c < 1 || tot > max_plans / c) { st = CPI_OVERFLOW; break; }
      tot *= c;
    }
  // key = makespan << b | index: b bits hold every index and the sentinel 2^b - 1 (> the last index),
  // the remaining 64 - b bits must hold the horizon
  int b = 1;
  while (b < 62 && (1LL << b) <= tot) ++b;
  if (!st && (64 - b >= 31 ? false : u >= (1LL << (64 - b)) - 1)) st = CPI_OVERFLOW;
  if (st) tot = 0;
  ibits[item] = b;
  total[item] = tot;
  chunks[item] = (tot + kExactChunk - 1) / kExactChunk;
  status[item] = st;
  // a known feasible makespan U (e.g. the greedy's) seeds the incumbent as (U << 36 | max index): plans
  // longer than U are cut from the start, and any plan of makespan <= U replaces it
  const int ub = upper ? upper[item] : -1;
  const bool seed = ub >= 0 && !st && (64 - b >= 31 || ub < (1LL << (64 - b)) - 1);
  keys[item] = seed ? (((unsigned long long)ub << b) | ((1ull << b) - 1)) : kExactNone;
}

// exclusive prefix over the chunk counts (one thread; n is at most a few thousand tiny searches)
__global__ void k_exact_scan(int n, long long* __restrict__ chunks) {
  long long acc = 0;
  for (int i = 0; i < n; ++i) { const long long c = chunks[i]; chunks[i] = acc; acc += c; }
  chunks[n] = acc;
}

__global__ void __launch_bounds__(128) k_exact_eval(const cp_inst_v1* __restrict__ inst, int n, int cap,
                                                    const unsigned long long* __restrict__ seqs,
                                                    const int32_t* __restrict__ cnt,
                                                    const int32_t* __restrict__ ibits,
                                                    const long long* __restrict__ total,
                                                    const long long* __restrict__ chunk_off,
                                                    unsigned long long* __restrict__ keys) {
  const long long n_chunks = chunk_off[n];
  for (long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x; c < n_chunks;
       c += (long long)gridDim.x * blockDim.x) {
    int lo = 0, hi = n - 1;                                      // instance: last offset <= c
    while (lo < hi) { const int mid = (lo + hi + 1) >> 1; if (chunk_off[mid] <= c) lo = mid; else hi = mid - 1; }
    const int item = lo;
    const cp_inst_v1* I = inst + item;
    const int p = I->n_pp, m = I->n_mb, L = 3 * m, ib = ibits[item];
    const long long i0 = (c - chunk_off[item]) * kExactChunk;
    const long long i1 = min(i0 + kExactChunk, total[item]);
    const bool zero1 = I->flags & 1;
    int tf[kExactMaxP], td[kExactMaxP], tw[kExactMaxP], tdp[kExactMaxP], nset[kExactMaxP], dig[kExactMaxP];
    int lf[kExactMaxP], bf[kExactMaxP], lb[kExactMaxP], bb[kExactMaxP], t0[kExactMaxP], work[kExactMaxP];
    unsigned long long seq[kExactMaxP];
    const unsigned long long* sbase = seqs + (long long)item * kExactMaxP * cap;
    long long r = i0;
    for (int s = p - 1; s >= 0; --s) {
      tf[s] = I->t_f[s]; td[s] = I->t_d[s]; tw[s] = I->t_w[s]; tdp[s] = I->t_dp[s];
      t0[s] = zero1 ? I->t_ag[s] : 0;
      work[s] = m * (tf[s] + td[s] + tw[s]);
      lf[s] = s < p - 1 ? I->lat_f[s] : 0; bf[s] = s < p - 1 ? I->bw_f[s] : 0;
      lb[s] = s < p - 1 ? I->lat_b[s] : 0; bb[s] = s < p - 1 ? I->bw_b[s] : 0;
      nset[s] = cnt[(long long)item * kExactMaxP + s];
      dig[s] = (int)(r % nset[s]); r /= nset[s];
      seq[s] = sbase[(long long)s * cap + dig[s]];
    }
    // Simulate stages 0..q-1 of the current plan; q < p relaxes stages q..p-1 to instantaneous and
    // free of their order (F_j passes through them and D_j comes back on arrival, each hop through its
    // FIFO link window).  Every start time can only drop, so the result bounds every plan with this
    // prefix from below, and a relaxed deadlock is a deadlock of all of them.  Returns the makespan
    // (q < p: the lower bound, including each relaxed stage's first arrival + work + DP tail), or -1
    // if it deadlocks or exceeds best.
    auto simulate = [&](int q, int best) -> int {
      const bool relax = q < p;
      int clk[kExactMaxP], pos[kExactMaxP], nF[kExactMaxP], nD[kExactMaxP], rem[kExactMaxP];
      int cF[kExactMaxP], cB[kExactMaxP];
      int rF[kExactMaxP][kExactMaxM], rD[kExactMaxP][kExactMaxM];
      for (int s = 0; s < p; ++s) { clk[s] = t0[s]; pos[s] = 0; nF[s] = 0; nD[s] = 0; rem[s] = work[s]; cF[s] = 0; cB[s] = 0; }
      int first[kExactMaxP];                                     // relax: F_0's arrival at each relaxed stage
      bool progress = true;
      int left = q * L;
      while (progress && left > 0) {
        progress = false;
        for (int s = 0; s < q; ++s) {
          while (pos[s] < L) {
            const int code = (int)((seq[s] >> (2 * pos[s])) & 3);
            int start, dur;
            if (code == (int)CP_OP_F) {
              const int j = nF[s];
              if (s > 0 && nF[s - 1] <= j) break;
              start = s > 0 ? max(clk[s], rF[s][j]) : clk[s];
              dur = tf[s];
              if (s < p - 1) {                                   // activation window on link s -> s+1
                const int w = max(start + dur, cF[s]);
                cF[s] = w + bf[s];
                rF[s + 1][j] = cF[s] + lf[s];
                if (relax && s == q - 1) {                       // through the relaxed stages and back
                  int t = rF[s + 1][j];
                  for (int k = q; k < p; ++k) {
                    if (j == 0) first[k] = t;
                    if (k < p - 1) { const int w2 = max(t, cF[k]); cF[k] = w2 + bf[k]; t = cF[k] + lf[k]; }
                  }
                  for (int k = p - 1; k >= q; --k) { const int w2 = max(t, cB[k - 1]); cB[k - 1] = w2 + bb[k - 1]; t = cB[k - 1] + lb[k - 1]; }
                  rD[s][j] = t;
                }
              }
              ++nF[s];
            } else if (code == (int)CP_OP_D) {
              const int j = nD[s];
              if (s < p - 1 && (relax && s == q - 1 ? nF[s] : nD[s + 1]) <= j) break;
              start = s < p - 1 ? max(clk[s], rD[s][j]) : clk[s];
              dur = td[s];
              if (s > 0) {                                       // gradient window on link s -> s-1
                const int w = max(start + dur, cB[s - 1]);
                cB[s - 1] = w + bb[s - 1];
                rD[s - 1][j] = cB[s - 1] + lb[s - 1];
              }
              ++nD[s];
            } else {
              start = clk[s];
              dur = tw[s];
            }
            clk[s] = start + dur;
            rem[s] -= dur;
            ++pos[s];
            --left;
            progress = true;
            if (clk[s] + rem[s] + tdp[s] > best) return -1;
          }
        }
      }
      if (left > 0) return -1;                                   // deadlock
      int ms = 0;
      for (int s = 0; s < q; ++s) ms = max(ms, clk[s] + tdp[s]);
      for (int k = q; k < p; ++k) ms = max(ms, max(first[k], t0[k]) + work[k] + tdp[k]);
      return ms > best ? -1 : ms;
    };
    // the stage digits that changed since the last prefix test (all at the chunk start)
    int chg = 0;
    for (long long idx = i0; idx < i1;) {
      const unsigned long long bk = *(volatile unsigned long long*)&keys[item] >> ib;   // racy incumbent: a bound only
      const int best = bk > 0x7fffffffull ? 0x7fffffff : (int)bk;
      // Test the deepest prefix (stages 0..p-2, the last stage relaxed) whenever it changed.  A chunk
      // covers 64 plans, so a cut at a shallower level could skip no further than the chunk's end:
      // testing those levels too measured slower (m = 4 E1 replicas 4.1 s against 2.8 s).
      int cut = -1;
      if (chg <= p - 2 && simulate(p - 1, best) < 0) cut = p - 2;
      if (cut >= 0) {
        // skip the rest of this prefix's block: every digit after `cut` back to 0, digit `cut` + 1
        long long block = 1, off = 0;
        for (int k = p - 1; k > cut; --k) { off += block * dig[k]; block *= nset[k]; }
        idx += block - off;
        for (int k = p - 1; k > cut; --k) { dig[k] = 0; seq[k] = sbase[(long long)k * cap]; }
        chg = cut;
        for (int k = cut; k >= 0; --k) {
          chg = k;
          if (++dig[k] < nset[k]) { seq[k] = sbase[(long long)k * cap + dig[k]]; break; }
          dig[k] = 0;
          seq[k] = sbase[(long long)k * cap];
        }
        continue;
      }
      chg = p - 1;                                               // (no prefix left to test at this plan)
      const int ms = simulate(p, best);
      if (ms >= 0) {
        const unsigned long long key = ((unsigned long long)ms << ib) | (unsigned long long)idx;
        if (key < *(volatile unsigned long long*)&keys[item]) atomicMin(&keys[item], key);
      }
      for (int s = p - 1; s >= 0; --s) {                         // odometer, last stage fastest
        chg = s;
        if (++dig[s] < nset[s]) { seq[s] = sbase[(long long)s * cap + dig[s]]; break; }
        dig[s] = 0;
        seq[s] = sbase[(long long)s * cap];
      }
      ++idx;
    }
  }
}

__global__ void k_exact_finish(const cp_inst_v1* __restrict__ inst, int n, int cap,
                               const unsigned long long* __restrict__ seqs, const int32_t* __restrict__ cnt,
                               const int32_t* __restrict__ ibits,
                               const unsigned long long* __restrict__ keys, int stride, int words,
                               uint32_t* __restrict__ ops, uint16_t* __restrict__ len, int32_t* __restrict__ makespan,
                               int32_t* __restrict__ status) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)n * stride) return;
  const int item = (int)(t / stride), s = (int)(t % stride);
  const int p = inst[item].n_pp, m = inst[item].n_mb;
  const unsigned long long key = keys[item];
  const int ib = ibits[item];
  const unsigned long long imask = (1ull << ib) - 1;
  const bool found = status[item] == 0 && key != kExactNone && (key & imask) != imask;
  unsigned long long sq = 0;
  int L = 0;
  if (found && s < p) {
    long long r = (long long)(key & imask);
    int d = 0;
    for (int q = p - 1; q >= s; --q) { const int c = cnt[(long long)item * kExactMaxP + q]; d = (int)(r % c); r /= c; }
    sq = seqs[((long long)item * kExactMaxP + s) * cap + d];
    L = 3 * m;
  }
  uint32_t* row = ops + (long long)item * words * stride + s;
  for (int k = 0; k < words; ++k) row[(long long)k * stride] = k < 2 ? (uint32_t)(sq >> (32 * k)) : 0u;
  len[t] = (uint16_t)L;
  if (s == 0) {
    makespan[item] = found ? (int32_t)(key >> ib) : -1;
    if (status[item] == 0 && !found) status[item] = CPI_DEADLOCK;
  }
}

int launch_exact(const cp_inst_v1* inst, int n, int cap, long long max_plans, const int32_t* upper, void* ws,
                 int stride, int words, uint32_t* ops, uint16_t* len, int32_t* makespan, int32_t* status,
                 void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  char* b = (char*)ws;
  unsigned long long* seqs = (unsigned long long*)b;   b += exact_ws_seq_bytes(n, cap);
  int32_t* cnt = (int32_t*)b;                          b += ((size_t)n * kExactMaxP * 4 + 255) & ~(size_t)255;
  long long* total = (long long*)b;                    b += ((size_t)n * 8 + 255) & ~(size_t)255;
  long long* chunks = (long long*)b;                   b += ((size_t)(n + 1) * 8 + 255) & ~(size_t)255;
  unsigned long long* keys = (unsigned long long*)b;   b += ((size_t)n * 8 + 255) & ~(size_t)255;
  int32_t* ibits = (int32_t*)b;
  const long long nt = (long long)n * kExactMaxP;
  k_exact_sets<<<(unsigned)((nt + 127) / 128), 128, 0, st>>>(inst, n, cap, seqs, cnt);
  k_exact_prep<<<(n + 127) / 128, 128, 0, st>>>(inst, n, cap, max_plans, upper, cnt, ibits, total, chunks, status,
                                                 keys);
  k_exact_scan<<<1, 1, 0, st>>>(n, chunks);
  k_exact_eval<<<device_sm_count() * 8, 128, 0, st>>>(inst, n, cap, seqs, cnt, ibits, total, chunks, keys);
  const long long nr = (long long)n * stride;
  k_exact_finish<<<(unsigned)((nr + 127) / 128), 128, 0, st>>>(inst, n, cap, seqs, cnt, ibits, keys, stride, words, ops, len,
                                                                makespan, status);
  return (int)cudaGetLastError();
}

size_t exact_ws_seq_bytes(int n, int cap) { return ((size_t)n * kExactMaxP * cap * 8 + 255) & ~(size_t)255; }

size_t exact_ws_bytes(int n, int cap) {
  return exact_ws_seq_bytes(n, cap) + (((size_t)n * kExactMaxP * 4 + 255) & ~(size_t)255) +
         (((size_t)n * 8 + 255) & ~(size_t)255) + (((size_t)(n + 1) * 8 + 255) & ~(size_t)255) +
         (((size_t)n * 8 + 255) & ~(size_t)255) + (((size_t)n * 4 + 255) & ~(size_t)255);
}

}  // namespace cpk
