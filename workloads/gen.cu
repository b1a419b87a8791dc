// gen.cu -- seeded generator of random VALID plans (workloads module; input generation only).
//
// Holds none of the method's arithmetic: no times, no link model, no greedy rule.  A plan
// is produced by a round-synchronous token game over the combinatorial dependency
// structure of the UD pattern (F_j on s needs F_j produced on s-1; D_j on s needs D_j
// produced on s+1, or F_j on the last stage; W sub-blocks of microbatch j need D_j) plus a
// per-stage counter of activations held (F adds m_f, D adds m_d, a W block's last sub-block
// adds m_w) that must stay <= m_lim.  Each round every stage appends at most one executable
// op: with probability q/4 a uniformly random one, else by the fixed preference D > F > W.
// Randomness is counter-based: u = splitmix64(seed ^ splitmix64(id ^ (s << 40) ^ (round << 8))),
// so the host and device versions (same source) produce identical plans.
// Output: the documented 2-bit plan format (word-major, stage-minor).
#include <cuda_runtime.h>
#include <stdint.h>

#define GEN_MAXP 32

__host__ __device__ static inline uint64_t gen_mix(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// returns 0 on success, 1 if the token game got stuck (never observed), 2 on bad args
__host__ __device__ static int gen_plan(int p, int m, int nsub, const int32_t* mf, const int32_t* md,
                                        const int32_t* mw, const int32_t* mlim, uint64_t seed, uint64_t id,
                                        int q, uint32_t* ops, uint16_t* len, int words, int stride) {
  if (p < 1 || p > GEN_MAXP || m < 1 || nsub < 1 || (2 + nsub) * m > 16 * words) return 2;
  int nF[GEN_MAXP], nD[GEN_MAXP], nW[GEN_MAXP], mem[GEN_MAXP], prevF[GEN_MAXP], prevD[GEN_MAXP];
  uint32_t cur[GEN_MAXP];
  for (int s = 0; s < p; ++s) { nF[s] = nD[s] = nW[s] = mem[s] = 0; cur[s] = 0; }
  const int total = (2 + nsub) * m;
  for (uint64_t r = 0;; ++r) {
    for (int s = 0; s < p; ++s) { prevF[s] = nF[s]; prevD[s] = nD[s]; }
    bool progress = false, done = true;
    for (int s = 0; s < p; ++s) {
      const int k = nF[s] + nD[s] + nW[s];
      if (k == total) continue;
      done = false;
      const bool canF = nF[s] < m && (s == 0 || prevF[s - 1] > nF[s]) && mem[s] + mf[s] <= mlim[s];
      const bool canD = nD[s] < m && (s == p - 1 ? nF[s] > nD[s] : prevD[s + 1] > nD[s]);
      const bool canW = nW[s] < nsub * nD[s];
      const int nx = (int)canF + (int)canD + (int)canW;
      if (nx == 0) continue;
      const uint64_t u = gen_mix(seed ^ gen_mix(id ^ ((uint64_t)s << 40) ^ (r << 8)));
      int code;
      if ((int)(u & 3u) < q) {
        int pick = (int)((u >> 8) % (uint64_t)nx);
        code = -1;
        if (canF) { if (pick == 0) code = 0; --pick; }
        if (code < 0 && canD) { if (pick == 0) code = 2; --pick; }
        if (code < 0) code = 3;
      } else {
        code = canD ? 2 : (canF ? 0 : 3);
      }
      if (code == 0) { nF[s]++; mem[s] += mf[s]; }
      else if (code == 2) { nD[s]++; mem[s] += md[s]; }
      else { nW[s]++; if (nW[s] % nsub == 0) mem[s] += mw[s]; }
      cur[s] |= (uint32_t)code << ((k & 15) * 2);
      if ((k & 15) == 15 || k + 1 == total) { ops[(k >> 4) * stride + s] = cur[s]; cur[s] = 0; }
      progress = true;
    }
    if (done) break;
    if (!progress) return 1;
  }
  for (int s = 0; s < p; ++s) len[s] = (uint16_t)total;
  return 0;
}

// Wave pattern (reading Q32): the same round-synchronous token game over the Wave data flow (F0
// needs F0 of s-1; F1 needs F1 of s+1, or the own F0 on the last stage; D1 needs D1 of s-1, or the
// own F1 on stage 0; D0 needs D0 of s+1, or the own D1 on the last stage; W sub-blocks of chunk c
// need a D of chunk c).  No memory gating, so the game cannot get stuck.  Preference: D (chunk 1
// first) > F (chunk 0 first) > W, or with probability q/4 a uniformly random executable entry.
// Output: 4-bit entries type | chunk << 2, 8 per word, word-major / stage-minor.
// loop = 1: the Loop pattern (reading Q33) instead: F1 on stage 0 needs F0 of the last stage (wrap),
// F1 elsewhere F1 of s-1; D1 needs D1 of s+1, or the own F1 on the last stage; D0 needs D0 of s+1,
// or D1 of stage 0 on the last stage (wrap).
__host__ __device__ static int gen_wave_plan(int p, int m, int nsub, uint64_t seed, uint64_t id, int q, uint32_t* ops,
                                             uint16_t* len, int words, int stride, int loop = 0) {
  const int total = 2 * (2 + nsub) * m;
  if (p < 1 || p > GEN_MAXP || m < 1 || nsub < 1 || total > 8 * words) return 2;
  int nF[2][GEN_MAXP], nD[2][GEN_MAXP], nW[2][GEN_MAXP], pF[2][GEN_MAXP], pD[2][GEN_MAXP];
  uint32_t cur[GEN_MAXP];
  for (int s = 0; s < p; ++s) {
    cur[s] = 0;
    for (int c = 0; c < 2; ++c) nF[c][s] = nD[c][s] = nW[c][s] = 0;
  }
  for (uint64_t r = 0;; ++r) {
    for (int s = 0; s < p; ++s)
      for (int c = 0; c < 2; ++c) { pF[c][s] = nF[c][s]; pD[c][s] = nD[c][s]; }
    bool progress = false, done = true;
    for (int s = 0; s < p; ++s) {
      const int k = nF[0][s] + nF[1][s] + nD[0][s] + nD[1][s] + nW[0][s] + nW[1][s];
      if (k == total) continue;
      done = false;
      int cand[6], nx = 0;                       // entry codes, in preference order
      if (!loop) {
        if (nD[1][s] < m && (s == 0 ? nF[1][s] > nD[1][s] : pD[1][s - 1] > nD[1][s])) cand[nx++] = 2 | 4;
        if (nD[0][s] < m && (s == p - 1 ? nD[1][s] > nD[0][s] : pD[0][s + 1] > nD[0][s])) cand[nx++] = 2;
        if (nF[0][s] < m && (s == 0 || pF[0][s - 1] > nF[0][s])) cand[nx++] = 0;
        if (nF[1][s] < m && (s == p - 1 ? nF[0][s] > nF[1][s] : pF[1][s + 1] > nF[1][s])) cand[nx++] = 4;
      } else {
        if (nD[1][s] < m && (s == p - 1 ? nF[1][s] > nD[1][s] : pD[1][s + 1] > nD[1][s])) cand[nx++] = 2 | 4;
        if (nD[0][s] < m && (s == p - 1 ? pD[1][0] > nD[0][s] : pD[0][s + 1] > nD[0][s])) cand[nx++] = 2;
        if (nF[0][s] < m && (s == 0 || pF[0][s - 1] > nF[0][s])) cand[nx++] = 0;
        if (nF[1][s] < m && (s == 0 ? pF[0][p - 1] > nF[1][s] : pF[1][s - 1] > nF[1][s])) cand[nx++] = 4;
      }
      if (nW[1][s] < nsub * nD[1][s]) cand[nx++] = 3 | 4;
      if (nW[0][s] < nsub * nD[0][s]) cand[nx++] = 3;
      if (nx == 0) continue;
      const uint64_t u = gen_mix(seed ^ gen_mix(id ^ ((uint64_t)s << 40) ^ (r << 8) ^ 0x57ull));
      const int x = ((int)(u & 3u) < q) ? cand[(int)((u >> 8) % (uint64_t)nx)] : cand[0];
      const int t = x & 3, c = x >> 2;
      if (t == 0) nF[c][s]++;
      else if (t == 2) nD[c][s]++;
      else nW[c][s]++;
      cur[s] |= (uint32_t)x << ((k & 7) * 4);
      if ((k & 7) == 7 || k + 1 == total) { ops[(k >> 3) * stride + s] = cur[s]; cur[s] = 0; }
      progress = true;
    }
    if (done) break;
    if (!progress) return 1;
  }
  for (int s = 0; s < p; ++s) len[s] = (uint16_t)total;
  return 0;
}

__global__ void k_gen_wave(int p, int m, int nsub, uint64_t seed, uint64_t id0, int q, long long n, int words,
                           int stride, uint32_t* ops, uint16_t* len, int32_t* err, int loop) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (gen_wave_plan(p, m, nsub, seed, id0 + (uint64_t)i, q, ops + i * (long long)words * stride,
                    len + i * (long long)stride, words, stride, loop))
    atomicAdd(err, 1);
}

struct GenArgs {
  int p, m, nsub, q, words, stride;
  int32_t mf[GEN_MAXP], md[GEN_MAXP], mw[GEN_MAXP], mlim[GEN_MAXP];
  uint64_t seed, id0;
  long long n;
};

__global__ void k_gen(const __grid_constant__ GenArgs a, uint32_t* ops, uint16_t* len, int32_t* err) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n) return;
  const int e = gen_plan(a.p, a.m, a.nsub, a.mf, a.md, a.mw, a.mlim, a.seed, a.id0 + (uint64_t)i, a.q,
                         ops + i * (long long)a.words * a.stride, len + i * (long long)a.stride, a.words, a.stride);
  if (e) atomicAdd(err, 1);
}

extern "C" {

// host: plans for ids id0 .. id0+n-1; returns number of failures
int cpgen_plans_host(int p, int m, int nsub, const int32_t* mf, const int32_t* md, const int32_t* mw,
                     const int32_t* mlim, uint64_t seed, uint64_t id0, int q, long long n, uint32_t* ops,
                     uint16_t* len, int words, int stride) {
  int err = 0;
  for (long long i = 0; i < n; ++i)
    err += gen_plan(p, m, nsub, mf, md, mw, mlim, seed, id0 + (uint64_t)i, q, ops + i * (long long)words * stride,
                    len + i * (long long)stride, words, stride) != 0;
  return err;
}

// Wave plans (host / device, identical for the same ids)
int cpgen_wave_plans_host(int p, int m, int nsub, uint64_t seed, uint64_t id0, int q, long long n, uint32_t* ops,
                          uint16_t* len, int words, int stride, int loop) {
  int err = 0;
  for (long long i = 0; i < n; ++i)
    err += gen_wave_plan(p, m, nsub, seed, id0 + (uint64_t)i, q, ops + i * (long long)words * stride,
                         len + i * (long long)stride, words, stride, loop) != 0;
  return err;
}
int cpgen_wave_plans_device(int p, int m, int nsub, uint64_t seed, uint64_t id0, int q, long long n, uint32_t* ops,
                            uint16_t* len, int words, int stride, int32_t* err, void* stream, int loop) {
  const int threads = 128;
  const long long blocks = (n + threads - 1) / threads;
  k_gen_wave<<<(unsigned)blocks, threads, 0, (cudaStream_t)stream>>>(p, m, nsub, seed, id0, q, n, words, stride, ops,
                                                                      len, err, loop);
  return (int)cudaGetLastError();
}

// device: same plans into device buffers (err: device int32, caller-zeroed)
int cpgen_plans_device(int p, int m, int nsub, const int32_t* mf, const int32_t* md, const int32_t* mw,
                       const int32_t* mlim, uint64_t seed, uint64_t id0, int q, long long n, uint32_t* ops,
                       uint16_t* len, int words, int stride, int32_t* err, void* stream) {
  GenArgs a;
  a.p = p; a.m = m; a.nsub = nsub; a.q = q; a.words = words; a.stride = stride;
  for (int s = 0; s < GEN_MAXP; ++s) {
    a.mf[s] = s < p ? mf[s] : 0; a.md[s] = s < p ? md[s] : 0; a.mw[s] = s < p ? mw[s] : 0; a.mlim[s] = s < p ? mlim[s] : 0;
  }
  a.seed = seed; a.id0 = id0; a.n = n;
  const int threads = 128;
  const long long blocks = (n + threads - 1) / threads;
  k_gen<<<(unsigned)blocks, threads, 0, (cudaStream_t)stream>>>(a, ops, len, err);
  return (int)cudaGetLastError();
}
}
