// exact_bnb.cu -- cp_exact_bnb: batched parallel branch and bound for the makespan-optimal split
// plan (n_sub = 1) of tiny instances (the stand-in for the paper's CO
// solver, §4.1 :313-360: per-stage order of F/D/W blocks respecting microbatch order per
// type, D_j after F_j, W_j after D_j and the memory capacity; objective = makespan, DP tail :363).
// Where cp_exact enumerates the plan product (m <= 4 on 4 stages), the search here reaches the
// paper's own 4 x 8 E1 setup (:486, :491) and beyond.
//
// Search space.  A node is a partial schedule: a prefix of every stage's sequence with fixed block
// starts.  A child appends one eligible block x to one stage s (next F if its input arrived and
// memory fits, next D if its gradient arrived, next W if its D is done) at
//   start = max(stage clock, input arrival, ZeRO-1 AG end, floor),
// where floor = the parent's own append start, plus one tick when s is below the parent's stage.
// Appends in increasing (start, stage) order reproduce every plan's semi-active schedule; other
// orders only delay it.  A node's future depends on its per-(stage, type) counts and its interface
// times (makespan so far; stage clocks raised to the floor; link clocks and pending arrivals raised
// to the consumer's clock), which gives the dominance cut below.
//
// Parallel search.  One warp is one worker, its node state in shared memory; lanes cooperate on
// the children (lane = (stage, type)), on the heads (one max-plus warp scan per stage and type),
// on the lower bound (lane = stage) and on the dominance test (lanes over vector components).
//   * Work items are search nodes given by their append path from the root.  Each round, warps
//     take items from a global frontier, replay the path, and search depth first (children in
//     increasing (start, stage, D < F < W)) for at most `budget` nodes; the unexplored children on
//     the warp's stack are then written to the next round's frontier.  The host repeats rounds
//     until the frontier is empty: the search is complete and the incumbent is optimal.
//   * Incumbent per instance: makespan in global memory (upper + 1 if a feasible makespan is given,
//     so a plan reaching it is found), improved under a per-instance lock together with its plan.
//   * Lower bound (cut when >= incumbent): the makespan so far, and per stage Jackson's preemptive
//     one-machine schedule of its remaining blocks, heads r from the dependency chains, link clocks
//     and floor, tails q = longest dependency path from a block's end to the end (DP tail
//     included).  Within a type heads increase and tails decrease with the microbatch, so the
//     preemptive rule (largest tail first) only ever chooses between the first unfinished block of
//     each type: three candidates per event, O(blocks) per stage.
//   * Dominance: a per-instance hash table in global memory of (counts, interface vector); a node
//     is cut when a recorded node with the same counts has every interface time <= its own (its
//     completions are matched, no later anywhere, by the same appends from the recorded node).  A
//     node is recorded only once its test passed, so it is always searched (in this round or from
//     the frontier); entries are claimed by atomicCAS and published with a ready flag after a fence.
// Result per instance: makespan and plan of the incumbent, status 0 when the search completed
// (optimal), CPI_INCOMPLETE when a node or frontier limit stopped it (makespan = best plan found,
// bound = root lower bound), CPI_DEADLOCK when no plan reaches `upper`, CPI_OVERFLOW when the
// instance is outside the limits (p <= 8, m <= 16, n_sub = 1, horizon < 2^30).
#include <cuda_runtime.h>
#include <stdint.h>

#include "engine.h"

namespace cpk {

constexpr int BP = kBnbMaxP, BM = kBnbMaxM;
constexpr int kBnbWarps = 4;                    // warps per block
constexpr int kInf = 0x3fffffff;

struct BInst {                                   // per-instance search constants (k_bnb_prep)
  int p, m, zero1, L, vlen_max, ok;
  int tf[BP], td[BP], tw[BP], mf[BP], md[BP], mw[BP], mlim[BP], tdp[BP], tag[BP];
  int latf[BP], bwf[BP], latb[BP], bwb[BP];
  int qF[BP][BM], qD[BP][BM], qW[BP][BM];
};

struct BCtl {                                    // per-instance shared search control
  int best;                                      // incumbent makespan (kInf: none)
  int lock;
  int incomplete;                                // a limit stopped the search
  int has_plan;
  unsigned long long nodes;
  int root_bound;
  int pad;
};

struct BState {                                  // one warp's node (shared memory)
  int clk[BP], mem[BP], linkF[BP], linkB[BP];
  int endF[BP][BM], endD[BP][BM], arrF[BP][BM], arrD[BP][BM];
  int hF[BP][BM], hD[BP][BM], hW[BP][BM];        // heads scratch of the bound
  unsigned char n[BP][3];                        // blocks done per (stage, type F/D/W)
  int t_last, s_last, M, depth;
};

struct BLevel {                                  // DFS level: last child tried + undo of that child
  int last_start, last_idx;
  int prev_clk, prev_link, prev_M, prev_tlast, prev_slast, code;
};

__device__ __forceinline__ int imax(int a, int b) { return a > b ? a : b; }

// ---------------------------------------------------------------------------------------------- prep
__global__ void k_bnb_prep(const cp_inst_v1* __restrict__ inst, int n, const int32_t* __restrict__ upper,
                           BInst* __restrict__ bi, BCtl* __restrict__ ctl, unsigned char* __restrict__ front,
                           int front_stride, int* __restrict__ front_n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const cp_inst_v1* I = inst + i;
  BInst& B = bi[i];
  BCtl& C = ctl[i];
  C.best = kInf; C.lock = 0; C.incomplete = 0; C.has_plan = 0; C.nodes = 0; C.root_bound = 0;
  const int p = I->n_pp, m = I->n_mb;
  bool ok = p >= 1 && p <= BP && m >= 1 && m <= BM && I->n_sub == 1;
  long long U = 0;
  if (ok)
    for (int s = 0; s < p; ++s) {
      ok = ok && I->t_f[s] > 0 && I->t_d[s] > 0 && I->t_w[s] > 0 && I->m_f[s] > 0 && I->m_d[s] <= 0 &&
           I->m_w[s] <= 0 && (long long)I->m_f[s] + I->m_d[s] + I->m_w[s] == 0 && I->m_lim[s] >= I->m_f[s] &&
           I->t_dp[s] >= 0 && I->t_ag[s] >= 0;
      if (s < p - 1) ok = ok && I->lat_f[s] >= 0 && I->bw_f[s] >= 0 && I->lat_b[s] >= 0 && I->bw_b[s] >= 0;
      U += (long long)m * ((long long)I->t_f[s] + I->t_d[s] + I->t_w[s]) + I->t_dp[s] + I->t_ag[s];
      if (s < p - 1) U += (long long)m * ((long long)I->lat_f[s] + I->bw_f[s] + I->lat_b[s] + I->bw_b[s]);
    }
  ok = ok && U < (1LL << 29);
  B.ok = ok;
  if (!ok) return;
  B.p = p; B.m = m; B.zero1 = I->flags & 1; B.L = 3 * m * p;
  for (int s = 0; s < BP; ++s) {
    const bool on = s < p, link = s < p - 1;
    B.tf[s] = on ? I->t_f[s] : 0; B.td[s] = on ? I->t_d[s] : 0; B.tw[s] = on ? I->t_w[s] : 0;
    B.mf[s] = on ? I->m_f[s] : 0; B.md[s] = on ? I->m_d[s] : 0; B.mw[s] = on ? I->m_w[s] : 0;
    B.mlim[s] = on ? I->m_lim[s] : 0; B.tdp[s] = on ? I->t_dp[s] : 0;
    B.tag[s] = on && B.zero1 ? I->t_ag[s] : 0;
    B.latf[s] = link ? I->lat_f[s] : 0; B.bwf[s] = link ? I->bw_f[s] : 0;
    B.latb[s] = link ? I->lat_b[s] : 0; B.bwb[s] = link ? I->bw_b[s] : 0;
  }
  // tails: W_j -> W_{j+1} and the DP tail; D_j -> W_j, D_{j+1}, D_j(s-1) over the link;
  // F_j -> F_{j+1}, F_j(s+1) over the link, or D_j(p-1) on the last stage
  for (int s = 0; s < p; ++s)
    for (int j = m - 1; j >= 0; --j) B.qW[s][j] = imax(B.tdp[s], j + 1 < m ? B.tw[s] + B.qW[s][j + 1] : 0);
  for (int j = m - 1; j >= 0; --j)
    for (int s = 0; s < p; ++s) {
      int q = imax(B.tdp[s], B.tw[s] + B.qW[s][j]);
      if (j + 1 < m) q = imax(q, B.td[s] + B.qD[s][j + 1]);
      if (s > 0) q = imax(q, B.bwb[s - 1] + B.latb[s - 1] + B.td[s - 1] + B.qD[s - 1][j]);
      B.qD[s][j] = q;
    }
  for (int j = m - 1; j >= 0; --j)
    for (int s = p - 1; s >= 0; --s) {
      int q = B.tdp[s];
      if (j + 1 < m) q = imax(q, B.tf[s] + B.qF[s][j + 1]);
      q = s < p - 1 ? imax(q, B.bwf[s] + B.latf[s] + B.tf[s + 1] + B.qF[s + 1][j]) : imax(q, B.td[s] + B.qD[s][j]);
      B.qF[s][j] = q;
    }
  B.vlen_max = 3 * p - 1 + 2 * (p - 1) * m;
  if (upper && upper[i] >= 0) C.best = upper[i] + 1;
  const int e = atomicAdd(front_n, 1);
  unsigned char* fe = front + (long long)e * front_stride;
  reinterpret_cast<int*>(fe)[0] = i;
  reinterpret_cast<int*>(fe)[1] = 0;
}

// ---------------------------------------------------------------------------------------------- node ops
// start of block (s, ty) appended to S (ty 0 F, 1 D, 2 W), -1 if not eligible
__device__ __forceinline__ int bnb_start(const BState& S, const BInst& B, int s, int ty) {
  const int j = S.n[s][ty];
  if (s >= B.p || j >= B.m) return -1;
  int a;
  if (ty == 0) {
    if (S.mem[s] + B.mf[s] > B.mlim[s]) return -1;
    if (s == 0) a = 0;
    else if (j < S.n[s - 1][0]) a = S.arrF[s][j];
    else return -1;
    a = imax(a, B.tag[s]);
  } else if (ty == 1) {
    if (j >= S.n[s][0]) return -1;
    if (s == B.p - 1) a = S.endF[s][j];
    else if (j < S.n[s + 1][1]) a = S.arrD[s][j];
    else return -1;
  } else {
    if (j >= S.n[s][1]) return -1;
    a = S.endD[s][j];
  }
  const int fl = S.t_last + (s < S.s_last ? 1 : 0);
  return imax(imax(S.clk[s], a), fl);
}

// append (lane 0 only); records the undo in lv
__device__ __forceinline__ void bnb_append(BState& S, const BInst& B, int s, int ty, int start, BLevel& lv,
                                           unsigned char* path) {
  const int j = S.n[s][ty];
  lv.prev_clk = S.clk[s];
  lv.prev_M = S.M;
  lv.prev_tlast = S.t_last;
  lv.prev_slast = S.s_last;
  lv.code = s * 3 + ty;
  lv.prev_link = 0;
  const int end = start + (ty == 0 ? B.tf[s] : (ty == 1 ? B.td[s] : B.tw[s]));
  path[S.depth] = (unsigned char)(s * 3 + ty);
  S.n[s][ty] = (unsigned char)(j + 1);
  S.clk[s] = end;
  if (ty == 0) {
    S.mem[s] += B.mf[s];
    S.endF[s][j] = end;
    if (s < B.p - 1) {               // Alg. 1 :404-407: window at or after ready (FIFO link, App. X1), then latency
      int ws = end;
      lv.prev_link = S.linkF[s];
      if (B.bwf[s] > 0) { ws = imax(end, S.linkF[s]); S.linkF[s] = ws + B.bwf[s]; }
      S.arrF[s + 1][j] = ws + B.bwf[s] + B.latf[s];
    }
  } else if (ty == 1) {
    S.mem[s] += B.md[s];
    S.endD[s][j] = end;
    if (s > 0) {
      int ws = end;
      lv.prev_link = S.linkB[s];
      if (B.bwb[s - 1] > 0) { ws = imax(end, S.linkB[s]); S.linkB[s] = ws + B.bwb[s - 1]; }
      S.arrD[s - 1][j] = ws + B.bwb[s - 1] + B.latb[s - 1];
    }
  } else {
    S.mem[s] += B.mw[s];
  }
  S.M = imax(S.M, end);
  if (ty == 2 && j + 1 == B.m) S.M = imax(S.M, end + B.tdp[s]);   // DP allreduce after the last W (:363)
  S.t_last = start;
  S.s_last = s;
  S.depth++;
}

__device__ __forceinline__ void bnb_undo(BState& S, const BInst& B, const BLevel& lv) {
  const int s = lv.code / 3, ty = lv.code % 3;
  const int j = S.n[s][ty] - 1;
  S.n[s][ty] = (unsigned char)j;
  S.clk[s] = lv.prev_clk;
  S.mem[s] -= ty == 0 ? B.mf[s] : (ty == 1 ? B.md[s] : B.mw[s]);
  if (ty == 0 && s < B.p - 1) S.linkF[s] = lv.prev_link;
  if (ty == 1 && s > 0) S.linkB[s] = lv.prev_link;
  S.M = lv.prev_M;
  S.t_last = lv.prev_tlast;
  S.s_last = lv.prev_slast;
  S.depth--;
}

// inclusive max-plus chain over lanes j in [j0, m): r_j = max(a_j, r_{j-1} + d), r_{j0-1} + d := c
__device__ __forceinline__ int chain_scan(int lane, int j0, int m, int a, int d, int c) {
  const bool on = lane >= j0 && lane < m;
  int v = on ? (lane == j0 ? imax(a, c) : a) - lane * d : -kInf;
#pragma unroll
  for (int k = 1; k < 32; k <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, v, k);
    if (lane >= k) v = imax(v, u);
  }
  return on ? v + lane * d : 0;
}

// lower bound of every completion of S (all lanes; result on every lane)
__device__ int bnb_bound(BState& S, const BInst& B, int lane) {
  const int p = B.p, m = B.m;
  auto cs = [&](int s) { return imax(S.clk[s], S.t_last + (s < S.s_last ? 1 : 0)); };
  // F heads, s ascending
  for (int s = 0; s < p; ++s) {
    const int j0 = S.n[s][0];
    int a = 0;
    if (lane >= j0 && lane < m) {
      if (s > 0) {
        if (lane < S.n[s - 1][0]) a = S.arrF[s][lane];
        else {
          const int e = S.hF[s - 1][lane] + B.tf[s - 1];
          a = (B.bwf[s - 1] > 0 ? imax(e, S.linkF[s - 1]) : e) + B.bwf[s - 1] + B.latf[s - 1];
        }
      }
      a = imax(a, B.tag[s]);
    }
    const int r = chain_scan(lane, j0, m, a, B.tf[s], cs(s));
    if (lane >= j0 && lane < m) S.hF[s][lane] = r;
    __syncwarp();
  }
  // D heads, s descending
  for (int s = p - 1; s >= 0; --s) {
    const int j0 = S.n[s][1];
    int a = 0;
    if (lane >= j0 && lane < m) {
      a = lane < S.n[s][0] ? S.endF[s][lane] : S.hF[s][lane] + B.tf[s];
      if (s < p - 1) {
        int g;
        if (lane < S.n[s + 1][1]) g = S.arrD[s][lane];
        else {
          const int e = S.hD[s + 1][lane] + B.td[s + 1];
          g = (B.bwb[s] > 0 ? imax(e, S.linkB[s + 1]) : e) + B.bwb[s] + B.latb[s];
        }
        a = imax(a, g);
      }
    }
    const int r = chain_scan(lane, j0, m, a, B.td[s], cs(s));
    if (lane >= j0 && lane < m) S.hD[s][lane] = r;
    __syncwarp();
  }
  // W heads
  for (int s = 0; s < p; ++s) {
    const int j0 = S.n[s][2];
    int a = 0;
    if (lane >= j0 && lane < m) a = lane < S.n[s][1] ? S.endD[s][lane] : S.hD[s][lane] + B.td[s];
    const int r = chain_scan(lane, j0, m, a, B.tw[s], cs(s));
    if (lane >= j0 && lane < m) S.hW[s][lane] = r;
  }
  __syncwarp();
  // per stage (lane s): Jackson's preemptive schedule over the three type chains
  int lb = S.M;
  if (lane < p) {
    const int s = lane;
    int j[3] = {S.n[s][0], S.n[s][1], S.n[s][2]};
    const int d[3] = {B.tf[s], B.td[s], B.tw[s]};
    int rem[3] = {d[0], d[1], d[2]};
    auto head = [&](int t) { return t == 0 ? S.hF[s][j[0]] : (t == 1 ? S.hD[s][j[1]] : S.hW[s][j[2]]); };
    auto tail = [&](int t) { return t == 0 ? B.qF[s][j[0]] : (t == 1 ? B.qD[s][j[1]] : B.qW[s][j[2]]); };
    int t = kInf;
    for (int k = 0; k < 3; ++k) if (j[k] < m) t = min(t, head(k));
    while (j[0] < m || j[1] < m || j[2] < m) {
      int pick = -1, pq = -1, nr = kInf;
      for (int k = 0; k < 3; ++k) {
        if (j[k] >= m) continue;
        const int h = head(k);
        if (h <= t) { const int q = tail(k); if (q > pq) { pq = q; pick = k; } }
        else nr = min(nr, h);
      }
      if (pick < 0) { t = nr; continue; }
      int run = rem[pick];
      if (nr != kInf && t + run > nr) run = nr - t;
      t += run;
      rem[pick] -= run;
      if (rem[pick] == 0) { lb = imax(lb, t + pq); ++j[pick]; rem[pick] = d[pick]; }
    }
  }
#pragma unroll
  for (int k = 16; k >= 1; k >>= 1) lb = imax(lb, __shfl_xor_sync(0xffffffffu, lb, k));
  return lb;
}

// ---------------------------------------------------------------------------------------------- dominance
__device__ __forceinline__ unsigned long long mix64(unsigned long long x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
  return x;
}

struct BTable { unsigned char* base; long long cap; int stride; };   // entries: k0, k1, ready, pad, vec[]

// builds the interface vector into vec (smem); returns its length (all lanes)
__device__ int bnb_vector(const BState& S, const BInst& B, int lane, int* vec) {
  const int p = B.p;
  auto cs = [&](int s) { return imax(S.clk[s], S.t_last + (s < S.s_last ? 1 : 0)); };
  if (lane == 0) vec[0] = S.M;
  if (lane < p) {
    vec[1 + lane] = cs(lane);
    if (lane < p - 1) vec[1 + p + lane] = imax(S.linkF[lane], cs(lane));
    if (lane >= 1) vec[2 * p + lane - 1] = imax(S.linkB[lane], cs(lane));
  }
  const int o0 = 3 * p - 1;
  int cnt = 0;
  if (lane < p) {
    if (lane >= 1) cnt += S.n[lane - 1][0] - S.n[lane][0];
    if (lane < p - 1) cnt += S.n[lane + 1][1] - S.n[lane][1];
  }
  int incl = cnt;
#pragma unroll
  for (int k = 1; k < 32; k <<= 1) {
    const int u = __shfl_up_sync(0xffffffffu, incl, k);
    if (lane >= k) incl += u;
  }
  const int total = __shfl_sync(0xffffffffu, incl, 31);
  if (lane < p) {
    int o = o0 + incl - cnt;
    const int s = lane, c = cs(s);
    if (s >= 1) for (int j = S.n[s][0]; j < S.n[s - 1][0]; ++j) vec[o++] = imax(S.arrF[s][j], c);
    if (s < p - 1) for (int j = S.n[s][1]; j < S.n[s + 1][1]; ++j) vec[o++] = imax(S.arrD[s][j], c);
  }
  __syncwarp();
  return o0 + total;
}

// true if a recorded node dominates S; otherwise records S (best effort) and returns false
__device__ bool bnb_dominated(const BState& S, const BInst& B, const BTable& T, int lane, int* vec, int max_probe) {
  const int vlen = bnb_vector(S, B, lane, vec);
  unsigned long long k0 = 1ull << 63, k1 = 0;
  for (int s = 0; s < B.p; ++s)
    for (int t = 0; t < 3; ++t) {
      const int b = 15 * (s & 3) + 5 * t;
      if (s < 4) k0 |= (unsigned long long)S.n[s][t] << b; else k1 |= (unsigned long long)S.n[s][t] << b;
    }
  long long h = (long long)(mix64(k0 ^ mix64(k1)) & (unsigned long long)(T.cap - 1));
  for (int probe = 0; probe < max_probe; ++probe, h = (h + 1) & (T.cap - 1)) {
    unsigned char* e = T.base + h * (long long)T.stride;
    unsigned long long* ek = reinterpret_cast<unsigned long long*>(e);
    volatile int* ready = reinterpret_cast<volatile int*>(e + 16);
    int* ev = reinterpret_cast<int*>(e + 32);
    unsigned long long cur = 0;
    if (lane == 0) {
      cur = *reinterpret_cast<volatile unsigned long long*>(ek);
      if (cur == 0) {
        cur = atomicCAS(ek, 0ull, k0);
        if (cur == 0) cur = ~0ull;                     // claimed by this warp
      }
    }
    cur = __shfl_sync(0xffffffffu, cur, 0);
    if (cur == ~0ull) {                                // publish: k1, vector, fence, ready
      if (lane == 0) ek[1] = k1;
      for (int i = lane; i < vlen; i += 32) ev[i] = vec[i];
      __threadfence();
      __syncwarp();
      if (lane == 0) *ready = 1;
      return false;
    }
    if (cur != k0) continue;
    int rd = 0;
    unsigned long long ek1 = 0;
    if (lane == 0) { rd = *ready; if (rd) { __threadfence(); ek1 = *reinterpret_cast<volatile unsigned long long*>(ek + 1); } }
    rd = __shfl_sync(0xffffffffu, rd, 0);
    ek1 = __shfl_sync(0xffffffffu, ek1, 0);
    if (!rd || ek1 != k1) continue;
    bool le = true;
    for (int i = lane; i < vlen; i += 32) le = le && __ldcg(ev + i) <= vec[i];
    if (__all_sync(0xffffffffu, le)) return true;
  }
  return false;
}

// ---------------------------------------------------------------------------------------------- search
struct BnbRound {
  const BInst* bi;
  BCtl* ctl;
  unsigned char* best_plan;          // [n][BP * 3 * BM] per-stage sequences of the incumbent
  const unsigned char* front;        // this round's items
  int front_n;
  int* front_head;                   // item counter
  unsigned char* next;               // next round's items
  int* next_n;
  int front_cap, front_stride;
  unsigned char* table;              // [n] tables of table_cap entries
  long long table_cap;
  int table_stride, max_probe;
  int budget;
  int Lmax;
  unsigned long long* nodes_total;   // nodes searched by all rounds
};

// next child of the node in S after (ls, li): lane l < 3p is (stage l / 3, type D, F, W); returns the
// lane index (or -1) and its start in *st (all lanes)
__device__ __forceinline__ int bnb_next_child(const BState& S, const BInst& B, int lane, int ls, int li, int* st) {
  int start = -1;
  if (lane < 3 * B.p) {
    const int s = lane / 3, k = lane % 3;
    const int ty = k == 0 ? 1 : (k == 1 ? 0 : 2);
    start = bnb_start(S, B, s, ty);
    if (start >= 0 && (start < ls || (start == ls && lane <= li))) start = -1;
  }
  const unsigned v = start >= 0 ? (unsigned)start : 0xffffffffu;
  const unsigned mn = __reduce_min_sync(0xffffffffu, v);
  if (mn == 0xffffffffu) return -1;
  const unsigned bal = __ballot_sync(0xffffffffu, v == mn);
  *st = (int)mn;
  return __ffs(bal) - 1;
}

__device__ __forceinline__ int lane_type(int l) { const int k = l % 3; return k == 0 ? 1 : (k == 1 ? 0 : 2); }

__global__ void __launch_bounds__(32 * kBnbWarps) k_bnb_round(const BnbRound R) {
  extern __shared__ __align__(16) unsigned char bsm[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int per_warp = (int)((sizeof(BState) + R.Lmax * sizeof(BLevel) + R.Lmax + 4 * (3 * BP + 2 * BP * BM) + 15) & ~15);
  unsigned char* mine = bsm + w * per_warp;
  BState& S = *reinterpret_cast<BState*>(mine);
  BLevel* lv = reinterpret_cast<BLevel*>(mine + sizeof(BState));
  unsigned char* path = mine + sizeof(BState) + R.Lmax * sizeof(BLevel);
  int* vec = reinterpret_cast<int*>((reinterpret_cast<uintptr_t>(path + R.Lmax) + 3) & ~uintptr_t(3));
  for (;;) {
    int e = 0;
    if (lane == 0) e = atomicAdd(R.front_head, 1);
    e = __shfl_sync(0xffffffffu, e, 0);
    if (e >= R.front_n) break;
    const unsigned char* fe = R.front + (long long)e * R.front_stride;
    const int inst = reinterpret_cast<const int*>(fe)[0];
    const int plen = reinterpret_cast<const int*>(fe)[1];
    const BInst& B = R.bi[inst];
    BCtl& C = R.ctl[inst];
    const BTable T{R.table + (long long)inst * R.table_cap * R.table_stride, R.table_cap, R.table_stride};
    // reset and replay the item's path
    for (int i = lane; i < (int)sizeof(BState) / 4; i += 32) reinterpret_cast<int*>(&S)[i] = 0;
    for (int i = lane; i < plen; i += 32) path[i] = fe[8 + i];
    __syncwarp();
    if (lane == 0)
      for (int k = 0; k < plen; ++k) {
        const int code = path[k], s = code / 3, ty = code % 3;
        const int st = bnb_start(S, B, s, ty);
        bnb_append(S, B, s, ty, st, lv[0], path);
      }
    __syncwarp();
    const int base = plen;
    long long nodes = 0;
    // visit: 1 = search below, 0 = leaf or cut
    auto visit = [&]() -> int {
      ++nodes;
      if (S.depth == B.L) {
        if (lane == 0 && S.M < *(volatile int*)&C.best) {
          while (atomicCAS(&C.lock, 0, 1) != 0) {}
          __threadfence();
          if (S.M < *(volatile int*)&C.best) {
            unsigned char* bp = R.best_plan + (long long)inst * BP * 3 * BM;
            int pos[BP] = {};
            for (int k = 0; k < B.L; ++k) {
              const int code = path[k], s = code / 3, ty = code % 3;
              bp[s * 3 * BM + pos[s]++] = (unsigned char)(ty == 0 ? CP_OP_F : (ty == 1 ? CP_OP_D : CP_OP_W));
            }
            C.has_plan = 1;
            __threadfence();
            atomicExch(&C.best, S.M);
          }
          __threadfence();
          atomicExch(&C.lock, 0);
        }
        __syncwarp();
        return 0;
      }
      const int lb = bnb_bound(S, B, lane);
      if (S.depth == 0 && lane == 0) C.root_bound = lb;
      int ub = lane == 0 ? *(volatile int*)&C.best : 0;
      ub = __shfl_sync(0xffffffffu, ub, 0);                  // one incumbent read per warp: uniform decision
      if (lb >= ub) return 0;
      if (bnb_dominated(S, B, T, lane, vec, R.max_probe)) return 0;
      return 1;
    };
    int top = -1;
    if (visit()) { top = 0; if (lane == 0) { lv[0].last_start = -1; lv[0].last_idx = -1; } }
    __syncwarp();
    int budget = R.budget;
    while (top >= 0) {
      int st = 0;
      const int c = bnb_next_child(S, B, lane, lv[top].last_start, lv[top].last_idx, &st);
      if (c < 0) {                                    // node exhausted: back to its parent
        if (top == 0) break;
        --top;
        if (lane == 0) bnb_undo(S, B, lv[top]);
        __syncwarp();
        continue;
      }
      if (budget <= 0) {
        // spill every unexplored child on the stack to the next round, deepest level first
        for (int t = top; t >= 0; --t) {
          int ls = lv[t].last_start, li = lv[t].last_idx;
          // lanes with an eligible child after (ls, li)
          int my = -1;
          if (lane < 3 * B.p) {
            my = bnb_start(S, B, lane / 3, lane_type(lane));
            if (my >= 0 && (my < ls || (my == ls && lane <= li))) my = -1;
          }
          const unsigned bal = __ballot_sync(0xffffffffu, my >= 0);
          const int cnt = __popc(bal);
          int at = 0;
          if (lane == 0 && cnt) at = atomicAdd(R.next_n, cnt);
          at = __shfl_sync(0xffffffffu, at, 0);
          const int slot = at + __popc(bal & ((1u << lane) - 1));
          if (my >= 0 && slot >= R.front_cap) atomicExch(&C.incomplete, 1);   // frontier full: item dropped
          else if (my >= 0) {
            unsigned char* ne = R.next + (long long)slot * R.front_stride;
            reinterpret_cast<int*>(ne)[0] = inst;
            reinterpret_cast<int*>(ne)[1] = S.depth + 1;
            for (int k = 0; k < S.depth; ++k) ne[8 + k] = path[k];
            ne[8 + S.depth] = (unsigned char)((lane / 3) * 3 + lane_type(lane));
          }
          __syncwarp();
          if (t > 0) { if (lane == 0) bnb_undo(S, B, lv[t - 1]); __syncwarp(); }
        }
        break;
      }
      --budget;
      if (lane == 0) {
        lv[top].last_start = st;
        lv[top].last_idx = c;
        bnb_append(S, B, c / 3, lane_type(c), st, lv[top], path);
      }
      __syncwarp();
      if (visit()) {
        ++top;
        if (lane == 0) { lv[top].last_start = -1; lv[top].last_idx = -1; }
        __syncwarp();
      } else {
        if (lane == 0) bnb_undo(S, B, lv[top]);
        __syncwarp();
      }
    }
    (void)base;
    if (lane == 0) { atomicAdd(&C.nodes, (unsigned long long)nodes); atomicAdd(R.nodes_total, (unsigned long long)nodes); }
    __syncwarp();
  }
}

// items left in a frontier mark their instance incomplete (the host stopped the search)
__global__ void k_bnb_mark(const unsigned char* __restrict__ front, int n, int stride, BCtl* __restrict__ ctl) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) atomicExch(&ctl[reinterpret_cast<const int*>(front + (long long)i * stride)[0]].incomplete, 1);
}

__global__ void k_bnb_finish(const BInst* __restrict__ bi, const BCtl* __restrict__ ctl,
                             const unsigned char* __restrict__ best_plan, int n, int stage_stride, int words,
                             uint32_t* __restrict__ ops, uint16_t* __restrict__ len, int32_t* __restrict__ makespan,
                             int32_t* __restrict__ status, int32_t* __restrict__ bound, long long* __restrict__ nodes) {
  const int i = blockIdx.x;
  const BInst& B = bi[i];
  const BCtl& C = ctl[i];
  const bool ok = B.ok;
  const bool found = ok && C.has_plan;
  for (int r = threadIdx.x; r < stage_stride; r += blockDim.x) {
    const bool on = found && r < B.p;
    const int L = on ? 3 * B.m : 0;
    len[(long long)i * stage_stride + r] = (uint16_t)L;
    for (int k = 0; k < words; ++k) {
      uint32_t wv = 0;
      for (int b = 0; b < 16; ++b) {
        const int idx = 16 * k + b;
        if (idx < L) wv |= (uint32_t)best_plan[(long long)i * BP * 3 * BM + r * 3 * BM + idx] << (2 * b);
      }
      ops[((long long)i * words + k) * stage_stride + r] = wv;
    }
  }
  if (threadIdx.x == 0) {
    makespan[i] = found ? C.best : -1;
    status[i] = !ok ? CPI_OVERFLOW : (!found ? (C.incomplete ? CPI_INCOMPLETE : CPI_DEADLOCK)
                                             : (C.incomplete ? CPI_INCOMPLETE : 0));
    if (bound) bound[i] = !ok ? -1 : (C.incomplete ? C.root_bound : (found ? C.best : C.root_bound));
    if (nodes) nodes[i] = (long long)C.nodes;
  }
}

// ---------------------------------------------------------------------------------------------- host
static size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

BnbLayout bnb_layout(int n, int lmax, int vlen_max, int front_cap, long long table_cap) {
  BnbLayout Lo;
  Lo.front_stride = (int)((8 + lmax + 15) & ~15);
  Lo.table_stride = (int)((32 + 4 * vlen_max + 15) & ~15);
  size_t o = 0;
  Lo.off_bi = o; o += al256(sizeof(BInst) * (size_t)n);
  Lo.off_ctl = o; o += al256(sizeof(BCtl) * (size_t)n);
  Lo.off_plan = o; o += al256((size_t)n * BP * 3 * BM);
  Lo.off_cnt = o; o += 256;
  Lo.off_front0 = o; o += al256((size_t)front_cap * Lo.front_stride);
  Lo.off_front1 = o; o += al256((size_t)front_cap * Lo.front_stride);
  Lo.off_table = o; o += al256((size_t)n * table_cap * Lo.table_stride);
  Lo.bytes = o;
  return Lo;
}

int launch_bnb(const cp_inst_v1* inst, int n, const int32_t* upper, int lmax, int vlen_max, int front_cap,
               long long table_cap, int budget, long long max_nodes, int max_rounds, void* ws, int stage_stride,
               int words, uint32_t* ops, uint16_t* len, int32_t* makespan, int32_t* status, int32_t* bound,
               long long* nodes_out, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const BnbLayout Lo = bnb_layout(n, lmax, vlen_max, front_cap, table_cap);
  unsigned char* base = static_cast<unsigned char*>(ws);
  BInst* bi = reinterpret_cast<BInst*>(base + Lo.off_bi);
  BCtl* ctl = reinterpret_cast<BCtl*>(base + Lo.off_ctl);
  unsigned char* plan = base + Lo.off_plan;
  int* cnt = reinterpret_cast<int*>(base + Lo.off_cnt);              // [0] front_n, [1] head, [2] next_n
  unsigned long long* ncount = reinterpret_cast<unsigned long long*>(base + Lo.off_cnt + 16);
  unsigned char* fr[2] = {base + Lo.off_front0, base + Lo.off_front1};
  unsigned char* table = base + Lo.off_table;
  cudaError_t e;
  if ((e = cudaMemsetAsync(cnt, 0, 256, st)) != cudaSuccess) return (int)e;
  if ((e = cudaMemsetAsync(plan, 0, (size_t)n * BP * 3 * BM, st)) != cudaSuccess) return (int)e;
  if ((e = cudaMemsetAsync(table, 0, (size_t)n * table_cap * Lo.table_stride, st)) != cudaSuccess) return (int)e;
  k_bnb_prep<<<(n + 127) / 128, 128, 0, st>>>(inst, n, upper, bi, ctl, fr[0], Lo.front_stride, cnt);
  if ((e = cudaGetLastError()) != cudaSuccess) return (int)e;
  alignas(8) int h_cnt[6] = {0, 0, 0, 0, 0, 0};                                 // ints 4-5: the node counter
  if ((e = cudaMemcpyAsync(h_cnt, cnt, sizeof(h_cnt), cudaMemcpyDeviceToHost, st)) != cudaSuccess) return (int)e;
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return (int)e;
  const size_t per_warp = (sizeof(BState) + lmax * sizeof(BLevel) + lmax + 4 * (3 * BP + 2 * BP * BM) + 15) & ~size_t(15);
  const size_t smem = per_warp * kBnbWarps;
  if (smem > 48 * 1024 && (e = cudaFuncSetAttribute(k_bnb_round, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) != cudaSuccess)
    return (int)e;
  int bps = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_bnb_round, 32 * kBnbWarps, smem);
  bps = bps > 0 ? bps : 1;
  const int sms = device_sm_count();
  int cur = 0, front_n = h_cnt[0];
  long long nodes_total = 0;
  for (int round = 0; front_n > 0; ++round) {
    if (round >= max_rounds || nodes_total >= max_nodes) {
      k_bnb_mark<<<(front_n + 255) / 256, 256, 0, st>>>(fr[cur], front_n, Lo.front_stride, ctl);
      break;
    }
    if ((e = cudaMemsetAsync(cnt + 1, 0, 2 * sizeof(int), st)) != cudaSuccess) return (int)e;
    BnbRound R;
    R.bi = bi; R.ctl = ctl; R.best_plan = plan;
    R.front = fr[cur]; R.front_n = front_n; R.front_head = cnt + 1;
    R.next = fr[cur ^ 1]; R.next_n = cnt + 2;
    R.front_cap = front_cap; R.front_stride = Lo.front_stride;
    R.table = table; R.table_cap = table_cap; R.table_stride = Lo.table_stride; R.max_probe = 4096;
    R.budget = budget; R.Lmax = lmax; R.nodes_total = ncount;
    const long long want = ((long long)front_n + kBnbWarps - 1) / kBnbWarps;
    const int blocks = (int)(want < (long long)sms * bps ? want : (long long)sms * bps);
    k_bnb_round<<<blocks, 32 * kBnbWarps, smem, st>>>(R);
    if ((e = cudaGetLastError()) != cudaSuccess) return (int)e;
    if ((e = cudaMemcpyAsync(h_cnt, cnt, sizeof(h_cnt), cudaMemcpyDeviceToHost, st)) != cudaSuccess) return (int)e;
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return (int)e;
    nodes_total = (long long)(*reinterpret_cast<unsigned long long*>(h_cnt + 4));
    front_n = h_cnt[2] < front_cap ? h_cnt[2] : front_cap;
    cur ^= 1;
  }
  k_bnb_finish<<<n, 32, 0, st>>>(bi, ctl, plan, n, stage_stride, words, ops, len, makespan, status, bound, nodes_out);
  return (int)cudaGetLastError();
}

}  // namespace cpk
