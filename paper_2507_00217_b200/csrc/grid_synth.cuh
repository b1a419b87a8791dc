// grid_synth.cuh -- sweep grid point -> per-lane instance fields, shared by the sweep paths of
// k_engine<MODE_SWEEP> (engine.cu) and k_greedy_fast<W, true> (greedy_fast.cu), so both evaluate
// exactly the same instance for a point.
//
// Point index (mixed radix, i_dp fastest): ((((i_pp * n_mb + i_mb) * n_lat + i_lat) * n_bw + i_bw)
// * n_mem + i_mem) * n_dp + i_dp.  Stages split evenly and contiguously over n_dc DCs: stage s
// sits in DC s*ndc/p; a boundary whose two stages sit in different DCs carries the point's
// (latency, T_bw) in both directions, every other boundary is zero-delay.
// M_L = round(x/1000 * p * m_f) (reading Q9).
#pragma once
#include <stdint.h>

#include "crosspipe.h"

namespace cpk {

constexpr unsigned long long KEY_NONE = 0x7fffffffffffffffull;   // no feasible candidate (INT64_MAX)
constexpr unsigned long long KEY_OVER = 0x7ffffffffffffffeull;   // point not evaluated (CPI_OVERFLOW)

struct GridLane {      // one lane's (stage's) view of a synthesized instance
  int p, m, zero1;
  int tf, td, tw, mf, md, mw, mlim, tdp, tag;
  int latF, bwF, latB, bwB;       // s -> s+1 (F) and s -> s-1 (D) link delays
};

// host + device: the host validates every synthesized instance class in check_grid (abi.cpp)
__host__ __device__ __forceinline__ GridLane grid_lane(const cp_grid& G, long long point, int s) {
  GridLane g = {};
  long long k = point;
  const int i_dp = (int)(k % G.n_dp); k /= G.n_dp;
  const int i_mem = (int)(k % G.n_mem); k /= G.n_mem;
  const int i_bw = (int)(k % G.n_bw); k /= G.n_bw;
  const int i_lat = (int)(k % G.n_lat); k /= G.n_lat;
  const int i_mb = (int)(k % G.n_mb_n); k /= G.n_mb_n;
  const int i_pp = (int)k;
  g.p = G.n_pp_vals[i_pp];
  g.m = G.n_mb_vals[i_mb];
  g.zero1 = G.base.flags & 1;
  const int ndc = G.n_dc < g.p ? G.n_dc : g.p;
  if (s < g.p) {
    g.tf = G.base.t_f[s]; g.td = G.base.t_d[s]; g.tw = G.base.t_w[s];
    g.mf = G.base.m_f[s]; g.md = G.base.m_d[s]; g.mw = G.base.m_w[s];
    g.mlim = (int)(((long long)G.mlim_x1000[i_mem] * g.p * g.mf + 500) / 1000);
    g.tdp = G.tdp[i_dp];
    g.tag = G.base.t_ag[s];
    const bool xf = (s < g.p - 1) && (s * ndc / g.p != (s + 1) * ndc / g.p);
    const bool xb = (s > 0) && ((s - 1) * ndc / g.p != s * ndc / g.p);
    g.latF = xf ? G.lat[i_lat] : 0; g.bwF = xf ? G.bw[i_bw] : 0;
    g.latB = xb ? G.lat[i_lat] : 0; g.bwB = xb ? G.bw[i_bw] : 0;
  }
  return g;
}

// A launch's point set: contiguous [lo, hi) when own_hi == own_lo; otherwise the blocked ownership
// of cp_sweep_shard_rank -- blocks [lo, hi) of `inner` consecutive points, slice [own_lo, own_hi)
// of each.  sweep_npts counts it, sweep_point_of maps index j (0 <= j < npts) to a point.
struct SweepSet {
  long long lo, hi, inner;
  int own_lo, own_hi;
};
__host__ __device__ __forceinline__ long long sweep_npts(const SweepSet& q) {
  return q.own_hi > q.own_lo ? (q.hi - q.lo) * (long long)(q.own_hi - q.own_lo) : q.hi - q.lo;
}
__host__ __device__ __forceinline__ long long sweep_point_of(const SweepSet& q, long long j) {
  if (q.own_hi <= q.own_lo) return q.lo + j;
  const long long span = q.own_hi - q.own_lo;
  return (q.lo + j / span) * q.inner + q.own_lo + j % span;
}

#ifdef __CUDACC__
// (point, candidate) of sweep task t: active candidates of `mask` as the slowest axis, visited in
// reverse so the most expensive tasks (highest candidate id, largest m) start first and
// neighbouring segments of a warp get the same candidate.  Returns the point (or -1).
__device__ __forceinline__ long long sweep_task(unsigned mask, const SweepSet& q, long long t, int& cand) {
  const long long npts = sweep_npts(q);
  const long long ntask = npts * __popc(mask);
  if (t >= ntask) return -1;
  const long long tid = ntask - 1 - t;
  int ci = (int)(tid / npts);
  unsigned mm = mask;
  while (ci-- > 0) mm &= mm - 1;       // ci-th set bit of the mask
  cand = __ffs(mm) - 1;
  return sweep_point_of(q, tid % npts);
}

#endif  // __CUDACC__

}  // namespace cpk
