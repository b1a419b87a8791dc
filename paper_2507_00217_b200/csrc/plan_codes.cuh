// plan_codes.cuh -- the 2-bit code at position `pos` of stage s's row of a static plan family,
// computed arithmetically (no storage): the sweep's static candidates (k_engine<SWEEP>) and
// cp_build_static (build.cu) share it.  Layouts (PAPER.md Table tab:ppschedules :468-473):
//   CP_PLAN_GPIPE (Q22): F x m, then B x m.
//   CP_PLAN_1F1B  (Q23): F x w, (F, B) x (m - w), B x w with w = min(p - s - 1, m).
//   CP_PLAN_ZBH1  (Q31): F x w (w = min(p - s, m)); for k = 0..m-1: D_k, W_{k-s} if k >= s,
//                        the next F if one remains; then the W blocks still owed.
#pragma once
#include "crosspipe.h"

namespace cpk {

__host__ __device__ __forceinline__ int plan_row_len(int kind, int m) {
  return kind == CP_PLAN_ZBH1 ? 3 * m : (kind == CP_PLAN_IV1F1B ? 4 * m : 2 * m);
}
__host__ __device__ __forceinline__ int plan_entry_bits(int kind) { return kind == CP_PLAN_IV1F1B ? 4 : 2; }

__host__ __device__ __forceinline__ int plan_code(int kind, int s, int p, int m, int pos) {
  if (kind == CP_PLAN_GPIPE) return pos < m ? (int)CP_OP_F : (int)CP_OP_B;
  if (kind == CP_PLAN_IV1F1B) {
    // 4-bit entries type | chunk << 2 (Q34): w forward units, (forward, backward) pairs, backward units;
    // forward unit u is chunk (u / p) % 2, backward unit u chunk 1 - (u / p) % 2
    const int w = (2 * (p - s - 1) + p) < 2 * m ? (2 * (p - s - 1) + p) : 2 * m;
    int u, fw;
    if (pos < w) { u = pos; fw = 1; }
    else {
      const int q = pos - w;
      if (q < 2 * (2 * m - w)) { fw = !(q & 1); u = fw ? w + (q >> 1) : (q >> 1); }
      else { fw = 0; u = (2 * m - w) + (q - 2 * (2 * m - w)); }
    }
    const int c = (u / p) % 2;
    return fw ? ((int)CP_OP_F | (c << 2)) : ((int)CP_OP_B | ((1 - c) << 2));
  }
  if (kind == CP_PLAN_1F1B) {
    const int w = (p - s - 1) < m ? (p - s - 1) : m;
    const int q = pos - w;
    if (q < 0) return (int)CP_OP_F;
    if (q < 2 * (m - w)) return (q & 1) ? (int)CP_OP_B : (int)CP_OP_F;
    return (int)CP_OP_B;
  }
  // ZB-H1: after the warm-up, block k holds D, then W if k >= s, then F if k < m - w; in k-order
  // the blocks fall into three runs of equal shape: k < lo, lo <= k < hi, hi <= k < m
  const int w = (p - s) < m ? (p - s) : m;
  int q = pos - w;
  if (q < 0) return (int)CP_OP_F;
  const int a = s < m ? s : m;             // first block with a W
  const int b = m - w;                     // first block without an F
  const int lo = a < b ? a : b, hi = a < b ? b : a;
  if (q < 2 * lo) return (q & 1) ? (int)CP_OP_F : (int)CP_OP_D;           // (D, F)
  q -= 2 * lo;
  if (a <= b) {                                                           // (D, W, F)
    if (q < 3 * (hi - lo)) { const int t = q % 3; return t == 0 ? (int)CP_OP_D : (t == 1 ? (int)CP_OP_W : (int)CP_OP_F); }
    q -= 3 * (hi - lo);
  } else {                                                                // (D)
    if (q < hi - lo) return (int)CP_OP_D;
    q -= hi - lo;
  }
  if (q < 2 * (m - hi)) return (q & 1) ? (int)CP_OP_W : (int)CP_OP_D;    // (D, W)
  return (int)CP_OP_W;                                                    // owed W blocks
}

}  // namespace cpk
