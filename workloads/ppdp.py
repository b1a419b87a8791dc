"""E2 scenario inputs: cross-DC PP vs cross-DC DP for Llama-3-405B (§5.2 :503-516,
Appendix E :855-858; reading Q36 in DESIGN.md).

Input generation and the scenario's closed-form costs only; the schedules are evaluated by the
product kernels (tools/e2_ppdp.py) or by the oracle (tests/test_ppdp.py).

- Model: Llama 3 405B (126 layers, d = 16384, FFN 53248, 128 query / 8 KV heads), n_TP = 8,
  n_PP = 16, n_DP = 64, s = 8192, b = 1, GBS = 2 n_PP n_DP (App. E :856), 2 DCs with the GPUs split
  evenly (:857).  Embedding and output layers count as transformer layers (§6.1), so each
  stage holds (126 + 2) / 16 = 8 layers.
- T_layer = C_layer / (P_GPU n_TP) with P_GPU = 500 TFLOP/s (App. E :857).  C_layer = forward FLOPs of
  one layer: 2 b s P_layer for the weight matmuls plus 2 b s^2 d for causal attention (QK^T and AV,
  half of the full 4 b s^2 d).  This gives T_F = 8 T_layer = 108.8 ms, the paper's anchor (:507,
  "T_F ~ 109 ms").  D and W each cost one forward (the backward is twice the forward).
- PP message per cross-DC transfer: b s d n_DP * 2 bytes: all n_DP pipelines cross
  the same DC boundary.
- DP cost: 2 alpha + 2 N beta with beta the per-parameter time of BF16 gradients, 2 bytes / bandwidth
  (App. E :858 "the extra factor 2 in the bandwidth term comes from the size of the BF16 datatype";
  SPEC.md:466 "BF16 factor folded"), i.e. 4N bytes at the link bandwidth (reading Q36).
"""
from __future__ import annotations

from . import configs as K

LLAMA3_405B = dict(layers=126, d=16384, ffn=53248, heads=128, kv_heads=8, s=8192, b=1, n_tp=8, n_pp=16, n_dp=64,
                   p_gpu=500e12, n_params=405e9)

BANDWIDTHS_GBS = [4, 8, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096]   # GB/s (Fig. cross_dc_dp_or_pp, and beyond)
LATENCIES_MS = [4, 8, 16, 32, 64, 128]                            # ms (:507 "ranging from 4-128 ms")
TICK_S = 1e-4                                                     # 0.1 ms ticks: t_PP <= ~150 s fits int32


def layer_params(c=LLAMA3_405B) -> int:
    d, hd = c["d"], c["d"] // c["heads"]
    return 2 * d * d + 2 * d * c["kv_heads"] * hd + 3 * d * c["ffn"]      # q, o, k, v, gate/up/down


def layer_flops(c=LLAMA3_405B) -> float:
    b, s, d = c["b"], c["s"], c["d"]
    return 2.0 * b * s * layer_params(c) + 2.0 * b * s * s * d


def stage_forward_s(c=LLAMA3_405B) -> float:
    layers_per_stage = (c["layers"] + 2) / c["n_pp"]
    return layers_per_stage * layer_flops(c) / (c["p_gpu"] * c["n_tp"])


def n_microbatches(c=LLAMA3_405B) -> int:
    return 2 * c["n_pp"] * c["n_dp"] // (c["n_dp"] * c["b"])               # GBS / (n_DP b) = 2 n_PP


def pp_message_bytes(c=LLAMA3_405B) -> int:
    return c["b"] * c["s"] * c["d"] * c["n_dp"] * 2


def dp_cost_s(alpha_s: float, bw_bytes_s: float, c=LLAMA3_405B) -> float:
    """Unoverlapped cross-DC DP cost 2 alpha + 2 N beta, beta = 2 bytes / bandwidth (Q36)."""
    return 2.0 * alpha_s + 2.0 * c["n_params"] * (2.0 / bw_bytes_s)


def dp_cost_literal_s(alpha_s: float, bw_bytes_s: float, c=LLAMA3_405B) -> float:
    """App. E :858 read literally: 2 x (alpha + 2 x N/2 x beta) with beta the time of ONE byte -- each of
    the two rounds moves N/2 parameters of 2 bytes, 2N bytes in total (half of Q36's 4N)."""
    return 2.0 * alpha_s + 2.0 * c["n_params"] / bw_bytes_s


def ticks(seconds: float, tick_s: float = TICK_S) -> int:
    return int(seconds / tick_s + 0.5)


def pp_instance(alpha_s: float, bw_bytes_s: float, n_sub: int = 1, c=LLAMA3_405B, tick_s: float = TICK_S):
    """Cross-DC PP, UD pattern: p = 16 over 2 DCs (8 + 8), m = 32, F = D = W = T_F, the DC boundary
    carries (alpha, message / bandwidth) both ways; memory budget = the 1F1B peak (PAPER.md:491
    "same memory limits as their static counterparts")."""
    tf = ticks(stage_forward_s(c), tick_s)
    return K.uniform_instance(c["n_pp"], n_microbatches(c), 2, tf, tf, tf, lat=ticks(alpha_s, tick_s),
                              bw=ticks(pp_message_bytes(c) / bw_bytes_s, tick_s), mlim_x1000=1000, n_sub=n_sub,
                              tick_s=tick_s)


def wave_instance(alpha_s: float, bw_bytes_s: float, c=LLAMA3_405B, tick_s: float = TICK_S):
    """The same stage as two half-cost chunks on the Wave pattern (ZBV, reading Q35): chunk blocks
    T_F / 2, activation freed by W, budget 2p chunk activations (= the 1F1B budget)."""
    th = ticks(stage_forward_s(c) / 2, tick_s)
    return K.uniform_instance(c["n_pp"], n_microbatches(c), 2, th, th, th, m_f=1, m_d=0, m_w=-1, mlim_x1000=2000,
                              lat=ticks(alpha_s, tick_s), bw=ticks(pp_message_bytes(c) / bw_bytes_s, tick_s),
                              tick_s=tick_s)
