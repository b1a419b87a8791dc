"""ctypes loader + struct mirrors of include/crosspipe.h (ABI v2).

Fails loudly: there is no CPU fallback anywhere in this package.  If the in-tree
libcrosspipe.so is missing, build it with `python -c "import __graft_entry__ as g; g.build()"`.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CROSSPIPE_LIB") or os.path.join(_HERE, "libcrosspipe.so")   # override: debug build

CP_OK, CP_EINVAL, CP_EUNSUPPORTED, CP_ECUDA, CP_EWORKSPACE = 0, -1, -2, -3, -4
CPI_DEADLOCK, CPI_MEM_EXCEEDED, CPI_BAD_PLAN, CPI_BAD_INSTANCE, CPI_OVERFLOW = 1, 2, 4, 8, 16
GRID_MAX_AXIS, GRID_MAX_SMALL = 128, 16

# numpy mirror of cp_inst_v1 (1792 B)
INST_DTYPE = np.dtype([
    ("n_pp", "u1"), ("n_dc", "u1"), ("n_sub", "u1"), ("flags", "u1"),
    ("n_mb", "<u2"), ("version", "<u2"), ("tick_ns", "<i4"),
    ("dc_first_stage", "u1", 4), ("_pad0", "u1", 16),
    ("t_f", "<i4", 32), ("t_d", "<i4", 32), ("t_w", "<i4", 32),
    ("m_f", "<i4", 32), ("m_d", "<i4", 32), ("m_w", "<i4", 32), ("m_lim", "<i4", 32),
    ("t_dp", "<i4", 32), ("t_ag", "<i4", 32),
    ("lat_f", "<i4", 32), ("bw_f", "<i4", 32), ("lat_b", "<i4", 32), ("bw_b", "<i4", 32),
    ("_tail", "u1", 96),
])
assert INST_DTYPE.itemsize == 1792


class CpInstV1(C.Structure):
    _fields_ = [("raw", C.c_uint8 * 1792)]


class CpInstances(C.Structure):
    _fields_ = [("n", C.c_int32), ("max_pp", C.c_int32), ("max_mb", C.c_int32), ("ring_hint", C.c_int32),
                ("inst", C.c_void_p)]


class CpSchedules(C.Structure):
    _fields_ = [("n", C.c_int32), ("stage_stride", C.c_int32), ("words", C.c_int32), ("pattern", C.c_int32),
                ("inst_of", C.c_void_p), ("ops", C.c_void_p), ("len", C.c_void_p)]


class CpResults(C.Structure):
    _fields_ = [("makespan", C.c_void_p), ("peak_mem", C.c_void_p), ("status", C.c_void_p),
                ("stage_stats", C.c_void_p), ("t_start", C.c_void_p), ("len_stride", C.c_int32),
                ("index_base", C.c_int32), ("best_key", C.c_void_p)]


class CpGrid(C.Structure):
    _fields_ = [("base", CpInstV1), ("n_dc", C.c_int32),
                ("n_pp_vals", C.c_int32 * 8), ("n_pp_n", C.c_int32),
                ("n_mb_vals", C.c_int32 * 8), ("n_mb_n", C.c_int32),
                ("lat", C.c_int32 * GRID_MAX_AXIS), ("n_lat", C.c_int32),
                ("bw", C.c_int32 * GRID_MAX_AXIS), ("n_bw", C.c_int32),
                ("mlim_x1000", C.c_int32 * GRID_MAX_SMALL), ("n_mem", C.c_int32),
                ("tdp", C.c_int32 * GRID_MAX_SMALL), ("n_dp", C.c_int32),
                ("cand_mask", C.c_uint32)]


_D32 = C.c_double * 32


class CpSpecSI(C.Structure):
    _fields_ = [("n_pp", C.c_int32), ("n_mb", C.c_int32), ("n_sub", C.c_int32), ("zero1", C.c_int32),
                ("n_dc", C.c_int32), ("dc_of_stage", C.c_int32 * 32)] + [
        (k, _D32) for k in ("t_f", "t_d", "t_w", "m_f", "m_d", "m_w", "m_lim", "t_dp", "t_ag")] + [
        ("alpha", (C.c_double * 4) * 4), ("beta", (C.c_double * 4) * 4),
        ("msg_f", _D32), ("msg_b", _D32), ("tick_s", C.c_double), ("mem_unit", C.c_double)]


EXPORTS = ("cp_abi_version", "cp_status_string", "cp_workspace_bytes", "cp_simulate", "cp_greedy",
           "cp_build_static", "cp_sweep_shard", "cp_sweep_shard_rank", "cp_sweep_partition", "cp_quantize",
           "cp_validate_instance", "cp_exact", "cp_exact_workspace_bytes", "cp_exact_bnb",
           "cp_exact_bnb_workspace_bytes")
ABI_VERSION = 3
N_CAND = 6                    # sweep candidates: 0 GPipe, 1 1F1B, 2/3/4 greedy n_sub 1/2/4, 5 ZB-H1
PLAN_KINDS = {"gpipe": 0, "1f1b": 1, "zbh1": 5, "iv1f1b": 6, "zbv": 7}   # iv1f1b: Loop, zbv: Wave plans (4-bit)

_lib = None


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"CrossPipe CUDA library not built: {LIB_PATH} missing "
                          "(run __graft_entry__.build()); there is no CPU fallback")
    L = C.CDLL(LIB_PATH)
    P = C.POINTER
    L.cp_abi_version.restype = C.c_uint32
    L.cp_status_string.restype = C.c_char_p
    L.cp_status_string.argtypes = [C.c_int32]
    L.cp_workspace_bytes.restype = C.c_size_t
    L.cp_workspace_bytes.argtypes = [C.c_int32, C.c_void_p, C.c_int64]
    L.cp_simulate.restype = C.c_int32
    L.cp_simulate.argtypes = [P(CpInstances), P(CpSchedules), P(CpResults), C.c_void_p, C.c_size_t, C.c_void_p]
    L.cp_greedy.restype = C.c_int32
    L.cp_greedy.argtypes = [P(CpInstances), P(CpSchedules), P(CpResults), C.c_void_p, C.c_size_t, C.c_void_p]
    L.cp_build_static.restype = C.c_int32
    L.cp_build_static.argtypes = [C.c_int32, P(CpInstances), P(CpSchedules), C.c_void_p]
    L.cp_sweep_shard.restype = C.c_int32
    L.cp_sweep_shard.argtypes = [P(CpGrid), C.c_int64, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p,
                                 C.c_size_t, C.c_void_p]
    L.cp_sweep_shard_rank.restype = C.c_int32
    L.cp_sweep_shard_rank.argtypes = [P(CpGrid), C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                      C.c_size_t, C.c_void_p]
    L.cp_sweep_partition.restype = C.c_int32
    L.cp_sweep_partition.argtypes = [P(CpGrid), C.c_int32, P(C.c_int64)]
    L.cp_exact_workspace_bytes.restype = C.c_size_t
    L.cp_exact_workspace_bytes.argtypes = [C.c_int32, C.c_int32]
    L.cp_exact.restype = C.c_int32
    L.cp_exact.argtypes = [P(CpInstances), P(CpSchedules), C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int64,
                           C.c_void_p, C.c_size_t, C.c_void_p]
    L.cp_exact_bnb_workspace_bytes.restype = C.c_size_t
    L.cp_exact_bnb_workspace_bytes.argtypes = [P(CpInstances), C.c_int32, C.c_int64]
    L.cp_exact_bnb.restype = C.c_int32
    L.cp_exact_bnb.argtypes = [P(CpInstances), P(CpSchedules), C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                               C.c_void_p, C.c_int32, C.c_int64, C.c_int32, C.c_int32, C.c_int64, C.c_void_p,
                               C.c_size_t, C.c_void_p]
    L.cp_quantize.restype = C.c_int32
    L.cp_quantize.argtypes = [P(CpSpecSI), C.c_void_p]
    L.cp_validate_instance.restype = C.c_int32
    L.cp_validate_instance.argtypes = [C.c_void_p, C.c_char_p, C.c_size_t]
    if L.cp_abi_version() != ABI_VERSION:
        raise ImportError("libcrosspipe ABI version mismatch")
    _lib = L
    return L


def check(rc: int, what: str):
    if rc != CP_OK:
        msg = load().cp_status_string(rc).decode()
        raise RuntimeError(f"{what} failed: rc={rc} ({msg})")
