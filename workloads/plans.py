"""Random valid plans (config 4 workload) -- ctypes wrapper of gen.cu (host or device).

Input generation only (see gen.cu header).  The packed output format is the documented
2-bit plan layout; unpack with workloads.unpack_plans for the oracle side.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "libcpgen.so")
_lib = None


def build():
    src = os.path.join(_HERE, "gen.cu")
    if not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(src):
        subprocess.check_call(["make", "-s", "-C", _HERE])
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        P32 = C.POINTER(C.c_int32)
        L.cpgen_plans_host.restype = C.c_int
        L.cpgen_plans_host.argtypes = [C.c_int, C.c_int, C.c_int, P32, P32, P32, P32, C.c_uint64, C.c_uint64,
                                       C.c_int, C.c_longlong, C.c_void_p, C.c_void_p, C.c_int, C.c_int]
        L.cpgen_plans_device.restype = C.c_int
        L.cpgen_plans_device.argtypes = [C.c_int, C.c_int, C.c_int, P32, P32, P32, P32, C.c_uint64, C.c_uint64,
                                         C.c_int, C.c_longlong, C.c_void_p, C.c_void_p, C.c_int, C.c_int,
                                         C.c_void_p, C.c_void_p]
        L.cpgen_wave_plans_host.restype = C.c_int
        L.cpgen_wave_plans_host.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_uint64, C.c_int, C.c_longlong,
                                            C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int]
        L.cpgen_wave_plans_device.restype = C.c_int
        L.cpgen_wave_plans_device.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_uint64, C.c_int,
                                              C.c_longlong, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_void_p,
                                              C.c_void_p, C.c_int]
        _lib = L
    return _lib


def _mem_arrays(batch, i=0):
    p = int(batch.p[i])
    arrs = [np.ascontiguousarray(np.asarray(getattr(batch, k))[i, :p], dtype=np.int32)
            for k in ("m_f", "m_d", "m_w", "m_lim")]
    return arrs, [a.ctypes.data_as(C.POINTER(C.c_int32)) for a in arrs]


def words_for(batch, i=0):
    return ((2 + int(batch.n_sub[i])) * int(batch.m[i]) + 15) // 16


def plans_host(batch, n, seed, id0=0, q=1, stride=None, i=0):
    """n random valid plans of instance i (host).  Returns (ops uint32 [n, words, stride], len uint16 [n, stride])."""
    p, m, ns = int(batch.p[i]), int(batch.m[i]), int(batch.n_sub[i])
    stride = stride or p
    words = words_for(batch, i)
    ops = np.zeros((n, words, stride), dtype=np.uint32)
    ln = np.zeros((n, stride), dtype=np.uint16)
    keep, ptrs = _mem_arrays(batch, i)
    err = lib().cpgen_plans_host(p, m, ns, *ptrs, seed, id0, q, n, ops.ctypes.data, ln.ctypes.data, words, stride)
    if err:
        raise RuntimeError(f"plan generator failed on {err} plans")
    return ops, ln


def plans_device(batch, n, seed, id0=0, q=1, stride=None, i=0, device="cuda"):
    """Same plans generated on the GPU (bench-scale workloads).  Returns torch tensors."""
    import torch
    p, m, ns = int(batch.p[i]), int(batch.m[i]), int(batch.n_sub[i])
    stride = stride or p
    words = words_for(batch, i)
    ops = torch.zeros((n, words, stride), dtype=torch.int32, device=device)
    ln = torch.zeros((n, stride), dtype=torch.int16, device=device)
    err = torch.zeros(1, dtype=torch.int32, device=device)
    keep, ptrs = _mem_arrays(batch, i)
    rc = lib().cpgen_plans_device(p, m, ns, *ptrs, seed, id0, q, n, ops.data_ptr(), ln.data_ptr(), words, stride,
                                  err.data_ptr(), torch.cuda.current_stream().cuda_stream)
    if rc:
        raise RuntimeError(f"cpgen launch failed: {rc}")
    if int(err.item()):
        raise RuntimeError(f"plan generator failed on {int(err.item())} plans")
    return ops, ln


def wave_words(p, m, n_sub=1):
    return (2 * (2 + n_sub) * m + 7) // 8


def wave_plans_host(p, m, n_sub, n, seed, id0=0, q=1, stride=None, loop=False):
    """n random valid Wave (reading Q32) or, loop=True, Loop (Q33) plans, 4-bit entries (host).  Returns
    (ops uint32 [n, words, stride], len uint16 [n, stride])."""
    stride = stride or p
    words = wave_words(p, m, n_sub)
    ops = np.zeros((n, words, stride), dtype=np.uint32)
    ln = np.zeros((n, stride), dtype=np.uint16)
    err = lib().cpgen_wave_plans_host(p, m, n_sub, seed, id0, q, n, ops.ctypes.data, ln.ctypes.data, words, stride,
                                      int(loop))
    if err:
        raise RuntimeError(f"wave plan generator failed on {err} plans")
    return ops, ln


def wave_plans_device(p, m, n_sub, n, seed, id0=0, q=1, stride=None, device="cuda", loop=False):
    """Same Wave / Loop plans generated on the GPU.  Returns torch tensors."""
    import torch
    stride = stride or p
    words = wave_words(p, m, n_sub)
    ops = torch.zeros((n, words, stride), dtype=torch.int32, device=device)
    ln = torch.zeros((n, stride), dtype=torch.int16, device=device)
    err = torch.zeros(1, dtype=torch.int32, device=device)
    rc = lib().cpgen_wave_plans_device(p, m, n_sub, seed, id0, q, n, ops.data_ptr(), ln.data_ptr(), words, stride,
                                       err.data_ptr(), torch.cuda.current_stream().cuda_stream, int(loop))
    if rc:
        raise RuntimeError(f"cpgen launch failed: {rc}")
    if int(err.item()):
        raise RuntimeError(f"wave plan generator failed on {int(err.item())} plans")
    return ops, ln
