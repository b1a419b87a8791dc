"""CPU-side checks of the product boundary (no GPU compute): the C-ABI library loads and
exports every symbol include/crosspipe.h declares; host entry points (quantizer, validator,
sweep partition) agree with the oracle / their definitions; format conversions round-trip."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2507_00217_b200 as cp
from paper_2507_00217_b200 import _lib as L
from workloads import configs as K, pack_plans, unpack_plans

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    syms = set()
    for fn in os.listdir(os.path.join(ROOT, "include")):
        if fn.endswith(".h"):
            txt = open(os.path.join(ROOT, "include", fn)).read()
            syms |= set(re.findall(r"^\s*(?:[A-Za-z_][\w\s\*]*?)\b(cp_\w+)\s*\(", txt, flags=re.M))
    return syms


def test_library_exports_every_declared_symbol():
    syms = declared_symbols()
    assert {"cp_simulate", "cp_greedy", "cp_sweep_shard", "cp_quantize"} <= syms
    lib = C.CDLL(L.LIB_PATH)
    for s in syms:
        assert hasattr(lib, s), s
    assert set(L.EXPORTS) == syms


def test_abi_version_and_strings():
    lib = L.load()
    assert lib.cp_abi_version() == 3
    assert b"workspace" in lib.cp_status_string(-4)
    assert b"deadlock" in lib.cp_status_string(1)


def test_record_layout():
    assert L.INST_DTYPE.itemsize == 1792
    assert C.sizeof(L.CpInstances) == 24 and C.sizeof(L.CpSchedules) == 40 and C.sizeof(L.CpResults) == 56
    assert L.INST_DTYPE.fields["t_f"][1] == 32 and L.INST_DTYPE.fields["bw_b"][1] == 32 + 12 * 128


def test_validator_matches_oracle(oracle_lib):
    """cp_validate_instance (host) flags BAD_INSTANCE exactly when the oracle's validator does."""
    rng = np.random.default_rng(3)
    batch = K.random_instances(300, seed=4, max_p=8, max_m=6)
    for i in range(len(batch)):
        if rng.random() < 0.7:
            k = int(rng.integers(7)); s = int(rng.integers(batch.p[i]))
            fld = ["t_f", "t_d", "t_w", "m_f", "m_d", "m_lim", "t_ag"][k]
            getattr(batch, fld)[i, s] += int(rng.integers(-3, 2))
    recs = cp.pack_instances(batch)
    for i in range(len(batch)):
        st, msg = cp.validate_record(recs[i:i + 1])
        want = oracle_lib.lib().or_validate_instance(C.byref(oracle_lib.to_or_inst(batch.item(i))))
        assert (st == 8) == (want == 8), (i, st, want, msg)
        if st == 8:
            assert msg


def test_quantizer_matches_oracle(oracle_lib):
    """cp_quantize (product, C++) and or_quantize (oracle, C) agree bit for bit on random SI specs
    (same double arithmetic, llround half away from zero; reading Q21)."""
    rng = np.random.default_rng(5)
    for _ in range(300):
        p = int(rng.integers(1, 9)); n_dc = int(rng.integers(1, 5))
        dc = sorted(int(x) for x in rng.integers(0, n_dc, size=p))
        spec = {"p": p, "m": int(rng.integers(1, 40)), "n_sub": int(rng.integers(1, 4)), "zero1": int(rng.integers(2)),
                "n_dc": n_dc, "dc_of_stage": dc,
                "t_f": rng.uniform(1e-4, 0.1, p), "t_d": rng.uniform(1e-4, 0.1, p), "t_w": rng.uniform(1e-4, 0.1, p),
                "m_f": [2e9] * p, "m_d": [-1e9] * p, "m_w": [-1e9] * p, "m_lim": rng.uniform(2e9, 4e10, p),
                "t_dp": rng.uniform(0, 0.2, p), "t_ag": rng.uniform(0, 0.1, p),
                "alpha": rng.uniform(0, 0.1, (4, 4)).tolist(), "beta": (8 / (rng.uniform(1, 800, (4, 4)) * 1e9)).tolist(),
                "msg_f": [1e9] * p, "msg_b": [1e9] * p, "tick_s": 1e-6, "mem_unit": 1e9}
        st, rec = cp.quantize(spec)
        o = oracle_lib.quantize(spec)
        assert (st == 8) == (o["status"] == 8)
        if st == 0:
            for k in ("t_f", "t_d", "t_w", "m_f", "m_d", "m_w", "m_lim", "t_dp", "t_ag"):
                assert np.array_equal(rec[k][0, :p], o[k]), k
            for k in ("lat_f", "bw_f", "lat_b", "bw_b"):
                assert np.array_equal(rec[k][0, :p - 1], o[k]), k


def test_sweep_partition_balances_cost():
    """cp_sweep_partition cuts at equal prefix sums of p*m*sum(2+n_sub)."""
    g = K.full_sweep_grid()
    for world in (1, 2, 3, 4, 8):
        b = cp.sweep_partition(g, world)
        assert b[0] == 0 and b[-1] == g.n_points and all(x <= y for x, y in zip(b, b[1:]))
        i_pp, i_mb, *_ = g.point_axes(np.arange(g.n_points))
        cost = np.array(g.pp_vals)[i_pp] * np.array(g.mb_vals)[i_mb] * 17
        shares = [cost[b[r]:b[r + 1]].sum() for r in range(world)]
        assert max(shares) - min(shares) <= cost.max() + 1, (world, shares)


def test_pack_unpack_roundtrip():
    rng = np.random.default_rng(6)
    codes = rng.integers(0, 4, size=(5, 7, 50)).astype(np.int8)
    lens = rng.integers(0, 51, size=(5, 7)).astype(np.int32)
    ops, ln = pack_plans(codes, lens, stage_stride=8)
    c2, l2 = unpack_plans(ops, ln, p=7)
    assert np.array_equal(l2, lens)
    for i in range(5):
        for s in range(7):
            assert np.array_equal(c2[i, s, :lens[i, s]], codes[i, s, :lens[i, s]])


def test_product_has_no_oracle_dependency():
    """The product never imports / links the oracle (independence)."""
    pkg = os.path.join(ROOT, "paper_2507_00217_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cpp", ".h", ".cuh", "Makefile")):
                txt = open(os.path.join(dirpath, fn)).read()
                assert "oracle" not in txt.replace("no CPU fallback", ""), fn
    assert b"or_simulate" not in open(L.LIB_PATH, "rb").read()


def test_compute_entry_points_fail_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        cp.sweep_shard(K.gpt16_grid())


def test_argument_errors_before_any_device_work():
    """The C ABI rejects bad arguments with CP_EINVAL / CP_EWORKSPACE before touching a device
    (include/crosspipe.h error behaviour of cp_build_static and cp_exact), so these run on CPU."""
    import ctypes as C
    lib = L.load()
    fake = C.c_void_p(0x1000)                                 # never dereferenced on these paths
    inst = L.CpInstances(4, 4, 8, 0, fake.value)
    good = L.CpSchedules(4, 4, 2, 0, None, fake.value, fake.value)
    ms = st = fake
    assert lib.cp_build_static(4, C.byref(inst), C.byref(good), None) == L.CP_EINVAL          # kind 4: no static family
    assert lib.cp_build_static(7, C.byref(inst), C.byref(L.CpSchedules(4, 4, 1, 0, None, fake.value, fake.value)),
                               None) == L.CP_EINVAL                                           # ZB-V: 8 entries < 6 * max_mb
    assert lib.cp_exact(None, C.byref(good), None, ms, st, 16, 100, None, 0, None) == L.CP_EINVAL
    assert lib.cp_exact(C.byref(inst), C.byref(good), None, ms, st, 0, 100, None, 0, None) == L.CP_EINVAL   # cap < 1
    assert lib.cp_exact(C.byref(inst), C.byref(good), None, ms, st, 16, 1 << 53, None, 0, None) == L.CP_EINVAL
    assert lib.cp_exact(C.byref(inst), C.byref(L.CpSchedules(3, 4, 2, 0, None, fake.value, fake.value)), None, ms, st,
                        16, 100, None, 0, None) == L.CP_EINVAL                                # n mismatch
    assert lib.cp_exact(C.byref(inst), C.byref(good), None, ms, st, 16, 100, None, 0, None) == L.CP_EWORKSPACE
    assert lib.cp_exact_workspace_bytes(0, 16) == 0
    assert lib.cp_exact_workspace_bytes(4, 16) >= 4 * 8 * 16 * 8


def test_validator_each_invariant_through_the_abi():
    """cp_validate_instance (host side of the C ABI) rejects each single-invariant violation of
    SPEC.md:46-50 / Q10 / Q12 / Q19 that tests/test_oracle_pins.py pins on the oracle, accepts the
    adjacent valid value, and names the violated invariant."""
    from tests.test_oracle_pins import _INVARIANT_CASES
    for why, fields, stage, bad, ok in _INVARIANT_CASES:
        p0 = 32 if ("p" in fields and bad[0] > 4) else 4
        for vals, want in ((bad, 8), (ok, 0)):
            b = K.uniform_instance(p0, 3, 2, 10, 10, 10, lat=5, bw=3, mlim_x1000=1000)
            for f, x in zip(fields, vals):
                if stage is None:
                    getattr(b, f)[0] = x
                else:
                    getattr(b, f)[0, stage] = x
            st, msg = cp.validate_record(cp.pack_instances(b))
            assert st == want, (why, vals, st, msg)
            if want:
                assert msg, why


def _grid(pp=(4,), mb=(8,), mlim=(1000,), lat=(0, 50), bw=(0, 20), tdp=(0,), p_base=4, m_f=2):
    from workloads.core import Grid
    base = K.uniform_instance(p_base, 8, 2, 100, 100, 100, m_f=m_f, m_d=-(m_f // 2), m_w=-(m_f - m_f // 2))
    return Grid(base=base, n_dc=2, pp_vals=list(pp), mb_vals=list(mb), lat=np.array(lat), bw=np.array(bw),
                mlim_x1000=np.array(mlim), tdp=np.array(tdp), cand_mask=0b11111)


def test_sweep_grid_validation_through_the_abi():
    """check_grid (cp_sweep_shard / cp_sweep_shard_rank / cp_sweep_partition) rejects grids whose
    synthesized instances would be invalid with CP_EINVAL, synchronously and before any device work,
    instead of reporting their points as "no feasible candidate": a p beyond the base record's stages
    (zero durations), a memory budget below m_f, a budget beyond int32, negative axes."""
    lib = cp._lib.load()
    b = (C.c_int64 * 3)()
    assert lib.cp_sweep_partition(C.byref(cp.api.to_cp_grid(_grid())), 2, b) == 0
    bad = {
        "p beyond the base record": cp.api.to_cp_grid(_grid(pp=(4, 8))),
        "M_L < m_f": cp.api.to_cp_grid(_grid(mlim=(1000, 100))),
        "M_L beyond int32": cp.api.to_cp_grid(_grid(mlim=(1000, 2**31 - 1), m_f=1000)),
    }
    g = cp.api.to_cp_grid(_grid())
    g.lat[1] = -5
    bad["negative latency"] = g
    g = cp.api.to_cp_grid(_grid())
    g.tdp[0] = -1
    bad["negative DP time"] = g
    for why, cg in bad.items():
        assert lib.cp_sweep_partition(C.byref(cg), 2, b) == -1, why              # CP_EINVAL
        assert lib.cp_sweep_shard(C.byref(cg), 0, 1, None, None, None, 0, None) == -1, why
        assert lib.cp_sweep_shard_rank(C.byref(cg), 0, 1, None, None, None, 0, None) == -1, why


def test_sweep_workspace_covers_global_rings():
    """A grid whose in-flight bound min(m, M_L / m_f) exceeds what one block's shared memory holds
    gets global-memory rings per p-class in the sweep workspace (cp_workspace_bytes(2, grid)).
    Grids with static candidates and n_mb <= 255 also hold the per-call plan library: 64 B of task
    counters, then 3 kinds x n_pp x n_mb plans of ceil(3 max_m / 16) words x 32 rows (256-B aligned);
    every sweep workspace ends with 256 B of task counters for the long-task launches."""
    lib = cp._lib.load()
    small = cp.api.to_cp_grid(_grid())
    words = (3 * 8 + 15) // 16
    lib_bytes = (64 + 3 * 1 * 1 * words * 32 * 4 + 255) // 256 * 256
    assert lib.cp_workspace_bytes(2, C.byref(small), 0) == 256 + lib_bytes + 256
    big = cp.api.to_cp_grid(_grid(pp=(2, 4), mb=(1024,), mlim=(600000,)))
    nb = lib.cp_workspace_bytes(2, C.byref(big), 0)
    assert nb >= 256 + 2 * 148 * 4 * 2 * 1024 * 32 * 4, nb


def test_bench_kernel_register_budget():
    """The bench kernel k_chunk32f<UD> keeps 7 resident 4-warp blocks per SM only at <= 72 registers
    per thread; small source changes have pushed it to 78 (6 blocks, -5% on config 4),
    so the built library is checked here (cuobjdump, no GPU needed)."""
    import shutil
    import subprocess
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([tool, "--dump-resource-usage", L.LIB_PATH], capture_output=True, text=True).stdout
    m = re.search(r"Function _ZN3cpk10k_chunk32fILi0ELb0EEEvNS_4ArgsE:\s*\n\s*REG:(\d+)", out)
    assert m, "k_chunk32f<UD, no timeline> not found in the library"
    assert int(m.group(1)) <= 72, f"k_chunk32f<UD> uses {m.group(1)} registers (> 72: 6 instead of 7 blocks per SM)"
