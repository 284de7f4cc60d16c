"""CPU checks of the C ABI library and the Python host mirror: the library
loads, exports every symbol include/parsweep_b200.h declares, and the
host-only logic (partition helpers, validation, the preliminary's error
behaviour) matches the reference — no device compute is issued here."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT, load_golden
from oracle.pyoracle import OracleError


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "parsweep_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(psw_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol(psw):
    L = psw.lib()
    names = declared_symbols()
    assert len(names) >= 20
    missing = [s for s in names if not hasattr(L, s)]
    assert not missing, missing


def test_library_is_sm100a_cuda(psw):
    # the .so carries sm_100a SASS (cuobjdump lists the ELF arch)
    import shutil
    import subprocess
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump unavailable")
    out = subprocess.run([exe, "--list-elf", psw.library_path()], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_abi_version(psw):
    assert psw.lib().psw_abi_version() == 4


def test_decompose_matches_reference(psw, orc):
    for n, P in ((1024, 4), (4096, 16), (333, 9), (16, 4), (10, 1), (7, 3), (65536, 512)):
        part = psw.decompose(n, P).induced_partition()
        assert part.boundaries == orc.decompose(n, P).tolist()
    d = psw.decompose(7, 3)
    assert [hi - lo + 1 for lo, hi in d.ranges] == [3, 2, 2]
    with pytest.raises(psw.TooManyPEs):
        psw.decompose(7, 4)
    with pytest.raises(psw.TooManyPEs):
        psw.decompose(4, 3)


def test_partition_validate_and_parse(psw):  # test_dichotomy.cpp:38-49
    part = psw.Partition(16, [4, 8, 12])
    part.validate()
    assert part.to_string() == "4,8,12"
    assert psw.Partition.parse(16, "4,8,12").boundaries == [4, 8, 12]
    for bad in ("4,4,12", "1,8", "8,16"):
        with pytest.raises(ValueError):
            psw.Partition.parse(16, bad)
    with pytest.raises(ValueError):
        psw.Partition.parse(16, "4,banana")


def test_plan_rejects_invalid_inputs(psw):
    A = psw.TridiagMatrix.constant(16, -1.0, 2.0, -1.0)
    with pytest.raises(ValueError):
        psw.Plan(A, psw.Partition(16, [4, 4]))
    with pytest.raises(ValueError):
        psw.Plan(A, psw.Partition(16, [1, 8]))
    with pytest.raises(ValueError):
        psw.Plan(psw.TridiagMatrix(np.ones(15), np.full(16, np.nan), np.ones(15)), psw.Partition(16, [8]))
    with pytest.raises(ValueError):  # unknown GRowStrategy
        psw.Plan(A, psw.Partition(16, [8]), strategy=7)


def test_plan_strategy_failures_like_reference(psw, orc):
    """Explicit GRowStrategy failures surface at setup with the reference's
    exception types and index, before any device is needed
    (preliminary.hpp:111-132; errors.hpp:29-43)."""
    from oracle.pyoracle import EXPLICIT_INVERSE, SYMMETRIZE, OracleError
    rng = np.random.default_rng(5)
    n = 40
    sub, sup = rng.uniform(-1, 1, n - 1), rng.uniform(-1, 1, n - 1)
    sup[::3] = -np.sign(sub[::3]) * np.abs(sup[::3])
    diag = np.r_[0, np.abs(sub)] + np.r_[np.abs(sup), 0] + 1.0
    A = psw.TridiagMatrix(sub, diag, sup)
    part = psw.Partition(n, [10, 20, 30])
    with pytest.raises(OracleError) as want:
        orc.preliminary(sub, diag, sup, [10, 20, 30], strategy=SYMMETRIZE)
    with pytest.raises(psw.NotSymmetrizable) as got:
        psw.Plan(A, part, strategy=psw.GROW_SYMMETRIZE)
    assert got.value.index == want.value.index
    red = psw.TridiagMatrix(-np.ones(5), 2.0 * np.ones(6), np.array([-1.0, -1.0, 0.0, -1.0, -1.0]))
    with pytest.raises(psw.OracleFallbackRequired):
        psw.Plan(red, psw.Partition(6, [3]), strategy=psw.GROW_EXPLICIT_INVERSE)
    with pytest.raises(OracleError):
        orc.preliminary(red.sub, red.diag, red.super, [3], strategy=EXPLICIT_INVERSE)


def test_plan_pivot_breakdown_like_reference(psw, orc):
    # singular Neumann matrix (test_core.cpp:48-55): the reference's
    # preliminary fails in the inverse-row sweep at row 2; with p = 0 the
    # first solve's sweep fails at the same row.
    A = psw.TridiagMatrix(np.array([-1.0, -1.0]), np.array([1.0, 2.0, 1.0]), np.array([-1.0, -1.0]))
    with pytest.raises(OracleError) as want:
        orc.preliminary(A.sub, A.diag, A.super, [2])
    for part in (psw.Partition(3, [2]), psw.Partition(3, [])):
        with pytest.raises(psw.PivotBreakdown) as got:
            psw.Plan(A, part)
        assert got.value.row == want.value.index == 2


def test_plan_requires_device_without_fallback(psw):
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    g = load_golden("c0_n1024_P4")
    A = psw.TridiagMatrix(g["sub"], g["diag"], g["super"])
    with pytest.raises(psw.CudaError, match="no CUDA device"):
        psw.Plan(A, psw.Partition(1024, g["bnd"].tolist()))


def test_header_cites_reference():
    text = open(os.path.join(ROOT, "include", "parsweep_b200.h")).read()
    for cite in ("preliminary.hpp:171-199", "batch.hpp:20-51", "decompose.hpp:33-47",
                 "partition.hpp:31-42", "batch.hpp:57-75"):
        assert cite in text


def test_configs_bytes_min_matches_baseline():
    from paper_0901_2859_b200.configs import CONFIGS
    assert CONFIGS["C0"].bytes_min() == 4_210_680
    assert CONFIGS["C1"].bytes_min() == 268_500_984
    assert CONFIGS["C2"].bytes_min() == 34_360_262_652
    assert CONFIGS["C3"].bytes_min() == 17_196_646_392
