"""The C-ABI library loads and exports every symbol include/nsfr_gpu.h declares;
host-only logic (halo plan) and the no-fallback rule. CPU only (no compute)."""
import os
import re
import subprocess

import pytest

import paper_2312_07725_b200 as P
from paper_2312_07725_b200 import solver

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "nsfr_gpu.h")


def declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(nsfr_gpu_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = P.load_library()
    names = declared()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n
    out = subprocess.run(["nm", "-D", "--defined-only", solver.LIB_PATH], capture_output=True, text=True).stdout
    for n in names:
        assert re.search(rf"\bT {n}\b", out), n


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", solver.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("m,n", [(128, 1), (128, 2), (128, 8), (7, 3), (16, 16)])
def test_halo_plan_partition(m, n):
    planes = []
    for r in range(n):
        h = P.halo_plan(m, 4, r, n)
        assert h["peer_lo"] == (r - 1) % n and h["peer_hi"] == (r + 1) % n
        assert h["count"] == m * m * 6 * 25  # NTR = 6 values per face node
        assert h["k1"] > h["k0"]
        planes += list(range(h["k0"], h["k1"]))
    assert planes == list(range(m))


def test_halo_plan_rejects_bad_partition():
    with pytest.raises(P.DimensionError):
        P.halo_plan(4, 3, 0, 8)


def test_no_cpu_fallback_without_device():
    try:
        import torch
        has = torch.cuda.is_available()
    except Exception:
        has = False
    if has:
        pytest.skip("CUDA device present")
    with pytest.raises(P.DeviceError):
        P.GpuSolver(P.SolverConfig(p=3, m=2))


def test_bad_config_raises_dimension_error():
    with pytest.raises(P.DimensionError):
        P.GpuSolver(P.SolverConfig(p=9, m=2))


def test_unknown_scheme_is_a_config_error():
    import paper_2312_07725_b200 as pkg
    with pytest.raises(pkg.ConfigError):
        pkg.GpuSolver(pkg.SolverConfig(p=3, m=2, scheme="bogus"))
