"""The C-ABI library builds, loads, exports every symbol include/cisdc_gpu.h declares, and refuses to
run without a GPU (no CPU fallback).  No GPU needed."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_1801_01201_b200 import _abi, api, problems as P

HDR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "cisdc_gpu.h")


def declared_functions():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cisdc_\w+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("cisdc_gpu_create", "cisdc_gpu_initialize", "cisdc_gpu_sweep", "cisdc_gpu_increment",
                 "cisdc_gpu_get_field", "cisdc_gpu_integrate", "cisdc_gpu_last_error", "cisdc_gpu_destroy",
                 "cisdc_make_quadrature_tables"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = _abi.load(build_if_missing=True)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    bound = {n for n, _, _ in _abi.GPU_SYMBOLS}
    assert set(declared_functions()) <= bound, set(declared_functions()) - bound


def test_library_is_sm100a():
    import subprocess
    lib = _abi.lib_path()
    out = subprocess.run(["cuobjdump", "--list-elf", lib], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_struct_layouts_match_header():
    # sizes as laid out by the C compiler
    assert C.sizeof(_abi.TablesC) == 8 + 8 * (9 + 8 + 72 + 8 + 64 + 72 + 64 + 64)
    assert C.sizeof(_abi.CountersC) == 5 * 8
    assert C.sizeof(_abi.StepReportC) == 8 + 40


def test_quadrature_tables_host_call():
    t = api.make_quadrature_tables(4)
    s = np.sqrt(3 / 7)
    assert abs(t.tau[1] - 0.5 * (1 - s)) <= 1e-14
    with pytest.raises(ValueError):
        api.make_quadrature_tables(0)


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    spec = P.config_c1(scale=4)
    with pytest.raises(api.CudaError, match="no CPU fallback"):
        api.integrate(spec.problem, spec.phi0, api.IntegrateOptions(scheme=1, dt=1e-3, M=2, n_sweeps=1))
