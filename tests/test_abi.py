"""The C-ABI library (no GPU): it loads, exports every symbol the header
declares, and its host-side entry points validate like the reference."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT


def header_symbols():
    text = open(os.path.join(ROOT, "include", "tessera_b200.h")).read()
    return sorted(set(re.findall(r"\b(tsr_[a-z_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol(ts):
    from paper_2303_08365_b200 import _abi
    L = _abi.lib()
    syms = header_symbols()
    assert len(syms) >= 12
    for name in syms:
        assert hasattr(L, name), name
    assert set(syms) == set(_abi.EXPORTED)
    assert L.tsr_abi_version() == _abi.ABI_VERSION == 3


def test_library_is_sm100a(ts):
    """The shipped fatbinary carries sm_100a SASS (no PTX-only / other arch)."""
    import subprocess
    from paper_2303_08365_b200 import _abi
    out = subprocess.run(["cuobjdump", "--list-elf", _abi.LIB_PATH], capture_output=True,
                         text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    archs = set(re.findall(r"sm_(\d+a?)", out.stdout))
    assert archs == {"100a"}, archs


def _grid(dims, ext, halo, dtype=0):
    from paper_2303_08365_b200 import _abi
    g = _abi.TsrGrid()
    g.dims, g.dtype = dims, dtype
    for a in range(3):
        g.extent[a] = ext[a] if a < dims else 1
        g.halo[a] = halo[a] if a < dims else 0
    return g


def test_layout_is_pitched_and_aligned(ts):
    from paper_2303_08365_b200 import _abi
    L = _abi.lib()
    for dims, ext, halo, dt in [(3, [512, 512, 512], [1, 1, 1], 0),
                                (3, [1024, 1024, 1024], [1, 1, 1], 1),
                                (2, [4096, 4096], [1, 1], 0), (1, [100], [2], 0),
                                (2, [33, 30], [2, 2], 1)]:
        lay = _abi.TsrLayout()
        assert L.tsr_layout_of(ctypes.byref(_grid(dims, ext, halo, dt)), ctypes.byref(lay)) == 0
        esize = 8 if dt == 0 else 4
        assert lay.pitch[dims - 1] == 1
        row = lay.pitch[dims - 2] if dims > 1 else None
        if row:
            assert (row * esize) % 128 == 0 and row >= ext[-1] + 2 * halo[-1]
        assert (lay.origin * esize) % 128 == 0  # interior rows start 128-B aligned
        assert lay.elements * esize >= np.prod([e + 2 * h for e, h in zip(ext, halo)]) * esize


def test_layout_rejects_degenerate(ts):
    from paper_2303_08365_b200 import _abi
    L = _abi.lib()
    lay = _abi.TsrLayout()
    rc = L.tsr_layout_of(ctypes.byref(_grid(2, [2, 8], [1, 1])), ctypes.byref(lay))
    assert rc == _abi.TSR_EINVAL
    assert b"degenerate extent" in L.tsr_last_error()


def test_check_kernel(ts):
    from paper_2303_08365_b200 import _abi
    L = _abi.lib()
    good = ts.find_benchmark("Box-3D27P").kernel
    assert L.tsr_check_kernel(ctypes.byref(good.c_struct())) == 0
    # non-canonical order is rejected (the C-ABI requires make_kernel order)
    taps = good.tap_list()[::-1]
    bad = ts.StencilKernel(3, "box", 1, taps)
    assert L.tsr_check_kernel(ctypes.byref(bad.c_struct())) == _abi.TSR_EINVAL
    short = ts.StencilKernel(3, "box", 1, good.tap_list()[:26])
    assert L.tsr_check_kernel(ctypes.byref(short.c_struct())) == _abi.TSR_EINVAL
    assert b"offset count mismatch" in L.tsr_last_error()


def test_run_validates_before_touching_the_device(ts):
    """Invalid arguments are reported as ValueError (std::invalid_argument)
    on any machine, GPU or not."""
    g = ts.Grid([8, 8], [1, 1])
    k3 = ts.find_benchmark("Heat-3D").kernel
    with pytest.raises(ValueError, match="dimensionality"):
        ts.naive_run(g, k3, 1)
    with pytest.raises(ValueError, match="halo too small"):
        ts.naive_run(g, ts.find_benchmark("Star-2D9P").kernel, 1)
    with pytest.raises(ValueError, match="negative"):
        ts.naive_run(g, ts.heat_coefficients(0.2), -1)
    ts.naive_run(g, ts.heat_coefficients(0.2), 0)  # T = 0 is a no-op
    assert g.parity == 0
