"""The header-only C++ drop-in (include/tessera_b200.hpp) with the reference's
own tessera::BasicGrid / StencilKernel, compiled against the unmodified
reference (oracle/Makefile target `adapter`)."""
import os
import subprocess

import pytest

from conftest import ROOT

BIN = os.path.join(ROOT, "oracle", "_ref", "adapter_test")


def _run():
    if not os.path.exists(BIN):
        pytest.skip("adapter_test not built (make -C oracle adapter)")
    return subprocess.run([BIN], capture_output=True, text=True, timeout=600)


def test_adapter_error_paths_without_gpu():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present: covered by the gpu test")
    except ImportError:
        pass
    r = _run()
    assert r.returncode == 0 and "PASSED (no-gpu)" in r.stdout, r.stdout + r.stderr


@pytest.mark.gpu
def test_adapter_bitwise_with_reference_types():
    r = _run()
    assert r.returncode == 0 and "PASSED (gpu)" in r.stdout, r.stdout + r.stderr
