"""The C++ drop-in (include/pmfgpu.hpp) used from parmf's own types: oracle/_ref/adapter_test trains
through pmfgpu::ccdpp_train / als_train and checks against parmf::ccdpp_train / als_train."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "oracle", "_ref", "adapter_test")


@pytest.mark.gpu
def test_cpp_adapter_drop_in():
    if not os.path.exists(EXE):
        pytest.skip("adapter_test not built (needs /root/reference at build time)")
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "OK" in r.stdout
