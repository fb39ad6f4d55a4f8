"""The repacked <=4-bit decode layout (csrc/repack.cuh) on the host: pack/decode
round trip, bit conservation (same bytes as the bit planes) and the exact f16
values the GEMV's one-LOP3 unpack produces.  Compiled with nvcc as host code."""
import os
import shutil
import subprocess

import pytest

from conftest import ROOT


@pytest.mark.skipif(shutil.which("nvcc") is None and not os.path.exists("/usr/local/cuda/bin/nvcc"),
                    reason="nvcc not available")
def test_repack_roundtrip(tmp_path):
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    exe = tmp_path / "repack_test"
    src = os.path.join(ROOT, "tests", "cpp", "repack_test.cu")
    r = subprocess.run([nvcc, "-std=c++17", "-O1", "-o", str(exe), src], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "mismatches: 0" in r.stdout
