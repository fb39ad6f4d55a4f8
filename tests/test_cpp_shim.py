"""The C++ drop-in (include/sfmp/cuda.hpp): it compiles against the
reference's own headers, and oracle/_ref/dropin_test -- the UNMODIFIED
reference sources linked with the product library through the shim -- agrees
with the reference's sfmp::gemv and maps errors to the reference exceptions."""
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT
from synth import activations, model_bytes

REF_INC = "/root/reference/proj/include"
DROPIN = os.path.join(ROOT, "oracle", "_ref", "dropin_test")


@pytest.mark.skipif(not os.path.isdir(REF_INC), reason="reference headers not present")
def test_shim_compiles_against_reference_headers(tmp_path):
    src = tmp_path / "t.cpp"
    src.write_text('#include "sfmp/layout.hpp"\n#include "sfmp/lutgemm.hpp"\n#include "sfmp/errors.hpp"\n'
                   '#include "sfmp/cuda.hpp"\nint main(){return 0;}\n')
    r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", f"-I{REF_INC}",
                        f"-I{os.path.join(ROOT, 'include')}", str(src)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


@pytest.mark.skipif(not os.path.exists(DROPIN), reason="dropin_test not built (needs /root/reference)")
def test_dropin_binary_links_product_library():
    out = subprocess.run(["ldd", DROPIN], capture_output=True, text=True).stdout
    assert "libsfmp_b200.so" in out and "not found" not in out


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(DROPIN), reason="dropin_test not built")
@pytest.mark.parametrize("bits,mode", [(3.5, 3), (2.5, 1), (4.0, 0)])
def test_dropin_matches_reference_gemv(gpu, port, tmp_path, bits, mode):
    data = model_bytes(port, 1024, 512, bits, mode=mode)
    x = activations(port, 3, 512, seed=4)
    (tmp_path / "m.sfmp").write_bytes(data)
    (tmp_path / "x.f32").write_bytes(np.ascontiguousarray(x, np.float32).tobytes())
    r = subprocess.run([DROPIN, str(tmp_path / "m.sfmp"), str(tmp_path / "x.f32"), "3"],
                       capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "format_error=1 shape_error=1" in r.stdout


@pytest.mark.gpu
def test_cpp_sharded_entry_world1(gpu, port, tmp_path):
    """A C++ caller of sfmp_gemm_sharded (NCCL communicator from sfmp_nccl_comm_init,
    world 1): bit-identical to sfmp_gemm; a size-mismatched communicator is refused."""
    exe = tmp_path / "sharded_test"
    lib_dir = os.path.join(ROOT, "paper_2602_01027_b200")
    r = subprocess.run(["g++", "-std=c++17", "-O1", "-o", str(exe), os.path.join(ROOT, "tests", "cpp", "sharded_test.cpp"),
                        f"-I{os.path.join(ROOT, 'include')}", "-I/usr/local/cuda/include", f"-L{lib_dir}", "-lsfmp_b200",
                        "-L/usr/local/cuda/lib64", "-lcudart", f"-Wl,-rpath,{lib_dir}"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    data = model_bytes(port, 1024, 1024, 3.25)
    (tmp_path / "m.sfmp").write_bytes(data)
    r = subprocess.run([str(exe), str(tmp_path / "m.sfmp")], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "sharded_vs_unsharded_bit_equal=1" in r.stdout
