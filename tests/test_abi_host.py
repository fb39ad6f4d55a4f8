"""Host-side checks of the product C ABI (no GPU): the library loads, exports every
symbol include/sfmp_cuda.h declares, and its SFMPPKD1 ingest matches the reference
(error kinds, header fields, block offsets).  No compute calls here."""
import os
import re

import numpy as np
import pytest

import paper_2602_01027_b200 as sfmp
from conftest import GOLDEN, ROOT, golden_cases, load_golden


def declared_symbols():
    txt = open(os.path.join(ROOT, "include", "sfmp_cuda.h")).read()
    return sorted(set(re.findall(r"^\s*(?:[\w\s\*]+?)\b(sfmp_\w+)\s*\(", txt, re.M)))


def test_library_exports_declared_symbols():
    L = sfmp.lib()
    decl = declared_symbols()
    assert len(decl) >= 18
    for name in decl:
        assert hasattr(L, name), name
    assert set(decl) == set(sfmp.EXPORTED_SYMBOLS)
    assert L.sfmp_abi_version() == 2


def test_library_is_sm100a_only():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", sfmp.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(7|8|9)\d", out)


@pytest.mark.parametrize("name", golden_cases())
def test_parse_header_matches_golden(index, name):
    meta, g = index[name], load_golden(name)
    data = bytes(g["model"])
    info = sfmp.parse_header(data)
    assert (info["rows"], info["cols"], info["m_b"], info["n_b"], info["mode"]) == (
        meta["rows"], meta["cols"], meta["m_b"], meta["n_b"], meta["mode"])
    assert abs(info["avg_code_bits"] - meta["avg_bits"]) < 0.26
    assert np.array_equal(sfmp.compute_block_offsets(data), g["offsets"])


def test_format_error_kinds_match_reference(index):
    for k, expect in index["_kat"]["format_errors"].items():
        buf = bytes(np.load(f"{GOLDEN}/err_{k}.npy"))
        try:
            sfmp.parse_header(buf)
            got = "ok"
        except sfmp.FormatError as e:
            got = e.kind
        assert got == expect, k


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    data = bytes(load_golden("small_rowcol_b3.25")["model"])
    assert sfmp.device_count() == 0
    with pytest.raises(sfmp.CudaError):
        sfmp.DeviceModel(data)


def test_shard_plan_snake_partition():
    data = bytes(load_golden("cfg1_mini_rowcol_b3.5")["model"])  # 2 block rows of 512
    gmap, sr = sfmp.shard_plan(data, 2)
    assert sr == 512 and gmap.shape == (2, 512)
    assert sorted(gmap.reshape(-1).tolist()) == list(range(1024))  # a bijection onto rows
    with pytest.raises(sfmp.ShapeError):
        sfmp.shard_plan(data, 4)  # 2 block rows cannot split 4 ways


def test_grouped_argument_checks():
    """sfmp_gemm_grouped(_v) validate before touching the device: an empty group is
    a no-op, missing arrays are argument errors, negative token counts shape errors."""
    import ctypes as C
    L = sfmp.lib()
    assert L.sfmp_gemm_grouped_v(None, None, 2, None, None, None, None, 0, None) == 0
    assert L.sfmp_gemm_grouped(None, None, 2, C.c_int64(0), None, None, None, 0, None) == 0
    assert L.sfmp_gemm_grouped_v(None, None, 2, None, None, None, None, 1, None) != 0
    assert b"null" in L.sfmp_last_error()
    one = (C.c_void_p * 1)(C.c_void_p(1))
    ms = (C.c_int64 * 1)(-3)
    st = L.sfmp_gemm_grouped_v(one, one, 2, ms, one, one, None, 1, None)
    assert st != 0 and b"negative" in L.sfmp_last_error()
    assert L.sfmp_gemm_grouped(one, one, 2, C.c_int64(-1), one, one, None, 1, None) != 0
