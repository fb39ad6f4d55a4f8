"""Pin the CPU oracle (oracle/sfmp_oracle.c) against golden vectors produced by the
unmodified reference (tests/golden/make_golden.py) and the spec's known answers."""
import hashlib
import math

import numpy as np
import pytest

from conftest import GOLDEN, golden_cases, load_golden


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("name", golden_cases())
def test_port_bit_exact_vs_reference_goldens(port, index, name):
    meta, g = index[name], load_golden(name)
    data = bytes(g["model"])
    # The port's offline packer reproduces the reference's SFMPPKD1 bytes exactly.
    W = port.gen_weights(meta["rows"], meta["cols"], meta["seed"])
    S = port.gen_salience(meta["rows"], meta["cols"], meta["seed"] + 1)
    assert port.build_model(W, S, meta["m_b"], meta["n_b"], meta["avg_bits"] + 32.0 / meta["n_b"],
                            meta["mode"]) == data
    x = port.gen_activation(meta["M"], meta["cols"], meta["seed"] + 2)
    assert np.array_equal(x, g["x"])
    m = port.load(data)
    assert np.array_equal(m.block_offsets(), g["offsets"])           # layout.cpp:301-314
    codes = m.unpack_codes()
    assert sha(codes) == meta["codes_sha256"]                          # layout.cpp:67-86
    w = m.dequantize()
    assert sha(w) == meta["w_sha256"]                                  # layout.cpp:316-332 bit-exact
    y = port.matmul(x, w)
    assert np.array_equal(y.view(np.uint32), g["y_ref"].view(np.uint32))  # matrix.cpp:5-17
    for t in range(meta["M"]):
        yl, lk = m.gemv_lut(x[t])
        assert np.array_equal(yl.view(np.uint32), g["y_lut"][t].view(np.uint32))  # lutgemm.cpp:95
        assert lk == meta["lookups"]
    if "w" in g:
        assert np.array_equal(w.view(np.uint32), g["w"].view(np.uint32))
        assert np.array_equal(codes, g["codes"])


def test_lookup_count_formula(port, index):
    # SPEC.md:528 work scaling: lookups == sum_k bits_k * m_b * n_b / 8
    for name in golden_cases():
        meta = index[name]
        m = port.load(bytes(load_golden(name)["model"]))
        assert meta["lookups"] == int(m.block_bits.astype(np.int64).sum()) * m.m_b * m.n_b // 8


def test_spec_kats(port, index):
    kat = index["_kat"]
    for key, vals in [("quantize_0123_b2", ([0, 1, 2, 3], 2)), ("quantize_const_b3", ([5, 5, 5], 3)),
                      ("quantize_03_b1", ([0, 3], 1))]:
        s, z, c = port.quantize_group(np.array(vals[0], np.float32), vals[1])
        assert (s, z, c.tolist()) == (kat[key]["scale"], kat[key]["zero"], kat[key]["codes"])
    # SPEC.md:352-354 literal expectations
    assert kat["quantize_0123_b2"] == {"scale": 1.0, "zero": 0.0, "codes": [0, 1, 2, 3]}
    assert kat["quantize_const_b3"]["codes"] == [0, 0, 0] and kat["quantize_const_b3"]["zero"] == 5.0
    assert kat["quantize_03_b1"] == {"scale": 3.0, "zero": 0.0, "codes": [0, 1]}
    for f, h in kat["fp16_from_float"].items():
        assert port.fp16_from_float(float(f)) == h, f
    allf = np.array([port.fp16_to_float(h) for h in range(65536)], np.float32)
    assert sha(allf) == kat["fp16_to_float_all"]


def test_bitplane_kat(port):
    # SPEC.md:428 / PAPER.md:610: codes (9,7,6,3), 4 bits -> plane0=(1,1,0,1), plane3=(1,0,0,0)
    import struct
    codes = [9, 7, 6, 3, 0, 0, 0, 0]
    planes = [sum(((c >> i) & 1) << k for k, c in enumerate(codes)) for i in range(4)]
    assert [(planes[0] >> k) & 1 for k in range(4)] == [1, 1, 0, 1]
    assert [(planes[3] >> k) & 1 for k in range(4)] == [1, 0, 0, 0]
    # Build a 1x8 block model by hand and check the port unpacks it.
    hdr = b"SFMPPKD1" + struct.pack("<HQQIIBBBB", 1, 1, 8, 1, 8, 4, 4, 0, 0) + struct.pack("<Q", 1) + bytes([4])
    blk = struct.pack("<HH", 0x3C00, 0x0000) + bytes(planes)
    m = port.load(hdr + blk)
    assert m.unpack_codes().tolist() == [codes]
    assert m.dequantize().tolist() == [[float(c) for c in codes]]


def test_format_error_kinds_match_reference(index):
    from oracle.oracle import OracleError, Port
    P = Port()
    for k, expect in index["_kat"]["format_errors"].items():
        buf = bytes(np.load(f"{GOLDEN}/err_{k}.npy"))
        try:
            P.load(buf)
            got = "ok"
        except OracleError as e:
            got = e.kind
        assert got == expect, k


def test_linearity_and_zero(port):
    d = load_golden("small_rowcol_b3.25")
    m = port.load(bytes(d["model"]))
    x = d["x"][0]
    y0, _ = m.gemv_lut(np.zeros_like(x))
    assert np.all(y0 == 0)
    y1, _ = m.gemv_lut(x)
    y2, _ = m.gemv_lut(2 * x)
    assert np.allclose(y2, 2 * y1, rtol=1e-5, atol=1e-6)


@pytest.mark.skipif(not __import__("oracle.oracle", fromlist=["x"]).reference_available(),
                    reason="reference library not built")
def test_port_vs_reference_random_models(port):
    from oracle.oracle import Reference
    R = Reference()
    rng = np.random.default_rng(0)
    for trial in range(6):
        m_b = int(rng.choice([8, 16, 32]))
        n_b = int(rng.choice([8, 16, 32]))
        rows, cols = m_b * int(rng.integers(1, 5)), n_b * int(rng.integers(1, 5))
        bits = float(rng.choice([1.0, 2.0, 2.5, 3.0, 3.75, 4.0, 6.5]))
        mode = int(rng.integers(0, 4))
        W = port.gen_weights(rows, cols, 100 + trial)
        S = port.gen_salience(rows, cols, 200 + trial)
        a = port.build_model(W, S, m_b, n_b, bits + 32.0 / n_b, mode)
        b = R.build_model(W, S, m_b, n_b, bits + 32.0 / n_b, mode)
        assert a == b
        pm, rm = port.load(a), R.load(b)
        assert np.array_equal(pm.dequantize().view(np.uint32), rm.dequantize().view(np.uint32))
        x = port.gen_activation(1, cols, 300 + trial)[0]
        assert np.array_equal(pm.gemv_lut(x)[0].view(np.uint32), rm.gemv(x)[0].view(np.uint32))
