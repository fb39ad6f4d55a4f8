"""Generate the golden fixtures in tests/golden/ from the UNMODIFIED reference.

Run here (where /root/reference exists):  python tests/golden/make_golden.py
Every array below is produced by the reference library compiled from
/root/reference/proj/src (oracle/_ref/libsfmpref.so via oracle/ref_shim.cpp):
model bytes by its own quantize_group/pack_block/serialize, W by
dequantize_model, y_ref by matmul_reference, y_lut by gemv, error kinds by
deserialize.  Inputs W, S, x come from the seeded generators in
oracle/sfmp_oracle.c.  The fixtures are small so they can be
committed; the GPU box never needs /root/reference.
"""
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.oracle import OracleError, Port, Reference  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

# (name, rows, cols, m_b, n_b, avg code bits, mode, M, store_w)
CASES = [
    ("tiny_rowcol_b2.5", 64, 64, 16, 16, 2.5, 3, 3, True),
    ("small_rowcol_b3.25", 512, 256, 128, 128, 3.25, 3, 4, True),
    ("small_row_b4_nb64", 256, 512, 128, 64, 4.0, 1, 4, True),
    ("small_col_b2.5_mb8", 128, 128, 8, 8, 2.5, 2, 2, True),
    ("small_none_b2", 256, 256, 64, 128, 2.0, 0, 3, True),
    ("small_rowcol_b1.5", 256, 256, 128, 128, 1.5, 3, 2, True),
    ("small_rowcol_b5.5", 256, 256, 128, 128, 5.5, 3, 2, True),
    ("small_rowcol_b7.75", 128, 256, 128, 128, 7.75, 3, 2, True),
    ("cfg1_mini_rowcol_b3.5", 1024, 512, 512, 128, 3.5, 3, 16, False),
    ("nb256_rowcol_b3", 512, 512, 256, 256, 3.0, 3, 5, False),
]


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    P, R = Port(), Reference()
    index = {}
    for name, rows, cols, m_b, n_b, b, mode, M, store_w in CASES:
        seed = sum(map(ord, name))
        W = P.gen_weights(rows, cols, seed)
        S = P.gen_salience(rows, cols, seed + 1)
        data = R.build_model(W, S, m_b, n_b, b + 32.0 / n_b, mode)
        rm = R.load(data)
        codes = rm.unpack_codes()
        w = rm.dequantize()
        x = P.gen_activation(M, cols, seed + 2)
        y_ref = R.matmul(x, w)
        y_lut = np.stack([rm.gemv(x[t])[0] for t in range(M)])
        lookups = rm.gemv(x[0])[1]
        arrs = dict(model=np.frombuffer(data, np.uint8), x=x, y_ref=y_ref, y_lut=y_lut,
                    offsets=rm.block_offsets())
        if store_w:
            arrs["w"] = w
            arrs["codes"] = codes
        np.savez_compressed(os.path.join(OUT, name + ".npz"), **arrs)
        index[name] = dict(rows=rows, cols=cols, m_b=m_b, n_b=n_b, avg_bits=b, mode=mode, M=M,
                           seed=seed, bytes=len(data), w_sha256=sha(w), codes_sha256=sha(codes),
                           lookups=lookups)
        print(name, len(data), "bytes")

    # Known-answer tests straight from the spec, evaluated by the reference.
    kat = {}
    g = R.quantize_group(np.array([0, 1, 2, 3], np.float32), 2)
    kat["quantize_0123_b2"] = dict(scale=g[0], zero=g[1], codes=g[2].tolist())
    g = R.quantize_group(np.array([5, 5, 5], np.float32), 3)
    kat["quantize_const_b3"] = dict(scale=g[0], zero=g[1], codes=g[2].tolist())
    g = R.quantize_group(np.array([0, 3], np.float32), 1)
    kat["quantize_03_b1"] = dict(scale=g[0], zero=g[1], codes=g[2].tolist())
    fl = [0.0, 1.0, -1.0, 0.5, 65504.0, 65520.0, 1e9, -1e9, 6.1e-5, 5.96e-8, 2.98e-8, 2.99e-8,
          1.0009765625, 1.00048828125, 1.000732421875, 3.14159265, -2.5e-6, float("inf"),
          float("-inf")]
    kat["fp16_from_float"] = {repr(f): R.fp16_from_float(f) for f in fl}
    kat["fp16_to_float_all"] = sha(np.array([R.fp16_to_float(h) for h in range(65536)],
                                            np.float32))

    # Format error kinds from the reference deserialize.
    base = bytes(np.load(os.path.join(OUT, "small_rowcol_b3.25.npz"))["model"])
    def kind(buf):
        try:
            R.load(buf)
            return "ok"
        except OracleError as e:
            return e.kind
    muts = {
        "bad_magic": b"X" + base[1:],
        "bad_version": base[:8] + b"\x02\x00" + base[10:],
        "truncated_header": base[:20],
        "truncated_perm": base[:38 + 100],
        "truncated_plane": base[:-5],
        "trailing_bytes": base + b"\x00",
        "bad_mode": base[:36] + b"\x07" + base[37:],
        "bad_perm_dup": base[:38] + base[42:46] + base[42:],
        "empty": b"",
        "bad_floor_bits": base[:34] + b"\x00" + base[35:],
    }
    kat["format_errors"] = {}
    for k, v in muts.items():
        kat["format_errors"][k] = kind(v)
        np.save(os.path.join(OUT, f"err_{k}.npy"), np.frombuffer(v, np.uint8)) if len(v) < 70000 else None
    index["_kat"] = kat
    with open(os.path.join(OUT, "index.json"), "w") as f:
        json.dump(index, f, indent=1, sort_keys=True)
    print(json.dumps(kat["format_errors"]))


if __name__ == "__main__":
    main()
