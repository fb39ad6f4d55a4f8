"""TEST INFRASTRUCTURE ONLY -- ctypes front-end to the CPU parity checkers.

Two implementations behind one API:

* ``Port``      -- ``oracle/liboracle.so``, the plain-C restatement of the
                   reference algorithms (``oracle/sfmp_oracle.c``).
* ``Reference`` -- ``oracle/_ref/libsfmpref.so``, the UNMODIFIED reference
                   compiled from ``/root/reference/proj/src`` plus an extern "C"
                   shim (``oracle/ref_shim.cpp``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline /
``--impl reference``) may import this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libsfmpref.so")

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")

STATUS_NAMES = {0: "ok", 1: "shape", 2: "config", 3: "bad_magic", 4: "bad_version",
                5: "truncated", 6: "invariant", 7: "io", 11: "nomem", 99: "unknown"}


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"{what}: {STATUS_NAMES.get(code, code)}")
        self.code = code
        self.kind = STATUS_NAMES.get(code, str(code))


def build(force: bool = False) -> None:
    """Build the checkers (make -C oracle).  The reference leg is built only
    where /root/reference exists; elsewhere a prebuilt _ref/ is used."""
    if force or not os.path.exists(PORT_SO) or (
            os.path.isdir("/root/reference/proj") and not os.path.exists(REF_SO)):
        subprocess.run(["make", "-s", "-C", HERE], check=True)


class _Model(C.Structure):
    _fields_ = [("version", C.c_uint16), ("rows", C.c_uint64), ("cols", C.c_uint64),
                ("m_b", C.c_uint32), ("n_b", C.c_uint32), ("floor_bits", C.c_int),
                ("ceil_bits", C.c_int), ("mode", C.c_int), ("row_perm", C.c_void_p),
                ("col_perm", C.c_void_p), ("K", C.c_uint64), ("block_bits", C.c_void_p),
                ("block_off", C.c_void_p), ("base", C.c_void_p)]


class Port:
    """The C restatement.  Model handles keep the byte buffer alive."""

    def __init__(self):
        build()
        L = C.CDLL(PORT_SO)
        self.L = L
        L.sfmpo_fp16_from_float.restype = C.c_uint16
        L.sfmpo_fp16_from_float.argtypes = [C.c_float]
        L.sfmpo_fp16_to_float.restype = C.c_float
        L.sfmpo_fp16_to_float.argtypes = [C.c_uint16]
        L.sfmpo_parse.argtypes = [C.c_void_p, C.c_size_t, C.POINTER(_Model)]
        L.sfmpo_free.argtypes = [C.POINTER(_Model)]
        L.sfmpo_unpack_codes.argtypes = [C.POINTER(_Model), _u8p]
        L.sfmpo_dequantize.argtypes = [C.POINTER(_Model), _f32p]
        L.sfmpo_matmul_reference.argtypes = [_f32p, _f32p, _f32p, C.c_int64, C.c_int64, C.c_int64]
        L.sfmpo_matmul_reference_mt.argtypes = [_f32p, _f32p, _f32p, C.c_int64, C.c_int64,
                                                C.c_int64, C.c_int]
        L.sfmpo_gemv_lut.argtypes = [C.POINTER(_Model), _f32p, _f32p, C.POINTER(C.c_uint64)]
        L.sfmpo_gemm_lut.argtypes = [C.POINTER(_Model), _f32p, _f32p, C.c_int64, C.c_int]
        L.sfmpo_quantize_group.argtypes = [_f32p, C.c_size_t, C.c_int, C.POINTER(C.c_float),
                                           C.POINTER(C.c_float), _u8p]
        L.sfmpo_build_model.argtypes = [_f32p, _f32p, C.c_uint64, C.c_uint64, C.c_uint32,
                                        C.c_uint32, C.c_double, C.c_int, C.c_void_p,
                                        C.POINTER(C.c_size_t)]
        L.sfmpo_block_offsets.argtypes = [C.c_void_p, C.c_size_t, _u64p, C.c_uint64]
        L.sfmpo_gen_normal.argtypes = [_f32p, C.c_size_t, C.c_uint64, C.c_float, C.c_float]
        L.sfmpo_gen_salience.argtypes = [_f32p, C.c_uint64, C.c_uint64, C.c_uint64]
        L.sfmpo_gen_activation.argtypes = [_f32p, C.c_size_t, C.c_uint64]

    # -- scalars
    def fp16_from_float(self, f: float) -> int:
        return int(self.L.sfmpo_fp16_from_float(f))

    def fp16_to_float(self, h: int) -> float:
        return float(self.L.sfmpo_fp16_to_float(h))

    def quantize_group(self, v, bits):
        v = np.ascontiguousarray(v, dtype=np.float32)
        s, z = C.c_float(), C.c_float()
        codes = np.zeros(v.size, np.uint8)
        rc = self.L.sfmpo_quantize_group(v, v.size, bits, C.byref(s), C.byref(z), codes)
        if rc:
            raise OracleError(rc, "quantize_group")
        return s.value, z.value, codes

    # -- synthetic inputs
    def gen_weights(self, rows, cols, seed, std=0.02):
        out = np.empty(rows * cols, np.float32)
        self.L.sfmpo_gen_normal(out, out.size, seed, 0.0, std)
        return out.reshape(rows, cols)

    def gen_salience(self, rows, cols, seed):
        out = np.empty(rows * cols, np.float32)
        self.L.sfmpo_gen_salience(out, rows, cols, seed)
        return out.reshape(rows, cols)

    def gen_activation(self, M, cols, seed):
        out = np.empty(M * cols, np.float32)
        self.L.sfmpo_gen_activation(out, out.size, seed)
        return out.reshape(M, cols)

    # -- model build / parse
    def build_model(self, W, S, m_b, n_b, target_bpw, mode) -> bytes:
        W = np.ascontiguousarray(W, np.float32)
        S = np.ascontiguousarray(S, np.float32)
        n = C.c_size_t(0)
        rc = self.L.sfmpo_build_model(W, S, W.shape[0], W.shape[1], m_b, n_b, target_bpw, mode,
                                      None, C.byref(n))
        if rc:
            raise OracleError(rc, "build_model(size)")
        buf = C.create_string_buffer(n.value)
        rc = self.L.sfmpo_build_model(W, S, W.shape[0], W.shape[1], m_b, n_b, target_bpw, mode,
                                      buf, C.byref(n))
        if rc:
            raise OracleError(rc, "build_model")
        return buf.raw[: n.value]

    def load(self, data: bytes) -> "PortModel":
        return PortModel(self, data)

    def block_offsets(self, data: bytes, K: int) -> np.ndarray:
        out = np.zeros(K, np.uint64)
        rc = self.L.sfmpo_block_offsets(data, len(data), out, K)
        if rc:
            raise OracleError(rc, "block_offsets")
        return out

    def matmul(self, x, w, threads: int = 1):
        x = np.ascontiguousarray(np.atleast_2d(x), np.float32)
        w = np.ascontiguousarray(w, np.float32)
        y = np.empty((x.shape[0], w.shape[0]), np.float32)
        if threads > 1:
            self.L.sfmpo_matmul_reference_mt(x, w, y, x.shape[0], w.shape[0], w.shape[1], threads)
        else:
            self.L.sfmpo_matmul_reference(x, w, y, x.shape[0], w.shape[0], w.shape[1])
        return y


class PortModel:
    def __init__(self, port: Port, data: bytes):
        self.port = port
        self._buf = C.create_string_buffer(bytes(data), len(data))
        self.m = _Model()
        rc = port.L.sfmpo_parse(self._buf, len(data), C.byref(self.m))
        if rc:
            raise OracleError(rc, "parse")
        self.rows, self.cols = int(self.m.rows), int(self.m.cols)
        self.m_b, self.n_b, self.K = int(self.m.m_b), int(self.m.n_b), int(self.m.K)
        self.mode = int(self.m.mode)
        self.floor_bits, self.ceil_bits = int(self.m.floor_bits), int(self.m.ceil_bits)
        self.block_bits = np.ctypeslib.as_array(
            C.cast(self.m.block_bits, C.POINTER(C.c_uint8)), (self.K,)).copy()
        self.row_perm = (np.ctypeslib.as_array(C.cast(self.m.row_perm, C.POINTER(C.c_uint32)),
                                               (self.rows,)).copy() if self.m.row_perm else None)
        self.col_perm = (np.ctypeslib.as_array(C.cast(self.m.col_perm, C.POINTER(C.c_uint32)),
                                               (self.cols,)).copy() if self.m.col_perm else None)

    def __del__(self):
        try:
            self.port.L.sfmpo_free(C.byref(self.m))
        except Exception:
            pass

    def block_offsets(self):
        return np.ctypeslib.as_array(C.cast(self.m.block_off, C.POINTER(C.c_uint64)),
                                     (self.K,)).copy()

    def unpack_codes(self):
        out = np.zeros(self.rows * self.cols, np.uint8)
        self.port.L.sfmpo_unpack_codes(C.byref(self.m), out)
        return out.reshape(self.rows, self.cols)

    def dequantize(self):
        out = np.zeros(self.rows * self.cols, np.float32)
        self.port.L.sfmpo_dequantize(C.byref(self.m), out)
        return out.reshape(self.rows, self.cols)

    def gemv_lut(self, x):
        x = np.ascontiguousarray(x, np.float32).reshape(-1)
        y = np.zeros(self.rows, np.float32)
        lk = C.c_uint64(0)
        rc = self.port.L.sfmpo_gemv_lut(C.byref(self.m), x, y, C.byref(lk))
        if rc:
            raise OracleError(rc, "gemv_lut")
        return y, int(lk.value)

    def gemm_lut(self, x, threads: int = 1):
        x = np.ascontiguousarray(np.atleast_2d(x), np.float32)
        y = np.zeros((x.shape[0], self.rows), np.float32)
        rc = self.port.L.sfmpo_gemm_lut(C.byref(self.m), x, y, x.shape[0], threads)
        if rc:
            raise OracleError(rc, "gemm_lut")
        return y

    def reference_output(self, x, threads: int = 1, w=None):
        """matmul_reference(x, dequantize_model(model)) -- the central oracle."""
        if w is None:
            w = self.dequantize()
        return self.port.matmul(x, w, threads)


def reference_available() -> bool:
    return os.path.exists(REF_SO)


class Reference:
    """The unmodified reference library (compiled from /root/reference sources)."""

    def __init__(self):
        build()
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(REF_SO)
        L = C.CDLL(REF_SO)
        self.L = L
        L.ref_fp16_from_float.restype = C.c_uint16
        L.ref_fp16_from_float.argtypes = [C.c_float]
        L.ref_fp16_to_float.restype = C.c_float
        L.ref_fp16_to_float.argtypes = [C.c_uint16]
        L.ref_quantize_group.argtypes = [_f32p, C.c_size_t, C.c_int, C.POINTER(C.c_float),
                                         C.POINTER(C.c_float), _u8p]
        L.ref_build_model.argtypes = [_f32p, _f32p, C.c_uint64, C.c_uint64, C.c_uint32,
                                      C.c_uint32, C.c_double, C.c_int, C.c_void_p,
                                      C.POINTER(C.c_size_t)]
        L.ref_load.restype = C.c_void_p
        L.ref_load.argtypes = [C.c_void_p, C.c_size_t, C.POINTER(C.c_int)]
        L.ref_free.argtypes = [C.c_void_p]
        L.ref_serialize.argtypes = [C.c_void_p, C.c_void_p, C.POINTER(C.c_size_t)]
        L.ref_block_offsets.argtypes = [C.c_void_p, _u64p]
        L.ref_unpack_codes.argtypes = [C.c_void_p, _u8p]
        L.ref_dequantize.argtypes = [C.c_void_p, _f32p]
        L.ref_matmul.argtypes = [_f32p, _f32p, _f32p, C.c_uint64, C.c_uint64]
        L.ref_gemv.argtypes = [C.c_void_p, _f32p, _f32p, C.POINTER(C.c_uint64)]
        L.ref_gemm_threads.argtypes = [C.c_void_p, _f32p, _f32p, C.c_int64, C.c_int]
        L.ref_bench_gemv.argtypes = [C.c_void_p, _f32p, C.c_uint64, C.POINTER(C.c_double)]

    def fp16_from_float(self, f):
        return int(self.L.ref_fp16_from_float(f))

    def fp16_to_float(self, h):
        return float(self.L.ref_fp16_to_float(h))

    def quantize_group(self, v, bits):
        v = np.ascontiguousarray(v, dtype=np.float32)
        s, z = C.c_float(), C.c_float()
        codes = np.zeros(v.size, np.uint8)
        rc = self.L.ref_quantize_group(v, v.size, bits, C.byref(s), C.byref(z), codes)
        if rc:
            raise OracleError(rc, "quantize_group")
        return s.value, z.value, codes

    def build_model(self, W, S, m_b, n_b, target_bpw, mode) -> bytes:
        W = np.ascontiguousarray(W, np.float32)
        S = np.ascontiguousarray(S, np.float32)
        n = C.c_size_t(0)
        rc = self.L.ref_build_model(W, S, W.shape[0], W.shape[1], m_b, n_b, target_bpw, mode,
                                    None, C.byref(n))
        if rc:
            raise OracleError(rc, "build_model(size)")
        buf = C.create_string_buffer(n.value)
        rc = self.L.ref_build_model(W, S, W.shape[0], W.shape[1], m_b, n_b, target_bpw, mode,
                                    buf, C.byref(n))
        if rc:
            raise OracleError(rc, "build_model")
        return buf.raw[: n.value]

    def load(self, data: bytes) -> "RefModel":
        return RefModel(self, data)

    def matmul(self, x, w):
        x = np.ascontiguousarray(np.atleast_2d(x), np.float32)
        w = np.ascontiguousarray(w, np.float32)
        y = np.empty((x.shape[0], w.shape[0]), np.float32)
        for t in range(x.shape[0]):
            yt = np.empty(w.shape[0], np.float32)
            rc = self.L.ref_matmul(np.ascontiguousarray(x[t]), w, yt, w.shape[0], w.shape[1])
            if rc:
                raise OracleError(rc, "matmul")
            y[t] = yt
        return y


class RefModel:
    def __init__(self, ref: Reference, data: bytes):
        self.ref = ref
        self._buf = C.create_string_buffer(bytes(data), len(data))
        st = C.c_int(0)
        self.h = ref.L.ref_load(self._buf, len(data), C.byref(st))
        if st.value:
            raise OracleError(st.value, "deserialize")
        pm = Port().load(data)  # header fields only (cheap)
        self.rows, self.cols, self.K = pm.rows, pm.cols, pm.K

    def __del__(self):
        try:
            if self.h:
                self.ref.L.ref_free(self.h)
        except Exception:
            pass

    def serialize(self) -> bytes:
        n = C.c_size_t(0)
        self.ref.L.ref_serialize(self.h, None, C.byref(n))
        buf = C.create_string_buffer(n.value)
        rc = self.ref.L.ref_serialize(self.h, buf, C.byref(n))
        if rc:
            raise OracleError(rc, "serialize")
        return buf.raw[: n.value]

    def block_offsets(self):
        out = np.zeros(self.K, np.uint64)
        self.ref.L.ref_block_offsets(self.h, out)
        return out

    def unpack_codes(self):
        out = np.zeros(self.rows * self.cols, np.uint8)
        rc = self.ref.L.ref_unpack_codes(self.h, out)
        if rc:
            raise OracleError(rc, "unpack")
        return out.reshape(self.rows, self.cols)

    def dequantize(self):
        out = np.zeros(self.rows * self.cols, np.float32)
        rc = self.ref.L.ref_dequantize(self.h, out)
        if rc:
            raise OracleError(rc, "dequantize")
        return out.reshape(self.rows, self.cols)

    def gemv(self, x):
        x = np.ascontiguousarray(x, np.float32).reshape(-1)
        y = np.zeros(self.rows, np.float32)
        lk = C.c_uint64(0)
        rc = self.ref.L.ref_gemv(self.h, x, y, C.byref(lk))
        if rc:
            raise OracleError(rc, "gemv")
        return y, int(lk.value)

    def gemm(self, x, threads: int = 1):
        x = np.ascontiguousarray(np.atleast_2d(x), np.float32)
        y = np.zeros((x.shape[0], self.rows), np.float32)
        rc = self.ref.L.ref_gemm_threads(self.h, x, y, x.shape[0], threads)
        if rc:
            raise OracleError(rc, "gemm")
        return y

    def bench_gemv(self, x, reps):
        x = np.ascontiguousarray(x, np.float32).reshape(-1)
        out = (C.c_double * 4)()
        rc = self.ref.L.ref_bench_gemv(self.h, x, reps, out)
        if rc:
            raise OracleError(rc, "bench_gemv")
        return {"median_us": out[0], "p10_us": out[1], "p90_us": out[2], "lookups": int(out[3])}
