"""B200-native SFMP mixed-precision GEMM -- Python host mirror of the reference API.

The product is ``libsfmp_b200.so`` (C ABI in ``include/sfmp_cuda.h``; CUDA
kernels for sm_100a in ``csrc/``).  This module binds it with ctypes and
mirrors the reference's operator interface for the hot path
(``/root/reference/proj``):

* ``PackedModel`` bytes (SFMPPKD1, ``layout.cpp:179-279``) -> ``DeviceModel``
* ``gemv(model, x)``                       -> ``lutgemm.hpp:57`` / ``lutgemm.cpp:95-135``
* ``DeviceModel.dequantize()``             -> ``dequantize_model`` (``layout.cpp:316-332``)
* ``DeviceModel.unpack_codes()``           -> ``unpack_block`` (``layout.cpp:67-86``)
* ``compute_block_offsets(bytes)``         -> ``layout.cpp:301-314``
* ``ShapeError`` / ``ConfigError`` / ``FormatError(kind)`` -> ``errors.hpp:9-36``

PyTorch is plumbing only (device memory and streams).  There is no CPU
fallback: without the built library or an sm_100 device the compute entry
points raise.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# SFMP_LIB: load an experiment build instead (tools/ only; the default is the product)
LIB_PATH = os.environ.get("SFMP_LIB") or os.path.join(HERE, "libsfmp_b200.so")

# status codes (include/sfmp_cuda.h)
OK, E_SHAPE, E_CONFIG, E_MAGIC, E_VERSION, E_TRUNC, E_INVARIANT, E_IO, E_CUDA, E_NCCL, E_ARG, \
    E_NOMEM, E_UNSUPPORTED = range(13)
F32, F16, BF16 = 0, 1, 2
PATH_AUTO, PATH_GEMV, PATH_GEMM, PATH_GENERIC, PATH_LUT = 0, 1, 2, 3, 4

EXPORTED_SYMBOLS = (
    "sfmp_abi_version", "sfmp_status_string", "sfmp_last_error", "sfmp_device_count",
    "sfmp_parse_header", "sfmp_block_offsets", "sfmp_model_create",
    "sfmp_model_create_from_parts", "sfmp_model_create_shard", "sfmp_model_destroy",
    "sfmp_model_get_info", "sfmp_workspace_size", "sfmp_gemm", "sfmp_gemm_ex", "sfmp_gemm_host",
    "sfmp_dequantize", "sfmp_unpack_codes", "sfmp_unpermute_gathered", "sfmp_shard_plan",
    "sfmp_shard_extract", "sfmp_gemm_grouped", "sfmp_gemm_grouped_v", "sfmp_gemm_stats",
    "sfmp_gemm_host_stats", "sfmp_launch_count", "sfmp_sharded_gather_bytes", "sfmp_gemm_sharded_local",
    "sfmp_sharded_unpermute", "sfmp_gemm_sharded", "sfmp_nccl_unique_id", "sfmp_nccl_comm_init",
    "sfmp_nccl_comm_destroy", "sfmp_gemv_block", "sfmp_model_create_ex", "sfmp_model_create_shard_ex",
    "sfmp_gemm_norm", "sfmp_gemm_grouped_v_norm",
)
MODEL_DECODE_ONLY = 1
MODEL_LUT_LAYOUT = 2
NCCL_ID_BYTES = 128


class SfmpError(RuntimeError):
    code = -1


class ShapeError(SfmpError, ValueError):
    """sfmp::ShapeError (errors.hpp:9-12)."""


class ConfigError(SfmpError, ValueError):
    """sfmp::ConfigError (errors.hpp:14-17)."""


class FormatError(SfmpError):
    """sfmp::FormatError with .kind in {bad_magic, bad_version, truncated, invariant, io}."""

    def __init__(self, kind: str, msg: str):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind


class CudaError(SfmpError):
    pass


class UnsupportedError(SfmpError):
    pass


_FORMAT_KINDS = {E_MAGIC: "bad_magic", E_VERSION: "bad_version", E_TRUNC: "truncated",
                 E_INVARIANT: "invariant", E_IO: "io"}


class ModelInfo(C.Structure):
    _fields_ = [("rows", C.c_uint64), ("cols", C.c_uint64), ("m_b", C.c_uint32),
                ("n_b", C.c_uint32), ("floor_bits", C.c_int32), ("ceil_bits", C.c_int32),
                ("mode", C.c_int32), ("block_count", C.c_uint64), ("blocks_high", C.c_uint64),
                ("avg_code_bits", C.c_double), ("payload_bytes", C.c_uint64),
                ("device_bytes", C.c_uint64), ("shard", C.c_uint32), ("num_shards", C.c_uint32),
                ("out_rows", C.c_uint64), ("global_rows", C.c_uint64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class Stats(C.Structure):
    """sfmp_stats: the GPU counterpart of GemvStats (lutgemm.hpp:47-52)."""
    _fields_ = [("device_us", C.c_double), ("h2d_us", C.c_double), ("d2h_us", C.c_double),
                ("wall_us", C.c_double), ("bytes", C.c_uint64), ("flops", C.c_double),
                ("path", C.c_int32), ("launches", C.c_int32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class PreNorm(C.Structure):
    """sfmp_prenorm: RMSNorm fused into the activation pre-pass."""
    _fields_ = [("gamma", C.c_void_p), ("gamma_dtype", C.c_int), ("eps", C.c_float), ("enabled", C.c_int32)]


def _prenorm(norm):
    """norm = (gamma tensor or None, eps) -> PreNorm; None -> a disabled entry."""
    if norm is None:
        return PreNorm(None, F32, 0.0, 0)
    gamma, eps = norm
    if gamma is None:
        return PreNorm(None, F32, float(eps), 1)
    gamma = gamma.contiguous()
    return PreNorm(gamma.data_ptr(), _dtype_code(gamma), float(eps), 1)


_lib = None


def build(force: bool = False) -> str:
    """Compile libsfmp_b200.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
    if force:
        subprocess.run(["make", "-s", "-C", HERE, "clean"], check=True)
    subprocess.run(["make", "-s", "-j8", "-C", HERE], check=True)
    return LIB_PATH


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run paper_2602_01027_b200.build() "
                          "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp, sz, i64 = C.c_void_p, C.c_size_t, C.c_int64
    L.sfmp_abi_version.restype = C.c_int
    L.sfmp_status_string.restype = C.c_char_p
    L.sfmp_status_string.argtypes = [C.c_int]
    L.sfmp_last_error.restype = C.c_char_p
    L.sfmp_device_count.restype = C.c_int
    L.sfmp_parse_header.argtypes = [vp, sz, C.POINTER(ModelInfo)]
    L.sfmp_block_offsets.argtypes = [vp, sz, vp, C.c_uint64]
    L.sfmp_model_create.argtypes = [vp, sz, C.c_int, C.POINTER(vp)]
    L.sfmp_model_create_shard.argtypes = [vp, sz, C.c_int, C.c_uint32, C.c_uint32, C.POINTER(vp)]
    L.sfmp_model_destroy.argtypes = [vp]
    L.sfmp_model_get_info.argtypes = [vp, C.POINTER(ModelInfo)]
    L.sfmp_workspace_size.argtypes = [vp, i64, C.c_int, C.POINTER(sz)]
    L.sfmp_gemm.argtypes = [vp, vp, C.c_int, i64, vp, vp, sz, vp]
    L.sfmp_gemm_ex.argtypes = [vp, vp, C.c_int, i64, vp, vp, sz, C.c_int, vp]
    L.sfmp_gemm_host.argtypes = [vp, vp, i64, vp, vp]
    L.sfmp_dequantize.argtypes = [vp, vp, vp]
    L.sfmp_unpack_codes.argtypes = [vp, vp, vp]
    L.sfmp_unpermute_gathered.argtypes = [vp, vp, i64, vp, vp]
    L.sfmp_shard_plan.argtypes = [vp, sz, C.c_uint32, vp, C.POINTER(C.c_uint64)]
    L.sfmp_gemm_grouped.argtypes = [vp, vp, C.c_int, i64, vp, vp, vp, C.c_int, vp]
    L.sfmp_gemm_grouped_v.argtypes = [vp, vp, C.c_int, vp, vp, vp, vp, C.c_int, vp]
    L.sfmp_shard_extract.argtypes = [vp, sz, C.c_uint32, C.c_uint32, vp, C.POINTER(C.c_size_t)]
    L.sfmp_gemm_stats.argtypes = [vp, vp, C.c_int, i64, vp, vp, sz, C.c_int, vp, C.POINTER(Stats)]
    L.sfmp_gemm_host_stats.argtypes = [vp, vp, i64, vp, vp, C.POINTER(Stats)]
    L.sfmp_launch_count.restype = C.c_uint64
    L.sfmp_sharded_gather_bytes.argtypes = [vp, vp, C.c_int, C.POINTER(sz)]
    L.sfmp_gemm_sharded_local.argtypes = [vp, vp, C.c_int, vp, vp, vp, C.c_int, vp, vp]
    L.sfmp_sharded_unpermute.argtypes = [vp, vp, C.c_int, vp, vp, vp]
    L.sfmp_gemm_sharded.argtypes = [vp, vp, C.c_int, vp, vp, vp, vp, C.c_int, vp, sz, vp, vp]
    L.sfmp_nccl_unique_id.argtypes = [vp]
    L.sfmp_nccl_comm_init.argtypes = [C.c_int, vp, C.c_int, C.c_int, C.POINTER(vp)]
    L.sfmp_nccl_comm_destroy.argtypes = [vp]
    L.sfmp_gemv_block.argtypes = [vp, C.c_uint64, vp, vp, vp]
    L.sfmp_gemm_norm.argtypes = [vp, vp, C.c_int, i64, vp, vp, sz, C.POINTER(PreNorm), vp]
    L.sfmp_gemm_grouped_v_norm.argtypes = [vp, vp, C.c_int, vp, vp, vp, vp, C.c_int, C.POINTER(PreNorm), vp]
    L.sfmp_model_create_ex.argtypes = [vp, sz, C.c_int, C.c_uint32, C.POINTER(vp)]
    L.sfmp_model_create_shard_ex.argtypes = [vp, sz, C.c_int, C.c_uint32, C.c_uint32, C.c_uint32, C.POINTER(vp)]
    for name in ("sfmp_parse_header", "sfmp_block_offsets", "sfmp_model_create",
                 "sfmp_model_create_shard", "sfmp_model_destroy", "sfmp_model_get_info",
                 "sfmp_workspace_size", "sfmp_gemm", "sfmp_gemm_ex", "sfmp_gemm_host",
                 "sfmp_dequantize", "sfmp_unpack_codes", "sfmp_unpermute_gathered",
                 "sfmp_shard_plan", "sfmp_shard_extract", "sfmp_gemm_grouped", "sfmp_gemm_grouped_v",
                 "sfmp_gemm_stats", "sfmp_gemm_host_stats", "sfmp_sharded_gather_bytes",
                 "sfmp_gemm_sharded_local", "sfmp_sharded_unpermute", "sfmp_gemm_sharded",
                 "sfmp_nccl_unique_id", "sfmp_nccl_comm_init", "sfmp_nccl_comm_destroy", "sfmp_gemv_block",
                 "sfmp_model_create_ex", "sfmp_model_create_shard_ex", "sfmp_gemm_norm",
                 "sfmp_gemm_grouped_v_norm"):
        getattr(L, name).restype = C.c_int
    _lib = L
    return L


def check(status: int) -> None:
    if status == OK:
        return
    msg = lib().sfmp_last_error().decode(errors="replace")
    if status == E_SHAPE:
        raise ShapeError(msg)
    if status == E_CONFIG:
        raise ConfigError(msg)
    if status in _FORMAT_KINDS:
        raise FormatError(_FORMAT_KINDS[status], msg)
    if status == E_CUDA:
        raise CudaError(msg)
    if status == E_UNSUPPORTED:
        raise UnsupportedError(msg)
    e = SfmpError(f"{lib().sfmp_status_string(status).decode()}: {msg}")
    e.code = status
    raise e


def launch_count() -> int:
    """Kernels enqueued by this host thread through the library so far."""
    return int(lib().sfmp_launch_count())


def device_count() -> int:
    return int(lib().sfmp_device_count())


def parse_header(data: bytes) -> dict:
    """Validate an SFMPPKD1 stream on the host (deserialize + validate)."""
    info = ModelInfo()
    check(lib().sfmp_parse_header(data, len(data), C.byref(info)))
    return info.as_dict()


def compute_block_offsets(data: bytes) -> np.ndarray:
    """compute_block_offsets (layout.cpp:301-314)."""
    K = parse_header(data)["block_count"]
    out = np.zeros(K, np.uint64)
    check(lib().sfmp_block_offsets(data, len(data), out.ctypes.data, K))
    return out


def shard_plan(data: bytes, num_shards: int):
    """Snake block-row partition: (gather_map[num_shards, shard_rows], shard_rows)."""
    sr = C.c_uint64(0)
    check(lib().sfmp_shard_plan(data, len(data), num_shards, None, C.byref(sr)))
    gmap = np.zeros(num_shards * sr.value, np.uint32)
    check(lib().sfmp_shard_plan(data, len(data), num_shards, gmap.ctypes.data, C.byref(sr)))
    return gmap.reshape(num_shards, sr.value), int(sr.value)


def shard_extract(data: bytes, shard: int, num_shards: int) -> bytes:
    """The shard's block rows as a stand-alone SFMPPKD1 stream (host only)."""
    n = C.c_size_t(0)
    check(lib().sfmp_shard_extract(data, len(data), shard, num_shards, None, C.byref(n)))
    buf = (C.c_uint8 * n.value)()
    check(lib().sfmp_shard_extract(data, len(data), shard, num_shards, buf, C.byref(n)))
    return bytes(buf)


def assemble_gathered(gathered: np.ndarray, gather_map: np.ndarray, rows: int) -> np.ndarray:
    """Host mirror of sfmp_unpermute_gathered: gathered[G, M, SR] -> y[M, rows]."""
    G, M, SR = gathered.shape
    y = np.zeros((M, rows), gathered.dtype)
    gm = gather_map.reshape(G * SR)
    valid = gm != 0xFFFFFFFF
    flat = gathered.transpose(1, 0, 2).reshape(M, G * SR)
    y[:, gm[valid]] = flat[:, valid]
    return y


def _dtype_code(t) -> int:
    import torch
    return {torch.float32: F32, torch.float16: F16, torch.bfloat16: BF16}[t.dtype]


def _stream_ptr(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


class DeviceModel:
    """A packed model resident on one B200 (sfmp_model_create)."""

    def __init__(self, data: bytes, device: int = 0, shard: int | None = None,
                 num_shards: int = 1, flags: int = 0):
        """flags: MODEL_DECODE_ONLY keeps only the decode layout (~1x payload)."""
        self._h = C.c_void_p()
        self._data_len = len(data)
        if shard is None:
            check(lib().sfmp_model_create_ex(data, len(data), device, flags, C.byref(self._h)))
        else:
            check(lib().sfmp_model_create_shard_ex(data, len(data), device, shard, num_shards, flags,
                                                   C.byref(self._h)))
        info = ModelInfo()
        check(lib().sfmp_model_get_info(self._h, C.byref(info)))
        self.info = info.as_dict()
        self.device = device
        self.rows, self.cols = self.info["rows"], self.info["cols"]
        self.out_rows = self.info["out_rows"]
        self._ws = {}

    def close(self):
        if self._h:
            lib().sfmp_model_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def workspace_bytes(self, M: int, path: int = PATH_AUTO) -> int:
        n = C.c_size_t(0)
        check(lib().sfmp_workspace_size(self._h, M, path, C.byref(n)))
        return int(n.value)

    def workspace(self, M: int, path: int = PATH_AUTO):
        import torch
        nbytes = self.workspace_bytes(M, path)
        key = (path, nbytes)
        if nbytes and key not in self._ws:
            self._ws[key] = torch.zeros(nbytes, dtype=torch.uint8, device=f"cuda:{self.device}")
        return self._ws.get(key)

    def gemm(self, x, out=None, path: int = PATH_AUTO, workspace=None, stream=None, norm=None):
        """y[M, out_rows] (f32) = x[M, cols] . W^T, x/y torch CUDA tensors, original order.
        norm=(gamma, eps): x is the unnormalised hidden state, RMSNorm fused (sfmp_gemm_norm)."""
        import torch
        if x.dim() == 1:
            x = x.unsqueeze(0)
        if x.shape[-1] != self.cols:
            raise ShapeError("gemv: x.len != model cols")
        x = x.contiguous()
        M = x.shape[0]
        if out is None:
            out = torch.empty(M, self.out_rows, dtype=torch.float32, device=x.device)
        ws = workspace if workspace is not None else self.workspace(M, path)
        if norm is not None:
            if path != PATH_AUTO:
                raise ConfigError("a fused norm takes the automatic path")
            pn = _prenorm(norm)
            check(lib().sfmp_gemm_norm(self._h, C.c_void_p(x.data_ptr()), _dtype_code(x), M,
                                       C.c_void_p(out.data_ptr()),
                                       C.c_void_p(ws.data_ptr()) if ws is not None else None,
                                       ws.numel() if ws is not None else 0, C.byref(pn), _stream_ptr(stream)))
            return out
        check(lib().sfmp_gemm_ex(self._h, C.c_void_p(x.data_ptr()), _dtype_code(x), M,
                                 C.c_void_p(out.data_ptr()),
                                 C.c_void_p(ws.data_ptr()) if ws is not None else None,
                                 ws.numel() if ws is not None else 0, path, _stream_ptr(stream)))
        return out

    def gemm_stats(self, x, out=None, path: int = PATH_AUTO, workspace=None, stream=None):
        """gemm() that also returns the call's sfmp_stats (synchronises the stream)."""
        import torch
        if x.dim() == 1:
            x = x.unsqueeze(0)
        x = x.contiguous()
        M = x.shape[0]
        if out is None:
            out = torch.empty(M, self.out_rows, dtype=torch.float32, device=x.device)
        ws = workspace if workspace is not None else self.workspace(M, path)
        st = Stats()
        check(lib().sfmp_gemm_stats(self._h, C.c_void_p(x.data_ptr()), _dtype_code(x), M,
                                    C.c_void_p(out.data_ptr()),
                                    C.c_void_p(ws.data_ptr()) if ws is not None else None,
                                    ws.numel() if ws is not None else 0, path, _stream_ptr(stream),
                                    C.byref(st)))
        return out, st.as_dict()

    def gemm_host(self, x: np.ndarray, stats: bool = False):
        """Reference calling convention: host f32 in, host f32 out (copies inside).
        stats=True also returns the sfmp_stats dict (GemvStats counterpart)."""
        x = np.ascontiguousarray(np.atleast_2d(x), np.float32)
        if x.shape[-1] != self.cols:
            raise ShapeError("gemv: x.len != model cols")
        y = np.empty((x.shape[0], self.out_rows), np.float32)
        st = Stats()
        check(lib().sfmp_gemm_host_stats(self._h, x.ctypes.data, x.shape[0], y.ctypes.data, None,
                                         C.byref(st) if stats else None))
        return (y, st.as_dict()) if stats else y

    def gemv_block(self, block: int, x_reordered, stream=None):
        """gemv_block (lutgemm.cpp:87-93): the m_b-row contribution of block k to
        y in STORED (reordered) row order, from the reordered x (device f32)."""
        import torch
        out = torch.empty(self.info["m_b"], dtype=torch.float32, device=x_reordered.device)
        x_reordered = x_reordered.contiguous().float()
        check(lib().sfmp_gemv_block(self._h, block, C.c_void_p(x_reordered.data_ptr()),
                                    C.c_void_p(out.data_ptr()), _stream_ptr(stream)))
        return out

    def dequantize(self, stream=None):
        import torch
        w = torch.empty(self.out_rows, self.cols, dtype=torch.float32,
                        device=f"cuda:{self.device}")
        check(lib().sfmp_dequantize(self._h, C.c_void_p(w.data_ptr()), _stream_ptr(stream)))
        return w

    def unpack_codes(self, stream=None):
        import torch
        c = torch.empty(self.rows, self.cols, dtype=torch.uint8, device=f"cuda:{self.device}")
        check(lib().sfmp_unpack_codes(self._h, C.c_void_p(c.data_ptr()), _stream_ptr(stream)))
        return c

    def unpermute_gathered(self, gathered, M: int, out=None, stream=None):
        """[num_shards, M, shard_rows] all-gathered shard outputs -> y[M, rows] original order."""
        import torch
        if out is None:
            out = torch.empty(M, self.info["global_rows"], dtype=torch.float32,
                              device=gathered.device)
        check(lib().sfmp_unpermute_gathered(self._h, C.c_void_p(gathered.data_ptr()), M,
                                            C.c_void_p(out.data_ptr()), _stream_ptr(stream)))
        return out


def gemm_grouped(models, xs, outs=None, workspaces=None, stream=None, norms=None):
    """Independent linears in one call: y_i = x_i . W_i^T, x_i [M_i, cols_i] of one
    dtype (M_i may differ: sfmp_gemm_grouped_v).  Decode problems (M_i <= 16) of
    one n-tile class (M <= 8 or 9..16) with distinct workspaces share one
    activation pre-pass + one GEMV launch."""
    import torch
    n = len(models)
    xs = [x.contiguous() for x in xs]
    dt = _dtype_code(xs[0])
    for m, x in zip(models, xs):
        if x.dim() != 2 or x.shape[1] != m.cols or _dtype_code(x) != dt:
            raise ShapeError("gemm_grouped: every x must be [M, cols] of one dtype")
    Ms = [x.shape[0] for x in xs]
    if outs is None:
        outs = [torch.empty(M, m.out_rows, dtype=torch.float32, device=x.device) for m, x, M in zip(models, xs, Ms)]
    if workspaces is None:
        workspaces = [m.workspace(min(M, 16) if M <= 16 else M) for m, M in zip(models, Ms)]
    P = C.c_void_p * n
    hs = P(*[m.handle for m in models])
    xp = P(*[x.data_ptr() for x in xs])
    yp = P(*[y.data_ptr() for y in outs])
    wp = P(*[(w.data_ptr() if w is not None else None) for w in workspaces])
    wb = (C.c_size_t * n)(*[(w.numel() if w is not None else 0) for w in workspaces])
    mp = (C.c_int64 * n)(*Ms)
    if norms is not None:  # one (gamma, eps) per problem: RMSNorm fused into the pre-pass
        pn = (PreNorm * n)(*[_prenorm(v) for v in norms])
        check(lib().sfmp_gemm_grouped_v_norm(hs, xp, dt, mp, yp, wp, wb, n, pn, _stream_ptr(stream)))
        return outs
    check(lib().sfmp_gemm_grouped_v(hs, xp, dt, mp, yp, wp, wb, n, _stream_ptr(stream)))
    return outs


def gemv(model: DeviceModel, x, stream=None):
    """sfmp::gemv (lutgemm.hpp:57): one token (or M tokens looped)."""
    y = model.gemm(x, stream=stream)
    return y[0] if x.dim() == 1 else y


# ---------------------------------------------------------------------------
# Sharded calls: several N-sharded linears, ONE collective
# ---------------------------------------------------------------------------
class NcclComm:
    """An NCCL communicator created through the library (libnccl.so.2 at run
    time).  The unique id travels over any channel, e.g. torch.distributed."""

    def __init__(self, nranks: int, rank: int, device: int, uid: bytes):
        self._h = C.c_void_p()
        buf = (C.c_uint8 * NCCL_ID_BYTES).from_buffer_copy(uid)
        check(lib().sfmp_nccl_comm_init(nranks, buf, rank, device, C.byref(self._h)))
        self.nranks, self.rank = nranks, rank

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * NCCL_ID_BYTES)()
        check(lib().sfmp_nccl_unique_id(buf))
        return bytes(buf)

    @property
    def handle(self):
        return self._h

    def close(self):
        if self._h:
            lib().sfmp_nccl_comm_destroy(self._h)
            self._h = C.c_void_p()


def _ptr_array(vals):
    return (C.c_void_p * len(vals))(*vals)


def sharded_gather_bytes(models, Ms) -> int:
    n = C.c_size_t(0)
    check(lib().sfmp_sharded_gather_bytes(_ptr_array([m.handle for m in models]),
                                          (C.c_int64 * len(Ms))(*Ms), len(models), C.byref(n)))
    return int(n.value)


def packed_offsets(models, Ms):
    """Float offsets of each problem in one rank's send block (+ total)."""
    off = [0]
    for m, M in zip(models, Ms):
        off.append(off[-1] + M * m.out_rows)
    return off


def gemm_sharded_local(models, xs, gather_buf, workspaces, stream=None):
    """Step 1 of a sharded call: the shard GEMMs into the send block of gather_buf."""
    n = len(models)
    xs = [x.contiguous() for x in xs]
    check(lib().sfmp_gemm_sharded_local(
        _ptr_array([m.handle for m in models]), _ptr_array([x.data_ptr() for x in xs]), _dtype_code(xs[0]),
        (C.c_int64 * n)(*[x.shape[0] for x in xs]), _ptr_array([w.data_ptr() for w in workspaces]),
        (C.c_size_t * n)(*[w.numel() for w in workspaces]), n, C.c_void_p(gather_buf.data_ptr()),
        _stream_ptr(stream)))


def sharded_unpermute(models, Ms, gather_buf, outs, stream=None):
    """Step 3: every problem's gathered rows to outs[i][M_i, global rows] (one launch)."""
    n = len(models)
    check(lib().sfmp_sharded_unpermute(_ptr_array([m.handle for m in models]), (C.c_int64 * n)(*Ms), n,
                                       C.c_void_p(gather_buf.data_ptr()), _ptr_array([y.data_ptr() for y in outs]),
                                       _stream_ptr(stream)))
    return outs


def gemm_sharded(models, xs, outs, workspaces, gather_buf, comm: NcclComm, stream=None):
    """Steps 1-3 with the library's NCCL all-gather (sfmp_gemm_sharded)."""
    n = len(models)
    xs = [x.contiguous() for x in xs]
    check(lib().sfmp_gemm_sharded(
        _ptr_array([m.handle for m in models]), _ptr_array([x.data_ptr() for x in xs]), _dtype_code(xs[0]),
        (C.c_int64 * n)(*[x.shape[0] for x in xs]), _ptr_array([y.data_ptr() for y in outs]),
        _ptr_array([w.data_ptr() for w in workspaces]), (C.c_size_t * n)(*[w.numel() for w in workspaces]), n,
        C.c_void_p(gather_buf.data_ptr()), gather_buf.numel() * gather_buf.element_size(), comm.handle,
        _stream_ptr(stream)))
    return outs
