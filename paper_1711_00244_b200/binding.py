"""ctypes marshalling for include/cdn.h.  Names mirror the C ABI."""
from __future__ import annotations

import ctypes as C
import os
from typing import List, Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
lib_path = os.path.join(_HERE, "libcdn.so")

CDN_LAYER_FC, CDN_LAYER_CONV = 0, 1

_STATUS = {0: "CDN_OK", -1: "CDN_E_ARG", -2: "CDN_E_MAGIC", -3: "CDN_E_VERSION", -4: "CDN_E_TRUNCATED",
           -5: "CDN_E_MALFORMED", -6: "CDN_E_UNSUPPORTED", -7: "CDN_E_SHAPE", -8: "CDN_E_OOM",
           -9: "CDN_E_INFEASIBLE", -10: "CDN_E_CUDA", -11: "CDN_E_NCCL", -12: "CDN_E_STATE"}


class CDNError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status
        self.name = _STATUS.get(status, str(status))


class LayerDesc(C.Structure):
    _fields_ = [("kind", C.c_int32), ("relu", C.c_int32), ("in_c", C.c_int32), ("in_h", C.c_int32),
                ("in_w", C.c_int32), ("kh", C.c_int32), ("kw", C.c_int32), ("stride", C.c_int32),
                ("pad", C.c_int32), ("groups", C.c_int32), ("lrn", C.c_int32), ("pool_k", C.c_int32),
                ("pool_s", C.c_int32)]

    @classmethod
    def conv(cls, in_c: int, in_h: int, in_w: int, kh: int, kw: int, stride: int, pad: int, groups: int = 1,
             relu: bool = True, lrn: bool = False, pool_k: int = 0, pool_s: int = 0) -> "LayerDesc":
        d = cls()
        d.kind = CDN_LAYER_CONV
        d.relu = int(bool(relu))
        d.in_c, d.in_h, d.in_w = in_c, in_h, in_w
        d.kh, d.kw, d.stride, d.pad, d.groups = kh, kw, stride, pad, groups
        d.lrn, d.pool_k, d.pool_s = int(bool(lrn)), pool_k, pool_s
        return d

    @classmethod
    def fc(cls, relu: bool) -> "LayerDesc":
        d = cls()
        d.kind = CDN_LAYER_FC
        d.relu = int(bool(relu))
        d.groups = 1
        return d


class LayerStats(C.Structure):
    _fields_ = [("rows", C.c_uint32), ("cols", C.c_uint32), ("row_begin", C.c_uint32),
                ("row_end", C.c_uint32), ("k", C.c_uint32), ("r", C.c_uint32),
                ("lanes_per_row", C.c_uint32), ("max_len_val", C.c_uint32), ("max_len_gap", C.c_uint32),
                ("tokens", C.c_uint64), ("nnz", C.c_uint64), ("stream_bytes", C.c_uint64),
                ("algo_bytes_fixed", C.c_uint64), ("index_bytes", C.c_uint64), ("ws_bytes", C.c_uint64),
                ("in_features", C.c_uint64), ("out_features", C.c_uint64), ("resident_bytes", C.c_uint64),
                ("call_index_bytes", C.c_uint64), ("col_begin", C.c_uint32), ("col_end", C.c_uint32)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


_lib = None

_SIGS = {
    "cdn_abi_version": (C.c_int, []),
    "cdn_last_error": (C.c_char_p, []),
    "cdn_nccl_unique_id": (C.c_int32, [C.c_void_p]),
    "cdn_model_create": (C.c_int32, [C.c_int, C.c_int, C.c_int, C.c_void_p, C.POINTER(C.c_void_p)]),
    "cdn_model_destroy": (None, [C.c_void_p]),
    "cdn_model_load_layer": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.POINTER(LayerDesc),
                                         C.POINTER(C.c_int)]),
    "cdn_model_set_memory_budget": (C.c_int32, [C.c_void_p, C.c_uint64, C.c_double]),
    "cdn_model_plan": (C.c_int32, [C.c_void_p, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_double)]),
    "cdn_model_set_plan": (C.c_int32, [C.c_void_p, C.POINTER(C.c_int), C.c_int]),
    "cdn_model_infer": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_void_p]),
    "cdn_model_set_sharding": (C.c_int32, [C.c_void_p, C.c_int]),
    "cdn_col_block": (C.c_int32, [C.c_uint32, C.c_int, C.c_int, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]),
    "cdn_model_scratch_bytes": (C.c_int32, [C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.c_int]),
    "cdn_model_release_scratch": (C.c_int32, [C.c_void_p]),
    "cdn_layer_forward": (C.c_int32, [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int,
                                      C.c_void_p]),
    "cdn_layer_decode": (C.c_int32, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                     C.POINTER(C.c_uint64), C.c_void_p]),
    "cdn_model_set_kernel_policy": (C.c_int32, [C.c_void_p, C.c_int, C.c_int]),
    "cdn_conv_forward": (C.c_int32, [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]),
    "cdn_layer_out_shape": (C.c_int32, [C.c_void_p, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                        C.POINTER(C.c_int)]),
    "cdn_debug_gemm_bf16": (C.c_int32, [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int,
                                        C.c_void_p, C.c_int, C.c_void_p]),
    "cdn_debug_kernel_launches": (C.c_int32, [C.POINTER(C.c_uint64)]),
    "cdn_debug_kernel_timer": (C.c_int32, [C.c_int]),
    "cdn_debug_kernel_timer_read": (C.c_int32, [C.c_char_p, C.POINTER(C.c_double), C.POINTER(C.c_int)]),
    "cdn_model_memory_model": (C.c_int32, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]),
    "cdn_layer_kernel_name": (C.c_char_p, [C.c_void_p, C.c_int, C.c_int]),
    "cdn_model_num_layers": (C.c_int32, [C.c_void_p, C.POINTER(C.c_int)]),
    "cdn_layer_stats_get": (C.c_int32, [C.c_void_p, C.c_int, C.POINTER(LayerStats)]),
    "cdn_model_profile": (C.c_int32, [C.c_void_p, C.c_int, C.c_int, C.c_void_p]),
    "cdn_compress_dense": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint32, C.c_double, C.c_int,
                                       C.c_int, C.POINTER(C.c_void_p), C.POINTER(C.c_size_t)]),
    "cdn_compress_dense_q": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint32, C.c_double, C.c_int,
                                         C.c_int, C.c_int, C.c_uint32, C.c_uint32, C.POINTER(C.c_void_p),
                                         C.POINTER(C.c_size_t)]),
    "cdn_free": (None, [C.c_void_p]),
    "cdn_plan_dp": (C.c_int32, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_uint64,
                                C.c_double, C.c_uint64, C.c_void_p, C.POINTER(C.c_double)]),
    "cdn_debug_host_walk_shard": (C.c_int32, [C.c_void_p, C.c_size_t, C.c_int, C.c_int, C.c_int, C.c_void_p,
                                              C.c_void_p, C.c_void_p, C.POINTER(C.c_uint64)]),
    "cdn_debug_host_walk": (C.c_int32, [C.c_void_p, C.c_size_t, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                        C.POINTER(C.c_uint64)]),
}


def load_library():
    """Load libcdn.so (raises if it is missing: there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(lib_path):
        raise ImportError(f"{lib_path} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(lib_path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def _check(status: int):
    if status != 0:
        msg = load_library().cdn_last_error()
        raise CDNError(status, msg.decode() if msg else "")


def abi_version() -> int:
    return load_library().cdn_abi_version()


def _ptr(t) -> int:
    """Device/host address of a torch tensor or numpy array."""
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _check(load_library().cdn_nccl_unique_id(buf))
    return bytes(buf)


def compress_dense(W: np.ndarray, density: float, r: int, k: int, bias: Optional[np.ndarray] = None,
                   quantizer: str = "linear", bh: int = 1, bw: int = 0) -> bytes:
    """Product-side compressor: dense fp32 -> single-layer CDNI bytes
    (quantizer "linear" = C-05 grid, "kmeans" = Lloyd refinement, C-33;
    bh x bw != 1 x cols: the block-contiguous container of Alg. 2, C-34)."""
    W = np.ascontiguousarray(W, dtype=np.float32)
    b = None if bias is None else np.ascontiguousarray(bias, dtype=np.float32)
    out = C.c_void_p()
    n = C.c_size_t()
    lib = load_library()
    qz = {"linear": 0, "kmeans": 1}[quantizer]
    _check(lib.cdn_compress_dense_q(W.ctypes.data, None if b is None else b.ctypes.data, W.shape[0], W.shape[1],
                                    float(density), int(r), int(k), qz, int(bh), int(bw), C.byref(out),
                                    C.byref(n)))
    try:
        return C.string_at(out, n.value)
    finally:
        lib.cdn_free(out)


def plan_dp(time_ms: np.ndarray, in_bytes: Sequence[int], out_bytes: Sequence[int], ws: Sequence[int],
            tot: int, latency_ms: float = 0.0, step: int = 1) -> Tuple[List[int], float]:
    """C++ DP on a given Time table (time_ms[i, B-1])."""
    t = np.ascontiguousarray(time_ms, dtype=np.float64)
    f, Bmax = t.shape
    ib = np.ascontiguousarray(in_bytes, dtype=np.uint64)
    ob = np.ascontiguousarray(out_bytes, dtype=np.uint64)
    wb = np.ascontiguousarray(ws, dtype=np.uint64)
    bs = np.zeros(f, dtype=np.int32)
    opt = C.c_double()
    _check(load_library().cdn_plan_dp(t.ctypes.data, ib.ctypes.data, ob.ctypes.data, wb.ctypes.data, f, Bmax,
                                      int(tot), float(latency_ms), int(step), bs.ctypes.data, C.byref(opt)))
    return bs.tolist(), opt.value


def kernel_launches() -> int:
    """Kernels the library has launched since it was loaded (cdn_debug_kernel_launches)."""
    out = C.c_uint64(0)
    _check(load_library().cdn_debug_kernel_launches(C.byref(out)))
    return int(out.value)


def kernel_timer(enable: bool):
    """Start (True) or stop (False) recording per-kernel CUDA-event durations; drops old records."""
    _check(load_library().cdn_debug_kernel_timer(1 if enable else 0))


def kernel_time(kernel: str):
    """(total ms, launches) recorded for `kernel` since kernel_timer(True)."""
    ms, n = C.c_double(0.0), C.c_int(0)
    _check(load_library().cdn_debug_kernel_timer_read(kernel.encode(), C.byref(ms), C.byref(n)))
    return float(ms.value), int(n.value)


def debug_gemm_bf16(A, M: int, Wt, N: int, Kpad: int, bias, relu: bool, out, ldo: int, stream: int = 0):
    """tcgen05 GEMM test hook (device tensors; A/Wt bf16 bit patterns)."""
    _check(load_library().cdn_debug_gemm_bf16(_ptr(A), int(M), _ptr(Wt), int(N), int(Kpad), _ptr(bias),
                                              int(bool(relu)), _ptr(out), int(ldo), stream or None))


CDN_SHARD_ROWS, CDN_SHARD_COLS = 0, 1


def col_block(cols: int, rank: int, world: int) -> Tuple[int, int]:
    """Input columns [k0, k1) rank `rank` of `world` multiplies in a column-sharded layer."""
    lib = load_library()
    k0, k1 = C.c_uint32(), C.c_uint32()
    _check(lib.cdn_col_block(int(cols), int(rank), int(world), C.byref(k0), C.byref(k1)))
    return k0.value, k1.value


def debug_host_walk_shard(cdni: bytes, rank: int, world: int, layer_in_file: int = 0):
    """Host walk of one rank's row-block shard (tokens with global row indices)."""
    lib = load_library()
    n = C.c_uint64()
    _check(lib.cdn_debug_host_walk_shard(cdni, len(cdni), layer_in_file, rank, world, None, None, None, C.byref(n)))
    row = np.zeros(n.value, np.int32)
    col = np.zeros(n.value, np.int32)
    sym = np.zeros(n.value, np.uint8)
    _check(lib.cdn_debug_host_walk_shard(cdni, len(cdni), layer_in_file, rank, world, row.ctypes.data,
                                         col.ctypes.data, sym.ctypes.data, C.byref(n)))
    return row, col, sym


def debug_host_walk(cdni: bytes, layer_in_file: int = 0):
    lib = load_library()
    n = C.c_uint64()
    _check(lib.cdn_debug_host_walk(cdni, len(cdni), layer_in_file, None, None, None, C.byref(n)))
    row = np.zeros(n.value, np.int32)
    col = np.zeros(n.value, np.int32)
    sym = np.zeros(n.value, np.uint8)
    _check(lib.cdn_debug_host_walk(cdni, len(cdni), layer_in_file, row.ctypes.data, col.ctypes.data,
                                   sym.ctypes.data, C.byref(n)))
    return row, col, sym


class Model:
    """Owns a cdn_model handle (one per GPU / rank)."""

    def __init__(self, device: int = 0, rank: int = 0, world: int = 1, nccl_id: Optional[bytes] = None):
        self._lib = load_library()
        h = C.c_void_p()
        idbuf = None if nccl_id is None else (C.c_uint8 * 128).from_buffer_copy(nccl_id)
        _check(self._lib.cdn_model_create(device, rank, world, idbuf, C.byref(h)))
        self._h = h
        self.device, self.rank, self.world = device, rank, world

    def close(self):
        if getattr(self, "_h", None):
            self._lib.cdn_model_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def load_layer(self, cdni: bytes, desc: LayerDesc, layer_in_file: int = 0) -> int:
        idx = C.c_int()
        _check(self._lib.cdn_model_load_layer(self._h, cdni, len(cdni), layer_in_file, C.byref(desc),
                                              C.byref(idx)))
        return idx.value

    def set_memory_budget(self, tot_bytes: int, latency_ms: float = 0.0):
        _check(self._lib.cdn_model_set_memory_budget(self._h, int(tot_bytes), float(latency_ms)))

    def set_plan(self, batches: Optional[Sequence[int]]):
        b = list(batches or [])
        arr = (C.c_int * max(1, len(b)))(*b)
        _check(self._lib.cdn_model_set_plan(self._h, arr, len(b)))

    def plan(self, K: int) -> Tuple[List[int], float]:
        n = self.num_layers()
        arr = (C.c_int * n)()
        ms = C.c_double()
        _check(self._lib.cdn_model_plan(self._h, int(K), arr, C.byref(ms)))
        return list(arr), ms.value

    def infer(self, inp, K: int, scores, on_device: bool, stream: int = 0):
        _check(self._lib.cdn_model_infer(self._h, _ptr(inp), int(K), _ptr(scores), int(bool(on_device)),
                                         stream or None))

    def layer_forward(self, layer: int, x, ldx: int, B: int, y, ldy: int, stream: int = 0):
        _check(self._lib.cdn_layer_forward(self._h, layer, _ptr(x), ldx, B, _ptr(y), ldy, stream or None))

    def conv_forward(self, layer: int, x, B: int, y, stream: int = 0):
        """NHWC device batch through one CONV layer (decode -> im2col -> tcgen05 GEMM -> ReLU/LRN/pool)."""
        _check(self._lib.cdn_conv_forward(self._h, layer, _ptr(x), int(B), _ptr(y), stream or None))

    def out_shape(self, layer: int) -> Tuple[int, int, int]:
        h, w, c = C.c_int(), C.c_int(), C.c_int()
        _check(self._lib.cdn_layer_out_shape(self._h, layer, C.byref(h), C.byref(w), C.byref(c)))
        return h.value, w.value, c.value

    def kernel_name(self, layer: int, B: int) -> str:
        return self._lib.cdn_layer_kernel_name(self._h, layer, int(B)).decode()

    def memory_model(self, Bmax: int):
        """(IN per image, OUT per image, WS) bytes per layer, as the planner sees them."""
        n = self.num_layers()
        a, b, c = (np.zeros(n, np.uint64) for _ in range(3))
        _check(self._lib.cdn_model_memory_model(self._h, int(Bmax), a.ctypes.data, b.ctypes.data, c.ctypes.data))
        return a.tolist(), b.tolist(), c.tolist()

    def set_kernel_policy(self, band_min_batch: int = 0, tc_min_batch: int = 0):
        """B >= tc_min_batch -> tensor-core kernel; B >= band_min_batch -> band kernel (0: defaults)."""
        _check(self._lib.cdn_model_set_kernel_policy(self._h, int(band_min_batch), int(tc_min_batch)))

    def set_sharding(self, mode: int):
        """CDN_SHARD_ROWS (0) or CDN_SHARD_COLS (1); before loading layers."""
        _check(self._lib.cdn_model_set_sharding(self._h, int(mode)))

    def scratch_bytes(self, reset_peak: bool = False) -> Tuple[int, int]:
        """(current, high-water) bytes of inference scratch (cdn_model_scratch_bytes)."""
        cur, peak = C.c_uint64(), C.c_uint64()
        _check(self._lib.cdn_model_scratch_bytes(self._h, C.byref(cur), C.byref(peak), int(bool(reset_peak))))
        return cur.value, peak.value

    def release_scratch(self):
        _check(self._lib.cdn_model_release_scratch(self._h))

    def decode_count(self, layer: int) -> int:
        n = C.c_uint64()
        _check(self._lib.cdn_layer_decode(self._h, layer, None, None, None, None, C.byref(n), None))
        return n.value

    def decode(self, layer: int, row, col, sym, val, stream: int = 0) -> int:
        n = C.c_uint64()
        _check(self._lib.cdn_layer_decode(self._h, layer, _ptr(row), _ptr(col), _ptr(sym), _ptr(val),
                                          C.byref(n), stream or None))
        return n.value

    def num_layers(self) -> int:
        n = C.c_int()
        _check(self._lib.cdn_model_num_layers(self._h, C.byref(n)))
        return n.value

    def stats(self, layer: int) -> dict:
        s = LayerStats()
        _check(self._lib.cdn_layer_stats_get(self._h, layer, C.byref(s)))
        return s.as_dict()

    def profile(self, Bmax: int, reps: int = 5) -> np.ndarray:
        n = self.num_layers()
        out = np.zeros((n, Bmax), dtype=np.float64)
        _check(self._lib.cdn_model_profile(self._h, int(Bmax), int(reps), out.ctypes.data))
        return out
