"""ctypes binding of libbitstack.so (include/bitstack.h) -- argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels; this module only
turns numpy arrays / torch tensors into pointers and status codes into
exceptions.  There is no CPU fallback: if the library is missing or the GPU is
not an sm_100 device, calls fail loudly.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BITSTACK_LIB", os.path.join(HERE, "libbitstack.so"))

F32, BF16, F16 = 0, 1, 2
KERNEL_AUTO, KERNEL_TC, KERNEL_SIMT, KERNEL_PREFILL, KERNEL_RGEMV = 0, 1, 2, 3, 4
_DTYPE_NAMES = {"f32": F32, "float32": F32, "bf16": BF16, "bfloat16": BF16, "f16": F16, "float16": F16}

STATUS = {
    0: "OK", -1: "E_INVALID_ARG", -2: "E_DIM_MISMATCH", -3: "E_LEVEL_OUT_OF_RANGE",
    -4: "E_MALFORMED_BUFFER", -5: "E_CAPACITY", -6: "E_OOM", -7: "E_CUDA", -8: "E_UNSUPPORTED", -9: "E_IO",
}

EXPORTED_SYMBOLS = (
    "bitstack_create", "bitstack_destroy", "bitstack_load_blocks", "bitstack_load_blocks_async",
    "bitstack_set_num_blocks",
    "bitstack_matmul", "bitstack_matmul_grouped", "bitstack_reconstruct", "bitstack_get_info", "bitstack_set_kernel",
    "bitstack_block_size_bits", "bitstack_last_error", "bitstack_compress", "bitstack_profile_begin",
    "bitstack_profile_end", "bitstack_launch_count",
    "bitstack_store_create", "bitstack_store_append", "bitstack_store_open", "bitstack_store_count",
    "bitstack_store_record_info", "bitstack_store_read", "bitstack_store_load_range", "bitstack_store_close",
)


class BitStackError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"{STATUS.get(status, status)}: {message}")
        self.status = status
        self.name = STATUS.get(status, str(status))


class Info(ctypes.Structure):
    _fields_ = [
        ("d_out", ctypes.c_int64), ("d_in", ctypes.c_int64),
        ("row_begin", ctypes.c_int64), ("row_end", ctypes.c_int64),
        ("k", ctypes.c_int32), ("n_capacity", ctypes.c_int32),
        ("n_resident", ctypes.c_int32), ("n_active", ctypes.c_int32),
        ("factor_dtype", ctypes.c_int32), ("device", ctypes.c_int32),
        ("device_bytes", ctypes.c_int64), ("block_bytes_device", ctypes.c_int64),
    ]


class StoreRecord(ctypes.Structure):
    _fields_ = [
        ("stack", ctypes.c_int32), ("block", ctypes.c_int32),
        ("d_out", ctypes.c_int64), ("d_in", ctypes.c_int64),
        ("k", ctypes.c_int32), ("factor_dtype", ctypes.c_int32),
        ("size_bits", ctypes.c_int64),
        ("sign_bytes", ctypes.c_int64), ("u_bytes", ctypes.c_int64), ("v_bytes", ctypes.c_int64),
        ("s_bytes", ctypes.c_int64), ("offset", ctypes.c_int64), ("crc32", ctypes.c_uint32),
    ]


_lib: Optional[ctypes.CDLL] = None


def load_library(path: Optional[str] = None) -> ctypes.CDLL:
    """Load libbitstack.so (build it first with paper_2410_23918_b200.build); the
    BITSTACK_LIB environment variable, read at first load, selects another build."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("BITSTACK_LIB", LIB_PATH)
    if not os.path.exists(path):
        raise FileNotFoundError(
            f"{path} not found: run `python -m paper_2410_23918_b200.build` (the CUDA "
            "library is required; there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    P, I32, I64, VP = ctypes.POINTER, ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p
    sig = {
        "bitstack_create": (I32, [I64, I64, I32, I32, I32, I64, I64, I32, P(VP)]),
        "bitstack_destroy": (I32, [VP]),
        "bitstack_load_blocks": (I32, [VP, I32, I32, VP, VP, VP, VP, VP]),
        "bitstack_load_blocks_async": (I32, [VP, I32, I32, VP, VP, VP, VP, VP]),
        "bitstack_set_num_blocks": (I32, [VP, I32]),
        "bitstack_matmul": (I32, [VP, VP, I32, VP, I32, I64, VP]),
        "bitstack_matmul_grouped": (I32, [P(VP), I32, P(VP), I32, P(VP), I32, I64, VP]),
        "bitstack_reconstruct": (I32, [VP, VP, I32, VP]),
        "bitstack_get_info": (I32, [VP, P(Info)]),
        "bitstack_set_kernel": (I32, [VP, I32]),
        "bitstack_block_size_bits": (I64, [I64, I64, I32, I32]),
        "bitstack_last_error": (ctypes.c_char_p, []),
        "bitstack_compress": (I32, [VP, VP, I64, I64, I64, I32, I32, I32, I32, I32, ctypes.c_uint64, VP, VP, VP, VP,
                                    VP, VP, VP]),
        "bitstack_profile_begin": (I32, [I32]),
        "bitstack_profile_end": (I32, [P(I32), P(ctypes.c_double)]),
        "bitstack_launch_count": (I64, []),
        "bitstack_store_create": (I32, [ctypes.c_char_p, P(VP)]),
        "bitstack_store_append": (I32, [VP, I32, I32, I64, I64, I32, I32, VP, VP, VP, VP]),
        "bitstack_store_open": (I32, [ctypes.c_char_p, P(VP)]),
        "bitstack_store_count": (I32, [VP, P(I64)]),
        "bitstack_store_record_info": (I32, [VP, I64, P(StoreRecord)]),
        "bitstack_store_read": (I32, [VP, I64, VP, VP, VP, VP]),
        "bitstack_store_load_range": (I32, [VP, VP, I64, I64, VP]),
        "bitstack_store_close": (I32, [VP]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def _check(status: int) -> None:
    if status != 0:
        msg = _lib.bitstack_last_error().decode(errors="replace")
        raise BitStackError(status, msg)


def dtype_code(dt) -> int:
    if isinstance(dt, int):
        return dt
    name = str(dt).replace("torch.", "").replace("numpy.", "")
    if name in _DTYPE_NAMES:
        return _DTYPE_NAMES[name]
    raise ValueError(f"unsupported dtype {dt}")


def _ptr(a) -> int:
    """Address of a contiguous numpy array or torch tensor (host or device)."""
    if a is None:
        return 0
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return a.ctypes.data
    if hasattr(a, "data_ptr"):
        if not a.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return a.data_ptr()
    raise TypeError(type(a))


def _stream_handle(stream) -> int:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def block_size_bits(m: int, n: int, k: int = 16, factor_bits: int = 16) -> int:
    """Eq.9, computed by the library."""
    return int(load_library().bitstack_block_size_bits(m, n, k, factor_bits))


def launch_count() -> int:
    return int(load_library().bitstack_launch_count())


def profile_begin(max_launches: int = 65536) -> None:
    load_library()
    _check(_lib.bitstack_profile_begin(max_launches))


def profile_end():
    """-> (launches, total_ms) of the decode launches bracketed since profile_begin."""
    n = ctypes.c_int32(0)
    ms = ctypes.c_double(0.0)
    _check(_lib.bitstack_profile_end(ctypes.byref(n), ctypes.byref(ms)))
    return int(n.value), float(ms.value)


class Layer:
    """One weight stack (bitstack_layer handle) -- the four calls of the north star:
    load_blocks / set_num_blocks / matmul / reconstruct."""

    def __init__(self, d_out: int, d_in: int, k: int = 16, n_capacity: int = 16,
                 factor_dtype="bf16", row_begin: int = 0, row_end: Optional[int] = None,
                 device: int = 0):
        lib = load_library()
        self.d_out, self.d_in, self.k = int(d_out), int(d_in), int(k)
        self.row_begin = int(row_begin)
        self.row_end = int(d_out if row_end is None else row_end)
        self.factor_dtype = dtype_code(factor_dtype)
        self.device = int(device)
        h = ctypes.c_void_p()
        _check(lib.bitstack_create(self.d_out, self.d_in, self.k, int(n_capacity), self.factor_dtype,
                                   self.row_begin, self.row_end, self.device, ctypes.byref(h)))
        self._h = h

    @property
    def rows(self) -> int:
        return self.row_end - self.row_begin

    def close(self) -> None:
        if getattr(self, "_h", None) and self._h.value:
            _lib.bitstack_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def load_blocks(self, first_block: int, signs, u, v, s=None, stream=None) -> None:
        """signs: [count, ceil(d_out*d_in/8)] uint8; u: [count, d_out, k], v: [count, d_in, k]
        in the storage dtype (bf16 as torch.bfloat16 or numpy uint16 bit patterns);
        s: [d_in] float32 (first_block == 0 only).  Host or device buffers."""
        count = int(signs.shape[0]) if signs is not None else 0
        _check(_lib.bitstack_load_blocks(self._h, int(first_block), count, _ptr(signs), _ptr(u),
                                         _ptr(v), _ptr(s), _stream_handle(stream)))

    def load_blocks_async(self, first_block: int, signs, u, v, s=None, stream=None) -> None:
        """bitstack_load_blocks_async: enqueue the load on `stream` and return; keep the (pinned
        host or device) buffers alive and unchanged until the stream has passed this call."""
        count = int(signs.shape[0]) if signs is not None else 0
        _check(_lib.bitstack_load_blocks_async(self._h, int(first_block), count, _ptr(signs), _ptr(u),
                                               _ptr(v), _ptr(s), _stream_handle(stream)))

    def set_num_blocks(self, n: int) -> None:
        _check(_lib.bitstack_set_num_blocks(self._h, int(n)))

    def set_kernel(self, kernel) -> None:
        code = {"auto": KERNEL_AUTO, "tc": KERNEL_TC, "simt": KERNEL_SIMT,
                "prefill": KERNEL_PREFILL, "rgemv": KERNEL_RGEMV}.get(kernel, kernel)
        _check(_lib.bitstack_set_kernel(self._h, int(code)))

    def info(self) -> dict:
        inf = Info()
        _check(_lib.bitstack_get_info(self._h, ctypes.byref(inf)))
        return {f: getattr(inf, f) for f, _ in Info._fields_}

    def matmul(self, x, y=None, y_dtype=None, stream=None):
        """y = W_hat_n x for x: device [batch, d_in] (float32 | bfloat16 | float16 torch tensor)."""
        import torch
        if x.dim() == 1:
            x = x.unsqueeze(0)
        if y is None:
            y = torch.empty((x.shape[0], self.rows), dtype=y_dtype or torch.float32, device=x.device)
        _check(_lib.bitstack_matmul(self._h, _ptr(x), dtype_code(x.dtype), _ptr(y), dtype_code(y.dtype),
                                    int(x.shape[0]), _stream_handle(stream)))
        return y

    def matmul_raw(self, x_ptr: int, x_dtype: int, y_ptr: int, y_dtype: int, batch: int, stream: int) -> None:
        """Pointer-level call (bench / CUDA-graph capture)."""
        _check(_lib.bitstack_matmul(self._h, x_ptr, x_dtype, y_ptr, y_dtype, batch, stream))

    def reconstruct(self, dtype=None, stream=None):
        import torch
        w = torch.empty((self.rows, self.d_in), dtype=dtype or torch.float32,
                        device=f"cuda:{self.device}")
        _check(_lib.bitstack_reconstruct(self._h, _ptr(w), dtype_code(w.dtype), _stream_handle(stream)))
        return w


class Group:
    """Pointer arrays of a fixed bitstack_matmul_grouped call (bench / CUDA-graph capture):
    members `layers`, inputs `x_ptrs`, outputs `y_ptrs`, built once, called many times."""

    def __init__(self, layers, x_ptrs, y_ptrs):
        n = len(layers)
        if not (n == len(x_ptrs) == len(y_ptrs)):
            raise ValueError("layers, x_ptrs and y_ptrs differ in length")
        self.count = n
        self._layers = list(layers)   # keep the handles alive
        self._h = (ctypes.c_void_p * n)(*[l._h.value for l in layers])
        self._x = (ctypes.c_void_p * n)(*[int(p) for p in x_ptrs])
        self._y = (ctypes.c_void_p * n)(*[int(p) for p in y_ptrs])

    def __call__(self, x_dtype: int, y_dtype: int, batch: int, stream: int) -> None:
        _check(_lib.bitstack_matmul_grouped(self._h, self.count, self._x, int(x_dtype), self._y, int(y_dtype),
                                            int(batch), int(stream)))


def matmul_grouped(layers, xs, y_dtype=None, stream=None):
    """ys[i] = W_hat(layers[i]) xs[i] in one grouped call (include/bitstack.h
    bitstack_matmul_grouped); xs: device tensors [batch, d_in_i] of one dtype and batch."""
    import torch
    xs = [x.unsqueeze(0) if x.dim() == 1 else x for x in xs]
    if len(xs) != len(layers):
        raise ValueError("one input per layer")
    batch = int(xs[0].shape[0]) if xs else 0
    ys = [torch.empty((x.shape[0], l.rows), dtype=y_dtype or torch.float32, device=x.device)
          for l, x in zip(layers, xs)]
    if not layers:
        return ys
    xdt = dtype_code(xs[0].dtype)
    for x in xs:
        if int(x.shape[0]) != batch or dtype_code(x.dtype) != xdt:
            raise ValueError("grouped inputs must share batch size and dtype")
    Group(layers, [_ptr(x) for x in xs], [_ptr(y) for y in ys])(xdt, dtype_code(ys[0].dtype), batch,
                                                                    _stream_handle(stream))
    return ys


def compress(w, x_cal, n: int, k: int = 16, factor_dtype="bf16", oversample: int = 16, power_iters: int = 4,
             seed: int = 0, stream=None):
    """bitstack_compress (include/bitstack.h): Alg.1 for one matrix on the device.
    w [d_out, d_in], x_cal [p, d_in]: device float32 tensors.  Returns device tensors
    (signs [n, nbytes] uint8, u [n, d_out, k], v [n, d_in, k] in factor_dtype, s [d_in] f32,
    sigma [n, k] f32, resid [n + 1] f32) -- the first four are bitstack_load_blocks' inputs."""
    import torch
    lib = load_library()
    d_out, d_in = int(w.shape[0]), int(w.shape[1])
    p = int(x_cal.shape[0])
    fdt = dtype_code(factor_dtype)
    tdt = {F32: torch.float32, BF16: torch.bfloat16, F16: torch.float16}[fdt]
    dev = w.device
    signs = torch.empty((n, (d_out * d_in + 7) // 8), dtype=torch.uint8, device=dev)
    u = torch.empty((n, d_out, k), dtype=tdt, device=dev)
    v = torch.empty((n, d_in, k), dtype=tdt, device=dev)
    s = torch.empty(d_in, dtype=torch.float32, device=dev)
    sigma = torch.empty((n, k), dtype=torch.float32, device=dev)
    resid = torch.empty(n + 1, dtype=torch.float32, device=dev)
    _check(lib.bitstack_compress(_ptr(w), _ptr(x_cal), p, d_out, d_in, int(n), int(k), fdt, int(oversample),
                                 int(power_iters), int(seed), _ptr(signs), _ptr(u), _ptr(v), _ptr(s), _ptr(sigma),
                                 _ptr(resid), _stream_handle(stream)))
    return signs, u, v, s, sigma, resid


# ---------------------------------------------------------------- block store (on disk)
_NP_FACTOR = {F32: np.float32, BF16: np.uint16, F16: np.float16}


class Store:
    """bitstack_store_* (include/bitstack.h): residual blocks on disk in universal-stack order,
    readable by record range.  Store.create(path) writes, Store.open(path) reads."""

    def __init__(self, handle, writer: bool):
        self._h = handle
        self.writer = writer

    @classmethod
    def create(cls, path: str) -> "Store":
        lib = load_library()
        h = ctypes.c_void_p()
        _check(lib.bitstack_store_create(os.fsencode(path), ctypes.byref(h)))
        return cls(h, True)

    @classmethod
    def open(cls, path: str) -> "Store":
        lib = load_library()
        h = ctypes.c_void_p()
        _check(lib.bitstack_store_open(os.fsencode(path), ctypes.byref(h)))
        return cls(h, False)

    def append(self, stack: int, block: int, signs, u, v, s=None, factor_dtype="bf16") -> None:
        """One block in the canonical host layouts of Layer.load_blocks (u / v: [d_out, k] /
        [d_in, k] in the factor dtype; bf16 as uint16 bit patterns); s with block 0 only."""
        fdt = dtype_code(factor_dtype)
        signs = np.ascontiguousarray(signs, dtype=np.uint8)
        u = np.ascontiguousarray(u)
        v = np.ascontiguousarray(v)
        s_arr = None if s is None else np.ascontiguousarray(s, dtype=np.float32)
        d_out, k = u.shape
        d_in = v.shape[0]
        _check(_lib.bitstack_store_append(self._h, stack, block, d_out, d_in, k, fdt, _ptr(signs), _ptr(u), _ptr(v),
                                          _ptr(s_arr)))

    def __len__(self) -> int:
        n = ctypes.c_int64()
        _check(_lib.bitstack_store_count(self._h, ctypes.byref(n)))
        return int(n.value)

    def info(self, record: int) -> dict:
        r = StoreRecord()
        _check(_lib.bitstack_store_record_info(self._h, record, ctypes.byref(r)))
        return {name: getattr(r, name) for name, _ in StoreRecord._fields_}

    def read(self, record: int):
        """(stack, block, signs, u, v, s or None) of one record, host numpy arrays."""
        r = self.info(record)
        signs = np.empty(r["sign_bytes"], np.uint8)
        ft = _NP_FACTOR[r["factor_dtype"]]
        u = np.empty((r["d_out"], r["k"]), ft)
        v = np.empty((r["d_in"], r["k"]), ft)
        s = np.empty(r["d_in"], np.float32) if r["s_bytes"] else None
        _check(_lib.bitstack_store_read(self._h, record, _ptr(signs), _ptr(u), _ptr(v), _ptr(s)))
        return r["stack"], r["block"], signs, u, v, s

    def read_range(self, first: int, count: int):
        return [self.read(first + j) for j in range(count)]

    def load_range(self, layer, first: int, count: int, stream=None) -> None:
        """Stream records [first, first + count) of one stack into `layer` (async on `stream`)."""
        _check(_lib.bitstack_store_load_range(self._h, layer._h, first, count, _stream_handle(stream)))

    def close(self) -> None:
        if self._h is not None:
            _check(_lib.bitstack_store_close(self._h))
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            if getattr(self, "_h", None) is not None and _lib is not None:
                _lib.bitstack_store_close(self._h)
                self._h = None
        except Exception:  # noqa: BLE001
            pass
