"""Python binding of libgear.so -- the B200-native GEAR replay hot path.

Argument marshalling only: every function below has the name of the C-ABI
entry point in ``include/gear.h`` it calls (``gear_table_create``,
``gear_insert``, ``gear_update_priorities``, ``gear_sample``,
``gear_collect``, ...), converts torch tensors / numpy arrays to pointers and
raises ``GearError`` on a non-zero status.  All compute runs in the CUDA
kernels of ``csrc/``; there is no CPU fallback -- importing this package on a
machine without the built library raises.

PyTorch is used for device memory, streams and process groups (the NCCL
unique id is broadcast with ``torch.distributed``).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GEAR_LIB", os.path.join(_HERE, "libgear.so"))  # override: dev A/B builds

# status codes (gear.h)
GEAR_OK = 0
GEAR_ERR_INVALID_ARG = -1
GEAR_ERR_OUT_OF_MEMORY = -2
GEAR_ERR_CUDA = -3
GEAR_ERR_NCCL = -4
GEAR_ERR_EMPTY = -5
GEAR_ERR_INDEX_RANGE = -6
GEAR_ERR_BAD_PRIORITY = -7
GEAR_ERR_STATE = -8
GEAR_ERR_UNSUPPORTED = -9
GEAR_DEVERR_INDEX_RANGE = 1
GEAR_DEVERR_BAD_PRIORITY = 2
GEAR_DEVERR_STALE = 4
GEAR_DEVERR_EMPTY = 8
GEAR_DEVERR_TIMEOUT = 16
GEAR_DEVERR_FULL = 32
GEAR_IDX_NONE = 0xFFFFFFFFFFFFFFFF

# dtypes / placements / strategies / removal (gear.h enums)
GEAR_U8, GEAR_I32, GEAR_I64, GEAR_F32, GEAR_F64, GEAR_BF16 = range(6)
GEAR_DEVICE, GEAR_HOST = 0, 1
GEAR_FIFO, GEAR_LIFO, GEAR_UNIFORM, GEAR_WEIGHTED, GEAR_PRIORITIZED, GEAR_TOPK = range(6)
GEAR_REMOVE_FIFO, GEAR_REMOVE_LIFO = 0, 1
GEAR_SAMPLE_OWNER_AFFINE = 0x100
GEAR_SAMPLE_DEVICE_SEED = 0x200

STRATEGIES = {"fifo": GEAR_FIFO, "lifo": GEAR_LIFO, "uniform": GEAR_UNIFORM,
              "weighted": GEAR_WEIGHTED, "prioritized": GEAR_PRIORITIZED, "topk": GEAR_TOPK}
DTYPES = {"u8": GEAR_U8, "i32": GEAR_I32, "i64": GEAR_I64, "f32": GEAR_F32, "f64": GEAR_F64,
          "bf16": GEAR_BF16}
DTYPE_BYTES = {GEAR_U8: 1, GEAR_I32: 4, GEAR_I64: 8, GEAR_F32: 4, GEAR_F64: 8, GEAR_BF16: 2}


class GearError(RuntimeError):
    def __init__(self, fn: str, status: int, msg: str):
        super().__init__(f"{fn} -> {status}: {msg}")
        self.status = status


class _ColumnDesc(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char_p), ("dtype", ctypes.c_int), ("ndim", ctypes.c_uint32),
                ("shape", ctypes.POINTER(ctypes.c_int64)), ("placement", ctypes.c_int)]


class _TableDesc(ctypes.Structure):
    _fields_ = [("capacity_global", ctypes.c_uint64), ("seq_len", ctypes.c_uint32),
                ("ncols", ctypes.c_uint32), ("cols", ctypes.POINTER(_ColumnDesc)),
                ("priority_frac_bits", ctypes.c_uint32), ("removal", ctypes.c_int),
                ("shards_per_rank", ctypes.c_uint32), ("max_batch", ctypes.c_uint32),
                ("priority_alpha", ctypes.c_double)]


class _TableInfo(ctypes.Structure):
    _fields_ = [("capacity_global", ctypes.c_uint64), ("shard_capacity", ctypes.c_uint64),
                ("n_ranks", ctypes.c_uint32), ("rank", ctypes.c_uint32),
                ("shards_per_rank", ctypes.c_uint32), ("ncols", ctypes.c_uint32),
                ("row_bytes_total", ctypes.c_uint64), ("q_max", ctypes.c_uint64),
                ("p_max", ctypes.c_double), ("frac_bits", ctypes.c_uint32),
                ("max_batch", ctypes.c_uint32), ("alpha", ctypes.c_double)]


# exported symbols and their signatures (also checked by the CPU tests)
_P = ctypes.c_void_p
_u32, _u64, _i32, _f64 = ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int, ctypes.c_double
SIGNATURES = {
    "gear_last_error": ([], ctypes.c_char_p),
    "gear_version": ([], ctypes.c_char_p),
    "gear_kernel_launches": ([], ctypes.c_uint64),
    "gear_get_unique_id": ([_P], _i32),
    "gear_comm_create": ([_i32, _i32, _P, _i32, _P], _i32),
    "gear_comm_create_host": ([_i32, _i32, _i32, _P, _P, _P], _i32),
    "gear_comm_destroy": ([_P], _i32),
    "gear_table_create": ([_P, _P, _P], _i32),
    "gear_table_destroy": ([_P], _i32),
    "gear_table_info_get": ([_P, _P], _i32),
    "gear_column_id": ([_P, ctypes.c_char_p, _P], _i32),
    "gear_column_row_bytes": ([_P, _u32, _P], _i32),
    "gear_insert": ([_P, _u32, _u32, _P, _P, _P, _P], _i32),
    "gear_allocate": ([_P, _u32, _u32, _P, _P], _i32),
    "gear_commit": ([_P, _u32, _u32, _P, _P, _P], _i32),
    "gear_column_base": ([_P, _u32, _P], _i32),
    "gear_update_priorities": ([_P, _u32, _P, _P, _i32, _P, _P], _i32),
    "gear_sample": ([_P, _i32, _u32, _u64, _f64, _P, _P, _P, _P, _u32, _P], _i32),
    "gear_collect": ([_P, _u32, _P, _u32, _P, _P, _P], _i32),
    "gear_table_sync": ([_P, _P, _P], _i32),
    "gear_read_state": ([_P, _P, _P, _P], _i32),
    "gear_read_cdf": ([_P, _P], _i32),
    "gear_table_set_tuning": ([_P, ctypes.c_char_p, ctypes.c_int64], _i32),
    "gear_table_save": ([_P, ctypes.c_char_p], _i32),
    "gear_table_load": ([_P, ctypes.c_char_p], _i32),
}

_lib = None


def load() -> ctypes.CDLL:
    """Load libgear.so (build it with ``python -m paper_2310_05205_b200.build``)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() -- "
                              "there is no CPU fallback")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (args, res) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _lib = lib
    return _lib


def _check(fn: str, st: int):
    if st != GEAR_OK:
        raise GearError(fn, st, load().gear_last_error().decode())


def _ptr(x) -> int | None:
    """Device/host address of a torch tensor, numpy array, int or None."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if isinstance(x, np.ndarray):
        assert x.flags["C_CONTIGUOUS"], "numpy arrays must be contiguous"
        return x.ctypes.data
    if hasattr(x, "data_ptr"):
        assert x.is_contiguous(), "tensors must be contiguous"
        return x.data_ptr()
    raise TypeError(f"cannot take the address of {type(x)}")


_I64 = ("int64", "uint64")
_I32 = ("int32", "uint32")


_DTYPE_NAMES: dict = {}


def _dtype_name(x) -> str:
    d = x.dtype
    s = _DTYPE_NAMES.get(d)
    if s is None:
        s = _DTYPE_NAMES[d] = str(d).replace("torch.", "")
    return s


def _arg(x, kinds, name: str, n: int = 0, fn: str = "") -> int | None:
    """_ptr(x) after checking that a tensor / array argument has one of the
    dtypes `kinds` and at least n elements (a wrong dtype would make the
    kernels read or write past the buffer).  Raw integer addresses are the
    caller's responsibility.  (Per-call cost matters for small batches: the
    dtype names are cached.)"""
    if x is None or isinstance(x, int):
        return x
    dt = _dtype_name(x)
    if dt not in kinds:
        raise TypeError(f"{fn}: {name} must have dtype {' or '.join(kinds)}, got {dt}")
    if isinstance(x, np.ndarray):
        if x.size < n:
            raise ValueError(f"{fn}: {name} has {x.size} elements, the call needs {n}")
        assert x.flags["C_CONTIGUOUS"], "numpy arrays must be contiguous"
        return x.ctypes.data
    numel = x.numel()
    if numel < n:
        raise ValueError(f"{fn}: {name} has {numel} elements, the call needs {n}")
    assert x.is_contiguous(), "tensors must be contiguous"
    return x.data_ptr()


def _nbytes(x) -> int | None:
    if isinstance(x, int) or x is None:
        return None
    if hasattr(x, "element_size"):
        return x.numel() * x.element_size()
    return x.nbytes


def _stream(stream) -> int | None:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def gear_kernel_launches() -> int:
    return int(load().gear_kernel_launches())


# ---------------------------------------------------------------- comm
def gear_get_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    _check("gear_get_unique_id", load().gear_get_unique_id(buf))
    return bytes(buf)


def gear_comm_create(nranks: int, rank: int, uid: bytes, device: int) -> int:
    out = ctypes.c_void_p()
    buf = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
    _check("gear_comm_create", load().gear_comm_create(nranks, rank, buf, device, ctypes.byref(out)))
    return out.value


# gear_allgather_fn: int (*)(void* ctx, const void* send, void* recv, size_t bytes)
ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                ctypes.c_size_t)
_host_comms: dict[int, object] = {}   # comm handle -> callback (kept alive until destroy)


def gear_comm_create_host(nranks: int, rank: int, device: int, allgather) -> int:
    """gear_comm_create_host with a Python all-gather ``allgather(bytes) ->
    list[bytes]`` (one entry per rank, rank order) as the host callback."""
    def cb(_ctx, send, recv, nbytes):
        try:
            parts = allgather(ctypes.string_at(send, nbytes))
            assert len(parts) == nranks and all(len(p) == nbytes for p in parts)
            ctypes.memmove(recv, b"".join(parts), nbytes * nranks)
            return 0
        except Exception as e:  # noqa: BLE001 -- reported as a status by the library
            print(f"gear host all-gather failed: {e!r}", flush=True)
            return 1
    fn = ALLGATHER_FN(cb)
    out = ctypes.c_void_p()
    _check("gear_comm_create_host",
           load().gear_comm_create_host(nranks, rank, device, ctypes.cast(fn, ctypes.c_void_p),
                                        None, ctypes.byref(out)))
    _host_comms[out.value] = fn
    return out.value


def gear_comm_destroy(comm: int):
    _check("gear_comm_destroy", load().gear_comm_destroy(comm))
    _host_comms.pop(comm, None)


def comm_from_process_group(device: int, group=None) -> int | None:
    """Create a gear comm bootstrapped through a torch.distributed group (any
    backend -- gloo works -- with no NCCL communicator of its own), so several
    ranks may share one CUDA device.  Returns None when the group has one
    rank."""
    import torch
    import torch.distributed as dist
    W = dist.get_world_size(group)
    if W == 1:
        return None

    def allgather(b: bytes) -> list[bytes]:
        t = torch.frombuffer(bytearray(b), dtype=torch.uint8)
        out = [torch.empty_like(t) for _ in range(W)]
        dist.all_gather(out, t, group=group)
        return [o.numpy().tobytes() for o in out]
    return gear_comm_create_host(W, dist.get_rank(group), device, allgather)


def comm_from_torch_distributed(device: int) -> int | None:
    """Create a gear comm over the ranks of the default torch.distributed
    group (rank 0's NCCL unique id is broadcast through it).  Returns None
    when the world has one rank."""
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return None
    obj = [gear_get_unique_id() if dist.get_rank() == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return gear_comm_create(dist.get_world_size(), dist.get_rank(), obj[0], device)


# ---------------------------------------------------------------- table
@dataclass
class Column:
    name: str
    dtype: int          # GEAR_U8 ...
    shape: tuple        # per-step shape
    placement: int = GEAR_DEVICE

    def row_bytes(self, seq_len: int) -> int:
        n = seq_len
        for s in self.shape:
            n *= s
        return n * DTYPE_BYTES[self.dtype]


def gear_table_create(capacity: int, seq_len: int, columns: Sequence[Column], comm: int | None = None,
                      frac_bits: int = 32, removal: int = GEAR_REMOVE_FIFO,
                      shards_per_rank: int = 1, max_batch: int = 4096,
                      alpha: float = 1.0) -> int:
    cols = (_ColumnDesc * len(columns))()
    keep = []
    for c, col in zip(cols, columns):
        shape = (ctypes.c_int64 * max(1, len(col.shape)))(*col.shape)
        name = col.name.encode()
        keep += [shape, name]
        c.name, c.dtype, c.ndim = name, col.dtype, len(col.shape)
        c.shape = ctypes.cast(shape, ctypes.POINTER(ctypes.c_int64))
        c.placement = col.placement
    d = _TableDesc(capacity, seq_len, len(columns), cols, frac_bits, removal, shards_per_rank,
                   max_batch, alpha)
    out = ctypes.c_void_p()
    _check("gear_table_create", load().gear_table_create(ctypes.byref(d), comm, ctypes.byref(out)))
    return out.value


def gear_table_destroy(t: int):
    _check("gear_table_destroy", load().gear_table_destroy(t))


def gear_table_info_get(t: int) -> dict:
    info = _TableInfo()
    _check("gear_table_info_get", load().gear_table_info_get(t, ctypes.byref(info)))
    return {f: getattr(info, f) for f, _ in _TableInfo._fields_}


def gear_column_id(t: int, name: str) -> int:
    out = ctypes.c_uint32()
    _check("gear_column_id", load().gear_column_id(t, name.encode(), ctypes.byref(out)))
    return out.value


def gear_column_row_bytes(t: int, col: int) -> int:
    out = ctypes.c_uint64()
    _check("gear_column_row_bytes", load().gear_column_row_bytes(t, col, ctypes.byref(out)))
    return out.value


def gear_insert(t: int, shard: int, n: int, col_src: Sequence, prio, out_idx=None, stream=None):
    for c, src in enumerate(col_src):
        nb = _nbytes(src)
        if nb is not None and nb < n * gear_column_row_bytes(t, c):
            raise ValueError(f"gear_insert: col_src[{c}] has {nb} bytes, {n} rows need "
                             f"{n * gear_column_row_bytes(t, c)}")
    srcs = (ctypes.c_void_p * len(col_src))(*[_ptr(s) for s in col_src])
    prio = np.ascontiguousarray(prio, dtype=np.float64) if not hasattr(prio, "data_ptr") else prio
    _check("gear_insert", load().gear_insert(t, shard, n, srcs, _arg(prio, ("float64",), "prio", n, "gear_insert"),
                                             _arg(out_idx, _I64, "out_idx", n, "gear_insert"),
                                             _stream(stream)))


def gear_allocate(t: int, shard: int, n: int, out_idx, stream=None):
    _check("gear_allocate", load().gear_allocate(t, shard, n, _arg(out_idx, _I64, "out_idx", n, "gear_allocate"),
                                                 _stream(stream)))


def gear_commit(t: int, shard: int, n: int, idx, prio, stream=None):
    prio = np.ascontiguousarray(prio, dtype=np.float64) if not hasattr(prio, "data_ptr") else prio
    _check("gear_commit", load().gear_commit(t, shard, n, _arg(idx, _I64, "idx", n, "gear_commit"),
                                             _arg(prio, ("float64",), "prio", n, "gear_commit"),
                                             _stream(stream)))


def gear_column_base(t: int, col: int) -> int:
    out = ctypes.c_void_p()
    _check("gear_column_base", load().gear_column_base(t, col, ctypes.byref(out)))
    return out.value or 0


def gear_update_priorities(t: int, n: int, idx, prio, prio_dtype: int, gen=None, stream=None):
    f = "gear_update_priorities"
    pk = {GEAR_F64: ("float64",), GEAR_F32: ("float32",)}.get(prio_dtype)
    pp = _arg(prio, pk, "prio", n, f) if pk else _ptr(prio)   # other dtypes: the C-ABI rejects them
    _check(f, load().gear_update_priorities(t, n, _arg(idx, _I64, "idx", n, f), pp,
                                            prio_dtype, _arg(gen, _I32, "gen", n, f), _stream(stream)))


def gear_sample(t: int, strategy: int, B: int, seed: int, beta: float, out_idx, out_w=None,
                out_p=None, out_gen=None, stream=None, flags: int = 0):
    """strategy: GEAR_FIFO ... GEAR_TOPK; flags: GEAR_SAMPLE_* bits (for
    compatibility, flag bits OR-ed into `strategy` are moved to `flags`)."""
    f = "gear_sample"
    flags |= strategy & ~0xFF
    strategy &= 0xFF
    _check(f, load().gear_sample(t, strategy, B, seed, beta, _arg(out_idx, _I64, "out_idx", B, f),
                                 _arg(out_w, ("float32",), "out_w", B, f),
                                 _arg(out_p, ("float64",), "out_p", B, f),
                                 _arg(out_gen, _I32, "out_gen", B, f), flags, _stream(stream)))


def gear_collect(t: int, n: int, idx, col_ids: Sequence[int], out: Sequence, stream=None):
    f = "gear_collect"
    if len(col_ids) != len(out):
        raise ValueError(f"{f}: {len(col_ids)} column ids but {len(out)} outputs")
    for c, o in zip(col_ids, out):
        nb = _nbytes(o)
        if nb is not None and nb < n * gear_column_row_bytes(t, c):
            raise ValueError(f"{f}: output of column {c} has {nb} bytes, {n} rows need "
                             f"{n * gear_column_row_bytes(t, c)}")
    ids = (ctypes.c_uint32 * len(col_ids))(*col_ids)
    outs = (ctypes.c_void_p * len(out))(*[_ptr(o) for o in out])
    _check(f, load().gear_collect(t, n, _arg(idx, _I64, "idx", n, f), len(col_ids), ids, outs,
                                  _stream(stream)))


def gear_table_sync(t: int) -> tuple[int, int]:
    """Returns (device error bits, stale update count); never raises for
    latched device errors (they are the return value)."""
    e = ctypes.c_uint32()
    ns = ctypes.c_uint64()
    st = load().gear_table_sync(t, ctypes.byref(e), ctypes.byref(ns))
    if st not in (GEAR_OK, GEAR_ERR_STATE):
        _check("gear_table_sync", st)
    return e.value, ns.value


def gear_read_state(t: int):
    info = gear_table_info_get(t)
    n = info["shard_capacity"] * info["shards_per_rank"]
    key = np.zeros(n, np.uint64)
    seq = np.zeros(n, np.uint64)
    gen = np.zeros(n, np.uint32)
    _check("gear_read_state", load().gear_read_state(t, _ptr(key), _ptr(seq), _ptr(gen)))
    return key, seq, gen


def gear_read_cdf(t: int):
    """The last built CDF as flat per-shard inclusive prefix sums (u64[R*C_s])."""
    info = gear_table_info_get(t)
    out = np.zeros(info["shard_capacity"] * info["shards_per_rank"], np.uint64)
    _check("gear_read_cdf", load().gear_read_cdf(t, _ptr(out)))
    return out


def gear_table_set_tuning(t: int, key: str, value: int):
    _check("gear_table_set_tuning", load().gear_table_set_tuning(t, key.encode(), value))


def gear_table_save(t: int, path: str):
    _check("gear_table_save", load().gear_table_save(t, str(path).encode()))


def gear_table_load(t: int, path: str):
    _check("gear_table_load", load().gear_table_load(t, str(path).encode()))


class Table:
    """Thin owner of a gear_table handle (destroys it on close)."""

    def __init__(self, capacity: int, seq_len: int, columns: Sequence[Column], comm=None, **kw):
        self.columns = list(columns)
        self.seq_len = seq_len
        self.handle = gear_table_create(capacity, seq_len, self.columns, comm, **kw)
        self.info = gear_table_info_get(self.handle)
        self.row_bytes = [gear_column_row_bytes(self.handle, i) for i in range(len(self.columns))]

    def close(self):
        if self.handle:
            gear_table_destroy(self.handle)
            self.handle = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def insert(self, shard, col_src, prio, out_idx=None, stream=None):
        gear_insert(self.handle, shard, len(prio), col_src, prio, out_idx, stream)

    def allocate(self, shard, n, out_idx, stream=None):
        gear_allocate(self.handle, shard, n, out_idx, stream)

    def commit(self, shard, idx, prio, stream=None):
        gear_commit(self.handle, shard, len(idx), idx, prio, stream)

    def column_base(self, col):
        return gear_column_base(self.handle, col)

    def update_priorities(self, idx, prio, gen=None, stream=None):
        dt = {"float64": GEAR_F64, "float32": GEAR_F32}.get(_dtype_name(prio))
        if dt is None:
            raise TypeError(f"priorities must be float32 or float64, got {_dtype_name(prio)}")
        gear_update_priorities(self.handle, len(idx), idx, prio, dt, gen, stream)

    def sample(self, strategy, B, seed, beta, out_idx, out_w=None, out_p=None, out_gen=None, stream=None,
               flags=0):
        gear_sample(self.handle, strategy, B, seed, beta, out_idx, out_w, out_p, out_gen, stream, flags)

    def collect(self, idx, col_ids, out, stream=None):
        gear_collect(self.handle, len(idx), idx, col_ids, out, stream)

    def sync(self):
        return gear_table_sync(self.handle)

    def read_state(self):
        return gear_read_state(self.handle)

    def save(self, path):
        gear_table_save(self.handle, path)

    def load(self, path):
        gear_table_load(self.handle, path)
