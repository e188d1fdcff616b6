"""Seeded synthetic inputs shared by the oracle and the CUDA path.

Input generation only -- this module holds none of the replay method's
arithmetic (no quantisation, CDF, RNG draw, search, selection or gather).
Both sides receive the SAME generated arrays: priorities come from numpy's
PCG64 and are handed to the oracle and to the GPU as identical f64 arrays;
row bytes are a splitmix64 hash of (seed, column, trajectory id, word) that
numpy (here) and a CUDA fill kernel (fill.cu -> libsynth.so) both compute, so
a test can regenerate any sampled row of a 100 GB table on the CPU.

The workload shapes follow BASELINE.json's configs.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "libsynth.so")
DATA_SEED = 0x47454152  # "GEAR"
SAMPLE_SEED_BASE = 0x5EED0000
PRIO_SEED = 1

_M64 = (1 << 64) - 1


def _splitmix64(z: np.ndarray) -> np.ndarray:
    z = z + np.uint64(0x9E3779B97F4A7C15)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def row_bytes_of(col: int, traj_ids, row_bytes: int, seed: int = DATA_SEED) -> np.ndarray:
    """uint8 [len(traj_ids), row_bytes]: the synthetic content of those rows."""
    t = np.asarray(traj_ids, dtype=np.uint64).reshape(-1, 1)
    with np.errstate(over="ignore"):
        base = _splitmix64(np.uint64(seed) ^ (np.uint64(col) * np.uint64(0xD1B54A32D192ED03))
                           ^ (t * np.uint64(0x9E3779B97F4A7C15)))
        w = np.arange((row_bytes + 7) // 8, dtype=np.uint64).reshape(1, -1)
        words = _splitmix64(base + w * np.uint64(0x632BE59BD9B4E019))
    return words.astype("<u8").view(np.uint8).reshape(t.shape[0], -1)[:, :row_bytes].copy()


def priorities(n: int, seed: int = PRIO_SEED, zero_frac: float = 0.0, sigma: float = 1.0) -> np.ndarray:
    """lognormal(0, sigma) f64 priorities with a fraction of exact zeros."""
    rng = np.random.default_rng(seed)
    p = rng.lognormal(0.0, sigma, size=n)
    if zero_frac > 0:
        p[rng.random(n) < zero_frac] = 0.0
    return p


def task_weights(n: int, tasks: int = 16, zero_frac: float = 0.005, seed: int = PRIO_SEED) -> np.ndarray:
    """c3: weights 1..tasks on contiguous id ranges, a fraction of zeros."""
    p = (np.arange(n, dtype=np.int64) * tasks // max(n, 1) + 1).astype(np.float64)
    rng = np.random.default_rng(seed)
    p[rng.random(n) < zero_frac] = 0.0
    return p


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "fill.cu")
    if not force and os.path.exists(_LIB) and os.path.getmtime(_LIB) >= os.path.getmtime(src):
        return _LIB
    tmp = _LIB + f".tmp{os.getpid()}"
    subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-O3", "-shared", "-Xcompiler", "-fPIC",
                           "-gencode", "arch=compute_100a,code=sm_100a", "-o", tmp, src])
    os.replace(tmp, _LIB)
    return _LIB


_lib = None


def _load():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(_LIB)
        _lib.synth_fill_rows.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64,
                                         ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                         ctypes.c_void_p]
        _lib.synth_fill_rows.restype = ctypes.c_int
        _lib.synth_fill_rows_ids.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64,
                                             ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                             ctypes.c_void_p]
        _lib.synth_fill_rows_ids.restype = ctypes.c_int
    return _lib


def fill_rows_ids(dst_ptr: int, ids_ptr: int, n_rows: int, row_bytes: int, col: int,
                  seed: int = DATA_SEED, stream: int = 0):
    """Write the rows of trajectories ids[0..n_rows) (device u64 array) of
    column `col` to device memory -- the expected batch of a gather."""
    st = _load().synth_fill_rows_ids(dst_ptr, ids_ptr, n_rows, row_bytes, col, seed, stream)
    if st != 0:
        raise RuntimeError(f"synth_fill_rows_ids: cuda error {st}")


def fill_rows(dst_ptr: int, n_rows: int, row_bytes: int, col: int, first_traj: int,
              seed: int = DATA_SEED, stream: int = 0):
    """Write rows first_traj .. first_traj+n_rows-1 of column `col` to device memory."""
    st = _load().synth_fill_rows(dst_ptr, n_rows, row_bytes, col, first_traj, seed, stream)
    if st != 0:
        raise RuntimeError(f"synth_fill_rows: cuda error {st}")


# ------------------------------------------------------------------ configs
@dataclass
class ColSpec:
    name: str
    dtype: str          # u8 / i32 / f32
    shape: tuple        # per step
    placement: str = "device"


@dataclass
class Config:
    name: str
    capacity: int
    seq_len: int
    cols: list
    strategy: str
    batch: int
    beta: float = 0.4
    update: bool = False
    prio: str = "lognormal"
    zero_frac: float = 0.01
    note: str = ""
    extra: dict = field(default_factory=dict)


BYTES = {"u8": 1, "i32": 4, "f32": 4, "i64": 8, "f64": 8}


def row_bytes(cfg: Config, c: ColSpec) -> int:
    n = cfg.seq_len * BYTES[c.dtype]
    for s in c.shape:
        n *= s
    return n


CONFIGS = {
    # BASELINE.json configs[0]: tiny table, the oracle finishes in seconds.
    "c1": Config("c1_tiny", 1024, 32,
                 [ColSpec("obs", "f32", (16,)), ColSpec("action", "i32", ()),
                  ColSpec("reward", "f32", ())],
                 "prioritized", 64, zero_frac=0.10, update=True),
    # configs[1]: Decision-Transformer-shaped Atari table, HBM-resident.
    "c2": Config("c2_dt_atari", 100_000, 30,
                 [ColSpec("obs", "u8", (4, 84, 84)), ColSpec("action", "i32", ()),
                  ColSpec("rtg", "f32", ()), ColSpec("timestep", "i32", ())],
                 "prioritized", 512, zero_frac=0.01, update=True),
    # configs[2]: Gato/DB1-shaped token table, host-pinned zero-copy.
    "c3": Config("c3_gato_db1", 1_000_000, 1024,
                 [ColSpec("tokens", "i32", (), "host")],
                 "weighted", 1024, prio="tasks", zero_frac=0.005),
    # configs[3]: MAT-shaped multi-agent table, mixed HBM + host columns.
    "c4": Config("c4_mat", 500_000, 64,
                 [ColSpec("obs", "f32", (8, 128)), ColSpec("action", "i32", (8,)),
                  ColSpec("reward", "f32", (8,)), ColSpec("done", "u8", (8,)),
                  ColSpec("share_obs", "f32", (8, 216), "host"), ColSpec("avail", "u8", (8, 14), "host")],
                 "prioritized", 256, zero_frac=0.0, update=True),
    # configs[4]: scale sweep, host-resident (N scaled to the box's RAM).
    "c5": Config("c5_scale", 10_000_000, 64,
                 [ColSpec("obs", "u8", (1600,), "host"), ColSpec("action", "i32", (), "host"),
                  ColSpec("reward", "f32", (), "host")],
                 "prioritized", 4096, zero_frac=0.01, update=True),
}
