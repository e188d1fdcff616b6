"""CPU oracle for the GEAR replay hot path -- TEST INFRASTRUCTURE ONLY.

This package is the plain, slow, single-threaded definition of what the CUDA
path computes (see gear_oracle.h for the per-function citations into
PAPER.md and the readings Q1..Q21 in DESIGN.md §3).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` legs may import it.  It shares no code with
``paper_2310_05205_b200`` and never imports it.

The C source is compiled with gcc into ``oracle/liboracle.so``; this module
only marshals numpy arrays into it.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gear_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

FIFO, LIFO, UNIFORM, WEIGHTED, PRIORITIZED, TOPK = 0, 1, 2, 3, 4, 5
OK, BAD_PRIORITY, INDEX_RANGE, STALE, EMPTY, INVALID, FULL = 0, 1, 2, 4, 8, 16, 32
IDX_NONE = np.uint64(0xFFFFFFFFFFFFFFFF)


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain C11, -O2, no fast-math)."""
    hdr = os.path.join(_HERE, "gear_oracle.h")
    if (not force and os.path.exists(_LIB)
            and os.path.getmtime(_LIB) >= max(os.path.getmtime(_SRC), os.path.getmtime(hdr))):
        return _LIB
    tmp = _LIB + f".tmp{os.getpid()}"
    subprocess.check_call(["gcc", "-std=gnu11", "-O2", "-fPIC", "-shared",
                           "-fno-fast-math", "-ffp-contract=off",
                           "-o", tmp, _SRC, "-lm"])
    os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        u32, u64, i32, f64 = ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int, ctypes.c_double
        L.gor_philox4x32_10.argtypes = [P, P, P]
        L.gor_q_max.argtypes = [u64]
        L.gor_q_max.restype = u64
        L.gor_quantize.argtypes = [f64, u32, u64, P]
        L.gor_quantize.restype = i32
        L.gor_cdf.argtypes = [P, u64, P]
        L.gor_draw.argtypes = [u64, u64, u64]
        L.gor_draw.restype = u64
        L.gor_inverse.argtypes = [P, u64, u64, P]
        L.gor_inverse.restype = u64
        L.gor_sample.argtypes = [i32, P, P, u64, u32, u32, u32, u32, u64, f64, P, P, P]
        L.gor_sample.restype = i32
        L.gor_sample_owner_affine.argtypes = [i32, P, P, u64, u32, u32, u32, u32, u64, f64, P, P, P]
        L.gor_sample_owner_affine.restype = i32
        L.gor_update.argtypes = [P, P, P, u64, u32, u32, P, P, P, P]
        L.gor_update.restype = i32
        L.gor_translate.argtypes = [u64, u64, P, P]
        L.gor_collect.argtypes = [P, u64, u64, u32, P, P]
        L.gor_collect.restype = i32
        L.gor_insert.argtypes = [P, P, P, u64, u64, u32, u32, u32, P, P, u32, P, P]
        L.gor_insert.restype = i32
        L.gor_allocate.argtypes = [P, P, P, u64, u32, u32, P, u32, P]
        L.gor_allocate.restype = i32
        L.gor_commit.argtypes = [P, P, P, u64, u64, u32, u32, P, u32, P, P]
        L.gor_commit.restype = i32
        _lib = L
    return _lib


def _p(a: np.ndarray | None):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.c_void_p)


def philox4x32_10(ctr, key) -> np.ndarray:
    c = np.ascontiguousarray(ctr, dtype=np.uint32)
    k = np.ascontiguousarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    lib().gor_philox4x32_10(_p(c), _p(k), _p(out))
    return out


def q_max(n_global: int) -> int:
    return int(lib().gor_q_max(n_global))


def quantize(p: float, frac_bits: int, qmax: int):
    """Returns (status, q)."""
    q = np.zeros(1, dtype=np.uint64)
    st = lib().gor_quantize(float(p), frac_bits, qmax, _p(q))
    return st, int(q[0])


def pow_alpha(p, alpha: float) -> np.ndarray:
    """PER priority exponent (Schaul et al. 2016, P(i) = p_i^alpha / sum_k p_k^alpha;
    the paper names PER at PAPER.md:55,121 and gives no formula -- reading Q7):
    every finite p > 0 becomes p^alpha rounded to the nearest double (ties to
    even).  The power is taken by mpmath at 200-bit precision -- exact when it
    fits in 200 bits (p^2, p^3, ...), else within a few 2^-200 -- and rounded
    once to 53 bits.  Results above DBL_MAX become DBL_MAX and results below
    the least subnormal become it, so a positive priority never turns into 0
    (below 2^-1022 only positivity matters: such keys are clamped to 1).
    p = 0 and invalid values (NaN, inf, negative) pass through unchanged for
    the quantiser to handle."""
    p = np.ascontiguousarray(p, dtype=np.float64)
    if alpha == 1.0:
        return p.copy()
    from mpmath import mp, mpf
    out = p.copy()
    with mp.workprec(200):
        a = mpf(float(alpha))
        for i, x in enumerate(p.tolist()):
            if not (x > 0.0 and math.isfinite(x)):
                continue
            f = float(mpf(x) ** a)
            if f == math.inf:
                f = float(np.finfo(np.float64).max)
            elif f == 0.0:
                f = 5e-324
            out[i] = f
    return out


def cdf(key: np.ndarray) -> np.ndarray:
    key = np.ascontiguousarray(key, dtype=np.uint64)
    C = np.zeros_like(key)
    lib().gor_cdf(_p(key), key.size, _p(C))
    return C


def draw(seed: int, j: int, T: int) -> int:
    return int(lib().gor_draw(seed, j, T))


def inverse(C: np.ndarray, u: int):
    """Returns (g, comparisons)."""
    C = np.ascontiguousarray(C, dtype=np.uint64)
    n = np.zeros(1, dtype=np.uint64)
    g = lib().gor_inverse(_p(C), C.size, u, _p(n))
    return int(g), int(n[0])


def sample(strategy: int, key: np.ndarray, seq: np.ndarray | None, shard_cap: int,
           n_shards: int, n_ranks: int, rank: int, B: int, seed: int, beta: float = 0.0):
    """Returns (status, idx u64[B], w f32[B], p f64[B])."""
    key = np.ascontiguousarray(key, dtype=np.uint64)
    seq = np.zeros_like(key) if seq is None else np.ascontiguousarray(seq, dtype=np.uint64)
    idx = np.zeros(B, dtype=np.uint64)
    w = np.zeros(B, dtype=np.float32)
    p = np.zeros(B, dtype=np.float64)
    st = lib().gor_sample(strategy, _p(key), _p(seq), shard_cap, n_shards, n_ranks, rank,
                          B, seed, float(beta), _p(idx), _p(w), _p(p))
    return st, idx, w, p


def sample_owner_affine(strategy: int, key: np.ndarray, seq: np.ndarray | None, shard_cap: int,
                        n_shards: int, n_ranks: int, rank: int, B: int, seed: int, beta: float = 0.0):
    """Reading Q19: the same global batch, assigned to ranks by owner."""
    key = np.ascontiguousarray(key, dtype=np.uint64)
    seq = np.zeros_like(key) if seq is None else np.ascontiguousarray(seq, dtype=np.uint64)
    idx = np.zeros(B, dtype=np.uint64)
    w = np.zeros(B, dtype=np.float32)
    p = np.zeros(B, dtype=np.float64)
    st = lib().gor_sample_owner_affine(strategy, _p(key), _p(seq), shard_cap, n_shards, n_ranks,
                                       rank, B, seed, float(beta), _p(idx), _p(w), _p(p))
    return st, idx, w, p


def update(key: np.ndarray, seq: np.ndarray, gen: np.ndarray, frac_bits: int, idx, p,
           gen_in=None):
    """In-place on key.  Returns (status bitmask, n_stale)."""
    assert key.dtype == np.uint64 and seq.dtype == np.uint64 and gen.dtype == np.uint32
    idx = np.ascontiguousarray(idx, dtype=np.uint64)
    p = np.ascontiguousarray(p, dtype=np.float64)
    gi = None if gen_in is None else np.ascontiguousarray(gen_in, dtype=np.uint32)
    ns = np.zeros(1, dtype=np.uint64)
    st = lib().gor_update(_p(key), _p(seq), _p(gen), key.size, frac_bits, idx.size, _p(idx), _p(p),
                          _p(gi), _p(ns))
    return st, int(ns[0])


def translate(g: int, shard_cap: int):
    s = np.zeros(1, dtype=np.uint64)
    i = np.zeros(1, dtype=np.uint64)
    lib().gor_translate(g, shard_cap, _p(s), _p(i))
    return int(s[0]), int(i[0])


def collect(col: np.ndarray, idx) -> np.ndarray:
    """col: uint8 [n_global, row_bytes] -> uint8 [len(idx), row_bytes]."""
    col = np.ascontiguousarray(col, dtype=np.uint8)
    idx = np.ascontiguousarray(idx, dtype=np.uint64)
    out = np.zeros((idx.size, col.shape[1]), dtype=np.uint8)
    st = lib().gor_collect(_p(col), col.shape[0], col.shape[1], idx.size, _p(idx), _p(out))
    if st != OK:
        raise IndexError("oracle collect: index out of range")
    return out


class Table:
    """Oracle-side replay table state: keys, seq, gen and per-shard queues.

    The whole table is one concatenated array in global id order; shards are
    only the unit of insertion and of FIFO tie-breaks.
    """

    def __init__(self, shard_cap: int, n_shards: int, frac_bits: int = 32, removal: int = 0,
                 alpha: float = 1.0):
        self.cap, self.S, self.F, self.removal = shard_cap, n_shards, frac_bits, removal
        self.alpha = alpha          # keys are Q_F(pow_alpha(p)) (reading Q7)
        n = shard_cap * n_shards
        self.key = np.zeros(n, dtype=np.uint64)
        self.seq = np.zeros(n, dtype=np.uint64)
        self.gen = np.zeros(n, dtype=np.uint32)
        self.next_free = np.zeros(n_shards, dtype=np.uint64)
        self.seq_ctr = np.ones(n_shards, dtype=np.uint64)   # seq 0 = never inserted

    @property
    def n(self) -> int:
        return self.cap * self.S

    def insert(self, shard: int, prio) -> tuple[int, np.ndarray]:
        prio = pow_alpha(prio, self.alpha)
        out = np.zeros(prio.size, dtype=np.uint64)
        nf = self.next_free[shard:shard + 1].copy()
        sc = self.seq_ctr[shard:shard + 1].copy()
        st = lib().gor_insert(_p(self.key), _p(self.seq), _p(self.gen), self.cap, self.n,
                              shard, self.removal, self.F, _p(nf), _p(sc), prio.size,
                              _p(prio), _p(out))
        self.next_free[shard] = nf[0]
        self.seq_ctr[shard] = sc[0]
        return st, out

    def update(self, idx, p, gen_in=None):
        return update(self.key, self.seq, self.gen, self.F, idx, pow_alpha(p, self.alpha), gen_in)

    def allocate(self, shard: int, n: int) -> tuple[int, np.ndarray]:
        """Split writer API (Q21): n ongoing slots of `shard`."""
        out = np.zeros(n, dtype=np.uint64)
        nf = self.next_free[shard:shard + 1].copy()
        st = lib().gor_allocate(_p(self.key), _p(self.seq), _p(self.gen), self.cap, shard,
                                self.removal, _p(nf), n, _p(out))
        self.next_free[shard] = nf[0]
        return st, out

    def commit(self, shard: int, idx, prio) -> int:
        idx = np.ascontiguousarray(idx, dtype=np.uint64)
        prio = pow_alpha(prio, self.alpha)
        sc = self.seq_ctr[shard:shard + 1].copy()
        st = lib().gor_commit(_p(self.key), _p(self.seq), _p(self.gen), self.cap, self.n, shard,
                              self.F, _p(sc), idx.size, _p(idx), _p(prio))
        self.seq_ctr[shard] = sc[0]
        return st

    def sample(self, strategy, n_ranks, rank, B, seed, beta=0.0, owner_affine=False):
        fn = sample_owner_affine if owner_affine else sample
        return fn(strategy, self.key, self.seq, self.cap, self.S, n_ranks, rank, B, seed, beta)
