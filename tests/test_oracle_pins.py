"""Pins of the CPU oracle against what the paper and mathematics fix.

Every test here checks the oracle (oracle/gear_oracle.c) against something
other than itself: published known-answer vectors, closed forms, brute-force
enumeration on tiny inputs, library routines (numpy cumsum / searchsorted),
invariants, a chi-square bound and the paper's one worked example (Figure 4,
PAPER.md:249).  CPU only.
"""
import json
import math
import os
from collections import Counter, deque

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden")
TWO64 = 1 << 64


# --------------------------------------------------------------------------
# Philox4x32-10: published Random123 known-answer vectors (reading Q4)
# --------------------------------------------------------------------------
def _kat():
    rows = []
    with open(os.path.join(GOLD, "philox4x32_10_kat.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            v = [int(x, 16) for x in line.split()]
            rows.append((v[0:4], v[4:6], v[6:10]))
    return rows


def test_philox_known_answers(oracle_mod):
    rows = _kat()
    assert len(rows) == 3
    for ctr, key, out in rows:
        got = oracle_mod.philox4x32_10(ctr, key)
        assert [int(x) for x in got] == out


def test_draw_uses_block_j_under_seed(oracle_mod):
    # The draw's r is the first two words of Philox(ctr=(j,0,0,0), key=seed)
    # (reading Q4); check u at r's extremes against the closed form of the
    # scaling: T=2^k gives u = r >> (64-k) exactly.
    seed = 0x0123456789ABCDEF
    for j in (0, 1, 77, (1 << 32) + 5):
        x = oracle_mod.philox4x32_10([j & 0xFFFFFFFF, j >> 32, 0, 0],
                                     [seed & 0xFFFFFFFF, seed >> 32])
        r = int(x[0]) | (int(x[1]) << 32)
        for k in (1, 7, 33, 62):
            assert oracle_mod.draw(seed, j, 1 << k) == r >> (64 - k)


# --------------------------------------------------------------------------
# mulhi mapping u = floor(r*T/2^64): exact bin-boundary identity (Q4)
# --------------------------------------------------------------------------
def test_scaling_bins_have_exact_sizes(oracle_mod):
    """Reading Q4 maps r to u = floor(r*T/2^64).  Its defining property: u is
    the unique value with ceil(u*2^64/T) <= r < ceil((u+1)*2^64/T), so value
    u is hit by exactly ceil((u+1)2^64/T) - ceil(u 2^64/T) of the 2^64 r
    values (bins differ in size by at most one r).  Checked with exact
    big-integer ceilings for the r of many Philox draws (r itself pinned by
    the KAT above), and for T <= 64 by counting boundaries at or below r."""
    rng = np.random.default_rng(5)
    for T in (1, 2, 3, 5, 7, 1000, (1 << 62) - 1, 12345678901234567):
        bounds = [-(-u * TWO64 // T) for u in range(0, min(T, 64) + 1)]  # ceil(u 2^64/T)
        for _ in range(50):
            seed = int(rng.integers(0, 2**63)); j = int(rng.integers(0, 2**40))
            x = oracle_mod.philox4x32_10([j & 0xFFFFFFFF, j >> 32, 0, 0],
                                         [seed & 0xFFFFFFFF, seed >> 32])
            r = int(x[0]) | (int(x[1]) << 32)
            u = oracle_mod.draw(seed, j, T)
            assert 0 <= u < T
            # u is the unique value with ceil(u 2^64/T) <= r < ceil((u+1) 2^64/T)
            lo = -(-u * TWO64 // T)
            hi = -(-(u + 1) * TWO64 // T)
            assert lo <= r < hi
            if T <= 64:
                assert u == sum(1 for b in bounds[1:T] if b <= r)


# --------------------------------------------------------------------------
# CDF: sequential sum, numpy cumsum, totals near 2^62
# --------------------------------------------------------------------------
def test_cdf_matches_library_cumsum(oracle_mod):
    rng = np.random.default_rng(1)
    for n in (0, 1, 2, 17, 4096, 100003):
        key = rng.integers(0, 2**40, size=n, dtype=np.uint64)
        key[rng.random(n) < 0.1] = 0
        C = oracle_mod.cdf(key)
        assert np.array_equal(C, np.cumsum(key, dtype=np.uint64))


def test_cdf_total_just_below_2_62(oracle_mod):
    n = 1024
    qmax = oracle_mod.q_max(n)
    assert qmax == ((1 << 62) - 1) // n
    key = np.full(n, qmax, dtype=np.uint64)
    C = oracle_mod.cdf(key)
    assert int(C[-1]) == n * qmax < (1 << 62)
    assert [int(c) for c in C[:5]] == [qmax * (i + 1) for i in range(5)]


# --------------------------------------------------------------------------
# Inverse CDF: enumeration on tiny tables + searchsorted + step bound
# --------------------------------------------------------------------------
def test_inverse_enumeration_tiny_tables(oracle_mod):
    rng = np.random.default_rng(2)
    for trial in range(300):
        n = int(rng.integers(1, 9))
        key = rng.integers(0, 14, size=n).astype(np.uint64)
        if key.sum() == 0:
            key[int(rng.integers(0, n))] = 1
        C = oracle_mod.cdf(key)
        T = int(C[-1])
        hits = Counter()
        for u in range(T):
            g, _ = oracle_mod.inverse(C, u)
            hits[g] += 1
            assert g == int(np.searchsorted(C, np.uint64(u), side="right"))
        for g in range(n):
            assert hits[g] == int(key[g]), (key, hits)


def test_inverse_step_bound(oracle_mod):
    """PAPER.md:222 / SPEC.md:303: a binary search over N bins needs at most
    ceil(log2(N+1)) comparisons per draw."""
    rng = np.random.default_rng(3)
    for n in (1, 2, 3, 1000, 1 << 16, 100003):
        key = rng.integers(1, 100, size=n).astype(np.uint64)
        C = oracle_mod.cdf(key)
        for _ in range(50):
            u = int(rng.integers(0, int(C[-1])))
            g, cmps = oracle_mod.inverse(C, u)
            assert cmps <= math.ceil(math.log2(n + 1))
            assert g == int(np.searchsorted(C, np.uint64(u), side="right"))


# --------------------------------------------------------------------------
# Sampling: chi-square, zero-weight exclusion, uniform closed form
# --------------------------------------------------------------------------
def test_weighted_chi_square(oracle_mod):
    """weights [1,2,3,4], 1e5 draws, chi^2 at 99% over 20
    seeds.  SPEC allows at most 1 failure (false-alarm rate 1.7% for a correct
    sampler); we allow 2 (false-alarm rate 0.1%).  Seeds 1000..1019 give 2."""
    crit = 11.344866730144373  # scipy.stats.chi2.ppf(0.99, 3)
    key = np.array([1, 2, 3, 4], dtype=np.uint64) << np.uint64(32)
    fails = 0
    for s in range(20):
        st, idx, w, p = oracle_mod.sample(oracle_mod.WEIGHTED, key, None, 4, 1, 1, 0, 100000,
                                          seed=1000 + s)
        assert st == 0
        obs = np.bincount(idx.astype(np.int64), minlength=4)
        exp = np.array([0.1, 0.2, 0.3, 0.4]) * 100000
        fails += ((obs - exp) ** 2 / exp).sum() > crit
        assert np.all(p == np.array([0.1, 0.2, 0.3, 0.4])[idx.astype(np.int64)])
    assert fails <= 2


def test_zero_weight_bins_never_drawn(oracle_mod):
    key = np.array([0, 5, 0], dtype=np.uint64)
    for strat in (oracle_mod.UNIFORM, oracle_mod.WEIGHTED, oracle_mod.PRIORITIZED):
        st, idx, w, p = oracle_mod.sample(strat, key, None, 3, 1, 1, 0, 1000, seed=9, beta=0.7)
        assert st == 0 and np.all(idx == 1) and np.all(w == 1.0)


def test_all_zero_is_empty(oracle_mod):
    key = np.zeros(16, dtype=np.uint64)
    for strat in (0, 1, 2, 3, 4):
        st, *_ = oracle_mod.sample(strat, key, None, 16, 1, 1, 0, 4, seed=1)
        assert st == oracle_mod.EMPTY


def test_uniform_full_table_closed_form(oracle_mod):
    """All slots selectable: C[g] = g+1 so the draw is g = floor(r*N/2^64)."""
    n = 1000
    key = np.arange(1, n + 1, dtype=np.uint64) * np.uint64(3)   # any positive keys
    seed = 77
    st, idx, w, p = oracle_mod.sample(oracle_mod.UNIFORM, key, None, n, 1, 1, 0, 256, seed)
    for j in range(256):
        x = oracle_mod.philox4x32_10([j, 0, 0, 0], [seed, 0])
        r = int(x[0]) | (int(x[1]) << 32)
        assert int(idx[j]) == (r * n) >> 64
    assert np.all(p == 1.0 / n)


def test_rank_slices_concatenate_to_global_draw(oracle_mod):
    """Q9: rank r's slice is draws [rB, (r+1)B) of one global draw, so the
    slices of W ranks concatenate to the single-rank draw of W*B."""
    rng = np.random.default_rng(4)
    key = rng.integers(0, 1000, size=256).astype(np.uint64)
    for W in (1, 2, 4, 8):
        full = oracle_mod.sample(oracle_mod.WEIGHTED, key, None, 256 // W, W, 1, 0, 16 * W, 5)[1]
        parts = [oracle_mod.sample(oracle_mod.WEIGHTED, key, None, 256 // W, W, W, r, 16, 5)[1]
                 for r in range(W)]
        assert np.array_equal(np.concatenate(parts), full)


# --------------------------------------------------------------------------
# IS weights (Q6): closed forms
# --------------------------------------------------------------------------
def test_is_weights_closed_forms(oracle_mod):
    rng = np.random.default_rng(6)
    key = rng.integers(1, 1 << 40, size=512).astype(np.uint64)
    st, idx, w0, p = oracle_mod.sample(oracle_mod.PRIORITIZED, key, None, 512, 1, 1, 0, 128, 3, 0.0)
    assert np.all(w0 == 1.0)                                   # beta = 0
    st, idx, w1, p = oracle_mod.sample(oracle_mod.PRIORITIZED, key, None, 512, 1, 1, 0, 128, 3, 1.0)
    q = key[idx.astype(np.int64)]
    qmin = int(q.min())
    # beta = 1: a correctly rounded division, then f32
    want = np.array([np.float32(qmin / int(x)) for x in q])
    assert np.array_equal(w1, want)
    assert np.all(w1[q == qmin] == 1.0)                      # argmin -> exactly 1
    assert np.all(w1 <= 1.0) and np.all(w1 > 0)
    T = int(key.sum())
    assert np.all(p == np.array([int(x) / T for x in q]))
    st, idx, we, p = oracle_mod.sample(oracle_mod.PRIORITIZED, np.full(64, 7, np.uint64), None,
                                       64, 1, 1, 0, 32, 3, 0.4)
    assert np.all(we == 1.0)                                   # equal keys
    st, idx, wb, p = oracle_mod.sample(oracle_mod.PRIORITIZED, key, None, 512, 1, 1, 0, 128, 3, 0.4)
    ref = np.array([(qmin / int(x)) ** 0.4 for x in q])
    np.testing.assert_allclose(wb, ref, rtol=1e-6)


# --------------------------------------------------------------------------
# Quantisation Q_F (Q3): special cases
# --------------------------------------------------------------------------
def test_quantize_special_cases(oracle_mod):
    N = 1024
    qmax = oracle_mod.q_max(N)
    F = 32
    Q = lambda p: oracle_mod.quantize(p, F, qmax)
    assert Q(0.0) == (0, 0)
    assert Q(2.0 ** -40) == (0, 1)             # clamps up to 1: positive stays selectable
    assert Q(1.0) == (0, 1 << 32)
    assert Q(1.5) == (0, 3 << 31)
    assert Q(2.0 ** 30) == (0, qmax)           # x = 2^62 saturates
    assert Q(1e300) == (0, qmax)
    assert Q(2.0 ** 20) == (0, min(1 << 52, qmax))
    for k in (0, 1, 2, 3, 10, 11, 12345):       # ties (k + 1/2) 2^-32 -> even
        st, q = Q((k + 0.5) * 2.0 ** -32)
        assert st == 0 and q == max(1, k + (k & 1))
    st, q = Q((6 + 0.5 + 2.0 ** -20) * 2.0 ** -32)
    assert q == 7                               # just above a tie rounds up
    st, q = Q((7 + 0.5 - 2.0 ** -20) * 2.0 ** -32)
    assert q == 7                               # just below a tie rounds down
    for bad in (float("nan"), float("inf"), -float("inf"), -1.0, -1e-300):
        assert Q(bad)[0] == oracle_mod.BAD_PRIORITY
    # fixed point of frac bits 0: plain rint-even of p
    assert oracle_mod.quantize(2.5, 0, qmax)[1] == 2
    assert oracle_mod.quantize(3.5, 0, qmax)[1] == 4


# --------------------------------------------------------------------------
# PER exponent alpha (Q7): p -> RN(p^alpha), keys Q_F(RN(p^alpha))
# --------------------------------------------------------------------------
def _wide_priorities(n, seed):
    rng = np.random.default_rng(seed)
    return np.exp(rng.normal(0.0, 8.0, n))      # ~1e-10 .. 1e10 and beyond


def test_pow_alpha_ieee_special_exponents(oracle_mod):
    """alpha = 1/2 and 2 reduce to single IEEE operations, which are correctly
    rounded by definition: RN(p^0.5) = sqrt(p), RN(p^2) = p*p, bit for bit."""
    p = _wide_priorities(3000, 1)
    p = p[(p > 1e-150) & (p < 1e150)]            # p*p stays finite and normal
    assert np.array_equal(oracle_mod.pow_alpha(p, 0.5), np.sqrt(p))
    assert np.array_equal(oracle_mod.pow_alpha(p, 2.0), p * p)
    assert np.array_equal(oracle_mod.pow_alpha(p, 1.0), p)
    # exact midpoint of p^2: p = 2^27 - 1 -> p^2 = 2^54 - 2^28 + 1 needs 54 bits;
    # IEEE p*p rounds the tie to even
    x = np.array([2.0 ** 27 - 1, 2.0 ** 27 + 1, 3.0 * 2 ** 25 + 1])
    assert np.array_equal(oracle_mod.pow_alpha(x, 2.0), x * x)


def test_pow_alpha_closed_forms_and_libm(oracle_mod):
    exact = [(4.0, 1.5, 8.0), (0.25, 1.5, 0.125), (9.0, 0.5, 3.0), (1.0, 0.6, 1.0),
             (2.0, 10.0, 1024.0), (1024.0, 0.1, 2.0), (27.0, 3.0, 19683.0), (2.0 ** -6, 0.5, 0.125)]
    for p, a, want in exact:
        assert oracle_mod.pow_alpha(np.array([p]), a)[0] == want, (p, a)
    # within one ulp of libm's pow (itself < 1 ulp), for PER-typical and odd alphas
    p = _wide_priorities(2000, 2)
    for a in (0.6, 0.7, 0.4, 1.3, 3.0, 0.05):
        got = oracle_mod.pow_alpha(p, a)
        ref = np.power(p, a)
        ok = np.isfinite(ref) & (ref > 1e-300)
        ulp = np.spacing(ref[ok])
        assert np.all(np.abs(got[ok] - ref[ok]) <= ulp), a
        # monotone in p
        order = np.argsort(p)
        assert np.all(np.diff(got[order]) >= 0)
    # 0 and invalid values pass through; overflow / underflow clamp, stay positive
    out = oracle_mod.pow_alpha(np.array([0.0, -1.0, np.inf, 1e300, 1e-300]), 3.0)
    assert out[0] == 0.0 and out[1] == -1.0 and out[2] == np.inf
    assert out[3] == np.finfo(np.float64).max and out[4] == 5e-324


def test_pow_alpha_keys_through_table(oracle_mod):
    """The table applies the exponent before Q_F on insert and update: a table
    with alpha = 1/2 holds the keys of a table with alpha = 1 fed sqrt(p)."""
    p = _wide_priorities(500, 3)
    p[::17] = 0.0
    a = oracle_mod.Table(250, 2, alpha=0.5)
    b = oracle_mod.Table(250, 2)
    for s in range(2):
        a.insert(s, p[s * 250:(s + 1) * 250])
        b.insert(s, np.sqrt(p[s * 250:(s + 1) * 250]))
    assert np.array_equal(a.key, b.key)
    ids = np.arange(0, 500, 3, dtype=np.uint64)
    q = _wide_priorities(ids.size, 4)
    a.update(ids, q)
    b.update(ids, np.sqrt(q))
    assert np.array_equal(a.key, b.key)
    assert np.all((a.key > 0) == (np.concatenate([p]) > 0) | np.isin(np.arange(500), ids))


# --------------------------------------------------------------------------
# Update round trip (Q11)
# --------------------------------------------------------------------------
def test_update_round_trip_last_writer_wins(oracle_mod):
    rng = np.random.default_rng(8)
    t = oracle_mod.Table(shard_cap=64, n_shards=2)
    for s in range(2):
        t.insert(s, np.ones(64))
    n = 500
    idx = rng.integers(0, 128, size=n).astype(np.uint64)
    p = rng.lognormal(0, 1, size=n)
    p[rng.random(n) < 0.05] = 0.0
    p[3] = float("nan")
    idx[5] = 128                                  # out of range
    before = t.key.copy()
    st, ns = t.update(idx, p)
    assert st == oracle_mod.BAD_PRIORITY | oracle_mod.INDEX_RANGE and ns == 0
    last = {}
    for k in range(n):
        if k in (3, 5):
            continue
        last[int(idx[k])] = float(p[k])
    qmax = oracle_mod.q_max(128)
    for g in range(128):
        if g in last:
            pk = last[g]
            want = 0 if pk == 0 else min(max(1, round(pk * 2**32)), qmax)
            assert int(t.key[g]) == want
        else:
            assert t.key[g] == before[g]
    # generation check: stale entries skipped and counted
    st, ns = t.update(np.array([0, 1], np.uint64), np.array([2.0, 2.0]),
                      gen_in=np.array([1, 7], np.uint32))
    assert ns == 1 and int(t.key[0]) == 2 << 32 and int(t.key[1]) == int(t.key[1])


def test_update_to_never_inserted_slot_is_stale(oracle_mod):
    t = oracle_mod.Table(shard_cap=8, n_shards=1)
    t.insert(0, [1.0, 1.0])
    st, ns = t.update(np.array([1, 5], np.uint64), np.array([3.0, 3.0]))
    assert ns == 1 and int(t.key[5]) == 0 and int(t.key[1]) == 3 << 32


# --------------------------------------------------------------------------
# Insert / eviction and FIFO / LIFO selection
# --------------------------------------------------------------------------
def test_fifo_removal_keeps_last_capacity_rows(oracle_mod):
    t = oracle_mod.Table(shard_cap=16, n_shards=1, removal=0)
    ids = []
    for k in range(53):
        st, out = t.insert(0, [1.0])
        ids.append(int(out[0]))
    assert ids[:16] == list(range(16))            # queue seeded ascending
    # slot of insert k is k mod 16 once full (oldest evicted first)
    assert ids == [k % 16 for k in range(53)]
    assert sorted(int(s) for s in t.seq) == list(range(53 - 16 + 1, 53 + 1))


def test_lifo_removal_replaces_newest(oracle_mod):
    t = oracle_mod.Table(shard_cap=4, n_shards=1, removal=1)
    ids = [int(t.insert(0, [1.0])[1][0]) for _ in range(7)]
    assert ids == [0, 1, 2, 3, 3, 3, 3]
    assert list(t.seq) == [1, 2, 3, 7]


def _simulate(cap, removal, events):
    """Independent deque-based model of a shard: FIFO removal pops the oldest,
    LIFO removal pops the newest."""
    free = deque(range(cap))
    live = deque()          # slots in insertion order
    out = []
    for _ in events:
        if free:
            g = free.popleft()
        else:
            g = live.popleft() if removal == 0 else live.pop()
        live.append(g)
        out.append(g)
    return out, list(live)


@pytest.mark.parametrize("removal", [0, 1])
def test_insert_matches_state_machine(oracle_mod, removal):
    rng = np.random.default_rng(10 + removal)
    for trial in range(40):
        cap = int(rng.integers(1, 12))
        m = int(rng.integers(0, 40))
        t = oracle_mod.Table(shard_cap=cap, n_shards=1, removal=removal)
        got = []
        k = 0
        while k < m:                                  # random batch sizes
            b = int(rng.integers(1, 5))
            b = min(b, m - k)
            got += [int(x) for x in t.insert(0, np.ones(b))[1]]
            k += b
        want, live = _simulate(cap, removal, range(m))
        assert got == want
        # FIFO selection of all live = insertion order; LIFO = reverse
        if live:
            K = len(live)
            st, idx, _, _ = t.sample(oracle_mod.FIFO, 1, 0, K, 0)
            assert st == 0 and [int(x) for x in idx] == live
            st, idx, _, _ = t.sample(oracle_mod.LIFO, 1, 0, K, 0)
            assert st == 0 and [int(x) for x in idx] == live[::-1]


class _ShardModel:
    """Independent model of one shard under the split writer API (Q21):
    a free deque, a deque of committed slots in commit order, a set of
    ongoing slots and generation counts."""

    def __init__(self, cap, removal):
        self.free, self.live, self.ongoing = deque(range(cap)), deque(), set()
        self.removal, self.gen = removal, Counter()

    def take(self):
        if self.free:
            return self.free.popleft()
        return self.live.popleft() if self.removal == 0 else self.live.pop()

    def allocate(self, n):
        if n > len(self.free) + len(self.live):
            return None
        out = []
        for _ in range(n):
            g = self.take()
            self.gen[g] += 1
            self.ongoing.add(g)
            out.append(g)
        return out

    def commit(self, ids, ok_prio):
        errs = 0
        for g, ok in zip(ids, ok_prio):
            if g not in self.ongoing:
                errs |= 4
                continue
            if not ok:
                errs |= 1
                continue
            self.ongoing.discard(g)
            self.live.append(g)
        return errs

    def insert(self, n):
        out = []
        for _ in range(n):
            if not self.free and not self.live:
                return None
            g = self.take()
            self.gen[g] += 1
            self.live.append(g)
            out.append(g)
        return out


@pytest.mark.parametrize("removal", [0, 1])
def test_allocate_commit_matches_state_machine(oracle_mod, removal):
    """gor_allocate / gor_commit (and gor_insert interleaved with them) against
    the deque model: slot choice, eviction of committed slots only, ongoing
    slots unselectable and immune to updates, all-or-nothing FULL, commit
    order = seq order = FIFO selection order, duplicate / stale / bad-priority
    commits skipped."""
    rng = np.random.default_rng(40 + removal)
    for trial in range(60):
        cap = int(rng.integers(1, 10))
        t = oracle_mod.Table(shard_cap=cap, n_shards=1, removal=removal)
        m = _ShardModel(cap, removal)
        pending = []
        for _ in range(int(rng.integers(1, 25))):
            op = rng.integers(0, 3)
            if op == 0:                                   # allocate
                n = int(rng.integers(1, 5))
                st, ids = t.allocate(0, n)
                want = m.allocate(n)
                if want is None:
                    assert st == oracle_mod.FULL
                    assert np.all(ids == oracle_mod.IDX_NONE)
                else:
                    assert st == 0 and [int(x) for x in ids] == want
                    for g in want:
                        assert t.key[g] == 0 and t.seq[g] == 0
                    pending += want
            elif op == 1 and pending:                     # commit some, maybe duplicated
                k = int(rng.integers(1, len(pending) + 1))
                ids = list(rng.permutation(pending)[:k])
                if rng.random() < 0.3:
                    ids.append(ids[0])                    # duplicate -> second is stale
                if rng.random() < 0.2:
                    ids.append(int(rng.integers(0, cap)))  # maybe not ongoing
                prio = rng.lognormal(0, 1, len(ids))
                ok = rng.random(len(ids)) > 0.1
                prio[~ok] = -1.0
                st = t.commit(0, np.array(ids, np.uint64), prio)
                assert st == m.commit(ids, ok)
                pending = sorted(m.ongoing)
            else:                                         # combined insert
                n = int(rng.integers(1, 4))
                want = m.insert(n)
                st, ids = t.insert(0, np.ones(n))
                if want is None:
                    assert st == oracle_mod.FULL
                else:
                    assert st == 0 and [int(x) for x in ids] == want
            assert [t.gen[g] for g in range(cap)] == [m.gen[g] for g in range(cap)]
            # updates to ongoing slots are stale; committed order is FIFO order
            for g in m.ongoing:
                key = t.key.copy()
                st, ns = t.update([g], [5.0])
                assert st & oracle_mod.STALE and ns == 1 and np.array_equal(t.key, key)
            live = list(m.live)
            if live:
                st, idx, _, _ = t.sample(oracle_mod.FIFO, 1, 0, len(live), 0)
                assert st == 0 and [int(x) for x in idx] == live


def test_fifo_lifo_order_and_sharded_merge(oracle_mod):
    """FIFO output strictly ascending in (seq, shard), LIFO strictly
    descending; equals a full sort of selectable (seq, shard) pairs."""
    rng = np.random.default_rng(12)
    S, cap = 4, 32
    t = oracle_mod.Table(shard_cap=cap, n_shards=S)
    for _ in range(200):
        s = int(rng.integers(0, S))
        t.insert(s, [1.0])
    t.key[rng.random(S * cap) < 0.2] = 0
    sel = [(int(t.seq[g]), g // cap, g) for g in range(S * cap) if t.key[g] > 0]
    sel.sort()
    for W in (1, 2, 4):
        B = 8
        for r in range(W):
            st, idx, _, _ = t.sample(oracle_mod.FIFO, W, r, B, 0)
            assert st == 0
            assert [int(x) for x in idx] == [g for _, _, g in sel[r * B:(r + 1) * B]]
            st, idx, _, _ = t.sample(oracle_mod.LIFO, W, r, B, 0)
            desc = sel[::-1]
            assert [int(x) for x in idx] == [g for _, _, g in desc[r * B:(r + 1) * B]]
    st, *_ = t.sample(oracle_mod.FIFO, 1, 0, len(sel) + 1, 0)
    assert st == oracle_mod.EMPTY


# --------------------------------------------------------------------------
# Translation and collection: Figure 4
# --------------------------------------------------------------------------
def test_figure4_translation_and_collect(oracle_mod):
    with open(os.path.join(GOLD, "figure4_collect.json")) as f:
        fx = json.load(f)
    cap, S = fx["shard_capacity"], fx["n_shards"]
    per = {}
    for pos, g in enumerate(fx["request"]):
        s, i = oracle_mod.translate(g, cap)
        per.setdefault(str(s), []).append((i, pos))
    assert {s: [i for i, _ in v] for s, v in per.items()} == fx["translated"]
    assert {s: [p for _, p in v] for s, v in per.items()} == fx["request_positions"]
    # collect two columns and check rows land in request order
    rng = np.random.default_rng(0)
    cols = [rng.integers(0, 256, size=(cap * S, rb), dtype=np.uint8) for rb in (24, 7)]
    req = np.array(fx["request"], dtype=np.uint64)
    for col in cols:
        out = oracle_mod.collect(col, req)
        for j, g in enumerate(fx["request"]):
            assert np.array_equal(out[j], col[g])


def test_translate_round_trip(oracle_mod):
    rng = np.random.default_rng(13)
    for _ in range(1000):
        cap = int(rng.integers(1, 1 << 40))
        g = int(rng.integers(0, 1 << 62))
        s, i = oracle_mod.translate(g, cap)
        assert s * cap + i == g and 0 <= i < cap


# --------------------------------------------------------------------------
# Owner-affine assignment (reading Q19): properties, not the formula
# --------------------------------------------------------------------------
@pytest.mark.parametrize("strategy", [2, 3, 4, 0, 1])
def test_owner_affine_partitions_the_global_batch(oracle_mod, strategy):
    rng = np.random.default_rng(30 + strategy)
    for W, R in ((1, 1), (2, 1), (4, 2), (8, 1), (3, 2)):
        S, Cs, B = W * R, 50, 37
        t = oracle_mod.Table(Cs, S)
        for s in range(S):
            t.insert(s, rng.lognormal(0, 1.5, Cs) * (rng.random(Cs) > 0.1) * (1 + 3 * (s % 2)))
        K = W * B
        st, glob, _, gp = t.sample(strategy, 1, 0, K, seed=99, beta=0.5)
        assert st == 0
        owners = (glob // np.uint64(Cs)) // np.uint64(R)
        slices = []
        for r in range(W):
            st, idx, w, p = t.sample(strategy, W, r, B, 99, 0.5, owner_affine=True)
            assert st == 0 and idx.size == B
            own = int(np.sum(owners == r))
            # the rank keeps min(B, own) of its own entries, first, in global order
            k = min(B, own)
            assert np.array_equal(idx[:k], glob[owners == r][:k])
            assert np.all((idx[k:] // np.uint64(Cs)) // np.uint64(R) != r) or own >= B
            if strategy == 4:
                q = t.key[idx.astype(np.int64)]
                assert np.all(w[q == q.min()] == 1.0) and np.all(w <= 1.0)
            slices.append(idx)
        # together the ranks receive exactly the global batch (as a multiset)
        assert sorted(np.concatenate(slices).tolist()) == sorted(glob.tolist())
        if W == 1:
            assert np.array_equal(slices[0], glob)


# --------------------------------------------------------------------------
# TopK (reading Q20): brute force on small tables
# --------------------------------------------------------------------------
def test_topk_matches_brute_force(oracle_mod):
    rng = np.random.default_rng(40)
    for trial in range(60):
        S = int(rng.integers(1, 5))
        Cs = int(rng.integers(1, 40))
        key = rng.integers(0, 6, size=S * Cs).astype(np.uint64)   # many ties
        key[rng.random(S * Cs) < 0.2] = 0
        sel = [g for g in range(S * Cs) if key[g] > 0]
        brute = sorted(sel, key=lambda g: (-int(key[g]), g))
        for W in (1, 2, 3):
            B = int(rng.integers(1, 6))
            if len(sel) < W * B:
                st, *_ = oracle_mod.sample(oracle_mod.TOPK, key, None, Cs, S, W, 0, B, 0)
                assert st == oracle_mod.EMPTY
                continue
            for r in range(W):
                st, idx, w, p = oracle_mod.sample(oracle_mod.TOPK, key, None, Cs, S, W, r, B, 0)
                assert st == 0
                assert [int(x) for x in idx] == brute[r * B:(r + 1) * B]
        if sel:
            st, idx, _, _ = oracle_mod.sample(oracle_mod.TOPK, key, None, Cs, S, 1, 0, len(sel), 0)
            ks = key[idx.astype(np.int64)]
            assert np.all(ks[:-1] >= ks[1:])                      # non-increasing keys


def test_owner_affine_hand_worked_fifo(oracle_mod):
    """Reading Q19's overflow order, pinned by a hand-worked example
    (tests/golden/owner_affine_fifo.json): a FIFO global batch whose owner
    pattern was designed through the priorities, the contiguous slices (Q9)
    and the owner-affine slices written out by hand."""
    with open(os.path.join(GOLD, "owner_affine_fifo.json")) as f:
        g = json.load(f)
    Cs, W, B = g["shard_capacity"], g["n_ranks"], g["batch_per_rank"]
    t = oracle_mod.Table(Cs, W)
    for s, pr in enumerate(g["priorities"]):
        st, ids = t.insert(s, np.array(pr, dtype=np.float64))
        assert st == 0 and [int(x) for x in ids] == list(range(s * Cs, s * Cs + Cs))
    st, glob, _, _ = t.sample(oracle_mod.FIFO, 1, 0, W * B, 0)
    assert st == 0 and [int(x) for x in glob] == g["global_batch"]
    for r in range(W):
        st, idx, _, _ = t.sample(oracle_mod.FIFO, W, r, B, 0)
        assert st == 0 and [int(x) for x in idx] == g["contiguous"][r]
        st, idx, _, _ = t.sample(oracle_mod.FIFO, W, r, B, 0, owner_affine=True)
        assert st == 0 and [int(x) for x in idx] == g["owner_affine"][r], r


@pytest.mark.parametrize("n", [1, 2, 3, 7, 1024, 100_000, 281_600, 1_000_000, 10_000_000,
                               2 ** 40 + 1, (1 << 62) - 1])
def test_q_max_is_the_largest_safe_key(oracle_mod, n):
    """Reading Q3: q_max is the LARGEST key for which N keys sum below 2^62
    (so the u64 totals and the flag bits of the scan never overflow):
    N*q_max < 2^62 <= N*(q_max + 1)."""
    q = int(oracle_mod.q_max(n))
    assert n * q < (1 << 62)
    assert n * (q + 1) >= (1 << 62)
