"""Shared harness of the GPU parity tests: one GPU table and one oracle table
fed the same seeded inputs (synth/), plus host mirrors of the columns."""
from __future__ import annotations

import ctypes

import numpy as np

import oracle
import synth
import paper_2310_05205_b200 as gear

DT = {"u8": gear.GEAR_U8, "i32": gear.GEAR_I32, "f32": gear.GEAR_F32}
ORACLE_STRATEGY = {gear.GEAR_FIFO: oracle.FIFO, gear.GEAR_LIFO: oracle.LIFO,
                   gear.GEAR_UNIFORM: oracle.UNIFORM, gear.GEAR_WEIGHTED: oracle.WEIGHTED,
                   gear.GEAR_PRIORITIZED: oracle.PRIORITIZED, gear.GEAR_TOPK: oracle.TOPK}


def oracle_bits_to_gear(st):
    """GOR_* status bits -> GEAR_DEVERR_* bits."""
    m = {oracle.BAD_PRIORITY: gear.GEAR_DEVERR_BAD_PRIORITY,
         oracle.INDEX_RANGE: gear.GEAR_DEVERR_INDEX_RANGE, oracle.STALE: gear.GEAR_DEVERR_STALE,
         oracle.EMPTY: gear.GEAR_DEVERR_EMPTY, oracle.FULL: gear.GEAR_DEVERR_FULL}
    return sum(g for o, g in m.items() if st & o)


class Pair:
    """A GPU table (W=1 rank, R virtual shards) and its oracle twin."""

    def __init__(self, capacity, seq_len, colspecs, R=1, placement=None, removal=0,
                 max_batch=4096, frac_bits=32, mirror=True, alpha=1.0):
        import torch
        self.torch = torch
        self.cols = []
        for c in colspecs:
            pl = placement if placement is not None else c.placement
            self.cols.append(gear.Column(c.name, DT[c.dtype], tuple(c.shape),
                                         gear.GEAR_HOST if pl == "host" else gear.GEAR_DEVICE))
        self.t = gear.Table(capacity, seq_len, self.cols, None, frac_bits=frac_bits, removal=removal,
                            shards_per_rank=R, max_batch=max_batch, alpha=alpha)
        self.R, self.N = R, capacity
        self.Cs = capacity // R
        self.o = oracle.Table(self.Cs, R, frac_bits=frac_bits, removal=removal, alpha=alpha)
        self.rb = self.t.row_bytes
        self.mirror = [np.zeros((capacity, rb), np.uint8) for rb in self.rb] if mirror else None
        self.content = np.full(capacity, -1, np.int64)   # trajectory id held by each slot
        self.next_traj = 0

    def insert(self, shard, prio, device_src=False):
        prio = np.asarray(prio, dtype=np.float64)
        n = prio.size
        traj = np.arange(self.next_traj, self.next_traj + n)
        self.next_traj += n
        rows = [synth.row_bytes_of(c, traj, rb) for c, rb in enumerate(self.rb)]
        srcs = [self.torch.from_numpy(r).cuda() for r in rows] if device_src else rows
        out = np.zeros(n, np.uint64)
        self.t.insert(shard, srcs, prio, out)
        st, oidx = self.o.insert(shard, prio)
        assert st == 0
        assert np.array_equal(out, oidx), "insert slot assignment differs from the oracle"
        for k, g in enumerate(oidx):
            self.content[int(g)] = traj[k]
            if self.mirror is not None:
                for c in range(len(self.rb)):
                    self.mirror[c][int(g)] = rows[c][k]
        return out

    def fill(self, prio_all):
        """Insert prio_all (length N) shard by shard, in batches."""
        for s in range(self.R):
            p = prio_all[s * self.Cs:(s + 1) * self.Cs]
            for k0 in range(0, p.size, 4096):
                self.insert(s, p[k0:k0 + 4096])

    def sample_gpu(self, strategy, B, seed, beta):
        torch = self.torch
        idx = torch.empty(B, dtype=torch.int64, device="cuda")
        w = torch.empty(B, dtype=torch.float32, device="cuda")
        p = torch.empty(B, dtype=torch.float64, device="cuda")
        gen = torch.empty(B, dtype=torch.int32, device="cuda")
        self.t.sample(strategy, B, seed, beta, idx, w, p, gen)
        torch.cuda.synchronize()
        return (idx.cpu().numpy().view(np.uint64), w.cpu().numpy(), p.cpu().numpy(),
                gen.cpu().numpy().view(np.uint32))

    def sample_oracle(self, strategy, B, seed, beta):
        return self.o.sample(ORACLE_STRATEGY[strategy], 1, 0, B, seed, beta)

    def check_sample(self, strategy, B, seed, beta=0.4):
        gi, gw, gp, gg = self.sample_gpu(strategy, B, seed, beta)
        st, oi, ow, op = self.sample_oracle(strategy, B, seed, beta)
        err, _ = self.t.sync()
        if st == oracle.EMPTY:
            assert err & gear.GEAR_DEVERR_EMPTY
            assert np.all(gi == np.uint64(gear.GEAR_IDX_NONE))
            return None
        assert st == 0 and err == 0, (st, err)
        assert np.array_equal(gi, oi), f"indices differ at {np.nonzero(gi != oi)[0][:10]}"
        np.testing.assert_allclose(gw, ow, rtol=1e-6, atol=0)
        assert np.array_equal(gp, op), "probabilities q/T differ"
        assert np.array_equal(gg, self.o.gen[oi.astype(np.int64)])
        return gi

    def collect_gpu(self, idx, col_ids=None):
        torch = self.torch
        col_ids = list(range(len(self.rb))) if col_ids is None else col_ids
        outs = [torch.empty((len(idx), self.rb[c]), dtype=torch.uint8, device="cuda") for c in col_ids]
        d_idx = torch.from_numpy(np.asarray(idx, np.uint64).view(np.int64)).cuda()
        self.t.collect(d_idx, col_ids, outs)
        torch.cuda.synchronize()
        return [o.cpu().numpy() for o in outs]

    def check_collect(self, idx, col_ids=None):
        col_ids = list(range(len(self.rb))) if col_ids is None else col_ids
        got = self.collect_gpu(idx, col_ids)
        for c, g in zip(col_ids, got):
            want = oracle.collect(self.mirror[c], np.asarray(idx, np.uint64))
            assert np.array_equal(g, want), f"column {c} differs"

    def update(self, idx, p, gen=None, f32=False):
        torch = self.torch
        idx = np.asarray(idx, np.uint64)
        p = np.asarray(p, np.float32 if f32 else np.float64)
        d_idx = torch.from_numpy(idx.view(np.int64)).cuda()
        d_p = torch.from_numpy(p).cuda()
        d_g = None if gen is None else torch.from_numpy(np.asarray(gen, np.uint32).view(np.int32)).cuda()
        gear.gear_update_priorities(self.t.handle, len(idx), d_idx, d_p,
                                    gear.GEAR_F32 if f32 else gear.GEAR_F64, d_g)
        ost, ons = self.o.update(idx, p.astype(np.float64), gen)
        err, ns = self.t.sync()
        return ost, ons, err, ns

    # --- split writer API (gear_allocate / in-place rows / gear_commit) -------
    def allocate(self, shard, n):
        torch = self.torch
        out = torch.empty(n, dtype=torch.int64, device="cuda")
        self.t.allocate(shard, n, out)
        torch.cuda.synchronize()
        gids = out.cpu().numpy().view(np.uint64)
        st, oids = self.o.allocate(shard, n)
        err, _ = self.t.sync()
        if st == oracle.FULL:
            assert err & gear.GEAR_DEVERR_FULL, err
            assert np.all(gids == np.uint64(gear.GEAR_IDX_NONE))
            return None
        assert st == 0 and err == 0, (st, err)
        assert np.array_equal(gids, oids), "allocated slots differ from the oracle"
        return gids

    def write_rows(self, ids):
        """Write new trajectories' rows IN PLACE at the allocated slots
        (gear_column_base), device columns with a device scatter, host
        columns through the mapped host pointer."""
        torch = self.torch
        ids = np.asarray(ids, np.uint64)
        traj = np.arange(self.next_traj, self.next_traj + ids.size)
        self.next_traj += ids.size
        for c, rb in enumerate(self.rb):
            rows = synth.row_bytes_of(c, traj, rb)
            base = self.t.column_base(c)
            if self.cols[c].placement == gear.GEAR_DEVICE:
                class _View:
                    __cuda_array_interface__ = {"shape": (self.N, rb), "typestr": "|u1",
                                                "data": (base, False), "version": 3}
                col = torch.as_tensor(_View(), device="cuda")
                col[torch.from_numpy(ids.astype(np.int64)).cuda()] = torch.from_numpy(rows).cuda()
            else:
                col = np.ctypeslib.as_array(ctypes.cast(base, ctypes.POINTER(ctypes.c_uint8)),
                                            shape=(self.N, rb))
                col[ids.astype(np.int64)] = rows
            if self.mirror is not None:
                self.mirror[c][ids.astype(np.int64)] = rows
        torch.cuda.synchronize()
        for k, g in enumerate(ids):
            self.content[int(g)] = traj[k]

    def commit(self, shard, ids, prio):
        torch = self.torch
        ids = np.asarray(ids, np.uint64)
        prio = np.asarray(prio, np.float64)
        self.t.commit(shard, torch.from_numpy(ids.view(np.int64)).cuda(),
                      torch.from_numpy(prio).cuda())
        torch.cuda.synchronize()
        ost = self.o.commit(shard, ids, prio)
        err, _ = self.t.sync()
        assert err == oracle_bits_to_gear(ost), (err, ost)
        return ost

    def check_state(self):
        key, seq, gen = self.t.read_state()
        assert np.array_equal(key, self.o.key)
        assert np.array_equal(seq, self.o.seq)
        assert np.array_equal(gen, self.o.gen)

    def close(self):
        self.t.close()
