"""bench.py -- sampled+collected trajectories/s of the GEAR replay hot path.

One step = the whole hot path on every rank: gear_sample (K1 scan of the
dirty CDF + K2 draw/search + IS weights) -> gear_collect (K5, every column of
the sampled rows into a contiguous batch) -> gear_update_priorities (K6, new
priorities for the sampled ids), for the configuration's strategy.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl reference]

Default workload at N=1: BASELINE.json configs[1] (c2, Decision-Transformer
Atari table: 100K trajectories x 847,080 B, HBM-resident, prioritized B=512
per rank with per-step priority updates).  N>1 (torchrun, one rank per GPU):
the same 100K-trajectory table sharded by id over N GPUs, B=512 per rank
(weak scaling), remote rows read over NVLink by the collect kernel.

Defaults: K = 1000 timed steps, W = 10 warm-up steps.  The headline is the
pipelined step (selection on one stream, collection on another) with the K
steps captured as ONE CUDA graph and replayed once inside the timed region;
the eager pipelined, serial and end-to-end (host buffers) variants, the
roofline of the collect kernel (its launch time taken from the timed replay),
live PCIe / NVLink probes, clocks and the selection-only time are in the same
line; at N > 1 also the other assignment of the global batch (DESIGN.md
Q9 / Q19).  --impl reference times the CPU oracle on the same workload.

Prints ONE JSON line (rank 0).  Time is measured with CUDA events on the
launching stream, barrier + synchronize on both sides, max over ranks.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
os.environ.setdefault("NCCL_DEBUG", "WARN")   # keep stdout to the one JSON line:
os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")  # (WARN still prints the version line)

L2_BYTES = 126 << 20   # B200 L2
METRIC = "sampled+collected trajectories/sec and collect GB/s vs HBM/PCIe roofline, 1/2/4/8 B200"
UNIT = "trajectories/s"
# Fallback peaks when the live probes below cannot run (labelled in the line):
PCIE_H2D_GBS = 55.62     # profiles/r01_probe_2gpu.jsonl: pinned cudaMemcpy H2D, 1 GiB, best of 5
NVLINK_PEER_GBS = 775.27  # profiles/r01_probe_2gpu.jsonl: cudaMemcpyPeer pull, 1 GiB


# dram__bytes_read.sum + dram__bytes_write.sum of one collect launch, from an
# ncu --set full capture of `bench.py --config X` (tools/run_ncu_suite.sh).
TRAFFIC = {
    ("c2_dt_atari", 1, None): ((432.961792 + 384.591872) * 1e6,
                               "profiles/r02s8/collect_tma_full.ncu-rep (one launch, final round-2 build)"),
    ("c3_gato_db1", 1, None): (109.824e3, "profiles/r02s8/collect_tma_c3_full.ncu-rep (one launch; "
                               "DRAM bytes only: the binding PCIe read is not a DRAM counter)"),
}


def probe_h2d_gbs(nbytes=1 << 30, reps=3):
    """Pinned host -> this GPU cudaMemcpy (copy engine), best of reps, GB/s:
    the PCIe denominator of host-resident collects, measured in this run."""
    import torch
    src = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    dst = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    best = 0.0
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        dst.copy_(src, non_blocking=True)
        b.record()
        b.synchronize()
        best = max(best, nbytes / (a.elapsed_time(b) / 1e3) / 1e9)
    del src, dst
    return best


def probe_peer_gbs(local, world, nbytes=1 << 30, reps=3):
    """Every rank pulls nbytes from the next rank's GPU at once (copy engine
    over NVLink), best of reps, GB/s per GPU: the NVLink denominator of
    peer-HBM rows, measured in this run under the same all-pull load."""
    import torch
    import torch.distributed as dist
    peer = (local + 1) % world
    src = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{peer}")
    dst = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{local}")
    dst.copy_(src)  # enables peer access
    torch.cuda.synchronize(peer)
    torch.cuda.synchronize(local)
    best = 0.0
    for _ in range(reps):
        dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        dst.copy_(src, non_blocking=True)
        b.record()
        b.synchronize()
        best = max(best, nbytes / (a.elapsed_time(b) / 1e3) / 1e9)
    del src, dst
    t = torch.tensor([best], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    return float(t.item())


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (copy, read+write bytes)"
    except Exception:
        return 6650.0, "fallback 6.65 TB/s of B200_PROFILING.md (MEASURED_PEAKS.json absent)"


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device, self.rows, self.proc = device, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        if not self.rows:  # a timed region shorter than the sampling period: one query now
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=10).stdout
                for line in out.splitlines():
                    parts = [p.strip() for p in line.split(",")]
                    if len(parts) == 7:
                        self.rows.append(parts)
                self.late = True
            except Exception:
                pass
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows),
                **({"note": "timed region shorter than the 20 ms sampling period: one query "
                            "right after it"} if getattr(self, "late", False) else {})}


# ---------------------------------------------------------------- workload
def scaled_capacity(cfg, n_ranks: int) -> tuple[int, str]:
    """Host-resident tables are scaled to fit this box's RAM: 60% at N=1,
    40% at N>1 (every rank registers every rank's shared host shard)."""
    import synth
    host_rb = sum(synth.row_bytes(cfg, c) for c in cfg.cols if c.placement == "host")
    N = cfg.capacity
    note = ""
    if host_rb:
        mem = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES")
        frac = 0.6 if n_ranks == 1 else 0.4
        frac = float(os.environ.get("GEAR_BENCH_HOST_FRAC", frac))
        fit = int(frac * mem) // host_rb
        if fit < N:
            N = max(n_ranks * 1024, (fit // (n_ranks * 1024)) * n_ranks * 1024)
            note = f"capacity scaled {cfg.capacity} -> {N} to fit {int(frac * 100)}% of {mem >> 30} GiB host RAM"
    N -= N % n_ranks
    return N, note


def _cudart():
    """The CUDA runtime library (for cudaEventRecordWithFlags), or None."""
    import glob
    import torch
    for path in sorted(glob.glob(os.path.join(os.path.dirname(torch.__file__), "lib",
                                              "libcudart*.so*"))) + \
            sorted(glob.glob("/usr/local/cuda/lib64/libcudart.so*")):
        try:
            lib = ctypes.CDLL(path)
            lib.cudaEventRecordWithFlags.restype = ctypes.c_int
            return lib
        except OSError:
            continue
    return None


def build_table(cfg, comm, n_ranks: int, rank: int, capacity: int, stream):
    """Create the config's table and fill this rank's shard through gear_insert
    (rows generated on the GPU by synth.fill_rows, priorities from synth)."""
    import torch
    import synth
    import paper_2310_05205_b200 as gear
    dt = {"u8": gear.GEAR_U8, "i32": gear.GEAR_I32, "f32": gear.GEAR_F32}
    cols = [gear.Column(c.name, dt[c.dtype], tuple(c.shape),
                        gear.GEAR_HOST if c.placement == "host" else gear.GEAR_DEVICE) for c in cfg.cols]
    B = cfg.batch
    t = gear.Table(capacity, cfg.seq_len, cols, comm, max_batch=max(4096, B))
    Cs = capacity // n_ranks
    if cfg.prio == "tasks":
        prio_all = synth.task_weights(capacity, zero_frac=cfg.zero_frac)
    else:
        prio_all = synth.priorities(capacity, seed=synth.PRIO_SEED, zero_frac=cfg.zero_frac)
    prio = prio_all[rank * Cs:(rank + 1) * Cs]
    rows_per = max(1, min(4096, (512 << 20) // max(1, sum(t.row_bytes))))
    stage = [torch.empty((rows_per, rb), dtype=torch.uint8, device="cuda") for rb in t.row_bytes]
    for k0 in range(0, Cs, rows_per):
        m = min(rows_per, Cs - k0)
        for c, rb in enumerate(t.row_bytes):
            synth.fill_rows(stage[c].data_ptr(), m, rb, c, rank * Cs + k0, stream=stream.cuda_stream)
        gear.gear_insert(t.handle, rank, m, stage, prio[k0:k0 + m], None, stream)
    stream.synchronize()
    del stage
    return t, prio_all


def effective_cfg(args):
    """The config with the --strategy override applied (both arms)."""
    import dataclasses
    import synth
    cfg = synth.CONFIGS[args.config]
    if args.strategy:
        cfg = dataclasses.replace(cfg, strategy=args.strategy,
                                  update=cfg.update and args.strategy == "prioritized")
    return cfg


def resolve_assign(args):
    """--assign auto: owner-affine (Q19) when the table has HBM-resident
    columns (local rows stay HBM-bound), contiguous slices (Q9) when every column
    is host-resident (any GPU reads any host row over its own PCIe: nothing to
    gain, and no assignment kernel)."""
    if args.assign != "auto":
        return args.assign
    cols = effective_cfg(args).cols
    return "owner" if any(c.placement == "device" for c in cols) else "contiguous"


def workload_config(cfg, capacity, world, args, cap_note):
    """The `config` object of the JSON line, identical for both arms."""
    import synth
    row_total = sum(synth.row_bytes(cfg, c) for c in cfg.cols)
    payload = cfg.batch * row_total
    return {"workload": cfg.name, "capacity": capacity, "seq_len": cfg.seq_len,
            "row_bytes": row_total, "strategy": cfg.strategy, "batch_per_rank": cfg.batch,
            "global_batch": world * cfg.batch, "update_per_step": cfg.update,
            "table_bytes": capacity * row_total,
            "l2": ("inputs larger than L2: random rows of a %.1f GB table, %.0f MB batch per rank"
                   % (capacity * row_total / 1e9, payload / 1e6)
                   if capacity * row_total > L2_BYTES else
                   "L2-resident table (%.1f MB < %d MB L2), not flushed: a latency case, "
                   "not a bandwidth measurement" % (capacity * row_total / 1e6, L2_BYTES >> 20)),
            "parallelism": f"dp{world} (table sharded by trajectory id, 1 shard per GPU)",
            "assignment": args.assign,
            **({"note": cap_note} if cap_note else {})}


def run_gpu(args):
    import torch
    import torch.distributed as dist
    import synth
    import paper_2310_05205_b200 as gear

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    gear.load()
    comm = gear.comm_from_torch_distributed(local) if world > 1 else None
    cfg = effective_cfg(args)
    capacity, cap_note = scaled_capacity(cfg, world)
    stream = torch.cuda.Stream()
    t, prio_all = build_table(cfg, comm, world, rank, capacity, stream)
    strategy = gear.STRATEGIES[cfg.strategy]
    sflags = gear.GEAR_SAMPLE_OWNER_AFFINE if args.assign == "owner" else 0
    # owner-affine batches are ~95% local: the few peer rows go through the
    # LSU warps (profiles/r01m, r01n: +1.7% at N=4); contiguous slices are
    # (W-1)/W remote: all rows by the bulk pipeline
    head_peer_lsu = int(os.environ.get("GEAR_COLLECT_PEER_LSU", "1" if sflags else "0"))
    if world > 1:
        gear.gear_table_set_tuning(t.handle, "collect_peer_lsu", head_peer_lsu)
    B = cfg.batch
    NB = args.depth   # id buffers: the selection may run NB - 1 steps ahead of the collect
    ncols = len(t.row_bytes)
    col_ids = list(range(ncols))
    row_total = sum(t.row_bytes)
    payload = B * row_total
    host_bytes = B * sum(rb for rb, c in zip(t.row_bytes, cfg.cols) if c.placement == "host")
    dev_bytes = payload - host_bytes

    with torch.cuda.stream(stream):
        idx = torch.empty(B, dtype=torch.int64, device="cuda")
        w = torch.empty(B, dtype=torch.float32, device="cuda")
        outs = [torch.empty((B, rb), dtype=torch.uint8, device="cuda") for rb in t.row_bytes]
        pool = [torch.from_numpy(synth.priorities(B, seed=1000 + k)).cuda() for k in range(16)]
        h_idx = torch.empty(B, dtype=torch.int64, pin_memory=True)
        h_w = torch.empty(B, dtype=torch.float32, pin_memory=True)
        h_prio = [torch.from_numpy(synth.priorities(B, seed=1000 + k)).pin_memory() for k in range(16)]
    # Second stream and idx double buffer for the pipelined step.
    # collection streams: with 2, collect(i) and collect(i+1) may overlap (the
    # next step's rows start streaming while this step's tail drains); each
    # stream has its own output batch
    # --collect-priority high: the collect streams get the higher CUDA stream
    # priority (the block scheduler then prefers the collect's CTAs over the
    # selection kernels that overlap it)
    cprio = -1 if args.collect_priority == "high" else 0
    cstreams = [torch.cuda.Stream(priority=cprio) for _ in range(args.collect_streams)]
    cstream = cstreams[0]
    with torch.cuda.stream(stream):
        outs2 = [outs] + [[torch.empty_like(o) for o in outs] for _ in range(len(cstreams) - 1)]
    with torch.cuda.stream(stream):
        idx2 = [idx] + [torch.empty(B, dtype=torch.int64, device="cuda") for _ in range(NB - 1)]
    ev_sampled = [torch.cuda.Event() for _ in range(NB)]
    ev_collected = [torch.cuda.Event() for _ in range(NB)]

    def step_serial(i, ev):
        """sample -> collect -> update, all on one stream."""
        gear.gear_sample(t.handle, strategy, B, synth.SAMPLE_SEED_BASE + i, cfg.beta, idx, w,
                         None, None, stream, flags=sflags)
        if ev:
            ev[0][i].record(stream)
        gear.gear_collect(t.handle, B, idx, col_ids, outs, stream)
        if ev:
            ev[1][i].record(stream)
        if cfg.update:
            gear.gear_update_priorities(t.handle, B, idx, pool[i % 16], gear.GEAR_F64, None, stream)

    def step_pipe(i, ev):
        """The same three calls; selection (sample + update, which share the
        keys) stays in order on `stream`, collection runs on `cstream`, so
        collect(i) overlaps update(i) and sample(i+1).  idx is double
        buffered: sample(i+2) waits until collect(i) has read idx[i%2]."""
        b = i % NB
        if i >= NB:
            stream.wait_event(ev_collected[b])
        gear.gear_sample(t.handle, strategy, B, synth.SAMPLE_SEED_BASE + i, cfg.beta, idx2[b], w,
                         None, None, stream, flags=sflags)
        ev_sampled[b].record(stream)
        if cfg.update:
            gear.gear_update_priorities(t.handle, B, idx2[b], pool[i % 16], gear.GEAR_F64, None,
                                        stream)
        cs = cstreams[b % len(cstreams)]
        cs.wait_event(ev_sampled[b])
        if ev:
            ev[0][i].record(cs)
        gear.gear_collect(t.handle, B, idx2[b], col_ids, outs2[b % len(cstreams)], cs)
        if ev:
            ev[1][i].record(cs)
        ev_collected[b].record(cs)

    def barrier():
        stream.synchronize()
        for cs in cstreams:
            cs.synchronize()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    def timed(step_fn):
        for i in range(args.warmup):
            step_fn(i, None)
        barrier()
        err, _ = t.sync()
        assert err == 0, f"device error bits {err} during warm-up"
        ev = tuple([torch.cuda.Event(enable_timing=True) for _ in range(args.steps)] for _ in range(2))
        clocks = ClockSampler(local)
        clocks.start()
        l0 = gear.gear_kernel_launches()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        e0.record(stream)
        for cs in cstreams:
            cs.wait_event(e0)
        for i in range(args.steps):
            step_fn(i, ev)
        for cs in cstreams:
            stream.wait_stream(cs)
        e1.record(stream)
        barrier()
        launches = gear.gear_kernel_launches() - l0
        clk = clocks.stop()
        err, _ = t.sync()
        assert err == 0, f"device error bits {err} in the timed region"
        coll = float(np.mean([a.elapsed_time(b) for a, b in zip(ev[0], ev[1])]))
        # per-step distribution: intervals between consecutive collect ends
        iv = [ev[1][i - 1].elapsed_time(ev[1][i]) for i in range(1, args.steps)]
        pct = ({f"p{q}": float(np.percentile(iv, q)) for q in (10, 50, 90)} if iv else {})
        timed.percentiles = pct
        return e0.elapsed_time(e1), coll, launches, clk

    def timed_graph(sflags, peer_lsu):
        """The pipelined step captured as ONE CUDA graph of S consecutive steps
        (S = K when K <= 2000: the collect-stream span then covers the whole timed region): the draw key comes from the table's device seed
        counter and the update epoch, the peer-mailbox epochs and the CDF
        parity are device-resident, so each replay performs S new, different
        (collective) steps.  K/S replays are timed.  Two events (external
        event nodes) on the collect stream, before the first and after the
        last collect of the captured steps, time the collect stream's busy
        span inside the timed replay itself; span / S is the collect's
        average launch duration INCLUDING the gaps between consecutive
        collects (an upper bound of the kernel time, so the roofline fraction
        is a lower bound) and can never exceed the time per step.  (Events
        around every collect cost ~6 us per step in the graph: not used.)"""
        S = next(d for d in range(min(args.steps, 2000), 0, -1) if args.steps % d == 0)
        gear.gear_table_set_tuning(t.handle, "device_seed", synth.SAMPLE_SEED_BASE + 100000)
        if world > 1:
            gear.gear_table_set_tuning(t.handle, "collect_peer_lsu", peer_lsu)
        gev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        for a in gev:  # create the events before capture
            a.record(stream)
        cudart = _cudart()

        def rec(ev, st):  # an external event node: keeps its timing inside the graph
            if cudart is None or cudart.cudaEventRecordWithFlags(
                    ctypes.c_void_p(ev.cuda_event), ctypes.c_void_p(st.cuda_stream), 1) != 0:
                raise RuntimeError("cudaEventRecordWithFlags(External) failed")

        def gstep(i, timing=False):
            b = i % NB
            if i >= NB:
                stream.wait_event(ev_collected[b])
            gear.gear_sample(t.handle, strategy, B, 0, cfg.beta, idx2[b], w, None, None, stream,
                             flags=sflags | gear.GEAR_SAMPLE_DEVICE_SEED)
            ev_sampled[b].record(stream)
            if cfg.update:
                gear.gear_update_priorities(t.handle, B, idx2[b], pool[i % 16], gear.GEAR_F64, None,
                                            stream)
            cs = cstreams[b % len(cstreams)]
            cs.wait_event(ev_sampled[b])
            if timing and i == 0:
                rec(gev[0], cs)
            gear.gear_collect(t.handle, B, idx2[b], col_ids, outs2[b % len(cstreams)], cs)
            if timing and i == S - 1:
                for c2 in cstreams:
                    if c2 is not cs:
                        cs.wait_stream(c2)
                rec(gev[1], cs)
            ev_collected[b].record(cs)

        for i in range(args.warmup):
            gstep(i)
        barrier()
        timing = cudart is not None
        g = torch.cuda.CUDAGraph()
        l0 = gear.gear_kernel_launches()
        with torch.cuda.graph(g, stream=stream, capture_error_mode="thread_local"):
            for i in range(S):
                gstep(i, timing=timing)
            for cs in cstreams:
                stream.wait_stream(cs)
        per_graph = gear.gear_kernel_launches() - l0
        barrier()
        clocks = ClockSampler(local)
        with torch.cuda.stream(stream):  # replay() launches on the current stream
            g.replay()  # warm replay
            barrier()
            clocks.start()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            barrier()
            e0.record(stream)
            for _ in range(args.steps // S):
                g.replay()
            e1.record(stream)
        barrier()
        clk = clocks.stop()
        err, _ = t.sync()
        assert err == 0, f"device error bits {err} in the graph replays"
        coll = None
        if timing:
            coll = gev[0].elapsed_time(gev[1]) / S
        return e0.elapsed_time(e1), coll, per_graph * (args.steps // S), S, clk

    def selection_only():
        """Diagnostic: K steps of the selection alone (sample + update, eager,
        one stream, no collect), device time per step -- what the pipelined
        step has to hide behind each collect."""
        for i in range(args.warmup):
            gear.gear_sample(t.handle, strategy, B, synth.SAMPLE_SEED_BASE + i, cfg.beta, idx, w,
                             None, None, stream, flags=sflags)
        barrier()
        a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for i in range(args.steps):
            gear.gear_sample(t.handle, strategy, B, synth.SAMPLE_SEED_BASE + i, cfg.beta, idx, w,
                             None, None, stream, flags=sflags)
            if cfg.update:
                gear.gear_update_priorities(t.handle, B, idx, pool[i % 16], gear.GEAR_F64, None,
                                            stream)
        z.record(stream)
        barrier()
        err, _ = t.sync()
        assert err == 0, f"device error bits {err} in the selection-only run"
        total = a.elapsed_time(z) / args.steps
        # the sample call alone (no update: the CDF stays clean after the first)
        a.record(stream)
        for i in range(args.steps):
            gear.gear_sample(t.handle, strategy, B, synth.SAMPLE_SEED_BASE + i, cfg.beta, idx, w,
                             None, None, stream, flags=sflags)
        z.record(stream)
        barrier()
        selection_only.sample_ms = a.elapsed_time(z) / args.steps
        return total

    sel_only_ms = selection_only()
    sel_sample_ms = selection_only.sample_ms
    ms, coll_ms_p, launches, clk = timed(step_pipe)
    coll_src = "eager pipelined run (events on the collect stream around each launch)"
    step_pct = dict(timed.percentiles)
    ms_serial, coll_ms_s, _, clk_s = timed(step_serial)
    graph = None
    assignments = None
    if args.graph:
        own_flags = gear.GEAR_SAMPLE_OWNER_AFFINE if args.assign == "owner" else 0
        ms_g, coll_g, launches_g, S_g, clk_g = timed_graph(own_flags, head_peer_lsu)
        graph = {"value": world * B * args.steps / (ms_g / 1e3), "ms_per_step": ms_g / args.steps,
                 "steps_per_graph": S_g, "gpu_launches": launches_g}
        if world > 1:
            # the other assignment of the same global batch, same K steps
            # (Q9 contiguous slices vs Q19 owner-affine)
            alt = "contiguous" if own_flags else "owner"
            ms_a, coll_a, _, _, _ = timed_graph(0 if own_flags else gear.GEAR_SAMPLE_OWNER_AFFINE,
                                                0 if own_flags else 1)
            ta = torch.tensor([ms_a, coll_a or 0.0], device="cuda")
            dist.all_reduce(ta, op=dist.ReduceOp.MAX)
            assignments = {alt: {"value": world * B * args.steps / (float(ta[0]) / 1e3),
                                 "ms_per_step": float(ta[0]) / args.steps,
                                 "collect_avg_ms": float(ta[1]),
                                 "note": "same K steps, graph replay, max over ranks"}}
            gear.gear_table_set_tuning(t.handle, "collect_peer_lsu", head_peer_lsu)
        if ms_g < ms:  # the graph-replayed pipelined step is the headline when faster
            graph["eager_pipelined"] = {"value": world * B * args.steps / (ms / 1e3),
                                        "ms_per_step": ms / args.steps,
                                        "collect_avg_ms": coll_ms_p}
            ms, launches, clk = ms_g, launches_g, clk_g
            if coll_g:
                # the headline's own collect launches: busy span of the collect
                # stream in the last timed replay / its S collects
                assert coll_g <= ms_g / args.steps * 1.0001, (coll_g, ms_g)
                coll_ms_p = coll_g
                coll_src = ("the timed graph replay itself: collect-stream span from before the "
                            "first to after the last of its %d collects (external event nodes) / "
                            "%d -- includes the gaps between collects, so frac is a lower bound"
                            % (S_g, S_g))

    # End-to-end through the C-ABI with HOST buffers, pipelined like the device
    # step.  Every step: gear_sample writes the IS weights straight to pinned
    # host memory (in place) and the ids to HBM, from where a third stream
    # copies them to pinned host memory for the host (a copy on the selection
    # stream delayed every rank's mailbox exchanges: N=4 e2e 9.6 M -> 13.5 M
    # traj/s without it); gear_update_priorities reads
    # that step's f64 priorities from pinned host memory (in place, over PCIe);
    # gear_collect (collect stream) gathers the rows into HBM.  The host
    # consumes every step's ids and weights LAG steps behind (waits for
    # sample(i-LAG) and reads its host buffers) while later steps run.
    barrier()
    LAG = 2                       # the host reads step i-LAG while steps i-LAG+1..i run
    NH = 2 * LAG                  # host buffers
    h_idx2 = [h_idx] + [torch.empty(B, dtype=torch.int64, pin_memory=True) for _ in range(NH - 1)]
    h_w2 = [h_w] + [torch.empty(B, dtype=torch.float32, pin_memory=True) for _ in range(NH - 1)]
    ev_hs = [torch.cuda.Event() for _ in range(NH)]
    xstream = torch.cuda.Stream()   # the ids' D2H copy: off the selection / collect streams
    ev_copied = [torch.cuda.Event() for _ in range(NB)]
    np_idx2 = [x.numpy() for x in h_idx2]   # host views of the pinned buffers
    np_w2 = [x.numpy() for x in h_w2]
    dw2 = [torch.empty(B, dtype=torch.float32, device="cuda") for _ in range(NB)]
    consumed = 0.0

    def step_e2e(i):
        b, hb = i % NB, i % NH
        if i >= NB:
            stream.wait_event(ev_collected[b])   # collect(i-NB) has read idx2[b]
            stream.wait_event(ev_copied[b])      # and so has its host copy
        gear.gear_sample(t.handle, strategy, B, synth.SAMPLE_SEED_BASE + 7919 + i, cfg.beta,
                         idx2[b], h_w2[hb] if args.e2e_weights == "host" else dw2[b], None, None,
                         stream, flags=sflags)
        ev_sampled[b].record(stream)
        xstream.wait_event(ev_sampled[b])
        with torch.cuda.stream(xstream):
            h_idx2[hb].copy_(idx2[b], non_blocking=True)
            if args.e2e_weights == "device":
                h_w2[hb].copy_(dw2[b], non_blocking=True)
        ev_copied[b].record(xstream)
        ev_hs[hb].record(xstream)
        if cfg.update:
            gear.gear_update_priorities(t.handle, B, idx2[b], h_prio[i % 16], gear.GEAR_F64,
                                        None, stream)
        cs = cstreams[b % len(cstreams)]
        cs.wait_event(ev_sampled[b])
        gear.gear_collect(t.handle, B, idx2[b], col_ids, outs2[b % len(cstreams)], cs)
        ev_collected[b].record(cs)

    for i in range(args.warmup):
        step_e2e(i)
    barrier()
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record(stream)
    for cs in cstreams:
        cs.wait_event(e2)
    for i in range(args.steps):
        step_e2e(i)
        if i >= LAG:   # the host reads step i-LAG's result while later steps run
            hb = (i - LAG) % NH
            ev_hs[hb].synchronize()
            consumed += float(np_w2[hb][0]) + float(np_idx2[hb][B - 1])
    for i in range(max(0, args.steps - LAG), args.steps):
        ev_hs[i % NH].synchronize()
        consumed += float(np_w2[i % NH][0]) + float(np_idx2[i % NH][B - 1])
    for cs in cstreams + [xstream]:
        stream.wait_stream(cs)
    e3.record(stream)
    barrier()
    assert consumed == consumed   # the host did read the results
    e2e_ms = e2.elapsed_time(e3)
    e2e_h2d = 8 * B if cfg.update else 0    # f64 priorities
    e2e_d2h = 12 * B                         # u64 ids + f32 weights

    times = torch.tensor([ms, e2e_ms, coll_ms_p, ms_serial, coll_ms_s, sel_only_ms, sel_sample_ms],
                         device="cuda")
    if world > 1:
        dist.all_reduce(times, op=dist.ReduceOp.MAX)
    ms, e2e_ms, coll_avg, ms_serial, coll_serial, sel_only_ms, sel_sample_ms = (float(x) for x in times.cpu())

    traj = world * B * args.steps
    value = traj / (ms / 1e3)
    hbm_peak, hbm_src = _peaks()
    # Algorithmic bytes of one collect launch: every
    # payload byte is read once from its source (local HBM, a peer's HBM over
    # NVLink, or host memory over this GPU's PCIe) and written once to local
    # HBM.  The remote fraction is measured on the step's sampled ids.
    Cl = capacity // world
    own = (idx2[(args.steps - 1) % NB].cpu().numpy().astype(np.uint64) // np.uint64(Cl))
    f_remote = torch.tensor([float(np.mean(own != rank))], device="cuda")
    if world > 1:
        dist.all_reduce(f_remote, op=dist.ReduceOp.MAX)
    f_remote = float(f_remote.item())
    remote = dev_bytes * f_remote
    # live probes of the PCIe / NVLink denominators (this box, this run)
    pcie_gbs, pcie_src = PCIE_H2D_GBS, "constant: pinned H2D cudaMemcpy probe of round 1 (profiles/r01_probe_2gpu.jsonl)"
    nvl_gbs, nvl_src = NVLINK_PEER_GBS, "constant: cudaMemcpyPeer pull probe of round 1 (profiles/r01_probe_2gpu.jsonl)"
    barrier()
    seq_ceiling = None
    if host_bytes > 0:
        try:
            pcie_gbs = probe_h2d_gbs()
            pcie_src = "measured in this run: pinned host -> GPU cudaMemcpy of 1 GiB, best of 3"
        except Exception as e:  # noqa: BLE001
            pcie_src += f" (live probe failed: {e!r})"
        # context: the same collect kernel on its best-case access pattern (B
        # consecutive rows of this rank's shard: sequential host reads), what
        # SM-initiated zero-copy reads reach on this box
        if dev_bytes == 0:
            seq = torch.arange(rank * (capacity // world), rank * (capacity // world) + B,
                               dtype=torch.int64, device="cuda")
            for _ in range(3):
                gear.gear_collect(t.handle, B, seq, col_ids, outs, stream)
            a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(20):
                gear.gear_collect(t.handle, B, seq, col_ids, outs, stream)
            z.record(stream)
            stream.synchronize()
            seq_ceiling = host_bytes / (a.elapsed_time(z) / 20 / 1e3) / 1e9
    if world > 1 and remote > 0:
        try:
            nvl_gbs = probe_peer_gbs(local, world)
            nvl_src = ("measured in this run: every rank pulls 1 GiB from the next GPU at once "
                       "(cudaMemcpyPeer), best of 3, min over ranks")
        except Exception as e:  # noqa: BLE001
            nvl_src += f" (live probe failed: {e!r})"
    t_ideal = {"hbm": (2 * dev_bytes - remote) / (hbm_peak * 1e9),
               "nvlink": remote / (nvl_gbs * 1e9),
               "pcie": host_bytes / (pcie_gbs * 1e9)}
    bound = max(t_ideal, key=t_ideal.get)
    alg = {"hbm": 2 * dev_bytes - remote, "nvlink": remote, "pcie": host_bytes}[bound]
    peak = {"hbm": hbm_peak, "nvlink": nvl_gbs, "pcie": pcie_gbs}[bound]
    roof = {"bound": bound, "achieved": alg / (coll_avg / 1e3) / 1e9, "peak": peak, "unit": "GB/s",
            "peak_source": {"hbm": hbm_src, "nvlink": nvl_src, "pcie": pcie_src}[bound]}
    roof["frac"] = roof["achieved"] / roof["peak"]
    roof["probes"] = {"pcie_h2d_GBps": pcie_gbs, "pcie_source": pcie_src,
                      "nvlink_pull_GBps": nvl_gbs, "nvlink_source": nvl_src}
    if seq_ceiling and bound == "pcie":
        roof["sequential_rows_GBps"] = seq_ceiling
        roof["frac_of_sequential"] = roof["achieved"] / seq_ceiling
        roof["sequential_note"] = ("context, not the peak: the same collect kernel gathering B "
                                   "consecutive rows (sequential host reads), 20 launches")
    if roof["frac"] < 0.2:  # e.g. c1: a few hundred KB per launch
        roof["note"] = ("latency-bound: %.0f KB per collect launch, far below what saturates %s"
                        % (alg / 1e3, bound.upper()))
    roof["kernel"] = "collect_tma_kernel" if max(t.row_bytes) >= 4096 else "collect_kernel"
    roof["avg_launch_ms"] = coll_avg
    roof["launch_timing"] = coll_src
    roof["algorithmic_bytes_per_launch"] = alg
    roof["remote_fraction"] = f_remote
    roof["traffic"] = args.traffic
    roof["traffic_source"] = ("--traffic (dram bytes of one collect launch, ncu --set full)"
                              if args.traffic is not None else "not captured for this config")
    key = (cfg.name, world, args.strategy)
    if args.traffic is None and key in TRAFFIC:
        # ncu cannot run inside the timed bench: a CONSTANT from the named
        # capture of this config (same kernel source), not measured in this run
        roof["traffic"], src = TRAFFIC[key]
        roof["traffic_source"] = "constant from " + src
    # The whole step against the same bound: the step's algorithmic bytes of
    # the binding resource over the (headline) time per step.
    roof["step_achieved"] = alg / (ms / args.steps / 1e3) / 1e9
    roof["step_frac"] = roof["step_achieved"] / roof["peak"]

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic (seeded splitmix64 row bytes, lognormal priorities)",
        "config": workload_config(cfg, capacity, world, args, cap_note),
        "collect_gbps": payload / (coll_avg / 1e3) / 1e9,
        "step": ("pipelined: collect(i) on a 2nd stream overlaps update(i) + sample(i+1)"
                 + ("; CUDA-graph replay" if graph and "eager_pipelined" in graph else "")),
        **({"graph": graph} if graph else {}),
        **({"assignments": {args.assign: {"value": value, "ms_per_step": ms / args.steps,
                                          "note": "headline"}, **assignments}}
           if assignments else {}),
        "serial": {"value": traj / (ms_serial / 1e3), "ms_per_step": ms_serial / args.steps,
                   "collect_avg_ms": coll_serial,
                   "note": "sample -> collect -> update on one stream, same K steps"},
        "step_ms_percentiles": {**step_pct, "from": ("eager pipelined run, rank 0: intervals "
                                                     "between consecutive collect completions")},
        "selection": {"only_ms_per_step": sel_only_ms, "sample_only_ms": sel_sample_ms,
                      "note": ("sample (+ update) alone, eager, one stream, K steps, max over ranks: "
                               "the pipelined step hides it behind each collect")},
        "roofline": roof,
        "e2e": {"value": traj / (e2e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": e2e_h2d,
                "d2h_bytes_per_step": e2e_d2h,
                "path": ("C-ABI; priorities from pinned host memory, ids and IS weights to "
                         "pinned host memory, batch in HBM; pipelined (collect on a 2nd stream), "
                         "the host reads every step's ids and weights two steps behind")},
        "gpu_launches": int(launches),
        "clocks": clk,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg, capacity, prio_all, budget_s=args.cpu_budget)
    if rank == 0:
        print(json.dumps(line), flush=True)
    t.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


# ---------------------------------------------------------------- CPU oracle
def cpu_baseline(cfg, capacity, prio_all, budget_s=15.0, max_steps=1000):
    """The oracle (oracle/, single thread) timed as it stands on this host: the
    same step (sample + collect of every column + update) on the same keys;
    row bytes come from a host mirror of M rows (row g read from g mod M) so
    the copy pattern is the same without a 2nd copy of the table."""
    import oracle
    import synth
    oracle.build()
    B = cfg.batch
    row_total = sum(synth.row_bytes(cfg, c) for c in cfg.cols)
    rbs = [synth.row_bytes(cfg, c) for c in cfg.cols]
    M = max(1, min(capacity, (2 << 30) // row_total))    # <= 2 GiB mirror (>> LLC)
    mirror = [np.zeros((M, rb), np.uint8) for rb in rbs]
    for c, rb in enumerate(rbs):
        for k0 in range(0, M, 256):
            mirror[c][k0:k0 + 256] = synth.row_bytes_of(c, np.arange(k0, min(M, k0 + 256)), rb)
    o = oracle.Table(capacity, 1)
    for k0 in range(0, capacity, 1 << 20):
        o.insert(0, prio_all[k0:k0 + (1 << 20)])
    strat = {"prioritized": oracle.PRIORITIZED, "weighted": oracle.WEIGHTED, "uniform": oracle.UNIFORM,
             "fifo": oracle.FIFO, "lifo": oracle.LIFO, "topk": oracle.TOPK}[cfg.strategy]
    steps = 0
    t0 = time.perf_counter()
    while True:
        st, idx, w, p = o.sample(strat, 1, 0, B, synth.SAMPLE_SEED_BASE + steps, cfg.beta)
        src = (idx % np.uint64(M)).astype(np.uint64)
        for c in range(len(rbs)):
            oracle.collect(mirror[c], src)
        if cfg.update:
            o.update(idx, synth.priorities(B, seed=1000 + steps % 16))
        steps += 1
        el = time.perf_counter() - t0
        if el >= budget_s or steps >= max_steps:
            break
    return {"value": steps * B / el, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"{steps} steps of {cfg.name} (B={B}, N={capacity} keys; rows from a "
                      f"{M}-row host mirror, row g <- g mod {M}), {el:.1f} s, single thread",
            "cpu": _cpu_model()}


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip() + f" ({os.cpu_count()} cores)"
    except Exception:
        pass
    return f"{os.cpu_count()} cores"


def run_reference(args):
    """--impl reference: the oracle as it stands, on rank 0's host cores."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    import synth
    cfg = effective_cfg(args)
    capacity, note = scaled_capacity(cfg, world)
    if cfg.prio == "tasks":
        prio_all = synth.task_weights(capacity, zero_frac=cfg.zero_frac)
    else:
        prio_all = synth.priorities(capacity, seed=synth.PRIO_SEED, zero_frac=cfg.zero_frac)
    steps_total = args.steps + args.warmup
    cb = cpu_baseline(cfg, capacity, prio_all, budget_s=args.cpu_budget, max_steps=max(steps_total, 1))
    line = {
        "impl": "reference", "metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": workload_config(cfg, capacity, world, args, note),
        "cpu_baseline": cb,
        "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--strategy", default=None,
                    choices=["fifo", "lifo", "uniform", "weighted", "prioritized", "topk"],
                    help="override the config's strategy")
    ap.add_argument("--collect-streams", type=int, default=1, choices=[1, 2],
                    help="2: consecutive collects on alternating streams may overlap")
    ap.add_argument("--depth", type=int, default=2,
                    help="pipeline depth: id buffers, the selection runs up to depth-1 steps ahead")
    ap.add_argument("--e2e-weights", default="host", choices=["host", "device"],
                    help="e2e: the sample kernel writes the IS weights to pinned host memory in "
                         "place (host) or to HBM, copied with the ids (device)")
    ap.add_argument("--collect-priority", default="normal", choices=["normal", "high"],
                    help="CUDA stream priority of the collect streams")
    ap.add_argument("--graph", type=int, default=1,
                    help="also time the pipelined step captured as a CUDA graph")
    ap.add_argument("--assign", default="auto", choices=["auto", "owner", "contiguous"],
                    help="owner-affine (DESIGN.md Q19) or contiguous rank slices of the global "
                         "batch; auto: owner-affine when the table has HBM-resident columns, "
                         "contiguous when every column is host-resident (every GPU reads any "
                         "host row over its own PCIe: no locality to gain, no assignment kernel)")
    ap.add_argument("--impl", default="gear", choices=["gear", "reference"])
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--traffic", type=float, default=None,
                    help="dram bytes per collect launch from an ncu --set full capture")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    args.assign = resolve_assign(args)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
