// collect.cu -- K5: gather the selected rows of several columns into
// contiguous batches; the same engine in scatter mode
// (CollectParams::meta) writes inserted rows into their table slots.
//
// The paper launches "one CUDA kernel per table" that reads pinned host
// memory zero-copy; here ONE launch covers every requested
// column.  The work is a flat list of warp tasks (column, row j, chunk k) of
// `chunk_bytes` each, decoded arithmetically (no work list in memory); a
// persistent grid of warps strides over it.  Index translation (shard = g div
// C_s) is fused: the row's owner rank picks the source base,
// which is local HBM, a peer GPU's HBM mapped through CUDA IPC (NVLink loads)
// or pinned host memory mapped into the device address space (PCIe loads).
// Each lane keeps kUnroll independent 16-byte loads in flight before it
// stores, so a warp has kUnroll*512 B outstanding -- what the PCIe path needs
// to cover its ~1-2 us round trip, and what HBM needs to reach its copy peak.
#include "common.cuh"

namespace gear {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kUnroll = 8;

// Copy `bytes` (a multiple of V) from src to dst with one warp.
template <int V>
__device__ __forceinline__ void warp_copy(uint8_t* __restrict__ dst,
                                          const uint8_t* __restrict__ src, uint64_t bytes,
                                          int lane) {
  if constexpr (V == 16) {
    const uint64_t n = bytes >> 4;
    uint64_t i = lane;
    for (; i + (kUnroll - 1) * 32 < n; i += kUnroll * 32) {
      int4 v[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) v[u] = ld_stream16(src + ((i + u * 32) << 4));
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) st_stream16(dst + ((i + u * 32) << 4), v[u]);
    }
    int4 v[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u)
      if (i + u * 32 < n) v[u] = ld_stream16(src + ((i + u * 32) << 4));
#pragma unroll
    for (int u = 0; u < kUnroll; ++u)
      if (i + u * 32 < n) st_stream16(dst + ((i + u * 32) << 4), v[u]);
  } else {
    using T = typename std::conditional<
        V == 8, uint64_t,
        typename std::conditional<V == 4, uint32_t,
                                  typename std::conditional<V == 2, uint16_t, uint8_t>::type>::type>::type;
    const uint64_t n = bytes / V;
    const T* s = reinterpret_cast<const T*>(src);
    T* d = reinterpret_cast<T*>(dst);
    uint64_t i = lane;
    for (; i + (kUnroll - 1) * 32 < n; i += kUnroll * 32) {
      T v[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) v[u] = s[i + u * 32];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) d[i + u * 32] = v[u];
    }
    for (; i < n; i += 32) d[i] = s[i];
  }
}

__device__ __forceinline__ void copy_dispatch(uint32_t vec, uint8_t* dst, const uint8_t* src,
                                              uint64_t bytes, int lane) {
  switch (vec) {
    case 16: warp_copy<16>(dst, src, bytes, lane); break;
    case 8: warp_copy<8>(dst, src, bytes, lane); break;
    case 4: warp_copy<4>(dst, src, bytes, lane); break;
    case 2: warp_copy<2>(dst, src, bytes, lane); break;
    default: warp_copy<1>(dst, src, bytes, lane); break;
  }
}

// Decode task `task` of a task space (columns `cols[0..ncols)` in order of
// chunk_begin) into (column, row j, chunk k).
__device__ __forceinline__ void decode_task(const CollectParams& p, const uint8_t* cols,
                                            uint32_t ncols, uint64_t task, uint32_t* c_out,
                                            uint64_t* j_out, uint64_t* k_out) {
  uint32_t ci = 0;
  while (ci + 1 < ncols && task >= p.col[cols[ci + 1]].chunk_begin) ++ci;
  const uint32_t c = cols[ci];
  const uint64_t rel = task - p.col[c].chunk_begin;
  const uint64_t jt = rel / p.col[c].chunks_per_row;
  *c_out = c;
  *j_out = jt;
  *k_out = rel - jt * p.col[c].chunks_per_row;
}

// Warps [w_first, w_first + w_count) of every CTA walk the LSU task space.
__device__ __forceinline__ void collect_lsu(const CollectParams& p, uint64_t warp0,
                                            uint64_t nwarps, int lane) {
  for (uint64_t task = warp0; task < p.lsu_total; task += nwarps) {
    uint32_t c;
    uint64_t j, k;
    decode_task(p, p.lsu_cols, p.n_lsu, task, &c, &j, &k);
    const CollectCol& col = p.col[c];
    const uint64_t off = k * (uint64_t)col.chunk;
    const uint64_t rem = col.rb - off;
    const uint64_t bytes = rem < col.chunk ? rem : col.chunk;
    if (p.meta) {  // insert scatter: source row -> table slot
      const uint64_t local = p.meta[j].local;
      if (local == kIdxNone) continue;
      copy_dispatch(col.vec, col.out + local * col.rb + off,
                    col.src[0] + (uint64_t)p.meta[j].src_row * col.rb + off, bytes, lane);
      continue;
    }
    const uint64_t g = __ldg(p.idx + j);
    if (g >= p.n_global) {
      if (lane == 0 && k == 0) atomicOr(p.err, kErrIndexRange);
      continue;
    }
    const uint64_t owner = g / p.rows_per_rank;
    const uint64_t local = g - owner * p.rows_per_rank;
    copy_dispatch(col.vec, col.out + j * col.rb + off, col.src[owner] + local * col.rb + off,
                  bytes, lane);
  }
}

__global__ void __launch_bounds__(kThreads) collect_kernel(const __grid_constant__ CollectParams p) {
  const uint64_t warp0 = (uint64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
  collect_lsu(p, warp0, (uint64_t)gridDim.x * kWarps, threadIdx.x & 31);
}

// The same engine in scatter mode (gear_insert), under its own name so that
// profiles tell the writer's launches from the collector's.
__global__ void __launch_bounds__(kThreads) insert_rows_kernel(const __grid_constant__ CollectParams p) {
  const uint64_t warp0 = (uint64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
  collect_lsu(p, warp0, (uint64_t)gridDim.x * kWarps, threadIdx.x & 31);
}

// ---- TMA bulk-copy variant -------------------------------------------------
// One CTA per SM.  Lane 0 of warp 0 runs a kStages-deep ring of shared-memory
// stages: cp.async.bulk global->shared completes on the stage's mbarrier,
// then cp.async.bulk shared->global writes the stage to the batch and a
// bulk async-group tracks when the stage may be refilled.  A CTA keeps up to
// kStages * stage bytes in flight with no register cost, independent of the
// source (local HBM, a peer's HBM over NVLink, or mapped host memory).  The
// other warps copy the columns whose rows are not 16-byte aligned.
#ifndef GEAR_TMA_THREADS
#define GEAR_TMA_THREADS 128
#endif
constexpr int kTmaThreads = GEAR_TMA_THREADS;  // warp 0: the bulk pipeline; the rest: LSU rows


// Rows the LSU warps of the bulk-copy kernel move instead of its single-lane
// pipeline, with 16-byte loads (8 independent loads in flight per lane):
//  * W > 1, `peer_lsu` columns: the peer-HBM rows (over NVLink), where one slow
//    NVLink chunk would hold up the in-order stages behind it;
//  * `host_lsu` columns (tuning "collect_host_lsu", default: host rows of at
//    most 16 KB): every row of a host-resident column (zero-copy over PCIe)
//    -- c3's 4 KB rows: collect 0.0875 -> 0.0853 ms, 0.86 -> 0.88 of the PCIe
//    probe, e2e -0.7%; the all-LSU kernel gains the same but its full-GPU
//    grid delays the next step's selection (e2e -4.6%, profiles/r02_c3lsu);
//    c4's 449 KB host rows lost 40% e2e at N=4 this way, so large rows keep
//    the bulk pipeline.
__device__ __forceinline__ void collect_peer_rows(const CollectParams& p, uint64_t warp0,
                                                  uint64_t nwarps, int lane) {
  for (uint64_t task = warp0; task < p.tma_total; task += nwarps) {
    uint32_t c;
    uint64_t j, k;
    decode_task(p, p.tma_cols, p.n_tma, task, &c, &j, &k);
    const CollectCol& col = p.col[c];
    if (!col.peer_lsu && !col.host_lsu) continue;
    const uint64_t g = __ldg(p.idx + j);
    if (g >= p.n_global) continue;  // latched by the TMA lane
    const uint64_t owner = g / p.rows_per_rank;
    if (!col.host_lsu && owner == p.self_rank) continue;
    const uint64_t local = g - owner * p.rows_per_rank;
    const uint64_t off = k * (uint64_t)col.chunk;
    const uint64_t rem = col.rb - off;
    const uint64_t bytes = rem < col.chunk ? rem : col.chunk;
    copy_dispatch(16, col.out + j * col.rb + off, col.src[owner] + local * col.rb + off, bytes,
                  lane);
  }
}

// L2 policy of the collect's bulk copies (tuning "collect_evict_first",
// default on at W > 1): the rows stream through once, so they can be marked
// evict-first and not push the selection's working set (keys, CDFs,
// mailboxes) out of L2 while the next step's selection runs next to this
// collect.  Measured (profiles/r02_ef): +7% at c2 TopK and +0.6% at c2 on 4
// GPUs, but -2.4% at c2 on 1 GPU, where the selection is small and hidden.
__device__ __forceinline__ uint64_t collect_l2_policy(bool evict_first) {
  uint64_t pol = 0;
  if (evict_first) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// pol == 0: plain copy
__device__ __forceinline__ void bulk_load_hint(uint32_t stage_addr, const void* src, uint32_t bytes,
                                               uint32_t bar, uint64_t pol) {
  if (pol)
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            stage_addr),
        "l"(src), "r"(bytes), "r"(bar), "l"(pol)
        : "memory");
  else
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            stage_addr),
        "l"(src), "r"(bytes), "r"(bar)
        : "memory");
}

__device__ __forceinline__ void bulk_store_hint(void* dst, uint32_t src, uint32_t bytes, uint64_t pol) {
  if (pol)
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(dst),
                 "r"(src), "r"(bytes), "l"(pol)
                 : "memory");
  else
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src),
                 "r"(bytes)
                 : "memory");
}

// Issue the bulk load of TMA task `task` into stage `s` (mbarrier bars[s]).
// Returns the bytes moved (0 for an invalid id: the barrier is still armed).
__device__ __forceinline__ uint32_t tma_issue_load(const CollectParams& p, uint64_t task,
                                                   uint32_t stage_addr, uint32_t bar,
                                                   uint8_t** dst, uint64_t pol) {
  uint32_t c;
  uint64_t j, k;
  decode_task(p, p.tma_cols, p.n_tma, task, &c, &j, &k);
  const CollectCol& col = p.col[c];
  if (p.meta) {  // insert scatter: source row -> table slot
    const uint64_t local = p.meta[j].local;
    if (local == kIdxNone) {
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
      return 0;
    }
    const uint64_t off = k * (uint64_t)col.chunk;
    const uint64_t rem = col.rb - off;
    const uint32_t bytes = (uint32_t)(rem < col.chunk ? rem : col.chunk);
    *dst = col.out + local * col.rb + off;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
    bulk_load_hint(stage_addr, col.src[0] + (uint64_t)p.meta[j].src_row * col.rb + off, bytes, bar,
                   pol);
    return bytes;
  }
  const uint64_t g = __ldg(p.idx + j);
  if (g >= p.n_global) {
    if (k == 0) atomicOr(p.err, kErrIndexRange);
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
    return 0;
  }
  const uint64_t owner = g / p.rows_per_rank;
  if ((col.peer_lsu && owner != p.self_rank) || col.host_lsu) {  // moved by the LSU warps
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
    return 0;
  }
  const uint64_t local = g - owner * p.rows_per_rank;
  const uint64_t off = k * (uint64_t)col.chunk;
  const uint64_t rem = col.rb - off;
  const uint32_t bytes = (uint32_t)(rem < col.chunk ? rem : col.chunk);
  *dst = col.out + j * col.rb + off;
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
  bulk_load_hint(stage_addr, col.src[owner] + local * col.rb + off, bytes, bar, pol);
  return bytes;
}

// Dynamic variant of the issuing lane's in-order ring (tuning
// "collect_dynamic", default on at W > 1 or with host rows: +6% c2 TopK at
// N=4, +3% c3 at N=1; off for HBM rows at W = 1, where it cost ~1% at c2 --
// profiles/r02_multi): each task is claimed from a
// per-launch counter instead of the static stride, so a CTA that starts late
// -- at W > 1 the next step's selection kernels (a 1024-thread assign CTA,
// spinning mailbox waits) can hold an SM's registers when the collect
// launches -- simply takes fewer tasks instead of finishing last with a full
// share.  The ticket for the next refill is fetched one task ahead, so the
// atomic's round trip stays off the critical path; the last CTA to finish
// re-arms the counter pair (graph-safe).
template <int kStages>
__device__ __forceinline__ void tma_lane_dynamic(const CollectParams& p, uint32_t base,
                                                 uint64_t* bars, uint32_t stage_bytes,
                                                 uint64_t pol) {
  unsigned long long* ctr = p.dyn_ctr;  // [0] next task, [1] CTAs done
  uint8_t* dst[kStages] = {};
  uint32_t nbytes[kStages] = {};
  uint32_t phase = 0;
  int inflight = 0;
  bool more = true;
  uint64_t next = atomicAdd(ctr, 1ull);  // prefetched ticket
  for (int s = 0; s < kStages; ++s) {
    const uint64_t task = next;
    if (task >= p.tma_total) {
      more = false;
      break;
    }
    next = atomicAdd(ctr, 1ull);
    nbytes[s] = tma_issue_load(p, task, base + (uint32_t)s * stage_bytes, smem_u32(&bars[s]),
                               &dst[s], pol);
    ++inflight;
  }
  for (uint64_t n = 0; inflight > 0; ++n) {
    const int s = (int)(n % kStages);
    while (!mbar_try_wait(smem_u32(&bars[s]), (phase >> s) & 1u)) {
    }
    phase ^= 1u << s;
    --inflight;
    if (nbytes[s]) bulk_store_hint(dst[s], base + (uint32_t)s * stage_bytes, nbytes[s], pol);
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    if (n >= 1 && more) {  // refill the previous stage (cyclic order is kept)
      const int sp = (int)((n - 1) % kStages);
      const uint64_t task = next;
      if (task < p.tma_total) {
        next = atomicAdd(ctr, 1ull);
        asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        nbytes[sp] = tma_issue_load(p, task, base + (uint32_t)sp * stage_bytes,
                                    smem_u32(&bars[sp]), &dst[sp], pol);
        ++inflight;
      } else {
        more = false;
      }
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  __threadfence();
  if (atomicAdd(ctr + 1, 1ull) == gridDim.x - 1) {  // every CTA has stopped claiming
    ctr[0] = 0;
    ctr[1] = 0;
  }
}

// Pipeline of the issuing lane, over its tasks n = 0, 1, ... (task id
// blockIdx.x + n * gridDim.x):  loads of tasks n+1 .. n+kStages-1 are in
// flight while task n is stored; the stage of task n-1 is refilled (task
// n-1+kStages) once its store has finished reading shared memory
// (wait_group.read 1: only the store of task n may still be reading).
template <int kStages>
__device__ __forceinline__ void tma_body(const CollectParams& p, uint32_t stage_bytes) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bars[kStages];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp != 0) {
    const uint64_t w0 = (uint64_t)blockIdx.x * (kTmaThreads / 32 - 1) + (warp - 1);
    const uint64_t nw = (uint64_t)gridDim.x * (kTmaThreads / 32 - 1);
    collect_lsu(p, w0, nw, lane);
    if (p.any_peer_lsu) collect_peer_rows(p, w0, nw, lane);
    return;
  }
  if (lane != 0) return;
  for (int s = 0; s < kStages; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[s])) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  const uint64_t first = blockIdx.x, step = gridDim.x;
  const uint64_t ntask = p.tma_total > first ? (p.tma_total - first + step - 1) / step : 0;
  const uint32_t base = smem_u32(smem);
  const uint64_t pol = collect_l2_policy(p.evict_first != 0);
  if (p.dyn_ctr != nullptr) {
    tma_lane_dynamic<kStages>(p, base, bars, stage_bytes, pol);
    return;
  }
  uint8_t* dst[kStages] = {};
  uint32_t nbytes[kStages] = {};
  uint32_t phase = 0;
  for (uint64_t n = 0; n < ntask && n < (uint64_t)kStages; ++n)
    nbytes[n] = tma_issue_load(p, first + n * step, base + (uint32_t)n * stage_bytes,
                               smem_u32(&bars[n]), &dst[n], pol);
  for (uint64_t n = 0; n < ntask; ++n) {
    const int s = (int)(n % kStages);
    while (!mbar_try_wait(smem_u32(&bars[s]), (phase >> s) & 1u)) {
    }
    phase ^= 1u << s;
    if (nbytes[s]) bulk_store_hint(dst[s], base + (uint32_t)s * stage_bytes, nbytes[s], pol);
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    if (n >= 1 && n - 1 + kStages < ntask) {
      const int sp = (int)((n - 1) % kStages);
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      nbytes[sp] = tma_issue_load(p, first + (n - 1 + kStages) * step,
                                  base + (uint32_t)sp * stage_bytes, smem_u32(&bars[sp]), &dst[sp],
                                  pol);
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void __launch_bounds__(kThreads)
    insert_meta_kernel(const InsMeta* __restrict__ meta, uint32_t m,
                       const OrdRec* __restrict__ ord_recs, uint32_t n_ord, Quant qz,
                       uint64_t* key, TileDirty td, uint64_t* seq, uint32_t* gen,
                       uint32_t* ord) {
  const uint32_t k = blockIdx.x * kThreads + threadIdx.x;
  if (k < m && meta[k].local != kIdxNone) {
    const InsMeta r = meta[k];
    uint64_t q = 0;
    quantize(r.prio, qz, &q);  // validated on the host
    key[r.local] = q;
    mark_tile(td, r.local);
    seq[r.local] = r.seq;
    gen[r.local] += r.gen_inc;
  }
  if (k < n_ord && ord_recs[k].pos != 0xffffffffu) ord[ord_recs[k].pos] = ord_recs[k].slot;
}

// Persistent grid: as many CTAs as can be resident at once (no second wave
// whose warps would start late on a static task split), capped by the work.
template <class K>
int grid_for(K kernel, uint64_t tasks) {
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kThreads, 0);
  const uint64_t want = (tasks + kWarps - 1) / kWarps;
  const uint64_t cap = (uint64_t)sms * (per_sm > 0 ? per_sm : 1);
  return (int)(want < cap ? (want > 0 ? want : 1) : cap);
}

template <int kStages>
__global__ void __launch_bounds__(kTmaThreads)
    collect_tma_kernel(const __grid_constant__ CollectParams p, uint32_t stage_bytes) {
  tma_body<kStages>(p, stage_bytes);
}

template <int kStages>
__global__ void __launch_bounds__(kTmaThreads)
    insert_rows_tma_kernel(const __grid_constant__ CollectParams p, uint32_t stage_bytes) {
  tma_body<kStages>(p, stage_bytes);
}

}  // namespace

// kStages stages of tma_chunk bytes per CTA, ctas CTAs per SM (192 KB of
// shared memory per SM either way).
template <int kStages>
cudaError_t launch_tma(const CollectParams& p, int ctas, cudaStream_t s) {
  const uint32_t stage_bytes = p.col[p.tma_cols[0]].chunk;
  const size_t smem = (size_t)kStages * stage_bytes;
  auto kern = p.meta ? insert_rows_tma_kernel<kStages> : collect_tma_kernel<kStages>;
  static size_t configured[2] = {0, 0};
  size_t& conf = configured[p.meta ? 1 : 0];
  if (smem > conf) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    conf = smem;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  count_launch();
  kern<<<sms * ctas, kTmaThreads, smem, s>>>(p, stage_bytes);
  return cudaGetLastError();
}

cudaError_t launch_tma_stages(const CollectParams& p, int ctas, cudaStream_t s) {
  switch (p.tma_stages) {
    case 2: return launch_tma<2>(p, ctas, s);
    case 3: return launch_tma<3>(p, ctas, s);
    case 4: return launch_tma<4>(p, ctas, s);
    case 6: return launch_tma<6>(p, ctas, s);
    default: return launch_tma<8>(p, ctas, s);
  }
}

cudaError_t launch_collect(const CollectParams& p, cudaStream_t s) {
  if (p.lsu_total + p.tma_total == 0) return cudaSuccess;
  if (p.tma_total == 0) {
    count_launch();
    if (p.meta)
      insert_rows_kernel<<<grid_for(insert_rows_kernel, p.lsu_total), kThreads, 0, s>>>(p);
    else
      collect_kernel<<<grid_for(collect_kernel, p.lsu_total), kThreads, 0, s>>>(p);
    return cudaGetLastError();
  }
  const int ctas = (int)p.tma_ctas_per_sm;
  return launch_tma_stages(p, ctas, s);
}

cudaError_t launch_insert_meta(const InsMeta* meta, uint32_t m, const OrdRec* ord_recs,
                               uint32_t n_ord, Quant qz,
                               uint64_t* key, TileDirty td, uint64_t* seq, uint32_t* gen,
                               uint32_t* ord, cudaStream_t s) {
  const uint32_t n = m > n_ord ? m : n_ord;
  if (n == 0) return cudaSuccess;
  count_launch();
  insert_meta_kernel<<<(n + kThreads - 1) / kThreads, kThreads, 0, s>>>(
      meta, m, ord_recs, n_ord, qz, key, td, seq, gen, ord);
  return cudaGetLastError();
}

}  // namespace gear
