// update.cu -- K6: priority update (quantise -> route -> last-writer-wins
// scatter).  The paper keeps priorities in the status table
// without a type; gear.h fixes the u64 fixed-point key Q_F(p).
//
// Duplicate ids must resolve deterministically to the LAST entry in (rank,
// position) order.  Racing stores cannot promise that, so the scatter is two
// passes over the concatenated entry list: a tag pass does
// atomicMax(tag[slot], epoch<<24 | k+1) and an apply pass lets only the entry
// whose tag survived write the key.  The 40-bit epoch (one per update call)
// makes the tags of earlier calls smaller, so the tag array never needs
// clearing (make_tag, gear_internal.h); it
// lives in device memory and the kernels advance it themselves, so an update
// captured in a CUDA graph stays correct when the graph is replayed.
//
// A table with a PER exponent alpha != 1 first raises the priorities to alpha
// (alpha_kernel, one f64 per entry); the update kernels then quantise with
// quantize_fixed, so the double-double code stays out of their registers.
#include "mbox.cuh"

namespace gear {

namespace {

constexpr int kThreads = 256;

__global__ void __launch_bounds__(kThreads)
    quantize_kernel(const uint64_t* __restrict__ idx, const void* __restrict__ prio,
                    int prio_is_f64, const uint32_t* __restrict__ gen, uint32_t n,
                    uint64_t n_global, Quant qz, UpdRec* out,
                    uint32_t* err) {
  const uint32_t k = blockIdx.x * kThreads + threadIdx.x;
  if (k >= n) return;
  UpdRec r;
  r.idx = idx[k];
  r.q = 0;
  r.gen = gen ? gen[k] : 0u;
  r.flags = gen ? 2u : 0u;
  const double p = prio_is_f64 ? static_cast<const double*>(prio)[k]
                               : (double)static_cast<const float*>(prio)[k];
  if (r.idx == kIdxNone) {
    // padding entry: ignored
  } else if (r.idx >= n_global) {
    atomicOr(err, kErrIndexRange);
  } else if (!quantize_fixed(p, qz, &r.q)) {
    atomicOr(err, kErrBadPriority);
  } else {
    r.flags |= 1u;
  }
  out[k] = r;
}

// Entry k is applied by the rank owning its id, if the slot holds a committed
// trajectory (gen != 0, seq != 0) and the optional generation matches.
__device__ __forceinline__ bool owned_and_fresh(const UpdRec& r, uint64_t local_begin,
                                                uint64_t local_rows, const uint32_t* gen,
                                                const uint64_t* seq,
                                                uint64_t* local, bool* stale) {
  *stale = false;
  if (!(r.flags & 1u)) return false;
  if (r.idx < local_begin || r.idx >= local_begin + local_rows) return false;
  *local = r.idx - local_begin;
  const uint32_t gcur = gen[*local];
  // never inserted (gen 0) or allocated and not yet committed (seq 0, Q21)
  if (gcur == 0 || seq[*local] == 0 || ((r.flags & 2u) && r.gen != gcur)) {
    *stale = true;
    return false;
  }
  return true;
}

__global__ void __launch_bounds__(kThreads)
    tag_kernel(const UpdRec* __restrict__ recs, uint32_t m, uint64_t local_begin,
               uint64_t local_rows, const uint32_t* __restrict__ gen,
                 const uint64_t* __restrict__ seq, unsigned long long* tag,
               uint64_t* epoch_dev, unsigned long long* n_stale, uint32_t* err) {
  const uint64_t epoch = *epoch_dev + 1;
  const uint32_t k = blockIdx.x * kThreads + threadIdx.x;
  if (k >= m) return;
  const UpdRec r = recs[k];
  uint64_t local;
  bool stale;
  if (owned_and_fresh(r, local_begin, local_rows, gen, seq, &local, &stale)) {
    atomicMax(tag + local, make_tag(epoch, k + 1));
  } else if (stale) {
    atomicAdd(n_stale, 1ull);
    atomicOr(err, kErrStale);
  }
}

__global__ void __launch_bounds__(kThreads)
    apply_kernel(const UpdRec* __restrict__ recs, uint32_t m, uint64_t local_begin,
                 uint64_t local_rows, const uint32_t* __restrict__ gen,
                 const uint64_t* __restrict__ seq,
                 const unsigned long long* __restrict__ tag, const uint64_t* epoch_dev,
                 uint64_t* key, TileDirty td) {
  const uint64_t epoch = *epoch_dev + 1;
  const uint32_t k = blockIdx.x * kThreads + threadIdx.x;
  if (k >= m) return;
  const UpdRec r = recs[k];
  uint64_t local;
  bool stale;
  if (owned_and_fresh(r, local_begin, local_rows, gen, seq, &local, &stale) &&
      tag[local] == (make_tag(epoch, k + 1))) {
    key[local] = r.q;
    mark_tile(td, local);
  }
}

// Single-CTA variant for up to kFusedMax entries: tag pass, block barrier,
// apply pass in one launch.  With `idx != nullptr` the entries are the raw
// (W = 1) inputs and are quantised in place; otherwise `recs` holds the
// all-gathered records of every rank.
constexpr int kFusedThreads = 1024;
constexpr uint32_t kFusedMax = 8192;
constexpr int kFusedPer = kFusedMax / kFusedThreads;

__global__ void __launch_bounds__(kFusedThreads)
    fused_kernel(const uint64_t* __restrict__ idx, const void* __restrict__ prio, int prio_is_f64,
                 const uint32_t* __restrict__ gen_in, const UpdRec* __restrict__ recs, uint32_t m,
                 uint64_t n_global, Quant qz, uint64_t local_begin,
                 uint64_t local_rows, const uint32_t* __restrict__ gen,
                 const uint64_t* __restrict__ seq, unsigned long long* tag,
                 uint64_t* epoch_dev, unsigned long long* n_stale, uint32_t* err, uint64_t* key,
                 TileDirty td) {
  const uint64_t epoch = *epoch_dev + 1;  // device-resident: graph-replayable
  UpdRec r[kFusedPer];
  bool mine[kFusedPer];
  uint64_t loc[kFusedPer];
  uint32_t e = 0, stale = 0;
#pragma unroll
  for (int u = 0; u < kFusedPer; ++u) {
    const uint32_t k = threadIdx.x + u * kFusedThreads;
    mine[u] = false;
    if (k >= m) continue;
    if (idx) {
      r[u].idx = idx[k];
      r[u].gen = gen_in ? gen_in[k] : 0u;
      r[u].flags = gen_in ? 2u : 0u;
      const double p = prio_is_f64 ? static_cast<const double*>(prio)[k]
                                   : (double)static_cast<const float*>(prio)[k];
      if (r[u].idx == kIdxNone) {
      } else if (r[u].idx >= n_global) {
        e |= kErrIndexRange;
      } else if (!quantize_fixed(p, qz, &r[u].q)) {
        e |= kErrBadPriority;
      } else {
        r[u].flags |= 1u;
      }
    } else {
      r[u] = recs[k];
    }
    bool st;
    mine[u] = owned_and_fresh(r[u], local_begin, local_rows, gen, seq, &loc[u], &st);
    stale += st ? 1u : 0u;
    if (mine[u])
      atomicMax(tag + loc[u], make_tag(epoch, k + 1));
  }
  if (stale) {
    atomicAdd(n_stale, (unsigned long long)stale);
    e |= kErrStale;
  }
  if (e) atomicOr(err, e);
  __syncthreads();
#pragma unroll
  for (int u = 0; u < kFusedPer; ++u) {
    const uint32_t k = threadIdx.x + u * kFusedThreads;
    if (mine[u] && __ldcg(tag + loc[u]) ==
                       (make_tag(epoch, k + 1))) {
      key[loc[u]] = r[u].q;
      mark_tile(td, loc[u]);
    }
  }
  __syncthreads();  // every thread has read the epoch before it advances
  if (threadIdx.x == 0) *epoch_dev = epoch;
}

// W > 1, W*n <= kFusedMax: one CTA quantises this rank's n entries, pushes
// the records into every peer's mailbox over NVLink (mbox.cuh), waits for the
// records of all W ranks, then runs the tag / barrier / apply passes over the
// W*n records in (rank, position) order -- the whole collective update in one
// launch, no NCCL call.
__global__ void __launch_bounds__(kFusedThreads)
    xchg_kernel(const uint64_t* __restrict__ idx, const void* __restrict__ prio, int prio_is_f64,
                const uint32_t* __restrict__ gen_in, uint32_t n, uint64_t n_global,
                Quant qz, const __grid_constant__ Mbox mb0,
                uint64_t local_begin, uint64_t local_rows, const uint32_t* __restrict__ gen,
                 const uint64_t* __restrict__ seq,
                unsigned long long* tag, uint64_t* epoch_dev, unsigned long long* n_stale,
                uint32_t* err, uint64_t* key, TileDirty td) {
  const uint64_t epoch = *epoch_dev + 1;  // device-resident tag epoch
  const Mbox mb = mbox_at_next_epoch(mb0);  // device-resident exchange epoch
  const MboxLayout L = mbox_layout(mb.W, mb.S, mb.MB);
  const uint32_t bsel = mbox_buf(mb);
  uint32_t e = 0;
  for (uint32_t k = threadIdx.x; k < n; k += kFusedThreads) {
    UpdRec r;
    r.idx = idx[k];
    r.q = 0;
    r.gen = gen_in ? gen_in[k] : 0u;
    r.flags = gen_in ? 2u : 0u;
    const double p = prio_is_f64 ? static_cast<const double*>(prio)[k]
                                 : (double)static_cast<const float*>(prio)[k];
    if (r.idx == kIdxNone) {
    } else if (r.idx >= n_global) {
      e |= kErrIndexRange;
    } else if (!quantize_fixed(p, qz, &r.q)) {
      e |= kErrBadPriority;
    } else {
      r.flags |= 1u;
    }
    for (uint32_t dst = 0; dst < mb.W; ++dst)
      mbox_at<UpdRec>(mb, dst, L.upd)[((uint64_t)bsel * mb.W + mb.rank) * mb.MB + k] = r;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbox_producer_fence();
    for (uint32_t dst = 0; dst < mb.W; ++dst)
      mbox_publish(mbox_at<uint64_t>(mb, dst, L.uflag) + bsel * mb.W + mb.rank, mb.epoch);
    mbox_wait(mbox_at<uint64_t>(mb, mb.rank, L.uflag) + bsel * mb.W, mb.W, mb.epoch, err);
  }
  __syncthreads();
  const UpdRec* recs = mbox_at<UpdRec>(mb, mb.rank, L.upd) + (uint64_t)bsel * mb.W * mb.MB;
  // a timed-out exchange: apply nothing (peers' records may be stale)
  const uint32_t m = mbox_failed(err) ? 0u : mb.W * n;
  UpdRec r[kFusedPer];
  bool mine[kFusedPer];
  uint64_t loc[kFusedPer];
  uint32_t stale = 0;
#pragma unroll
  for (int u = 0; u < kFusedPer; ++u) {
    const uint32_t k = threadIdx.x + u * kFusedThreads;  // (rank, position) order
    mine[u] = false;
    if (k >= m) continue;
    const uint32_t src = k / n, pos = k - src * n;
    const UpdRec* rp = recs + (uint64_t)src * mb.MB + pos;
    r[u].idx = __ldcg(&rp->idx);
    r[u].q = __ldcg(&rp->q);
    r[u].gen = __ldcg(&rp->gen);
    r[u].flags = __ldcg(&rp->flags);
    bool st;
    mine[u] = owned_and_fresh(r[u], local_begin, local_rows, gen, seq, &loc[u], &st);
    stale += st ? 1u : 0u;
    if (mine[u])
      atomicMax(tag + loc[u], make_tag(epoch, k + 1));
  }
  if (stale) {
    atomicAdd(n_stale, (unsigned long long)stale);
    e |= kErrStale;
  }
  if (e) atomicOr(err, e);
  __syncthreads();
#pragma unroll
  for (int u = 0; u < kFusedPer; ++u) {
    const uint32_t k = threadIdx.x + u * kFusedThreads;
    if (mine[u] && __ldcg(tag + loc[u]) ==
                       (make_tag(epoch, k + 1))) {
      key[loc[u]] = r[u].q;
      mark_tile(td, loc[u]);
    }
  }
  __syncthreads();  // every thread has read the epoch before it advances
  if (threadIdx.x == 0) {
    *epoch_dev = epoch;
    *mb0.epoch_dev = mb.epoch;
  }
}

__global__ void epoch_bump_kernel(uint64_t* epoch_dev) { *epoch_dev += 1; }

}  // namespace

uint32_t update_fused_max() { return kFusedMax; }

cudaError_t launch_update_xchg(const uint64_t* idx, const void* prio, int prio_is_f64,
                               const uint32_t* gen_in, uint32_t n, uint64_t n_global,
                               Quant qz, const Mbox& mb,
                               uint64_t local_begin, uint64_t local_rows, const uint32_t* gen,
                               const uint64_t* seq,
                               unsigned long long* tag, uint64_t* epoch_dev,
                               unsigned long long* n_stale, uint32_t* err, uint64_t* key,
                               TileDirty td, cudaStream_t s) {
  count_launch();
  xchg_kernel<<<1, kFusedThreads, 0, s>>>(idx, prio, prio_is_f64, gen_in, n, n_global, qz, mb,
                                          local_begin, local_rows, gen, seq, tag, epoch_dev,
                                          n_stale, err, key, td);
  return cudaGetLastError();
}

cudaError_t launch_update_fused(const uint64_t* idx, const void* prio, int prio_is_f64,
                                const uint32_t* gen_in, const UpdRec* recs, uint32_t m,
                                uint64_t n_global, Quant qz,
                                uint64_t local_begin, uint64_t local_rows, const uint32_t* gen,
                                const uint64_t* seq,
                                unsigned long long* tag, uint64_t* epoch_dev,
                                unsigned long long* n_stale, uint32_t* err, uint64_t* key,
                                TileDirty td, cudaStream_t s) {
  if (m == 0) return cudaSuccess;
  count_launch();
  fused_kernel<<<1, kFusedThreads, 0, s>>>(idx, prio, prio_is_f64, gen_in, recs, m, n_global,
                                           qz, local_begin, local_rows, gen, seq, tag,
                                           epoch_dev, n_stale, err, key, td);
  return cudaGetLastError();
}

namespace {
__global__ void __launch_bounds__(kThreads)
    alpha_kernel(const void* __restrict__ prio, int prio_is_f64, uint32_t n, double alpha,
                 double* __restrict__ out) {
  const uint32_t k = blockIdx.x * kThreads + threadIdx.x;
  if (k >= n) return;
  const double p = prio_is_f64 ? static_cast<const double*>(prio)[k]
                               : (double)static_cast<const float*>(prio)[k];
  out[k] = apply_alpha(p, alpha);
}
}  // namespace

cudaError_t launch_alpha(const void* prio, int prio_is_f64, uint32_t n, double alpha,
                         double* out, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  count_launch();
  alpha_kernel<<<(n + kThreads - 1) / kThreads, kThreads, 0, s>>>(prio, prio_is_f64, n, alpha,
                                                                 out);
  return cudaGetLastError();
}

cudaError_t launch_update_quantize(const uint64_t* idx, const void* prio, int prio_is_f64,
                                   const uint32_t* gen, uint32_t n, uint64_t n_global,
                                   Quant qz, UpdRec* out,
                                   uint32_t* err, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  count_launch();
  quantize_kernel<<<(n + kThreads - 1) / kThreads, kThreads, 0, s>>>(
      idx, prio, prio_is_f64, gen, n, n_global, qz, out, err);
  return cudaGetLastError();
}

cudaError_t launch_update_tag(const UpdRec* recs, uint32_t m, uint64_t local_begin,
                              uint64_t local_rows, const uint32_t* gen, const uint64_t* seq, unsigned long long* tag,
                              uint64_t* epoch_dev, unsigned long long* n_stale, uint32_t* err,
                              cudaStream_t s) {
  if (m == 0) return cudaSuccess;
  count_launch();
  tag_kernel<<<(m + kThreads - 1) / kThreads, kThreads, 0, s>>>(
      recs, m, local_begin, local_rows, gen, seq, tag, epoch_dev, n_stale, err);
  return cudaGetLastError();
}

cudaError_t launch_update_apply(const UpdRec* recs, uint32_t m, uint64_t local_begin,
                                uint64_t local_rows, const uint32_t* gen,
                                const uint64_t* seq,
                                const unsigned long long* tag, uint64_t* epoch_dev, uint64_t* key,
                                TileDirty td, cudaStream_t s) {
  if (m == 0) return cudaSuccess;
  count_launch(2);
  apply_kernel<<<(m + kThreads - 1) / kThreads, kThreads, 0, s>>>(recs, m, local_begin,
                                                                  local_rows, gen, seq, tag,
                                                                  epoch_dev, key, td);
  epoch_bump_kernel<<<1, 1, 0, s>>>(epoch_dev);  // after every apply block read it
  return cudaGetLastError();
}

}  // namespace gear
