// alloc.cu -- NEXT-1: the block allocator on the device.
//
// Each local shard keeps, in device memory, a free-queue cursor (the queue is
// seeded 0..C_s-1 ascending, so the free slots are [next_free, C_s)), the
// ring of committed slots in commit order (`ord`, head + len) and the next
// seq value.  Every writer call is one single-CTA launch that reads and
// advances that state on the stream, so inserts need no host round trip and
// can be captured in a CUDA graph.
//
//  * insert (gear_insert): each row is allocated and committed before the
//    next (reading Q12) -- the slot, ring position and seq of row k have a
//    closed form, so all rows are planned in parallel:
//      F = free slots, L = ring length, C = F + L (slots not ongoing)
//      FIFO removal: row k takes j = k mod C: j < F ? next_free + j
//                    : ord[head + j - F]; it is appended at head + L + k
//      LIFO removal: rows k < F take next_free + k; every later row evicts
//                    the newest, i.e. the previous row (or, with F = 0, the
//                    ring's newest) and reuses its slot and ring position.
//    Several rows can land in one slot / position: the last one wins (the
//    plan marks the winners; gen counts every row that landed).
//  * allocate (gear_allocate): n ongoing slots -- free ones first, then
//    victims popped from the ring's old (FIFO) / new (LIFO) end; key = seq =
//    0 and gen += 1 (reading Q21).  All or nothing (FULL).
//  * commit (gear_commit): in order, each ongoing id of the shard gets seq =
//    seq_ctr++ and key = Q_F(p^alpha) and is appended to the ring.  The first
//    copy of a duplicated id wins (tag pass, like the priority update);
//    entries outside the shard, not ongoing, or with a bad priority are
//    skipped and latched.
#include "common.cuh"

namespace gear {

namespace {

constexpr int kThreads = 1024;

__device__ __forceinline__ uint32_t block_excl_scan(uint32_t x, uint32_t* s_warp,
                                                    uint32_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t incl = x;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, incl, d);
    if (lane >= d) incl += y;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  uint32_t before = 0, all = 0;
  for (int w = 0; w < kThreads / 32; ++w) {
    const uint32_t v = s_warp[w];
    before += w < warp ? v : 0u;
    all += v;
  }
  __syncthreads();
  *total = all;
  return before + incl - x;
}

// Device-side priority check of a whole gear_insert call (all or nothing):
// *bad = 1 (and BAD_PRIORITY latched) if any p is NaN, infinite or negative.
__global__ void __launch_bounds__(kThreads)
    validate_prio_kernel(const double* __restrict__ prio, uint32_t n, uint32_t* bad,
                         uint32_t* err) {
  bool b = false;
  for (uint32_t k = threadIdx.x; k < n; k += kThreads) {
    const double p = prio[k];
    b |= !(p >= 0.0) || isinf(p);
  }
  const int any = __syncthreads_or(b);
  if (threadIdx.x == 0) {
    *bad = any ? 1u : 0u;
    if (any) atomicOr(err, kErrBadPriority);
  }
}

__global__ void __launch_bounds__(kThreads)
    insert_plan_kernel(AllocState* st, uint32_t ls, uint32_t shard, uint64_t Cs, int lifo,
                       uint32_t m, const double* __restrict__ prio, const uint32_t* __restrict__ ord,
                       const uint32_t* abort_flag, InsMeta* __restrict__ meta,
                       OrdRec* __restrict__ ord_recs, uint64_t* __restrict__ out_idx,
                       uint32_t* err) {
  const AllocState a = st[ls];
  const uint64_t F = Cs - a.next_free, L = a.len, C = F + L;
  const uint64_t base = (uint64_t)ls * Cs;
  const bool aborted = abort_flag != nullptr && *abort_flag != 0;  // a bad priority
  if (C == 0 || aborted) {  // every slot is ongoing, or the call is rejected
    for (uint32_t k = threadIdx.x; k < m; k += kThreads) {
      meta[k].local = kIdxNone;
      ord_recs[k].pos = 0xffffffffu;
      out_idx[k] = kIdxNone;
    }
    if (threadIdx.x == 0 && !aborted) atomicOr(err, kErrFull);
    return;
  }
  auto old_ring = [&](uint64_t i) -> uint32_t {  // i-th entry from the oldest
    return ord[base + (a.head + i) % Cs];
  };
  for (uint32_t k = threadIdx.x; k < m; k += kThreads) {
    uint64_t slot, pos;
    bool win_slot, win_pos;
    uint32_t gen_inc = 1;
    if (!lifo) {
      const uint64_t j = k % C;
      slot = j < F ? a.next_free + j : old_ring(j - F);
      pos = (a.head + L + k) % Cs;
      win_slot = (uint64_t)k + C >= m;
      win_pos = (uint64_t)k + Cs >= m;
      gen_inc = (uint32_t)(k / C) + 1;
    } else if (F > 0) {
      const uint64_t kk = k < F ? k : F - 1;
      slot = a.next_free + kk;
      pos = (a.head + L + kk) % Cs;
      win_slot = win_pos = (uint64_t)k + 1 < F || k == m - 1;
      gen_inc = (uint64_t)k + 1 < F ? 1u : (uint32_t)(m - (F - 1));
    } else {  // LIFO, no free slot: every row replaces the newest entry
      slot = old_ring(L - 1);
      pos = (a.head + L - 1) % Cs;
      win_slot = win_pos = k == m - 1;
      gen_inc = m;
    }
    InsMeta im;
    im.local = win_slot ? base + slot : kIdxNone;
    im.seq = a.seq_ctr + k;
    im.gen_inc = gen_inc;
    im.src_row = k;
    im.prio = prio[k];
    meta[k] = im;
    OrdRec orr;
    orr.pos = win_pos ? (uint32_t)(base + pos) : 0xffffffffu;
    orr.slot = (uint32_t)slot;
    ord_recs[k] = orr;
    out_idx[k] = (uint64_t)shard * Cs + slot;
  }
  if (threadIdx.x == 0) {
    AllocState b = a;
    const uint64_t from_free = m < F ? m : F;
    b.next_free = a.next_free + from_free;
    b.seq_ctr = a.seq_ctr + m;
    if (!lifo) {
      const uint64_t evict = m - from_free;  // pops from the old end
      b.head = (uint32_t)((a.head + evict) % Cs);
      b.len = (uint32_t)(L + m - evict);
    } else {
      b.len = (uint32_t)(L + from_free);  // the rest replaced the newest
    }
    st[ls] = b;
  }
}

__global__ void __launch_bounds__(kThreads)
    allocate_kernel(AllocState* st, uint32_t ls, uint32_t shard, uint64_t Cs, int lifo, uint32_t n,
                    const uint32_t* __restrict__ ord, uint64_t* key, uint64_t* seq, uint32_t* gen,
                    TileDirty td, uint64_t* __restrict__ out_idx, uint32_t* err) {
  const AllocState a = st[ls];
  const uint64_t F = Cs - a.next_free, L = a.len;
  const uint64_t base = (uint64_t)ls * Cs;
  if ((uint64_t)n > F + L) {
    for (uint32_t k = threadIdx.x; k < n; k += kThreads) out_idx[k] = kIdxNone;
    if (threadIdx.x == 0) atomicOr(err, kErrFull);
    return;
  }
  for (uint32_t k = threadIdx.x; k < n; k += kThreads) {
    uint64_t slot;
    if (k < F) {
      slot = a.next_free + k;
    } else {
      const uint64_t v = k - F;  // v-th victim: oldest first (FIFO) / newest first (LIFO)
      const uint64_t i = lifo ? L - 1 - v : v;
      slot = ord[base + (a.head + i) % Cs];
    }
    const uint64_t local = base + slot;
    gen[local] += 1;
    key[local] = 0;
    seq[local] = 0;
    mark_tile(td, local);
    out_idx[k] = (uint64_t)shard * Cs + slot;
  }
  if (threadIdx.x == 0) {
    AllocState b = a;
    const uint64_t from_free = n < F ? n : F;
    const uint64_t evict = n - from_free;
    b.next_free = a.next_free + from_free;
    if (!lifo) b.head = (uint32_t)((a.head + evict) % Cs);
    b.len = (uint32_t)(L - evict);
    st[ls] = b;
  }
}

__global__ void __launch_bounds__(kThreads)
    commit_kernel(AllocState* st, uint32_t ls, uint32_t shard, uint64_t Cs, uint32_t n,
                  const uint64_t* __restrict__ idx, const double* __restrict__ prio, Quant qz,
                  uint64_t* key, uint64_t* seq, const uint32_t* __restrict__ gen, uint32_t* ord,
                  unsigned long long* tag, uint64_t* epoch_dev, TileDirty td, uint32_t* err) {
  __shared__ uint32_t s_warp[kThreads / 32];
  __shared__ uint32_t s_err;
  const AllocState a = st[ls];
  const uint64_t epoch = *epoch_dev + 1;  // shares the update's tag epochs
  const uint64_t base = (uint64_t)ls * Cs;
  const uint64_t g0 = (uint64_t)shard * Cs;
  if (threadIdx.x == 0) s_err = 0;
  __syncthreads();
  // Pass 1: the smallest position of every ongoing id claims its slot.
  for (uint32_t k = threadIdx.x; k < n; k += kThreads) {
    const uint64_t g = idx[k];
    if (g < g0 || g >= g0 + Cs) continue;
    const uint64_t local = base + (g - g0);
    if (gen[local] == 0 || seq[local] != 0) continue;
    atomicMax(tag + local, make_tag(epoch, kTagLowMax - k));
  }
  __syncthreads();
  // Pass 2: in order, the valid entries get consecutive seq and ring slots.
  uint32_t done = 0;
  for (uint32_t k0 = 0; k0 < n; k0 += kThreads) {
    const uint32_t k = k0 + threadIdx.x;
    bool ok = false;
    uint64_t local = 0, q = 0;
    uint32_t e = 0;
    if (k < n) {
      const uint64_t g = idx[k];
      if (g < g0 || g >= g0 + Cs) {
        e = kErrIndexRange;
      } else {
        local = base + (g - g0);
        if (gen[local] == 0 || seq[local] != 0 ||
            __ldcg(tag + local) != (make_tag(epoch, kTagLowMax - k)))
          e = kErrStale;
        else if (!quantize(prio[k], qz, &q))
          e = kErrBadPriority;
        else
          ok = true;
      }
    }
    if (e) atomicOr(&s_err, e);
    uint32_t total;
    const uint32_t r = block_excl_scan(ok ? 1u : 0u, s_warp, &total);
    if (ok) {
      const uint64_t rank = done + r;
      seq[local] = a.seq_ctr + rank;
      key[local] = q;
      mark_tile(td, local);
      ord[base + (a.head + a.len + rank) % Cs] = (uint32_t)(local - base);
    }
    done += total;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    AllocState b = a;
    b.seq_ctr = a.seq_ctr + done;
    b.len = (uint32_t)(a.len + done);
    st[ls] = b;
    *epoch_dev = epoch;
    if (s_err) atomicOr(err, s_err);
  }
}

}  // namespace

cudaError_t launch_validate_prio(const double* prio, uint32_t n, uint32_t* bad, uint32_t* err,
                                 cudaStream_t s) {
  count_launch();
  validate_prio_kernel<<<1, kThreads, 0, s>>>(prio, n, bad, err);
  return cudaGetLastError();
}

cudaError_t launch_insert_plan(AllocState* st, uint32_t ls, uint32_t shard, uint64_t Cs, int lifo,
                               uint32_t m, const double* prio, const uint32_t* ord,
                               const uint32_t* abort_flag, InsMeta* meta, OrdRec* ord_recs,
                               uint64_t* out_idx, uint32_t* err, cudaStream_t s) {
  if (m == 0) return cudaSuccess;
  count_launch();
  insert_plan_kernel<<<1, kThreads, 0, s>>>(st, ls, shard, Cs, lifo, m, prio, ord, abort_flag,
                                            meta, ord_recs, out_idx, err);
  return cudaGetLastError();
}

cudaError_t launch_allocate(AllocState* st, uint32_t ls, uint32_t shard, uint64_t Cs, int lifo,
                            uint32_t n, const uint32_t* ord, uint64_t* key, uint64_t* seq,
                            uint32_t* gen, TileDirty td, uint64_t* out_idx, uint32_t* err,
                            cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  count_launch();
  allocate_kernel<<<1, kThreads, 0, s>>>(st, ls, shard, Cs, lifo, n, ord, key, seq, gen, td,
                                         out_idx, err);
  return cudaGetLastError();
}

cudaError_t launch_commit(AllocState* st, uint32_t ls, uint32_t shard, uint64_t Cs, uint32_t n,
                          const uint64_t* idx, const double* prio, Quant qz, uint64_t* key,
                          uint64_t* seq, const uint32_t* gen, uint32_t* ord,
                          unsigned long long* tag, uint64_t* epoch_dev, TileDirty td,
                          uint32_t* err, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  count_launch();
  commit_kernel<<<1, kThreads, 0, s>>>(st, ls, shard, Cs, n, idx, prio, qz, key, seq, gen, ord,
                                       tag, epoch_dev, td, err);
  return cudaGetLastError();
}

}  // namespace gear
