// mbox.cuh -- peer-mailbox exchange over NVLink (see gear_internal.h Mbox).
//
// Producer: plain stores of the payload into every peer's mailbox (CUDA-IPC
// mapped device memory, so each store crosses NVLink), a block barrier, then
// ONE thread issues ONE system-scope fence (fence.acq_rel.sys) followed by
// relaxed system-scope stores of the epoch into each peer's flag slot for
// this producer -- the fence + strong-store release pattern of the PTX memory
// model, covering the payload stores the barrier ordered before the fence.
// Consumer: one thread polls its own mailbox flags with relaxed system-scope
// loads until every producer has published this epoch (flags only grow), then
// ONE fence.acq_rel.sys (acquire pattern), a block barrier, and the block
// reads the payload with L1-bypassing loads.  A spin longer than ~4 s latches
// kErrTimeout and gives up instead of hanging the GPU.
//
// Round 1 used a release store per peer flag and an acquire load per poll:
// each compiles to a MEMBAR.ALL.SYS, which drains the SM's outstanding
// memory operations -- with a zero-copy collect running on the same SMs the
// per-poll / per-flag system barriers cost c3 (4 KB host rows) 6-16% at N=4
// (profiles/r02_multi: mailbox vs NCCL exchange, protocol A/B).
// (The round-1 protocol was deleted after the A/B.)
#pragma once

#include "common.cuh"

#ifndef GEAR_MBOX_SLEEP_NS
#define GEAR_MBOX_SLEEP_NS 64
#endif

namespace gear {

__device__ __forceinline__ uint64_t ld_relaxed_sys_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_relaxed_sys_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Producer, by the one publishing thread after the block barrier that follows
// the payload stores: the release fence ...
__device__ __forceinline__ void mbox_producer_fence() {
  asm volatile("fence.acq_rel.sys;" ::: "memory");
}

// ... then one flag store per peer (after mbox_producer_fence).
__device__ __forceinline__ void mbox_publish(uint64_t* flag, uint64_t epoch) {
  st_relaxed_sys_u64(flag, epoch);
}

// Spin until flags[0..n) >= epoch.  Returns false on timeout (error latched).
__device__ __forceinline__ bool mbox_wait(const uint64_t* flags, uint32_t n, uint64_t epoch,
                                          uint32_t* err) {
  const uint64_t t0 = global_ns();
  for (uint32_t i = 0; i < n; ++i) {
    while (ld_relaxed_sys_u64(flags + i) < epoch) {
      if (global_ns() - t0 > 4000000000ull) {
        atomicOr(err, kErrTimeout);
        return false;
      }
      __nanosleep(GEAR_MBOX_SLEEP_NS);
    }
  }
  asm volatile("fence.acq_rel.sys;" ::: "memory");  // acquire: the relaxed loads saw the flags
  return true;
}

__device__ __forceinline__ bool mbox_failed(const uint32_t* err) {
  return (*(const volatile uint32_t*)err & kErrTimeout) != 0;
}

__device__ __forceinline__ uint32_t mbox_buf(const Mbox& m) { return (uint32_t)(m.epoch & 1); }

// The epochs live in device memory so a captured step stays correct when a
// CUDA graph replays it: a kernel that takes part in exchange e reads
// e = *epoch_dev + 1 on entry, and exactly one party advances the counter
// once every reader of this rank is done (see each kernel).
__device__ __forceinline__ Mbox mbox_at_next_epoch(const Mbox& m) {
  Mbox r = m;
  r.epoch = ld_relaxed_u64(m.epoch_dev) + 1;
  return r;
}

template <class T>
__device__ __forceinline__ T* mbox_at(const Mbox& m, uint32_t r, uint64_t off) {
  return reinterpret_cast<T*>(m.base[r] + off);
}

// Shard totals: every rank writes its R records to all peers, then flags.
// Called by one whole block; returns this rank's view of all S totals in
// its own mailbox (valid after the wait), or nullptr after a timeout.
__device__ __forceinline__ const ShardTotals* mbox_exchange_totals(const Mbox& m,
                                                                   const ShardTotals* local,
                                                                   uint32_t* err) {
  const MboxLayout L = mbox_layout(m.W, m.S, m.MB);
  const uint32_t b = mbox_buf(m);
  const int tid = threadIdx.x;
  for (uint32_t i = tid; i < m.W * m.R; i += blockDim.x) {
    const uint32_t r = i / m.R, ls = i - r * m.R;
    mbox_at<ShardTotals>(m, r, L.totals)[b * m.S + m.rank * m.R + ls] = local[ls];
  }
  __syncthreads();
  if (tid == 0) {
    mbox_producer_fence();
    for (uint32_t r = 0; r < m.W; ++r)
      mbox_publish(mbox_at<uint64_t>(m, r, L.tflag) + b * m.W + m.rank, m.epoch);
    mbox_wait(mbox_at<uint64_t>(m, m.rank, L.tflag) + b * m.W, m.W, m.epoch, err);
  }
  __syncthreads();
  if (mbox_failed(err)) return nullptr;
  return mbox_at<ShardTotals>(m, m.rank, L.totals) + b * m.S;
}

}  // namespace gear
