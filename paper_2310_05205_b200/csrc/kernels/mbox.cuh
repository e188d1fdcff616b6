// mbox.cuh -- peer-mailbox exchange over NVLink (see gear_internal.h Mbox).
//
// Producer: plain stores of the payload into every peer's mailbox (CUDA-IPC
// mapped device memory, so each store crosses NVLink), a block barrier, then
// one thread issues a system-scope fence and a release store of the epoch
// into the peer's flag slot for this producer.  Consumer: one thread spins
// with acquire loads on its own mailbox flags until every producer has
// published this epoch (flags only grow), a block barrier, then the block
// reads the payload with L1-bypassing loads.  A spin longer than ~4 s latches
// kErrTimeout and gives up instead of hanging the GPU.
#pragma once

#include "common.cuh"

namespace gear {

__device__ __forceinline__ uint64_t ld_acquire_sys_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_sys_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Spin until flags[0..n) >= epoch.  Returns false on timeout (error latched).
__device__ __forceinline__ bool mbox_wait(const uint64_t* flags, uint32_t n, uint64_t epoch,
                                          uint32_t* err) {
  const uint64_t t0 = global_ns();
  for (uint32_t i = 0; i < n; ++i) {
    while (ld_acquire_sys_u64(flags + i) < epoch) {
      if (global_ns() - t0 > 4000000000ull) {
        atomicOr(err, kErrTimeout);
        return false;
      }
      __nanosleep(64);
    }
  }
  return true;
}

// True once any exchange of this table timed out (the bit stays latched until
// gear_table_sync): the SPMD protocol is broken, so consumers of exchanged
// data write GEAR_IDX_NONE / skip their writes instead of using stale data.
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
    __threadfence_system();
    for (uint32_t r = 0; r < m.W; ++r)
      st_release_sys_u64(mbox_at<uint64_t>(m, r, L.tflag) + b * m.W + m.rank, m.epoch);
    mbox_wait(mbox_at<uint64_t>(m, m.rank, L.tflag) + b * m.W, m.W, m.epoch, err);
  }
  __syncthreads();
  if (mbox_failed(err)) return nullptr;
  return mbox_at<ShardTotals>(m, m.rank, L.totals) + b * m.S;
}

}  // namespace gear
