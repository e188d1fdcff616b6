// fifo.cu -- K4: decentralised FIFO/LIFO selection.
//
// "all servers can perform a local scan to generate k samples before the
// global gathering operation, which can significantly reduce the
// communication overhead from O(n) to O(mk)".  Each shard keeps its committed
// slots in commit order in a ring (`ord`, maintained by the device-side
// allocator, kernels/alloc.cu), so
// seq is increasing along the ring.  Local step: one CTA per local shard
// walks the ring from the oldest (FIFO) or newest (LIFO) end and compacts the
// first K = W*B selectable slots (key > 0) with a block-wide ballot scan,
// stopping as soon as it has K.  After the candidates of all S shards are
// all-gathered, every rank runs the same merge: a candidate's global position
// is its position in its own (sorted) list plus, for every other list, the
// number of entries that order before it under (seq, shard) -- a binary
// search per list.  Rank r keeps positions [r*B, (r+1)*B).
#include "mbox.cuh"

namespace gear {

namespace {

constexpr int kLocalThreads = 1024;
constexpr int kMergeThreads = 256;

__global__ void __launch_bounds__(kLocalThreads)
    fifo_local_kernel(const uint64_t* __restrict__ key, const uint64_t* __restrict__ seq,
                      const uint32_t* __restrict__ ord, const AllocState* __restrict__ alloc,
                      uint64_t shard_cap, uint32_t first_shard, uint32_t K, int lifo,
                      Cand* __restrict__ cand_out, ShardTotals* __restrict__ totals_out,
                      const __grid_constant__ Mbox m0, int xchg) {
  const Mbox m = xchg ? mbox_at_next_epoch(m0) : m0;  // the FIFO epoch advances after the step
  __shared__ uint32_t s_warp[kLocalThreads / 32];
  __shared__ uint32_t s_count;
  const uint32_t ls = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t base = (uint64_t)ls * shard_cap;
  const uint32_t head = alloc[ls].head, len = alloc[ls].len;
  Cand* out = cand_out + (uint64_t)ls * K;
  if (tid == 0) s_count = 0;
  __syncthreads();
  for (uint32_t k0 = 0; k0 < len; k0 += kLocalThreads) {
    const uint32_t count = s_count;
    if (count >= K) break;
    const uint32_t k = k0 + tid;
    bool sel = false;
    uint32_t slot = 0;
    if (k < len) {
      const uint64_t step = lifo ? (uint64_t)len - 1 - k : (uint64_t)k;
      const uint64_t pos = ((uint64_t)head + step) % shard_cap;
      slot = ord[base + pos];
      sel = key[base + slot] > 0;
    }
    const unsigned m = __ballot_sync(kFull, sel);
    if (lane == 0) s_warp[warp] = __popc(m);
    __syncthreads();
    uint32_t before = 0, total = 0;
#pragma unroll 4
    for (int w = 0; w < kLocalThreads / 32; ++w) {
      const uint32_t x = s_warp[w];
      before += w < warp ? x : 0u;
      total += x;
    }
    const uint32_t at = count + before + __popc(m & ((1u << lane) - 1u));
    if (sel && at < K) {
      Cand c;
      c.seq = seq[base + slot];
      c.shard = first_shard + ls;
      c.slot = slot;
      out[at] = c;
    }
    __syncthreads();
    if (tid == 0) s_count = count + total;
    __syncthreads();
  }
  if (tid == 0) {
    ShardTotals t;
    t.total_and_parity = 0;
    t.aux = s_count < K ? s_count : K;
    totals_out[ls] = t;
  }
  if (!xchg) return;
  // W > 1: push this shard's candidates and count into every peer's mailbox
  // over NVLink, then release the shard's flag there (mbox.cuh).
  __syncthreads();
  const MboxLayout L = mbox_layout(m.W, m.S, m.MB);
  const uint32_t b = mbox_buf(m), shard = first_shard + ls;
  const uint32_t n = s_count < K ? s_count : K;
  for (uint32_t r = 0; r < m.W; ++r) {
    Cand* dst = mbox_at<Cand>(m, r, L.cand) + ((uint64_t)b * m.S + shard) * K;
    for (uint32_t i = tid; i < n; i += kLocalThreads) dst[i] = out[i];
    if (tid == 0) {
      ShardTotals t;
      t.total_and_parity = 0;
      t.aux = n;
      mbox_at<ShardTotals>(m, r, L.ccnt)[b * m.S + shard] = t;
    }
  }
  __syncthreads();
  if (tid == 0) {
    mbox_producer_fence();
    for (uint32_t r = 0; r < m.W; ++r)
      mbox_publish(mbox_at<uint64_t>(m, r, L.cflag) + b * m.S + shard, m.epoch);
  }
}

// Number of entries of the sorted list c[0..n) that order before (sq, s)
// under (seq, shard) -- ascending lists for FIFO, descending for LIFO, and
// (key descending, shard ascending) for TopK (lifo == 2, topk.cu).
__device__ __forceinline__ uint32_t count_before(const Cand* __restrict__ c, uint32_t n,
                                                 uint32_t list_shard, uint64_t sq, uint32_t s,
                                                 int lifo) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    const uint64_t e = c[mid].seq;
    bool b;
    if (lifo == 0) b = e < sq || (e == sq && list_shard < s);        // FIFO
    else if (lifo == 1) b = e > sq || (e == sq && list_shard > s);   // LIFO
    else b = e > sq || (e == sq && list_shard < s);                  // TopK (seq = key)
    if (b) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__global__ void __launch_bounds__(kMergeThreads)
    fifo_merge_kernel(const Cand* __restrict__ cand_all, const ShardTotals* __restrict__ totals,
                      uint32_t S, uint32_t K, int lifo, uint64_t shard_cap, uint32_t rank,
                      uint32_t B, const uint32_t* const* gen_ptrs, uint32_t shards_per_rank,
                      uint64_t* out_idx, float* out_w, double* out_p, uint32_t* out_gen,
                      uint32_t* err, uint32_t* glob_shard, uint32_t* glob_slot,
                      const __grid_constant__ Mbox m0, int xchg) {
  const Mbox m = xchg ? mbox_at_next_epoch(m0) : m0;  // the FIFO epoch advances after the step
  const uint64_t t = (uint64_t)blockIdx.x * kMergeThreads + threadIdx.x;
  if (xchg) {  // candidates of all S shards arrive in this rank's mailbox
    const MboxLayout L = mbox_layout(m.W, m.S, m.MB);
    const uint32_t b = mbox_buf(m);
    if (threadIdx.x == 0)
      mbox_wait(mbox_at<uint64_t>(m, m.rank, L.cflag) + b * m.S, m.S, m.epoch, err);
    __syncthreads();
    cand_all = mbox_at<Cand>(m, m.rank, L.cand) + (uint64_t)b * m.S * K;
    totals = mbox_at<ShardTotals>(m, m.rank, L.ccnt) + b * m.S;
  }
  const bool failed = xchg && mbox_failed(err);  // a timed-out exchange: no candidates
  uint64_t avail = 0;
  for (uint32_t s = 0; s < S && !failed; ++s) avail += totals[s].aux;
  if (avail < K) {  // fewer than W*B selectable: EMPTY
    if (t < B) {
      out_idx[t] = kIdxNone;
      if (out_w) out_w[t] = 0.0f;
      if (out_p) out_p[t] = 0.0;
      if (out_gen) out_gen[t] = 0;
    }
    if (t == 0 && !failed) atomicOr(err, kErrEmpty);
    return;
  }
  if (t >= (uint64_t)S * K) return;
  const uint32_t s = (uint32_t)(t / K), p = (uint32_t)(t - (uint64_t)s * K);
  if (p >= totals[s].aux) return;
  const Cand me = cand_all[t];
  uint64_t pos = p;
  for (uint32_t s2 = 0; s2 < S; ++s2) {
    if (s2 == s) continue;
    pos += count_before(cand_all + (uint64_t)s2 * K, (uint32_t)totals[s2].aux, s2, me.seq, s,
                        lifo);
  }
  if (glob_shard) {  // whole merged list for the owner-affine assignment
    if (pos < K) {
      glob_shard[pos] = me.shard;
      glob_slot[pos] = me.slot;
    }
    return;
  }
  const uint64_t lo = (uint64_t)rank * B;
  if (pos < lo || pos >= lo + B) return;
  const uint32_t b = (uint32_t)(pos - lo);
  out_idx[b] = (uint64_t)me.shard * shard_cap + me.slot;
  if (out_w) out_w[b] = 1.0f;
  if (out_p) out_p[b] = 1.0;
  if (out_gen) {
    const uint32_t owner = me.shard / shards_per_rank;
    const uint64_t local = (uint64_t)(me.shard % shards_per_rank) * shard_cap + me.slot;
    out_gen[b] = gen_ptrs[owner][local];
  }
}

}  // namespace

cudaError_t launch_fifo_local(const uint64_t* key, const uint64_t* seq, const uint32_t* ord,
                              const AllocState* alloc, uint64_t shard_cap,
                              uint32_t n_shards_local, uint32_t first_shard, uint32_t K,
                              int lifo, Cand* cand_out, ShardTotals* totals_out,
                              const Mbox* mbox, cudaStream_t s) {
  count_launch();
  fifo_local_kernel<<<n_shards_local, kLocalThreads, 0, s>>>(
      key, seq, ord, alloc, shard_cap, first_shard, K, lifo, cand_out, totals_out,
      mbox ? *mbox : Mbox{}, mbox != nullptr);
  return cudaGetLastError();
}

cudaError_t launch_fifo_merge(const Cand* cand_all, const ShardTotals* totals_all,
                              uint32_t n_shards, uint32_t K, int lifo, uint64_t shard_cap,
                              uint32_t rank, uint32_t B, const uint32_t* const* gen_ptrs,
                              uint32_t shards_per_rank, uint64_t* out_idx, float* out_w,
                              double* out_p, uint32_t* out_gen, uint32_t* err,
                              uint32_t* glob_shard, uint32_t* glob_slot, const Mbox* mbox,
                              cudaStream_t s) {
  const uint64_t n = (uint64_t)n_shards * K;
  const uint64_t threads = n > B ? n : B;
  const uint32_t grid = (uint32_t)((threads + kMergeThreads - 1) / kMergeThreads);
  count_launch();
  fifo_merge_kernel<<<grid, kMergeThreads, 0, s>>>(cand_all, totals_all, n_shards, K, lifo,
                                                   shard_cap, rank, B, gen_ptrs, shards_per_rank,
                                                   out_idx, out_w, out_p, out_gen, err,
                                                   glob_shard, glob_slot,
                                                   mbox ? *mbox : Mbox{}, mbox != nullptr);
  return cudaGetLastError();
}

}  // namespace gear

namespace gear {

namespace {
__global__ void epoch_bump_u64_kernel(uint64_t* p) { *p += 1; }
}  // namespace

cudaError_t launch_epoch_bump(uint64_t* counter, cudaStream_t s) {
  count_launch();
  epoch_bump_u64_kernel<<<1, 1, 0, s>>>(counter);
  return cudaGetLastError();
}

}  // namespace gear
