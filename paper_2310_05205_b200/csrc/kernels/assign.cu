// assign.cu -- owner-affine assignment of the global batch to DP ranks
// (reading Q19 of DESIGN.md; "the majority of the trajectories
// collected by the servers reside in local memory").
//
// The global batch is the same W*B entries as the contiguous assignment
// (draws j of the Philox stream, or FIFO/LIFO merged positions); only which
// rank consumes which entry changes.  Rank r keeps its own entries (owner rank
// = shard / R) in j order, at most B; the entries beyond B of over-full
// owners form an overflow list in j order and under-full ranks take
// consecutive runs of it in rank order.  Every rank evaluates the rule over
// all W*B entries (only the owner is needed: Philox + mulhi + the 32 shard
// offsets for draws, the merged shard list for FIFO/LIFO), so no extra
// communication is needed and the result is identical on every rank.
//
// One CTA of 1024 threads; K = W*B <= 8*4096 entries are walked in chunks of
// 1024 with a per-owner ballot scan (W <= 8 owners).
#include "mbox.cuh"

namespace gear {

namespace {

constexpr int kThreads = 1024;
constexpr int kWarps = kThreads / 32;

__global__ void __launch_bounds__(kThreads) assign_kernel(const __grid_constant__ AssignParams p) {
  __shared__ uint64_t s_G[kMaxShards];        // inclusive shard offsets
  __shared__ uint32_t s_cnt[kWarps][kMaxRanks + 1];
  __shared__ uint32_t s_run[kMaxRanks + 1];   // running per-owner counts (+ overflow at [W])
  __shared__ uint64_t s_T;
  __shared__ uint32_t s_bail;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t W = p.W, B = p.B, K = W * B;
  const uint32_t S = p.n_shards;
  // W > 1 draws: exchange the shard totals through the peer mailboxes here;
  // the sample kernel that follows reads them from this rank's mailbox.
  const Mbox mm = (p.xchg || p.fifo_mbox) ? mbox_at_next_epoch(p.mbox) : p.mbox;
  const ShardTotals* totals = p.totals;
  if (p.xchg) {
    totals = mbox_exchange_totals(mm, p.totals_local, p.err);  // ends with a barrier:
    if (tid == 0) *p.mbox.epoch_dev = mm.epoch;                // every thread read it
  }
  // FIFO/LIFO through the mailboxes: the candidate counts of this exchange
  // (the FIFO epoch advances after this kernel)
  const ShardTotals* fifo_totals = p.fifo_totals;
  if (p.fifo_mbox) {
    const MboxLayout L = mbox_layout(mm.W, mm.S, mm.MB);
    fifo_totals = mbox_at<ShardTotals>(mm, mm.rank, L.ccnt) + mbox_buf(mm) * mm.S;
  }
  if (p.xchg && totals == nullptr) {  // timed out: the sample kernel writes GEAR_IDX_NONE
    for (uint32_t b = tid; b < B; b += kThreads) p.draw_list[b] = p.rank * B + b;
    return;
  }
  if (tid < 32) {
    uint64_t Ts = 0;
    if ((uint32_t)lane < S && totals)
      Ts = __ldcg(&totals[lane].total_and_parity) & ((1ull << 62) - 1);
    const uint64_t G = warp_incl_scan_u64(Ts, lane);
    if ((uint32_t)lane < S) s_G[lane] = G;
    if (lane == 31) s_T = G;
  }
  if (tid <= (int)kMaxRanks) s_run[tid] = 0;
  if (tid == 0) {
    s_bail = 0;
    if (fifo_totals) {  // FIFO/LIFO: fewer than K candidates -> EMPTY (merge wrote it)
      uint64_t avail = 0;
      for (uint32_t s = 0; s < S; ++s) avail += __ldcg(&fifo_totals[s].aux);
      s_bail = avail < K || (p.fifo_mbox && mbox_failed(p.err));  // timed out: likewise
    }
  }
  __syncthreads();
  if (s_bail) return;
  const uint64_t T = s_T;
  // (an asm load under a branch: a plain conditional load from a possibly
  // null pointer was hoisted by the compiler and faulted)
  uint64_t seed = p.seed;
  if (p.seed_dev != nullptr) seed = ld_relaxed_u64(p.seed_dev);
  if (!p.glob_shard && T == 0) {  // nothing selectable: the sample kernel latches EMPTY
    for (uint32_t b = tid; b < B; b += kThreads) p.draw_list[b] = p.rank * B + b;
    return;
  }
  // Pass 1: position of each entry among its owner's entries, overflow index.
  for (uint32_t c0 = 0; c0 < K; c0 += kThreads) {
    const uint32_t j = c0 + tid;
    uint32_t o = kMaxRanks;  // out of range: matches no owner
    if (j < K) {
      uint32_t s;
      if (p.glob_shard) {
        s = p.glob_shard[j];
      } else {
        const uint64_t u = __umul64hi(draw_bits(seed, j), T);
        s = 0;
        while (s + 1 < S && s_G[s] <= u) ++s;
      }
      o = s / p.shards_per_rank;
    }
    uint32_t before_mine = 0;
    for (uint32_t r = 0; r < W; ++r) {
      const unsigned m = __ballot_sync(kFull, o == r);
      if (lane == 0) s_cnt[warp][r] = __popc(m);
      if (o == r) before_mine = __popc(m & ((1u << lane) - 1u));
    }
    __syncthreads();
    uint32_t pos = 0;
    if (o < W) {
      for (int w = 0; w < warp; ++w) before_mine += s_cnt[w][o];
      pos = s_run[o] + before_mine;
    }
    const bool over = o < W && pos >= B;
    const unsigned mo = __ballot_sync(kFull, over);
    __syncthreads();  // everyone has read s_cnt / s_run
    if (lane == 0) s_cnt[warp][kMaxRanks] = __popc(mo);
    __syncthreads();
    uint32_t ov = s_run[kMaxRanks] + __popc(mo & ((1u << lane) - 1u));
    for (int w = 0; w < warp; ++w) ov += s_cnt[w][kMaxRanks];
    if (j < K) {
      p.pos_scratch[j] = (o == p.rank && pos < B) ? pos : ~0u;
      p.ov_scratch[j] = over ? ov : ~0u;
    }
    __syncthreads();
    if (tid < (int)W) {
      uint32_t add = 0;
      for (int w = 0; w < kWarps; ++w) add += s_cnt[w][tid];
      s_run[tid] += add;
    }
    if (tid == 0) {
      uint32_t add = 0;
      for (int w = 0; w < kWarps; ++w) add += s_cnt[w][kMaxRanks];
      s_run[kMaxRanks] += add;
    }
    __syncthreads();
  }
  // Run of the overflow list this rank takes.
  uint32_t offset = 0;
  for (uint32_t r = 0; r < p.rank; ++r) offset += s_run[r] < B ? B - s_run[r] : 0;
  const uint32_t own = s_run[p.rank] < B ? s_run[p.rank] : B;
  const uint32_t need = B - own;
  // Pass 2: scatter this rank's entries into its slice.
  for (uint32_t j = tid; j < K; j += kThreads) {
    const uint32_t ps = p.pos_scratch[j], ov = p.ov_scratch[j];
    if (ps != ~0u) p.draw_list[ps] = j;
    else if (ov != ~0u && ov >= offset && ov < offset + need) p.draw_list[own + ov - offset] = j;
  }
  if (!p.glob_shard) return;
  // FIFO/LIFO: emit the outputs straight from the merged global list.
  __syncthreads();
  for (uint32_t b = tid; b < B; b += kThreads) {
    const uint32_t j = p.draw_list[b];
    const uint32_t s = p.glob_shard[j], slot = p.glob_slot[j];
    p.out_idx[b] = (uint64_t)s * p.shard_cap + slot;
    if (p.out_w) p.out_w[b] = 1.0f;
    if (p.out_p) p.out_p[b] = 1.0;
    if (p.out_gen) {
      const uint32_t owner = s / p.shards_per_rank;
      p.out_gen[b] = p.gen_ptrs[owner][(uint64_t)(s % p.shards_per_rank) * p.shard_cap + slot];
    }
  }
}

}  // namespace

cudaError_t launch_assign(const AssignParams& p, cudaStream_t s) {
  if (p.B == 0) return cudaSuccess;
  count_launch();
  assign_kernel<<<1, kThreads, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace gear
