// topk.cu -- decentralised TopK selection ("GEAR provides
// FIFO and TopK selection implementation, which are deterministic in
// decentralized selection scenarios ... all servers can perform a local scan
// to generate k samples before the global gathering").  Reading Q20: the
// K = W*B selectable trajectories with the largest keys, ties by the smaller
// global id, in that order.
//
// Local step for each of the rank's R shards, spread over the whole GPU
// (G CTAs per shard, each owning a contiguous slice of the shard's keys):
//  1. stats: selectable count and maximum key (block reduce + atomics);
//  2. radix select of the K-th largest key, one launch per key byte from the
//     top: every CTA histograms the byte of the keys that match the prefix
//     chosen so far into shared memory and adds it to the shard's global
//     histogram; the last CTA of the shard (threadfence + counter) picks the
//     digit, extends the prefix and re-arms the histogram.  The result is the
//     threshold key T* and the number of keys == T* that complete the K;
//  3. count: per CTA, the keys > T* and the keys == T* of its slice;
//  4. write: each CTA turns the counts of the CTAs before it into offsets and
//     compacts its selected keys in slot order (ties: only the first needed
//     keys == T* in slot order);
//  5. sort: rank sort of the <= K candidates by (key desc, slot asc), one
//     thread per candidate counting the candidates before it in shared memory;
//     each writes itself at its rank (W > 1: also into every peer's mailbox).
// The global merge is the FIFO/LIFO merge with the TopK order (fifo.cu).
// Every launch is stream-ordered and every counter re-arms itself, so the
// sequence can be captured in a CUDA graph.
#include <cooperative_groups.h>

#include "mbox.cuh"

namespace gear {

namespace {

constexpr int kThreads = 256;
constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;

struct Slice {
  uint64_t begin, end;  // slot range of this CTA within its shard
};

__device__ __forceinline__ Slice cta_slice(uint64_t shard_cap, uint32_t G, uint32_t g) {
  const uint64_t per = ((shard_cap + G - 1) / G + kThreads - 1) / kThreads * kThreads;
  Slice s;
  s.begin = min(shard_cap, (uint64_t)g * per);
  s.end = min(shard_cap, s.begin + per);
  return s;
}

// Last CTA of shard `ls` to arrive (threadfence + counter); re-arms it.
__device__ __forceinline__ bool last_cta(uint32_t* ctr, uint32_t G, bool* s_flag) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    *s_flag = atomicAdd(ctr, 1u) == G - 1;
    if (*s_flag) *ctr = 0;
  }
  __syncthreads();
  if (*s_flag) __threadfence();
  return *s_flag;
}

__global__ void __launch_bounds__(kThreads)
    stats_kernel(const uint64_t* __restrict__ key, uint64_t shard_cap, uint32_t G, uint32_t K,
                 TopkState* st) {
  __shared__ bool s_last;
  __shared__ unsigned long long s_max;
  __shared__ uint32_t s_cnt;
  const uint32_t ls = blockIdx.y;
  const Slice sl = cta_slice(shard_cap, G, blockIdx.x);
  const uint64_t* k = key + (uint64_t)ls * shard_cap;
  if (threadIdx.x == 0) {
    s_max = 0;
    s_cnt = 0;
  }
  __syncthreads();
  uint32_t cnt = 0;
  unsigned long long mx = 0;
  for (uint64_t i = sl.begin + threadIdx.x; i < sl.end; i += kThreads) {
    const uint64_t x = k[i];
    cnt += x > 0;
    mx = x > mx ? x : mx;
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    cnt += __shfl_xor_sync(kFull, cnt, d);
    const unsigned long long o = __shfl_xor_sync(kFull, mx, d);
    mx = o > mx ? o : mx;
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&s_cnt, cnt);
    atomicMax(&s_max, mx);
  }
  __syncthreads();
  TopkState& S = st[ls];
  if (threadIdx.x == 0) {
    atomicAdd(&S.n_sel, s_cnt);
    atomicMax(&S.max_key, s_max);
  }
  if (!last_cta(&S.ctr, G, &s_last)) return;
  if (threadIdx.x == 0) {  // set up the radix select
    const uint64_t mxk = *(volatile unsigned long long*)&S.max_key;
    const uint32_t n = *(volatile uint32_t*)&S.n_sel;
    S.all = n <= K;
    S.eq_all = 0;
    S.k_remain = K;
    S.prefix = 0;
    S.mask = 0;
    S.shift = mxk ? ((63 - __clzll(mxk)) / 8) * 8 : 0;
  }
  for (int b = threadIdx.x; b < 256; b += kThreads) S.hist[b] = 0;
}

__global__ void __launch_bounds__(kThreads)
    hist_kernel(const uint64_t* __restrict__ key, uint64_t shard_cap, uint32_t G, TopkState* st) {
  __shared__ uint32_t s_hist[256];
  __shared__ bool s_last;
  const uint32_t ls = blockIdx.y;
  TopkState& S = st[ls];
  const int shift = *(volatile int*)&S.shift;
  if (S.all || shift < 0) return;  // selection finished (uniform over the shard)
  const uint64_t prefix = S.prefix, mask = S.mask;
  const Slice sl = cta_slice(shard_cap, G, blockIdx.x);
  const uint64_t* k = key + (uint64_t)ls * shard_cap;
  for (int b = threadIdx.x; b < 256; b += kThreads) s_hist[b] = 0;
  __syncthreads();
  for (uint64_t i = sl.begin + threadIdx.x; i < sl.end; i += kThreads) {
    const uint64_t x = k[i];
    if (x > 0 && (x & mask) == prefix) atomicAdd(&s_hist[(x >> shift) & 255], 1u);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < 256; b += kThreads)
    if (s_hist[b]) atomicAdd(&S.hist[b], s_hist[b]);
  if (!last_cta(&S.ctr, G, &s_last)) return;
  // The digit: the largest v whose suffix count sum_{u >= v} hist[u] reaches
  // k_remain.  Thread t owns bin 255 - t; block-wide inclusive scan over t.
  static_assert(kThreads == 256, "one thread per digit");
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const uint32_t kk = S.k_remain;
  const uint32_t h = *(volatile uint32_t*)&S.hist[255 - t];
  uint32_t suf = h;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t o = __shfl_up_sync(kFull, suf, d);
    if (lane >= d) suf += o;
  }
  if (lane == 31) s_hist[warp] = suf;  // warp totals (the local histogram is dead)
  __syncthreads();
  for (int w = 0; w < warp; ++w) suf += s_hist[w];
  if (suf >= kk && suf - h < kk) {  // exactly one thread
    const uint32_t v = 255 - t;
    const uint32_t need = kk - (suf - h);
    S.prefix = prefix | ((uint64_t)v << shift);
    S.mask = mask | (255ull << shift);
    S.k_remain = need;
    // Done after the last byte, or as soon as the boundary bin is small: then
    // every key of the bin becomes a candidate (at most kTopkEqMax beyond the
    // K) and the rank sort keeps the first K by (key desc, slot asc).  After
    // the last byte with a large bin the bin holds equal keys: the first
    // `need` in slot order are taken.
    const bool small = h - need <= kTopkEqMax;
    S.eq_all = small ? 1u : 0u;
    S.shift = (small || shift == 0) ? -1 : shift - 8;
  }
  __syncthreads();  // every thread has read the histogram
  for (int b = threadIdx.x; b < 256; b += kThreads) S.hist[b] = 0;
}

// Candidates: all selectable keys (all), or the keys whose resolved bytes
// (x & mask) exceed the prefix plus those whose resolved bytes equal it --
// all of them (eq_all: a bin of at most K + kTopkEqMax keys, ranked by the
// sort) or the first k_remain in slot order (every byte resolved: the prefix
// is the K-th largest key T* itself, "key > T*, then ties by slot").
__device__ __forceinline__ void classify(const TopkState& S, uint64_t x, bool* gt, bool* eq) {
  if (S.all) {
    *gt = x > 0;
    *eq = false;
  } else {
    const uint64_t xm = x & S.mask;
    *gt = x > 0 && xm > S.prefix;
    *eq = x > 0 && xm == S.prefix;
  }
}

__global__ void __launch_bounds__(kThreads)
    count_kernel(const uint64_t* __restrict__ key, uint64_t shard_cap, uint32_t G, TopkState* st,
                 uint32_t* cnt /* [R][G][2] */) {
  __shared__ uint32_t s_gt, s_eq;
  const uint32_t ls = blockIdx.y;
  const TopkState& S = st[ls];
  const Slice sl = cta_slice(shard_cap, G, blockIdx.x);
  const uint64_t* k = key + (uint64_t)ls * shard_cap;
  if (threadIdx.x == 0) s_gt = s_eq = 0;
  __syncthreads();
  uint32_t g = 0, e = 0;
  for (uint64_t i = sl.begin + threadIdx.x; i < sl.end; i += kThreads) {
    bool gt, eq;
    classify(S, k[i], &gt, &eq);
    g += gt;
    e += eq;
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    g += __shfl_xor_sync(kFull, g, d);
    e += __shfl_xor_sync(kFull, e, d);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&s_gt, g);
    atomicAdd(&s_eq, e);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    cnt[((uint64_t)ls * G + blockIdx.x) * 2 + 0] = s_gt;
    cnt[((uint64_t)ls * G + blockIdx.x) * 2 + 1] = s_eq;
  }
}

__global__ void __launch_bounds__(kThreads)
    write_kernel(const uint64_t* __restrict__ key, uint64_t shard_cap, uint32_t G, uint32_t K,
                 uint32_t first_shard, const TopkState* st, const uint32_t* __restrict__ cnt,
                 Cand* __restrict__ cand_out, ShardTotals* __restrict__ totals_out) {
  __shared__ uint32_t s_red[kThreads / 32];
  __shared__ uint32_t s_base_gt, s_base_eq, s_tot;
  const uint32_t ls = blockIdx.y;
  const TopkState& S = st[ls];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t need = S.all ? 0u : (S.eq_all ? 0xffffffffu : S.k_remain);
  const uint32_t cap = K + kTopkEqMax;  // candidate slots per shard
  __shared__ uint32_t s_tg, s_te;
  if (tid == 0) s_base_gt = s_base_eq = s_tg = s_te = 0;
  __syncthreads();
  {  // offsets from the CTAs before this one (slot order), block-wide
    uint32_t bg = 0, be = 0, tg = 0, te = 0;
    for (uint32_t c = tid; c < G; c += kThreads) {
      const uint2 ge = *reinterpret_cast<const uint2*>(cnt + ((uint64_t)ls * G + c) * 2);
      if (c < blockIdx.x) {
        bg += ge.x;
        be += ge.y;
      }
      tg += ge.x;
      te += ge.y;
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      bg += __shfl_xor_sync(kFull, bg, d);
      be += __shfl_xor_sync(kFull, be, d);
      tg += __shfl_xor_sync(kFull, tg, d);
      te += __shfl_xor_sync(kFull, te, d);
    }
    if (lane == 0 && (tg | te)) {
      atomicAdd(&s_base_gt, bg);
      atomicAdd(&s_base_eq, be);
      atomicAdd(&s_tg, tg);
      atomicAdd(&s_te, te);
    }
    __syncthreads();
    if (tid == 0) s_tot = min(cap, s_tg + min(need, s_te));
    __syncthreads();
  }
  const uint32_t base_gt = s_base_gt;
  uint32_t eq_seen = s_base_eq;  // keys == T* in earlier slots (block-uniform)
  // taken so far = gt before + ties taken before
  uint32_t taken = base_gt + min(need, eq_seen);
  const Slice sl = cta_slice(shard_cap, G, blockIdx.x);
  const uint64_t* k = key + (uint64_t)ls * shard_cap;
  Cand* out = cand_out + (uint64_t)ls * cap;
  for (uint64_t i0 = sl.begin; i0 < sl.end; i0 += kThreads) {
    const uint64_t i = i0 + tid;
    const uint64_t x = i < sl.end ? k[i] : 0;
    bool gt = false, eq = false;
    if (i < sl.end) classify(S, x, &gt, &eq);
    const unsigned mg = __ballot_sync(kFull, gt), me = __ballot_sync(kFull, eq);
    if (lane == 0) s_red[warp] = (__popc(me) << 16) | __popc(mg);
    __syncthreads();
    uint32_t gt_before = 0, eq_before = 0, gt_total = 0, eq_total = 0;
    for (int w = 0; w < kThreads / 32; ++w) {
      const uint32_t c = s_red[w];
      if (w < warp) {
        gt_before += c & 0xffff;
        eq_before += c >> 16;
      }
      gt_total += c & 0xffff;
      eq_total += c >> 16;
    }
    const uint32_t lt = (1u << lane) - 1u;
    const uint32_t my_eq_rank = eq_seen + eq_before + __popc(me & lt);  // among keys == T*
    const uint32_t eq_taken_before = min(need, my_eq_rank) - min(need, eq_seen);
    if (gt || (eq && my_eq_rank < need)) {
      Cand c;
      c.seq = x;
      c.shard = first_shard + ls;
      c.slot = (uint32_t)i;
      const uint32_t pos = taken + gt_before + __popc(mg & lt) + eq_taken_before;
      if (pos < cap) out[pos] = c;  // always true when the selection invariant holds
    }
    taken += gt_total + (min(need, eq_seen + eq_total) - min(need, eq_seen));
    eq_seen += eq_total;
    __syncthreads();
  }
  if (blockIdx.x == 0 && tid == 0) {  // candidates for the sort, list length for the merge
    ShardTotals t;
    t.total_and_parity = s_tot;
    t.aux = min(s_tot, K);
    totals_out[ls] = t;
  }
}

// ---- small shards: the whole local select in ONE launch on a thread-block
// cluster (B200 distributed shared memory) --------------------------------
// kClusterCtas CTAs of one cluster share a shard (a contiguous slice each).
// Every step that the grid-wide path does with a separate launch and global
// atomics -- stats, each radix pass, the counts -- is a cluster barrier here:
// each CTA builds its partial (count, max, 256-bin histogram, gt/eq counts)
// in its own shared memory and every CTA reads all of them through DSMEM
// (cluster.map_shared_rank) and takes the same decision.  The candidates go
// to the same unsorted list and totals as write_kernel's, for sort_kernel.
constexpr int kClusterCtas = 8;          // portable cluster size
constexpr int kClusterThreads = 512;
// Shards up to 64 K keys (c2 at W >= 2): the cluster holds 8 SMs for the
// select, so bigger shards keep the grid-wide path, which at c2 W = 1
// (100 K keys) measured 2.6% faster next to the collect (profiles/r02_topk2).
constexpr uint64_t kClusterMaxKeys = 1u << 16;

namespace cg = cooperative_groups;

__global__ void __cluster_dims__(kClusterCtas, 1, 1) __launch_bounds__(kClusterThreads)
    topk_cluster_kernel(const uint64_t* __restrict__ key, uint64_t shard_cap, uint32_t K,
                        uint32_t first_shard, Cand* __restrict__ cand_out,
                        ShardTotals* __restrict__ totals_out) {
  cg::cluster_group cluster = cg::this_cluster();
  __shared__ uint32_t s_hist[256];
  __shared__ uint32_t s_scan[kClusterThreads / 32];
  __shared__ uint32_t s_cnt, s_gt, s_eq;
  __shared__ unsigned long long s_max;
  __shared__ uint64_t s_prefix, s_mask;
  __shared__ uint32_t s_kremain, s_all, s_eqall;
  __shared__ int s_shift;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t cr = cluster.block_rank();
  const uint32_t ls = blockIdx.y;
  const Slice sl = cta_slice(shard_cap, kClusterCtas, cr);
  const uint64_t* k = key + (uint64_t)ls * shard_cap;

  // stats: selectable count and maximum key of the shard
  if (tid == 0) {
    s_cnt = 0;
    s_max = 0;
  }
  __syncthreads();
  {
    uint32_t cnt = 0;
    unsigned long long mx = 0;
    for (uint64_t i = sl.begin + tid; i < sl.end; i += kClusterThreads) {
      const uint64_t x = k[i];
      cnt += x > 0;
      mx = x > mx ? x : mx;
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      cnt += __shfl_xor_sync(kFull, cnt, d);
      const unsigned long long o = __shfl_xor_sync(kFull, mx, d);
      mx = o > mx ? o : mx;
    }
    if (lane == 0) {
      atomicAdd(&s_cnt, cnt);
      atomicMax(&s_max, mx);
    }
  }
  cluster.sync();
  if (tid == 0) {
    uint32_t n = 0;
    unsigned long long mx = 0;
    for (int r = 0; r < kClusterCtas; ++r) {
      n += *cluster.map_shared_rank(&s_cnt, r);
      const unsigned long long m = *cluster.map_shared_rank(&s_max, r);
      mx = m > mx ? m : mx;
    }
    s_all = n <= K;
    s_eqall = 0;
    s_kremain = K;
    s_prefix = 0;
    s_mask = 0;
    s_shift = s_all ? -1 : (mx ? ((63 - __clzll(mx)) / 8) * 8 : 0);
  }
  __syncthreads();

  // radix select of the K-th largest key, one byte per pass from the top
  while (s_shift >= 0) {
    const int shift = s_shift;
    const uint64_t prefix = s_prefix, mask = s_mask;
    cluster.sync();  // every CTA is done reading the previous pass's histograms
    for (int b = tid; b < 256; b += kClusterThreads) s_hist[b] = 0;
    __syncthreads();
    for (uint64_t i = sl.begin + tid; i < sl.end; i += kClusterThreads) {
      const uint64_t x = k[i];
      if (x > 0 && (x & mask) == prefix) atomicAdd(&s_hist[(x >> shift) & 255], 1u);
    }
    cluster.sync();  // every CTA's histogram is complete
    // the shard's histogram (thread t < 256 owns bin 255 - t, summed over the
    // cluster through DSMEM), then the digit: the largest v whose suffix
    // count reaches k_remain (block-wide inclusive scan over t)
    uint32_t h = 0;
    if (tid < 256)
      for (int r = 0; r < kClusterCtas; ++r) h += cluster.map_shared_rank(s_hist, r)[255 - tid];
    uint32_t suf = h;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t o = __shfl_up_sync(kFull, suf, d);
      if (lane >= d) suf += o;
    }
    if (lane == 31) s_scan[warp] = suf;
    __syncthreads();
    for (int w = 0; w < warp && tid < 256; ++w) suf += s_scan[w];
    const uint32_t kk = s_kremain;
    __syncthreads();  // s_kremain read by every thread before it changes
    if (tid < 256 && suf >= kk && suf - h < kk) {  // exactly one thread
      const uint32_t v = 255 - tid;
      const uint32_t need = kk - (suf - h);
      s_prefix = prefix | ((uint64_t)v << shift);
      s_mask = mask | (255ull << shift);
      s_kremain = need;
      const bool small = h - need <= kTopkEqMax;  // as hist_kernel
      s_eqall = small ? 1u : 0u;
      s_shift = (small || shift == 0) ? -1 : shift - 8;
    }
    __syncthreads();
  }

  // counts of keys > T* and == T* per CTA, offsets from the CTAs before it
  TopkState S{};
  S.all = s_all;
  S.prefix = s_prefix;
  S.mask = s_mask;
  const uint32_t need = s_all ? 0u : (s_eqall ? 0xffffffffu : s_kremain);
  if (tid == 0) s_gt = s_eq = 0;
  __syncthreads();
  {
    uint32_t g = 0, e = 0;
    for (uint64_t i = sl.begin + tid; i < sl.end; i += kClusterThreads) {
      bool gt, eq;
      classify(S, k[i], &gt, &eq);
      g += gt;
      e += eq;
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      g += __shfl_xor_sync(kFull, g, d);
      e += __shfl_xor_sync(kFull, e, d);
    }
    if (lane == 0) {
      atomicAdd(&s_gt, g);
      atomicAdd(&s_eq, e);
    }
  }
  cluster.sync();
  uint32_t base_gt = 0, eq_seen = 0, tg = 0, te = 0;
  for (int r = 0; r < kClusterCtas; ++r) {
    const uint32_t g = *cluster.map_shared_rank(&s_gt, r), e = *cluster.map_shared_rank(&s_eq, r);
    if (r < (int)cr) {
      base_gt += g;
      eq_seen += e;
    }
    tg += g;
    te += e;
  }
  cluster.sync();  // no DSMEM access after this: any CTA may exit
  const uint32_t cap = K + kTopkEqMax;
  const uint32_t tot = min(cap, tg + min(need, te));

  // write: compaction in slot order (ties: the first `need` in slot order)
  uint32_t taken = base_gt + min(need, eq_seen);
  Cand* out = cand_out + (uint64_t)ls * cap;
  for (uint64_t i0 = sl.begin; i0 < sl.end; i0 += kClusterThreads) {
    const uint64_t i = i0 + tid;
    const uint64_t x = i < sl.end ? k[i] : 0;
    bool gt = false, eq = false;
    if (i < sl.end) classify(S, x, &gt, &eq);
    const unsigned mg = __ballot_sync(kFull, gt), me = __ballot_sync(kFull, eq);
    if (lane == 0) s_scan[warp] = (__popc(me) << 16) | __popc(mg);
    __syncthreads();
    uint32_t gt_before = 0, eq_before = 0, gt_total = 0, eq_total = 0;
    for (int w = 0; w < kClusterThreads / 32; ++w) {
      const uint32_t c = s_scan[w];
      if (w < warp) {
        gt_before += c & 0xffff;
        eq_before += c >> 16;
      }
      gt_total += c & 0xffff;
      eq_total += c >> 16;
    }
    const uint32_t lt = (1u << lane) - 1u;
    const uint32_t my_eq_rank = eq_seen + eq_before + __popc(me & lt);
    const uint32_t eq_taken_before = min(need, my_eq_rank) - min(need, eq_seen);
    if (gt || (eq && my_eq_rank < need)) {
      Cand c;
      c.seq = x;
      c.shard = first_shard + ls;
      c.slot = (uint32_t)i;
      const uint32_t pos = taken + gt_before + __popc(mg & lt) + eq_taken_before;
      if (pos < cap) out[pos] = c;
    }
    taken += gt_total + (min(need, eq_seen + eq_total) - min(need, eq_seen));
    eq_seen += eq_total;
    __syncthreads();
  }
  if (cr == 0 && tid == 0) {  // candidates for the sort, list length for the merge
    ShardTotals t;
    t.total_and_parity = tot;
    t.aux = min(tot, K);
    totals_out[ls] = t;
  }
}

// Candidate order of TopK: larger key first, then smaller slot.
__device__ __forceinline__ bool before(const Cand& a, const Cand& b) {
  return a.seq > b.seq || (a.seq == b.seq && a.slot < b.slot);
}

// Rank sort: the position of a candidate is the number of candidates before
// it in the TopK order (keys and slots are distinct, so the ranks are a
// permutation).
//  * n <= kSortDirect candidates (one launch, kMerge = false): one warp per
//    candidate, the lanes compare it with a strided 1/32 of the list
//    (L1-resident after the first warps) and sum; kSortWarps candidates per
//    CTA, ceil(n / kSortWarps) CTAs per shard.
//  * more (kMerge = true, after run_rank_kernel): the list is cut into runs of
//    kSortRun candidates, each already sorted by run_rank_kernel (the same
//    warp rank within the run); a candidate's rank is its position in its run
//    plus, for every other run, the number of that run's candidates before it
//    -- one binary search per run, one lane per run (<= 32 runs) -- so the
//    work is O(n log n) instead of O(n^2).
// The output (and at W > 1 every peer's mailbox) gets the first K ranks.
constexpr uint32_t kSortDirect = 8192;
constexpr uint32_t kSortRun = 4096;

__global__ void __launch_bounds__(kSortThreads)
    run_rank_kernel(uint32_t K, const Cand* __restrict__ unsorted, Cand* __restrict__ runs,
                    const ShardTotals* __restrict__ totals) {
  const uint32_t ls = blockIdx.y;
  const int lane = threadIdx.x & 31;
  const uint32_t n = (uint32_t)totals[ls].total_and_parity;
  const uint32_t i = blockIdx.x * kSortWarps + (threadIdx.x >> 5);
  if (i >= n) return;
  const uint64_t cap = (uint64_t)K + kTopkEqMax;
  const Cand* in = unsorted + (uint64_t)ls * cap;
  const Cand me = in[i];
  const uint32_t q0 = i / kSortRun * kSortRun, q1 = min(n, q0 + kSortRun);
  uint32_t rank = 0;
#pragma unroll 4
  for (uint32_t j = q0 + lane; j < q1; j += 32) rank += before(in[j], me);
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) rank += __shfl_xor_sync(kFull, rank, d);
  if (lane == 0) runs[(uint64_t)ls * cap + q0 + rank] = me;
}

template <bool kMerge>
__global__ void __launch_bounds__(kSortThreads)
    sort_kernel(uint32_t K, uint32_t first_shard, const Cand* __restrict__ unsorted,
                Cand* __restrict__ sorted, const ShardTotals* __restrict__ totals, TopkState* st,
                const __grid_constant__ Mbox m0, int xchg) {
  __shared__ bool s_last;
  const Mbox m = xchg ? mbox_at_next_epoch(m0) : m0;  // the FIFO/TopK epoch advances later
  const uint32_t ls = blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31;
  const uint32_t n = (uint32_t)totals[ls].total_and_parity;  // candidates (write_kernel)
  const uint32_t n_out = n < K ? n : K;
  const uint32_t i = blockIdx.x * kSortWarps + (tid >> 5);
  const uint32_t shard = first_shard + ls;
  if (blockIdx.x == 0 && tid == 0) {  // re-arm this shard's selection state for the next call
    TopkState& S = st[ls];
    S.n_sel = 0;
    S.max_key = 0;
  }
  if (i < n) {
    const Cand* in = unsorted + (uint64_t)ls * (K + kTopkEqMax);
    const Cand me = in[i];
    uint32_t rank = 0;
    if (kMerge) {  // `in` holds sorted runs: position in the own run + searches in the others
      const uint32_t q = i / kSortRun, runs = (n + kSortRun - 1) / kSortRun;
      if ((uint32_t)lane < runs && (uint32_t)lane != q) {
        uint32_t lo = lane * kSortRun, hi = min(n, lo + kSortRun);  // first x with !before(x, me)
        const uint32_t base = lo;
        while (lo < hi) {
          const uint32_t mid = (lo + hi) >> 1;
          if (before(in[mid], me)) lo = mid + 1;
          else hi = mid;
        }
        rank = lo - base;
      }
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) rank += __shfl_xor_sync(kFull, rank, d);
      rank += i - q * kSortRun;
    } else {
#pragma unroll 4
      for (uint32_t j = lane; j < n; j += 32) rank += before(in[j], me);
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) rank += __shfl_xor_sync(kFull, rank, d);
    }
    if (rank < K && lane == 0) sorted[(uint64_t)ls * K + rank] = me;
    if (rank < K && xchg && lane < m.W) {  // W > 1: straight into every peer's mailbox too
      const MboxLayout L = mbox_layout(m.W, m.S, m.MB);
      const uint32_t b = mbox_buf(m);
      mbox_at<Cand>(m, lane, L.cand)[((uint64_t)b * m.S + shard) * K + rank] = me;
    }
  }
  if (!xchg) return;
  // The last CTA of the shard publishes the list length and the epoch flag.
  __syncthreads();
  if (tid == 0) {
    mbox_producer_fence();
    s_last = atomicAdd(&st[ls].ctr, 1u) == gridDim.x - 1;
    if (s_last) st[ls].ctr = 0;
  }
  __syncthreads();
  if (!s_last || tid != 0) return;
  mbox_producer_fence();
  const MboxLayout L = mbox_layout(m.W, m.S, m.MB);
  const uint32_t b = mbox_buf(m);
  ShardTotals t;
  t.total_and_parity = 0;
  t.aux = n_out;
  for (uint32_t r = 0; r < m.W; ++r) mbox_at<ShardTotals>(m, r, L.ccnt)[b * m.S + shard] = t;
  mbox_producer_fence();
  for (uint32_t r = 0; r < m.W; ++r)
    mbox_publish(mbox_at<uint64_t>(m, r, L.cflag) + b * m.S + shard, m.epoch);
}

}  // namespace

// (<= 32 runs of kSortRun candidates, K + kTopkEqMax of them)
uint32_t topk_max_k() { return 32 * kSortRun - kTopkEqMax; }

// GEAR_TOPK_CLUSTER=0 forces the grid-wide path for every shard size (A/B).
bool topk_cluster_enabled() {
  static const bool on = [] {
    const char* e = getenv("GEAR_TOPK_CLUSTER");
    return e == nullptr || e[0] != '0';
  }();
  return on;
}

#ifndef GEAR_TOPK_KEYS_PER_CTA
#define GEAR_TOPK_KEYS_PER_CTA 256
#endif
constexpr uint64_t kTopkKeysPerCta = GEAR_TOPK_KEYS_PER_CTA;

cudaError_t launch_topk_local(const uint64_t* key, uint64_t shard_cap, uint64_t q_max,
                              uint32_t n_shards_local,
                              uint32_t first_shard, uint32_t K, Cand* cand_tmp, Cand* cand_out,
                              ShardTotals* totals_out, TopkState* state, uint32_t* cnt,
                              const Mbox* mbox, cudaStream_t s) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // CTAs per shard: ~2 waves of the GPU over all local shards, >= 1 slice of
  // kTopkKeysPerCta keys (256; 4096 and 16384 measured 8% / 27% slower at c2
  // TopK, W = 4: profiles/r02_topk)
  uint32_t G = (uint32_t)(2 * sms) / n_shards_local;
  G = G < 1 ? 1 : G;
  const uint64_t max_g = (shard_cap + kTopkKeysPerCta - 1) / kTopkKeysPerCta;
  G = (uint64_t)G > max_g ? (uint32_t)max_g : G;
  G = G > kTopkMaxCtas ? kTopkMaxCtas : G;
  const dim3 grid(G, n_shards_local);
  // Every key is <= q_max: the select never needs more passes than q_max has
  // bytes (6 at c2); the passes after an early exit are no-op launches.
  int passes = 1;
  while (passes < 8 && (q_max >> (8 * passes)) != 0) ++passes;
  if (shard_cap <= kClusterMaxKeys && topk_cluster_enabled()) {
    // small shards: stats + every radix pass + counts + compaction in one
    // cluster launch (DSMEM instead of global atomics between launches)
    count_launch(2);
    topk_cluster_kernel<<<dim3(kClusterCtas, n_shards_local), kClusterThreads, 0, s>>>(
        key, shard_cap, K, first_shard, cand_tmp, totals_out);
  } else {
    count_launch(4 + passes);
    stats_kernel<<<grid, kThreads, 0, s>>>(key, shard_cap, G, K, state);
    for (int pass = 0; pass < passes; ++pass)  // one per key byte from the top
      hist_kernel<<<grid, kThreads, 0, s>>>(key, shard_cap, G, state);
    count_kernel<<<grid, kThreads, 0, s>>>(key, shard_cap, G, state, cnt);
    write_kernel<<<grid, kThreads, 0, s>>>(key, shard_cap, G, K, first_shard, state, cnt, cand_tmp,
                                           totals_out);
  }
  // candidates n <= K + kTopkEqMax: the direct rank sort while that bound is
  // small, runs + merge ranks above it (cand_tmp holds 2 x R x (K + kTopkEqMax))
  const dim3 sgrid((K + kTopkEqMax + kSortWarps - 1) / kSortWarps, n_shards_local);
  if (K + kTopkEqMax <= kSortDirect) {  // (the sort launch is counted above)
    sort_kernel<false><<<sgrid, kSortThreads, 0, s>>>(K, first_shard, cand_tmp, cand_out,
                                                      totals_out, state, mbox ? *mbox : Mbox{},
                                                      mbox != nullptr);
  } else {
    Cand* runs = cand_tmp + (uint64_t)n_shards_local * (K + kTopkEqMax);
    count_launch();  // run_rank_kernel (the sort launch is counted above)
    run_rank_kernel<<<sgrid, kSortThreads, 0, s>>>(K, cand_tmp, runs, totals_out);
    sort_kernel<true><<<sgrid, kSortThreads, 0, s>>>(K, first_shard, runs, cand_out, totals_out,
                                                     state, mbox ? *mbox : Mbox{}, mbox != nullptr);
  }
  return cudaGetLastError();
}

}  // namespace gear
