// topk.cu -- decentralised TopK selection ("GEAR provides
// FIFO and TopK selection implementation, which are deterministic in
// decentralized selection scenarios ... all servers can perform a local scan
// to generate k samples before the global gathering").  Reading Q20: the
// K = W*B selectable trajectories with the largest keys, ties by the smaller
// global id, in that order.
//
// Local step, one CTA per local shard:
//  1. count the selectable keys and their maximum (block reduction);
//  2. if more than K are selectable, radix-select the K-th largest key: one
//     256-bin shared-memory histogram pass per byte of the key, from the
//     highest non-zero byte down, keeping only keys that match the prefix
//     chosen so far -- this yields the threshold key T* and how many keys
//     equal to T* are needed;
//  3. compact, in slot order, the keys > T* and the first needed keys == T*
//     (block ballot scan), into shared memory;
//  4. bitonic-sort the <= K candidates by (key desc, slot asc) in shared
//     memory and write them (with W > 1 also into every peer's mailbox).
// The global merge is the FIFO/LIFO merge with the TopK order (fifo.cu).
#include "mbox.cuh"

namespace gear {

namespace {

constexpr int kThreads = 1024;
constexpr int kWarps = kThreads / 32;

__device__ __forceinline__ uint32_t block_sum_u32(uint32_t v, uint32_t* s_red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(kFull, v, d);
  if (lane == 0) s_red[warp] = v;
  __syncthreads();
  uint32_t t = 0;
  for (int w = 0; w < kWarps; ++w) t += s_red[w];
  __syncthreads();
  return t;
}

// Candidate order of TopK: larger key first, then smaller slot.
__device__ __forceinline__ bool before(const Cand& a, const Cand& b) {
  return a.seq > b.seq || (a.seq == b.seq && a.slot < b.slot);
}

__global__ void __launch_bounds__(kThreads)
    topk_local_kernel(const uint64_t* __restrict__ key, uint64_t shard_cap, uint32_t first_shard,
                      uint32_t K, uint32_t Kpow2, Cand* __restrict__ cand_out,
                      ShardTotals* __restrict__ totals_out, const __grid_constant__ Mbox m0,
                      int xchg) {
  extern __shared__ __align__(16) Cand s_sel[];  // [Kpow2]
  __shared__ uint32_t s_hist[256];
  __shared__ uint32_t s_red[kWarps];
  __shared__ unsigned long long s_max;
  __shared__ uint32_t s_digit, s_need, s_count;
  const Mbox m = xchg ? mbox_at_next_epoch(m0) : m0;  // the FIFO/TopK epoch advances later
  const uint32_t ls = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t* k = key + (uint64_t)ls * shard_cap;
  const uint32_t shard = first_shard + ls;

  // 1. selectable count and maximum key
  if (tid == 0) s_max = 0;
  __syncthreads();
  uint32_t cnt = 0;
  unsigned long long mx = 0;
  for (uint64_t i = tid; i < shard_cap; i += kThreads) {
    const uint64_t x = k[i];
    cnt += x > 0;
    mx = x > mx ? x : mx;
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    const unsigned long long o = __shfl_xor_sync(kFull, mx, d);
    mx = o > mx ? o : mx;
  }
  if (lane == 0) atomicMax(&s_max, mx);
  const uint32_t n_sel = block_sum_u32(cnt, s_red);

  // 2. radix select of the K-th largest key (only if needed)
  uint64_t thr = 1, mask = 0;  // select keys > thr, plus `need` keys == thr
  uint32_t need = 0;
  if (n_sel > K) {
    uint32_t kk = K;  // rank of the wanted key among the keys matching the prefix
    uint64_t prefix = 0;
    const int top = s_max ? 63 - __clzll(s_max) : 0;
    for (int shift = (top / 8) * 8; shift >= 0; shift -= 8) {
      for (int b = tid; b < 256; b += kThreads) s_hist[b] = 0;
      __syncthreads();
      for (uint64_t i = tid; i < shard_cap; i += kThreads) {
        const uint64_t x = k[i];
        if (x > 0 && (x & mask) == prefix) atomicAdd(&s_hist[(x >> shift) & 255], 1u);
      }
      __syncthreads();
      if (tid == 0) {  // walk the digits from the top
        uint32_t above = 0;
        int v = 255;
        for (; v > 0; --v) {
          if (above + s_hist[v] >= kk) break;
          above += s_hist[v];
        }
        s_digit = (uint32_t)v;
        s_need = kk - above;
      }
      __syncthreads();
      prefix |= (uint64_t)s_digit << shift;
      mask |= 255ull << shift;
      kk = s_need;
      __syncthreads();
    }
    thr = prefix;  // the K-th largest key
    need = kk;     // how many keys equal to thr complete the K
  }
  const bool all = n_sel <= K;

  // 3. stable compaction in slot order into shared memory
  if (tid == 0) s_count = 0;
  uint32_t eq_seen = 0;  // keys == thr passed so far (block-uniform)
  __syncthreads();
  for (uint64_t i0 = 0; i0 < shard_cap; i0 += kThreads) {
    const uint64_t i = i0 + tid;
    const uint64_t x = i < shard_cap ? k[i] : 0;
    const bool gt = all ? x > 0 : x > thr;
    const bool eq = !all && x == thr && x > 0;
    const unsigned mg = __ballot_sync(kFull, gt), me = __ballot_sync(kFull, eq);
    if (lane == 0) s_red[warp] = (__popc(me) << 16) | __popc(mg);
    __syncthreads();
    uint32_t gt_before = 0, eq_before = 0, eq_total = 0, gt_total = 0;
    for (int w = 0; w < kWarps; ++w) {
      const uint32_t c = s_red[w];
      if (w < warp) {
        gt_before += c & 0xffff;
        eq_before += c >> 16;
      }
      gt_total += c & 0xffff;
      eq_total += c >> 16;
    }
    const uint32_t lt = (1u << lane) - 1u;
    const uint32_t my_eq = eq_seen + eq_before + __popc(me & lt);
    const bool take_eq = eq && my_eq < need;
    // position = #taken before me in slot order
    const uint32_t eq_taken_before =
        min(need, eq_seen + eq_before + __popc(me & lt)) - min(need, eq_seen);
    const uint32_t base = s_count;
    if (gt || take_eq) {
      Cand c;
      c.seq = x;
      c.shard = shard;
      c.slot = (uint32_t)i;
      s_sel[base + gt_before + __popc(mg & lt) + eq_taken_before] = c;
    }
    __syncthreads();
    if (tid == 0) s_count = base + gt_total + (min(need, eq_seen + eq_total) - min(need, eq_seen));
    eq_seen += eq_total;
    __syncthreads();
  }
  const uint32_t n = s_count;  // == min(K, n_sel)
  for (uint32_t i = n + tid; i < Kpow2; i += kThreads) {  // sentinels sort last
    Cand c;
    c.seq = 0;
    c.shard = 0;
    c.slot = 0xffffffffu;
    s_sel[i] = c;
  }
  __syncthreads();

  // 4. bitonic sort of Kpow2 entries: (key desc, slot asc)
  for (uint32_t size = 2; size <= Kpow2; size <<= 1) {
    for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
      for (uint32_t i = tid; i < Kpow2; i += kThreads) {
        const uint32_t j = i ^ stride;
        if (j > i) {
          const bool asc = (i & size) == 0;  // "ascending" in the `before` order
          const Cand a = s_sel[i], b = s_sel[j];
          if (asc ? before(b, a) : before(a, b)) {
            s_sel[i] = b;
            s_sel[j] = a;
          }
        }
      }
      __syncthreads();
    }
  }
  Cand* out = cand_out + (uint64_t)ls * K;
  for (uint32_t i = tid; i < n; i += kThreads) out[i] = s_sel[i];
  if (tid == 0) {
    ShardTotals t;
    t.total_and_parity = 0;
    t.aux = n;
    totals_out[ls] = t;
  }
  if (!xchg) return;
  // W > 1: push the sorted list and its length into every peer's mailbox.
  const MboxLayout L = mbox_layout(m.W, m.S, m.MB);
  const uint32_t b = mbox_buf(m);
  for (uint32_t r = 0; r < m.W; ++r) {
    Cand* dst = mbox_at<Cand>(m, r, L.cand) + ((uint64_t)b * m.S + shard) * K;
    for (uint32_t i = tid; i < n; i += kThreads) dst[i] = s_sel[i];
    if (tid == 0) {
      ShardTotals t;
      t.total_and_parity = 0;
      t.aux = n;
      mbox_at<ShardTotals>(m, r, L.ccnt)[b * m.S + shard] = t;
    }
  }
  __syncthreads();
  if (tid == 0) {
    __threadfence_system();
    for (uint32_t r = 0; r < m.W; ++r)
      st_release_sys_u64(mbox_at<uint64_t>(m, r, L.cflag) + b * m.S + shard, m.epoch);
  }
}

}  // namespace

uint32_t topk_max_k() { return 8192; }

cudaError_t launch_topk_local(const uint64_t* key, uint64_t shard_cap, uint32_t n_shards_local,
                              uint32_t first_shard, uint32_t K, Cand* cand_out,
                              ShardTotals* totals_out, const Mbox* mbox, cudaStream_t s) {
  uint32_t Kpow2 = 1;
  while (Kpow2 < K) Kpow2 <<= 1;
  const size_t smem = (size_t)Kpow2 * sizeof(Cand);
  static size_t configured = 0;
  if (smem > configured) {
    cudaError_t e = cudaFuncSetAttribute(topk_local_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)(smem < 48 * 1024 ? 48 * 1024 : smem));
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  count_launch();
  topk_local_kernel<<<n_shards_local, kThreads, smem, s>>>(key, shard_cap, first_shard, K, Kpow2,
                                                           cand_out, totals_out,
                                                           mbox ? *mbox : Mbox{}, mbox != nullptr);
  return cudaGetLastError();
}

}  // namespace gear
