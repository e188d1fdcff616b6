// sample.cu -- K2/K3/K7: batched inverse-CDF sampling.
//
// "performs binary searching to locate the bins associated with
// uniformly generated random numbers".  One warp per draw j of the rank's
// slice [rank*B, rank*B + B) of the global batch:
//   r  = Philox4x32-10(counter j, key seed)            (64 bits)
//   u  = floor(r * T / 2^64), T = sum of the S shard totals (exact, mulhi)
//   s  = the shard whose exclusive offset range [G_s, G_s + T_s) holds u
//   i  = min{ i : cdf_s[i] > u - G_s }  -- 32-ary warp-cooperative search:
//        each round the 32 lanes probe 32 evenly spaced pivots of the live
//        range and a ballot keeps the first bin that can hold the answer, so
//        a shard of C_s keys takes ceil(log32 C_s) dependent rounds instead
//        of ceil(log2 C_s).  With the two-level CDF (default) the search runs
//        first over the shard's tile prefixes, then inside the chosen tile.
//        cdf_s may live in a peer GPU's HBM (read over NVLink through a
//        CUDA-IPC mapping).
//   g  = s*C_s + i,  q = cdf_s[i] - cdf_s[i-1]
// The IS weights (q_min/q)^beta need the min over the whole slice; the last
// block to finish (threadfence + counter) computes them and re-arms the
// counter and the min slot for the next launch.
#include "mbox.cuh"

namespace gear {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

// min{ i < n : c[i] > u } for a non-decreasing c with c[n-1] > u; also
// returns c[i] and c[i-1] (0 for i == 0).
__device__ __forceinline__ uint64_t search_bin(const uint64_t* __restrict__ c, uint64_t n,
                                               uint64_t u, int lane, uint64_t* c_at,
                                               uint64_t* c_prev) {
  uint64_t lo = 0, hi = n;  // answer in [lo, hi); c[hi-1] > u
  while (hi - lo > 32) {
    const uint64_t len = hi - lo;
    const uint64_t step = (len + 31) >> 5;
    uint64_t piv = lo + (uint64_t)(lane + 1) * step - 1;
    piv = piv > hi - 1 ? hi - 1 : piv;
    const bool gt = c[piv] > u;
    const unsigned m = __ballot_sync(kFull, gt);
    const int f = m ? __ffs(m) - 1 : 31;  // m == 0 only on a corrupt CDF: still terminates
    const uint64_t piv_f = __shfl_sync(kFull, piv, f);
    const uint64_t piv_b = __shfl_sync(kFull, piv, f > 0 ? f - 1 : 0);
    hi = piv_f + 1;
    lo = f > 0 ? piv_b + 1 : lo;
  }
  const uint64_t pos = lo + lane;
  const uint64_t cv = pos < hi ? c[pos] : ~0ull;
  const uint64_t before = (lane == 0 && lo > 0) ? c[lo - 1] : 0ull;
  const unsigned m = __ballot_sync(kFull, pos < hi && cv > u);
  const int f = m ? __ffs(m) - 1 : 0;
  const uint64_t cprev_lane = __shfl_sync(kFull, cv, f > 0 ? f - 1 : 0);
  const uint64_t cprev0 = __shfl_sync(kFull, before, 0);
  *c_at = __shfl_sync(kFull, cv, f);
  *c_prev = f > 0 ? cprev_lane : cprev0;
  return lo + (uint64_t)f;
}

// Bin of offset u within shard s (0 <= u < T_s); q = its weight.
//  levels 1: flat inclusive prefix C of the shard (decoupled look-back scan).
//  levels 2: tile prefixes P then the tile's own prefix L (scan2_kernel);
//            L_s sits at cdf, P_s after the R*C_s tile-local prefixes.
__device__ __forceinline__ uint64_t search_shard(const uint64_t* __restrict__ cdf,
                                                 const SampleParams& p, uint32_t s, uint64_t u,
                                                 int lane, uint64_t* q_out) {
  uint64_t at, prev;
  if (p.cdf_levels != 2) {
    const uint64_t i = search_bin(cdf, p.shard_cap, u, lane, &at, &prev);
    *q_out = at - prev;
    return i;
  }
  const uint64_t ls = s % p.shards_per_rank;
  const uint64_t tps = p.tiles_per_shard;
  const uint64_t* P = cdf - ls * p.shard_cap + (uint64_t)p.shards_per_rank * p.shard_cap + ls * tps;
  const uint64_t t = search_bin(P, tps, u, lane, &at, &prev);
  const uint64_t begin = t * kCdfTile;
  const uint64_t cnt = min((uint64_t)kCdfTile, p.shard_cap - begin);
  const uint64_t i = search_bin(cdf + begin, cnt, u - prev, lane, &at, &prev);
  *q_out = at - prev;
  return begin + i;
}

__global__ void __launch_bounds__(kThreads) sample_kernel(const __grid_constant__ SampleParams p) {
  __shared__ unsigned long long s_min[kWarps];
  __shared__ bool s_last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t b = blockIdx.x * kWarps + warp;
  const bool prioritized = p.strategy == kPrioritized;
  // Device seed counter (graph-replayable draws): read here, advanced by the
  // last block once every block has read it.
  uint64_t seed = p.seed;
  if (p.seed_dev != nullptr) seed = ld_relaxed_u64(p.seed_dev);  // asm: never hoisted

  // W > 1: every block publishes this rank's shard totals into every peer's
  // mailbox over NVLink and waits for all peers' (mbox.cuh).
  // xchg 2: the owner-affine assign kernel already exchanged them (and
  // advanced the epoch): read this rank's mailbox at the current epoch.
  const Mbox mm = p.xchg ? mbox_at_next_epoch(p.mbox) : p.mbox;
  const ShardTotals* totals = p.totals;
  if (p.xchg == 1) {
    totals = mbox_exchange_totals(mm, p.totals_local, p.err);
  } else if (p.xchg == 2) {
    const MboxLayout L = mbox_layout(mm.W, mm.S, mm.MB);
    totals = mbox_failed(p.err) ? nullptr
                                : mbox_at<ShardTotals>(mm, mm.rank, L.totals) + ((mm.epoch - 1) & 1) * mm.S;
  }
  // A timed-out exchange (totals == nullptr): no shard totals, so T = 0 and
  // every output is GEAR_IDX_NONE (kErrTimeout latched, not kErrEmpty).
  const bool failed = totals == nullptr;
  // Shard totals -> exclusive offsets (S <= 32: one lane per shard).
  const uint32_t S = p.n_shards;
  uint64_t Ts = 0;
  uint32_t par = 0;
  if ((uint32_t)lane < S && !failed) {
    const uint64_t tp = __ldcg(&totals[lane].total_and_parity);
    Ts = tp & ((1ull << 62) - 1);
    par = (uint32_t)(tp >> 63);
  }
  const uint64_t G = warp_incl_scan_u64(Ts, lane);
  const uint64_t T = __shfl_sync(kFull, G, 31);

  uint64_t my_q = ~0ull;
  if (b < p.B) {
    const uint64_t j = p.draw_list ? (uint64_t)p.draw_list[b] : (uint64_t)p.rank * p.B + b;
    uint64_t g = kIdxNone, q = 0;
    if (T > 0) {
      const uint64_t r = draw_bits(seed, j);
      const uint64_t u = __umul64hi(r, T);
      const unsigned own = __ballot_sync(kFull, (uint32_t)lane < S && G > u);
      const int s = __ffs(own) - 1;
      const uint64_t Gs_incl = __shfl_sync(kFull, G, s);
      const uint64_t Ts_s = __shfl_sync(kFull, Ts, s);
      const uint32_t par_s = __shfl_sync(kFull, par, s);
      const uint64_t* cdf = p.cdf_ptrs[(uint64_t)par_s * S + s];
      const uint64_t i = search_shard(cdf, p, (uint32_t)s, u - (Gs_incl - Ts_s), lane, &q);
      g = (uint64_t)s * p.shard_cap + i;
      if (lane == 0) {
        if (p.out_gen) {
          const uint32_t r_owner = (uint32_t)s / p.shards_per_rank;
          const uint64_t local = (uint64_t)(s % p.shards_per_rank) * p.shard_cap + i;
          p.out_gen[b] = p.gen_ptrs[r_owner][local];
        }
      }
    } else if (lane == 0) {
      if (!failed) atomicOr(p.err, kErrEmpty);
      if (p.out_gen) p.out_gen[b] = 0;
    }
    if (lane == 0) {
      p.out_idx[b] = g;
      if (p.out_p) p.out_p[b] = T > 0 ? (double)q / (double)T : 0.0;
      if (p.out_w && !prioritized) p.out_w[b] = T > 0 ? 1.0f : 0.0f;
      p.q_scratch[b] = q;
    }
    my_q = T > 0 ? q : ~0ull;
  }
  const bool need_w = prioritized && p.out_w != nullptr;
  const bool bump_epoch = p.xchg == 1;  // this kernel ran the exchange
  if (!need_w && !p.seed_dev && !bump_epoch) return;

  // Slice-wide q_min, then the last block writes the weights (and advances
  // the device seed counter).
  if (lane == 0) s_min[warp] = my_q;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long m = ~0ull;
    for (int w = 0; w < kWarps; ++w) m = s_min[w] < m ? s_min[w] : m;
    if (need_w) atomicMin(p.qmin_slot, m);
    __threadfence();
    const uint32_t done = atomicAdd(p.done_ctr, 1u);
    s_last = (done == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (need_w) {
    const unsigned long long qmin = *(volatile unsigned long long*)p.qmin_slot;
    for (uint32_t k = threadIdx.x; k < p.B; k += kThreads) {
      const uint64_t q = *(volatile uint64_t*)(p.q_scratch + k);
      p.out_w[k] = (T > 0 && q > 0) ? (float)pow((double)qmin / (double)q, p.beta) : 0.0f;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    *p.qmin_slot = ~0ull;
    *p.done_ctr = 0;
    if (p.seed_dev) *p.seed_dev = seed + 1;
    if (bump_epoch) *p.mbox.epoch_dev = mm.epoch;  // every block has read it
  }
}

}  // namespace

cudaError_t launch_sample(const SampleParams& p, cudaStream_t s) {
  if (p.B == 0) return cudaSuccess;
  const uint32_t grid = (p.B + kWarps - 1) / kWarps;
  count_launch();
  sample_kernel<<<grid, kThreads, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace gear
