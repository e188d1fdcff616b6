// scan.cu -- K1: the CDF of each shard as a single-pass u64 inclusive scan
// with decoupled look-back ("computes a prefix sum array using
// the decoupled look-back algorithm").
//
// Layout: a rank's R shards are contiguous in `key` (R * C_s u64); tile t of
// the launch covers kTile keys of shard t / tiles_per_shard.  Tile ids come
// from an atomic ticket so a tile only ever waits on tiles that already run
// (forward progress).  Each tile publishes one 64-bit status word: the top
// two bits are the flag (0 = not ready, 1 = aggregate, 2 = inclusive prefix)
// and the low 62 bits the value -- the keys are capped so every shard total
// is < 2^62 (gear.h q_max), so flag and value travel in one relaxed 64-bit
// store and need no fence.  Integer addition is associative, so the result is
// bit-identical to a sequential sum whatever the tiling.
//
// Memory path: the tile is moved HBM -> shared memory with coalesced 16-byte
// loads and back with coalesced 16-byte stores; threads own 16 consecutive
// keys in a padded shared layout (one u64 of padding per 16, conflict-free
// per half-warp).  The last tile to finish its look-back (done counter)
// clears the status words, the ticket and the counter, so every launch starts
// from the same state and the launch can be replayed from a CUDA graph.
#include "common.cuh"

namespace gear {

namespace {

constexpr int kThreads = 256;
constexpr int kItems = 16;                  // keys per thread
constexpr int kTile = kThreads * kItems;    // 4096 keys = 32 KB per tile
constexpr uint64_t kFlagA = 1ull << 62;
constexpr uint64_t kFlagP = 2ull << 62;
constexpr uint64_t kValMask = (1ull << 62) - 1;

__device__ __forceinline__ int pad(int e) { return e + (e >> 4); }

template <bool kIndicator>
__global__ void __launch_bounds__(kThreads) scan_kernel(
    const uint64_t* __restrict__ key, uint64_t* __restrict__ cdf0, uint64_t* __restrict__ cdf1,
    uint64_t shard_cap, uint32_t tiles_per_shard, uint32_t n_tiles, uint64_t* par_dev,
    ShardTotals* totals, uint64_t* status, uint32_t* ticket, uint32_t* done) {
  // The CDF is rebuilt into the buffer peers are NOT reading: the parity of
  // the last build lives in device memory (graph-replayable) and is flipped
  // by the last tile; the parity travels with the shard totals.
  const uint32_t parity = (uint32_t)(ld_relaxed_u64(par_dev) & 1) ^ 1u;
  uint64_t* __restrict__ cdf = parity ? cdf1 : cdf0;
  __shared__ uint64_t s_k[kTile + kTile / 16];
  __shared__ uint32_t s_tile;
  __shared__ uint64_t s_warp[kThreads / 32];
  __shared__ uint64_t s_excl;
  __shared__ bool s_last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  if (tid == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const uint32_t t = s_tile;
  const uint32_t shard = t / tiles_per_shard;
  const uint32_t tt = t - shard * tiles_per_shard;
  const uint64_t tile_begin = (uint64_t)tt * kTile;                   // within shard
  const uint64_t gbase = (uint64_t)shard * shard_cap + tile_begin;    // within key[]
  const uint32_t count = (uint32_t)min((uint64_t)kTile, shard_cap - tile_begin);
  const bool vec = count == (uint32_t)kTile && (gbase & 1) == 0;

  // HBM -> shared, coalesced.
  if (vec) {
    const ulonglong2* src = reinterpret_cast<const ulonglong2*>(key + gbase);
#pragma unroll
    for (int it = 0; it < kItems / 2; ++it) {
      const int vi = it * kThreads + tid;
      const ulonglong2 x = __ldg(src + vi);
      const int p = pad(2 * vi);
      s_k[p] = x.x;
      s_k[p + 1] = x.y;
    }
  } else {
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
      const int e = it * kThreads + tid;
      s_k[pad(e)] = (uint32_t)e < count ? key[gbase + e] : 0ull;
    }
  }
  __syncthreads();
  uint64_t v[kItems];
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const uint64_t x = s_k[tid * (kItems + 1) + i];
    v[i] = kIndicator ? (x > 0 ? 1ull : 0ull) : x;
  }
  // Thread-local inclusive prefix.
#pragma unroll
  for (int i = 1; i < kItems; ++i) v[i] += v[i - 1];
  // Warp and block scan of the thread totals.
  const uint64_t incl = warp_incl_scan_u64(v[kItems - 1], lane);
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  uint64_t warp_excl = 0, agg = 0;
#pragma unroll
  for (int w = 0; w < kThreads / 32; ++w) {
    const uint64_t x = s_warp[w];
    warp_excl += (w < warp) ? x : 0ull;
    agg += x;
  }
  const uint64_t thread_excl = warp_excl + incl - v[kItems - 1];

  // Publish the aggregate (or the inclusive prefix for a shard's first tile)
  // and look back over the predecessors of the same shard.
  if (warp == 0) {
    uint64_t excl = 0;
    if (tt == 0) {
      if (lane == 0) st_relaxed_u64(status + t, kFlagP | agg);
    } else {
      if (lane == 0) st_relaxed_u64(status + t, kFlagA | agg);
      const int64_t first = (int64_t)t - (int64_t)tt;  // shard's first tile
      int64_t pred = (int64_t)t - 1;
      while (true) {
        const int64_t idx = pred - lane;
        const bool valid = idx >= first;
        uint64_t s = valid ? ld_relaxed_u64(status + idx) : kFlagP;
        while (__any_sync(kFull, (s >> 62) == 0)) {
          if ((s >> 62) == 0) s = ld_relaxed_u64(status + idx);
        }
        const unsigned pmask = __ballot_sync(kFull, valid && (s >> 62) == 2);
        const uint64_t val = valid ? (s & kValMask) : 0ull;
        if (pmask) {
          const int lp = __ffs(pmask) - 1;  // closest inclusive predecessor
          uint64_t part = lane <= lp ? val : 0ull;
#pragma unroll
          for (int d = 16; d > 0; d >>= 1) part += __shfl_xor_sync(kFull, part, d);
          excl += part;
          break;
        }
        uint64_t part = val;
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) part += __shfl_xor_sync(kFull, part, d);
        excl += part;
        pred -= 32;
      }
      if (lane == 0) st_relaxed_u64(status + t, kFlagP | (excl + agg));
    }
    if (lane == 0) {
      s_excl = excl;
      // This tile no longer reads or writes status words: count it done.
      // The fence only has to drain the status store above (the CDF stores
      // come later), and the last tile to get here re-arms the status
      // words, the ticket and the counter after its stores.
      __threadfence();
      s_last = atomicAdd(done, 1u) == n_tiles - 1;
    }
  }
  __syncthreads();
  const uint64_t base = s_excl + thread_excl;
#pragma unroll
  for (int i = 0; i < kItems; ++i) s_k[tid * (kItems + 1) + i] = base + v[i];
  __syncthreads();

  // shared -> HBM, coalesced.
  if (vec) {
    ulonglong2* dst = reinterpret_cast<ulonglong2*>(cdf + gbase);
#pragma unroll
    for (int it = 0; it < kItems / 2; ++it) {
      const int vi = it * kThreads + tid;
      const int p = pad(2 * vi);
      dst[vi] = make_ulonglong2(s_k[p], s_k[p + 1]);
    }
  } else {
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
      const int e = it * kThreads + tid;
      if ((uint32_t)e < count) cdf[gbase + e] = s_k[pad(e)];
    }
  }
  if (tt == tiles_per_shard - 1 && tid == 0) {
    ShardTotals r;
    r.total_and_parity = (s_excl + agg) | ((uint64_t)parity << 63);
    r.aux = 0;
    totals[shard] = r;
  }
  if (s_last) {
    for (uint32_t i = tid; i < n_tiles; i += kThreads) status[i] = 0;
    if (tid == 0) {
      *ticket = 0;
      *done = 0;
      *par_dev = parity;  // every tile read the old parity before counting done
    }
  }
}

// Two-level CDF (NEXT-3, incremental): tile t of shard s holds the inclusive
// prefix of its own keys, L[i] = sum of the tile's keys up to i, and the
// shard holds P[t] = sum of the totals of tiles 0..t, so the flat CDF is
// C[t*kTile + i] = P[t-1] + L[i].  No look-back: tiles are independent.  A
// rebuild of buffer b rescans only the tiles whose dirty bit b is set (every
// key writer sets both bits of its tile), or every tile when the buffer was
// last built in the other mode (weights vs indicator); the last tile of each
// shard to arrive recomputes P from the tile totals, and the last shard flips
// the parity and records the buffer's mode.  Buffer layout: L of the R shards
// (R*C_s u64) followed by P of the R shards (R*tiles_per_shard u64).
template <bool kIndicator>
__global__ void __launch_bounds__(kThreads) scan2_kernel(
    const uint64_t* __restrict__ key, uint64_t* __restrict__ cdf0, uint64_t* __restrict__ cdf1,
    uint64_t shard_cap, uint32_t tiles_per_shard, uint32_t n_shards_local, uint64_t* par_dev,
    ShardTotals* totals, uint32_t* __restrict__ dirty, uint64_t* __restrict__ ttot0,
    uint64_t* __restrict__ ttot1, uint32_t* buf_mode, uint32_t* shard_ctr, uint32_t* done) {
  static_assert(kTile == (int)kCdfTile, "tile of the dirty map");
  const uint32_t t = blockIdx.x;
  // The four control words only change at kernel boundaries (the last CTA
  // writes parity and mode after every CTA has read them): one round trip.
  const uint64_t par_old = __ldcg(par_dev);
  const uint32_t mode0 = __ldcg(buf_mode), mode1 = __ldcg(buf_mode + 1);
  const uint32_t dirty_t = __ldcg(dirty + t);
  const uint32_t parity = (uint32_t)(par_old & 1) ^ 1u;
  uint64_t* __restrict__ cdf = parity ? cdf1 : cdf0;
  uint64_t* __restrict__ ttot = parity ? ttot1 : ttot0;  // this buffer's tile totals
  const uint32_t mode = kIndicator ? 2u : 1u;
  __shared__ uint64_t s_k[kTile + kTile / 16];
  __shared__ uint64_t s_warp[kThreads / 32];
  __shared__ bool s_last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t shard = t / tiles_per_shard;
  const uint32_t tt = t - shard * tiles_per_shard;
  const bool full = (parity ? mode1 : mode0) != mode;
  const uint32_t bit = 1u << parity;

  if (full || (dirty_t & bit)) {
    const uint64_t tile_begin = (uint64_t)tt * kTile;
    const uint64_t gbase = (uint64_t)shard * shard_cap + tile_begin;
    const uint32_t count = (uint32_t)min((uint64_t)kTile, shard_cap - tile_begin);
    const bool vec = count == (uint32_t)kTile && (gbase & 1) == 0;
    if (vec) {
      const ulonglong2* src = reinterpret_cast<const ulonglong2*>(key + gbase);
#pragma unroll
      for (int it = 0; it < kItems / 2; ++it) {
        const int vi = it * kThreads + tid;
        const ulonglong2 x = __ldg(src + vi);
        const int p = pad(2 * vi);
        s_k[p] = x.x;
        s_k[p + 1] = x.y;
      }
    } else {
#pragma unroll
      for (int it = 0; it < kItems; ++it) {
        const int e = it * kThreads + tid;
        s_k[pad(e)] = (uint32_t)e < count ? key[gbase + e] : 0ull;
      }
    }
    __syncthreads();
    uint64_t v[kItems];
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
      const uint64_t x = s_k[tid * (kItems + 1) + i];
      v[i] = kIndicator ? (x > 0 ? 1ull : 0ull) : x;
    }
#pragma unroll
    for (int i = 1; i < kItems; ++i) v[i] += v[i - 1];
    const uint64_t incl = warp_incl_scan_u64(v[kItems - 1], lane);
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    uint64_t warp_excl = 0, agg = 0;
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) {
      const uint64_t x = s_warp[w];
      warp_excl += (w < warp) ? x : 0ull;
      agg += x;
    }
    const uint64_t base = warp_excl + incl - v[kItems - 1];
#pragma unroll
    for (int i = 0; i < kItems; ++i) s_k[tid * (kItems + 1) + i] = base + v[i];
    __syncthreads();
    uint64_t* dst_l = cdf + gbase;
    if (vec) {
      ulonglong2* dst = reinterpret_cast<ulonglong2*>(dst_l);
#pragma unroll
      for (int it = 0; it < kItems / 2; ++it) {
        const int vi = it * kThreads + tid;
        const int p = pad(2 * vi);
        dst[vi] = make_ulonglong2(s_k[p], s_k[p + 1]);
      }
    } else {
#pragma unroll
      for (int it = 0; it < kItems; ++it) {
        const int e = it * kThreads + tid;
        if ((uint32_t)e < count) dst_l[e] = s_k[pad(e)];
      }
    }
    if (tid == 0) {
      ttot[t] = agg;
      dirty[t] = dirty_t & ~bit;
    }
  }
  // Arrival of this tile; the shard's last tile builds P.
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    s_last = atomicAdd(shard_ctr + shard, 1u) == tiles_per_shard - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // Level 2: P = inclusive prefix of this buffer's tile totals (rescanned
  // now or kept from this buffer's last build, in this buffer's mode), in
  // coalesced chunks of 4 totals per thread.
  uint64_t* P = cdf + (uint64_t)n_shards_local * shard_cap + (uint64_t)shard * tiles_per_shard;
  const uint64_t* tot = ttot + (uint64_t)shard * tiles_per_shard;
  uint64_t carry = 0;
  for (uint32_t c0 = 0; c0 < tiles_per_shard; c0 += 4 * kThreads) {
    uint64_t x[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t c = c0 + 4 * tid + k;
      x[k] = c < tiles_per_shard ? __ldcg(tot + c) : 0ull;
    }
    x[1] += x[0];
    x[2] += x[1];
    x[3] += x[2];
    const uint64_t incl = warp_incl_scan_u64(x[3], lane);
    __syncthreads();  // s_warp of the previous use consumed
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    uint64_t warp_excl = 0, agg = 0;
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) {
      const uint64_t y = s_warp[w];
      warp_excl += (w < warp) ? y : 0ull;
      agg += y;
    }
    const uint64_t base = carry + warp_excl + incl - x[3];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t c = c0 + 4 * tid + k;
      if (c < tiles_per_shard) P[c] = base + x[k];
    }
    carry += agg;
  }
  if (tid == 0) {
    ShardTotals r;
    r.total_and_parity = carry | ((uint64_t)parity << 63);
    r.aux = 0;
    totals[shard] = r;
    shard_ctr[shard] = 0;
    __threadfence();
    if (atomicAdd(done, 1u) == n_shards_local - 1) {  // every shard is built
      *done = 0;
      buf_mode[parity] = mode;
      *par_dev = parity;  // every tile read the old parity before arriving
    }
  }
}

}  // namespace

cudaError_t launch_scan2(const uint64_t* key, uint64_t* cdf0, uint64_t* cdf1, uint64_t shard_cap,
                         uint32_t n_shards_local, int indicator, uint64_t* par_dev,
                         ShardTotals* totals_out, uint32_t* dirty, uint64_t* ttot,
                         uint32_t* buf_mode, uint32_t* shard_ctr, uint32_t* done,
                         cudaStream_t s) {
  const uint32_t tps = scan_tiles_per_shard(shard_cap);
  const uint32_t n_tiles = tps * n_shards_local;
  count_launch();
  if (indicator)
    scan2_kernel<true><<<n_tiles, kThreads, 0, s>>>(key, cdf0, cdf1, shard_cap, tps,
                                                    n_shards_local, par_dev, totals_out, dirty,
                                                    ttot, ttot + n_tiles, buf_mode, shard_ctr,
                                                    done);
  else
    scan2_kernel<false><<<n_tiles, kThreads, 0, s>>>(key, cdf0, cdf1, shard_cap, tps,
                                                     n_shards_local, par_dev, totals_out, dirty,
                                                     ttot, ttot + n_tiles, buf_mode, shard_ctr,
                                                     done);
  return cudaGetLastError();
}

uint32_t scan_tiles_per_shard(uint64_t shard_cap) {
  return (uint32_t)((shard_cap + kTile - 1) / kTile);
}

cudaError_t launch_scan(const uint64_t* key, uint64_t* cdf0, uint64_t* cdf1, uint64_t shard_cap,
                        uint32_t n_shards_local, int indicator, uint64_t* par_dev,
                        ShardTotals* totals_out, uint64_t* status, uint32_t* ticket,
                        uint32_t* done, cudaStream_t s) {
  const uint32_t tps = scan_tiles_per_shard(shard_cap);
  const uint32_t n_tiles = tps * n_shards_local;
  count_launch();
  if (indicator)
    scan_kernel<true><<<n_tiles, kThreads, 0, s>>>(key, cdf0, cdf1, shard_cap, tps, n_tiles,
                                                   par_dev, totals_out, status, ticket, done);
  else
    scan_kernel<false><<<n_tiles, kThreads, 0, s>>>(key, cdf0, cdf1, shard_cap, tps, n_tiles,
                                                    par_dev, totals_out, status, ticket, done);
  return cudaGetLastError();
}

}  // namespace gear
