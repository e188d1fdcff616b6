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
#include <algorithm>
#include <cstdio>

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

// GEAR_SCAN_TL (A/B builds only): per-CTA timeline of the persistent scans,
// %globaltimer (ns) at entry, at the phase boundaries and at exit, printed by
// every 8th CTA.
#ifdef GEAR_SCAN_TL
__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define TL_DECL uint64_t tl_[4] = {gtimer(), 0, 0, 0};
#define TL_MARK(i) do { if (tl_[i] == 0) tl_[i] = gtimer(); } while (0)
#define TL_PRINT(name) do { if (threadIdx.x == 0 && blockIdx.x % 8 == 0) { unsigned sm_; \
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm_)); \
    printf("TL %s cta %u sm %u %llu %llu %llu %llu\n", name, blockIdx.x, sm_, tl_[0], tl_[1], tl_[2], gtimer()); } } while (0)
#else
#define TL_DECL
#define TL_MARK(i) do {} while (0)
#define TL_PRINT(name) do {} while (0)
#endif

// Persistent, software-pipelined decoupled look-back scan.
//
// kScanCtasPerSm CTAs per SM stay resident and claim 4096-key tiles from an
// atomic ticket, one per iteration.  Iteration n of a CTA:
//   1. issues the look-back loads for its PREVIOUS tile n-1 (block-wide: each
//      thread polls kScanLookPer status words, a window of 512 predecessors
//      per L2 round trip),
//   2. claims tile n+1 and starts its TMA bulk load (cp.async.bulk +
//      mbarrier) into the buffer freed by tile n-2's bulk store,
//   3. waits for tile n's data, scans it in shared memory (tile-local
//      inclusive prefix, in place) and publishes its aggregate,
//   4. consumes the look-back loads of tile n-1 (re-polling words that are
//      not published yet), publishes its inclusive prefix, adds the prefix to
//      tile n-1's local prefixes and writes it out with a bulk store.
// So the L2 round trips of tile n-1's look-back overlap the scan of tile n,
// and by the time they are consumed every predecessor has published: the
// tiles being resolved (round j-1) only need the aggregates of their own
// round and the inclusive prefixes of round j-2, published one iteration
// earlier.  A tile waits only on tiles with smaller tickets, which running
// CTAs hold and publish in ticket order (forward progress).  The look-back of
// a tile that holds the shard's first tile is empty (prefix 0).
//
// Round 1's kernel (one CTA per tile, warp-0 look-back after the scan)
// stalled 7 of 8 warps at the barrier behind a 1.2 us L2 round trip per
// poll: 0.38 of the HBM copy peak.
//
// Shared layout: a tile is kTile consecutive u64 as the bulk copy lands it;
// thread i owns elements [16i, 16i+16) and touches them in the rotated order
// (k + i) mod 16, conflict-free per half-warp for 64-bit accesses.
#ifndef GEAR_STATUS_STRIDE
#define GEAR_STATUS_STRIDE 16
#endif
constexpr int kStatusStride = GEAR_STATUS_STRIDE;  // u64 words between two tiles' status words
constexpr int kScanBufs = 3;
constexpr int kScanCtasPerSm = 2;
#ifndef GEAR_SCAN_LOOK_PER
#define GEAR_SCAN_LOOK_PER 1
#endif
constexpr int kScanLookPer = GEAR_SCAN_LOOK_PER;
constexpr uint32_t kNoTile = 0xffffffffu;

template <bool kIndicator>
__global__ void __launch_bounds__(kThreads, kScanCtasPerSm) scan_kernel(
    const uint64_t* __restrict__ key, uint64_t* __restrict__ cdf0, uint64_t* __restrict__ cdf1,
    uint64_t shard_cap, uint32_t tiles_per_shard, uint32_t n_tiles, uint64_t* par_dev,
    ShardTotals* totals, uint64_t* status0, uint64_t* status1, uint32_t* ticket, uint32_t* done) {
  extern __shared__ __align__(128) uint64_t s_buf[];  // kScanBufs * kTile
  __shared__ __align__(8) uint64_t s_bar[kScanBufs];
  __shared__ uint32_t s_t[kScanBufs];    // ticket held by each buffer
  __shared__ uint32_t s_tma[kScanBufs];  // 1: the buffer's tile arrives by TMA
  __shared__ uint32_t s_shard[kScanBufs], s_tt[kScanBufs], s_count[kScanBufs];
  __shared__ uint64_t s_gbase[kScanBufs];  // each buffer's tile geometry
  __shared__ uint64_t s_agg[kScanBufs];  // each buffer's tile aggregate
  __shared__ uint64_t s_red[kThreads / 32];   // scan: warp totals
  __shared__ uint64_t s_part[kScanLookPer][kThreads / 32];  // look-back: warp sums up to its first P
  __shared__ uint32_t s_pmask[kScanLookPer][kThreads / 32];
  __shared__ bool s_last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  TL_DECL
  // The CDF is rebuilt into the buffer peers are NOT reading: the parity of
  // the last build lives in device memory (graph-replayable) and is flipped
  // by the last CTA to exit; the parity travels with the shard totals.
  const uint32_t parity = (uint32_t)(ld_relaxed_u64(par_dev) & 1) ^ 1u;
  uint64_t* __restrict__ cdf = parity ? cdf1 : cdf0;
  // Status words: launches of this kernel alternate between two arrays (the
  // scan epoch in ticket[1], advanced by the last CTA): this launch uses one
  // and clears the other -- the previous launch's -- for the next launch.
  const uint32_t epoch = *(volatile uint32_t*)(ticket + 1);
  uint64_t* __restrict__ status = (epoch & 1) ? status1 : status0;
  {
    uint64_t* other = (epoch & 1) ? status0 : status1;
    for (uint32_t i = blockIdx.x * kThreads + tid; i < n_tiles; i += gridDim.x * kThreads)
      other[(uint64_t)i * kStatusStride] = 0;
  }

  auto tile_geom = [&](uint32_t t, uint32_t* shard, uint32_t* tt, uint64_t* gbase,
                       uint32_t* count) {
    *shard = t / tiles_per_shard;
    *tt = t - *shard * tiles_per_shard;
    const uint64_t tb = (uint64_t)*tt * kTile;
    *gbase = (uint64_t)*shard * shard_cap + tb;
    *count = (uint32_t)min((uint64_t)kTile, shard_cap - tb);
  };
  // thread 0: give buffer b ticket t, cache the tile's geometry and start
  // its bulk load
  auto claim_t = [&](int b, uint32_t t) {
    s_t[b] = t < n_tiles ? t : kNoTile;
    s_tma[b] = 0;
    if (t >= n_tiles) return;
    uint32_t sh, tt, count;
    uint64_t gb;
    tile_geom(t, &sh, &tt, &gb, &count);
    s_shard[b] = sh;
    s_tt[b] = tt;
    s_count[b] = count;
    s_gbase[b] = gb;
    if (count == (uint32_t)kTile && (gb & 1) == 0) {
      s_tma[b] = 1;
      bulk_g2s(smem_u32(s_buf + (size_t)b * kTile), key + gb, kTile * 8, smem_u32(&s_bar[b]));
    }
  };
  // ... with the prefetched ticket, prefetching the next one (the atomic's
  // round trip is consumed one iteration later, off the critical path; it is
  // issued after the previous result was used, so tickets grow)
  uint32_t next_ticket = 0;
  auto claim = [&](int b) {
    const uint32_t t = next_ticket;
    claim_t(b, t);
    next_ticket = atomicAdd(ticket, 1u);
  };
  // Look-back loads of the tile in buffer b (window at distances 1 + tid + 256k).
  auto poll = [&](int b, int64_t pred, uint64_t* st) {
    const int64_t first = (int64_t)s_t[b] - (int64_t)s_tt[b];
#pragma unroll
    for (int k = 0; k < kScanLookPer; ++k) {
      const int64_t idx = pred - tid - (int64_t)k * kThreads;
      st[k] = idx >= first ? ld_relaxed_u64(status + idx * kStatusStride) : kFlagP;
    }
  };
  if (tid == 0) {
    for (int b = 0; b < kScanBufs; ++b) {
      mbar_init(smem_u32(&s_bar[b]), 1);
      s_t[b] = kNoTile;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const uint32_t t0 = atomicAdd(ticket, 2u);  // two tickets in one round trip
    claim_t(0, t0);
    claim_t(1, t0 + 1);
    next_ticket = atomicAdd(ticket, 1u);
  }
  __syncthreads();

  uint32_t phase = 0;  // bit b: parity of buffer b's mbarrier
#ifdef GEAR_SCAN_PROF
  uint64_t pr[8] = {0, 0, 0, 0, 0, 0, 0, 0}, pt = clock64(), iters = 0, polls = 0;
#define PROF(i) do { const uint64_t c_ = clock64(); pr[i] += c_ - pt; pt = c_; } while (0)
#else
#define PROF(i) do {} while (0)
#endif
  for (uint32_t n = 0;; ++n) {
    const int b = (int)(n % kScanBufs);
    const int bp = (int)((n + kScanBufs - 1) % kScanBufs);  // tile n-1 (pending prefix)
    const int bn = (int)((n + 1) % kScanBufs);              // tile n+1 (in flight)
    const uint32_t t = s_t[b];
    const uint32_t tp = n >= 1 ? s_t[bp] : kNoTile;
    // 1. the look-back loads of tile n-1 fly while tile n is scanned
    uint64_t st[kScanLookPer];
    if (tp != kNoTile) poll(bp, (int64_t)tp - 1, st);
    PROF(0);
    // 2. scan tile n in place (tile-local inclusive prefix) and publish it
    if (t != kNoTile) {
      const uint32_t tt = s_tt[b], count = s_count[b];
      const uint64_t gbase = s_gbase[b];
      uint64_t* buf = s_buf + (size_t)b * kTile;
      if (s_tma[b]) {
        while (!mbar_try_wait(smem_u32(&s_bar[b]), (phase >> b) & 1u)) {
        }
        phase ^= 1u << b;
      } else {  // a ragged or unaligned tile: plain loads, zero-padded
        for (int e = tid; e < kTile; e += kThreads)
          buf[e] = (uint32_t)e < count ? key[gbase + e] : 0ull;
        __syncthreads();
      }
      PROF(1);
      // thread i owns the 8 pairs [16i + 2j, 16i + 2j + 1] and visits them in
      // the rotated order j = (k + r) mod 8, r = i mod 8 (128-bit accesses,
      // conflict-free per quarter-warp); S_k = prefix over the visited pairs,
      // and the natural prefix of pair j = (k + r) mod 8 is
      // S_k - S_{7-r} + (k < 8 - r ? total : 0)
      const int r = tid & 7;
      ulonglong2* b2 = reinterpret_cast<ulonglong2*>(buf) + tid * (kItems / 2);
      uint64_t lo[kItems / 2], hi[kItems / 2];
#pragma unroll
      for (int k = 0; k < kItems / 2; ++k) {
        const ulonglong2 x = b2[(k + r) & 7];
        lo[k] = kIndicator ? (x.x > 0 ? 1ull : 0ull) : x.x;
        hi[k] = kIndicator ? (x.y > 0 ? 1ull : 0ull) : x.y;
      }
      uint64_t run = 0;
#pragma unroll
      for (int k = 0; k < kItems / 2; ++k) {
        lo[k] += run;
        hi[k] += lo[k];
        run = hi[k];
      }
      const uint64_t total = run;
      uint64_t s_rot = 0;
#pragma unroll
      for (int k = 0; k < kItems / 2; ++k) s_rot = (k == 7 - r) ? hi[k] : s_rot;
      const uint64_t incl = warp_incl_scan_u64(total, lane);
      if (lane == 31) s_red[warp] = incl;  // (last read before the previous end-of-iteration barrier)
      __syncthreads();
      uint64_t warp_excl = 0, agg = 0;
#pragma unroll
      for (int w = 0; w < kThreads / 32; ++w) {
        const uint64_t x = s_red[w];
        warp_excl += (w < warp) ? x : 0ull;
        agg += x;
      }
      const uint64_t base = warp_excl + incl - total;
#pragma unroll
      for (int k = 0; k < kItems / 2; ++k) {
        const uint64_t off = base - s_rot + (k < 8 - r ? total : 0ull);
        b2[(k + r) & 7] = make_ulonglong2(lo[k] + off, hi[k] + off);
      }
      if (tid == 0) {
        s_agg[b] = agg;
        // a shard's first tile: its aggregate IS its inclusive prefix
        st_relaxed_u64(status + (uint64_t)t * kStatusStride, (tt == 0 ? kFlagP : kFlagA) | agg);
      }
    }
    PROF(2);
    // 3. resolve tile n-1: consume the look-back, publish, add, store
    if (tp != kNoTile) {
      const uint32_t shard = s_shard[bp], tt = s_tt[bp], count = s_count[bp];
      const uint64_t gbase = s_gbase[bp];
      uint64_t excl = 0;
      if (tt != 0) {
        int64_t pred = (int64_t)tp - 1;
        while (true) {
#pragma unroll
          for (int k = 0; k < kScanLookPer; ++k) {
            const int64_t idx = pred - tid - (int64_t)k * kThreads;
            while ((st[k] >> 62) == 0) {
              st[k] = ld_relaxed_u64(status + idx * kStatusStride);
#ifdef GEAR_SCAN_PROF
              ++polls;
#endif
            }
          }
          PROF(6);
          // closest inclusive prefix: the smallest distance tid + 256k with a
          // P flag.  ONE block barrier: every warp publishes its ballot and the
          // sum of its values up to and including its own first P (all of them
          // if it has none); the combine walks the (word, warp) pairs in
          // distance order up to the first one with a P
#pragma unroll
          for (int k = 0; k < kScanLookPer; ++k) {
            const unsigned m = __ballot_sync(kFull, (st[k] >> 62) == 2);
            const int f = m ? __ffs(m) - 1 : 31;
            uint64_t v = lane <= f ? (st[k] & kValMask) : 0ull;
#pragma unroll
            for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(kFull, v, d);
            if (lane == 0) {
              s_pmask[k][warp] = m;
              s_part[k][warp] = v;
            }
          }
          __syncthreads();
          PROF(7);
          bool found = false;
#pragma unroll
          for (int k = 0; k < kScanLookPer; ++k)
#pragma unroll
            for (int w = 0; w < kThreads / 32; ++w)
              if (!found) {
                excl += s_part[k][w];
                found = s_pmask[k][w] != 0;
              }
          if (found) break;
          __syncthreads();  // s_pmask / s_part read before the next round
          pred -= (int64_t)kThreads * kScanLookPer;  // no prefix in this window
          poll(bp, pred, st);
        }
        if (tid == 0) st_relaxed_u64(status + (uint64_t)tp * kStatusStride, kFlagP | (excl + s_agg[bp]));
      }
      PROF(3);
      if (tt == tiles_per_shard - 1 && tid == 0) {
        ShardTotals rec;
        rec.total_and_parity = (excl + s_agg[bp]) | ((uint64_t)parity << 63);
        rec.aux = 0;
        totals[shard] = rec;
      }
      // out: prefix + local prefix, coalesced 16-byte stores straight from
      // registers (the buffer is free as soon as this pass has read it)
      const uint64_t* buf = s_buf + (size_t)bp * kTile;
      if (s_tma[bp]) {
        const ulonglong2* src = reinterpret_cast<const ulonglong2*>(buf);
        ulonglong2* dst = reinterpret_cast<ulonglong2*>(cdf + gbase);
#pragma unroll
        for (int k = 0; k < kItems / 2; ++k) {
          const ulonglong2 x = src[k * kThreads + tid];
          dst[k * kThreads + tid] = make_ulonglong2(x.x + excl, x.y + excl);
        }
      } else {
        for (int e = tid; e < (int)count; e += kThreads) cdf[gbase + e] = buf[e] + excl;
      }
    }
    PROF(4);
    __syncthreads();  // tile n-1's buffer read by every thread: free
    // 4. claim tile n+2 into tile n-1's buffer, just freed: its load has a
    //    whole iteration (tile n+1 is already in flight in the third buffer)
    if (tid == 0 && t != kNoTile) {
      if (s_t[bn] != kNoTile) claim(bp);
      else s_t[bp] = kNoTile;  // tickets only grow: nothing more for this CTA
    }
    // (s_t / s_tma of the claimed buffer are read two iterations from now,
    // after several barriers)
    PROF(5);
#ifdef GEAR_SCAN_PROF
    ++iters;
#endif
    if (t == kNoTile) break;  // tile n-1 was the last: done
  }
#ifdef GEAR_SCAN_PROF
  if (tid == 0 && (blockIdx.x % 37) == 0)
    printf("scanprof cta %u iters %llu cyc/iter: poll-issue %llu tma-wait %llu scan %llu resolve-spin %llu resolve-bar1 %llu resolve-rest %llu out %llu claim %llu polls %llu\n",
           blockIdx.x, iters, pr[0] / iters, pr[1] / iters, pr[2] / iters, pr[6] / iters, pr[7] / iters, pr[3] / iters,
           pr[4] / iters, pr[5] / iters, polls);
#endif
  TL_PRINT("tile");
  // The last CTA to exit re-arms the ticket and the exit counter and
  // publishes the new parity.
  if (tid == 0) {
    __threadfence();
    s_last = atomicAdd(done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (s_last) {
    if (tid == 0) {
      *ticket = 0;
      ticket[1] = epoch + 1;  // every CTA read the epoch before exiting
      *done = 0;
      *par_dev = parity;  // every CTA read the old parity before exiting
    }
  }
}

// Chunked decoupled look-back (K1c; `cdf_levels = 1` for mid-sized tables).
//
// The look-back runs over CHUNKS -- contiguous key ranges, one per resident
// CTA -- instead of 4096-key tiles, so it is resolved once per CTA instead of
// once per tile:
//   phase 1: stream the chunk's tiles (TMA, kCBufs ahead) and reduce each to
//            its tile sum; the last kCBufs tiles stay in shared memory;
//            publish the chunk aggregate (flag A; flag P for a shard's first
//            chunk) -- the same 64-bit flag+value status word as scan_kernel;
//   look-back: block-wide over up to 2 * kThreads predecessors per round trip
//            (every chunk of a shard is in flight at once, so the first
//            window normally reaches the shard's first chunk), publish P;
//   phase 2: scan the chunk's tiles in REVERSE order -- the resident ones
//            first, then the most recently streamed (still in L2 while the
//            table's keys are a fraction of the 126 MB L2), each tile's
//            prefix being the chunk prefix + the tile sums before it -- and
//            write each tile of the CDF with one bulk (TMA) store.
// DRAM traffic stays 8 B read + 8 B written per key as long as the keys
// re-read in phase 2 hit L2, and HBM sees a read phase and a write phase
// instead of a per-tile mix; the per-tile look-back pipeline of scan_kernel
// (and its fill / drain) is gone.  Chunk boundaries are key offsets rounded to
// 16 keys, so every CTA gets the same work (+- 16 keys); a chunk's last tile
// is ragged (masked).  Chunks are claimed from the ticket, so a chunk only
// waits on chunks that already run (forward progress), and the kernel shares
// scan_kernel's status arrays / epoch / ticket / exit counter protocol.
// Measured (profiles/r02_scan/chunk, final_full): 10 M keys 36 us under ncu
// (scan_kernel ~41), but at 40 M keys most of phase 2's re-read misses L2, so
// launch_scan picks this kernel only while the rank's keys are <= 96 MB.
#ifndef GEAR_CHUNK_BUFS
#define GEAR_CHUNK_BUFS 3
#endif
#ifndef GEAR_CHUNK_CTAS
#define GEAR_CHUNK_CTAS 2
#endif
#ifndef GEAR_CHUNKS_PER_CTA
#define GEAR_CHUNKS_PER_CTA 1
#endif
constexpr int kCBufs = GEAR_CHUNK_BUFS;
constexpr int kChunksPerCta = GEAR_CHUNKS_PER_CTA;  // chunks per CTA (a CTA's phase 1 overlaps others' phase 2)
constexpr int kChunkCtasPerSm = GEAR_CHUNK_CTAS;
constexpr int kMaxChunkTiles = 64;  // tile sums kept in shared memory

template <bool kIndicator>
__global__ void __launch_bounds__(kThreads, kChunkCtasPerSm) scan_chunk_kernel(
    const uint64_t* __restrict__ key, uint64_t* __restrict__ cdf0, uint64_t* __restrict__ cdf1,
    uint64_t shard_cap, uint32_t chunks_per_shard, uint32_t n_chunks, uint32_t n_status_clear,
    uint64_t* par_dev, ShardTotals* totals, uint64_t* status0, uint64_t* status1,
    uint32_t* ticket, uint32_t* done) {
  extern __shared__ __align__(128) uint64_t s_buf[];  // kCBufs * kTile
  __shared__ __align__(8) uint64_t s_bar[kCBufs];
  __shared__ uint64_t s_tsum[kMaxChunkTiles];  // phase 1: tile sums; phase 2: tile prefixes
  __shared__ uint64_t s_red[2][kThreads / 32];
  __shared__ uint32_t s_pmask[2][kThreads / 32];
  __shared__ uint64_t s_excl;
  __shared__ uint32_t s_chunk;
  __shared__ bool s_last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  TL_DECL
  const uint32_t parity = (uint32_t)(ld_relaxed_u64(par_dev) & 1) ^ 1u;
  uint64_t* __restrict__ cdf = parity ? cdf1 : cdf0;
  const uint32_t epoch = *(volatile uint32_t*)(ticket + 1);
  uint64_t* __restrict__ status = (epoch & 1) ? status1 : status0;
  {
    uint64_t* other = (epoch & 1) ? status0 : status1;
    for (uint32_t i = blockIdx.x * kThreads + tid; i < n_status_clear; i += gridDim.x * kThreads)
      other[(uint64_t)i * kStatusStride] = 0;
  }
  if (tid == 0) {
    for (int b = 0; b < kCBufs; ++b) mbar_init(smem_u32(&s_bar[b]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  uint32_t phase = 0;  // bit b: parity of buffer b's mbarrier

  while (true) {
    if (tid == 0) s_chunk = atomicAdd(ticket, 1u);
    __syncthreads();
    const uint32_t c = s_chunk;
    if (c >= n_chunks) break;
    const uint32_t shard = c / chunks_per_shard, ci = c - shard * chunks_per_shard;
    // chunk ci of the shard: keys [k0, k1), k0 rounded down to 16 keys
    const uint64_t k0 = ((uint64_t)ci * shard_cap / chunks_per_shard) & ~15ull;
    const uint64_t k1 = ci + 1 == chunks_per_shard
                            ? shard_cap
                            : (((uint64_t)(ci + 1) * shard_cap / chunks_per_shard) & ~15ull);
    const uint32_t nt = (uint32_t)((k1 - k0 + kTile - 1) / kTile);
    const uint64_t sbase = (uint64_t)shard * shard_cap;
    auto tcount = [&](uint32_t j) { return (uint32_t)min((uint64_t)kTile, k1 - k0 - (uint64_t)j * kTile); };
    auto is_tma = [&](uint32_t j) {
      return ((sbase + k0 + (uint64_t)j * kTile) & 1) == 0 && (tcount(j) & 1) == 0;
    };
    // thread 0: bulk load of tile j into its buffer j % kCBufs (L2 evict-last
    // hints on phase-1 loads / evict-first on phase-2 reloads were measured no
    // faster, profiles/r02_scan/chunk)
    auto issue = [&](uint32_t j) {
      if (!is_tma(j)) return;
      bulk_g2s(smem_u32(s_buf + (size_t)(j % kCBufs) * kTile), key + sbase + k0 + (uint64_t)j * kTile,
               tcount(j) * 8, smem_u32(&s_bar[j % kCBufs]));
    };
    // every thread: tile j is in its buffer (TMA wait, or plain zero-padded loads)
    auto land = [&](uint32_t j) {
      const int b = (int)(j % kCBufs);
      if (is_tma(j)) {
        while (!mbar_try_wait(smem_u32(&s_bar[b]), (phase >> b) & 1u)) {
        }
        phase ^= 1u << b;
      } else {
        uint64_t* buf = s_buf + (size_t)b * kTile;
        const uint64_t* src = key + sbase + k0 + (uint64_t)j * kTile;
        const uint32_t count = tcount(j);
        for (int e = tid; e < kTile; e += kThreads) buf[e] = (uint32_t)e < count ? src[e] : 0ull;
        __syncthreads();
      }
    };
    if (tid == 0)
      for (uint32_t j = 0; j < nt && j < (uint32_t)kCBufs; ++j) issue(j);

    // phase 1: tile sums
    for (uint32_t j = 0; j < nt; ++j) {
      land(j);
      const uint32_t count = tcount(j);
      const ulonglong2* b2 = reinterpret_cast<const ulonglong2*>(s_buf + (size_t)(j % kCBufs) * kTile);
      uint64_t sum = 0;
#pragma unroll
      for (int k = 0; k < kItems / 2; ++k) {
        const uint32_t e = 2u * (uint32_t)(k * kThreads + tid);
        const ulonglong2 x = b2[k * kThreads + tid];
        const uint64_t a = e < count ? x.x : 0ull, bb = e + 1 < count ? x.y : 0ull;
        sum += kIndicator ? (uint64_t)(a > 0) + (uint64_t)(bb > 0) : a + bb;
      }
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) sum += __shfl_xor_sync(kFull, sum, d);
      if (lane == 0) s_red[j & 1][warp] = sum;
      __syncthreads();  // buffer j % kCBufs read by every thread; s_red[j & 1] complete
      if (tid == 0) {
        uint64_t ts = 0;
#pragma unroll
        for (int w = 0; w < kThreads / 32; ++w) ts += s_red[j & 1][w];
        s_tsum[j] = ts;
        if (j + kCBufs < nt) issue(j + kCBufs);  // the last kCBufs tiles stay resident
      }
    }
    __syncthreads();  // s_tsum complete
    TL_MARK(1);
    // chunk aggregate -> status; tile sums -> tile-exclusive prefixes (thread 0)
    if (tid == 0) {
      uint64_t run = 0;
      for (uint32_t j = 0; j < nt; ++j) {
        const uint64_t x = s_tsum[j];
        s_tsum[j] = run;
        run += x;
      }
      st_relaxed_u64(status + (uint64_t)c * kStatusStride, (ci == 0 ? kFlagP : kFlagA) | run);
      s_excl = run;  // (aggregate, until the look-back below)
    }
    __syncthreads();
    const uint64_t agg = s_excl;
    // look-back over the shard's preceding chunks, 2 * kThreads per round
    uint64_t excl = 0;
    if (ci != 0) {
      const int64_t first = (int64_t)c - (int64_t)ci;
      int64_t pred = (int64_t)c - 1;
      while (true) {
        uint64_t st[2];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const int64_t idx = pred - tid - (int64_t)k * kThreads;
          st[k] = idx >= first ? ld_relaxed_u64(status + idx * kStatusStride) : kFlagP;
        }
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const int64_t idx = pred - tid - (int64_t)k * kThreads;
          while ((st[k] >> 62) == 0) st[k] = ld_relaxed_u64(status + idx * kStatusStride);
        }
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const unsigned m = __ballot_sync(kFull, (st[k] >> 62) == 2);
          if (lane == 0) s_pmask[k][warp] = m;
        }
        __syncthreads();
        uint32_t dp = 0xffffffffu;
#pragma unroll
        for (int k = 1; k >= 0; --k)
#pragma unroll
          for (int w = kThreads / 32 - 1; w >= 0; --w) {
            const unsigned m = s_pmask[k][w];
            if (m) dp = (uint32_t)(k * kThreads + w * 32 + __ffs(m) - 1);
          }
        uint64_t part = 0;
#pragma unroll
        for (int k = 0; k < 2; ++k)
          part += ((uint32_t)(tid + k * kThreads) <= dp) ? (st[k] & kValMask) : 0ull;
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) part += __shfl_xor_sync(kFull, part, d);
        if (lane == 0) s_red[0][warp] = part;
        __syncthreads();
#pragma unroll
        for (int w = 0; w < kThreads / 32; ++w) excl += s_red[0][w];
        __syncthreads();  // s_pmask / s_red read before their next use
        if (dp != 0xffffffffu) break;
        pred -= 2 * kThreads;  // no inclusive prefix in this window
      }
      if (tid == 0) st_relaxed_u64(status + (uint64_t)c * kStatusStride, kFlagP | (excl + agg));
    }
    if (tid == 0 && ci + 1 == chunks_per_shard) {
      ShardTotals rec;
      rec.total_and_parity = (excl + agg) | ((uint64_t)parity << 63);
      rec.aux = 0;
      totals[shard] = rec;
    }

    TL_MARK(2);
    // phase 2: tiles in reverse order; tile j - kCBufs is loaded into tile j's
    // buffer once tile j is written out
    const int r = tid & 7;
    for (int64_t jj = (int64_t)nt - 1; jj >= 0; --jj) {
      const uint32_t j = (uint32_t)jj;
      if (j + kCBufs < nt) land(j);  // reloaded (the resident ones landed in phase 1)
      const uint32_t count = tcount(j);
      uint64_t* buf = s_buf + (size_t)(j % kCBufs) * kTile;
      ulonglong2* b2 = reinterpret_cast<ulonglong2*>(buf) + tid * (kItems / 2);
      uint64_t lo[kItems / 2], hi[kItems / 2];
#pragma unroll
      for (int k = 0; k < kItems / 2; ++k) {
        const uint32_t e = (uint32_t)(tid * kItems + 2 * ((k + r) & 7));
        const ulonglong2 x = b2[(k + r) & 7];
        const uint64_t a = e < count ? x.x : 0ull, bb = e + 1 < count ? x.y : 0ull;
        lo[k] = kIndicator ? (a > 0 ? 1ull : 0ull) : a;
        hi[k] = kIndicator ? (bb > 0 ? 1ull : 0ull) : bb;
      }
      uint64_t run = 0;
#pragma unroll
      for (int k = 0; k < kItems / 2; ++k) {
        lo[k] += run;
        hi[k] += lo[k];
        run = hi[k];
      }
      const uint64_t total = run;
      uint64_t s_rot = 0;
#pragma unroll
      for (int k = 0; k < kItems / 2; ++k) s_rot = (k == 7 - r) ? hi[k] : s_rot;
      const uint64_t incl = warp_incl_scan_u64(total, lane);
      if (lane == 31) s_red[j & 1][warp] = incl;
      __syncthreads();
      uint64_t warp_excl = excl + s_tsum[j];  // chunk prefix + tile prefix
#pragma unroll
      for (int w = 0; w < kThreads / 32; ++w) warp_excl += (w < warp) ? s_red[j & 1][w] : 0ull;
      const uint64_t base = warp_excl + incl - total;
#pragma unroll
      for (int k = 0; k < kItems / 2; ++k) {
        const uint64_t off = base - s_rot + (k < 8 - r ? total : 0ull);
        b2[(k + r) & 7] = make_ulonglong2(lo[k] + off, hi[k] + off);
      }
      uint64_t* dst = cdf + sbase + k0 + (uint64_t)j * kTile;
      if (count == (uint32_t)kTile && ((sbase + k0) & 1) == 0) {
        // full aligned tile: one bulk store (smem -> global, UBLKCP) by thread
        // 0; no thread reads the buffer afterwards, so no barrier -- the
        // reload into this buffer waits until the store has read it (bulk
        // stores measured 3-14% faster than 16-B stores from every thread at
        // 5-20 M keys, profiles/r02_scan/chunk)
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();  // the tile's CDF is in shared memory (async proxy)
        if (tid == 0) {
          bulk_s2g(dst, smem_u32(buf), kTile * 8);
          if (j >= (uint32_t)kCBufs) {
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            issue(j - kCBufs);
          }
        }
        continue;
      }
      __syncthreads();  // the tile's CDF is in shared memory
      for (int e = tid; e < (int)count; e += kThreads) dst[e] = buf[e];  // ragged / unaligned
      __syncthreads();  // buffer read by every thread
      if (tid == 0 && j >= (uint32_t)kCBufs) issue(j - kCBufs);
    }
    // the next chunk's loads reuse the buffers: every bulk store has read them
    if (tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    __syncthreads();
  }
  if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  TL_PRINT("chunk");
  // The last CTA to exit re-arms the ticket and the exit counter and
  // publishes the new parity (as scan_kernel).
  if (tid == 0) {
    __threadfence();
    s_last = atomicAdd(done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (s_last && tid == 0) {
    *ticket = 0;
    ticket[1] = epoch + 1;
    *done = 0;
    *par_dev = parity;
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

// Persistent two-level rebuild (default for large shards; `scan2_kernel`,
// one CTA per tile, stays for small ones).  2 CTAs per SM; CTA b owns the
// tiles b, b + G, b + 2G, ...  It first reads the dirty words of its tiles
// (block-wide, in chunks of kThreads) and compacts the ones to rescan into a
// shared-memory work list, so a clean tile costs one coalesced word -- the
// incremental no-op of a 40 M-key table no longer launches 9766 CTAs.  Work
// tiles stream through three shared-memory buffers: TMA bulk loads
// (cp.async.bulk + mbarrier) two tiles ahead, the tile-local scan in place
// (the rotated 128-bit layout of scan_kernel), one TMA bulk store per tile
// (16-B stores from every thread for a ragged / unaligned tile).  Each
// CTA then adds its tiles to every shard's arrival counter in one atomic;
// the CTA that completes a shard builds that shard's prefix of tile totals,
// and the last shard flips the parity and records the buffer's mode, as in
// scan2_kernel.
#ifndef GEAR_S2_CTAS
#define GEAR_S2_CTAS 2
#endif
#ifndef GEAR_S2_BUFS
#define GEAR_S2_BUFS 3
#endif
constexpr int kS2Ctas = GEAR_S2_CTAS;  // scan2p CTAs per SM
constexpr int kS2Bufs = GEAR_S2_BUFS;  // scan2p tile buffers per CTA (loads kS2Bufs - 1 ahead)

template <bool kIndicator>
__global__ void __launch_bounds__(kThreads, kS2Ctas) scan2p_kernel(
    const uint64_t* __restrict__ key, uint64_t* __restrict__ cdf0, uint64_t* __restrict__ cdf1,
    uint64_t shard_cap, uint32_t tiles_per_shard, uint32_t n_shards_local, uint64_t* par_dev,
    ShardTotals* totals, uint32_t* __restrict__ dirty, uint64_t* __restrict__ ttot0,
    uint64_t* __restrict__ ttot1, uint32_t* buf_mode, uint32_t* shard_ctr, uint32_t* done) {
  static_assert(kTile == (int)kCdfTile, "tile of the dirty map");
  extern __shared__ __align__(128) uint64_t s_buf[];  // kS2Bufs * kTile
  __shared__ __align__(8) uint64_t s_bar[kS2Bufs];
  __shared__ uint32_t s_work[kThreads];   // work tiles of the current chunk
  __shared__ uint32_t s_wcnt[kThreads / 32];
  __shared__ uint32_t s_shcnt[kMaxShards];  // tiles of each shard this CTA covers
  __shared__ uint64_t s_red[kThreads / 32];
  __shared__ bool s_last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  TL_DECL
  const uint64_t par_old = __ldcg(par_dev);
  const uint32_t mode0 = __ldcg(buf_mode), mode1 = __ldcg(buf_mode + 1);
  const uint32_t parity = (uint32_t)(par_old & 1) ^ 1u;
  uint64_t* __restrict__ cdf = parity ? cdf1 : cdf0;
  uint64_t* __restrict__ ttot = parity ? ttot1 : ttot0;
  const uint32_t mode = kIndicator ? 2u : 1u;
  const bool full = (parity ? mode1 : mode0) != mode;
  const uint32_t bit = 1u << parity;
  const uint32_t n_tiles = tiles_per_shard * n_shards_local;
  const uint32_t G = gridDim.x;
  if (tid < kMaxShards) s_shcnt[tid] = 0;
  if (tid == 0)
    for (int b = 0; b < kS2Bufs; ++b) mbar_init(smem_u32(&s_bar[b]), 1);
  if (tid == 0) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();

  auto geom = [&](uint32_t t, uint64_t* gbase, uint32_t* count) {
    const uint32_t sh = t / tiles_per_shard, tt = t - sh * tiles_per_shard;
    const uint64_t tb = (uint64_t)tt * kTile;
    *gbase = (uint64_t)sh * shard_cap + tb;
    *count = (uint32_t)min((uint64_t)kTile, shard_cap - tb);
  };
  // thread 0: start the bulk load of work tile j of the chunk into its buffer
  auto issue = [&](uint32_t j) {
    uint64_t gb;
    uint32_t count;
    geom(s_work[j], &gb, &count);
    if (count == (uint32_t)kTile && (gb & 1) == 0)
      bulk_g2s(smem_u32(s_buf + (size_t)(j % kS2Bufs) * kTile), key + gb, kTile * 8,
               smem_u32(&s_bar[j % kS2Bufs]));
  };

  uint32_t phase = 0;
  // this CTA's tile list, in chunks of kThreads entries
  for (uint32_t c0 = 0; blockIdx.x + (uint64_t)c0 * G < n_tiles; c0 += kThreads) {
    const uint64_t t64 = blockIdx.x + (uint64_t)(c0 + tid) * G;
    const bool have = t64 < n_tiles;
    const uint32_t t = (uint32_t)t64;
    // a full rebuild takes every tile: no dirty word on the critical path
    const uint32_t dw = (have && !full) ? __ldcg(dirty + t) : 0u;
    const bool work = have && (full || (dw & bit));
    if (have) atomicAdd(&s_shcnt[t / tiles_per_shard], 1u);
    // compact the work tiles in tile order
    const unsigned m = __ballot_sync(kFull, work);
    if (lane == 0) s_wcnt[warp] = __popc(m);
    __syncthreads();
    uint32_t before = 0, nwork = 0;
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) {
      before += (w < warp) ? s_wcnt[w] : 0u;
      nwork += s_wcnt[w];
    }
    if (work) {
      const uint32_t pos = before + __popc(m & ((1u << lane) - 1u));
      s_work[pos] = t;
    }
    __syncthreads();
    if (tid == 0)
      for (uint32_t j = 0; j < nwork && j < (uint32_t)kS2Bufs - 1; ++j) issue(j);
    for (uint32_t j = 0; j < nwork; ++j) {
      const int b = (int)(j % kS2Bufs);
      const uint32_t wt = s_work[j];
      uint64_t gbase;
      uint32_t count;
      geom(wt, &gbase, &count);
      const bool tma = count == (uint32_t)kTile && (gbase & 1) == 0;
      uint64_t* buf = s_buf + (size_t)b * kTile;
      if (tma) {
        while (!mbar_try_wait(smem_u32(&s_bar[b]), (phase >> b) & 1u)) {
        }
        phase ^= 1u << b;
      } else {
        for (int e = tid; e < kTile; e += kThreads)
          buf[e] = (uint32_t)e < count ? key[gbase + e] : 0ull;
        __syncthreads();
      }
      const int r = tid & 7;
      ulonglong2* b2 = reinterpret_cast<ulonglong2*>(buf) + tid * (kItems / 2);
      uint64_t lo[kItems / 2], hi[kItems / 2];
#pragma unroll
      for (int k = 0; k < kItems / 2; ++k) {
        const ulonglong2 x = b2[(k + r) & 7];
        lo[k] = kIndicator ? (x.x > 0 ? 1ull : 0ull) : x.x;
        hi[k] = kIndicator ? (x.y > 0 ? 1ull : 0ull) : x.y;
      }
      uint64_t run = 0;
#pragma unroll
      for (int k = 0; k < kItems / 2; ++k) {
        lo[k] += run;
        hi[k] += lo[k];
        run = hi[k];
      }
      const uint64_t total = run;
      uint64_t s_rot = 0;
#pragma unroll
      for (int k = 0; k < kItems / 2; ++k) s_rot = (k == 7 - r) ? hi[k] : s_rot;
      const uint64_t incl = warp_incl_scan_u64(total, lane);
      if (lane == 31) s_red[warp] = incl;
      __syncthreads();
      uint64_t warp_excl = 0, agg = 0;
#pragma unroll
      for (int w = 0; w < kThreads / 32; ++w) {
        const uint64_t x = s_red[w];
        warp_excl += (w < warp) ? x : 0ull;
        agg += x;
      }
      const uint64_t base = warp_excl + incl - total;
#pragma unroll
      for (int k = 0; k < kItems / 2; ++k) {
        const uint64_t off = base - s_rot + (k < 8 - r ? total : 0ull);
        b2[(k + r) & 7] = make_ulonglong2(lo[k] + off, hi[k] + off);
      }
      if (tma) {
        // one bulk store of the tile (smem -> global) by thread 0; the next
        // load goes into the PREVIOUS tile's buffer once its store has read
        // it (only the newest store may still be reading) -- no barrier here
        // (vs 16-B stores from every thread: full rebuild of 10 M keys 28.6-31.6
        // instead of 34.0-36.1 us under ncu; event-timed +22% at 5 M keys,
        // -5% at 20 M, even at 10 / 40 M; profiles/r02_scan/s2store)
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();  // the tile's prefixes are in shared memory; s_red read
        if (tid == 0) {
          bulk_s2g(cdf + gbase, smem_u32(buf), kTile * 8);
          ttot[wt] = agg;
          atomicAnd(dirty + wt, ~bit);  // this buffer's bit; the other buffer's stays
          if (j + kS2Bufs - 1 < nwork) {
            asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            issue(j + kS2Bufs - 1);
          }
        }
        continue;
      }
      __syncthreads();  // the tile's prefixes are in shared memory; s_red read
      if (tma) {
        const ulonglong2* src = reinterpret_cast<const ulonglong2*>(buf);
        ulonglong2* dst = reinterpret_cast<ulonglong2*>(cdf + gbase);
#pragma unroll
        for (int k = 0; k < kItems / 2; ++k) dst[k * kThreads + tid] = src[k * kThreads + tid];
      } else {
        for (int e = tid; e < (int)count; e += kThreads) cdf[gbase + e] = buf[e];
      }
      if (tid == 0) {
        ttot[wt] = agg;
        atomicAnd(dirty + wt, ~bit);  // this buffer's bit; the other buffer's stays
      }
      __syncthreads();  // buffer read by every thread: free for tile j + kS2Bufs
      if (tid == 0 && j + kS2Bufs - 1 < nwork) {
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // a bulk-stored buffer
        issue(j + kS2Bufs - 1);
      }
    }
    // the next chunk of the tile list reuses the buffers
    if (tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    __syncthreads();
  }
  if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // before the arrivals

  // Arrivals: this CTA's tiles of every shard in one atomic; the CTA that
  // completes a shard builds its prefix of tile totals P.
  __syncthreads();
  TL_MARK(1);
  if (tid == 0) __threadfence();  // this CTA's cdf / ttot / dirty writes before its arrivals
  for (uint32_t ls = 0; ls < n_shards_local; ++ls) {
    const uint32_t mine = s_shcnt[ls];
    if (mine == 0) continue;  // block-uniform
    if (tid == 0) s_last = atomicAdd(shard_ctr + ls, mine) + mine == tiles_per_shard;
    __syncthreads();
    const bool last = s_last;
    __syncthreads();  // s_last read by every thread before the next shard's write
    if (!last) continue;
    __threadfence();
    uint64_t* P = cdf + (uint64_t)n_shards_local * shard_cap + (uint64_t)ls * tiles_per_shard;
    const uint64_t* tot = ttot + (uint64_t)ls * tiles_per_shard;
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
      __syncthreads();  // s_red of the previous use consumed
      if (lane == 31) s_red[warp] = incl;
      __syncthreads();
      uint64_t warp_excl = 0, agg = 0;
#pragma unroll
      for (int w = 0; w < kThreads / 32; ++w) {
        const uint64_t y = s_red[w];
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
      ShardTotals rec;
      rec.total_and_parity = carry | ((uint64_t)parity << 63);
      rec.aux = 0;
      totals[ls] = rec;
      shard_ctr[ls] = 0;
      __threadfence();
      if (atomicAdd(done, 1u) == n_shards_local - 1) {  // every shard is built
        *done = 0;
        buf_mode[parity] = mode;
        *par_dev = parity;  // every CTA read the old parity before arriving
      }
    }
    __syncthreads();
  }
  TL_PRINT("s2p");
}

}  // namespace

cudaError_t launch_scan2(const uint64_t* key, uint64_t* cdf0, uint64_t* cdf1, uint64_t shard_cap,
                         uint32_t n_shards_local, int indicator, uint64_t* par_dev,
                         ShardTotals* totals_out, uint32_t* dirty, uint64_t* ttot,
                         uint32_t* buf_mode, uint32_t* shard_ctr, uint32_t* done,
                         cudaStream_t s) {
  const uint32_t tps = scan_tiles_per_shard(shard_cap);
  const uint32_t n_tiles = tps * n_shards_local;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  static const bool persistent = [] {
    const char* e = getenv("GEAR_SCAN2_PERSISTENT");
    return e == nullptr || e[0] != '0';
  }();
  // persistent rebuild once the table has more tiles than the resident CTAs
  // (small tables: one CTA per tile launches no idle CTAs and needs no list)
  if (persistent && n_tiles > (uint32_t)sms * kS2Ctas) {
    const size_t smem = (size_t)kS2Bufs * kTile * 8;
    static bool configured = false;
    if (!configured) {
      cudaError_t e = cudaFuncSetAttribute(scan2p_kernel<true>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(scan2p_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem);
      if (e != cudaSuccess) return e;
      configured = true;
    }
    const uint32_t grid = (uint32_t)sms * kS2Ctas;
    count_launch();
    if (indicator)
      scan2p_kernel<true><<<grid, kThreads, smem, s>>>(key, cdf0, cdf1, shard_cap, tps,
                                                       n_shards_local, par_dev, totals_out, dirty,
                                                       ttot, ttot + n_tiles, buf_mode, shard_ctr,
                                                       done);
    else
      scan2p_kernel<false><<<grid, kThreads, smem, s>>>(key, cdf0, cdf1, shard_cap, tps,
                                                        n_shards_local, par_dev, totals_out, dirty,
                                                        ttot, ttot + n_tiles, buf_mode, shard_ctr,
                                                        done);
    return cudaGetLastError();
  }
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
                        ShardTotals* totals_out, uint64_t* status0, uint64_t* status1,
                        uint32_t* ticket, uint32_t* done, int chunked, cudaStream_t s) {
  const uint32_t tps = scan_tiles_per_shard(shard_cap);
  const uint32_t n_tiles = tps * n_shards_local;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // Chunked look-back (scan_chunk_kernel): one chunk per resident CTA, so
  // its phase-2 re-read hits L2 while the rank's keys are a fraction of it.
  // chunked: 1 = whenever the geometry allows, 0 = never, -1 = auto (keys of
  // the rank <= chunk_max_bytes, and at least one tile per CTA); >= 2: as 1
  // for a grid of that many CTAs (tests).
  {
    // (chunked >= 2: chunks sized for that many CTAs, and at most that many
    // CTAs, so chunks are long -- phase-2 reloads -- and CTAs claim several)
    const uint32_t G = chunked >= 2 ? (uint32_t)chunked : (uint32_t)sms * kChunkCtasPerSm;
    uint64_t cps = std::min<uint64_t>(std::max<uint64_t>(1, (uint64_t)G * kChunksPerCta / n_shards_local), tps);
    const uint64_t max_keys = (uint64_t)kMaxChunkTiles * kTile - 32;
    cps = std::max<uint64_t>(cps, (shard_cap + max_keys - 1) / max_keys);
    const uint64_t n_chunks = cps * n_shards_local;
    static const uint64_t chunk_max_bytes = [] {
      const char* e = getenv("GEAR_SCAN_CHUNK_MAX_MB");
      return (uint64_t)(e ? atoll(e) : 96) << 20;
    }();
    const bool fits = n_chunks <= n_tiles && shard_cap >= cps * 16;
    const bool want = chunked >= 1 ||
                      (chunked == -1 && (uint64_t)n_shards_local * shard_cap * 8 <= chunk_max_bytes &&
                       n_tiles >= G);
    if (fits && want) {
      const size_t smem = (size_t)kCBufs * kTile * 8;
      static bool configured = false;
      if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(scan_chunk_kernel<true>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e == cudaSuccess)
          e = cudaFuncSetAttribute(scan_chunk_kernel<false>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        configured = true;
      }
      const uint32_t grid = (uint32_t)std::min<uint64_t>(n_chunks, G);
      count_launch();
      if (indicator)
        scan_chunk_kernel<true><<<grid, kThreads, smem, s>>>(
            key, cdf0, cdf1, shard_cap, (uint32_t)cps, (uint32_t)n_chunks, n_tiles, par_dev,
            totals_out, status0, status1, ticket, done);
      else
        scan_chunk_kernel<false><<<grid, kThreads, smem, s>>>(
            key, cdf0, cdf1, shard_cap, (uint32_t)cps, (uint32_t)n_chunks, n_tiles, par_dev,
            totals_out, status0, status1, ticket, done);
      return cudaGetLastError();
    }
  }
  const size_t smem = (size_t)kScanBufs * kTile * 8;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(scan_kernel<true>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(scan_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  const uint32_t grid = std::min<uint32_t>(n_tiles, (uint32_t)sms * kScanCtasPerSm);
  count_launch();
  if (indicator)
    scan_kernel<true><<<grid, kThreads, smem, s>>>(key, cdf0, cdf1, shard_cap, tps, n_tiles,
                                                   par_dev, totals_out, status0, status1, ticket, done);
  else
    scan_kernel<false><<<grid, kThreads, smem, s>>>(key, cdf0, cdf1, shard_cap, tps, n_tiles,
                                                    par_dev, totals_out, status0, status1, ticket, done);
  return cudaGetLastError();
}

}  // namespace gear
