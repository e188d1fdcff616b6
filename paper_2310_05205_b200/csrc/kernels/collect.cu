// collect.cu -- K5: gather the selected rows of several columns into
// contiguous batches, and the insert-side scatter.
//
// The paper launches "one CUDA kernel per table" that reads pinned host
// memory zero-copy; here ONE launch covers every requested
// column.  The work is a flat list of warp tasks (column, row j, chunk k) of
// `chunk_bytes` each, decoded arithmetically (no work list in memory); a
// persistent grid of warps strides over it.  Index translation (shard = g div
// C_s) is fused: the row's owner rank picks the source base,
// which is local HBM, a peer GPU's HBM mapped through CUDA IPC (NVLink loads)
// or pinned host memory mapped into the device address space (PCIe loads).
// Each lane keeps kUnroll independent 16-byte loads in flight before it
// stores, so a warp has kUnroll*512 B outstanding -- what the PCIe path needs
// to cover its ~1-2 us round trip, and what HBM needs to reach its copy peak.
#include "common.cuh"

namespace gear {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kUnroll = 8;

// Copy `bytes` (a multiple of V) from src to dst with one warp.
template <int V>
__device__ __forceinline__ void warp_copy(uint8_t* __restrict__ dst,
                                          const uint8_t* __restrict__ src, uint64_t bytes,
                                          int lane) {
  if constexpr (V == 16) {
    const uint64_t n = bytes >> 4;
    uint64_t i = lane;
    for (; i + (kUnroll - 1) * 32 < n; i += kUnroll * 32) {
      int4 v[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) v[u] = ld_stream16(src + ((i + u * 32) << 4));
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) st_stream16(dst + ((i + u * 32) << 4), v[u]);
    }
    int4 v[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u)
      if (i + u * 32 < n) v[u] = ld_stream16(src + ((i + u * 32) << 4));
#pragma unroll
    for (int u = 0; u < kUnroll; ++u)
      if (i + u * 32 < n) st_stream16(dst + ((i + u * 32) << 4), v[u]);
  } else {
    using T = typename std::conditional<
        V == 8, uint64_t,
        typename std::conditional<V == 4, uint32_t,
                                  typename std::conditional<V == 2, uint16_t, uint8_t>::type>::type>::type;
    const uint64_t n = bytes / V;
    const T* s = reinterpret_cast<const T*>(src);
    T* d = reinterpret_cast<T*>(dst);
    uint64_t i = lane;
    for (; i + (kUnroll - 1) * 32 < n; i += kUnroll * 32) {
      T v[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) v[u] = s[i + u * 32];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) d[i + u * 32] = v[u];
    }
    for (; i < n; i += 32) d[i] = s[i];
  }
}

__device__ __forceinline__ void copy_dispatch(uint32_t vec, uint8_t* dst, const uint8_t* src,
                                              uint64_t bytes, int lane) {
  switch (vec) {
    case 16: warp_copy<16>(dst, src, bytes, lane); break;
    case 8: warp_copy<8>(dst, src, bytes, lane); break;
    case 4: warp_copy<4>(dst, src, bytes, lane); break;
    case 2: warp_copy<2>(dst, src, bytes, lane); break;
    default: warp_copy<1>(dst, src, bytes, lane); break;
  }
}

__global__ void __launch_bounds__(kThreads) collect_kernel(const __grid_constant__ CollectParams p) {
  const int lane = threadIdx.x & 31;
  const uint64_t warp0 = (uint64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
  const uint64_t nwarps = (uint64_t)gridDim.x * kWarps;
  for (uint64_t task = warp0; task < p.total_chunks; task += nwarps) {
    uint32_t c = 0;
    while (c + 1 < p.ncols && task >= p.col[c + 1].chunk_begin) ++c;
    const CollectCol& col = p.col[c];
    const uint64_t rel = task - col.chunk_begin;
    const uint64_t j = rel / col.chunks_per_row;
    const uint64_t k = rel - j * col.chunks_per_row;
    const uint64_t g = __ldg(p.idx + j);
    if (g >= p.n_global) {
      if (lane == 0 && k == 0) atomicOr(p.err, kErrIndexRange);
      continue;
    }
    const uint64_t owner = g / p.rows_per_rank;
    const uint64_t local = g - owner * p.rows_per_rank;
    const uint64_t off = k * (uint64_t)p.chunk_bytes;
    const uint64_t rem = col.rb - off;
    const uint64_t bytes = rem < p.chunk_bytes ? rem : p.chunk_bytes;
    copy_dispatch(col.vec, col.out + j * col.rb + off, col.src[owner] + local * col.rb + off,
                  bytes, lane);
  }
}

__global__ void __launch_bounds__(kThreads) scatter_kernel(const __grid_constant__ ScatterParams p) {
  const int lane = threadIdx.x & 31;
  const uint64_t warp0 = (uint64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
  const uint64_t nwarps = (uint64_t)gridDim.x * kWarps;
  for (uint64_t task = warp0; task < p.total_chunks; task += nwarps) {
    uint32_t c = 0;
    while (c + 1 < p.ncols && task >= p.col[c + 1].chunk_begin) ++c;
    const ScatterCol& col = p.col[c];
    const uint64_t rel = task - col.chunk_begin;
    const uint64_t j = rel / col.chunks_per_row;
    const uint64_t k = rel - j * col.chunks_per_row;
    const InsMeta m = p.meta[j];
    const uint64_t off = k * (uint64_t)p.chunk_bytes;
    const uint64_t rem = col.rb - off;
    const uint64_t bytes = rem < p.chunk_bytes ? rem : p.chunk_bytes;
    copy_dispatch(col.vec, col.dst + m.local * col.rb + off,
                  col.src + (uint64_t)m.src_row * col.rb + off, bytes, lane);
  }
}

__global__ void __launch_bounds__(kThreads)
    insert_meta_kernel(const InsMeta* __restrict__ meta, uint32_t m,
                       const OrdRec* __restrict__ ord_recs, uint32_t n_ord, uint32_t frac_bits,
                       uint64_t q_max, uint64_t* key, uint64_t* seq, uint32_t* gen,
                       uint32_t* ord) {
  const uint32_t k = blockIdx.x * kThreads + threadIdx.x;
  if (k < m) {
    const InsMeta r = meta[k];
    uint64_t q = 0;
    quantize(r.prio, frac_bits, q_max, &q);  // validated on the host
    key[r.local] = q;
    seq[r.local] = r.seq;
    gen[r.local] += r.gen_inc;
  }
  if (k < n_ord) ord[ord_recs[k].pos] = ord_recs[k].slot;
}

// Persistent grid: as many CTAs as can be resident at once (no second wave
// whose warps would start late on a static task split), capped by the work.
template <class K>
int grid_for(K kernel, uint64_t tasks) {
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kThreads, 0);
  const uint64_t want = (tasks + kWarps - 1) / kWarps;
  const uint64_t cap = (uint64_t)sms * (per_sm > 0 ? per_sm : 1);
  return (int)(want < cap ? (want > 0 ? want : 1) : cap);
}

}  // namespace

cudaError_t launch_collect(const CollectParams& p, cudaStream_t s) {
  if (p.total_chunks == 0) return cudaSuccess;
  count_launch();
  collect_kernel<<<grid_for(collect_kernel, p.total_chunks), kThreads, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_scatter(const ScatterParams& p, cudaStream_t s) {
  if (p.total_chunks == 0) return cudaSuccess;
  count_launch();
  scatter_kernel<<<grid_for(scatter_kernel, p.total_chunks), kThreads, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_insert_meta(const InsMeta* meta, uint32_t m, const OrdRec* ord_recs,
                               uint32_t n_ord, uint32_t frac_bits, uint64_t q_max,
                               uint64_t* key, uint64_t* seq, uint32_t* gen, uint32_t* ord,
                               cudaStream_t s) {
  const uint32_t n = m > n_ord ? m : n_ord;
  if (n == 0) return cudaSuccess;
  count_launch();
  insert_meta_kernel<<<(n + kThreads - 1) / kThreads, kThreads, 0, s>>>(
      meta, m, ord_recs, n_ord, frac_bits, q_max, key, seq, gen, ord);
  return cudaGetLastError();
}

}  // namespace gear
