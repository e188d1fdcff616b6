// fill.cu -- seeded synthetic row bytes on the GPU (input generation only;
// holds none of the replay method's arithmetic).  Row t of column c is the
// little-endian byte stream of 64-bit words
//   word_w = splitmix64(base + w * 0x632BE59BD9B4E019),
//   base   = splitmix64(seed ^ c * 0xD1B54A32D192ED03 ^ t * 0x9E3779B97F4A7C15),
// truncated to row_bytes; synth/__init__.py computes the same bytes with numpy
// so tests can regenerate any sampled row without a second copy of a table.
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void fill_rows_kernel(uint8_t* dst, uint64_t n_rows, uint64_t row_bytes, uint64_t col,
                                 uint64_t first_traj, uint64_t seed) {
  const uint64_t words_per_row = (row_bytes + 7) / 8;
  const uint64_t total = n_rows * words_per_row;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = i / words_per_row, w = i - r * words_per_row;
    const uint64_t t = first_traj + r;
    const uint64_t base = splitmix64(seed ^ (col * 0xD1B54A32D192ED03ull) ^ (t * 0x9E3779B97F4A7C15ull));
    const uint64_t v = splitmix64(base + w * 0x632BE59BD9B4E019ull);
    uint8_t* row = dst + r * row_bytes;
    const uint64_t off = w * 8;
    if (off + 8 <= row_bytes && (row_bytes % 8) == 0) {
      *reinterpret_cast<uint64_t*>(row + off) = v;
    } else {
      for (int b = 0; b < 8 && off + b < row_bytes; ++b) row[off + b] = (uint8_t)(v >> (8 * b));
    }
  }
}

extern "C" int synth_fill_rows(void* dst, uint64_t n_rows, uint64_t row_bytes, uint64_t col,
                               uint64_t first_traj, uint64_t seed, void* stream) {
  if (n_rows == 0) return 0;
  fill_rows_kernel<<<148 * 16, 256, 0, (cudaStream_t)stream>>>((uint8_t*)dst, n_rows, row_bytes,
                                                               col, first_traj, seed);
  return (int)cudaGetLastError();
}

// Row k of dst is the row of trajectory ids[k] (device u64 ids): expected
// batches of a gather are regenerated whole, without a copy of the table.
__global__ void fill_rows_ids_kernel(uint8_t* dst, const uint64_t* ids, uint64_t n_rows,
                                     uint64_t row_bytes, uint64_t col, uint64_t seed) {
  const uint64_t words_per_row = (row_bytes + 7) / 8;
  const uint64_t total = n_rows * words_per_row;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = i / words_per_row, w = i - r * words_per_row;
    const uint64_t t = ids[r];
    const uint64_t base = splitmix64(seed ^ (col * 0xD1B54A32D192ED03ull) ^ (t * 0x9E3779B97F4A7C15ull));
    const uint64_t v = splitmix64(base + w * 0x632BE59BD9B4E019ull);
    uint8_t* row = dst + r * row_bytes;
    const uint64_t off = w * 8;
    if (off + 8 <= row_bytes && (row_bytes % 8) == 0) {
      *reinterpret_cast<uint64_t*>(row + off) = v;
    } else {
      for (int b = 0; b < 8 && off + b < row_bytes; ++b) row[off + b] = (uint8_t)(v >> (8 * b));
    }
  }
}

extern "C" int synth_fill_rows_ids(void* dst, const void* ids, uint64_t n_rows, uint64_t row_bytes,
                                   uint64_t col, uint64_t seed, void* stream) {
  if (n_rows == 0) return 0;
  fill_rows_ids_kernel<<<148 * 16, 256, 0, (cudaStream_t)stream>>>(
      (uint8_t*)dst, (const uint64_t*)ids, n_rows, row_bytes, col, seed);
  return (int)cudaGetLastError();
}
