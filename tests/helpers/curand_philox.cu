// Test helper (not product code): 64-bit draws r_j = x0 | x1 << 32 of the
// library generator curand Philox4_32_10 with counter block j and key `seed`
// -- curand_init(seed, subsequence 0, offset 4*j) positions the generator at
// block j -- for pinning the product's Philox (reading Q4) to a library
// routine.  Built by tests/test_gpu_curand_pin.py with nvcc.
#include <cstdint>
#include <curand_kernel.h>

__global__ void draws(uint64_t seed, const uint64_t* j, uint32_t n, uint64_t* out) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  curandStatePhilox4_32_10_t st;
  curand_init(seed, 0ull, 4ull * j[k], &st);
  const uint4 x = curand4(&st);
  out[k] = (uint64_t)x.x | ((uint64_t)x.y << 32);
}

extern "C" int curand_philox_draws(uint64_t seed, const uint64_t* j_host, uint32_t n,
                                   uint64_t* out_host) {
  uint64_t *dj = nullptr, *dout = nullptr;
  if (cudaMalloc(&dj, n * 8) != cudaSuccess || cudaMalloc(&dout, n * 8) != cudaSuccess) return 1;
  cudaMemcpy(dj, j_host, n * 8, cudaMemcpyHostToDevice);
  draws<<<(n + 255) / 256, 256>>>(seed, dj, n, dout);
  const cudaError_t e = cudaMemcpy(out_host, dout, n * 8, cudaMemcpyDeviceToHost);
  cudaFree(dj);
  cudaFree(dout);
  return e == cudaSuccess ? 0 : 2;
}
