// Hardware probe: PCIe H2D/D2H copy, zero-copy host reads from a kernel,
// HBM copy kernel, and peer copies / peer kernel reads when >1 GPU is visible.
// Prints one JSON object per measurement. Not part of the product path.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <vector>
#include <chrono>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

template <int U>
__global__ void copy_kernel(const int4* __restrict__ src, int4* __restrict__ dst, size_t n) {
  size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = tid;
  for (; i + (U - 1) * stride < n; i += U * stride) {
    int4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = src[i + u * stride];
#pragma unroll
    for (int u = 0; u < U; ++u) dst[i + u * stride] = v[u];
  }
  for (; i < n; i += stride) dst[i] = src[i];
}

static float time_copy(int grid, int block, const void* s, void* d, size_t bytes, int reps) {
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  size_t n = bytes / 16;
  copy_kernel<8><<<grid, block>>>((const int4*)s, (int4*)d, n);
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(a));
    copy_kernel<8><<<grid, block>>>((const int4*)s, (int4*)d, n);
    CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
    float ms; CK(cudaEventElapsedTime(&ms, a, b)); if (ms < best) best = ms;
  }
  return best;
}

static float time_memcpy(void* d, const void* s, size_t bytes, cudaMemcpyKind k, int reps) {
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  CK(cudaMemcpy(d, s, bytes, k));
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(a)); CK(cudaMemcpyAsync(d, s, bytes, k)); CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms; CK(cudaEventElapsedTime(&ms, a, b)); if (ms < best) best = ms;
  }
  return best;
}

// Sustained single-device loop for the concurrent probes:
//   probe zc <dev> <seconds>   zero-copy kernel reads of 1 GiB pinned host memory
//   probe h2d <dev> <seconds>  pinned cudaMemcpy H2D of 1 GiB
static int sustained(const char* mode, int dev, double secs) {
  CK(cudaSetDevice(dev));
  size_t bytes = (size_t)1 << 30;
  void *h, *d;
  CK(cudaHostAlloc(&h, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
  memset(h, 1, bytes);
  CK(cudaMalloc(&d, bytes));
  void* hd; CK(cudaHostGetDevicePointer(&hd, h, 0));
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  double moved = 0, ms_total = 0;
  auto t0 = std::chrono::steady_clock::now();
  while (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() < secs) {
    CK(cudaEventRecord(a));
    if (mode[0] == 'z') copy_kernel<8><<<1184, 512>>>((const int4*)hd, (int4*)d, bytes / 16);
    else CK(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice));
    CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
    float ms; CK(cudaEventElapsedTime(&ms, a, b));
    moved += bytes; ms_total += ms;
  }
  printf("{\"probe\":\"sustained_%s\",\"dev\":%d,\"GBps\":%.2f,\"seconds\":%.2f}\n", mode, dev,
         moved / ms_total / 1e6, ms_total / 1e3);
  return 0;
}

int main(int argc, char** argv) {
  if (argc >= 4) return sustained(argv[1], atoi(argv[2]), atof(argv[3]));
  int ndev = 0; CK(cudaGetDeviceCount(&ndev));
  printf("{\"probe\":\"devices\",\"n\":%d}\n", ndev);
  size_t bytes = (size_t)1 << 30;
  for (int dev = 0; dev < ndev; ++dev) {
    CK(cudaSetDevice(dev));
    cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
    printf("{\"probe\":\"prop\",\"dev\":%d,\"name\":\"%s\",\"sms\":%d,\"pci_bus\":%d,\"l2\":%d,\"canMapHost\":%d}\n",
           dev, p.name, p.multiProcessorCount, p.pciBusID, p.l2CacheSize, p.canMapHostMemory);
    void *h, *d0, *d1;
    CK(cudaHostAlloc(&h, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
    memset(h, 1, bytes);
    CK(cudaMalloc(&d0, bytes)); CK(cudaMalloc(&d1, bytes));
    float ms = time_memcpy(d0, h, bytes, cudaMemcpyHostToDevice, 5);
    printf("{\"probe\":\"h2d_memcpy\",\"dev\":%d,\"GBps\":%.2f}\n", dev, bytes / ms / 1e6);
    ms = time_memcpy(h, d0, bytes, cudaMemcpyDeviceToHost, 5);
    printf("{\"probe\":\"d2h_memcpy\",\"dev\":%d,\"GBps\":%.2f}\n", dev, bytes / ms / 1e6);
    ms = time_memcpy(d1, d0, bytes, cudaMemcpyDeviceToDevice, 5);
    printf("{\"probe\":\"d2d_memcpy\",\"dev\":%d,\"GBps_rw\":%.2f}\n", dev, 2 * bytes / ms / 1e6);
    for (int grid : {148, 296, 592, 1184, 2368}) for (int block : {256, 512}) {
      ms = time_copy(grid, block, d0, d1, bytes, 5);
      printf("{\"probe\":\"hbm_copy_kernel\",\"dev\":%d,\"grid\":%d,\"block\":%d,\"GBps_rw\":%.2f}\n", dev, grid, block, 2 * bytes / ms / 1e6);
    }
    void* hd; CK(cudaHostGetDevicePointer(&hd, h, 0));
    size_t zb = (size_t)256 << 20;
    for (int grid : {148, 296, 592, 1184, 2368}) for (int block : {256, 512, 1024}) {
      ms = time_copy(grid, block, hd, d1, zb, 3);
      printf("{\"probe\":\"zerocopy_read_kernel\",\"dev\":%d,\"grid\":%d,\"block\":%d,\"GBps\":%.2f}\n", dev, grid, block, zb / ms / 1e6);
    }
    CK(cudaFreeHost(h)); CK(cudaFree(d0)); CK(cudaFree(d1));
    if (dev >= 1) break;  // two devices is enough for per-GPU numbers
  }
  // host register of a large malloc'ed region: time + feasibility
  {
    CK(cudaSetDevice(0));
    for (size_t gb : {4, 32}) {
      size_t nb = gb << 30;
      void* m = aligned_alloc(1 << 21, nb);
      if (!m) { printf("{\"probe\":\"hostreg\",\"GB\":%zu,\"alloc\":0}\n", gb); continue; }
      memset(m, 0, nb);
      cudaEvent_t a; (void)a;
      auto t0 = std::chrono::steady_clock::now();
      cudaError_t e = cudaHostRegister(m, nb, cudaHostRegisterMapped | cudaHostRegisterPortable);
      auto t1 = std::chrono::steady_clock::now();
      printf("{\"probe\":\"hostreg\",\"GB\":%zu,\"ok\":%d,\"s\":%.3f}\n", gb, e == cudaSuccess,
             std::chrono::duration<double>(t1 - t0).count());
      if (e == cudaSuccess) {
        void* dd; CK(cudaMalloc(&dd, (size_t)256 << 20)); void* hd;
        CK(cudaHostGetDevicePointer(&hd, m, 0));
        float ms = time_copy(1184, 512, hd, dd, (size_t)256 << 20, 3);
        printf("{\"probe\":\"zerocopy_registered\",\"GB\":%zu,\"GBps\":%.2f}\n", gb, ((size_t)256 << 20) / ms / 1e6);
        CK(cudaFree(dd)); CK(cudaHostUnregister(m));
      } else cudaGetLastError();
      free(m);
    }
  }
  if (ndev > 1) {
    for (int a = 0; a < ndev; ++a) for (int b = 0; b < ndev; ++b) if (a != b) {
      int can; CK(cudaDeviceCanAccessPeer(&can, a, b));
      if (!can) { printf("{\"probe\":\"peer\",\"a\":%d,\"b\":%d,\"can\":0}\n", a, b); continue; }
      CK(cudaSetDevice(a)); cudaDeviceEnablePeerAccess(b, 0); cudaGetLastError();
      CK(cudaSetDevice(b)); cudaDeviceEnablePeerAccess(a, 0); cudaGetLastError();
    }
    for (int b = 1; b < ndev; ++b) {
      void *da, *db;
      CK(cudaSetDevice(b)); CK(cudaMalloc(&db, bytes));
      CK(cudaSetDevice(0)); CK(cudaMalloc(&da, bytes));
      float ms = time_memcpy(da, db, bytes, cudaMemcpyDeviceToDevice, 5);
      printf("{\"probe\":\"peer_memcpy_pull\",\"dst\":0,\"src\":%d,\"GBps\":%.2f}\n", b, bytes / ms / 1e6);
      for (int grid : {148, 296, 592, 1184}) for (int block : {256, 512}) {
        ms = time_copy(grid, block, db, da, bytes, 3);
        printf("{\"probe\":\"peer_kernel_read\",\"dst\":0,\"src\":%d,\"grid\":%d,\"block\":%d,\"GBps\":%.2f}\n", b, grid, block, bytes / ms / 1e6);
      }
      CK(cudaFree(da)); CK(cudaSetDevice(b)); CK(cudaFree(db));
    }
  }
  return 0;
}
