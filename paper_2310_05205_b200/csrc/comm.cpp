// comm.cpp -- error reporting, pointer classification and the NCCL plumbing
// of the replay hot path (one NCCL communicator per rank; NVLink 5 /
// NVSwitch inside the box).  The exchanges the path needs are tiny: shard
// totals (16 B per shard), FIFO/LIFO candidates (16 B each) and priority
// updates (24 B each); the payload itself is read peer-to-peer by the
// collect kernel, never through NCCL.
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <vector>

#include "runtime.h"

namespace gear {

namespace {
thread_local char g_err[1024] = "";
std::atomic<uint64_t> g_launches{0};
}

void count_launch(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

gear_status set_error(gear_status code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

void clear_error() { g_err[0] = 0; }

const char* last_error() { return g_err; }

MemKind mem_kind(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return MemKind::HostPageable;
  }
  switch (a.type) {
    case cudaMemoryTypeDevice:
    case cudaMemoryTypeManaged:
      return MemKind::Device;
    case cudaMemoryTypeHost:
      return MemKind::HostPinned;
    default:
      return MemKind::HostPageable;
  }
}

// Host-callback all-gather: stream-ordered by synchronising the stream
// (device buffers are staged through host memory).  Not graph-capturable.
gear_status host_allgather(gear_comm* c, const void* send, void* recv, size_t bytes,
                           cudaStream_t s) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  GEAR_CUDA(cudaStreamIsCapturing(s, &cs));
  if (cs != cudaStreamCaptureStatusNone)
    return set_error(GEAR_ERR_UNSUPPORTED,
                     "a host-bootstrapped comm cannot run an all-gather inside stream capture "
                     "(use peer_xchg = 1)");
  GEAR_CUDA(cudaStreamSynchronize(s));
  const bool dev_send = mem_kind(send) == MemKind::Device;
  const bool dev_recv = mem_kind(recv) == MemKind::Device;
  std::vector<uint8_t> hs, hr;
  const void* sp = send;
  void* rp = recv;
  if (dev_send) {
    hs.resize(bytes);
    GEAR_CUDA(cudaMemcpy(hs.data(), send, bytes, cudaMemcpyDeviceToHost));
    sp = hs.data();
  }
  if (dev_recv) {
    hr.resize(bytes * (size_t)c->nranks);
    rp = hr.data();
  }
  if (c->host_ag(c->host_ctx, sp, rp, bytes) != 0)
    return set_error(GEAR_ERR_NCCL, "host all-gather callback failed (%zu bytes)", bytes);
  if (dev_recv)
    GEAR_CUDA(cudaMemcpy(recv, hr.data(), bytes * (size_t)c->nranks, cudaMemcpyHostToDevice));
  return GEAR_OK;
}

gear_status allgather_bytes(gear_comm* c, const void* send, void* recv, size_t bytes,
                            cudaStream_t s) {
  if (c == nullptr || c->nranks == 1) {
    if (send != recv) GEAR_CUDA(cudaMemcpyAsync(recv, send, bytes, cudaMemcpyDeviceToDevice, s));
    return GEAR_OK;
  }
  if (c->host_ag) return host_allgather(c, send, recv, bytes, s);
  GEAR_NCCL(ncclAllGather(send, recv, bytes, ncclUint8, c->nccl, s));
  return GEAR_OK;
}

gear_status barrier(gear_comm* c) {
  if (c == nullptr || c->nranks == 1) return GEAR_OK;
  if (c->host_ag) {
    GEAR_CUDA(cudaDeviceSynchronize());
    uint8_t one = 1;
    std::vector<uint8_t> all((size_t)c->nranks);
    if (c->host_ag(c->host_ctx, &one, all.data(), 1) != 0)
      return set_error(GEAR_ERR_NCCL, "host all-gather callback failed (barrier)");
    return GEAR_OK;
  }
  int* d = nullptr;
  GEAR_CUDA(cudaMallocAsync(&d, sizeof(int), c->stream));
  GEAR_CUDA(cudaMemsetAsync(d, 0, sizeof(int), c->stream));
  GEAR_NCCL(ncclAllReduce(d, d, 1, ncclInt32, ncclSum, c->nccl, c->stream));
  GEAR_CUDA(cudaFreeAsync(d, c->stream));
  GEAR_CUDA(cudaStreamSynchronize(c->stream));
  return GEAR_OK;
}

}  // namespace gear

extern "C" {

const char* gear_last_error(void) { return gear::last_error(); }

const char* gear_version(void) { return "gear-b200 0.1 (sm_100a)"; }

uint64_t gear_kernel_launches(void) { return gear::g_launches.load(); }

gear_status gear_get_unique_id(uint8_t out[128]) {
  GEAR_NVTX("gear_get_unique_id");
  static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id is 128 bytes");
  if (out == nullptr) return gear::set_error(GEAR_ERR_INVALID_ARG, "out is NULL");
  ncclUniqueId id;
  GEAR_NCCL(ncclGetUniqueId(&id));
  std::memcpy(out, &id, sizeof(id));
  return GEAR_OK;
}

gear_status gear_comm_create(int nranks, int rank, const uint8_t id[128], int device,
                             gear_comm** out) {
  GEAR_NVTX("gear_comm_create");
  gear::clear_error();
  if (out == nullptr || id == nullptr || nranks < 1 || nranks > gear::kMaxRanks || rank < 0 ||
      rank >= nranks || device < 0)
    return gear::set_error(GEAR_ERR_INVALID_ARG, "bad comm arguments (nranks=%d rank=%d)",
                           nranks, rank);
  GEAR_CUDA(cudaSetDevice(device));
  auto* c = new gear_comm();
  c->nranks = nranks;
  c->rank = rank;
  c->device = device;
  cudaError_t e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete c;
    return gear::set_error(GEAR_ERR_CUDA, "cudaStreamCreate: %s", cudaGetErrorString(e));
  }
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  ncclResult_t r = ncclCommInitRank(&c->nccl, nranks, uid, rank);
  if (r != ncclSuccess) {
    cudaStreamDestroy(c->stream);
    delete c;
    return gear::set_error(GEAR_ERR_NCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
  }
  *out = c;
  return GEAR_OK;
}

gear_status gear_comm_create_host(int nranks, int rank, int device, gear_allgather_fn fn,
                                  void* ctx, gear_comm** out) {
  GEAR_NVTX("gear_comm_create_host");
  gear::clear_error();
  if (out == nullptr || fn == nullptr || nranks < 1 || nranks > gear::kMaxRanks || rank < 0 ||
      rank >= nranks || device < 0)
    return gear::set_error(GEAR_ERR_INVALID_ARG, "bad comm arguments (nranks=%d rank=%d)",
                           nranks, rank);
  GEAR_CUDA(cudaSetDevice(device));
  auto* c = new gear_comm();
  c->nranks = nranks;
  c->rank = rank;
  c->device = device;
  c->host_ag = fn;
  c->host_ctx = ctx;
  cudaError_t e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete c;
    return gear::set_error(GEAR_ERR_CUDA, "cudaStreamCreate: %s", cudaGetErrorString(e));
  }
  // every rank agrees on nranks (a mismatch would hang the first exchange)
  std::vector<int32_t> all((size_t)nranks);
  int32_t mine = nranks;
  if (fn(ctx, &mine, all.data(), sizeof(mine)) != 0) {
    cudaStreamDestroy(c->stream);
    delete c;
    return gear::set_error(GEAR_ERR_NCCL, "host all-gather callback failed (bootstrap)");
  }
  for (int r = 0; r < nranks; ++r)
    if (all[r] != nranks) {
      cudaStreamDestroy(c->stream);
      delete c;
      return gear::set_error(GEAR_ERR_INVALID_ARG, "rank %d passed nranks=%d, this rank %d", r,
                             all[r], nranks);
    }
  *out = c;
  return GEAR_OK;
}

gear_status gear_comm_destroy(gear_comm* c) {
  GEAR_NVTX("gear_comm_destroy");
  if (c == nullptr) return GEAR_OK;
  cudaSetDevice(c->device);
  if (c->nccl) ncclCommDestroy(c->nccl);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
  return GEAR_OK;
}

}  // extern "C"
