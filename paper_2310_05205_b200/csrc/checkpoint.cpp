// checkpoint.cpp -- shard checkpoint / restore ("GEAR allows
// for trajectory shards to be checkpointed on local SSDs ... at data epoch
// boundaries").  One file per rank holds that rank's R shards: a header that
// pins the layout, the slot state (keys, seq, gen), the insertion rings and
// every column's rows.  Device rows stream through a pinned staging buffer.
#include <cstdio>
#include <cstring>
#include <vector>

#include "runtime.h"

using namespace gear;

namespace {

constexpr char kMagic[8] = {'G', 'E', 'A', 'R', 'C', 'K', 'P', 'T'};
constexpr uint32_t kVersion = 2;
constexpr size_t kStage = 64ull << 20;

struct Header {
  char magic[8];
  uint32_t version, W, R, rank, ncols, F, removal, pad;
  uint64_t N, Cs;
  uint64_t rb[kMaxCols];
  uint32_t placement[kMaxCols];
  double alpha;  // PER exponent the keys were made with
};

Header make_header(const gear_table* t) {
  Header h{};
  std::memcpy(h.magic, kMagic, 8);
  h.version = kVersion;
  h.W = t->W;
  h.R = t->R;
  h.rank = t->rank;
  h.ncols = (uint32_t)t->cols.size();
  h.F = t->F;
  h.removal = (uint32_t)t->removal;
  h.N = t->N;
  h.Cs = t->Cs;
  h.alpha = t->alpha;
  for (size_t c = 0; c < t->cols.size(); ++c) {
    h.rb[c] = t->cols[c].rb;
    h.placement[c] = (uint32_t)t->cols[c].placement;
  }
  return h;
}

struct File {
  FILE* f = nullptr;
  ~File() {
    if (f) fclose(f);
  }
};

gear_status wr(FILE* f, const void* p, size_t n) {
  if (n && fwrite(p, 1, n, f) != n) return set_error(GEAR_ERR_INVALID_ARG, "checkpoint write failed");
  return GEAR_OK;
}

gear_status rd(FILE* f, void* p, size_t n) {
  if (n && fread(p, 1, n, f) != n) return set_error(GEAR_ERR_INVALID_ARG, "checkpoint truncated");
  return GEAR_OK;
}

// Device <-> file through a pinned staging buffer.
gear_status dev_to_file(FILE* f, const void* d, size_t n, uint8_t* stage) {
  for (size_t o = 0; o < n; o += kStage) {
    const size_t m = n - o < kStage ? n - o : kStage;
    GEAR_CUDA(cudaMemcpy(stage, (const uint8_t*)d + o, m, cudaMemcpyDeviceToHost));
    GEAR_TRY(wr(f, stage, m));
  }
  return GEAR_OK;
}

gear_status file_to_dev(FILE* f, void* d, size_t n, uint8_t* stage) {
  for (size_t o = 0; o < n; o += kStage) {
    const size_t m = n - o < kStage ? n - o : kStage;
    GEAR_TRY(rd(f, stage, m));
    GEAR_CUDA(cudaMemcpy((uint8_t*)d + o, stage, m, cudaMemcpyHostToDevice));
  }
  return GEAR_OK;
}

struct Pinned {
  uint8_t* p = nullptr;
  ~Pinned() {
    if (p) cudaFreeHost(p);
  }
};

}  // namespace

extern "C" {

gear_status gear_table_save(gear_table* t, const char* path) {
  clear_error();
  if (t == nullptr || path == nullptr) return set_error(GEAR_ERR_INVALID_ARG, "NULL argument");
  GEAR_CUDA(cudaSetDevice(t->device));
  GEAR_CUDA(cudaDeviceSynchronize());
  File file;
  file.f = fopen(path, "wb");
  if (!file.f) return set_error(GEAR_ERR_INVALID_ARG, "cannot open %s for writing", path);
  Pinned stage;
  GEAR_CUDA(cudaHostAlloc((void**)&stage.p, kStage, cudaHostAllocDefault));
  const Header h = make_header(t);
  GEAR_TRY(wr(file.f, &h, sizeof(h)));
  GEAR_TRY(dev_to_file(file.f, t->key, t->Clocal * 8, stage.p));
  GEAR_TRY(dev_to_file(file.f, t->seq, t->Clocal * 8, stage.p));
  GEAR_TRY(dev_to_file(file.f, t->gen, t->Clocal * 4, stage.p));
  // the device-resident allocator state and ring of every local shard
  std::vector<AllocState> a(t->R);
  GEAR_CUDA(cudaMemcpy(a.data(), t->d_alloc, t->R * sizeof(AllocState), cudaMemcpyDeviceToHost));
  std::vector<uint32_t> ord(t->Cs);
  for (uint32_t ls = 0; ls < t->R; ++ls) {
    const uint64_t st[4] = {a[ls].next_free, a[ls].head, a[ls].len, a[ls].seq_ctr};
    GEAR_TRY(wr(file.f, st, sizeof(st)));
    GEAR_CUDA(cudaMemcpy(ord.data(), t->ord + (uint64_t)ls * t->Cs, t->Cs * 4,
                         cudaMemcpyDeviceToHost));
    GEAR_TRY(wr(file.f, ord.data(), t->Cs * 4));
  }
  for (const ColumnState& c : t->cols) {
    if (c.placement == GEAR_DEVICE) GEAR_TRY(dev_to_file(file.f, c.local, c.bytes_local, stage.p));
    else GEAR_TRY(wr(file.f, c.local, c.bytes_local));
  }
  if (fflush(file.f) != 0) return set_error(GEAR_ERR_INVALID_ARG, "checkpoint flush failed");
  return GEAR_OK;
}

gear_status gear_table_load(gear_table* t, const char* path) {
  clear_error();
  if (t == nullptr || path == nullptr) return set_error(GEAR_ERR_INVALID_ARG, "NULL argument");
  GEAR_CUDA(cudaSetDevice(t->device));
  GEAR_CUDA(cudaDeviceSynchronize());
  File file;
  file.f = fopen(path, "rb");
  if (!file.f) return set_error(GEAR_ERR_INVALID_ARG, "cannot open %s", path);
  Header h{};
  GEAR_TRY(rd(file.f, &h, sizeof(h)));
  const Header want = make_header(t);
  if (std::memcmp(h.magic, kMagic, 8) != 0 || h.version != kVersion)
    return set_error(GEAR_ERR_INVALID_ARG, "%s is not a gear checkpoint (v%u)", path, kVersion);
  if (std::memcmp(&h, &want, sizeof(h)) != 0)
    return set_error(GEAR_ERR_INVALID_ARG,
                     "%s was written by a table of another layout or world (N, W, R, rank, columns)",
                     path);
  Pinned stage;
  GEAR_CUDA(cudaHostAlloc((void**)&stage.p, kStage, cudaHostAllocDefault));
  GEAR_TRY(file_to_dev(file.f, t->key, t->Clocal * 8, stage.p));
  GEAR_TRY(file_to_dev(file.f, t->seq, t->Clocal * 8, stage.p));
  GEAR_TRY(file_to_dev(file.f, t->gen, t->Clocal * 4, stage.p));
  std::vector<AllocState> a(t->R);
  std::vector<uint32_t> ord(t->Cs);
  for (uint32_t ls = 0; ls < t->R; ++ls) {
    uint64_t st[4];
    GEAR_TRY(rd(file.f, st, sizeof(st)));
    a[ls].next_free = st[0];
    a[ls].head = (uint32_t)st[1];
    a[ls].len = (uint32_t)st[2];
    a[ls].seq_ctr = st[3];
    GEAR_TRY(rd(file.f, ord.data(), t->Cs * 4));
    GEAR_CUDA(cudaMemcpy(t->ord + (uint64_t)ls * t->Cs, ord.data(), t->Cs * 4,
                         cudaMemcpyHostToDevice));
  }
  GEAR_CUDA(cudaMemcpy(t->d_alloc, a.data(), t->R * sizeof(AllocState), cudaMemcpyHostToDevice));
  for (ColumnState& c : t->cols) {
    if (c.placement == GEAR_DEVICE) GEAR_TRY(file_to_dev(file.f, c.local, c.bytes_local, stage.p));
    else GEAR_TRY(rd(file.f, c.local, c.bytes_local));
  }
  // tags of the update pass are scratch: clear them; the CDF is rebuilt by
  // the next sample
  GEAR_CUDA(cudaMemset(t->tag, 0, t->Clocal * 8));
  GEAR_CUDA(cudaDeviceSynchronize());
  t->dirty = true;
  GEAR_CUDA(cudaMemset(t->cdf_buf_mode, 0, 8));  // two-level CDF: rescan every tile
  return GEAR_OK;
}

}  // extern "C"
