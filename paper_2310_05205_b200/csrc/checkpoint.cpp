// checkpoint.cpp -- shard checkpoint / restore ("GEAR allows
// for trajectory shards to be checkpointed on local SSDs ... at data epoch
// boundaries").  One file per rank holds that rank's R shards: a header that
// pins the layout and the schema, the slot state (keys, seq, gen), the
// insertion rings and every column's rows.  Device rows stream through a
// pinned staging buffer.
//
// File format v3 (every integer little-endian, written field by field):
//   magic "GEARCKPT", u32 version, u32 W, u32 R, u32 rank, u32 ncols, u32 F,
//   u32 removal, u64 N, u64 C_s, f64 alpha (IEEE bits as u64), u64 schema
//   hash (FNV-1a of seq_len and every column's name, dtype, shape,
//   placement), ncols x {u64 row bytes, u32 placement}; then key u64[R*C_s],
//   seq u64[R*C_s], gen u32[R*C_s], R x {u64 next_free, head, len, seq_ctr,
//   u32 ord[C_s]}, then every column's R*C_s rows.
// Save writes `path`.tmp, flushes and fsyncs it, and renames it over `path`,
// so a failed save never destroys the previous checkpoint.  Load checks the
// header AND the file size before it overwrites anything.
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "runtime.h"

using namespace gear;

namespace {

constexpr char kMagic[8] = {'G', 'E', 'A', 'R', 'C', 'K', 'P', 'T'};
constexpr uint32_t kVersion = 3;
constexpr size_t kStage = 64ull << 20;

void put(std::vector<uint8_t>& b, uint64_t v, int nbytes) {
  for (int k = 0; k < nbytes; ++k) b.push_back((uint8_t)(v >> (8 * k)));
}

std::vector<uint8_t> make_header(const gear_table* t) {
  std::vector<uint8_t> b(kMagic, kMagic + 8);
  put(b, kVersion, 4);
  put(b, t->W, 4);
  put(b, t->R, 4);
  put(b, t->rank, 4);
  put(b, t->cols.size(), 4);
  put(b, t->F, 4);
  put(b, (uint32_t)t->removal, 4);
  put(b, t->N, 8);
  put(b, t->Cs, 8);
  uint64_t ab;
  std::memcpy(&ab, &t->alpha, 8);
  put(b, ab, 8);
  put(b, t->schema_hash, 8);
  for (const ColumnState& c : t->cols) {
    put(b, c.rb, 8);
    put(b, (uint32_t)c.placement, 4);
  }
  return b;
}

uint64_t payload_bytes(const gear_table* t) {
  uint64_t n = t->Clocal * (8 + 8 + 4) + (uint64_t)t->R * (32 + 4 * t->Cs);
  for (const ColumnState& c : t->cols) n += c.bytes_local;
  return n;
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

uint64_t get(const uint8_t* p, int nbytes) {
  uint64_t v = 0;
  for (int k = 0; k < nbytes; ++k) v |= (uint64_t)p[k] << (8 * k);
  return v;
}

// Device <-> file through a pinned staging buffer (the u64 / u32 state
// arrays are stored in the host's byte order, little-endian on every
// platform this library builds for: x86-64 / aarch64 hosts of a B200).
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

static_assert(__BYTE_ORDER__ == __ORDER_LITTLE_ENDIAN__, "checkpoint arrays are little-endian");

gear_status save_to(gear_table* t, FILE* f, const std::vector<AllocState>& a) {
  Pinned stage;
  GEAR_CUDA(cudaHostAlloc((void**)&stage.p, kStage, cudaHostAllocDefault));
  const std::vector<uint8_t> h = make_header(t);
  GEAR_TRY(wr(f, h.data(), h.size()));
  GEAR_TRY(dev_to_file(f, t->key, t->Clocal * 8, stage.p));
  GEAR_TRY(dev_to_file(f, t->seq, t->Clocal * 8, stage.p));
  GEAR_TRY(dev_to_file(f, t->gen, t->Clocal * 4, stage.p));
  std::vector<uint32_t> ord(t->Cs);
  for (uint32_t ls = 0; ls < t->R; ++ls) {
    const uint64_t st[4] = {a[ls].next_free, a[ls].head, a[ls].len, a[ls].seq_ctr};
    GEAR_TRY(wr(f, st, sizeof(st)));
    GEAR_CUDA(cudaMemcpy(ord.data(), t->ord + (uint64_t)ls * t->Cs, t->Cs * 4,
                         cudaMemcpyDeviceToHost));
    GEAR_TRY(wr(f, ord.data(), t->Cs * 4));
  }
  for (const ColumnState& c : t->cols) {
    if (c.placement == GEAR_DEVICE) GEAR_TRY(dev_to_file(f, c.local, c.bytes_local, stage.p));
    else GEAR_TRY(wr(f, c.local, c.bytes_local));
  }
  if (fflush(f) != 0 || fsync(fileno(f)) != 0)
    return set_error(GEAR_ERR_INVALID_ARG, "checkpoint flush / fsync failed");
  return GEAR_OK;
}

}  // namespace

extern "C" {

gear_status gear_table_save(gear_table* t, const char* path) {
  GEAR_NVTX("gear_table_save");
  clear_error();
  if (t == nullptr || path == nullptr) return set_error(GEAR_ERR_INVALID_ARG, "NULL argument");
  GEAR_CUDA(cudaSetDevice(t->device));
  GEAR_CUDA(cudaDeviceSynchronize());
  // the device-resident allocator state of every local shard; slots taken
  // from the free queue or evicted (next_free) but not in the commit ring
  // (len) are ongoing allocations (reading Q21): they would be lost on
  // restore, so a checkpoint with one in flight is refused
  std::vector<AllocState> a(t->R);
  GEAR_CUDA(cudaMemcpy(a.data(), t->d_alloc, t->R * sizeof(AllocState), cudaMemcpyDeviceToHost));
  for (uint32_t ls = 0; ls < t->R; ++ls)
    if (a[ls].next_free != a[ls].len)
      return set_error(GEAR_ERR_STATE,
                       "shard %u has %llu allocated but uncommitted slots: commit them before "
                       "gear_table_save",
                       t->rank * t->R + ls, (unsigned long long)(a[ls].next_free - a[ls].len));
  const std::string tmp = std::string(path) + ".tmp";
  gear_status st;
  {
    File file;
    file.f = fopen(tmp.c_str(), "wb");
    if (!file.f) return set_error(GEAR_ERR_INVALID_ARG, "cannot open %s for writing", tmp.c_str());
    st = save_to(t, file.f, a);
    if (st == GEAR_OK) {
      const int rc = fclose(file.f);
      file.f = nullptr;
      if (rc != 0) st = set_error(GEAR_ERR_INVALID_ARG, "checkpoint close failed");
    }
  }
  if (st != GEAR_OK) {
    unlink(tmp.c_str());
    return st;
  }
  if (rename(tmp.c_str(), path) != 0) {
    unlink(tmp.c_str());
    return set_error(GEAR_ERR_INVALID_ARG, "cannot rename %s to %s", tmp.c_str(), path);
  }
  return GEAR_OK;
}

gear_status gear_table_load(gear_table* t, const char* path) {
  GEAR_NVTX("gear_table_load");
  clear_error();
  if (t == nullptr || path == nullptr) return set_error(GEAR_ERR_INVALID_ARG, "NULL argument");
  GEAR_CUDA(cudaSetDevice(t->device));
  GEAR_CUDA(cudaDeviceSynchronize());
  File file;
  file.f = fopen(path, "rb");
  if (!file.f) return set_error(GEAR_ERR_INVALID_ARG, "cannot open %s", path);
  const std::vector<uint8_t> want = make_header(t);
  std::vector<uint8_t> h(want.size());
  if (fread(h.data(), 1, 12, file.f) != 12 || std::memcmp(h.data(), kMagic, 8) != 0)
    return set_error(GEAR_ERR_INVALID_ARG, "%s is not a gear checkpoint", path);
  if (get(h.data() + 8, 4) != kVersion)
    return set_error(GEAR_ERR_INVALID_ARG, "%s is checkpoint version %llu, this library reads v%u",
                     path, (unsigned long long)get(h.data() + 8, 4), kVersion);
  GEAR_TRY(rd(file.f, h.data() + 12, h.size() - 12));
  if (h != want) {
    const size_t hash_at = 8 + 4 * 7 + 8 * 3;
    if (std::memcmp(h.data(), want.data(), hash_at) == 0 &&
        std::memcmp(h.data() + hash_at, want.data() + hash_at, 8) != 0)
      return set_error(GEAR_ERR_INVALID_ARG,
                       "%s was written by a table of another schema (column names, dtypes, shapes, "
                       "placement or seq_len differ)", path);
    return set_error(GEAR_ERR_INVALID_ARG,
                     "%s was written by a table of another layout or world (N, W, R, rank, F, "
                     "alpha, columns)", path);
  }
  struct stat sb;
  if (fstat(fileno(file.f), &sb) != 0 ||
      (uint64_t)sb.st_size != want.size() + payload_bytes(t))
    return set_error(GEAR_ERR_INVALID_ARG, "%s has %lld bytes, a checkpoint of this table has %llu",
                     path, (long long)sb.st_size,
                     (unsigned long long)(want.size() + payload_bytes(t)));
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
  // tags of the update pass are scratch: clear them (every later tag's epoch
  // is above 0); the CDF is rebuilt by the next sample
  GEAR_CUDA(cudaMemset(t->tag, 0, t->Clocal * 8));
  GEAR_CUDA(cudaDeviceSynchronize());
  t->dirty = true;
  GEAR_CUDA(cudaMemset(t->cdf_buf_mode, 0, 8));  // two-level CDF: rescan every tile
  return GEAR_OK;
}

}  // extern "C"
