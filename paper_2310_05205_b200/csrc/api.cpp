// api.cpp -- the C-ABI of include/gear.h: argument validation, table memory,
// peer mappings and the orchestration of the sm_100a kernels.
//
// Every step of the hot path runs on the GPU, the block allocator of the
// writers included (kernels/alloc.cu): this file only validates, allocates,
// stages small host arrays and enqueues kernels / NCCL calls on the caller's
// stream.
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <random>

#include "runtime.h"

using namespace gear;

namespace {

TileDirty tile_dirty(const gear_table* t) {
  TileDirty d{};
  d.bits = t->tile_dirty;
  d.shard_cap = t->Cs;
  d.tiles_per_shard = scan_tiles_per_shard(t->Cs);
  return d;
}

Quant quant(const gear_table* t) {
  Quant q{};
  q.q_max = t->qmax;
  q.frac_bits = t->F;
  q.alpha = t->alpha;
  return q;
}

uint64_t dtype_size(gear_dtype d) {
  switch (d) {
    case GEAR_U8: return 1;
    case GEAR_I32: return 4;
    case GEAR_I64: return 8;
    case GEAR_F32: return 4;
    case GEAR_F64: return 8;
    case GEAR_BF16: return 2;
  }
  return 0;
}

template <class T>
gear_status dalloc(T** p, size_t n) {
  *p = nullptr;
  if (n == 0) n = 1;
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), n * sizeof(T));
  if (e != cudaSuccess) {
    cudaGetLastError();
    return set_error(GEAR_ERR_OUT_OF_MEMORY, "cudaMalloc(%zu bytes): %s", n * sizeof(T),
                     cudaGetErrorString(e));
  }
  return GEAR_OK;
}

template <class T>
void dfree(T*& p) {
  if (p) cudaFree(const_cast<void*>(reinterpret_cast<const void*>(p)));
  p = nullptr;
}

// Maps `bytes` of host memory and registers it with CUDA as mapped pinned
// memory.  shm_name empty: private anonymous memory (W = 1); otherwise a POSIX
// shared-memory object (created if `create`), so every rank's GPU can map the
// same pages.
constexpr size_t kHostRegChunkDefault = size_t(64) << 30;

// GEAR_HOST_REG_CHUNK (bytes, a multiple of 2 MiB): a smaller piece size, so
// tests cover rows that straddle two registrations.
size_t host_reg_chunk() {
  if (const char* e = getenv("GEAR_HOST_REG_CHUNK")) {
    const size_t v = (size_t)strtoull(e, nullptr, 10);
    if (v >= (size_t(2) << 20) && v % (size_t(2) << 20) == 0) return v;
  }
  return kHostRegChunkDefault;
}

gear_status map_host(const std::string& shm_name, bool create, size_t bytes, size_t piece,
                     void** out) {
  *out = nullptr;
  void* p = MAP_FAILED;
  if (shm_name.empty()) {
    p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
  } else {
    int fd = shm_open(shm_name.c_str(), create ? (O_CREAT | O_EXCL | O_RDWR) : O_RDWR, 0600);
    if (fd < 0) return set_error(GEAR_ERR_OUT_OF_MEMORY, "shm_open(%s) failed", shm_name.c_str());
    if (create && ftruncate(fd, (off_t)bytes) != 0) {
      close(fd);
      shm_unlink(shm_name.c_str());
      return set_error(GEAR_ERR_OUT_OF_MEMORY, "ftruncate(%s, %zu) failed", shm_name.c_str(),
                       bytes);
    }
    p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
  }
  if (p == MAP_FAILED) return set_error(GEAR_ERR_OUT_OF_MEMORY, "mmap(%zu) failed", bytes);
  madvise(p, bytes, MADV_HUGEPAGE);
  // One registration per piece: a single cudaHostRegister of ~300 GB
  // fails on the 4-GPU boxes ("OS call failed"), 64 GiB pieces do not.  The
  // pieces form one contiguous device range because registered memory is
  // mapped at its host address (checked below; UVA).
  size_t done = 0;
  cudaError_t e = cudaSuccess;
  for (; done < bytes; done += piece) {
    uint8_t* c = (uint8_t*)p + done;
    size_t n = std::min(piece, bytes - done);
    e = cudaHostRegister(c, n, cudaHostRegisterMapped | cudaHostRegisterPortable);
    if (e != cudaSuccess) break;
    void* dp = nullptr;
    if (cudaHostGetDevicePointer(&dp, c, 0) != cudaSuccess || dp != (void*)c) {
      cudaHostUnregister(c);
      e = cudaErrorNotSupported;
      break;
    }
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    for (size_t o = 0; o < done; o += piece) cudaHostUnregister((uint8_t*)p + o);
    munmap(p, bytes);
    return set_error(GEAR_ERR_OUT_OF_MEMORY, "cudaHostRegister(%zu of %zu bytes at offset %zu): %s",
                     std::min(piece, bytes - done), bytes, done, cudaGetErrorString(e));
  }
  *out = p;
  return GEAR_OK;
}

void unmap_host(void* p, size_t bytes, size_t piece) {
  for (size_t o = 0; o < bytes; o += piece) cudaHostUnregister((uint8_t*)p + o);
  munmap(p, bytes);
}

// Exchange a CUDA-IPC handle for `local` and open every peer's allocation.
gear_status exchange_ipc(gear_table* t, void* local, void** views, std::vector<void*>& opened) {
  gear_comm* c = t->comm;
  cudaIpcMemHandle_t h;
  GEAR_CUDA(cudaIpcGetMemHandle(&h, local));
  uint8_t* d_send = nullptr;
  uint8_t* d_recv = nullptr;
  GEAR_TRY(dalloc(&d_send, sizeof(h)));
  GEAR_TRY(dalloc(&d_recv, sizeof(h) * t->W));
  GEAR_CUDA(cudaMemcpy(d_send, &h, sizeof(h), cudaMemcpyHostToDevice));
  GEAR_TRY(allgather_bytes(c, d_send, d_recv, sizeof(h), c->stream));
  GEAR_CUDA(cudaStreamSynchronize(c->stream));
  std::vector<cudaIpcMemHandle_t> all(t->W);
  GEAR_CUDA(cudaMemcpy(all.data(), d_recv, sizeof(h) * t->W, cudaMemcpyDeviceToHost));
  dfree(d_send);
  dfree(d_recv);
  for (uint32_t r = 0; r < t->W; ++r) {
    if (r == t->rank) {
      views[r] = local;
      continue;
    }
    void* p = nullptr;
    GEAR_CUDA(cudaIpcOpenMemHandle(&p, all[r], cudaIpcMemLazyEnablePeerAccess));
    views[r] = p;
    opened.push_back(p);
  }
  return GEAR_OK;
}

void destroy_table(gear_table* t) {
  if (!t) return;
  cudaSetDevice(t->device);
  cudaDeviceSynchronize();
  for (auto& c : t->cols) {
    for (void* p : c.ipc_opened) cudaIpcCloseMemHandle(p);
    for (auto& m : c.host_maps) unmap_host(m.first, m.second, c.host_reg_chunk);
    if (c.placement == GEAR_DEVICE && c.local) cudaFree(c.local);
  }
  for (void* p : t->ipc_opened) cudaIpcCloseMemHandle(p);
  for (void* p : t->mbox_opened) cudaIpcCloseMemHandle(p);
  dfree(t->mbox);
  dfree(t->key); dfree(t->seq); dfree(t->gen); dfree(t->tag); dfree(t->ord);
  for (int i = 0; i < 2; ++i) {
    dfree(t->cdf[i]); dfree(t->scan_status[i]); dfree(t->scan_ticket[i]);
  }
  dfree(t->cdf_totals_local); dfree(t->cdf_totals_all);
  dfree(t->tile_dirty); dfree(t->tile_tot); dfree(t->cdf_buf_mode); dfree(t->scan2_ctr);
  dfree(t->fifo_totals_local); dfree(t->fifo_totals_all);
  dfree(t->d_cdf_ptrs); dfree(t->d_gen_ptrs);
  dfree(t->q_scratch); dfree(t->qmin_slot); dfree(t->done_ctr);
  dfree(t->tmp_idx); dfree(t->tmp_w); dfree(t->tmp_p); dfree(t->tmp_gen);
  dfree(t->cand_local); dfree(t->cand_all);
  dfree(t->topk_state); dfree(t->topk_cnt); dfree(t->topk_tmp);
  dfree(t->draw_list); dfree(t->pos_scratch); dfree(t->ov_scratch);
  dfree(t->glob_shard); dfree(t->glob_slot);
  dfree(t->upd_local); dfree(t->upd_all); dfree(t->upd_idx); dfree(t->upd_prio); dfree(t->upd_pow); dfree(t->upd_gen);
  dfree(t->n_stale); dfree(t->err); dfree(t->d_epoch); dfree(t->d_seed); dfree(t->d_xep);
  for (auto& b : t->col_idx) dfree(b.p);
  dfree(t->d_meta); dfree(t->d_ord); dfree(t->d_out); dfree(t->d_rows);
  dfree(t->d_prio_ins); dfree(t->d_alloc); dfree(t->ins_bad); dfree(t->dyn_pool);
  if (t->h_prio) cudaFreeHost(t->h_prio);
  if (t->h_out) cudaFreeHost(t->h_out);
  if (t->staging_ev) cudaEventDestroy(t->staging_ev);
  delete t;
}

gear_status create_table(const gear_table_desc* d, gear_comm* comm, gear_table* t) {
  t->comm = comm;
  GEAR_CUDA(cudaGetDevice(&t->device));
  if (comm) {
    t->device = comm->device;
    GEAR_CUDA(cudaSetDevice(t->device));
    t->W = (uint32_t)comm->nranks;
    t->rank = (uint32_t)comm->rank;
  }
  t->R = d->shards_per_rank ? d->shards_per_rank : 1;
  t->S = t->W * t->R;
  if (t->S > (uint32_t)kMaxShards)
    return set_error(GEAR_ERR_INVALID_ARG, "W*R = %u shards > %d", t->S, kMaxShards);
  t->N = d->capacity_global;
  if (t->N == 0 || t->N % t->S)
    return set_error(GEAR_ERR_INVALID_ARG, "capacity_global %llu not a positive multiple of %u shards",
                     (unsigned long long)t->N, t->S);
  t->Cs = t->N / t->S;
  if (t->Cs >= (1ull << 32))
    return set_error(GEAR_ERR_INVALID_ARG, "shard capacity must be < 2^32");
  t->Clocal = t->Cs * t->R;
  t->F = d->priority_frac_bits ? d->priority_frac_bits : 32;
  if (t->F > 62) return set_error(GEAR_ERR_INVALID_ARG, "priority_frac_bits > 62");
  t->qmax = ((1ull << 62) - 1) / t->N;
  if (!std::isfinite(d->priority_alpha) || d->priority_alpha < 0.0)
    return set_error(GEAR_ERR_INVALID_ARG, "priority_alpha must be finite and >= 0");
  t->alpha = d->priority_alpha == 0.0 ? 1.0 : d->priority_alpha;
  t->removal = d->removal;
  if (t->removal != GEAR_REMOVE_FIFO && t->removal != GEAR_REMOVE_LIFO)
    return set_error(GEAR_ERR_INVALID_ARG, "bad removal");
  t->max_batch = d->max_batch ? d->max_batch : 4096;
  if ((uint64_t)t->W * t->max_batch >= (1ull << kTagLowBits))
    return set_error(GEAR_ERR_INVALID_ARG, "W * max_batch must be < 2^%d", kTagLowBits);
  if (d->seq_len == 0) return set_error(GEAR_ERR_INVALID_ARG, "seq_len == 0");
  if (d->ncols == 0 || d->ncols > (uint32_t)kMaxCols || d->cols == nullptr)
    return set_error(GEAR_ERR_INVALID_ARG, "ncols must be 1..%d", kMaxCols);
  if (const char* e = getenv("GEAR_COLLECT_CHUNK")) t->chunk_bytes = (uint32_t)atoi(e);
  if (const char* e = getenv("GEAR_TMA_CHUNK")) t->tma_chunk = (uint32_t)atoi(e);
  if (const char* e = getenv("GEAR_COLLECT_PEER_LSU")) t->collect_peer_lsu = atoi(e) != 0;
  if (const char* e = getenv("GEAR_COLLECT_HOST_LSU")) t->collect_host_lsu = atoi(e) < 0 ? -1 : (atoi(e) != 0);
  if (const char* e = getenv("GEAR_PEER_XCHG")) t->peer_xchg = atoi(e) != 0;  // A/B (same on every rank)
  if (const char* e = getenv("GEAR_COLLECT_DYNAMIC")) t->collect_dynamic = atoi(e);
  if (const char* e = getenv("GEAR_COLLECT_EVICT_FIRST")) t->evict_first = atoi(e);
  if (const char* e = getenv("GEAR_TMA_STAGES")) {
    const int v = atoi(e);
    if (v == 2 || v == 3 || v == 4 || v == 6 || v == 8) t->tma_stages = v;
  }
  if (const char* e = getenv("GEAR_TMA_CTAS")) {
    const int v = atoi(e);
    if (v >= 1 && v <= 8) t->tma_ctas = v;
  }
  if ((uint64_t)t->tma_ctas * t->tma_stages * t->tma_chunk > (220u << 10))
    return set_error(GEAR_ERR_INVALID_ARG, "GEAR_TMA_CTAS * GEAR_TMA_STAGES * tma_chunk > 220 KB");
  if (const char* e = getenv("GEAR_COLLECT_IMPL")) t->collect_impl = strcmp(e, "lsu") == 0 ? 0 : 1;
  if (t->tma_chunk < 4096 || t->tma_chunk % 16 || t->tma_chunk > 32768)
    return set_error(GEAR_ERR_INVALID_ARG, "GEAR_TMA_CHUNK must be a multiple of 16 in [4096, 32768]");
  if (t->chunk_bytes < 512 || t->chunk_bytes % 512)
    return set_error(GEAR_ERR_INVALID_ARG, "GEAR_COLLECT_CHUNK must be a multiple of 512");

  // Column layout.
  t->cols.resize(d->ncols);
  for (uint32_t c = 0; c < d->ncols; ++c) {
    const gear_column_desc& cd = d->cols[c];
    ColumnState& cs = t->cols[c];
    if (cd.name == nullptr || cd.name[0] == 0 || strlen(cd.name) > 63)
      return set_error(GEAR_ERR_INVALID_ARG, "column %u: empty or long name", c);
    for (uint32_t o = 0; o < c; ++o)
      if (t->cols[o].name == cd.name)
        return set_error(GEAR_ERR_INVALID_ARG, "duplicate column name %s", cd.name);
    if (dtype_size(cd.dtype) == 0) return set_error(GEAR_ERR_INVALID_ARG, "column %s: bad dtype", cd.name);
    if (cd.ndim > 8 || (cd.ndim > 0 && cd.shape == nullptr))
      return set_error(GEAR_ERR_INVALID_ARG, "column %s: bad shape", cd.name);
    uint64_t elems = d->seq_len;
    for (uint32_t k = 0; k < cd.ndim; ++k) {
      if (cd.shape[k] <= 0) return set_error(GEAR_ERR_INVALID_ARG, "column %s: zero-size shape", cd.name);
      elems *= (uint64_t)cd.shape[k];
    }
    if (cd.placement != GEAR_DEVICE && cd.placement != GEAR_HOST)
      return set_error(GEAR_ERR_INVALID_ARG, "column %s: bad placement", cd.name);
    cs.name = cd.name;
    cs.dtype = cd.dtype;
    cs.placement = cd.placement;
    cs.rb = elems * dtype_size(cd.dtype);
    cs.bytes_local = cs.rb * t->Clocal;
  }
  // schema hash (checkpoints): FNV-1a 64 over little-endian field encodings
  t->seq_len = d->seq_len;
  {
    uint64_t h = 0xcbf29ce484222325ull;
    auto mix = [&h](uint64_t v, int nbytes) {
      for (int b = 0; b < nbytes; ++b) {
        h ^= (v >> (8 * b)) & 0xff;
        h *= 0x100000001b3ull;
      }
    };
    mix(d->seq_len, 4);
    mix(d->ncols, 4);
    for (uint32_t c = 0; c < d->ncols; ++c) {
      const gear_column_desc& cd = d->cols[c];
      const size_t L = strlen(cd.name);
      mix(L, 4);
      for (size_t k = 0; k < L; ++k) mix((uint8_t)cd.name[k], 1);
      mix((uint32_t)cd.dtype, 4);
      mix(cd.ndim, 4);
      for (uint32_t k = 0; k < cd.ndim; ++k) mix((uint64_t)cd.shape[k], 8);
      mix((uint32_t)cd.placement, 4);
    }
    t->schema_hash = h;
  }

  // A per-table tag for shared-memory names (rank 0 draws it, all-gathered).
  uint64_t tag = 0;
  if (t->W > 1) {
    std::random_device rd;
    uint64_t mine = ((uint64_t)rd() << 32) ^ rd() ^ (uint64_t)getpid();
    uint64_t *d_s = nullptr, *d_r = nullptr;
    GEAR_TRY(dalloc(&d_s, 1));
    GEAR_TRY(dalloc(&d_r, t->W));
    GEAR_CUDA(cudaMemcpy(d_s, &mine, 8, cudaMemcpyHostToDevice));
    GEAR_TRY(allgather_bytes(comm, d_s, d_r, 8, comm->stream));
    GEAR_CUDA(cudaStreamSynchronize(comm->stream));
    GEAR_CUDA(cudaMemcpy(&tag, d_r, 8, cudaMemcpyDeviceToHost));  // rank 0's value
    dfree(d_s);
    dfree(d_r);
  }

  // Column memory.
  for (uint32_t c = 0; c < d->ncols; ++c) {
    ColumnState& cs = t->cols[c];
    if (cs.placement == GEAR_DEVICE) {
      GEAR_TRY(dalloc(&cs.local, cs.bytes_local));
      if (t->W > 1) {
        void* views[kMaxRanks] = {};
        GEAR_TRY(exchange_ipc(t, cs.local, views, cs.ipc_opened));
        for (uint32_t r = 0; r < t->W; ++r) cs.view[r] = (const uint8_t*)views[r];
      } else {
        cs.view[0] = cs.local;
      }
    } else {
      cs.host_reg_chunk = host_reg_chunk();
      if (t->W == 1) {
        void* p = nullptr;
        // GEAR_HOST_SHM=1: use a shared-memory object even at W = 1 (to
        // compare page backing with the W > 1 path)
        std::string nm;
        if (const char* e = getenv("GEAR_HOST_SHM"); e && e[0] == '1') {
          char b[96];
          snprintf(b, sizeof(b), "/gear_w1_%d_c%u", (int)getpid(), c);
          nm = b;
        }
        GEAR_TRY(map_host(nm, true, cs.bytes_local, cs.host_reg_chunk, &p));
        if (!nm.empty()) shm_unlink(nm.c_str());
        cs.host_maps.emplace_back(p, cs.bytes_local);
        cs.local = (uint8_t*)p;
        void* dp = nullptr;
        GEAR_CUDA(cudaHostGetDevicePointer(&dp, p, 0));
        cs.view[0] = (const uint8_t*)dp;
      } else {
        char nm[96];
        snprintf(nm, sizeof(nm), "/gear_%016llx_c%u_r%u", (unsigned long long)tag, c, t->rank);
        cs.shm_name = nm;
        void* p = nullptr;
        GEAR_TRY(map_host(cs.shm_name, true, cs.bytes_local, cs.host_reg_chunk, &p));
        cs.host_maps.emplace_back(p, cs.bytes_local);
        cs.local = (uint8_t*)p;
        GEAR_TRY(barrier(comm));
        for (uint32_t r = 0; r < t->W; ++r) {
          void* q = p;
          if (r != t->rank) {
            snprintf(nm, sizeof(nm), "/gear_%016llx_c%u_r%u", (unsigned long long)tag, c, r);
            GEAR_TRY(map_host(nm, false, cs.bytes_local, cs.host_reg_chunk, &q));
            cs.host_maps.emplace_back(q, cs.bytes_local);
          }
          void* dp = nullptr;
          GEAR_CUDA(cudaHostGetDevicePointer(&dp, q, 0));
          cs.view[r] = (const uint8_t*)dp;
        }
        GEAR_TRY(barrier(comm));
        shm_unlink(cs.shm_name.c_str());
      }
    }
  }

  // Slot state.
  GEAR_TRY(dalloc(&t->key, t->Clocal));
  GEAR_TRY(dalloc(&t->seq, t->Clocal));
  GEAR_TRY(dalloc(&t->gen, t->Clocal));
  GEAR_TRY(dalloc(&t->tag, t->Clocal));
  GEAR_TRY(dalloc(&t->ord, t->Clocal));
  GEAR_CUDA(cudaMemset(t->key, 0, t->Clocal * 8));
  GEAR_CUDA(cudaMemset(t->seq, 0, t->Clocal * 8));
  GEAR_CUDA(cudaMemset(t->gen, 0, t->Clocal * 4));
  GEAR_CUDA(cudaMemset(t->tag, 0, t->Clocal * 8));
  GEAR_CUDA(cudaMemset(t->ord, 0, t->Clocal * 4));
  const uint32_t tiles = scan_tiles_per_shard(t->Cs) * t->R;
  for (int i = 0; i < 2; ++i) {
    // flat CDF (R*C_s), or tile-local prefixes (R*C_s) + tile prefixes (tiles)
    GEAR_TRY(dalloc(&t->cdf[i], t->Clocal + tiles));
    GEAR_CUDA(cudaMemset(t->cdf[i], 0, (t->Clocal + tiles) * 8));
    GEAR_TRY(dalloc(&t->scan_status[i], (size_t)tiles * 16));  // room for a padded layout
    GEAR_CUDA(cudaMemset(t->scan_status[i], 0, (size_t)tiles * 16 * 8));
    GEAR_TRY(dalloc(&t->scan_ticket[i], 2));  // [0] counter, [1] scan epoch (flat scan)
    GEAR_CUDA(cudaMemset(t->scan_ticket[i], 0, 8));
  }
  // two-level CDF bookkeeping: nothing built yet (buffer modes 0) -> the first
  // rebuild of each buffer rescans every tile
  GEAR_TRY(dalloc(&t->tile_dirty, tiles));
  GEAR_CUDA(cudaMemset(t->tile_dirty, 0, tiles * 4));
  GEAR_TRY(dalloc(&t->tile_tot, 2 * (size_t)tiles));
  GEAR_TRY(dalloc(&t->cdf_buf_mode, 2));
  GEAR_CUDA(cudaMemset(t->cdf_buf_mode, 0, 8));
  GEAR_TRY(dalloc(&t->scan2_ctr, t->R + 1));
  GEAR_CUDA(cudaMemset(t->scan2_ctr, 0, (t->R + 1) * 4));
  GEAR_TRY(dalloc(&t->cdf_totals_local, t->R));
  GEAR_TRY(dalloc(&t->cdf_totals_all, t->S));
  GEAR_TRY(dalloc(&t->fifo_totals_local, t->R));
  GEAR_TRY(dalloc(&t->fifo_totals_all, t->S));
  GEAR_CUDA(cudaMemset(t->cdf_totals_local, 0, t->R * sizeof(ShardTotals)));
  GEAR_CUDA(cudaMemset(t->cdf_totals_all, 0, t->S * sizeof(ShardTotals)));

  // Pointer tables: every shard's two CDF buffers and every rank's gen array.
  std::vector<const uint64_t*> cdf_ptrs(2 * t->S);
  std::vector<const uint32_t*> gen_ptrs(t->W);
  if (t->W > 1) {
    void* v0[kMaxRanks] = {};
    void* v1[kMaxRanks] = {};
    void* vg[kMaxRanks] = {};
    GEAR_TRY(exchange_ipc(t, t->cdf[0], v0, t->ipc_opened));
    GEAR_TRY(exchange_ipc(t, t->cdf[1], v1, t->ipc_opened));
    GEAR_TRY(exchange_ipc(t, t->gen, vg, t->ipc_opened));
    for (uint32_t r = 0; r < t->W; ++r) {
      gen_ptrs[r] = (const uint32_t*)vg[r];
      for (uint32_t ls = 0; ls < t->R; ++ls) {
        cdf_ptrs[0 * t->S + r * t->R + ls] = (const uint64_t*)v0[r] + ls * t->Cs;
        cdf_ptrs[1 * t->S + r * t->R + ls] = (const uint64_t*)v1[r] + ls * t->Cs;
      }
    }
  } else {
    gen_ptrs[0] = t->gen;
    for (uint32_t ls = 0; ls < t->R; ++ls) {
      cdf_ptrs[ls] = t->cdf[0] + ls * t->Cs;
      cdf_ptrs[t->S + ls] = t->cdf[1] + ls * t->Cs;
    }
  }
  GEAR_TRY(dalloc(&t->d_cdf_ptrs, 2 * t->S));
  GEAR_TRY(dalloc(&t->d_gen_ptrs, t->W));
  GEAR_CUDA(cudaMemcpy(t->d_cdf_ptrs, cdf_ptrs.data(), 2 * t->S * sizeof(void*), cudaMemcpyHostToDevice));
  GEAR_CUDA(cudaMemcpy(t->d_gen_ptrs, gen_ptrs.data(), t->W * sizeof(void*), cudaMemcpyHostToDevice));

  // Peer mailboxes for the per-step exchanges (W > 1), mapped by every rank.
  if (t->W > 1) {
    const MboxLayout L = mbox_layout(t->W, t->S, t->max_batch);
    GEAR_TRY(dalloc(&t->mbox, L.bytes));
    GEAR_CUDA(cudaMemset(t->mbox, 0, L.bytes));
    void* views[kMaxRanks] = {};
    GEAR_TRY(exchange_ipc(t, t->mbox, views, t->mbox_opened));
    for (uint32_t r = 0; r < t->W; ++r) t->mb.base[r] = (uint8_t*)views[r];
    t->mb.W = t->W;
    t->mb.rank = t->rank;
    t->mb.S = t->S;
    t->mb.R = t->R;
    t->mb.MB = t->max_batch;
    GEAR_CUDA(cudaDeviceSynchronize());
    GEAR_TRY(barrier(comm));  // every mailbox is zeroed before anyone writes
  }

  // Scratch.
  const uint64_t MB = t->max_batch, K = (uint64_t)t->W * MB;
  GEAR_TRY(dalloc(&t->q_scratch, MB));
  GEAR_TRY(dalloc(&t->qmin_slot, 1));
  GEAR_CUDA(cudaMemset(t->qmin_slot, 0xff, 8));
  GEAR_TRY(dalloc(&t->done_ctr, 1));
  GEAR_CUDA(cudaMemset(t->done_ctr, 0, 4));
  GEAR_TRY(dalloc(&t->tmp_idx, MB));
  GEAR_TRY(dalloc(&t->tmp_w, MB));
  GEAR_TRY(dalloc(&t->tmp_p, MB));
  GEAR_TRY(dalloc(&t->tmp_gen, MB));
  GEAR_TRY(dalloc(&t->draw_list, MB));
  GEAR_TRY(dalloc(&t->pos_scratch, K));
  GEAR_TRY(dalloc(&t->ov_scratch, K));
  GEAR_TRY(dalloc(&t->glob_shard, K));
  GEAR_TRY(dalloc(&t->glob_slot, K));
  GEAR_TRY(dalloc(&t->cand_local, t->R * K));
  GEAR_TRY(dalloc(&t->cand_all, t->S * K));
  GEAR_TRY(dalloc(&t->topk_tmp, 2 * t->R * (K + kTopkEqMax)));  // candidates + sorted runs
  GEAR_TRY(dalloc(&t->topk_state, t->R));
  GEAR_CUDA(cudaMemset(t->topk_state, 0, t->R * sizeof(TopkState)));
  GEAR_TRY(dalloc(&t->topk_cnt, (size_t)t->R * kTopkMaxCtas * 2));
  GEAR_TRY(dalloc(&t->upd_local, MB));
  GEAR_TRY(dalloc(&t->upd_all, K));
  GEAR_TRY(dalloc(&t->upd_idx, MB));
  GEAR_TRY(dalloc(&t->upd_prio, MB));
  GEAR_TRY(dalloc(&t->upd_pow, MB));
  GEAR_TRY(dalloc(&t->upd_gen, MB));
  GEAR_TRY(dalloc(&t->d_xep, 4));
  GEAR_CUDA(cudaMemset(t->d_xep, 0, 32));
  GEAR_TRY(dalloc(&t->d_epoch, 1));
  GEAR_CUDA(cudaMemset(t->d_epoch, 0, 8));
  GEAR_TRY(dalloc(&t->d_seed, 1));
  GEAR_CUDA(cudaMemset(t->d_seed, 0, 8));
  GEAR_TRY(dalloc(&t->n_stale, 1));
  GEAR_TRY(dalloc(&t->err, 1));
  GEAR_CUDA(cudaMemset(t->n_stale, 0, 8));
  GEAR_CUDA(cudaMemset(t->err, 0, 4));
  GEAR_CUDA(cudaHostAlloc((void**)&t->h_prio, MB * sizeof(double), cudaHostAllocDefault));
  GEAR_CUDA(cudaHostAlloc((void**)&t->h_out, MB * sizeof(uint64_t), cudaHostAllocDefault));
  GEAR_TRY(dalloc(&t->d_prio_ins, MB));
  GEAR_TRY(dalloc(&t->d_alloc, t->R));
  GEAR_TRY(dalloc(&t->dyn_pool, 2 * gear_table::kDynSlots));
  GEAR_CUDA(cudaMemset(t->dyn_pool, 0, 2 * gear_table::kDynSlots * sizeof(unsigned long long)));
  GEAR_TRY(dalloc(&t->ins_bad, 1));
  GEAR_CUDA(cudaMemset(t->ins_bad, 0, 4));
  {
    std::vector<AllocState> a0(t->R);
    for (auto& a : a0) a = AllocState{0, 1, 0, 0};  // free queue full, seq counter at 1
    GEAR_CUDA(cudaMemcpy(t->d_alloc, a0.data(), t->R * sizeof(AllocState),
                         cudaMemcpyHostToDevice));
  }
  GEAR_TRY(dalloc(&t->d_meta, MB));
  GEAR_TRY(dalloc(&t->d_ord, MB));
  GEAR_TRY(dalloc(&t->d_out, MB));
  GEAR_CUDA(cudaEventCreateWithFlags(&t->staging_ev, cudaEventDisableTiming));
  GEAR_CUDA(cudaEventRecord(t->staging_ev, 0));

  GEAR_CUDA(cudaDeviceSynchronize());
  return GEAR_OK;
}

// Make `n` elements at `user` available on the device: device pointers pass
// through, host pointers are copied into `scratch` on the stream -- except
// pinned host memory with `zero_copy`, which the kernel reads in place over
// PCIe through its mapped address (for arrays every element of which is read
// once: no copy-engine operation on the step, same stream-order lifetime rule
// as an async copy).
template <class T>
gear_status stage_in(const T* user, size_t n, T* scratch, cudaStream_t s, const T** out,
                     bool zero_copy = false) {
  const MemKind k = n == 0 ? MemKind::Device : mem_kind(user);
  if (k == MemKind::Device) {
    *out = user;
    return GEAR_OK;
  }
  if (zero_copy && k == MemKind::HostPinned) {
    void* dp = nullptr;
    if (cudaHostGetDevicePointer(&dp, const_cast<T*>(user), 0) == cudaSuccess) {
      *out = static_cast<const T*>(dp);
      return GEAR_OK;
    }
    cudaGetLastError();  // not mapped: copy instead
  }
  GEAR_CUDA(cudaMemcpyAsync(scratch, user, n * sizeof(T), cudaMemcpyHostToDevice, s));
  *out = scratch;
  return GEAR_OK;
}

// Where a kernel writes an output the caller passed: device memory as is,
// pinned host memory through its mapped address, pageable host memory into
// `scratch` (*copy_back = true: copied to the caller at the end).
template <class T>
T* out_device(T* user, T* scratch, bool* copy_back) {
  *copy_back = false;
  if (user == nullptr) return nullptr;
  const MemKind k = mem_kind(user);
  if (k == MemKind::Device) return user;
  if (k == MemKind::HostPinned) {
    void* dp = nullptr;
    if (cudaHostGetDevicePointer(&dp, user, 0) == cudaSuccess) return static_cast<T*>(dp);
    cudaGetLastError();
  }
  *copy_back = true;
  return scratch;
}

uint32_t vec_width(uint64_t rb, uint32_t chunk, std::initializer_list<uintptr_t> ptrs) {
  for (uint32_t v : {16u, 8u, 4u, 2u}) {
    bool ok = rb % v == 0 && chunk % v == 0;
    for (uintptr_t p : ptrs) ok = ok && (p % v == 0);
    if (ok) return v;
  }
  return 1;
}

AssignParams assign_params(gear_table* t, uint32_t B, uint64_t seed) {
  AssignParams ap{};
  ap.n_shards = t->S;
  ap.shards_per_rank = t->R;
  ap.W = t->W;
  ap.rank = t->rank;
  ap.B = B;
  ap.seed = seed;
  ap.shard_cap = t->Cs;
  ap.draw_list = t->draw_list;
  ap.pos_scratch = t->pos_scratch;
  ap.ov_scratch = t->ov_scratch;
  ap.gen_ptrs = t->d_gen_ptrs;
  ap.err = t->err;
  return ap;
}

gear_status check_table(const gear_table* t) {
  if (t == nullptr) return set_error(GEAR_ERR_INVALID_ARG, "table is NULL");
  return GEAR_OK;
}

}  // namespace

extern "C" {

gear_status gear_table_create(const gear_table_desc* desc, gear_comm* comm, gear_table** out) {
  GEAR_NVTX("gear_table_create");
  clear_error();
  if (desc == nullptr || out == nullptr) return set_error(GEAR_ERR_INVALID_ARG, "NULL argument");
  *out = nullptr;
  auto* t = new gear_table();
  gear_status st = create_table(desc, comm, t);
  if (st != GEAR_OK) {
    std::string msg = gear_last_error();
    destroy_table(t);
    set_error(st, "%s", msg.c_str());
    return st;
  }
  *out = t;
  return GEAR_OK;
}

gear_status gear_table_destroy(gear_table* t) {
  GEAR_NVTX("gear_table_destroy");
  if (t == nullptr) return GEAR_OK;
  gear_comm* c = t->comm;
  destroy_table(t);
  if (c) GEAR_TRY(barrier(c));
  return GEAR_OK;
}

gear_status gear_table_info_get(const gear_table* t, gear_table_info* info) {
  GEAR_NVTX("gear_table_info_get");
  GEAR_TRY(check_table(t));
  if (info == nullptr) return set_error(GEAR_ERR_INVALID_ARG, "info is NULL");
  info->capacity_global = t->N;
  info->shard_capacity = t->Cs;
  info->n_ranks = t->W;
  info->rank = t->rank;
  info->shards_per_rank = t->R;
  info->ncols = (uint32_t)t->cols.size();
  info->row_bytes_total = 0;
  for (auto& c : t->cols) info->row_bytes_total += c.rb;
  info->q_max = t->qmax;
  info->p_max = std::ldexp((double)t->qmax, -(int)t->F);
  info->frac_bits = t->F;
  info->alpha = t->alpha;
  info->max_batch = t->max_batch;
  return GEAR_OK;
}

gear_status gear_column_id(const gear_table* t, const char* name, uint32_t* out) {
  GEAR_NVTX("gear_column_id");
  GEAR_TRY(check_table(t));
  if (name == nullptr || out == nullptr) return set_error(GEAR_ERR_INVALID_ARG, "NULL argument");
  for (uint32_t c = 0; c < t->cols.size(); ++c)
    if (t->cols[c].name == name) {
      *out = c;
      return GEAR_OK;
    }
  return set_error(GEAR_ERR_INVALID_ARG, "no column named %s", name);
}

gear_status gear_column_row_bytes(const gear_table* t, uint32_t col, uint64_t* out) {
  GEAR_NVTX("gear_column_row_bytes");
  GEAR_TRY(check_table(t));
  if (out == nullptr || col >= t->cols.size())
    return set_error(GEAR_ERR_INVALID_ARG, "bad column %u", col);
  *out = t->cols[col].rb;
  return GEAR_OK;
}

gear_status gear_insert(gear_table* t, uint32_t shard, uint32_t n, const void* const* col_src,
                        const double* prio, uint64_t* out_idx, gear_stream stream) {
  GEAR_NVTX("gear_insert");
  clear_error();
  GEAR_TRY(check_table(t));
  GEAR_CUDA(cudaSetDevice(t->device));
  cudaStream_t s = (cudaStream_t)stream;
  if (shard / t->R != t->rank || shard >= t->S)
    return set_error(GEAR_ERR_INVALID_ARG, "shard %u is not owned by rank %u", shard, t->rank);
  if (n == 0) return GEAR_OK;
  if (col_src == nullptr || prio == nullptr)
    return set_error(GEAR_ERR_INVALID_ARG, "col_src / prio is NULL");
  for (size_t c = 0; c < t->cols.size(); ++c)
    if (col_src[c] == nullptr) return set_error(GEAR_ERR_INVALID_ARG, "col_src[%zu] is NULL", c);
  // Host priorities are validated here before anything is inserted (error
  // returned); device priorities by a kernel (BAD_PRIORITY latched, nothing
  // inserted), so a call with device sources and priorities never blocks the
  // host and can be captured in a CUDA graph.
  const bool dev_prio = mem_kind(prio) == MemKind::Device;
  std::vector<double> p;
  if (!dev_prio) {
    p.assign(prio, prio + n);
    for (uint32_t k = 0; k < n; ++k)
      if (!(p[k] >= 0.0) || std::isinf(p[k]))
        return set_error(GEAR_ERR_BAD_PRIORITY, "prio[%u] = %g is not a finite non-negative number",
                         k, p[k]);
  } else {
    GEAR_CUDA(launch_validate_prio(prio, n, t->ins_bad, t->err, s));
  }
  const uint32_t ls = shard % t->R;
  uint64_t row_total = 0;
  for (auto& c : t->cols) row_total += c.rb;
  // Rows per chunk: bounded by the staging arrays and by 256 MB of row data.
  const uint64_t by_bytes = std::max<uint64_t>(1, (256ull << 20) / row_total);
  const uint32_t chunk_rows = (uint32_t)std::min<uint64_t>(t->max_batch, by_bytes);
  std::vector<MemKind> kinds(t->cols.size());
  for (size_t c = 0; c < t->cols.size(); ++c) kinds[c] = mem_kind(col_src[c]);

  bool staging = !dev_prio;  // pinned host staging in use (reused per call)
  for (auto k : kinds) staging = staging || k == MemKind::HostPageable;
  for (uint32_t k0 = 0; k0 < n; k0 += chunk_rows) {
    const uint32_t m = std::min(chunk_rows, n - k0);
    if (staging) GEAR_CUDA(cudaEventSynchronize(t->staging_ev));  // staging buffers free again
    // The allocator runs on the device (kernels/alloc.cu): slots, ring
    // positions, seq and generation counts of the m rows in one launch.
    const double* d_p = prio + k0;
    if (!dev_prio) {
      std::memcpy(t->h_prio, p.data() + k0, m * sizeof(double));
      GEAR_CUDA(cudaMemcpyAsync(t->d_prio_ins, t->h_prio, m * sizeof(double),
                                cudaMemcpyHostToDevice, s));
      d_p = t->d_prio_ins;
    }
    GEAR_CUDA(launch_insert_plan(t->d_alloc, ls, shard, t->Cs, t->removal == GEAR_REMOVE_LIFO, m,
                                 d_p, t->ord, dev_prio ? t->ins_bad : nullptr, t->d_meta,
                                 t->d_ord, t->d_out, t->err, s));
    const uint32_t n_meta = m, n_ord = m;  // rows a later row overrides are skipped
    // Row sources: device / pinned host are read in place; pageable host is
    // staged into device memory first.  The rows move with the collect
    // engine in scatter mode (source row -> table slot): TMA bulk copies for
    // 16-byte aligned rows of >= 4 KB, warp LSU copies otherwise.
    uint64_t stage_off = 0, stage_need = 0;
    for (size_t c = 0; c < t->cols.size(); ++c)
      if (kinds[c] == MemKind::HostPageable) stage_need += (uint64_t)m * t->cols[c].rb;
    if (stage_need > t->d_rows_bytes) {
      dfree(t->d_rows);
      GEAR_TRY(dalloc(&t->d_rows, stage_need));
      t->d_rows_bytes = stage_need;
    }
    CollectParams cp{};
    cp.meta = t->d_meta;
    cp.rows_per_rank = t->Clocal;
    cp.n_global = t->N;
    cp.ncols = (uint32_t)t->cols.size();
    cp.n = n_meta;
    cp.err = t->err;
    cp.self_rank = t->rank;
    cp.tma_ctas_per_sm = (uint32_t)t->tma_ctas;
    cp.tma_stages = (uint32_t)t->tma_stages;
    for (size_t c = 0; c < t->cols.size(); ++c) {
      ColumnState& cs = t->cols[c];
      const uint8_t* src = (const uint8_t*)col_src[c] + (uint64_t)k0 * cs.rb;
      if (kinds[c] == MemKind::HostPageable) {
        GEAR_CUDA(cudaMemcpyAsync(t->d_rows + stage_off, src, (uint64_t)m * cs.rb,
                                  cudaMemcpyHostToDevice, s));
        src = t->d_rows + stage_off;
        stage_off += (uint64_t)m * cs.rb;
      } else if (kinds[c] == MemKind::HostPinned) {
        void* dp = nullptr;
        GEAR_CUDA(cudaHostGetDevicePointer(&dp, (void*)src, 0));
        src = (const uint8_t*)dp;
      }
      CollectCol& cc = cp.col[c];
      cc.out = (uint8_t*)cs.view[t->rank];  // the table column (destination)
      cc.src[0] = src;                      // the caller's rows (source)
      cc.rb = cs.rb;
      cc.vec = vec_width(cs.rb, 512, {(uintptr_t)cc.out | (uintptr_t)src});
      cc.tma = (t->collect_impl == 1 && cc.vec == 16 && cs.rb >= 4096) ? 1u : 0u;
      cc.chunk = cc.tma ? t->tma_chunk : t->chunk_bytes;
      if (cc.vec < 16 && cc.chunk % cc.vec) cc.chunk = t->chunk_bytes;
      cc.chunks_per_row = (uint32_t)((cs.rb + cc.chunk - 1) / cc.chunk);
      if (cc.tma) {
        cc.chunk_begin = cp.tma_total;
        cp.tma_total += (uint64_t)n_meta * cc.chunks_per_row;
        cp.tma_cols[cp.n_tma++] = (uint8_t)c;
      } else {
        cc.chunk_begin = cp.lsu_total;
        cp.lsu_total += (uint64_t)n_meta * cc.chunks_per_row;
        cp.lsu_cols[cp.n_lsu++] = (uint8_t)c;
      }
    }
    GEAR_CUDA(launch_collect(cp, s));
    GEAR_CUDA(launch_insert_meta(t->d_meta, n_meta, t->d_ord, n_ord, quant(t), t->key,
                                 tile_dirty(t), t->seq, t->gen, t->ord, s));
    if (out_idx) {
      if (mem_kind(out_idx) == MemKind::Device) {
        GEAR_CUDA(cudaMemcpyAsync(out_idx + k0, t->d_out, m * 8, cudaMemcpyDeviceToDevice, s));
      } else {  // a host id list: the ids are known once the plan ran
        GEAR_CUDA(cudaMemcpyAsync(t->h_out, t->d_out, m * 8, cudaMemcpyDeviceToHost, s));
        GEAR_CUDA(cudaStreamSynchronize(s));
        std::memcpy(out_idx + k0, t->h_out, m * 8);
      }
    }
    if (staging) GEAR_CUDA(cudaEventRecord(t->staging_ev, s));
  }
  t->dirty = true;
  return GEAR_OK;
}

gear_status gear_update_priorities(gear_table* t, uint32_t n, const uint64_t* idx,
                                   const void* prio, gear_dtype prio_dtype, const uint32_t* gen,
                                   gear_stream stream) {
  GEAR_NVTX("gear_update_priorities");
  clear_error();
  GEAR_TRY(check_table(t));
  GEAR_CUDA(cudaSetDevice(t->device));
  cudaStream_t s = (cudaStream_t)stream;
  if (n > t->max_batch) return set_error(GEAR_ERR_INVALID_ARG, "n %u > max_batch %u", n, t->max_batch);
  if (prio_dtype != GEAR_F32 && prio_dtype != GEAR_F64)
    return set_error(GEAR_ERR_INVALID_ARG, "prio_dtype must be GEAR_F32 or GEAR_F64");
  if (n > 0 && (idx == nullptr || prio == nullptr))
    return set_error(GEAR_ERR_INVALID_ARG, "idx / prio is NULL");
  const uint64_t* d_idx = idx;
  const void* d_prio = prio;
  const uint32_t* d_gen = gen;
  if (n > 0) {
    GEAR_TRY(stage_in(idx, n, t->upd_idx, s, &d_idx, true));
    if (prio_dtype == GEAR_F64) {
      const double* dp = nullptr;
      GEAR_TRY(stage_in((const double*)prio, n, t->upd_prio, s, &dp, true));
      d_prio = dp;
    } else {
      const float* dp = nullptr;
      GEAR_TRY(stage_in((const float*)prio, n, (float*)t->upd_prio, s, &dp, true));
      d_prio = dp;
    }
    if (gen) GEAR_TRY(stage_in(gen, n, t->upd_gen, s, &d_gen, true));
  }
  // PER exponent: the update kernels quantise p^alpha computed here first
  Quant qz = quant(t);
  if (t->alpha != 1.0 && n > 0) {
    GEAR_CUDA(launch_alpha(d_prio, prio_dtype == GEAR_F64, n, t->alpha, t->upd_pow, s));
    d_prio = t->upd_pow;
    prio_dtype = GEAR_F64;
  }
  qz.alpha = 1.0;
  const uint64_t local_begin = (uint64_t)t->rank * t->Clocal;
  const bool fused = t->update_fused && (uint64_t)n * t->W <= update_fused_max();
  if (t->W == 1 && fused) {
    // one launch: quantise, tag, block barrier, apply
    GEAR_CUDA(launch_update_fused(d_idx, d_prio, prio_dtype == GEAR_F64, d_gen, nullptr, n, t->N,
                                  qz, local_begin, t->Clocal, t->gen, t->seq, t->tag, t->d_epoch,
                                  t->n_stale, t->err, t->key, tile_dirty(t), s));
  } else if (t->W > 1 && fused && t->peer_xchg) {
    // one launch: quantise, push records to every peer over NVLink, wait for
    // every rank's records, tag, barrier, apply
    Mbox mb = t->mb;
    mb.epoch_dev = t->d_xep + 1;  // update-exchange epoch (advanced by the kernel)
    GEAR_CUDA(launch_update_xchg(d_idx, d_prio, prio_dtype == GEAR_F64, d_gen, n, t->N, qz,
                                 mb, local_begin, t->Clocal, t->gen, t->seq, t->tag, t->d_epoch,
                                 t->n_stale, t->err, t->key, tile_dirty(t), s));
  } else {
    GEAR_CUDA(launch_update_quantize(d_idx, d_prio, prio_dtype == GEAR_F64, d_gen, n, t->N,
                                     qz, t->upd_local, t->err, s));
    const UpdRec* recs = t->upd_local;
    uint32_t m = n;
    if (t->W > 1) {
      GEAR_TRY(allgather_bytes(t->comm, t->upd_local, t->upd_all, (size_t)n * sizeof(UpdRec), s));
      recs = t->upd_all;
      m = n * t->W;
    }
    if (fused) {
      GEAR_CUDA(launch_update_fused(nullptr, nullptr, 0, nullptr, recs, m, t->N, qz,
                                    local_begin, t->Clocal, t->gen, t->seq, t->tag, t->d_epoch, t->n_stale,
                                    t->err, t->key, tile_dirty(t), s));
    } else {
      GEAR_CUDA(launch_update_tag(recs, m, local_begin, t->Clocal, t->gen, t->seq, t->tag, t->d_epoch,
                                  t->n_stale, t->err, s));
      GEAR_CUDA(launch_update_apply(recs, m, local_begin, t->Clocal, t->gen, t->seq, t->tag, t->d_epoch,
                                    t->key, tile_dirty(t), s));
    }
  }
  t->dirty = true;
  return GEAR_OK;
}

gear_status gear_sample(gear_table* t, gear_strategy strategy, uint32_t B, uint64_t seed,
                        double beta, uint64_t* out_idx, float* out_w, double* out_p,
                        uint32_t* out_gen, uint32_t flags, gear_stream stream) {
  GEAR_NVTX("gear_sample");
  clear_error();
  GEAR_TRY(check_table(t));
  GEAR_CUDA(cudaSetDevice(t->device));
  cudaStream_t s = (cudaStream_t)stream;
  if (flags & ~(uint32_t)(GEAR_SAMPLE_OWNER_AFFINE | GEAR_SAMPLE_DEVICE_SEED))
    return set_error(GEAR_ERR_INVALID_ARG, "unknown sample flags 0x%x", flags);
  // With one rank every entry is local: the owner-affine slice is the
  // contiguous one, so the assignment kernel is skipped.
  const bool affine = (flags & GEAR_SAMPLE_OWNER_AFFINE) != 0 && t->W > 1;
  const bool dseed = (flags & GEAR_SAMPLE_DEVICE_SEED) != 0;
  if ((int)strategy < GEAR_FIFO || (int)strategy > GEAR_TOPK)
    return set_error(GEAR_ERR_INVALID_ARG, "bad strategy %d", (int)strategy);
  t->last_topk = strategy == GEAR_TOPK;
  if (B > t->max_batch) return set_error(GEAR_ERR_INVALID_ARG, "B %u > max_batch %u", B, t->max_batch);
  if (B == 0) return GEAR_OK;
  if (out_idx == nullptr) return set_error(GEAR_ERR_INVALID_ARG, "out_idx is NULL");
  if (!std::isfinite(beta)) return set_error(GEAR_ERR_INVALID_ARG, "beta is not finite");
  // Outputs: device and pinned host buffers are written in place by the
  // kernels (pinned ones through their mapped address, over PCIe); pageable
  // host buffers through device scratch and a copy at the end.
  bool h_idx = false, h_w = false, h_p = false, h_gen = false;
  uint64_t* d_idx = out_device(out_idx, t->tmp_idx, &h_idx);
  float* d_w = out_device(out_w, t->tmp_w, &h_w);
  double* d_p = out_device(out_p, t->tmp_p, &h_p);
  uint32_t* d_gen = out_device(out_gen, t->tmp_gen, &h_gen);

  if (strategy == GEAR_FIFO || strategy == GEAR_LIFO || strategy == GEAR_TOPK) {
    const uint32_t K = t->W * B;
    const bool topk = strategy == GEAR_TOPK;
    if (topk && K > topk_max_k())
      return set_error(GEAR_ERR_UNSUPPORTED, "TopK needs W*B <= %u (got %u)", topk_max_k(), K);
    const int lifo = topk ? 2 : (strategy == GEAR_LIFO ? 1 : 0);  // merge order
    const bool xchg = t->W > 1 && t->peer_xchg;
    Mbox mb = t->mb;
    const ShardTotals* fifo_totals = t->fifo_totals_all;
    // candidates go straight into every peer's mailbox from the local kernel;
    // the FIFO-exchange epoch advances after the merge (and assignment)
    mb.epoch_dev = t->d_xep + 2;
    if (topk)
      GEAR_CUDA(launch_topk_local(t->key, t->Cs, t->qmax, t->R, t->rank * t->R, K, t->topk_tmp,
                                  t->cand_local,
                                  t->fifo_totals_local, t->topk_state, t->topk_cnt,
                                  xchg ? &mb : nullptr, s));
    else
      GEAR_CUDA(launch_fifo_local(t->key, t->seq, t->ord, t->d_alloc, t->Cs, t->R, t->rank * t->R, K,
                                  lifo, t->cand_local, t->fifo_totals_local, xchg ? &mb : nullptr,
                                  s));
    const Cand* cand_all = t->cand_all;
    const ShardTotals* merge_totals = t->fifo_totals_all;
    if (t->W == 1) {  // the local lists are all the lists
      cand_all = t->cand_local;
      merge_totals = fifo_totals = t->fifo_totals_local;
    } else if (!xchg) {
      GEAR_TRY(allgather_bytes(t->comm, t->cand_local, t->cand_all,
                               (size_t)t->R * K * sizeof(Cand), s));
      GEAR_TRY(allgather_bytes(t->comm, t->fifo_totals_local, t->fifo_totals_all,
                               t->R * sizeof(ShardTotals), s));
    }
    GEAR_CUDA(launch_fifo_merge(cand_all, merge_totals, t->S, K, lifo, t->Cs, t->rank,
                                B, t->d_gen_ptrs, t->R, d_idx, d_w, d_p, d_gen, t->err,
                                affine ? t->glob_shard : nullptr, affine ? t->glob_slot : nullptr,
                                xchg ? &mb : nullptr, s));
    if (affine) {
      AssignParams ap = assign_params(t, B, seed);
      ap.fifo_totals = fifo_totals;
      ap.fifo_mbox = xchg;
      ap.mbox = mb;
      ap.glob_shard = t->glob_shard;
      ap.glob_slot = t->glob_slot;
      ap.out_idx = d_idx;
      ap.out_w = d_w;
      ap.out_p = d_p;
      ap.out_gen = d_gen;
      GEAR_CUDA(launch_assign(ap, s));
    }
    if (xchg) GEAR_CUDA(launch_epoch_bump(t->d_xep + 2, s));
  } else {
    const int mode = strategy == GEAR_UNIFORM ? 1 : 0;
    // Two-level CDF: always launched -- it rescans only tiles the device-side
    // dirty bits name, so writers replayed from a CUDA graph (which the host
    // does not see) are picked up; a clean table costs one short launch.
    if (t->cdf_levels == 2 || t->dirty || t->cdf_mode != mode) {
      // Rebuild into the buffer peers are not reading (device-resident parity).
      if (t->cdf_levels == 2)  // incremental: only tiles changed since this buffer's build
        GEAR_CUDA(launch_scan2(t->key, t->cdf[0], t->cdf[1], t->Cs, t->R, mode, t->d_xep + 3,
                               t->cdf_totals_local, t->tile_dirty, t->tile_tot, t->cdf_buf_mode,
                               t->scan2_ctr, t->scan2_ctr + t->R, s));
      else
        GEAR_CUDA(launch_scan(t->key, t->cdf[0], t->cdf[1], t->Cs, t->R, mode, t->d_xep + 3,
                              t->cdf_totals_local, t->scan_status[0], t->scan_status[1],
                              t->scan_ticket[0], t->scan_ticket[1], t->scan_chunk, s));
      t->scan_launches += 1;
      t->cdf_mode = mode;
      t->dirty = false;
    }
    // If a later step of this call fails (e.g. a host all-gather refused
    // inside stream capture), the rebuild enqueued above may never run: keep
    // the host's "CDF is current" flag honest (flat layout) by marking it
    // dirty again on every error return below.
    struct DirtyOnError {
      gear_table* t;
      bool ok = false;
      ~DirtyOnError() {
        if (!ok) t->dirty = true;
      }
    } dirty_guard{t};
    // Every step publishes the totals; the exchange is also the barrier that
    // makes every shard's CDF visible before anyone searches it.  W > 1: the
    // first kernel of the step (assign or sample) pushes this rank's totals
    // into every peer's mailbox over NVLink and waits for all of them;
    // otherwise an NCCL all-gather (or a copy at W = 1).
    const bool xchg = t->W > 1 && t->peer_xchg;
    Mbox mb = t->mb;
    const ShardTotals* totals_all = t->cdf_totals_all;
    mb.epoch_dev = t->d_xep + 0;  // totals-exchange epoch (advanced by the kernels)
    if (xchg) {
      totals_all = nullptr;  // the kernels find them in the mailbox
    } else if (t->W == 1) {
      totals_all = t->cdf_totals_local;  // R local shards are all the shards
    } else {
      GEAR_TRY(allgather_bytes(t->comm, t->cdf_totals_local, t->cdf_totals_all,
                               t->R * sizeof(ShardTotals), s));
    }
    SampleParams sp{};
    sp.totals = totals_all;
    sp.totals_local = t->cdf_totals_local;
    sp.mbox = mb;
    // 1: the sample kernel exchanges; 2: the assign kernel did, read the mailbox
    sp.xchg = xchg ? (affine ? 2 : 1) : 0;
    sp.cdf_ptrs = t->d_cdf_ptrs;
    sp.cdf_levels = (uint32_t)t->cdf_levels;
    sp.tiles_per_shard = scan_tiles_per_shard(t->Cs);
    sp.gen_ptrs = t->d_gen_ptrs;
    sp.shard_cap = t->Cs;
    sp.n_shards = t->S;
    sp.shards_per_rank = t->R;
    sp.seed = seed;
    sp.rank = t->rank;
    sp.B = B;
    sp.beta = beta;
    sp.strategy = (int)strategy;
    sp.out_idx = d_idx;
    sp.out_w = d_w;
    sp.out_p = d_p;
    sp.out_gen = d_gen;
    sp.q_scratch = t->q_scratch;
    sp.qmin_slot = t->qmin_slot;
    sp.done_ctr = t->done_ctr;
    sp.err = t->err;
    sp.seed_dev = dseed ? t->d_seed : nullptr;
    if (affine) {
      AssignParams ap = assign_params(t, B, seed);
      ap.seed_dev = sp.seed_dev;
      ap.totals = totals_all;
      ap.totals_local = t->cdf_totals_local;
      ap.mbox = mb;
      ap.xchg = xchg;
      GEAR_CUDA(launch_assign(ap, s));
      sp.draw_list = t->draw_list;
    }
    GEAR_CUDA(launch_sample(sp, s));
    dirty_guard.ok = true;
  }
  if (h_idx) GEAR_CUDA(cudaMemcpyAsync(out_idx, d_idx, B * 8ull, cudaMemcpyDeviceToHost, s));
  if (h_w) GEAR_CUDA(cudaMemcpyAsync(out_w, d_w, B * 4ull, cudaMemcpyDeviceToHost, s));
  if (h_p) GEAR_CUDA(cudaMemcpyAsync(out_p, d_p, B * 8ull, cudaMemcpyDeviceToHost, s));
  if (h_gen) GEAR_CUDA(cudaMemcpyAsync(out_gen, d_gen, B * 4ull, cudaMemcpyDeviceToHost, s));
  return GEAR_OK;
}

gear_status gear_allocate(gear_table* t, uint32_t shard, uint32_t n, uint64_t* out_idx,
                          gear_stream stream) {
  GEAR_NVTX("gear_allocate");
  clear_error();
  GEAR_TRY(check_table(t));
  GEAR_CUDA(cudaSetDevice(t->device));
  cudaStream_t s = (cudaStream_t)stream;
  if (shard / t->R != t->rank || shard >= t->S)
    return set_error(GEAR_ERR_INVALID_ARG, "shard %u is not owned by rank %u", shard, t->rank);
  if (n > t->max_batch) return set_error(GEAR_ERR_INVALID_ARG, "n %u > max_batch %u", n, t->max_batch);
  if (n == 0) return GEAR_OK;
  if (out_idx == nullptr) return set_error(GEAR_ERR_INVALID_ARG, "out_idx is NULL");
  const bool host_out = mem_kind(out_idx) != MemKind::Device;
  uint64_t* d_out = host_out ? t->d_out : out_idx;
  GEAR_CUDA(launch_allocate(t->d_alloc, shard % t->R, shard, t->Cs,
                            t->removal == GEAR_REMOVE_LIFO, n, t->ord, t->key, t->seq, t->gen,
                            tile_dirty(t), d_out, t->err, s));
  if (host_out) {
    GEAR_CUDA(cudaMemcpyAsync(out_idx, d_out, n * 8ull, cudaMemcpyDeviceToHost, s));
    GEAR_CUDA(cudaStreamSynchronize(s));
  }
  t->dirty = true;
  return GEAR_OK;
}

gear_status gear_commit(gear_table* t, uint32_t shard, uint32_t n, const uint64_t* idx,
                        const double* prio, gear_stream stream) {
  GEAR_NVTX("gear_commit");
  clear_error();
  GEAR_TRY(check_table(t));
  GEAR_CUDA(cudaSetDevice(t->device));
  cudaStream_t s = (cudaStream_t)stream;
  if (shard / t->R != t->rank || shard >= t->S)
    return set_error(GEAR_ERR_INVALID_ARG, "shard %u is not owned by rank %u", shard, t->rank);
  if (n > t->max_batch) return set_error(GEAR_ERR_INVALID_ARG, "n %u > max_batch %u", n, t->max_batch);
  if (n == 0) return GEAR_OK;
  if (idx == nullptr || prio == nullptr) return set_error(GEAR_ERR_INVALID_ARG, "idx / prio is NULL");
  const uint64_t* d_idx = nullptr;
  const double* d_prio = nullptr;
  GEAR_TRY(stage_in(idx, n, t->upd_idx, s, &d_idx));
  GEAR_TRY(stage_in(prio, n, t->upd_prio, s, &d_prio));
  GEAR_CUDA(launch_commit(t->d_alloc, shard % t->R, shard, t->Cs, n, d_idx, d_prio, quant(t),
                          t->key, t->seq, t->gen, t->ord, t->tag, t->d_epoch, tile_dirty(t),
                          t->err, s));
  t->dirty = true;
  return GEAR_OK;
}

gear_status gear_column_base(const gear_table* t, uint32_t col, void** out) {
  GEAR_NVTX("gear_column_base");
  clear_error();
  if (t == nullptr || out == nullptr || col >= t->cols.size())
    return set_error(GEAR_ERR_INVALID_ARG, "bad table, column %u or NULL output", col);
  *out = t->cols[col].local;
  return GEAR_OK;
}

gear_status gear_collect(gear_table* t, uint32_t n, const uint64_t* idx, uint32_t ncols,
                         const uint32_t* col_ids, void* const* out, gear_stream stream) {
  GEAR_NVTX("gear_collect");
  clear_error();
  GEAR_TRY(check_table(t));
  GEAR_CUDA(cudaSetDevice(t->device));
  cudaStream_t s = (cudaStream_t)stream;
  if (n == 0 || ncols == 0) return GEAR_OK;
  if (idx == nullptr || col_ids == nullptr || out == nullptr)
    return set_error(GEAR_ERR_INVALID_ARG, "NULL argument");
  if (ncols > (uint32_t)kMaxCols) return set_error(GEAR_ERR_INVALID_ARG, "ncols > %d", kMaxCols);
  const uint64_t* d_idx = idx;
  if (mem_kind(idx) != MemKind::Device) {
    DevBuf<uint64_t>& buf = t->col_idx[t->col_idx_next++ % 4];
    if (buf.n < n) {
      dfree(buf.p);
      GEAR_TRY(dalloc(&buf.p, n));
      buf.n = n;
    }
    GEAR_CUDA(cudaMemcpyAsync(buf.p, idx, n * 8ull, cudaMemcpyHostToDevice, s));
    d_idx = buf.p;
  }
  CollectParams cp{};
  cp.idx = d_idx;
  cp.rows_per_rank = t->Clocal;
  cp.n_global = t->N;
  cp.ncols = ncols;
  cp.n = n;
  cp.err = t->err;
  cp.self_rank = t->rank;
  // L2 evict-first bulk copies: auto = at W > 1 after a TopK selection, whose
  // grid-wide radix passes re-read the keys from L2 while this collect runs
  // (+7-11% c2 TopK at N=4); for the other strategies it cost ~1.5% (c2, N=2/4)
  cp.evict_first = t->evict_first < 0 ? (t->W > 1 && t->last_topk ? 1u : 0u)
                                      : (uint32_t)t->evict_first;
  bool any_host = false;
  for (uint32_t c = 0; c < ncols; ++c)
    any_host |= col_ids[c] < t->cols.size() && t->cols[col_ids[c]].placement == GEAR_HOST;
  // dynamic task claiming: auto = at W > 1 (selection kernels next to the
  // collect) or with host rows (uneven PCIe row latencies); HBM-only at W = 1
  // keeps the static stride (measured 1% faster at c2)
  const bool dynamic = t->collect_dynamic < 0 ? (t->W > 1 || any_host) : t->collect_dynamic != 0;
  if (dynamic)  // rotating counter pairs: overlapping collects differ
    cp.dyn_ctr = t->dyn_pool + 2 * (t->dyn_slot++ % gear_table::kDynSlots);
  cp.tma_ctas_per_sm = (uint32_t)t->tma_ctas;
  cp.tma_stages = (uint32_t)t->tma_stages;
  for (uint32_t c = 0; c < ncols; ++c) {
    if (col_ids[c] >= t->cols.size()) return set_error(GEAR_ERR_INVALID_ARG, "bad column id %u", col_ids[c]);
    if (out[c] == nullptr) return set_error(GEAR_ERR_INVALID_ARG, "out[%u] is NULL", c);
    const ColumnState& cs = t->cols[col_ids[c]];
    CollectCol& cc = cp.col[c];
    cc.out = (uint8_t*)out[c];
    cc.rb = cs.rb;
    uintptr_t align_or = (uintptr_t)out[c];
    for (uint32_t r = 0; r < t->W; ++r) {
      cc.src[r] = cs.view[r];
      align_or |= (uintptr_t)cs.view[r];
    }
    cc.vec = vec_width(cs.rb, 512, {align_or});
    // Rows of >= 4 KB with 16-byte alignment go to the TMA bulk-copy path.
    cc.tma = (t->collect_impl == 1 && cc.vec == 16 && cs.rb >= 4096) ? 1u : 0u;
    cc.chunk = cc.tma ? t->tma_chunk : t->chunk_bytes;
    if (cc.vec < 16 && cc.chunk % cc.vec) cc.chunk = t->chunk_bytes;
    cc.chunks_per_row = (uint32_t)((cs.rb + cc.chunk - 1) / cc.chunk);
    cc.peer_lsu = (cc.tma && t->W > 1 && cs.placement == GEAR_DEVICE && t->collect_peer_lsu) ? 1u : 0u;
    // host rows by the LSU warps: auto = rows of at most one 16 KB bulk task
    // (c3's 4 KB rows: +2.5%; c4's 449 KB host rows lost 40% e2e at N=4)
    cc.host_lsu = (cc.tma && cs.placement == GEAR_HOST &&
                   (t->collect_host_lsu == 1 || (t->collect_host_lsu < 0 && cs.rb <= 16384)))
                      ? 1u : 0u;
    cp.any_peer_lsu |= cc.peer_lsu | cc.host_lsu;
    if (cc.tma) {
      cc.chunk_begin = cp.tma_total;
      cp.tma_total += (uint64_t)n * cc.chunks_per_row;
      cp.tma_cols[cp.n_tma++] = (uint8_t)c;
    } else {
      cc.chunk_begin = cp.lsu_total;
      cp.lsu_total += (uint64_t)n * cc.chunks_per_row;
      cp.lsu_cols[cp.n_lsu++] = (uint8_t)c;
    }
  }
  GEAR_CUDA(launch_collect(cp, s));
  return GEAR_OK;
}

gear_status gear_table_sync(gear_table* t, uint32_t* dev_errors, uint64_t* n_stale) {
  GEAR_NVTX("gear_table_sync");
  clear_error();
  GEAR_TRY(check_table(t));
  GEAR_CUDA(cudaSetDevice(t->device));
  GEAR_CUDA(cudaDeviceSynchronize());
  uint32_t e = 0;
  unsigned long long ns = 0;
  GEAR_CUDA(cudaMemcpy(&e, t->err, 4, cudaMemcpyDeviceToHost));
  GEAR_CUDA(cudaMemcpy(&ns, t->n_stale, 8, cudaMemcpyDeviceToHost));
  GEAR_CUDA(cudaMemset(t->err, 0, 4));
  GEAR_CUDA(cudaMemset(t->n_stale, 0, 8));
  if (dev_errors) *dev_errors = e;
  if (n_stale) *n_stale = ns;
  if (e) return set_error(GEAR_ERR_STATE, "device error bits 0x%x", e);
  return GEAR_OK;
}

gear_status gear_table_set_tuning(gear_table* t, const char* key, int64_t value) {
  GEAR_NVTX("gear_table_set_tuning");
  clear_error();
  GEAR_TRY(check_table(t));
  if (key == nullptr) return set_error(GEAR_ERR_INVALID_ARG, "key is NULL");
  if (!strcmp(key, "collect_impl") && (value == 0 || value == 1)) {
    t->collect_impl = (int)value;
  } else if (!strcmp(key, "lsu_chunk") && value >= 512 && value % 512 == 0 && value <= (1 << 20)) {
    t->chunk_bytes = (uint32_t)value;
  } else if (!strcmp(key, "device_seed")) {
    const uint64_t v = (uint64_t)value;  // synchronous: not for use while capturing
    GEAR_CUDA(cudaSetDevice(t->device));
    GEAR_CUDA(cudaDeviceSynchronize());
    GEAR_CUDA(cudaMemcpy(t->d_seed, &v, 8, cudaMemcpyHostToDevice));
  } else if (!strcmp(key, "peer_xchg") && (value == 0 || value == 1)) {
    t->peer_xchg = (int)value;  // must be set identically on every rank
  } else if (!strcmp(key, "cdf_levels") && (value == 1 || value == 2)) {
    // must be set identically on every rank (peers search each other's CDFs)
    GEAR_CUDA(cudaDeviceSynchronize());
    GEAR_CUDA(cudaMemset(t->cdf_buf_mode, 0, 8));  // both buffers: full rebuild
    t->cdf_levels = (int)value;
    t->dirty = true;
  } else if (!strcmp(key, "scan_chunk") && value >= -1 && value <= 4096) {
    t->scan_chunk = (int)value;  // flat CDF kernel choice (same CDF either way)
  } else if (!strcmp(key, "collect_dynamic") && value >= -1 && value <= 1) {
    t->collect_dynamic = (int)value;
  } else if (!strcmp(key, "collect_evict_first") && value >= -1 && value <= 1) {
    t->evict_first = (int)value;
  } else if (!strcmp(key, "collect_host_lsu") && value >= -1 && value <= 1) {
    t->collect_host_lsu = (int)value;
  } else if (!strcmp(key, "collect_peer_lsu") && (value == 0 || value == 1)) {
    t->collect_peer_lsu = (int)value;
  } else if (!strcmp(key, "update_fused") && (value == 0 || value == 1)) {
    t->update_fused = (int)value;
  } else if (!strcmp(key, "tma_ctas_per_sm") && value >= 1 && value <= 8 &&
             (uint64_t)value * t->tma_stages * t->tma_chunk <= (220u << 10)) {
    t->tma_ctas = (int)value;
  } else if (!strcmp(key, "tma_stages") &&
             (value == 2 || value == 3 || value == 4 || value == 6 || value == 8) &&
             (uint64_t)value * t->tma_ctas * t->tma_chunk <= (220u << 10)) {
    t->tma_stages = (int)value;
  } else if (!strcmp(key, "tma_chunk") && value >= 4096 && value % 16 == 0 && value <= 32768 &&
             (uint64_t)value * t->tma_ctas * t->tma_stages <= (220u << 10)) {
    t->tma_chunk = (uint32_t)value;
  } else {
    return set_error(GEAR_ERR_INVALID_ARG, "bad tuning %s = %lld", key, (long long)value);
  }
  return GEAR_OK;
}

gear_status gear_read_cdf(gear_table* t, uint64_t* cdf) {
  GEAR_NVTX("gear_read_cdf");
  clear_error();
  GEAR_TRY(check_table(t));
  if (cdf == nullptr) return set_error(GEAR_ERR_INVALID_ARG, "cdf is NULL");
  if (t->cdf_mode < 0) return set_error(GEAR_ERR_STATE, "no CDF built yet (call gear_sample)");
  GEAR_CUDA(cudaSetDevice(t->device));
  GEAR_CUDA(cudaDeviceSynchronize());
  uint64_t par = 0;
  GEAR_CUDA(cudaMemcpy(&par, t->d_xep + 3, 8, cudaMemcpyDeviceToHost));
  const uint64_t* buf = t->cdf[par & 1];
  GEAR_CUDA(cudaMemcpy(cdf, buf, t->Clocal * 8, cudaMemcpyDeviceToHost));
  if (t->cdf_levels == 2) {  // tile-local prefixes + each shard's prefix of tile totals
    const uint32_t tps = scan_tiles_per_shard(t->Cs);
    std::vector<uint64_t> P((size_t)t->R * tps);
    GEAR_CUDA(cudaMemcpy(P.data(), buf + t->Clocal, P.size() * 8, cudaMemcpyDeviceToHost));
    for (uint32_t ls = 0; ls < t->R; ++ls)
      for (uint64_t i = kCdfTile; i < t->Cs; ++i)
        cdf[ls * t->Cs + i] += P[(size_t)ls * tps + i / kCdfTile - 1];
  }
  return GEAR_OK;
}

gear_status gear_read_state(gear_table* t, uint64_t* key, uint64_t* seq, uint32_t* gen) {
  GEAR_NVTX("gear_read_state");
  clear_error();
  GEAR_TRY(check_table(t));
  GEAR_CUDA(cudaSetDevice(t->device));
  GEAR_CUDA(cudaDeviceSynchronize());
  if (key) GEAR_CUDA(cudaMemcpy(key, t->key, t->Clocal * 8, cudaMemcpyDeviceToHost));
  if (seq) GEAR_CUDA(cudaMemcpy(seq, t->seq, t->Clocal * 8, cudaMemcpyDeviceToHost));
  if (gen) GEAR_CUDA(cudaMemcpy(gen, t->gen, t->Clocal * 4, cudaMemcpyDeviceToHost));
  return GEAR_OK;
}

}  // extern "C"
