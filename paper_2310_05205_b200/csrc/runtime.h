// runtime.h -- host-side state of a gear_table / gear_comm (C++17).
#pragma once

#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "../../include/gear.h"
#include "gear_internal.h"

struct gear_comm {
  ncclComm_t nccl = nullptr;
  int nranks = 1;
  int rank = 0;
  int device = 0;
  cudaStream_t stream = nullptr;  // for create-time exchanges
  // gear_comm_create_host: no NCCL; create-time plumbing and the peer_xchg = 0
  // exchanges go through the caller's host all-gather
  gear_allgather_fn host_ag = nullptr;
  void* host_ctx = nullptr;
};

namespace gear {

// Thread-local error string + status helpers.
gear_status set_error(gear_status code, const char* fmt, ...);
void clear_error();

#define GEAR_CUDA(x)                                                                    \
  do {                                                                                  \
    cudaError_t e_ = (x);                                                               \
    if (e_ != cudaSuccess)                                                              \
      return ::gear::set_error(GEAR_ERR_CUDA, "%s failed: %s (%s:%d)", #x,              \
                               cudaGetErrorString(e_), __FILE__, __LINE__);             \
  } while (0)

#define GEAR_NCCL(x)                                                                    \
  do {                                                                                  \
    ncclResult_t r_ = (x);                                                              \
    if (r_ != ncclSuccess)                                                              \
      return ::gear::set_error(GEAR_ERR_NCCL, "%s failed: %s (%s:%d)", #x,              \
                               ncclGetErrorString(r_), __FILE__, __LINE__);             \
  } while (0)

#define GEAR_TRY(x)                      \
  do {                                   \
    gear_status s_ = (x);                \
    if (s_ != GEAR_OK) return s_;        \
  } while (0)

// NVTX range around every C-ABI call (header-only NVTX v3: a no-op unless a
// tool such as nsys / ncu is attached), so timelines show gear_sample /
// gear_collect / ... next to the kernels they enqueue.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
#define GEAR_NVTX(name) ::gear::NvtxRange gear_nvtx_range_(name)

enum class MemKind { Device, HostPinned, HostPageable };
MemKind mem_kind(const void* p);

// Comm helpers (comm.cpp).  With comm == nullptr they are copies / no-ops.
gear_status allgather_bytes(gear_comm* c, const void* send, void* recv, size_t bytes,
                            cudaStream_t s);
gear_status barrier(gear_comm* c);

struct ColumnState {
  std::string name;
  gear_dtype dtype = GEAR_U8;
  gear_placement placement = GEAR_DEVICE;
  uint64_t rb = 0;                      // row bytes
  uint64_t bytes_local = 0;             // R * C_s * rb
  uint8_t* local = nullptr;             // this rank's rows (device ptr or host ptr)
  const uint8_t* view[kMaxRanks] = {};  // device-accessible base of each rank's rows
  std::vector<void*> ipc_opened;        // peer device mappings to close
  std::vector<std::pair<void*, size_t>> host_maps;  // host mappings (own + peers) to unmap
  size_t host_reg_chunk = 0;            // bytes per cudaHostRegister piece of those mappings
  std::string shm_name;                 // own shm object (W > 1 HOST columns)
};

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
};

}  // namespace gear

struct gear_table {
  gear_comm* comm = nullptr;
  int device = 0;
  uint32_t W = 1, rank = 0, R = 1, S = 1;
  uint64_t Cs = 0, Clocal = 0, N = 0;
  uint32_t F = 32;
  double alpha = 1.0;  // PER priority exponent (keys are Q_F(p^alpha))
  uint64_t qmax = 0;
  gear_removal removal = GEAR_REMOVE_FIFO;
  uint32_t max_batch = 4096;
  uint32_t seq_len = 0;
  uint64_t schema_hash = 0;  // FNV-1a over seq_len and every column's name, dtype, shape, placement
  std::vector<gear::ColumnState> cols;

  // slot state (rank-local, R*C_s entries)
  uint64_t* key = nullptr;
  uint64_t* seq = nullptr;
  uint32_t* gen = nullptr;
  unsigned long long* tag = nullptr;
  uint32_t* ord = nullptr;

  // CDF double buffer + scan bookkeeping
  uint64_t* cdf[2] = {nullptr, nullptr};
  uint64_t* scan_status[2] = {nullptr, nullptr};
  uint32_t* scan_ticket[2] = {nullptr, nullptr};
  uint64_t scan_launches = 0;
  int cdf_mode = -1;      // -1 none, 0 weighted keys, 1 indicator
  bool dirty = true;
  int cdf_levels = 2;     // 1: flat CDF (decoupled look-back), 2: two-level incremental
  int scan_chunk = -1;    // flat CDF: 1 chunked look-back, 0 per-tile look-back, -1 auto by size
  uint32_t* tile_dirty = nullptr;    // [R*tiles] bit b: tile changed since buffer b's build
  uint64_t* tile_tot = nullptr;      // [2][R*tiles] each buffer's tile totals
  uint32_t* cdf_buf_mode = nullptr;  // [2] mode each buffer was built in (0 none, 1 w, 2 ind)
  uint32_t* scan2_ctr = nullptr;     // [R+1] per-shard arrivals, shards done
  gear::ShardTotals* cdf_totals_local = nullptr;  // [R]
  gear::ShardTotals* cdf_totals_all = nullptr;    // [S]
  gear::ShardTotals* fifo_totals_local = nullptr; // [R]
  gear::ShardTotals* fifo_totals_all = nullptr;   // [S]
  const uint64_t** d_cdf_ptrs = nullptr;          // [2*S]
  const uint32_t** d_gen_ptrs = nullptr;          // [W]
  std::vector<void*> ipc_opened;                  // peer cdf/gen mappings

  // sample scratch
  uint64_t* q_scratch = nullptr;
  unsigned long long* qmin_slot = nullptr;
  uint32_t* done_ctr = nullptr;
  uint64_t* tmp_idx = nullptr;
  float* tmp_w = nullptr;
  double* tmp_p = nullptr;
  uint32_t* tmp_gen = nullptr;
  // peer mailboxes (W > 1): this rank's allocation, every rank's mapping, and
  // one epoch counter per exchange kind (identical on all ranks: SPMD)
  uint8_t* mbox = nullptr;
  gear::Mbox mb{};
  std::vector<void*> mbox_opened;
  // device counters [4]: totals / update / FIFO exchange epochs, CDF parity
  // (device-resident so that captured steps replay correctly)
  uint64_t* d_xep = nullptr;
  int peer_xchg = 1;                 // 1: mailbox exchanges, 0: NCCL all-gathers

  uint32_t* draw_list = nullptr;     // [max_batch] owner-affine slice -> draw number
  uint32_t* pos_scratch = nullptr;   // [W*max_batch]
  uint32_t* ov_scratch = nullptr;    // [W*max_batch]
  uint32_t* glob_shard = nullptr;    // [W*max_batch] merged FIFO/LIFO list
  uint32_t* glob_slot = nullptr;
  gear::Cand* cand_local = nullptr;  // [R * W*max_batch]
  gear::TopkState* topk_state = nullptr;  // [R]
  gear::Cand* topk_tmp = nullptr;         // [2][R * (W*max_batch + kTopkEqMax)] TopK candidates, sorted runs
  uint32_t* topk_cnt = nullptr;           // [R][kTopkMaxCtas][2]
  gear::Cand* cand_all = nullptr;    // [S * W*max_batch]

  // update scratch
  gear::UpdRec* upd_local = nullptr;  // [max_batch]
  gear::UpdRec* upd_all = nullptr;    // [W*max_batch]
  uint64_t* upd_idx = nullptr;
  double* upd_prio = nullptr;
  double* upd_pow = nullptr;        // [max_batch] p^alpha (alpha != 1)
  uint32_t* upd_gen = nullptr;
  uint64_t* d_epoch = nullptr;      // update tag epoch (device-resident, advanced by the kernels)
  uint64_t* d_seed = nullptr;       // device seed counter (gear_sample with GEAR_SAMPLE_DEVICE_SEED)
  unsigned long long* n_stale = nullptr;
  uint32_t* err = nullptr;

  // collect scratch (host-resident id lists)
  gear::DevBuf<uint64_t> col_idx[4];  // rotating: collects on different streams do not share one
  uint32_t col_idx_next = 0;

  // block allocator (device-resident, kernels/alloc.cu) and insert staging
  gear::AllocState* d_alloc = nullptr;  // [R]
  double* h_prio = nullptr;         // pinned [max_batch]
  double* d_prio_ins = nullptr;     // [max_batch]
  uint32_t* ins_bad = nullptr;      // device priorities of the current insert invalid
  uint64_t* h_out = nullptr;        // pinned
  gear::InsMeta* d_meta = nullptr;
  gear::OrdRec* d_ord = nullptr;
  uint64_t* d_out = nullptr;
  uint8_t* d_rows = nullptr;        // staging for pageable row sources
  size_t d_rows_bytes = 0;
  cudaEvent_t staging_ev = nullptr;
  uint32_t chunk_bytes = 8192;      // collect warp-task size (LSU path)
  uint32_t tma_chunk = 16384;       // collect TMA stage size
  int update_fused = 1;             // single-CTA tag+apply update when it fits
  int tma_ctas = 2;                 // TMA collect CTAs per SM
  int tma_stages = 3;               // shared-memory stages per TMA CTA
  int collect_impl = 1;             // 1: TMA bulk copies for large aligned rows, 0: LSU only
  int evict_first = -1;             // collect copies L2 evict-first: -1 auto (W > 1 after TopK), 0, 1
  bool last_topk = false;           // the most recent gear_sample was TopK
  int collect_dynamic = -1;         // TMA tasks from a counter: -1 auto (W > 1 or host rows), 0, 1
  static constexpr uint32_t kDynSlots = 64;  // collects of one table in flight at once (gear.h)
  unsigned long long* dyn_pool = nullptr;  // [kDynSlots][2] task counters (rotating)
  uint64_t dyn_slot = 0;
  int collect_peer_lsu = 0;         // W > 1: peer-HBM rows of TMA columns via LSU warps
  int collect_host_lsu = -1;        // host-resident TMA columns via the TMA kernel's LSU warps (-1: rows <= 16 KB)
};
