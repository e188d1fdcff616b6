// gear_internal.h -- structures shared by the host runtime (api.cpp, comm.cpp)
// and the sm_100a kernels (kernels/*.cu).  Not part of the C-ABI.
#pragma once

#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>

namespace gear {

constexpr int kMaxCols = 16;
constexpr int kMaxRanks = 8;
constexpr int kMaxShards = 32;
constexpr uint64_t kIdxNone = ~0ull;

// Device error latch bits (mirror GEAR_DEVERR_* of gear.h).
constexpr uint32_t kErrIndexRange = 1u;
constexpr uint32_t kErrBadPriority = 2u;
constexpr uint32_t kErrStale = 4u;
constexpr uint32_t kErrEmpty = 8u;

constexpr uint32_t kErrTimeout = 16u;
constexpr uint32_t kErrFull = 32u;

// Last-writer-wins tags of the update / commit passes (kernels/update.cu,
// alloc.cu): tag = epoch << 24 | low, low = an entry's rank in its call
// (< 2^24: create checks W * max_batch < 2^24).  The epoch is a 40-bit
// device counter advanced once per update / commit call, so tags of earlier
// calls compare smaller and the tag array never needs clearing; it wraps
// after 2^40 calls (~4.8 years at 7,300 calls/s).
constexpr int kTagLowBits = 24;
constexpr uint32_t kTagLowMax = (1u << kTagLowBits) - 1;
__host__ __device__ __forceinline__ unsigned long long make_tag(uint64_t epoch, uint32_t low) {
  return ((unsigned long long)epoch << kTagLowBits) | (unsigned long long)low;
}

// Strategy codes (mirror gear_strategy).
constexpr int kFifo = 0, kLifo = 1, kUniform = 2, kWeighted = 3, kPrioritized = 4;

// Priority quantisation parameters (common.cuh quantize): key = Q_F(p^alpha).
struct Quant {
  uint64_t q_max;
  uint32_t frac_bits;
  uint32_t pad;
  double alpha;  // PER exponent (1: the priority itself)
};

// Two-level CDF (kernels/scan.cu, scan2): tiles of kCdfTile keys per shard,
// each with its own inclusive prefix, plus a per-shard inclusive prefix of
// the tile totals.  Key writers mark the tile of every key they change dirty
// for both CDF buffers (bits 0 and 1); a rebuild of buffer b rescans only the
// tiles whose bit b is set.
constexpr uint32_t kCdfTile = 4096;
struct TileDirty {
  uint32_t* bits;           // [R * tiles_per_shard]
  uint64_t shard_cap;       // C_s
  uint32_t tiles_per_shard;
  uint32_t pad;
};

// Per-shard totals record exchanged between ranks (16 B): total weight T_s of
// the shard's CDF with the CDF buffer parity in bit 63 (T_s < 2^62 by q_max),
// and the number of valid FIFO/LIFO candidates the shard offers.
struct ShardTotals {
  uint64_t total_and_parity;
  uint64_t aux;
};

// One priority-update entry after quantisation (24 B), exchanged between
// ranks for a collective update.
struct UpdRec {
  uint64_t idx;    // global id, or kIdxNone for a skipped entry
  uint64_t q;      // fixed-point key Q_F(p)
  uint32_t gen;    // expected generation when flags & 2
  uint32_t flags;  // bit0 valid, bit1 has generation
};

// Device-resident block allocator state of one local shard (kernels/alloc.cu):
// free slots are [next_free, C_s); committed slots sit in commit order in the
// ring ord[shard_local*C_s + (head + i) % C_s], i < len.
struct AllocState {
  uint64_t next_free;
  uint64_t seq_ctr;  // next seq (starts at 1; 0 = never committed / ongoing)
  uint32_t head;
  uint32_t len;
};

// One row written by gear_insert (planned on the device, kernels/alloc.cu).
struct InsMeta {
  uint64_t local;    // rank-local slot (shard_local * C_s + i); kIdxNone: a later row wins
  uint64_t seq;      // new seq value
  uint32_t gen_inc;  // how many inserts landed in the slot in this call
  uint32_t src_row;  // row of the caller's source arrays that wins the slot
  double prio;       // priority of that row (validated on the host)
};

// One ring-order entry written by gear_insert: ord[pos] = slot (both
// rank-local; pos indexes the rank's concatenated per-shard rings;
// 0xffffffff: a later row owns the position).
struct OrdRec {
  uint32_t pos;
  uint32_t slot;
};

// FIFO/LIFO candidate (16 B): the ordering key is (seq, shard).
struct Cand {
  uint64_t seq;
  uint32_t shard;
  uint32_t slot;  // shard-local slot
};

// Per-shard state of the multi-CTA TopK radix select (kernels/topk.cu);
// zero-initialised once, re-armed by the kernels themselves.
constexpr uint32_t kTopkMaxCtas = 512;  // CTAs per shard
constexpr uint32_t kTopkEqMax = 2048;   // extra candidates beyond K the sort may rank
struct TopkState {
  unsigned long long max_key;  // stats: largest key
  uint64_t prefix;             // select: key bits fixed so far (== T* when done)
  uint64_t mask;
  uint32_t n_sel;     // stats: selectable keys
  uint32_t k_remain;  // keys still to take among those matching the prefix
  int shift;          // next byte to resolve; < 0 when done
  uint32_t all;       // n_sel <= K: take every selectable key
  uint32_t ctr;       // last-CTA counter
  uint32_t eq_all;    // select stopped on a small bin: take all of it, the sort keeps K
  uint32_t hist[256];
};

// Peer mailboxes (W > 1).  Every rank owns one device allocation that all
// peers map through CUDA IPC and write over NVLink; the small per-step
// exchanges (shard totals, update records, FIFO/LIFO candidates) are remote
// stores + a release flag carrying the exchange's epoch, consumed in place by
// the next kernel -- no NCCL launch on the step.  Two buffers (epoch & 1)
// alternate: a peer can only be one exchange ahead.
struct MboxLayout {
  uint64_t totals;  // ShardTotals [2][S]
  uint64_t tflag;   // u64 [2][W]
  uint64_t upd;     // UpdRec [2][W][MB]
  uint64_t uflag;   // u64 [2][W]
  uint64_t cand;    // Cand [2][S][K], K = W*MB
  uint64_t ccnt;    // ShardTotals [2][S] (aux = candidate count)
  uint64_t cflag;   // u64 [2][S]
  uint64_t bytes;
};

__host__ __device__ inline MboxLayout mbox_layout(uint32_t W, uint32_t S, uint32_t MB) {
  MboxLayout l;
  const uint64_t K = (uint64_t)W * MB;
  uint64_t o = 0;
  l.totals = o; o += 2ull * S * sizeof(ShardTotals);
  l.tflag = o;  o += 2ull * W * 8;
  l.upd = o;    o += 2ull * W * MB * sizeof(UpdRec);
  l.uflag = o;  o += 2ull * W * 8;
  l.cand = o;   o += 2ull * S * K * sizeof(Cand);
  l.ccnt = o;   o += 2ull * S * sizeof(ShardTotals);
  l.cflag = o;  o += 2ull * S * 8;
  l.bytes = (o + 255) & ~255ull;
  return l;
}

// Kernel-parameter view of every rank's mailbox.
struct Mbox {
  uint8_t* base[kMaxRanks];  // base[rank] is this rank's own mailbox
  uint32_t W, rank, S, R, MB;
  uint64_t* epoch_dev;       // this exchange kind's counter (device): the next
                             // exchange is *epoch_dev + 1; the kernels advance it
  uint64_t epoch;            // filled in-kernel from epoch_dev (buffer = epoch & 1)
};

struct CollectCol {
  uint8_t* out;                       // [n][rb] output batch
  const uint8_t* src[kMaxRanks];      // device-accessible base of each rank's rows
  uint64_t rb;                        // row bytes
  uint64_t chunk_begin;               // first task id of this column in its task space
  uint32_t chunks_per_row;
  uint32_t chunk;                     // bytes per task of this column
  uint32_t vec;                       // LSU vector width in bytes: 16, 8, 4, 2 or 1
  uint32_t tma;                       // 1: moved by TMA bulk copies (16-B aligned rows)
  uint32_t peer_lsu;                  // TMA column whose peer-HBM rows the LSU warps move
  uint32_t host_lsu;                  // TMA column (host-resident) whose rows the LSU warps move
};

struct CollectParams {
  CollectCol col[kMaxCols];
  const uint64_t* idx;                // [n] global ids (device)
  const InsMeta* meta;                // non-null: insert scatter -- row j of the source
                                      // (col.src[0], row meta[j].src_row) goes to table slot
                                      // meta[j].local of col.out; kIdxNone rows are skipped
  uint64_t rows_per_rank;             // R * C_s
  uint64_t n_global;                  // N
  uint64_t lsu_total;                 // tasks of the LSU (warp-copy) space
  uint64_t tma_total;                 // tasks of the TMA bulk-copy space
  uint8_t lsu_cols[kMaxCols];
  uint8_t tma_cols[kMaxCols];
  uint32_t n_lsu;
  uint32_t n_tma;
  uint32_t tma_ctas_per_sm;           // CTAs of the TMA kernel per SM
  uint32_t tma_stages;                // 2, 3, 4, 6 or 8 shared-memory stages per CTA
  uint32_t ncols;
  uint32_t n;
  uint32_t self_rank;                 // this rank (peer rows: owner != self_rank)
  uint32_t any_peer_lsu;              // some column has peer_lsu or host_lsu
  uint32_t evict_first;               // bulk copies with an L2 evict-first policy
  unsigned long long* dyn_ctr;        // non-null: TMA tasks claimed from this counter pair
  uint32_t* err;
};

struct SampleParams {
  const ShardTotals* totals;          // [S] (ignored when xchg: taken from the mailbox)
  const ShardTotals* totals_local;    // [R] this rank's totals (xchg)
  Mbox mbox;
  int xchg;                           // 1: exchange the totals through the mailboxes first
  const uint64_t* const* cdf_ptrs;    // [2*S]: parity p of shard s at [p*S + s]
  const uint32_t* const* gen_ptrs;    // [W]: each rank's gen array
  uint64_t shard_cap;                 // C_s
  uint32_t n_shards;                  // S
  uint32_t shards_per_rank;           // R
  uint32_t cdf_levels;                // 1: flat CDF (scan_kernel), 2: two-level (scan2_kernel)
  uint32_t tiles_per_shard;           // two-level: tiles of kCdfTile keys per shard
  uint64_t seed;
  uint32_t rank;
  uint32_t B;
  double beta;
  int strategy;
  uint64_t* out_idx;
  float* out_w;
  double* out_p;
  uint32_t* out_gen;
  const uint32_t* draw_list;          // [B] draw numbers j of the slice, or null: rank*B + b
  uint64_t* seed_dev;                 // non-null: key = *seed_dev, advanced by the kernel
  uint64_t* q_scratch;                // [B]
  unsigned long long* qmin_slot;      // reset to ~0 by the last block
  uint32_t* done_ctr;                 // reset to 0 by the last block
  uint32_t* err;
};

// Owner-affine assignment of the global batch (kernels/assign.cu).
struct AssignParams {
  const ShardTotals* totals;        // draws: CDF totals [S] (null for FIFO/LIFO)
  const ShardTotals* totals_local;  // draws with xchg: this rank's [R] totals
  Mbox mbox;
  int xchg;                         // 1: exchange the totals through the mailboxes first
  const ShardTotals* fifo_totals;   // FIFO/LIFO: candidate counts [S] (null for draws)
  int fifo_mbox;                    // 1: FIFO/LIFO counts are in the mailbox (fifo_totals unused)
  const uint32_t* glob_shard;       // FIFO/LIFO merged global list [K] (null for draws)
  const uint32_t* glob_slot;
  uint32_t n_shards;
  uint32_t shards_per_rank;
  uint32_t W;
  uint32_t rank;
  uint32_t B;
  uint64_t seed;
  const uint64_t* seed_dev;         // non-null: the key is *seed_dev (read only)
  uint64_t shard_cap;
  uint32_t* draw_list;              // [B] out: global entry j of each slice position
  uint32_t* pos_scratch;            // [K]
  uint32_t* ov_scratch;             // [K]
  uint64_t* out_idx;                // FIFO/LIFO outputs (written by the assign kernel)
  float* out_w;
  double* out_p;
  uint32_t* out_gen;
  const uint32_t* const* gen_ptrs;
  uint32_t* err;
};

// ---- kernel launchers (kernels/*.cu) --------------------------------------

// Counts every kernel launch of the library (gear_kernel_launches()).
void count_launch(uint64_t n = 1);

// K1: per-shard inclusive u64 scan with decoupled look-back.  Writes cdf for
// `n_shards_local` contiguous shards of `shard_cap` keys and their totals.
// indicator != 0 scans [key > 0] instead of key.
// status [tiles], ticket and done counter start at 0 and are left at 0 by the
// kernel itself (the last tile re-arms them), so launches can be replayed.
// Builds into cdf1 if the device parity *par_dev is 0, else cdf0, then flips it.
cudaError_t launch_scan(const uint64_t* key, uint64_t* cdf0, uint64_t* cdf1, uint64_t shard_cap,
                        uint32_t n_shards_local, int indicator, uint64_t* par_dev,
                        ShardTotals* totals_out, uint64_t* status0, uint64_t* status1, uint32_t* ticket,
                        uint32_t* done, int chunked, cudaStream_t s);
uint32_t scan_tiles_per_shard(uint64_t shard_cap);
// Two-level incremental CDF (scan.cu, scan2_kernel): cdf0/cdf1 hold
// R*C_s tile-local prefixes followed by R*tiles_per_shard tile prefixes;
// ttot holds each buffer's tile totals ([2][R*tiles_per_shard]).
cudaError_t launch_scan2(const uint64_t* key, uint64_t* cdf0, uint64_t* cdf1, uint64_t shard_cap,
                         uint32_t n_shards_local, int indicator, uint64_t* par_dev,
                         ShardTotals* totals_out, uint32_t* dirty, uint64_t* ttot,
                         uint32_t* buf_mode, uint32_t* shard_ctr, uint32_t* done,
                         cudaStream_t s);

// K2/K3/K7: draw + warp-cooperative search + IS weights.
cudaError_t launch_sample(const SampleParams& p, cudaStream_t s);

// K6: priority update.
// prio (f32 or f64) -> RN(p^alpha) as f64 (0 and invalid values unchanged).
cudaError_t launch_alpha(const void* prio, int prio_is_f64, uint32_t n, double alpha,
                         double* out, cudaStream_t s);
cudaError_t launch_update_quantize(const uint64_t* idx, const void* prio, int prio_is_f64,
                                   const uint32_t* gen, uint32_t n, uint64_t n_global,
                                   Quant qz, UpdRec* out,
                                   uint32_t* err, cudaStream_t s);
cudaError_t launch_update_tag(const UpdRec* recs, uint32_t m, uint64_t local_begin,
                              uint64_t local_rows, const uint32_t* gen, const uint64_t* seq, unsigned long long* tag,
                              uint64_t* epoch_dev, unsigned long long* n_stale, uint32_t* err,
                              cudaStream_t s);
cudaError_t launch_update_apply(const UpdRec* recs, uint32_t m, uint64_t local_begin,
                                uint64_t local_rows, const uint32_t* gen,
                               const uint64_t* seq,
                                const unsigned long long* tag, uint64_t* epoch_dev, uint64_t* key,
                                TileDirty td, cudaStream_t s);

// Single-launch update for m <= update_fused_max() entries (one CTA): raw
// W = 1 inputs when idx != nullptr, else all-gathered records.
uint32_t update_fused_max();
cudaError_t launch_update_fused(const uint64_t* idx, const void* prio, int prio_is_f64,
                                const uint32_t* gen_in, const UpdRec* recs, uint32_t m,
                                uint64_t n_global, Quant qz,
                                uint64_t local_begin, uint64_t local_rows, const uint32_t* gen,
                               const uint64_t* seq,
                                unsigned long long* tag, uint64_t* epoch_dev,
                                unsigned long long* n_stale, uint32_t* err, uint64_t* key,
                                TileDirty td, cudaStream_t s);

// W > 1 collective update through the peer mailboxes, one launch (n*W <=
// update_fused_max()).
cudaError_t launch_update_xchg(const uint64_t* idx, const void* prio, int prio_is_f64,
                               const uint32_t* gen_in, uint32_t n, uint64_t n_global,
                               Quant qz, const Mbox& mb,
                               uint64_t local_begin, uint64_t local_rows, const uint32_t* gen,
                               const uint64_t* seq,
                               unsigned long long* tag, uint64_t* epoch_dev,
                               unsigned long long* n_stale, uint32_t* err, uint64_t* key,
                               TileDirty td, cudaStream_t s);

// K5: collect (gather) and the insert-side scatter.
cudaError_t launch_collect(const CollectParams& p, cudaStream_t s);
cudaError_t launch_insert_meta(const InsMeta* meta, uint32_t m, const OrdRec* ord_recs,
                               uint32_t n_ord, Quant qz,
                               uint64_t* key, TileDirty td, uint64_t* seq, uint32_t* gen,
                               uint32_t* ord, cudaStream_t s);

// NEXT-1: device-resident allocator (kernels/alloc.cu).
// Device priorities of gear_insert: *bad = any invalid (all or nothing).
cudaError_t launch_validate_prio(const double* prio, uint32_t n, uint32_t* bad, uint32_t* err,
                                 cudaStream_t s);
// abort_flag != null: plan nothing when *abort_flag (the validation failed).
cudaError_t launch_insert_plan(AllocState* st, uint32_t ls, uint32_t shard, uint64_t Cs, int lifo,
                               uint32_t m, const double* prio, const uint32_t* ord,
                               const uint32_t* abort_flag, InsMeta* meta, OrdRec* ord_recs,
                               uint64_t* out_idx, uint32_t* err, cudaStream_t s);
cudaError_t launch_allocate(AllocState* st, uint32_t ls, uint32_t shard, uint64_t Cs, int lifo,
                            uint32_t n, const uint32_t* ord, uint64_t* key, uint64_t* seq,
                            uint32_t* gen, TileDirty td, uint64_t* out_idx, uint32_t* err,
                            cudaStream_t s);
cudaError_t launch_commit(AllocState* st, uint32_t ls, uint32_t shard, uint64_t Cs, uint32_t n,
                          const uint64_t* idx, const double* prio, Quant qz, uint64_t* key,
                          uint64_t* seq, const uint32_t* gen, uint32_t* ord,
                          unsigned long long* tag, uint64_t* epoch_dev, TileDirty td,
                          uint32_t* err, cudaStream_t s);

// K4: FIFO/LIFO local selection and merge (ring state read from `alloc`).
cudaError_t launch_fifo_local(const uint64_t* key, const uint64_t* seq, const uint32_t* ord,
                              const AllocState* alloc, uint64_t shard_cap,
                              uint32_t n_shards_local, uint32_t first_shard, uint32_t K,
                              int lifo, Cand* cand_out, ShardTotals* totals_out,
                              const Mbox* mbox, cudaStream_t s);
// glob_shard != null: write the whole merged list (glob_shard/glob_slot[K])
// for the owner-affine assignment instead of this rank's slice.
cudaError_t launch_fifo_merge(const Cand* cand_all, const ShardTotals* totals_all,
                              uint32_t n_shards, uint32_t K, int lifo, uint64_t shard_cap,
                              uint32_t rank, uint32_t B, const uint32_t* const* gen_ptrs,
                              uint32_t shards_per_rank, uint64_t* out_idx, float* out_w,
                              double* out_p, uint32_t* out_gen, uint32_t* err,
                              uint32_t* glob_shard, uint32_t* glob_slot, const Mbox* mbox,
                              cudaStream_t s);
cudaError_t launch_assign(const AssignParams& p, cudaStream_t s);
// TopK local selection (kernels/topk.cu): sorted top-K of each local shard;
// merged by launch_fifo_merge with lifo == 2.  K <= topk_max_k().
uint32_t topk_max_k();
cudaError_t launch_topk_local(const uint64_t* key, uint64_t shard_cap, uint64_t q_max,
                              uint32_t n_shards_local,
                              uint32_t first_shard, uint32_t K, Cand* cand_tmp, Cand* cand_out,
                              ShardTotals* totals_out, TopkState* state, uint32_t* cnt,
                              const Mbox* mbox, cudaStream_t s);
// Advances a device-resident exchange epoch by one (FIFO/LIFO exchange).
cudaError_t launch_epoch_bump(uint64_t* counter, cudaStream_t s);

}  // namespace gear
