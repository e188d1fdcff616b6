/*
 * gear.h -- C-ABI of the B200-native GEAR replay hot path.
 *
 * GEAR (arXiv 2310.05205, /root/reference/PAPER.md) keeps RL trajectories in
 * column tables sharded across the training servers' memory,
 * selects a batch with GPU kernels and collects the selected
 * rows into a training batch with GPU kernels that read HBM, host memory
 * (zero-copy) and remote shards.  This library is that hot
 * path for one 8xB200 box: one process (rank) per GPU, the table sharded by
 * trajectory id, one or more shards per rank.
 *
 * Conventions (all functions):
 *  - Every function returns gear_status; GEAR_OK is 0, errors are negative.
 *    On error the thread-local gear_last_error() string explains it.
 *  - `stream` is a cudaStream_t passed as void* (0 = legacy default stream).
 *    All device work of a call is enqueued on that stream; calls return
 *    before the work completes.  Outputs are valid after the stream reaches
 *    the call.  Errors that only the device can see (an id out of range, a
 *    bad priority, nothing selectable) are latched into a per-table word and
 *    returned by gear_table_sync().
 *  - Small per-call arrays (ids, priorities, generations, sample outputs) may
 *    be DEVICE or HOST pointers; the library detects which.  Pinned host
 *    memory keeps the call asynchronous (update inputs and sample outputs are
 *    read / written in place by the kernels through their mapped address);
 *    pageable host memory goes through per-table scratch with a synchronous
 *    copy, so calls with pageable arrays must be ordered among themselves
 *    (one stream).  Collect outputs must be device memory (or mapped pinned).
 *  - Streams: sample and update of a table must be issued in one order (they
 *    share the keys and, at W > 1, the exchange epochs); collects and writers
 *    may run on other streams ordered by events, as bench.py does.  At most
 *    64 collects of one table may be in flight at once (each launch takes one
 *    of 64 rotating task counters).
 *  - The caller owns every argument buffer and must keep it alive until the
 *    stream has reached the call.  The table owns its columns, keys, CDFs and
 *    scratch.
 *  - "Collective" calls must be made by every rank of the table's comm, in
 *    the same order, with the same scalar arguments (SPMD).
 *  - One host thread per table per rank.
 *
 * Global ids.  With W ranks and R shards per rank there are S = W*R shards
 * of equal capacity C_s = capacity_global / S; shard s owns global ids
 * [s*C_s, (s+1)*C_s) and lives on rank s / R.  Translation of a global id g
 * is shard = g / C_s, local = g mod C_s.
 */
#ifndef GEAR_H
#define GEAR_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t gear_status;
#define GEAR_OK 0
#define GEAR_ERR_INVALID_ARG (-1)   /* bad argument, size or combination */
#define GEAR_ERR_OUT_OF_MEMORY (-2) /* device or pinned host allocation failed */
#define GEAR_ERR_CUDA (-3)          /* a CUDA runtime call failed */
#define GEAR_ERR_NCCL (-4)          /* an NCCL call failed */
#define GEAR_ERR_EMPTY (-5)         /* nothing (or too little) selectable */
#define GEAR_ERR_INDEX_RANGE (-6)   /* a global id >= capacity_global */
#define GEAR_ERR_BAD_PRIORITY (-7)  /* NaN, +-inf or negative priority */
#define GEAR_ERR_STATE (-8)         /* wrong call order / latched device error */
#define GEAR_ERR_UNSUPPORTED (-9)   /* valid request this build does not do */

/* Bits of the device-side error word returned by gear_table_sync(). */
#define GEAR_DEVERR_INDEX_RANGE 1u  /* an update/collect id was >= capacity_global */
#define GEAR_DEVERR_BAD_PRIORITY 2u /* an update priority was NaN/inf/negative */
#define GEAR_DEVERR_STALE 4u        /* an update hit a never-inserted slot or a stale generation */
#define GEAR_DEVERR_EMPTY 8u        /* a sample found nothing (or < W*B for FIFO/LIFO) selectable */
#define GEAR_DEVERR_TIMEOUT 16u     /* a peer-mailbox exchange waited > 4 s for a peer (SPMD broken) */
#define GEAR_DEVERR_FULL 32u        /* an insert / allocate found too few free or committed slots */

/* Padding id: update entries with this id are ignored (lets ranks with fewer
 * updates pass the common n of a collective update). */
#define GEAR_IDX_NONE UINT64_MAX

typedef void* gear_stream; /* cudaStream_t */

typedef enum {
  GEAR_U8 = 0,
  GEAR_I32 = 1,
  GEAR_I64 = 2,
  GEAR_F32 = 3,
  GEAR_F64 = 4,
  GEAR_BF16 = 5
} gear_dtype;

/* Where a column's rows live: device HBM of the owning rank, or pinned host
 * memory read by the GPUs zero-copy over PCIe. */
typedef enum { GEAR_DEVICE = 0, GEAR_HOST = 1 } gear_placement;

/* Selection strategies.  FIFO/LIFO select the W*B
 * oldest / newest selectable trajectories (decentralised);
 * UNIFORM/WEIGHTED/PRIORITIZED draw W*B ids with replacement from the CDF of
 * [key>0] / key (centralised).  PRIORITIZED also returns
 * importance-sampling weights (q_min/q)^beta over the rank's slice.  TOPK
 * (decentralised like FIFO) selects the W*B selectable
 * trajectories with the largest priority keys, ties by the smaller global id,
 * in that order (W*B <= 129024). */
typedef enum {
  GEAR_FIFO = 0,
  GEAR_LIFO = 1,
  GEAR_UNIFORM = 2,
  GEAR_WEIGHTED = 3,
  GEAR_PRIORITIZED = 4,
  GEAR_TOPK = 5
} gear_strategy;

/* Bit of gear_sample's `flags`: owner-affine assignment of
 * the same global batch (Q19; data locality, "the
 * majority of the trajectories collected by the servers reside in local
 * memory").  Instead of the contiguous positions [r*B, (r+1)*B), rank r keeps
 * up to B entries of the global batch that its own shards own (in global
 * order); the surplus of over-full owners, in global order, fills the
 * under-full ranks in rank order.  Same W*B entries, same distribution, so
 * each rank mostly collects rows from its own HBM instead of over NVLink. */
#define GEAR_SAMPLE_OWNER_AFFINE 0x100

/* Bit of gear_sample's `flags`: the draw key is the table's
 * device-resident seed counter instead of the `seed` argument, and the call
 * advances the counter on the device (set it with gear_table_set_tuning(t,
 * "device_seed", value)).  Consecutive calls use value, value+1, ... even when
 * the calls are captured once in a CUDA graph and replayed (every other
 * per-call counter -- update epoch, mailbox epochs, CDF parity -- is
 * device-resident too, so captured steps replay correctly at any W). */
#define GEAR_SAMPLE_DEVICE_SEED 0x200

/* Victim choice when a shard is full. */
typedef enum { GEAR_REMOVE_FIFO = 0, GEAR_REMOVE_LIFO = 1 } gear_removal;

/* One column table: a field of every trajectory; its row
 * ("block") is seq_len * prod(shape) elements of dtype, stored contiguously. */
typedef struct {
  const char* name;        /* unique, non-empty, <= 63 chars */
  gear_dtype dtype;
  uint32_t ndim;           /* <= 8; 0 means a scalar per step */
  const int64_t* shape;    /* per-step shape, ndim entries, all > 0 */
  gear_placement placement;
} gear_column_desc;

typedef struct {
  uint64_t capacity_global;    /* N: trajectories in the whole table; divisible by S */
  uint32_t seq_len;            /* steps per trajectory (>= 1), folded into every row */
  uint32_t ncols;              /* 1..16 */
  const gear_column_desc* cols;
  uint32_t priority_frac_bits; /* F of the fixed-point priority Q_F (0 -> 32; max 62) */
  gear_removal removal;        /* victim rule of gear_insert when a shard is full */
  uint32_t shards_per_rank;    /* R (0 -> 1); W*R <= 32.  R > 1 emulates a
                                  larger world on fewer GPUs (tests). */
  uint32_t max_batch;          /* upper bound of B and of per-call n (0 -> 4096);
                                  W * max_batch < 2^24 */
  double priority_alpha;       /* PER exponent alpha (Schaul et al.; Q7):
                                  every priority p of gear_insert and
                                  gear_update_priorities becomes the key
                                  Q_F(p^alpha) with p^alpha rounded to the nearest
                                  double (p = 0 stays 0).  0 -> 1 (the priority
                                  itself); alpha = 0 is GEAR_UNIFORM.  Finite,
                                  >= 0, else INVALID_ARG. */
} gear_table_desc;

typedef struct {
  uint64_t capacity_global;  /* N */
  uint64_t shard_capacity;   /* C_s */
  uint32_t n_ranks;          /* W */
  uint32_t rank;
  uint32_t shards_per_rank;  /* R */
  uint32_t ncols;
  uint64_t row_bytes_total;  /* sum of the columns' row bytes */
  uint64_t q_max;            /* largest fixed-point key = floor((2^62-1)/N) */
  double p_max;              /* q_max / 2^F: values of p^alpha above it saturate */
  uint32_t frac_bits;
  uint32_t max_batch;
  double alpha;              /* PER exponent of the keys */
} gear_table_info;

typedef struct gear_comm gear_comm;
typedef struct gear_table gear_table;

/* Thread-local description of the last error on this thread ("" if none). */
const char* gear_last_error(void);

/* Library version string. */
const char* gear_version(void);

/* Number of kernels this library has launched in the process so far
 * (diagnostics: bench.py reports the count inside its timed region). */
uint64_t gear_kernel_launches(void);

/* --- communicator (one per rank; wraps an NCCL communicator, or a host
 *     all-gather callback: gear_comm_create_host) --------------------------- */

/* Rank 0 creates the 128-byte unique id and the caller broadcasts it to the
 * other ranks by any means (the Python binding uses torch.distributed). */
gear_status gear_get_unique_id(uint8_t out[128]);

/* Collective over all nranks.  `device` is this rank's CUDA device; it is
 * made current.  (Peer memory is mapped per table, through CUDA IPC, by
 * gear_table_create.) */
gear_status gear_comm_create(int nranks, int rank, const uint8_t id[128], int device,
                             gear_comm** out);

/* Host all-gather callback of gear_comm_create_host: gather `bytes` bytes of
 * `send` from every rank into `recv` (nranks * bytes, rank order).  Host
 * pointers.  Returns 0 on success.  Called only from the thread that makes
 * the gear call, and only by calls every rank makes (create, destroy,
 * barriers, the peer_xchg = 0 exchanges). */
typedef int (*gear_allgather_fn)(void* ctx, const void* send, void* recv, size_t bytes);

/* Collective over all nranks: a communicator bootstrapped WITHOUT NCCL, through
 * the caller's host all-gather (the Python binding passes a torch.distributed
 * gloo group).  Unlike gear_comm_create, several ranks may share one CUDA
 * device (NCCL refuses that): every per-step exchange of the hot path is a
 * peer-mailbox store through CUDA-IPC mappings, which work between processes
 * on one device as between devices, so the multi-rank device path (totals /
 * update / FIFO / TopK mailboxes, owner-CDF search, peer collect, shared host
 * shards) runs unchanged -- kernels of different processes on one GPU are
 * time-sliced, so it is a correctness vehicle, not a performance one.  The
 * peer_xchg = 0 fallback exchanges go through the callback synchronously
 * (device -> host copy, all-gather, host -> device copy; not capturable in a
 * CUDA graph: UNSUPPORTED while the stream is capturing).  `fn` and `ctx`
 * must stay valid until gear_comm_destroy. */
gear_status gear_comm_create_host(int nranks, int rank, int device, gear_allgather_fn fn,
                                  void* ctx, gear_comm** out);
gear_status gear_comm_destroy(gear_comm* comm);

/* --- table ------------------------------------------------------------- */

/* Collective when comm != NULL (comm == NULL means W = 1).  Allocates this
 * rank's R shards: DEVICE columns with cudaMalloc, HOST columns as pinned
 * mapped host memory (W > 1: POSIX shared memory registered with every GPU so
 * any rank can read any shard's host rows over its own PCIe link), plus keys
 * (u64 fixed point), seq (u64), gen (u32), two CDF buffers and scratch, and
 * exchanges peer pointers (CUDA IPC) so kernels can read peer shards over
 * NVLink.  Errors: INVALID_ARG (N not divisible by S, duplicate or empty
 * names, zero-size rows, S > 32, ncols > 16, W * max_batch >= 2^24),
 * OUT_OF_MEMORY, CUDA, NCCL. */
gear_status gear_table_create(const gear_table_desc* desc, gear_comm* comm, gear_table** out);

/* Collective when the table has a comm.  Frees everything. */
gear_status gear_table_destroy(gear_table* t);

gear_status gear_table_info_get(const gear_table* t, gear_table_info* info);

/* Column index of `name`, or INVALID_ARG. */
gear_status gear_column_id(const gear_table* t, const char* name, uint32_t* out);

/* Row bytes of column `col`. */
gear_status gear_column_row_bytes(const gear_table* t, uint32_t col, uint64_t* out);

/* --- hot path ---------------------------------------------------------- */

/* Insert n trajectories into global shard `shard`, which must be owned by
 * this rank (online data goes to the local shard).  Not
 * collective.  Allocation follows PAPER.md:186-195: a per-shard free queue
 * seeded 0..C_s-1 ascending; when it is empty the victim is the oldest (FIFO
 * removal) or newest (LIFO removal) committed slot.  Each inserted slot gets
 * seq = the shard's next counter value (starting at 1), gen += 1, and
 * key = Q_F(prio[k]).
 *   col_src[c]: n rows of column c, [n][row_bytes_c], host or device.
 *   prio:       n f64 priorities (0 = stored, not selectable), host or
 *               device.  Host priorities are validated before anything is
 *               inserted (BAD_PRIORITY returned); device priorities by a
 *               kernel (GEAR_DEVERR_BAD_PRIORITY latched, nothing inserted),
 *               so a call with device rows and priorities and a device (or
 *               NULL) out_idx never blocks the host and can be captured.
 *   out_idx:    n u64 global ids (host or device), may be NULL.
 * Each row is allocated and committed before the next (victims are
 * committed slots only -- never ongoing ones of gear_allocate).  If two of
 * the n rows land in one slot (LIFO removal, or n > free + committed slots)
 * the later row wins.  The allocation runs on the device (kernels/alloc.cu);
 * a host out_idx makes the call synchronise the stream.  Errors: INVALID_ARG,
 * BAD_PRIORITY (nothing inserted); GEAR_DEVERR_FULL is latched (nothing
 * inserted) when every slot of the shard is ongoing.  Must not overlap a
 * sample/collect of the same step on any rank (caller barrier). */
gear_status gear_insert(gear_table* t, uint32_t shard, uint32_t n, const void* const* col_src,
                        const double* prio, uint64_t* out_idx, gear_stream stream);

/* Split writer API ("the client initiates an allocate
 * operation, which generates a buffer containing memory views of the blocks
 * ... fills with trajectory data ... commits the buffer, triggering an update
 * in the Status Table"; reading Q21).  Not collective; the block allocator of
 * each shard lives in device memory, so both calls are stream-ordered, need
 * no host round trip (unless out_idx is a host pointer: then the call
 * synchronises the stream) and can be captured in a CUDA graph.
 *
 * gear_allocate: n slots of global shard `shard` (owned by this rank): free
 *   slots first (queue seeded 0..C_s-1 ascending), then victims evicted from
 *   the committed slots -- the oldest first (FIFO removal) or the newest
 *   first (LIFO removal).  Each allocated slot is ongoing:
 *   gen += 1, key = 0 and seq = 0, so it is not selectable, not a victim, and
 *   updates to it are skipped as stale, until it is committed.  out_idx:
 *   u64[n] global ids (device or host).  All or nothing: with fewer than n
 *   free + committed slots, nothing is allocated, out_idx gets GEAR_IDX_NONE
 *   and GEAR_DEVERR_FULL is latched.
 * The caller writes each allocated trajectory's rows IN PLACE: row of global
 *   id g in column c is at gear_column_base(c) + (g - rank*R*C_s) * row_bytes
 *   (device memory for DEVICE columns, mapped host memory for HOST columns),
 *   ordered before the commit on the stream.
 * gear_commit: in order, every ongoing id of `shard` gets seq = the shard's
 *   next counter value and key = Q_F(prio[k]^alpha), and joins the shard's
 *   FIFO/LIFO order.  idx: u64[n] (device or host); prio: f64[n] (device or
 *   host).  Entries outside the shard (INDEX_RANGE), not ongoing -- never
 *   allocated, already committed, the second copy of a duplicate -- (STALE)
 *   or with an invalid priority (BAD_PRIORITY; the slot stays ongoing) are
 *   skipped and latched.  n <= max_batch for both calls. */
gear_status gear_allocate(gear_table* t, uint32_t shard, uint32_t n, uint64_t* out_idx,
                          gear_stream stream);
gear_status gear_commit(gear_table* t, uint32_t shard, uint32_t n, const uint64_t* idx,
                        const double* prio, gear_stream stream);

/* Base address of this rank's rows of column `col` (R*C_s rows of
 * row_bytes, rank-local slot order): a device pointer for DEVICE columns, the
 * mapped host pointer for HOST columns. */
gear_status gear_column_base(const gear_table* t, uint32_t col, void** out);

/* Set the priorities of n trajectories.  Collective: every rank passes the
 * same n; pad with GEAR_IDX_NONE.  idx: u64 global ids; prio: n values of
 * prio_dtype (GEAR_F32 or GEAR_F64); gen: optional u32 generations (entries
 * whose generation differs from the slot's are skipped as stale, as are
 * never-inserted slots and allocated but uncommitted ones).  The
 * priority becomes key = Q_F(v), v = RN(p^alpha) (v = p for alpha 1):
 * p == 0 -> 0 (not selectable), else clamp(round_half_even(v * 2^F), 1,
 * q_max).  Entries of all ranks are applied in (rank, position) order -- the
 * last writer wins.  idx / prio / gen may be device memory, pinned host
 * memory (read in place by the kernel over PCIe) or pageable host memory
 * (copied).  Device-side errors (id >= N, bad p, stale) skip the entry and
 * are latched.  n <= max_batch; n == 0 is valid and applies nothing (still
 * collective at W > 1). */
gear_status gear_update_priorities(gear_table* t, uint32_t n, const uint64_t* idx,
                                   const void* prio, gear_dtype prio_dtype, const uint32_t* gen,
                                   gear_stream stream);

/* Select this rank's B trajectories.  Collective.  One global batch of W*B
 * is selected; rank r receives positions [r*B, (r+1)*B).
 *  UNIFORM/WEIGHTED/PRIORITIZED: draw j uses
 *    Philox4x32-10(counter=(j_lo, j_hi, 0, 0), key=(seed_lo, seed_hi)),
 *    r = x0 | x1<<32, u = floor(r*T/2^64) with T the total weight, and
 *    returns min{g : CDF[g] > u}.  Deterministic in (table, seed), independent
 *    of W, R and launch shape.
 *  FIFO/LIFO: the W*B selectable trajectories with the
 *    smallest / largest (seq, shard), in that order.
 *  out_idx: u64[B] global ids (required).  out_w: f32[B] importance weights
 *  (PRIORITIZED: (q_min/q)^beta in f64 rounded to f32; otherwise 1).
 *  out_p: f64[B] selection probability q/T (FIFO/LIFO/TOPK: 1).  out_gen:
 *  u32[B] generation of each selected slot.  Optional outputs may be NULL.
 *  Outputs may be device memory or pinned host memory (written in place by
 *  the kernels through the mapped address, stream-ordered) or pageable host
 *  memory (copied at the end of the call).
 *  TOPK: the W*B selectable trajectories with the largest keys, ties by the
 *  smaller global id, in that order (reading Q20; W*B <= 129024).
 *  flags: 0 or GEAR_SAMPLE_OWNER_AFFINE | GEAR_SAMPLE_DEVICE_SEED (other
 *  bits: INVALID_ARG); same value on every rank.
 *  Nothing selectable: outputs get GEAR_IDX_NONE and EMPTY is latched.
 *  B == 0 (on every rank): returns OK with no work (outputs, keys and the
 *  device seed counter untouched). */
gear_status gear_sample(gear_table* t, gear_strategy strategy, uint32_t B, uint64_t seed,
                        double beta, uint64_t* out_idx, float* out_w, double* out_p,
                        uint32_t* out_gen, uint32_t flags, gear_stream stream);

/* Gather rows of ncols columns for n global ids into contiguous batches,
 * rows in request order.  out[c] is a device buffer of
 * n * row_bytes(col_ids[c]) bytes.  DEVICE columns are read from local HBM
 * or a peer's HBM over NVLink; HOST columns are read zero-copy over PCIe.
 * Not collective (peers' memory is read directly).  idx: device or host.
 * An id >= N leaves its output row untouched and latches INDEX_RANGE.
 * n == 0 or ncols == 0: OK, no work. */
gear_status gear_collect(gear_table* t, uint32_t n, const uint64_t* idx, uint32_t ncols,
                         const uint32_t* col_ids, void* const* out, gear_stream stream);

/* Synchronise the device, return and clear the latched device error bits
 * (GEAR_DEVERR_*) and the count of stale update entries.  Either output may
 * be NULL.  Returns STATE if any bit was set, else OK. */
gear_status gear_table_sync(gear_table* t, uint32_t* dev_errors, uint64_t* n_stale);

/* Shard checkpoint ("GEAR allows for trajectory shards to
 * be checkpointed on local SSDs").  gear_table_save writes this rank's R
 * shards -- keys, seq, gen, insertion rings and every column's rows -- to
 * `path` (one file per rank; pass a rank-specific path).  gear_table_load
 * restores such a file into a table created with the same descriptor, world
 * and rank (INVALID_ARG otherwise); the CDF is rebuilt by the next sample.
 * Both synchronise the device and must not overlap other calls on the
 * table; neither is collective. */
gear_status gear_table_save(gear_table* t, const char* path);
gear_status gear_table_load(gear_table* t, const char* path);

/* Tuning knobs of the collect kernel (not collective, no device work):
 *   "collect_impl": 1 = rows >= 4 KB with 16-byte alignment move by TMA bulk
 *                   copies through shared memory (default), 0 = every row
 *                   by warp-wide 16-byte LSU copies;
 *   "lsu_chunk":    bytes per warp task of the LSU path (multiple of 512);
 *   "tma_chunk":    bytes per TMA stage (multiple of 16, 4096..32768;
 *                   default 16384);
 *   "tma_ctas_per_sm": TMA CTAs per SM (default 2), "tma_stages": stages per
 *                   CTA (2, 3, 4, 6, 8; default 3); ctas * stages * tma_chunk
 *                   must stay <= 220 KB (set the smaller knob first);
 *   "device_seed":  set the device seed counter used by GEAR_SAMPLE_DEVICE_SEED
 *                   (synchronises the device);
 *   "peer_xchg":    W > 1 only, same value on every rank: 1 = the per-step
 *                   exchanges (shard totals, update records, FIFO/LIFO
 *                   candidates) are NVLink stores into the peers' mailboxes
 *                   inside the step's kernels (default), 0 = NCCL all-gathers;
 *   "update_fused": 1 = priority updates of <= 8192 entries (all ranks) run
 *                   tag + apply in one single-CTA launch (default), 0 = two
 *                   grid-wide launches;
 *   "collect_dynamic": 1 = the bulk pipeline claims its tasks from a
 *                   per-launch counter, so CTAs that start late (an SM held
 *                   by a concurrent selection kernel) or hit slow rows take
 *                   fewer tasks; 0 = a static stride; -1 = auto (default):
 *                   dynamic at W > 1 or when host-resident rows are read;
 *   "collect_evict_first": the collect's bulk copies carry an L2 evict-first
 *                   policy (the rows stream through once and stop evicting
 *                   the selection's keys / CDFs / mailboxes): -1 = auto
 *                   (default): on at W > 1 after a TopK selection, 0 = off,
 *                   1 = on;
 *   "collect_host_lsu": 1 = the rows of host-resident columns are gathered
 *                   by the bulk-copy kernel's LSU warps (16-B zero-copy
 *                   loads) instead of its bulk pipeline; 0 = bulk pipeline;
 *                   -1 = auto (default): LSU warps for host rows of at most
 *                   16 KB (+2.5% c3 throughput; large host rows keep the
 *                   bulk pipeline);
 *   "collect_peer_lsu": W > 1: 1 = the peer-HBM rows of bulk-copied (TMA)
 *                   columns are moved by the LSU warps instead of the bulk
 *                   pipeline (+3% collect throughput when few rows are
 *                   remote, -11% when half are); 0 = all by the bulk
 *                   pipeline (default);
 *   "cdf_levels":   same value on every rank; 2 = two-level CDF (default):
 *                   every 4096-key tile of a shard holds its own prefix sum,
 *                   the shard a prefix sum of the tile totals, and a rebuild
 *                   rescans only the tiles whose keys changed since that CDF
 *                   buffer was last built (incremental, no look-back);
 *                   1 = one flat prefix sum per shard rebuilt whole by the
 *                   decoupled look-back scan, only when the
 *                   host saw a writer call since the last build (so writers
 *                   replayed from a CUDA graph need cdf_levels 2).  The
 *                   sampled ids are identical (synchronises the device);
 *   "scan_chunk":   cdf_levels 1 only: 1 = the look-back runs over one
 *                   contiguous chunk of keys per resident CTA (two passes
 *                   over the chunk, the second from shared memory / L2),
 *                   0 = over 4096-key tiles (persistent, pipelined), -1 =
 *                   auto (default): chunks when the rank's keys are at most
 *                   GEAR_SCAN_CHUNK_MAX_MB (default 96) MB and span at least
 *                   one tile per CTA; k >= 2 (tests): chunked on at most k
 *                   CTAs, each claiming several chunks.  Identical CDF
 *                   either way.
 * Initial values also come from the environment (GEAR_COLLECT_IMPL=lsu|tma,
 * GEAR_COLLECT_CHUNK, GEAR_TMA_CHUNK, GEAR_COLLECT_HOST_LSU).  INVALID_ARG for an unknown key or
 * value. */
gear_status gear_table_set_tuning(gear_table* t, const char* key, int64_t value);

/* Read back this rank's slot state (device -> host, synchronous), for tests
 * and checkpoints: keys u64[R*C_s], seq u64[R*C_s], gen u32[R*C_s]; any
 * pointer may be NULL. */
gear_status gear_read_state(gear_table* t, uint64_t* key, uint64_t* seq, uint32_t* gen);

/* Diagnostics (tests): the CDF the last gear_sample built, as this rank's R
 * flat per-shard inclusive prefix sums cdf[ls*C_s + i] = sum of the keys
 * (UNIFORM: of [key > 0]) of local shard ls up to slot i,
 * whichever layout (cdf_levels) holds it; host u64[R*C_s], synchronous.
 * STATE before the first sample. */
gear_status gear_read_cdf(gear_table* t, uint64_t* cdf);

#ifdef __cplusplus
}
#endif
#endif /* GEAR_H */
