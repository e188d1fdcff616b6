/*
 * gear_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, single-threaded CPU oracle for the GEAR (arXiv 2310.05205)
 * replay hot path: quantised priority update, CDF, Philox draw, inverse-CDF
 * search, uniform/weighted/prioritized sampling with importance weights,
 * FIFO/LIFO/TopK selection (plain and owner-affine), index translation,
 * collection, insertion and the split allocate / commit writer.  The PER
 * exponent (RN(p^alpha), reading Q7) is applied by oracle/__init__.py with
 * mpmath before the priorities reach this code.
 *
 * It treats the W shards as ONE concatenated global table (global id order),
 * which is the plain definition of what the sharded GPU path must reproduce
 * (SURVEY.md §8(c) c.1).  It shares no code, header, table or constant with
 * the CUDA path under paper_2310_05205_b200/ and include/; neither side
 * includes or links the other.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load it.
 *
 * Citations: "PAPER.md:N" is a line of /root/reference/PAPER.md (the paper's
 * LaTeX); "Qn" is the reading of a silent/ambiguous passage listed in
 * DESIGN.md §3 (mirrors SURVEY.md §8(c) c.2).
 */
#ifndef GEAR_ORACLE_H
#define GEAR_ORACLE_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes of the oracle (plain ints; deliberately not shared with gear.h). */
#define GOR_OK 0
#define GOR_BAD_PRIORITY 1
#define GOR_INDEX_RANGE 2
#define GOR_STALE 4
#define GOR_EMPTY 8
#define GOR_INVALID 16
#define GOR_FULL 32

/* Strategies (paper PAPER.md:55 lists FIFO, LIFO, weighted, prioritized;
 * PAPER.md:222 adds uniform). */
#define GOR_FIFO 0
#define GOR_LIFO 1
#define GOR_UNIFORM 2
#define GOR_WEIGHTED 3
#define GOR_PRIORITIZED 4
/* TopK ("GEAR provides FIFO and TopK selection"; reading
 * Q20): the n_ranks*B selectable slots with the largest keys, ties by the
 * smaller global id, in that order. */
#define GOR_TOPK 5

/* Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11 "Parallel random numbers:
 * as easy as 1, 2, 3"); the counter-based RNG of reading Q4, which supplies
 * the "uniformly generated random numbers" of PAPER.md:222. */
void gor_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);

/* q_max = floor((2^62 - 1) / N): every total of N keys stays below 2^62 (Q3). */
uint64_t gor_q_max(uint64_t n_global);

/* Q_F(p) (Q3): returns GOR_OK and writes *q, or GOR_BAD_PRIORITY for NaN,
 * +-inf or negative p (then *q is untouched). */
int gor_quantize(double p, uint32_t frac_bits, uint64_t q_max, uint64_t* q);

/* CDF, "computes a prefix sum array": C[g] = sum_{h<=g} key[h]. */
void gor_cdf(const uint64_t* key, uint64_t n, uint64_t* C);

/* Draw j (Q4): Philox4x32-10(ctr=(j_lo, j_hi, 0, 0), key=(seed_lo, seed_hi)),
 * r = x0 | x1 << 32, u = floor(r * T / 2^64).  Returns u in [0, T). */
uint64_t gor_draw(uint64_t seed, uint64_t j, uint64_t T);

/* Inverse CDF, "binary searching to locate the bins":
 * min{ g : C[g] > u } (half-open bins, Q5).  Counts comparisons in *ncmp
 * (may be NULL) for the k*log N bound of PAPER.md:222. */
uint64_t gor_inverse(const uint64_t* C, uint64_t n, uint64_t u, uint64_t* ncmp);

/* Sample (PAPER.md:216-222 centralized selection; Q1, Q2, Q6, Q8, Q9):
 * global table of n_global = n_shards * shard_cap slots; draws the GLOBAL
 * batch of n_ranks*B and returns rank's slice [rank*B, (rank+1)*B).
 *   key[n_global], seq[n_global] (seq only read for FIFO/LIFO).
 *   out_idx[B]  global ids; out_w[B] IS weights (f32); out_p[B] = q/T.
 * Returns GOR_OK or GOR_EMPTY (nothing selectable / fewer than n_ranks*B for
 * FIFO/LIFO) or GOR_INVALID. */
int gor_sample(int strategy, const uint64_t* key, const uint64_t* seq,
               uint64_t shard_cap, uint32_t n_shards, uint32_t n_ranks, uint32_t rank,
               uint32_t B, uint64_t seed, double beta,
               uint64_t* out_idx, float* out_w, double* out_p);

/* Owner-affine assignment of the same global batch (reading Q19; data
 * locality, "the majority of the trajectories collected by the
 * servers reside in local memory").  The global batch of n_ranks*B entries
 * (draws j = 0.. for UNIFORM/WEIGHTED/PRIORITIZED, merged order for
 * FIFO/LIFO) is computed exactly as gor_sample with one rank; entry j is
 * owned by rank (g_j / shard_cap) / (n_shards / n_ranks).  Rank r keeps its
 * own entries in j order, at most B of them; the entries beyond B of
 * over-full owners form an overflow list in j order, and under-full ranks
 * take consecutive runs of it in rank order (rank r takes
 * max(0, B - count_r) entries after those of ranks < r).  The slice is own
 * entries then overflow entries; IS weights use q_min over that slice. */
int gor_sample_owner_affine(int strategy, const uint64_t* key, const uint64_t* seq,
                            uint64_t shard_cap, uint32_t n_shards, uint32_t n_ranks,
                            uint32_t rank, uint32_t B, uint64_t seed, double beta,
                            uint64_t* out_idx, float* out_w, double* out_p);

/* Priority update, applied as the concatenation of every rank's list in
 * (rank, position) order, so the last writer wins (Q11).  Entries with an
 * out-of-range id, an invalid priority, a never-inserted slot (gen == 0), an
 * allocated but uncommitted one (seq == 0, Q21) or
 * (when gen_in != NULL) a generation mismatch are skipped.  Returns a bitmask
 * of GOR_INDEX_RANGE | GOR_BAD_PRIORITY | GOR_STALE; *n_stale counts stale
 * skips (may be NULL).  p is f64; callers holding f32 widen exactly. */
int gor_update(uint64_t* key, const uint64_t* seq, const uint32_t* gen, uint64_t n_global,
               uint32_t frac_bits, uint32_t n, const uint64_t* idx, const double* p,
               const uint32_t* gen_in, uint64_t* n_stale);

/* Index translation: shard = g / cap, local = g mod cap. */
void gor_translate(uint64_t g, uint64_t shard_cap, uint64_t* shard, uint64_t* local);

/* Collection: out[j] = row(idx[j]) for one column whose
 * global table is `col` with row_bytes per row; rows in request order. */
int gor_collect(const uint8_t* col, uint64_t n_global, uint64_t row_bytes,
                uint32_t n, const uint64_t* idx, uint8_t* out);

/* Insertion into shard s:
 * a free queue per shard seeded 0..cap-1 ascending (*next_free counts the
 * dequeued entries); when it is empty the victim is the committed slot of
 * the shard (seq != 0) with the smallest seq (FIFO removal, removal=0) or the
 * largest (LIFO removal, removal=1).  Then seq[g] = (*seq_ctr)++, gen[g]++,
 * key[g] = Q_F(prio[k]); row bytes are copied by the caller using out_idx.
 * Row by row (allocate + commit each).  Returns GOR_OK, GOR_BAD_PRIORITY or
 * GOR_FULL (no free or committed slot at all); nothing inserted on error. */
int gor_insert(uint64_t* key, uint64_t* seq, uint32_t* gen, uint64_t shard_cap,
               uint64_t n_global, uint32_t shard, uint32_t removal, uint32_t frac_bits,
               uint64_t* next_free, uint64_t* seq_ctr,
               uint32_t n, const double* prio, uint64_t* out_idx);

/* Split writer API (reading Q21): allocate n ongoing slots of
 * shard s (gen += 1, key = seq = 0; all or nothing, GOR_FULL), the caller
 * writes the rows in place, then commit them (seq = (*seq_ctr)++, key =
 * Q_F(prio)).  See gear_oracle.c for the per-entry errors of commit. */
int gor_allocate(uint64_t* key, uint64_t* seq, uint32_t* gen, uint64_t shard_cap,
                 uint32_t shard, uint32_t removal, uint64_t* next_free, uint32_t n,
                 uint64_t* out_idx);
int gor_commit(uint64_t* key, uint64_t* seq, const uint32_t* gen, uint64_t shard_cap,
               uint64_t n_global, uint32_t shard, uint32_t frac_bits, uint64_t* seq_ctr,
               uint32_t n, const uint64_t* idx, const double* prio);

#ifdef __cplusplus
}
#endif
#endif
