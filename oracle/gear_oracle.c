/*
 * gear_oracle.c -- TEST INFRASTRUCTURE ONLY (see gear_oracle.h).
 *
 * Plain C11, one thread, no CUDA, no blocking, fusion or reordering beyond
 * the definitions it restates.  Each function cites the passage it follows.
 * Loaded only by tests/, __graft_entry__.smoke() and bench.py's CPU legs.
 */
#include "gear_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ */
/* Philox4x32-10 (Salmon et al., SC'11, Fig. 2 / Random123 philox.h    */
/* reference description): 10 rounds of                                */
/*   (hi0,lo0) = M0*c0, (hi1,lo1) = M1*c2,                              */
/*   c' = (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0),                     */
/* with the Weyl key bump k += (W0, W1) between rounds.                 */
/* ------------------------------------------------------------------ */
void gor_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint32_t k0 = key[0], k1 = key[1];
  for (int round = 0; round < 10; ++round) {
    if (round > 0) {
      k0 += W0;
      k1 += W1;
    }
    uint64_t p0 = (uint64_t)M0 * (uint64_t)c0;
    uint64_t p1 = (uint64_t)M1 * (uint64_t)c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    uint32_t n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* Q3: q_max = floor((2^62 - 1) / N), so sum of N keys < 2^62. */
uint64_t gor_q_max(uint64_t n_global) {
  if (n_global == 0) return 0;
  return (((uint64_t)1 << 62) - 1) / n_global;
}

/* Q3: Q_F(p).  PAPER.md:186 gives priorities with no type; priority 0 means
 * "not selectable".  x = p * 2^F exactly; x >= 2^62 saturates to q_max;
 * otherwise round half to even, written out (floor, fraction, tie -> even);
 * then clamp into [1, q_max] so a positive p never becomes unselectable. */
int gor_quantize(double p, uint32_t frac_bits, uint64_t q_max, uint64_t* q) {
  if (p != p) return GOR_BAD_PRIORITY;          /* NaN */
  if (p < 0.0) return GOR_BAD_PRIORITY;
  if (p == INFINITY) return GOR_BAD_PRIORITY;
  if (p == 0.0) { *q = 0; return GOR_OK; }
  double scale = 1.0;
  for (uint32_t b = 0; b < frac_bits; ++b) scale *= 2.0;   /* 2^F, exact */
  double x = p * scale;                                      /* exact (power of two) */
  const double two62 = 4611686018427387904.0;               /* 2^62 */
  uint64_t r;
  if (x >= two62) {
    r = q_max;
  } else {
    double fl = floor(x);
    double frac = x - fl;                                    /* exact */
    r = (uint64_t)fl;
    if (frac > 0.5) r += 1;
    else if (frac == 0.5 && (r & 1u)) r += 1;                /* tie -> even */
  }
  if (r < 1) r = 1;
  if (r > q_max) r = q_max;
  *q = r;
  return GOR_OK;
}

/* PAPER.md:222 "prefix sum array": inclusive running sum, left to right. */
void gor_cdf(const uint64_t* key, uint64_t n, uint64_t* C) {
  uint64_t run = 0;
  for (uint64_t g = 0; g < n; ++g) {
    run += key[g];
    C[g] = run;
  }
}

/* Q4: r from Philox block j under key = seed; u = floor(r*T / 2^64). */
uint64_t gor_draw(uint64_t seed, uint64_t j, uint64_t T) {
  uint32_t ctr[4] = {(uint32_t)j, (uint32_t)(j >> 32), 0u, 0u};
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t x[4];
  gor_philox4x32_10(ctr, key, x);
  uint64_t r = (uint64_t)x[0] | ((uint64_t)x[1] << 32);
  unsigned __int128 prod = (unsigned __int128)r * (unsigned __int128)T;
  return (uint64_t)(prod >> 64);
}

/* PAPER.md:222 "binary searching to locate the bins": textbook lower-bound
 * style binary search for the first C[g] > u (Q5). */
uint64_t gor_inverse(const uint64_t* C, uint64_t n, uint64_t u, uint64_t* ncmp) {
  uint64_t lo = 0, hi = n;   /* answer in [lo, hi) */
  uint64_t cmps = 0;
  while (lo < hi) {
    uint64_t mid = lo + (hi - lo) / 2;
    ++cmps;
    if (C[mid] > u) hi = mid;
    else lo = mid + 1;
  }
  if (ncmp) *ncmp += cmps;
  return lo;
}

/* ---- FIFO / LIFO ordering (Q8) ---- */
typedef struct {
  uint64_t seq;
  uint64_t shard;
  uint64_t g;
} gor_cand;

static int gor_cand_cmp(const void* a, const void* b) {
  const gor_cand* x = (const gor_cand*)a;
  const gor_cand* y = (const gor_cand*)b;
  if (x->seq != y->seq) return x->seq < y->seq ? -1 : 1;
  if (x->shard != y->shard) return x->shard < y->shard ? -1 : 1;
  if (x->g != y->g) return x->g < y->g ? -1 : 1;
  return 0;
}

int gor_sample(int strategy, const uint64_t* key, const uint64_t* seq,
               uint64_t shard_cap, uint32_t n_shards, uint32_t n_ranks, uint32_t rank,
               uint32_t B, uint64_t seed, double beta,
               uint64_t* out_idx, float* out_w, double* out_p) {
  if (n_shards == 0 || n_ranks == 0 || rank >= n_ranks || shard_cap == 0) return GOR_INVALID;
  uint64_t n = shard_cap * (uint64_t)n_shards;
  uint64_t K = (uint64_t)n_ranks * (uint64_t)B;   /* global batch (Q9) */
  if (B == 0) return GOR_OK;

  if (strategy == GOR_FIFO || strategy == GOR_LIFO) {
    /* Sort every selectable slot by (seq, shard); FIFO takes the first K
     * ascending, LIFO the last K descending; rank keeps [rank*B, rank*B+B). */
    gor_cand* c = (gor_cand*)malloc(sizeof(gor_cand) * (n ? n : 1));
    uint64_t m = 0;
    for (uint64_t g = 0; g < n; ++g) {
      if (key[g] > 0) {
        c[m].seq = seq[g];
        c[m].shard = g / shard_cap;
        c[m].g = g;
        ++m;
      }
    }
    if (m < K) { free(c); return GOR_EMPTY; }
    qsort(c, m, sizeof(gor_cand), gor_cand_cmp);
    for (uint32_t b = 0; b < B; ++b) {
      uint64_t pos = (uint64_t)rank * B + b;
      uint64_t at = (strategy == GOR_FIFO) ? pos : (m - 1 - pos);
      out_idx[b] = c[at].g;
      if (out_w) out_w[b] = 1.0f;
      if (out_p) out_p[b] = 1.0;
    }
    free(c);
    return GOR_OK;
  }

  if (strategy == GOR_TOPK) {
    /* Q20: sort every selectable slot by (key descending, global id
     * ascending) and take the first K; rank keeps [rank*B, rank*B+B).  The
     * comparator negates the key through the `seq` field: sort ascending by
     * (-key, g) written as (UINT64_MAX - key, g). */
    gor_cand* c = (gor_cand*)malloc(sizeof(gor_cand) * (n ? n : 1));
    uint64_t m = 0;
    for (uint64_t g = 0; g < n; ++g) {
      if (key[g] > 0) {
        c[m].seq = UINT64_MAX - key[g];
        c[m].shard = 0;      /* ties go by global id alone */
        c[m].g = g;
        ++m;
      }
    }
    if (m < K) { free(c); return GOR_EMPTY; }
    qsort(c, m, sizeof(gor_cand), gor_cand_cmp);
    for (uint32_t b = 0; b < B; ++b) {
      out_idx[b] = c[(uint64_t)rank * B + b].g;
      if (out_w) out_w[b] = 1.0f;
      if (out_p) out_p[b] = 1.0;
    }
    free(c);
    return GOR_OK;
  }

  if (strategy != GOR_UNIFORM && strategy != GOR_WEIGHTED && strategy != GOR_PRIORITIZED)
    return GOR_INVALID;

  /* Weights: the keys themselves, or the indicator [key>0] for UNIFORM (Q2). */
  uint64_t* wts = (uint64_t*)malloc(sizeof(uint64_t) * (n ? n : 1));
  uint64_t* C = (uint64_t*)malloc(sizeof(uint64_t) * (n ? n : 1));
  for (uint64_t g = 0; g < n; ++g)
    wts[g] = (strategy == GOR_UNIFORM) ? (key[g] > 0 ? 1u : 0u) : key[g];
  gor_cdf(wts, n, C);
  uint64_t T = n ? C[n - 1] : 0;
  if (T == 0) { free(wts); free(C); return GOR_EMPTY; }

  uint64_t* q = (uint64_t*)malloc(sizeof(uint64_t) * B);
  for (uint32_t b = 0; b < B; ++b) {
    uint64_t j = (uint64_t)rank * B + b;        /* global draw number */
    uint64_t u = gor_draw(seed, j, T);
    uint64_t g = gor_inverse(C, n, u, NULL);
    out_idx[b] = g;
    q[b] = wts[g];
  }
  /* Q6: PER weights w = (N*P)^-beta / max w over the rank's slice,
   * which is (q_min / q)^beta; f64 arithmetic, stored as f32. */
  uint64_t qmin = q[0];
  for (uint32_t b = 1; b < B; ++b) if (q[b] < qmin) qmin = q[b];
  for (uint32_t b = 0; b < B; ++b) {
    if (out_w) {
      if (strategy == GOR_PRIORITIZED)
        out_w[b] = (float)pow((double)qmin / (double)q[b], beta);
      else
        out_w[b] = 1.0f;
    }
    if (out_p) out_p[b] = (double)q[b] / (double)T;
  }
  free(q);
  free(wts);
  free(C);
  return GOR_OK;
}

/* Q19: owner-affine assignment of the global batch (see gear_oracle.h). */
int gor_sample_owner_affine(int strategy, const uint64_t* key, const uint64_t* seq,
                            uint64_t shard_cap, uint32_t n_shards, uint32_t n_ranks,
                            uint32_t rank, uint32_t B, uint64_t seed, double beta,
                            uint64_t* out_idx, float* out_w, double* out_p) {
  if (n_ranks == 0 || rank >= n_ranks || n_shards % n_ranks) return GOR_INVALID;
  if (B == 0) return GOR_OK;
  uint64_t K = (uint64_t)n_ranks * B;
  uint64_t* g = (uint64_t*)malloc(sizeof(uint64_t) * K);
  double* p = (double*)malloc(sizeof(double) * K);
  /* the global batch, in global order */
  int st = gor_sample(strategy, key, seq, shard_cap, n_shards, 1, 0, (uint32_t)K, seed, beta,
                      g, NULL, p);
  if (st != GOR_OK) { free(g); free(p); return st; }
  uint32_t R = n_shards / n_ranks;
  uint64_t* count = (uint64_t*)calloc(n_ranks, sizeof(uint64_t));
  for (uint64_t j = 0; j < K; ++j) count[(g[j] / shard_cap) / R] += 1;
  uint64_t offset = 0;           /* overflow entries taken by ranks before `rank` */
  for (uint32_t r = 0; r < rank; ++r) offset += count[r] < B ? B - count[r] : 0;
  uint64_t need = count[rank] < B ? B - count[rank] : 0;
  uint64_t* seen = (uint64_t*)calloc(n_ranks, sizeof(uint64_t));
  uint64_t nown = 0, nover = 0, ov = 0;
  uint64_t* own = (uint64_t*)malloc(sizeof(uint64_t) * B);
  uint64_t* over = (uint64_t*)malloc(sizeof(uint64_t) * B);
  for (uint64_t j = 0; j < K; ++j) {
    uint32_t o = (uint32_t)((g[j] / shard_cap) / R);
    uint64_t pos = seen[o]++;    /* position of j among its owner's entries */
    if (pos < B) {
      if (o == rank) own[nown++] = j;
    } else {
      if (ov >= offset && ov < offset + need) over[nover++] = j;
      ++ov;
    }
  }
  uint32_t b = 0;
  for (uint64_t k = 0; k < nown; ++k, ++b) out_idx[b] = g[own[k]], out_p ? out_p[b] = p[own[k]] : 0;
  for (uint64_t k = 0; k < nover; ++k, ++b) out_idx[b] = g[over[k]], out_p ? out_p[b] = p[over[k]] : 0;
  if (out_w) {
    uint64_t qmin = UINT64_MAX;
    for (uint32_t k = 0; k < B; ++k) if (key[out_idx[k]] < qmin) qmin = key[out_idx[k]];
    for (uint32_t k = 0; k < B; ++k)
      out_w[k] = strategy == GOR_PRIORITIZED ? (float)pow((double)qmin / (double)key[out_idx[k]], beta)
                                             : 1.0f;
  }
  free(g); free(p); free(count); free(seen); free(own); free(over);
  return GOR_OK;
}

/* Q11: apply the list in order; the last valid writer of a slot wins. */
int gor_update(uint64_t* key, const uint64_t* seq, const uint32_t* gen, uint64_t n_global,
               uint32_t frac_bits, uint32_t n, const uint64_t* idx, const double* p,
               const uint32_t* gen_in, uint64_t* n_stale) {
  int err = GOR_OK;
  uint64_t qmax = gor_q_max(n_global);
  for (uint32_t k = 0; k < n; ++k) {
    uint64_t g = idx[k];
    if (g == UINT64_MAX) continue;                  /* padding entry */
    if (g >= n_global) { err |= GOR_INDEX_RANGE; continue; }
    uint64_t q;
    if (gor_quantize(p[k], frac_bits, qmax, &q) != GOR_OK) { err |= GOR_BAD_PRIORITY; continue; }
    /* never inserted (gen 0) or allocated but not committed (seq 0, Q21) */
    if (gen[g] == 0 || seq[g] == 0 || (gen_in && gen_in[k] != gen[g])) {
      err |= GOR_STALE;
      if (n_stale) ++*n_stale;
      continue;
    }
    key[g] = q;
  }
  return err;
}

/* PAPER.md:243 "dividing the index by the capacity". */
void gor_translate(uint64_t g, uint64_t shard_cap, uint64_t* shard, uint64_t* local) {
  *shard = g / shard_cap;
  *local = g % shard_cap;
}

/* rows concatenated in request order. */
int gor_collect(const uint8_t* col, uint64_t n_global, uint64_t row_bytes,
                uint32_t n, const uint64_t* idx, uint8_t* out) {
  for (uint32_t j = 0; j < n; ++j) {
    if (idx[j] >= n_global) return GOR_INDEX_RANGE;
    memcpy(out + (uint64_t)j * row_bytes, col + idx[j] * row_bytes, row_bytes);
  }
  return GOR_OK;
}

/* The committed slot of shard [base, base+cap) a full free queue evicts:
 * smallest seq (FIFO removal) or largest (LIFO removal) among committed slots
 * (seq != 0; ongoing slots -- allocated, not committed -- have seq 0).
 * UINT64_MAX if none. */
static uint64_t victim(const uint64_t* seq, uint64_t base, uint64_t cap, uint32_t removal) {
  uint64_t best = UINT64_MAX;
  for (uint64_t i = 0; i < cap; ++i) {
    uint64_t h = base + i;
    if (seq[h] == 0) continue;
    if (best == UINT64_MAX || (removal == 0 ? (seq[h] < seq[best]) : (seq[h] > seq[best])))
      best = h;
  }
  return best;
}

/* Free entries plus committed slots of a shard: what n allocations can use. */
static uint64_t available(const uint64_t* seq, uint64_t base, uint64_t cap, uint64_t next_free) {
  uint64_t c = cap - next_free;
  for (uint64_t i = 0; i < cap; ++i) c += seq[base + i] != 0;
  return c;
}

/* PAPER.md:186 single free queue; PAPER.md:193 allocate/commit;
 * PAPER.md:195 victim by removal strategy when no index is free.  Each row is
 * allocated and committed before the next one (a later row can evict an
 * earlier one of the same call). */
int gor_insert(uint64_t* key, uint64_t* seq, uint32_t* gen, uint64_t shard_cap,
               uint64_t n_global, uint32_t shard, uint32_t removal, uint32_t frac_bits,
               uint64_t* next_free, uint64_t* seq_ctr,
               uint32_t n, const double* prio, uint64_t* out_idx) {
  uint64_t qmax = gor_q_max(n_global);
  uint64_t base = (uint64_t)shard * shard_cap;
  for (uint32_t k = 0; k < n; ++k) {
    uint64_t q;
    if (gor_quantize(prio[k], frac_bits, qmax, &q) != GOR_OK) return GOR_BAD_PRIORITY;
  }
  if (n > 0 && available(seq, base, shard_cap, *next_free) == 0) return GOR_FULL;
  for (uint32_t k = 0; k < n; ++k) {
    uint64_t g;
    if (*next_free < shard_cap) {
      g = base + *next_free;                 /* dequeue from the free queue */
      *next_free += 1;
    } else {
      g = victim(seq, base, shard_cap, removal);
    }
    uint64_t q;
    gor_quantize(prio[k], frac_bits, qmax, &q);
    seq[g] = *seq_ctr;
    *seq_ctr += 1;
    gen[g] += 1;
    key[g] = q;
    out_idx[k] = g;
  }
  return GOR_OK;
}

/* PAPER.md:193 steps 3-4 ("requests a free index from the block allocator"),
 * reading Q21: n indices of shard s, each from the free queue or, when it is
 * empty, by evicting the victim of the removal strategy.  An
 * allocated slot is ongoing: gen += 1, key = 0 and seq = 0 (not selectable,
 * not a victim, updates to it are stale) until it is committed.  All or
 * nothing: GOR_FULL (and nothing allocated) when fewer than n free or
 * committed slots exist. */
int gor_allocate(uint64_t* key, uint64_t* seq, uint32_t* gen, uint64_t shard_cap,
                 uint32_t shard, uint32_t removal, uint64_t* next_free, uint32_t n,
                 uint64_t* out_idx) {
  uint64_t base = (uint64_t)shard * shard_cap;
  if (available(seq, base, shard_cap, *next_free) < n) {
    for (uint32_t k = 0; k < n; ++k) out_idx[k] = UINT64_MAX;
    return GOR_FULL;
  }
  for (uint32_t k = 0; k < n; ++k) {
    uint64_t g;
    if (*next_free < shard_cap) {
      g = base + *next_free;
      *next_free += 1;
    } else {
      g = victim(seq, base, shard_cap, removal);
    }
    gen[g] += 1;
    key[g] = 0;
    seq[g] = 0;
    out_idx[k] = g;
  }
  return GOR_OK;
}

/* PAPER.md:193 step 5 ("commits the buffer, triggering an update in the
 * Status Table ... designates the index as available for selection"): in
 * order, each ongoing id of shard s gets seq = (*seq_ctr)++ and key =
 * Q_F(prio[k]).  An id outside the shard is skipped with GOR_INDEX_RANGE, one
 * that is not ongoing (never allocated, already committed -- e.g. the second
 * copy of a duplicate) with GOR_STALE, an invalid priority with
 * GOR_BAD_PRIORITY (the slot stays ongoing).  Returns the bitmask. */
int gor_commit(uint64_t* key, uint64_t* seq, const uint32_t* gen, uint64_t shard_cap,
               uint64_t n_global, uint32_t shard, uint32_t frac_bits, uint64_t* seq_ctr,
               uint32_t n, const uint64_t* idx, const double* prio) {
  int err = GOR_OK;
  uint64_t qmax = gor_q_max(n_global);
  uint64_t base = (uint64_t)shard * shard_cap;
  for (uint32_t k = 0; k < n; ++k) {
    uint64_t g = idx[k];
    if (g < base || g >= base + shard_cap) { err |= GOR_INDEX_RANGE; continue; }
    if (gen[g] == 0 || seq[g] != 0) { err |= GOR_STALE; continue; }
    uint64_t q;
    if (gor_quantize(prio[k], frac_bits, qmax, &q) != GOR_OK) { err |= GOR_BAD_PRIORITY; continue; }
    seq[g] = *seq_ctr;
    *seq_ctr += 1;
    key[g] = q;
  }
  return err;
}
