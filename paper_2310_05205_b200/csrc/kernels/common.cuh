// common.cuh -- device helpers for the sm_100a kernels of the replay hot path.
#pragma once

#include <cstdint>
#include <type_traits>

#include "../gear_internal.h"
#include "pow_dd.cuh"

namespace gear {

constexpr unsigned kFull = 0xffffffffu;

// Philox4x32-10 (Salmon et al., SC'11): the counter-based generator of the
// draw (gear.h, gear_sample).  10 rounds, Weyl key schedule.
struct U4 {
  uint32_t x, y, z, w;
};

__device__ __forceinline__ U4 philox4x32_10(U4 c, uint32_t k0, uint32_t k1) {
  const uint32_t kM0 = 0xD2511F53u, kM1 = 0xCD9E8D57u;
  const uint32_t kW0 = 0x9E3779B9u, kW1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(kM0, c.x), lo0 = kM0 * c.x;
    const uint32_t hi1 = __umulhi(kM1, c.z), lo1 = kM1 * c.z;
    c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
    k0 += kW0;
    k1 += kW1;
  }
  return c;
}

// Draw j of the global batch: 64 random bits from Philox block j under key seed.
__device__ __forceinline__ uint64_t draw_bits(uint64_t seed, uint64_t j) {
  const U4 x = philox4x32_10(U4{(uint32_t)j, (uint32_t)(j >> 32), 0u, 0u}, (uint32_t)seed,
                             (uint32_t)(seed >> 32));
  return (uint64_t)x.x | ((uint64_t)x.y << 32);
}

// Fixed-point key Q_F(v) (gear.h, gear_update_priorities) of a value already
// raised to the table's alpha.  Returns false for NaN, +-inf or negative v.
// v == 0 is key 0; x = v*2^F is exact, __double2ull_rn rounds half to even,
// x >= 2^62 saturates and the key is clamped to [1, q_max].
__device__ __forceinline__ bool quantize_fixed(double v, const Quant& qz, uint64_t* q) {
  if (!(v >= 0.0) || isinf(v)) return false;  // NaN fails v >= 0
  if (v == 0.0) {
    *q = 0;
    return true;
  }
  const double x = scalbn(v, (int)qz.frac_bits);
  uint64_t r = (x >= 4611686018427387904.0) ? qz.q_max : __double2ull_rn(x);
  r = r < 1 ? 1 : r;
  r = r > qz.q_max ? qz.q_max : r;
  *q = r;
  return true;
}

// The PER exponent (reading Q7): a finite p > 0 becomes RN(p^alpha)
// (pow_dd.cuh); 0 and invalid values pass through to quantize_fixed.
__device__ __forceinline__ double apply_alpha(double p, double alpha) {
  return (p > 0.0 && !isinf(p)) ? pow_rn(p, alpha) : p;
}

// Q_F(p^alpha).
__device__ __forceinline__ bool quantize(double p, const Quant& qz, uint64_t* q) {
  return quantize_fixed(apply_alpha(p, qz.alpha), qz, q);
}

// A key of rank-local slot `local` changed: its CDF tile is stale in both
// buffers.
__device__ __forceinline__ void mark_tile(const TileDirty& d, uint64_t local) {
  const uint64_t ls = local / d.shard_cap;
  const uint64_t i = local - ls * d.shard_cap;
  d.bits[ls * d.tiles_per_shard + i / kCdfTile] = 3u;
}

// Relaxed 64-bit global loads/stores for the look-back status words.
__device__ __forceinline__ uint64_t ld_relaxed_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Streaming 16-byte loads/stores for the collect path (no L1 allocation).
__device__ __forceinline__ int4 ld_stream16(const void* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void st_stream16(void* p, int4 v) {
  asm volatile("st.global.L1::no_allocate.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

__device__ __forceinline__ uint64_t warp_incl_scan_u64(uint64_t v, int lane) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint64_t o = __shfl_up_sync(kFull, v, d);
    if (lane >= d) v += o;
  }
  return v;
}

// Shared-memory address, mbarrier and bulk-copy (TMA) helpers.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

// cp.async.bulk global -> shared of `bytes` (multiple of 16, both ends
// 16-byte aligned), completing on mbarrier `bar` (armed with the bytes).
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes,
                                         uint32_t bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}

// cp.async.bulk shared -> global, tracked by this thread's bulk async-groups.
__device__ __forceinline__ void bulk_s2g(void* dst, uint32_t src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src),
               "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

__device__ __forceinline__ uint64_t warp_min_u64(uint64_t v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    const uint64_t o = __shfl_xor_sync(kFull, v, d);
    v = o < v ? o : v;
  }
  return v;
}

}  // namespace gear
