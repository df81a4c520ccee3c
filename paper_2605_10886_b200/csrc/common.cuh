// common.cuh — sm_100a device helpers shared by the LoKA kernels (PTX wrappers for FP8 casts,
// mbarrier, TMA, tcgen05/TMEM, clusters).  Product code only; nothing here is used by oracle/.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include "../../include/loka.h"

#define LOKA_DEVINL __device__ __forceinline__

namespace loka {

// ------------------------------------------------------------------------------------------
// FP8 constants (OCP E4M3FN / E5M2; D4)
// ------------------------------------------------------------------------------------------
template <int FMT> struct Fp8Traits;
template <> struct Fp8Traits<LOKA_E4M3> {
  static constexpr float kMax = 448.0f;
  static constexpr int kMaxExp = 8;  // 448 = 1.75 * 2^8
};
template <> struct Fp8Traits<LOKA_E5M2> {
  static constexpr float kMax = 57344.0f;
  static constexpr int kMaxExp = 15;  // 57344 = 1.75 * 2^15
};

// Two FP32 -> two FP8 codes, saturating RNE (F2FP.SATFINITE).  lo goes to the low byte.
template <int FMT> LOKA_DEVINL uint32_t cvt_fp8x2(float lo, float hi) {
  uint16_t r;
  if constexpr (FMT == LOKA_E4M3)
    asm("{ cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2; }" : "=h"(r) : "f"(hi), "f"(lo));
  else
    asm("{ cvt.rn.satfinite.e5m2x2.f32 %0, %1, %2; }" : "=h"(r) : "f"(hi), "f"(lo));
  return (uint32_t)r;
}
// Four codes in one register (a in the low byte): the two pair conversions are packed with one
// mov.b32 {lo, hi}, which ptxas folds into the second F2FP's MERGE_C operand (no shift / OR).
template <int FMT> LOKA_DEVINL uint32_t cvt_fp8x4(float a, float b, float c, float d) {
  uint32_t r;
  if constexpr (FMT == LOKA_E4M3)
    asm("{ .reg .b16 lo, hi;\n cvt.rn.satfinite.e4m3x2.f32 lo, %2, %1;\n cvt.rn.satfinite.e4m3x2.f32 hi, %4, %3;\n"
        " mov.b32 %0, {lo, hi}; }"
        : "=r"(r) : "f"(a), "f"(b), "f"(c), "f"(d));
  else
    asm("{ .reg .b16 lo, hi;\n cvt.rn.satfinite.e5m2x2.f32 lo, %2, %1;\n cvt.rn.satfinite.e5m2x2.f32 hi, %4, %3;\n"
        " mov.b32 %0, {lo, hi}; }"
        : "=r"(r) : "f"(a), "f"(b), "f"(c), "f"(d));
  return r;
}

// Exact IEEE scale computation for one granule (D1/D2/D7).  amax >= 0, finite.
template <int FMT, int SCALE_FMT>
LOKA_DEVINL void scales_from_amax(float amax, float& s, float& r) {
  constexpr float kMax = Fp8Traits<FMT>::kMax;
  if (!(amax > 0.0f)) { s = 1.0f; r = 1.0f; return; }
  if constexpr (SCALE_FMT == LOKA_SCALE_F32) {
    s = __fdiv_rn(amax, kMax);
    // D1b: max/amax overflows FP32 for amax < max/FLT_MAX; the reciprocal is then FLT_MAX
    // (fminf(+Inf, FLT_MAX)), so x*r stays finite and zeros keep their sign (no 0*Inf NaN)
    r = fminf(__fdiv_rn(kMax, amax), 3.402823466e38f);
  } else {
    // s = 2^e, e = smallest integer >= -127 with amax <= kMax * 2^e.  With amax = m * 2^ea
    // (m in [1,2)) and kMax = 1.75 * 2^kMaxExp:  e = ea - kMaxExp + (m > 1.75).
    uint32_t b = __float_as_uint(amax);
    int ef = (int)(b >> 23);
    uint32_t mf = b & 0x7FFFFFu;
    int e;
    if (ef == 0) {
      e = -127;  // subnormal amax < 2^-126: amax/kMax < 2^-134
    } else {
      e = (ef - 127) - Fp8Traits<FMT>::kMaxExp + (mf > 0x600000u ? 1 : 0);
      if (e < -127) e = -127;
    }
    s = (e >= -126) ? __uint_as_float((uint32_t)(e + 127) << 23) : __uint_as_float(0x00400000u);
    r = __uint_as_float((uint32_t)(127 - e) << 23);  // 2^-e, e in [-127, 127]: exponent 0..254
  }
}

// ------------------------------------------------------------------------------------------
// misc
// ------------------------------------------------------------------------------------------
LOKA_DEVINL int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }
LOKA_DEVINL uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

LOKA_DEVINL float bf16lo_to_f32(uint32_t w) { return __uint_as_float(w << 16); }
LOKA_DEVINL float bf16hi_to_f32(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }

LOKA_DEVINL uint32_t warp_max_u32(uint32_t v) {
  return __reduce_max_sync(0xFFFFFFFFu, v);
}

// Packed FP32x2 arithmetic (SASS FMUL2 / FFMA2 / FADD2), IEEE round-to-nearest per lane.
LOKA_DEVINL float2 fmul2(float2 a, float2 b) {
  float2 d;
  asm("{.reg .b64 ra, rb, rd;\n mov.b64 ra, {%2,%3};\n mov.b64 rb, {%4,%5};\n mul.rn.f32x2 rd, ra, rb;\n"
      " mov.b64 {%0,%1}, rd;}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
LOKA_DEVINL float2 ffma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{.reg .b64 ra, rb, rc, rd;\n mov.b64 ra, {%2,%3};\n mov.b64 rb, {%4,%5};\n mov.b64 rc, {%6,%7};\n"
      " fma.rn.f32x2 rd, ra, rb, rc;\n mov.b64 {%0,%1}, rd;}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}
LOKA_DEVINL float2 fadd2(float2 a, float2 b) {
  float2 d;
  asm("{.reg .b64 ra, rb, rd;\n mov.b64 ra, {%2,%3};\n mov.b64 rb, {%4,%5};\n add.rn.f32x2 rd, ra, rb;\n"
      " mov.b64 {%0,%1}, rd;}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
// 3-input min/max (SASS FMNMX3)
LOKA_DEVINL float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
LOKA_DEVINL float fmin3(float a, float b, float c) {
  float d;
  asm("min.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
LOKA_DEVINL float4 lds_f4(uint32_t saddr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(saddr));
  return v;
}
// NEXT-4: fold a thread's max |v| into a device float by warp reduction + one atomicMax of the
// IEEE bit pattern (non-negative floats order like their bits; NaN > Inf > finite).  Whole warp.
LOKA_DEVINL void warp_amax_to(float* dst, float m) {
  uint32_t b = __float_as_uint(m) & 0x7FFFFFFFu;
  b = __reduce_max_sync(0xFFFFFFFFu, b);
  if ((threadIdx.x & 31) == 0 && b) atomicMax(reinterpret_cast<unsigned int*>(dst), b);
}
// value as stored in the output dtype (bf16 rounding) for the producer amax
LOKA_DEVINL float stored_bf16(float v) { return __bfloat162float(__float2bfloat16_rn(v)); }
// named barrier among `n` threads (id 1..15; id 0 is __syncthreads)
LOKA_DEVINL void named_bar_sync(uint32_t id, uint32_t n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
// programmatic dependent launch (PDL)
LOKA_DEVINL void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
LOKA_DEVINL void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ------------------------------------------------------------------------------------------
// mbarrier
// ------------------------------------------------------------------------------------------
LOKA_DEVINL void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
LOKA_DEVINL void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
LOKA_DEVINL void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
LOKA_DEVINL void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
LOKA_DEVINL bool mbar_try_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
LOKA_DEVINL uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Watchdog state (one copy per translation unit; linear.cu reads its own): a wait that exceeds kHangNs records where it hung,
// raises g_loka_abort so every other wait returns at once, and returns — the kernel then
// finishes with garbage output instead of hanging the GPU (read via loka_debug_hang_info).
static __device__ unsigned long long g_loka_hang[4];  // per translation unit
static __device__ int g_loka_abort;
constexpr uint64_t kHangNs = 4000000000ull;

LOKA_DEVINL void mbar_wait(uint64_t* bar, uint32_t parity, int tag = 0) {
  const uint32_t a = smem_u32(bar);
  if (mbar_try_wait(a, parity)) return;
  uint64_t t0 = 0;
  uint32_t spins = 0;
  while (!mbar_try_wait(a, parity)) {
    if ((++spins & 1023u) != 0) continue;  // the watchdog costs nothing on the normal path
    const uint64_t t = globaltimer_ns();
    if (t0 == 0) t0 = t;
    if (*reinterpret_cast<volatile int*>(&g_loka_abort)) return;
    if (t - t0 > kHangNs) {
      if (atomicAdd(&g_loka_hang[0], 1ull) == 0) {
        g_loka_hang[1] = (unsigned long long)tag;
        g_loka_hang[2] = (unsigned long long)(blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z));
        g_loka_hang[3] = (unsigned long long)threadIdx.x | ((unsigned long long)parity << 32);
      }
      atomicExch(&g_loka_abort, 1);
      return;
    }
  }
}

// ------------------------------------------------------------------------------------------
// TMA
// ------------------------------------------------------------------------------------------
LOKA_DEVINL void tma_prefetch_desc(const CUtensorMap* m) {
  asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)m) : "memory");
}
LOKA_DEVINL void tma_load_2d(void* dst, const CUtensorMap* m, uint64_t* bar, int32_t c0, int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"((uint64_t)m), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// TMA store (smem -> global), bulk-group completion
LOKA_DEVINL void tma_store_2d(const CUtensorMap* m, const void* src, int32_t c0, int32_t c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"((uint64_t)m),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
LOKA_DEVINL void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
LOKA_DEVINL void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
LOKA_DEVINL void bulk_wait_read_le1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
// make generic-proxy shared-memory writes visible to the async (TMA) proxy
LOKA_DEVINL void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
LOKA_DEVINL void sts_u4(uint32_t saddr, uint4 v) {
  asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(saddr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

// ------------------------------------------------------------------------------------------
// tcgen05 / TMEM
// ------------------------------------------------------------------------------------------
template <uint32_t kCols>
LOKA_DEVINL void tmem_alloc(uint32_t* dst_smem) {  // whole warp
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "n"(kCols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
template <uint32_t kCols>
LOKA_DEVINL void tmem_dealloc(uint32_t taddr) {  // whole warp
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols));
}
LOKA_DEVINL void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
LOKA_DEVINL void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// SMEM matrix descriptor, K-major operand, 128-byte swizzle: rows of 128 B, 8-row groups 1024 B
// apart (SBO), LBO unused (16 B), version 1 (sm_100), layout type 2 = SWIZZLE_128B.
LOKA_DEVINL uint64_t smem_desc_kmajor_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;                 // LBO = 16 B (ignored for swizzled K-major)
  d |= (uint64_t)(1024u >> 4) << 32;       // SBO = 1024 B
  d |= (uint64_t)1u << 46;                 // version
  d |= (uint64_t)2u << 61;                 // SWIZZLE_128B
  return d;
}

// Instruction descriptor for kind::f8f6f4, FP32 accumulate, both operands K-major.
LOKA_DEVINL uint32_t idesc_f8f6f4(int a_fmt, int b_fmt, uint32_t M, uint32_t N) {
  uint32_t d = 0;
  d |= 1u << 4;                     // D format F32
  d |= (uint32_t)a_fmt << 7;        // 0 = E4M3, 1 = E5M2
  d |= (uint32_t)b_fmt << 10;
  d |= (N >> 3) << 17;
  d |= (M >> 4) << 24;
  return d;
}

LOKA_DEVINL void mma_f8f6f4(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate)
      : "memory");
}
// ---- block-scaled (MX) MMA: kind::mxf8f6f4.block_scale, UE8M0 scale per 32 K, scales in TMEM ----
// Instruction descriptor (block-scaled form): b_sf_id [4,6), a/b format [7,10)/[10,13), N>>3
// [17,23), scale format [23] (1 = UE8M0), M>>4 [24,29), a_sf_id [29,31).
LOKA_DEVINL uint32_t idesc_mxf8f6f4(int a_fmt, int b_fmt, uint32_t M, uint32_t N) {
  uint32_t d = 0;
  d |= (uint32_t)a_fmt << 7;
  d |= (uint32_t)b_fmt << 10;
  d |= (N >> 3) << 17;
  d |= 1u << 23;  // UE8M0 scales
  d |= (M >> 4) << 24;
  return d;
}
// sf_id k selects byte k of the 32-bit TMEM scale word (the k-th 32-wide K block of a 128-K
// group); it is carried both in the descriptor and in the top two bits of the TMEM addresses.
LOKA_DEVINL void mma_mxf8f6f4(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t tsfa, uint32_t tsfb,
                              uint32_t k, uint32_t accumulate) {
  const uint32_t id = idesc | (k << 29) | (k << 4);
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %6, 0;\n"
      " tcgen05.mma.cta_group::1.kind::mxf8f6f4.block_scale [%0], %1, %2, %3, [%4], [%5], p;\n}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(id), "r"(tsfa | (k << 30)), "r"(tsfb | (k << 30)), "r"(accumulate)
      : "memory");
}
// NVFP4 (kind::mxf4nvf4, E2M1 x E2M1, UE4M3 scales, K = 64 per instruction)
LOKA_DEVINL uint32_t idesc_nvf4(uint32_t M, uint32_t N) {
  uint32_t d = 0;
  d |= 1u << 7;   // A: E2M1
  d |= 1u << 10;  // B: E2M1
  d |= (N >> 3) << 17;
  // bit 23 = 0: UE4M3 scales; bit 31 = 0: K = 64
  d |= (M >> 4) << 24;
  return d;
}
// scale_vec::4X: four 16-element scales per row per MMA = one full 32-bit TMEM column per row
LOKA_DEVINL void mma_nvf4(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t tsfa, uint32_t tsfb,
                          uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %6, 0;\n"
      " tcgen05.mma.cta_group::1.kind::mxf4nvf4.block_scale.scale_vec::4X [%0], %1, %2, %3, [%4], [%5], p;\n}" ::"r"(
          tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(tsfa), "r"(tsfb), "r"(accumulate)
      : "memory");
}
// smem -> TMEM copy of one 32 x 16 B scale-factor atom, broadcast to the four 32-lane groups
// (lane i of every group gets row i: 4 TMEM columns).  Source: no-swizzle K-major descriptor,
// 8-row core matrices 128 B apart (SBO).
LOKA_DEVINL void utccp_32x128b_warpx4(uint32_t tmem_dst, uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)(128u >> 4) << 16;  // LBO (single 16 B column: unused)
  d |= (uint64_t)(128u >> 4) << 32;  // SBO = 128 B
  d |= (uint64_t)1u << 46;           // version; layout type 0 = no swizzle
  asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;" ::"r"(tmem_dst), "l"(d) : "memory");
}
// ---- CTA pair (cta_group::2): one MMA spans the two SMs of a 2-CTA cluster ----
template <uint32_t kCols>
LOKA_DEVINL void tmem_alloc_cg2(uint32_t* dst_smem) {  // one warp in EACH CTA of the pair (same warp id)
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "n"(kCols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
}
template <uint32_t kCols>
LOKA_DEVINL void tmem_dealloc_cg2(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols));
}
// D[256 x N] (+)= A[256 x 32] . B[N x 32]^T: rows 0-127 of A / D and B rows 0..N/2-1 live in the
// leader CTA, the rest at the same shared-memory / TMEM offsets in the peer.  Leader issues.
LOKA_DEVINL void mma_f8f6f4_cg2(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::2.kind::f8f6f4 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate)
      : "memory");
}
// BF16 x BF16 -> FP32 pair MMA (kind::f16, K = 16 per instruction = 32 bytes of a 128-byte row)
LOKA_DEVINL uint32_t idesc_bf16(uint32_t M, uint32_t N) {
  uint32_t d = 0;
  d |= 1u << 4;   // D format F32
  d |= 1u << 7;   // A format BF16
  d |= 1u << 10;  // B format BF16
  d |= (N >> 3) << 17;
  d |= (M >> 4) << 24;
  return d;
}
LOKA_DEVINL void mma_bf16_cg2(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate)
      : "memory");
}
// block-scaled (UE8M0 per 32-K) variant of the pair MMA; scale factors in each CTA's TMEM
LOKA_DEVINL void mma_mxf8f6f4_cg2(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t tsfa,
                                  uint32_t tsfb, uint32_t k, uint32_t accumulate) {
  const uint32_t id = idesc | (k << 29) | (k << 4);
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %6, 0;\n"
      " tcgen05.mma.cta_group::2.kind::mxf8f6f4.block_scale [%0], %1, %2, %3, [%4], [%5], p;\n}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(id), "r"(tsfa | (k << 30)), "r"(tsfb | (k << 30)), "r"(accumulate)
      : "memory");
}
LOKA_DEVINL void mma_nvf4_cg2(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t tsfa, uint32_t tsfb,
                              uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %6, 0;\n"
      " tcgen05.mma.cta_group::2.kind::mxf4nvf4.block_scale.scale_vec::4X [%0], %1, %2, %3, [%4], [%5], p;\n}" ::"r"(
          tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(tsfa), "r"(tsfb), "r"(accumulate)
      : "memory");
}
// smem -> TMEM scale-factor atom copy in both CTAs of the pair (each from its own smem)
LOKA_DEVINL void utccp_32x128b_warpx4_cg2(uint32_t tmem_dst, uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)(128u >> 4) << 16;
  d |= (uint64_t)(128u >> 4) << 32;
  d |= (uint64_t)1u << 46;
  asm volatile("tcgen05.cp.cta_group::2.32x128b.warpx4 [%0], %1;" ::"r"(tmem_dst), "l"(d) : "memory");
}
// arrive on `bar` (same offset) in every CTA of cta_mask once the issued MMAs complete
LOKA_DEVINL void mma_commit_cg2_mc(uint64_t* bar, uint16_t cta_mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(cta_mask)
      : "memory");
}
// TMA 2-D load into this CTA's shared memory whose completion is counted on the LEADER's
// barrier (bar_cluster: a shared::cluster address, e.g. mapa(bar, 0)).
LOKA_DEVINL void tma_load_2d_cg2(void* dst, const CUtensorMap* m, uint32_t bar_cluster, int32_t c0, int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4}], [%2];" ::"r"(smem_u32(dst)),
      "l"((uint64_t)m), "r"(bar_cluster), "r"(c0), "r"(c1)
      : "memory");
}
// the same, multicast to the CTAs of cta_mask (cluster ranks): each destination's transaction bytes
// complete on the barrier at bar_cluster's offset in that destination's pair leader
LOKA_DEVINL void tma_load_2d_cg2_mc(void* dst, const CUtensorMap* m, uint32_t bar_cluster, int32_t c0, int32_t c1,
                                   uint16_t cta_mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"((uint64_t)m), "r"(bar_cluster), "r"(c0), "r"(c1), "h"(cta_mask)
      : "memory");
}
LOKA_DEVINL void mbar_arrive_expect_tx_cluster(uint32_t bar_cluster, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cluster.shared::cluster.b64 _, [%0], %1;" ::"r"(bar_cluster),
               "r"(bytes)
               : "memory");
}
LOKA_DEVINL void mbar_arrive_cluster(uint32_t bar_cluster) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster) : "memory");
}
LOKA_DEVINL void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// TMA 2-D load multicast to every CTA in cta_mask: the tile lands at dst's offset in each of
// them and completes as transaction bytes on the mbarrier at bar's offset in each of them.
LOKA_DEVINL void tma_load_2d_mc(void* dst, const CUtensorMap* m, uint64_t* bar, int32_t c0, int32_t c1,
                                uint16_t cta_mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, "
      "{%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"((uint64_t)m), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "h"(cta_mask)
      : "memory");
}
// make this thread's generic-proxy global writes visible to later async-proxy (TMA) reads
LOKA_DEVINL void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
// 1-D bulk copy global -> own shared memory, completing as transaction bytes on `bar`.
LOKA_DEVINL void bulk_load_g2s(void* dst_smem, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst_smem)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
LOKA_DEVINL void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// 32 lanes x 32 columns of 32-bit: thread t of the warp gets lane (base + t), 32 consecutive cols.
LOKA_DEVINL void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Split-phase TMEM loads: issue several loads, then ONE wait.  The wait carries every
// destination register as an in/out operand so the compiler cannot read them before it.
LOKA_DEVINL void tmem_ld32_nowait(uint32_t taddr, float* v) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
LOKA_DEVINL void tmem_ld16_nowait(uint32_t taddr, float* v) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
LOKA_DEVINL void tmem_wait16(float* v) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                 "+r"(r[15])::"memory");
}

LOKA_DEVINL void tmem_wait32(float* v) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                 "+r"(r[15]), "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]),
                 "+r"(r[22]), "+r"(r[23]), "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]),
                 "+r"(r[29]), "+r"(r[30]), "+r"(r[31])::"memory");
}

// ------------------------------------------------------------------------------------------
// clusters / DSMEM
// ------------------------------------------------------------------------------------------
LOKA_DEVINL uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
LOKA_DEVINL void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
LOKA_DEVINL uint32_t mapa_shared(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
LOKA_DEVINL void st_dsmem_f4(uint32_t addr, float4 v) {
  asm volatile("st.shared::cluster.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
               : "memory");
}
// Bulk (TMA-engine) copy of `bytes` (multiple of 16) from this CTA's shared memory to a cluster
// peer's; completes as transaction bytes on the peer's mbarrier (both cluster addresses, mapa).
LOKA_DEVINL void bulk_copy_s2cluster(uint32_t dst_cluster, uint32_t src_cta, uint32_t bytes, uint32_t mbar_cluster) {
  asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   dst_cluster),
               "r"(src_cta), "r"(bytes), "r"(mbar_cluster)
               : "memory");
}
// Remote (cluster peer) 16-B store that completes as 16 transaction bytes on the peer's mbarrier
// (st.async: no barrier on the sender's side; the receiver waits on its own mbarrier).
LOKA_DEVINL void st_async_u4(uint32_t dst_cluster, uint4 v, uint32_t mbar_cluster) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1,%2,%3,%4}, [%5];" ::"r"(
                   dst_cluster),
               "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "r"(mbar_cluster)
               : "memory");
}
LOKA_DEVINL void st_dsmem_f32(uint32_t addr, float v) {
  asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}
LOKA_DEVINL float ld_dsmem_f32(uint32_t addr) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(addr) : "memory");
  return v;
}

}  // namespace loka
