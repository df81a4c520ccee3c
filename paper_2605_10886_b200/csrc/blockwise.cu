// blockwise.cu — a4 with blockwise FP32 scales (BW-F32; D6/D7, PAPER.md:171/692
// "DeepGEMM BW": 1x128 activation scales, 128x128 weight scales).  Scales change every 128
// elements of K, so they cannot be factored out of the K sum: each 128-K block's MMA result is a
// separate partial sum that is promoted into an FP32 register accumulator,
//     y[m,n] += partial_kb[m,n] * s_a[m,kb] * s_b[n,kb]
// (s_b per 128x128 block of B, or per row of B for the 1x128 K-major copies of wgrad).
//
// CTA tile 128 x 128; warp 0 lane 0 = TMA producer, warp 1 lane 0 = MMA issuer writing k-block
// kb into TMEM buffer kb & 1 (fresh accumulation), warps 2-9 = promotion/epilogue (one row x 64
// columns per thread, in registers); the epilogue frees a TMEM buffer right after its tcgen05.ld,
// so the MMA of block kb+1 overlaps the promotion of block kb.  Output: (+bias) -> f32 / bf16 /
// e4m3 with ROW scales (row amax over N <= 128 within the CTA), TMA store of a swizzled tile.
#include "common.cuh"
#include "launch.h"

namespace loka {

constexpr int kWBN = 128;
constexpr int kWEpiWarps = 8;
constexpr int kWThreads = 64 + 32 * kWEpiWarps;
constexpr int kWCPT = kWBN / 2;
constexpr int kWStageBytes = 128 * 128 + kWBN * 128;
constexpr int kWStages = 5;
constexpr int kWOffOut = kWStages * kWStageBytes;            // staging tile (<= 128 x 128 f32 = 64 KB)
constexpr int kWOffRed = kWOffOut + 128 * kWBN * 4;          // [3][128]: B row scales / row amax halves
constexpr int kWOffBar = kWOffRed + 3 * 128 * 4;
constexpr int kWSmem = kWOffBar + 256 + 1024;
static_assert(kWSmem <= 227 * 1024, "blockwise smem");

__global__ void __launch_bounds__(kWThreads, 1)
    linear_bw_kernel(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
                     const __grid_constant__ CUtensorMap tma_y, const BwParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + kWOffBar);
  uint64_t* empty_bar = full_bar + kWStages;
  uint64_t* acc_full = empty_bar + kWStages;  // [2]
  uint64_t* acc_empty = acc_full + 2;          // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  float* red = reinterpret_cast<float*>(smem + kWOffRed);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * 128, n0 = blockIdx.y * kWBN;
  const int nkb = (p.K + 127) / 128;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tma_a);
    tma_prefetch_desc(&tma_b);
    tma_prefetch_desc(&tma_y);
    for (int s = 0; s < kWStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], kWEpiWarps);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<2 * kWBN>(tmem_slot);
  pdl_wait();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % kWStages;
        mbar_wait(&empty_bar[s], ((uint32_t)(kb / kWStages) & 1u) ^ 1u, 1);
        mbar_arrive_expect_tx(&full_bar[s], kWStageBytes);
        tma_load_2d(smem + s * kWStageBytes, &tma_a, &full_bar[s], kb * 128, m0);
        tma_load_2d(smem + s * kWStageBytes + 128 * 128, &tma_b, &full_bar[s], kb * 128, n0);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = idesc_f8f6f4(p.a_fmt, p.b_fmt, 128, kWBN);
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % kWStages, buf = kb & 1;
        mbar_wait(&acc_empty[buf], ((uint32_t)(kb >> 1) & 1u) ^ 1u, 4);
        mbar_wait(&full_bar[s], (uint32_t)(kb / kWStages) & 1u, 2);
        tc_fence_after();
        const uint32_t a0 = smem_u32(smem + s * kWStageBytes), b0 = a0 + 128 * 128;
        const uint32_t d = tmem_base + (uint32_t)(buf * kWBN);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          mma_f8f6f4(d, smem_desc_kmajor_sw128(a0 + k * 32), smem_desc_kmajor_sw128(b0 + k * 32), idesc, k != 0);
        mma_commit(&empty_bar[s]);
        mma_commit(&acc_full[buf]);
      }
    }
    __syncwarp();
  } else {
    const int q = warp & 3, h = (warp - 2) >> 2;
    const int r = q * 32 + lane;
    const int grow = m0 + r;
    const bool row_ok = grow < p.M;
    const int cb = h * kWCPT;
    const int nblk_b = (p.N + 127) / 128;
    float y[kWCPT];
#pragma unroll
    for (int j = 0; j < kWCPT; ++j) y[j] = 0.f;
    // per-row B scales (1x128 K-major copies): the CTA's 128 scales of k-block kb are staged in
    // smem (triple-buffered, one k-block ahead) instead of 64 strided global loads per thread
    float* sbs = red;  // [3][128] (red is reused for the FP8 row amax only after the loop)
    const int te = threadIdx.x - 64;
    auto stage_sb = [&](int kb) {
      if (te < 128) {
        const int n = n0 + te;
        sbs[(kb % 3) * 128 + te] = n < p.N ? __ldg(p.sb + (int64_t)n * p.sb_ld + kb) : 0.f;
      }
    };
    if (p.sb_rows) stage_sb(0);
    for (int kb = 0; kb < nkb; ++kb) {
      const int buf = kb & 1;
      if (p.sb_rows) {
        if (kb + 1 < nkb) stage_sb(kb + 1);
        named_bar_sync(1, 32 * kWEpiWarps);  // kb's scales visible; kb-2's buffer no longer read
      }
      // scales of this k-block (issued before the wait to hide their latency)
      const float sa = row_ok ? __ldg(p.sa + (int64_t)grow * p.sa_ld + kb) : 0.f;
      float sbk = 0.f;
      if (!p.sb_rows) sbk = __ldg(p.sb + (int64_t)(n0 / 128) * p.sb_ld + kb);  // one 128x128 block per CTA
      if (lane == 0) mbar_wait(&acc_full[buf], (uint32_t)(kb >> 1) & 1u, 3);
      __syncwarp();
      tc_fence_after();
      float part[kWCPT];
      const uint32_t ta = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * kWBN + cb);
      tmem_ld32_nowait(ta, part);
      tmem_ld32_nowait(ta + 32, part + 32);
#pragma unroll
      for (int i = 0; i < kWCPT / 16; ++i) tmem_wait16(part + 16 * i);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[buf]);
      if (!p.sb_rows) {
        const float s = sa * sbk;
        const float2 s2 = make_float2(s, s);
#pragma unroll
        for (int j = 0; j < kWCPT; j += 2) {
          const float2 t = ffma2(make_float2(part[j], part[j + 1]), s2, make_float2(y[j], y[j + 1]));
          y[j] = t.x;
          y[j + 1] = t.y;
        }
      } else {  // per-row scales of B (1x128 K-major copy): s_b[n, kb] from the staged smem copy
        const uint32_t sbase = smem_u32(sbs + (kb % 3) * 128 + cb);
        const float2 sa2 = make_float2(sa, sa);
#pragma unroll
        for (int j = 0; j < kWCPT; j += 4) {
          const float4 b4 = lds_f4(sbase + j * 4);
          const float2 s01 = fmul2(sa2, make_float2(b4.x, b4.y)), s23 = fmul2(sa2, make_float2(b4.z, b4.w));
          const float2 t0 = ffma2(make_float2(part[j], part[j + 1]), s01, make_float2(y[j], y[j + 1]));
          const float2 t1 = ffma2(make_float2(part[j + 2], part[j + 3]), s23, make_float2(y[j + 2], y[j + 3]));
          y[j] = t0.x; y[j + 1] = t0.y; y[j + 2] = t1.x; y[j + 3] = t1.y;
        }
      }
    }
    (void)nblk_b;
    if (p.sb_rows) named_bar_sync(1, 32 * kWEpiWarps);  // sbs (aliasing red) fully consumed
    // ---- bias, optional FP8 cast with row scale, TMA store ----
    const int nv = max(0, min(kWCPT, p.N - (n0 + cb)));
    if (p.bias) {
#pragma unroll
      for (int j = 0; j < kWCPT; ++j) {
        const int n = n0 + cb + j;
        if (j < nv) y[j] += p.bias_bf16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p.bias)[n])
                                        : reinterpret_cast<const float*>(p.bias)[n];
      }
    }
    const int esz = p.out_dtype == LOKA_F32 ? 4 : p.out_dtype == LOKA_BF16 ? 2 : 1;
    float r_out = 1.f;
    if (esz == 1) {  // row amax over the tile's <= 128 columns (N <= 128 checked on the host)
      float am = 0.f;
#pragma unroll
      for (int j = 0; j < kWCPT; ++j)
        if (j < nv) am = fmaxf(am, fabsf(y[j]));
      red[h * 128 + r] = am;
      named_bar_sync(1, 32 * kWEpiWarps);
      am = fmaxf(red[r], red[128 + r]);
      float s_out;
      if (p.out_dtype == LOKA_E4M3) scales_from_amax<LOKA_E4M3, LOKA_SCALE_F32>(am, s_out, r_out);
      else scales_from_amax<LOKA_E5M2, LOKA_SCALE_F32>(am, s_out, r_out);
      if (row_ok && h == 0 && p.y_scales) p.y_scales[grow] = s_out;
    }
    if (p.precast && row_ok) {
#pragma unroll
      for (int j = 0; j < kWCPT; ++j)
        if (j < nv) p.precast[(int64_t)grow * p.ld_pre + n0 + cb + j] = y[j];
    }
    const uint32_t box_bytes = (uint32_t)min(128, kWBN * esz);
    const uint32_t stage_s = smem_u32(smem + kWOffOut);
    auto put16 = [&](int chunk, uint4 v) {
      const uint32_t bofs = (uint32_t)(cb * esz + 16 * chunk);
      const uint32_t c16 = (bofs % box_bytes) >> 4;
      const uint32_t sw = box_bytes == 128u ? (c16 ^ ((uint32_t)r & 7u)) : (c16 ^ (((uint32_t)r >> 1) & 3u));
      sts_u4(stage_s + (bofs / box_bytes) * (128u * box_bytes) + (uint32_t)r * box_bytes + (sw << 4), v);
    };
    if (esz == 4) {
#pragma unroll
      for (int k = 0; k < kWCPT / 4; ++k)
        put16(k, make_uint4(__float_as_uint(y[4 * k]), __float_as_uint(y[4 * k + 1]), __float_as_uint(y[4 * k + 2]),
                            __float_as_uint(y[4 * k + 3])));
    } else if (esz == 2) {
#pragma unroll
      for (int k = 0; k < kWCPT / 8; ++k) {
        uint32_t w[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          __nv_bfloat162 hh = __floats2bfloat162_rn(y[8 * k + 2 * i], y[8 * k + 2 * i + 1]);
          w[i] = *reinterpret_cast<uint32_t*>(&hh);
        }
        put16(k, make_uint4(w[0], w[1], w[2], w[3]));
      }
    } else {
#pragma unroll
      for (int k = 0; k < kWCPT / 16; ++k) {
        uint32_t w[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int j = 16 * k + 4 * i;
          const float a0 = __fmul_rn(y[j], r_out), a1 = __fmul_rn(y[j + 1], r_out);
          const float a2 = __fmul_rn(y[j + 2], r_out), a3 = __fmul_rn(y[j + 3], r_out);
          w[i] = p.out_dtype == LOKA_E4M3 ? cvt_fp8x4<LOKA_E4M3>(a0, a1, a2, a3) : cvt_fp8x4<LOKA_E5M2>(a0, a1, a2, a3);
        }
        put16(k, make_uint4(w[0], w[1], w[2], w[3]));
      }
    }
    fence_proxy_async_smem();
    named_bar_sync(1, 32 * kWEpiWarps);
    if (threadIdx.x == 64) {
      const int per_box = (int)box_bytes / esz, nbox = kWBN * esz / (int)box_bytes;
      for (int b = 0; b < nbox; ++b) {
        const int c0 = n0 + b * per_box;
        if (c0 < p.N) tma_store_2d(&tma_y, smem + kWOffOut + b * 128 * (int)box_bytes, c0, m0);
      }
      bulk_commit();
      bulk_wait_read0();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<2 * kWBN>(tmem_base);
  }
}

cudaError_t launch_linear_bw(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& ty, const BwParams& p,
                             cudaStream_t st) {
  {
    cudaError_t e = ensure_func_attrs(reinterpret_cast<const void*>(linear_bw_kernel), kWSmem);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)((p.M + 127) / 128), (unsigned)((p.N + kWBN - 1) / kWBN), 1);
  cfg.blockDim = dim3(kWThreads, 1, 1);
  cfg.dynamicSmemBytes = kWSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, linear_bw_kernel, ta, tb, ty, p);
  note_launch();
  return e;
}

}  // namespace loka
