// grouped.cu — a6: many small FP8 GEMMs ("architecturally heterogeneous ... wide
// ensembles"; DHEN/Wukong-style, BJ configs[2]) in ONE persistent launch.
//
// Design:
//   * The tiles (128 x BN, BN = 128) of up to kMaxGroups GEMMs form one list, groups ordered
//     longest-K first on the host; a persistent grid of <= #SM CTAs walks the list round-robin.
//   * Warp 0 lane 0 = TMA producer running ahead through tiles and k-blocks over one smem ring;
//     warp 1 lane 0 = tcgen05.mma issuer writing tile t into TMEM accumulator buffer t & 1;
//     warps 2-9 = epilogue (two warps per TMEM lane quadrant, BN/2 columns per thread held in
//     registers).  The epilogue releases the accumulator buffer right after its tcgen05.ld, so the
//     MMAs of tile t+1 overlap the dequant / cast / store of tile t.
//   * Epilogue: y = acc * s_a[m] * s_b[n] (+ bias[n]) -> f32 / bf16 into a 128B-swizzled smem tile
//     (double-buffered) -> TMA bulk-tensor store.
// Row-coupled epilogues (LayerNorm / RMSNorm / FP8 output with row scales) and BlockNorm are
// served by per-group launches of linear_norm_kernel (api.cu decides).
#include "common.cuh"
#include "launch.h"

namespace loka {

constexpr int kGBN = 128;                  // tile N
constexpr int kGEpiWarps = 8;
constexpr int kGThreads = 64 + 32 * kGEpiWarps;
constexpr int kGCPT = kGBN / 2;            // columns per epilogue thread
constexpr int kGStageA = 128 * 128, kGStageB = kGBN * 128, kGStageBytes = kGStageA + kGStageB;
constexpr int kGStages = 5;
constexpr int kGStageOut = 128 * kGBN * 2;  // one bf16 output staging tile (double-buffered)
constexpr int kGOffB = kGStages * kGStageA;
constexpr int kGOffOut = kGOffB + kGStages * kGStageB;       // 2 staging tiles
constexpr int kGOffBar = kGOffOut + 2 * kGStageOut;
constexpr int kGSmem = kGOffBar + 256 + 1024;
static_assert(kGSmem <= 227 * 1024, "grouped smem");

__global__ void __launch_bounds__(kGThreads, 1) grouped_linear_kernel(const __grid_constant__ GroupedParams gp) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + kGOffB;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + kGOffBar);
  uint64_t* empty_bar = full_bar + kGStages;
  uint64_t* acc_full = empty_bar + kGStages;  // [2]
  uint64_t* acc_empty = acc_full + 2;          // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int T = gp.tile_start[gp.G];

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kGStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], kGEpiWarps);  // one arrival per epilogue warp
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<2 * kGBN>(tmem_slot);
  pdl_wait();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  auto locate = [&](int t, int& g, int& mb, int& nb) {
    g = 0;
    while (t >= gp.tile_start[g + 1]) ++g;
    const int local = t - gp.tile_start[g];
    const int tn = gp.g[g].tiles_n;
    mb = local / tn;
    nb = local - mb * tn;
  };

  if (warp == 0) {
    // ===== TMA producer: runs ahead across tiles =====
    if (lane == 0) {
      int it = 0;  // global k-block counter (ring position)
      for (int t = blockIdx.x; t < T; t += gridDim.x) {
        int g, mb, nb;
        locate(t, g, mb, nb);
        const int nkb = (gp.g[g].K + 127) / 128;
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % kGStages;
          const uint32_t ph = (uint32_t)(it / kGStages) & 1u;
          mbar_wait(&empty_bar[s], ph ^ 1u, 1);
          mbar_arrive_expect_tx(&full_bar[s], kGStageBytes);
          tma_load_2d(sA + s * kGStageA, &gp.ta[g], &full_bar[s], kb * 128, mb * 128);
          tma_load_2d(sB + s * kGStageB, &gp.tb[g], &full_bar[s], kb * 128, nb * kGBN);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ===== MMA issuer: tile j -> accumulator buffer j & 1 =====
    if (lane == 0) {
      int it = 0, j = 0;
      for (int t = blockIdx.x; t < T; t += gridDim.x, ++j) {
        int g, mb, nb;
        locate(t, g, mb, nb);
        const int nkb = (gp.g[g].K + 127) / 128;
        const int buf = j & 1;
        mbar_wait(&acc_empty[buf], ((uint32_t)(j >> 1) & 1u) ^ 1u, 4);  // epilogue drained it
        tc_fence_after();
        const uint32_t idesc = idesc_f8f6f4(gp.g[g].a_fmt, gp.g[g].b_fmt, 128, kGBN);
        const uint32_t dacc = tmem_base + (uint32_t)(buf * kGBN);
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % kGStages;
          const uint32_t ph = (uint32_t)(it / kGStages) & 1u;
          mbar_wait(&full_bar[s], ph, 2);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + s * kGStageA);
          const uint32_t b0 = smem_u32(sB + s * kGStageB);
#pragma unroll
          for (int k = 0; k < 4; ++k)
            mma_f8f6f4(dacc, smem_desc_kmajor_sw128(a0 + k * 32), smem_desc_kmajor_sw128(b0 + k * 32), idesc,
                       (kb | k) != 0);
          mma_commit(&empty_bar[s]);
        }
        mma_commit(&acc_full[buf]);
      }
    }
    __syncwarp();
  } else {
    // ===== epilogue: warps 2..9, thread = row x column half =====
    const int q = warp & 3;
    const int h = (warp - 2) >> 2;
    const int r = q * 32 + lane;
    const int cb = h * kGCPT;
    int j = 0;
    for (int t = blockIdx.x; t < T; t += gridDim.x, ++j) {
      int g, mb, nb;
      locate(t, g, mb, nb);
      const GroupDesc& d = gp.g[g];
      const int buf = j & 1;
      if (lane == 0) mbar_wait(&acc_full[buf], (uint32_t)(j >> 1) & 1u, 3);
      __syncwarp();
      tc_fence_after();
      float y[kGCPT];
      const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * kGBN + cb);
      tmem_ld32_nowait(taddr, y);
      tmem_ld32_nowait(taddr + 32, y + 32);
#pragma unroll
      for (int i = 0; i < kGCPT / 16; ++i) tmem_wait16(y + 16 * i);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[buf]);  // accumulator buffer free for tile j+2

      const int grow = mb * 128 + r;
      const int n0 = nb * kGBN + cb;
      const float sa = grow < d.M ? d.sa[d.sa_row ? grow : 0] : 0.f;
      // dequant (+ bias); columns >= N read s_b / bias as 0 (clipped by the TMA store anyway)
#pragma unroll
      for (int c = 0; c < kGCPT; c += 2) {
        const int n = n0 + c;
        const float s0 = n < d.N ? __ldg(d.sb + (d.sb_row ? n : 0)) : 0.f;
        const float s1 = n + 1 < d.N ? __ldg(d.sb + (d.sb_row ? n + 1 : 0)) : 0.f;
        float2 a = fmul2(make_float2(y[c], y[c + 1]), make_float2(sa * s0, sa * s1));
        if (d.bias) {
          float b0 = 0.f, b1 = 0.f;
          if (n < d.N) b0 = d.bias_bf16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(d.bias)[n])
                                        : reinterpret_cast<const float*>(d.bias)[n];
          if (n + 1 < d.N) b1 = d.bias_bf16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(d.bias)[n + 1])
                                            : reinterpret_cast<const float*>(d.bias)[n + 1];
          a = fadd2(a, make_float2(b0, b1));
        }
        y[c] = a.x;
        y[c + 1] = a.y;
      }
      // staging buffer j & 1: make sure the TMA store that used it two tiles ago has read it
      if (threadIdx.x == 64) bulk_wait_read_le1();
      named_bar_sync(2, 32 * kGEpiWarps);
      const int esz = 2;  // bf16 output (api.cu routes other output types to per-group launches)
      const uint32_t stage_s = smem_u32(smem + kGOffOut + buf * kGStageOut);
      auto put16 = [&](int chunk, uint4 v) {
        const uint32_t bofs = (uint32_t)(cb * esz + 16 * chunk);
        const uint32_t a = stage_s + (bofs >> 7) * 16384u + (uint32_t)r * 128u +
                           ((((bofs >> 4) & 7u) ^ ((uint32_t)r & 7u)) << 4);
        sts_u4(a, v);
      };
#pragma unroll
      for (int k = 0; k < kGCPT / 8; ++k) {
        uint32_t w[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          __nv_bfloat162 hh = __floats2bfloat162_rn(y[8 * k + 2 * i], y[8 * k + 2 * i + 1]);
          w[i] = *reinterpret_cast<uint32_t*>(&hh);
        }
        put16(k, make_uint4(w[0], w[1], w[2], w[3]));
      }
      fence_proxy_async_smem();
      named_bar_sync(2, 32 * kGEpiWarps);
      if (threadIdx.x == 64) {
        const int per_box = 128 / esz;
        const int nbox = kGBN * esz / 128;
        for (int b = 0; b < nbox; ++b) {
          const int c0 = nb * kGBN + b * per_box;
          if (c0 < d.N) tma_store_2d(&gp.ty[g], smem + kGOffOut + buf * kGStageOut + b * 16384, c0, mb * 128);
        }
        bulk_commit();
      }
    }
    if (threadIdx.x == 64) bulk_wait_read0();
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<2 * kGBN>(tmem_base);
  }
}

cudaError_t launch_grouped(const GroupedParams& gp, int num_sms, cudaStream_t st) {
  {
    cudaError_t e = ensure_func_attrs(reinterpret_cast<const void*>(grouped_linear_kernel), kGSmem);
    if (e != cudaSuccess) return e;
  }
  const int T = gp.tile_start[gp.G];
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(T < num_sms ? T : num_sms), 1, 1);
  cfg.blockDim = dim3(kGThreads, 1, 1);
  cfg.dynamicSmemBytes = kGSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, grouped_linear_kernel, gp);
  note_launch();
  return e;
}

}  // namespace loka
