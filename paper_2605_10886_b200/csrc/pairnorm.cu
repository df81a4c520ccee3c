// pairnorm.cu — a4 + a5 at scale: the CTA-pair FP8 GEMM (gemm2.cu's engine) with the row norm
// fused into its epilogue, so the FP32 tile never goes to HBM ("fuse normalization
// directly into the GEMM epilogue to minimize HBM I/O"; Case 1 / Case 2).
//
// Tile: a 2-CTA cluster (tcgen05.mma.cta_group::2, M = 256) computes 256 rows x TN columns; each
// CTA holds its 128 rows x TN columns of FP32 accumulator in TMEM.
//   * TN = 256: two accumulator buffers; tile j+1's MMAs run while the epilogue drains tile j.
//   * TN = 512 ("WIDE"): two N = 256 MMAs per K step share the A stage (gemm2's L2 -> SM port
//     saving); one accumulator, so a tile's epilogue does not overlap the next tile's MMAs.
// Epilogue (8 warps per CTA; warp = TMEM lane quadrant q x column half h; thread = one row x TN/2
// columns, streamed out of TMEM in 32-column chunks with the next chunk's load in flight):
//   pass S  y = acc * s_a[m] * s_b[n] (+ bias[n]) -> per-chunk (mean, M2) merged in order with
//           Chan's update (LayerNorm; the parallel merge of PAPER.md:293-299 applied to column
//           partitions) or the sum of squares (RMS / BlockNorm), y max / min (FP8 row amax); the two
//           column halves merged through smem.  With a tensor-wide s_b and no bias the statistics are
//           taken on acc and scaled (mean * c, M2 * c^2; c = s_a s_b), and pass N is one FMA;
//   xchg    rows wider than one tile (Case 2): the G = ceil(N / TN) tiles of a row are
//           computed by G different pairs.  Each CTA stores its 128 row records (float4) to the
//           workspace, which the host fills with a sentinel NaN pattern before the launch; the
//           readers load the G records of their row directly and re-load any element still holding
//           the sentinel (a 32-bit store is single-copy atomic, and no statistic of finite data is
//           that NaN), so the exchange is one L2 round trip after the last peer's store — no flags,
//           no fences; the G records are merged in tile order (bit-identical in every CTA of a row);
//   pass N  the same y -> (y - mu) * rstd [* gamma + beta] [h-swish] -> bf16 / f32 / FP8 (row scale
//           from the merged y max / min: the map is monotone) -> swizzled smem box -> TMA store.
// Exchange through global memory (L2), not DSMEM: a 4096-wide row spans 16 (TN = 256) or 8 WIDE
// pairs, and clusters of 16+ CTAs would leave ~14% of the SMs idle.  Co-residency: one CTA per SM,
// at most 2 x 74 CTAs, every CTA resident (a reader only waits for tiles other resident pairs own).
#include <algorithm>

#include "common.cuh"
#include "launch.h"

namespace loka {

constexpr int kPnEpiWarps = 8;
constexpr int kPnThreads = 64 + 32 * kPnEpiWarps;
constexpr int kPnCastWarps = 2;  // CASTX: warps that quantize X for the tiles ahead of the MMAs
constexpr int kPnCastAhead = 3;  // CASTX default: the cast warps stay <= this many tiles ahead of the epilogue
                                 // (spreads their HBM / L2 traffic over the GEMM instead of bursting it)
constexpr uint32_t kPnSentinel = 0xFFFFFFFFu;  // a NaN no statistic of finite data can take

template <int TN>
struct PnCfg {
  static constexpr int kStages = TN == 512 ? 3 : 4;
  static constexpr int kAcc = TN == 512 ? 1 : 2;      // accumulator buffers in the 512 TMEM columns
  static constexpr int kColBufs = TN == 512 ? 1 : 2;  // column-parameter buffers (sb, bias, gamma, beta)
  static constexpr int kStageA = 128 * 128;
  static constexpr int kStageB = (TN / 2) * 128;      // per CTA: 128 rows of each 256-column half
  static constexpr int kOffB = kStages * kStageA;
  static constexpr int kOffOut = kOffB + kStages * kStageB;      // [8 warps][2][32 rows x 128 B]
  static constexpr int kOffCol = kOffOut + kPnEpiWarps * 2 * 4096;
  static constexpr int kOffRec = kOffCol + kColBufs * 4 * TN * 4;  // [2 halves][128 rows] float4
  static constexpr int kOffBar = kOffRec + 2 * 128 * 16;
  static constexpr int kSmem = kOffBar + 256 + 1024;
  static_assert(kSmem <= 227 * 1024, "pairnorm smem");
};

// Case 2 records (caller's workspace): float4 [row blocks][tiles_n][2 CTA ranks][128 rows], set to
// the sentinel by the host (a memset node in the same stream) before every launch.
size_t pair_xchg_bytes(int64_t row_blocks, int tiles_n) { return (size_t)row_blocks * tiles_n * 2 * 128 * 16; }

LOKA_DEVINL float4 ld_relaxed_f4(const float4* p) {
  float4 v;
  asm volatile("ld.relaxed.gpu.global.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p)
               : "memory");
  return v;
}
LOKA_DEVINL bool rec_pending(const float4& v) {
  return __float_as_uint(v.x) == kPnSentinel || __float_as_uint(v.y) == kPnSentinel ||
         __float_as_uint(v.z) == kPnSentinel || __float_as_uint(v.w) == kPnSentinel;
}
// re-load a peer's record until no element holds the sentinel; the watchdog of mbar_wait
// (common.cuh): a wait longer than 4 s records where it stalled and gives up instead of hanging
LOKA_DEVINL float4 rec_wait(const float4* p) {
  float4 v = ld_relaxed_f4(p);
  uint32_t spins = 0;
  uint64_t t0 = 0;
  while (rec_pending(v)) {
    if ((++spins & 15u) == 0) {
      __nanosleep(64);
      const uint64_t t = globaltimer_ns();
      if (t0 == 0) t0 = t;
      if (*reinterpret_cast<volatile int*>(&g_loka_abort)) break;
      if (t - t0 > kHangNs) {
        if (atomicAdd(&g_loka_hang[0], 1ull) == 0) {
          g_loka_hang[1] = 100ull;
          g_loka_hang[2] = (unsigned long long)blockIdx.x;
          g_loka_hang[3] = (unsigned long long)threadIdx.x;
        }
        atomicExch(&g_loka_abort, 1);
        break;
      }
    }
    v = ld_relaxed_f4(p);
  }
  return v;
}

// CASTX producer side: wait until a row block's cast parts are all published (acquire), with the watchdog
LOKA_DEVINL void xcnt_wait(const uint32_t* c, uint32_t need) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(c) : "memory");
  if (v >= need) return;
  uint32_t spins = 0;
  uint64_t t0 = 0;
  for (;;) {
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(c) : "memory");
    if (v >= need) return;
    __nanosleep(64);
    if ((++spins & 63u) != 0) continue;
    const uint64_t t = globaltimer_ns();
    if (t0 == 0) t0 = t;
    if (*reinterpret_cast<volatile int*>(&g_loka_abort)) return;
    if (t - t0 > kHangNs) {
      if (atomicAdd(&g_loka_hang[0], 1ull) == 0) {
        g_loka_hang[1] = 101ull;
        g_loka_hang[2] = (unsigned long long)blockIdx.x;
        g_loka_hang[3] = (unsigned long long)threadIdx.x;
      }
      atomicExch(&g_loka_abort, 1);
      return;
    }
  }
}

LOKA_DEVINL float hswish(float x) {  // x * ReLU6(x + 3) / 6
  const float t = fminf(fmaxf(x + 3.f, 0.f), 6.f);
  return __fdiv_rn(__fmul_rn(x, t), 6.f);
}

// BF16IN: BF16 operands (kind::f16; a 128-byte stage row holds 64 K elements; the maps are byte views
// of the bf16 data): the library's own BF16 path with the same fused epilogue (SURVEY.md §8(d)'s
// secondary denominator, separating the FP8 gain from the fusion gain)
// BWD: the NEXT-1 norm backward epilogue (a separate instance, so the forward carries none of it).
// CASTX: the tensorwise cast of X fused into the GEMM (x_recipe, "quantization overhead"):
// two extra warps per CTA cast this pair's share of each upcoming row block from bf16 to FP8 codes with
// the given (all-reduced) amax, publishing per-row-block counters that the TMA producers wait on.
template <int TN, int NORM, bool BF16IN, bool BWD, bool CASTX = false>
__global__ void __launch_bounds__(kPnThreads + (CASTX ? 32 * kPnCastWarps : 0), 1)
    pair_norm_kernel(const __grid_constant__ PairNormParams p) {
  using Cf = PnCfg<TN>;
  constexpr int kHN = TN / 2;     // columns per epilogue thread
  constexpr int kNch = kHN / 32;  // 32-column chunks per thread
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + Cf::kOffB;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + Cf::kOffBar);
  uint64_t* empty_bar = full_bar + Cf::kStages;
  uint64_t* acc_full = empty_bar + Cf::kStages;  // [2]
  uint64_t* acc_empty = acc_full + 2;           // [2] (the leader's is used)
  uint64_t* xbar = acc_empty + 2;  // [8] backward: the warps' staged xhat sub-tiles landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(xbar + kPnEpiWarps);
  float4* hrec = reinterpret_cast<float4*>(smem + Cf::kOffRec);
  volatile int* ep_tile = reinterpret_cast<volatile int*>(tmem_slot + 1);  // CASTX pacing: the epilogue's tile

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // cluster rank: bit 0 = the CTA within its pair (the cta_group::2 peer), bit 1 = the pair within a
  // 4-CTA cluster (mc); `rank` below is the CTA's rank within its pair
  const int crank = (int)cluster_ctarank();
  const int rank = crank & 1, lead = crank & ~1, cq = crank >> 1;
  const bool mc = p.mc != 0;
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const int G = p.tiles_n;
  // schedule: order 0 = round-robin over the tile list (row-block major: the G tiles of a row are
  // computed by G consecutive pairs, mostly in the same wave); order 1 = static groups of G pairs
  // that walk row blocks gi, gi + #groups, ... in lock step (for the single-accumulator WIDE tile,
  // which cannot wait for a peer's next wave without idling its tensor core)
  const bool xchg = p.xchg != 0;
  const int gi = p.order == 1 ? cid / G : 0, gj = p.order == 1 ? cid - (cid / G) * G : 0;
  const int T = p.row_blocks * G;
  auto tile_of = [&](int k, int& mb, int& nb) -> bool {  // k-th tile of this pair
    if (p.order == 1) {
      mb = gi + k * p.ngroups;
      nb = gj;
      return mb < p.row_blocks;
    }
    const int t = cid + k * ncl;
    mb = t / G;
    nb = t - mb * G;
    return t < T;
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&p.ta);
    tma_prefetch_desc(&p.tb);
    tma_prefetch_desc(&p.ty);
    for (int s = 0; s < Cf::kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], mc ? 2 : 1);  // mc: both pairs' MMAs read this CTA's A stage
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 2 * kPnEpiWarps);
    }
    for (int w = 0; w < kPnEpiWarps; ++w) mbar_init(&xbar[w], 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_cg2<512>(tmem_slot);
  if (threadIdx.x == 0) *ep_tile = 0;
  pdl_wait();
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int nkb = (p.K * (BF16IN ? 2 : 1) + 127) / 128;  // 128-byte K stages

  if (warp == 0) {
    // ===== TMA producer (both CTAs): this CTA's 128 A rows and half of each 256-row B half =====
    if (lane == 0) {
      const uint32_t full0 = mapa_shared(smem_u32(full_bar), (uint32_t)lead);
      int it = 0, mb, nb;
      for (int k = 0; tile_of(k, mb, nb); ++k) {
        if constexpr (CASTX) {  // this row block's codes: all 4 G cast parts published
          xcnt_wait(&p.xcnt[mb], 4u * (uint32_t)G);
          fence_proxy_async_global();  // (generic-proxy stores of other SMs -> this SM's TMA reads)
        }
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % Cf::kStages;
          const uint32_t ph = (uint32_t)(it / Cf::kStages) & 1u;
          mbar_wait(&empty_bar[s], ph ^ 1u, 1);
          if (rank == 0) mbar_arrive_expect_tx(&full_bar[s], 2u * (Cf::kStageA + Cf::kStageB));
          if (mc)  // half of the 128 A rows, to this CTA and its counterpart in the other pair
            tma_load_2d_cg2_mc(sA + s * Cf::kStageA + cq * 8192, &p.ta64, full0 + 8u * s, kb * 128,
                               mb * 256 + rank * 128 + cq * 64, (uint16_t)((1u << rank) | (1u << (2 + rank))));
          else
            tma_load_2d_cg2(sA + s * Cf::kStageA, &p.ta, full0 + 8u * s, kb * 128, mb * 256 + rank * 128);
#pragma unroll
          for (int hh = 0; hh < TN / 256; ++hh)
            tma_load_2d_cg2(sB + s * Cf::kStageB + hh * 16384, &p.tb, full0 + 8u * s, kb * 128,
                            nb * TN + hh * 256 + rank * 128);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ===== MMA issuer (leader only) =====
    if (lane == 0 && rank == 0) {
      const uint32_t idesc = BF16IN ? idesc_bf16(256, 256) : idesc_f8f6f4(p.a_fmt, p.b_fmt, 256, 256);
      int it = 0, mb, nb;
      for (int j = 0; tile_of(j, mb, nb); ++j) {
        const int buf = Cf::kAcc == 1 ? 0 : (j & 1);
        const uint32_t use = Cf::kAcc == 1 ? (uint32_t)j : (uint32_t)(j >> 1);
        uint64_t* tr = (p.trace && j < 64) ? p.trace + ((size_t)blockIdx.x * 64 + j) * 8 : nullptr;
        if (tr) tr[4] = globaltimer_ns();
        mbar_wait(&acc_empty[buf], (use & 1u) ^ 1u, 4);
        if (tr) tr[5] = globaltimer_ns();
        tc_fence_after();
        const uint32_t dacc = tmem_base + (uint32_t)(buf * 256);
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % Cf::kStages;
          const uint32_t ph = (uint32_t)(it / Cf::kStages) & 1u;
          mbar_wait(&full_bar[s], ph, 2);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + s * Cf::kStageA);
          const uint32_t b0 = smem_u32(sB + s * Cf::kStageB);
#pragma unroll
          for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int hh = 0; hh < TN / 256; ++hh) {
              const uint64_t da = smem_desc_kmajor_sw128(a0 + k * 32);
              const uint64_t db = smem_desc_kmajor_sw128(b0 + hh * 16384 + k * 32);
              if constexpr (BF16IN) mma_bf16_cg2(dacc + hh * 256, da, db, idesc, (kb | k) ? 1u : 0u);
              else mma_f8f6f4_cg2(dacc + hh * 256, da, db, idesc, (kb | k) ? 1u : 0u);
            }
          mma_commit_cg2_mc(&empty_bar[s], mc ? (uint16_t)0xF : (uint16_t)(3u << lead));
        }
        mma_commit_cg2_mc(&acc_full[buf], (uint16_t)(3u << lead));
        if (tr) tr[6] = globaltimer_ns();
      }
    }
    __syncwarp();
  } else if (CASTX && warp >= 2 + kPnEpiWarps) {
    // ===== X cast warps (both CTAs): row block mb's 256 rows are split over its G tiles' pairs, and a
    // pair's share over its 2 CTAs x 2 cast warps; each warp casts its rows (fl32(x r), satRNE, the
    // arithmetic of loka_quantize's tensorwise cast: bit-identical codes), then publishes one part ====
    const int cw = warp - (2 + kPnEpiWarps);
    float s_x, r_x;
    if (p.a_fmt) scales_from_amax<LOKA_E5M2, LOKA_SCALE_F32>(*p.xamax, s_x, r_x);
    else scales_from_amax<LOKA_E4M3, LOKA_SCALE_F32>(*p.xamax, s_x, r_x);
    if (blockIdx.x == 0 && cw == 0 && lane == 0 && p.xs_out) p.xs_out[0] = s_x;
    int mb, nb;
    for (int k = 0; tile_of(k, mb, nb); ++k) {
      if (k > p.cast_ahead) {  // pacing: wait for the epilogue to reach tile k - cast_ahead
        while (*ep_tile < k - p.cast_ahead) __nanosleep(256);
      }
      const int j0 = (256 * nb) / G, j1 = (256 * (nb + 1)) / G, part = rank * kPnCastWarps + cw;
      const int r0 = j0 + ((j1 - j0) * part) / 4, r1 = j0 + ((j1 - j0) * (part + 1)) / 4;
      for (int rr = r0; rr < r1; ++rr) {
        const int64_t row = (int64_t)mb * 256 + rr;
        if (row >= p.M) break;
        const __nv_bfloat16* xr = p.xb + row * p.ld_xb;
        uint8_t* qr = p.xq + row * p.ld_xq;
        for (int c0 = lane * 8; c0 < p.K; c0 += 256 * 4) {
          uint4 v[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int c = c0 + 256 * u;
            v[u] = c < p.K ? __ldcs(reinterpret_cast<const uint4*>(xr + c)) : make_uint4(0u, 0u, 0u, 0u);
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int c = c0 + 256 * u;
            if (c >= p.K) break;
            float f[8] = {bf16lo_to_f32(v[u].x), bf16hi_to_f32(v[u].x), bf16lo_to_f32(v[u].y), bf16hi_to_f32(v[u].y),
                          bf16lo_to_f32(v[u].z), bf16hi_to_f32(v[u].z), bf16lo_to_f32(v[u].w), bf16hi_to_f32(v[u].w)};
#pragma unroll
            for (int i = 0; i < 8; ++i) f[i] = __fmul_rn(f[i], r_x);
            const uint2 code = p.a_fmt ? make_uint2(cvt_fp8x4<LOKA_E5M2>(f[0], f[1], f[2], f[3]),
                                                    cvt_fp8x4<LOKA_E5M2>(f[4], f[5], f[6], f[7]))
                                       : make_uint2(cvt_fp8x4<LOKA_E4M3>(f[0], f[1], f[2], f[3]),
                                                    cvt_fp8x4<LOKA_E4M3>(f[4], f[5], f[6], f[7]));
            *reinterpret_cast<uint2*>(qr + c) = code;
          }
        }
      }
      __syncwarp();
      if (lane == 0) {  // release this part: the codes above, then the counter
        __threadfence();
        fence_proxy_async_global();
        atomicAdd(&p.xcnt[mb], 1u);
      }
    }
  } else {
    // ===== epilogue (both CTAs) =====
    const int q = warp & 3;          // TMEM lane quadrant (hardware: warp w reads lanes 32 (w % 4) ..)
    const int h = (warp - 2) >> 2;   // column half
    const int r = q * 32 + lane;     // row within this CTA's 128
    const int et = threadIdx.x - 64;  // 0..255
    uint8_t* stg = smem + Cf::kOffOut + (warp - 2) * 8192;
    const uint32_t acc_empty0 = mapa_shared(smem_u32(acc_empty), (uint32_t)lead);
    const int esz = p.out_dtype == LOKA_F32 ? 4 : p.out_dtype == LOKA_BF16 ? 2 : 1;
    const bool fp8_out = esz == 1;
    const int cpb = 128 / esz;  // columns per 128-byte box row
    const bool has_gb = p.gamma != nullptr || p.beta != nullptr;
    const bool act = p.act == LOKA_ACT_HARDSWISH;
    // fold: with a tensor-wide s_b and no bias, y = acc * c (c = s_a s_b per row), so the statistics
    // are taken on acc and scaled (mean * c, M2 * c^2), and pass N is one FMA per element
    constexpr bool bwd = BWD;  // NEXT-1 norm backward (dL/dz from dL/dh, the forward's saved xhat / rstd)
    float sa_castx = 1.f;
    if constexpr (CASTX) {
      float r_unused;
      if (p.a_fmt) scales_from_amax<LOKA_E5M2, LOKA_SCALE_F32>(*p.xamax, sa_castx, r_unused);
      else scales_from_amax<LOKA_E4M3, LOKA_SCALE_F32>(*p.xamax, sa_castx, r_unused);
    }
    const bool xs_stage = BWD && p.out_dtype == LOKA_BF16;  // xhat staged in smem (bf16 dz boxes match it)
    uint32_t xph = 0;
    const bool fold = !p.sb_row && p.bias == nullptr && !bwd;
    // (BlockNorm exchanges only for the forward FP8 row amax; the backward's block sums are tile-local
    // and its FP8 dz takes 1x128 granules)
    const bool need_x = xchg && (NORM != LOKA_NORM_BLOCK_RMS || (fp8_out && !bwd));
    float4* xrec = reinterpret_cast<float4*>(p.xws);
    int nbox = 0;
    int mb, nb;
    for (int j = 0; tile_of(j, mb, nb); ++j) {
      const int buf = Cf::kAcc == 1 ? 0 : (j & 1);
      const uint32_t use = Cf::kAcc == 1 ? (uint32_t)j : (uint32_t)(j >> 1);
      // ---- column parameters of this tile -> smem (sb, bias, gamma, beta) ----
      float* colp = reinterpret_cast<float*>(smem + Cf::kOffCol) + (Cf::kColBufs == 1 ? 0 : (j & 1)) * 4 * TN;
      if (Cf::kColBufs == 1) named_bar_sync(2, 32 * kPnEpiWarps);  // the previous tile's reads are done
      if (!fold || has_gb) {
        for (int e = et; e < TN; e += 32 * kPnEpiWarps) {
          const int n = nb * TN + e;
          const bool ok = n < p.N;
          colp[e] = ok ? __ldg(p.sb + (p.sb_row ? n : 0)) : 0.f;
          float b = 0.f;
          if (ok && p.bias) b = p.bias_bf16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p.bias)[n])
                                            : reinterpret_cast<const float*>(p.bias)[n];
          colp[TN + e] = b;
          colp[2 * TN + e] = (ok && p.gamma) ? __ldg(p.gamma + n) : 1.f;
          colp[3 * TN + e] = (ok && p.beta) ? __ldg(p.beta + n) : 0.f;
        }
      }
      named_bar_sync(2, 32 * kPnEpiWarps);
      // backward with bf16 dz: this warp's xhat sub-tile (32 rows x 128 columns, 8 KB) is TMA-loaded into
      // its output staging area (two 32 x 64 SW128 boxes, exactly the layout of the dz boxes it will
      // store), so both passes read it from smem and pass N overwrites each chunk's xhat with its dz
      if constexpr (BWD) {
        if (xs_stage && lane == 0) {
          bulk_wait_read0();  // the previous tile's dz boxes have been read out of the staging area
          mbar_arrive_expect_tx(&xbar[warp - 2], 8192u);
          const int xr0 = mb * 256 + rank * 128 + q * 32, xc0 = nb * TN + h * kHN;
          tma_load_2d(stg, &p.tx, &xbar[warp - 2], xc0, xr0);
          tma_load_2d(stg + 4096, &p.tx, &xbar[warp - 2], xc0 + 64, xr0);
        }
      }
      if (lane == 0) mbar_wait(&acc_full[buf], use & 1u, 3);
      __syncwarp();
      tc_fence_after();
      if (CASTX && et == 0) *ep_tile = j;  // (the cast warps pace themselves on this)
      uint64_t* tr = (p.trace && j < 64 && et == 0) ? p.trace + ((size_t)blockIdx.x * 64 + j) * 8 : nullptr;
      if (tr) tr[0] = globaltimer_ns();

      const int grow = mb * 256 + rank * 128 + r;
      const bool row_ok = grow < p.M;
      // (CASTX: X's scale from the amax itself — p.sa is written by another CTA's cast warps)
      const float sa = !row_ok ? 0.f : CASTX ? sa_castx : __ldg(p.sa + (p.sa_row ? grow : 0));
      const float cfold = fold ? __fmul_rn(sa, __ldg(p.sb)) : 1.f;  // y = acc * cfold when folding
      const float2 sa2 = make_float2(sa, sa);
      const int col0 = nb * TN + h * kHN;  // first column of this thread
      const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * 256 + h * kHN);
      const uint32_t cs = smem_u32(colp + h * kHN);
      // y = acc * (s_a s_b[n]) + bias[n] for one 32-column chunk (identical instructions in both passes)
      auto dequant = [&](float (&y)[32], int cb) {
#pragma unroll
        for (int c = 0; c < 32; c += 4) {
          const float4 s4 = lds_f4(cs + 4u * (cb + c)), b4 = lds_f4(cs + 4u * TN + 4u * (cb + c));
          const float2 a = fadd2(fmul2(make_float2(y[c], y[c + 1]), fmul2(sa2, make_float2(s4.x, s4.y))),
                                 make_float2(b4.x, b4.y));
          const float2 b = fadd2(fmul2(make_float2(y[c + 2], y[c + 3]), fmul2(sa2, make_float2(s4.z, s4.w))),
                                 make_float2(b4.z, b4.w));
          y[c] = a.x; y[c + 1] = a.y; y[c + 2] = b.x; y[c + 3] = b.y;
        }
      };
      // backward: g = dh * act'(xhat gamma + beta) * gamma for one chunk (y: dequantized dh in, g out), and
      // the chunk's saved xhat values (bf16, global) into xv
      auto load_g = [&](float (&y)[32], int cb, float (&xv)[32]) {
        if (xs_stage) {  // from the staged SW128 box (cb / 64), 16-B pieces (cb % 64) / 8 .. + 3 of row `lane`
          const uint32_t base = smem_u32(stg) + (uint32_t)(cb / 64) * 4096u + (uint32_t)lane * 128u;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const uint32_t pc = ((uint32_t)((cb % 64) / 8 + u)) ^ ((uint32_t)lane & 7u);
            uint4 w;
            asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(w.x), "=r"(w.y), "=r"(w.z), "=r"(w.w)
                         : "r"(base + (pc << 4)));
            xv[8 * u + 0] = bf16lo_to_f32(w.x); xv[8 * u + 1] = bf16hi_to_f32(w.x);
            xv[8 * u + 2] = bf16lo_to_f32(w.y); xv[8 * u + 3] = bf16hi_to_f32(w.y);
            xv[8 * u + 4] = bf16lo_to_f32(w.z); xv[8 * u + 5] = bf16hi_to_f32(w.z);
            xv[8 * u + 6] = bf16lo_to_f32(w.w); xv[8 * u + 7] = bf16hi_to_f32(w.w);
          }
        } else if (row_ok) {
          const uint4* src = reinterpret_cast<const uint4*>(p.xhat + (int64_t)grow * p.ld_xhat + col0 + cb);
          uint4 w[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) w[u] = (col0 + cb + 8 * u < p.N) ? __ldg(src + u) : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            xv[8 * u + 0] = bf16lo_to_f32(w[u].x); xv[8 * u + 1] = bf16hi_to_f32(w[u].x);
            xv[8 * u + 2] = bf16lo_to_f32(w[u].y); xv[8 * u + 3] = bf16hi_to_f32(w[u].y);
            xv[8 * u + 4] = bf16lo_to_f32(w[u].z); xv[8 * u + 5] = bf16hi_to_f32(w[u].z);
            xv[8 * u + 6] = bf16lo_to_f32(w[u].w); xv[8 * u + 7] = bf16hi_to_f32(w[u].w);
          }
        } else {
#pragma unroll
          for (int k = 0; k < 32; ++k) xv[k] = 0.f;
        }
        if (has_gb || act) {
#pragma unroll
          for (int k = 0; k < 32; ++k) {
            const float ga = colp[2 * TN + h * kHN + cb + k], be = colp[3 * TN + h * kHN + cb + k];
            float g = y[k];
            if (act) {  // h-swish' at u = xhat gamma + beta (PyTorch at the kinks: 0 below -3, 1 above 3)
              const float u = fmaf(xv[k], ga, be);
              g = g * (u < -3.f ? 0.f : (u > 3.f ? 1.f : __fdiv_rn(fmaf(2.f, u, 3.f), 6.f)));
            }
            y[k] = g * ga;
          }
        }
      };
      // both passes stream the thread's kHN columns out of TMEM in 32-column chunks, the next chunk's
      // tcgen05.ld in flight while the current one is processed (two register buffers)
      auto stream_tmem = [&](auto&& fn, bool release) {
        float ya[32], yb[32];
        tmem_ld32_nowait(tbase, ya);
        tmem_wait32(ya);
#pragma unroll 1
        for (int c = 0; c < kNch; c += 2) {
          tmem_ld32_nowait(tbase + (uint32_t)(32 * (c + 1)), yb);
          fn(ya, c);
          tmem_wait32(yb);
          if (c + 2 < kNch) {
            tmem_ld32_nowait(tbase + (uint32_t)(32 * (c + 2)), ya);
          } else if (release) {  // the whole accumulator is in registers: hand it back to the MMA
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(acc_empty0 + 8u * buf);
          }
          fn(yb, c + 1);
          if (c + 2 < kNch) tmem_wait32(ya);
        }
      };

      // ---- pass S: this thread's statistics over its kHN columns (of acc when folding, else y) ----
      // Columns >= N hold exact zeros (zero-filled B rows, s_b = bias = 0): sums need no mask,
      // the LayerNorm chunk M2 is corrected for them and max / min skip them.
      float ss = 0.f, ymax = -INFINITY, ymin = INFINITY;
      float mean = 0.f, m2 = 0.f, nacc = 0.f;
      float sg = 0.f, sgx = 0.f;  // backward: sum g, sum g xhat
      auto stats_chunk = [&](float (&y)[32], int c) {
        const int cb = 32 * c;
        const int nv = max(0, min(32, p.N - (col0 + cb)));
        if (!fold) dequant(y, cb);
        if constexpr (BWD) {  // (columns >= N: dh = 0 and xhat = 0)
          float xv[32];
          load_g(y, cb, xv);
          float2 a0 = make_float2(0.f, 0.f), a1 = a0;
#pragma unroll
          for (int k = 0; k < 32; k += 4) {
            a0 = ffma2(make_float2(y[k], y[k + 1]), make_float2(xv[k], xv[k + 1]), a0);
            a1 = ffma2(make_float2(y[k + 2], y[k + 3]), make_float2(xv[k + 2], xv[k + 3]), a1);
          }
          a0 = fadd2(a0, a1);
          sgx += a0.x + a0.y;
          if constexpr (NORM == LOKA_NORM_LAYER) {
            float t = 0.f;
#pragma unroll
            for (int k = 0; k < 32; ++k) t += y[k];
            sg += t;
          }
          return;
        }
        if (nv > 0 && fp8_out) {
          if (nv == 32) {
#pragma unroll
            for (int k = 0; k < 32; k += 2) ymax = fmax3(ymax, y[k], y[k + 1]), ymin = fmin3(ymin, y[k], y[k + 1]);
          } else {
#pragma unroll
            for (int k = 0; k < 32; ++k)
              if (k < nv) ymax = fmaxf(ymax, y[k]), ymin = fminf(ymin, y[k]);
          }
        }
        if constexpr (NORM == LOKA_NORM_LAYER) {
          float2 s0 = make_float2(0.f, 0.f), s1 = s0, s2 = s0, s3 = s0;
#pragma unroll
          for (int k = 0; k < 32; k += 8) {
            s0 = fadd2(s0, make_float2(y[k], y[k + 1]));
            s1 = fadd2(s1, make_float2(y[k + 2], y[k + 3]));
            s2 = fadd2(s2, make_float2(y[k + 4], y[k + 5]));
            s3 = fadd2(s3, make_float2(y[k + 6], y[k + 7]));
          }
          s0 = fadd2(fadd2(s0, s1), fadd2(s2, s3));
          const float mc = nv > 0 ? (s0.x + s0.y) / (float)nv : 0.f;
          const float2 nm = make_float2(-mc, -mc);
          float2 q0 = make_float2(0.f, 0.f), q1 = q0;
#pragma unroll
          for (int k = 0; k < 32; k += 4) {
            const float2 d0 = fadd2(make_float2(y[k], y[k + 1]), nm);
            const float2 d1 = fadd2(make_float2(y[k + 2], y[k + 3]), nm);
            q0 = ffma2(d0, d0, q0);
            q1 = ffma2(d1, d1, q1);
          }
          q0 = fadd2(q0, q1);
          float mc2 = q0.x + q0.y;
          if (nv < 32) mc2 = nv > 0 ? fmaxf(0.f, mc2 - (float)(32 - nv) * mc * mc) : 0.f;
          if (nv > 0) {  // Chan's pairwise update: (nacc, mean, m2) += (nv, mc, mc2)
            const float nn = nacc + (float)nv;
            const float d = mc - mean;
            const float f = __fdiv_rn((float)nv, nn);
            mean = fmaf(d, f, mean);
            m2 += mc2 + d * d * nacc * f;
            nacc = nn;
          }
        } else {
          float2 q0 = make_float2(0.f, 0.f), q1 = q0;
#pragma unroll
          for (int k = 0; k < 32; k += 4) {
            const float2 a = make_float2(y[k], y[k + 1]), b = make_float2(y[k + 2], y[k + 3]);
            q0 = ffma2(a, a, q0);
            q1 = ffma2(b, b, q1);
          }
          q0 = fadd2(q0, q1);
          ss += q0.x + q0.y;
        }
      };
      if constexpr (BWD) {
        if (xs_stage) {
          if (lane == 0) mbar_wait(&xbar[warp - 2], xph, 8);
          xph ^= 1u;
          __syncwarp();
        }
      }
      if (!(p.dbg & 2)) stream_tmem(stats_chunk, false);
      if (tr) tr[1] = globaltimer_ns();
      if (fold) {  // back to y = c acc (the statistics of y)
        mean = __fmul_rn(mean, cfold);
        m2 = __fmul_rn(m2, __fmul_rn(cfold, cfold));
        ss = __fmul_rn(ss, __fmul_rn(cfold, cfold));
      }

      // ---- the two halves of the row (fixed order h = 0, 1), then the Case 2 exchange ----
      hrec[h * 128 + r] = bwd ? make_float4(sg, sgx, 0.f, 0.f)
                              : make_float4(NORM == LOKA_NORM_LAYER ? mean : ss, m2, ymax, ymin);
      named_bar_sync(1, 32 * kPnEpiWarps);
      // z = y rstd + c0; with folding z = acc (c rstd) + c0 and ymax / ymin are of acc
      float rstd = 1.f, c0 = 0.f, amax = 0.f;
      const float sc = fold ? cfold : 1.f;
      {
        const float4 v0 = hrec[r], v1 = hrec[128 + r];
        const int n0 = max(0, min(kHN, p.N - nb * TN)), n1 = max(0, min(kHN, p.N - nb * TN - kHN));
        float4 cr;  // this CTA's record of the row: (mean | ss, M2, ymax, ymin); backward (sum g, sum g xhat)
        if (bwd) {
          cr = (NORM == LOKA_NORM_BLOCK_RMS && TN == 512) ? (h ? v1 : v0)
                                                            : make_float4(v0.x + v1.x, v0.y + v1.y, 0.f, 0.f);
        } else if constexpr (NORM == LOKA_NORM_LAYER) {
          const float n = (float)(n0 + n1);
          const float mu = n > 0.f ? __fdiv_rn(fmaf((float)n0, v0.x, (float)n1 * v1.x), n) : 0.f;
          const float d0 = v0.x - mu, d1 = v1.x - mu;
          cr = make_float4(mu, v0.y + (float)n0 * d0 * d0 + (v1.y + (float)n1 * d1 * d1), fmaxf(v0.z, v1.z),
                           fminf(v0.w, v1.w));
        } else if constexpr (NORM == LOKA_NORM_RMS) {
          cr = make_float4(v0.x + v1.x, 0.f, fmaxf(v0.z, v1.z), fminf(v0.w, v1.w));
        } else {  // BlockNorm-256: TN = 512 -> each half is one block; TN = 256 -> the two halves are
          const float ssb = TN == 512 ? (h ? v1.x : v0.x) : v0.x + v1.x;
          rstd = __fdiv_rn(1.f, __fsqrt_rn(__fadd_rn(__fdiv_rn(ssb, 256.f), p.eps)));
          if (fp8_out) {  // the row amax candidate of this CTA's blocks (max |stored value| per block)
            if (TN == 512) {
              const float r0 = __fmul_rn(sc, __fdiv_rn(1.f, __fsqrt_rn(__fadd_rn(__fdiv_rn(v0.x, 256.f), p.eps))));
              const float r1 = __fmul_rn(sc, __fdiv_rn(1.f, __fsqrt_rn(__fadd_rn(__fdiv_rn(v1.x, 256.f), p.eps))));
              amax = fmaxf(n0 > 0 ? fmaxf(fabsf(fmaf(v0.z, r0, 0.f)), fabsf(fmaf(v0.w, r0, 0.f))) : 0.f,
                           n1 > 0 ? fmaxf(fabsf(fmaf(v1.z, r1, 0.f)), fabsf(fmaf(v1.w, r1, 0.f))) : 0.f);
            } else {
              const float rs = __fmul_rn(sc, rstd);
              amax = (n0 + n1) > 0 ? fmaxf(fabsf(fmaf(fmaxf(v0.z, v1.z), rs, 0.f)), fabsf(fmaf(fminf(v0.w, v1.w), rs, 0.f)))
                                   : 0.f;
            }
          }
          cr = make_float4(0.f, 0.f, amax, 0.f);
        }
        if (need_x) {
          // publish this CTA's record of row r: one float4 store, waited for element-wise by readers
          const size_t rb = (size_t)mb * G * 2 + rank;  // record of tile k, row i: xrec[(rb + 2 k) * 128 + i]
          if (h == 0) xrec[(rb + 2 * nb) * 128 + r] = cr;
          if (tr) tr[7] = globaltimer_ns();
          // each column half of the row's threads loads half of the G records (all loads in flight),
          // merges them in tile order; the two partial records meet in smem (order h = 0, 1)
          const int kb0 = h ? (G + 1) / 2 : 0, kb1 = h ? G : (G + 1) / 2;
          float n = 0.f, sm = 0.f, mx = -INFINITY, mn = INFINITY;
          float4 v[8];
          auto load8 = [&](int k0) {
#pragma unroll
            for (int u = 0; u < 8; ++u)
              if (k0 + u < kb1)
                v[u] = (p.dbg & 1) ? make_float4(0.f, 0.f, 0.f, 0.f) : ld_relaxed_f4(xrec + (rb + 2 * (k0 + u)) * 128 + r);
#pragma unroll
            for (int u = 0; u < 8; ++u)
              if (k0 + u < kb1 && rec_pending(v[u])) v[u] = rec_wait(xrec + (rb + 2 * (k0 + u)) * 128 + r);
          };
          float sy = 0.f;  // backward: sum of the records' sum g xhat
          for (int k0 = kb0; k0 < kb1; k0 += 8) {  // sum n_k mean_k (LayerNorm) | sum ss_k; max / min
            load8(k0);
#pragma unroll
            for (int u = 0; u < 8; ++u)
              if (k0 + u < kb1) {
                const float nk = (float)max(0, min(TN, p.N - (k0 + u) * TN));
                n += nk;
                sm = (NORM == LOKA_NORM_LAYER && !bwd) ? fmaf(nk, v[u].x, sm) : sm + v[u].x;
                sy += v[u].y;
                mx = fmaxf(mx, v[u].z);
                mn = fminf(mn, v[u].w);
              }
          }
          float pm = sm, pm2 = bwd ? sy : 0.f;  // LayerNorm: this half's (mean, M2) of its tiles
          if (NORM == LOKA_NORM_LAYER && !bwd) {
            pm = n > 0.f ? __fdiv_rn(sm, n) : 0.f;
            for (int k0 = kb0; k0 < kb1; k0 += 8) {
              if (kb1 - kb0 > 8) load8(k0);  // (more than 8 tiles per half, G > 16: load again)
#pragma unroll
              for (int u = 0; u < 8; ++u)
                if (k0 + u < kb1) {
                  const float nk = (float)max(0, min(TN, p.N - (k0 + u) * TN));
                  const float dk = v[u].x - pm;
                  pm2 += v[u].y + nk * dk * dk;
                }
            }
          }
          named_bar_sync(1, 32 * kPnEpiWarps);  // the halves' hrec reads above are done
          hrec[h * 128 + r] = make_float4(pm, pm2, mx, mn);
          named_bar_sync(1, 32 * kPnEpiWarps);
          const float4 a0 = hrec[r], a1 = hrec[128 + r];
          if (bwd) {
            cr = make_float4(a0.x + a1.x, a0.y + a1.y, 0.f, 0.f);
          } else if constexpr (NORM == LOKA_NORM_LAYER) {
            const float na = (float)min((G + 1) / 2 * TN, p.N), nbb = (float)p.N - na;
            const float mu = __fdiv_rn(fmaf(na, a0.x, nbb * a1.x), (float)p.N);
            const float d0 = a0.x - mu, d1 = a1.x - mu;
            cr = make_float4(mu, a0.y + na * d0 * d0 + (a1.y + nbb * d1 * d1), fmaxf(a0.z, a1.z), fminf(a0.w, a1.w));
          } else if constexpr (NORM == LOKA_NORM_RMS) {
            cr = make_float4(a0.x + a1.x, 0.f, fmaxf(a0.z, a1.z), fminf(a0.w, a1.w));
          } else {
            cr = make_float4(0.f, 0.f, fmaxf(a0.z, a1.z), 0.f);
          }
        }
        named_bar_sync(1, 32 * kPnEpiWarps);  // hrec reads done before the next tile's writes
        const float nrow = (float)p.N;
        if (bwd) {  // mean(g) (LayerNorm), mean(g xhat) over the row (BlockNorm: its 256-column block)
          const float nb = NORM == LOKA_NORM_BLOCK_RMS ? 256.f : nrow;
          c0 = NORM == LOKA_NORM_LAYER ? __fdiv_rn(cr.x, nb) : 0.f;
          amax = __fdiv_rn(cr.y, nb);  // (mean(g xhat), kept in amax's register)
          rstd = row_ok ? (NORM == LOKA_NORM_BLOCK_RMS ? __ldg(p.rstd_in + (int64_t)grow * (p.N / 256) + (col0 / 256))
                                                       : __ldg(p.rstd_in + grow))
                        : 0.f;
        } else if constexpr (NORM == LOKA_NORM_LAYER) {
          rstd = __fdiv_rn(1.f, __fsqrt_rn(__fadd_rn(__fdiv_rn(cr.y, nrow), p.eps)));
          c0 = -__fmul_rn(cr.x, rstd);
        } else if constexpr (NORM == LOKA_NORM_RMS) {
          rstd = __fdiv_rn(1.f, __fsqrt_rn(__fadd_rn(__fdiv_rn(cr.x, nrow), p.eps)));
        }
        if (bwd) {
        } else if constexpr (NORM != LOKA_NORM_BLOCK_RMS) {
          if (fp8_out) {  // the stored values are fma(y_or_acc, rs, c0): monotone, exact at ymax / ymin
            const float rs = __fmul_rn(sc, rstd);
            amax = fmaxf(fabsf(fmaf(cr.z, rs, c0)), fabsf(fmaf(cr.w, rs, c0)));
          }
        } else {
          if (fp8_out) amax = cr.z;
        }
      }
      if (tr) tr[2] = globaltimer_ns();
      const float mgx_keep = amax;  // backward: mean(g xhat) (the forward never reads it)
      // backward with FP8 dz (1x128 granules, TN = 256): this thread's 128 columns are one granule; an
      // extra TMEM pass computes dz exactly as pass N will (the same non-contracted operations) and
      // keeps max |dz| — the granule's scale must exist before the cast
      float dz_amax = 0.f;
      if constexpr (BWD) {
        if (fp8_out) {
          auto amax_chunk = [&](float (&y)[32], int c) {
            const int cb = 32 * c;
            if (!fold) dequant(y, cb);
            float xv[32];
            load_g(y, cb, xv);
            const int nv = max(0, min(32, p.N - (col0 + cb)));
#pragma unroll
            for (int k = 0; k < 32; ++k)
              if (k < nv) dz_amax = fmaxf(dz_amax, fabsf(__fmul_rn(rstd, __fsub_rn(__fsub_rn(y[k], c0), __fmul_rn(xv[k], amax)))));
          };
          stream_tmem(amax_chunk, false);
        }
      }
      float r_out = 1.f;
      if (fp8_out) {
        if (bwd) amax = dz_amax;  // (amax carried mean(g xhat) so far; pass N gets it from mgx below)
        // 1x128 scales (TN = 256): this thread's 128 columns are one granule; its amax comes from the
        // thread's own y max / min of pass S through the same monotone map as the row amax
        if (TN == 256 && !bwd && p.y_blk)
          amax = col0 < p.N ? fmaxf(fabsf(fmaf(ymax, __fmul_rn(sc, rstd), c0)), fabsf(fmaf(ymin, __fmul_rn(sc, rstd), c0)))
                            : 0.f;
        if (__float_as_uint(amax) >= 0x7F800000u && p.status) atomicOr(p.status, LOKA_DEVSTATUS_NONFINITE);
        float s_out;
        if (p.out_dtype == LOKA_E4M3) scales_from_amax<LOKA_E4M3, LOKA_SCALE_F32>(amax, s_out, r_out);
        else scales_from_amax<LOKA_E5M2, LOKA_SCALE_F32>(amax, s_out, r_out);
        if (p.y_blk) {
          if (row_ok && col0 < p.N && p.y_scales) p.y_scales[(int64_t)grow * ((p.N + 127) / 128) + col0 / 128] = s_out;
        } else if (row_ok && nb == 0 && h == 0 && p.y_scales) {
          p.y_scales[grow] = s_out;
        }
      }

      // ---- pass N: normalise, activation, cast, store ----
      const float rs = __fmul_rn(sc, rstd);
      const float2 r2 = make_float2(rs, rs), c02 = make_float2(c0, c0);
      float amx = 0.f;
      const float mgx = bwd ? mgx_keep : 0.f;
      auto out_chunk = [&](float (&y)[32], int c) {
        const int cb = 32 * c;
        if (!fold) dequant(y, cb);
        if constexpr (BWD) {  // dz = rstd (g - mean(g) - xhat mean(g xhat))
          float xv[32];
          load_g(y, cb, xv);
#pragma unroll
          for (int k = 0; k < 32; ++k) y[k] = __fmul_rn(rstd, __fsub_rn(__fsub_rn(y[k], c0), __fmul_rn(xv[k], mgx)));
        } else {
#pragma unroll
        for (int k = 0; k < 32; k += 4) {
          float2 a = ffma2(make_float2(y[k], y[k + 1]), r2, c02);
          float2 b = ffma2(make_float2(y[k + 2], y[k + 3]), r2, c02);
          if (has_gb) {
            const uint32_t o = cs + 2u * TN * 4u + 4u * (cb + k);
            const float4 g4 = lds_f4(o), e4 = lds_f4(o + TN * 4u);
            a = ffma2(a, make_float2(g4.x, g4.y), make_float2(e4.x, e4.y));
            b = ffma2(b, make_float2(g4.z, g4.w), make_float2(e4.z, e4.w));
          }
          y[k] = a.x; y[k + 1] = a.y; y[k + 2] = b.x; y[k + 3] = b.y;
        }
        if (act) {
#pragma unroll
          for (int k = 0; k < 32; ++k) y[k] = hswish(y[k]);
        }
        }
        const int nv = max(0, min(32, p.N - (col0 + cb)));
        if (p.amax_out && row_ok) {
#pragma unroll
          for (int k = 0; k < 32; ++k)
            if (k < nv) amx = fmaxf(amx, fabsf(esz == 2 ? stored_bf16(y[k]) : y[k]));
        }
        if (p.precast && row_ok) {
          float* dst = p.precast + (int64_t)grow * p.ld_pre + col0 + cb;
#pragma unroll
          for (int k = 0; k < 32; ++k)
            if (k < nv) dst[k] = y[k];
        }
        const int in_box = cb % cpb;
        // (backward with staged xhat: 2 bf16 boxes per tile, so box (nbox & 1) == cb / 64 and each chunk's
        // dz overwrites exactly its own, already consumed, xhat pieces of this lane's row)
        uint8_t* box = stg + (xs_stage ? (cb / 64) : (nbox & 1)) * 4096;
        if (in_box == 0 && !xs_stage) {  // this buffer's previous store (two boxes ago) must have been read
          if (lane == 0) bulk_wait_read_le1();
          __syncwarp();
        }
        const uint32_t rowa = smem_u32(box) + (uint32_t)lane * 128u;
        if (esz == 4) {
#pragma unroll
          for (int k = 0; k < 8; ++k)
            sts_u4(rowa + ((((uint32_t)k) ^ ((uint32_t)lane & 7u)) << 4),
                   make_uint4(__float_as_uint(y[4 * k]), __float_as_uint(y[4 * k + 1]), __float_as_uint(y[4 * k + 2]),
                              __float_as_uint(y[4 * k + 3])));
        } else if (esz == 2) {
          const uint32_t p0 = (uint32_t)(in_box * 2) >> 4;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            uint32_t w[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              __nv_bfloat162 hh = __floats2bfloat162_rn(y[8 * k + 2 * i], y[8 * k + 2 * i + 1]);
              w[i] = *reinterpret_cast<uint32_t*>(&hh);
            }
            sts_u4(rowa + (((p0 + (uint32_t)k) ^ ((uint32_t)lane & 7u)) << 4), make_uint4(w[0], w[1], w[2], w[3]));
          }
        } else {
          const uint32_t p0 = (uint32_t)in_box >> 4;
          const float2 rr = make_float2(r_out, r_out);
#pragma unroll
          for (int k = 0; k < 2; ++k) {
            uint32_t w[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int e = 16 * k + 4 * i;
              const float2 a = fmul2(make_float2(y[e], y[e + 1]), rr);
              const float2 b = fmul2(make_float2(y[e + 2], y[e + 3]), rr);
              w[i] = p.out_dtype == LOKA_E4M3 ? cvt_fp8x4<LOKA_E4M3>(a.x, a.y, b.x, b.y)
                                              : cvt_fp8x4<LOKA_E5M2>(a.x, a.y, b.x, b.y);
            }
            sts_u4(rowa + (((p0 + (uint32_t)k) ^ ((uint32_t)lane & 7u)) << 4), make_uint4(w[0], w[1], w[2], w[3]));
          }
        }
        if (in_box + 32 == cpb) {  // box complete: store it
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            const int cbox = col0 + cb + 32 - cpb;
            const int row0 = mb * 256 + rank * 128 + q * 32;
            if (cbox < p.N && row0 < p.M) tma_store_2d(&p.ty, box, cbox, row0);
            bulk_commit();
          }
          ++nbox;
        }
      };
      stream_tmem(out_chunk, true);
      if (tr) tr[3] = globaltimer_ns();
      if (p.amax_out) warp_amax_to(p.amax_out, amx);
    }
    if (lane == 0) bulk_wait0();
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_cg2<512>(tmem_base);
  }
}

template <int TN, int NORM, bool BF16IN, bool BWD = false, bool CASTX = false>
static cudaError_t launch_pn(const PairNormParams& p_in, int pairs, cudaStream_t st) {
  auto kern = pair_norm_kernel<TN, NORM, BF16IN, BWD, CASTX>;
  {
    cudaError_t e = ensure_func_attrs(reinterpret_cast<const void*>(kern), PnCfg<TN>::kSmem);
    if (e != cudaSuccess) return e;
  }
  PairNormParams p = p_in;
  if (p.mc) {  // 4-CTA clusters: only as many as are co-resident (the record exchange needs every pair resident)
    if (TN != 256 || p.order != 0 || CASTX || (p.tiles_n & 1)) {
      p.mc = 0;
    } else {
      static int max_clusters = -1;  // per instance (one device type per process)
      if (max_clusters < 0) {
        cudaLaunchConfig_t q = {};
        q.gridDim = dim3(4 * 64, 1, 1);
        q.blockDim = dim3(kPnThreads + (CASTX ? 32 * kPnCastWarps : 0), 1, 1);
        q.dynamicSmemBytes = PnCfg<TN>::kSmem;
        cudaLaunchAttribute qa[1];
        qa[0].id = cudaLaunchAttributeClusterDimension;
        qa[0].val.clusterDim.x = 4;
        qa[0].val.clusterDim.y = 1;
        qa[0].val.clusterDim.z = 1;
        q.attrs = qa;
        q.numAttrs = 1;
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, kern, &q) != cudaSuccess) n = 0;
        max_clusters = n;
      }
      const int np = std::min(pairs, 2 * max_clusters) & ~1;
      if (np < 2) p.mc = 0;
      else pairs = np;
    }
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(2 * pairs), 1, 1);
  cfg.blockDim = dim3(kPnThreads + (CASTX ? 32 * kPnCastWarps : 0), 1, 1);
  cfg.dynamicSmemBytes = PnCfg<TN>::kSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = p.mc ? 4 : 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, p);
  note_launch();
  return e;
}

template <int TN>
static cudaError_t launch_pn_norm(const PairNormParams& p, int pairs, cudaStream_t st) {
  switch (p.norm) {
    case LOKA_NORM_LAYER: return launch_pn<TN, LOKA_NORM_LAYER, false>(p, pairs, st);
    case LOKA_NORM_RMS: return launch_pn<TN, LOKA_NORM_RMS, false>(p, pairs, st);
    case LOKA_NORM_BLOCK_RMS: return launch_pn<TN, LOKA_NORM_BLOCK_RMS, false>(p, pairs, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_pair_norm(const PairNormParams& p, int tn, int pairs, cudaStream_t st) {
  if (p.castx) {  // (256-wide tiles, FP8, forward)
    switch (p.norm) {
      case LOKA_NORM_LAYER: return launch_pn<256, LOKA_NORM_LAYER, false, false, true>(p, pairs, st);
      case LOKA_NORM_RMS: return launch_pn<256, LOKA_NORM_RMS, false, false, true>(p, pairs, st);
      case LOKA_NORM_BLOCK_RMS: return launch_pn<256, LOKA_NORM_BLOCK_RMS, false, false, true>(p, pairs, st);
      default: return cudaErrorInvalidValue;
    }
  }
  if (p.bwd) {  // (256-wide tiles, FP8 operands)
    switch (p.norm) {
      case LOKA_NORM_LAYER: return launch_pn<256, LOKA_NORM_LAYER, false, true>(p, pairs, st);
      case LOKA_NORM_RMS: return launch_pn<256, LOKA_NORM_RMS, false, true>(p, pairs, st);
      case LOKA_NORM_BLOCK_RMS: return launch_pn<256, LOKA_NORM_BLOCK_RMS, false, true>(p, pairs, st);
      default: return cudaErrorInvalidValue;
    }
  }
  if (p.bf16_in) {  // (256-wide tiles only)
    switch (p.norm) {
      case LOKA_NORM_LAYER: return launch_pn<256, LOKA_NORM_LAYER, true>(p, pairs, st);
      case LOKA_NORM_RMS: return launch_pn<256, LOKA_NORM_RMS, true>(p, pairs, st);
      case LOKA_NORM_BLOCK_RMS: return launch_pn<256, LOKA_NORM_BLOCK_RMS, true>(p, pairs, st);
      default: return cudaErrorInvalidValue;
    }
  }
  return tn == 512 ? launch_pn_norm<512>(p, pairs, st) : launch_pn_norm<256>(p, pairs, st);
}

__device__ const float g_pn_one = 1.0f;  // the unit scale of the BF16 path
const float* pair_norm_unit_scale() {
  void* a = nullptr;
  return cudaGetSymbolAddress(&a, g_pn_one) == cudaSuccess ? static_cast<const float*>(a) : nullptr;
}

}  // namespace loka
