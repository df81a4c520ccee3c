// gemm2.cu — a4/a6 on CTA pairs: persistent FP8 GEMM with 256 x 256 tiles computed by ONE
// tcgen05.mma.cta_group::2 per 32-wide K step across the two SMs of a 2-CTA cluster.
//
// Why: a 128 x 128 (or 128 x 256) single-CTA tile needs 32 KB (48 KB) of
// operands per 128-K stage for 4.2 (8.4) MFLOP, i.e. ~19-25 TB/s of L2 -> SM traffic chip-wide at
// the tensor-core rate — more than L2 delivers, so the many-small-GEMM mix (BJ configs[2])
// and the big training GEMMs (configs[3]) were L2-bound.  A CTA pair computes a 256 x 256 tile:
// each CTA stages its 128 rows of A and HALF of the 256 rows of B (32 KB per stage per SM for
// 16.8 MFLOP per pair), halving the traffic per FLOP of the 128 x 256 tile.
//
//   * cluster (2,1,1); rank 0 is the leader.  Both CTAs' producers (warp 0 lane 0) TMA-load their
//     halves with .cta_group::2 loads whose transaction bytes land on the LEADER's full barrier;
//     the leader's MMA thread (warp 1 lane 0) issues the M=256, N=256 MMAs and commits with
//     .multicast::cluster to the empty barriers of both CTAs (stage free in both).
//   * Each CTA's TMEM holds its 128 rows x 256 columns; two accumulator buffers (all 512 columns)
//     let the MMAs of tile j+1 run while the epilogue drains tile j.  The 8 epilogue warps of both
//     CTAs (16 arrivals) release a buffer on the leader's acc_empty barrier.
//   * Epilogue per warp: 32 rows (its TMEM lane quadrant) x 128 columns in 32-column chunks:
//     y = acc * s_a[m] * s_b[n] (+ bias[n]) -> bf16 / f32 into a per-warp double-buffered
//     32-row x 128-byte swizzled box -> TMA store (no CTA-wide barrier in the epilogue).
//   * Persistent: pair c walks tiles c, c + #pairs, ... of the concatenated tile list of up to
//     kMaxGroups GEMMs (longest K first, host order), tile = (256-row block, 256-col block).
#include "common.cuh"
#include "launch.h"

namespace loka {

constexpr int k2Stages = 4;
constexpr int k2EpiWarps = 8;
constexpr int k2Threads = 64 + 32 * k2EpiWarps;
constexpr int k2StageA = 128 * 128, k2StageB = 128 * 128;  // per CTA: 128 rows x 128 K each
constexpr int k2OffB = k2Stages * k2StageA;
constexpr int k2OffOut = k2OffB + k2Stages * k2StageB;       // [8 warps][2][32 rows x 128 B]
constexpr int k2OffCol = k2OffOut + k2EpiWarps * 2 * 4096;  // [2 tiles][s_b | bias][256] FP32
constexpr int k2OffBar = k2OffCol + 2 * 2 * 256 * 4;
constexpr int k2Smem = k2OffBar + 256 + 1024;
static_assert(k2Smem <= 227 * 1024, "gemm2 smem");

// WIDE: 256 x 512 pair tiles — two N = 256 MMAs per K step share the A stage, so a pair moves
// 96 KB of operands per 33.6 MFLOP instead of 64 KB per 16.8 MFLOP: 25% fewer bytes per FLOP
// through each SM's L2 -> SM port (~40 B/clk, the bound of the 256 x 256 tile at ~80% of the MMA
// rate).  All 512 TMEM columns hold one accumulator (no overlap of a tile's epilogue with the next
// tile's MMAs), so WIDE is for long-K work units (split-K slices of the paper's largest layer).
template <bool WIDE>
struct G2 {
  static constexpr int kTN = WIDE ? 512 : 256;  // tile columns
  static constexpr int kStages = WIDE ? 3 : 4;
  static constexpr int kStageA = 128 * 128;
  static constexpr int kStageB = (WIDE ? 256 : 128) * 128;  // per CTA: 128 rows of each 256-col half
  static constexpr int kOffB = kStages * kStageA;
  static constexpr int kOffOut = kOffB + kStages * kStageB;
  static constexpr int kOffCol = kOffOut + k2EpiWarps * 2 * 4096;  // [2 tiles][s_b | bias][kTN] FP32
  static constexpr int kOffBar = kOffCol + 2 * 2 * kTN * 4;
  static constexpr int kSmem = kOffBar + 256 + 1024;
};
static_assert(G2<true>::kSmem <= 227 * 1024 && G2<false>::kSmem == k2Smem, "gemm2 smem");

// BF16IN: BF16 operands (kind::f16; a 128-byte stage row holds 64 K elements) — the probe
// tracker's scatter GEMM (NEXT-2); otherwise FP8 (kind::f8f6f4, 128 K elements per row).
// SPLIT: the launch is one split-K problem (raw FP32 partials to gp.tp); a template parameter so the
// many-small-GEMM epilogue carries none of that code (it is epilogue-bound: ~1 K-block per tile).
template <bool BF16IN, bool WIDE, bool SPLIT>
__global__ void __launch_bounds__(k2Threads, 1) grouped2_kernel(const __grid_constant__ GroupedParams gp) {
  using C2 = G2<WIDE>;
  constexpr int kKE = BF16IN ? 64 : 128;  // K elements per 128-byte stage row
  constexpr int kTN = C2::kTN, kHN = kTN / 2;  // tile columns; columns per epilogue warp
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C2::kOffB;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + C2::kOffBar);
  uint64_t* empty_bar = full_bar + C2::kStages;
  uint64_t* acc_full = empty_bar + C2::kStages;  // [2]
  uint64_t* acc_empty = acc_full + 2;          // [2] (leader's is the one used)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rank = (int)cluster_ctarank();
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const int T = gp.tile_start[gp.G];

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < C2::kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 2 * k2EpiWarps);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_cg2<512>(tmem_slot);
  pdl_wait();
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // barriers of both CTAs initialised before any remote arrive / TMA
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  int ks = 0;
  auto locate = [&](int t, int& g, int& mb, int& nb) {  // binary search of the tile prefix sum
    int lo = 0, hi = gp.G - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (t >= gp.tile_start[mid]) lo = mid;
      else hi = mid - 1;
    }
    g = lo;
    int local = t - gp.tile_start[g];
    const int tn = gp.g[g].tiles_n;
    if constexpr (SPLIT) {
      const int per = ((gp.g[g].M + 255) / 256) * tn;  // tiles of one K slice
      ks = local / per;                                   // split-K slice
      local -= ks * per;
    }
    mb = local / tn;
    nb = local - mb * tn;
  };
  auto krange = [&](int g, int ks, int& kb0, int& kb1) {
    const int nkb = (gp.g[g].K + kKE - 1) / kKE;
    if (SPLIT) {
      kb0 = ks * gp.g[g].kb_per_split;
      kb1 = min(nkb, kb0 + gp.g[g].kb_per_split);
    } else {
      kb0 = 0;
      kb1 = nkb;
    }
  };

  if (warp == 0) {
    // ===== TMA producer (both CTAs): this CTA's A rows and half of the tile's B rows =====
    if (lane == 0) {
      const uint32_t full0 = mapa_shared(smem_u32(full_bar), 0);  // leader's full_bar[0]
      int it = 0;
      for (int t = cid; t < T; t += ncl) {
        int g, mb, nb;
        locate(t, g, mb, nb);
        int kb0, kb1;
        krange(g, ks, kb0, kb1);
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % C2::kStages;
          const uint32_t ph = (uint32_t)(it / C2::kStages) & 1u;
          mbar_wait(&empty_bar[s], ph ^ 1u, 1);
          if (rank == 0) mbar_arrive_expect_tx(&full_bar[s], 2u * (C2::kStageA + C2::kStageB));
          tma_load_2d_cg2(sA + s * C2::kStageA, &gp.ta[g], full0 + 8u * s, kb * kKE, mb * 256 + rank * 128);
#pragma unroll
          for (int hh = 0; hh < kTN / 256; ++hh)  // this CTA's 128 rows of each 256-column half
            tma_load_2d_cg2(sB + s * C2::kStageB + hh * 16384, &gp.tb[g], full0 + 8u * s, kb * kKE,
                            nb * kTN + hh * 256 + rank * 128);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ===== MMA issuer (leader only): tile j -> accumulator buffer j & 1 of both CTAs =====
    if (lane == 0 && rank == 0) {
      int it = 0, j = 0;
      for (int t = cid; t < T; t += ncl, ++j) {
        int g, mb, nb;
        locate(t, g, mb, nb);
        int kb0, kb1;
        krange(g, ks, kb0, kb1);
        const int buf = WIDE ? 0 : (j & 1);
        const uint32_t use = WIDE ? (uint32_t)j : (uint32_t)(j >> 1);  // earlier uses of this buffer
        mbar_wait(&acc_empty[buf], (use & 1u) ^ 1u, 4);  // both CTAs drained it
        tc_fence_after();
        const uint32_t idesc = BF16IN ? idesc_bf16(256, 256) : idesc_f8f6f4(gp.g[g].a_fmt, gp.g[g].b_fmt, 256, 256);
        const uint32_t dacc = tmem_base + (uint32_t)(buf * 256);
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % C2::kStages;
          const uint32_t ph = (uint32_t)(it / C2::kStages) & 1u;
          mbar_wait(&full_bar[s], ph, 2);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + s * C2::kStageA);
          const uint32_t b0 = smem_u32(sB + s * C2::kStageB);
#pragma unroll
          for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int hh = 0; hh < kTN / 256; ++hh) {  // WIDE: two N = 256 MMAs share the A stage
              const uint64_t da = smem_desc_kmajor_sw128(a0 + k * 32);
              const uint64_t db = smem_desc_kmajor_sw128(b0 + hh * 16384 + k * 32);
              if constexpr (BF16IN)
                mma_bf16_cg2(dacc + hh * 256, da, db, idesc, (kb > kb0 || k) ? 1u : 0u);
              else
                mma_f8f6f4_cg2(dacc + hh * 256, da, db, idesc, (kb > kb0 || k) ? 1u : 0u);
            }
          mma_commit_cg2_mc(&empty_bar[s], 3);
        }
        mma_commit_cg2_mc(&acc_full[buf], 3);
      }
    }
    __syncwarp();
  } else {
    // ===== epilogue (both CTAs): warp = TMEM lane quadrant q x column half h =====
    const int q = warp & 3;
    const int h = (warp - 2) >> 2;
    uint8_t* stg = smem + C2::kOffOut + (warp - 2) * 8192;
    const uint32_t acc_empty0 = mapa_shared(smem_u32(acc_empty), 0);
    int nbox = 0;
    int j = 0;
    for (int t = cid; t < T; t += ncl, ++j) {
      int g, mb, nb;
      locate(t, g, mb, nb);
      const GroupDesc& d = gp.g[g];
      const int buf = WIDE ? 0 : (j & 1);
      const uint32_t use = WIDE ? (uint32_t)j : (uint32_t)(j >> 1);
      // this tile's kTN column parameters -> smem (while the MMAs run); buffer j & 1 was last read
      // in tile j - 2, which every epilogue warp finished before the barrier of tile j - 1
      float* colp = reinterpret_cast<float*>(smem + C2::kOffCol) + (j & 1) * 2 * kTN;
      for (int e = threadIdx.x - 64; e < kTN; e += 32 * k2EpiWarps) {
        const int n = nb * kTN + e;
        const bool ok = n < d.N;
        colp[e] = ok ? __ldg(d.sb + (d.sb_row ? n : 0)) : 0.f;
        float b = 0.f;
        if (ok && d.bias) b = d.bias_bf16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(d.bias)[n])
                                          : reinterpret_cast<const float*>(d.bias)[n];
        colp[kTN + e] = b;
      }
      named_bar_sync(2, 32 * k2EpiWarps);
      if (lane == 0) mbar_wait(&acc_full[buf], use & 1u, 3);
      __syncwarp();
      tc_fence_after();
      const int row0 = mb * 256 + rank * 128 + q * 32;  // first row of this warp's box
      const int grow = row0 + lane;
      constexpr bool split = SPLIT;  // raw FP32 partial of K slice ks -> partial buffer
      const float sa = grow < d.M ? (split ? 1.f : d.sa[d.sa_row ? grow : 0]) : 0.f;
      const int esz = (split || d.out_dtype == LOKA_F32) ? 4 : 2;
      const int cpb = 128 / esz;  // columns per 128-byte box row
      const int col0 = nb * kTN + h * kHN;
      const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * 256 + h * kHN);
      float amx = 0.f;  // NEXT-4 producer amax of this warp's stored values
      // 32-column chunks streamed out of TMEM with the next chunk's load in flight (two buffers)
      auto chunk = [&](float (&y)[32], int cb) {
        const uint32_t cs = smem_u32(colp + h * kHN + cb);
        const float2 sa2 = make_float2(sa, sa);
        if (!split) {
#pragma unroll
          for (int c = 0; c < 32; c += 4) {  // y = acc * (s_a s_b) + bias, column params from smem
            const float4 s4 = lds_f4(cs + 4u * c), b4 = lds_f4(cs + 4u * kTN + 4u * c);
            const float2 a = fadd2(fmul2(make_float2(y[c], y[c + 1]), fmul2(sa2, make_float2(s4.x, s4.y))),
                                   make_float2(b4.x, b4.y));
            const float2 b = fadd2(fmul2(make_float2(y[c + 2], y[c + 3]), fmul2(sa2, make_float2(s4.z, s4.w))),
                                   make_float2(b4.z, b4.w));
            y[c] = a.x; y[c + 1] = a.y; y[c + 2] = b.x; y[c + 3] = b.y;
          }
        }
        if (d.amax_out && !split && grow < d.M) {
#pragma unroll
          for (int c = 0; c < 32; ++c)
            if (col0 + cb + c < d.N) amx = fmaxf(amx, fabsf(esz == 2 ? stored_bf16(y[c]) : y[c]));
        }
        const int in_box = cb % cpb;  // first column of this chunk inside its box
        uint8_t* box = stg + (nbox & 1) * 4096;
        if (in_box == 0) {  // the buffer's previous store (two boxes ago) must have been read
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
        } else {
          const uint32_t p0 = (uint32_t)(in_box * 2) >> 4;  // first 16-byte piece (0 or 4)
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
        }
        if (in_box + 32 == cpb) {  // box complete: store it
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            const int c0 = col0 + cb + 32 - cpb;
            if (c0 < d.N && row0 < d.M) {
              if (split) tma_store_2d(&gp.tp[0], box, c0, ks * d.M + row0);  // (M % 32 == 0 for split)
              else tma_store_2d(&gp.ty[g], box, c0, row0);
            }
            bulk_commit();
          }
          ++nbox;
        }
      };
      {
        float ya[32], yb[32];
        tmem_ld32_nowait(tbase, ya);
        tmem_wait32(ya);
#pragma unroll 1
        for (int cb = 0; cb < kHN; cb += 64) {
          tmem_ld32_nowait(tbase + (uint32_t)(cb + 32), yb);
          chunk(ya, cb);
          tmem_wait32(yb);
          if (cb + 64 < kHN) {
            tmem_ld32_nowait(tbase + (uint32_t)(cb + 64), ya);
          } else {  // accumulator fully in registers: hand the buffer back to the MMA
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(acc_empty0 + 8u * buf);
          }
          chunk(yb, cb + 32);
          if (cb + 64 < kHN) tmem_wait32(ya);
        }
      }
      if (d.amax_out && !split) warp_amax_to(d.amax_out, amx);
    }
    if (lane == 0) bulk_wait0();
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // the peer's TMEM is written by the leader's MMAs until the very end
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_cg2<512>(tmem_base);
  }
}

// ---- native block-scaled (UE8M0, MX) GEMM on the CTA pair --------------------------------------
// One problem, 256 x 256 tiles, tcgen05.mma.cta_group::2.kind::mxf8f6f4.block_scale.  Per 128-K stage
// each CTA stages, next to its A rows and half of B, the UE8M0 atoms the MMA needs in ITS TMEM:
// SFA for its 128 rows (512 B) and SFB for all 256 columns of the tile (2 x 512 B; CUTLASS's 2-SM
// block-scaled layout); the leader copies them smem -> TMEM in both CTAs with
// tcgen05.cp.cta_group::2 right before the stage's MMAs (same pipeline, issue order).  TMEM: one
// 256-column accumulator + a 4-stage ring of 12 scale columns, so the accumulator is single-
// buffered: the epilogue warps pull their 128 columns into registers first and release it at once.
// NV = true: NVFP4 (kind::mxf4nvf4.block_scale.scale_vec::4X; a stage row = 256 packed E2M1
// elements = 4 MMAs of K = 64, each reading its own atoms: SFA 4 x 512 B and SFB 2 x 4 x 512 B per
// stage; TMEM ring of 48 scale columns per stage; the FP32 tensor scales sa[0] * sb[0] applied in
// the epilogue).

template <bool NV> struct MxCfg {
  // NVFP4: a stage's MMAs take half the time of FP8's, so the ring is deeper (5 stages) and the
  // epilogue's staging boxes single-buffered to make room
  static constexpr int kStages = NV ? 5 : 4;
  static constexpr int kOutBufs = NV ? 1 : 2;
  static constexpr int kSf = NV ? 512 * 12 : 512 * 3;              // SFA + SFB atoms per stage
  static constexpr int kSfCols = NV ? 48 : 12;                     // TMEM scale columns per stage
  static constexpr int kOffB = kStages * k2StageA;
  static constexpr int kOffSf = kOffB + kStages * k2StageB;
  static constexpr int kOffOut = kOffSf + kStages * kSf;            // [8 warps][kOutBufs][4096]
  static constexpr int kOffCol = kOffOut + k2EpiWarps * kOutBufs * 4096;  // bias [256]
  static constexpr int kOffBar = kOffCol + 256 * 4;
  static constexpr int kSmem = kOffBar + 256 + 1024;
  static_assert(kSmem <= 227 * 1024, "mx pair smem");
  static_assert(256 + kStages * kSfCols <= 512, "mx pair tmem");
};

template <bool NV>
__global__ void __launch_bounds__(k2Threads, 1) mx_pair_kernel(const __grid_constant__ MxPairParams mp) {
  using Cf = MxCfg<NV>;
  constexpr int kMxSf = Cf::kSf;
  constexpr int kMxOffB = Cf::kOffB, kMxOffSf = Cf::kOffSf, kMxOffOut = Cf::kOffOut, kMxOffCol = Cf::kOffCol,
                kMxOffBar = Cf::kOffBar;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + kMxOffB;
  uint8_t* sSf = smem + kMxOffSf;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + kMxOffBar);
  uint64_t* empty_bar = full_bar + Cf::kStages;
  uint64_t* acc_full = empty_bar + Cf::kStages;
  uint64_t* acc_empty = acc_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 1);
  const GroupDesc& d = mp.d;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rank = (int)cluster_ctarank();
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const int T = mp.tiles;
  const int nkb = (d.K + 127) / 128;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&mp.ta);
    tma_prefetch_desc(&mp.tb);
    tma_prefetch_desc(&mp.tsa);
    tma_prefetch_desc(&mp.tsb);
    for (int s = 0; s < Cf::kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    mbar_init(acc_full, 1);
    mbar_init(acc_empty, 2 * k2EpiWarps);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_cg2<512>(tmem_slot);
  pdl_wait();
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ===== TMA producer (both CTAs) =====
    if (lane == 0) {
      const uint32_t full0 = mapa_shared(smem_u32(full_bar), 0);
      int it = 0;
      for (int t = cid; t < T; t += ncl) {
        const int mb = t / d.tiles_n, nb = t - (t / d.tiles_n) * d.tiles_n;
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % Cf::kStages;
          const uint32_t ph = (uint32_t)(it / Cf::kStages) & 1u;
          mbar_wait(&empty_bar[s], ph ^ 1u, 1);
          if (rank == 0) mbar_arrive_expect_tx(&full_bar[s], 2u * (k2StageA + k2StageB + kMxSf));
          tma_load_2d_cg2(sA + s * k2StageA, &mp.ta, full0 + 8u * s, kb * 128, mb * 256 + rank * 128);
          tma_load_2d_cg2(sB + s * k2StageB, &mp.tb, full0 + 8u * s, kb * 128, nb * 256 + rank * 128);
          // scale atoms: (atom, kb) starts at 256-byte row (atom * kbs + kb) * 2 of the pack
          uint8_t* sf = sSf + s * kMxSf;
          constexpr int kR = NV ? 8 : 2;  // 256-byte pack rows per 128 rows per stage (the map's box)
          tma_load_2d_cg2(sf, &mp.tsa, full0 + 8u * s, 0, ((mb * 2 + rank) * mp.sf_kbs + kb) * kR);
          tma_load_2d_cg2(sf + 256 * kR, &mp.tsb, full0 + 8u * s, 0, ((nb * 2) * mp.sf_kbs + kb) * kR);
          tma_load_2d_cg2(sf + 512 * kR, &mp.tsb, full0 + 8u * s, 0, ((nb * 2 + 1) * mp.sf_kbs + kb) * kR);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ===== MMA issuer (leader only) =====
    if (lane == 0 && rank == 0) {
      int it = 0, j = 0;
      const uint32_t idesc = NV ? idesc_nvf4(256, 256) : idesc_mxf8f6f4(d.a_fmt, d.b_fmt, 256, 256);
      for (int t = cid; t < T; t += ncl, ++j) {
        mbar_wait(acc_empty, ((uint32_t)j & 1u) ^ 1u, 4);  // both CTAs drained the accumulator
        tc_fence_after();
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % Cf::kStages;
          const uint32_t ph = (uint32_t)(it / Cf::kStages) & 1u;
          mbar_wait(&full_bar[s], ph, 2);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + s * k2StageA);
          const uint32_t b0 = smem_u32(sB + s * k2StageB);
          const uint32_t sft = tmem_base + 256u + (uint32_t)(Cf::kSfCols * s);
          const uint32_t sfs = smem_u32(sSf + s * kMxSf);
          if constexpr (NV) {
            // SFA atom k -> columns +4k; SFB (column half j, atom k) -> +16 + 8k + 4j: MMA k reads
            // its 256 B-scale rows from 8 consecutive columns
#pragma unroll
            for (int k = 0; k < 4; ++k) utccp_32x128b_warpx4_cg2(sft + 4u * k, sfs + 512u * k);
#pragma unroll
            for (int j = 0; j < 2; ++j)
#pragma unroll
              for (int k = 0; k < 4; ++k)
                utccp_32x128b_warpx4_cg2(sft + 16u + 8u * k + 4u * j, sfs + 2048u * (j + 1) + 512u * k);
#pragma unroll
            for (int k = 0; k < 4; ++k)
              mma_nvf4_cg2(tmem_base, smem_desc_kmajor_sw128(a0 + k * 32), smem_desc_kmajor_sw128(b0 + k * 32),
                           idesc, sft + 4u * k, sft + 16u + 8u * k, (kb | k) != 0);
          } else {
            utccp_32x128b_warpx4_cg2(sft, sfs);               // SFA (this CTA's 128 rows)
            utccp_32x128b_warpx4_cg2(sft + 4u, sfs + 512u);   // SFB columns 0..127
            utccp_32x128b_warpx4_cg2(sft + 8u, sfs + 1024u);  // SFB columns 128..255
#pragma unroll
            for (int k = 0; k < 4; ++k)
              mma_mxf8f6f4_cg2(tmem_base, smem_desc_kmajor_sw128(a0 + k * 32), smem_desc_kmajor_sw128(b0 + k * 32),
                               idesc, sft, sft + 4u, (uint32_t)k, (kb | k) != 0);
          }
          mma_commit_cg2_mc(&empty_bar[s], 3);
        }
        mma_commit_cg2_mc(acc_full, 3);
      }
    }
    __syncwarp();
  } else {
    // ===== epilogue (both CTAs): warp = TMEM lane quadrant q x column half h =====
    const int q = warp & 3;
    const int h = (warp - 2) >> 2;
    uint8_t* stg = smem + kMxOffOut + (warp - 2) * (Cf::kOutBufs * 4096);
    float* colb = reinterpret_cast<float*>(smem + kMxOffCol);
    const uint32_t acc_empty0 = mapa_shared(smem_u32(acc_empty), 0);
    const int esz = d.out_dtype == LOKA_F32 ? 4 : 2;
    const int cpb = 128 / esz;
    int nbox = 0, j = 0;
    for (int t = cid; t < T; t += ncl, ++j) {
      const int mb = t / d.tiles_n, nb = t - (t / d.tiles_n) * d.tiles_n;
      named_bar_sync(2, 32 * k2EpiWarps);  // the previous tile's bias reads are done
      {
        const int e = threadIdx.x - 64, n = nb * 256 + e;
        float b = 0.f;
        if (n < d.N && d.bias) b = d.bias_bf16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(d.bias)[n])
                                               : reinterpret_cast<const float*>(d.bias)[n];
        colb[e] = b;
      }
      named_bar_sync(2, 32 * k2EpiWarps);
      if (lane == 0) mbar_wait(acc_full, (uint32_t)j & 1u, 3);
      __syncwarp();
      tc_fence_after();
      // the whole 128-column half into registers, then the accumulator goes back to the MMA
      float y[128];
      const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(h * 128);
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld32_nowait(tbase + 32u * c, y + 32 * c);
#pragma unroll
      for (int c = 0; c < 8; ++c) tmem_wait16(y + 16 * c);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(acc_empty0);
      const int row0 = mb * 256 + rank * 128 + q * 32;
      const int col0 = nb * 256 + h * 128;
      float amx = 0.f;
      if constexpr (NV) {  // the FP32 tensor scales (the block scales were applied by the MMA)
        const float st = __fmul_rn(d.sa[0], d.sb[0]);
#pragma unroll
        for (int c = 0; c < 128; c += 2) {
          const float2 v = fmul2(make_float2(y[c], y[c + 1]), make_float2(st, st));
          y[c] = v.x;
          y[c + 1] = v.y;
        }
      }
#pragma unroll
      for (int cb = 0; cb < 128; cb += 32) {
        float* yc = y + cb;
        if (d.bias) {
          const uint32_t cs = smem_u32(colb + h * 128 + cb);
#pragma unroll
          for (int c = 0; c < 32; c += 4) {
            const float4 b4 = lds_f4(cs + 4u * c);
            const float2 a = fadd2(make_float2(yc[c], yc[c + 1]), make_float2(b4.x, b4.y));
            const float2 b = fadd2(make_float2(yc[c + 2], yc[c + 3]), make_float2(b4.z, b4.w));
            yc[c] = a.x; yc[c + 1] = a.y; yc[c + 2] = b.x; yc[c + 3] = b.y;
          }
        }
        if (d.amax_out && row0 + lane < d.M) {
#pragma unroll
          for (int c = 0; c < 32; ++c)
            if (col0 + cb + c < d.N) amx = fmaxf(amx, fabsf(esz == 2 ? stored_bf16(yc[c]) : yc[c]));
        }
        const int in_box = cb % cpb;
        uint8_t* box = stg + (Cf::kOutBufs == 2 ? (nbox & 1) * 4096 : 0);
        if (in_box == 0) {
          if (lane == 0) {
            if constexpr (Cf::kOutBufs == 2) bulk_wait_read_le1();
            else bulk_wait_read0();
          }
          __syncwarp();
        }
        const uint32_t rowa = smem_u32(box) + (uint32_t)lane * 128u;
        if (esz == 4) {
#pragma unroll
          for (int k = 0; k < 8; ++k)
            sts_u4(rowa + ((((uint32_t)k) ^ ((uint32_t)lane & 7u)) << 4),
                   make_uint4(__float_as_uint(yc[4 * k]), __float_as_uint(yc[4 * k + 1]),
                              __float_as_uint(yc[4 * k + 2]), __float_as_uint(yc[4 * k + 3])));
        } else {
          const uint32_t p0 = (uint32_t)(in_box * 2) >> 4;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            uint32_t w[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              __nv_bfloat162 hh = __floats2bfloat162_rn(yc[8 * k + 2 * i], yc[8 * k + 2 * i + 1]);
              w[i] = *reinterpret_cast<uint32_t*>(&hh);
            }
            sts_u4(rowa + (((p0 + (uint32_t)k) ^ ((uint32_t)lane & 7u)) << 4), make_uint4(w[0], w[1], w[2], w[3]));
          }
        }
        if (in_box + 32 == cpb) {
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            const int c0 = col0 + cb + 32 - cpb;
            if (c0 < d.N && row0 < d.M) tma_store_2d(&mp.ty, box, c0, row0);
            bulk_commit();
          }
          ++nbox;
        }
      }
      if (d.amax_out) warp_amax_to(d.amax_out, amx);
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

template <bool NV>
static cudaError_t launch_mx_pair_t(const MxPairParams& mp, int num_sms, cudaStream_t st) {
  {
    cudaError_t e = ensure_func_attrs(reinterpret_cast<const void*>(mx_pair_kernel<NV>), MxCfg<NV>::kSmem);
    if (e != cudaSuccess) return e;
  }
  const int pairs = mp.tiles < num_sms / 2 ? mp.tiles : num_sms / 2;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(2 * pairs), 1, 1);
  cfg.blockDim = dim3(k2Threads, 1, 1);
  cfg.dynamicSmemBytes = MxCfg<NV>::kSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  cudaError_t e = cudaLaunchKernelEx(&cfg, mx_pair_kernel<NV>, mp);
  note_launch();
  return e;
}
cudaError_t launch_mx_pair(const MxPairParams& mp, int num_sms, cudaStream_t st) {
  return mp.nvfp4 ? launch_mx_pair_t<true>(mp, num_sms, st) : launch_mx_pair_t<false>(mp, num_sms, st);
}

// ---- split-K reduction: y = (sum over slices) * s_a[m] * s_b[n] (+ bias[n]), fixed slice order ----
__global__ void __launch_bounds__(256) splitk_reduce_kernel(const GroupDesc d, const float* __restrict__ part,
                                                            void* y, int64_t ldy) {
  pdl_wait();
  const int64_t n4 = d.N / 4, total = (int64_t)d.M * n4, slice = (int64_t)d.M * d.N;
  float amx = 0.f;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = i / n4;
    const int n = (int)(i - m * n4) * 4;
    float4 acc = __ldg(reinterpret_cast<const float4*>(part + m * d.N + n));
    for (int s = 1; s < d.ksplit; ++s) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(part + s * slice + m * d.N + n));
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    const float sa = d.sa[d.sa_row ? m : 0];
    float o[4] = {acc.x, acc.y, acc.z, acc.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      o[k] = o[k] * (sa * d.sb[d.sb_row ? n + k : 0]);
      if (d.bias)
        o[k] += d.bias_bf16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(d.bias)[n + k])
                            : reinterpret_cast<const float*>(d.bias)[n + k];
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) amx = fmaxf(amx, fabsf(d.out_dtype == LOKA_F32 ? o[k] : stored_bf16(o[k])));
    if (d.out_dtype == LOKA_F32) {
      *reinterpret_cast<float4*>(reinterpret_cast<float*>(y) + m * ldy + n) = make_float4(o[0], o[1], o[2], o[3]);
    } else {
      __nv_bfloat162 a = __floats2bfloat162_rn(o[0], o[1]), b = __floats2bfloat162_rn(o[2], o[3]);
      *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(y) + m * ldy + n) =
          make_uint2(*reinterpret_cast<uint32_t*>(&a), *reinterpret_cast<uint32_t*>(&b));
    }
  }
  if (d.amax_out) warp_amax_to(d.amax_out, amx);
}

cudaError_t launch_splitk_reduce(const GroupDesc& d, const float* part, void* y, int64_t ldy, cudaStream_t st) {
  const int64_t total = (int64_t)d.M * (d.N / 4);
  int64_t nb = (total + 255) / 256;
  if (nb > 148 * 8) nb = 148 * 8;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)nb);
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  note_launch();
  return cudaLaunchKernelEx(&cfg, splitk_reduce_kernel, d, part, y, ldy);
}

template <bool BF16IN, bool WIDE, bool SPLIT>
static cudaError_t launch_grouped2_t(const GroupedParams& gp, int num_sms, cudaStream_t st) {
  {
    cudaError_t e = ensure_func_attrs(reinterpret_cast<const void*>(grouped2_kernel<BF16IN, WIDE, SPLIT>), G2<WIDE>::kSmem);
    if (e != cudaSuccess) return e;
  }
  const int T = gp.tile_start[gp.G];
  const int pairs = T < num_sms / 2 ? T : num_sms / 2;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(2 * pairs), 1, 1);
  cfg.blockDim = dim3(k2Threads, 1, 1);
  cfg.dynamicSmemBytes = G2<WIDE>::kSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  cudaError_t e = cudaLaunchKernelEx(&cfg, grouped2_kernel<BF16IN, WIDE, SPLIT>, gp);
  note_launch();
  return e;
}
template <bool BF16IN>
static cudaError_t launch_grouped2_any(const GroupedParams& gp, int num_sms, cudaStream_t st) {
  const bool split = gp.G == 1 && gp.g[0].ksplit > 1;
  if (gp.wide)
    return split ? launch_grouped2_t<BF16IN, true, true>(gp, num_sms, st)
                 : launch_grouped2_t<BF16IN, true, false>(gp, num_sms, st);
  return split ? launch_grouped2_t<BF16IN, false, true>(gp, num_sms, st)
               : launch_grouped2_t<BF16IN, false, false>(gp, num_sms, st);
}
cudaError_t launch_grouped2(const GroupedParams& gp, int num_sms, cudaStream_t st) {
  return launch_grouped2_any<false>(gp, num_sms, st);
}
cudaError_t launch_grouped2_bf16(const GroupedParams& gp, int num_sms, cudaStream_t st) {
  return launch_grouped2_any<true>(gp, num_sms, st);
}

}  // namespace loka
