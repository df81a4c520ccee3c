// linear.cu — a4/a5: FP8 GEMM on tcgen05 (FP32 accumulator in TMEM, operands by TMA) fused
// with the dequant / bias / LayerNorm / RMSNorm / BlockNorm epilogue and the optional FP8 cast
// of the normalised output (next layer's rowwise input).
//
// Paper: PAPER.md:456 (§III-B.2) "fuse normalization directly into the GEMM epilogue ... while
// the output tiles still reside in on-chip memory"; formula PAPER.md:460; Case 1/Case 2
// PAPER.md:464-468 (a row that spans several thread blocks needs cross-block statistics).
//
// B200 design:
//   * CTA tile 128 x BN (BN in {64,128,256}), K staged 128 FP8 (= one 128B swizzle atom) per
//     pipeline stage; warp 0 = TMA producer, warp 1 = tcgen05.mma issuer (one elected lane),
//     warps 2-5 = epilogue (warp w reads TMEM lanes 32*(w%4)..+31, one row per thread).
//   * The 128 x BN FP32 accumulator lives in TMEM; it never goes to HBM (a5).
//   * Case 2 (row wider than one CTA) is a thread-block cluster along N (<= 8 CTAs): per-row
//     partial statistics (Chan's (n, mean, M2) for LayerNorm, sum of squares for RMSNorm, amax
//     for an FP8 output) are exchanged through distributed shared memory and merged in
//     cluster-rank order, so every CTA derives bit-identical row statistics.
#include "common.cuh"
#include "launch.h"

namespace loka {


constexpr int kThreads = 192;  // 6 warps
constexpr int kBK = 128;       // FP8 elements of K per stage (128 B rows, SW128 atom)

template <int BN> struct LinCfg {
  static constexpr int kStageA = 128 * kBK;  // bytes
  static constexpr int kStageB = BN * kBK;
  static constexpr int kStageBytes = kStageA + kStageB;
  static constexpr int kStages = (196 * 1024) / kStageBytes > 8 ? 8 : (196 * 1024) / kStageBytes;
  static constexpr uint32_t kTmemCols = BN < 32 ? 32 : BN;
  // smem: [stages A][stages B][barriers][tmem slot][column params 4*BN][stats 128*4]
  static constexpr int kOffB = kStages * kStageA;
  static constexpr int kOffBar = kOffB + kStages * kStageB;
  static constexpr int kOffTmem = kOffBar + (2 * kStages + 1) * 8;
  static constexpr int kOffCol = (kOffTmem + 4 + 15) & ~15;
  static constexpr int kOffStat = kOffCol + 4 * BN * 4;
  static constexpr int kOffStat2 = kOffStat + 128 * 4 * 4;
  static constexpr int kSmemBytes = kOffStat2 + 128 * 4 + 1024;  // + alignment slack
};

// Chan et al. pairwise merge of (n, mean, M2) — the same update as PAPER.md:293-299
// (batched Welford merge) applied to column partitions of one row.
LOKA_DEVINL void chan_merge(float& n, float& mean, float& m2, float nb, float meanb, float m2b) {
  if (nb <= 0.f) return;
  if (n <= 0.f) { n = nb; mean = meanb; m2 = m2b; return; }
  const float nt = n + nb;
  const float d = meanb - mean;
  mean = mean + d * (nb / nt);
  m2 = m2 + m2b + d * d * (n * nb / nt);
  n = nt;
}

template <int BN>
__global__ void __launch_bounds__(kThreads, 1)
    linear_norm_kernel(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
                       const LinearParams p) {
  using C = LinCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::kOffB;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
  uint64_t* empty_bar = full_bar + C::kStages;
  uint64_t* tmem_full = empty_bar + C::kStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::kOffTmem);
  float* col_sb = reinterpret_cast<float*>(smem + C::kOffCol);
  float* col_bias = col_sb + BN;
  float* col_gamma = col_bias + BN;
  float* col_beta = col_gamma + BN;
  float* stat = reinterpret_cast<float*>(smem + C::kOffStat);    // [128][4]
  float* stat2 = reinterpret_cast<float*>(smem + C::kOffStat2);  // [128]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * 128;
  const int n0 = blockIdx.y * BN;
  const int ncols = min(BN, p.N - n0);  // valid columns of this CTA (> 0)
  const int num_kb = (p.K + kBK - 1) / kBK;
  const int csize = p.cluster_n;

  // ---- one-time setup ----
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tma_a);
    tma_prefetch_desc(&tma_b);
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    mbar_init(tmem_full, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<C::kTmemCols>(tmem_slot);
  if (warp >= 2) {  // per-column epilogue parameters -> smem
    for (int j = threadIdx.x - 64; j < BN; j += 128) {
      const int n = n0 + j;
      const bool ok = n < p.N;
      col_sb[j] = ok ? p.sb[p.sb_row ? n : 0] : 0.f;
      float b = 0.f;
      if (ok && p.bias) b = p.bias_bf16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p.bias)[n])
                                         : reinterpret_cast<const float*>(p.bias)[n];
      col_bias[j] = b;
      col_gamma[j] = (ok && p.gamma) ? p.gamma[n] : 1.f;
      col_beta[j] = (ok && p.beta) ? p.beta[n] : 0.f;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  // number of cluster-wide barriers every thread of the CTA executes (uniform)
  const bool is_fp8_out = p.out_dtype == LOKA_E4M3 || p.out_dtype == LOKA_E5M2;
  const bool affine = p.gamma != nullptr || p.beta != nullptr;
  const bool xchg_stats = csize > 1 && (p.norm == LOKA_NORM_LAYER || p.norm == LOKA_NORM_RMS);
  const bool xchg_amax = csize > 1 && is_fp8_out;
  const int n_cluster_bars = csize > 1 ? (int)xchg_stats + (int)xchg_amax + 1 : 0;

  if (warp == 0) {
    // ===== TMA producer =====
    if (lane == 0) {
      for (int kb = 0; kb < num_kb; ++kb) {
        const int s = kb % C::kStages;
        const uint32_t ph = (uint32_t)(kb / C::kStages) & 1u;
        mbar_wait(&empty_bar[s], ph ^ 1u, 1);
        mbar_arrive_expect_tx(&full_bar[s], C::kStageBytes);
        tma_load_2d(sA + s * C::kStageA, &tma_a, &full_bar[s], kb * kBK, m0);
        tma_load_2d(sB + s * C::kStageB, &tma_b, &full_bar[s], kb * kBK, n0);
      }
    }
    __syncwarp();
    for (int i = 0; i < n_cluster_bars; ++i) cluster_sync_all();
  } else if (warp == 1) {
    // ===== MMA issuer =====
    if (lane == 0) {
      const uint32_t idesc = idesc_f8f6f4(p.a_fmt, p.b_fmt, 128, BN);
      for (int kb = 0; kb < num_kb; ++kb) {
        const int s = kb % C::kStages;
        const uint32_t ph = (uint32_t)(kb / C::kStages) & 1u;
        mbar_wait(&full_bar[s], ph, 2);
        tc_fence_after();
        const uint32_t a0 = smem_u32(sA + s * C::kStageA);
        const uint32_t b0 = smem_u32(sB + s * C::kStageB);
#pragma unroll
        for (int k = 0; k < kBK / 32; ++k) {
          mma_f8f6f4(tmem_base, smem_desc_kmajor_sw128(a0 + k * 32), smem_desc_kmajor_sw128(b0 + k * 32), idesc,
                     (kb | k) != 0);
        }
        mma_commit(&empty_bar[s]);
      }
      mma_commit(tmem_full);
    }
    __syncwarp();
    for (int i = 0; i < n_cluster_bars; ++i) cluster_sync_all();
  } else {
    // ===== epilogue: thread = one row of the 128 x BN tile =====
    const int q = warp & 3;  // TMEM lane quadrant this warp may access
    const int r = q * 32 + lane;
    const int grow = m0 + r;
    const bool row_ok = grow < p.M;
    const float sa = row_ok ? p.sa[p.sa_row ? grow : 0] : 0.f;
    const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16);
    const int nchunks = (ncols + 31) / 32;
    const int norm = p.norm;
    const int blk = norm == LOKA_NORM_BLOCK_RMS ? p.norm_block : BN;
    const int nblk_cta = (ncols + blk - 1) / blk;  // <= 8 (blk >= 32)

    mbar_wait(tmem_full, 0, 3);
    tc_fence_after();

    // y_j = acc_j * sa * sb_j + bias_j (identical in every pass)
    auto load_y = [&](int c, float (&v)[32]) {
      tmem_ld32(taddr + (uint32_t)(c * 32), v);
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int jj = c * 32 + j;
        v[j] = __fadd_rn(__fmul_rn(__fmul_rn(v[j], sa), col_sb[jj]), col_bias[jj]);
      }
    };

    // ---- pass 1: row statistics over this CTA's columns ----
    float st_n = 0.f, st_mean = 0.f, st_m2 = 0.f;  // LayerNorm (Chan)
    float st_ss = 0.f;                              // RMSNorm
    float blk_ss[8], blk_max[8];
#pragma unroll
    for (int b = 0; b < 8; ++b) blk_ss[b] = 0.f, blk_max[b] = 0.f;
    float ymax = -INFINITY, ymin = INFINITY;
    const bool need_pass1 = norm != LOKA_NORM_NONE || (is_fp8_out && !affine);
    if (need_pass1) {
      for (int c = 0; c < nchunks; ++c) {
        float v[32];
        load_y(c, v);
        const int nv = min(32, ncols - c * 32);
        if (norm == LOKA_NORM_LAYER) {
          float s = 0.f;
#pragma unroll
          for (int j = 0; j < 32; ++j) s += j < nv ? v[j] : 0.f;
          const float mc = s / (float)nv;
          float m2 = 0.f;
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float d = j < nv ? v[j] - mc : 0.f;
            m2 = fmaf(d, d, m2);
          }
          chan_merge(st_n, st_mean, st_m2, (float)nv, mc, m2);
        } else if (norm == LOKA_NORM_RMS) {
#pragma unroll
          for (int j = 0; j < 32; ++j) st_ss = j < nv ? fmaf(v[j], v[j], st_ss) : st_ss;
        } else if (norm == LOKA_NORM_BLOCK_RMS) {
          const int b = (c * 32) / blk;
          float ss = 0.f, mx = 0.f;
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            if (j < nv) {
              ss = fmaf(v[j], v[j], ss);
              mx = fmaxf(mx, fabsf(v[j]));
            }
          }
#pragma unroll
          for (int bb = 0; bb < 8; ++bb)
            if (bb == b) blk_ss[bb] += ss, blk_max[bb] = fmaxf(blk_max[bb], mx);
        }
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (j < nv) ymax = fmaxf(ymax, v[j]), ymin = fminf(ymin, v[j]);
      }
    }

    // ---- cross-CTA statistics (Case 2) ----
    float mu = 0.f, rstd = 1.f;
    if (norm == LOKA_NORM_LAYER || norm == LOKA_NORM_RMS) {
      float n_tot = st_n, mean = st_mean, m2 = st_m2, ss = st_ss, mx = ymax, mn = ymin;
      if (xchg_stats) {
        stat[r * 4 + 0] = norm == LOKA_NORM_LAYER ? st_mean : st_ss;
        stat[r * 4 + 1] = st_m2;
        stat[r * 4 + 2] = ymax;
        stat[r * 4 + 3] = ymin;
        cluster_sync_all();
        n_tot = 0.f; mean = 0.f; m2 = 0.f; ss = 0.f; mx = -INFINITY; mn = INFINITY;
        const uint32_t la = smem_u32(&stat[r * 4]);
        for (int rk = 0; rk < csize; ++rk) {
          const uint32_t ra = mapa_shared(la, (uint32_t)rk);
          const float a0 = ld_dsmem_f32(ra), a1 = ld_dsmem_f32(ra + 4);
          const float a2 = ld_dsmem_f32(ra + 8), a3 = ld_dsmem_f32(ra + 12);
          const float nk = (float)min(BN, p.N - rk * BN);
          if (norm == LOKA_NORM_LAYER) chan_merge(n_tot, mean, m2, nk, a0, a1);
          else ss += a0, n_tot += nk;
          mx = fmaxf(mx, a2);
          mn = fminf(mn, a3);
        }
      } else if (norm == LOKA_NORM_RMS) {
        n_tot = (float)ncols;
      }
      ymax = mx;
      ymin = mn;
      if (norm == LOKA_NORM_LAYER) {
        mu = mean;
        rstd = __fdiv_rn(1.f, __fsqrt_rn(__fadd_rn(__fdiv_rn(m2, n_tot), p.eps)));
      } else {
        mu = 0.f;
        rstd = __fdiv_rn(1.f, __fsqrt_rn(__fadd_rn(__fdiv_rn(ss, n_tot), p.eps)));
      }
    }
    float blk_rstd[8];
#pragma unroll
    for (int b = 0; b < 8; ++b)
      blk_rstd[b] = __fdiv_rn(1.f, __fsqrt_rn(__fadd_rn(__fdiv_rn(blk_ss[b], (float)blk), p.eps)));

    // out_j = norm(y_j) (identical in every pass)
    auto norm_out = [&](int c, float (&v)[32]) {
      if (norm == LOKA_NORM_LAYER || norm == LOKA_NORM_RMS) {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int jj = c * 32 + j;
          float o = __fmul_rn(__fsub_rn(v[j], mu), rstd);
          if (affine) o = __fadd_rn(__fmul_rn(o, col_gamma[jj]), col_beta[jj]);
          v[j] = o;
        }
      } else if (norm == LOKA_NORM_BLOCK_RMS) {
        const int b = (c * 32) / blk;
        float rs = blk_rstd[0];
#pragma unroll
        for (int bb = 1; bb < 8; ++bb)
          if (bb == b) rs = blk_rstd[bb];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __fmul_rn(v[j], rs);
      }
    };

    // ---- FP8 output: row amax of the normalised values -> row scale ----
    float r_out = 1.f;
    if (is_fp8_out) {
      float amax = 0.f;
      if (!affine) {  // out is monotone in y: the amax is attained at ymax or ymin exactly
        if (norm == LOKA_NORM_LAYER || norm == LOKA_NORM_RMS) {
          const float hi = __fmul_rn(__fsub_rn(ymax, mu), rstd);
          const float lo = __fmul_rn(__fsub_rn(ymin, mu), rstd);
          amax = fmaxf(fabsf(hi), fabsf(lo));
        } else if (norm == LOKA_NORM_BLOCK_RMS) {
          for (int b = 0; b < nblk_cta; ++b) amax = fmaxf(amax, __fmul_rn(blk_max[b], blk_rstd[b]));
        } else {
          amax = fmaxf(fabsf(ymax), fabsf(ymin));
        }
      } else {  // affine: one more pass over TMEM
        for (int c = 0; c < nchunks; ++c) {
          float v[32];
          load_y(c, v);
          norm_out(c, v);
          const int nv = min(32, ncols - c * 32);
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (j < nv) amax = fmaxf(amax, fabsf(v[j]));
        }
      }
      if (nchunks == 0) amax = 0.f;
      if (xchg_amax) {
        stat2[r] = amax;
        cluster_sync_all();
        amax = 0.f;
        const uint32_t la = smem_u32(&stat2[r]);
        for (int rk = 0; rk < csize; ++rk) amax = fmaxf(amax, ld_dsmem_f32(mapa_shared(la, (uint32_t)rk)));
      }
      if (__float_as_uint(amax) >= 0x7F800000u && p.status) atomicOr(p.status, LOKA_DEVSTATUS_NONFINITE);
      float s_out;
      if (p.out_dtype == LOKA_E4M3) scales_from_amax<LOKA_E4M3, LOKA_SCALE_F32>(amax, s_out, r_out);
      else scales_from_amax<LOKA_E5M2, LOKA_SCALE_F32>(amax, s_out, r_out);
      if (row_ok && blockIdx.y == 0 && p.y_scales) p.y_scales[grow] = s_out;
    }

    // ---- pass 2: normalise, cast, store ----
    {  // every lane executes the .sync.aligned TMEM loads; only rows < M store
      for (int c = 0; c < nchunks; ++c) {
        float v[32];
        load_y(c, v);
        norm_out(c, v);
        if (!row_ok) continue;
        const int col0 = n0 + c * 32;
        const int nv = min(32, ncols - c * 32);
        if (p.precast) {
          float* dst = p.precast + (int64_t)grow * p.ld_pre + col0;
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (j < nv) dst[j] = v[j];
        }
        if (p.out_dtype == LOKA_F32) {
          float* dst = reinterpret_cast<float*>(p.y) + (int64_t)grow * p.ldy + col0;
          if (nv == 32) {
#pragma unroll
            for (int j = 0; j < 32; j += 4)
              *reinterpret_cast<float4*>(dst + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (j < nv) dst[j] = v[j];
          }
        } else if (p.out_dtype == LOKA_BF16) {
          __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(p.y) + (int64_t)grow * p.ldy + col0;
          if (nv == 32) {
#pragma unroll
            for (int j = 0; j < 32; j += 8) {
              uint4 w;
              __nv_bfloat162 h0 = __floats2bfloat162_rn(v[j], v[j + 1]);
              __nv_bfloat162 h1 = __floats2bfloat162_rn(v[j + 2], v[j + 3]);
              __nv_bfloat162 h2 = __floats2bfloat162_rn(v[j + 4], v[j + 5]);
              __nv_bfloat162 h3 = __floats2bfloat162_rn(v[j + 6], v[j + 7]);
              w.x = *reinterpret_cast<uint32_t*>(&h0);
              w.y = *reinterpret_cast<uint32_t*>(&h1);
              w.z = *reinterpret_cast<uint32_t*>(&h2);
              w.w = *reinterpret_cast<uint32_t*>(&h3);
              *reinterpret_cast<uint4*>(dst + j) = w;
            }
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (j < nv) dst[j] = __float2bfloat16_rn(v[j]);
          }
        } else {
          uint8_t* dst = reinterpret_cast<uint8_t*>(p.y) + (int64_t)grow * p.ldy + col0;
          uint32_t w[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float a = __fmul_rn(v[4 * j], r_out), b = __fmul_rn(v[4 * j + 1], r_out);
            const float c2 = __fmul_rn(v[4 * j + 2], r_out), d = __fmul_rn(v[4 * j + 3], r_out);
            w[j] = p.out_dtype == LOKA_E4M3 ? cvt_fp8x4<LOKA_E4M3>(a, b, c2, d) : cvt_fp8x4<LOKA_E5M2>(a, b, c2, d);
          }
          if (nv == 32) {
            *reinterpret_cast<uint4*>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
            *reinterpret_cast<uint4*>(dst + 16) = make_uint4(w[4], w[5], w[6], w[7]);
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (j < nv) dst[j] = (uint8_t)(w[j >> 2] >> (8 * (j & 3)));
          }
        }
      }
    }
    if (csize > 1) cluster_sync_all();  // peers may still read our stats from DSMEM
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<C::kTmemCols>(tmem_base);
  }
}

template <int BN>
static cudaError_t launch_bn(const CUtensorMap& ta, const CUtensorMap& tb, const LinearParams& p, cudaStream_t st) {
  using C = LinCfg<BN>;
  static bool attr_done = false;  // idempotent; racing threads set the same value
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(linear_norm_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         C::kSmemBytes);
    if (e != cudaSuccess) return e;
    attr_done = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)((p.M + 127) / 128), (unsigned)((p.N + BN - 1) / BN), 1);
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = C::kSmemBytes;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 1;
  attr[0].val.clusterDim.y = (unsigned)p.cluster_n;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, linear_norm_kernel<BN>, ta, tb, p);
  note_launch();
  return e;
}

// Host accessor for the watchdog: returns the number of timed-out waits since the last reset
// and fills info[3] = {tag (1 empty, 2 full, 3 tmem_full), linear block id, thread | parity<<32}.
long long debug_hang_info(unsigned long long* info, int reset) {
  unsigned long long h[4] = {0, 0, 0, 0};
  if (cudaMemcpyFromSymbol(h, g_loka_hang, sizeof(h)) != cudaSuccess) return -1;
  if (info) info[0] = h[1], info[1] = h[2], info[2] = h[3];
  if (reset) {
    unsigned long long z[4] = {0, 0, 0, 0};
    int zi = 0;
    cudaMemcpyToSymbol(g_loka_hang, z, sizeof(z));
    cudaMemcpyToSymbol(g_loka_abort, &zi, sizeof(zi));
  }
  return (long long)h[0];
}

cudaError_t launch_linear(const CUtensorMap& ta, const CUtensorMap& tb, const LinearParams& p, int bn,
                          cudaStream_t st) {
  switch (bn) {
    case 64: return launch_bn<64>(ta, tb, p, st);
    case 128: return launch_bn<128>(ta, tb, p, st);
    case 256: return launch_bn<256>(ta, tb, p, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace loka
