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
//     warps 2-17 = epilogue: warp w reads TMEM lanes 32*(w%4)..+31 (one row per thread) and the
//     column quarter (w-2)/4 of the tile, i.e. BN/4 columns held entirely in registers: ONE
//     batch of TMEM loads and one wait, statistics, exchange and output all from registers.
//   * The 128 x BN FP32 accumulator lives in TMEM; it never goes to HBM (a5).
//   * Epilogue arithmetic is packed FP32x2 (FMUL2/FFMA2/FADD2) with 3-input min/max; for norms
//     without bias the per-row dequant scale s_a is folded into eps
//     ((s z - s mu)/sqrt(s^2 var + eps) == (z - mu)/sqrt(var + eps/s^2)), and the normalised
//     value is one FFMA: v = fma(y, rstd, -mu*rstd).
//   * The four column quarters of a row merge their statistics through shared memory (aliased on
//     the drained operand ring); Case 2 (row wider than one CTA) is a thread-block cluster along
//     N (<= 8 CTAs): every CTA pushes its per-row record (Chan (mean, M2) | sum of squares, y max,
//     y min) into each peer with one st.shared::cluster.v4, and all CTAs merge the records in
//     cluster-rank order, so every CTA derives bit-identical row statistics.
//   * Programmatic dependent launch: the prologue (barrier init, TMEM alloc, descriptor
//     prefetch) overlaps the previous kernel's tail; global inputs are read after
//     griddepcontrol.wait.
#include "common.cuh"
#include "launch.h"

namespace loka {

// Opt-in phase trace (loka_debug_trace): per CTA, 16 globaltimer stamps
//   0 entry | 1 after griddepcontrol.wait | 2 first TMA issued | 3 first stage landed (MMA)
//   4 last MMA committed | 5 accumulator ready (epilogue) | 6 statistics done | 7 stores done
//   8 accumulator in registers | 9 quarters merged | 10 cluster merged | 11 finalized
constexpr int kTraceCtas = 4096;
static __device__ unsigned long long g_trace[kTraceCtas * 16];
static __device__ int g_trace_on;
#define LOKA_TRACE(slot)                                                                    \
  do {                                                                                      \
    if (trace_on && cta_lin < kTraceCtas) g_trace[cta_lin * 16 + (slot)] = globaltimer_ns(); \
  } while (0)

constexpr int kEpiWarps = 16;               // every warp runs the epilogue ...
constexpr int kEpiThreads = 32 * kEpiWarps;
constexpr int kThreads = kEpiThreads;       // ... after warp 0 lane 0 (TMA) / warp 1 lane 0 (MMA) roles
constexpr int kBK = 128;                    // FP8 elements of K per stage (128 B rows, SW128 atom)
constexpr int kRec = 6;                     // floats per (row, quarter) record: n, mean, m2, ss, ymax, ymin
constexpr int kMaxCluster = 8;   // portable cluster size
constexpr int kBigCluster = 16;  // non-portable (opt-in): rows up to 16 x 256 = 4096 columns

constexpr uint32_t pow2_cols(uint32_t c) { return c <= 32 ? 32 : c <= 64 ? 64 : c <= 128 ? 128 : c <= 256 ? 256 : 512; }

// MX: 0 = plain FP8 (scales in the epilogue), 1 = MXFP8 / UE8M0 blockwise (kind::mxf8f6f4
// .block_scale: one 512 B atom per 128-K stage and 128 rows), 2 = NVFP4 (kind::mxf4nvf4
// .block_scale.scale_vec::4X: a stage row is 128 B = 256 packed E2M1 elements = 4 MMAs of K = 64,
// each MMA reading one 512 B atom (128 rows x four 16-element E4M3 scales) per 128 rows).
template <int BN, int MX = 0, int MAXC = kMaxCluster> struct LinCfg {
  static constexpr int kCPT = BN / 4;  // columns per epilogue thread
  static constexpr int kStageA = 128 * kBK;  // bytes
  static constexpr int kStageB = BN * kBK;
  static constexpr int kStageBytes = kStageA + kStageB;
  // MX mode: per stage one 512 B UE8M0 atom for A and BN/128 for B (bulk-copied with the stage),
  // copied to TMEM columns [BN + s*kSfCols, ...) by tcgen05.cp
  static constexpr int kSfAtoms = MX == 2 ? 4 : 1;  // atoms per stage per 128 rows
  static constexpr int kSf = MX ? 512 * kSfAtoms * (1 + BN / 128) : 0;
  static constexpr int kSfCols = 4 * kSfAtoms * (1 + BN / 128);
  // everything but the operand ring: column params, pushed cluster records (+ amax), barriers
  static constexpr int kFixed = 4 * BN * 4 + MAXC * 128 * 16 + MAXC * 128 * 4 + 512 + 1024;
  static constexpr int kStagesFit = (227 * 1024 - kFixed) / (kStageBytes + kSf);
  static constexpr int kStages = kStagesFit > 8 ? 8 : kStagesFit;
  static constexpr uint32_t kTmemCols = pow2_cols(MX ? BN + kStages * kSfCols : BN);
  static constexpr int kOffB = kStages * kStageA;
  static constexpr int kOffBar = kOffB + kStages * kStageB;
  static constexpr int kOffTmem = kOffBar + (2 * kStages + 1) * 8;
  static constexpr int kOffCol = (kOffTmem + 4 + 15) & ~15;         // sb, bias, gamma, beta [BN]
  static constexpr int kOffCs = kOffCol + 4 * BN * 4;                // [MAXC][128] float4 records
  static constexpr int kOffCs2 = kOffCs + MAXC * 128 * 16;           // [MAXC][128] amax
  static constexpr int kOffSf = kOffCs2 + MAXC * 128 * 4;            // [kStages][kSf] (MX)
  static constexpr int kSmemBytes = kOffSf + kStages * kSf + 1024;       // + alignment slack
  // after the mainloop the (drained) operand ring holds the quarter exchange [4][kRec + 1][128]
  // floats at offset 0 and the output staging tile (128 rows x BN x <= 4 bytes) at kOffStage
  static constexpr int kOffStage = 16384;
  static_assert(4 * (kRec + 1) * 128 * 4 <= kOffStage, "hx alias");
  static_assert(kOffStage + 128 * BN * 4 <= kStages * kStageBytes, "staging alias");
  static_assert(kStages >= 2 && kSmemBytes <= 227 * 1024, "smem");
  static_assert(!MX || BN % 128 == 0, "MX scale atoms cover 128 rows of B");
};

// Row statistics of a column partition: (n, mean, M2) for LayerNorm (merged with the batched
// Welford / Chan update of PAPER.md:293-299 applied to column partitions), sum of squares for
// RMS/BlockNorm, y max / min for the FP8 output's row amax.
struct RowRec {
  float n, mean, m2, ss, ymax, ymin;
  LOKA_DEVINL void init() { n = 0.f; mean = 0.f; m2 = 0.f; ss = 0.f; ymax = -INFINITY; ymin = INFINITY; }
};

// n-way parallel merge of K partial records (fixed order -> bit-identical wherever it runs):
//   n = sum n_k, mean = sum n_k mean_k / n, M2 = sum M2_k + sum n_k (mean_k - mean)^2
// (Chan et al.'s pairwise update applied to all parts at once: one division).
template <int K>
LOKA_DEVINL RowRec merge_recs(const RowRec (&r)[K]) {
  RowRec o;
  o.init();
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    o.n += r[k].n;
    s = fmaf(r[k].n, r[k].mean, s);
    o.ss += r[k].ss;
    o.ymax = fmaxf(o.ymax, r[k].ymax);
    o.ymin = fminf(o.ymin, r[k].ymin);
  }
  o.mean = o.n > 0.f ? __fdiv_rn(s, o.n) : 0.f;
  float m2 = 0.f;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const float d = r[k].mean - o.mean;
    m2 += r[k].m2 + r[k].n * d * d;
  }
  o.m2 = m2;
  return o;
}

template <int BN, int MX, int MAXC>
__global__ void __launch_bounds__(kThreads, 1)
    linear_norm_kernel(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
                       const __grid_constant__ CUtensorMap tma_y, const LinearParams p) {
  using C = LinCfg<BN, MX, MAXC>;
  constexpr int CPT = C::kCPT;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::kOffB;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + C::kOffBar);
  uint64_t* empty_bar = full_bar + C::kStages;
  uint64_t* tmem_full = empty_bar + C::kStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::kOffTmem);
  float* col = reinterpret_cast<float*>(smem + C::kOffCol);  // [4][BN]: sb, bias, gamma, beta
  float* hx = reinterpret_cast<float*>(smem);                // [4][kRec+1][128], valid after tmem_full
  float* cs = reinterpret_cast<float*>(smem + C::kOffCs);
  float* cs2 = reinterpret_cast<float*>(smem + C::kOffCs2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * 128;
  const int n0 = blockIdx.y * BN;
  const int ncols = min(BN, p.N - n0);  // valid columns of this CTA (> 0)
  const int num_kb = (p.K + kBK - 1) / kBK;
  const int csize = p.cluster_n;
  const int trace_on = *reinterpret_cast<volatile int*>(&g_trace_on);
  const int cta_lin = blockIdx.x + gridDim.x * blockIdx.y;
  if (threadIdx.x == 0) LOKA_TRACE(0);

  // ---- one-time setup (overlaps the previous kernel under PDL) ----
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tma_a);
    tma_prefetch_desc(&tma_b);
    tma_prefetch_desc(&tma_y);
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    mbar_init(tmem_full, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<C::kTmemCols>(tmem_slot);
  pdl_wait();  // inputs written by the previous kernel are visible from here on
  if (threadIdx.x == 0) LOKA_TRACE(1);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int norm = p.norm;
  const bool is_fp8_out = p.out_dtype == LOKA_E4M3 || p.out_dtype == LOKA_E5M2;
  // affine (gamma/beta) and the activation make the output non-monotone in y: the FP8 row amax
  // is then reduced over the final values instead of derived from y max / min
  const bool bwd = p.bwd != 0;  // NEXT-1 norm backward epilogue (y = dL/dz: not monotone in acc)
  const bool affine = p.gamma != nullptr || p.beta != nullptr || p.act != LOKA_ACT_NONE || bwd;
  const bool has_gb = p.gamma != nullptr || p.beta != nullptr;
  const bool is_block = norm == LOKA_NORM_BLOCK_RMS;
  // cluster-wide barriers: every thread of the CTA executes the same count (uniform)
  const bool xchg_stats = csize > 1 && !is_block && (norm != LOKA_NORM_NONE || (is_fp8_out && !affine));
  const bool xchg_amax = csize > 1 && is_fp8_out && (is_block || affine);

  if (warp == 0) {
    // ===== TMA producer =====
    if (lane == 0) {
      for (int kb = 0; kb < num_kb; ++kb) {
        const int s = kb % C::kStages;
        const uint32_t ph = (uint32_t)(kb / C::kStages) & 1u;
        mbar_wait(&empty_bar[s], ph ^ 1u, 1);
        mbar_arrive_expect_tx(&full_bar[s], C::kStageBytes + C::kSf);
        tma_load_2d(sA + s * C::kStageA, &tma_a, &full_bar[s], kb * kBK, m0);
        tma_load_2d(sB + s * C::kStageB, &tma_b, &full_bar[s], kb * kBK, n0);
        if constexpr (MX) {  // the stage's scale atoms: A rows m0.., B rows n0.. (BN/128 row blocks)
          constexpr int kA = 512 * C::kSfAtoms;  // bytes per 128 rows per stage
          uint8_t* sf = smem + C::kOffSf + s * C::kSf;
          bulk_load_g2s(sf, p.sfa_pack + ((size_t)(m0 >> 7) * p.sf_kblocks + kb) * kA, kA, &full_bar[s]);
#pragma unroll
          for (int j = 0; j < BN / 128; ++j)
            bulk_load_g2s(sf + kA * (j + 1), p.sfb_pack + ((size_t)((n0 >> 7) + j) * p.sf_kblocks + kb) * kA, kA,
                          &full_bar[s]);
        }
        if (kb == 0) LOKA_TRACE(2);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ===== MMA issuer =====
    if (lane == 0) {
      const uint32_t idesc = MX == 2   ? idesc_nvf4(128, BN)
                             : MX == 1 ? idesc_mxf8f6f4(p.a_fmt, p.b_fmt, 128, BN)
                                       : idesc_f8f6f4(p.a_fmt, p.b_fmt, 128, BN);
      for (int kb = 0; kb < num_kb; ++kb) {
        const int s = kb % C::kStages;
        const uint32_t ph = (uint32_t)(kb / C::kStages) & 1u;
        mbar_wait(&full_bar[s], ph, 2);
        if (kb == 0) LOKA_TRACE(3);
        tc_fence_after();
        const uint32_t a0 = smem_u32(sA + s * C::kStageA);
        const uint32_t b0 = smem_u32(sB + s * C::kStageB);
        if constexpr (MX == 2) {
          // scale atoms smem -> TMEM: A atom k at columns sft + 4k; B atom (row block j, k) at
          // sft + 16 + 4 (k BN/128 + j), so MMA k reads B's BN rows from consecutive columns
          const uint32_t sft = tmem_base + (uint32_t)(BN + s * C::kSfCols);
          const uint32_t sfs = smem_u32(smem + C::kOffSf + s * C::kSf);
#pragma unroll
          for (int k = 0; k < 4; ++k) utccp_32x128b_warpx4(sft + 4u * k, sfs + 512u * k);
#pragma unroll
          for (int j = 0; j < BN / 128; ++j)
#pragma unroll
            for (int k = 0; k < 4; ++k)
              utccp_32x128b_warpx4(sft + 16u + 4u * (k * (BN / 128) + j), sfs + 2048u * (j + 1) + 512u * k);
#pragma unroll
          for (int k = 0; k < 4; ++k)
            mma_nvf4(tmem_base, smem_desc_kmajor_sw128(a0 + k * 32), smem_desc_kmajor_sw128(b0 + k * 32), idesc,
                     sft + 4u * k, sft + 16u + 4u * k * (BN / 128), (kb | k) != 0);
        } else if constexpr (MX == 1) {
          // scales smem -> TMEM (executes in order with the MMAs issued by this thread)
          const uint32_t sft = tmem_base + (uint32_t)(BN + s * C::kSfCols);
          const uint32_t sfs = smem_u32(smem + C::kOffSf + s * C::kSf);
#pragma unroll
          for (int j = 0; j <= BN / 128; ++j) utccp_32x128b_warpx4(sft + 4u * j, sfs + 512u * j);
#pragma unroll
          for (int k = 0; k < kBK / 32; ++k)
            mma_mxf8f6f4(tmem_base, smem_desc_kmajor_sw128(a0 + k * 32), smem_desc_kmajor_sw128(b0 + k * 32), idesc,
                         sft, sft + 4u, (uint32_t)k, (kb | k) != 0);
        } else {
#pragma unroll
          for (int k = 0; k < kBK / 32; ++k) {
            mma_f8f6f4(tmem_base, smem_desc_kmajor_sw128(a0 + k * 32), smem_desc_kmajor_sw128(b0 + k * 32), idesc,
                       (kb | k) != 0);
          }
        }
        mma_commit(&empty_bar[s]);
      }
      mma_commit(tmem_full);
      LOKA_TRACE(4);
    }
    __syncwarp();
  }
  {
    // ===== epilogue (all 16 warps): thread = one row x one column quarter (CPT cols, registers) =====
    const int q = warp & 3;              // TMEM lane quadrant this warp may access
    const int cq = warp >> 2;            // column quarter
    const int r = q * 32 + lane;
    const int grow = m0 + r;
    const bool row_ok = grow < p.M;
    const int cb = cq * CPT;                         // first local column of this thread
    const int nv = max(0, min(CPT, ncols - cb));     // valid columns of this thread
    const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)cb;
    // MX: block scales applied by the MMA (NVFP4: the FP32 tensor scales remain, as sa / sb)
    const float sa = row_ok ? (MX == 1 ? 1.f : p.sa[p.sa_row ? grow : 0]) : 0.f;
    const bool has_bias = p.bias != nullptr;
    const bool fold = !has_bias && norm != LOKA_NORM_NONE && !bwd;  // s_a folded into eps
    const float ys = fold ? 1.f : sa;
    const int blk = is_block ? p.norm_block : BN;
    const uint32_t col_s = smem_u32(col);

    // per-column epilogue parameters -> smem (while the producer / MMA warps run the mainloop)
    for (int j = threadIdx.x; j < BN; j += kEpiThreads) {
      const int n = n0 + j;
      const bool ok = n < p.N;
      col[j] = ok ? (MX == 1 ? 1.f : p.sb[p.sb_row ? n : 0]) : 0.f;
      float b = 0.f;
      if (ok && p.bias) b = p.bias_bf16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p.bias)[n])
                                         : reinterpret_cast<const float*>(p.bias)[n];
      col[BN + j] = b;
      col[2 * BN + j] = (ok && p.gamma) ? p.gamma[n] : 1.f;
      col[3 * BN + j] = (ok && p.beta) ? p.beta[n] : 0.f;
    }
    named_bar_sync(1, kEpiThreads);

    if (bwd && row_ok) {  // NEXT-1: pull this thread's x-hat row segment into L2 while the MMAs run
      const __nv_bfloat16* xr = p.xhat + (int64_t)grow * p.ld_xhat + n0 + cb;
      for (int j = 0; j < CPT; j += 64) asm volatile("prefetch.global.L2 [%0];" ::"l"(xr + j));
    }
    if (lane == 0) mbar_wait(tmem_full, 0, 3);  // one waiter per warp
    __syncwarp();
    tc_fence_after();
    pdl_launch_dependents();
    if (threadIdx.x == 64) LOKA_TRACE(5);

    // ---- accumulator -> registers: all loads in flight, one wait ----
    float y[CPT];
    if constexpr (CPT >= 32) {
#pragma unroll
      for (int i = 0; i < CPT / 32; ++i) tmem_ld32_nowait(taddr + (uint32_t)(32 * i), y + 32 * i);
#pragma unroll
      for (int i = 0; i < CPT / 16; ++i) tmem_wait16(y + 16 * i);
    } else {
      tmem_ld16_nowait(taddr, y);
      tmem_wait16(y);
    }
    // y_j = acc_j * s_a * s_b[n] (+ bias[n]); with fold: acc_j * s_b[n]
#pragma unroll
    for (int j = 0; j < CPT; j += 4) {
      const uint32_t o = (uint32_t)(cb + j) * 4u;
      const float4 s4 = lds_f4(col_s + o);
      float2 s01 = make_float2(s4.x, s4.y), s23 = make_float2(s4.z, s4.w);
      if (!fold) {
        s01 = fmul2(s01, make_float2(ys, ys));
        s23 = fmul2(s23, make_float2(ys, ys));
      }
      float2 a01 = make_float2(y[j], y[j + 1]), a23 = make_float2(y[j + 2], y[j + 3]);
      if (has_bias) {
        const float4 b4 = lds_f4(col_s + (uint32_t)BN * 4u + o);
        a01 = ffma2(a01, s01, make_float2(b4.x, b4.y));
        a23 = ffma2(a23, s23, make_float2(b4.z, b4.w));
      } else {
        a01 = fmul2(a01, s01);
        a23 = fmul2(a23, s23);
      }
      y[j] = a01.x; y[j + 1] = a01.y; y[j + 2] = a23.x; y[j + 3] = a23.y;
    }
    if (threadIdx.x == 64) LOKA_TRACE(8);

    // ---- per-thread statistics over its nv valid columns ----
    RowRec rec;
    rec.init();
    const bool need_minmax = is_fp8_out && !affine;
    const bool need_stats = norm != LOKA_NORM_NONE || need_minmax;
    // ---- NEXT-1 backward: g = dh * act'(xhat*gamma + beta) * gamma; per-row sums of g and g*xhat
    //      (the LayerNorm / RMSNorm backward's two reductions) in the forward's record slots:
    //      rec.mean = mean(g) over the thread's columns, rec.ss = sum(g * xhat) ----
    // x-hat of this thread's 8 columns j..j+7 (bf16, one 16-byte load; re-read in the finalize pass
    // instead of being held next to dh, so the backward fits every tile width)
    auto load_xh8 = [&](int j, float (&xv)[8]) {
      const __nv_bfloat16* xr = p.xhat + (int64_t)(row_ok ? grow : 0) * p.ld_xhat + n0 + cb + j;
      if (row_ok && cb + j + 8 <= ncols) {
        const uint4 w = __ldg(reinterpret_cast<const uint4*>(xr));
        xv[0] = bf16lo_to_f32(w.x); xv[1] = bf16hi_to_f32(w.x); xv[2] = bf16lo_to_f32(w.y); xv[3] = bf16hi_to_f32(w.y);
        xv[4] = bf16lo_to_f32(w.z); xv[5] = bf16hi_to_f32(w.z); xv[6] = bf16lo_to_f32(w.w); xv[7] = bf16hi_to_f32(w.w);
      } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) xv[k] = (row_ok && cb + j + k < ncols) ? __bfloat162float(xr[k]) : 0.f;
      }
    };
    if (bwd) {
      float sg = 0.f, sgx = 0.f;
#pragma unroll
      for (int j = 0; j < CPT; j += 8) {
        float xv[8];
        load_xh8(j, xv);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t o = (uint32_t)(cb + j + k) * 4u;
          const float gam = col[2 * BN + cb + j + k], bet = col[3 * BN + cb + j + k];
          (void)o;
          float g = y[j + k];
          if (p.act == LOKA_ACT_HARDSWISH) {  // PyTorch's hardswish' convention at the kinks
            const float yp = fmaf(xv[k], gam, bet);
            g *= yp < -3.f ? 0.f : (yp <= 3.f ? fmaf(yp, 1.f / 3.f, 0.5f) : 1.f);
          }
          g = (cb + j + k < ncols) ? g * gam : 0.f;
          y[j + k] = g;
          sg += g;
          sgx = fmaf(g, xv[k], sgx);
        }
      }
      rec.init();
      rec.n = (float)nv;
      rec.mean = nv > 0 ? sg / (float)nv : 0.f;
      rec.m2 = 0.f;
      rec.ss = sgx;
      rec.ymax = rec.ymin = 0.f;
    }
    if (need_stats && nv > 0 && !bwd) {
      // Columns >= N of a ragged tile hold exact zeros (zero-filled B rows, s_b = bias = 0), so
      // sums need no mask; only max/min must skip them.
      const float* t = y;
      float cmax = y[0], cmin = y[0];
      if (nv == CPT) {
#pragma unroll
        for (int j = 0; j < CPT; j += 2) cmax = fmax3(cmax, y[j], y[j + 1]), cmin = fmin3(cmin, y[j], y[j + 1]);
      } else {
#pragma unroll
        for (int j = 0; j < CPT; ++j)
          if (j < nv) cmax = fmaxf(cmax, y[j]), cmin = fminf(cmin, y[j]);
      }
      rec.n = (float)nv;
      rec.ymax = cmax;
      rec.ymin = cmin;
      if (norm == LOKA_NORM_LAYER) {
        float2 s0 = make_float2(0.f, 0.f), s1 = s0, s2 = s0, s3 = s0;
#pragma unroll
        for (int j = 0; j < CPT; j += 8) {
          s0 = fadd2(s0, make_float2(t[j], t[j + 1]));
          s1 = fadd2(s1, make_float2(t[j + 2], t[j + 3]));
          s2 = fadd2(s2, make_float2(t[j + 4], t[j + 5]));
          s3 = fadd2(s3, make_float2(t[j + 6], t[j + 7]));
        }
        s0 = fadd2(fadd2(s0, s1), fadd2(s2, s3));
        const float mc = (s0.x + s0.y) / (float)nv;
        const float2 nm = make_float2(-mc, -mc);
        float2 q0 = make_float2(0.f, 0.f), q1 = q0;
#pragma unroll
        for (int j = 0; j < CPT; j += 4) {
          const float2 d0 = fadd2(make_float2(t[j], t[j + 1]), nm);
          const float2 d1 = fadd2(make_float2(t[j + 2], t[j + 3]), nm);
          q0 = ffma2(d0, d0, q0);
          q1 = ffma2(d1, d1, q1);
        }
        q0 = fadd2(q0, q1);
        float m2 = q0.x + q0.y;
        if (nv < CPT) m2 = fmaxf(0.f, m2 - (float)(CPT - nv) * mc * mc);  // masked lanes added mc^2 each
        rec.mean = mc;
        rec.m2 = m2;
      } else if (norm == LOKA_NORM_RMS || is_block) {
        float2 q0 = make_float2(0.f, 0.f), q1 = q0;
#pragma unroll
        for (int j = 0; j < CPT; j += 4) {
          const float2 a = make_float2(t[j], t[j + 1]), b = make_float2(t[j + 2], t[j + 3]);
          q0 = ffma2(a, a, q0);
          q1 = ffma2(b, b, q1);
        }
        q0 = fadd2(q0, q1);
        rec.ss = q0.x + q0.y;
      }
    }

    // ---- merge the four column quarters of each row (fixed order -> identical in all four) ----
    // BlockNorm blocks cover whole quarters (blk % CPT == 0): a thread keeps its own block's sum
    // and the per-quarter (ss, max|y|) needed for the row amax.
    float q_ss[4], q_ma[4];
    if (need_stats) {
      float* my = hx + (size_t)cq * (kRec + 1) * 128 + r;  // component-major: conflict-free
      my[0] = rec.n; my[128] = rec.mean; my[256] = rec.m2; my[384] = rec.ss; my[512] = rec.ymax; my[640] = rec.ymin;
      named_bar_sync(1, kEpiThreads);
      RowRec parts[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float* o = hx + (size_t)k * (kRec + 1) * 128 + r;
        RowRec& t = parts[k];
        t.n = o[0]; t.mean = o[128]; t.m2 = o[256]; t.ss = o[384]; t.ymax = o[512]; t.ymin = o[640];
        q_ss[k] = t.ss;
        q_ma[k] = t.n > 0.f ? fmaxf(t.ymax, -t.ymin) : 0.f;
      }
      rec = merge_recs(parts);
    }
    if (threadIdx.x == 64) LOKA_TRACE(9);

    // ---- cross-CTA statistics (Case 2): push records, cluster barrier, merge in rank order ----
    if (xchg_stats) {
      const uint32_t my_rank = cluster_ctarank();
      if (cq == 0) {
        const float4 v = bwd ? make_float4(rec.mean, rec.ss, 0.f, 0.f)
                             : make_float4(norm == LOKA_NORM_LAYER ? rec.mean : rec.ss, rec.m2, rec.ymax, rec.ymin);
        const uint32_t la = smem_u32(cs + ((size_t)my_rank * 128 + r) * 4);
        for (int rk = 0; rk < csize; ++rk) st_dsmem_f4(mapa_shared(la, (uint32_t)rk), v);
      }
      cluster_sync_all();
      // n-way merge in rank order straight from the pushed records (two passes over smem: the
      // same sums as merge_recs over the ranks, without a register array per rank)
      RowRec o;
      o.init();
      float sm = 0.f;
      for (int rk = 0; rk < csize; ++rk) {
        const float4 v = lds_f4(smem_u32(cs + ((size_t)rk * 128 + r) * 4));
        const float nk = (float)min(BN, p.N - rk * BN);
        o.n += nk;
        sm = fmaf(nk, (norm == LOKA_NORM_LAYER || bwd) ? v.x : 0.f, sm);
        o.ss += bwd ? v.y : (norm == LOKA_NORM_LAYER ? 0.f : v.x);
        o.ymax = fmaxf(o.ymax, v.z);
        o.ymin = fminf(o.ymin, v.w);
      }
      o.mean = o.n > 0.f ? __fdiv_rn(sm, o.n) : 0.f;
      float m2 = 0.f;
      for (int rk = 0; rk < csize && !bwd; ++rk) {
        const float4 v = lds_f4(smem_u32(cs + ((size_t)rk * 128 + r) * 4));
        const float nk = (float)min(BN, p.N - rk * BN);
        const float dk = (norm == LOKA_NORM_LAYER ? v.x : 0.f) - o.mean;
        m2 += v.y + nk * dk * dk;
      }
      o.m2 = m2;
      rec = o;
    }
    if (threadIdx.x == 64) LOKA_TRACE(10);

    // ---- finalize: v = fma(y, rstd, c0) (BlockNorm: rstd of the thread's block) ----
    const float eps_eff = fold ? __fdiv_rn(p.eps, __fmul_rn(sa, sa)) : p.eps;
    float rstd = 1.f, c0 = 0.f;
    if (norm == LOKA_NORM_LAYER) {
      rstd = __fdiv_rn(1.f, __fsqrt_rn(__fadd_rn(__fdiv_rn(rec.m2, rec.n), eps_eff)));
      c0 = -__fmul_rn(rec.mean, rstd);
    } else if (norm == LOKA_NORM_RMS) {
      rstd = __fdiv_rn(1.f, __fsqrt_rn(__fadd_rn(__fdiv_rn(rec.ss, rec.n), eps_eff)));
    }
    float q_rs[4] = {1.f, 1.f, 1.f, 1.f};  // BlockNorm: rstd of each quarter's block
    if (is_block) {
      const int qpb = blk / CPT;  // quarters per block
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int kb0 = (k / qpb) * qpb;
        float ss = 0.f;
#pragma unroll
        for (int k2 = 0; k2 < 4; ++k2)
          if (k2 >= kb0 && k2 < kb0 + qpb) ss += q_ss[k2];
        q_rs[k] = __fdiv_rn(1.f, __fsqrt_rn(__fadd_rn(__fdiv_rn(ss, (float)blk), eps_eff)));
      }
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (k == cq) rstd = q_rs[k];
    }
    if (threadIdx.x == 64) LOKA_TRACE(11);

    // ---- NEXT-1 backward finalize: dz = rstd (g - mean(g) - xhat mean(g xhat)) (LayerNorm),
    //      rstd (g - xhat mean(g xhat)) (RMSNorm; BlockNorm per block with the block's sums) ----
    {
      if (bwd) {
        float mg = 0.f, mgx = 0.f, rs = 0.f;
        if (is_block) {
          const int qpb = blk / CPT;
          const int kb0 = (cq / qpb) * qpb;
          float ss = 0.f;
#pragma unroll
          for (int k2 = 0; k2 < 4; ++k2)
            if (k2 >= kb0 && k2 < kb0 + qpb) ss += q_ss[k2];
          mgx = ss / (float)blk;
          rs = row_ok ? p.rstd_in[(int64_t)grow * (p.N / blk) + (n0 + cb) / blk] : 0.f;
        } else {
          mg = norm == LOKA_NORM_LAYER ? rec.mean : 0.f;
          mgx = rec.ss / rec.n;
          rs = row_ok ? p.rstd_in[grow] : 0.f;
        }
#pragma unroll
        for (int j = 0; j < CPT; j += 8) {
          float xv[8];
          load_xh8(j, xv);
#pragma unroll
          for (int k = 0; k < 8; ++k) y[j + k] = rs * (y[j + k] - mg - xv[k] * mgx);
        }
      }
    }
    // normalised values in place (registers)
    if (norm != LOKA_NORM_NONE && !bwd) {
      const float2 r2 = make_float2(rstd, rstd), c2 = make_float2(c0, c0);
      const bool save = p.save_xhat != nullptr && row_ok;
#pragma unroll
      for (int j = 0; j < CPT; j += 4) {
        float2 a = ffma2(make_float2(y[j], y[j + 1]), r2, c2);
        float2 b = ffma2(make_float2(y[j + 2], y[j + 3]), r2, c2);
        if (save) {  // NEXT-1: the normalised values (before gamma / beta / act) for the backward
          __nv_bfloat162 h0 = __floats2bfloat162_rn(a.x, a.y), h1 = __floats2bfloat162_rn(b.x, b.y);
          __nv_bfloat16* d = p.save_xhat + (int64_t)grow * p.ld_save_xhat + n0 + cb + j;
          if (cb + j + 4 <= ncols) {
            *reinterpret_cast<uint2*>(d) = make_uint2(*reinterpret_cast<uint32_t*>(&h0), *reinterpret_cast<uint32_t*>(&h1));
          } else {
            const __nv_bfloat16 hv[4] = {h0.x, h0.y, h1.x, h1.y};
            for (int k = 0; k < 4; ++k)
              if (cb + j + k < ncols) d[k] = hv[k];
          }
        }
        if (has_gb) {
          const uint32_t o = (uint32_t)(cb + j) * 4u;
          const float4 g4 = lds_f4(col_s + 2u * BN * 4u + o);
          const float4 e4 = lds_f4(col_s + 3u * BN * 4u + o);
          a = ffma2(a, make_float2(g4.x, g4.y), make_float2(e4.x, e4.y));
          b = ffma2(b, make_float2(g4.z, g4.w), make_float2(e4.z, e4.w));
        }
        y[j] = a.x; y[j + 1] = a.y; y[j + 2] = b.x; y[j + 3] = b.y;
      }
    }

    if (p.save_rstd && row_ok && !bwd && norm != LOKA_NORM_NONE) {  // rstd of z = acc * s_a * s_b (+ bias)
      const float rz = fold ? __fdiv_rn(rstd, sa) : rstd;
      if (is_block) {
        if (cb % blk == 0 && nv > 0) p.save_rstd[(int64_t)grow * (p.N / blk) + (n0 + cb) / blk] = rz;
      } else if (cq == 0 && blockIdx.y == 0) {
        p.save_rstd[grow] = rz;
      }
    }

    // ---- activation (PAPER.md:502 Hard Swish): x * ReLU6(x + 3) / 6 ----
    if (p.act == LOKA_ACT_HARDSWISH && !bwd) {
#pragma unroll
      for (int j = 0; j < CPT; ++j) {
        const float t = fminf(fmaxf(y[j] + 3.f, 0.f), 6.f);
        y[j] = __fdiv_rn(__fmul_rn(y[j], t), 6.f);
      }
    }

    // ---- FP8 output: row amax of the normalised values -> row scale ----
    float r_out = 1.f;
    if (is_fp8_out) {
      float amax = 0.f;
      if (!affine) {  // v is monotone in y: max |v| is attained at ymax or ymin, exactly
        if (is_block) {
#pragma unroll
          for (int k = 0; k < 4; ++k) amax = fmaxf(amax, __fmul_rn(q_ma[k], q_rs[k]));
        } else if (norm == LOKA_NORM_NONE) {
          amax = fmaxf(fabsf(rec.ymax), fabsf(rec.ymin));
        } else {
          amax = fmaxf(fabsf(fmaf(rec.ymax, rstd, c0)), fabsf(fmaf(rec.ymin, rstd, c0)));
        }
      } else {  // affine: max over this thread's values, then over the four quarters
#pragma unroll
        for (int j = 0; j < CPT; ++j)
          if (j < nv) amax = fmaxf(amax, fabsf(y[j]));
        hx[((size_t)cq * (kRec + 1) + kRec) * 128 + r] = amax;  // slot kRec: not read by the stats merge
        named_bar_sync(1, kEpiThreads);
        amax = 0.f;
#pragma unroll
        for (int k = 0; k < 4; ++k) amax = fmaxf(amax, hx[((size_t)k * (kRec + 1) + kRec) * 128 + r]);
      }
      if (xchg_amax) {  // push this CTA's row amax into slot [my rank] of every peer
        const uint32_t my_rank = cluster_ctarank();
        if (cq == 0) {
          const uint32_t la = smem_u32(&cs2[my_rank * 128 + r]);
          for (int rk = 0; rk < csize; ++rk) st_dsmem_f32(mapa_shared(la, (uint32_t)rk), amax);
        }
        cluster_sync_all();
        amax = 0.f;
        for (int rk = 0; rk < csize; ++rk) amax = fmaxf(amax, cs2[rk * 128 + r]);
      }
      if (__float_as_uint(amax) >= 0x7F800000u && p.status) atomicOr(p.status, LOKA_DEVSTATUS_NONFINITE);
      float s_out;
      if (p.out_dtype == LOKA_E4M3) scales_from_amax<LOKA_E4M3, LOKA_SCALE_F32>(amax, s_out, r_out);
      else scales_from_amax<LOKA_E5M2, LOKA_SCALE_F32>(amax, s_out, r_out);
      if (row_ok && blockIdx.y == 0 && cq == 0 && p.y_scales) p.y_scales[grow] = s_out;
    }
    if (threadIdx.x == 64) LOKA_TRACE(6);

    // ---- cast into a 128B-swizzled smem tile (aliasing the drained ring), then TMA store ----
    // Box b of the tile holds output bytes [128 b, 128 b + 128) of every row; 16-byte chunk c of
    // row r lives at b*16K + r*128 + ((c ^ (r & 7)) << 4), the TMA SWIZZLE_128B pattern, so the
    // 8 rows a quarter-warp writes land in 8 different bank groups (conflict-free) and the global
    // writes are whole 128-byte lines (OOB rows / columns are clipped by the TMA unit).
    if (p.amax_out) {  // NEXT-4: producer-side tensor amax over the stored values
      float m = 0.f;
#pragma unroll
      for (int j = 0; j < CPT; ++j)
        if (j < nv && row_ok) m = fmaxf(m, fabsf(p.out_dtype == LOKA_BF16 ? stored_bf16(y[j]) : y[j]));
      warp_amax_to(p.amax_out, m);
    }
    if (p.precast && row_ok) {
      float* dst = p.precast + (int64_t)grow * p.ld_pre + n0 + cb;
#pragma unroll
      for (int j = 0; j < CPT; ++j)
        if (j < nv) dst[j] = y[j];
    }
    const int esz = p.out_dtype == LOKA_F32 ? 4 : p.out_dtype == LOKA_BF16 ? 2 : 1;
    // box row width: 128 B (SWIZZLE_128B, chunk ^= r & 7) or, when a CTA row is only 64 B
    // (FP8 output, BN = 64), 64 B (SWIZZLE_64B, chunk ^= (r >> 1) & 3); must match make_map_out
    const uint32_t box_bytes = (uint32_t)min(128, BN * esz);
    const uint32_t stage_s = smem_u32(smem) + (uint32_t)C::kOffStage;
    auto put16 = [&](int chunk, uint4 v) {  // chunk = 16-byte chunk index within this thread's bytes
      const uint32_t bofs = (uint32_t)(cb * esz + 16 * chunk);
      const uint32_t c16 = (bofs % box_bytes) >> 4;
      const uint32_t sw = box_bytes == 128u ? (c16 ^ ((uint32_t)r & 7u)) : (c16 ^ (((uint32_t)r >> 1) & 3u));
      const uint32_t a = stage_s + (bofs / box_bytes) * (128u * box_bytes) + (uint32_t)r * box_bytes + (sw << 4);
      sts_u4(a, v);
    };
    if (p.out_dtype == LOKA_F32) {
#pragma unroll
      for (int k = 0; k < CPT / 4; ++k)
        put16(k, make_uint4(__float_as_uint(y[4 * k]), __float_as_uint(y[4 * k + 1]), __float_as_uint(y[4 * k + 2]),
                            __float_as_uint(y[4 * k + 3])));
    } else if (p.out_dtype == LOKA_BF16) {
#pragma unroll
      for (int k = 0; k < CPT / 8; ++k) {
        uint32_t w[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          __nv_bfloat162 hh = __floats2bfloat162_rn(y[8 * k + 2 * i], y[8 * k + 2 * i + 1]);
          w[i] = *reinterpret_cast<uint32_t*>(&hh);
        }
        put16(k, make_uint4(w[0], w[1], w[2], w[3]));
      }
    } else {
      const float2 rr = make_float2(r_out, r_out);
#pragma unroll
      for (int k = 0; k < CPT / 16; ++k) {
        uint32_t w[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int j = 16 * k + 4 * i;
          const float2 a = fmul2(make_float2(y[j], y[j + 1]), rr);
          const float2 b = fmul2(make_float2(y[j + 2], y[j + 3]), rr);
          w[i] = p.out_dtype == LOKA_E4M3 ? cvt_fp8x4<LOKA_E4M3>(a.x, a.y, b.x, b.y)
                                           : cvt_fp8x4<LOKA_E5M2>(a.x, a.y, b.x, b.y);
        }
        put16(k, make_uint4(w[0], w[1], w[2], w[3]));
      }
    }
    fence_proxy_async_smem();
    named_bar_sync(1, kEpiThreads);
    if (threadIdx.x == 0) {
      const int per_box = (int)box_bytes / esz;  // output elements per box row
      const int nbox = BN * esz / (int)box_bytes;
      for (int b = 0; b < nbox; ++b) {
        const int c0 = n0 + b * per_box;
        if (c0 < p.N)
          tma_store_2d(&tma_y, reinterpret_cast<const uint8_t*>(smem) + C::kOffStage + b * 128 * (int)box_bytes, c0, m0);
      }
      bulk_commit();
      bulk_wait_read0();  // the tile must stay in smem until the TMA unit has read it
    }
    if (threadIdx.x == 64) LOKA_TRACE(7);
    if (csize > 1) cluster_sync_all();  // peers may still be pushing into / reading our smem
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<C::kTmemCols>(tmem_base);
  }
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

long long debug_trace(int enable, unsigned long long* out, long long n) {
  long long got = 0;
  if (out && n > 0) {
    got = n < (long long)kTraceCtas * 16 ? n : (long long)kTraceCtas * 16;
    if (cudaMemcpyFromSymbol(out, g_trace, (size_t)got * 8) != cudaSuccess) return -1;
  }
  if (n > (long long)kTraceCtas * 16) {
    const long long g2 = stack_debug_trace(enable, out + (size_t)kTraceCtas * 16, n - (long long)kTraceCtas * 16);
    if (g2 < 0) return -1;
    got += g2;
  } else if (stack_debug_trace(enable, nullptr, 0) < 0) {
    return -1;
  }
  if (enable >= 0) {
    if (enable) {
      static unsigned long long zero[kTraceCtas * 16];
      cudaMemcpyToSymbol(g_trace, zero, sizeof(zero));
    }
    cudaMemcpyToSymbol(g_trace_on, &enable, sizeof(int));
  }
  return got;
}

template <int BN, int MX, int MAXC = kMaxCluster>
static cudaError_t launch_bn(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& ty, const LinearParams& p,
                             cudaStream_t st) {
  using C = LinCfg<BN, MX, MAXC>;
  {
    cudaError_t e = ensure_func_attrs(reinterpret_cast<const void*>(linear_norm_kernel<BN, MX, MAXC>), C::kSmemBytes,
                                      MAXC > 8);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)((p.M + 127) / 128), (unsigned)((p.N + BN - 1) / BN), 1);
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = C::kSmemBytes;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 1;
  attr[0].val.clusterDim.y = (unsigned)p.cluster_n;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  cudaError_t e = cudaLaunchKernelEx(&cfg, linear_norm_kernel<BN, MX, MAXC>, ta, tb, ty, p);
  note_launch();
  return e;
}

cudaError_t launch_linear(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& ty, const LinearParams& p,
                          int bn, cudaStream_t st) {
  if (p.cluster_n > kMaxCluster) {  // rows of 2304..4096 columns: 16-CTA cluster, BN = 256
    if (bn != 256 || p.mx || p.cluster_n > kBigCluster) return cudaErrorInvalidValue;
    return launch_bn<256, 0, kBigCluster>(ta, tb, ty, p, st);
  }
  if (p.mx == 2) {
    switch (bn) {
      case 128: return launch_bn<128, 2>(ta, tb, ty, p, st);
      case 256: return launch_bn<256, 2>(ta, tb, ty, p, st);
      default: return cudaErrorInvalidValue;
    }
  }
  if (p.mx) {
    switch (bn) {
      case 128: return launch_bn<128, 1>(ta, tb, ty, p, st);
      case 256: return launch_bn<256, 1>(ta, tb, ty, p, st);
      default: return cudaErrorInvalidValue;
    }
  }
  switch (bn) {
    case 64: return launch_bn<64, 0>(ta, tb, ty, p, st);
    case 128: return launch_bn<128, 0>(ta, tb, ty, p, st);
    case 256: return launch_bn<256, 0>(ta, tb, ty, p, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace loka
