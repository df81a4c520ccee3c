// stack.cu — a whole LRM MLP stack (BASELINE.json configs[1]: L layers of rowwise-e4m3 FP8 linear
// + LayerNorm, "many small GEMMs followed immediately by normalization") in ONE launch.
//
// A thread-block cluster of C CTAs owns a 128-row block of the batch; CTA `rank` owns the column
// slice [rank*BN_l, (rank+1)*BN_l) of every layer (BN_l = N_l / C).  Per layer:
//   * the layer input h_l (the MMA's A operand, 128 x K_l FP8) lives in every CTA's shared memory
//     in the 128B-swizzled K-major layout tcgen05 reads; only the weight slice streams (2-stage TMA
//     ring of BN_l x 128 stages, running ahead across layers);
//   * h_l arrives slice by slice (slice s = the columns rank s produced in layer l-1): one mbarrier
//     per slice; the MMAs consume the CTA's own slice first, then the peers' slices in the order
//     they are sent, so the all-gather of h_l overlaps layer l's MMAs;
//   * the epilogue (s_a folded into eps, packed FP32x2 statistics, quarter merge in smem, cluster
//     exchange of (mean|ss, M2, ymax, ymin) records pushed with DSMEM stores, one-FFMA
//     normalisation, row amax from ymax/ymin) produces the next layer's e4m3 codes and row scale
//     and writes the codes into the CTA's own A tile; the slice then reaches the peers through L2:
//     TMA store of its K blocks to a global hand-off buffer, then one TMA load per K block
//     multicast to every peer, completing on the peer's slice barrier (kStackGatherL2; the SM-to-SM
//     alternative — one bulk DSMEM copy per peer — measured ~4% slower).  Slices narrower than a
//     128-wide K block go by per-thread DSMEM stores + a cluster barrier;
//   * only the last layer's output goes to HBM (swizzled staging tile + TMA store); the global
//     hand-offs double as the saved activations training needs (loka_stack_args.h).
// Each layer is the arithmetic of a loka_fp8_linear_norm call with an E4M3/ROW output, up to the
// order of the FP32 accumulation and of the row-statistics merge.
//
// Where the time goes (tools/trace_stack.py): per CTA and layer, the L2 -> SM
// ingress (~40 B/clk per SM: the weight slice plus 3/4 of h_l) bounds the MMA phase; the FP32
// accumulator drain from TMEM (~64 B/clk: 1 us for 128 x 256) and the two cluster-wide merges
// bound the epilogue.
#include "common.cuh"
#include "launch.h"

namespace loka {

constexpr int kSThreads = 512;  // 16 warps: warp 0 lane 0 = TMA producer, warp 1 lane 0 = MMA issuer,
                                // then all 16 warps run each layer's epilogue
constexpr int kSStages = 2;
constexpr int kSKMax = 1024;
constexpr int kSOffA = 0;                                // [kb][128 rows][128 B] (<= 128 KB)
constexpr int kSOffW = 128 * kSKMax;                     // weight ring [stage][<= 256 rows][128 B]
constexpr int kSStageW = 256 * 128;
constexpr int kSOffCs = kSOffW + kSStages * kSStageW;    // [8][128] float4 cluster records
constexpr int kSOffCol = kSOffCs + 8 * 128 * 16;         // [256] W row scales of this slice
constexpr int kSOffHx = kSOffCol + 256 * 4;             // [4][128] float4 column-quarter records
constexpr int kSOffBar = kSOffHx + 4 * 128 * 16;
constexpr int kSSmem = kSOffBar + 256 + 1024;
static_assert(kSSmem <= 227 * 1024, "stack smem");

// Opt-in phase trace (loka_debug_trace): per CTA 64 globaltimer stamps — 0 entry, 1 setup done,
// then per layer l at 2 + 7 l: +0 first weight stage landed (MMA), +1 last MMA issued,
// +2 first accumulator half ready (epilogue), +3 quarters merged, +4 cluster merged,
// +5 codes pushed, +6 next layer's A complete (MMA issuer saw its last slice).
constexpr int kSTraceCtas = 512;
static __device__ unsigned long long g_strace[kSTraceCtas * 64];
static __device__ int g_strace_on;
// fine trace of layer 1 (clock64 per CTA: slots 0-31 thread 0, 32-63 warp 15 lane 0)
static __device__ unsigned long long g_sfine[kSTraceCtas * 64];
#define LOKA_FST(c, l, i)                                                                          \
  do {                                                                                             \
    if ((c).trace && (l) == 1 && (c).cta < kSTraceCtas && (threadIdx.x == 0 || threadIdx.x == 480)) \
      g_sfine[(c).cta * 64 + (threadIdx.x ? 32 : 0) + (i)] = clock64();                            \
  } while (0)
#define LOKA_STRACE(c, slot)                                                                    \
  do {                                                                                          \
    if ((c).trace && (c).cta < kSTraceCtas) g_strace[(c).cta * 64 + (slot)] = globaltimer_ns(); \
  } while (0)

struct SRow {
  float n, mean, m2, ss, ymax, ymin;
  LOKA_DEVINL void init() { n = 0.f; mean = 0.f; m2 = 0.f; ss = 0.f; ymax = -INFINITY; ymin = INFINITY; }
};
// Record of a row segment as one float4: (mean | sum of squares, M2, ymax, ymin); n is implicit.
LOKA_DEVINL float4 rec4(const SRow& r, int norm) {
  return make_float4(norm == LOKA_NORM_LAYER ? r.mean : r.ss, r.m2, r.ymax, r.ymin);
}
// Merge of kv <= K records of equal counts n_each (Chan et al. with equal weights: no division;
// inv_k = 1/kv).  Every CTA merges the same records in the same order: identical statistics.
template <int K>
LOKA_DEVINL SRow merge_eq(const float4 (&v)[K], int kv, float n_each, float inv_k, int norm) {
  SRow o;
  o.init();
  o.n = (float)kv * n_each;
  float s = 0.f, m2 = 0.f;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    if (k < kv) {
      s += v[k].x;
      m2 += v[k].y;
      o.ymax = fmaxf(o.ymax, v[k].z);
      o.ymin = fminf(o.ymin, v[k].w);
    }
  }
  if (norm == LOKA_NORM_LAYER) {
    o.mean = s * inv_k;
    float d2 = 0.f;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (k < kv) {
        const float d = v[k].x - o.mean;
        d2 = fmaf(d, d, d2);
      }
    }
    o.m2 = fmaf(n_each, d2, m2);
  } else {
    o.ss = s;
  }
  return o;
}
template <int K>
LOKA_DEVINL SRow merge_rows(const SRow (&r)[K]) {
  SRow o;
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
  o.mean = o.n > 0.f ? s * __frcp_rn(o.n) : 0.f;  // (statistics need not be correctly rounded)
  float m2 = 0.f;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const float d = r[k].mean - o.mean;
    m2 += r[k].m2 + r[k].n * d * d;
  }
  o.m2 = m2;
  return o;
}

// Issuing the MMAs per 128-column half (so the epilogue could drain half 0 while half 1 is being
// multiplied) was measured SLOWER: two N=128 passes re-read A from shared memory and the MMA
// becomes shared-memory-bandwidth bound (A + B bytes per FLOP double).  Kept switchable.
constexpr bool kSplitHalves = false;
// All-gather of a layer's hand-off among the cluster (StackParams::gather): through L2 (codes
// stored to global memory, multicast TMA loads back into the peers' A tiles), SM-to-SM by bulk
// DSMEM copies of the staged slice, or SM-to-SM straight from registers (st.async, each 16-B piece
// completing on the peer's slice mbarrier: no staging, fence, CTA barrier or store/load round trip).

// Layer schedule shared by the producer and the MMA issuer: unit u in [0, nh * nkb) is
// (half h = u / nkb, K block kb); within a half the K blocks go slice by slice, own slice first.
struct SPlan {
  int nh, hn, nkb, kps;
  bool sliced;
};
LOKA_DEVINL SPlan splan(const StackParams& p, int l) {
  SPlan s;
  const int bn = p.BN[l];
  s.nh = kSplitHalves && bn > 128 ? 2 : 1;
  s.hn = s.nh == 2 ? 128 : bn;
  s.nkb = (p.K[l] + 127) / 128;
  s.sliced = l > 0 && p.C > 1 && p.BN[l - 1] >= 128;
  s.kps = s.sliced ? p.BN[l - 1] / 128 : s.nkb;
  return s;
}
LOKA_DEVINL int unit_kb(const SPlan& s, int i, int rank, int C) {  // i = index within the half
  if (!s.sliced) return i;
  const int t = i / s.kps;
  const int src = (rank - t + C) % C;
  return src * s.kps + (i - t * s.kps);
}

struct SCtx {
  uint8_t* smem;
  uint32_t tmem_base;
  int warp, lane, q, cq, r, grow, m0, rank, C;
  int trace, cta;
  bool dbg;       // the debug (traced) instance: also honours p.precast (compile-time false otherwise)
  int norm_c;     // >= 0: every layer's norm, a compile-time constant in the specialised instance
  int gather_c;   // >= 0: the all-gather transport, a compile-time constant in the specialised instance
  uint64_t* a_bar;     // [8] per-slice "layer input complete" barriers
  uint64_t* half_bar;  // [2] accumulator half ready
  uint64_t* stat_bar;  // cluster row-statistics records arrived (one phase per layer)
  bool row_ok;
};

template <int SEG>
LOKA_DEVINL SRow seg_stats(const float* y, int norm) {
  SRow rec;
  rec.init();
  rec.n = (float)SEG;
  float cmax = y[0], cmin = y[0];
#pragma unroll
  for (int j = 0; j < SEG; j += 2) cmax = fmax3(cmax, y[j], y[j + 1]), cmin = fmin3(cmin, y[j], y[j + 1]);
  rec.ymax = cmax;
  rec.ymin = cmin;
  if (norm == LOKA_NORM_LAYER) {
    float2 s0 = make_float2(0.f, 0.f), s1 = s0, s2 = s0, s3 = s0;
#pragma unroll
    for (int j = 0; j < SEG; j += 8) {
      s0 = fadd2(s0, make_float2(y[j], y[j + 1]));
      s1 = fadd2(s1, make_float2(y[j + 2], y[j + 3]));
      s2 = fadd2(s2, make_float2(y[j + 4], y[j + 5]));
      s3 = fadd2(s3, make_float2(y[j + 6], y[j + 7]));
    }
    s0 = fadd2(fadd2(s0, s1), fadd2(s2, s3));
    const float mc = (s0.x + s0.y) / (float)SEG;
    const float2 nm = make_float2(-mc, -mc);
    float2 q0 = make_float2(0.f, 0.f), q1 = q0;
#pragma unroll
    for (int j = 0; j < SEG; j += 4) {
      const float2 d0 = fadd2(make_float2(y[j], y[j + 1]), nm);
      const float2 d1 = fadd2(make_float2(y[j + 2], y[j + 3]), nm);
      q0 = ffma2(d0, d0, q0);
      q1 = ffma2(d1, d1, q1);
    }
    q0 = fadd2(q0, q1);
    rec.mean = mc;
    rec.m2 = q0.x + q0.y;
  } else if (norm == LOKA_NORM_RMS) {
    float2 q0 = make_float2(0.f, 0.f), q1 = q0;
#pragma unroll
    for (int j = 0; j < SEG; j += 4) {
      const float2 a = make_float2(y[j], y[j + 1]), b = make_float2(y[j + 2], y[j + 3]);
      q0 = ffma2(a, a, q0);
      q1 = ffma2(b, b, q1);
    }
    q0 = fadd2(q0, q1);
    rec.ss = q0.x + q0.y;
  }
  return rec;
}

// One layer's epilogue: NH accumulator halves of SEG columns per thread (thread (q, cq) owns row
// r = 32 q + lane and, in half h, the columns h*128 + cq*SEG + [0, SEG)).  `sa` is the layer
// input's row scale; returns the next layer's row scale (or 1 for the last layer).
template <int NH, int SEG>
LOKA_DEVINL float stack_epilogue(const StackParams& p, const SCtx& c, int l, float sa, uint32_t& hph) {
  static_assert(NH == 1 || SEG == 32, "halves are 128 columns");
  constexpr int BN = NH == 2 ? 256 : 4 * SEG;
  constexpr int CPT = NH * SEG;
  const int norm = c.norm_c >= 0 ? c.norm_c : p.norm[l];
  const int N = p.N[l];
  const int n0 = c.rank * BN;
  const bool last = l + 1 == p.L;
  const bool fold = norm != LOKA_NORM_NONE;  // no bias in the stack: s_a goes into eps
  const uint32_t cs = smem_u32(c.smem + kSOffCs);
  const uint32_t hx = smem_u32(c.smem + kSOffHx);
  const uint32_t col_s = smem_u32(c.smem + kSOffCol);
  const float ys = fold ? 1.f : sa;
  // the cluster's records of this layer arrive as st.async transactions on stat_bar
  if (c.C > 1 && threadIdx.x == 0) mbar_arrive_expect_tx(c.stat_bar, (uint32_t)c.C * 128u * 16u);

  // ---- accumulator halves -> registers (dequant, partial statistics) as each half completes ----
  float y[CPT];
  SRow hrec[NH];
#pragma unroll
  for (int h = 0; h < NH; ++h) {
    LOKA_FST(c, l, 0);
    if (c.lane == 0) mbar_wait(&c.half_bar[h], (hph >> h) & 1u, 3);
    __syncwarp();
    tc_fence_after();
    LOKA_FST(c, l, 1);
    if (h == 0 && threadIdx.x == 0) LOKA_STRACE(c, 2 + 7 * l + 2);
    const int cbh = h * 128 + c.cq * SEG;
    const uint32_t taddr = c.tmem_base + ((uint32_t)(c.q * 32) << 16) + (uint32_t)cbh;
    float* yh = y + h * SEG;
    if constexpr (SEG >= 32) {
#pragma unroll
      for (int i = 0; i < SEG / 32; ++i) tmem_ld32_nowait(taddr + (uint32_t)(32 * i), yh + 32 * i);
    } else {
      tmem_ld16_nowait(taddr, yh);
    }
#pragma unroll
    for (int i = 0; i < SEG / 16; ++i) tmem_wait16(yh + 16 * i);
    LOKA_FST(c, l, 2);
#pragma unroll
    for (int j = 0; j < SEG; j += 4) {
      float4 s4 = lds_f4(col_s + (uint32_t)(cbh + j) * 4u);
      if (!fold) {
        const float2 u = fmul2(make_float2(s4.x, s4.y), make_float2(ys, ys));
        const float2 v = fmul2(make_float2(s4.z, s4.w), make_float2(ys, ys));
        s4 = make_float4(u.x, u.y, v.x, v.y);
      }
      const float2 a = fmul2(make_float2(yh[j], yh[j + 1]), make_float2(s4.x, s4.y));
      const float2 b = fmul2(make_float2(yh[j + 2], yh[j + 3]), make_float2(s4.z, s4.w));
      yh[j] = a.x; yh[j + 1] = a.y; yh[j + 2] = b.x; yh[j + 3] = b.y;
    }
    LOKA_FST(c, l, 3);
    hrec[h] = seg_stats<SEG>(yh, norm);
    LOKA_FST(c, l, 4);
  }
  hph ^= NH == 2 ? 3u : 1u;
  SRow rec = NH == 2 ? merge_rows(hrec) : hrec[0];

  // ---- merge the four column quarters (float4 records in a dedicated smem area) ----
  {
    const float4 mine = rec4(rec, norm);
    asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(hx + (uint32_t)(c.cq * 128 + c.r) * 16u), "f"(mine.x),
                 "f"(mine.y), "f"(mine.z), "f"(mine.w)
                 : "memory");
    named_bar_sync(1, kSThreads);
    LOKA_FST(c, l, 5);
    float4 parts[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) parts[k] = lds_f4(hx + (uint32_t)(k * 128 + c.r) * 16u);
    rec = merge_eq(parts, 4, (float)CPT, 0.25f, norm);
    LOKA_FST(c, l, 6);
    if (threadIdx.x == 0) LOKA_STRACE(c, 2 + 7 * l + 3);
  }
  // ---- cluster exchange: every CTA's row records st.async'ed to every CTA (own included),
  //      completing on each receiver's stat_bar; merged in rank order ----
  if (c.C > 1) {
    if (c.cq == 0) {
      const float4 v = rec4(rec, norm);
      const uint32_t la = cs + (uint32_t)(c.rank * 128 + c.r) * 16u, lb = smem_u32(c.stat_bar);
      for (int t = 0; t < c.C; ++t) {
        const uint32_t rk = (uint32_t)((c.rank + t) % c.C);
        st_async_u4(mapa_shared(la, rk), make_uint4(__float_as_uint(v.x), __float_as_uint(v.y), __float_as_uint(v.z),
                                                    __float_as_uint(v.w)),
                    mapa_shared(lb, rk));
      }
    }
    LOKA_FST(c, l, 7);
    // Receiving every peer's record also proves every cluster CTA finished this layer's MMAs
    // (a record is sent after its CTA's accumulator was ready): the peers' A tiles are free.
    mbar_wait(c.stat_bar, (uint32_t)l & 1u, 6);
    LOKA_FST(c, l, 8);
    if (threadIdx.x == 0) LOKA_STRACE(c, 2 + 7 * l + 4);
    float4 parts[8];
#pragma unroll
    for (int rk = 0; rk < 8; ++rk)
      parts[rk] = rk < c.C ? lds_f4(cs + (uint32_t)(rk * 128 + c.r) * 16u) : make_float4(0.f, 0.f, -INFINITY, INFINITY);
    rec = merge_eq(parts, c.C, (float)BN, __fdividef(1.f, (float)c.C), norm);  // (exact for C = 2, 4, 8)
    LOKA_FST(c, l, 9);
  }
  // ---- normalise (one FFMA) ----
  const float eps = p.eps[l];
  // rstd by the hardware reciprocal square root (~2 ulp): the statistics are FP32 estimates of
  // FP64 quantities anyway; only the FP8 scales derived from the normalised values are IEEE-exact
  const float eps_eff = fold ? __fdividef(eps, sa * sa) : eps;
  const float inv_n = __fdividef(1.f, rec.n);  // (exact for the power-of-two row widths)
  float rstd = 1.f, c0 = 0.f;
  if (norm == LOKA_NORM_LAYER) {
    rstd = rsqrtf(fmaf(rec.m2, inv_n, eps_eff));
    c0 = -__fmul_rn(rec.mean, rstd);
  } else if (norm == LOKA_NORM_RMS) {
    rstd = rsqrtf(fmaf(rec.ss, inv_n, eps_eff));
  }
  if (norm != LOKA_NORM_NONE) {
    const float2 r2 = make_float2(rstd, rstd), c2 = make_float2(c0, c0);
#pragma unroll
    for (int j = 0; j < CPT; j += 2) {
      const float2 a = ffma2(make_float2(y[j], y[j + 1]), r2, c2);
      y[j] = a.x;
      y[j + 1] = a.y;
    }
  }
  LOKA_FST(c, l, 10);
  if (l == 1 && threadIdx.x == 0) LOKA_STRACE(c, 58);
  const bool fp8_next = !last || p.out_dtype == LOKA_E4M3 || p.out_dtype == LOKA_E5M2;
  const int ofmt = last ? p.out_dtype : LOKA_E4M3;
  float s_out = 1.f, r_out = 1.f;
  if (fp8_next) {  // row amax of the normalised row (monotone in y: from ymax / ymin, exact)
    const float amax = norm == LOKA_NORM_NONE ? fmaxf(fabsf(rec.ymax), fabsf(rec.ymin))
                                              : fmaxf(fabsf(fmaf(rec.ymax, rstd, c0)), fabsf(fmaf(rec.ymin, rstd, c0)));
    if (__float_as_uint(amax) >= 0x7F800000u && p.status) atomicOr(p.status, LOKA_DEVSTATUS_NONFINITE);
    if (ofmt == LOKA_E5M2) scales_from_amax<LOKA_E5M2, LOKA_SCALE_F32>(amax, s_out, r_out);
    else scales_from_amax<LOKA_E4M3, LOKA_SCALE_F32>(amax, s_out, r_out);
  }
  if (c.dbg && fp8_next && p.precast[l] && c.row_ok) {  // tests: the values the cast below consumes
    float* dst = p.precast[l] + (size_t)c.grow * p.N[l] + n0 + c.cq * SEG;
#pragma unroll
    for (int h = 0; h < NH; ++h)
#pragma unroll
      for (int j = 0; j < SEG; ++j) dst[h * 128 + j] = y[h * SEG + j];
  }
  LOKA_FST(c, l, 11);
  if (l == 1 && threadIdx.x == 0) LOKA_STRACE(c, 59);
  if (!last) {
    // ---- next layer's A operand: codes into this CTA's swizzled A tile (+ saved hand-off) ----
    const float2 rr = make_float2(r_out, r_out);
    const uint32_t a_local = smem_u32(c.smem + kSOffA);
    uint8_t* hsave = p.h_save[l];
    const int gather = c.gather_c >= 0 ? c.gather_c : p.gather;
    const bool hybrid = gather == kStackGatherL2StAsync || gather == kStackGatherL2StAsync256;
    const int l2min = gather == kStackGatherL2StAsync256 ? 256 : 128;
    const bool gl2 = gather == kStackGatherL2 || hybrid;
    const bool st_async = (gather == kStackGatherStAsync || (hybrid && BN < l2min)) && c.C > 1;
    const bool l2_path = gl2 && BN >= l2min && c.C > 1;
    // st.async pieces complete on the receiver's barrier of this CTA's slice (a_bar[0] when the
    // slices are narrower than a K block and the next layer waits for the whole input at once)
    const uint32_t bar_own = smem_u32(&c.a_bar[BN >= 128 ? c.rank : 0]);
#pragma unroll
    for (int h = 0; h < NH; ++h) {
#pragma unroll
      for (int ch = 0; ch < SEG / 16; ++ch) {
        uint32_t w[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int j = h * SEG + 16 * ch + 4 * i;
          const float2 a = fmul2(make_float2(y[j], y[j + 1]), rr);
          const float2 b = fmul2(make_float2(y[j + 2], y[j + 3]), rr);
          w[i] = cvt_fp8x4<LOKA_E4M3>(a.x, a.y, b.x, b.y);
        }
        const int k = n0 + h * 128 + c.cq * SEG + 16 * ch;  // K index of the next layer
        const uint32_t off = (uint32_t)(k >> 7) * 16384u + (uint32_t)c.r * 128u +
                             ((((uint32_t)(k & 127) >> 4) ^ ((uint32_t)c.r & 7u)) << 4);
        sts_u4(a_local + off, make_uint4(w[0], w[1], w[2], w[3]));
        if (st_async) {
          for (int t = 1; t < c.C; ++t) {
            const uint32_t rk = (uint32_t)((c.rank + t) % c.C);
            st_async_u4(mapa_shared(a_local + off, rk), make_uint4(w[0], w[1], w[2], w[3]), mapa_shared(bar_own, rk));
          }
        } else if constexpr (BN < 128) {  // slice not contiguous in the swizzled tile: per-thread DSMEM stores
          const float4 v = make_float4(__uint_as_float(w[0]), __uint_as_float(w[1]), __uint_as_float(w[2]),
                                       __uint_as_float(w[3]));
          for (int rk = 0; rk < c.C; ++rk)
            if (rk != c.rank) st_dsmem_f4(mapa_shared(a_local + off, (uint32_t)rk), v);
        }
        if (hsave && c.row_ok && !l2_path)  // (L2 gather: TMA-stored below)
          *reinterpret_cast<uint4*>(hsave + (size_t)c.grow * p.h_ld[l] + k) = make_uint4(w[0], w[1], w[2], w[3]);
      }
    }
    if (p.hs_save[l] && c.row_ok && c.rank == 0 && c.cq == 0) p.hs_save[l][c.grow] = s_out;
    LOKA_FST(c, l, 15);
    LOKA_FST(c, l, 12);
    if (l == 1 && threadIdx.x == 0) LOKA_STRACE(c, 60);
    if (c.C == 1) {
      fence_proxy_async_smem();  // generic writes -> async proxy (own MMA)
      named_bar_sync(1, kSThreads);
      LOKA_FST(c, l, 13);
      if (threadIdx.x == 0) {
        mbar_arrive(&c.a_bar[0]);
        LOKA_STRACE(c, 2 + 7 * l + 5);
      }
    } else if (st_async) {
      // own codes: generic smem writes -> async proxy (own MMA); the peers' pieces are in flight
      fence_proxy_async_smem();
      named_bar_sync(1, kSThreads);
      if (threadIdx.x == 0) {
        const uint32_t bytes = (uint32_t)BN * 128u;
        if (BN >= 128) {
          mbar_arrive(&c.a_bar[c.rank]);  // own slice
          for (int s = 0; s < c.C; ++s)
            if (s != c.rank) mbar_arrive_expect_tx(&c.a_bar[s], bytes);  // peers' slices (same BN)
        } else {
          mbar_arrive_expect_tx(&c.a_bar[0], (uint32_t)(c.C - 1) * bytes);  // whole input, one barrier
        }
        LOKA_STRACE(c, 2 + 7 * l + 5);
      }
    } else if (l2_path) {
      // The slice [n0, n0 + BN) of h_{l+1} is BN/128 whole 16 KB K blocks of the A tile.  Its
      // codes also went to global memory (p.h_save[l], L2-resident); one TMA load per K block,
      // multicast to every peer, brings them back into the peers' A tiles and completes on each
      // peer's slice barrier a_bar[rank] — the all-gather runs on the L2 -> SM path instead of the
      // SM -> SM network (DSMEM: ~14-21 B/clk per SM, measured ~2x slower here).  Peers' A tiles
      // are free: the stat_bar wait above proved every cluster CTA's layer-l MMAs completed.
      // The data are this CTA's own writes, so a CTA-wide barrier orders them before the load.
      fence_proxy_async_smem();  // generic smem writes -> async proxy (TMA store source, own MMA)
      named_bar_sync(1, kSThreads);
      LOKA_FST(c, l, 13);
      if (l == 1 && threadIdx.x == 0) LOKA_STRACE(c, 61);
      if (threadIdx.x == 0) {
        const uint32_t bytes = (uint32_t)BN * 128u;
        // own slice complete: the next layer's MMAs on it start now, under the store round trip
        mbar_arrive(&c.a_bar[c.rank]);
        for (int s = 0; s < c.C; ++s)
          if (s != c.rank) mbar_arrive_expect_tx(&c.a_bar[s], bytes);  // peers' slices (same BN)
        // the slice's K blocks (already swizzled in A) -> global with TMA stores; wait until written
        for (int kb = n0 >> 7; kb < (n0 + BN) >> 7; ++kb) tma_store_2d(&p.th[l], c.smem + kSOffA + kb * 16384, kb * 128, c.m0);
        bulk_commit();
        bulk_wait0();
        fence_proxy_async_global();
        LOKA_FST(c, l, 14);
        const uint16_t mask = (uint16_t)(((1u << c.C) - 1u) & ~(1u << c.rank));
        for (int kb = n0 >> 7; kb < (n0 + BN) >> 7; ++kb)
          tma_load_2d_mc(c.smem + kSOffA + kb * 16384, &p.th[l], &c.a_bar[c.rank], kb * 128, c.m0, mask);
        LOKA_STRACE(c, 2 + 7 * l + 5);
      }
    } else if (BN >= 128) {
      // DSMEM variant of the all-gather: one bulk (TMA-engine) shared::cta -> shared::cluster copy
      // of the slice per peer, completing on the peer's slice barrier a_bar[rank]; peers served in
      // rank order starting after this CTA (the order in which every receiver consumes slices).
      fence_proxy_async_smem();  // generic writes -> async proxy (bulk-copy source, own MMA)
      named_bar_sync(1, kSThreads);
      if (l == 1 && threadIdx.x == 0) LOKA_STRACE(c, 61);
      if (threadIdx.x == 0) {
        const uint32_t src = a_local + (uint32_t)(n0 >> 7) * 16384u, bytes = (uint32_t)BN * 128u;
        for (int t = 1; t < c.C; ++t) {
          const int rk = (c.rank + t) % c.C;
          bulk_copy_s2cluster(mapa_shared(src, (uint32_t)rk), src, bytes,
                              mapa_shared(smem_u32(&c.a_bar[c.rank]), (uint32_t)rk));
        }
        mbar_arrive(&c.a_bar[c.rank]);  // own slice
        for (int s = 0; s < c.C; ++s)
          if (s != c.rank) mbar_arrive_expect_tx(&c.a_bar[s], bytes);  // peers' slices (same BN)
        LOKA_STRACE(c, 2 + 7 * l + 5);
      }
    } else {
      asm volatile("fence.proxy.async.shared::cluster;" ::: "memory");  // generic writes -> tensor-core reads
      if (threadIdx.x == 0) LOKA_STRACE(c, 2 + 7 * l + 5);
      cluster_sync_all();  // barrier 2: h_{l+1} complete in every CTA
      if (threadIdx.x == 0) mbar_arrive(&c.a_bar[0]);
    }
    return s_out;
  }
  // ---- last layer: output tile -> swizzled staging (reuses A) -> TMA store ----
  if (fp8_next && c.row_ok && c.rank == 0 && c.cq == 0 && p.y_scales) p.y_scales[c.grow] = s_out;
  const int esz = p.out_dtype == LOKA_F32 ? 4 : p.out_dtype == LOKA_BF16 ? 2 : 1;
  const uint32_t box_bytes = (uint32_t)min(128, BN * esz);
  const uint32_t stage_s = smem_u32(c.smem + kSOffA);
  auto put16 = [&](int lcol, uint4 v) {  // lcol: local column (within BN) of the piece's first element
    const uint32_t bofs = (uint32_t)(lcol * esz);
    const uint32_t c16 = (bofs % box_bytes) >> 4;
    const uint32_t sw = box_bytes == 128u ? (c16 ^ ((uint32_t)c.r & 7u)) : (c16 ^ (((uint32_t)c.r >> 1) & 3u));
    sts_u4(stage_s + (bofs / box_bytes) * (128u * box_bytes) + (uint32_t)c.r * box_bytes + (sw << 4), v);
  };
#pragma unroll
  for (int h = 0; h < NH; ++h) {
    const int lc = h * 128 + c.cq * SEG;
    const float* yh = y + h * SEG;
    if (esz == 4) {
#pragma unroll
      for (int k = 0; k < SEG / 4; ++k)
        put16(lc + 4 * k, make_uint4(__float_as_uint(yh[4 * k]), __float_as_uint(yh[4 * k + 1]),
                                     __float_as_uint(yh[4 * k + 2]), __float_as_uint(yh[4 * k + 3])));
    } else if (esz == 2) {
#pragma unroll
      for (int k = 0; k < SEG / 8; ++k) {
        uint32_t w[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          __nv_bfloat162 hh = __floats2bfloat162_rn(yh[8 * k + 2 * i], yh[8 * k + 2 * i + 1]);
          w[i] = *reinterpret_cast<uint32_t*>(&hh);
        }
        put16(lc + 8 * k, make_uint4(w[0], w[1], w[2], w[3]));
      }
    } else {
      const float2 rr = make_float2(r_out, r_out);
#pragma unroll
      for (int k = 0; k < SEG / 16; ++k) {
        uint32_t w[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int j = 16 * k + 4 * i;
          const float2 a = fmul2(make_float2(yh[j], yh[j + 1]), rr);
          const float2 b = fmul2(make_float2(yh[j + 2], yh[j + 3]), rr);
          w[i] = ofmt == LOKA_E5M2 ? cvt_fp8x4<LOKA_E5M2>(a.x, a.y, b.x, b.y) : cvt_fp8x4<LOKA_E4M3>(a.x, a.y, b.x, b.y);
        }
        put16(lc + 16 * k, make_uint4(w[0], w[1], w[2], w[3]));
      }
    }
  }
  fence_proxy_async_smem();
  named_bar_sync(1, kSThreads);
  if (threadIdx.x == 0) {
    const int per_box = (int)box_bytes / esz, nbox = BN * esz / (int)box_bytes;
    for (int b = 0; b < nbox; ++b) {
      const int c0b = n0 + b * per_box;
      if (c0b < N) tma_store_2d(&p.ty, c.smem + kSOffA + b * 128 * (int)box_bytes, c0b, c.m0);
    }
    bulk_commit();
    bulk_wait_read0();
  }
  return 1.f;
}

// TRACE = false (the production instance) makes c.trace a compile-time 0: every trace stamp and
// its predicate logic is compiled out of the epilogue (~10% of its instructions).
// CT > 0: the cluster size as a compile-time constant (CT = p.C), so the rank-order loops unroll and
// the modular rank arithmetic of the exchange and of the slice order folds (cfg2: C = 4).
// GT >= 0: every layer is LayerNorm and the all-gather transport is GT (cfg2: L2), both compile-time.
template <bool TRACE, int CT, int GT>
__global__ void __launch_bounds__(kSThreads, 1) stack_kernel(const __grid_constant__ StackParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem + kSOffA;
  uint8_t* sW = smem + kSOffW;
  float* col = reinterpret_cast<float*>(smem + kSOffCol);
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + kSOffBar);
  uint64_t* empty_bar = full_bar + kSStages;
  uint64_t* a_bar = empty_bar + kSStages;  // [8]
  uint64_t* half_bar = a_bar + 8;          // [2]
  uint64_t* stat_bar = half_bar + 2;       // [1]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(stat_bar + 1);

  SCtx c;
  c.smem = smem;
  c.warp = threadIdx.x >> 5;
  c.lane = threadIdx.x & 31;
  c.q = c.warp & 3;
  c.cq = c.warp >> 2;
  c.r = c.q * 32 + c.lane;
  c.m0 = blockIdx.x * 128;
  c.grow = c.m0 + c.r;
  c.row_ok = c.grow < p.M;
  c.C = CT > 0 ? CT : p.C;
  c.norm_c = GT >= 0 ? (int)LOKA_NORM_LAYER : -1;
  c.gather_c = GT;
  c.rank = c.C > 1 ? (int)cluster_ctarank() : 0;
  c.a_bar = a_bar;
  c.half_bar = half_bar;
  c.stat_bar = stat_bar;
  c.trace = TRACE ? *reinterpret_cast<volatile int*>(&g_strace_on) : 0;
  c.dbg = TRACE;
  c.cta = blockIdx.x + gridDim.x * blockIdx.y;
  if (threadIdx.x == 0) LOKA_STRACE(c, 0);

  if (c.warp == 0 && c.lane == 0) {
    tma_prefetch_desc(&p.tx);
    tma_prefetch_desc(&p.ty);
    for (int l = 0; l < p.L; ++l) tma_prefetch_desc(&p.tw[l]);
    for (int s = 0; s < kSStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 8; ++s) mbar_init(&a_bar[s], 1);
    for (int h = 0; h < 2; ++h) mbar_init(&half_bar[h], 1);
    mbar_init(stat_bar, 1);
    fence_barrier_init();
  }
  if (c.warp == 1) tmem_alloc<256>(tmem_slot);
  pdl_wait();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  c.tmem_base = *tmem_slot;
  if (c.C > 1) cluster_sync_all();  // every cluster CTA is running before any DSMEM traffic
  if (threadIdx.x == 0) LOKA_STRACE(c, 1);

  float sa = c.row_ok ? p.xs[c.grow] : 0.f;  // row scale of the current layer input
  int prod_it = 0, mma_it = 0;
  uint32_t aph = 0;  // MMA issuer: parity of each slice barrier's next phase
  uint32_t hph = 0;  // epilogue: parity of each accumulator-half barrier's next phase
  auto produce = [&](int l, int u) {
    const SPlan s = splan(p, l);
    const int h = u / s.nkb;
    const int kb = unit_kb(s, u - h * s.nkb, c.rank, c.C);
    const int st = prod_it % kSStages;
    mbar_wait(&empty_bar[st], ((uint32_t)(prod_it / kSStages) & 1u) ^ 1u, 1);
    mbar_arrive_expect_tx(&full_bar[st], (uint32_t)(s.hn * 128));
    tma_load_2d(sW + st * kSStageW, &p.tw[l], &full_bar[st], kb * 128, c.rank * p.BN[l] + h * 128);
    ++prod_it;
  };
  int prefetched = 0;  // units of the current layer already issued during the previous layer
  for (int l = 0; l < p.L; ++l) {
    const SPlan pl = splan(p, l);
    const int units = pl.nh * pl.nkb;
    if (c.warp == 0 && c.lane == 0) {  // ===== producer =====
      if (l == 0) {
        mbar_arrive_expect_tx(&a_bar[0], (uint32_t)(pl.nkb * 128 * 128));
        for (int kb = 0; kb < pl.nkb; ++kb) tma_load_2d(sA + kb * 16384, &p.tx, &a_bar[0], kb * 128, c.m0);
      }
      for (int u = prefetched; u < units; ++u) produce(l, u);
      prefetched = 0;
      if (l + 1 < p.L) {  // run ahead into the next layer's weights while this layer finishes
        const SPlan nx = splan(p, l + 1);
        const int nn = min(kSStages, nx.nh * nx.nkb);
        for (int u = 0; u < nn; ++u) produce(l + 1, u);
        prefetched = nn;
      }
    }
    if (c.warp == 1 && c.lane == 0) {  // ===== MMA issuer =====
      const uint32_t idesc = idesc_f8f6f4(0, 0, 128, (uint32_t)pl.hn);
      for (int h = 0; h < pl.nh; ++h) {
        for (int i = 0; i < pl.nkb; ++i) {
          const int kb = unit_kb(pl, i, c.rank, c.C);
          if (h == 0 && i % pl.kps == 0) {  // first use of a slice of h_l: wait until it is complete
            const int src = kb / pl.kps;
            mbar_wait(&a_bar[src], (aph >> src) & 1u, 5);
            aph ^= 1u << src;
            tc_fence_after();
            fence_proxy_async_smem();  // peers' st.async pieces (generic proxy) -> this thread's MMAs
            if (l > 0) LOKA_STRACE(c, 2 + 7 * (l - 1) + 6);
          }
          const int st = mma_it % kSStages;
          mbar_wait(&full_bar[st], (uint32_t)(mma_it / kSStages) & 1u, 2);
          tc_fence_after();
          if (h == 0 && i == 0) LOKA_STRACE(c, 2 + 7 * l);
          const uint32_t a0 = smem_u32(sA + kb * 16384), b0 = smem_u32(sW + st * kSStageW);
#pragma unroll
          for (int k = 0; k < 4; ++k)
            mma_f8f6f4(c.tmem_base + (uint32_t)(h * 128), smem_desc_kmajor_sw128(a0 + k * 32),
                       smem_desc_kmajor_sw128(b0 + k * 32), idesc, (i | k) != 0);
          mma_commit(&empty_bar[st]);
          ++mma_it;
        }
        mma_commit(&half_bar[h]);
      }
      LOKA_STRACE(c, 2 + 7 * l + 1);
    }
    __syncwarp();
    LOKA_FST(c, l, 16);
    // ===== epilogue (all warps) =====
    const float* ws = p.ws[l];
    for (int j = threadIdx.x; j < p.BN[l]; j += kSThreads) col[j] = ws[c.rank * p.BN[l] + j];
    named_bar_sync(1, kSThreads);
    LOKA_FST(c, l, 17);
    float s_next;
    switch (p.BN[l]) {
      case 64: s_next = stack_epilogue<1, 16>(p, c, l, sa, hph); break;
      case 128: s_next = stack_epilogue<1, 32>(p, c, l, sa, hph); break;
      default:
        s_next = kSplitHalves ? stack_epilogue<2, 32>(p, c, l, sa, hph) : stack_epilogue<1, 64>(p, c, l, sa, hph);
        break;
    }
    sa = c.row_ok ? s_next : 0.f;
    tc_fence_before();  // this layer's tcgen05.ld done before the next layer's MMAs overwrite TMEM
  }
  if (c.C > 1) cluster_sync_all();
  __syncthreads();
  if (c.warp == 1) {
    tc_fence_after();
    tmem_dealloc<256>(c.tmem_base);
  }
}

static bool g_strace_host = false;  // launch the traced instance (set by loka_debug_trace)

long long stack_debug_trace(int enable, unsigned long long* out, long long n) {
  long long got = 0;
  if (out && n > 0) {
    got = n < (long long)kSTraceCtas * 64 ? n : (long long)kSTraceCtas * 64;
    if (cudaMemcpyFromSymbol(out, g_strace, (size_t)got * 8) != cudaSuccess) return -1;
    if (n > got) {  // the fine layer-1 trace follows
      const long long g2 = n - got < (long long)kSTraceCtas * 64 ? n - got : (long long)kSTraceCtas * 64;
      if (cudaMemcpyFromSymbol(out + got, g_sfine, (size_t)g2 * 8) != cudaSuccess) return -1;
      got += g2;
    }
  }
  if (enable >= 0) {
    if (enable) {
      static unsigned long long zero[kSTraceCtas * 64];
      if (cudaMemcpyToSymbol(g_strace, zero, sizeof(zero)) != cudaSuccess) return -1;
      if (cudaMemcpyToSymbol(g_sfine, zero, sizeof(zero)) != cudaSuccess) return -1;
    }
    if (cudaMemcpyToSymbol(g_strace_on, &enable, sizeof(int)) != cudaSuccess) return -1;
    g_strace_host = enable != 0;
  }
  return got;
}

cudaError_t launch_stack(const StackParams& p, cudaStream_t st) {
  bool all_ln = true;
  for (int l = 0; l < p.L; ++l) all_ln = all_ln && p.norm[l] == LOKA_NORM_LAYER;
  // (a DSMEM-gather instance was measured 2 us slower per step than the L2 one: not instantiated)
  const bool spec = p.C == 4 && all_ln && (p.gather == kStackGatherL2 || p.gather == kStackGatherL2StAsync);
  const bool hyb = p.gather == kStackGatherL2StAsync;
  bool dump = false;  // debug pre-cast dump: the traced instance carries it
  for (int l = 0; l < p.L; ++l) dump = dump || p.precast[l] != nullptr;
  const int inst = ((g_strace_host || dump) ? 3 : 0) + (spec ? (hyb ? 2 : 1) : 0);  // (mode 4: generic instance)
  auto kern = inst == 0   ? stack_kernel<false, 0, -1>
              : inst == 1 ? stack_kernel<false, 4, kStackGatherL2>
              : inst == 2 ? stack_kernel<false, 4, kStackGatherL2StAsync>
              : inst == 3 ? stack_kernel<true, 0, -1>
              : inst == 4 ? stack_kernel<true, 4, kStackGatherL2>
                          : stack_kernel<true, 4, kStackGatherL2StAsync>;
  {
    cudaError_t e = ensure_func_attrs(reinterpret_cast<const void*>(kern), kSSmem);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)((p.M + 127) / 128), (unsigned)p.C, 1);
  cfg.blockDim = dim3(kSThreads, 1, 1);
  cfg.dynamicSmemBytes = kSSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 1;
  attr[0].val.clusterDim.y = (unsigned)p.C;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, p);
  note_launch();
  return e;
}

}  // namespace loka
