// quantize_t.cu — a3: quantize with a K-major transposed copy (cast-transpose) and the column-
// spanning granularities (COL, BLK_128x1) the backward directions need ("separate
// optimization decisions for each direction", "RW GW HP"; D6):
//   dgrad dX = dY W    : B operand = W^T (K-major over N) -> W quantized per COLUMN, written transposed
//   wgrad dW = dY^T X  : A = dY^T, B = X^T (K-major over M) -> per COLUMN / 128x1, written transposed
//
// One CTA (256 threads) per 128 x 128 input tile: the tile is loaded with 16-byte loads into
// registers (64 elements per thread), granule amax is reduced within the tile (1x128: half warp,
// 128x1: per column across the tile, 128x128: whole CTA) or read from a pre-pass array
// (TENSOR / ROW / COL span beyond one tile), codes are written row-major directly and the
// transposed copy goes through a swizzled shared-memory tile and an in-register byte transpose so
// both layouts are written with coalesced 128-byte rows.  Same arithmetic as quantize.cu (bit-identical codes and scales).
#include "common.cuh"
#include "launch.h"

namespace loka {

template <typename Tin> struct In8;
template <> struct In8<__nv_bfloat16> {
  static LOKA_DEVINL void load(const __nv_bfloat16* p, int n, float (&f)[8]) {
    if (n == 8) {
      const uint4 w = __ldg(reinterpret_cast<const uint4*>(p));
      f[0] = bf16lo_to_f32(w.x); f[1] = bf16hi_to_f32(w.x); f[2] = bf16lo_to_f32(w.y); f[3] = bf16hi_to_f32(w.y);
      f[4] = bf16lo_to_f32(w.z); f[5] = bf16hi_to_f32(w.z); f[6] = bf16lo_to_f32(w.w); f[7] = bf16hi_to_f32(w.w);
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) f[i] = i < n ? __bfloat162float(p[i]) : 0.f;
    }
  }
};
template <> struct In8<float> {
  static LOKA_DEVINL void load(const float* p, int n, float (&f)[8]) {
    if (n == 8) {
      const float4 a = __ldg(reinterpret_cast<const float4*>(p)), b = __ldg(reinterpret_cast<const float4*>(p) + 1);
      f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w; f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) f[i] = i < n ? p[i] : 0.f;
    }
  }
};

LOKA_DEVINL uint32_t absbits(float v) { return __float_as_uint(v) & 0x7FFFFFFFu; }

// 8 input elements kept in their storage form (bf16: 4 registers) until the cast.
template <typename Tin> struct Raw8;
template <> struct Raw8<__nv_bfloat16> {
  uint32_t w[4];
  LOKA_DEVINL void load(const __nv_bfloat16* p, int n) {
    if (n == 8) {
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(p));
      w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w;
    } else {
      const uint16_t* h = reinterpret_cast<const uint16_t*>(p);
#pragma unroll
      for (int i = 0; i < 4; ++i)
        w[i] = (2 * i < n ? h[2 * i] : 0u) | ((2 * i + 1 < n ? (uint32_t)h[2 * i + 1] : 0u) << 16);
    }
  }
  LOKA_DEVINL void zero() { w[0] = w[1] = w[2] = w[3] = 0u; }
  LOKA_DEVINL float f(int k) const { return (k & 1) ? bf16hi_to_f32(w[k >> 1]) : bf16lo_to_f32(w[k >> 1]); }
  LOKA_DEVINL uint32_t abits(int k) const { return absbits(f(k)); }
};
template <> struct Raw8<float> {
  float v[8];
  LOKA_DEVINL void load(const float* p, int n) { In8<float>::load(p, n, v); }
  LOKA_DEVINL void zero() {
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = 0.f;
  }
  LOKA_DEVINL float f(int k) const { return v[k]; }
  LOKA_DEVINL uint32_t abits(int k) const { return absbits(v[k]); }
};

// ---- pre-pass: per-row amax (bit patterns) ------------------------------------------------
template <typename Tin>
__global__ void __launch_bounds__(256) row_amax_kernel(QuantParams p, uint32_t* amax_row) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (row >= p.rows) return;
  const Tin* xr = reinterpret_cast<const Tin*>(p.x) + row * p.ldx;
  uint32_t am = 0;
  int64_t c = lane * 8;
  for (; c + 768 + 8 <= p.cols; c += 1024) {  // 4 independent 16-byte loads in flight per lane
    float f[4][8];
#pragma unroll
    for (int u = 0; u < 4; ++u) In8<Tin>::load(xr + c + 256 * u, 8, f[u]);
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int i = 0; i < 8; ++i) am = max(am, absbits(f[u][i]));
  }
  for (; c < p.cols; c += 256) {
    float f[8];
    In8<Tin>::load(xr + c, (int)imin64(8, p.cols - c), f);
#pragma unroll
    for (int i = 0; i < 8; ++i) am = max(am, absbits(f[i]));
  }
  am = warp_max_u32(am);
  if (lane == 0) amax_row[row] = am;
  if (am >= 0x7F800000u && lane == 0 && p.status) atomicOr(p.status, LOKA_DEVSTATUS_NONFINITE);
}

// ---- pre-pass: per-column amax over all rows (atomicMax into a zeroed array) ---------------
template <typename Tin>
__global__ void __launch_bounds__(256) col_amax_kernel(QuantParams p, uint32_t* amax_col) {
  pdl_wait();
  __shared__ uint32_t red[8][128];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t c0 = (int64_t)blockIdx.x * 128, r0 = (int64_t)blockIdx.y * 128;
  const int cl = (lane & 15) * 8;
  uint32_t cm[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t row = r0 + warp * 16 + i * 2 + (lane >> 4);
    const int64_t c = c0 + cl;
    if (row < p.rows && c < p.cols) {
      float f[8];
      In8<Tin>::load(reinterpret_cast<const Tin*>(p.x) + row * p.ldx + c, (int)imin64(8, p.cols - c), f);
#pragma unroll
      for (int k = 0; k < 8; ++k) cm[k] = max(cm[k], absbits(f[k]));
    }
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) cm[k] = max(cm[k], __shfl_xor_sync(0xFFFFFFFFu, cm[k], 16));
  if (lane < 16) {
#pragma unroll
    for (int k = 0; k < 8; ++k) red[warp][cl + k] = cm[k];
  }
  __syncthreads();
  if (threadIdx.x < 128 && c0 + threadIdx.x < p.cols) {
    uint32_t m = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) m = max(m, red[w][threadIdx.x]);
    if (m) atomicMax(&amax_col[c0 + threadIdx.x], m);
    if (m >= 0x7F800000u && p.status) atomicOr(p.status, LOKA_DEVSTATUS_NONFINITE);
  }
}

// ---- tile kernel: granule scales + cast + row-major and/or transposed codes ----------------
// GRAN is a template parameter so the granularities whose scales come from a pre-pass (TENSOR /
// ROW / COL) carry no reduction state and run at 3 CTAs per SM.  amax_g: pre-pass array for
// TENSOR ([1], float bits) / ROW ([rows]) / COL ([cols]); else null.
//
// Transposed copy: the 128 x 128 code tile goes to shared memory row-major with its 16-byte chunks
// XOR-swizzled by (row / 8) & 7; each thread then reads an 8-row x 4-column block as eight 32-bit
// words (2-way bank conflicts at most), transposes it in registers with byte permutes (PRMT) and
// writes 4 transposed rows x 8 bytes; 16 lanes cover 128 contiguous bytes of a transposed row.
// GRAN = kGranDual: two quantizations of the same tile in one pass (the blockwise training recipe's
// X and dY, DeepSeek-V3 style): q = 1x128 granules (row-major codes for the forward / dgrad A
// operand) and qt = the 128x1 granules of x written transposed (K-major A / B of wgrad), i.e. the
// input is read once for both instead of once per granularity.
constexpr int kGranDual = 64;

template <typename Tin, int GRAN> struct TileOcc {
  static constexpr int kBlocks =
      sizeof(Tin) == 2 && (GRAN == LOKA_GRAN_TENSOR || GRAN == LOKA_GRAN_ROW || GRAN == LOKA_GRAN_COL) ? 3 : 2;
};

LOKA_DEVINL uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
  return d;
}
// 4 x 4 byte transpose: in[i] holds row i (bytes = columns 0..3); out[k] = column k (bytes = rows)
LOKA_DEVINL void transpose4x4(const uint32_t (&in)[4], uint32_t (&out)[4]) {
  const uint32_t t0 = prmt(in[0], in[1], 0x5140u), t1 = prmt(in[2], in[3], 0x5140u);
  const uint32_t t2 = prmt(in[0], in[1], 0x7362u), t3 = prmt(in[2], in[3], 0x7362u);
  out[0] = prmt(t0, t1, 0x5410u);
  out[1] = prmt(t0, t1, 0x7632u);
  out[2] = prmt(t2, t3, 0x5410u);
  out[3] = prmt(t2, t3, 0x7632u);
}
LOKA_DEVINL uint32_t tq_off(int row, int col) {  // byte offset of (row, col) in the swizzled code tile
  return (uint32_t)row * 128u + ((((uint32_t)col >> 4) ^ (((uint32_t)row >> 3) & 7u)) << 4) + ((uint32_t)col & 15u);
}

template <typename Tin, int FMT, int SF, int GRAN>
__global__ void __launch_bounds__(256, TileOcc<Tin, GRAN>::kBlocks) quant_tile_kernel(QuantParams p, const uint32_t* amax_g) {
  pdl_wait();
  __shared__ uint32_t red[8][128];
  __shared__ __align__(16) uint8_t tq[128 * 128];  // codes tile for the transposed write (swizzled)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t c0 = (int64_t)blockIdx.x * 128, r0 = (int64_t)blockIdx.y * 128;
  const int64_t nbc = (p.cols + 127) / 128, nbr = (p.rows + 127) / 128;
  const int cl = (lane & 15) * 8;  // local column of this lane's 8 elements
  const int64_t c = c0 + cl;
  const int nc = (int)max((int64_t)0, imin64(8, p.cols - c));
  Raw8<Tin> v[8];  // [row iteration], 8 elements each, storage form
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t row = r0 + warp * 16 + i * 2 + (lane >> 4);
    if (row < p.rows && nc > 0) v[i].load(reinterpret_cast<const Tin*>(p.x) + row * p.ldx + c, nc);
    else v[i].zero();
  }
  // ---- granule amax -> cast multiplier per element: rrow[i] (row-like) or rcol[k] (column-like) ----
  constexpr bool kColwise = GRAN == LOKA_GRAN_BLK_128x1 || GRAN == LOKA_GRAN_COL;
  constexpr bool kDual = GRAN == kGranDual;
  float rrow[8], rcol[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) rrow[i] = rcol[i] = 1.f;
  if constexpr (kDual) {  // 128x1 of x for the transposed copy (t-frame 1x128 scales [cols, nbr])
    uint32_t colm[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int k = 0; k < 8; ++k) colm[k] = max(colm[k], v[i].abits(k));
#pragma unroll
    for (int k = 0; k < 8; ++k) colm[k] = max(colm[k], __shfl_xor_sync(0xFFFFFFFFu, colm[k], 16));
    if (lane < 16) {
#pragma unroll
      for (int k = 0; k < 8; ++k) red[warp][cl + k] = colm[k];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      uint32_t m = 0;
#pragma unroll
      for (int w = 0; w < 8; ++w) m = max(m, red[w][cl + k]);
      float s, r;
      scales_from_amax<FMT, SF>(__uint_as_float(m), s, r);
      rcol[k] = r;
      if (warp == 0 && lane < 16 && k < nc && p.scales_t) p.scales_t[(c + k) * nbr + blockIdx.y] = s;
    }
  }
  if constexpr (GRAN == LOKA_GRAN_BLK_1x128 || kDual) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      uint32_t m = 0;
#pragma unroll
      for (int k = 0; k < 8; ++k) m = max(m, v[i].abits(k));
#pragma unroll
      for (int o = 8; o >= 1; o >>= 1) m = max(m, __shfl_xor_sync(0xFFFFFFFFu, m, o));
      if (m >= 0x7F800000u && (lane & 15) == 0 && p.status) atomicOr(p.status, LOKA_DEVSTATUS_NONFINITE);
      float s, r;
      scales_from_amax<FMT, SF>(__uint_as_float(m), s, r);
      const int64_t row = r0 + warp * 16 + i * 2 + (lane >> 4);
      if ((lane & 15) == 0 && row < p.rows) {
        if (p.scales) p.scales[row * nbc + blockIdx.x] = s;
        if (!kDual && p.scales_t) p.scales_t[(int64_t)blockIdx.x * p.rows + row] = s;  // t-frame BLK_128x1 [nbc, rows]
      }
      rrow[i] = r;
    }
  } else if constexpr (GRAN == LOKA_GRAN_BLK_1x32) {  // MX block: 4 lanes x 8 columns
    const int64_t nb32 = (p.cols + 31) / 32;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      uint32_t m = 0;
#pragma unroll
      for (int k = 0; k < 8; ++k) m = max(m, v[i].abits(k));
#pragma unroll
      for (int o = 2; o >= 1; o >>= 1) m = max(m, __shfl_xor_sync(0xFFFFFFFFu, m, o));
      if (m >= 0x7F800000u && (lane & 3) == 0 && p.status) atomicOr(p.status, LOKA_DEVSTATUS_NONFINITE);
      float s, r;
      scales_from_amax<FMT, SF>(__uint_as_float(m), s, r);
      const int64_t row = r0 + warp * 16 + i * 2 + (lane >> 4);
      if ((lane & 3) == 0 && row < p.rows && nc > 0 && p.scales) p.scales[row * nb32 + (c >> 5)] = s;
      rrow[i] = r;
    }
  } else if constexpr (GRAN == LOKA_GRAN_BLK_128x1 || GRAN == LOKA_GRAN_BLK_128x128) {
    uint32_t colm[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int k = 0; k < 8; ++k) colm[k] = max(colm[k], v[i].abits(k));
#pragma unroll
    for (int k = 0; k < 8; ++k) colm[k] = max(colm[k], __shfl_xor_sync(0xFFFFFFFFu, colm[k], 16));
    if (lane < 16) {
#pragma unroll
      for (int k = 0; k < 8; ++k) red[warp][cl + k] = colm[k];
    }
    __syncthreads();
    if constexpr (GRAN == LOKA_GRAN_BLK_128x1) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        uint32_t m = 0;
#pragma unroll
        for (int w = 0; w < 8; ++w) m = max(m, red[w][cl + k]);
        float s, r;
        scales_from_amax<FMT, SF>(__uint_as_float(m), s, r);
        rcol[k] = r;
        if (warp == 0 && lane < 16 && k < nc) {
          if (m >= 0x7F800000u && p.status) atomicOr(p.status, LOKA_DEVSTATUS_NONFINITE);
          if (p.scales) p.scales[(int64_t)blockIdx.y * p.cols + c + k] = s;     // [nbr, cols]
          if (p.scales_t) p.scales_t[(c + k) * nbr + blockIdx.y] = s;           // t-frame 1x128 [cols, nbr]
        }
      }
    } else {
      __shared__ uint32_t red2[8];
      uint32_t m = 0;
      if (threadIdx.x < 128) {
#pragma unroll
        for (int w = 0; w < 8; ++w) m = max(m, red[w][threadIdx.x]);
      }
      m = warp_max_u32(m);
      if (lane == 0) red2[warp] = m;
      __syncthreads();
      m = max(max(red2[0], red2[1]), max(red2[2], red2[3]));
      float s, r;
      scales_from_amax<FMT, SF>(__uint_as_float(m), s, r);
#pragma unroll
      for (int i = 0; i < 8; ++i) rrow[i] = r;
      if (threadIdx.x == 0) {
        if (m >= 0x7F800000u && p.status) atomicOr(p.status, LOKA_DEVSTATUS_NONFINITE);
        if (p.scales) p.scales[(int64_t)blockIdx.y * nbc + blockIdx.x] = s;
        if (p.scales_t) p.scales_t[(int64_t)blockIdx.x * nbr + blockIdx.y] = s;
      }
    }
  } else if constexpr (GRAN == LOKA_GRAN_TENSOR) {  // from the pre-pass amax word
    float s, r;
    scales_from_amax<FMT, SF>(__uint_as_float(amax_g[0]), s, r);
#pragma unroll
    for (int i = 0; i < 8; ++i) rrow[i] = r;
    if (threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0) {
      if (p.scales) p.scales[0] = s;
      if (p.scales_t) p.scales_t[0] = s;
    }
  } else if constexpr (GRAN == LOKA_GRAN_ROW) {  // from the pre-pass row amax array
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int64_t row = r0 + warp * 16 + i * 2 + (lane >> 4);
      float s, r;
      scales_from_amax<FMT, SF>(__uint_as_float(row < p.rows ? amax_g[row] : 0u), s, r);
      rrow[i] = r;
      if (cl == 0 && blockIdx.x == 0 && row < p.rows) {
        if (p.scales) p.scales[row] = s;
        if (p.scales_t) p.scales_t[row] = s;
      }
    }
  } else {  // COL from the pre-pass column amax array
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      float s, r;
      scales_from_amax<FMT, SF>(__uint_as_float(k < nc ? amax_g[c + k] : 0u), s, r);
      rcol[k] = r;
      if (warp == 0 && lane < 16 && blockIdx.y == 0 && k < nc) {
        if (p.scales) p.scales[c + k] = s;
        if (p.scales_t) p.scales_t[c + k] = s;
      }
    }
  }
  // ---- cast; row-major codes straight to global, the transposed copy through smem ----
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    float f[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) f[k] = __fmul_rn(v[i].f(k), kColwise ? rcol[k] : rrow[i]);
    const uint32_t lo = cvt_fp8x4<FMT>(f[0], f[1], f[2], f[3]), hi = cvt_fp8x4<FMT>(f[4], f[5], f[6], f[7]);
    const int lr = warp * 16 + i * 2 + (lane >> 4);
    const int64_t row = r0 + lr;
    if (p.q && row < p.rows && nc > 0) {
      uint8_t* dst = p.q + row * p.ldq + c;
      if (nc == 8) *reinterpret_cast<uint2*>(dst) = make_uint2(lo, hi);
      else
        for (int k = 0; k < nc; ++k) dst[k] = (uint8_t)((k < 4 ? lo : hi) >> (8 * (k & 3)));
    }
    if (p.qt) {
      if constexpr (kDual) {  // the 128x1 quantization for the transposed copy
#pragma unroll
        for (int k = 0; k < 8; ++k) f[k] = __fmul_rn(v[i].f(k), rcol[k]);
        *reinterpret_cast<uint2*>(&tq[tq_off(lr, cl)]) =
            make_uint2(cvt_fp8x4<FMT>(f[0], f[1], f[2], f[3]), cvt_fp8x4<FMT>(f[4], f[5], f[6], f[7]));
      } else {
        *reinterpret_cast<uint2*>(&tq[tq_off(lr, cl)]) = make_uint2(lo, hi);
      }
    }
  }
  if (p.qt) {
    __syncthreads();
#pragma unroll
    for (int it = 0; it < 2; ++it) {
      const int item = threadIdx.x + 256 * it;
      const int rg = item & 15, cg = item >> 4;  // rows 8rg..8rg+7, columns 4cg..4cg+3 of the tile
      uint32_t w[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) w[i] = *reinterpret_cast<const uint32_t*>(&tq[tq_off(8 * rg + i, 4 * cg)]);
      uint32_t lo[4], hi[4];
      transpose4x4({w[0], w[1], w[2], w[3]}, lo);
      transpose4x4({w[4], w[5], w[6], w[7]}, hi);
      const int64_t rb = r0 + 8 * rg;
      if (rb >= p.rows) continue;
      const int nr = (int)imin64(8, p.rows - rb);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int64_t orow = c0 + 4 * cg + k;
        if (orow >= p.cols) break;
        uint8_t* dst = p.qt + orow * p.ldqt + rb;
        if (nr == 8) *reinterpret_cast<uint2*>(dst) = make_uint2(lo[k], hi[k]);
        else
          for (int j = 0; j < nr; ++j) dst[j] = (uint8_t)((j < 4 ? lo[k] : hi[k]) >> (8 * (j & 3)));
      }
    }
  }
}

template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl_t(void (*kern)(KArgs...), dim3 grid, dim3 block, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  note_launch();
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

template <typename Tin, int FMT, int SF>
static cudaError_t launch_tiled_t(const QuantParams& p, int gran, int phase, float* amax_dev, void* ws,
                                  cudaStream_t st, QuantTileParams* tile, int num_sms) {
  const dim3 tiles((unsigned)((p.cols + 127) / 128), (unsigned)((p.rows + 127) / 128));
  uint32_t* amax = nullptr;
  cudaError_t e = cudaSuccess;
  if (gran == LOKA_GRAN_TENSOR) {
    amax = reinterpret_cast<uint32_t*>(amax_dev);
    if (phase != LOKA_PHASE_CAST_WITH_AMAX)  // FULL (AMAX_ONLY is handled by quantize.cu alone)
      e = launch_quantize(p, sizeof(Tin) == 2, FMT, SF, LOKA_GRAN_TENSOR, LOKA_PHASE_AMAX_ONLY, amax_dev, st, 148);
  } else if (gran == LOKA_GRAN_ROW) {
    amax = reinterpret_cast<uint32_t*>(ws);
    e = launch_pdl_t(row_amax_kernel<Tin>, dim3((unsigned)((p.rows + 7) / 8)), dim3(256), st, p, amax);
  } else if (gran == LOKA_GRAN_COL) {
    // ws: the pre-pass array (FULL) or the caller's column amax vector (split phases: AMAX_ONLY writes
    // it, CAST_WITH_AMAX reads the all-reduced one); |x| bit patterns order like the floats they are
    amax = reinterpret_cast<uint32_t*>(ws);
    if (phase != LOKA_PHASE_CAST_WITH_AMAX) {
      e = cudaMemsetAsync(amax, 0, (size_t)p.cols * 4, st);
      if (e == cudaSuccess) e = launch_pdl_t(col_amax_kernel<Tin>, tiles, dim3(256), st, p, amax);
      if (e != cudaSuccess || phase == LOKA_PHASE_AMAX_ONLY) return e;
    }
  }
  if (e != cudaSuccess) return e;
  const uint32_t* ag = amax;
  if (tile && sizeof(Tin) == 2) {  // the streaming kernel (bf16 input; api.cu built the maps)
    tile->amax_g = ag;
    return launch_quant_tile_tma(*tile, FMT, SF, gran, num_sms, st);
  }
  switch (gran) {
    case LOKA_GRAN_TENSOR: return launch_pdl_t(quant_tile_kernel<Tin, FMT, SF, LOKA_GRAN_TENSOR>, tiles, dim3(256), st, p, ag);
    case LOKA_GRAN_ROW: return launch_pdl_t(quant_tile_kernel<Tin, FMT, SF, LOKA_GRAN_ROW>, tiles, dim3(256), st, p, ag);
    case LOKA_GRAN_COL: return launch_pdl_t(quant_tile_kernel<Tin, FMT, SF, LOKA_GRAN_COL>, tiles, dim3(256), st, p, ag);
    case LOKA_GRAN_BLK_1x128:
      return launch_pdl_t(quant_tile_kernel<Tin, FMT, SF, LOKA_GRAN_BLK_1x128>, tiles, dim3(256), st, p, ag);
    case LOKA_GRAN_BLK_128x1:
      return launch_pdl_t(quant_tile_kernel<Tin, FMT, SF, LOKA_GRAN_BLK_128x1>, tiles, dim3(256), st, p, ag);
    case LOKA_GRAN_BLK_128x128:
      return launch_pdl_t(quant_tile_kernel<Tin, FMT, SF, LOKA_GRAN_BLK_128x128>, tiles, dim3(256), st, p, ag);
    case kGranDual: return launch_pdl_t(quant_tile_kernel<Tin, FMT, SF, kGranDual>, tiles, dim3(256), st, p, ag);
    case LOKA_GRAN_BLK_1x32:
      return launch_pdl_t(quant_tile_kernel<Tin, FMT, SF, LOKA_GRAN_BLK_1x32>, tiles, dim3(256), st, p, ag);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_quantize_tiled(const QuantParams& p, bool in_bf16, int fmt, int scale_fmt, int gran, int phase,
                                  float* amax_dev, void* ws, cudaStream_t st, QuantTileParams* tile, int num_sms) {
#define LOKA_T(T, F, S) \
  if (fmt == F && scale_fmt == S) return launch_tiled_t<T, F, S>(p, gran, phase, amax_dev, ws, st, tile, num_sms);
  if (in_bf16) {
    LOKA_T(__nv_bfloat16, LOKA_E4M3, LOKA_SCALE_F32)
    LOKA_T(__nv_bfloat16, LOKA_E4M3, LOKA_SCALE_UE8M0)
    LOKA_T(__nv_bfloat16, LOKA_E5M2, LOKA_SCALE_F32)
    LOKA_T(__nv_bfloat16, LOKA_E5M2, LOKA_SCALE_UE8M0)
  } else {
    LOKA_T(float, LOKA_E4M3, LOKA_SCALE_F32)
    LOKA_T(float, LOKA_E4M3, LOKA_SCALE_UE8M0)
    LOKA_T(float, LOKA_E5M2, LOKA_SCALE_F32)
    LOKA_T(float, LOKA_E5M2, LOKA_SCALE_UE8M0)
  }
#undef LOKA_T
  return cudaErrorNotSupported;
}

}  // namespace loka
