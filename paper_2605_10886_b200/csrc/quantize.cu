// quantize.cu — a1/a2/a3: granule amax -> scale -> saturating RNE cast to e4m3/e5m2.
//
// Definition (D1-D3, D7):
//   amax = max |x| over the granule (exact), s = fl32(amax/max), r = fl32(max/amax)
//   (UE8M0: s = 2^e smallest power of two >= amax/max), q = satRNE_fp8(fl32(x * r)).
//
// HBM-bound: 2 B (bf16) read + 1 B written per element.  Kernels read 16 B per lane per
// load (8 bf16), keep the row/block in registers between the amax reduction and the cast
// when it fits (one HBM read), and reduce amax on the integer bit pattern of |x|
// (NaN > Inf > finite, so a non-finite element is detected from the reduced amax alone).
#include <cstdlib>

#include "common.cuh"
#include "launch.h"

namespace loka {

// ----- element loading: 8 elements per lane as FP32 + max of |x| bit patterns ------------
template <typename Tin> struct Vec8;

template <> struct Vec8<__nv_bfloat16> {
  uint4 w;  // 8 bf16
  LOKA_DEVINL void load(const __nv_bfloat16* p) { w = __ldg(reinterpret_cast<const uint4*>(p)); }
  LOKA_DEVINL void load_partial(const __nv_bfloat16* p, int n) {
    uint16_t h[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) h[i] = i < n ? reinterpret_cast<const uint16_t*>(p)[i] : 0;
    w.x = h[0] | ((uint32_t)h[1] << 16);
    w.y = h[2] | ((uint32_t)h[3] << 16);
    w.z = h[4] | ((uint32_t)h[5] << 16);
    w.w = h[6] | ((uint32_t)h[7] << 16);
  }
  LOKA_DEVINL void zero() { w = make_uint4(0, 0, 0, 0); }
  // max of |x| as FP32 bit patterns (bf16 -> fp32 is a 16-bit shift, order preserved)
  LOKA_DEVINL uint32_t amax_bits() const {
    uint32_t m;
    uint32_t a = w.x & 0x7FFF7FFFu, b = w.y & 0x7FFF7FFFu, c = w.z & 0x7FFF7FFFu, d = w.w & 0x7FFF7FFFu;
    asm("max.u16x2 %0, %1, %2;" : "=r"(a) : "r"(a), "r"(b));
    asm("max.u16x2 %0, %1, %2;" : "=r"(c) : "r"(c), "r"(d));
    asm("max.u16x2 %0, %1, %2;" : "=r"(m) : "r"(a), "r"(c));
    return max(m & 0xFFFFu, m >> 16) << 16;
  }
  LOKA_DEVINL void to_f32(float (&f)[8]) const {
    f[0] = bf16lo_to_f32(w.x); f[1] = bf16hi_to_f32(w.x);
    f[2] = bf16lo_to_f32(w.y); f[3] = bf16hi_to_f32(w.y);
    f[4] = bf16lo_to_f32(w.z); f[5] = bf16hi_to_f32(w.z);
    f[6] = bf16lo_to_f32(w.w); f[7] = bf16hi_to_f32(w.w);
  }
};

template <> struct Vec8<float> {
  float4 a, b;
  LOKA_DEVINL void load(const float* p) {
    a = __ldg(reinterpret_cast<const float4*>(p));
    b = __ldg(reinterpret_cast<const float4*>(p) + 1);
  }
  LOKA_DEVINL void load_partial(const float* p, int n) {
    float h[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) h[i] = i < n ? p[i] : 0.0f;
    a = make_float4(h[0], h[1], h[2], h[3]);
    b = make_float4(h[4], h[5], h[6], h[7]);
  }
  LOKA_DEVINL void zero() { a = b = make_float4(0.f, 0.f, 0.f, 0.f); }
  LOKA_DEVINL uint32_t amax_bits() const {
    uint32_t m = __float_as_uint(a.x) & 0x7FFFFFFFu;
    m = max(m, __float_as_uint(a.y) & 0x7FFFFFFFu);
    m = max(m, __float_as_uint(a.z) & 0x7FFFFFFFu);
    m = max(m, __float_as_uint(a.w) & 0x7FFFFFFFu);
    m = max(m, __float_as_uint(b.x) & 0x7FFFFFFFu);
    m = max(m, __float_as_uint(b.y) & 0x7FFFFFFFu);
    m = max(m, __float_as_uint(b.z) & 0x7FFFFFFFu);
    m = max(m, __float_as_uint(b.w) & 0x7FFFFFFFu);
    return m;
  }
  LOKA_DEVINL void to_f32(float (&f)[8]) const {
    f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w;
    f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
  }
};

// 8 elements * r -> 8 codes (two u32).  fl32(x*r) is a plain IEEE multiply (no FMA, no FTZ).
template <int FMT, typename Tin>
LOKA_DEVINL uint2 cast8(const Vec8<Tin>& v, float r) {
  float f[8];
  v.to_f32(f);
#pragma unroll
  for (int i = 0; i < 8; ++i) f[i] = __fmul_rn(f[i], r);
  return make_uint2(cvt_fp8x4<FMT>(f[0], f[1], f[2], f[3]), cvt_fp8x4<FMT>(f[4], f[5], f[6], f[7]));
}

LOKA_DEVINL void store8(uint8_t* p, uint2 c, int n) {
  if (n >= 8) {
    *reinterpret_cast<uint2*>(p) = c;
  } else {
    const uint8_t* b = reinterpret_cast<const uint8_t*>(&c);
    for (int i = 0; i < n; ++i) p[i] = b[i];
  }
}

LOKA_DEVINL void flag_nonfinite(uint32_t amax_bits, int32_t* status) {
  if (amax_bits >= 0x7F800000u && status != nullptr) atomicOr(status, LOKA_DEVSTATUS_NONFINITE);
}

// ----- ROW: one warp per row; rows of <= 256*NREG elements stay in registers -------------
template <typename Tin, int FMT, int SF, int NREG>
LOKA_DEVINL void quant_row_body(const QuantParams& p, int64_t row, int lane) {
  const Tin* xr = reinterpret_cast<const Tin*>(p.x) + row * p.ldx;
  const int64_t cols = p.cols;
  const bool cached = cols <= 256 * NREG;
  Vec8<Tin> v[NREG];
  uint32_t am = 0;
  if (cached) {  // the whole row in registers: all loads in flight at once, one HBM read
#pragma unroll
    for (int i = 0; i < NREG; ++i) {
      const int64_t c = i * 256 + lane * 8;
      if (c + 8 <= cols) v[i].load(xr + c);
      else if (c < cols) v[i].load_partial(xr + c, (int)(cols - c));
      else v[i].zero();
    }
#pragma unroll
    for (int i = 0; i < NREG; ++i) am = max(am, v[i].amax_bits());
  } else {
    for (int64_t c0 = 0; c0 < cols; c0 += 256) {
      const int64_t c = c0 + lane * 8;
      Vec8<Tin> t;
      if (c + 8 <= cols) t.load(xr + c);
      else if (c < cols) t.load_partial(xr + c, (int)(cols - c));
      else t.zero();
      am = max(am, t.amax_bits());
    }
  }
  am = warp_max_u32(am);
  flag_nonfinite(am, p.status);
  float s, r;
  scales_from_amax<FMT, SF>(__uint_as_float(am), s, r);
  if (lane == 0) {
    if (p.scales) p.scales[row] = s;
    if (p.scales_t) p.scales_t[row] = s;
  }
  uint8_t* qr = p.q ? p.q + row * p.ldq : nullptr;
  auto emit = [&](int64_t c, const Vec8<Tin>& t) {
    const uint2 code = cast8<FMT>(t, r);
    const int n = (int)imin64(8, cols - c);
    if (qr) store8(qr + c, code, n);
    if (p.qt) {  // transposed copy: element (row, c+i) -> qt[(c+i) * ldqt + row]
      const uint8_t* b = reinterpret_cast<const uint8_t*>(&code);
      for (int i = 0; i < n; ++i) p.qt[(c + i) * p.ldqt + row] = b[i];
    }
  };
  if (cached) {
#pragma unroll
    for (int i = 0; i < NREG; ++i) {
      const int64_t c = i * 256 + lane * 8;
      if (c < cols) emit(c, v[i]);
    }
  } else {
    for (int64_t c0 = 0; c0 < cols; c0 += 256) {
      const int64_t c = c0 + lane * 8;
      if (c >= cols) continue;
      Vec8<Tin> t;
      if (c + 8 <= cols) t.load(xr + c);
      else t.load_partial(xr + c, (int)(cols - c));
      emit(c, t);
    }
  }
}

template <typename Tin, int FMT, int SF, int NREG>
__global__ void __launch_bounds__(256) quant_row_kernel(QuantParams p) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= p.rows) return;
  quant_row_body<Tin, FMT, SF, NREG>(p, row, lane);
}

// ----- ROW, streaming variant (no transposed copy, row fits NREG registers per lane): a
// persistent grid of warps walks rows w, w + #warps, ...; the NEXT row's loads are issued before
// the current row is reduced, cast and stored, so every warp keeps a row's worth of loads in
// flight continuously (the one-row-per-warp kernel above idles between load bursts).
template <typename Tin, int NREG>
LOKA_DEVINL void load_row(Vec8<Tin> (&v)[NREG], const Tin* xr, int64_t cols, int lane) {
#pragma unroll
  for (int i = 0; i < NREG; ++i) {
    const int64_t c = i * 256 + lane * 8;
    if (c + 8 <= cols) v[i].load(xr + c);
    else if (c < cols) v[i].load_partial(xr + c, (int)(cols - c));
    else v[i].zero();
  }
}
template <typename Tin, int FMT, int SF, int NREG>
LOKA_DEVINL void emit_row(const Vec8<Tin> (&v)[NREG], const QuantParams& p, int64_t row, int lane) {
  uint32_t am = 0;
#pragma unroll
  for (int i = 0; i < NREG; ++i) am = max(am, v[i].amax_bits());
  am = warp_max_u32(am);
  flag_nonfinite(am, p.status);
  float s, r;
  scales_from_amax<FMT, SF>(__uint_as_float(am), s, r);
  if (lane == 0) {
    if (p.scales) p.scales[row] = s;
    if (p.scales_t) p.scales_t[row] = s;
  }
  uint8_t* qr = p.q + row * p.ldq;
#pragma unroll
  for (int i = 0; i < NREG; ++i) {
    const int64_t c = i * 256 + lane * 8;
    if (c < p.cols) store8(qr + c, cast8<FMT>(v[i], r), (int)imin64(8, p.cols - c));
  }
}
template <typename Tin, int FMT, int SF, int NREG>
__global__ void __launch_bounds__(256, 1) quant_row_stream_kernel(QuantParams p) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * 8;
  int64_t row = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const Tin* x = reinterpret_cast<const Tin*>(p.x);
  Vec8<Tin> a[NREG];
  if (row < p.rows) load_row<Tin, NREG>(a, x + row * p.ldx, p.cols, lane);
  while (row < p.rows) {
    const int64_t nrow = row + nw;
    Vec8<Tin> b[NREG];
    if (nrow < p.rows) load_row<Tin, NREG>(b, x + nrow * p.ldx, p.cols, lane);
    emit_row<Tin, FMT, SF, NREG>(a, p, row, lane);
#pragma unroll
    for (int i = 0; i < NREG; ++i) a[i] = b[i];
    row = nrow;
  }
}

// ----- grouped ROW quantize: many tensors (e.g. an activation + every layer's weight) in one
// launch; warp w of the grid takes global row w, located in tensor g by a prefix sum of rows.
template <typename Tin, int FMT, int SF, int NREG>
__global__ void __launch_bounds__(256) quant_row_grouped_kernel(const __grid_constant__ QuantGroup grp) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int64_t grow = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (grow >= grp.row_start[grp.G]) return;
  int g = 0;
  while (grow >= grp.row_start[g + 1]) ++g;
  quant_row_body<Tin, FMT, SF, NREG>(grp.p[g], grow - grp.row_start[g], lane);
}

// ----- BLK_1x128: one warp per row, 16 lanes per 128-column block -------------------------
template <typename Tin, int FMT, int SF>
__global__ void __launch_bounds__(256) quant_1x128_kernel(QuantParams p) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= p.rows) return;
  const Tin* xr = reinterpret_cast<const Tin*>(p.x) + row * p.ldx;
  const int64_t cols = p.cols;
  const int64_t nblk = (cols + 127) / 128;
  constexpr int U = 4;  // 256-column steps whose loads are in flight together (x and q may alias: all
                        // loads of a group precede its stores, and the groups cover disjoint columns)
  for (int64_t g0 = 0; g0 < cols; g0 += 256 * U) {
    Vec8<Tin> t[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t c = g0 + 256 * u + lane * 8;
      if (c + 8 <= cols) t[u].load(xr + c);
      else if (c < cols) t[u].load_partial(xr + c, (int)(cols - c));
      else t[u].zero();
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t c0 = g0 + 256 * u;
      if (c0 >= cols) break;  // (uniform over the warp)
      const int64_t c = c0 + lane * 8;
      uint32_t am = t[u].amax_bits();
#pragma unroll
      for (int o = 8; o >= 1; o >>= 1) am = max(am, __shfl_xor_sync(0xFFFFFFFFu, am, o));
      flag_nonfinite(am, p.status);
      float s, r;
      scales_from_amax<FMT, SF>(__uint_as_float(am), s, r);
      const int64_t blk = c0 / 128 + (lane >> 4);
      if ((lane & 15) == 0 && blk < nblk) {
        if (p.scales) p.scales[row * nblk + blk] = s;
        if (p.scales_t) p.scales_t[blk * p.rows + row] = s;  // transposed frame: BLK_128x1 [nblk, rows]
      }
      if (c < cols) {
        uint2 code = cast8<FMT>(t[u], r);
        const int n = (int)imin64(8, cols - c);
        if (p.q) store8(p.q + row * p.ldq + c, code, n);
        if (p.qt) {
          const uint8_t* b = reinterpret_cast<const uint8_t*>(&code);
          for (int i = 0; i < n; ++i) p.qt[(c + i) * p.ldqt + row] = b[i];
        }
      }
    }
  }
}

// ----- BLK_128x128: one CTA (8 warps) per 128x128 block, block held in registers --------
template <typename Tin, int FMT, int SF>
__global__ void __launch_bounds__(256) quant_128x128_kernel(QuantParams p) {
  // two horizontally adjacent 128x128 blocks per CTA: all 16 loads per thread in flight before the
  // first reduction (one block's 8 left the SMs' memory pipes half empty: 3.6 TB/s)
  pdl_wait();
  __shared__ uint32_t red[2][8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t br = blockIdx.y;
  const int64_t nbc = (p.cols + 127) / 128, nbr = (p.rows + 127) / 128;
  Vec8<Tin> v[2][8];
  uint32_t am[2] = {0u, 0u};
#pragma unroll
  for (int b = 0; b < 2; ++b) {
    const int64_t col = (2 * (int64_t)blockIdx.x + b) * 128 + (lane & 15) * 8;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int64_t row = br * 128 + warp * 16 + i * 2 + (lane >> 4);
      const Tin* xr = reinterpret_cast<const Tin*>(p.x) + row * p.ldx;
      if (row < p.rows && col + 8 <= p.cols) v[b][i].load(xr + col);
      else if (row < p.rows && col < p.cols) v[b][i].load_partial(xr + col, (int)(p.cols - col));
      else v[b][i].zero();
    }
  }
#pragma unroll
  for (int b = 0; b < 2; ++b) {
#pragma unroll
    for (int i = 0; i < 8; ++i) am[b] = max(am[b], v[b][i].amax_bits());
    am[b] = warp_max_u32(am[b]);
    if (lane == 0) red[b][warp] = am[b];
  }
  __syncthreads();
#pragma unroll
  for (int b = 0; b < 2; ++b) {
    const int64_t bc = 2 * (int64_t)blockIdx.x + b;
    if (bc >= nbc) break;
    uint32_t a = red[b][0];
#pragma unroll
    for (int w = 1; w < 8; ++w) a = max(a, red[b][w]);
    if (threadIdx.x == 0) flag_nonfinite(a, p.status);
    float s, r;
    scales_from_amax<FMT, SF>(__uint_as_float(a), s, r);
    if (threadIdx.x == 0) {
      if (p.scales) p.scales[br * nbc + bc] = s;
      if (p.scales_t) p.scales_t[bc * nbr + br] = s;
    }
    const int64_t col = bc * 128 + (lane & 15) * 8;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int64_t row = br * 128 + warp * 16 + i * 2 + (lane >> 4);
      if (row >= p.rows || col >= p.cols) continue;
      uint2 code = cast8<FMT>(v[b][i], r);
      const int n = (int)imin64(8, p.cols - col);
      if (p.q) store8(p.q + row * p.ldq + col, code, n);
      if (p.qt) {
        const uint8_t* bb = reinterpret_cast<const uint8_t*>(&code);
        for (int k = 0; k < n; ++k) p.qt[(col + k) * p.ldqt + row] = bb[k];
      }
    }
  }
}

// ----- TENSOR: amax pass (atomicMax on bit patterns into a zeroed word) + cast pass -------
template <typename Tin>
__global__ void __launch_bounds__(256) amax_tensor_kernel(QuantParams p, uint32_t* amax_bits) {
  pdl_wait();
  __shared__ uint32_t red[8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nwarps = (int64_t)gridDim.x * 8;
  uint32_t am = 0;
  for (int64_t row = (int64_t)blockIdx.x * 8 + warp; row < p.rows; row += nwarps) {
    const Tin* xr = reinterpret_cast<const Tin*>(p.x) + row * p.ldx;
    for (int64_t c = lane * 8; c < p.cols; c += 256) {
      Vec8<Tin> t;
      if (c + 8 <= p.cols) t.load(xr + c);
      else t.load_partial(xr + c, (int)(p.cols - c));
      am = max(am, t.amax_bits());
    }
  }
  am = warp_max_u32(am);
  if (lane == 0) red[warp] = am;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 8; ++w) am = max(am, red[w]);
    am = max(am, red[0]);
    if (am) atomicMax(amax_bits, am);
    flag_nonfinite(am, p.status);
  }
}

// Dense (ld == cols) tensors: the tensor is one flat array of 16-byte vectors; every lane keeps 8
// streaming (evict-first) 16-B loads in flight before reducing them, persistent grid of 4 CTAs per SM.
template <typename Tin>
__global__ void __launch_bounds__(256) amax_flat_kernel(QuantParams p, uint32_t* amax_bits) {
  pdl_wait();
  __shared__ uint32_t red[8];
  constexpr int E = 16 / sizeof(Tin);  // elements per 16-B vector
  constexpr int U = 8;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t n = p.rows * p.cols;
  const int64_t nv = n / E;
  const uint4* xv = reinterpret_cast<const uint4*>(p.x);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  uint32_t am = 0;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < nv; i += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcs(xv + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      Vec8<Tin> t;
      if constexpr (sizeof(Tin) == 2) {
        t.w = v[u];
      } else {
        t.a = make_float4(__uint_as_float(v[u].x), __uint_as_float(v[u].y), __uint_as_float(v[u].z),
                          __uint_as_float(v[u].w));
        t.b = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      am = max(am, t.amax_bits());
    }
  }
  for (; i < nv; i += stride) {
    Vec8<Tin> t;
    const uint4 v = __ldcs(xv + i);
    if constexpr (sizeof(Tin) == 2) {
      t.w = v;
    } else {
      t.a = make_float4(__uint_as_float(v.x), __uint_as_float(v.y), __uint_as_float(v.z), __uint_as_float(v.w));
      t.b = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    am = max(am, t.amax_bits());
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {  // the n % E tail elements
    const Tin* xt = reinterpret_cast<const Tin*>(p.x) + nv * E;
    Vec8<Tin> t;
    t.load_partial(xt, (int)(n - nv * E));
    am = max(am, t.amax_bits());
  }
  am = warp_max_u32(am);
  if (lane == 0) red[warp] = am;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 8; ++w) am = max(am, red[w]);
    am = max(am, red[0]);
    if (am) atomicMax(amax_bits, am);
    flag_nonfinite(am, p.status);
  }
}

template <typename Tin, int FMT, int SF>
__global__ void __launch_bounds__(256) cast_tensor_kernel(QuantParams p, const float* amax_dev) {
  pdl_wait();
  const float amax = *amax_dev;
  float s, r;
  scales_from_amax<FMT, SF>(amax, s, r);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (p.scales) p.scales[0] = s;
    if (p.scales_t) p.scales_t[0] = s;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nwarps = (int64_t)gridDim.x * 8;
  constexpr int U = 4;  // loads in flight per lane before the first store (x and q may alias)
  for (int64_t row = (int64_t)blockIdx.x * 8 + warp; row < p.rows; row += nwarps) {
    const Tin* xr = reinterpret_cast<const Tin*>(p.x) + row * p.ldx;
    for (int64_t c0 = lane * 8; c0 < p.cols; c0 += 256 * U) {
      Vec8<Tin> t[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t c = c0 + 256 * u;
        const int n = (int)imin64(8, p.cols - c);
        if (n >= 8) t[u].load(xr + c);
        else if (n > 0) t[u].load_partial(xr + c, n);
        else t[u].zero();
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t c = c0 + 256 * u;
        if (c >= p.cols) break;
        const int n = (int)imin64(8, p.cols - c);
        uint2 code = cast8<FMT>(t[u], r);
        if (p.q) store8(p.q + row * p.ldq + c, code, n);
        if (p.qt) {
          const uint8_t* b = reinterpret_cast<const uint8_t*>(&code);
          for (int k = 0; k < n; ++k) p.qt[(c + k) * p.ldqt + row] = b[k];
        }
      }
    }
  }
}

// ----- host-side launch (programmatic dependent launch: prologue overlaps the previous kernel)
template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  note_launch();
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

// LOKA_QUANT_TMA=0 keeps the register-resident kernels (A/B measurement; the outputs are identical)
static bool quant_tma_use() {
  static const bool off = [] {
    const char* e = std::getenv("LOKA_QUANT_TMA");
    return e && e[0] == '0';
  }();
  return !off;
}

template <typename Tin, int FMT, int SF>
static cudaError_t launch_quant_t(const QuantParams& p, int gran, int phase, float* amax_dev, cudaStream_t st,
                                  int num_sms) {
  const dim3 blk(256);
  cudaError_t e = cudaSuccess;
  const bool tma = quant_tma_use() && quant_tma_eligible(p, sizeof(Tin) == 2, gran) && p.rows >= 64;
  if (tma && gran != LOKA_GRAN_TENSOR) return launch_quantize_tma(p, FMT, SF, gran, nullptr, num_sms, st);
  switch (gran) {
    case LOKA_GRAN_ROW: {
      const dim3 grd((unsigned)((p.rows + 7) / 8));
      constexpr int kBig = sizeof(Tin) == 2 ? 16 : 8;  // <= 64 data registers per lane
      const int64_t rows_per_pass = (int64_t)num_sms * 8;
      if (p.q && !p.qt && p.rows > 2 * rows_per_pass && p.cols <= 256 * kBig) {  // streaming variant
        const dim3 sg((unsigned)num_sms);
        if (p.cols <= 256 * 4) e = launch_pdl(quant_row_stream_kernel<Tin, FMT, SF, 4>, sg, blk, st, p);
        else e = launch_pdl(quant_row_stream_kernel<Tin, FMT, SF, kBig>, sg, blk, st, p);
      } else if (p.cols <= 256 * 4) {
        e = launch_pdl(quant_row_kernel<Tin, FMT, SF, 4>, grd, blk, st, p);
      } else {
        e = launch_pdl(quant_row_kernel<Tin, FMT, SF, kBig>, grd, blk, st, p);
      }
      break;
    }
    case LOKA_GRAN_BLK_1x128:
      e = launch_pdl(quant_1x128_kernel<Tin, FMT, SF>, dim3((unsigned)((p.rows + 7) / 8)), blk, st, p);
      break;
    case LOKA_GRAN_BLK_128x128:
      e = launch_pdl(quant_128x128_kernel<Tin, FMT, SF>,
                     dim3((unsigned)((p.cols + 255) / 256), (unsigned)((p.rows + 127) / 128)), blk, st, p);
      break;
    case LOKA_GRAN_TENSOR: {
      int64_t nb = (p.rows + 7) / 8;
      const int64_t cap = (int64_t)num_sms * 8;
      if (nb > cap) nb = cap;
      if (nb < 1) nb = 1;
      if (phase == LOKA_PHASE_FULL || phase == LOKA_PHASE_AMAX_ONLY) {
        e = cudaMemsetAsync(amax_dev, 0, sizeof(float), st);
        if (e != cudaSuccess) return e;
        const bool flat = p.ldx == p.cols && (reinterpret_cast<uintptr_t>(p.x) & 15) == 0;
        if (flat)
          e = launch_pdl(amax_flat_kernel<Tin>, dim3((unsigned)(num_sms * 4)), blk, st, p,
                         reinterpret_cast<uint32_t*>(amax_dev));
        else
          e = launch_pdl(amax_tensor_kernel<Tin>, dim3((unsigned)nb), blk, st, p, reinterpret_cast<uint32_t*>(amax_dev));
        if (e != cudaSuccess) return e;
      }
      if (phase == LOKA_PHASE_FULL || phase == LOKA_PHASE_CAST_WITH_AMAX) {
        if (tma) e = launch_quantize_tma(p, FMT, SF, gran, amax_dev, num_sms, st);
        else e = launch_pdl(cast_tensor_kernel<Tin, FMT, SF>, dim3((unsigned)nb), blk, st, p, (const float*)amax_dev);
      }
      if (phase == LOKA_PHASE_CAST_DELAYED) {  // cast with amax_dev[0], this tensor's amax -> amax_dev[1]
        uint32_t* next = reinterpret_cast<uint32_t*>(amax_dev + 1);
        e = cudaMemsetAsync(next, 0, sizeof(float), st);
        if (e != cudaSuccess) return e;
        if (tma) {  // one pass: the bulk-copy cast reduces max |x| of the rows it casts
          e = launch_quantize_tma(p, FMT, SF, gran, amax_dev, num_sms, st, next);
        } else {    // (same result in two passes)
          e = launch_pdl(amax_tensor_kernel<Tin>, dim3((unsigned)nb), blk, st, p, next);
          if (e != cudaSuccess) return e;
          e = launch_pdl(cast_tensor_kernel<Tin, FMT, SF>, dim3((unsigned)nb), blk, st, p, (const float*)amax_dev);
        }
      }
      break;
    }
    default:
      return cudaErrorNotSupported;
  }
  return e;
}

cudaError_t launch_quantize(const QuantParams& p, bool in_bf16, int fmt, int scale_fmt, int gran, int phase,
                            float* amax_dev, cudaStream_t st, int num_sms) {
#define LOKA_Q(T, F, S)                                 \
  if (fmt == F && scale_fmt == S)                       \
    return launch_quant_t<T, F, S>(p, gran, phase, amax_dev, st, num_sms);
  if (in_bf16) {
    LOKA_Q(__nv_bfloat16, LOKA_E4M3, LOKA_SCALE_F32)
    LOKA_Q(__nv_bfloat16, LOKA_E4M3, LOKA_SCALE_UE8M0)
    LOKA_Q(__nv_bfloat16, LOKA_E5M2, LOKA_SCALE_F32)
    LOKA_Q(__nv_bfloat16, LOKA_E5M2, LOKA_SCALE_UE8M0)
  } else {
    LOKA_Q(float, LOKA_E4M3, LOKA_SCALE_F32)
    LOKA_Q(float, LOKA_E4M3, LOKA_SCALE_UE8M0)
    LOKA_Q(float, LOKA_E5M2, LOKA_SCALE_F32)
    LOKA_Q(float, LOKA_E5M2, LOKA_SCALE_UE8M0)
  }
#undef LOKA_Q
  return cudaErrorNotSupported;
}

}  // namespace loka

namespace loka {

template <typename Tin, int FMT, int SF>
static cudaError_t launch_grouped_t(const QuantGroup& grp, int64_t max_cols, cudaStream_t st) {
  bool tma = quant_tma_use() && sizeof(Tin) == 2;
  for (int g = 0; g < grp.G && tma; ++g) tma = quant_tma_eligible(grp.p[g], true, LOKA_GRAN_ROW);
  if (tma) return launch_quantize_tma_group(grp, max_cols, FMT, SF, LOKA_GRAN_ROW, nullptr, 148, st);
  const int64_t rows = grp.row_start[grp.G];
  const dim3 grd((unsigned)((rows + 7) / 8)), blk(256);
  constexpr int kBig = sizeof(Tin) == 2 ? 16 : 8;
  if (max_cols <= 256 * 4) return launch_pdl(quant_row_grouped_kernel<Tin, FMT, SF, 4>, grd, blk, st, grp);
  return launch_pdl(quant_row_grouped_kernel<Tin, FMT, SF, kBig>, grd, blk, st, grp);
}

cudaError_t launch_quantize_grouped(const QuantGroup& grp, bool in_bf16, int fmt, int scale_fmt, int64_t max_cols,
                                    cudaStream_t st) {
#define LOKA_G(T, F, S) \
  if (fmt == F && scale_fmt == S) return launch_grouped_t<T, F, S>(grp, max_cols, st);
  if (in_bf16) {
    LOKA_G(__nv_bfloat16, LOKA_E4M3, LOKA_SCALE_F32)
    LOKA_G(__nv_bfloat16, LOKA_E4M3, LOKA_SCALE_UE8M0)
    LOKA_G(__nv_bfloat16, LOKA_E5M2, LOKA_SCALE_F32)
    LOKA_G(__nv_bfloat16, LOKA_E5M2, LOKA_SCALE_UE8M0)
  } else {
    LOKA_G(float, LOKA_E4M3, LOKA_SCALE_F32)
    LOKA_G(float, LOKA_E4M3, LOKA_SCALE_UE8M0)
    LOKA_G(float, LOKA_E5M2, LOKA_SCALE_F32)
    LOKA_G(float, LOKA_E5M2, LOKA_SCALE_UE8M0)
  }
#undef LOKA_G
  return cudaErrorNotSupported;
}

}  // namespace loka
