// nvfp4.cu — NEXT-4: NVFP4 quantize and the scale-atom packing for the
// NVFP4 block-scaled GEMM (linear.cu, kind::mxf4nvf4.block_scale.scale_vec::4X).
//
// Quantize (D35-D37; the paper names FP4 as future work): with the tensor
// amax A (computed by quantize.cu's amax pass, or the caller's all-reduced value),
//   s_t = fl32(A / 2688), r_t = fl32(2688 / A)                       (A = 0: s_t = r_t = 1)
//   per 1x16 block: sf = E4M3_satRNE(fl32(fl32(a_b * r_t) / 6)), d = decode(sf),
//                   codes = E2M1_satRNE(fl32(x * fl32(r_t / d)))     (d = 0: signed zeros)
// one thread per 16-element block: 32 B of bf16 in (two 16-B loads), 8 B of packed codes and one
// scale byte out (consecutive threads -> consecutive blocks: coalesced).  HBM-bound.
#include "common.cuh"
#include "launch.h"

namespace loka {

LOKA_DEVINL float e4m3_value(uint32_t c) {  // exact value of a non-negative E4M3 code (< 0x7F)
  const uint32_t e = (c >> 3) & 15u, m = c & 7u;
  return e == 0 ? (float)m * 0x1p-9f : __uint_as_float(((e + 120u) << 23) | (m << 20));
}

// 8 values -> 8 E2M1 codes packed in 32 bits (element 2j in the low nibble of byte j)
LOKA_DEVINL uint32_t cvt_e2m1x8(const float* v) {
  uint32_t w;
  asm("{\n .reg .b8 b0, b1, b2, b3;\n"
      " cvt.rn.satfinite.e2m1x2.f32 b0, %2, %1;\n"
      " cvt.rn.satfinite.e2m1x2.f32 b1, %4, %3;\n"
      " cvt.rn.satfinite.e2m1x2.f32 b2, %6, %5;\n"
      " cvt.rn.satfinite.e2m1x2.f32 b3, %8, %7;\n"
      " mov.b32 %0, {b0, b1, b2, b3};\n}"
      : "=r"(w)
      : "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]));
  return w;
}

template <typename Tin> LOKA_DEVINL void load16(const Tin* p, float* f);
template <> LOKA_DEVINL void load16<__nv_bfloat16>(const __nv_bfloat16* p, float* f) {
  const uint4 a = *reinterpret_cast<const uint4*>(p), b = *reinterpret_cast<const uint4*>(p + 8);
  const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    f[2 * i] = bf16lo_to_f32(w[i]);
    f[2 * i + 1] = bf16hi_to_f32(w[i]);
  }
}
template <> LOKA_DEVINL void load16<float>(const float* p, float* f) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float4 v = reinterpret_cast<const float4*>(p)[i];
    f[4 * i] = v.x; f[4 * i + 1] = v.y; f[4 * i + 2] = v.z; f[4 * i + 3] = v.w;
  }
}

template <typename Tin>
__global__ void __launch_bounds__(256) nvfp4_cast_kernel(const Nvfp4QParams p) {
  pdl_wait();
  const float A = *p.amax;
  float s_t = 1.f, r_t = 1.f;
  if (A > 0.f) {
    s_t = __fdiv_rn(A, 2688.f);
    r_t = fminf(__fdiv_rn(2688.f, A), 3.402823466e38f);  // D1b
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && p.s_tensor) *p.s_tensor = s_t;
  const int64_t nb = p.cols / 16, total = p.rows * nb;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = t / nb, b = t - row * nb;
    float f[16];
    load16<Tin>(reinterpret_cast<const Tin*>(p.x) + row * p.ldx + b * 16, f);
    float ab = 0.f;
#pragma unroll
    for (int i = 0; i < 16; ++i) ab = fmaxf(ab, fabsf(f[i]));
    const float sbv = __fdiv_rn(__fmul_rn(ab, r_t), 6.f);
    const uint32_t sf = cvt_fp8x2<LOKA_E4M3>(sbv, 0.f) & 0xFFu;  // (non-negative: UE4M3)
    const float d = e4m3_value(sf);
    if (d > 0.f) {
      const float rb = fminf(__fdiv_rn(r_t, d), 3.402823466e38f);  // D1b
#pragma unroll
      for (int i = 0; i < 16; ++i) f[i] = __fmul_rn(f[i], rb);
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) f[i] = copysignf(0.f, f[i]);
    }
    uint2 w;
    w.x = cvt_e2m1x8(f);
    w.y = cvt_e2m1x8(f + 8);
    *reinterpret_cast<uint2*>(p.q + row * p.ldq + b * 8) = w;
    p.sf[row * p.ld_sf + b] = (uint8_t)sf;
  }
}

// Block-scale codes [rows, ld] (one E4M3 byte per 16 columns) -> the MMA's 512-byte scale atoms,
// one per 128 rows x 64 columns: byte 16*(r%32) + 4*((r%128)/32) + kk holds row r's scale for
// the kk-th 16-column block of the atom's 64 columns ([row_blocks][k64 blocks][512], zero-padded).
__global__ void __launch_bounds__(256) nvfp4_sf_pack_kernel(const uint8_t* sf, int64_t ld, int64_t rows, int64_t nblk,
                                                            int64_t row_blocks, int64_t k64, uint8_t* out) {
  pdl_wait();
  const int64_t total = row_blocks * k64 * 512;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t atom = i >> 9;
    const int byte = (int)(i & 511);
    const int64_t rb = atom / k64, kb = atom - rb * k64;
    const int64_t r = rb * 128 + 32 * ((byte & 15) >> 2) + (byte >> 4);
    const int64_t blk = 4 * kb + (byte & 3);
    out[i] = (r < rows && blk < nblk) ? sf[r * ld + blk] : (uint8_t)0;
  }
}

template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl_n4(void (*kern)(KArgs...), dim3 grid, dim3 block, cudaStream_t st, Args... args) {
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

cudaError_t launch_nvfp4_cast(const Nvfp4QParams& p, bool in_bf16, int num_sms, cudaStream_t st) {
  const int64_t total = p.rows * (p.cols / 16);
  if (total == 0) return cudaSuccess;
  int64_t nb = (total + 255) / 256;
  if (nb > (int64_t)num_sms * 16) nb = (int64_t)num_sms * 16;
  if (in_bf16) return launch_pdl_n4(nvfp4_cast_kernel<__nv_bfloat16>, dim3((unsigned)nb), dim3(256), st, p);
  return launch_pdl_n4(nvfp4_cast_kernel<float>, dim3((unsigned)nb), dim3(256), st, p);
}

cudaError_t launch_nvfp4_sf_pack(const uint8_t* sf, int64_t ld, int64_t rows, int64_t nblk, int64_t row_blocks,
                                 int64_t k64, uint8_t* out, cudaStream_t st) {
  const int64_t total = row_blocks * k64 * 512;
  if (total == 0) return cudaSuccess;
  int64_t nb = (total + 255) / 256;
  if (nb > 148 * 16) nb = 148 * 16;
  return launch_pdl_n4(nvfp4_sf_pack_kernel, dim3((unsigned)nb), dim3(256), st, sf, ld, rows, nblk, row_blocks, k64,
                       out);
}

}  // namespace loka
