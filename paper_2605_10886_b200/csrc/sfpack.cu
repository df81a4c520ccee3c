// sfpack.cu — UE8M0 scale-factor packing for the native block-scaled GEMM (a4, SURVEY §8(a)
// "UE8M0: kind::mxf8f6f4.block_scale with scales in TMEM").
//
// A blockwise recipe with UE8M0 scales ("blockwise"; D7: s = 2^e) can run
// on the tensor core's own block scaling instead of FP32 promotion: a 1x128 (or 128x128) scale is
// four identical 1x32 MX scales.  The MMA reads its scales from TMEM, copied there from shared
// memory by tcgen05.cp in 512-byte atoms: for 128 rows r and the four 32-wide K blocks kk of one
// 128-K group, byte 16*(r%32) + 4*(r/32) + kk holds the biased exponent of row r's scale.
// This kernel writes those atoms for a whole operand, [row_blocks][kblocks][512], so the GEMM's
// producer fetches one atom per operand per pipeline stage with a 1-D bulk copy.
//
// FP32 2^e (e >= -127) has biased exponent field e + 127 (2^-127 is the subnormal 0x00400000,
// field 0), which IS the UE8M0 encoding: the byte is (bits >> 23) & 0xFF, exact.  Rows past the
// operand's end get 127 (scale 1; their codes are TMA zero fill).
#include "common.cuh"
#include "launch.h"

namespace loka {

__global__ void __launch_bounds__(256) sf_pack_kernel(const SfPackParams p) {
  const int seg_total0 = p.seg[0].row_blocks * p.kblocks * 32;
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int sg = 0;
  if (t >= seg_total0) {
    t -= seg_total0;
    sg = 1;
    if (t >= (int64_t)p.seg[1].row_blocks * p.kblocks * 32) return;
  }
  const SfPackSeg& s = p.seg[sg];
  pdl_wait();
  const int i = (int)(t & 31);
  const int64_t rk = t >> 5;
  const int kb = (int)(rk % p.kblocks);
  const int64_t rb = rk / p.kblocks;
  uint32_t w[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int64_t r = rb * 128 + 32 * j + i;
    uint32_t e = 127u;
    if (s.k32) {  // MX 1x32: byte kk = the scale of K block 4 kb + kk (127 past the end)
      uint32_t b = 0;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const int64_t col = (int64_t)kb * 4 + kk;
        const uint32_t ek = (r < s.rows && col < s.ld) ? (__float_as_uint(s.scales[r * s.ld + col]) >> 23) & 0xFFu : 127u;
        b |= ek << (8 * kk);
      }
      w[j] = b;
      continue;
    }
    if (r < s.rows) e = (__float_as_uint(s.scales[(r / s.row_div) * s.ld + kb]) >> 23) & 0xFFu;
    w[j] = e * 0x01010101u;
  }
  reinterpret_cast<uint4*>(s.out)[t] = make_uint4(w[0], w[1], w[2], w[3]);
  pdl_launch_dependents();
}

cudaError_t launch_sf_pack(const SfPackParams& p, cudaStream_t st) {
  const int64_t total = (int64_t)(p.seg[0].row_blocks + p.seg[1].row_blocks) * p.kblocks * 32;
  if (total <= 0) return cudaSuccess;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)((total + 255) / 256), 1, 1);
  cfg.blockDim = dim3(256, 1, 1);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, sf_pack_kernel, p);
  note_launch();
  return e;
}

}  // namespace loka
