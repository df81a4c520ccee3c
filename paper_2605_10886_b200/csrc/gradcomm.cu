// gradcomm.cu — NEXT-4: the reduction side of quantized data-parallel gradient
// communication (D39, oracle/gradcomm.py).  Every rank quantizes its gradient rowwise
// (loka_quantize); the owner of a row shard reduces the P ranks' codes of its rows:
//     out[i, j] = sum_{p = 0..P-1} decode(q_p[i, j]) * s_p[i]      (FP32, fmaf in rank order)
// The P code / scale pointers may be peer memory (CUDA IPC over NVLink / NVSwitch): the kernel then
// IS the collective's data movement — each rank pulls 1 byte per element from every peer straight
// into the reduction, instead of receiving FP32 partial sums (4 bytes) through NCCL.
// One thread per 16 consecutive elements of a row: one 16-B load per rank, 16 FP32 out.
#include "common.cuh"
#include "launch.h"

namespace loka {

template <int FMT>
LOKA_DEVINL void decode16(uint4 v, float* f) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint16_t pair = (uint16_t)(w[i] >> (16 * h));
      uint32_t hh;
      if constexpr (FMT == LOKA_E4M3)
        asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(hh) : "h"(pair));
      else
        asm("cvt.rn.f16x2.e5m2x2 %0, %1;" : "=r"(hh) : "h"(pair));
      const float2 t = __half22float2(*reinterpret_cast<__half2*>(&hh));  // exact
      f[4 * i + 2 * h] = t.x;
      f[4 * i + 2 * h + 1] = t.y;
    }
  }
}

template <int FMT>
__global__ void __launch_bounds__(256) dequant_reduce_kernel(const DeqReduceParams p) {
  pdl_wait();
  const int64_t n16 = p.cols / 16, total = p.rows * n16;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = t / n16, c = (t - row * n16) * 16;
    float acc[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = 0.f;
    for (int r = 0; r < p.P; ++r) {
      const uint4 v = *reinterpret_cast<const uint4*>(p.codes[r] + row * p.ld + c);
      const float s = p.scales[r][row];
      float f[16];
      decode16<FMT>(v, f);
#pragma unroll
      for (int i = 0; i < 16; ++i) acc[i] = fmaf(f[i], s, acc[i]);
    }
    float4* o = reinterpret_cast<float4*>(p.out + row * p.ld_out + c);
#pragma unroll
    for (int i = 0; i < 4; ++i) o[i] = make_float4(acc[4 * i], acc[4 * i + 1], acc[4 * i + 2], acc[4 * i + 3]);
  }
}

cudaError_t launch_dequant_reduce(const DeqReduceParams& p, int num_sms, cudaStream_t st) {
  const int64_t total = p.rows * (p.cols / 16);
  if (total == 0) return cudaSuccess;
  int64_t nb = (total + 255) / 256;
  if (nb > (int64_t)num_sms * 8) nb = (int64_t)num_sms * 8;
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
  if (p.fmt == LOKA_E5M2) return cudaLaunchKernelEx(&cfg, dequant_reduce_kernel<LOKA_E5M2>, p);
  return cudaLaunchKernelEx(&cfg, dequant_reduce_kernel<LOKA_E4M3>, p);
}

}  // namespace loka
