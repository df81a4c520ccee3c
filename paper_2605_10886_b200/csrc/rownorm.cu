// rownorm.cu — a5 for rows too wide to fuse profitably: LayerNorm / RMSNorm (+ gamma / beta, Hard
// Swish, FP8 output with row scales) over an FP32 GEMM output written by the CTA-pair engine.
//
// PAPER.md:464-468 (§III-B.2, Case 2): when a row spans several thread blocks, fusing the norm into
// the GEMM needs cross-block synchronisation "which negates most of the performance gains".  On
// sm_100a the fused form exists up to 4096 columns (16-CTA clusters, linear.cu), but for N > 2048
// it runs on single-CTA 128 x 256 tiles at ~half the CTA-pair engine's tensor throughput; measured
// on BASELINE configs[4] (M = 262144, N = K = 4096) the unfused pair-engine GEMM (FP32 out) + this
// pass is faster.  Same arithmetic as the fused epilogue: FP32 statistics (mean and
// M2 two-pass, biased variance), one-FFMA normalisation, h-swish, FP8 row amax over the final
// values, IEEE scales.
//
#include "common.cuh"
#include "launch.h"

namespace loka {

// One CTA (256 threads) per row, grid-stride over rows: each thread holds 8 * V consecutive
// columns (V = N / 2048, <= 2) in registers, block reductions through shared memory.  Small
// register footprint -> 8 CTAs per SM, i.e. many rows' loads in flight (HBM-bound pass).
template <int V>
__global__ void __launch_bounds__(256) rownorm_kernel(const RowNormParams p) {
  pdl_wait();
  __shared__ float red[8];
  __shared__ float bc;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const float n = (float)p.N;
  auto bsum = [&](float v) {  // fixed-shape block sum (every thread gets the same value)
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    float r = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) r += red[w];
    return r;
  };
  float amx_out = 0.f;  // NEXT-4 producer amax over the stored values of this thread's rows
  auto rowout = [&](int64_t row, float (&v)[8 * V], const bool (&ok)[V], float amax) {
      if (p.amax_out) {
#pragma unroll
        for (int u = 0; u < V; ++u)
          if (ok[u])
#pragma unroll
            for (int k = 0; k < 8; ++k)
              amx_out = fmaxf(amx_out, fabsf(p.out_dtype == LOKA_BF16 ? stored_bf16(v[8 * u + k]) : v[8 * u + k]));
      }
      const bool fp8 = p.out_dtype == LOKA_E4M3 || p.out_dtype == LOKA_E5M2;
      float r_out = 1.f;
      if (fp8) {
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xFFFFFFFFu, amax, o));
        __syncthreads();
        if (lane == 0) red[warp] = amax;
        __syncthreads();
        if (t == 0) {
          float m = red[0];
          for (int w = 1; w < 8; ++w) m = fmaxf(m, red[w]);
          if (__float_as_uint(m) >= 0x7F800000u && p.status) atomicOr(p.status, LOKA_DEVSTATUS_NONFINITE);
          float s_out, r;
          if (p.out_dtype == LOKA_E4M3) scales_from_amax<LOKA_E4M3, LOKA_SCALE_F32>(m, s_out, r);
          else scales_from_amax<LOKA_E5M2, LOKA_SCALE_F32>(m, s_out, r);
          if (p.y_scales) p.y_scales[row] = s_out;
          bc = r;
        }
        __syncthreads();
        r_out = bc;
      }
#pragma unroll
      for (int u = 0; u < V; ++u) {
        if (!ok[u]) continue;
        const int c = (u * 256 + t) * 8;
        const float* x = v + 8 * u;
        if (p.precast) {
          float* d = p.precast + row * p.ld_pre + c;
          *reinterpret_cast<float4*>(d) = make_float4(x[0], x[1], x[2], x[3]);
          *reinterpret_cast<float4*>(d + 4) = make_float4(x[4], x[5], x[6], x[7]);
        }
        if (p.out_dtype == LOKA_F32) {
          float* d = reinterpret_cast<float*>(p.y) + row * p.ldy + c;
          *reinterpret_cast<float4*>(d) = make_float4(x[0], x[1], x[2], x[3]);
          *reinterpret_cast<float4*>(d + 4) = make_float4(x[4], x[5], x[6], x[7]);
        } else if (p.out_dtype == LOKA_BF16) {
          uint32_t w[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            __nv_bfloat162 hh = __floats2bfloat162_rn(x[2 * k], x[2 * k + 1]);
            w[k] = *reinterpret_cast<uint32_t*>(&hh);
          }
          *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(p.y) + row * p.ldy + c) =
              make_uint4(w[0], w[1], w[2], w[3]);
        } else {
          float f[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) f[k] = __fmul_rn(x[k], r_out);
          const uint2 code = p.out_dtype == LOKA_E4M3
                                 ? make_uint2(cvt_fp8x4<LOKA_E4M3>(f[0], f[1], f[2], f[3]),
                                              cvt_fp8x4<LOKA_E4M3>(f[4], f[5], f[6], f[7]))
                                 : make_uint2(cvt_fp8x4<LOKA_E5M2>(f[0], f[1], f[2], f[3]),
                                              cvt_fp8x4<LOKA_E5M2>(f[4], f[5], f[6], f[7]));
          *reinterpret_cast<uint2*>(reinterpret_cast<uint8_t*>(p.y) + row * p.ldy + c) = code;
        }
      }
  };
  // the next row's loads are issued before this row's reductions (register double buffer): two
  // rows in flight per CTA keep HBM busy across the block barriers
  bool ok[V];
  float4 nx[2 * V];
  auto load_row = [&](int64_t row) {
    const float* xr = p.y32 + row * p.ld32;
#pragma unroll
    for (int u = 0; u < V; ++u) {
      const int c = (u * 256 + t) * 8;
      if (row < p.M && c < p.N) {
        nx[2 * u] = __ldg(reinterpret_cast<const float4*>(xr + c));
        nx[2 * u + 1] = __ldg(reinterpret_cast<const float4*>(xr + c) + 1);
      } else {
        nx[2 * u] = nx[2 * u + 1] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
  };
#pragma unroll
  for (int u = 0; u < V; ++u) ok[u] = (u * 256 + t) * 8 < p.N;
  load_row(blockIdx.x);
  for (int64_t row = blockIdx.x; row < p.M; row += gridDim.x) {
    float v[8 * V];
#pragma unroll
    for (int u = 0; u < V; ++u) {
      const float4 a = nx[2 * u], b = nx[2 * u + 1];
      v[8 * u] = a.x; v[8 * u + 1] = a.y; v[8 * u + 2] = a.z; v[8 * u + 3] = a.w;
      v[8 * u + 4] = b.x; v[8 * u + 5] = b.y; v[8 * u + 6] = b.z; v[8 * u + 7] = b.w;
    }
    load_row(row + gridDim.x);
    float rstd = 1.f, c0 = 0.f;
    if (p.bwd) {
      // NEXT-1 norm backward: g = dh * act'(xhat*gamma + beta) * gamma,
      // dz = rstd (g - mean(g) - xhat mean(g xhat)) (LayerNorm; RMS / BlockNorm without mean(g))
      float xv[8 * V];
#pragma unroll
      for (int u = 0; u < V; ++u) {
        const int c = (u * 256 + t) * 8;
        if (ok[u]) {
          const uint4 w = __ldg(reinterpret_cast<const uint4*>(p.xhat + row * p.ld_xhat + c));
          xv[8 * u] = bf16lo_to_f32(w.x); xv[8 * u + 1] = bf16hi_to_f32(w.x); xv[8 * u + 2] = bf16lo_to_f32(w.y);
          xv[8 * u + 3] = bf16hi_to_f32(w.y); xv[8 * u + 4] = bf16lo_to_f32(w.z); xv[8 * u + 5] = bf16hi_to_f32(w.z);
          xv[8 * u + 6] = bf16lo_to_f32(w.w); xv[8 * u + 7] = bf16hi_to_f32(w.w);
        } else {
#pragma unroll
          for (int k = 0; k < 8; ++k) xv[8 * u + k] = 0.f;
        }
      }
      float sg[V], sgx[V];
#pragma unroll
      for (int u = 0; u < V; ++u) {
        const int c = (u * 256 + t) * 8;
        sg[u] = sgx[u] = 0.f;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float gam = (ok[u] && p.gamma) ? __ldg(p.gamma + c + k) : 1.f;
          const float bet = (ok[u] && p.beta) ? __ldg(p.beta + c + k) : 0.f;
          float g = v[8 * u + k];
          if (p.act == LOKA_ACT_HARDSWISH) {
            const float yp = fmaf(xv[8 * u + k], gam, bet);
            g *= yp < -3.f ? 0.f : (yp <= 3.f ? fmaf(yp, 1.f / 3.f, 0.5f) : 1.f);
          }
          g = ok[u] ? g * gam : 0.f;
          v[8 * u + k] = g;
          sg[u] += g;
          sgx[u] = fmaf(g, xv[8 * u + k], sgx[u]);
        }
      }
      float amax = 0.f;
      if (p.norm == LOKA_NORM_BLOCK_RMS) {  // blocks of 256 columns = one warp's span per u
#pragma unroll
        for (int u = 0; u < V; ++u) {
          float s2 = sgx[u];
#pragma unroll
          for (int o = 16; o >= 1; o >>= 1) s2 += __shfl_xor_sync(0xFFFFFFFFu, s2, o);
          const int c = (u * 256 + t) * 8;
          const float rs = ok[u] ? p.rstd_in[row * (p.N / 256) + c / 256] : 0.f;
          const float mgx = s2 / 256.f;
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            v[8 * u + k] = rs * (v[8 * u + k] - xv[8 * u + k] * mgx);
            if (ok[u]) amax = fmaxf(amax, fabsf(v[8 * u + k]));
          }
        }
      } else {
        float a1 = 0.f, a2 = 0.f;
#pragma unroll
        for (int u = 0; u < V; ++u) a1 += sg[u], a2 += sgx[u];
        const float mg = p.norm == LOKA_NORM_LAYER ? __fdiv_rn(bsum(a1), n) : 0.f;
        const float mgx = __fdiv_rn(bsum(a2), n);
        const float rs = p.rstd_in[row];
#pragma unroll
        for (int u = 0; u < V; ++u)
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            v[8 * u + k] = rs * (v[8 * u + k] - mg - xv[8 * u + k] * mgx);
            if (ok[u]) amax = fmaxf(amax, fabsf(v[8 * u + k]));
          }
      }
      rowout(row, v, ok, amax);
      continue;
    }
    if (p.norm == LOKA_NORM_LAYER) {
      float s = 0.f;
#pragma unroll
      for (int j = 0; j < 8 * V; ++j) s += v[j];
      const float mean = __fdiv_rn(bsum(s), n);
      float m2 = 0.f;
#pragma unroll
      for (int u = 0; u < V; ++u)
        if (ok[u]) {
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const float d = v[8 * u + k] - mean;
            m2 = fmaf(d, d, m2);
          }
        }
      rstd = __fdiv_rn(1.f, __fsqrt_rn(__fadd_rn(__fdiv_rn(bsum(m2), n), p.eps)));
      c0 = -__fmul_rn(mean, rstd);
    } else if (p.norm == LOKA_NORM_RMS) {
      float ss = 0.f;
#pragma unroll
      for (int j = 0; j < 8 * V; ++j) ss = fmaf(v[j], v[j], ss);
      rstd = __fdiv_rn(1.f, __fsqrt_rn(__fadd_rn(__fdiv_rn(bsum(ss), n), p.eps)));
    }
    float amax = 0.f;
#pragma unroll
    for (int u = 0; u < V; ++u) {
      const int c = (u * 256 + t) * 8;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        float x = p.norm == LOKA_NORM_NONE ? v[8 * u + k] : fmaf(v[8 * u + k], rstd, c0);
        if (ok[u] && (p.gamma || p.beta)) x = fmaf(x, p.gamma ? __ldg(p.gamma + c + k) : 1.f, p.beta ? __ldg(p.beta + c + k) : 0.f);
        if (p.act == LOKA_ACT_HARDSWISH) x = __fdiv_rn(__fmul_rn(x, fminf(fmaxf(x + 3.f, 0.f), 6.f)), 6.f);
        v[8 * u + k] = x;
        if (ok[u]) amax = fmaxf(amax, fabsf(x));
      }
    }
    rowout(row, v, ok, amax);
  }
  if (p.amax_out) warp_amax_to(p.amax_out, amx_out);
}

cudaError_t launch_rownorm(const RowNormParams& p, int num_sms, cudaStream_t st) {
  int64_t nb = p.M;
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
  if (p.N <= 2048) return cudaLaunchKernelEx(&cfg, rownorm_kernel<1>, p);
  if (p.N <= 4096) return cudaLaunchKernelEx(&cfg, rownorm_kernel<2>, p);
  return cudaErrorInvalidValue;
}

}  // namespace loka
