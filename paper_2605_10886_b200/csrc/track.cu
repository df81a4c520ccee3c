// track.cu — NEXT-2: LoKA Probe's online input-distribution tracker, the batched
// Welford (Chan) merge of PAPER.md:282-305 (§III LoKA Probe, "Optimized Input Distribution Modeling"):
//   n_new = n_old + B, delta = mu_b - mu_old, mu_new = mu_old + (B / n_new) delta,
//   Sigma_new = Sigma_old + S_b + (n_old B / n_new) delta delta^T,  S_b = (X - 1 mu_b^T)^T (X - 1 mu_b^T)
// with the running summaries in FP32 (the paper: "accumulates Sigma in higher precision (e.g., FP32)").
//
// B200 mapping: S_b is a K x K x B dense contraction -> the CTA-pair tensor-core engine on BF16
// operands (gemm2.cu, kind::f16, FP32 accumulation in TMEM).  Around it three HBM-bound passes:
//   1. column sums of X in fixed row chunks (deterministic), then mu_b, delta, the mean update;
//   2. the centred transpose Xc^T [K, B] in bf16 (the GEMM's K-major operand; centring before the
//      product avoids the cancellation of X^T X - B mu mu^T when |mu| >> sigma);
//   3. the merge Sigma += S_b + c delta delta^T (element-wise over K x K).
#include "common.cuh"
#include "launch.h"

namespace loka {

// 1a. partial column sums: block (column block of 256, row chunk)
__global__ void __launch_bounds__(256) track_colsum_kernel(const TrackParams p) {
  pdl_wait();
  const int64_t k = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (k >= p.K) return;
  const int64_t rows_per = (p.B + p.nchunk - 1) / p.nchunk;
  const int64_t r0 = (int64_t)blockIdx.y * rows_per, r1 = min(p.B, r0 + rows_per);
  float s = 0.f;
  for (int64_t b = r0; b < r1; ++b) s += __bfloat162float(p.x[b * p.ldx + k]);
  p.colpart[(int64_t)blockIdx.y * p.K + k] = s;
}

// 1b. mu_b (into colpart row 0), delta, the tracked mean's update; one[0] = 1
__global__ void __launch_bounds__(256) track_mean_kernel(const TrackParams p) {
  const int64_t k = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (blockIdx.x == 0 && threadIdx.x == 0) p.one[0] = 1.f;
  if (k >= p.K) return;
  float s = 0.f;
  for (int c = 0; c < p.nchunk; ++c) s += p.colpart[(int64_t)c * p.K + k];  // fixed order
  const float mub = s / (float)p.B;
  const float d = mub - p.mean[k];
  const double n_new = (double)p.n_old + (double)p.B;
  p.mean[k] = p.mean[k] + (float)((double)p.B / n_new) * d;
  p.delta[k] = d;
  p.colpart[k] = mub;
}

// 2. Xc^T [K, B] = (X - mu_b)^T in bf16: 64 x 64 tiles through smem (coalesced on both sides)
__global__ void __launch_bounds__(256) track_center_t_kernel(const TrackParams p) {
  __shared__ float tile[64][65];
  const int64_t b0 = (int64_t)blockIdx.y * 64, k0 = (int64_t)blockIdx.x * 64;
  const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;  // 64 x 4
  const int64_t k = k0 + tx;
  const float mu = k < p.K ? p.colpart[k] : 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int64_t b = b0 + ty + 4 * i;
    tile[ty + 4 * i][tx] = (b < p.B && k < p.K) ? __bfloat162float(p.x[b * p.ldx + k]) - mu : 0.f;
  }
  __syncthreads();
  const int64_t bb = b0 + tx;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int64_t kk = k0 + ty + 4 * i;
    if (kk < p.K && bb < p.B) p.xct[kk * p.ldxct + bb] = __float2bfloat16_rn(tile[tx][ty + 4 * i]);
  }
}

// 3. Sigma += S_b + c delta delta^T, c = n_old B / n_new
__global__ void __launch_bounds__(256) track_merge_kernel(const TrackParams p) {
  pdl_wait();
  const double n_new = (double)p.n_old + (double)p.B;
  const float c = (float)((double)p.n_old * (double)p.B / n_new);
  const int64_t total = p.K * p.K;
  for (int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x; i < total; i += (int64_t)gridDim.x * 256) {
    const int64_t r = i / p.K, col = i - r * p.K;
    p.scatter[i] = p.scatter[i] + p.sb[i] + c * p.delta[r] * p.delta[col];
  }
}

cudaError_t launch_track_prep(const TrackParams& p, cudaStream_t st) {
  const unsigned kb = (unsigned)((p.K + 255) / 256);
  track_colsum_kernel<<<dim3(kb, (unsigned)p.nchunk), 256, 0, st>>>(p);
  track_mean_kernel<<<kb, 256, 0, st>>>(p);
  track_center_t_kernel<<<dim3((unsigned)((p.K + 63) / 64), (unsigned)((p.B + 63) / 64)), 256, 0, st>>>(p);
  note_launch(3);
  return cudaGetLastError();
}

cudaError_t launch_track_merge(const TrackParams& p, cudaStream_t st) {
  int64_t nb = (p.K * p.K + 255) / 256;
  if (nb > 148 * 8) nb = 148 * 8;
  track_merge_kernel<<<(unsigned)nb, 256, 0, st>>>(p);
  note_launch(1);
  return cudaGetLastError();
}

// the unbiased covariance Sigma / (n - 1) of the tracked statistics, K x K
__global__ void __launch_bounds__(256) track_cov_kernel(const float* scatter, float* out, int64_t nel, float inv) {
  pdl_wait();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nel; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = scatter[i] * inv;
}
cudaError_t launch_track_cov(const float* scatter, float* out, int64_t K, int64_t n, cudaStream_t st) {
  const int64_t nel = K * K;
  const float inv = (float)(1.0 / (double)(n - 1));  // one FP32 rounding of 1/(n-1), then one multiply
  int64_t nb = (nel + 255) / 256;
  if (nb > 148 * 16) nb = 148 * 16;
  note_launch();
  track_cov_kernel<<<dim3((unsigned)nb), 256, 0, st>>>(scatter, out, nel, inv);
  return cudaGetLastError();
}

}  // namespace loka
