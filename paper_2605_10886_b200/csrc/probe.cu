// probe.cu — a7: LoKA Probe per-layer error statistic (PAPER.md:192 MERE; D8-D10).
//
//   mere = (1/(M N)) sum |out - ref| / max(|ref|, f),   f = floor_rel * mean |ref|
//   plus max relative error, sum |ref|, count, n_floored (|ref| < f).
//
// HBM-bound reduction over L layers in one launch sequence:
//   P1  grid (nblk, L): per-block FP64 partial sums of |ref|
//   P2  grid (nblk, L): every block re-derives f_l from the P1 partials (same order -> same
//       value in every block), then per element the FP32 relative error, FP64 block sums,
//       FP32 max, int64 floored count
//   P3  grid (L): fixed-order reduction of the partials -> loka_probe_stats[l]
// Deterministic: no floating-point atomics; all reductions are in a fixed order.
#include "common.cuh"
#include "launch.h"

namespace loka {

constexpr int kMaxProbeLayers = 64;
struct ProbeBatch {
  ProbeLayer layer[kMaxProbeLayers];
};

struct ProbeStatsDev {  // == loka_probe_stats
  double mere, max_rel, sum_abs_ref;
  long long count, n_floored;
};

LOKA_DEVINL void load4(const void* base, int bf16, int64_t off, float (&v)[4], int n, int vec) {
  if (n == 4 && vec) {
    if (bf16) {
      const uint2 w = *reinterpret_cast<const uint2*>(reinterpret_cast<const __nv_bfloat16*>(base) + off);
      v[0] = bf16lo_to_f32(w.x); v[1] = bf16hi_to_f32(w.x);
      v[2] = bf16lo_to_f32(w.y); v[3] = bf16hi_to_f32(w.y);
    } else {
      const float4 w = *reinterpret_cast<const float4*>(reinterpret_cast<const float*>(base) + off);
      v[0] = w.x; v[1] = w.y; v[2] = w.z; v[3] = w.w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (i < n) v[i] = bf16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(base)[off + i])
                             : reinterpret_cast<const float*>(base)[off + i];
      else v[i] = 0.f;
    }
  }
}

template <typename T>
LOKA_DEVINL T block_sum(T v, T* red) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
  const int w = threadIdx.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[w] = v;
  __syncthreads();
  T t = 0;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];
  return t;
}

__global__ void __launch_bounds__(256) probe_p1(const __grid_constant__ ProbeBatch b, double* part1, int nblk) {
  __shared__ double red[8];
  const ProbeLayer& L = b.layer[blockIdx.y];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nw = (int64_t)nblk * 8;
  double acc = 0.0;
  for (int64_t row = (int64_t)blockIdx.x * 8 + warp; row < L.M; row += nw) {
    for (int64_t c = lane * 4; c < L.N; c += 128) {
      float v[4];
      load4(L.ref, L.ref_bf16, row * L.ld_ref + c, v, (int)imin64(4, L.N - c), L.ref_vec);
      acc += (double)(fabsf(v[0]) + fabsf(v[1])) + (double)(fabsf(v[2]) + fabsf(v[3]));
    }
  }
  const double t = block_sum(acc, red);
  if (threadIdx.x == 0) part1[(int64_t)blockIdx.y * nblk + blockIdx.x] = t;
}

__global__ void __launch_bounds__(256) probe_p2(const __grid_constant__ ProbeBatch b, const double* part1,
                                                double* part2, float* partmax, long long* partfl, int nblk,
                                                double floor_rel) {
  __shared__ double red[8];
  __shared__ long long redl[8];
  __shared__ float redf[8];
  const ProbeLayer& L = b.layer[blockIdx.y];
  double sabs = 0.0;
  for (int i = 0; i < nblk; ++i) sabs += part1[(int64_t)blockIdx.y * nblk + i];
  const int64_t count = L.M * L.N;
  const double f = count > 0 ? floor_rel * (sabs / (double)count) : 0.0;
  const float f32 = (float)f;  // used only as the denominator; the floored decision is in FP64
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nw = (int64_t)nblk * 8;
  double acc = 0.0;
  float mx = 0.f;
  long long nfl = 0;
  for (int64_t row = (int64_t)blockIdx.x * 8 + warp; row < L.M; row += nw) {
    for (int64_t c = lane * 4; c < L.N; c += 128) {
      const int n = (int)imin64(4, L.N - c);
      float o[4], r[4];
      load4(L.out, L.out_bf16, row * L.ld_out + c, o, n, L.out_vec);
      load4(L.ref, L.ref_bf16, row * L.ld_ref + c, r, n, L.ref_vec);
      float part = 0.f;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (i < n) {
          const float ar = fabsf(r[i]);
          const bool floored = (double)ar < f;
          nfl += floored ? 1 : 0;
          const float den = floored ? f32 : ar;
          const float d = fabsf(__fsub_rn(o[i], r[i]));
          float rel;
          if (den > 0.f) rel = __fdiv_rn(d, den);
          else rel = d > 0.f ? INFINITY : 0.f;
          part += rel;
          mx = fmaxf(mx, rel);
        }
      }
      acc += (double)part;
    }
  }
  const double t = block_sum(acc, red);
  const long long tf = block_sum(nfl, redl);
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
  __syncthreads();
  if (lane == 0) redf[warp] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    float m = redf[0];
    for (int i = 1; i < 8; ++i) m = fmaxf(m, redf[i]);
    const int64_t k = (int64_t)blockIdx.y * nblk + blockIdx.x;
    part2[k] = t;
    partmax[k] = m;
    partfl[k] = tf;
  }
}

__global__ void probe_p3(const __grid_constant__ ProbeBatch b, const double* part1, const double* part2,
                         const float* partmax, const long long* partfl, int nblk, ProbeStatsDev* out) {
  if (threadIdx.x != 0) return;
  const int l = blockIdx.x;
  const ProbeLayer& L = b.layer[l];
  double s1 = 0.0, s2 = 0.0;
  float m = 0.f;
  long long nf = 0;
  for (int i = 0; i < nblk; ++i) {
    const int64_t k = (int64_t)l * nblk + i;
    s1 += part1[k];
    s2 += part2[k];
    m = fmaxf(m, partmax[k]);
    nf += partfl[k];
  }
  const long long count = (long long)(L.M * L.N);
  ProbeStatsDev st;
  st.mere = count > 0 ? s2 / (double)count : 0.0;
  st.max_rel = (double)m;
  st.sum_abs_ref = s1;
  st.count = count;
  st.n_floored = nf;
  out[l] = st;
}

cudaError_t launch_probe(const ProbeLayer* layers, int L, int64_t /*max_elems*/, double floor_rel, void* stats_dev,
                         double* ws, int nblk, cudaStream_t st) {
  // ws layout per batch of <= 64 layers: part1 [64*nblk] f64 | part2 [64*nblk] f64 | partfl [64*nblk] i64
  //                                      | partmax [64*nblk] f32
  for (int l0 = 0; l0 < L; l0 += kMaxProbeLayers) {
    const int nl = L - l0 < kMaxProbeLayers ? L - l0 : kMaxProbeLayers;
    ProbeBatch b;
    for (int i = 0; i < nl; ++i) b.layer[i] = layers[l0 + i];
    const int64_t n = (int64_t)kMaxProbeLayers * nblk;
    double* part1 = ws;
    double* part2 = ws + n;
    long long* partfl = reinterpret_cast<long long*>(ws + 2 * n);
    float* partmax = reinterpret_cast<float*>(ws + 3 * n);
    probe_p1<<<dim3((unsigned)nblk, (unsigned)nl), 256, 0, st>>>(b, part1, nblk);
    probe_p2<<<dim3((unsigned)nblk, (unsigned)nl), 256, 0, st>>>(b, part1, part2, partmax, partfl, nblk, floor_rel);
    probe_p3<<<dim3((unsigned)nl), 32, 0, st>>>(b, part1, part2, partmax, partfl, nblk,
                                                reinterpret_cast<ProbeStatsDev*>(stats_dev) + l0);
    note_launch(3);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace loka
