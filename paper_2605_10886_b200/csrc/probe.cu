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

// 8 consecutive elements (16 B of bf16 / 32 B of f32 when the row is 16-byte aligned)
LOKA_DEVINL void load8(const void* base, int bf16, int64_t off, float (&v)[8], int n, int vec) {
  if (n == 8 && vec) {
    if (bf16) {
      const uint4 w = __ldg(reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(base) + off));
      v[0] = bf16lo_to_f32(w.x); v[1] = bf16hi_to_f32(w.x); v[2] = bf16lo_to_f32(w.y); v[3] = bf16hi_to_f32(w.y);
      v[4] = bf16lo_to_f32(w.z); v[5] = bf16hi_to_f32(w.z); v[6] = bf16lo_to_f32(w.w); v[7] = bf16hi_to_f32(w.w);
    } else {
      const float4 a = __ldg(reinterpret_cast<const float4*>(reinterpret_cast<const float*>(base) + off));
      const float4 b = __ldg(reinterpret_cast<const float4*>(reinterpret_cast<const float*>(base) + off) + 1);
      v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    }
  } else {
    float t[4];
    load4(base, bf16, off, t, n < 4 ? n : 4, 0);
    v[0] = t[0]; v[1] = t[1]; v[2] = t[2]; v[3] = t[3];
    load4(base, bf16, off + 4, t, n > 4 ? n - 4 : 0, 0);
    v[4] = t[0]; v[5] = t[1]; v[6] = t[2]; v[7] = t[3];
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
  const bool fast = L.ref_vec && L.ref_bf16;
  for (int64_t row = (int64_t)blockIdx.x * 8 + warp; row < L.M; row += nw) {
    int64_t cstart = lane * 8;
    if (fast) {  // whole 256*U-column spans: U independent 16-B loads per lane in flight
      constexpr int U = 8;
      for (; (cstart - lane * 8) + 256 * U <= L.N; cstart += 256 * U) {  // warp-uniform span test
        const __nv_bfloat16* rp = reinterpret_cast<const __nv_bfloat16*>(L.ref) + row * L.ld_ref + cstart;
        uint4 rv4[U];
#pragma unroll
        for (int u = 0; u < U; ++u) rv4[u] = __ldg(reinterpret_cast<const uint4*>(rp + 256 * u));
        float s = 0.f;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t w[4] = {rv4[u].x, rv4[u].y, rv4[u].z, rv4[u].w};
#pragma unroll
          for (int i = 0; i < 4; ++i) s += fabsf(bf16lo_to_f32(w[i])) + fabsf(bf16hi_to_f32(w[i]));
        }
        acc += (double)s;
      }
    }
    for (int64_t c0 = cstart; c0 < L.N; c0 += 512) {  // two independent 16-B loads per lane in flight
      float v[8], u[8];
      load8(L.ref, L.ref_bf16, row * L.ld_ref + c0, v, (int)max((int64_t)0, imin64(8, L.N - c0)), L.ref_vec);
      load8(L.ref, L.ref_bf16, row * L.ld_ref + c0 + 256, u, (int)max((int64_t)0, imin64(8, L.N - c0 - 256)),
            L.ref_vec);
      float s = 0.f;
#pragma unroll
      for (int i = 0; i < 8; ++i) s += fabsf(v[i]) + fabsf(u[i]);
      acc += (double)s;
    }
  }
  const double t = block_sum(acc, red);
  if (threadIdx.x == 0) part1[(int64_t)blockIdx.y * nblk + blockIdx.x] = t;
}

__global__ void __launch_bounds__(256) probe_p2(const __grid_constant__ ProbeBatch b, const double* part1,
                                                double* part2, float* partmax, long long* partfl, int nblk,
                                                double floor_rel, const double* gsum) {
  __shared__ double red[8];
  __shared__ long long redl[8];
  __shared__ float redf[8];
  const ProbeLayer& L = b.layer[blockIdx.y];
  // f from the P1 partials: a fixed-shape parallel reduction (every block derives the same value)
  double sabs = 0.0;
  for (int i = threadIdx.x; i < nblk; i += blockDim.x) sabs += part1[(int64_t)blockIdx.y * nblk + i];
  sabs = block_sum(sabs, red);
  const int64_t count = L.M * L.N;
  double f = count > 0 ? floor_rel * (sabs / (double)count) : 0.0;
  // data-parallel form: the floor from the global sum |ref| and count (all-reduced over the ranks
  // that hold shards of this layer's pair), so every shard is measured against the same f
  if (gsum) f = gsum[2 * blockIdx.y + 1] > 0.0 ? floor_rel * (gsum[2 * blockIdx.y] / gsum[2 * blockIdx.y + 1]) : 0.0;
  const float f32 = (float)f;  // used only as the denominator
  // floored <=> |r| < f (FP64).  For an FP32 |r| that is |r| < t with t = f rounded UP to FP32
  // (no FP32 value lies in [f, t)), so the decision stays exact with an FP32 compare.
  const float ft = __double2float_ru(f);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t nw = (int64_t)nblk * 8;
  double acc = 0.0;
  float mx = 0.f;
  unsigned nfl32 = 0;
  for (int64_t row = (int64_t)blockIdx.x * 8 + warp; row < L.M; row += nw) {
    // fast path for whole 512-column spans of aligned rows: two independent 16-B loads of each
    // operand per lane in flight
    const bool fast = L.out_vec && L.ref_vec && L.out_bf16 && L.ref_bf16 && f32 > 0.f;
    int64_t cstart = lane * 8;
    if (fast) {
      constexpr int U = 8;  // 16-B loads of each operand per lane in flight
      for (; (cstart - lane * 8) + 256 * U <= L.N; cstart += 256 * U) {  // warp-uniform span test
        const __nv_bfloat16* op = reinterpret_cast<const __nv_bfloat16*>(L.out) + row * L.ld_out + cstart;
        const __nv_bfloat16* rp = reinterpret_cast<const __nv_bfloat16*>(L.ref) + row * L.ld_ref + cstart;
        uint4 ov4[U], rv4[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          ov4[u] = __ldg(reinterpret_cast<const uint4*>(op + 256 * u));
          rv4[u] = __ldg(reinterpret_cast<const uint4*>(rp + 256 * u));
        }
        uint32_t ow[4 * U], rw[4 * U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          ow[4 * u] = ov4[u].x; ow[4 * u + 1] = ov4[u].y; ow[4 * u + 2] = ov4[u].z; ow[4 * u + 3] = ov4[u].w;
          rw[4 * u] = rv4[u].x; rw[4 * u + 1] = rv4[u].y; rw[4 * u + 2] = rv4[u].z; rw[4 * u + 3] = rv4[u].w;
        }
        float part = 0.f;
#pragma unroll
        for (int i = 0; i < 8 * U; ++i) {
          const float ov = (i & 1) ? bf16hi_to_f32(ow[i >> 1]) : bf16lo_to_f32(ow[i >> 1]);
          const float rv = (i & 1) ? bf16hi_to_f32(rw[i >> 1]) : bf16lo_to_f32(rw[i >> 1]);
          const float ar = fabsf(rv);
          nfl32 += ar < ft ? 1u : 0u;
          // den = max(|r|, f32) equals the floored select exactly (the only FP32 value in
          // [f32, ft) is f32 itself); the fast division (<= 2 ulp) is far inside the 1e-5 bar
          const float rel = __fdividef(fabsf(__fsub_rn(ov, rv)), fmaxf(ar, f32));
          part += rel;
          mx = fmaxf(mx, rel);
        }
        acc += (double)part;
      }
    }
    for (int64_t c = cstart; c < L.N; c += 256) {
      const int n = (int)imin64(8, L.N - c);
      float o[8], r[8];
      load8(L.out, L.out_bf16, row * L.ld_out + c, o, n, L.out_vec);
      load8(L.ref, L.ref_bf16, row * L.ld_ref + c, r, n, L.ref_vec);
      float part = 0.f;
      if (n == 8 && f32 > 0.f) {
        // fast path: den = max(|r|, f32) equals the floored select exactly (the only FP32 value in
        // [f32, ft) is f32 itself), so no branches; ~10 instructions per element
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float ar = fabsf(r[i]);
          nfl32 += ar < ft ? 1u : 0u;
          const float rel = __fdividef(fabsf(__fsub_rn(o[i], r[i])), fmaxf(ar, f32));
          part += rel;
          mx = fmaxf(mx, rel);
        }
        acc += (double)part;
        continue;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (i < n) {
          const float ar = fabsf(r[i]);
          const bool floored = ar < ft;  // == (double)ar < f (D10)
          nfl32 += floored ? 1u : 0u;
          const float den = floored ? f32 : ar;
          const float d = fabsf(__fsub_rn(o[i], r[i]));
          // the fast division (<= 2 ulp, far inside the statistic's 1e-5 tolerance) is exact enough
          // only for a denominator in [2^-126, 2^126]; a floor f = 1e-6 mean|ref| can be subnormal or
          // the refs huge, so outside that range the IEEE division is taken
          float rel;
          if (den >= 1.17549435e-38f && den <= 8.5070592e37f) rel = __fdividef(d, den);
          else if (den > 0.f) rel = __fdiv_rn(d, den);
          else rel = d > 0.f ? INFINITY : 0.f;
          part += rel;
          mx = fmaxf(mx, rel);
        }
      }
      acc += (double)part;
    }
  }
  const double t = block_sum(acc, red);
  const long long tf = block_sum((long long)nfl32, redl);
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

// One 256-thread block per layer: strided per-thread sums in a fixed order, then the fixed shuffle
// tree of block_sum (deterministic; s1 is bit-identical to the sum P2 derived f from).  (A single
// thread walking nblk ~ 1200 partials serially took 130 us for one 32768 x 4096 layer.)
__global__ void __launch_bounds__(256) probe_p3(const __grid_constant__ ProbeBatch b, const double* part1,
                                                const double* part2, const float* partmax,
                                                const long long* partfl, int nblk, ProbeStatsDev* out) {
  __shared__ double red[8];
  __shared__ long long redl[8];
  __shared__ float redf[8];
  const int l = blockIdx.x;
  const ProbeLayer& L = b.layer[l];
  double s1 = 0.0, s2 = 0.0;
  float m = 0.f;
  long long nf = 0;
  for (int i = threadIdx.x; i < nblk; i += blockDim.x) {
    const int64_t k = (int64_t)l * nblk + i;
    s1 += part1[k];
    s2 += part2[k];
    m = fmaxf(m, partmax[k]);
    nf += partfl[k];
  }
  s1 = block_sum(s1, red);
  s2 = block_sum(s2, red);
  nf = block_sum(nf, redl);
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xFFFFFFFFu, m, o));
  if ((threadIdx.x & 31) == 0) redf[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x != 0) return;
  for (int i = 1; i < 8; ++i) m = fmaxf(m, redf[i]);
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
                         double* ws, int nblk, cudaStream_t st, const double* gsum) {
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
    probe_p2<<<dim3((unsigned)nblk, (unsigned)nl), 256, 0, st>>>(b, part1, part2, partmax, partfl, nblk, floor_rel,
                                                                 gsum ? gsum + 2 * l0 : nullptr);
    probe_p3<<<dim3((unsigned)nl), 256, 0, st>>>(b, part1, part2, partmax, partfl, nblk,
                                                reinterpret_cast<ProbeStatsDev*>(stats_dev) + l0);
    note_launch(3);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace loka
