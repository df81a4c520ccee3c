// linalg.cu — NEXT-3: LoKA Probe's matrix-normal weight tracker and the
// learned-distribution sampling, as FP32 device kernels.
//
//   * Cholesky of a regularised covariance: blocked right-looking,
//     64-column panels: potf2 on the diagonal block (one CTA, in shared memory), the panel below
//     by a row-parallel triangular solve (one thread per row, the 64x64 factor in shared memory),
//     the trailing update A22 -= L21 L21^T on the lower tiles only (SIMT FP32 GEMM below);
//   * triangular solves L X = B in place (the "linear solves with Cholesky factors" that replace
//     the inverses): 64-row panels of B by a column-parallel substitution, then a GEMM
//     update of the rows below;
//   * the Gram products U' = (1/N) W~ W~^T, V' = (1/M) W^^T W^, the EMA + symmetrisation + eps I,
//     and the trace renormalisation — traces accumulated in FP64 on the device,
//     so one tracker update never synchronises with the host;
//   * Philox4x64-10 normals (Box-Muller on 24-bit uniforms, D31) and the sampling GEMMs
//     T' = 1 mu^T + Z L_Sigma^T, W' = M + L_U (Z L_V^T) with the triangular factor's zero half
//     skipped.
//
// Why FP32 SIMT and not the tensor cores: the tracker is off the hot path (it runs every 100
// iterations) and keeps its statistics in FP32 or wider; tcgen05
// offers TF32 at best for FP32 operands, whose 10-bit mantissa would enter the Cholesky solves.
#include "common.cuh"
#include "launch.h"

namespace loka {

LOKA_DEVINL float to_f32(float x) { return x; }
LOKA_DEVINL float to_f32(__nv_bfloat16 x) { return __bfloat162float(x); }

// ---------------------------------------------------------------------------------------------
// FP32 GEMM: C[m][n] = alpha sum_k A(m,k) B(k,n) + beta Cin[m][n] + bias[n]
//   AT = false: A(m,k) = A[m lda + k]   AT = true: A(m,k) = A[k lda + m]
//   BT = false: B(k,n) = B[k ldb + n]   BT = true: B(k,n) = B[n ldb + k]
// 128 x 128 tiles, 256 threads, 8 x 8 outputs per thread, K steps of 8 double-buffered in smem.
// tri_a / tri_b: A(m,k) = 0 for k > m / B(k,n) = 0 for k > n (the K loop stops at the tile's
// diagonal); lower_only: tiles entirely above the diagonal are skipped.
// ---------------------------------------------------------------------------------------------
constexpr int kGBM = 128, kGBN = 128, kGBK = 8;

template <bool AT, bool BT>
__global__ void __launch_bounds__(256) gemm_f32_kernel(const GemmF32Params p) {
  __shared__ __align__(16) float As[2][kGBK][kGBM + 4];
  __shared__ __align__(16) float Bs[2][kGBK][kGBN + 4];
  const int64_t m0 = (int64_t)blockIdx.y * kGBM, n0 = (int64_t)blockIdx.x * kGBN;
  if (p.lower_only && n0 > m0 + kGBM - 1) return;
  int64_t kend = p.K;
  if (p.tri_a) kend = min(kend, m0 + kGBM);
  if (p.tri_b) kend = min(kend, n0 + kGBN);
  const int t = threadIdx.x;
  const int tx = t & 15, ty = t >> 4;
  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
  float ra[4], rb[4];
  auto a_idx = [&](int i, int& mm, int& kk) {
    const int idx = t + 256 * i;
    if (AT) { kk = idx >> 7; mm = idx & 127; } else { mm = idx >> 3; kk = idx & 7; }
  };
  auto b_idx = [&](int i, int& nn, int& kk) {
    const int idx = t + 256 * i;
    if (BT) { nn = idx >> 3; kk = idx & 7; } else { kk = idx >> 7; nn = idx & 127; }
  };
  auto load = [&](int64_t k0) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      int mm, kk;
      a_idx(i, mm, kk);
      const int64_t gm = m0 + mm, gk = k0 + kk;
      ra[i] = (gm < p.M && gk < kend) ? (AT ? p.A[gk * p.lda + gm] : p.A[gm * p.lda + gk]) : 0.f;
      int nn, kb;
      b_idx(i, nn, kb);
      const int64_t gn = n0 + nn, gkb = k0 + kb;
      rb[i] = (gn < p.N && gkb < kend) ? (BT ? p.B[gn * p.ldb + gkb] : p.B[gkb * p.ldb + gn]) : 0.f;
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      int mm, kk;
      a_idx(i, mm, kk);
      As[buf][kk][mm] = ra[i];
      int nn, kb;
      b_idx(i, nn, kb);
      Bs[buf][kb][nn] = rb[i];
    }
  };
  const int64_t nk = kend > 0 ? (kend + kGBK - 1) / kGBK : 0;
  if (nk > 0) {
    load(0);
    store(0);
  }
  __syncthreads();
  for (int64_t kt = 0; kt < nk; ++kt) {
    const int buf = (int)(kt & 1);
    if (kt + 1 < nk) load((kt + 1) * kGBK);
#pragma unroll
    for (int k = 0; k < kGBK; ++k) {
      const float4 a0 = *reinterpret_cast<const float4*>(&As[buf][k][ty * 4]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[buf][k][64 + ty * 4]);
      const float4 b0 = *reinterpret_cast<const float4*>(&Bs[buf][k][tx * 4]);
      const float4 b1 = *reinterpret_cast<const float4*>(&Bs[buf][k][64 + tx * 4]);
      const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    if (kt + 1 < nk) store(buf ^ 1);
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t r = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + i - 4);
    if (r >= p.M) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int64_t c = n0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + j - 4);
      if (c >= p.N) continue;
      float v = p.alpha * acc[i][j];
      if (p.beta != 0.f) v = fmaf(p.beta, p.Cin[r * p.ldcin + c], v);
      if (p.bias) v += p.bias[c];
      if (p.c_bf16) reinterpret_cast<__nv_bfloat16*>(p.C)[r * p.ldc + c] = __float2bfloat16_rn(v);
      else reinterpret_cast<float*>(p.C)[r * p.ldc + c] = v;
    }
  }
}

cudaError_t launch_gemm_f32(const GemmF32Params& p, bool at, bool bt, cudaStream_t st) {
  if (p.M <= 0 || p.N <= 0) return cudaSuccess;
  const dim3 grid((unsigned)((p.N + kGBN - 1) / kGBN), (unsigned)((p.M + kGBM - 1) / kGBM));
  if (!at && !bt) gemm_f32_kernel<false, false><<<grid, 256, 0, st>>>(p);
  else if (!at && bt) gemm_f32_kernel<false, true><<<grid, 256, 0, st>>>(p);
  else if (at && !bt) gemm_f32_kernel<true, false><<<grid, 256, 0, st>>>(p);
  else gemm_f32_kernel<true, true><<<grid, 256, 0, st>>>(p);
  note_launch();
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// Cholesky pieces
// ---------------------------------------------------------------------------------------------
constexpr int kNB = 64;

// Unblocked right-looking Cholesky of the jb x jb diagonal block (lower part read, upper zeroed).
// Thread (ty, tx) of 4 x 64 holds column tx, rows i = ty + 4 q (q < 16), in registers.  Step j:
// the owners of column j publish it (unscaled) to a double-buffered shared vector, one barrier,
// then every thread updates its entries a[i][k] -= a[i][j] a[k][j] / d_j (= L[i][j] L[k][j]) for
// i, k > j.  The column scaling by 1/sqrt(d_k) is deferred to the end, so one barrier per step.
// A pivot d_j that is not positive and finite sets bit 0 of *status (the factor is then garbage).
// (One warp instead — the block in registers with every step unrolled, or in shared memory with
// runtime loops — measured 117 / 98 us per panel against this kernel's 22: instruction fetch of
// ~12K straight-line instructions, resp. a 2K-long dependent load-FMA-store chain per lane.)
__global__ void __launch_bounds__(256) potf2_kernel(float* a, int64_t lda, int jb, int32_t* status) {
  __shared__ float col[2][kNB];
  __shared__ float dvec[kNB];
  pdl_wait();
  pdl_launch_dependents();
  const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;
  float r[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const int i = ty + 4 * q;
    r[q] = (i < jb && tx < jb && tx <= i) ? a[(int64_t)i * lda + tx] : 0.f;
  }
  for (int j = 0; j < jb; ++j) {
    float* cj = col[j & 1];
    if (tx == j) {
#pragma unroll
      for (int q = 0; q < 16; ++q) cj[ty + 4 * q] = r[q];
    }
    __syncthreads();
    const float d = cj[j];
    if (threadIdx.x == 0) {
      dvec[j] = d;
      if ((!(d > 0.f) || !(d < INFINITY)) && status) atomicOr(status, 1);
    }
    if (tx > j && tx < jb) {
      const float lk = cj[tx] / d;
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int i = ty + 4 * q;
        if (i >= tx) r[q] = fmaf(-cj[i], lk, r[q]);
      }
    }
  }
  __syncthreads();
  if (tx < jb) {
    const float rs = 1.f / sqrtf(dvec[tx]);
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int i = ty + 4 * q;
      if (i < jb) a[(int64_t)i * lda + tx] = tx < i ? r[q] * rs : (tx == i ? sqrtf(dvec[i]) : 0.f);
    }
  }
}

// Trailing update of one Cholesky panel, C -= L21 L21^T (K = jb <= 64), on the lower 64 x 64 tiles:
// the whole K extent of both operand tiles is loaded once (no K loop, one barrier), 4 x 4 outputs
// per thread.  The 128 x 128 / K-steps-of-8 SIMT GEMM spent ~27 us per panel here (36 CTAs, eight
// dependent load rounds); these tiles give ~4x the CTAs and one load round.  Tiles on the diagonal
// also update their upper part, which zero_upper clears at the end (nothing reads it before).
__global__ void __launch_bounds__(256) syrk_k64_kernel(float* c, int64_t ldc, const float* l21, int64_t ldl,
                                                       int64_t n, int jb) {
  pdl_wait();
  pdl_launch_dependents();
  const int64_t m0 = (int64_t)blockIdx.y * 64, n0 = (int64_t)blockIdx.x * 64;
  if (n0 > m0) return;
  __shared__ __align__(16) float As[kNB][64 + 4];
  __shared__ __align__(16) float Bs[kNB][64 + 4];
  const int t = threadIdx.x;
  for (int idx = t; idx < 64 * kNB; idx += 256) {  // row r, column k of L21 (coalesced along k)
    const int r = idx / kNB, k = idx - r * kNB;
    const bool kin = k < jb;
    As[k][r] = (kin && m0 + r < n) ? l21[(m0 + r) * ldl + k] : 0.f;
    Bs[k][r] = (kin && n0 + r < n) ? l21[(n0 + r) * ldl + k] : 0.f;
  }
  __syncthreads();
  const int tx = t & 15, ty = t >> 4;
  float acc[4][4] = {};
  for (int k = 0; k < jb; ++k) {
    const float4 a = *reinterpret_cast<const float4*>(&As[k][ty * 4]);
    const float4 b = *reinterpret_cast<const float4*>(&Bs[k][tx * 4]);
    const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t r = m0 + ty * 4 + i;
    if (r >= n) continue;
    float* cr = c + r * ldc + n0 + tx * 4;
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (n0 + tx * 4 + j < n) cr[j] -= acc[i][j];
  }
}

// Solve X L^T = B in place for a panel of jb <= 64 columns: X(r, c) = b[r sr + c sc], r < R.
// A CTA stages 128 rows x jb columns through shared memory with coalesced loads/stores (along c
// when sc == 1, along r otherwise), then one thread per row solves right-looking inside the thread
// (x_j = v_j / L[j][j], then v_c -= x_j L[c][j] for all c > j: independent FMAs), the jb x jb
// lower factor and its inverse diagonal in shared memory (broadcast reads).  Used for the
// Cholesky panel (rows of A21: sr = lda, sc = 1) and for L X = B (the transposed view of B's panel
// rows: sr = 1, sc = ldb).
__global__ void __launch_bounds__(128) panel_trsm_kernel(float* b, int64_t sr, int64_t sc, int64_t R,
                                                         const float* l, int64_t ldl, int jb, int nr) {
  // smem: Lt [64][68] (L transposed: the 16 factors a chunk update needs are one float4 run),
  // rinv [64], tile [nr][65]; 128 threads stage L and the tile, then threads < nr solve a row each
  // (nr = 32 for the Cholesky panel, so the ~1000-row panels spread over ~30 SMs; 128 for the wide
  // L X = B solves)
  extern __shared__ float trsm_smem[];
  pdl_wait();
  pdl_launch_dependents();
  float (*Lt)[kNB + 4] = reinterpret_cast<float (*)[kNB + 4]>(trsm_smem);
  float* rinv = trsm_smem + kNB * (kNB + 4);
  float (*tile)[kNB + 1] = reinterpret_cast<float (*)[kNB + 1]>(trsm_smem + kNB * (kNB + 4) + kNB);
  const int nt = blockDim.x;
  for (int idx = threadIdx.x; idx < kNB * kNB; idx += nt) {
    const int i = idx / kNB, j = idx - i * kNB;
    Lt[j][i] = (i < jb && j <= i) ? l[(int64_t)i * ldl + j] : 0.f;
  }
  const int64_t r0 = (int64_t)blockIdx.x * nr;
  if (sc == 1) {  // along a row: coalesced
    for (int idx = threadIdx.x; idx < nr * kNB; idx += nt) {
      const int rr = idx / kNB, c = idx - rr * kNB;
      if (c < jb && r0 + rr < R) tile[rr][c] = b[(r0 + rr) * sr + c];
    }
  } else {
    for (int c = 0; c < jb; ++c)
      if (threadIdx.x < nr && r0 + threadIdx.x < R) tile[threadIdx.x][c] = b[(r0 + threadIdx.x) * sr + c * sc];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < jb; i += nt) rinv[i] = 1.f / Lt[i][i];
  __syncthreads();
  if (threadIdx.x < nr && r0 + threadIdx.x < R) {
    // 16-column chunks (a fully unrolled 64-column solve is ~4K instructions: i-cache bound):
    // chunk a first takes the updates of the already-solved columns j < 16a (runtime loop), then
    // solves its own 16 columns with the unrolled right-looking step.
    float* trow = tile[threadIdx.x];
    for (int a0 = 0; a0 < jb; a0 += 16) {
      float v[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) v[c] = a0 + c < jb ? trow[a0 + c] : 0.f;
      for (int j = 0; j < a0; ++j) {
        const float x = trow[j];
        const float4* lj = reinterpret_cast<const float4*>(&Lt[j][a0]);  // L[a0 .. a0+15][j]
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float4 f = lj[q];
          v[4 * q] = fmaf(-x, f.x, v[4 * q]);
          v[4 * q + 1] = fmaf(-x, f.y, v[4 * q + 1]);
          v[4 * q + 2] = fmaf(-x, f.z, v[4 * q + 2]);
          v[4 * q + 3] = fmaf(-x, f.w, v[4 * q + 3]);
        }
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        if (a0 + j < jb) {
          const float x = v[j] * rinv[a0 + j];
          v[j] = x;
          const float* lcol = &Lt[a0 + j][a0];  // L[a0 + c][a0 + j]
#pragma unroll
          for (int c = j + 1; c < 16; ++c) v[c] = fmaf(-x, lcol[c], v[c]);
        }
      }
#pragma unroll
      for (int c = 0; c < 16; ++c)
        if (a0 + c < jb) trow[a0 + c] = v[c];
    }
  }
  __syncthreads();
  if (sc == 1) {
    for (int idx = threadIdx.x; idx < nr * kNB; idx += nt) {
      const int rr = idx / kNB, c = idx - rr * kNB;
      if (c < jb && r0 + rr < R) b[(r0 + rr) * sr + c] = tile[rr][c];
    }
  } else {
    for (int c = 0; c < jb; ++c)
      if (threadIdx.x < nr && r0 + threadIdx.x < R) b[(r0 + threadIdx.x) * sr + c * sc] = tile[threadIdx.x][c];
  }
}

constexpr int kTrsmSmem = (kNB * (kNB + 4) + kNB + 128 * (kNB + 1)) * 4;
static cudaError_t trsm_attr() {
  return ensure_func_attrs(reinterpret_cast<const void*>(panel_trsm_kernel), kTrsmSmem);
}

__global__ void zero_upper_kernel(float* a, int64_t lda, int64_t n) {
  pdl_wait();
  const int64_t total = n * n;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / n, c = i - r * n;
    if (c > r) a[r * lda + c] = 0.f;
  }
}

// the Cholesky's ~3 dependent launches per 64-column panel go out with programmatic dependent launch:
// each kernel's launch and CTA scheduling overlap the previous one (its griddepcontrol.wait still
// waits for the previous grid's completion and memory flush before reading its output)
template <typename... KArgs, typename... Args>
static cudaError_t launch_la(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                             Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  note_launch();
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

static unsigned grid_for(int64_t n, int threads) {
  int64_t b = (n + threads - 1) / threads;
  if (b > 148 * 16) b = 148 * 16;
  return (unsigned)(b < 1 ? 1 : b);
}

cudaError_t launch_cholesky(float* a, int64_t lda, int64_t n, int32_t* status, cudaStream_t st) {
  if (cudaError_t e = trsm_attr()) return e;
  for (int64_t j0 = 0; j0 < n; j0 += kNB) {
    const int jb = (int)(n - j0 < kNB ? n - j0 : kNB);
    float* d = a + j0 * lda + j0;
    if (cudaError_t e = launch_la(potf2_kernel, dim3(1), dim3(256), 0, st, d, lda, jb, status)) return e;
    const int64_t rest = n - j0 - jb;
    if (rest > 0) {
      float* l21 = a + (j0 + jb) * lda + j0;
      if (cudaError_t e = launch_la(panel_trsm_kernel, dim3((unsigned)((rest + 31) / 32)), dim3(128), (size_t)kTrsmSmem, st,
                                    l21, (int64_t)lda, (int64_t)1, rest, static_cast<const float*>(d), (int64_t)lda, jb, 32))
        return e;
      const unsigned nt = (unsigned)((rest + 63) / 64);
      if (cudaError_t e = launch_la(syrk_k64_kernel, dim3(nt, nt), dim3(256), 0, st, a + (j0 + jb) * lda + (j0 + jb),
                                    (int64_t)lda, static_cast<const float*>(l21), (int64_t)lda, rest, jb))
        return e;
    }
  }
  return launch_la(zero_upper_kernel, dim3(grid_for(n * n, 256)), dim3(256), 0, st, a, (int64_t)lda, n);
}

cudaError_t launch_trsm_left(const float* l, int64_t ldl, int64_t n, float* b, int64_t ldb, int64_t ncols,
                             cudaStream_t st) {
  for (int64_t j0 = 0; j0 < n; j0 += kNB) {
    const int jb = (int)(n - j0 < kNB ? n - j0 : kNB);
    if (cudaError_t e = trsm_attr()) return e;
    panel_trsm_kernel<<<(unsigned)((ncols + 127) / 128), 128, kTrsmSmem, st>>>(b + j0 * ldb, 1, ldb, ncols,
                                                                         l + j0 * ldl + j0, ldl, jb, 128);
    note_launch();
    const int64_t rest = n - j0 - jb;
    if (rest > 0) {
      GemmF32Params g = {};
      g.M = rest; g.N = ncols; g.K = jb;
      g.A = l + (j0 + jb) * ldl + j0; g.lda = ldl;
      g.B = b + j0 * ldb; g.ldb = ldb;
      g.C = b + (j0 + jb) * ldb; g.ldc = ldb;
      g.Cin = static_cast<const float*>(g.C); g.ldcin = ldb;
      g.alpha = -1.f; g.beta = 1.f;
      cudaError_t e = launch_gemm_f32(g, false, false, st);
      if (e != cudaSuccess) return e;
    }
  }
  return cudaSuccess;
}

// ---------------------------------------------------------------------------------------------
// element-wise pieces
// ---------------------------------------------------------------------------------------------
// tr[i] = sum_j mats[i][j][j] in FP64, for up to two square matrices (one CTA)
__global__ void __launch_bounds__(256) trace2_kernel(const float* a, int64_t na, int64_t lda, const float* b,
                                                     int64_t nb, int64_t ldb, double* tr) {
  __shared__ double red[2][256];
  double sa = 0.0, sb = 0.0;
  for (int64_t i = threadIdx.x; i < na; i += 256) sa += (double)a[i * lda + i];
  if (b)
    for (int64_t i = threadIdx.x; i < nb; i += 256) sb += (double)b[i * ldb + i];
  red[0][threadIdx.x] = sa;
  red[1][threadIdx.x] = sb;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      red[0][threadIdx.x] += red[0][threadIdx.x + s];
      red[1][threadIdx.x] += red[1][threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    tr[0] = red[0][0];
    if (b) tr[1] = red[1][0];
  }
}

cudaError_t launch_trace2(const float* a, int64_t na, int64_t lda, const float* b, int64_t nb, int64_t ldb,
                          double* tr, cudaStream_t st) {
  trace2_kernel<<<1, 256, 0, st>>>(a, na, lda, b, nb, ldb, tr);
  note_launch();
  return cudaGetLastError();
}

// l = lower(scale * sym(a)) + eps I (upper zeroed); eps = tr_dev ? eps_rel * t : eps_host with
// t = tr_dev[0] * tr_scale, and t <= 0 -> 1 (D30)
__global__ void jitter_copy_kernel(const float* a, int64_t lda, float* l, int64_t ldl, int64_t n, float scale,
                                   float eps_host, const double* tr_dev, double tr_scale, float eps_rel) {
  float eps = eps_host;
  if (tr_dev) {
    const double t = tr_dev[0] * tr_scale;
    eps = (float)((double)eps_rel * (t > 0.0 ? t : 1.0));
  }
  const int64_t total = n * n;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / n, c = i - r * n;
    float v = 0.f;
    if (c <= r) {
      v = scale * (0.5f * (a[r * lda + c] + a[c * lda + r]));
      if (c == r) v += eps;
    }
    l[r * ldl + c] = v;
  }
}

cudaError_t launch_jitter_copy(const float* a, int64_t lda, float* l, int64_t ldl, int64_t n, float scale,
                               float eps_host, const double* tr_dev, double tr_scale, float eps_rel, cudaStream_t st) {
  jitter_copy_kernel<<<grid_for(n * n, 256), 256, 0, st>>>(a, lda, l, ldl, n, scale, eps_host, tr_dev, tr_scale, eps_rel);
  note_launch();
  return cudaGetLastError();
}

// out = sym(m X + (1 - m) X1) + eps I, eps = eps_rel * tr_dev[0] / n; X1 is a
// Gram product of which only the lower triangle is valid (it is symmetric by construction)
__global__ void ema_sym_kernel(const float* x, const float* x1, float* out, int64_t n, float m, float eps_rel,
                               const double* tr_dev) {
  const float eps = (float)((double)eps_rel * tr_dev[0] / (double)n);
  const int64_t total = n * n;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / n, c = i - r * n;
    const float g = x1[r >= c ? r * n + c : c * n + r];
    const float a = fmaf(m, x[r * n + c], (1.f - m) * g);
    const float b = fmaf(m, x[c * n + r], (1.f - m) * g);
    float v = 0.5f * (a + b);
    if (r == c) v += eps;
    out[i] = v;
  }
}

// U = Ut / s, V = Vt * s with s = tr(Ut) / M
__global__ void renorm_kernel(const float* ut, float* u, int64_t mm, const float* vt, float* v, int64_t nn,
                              const double* tr_dev) {
  const double s = tr_dev[0] / (double)mm;
  const float inv = (float)(1.0 / s), sf = (float)s;
  const int64_t tu = mm * mm, tv = nn * nn;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tu + tv; i += (int64_t)gridDim.x * blockDim.x) {
    if (i < tu) u[i] = ut[i] * inv;
    else v[i - tu] = vt[i - tu] * sf;
  }
}

// W_c = W - Mean (row-major and transposed copies), Mean <- m Mean + (1 - m) W; 32 x 32 tiles
template <typename T>
__global__ void __launch_bounds__(256) center_kernel(const T* w, int64_t ldw, float* mean, int64_t mm, int64_t nn,
                                                     float m, float* wc, float* wct) {
  __shared__ float tile[32][33];
  const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t r = r0 + ty + 8 * i, c = c0 + tx;
    float d = 0.f;
    if (r < mm && c < nn) {
      const float x = to_f32(w[r * ldw + c]);
      const float mu = mean[r * nn + c];
      d = x - mu;
      wc[r * nn + c] = d;
      mean[r * nn + c] = fmaf(m, mu, (1.f - m) * x);
    }
    tile[ty + 8 * i][tx] = d;
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t c = c0 + ty + 8 * i, r = r0 + tx;
    if (r < mm && c < nn) wct[c * mm + r] = tile[tx][ty + 8 * i];
  }
}

template <typename T>
__global__ void matnorm_init_kernel(const T* w, int64_t ldw, float* mean, float* u, int64_t mm, float* v, int64_t nn) {
  const int64_t tw = mm * nn, tu = mm * mm, tv = nn * nn;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < tw + tu + tv; i += (int64_t)gridDim.x * blockDim.x) {
    if (i < tw) {
      const int64_t r = i / nn, c = i - r * nn;
      mean[i] = to_f32(w[r * ldw + c]);
    } else if (i < tw + tu) {
      const int64_t j = i - tw;
      u[j] = (j / mm == j % mm) ? 1.f : 0.f;
    } else {
      const int64_t j = i - tw - tu;
      v[j] = (j / nn == j % nn) ? 1.f : 0.f;
    }
  }
}

cudaError_t launch_matnorm_init(const void* w, bool bf16, int64_t ldw, float* mean, float* u, int64_t mm, float* v,
                                int64_t nn, cudaStream_t st) {
  const unsigned g = grid_for(mm * nn + mm * mm + nn * nn, 256);
  if (bf16) matnorm_init_kernel<<<g, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(w), ldw, mean, u, mm, v, nn);
  else matnorm_init_kernel<<<g, 256, 0, st>>>(static_cast<const float*>(w), ldw, mean, u, mm, v, nn);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_matnorm_update(const MatnormParams& p, cudaStream_t st) {
  const int64_t mm = p.M, nn = p.N;
  cudaError_t e;
  // traces of the current factors (eps_U, eps_V)
  if ((e = launch_trace2(p.u, mm, mm, p.v, nn, nn, p.tr, st)) != cudaSuccess) return e;
  // W_c, W_c^T, Mean EMA
  {
    const dim3 grid((unsigned)((nn + 31) / 32), (unsigned)((mm + 31) / 32));
    if (p.w_bf16)
      center_kernel<<<grid, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(p.w), p.ldw, p.mean, mm, nn, p.m, p.wc, p.wct);
    else
      center_kernel<<<grid, 256, 0, st>>>(static_cast<const float*>(p.w), p.ldw, p.mean, mm, nn, p.m, p.wc, p.wct);
    note_launch();
  }
  // L_V L_V^T = V + eps_V I, L_U L_U^T = U + eps_U I
  if ((e = launch_jitter_copy(p.v, nn, p.lv, nn, nn, 1.f, 0.f, p.tr + 1, 1.0 / (double)nn, p.eps_rel, st)) != cudaSuccess)
    return e;
  if ((e = launch_cholesky(p.lv, nn, nn, p.status, st)) != cudaSuccess) return e;
  if ((e = launch_jitter_copy(p.u, mm, p.lu, mm, mm, 1.f, 0.f, p.tr, 1.0 / (double)mm, p.eps_rel, st)) != cudaSuccess)
    return e;
  if ((e = launch_cholesky(p.lu, mm, mm, p.status, st)) != cudaSuccess) return e;
  // W~^T = L_V^{-1} W_c^T (i.e. W~ = W_c L_V^{-T}),  W^ = L_U^{-1} W_c
  if ((e = launch_trsm_left(p.lv, nn, nn, p.wct, mm, mm, st)) != cudaSuccess) return e;
  if ((e = launch_trsm_left(p.lu, mm, mm, p.wc, nn, nn, st)) != cudaSuccess) return e;
  // U' = (1/N) W~ W~^T = (1/N) (W~^T)^T (W~^T),  V' = (1/M) W^^T W^
  {
    GemmF32Params g = {};
    g.M = mm; g.N = mm; g.K = nn;
    g.A = p.wct; g.lda = mm;
    g.B = p.wct; g.ldb = mm;
    g.C = p.u1; g.ldc = mm;
    g.alpha = (float)(1.0 / (double)nn);
    g.lower_only = 1;  // symmetric: the strict upper tiles are not computed (ema_sym reads the lower)
    if ((e = launch_gemm_f32(g, true, false, st)) != cudaSuccess) return e;
    g.M = nn; g.N = nn; g.K = mm;
    g.A = p.wc; g.lda = nn;
    g.B = p.wc; g.ldb = nn;
    g.C = p.v1; g.ldc = nn;
    g.alpha = (float)(1.0 / (double)mm);
    if ((e = launch_gemm_f32(g, true, false, st)) != cudaSuccess) return e;
  }
  // EMA + symmetrise + eps I into the (now free) factor buffers, then the trace renormalisation
  ema_sym_kernel<<<grid_for(mm * mm, 256), 256, 0, st>>>(p.u, p.u1, p.lu, mm, p.m, p.eps_rel, p.tr);
  ema_sym_kernel<<<grid_for(nn * nn, 256), 256, 0, st>>>(p.v, p.v1, p.lv, nn, p.m, p.eps_rel, p.tr + 1);
  note_launch(2);
  if ((e = launch_trace2(p.lu, mm, mm, nullptr, 0, 0, p.tr + 2, st)) != cudaSuccess) return e;
  renorm_kernel<<<grid_for(mm * mm + nn * nn, 256), 256, 0, st>>>(p.lu, p.u, mm, p.lv, p.v, nn, p.tr + 2);
  note_launch();
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// Philox4x64-10 normals (D31)
// ---------------------------------------------------------------------------------------------
LOKA_DEVINL void philox4x64_10(uint64_t c[4], uint64_t k0, uint64_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t lo0 = c[0] * 0xD2E7470EE14C6C93ull, hi0 = __umul64hi(c[0], 0xD2E7470EE14C6C93ull);
    const uint64_t lo1 = c[2] * 0xCA5A826395121157ull, hi1 = __umul64hi(c[2], 0xCA5A826395121157ull);
    const uint64_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
    k0 += 0x9E3779B97F4A7C15ull;
    k1 += 0xBB67AE8584CAA73Bull;
  }
}

LOKA_DEVINL void box_muller(uint64_t xa, uint64_t xb, float& z0, float& z1) {
  const float u1 = (float)((xa >> 40) + 1ull) * 0x1p-24f;  // (0, 1], exact
  const float u2 = (float)(xb >> 40) * 0x1p-24f;           // [0, 1), exact
  const float r = sqrtf(-2.f * logf(u1));
  float s, c;
  sincospif(2.f * u2, &s, &c);
  z0 = r * c;
  z1 = r * s;
}

// out[e] = normal number (offset + e) of the stream keyed by seed; one thread per Philox block
__global__ void __launch_bounds__(256) philox_normal_kernel(uint64_t seed, uint64_t offset, int64_t n, float* out) {
  const uint64_t b0 = offset >> 2;
  const uint64_t nblk = ((offset + (uint64_t)n - 1) >> 2) - b0 + 1;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nblk; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t blk = b0 + i;
    uint64_t c[4] = {blk, 0ull, 0ull, 0ull};
    philox4x64_10(c, seed, 0ull);
    float z[4];
    box_muller(c[0], c[1], z[0], z[1]);
    box_muller(c[2], c[3], z[2], z[3]);
    const uint64_t g0 = blk * 4;
    if (g0 >= offset && g0 + 3 < offset + (uint64_t)n && ((g0 - offset) & 3) == 0 &&
        (reinterpret_cast<uintptr_t>(out) & 15) == 0) {
      *reinterpret_cast<float4*>(out + (g0 - offset)) = make_float4(z[0], z[1], z[2], z[3]);
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint64_t g = g0 + j;
        if (g >= offset && g < offset + (uint64_t)n) out[g - offset] = z[j];
      }
    }
  }
}

cudaError_t launch_philox_normal(uint64_t seed, uint64_t offset, int64_t n, float* out, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int64_t nblk = (int64_t)(((offset + (uint64_t)n - 1) >> 2) - (offset >> 2) + 1);
  philox_normal_kernel<<<grid_for(nblk, 256), 256, 0, st>>>(seed, offset, n, out);
  note_launch();
  return cudaGetLastError();
}

}  // namespace loka
