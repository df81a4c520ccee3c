// quantize_tma.cu — a1/a2: ROW / TENSOR-cast quantize streamed through shared memory
// with bulk (TMA-engine) copies: the HBM-bound form of the quantize step (PAPER.md:207-213
// "Quantization overhead consumes over 30% of end-to-end GEMM latency").
//
// Same arithmetic as quantize.cu (bit-identical codes and scales; D1-D3, D7):
// granule amax on |x| bit patterns, s = fl32(amax/max), r = fl32(max/amax) (UE8M0: powers of
// two), q = satRNE(fl32(x * r)).
//
// Why a second implementation: the register-resident warp-per-row kernels issue 16-byte loads
// and 8-byte stores per lane; with reads and writes interleaved at that granularity they reach
// ~60% of the measured HBM copy bandwidth.  Here a persistent CTA per SM moves whole rows:
//   * one producer lane issues 1-D bulk copies global -> smem (one per input row, <= 16 KB) into
//     a ring of stages of 8 rows, completing on the stage's mbarrier;
//   * 8 consumer warps (one row each) read their row from smem, reduce the granule amax, cast, and
//     write the codes into a per-warp smem staging row that one lane stores back with a single
//     1-D bulk copy smem -> global (bulk_group; the staging row is reused after wait_group.read);
//   * the stage is released (empty mbarrier, 8 arrivals) as soon as every warp has read its row.
// Requirements (else quantize.cu's kernels run): rows of cols * elem bytes that are multiples of
// 16 and <= 16 KB, 16-byte aligned row starts (ld * elem % 16 == 0 by the ABI), no transposed copy.
#include "common.cuh"
#include "launch.h"

namespace loka {

constexpr int kQtMaxStages = 12;  // ring depth: as many 8-row stages as fit (>= 2), so a CTA's whole
                                  // share of a small grouped launch (cfg2: ~8 stages) is in flight at once
// rows per stage = consumer warps (template R): 8 for long rows, 16 for rows <= 4 KB (each warp
// works through its rows one after another, so short rows want more warps in flight per SM)
constexpr int kQtMaxRowBytes = 16384;              // input row bytes per stage slot

template <typename Tin> struct QtIn;
template <> struct QtIn<__nv_bfloat16> {
  // 8 elements from 16 bytes of smem: |x| max bits + values
  static LOKA_DEVINL uint4 ld(uint32_t a) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
  }
  static LOKA_DEVINL uint32_t amax(uint4 w) {
    uint32_t a = w.x & 0x7FFF7FFFu, b = w.y & 0x7FFF7FFFu, c = w.z & 0x7FFF7FFFu, d = w.w & 0x7FFF7FFFu, m;
    asm("max.u16x2 %0, %1, %2;" : "=r"(a) : "r"(a), "r"(b));
    asm("max.u16x2 %0, %1, %2;" : "=r"(c) : "r"(c), "r"(d));
    asm("max.u16x2 %0, %1, %2;" : "=r"(m) : "r"(a), "r"(c));
    return max(m & 0xFFFFu, m >> 16) << 16;
  }
  template <int FMT>
  static LOKA_DEVINL uint2 cast(uint4 w, float r) {
    float f[8] = {bf16lo_to_f32(w.x), bf16hi_to_f32(w.x), bf16lo_to_f32(w.y), bf16hi_to_f32(w.y),
                  bf16lo_to_f32(w.z), bf16hi_to_f32(w.z), bf16lo_to_f32(w.w), bf16hi_to_f32(w.w)};
#pragma unroll
    for (int i = 0; i < 8; ++i) f[i] = __fmul_rn(f[i], r);
    return make_uint2(cvt_fp8x4<FMT>(f[0], f[1], f[2], f[3]), cvt_fp8x4<FMT>(f[4], f[5], f[6], f[7]));
  }
  static constexpr int kElemsPer16B = 8;
};

// cast a row held in smem into the staging row: 4 chunks of 16 B per lane loaded before any is
// converted (the smem latency of one chunk hides behind the others' conversion)
// AMAX (bf16): a running max of the 16-bit |x| patterns, two per word (max.u16x2), folded once at the end
LOKA_DEVINL uint32_t vmax16x2(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("max.u16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
LOKA_DEVINL void amax_acc(uint32_t& pm, uint4 w) {
  pm = vmax16x2(vmax16x2(pm, w.x & 0x7FFF7FFFu), vmax16x2(w.y & 0x7FFF7FFFu, vmax16x2(w.z & 0x7FFF7FFFu,
                                                                                   w.w & 0x7FFF7FFFu)));
}
template <typename Tin, int FMT, bool AMAX = false>
LOKA_DEVINL uint32_t qt_cast_row(uint32_t src, uint32_t dsts, int nchunks, int lane, float r) {
  static_assert(!AMAX || sizeof(Tin) == 2, "packed amax: bf16 rows");
  uint32_t pm = 0;  // AMAX: this lane's max |x| over the row, 16-bit patterns packed in pairs
  int c = lane;
  for (; c + 96 < nchunks; c += 128) {
    uint4 w[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) w[u] = QtIn<Tin>::ld(src + 16u * (c + 32 * u));
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (AMAX) amax_acc(pm, w[u]);
      const uint2 code = QtIn<Tin>::template cast<FMT>(w[u], r);
      asm volatile("st.shared.v2.u32 [%0], {%1,%2};" ::"r"(dsts + 8u * (c + 32 * u)), "r"(code.x), "r"(code.y)
                   : "memory");
    }
  }
  for (; c < nchunks; c += 32) {
    const uint4 w = QtIn<Tin>::ld(src + 16u * c);
    if (AMAX) amax_acc(pm, w);
    const uint2 code = QtIn<Tin>::template cast<FMT>(w, r);
    asm volatile("st.shared.v2.u32 [%0], {%1,%2};" ::"r"(dsts + 8u * c), "r"(code.x), "r"(code.y) : "memory");
  }
  return max(pm & 0xFFFFu, pm >> 16) << 16;  // as FP32 bits
}

// Work items are groups of 8 consecutive rows of one tensor of the QuantGroup (a single tensor
// is a group of one); item gg belongs to tensor t with rgs[t] <= gg < rgs[t+1] (row-group prefix).
template <int R>
LOKA_DEVINL int qt_locate(const QuantGroup& grp, int64_t gg, int64_t& first_row) {
  int64_t acc = 0;
  for (int t = 0; t < grp.G; ++t) {
    const int64_t n = (grp.p[t].rows + R - 1) / R;
    if (gg < acc + n) {
      first_row = (gg - acc) * R;
      return t;
    }
    acc += n;
  }
  first_row = 0;
  return -1;
}

template <typename Tin, int FMT, int SF, int GRAN, int kQtRows>
__global__ void __launch_bounds__(32 * (kQtRows + 1), 1)
    quant_tma_kernel(const __grid_constant__ QuantGroup grp, int64_t ngroups, int max_cols, int nstages,
                     const float* amax_dev, uint32_t* amax_next) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
  const int slot_in = (max_cols * (int)sizeof(Tin) + 127) & ~127, slot_out = (max_cols + 127) & ~127;
  uint8_t* sin = smem;                                          // [stage][row][slot_in]
  uint8_t* sout = smem + nstages * kQtRows * slot_in;           // [warp][2][slot_out]
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(sout + kQtRows * 2 * slot_out);
  uint64_t* empty_bar = full_bar + kQtMaxStages;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < nstages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], kQtRows);
    }
    fence_barrier_init();
  }
  __syncthreads();
  pdl_wait();
  // Every CTA of this grid is resident (grid <= SMs): let the dependent launch (the layer stack /
  // GEMM that consumes these codes) start its prologue on SMs as they free up.  Safe at any point:
  // the dependent's griddepcontrol.wait still waits for this grid's completion and memory flush.
  pdl_launch_dependents();

  if (warp == kQtRows) {  // ===== producer =====
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int64_t g = blockIdx.x; g < ngroups; g += gridDim.x) {
        mbar_wait(&empty_bar[s], ph ^ 1u, 1);
        int64_t r0;
        const QuantParams& p = grp.p[qt_locate<kQtRows>(grp, g, r0)];
        const int in_bytes = (int)(p.cols * (int64_t)sizeof(Tin));
        const int nr = (int)imin64(kQtRows, p.rows - r0);
        mbar_arrive_expect_tx(&full_bar[s], (uint32_t)(nr * in_bytes));
        for (int i = 0; i < nr; ++i) {
          const int64_t row = r0 + i;
          bulk_load_g2s(sin + (s * kQtRows + i) * slot_in,
                        reinterpret_cast<const uint8_t*>(p.x) + row * p.ldx * (int64_t)sizeof(Tin),
                        (uint32_t)in_bytes, &full_bar[s]);
        }
        if (++s == nstages) s = 0, ph ^= 1u;
      }
    }
    return;
  }

  // ===== consumers: warp w takes row w of every stage =====
  float r_tensor = 1.f;
  if constexpr (GRAN == LOKA_GRAN_TENSOR) {  // (G == 1)
    float s_t;
    scales_from_amax<FMT, SF>(*amax_dev, s_t, r_tensor);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      if (grp.p[0].scales) grp.p[0].scales[0] = s_t;
      if (grp.p[0].scales_t) grp.p[0].scales_t[0] = s_t;
    }
  }
  int nst = 0, s = -1;
  uint32_t ph = 1;
  uint32_t am_next = 0;
  for (int64_t g = blockIdx.x; g < ngroups; g += gridDim.x) {
    if (++s == nstages) s = 0;
    if (s == 0) ph ^= 1u;
    int64_t r0;
    const QuantParams& p = grp.p[qt_locate<kQtRows>(grp, g, r0)];
    const int in_bytes = (int)(p.cols * (int64_t)sizeof(Tin)), out_bytes = (int)p.cols;
    const int64_t row = r0 + warp;
    if (lane == 0) mbar_wait(&full_bar[s], ph, 2);
    __syncwarp();
    if (row >= p.rows) {  // ragged last group: nothing to read, release the slot
      if (lane == 0) mbar_arrive(&empty_bar[s]);
      continue;
    }
    const uint32_t src = smem_u32(sin + (s * kQtRows + warp) * slot_in);
    uint8_t* dst = sout + (warp * 2 + (nst & 1)) * slot_out;
    if (lane == 0) bulk_wait_read_le1();  // this staging row's previous store has been read
    __syncwarp();
    const uint32_t dsts = smem_u32(dst);
    const int nchunks = in_bytes / 16;  // 16-byte input chunks of the row
    if constexpr (GRAN == LOKA_GRAN_ROW) {
      uint32_t am = 0;
      for (int c = lane; c < nchunks; c += 32) am = max(am, QtIn<Tin>::amax(QtIn<Tin>::ld(src + 16u * c)));
      am = warp_max_u32(am);
      if (am >= 0x7F800000u && lane == 0 && p.status) atomicOr(p.status, LOKA_DEVSTATUS_NONFINITE);
      float sc, r;
      scales_from_amax<FMT, SF>(__uint_as_float(am), sc, r);
      if (lane == 0) {
        if (p.scales) p.scales[row] = sc;
        if (p.scales_t) p.scales_t[row] = sc;
      }
      qt_cast_row<Tin, FMT>(src, dsts, nchunks, lane, r);
    } else if constexpr (GRAN == LOKA_GRAN_BLK_1x128) {
      // 1x128 granules: chunk c (8 elements) lies in block c / 16, so in each 32-chunk step the two
      // half-warps hold one block each: half-warp max reduction, then scale and cast in registers
      const int nblk = (int)((p.cols + 127) / 128);
      for (int c0 = 0; c0 < nchunks; c0 += 128) {
        uint4 w[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int c = c0 + 32 * u + lane;
          w[u] = c < nchunks ? QtIn<Tin>::ld(src + 16u * c) : make_uint4(0u, 0u, 0u, 0u);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int c = c0 + 32 * u + lane;
          if (c0 + 32 * u >= nchunks) break;  // (uniform over the warp)
          uint32_t am = QtIn<Tin>::amax(w[u]);
#pragma unroll
          for (int o = 8; o >= 1; o >>= 1) am = max(am, __shfl_xor_sync(0xFFFFFFFFu, am, o));
          if (am >= 0x7F800000u && (lane & 15) == 0 && p.status) atomicOr(p.status, LOKA_DEVSTATUS_NONFINITE);
          float sc, r;
          scales_from_amax<FMT, SF>(__uint_as_float(am), sc, r);
          const int blk = (c0 + 32 * u) / 16 + (lane >> 4);
          if ((lane & 15) == 0 && blk < nblk && p.scales) p.scales[row * nblk + blk] = sc;
          if (c < nchunks) {
            const uint2 code = QtIn<Tin>::template cast<FMT>(w[u], r);
            asm volatile("st.shared.v2.u32 [%0], {%1,%2};" ::"r"(dsts + 8u * c), "r"(code.x), "r"(code.y)
                         : "memory");
          }
        }
      }
    } else if (amax_next) {  // TENSOR, delayed scaling: cast with the given amax, record this tensor's
      am_next = max(am_next, qt_cast_row<Tin, FMT, true>(src, dsts, nchunks, lane, r_tensor));
    } else {  // TENSOR cast with the pre-computed amax
      qt_cast_row<Tin, FMT>(src, dsts, nchunks, lane, r_tensor);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty_bar[s]);  // input row consumed
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(p.q + row * p.ldq),
                   "r"(dsts), "r"((uint32_t)out_bytes)
                   : "memory");
      bulk_commit();
    }
    ++nst;
  }
  if (lane == 0) bulk_wait0();
  if (GRAN == LOKA_GRAN_TENSOR && amax_next) {  // one atomicMax of the bit pattern per warp
    am_next = warp_max_u32(am_next);
    if (lane == 0 && am_next) {
      atomicMax(amax_next, am_next);
      if (am_next >= 0x7F800000u && grp.p[0].status) atomicOr(grp.p[0].status, LOKA_DEVSTATUS_NONFINITE);
    }
  }
}

static int quant_tma_rows(int64_t cols, int in_elem) { return cols * in_elem <= 4096 ? 16 : 8; }
static size_t quant_tma_smem_n(int64_t cols, int in_elem, int nstages) {
  const int64_t slot_in = (cols * in_elem + 127) & ~int64_t(127), slot_out = (cols + 127) & ~int64_t(127);
  const int R = quant_tma_rows(cols, in_elem);
  return (size_t)(nstages * R * slot_in + R * 2 * slot_out + 2 * kQtMaxStages * 8 + 128);
}
// deepest ring (<= kQtMaxStages) that fits in 227 KB; 0 if not even two stages fit
static int quant_tma_stages(int64_t cols, int in_elem) {
  for (int n = kQtMaxStages; n >= 2; --n)
    if (quant_tma_smem_n(cols, in_elem, n) <= 227 * 1024) return n;
  return 0;
}
size_t quant_tma_smem(int64_t cols, int in_elem) {
  const int n = quant_tma_stages(cols, in_elem);
  return n ? quant_tma_smem_n(cols, in_elem, n) : (size_t)-1;
}

bool quant_tma_eligible(const QuantParams& p, bool in_bf16, int gran) {
  if (!in_bf16 || !p.q || p.qt || p.rows <= 0) return false;
  // (BLK_1x128 runs here too, but measured slower than quantize.cu's register-resident kernel at
  // 262144 x 4096: 1.18 vs 0.81 ms (profiles/r02g_quantize_262k.json) — ROW and TENSOR only)
  if (gran != LOKA_GRAN_ROW && gran != LOKA_GRAN_TENSOR) return false;
  if (p.cols % 16 || p.cols * 2 > kQtMaxRowBytes) return false;
  if ((p.ldx * 2) % 16 || p.ldq % 16) return false;
  if ((reinterpret_cast<uintptr_t>(p.x) & 15) || (reinterpret_cast<uintptr_t>(p.q) & 15)) return false;
  return quant_tma_smem(p.cols, 2) <= 227 * 1024;
}

template <int FMT, int SF, int GRAN, int kQtRows>
static cudaError_t launch_qt_r(const QuantGroup& grp, int64_t max_cols, const float* amax_dev, int num_sms,
                               cudaStream_t st, uint32_t* amax_next) {
  auto kern = quant_tma_kernel<__nv_bfloat16, FMT, SF, GRAN, kQtRows>;
  const size_t smem = quant_tma_smem(max_cols, 2);
  const int nstages = quant_tma_stages(max_cols, 2);
  {
    cudaError_t e = ensure_func_attrs(reinterpret_cast<const void*>(kern), 227 * 1024);
    if (e != cudaSuccess) return e;
  }
  int64_t ngroups = 0;
  for (int t = 0; t < grp.G; ++t) ngroups += (grp.p[t].rows + kQtRows - 1) / kQtRows;
  if (ngroups == 0) return cudaSuccess;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(ngroups < num_sms ? ngroups : num_sms));
  cfg.blockDim = dim3(32 * (kQtRows + 1));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  note_launch();
  return cudaLaunchKernelEx(&cfg, kern, grp, ngroups, (int)max_cols, nstages, amax_dev, amax_next);
}
template <int FMT, int SF, int GRAN>
static cudaError_t launch_qt(const QuantGroup& grp, int64_t max_cols, const float* amax_dev, int num_sms,
                             cudaStream_t st, uint32_t* amax_next) {
  if (quant_tma_rows(max_cols, 2) == 16)
    return launch_qt_r<FMT, SF, GRAN, 16>(grp, max_cols, amax_dev, num_sms, st, amax_next);
  return launch_qt_r<FMT, SF, GRAN, 8>(grp, max_cols, amax_dev, num_sms, st, amax_next);
}

cudaError_t launch_quantize_tma_group(const QuantGroup& grp, int64_t max_cols, int fmt, int scale_fmt, int gran,
                                      const float* amax_dev, int num_sms, cudaStream_t st, uint32_t* amax_next) {
#define LOKA_QT(F, S, G) \
  if (fmt == F && scale_fmt == S && gran == G) \
    return launch_qt<F, S, G>(grp, max_cols, amax_dev, num_sms, st, amax_next);
#define LOKA_QT_G(F, S)                     \
  LOKA_QT(F, S, LOKA_GRAN_ROW)              \
  LOKA_QT(F, S, LOKA_GRAN_TENSOR)           \
  LOKA_QT(F, S, LOKA_GRAN_BLK_1x128)
  LOKA_QT_G(LOKA_E4M3, LOKA_SCALE_F32)
  LOKA_QT_G(LOKA_E4M3, LOKA_SCALE_UE8M0)
  LOKA_QT_G(LOKA_E5M2, LOKA_SCALE_F32)
  LOKA_QT_G(LOKA_E5M2, LOKA_SCALE_UE8M0)
#undef LOKA_QT_G
#undef LOKA_QT
  return cudaErrorNotSupported;
}

cudaError_t launch_quantize_tma(const QuantParams& p, int fmt, int scale_fmt, int gran, const float* amax_dev,
                                int num_sms, cudaStream_t st, uint32_t* amax_next) {
  static thread_local QuantGroup grp;  // ~7 KB: not on the stack
  grp.G = 1;
  grp.row_start[0] = 0;
  grp.row_start[1] = p.rows;
  grp.p[0] = p;
  return launch_quantize_tma_group(grp, p.cols, fmt, scale_fmt, gran, amax_dev, num_sms, st, amax_next);
}

}  // namespace loka
