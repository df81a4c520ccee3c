// quantize_tile.cu — a1-a3 for the tile-shaped granularities, streamed through shared memory with
// TMA: 1x128 / 128x128 / 128x1 blocks (PAPER.md:161-169 blockwise scaling, P:547 per-direction
// layouts), COL (with its amax pre-pass), and every cast-transpose (ROW / COL / TENSOR / 1x128 /
// 128x1 / 128x128 with the K-major copy qt; the blockwise recipe's dual 1x128 + 128x1 pass).
// "Quantization overhead consumes over 30% of end-to-end GEMM latency" — this is
// HBM-bound work, so the design is about keeping loads in flight, not about arithmetic.
//
// Same arithmetic as quantize_t.cu / quantize.cu (bit-identical codes and scales; D1-D3,
// D6, D7): granule amax on |x| bit patterns, s = fl32(amax/max), r = fl32(max/amax) (UE8M0: powers
// of two), q = satRNE(fl32(x * r)).
//
// Why it replaces the one-shot tile kernel for bf16 input: that kernel loads a 128 x 128 tile into
// registers, reduces, casts and stores, then exits — with 2-3 CTAs per SM the loads of the next
// tile only start when a CTA retires, and it reached 3.1-4.4 TB/s.  Here a persistent CTA per SM:
//   * one producer lane streams 128 x 128 bf16 tiles (32 KB, rows of 256 B, no swizzle: a
//     half-warp's 16-byte reads of one row are conflict-free) into a 4-stage ring (3 with a
//     transposed copy) with 2D TMA loads;
//   * two consumer groups of 4 warps take alternate tiles and synchronise only among themselves
//     (named barriers 1 / 2), so one group's barrier waits and reciprocal latencies overlap the
//     other's loads and casts; full barriers are per (group, stage) — with 3 stages both groups use
//     every stage, and a shared barrier's parity would let a group take the other group's pending
//     fill for its own completed phase;
//   * a warp owns 32 rows of its group's tile, 8 elements per lane per row, in two half-passes of 16
//     rows: reduce the granule amax (16-bit maxima of two rows / columns per word; half-warp
//     shuffles for row-like granules, a shared-memory column reduction for column-like ones),
//     compute ONE reciprocal per lane (the granule's lanes share it by shuffle or through shared
//     memory instead of each dividing), cast, and write the codes into a 128B-swizzled staging tile;
//   * the transposed copy goes through a code tile (XOR-swizzled by row/8 so the 4 x 4 byte
//     transposes read it with at most 2-way conflicts) into its own staging tile;
//   * one thread per group stores its staging tiles with 2D TMA stores (bulk group, reused after
//     wait_group.read).
// Ragged edges cost nothing: TMA zero-fills out-of-range input (|0| never raises an amax) and
// clips out-of-range output; only the scale writes are bounds-checked.
#include "common.cuh"
#include "launch.h"

namespace loka {

constexpr int kQlThreads = 288;                          // 2 consumer groups of 4 warps + the producer warp
constexpr int kQlIn = 128 * 256;                         // one tile: 128 rows x 256 B (bf16)
// Shared memory per instance (QT: a transposed copy is written).  Per consumer group: a q staging
// tile [128 rows][128 B] SW128, with QT a qt staging tile and the transpose's code tile.
template <bool QT> struct QlLayout {
  static constexpr int kStages = QT ? 3 : 4;
  static constexpr int kOffQ = kStages * kQlIn;                    // [2 groups][16 KB]
  static constexpr int kOffQT = kOffQ + 2 * 16384;                 // [2][16 KB] (QT)
  static constexpr int kOffTQ = kOffQT + (QT ? 2 * 16384 : 0);     // [2][16 KB] (QT)
  static constexpr int kOffRed = kOffTQ + (QT ? 2 * 16384 : 0);    // u32 [2][4 warps][128 columns]
  static constexpr int kOffR = kOffRed + 2 * 4 * 128 * 4;          // f32 [2][128] per-row / per-column r
  static constexpr int kOffRed2 = kOffR + 2 * 128 * 4;             // u32 [2][4] 128x128 partials
  static constexpr int kOffBar = kOffRed2 + 64;
  static constexpr int kSmem = kOffBar + 3 * 4 * 8 + 1024;         // + alignment slack
  static_assert(kSmem <= 227 * 1024, "quantize tile smem");
};
constexpr int kGranDualT = 64;                           // (= quantize_t.cu's kGranDual)

LOKA_DEVINL uint4 lds_u4(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
LOKA_DEVINL uint32_t lds_u32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
LOKA_DEVINL void sts_u2(uint32_t a, uint32_t x, uint32_t y) {
  asm volatile("st.shared.v2.u32 [%0], {%1,%2};" ::"r"(a), "r"(x), "r"(y) : "memory");
}
LOKA_DEVINL uint32_t prmt_b32(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
  return d;
}
// 4 x 4 byte transpose: in[i] = row i (bytes = columns 0..3) -> out[k] = column k (bytes = rows)
LOKA_DEVINL void tr4x4(uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t (&o)[4]) {
  const uint32_t t0 = prmt_b32(a0, a1, 0x5140u), t1 = prmt_b32(a2, a3, 0x5140u);
  const uint32_t t2 = prmt_b32(a0, a1, 0x7362u), t3 = prmt_b32(a2, a3, 0x7362u);
  o[0] = prmt_b32(t0, t1, 0x5410u);
  o[1] = prmt_b32(t0, t1, 0x7632u);
  o[2] = prmt_b32(t2, t3, 0x5410u);
  o[3] = prmt_b32(t2, t3, 0x7632u);
}
LOKA_DEVINL uint32_t vmax_u16x2(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("max.u16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
// the same as two 16-bit partial maxima (halves of one word; the caller combines them)
LOKA_DEVINL uint32_t amax8_u16x2(uint4 w) {
  return vmax_u16x2(vmax_u16x2(w.x & 0x7FFF7FFFu, w.y & 0x7FFF7FFFu), vmax_u16x2(w.z & 0x7FFF7FFFu, w.w & 0x7FFF7FFFu));
}
template <int FMT>
LOKA_DEVINL uint2 cast8_row(uint4 w, float r) {
  float f[8] = {bf16lo_to_f32(w.x), bf16hi_to_f32(w.x), bf16lo_to_f32(w.y), bf16hi_to_f32(w.y),
                bf16lo_to_f32(w.z), bf16hi_to_f32(w.z), bf16lo_to_f32(w.w), bf16hi_to_f32(w.w)};
#pragma unroll
  for (int i = 0; i < 8; ++i) f[i] = __fmul_rn(f[i], r);
  return make_uint2(cvt_fp8x4<FMT>(f[0], f[1], f[2], f[3]), cvt_fp8x4<FMT>(f[4], f[5], f[6], f[7]));
}
template <int FMT>
LOKA_DEVINL uint2 cast8_col(uint4 w, const float (&r)[8]) {
  float f[8] = {bf16lo_to_f32(w.x), bf16hi_to_f32(w.x), bf16lo_to_f32(w.y), bf16hi_to_f32(w.y),
                bf16lo_to_f32(w.z), bf16hi_to_f32(w.z), bf16lo_to_f32(w.w), bf16hi_to_f32(w.w)};
#pragma unroll
  for (int i = 0; i < 8; ++i) f[i] = __fmul_rn(f[i], r[i]);
  return make_uint2(cvt_fp8x4<FMT>(f[0], f[1], f[2], f[3]), cvt_fp8x4<FMT>(f[4], f[5], f[6], f[7]));
}
// byte offset of (row, col) in the transpose's code tile (16-byte chunks XOR-swizzled by row / 8)
LOKA_DEVINL uint32_t tql_off(int row, int col) {
  return (uint32_t)row * 128u + ((((uint32_t)col >> 4) ^ (((uint32_t)row >> 3) & 7u)) << 4) + ((uint32_t)col & 15u);
}
// byte offset of (row, byte col) in a 128-row x 128-byte SW128 staging tile (the TMA store layout)
LOKA_DEVINL uint32_t sw128_off(int row, int col) {
  return (uint32_t)row * 128u + ((((uint32_t)col >> 4) ^ ((uint32_t)row & 7u)) << 4) + ((uint32_t)col & 15u);
}

// Tile t -> (row tile tr, column tile tc), row-major: the CTAs in flight read whole row bands.
// (Bands of 8 row tiles taken column tile by column tile for the transposed copy — 1 KB runs of each
// transposed row instead of 128-byte pieces — measured slower: 3.96 vs 4.46 TB/s for ROW + transpose
// at 262144 x 4096; kept switchable.)
constexpr bool kQlBandOrder = false;
template <bool QT>
LOKA_DEVINL void ql_tile(int64_t t, int nbc, int nbr, int& tr, int& tc) {
  if constexpr (!QT || !kQlBandOrder) {
    tr = (int)(t / nbc);
    tc = (int)(t % nbc);
  } else {
    const int64_t band = t / (8 * (int64_t)nbc);
    const int w = (int)(t - band * 8 * (int64_t)nbc);
    const int gsz = min(8, nbr - (int)band * 8);
    tc = w / gsz;
    tr = (int)band * 8 + w % gsz;
  }
}

// NG consumer groups: 2 (4 warps each, alternate tiles) or 1 (all 8 warps on every tile).  Two groups
// hide each other's barrier and reciprocal latencies — better when a CTA has few tiles (32768 x 4096:
// ~55); one group keeps more loads in flight per tile in the long steady state (262144 x 4096: ~440
// tiles per CTA, 8-10% faster there).  The launch picks by tiles per CTA.
template <int FMT, int SF, int GRAN, bool QT, int NG>
__global__ void __launch_bounds__(kQlThreads, 1) quant_tile_tma_kernel(const __grid_constant__ QuantTileParams P) {
  using L = QlLayout<QT>;
  constexpr int WG = 8 / NG;    // warps per group
  constexpr int TG = 32 * WG;   // threads per group
  constexpr int RW = 128 / WG;  // tile rows per warp (16 or 32): RW / 16 half-passes of 8 rows per lane
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const QuantParams& p = P.p;
  // full barriers per (consumer group, stage): with an odd stage count both groups use every stage,
  // and a group waiting on a shared barrier could see the parity of the OTHER group's pending fill
  // as its own completed phase; per-group barriers complete only for that group's tiles, in order
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + L::kOffBar);  // [2][kStages]
  uint64_t* empty_bar = full_bar + 2 * L::kStages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < L::kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&full_bar[L::kStages + s], 1);
      mbar_init(&empty_bar[s], WG);  // the consuming group's warps
    }
    fence_barrier_init();
  }
  __syncthreads();
  pdl_wait();
  pdl_launch_dependents();  // (the dependent's griddepcontrol.wait still waits for this grid)

  if (warp == 8) {  // ===== producer: the CTA's tiles k = 0, 1, ... in order =====
    if (lane == 0) {
      tma_prefetch_desc(&P.tx);
      int s = 0, k = 0;
      uint32_t ph = 0;
      for (int64_t t = blockIdx.x; t < P.ntiles; t += gridDim.x, ++k) {
        mbar_wait(&empty_bar[s], ph ^ 1u, 1);
        uint64_t* fb = &full_bar[(k % NG) * L::kStages + s];  // tile k goes to group k % NG
        mbar_arrive_expect_tx(fb, (uint32_t)kQlIn);
        int tr, tc;
        ql_tile<QT>(t, P.nbc, P.nbr, tr, tc);
        tma_load_2d(smem + s * kQlIn, &P.tx, fb, tc * 128, tr * 128);
        if (++s == L::kStages) s = 0, ph ^= 1u;
      }
    }
    return;
  }

  // ===== two consumer groups of 4 warps, each on every other tile of the CTA (k = g, g + 2, ...),
  // synchronising only among themselves (named barrier 1 + g): one group's barrier waits and
  // reciprocal latencies overlap the other's loads and casts.  Warp gw of a group owns tile rows
  // 32 gw .. 32 gw + 31: lane (hw, hl) row 32 gw + 2 i + hw of step i (0..15), columns 8 hl .. 8 hl + 7.
  constexpr bool kDual = GRAN == kGranDualT;
  constexpr bool kRowBlk = GRAN == LOKA_GRAN_BLK_1x128 || kDual;       // half-warp granules
  constexpr bool kColRed = GRAN == LOKA_GRAN_BLK_128x1 || GRAN == LOKA_GRAN_BLK_128x128 || kDual;
  constexpr bool kColwise = GRAN == LOKA_GRAN_BLK_128x1 || GRAN == LOKA_GRAN_COL;  // q's r per column
  const int g = warp / WG, gw = warp % WG, gt = threadIdx.x % TG;
  const uint32_t bar_id = 1u + (uint32_t)g;
  const int hl = lane & 15, hw = lane >> 4, cl = hl * 8;
  const uint32_t red = smem_u32(smem + L::kOffRed) + (uint32_t)g * 2048u;  // [WG][128] per group
  const uint32_t rb = smem_u32(smem + L::kOffR) + (uint32_t)g * 512u;
  const uint32_t red2 = smem_u32(smem + L::kOffRed2) + (uint32_t)g * 16u;
  const uint32_t tq = smem_u32(smem + L::kOffTQ) + (uint32_t)g * 16384u;
  const bool want_q = p.q != nullptr;
  float r_tensor = 1.f;
  if constexpr (GRAN == LOKA_GRAN_TENSOR) {  // from the pre-pass amax word
    float s_t;
    scales_from_amax<FMT, SF>(__uint_as_float(P.amax_g[0]), s_t, r_tensor);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      if (p.scales) p.scales[0] = s_t;
      if (p.scales_t) p.scales_t[0] = s_t;
    }
  }
  for (int64_t k = g;; k += NG) {
    const int64_t t = blockIdx.x + k * (int64_t)gridDim.x;
    if (t >= P.ntiles) break;
    const int s = (int)(k % L::kStages);
    constexpr int kPeriod = (NG == 2 && L::kStages % 2) ? 2 * L::kStages : L::kStages;  // lcm(stages, NG)
    const uint32_t ph = (uint32_t)((k / kPeriod) & 1);  // this group's earlier fills of its barrier
    int tr, tc;
    ql_tile<QT>(t, P.nbc, P.nbr, tr, tc);
    const int64_t c0 = (int64_t)tc * 128, r0 = (int64_t)tr * 128;
    if (lane == 0) mbar_wait(&full_bar[g * L::kStages + s], ph, 2);
    __syncwarp();
    const uint32_t src = smem_u32(smem + s * kQlIn) + (uint32_t)(gw * RW + hw) * 256u + (uint32_t)hl * 16u;
    // staging tiles: one per group (NG = 2), or double-buffered for the single group (NG = 1)
    const int sbuf = NG == 2 ? g : (int)(k & 1);
    const uint32_t sq = smem_u32(smem + L::kOffQ) + (uint32_t)sbuf * 16384u;
    const uint32_t sqt = smem_u32(smem + L::kOffQT) + (uint32_t)sbuf * 16384u;
    // ---- column-like granules: per-column partial max of this warp's 32 rows ----
    if constexpr (kColRed) {
      // columns (2j, 2j+1) share a word: 16-bit |x| maxima, two per max.u16x2
      uint32_t pk[4] = {0u, 0u, 0u, 0u};
#pragma unroll
      for (int i = 0; i < RW / 2; ++i) {
        const uint4 w = lds_u4(src + (uint32_t)i * 512u);
        pk[0] = vmax_u16x2(pk[0], w.x & 0x7FFF7FFFu);
        pk[1] = vmax_u16x2(pk[1], w.y & 0x7FFF7FFFu);
        pk[2] = vmax_u16x2(pk[2], w.z & 0x7FFF7FFFu);
        pk[3] = vmax_u16x2(pk[3], w.w & 0x7FFF7FFFu);
      }
      uint32_t cm[8];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        pk[j] = vmax_u16x2(pk[j], __shfl_xor_sync(0xFFFFFFFFu, pk[j], 16));
        cm[2 * j] = pk[j] << 16;
        cm[2 * j + 1] = pk[j] & 0xFFFF0000u;
      }
      if (lane < 16) {
        const uint32_t a = red + (uint32_t)(gw * 128 + cl) * 4u;
        sts_u4(a, make_uint4(cm[0], cm[1], cm[2], cm[3]));
        sts_u4(a + 16u, make_uint4(cm[4], cm[5], cm[6], cm[7]));
      }
      named_bar_sync(bar_id, TG);  // (A) partials complete
    }
    if constexpr (GRAN == LOKA_GRAN_BLK_128x1 || kDual) {  // thread gt finalises column c0 + gt
     if (gt < 128) {
      uint32_t m = 0;
#pragma unroll
      for (int w = 0; w < WG; ++w) m = max(m, lds_u32(red + (uint32_t)(w * 128 + gt) * 4u));
      float sc, r;
      scales_from_amax<FMT, SF>(__uint_as_float(m), sc, r);
      asm volatile("st.shared.f32 [%0], %1;" ::"r"(rb + (uint32_t)gt * 4u), "f"(r) : "memory");
      const int64_t cc = c0 + gt;
      if (cc < p.cols) {
        if (m >= 0x7F800000u && p.status) atomicOr(p.status, LOKA_DEVSTATUS_NONFINITE);
        if (!kDual && p.scales) p.scales[(int64_t)tr * p.cols + cc] = sc;  // [nbr, cols]
        if (p.scales_t) p.scales_t[cc * P.nbr + tr] = sc;                   // t-frame 1x128 [cols, nbr]
      }
     }
    } else if constexpr (GRAN == LOKA_GRAN_BLK_128x128) {
      if (gt < 128) {  // warps gw = 0..3 each reduce 32 columns
        uint32_t m = 0;
#pragma unroll
        for (int w = 0; w < WG; ++w) m = max(m, lds_u32(red + (uint32_t)(w * 128 + gt) * 4u));
        m = warp_max_u32(m);
        if (lane == 0) asm volatile("st.shared.u32 [%0], %1;" ::"r"(red2 + (uint32_t)gw * 4u), "r"(m) : "memory");
      }
    } else if constexpr (GRAN == LOKA_GRAN_ROW || GRAN == LOKA_GRAN_COL) {  // from the pre-pass array
     if (gt < 128) {
      const bool row_g = GRAN == LOKA_GRAN_ROW;
      const int64_t idx = (row_g ? r0 : c0) + gt;
      const bool ok = idx < (row_g ? p.rows : p.cols);
      float sc, r;
      scales_from_amax<FMT, SF>(__uint_as_float(ok ? P.amax_g[idx] : 0u), sc, r);
      asm volatile("st.shared.f32 [%0], %1;" ::"r"(rb + (uint32_t)gt * 4u), "f"(r) : "memory");
      if (ok && (row_g ? tc : tr) == 0) {
        if (p.scales) p.scales[idx] = sc;
        if (p.scales_t) p.scales_t[idx] = sc;
      }
     }
    }
    // (B) the group's staging tiles free (its store thread waits for the previous stores' reads
    // here) and this tile's per-row / per-column r ready
    if (gt == 0) {
      if constexpr (NG == 2) bulk_wait_read0();
      else bulk_wait_read_le1();  // (double-buffered staging)
    }
    named_bar_sync(bar_id, TG);
    float rcol[8];
    if constexpr (kColwise || kDual) {
      const float4 a = lds_f4(rb + (uint32_t)cl * 4u), b = lds_f4(rb + (uint32_t)cl * 4u + 16u);
      rcol[0] = a.x; rcol[1] = a.y; rcol[2] = a.z; rcol[3] = a.w;
      rcol[4] = b.x; rcol[5] = b.y; rcol[6] = b.z; rcol[7] = b.w;
    }
    float r_blk = r_tensor;
    if constexpr (GRAN == LOKA_GRAN_BLK_128x128) {
      const uint32_t m = max(max(lds_u32(red2), lds_u32(red2 + 4u)), max(lds_u32(red2 + 8u), lds_u32(red2 + 12u)));
      float sc;
      scales_from_amax<FMT, SF>(__uint_as_float(m), sc, r_blk);
      if (gt == 0) {
        if (m >= 0x7F800000u && p.status) atomicOr(p.status, LOKA_DEVSTATUS_NONFINITE);
        if (p.scales) p.scales[(int64_t)tr * P.nbc + tc] = sc;
        if (p.scales_t) p.scales_t[(int64_t)tc * P.nbr + tr] = sc;
      }
    }
    // ---- two half-passes of 8 rows: load, (1x128) reduce, cast into the staging tiles (a lane's
    // 16 rows at once measured slower: 168 registers, and no gain from the earlier stage release) ----
#pragma unroll 1
    for (int h = 0; h < RW / 16; ++h) {
      uint4 vh[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) vh[i] = lds_u4(src + (uint32_t)(8 * h + i) * 512u);
      if (h == RW / 16 - 1) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty_bar[s]);  // the group's last read of the stage
      }
      float rrow[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) rrow[i] = r_blk;
      if constexpr (kRowBlk) {
        // two rows' 16-bit |x| maxima per word (rows 2j, 2j+1 in the low / high half): half the shuffles
        uint32_t m[8];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t a = amax8_u16x2(vh[2 * j]), b = amax8_u16x2(vh[2 * j + 1]);
          uint32_t pk = vmax_u16x2(prmt_b32(a, b, 0x5410u), prmt_b32(a, b, 0x7632u));
#pragma unroll
          for (int o = 8; o >= 1; o >>= 1) pk = vmax_u16x2(pk, __shfl_xor_sync(0xFFFFFFFFu, pk, o));
          m[2 * j] = pk << 16;
          m[2 * j + 1] = pk & 0xFFFF0000u;
        }
        // lane (hw, j), j = lane & 7, divides for step j's row (a select tree: a loop of predicated
        // selects is turned into a dynamically indexed local array)
        const bool b0 = lane & 1, b1 = lane & 2, b2 = lane & 4;
        const uint32_t x0 = b0 ? m[1] : m[0], x1 = b0 ? m[3] : m[2], x2 = b0 ? m[5] : m[4], x3 = b0 ? m[7] : m[6];
        const uint32_t mine = b2 ? (b1 ? x3 : x2) : (b1 ? x1 : x0);
        float sc, r;
        scales_from_amax<FMT, SF>(__uint_as_float(mine), sc, r);
        const int64_t row = r0 + gw * RW + 2 * (8 * h + (lane & 7)) + hw;
        if ((lane & 8) == 0 && row < p.rows) {
          if (mine >= 0x7F800000u && p.status) atomicOr(p.status, LOKA_DEVSTATUS_NONFINITE);
          if (p.scales) p.scales[row * P.nbc + tc] = sc;
          if (!kDual && p.scales_t) p.scales_t[(int64_t)tc * p.rows + row] = sc;  // t-frame 128x1 [nbc, rows]
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) rrow[i] = __shfl_sync(0xFFFFFFFFu, r, (lane & 16) + i);
      }
      if constexpr (GRAN == LOKA_GRAN_ROW) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          float r;
          asm volatile("ld.shared.f32 %0, [%1];" : "=f"(r) : "r"(rb + (uint32_t)(gw * RW + 2 * (8 * h + i) + hw) * 4u));
          rrow[i] = r;
        }
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int lr = gw * RW + 2 * (8 * h + i) + hw;
        const uint2 code = kColwise ? cast8_col<FMT>(vh[i], rcol) : cast8_row<FMT>(vh[i], rrow[i]);
        if (want_q) sts_u2(sq + sw128_off(lr, cl), code.x, code.y);
        if constexpr (QT) {
          const uint2 ct = kDual ? cast8_col<FMT>(vh[i], rcol) : code;  // dual: x's 128x1 quantization
          sts_u2(tq + tql_off(lr, cl), ct.x, ct.y);
        }
      }
    }
    if constexpr (QT) {
      named_bar_sync(bar_id, TG);  // (C) the code tile is complete
#pragma unroll
      for (int u = 0; u < 512 / TG; ++u) {
        const int item = gt + TG * u;
        const int rg = item & 15, cg = item >> 4;  // rows 8rg .. 8rg+7, columns 4cg .. 4cg+3
        uint32_t w[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) w[i] = lds_u32(tq + tql_off(8 * rg + i, 4 * cg));
        uint32_t lo[4], hi[4];
        tr4x4(w[0], w[1], w[2], w[3], lo);
        tr4x4(w[4], w[5], w[6], w[7], hi);
#pragma unroll
        for (int j = 0; j < 4; ++j) sts_u2(sqt + sw128_off(4 * cg + j, 8 * rg), lo[j], hi[j]);
      }
    }
    fence_proxy_async_smem();     // staging writes -> the TMA stores
    named_bar_sync(bar_id, TG);  // (D) staging complete (and, with QT, the code tile's reads done)
    if (gt == 0) {
      if (want_q) tma_store_2d(&P.tq, smem + L::kOffQ + sbuf * 16384, (int32_t)c0, (int32_t)r0);
      if constexpr (QT) tma_store_2d(&P.tqt, smem + L::kOffQT + sbuf * 16384, (int32_t)r0, (int32_t)c0);
      bulk_commit();
    }
  }
  if (gt == 0) bulk_wait0();
}

bool quant_tile_tma_eligible(int gran) {
  static const bool off = [] {
    const char* e = std::getenv("LOKA_QUANT_TILE");
    return e && e[0] == '0';
  }();
  if (off) return false;
  // (TENSOR + transpose stays on quantize_t.cu's kernel: 3 CTAs per SM with no reduction state
  // measured faster there, 4.28 vs 3.80 TB/s at 262144 x 4096)
  return gran == LOKA_GRAN_BLK_1x128 || gran == LOKA_GRAN_BLK_128x1 || gran == LOKA_GRAN_BLK_128x128 ||
         gran == LOKA_GRAN_ROW || gran == LOKA_GRAN_COL || gran == kGranDualT;
}

template <int FMT, int SF, int GRAN, bool QT>
static cudaError_t launch_ql(const QuantTileParams& tp, int num_sms, cudaStream_t st) {
  // two consumer groups when each CTA gets few tiles; one in the long steady state for the granules
  // measured faster that way at 262144 x 4096 (~440 tiles per CTA): 1x128 5.91 vs 5.53, 128x128 6.29
  // vs 5.90, 128x1 + transpose 5.71 vs 4.97 TB/s — while 128x1 (5.52 vs 5.82) and ROW + transpose
  // (3.59 vs 4.46) stay faster with two (profiles/r02ai_quantize_262k_groups.json)
  constexpr bool kOneWhenLong = GRAN == LOKA_GRAN_BLK_1x128 || GRAN == LOKA_GRAN_BLK_128x128 ||
                                (GRAN == LOKA_GRAN_BLK_128x1 && QT);
  bool two = !kOneWhenLong || tp.ntiles <= (int64_t)num_sms * 128;
  if (const char* e = std::getenv("LOKA_QUANT_GROUPS")) two = e[0] != '1';  // (tests / A-B: 1 or 2)
  auto kern = two ? quant_tile_tma_kernel<FMT, SF, GRAN, QT, 2> : quant_tile_tma_kernel<FMT, SF, GRAN, QT, 1>;
  constexpr int smem = QlLayout<QT>::kSmem;
  cudaError_t e = ensure_func_attrs(reinterpret_cast<const void*>(kern), smem);
  if (e != cudaSuccess) return e;
  if (tp.ntiles == 0) return cudaSuccess;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(tp.ntiles < num_sms ? tp.ntiles : num_sms));
  cfg.blockDim = dim3(kQlThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  note_launch();
  return cudaLaunchKernelEx(&cfg, kern, tp);
}

cudaError_t launch_quant_tile_tma(const QuantTileParams& tp, int fmt, int scale_fmt, int gran, int num_sms,
                                  cudaStream_t st) {
#define LOKA_QL(F, S, G)                                                          \
  if (fmt == F && scale_fmt == S && gran == G)                                    \
    return tp.p.qt ? launch_ql<F, S, G, true>(tp, num_sms, st) : launch_ql<F, S, G, false>(tp, num_sms, st);
#define LOKA_QL_G(F, S)                  \
  LOKA_QL(F, S, LOKA_GRAN_TENSOR)        \
  LOKA_QL(F, S, LOKA_GRAN_ROW)           \
  LOKA_QL(F, S, LOKA_GRAN_COL)           \
  LOKA_QL(F, S, LOKA_GRAN_BLK_1x128)     \
  LOKA_QL(F, S, LOKA_GRAN_BLK_128x1)     \
  LOKA_QL(F, S, LOKA_GRAN_BLK_128x128)   \
  LOKA_QL(F, S, kGranDualT)
  LOKA_QL_G(LOKA_E4M3, LOKA_SCALE_F32)
  LOKA_QL_G(LOKA_E4M3, LOKA_SCALE_UE8M0)
  LOKA_QL_G(LOKA_E5M2, LOKA_SCALE_F32)
  LOKA_QL_G(LOKA_E5M2, LOKA_SCALE_UE8M0)
#undef LOKA_QL_G
#undef LOKA_QL
  return cudaErrorNotSupported;
}

}  // namespace loka
