// launch.h — internal (non-ABI) launch interfaces between api.cu and the kernel files.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

namespace loka {

void note_launch(int n = 1);
// set a kernel's max dynamic smem (and optionally non-portable cluster size) once per (function,
// device), thread-safe (attrs.cu)
cudaError_t ensure_func_attrs(const void* func, int smem_bytes, bool nonportable_cluster = false);
long long debug_hang_info(unsigned long long* info, int reset);
long long debug_trace(int enable, unsigned long long* out, long long n);  // process-wide launch counter (loka_launch_count)

struct QuantParams {
  const void* x;
  int64_t rows, cols, ldx;
  uint8_t* q;        // nullable
  int64_t ldq;
  float* scales;     // scales in x's frame (nullable when only the transposed copy is wanted)
  uint8_t* qt;       // nullable transposed codes [cols, rows]
  int64_t ldqt;
  float* scales_t;   // nullable scales in the transposed frame
  int32_t* status;
};

// ---- NVFP4 (nvfp4.cu, NEXT-4) ----
struct Nvfp4QParams {
  const void* x;
  int64_t rows, cols, ldx;  // cols % 16 == 0
  uint8_t* q;               // packed E2M1 codes [rows, cols/2], ldq bytes
  int64_t ldq;
  uint8_t* sf;              // E4M3 block-scale codes [rows, cols/16], ld_sf
  int64_t ld_sf;
  const float* amax;        // device: the tensor amax
  float* s_tensor;          // device: s_t out (nullable)
};
cudaError_t launch_nvfp4_cast(const Nvfp4QParams& p, bool in_bf16, int num_sms, cudaStream_t st);
cudaError_t launch_nvfp4_sf_pack(const uint8_t* sf, int64_t ld, int64_t rows, int64_t nblk, int64_t row_blocks,
                                 int64_t k64, uint8_t* out, cudaStream_t st);

// ---- quantized DP gradient reduction (gradcomm.cu, NEXT-4) ----
constexpr int kMaxRanks = 8;
struct DeqReduceParams {
  const uint8_t* codes[kMaxRanks];  // per rank: FP8 codes of the shard rows (may be peer memory)
  const float* scales[kMaxRanks];   // per rank: row scales of the shard rows
  int32_t P, fmt;
  int64_t rows, cols, ld;           // cols % 16 == 0, ld % 16 == 0 (bytes = elements)
  float* out;
  int64_t ld_out;
};
cudaError_t launch_dequant_reduce(const DeqReduceParams& p, int num_sms, cudaStream_t st);

cudaError_t launch_quantize(const QuantParams& p, bool in_bf16, int fmt, int scale_fmt, int gran, int phase,
                            float* amax_dev, cudaStream_t st, int num_sms);

// Streaming quantize through smem with bulk copies (quantize_tma.cu): ROW / TENSOR
// cast (amax_dev = the tensor amax), bf16 input, no transposed copy; see quant_tma_eligible.
bool quant_tma_eligible(const QuantParams& p, bool in_bf16, int gran);
// amax_next (nullable, TENSOR only): also atomicMax the tensor's own max |x| bits into it (delayed scaling)
cudaError_t launch_quantize_tma(const QuantParams& p, int fmt, int scale_fmt, int gran, const float* amax_dev,
                                int num_sms, cudaStream_t st, uint32_t* amax_next = nullptr);
struct QuantGroup;
cudaError_t launch_quantize_tma_group(const QuantGroup& grp, int64_t max_cols, int fmt, int scale_fmt, int gran,
                                      const float* amax_dev, int num_sms, cudaStream_t st,
                                      uint32_t* amax_next = nullptr);

// Streaming tile quantize (quantize_tile.cu, bf16 input): maps built by api.cu — tx over x
// [rows, cols] bf16 box {128, 128} no swizzle; tq over q [rows, cols] u8 and tqt over qt
// [cols, rows] u8, box {128, 128} SW128 (unused maps when q / qt are null).
struct QuantTileParams {
  CUtensorMap tx, tq, tqt;
  QuantParams p;
  const uint32_t* amax_g;  // TENSOR: [1] amax bits; ROW / COL: the pre-pass array; else null
  int64_t ntiles;          // nbr * nbc
  int nbc, nbr;            // 128-wide column / row tiles
};
bool quant_tile_tma_eligible(int gran);
cudaError_t launch_quant_tile_tma(const QuantTileParams& tp, int fmt, int scale_fmt, int gran, int num_sms,
                                  cudaStream_t st);

// Tiled quantize (quantize_t.cu): any granularity incl. COL / BLK_128x1, optional transposed
// copy; ws holds the ROW / COL amax pre-pass array (4 * max(rows, cols) bytes).  tile (nullable,
// bf16 input only): the streaming kernel's maps — the tile pass then runs in quantize_tile.cu.
cudaError_t launch_quantize_tiled(const QuantParams& p, bool in_bf16, int fmt, int scale_fmt, int gran, int phase,
                                  float* amax_dev, void* ws, cudaStream_t st, QuantTileParams* tile = nullptr,
                                  int num_sms = 148);

constexpr int kMaxQuantGroup = 64;
struct QuantGroup {
  int32_t G;
  int64_t row_start[kMaxQuantGroup + 1];  // prefix sum of rows
  QuantParams p[kMaxQuantGroup];
};
// ROW granularity, every tensor the same input dtype / FP8 format / scale format.
cudaError_t launch_quantize_grouped(const QuantGroup& grp, bool in_bf16, int fmt, int scale_fmt, int64_t max_cols,
                                    cudaStream_t st);

struct LinearParams {
  int32_t M, N, K;
  int32_t a_fmt, b_fmt;          // 0 = e4m3, 1 = e5m2 (tcgen05 kind::f8f6f4 encoding)
  const float* sa; int32_t sa_row;  // per-row (1) or tensor (0) scale of A
  const float* sb; int32_t sb_row;  // per-row of B (= per output column n) or tensor
  const void* bias; int32_t bias_bf16;
  const float* gamma;
  const float* beta;
  float eps;
  int32_t norm, norm_block;
  int32_t out_dtype;             // loka_dtype
  void* y; int64_t ldy;
  float* y_scales;               // ROW scales of an FP8 output
  float* precast; int64_t ld_pre;
  int32_t* status;
  int32_t cluster_n;             // CTAs per cluster along N (1 = no cross-CTA row exchange)
  int32_t act;                   // loka_act, applied after the norm (and gamma / beta)
  // NEXT-1 norm backward (bwd): the accumulator is dL/dh of a forward h = act(norm(z)*gamma+beta)
  // whose saved xhat (bf16 [M, N], ld_xhat) and rstd (rstd_in: [M], BLOCK_RMS [M, N/block]) are
  // given; the epilogue emits dL/dz.  Forward saves (nullable): save_xhat (bf16) / save_rstd.
  int32_t bwd;
  const __nv_bfloat16* xhat; int64_t ld_xhat;
  const float* rstd_in;
  __nv_bfloat16* save_xhat; int64_t ld_save_xhat;
  float* save_rstd;
  float* amax_out;               // NEXT-4: atomicMax of |stored y| (bit pattern), nullable
  // native block-scaled mode: 1 = MX (UE8M0 blockwise scales applied by the tensor core; sa/sb
  // unused), 2 = NVFP4 (E4M3 block scales by the tensor core; sa/sb = the FP32 tensor scales;
  // K counts bytes of packed E2M1 codes; atoms [row blocks][sf_kblocks][4][512])
  int32_t mx;
  const uint8_t* sfa_pack;       // [ceil(M/128)][kblocks][512] (sfpack.cu layout)
  const uint8_t* sfb_pack;       // [ceil(N/256)*2][kblocks][512]
  int32_t sf_kblocks;            // ceil(K/128)
};

// ---- UE8M0 scale packing for the MX mode (sfpack.cu) ----
struct SfPackSeg {
  const float* scales;  // FP32 powers of two, [rows / row_div, ld] row-major
  int64_t ld;
  int64_t rows;         // operand rows
  int32_t row_div;      // 1 (1x128 scales) or 128 (128x128 scales)
  int32_t row_blocks;   // 128-row atoms to write (>= ceil(rows/128))
  uint8_t* out;         // [row_blocks][kblocks][512]
  int32_t k32;          // 1: MX 1x32 scales (one per 32-wide K block, [rows, ld = ceil(K/32)])
};
struct SfPackParams {
  SfPackSeg seg[2];
  int32_t kblocks;
};
cudaError_t launch_sf_pack(const SfPackParams& p, cudaStream_t st);

// Launch one linear+norm problem.  tma_a/tma_b are 2D maps over the FP8 operands with box
// {128 (K), 128 (A rows)} and {128 (K), bn (B rows)}, 128B swizzle.
// tma_y: 2D map over the output [M, N] (element type of y), box {128 bytes, 128 rows}, SW128.
cudaError_t launch_linear(const CUtensorMap& tma_a, const CUtensorMap& tma_b, const CUtensorMap& tma_y,
                          const LinearParams& p, int bn, cudaStream_t st);

// ---- fused layer stack (stack.cu) ----
constexpr int kMaxStackLayers = 8;
struct StackParams {
  CUtensorMap tx;                    // X codes [M, K0], box {128, 128}
  CUtensorMap tw[kMaxStackLayers];   // W_l codes [N_l, K_l], box {128, min(BN_l, 128)}
  CUtensorMap ty;                    // output [M, N_last], box {min(128, BN*e) bytes, 128}
  const float* xs;                   // X row scales
  const float* ws[kMaxStackLayers];  // W_l row scales (per output column)
  int32_t L, M, C;
  int32_t K[kMaxStackLayers], N[kMaxStackLayers], BN[kMaxStackLayers];
  int32_t norm[kMaxStackLayers];
  float eps[kMaxStackLayers];
  int32_t out_dtype;
  float* y_scales;
  int32_t* status;
  // hand-off h_{l+1} codes in global memory [M, N_l] (ld h_ld): the caller's saved copy or the
  // workspace; required where the cluster all-gathers through L2 (C > 1, BN_l >= 128), else nullable
  uint8_t* h_save[kMaxStackLayers];
  int32_t h_ld[kMaxStackLayers];
  float* hs_save[kMaxStackLayers];    // nullable: its row scales [M]
  CUtensorMap th[kMaxStackLayers];    // map over h_save[l], box {128, 128}, SW128 (multicast loads)
  int32_t gather;                     // all-gather transport: kStackGather* (stack.cu)
  float* precast[kMaxStackLayers];    // tests: FP32 [M, N_l] pre-cast values (debug instance only)
};
constexpr int kStackGatherDsmemBulk = 0, kStackGatherL2 = 1, kStackGatherStAsync = 2;
// L2 for slices of whole K blocks (BN >= 128), st.async pieces on the receiver's barrier for
// narrower slices (instead of per-thread DSMEM stores + a cluster barrier)
constexpr int kStackGatherL2StAsync = 3;
constexpr int kStackGatherL2StAsync256 = 4;  // the same split at BN = 256 (measurement variant)
cudaError_t launch_stack(const StackParams& p, cudaStream_t st);
long long stack_debug_trace(int enable, unsigned long long* out, long long n);  // see loka_debug_trace

// ---- blockwise-scaled GEMM with FP32 promotion (blockwise.cu) ----
struct BwParams {
  int32_t M, N, K;
  int32_t a_fmt, b_fmt;
  const float* sa; int32_t sa_ld;   // A: 1x128 scales [M, ceil(K/128)]
  const float* sb; int32_t sb_ld;   // B: 128x128 [ceil(N/128), ceil(K/128)] or 1x128 [N, ceil(K/128)]
  int32_t sb_rows;                  // 1: B scales are 1x128 (per row of B)
  const void* bias; int32_t bias_bf16;
  int32_t out_dtype;
  float* y_scales;                  // FP8 output ROW scales (N <= 128)
  float* precast; int64_t ld_pre;
};
cudaError_t launch_linear_bw(const CUtensorMap& tma_a, const CUtensorMap& tma_b, const CUtensorMap& tma_y,
                             const BwParams& p, cudaStream_t st);

// ---- grouped persistent launch (grouped.cu) ----
constexpr int kMaxGroups = 64;  // per launch (kernel-parameter space: 3 tensor maps per group, ~30.8 KB of the 32 KB)
struct GroupDesc {
  int32_t M, N, K, tiles_n;
  int32_t a_fmt, b_fmt;
  const float* sa; int32_t sa_row;
  const float* sb; int32_t sb_row;
  const void* bias; int32_t bias_bf16;
  int32_t out_dtype;
  // split-K (CTA-pair engine only): ksplit slices of kb_per_split 128-K blocks; each writes its raw
  // FP32 accumulator to the [ksplit][M][N] partial buffer (map tp), reduced by splitk_reduce
  int32_t ksplit, kb_per_split;
  float* amax_out;  // NEXT-4: atomicMax of |stored y| (bit pattern), nullable
};
struct GroupedParams {
  CUtensorMap ta[kMaxGroups], tb[kMaxGroups], ty[kMaxGroups];  // A box {128,128}, B box {128,128}, Y out
  CUtensorMap tp[1];  // split-K partials [ksplit*M, N] f32 (split-K is for lone problems: G == 1)
  GroupDesc g[kMaxGroups];
  int32_t G;
  int32_t tile_start[kMaxGroups + 1];  // prefix sum of 128x128 tiles
  int32_t wide;                        // CTA-pair engine: 256 x 512 tiles (tiles_n = ceil(N/512))
};
cudaError_t launch_grouped(const GroupedParams& gp, int num_sms, cudaStream_t st);
// CTA-pair variant (gemm2.cu): tiles 256 x 256 (tiles_n = ceil(N/256), tile_start counts them);
// ta/tb boxes {128, 128}; ty box {128 bytes, 32 rows}, SW128; bf16 / f32 output.
cudaError_t launch_grouped2(const GroupedParams& gp, int num_sms, cudaStream_t st);
// the same engine on BF16 operands (K-major, 64 elements per stage row): FP32 C = A . B^T (sa = sb =
// pointers to 1.0f, tensor scales), bf16 / f32 output
cudaError_t launch_grouped2_bf16(const GroupedParams& gp, int num_sms, cudaStream_t st);

// ---- NEXT-2 input tracker (track.cu): batched Welford merge of one bf16 batch X [B, K] ----
struct TrackParams {
  const __nv_bfloat16* x; int64_t ldx;
  int64_t B, K;
  float* mean;             // [K] tracked mean (updated in place)
  float* scatter;          // [K, K] tracked unnormalised scatter (updated in place)
  int64_t n_old;
  float* colpart;          // ws [nchunk][K] column partial sums
  float* delta;            // ws [K]
  float* one;              // ws [1] = 1.0f (GEMM tensor scales)
  __nv_bfloat16* xct;      // ws [K, ldxct] centred transpose
  int64_t ldxct;
  float* sb;               // ws [K, K] batch scatter
  int32_t nchunk;
};
cudaError_t launch_track_prep(const TrackParams& p, cudaStream_t st);   // column means, delta, mean update, Xc^T
cudaError_t launch_track_merge(const TrackParams& p, cudaStream_t st);  // scatter += S_b + c delta delta^T
cudaError_t launch_track_cov(const float* scatter, float* out, int64_t K, int64_t n, cudaStream_t st);
// Native block-scaled (UE8M0 blockwise, MX) problem on the CTA pair (gemm2.cu): 256 x 256 tiles,
// kind::mxf8f6f4.block_scale with cta_group::2; scale atoms TMA-loaded from the sfpack layout
// viewed as rows of 256 B (maps tsa / tsb, box {256, 2} = one 512 B atom).  Plain epilogue
// (+ bias), bf16 / f32 output.
struct MxPairParams {
  CUtensorMap ta, tb, ty, tsa, tsb;
  GroupDesc d;     // sa / sb unused (the MMA applies the scales); NVFP4: the tensor scales [1]
  int32_t sf_kbs;  // 128-byte K stages (MX: one atom, NVFP4: four atoms per operand row block)
  int32_t tiles;
  int32_t nvfp4;   // 1: E2M1 operands (K counts bytes), kind::mxf4nvf4 scale_vec::4X
};
cudaError_t launch_mx_pair(const MxPairParams& mp, int num_sms, cudaStream_t st);
// Row-wise norm / act / cast over an FP32 GEMM output (rownorm.cu; the unfused form for wide rows)
struct RowNormParams {
  const float* y32; int64_t ld32;
  int64_t M, N;
  int32_t norm, act, out_dtype;
  float eps;
  const float* gamma; const float* beta;
  void* y; int64_t ldy;
  float* y_scales;
  float* precast; int64_t ld_pre;
  int32_t* status;
  // NEXT-1 backward mode (bwd): y32 holds dL/dh; xhat / rstd_in are the forward's saves
  int32_t bwd, block;
  const __nv_bfloat16* xhat; int64_t ld_xhat;
  const float* rstd_in;
  float* amax_out;  // NEXT-4, nullable
};
cudaError_t launch_rownorm(const RowNormParams& p, int num_sms, cudaStream_t st);
// y[m,n] = (sum_s part[s][m][n]) * s_a[m] * s_b[n] (+ bias[n]) -> y (bf16 / f32)
cudaError_t launch_splitk_reduce(const GroupDesc& d, const float* part, void* y, int64_t ldy, cudaStream_t st);

struct ProbeLayer {
  const void* out; const void* ref;
  int32_t out_bf16, ref_bf16;
  int64_t M, N, ld_out, ld_ref;
  int32_t out_vec, ref_vec;  // rows 16B-aligned: vector loads allowed
};
// gsum (nullable, device [L][2]): the global (sum |ref|, count) of each layer for the floor
cudaError_t launch_probe(const ProbeLayer* layers_dev, int L, int64_t max_elems, double floor_rel,
                         void* stats_dev, double* partials, int nblk, cudaStream_t st, const double* gsum = nullptr);

// ---- NEXT-3 (linalg.cu): FP32 linear algebra for the matrix-normal tracker and the sampling ----
struct GemmF32Params {  // C = alpha op(A) op(B) + beta Cin + bias[n]  (see linalg.cu)
  int64_t M, N, K;
  const float* A; int64_t lda;
  const float* B; int64_t ldb;
  const float* Cin; int64_t ldcin;
  void* C; int64_t ldc;
  int32_t c_bf16;
  const float* bias;
  float alpha, beta;
  int32_t tri_a, tri_b, lower_only;
};
cudaError_t launch_gemm_f32(const GemmF32Params& p, bool at, bool bt, cudaStream_t st);
cudaError_t launch_cholesky(float* a, int64_t lda, int64_t n, int32_t* status, cudaStream_t st);
cudaError_t launch_trsm_left(const float* l, int64_t ldl, int64_t n, float* b, int64_t ldb, int64_t ncols,
                             cudaStream_t st);
cudaError_t launch_trace2(const float* a, int64_t na, int64_t lda, const float* b, int64_t nb, int64_t ldb,
                          double* tr, cudaStream_t st);
cudaError_t launch_jitter_copy(const float* a, int64_t lda, float* l, int64_t ldl, int64_t n, float scale,
                               float eps_host, const double* tr_dev, double tr_scale, float eps_rel, cudaStream_t st);
cudaError_t launch_philox_normal(uint64_t seed, uint64_t offset, int64_t n, float* out, cudaStream_t st);
struct MatnormParams {
  const void* w; int32_t w_bf16; int64_t ldw;
  int64_t M, N;
  float m, eps_rel;
  float *mean, *u, *v;              // state (updated in place)
  float *wc, *wct, *lu, *lv, *u1, *v1;  // workspace
  double* tr;                        // [4]
  int32_t* status;                   // nullable: bit 0 = a Cholesky pivot was not positive
};
cudaError_t launch_matnorm_init(const void* w, bool bf16, int64_t ldw, float* mean, float* u, int64_t mm, float* v,
                                int64_t nn, cudaStream_t st);
cudaError_t launch_matnorm_update(const MatnormParams& p, cudaStream_t st);

// ---- a4 + a5 at scale: CTA-pair GEMM with the norm fused in the epilogue (pairnorm.cu) ----
constexpr int kPnMaxPairs = 128;  // CTA pairs per launch (148 SMs -> 74)
// workspace of the Case 2 row-record exchange: float4 records [row_blocks][tiles_n][2][128], filled
// with 0xFF bytes (a sentinel NaN) by the host before each launch
size_t pair_xchg_bytes(int64_t row_blocks, int tiles_n);
struct PairNormParams {
  CUtensorMap ta, tb, ty;  // A [M,K] / B [N,K] codes box {128, 128}; Y box {128 bytes, 32 rows} SW128
  int32_t M, N, K;
  int32_t a_fmt, b_fmt;
  const float* sa; int32_t sa_row;
  const float* sb; int32_t sb_row;
  const void* bias; int32_t bias_bf16;
  const float* gamma; const float* beta;  // nullable (FP8 output: both null)
  float eps;
  int32_t norm;       // LAYER, RMS, BLOCK_RMS (block 256, N % 256 == 0)
  int32_t act;        // loka_act (bf16 / f32 output)
  int32_t out_dtype;  // f32, bf16, e4m3, e5m2 (+ ROW scales y_scales)
  float* y_scales;
  int32_t y_blk;      // FP8 output scales: 0 = ROW [M]; 1 = BLK_1x128 [M, ceil(N/128)] (TN = 256)
  float* precast; int64_t ld_pre;
  float* amax_out;
  int32_t* status;
  int32_t tiles_n;     // ceil(N / TN)
  int32_t row_blocks;  // ceil(M / 256)
  int32_t xchg;        // 1: the tiles_n pairs of a row block exchange row records (Case 2)
  int32_t order;       // 0: round-robin over the tile list; 1: static groups of tiles_n pairs (TN 512)
  int32_t ngroups;     // order 1: the launch is ngroups x tiles_n pairs
  uint8_t* xws;        // xchg: the records (pair_xchg_bytes)
  int32_t dbg;         // measurement knobs (LOKA_PN_DEBUG; results are wrong when set): 1 = no
                       // waits for peers' records, 2 = no statistics pass
  uint64_t* trace;     // nullable: globaltimer stamps [CTA][tile < 64][8] (loka_debug_pairnorm_trace)
  int32_t bf16_in;     // 1: BF16 operands (kind::f16), K in elements, maps are byte views (2K wide)
  // NEXT-1 backward: the accumulator is dL/dh; xhat (bf16 [M, N], ld_xhat) and rstd_in ([M], BLOCK_RMS
  // [M, N/256]) are the forward's saves; bf16 / f32 dz out
  int32_t bwd;
  const __nv_bfloat16* xhat; int64_t ld_xhat;
  const float* rstd_in;
  CUtensorMap tx;      // bwd with bf16 dz: xhat [M, N] box {64 elements, 32 rows} SW128
  // castx (x_recipe, tensorwise): the kernel casts X itself (bf16 xb -> codes xq, the buffer ta maps)
  // with the amax at xamax; xcnt [row_blocks] counters (zeroed before the launch); xs_out: X's scale
  int32_t castx;
  const __nv_bfloat16* xb; int64_t ld_xb;
  uint8_t* xq; int64_t ld_xq;
  const float* xamax;
  uint32_t* xcnt;
  float* xs_out;
  int32_t cast_ahead;  // castx pacing (tiles ahead of the epilogue; LOKA_CAST_AHEAD, default 3)
  // mc: 4-CTA clusters of two pairs that own adjacent column tiles of the same row block; each CTA
  // loads half of its A rows (box {128, 64}: ta64) multicast to itself and its counterpart in the
  // other pair (TN = 256, order 0, tiles_n and the pair count even)
  int32_t mc;
  CUtensorMap ta64;
};
const float* pair_norm_unit_scale();  // device address of 1.0f (the BF16 path's s_a = s_b)
// tn = 512 (one accumulator, two N = 256 MMAs per K step) or 256 (double-buffered accumulators)
cudaError_t launch_pair_norm(const PairNormParams& p, int tn, int pairs, cudaStream_t st);
}  // namespace loka
