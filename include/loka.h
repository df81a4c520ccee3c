/*
 * loka.h — C ABI of the B200-native (sm_100a) LoKA FP8 linear+norm hot path.
 *
 * LoKA (arXiv 2605.10886) makes FP8 practical for large recommendation models.  This library
 * implements the data-parallel hot path named by BASELINE.json's north_star:
 *   a1-a3  quantize (granule amax -> scale -> saturating RNE cast)        loka_quantize
 *   a4-a5  FP8 GEMM (tcgen05, FP32 accumulation in TMEM) fused with
 *          dequant / bias / LayerNorm / RMSNorm / BlockNorm epilogue      loka_fp8_linear_norm
 *   a6     many small GEMMs in one launch                                  loka_grouped_fp8_linear
 *   a7     LoKA Probe error statistic (MERE)                               loka_probe_error
 *   a8     LoKA Dispatch constrained selection                             loka_dispatch_select
 *
 * Conventions (every call):
 *   - Returns loka_status; no C++ exception crosses the ABI.  loka_status_string() gives text.
 *   - Ownership: the caller owns all memory.  Tensor data/scales are DEVICE pointers; descriptor
 *     structs and arrays passed by pointer are HOST memory read only during the call.  The library
 *     never allocates device memory in a hot call; workspace is sized by loka_*_workspace_size().
 *   - Asynchrony: device work is enqueued on the caller's stream and never synchronized.  Errors
 *     detected on the device (non-finite input) are OR'ed into an optional device int32
 *     *status_dev (bit LOKA_DEVSTATUS_NONFINITE); the caller reads it after its own sync.
 *   - No CPU fallback: on a device that is not sm_100 the calls return LOKA_ERR_UNSUPPORTED.
 *   - Layouts: row-major, last dimension contiguous, leading dimension `ld` in elements.  Base
 *     pointers 16-byte aligned; ld*elem_size % 16 == 0 (TMA requirement) else LOKA_ERR_INVALID_ARG.
 *   - Thread safety: calls may be made concurrently; the only global state is a mutex-guarded
 *     per-device tensor-map/attribute cache.
 */
#ifndef LOKA_H_
#define LOKA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LOKA_VERSION_MAJOR 0
#define LOKA_VERSION_MINOR 1

#if defined(__GNUC__)
#define LOKA_API __attribute__((visibility("default")))
#else
#define LOKA_API
#endif

typedef struct CUstream_st* loka_stream_t; /* identical to cudaStream_t */

typedef enum loka_status {
  LOKA_OK = 0,
  LOKA_ERR_INVALID_ARG = 1, /* null pointer, bad enum, misalignment, bad leading dimension   */
  LOKA_ERR_SHAPE = 2,       /* inconsistent shapes; BLOCK_RMS with N % block != 0     */
  LOKA_ERR_UNSUPPORTED = 3, /* not sm_100, or a combination this build does not implement     */
  LOKA_ERR_NONFINITE = 4,   /* (host-visible form of the device status bit)                  */
  LOKA_ERR_WORKSPACE = 5,   /* workspace pointer null or smaller than loka_*_workspace_size() */
  LOKA_ERR_CUDA = 6,        /* a CUDA runtime call or launch failed                           */
  LOKA_ERR_NOT_PD = 7       /* Cholesky: not positive definite after the jitter escalation    */
} loka_status;

#define LOKA_DEVSTATUS_NONFINITE 0x1 /* OR'ed into *status_dev when an input holds NaN/Inf */

typedef enum loka_dtype {
  LOKA_F32 = 0,
  LOKA_BF16 = 1,
  LOKA_E4M3 = 2, /* OCP E4M3FN, max 448   (D4) */
  LOKA_E5M2 = 3  /* OCP E5M2,   max 57344                */
} loka_dtype;

/* Scale granularity in the tensor's own [rows, cols] frame ("tensorwise, rowwise,
 * blockwise"; D6).  FP32 scale array layouts (row-major):
 *   TENSOR [1] | ROW [rows] | COL [cols] | BLK_1x128 [rows, ceil(cols/128)]
 *   | BLK_128x1 [ceil(rows/128), cols] | BLK_128x128 [ceil(rows/128), ceil(cols/128)]        */
typedef enum loka_gran {
  LOKA_GRAN_TENSOR = 0,
  LOKA_GRAN_ROW = 1,
  LOKA_GRAN_COL = 2,
  LOKA_GRAN_BLK_1x128 = 3,
  LOKA_GRAN_BLK_128x1 = 4,
  LOKA_GRAN_BLK_128x128 = 5,
  /* MXFP8 block (NEXT-4): 1 row x 32 columns, scales [rows, ceil(cols/32)].  Quantize: row-major
   * codes only (no transposed copy).  GEMM: with UE8M0 scales on A and/or B it runs on the
   * block-scaled MMA (kind::mxf8f6f4.block_scale, one scale per 32-wide K block, its native
   * granule); combinations: A in {1x128, 1x32} x B in {128x128, 1x128, 1x32}.                  */
  LOKA_GRAN_BLK_1x32 = 6
} loka_gran;

/* F32: s = fl32(amax/max), r = fl32(max/amax) (D1).  UE8M0: s = 2^e, the smallest
 * power of two (e >= -127) with amax <= max*s, r = 2^-e (D7).  Both stored as FP32.
 * amax == 0 gives s = r = 1 (D2).                                                            */
typedef enum loka_scale_fmt { LOKA_SCALE_F32 = 0, LOKA_SCALE_UE8M0 = 1 } loka_scale_fmt;

typedef enum loka_phase {
  LOKA_PHASE_FULL = 0,          /* amax + cast in one call                                   */
  LOKA_PHASE_AMAX_ONLY = 1,     /* TENSOR: write the local amax to *amax_dev; COL: the local
                                   per-column amax to amax_dev[cols] (float, >= 0)            */
  LOKA_PHASE_CAST_WITH_AMAX = 2, /* TENSOR / COL: cast with the (all-reduced MAX) amax in
                                   amax_dev[0] / amax_dev[cols].  COL split-phase: the rowwise
                                   recipe's wgrad operands (per-column scales over M) stay
                                   bit-identical to one device when M is sharded (SURVEY.md
                                   §8(e): all-reduce MAX of the K- and N-length vectors)        */
  /* TENSOR only, delayed scaling: cast with amax_dev[0] (a previous step's
   * all-reduced amax; values beyond it saturate, D3) and write max |x| of THIS tensor to amax_dev[1]
   * in the same read of x (the next step's scale source: its all-reduce runs off the critical path). */
  LOKA_PHASE_CAST_DELAYED = 3
} loka_phase;

typedef enum loka_norm {
  LOKA_NORM_NONE = 0,
  LOKA_NORM_LAYER = 1,    /* (y-mu)/sqrt(var+eps) * gamma + beta, biased var (D13)  */
  LOKA_NORM_RMS = 2,      /* y/sqrt(mean(y^2)+eps) * gamma (D14)                    */
  LOKA_NORM_BLOCK_RMS = 3 /* RMSNorm per contiguous block of norm_block columns, unparameterized
                             ("RMSNorm((Wx + b).view(-1, BlockN)).view(B, N)")   */
} loka_norm;

/* Activation applied after the norm (PAPER.md:497-518 Hard Swish, "integrates seamlessly with
 * BlockNorm, allowing both operations to be fused").                 */
typedef enum loka_act {
  LOKA_ACT_NONE = 0,
  LOKA_ACT_HARDSWISH = 1 /* x * ReLU6(x + 3) / 6                              */
} loka_act;

/* GEMM direction ("separate optimization decisions for each direction").  The
 * kernel always computes C[M,N] = A[M,K] . B[N,K]^T with both operands K-major; the direction
 * says how the caller laid the operands out:
 *   FWD   Y  = X  W^T : A = Xq [M,K],        B = Wq [N,K]
 *   DGRAD dX = dY W   : A = dYq [M,N_out],   B = (W^T)q [K_in, N_out]   (K-major copy of W)
 *   WGRAD dW = dY^T X : A = (dY^T)q [N,M],   B = (X^T)q [K,M]           (K-major copies)      */
typedef enum loka_direction { LOKA_DIR_FWD = 0, LOKA_DIR_DGRAD = 1, LOKA_DIR_WGRAD = 2 } loka_direction;

typedef struct loka_tensor {
  void* data;               /* device pointer, row-major [rows, cols], leading dimension ld    */
  loka_dtype dtype;
  int64_t rows, cols, ld;
  float* scales;            /* device FP32 scale array for FP8 tensors (layout per gran)      */
  loka_gran gran;
  loka_scale_fmt scale_fmt;
} loka_tensor;

/* ---- a1-a3: quantize ----------------------------------------------------------------------
 * The FP8 recipes' quantize step: per granule amax -> scale -> saturating RNE cast (PAPER.md:535
 * "tensorwise, rowwise, blockwise" recipes; P:425 values are "clamped and quantized"
 * the quantization overhead this kernel has to keep small, D1-D7).
 * Errors: INVALID_ARG (null / misaligned pointers, ld * elem % 16 != 0, bad enums, phase != FULL
 * with a granularity other than TENSOR / COL), SHAPE (rows / cols mismatch), UNSUPPORTED (not sm_100, or a
 * transposed copy of 1x32 granules), WORKSPACE, CUDA; non-finite input -> status_dev bit.
 * x  : bf16 or f32 [rows, cols].
 * q  : e4m3/e5m2 codes [rows, cols] (q->data may be NULL when only qt is wanted) + q->scales in
 *      q->gran layout (required).  q->rows/cols must equal x's.
 * qt : nullable.  K-major copy for backward: codes of the SAME quantization written transposed,
 *      [cols, rows]; qt->scales gets the same scales in the transposed frame's layout
 *      (qt->gran must be the transpose of q->gran: ROW<->COL, 1x128<->128x1, others equal).
 *      One other combination: q->gran = qt->gran = BLK_1x128 quantizes x TWICE in one pass —
 *      q = x at 1x128 granules, qt = x at 128x1 granules written transposed (in qt's frame those
 *      granules are 1x128): the blockwise training recipe's forward and wgrad operands from one
 *      read of x.
 * phase, amax_dev: see loka_phase; amax_dev is a device float (TENSOR) or float[cols] (COL, split
 *      phases), else ignored.
 * Bit-exact with oracle/quantize.py (codes as bytes, scales as FP32 bit patterns).            */
LOKA_API loka_status loka_quantize(const loka_tensor* x, loka_tensor* q, loka_tensor* qt, loka_phase phase,
                          float* amax_dev, int32_t* status_dev, void* ws, size_t ws_bytes,
                          loka_stream_t stream);
LOKA_API size_t loka_quantize_workspace_size(const loka_tensor* x, const loka_tensor* q);

/* Grouped a1/a2: G (<= 64) independent ROW-granular quantizations in ONE launch (e.g. a layer
 * stack's input activation plus every layer's weight).  x[g], q[g] as for loka_quantize with
 * phase FULL and no transposed copy; all x[g] share one input dtype and all q[g] one FP8 format
 * and scale format, q[g].gran == LOKA_GRAN_ROW.  Results are bit-identical to G separate
 * loka_quantize calls.                                                                        */
LOKA_API loka_status loka_quantize_grouped(int32_t G, const loka_tensor* x, loka_tensor* q, int32_t* status_dev,
                                           loka_stream_t stream);

/* ---- a4-a5: FP8 GEMM + fused epilogue ----------------------------------------------------- */
typedef struct loka_linear_args {
  int64_t M, N, K;
  loka_direction dir;       /* metadata; see loka_direction                                   */
  loka_tensor a;            /* e4m3/e5m2 [M,K] K-major, scales gran TENSOR | ROW | BLK_1x128  */
  loka_tensor b;            /* e4m3/e5m2 [N,K] K-major, scales gran TENSOR | ROW, or with a
                               BLK_1x128 A: BLK_128x128 | BLK_1x128 (blockwise recipe, FP32
                               promotion per 128-K block; epilogue NONE (+bias), FP8 output
                               only for N <= 128)                                             */
  const void* bias;         /* nullable [N], dtype bias_dtype (F32 | BF16); added before norm */
  loka_dtype bias_dtype;
  loka_norm norm;
  int32_t norm_block;       /* BLOCK_RMS block size (256 in the paper)          */
  float eps;                /* <= 0 selects the default: 1e-5 LAYER, 1e-6 RMS/BLOCK_RMS       */
  const float* gamma;       /* nullable [N] (LAYER, RMS)                                      */
  const float* beta;        /* nullable [N] (LAYER)                                           */
  loka_tensor y;            /* [M,N]: F32 | BF16 | E4M3/E5M2 with y.scales ROW (next layer's
                               rowwise input, amax over the full normalised row) or, with a
                               LAYER / RMS / BLOCK_RMS norm and no gamma / beta / act,
                               BLK_1x128 [M, ceil(N/128)] (the blockwise recipe's next input;
                               the CTA-pair route, PAPER.md:535 + P:464; other routes ->
                               LOKA_ERR_UNSUPPORTED)                                           */
  float* debug_precast;     /* nullable [M,N] FP32 (ld = N): post-norm values before the
                               output cast, for tests                                        */
  int32_t* status_dev;      /* nullable                                                       */
  loka_act act;             /* applied after the norm (and gamma/beta); NONE by default.  The
                               FP8 output's row amax is then taken over the activated values  */
  /* NEXT-1 norm backward fused into the (dgrad) GEMM epilogue: when bwd_xhat is
     set, A.B^T (dequantized) is dL/dh for a forward h = act(norm(z)*gamma + beta) with this args'
     norm / norm_block / gamma / beta / act, and y receives dL/dz:
       g = dh * act'(xhat*gamma + beta) * gamma,
       LAYER: dz = rstd (g - mean(g) - xhat mean(g xhat));  RMS: dz = rstd (g - xhat mean(g xhat));
       BLOCK_RMS: RMS per block.  bwd_xhat: the forward's normalised values (bf16 [M, N], ld
       bwd_xhat_ld, ld*2 % 16 == 0); bwd_rstd: [M] (LAYER/RMS) or [M, N/norm_block].  No bias;
       the fused-epilogue row limits of the forward apply (N <= 4096 for LAYER/RMS).               */
  const void* bwd_xhat;
  int64_t bwd_xhat_ld;
  const float* bwd_rstd;
  /* forward saves for that backward (nullable): xhat (bf16, ld save_xhat_ld) and rstd of z        */
  void* save_xhat;
  int64_t save_xhat_ld;
  float* save_rstd;
  /* NEXT-4: producer-side tensor amax.  Nullable device float, zeroed by the
     caller: the epilogue folds max |y| over the values it stores (after their rounding to the
     output dtype; F32 / BF16 outputs) into it (atomicMax on the IEEE bit pattern), so the next
     layer's tensorwise quantize can skip its amax pass (LOKA_PHASE_CAST_WITH_AMAX), and a data-
     parallel job all-reduces this word instead (a9).  Non-finite outputs raise it to Inf/NaN.    */
  float* amax_out;
  /* x_recipe with a TENSOR-granular unquantized A (see loka_fp8_linear_norm): nullable device float,
     the amax to cast A with (a data-parallel caller's all-reduced global amax, a9); NULL = the call
     computes A's own amax first.                                                                 */
  const float* x_amax;
} loka_linear_args;

/* x_recipe: a->a may also be the UNQUANTIZED activation (bf16 / f32, ld * elem % 16
 * == 0): the call then quantizes it first, with a->a.gran (TENSOR | ROW | BLK_1x128 | BLK_1x32) and
 * a->a.scale_fmt, to e4m3 (e5m2 when dir == DGRAD: the gradient dY, reading D5), into the front of the
 * workspace (loka_linear_workspace_size includes it), and runs the FP8 problem on those codes — the
 * same bytes a separate loka_quantize would produce.
 * Y = epilogue(A . B^T): acc(FP32, TMEM) -> y = acc*sa[m]*sb[n] (+bias[n]) -> norm -> act -> cast
 * ("fuse normalization directly into the GEMM epilogue"; formula P:460; Case 1 / 2
 * P:464-473).  Routes (chosen per call, identical semantics):
 *   * >= 74 256x256 tiles, or a LAYER/RMS row wider than 2048, with TENSOR/ROW scales and LAYER /
 *     RMS / BLOCK_RMS(256): the CTA-pair engine with the norm in its epilogue (pairnorm.cu).  Rows
 *     wider than 256 columns exchange per-row statistics between the pairs that own the row's
 *     column tiles through the workspace (loka_linear_workspace_size: 4 KB per 256-row x 256-column
 *     tile; a memset node fills it before the kernel).  N <= 8192.  FP8 output requires no gamma /
 *     beta / act on this route (else the next one).
 *   * otherwise the single-CTA engine: full-row norms span a thread-block cluster (<= 8 CTAs, or 16
 *     of 256 columns for N <= 4096); N > 4096 full-row norms there -> UNSUPPORTED.
 * BLOCK_RMS and NONE take any N.  K % 16 == 0.                                                   */
LOKA_API loka_status loka_fp8_linear_norm(const loka_linear_args* args, void* ws, size_t ws_bytes,
                                 loka_stream_t stream);
LOKA_API size_t loka_linear_workspace_size(const loka_linear_args* args);

/* The library's own BF16 path with the same fused epilogue (the secondary BF16
 * denominator, which separates the gain of FP8 from the gain of fusion): A [M,K] and B [N,K] are
 * BF16 (a/b dtype LOKA_BF16, K-major, ld * 2 % 16 == 0; scales ignored, unit), C = A . B^T by
 * tcgen05.mma.cta_group::2.kind::f16 (FP32 accumulation in TMEM) on the CTA-pair engine, then the
 * pair-norm epilogue (LAYER / RMS / BLOCK_RMS(256), bias, gamma / beta, h-swish, FP8 row-scale
 * output without gamma / beta / act).  Workspace: loka_bf16_linear_workspace_size.  Errors as
 * loka_fp8_linear_norm; other norms or the NEXT-1 backward fields -> UNSUPPORTED.              */
LOKA_API loka_status loka_bf16_linear_norm(const loka_linear_args* args, void* ws, size_t ws_bytes,
                                           loka_stream_t stream);
LOKA_API size_t loka_bf16_linear_workspace_size(const loka_linear_args* args);

/* ---- a4+a5 for a whole LRM MLP stack in ONE launch (BASELINE.json configs[1]) --------------
 * Layer l: h_{l+1} = norm_l(h_l . W_l^T) with h_0 = x (e4m3 + ROW scales) and W_l e4m3 + ROW
 * scales (No Bias, unparameterized norm: PAPER.md:443, 483).  Every intermediate h_l (l = 1..L-1)
 * is quantized rowwise to e4m3 exactly as loka_fp8_linear_norm with an E4M3/ROW output would,
 * but never leaves the chip: a cluster of C CTAs keeps a 128-row block's activation in shared
 * memory (the next layer's A operand) and streams only the weights.  Only y (the last layer's
 * output) is written (plus the hand-offs the caller asks for in h[]).  Every layer is the
 * arithmetic of a loka_fp8_linear_norm call with an E4M3/ROW output (the last: y's dtype), up to
 * the order of the FP32 accumulation (the A operand arrives slice by slice and is consumed in
 * arrival order) and of the row-statistics merge.
 * Limits: L <= 8, dims[l] <= 1024 for l < L (K of each layer), with C = ceil(max N / 256), every
 * N = dims[l+1] in {64C, 128C, 256C} (C <= 8); norm in {NONE, LAYER, RMS}.                     */
typedef struct loka_stack_args {
  int32_t L;
  int64_t M;
  int64_t dims[9];          /* dims[0] = K of layer 0, dims[l+1] = N of layer l                 */
  loka_tensor x;            /* e4m3 [M, dims[0]] + ROW scales                                    */
  loka_tensor w[8];         /* e4m3 [dims[l+1], dims[l]] + ROW scales                           */
  loka_norm norm[8];
  float eps[8];             /* <= 0: default (1e-5 LAYER, 1e-6 RMS)                              */
  loka_tensor y;            /* [M, dims[L]]: F32 | BF16 | E4M3/E5M2 with ROW scales             */
  int32_t* status_dev;      /* nullable                                                          */
  loka_tensor h[7];         /* optional saved hand-offs: h[l] = h_{l+1} (e4m3 [M, dims[l+1]],
                               ld % 16 == 0, ROW scales) for l < L-1; data NULL = not saved
                               (training keeps them for the backward pass)                        */
  void* ws;                 /* device workspace, >= loka_stack_workspace_size(args) bytes (the
                               cluster all-gathers a hand-off through L2; a saved h[l] doubles
                               as that buffer), 16-byte aligned; may be NULL when the size is 0   */
  size_t ws_bytes;
  float* debug_precast[8];  /* tests: nullable device FP32 [M, dims[l+1]] (dense): layer l's
                               normalised values just before the cast of an FP8 hand-off / output
                               (the hand-off codes and row scales are checked
                               bit-exactly against the oracle's quantize of these values).  Any
                               non-null entry selects the kernel's debug instance.                */
} loka_stack_args;
LOKA_API loka_status loka_fp8_mlp_stack(const loka_stack_args* args, loka_stream_t stream);
LOKA_API size_t loka_stack_workspace_size(const loka_stack_args* args);

/* ---- a6: grouped launch: G independent linear+norm problems ------------------------------- *
 * The paper's "many small GEMMs" of heterogeneous LRM layers (PAPER.md:78-79 DHEN / Wukong wide
 * ensembles; "< 20% of hardware capacity") in one persistent launch: problems with the plain
 * dequant(+bias) epilogue and bf16 / f32 output share one CTA-pair launch (<= 64 problems per launch,
 * longest K first, 256x256 tiles); the others run their own loka_fp8_linear_norm route.  Same
 * arguments, errors and bit-exact results as G separate loka_fp8_linear_norm calls (args is a host
 * array of G structs, read during the call).                                                      */
LOKA_API loka_status loka_grouped_fp8_linear(int32_t G, const loka_linear_args* args, void* ws, size_t ws_bytes,
                                    loka_stream_t stream);
LOKA_API size_t loka_grouped_workspace_size(int32_t G, const loka_linear_args* args);

/* The library's own BF16 form of a6 (the secondary BF16 denominator of the
 * ensemble, "many small GEMMs"): G problems with BF16 A [M,K] and B [N,K] (a/b dtype
 * LOKA_BF16, K-major, ld * 2 % 16 == 0, scales ignored), Y = A . B^T (+ bias[n]) in bf16 or f32,
 * in persistent launches of the CTA-pair engine (one per 64 problems) with tcgen05.mma.cta_group::2.kind::f16 (FP32
 * accumulation in TMEM), longest K first, 256x256 tiles.  norm / act must be NONE, no FP8 output, no
 * backward fields (else UNSUPPORTED).  No workspace.  args: a host array of G
 * structs, read during the call.                                                                  */
LOKA_API loka_status loka_grouped_bf16_linear(int32_t G, const loka_linear_args* args, loka_stream_t stream);

/* ---- NEXT-4: NVFP4 ----------------------------------------------------------
 * The paper names FP4 as future work; the recipe is DESIGN.md D35-D38 (oracle/nvfp4.py):
 * E2M1 codes (values {0, .5, 1, 1.5, 2, 3, 4, 6}, saturating RNE), one E4M3 block-scale code per
 * 16 consecutive elements of a row, one FP32 tensor scale s_t = fl32(A / 2688) from the tensor amax A:
 *   sf = E4M3(fl32(fl32(a_block * r_t) / 6)), codes = E2M1(fl32(x * fl32(r_t / decode(sf)))),
 *   r_t = fl32(2688 / A); x_hat = e2m1(code) * decode(sf) * s_t.
 * Ownership and errors as everywhere: caller-owned device memory, async on `stream`.            */
typedef struct loka_nvfp4_tensor {
  void* data;               /* packed E2M1 codes [rows, cols/2] bytes; element 2j in the low nibble
                               of byte j; 16-byte aligned                                         */
  int64_t rows, cols;       /* logical elements; cols % 64 == 0                                  */
  int64_t ld;               /* bytes between row starts: >= cols/2, multiple of 16               */
  uint8_t* block_scales;    /* E4M3 codes [rows, cols/16], row-major, leading dimension cols/16  */
  float* tensor_scale;      /* device FP32 [1]: s_t                                              */
} loka_nvfp4_tensor;

/* x: bf16 or f32 [rows, cols] (ld elements, 16-byte aligned rows).  amax_dev: nullable device float
 * holding the tensor amax to use (data parallel: the all-reduced global amax, as the FP8 tensorwise
 * split phase); NULL = computed here (workspace >= loka_quantize_nvfp4_workspace_size bytes).
 * Non-finite input sets LOKA_DEVSTATUS_NONFINITE in *status_dev (when computing the amax).
 * Bit-exact with oracle/nvfp4.py: codes, block-scale codes and s_t.                              */
LOKA_API loka_status loka_quantize_nvfp4(const loka_tensor* x, loka_nvfp4_tensor* q, const float* amax_dev,
                                         int32_t* status_dev, void* ws, size_t ws_bytes, loka_stream_t stream);
LOKA_API size_t loka_quantize_nvfp4_workspace_size(const loka_tensor* x);

/* y = epilogue(A_hat B_hat^T): A [M,K], B [N,K] NVFP4 (both K-major), on the block-scaled tensor
 * cores (tcgen05.mma kind::mxf4nvf4.block_scale.scale_vec::4X; FP32 accumulation in TMEM), the
 * tensor scales s_t(A) s_t(B) applied in the epilogue, then bias / LayerNorm / RMSNorm / BlockNorm
 * and the output cast exactly as loka_fp8_linear_norm (y: F32 | BF16 | E4M3 + ROW scales).
 * K % 64 == 0.  Workspace: the scale atoms (loka_nvfp4_linear_workspace_size).                  */
typedef struct loka_nvfp4_linear_args {
  int64_t M, N, K;
  loka_nvfp4_tensor a, b;
  const void* bias;         /* nullable [N] */
  loka_dtype bias_dtype;
  loka_norm norm;
  int32_t norm_block;
  float eps;
  const float* gamma;       /* nullable [N] */
  const float* beta;        /* nullable [N] */
  loka_tensor y;
  int32_t* status_dev;      /* nullable */
} loka_nvfp4_linear_args;
LOKA_API loka_status loka_nvfp4_linear_norm(const loka_nvfp4_linear_args* args, void* ws, size_t ws_bytes,
                                            loka_stream_t stream);
LOKA_API size_t loka_nvfp4_linear_workspace_size(const loka_nvfp4_linear_args* args);

/* ---- NEXT-4: quantized data-parallel gradient reduction (D39) ------------------------
 * out[i, j] = sum_{p=0}^{P-1} decode(codes[p][i*ld + j]) * scales[p][i]   (FP32 fmaf, rank order)
 * codes / scales: host arrays of P (1..8) device pointers to each rank's rowwise-quantized shard
 * (loka_quantize ROW codes + FP32 row scales, already offset to the shard's first row); they may
 * point into peer GPUs' memory mapped into this device (symmetric memory over NVLink / NVSwitch):
 * the kernel then pulls one byte per element from every rank.  fmt: E4M3 | E5M2.  cols % 16 == 0, ld % 16 == 0, 16-byte aligned rows; out FP32
 * [rows, cols] (ld_out % 4 == 0).  The caller orders the peers' writes before the launch (stream
 * sync + barrier) and the launch before the peers' next writes.                                 */
LOKA_API loka_status loka_dequant_reduce(int32_t P, const uint8_t* const* codes, const float* const* scales,
                                         loka_dtype fmt, int64_t rows, int64_t cols, int64_t ld, float* out,
                                         int64_t ld_out, loka_stream_t stream);

/* ---- a7: LoKA Probe error statistic ------------------------------------------------------- */
typedef struct loka_probe_pair {
  const void* out;          /* device [M,N], dtype out_dtype (F32 | BF16): low-precision path */
  loka_dtype out_dtype;
  const void* ref;          /* device [M,N], dtype ref_dtype (F32 | BF16): BF16 path (D9)     */
  loka_dtype ref_dtype;
  int64_t M, N, ld_out, ld_ref;
} loka_probe_pair;

typedef struct loka_probe_stats {
  double mere;              /* (1/(M N)) sum |out-ref| / max(|ref|, f), f = floor_rel*mean|ref| */
  double max_rel;
  double sum_abs_ref;
  int64_t count;
  int64_t n_floored;        /* elements with |ref| < f                                        */
} loka_probe_stats;

/* One launch sequence for L layers; stats_dev is a DEVICE array of L loka_probe_stats.
 * Any leading dimension is accepted (16-byte-aligned rows take the vector path).
 * Within 1e-5 relative of oracle/probe.py (D8-D10).                  */
LOKA_API loka_status loka_probe_error(int32_t L, const loka_probe_pair* pairs, double floor_rel,
                             loka_probe_stats* stats_dev, void* ws, size_t ws_bytes, loka_stream_t stream);
LOKA_API size_t loka_probe_workspace_size(int32_t L, const loka_probe_pair* pairs);
/* Data-parallel probe (SURVEY.md §8(e) "probe sums and max values can be all-reduced"): each rank
 * holds row shards of the layers' pairs.  global_sum_count_dev (DEVICE, [L][2] doubles) holds each
 * layer's (sum |ref|, element count) summed over all ranks (the caller's all-reduce of the local
 * loka_probe_error results' sum_abs_ref and count), so every shard uses the floor
 * f = floor_rel * sum / count of the whole layer; the per-rank results then combine exactly with
 * loka_probe_merge into the statistic of the concatenated tensor.  Same workspace as above.      */
LOKA_API loka_status loka_probe_error_global(int32_t L, const loka_probe_pair* pairs, double floor_rel,
                                            const double* global_sum_count_dev, loka_probe_stats* stats_dev,
                                            void* ws, size_t ws_bytes, loka_stream_t stream);
/* Host: combine R ranks' stats of L layers, parts[r * L + l] -> out[l] (counts, floored counts and
 * sum |ref| add; max_rel max; mere = sum mere_r count_r / sum count_r).                         */
LOKA_API loka_status loka_probe_merge(int32_t R, int32_t L, const loka_probe_stats* parts, loka_probe_stats* out);

/* ---- NEXT-2: LoKA Probe online input tracker (batched Welford) ------------
 * Running summaries of one layer's input distribution, feature dimension only (the batch rows are
 * independent): n (host), mean [K] and the unnormalised scatter Sigma [K, K]
 * (row-major, ld K), both FP32 device arrays owned by the caller (zero them for n = 0).
 * loka_probe_track_input merges one batch X [B, K] (bf16, ld*2 % 16 == 0, K % 8 == 0):
 *   delta = mu_b - mean, mean += (B / n_new) delta,
 *   Sigma += S_b + (n B / n_new) delta delta^T with S_b = (X - mu_b)^T (X - mu_b)
 * (S_b on the tensor cores from a centred bf16 transpose, FP32 accumulation) and sets n += B.
 * The unbiased covariance is Sigma / (n - 1).  Async on the stream; ws >= the workspace size.   */
typedef struct loka_welford_state {
  int64_t n;
  int64_t K;
  float* mean;
  float* scatter;
} loka_welford_state;
LOKA_API size_t loka_probe_track_workspace_size(const loka_welford_state* st, int64_t B);
LOKA_API loka_status loka_probe_track_input(loka_welford_state* st, const loka_tensor* x, void* ws, size_t ws_bytes,
                                           loka_stream_t stream);
/* out [K, K] (device FP32, caller-owned) = scatter / (n - 1): the unbiased covariance of the tracked
 * inputs.  n < 2 -> LOKA_ERR_SHAPE.  Asynchronous.                                  */
LOKA_API loka_status loka_probe_track_covariance(const loka_welford_state* st, float* out, loka_stream_t stream);

/* ---- NEXT-3: LoKA Probe weight tracker and learned-distribution sampling ----
 * All matrices are FP32, row-major and dense (ld = number of columns unless an ld is passed),
 * device pointers owned by the caller; calls are asynchronous on
 * the stream unless stated.  Readings of the paper: DESIGN.md D30-D34.
 *
 * loka_philox_normal: out[e] = standard normal number (offset + e) of the stream keyed by seed:
 * Philox4x64-10 (counter (b, 0, 0, 0), key (seed, 0)) for block b = (offset + e) / 4, Box-Muller on
 * the top 24 bits of the word pairs (x0, x1) and (x2, x3) (D31); FP32.  n >= 0.        */
LOKA_API loka_status loka_philox_normal(uint64_t seed, uint64_t offset, int64_t n, float* out, loka_stream_t stream);

/* loka_cholesky_jittered (PAPER.md:377-381 and its footnote): l = lower Cholesky factor of
 * a_scale * (a + a^T)/2 + eps I, eps = eps_rel * trace(a_scale * a) / n (a non-positive trace
 * uses scale 1, D30), escalated x10 up to `escalations` times while a pivot is not positive
 * (SPEC.md:262).  a [n, n] (lda), l [n, n] (ldl, strict upper part zeroed) must not overlap.
 * *eps_used (host) receives the eps of the successful factorisation.  SYNCHRONOUS: it reads the
 * trace and the pivot status back (the factorisation itself runs on the device: 64-column
 * panels, FP32).  LOKA_ERR_NOT_PD after the escalations.  ws >= loka_cholesky_workspace_size(). */
LOKA_API size_t loka_cholesky_workspace_size(int64_t n);
LOKA_API loka_status loka_cholesky_jittered(const float* a, int64_t lda, int64_t n, float a_scale, float eps_rel,
                                            int32_t escalations, float* l, int64_t ldl, float* eps_used, void* ws,
                                            size_t ws_bytes, loka_stream_t stream);

/* Matrix-normal weight tracker: W [M, N] ~ MN(mean, U, V).  mean [M, N],
 * U [M, M], V [N, N] are the caller's device arrays (ld = M / N); count, momentum m and eps_rel
 * are host fields.  loka_probe_track_weight_init sets mean = W, U = I, V = I, count = 0
 * (SPEC.md:216).  loka_probe_track_weight applies one update in the paper's order
 * (PAPER.md:319-348): eps_U = eps_rel tr(U)/M, eps_V = eps_rel tr(V)/N; W_c = W - mean;
 * L_V L_V^T = V + eps_V I, W~ = W_c L_V^{-T}, U' = W~ W~^T / N; L_U L_U^T = U + eps_U I,
 * W^ = L_U^{-1} W_c, V' = W^^T W^ / M; U = sym(m U + (1-m) U') + eps_U I, V likewise;
 * s = tr(U)/M, U /= s, V *= s; mean = m mean + (1-m) W (D32-D34); count += 1.  W is F32 or BF16
 * (any ld >= N).  No host synchronisation: a non-positive pivot sets bit 0 of *status_dev
 * (nullable).  ws >= loka_probe_track_weight_workspace_size().                                 */
typedef struct loka_matnorm_state {
  int64_t M, N;
  int64_t count;
  float momentum;
  float eps_rel;
  float* mean;
  float* U;
  float* V;
} loka_matnorm_state;
LOKA_API loka_status loka_probe_track_weight_init(loka_matnorm_state* st, const loka_tensor* w, loka_stream_t stream);
LOKA_API size_t loka_probe_track_weight_workspace_size(const loka_matnorm_state* st);
LOKA_API loka_status loka_probe_track_weight(loka_matnorm_state* st, const loka_tensor* w, int32_t* status_dev,
                                             void* ws, size_t ws_bytes, loka_stream_t stream);

/* Sampling learned distributions, Z from loka_philox_normal's stream:
 *   loka_probe_sample_input:  out [B, K] = 1 mean^T + Z L_Sigma^T, Z [B, K] row-major (elements
 *                             offset .. offset + B K - 1 of the stream);
 *   loka_probe_sample_weight: out [M, N] = mean + L_U (Z L_V^T), Z [M, N] row-major.
 * L_* are lower-triangular factors with a ZERO strict upper part (as loka_cholesky_jittered
 * writes them; the GEMMs skip the zero tiles but read inside the diagonal tiles).  out: F32 or BF16, rows x cols = B x K / M x N, any ld >= cols.
 * ws >= loka_probe_sample_workspace_size(rows, cols, is_weight).                               */
LOKA_API size_t loka_probe_sample_workspace_size(int64_t rows, int64_t cols, int32_t is_weight);
LOKA_API loka_status loka_probe_sample_input(const float* mean, const float* l_sigma, int64_t K, int64_t B,
                                             uint64_t seed, uint64_t offset, loka_tensor* out, void* ws,
                                             size_t ws_bytes, loka_stream_t stream);
LOKA_API loka_status loka_probe_sample_weight(const float* mean, const float* l_u, const float* l_v, int64_t M,
                                              int64_t N, uint64_t seed, uint64_t offset, loka_tensor* out, void* ws,
                                              size_t ws_bytes, loka_stream_t stream);

/* ---- a8: LoKA Dispatch (host) -------------------------------------------------------------- */
typedef struct loka_candidate {
  const char* id;
  loka_direction dir;
  double mere;
  double time_us;           /* end-to-end time of the op with this recipe (D19)               */
} loka_candidate;

/* keep candidates with mere < mere_budget and baseline_time_us/time_us >
 * min_speedup (both strict); choose the smallest time; ties -> lexicographically smallest id;
 * *chosen = index, or -1 for the baseline when none passes.  Pure host function.             */
LOKA_API loka_status loka_dispatch_select(const loka_candidate* c, int32_t n, double baseline_time_us,
                                 double mere_budget, double min_speedup, int32_t* chosen);

/* ---- helpers -------------------------------------------------------------------------------- */
LOKA_API const char* loka_status_string(loka_status s);
LOKA_API int32_t loka_device_supported(int32_t device); /* 1 if sm_100, else 0 */
LOKA_API int32_t loka_version(void);                    /* major*100 + minor */
/* Hash of the sources and flags the library was built from (paper_2605_10886_b200/build.py); the
 * Python binding refuses a library whose hash differs from the source tree's (a stale binary).   */
LOKA_API const char* loka_source_hash(void);
/* Number of kernel launches the library made since load (process-wide counter; for bench
 * evidence of "gpu_launches").                                                               */
LOKA_API int64_t loka_launch_count(void);
/* Pipeline watchdog (debug): every mbarrier wait in the GEMM kernels gives up after 4 s, records
 * where it stalled and lets the kernel finish (with garbage output) instead of hanging the GPU.
 * Returns the number of timed-out waits since the last reset (0 = healthy; -1 = CUDA error) and
 * fills info3 = {tag (1 smem-empty, 2 smem-full, 3 accumulator-ready), block id,
 * thread | parity << 32}.  reset != 0 clears the record.  Synchronous.                      */
LOKA_API int64_t loka_debug_hang_info(uint64_t* info3, int32_t reset);
/* Phase trace (debug/profiling): enable = 1 clears the buffer and makes every later GEMM CTA
 * record 16 globaltimer stamps (entry, after grid-dependency wait, first TMA issued, first stage
 * landed, last MMA committed, accumulator ready, statistics done, stores done, pass-1 done,
 * halves merged, cluster merged, finalized) at
 * out[(blockIdx.x + gridDim.x*blockIdx.y)*16 + slot] for the first 4096 CTAs of the LAST launch;
 * the fused stack kernel records 64 stamps per CTA (2 + 7 per layer, see stack.cu) at
 * out[65536 + (blockIdx.x + gridDim.x*blockIdx.y)*64 + slot] for its first 512 CTAs.
 * enable = 0 turns it off, enable = -1 leaves it unchanged.  Copies up to n stamps into out
 * (host, may be NULL).  Returns the number copied, -1 on a CUDA error.  Synchronous.          */
LOKA_API int64_t loka_debug_trace(int32_t enable, uint64_t* out, int64_t n);
/* Pair-norm phase trace (debug/profiling): dev_buf (device, >= 148 * 64 * 8 u64, caller-owned) makes
 * later pair-norm launches record globaltimer stamps per CTA and tile (< 64) at
 * dev_buf[(blockIdx.x * 64 + tile) * 8 + slot]: 0 accumulator ready, 1 statistics pass done,
 * 2 row records merged, 3 stores issued (epilogue thread 0); 4 / 5 / 6 MMA thread (leader CTAs):
 * waiting for the accumulator buffer, buffer acquired, last MMA committed.  NULL turns it off.    */
LOKA_API void loka_debug_pairnorm_trace(unsigned long long* dev_buf);

#ifdef __cplusplus
}
#endif
#endif /* LOKA_H_ */
