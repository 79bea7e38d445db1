/*
 * zo_b200.h -- C ABI of the B200 (sm_100a) zeroth-order training-step kernels.
 *
 * Drop-in boundary for the hot path of the DistZO2 reference package
 * `zosim` (/root/reference/pkg/src/zosim).  The reference has no FFI: its
 * boundary is a Python function API.  Each entry below replaces one
 * numpy call site of that API (file:line cited per entry); the Python
 * package paper_2507_03211_b200 mirrors the reference's function names and
 * binds these symbols with ctypes.
 *
 * Conventions
 *  - every entry returns an int status: ZO_OK or one of the ZO_ERR_* codes
 *    below, which map 1:1 onto the reference's exception hierarchy
 *    (src/zosim/errors.py:8-56); zo_last_error() returns the message.
 *  - all device pointers are plain CUDA device addresses; `stream` is a
 *    cudaStream_t passed as void* (NULL = legacy default stream); every
 *    compute entry is asynchronous on that stream.
 *  - element offsets ("keys") are GLOBAL parameter indices in the
 *    reference's (block, tensor, element) order (src/zosim/model.py:81-101);
 *    they key the counter-based direction z, so z never depends on how a
 *    block is sliced or which rank computes it.
 *  - bf16 buffers are passed as void* (bit pattern of __nv_bfloat16).
 */
#ifndef ZO_B200_H_
#define ZO_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes <-> src/zosim/errors.py (CLI exit codes src/zosim/cli.py:176-192) */
#define ZO_OK 0
#define ZO_ERR_PROTOCOL 1 /* ProtocolError       (errors.py:47-51)  */
#define ZO_ERR_CONFIG 2   /* ConfigurationError / DimensionError (errors.py:13-20) */
#define ZO_ERR_NUMERIC 3  /* NumericError        (errors.py:31-34)  */
#define ZO_ERR_FABRIC 4   /* FabricFault         (errors.py:37-40)  */
#define ZO_ERR_CUDA 5     /* CUDA runtime failure (no reference analogue) */

/* direction source */
#define ZO_Z_PHILOX 0 /* z = Philox4x32-10(seed, key) + Box-Muller, in-register   */
#define ZO_Z_ORACLE 1 /* z = injected f64 array (the reference's PCG64 stream)   */

/* shadow kinds of a segment */
#define ZO_SHADOW_BF16 0 /* perturbed copy rounded to bf16 (GEMM operand)        */
#define ZO_SHADOW_F32 1  /* perturbed copy kept in fp32 (LN gains, biases)       */
#define ZO_SHADOW_NONE 2 /* update only; consumer perturbs on read (embedding)  */

/* zo_perturb_update flags */
#define ZO_PU_UPDATE 1u  /* apply the pending update theta -= (lr g_prev) z_prev  */
#define ZO_PU_SHADOW_A 2u /* write shadow A = theta' + scale_a z_cur             */
#define ZO_PU_SHADOW_B 4u /* write shadow B = theta' + scale_b z_cur             */
#define ZO_PU_FILL 8u     /* launch as short-lived CTAs (one chunk per warp) so a
                             pass on a low-priority stream only fills SMs that the
                             forward leaves idle and never holds one for long    */

/* zo_gemm_bf16 epilogues */
#define ZO_EPI_F32 0          /* out f32  = acc                                   */
#define ZO_EPI_BIAS_BF16 1    /* out bf16 = acc + bias            (QKV)           */
#define ZO_EPI_BIAS_GELU_BF16 2 /* out bf16 = gelu_tanh(acc + bias) (FFN up)      */
#define ZO_EPI_BIAS_RESID_F32 3 /* out f32 += (acc + bias)        (O-proj, FFN down) */
#define ZO_EPI_CE 4           /* LM head: per-row partial max/sum-exp + target logit */
#define ZO_EPI_BIAS_RELU_BF16 5 /* out bf16 = relu(acc + bias)    (real-OPT FFN up) */
/* OR-ed into `epilogue`: B is given transposed, [N, K] row-major (K
 * contiguous, ldb >= K) -- e.g. a tied LM head reading the [V, d] token
 * embedding.  Supported with ZO_EPI_F32 and ZO_EPI_CE. */
#define ZO_GEMM_B_KMAJOR 0x100

/* One tensor of a parameter block, as the perturb/update kernel sees it. */
typedef struct ZoSegment {
  int64_t src;    /* global element offset (z key) of the tensor's element 0  */
  int64_t rows;   /* rows x cols elements, row-major in the master buffer     */
  int64_t cols;
  int64_t dst;    /* element offset of the tensor inside its shadow buffer    */
  int64_t dst_ld; /* shadow row stride in elements (>= cols)                  */
  int32_t kind;   /* ZO_SHADOW_*                                              */
  int32_t reserved; /* block index (completion counters of zo_perturb_update_bg) */
} ZoSegment;

/* Per-iteration scalars, device-resident so a captured CUDA graph can replay
 * steps: the host writes seed_cur; zo_grad_finalize writes the rest. */
typedef struct ZoStepScalars {
  uint64_t seed_cur;  /* key of this iteration's direction z_j              */
  uint64_t seed_prev; /* key of the pending update's direction z_{j-1}      */
  double lr_g_prev;   /* lr * g_{j-1}; formed as (lr*g) like zo.py:125      */
  int64_t pending;    /* 1 when an update is pending (zo.py:267-271 flag)    */
} ZoStepScalars;

const char* zo_version(void);
const char* zo_last_error(void);
/* 0 when device `dev` is an sm_100 part the library was built for. */
int zo_device_check(int dev);

/*
 * Fused perturb / update over a set of tensors (one block or a whole model).
 * Replaces perturb_block / perturb_params (src/zosim/zo.py:90-113) and
 * update_block / update_params (src/zosim/zo.py:116-130), and the per-block
 * deferred update of dual_forward (src/zosim/zo.py:204-211).
 *   theta        fp32 master; element with key e lives at theta[e - theta_key0]
 *   segs/prefix  device table: prefix[i] = first tile of segs[i], prefix[n]=total
 *   flags        ZO_PU_*; the update is applied only when scal->pending != 0
 *   zmode        ZO_Z_PHILOX (keys scal->seed_cur/seed_prev) or ZO_Z_ORACLE
 *                (z_cur/z_prev f64 arrays indexed by key - z_key0; exact f64
 *                arithmetic, bit-identical to the reference's f32 results)
 *   scale_a/b    cumulative perturbation of shadows A/B (e.g. +eps, -eps)
 */
int zo_perturb_update(float* theta, int64_t theta_key0, const ZoSegment* segs,
                      const int64_t* tile_prefix, int32_t n_segs, int64_t n_tiles,
                      void* wsh_a, float* vsh_a, void* wsh_b, float* vsh_b,
                      double scale_a, double scale_b, uint32_t flags,
                      const ZoStepScalars* scal, int32_t zmode,
                      const double* z_cur, const double* z_prev, int64_t z_key0,
                      void* stream);
/*
 * CUDA-graph capture of a step that honours per-launch priorities (torch's
 * graphs instantiate without cudaGraphInstantiateFlagUseNodePriority): every
 * kernel this library launches carries its stream's priority as a launch
 * attribute, and a graph instantiated here replays with those priorities, so
 * a low-priority ZO_PU_FILL pass keeps yielding SMs to the forward.
 *   zo_graph_begin(stream)            cudaStreamBeginCapture (thread-local mode)
 *   zo_graph_end(stream, &exec)       end capture, instantiate with node priorities
 *   zo_graph_launch(exec, stream)     replay
 *   zo_graph_destroy(exec)
 */
int zo_graph_begin(void* stream);
/* Asynchronous copy on `stream` (pinned host <-> device, device <-> device);
 * captured as a graph node, so a replayed step carries its own batch upload
 * and record read-back and the host only fills / reads pinned memory. */
int zo_copy_async(void* dst, const void* src, int64_t bytes, void* stream);
int zo_graph_end(void* stream, void** exec_out);
int zo_graph_launch(void* exec, void* stream);
int zo_graph_destroy(void* exec);

/* Tile granularity (elements) the host must use to build tile_prefix. */
int64_t zo_perturb_tile_elems(void);

/*
 * Embedding forward with perturb-on-gather (src/zosim/model.py:300-310):
 * x[b,t,:] = f32(tok[ids[b,t]] + s z) + f32(pos[t] + s z), z keyed by the
 * gathered element's global key.  Only gathered rows are perturbed.
 */
int zo_embed_fwd(const float* tok, int64_t tok_key0, const float* pos, int64_t pos_key0,
                 const int32_t* ids, int64_t batch, int64_t seq, int64_t d, int64_t vocab,
                 double scale, const ZoStepScalars* scal, int32_t zmode,
                 const double* z, int64_t z_key0, float* x, int64_t ldx,
                 int32_t* err_flag, void* stream);

/* LayerNorm over the last dim, eps 1e-5, biased variance, fp32 statistics,
 * bf16 output (src/zosim/model.py:280-283). */
int zo_layernorm_fwd(const float* x, int64_t ldx, const float* gamma, const float* beta,
                     int64_t rows, int64_t d, void* out_bf16, int64_t ldo, void* stream);

/* LayerNorm over stacked +eps / -eps rows: rows >= row_split use gamma2 /
 * beta2 (each direction's perturbed LN parameters). */
int zo_layernorm_fwd_split(const float* x, int64_t ldx, const float* gamma, const float* beta,
                           const float* gamma2, const float* beta2, int64_t rows, int64_t row_split,
                           int64_t d, void* out_bf16, int64_t ldo, void* stream);

/*
 * C[M,N] = A[M,K] (bf16, K-major) x B[K,N] (bf16, N-major = the reference's
 * (d_in, d_out) weight layout, src/zosim/model.py:325) on tcgen05 tensor
 * cores with TMA-fed shared memory and fp32 TMEM accumulators, plus a fused
 * epilogue.  Replaces h @ W + b, the residual adds and GELU of
 * src/zosim/model.py:325-344, and (ZO_EPI_CE) the logits half of loss
 * (src/zosim/model.py:357-372): ce_part[m, tile] = (max, sum exp(l-max)) over
 * the tile's columns and ce_tgt[m] = logit of targets[m].
 * Leading dimensions are in elements and must be multiples of 8.
 */
int zo_gemm_bf16(const void* A, int64_t lda, const void* B, int64_t ldb,
                 int64_t M, int64_t N, int64_t K, int32_t epilogue,
                 const float* bias, void* out, int64_t ldo,
                 const int32_t* targets, float* ce_part, float* ce_tgt,
                 int32_t* err_flag, void* stream);
/*
 * The +eps and -eps forwards of one ZO step as ONE launch ("stacked"): the
 * activations of both directions are stacked as A = [a+; a-] (M rows), rows
 * [0, m_split) multiply B (the +eps shadow) and add bias, rows [m_split, M)
 * multiply B2 / add bias2.  Same kernel, tile schedule and per-tile
 * arithmetic as zo_gemm_bf16 on each half (results are bit-identical); one
 * launch fills twice the tiles, so the partial last wave and the launch
 * prologue / tail are paid once per layer instead of once per direction.
 * m_split must be a multiple of 256 and M > 256 (CTA-pair kernel).
 */
int zo_gemm_bf16_split(const void* A, int64_t lda, const void* B, const void* B2, int64_t ldb,
                       int64_t M, int64_t N, int64_t K, int64_t m_split, int32_t epilogue,
                       const float* bias, const float* bias2, void* out, int64_t ldo,
                       const int32_t* targets, float* ce_part, float* ce_tgt,
                       int32_t* err_flag, void* stream);
/* number of N tiles the ZO_EPI_CE epilogue writes per row for a given N */
int64_t zo_gemm_ce_tiles(int64_t N);

/*
 * fp32 forward of the f32 parity mode (SURVEY.md 8c mode (i)): the same ops
 * as the bf16 production path with every operand and activation in fp32 and
 * accurate expf / tanhf (CUDA-core FFMA; checker-grade, not the hot path).
 *   zo_gemm_f32: C = A[M,K] B[K,N] with ZO_EPI_F32 / BIAS_BF16 (here: fp32
 *     out) / BIAS_GELU_BF16 (fp32 out) / BIAS_RELU_BF16 / BIAS_RESID_F32.
 *   zo_ce_rows_f32: per-row (max, sum exp) and target logit of fp32 logits
 *     written as the CE partials zo_ce_finalize combines (slot 0 of n_tiles).
 */
int zo_gemm_f32(const float* A, int64_t lda, const float* B, int64_t ldb, int64_t M, int64_t N, int64_t K,
                int32_t epilogue, const float* bias, float* out, int64_t ldo, void* stream);
int zo_attn_causal_fwd_f32(const float* qkv, int64_t ldqkv, int64_t batch, int64_t seq, int64_t heads,
                           int64_t head_dim, float* ctx, int64_t ldc, void* stream);
int zo_layernorm_fwd_f32(const float* x, int64_t ldx, const float* gamma, const float* beta, int64_t rows,
                         int64_t d, float* out, int64_t ldo, void* stream);
int zo_ce_rows_f32(const float* logits, int64_t ld, int64_t rows, int64_t vocab, const int32_t* targets,
                   float* ce_part, float* ce_tgt, int64_t n_tiles, int32_t* err_flag, void* stream);

/* Causal exact-softmax attention (src/zosim/model.py:325-332): qkv rows are
 * [q | k | v] (each H*hd wide), out ctx[B*T, H*hd] bf16. */
int zo_attn_causal_fwd(const void* qkv, int64_t ldqkv, int64_t batch, int64_t seq,
                       int64_t heads, int64_t head_dim, void* ctx, int64_t ldc, void* stream);

/* Mean cross-entropy over rows from the ZO_EPI_CE partials, combined and
 * summed in f64 in a fixed order (src/zosim/model.py:366-372). Sets
 * err_flag bit 1 on non-finite logits (-> NumericError). */
int zo_ce_finalize(const float* ce_part, const float* ce_tgt, int64_t rows, int64_t n_tiles,
                   double* loss_out, double* row_scratch /* >= rows */, int32_t* err_flag,
                   void* stream);

/* g = (loss_pos - loss_neg) / (2 eps) (src/zosim/zo.py:80-84); record =
 * {loss_pos, loss_neg, g}; then scal->{seed_prev, lr_g_prev, pending} =
 * {seed_cur, lr*g, 1} so the next zo_perturb_update folds the update in. */
int zo_grad_finalize(const double* loss_pos, const double* loss_neg, double eps, double lr,
                     ZoStepScalars* scal, double* record, void* stream);

/* g from n per-group central differences gathered from the mesh: an ordered
 * ascending sum of (L+_i - L-_i)/(2 eps), divided by n -- the DDP / 2D
 * reduction of src/zosim/strategies.py:145-147, 197-216 with the fixed
 * ascending order of src/zosim/fabric.py:105-113.  L+_i =
 * losses[i*plus_stride + plus_off], L-_i = losses[i*minus_stride + minus_off]
 * (the layout of the rank-ordered all_gather).  record = {L+_mine, L-_mine, g}. */
int zo_grad_finalize_groups(const double* losses, int32_t n_groups, int32_t plus_stride, int32_t plus_off,
                            int32_t minus_stride, int32_t minus_off, int32_t mine, double eps,
                            double lr, ZoStepScalars* scal, double* record, void* stream);

/* 64-bit FNV-style hash of a device buffer (replica-divergence guard that
 * replaces the SHA-256 all_gather of src/zosim/strategies.py:86-89). */
int zo_hash_u64(const void* data, int64_t nbytes, uint64_t* out_dev,
                uint64_t* scratch_dev /* >= 256 words */, void* stream);

/* 16-bit planes of the fp32 master for transfer-compressed offload (SURVEY
 * 8f row 4; no reference counterpart: it replaces the fp32 H2D / D2H of
 * src/zosim/comm.py:314-342 with half the bytes): bits(theta[i]) =
 * hi[i] << 16 | lo[i], exact both ways.  hi (the bf16 truncation) crosses
 * PCIe, lo stays in device memory. */
int zo_planes_join(const uint16_t* hi, const uint16_t* lo, float* theta, int64_t n, void* stream);
int zo_planes_split(const float* theta, uint16_t* hi, uint16_t* lo, int64_t n, void* stream);

/* Debug/test: the Philox direction itself, z[i] for keys e0 .. e0+n-1. */
int zo_philox_normals(uint64_t seed, int64_t e0, int64_t n, float* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* ZO_B200_H_ */
