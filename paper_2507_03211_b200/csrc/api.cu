// extern "C" entry points of libzo_b200.so (declared in include/zo_b200.h).
// Argument validation maps onto the reference's exception classes through
// the ZO_ERR_* codes; kernels live in perturb.cu / ops.cu / attention.cu /
// gemm_tcgen05.cu.
#include <stdarg.h>
#include <stdlib.h>
#include <string.h>

#include <mutex>

#include "common.cuh"

namespace zo {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

// Programmatic dependent launch measured no gain on the step's launch chain
// (profiles/r01_*): kernels keep the griddepcontrol hooks, launches do not set it.
bool pdl_enabled() { return false; }

int num_sms() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!cached[dev]) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cached[dev] = n > 0 ? n : 148;
  }
  return cached[dev];
}

int perturb_update_launch(const PuParams& p, int zmode, cudaStream_t stream);
int philox_normals_launch(uint64_t seed, int64_t e0, int64_t n, float* out, cudaStream_t stream);
int embed_launch(const float*, int64_t, const float*, int64_t, const int32_t*, int64_t, int64_t, int64_t, int64_t,
                 double, const ZoStepScalars*, int32_t, const double*, int64_t, float*, int64_t, int32_t*,
                 cudaStream_t);
int layernorm_launch(const float*, int64_t, const float*, const float*, int64_t, int64_t, __nv_bfloat16*, int64_t,
                     cudaStream_t, const float*, const float*, int64_t);
int attention_launch(const __nv_bfloat16*, int64_t, int64_t, int64_t, int64_t, int64_t, __nv_bfloat16*, int64_t,
                     cudaStream_t);
int ce_finalize_launch(const float*, const float*, int64_t, int64_t, double*, double*, int32_t*, cudaStream_t);
int grad_finalize_launch(const double*, const double*, double, double, ZoStepScalars*, double*, cudaStream_t);
int grad_groups_launch(const double*, int, int, int, int, int, int, double, double, ZoStepScalars*, double*,
                       cudaStream_t);
int hash_launch(const void*, int64_t, uint64_t*, uint64_t*, int, cudaStream_t);
int planes_join_launch(const uint16_t*, const uint16_t*, float*, int64_t, cudaStream_t);
int planes_split_launch(const float*, uint16_t*, uint16_t*, int64_t, cudaStream_t);
int gemm_launch(const void*, int64_t, const void*, int64_t, int64_t, int64_t, int64_t, int, const float*, void*,
                int64_t, const int32_t*, float*, float*, int32_t*, cudaStream_t, const void*, const float*, int64_t);
int64_t perturb_tile_elems();
int64_t gemm_ce_tiles(int64_t N);
int gemm_f32_launch(const float*, int64_t, const float*, int64_t, int64_t, int64_t, int64_t, int, const float*,
                    float*, int64_t, cudaStream_t);
int attn_f32_launch(const float*, int64_t, int64_t, int64_t, int64_t, int64_t, float*, int64_t, cudaStream_t);
int layernorm_f32_launch(const float*, int64_t, const float*, const float*, int64_t, int64_t, float*, int64_t,
                         cudaStream_t);
int ce_rows_f32_launch(const float*, int64_t, int64_t, int64_t, const int32_t*, float*, float*, int64_t, int32_t*,
                       cudaStream_t);

}  // namespace zo

#define ZO_STREAM(s) reinterpret_cast<cudaStream_t>(s)

extern "C" {

const char* zo_version(void) { return "zo_b200 0.1.0 (sm_100a tcgen05/TMA)"; }

const char* zo_last_error(void) { return zo::g_err; }

int zo_device_check(int dev) {
  cudaDeviceProp prop;
  cudaError_t e = cudaGetDeviceProperties(&prop, dev);
  if (e != cudaSuccess) {
    zo::set_error("cudaGetDeviceProperties(%d): %s", dev, cudaGetErrorString(e));
    return ZO_ERR_CUDA;
  }
  if (prop.major != 10 || prop.minor != 0) {
    zo::set_error("device %d is sm_%d%d; this library is built for sm_100a only", dev, prop.major, prop.minor);
    return ZO_ERR_CONFIG;
  }
  return ZO_OK;
}

int64_t zo_perturb_tile_elems(void) { return zo::perturb_tile_elems(); }

int zo_perturb_update(float* theta, int64_t theta_key0, const ZoSegment* segs, const int64_t* tile_prefix,
                      int32_t n_segs, int64_t n_tiles, void* wsh_a, float* vsh_a, void* wsh_b, float* vsh_b,
                      double scale_a, double scale_b, uint32_t flags, const ZoStepScalars* scal, int32_t zmode,
                      const double* z_cur, const double* z_prev, int64_t z_key0, void* stream) {
  ZO_CHECK_ARG(theta && segs && tile_prefix && scal, ZO_ERR_CONFIG, "zo_perturb_update: null argument");
  ZO_CHECK_ARG(n_segs > 0 || n_tiles == 0, ZO_ERR_CONFIG, "zo_perturb_update: no segments");
  ZO_CHECK_ARG(zmode == ZO_Z_PHILOX || zmode == ZO_Z_ORACLE, ZO_ERR_CONFIG, "zo_perturb_update: bad zmode %d", zmode);
  if (zmode == ZO_Z_ORACLE) {
    ZO_CHECK_ARG(!((flags & (ZO_PU_SHADOW_A | ZO_PU_SHADOW_B)) && (scale_a != 0.0 || scale_b != 0.0)) || z_cur,
                 ZO_ERR_CONFIG, "zo_perturb_update: oracle mode needs z_cur");
    ZO_CHECK_ARG(!(flags & ZO_PU_UPDATE) || z_prev, ZO_ERR_CONFIG, "zo_perturb_update: oracle update needs z_prev");
  }
  zo::PuParams p;
  p.theta = theta;
  p.theta_key0 = theta_key0;
  p.segs = segs;
  p.prefix = tile_prefix;
  p.n_segs = n_segs;
  p.n_tiles = n_tiles;
  p.wsh[0] = static_cast<__nv_bfloat16*>(wsh_a);
  p.wsh[1] = static_cast<__nv_bfloat16*>(wsh_b);
  p.vsh[0] = vsh_a;
  p.vsh[1] = vsh_b;
  p.scale[0] = scale_a;
  p.scale[1] = scale_b;
  p.flags = flags;
  p.scal = scal;
  p.z_cur = z_cur;
  p.z_prev = z_prev;
  p.z_key0 = z_key0;
  return zo::perturb_update_launch(p, zmode, ZO_STREAM(stream));
}

int zo_embed_fwd(const float* tok, int64_t tok_key0, const float* pos, int64_t pos_key0, const int32_t* ids,
                 int64_t batch, int64_t seq, int64_t d, int64_t vocab, double scale, const ZoStepScalars* scal,
                 int32_t zmode, const double* z, int64_t z_key0, float* x, int64_t ldx, int32_t* err_flag,
                 void* stream) {
  ZO_CHECK_ARG(tok && pos && ids && x && err_flag, ZO_ERR_CONFIG, "zo_embed_fwd: null argument");
  ZO_CHECK_ARG(ldx >= d, ZO_ERR_CONFIG, "zo_embed_fwd: ldx < d");
  ZO_CHECK_ARG(scale == 0.0 || (zmode == ZO_Z_PHILOX ? scal != nullptr : z != nullptr), ZO_ERR_CONFIG,
               "zo_embed_fwd: perturbation needs a z source");
  return zo::embed_launch(tok, tok_key0, pos, pos_key0, ids, batch, seq, d, vocab, scale, scal, zmode, z, z_key0, x,
                          ldx, err_flag, ZO_STREAM(stream));
}

int zo_layernorm_fwd(const float* x, int64_t ldx, const float* gamma, const float* beta, int64_t rows, int64_t d,
                     void* out_bf16, int64_t ldo, void* stream) {
  ZO_CHECK_ARG(x && gamma && beta && out_bf16, ZO_ERR_CONFIG, "zo_layernorm_fwd: null argument");
  ZO_CHECK_ARG(d > 0 && d <= 49152, ZO_ERR_CONFIG, "zo_layernorm_fwd: d=%lld out of range", (long long)d);
  return zo::layernorm_launch(x, ldx, gamma, beta, rows, d, static_cast<__nv_bfloat16*>(out_bf16), ldo,
                              ZO_STREAM(stream), nullptr, nullptr, 0);
}

int zo_layernorm_fwd_split(const float* x, int64_t ldx, const float* gamma, const float* beta,
                           const float* gamma2, const float* beta2, int64_t rows, int64_t row_split, int64_t d,
                           void* out_bf16, int64_t ldo, void* stream) {
  ZO_CHECK_ARG(x && gamma && beta && gamma2 && beta2 && out_bf16, ZO_ERR_CONFIG,
               "zo_layernorm_fwd_split: null argument");
  ZO_CHECK_ARG(d > 0 && d <= 49152, ZO_ERR_CONFIG, "zo_layernorm_fwd_split: d=%lld out of range", (long long)d);
  ZO_CHECK_ARG(row_split >= 0 && row_split <= rows, ZO_ERR_CONFIG, "zo_layernorm_fwd_split: bad row_split");
  return zo::layernorm_launch(x, ldx, gamma, beta, rows, d, static_cast<__nv_bfloat16*>(out_bf16), ldo,
                              ZO_STREAM(stream), gamma2, beta2, row_split);
}

int zo_gemm_bf16(const void* A, int64_t lda, const void* B, int64_t ldb, int64_t M, int64_t N, int64_t K,
                 int32_t epilogue, const float* bias, void* out, int64_t ldo, const int32_t* targets, float* ce_part,
                 float* ce_tgt, int32_t* err_flag, void* stream) {
  ZO_CHECK_ARG(A && B, ZO_ERR_CONFIG, "zo_gemm_bf16: null operand");
  const int32_t epi = epilogue & ~ZO_GEMM_B_KMAJOR;
  ZO_CHECK_ARG(epi == ZO_EPI_CE ? (targets && ce_part && ce_tgt && err_flag) : (out != nullptr),
               ZO_ERR_CONFIG, "zo_gemm_bf16: missing epilogue buffers");
  ZO_CHECK_ARG(epi == ZO_EPI_F32 || epi == ZO_EPI_CE || bias, ZO_ERR_CONFIG, "zo_gemm_bf16: bias required");
  return zo::gemm_launch(A, lda, B, ldb, M, N, K, epilogue, bias, out, ldo, targets, ce_part, ce_tgt, err_flag,
                         ZO_STREAM(stream), nullptr, nullptr, 0);
}

int zo_gemm_bf16_split(const void* A, int64_t lda, const void* B, const void* B2, int64_t ldb, int64_t M, int64_t N,
                       int64_t K, int64_t m_split, int32_t epilogue, const float* bias, const float* bias2, void* out,
                       int64_t ldo, const int32_t* targets, float* ce_part, float* ce_tgt, int32_t* err_flag,
                       void* stream) {
  ZO_CHECK_ARG(A && B && B2, ZO_ERR_CONFIG, "zo_gemm_bf16_split: null operand");
  const int32_t epi = epilogue & ~ZO_GEMM_B_KMAJOR;
  ZO_CHECK_ARG(epi == ZO_EPI_CE ? (targets && ce_part && ce_tgt && err_flag) : (out != nullptr),
               ZO_ERR_CONFIG, "zo_gemm_bf16_split: missing epilogue buffers");
  ZO_CHECK_ARG(epi == ZO_EPI_F32 || epi == ZO_EPI_CE || (bias && bias2), ZO_ERR_CONFIG,
               "zo_gemm_bf16_split: bias required");
  ZO_CHECK_ARG(m_split > 0, ZO_ERR_CONFIG, "zo_gemm_bf16_split: m_split must be positive");
  return zo::gemm_launch(A, lda, B, ldb, M, N, K, epilogue, bias, out, ldo, targets, ce_part, ce_tgt, err_flag,
                         ZO_STREAM(stream), B2, bias2, m_split);
}

int zo_gemm_f32(const float* A, int64_t lda, const float* B, int64_t ldb, int64_t M, int64_t N, int64_t K,
                int32_t epilogue, const float* bias, float* out, int64_t ldo, void* stream) {
  ZO_CHECK_ARG(A && B && out, ZO_ERR_CONFIG, "zo_gemm_f32: null operand");
  ZO_CHECK_ARG(epilogue == ZO_EPI_F32 || bias, ZO_ERR_CONFIG, "zo_gemm_f32: bias required");
  ZO_CHECK_ARG(lda >= K && ldb >= N && ldo >= N, ZO_ERR_CONFIG, "zo_gemm_f32: leading dimension too small");
  return zo::gemm_f32_launch(A, lda, B, ldb, M, N, K, epilogue, bias, out, ldo, ZO_STREAM(stream));
}

int zo_attn_causal_fwd_f32(const float* qkv, int64_t ldqkv, int64_t batch, int64_t seq, int64_t heads,
                           int64_t head_dim, float* ctx, int64_t ldc, void* stream) {
  ZO_CHECK_ARG(qkv && ctx, ZO_ERR_CONFIG, "zo_attn_causal_fwd_f32: null argument");
  ZO_CHECK_ARG(head_dim >= 1 && head_dim <= 128, ZO_ERR_CONFIG, "zo_attn_causal_fwd_f32: head_dim %lld > 128",
               (long long)head_dim);
  return zo::attn_f32_launch(qkv, ldqkv, batch, seq, heads, head_dim, ctx, ldc, ZO_STREAM(stream));
}

int zo_layernorm_fwd_f32(const float* x, int64_t ldx, const float* gamma, const float* beta, int64_t rows,
                         int64_t d, float* out, int64_t ldo, void* stream) {
  ZO_CHECK_ARG(x && gamma && beta && out, ZO_ERR_CONFIG, "zo_layernorm_fwd_f32: null argument");
  return zo::layernorm_f32_launch(x, ldx, gamma, beta, rows, d, out, ldo, ZO_STREAM(stream));
}

int zo_ce_rows_f32(const float* logits, int64_t ld, int64_t rows, int64_t vocab, const int32_t* targets,
                   float* ce_part, float* ce_tgt, int64_t n_tiles, int32_t* err_flag, void* stream) {
  ZO_CHECK_ARG(logits && targets && ce_part && ce_tgt && err_flag, ZO_ERR_CONFIG, "zo_ce_rows_f32: null argument");
  ZO_CHECK_ARG(n_tiles >= 1, ZO_ERR_CONFIG, "zo_ce_rows_f32: n_tiles must be >= 1");
  return zo::ce_rows_f32_launch(logits, ld, rows, vocab, targets, ce_part, ce_tgt, n_tiles, err_flag,
                                ZO_STREAM(stream));
}

int64_t zo_gemm_ce_tiles(int64_t N) { return zo::gemm_ce_tiles(N); }

int zo_attn_causal_fwd(const void* qkv, int64_t ldqkv, int64_t batch, int64_t seq, int64_t heads, int64_t head_dim,
                       void* ctx, int64_t ldc, void* stream) {
  ZO_CHECK_ARG(qkv && ctx, ZO_ERR_CONFIG, "zo_attn_causal_fwd: null argument");
  ZO_CHECK_ARG(ldqkv >= 3 * heads * head_dim && ldc >= heads * head_dim, ZO_ERR_CONFIG,
               "zo_attn_causal_fwd: leading dimension too small");
  return zo::attention_launch(static_cast<const __nv_bfloat16*>(qkv), ldqkv, batch, seq, heads, head_dim,
                              static_cast<__nv_bfloat16*>(ctx), ldc, ZO_STREAM(stream));
}

int zo_ce_finalize(const float* ce_part, const float* ce_tgt, int64_t rows, int64_t n_tiles, double* loss_out,
                   double* row_scratch, int32_t* err_flag, void* stream) {
  ZO_CHECK_ARG(ce_part && ce_tgt && loss_out && row_scratch && err_flag, ZO_ERR_CONFIG,
               "zo_ce_finalize: null argument");
  return zo::ce_finalize_launch(ce_part, ce_tgt, rows, n_tiles, loss_out, row_scratch, err_flag, ZO_STREAM(stream));
}

int zo_grad_finalize(const double* loss_pos, const double* loss_neg, double eps, double lr, ZoStepScalars* scal,
                     double* record, void* stream) {
  ZO_CHECK_ARG(eps != 0.0, ZO_ERR_NUMERIC, "epsilon must be nonzero");
  ZO_CHECK_ARG(loss_pos && loss_neg && scal && record, ZO_ERR_CONFIG, "zo_grad_finalize: null argument");
  return zo::grad_finalize_launch(loss_pos, loss_neg, eps, lr, scal, record, ZO_STREAM(stream));
}

int zo_grad_finalize_groups(const double* losses, int32_t n_groups, int32_t plus_stride, int32_t plus_off,
                            int32_t minus_stride, int32_t minus_off, int32_t mine, double eps, double lr,
                            ZoStepScalars* scal, double* record, void* stream) {
  ZO_CHECK_ARG(eps != 0.0, ZO_ERR_NUMERIC, "epsilon must be nonzero");
  ZO_CHECK_ARG(losses && scal && record && n_groups > 0 && mine >= 0 && mine < n_groups, ZO_ERR_CONFIG,
               "zo_grad_finalize_groups: bad argument");
  return zo::grad_groups_launch(losses, n_groups, plus_stride, plus_off, minus_stride, minus_off, mine, eps, lr,
                                scal, record, ZO_STREAM(stream));
}

int zo_hash_u64(const void* data, int64_t nbytes, uint64_t* out_dev, uint64_t* scratch_dev, void* stream) {
  ZO_CHECK_ARG(data && out_dev && scratch_dev && nbytes >= 0, ZO_ERR_CONFIG, "zo_hash_u64: bad argument");
  return zo::hash_launch(data, nbytes, out_dev, scratch_dev, 256, ZO_STREAM(stream));
}

int zo_planes_join(const uint16_t* hi, const uint16_t* lo, float* theta, int64_t n, void* stream) {
  ZO_CHECK_ARG(n >= 0 && (n == 0 || (hi && lo && theta)), ZO_ERR_CONFIG, "zo_planes_join: bad argument");
  return zo::planes_join_launch(hi, lo, theta, n, ZO_STREAM(stream));
}

int zo_planes_split(const float* theta, uint16_t* hi, uint16_t* lo, int64_t n, void* stream) {
  ZO_CHECK_ARG(n >= 0 && (n == 0 || (hi && lo && theta)), ZO_ERR_CONFIG, "zo_planes_split: bad argument");
  return zo::planes_split_launch(theta, hi, lo, n, ZO_STREAM(stream));
}

int zo_philox_normals(uint64_t seed, int64_t e0, int64_t n, float* out, void* stream) {
  ZO_CHECK_ARG(out || n == 0, ZO_ERR_CONFIG, "zo_philox_normals: null output");
  return zo::philox_normals_launch(seed, e0, n, out, ZO_STREAM(stream));
}

int zo_copy_async(void* dst, const void* src, int64_t bytes, void* stream) {
  ZO_CHECK_ARG(bytes >= 0 && (bytes == 0 || (dst && src)), ZO_ERR_CONFIG, "zo_copy_async: bad argument");
  if (bytes) ZO_CUDA_TRY(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDefault, ZO_STREAM(stream)));
  return ZO_OK;
}

int zo_graph_begin(void* stream) {
  ZO_CUDA_TRY(cudaStreamBeginCapture(ZO_STREAM(stream), cudaStreamCaptureModeThreadLocal));
  return ZO_OK;
}

int zo_graph_end(void* stream, void** exec_out) {
  ZO_CHECK_ARG(exec_out, ZO_ERR_CONFIG, "zo_graph_end: null output");
  cudaGraph_t g = nullptr;
  ZO_CUDA_TRY(cudaStreamEndCapture(ZO_STREAM(stream), &g));
  cudaGraphExec_t ex = nullptr;
  const cudaError_t e = cudaGraphInstantiateWithFlags(&ex, g, cudaGraphInstantiateFlagUseNodePriority);
  cudaGraphDestroy(g);
  ZO_CUDA_TRY(e);
  *exec_out = ex;
  return ZO_OK;
}

int zo_graph_launch(void* exec, void* stream) {
  ZO_CHECK_ARG(exec, ZO_ERR_CONFIG, "zo_graph_launch: null graph");
  ZO_CUDA_TRY(cudaGraphLaunch(static_cast<cudaGraphExec_t>(exec), ZO_STREAM(stream)));
  return ZO_OK;
}

int zo_graph_destroy(void* exec) {
  if (exec) ZO_CUDA_TRY(cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(exec)));
  return ZO_OK;
}

}  // extern "C"
