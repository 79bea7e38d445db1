// Row-wise forward ops of the zosim decoder block and the step's scalar tail.
//   embedding gather (model.py:300-310) with perturb-on-gather
//   LayerNorm (model.py:280-283)
//   cross-entropy finalize (model.py:357-372), projected gradient (zo.py:80-84)
//   replica hash (strategies.py:86-89 guard)
#include "common.cuh"

namespace zo {

// ---------------------------------------------------------------------------
// embedding: x = f32(tok[id] + s z) + f32(pos[t] + s z)
// ---------------------------------------------------------------------------
template <int ZMODE>
__global__ void embed_kernel(const float* __restrict__ tok, int64_t tok_key0,
                             const float* __restrict__ pos, int64_t pos_key0,
                             const int32_t* __restrict__ ids, int64_t seq, int64_t d, int64_t vocab,
                             double scale, const ZoStepScalars* scal, const double* z, int64_t z_key0,
                             float* __restrict__ x, int64_t ldx, int32_t* err, bool vec) {
  pdl_trigger();
  pdl_wait();
  const int64_t m = blockIdx.x;
  const int64_t t = m % seq;
  int64_t id = ids[m];
  if (id < 0 || id >= vocab) {
    if (threadIdx.x == 0) atomicOr(err, 4);
    id = 0;
  }
  const uint64_t seed = scal ? scal->seed_cur : 0ull;
  const float s32 = (float)scale;
  if constexpr (ZMODE == ZO_Z_PHILOX) {
    if (vec) {
      // 4 consecutive elements per thread = one Philox4x32 counter (keys
      // 4-aligned): one generator call per 4 outputs instead of per output,
      // the same z values and arithmetic as the scalar loop below
      const int64_t kt0 = tok_key0 + id * d, kp0 = pos_key0 + t * d;
      for (int64_t c = 4 * (int64_t)threadIdx.x; c < d; c += 4 * (int64_t)blockDim.x) {
        float4 a = *reinterpret_cast<const float4*>(tok + id * d + c);
        float4 b = *reinterpret_cast<const float4*>(pos + t * d + c);
        if (scale != 0.0) {
          const f32x4 za = philox_normal4(seed, (uint64_t)(kt0 + c) >> 2);
          const f32x4 zb = philox_normal4(seed, (uint64_t)(kp0 + c) >> 2);
          a.x = fmaf(s32, za.x, a.x); a.y = fmaf(s32, za.y, a.y); a.z = fmaf(s32, za.z, a.z); a.w = fmaf(s32, za.w, a.w);
          b.x = fmaf(s32, zb.x, b.x); b.y = fmaf(s32, zb.y, b.y); b.z = fmaf(s32, zb.z, b.z); b.w = fmaf(s32, zb.w, b.w);
        }
        *reinterpret_cast<float4*>(x + m * ldx + c) =
            make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z), __fadd_rn(a.w, b.w));
      }
      return;
    }
  }
  for (int64_t c = threadIdx.x; c < d; c += blockDim.x) {
    const int64_t kt = tok_key0 + id * d + c, kp = pos_key0 + t * d + c;
    float a = tok[id * d + c], b = pos[t * d + c];
    if (scale != 0.0) {
      if constexpr (ZMODE == ZO_Z_PHILOX) {
        a = fmaf(s32, philox_normal1(seed, (uint64_t)kt), a);
        b = fmaf(s32, philox_normal1(seed, (uint64_t)kp), b);
      } else {
        a = __double2float_rn(__dadd_rn((double)a, __dmul_rn(scale, z[kt - z_key0])));
        b = __double2float_rn(__dadd_rn((double)b, __dmul_rn(scale, z[kp - z_key0])));
      }
    }
    x[m * ldx + c] = __fadd_rn(a, b);
  }
}

int embed_launch(const float* tok, int64_t tok_key0, const float* pos, int64_t pos_key0,
                 const int32_t* ids, int64_t batch, int64_t seq, int64_t d, int64_t vocab,
                 double scale, const ZoStepScalars* scal, int32_t zmode, const double* z,
                 int64_t z_key0, float* x, int64_t ldx, int32_t* err, cudaStream_t st) {
  const int64_t rows = batch * seq;
  if (rows == 0) return ZO_OK;
  const bool vec = zmode == ZO_Z_PHILOX && d % 4 == 0 && tok_key0 % 4 == 0 && pos_key0 % 4 == 0 && ldx % 4 == 0 &&
                   ((reinterpret_cast<uintptr_t>(tok) | reinterpret_cast<uintptr_t>(pos) |
                     reinterpret_cast<uintptr_t>(x)) & 15) == 0;
  const int64_t lanes = vec ? d / 4 : d;
  const int threads = lanes >= 256 ? 256 : (int)((lanes + 31) / 32 * 32);
  if (zmode == ZO_Z_PHILOX)
    launch_k(embed_kernel<ZO_Z_PHILOX>, dim3((unsigned)rows), dim3(threads), 0, st, tok, tok_key0, pos, pos_key0, ids,
             seq, d, vocab, scale, scal, z, z_key0, x, ldx, err, vec);
  else
    launch_k(embed_kernel<ZO_Z_ORACLE>, dim3((unsigned)rows), dim3(threads), 0, st, tok, tok_key0, pos, pos_key0, ids,
             seq, d, vocab, scale, scal, z, z_key0, x, ldx, err, false);
  return launch_status("embed_kernel");
}

// ---------------------------------------------------------------------------
// LayerNorm: one CTA per row, row cached in shared memory, fp32 two-pass stats
// ---------------------------------------------------------------------------
__device__ __forceinline__ float block_sum(float v, float* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float tot = 0.f;
  for (int i = 0; i < nw; ++i) tot += red[i];   // fixed order: deterministic
  return tot;
}

__global__ void layernorm_kernel(const float* __restrict__ x, int64_t ldx, const float* __restrict__ g,
                                 const float* __restrict__ b, int64_t d, __nv_bfloat16* __restrict__ out,
                                 int64_t ldo, const float* __restrict__ g2, const float* __restrict__ b2,
                                 int64_t row_split) {
  extern __shared__ float srow[];
  if (row_split && (int64_t)blockIdx.x >= row_split) { g = g2; b = b2; }   // stacked +eps / -eps rows
  __shared__ float red[32];
  pdl_trigger();
  pdl_wait();
  const float* xr = x + blockIdx.x * ldx;
  float s = 0.f;
  for (int64_t c = threadIdx.x; c < d; c += blockDim.x) {
    const float v = xr[c];
    srow[c] = v;
    s += v;
  }
  const float mu = block_sum(s, red) / (float)d;
  float q = 0.f;
  for (int64_t c = threadIdx.x; c < d; c += blockDim.x) {
    const float dv = srow[c] - mu;
    q += dv * dv;
  }
  const float var = block_sum(q, red) / (float)d;
  const float rstd = 1.0f / sqrtf(var + 1e-5f);
  __nv_bfloat16* orow = out + blockIdx.x * ldo;
  for (int64_t c = threadIdx.x; c < d; c += blockDim.x)
    orow[c] = __float2bfloat16_rn(fmaf((srow[c] - mu) * rstd, g[c], b[c]));
}

// Wide rows (4096 < d <= 1024 NV: the 13B / 66B / 175B widths): one CTA of 256
// threads per row, NV float4 per thread kept in registers (one pass over
// memory), the two statistics by warp shuffles + a fixed-order sum of the 8
// warp partials.  (The smem kernel above re-reads the row from shared memory
// and ran at ~0.2 of HBM at d = 5120.)
template <int NV>
__global__ void __launch_bounds__(256) layernorm_row_kernel(const float* __restrict__ x, int64_t ldx,
                                                            const float* __restrict__ g,
                                                            const float* __restrict__ b, int d,
                                                            __nv_bfloat16* __restrict__ out, int64_t ldo,
                                                            const float* __restrict__ g2,
                                                            const float* __restrict__ b2, int64_t row_split) {
  __shared__ float red[8];
  pdl_trigger();
  pdl_wait();
  const int64_t r = blockIdx.x;
  if (row_split && r >= row_split) { g = g2; b = b2; }   // stacked +eps / -eps rows
  const float4* xr = reinterpret_cast<const float4*>(x + r * ldx);
  float4 v[NV];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = (i * 256 + threadIdx.x) * 4;
    v[i] = c < d ? xr[i * 256 + threadIdx.x] : make_float4(0.f, 0.f, 0.f, 0.f);
    s += (v[i].x + v[i].y) + (v[i].z + v[i].w);
  }
  const float mu = block_sum(s, red) / (float)d;
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = (i * 256 + threadIdx.x) * 4;
    if (c < d) {
      const float a0 = v[i].x - mu, a1 = v[i].y - mu, a2 = v[i].z - mu, a3 = v[i].w - mu;
      q += (a0 * a0 + a1 * a1) + (a2 * a2 + a3 * a3);
    }
  }
  const float rstd = 1.0f / sqrtf(block_sum(q, red) / (float)d + 1e-5f);
  __nv_bfloat16* orow = out + r * ldo;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = (i * 256 + threadIdx.x) * 4;
    if (c < d) {
      const float4 gg = *reinterpret_cast<const float4*>(g + c);
      const float4 bb = *reinterpret_cast<const float4*>(b + c);
      __nv_bfloat162 lo = __floats2bfloat162_rn(fmaf((v[i].x - mu) * rstd, gg.x, bb.x),
                                                fmaf((v[i].y - mu) * rstd, gg.y, bb.y));
      __nv_bfloat162 hi = __floats2bfloat162_rn(fmaf((v[i].z - mu) * rstd, gg.z, bb.z),
                                                fmaf((v[i].w - mu) * rstd, gg.w, bb.w));
      uint2 pk;
      pk.x = *reinterpret_cast<uint32_t*>(&lo);
      pk.y = *reinterpret_cast<uint32_t*>(&hi);
      *reinterpret_cast<uint2*>(orow + c) = pk;
    }
  }
}

// Warp-per-row variant for d <= 32*4*NV: the row lives in registers as float4,
// statistics via warp shuffles only (no block barriers); 8 rows per CTA.
template <int NV>
__global__ void __launch_bounds__(256) layernorm_warp_kernel(const float* __restrict__ x, int64_t ldx,
                                                              const float* __restrict__ g,
                                                              const float* __restrict__ b, int64_t rows, int d,
                                                              __nv_bfloat16* __restrict__ out, int64_t ldo,
                                                              const float* __restrict__ g2,
                                                              const float* __restrict__ b2, int64_t row_split) {
  pdl_trigger();
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int64_t warp_g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp_g; r < rows; r += nwarps) {
    const float4* xr = reinterpret_cast<const float4*>(x + r * ldx);
    float4 v[NV];
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c = (i * 32 + lane) * 4;
      v[i] = c < d ? xr[i * 32 + lane] : make_float4(0.f, 0.f, 0.f, 0.f);
      s += (v[i].x + v[i].y) + (v[i].z + v[i].w);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const float mu = s / (float)d;
    float q = 0.f;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c = (i * 32 + lane) * 4;
      if (c < d) {
        const float a0 = v[i].x - mu, a1 = v[i].y - mu, a2 = v[i].z - mu, a3 = v[i].w - mu;
        q += (a0 * a0 + a1 * a1) + (a2 * a2 + a3 * a3);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
    const float rstd = 1.0f / sqrtf(q / (float)d + 1e-5f);
    __nv_bfloat16* orow = out + r * ldo;
    const bool second = row_split && r >= row_split;      // stacked +eps / -eps rows
    const float* gr = second ? g2 : g;
    const float* br = second ? b2 : b;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c = (i * 32 + lane) * 4;
      if (c < d) {
        const float4 gg = *reinterpret_cast<const float4*>(gr + c);
        const float4 bb = *reinterpret_cast<const float4*>(br + c);
        __nv_bfloat162 lo = __floats2bfloat162_rn(fmaf((v[i].x - mu) * rstd, gg.x, bb.x),
                                                  fmaf((v[i].y - mu) * rstd, gg.y, bb.y));
        __nv_bfloat162 hi = __floats2bfloat162_rn(fmaf((v[i].z - mu) * rstd, gg.z, bb.z),
                                                  fmaf((v[i].w - mu) * rstd, gg.w, bb.w));
        uint2 pk;
        pk.x = *reinterpret_cast<uint32_t*>(&lo);
        pk.y = *reinterpret_cast<uint32_t*>(&hi);
        *reinterpret_cast<uint2*>(orow + c) = pk;
      }
    }
  }
}

int layernorm_launch(const float* x, int64_t ldx, const float* g, const float* b, int64_t rows, int64_t d,
                     __nv_bfloat16* out, int64_t ldo, cudaStream_t st, const float* g2, const float* b2,
                     int64_t row_split) {
  if (rows == 0) return ZO_OK;
  if (!row_split) { g2 = g; b2 = b; }
  const bool vec = (d % 4 == 0) && (ldx % 4 == 0) && (ldo % 4 == 0) &&
                   ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(g) | reinterpret_cast<uintptr_t>(b) |
                     reinterpret_cast<uintptr_t>(g2) | reinterpret_cast<uintptr_t>(b2)) & 15) == 0 &&
                   ((reinterpret_cast<uintptr_t>(out) & 7) == 0);
  if (vec && d <= 4096) {
    const int64_t want = (rows + 7) / 8;
    const int grid = (int)(want < (int64_t)num_sms() * 8 ? want : (int64_t)num_sms() * 8);
    const int nv = (int)((d + 127) / 128);
#define ZO_LN_CASE(N)                                                                                   \
  if (nv <= N) {                                                                                        \
    launch_k(layernorm_warp_kernel<N>, dim3(grid), dim3(256), 0, st, x, ldx, g, b, rows, (int)d, out, ldo,  \
             g2, b2, row_split);                                                                        \
    return launch_status("layernorm_warp_kernel");                                                      \
  }
    ZO_LN_CASE(1) ZO_LN_CASE(2) ZO_LN_CASE(4) ZO_LN_CASE(8) ZO_LN_CASE(16) ZO_LN_CASE(32)
#undef ZO_LN_CASE
  }
  if (vec && d <= 12288) {
    const int nv = (int)((d + 1023) / 1024);
#define ZO_LN_ROW(N)                                                                                  \
  if (nv <= N) {                                                                                      \
    launch_k(layernorm_row_kernel<N>, dim3((unsigned)rows), dim3(256), 0, st, x, ldx, g, b, (int)d, out, ldo, \
             g2, b2, row_split);                                                                      \
    return launch_status("layernorm_row_kernel");                                                     \
  }
    ZO_LN_ROW(5) ZO_LN_ROW(6) ZO_LN_ROW(8) ZO_LN_ROW(9) ZO_LN_ROW(10) ZO_LN_ROW(12)
#undef ZO_LN_ROW
  }
  const size_t smem = (size_t)d * sizeof(float);
  static bool big_smem = false;
  if (smem + 256 > 48 * 1024 && !big_smem) {
    cudaFuncSetAttribute(layernorm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    big_smem = true;
  }
  const int threads = d >= 1024 ? 512 : (d >= 256 ? 256 : 64);
  launch_k(layernorm_kernel, dim3((unsigned)rows), dim3(threads), smem, st, x, ldx, g, b, d, out, ldo, g2, b2,
           row_split);
  return launch_status("layernorm_kernel");
}

// ---------------------------------------------------------------------------
// cross-entropy finalize: per row combine the N-tile partials (fixed order),
// then a single-CTA fixed-order f64 mean -- bit-stable run to run.
// ---------------------------------------------------------------------------
// One warp per row: lanes stride the row's (max, sum-exp) tile partials
// (coalesced 8-B pairs), then fixed-shape xor-shuffle trees combine them,
// so the result is deterministic run to run.
__global__ void ce_rows_kernel(const float* __restrict__ part, const float* __restrict__ tgt, int64_t rows,
                               int64_t n_tiles, double* __restrict__ row_loss, int32_t* err) {
  pdl_trigger();
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int64_t r = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= rows) return;
  const float2* p = reinterpret_cast<const float2*>(part + r * n_tiles * 2);
  double m = -INFINITY;
  bool bad = false;
  for (int64_t i = lane; i < n_tiles; i += 32) {
    const float2 v = p[i];
    if (v.x == -INFINITY && v.y == 0.f) continue;   // empty (out-of-range) partial
    if (!isfinite(v.x)) bad = true;
    m = fmax(m, (double)v.x);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  double s = 0.0;
  for (int64_t i = lane; i < n_tiles; i += 32) {
    const float2 v = p[i];
    if (v.x == -INFINITY && v.y == 0.f) continue;
    if (!isfinite(v.y)) bad = true;
    s += (double)v.y * exp((double)v.x - m);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  bad = __any_sync(0xffffffffu, bad);
  if (lane == 0) {
    const float tl = tgt[r];
    if (!isfinite(tl)) bad = true;
    if (bad) atomicOr(err, 2);
    row_loss[r] = bad ? (double)NAN : m + log(s) - (double)tl;   // a flagged row poisons the mean (gate below)
  }
}

__global__ void mean_f64_kernel(const double* __restrict__ v, int64_t n, double* out) {
  __shared__ double red[1024];
  pdl_trigger();
  pdl_wait();
  double s = 0.0;
  // contiguous chunk per thread, then a fixed-shape tree: deterministic
  const int64_t per = (n + blockDim.x - 1) / blockDim.x;
  const int64_t lo = threadIdx.x * per, hi = min(lo + per, n);
  for (int64_t i = lo; i < hi; ++i) s += v[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int st = blockDim.x / 2; st > 0; st >>= 1) {
    if ((int)threadIdx.x < st) red[threadIdx.x] += red[threadIdx.x + st];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = red[0] / (double)n;
}

int ce_finalize_launch(const float* part, const float* tgt, int64_t rows, int64_t n_tiles, double* loss,
                       double* row_scratch, int32_t* err, cudaStream_t st) {
  if (rows == 0) return ZO_OK;
  launch_k(ce_rows_kernel, dim3((unsigned)((rows + 7) / 8)), dim3(256), 0, st, part, tgt, rows, n_tiles,
           row_scratch, err);
  launch_k(mean_f64_kernel, dim3(1), dim3(1024), 0, st, (const double*)row_scratch, rows, loss);
  return launch_status("ce_finalize");
}

// ---------------------------------------------------------------------------
// projected gradient + scalar state for the folded update
// ---------------------------------------------------------------------------
// The deferred update is armed only for a finite g: a step whose losses are
// non-finite (the CE kernels flag the rows and write NaN) leaves pending = 0
// and lr_g_prev = 0, so the next fused pass / the eager update pass is a
// value no-op and the master never sees theta -= NaN * z.  The host raises
// NumericError from the workspace flag after the step (model.py:366-367).
__device__ __forceinline__ void arm_update(ZoStepScalars* scal, double lr, double g) {
  const bool ok = isfinite(g) && isfinite(lr * g);
  scal->seed_prev = scal->seed_cur;
  scal->lr_g_prev = ok ? lr * g : 0.0;
  scal->pending = ok ? 1 : 0;
}

__global__ void grad_finalize_kernel(const double* lp, const double* ln, double eps, double lr,
                                     ZoStepScalars* scal, double* rec) {
  pdl_wait();
  const double a = *lp, b = *ln;
  const double g = (a - b) / (2.0 * eps);
  rec[0] = a; rec[1] = b; rec[2] = g;
  arm_update(scal, lr, g);
}

__global__ void grad_groups_kernel(const double* losses, int n, int sp, int op, int sm, int om, int mine,
                                   double eps, double lr, ZoStepScalars* scal, double* rec) {
  pdl_wait();
  double tot = 0.0;
  for (int i = 0; i < n; ++i) tot += (losses[i * sp + op] - losses[i * sm + om]) / (2.0 * eps);
  const double g = tot / (double)n;
  rec[0] = losses[mine * sp + op]; rec[1] = losses[mine * sm + om]; rec[2] = g;
  arm_update(scal, lr, g);
}

int grad_finalize_launch(const double* lp, const double* ln, double eps, double lr, ZoStepScalars* scal,
                         double* rec, cudaStream_t st) {
  launch_k(grad_finalize_kernel, dim3(1), dim3(1), 0, st, lp, ln, eps, lr, scal, rec);
  return launch_status("grad_finalize_kernel");
}

int grad_groups_launch(const double* losses, int n, int sp, int op, int sm, int om, int mine, double eps, double lr,
                       ZoStepScalars* scal, double* rec, cudaStream_t st) {
  launch_k(grad_groups_kernel, dim3(1), dim3(1), 0, st, losses, n, sp, op, sm, om, mine, eps, lr, scal, rec);
  return launch_status("grad_groups_kernel");
}

// ---------------------------------------------------------------------------
// replica hash: per-CTA FNV-1a-style mix of 8-byte words, combined in order
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t mix64(uint64_t h, uint64_t v) {
  h ^= v + 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2);
  h *= 0x100000001B3ull;
  return h;
}

__global__ void hash_partial_kernel(const uint8_t* __restrict__ p, int64_t nbytes, uint64_t* partial) {
  __shared__ uint64_t red[256];
  const int64_t nblk = gridDim.x;
  const int64_t chunk = ((nbytes + nblk - 1) / nblk + 7) & ~int64_t(7);
  const int64_t lo = blockIdx.x * chunk, hi = min(lo + chunk, nbytes);
  uint64_t h = 0xcbf29ce484222325ull ^ (uint64_t)threadIdx.x;
  for (int64_t i = lo + threadIdx.x * 8; i < hi; i += blockDim.x * 8) {
    uint64_t w = 0;
    if (i + 8 <= hi) w = *reinterpret_cast<const uint64_t*>(p + i);
    else for (int64_t j = i; j < hi; ++j) w |= (uint64_t)p[j] << (8 * (j - i));
    h = mix64(h, w ^ (uint64_t)i);
  }
  red[threadIdx.x] = h;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t acc = 0x84222325cbf29ce4ull;
    for (int i = 0; i < (int)blockDim.x; ++i) acc = mix64(acc, red[i]);
    partial[blockIdx.x] = acc;
  }
}

__global__ void hash_final_kernel(const uint64_t* partial, int n, uint64_t* out) {
  uint64_t acc = 0x1234567887654321ull;
  for (int i = 0; i < n; ++i) acc = mix64(acc, partial[i]);
  *out = acc;
}

// ---------------------------------------------------------------------------
// 16-bit planes of the fp32 master (transfer compression):
// bits(theta) = hi << 16 | lo.  The hi plane (the bf16 truncation of theta)
// crosses PCIe; the lo plane stays in HBM; join / split are exact.  HBM-bound
// elementwise passes, 8 elements per thread when all three pointers are
// 16-byte aligned, a scalar grid-stride loop otherwise.
// ---------------------------------------------------------------------------
__global__ void planes_join_kernel(const uint16_t* __restrict__ hi, const uint16_t* __restrict__ lo,
                                   uint32_t* __restrict__ out, int64_t n, bool vec) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  int64_t done = 0;
  if (vec) {
    const int64_t n8 = n >> 3;
    for (int64_t i = tid; i < n8; i += nth) {
      const uint4 h = reinterpret_cast<const uint4*>(hi)[i];
      const uint4 l = reinterpret_cast<const uint4*>(lo)[i];
      const uint32_t hw[4] = {h.x, h.y, h.z, h.w}, lw[4] = {l.x, l.y, l.z, l.w};
      uint32_t o[8];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        o[2 * j] = (hw[j] << 16) | (lw[j] & 0xFFFFu);
        o[2 * j + 1] = (hw[j] & 0xFFFF0000u) | (lw[j] >> 16);
      }
      reinterpret_cast<uint4*>(out)[2 * i] = make_uint4(o[0], o[1], o[2], o[3]);
      reinterpret_cast<uint4*>(out)[2 * i + 1] = make_uint4(o[4], o[5], o[6], o[7]);
    }
    done = n8 << 3;
  }
  for (int64_t i = done + tid; i < n; i += nth) out[i] = ((uint32_t)hi[i] << 16) | lo[i];
}

__global__ void planes_split_kernel(const uint32_t* __restrict__ in, uint16_t* __restrict__ hi,
                                    uint16_t* __restrict__ lo, int64_t n, bool vec) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  int64_t done = 0;
  if (vec) {
    const int64_t n8 = n >> 3;
    for (int64_t i = tid; i < n8; i += nth) {
      const uint4 a = reinterpret_cast<const uint4*>(in)[2 * i];
      const uint4 b = reinterpret_cast<const uint4*>(in)[2 * i + 1];
      const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
      uint32_t h[4], l[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        h[j] = (w[2 * j] >> 16) | (w[2 * j + 1] & 0xFFFF0000u);
        l[j] = (w[2 * j] & 0xFFFFu) | (w[2 * j + 1] << 16);
      }
      reinterpret_cast<uint4*>(hi)[i] = make_uint4(h[0], h[1], h[2], h[3]);
      reinterpret_cast<uint4*>(lo)[i] = make_uint4(l[0], l[1], l[2], l[3]);
    }
    done = n8 << 3;
  }
  for (int64_t i = done + tid; i < n; i += nth) {
    const uint32_t w = in[i];
    hi[i] = (uint16_t)(w >> 16);
    lo[i] = (uint16_t)(w & 0xFFFFu);
  }
}

static int planes_grid(int64_t n) {
  const int64_t want = (n / 8 + 255) / 256;
  const int64_t cap = (int64_t)num_sms() * 8;
  return (int)(want < 1 ? 1 : (want < cap ? want : cap));
}

int planes_join_launch(const uint16_t* hi, const uint16_t* lo, float* out, int64_t n, cudaStream_t st) {
  if (n == 0) return ZO_OK;
  const bool vec = ((reinterpret_cast<uintptr_t>(hi) | reinterpret_cast<uintptr_t>(lo) |
                     reinterpret_cast<uintptr_t>(out)) & 15) == 0;
  planes_join_kernel<<<planes_grid(n), 256, 0, st>>>(hi, lo, reinterpret_cast<uint32_t*>(out), n, vec);
  return launch_status("planes_join");
}

int planes_split_launch(const float* in, uint16_t* hi, uint16_t* lo, int64_t n, cudaStream_t st) {
  if (n == 0) return ZO_OK;
  const bool vec = ((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(hi) |
                     reinterpret_cast<uintptr_t>(lo)) & 15) == 0;
  planes_split_kernel<<<planes_grid(n), 256, 0, st>>>(reinterpret_cast<const uint32_t*>(in), hi, lo, n, vec);
  return launch_status("planes_split");
}

int hash_launch(const void* data, int64_t nbytes, uint64_t* out, uint64_t* scratch, int nblk, cudaStream_t st) {
  const bool aligned = (reinterpret_cast<uintptr_t>(data) & 7) == 0;
  if (!aligned) { set_error("zo_hash_u64: buffer must be 8-byte aligned"); return ZO_ERR_CONFIG; }
  hash_partial_kernel<<<nblk, 256, 0, st>>>(static_cast<const uint8_t*>(data), nbytes, scratch);
  hash_final_kernel<<<1, 1, 0, st>>>(scratch, nblk, out);
  return launch_status("hash");
}

}  // namespace zo
