// Causal exact-softmax attention of the zosim block (src/zosim/model.py:325-332):
//   scores = q k^T / sqrt(hd), -inf above the diagonal, max-subtracted softmax, @ v.
// qkv is the fused QKV GEMM output: row m = b*T + t holds [q | k | v], each H*hd wide.
//
// Dispatch:
//  * hd 64  -> attn_pp_kernel (attention_tc.cu): tcgen05, two query tiles in
//              flight per CTA (the OPT-125M .. 2.7B shapes, the headline)
//  * hd 128 -> attn_tc_kernel<128> (attention_tc.cu): tcgen05 (OPT-6.7B .. 175B)
//  * other head dims / unaligned operands -> attn_simt_kernel below: warp per
//    query, fp32 throughout (the small shapes of the parity suite)
#include <stdlib.h>

#include "common.cuh"

namespace zo {

// ------------------------------- SIMT path ---------------------------------
__global__ void attn_simt_kernel(const __nv_bfloat16* __restrict__ qkv, int64_t ldq, int seq, int heads,
                                 int hd, __nv_bfloat16* __restrict__ ctx, int64_t ldc, float scale) {
  extern __shared__ float sbuf[];  // per warp: seq scores
  pdl_trigger();
  pdl_wait();
  const int warps = blockDim.x >> 5, w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t qidx = (int64_t)blockIdx.x * warps + w;   // over B*H*T
  const int64_t total = (int64_t)gridDim.y * heads * seq;  // gridDim.y = batch
  (void)total;
  const int t = (int)(qidx % seq);
  const int h = (int)((qidx / seq) % heads);
  const int b = blockIdx.y;
  if (qidx >= (int64_t)heads * seq) return;
  float* sc = sbuf + (size_t)w * seq;
  const int64_t d = (int64_t)heads * hd;
  const __nv_bfloat16* qrow = qkv + ((int64_t)b * seq + t) * ldq + (int64_t)h * hd;
  float mx = -INFINITY;
  for (int s = lane; s <= t; s += 32) {
    const __nv_bfloat16* krow = qkv + ((int64_t)b * seq + s) * ldq + d + (int64_t)h * hd;
    float acc = 0.f;
    for (int c = 0; c < hd; ++c) acc = fmaf(__bfloat162float(qrow[c]), __bfloat162float(krow[c]), acc);
    acc *= scale;
    sc[s] = acc;
    mx = fmaxf(mx, acc);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  float sum = 0.f;
  for (int s = lane; s <= t; s += 32) {
    const float e = expf(sc[s] - mx);
    sc[s] = e;
    sum += e;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  __syncwarp();
  const float inv = 1.0f / sum;
  for (int c = lane; c < hd; c += 32) {
    float acc = 0.f;
    for (int s = 0; s <= t; ++s) {
      const __nv_bfloat16* vrow = qkv + ((int64_t)b * seq + s) * ldq + 2 * d + (int64_t)h * hd;
      acc = fmaf(sc[s], __bfloat162float(vrow[c]), acc);
    }
    ctx[((int64_t)b * seq + t) * ldc + (int64_t)h * hd + c] = __float2bfloat16_rn(acc * inv);
  }
}

int attention_tc_launch(const __nv_bfloat16* qkv, int64_t ldq, int64_t batch, int64_t seq, int64_t heads,
                        int64_t hd, __nv_bfloat16* ctx, int64_t ldc, cudaStream_t st);

int attention_launch(const __nv_bfloat16* qkv, int64_t ldq, int64_t batch, int64_t seq, int64_t heads,
                     int64_t hd, __nv_bfloat16* ctx, int64_t ldc, cudaStream_t st) {
  if (batch * seq == 0) return ZO_OK;
  const float scale = 1.0f / sqrtf((float)hd);
  const bool aligned = (ldq % 8 == 0) && (ldc % 8 == 0) &&
                       ((reinterpret_cast<uintptr_t>(qkv) & 15) == 0) && ((reinterpret_cast<uintptr_t>(ctx) & 15) == 0);
  if ((hd == 64 || hd == 128) && aligned) return attention_tc_launch(qkv, ldq, batch, seq, heads, hd, ctx, ldc, st);
  if (hd > 256) { set_error("attention: head_dim %lld unsupported", (long long)hd); return ZO_ERR_CONFIG; }
  const int warps = 4;
  const size_t smem = (size_t)warps * seq * sizeof(float);
  if (smem > 48 * 1024) cudaFuncSetAttribute(attn_simt_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const dim3 grid((unsigned)((heads * seq + warps - 1) / warps), (unsigned)batch);
  launch_k(attn_simt_kernel, grid, dim3(warps * 32), smem, st, qkv, ldq, (int)seq, (int)heads, (int)hd, ctx, ldc,
           scale);
  return launch_status("attn_simt_kernel");
}

}  // namespace zo
