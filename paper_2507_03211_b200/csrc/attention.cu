// Causal exact-softmax attention of the zosim block (src/zosim/model.py:325-332):
//   scores = q k^T / sqrt(hd), -inf above the diagonal, max-subtracted softmax, @ v.
// qkv is the fused QKV GEMM output: row m = b*T + t holds [q | k | v], each H*hd wide.
//
// Two kernels:
//  * flash_attn_kernel<HD>  (hd in {64, 128}): FlashAttention-2 style tiling,
//    64-query x 64-key tiles, bf16 mma.sync m16n8k16 with fp32 accumulation,
//    online softmax in fp32 (exp2), no T x T materialisation. Attention is
//    2-3% of the step's FLOPs at the benchmark shapes (SURVEY shape sheet).
//  * attn_simt_kernel (any hd <= 256): warp per query, fp32 throughout; used
//    for the small/ragged shapes of the parity suite.
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

// ------------------------------- flash path --------------------------------
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
__device__ __forceinline__ void mma_bf16_16816(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void cp_async16(uint32_t saddr, const void* g, bool pred) {
  const int sz = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(saddr), "l"(g), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// smem tile [64 rows][HD] bf16, 16-byte chunks XOR-swizzled by (row & 7)
template <int HD>
__device__ __forceinline__ uint32_t swz(int row, int chunk) {
  constexpr int CH = HD / 8;
  return (uint32_t)((row * CH + (chunk ^ (row & 7))) * 16);
}

template <int HD>
__global__ void __launch_bounds__(128) flash_attn_kernel(const __nv_bfloat16* __restrict__ qkv, int64_t ldq,
                                                         int seq, int heads, __nv_bfloat16* __restrict__ ctx,
                                                         int64_t ldc, float scale_log2) {
  constexpr int BQ = 64, BK = 64, CH = HD / 8;
  extern __shared__ __align__(128) uint8_t smem[];
  pdl_trigger();
  pdl_wait();
  uint8_t* sQ = smem;
  uint8_t* sK = smem + BQ * HD * 2;            // 2 stages
  uint8_t* sV = sK + 2 * BK * HD * 2;          // 2 stages
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int qt = (int)gridDim.x - 1 - (int)blockIdx.x;   // heavy (late) query tiles first
  const int h = blockIdx.y, b = blockIdx.z;
  const int q0 = qt * BQ;
  const int64_t d = (int64_t)heads * HD;
  const __nv_bfloat16* base = qkv + (int64_t)b * seq * ldq + (int64_t)h * HD;

  auto load_tile = [&](uint8_t* dst, int row0, int64_t col_off) {
    for (int i = tid; i < 64 * CH; i += 128) {
      const int r = i / CH, c = i % CH;
      const int gr = row0 + r;
      const bool ok = gr < seq;
      const __nv_bfloat16* src = base + (int64_t)(ok ? gr : 0) * ldq + col_off + c * 8;
      cp_async16(smem_u32(dst) + swz<HD>(r, c), src, ok);
    }
  };

  load_tile(sQ, q0, 0);
  load_tile(sK, 0, d);
  load_tile(sV, 0, 2 * d);
  cp_async_commit();

  float o[HD / 8][4];
#pragma unroll
  for (int j = 0; j < HD / 8; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
  float mrow[2] = {-INFINITY, -INFINITY}, lrow[2] = {0.f, 0.f};
  uint32_t qf[HD / 16][4];

  const int n_kt = min((q0 + BQ - 1) / BK, (seq - 1) / BK) + 1;
  const int g = lane >> 2, tq = lane & 3;
  const int qrow_base = q0 + warp * 16;

  for (int kt = 0; kt < n_kt; ++kt) {
    const int stage = kt & 1;
    if (kt + 1 < n_kt) {
      load_tile(sK + (stage ^ 1) * BK * HD * 2, (kt + 1) * BK, d);
      load_tile(sV + (stage ^ 1) * BK * HD * 2, (kt + 1) * BK, 2 * d);
    }
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    if (kt == 0) {
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk) {
        const int r = warp * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
        const int c = kk * 2 + (lane >> 4);
        ldsm_x4(smem_u32(sQ) + swz<HD>(r, c), qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3]);
      }
    }
    const uint8_t* cK = sK + stage * BK * HD * 2;
    const uint8_t* cV = sV + stage * BK * HD * 2;
    // S = Q K^T  (16 x 64 per warp)
    float s[8][4];
#pragma unroll
    for (int j = 0; j < 8; ++j) s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk) {
#pragma unroll
      for (int jp = 0; jp < 4; ++jp) {   // pairs of 8-key n-tiles
        const int r = jp * 16 + (lane & 7) + (lane >> 4) * 8;
        const int c = kk * 2 + ((lane >> 3) & 1);
        uint32_t b0, b1, b2, b3;
        ldsm_x4(smem_u32(cK) + swz<HD>(r, c), b0, b1, b2, b3);
        mma_bf16_16816(s[2 * jp], qf[kk], b0, b1);
        mma_bf16_16816(s[2 * jp + 1], qf[kk], b2, b3);
      }
    }
    // causal mask + online softmax (rows g and g+8 of this warp)
    const int k0 = kt * BK;
    float mnew[2] = {mrow[0], mrow[1]};
#pragma unroll
    for (int j = 0; j < 8; ++j) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int qi = qrow_base + g + (e >> 1) * 8;
        const int ki = k0 + j * 8 + tq * 2 + (e & 1);
        float v = s[j][e] * scale_log2;
        if (ki > qi || ki >= seq) v = -INFINITY;
        s[j][e] = v;
        mnew[e >> 1] = fmaxf(mnew[e >> 1], v);
      }
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      mnew[r] = fmaxf(mnew[r], __shfl_xor_sync(0xffffffffu, mnew[r], 1));
      mnew[r] = fmaxf(mnew[r], __shfl_xor_sync(0xffffffffu, mnew[r], 2));
    }
    float alpha[2], msafe[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      msafe[r] = mnew[r] == -INFINITY ? 0.f : mnew[r];
      alpha[r] = exp2f(mrow[r] - msafe[r]);
      mrow[r] = mnew[r];
      lrow[r] *= alpha[r];
    }
#pragma unroll
    for (int j = 0; j < HD / 8; ++j) {
      o[j][0] *= alpha[0]; o[j][1] *= alpha[0];
      o[j][2] *= alpha[1]; o[j][3] *= alpha[1];
    }
    uint32_t pf[4][4];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float p0 = exp2f(s[j][0] - msafe[0]), p1 = exp2f(s[j][1] - msafe[0]);
      const float p2 = exp2f(s[j][2] - msafe[1]), p3 = exp2f(s[j][3] - msafe[1]);
      lrow[0] += p0 + p1;
      lrow[1] += p2 + p3;
      const int kk = j >> 1;
      if ((j & 1) == 0) { pf[kk][0] = pack_bf16(p0, p1); pf[kk][1] = pack_bf16(p2, p3); }
      else              { pf[kk][2] = pack_bf16(p0, p1); pf[kk][3] = pack_bf16(p2, p3); }
    }
    // O += P V
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
#pragma unroll
      for (int np = 0; np < HD / 16; ++np) {
        const int r = kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
        const int c = np * 2 + (lane >> 4);
        uint32_t b0, b1, b2, b3;
        ldsm_x4_t(smem_u32(cV) + swz<HD>(r, c), b0, b1, b2, b3);
        mma_bf16_16816(o[2 * np], pf[kk], b0, b1);
        mma_bf16_16816(o[2 * np + 1], pf[kk], b2, b3);
      }
    }
    __syncthreads();
  }
  cp_async_wait<0>();
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    lrow[r] += __shfl_xor_sync(0xffffffffu, lrow[r], 1);
    lrow[r] += __shfl_xor_sync(0xffffffffu, lrow[r], 2);
  }
  const float inv0 = 1.f / lrow[0], inv1 = 1.f / lrow[1];
  const int r0 = qrow_base + g, r1 = r0 + 8;
  __nv_bfloat16* out = ctx + (int64_t)b * seq * ldc + (int64_t)h * HD;
#pragma unroll
  for (int j = 0; j < HD / 8; ++j) {
    const int c = j * 8 + tq * 2;
    if (r0 < seq) *reinterpret_cast<uint32_t*>(out + (int64_t)r0 * ldc + c) = pack_bf16(o[j][0] * inv0, o[j][1] * inv0);
    if (r1 < seq) *reinterpret_cast<uint32_t*>(out + (int64_t)r1 * ldc + c) = pack_bf16(o[j][2] * inv1, o[j][3] * inv1);
  }
}


// 128-query CTAs (8 warps x 16 rows) share each 64-key K/V tile; masks only on
// tiles that straddle a warp's diagonal, fully-masked tiles skipped per warp,
// softmax scale folded into one FFMA before exp2.
template <int HD>
__global__ void __launch_bounds__(256) flash_attn_q128_kernel(const __nv_bfloat16* __restrict__ qkv, int64_t ldq,
                                                              int seq, int heads, __nv_bfloat16* __restrict__ ctx,
                                                              int64_t ldc, float scale_log2) {
  constexpr int BQ = 128, BK = 64, CH = HD / 8;
  extern __shared__ __align__(128) uint8_t smem[];
  pdl_trigger();
  pdl_wait();
  uint8_t* sQ = smem;                              // [128][HD]
  uint8_t* sK = smem + BQ * HD * 2;                // 2 stages of [64][HD]
  uint8_t* sV = sK + 2 * BK * HD * 2;              // 2 stages
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int qt = (int)gridDim.x - 1 - (int)blockIdx.x;   // heavy tiles first
  const int h = blockIdx.y, b = blockIdx.z;
  const int q0 = qt * BQ;
  const int64_t d = (int64_t)heads * HD;
  const __nv_bfloat16* base = qkv + (int64_t)b * seq * ldq + (int64_t)h * HD;

  auto load_rows = [&](uint8_t* dst, int rows, int row0, int64_t col_off) {
    for (int i = tid; i < rows * CH; i += 256) {
      const int r = i / CH, c = i % CH;
      const int gr = row0 + r;
      const bool ok = gr < seq;
      const __nv_bfloat16* src = base + (int64_t)(ok ? gr : 0) * ldq + col_off + c * 8;
      cp_async16(smem_u32(dst) + swz<HD>(r, c), src, ok);
    }
  };

  load_rows(sQ, BQ, q0, 0);
  load_rows(sK, BK, 0, d);
  load_rows(sV, BK, 0, 2 * d);
  cp_async_commit();

  float o[HD / 8][4];
#pragma unroll
  for (int j = 0; j < HD / 8; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
  float mrow[2] = {-INFINITY, -INFINITY}, lrow[2] = {0.f, 0.f};
  uint32_t qf[HD / 16][4];

  const int last_q = min(q0 + BQ, seq) - 1;
  const int n_kt = last_q / BK + 1;
  const int g = lane >> 2, tq = lane & 3;
  const int qw = q0 + warp * 16;              // this warp's first query row

  for (int kt = 0; kt < n_kt; ++kt) {
    const int stage = kt & 1;
    if (kt + 1 < n_kt) {
      load_rows(sK + (stage ^ 1) * BK * HD * 2, BK, (kt + 1) * BK, d);
      load_rows(sV + (stage ^ 1) * BK * HD * 2, BK, (kt + 1) * BK, 2 * d);
    }
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    if (kt == 0) {
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk) {
        const int r = warp * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
        const int c = kk * 2 + (lane >> 4);
        ldsm_x4(smem_u32(sQ) + swz<HD>(r, c), qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3]);
      }
    }
    const int k0 = kt * BK;
    if (k0 <= qw + 15 && qw < seq) {          // tile has keys visible to some row of this warp
      const uint8_t* cK = sK + stage * BK * HD * 2;
      const uint8_t* cV = sV + stage * BK * HD * 2;
      float s[8][4];
#pragma unroll
      for (int j = 0; j < 8; ++j) s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk) {
#pragma unroll
        for (int jp = 0; jp < 4; ++jp) {
          const int r = jp * 16 + (lane & 7) + (lane >> 4) * 8;
          const int c = kk * 2 + ((lane >> 3) & 1);
          uint32_t b0, b1, b2, b3;
          ldsm_x4(smem_u32(cK) + swz<HD>(r, c), b0, b1, b2, b3);
          mma_bf16_16816(s[2 * jp], qf[kk], b0, b1);
          mma_bf16_16816(s[2 * jp + 1], qf[kk], b2, b3);
        }
      }
      const bool need_mask = (k0 + BK - 1 > qw) || (k0 + BK > seq);
      if (need_mask) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int qi = qw + g + (e >> 1) * 8;
            const int ki = k0 + j * 8 + tq * 2 + (e & 1);
            if (ki > qi || ki >= seq) s[j][e] = -INFINITY;
          }
        }
      }
      float mnew[2] = {mrow[0], mrow[1]};
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        mnew[0] = fmaxf(mnew[0], fmaxf(s[j][0], s[j][1]));
        mnew[1] = fmaxf(mnew[1], fmaxf(s[j][2], s[j][3]));
      }
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        mnew[r] = fmaxf(mnew[r], __shfl_xor_sync(0xffffffffu, mnew[r], 1));
        mnew[r] = fmaxf(mnew[r], __shfl_xor_sync(0xffffffffu, mnew[r], 2));
      }
      float alpha[2], mb[2];
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        // raw-score max; exp2(scale*s - scale*m): one FFMA per element
        mb[r] = mnew[r] == -INFINITY ? 0.f : mnew[r] * scale_log2;
        alpha[r] = exp2f(fmaf(mrow[r], scale_log2, -mb[r]));
        mrow[r] = mnew[r];
        lrow[r] *= alpha[r];
      }
#pragma unroll
      for (int j = 0; j < HD / 8; ++j) {
        o[j][0] *= alpha[0]; o[j][1] *= alpha[0];
        o[j][2] *= alpha[1]; o[j][3] *= alpha[1];
      }
      uint32_t pf[4][4];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float p0 = exp2f(fmaf(s[j][0], scale_log2, -mb[0])), p1 = exp2f(fmaf(s[j][1], scale_log2, -mb[0]));
        const float p2 = exp2f(fmaf(s[j][2], scale_log2, -mb[1])), p3 = exp2f(fmaf(s[j][3], scale_log2, -mb[1]));
        lrow[0] += p0 + p1;
        lrow[1] += p2 + p3;
        const int kk = j >> 1;
        if ((j & 1) == 0) { pf[kk][0] = pack_bf16(p0, p1); pf[kk][1] = pack_bf16(p2, p3); }
        else              { pf[kk][2] = pack_bf16(p0, p1); pf[kk][3] = pack_bf16(p2, p3); }
      }
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
#pragma unroll
        for (int np = 0; np < HD / 16; ++np) {
          const int r = kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
          const int c = np * 2 + (lane >> 4);
          uint32_t b0, b1, b2, b3;
          ldsm_x4_t(smem_u32(cV) + swz<HD>(r, c), b0, b1, b2, b3);
          mma_bf16_16816(o[2 * np], pf[kk], b0, b1);
          mma_bf16_16816(o[2 * np + 1], pf[kk], b2, b3);
        }
      }
    }
    __syncthreads();
  }
  cp_async_wait<0>();
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    lrow[r] += __shfl_xor_sync(0xffffffffu, lrow[r], 1);
    lrow[r] += __shfl_xor_sync(0xffffffffu, lrow[r], 2);
  }
  const float inv0 = lrow[0] > 0.f ? 1.f / lrow[0] : 0.f, inv1 = lrow[1] > 0.f ? 1.f / lrow[1] : 0.f;
  const int r0 = qw + g, r1 = r0 + 8;
  __nv_bfloat16* out = ctx + (int64_t)b * seq * ldc + (int64_t)h * HD;
#pragma unroll
  for (int j = 0; j < HD / 8; ++j) {
    const int c = j * 8 + tq * 2;
    if (r0 < seq) *reinterpret_cast<uint32_t*>(out + (int64_t)r0 * ldc + c) = pack_bf16(o[j][0] * inv0, o[j][1] * inv0);
    if (r1 < seq) *reinterpret_cast<uint32_t*>(out + (int64_t)r1 * ldc + c) = pack_bf16(o[j][2] * inv1, o[j][3] * inv1);
  }
}

int attention_tc_launch(const __nv_bfloat16* qkv, int64_t ldq, int64_t batch, int64_t seq, int64_t heads,
                        int64_t hd, __nv_bfloat16* ctx, int64_t ldc, cudaStream_t st);

int attention_launch(const __nv_bfloat16* qkv, int64_t ldq, int64_t batch, int64_t seq, int64_t heads,
                     int64_t hd, __nv_bfloat16* ctx, int64_t ldc, cudaStream_t st) {
  if (batch * seq == 0) return ZO_OK;
  const float scale = 1.0f / sqrtf((float)hd);
  const bool aligned = (ldq % 8 == 0) && (ldc % 8 == 0) &&
                       ((reinterpret_cast<uintptr_t>(qkv) & 15) == 0) && ((reinterpret_cast<uintptr_t>(ctx) & 3) == 0);
  static const int use_tc = [] {
    const char* e = getenv("ZO_ATTN_TC");   // 0: the mma.sync kernels (A/B testing)
    return e ? atoi(e) : 1;
  }();
  // tcgen05 path for hd 64 and 128 (hd 128, T=2048: 91 us vs 222 us for the mma.sync kernel)
  if ((hd == 64 || hd == 128) && aligned && use_tc)
    return attention_tc_launch(qkv, ldq, batch, seq, heads, hd, ctx, ldc, st);
  static const int variant = [] {
    const char* e = getenv("ZO_ATTN_Q64");   // 1: the 64-query kernel (A/B testing)
    return e ? atoi(e) : 0;
  }();
  if ((hd == 64 || hd == 128) && aligned && variant == 0) {
    const dim3 grid((unsigned)((seq + 127) / 128), (unsigned)heads, (unsigned)batch);
    const float sl2 = scale * 1.4426950408889634f;
    if (hd == 64) {
      const int smem = (128 + 4 * 64) * 64 * 2;     // 48 KB
      launch_k(flash_attn_q128_kernel<64>, grid, dim3(256), smem, st, qkv, ldq, (int)seq, (int)heads, ctx, ldc, sl2);
    } else {
      const int smem = (128 + 4 * 64) * 128 * 2;    // 96 KB
      static bool attr = false;
      if (!attr) {
        cudaFuncSetAttribute(flash_attn_q128_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        attr = true;
      }
      launch_k(flash_attn_q128_kernel<128>, grid, dim3(256), smem, st, qkv, ldq, (int)seq, (int)heads, ctx, ldc, sl2);
    }
    return launch_status("flash_attn_q128_kernel");
  }
  if ((hd == 64 || hd == 128) && aligned) {
    const dim3 grid((unsigned)((seq + 63) / 64), (unsigned)heads, (unsigned)batch);
    const float sl2 = scale * 1.4426950408889634f;
    if (hd == 64) {
      const int smem = 64 * 64 * 2 * 5;
      launch_k(flash_attn_kernel<64>, grid, dim3(128), smem, st, qkv, ldq, (int)seq, (int)heads, ctx, ldc, sl2);
    } else {
      const int smem = 64 * 128 * 2 * 5;
      cudaFuncSetAttribute(flash_attn_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      launch_k(flash_attn_kernel<128>, grid, dim3(128), smem, st, qkv, ldq, (int)seq, (int)heads, ctx, ldc, sl2);
    }
    return launch_status("flash_attn_kernel");
  }
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
