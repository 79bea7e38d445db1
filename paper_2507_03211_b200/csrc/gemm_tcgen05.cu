// bf16 GEMM on the 5th-generation tensor cores (tcgen05) with TMA-fed shared
// memory, fp32 accumulators in TMEM and a fused epilogue.
//
//   C[M,N] = A[M,K] . B[K,N]
//   A: activations, row-major, K contiguous          -> UMMA K-major operand
//   B: weights in the reference's (d_in, d_out) layout, N contiguous
//      (src/zosim/model.py:325 `h @ W`)                 -> UMMA MN-major operand
//      or, with ZO_GEMM_B_KMAJOR, B^T stored [N, K] row-major (K contiguous:
//      a tied LM head reading the [V, d] token embedding) -> UMMA K-major
//
// Persistent, warp-specialised CTA (192 threads, 1 CTA per SM):
//   warp 0      TMA producer (one lane): A 128x64 box + B 64x64 boxes per stage
//   warp 1      TMEM allocator + MMA issuer (one lane issues tcgen05.mma)
//   warps 2..5  epilogue: tcgen05.ld 32x32b -> registers -> fused op -> global
// Pipelines: smem ring full/empty mbarriers (TMA <-> MMA) and a 2-deep TMEM
// accumulator ring tfull/tempty (MMA <-> epilogue), so the epilogue of tile i
// overlaps the MMAs of tile i+1.
//
// Epilogues (the ops that follow each GEMM in model.py:325-344):
//   ZO_EPI_BIAS_BF16       qkv  = h @ Wqkv + b                 (bf16 out)
//   ZO_EPI_BIAS_GELU_BF16  f    = gelu_tanh(h2 @ W1 + b1)      (bf16 out)
//   ZO_EPI_BIAS_RELU_BF16  f    = relu(h2 @ W1 + b1)           (bf16 out, real OPT)
//   ZO_EPI_BIAS_RESID_F32  x   += ctx @ Wo + bo / f @ W2 + b2  (fp32 residual)
//   ZO_EPI_CE              per-row (max, sum exp) of logits + target logit;
//                          the [M, V] logits never reach HBM
#include <cuda.h>
#include <cudaTypedefs.h>
#include <stdlib.h>

#include <mutex>
#include <unordered_map>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace zo {

constexpr int kBM = 128;
constexpr int kBK = 64;
// Epilogue warps: 8 (each owns a TMEM lane quarter x one column half), or 4
// (each walks both halves) -- the 6-warp CTA at <= 168 registers leaves half
// of the SM's register file for a co-resident perturb pass.
#ifndef ZO_GEMM_EPI_WARPS
#define ZO_GEMM_EPI_WARPS 8
#endif
constexpr int kEpiWarps = ZO_GEMM_EPI_WARPS;
static_assert(kEpiWarps == 8 || kEpiWarps == 4, "epilogue warps");
constexpr int kGemmThreads = 64 + 32 * kEpiWarps;   // warp 0 TMA, warp 1 MMA/TMEM, warps 2.. epilogue
constexpr int kGemmMinBlocks = kEpiWarps == 4 ? 2 : 1;   // 4 epilogue warps: cap registers at 170

template <int BN>
struct GemmCfg {
  static constexpr int kStages = BN == 256 ? 4 : 6;
  static constexpr int kABytes = kBM * kBK * 2;   // 16 KB
  static constexpr int kBBytes = kBK * BN * 2;    // 32 KB / 16 KB
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kTmemCols = 2 * BN;        // double-buffered accumulator
  static constexpr int kSmem = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;
};

struct GemmArgs {
  int64_t M, N, K;
  const float* bias;
  void* out;
  int64_t ldo;
  const int32_t* targets;
  float* ce_part;
  float* ce_tgt;
  int32_t* err;
  int64_t ce_tiles;
  // row-split ("stacked") problem: rows >= m_split use the second B operand
  // (tmB2) and bias2 -- the +eps / -eps forwards of one ZO step as ONE launch
  // over [x+; x-] (0 = off; a multiple of 256 so every pair tile is one side)
  int64_t m_split;
  const float* bias2;
};

template <int BN, bool BKM = false>
__device__ __forceinline__ uint32_t make_idesc() {
  // c_format F32 [4,6)=1, a_format BF16 [7,10)=1, b_format BF16 [10,13)=1,
  // a_major K (bit 15 = 0), b_major MN (bit 16 = 1) or K (0), N>>3 at [17,23), M>>4 at [24,29)
  return (1u << 4) | (1u << 7) | (1u << 10) | (BKM ? 0u : (1u << 16)) | ((uint32_t)(BN >> 3) << 17) |
         ((uint32_t)(kBM >> 4) << 24);
}

__device__ __forceinline__ float ex2_fast(float x) {   // MUFU.EX2, ex2(-inf) = 0
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// tanh-GELU (model.py:286-289).  tanh via MUFU.TANH (rel. error ~2^-11), far
// below the bf16 rounding of the output that follows.
__device__ __forceinline__ float tanh_fast(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float gelu_tanh(float x) {
  const float c = 0.7978845608028654f;  // sqrt(2/pi)
  const float u = c * fmaf(0.044715f * x, x * x, x);
  const float hx = 0.5f * x;
  return fmaf(hx, tanh_fast(u), hx);
}

// One 128 x BN accumulator tile from TMEM -> fused epilogue -> global.
// Thread (quarter, lane) owns output row m0 + 32*quarter + lane.
// Epilogue warp e (0..7) owns TMEM lane quarter (warp % 4) and column half
// e / 4, so two warps share each quarter and each thread stores half a row.
__device__ __forceinline__ void ld_v8_na(const float* p, float* v) {
  asm volatile("ld.global.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
               : "l"(p));
}
__device__ __forceinline__ void st_v8(float* p, const float* v) {
  asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(v[0]), "f"(v[1]), "f"(v[2]),
               "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
               : "memory");
}

template <int BN, int EPI>
__device__ __forceinline__ void epilogue_tile(const GemmArgs& args, uint32_t tmem_base, int acc, int quarter,
                                              int half, int lane, int64_t m0, int64_t n0, int64_t tn) {
  const int64_t row_base = m0 + quarter * 32;
  const int64_t row = row_base + lane;
  const bool second = args.m_split && row_base >= args.m_split;
  const float* __restrict__ bias = second ? args.bias2 : args.bias;
  const bool row_ok = row < args.M;
  float ce_m = -INFINITY, ce_s = 0.f;
  int32_t tgt = -1;
  bool bad = false;
  if constexpr (EPI == ZO_EPI_CE) {
    if (row_ok) tgt = args.targets[second ? row - args.m_split : row];   // stacked rows share the targets
  }
  constexpr int CH = BN / 64;   // 32-column chunks per half
#pragma unroll 1
  for (int c = half * CH; c < (half + 1) * CH; ++c) {
    const int64_t col0 = n0 + c * 32;
    const uint32_t taddr = tmem_base + (uint32_t)(acc * BN + c * 32) + ((uint32_t)(quarter * 32) << 16);
    if constexpr (EPI == ZO_EPI_CE) {
      // thread-per-row: online (max, sum exp) over this row's columns, target logit
      float v[32];
      tmem_ld_32x32b_x32(taddr, v);
      if (!row_ok || col0 >= args.N) continue;
      const int lim = col0 + 32 <= args.N ? 32 : (int)(args.N - col0);
      const bool has_bias = bias != nullptr;   // a tied head has no bias (real OPT)
      if (lim == 32) {
        // full chunk (all but a row's last): float4 bias, 4-way max / min / sum
        // chains, exp2 with the log2(e) scale folded into one FFMA; non-finite
        // logits surface as an infinite max / min or a NaN sum
        if (has_bias) {
          if ((reinterpret_cast<uintptr_t>(bias + col0) & 15) == 0) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const float4 b4 = __ldg(reinterpret_cast<const float4*>(bias + col0) + i);
              v[4 * i] += b4.x; v[4 * i + 1] += b4.y; v[4 * i + 2] += b4.z; v[4 * i + 3] += b4.w;
            }
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] += __ldg(bias + col0 + i);
          }
        }
        float mx[4], mn[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) { mx[k] = v[k]; mn[k] = v[k]; }
#pragma unroll
        for (int i = 4; i < 32; ++i) { mx[i & 3] = fmaxf(mx[i & 3], v[i]); mn[i & 3] = fminf(mn[i & 3], v[i]); }
        const float cm = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3]));
        const float cmin = fminf(fminf(mn[0], mn[1]), fminf(mn[2], mn[3]));
        const float nm = fmaxf(ce_m, cm);
        const float nl = nm * 1.4426950408889634f;
        float sk[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int i = 0; i < 32; ++i) sk[i & 3] += ex2_fast(fmaf(v[i], 1.4426950408889634f, -nl));
        const float prev = ce_m == -INFINITY ? 0.f : ce_s * ex2_fast((ce_m - nm) * 1.4426950408889634f);
        ce_s = prev + ((sk[0] + sk[1]) + (sk[2] + sk[3]));
        ce_m = nm;
        bad |= !(isfinite(cm) && isfinite(cmin) && isfinite(ce_s));
        if (tgt >= col0 && tgt < col0 + 32) {
          const int ti = (int)(tgt - col0);
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (i == ti) args.ce_tgt[row] = v[i];
        }
        continue;
      }
      float cm = -INFINITY;
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        if (i < lim) {
          if (has_bias) v[i] += __ldg(bias + col0 + i);
          bad |= !isfinite(v[i]);
          cm = fmaxf(cm, v[i]);
        }
      }
      const float nm = fmaxf(ce_m, cm);
      float s = ce_s * __expf(ce_m - nm);
      if (ce_m == -INFINITY) s = 0.f;
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (i < lim) s += __expf(v[i] - nm);
      ce_m = nm;
      ce_s = s;
      if (tgt >= col0 && tgt < col0 + lim) {
        const int ti = (int)(tgt - col0);
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (i == ti) args.ce_tgt[row] = v[i];
      }
    } else if constexpr (EPI == ZO_EPI_BIAS_BF16 || EPI == ZO_EPI_BIAS_GELU_BF16 || EPI == ZO_EPI_BIAS_RELU_BF16) {
      // bf16 out: each thread writes 64 contiguous bytes of its row (4 x 16 B)
      float4 bias4[8];
      const bool full = row_ok && col0 + 32 <= args.N;
      if (full && ((reinterpret_cast<uintptr_t>(bias + col0) & 15) == 0)) {
#pragma unroll
        for (int i = 0; i < 8; ++i) bias4[i] = __ldg(reinterpret_cast<const float4*>(bias + col0) + i);
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          float t[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) t[j] = (col0 + 4 * i + j < args.N) ? bias[col0 + 4 * i + j] : 0.f;
          bias4[i] = make_float4(t[0], t[1], t[2], t[3]);
        }
      }
      float v[32];
      tmem_ld_32x32b_x32(taddr, v);
      if (!row_ok || col0 >= args.N) continue;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        v[4 * i] += bias4[i].x; v[4 * i + 1] += bias4[i].y;
        v[4 * i + 2] += bias4[i].z; v[4 * i + 3] += bias4[i].w;
      }
      if constexpr (EPI == ZO_EPI_BIAS_GELU_BF16) {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = gelu_tanh(v[i]);
      }
      if constexpr (EPI == ZO_EPI_BIAS_RELU_BF16) {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = fmaxf(v[i], 0.f);
      }
      __nv_bfloat16* o = static_cast<__nv_bfloat16*>(args.out) + row * args.ldo + col0;
      if (full && ((reinterpret_cast<uintptr_t>(o) & 15) == 0)) {
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
          uint32_t pk[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            __nv_bfloat162 h2 = __floats2bfloat162_rn(v[i + 2 * j], v[i + 2 * j + 1]);
            pk[j] = *reinterpret_cast<uint32_t*>(&h2);
          }
          *reinterpret_cast<uint4*>(o + i) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        }
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (col0 + i < args.N) o[i] = __float2bfloat16_rn(v[i]);
      }
    } else {
      // fp32 out (+ residual): row-per-thread like the bf16 path, 32 B
      // (full-sector) accesses, no shared-memory staging -- the tensor core's
      // operand reads already keep the SM's shared-memory pipe ~93% busy
      float* o = static_cast<float*>(args.out) + row * args.ldo + col0;
      const bool full = row_ok && col0 + 32 <= args.N;
      const bool vec = full && ((reinterpret_cast<uintptr_t>(o) & 31) == 0) &&
                       (EPI == ZO_EPI_F32 || (reinterpret_cast<uintptr_t>(bias + col0) & 15) == 0);
      float res[32];
      if constexpr (EPI == ZO_EPI_BIAS_RESID_F32) {
        // residual (the previous contents of out) read before the TMEM load so
        // the latency overlaps it
        if (vec) {
#pragma unroll
          for (int i = 0; i < 4; ++i) ld_v8_na(o + 8 * i, res + 8 * i);
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) res[i] = (row_ok && col0 + i < args.N) ? o[i] : 0.f;
        }
      }
      float v[32];
      tmem_ld_32x32b_x32(taddr, v);
      if (!row_ok || col0 >= args.N) continue;
      if constexpr (EPI == ZO_EPI_BIAS_RESID_F32) {
        if (vec) {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float4 b4 = __ldg(reinterpret_cast<const float4*>(bias + col0) + i);
            v[4 * i] = res[4 * i] + (v[4 * i] + b4.x);
            v[4 * i + 1] = res[4 * i + 1] + (v[4 * i + 1] + b4.y);
            v[4 * i + 2] = res[4 * i + 2] + (v[4 * i + 2] + b4.z);
            v[4 * i + 3] = res[4 * i + 3] + (v[4 * i + 3] + b4.w);
          }
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (col0 + i < args.N) v[i] = res[i] + (v[i] + bias[col0 + i]);
        }
      }
      if (vec) {
#pragma unroll
        for (int i = 0; i < 4; ++i) st_v8(o + 8 * i, v + 8 * i);
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (col0 + i < args.N) o[i] = v[i];
      }
    }
  }
  if constexpr (EPI == ZO_EPI_CE) {
    if (row_ok) {
      const int64_t slot = tn * 2 + half;
      args.ce_part[(row * args.ce_tiles + slot) * 2] = ce_m;
      args.ce_part[(row * args.ce_tiles + slot) * 2 + 1] = ce_s;
      if (bad) atomicOr(args.err, 2);
    }
  }
}

template <int BN, int EPI, bool BKM>
__global__ void __launch_bounds__(kGemmThreads, kGemmMinBlocks)
    gemm_tcgen05_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                        const GemmArgs args) {
  using C = GemmCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);
  const uint32_t sA = base;
  const uint32_t sB = base + C::kStages * C::kABytes;
  const uint32_t bars = base + C::kStages * C::kStageBytes;
  // barrier layout: full[S], empty[S], tfull[2], tempty[2], then tmem ptr
  auto full_bar = [&](int s) { return bars + 8u * s; };
  auto empty_bar = [&](int s) { return bars + 8u * (C::kStages + s); };
  auto tfull_bar = [&](int a) { return bars + 8u * (2 * C::kStages + a); };
  auto tempty_bar = [&](int a) { return bars + 8u * (2 * C::kStages + 2 + a); };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gbase + C::kStages * C::kStageBytes + 8 * (2 * C::kStages + 4));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t num_m = (args.M + kBM - 1) / kBM;
  const int64_t num_n = (args.N + BN - 1) / BN;
  const int64_t tiles = num_m * num_n;
  const int nk = (int)((args.K + kBK - 1) / kBK);

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
    for (int s = 0; s < C::kStages; ++s) { mbar_init(full_bar(s), 1); mbar_init(empty_bar(s), 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(tfull_bar(a), 1); mbar_init(tempty_bar(a), kEpiWarps); }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "r"((uint32_t)C::kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_trigger();
  pdl_wait();   // inputs of the previous kernel in the stream are visible from here

  if (warp == 0) {
    // ============================ TMA producer ============================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        const int m0 = (int)((tile % num_m) * kBM);
        const int n0 = (int)((tile / num_m) * BN);
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(empty_bar(stage), phase ^ 1u);
          mbar_expect_tx(full_bar(stage), (uint32_t)C::kStageBytes);
          tma_load_2d(sA + stage * C::kABytes, &tmA, full_bar(stage), kb * kBK, m0);
          if constexpr (BKM) {
            tma_load_2d(sB + stage * C::kBBytes, &tmB, full_bar(stage), kb * kBK, n0);   // BN rows x 64 k
          } else {
#pragma unroll
            for (int j = 0; j < BN / 64; ++j)
              tma_load_2d(sB + stage * C::kBBytes + j * (kBK * 128), &tmB, full_bar(stage), n0 + 64 * j, kb * kBK);
          }
          if (++stage == C::kStages) { stage = 0; phase ^= 1u; }
        }
      }
    }
  } else if (warp == 1) {
    // ============================ MMA issuer ==============================
    const uint32_t idesc = make_idesc<BN, BKM>();
    int stage = 0;
    uint32_t phase = 0;
    int64_t local = 0;
    for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++local) {
      const int acc = (int)(local & 1);
      const uint32_t acc_phase = (uint32_t)((local >> 1) & 1);
      mbar_wait(tempty_bar(acc), acc_phase ^ 1u);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + (uint32_t)(acc * BN);
      for (int kb = 0; kb < nk; ++kb) {
        mbar_wait(full_bar(stage), phase);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t a0 = sA + stage * C::kABytes;
          const uint32_t b0 = sB + stage * C::kBBytes;
#pragma unroll
          for (int kk = 0; kk < kBK / 16; ++kk) {
            const uint64_t ad = desc_sw128(a0 + kk * 32, 16, 1024);
            const uint64_t bd = BKM ? desc_sw128(b0 + kk * 32, 16, 1024) : desc_sw128(b0 + kk * 2048, kBK * 128, 1024);
            tc_mma_f16(d_tmem, ad, bd, idesc, (kb | kk) != 0 ? 1u : 0u);
          }
          tc_commit(empty_bar(stage));   // frees the smem slot once these MMAs retire
        }
        __syncwarp();
        if (++stage == C::kStages) { stage = 0; phase ^= 1u; }
      }
      if (lane == 0) tc_commit(tfull_bar(acc));  // accumulator ready for the epilogue
      __syncwarp();
    }
  } else {
    // ============================ epilogue ================================
    const int quarter = warp & 3;   // TMEM lanes 32*quarter .. +31
    int64_t local = 0;
    for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++local) {
      const int acc = (int)(local & 1);
      const uint32_t acc_phase = (uint32_t)((local >> 1) & 1);
      const int64_t m0 = (tile % num_m) * kBM;
      const int64_t tn = tile / num_m;
      mbar_wait(tfull_bar(acc), acc_phase);
      tc_fence_after();
#pragma unroll 1
      for (int e = warp - 2; e < 8; e += kEpiWarps)        // logical epilogue slot e: column half e / 4
        epilogue_tile<BN, EPI>(args, tmem_base, acc, quarter, e >> 2, lane, m0, tn * BN, tn);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty_bar(acc));
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem_base),
                 "r"((uint32_t)C::kTmemCols));
  }
}


// ----------------------------------------------------------------------------
// CTA-pair variant (tcgen05 cta_group::2): a cluster of 2 CTAs on one TPC
// computes a 256 x 256 tile with M=256 UMMAs issued by the leader CTA.  Each
// CTA stages its own 128 A rows and HALF of the B tile (128 columns), so per
// pair and K-block the pair moves 64 KB for 8.4 MFLOP (128 FLOP/B, 1.5x the
// single-CTA tile) -- the L2->SMEM feed, not the tensor pipe, bounds the
// single-CTA kernel at these shapes.  TMEM: each CTA holds its 128 rows x 256
// fp32 columns, double buffered (512 columns).
//   full[s]   leader only; expects both CTAs' bytes (cta_group::2 TMA signals it)
//   empty[s]  both CTAs; leader's tcgen05.commit multicasts to the pair
//   tfull[a]  both CTAs; multicast commit
//   tempty[a] leader only; 16 arrivals = 8 epilogue warps x 2 CTAs (remote)
// ----------------------------------------------------------------------------
#ifndef ZO_K2_STAGES
#define ZO_K2_STAGES 6
#endif
constexpr int k2Stages = ZO_K2_STAGES;   // 6 x 32 KB operand stages (no epilogue staging buffer)
constexpr int k2ABytes = kBM * kBK * 2;        // 16 KB: this CTA's 128 rows
constexpr int k2BBytes = kBK * 128 * 2;        // 16 KB: this CTA's half of B
constexpr int k2StageBytes = k2ABytes + k2BBytes;
constexpr int k2Smem = k2Stages * k2StageBytes + 1024 + 256;
static_assert(k2Smem <= 232448, "pair kernel smem");

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void tma_load_2d_cg2(uint32_t dst, const CUtensorMap* map, uint32_t bar_cluster, int c0,
                                                int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3}], [%4];\n" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar_cluster)
      : "memory");
}
__device__ __forceinline__ void tc_commit_pair(uint32_t bar) {
  asm volatile(
      "{\n.reg .b16 m;\nmov.b16 m, 3;\n"
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n}\n" ::"r"(
          bar)
      : "memory");
}
__device__ __forceinline__ void tc_mma_f16_pair(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                                uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

template <int EPI, bool BKM>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kGemmThreads, kGemmMinBlocks)
    gemm_tcgen05_pair_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                             const __grid_constant__ CUtensorMap tmB2, const GemmArgs args) {
  constexpr int BN = 256;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);
  const uint32_t sA = base;
  const uint32_t sB = base + k2Stages * k2ABytes;
  const uint32_t bars = base + k2Stages * k2StageBytes;
  auto full_bar = [&](int s) { return bars + 8u * s; };
  auto empty_bar = [&](int s) { return bars + 8u * (k2Stages + s); };
  auto tfull_bar = [&](int a) { return bars + 8u * (2 * k2Stages + a); };
  auto tempty_bar = [&](int a) { return bars + 8u * (2 * k2Stages + 2 + a); };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gbase + k2Stages * k2StageBytes + 8 * (2 * k2Stages + 4));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int64_t cluster_id = blockIdx.x >> 1, n_clusters = gridDim.x >> 1;
  const int64_t num_m = (args.M + 2 * kBM - 1) / (2 * kBM);
  const int64_t num_n = (args.N + BN - 1) / BN;
  const int nk = (int)((args.K + kBK - 1) / kBK);

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
    if (args.m_split) prefetch_tmap(&tmB2);
    for (int s = 0; s < k2Stages; ++s) { mbar_init(full_bar(s), 1); mbar_init(empty_bar(s), 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(tfull_bar(a), 1); mbar_init(tempty_bar(a), 2 * kEpiWarps); }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "r"(512u));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_trigger();
  pdl_wait();

  if (warp == 0) {
    // ====== TMA producer (both CTAs): own A rows + own half of B ======
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      const int64_t tiles = num_m * num_n;
      for (int64_t tile = cluster_id; tile < tiles; tile += n_clusters) {
        const int m0 = (int)((tile % num_m) * (2 * kBM) + rank * kBM);
        const int n0 = (int)((tile / num_m) * BN + rank * 128);
        const CUtensorMap* mb = (args.m_split && (tile % num_m) * (2 * kBM) >= args.m_split) ? &tmB2 : &tmB;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(empty_bar(stage), phase ^ 1u);
          if (leader) mbar_expect_tx(full_bar(stage), (uint32_t)(2 * k2StageBytes));
          const uint32_t fb = mapa_shared(full_bar(stage), 0);
          tma_load_2d_cg2(sA + stage * k2ABytes, &tmA, fb, kb * kBK, m0);
          if constexpr (BKM) {
            tma_load_2d_cg2(sB + stage * k2BBytes, mb, fb, kb * kBK, n0);    // 128 rows x 64 k
          } else {
            tma_load_2d_cg2(sB + stage * k2BBytes, mb, fb, n0, kb * kBK);
            tma_load_2d_cg2(sB + stage * k2BBytes + kBK * 128, mb, fb, n0 + 64, kb * kBK);
          }
          if (++stage == k2Stages) { stage = 0; phase ^= 1u; }
        }
      }
    }
  } else if (warp == 1) {
    // ====== MMA issuer (leader CTA only): M=256 x N=256 per instruction ======
    if (leader) {
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (BKM ? 0u : (1u << 16)) |
                             ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
      int stage = 0;
      uint32_t phase = 0;
      const int64_t tiles = num_m * num_n;
      int64_t local = 0;
      for (int64_t tile = cluster_id; tile < tiles; tile += n_clusters, ++local) {
        const int acc = (int)(local & 1);
        const uint32_t acc_phase = (uint32_t)((local >> 1) & 1);
        mbar_wait(tempty_bar(acc), acc_phase ^ 1u);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + (uint32_t)(acc * BN);
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(full_bar(stage), phase);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t a0 = sA + stage * k2ABytes;
            const uint32_t b0 = sB + stage * k2BBytes;
#pragma unroll
            for (int kk = 0; kk < kBK / 16; ++kk) {
              const uint64_t ad = desc_sw128(a0 + kk * 32, 16, 1024);
              const uint64_t bd =
                  BKM ? desc_sw128(b0 + kk * 32, 16, 1024) : desc_sw128(b0 + kk * 2048, kBK * 128, 1024);
              tc_mma_f16_pair(d_tmem, ad, bd, idesc, (kb | kk) != 0 ? 1u : 0u);
            }
            tc_commit_pair(empty_bar(stage));
          }
          __syncwarp();
          if (++stage == k2Stages) { stage = 0; phase ^= 1u; }
        }
        if (lane == 0) tc_commit_pair(tfull_bar(acc));
        __syncwarp();
      }
    }
  } else {
    // ====== epilogue (both CTAs): this CTA's 128 rows x 256 columns ======
    const int quarter = warp & 3;
    const int64_t tiles = num_m * num_n;
    int64_t local = 0;
    for (int64_t tile = cluster_id; tile < tiles; tile += n_clusters, ++local) {
      const int acc = (int)(local & 1);
      const uint32_t acc_phase = (uint32_t)((local >> 1) & 1);
      const int64_t m0 = (tile % num_m) * (2 * kBM) + rank * kBM;
      const int64_t tn = tile / num_m;
      mbar_wait(tfull_bar(acc), acc_phase);
      tc_fence_after();
#pragma unroll 1
      for (int e = warp - 2; e < 8; e += kEpiWarps)        // logical slot e: lane quarter, column half e / 4
        epilogue_tile<BN, EPI>(args, tmem_base, acc, quarter, e >> 2, lane, m0, tn * BN, tn);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(mapa_shared(tempty_bar(acc), 0));
    }
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tmem_base), "r"(512u));
  }
}

// ------------------------------ host side -----------------------------------
namespace {

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

struct MapKey {
  uint64_t ptr, inner, outer, ld, box_in, box_out;
  bool operator==(const MapKey& o) const {
    return ptr == o.ptr && inner == o.inner && outer == o.outer && ld == o.ld && box_in == o.box_in &&
           box_out == o.box_out;
  }
};
struct MapKeyHash {
  size_t operator()(const MapKey& k) const {
    uint64_t h = k.ptr * 0x9E3779B97F4A7C15ull;
    h ^= k.inner + 0x7F4A7C15ull + (h << 6) + (h >> 2);
    h ^= k.outer + (h << 6) + (h >> 2);
    h ^= k.ld + (h << 6) + (h >> 2);
    h ^= (k.box_in << 20) ^ k.box_out;
    return (size_t)h;
  }
};

std::mutex g_map_mu;
std::unordered_map<MapKey, CUtensorMap, MapKeyHash> g_maps;

// 2-D bf16 tensor map, inner dim contiguous, 128B swizzle, zero OOB fill.
int get_map(const void* ptr, int64_t inner, int64_t outer, int64_t ld, int box_in, int box_out, CUtensorMap* out) {
  MapKey key{(uint64_t)ptr, (uint64_t)inner, (uint64_t)outer, (uint64_t)ld, (uint64_t)box_in, (uint64_t)box_out};
  std::lock_guard<std::mutex> lk(g_map_mu);
  auto it = g_maps.find(key);
  if (it != g_maps.end()) { *out = it->second; return ZO_OK; }
  auto enc = get_encode();
  if (!enc) { set_error("cuTensorMapEncodeTiled unavailable (driver too old?)"); return ZO_ERR_CUDA; }
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {(cuuint32_t)box_in, (cuuint32_t)box_out};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d): ptr=%p inner=%lld outer=%lld ld=%lld", (int)r, ptr,
              (long long)inner, (long long)outer, (long long)ld);
    return ZO_ERR_CONFIG;
  }
  if (g_maps.size() > 4096) g_maps.clear();
  g_maps.emplace(key, m);
  *out = m;
  return ZO_OK;
}

template <int BN, int EPI, bool BKM = false>
int launch_t(const CUtensorMap& ma, const CUtensorMap& mb, const GemmArgs& a, cudaStream_t st) {
  using C = GemmCfg<BN>;
  static bool attr_done = false;   // per-instantiation (benign race: idempotent)
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(gemm_tcgen05_kernel<BN, EPI, BKM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         C::kSmem);
    if (e != cudaSuccess) { set_error("gemm smem attribute: %s", cudaGetErrorString(e)); return ZO_ERR_CUDA; }
    attr_done = true;
  }
  const int64_t tiles = ((a.M + kBM - 1) / kBM) * ((a.N + BN - 1) / BN);
  const int grid = (int)(tiles < num_sms() ? tiles : num_sms());
  launch_k(gemm_tcgen05_kernel<BN, EPI, BKM>, dim3(grid), dim3(kGemmThreads), C::kSmem, st, ma, mb, a);
  return launch_status("gemm_tcgen05_kernel");
}

template <int BN>
int launch_bn(int epi, bool bkm, const CUtensorMap& ma, const CUtensorMap& mb, const GemmArgs& a, cudaStream_t st) {
  if (bkm) {
    switch (epi) {
      case ZO_EPI_F32: return launch_t<BN, ZO_EPI_F32, true>(ma, mb, a, st);
      case ZO_EPI_CE: return launch_t<BN, ZO_EPI_CE, true>(ma, mb, a, st);
    }
    set_error("zo_gemm_bf16: ZO_GEMM_B_KMAJOR supports the F32 and CE epilogues only (got %d)", epi);
    return ZO_ERR_CONFIG;
  }
  switch (epi) {
    case ZO_EPI_F32: return launch_t<BN, ZO_EPI_F32>(ma, mb, a, st);
    case ZO_EPI_BIAS_BF16: return launch_t<BN, ZO_EPI_BIAS_BF16>(ma, mb, a, st);
    case ZO_EPI_BIAS_GELU_BF16: return launch_t<BN, ZO_EPI_BIAS_GELU_BF16>(ma, mb, a, st);
    case ZO_EPI_BIAS_RELU_BF16: return launch_t<BN, ZO_EPI_BIAS_RELU_BF16>(ma, mb, a, st);
    case ZO_EPI_BIAS_RESID_F32: return launch_t<BN, ZO_EPI_BIAS_RESID_F32>(ma, mb, a, st);
    case ZO_EPI_CE: return launch_t<BN, ZO_EPI_CE>(ma, mb, a, st);
  }
  set_error("zo_gemm_bf16: unknown epilogue %d", epi);
  return ZO_ERR_CONFIG;
}


template <int EPI, bool BKM = false>
int launch_pair_t(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mb2, const GemmArgs& a,
                  cudaStream_t st) {
  static bool attr_done = false;
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(gemm_tcgen05_pair_kernel<EPI, BKM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         k2Smem);
    if (e != cudaSuccess) { set_error("gemm pair smem attribute: %s", cudaGetErrorString(e)); return ZO_ERR_CUDA; }
    attr_done = true;
  }
  const int64_t tiles = ((a.M + 255) / 256) * ((a.N + 255) / 256);
  const int64_t pairs = num_sms() / 2;
  const int grid = 2 * (int)(tiles < pairs ? tiles : pairs);
  launch_k(gemm_tcgen05_pair_kernel<EPI, BKM>, dim3(grid), dim3(kGemmThreads), k2Smem, st, ma, mb, mb2, a);
  return launch_status("gemm_tcgen05_pair_kernel");
}

int launch_pair(int epi, bool bkm, const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mb2,
                const GemmArgs& a, cudaStream_t st) {
  if (bkm) {
    switch (epi) {
      case ZO_EPI_F32: return launch_pair_t<ZO_EPI_F32, true>(ma, mb, mb2, a, st);
      case ZO_EPI_CE: return launch_pair_t<ZO_EPI_CE, true>(ma, mb, mb2, a, st);
    }
    set_error("zo_gemm_bf16: ZO_GEMM_B_KMAJOR supports the F32 and CE epilogues only (got %d)", epi);
    return ZO_ERR_CONFIG;
  }
  switch (epi) {
    case ZO_EPI_F32: return launch_pair_t<ZO_EPI_F32>(ma, mb, mb2, a, st);
    case ZO_EPI_BIAS_BF16: return launch_pair_t<ZO_EPI_BIAS_BF16>(ma, mb, mb2, a, st);
    case ZO_EPI_BIAS_GELU_BF16: return launch_pair_t<ZO_EPI_BIAS_GELU_BF16>(ma, mb, mb2, a, st);
    case ZO_EPI_BIAS_RELU_BF16: return launch_pair_t<ZO_EPI_BIAS_RELU_BF16>(ma, mb, mb2, a, st);
    case ZO_EPI_BIAS_RESID_F32: return launch_pair_t<ZO_EPI_BIAS_RESID_F32>(ma, mb, mb2, a, st);
    case ZO_EPI_CE: return launch_pair_t<ZO_EPI_CE>(ma, mb, mb2, a, st);
  }
  set_error("zo_gemm_bf16: unknown epilogue %d", epi);
  return ZO_ERR_CONFIG;
}

}  // namespace

// shared with attention_tc.cu: cached 2-D bf16 SW128 tensor map
int tma_map_bf16(const void* ptr, int64_t inner, int64_t outer, int64_t ld, int box_in, int box_out,
                 CUtensorMap* out) {
  return get_map(ptr, inner, outer, ld, box_in, box_out, out);
}

int64_t gemm_ce_tiles(int64_t N) { return 2 * ((N + 255) / 256); }   // one partial per 128-column half

int gemm_launch(const void* A, int64_t lda, const void* B, int64_t ldb, int64_t M, int64_t N, int64_t K, int epi,
                const float* bias, void* out, int64_t ldo, const int32_t* targets, float* ce_part, float* ce_tgt,
                int32_t* err, cudaStream_t st, const void* B2, const float* bias2, int64_t m_split) {
  const bool bkm = (epi & ZO_GEMM_B_KMAJOR) != 0;
  epi &= ~ZO_GEMM_B_KMAJOR;
  if (M == 0 || N == 0) return ZO_OK;
  if (K <= 0) { set_error("zo_gemm_bf16: K must be positive"); return ZO_ERR_CONFIG; }
  if (lda % 8 || ldb % 8 || lda < K || ldb < (bkm ? K : N)) {
    set_error("zo_gemm_bf16: lda/ldb must be multiples of 8 and >= K / (N, or K with B_KMAJOR) (lda=%lld ldb=%lld)",
              (long long)lda,
              (long long)ldb);
    return ZO_ERR_CONFIG;
  }
  if ((reinterpret_cast<uintptr_t>(A) & 15) || (reinterpret_cast<uintptr_t>(B) & 15) ||
      (reinterpret_cast<uintptr_t>(B2) & 15)) {
    set_error("zo_gemm_bf16: operands must be 16-byte aligned");
    return ZO_ERR_CONFIG;
  }
  // 128 x 256 tiles (measured: BN=256 beats BN=128 even below one wave), CTA
  // pairs with 256 x 256 tiles once M spans more than one 128-row tile
  constexpr int bn = 256;
  CUtensorMap ma, mb;
  int rc = get_map(A, K, M, lda, kBK, kBM, &ma);
  if (rc) return rc;
  const bool pair = M > kBM;
  // B tile: MN-major 64-column boxes, or K-major (rows = N) boxes of 128 (pair half) / BN rows
  rc = bkm ? get_map(B, K, N, ldb, kBK, pair ? 128 : bn, &mb) : get_map(B, N, K, ldb, 64, kBK, &mb);
  if (rc) return rc;
  CUtensorMap mb2 = mb;
  if (m_split) {
    if (!pair || m_split % 256 || m_split >= M || !B2) {
      set_error("zo_gemm_bf16_split: m_split=%lld must be a multiple of 256 in (0, M=%lld) with M > 128",
                (long long)m_split, (long long)M);
      return ZO_ERR_CONFIG;
    }
    rc = bkm ? get_map(B2, K, N, ldb, kBK, 128, &mb2) : get_map(B2, N, K, ldb, 64, kBK, &mb2);
    if (rc) return rc;
  }
  GemmArgs a{M, N, K, bias, out, ldo, targets, ce_part, ce_tgt, err, gemm_ce_tiles(N), m_split, bias2};
  if (pair) return launch_pair(epi, bkm, ma, mb, mb2, a, st);
  return launch_bn<bn>(epi, bkm, ma, mb, a, st);
}

}  // namespace zo
