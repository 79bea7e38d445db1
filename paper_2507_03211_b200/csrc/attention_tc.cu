// Causal attention on the 5th-generation tensor cores (src/zosim/model.py:
// 325-332), head_dim 64 or 128.  One CTA per SM, persistent over (query tile of 128,
// head, batch) work items, heaviest (latest) query tiles first.
//
//   warp 0      TMA producer: Q tile (once per item), K/V blocks of 128 keys
//               (kKV-stage ring, so loads run ahead across short items) from
//               the fused QKV activation
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer:
//                 S_j  = Q K_j^T      M=128 N=128 K=64   -> TMEM S[j%2]
//                 PV_j = P_j V_j      M=128 N=64  K=128  -> TMEM PV[j%2]
//               S_{j+1} is issued before PV_j so the tensor core computes the
//               next scores while the softmax warps work on the current ones
//   warps 2..9  softmax, two warps per query row group (each owns 64 of the 128
//               key columns and 32 output columns): S from TMEM, causal mask,
//               online max / sum (fp32, exp2), P = bf16(exp2(s - m)) written
//               straight into shared memory in the UMMA K-major SW128 layout,
//               O = O * alpha + PV_j kept in registers, final O / l to global.
// TMEM: S0 [0,128) S1 [128,256) PV0 [256,320) PV1 [320,384) of 512 columns.
#include <stdlib.h>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace zo {

int tma_map_bf16(const void* ptr, int64_t inner, int64_t outer, int64_t ld, int box_in, int box_out,
                 CUtensorMap* out);

// ZO_ATTN_TRACE (debug builds only): clock64 stamps of CTA 0's softmax warp 2
// (TR), MMA warp (TRW) and producer (TRP), read back by zo_attn_trace_read;
// tools/attn_trace.py prints the timeline.  Compiled out otherwise.
#ifdef ZO_ATTN_TRACE
__device__ long long g_attn_trace[4096];
#define TR(slot) do { if (blockIdx.x == 0 && threadIdx.x == 64 && (slot) < 4096) g_attn_trace[(slot)] = clock64(); } while (0)
#define TRW(slot) do { if (blockIdx.x == 0 && threadIdx.x == 32 && (slot) < 4096) g_attn_trace[(slot)] = clock64(); } while (0)
#define TRP(slot) do { if (blockIdx.x == 0 && threadIdx.x == 0 && (slot) < 4096) g_attn_trace[(slot)] = clock64(); } while (0)
#else
#define TR(slot)
#define TRW(slot)
#define TRP(slot)
#endif

namespace {

// Softmax warps: 8 (2 per TMEM lane quarter, 64 key columns each) or 16 (4
// per quarter, 32 key columns each: half the work per thread and twice the
// warps per scheduler to hide the TMEM-load / exchange / MUFU latencies).
#ifndef ZO_ATTN_SOFTMAX_WARPS
#define ZO_ATTN_SOFTMAX_WARPS 8
#endif
constexpr int kSW = ZO_ATTN_SOFTMAX_WARPS;
static_assert(kSW == 8 || kSW == 16, "softmax warps");
constexpr int kNCG = kSW / 4;                // column groups per lane quarter
constexpr int kKC = 128 / kNCG;              // key columns of S per softmax warp
constexpr int kAttnThreads = 64 + 32 * kSW;  // producer, MMA, softmax warps
constexpr int kChunkBytes = 128 * 64 * 2;    // 16 KB: 128 rows x 64 bf16, one SW128 K-chunk
constexpr int kPBytes = 128 * 128 * 2;       // 32 KB: P tile, two 64-key K-chunks

// Per-head-dim layout.  hd 64: Q[2] | K[kKV] | V[kKV] | P[2], 4 K/V stages
// (3 with 16 softmax warps).  hd 128: every Q/K/V tile is two 64-column
// chunks (32 KB); Q single-buffered, 2 K/V stages: 224 KB.  TMEM: S[2] in
// columns [0, 256), PV[2] (hd columns each) from column 256.
template <int HD>
struct AttnCfg {
  static constexpr int kTile = 128 * HD * 2;                 // Q / K / V tile bytes
  static constexpr int kChunks = HD / 64;                    // 64-column SW128 chunks per tile
  static constexpr int kQB = HD == 64 ? 2 : 1;               // Q buffers
#ifdef ZO_ATTN_KV_STAGES
  static constexpr int kKV = ZO_ATTN_KV_STAGES;
#else
  static constexpr int kKV = HD == 64 ? (kSW == 16 ? 3 : 4) : 2;
#endif
  static constexpr int kOC = HD / kNCG;                      // output columns per softmax warp
  static constexpr int kOffQ = 0;
  static constexpr int kOffK = kOffQ + kQB * kTile;
  static constexpr int kOffV = kOffK + kKV * kTile;
  static constexpr int kOffP = kOffV + kKV * kTile;
  static constexpr int kOffBar = kOffP + 2 * kPBytes;
  // row-max / row-sum exchange [kRedBufs][kNCG][128] fp32: parity-double-buffered
  // (one barrier per exchange) when it fits, else one buffer and a second barrier
  static constexpr int kRedBufs = (kOffBar + 256 + 2 * kNCG * 128 * 4 + 1024 <= 232448) ? 2 : 1;
  static constexpr int kOffRed = kOffBar + 256;
  static constexpr int kSmem = kOffRed + kRedBufs * kNCG * 128 * 4 + 1024;
  static_assert(kSmem <= 232448, "attention smem");
  static_assert(8 * (20 + 2 * kKV) + 4 <= 256, "barrier area");
};

struct AttnArgs {
  int batch, seq, heads, ldc;
  int64_t d;            // heads * head_dim
  int n_qt;             // query tiles per sequence
  int items;
  float sl2;            // log2(e) / sqrt(hd)
  __nv_bfloat16* ctx;
};

__device__ __forceinline__ float ex2_approx(float x) {   // MUFU.EX2; ex2(-inf) = 0
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

template <int HD>
__global__ void __launch_bounds__(kAttnThreads, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tm, const AttnArgs a) {
  using C = AttnCfg<HD>;
  constexpr int kKV = C::kKV, kOC = C::kOC, kTile = C::kTile, kCh = C::kChunks;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);
  const uint32_t sQ = base + C::kOffQ, sK = base + C::kOffK, sV = base + C::kOffV, sP = base + C::kOffP;
  const uint32_t bars = base + C::kOffBar;
  // barriers: 0 q_full0, 1 q_empty0, 6-7 s_full, 8-9 s_empty, 10-11 p_full, 12-13 p_empty,
  //           14-15 pv_full, 16-17 pv_empty, 18 q_full1, 19 q_empty1,
  //           20.. kv_full[kKV], 20+kKV.. kv_empty[kKV]
  auto bar = [&](int i) { return bars + 8u * i; };
  auto qfull = [&](uint32_t qb) { return bar(qb ? 18 : 0); };
  auto qempty = [&](uint32_t qb) { return bar(qb ? 19 : 1); };
  auto kvfull = [&](uint32_t st) { return bar(20 + (int)st); };
  auto kvempty = [&](uint32_t st) { return bar(20 + kKV + (int)st); };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gbase + C::kOffBar + 8 * (20 + 2 * kKV));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tm);
    mbar_init(bar(0), 1); mbar_init(bar(1), 1); mbar_init(bar(18), 1); mbar_init(bar(19), 1);
    for (int i = 0; i < kKV; ++i) { mbar_init(kvfull(i), 1); mbar_init(kvempty(i), 1); }
    for (int i = 0; i < 2; ++i) {
      mbar_init(bar(6 + i), 1); mbar_init(bar(8 + i), kSW);
      mbar_init(bar(10 + i), kSW); mbar_init(bar(12 + i), 1);
      mbar_init(bar(14 + i), 1); mbar_init(bar(16 + i), kSW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "r"(512u));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();
  pdl_wait();

  const int n_bh = a.batch * a.heads;
  auto item_coords = [&](int it, int& qt, int& h, int& b) {
    qt = a.n_qt - 1 - it / n_bh;           // heavy (late) query tiles first
    const int bh = it % n_bh;
    h = bh % a.heads;
    b = bh / a.heads;
  };
  auto n_blocks = [&](int qt) {
    const int by_causal = qt + 1;
    const int by_len = (a.seq + 127) / 128;
    return by_causal < by_len ? by_causal : by_len;
  };

  if (warp == 0) {
    // ================= TMA producer =================
    if (lane == 0) {
      uint32_t kvc = 0, it_local = 0;
      for (int it = blockIdx.x; it < a.items; it += gridDim.x, ++it_local) {
        int qt, h, b;
        item_coords(it, qt, h, b);
        const int row0 = b * a.seq;
        const uint32_t qb = it_local % C::kQB, qph = (it_local / C::kQB) & 1u;
        mbar_wait(qempty(qb), qph ^ 1u);
        TRP(3072 + (int)it_local);
        mbar_expect_tx(qfull(qb), kTile);
#pragma unroll
        for (int ch = 0; ch < kCh; ++ch)
          tma_load_2d(sQ + qb * kTile + ch * kChunkBytes, &tm, qfull(qb), h * HD + ch * 64, row0 + qt * 128);
        const int nkb = n_blocks(qt);
        for (int j = 0; j < nkb; ++j, ++kvc) {
          const uint32_t st = kvc % kKV, ph = (kvc / kKV) & 1u;
          mbar_wait(kvempty(st), ph ^ 1u);
          TRP(2048 + (int)kvc);
          mbar_expect_tx(kvfull(st), 2 * kTile);
#pragma unroll
          for (int ch = 0; ch < kCh; ++ch) {
            tma_load_2d(sK + st * kTile + ch * kChunkBytes, &tm, kvfull(st), (int)(a.d + h * HD + ch * 64),
                        row0 + j * 128);
            tma_load_2d(sV + st * kTile + ch * kChunkBytes, &tm, kvfull(st), (int)(2 * a.d + h * HD + ch * 64),
                        row0 + j * 128);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer =================
    // S: A = Q (K-major), B = K (K-major), M=N=128, K = hd in 64-column chunks.
    // PV: A = P (K-major), B = V (MN-major: hd contiguous, 64-wide N chunks
    // 16 KB apart), M=128, N=hd.
    const uint32_t idesc_s = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(128 >> 3) << 17) |
                             ((uint32_t)(128 >> 4) << 24);
    const uint32_t idesc_pv = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | ((uint32_t)(HD >> 3) << 17) |
                              ((uint32_t)(128 >> 4) << 24);
    uint32_t kvc = 0, sc = 0, it_local = 0;
    auto issue_pv = [&](uint32_t c, uint32_t kv) {
      const uint32_t pb = c & 1u, ph = (c >> 1) & 1u, st = kv % kKV;
      mbar_wait(bar(10 + pb), ph);               // P_c written
      TRW(1024 + 4 * (int)c + 3);
      mbar_wait(bar(16 + pb), ph ^ 1u);          // PV buffer drained by the softmax warps
      tc_fence_after();
      if (lane == 0) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {         // 128 keys = 8 x K16
          const uint64_t ad = desc_sw128(sP + pb * kPBytes + (kk >> 2) * kChunkBytes + (kk & 3) * 32, 16, 1024);
          const uint64_t bd = desc_sw128(sV + st * kTile + kk * 2048, kChunkBytes, 1024);
          tc_mma_f16(tmem + 256 + pb * HD, ad, bd, idesc_pv, kk != 0 ? 1u : 0u);
        }
        tc_commit(bar(14 + pb));                  // PV ready
        tc_commit(kvempty(st));                   // K/V stage free
        tc_commit(bar(12 + pb));                  // P buffer free
      }
      __syncwarp();
    };
    // PV of the previous block is issued after the next S, and that chain
    // runs across item boundaries: the first S of item i+1 is already on the
    // tensor core while the softmax warps finish item i (no per-item bubble)
    bool have_prev = false;
    uint32_t prev_c = 0, prev_kv = 0;
    for (int it = blockIdx.x; it < a.items; it += gridDim.x, ++it_local) {
      int qt, h, b;
      item_coords(it, qt, h, b);
      const int nkb = n_blocks(qt);
      const uint32_t qb = it_local % C::kQB;
      mbar_wait(qfull(qb), (it_local / C::kQB) & 1u);
      for (int j = 0; j < nkb; ++j) {
        const uint32_t c = sc + j, kv = kvc + j;
        const uint32_t sb = c & 1u, ph = (c >> 1) & 1u;
        TRW(1024 + 4 * (int)c + 0);
        mbar_wait(kvfull(kv % kKV), (kv / kKV) & 1u);    // K_j, V_j landed
        TRW(1024 + 4 * (int)c + 1);
        mbar_wait(bar(8 + sb), ph ^ 1u);                 // S buffer free
        TRW(1024 + 4 * (int)c + 2);
        tc_fence_after();
        if (lane == 0) {
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk) {     // K16 steps; 4 per 64-column chunk
            const uint32_t off = (kk >> 2) * kChunkBytes + (kk & 3) * 32;
            const uint64_t ad = desc_sw128(sQ + qb * kTile + off, 16, 1024);
            const uint64_t bd = desc_sw128(sK + (kv % kKV) * kTile + off, 16, 1024);
            tc_mma_f16(tmem + sb * 128, ad, bd, idesc_s, kk != 0 ? 1u : 0u);
          }
          tc_commit(bar(6 + sb));                 // S ready
          if (j == nkb - 1) tc_commit(qempty(qb));  // Q buffer no longer needed
        }
        __syncwarp();
        if (have_prev) issue_pv(prev_c, prev_kv);
        prev_c = c;
        prev_kv = kv;
        have_prev = true;
      }
      sc += nkb;
      kvc += nkb;
    }
    if (have_prev) issue_pv(prev_c, prev_kv);
  } else {
    // ================= softmax / output =================
    // warp (quarter q, column group cg): rows 32q..32q+31, key columns
    // [kKC*cg, +kKC) of S, output columns [kOC*cg, +kOC).  The row max and the
    // final row sum are exchanged between the kNCG warps of a quarter through a
    // parity-double-buffered shared array: one named barrier per exchange.
    const int quarter = warp & 3, cg = (warp - 2) >> 2;
    const int r = quarter * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    float* red = reinterpret_cast<float*>(gbase + C::kOffRed);   // [kRedBufs][kNCG][128]
    auto group_sync = [&]() { asm volatile("bar.sync %0, %1;\n" ::"r"(1 + quarter), "r"(kNCG * 32) : "memory"); };
    uint32_t par = 0;
    auto exchange = [&](float v, bool is_max) {
      float* rb = red + par * (kNCG * 128);
      rb[cg * 128 + r] = v;
      group_sync();
      float t = rb[r];
#pragma unroll
      for (int g = 1; g < kNCG; ++g) t = is_max ? fmaxf(t, rb[g * 128 + r]) : t + rb[g * 128 + r];
      if constexpr (C::kRedBufs == 2) par ^= 1u;
      else group_sync();                        // all read before the next exchange overwrites
      return t;
    };
    uint32_t sc = 0;
    for (int it = blockIdx.x; it < a.items; it += gridDim.x) {
      int qt, h, b;
      item_coords(it, qt, h, b);
      const int nkb = n_blocks(qt);
      const int qi = qt * 128 + r;
      float m = -INFINITY, l = 0.f, alpha_prev = 0.f;
      const int tr_item = (it - blockIdx.x) / gridDim.x;
      TR(tr_item * 32 + 0);
      (void)tr_item;
      float o[kOC];
#pragma unroll
      for (int i = 0; i < kOC; ++i) o[i] = 0.f;
      // O <- O * alpha_c + PV_c  (alpha_c rescales O to block c's running max)
      auto accumulate_pv = [&](uint32_t cc, float al) {
        const uint32_t pb = cc & 1u, pph = (cc >> 1) & 1u;
        mbar_wait(bar(14 + pb), pph);
        tc_fence_after();
        constexpr int W = kOC < 32 ? kOC : 32;     // TMEM load width
        uint32_t pv[kOC / W][W];
#pragma unroll
        for (int q = 0; q < kOC / W; ++q) tmem_ld_nw(tmem + 256 + pb * HD + cg * kOC + q * W + lane_off, pv[q]);
        tmem_wait_ld();
#pragma unroll
        for (int q = 0; q < kOC / W; ++q)
#pragma unroll
          for (int i = 0; i < W; ++i) o[q * W + i] = fmaf(o[q * W + i], al, __uint_as_float(pv[q][i]));
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar(16 + pb));
      };
      for (int j = 0; j < nkb; ++j) {
        const uint32_t c = sc + j, sb = c & 1u, ph = (c >> 1) & 1u;
        const bool need_mask = (j * 128 + 127 > qt * 128) || ((j + 1) * 128 > a.seq);
        TR(tr_item * 32 + 1 + 3 * j);
        mbar_wait(bar(6 + sb), ph);
        TR(tr_item * 32 + 2 + 3 * j);
        tc_fence_after();
        constexpr int NCH = kKC / 32;
        uint32_t sv[NCH][32];
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch)
          tmem_ld_32x32b_x32_nw(tmem + sb * 128 + cg * kKC + ch * 32 + lane_off, sv[ch]);
        tmem_wait_ld();
        if (need_mask) {
#pragma unroll
          for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const int ki = j * 128 + cg * kKC + ch * 32 + i;
              if (!(ki <= qi && ki < a.seq)) sv[ch][i] = __float_as_uint(-INFINITY);
            }
        }
        float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            mx0 = fmaxf(mx0, __uint_as_float(sv[ch][i]));
            mx1 = fmaxf(mx1, __uint_as_float(sv[ch][i + 1]));
          }
        const float mx = exchange(fmaxf(mx0, mx1), true);
        const float m_new = fmaxf(m, mx);
        const float mb = m_new == -INFINITY ? 0.f : m_new * a.sl2;
        const float alpha = m == -INFINITY ? 0.f : ex2_approx(fmaf(m, a.sl2, -mb));
        mbar_wait(bar(12 + sb), ph ^ 1u);         // P buffer free
        float sum0 = 0.f, sum1 = 0.f;
        // this warp's keys: 64-key K-chunk (cg * kKC) / 64, 16-B units from ((cg * kKC) % 64) / 8
        const uint32_t region = sP + sb * kPBytes + ((cg * kKC) >> 6) * kChunkBytes + r * 128;
        const int unit0 = ((cg * kKC) & 63) >> 3;
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) {
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            const float p0 = ex2_approx(fmaf(__uint_as_float(sv[ch][i]), a.sl2, -mb));
            const float p1 = ex2_approx(fmaf(__uint_as_float(sv[ch][i + 1]), a.sl2, -mb));
            sum0 += p0;
            sum1 += p1;
            __nv_bfloat162 h2 = __floats2bfloat162_rn(p0, p1);
            pk[i >> 1] = *reinterpret_cast<uint32_t*>(&h2);
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int unit = unit0 + ch * 4 + q;
            const uint32_t addr = region + ((unit ^ (r & 7)) << 4);
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(addr), "r"(pk[4 * q]),
                         "r"(pk[4 * q + 1]), "r"(pk[4 * q + 2]), "r"(pk[4 * q + 3])
                         : "memory");
          }
        }
        tc_fence_before();
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) { mbar_arrive(bar(8 + sb)); mbar_arrive(bar(10 + sb)); }   // S read, P written
        TR(tr_item * 32 + 3 + 3 * j);
        l = fmaf(l, alpha, sum0 + sum1);          // this warp's running sum over its key columns
        m = m_new;
        // deferred: fold PV of the PREVIOUS block (ready while we computed this one)
        if (j > 0) accumulate_pv(c - 1, alpha_prev);
        alpha_prev = alpha;
      }
      TR(tr_item * 32 + 20);
      accumulate_pv(sc + nkb - 1, alpha_prev);
      TR(tr_item * 32 + 21);
      sc += nkb;
      const float lt = exchange(l, false);
      if (qi < a.seq) {
        const float inv = lt > 0.f ? 1.f / lt : 0.f;
        __nv_bfloat16* out = a.ctx + ((int64_t)b * a.seq + qi) * a.ldc + (int64_t)h * HD + cg * kOC;
#pragma unroll
        for (int i = 0; i < kOC; i += 8) {
          uint32_t pk[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            __nv_bfloat162 h2 = __floats2bfloat162_rn(o[i + 2 * k] * inv, o[i + 2 * k + 1] * inv);
            pk[k] = *reinterpret_cast<uint32_t*>(&h2);
          }
          *reinterpret_cast<uint4*>(out + i) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        }
      }
      TR(tr_item * 32 + 22);
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512u));
  }
}

// ----------------------------------------------------------------------------
// hd 64: two query tiles in flight per CTA ("ping-pong").  A work item is the
// same query tile qt of two (batch, head) pairs -- tiles A and B have the same
// causal length, so their pipelines stay in step.  Each tile has its own four
// softmax warps (one thread per query row, the whole 128-key row of S in
// registers: no cross-warp row exchange), so while one tile's warps run the
// exponentials the other tile's S / PV MMAs run on the tensor core, and one
// tile's per-item tail (last PV wait, output store) hides under the other's
// softmax.  O accumulates in TMEM (PV with accumulate = 1); a row's running
// max is only raised -- and O, l rescaled -- when it grows by more than 2^8,
// so the rescale (a TMEM read-modify-write by the row's own thread) is rare.
//   warp 0     TMA: Q_A, Q_B once per item; K/V blocks (A0, B0, A1, B1, ...)
//              through a 4-stage ring
//   warp 1     TMEM alloc + MMA issue: per block j and tile t:
//                S_t,j+1 = Q_t K_t,j+1^T  (issued as soon as S_t,j is in registers)
//                PV:  O_t += P_t,j V_t,j  (after the softmax wrote P_t,j)
//   warps 2-5  softmax + output of tile A, warps 6-9 of tile B
// TMEM: S_A [0,128) S_B [128,256) O_A[2] [256,384) O_B[2] [384,512)  (O
// double-buffered across items so the next item's first PV never waits for
// the previous item's output read).
// ----------------------------------------------------------------------------
namespace pp {
constexpr int kThreads = 320;
constexpr int kQB = 128 * 64 * 2;          // 16 KB Q tile
constexpr int kKVB = 2 * kQB;              // K + V of one block: 32 KB
constexpr int kStages = 4;
constexpr int kPB = 128 * 128 * 2;         // 32 KB P tile (two 64-key SW128 chunks)
constexpr int kOffQ = 0;
constexpr int kOffKV = kOffQ + 2 * kQB;
constexpr int kOffP = kOffKV + kStages * kKVB;
constexpr int kOffBar = kOffP + 2 * kPB;
constexpr int kNBar = 26;
constexpr int kSmem = kOffBar + 8 * kNBar + 16 + 1024;
static_assert(kSmem <= 232448, "attention pp smem");
// barrier indices
constexpr int QF = 0, QE = 2, KVF = 4, KVE = 8, SF = 12, SE = 14, PF = 16, PVD = 18, OE = 20;  // OE: [t][2]
}  // namespace pp

__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}
// sm_100 packed-fp32 and 3-input ops (FFMA2 / FADD2 / FMNMX3)
__device__ __forceinline__ uint64_t pack_f32x2(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ uint64_t pack_u32x2(uint32_t lo, uint32_t hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "r"(lo), "r"(hi));
  return r;
}
__device__ __forceinline__ void unpack_f32x2(uint64_t v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ uint64_t ffma_f32x2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t add_f32x2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

__global__ void __launch_bounds__(pp::kThreads, 1)
    attn_pp_kernel(const __grid_constant__ CUtensorMap tm, const AttnArgs a) {
  using namespace pp;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);
  const uint32_t sQ = base + kOffQ, sKV = base + kOffKV, sP = base + kOffP;
  const uint32_t bars = base + kOffBar;
  auto bar = [&](int i) { return bars + 8u * i; };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gbase + kOffBar + 8 * kNBar);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tm);
    for (int t = 0; t < 2; ++t) {
      mbar_init(bar(QF + t), 1); mbar_init(bar(QE + t), 1);
      mbar_init(bar(SF + t), 1); mbar_init(bar(SE + t), 4);
      mbar_init(bar(PF + t), 4); mbar_init(bar(PVD + t), 1);
      mbar_init(bar(OE + 2 * t), 4); mbar_init(bar(OE + 2 * t + 1), 4);
    }
    for (int s = 0; s < kStages; ++s) { mbar_init(bar(KVF + s), 1); mbar_init(bar(KVE + s), 1); }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "r"(512u));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();
  pdl_wait();

  const int n_bh = a.batch * a.heads;
  const int n_pairs = (n_bh + 1) >> 1;
  // item -> (query tile, first (b,h) of the pair); heaviest (latest) tiles first
  auto coords = [&](int it, int& qt, int& bh0) {
    qt = a.n_qt - 1 - it / n_pairs;
    bh0 = 2 * (it % n_pairs);
  };

  if (warp == 0) {
    // ============================ TMA producer ============================
    if (lane == 0) {
      uint32_t kvc = 0, qc[2] = {0u, 0u};
      for (int it = blockIdx.x; it < a.items; it += gridDim.x) {
        int qt, bh0;
        coords(it, qt, bh0);
        const int T = bh0 + 1 < n_bh ? 2 : 1;
        for (int t = 0; t < T; ++t) {
          const int bh = bh0 + t, b = bh / a.heads, h = bh % a.heads;
          mbar_wait(bar(QE + t), (qc[t]++ & 1u) ^ 1u);
          mbar_expect_tx(bar(QF + t), kQB);
          tma_load_2d(sQ + t * kQB, &tm, bar(QF + t), h * 64, b * a.seq + qt * 128);
        }
        for (int j = 0; j <= qt; ++j) {
          for (int t = 0; t < T; ++t, ++kvc) {
            const int bh = bh0 + t, b = bh / a.heads, h = bh % a.heads;
            const uint32_t st = kvc % kStages, ph = (kvc / kStages) & 1u;
            TRP(2048 + 2 * (int)kvc);
            mbar_wait(bar(KVE + st), ph ^ 1u);
            TRP(2048 + 2 * (int)kvc + 1);
            mbar_expect_tx(bar(KVF + st), kKVB);
            tma_load_2d(sKV + st * kKVB, &tm, bar(KVF + st), (int)(a.d + h * 64), b * a.seq + j * 128);
            tma_load_2d(sKV + st * kKVB + kQB, &tm, bar(KVF + st), (int)(2 * a.d + h * 64), b * a.seq + j * 128);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ============================ MMA issuer =============================
    const uint32_t idesc_s = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(128 >> 3) << 17) |
                             ((uint32_t)(128 >> 4) << 24);
    const uint32_t idesc_pv = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | ((uint32_t)(64 >> 3) << 17) |
                              ((uint32_t)(128 >> 4) << 24);
    uint32_t kvc = 0;
    uint32_t qc[2] = {0u, 0u}, sc[2] = {0u, 0u}, pc[2] = {0u, 0u}, ic[2] = {0u, 0u};
    int trm = 0;
    auto issue_s = [&](int t, uint32_t kv, bool last) {
      TRW(1024 + 4 * trm);
      mbar_wait(bar(KVF + kv % kStages), (kv / kStages) & 1u);     // K, V landed
      TRW(1024 + 4 * trm + 1);
      mbar_wait(bar(SE + t), (sc[t] & 1u) ^ 1u);                   // S_t drained into registers
      TRW(1024 + 4 * trm + 2);
      ++trm;
      tc_fence_after();
      if (lane == 0) {
        const uint32_t k0 = sKV + (kv % kStages) * kKVB;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          tc_mma_f16(tmem + t * 128, desc_sw128(sQ + t * kQB + kk * 32, 16, 1024), desc_sw128(k0 + kk * 32, 16, 1024),
                     idesc_s, kk != 0 ? 1u : 0u);
        tc_commit(bar(SF + t));
        if (last) tc_commit(bar(QE + t));                          // Q_t no longer read
      }
      __syncwarp();
      ++sc[t];
    };
    auto issue_pv = [&](int t, uint32_t kv, bool first) {
      TRW(1024 + 4 * trm);
      mbar_wait(bar(PF + t), pc[t] & 1u);                          // P_t written (and O_t rescaled)
      TRW(1024 + 4 * trm + 1);
      ++trm;
      const uint32_t ob = ic[t] & 1u;
      if (first) mbar_wait(bar(OE + 2 * t + ob), ((ic[t] >> 1) & 1u) ^ 1u);   // O buffer read out
      tc_fence_after();
      if (lane == 0) {
        const uint32_t v0 = sKV + (kv % kStages) * kKVB + kQB;
        const uint32_t p0 = sP + t * kPB;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)                              // 128 keys = 8 x K16
          tc_mma_f16(tmem + 256 + t * 128 + ob * 64, desc_sw128(p0 + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024),
                     desc_sw128(v0 + kk * 2048, 16384, 1024), idesc_pv, (!first || kk != 0) ? 1u : 0u);
        tc_commit(bar(PVD + t));                                     // PV done: O_t final / P_t free
        tc_commit(bar(KVE + kv % kStages));                          // K/V stage free
      }
      __syncwarp();
      ++pc[t];
    };
    for (int it = blockIdx.x; it < a.items; it += gridDim.x) {
      int qt, bh0;
      coords(it, qt, bh0);
      const int T = bh0 + 1 < n_bh ? 2 : 1;
      const int nkb = qt + 1;
      for (int t = 0; t < T; ++t) mbar_wait(bar(QF + t), qc[t]++ & 1u);
      for (int t = 0; t < T; ++t) issue_s(t, kvc + t, nkb == 1);
      for (int j = 0; j < nkb; ++j) {
        // the next block's S of both tiles first: a tile's softmax finds S_j+1
        // ready when it finishes block j whatever the other tile is doing
        if (j + 1 < nkb)
          for (int t = 0; t < T; ++t) issue_s(t, kvc + (j + 1) * T + t, j + 2 == nkb);
        for (int t = 0; t < T; ++t) issue_pv(t, kvc + j * T + t, j == 0);
      }
      kvc += nkb * T;
      for (int t = 0; t < T; ++t) ++ic[t];
    }
  } else {
    // ====================== softmax + output (tile t) =====================
    // Warp (t, quarter) owns query rows 32*quarter .. +31 of tile t; tile A's
    // and tile B's warps of a quarter share one SM sub-partition (and its MUFU
    // pipe: two warps issuing exponentials together keep it busy, one alone
    // reaches about half its rate -- measured with an alternating hand-off).
    const int t = (warp - 2) >> 2;
    const int quarter = warp & 3;               // TMEM lane quarter this warp may access
    const int r = quarter * 32 + lane;          // query row within the tile
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const uint32_t s_tm = tmem + t * 128 + lane_off;
    const uint32_t prow = sP + t * kPB + r * 128;   // row r of chunk 0 (keys 0-63); chunk 1 at +16 KB
    const uint64_t sl2x2 = pack_f32x2(a.sl2, a.sl2);
    uint32_t sc = 0, pw = 0, ic = 0;
    int trn = 0;
    (void)trn;
    for (int it = blockIdx.x; it < a.items; it += gridDim.x) {
      int qt, bh0;
      coords(it, qt, bh0);
      if (bh0 + t >= n_bh) continue;            // odd (b,h) count: no tile B in the last pair
      const int bh = bh0 + t, b = bh / a.heads, h = bh % a.heads;
      const int qi = qt * 128 + r;
      const int q_lo = qt * 128 + quarter * 32, q_hi = q_lo + 31;   // this warp's query rows
      const uint32_t ob = ic & 1u;
      const uint32_t o_tm = tmem + 256 + t * 128 + ob * 64 + lane_off;
      float m = -INFINITY, l = 0.f;
      for (int j = 0; j <= qt; ++j) {
        const int tr = (trn++) * 8;
        (void)tr;
        TR(tr + 0);
        mbar_wait(bar(SF + t), sc & 1u);
        ++sc;
        TR(tr + 1);
        tc_fence_after();
        uint32_t s[4][32];
#pragma unroll
        for (int c = 0; c < 4; ++c) tmem_ld_32x32b_x32_nw(s_tm + c * 32, s[c]);
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar(SE + t));  // S_t may be overwritten by S_t,j+1
        // 32-key chunk c: dead (no row of the warp sees a key of it), full (every
        // row sees every key) or ragged (element mask: causal diagonal / seq end)
        const int k0 = j * 128;
        bool live[4], full[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int kc = k0 + c * 32;
          live[c] = kc <= q_hi && kc < a.seq;
          full[c] = kc + 31 <= q_lo && kc + 32 <= a.seq;
        }
        float mc[3] = {-INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          if (!live[c]) continue;
          if (!full[c]) {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const int ki = k0 + c * 32 + i;
              if (!(ki <= qi && ki < a.seq)) s[c][i] = __float_as_uint(-INFINITY);
            }
          }
#pragma unroll
          for (int i = 0; i < 30; i += 6) {
            mc[0] = fmax3(mc[0], __uint_as_float(s[c][i]), __uint_as_float(s[c][i + 1]));
            mc[1] = fmax3(mc[1], __uint_as_float(s[c][i + 2]), __uint_as_float(s[c][i + 3]));
            mc[2] = fmax3(mc[2], __uint_as_float(s[c][i + 4]), __uint_as_float(s[c][i + 5]));
          }
          mc[0] = fmax3(mc[0], __uint_as_float(s[c][30]), __uint_as_float(s[c][31]));
        }
        const float mx = fmax3(mc[0], mc[1], mc[2]);
        // lazy max: raise the scaling max only when the row max grew by > 2^8
        const float m_new = fmaxf(m, mx);
        float m_use = m, alpha = 1.f;
        bool rescale = false;
        if (m == -INFINITY) {
          m_use = m_new;
        } else if ((m_new - m) * a.sl2 > 8.f) {
          m_use = m_new;
          alpha = ex2_approx((m - m_new) * a.sl2);
          rescale = true;
        }
        const float mb = m_use == -INFINITY ? 0.f : m_use * a.sl2;
        const uint64_t nmb2 = pack_f32x2(-mb, -mb);
        TR(tr + 2);
        if (j > 0) {                               // PV_t,j-1 done: P_t free, O_t stable
          mbar_wait(bar(PVD + t), pw & 1u);
          ++pw;
        }
        TR(tr + 3);
        // P = exp2(s * log2e / sqrt(hd) - mb) -> bf16, straight into the K-major SW128 P tile
        uint64_t sum2[2] = {0ull, 0ull};
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const uint32_t rowc = prow + (c >> 1) * 16384;
          const int u0 = (c & 1) * 4;              // 16-B units of this 32-key chunk within the 128-B row
          if (!live[c]) {
#pragma unroll
            for (int q = 0; q < 4; ++q) st_shared_v4(rowc + (((u0 + q) ^ (r & 7)) << 4), 0u, 0u, 0u, 0u);
            continue;
          }
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 32; i += 2) {
            const uint64_t x2 = ffma_f32x2(pack_u32x2(s[c][i], s[c][i + 1]), sl2x2, nmb2);
            float x0, x1;
            unpack_f32x2(x2, x0, x1);
            const float p0 = ex2_approx(x0), p1 = ex2_approx(x1);
            sum2[(i >> 1) & 1] = add_f32x2(sum2[(i >> 1) & 1], pack_f32x2(p0, p1));
            __nv_bfloat162 h2 = __floats2bfloat162_rn(p0, p1);
            pk[i >> 1] = *reinterpret_cast<uint32_t*>(&h2);
          }
#pragma unroll
          for (int q = 0; q < 4; ++q)
            st_shared_v4(rowc + (((u0 + q) ^ (r & 7)) << 4), pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
        }
        TR(tr + 4);
        float s0, s1, s2, s3;
        unpack_f32x2(sum2[0], s0, s1);
        unpack_f32x2(sum2[1], s2, s3);
        l = fmaf(l, alpha, (s0 + s1) + (s2 + s3));
        m = m_use;
        if (__any_sync(0xffffffffu, rescale)) {   // O_t *= alpha (rows that did not rescale: alpha = 1)
          tc_fence_after();
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            uint32_t o[32];
            tmem_ld_32x32b_x32_nw(o_tm + c * 32, o);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
            tmem_st_32x32b_x32(o_tm + c * 32, o);
          }
          tmem_wait_st();
        }
        fence_proxy_async_smem();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar(PF + t));
        TR(tr + 5);
      }
      // item end: O_t = sum_j P_t,j V_t,j (up to the lazy scale), out = O / l
      mbar_wait(bar(PVD + t), pw & 1u);
      ++pw;
      TR(trn * 8 - 2);
      tc_fence_after();
      uint32_t o[2][32];
      tmem_ld_32x32b_x32_nw(o_tm, o[0]);
      tmem_ld_32x32b_x32_nw(o_tm + 32, o[1]);
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar(OE + 2 * t + ob));
      ++ic;
      if (qi < a.seq) {
        const float inv = l > 0.f ? 1.f / l : 0.f;
        __nv_bfloat16* out = a.ctx + ((int64_t)b * a.seq + qi) * a.ldc + (int64_t)h * 64;
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int i = 0; i < 32; i += 8) {
            uint32_t pk[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              __nv_bfloat162 h2 = __floats2bfloat162_rn(__uint_as_float(o[c][i + 2 * k]) * inv,
                                                        __uint_as_float(o[c][i + 2 * k + 1]) * inv);
              pk[k] = *reinterpret_cast<uint32_t*>(&h2);
            }
            *reinterpret_cast<uint4*>(out + c * 32 + i) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
          }
      }
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512u));
  }
}

int attention_pp_launch(const __nv_bfloat16* qkv, int64_t ldq, int64_t batch, int64_t seq, int64_t heads,
                        __nv_bfloat16* ctx, int64_t ldc, cudaStream_t st) {
  CUtensorMap tm;
  int rc = tma_map_bf16(qkv, 3 * heads * 64, batch * seq, ldq, 64, 128, &tm);
  if (rc) return rc;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(attn_pp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, pp::kSmem);
    if (e != cudaSuccess) { set_error("attn_pp smem attribute: %s", cudaGetErrorString(e)); return ZO_ERR_CUDA; }
    attr = true;
  }
  AttnArgs a;
  a.batch = (int)batch;
  a.seq = (int)seq;
  a.heads = (int)heads;
  a.ldc = (int)ldc;
  a.d = heads * 64;
  a.n_qt = (int)((seq + 127) / 128);
  a.items = a.n_qt * (int)((batch * heads + 1) / 2);
  a.sl2 = 1.4426950408889634f / 8.0f;   // log2(e) / sqrt(64)
  a.ctx = ctx;
  const int grid = a.items < num_sms() ? a.items : num_sms();
  launch_k(attn_pp_kernel, dim3(grid), dim3(pp::kThreads), pp::kSmem, st, tm, a);
  return launch_status("attn_pp_kernel");
}

template <int HD>
int attention_tc_launch_t(const __nv_bfloat16* qkv, int64_t ldq, int64_t batch, int64_t seq, int64_t heads,
                          __nv_bfloat16* ctx, int64_t ldc, cudaStream_t st) {
  using C = AttnCfg<HD>;
  CUtensorMap tm;
  const int64_t rows = batch * seq;
  int rc = tma_map_bf16(qkv, 3 * heads * HD, rows, ldq, 64, 128, &tm);
  if (rc) return rc;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(attn_tc_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
    if (e != cudaSuccess) { set_error("attn_tc smem attribute: %s", cudaGetErrorString(e)); return ZO_ERR_CUDA; }
    attr = true;
  }
  AttnArgs a;
  a.batch = (int)batch;
  a.seq = (int)seq;
  a.heads = (int)heads;
  a.ldc = (int)ldc;
  a.d = heads * HD;
  a.n_qt = (int)((seq + 127) / 128);
  a.items = a.n_qt * (int)(batch * heads);
  a.sl2 = 1.4426950408889634f / sqrtf((float)HD);   // log2(e) / sqrt(hd)
  a.ctx = ctx;
  const int grid = a.items < num_sms() ? a.items : num_sms();
  launch_k(attn_tc_kernel<HD>, dim3(grid), dim3(kAttnThreads), C::kSmem, st, tm, a);
  return launch_status("attn_tc_kernel");
}

}  // namespace

// head_dim 64 or 128, qkv / ctx leading dims multiples of 8, 16-byte aligned.
int attention_tc_launch(const __nv_bfloat16* qkv, int64_t ldq, int64_t batch, int64_t seq, int64_t heads,
                        int64_t hd, __nv_bfloat16* ctx, int64_t ldc, cudaStream_t st) {
  if (hd == 128) return attention_tc_launch_t<128>(qkv, ldq, batch, seq, heads, ctx, ldc, st);
  return attention_pp_launch(qkv, ldq, batch, seq, heads, ctx, ldc, st);
}

}  // namespace zo

#ifdef ZO_ATTN_TRACE
extern "C" int zo_attn_trace_read(long long* host) {
  return (int)cudaMemcpyFromSymbol(host, zo::g_attn_trace, sizeof(long long) * 4096);
}
#endif
