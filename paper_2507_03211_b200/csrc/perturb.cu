// Fused perturb / restore / update kernel (one launch per block or per model).
//
// Reference semantics (src/zosim/zo.py:90-130):
//   perturbed  = dtype(f64(base) + (scale * z))      -- always from the base
//   updated    = dtype(f64(theta) - ((lr*g) * z))
// On the GPU the fp32 master `theta` is never perturbed in place: the
// perturbed copies are written as "shadows" (bf16 GEMM operands / fp32
// vectors) and the master only ever receives the update, so the reference's
// snapshot/restore (zo.py:97-107) is free and exact.  The update of step j is
// folded into the pass that perturbs step j+1 (Alg. 2, zo.py:204-215): one
// read + one write of theta and one write per shadow per element per step.
//
// HBM-bound streaming kernel: 4-element groups (one Philox4x32 call yields
// the 4 normals of a group), float4 theta I/O, persistent grid over tiles.
#include "common.cuh"

namespace zo {

constexpr int kPuThreads = 128;
#ifndef ZO_PU_G
#define ZO_PU_G 4
#endif
constexpr int kPuGroupsPerThread = ZO_PU_G;   // 4-element groups per lane per tile
constexpr int64_t kPuTile = 32 * kPuGroupsPerThread * 4;  // elements per warp tile (512 at G = 4)
constexpr int kPuMaxSmemSegs = 4096;   // prefix entries staged in shared memory (32 KB)

__device__ __forceinline__ void store_shadow(const ZoSegment& s, __nv_bfloat16* w, float* v,
                                             int64_t di, float val) {
  if (s.kind == ZO_SHADOW_BF16) w[di] = __float2bfloat16_rn(val);
  else v[di] = val;
}

template <int ZMODE>
__device__ __forceinline__ void pu_group(const PuParams& p, const ZoSegment& s, int64_t q, int64_t e0, int64_t e1,
                                         int64_t drow, float (&th)[4], bool full, bool theta_vec, bool pending,
                                         bool need_z, bool want_sh, const bool (&sh)[2], const float (&sc32)[2],
                                         uint64_t seed_cur, uint64_t seed_prev, double lrg64, float lrg32) {
  const int64_t eg = q << 2;
  if (pending) {
    if constexpr (ZMODE == ZO_Z_PHILOX) {
      const f32x4 zp = philox_normal4(seed_prev, (uint64_t)q);
      th[0] = fmaf(-lrg32, zp.x, th[0]); th[1] = fmaf(-lrg32, zp.y, th[1]);
      th[2] = fmaf(-lrg32, zp.z, th[2]); th[3] = fmaf(-lrg32, zp.w, th[3]);
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int64_t e = eg + i;
        if (e >= e0 && e < e1)
          th[i] = __double2float_rn(__dsub_rn((double)th[i], __dmul_rn(lrg64, p.z_prev[e - p.z_key0])));
      }
    }
    if (full && theta_vec) {
      *reinterpret_cast<float4*>(p.theta + (eg - p.theta_key0)) = make_float4(th[0], th[1], th[2], th[3]);
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (eg + i >= e0 && eg + i < e1) p.theta[eg + i - p.theta_key0] = th[i];
    }
  }
  if (!want_sh) return;
  float zc[4] = {0.f, 0.f, 0.f, 0.f};
  double zc64[4] = {0.0, 0.0, 0.0, 0.0};
  if (need_z) {
    if constexpr (ZMODE == ZO_Z_PHILOX) {
      const f32x4 z4 = philox_normal4(seed_cur, (uint64_t)q);
      zc[0] = z4.x; zc[1] = z4.y; zc[2] = z4.z; zc[3] = z4.w;
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int64_t e = eg + i;
        if (e >= e0 && e < e1) zc64[i] = p.z_cur[e - p.z_key0];
      }
    }
  }
#pragma unroll
  for (int d = 0; d < 2; ++d) {
    if (!sh[d]) continue;
    float v[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (p.scale[d] == 0.0) v[i] = th[i];
      else if constexpr (ZMODE == ZO_Z_PHILOX) v[i] = fmaf(sc32[d], zc[i], th[i]);
      else v[i] = __double2float_rn(__dadd_rn((double)th[i], __dmul_rn(p.scale[d], zc64[i])));
    }
    const int64_t di = eg + drow;
    if (full && ((di & 3) == 0)) {
      if (s.kind == ZO_SHADOW_BF16) {
        __nv_bfloat162 lo2 = __floats2bfloat162_rn(v[0], v[1]);
        __nv_bfloat162 hi2 = __floats2bfloat162_rn(v[2], v[3]);
        uint2 packed;
        packed.x = *reinterpret_cast<uint32_t*>(&lo2);
        packed.y = *reinterpret_cast<uint32_t*>(&hi2);
        *reinterpret_cast<uint2*>(p.wsh[d] + di) = packed;
      } else {
        *reinterpret_cast<float4*>(p.vsh[d] + di) = make_float4(v[0], v[1], v[2], v[3]);
      }
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (eg + i >= e0 && eg + i < e1) store_shadow(s, p.wsh[d], p.vsh[d], di + i, v[i]);
    }
  }
}


// Fast tile: Philox direction, every group 16-B aligned (all real model
// tensors).  Specialised at compile time on (pending update, bf16) so the hot
// loop has no runtime-flag branches; 32-bit lane offsets from per-tile base
// pointers; the lane's groups run their Philox streams in lockstep.  The
// caller loads theta (one tile ahead).
template <int G>
__device__ __forceinline__ void pu_load_fast(const PuParams& p, int64_t e0, int ngroups, int lane, float4 (&th)[G]) {
  const float4* tp = reinterpret_cast<const float4*>(p.theta + (e0 - p.theta_key0)) + lane;
  const bool full = ngroups >= 32 * G;
#pragma unroll
  for (int g = 0; g < G; ++g)
    if (full || lane + 32 * g < ngroups) th[g] = tp[32 * g];
}

// FULL: a whole 512-element tile, no per-group guards; FULL_MASK says which
// shadows it writes at compile time (3: both, the single-GPU step; 1 / 2: one,
// a PertP / 2D rank's own direction) so the hot loop has no direction branches
template <bool PEND, bool BF16, int G, bool FULL = false, int FULL_MASK = 3>
__device__ __forceinline__ void pu_compute_fast(const PuParams& p, int64_t e0, int ngroups, int64_t dbase,
                                                bool SA, bool SB, float sa, float sb, uint64_t seed_cur,
                                                uint64_t seed_prev, float lrg32, int lane, float4 (&th)[G]) {
  if constexpr (FULL) { SA = (FULL_MASK & 1) != 0; SB = (FULL_MASK & 2) != 0; }
  float4* tp = reinterpret_cast<float4*>(p.theta + (e0 - p.theta_key0)) + lane;
  const uint64_t qa = (uint64_t)(e0 >> 2) + (uint64_t)lane;
  const bool full = FULL || ngroups >= 32 * G;
  uint64_t q[G];
#pragma unroll
  for (int g = 0; g < G; ++g) q[g] = qa + (uint64_t)(32 * g);
  if constexpr (PEND) {
    u32x4 r[G];
    philox4x32_10_xn<G>(q, seed_prev, r);
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const f32x4 zp = normals_from_bits(r[g]);
      th[g].x = fmaf(-lrg32, zp.x, th[g].x); th[g].y = fmaf(-lrg32, zp.y, th[g].y);
      th[g].z = fmaf(-lrg32, zp.z, th[g].z); th[g].w = fmaf(-lrg32, zp.w, th[g].w);
      if (full || lane + 32 * g < ngroups) tp[32 * g] = th[g];
    }
  }
  if (SA || SB) {
    u32x4 r[G];
    philox4x32_10_xn<G>(q, seed_cur, r);
#pragma unroll
    for (int g = 0; g < G; ++g) {
      if (!full && lane + 32 * g >= ngroups) continue;
      const f32x4 z = normals_from_bits(r[g]);
      const float4 t = th[g];
#pragma unroll
      for (int d = 0; d < 2; ++d) {
        if constexpr (FULL) {
          if (!((FULL_MASK >> d) & 1)) continue;              // compile-time
        } else if ((d == 0 && !SA) || (d == 1 && !SB)) {
          continue;                                           // warp-uniform
        }
        const float sc = d == 0 ? sa : sb;
        const float a = fmaf(sc, z.x, t.x), b = fmaf(sc, z.y, t.y);
        const float c = fmaf(sc, z.z, t.z), e = fmaf(sc, z.w, t.w);
        if constexpr (BF16) {
          __nv_bfloat162 lo2 = __floats2bfloat162_rn(a, b), hi2 = __floats2bfloat162_rn(c, e);
          uint2 pk;
          pk.x = *reinterpret_cast<uint32_t*>(&lo2);
          pk.y = *reinterpret_cast<uint32_t*>(&hi2);
          (reinterpret_cast<uint2*>(p.wsh[d] + dbase) + lane)[32 * g] = pk;
        } else {
          (reinterpret_cast<float4*>(p.vsh[d] + dbase) + lane)[32 * g] = make_float4(a, b, c, e);
        }
      }
    }
  }
}

__device__ __forceinline__ void pu_tile_fast(const PuParams& p, int64_t e0, int ngroups, int64_t dbase,
                                             bool pending, bool want_sh, const bool (&sh)[2],
                                             const float (&sc32)[2], uint64_t seed_cur, uint64_t seed_prev,
                                             float lrg32, int kind, int lane, float4 (&th)[kPuGroupsPerThread]) {
  constexpr int G = kPuGroupsPerThread;
  const bool sa = want_sh && sh[0], sb = want_sh && sh[1];
#define ZO_PU_FULL(M)                                                                                              \
  {                                                                                                                \
    if (kind == ZO_SHADOW_BF16) {                                                                                  \
      if (pending) pu_compute_fast<true, true, G, true, M>(p, e0, ngroups, dbase, sa, sb, sc32[0], sc32[1], seed_cur, seed_prev, lrg32, lane, th); \
      else pu_compute_fast<false, true, G, true, M>(p, e0, ngroups, dbase, sa, sb, sc32[0], sc32[1], seed_cur, seed_prev, lrg32, lane, th); \
    } else {                                                                                                       \
      if (pending) pu_compute_fast<true, false, G, true, M>(p, e0, ngroups, dbase, sa, sb, sc32[0], sc32[1], seed_cur, seed_prev, lrg32, lane, th); \
      else pu_compute_fast<false, false, G, true, M>(p, e0, ngroups, dbase, sa, sb, sc32[0], sc32[1], seed_cur, seed_prev, lrg32, lane, th); \
    }                                                                                                              \
    return;                                                                                                        \
  }
  if (ngroups == 32 * G) {
    if (sa && sb) ZO_PU_FULL(3)
    if (sa) ZO_PU_FULL(1)
    if (sb) ZO_PU_FULL(2)
  }
#undef ZO_PU_FULL
  if (kind == ZO_SHADOW_BF16) {
    if (pending) pu_compute_fast<true, true, G>(p, e0, ngroups, dbase, sa, sb, sc32[0], sc32[1], seed_cur, seed_prev, lrg32, lane, th);
    else pu_compute_fast<false, true, G>(p, e0, ngroups, dbase, sa, sb, sc32[0], sc32[1], seed_cur, seed_prev, lrg32, lane, th);
  } else {
    if (pending) pu_compute_fast<true, false, G>(p, e0, ngroups, dbase, sa, sb, sc32[0], sc32[1], seed_cur, seed_prev, lrg32, lane, th);
    else pu_compute_fast<false, false, G>(p, e0, ngroups, dbase, sa, sb, sc32[0], sc32[1], seed_cur, seed_prev, lrg32, lane, th);
  }
}

// Generic tile (unaligned groups, oracle z, shadow-less segments): one group
// per lane at a time, element-guarded; rare, so kept register-light.
template <int ZMODE>
__device__ __forceinline__ void pu_tile_generic(const PuParams& p, const ZoSegment& s, int64_t e0, int64_t e1,
                                             int64_t drow, bool theta_vec, bool pending, bool need_z,
                                             const bool (&sh)[2], const float (&sc32)[2], uint64_t seed_cur,
                                             uint64_t seed_prev, double lrg64, float lrg32, int lane) {
  const bool want_sh = s.kind != ZO_SHADOW_NONE;
  const int64_t qa = e0 >> 2, qb = (e1 + 3) >> 2;
  for (int64_t q = qa + lane; q < qb; q += 32) {
    const int64_t eg = q << 2;
    const bool full = eg >= e0 && eg + 4 <= e1;
    float th[4];
    if (full && theta_vec) {
      const float4 v4 = *reinterpret_cast<const float4*>(p.theta + (eg - p.theta_key0));
      th[0] = v4.x; th[1] = v4.y; th[2] = v4.z; th[3] = v4.w;
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i) th[i] = (eg + i >= e0 && eg + i < e1) ? p.theta[eg + i - p.theta_key0] : 0.f;
    }
    pu_group<ZMODE>(p, s, q, e0, e1, drow, th, full, theta_vec, pending, need_z, want_sh, sh, sc32, seed_cur,
                    seed_prev, lrg64, lrg32);
  }
}

// Walks the tiles of a contiguous chunk in order: one prefix search per
// chunk, then row / column-tile counters advance without division.
struct PuCursor {
  int si;
  int64_t t, seg_end;          // current tile, first tile of the next segment
  ZoSegment s;
  uint32_t tpr, row, ct;       // tiles per row, row, column tile

  __device__ __forceinline__ void load_seg(const PuParams& p, const int64_t* pref, int64_t local) {
    s = p.segs[si];
    seg_end = pref[si + 1];
    tpr = (uint32_t)((s.cols + kPuTile - 1) / kPuTile);
    if (s.rows == 1) { row = 0; ct = (uint32_t)local; }
    else { row = (uint32_t)local / tpr; ct = (uint32_t)local - row * tpr; }
  }
  __device__ __forceinline__ void seek(const PuParams& p, const int64_t* pref, int64_t t0) {
    int lo = 0, hi = p.n_segs - 1;     // last segment with pref[lo] <= t0 (skips empty segments)
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (pref[mid] <= t0) lo = mid; else hi = mid - 1;
    }
    si = lo;
    t = t0;
    load_seg(p, pref, t0 - pref[lo]);
  }
  __device__ __forceinline__ void next(const PuParams& p, const int64_t* pref) {
    ++t;
    if (t >= seg_end) {
      do { ++si; } while (pref[si + 1] <= t);
      load_seg(p, pref, 0);
    } else if (++ct == tpr && s.rows > 1) {
      ct = 0;
      ++row;
    }
  }
  // tile extent in theta keys and the destination offset (dst - src) of its row
  __device__ __forceinline__ void geo(int64_t& e0, int64_t& e1, int64_t& drow) const {
    const int64_t c0 = (int64_t)ct * kPuTile;
    const int64_t c1 = min(c0 + kPuTile, s.cols);
    const int64_t rk = s.src + (int64_t)row * s.cols;
    e0 = rk + c0;
    e1 = rk + c1;
    drow = s.dst + (int64_t)row * s.dst_ld - rk;
  }
};

// Warp-independent streaming over chunks of kPuChunk consecutive tiles (512
// elements each = 32 lanes x 4 groups of 4).  Warps never synchronise with
// each other; within a chunk the next fast tile's theta is loaded before the
// current tile's Philox/Box-Muller math, so the loads overlap the compute.
constexpr int kPuChunk = 8;

template <int ZMODE>
__device__ __forceinline__ void perturb_update_body(const PuParams& p) {
  extern __shared__ int64_t s_prefix[];
  pdl_trigger();
  pdl_wait();
  const bool prefix_in_smem = p.n_segs + 1 <= kPuMaxSmemSegs;
  if (prefix_in_smem)
    for (int i = threadIdx.x; i <= p.n_segs; i += kPuThreads) s_prefix[i] = p.prefix[i];
  __syncthreads();
  const int64_t* pref = prefix_in_smem ? s_prefix : p.prefix;
  const bool pending = (p.flags & ZO_PU_UPDATE) && p.scal->pending != 0;
  const uint64_t seed_cur = p.scal->seed_cur;
  const uint64_t seed_prev = p.scal->seed_prev;
  const double lrg64 = p.scal->lr_g_prev;
  const float lrg32 = (float)lrg64;
  const bool sh[2] = {(p.flags & ZO_PU_SHADOW_A) != 0, (p.flags & ZO_PU_SHADOW_B) != 0};
  const float sc32[2] = {(float)p.scale[0], (float)p.scale[1]};
  const bool need_z = (sh[0] && p.scale[0] != 0.0) || (sh[1] && p.scale[1] != 0.0);
  const bool theta_vec = ((p.theta_key0 & 3) == 0) && ((reinterpret_cast<uintptr_t>(p.theta) & 15) == 0);
  const bool fast_ok = ZMODE == ZO_Z_PHILOX && theta_vec;
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = (blockIdx.x * (int64_t)kPuThreads + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * kPuThreads) >> 5;
  const int64_t n_chunks = (p.n_tiles + kPuChunk - 1) / kPuChunk;

  for (int64_t c = warp0; c < n_chunks; c += n_warps) {
    const int64_t t_end = min((c + 1) * kPuChunk, p.n_tiles);
    PuCursor cur;
    cur.seek(p, pref, c * kPuChunk);
    int64_t e0, e1, drow;
    cur.geo(e0, e1, drow);
    auto is_fast = [&](const ZoSegment& s, int64_t a0, int64_t a1, int64_t dr) {
      const bool any_sh = s.kind != ZO_SHADOW_NONE && (sh[0] || sh[1]);
      return fast_ok && ((a0 | a1 | (a0 + dr)) & 3) == 0 && (need_z || !any_sh);
    };
    bool fast = is_fast(cur.s, e0, e1, drow);
    float4 th[kPuGroupsPerThread];
    if (fast) pu_load_fast<kPuGroupsPerThread>(p, e0, (int)((e1 - e0) >> 2), lane, th);
    while (true) {
      const ZoSegment s = cur.s;
      const int64_t ce0 = e0, ce1 = e1, cdrow = drow;
      const bool cfast = fast;
      float4 thc[kPuGroupsPerThread];
#pragma unroll
      for (int g = 0; g < kPuGroupsPerThread; ++g) thc[g] = th[g];
      const bool more = cur.t + 1 < t_end;
      if (more) {                                   // prefetch the next tile's theta
        cur.next(p, pref);
        cur.geo(e0, e1, drow);
        fast = is_fast(cur.s, e0, e1, drow);
        if (fast) pu_load_fast<kPuGroupsPerThread>(p, e0, (int)((e1 - e0) >> 2), lane, th);
      }
      if (cfast) {
        pu_tile_fast(p, ce0, (int)((ce1 - ce0) >> 2), ce0 + cdrow, pending, s.kind != ZO_SHADOW_NONE, sh, sc32,
                     seed_cur, seed_prev, lrg32, s.kind, lane, thc);
      } else {
        pu_tile_generic<ZMODE>(p, s, ce0, ce1, cdrow, theta_vec, pending, need_z, sh, sc32, seed_cur, seed_prev,
                               lrg64, lrg32, lane);
      }
      if (!more) break;
    }
  }
}

// 126 registers x 4 CTAs of 4 warps per SM; a grid of 4 resident waves of
// chunks (measured best of 1 / 2 / 4: late-starting CTAs even out the tail)
template <int ZMODE>
__global__ void __launch_bounds__(kPuThreads, 4) perturb_update_kernel(const PuParams p) {
  perturb_update_body<ZMODE>(p);
}

int64_t perturb_tile_elems() { return kPuTile; }   // the host builds its tile prefixes with this

int perturb_update_launch(const PuParams& p, int zmode, cudaStream_t stream) {
  if (p.n_tiles <= 0) return ZO_OK;
  const int64_t n_chunks = (p.n_tiles + kPuChunk - 1) / kPuChunk;
  // ZO_PU_FILL: one chunk per warp, CTAs live a few microseconds; otherwise a
  // persistent grid of four resident waves
  const int64_t want = (p.flags & ZO_PU_FILL) ? (n_chunks + 3) / 4 : (int64_t)num_sms() * 4 * 4;
  const int grid = (int)(p.n_tiles < want ? p.n_tiles : want);
  const size_t smem = p.n_segs + 1 <= kPuMaxSmemSegs ? (size_t)(p.n_segs + 1) * sizeof(int64_t) : 0;
  if (zmode == ZO_Z_PHILOX)
    launch_k(perturb_update_kernel<ZO_Z_PHILOX>, dim3(grid), dim3(kPuThreads), smem, stream, p);
  else
    launch_k(perturb_update_kernel<ZO_Z_ORACLE>, dim3(grid), dim3(kPuThreads), smem, stream, p);
  return launch_status("perturb_update_kernel");
}

// ---------------------------------------------------------------------------
// debug: the Philox direction itself
// ---------------------------------------------------------------------------
__global__ void philox_normals_kernel(uint64_t seed, int64_t e0, int64_t n, float* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = philox_normal1(seed, (uint64_t)(e0 + i));
}

int philox_normals_launch(uint64_t seed, int64_t e0, int64_t n, float* out, cudaStream_t stream) {
  if (n <= 0) return ZO_OK;
  const int grid = (int)((n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096);
  philox_normals_kernel<<<grid, 256, 0, stream>>>(seed, e0, n, out);
  return launch_status("philox_normals_kernel");
}

}  // namespace zo
