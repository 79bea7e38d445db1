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

constexpr int kPuThreads = 256;
constexpr int kPuGroupsPerThread = 4;
constexpr int64_t kPuTile = (int64_t)kPuThreads * kPuGroupsPerThread * 4;  // elements per tile

__device__ __forceinline__ void store_shadow(const ZoSegment& s, __nv_bfloat16* w, float* v,
                                             int64_t di, float val) {
  if (s.kind == ZO_SHADOW_BF16) w[di] = __float2bfloat16_rn(val);
  else v[di] = val;
}

template <int ZMODE>
__global__ void __launch_bounds__(kPuThreads) perturb_update_kernel(const PuParams p) {
  __shared__ int s_seg;
  const bool pending = (p.flags & ZO_PU_UPDATE) && p.scal->pending != 0;
  const uint64_t seed_cur = p.scal->seed_cur;
  const uint64_t seed_prev = p.scal->seed_prev;
  const double lrg64 = p.scal->lr_g_prev;
  const float lrg32 = (float)lrg64;
  const bool sh[2] = {(p.flags & ZO_PU_SHADOW_A) != 0, (p.flags & ZO_PU_SHADOW_B) != 0};
  const float sc32[2] = {(float)p.scale[0], (float)p.scale[1]};
  const bool need_z = (sh[0] && p.scale[0] != 0.0) || (sh[1] && p.scale[1] != 0.0);
  const bool theta_vec = ((p.theta_key0 & 3) == 0) && ((reinterpret_cast<uintptr_t>(p.theta) & 15) == 0);

  for (int64_t t = blockIdx.x; t < p.n_tiles; t += gridDim.x) {
    if (threadIdx.x == 0) {  // segment owning tile t: largest i with prefix[i] <= t
      int lo = 0, hi = p.n_segs - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (p.prefix[mid] <= t) lo = mid; else hi = mid - 1;
      }
      s_seg = lo;
    }
    __syncthreads();
    const int si = s_seg;
    __syncthreads();
    const ZoSegment s = p.segs[si];
    const int64_t tpr = (s.cols + kPuTile - 1) / kPuTile;
    const int64_t local = t - p.prefix[si];
    const int64_t row = local / tpr;
    const int64_t c0 = (local % tpr) * kPuTile;
    const int64_t c1 = min(c0 + kPuTile, s.cols);
    const int64_t rk = s.src + row * s.cols;         // key of (row, col 0)
    const int64_t e0 = rk + c0, e1 = rk + c1;
    const int64_t drow = s.dst + row * s.dst_ld - rk;  // shadow index = key + drow
    const bool want_sh = s.kind != ZO_SHADOW_NONE;

    for (int64_t q = (e0 >> 2) + threadIdx.x; q < ((e1 + 3) >> 2); q += kPuThreads) {
      const int64_t eg = q << 2;
      float th[4];
      const bool full = eg >= e0 && eg + 4 <= e1;
      if (full && theta_vec) {
        const float4 v4 = *reinterpret_cast<const float4*>(p.theta + (eg - p.theta_key0));
        th[0] = v4.x; th[1] = v4.y; th[2] = v4.z; th[3] = v4.w;
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i)
          th[i] = (eg + i >= e0 && eg + i < e1) ? p.theta[eg + i - p.theta_key0] : 0.f;
      }

      if (pending) {
        if constexpr (ZMODE == ZO_Z_PHILOX) {
          const f32x4 zp = philox_normal4(seed_prev, (uint64_t)q);
#pragma unroll
          for (int i = 0; i < 4; ++i) th[i] = fmaf(-lrg32, f4get(zp, i), th[i]);
        } else {
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int64_t e = eg + i;
            if (e >= e0 && e < e1) {
              const double z = p.z_prev[e - p.z_key0];
              th[i] = __double2float_rn(__dsub_rn((double)th[i], __dmul_rn(lrg64, z)));
            }
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

      if (!want_sh) continue;
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
  }
}

int perturb_update_launch(const PuParams& p, int zmode, cudaStream_t stream) {
  if (p.n_tiles <= 0) return ZO_OK;
  const int64_t want = (int64_t)num_sms() * 8;   // 8 x 256 threads resident per SM
  const int grid = (int)(p.n_tiles < want ? p.n_tiles : want);
  if (zmode == ZO_Z_PHILOX) perturb_update_kernel<ZO_Z_PHILOX><<<grid, kPuThreads, 0, stream>>>(p);
  else perturb_update_kernel<ZO_Z_ORACLE><<<grid, kPuThreads, 0, stream>>>(p);
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
