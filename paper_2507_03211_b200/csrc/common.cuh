// Shared device/host helpers for the sm_100a ZO-step kernels.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <stdio.h>

#include <utility>

#include "../../include/zo_b200.h"

namespace zo {

// ---------------------------------------------------------------------------
// status / last error (thread-local, read through zo_last_error())
// ---------------------------------------------------------------------------
void set_error(const char* fmt, ...);

#define ZO_CHECK_ARG(cond, code, ...)     \
  do {                                    \
    if (!(cond)) {                        \
      ::zo::set_error(__VA_ARGS__);       \
      return (code);                      \
    }                                     \
  } while (0)

#define ZO_CUDA_TRY(expr)                                                        \
  do {                                                                           \
    cudaError_t _e = (expr);                                                     \
    if (_e != cudaSuccess) {                                                     \
      ::zo::set_error("%s failed: %s", #expr, cudaGetErrorString(_e));           \
      return ZO_ERR_CUDA;                                                        \
    }                                                                            \
  } while (0)

inline int launch_status(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s launch failed: %s", what, cudaGetErrorString(e));
    return ZO_ERR_CUDA;
  }
  return ZO_OK;
}

int num_sms();

// ---------------------------------------------------------------------------
// Philox4x32-10 (Salmon et al., SC'11): counter-based, so z for global
// element e is a pure function of (seed, e) -- identical on every rank and
// for every slicing of a block.  counter = (e/4 lo, e/4 hi, 0, 0),
// key = (seed lo, seed hi); the 4 outputs become z[4q .. 4q+3].
// ---------------------------------------------------------------------------
struct u32x4 { uint32_t x, y, z, w; };

__host__ __device__ __forceinline__ uint32_t mulhi32(uint32_t a, uint32_t b) {
#ifdef __CUDA_ARCH__
  return __umulhi(a, b);
#else
  return (uint32_t)(((uint64_t)a * (uint64_t)b) >> 32);
#endif
}

// Philox4x32 round count: 10 (Random123's recommended default; the value
// every test and measurement uses).  Overridable at build time only for
// experiments (-DZO_PHILOX_ROUNDS=7, the smallest count that passes BigCrush).
#ifndef ZO_PHILOX_ROUNDS
#define ZO_PHILOX_ROUNDS 10
#endif
__host__ __device__ __forceinline__ u32x4 philox4x32_10(uint64_t ctr, uint64_t seed) {
  uint32_t c0 = (uint32_t)ctr, c1 = (uint32_t)(ctr >> 32), c2 = 0u, c3 = 0u;
  uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
#pragma unroll
  for (int r = 0; r < ZO_PHILOX_ROUNDS; ++r) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * c0;   // one IMAD.WIDE.U32: hi and lo
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0, n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
    c0 = n0; c1 = (uint32_t)p1; c2 = n2; c3 = (uint32_t)p0;
    k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
  }
  return {c0, c1, c2, c3};
}

// Box-Muller on 24-bit uniforms: u1 in (0,1) (never 0), angle in [-pi, pi).
// Fast MUFU intrinsics; outputs are a deterministic function of the bits.
__device__ __forceinline__ void box_muller(uint32_t a, uint32_t b, float& z0, float& z1) {
  // uniforms from the mantissa bits (no int->float conversion):
  //   u1 = 2 - [1,2)  in (0, 1];   ang = pi * [2,4) - 3 pi  in [-pi, pi)
  const float u1 = 2.0f - __uint_as_float(0x3F800000u | (a >> 9));
  const float ang = fmaf(__uint_as_float(0x40000000u | (b >> 9)), 3.14159265358979f, -9.42477796076938f);
  // single MUFU ops, flush-to-zero (u1 >= 2^-23 and |ang| <= pi: no denormals)
  float lg, r, s, c;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(lg) : "f"(u1));
  const float t = -1.3862943611198906f * lg;                                      // -2 ln u >= 0
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(t));                          // one MUFU, sqrt(0) = 0
  asm("sin.approx.ftz.f32 %0, %1;" : "=f"(s) : "f"(ang));
  asm("cos.approx.ftz.f32 %0, %1;" : "=f"(c) : "f"(ang));
  z0 = r * c;
  z1 = r * s;
}


// ---------------------------------------------------------------------------
// Keyed Philox for the streaming kernels: the 10 round keys of a seed are
// computed once per thread (PhiloxKeys) and each round is 2 IMAD.WIDE.U32 +
// 2 LOP3.  Produces exactly the words of philox4x32_10 (same z everywhere).
// ---------------------------------------------------------------------------
struct PhiloxKeys { uint32_t k0[ZO_PHILOX_ROUNDS], k1[ZO_PHILOX_ROUNDS]; };

__host__ __device__ __forceinline__ PhiloxKeys philox_keys(uint64_t seed) {
  PhiloxKeys k;
  uint32_t a = (uint32_t)seed, b = (uint32_t)(seed >> 32);
#pragma unroll
  for (int r = 0; r < ZO_PHILOX_ROUNDS; ++r) { k.k0[r] = a; k.k1[r] = b; a += 0x9E3779B9u; b += 0xBB67AE85u; }
  return k;
}

__device__ __forceinline__ u32x4 philox4x32_10_k(uint64_t ctr, const PhiloxKeys& k) {
  uint32_t c0 = (uint32_t)ctr, c1 = (uint32_t)(ctr >> 32), c2 = 0u, c3 = 0u;
#pragma unroll
  for (int r = 0; r < ZO_PHILOX_ROUNDS; ++r) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k.k0[r];
    const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k.k1[r];
    c1 = (uint32_t)p1; c3 = (uint32_t)p0; c0 = n0; c2 = n2;
  }
  return {c0, c1, c2, c3};
}

struct f32x4 { float x, y, z, w; };

__device__ __forceinline__ f32x4 philox_normal4(uint64_t seed, uint64_t q) {
  const u32x4 r = philox4x32_10(q, seed);
  f32x4 o;
  box_muller(r.x, r.y, o.x, o.y);
  box_muller(r.z, r.w, o.z, o.w);
  return o;
}

__device__ __forceinline__ float philox_normal1(uint64_t seed, uint64_t e) {
  const f32x4 v = philox_normal4(seed, e >> 2);
  switch (e & 3) { case 0: return v.x; case 1: return v.y; case 2: return v.z; default: return v.w; }
}

// Four Philox4x32-10 streams in lockstep: each round key is formed once and
// shared by the four counters (and the four dependency chains interleave).
template <int N>
__device__ __forceinline__ void philox4x32_10_xn(const uint64_t (&ctr)[N], uint64_t seed, u32x4 (&out)[N]) {
  uint32_t c0[N], c1[N], c2[N], c3[N];
#pragma unroll
  for (int i = 0; i < N; ++i) { c0[i] = (uint32_t)ctr[i]; c1[i] = (uint32_t)(ctr[i] >> 32); c2[i] = 0u; c3[i] = 0u; }
  uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
#pragma unroll
  for (int r = 0; r < ZO_PHILOX_ROUNDS; ++r) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const uint64_t p0 = (uint64_t)0xD2511F53u * c0[i];
      const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2[i];
      const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1[i] ^ k0, n2 = (uint32_t)(p0 >> 32) ^ c3[i] ^ k1;
      c0[i] = n0; c1[i] = (uint32_t)p1; c2[i] = n2; c3[i] = (uint32_t)p0;
    }
    k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
  }
#pragma unroll
  for (int i = 0; i < N; ++i) out[i] = {c0[i], c1[i], c2[i], c3[i]};
}

__device__ __forceinline__ f32x4 normals_from_bits(const u32x4& r) {
  f32x4 o;
  box_muller(r.x, r.y, o.x, o.y);
  box_muller(r.z, r.w, o.z, o.w);
  return o;
}

__device__ __forceinline__ f32x4 philox_normal4_k(const PhiloxKeys& k, uint64_t q) {
  const u32x4 r = philox4x32_10_k(q, k);
  f32x4 o;
  box_muller(r.x, r.y, o.x, o.y);
  box_muller(r.z, r.w, o.z, o.w);
  return o;
}

__device__ __forceinline__ float f4get(const f32x4& v, int i) {
  return i == 0 ? v.x : (i == 1 ? v.y : (i == 2 ? v.z : v.w));
}

// Direction source shared by every kernel that perturbs on the fly.
// mode ZO_Z_PHILOX: z = philox(seed, e).  mode ZO_Z_ORACLE: z = zsrc[e - zbase]
// (the reference's f64 z, injected), with exact f64 arithmetic.
struct ZSource {
  int mode;
  uint64_t seed;
  const double* zsrc;
  int64_t zbase;
};

// Parameter block of the perturb/update kernel (perturb.cu; filled by api.cu).
struct PuParams {
  float* theta;
  int64_t theta_key0;
  const ZoSegment* segs;
  const int64_t* prefix;
  int32_t n_segs;
  int64_t n_tiles;
  __nv_bfloat16* wsh[2];
  float* vsh[2];
  double scale[2];
  uint32_t flags;
  const ZoStepScalars* scal;
  const double* z_cur;
  const double* z_prev;
  int64_t z_key0;
};

// ---------------------------------------------------------------------------
// Programmatic dependent launch: every kernel lets its stream successor start
// launching immediately (the successor's CTAs still only run where resources
// free up), and waits for its predecessor's memory to be visible before
// reading any input.  Both are no-ops for kernels launched without PDL.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

bool pdl_enabled();

// cudaLaunchKernelEx with programmatic stream serialisation (PDL)
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                            Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  // the stream's priority as a launch attribute: kept by graph capture, and
  // honoured on replay of graphs instantiated by zo_graph_end
  int prio = 0;
  cudaStreamGetPriority(st, &prio);
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributePriority;
  attr[0].val.priority = prio;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// ---------------------------------------------------------------------------
// small PTX wrappers (mbarrier / TMA / tcgen05) for the GEMM
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

}  // namespace zo
