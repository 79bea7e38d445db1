// LayerNorm launch-shape study at the stacked step's shape (rows x d fp32 ->
// bf16): the shipped warp-per-row kernel vs a software-pipelined persistent
// warp loop vs a CTA-per-row kernel, and a plain copy of the same bytes as the
// floor.  x is either flushed from L2 (a 256 MB write between launches) or
// L2-warm.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ln tools/ln_bench.cu
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ uint2 pack4(float a, float b, float c, float d) {
  __nv_bfloat162 lo = __floats2bfloat162_rn(a, b), hi = __floats2bfloat162_rn(c, d);
  uint2 r;
  r.x = *reinterpret_cast<uint32_t*>(&lo);
  r.y = *reinterpret_cast<uint32_t*>(&hi);
  return r;
}

// A: the shipped kernel (warp per row, whole row in registers, grid <= 8 CTAs/SM)
template <int NV>
__global__ void __launch_bounds__(256) ln_warp(const float* __restrict__ x, const float* __restrict__ g,
                                               const float* __restrict__ b, int rows, int d,
                                               __nv_bfloat16* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const long warp_g = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  const long nwarps = ((long)gridDim.x * blockDim.x) >> 5;
  for (long r = warp_g; r < rows; r += nwarps) {
    const float4* xr = reinterpret_cast<const float4*>(x + r * d);
    float4 v[NV];
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < NV; ++i) { v[i] = xr[i * 32 + lane]; s += (v[i].x + v[i].y) + (v[i].z + v[i].w); }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const float mu = s / d;
    float q = 0.f;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const float a0 = v[i].x - mu, a1 = v[i].y - mu, a2 = v[i].z - mu, a3 = v[i].w - mu;
      q += (a0 * a0 + a1 * a1) + (a2 * a2 + a3 * a3);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
    const float rs = 1.0f / sqrtf(q / d + 1e-5f);
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c = (i * 32 + lane) * 4;
      const float4 gg = *reinterpret_cast<const float4*>(g + c), bb = *reinterpret_cast<const float4*>(b + c);
      *reinterpret_cast<uint2*>(out + r * d + c) =
          pack4(fmaf((v[i].x - mu) * rs, gg.x, bb.x), fmaf((v[i].y - mu) * rs, gg.y, bb.y),
                fmaf((v[i].z - mu) * rs, gg.z, bb.z), fmaf((v[i].w - mu) * rs, gg.w, bb.w));
    }
  }
}

// B: persistent warps, next row prefetched into registers while the current
// one is reduced and stored
template <int NV>
__global__ void __launch_bounds__(128, 3) ln_pipe(const float* __restrict__ x, const float* __restrict__ g,
                                                  const float* __restrict__ b, int rows, int d,
                                                  __nv_bfloat16* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const long warp_g = (blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5;
  const long nwarps = ((long)gridDim.x * blockDim.x) >> 5;
  float4 v[NV], w[NV];
  long r = warp_g;
  if (r < rows) {
    const float4* xr = reinterpret_cast<const float4*>(x + r * d);
#pragma unroll
    for (int i = 0; i < NV; ++i) v[i] = xr[i * 32 + lane];
  }
  for (; r < rows; r += nwarps) {
    const long rn = r + nwarps;
    if (rn < rows) {
      const float4* xn = reinterpret_cast<const float4*>(x + rn * d);
#pragma unroll
      for (int i = 0; i < NV; ++i) w[i] = xn[i * 32 + lane];
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < NV; ++i) s += (v[i].x + v[i].y) + (v[i].z + v[i].w);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const float mu = s / d;
    float q = 0.f;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const float a0 = v[i].x - mu, a1 = v[i].y - mu, a2 = v[i].z - mu, a3 = v[i].w - mu;
      q += (a0 * a0 + a1 * a1) + (a2 * a2 + a3 * a3);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
    const float rs = 1.0f / sqrtf(q / d + 1e-5f);
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c = (i * 32 + lane) * 4;
      const float4 gg = *reinterpret_cast<const float4*>(g + c), bb = *reinterpret_cast<const float4*>(b + c);
      *reinterpret_cast<uint2*>(out + r * d + c) =
          pack4(fmaf((v[i].x - mu) * rs, gg.x, bb.x), fmaf((v[i].y - mu) * rs, gg.y, bb.y),
                fmaf((v[i].z - mu) * rs, gg.z, bb.z), fmaf((v[i].w - mu) * rs, gg.w, bb.w));
    }
#pragma unroll
    for (int i = 0; i < NV; ++i) v[i] = w[i];
  }
}

// C: one CTA of 256 threads per row (2 float4 per thread), block reduction
__device__ __forceinline__ float block_sum256(float s, float* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = s;
  __syncthreads();
  float t = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) t += red[i];
  return t;
}
template <int PT>
__global__ void __launch_bounds__(256) ln_cta(const float* __restrict__ x, const float* __restrict__ g,
                                              const float* __restrict__ b, int rows, int d,
                                              __nv_bfloat16* __restrict__ out) {
  __shared__ float red[8];
  const long r = blockIdx.x;
  const float4* xr = reinterpret_cast<const float4*>(x + r * d);
  float4 v[PT];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < PT; ++i) { v[i] = xr[i * 256 + threadIdx.x]; s += (v[i].x + v[i].y) + (v[i].z + v[i].w); }
  const float mu = block_sum256(s, red) / d;
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < PT; ++i) {
    const float a0 = v[i].x - mu, a1 = v[i].y - mu, a2 = v[i].z - mu, a3 = v[i].w - mu;
    q += (a0 * a0 + a1 * a1) + (a2 * a2 + a3 * a3);
  }
  const float rs = 1.0f / sqrtf(block_sum256(q, red) / d + 1e-5f);
#pragma unroll
  for (int i = 0; i < PT; ++i) {
    const int c = (i * 256 + threadIdx.x) * 4;
    const float4 gg = *reinterpret_cast<const float4*>(g + c), bb = *reinterpret_cast<const float4*>(b + c);
    *reinterpret_cast<uint2*>(out + r * d + c) =
        pack4(fmaf((v[i].x - mu) * rs, gg.x, bb.x), fmaf((v[i].y - mu) * rs, gg.y, bb.y),
              fmaf((v[i].z - mu) * rs, gg.z, bb.z), fmaf((v[i].w - mu) * rs, gg.w, bb.w));
  }
}

// D: two warps per row (64-thread CTA), 8 float4 per lane, smem exchange
template <int NV>
__global__ void __launch_bounds__(64) ln_2w(const float* __restrict__ x, const float* __restrict__ g,
                                            const float* __restrict__ b, int rows, int d,
                                            __nv_bfloat16* __restrict__ out) {
  __shared__ float red[2];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const long r = blockIdx.x;
  const float4* xr = reinterpret_cast<const float4*>(x + r * d) + w * NV * 32;
  float4 v[NV];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) { v[i] = xr[i * 32 + lane]; s += (v[i].x + v[i].y) + (v[i].z + v[i].w); }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) red[w] = s;
  __syncthreads();
  const float mu = (red[0] + red[1]) / d;
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const float a0 = v[i].x - mu, a1 = v[i].y - mu, a2 = v[i].z - mu, a3 = v[i].w - mu;
    q += (a0 * a0 + a1 * a1) + (a2 * a2 + a3 * a3);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
  __syncthreads();
  if (lane == 0) red[w] = q;
  __syncthreads();
  const float rs = 1.0f / sqrtf((red[0] + red[1]) / d + 1e-5f);
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = ((w * NV + i) * 32 + lane) * 4;
    const float4 gg = *reinterpret_cast<const float4*>(g + c), bb = *reinterpret_cast<const float4*>(b + c);
    *reinterpret_cast<uint2*>(out + r * d + c) =
        pack4(fmaf((v[i].x - mu) * rs, gg.x, bb.x), fmaf((v[i].y - mu) * rs, gg.y, bb.y),
              fmaf((v[i].z - mu) * rs, gg.z, bb.z), fmaf((v[i].w - mu) * rs, gg.w, bb.w));
  }
}

// E: copy floor -- read the same fp32 bytes, write the same bf16 bytes
__global__ void copy_floor(const float4* __restrict__ x, uint2* __restrict__ out, long n4) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n4; i += (long)gridDim.x * blockDim.x) {
    const float4 v = x[i];
    out[i] = pack4(v.x, v.y, v.z, v.w);
  }
}

__global__ void flush_k(float4* p, long n4, float v) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n4; i += (long)gridDim.x * blockDim.x)
    p[i] = make_float4(v, v, v, v);
}

int main() {
  const int rows = 4096, d = 2048;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  float *x, *g, *b, *fl;
  __nv_bfloat16 *o, *o2;
  CK(cudaMalloc(&x, (size_t)rows * d * 4));
  CK(cudaMalloc(&g, d * 4));
  CK(cudaMalloc(&b, d * 4));
  CK(cudaMalloc(&o, (size_t)rows * d * 2));
  CK(cudaMalloc(&o2, (size_t)rows * d * 2));
  const long nfl = 256l << 20;
  CK(cudaMalloc(&fl, nfl));
  {
    float* h = (float*)malloc((size_t)rows * d * 4);
    for (long i = 0; i < (long)rows * d; ++i) h[i] = (float)((i * 2654435761u) % 1000) / 250.f - 2.f;
    CK(cudaMemcpy(x, h, (size_t)rows * d * 4, cudaMemcpyHostToDevice));
    for (int i = 0; i < d; ++i) h[i] = 1.f + 0.001f * i;
    CK(cudaMemcpy(g, h, d * 4, cudaMemcpyHostToDevice));
    for (int i = 0; i < d; ++i) h[i] = 0.01f * (i % 7);
    CK(cudaMemcpy(b, h, d * 4, cudaMemcpyHostToDevice));
    free(h);
  }
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  auto run = [&](const char* name, auto launch) {
    for (int flush = 1; flush >= 0; --flush) {
      float best = 1e9, tot = 0;
      const int it = 30;
      for (int i = 0; i < it + 3; ++i) {
        if (flush) flush_k<<<sms * 4, 256>>>((float4*)fl, nfl / 16, (float)i);
        else launch();   // warm x into L2
        CK(cudaEventRecord(e0));
        launch();
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        if (i >= 3) { best = ms < best ? ms : best; tot += ms; }
      }
      const double bytes = (double)rows * d * 6;
      printf("%-34s %s  mean %6.2f us  best %6.2f us  (%.0f GB/s mean)\n", name, flush ? "x cold " : "x in L2",
             tot / it * 1e3, best * 1e3, bytes / (tot / it * 1e-3) / 1e9);
    }
  };
  const int grid_a = rows / 8 < sms * 8 ? rows / 8 : sms * 8;
  run("A warp/row (shipped)", [&] { ln_warp<16><<<grid_a, 256>>>(x, g, b, rows, d, o); });
  run("B pipelined warp loop 3x128/SM", [&] { ln_pipe<16><<<sms * 3, 128>>>(x, g, b, rows, d, o2); });
  run("B' pipelined warp loop 2x128/SM", [&] { ln_pipe<16><<<sms * 2, 128>>>(x, g, b, rows, d, o2); });
  run("C CTA(256)/row", [&] { ln_cta<2><<<rows, 256>>>(x, g, b, rows, d, o2); });
  run("D 2 warps/row", [&] { ln_2w<8><<<rows, 64>>>(x, g, b, rows, d, o2); });
  run("E copy floor (same bytes)", [&] { copy_floor<<<sms * 8, 256>>>((const float4*)x, (uint2*)o2, (long)rows * d / 4); });
  // results of B / C / D equal A bit for bit? (same arithmetic order only for A/B)
  ln_warp<16><<<grid_a, 256>>>(x, g, b, rows, d, o);
  ln_pipe<16><<<sms * 3, 128>>>(x, g, b, rows, d, o2);
  CK(cudaDeviceSynchronize());
  unsigned short *h1 = (unsigned short*)malloc((size_t)rows * d * 2), *h2 = (unsigned short*)malloc((size_t)rows * d * 2);
  CK(cudaMemcpy(h1, o, (size_t)rows * d * 2, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(h2, o2, (size_t)rows * d * 2, cudaMemcpyDeviceToHost));
  long diff = 0;
  for (long i = 0; i < (long)rows * d; ++i) diff += h1[i] != h2[i];
  printf("A vs B differing outputs: %ld\n", diff);
  return 0;
}
