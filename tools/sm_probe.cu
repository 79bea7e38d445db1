// Per-SM rates that bound the hd-64 attention softmax (attention_tc.cu):
//  (1) MUFU.EX2 with the softmax's instruction mix (FFMA2 scale, 2 x EX2,
//      FADD2 row sum, bf16 pack) for 1..4 warps per SM sub-partition;
//  (2) tcgen05.ld 32x32b.x32 read bandwidth for 1..4 warps per sub-partition.
// One CTA per SM, clock64 around the timed loop, exps (bytes) per SM clock.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2507_03211_b200/csrc -o /tmp/probe tools/sm_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint64_t pk2(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void up2(uint64_t v, float& lo, float& hi) { asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v)); }
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// each warp: ITER x 128 exps per lane, the softmax's mix
__global__ void __launch_bounds__(512, 1) ex2_probe(int iters, float seed, uint32_t* sink, unsigned long long* cyc) {
  float s[64];
#pragma unroll
  for (int i = 0; i < 64; ++i) s[i] = seed * (threadIdx.x + i) * 1e-3f;
  const uint64_t sc = pk2(0.18f, 0.18f), nm = pk2(-1.f, -1.f);
  uint64_t sum2[2] = {0ull, 0ull};
  uint32_t acc = 0;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 2; ++c) {
#pragma unroll
      for (int i = 0; i < 32; i += 2) {
        const uint64_t x2 = ffma2(pk2(s[c * 32 + i], s[c * 32 + i + 1]), sc, nm);
        float x0, x1;
        up2(x2, x0, x1);
        const float p0 = ex2(x0), p1 = ex2(x1);
        s[c * 32 + i] = p0;
        s[c * 32 + i + 1] = p1;
        sum2[(i >> 1) & 1] = fadd2(sum2[(i >> 1) & 1], pk2(p0, p1));
        uint32_t h;
        asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(p1), "f"(p0));
        acc ^= h;
      }
    }
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  float a, b, c, d;
  up2(sum2[0], a, b);
  up2(sum2[1], c, d);
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc ^ __float_as_uint(a + b + c + d);
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// tcgen05.ld throughput: warp w reads its lane quarter (w % 4), 4 x32 loads then wait
__global__ void tmem_probe(int iters, uint32_t* sink, unsigned long long* cyc) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&slot)),
                 "r"(512u));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tm = slot + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) & 3) * 128;
  uint32_t acc = 0;
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t r[4][32];
#pragma unroll
    for (int c = 0; c < 4; ++c)
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
          "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
          : "=r"(r[c][0]), "=r"(r[c][1]), "=r"(r[c][2]), "=r"(r[c][3]), "=r"(r[c][4]), "=r"(r[c][5]), "=r"(r[c][6]),
            "=r"(r[c][7]), "=r"(r[c][8]), "=r"(r[c][9]), "=r"(r[c][10]), "=r"(r[c][11]), "=r"(r[c][12]),
            "=r"(r[c][13]), "=r"(r[c][14]), "=r"(r[c][15]), "=r"(r[c][16]), "=r"(r[c][17]), "=r"(r[c][18]),
            "=r"(r[c][19]), "=r"(r[c][20]), "=r"(r[c][21]), "=r"(r[c][22]), "=r"(r[c][23]), "=r"(r[c][24]),
            "=r"(r[c][25]), "=r"(r[c][26]), "=r"(r[c][27]), "=r"(r[c][28]), "=r"(r[c][29]), "=r"(r[c][30]),
            "=r"(r[c][31])
          : "r"(tm + c * 32));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int i = 0; i < 32; ++i) acc += r[c][i];
  }
  const unsigned long long t1 = clock64();
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(slot), "r"(512u));
}

int main() {
  uint32_t* sink;
  unsigned long long* cyc;
  cudaMalloc(&sink, 1 << 22);
  cudaMalloc(&cyc, 4096 * 8);
  unsigned long long h[148];
  for (int wps = 1; wps <= 4; ++wps) {
    const int threads = 128 * wps, iters = 256;
    ex2_probe<<<148, threads>>>(iters, 1.f, sink, cyc);
    if (cudaDeviceSynchronize() != cudaSuccess) { printf("ex2 probe failed\n"); return 1; }
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    const double exps = (double)threads * iters * 64;
    printf("ex2 mix : %d warp(s)/SMSP  %.2f exps/clk/SM  (%.0f clk)\n", wps, exps / h[0], (double)h[0]);
  }
  for (int wps = 1; wps <= 4; ++wps) {
    const int threads = 128 * wps, iters = 256;
    tmem_probe<<<148, threads>>>(iters, sink, cyc);
    tmem_probe<<<148, threads>>>(iters, sink, cyc);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("tmem probe: %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    const double bytes = (double)threads * iters * 128 * 4;
    printf("tcgen05.ld 32x32b.x32: %d warp(s)/SMSP  %.1f B/clk/SM  (%.0f clk)\n", wps, bytes / h[0], (double)h[0]);
  }
  return 0;
}
