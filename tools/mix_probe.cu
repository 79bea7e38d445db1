// Bandwidth ceiling of the perturb pass's access mix, with no arithmetic:
// per element read 4 B (theta) and write 4 B (theta) + 2 x 2 B (bf16 shadows)
// -- 12 B -- over the 1.42 G parameters of the OPT-1.3B shape, next to a plain
// copy (4 B + 4 B) and the 8 B mixes of the shadow-only / update-only passes.
// Grid-stride float4 loop, 8 CTAs of 256 per SM; CUDA events, best of 10.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mix tools/mix_probe.cu
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint2 pk(float4 v) {
  __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
  return make_uint2(*reinterpret_cast<uint32_t*>(&lo), *reinterpret_cast<uint32_t*>(&hi));
}

template <int MODE>   // 0 copy (R4 W4), 1 perturb mix (R4 W4 W2 W2), 2 shadows only (R4 W2 W2), 3 update only (R4 W4)
__global__ void __launch_bounds__(256) mix(float4* th, uint2* a, uint2* b, float4* dst, long n4, float s) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n4; i += (long)gridDim.x * blockDim.x) {
    float4 v = th[i];
    if (MODE == 0) { dst[i] = v; continue; }
    v.x += s; v.y += s; v.z += s; v.w += s;
    if (MODE == 1 || MODE == 3) th[i] = v;
    if (MODE == 1 || MODE == 2) { a[i] = pk(v); b[i] = pk(make_float4(-v.x, -v.y, -v.z, -v.w)); }
  }
}

int main() {
  const long n = 1415615584l / 4 * 4, n4 = n / 4;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float4 *th, *dst;
  uint2 *a, *b;
  if (cudaMalloc(&th, n * 4) || cudaMalloc(&dst, n * 4) || cudaMalloc(&a, n * 2) || cudaMalloc(&b, n * 2)) {
    printf("alloc failed\n");
    return 1;
  }
  cudaMemset(th, 0, n * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char* names[4] = {"copy          R4 W4   (8 B/elem)", "perturb mix   R4 W4 W2 W2 (12 B)",
                          "shadows only  R4 W2 W2 (8 B)", "update only   R4 W4   (8 B)"};
  const double bytes[4] = {8.0, 12.0, 8.0, 8.0};
  for (int rep = 0; rep < 2; ++rep)
    for (int m = 0; m < 4; ++m) {
      float best = 1e9;
      for (int it = 0; it < 10; ++it) {
        cudaEventRecord(e0);
        switch (m) {
          case 0: mix<0><<<sms * 8, 256>>>(th, a, b, dst, n4, 1e-7f); break;
          case 1: mix<1><<<sms * 8, 256>>>(th, a, b, dst, n4, 1e-7f); break;
          case 2: mix<2><<<sms * 8, 256>>>(th, a, b, dst, n4, 1e-7f); break;
          default: mix<3><<<sms * 8, 256>>>(th, a, b, dst, n4, 1e-7f); break;
        }
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
      }
      printf("%s  %7.3f ms  %6.0f GB/s\n", names[m], best, bytes[m] * n / (best * 1e-3) / 1e9);
    }
  return 0;
}
