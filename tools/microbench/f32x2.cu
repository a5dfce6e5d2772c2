// FP32 scalar vs packed f32x2 (add.rn.f32x2 / mul.rn.f32x2) throughput on B200.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t add2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t mul2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

template <int CH>
__global__ void k_scalar(float* out, int iters, float s) {
  float x[CH];
  for (int c = 0; c < CH; ++c) x[c] = threadIdx.x + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      x[c] = __fmul_rn(x[c], s);
      x[c] = __fadd_rn(x[c], s);
    }
  }
  float t = 0;
  for (int c = 0; c < CH; ++c) t += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

template <int CH>
__global__ void k_pair(float* out, int iters, float s) {
  uint64_t x[CH];
  const uint64_t ss = ((uint64_t)__float_as_uint(s) << 32) | __float_as_uint(s);
  for (int c = 0; c < CH; ++c) x[c] = ((uint64_t)__float_as_uint(threadIdx.x + c) << 32) | __float_as_uint(c);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      x[c] = mul2(x[c], ss);
      x[c] = add2(x[c], ss);
    }
  }
  float t = 0;
  for (int c = 0; c < CH; ++c) t += __uint_as_float((uint32_t)x[c]) + __uint_as_float((uint32_t)(x[c] >> 32));
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  cudaMalloc(&out, sizeof(float) * sms * 8 * 1024);
  const int iters = 4096;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int warps : {4, 8, 16}) {
    for (int kind = 0; kind < 2; ++kind) {
      auto run = [&]() {
        if (kind == 0) k_scalar<8><<<sms, warps * 32>>>(out, iters, 1.0001f);
        else k_pair<4><<<sms, warps * 32>>>(out, iters, 1.0001f);
      };
      run();
      cudaEventRecord(a);
      run();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      // values per thread per iter: 8 (scalar: 8 chains x 2 ops; pair: 4 chains x 2 vals x 2 ops)
      const double ops = (double)sms * warps * 32 * iters * 8 * 2;
      printf("%s warps/SM %2d: %.1f Gop/s (%.1f op/SM/ns)\n", kind ? "f32x2 " : "scalar", warps,
             ops / ms / 1e6, ops / ms / 1e6 / sms);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
