// Column-strip halo copy into a 1 KB-row shared tile: 16-byte cp.async of a
// 211-row x 2-chunk strip per warp (the resident kernel's W/E refresh), with
// the destination chunks either in the same bank group for every row (the
// row-independent tile swizzle) or XOR-spread by row & 7. Cycles per strip.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o strip_copy strip_copy.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void cp16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}

template <int SPREAD>
__global__ void strips(const double* __restrict__ g, int64_t pitch, int rows, int warps_copying,
                       int reps, unsigned long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(sm);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double* src = g + (int64_t)blockIdx.x * 2 * rows * pitch;
  unsigned long long t = 0;
  for (int rep = 0; rep < reps; ++rep) {
    __syncthreads();
    const unsigned long long t0 = clock64();
    if (warp < warps_copying) {
      // this warp's share of the strip rows
      const int r0 = rows * warp / warps_copying, r1 = rows * (warp + 1) / warps_copying;
      const int n = (r1 - r0) * 2;
      for (int i = lane; i < n; i += 32) {
        const int r = r0 + i / 2, q = i & 1;
        const int pq = SPREAD ? (q ^ (r & 7)) : q;
        cp16(base + (uint32_t)(r * 1024 + pq * 16), src + (int64_t)r * pitch + q * 2);
      }
      asm volatile("cp.async.wait_all;" ::: "memory");
    }
    __syncthreads();
    t += clock64() - t0;
  }
  if (threadIdx.x == 0) out[blockIdx.x] = t / reps;
}

// The same strip copy of data a neighbour CTA has just written: every
// iteration CTA i stores its strip (st.cg), releases flag i, waits for flag
// (i+1) % n and copies that CTA's strip; cycles of the copy after the flag.
__global__ void fresh(double* __restrict__ g, int64_t pitch, int rows, int* flags, int iters,
                      int warps_copying, int far, unsigned long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(sm);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n = gridDim.x, me = blockIdx.x, nb = (me + (far ? n / 2 : 1)) % n;
  double* mine = g + (int64_t)me * 2 * rows * pitch;
  const double* theirs = g + (int64_t)nb * 2 * rows * pitch;
  unsigned long long t = 0;
  for (int it = 1; it <= iters; ++it) {
    for (int i = threadIdx.x; i < rows * 4; i += blockDim.x)
      asm volatile("st.global.cg.f64 [%0], %1;" ::"l"(mine + (int64_t)(i / 4) * pitch + (i % 4)),
                   "d"((double)it) : "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      atomicExch(flags + me, it);
    }
    if (threadIdx.x == 0) {
      while (true) {
        int v;
        asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(flags + nb) : "memory");
        if (v >= it) break;
      }
    }
    __syncthreads();
    const unsigned long long t0 = clock64();
    if (warp < warps_copying) {
      const int r0 = rows * warp / warps_copying, r1 = rows * (warp + 1) / warps_copying;
      const int m = (r1 - r0) * 2;
      for (int i = lane; i < m; i += 32) {
        const int r = r0 + i / 2, q = i & 1;
        cp16(base + (uint32_t)(r * 1024 + q * 16), theirs + (int64_t)r * pitch + q * 2);
      }
      asm volatile("cp.async.wait_all;" ::: "memory");
    }
    __syncthreads();
    t += clock64() - t0;
    // keep the next iteration's stores from overtaking a slow reader
    if (threadIdx.x == 0) {
      atomicAdd(flags + n + nb, 1);
      while (atomicAdd(flags + n + me, 0) < it) {}
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = t / iters;
}

int main() {
  const int rows = 211, ctas = 144, reps = 200;
  const int64_t pitch = 1920;
  double* g;
  unsigned long long* out;
  cudaMalloc(&g, (size_t)ctas * 2 * rows * pitch * sizeof(double));
  cudaMemset(g, 0, (size_t)ctas * 2 * rows * pitch * sizeof(double));
  cudaMallocManaged(&out, ctas * sizeof(unsigned long long));
  cudaFuncSetAttribute(strips<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaFuncSetAttribute(strips<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  for (int wc : {1, 2, 3, 8}) {
    for (int spread = 0; spread < 2; ++spread) {
      if (spread) strips<1><<<ctas, 256, 212 * 1024>>>(g, pitch, rows, wc, reps, out);
      else strips<0><<<ctas, 256, 212 * 1024>>>(g, pitch, rows, wc, reps, out);
      cudaDeviceSynchronize();
      unsigned long long s = 0, mx = 0;
      for (int i = 0; i < ctas; ++i) { s += out[i]; mx = out[i] > mx ? out[i] : mx; }
      printf("{\"warps_copying\": %d, \"spread\": %d, \"cycles_avg\": %llu, \"cycles_max\": %llu}\n",
             wc, spread, s / ctas, mx);
    }
  }
  int* flags;
  cudaMalloc(&flags, 2 * ctas * sizeof(int));
  cudaFuncSetAttribute(fresh, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  for (int far = 0; far < 2; ++far)
    for (int wc : {1, 3}) {
      cudaMemset(flags, 0, 2 * ctas * sizeof(int));
      int iters = 200;
      void* args[] = {&g, (void*)&pitch, (void*)&rows, &flags, &iters, &wc, &far, &out};
      cudaLaunchCooperativeKernel((void*)fresh, ctas, 256, args, 212 * 1024, 0);
      cudaError_t e = cudaDeviceSynchronize();
      unsigned long long s = 0, mx = 0;
      for (int i = 0; i < ctas; ++i) { s += out[i]; mx = out[i] > mx ? out[i] : mx; }
      printf("{\"fresh\": 1, \"far\": %d, \"warps_copying\": %d, \"cycles_avg\": %llu, \"cycles_max\": %llu, \"err\": \"%s\"}\n",
             far, wc, s / ctas, mx, cudaGetErrorString(e));
    }
  return 0;
}
