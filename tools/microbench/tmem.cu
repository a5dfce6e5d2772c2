// TMEM as a second tile store for the resident kernel: how fast
// can a warp stream rows through tensor memory with tcgen05.ld / tcgen05.st?
// One CTA per SM allocates all 512 columns; warp w reaches TMEM lanes
// 32*(w%4)..+31 (its quarter), warps w and w+4 use disjoint column halves.
// Reports per-SM bytes/clock for loads and stores (x16 = 16 words per thread
// per instruction, NB instructions in flight before the wait) and the
// single-instruction load-to-use latency.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem tmem.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

#define LD16(a, r)                                                                            \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11," \
               "%12,%13,%14,%15}, [%16];"                                                     \
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),      \
                 "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]),   \
                 "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])                          \
               : "r"(a))
#define ST16(a, r)                                                                            \
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10," \
               "%11,%12,%13,%14,%15,%16};"                                                    \
               ::"r"(a), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]),    \
                 "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]),         \
                 "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]))

template <int NB>
__global__ void __launch_bounds__(256, 1) tmem_bw(long long* cyc, uint32_t* sink, int iters,
                                                   int mode) {
  __shared__ uint32_t taddr_s;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;"
                 ::"r"((uint32_t)__cvta_generic_to_shared(&taddr_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = taddr_s + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * 256);
  uint32_t r[NB][16];
#pragma unroll
  for (int b = 0; b < NB; ++b)
#pragma unroll
    for (int j = 0; j < 16; ++j) r[b][j] = threadIdx.x * 31 + j + b;
  // fill once so loads read defined data
#pragma unroll
  for (int b = 0; b < NB; ++b) ST16(base + b * 16, r[b]);
  asm volatile("tcgen05.wait::st.sync.aligned;");
  uint32_t acc = 0;
  __syncwarp();
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    const uint32_t a = base + (uint32_t)((i & 7) * NB * 16) % 256;
    if (mode == 0) {
#pragma unroll
      for (int b = 0; b < NB; ++b) LD16(a + b * 16, r[b]);
      asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
      for (int b = 0; b < NB; ++b) acc ^= r[b][0] ^ r[b][15];
    } else {
#pragma unroll
      for (int b = 0; b < NB; ++b) { r[b][0] += i; ST16(a + b * 16, r[b]); }
      asm volatile("tcgen05.wait::st.sync.aligned;");
    }
  }
  const long long t1 = clock64();
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if ((threadIdx.x & 31) == 0) cyc[blockIdx.x * 8 + warp] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(taddr_s));
}

template <int NB>
int run(int warps_per_cta, int mode, long long* d_cyc, uint32_t* d_sink) {
  const int iters = 4096, ctas = 148;
  tmem_bw<NB><<<ctas, warps_per_cta * 32>>>(d_cyc, d_sink, iters, mode);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  long long h[148 * 8];
  CK(cudaMemcpy(h, d_cyc, sizeof h, cudaMemcpyDeviceToHost));
  double mx = 0;
  for (int c = 0; c < ctas; ++c)
    for (int w = 0; w < warps_per_cta; ++w) mx = h[c * 8 + w] > mx ? (double)h[c * 8 + w] : mx;
  const double bytes = (double)warps_per_cta * iters * NB * 16 * 32 * 4;  // per SM
  printf("%s x16*%d in flight, %d warps/CTA: %.1f B/clk/SM (%.1f clk per wait round)\n",
         mode == 0 ? "tcgen05.ld" : "tcgen05.st", NB, warps_per_cta, bytes / mx, mx / iters);
  return 0;
}

int main() {
  long long* d_cyc;
  uint32_t* d_sink;
  CK(cudaMalloc(&d_cyc, 148 * 8 * sizeof(long long)));
  CK(cudaMalloc(&d_sink, 148 * 256 * sizeof(uint32_t)));
  CK(cudaMemset(d_cyc, 0, 148 * 8 * sizeof(long long)));
  for (int mode = 0; mode < 2; ++mode) {
    if (run<1>(1, mode, d_cyc, d_sink)) return 1;  // latency-ish: one warp, one in flight
    if (run<1>(4, mode, d_cyc, d_sink)) return 1;
    if (run<4>(4, mode, d_cyc, d_sink)) return 1;
    if (run<4>(8, mode, d_cyc, d_sink)) return 1;
    if (run<2>(8, mode, d_cyc, d_sink)) return 1;
  }
  return 0;
}
