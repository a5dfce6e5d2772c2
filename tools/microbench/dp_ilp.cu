// FP64 issue rate on sm_100a as a function of independent chains per warp (ILP)
// and warps per SM — tells how much ILP the stencil's FP64 pipeline needs.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o dp_ilp dp_ilp.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int C>
__global__ void chains(double* out, int iters, double a, double b) {
  double r[C];
#pragma unroll
  for (int i = 0; i < C; ++i) r[i] = threadIdx.x + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < C; ++i) r[i] = __dadd_rn(__dmul_rn(r[i], a), b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < C; ++i) s += r[i];
  if (s == 1.2345) out[threadIdx.x] = s;
}

template <int C>
void run(double* d, int warps, int nsm) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 20000 / C * 8;
  chains<C><<<nsm, warps * 32>>>(d, 10, 1.0000001, 1e-9);
  cudaEventRecord(e0);
  chains<C><<<nsm, warps * 32>>>(d, iters, 1.0000001, 1e-9);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double ops = 2.0 * C * iters * warps * 32.0 * nsm;
  printf("{\"chains\": %d, \"warps_per_sm\": %d, \"dp_ops_per_sm_per_ns\": %.2f}\n", C, warps,
         ops / (ms * 1e-3) / nsm / 1e9);
}

int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double* d; cudaMalloc(&d, 1 << 20);
  int ws[] = {4, 8, 16, 32};
  for (int w : ws) { run<1>(d, w, nsm); run<2>(d, w, nsm); run<4>(d, w, nsm); run<8>(d, w, nsm); run<16>(d, w, nsm); }
  // dependent-chain latency: 1 warp per SM, 1 chain
  cudaDeviceSynchronize();
  return 0;
}
