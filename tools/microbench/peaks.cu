// Microbenchmarks for the j2d5pt roofline denominators on B200 (sm_100a).
// Measures: FP64/FP32 mul+add issue rate (no FMA), SHFL and LDS throughput,
// cooperative grid.sync latency, and an L2 flag ping-pong between two CTAs.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o peaks peaks.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

template <typename T>
__global__ void fp_rate(T* out, int iters, T a, T b) {
  // 8 independent chains of alternating mul/add, every op separately rounded
  T r[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) r[i] = (T)(threadIdx.x + i);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) { r[i] = r[i] * a; r[i] = r[i] + b; }
  }
  T s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += r[i];
  if (s == (T)12345.678) out[threadIdx.x] = s;
}

__global__ void shfl_rate(int* out, int iters) {
  int v = threadIdx.x, w = threadIdx.x * 3;
  for (int it = 0; it < iters; ++it) {
    v = __shfl_sync(0xffffffff, v, (threadIdx.x + 1) & 31);
    w = __shfl_sync(0xffffffff, w, (threadIdx.x + 31) & 31);
  }
  if (v + w == -7) out[threadIdx.x] = v;
}

__global__ void lds_rate(double* out, int iters) {
  extern __shared__ double2 sm[];
  int n = blockDim.x;
  sm[threadIdx.x] = make_double2(threadIdx.x, 1.0);
  __syncthreads();
  double acc = 0;
  int idx = threadIdx.x;
  for (int it = 0; it < iters; ++it) {
    double2 v = sm[idx];
    acc += v.x;
    idx = (idx + 32) % n;
  }
  if (acc == -1.0) out[threadIdx.x] = acc;
}

__global__ void gridsync_lat(int iters, long long* cyc) {
  cg::grid_group g = cg::this_grid();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) g.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) *cyc = clock64() - t0;
}

__global__ void pingpong(volatile int* flags, int iters, long long* cyc) {
  // block 0 and block 1 bounce a counter through L2
  if (threadIdx.x != 0) return;
  int me = blockIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (me == 0) {
      flags[0] = 2 * i + 1;
      __threadfence();
      while (flags[32] != 2 * i + 1) {}
    } else {
      while (flags[0] != 2 * i + 1) {}
      flags[32] = 2 * i + 1;
      __threadfence();
    }
  }
  if (me == 0) *cyc = clock64() - t0;
}

__global__ void clk_probe(long long* c) { *c = clock64(); }

int main() {
  int dev = 0, nsm = 0, clk_khz = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev));
  int smem_optin = 0;
  CK(cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  printf("{\"sms\": %d, \"clock_khz_attr\": %d, \"smem_optin\": %d}\n", nsm, clk_khz, smem_optin);
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  void* dbuf; CK(cudaMalloc(&dbuf, 1 << 20));
  long long* dcyc; CK(cudaMalloc(&dcyc, 64));
  float ms;

  // measure effective SM clock with a long fp64 run: cycles from clock64 unavailable
  // across SMs, so derive rate per second directly.
  {
    int iters = 20000, threads = 512, blocks = nsm * 4;
    fp_rate<double><<<blocks, threads>>>((double*)dbuf, 100, 1.0000001, 1e-9);
    CK(cudaEventRecord(e0));
    fp_rate<double><<<blocks, threads>>>((double*)dbuf, iters, 1.0000001, 1e-9);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    double ops = 16.0 * iters * threads * (double)blocks;
    printf("{\"fp64_ops_per_s\": %.4e, \"fp64_ops_per_sm_per_ns\": %.3f, \"ms\": %.3f}\n",
           ops / (ms * 1e-3), ops / (ms * 1e-3) / nsm / 1e9, ms);
  }
  {
    int iters = 20000, threads = 512, blocks = nsm * 4;
    fp_rate<float><<<blocks, threads>>>((float*)dbuf, 100, 1.0000001f, 1e-9f);
    CK(cudaEventRecord(e0));
    fp_rate<float><<<blocks, threads>>>((float*)dbuf, iters, 1.0000001f, 1e-9f);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    double ops = 16.0 * iters * threads * (double)blocks;
    printf("{\"fp32_ops_per_s\": %.4e, \"fp32_ops_per_sm_per_ns\": %.3f, \"ms\": %.3f}\n",
           ops / (ms * 1e-3), ops / (ms * 1e-3) / nsm / 1e9, ms);
  }
  {
    int iters = 100000, threads = 512, blocks = nsm * 4;
    shfl_rate<<<blocks, threads>>>((int*)dbuf, 100);
    CK(cudaEventRecord(e0));
    shfl_rate<<<blocks, threads>>>((int*)dbuf, iters);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    double warp_shfl = 2.0 * iters * (threads / 32) * (double)blocks;
    printf("{\"shfl_warp_instr_per_sm_per_ns\": %.3f}\n", warp_shfl / (ms * 1e-3) / nsm / 1e9);
  }
  {
    int iters = 100000, threads = 1024, blocks = nsm * 2;
    CK(cudaFuncSetAttribute(lds_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
    lds_rate<<<blocks, threads, threads * 16>>>((double*)dbuf, 100);
    CK(cudaEventRecord(e0));
    lds_rate<<<blocks, threads, threads * 16>>>((double*)dbuf, iters);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    double bytes = 16.0 * iters * threads * (double)blocks;
    printf("{\"lds128_bytes_per_sm_per_ns\": %.3f}\n", bytes / (ms * 1e-3) / nsm / 1e9);
  }
  {
    int iters = 2000;
    void* args[] = {&iters, &dcyc};
    CK(cudaLaunchCooperativeKernel((void*)gridsync_lat, nsm, 256, args, 0, 0));
    CK(cudaEventRecord(e0));
    CK(cudaLaunchCooperativeKernel((void*)gridsync_lat, nsm, 256, args, 0, 0));
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    long long cyc; CK(cudaMemcpy(&cyc, dcyc, 8, cudaMemcpyDeviceToHost));
    printf("{\"gridsync_us\": %.3f, \"gridsync_cycles\": %.1f}\n", ms * 1e3 / iters, (double)cyc / iters);
  }
  {
    int iters = 20000;
    CK(cudaMemset(dbuf, 0, 4096));
    pingpong<<<2, 32>>>((volatile int*)dbuf, 10, dcyc);
    CK(cudaMemset(dbuf, 0, 4096));
    CK(cudaEventRecord(e0));
    pingpong<<<2, 32>>>((volatile int*)dbuf, iters, dcyc);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    long long cyc; CK(cudaMemcpy(&cyc, dcyc, 8, cudaMemcpyDeviceToHost));
    printf("{\"l2_pingpong_roundtrip_us\": %.3f, \"cycles\": %.1f}\n", ms * 1e3 / iters, (double)cyc / iters);
  }
  CK(cudaDeviceSynchronize());
  return 0;
}
