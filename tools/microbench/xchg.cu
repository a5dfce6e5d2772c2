// Cost of the resident halo-exchange primitives on sm_100a, one CTA (256
// threads) per SM, all SMs at once (like the resident kernel):
//   store N 8-byte values in a column pattern (stride = one grid row) or a
//   row pattern (contiguous), then fence; load N values back via cp.async.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o xchg xchg.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void stores(double* g, long pitch, int n, int colmode, int fence, long long* cyc) {
  extern __shared__ double sm[];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = i;
  __syncthreads();
  long long t0 = clock64();
  double* base = g + (long)blockIdx.x * 1100 * pitch;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    long off = colmode ? (long)(i / 4) * pitch + (i % 4) : i;
    __stcg(base + off, sm[i & 4095]);
  }
  if (fence == 1) __threadfence();
  __syncthreads();
  if (fence == 2 && threadIdx.x == 0) __threadfence();
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void loads(const double* g, long pitch, int n, int colmode, long long* cyc) {
  extern __shared__ double sm[];
  unsigned sbase = (unsigned)__cvta_generic_to_shared(sm);
  __syncthreads();
  long long t0 = clock64();
  const double* base = g + (long)blockIdx.x * 1100 * pitch;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    long off = colmode ? (long)(i / 4) * pitch + (i % 4) : i;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sbase + 8u * (i & 4095)),
                 "l"(base + off) : "memory");
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  long pitch = 1902;
  double* g; cudaMalloc(&g, (size_t)nsm * 1100 * pitch * 8 + 65536);
  long long* cyc; cudaMalloc(&cyc, nsm * 8);
  long long h[256];
  int ns[] = {256, 1024, 2048, 4096};
  for (int colmode = 0; colmode < 2; ++colmode)
    for (int n : ns)
      for (int fence = 0; fence < 3; ++fence) {
        stores<<<nsm, 256, 32768>>>(g, pitch, n, colmode, fence, cyc);
        stores<<<nsm, 256, 32768>>>(g, pitch, n, colmode, fence, cyc);
        cudaMemcpy(h, cyc, nsm * 8, cudaMemcpyDeviceToHost);
        long long mx = 0, sum = 0;
        for (int i = 0; i < nsm; ++i) { mx = h[i] > mx ? h[i] : mx; sum += h[i]; }
        printf("{\"op\": \"store\", \"col\": %d, \"n\": %d, \"fence\": %d, \"cyc_avg\": %lld, \"cyc_max\": %lld}\n",
               colmode, n, fence, sum / nsm, mx);
      }
  for (int colmode = 0; colmode < 2; ++colmode)
    for (int n : ns) {
      loads<<<nsm, 256, 32768>>>(g, pitch, n, colmode, cyc);
      loads<<<nsm, 256, 32768>>>(g, pitch, n, colmode, cyc);
      cudaMemcpy(h, cyc, nsm * 8, cudaMemcpyDeviceToHost);
      long long mx = 0, sum = 0;
      for (int i = 0; i < nsm; ++i) { mx = h[i] > mx ? h[i] : mx; sum += h[i]; }
      printf("{\"op\": \"cp.async\", \"col\": %d, \"n\": %d, \"cyc_avg\": %lld, \"cyc_max\": %lld}\n",
             colmode, n, sum / nsm, mx);
    }
  return 0;
}
