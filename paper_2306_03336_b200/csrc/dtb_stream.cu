// dtb_stream.cu — the tile-sweep streaming kernel (one HBM pass of h fused
// steps per launch; the planner's fallback for shapes the pipelined kernel
// does not take), the one-step-per-launch naive kernel (the T=1 HBM
// baseline), and the on-device splitmix64 input fill.
#include <algorithm>
#include <cstring>

#include "dtb_internal.h"
#include "dtb_tile_io.cuh"

namespace dtb {

// One HBM pass over every tile. nbuf == 2: the CTA's smem holds two tile
// buffers; tile i+1 streams in (cp.async) while tile i is advanced and
// stored, so HBM traffic overlaps the FP64/FP32 work. nbuf == 1: tall tiles,
// load / compute / store in sequence.
template <typename T, int K, int NW, bool SYM, bool DYN>
__global__ void __launch_bounds__(NW * 32, 1)
stream_kernel(const T* __restrict__ src, T* __restrict__ dst, int64_t pitch, int nx, int ny,
              Weights<T> wt, int steps, int poison, int nbuf, int buf_elems,
              unsigned long long* __restrict__ trace, const __grid_constant__ Geometry geo,
              unsigned long long* __restrict__ cnt) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* bufs[2] = {reinterpret_cast<T*>(smem_raw), reinterpret_cast<T*>(smem_raw) + buf_elems};
  const bool tracing = trace != nullptr && threadIdx.x == 0;
  unsigned long long t_wait = 0, t_comp = 0, t_store = 0, tc = tracing ? clock64() : 0;
#define DTB_MARK(acc)                          \
  if (tracing) {                               \
    const unsigned long long now_ = clock64(); \
    acc += now_ - tc;                          \
    tc = now_;                                 \
  }
  const int ntiles = geo.ntx * geo.nty;
  auto issue_load = [&](int t, T* tile) {
    const int tx = t % geo.ntx, ty = t / geo.ntx;
    const int4 cx = geo.col[tx], cy = geo.row[ty];
    g2s_rows<T, K>(tile, src, pitch, cx.z + 1, cy.z + 1, 0, cy.w - cy.z, 0, cx.w - cx.z);
  };
  int i = 0;
  if (nbuf == 2 && (int)blockIdx.x < ntiles) issue_load(blockIdx.x, bufs[0]);
  cp_async_commit();
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++i) {
    T* tile = bufs[nbuf == 2 ? (i & 1) : 0];
    if (nbuf == 2) {
      const int tn = t + gridDim.x;
      if (tn < ntiles) issue_load(tn, bufs[(i + 1) & 1]);  // prefetch the next tile
      cp_async_commit();
      cp_async_wait_1();  // this tile's copies have landed
    } else {
      issue_load(t, tile);
      cp_async_wait_all();
    }
    __syncthreads();
    DTB_MARK(t_wait)
    const int tx = t % geo.ntx, ty = t / geo.ntx;
    const int4 cx = geo.col[tx], cy = geo.row[ty];
    const int Lw = cx.w - cx.z, Lh = cy.w - cy.z;
    advance<T, K, SYM, DYN>(tile, Lw, Lh, steps, wt, poison != 0, cx.z > -1, cx.w < nx + 1,
                            cy.z > -1, cy.w < ny + 1, nullptr, cnt);
    if (cnt && threadIdx.x == 0) {  // the tile's load and owned store (domain cells)
      atomicAdd(cnt + 0, (unsigned long long)(span_in(cy.z + 1, cy.w + 1, 1, ny + 1) *
                                              span_in(cx.z + 1, cx.w + 1, 1, nx + 1)));
      atomicAdd(cnt + 1, (unsigned long long)((cy.y - cy.x) * (cx.y - cx.x)));
    }
    DTB_MARK(t_comp)
    // owned cells, plus the ghost ring where the tile touches the domain edge
    const int sx0 = cx.x - (cx.x == 0), sx1 = cx.y + (cx.y == nx);
    const int sy0 = cy.x - (cy.x == 0), sy1 = cy.y + (cy.y == ny);
    s2g_rows<T, K>(tile, dst, pitch, cx.z + 1, cy.z + 1, sy0 - cy.z, sy1 - cy.z, sx0 - cx.z,
                   sx1 - cx.z);
    __syncthreads();  // every read of this buffer is done before it is refilled
    DTB_MARK(t_store)
  }
  cp_async_wait_all();
#undef DTB_MARK
  if (tracing) {
    unsigned long long* tr = trace + 8 * blockIdx.x;
    tr[0] += t_comp; tr[1] += t_store; tr[2] += t_wait; tr[4] += i;
  }
}

// one step, global memory (the T=1 HBM baseline)
template <typename T>
__global__ void naive_kernel(const T* __restrict__ a, T* __restrict__ b, int64_t pitch, int nx,
                             int ny, Weights<T> wt) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  for (int y = blockIdx.y; y < ny + 2; y += gridDim.y) {
    if (x >= nx + 2) return;
    const int64_t i = (int64_t)y * pitch + x;
    if (x == 0 || y == 0 || x == nx + 1 || y == ny + 1) {
      b[i] = a[i];
    } else {
      b[i] = cell_update(a[i - 1], a[i + 1], a[i - pitch], a[i], a[i + pitch], wt);
    }
  }
}

// splitmix64 fill (prng.py:45-67): interior (x, y) = value i = y*nx + x.
// Rows [row0, row0 + nrows) of the padded global grid, written to out[0..].
template <typename T>
__global__ void fill_random_kernel(T* out, int64_t pitch, int nx, int ny, uint64_t seed,
                                   double ghost, int64_t row0, int64_t nrows) {
  const int64_t total = (int64_t)(nx + 2) * nrows;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t yl = k / (nx + 2), x = k % (nx + 2), y = row0 + yl;
    double v;
    if (x == 0 || y == 0 || x == nx + 1 || y == ny + 1) {
      v = ghost;
    } else {
      const uint64_t i = (uint64_t)((y - 1) * nx + (x - 1));
      uint64_t z = seed + (i + 1) * 0x9E3779B97F4B7C15ull;
      z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
      z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
      z = z ^ (z >> 31);
      v = (double)(z >> 11) * (1.0 / 9007199254740992.0);
    }
    out[yl * pitch + x] = (T)v;
  }
}

template <typename T, int K, int NW, bool SYM, bool DYN>
int launch_stream_kernel(const Plan& p, const Geometry& geo, const T* d_in, T* d_out,
                         int64_t pitch, int nx, int ny, const Weights<T>& wt, int64_t steps,
                         bool poison, cudaStream_t st, unsigned long long* cnt) {
  const bool tracing = (g_flags & DTB_FLAG_TRACE) != 0;
  const int threads = NW * 32;
  const int smem = (int)p.smem_bytes;
  const size_t grid_bytes = (size_t)(ny + 2) * pitch * sizeof(T);
  int device;
  CUDA_TRY(cudaGetDevice(&device));
  auto kern = stream_kernel<T, K, NW, SYM, DYN>;
  if (int rc = prepare_kernel((const void*)kern, device, smem * p.ctas_per_sm, threads, nullptr))
    return rc;
  const int64_t passes = (steps + p.h - 1) / p.h;
  T* tmp = nullptr;
  if (passes > 1) {
    void* scratch = nullptr;
    if (int rc = arena_get(kArenaScratch, device, grid_bytes, &scratch)) return rc;
    tmp = reinterpret_cast<T*>(scratch);
  }
  const T* src = d_in;
  int64_t done = 0;
  const int nbuf = p.ctas_per_sm;  // the planner's occupancy 2 == double-buffered CTA
  const int buf_elems = (int)(p.smem_bytes / (int64_t)sizeof(T));
  unsigned long long* strace = nullptr;
  const size_t strace_bytes = (size_t)p.ctas * 8 * sizeof(unsigned long long);
  if (tracing) {
    CUDA_TRY(cudaMallocAsync((void**)&strace, strace_bytes, st));
    CUDA_TRY(cudaMemsetAsync(strace, 0, strace_bytes, st));
  }
  for (int64_t i = 0; i < passes; ++i) {
    const int s = (int)std::min<int64_t>(p.h, steps - done);
    T* dst = ((passes - 1 - i) % 2 == 0) ? d_out : tmp;
    kern<<<p.ctas, threads, (size_t)smem * nbuf, st>>>(src, dst, pitch, nx, ny, wt, s,
                                                       poison ? 1 : 0, nbuf, buf_elems, strace,
                                                       geo, cnt);
    g_launches += 1;
    CUDA_TRY(cudaGetLastError());
    src = dst;
    done += s;
  }
  if (tracing) {
    std::vector<unsigned long long> h_tr((size_t)p.ctas * 8);
    CUDA_TRY(cudaMemcpyAsync(h_tr.data(), strace, strace_bytes, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    CUDA_TRY(cudaFreeAsync(strace, st));
    g_trace.assign(h_tr.begin(), h_tr.end());
  }
  return DTB_OK;
}

template <typename T>
int launch_stream(const Plan& p, const Geometry& geo, const T* d_in, T* d_out, int64_t pitch,
                  int nx, int ny, const T w[5], int64_t steps, bool poison, cudaStream_t st,
                  unsigned long long* cnt) {
  constexpr int K = sizeof(T) == 8 ? 4 : 8, NW = 8;
  if (p.K != K || p.warps != NW)
    return fail(DTB_EINFEASIBLE, "no streaming kernel for elem %d K %d warps %d",
                (int)sizeof(T), p.K, p.warps);
  Weights<T> wt{w[0], w[1], w[2], w[3], w[4]};
  const bool sym = weights_isotropic<T>(w);
#define DTB_GO(S, D) \
  return launch_stream_kernel<T, K, NW, S, D>(p, geo, d_in, d_out, pitch, nx, ny, wt, steps, poison, st, cnt)
  if (sym) {
    if (p.dyn()) DTB_GO(true, true);
    DTB_GO(true, false);
  }
  if (p.dyn()) DTB_GO(false, true);
  DTB_GO(false, false);
#undef DTB_GO
}

template <typename T>
int launch_naive(const T* d_in, T* d_out, T* d_tmp, int64_t pitch, int nx, int ny, const T w[5],
                 int64_t steps, cudaStream_t st) {
  Weights<T> wt{w[0], w[1], w[2], w[3], w[4]};
  const T* src = d_in;
  dim3 block(256), grid((unsigned)((nx + 2 + 255) / 256), (unsigned)std::min<int64_t>(ny + 2, 65535));
  for (int64_t i = 0; i < steps; ++i) {
    T* dst = ((steps - 1 - i) % 2 == 0) ? d_out : d_tmp;
    naive_kernel<T><<<grid, block, 0, st>>>(src, dst, pitch, nx, ny, wt);
    g_launches += 1;
    src = dst;
  }
  CUDA_TRY(cudaGetLastError());
  return DTB_OK;
}

template <typename T>
int launch_fill(T* d_out, int64_t pitch, int nx, int ny, uint64_t seed, double ghost,
                int64_t row0, int64_t nrows, cudaStream_t st) {
  fill_random_kernel<T><<<1184, 256, 0, st>>>(d_out, pitch, nx, ny, seed, ghost, row0, nrows);
  CUDA_TRY(cudaGetLastError());
  return DTB_OK;
}

#define DTB_INST(T)                                                                            \
  template int launch_stream<T>(const Plan&, const Geometry&, const T*, T*, int64_t, int, int, \
                                const T*, int64_t, bool, cudaStream_t, unsigned long long*);   \
  template int launch_naive<T>(const T*, T*, T*, int64_t, int, int, const T*, int64_t,         \
                               cudaStream_t);                                                  \
  template int launch_fill<T>(T*, int64_t, int, int, uint64_t, double, int64_t, int64_t,       \
                              cudaStream_t);
DTB_INST(double)
DTB_INST(float)
#undef DTB_INST

}  // namespace dtb
