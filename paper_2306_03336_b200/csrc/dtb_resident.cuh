// dtb_resident.cuh — the smem-resident persistent kernel and its launcher
// (instantiated per element type by dtb_resident_f64.cu / dtb_resident_f32.cu).
//
// One CTA per tile, all tiles co-resident (cooperative launch, one CTA per
// SM); the whole grid stays in shared memory for the whole solve. Every h
// steps each warp publishes the owned cells of its band that the neighbours'
// halos cover into an L2-resident exchange buffer and bumps its CTA's epoch
// flag (release-add); the halo ring is then refreshed with 16-byte cp.async
// — on fp64 tiles by one warp per neighbour direction that polls only that
// neighbour (acquire, refresh_by_direction), on fp32 tiles split evenly over
// the warps after warp 0 has seen every flag (refresh_flat; dtb_tile_io.cuh).
// This replaces the reference's serial-tile BSP loop
// (engine.py:265-290) and its modelled grid-level barrier
// with point-to-point neighbour synchronisation.
#pragma once
#include <algorithm>
#include <cstdlib>

#include "dtb_internal.h"
#include "dtb_tile_io.cuh"

namespace dtb {

template <typename T, int K, int NW, bool SYM, bool DYN>
__global__ void __launch_bounds__(NW * 32, 1)
resident_kernel(const T* __restrict__ in, T* __restrict__ out, T* __restrict__ xb0,
                T* __restrict__ xb1, int* __restrict__ flags, int64_t pitch, int nx, int ny,
                Weights<T> wt, int64_t total_steps, int h, int poison,
                unsigned long long* __restrict__ trace, const __grid_constant__ Geometry geo,
                unsigned long long* __restrict__ cnt) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  typedef Tile<T, K> L;
  T* tile = reinterpret_cast<T*>(smem_raw);
  const int tx = blockIdx.x % geo.ntx, ty = blockIdx.x / geo.ntx;
  const int vcta = blockIdx.x;
  const int4 cx = geo.col[tx], cy = geo.row[ty];
  const int Lw = cx.w - cx.z, Lh = cy.w - cy.z;
  const int gx0 = cx.z + 1, gy0 = cy.z + 1;  // padded coords of tile (0,0)
  const bool hl = cx.z > -1, hr = cx.w < nx + 1, ht = cy.z > -1, hb = cy.w < ny + 1;

  g2s_rows<T, K>(tile, in, pitch, gx0, gy0, 0, Lh, 0, Lw);
  cp_async_wait_all();
  __syncthreads();
  if (cnt && threadIdx.x == 0)  // domain cells of the load (the ghost ring is not counted)
    atomicAdd(cnt + 0, (unsigned long long)(span_in(gy0, gy0 + Lh, 1, ny + 1) *
                                            span_in(gx0, gx0 + Lw, 1, nx + 1)));

  // how deep each neighbour's load region reaches into my owned cells
  const int bl = tx > 0 ? max(0, geo.col[tx - 1].w - cx.x) : 0;
  const int br = tx + 1 < geo.ntx ? max(0, cx.y - geo.col[tx + 1].z) : 0;
  const int bt = ty > 0 ? max(0, geo.row[ty - 1].w - cy.x) : 0;
  const int bb = ty + 1 < geo.nty ? max(0, cy.y - geo.row[ty + 1].z) : 0;
  // owned rect in tile coordinates
  const int ox0 = cx.x - cx.z, ox1 = cx.y - cx.z, oy0 = cy.x - cy.z, oy1 = cy.y - cy.z;
  // halo ring cells to refresh exclude the frozen ghost ring of the domain
  const int rx0 = hl ? 0 : 1, rx1 = hr ? Lw : Lw - 1, ry0 = ht ? 0 : 1, ry1 = hb ? Lh : Lh - 1;

  int64_t done = 0;
  int epoch = 0;
  unsigned long long t_comp = 0, t_wait = 0, t_ref = 0, t_copy = 0, tc = 0;
  const bool tracing = trace != nullptr && threadIdx.x == 0;
  if (tracing) tc = clock64();
#define DTB_MARK(acc)                          \
  if (tracing) {                               \
    const unsigned long long now_ = clock64(); \
    acc += now_ - tc;                          \
    tc = now_;                                 \
  }
  Publisher<T, K> pub;
  pub.pitch = pitch;
  pub.own0 = oy0;
  pub.own1 = oy1;
  pub.top1 = oy0 + bt;
  pub.bot0 = oy1 - bb;
  pub.full_mask = 0;
  pub.flag = flags + vcta;
  pub.cl0 = ox0;
  pub.wl = bl;
  pub.cr0 = max(ox1 - br, ox0 + bl);
  pub.wr = ox1 - pub.cr0;
  {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int e = 0; e < K; ++e) {
      const int c = lane * K + e;
      if (c >= ox0 && c < ox1) pub.full_mask |= 1u << e;
    }
  }
  // "epoch e published": NW release-adds (one per warp), or one CTA-level
  // release in poison mode (which publishes through smem after the epoch)
  const int flag_per_epoch = poison ? 1 : NW;
  while (true) {
    const int steps = (int)((total_steps - done) < (int64_t)h ? (total_steps - done) : (int64_t)h);
    const bool last = done + steps >= total_steps;
    T* xb = ((epoch + 1) & 1) ? xb1 : xb0;
    pub.g0 = xb + (int64_t)gy0 * pitch + gx0;
    pub.g = pub.g0 + (threadIdx.x & 31) * K;
    // 1. compute the epoch; each warp publishes its band right after its last sweep
    advance<T, K, SYM, DYN>(tile, Lw, Lh, steps, wt, poison != 0, hl, hr, ht, hb,
                            (last || poison) ? nullptr : &pub, cnt, ox1 - ox0);
    done += steps;
    DTB_MARK(t_comp)
    if (last) break;
    ++epoch;
    if (poison) {
      // owned cells the neighbours' halos cover, through smem
      const int t1 = min(oy0 + bt, oy1), b0 = max(oy1 - bb, t1);
      s2g_rows<T, K>(tile, xb, pitch, gx0, gy0, oy0, t1, ox0, ox1);
      s2g_rows<T, K>(tile, xb, pitch, gx0, gy0, b0, oy1, ox0, ox1);
      s2g_rows<T, K>(tile, xb, pitch, gx0, gy0, t1, b0, ox0, ox0 + bl);
      s2g_rows<T, K>(tile, xb, pitch, gx0, gy0, t1, b0, max(ox1 - br, ox0 + bl), ox1);
      if (cnt && threadIdx.x == 0)
        atomicAdd(cnt + 1, (unsigned long long)((t1 - oy0 + oy1 - b0) * (ox1 - ox0) +
                                                (b0 - t1) * (bl + ox1 - max(ox1 - br, ox0 + bl))));
      __syncthreads();
      if (threadIdx.x == 0) st_release_gpu(flags + vcta, epoch);
    }
    // 2+3. wait for the neighbours' epoch flags, stream the halo ring in
    unsigned long long t_poll[2] = {tc, tc};
    // (measured per type: the balanced split wins on 256-column fp32 tiles,
    // C3a +6 %; one warp per neighbour on 128-column fp64 tiles, C2 +2 %)
    if constexpr (sizeof(T) == 4) {
      refresh_flat<T, K>(tile, xb, pitch, gx0, gy0, flags, epoch * flag_per_epoch, geo.ntx,
                         geo.nty, tx, ty, ry0, oy0, oy1, ry1, rx0, ox0, ox1, rx1,
                         tracing ? t_poll : nullptr, cnt);
    } else {
      refresh_by_direction<T, K>(tile, xb, pitch, gx0, gy0, flags, epoch * flag_per_epoch,
                                 geo.ntx, geo.nty, tx, ty, ry0, oy0, oy1, ry1, rx0, ox0, ox1,
                                 rx1, tracing ? t_poll : nullptr, cnt);
      t_poll[1] = t_poll[0];
    }
    if (tracing) {
      t_wait += t_poll[0] - tc;  // warp 0: until the neighbour flags arrived
      t_copy += t_poll[1] - t_poll[0];
      tc = t_poll[1];
    }
    __syncthreads();
    DTB_MARK(t_ref)
  }
#undef DTB_MARK
  if (tracing) {
    unsigned long long* tr = trace + 8 * vcta;
    tr[0] = t_comp; tr[1] = 0; tr[2] = t_wait; tr[3] = t_ref + t_copy; tr[4] = epoch;
    tr[5] = t_copy;
  }
  s2g_rows<T, K>(tile, out, pitch, gx0, gy0, oy0 - !ht, oy1 + !hb, ox0 - !hl, ox1 + !hr);
  if (cnt && threadIdx.x == 0)  // owned cells (the ghost ring copy is not counted)
    atomicAdd(cnt + 1, (unsigned long long)((oy1 - oy0) * (ox1 - ox0)));
}

template <typename T, int K, int NW, bool SYM, bool DYN>
int launch_resident_kernel(const Plan& p, const Geometry& geo, const T* d_in, T* d_out,
                           int64_t pitch, int nx, int ny, const Weights<T>& wt, int64_t steps,
                           bool poison, cudaStream_t st, unsigned long long* cnt) {
  const bool tracing = (g_flags & DTB_FLAG_TRACE) != 0;
  const int threads = NW * 32;
  const int64_t tiles = p.ctas;
  const int smem = (int)p.smem_bytes;
  const size_t grid_bytes = (size_t)(ny + 2) * pitch * sizeof(T);
  int device;
  CUDA_TRY(cudaGetDevice(&device));
  auto kern = resident_kernel<T, K, NW, SYM, DYN>;
  DevInfo di;
  if (int rc = query_dev(di)) return rc;
  int per_sm = 0;
  if (int rc = prepare_kernel((const void*)kern, device, smem, threads, &per_sm)) return rc;
  if (per_sm < 1 || p.ctas > per_sm * di.sms)
    return fail(DTB_ECAPACITY, "resident plan needs %d co-resident CTAs, device holds %d",
                p.ctas, per_sm * di.sms);
  void* scratch = nullptr;
  const size_t flag_bytes = 256 + (size_t)tiles * sizeof(int);
  const size_t trace_bytes = (size_t)tiles * 8 * sizeof(unsigned long long);
  if (int rc = arena_get(kArenaScratch, device, 2 * grid_bytes + flag_bytes + trace_bytes + 256,
                         &scratch))
    return rc;
  T* xb0 = reinterpret_cast<T*>(scratch);
  T* xb1 = reinterpret_cast<T*>(reinterpret_cast<char*>(scratch) + grid_bytes);
  int* flags = reinterpret_cast<int*>(reinterpret_cast<char*>(scratch) + 2 * grid_bytes);
  CUDA_TRY(cudaMemsetAsync(flags, 0, (size_t)tiles * sizeof(int), st));
  unsigned long long* trace = nullptr;
  if (tracing) {
    trace = reinterpret_cast<unsigned long long*>(
        reinterpret_cast<char*>(scratch) + ((2 * grid_bytes + flag_bytes + 255) & ~(size_t)255));
    CUDA_TRY(cudaMemsetAsync(trace, 0, trace_bytes, st));
  }
  int h = p.h;
  int pois = poison ? 1 : 0;
  void* args[] = {(void*)&d_in, (void*)&d_out, (void*)&xb0, (void*)&xb1, (void*)&flags,
                  (void*)&pitch, (void*)&nx, (void*)&ny, (void*)&wt, (void*)&steps,
                  (void*)&h, (void*)&pois, (void*)&trace, (void*)&geo, (void*)&cnt};
  CUDA_TRY(cudaLaunchCooperativeKernel((const void*)kern, dim3(p.ctas), dim3(threads), args,
                                       (size_t)smem, st));
  g_launches += 1;
  CUDA_TRY(cudaGetLastError());
  if (tracing) {
    std::vector<unsigned long long> h_tr((size_t)tiles * 8);
    CUDA_TRY(cudaMemcpyAsync(h_tr.data(), trace, trace_bytes, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    g_trace.assign(h_tr.begin(), h_tr.end());
  }
  return DTB_OK;
}

// kernel shapes compiled (the planner's candidates, dtb_plan.cpp shapes_for):
// fp64 K=4 / fp32 K=8 (a 1 KB smem row per warp-row), 8 warps
template <typename T>
int launch_resident_impl(const Plan& p, const Geometry& geo, const T* d_in, T* d_out,
                         int64_t pitch, int nx, int ny, const T w[5], int64_t steps, bool poison,
                         cudaStream_t st, unsigned long long* cnt) {
  constexpr int K = sizeof(T) == 8 ? 4 : 8, NW = 8;
  if (p.K != K || p.warps != NW)
    return fail(DTB_EINFEASIBLE, "no resident kernel for elem %d K %d warps %d", (int)sizeof(T),
                p.K, p.warps);
  Weights<T> wt{w[0], w[1], w[2], w[3], w[4]};
  const bool sym = weights_isotropic<T>(w);
#define DTB_GO(S, D) \
  return launch_resident_kernel<T, K, NW, S, D>(p, geo, d_in, d_out, pitch, nx, ny, wt, steps, poison, st, cnt)
  if (sym) {
    if (p.dyn()) DTB_GO(true, true);
    DTB_GO(true, false);
  }
  if (p.dyn()) DTB_GO(false, true);
  DTB_GO(false, false);
#undef DTB_GO
}

template <typename T>
int launch_resident(const Plan& p, const Geometry& geo, const T* d_in, T* d_out, int64_t pitch,
                    int nx, int ny, const T w[5], int64_t steps, bool poison, cudaStream_t st,
                    unsigned long long* cnt) {
  return launch_resident_impl<T>(p, geo, d_in, d_out, pitch, nx, ny, w, steps, poison, st, cnt);
}

}  // namespace dtb
