// dtb_kernels.cu — sm_100a kernels and the C ABI (include/dtb_b200.h).
//
//   resident_kernel  persistent cooperative launch, one CTA per SM; the whole
//                    grid stays in shared memory for the whole solve. Every h
//                    steps each CTA publishes the owned cells its neighbours'
//                    halos cover into an L2-resident exchange buffer, bumps an
//                    epoch flag (release), waits only for its <= 8 neighbours'
//                    flags (acquire) and refreshes its halo ring. Replaces the
//                    reference's serial-tile BSP loop (engine.py:265-290) and
//                    its modelled "grid-level barrier".
//   stream_kernel    one HBM pass: every tile loads owned+h halo from `src`,
//                    fuses h steps in smem, stores owned cells to `dst`.
//   naive_kernel     one global-memory step per launch (T=1 baseline).
//   fill_random      on-device splitmix64, bit-identical to prng.py:45-67.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/dtb_b200.h"
#include "dtb_core.cuh"
#include "dtb_pipe.cuh"
#include "dtb_plan.h"

namespace dtb {

constexpr int kMaxTiles = 512;  // per dimension


// Tile geometry as kernel parameters (<= 32 KB param space on sm_70+ / CUDA 12.1+).
// col[i] = (owned x0, owned x1, load x0, load x1) in interior coordinates.
struct Geometry {
  int ntx, nty;
  int4 col[kMaxTiles];
  int4 row[kMaxTiles];
};

template <typename T>
struct Problem {
  const T* in;
  T* out;
  int64_t pitch;  // elements per row of in/out
  int nx, ny;
  Weights<T> wt;
};

// ---------------------------------------------------------------------------
// global <-> smem movement. A copy is a list of up to 4 tile rectangles
// spread over all CTA threads. Index -> (row, col) uses a 64-bit multiply by
// a precomputed reciprocal m = ceil(2^32 / width), exact for idx < 2^32/width.
// ---------------------------------------------------------------------------
template <int N>
struct RectList {
  // rect j: rows [r0, r0 + n/w), cols [c0, c0 + w); cells [end[j-1], end[j]) of the
  // flattened space. set() is called with literal j in order, so after inlining
  // every array index is static and the struct lives in registers.
  int r0[N], c0[N], w[N], end[N];
  uint64_t m[N];
  __device__ __forceinline__ void set(int j, int ra, int rb, int ca, int cb) {
    const bool empty = rb <= ra || cb <= ca;
    r0[j] = ra;
    c0[j] = ca;
    w[j] = empty ? 1 : cb - ca;
    m[j] = (0xFFFFFFFFull + (uint64_t)w[j]) / (uint64_t)w[j];
    end[j] = (j ? end[j - 1] : 0) + (empty ? 0 : (rb - ra) * (cb - ca));
  }
  __device__ __forceinline__ int total() const { return end[N - 1]; }
  __device__ __forceinline__ void locate(int i, int& r, int& c) const {
    int rr = r0[0], cc = c0[0], ww = w[0], st = 0;
    uint64_t mm = m[0];
#pragma unroll
    for (int j = 1; j < N; ++j)
      if (i >= end[j - 1]) { rr = r0[j]; cc = c0[j]; ww = w[j]; mm = m[j]; st = end[j - 1]; }
    const uint32_t li = (uint32_t)(i - st);
    const uint32_t q = (uint32_t)(((uint64_t)li * mm) >> 32);
    r = rr + (int)q;
    c = cc + (int)(li - q * (uint32_t)ww);
  }
};


__device__ __forceinline__ void cp_async(uint32_t dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async(uint32_t dst, const float* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;" ::: "memory");
}

// tile cells of `rl` <- global (padded coords gy0 + r, gx0 + c), as
// asynchronous global->shared copies (LDGSTS): no registers are held, every
// copy of the CTA is in flight at once, one L2/HBM latency covers the lot.
// The caller must __syncthreads() afterwards.
template <typename T, int K, int N, int GT = 0>
__device__ __forceinline__ void g2s(T* tile, const T* __restrict__ g, int64_t pitch, int gx0,
                                    int gy0, const RectList<N>& rl) {
  typedef Tile<T, K> L;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(tile);
  const int nt = gt_n<GT>();
#pragma unroll
  for (int j = 0; j < N; ++j) {
    const int n = rl.end[j] - (j ? rl.end[j - 1] : 0);
    const uint32_t w = (uint32_t)rl.w[j];
    const uint64_t m = rl.m[j];
    for (int i = gt_tid<GT>(); i < n; i += nt) {
      const uint32_t q = (uint32_t)(((uint64_t)(uint32_t)i * m) >> 32);
      const int r = rl.r0[j] + (int)q, c = rl.c0[j] + (int)((uint32_t)i - q * w);
      cp_async(sbase + (uint32_t)(L::at(r, c) * (int)sizeof(T)),
               g + (int64_t)(gy0 + r) * pitch + (gx0 + c));
    }
  }
  cp_async_wait_all();
}

// global (padded coords) <- tile cells of `rl`
template <typename T, int K, int N, int GT = 0>
__device__ __forceinline__ void s2g(const T* tile, T* __restrict__ g, int64_t pitch, int gx0,
                                    int gy0, const RectList<N>& rl) {
  typedef Tile<T, K> L;
  const int nt = gt_n<GT>();
  for (int i = gt_tid<GT>(); i < rl.total(); i += nt) {
    int r, c;
    rl.locate(i, r, c);
    __stcg(g + (int64_t)(gy0 + r) * pitch + (gx0 + c), tile[L::at(r, c)]);
  }
}

// Resident halo refresh: top/bottom ring rows one warp per row (coalesced),
// side ring columns one thread per row; all as cp.async, one latency.
template <typename T, int K, int GT = 0>
__device__ __forceinline__ void refresh_ring(T* tile, const T* __restrict__ g, int64_t pitch,
                                             int gx0, int gy0, int ry0, int oy0, int oy1, int ry1,
                                             int rx0, int ox0, int ox1, int rx1) {
  typedef Tile<T, K> L;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(tile);
  const int warp = gt_tid<GT>() >> 5, lane = threadIdx.x & 31, nw = gt_n<GT>() >> 5;
  const int ntop = oy0 - ry0, nrows = ntop + (ry1 - oy1);
  for (int k = warp; k < nrows; k += nw) {
    const int r = k < ntop ? ry0 + k : oy1 + (k - ntop);
    const T* src = g + (int64_t)(gy0 + r) * pitch + gx0;
    for (int c = rx0 + lane; c < rx1; c += 32)
      cp_async(sbase + (uint32_t)(L::at(r, c) * (int)sizeof(T)), src + c);
  }
  for (int r = oy0 + gt_tid<GT>(); r < oy1; r += gt_n<GT>()) {
    const T* src = g + (int64_t)(gy0 + r) * pitch + gx0;
    for (int c = rx0; c < ox0; ++c) cp_async(sbase + (uint32_t)(L::at(r, c) * (int)sizeof(T)), src + c);
    for (int c = ox1; c < rx1; ++c) cp_async(sbase + (uint32_t)(L::at(r, c) * (int)sizeof(T)), src + c);
  }
  cp_async_wait_all();
}

__device__ __forceinline__ double lds_elem(uint32_t a, double) {
  double v;
  asm("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts_elem(uint32_t a, double v) {
  asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
__device__ __forceinline__ void sts_elem(uint32_t a, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
}
__device__ __forceinline__ float lds_elem(uint32_t a, float) {
  float v;
  asm("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}

// Whole-rectangle tile copies, one warp per row, one 16-byte smem chunk per
// lane-iteration (the swizzled chunk address is computed once per chunk):
// tile rows [r0, r1) x cols [c0, c1) <-> global padded (gy0 + r, gx0 + c).
// When the global side is 16-byte aligned chunk-for-chunk (gx0 and pitch
// multiples of the chunk), whole chunks move as one 16-byte cp.async / STG;
// otherwise element by element. Loads are cp.async (caller waits + syncs).
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}

template <typename T, int K, int GT = 0>
__device__ __forceinline__ void g2s_rows(T* tile, const T* __restrict__ g, int64_t pitch, int gx0,
                                         int gy0, int r0, int r1, int c0, int c1) {
  typedef Tile<T, K> L;
  constexpr int E = L::EPC;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(tile);
  const int warp = gt_tid<GT>() >> 5, lane = threadIdx.x & 31, nw = gt_n<GT>() >> 5;
  const bool vec = ((gx0 % E) == 0) && ((pitch % E) == 0);
  const int q0 = c0 / E, q1 = (c1 + E - 1) / E;
  for (int r = r0 + warp; r < r1; r += nw) {
    const T* src = g + (int64_t)(gy0 + r) * pitch + gx0;
    const uint32_t srow = sbase + (uint32_t)(r * L::ROW * (int)sizeof(T));
    for (int q = q0 + lane; q < q1; q += 32) {
      const uint32_t sa = srow + (uint32_t)(L::swz(q) * 16);
      const int cb = q * E;
      if (vec && cb >= c0 && cb + E <= c1) {
        cp_async16(sa, src + cb);
      } else {
#pragma unroll
        for (int e = 0; e < E; ++e)
          if (cb + e >= c0 && cb + e < c1) cp_async(sa + (uint32_t)(e * sizeof(T)), src + cb + e);
      }
    }
  }
}

template <typename T, int K, int GT = 0>
__device__ __forceinline__ void s2g_rows(const T* tile, T* __restrict__ g, int64_t pitch, int gx0,
                                         int gy0, int r0, int r1, int c0, int c1) {
  typedef Tile<T, K> L;
  typedef typename Arith<T>::vec_t V;
  constexpr int E = L::EPC;
  const int warp = gt_tid<GT>() >> 5, lane = threadIdx.x & 31, nw = gt_n<GT>() >> 5;
  const bool vec = ((gx0 % E) == 0) && ((pitch % E) == 0);
  const int q0 = c0 / E, q1 = (c1 + E - 1) / E;
  for (int r = r0 + warp; r < r1; r += nw) {
    T* dst = g + (int64_t)(gy0 + r) * pitch + gx0;
    const T* srow = tile + r * L::ROW;
    for (int q = q0 + lane; q < q1; q += 32) {
      const V x = *reinterpret_cast<const V*>(srow + L::swz(q) * E);
      const T* px = reinterpret_cast<const T*>(&x);
      const int cb = q * E;
      if (vec && cb >= c0 && cb + E <= c1) {
        *reinterpret_cast<V*>(dst + cb) = x;
      } else {
#pragma unroll
        for (int e = 0; e < E; ++e)
          if (cb + e >= c0 && cb + e < c1) dst[cb + e] = px[e];
      }
    }
  }
}

// Halo refresh, warp-specialised by direction: region k (N, S, W, E, NW, NE,
// SW, SE) of the ring is owned by one neighbour; warp k polls that
// neighbour's epoch flag and streams the region in with cp.async as soon as
// it is published, so the eight waits and loads overlap.
__device__ __forceinline__ int ld_relaxed_gpu(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Copy tile rect [r0, r1) x [c0, c1) from global by 16-byte smem chunks,
// flattened over (row, chunk) across the 32 lanes of one warp. Whole chunks
// use a 16-byte cp.async when the global side is aligned (vec).
template <typename T, int K>
__device__ __forceinline__ void warp_g2s_chunks(uint32_t sbase, const T* __restrict__ g,
                                                int64_t pitch, int gx0, int gy0, int r0, int r1,
                                                int c0, int c1, bool vec, int lane) {
  typedef Tile<T, K> L;
  constexpr int E = L::EPC;
  const int q0 = c0 / E, nq = (c1 + E - 1) / E - q0, n = (r1 - r0) * nq;
  if (n <= 0) return;
  const uint64_t m = (0xFFFFFFFFull + (uint64_t)nq) / (uint64_t)nq;
  for (int i = lane; i < n; i += 32) {
    const uint32_t rr = (uint32_t)(((uint64_t)(uint32_t)i * m) >> 32);
    const int r = r0 + (int)rr, q = q0 + i - (int)rr * nq, cb = q * E;
    const uint32_t sa = sbase + (uint32_t)((r * L::ROW + L::swz(q) * E) * (int)sizeof(T));
    const T* src = g + (int64_t)(gy0 + r) * pitch + gx0 + cb;
    if (vec && cb >= c0 && cb + E <= c1) {
      cp_async16(sa, src);
    } else {
#pragma unroll
      for (int e = 0; e < E; ++e)
        if (cb + e >= c0 && cb + e < c1) cp_async(sa + (uint32_t)(e * sizeof(T)), src + e);
    }
  }
}

// Thread-block cluster pair (DTB_CLUSTER): horizontally adjacent tiles
// (tx, tx^1) run as one 2-CTA cluster, and the side strip a tile needs from
// its partner is read straight out of the partner's shared memory (DSMEM)
// instead of the L2 exchange buffer. Ordering: every thread arrives
// (release) on the cluster barrier after its epoch's sweeps; the warp that
// copies the partner strip waits (acquire) first, the others after their
// tasks; the refresh closes with a full cluster barrier so the partner has
// read my seam columns before my next sweep overwrites them.
#ifndef DTB_CLUSTER
#define DTB_CLUSTER 0
#endif
#ifndef DTB_CLUSTER_RELAXED
#define DTB_CLUSTER_RELAXED 0  // 1: relaxed arrives (timing probe only: no release ordering)
#endif
__device__ __forceinline__ void cluster_arrive() {
  if (DTB_CLUSTER_RELAXED)
    asm volatile("barrier.cluster.arrive.relaxed;" ::: "memory");
  else
    asm volatile("barrier.cluster.arrive.release;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire;" ::: "memory");
}
__device__ __forceinline__ uint32_t dsmem_map(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
// remote loads carry no memory clobber so a batch of them is in flight at
// once; the cluster barrier asm (volatile, clobbers memory) orders them
__device__ __forceinline__ double dsmem_ld(uint32_t a, double) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ float dsmem_ld(uint32_t a, float) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}
// tile rect [r0, r1) x [c0, c1) <- partner tile (r, c + dc), one warp; each
// lane issues 8 remote loads before its 8 local stores
template <typename T, int K>
__device__ __forceinline__ void warp_dsmem_strip(T* tile, uint32_t pbase, int r0, int r1,
                                                 int c0, int c1, int dc, int lane) {
  typedef Tile<T, K> L;
  constexpr int B = 8;
  const int w = c1 - c0, n = (r1 - r0) * w;
  for (int i0 = lane; i0 < n; i0 += 32 * B) {
    T v[B];
    int d[B];
#pragma unroll
    for (int u = 0; u < B; ++u) {
      const int i = i0 + 32 * u;
      if (i < n) {
        const int q = i / w, r = r0 + q, c = c0 + (i - q * w);
        d[u] = L::at(r, c);
        v[u] = dsmem_ld(pbase + (uint32_t)(L::at(r, c + dc) * (int)sizeof(T)), T());
      }
    }
#pragma unroll
    for (int u = 0; u < B; ++u)
      if (i0 + 32 * u < n) tile[d[u]] = v[u];
  }
}

// Halo refresh, warp-specialised: the ring is cut into 16 tasks (N, S, the 4
// corners, and the W and E side columns in 5 row slices each), each owned by
// one neighbour; a warp polls that neighbour's epoch flag and streams the
// task's cells in with cp.async as soon as they are published, so the waits
// and loads overlap across warps.
template <typename T, int K, int GT = 0>
__device__ __forceinline__ void refresh_by_direction(T* tile, const T* __restrict__ g,
                                                     int64_t pitch, int gx0, int gy0,
                                                     const int* flags, int epoch, int ntx, int nty,
                                                     int tx, int ty, int ry0, int oy0, int oy1,
                                                     int ry1, int rx0, int ox0, int ox1, int rx1,
                                                     unsigned long long* mark = nullptr,
                                                     int ptx = -1, uint32_t pbase = 0, int pdc = 0) {
  typedef Tile<T, K> L;
#ifndef DTB_SIDE_PARTS
#define DTB_SIDE_PARTS 1
#endif
  constexpr int kSideParts = DTB_SIDE_PARTS;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(tile);
  const int warp = gt_tid<GT>() >> 5, lane = threadIdx.x & 31, nw = gt_n<GT>() >> 5;
  const bool vec = ((gx0 % L::EPC) == 0) && ((pitch % L::EPC) == 0);
  const int side_rows = oy1 - oy0;
  int polled = -1;  // neighbour this warp last waited for
  // Cluster phases per epoch: P1 (arrived by the caller after the sweeps)
  // gates the partner-strip copy; P2 tells the partner its seam columns have
  // been read. Warps without the copy pass P1 and arrive on P2 up front so
  // the partner never waits for this CTA's global-memory refresh.
  bool copy_warp = false;
  if (DTB_CLUSTER && ptx >= 0) {
    for (int k = warp; k < 6 + 2 * kSideParts; k += nw)
      copy_warp |= k >= 6 && (((k - 6) < kSideParts) ? tx - 1 : tx + 1) == ptx;
    if (!copy_warp) {
      cluster_wait();
      cluster_arrive();
    }
  }
  bool waited = !copy_warp;
  for (int k = warp; k < 6 + 2 * kSideParts; k += nw) {
    int dx, dy, r0, r1, c0, c1;
    if (k < 6) {
      switch (k) {
        case 0: dx = 0; dy = -1; r0 = ry0; r1 = oy0; c0 = ox0; c1 = ox1; break;
        case 1: dx = 0; dy = 1; r0 = oy1; r1 = ry1; c0 = ox0; c1 = ox1; break;
        case 2: dx = -1; dy = -1; r0 = ry0; r1 = oy0; c0 = rx0; c1 = ox0; break;
        case 3: dx = 1; dy = -1; r0 = ry0; r1 = oy0; c0 = ox1; c1 = rx1; break;
        case 4: dx = -1; dy = 1; r0 = oy1; r1 = ry1; c0 = rx0; c1 = ox0; break;
        default: dx = 1; dy = 1; r0 = oy1; r1 = ry1; c0 = ox1; c1 = rx1; break;
      }
    } else {
      const int j = (k - 6) % kSideParts;
      const bool west = (k - 6) < kSideParts;
      dx = west ? -1 : 1;
      dy = 0;
      r0 = oy0 + side_rows * j / kSideParts;
      r1 = oy0 + side_rows * (j + 1) / kSideParts;
      c0 = west ? rx0 : ox1;
      c1 = west ? ox0 : rx1;
    }
    const int nxt = tx + dx, nyt = ty + dy;
    if (r1 <= r0 || c1 <= c0 || nxt < 0 || nxt >= ntx || nyt < 0 || nyt >= nty) continue;
    if (DTB_CLUSTER && dy == 0 && nxt == ptx) {  // the cluster partner's strip: DSMEM
      if (!waited) cluster_wait();
#ifndef DTB_CLUSTER_NOCOPY
#define DTB_CLUSTER_NOCOPY 0  // 1: timing probe, partner strip not copied (wrong results)
#endif
      if (!DTB_CLUSTER_NOCOPY) warp_dsmem_strip<T, K>(tile, pbase, r0, r1, c0, c1, pdc, lane);
      if (!waited) cluster_arrive();
      waited = true;
      continue;
    }
    const int nb = nyt * ntx + nxt;
    if (nb != polled) {
#ifndef DTB_POLL
#define DTB_POLL 0  // 0: acquire load per poll; 1: relaxed polls + one acquire load;
                    // 2: relaxed polls (no sleep) + one acquire load
#endif
      if (lane == 0) {
        if (DTB_POLL == 0) {
          while (ld_acquire_gpu(flags + nb) < epoch) __nanosleep(32);
        } else {
          while (ld_relaxed_gpu(flags + nb) < epoch)
            if (DTB_POLL == 1) __nanosleep(32);
          (void)ld_acquire_gpu(flags + nb);
        }
      }
      __syncwarp();
      if (mark && polled < 0) *mark = clock64();
      polled = nb;
    }
    warp_g2s_chunks<T, K>(sbase, g, pitch, gx0, gy0, r0, r1, c0, c1, vec, lane);
  }
  if (DTB_CLUSTER && !waited) {  // copy task was empty
    cluster_wait();
    cluster_arrive();
  }
  cp_async_wait_all();
}

// Resident publish of the owned band: rows [oy0, t1) and [b0, oy1) in full
// (one warp per row, coalesced), and the side columns [ox0, c1), [c2, ox1) of
// the rows in between (one thread per row).
template <typename T, int K, int GT = 0>
__device__ __forceinline__ void publish_band(const T* tile, T* __restrict__ g, int64_t pitch,
                                             int gx0, int gy0, int oy0, int t1, int b0, int oy1,
                                             int ox0, int c1, int c2, int ox1) {
  typedef Tile<T, K> L;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(tile);
  const int warp = gt_tid<GT>() >> 5, lane = threadIdx.x & 31, nw = gt_n<GT>() >> 5;
  const int ntop = t1 - oy0, nrows = ntop + (oy1 - b0);
  for (int k = warp; k < nrows; k += nw) {
    const int r = k < ntop ? oy0 + k : b0 + (k - ntop);
    T* dst = g + (int64_t)(gy0 + r) * pitch + gx0;
#pragma unroll 4
    for (int c = ox0 + lane; c < ox1; c += 32)
      dst[c] = lds_elem(sbase + (uint32_t)(L::at(r, c) * (int)sizeof(T)), T());
  }
  // side columns, flattened column-fastest so a warp's stores hit few sectors
  const int wl = c1 - ox0, wr = ox1 - c2, nr = b0 - t1;
  const int nl = wl > 0 ? nr * wl : 0, ntot = nl + (wr > 0 ? nr * wr : 0);
  const uint32_t ml = wl > 0 ? (65535u + wl) / wl : 0, mr = wr > 0 ? (65535u + wr) / wr : 0;
  for (int i = gt_tid<GT>(); i < ntot; i += gt_n<GT>()) {
    int r, c;
    if (i < nl) {
      const uint32_t q = ((uint32_t)i * ml) >> 16;
      r = t1 + (int)q;
      c = ox0 + i - (int)q * wl;
    } else {
      const uint32_t j = (uint32_t)(i - nl), q = (j * mr) >> 16;
      r = t1 + (int)q;
      c = c2 + (int)j - (int)q * wr;
    }
    g[(int64_t)(gy0 + r) * pitch + gx0 + c] =
        lds_elem(sbase + (uint32_t)(L::at(r, c) * (int)sizeof(T)), T());
  }
}

// Resident publish of the side columns [c0, c1) and [c2, c3) of rows [r0, r1):
// one thread per row.
template <typename T, int K, int GT = 0>
__device__ __forceinline__ void publish_sides(const T* tile, T* __restrict__ g, int64_t pitch,
                                              int gx0, int gy0, int r0, int r1, int c0, int c1,
                                              int c2, int c3) {
  typedef Tile<T, K> L;
  for (int r = r0 + gt_tid<GT>(); r < r1; r += gt_n<GT>()) {
    T* dst = g + (int64_t)(gy0 + r) * pitch + gx0;
    for (int c = c0; c < c1; ++c) __stcg(dst + c, tile[L::at(r, c)]);
    for (int c = c2; c < c3; ++c) __stcg(dst + c, tile[L::at(r, c)]);
  }
}

// Poison (debug, DTB_FLAG_POISON): NaN every tile cell a correct schedule can
// no longer read after `done` steps of the epoch — the ring of width `done`
// along halo sides (the trapezoid rim, planner.py:272-286) plus the unused
// lane columns. A stale read anywhere then propagates NaN into the owned
// cells and fails the bitwise comparison (the reference's poison mode,
// engine.py:16-20,174-177).
template <typename T, int K, int GT = 0>
__device__ void poison_rim(T* tile, int Lw, int Lh, int done, bool hl, bool hr, bool ht, bool hb) {
  typedef Tile<T, K> L;
  const T nanv = (T)NAN;
  for (int i = gt_tid<GT>(); i < Lh * L::ROW; i += gt_n<GT>()) {
    const int r = i / L::ROW, c = i % L::ROW;
    bool p = c >= Lw;
    p |= hl && c < done;
    p |= hr && c >= Lw - done;
    p |= ht && r < done;
    p |= hb && r >= Lh - done;
    if (p) tile[L::at(r, c)] = nanv;
  }
}

#ifndef DTB_FREEZE_HALO_COLS
#define DTB_FREEZE_HALO_COLS 1  // 0: freeze only domain-ghost columns (parity-green, no gain)
#endif
template <typename T, int K, bool DYN, int GT = 0>
__device__ void advance(T* tile, int Lw, int Lh, int steps, const Weights<T>& wt, bool poison,
                        bool hl, bool hr, bool ht, bool hb,
                        const Publisher<T, K>* pub = nullptr, int* bsmem = nullptr,
                        int* bseq = nullptr) {
  if (!poison) {
    // freeze only the domain's ghost columns; stale halo columns are harmless
    advance_tile<T, K, DYN, GT>(tile, Lw, Lh, steps, wt, pub, bsmem, bseq,
                                !DTB_FREEZE_HALO_COLS ? !hl : true,
                                !DTB_FREEZE_HALO_COLS ? !hr : true);
    return;
  }
  // poison mode: one step at a time, NaN the stale rim after each
  for (int s = 0; s < steps; ++s) {
    advance_tile<T, K, DYN, GT>(tile, Lw, Lh, 1, wt);
    poison_rim<T, K, GT>(tile, Lw, Lh, s + 1, hl, hr, ht, hb);
    gt_sync<GT>();
  }
}

// ---------------------------------------------------------------------------
// streaming: one pass of h fused steps over every tile
// ---------------------------------------------------------------------------
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// One HBM pass over every tile. nbuf == 2: the CTA's smem holds two tile
// buffers; tile i+1 streams in (cp.async) while tile i is advanced and
// stored, so HBM traffic overlaps the FP64/FP32 work. nbuf == 1: tall tiles,
// load / compute / store in sequence.
template <typename T, int K, int NW, bool DYN>
__global__ void __launch_bounds__(NW * 32, 1)
stream_kernel(const T* __restrict__ src, T* __restrict__ dst, int64_t pitch, int nx, int ny,
              Weights<T> wt, int steps, int poison, int nbuf, int buf_elems,
              unsigned long long* __restrict__ trace, const __grid_constant__ Geometry geo) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* bufs[2] = {reinterpret_cast<T*>(smem_raw), reinterpret_cast<T*>(smem_raw) + buf_elems};
  const bool tracing = trace != nullptr && threadIdx.x == 0;
  unsigned long long t_wait = 0, t_comp = 0, t_store = 0, tc = tracing ? clock64() : 0;
#define DTB_MARK(acc)                                  \
  if (tracing) {                                       \
    const unsigned long long now_ = clock64();         \
    acc += now_ - tc;                                  \
    tc = now_;                                         \
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
    advance<T, K, DYN>(tile, Lw, Lh, steps, wt, poison != 0, cx.z > -1, cx.w < nx + 1,
                       cy.z > -1, cy.w < ny + 1);
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

// ---------------------------------------------------------------------------
// pipelined streaming pass (dtb_pipe.cuh): NW/S pipelines of S warps per CTA,
// each pipeline marching column-strip segments; h = 2S steps per pass.
// ---------------------------------------------------------------------------
template <int S>
struct PipeSmem {
  int prod[S], cons[S];
};

template <typename T, int K, int NW, int S, bool DYN, bool MIR = false>
__global__ void __launch_bounds__(NW * 32, 1)
pipe_kernel(const T* __restrict__ src, T* __restrict__ dst, int64_t pitch, int nx, int ny,
            Weights<T> wt, int steps, const __grid_constant__ Geometry geo,
            const __grid_constant__ HaloMirror<T> mir) {
  constexpr int P = NW / S;
  typedef Tile<T, K> L;
  constexpr int RB = L::ROW * (int)sizeof(T);
  constexpr int kRing0Rows = PipeCfg<NW, T>::kRing0Rows, kRingRows = PipeCfg<NW, T>::kRingRows;
  constexpr int kPipeBytes = (kRing0Rows + (S - 1) * kRingRows) * RB;
  extern __shared__ __align__(128) unsigned char smem_raw[];
#ifndef DTB_PIPE_MAP
#define DTB_PIPE_MAP 1
#endif
  // DTB_PIPE_MAP 1: warp = s * P + p, so SM sub-partition (warp % 4) p hosts all
  // S stages of pipeline p and a stage's slack goes to its own upstream/downstream
  // warps; 0: warp = p * S + s (all stage-0 warps share one sub-partition)
  const int warp = threadIdx.x >> 5;
  const int p = DTB_PIPE_MAP ? warp % P : warp / S, s = DTB_PIPE_MAP ? warp / P : warp % S;
  PipeSmem<S>* ctl = reinterpret_cast<PipeSmem<S>*>(smem_raw + P * kPipeBytes);
  if (threadIdx.x < P * S) {
    ctl[threadIdx.x / S].prod[threadIdx.x % S] = 0;
    ctl[threadIdx.x / S].cons[threadIdx.x % S] = 0;
  }
  __syncthreads();
  const uint32_t pbase = (uint32_t)__cvta_generic_to_shared(smem_raw + p * kPipeBytes);
  // ring s (s >= 1) follows ring0
  const uint32_t ring_in = s == 0 ? pbase : pbase + (uint32_t)(kRing0Rows + (s - 1) * kRingRows) * RB;
  const uint32_t ring_out = pbase + (uint32_t)(kRing0Rows + s * kRingRows) * RB;
  const int levels = max(0, min(2, steps - 2 * s));
  LaneCtx lc;
  lc.lane = threadIdx.x & 31;
  lc.first = lc.lane == 0;
  const int ntiles = geo.ntx * geo.nty;
  int seq = 0;
  for (int t = blockIdx.x * P + p; t < ntiles; t += gridDim.x * P) {
    const int tx = t % geo.ntx, ty = t / geo.ntx;
    const int4 cx = geo.col[tx], cy = geo.row[ty];
    PipeTile pt;
    pt.Lw = cx.w - cx.z;
    pt.Lh = cy.w - cy.z;
    pt.gx0 = cx.z + 1;
    pt.gy0 = cy.z + 1;
    pt.ox0 = cx.x - (cx.x == 0) - cx.z;
    pt.ox1 = cx.y + (cx.y == nx) - cx.z;
    pt.oy0 = cy.x - (cy.x == 0) - cy.z;
    pt.oy1 = cy.y + (cy.y == ny) - cy.z;
    pt.qy0 = pt.oy0;
    pt.qy1 = pt.oy1;
    if (MIR) {  // own stores only inside the window; the neighbours fill the rest
      pt.oy0 = max(pt.oy0, (int)(mir.sw0 - pt.gy0));
      pt.oy1 = min(pt.oy1, (int)(mir.sw1 - pt.gy0));
    }
    pt.vec = ((pt.gx0 % L::EPC) == 0) && ((pitch % L::EPC) == 0);
    lc.last = lc.lane == (pt.Lw - 1) / K;
    lc.last_e = (pt.Lw - 1) % K;
    pipe_stage<T, K, NW, DYN, MIR>(pt, s, S, levels, seq, src, dst, pitch, ring_in, ring_out,
                               ctl[p].prod, ctl[p].cons, wt, lc, &mir);
    seq += pt.Lh;
  }
}

// ---------------------------------------------------------------------------
// resident: persistent cooperative kernel, neighbour-flag halo exchange
// ---------------------------------------------------------------------------
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// G > 1: G independent tiles per CTA, NW warps each (own named barrier, own
// flags and epochs), stacked in shared memory; a tile's halo wait overlaps
// the other tiles' sweeps.
template <typename T, int K, int NW, bool DYN, int G = 1>
__global__ void __launch_bounds__(NW * 32 * G, 1)
resident_kernel(const T* __restrict__ in, T* __restrict__ out, T* __restrict__ xb0,
                T* __restrict__ xb1, int* __restrict__ flags, int64_t pitch, int nx, int ny,
                Weights<T> wt, int64_t total_steps, int h, int poison, int bs_on,
                unsigned long long* __restrict__ trace, const __grid_constant__ Geometry geo,
                int cl_on) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  constexpr int GT = G > 1 ? NW * 32 : 0;  // thread group = one tile
  const int group = G > 1 ? (int)(threadIdx.x / (NW * 32)) : 0;
  // tile (tx, ty); a CTA's G tiles are vertically adjacent (ty = G*cy + group)
  const int tx = blockIdx.x % geo.ntx, ty = G * (blockIdx.x / geo.ntx) + group;
  const int vcta = ty * geo.ntx + tx;
  int row_off = 0;  // rows of this CTA's earlier tiles in shared memory
  for (int g = 0; g < group; ++g) row_off += geo.row[ty - group + g].w - geo.row[ty - group + g].z;
  T* tile = reinterpret_cast<T*>(smem_raw) + (size_t)row_off * Tile<T, K>::ROW;
  const int4 cx = geo.col[tx], cy = geo.row[ty];
  const int Lw = cx.w - cx.z, Lh = cy.w - cy.z;
  const int gx0 = cx.z + 1, gy0 = cy.z + 1;  // padded coords of tile (0,0)
  const bool hl = cx.z > -1, hr = cx.w < nx + 1, ht = cy.z > -1, hb = cy.w < ny + 1;

  // band-sync counters (DTB_BANDSYNC) after all of the CTA's tiles
  int* bsmem = nullptr;
  int bseq = 0;
  if (bs_on) {
    int rows_all = 0;
    for (int g = 0; g < G; ++g) rows_all += geo.row[ty - group + g].w - geo.row[ty - group + g].z;
    bsmem = reinterpret_cast<int*>(smem_raw + (size_t)rows_all * Tile<T, K>::ROW * sizeof(T)) +
            group * 2 * NW;
    if (gt_tid<GT>() < 2 * NW) bsmem[gt_tid<GT>()] = 0;
  }
  g2s_rows<T, K, GT>(tile, in, pitch, gx0, gy0, 0, Lh, 0, Lw);
  cp_async_wait_all();
  gt_sync<GT>();

  // how deep each neighbour's load region reaches into my owned cells
  const int bl = tx > 0 ? max(0, geo.col[tx - 1].w - cx.x) : 0;
  const int br = tx + 1 < geo.ntx ? max(0, cx.y - geo.col[tx + 1].z) : 0;
  const int bt = ty > 0 ? max(0, geo.row[ty - 1].w - cy.x) : 0;
  const int bb = ty + 1 < geo.nty ? max(0, cy.y - geo.row[ty + 1].z) : 0;
  // owned rect in tile coordinates
  const int ox0 = cx.x - cx.z, ox1 = cx.y - cx.z, oy0 = cy.x - cy.z, oy1 = cy.y - cy.z;
  // halo ring cells to refresh exclude the frozen ghost ring of the domain
  const int rx0 = hl ? 0 : 1, rx1 = hr ? Lw : Lw - 1, ry0 = ht ? 0 : 1, ry1 = hb ? Lh : Lh - 1;

  // cluster partner (DTB_CLUSTER, launched as 2-CTA clusters along x): its tile
  // index, its smem tile in the cluster window, and the column offset from my
  // tile coordinates to its
  int ptx = -1, pdc = 0;
  uint32_t pbase = 0;
  if (DTB_CLUSTER && cl_on) {
    ptx = tx ^ 1;
    pbase = dsmem_map((uint32_t)__cvta_generic_to_shared(tile), (uint32_t)(tx & 1) ^ 1u);
    pdc = cx.z - geo.col[ptx].z;
  }
  int64_t done = 0;
  int epoch = 0;
  unsigned long long t_comp = 0, t_pub = 0, t_wait = 0, t_ref = 0, t_pst = 0, t_pbar = 0, tc = 0;
  const bool tracing = trace != nullptr && gt_tid<GT>() == 0;
  if (tracing) tc = clock64();
#define DTB_MARK(acc)                                  \
  if (tracing) {                                       \
    const unsigned long long now_ = clock64();         \
    acc += now_ - tc;                                  \
    tc = now_;                                         \
  }
  // per-lane publish masks over the lane's K columns (tile coordinates)
  Publisher<T, K> pub;
  pub.pitch = pitch;
  pub.own0 = oy0;
  pub.own1 = oy1;
  pub.top1 = oy0 + bt;
  pub.bot0 = oy1 - bb;
  pub.full_mask = 0;
  pub.side_mask = 0;
  pub.flag = flags + vcta;
  pub.cl0 = ox0;
  pub.wl = bl;
  pub.cr0 = max(ox1 - br, ox0 + bl);
  pub.wr = ox1 - pub.cr0;
  // flag value that marks "epoch e published": e (CTA-level release) or
  // e * warps (mode 3: one release-add per warp)
  const int flag_per_epoch =
      ((DTB_PUBREG == 3 || DTB_PUBREG == 4 || DTB_PUBREG == 6) && !poison) ? NW : 1;
  {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int e = 0; e < K; ++e) {
      const int c = lane * K + e;
      if (c >= ox0 && c < ox1) {
        pub.full_mask |= 1u << e;
        if (c < ox0 + bl || c >= ox1 - br) pub.side_mask |= 1u << e;
      }
    }
  }
  while (true) {
    const int steps = (int)((total_steps - done) < (int64_t)h ? (total_steps - done) : (int64_t)h);
    const bool last = done + steps >= total_steps;
    T* xb = ((epoch + 1) & 1) ? xb1 : xb0;
    pub.g0 = xb + (int64_t)gy0 * pitch + gx0;
    pub.g = pub.g0 + (threadIdx.x & 31) * K;
    // 1. compute the epoch; its final sweep publishes the owned band from registers
    advance<T, K, DYN, GT>(tile, Lw, Lh, steps, wt, poison != 0, hl, hr, ht, hb,
                           (last || poison || !DTB_PUBREG) ? nullptr : &pub, bsmem, &bseq);
    done += steps;
    DTB_MARK(t_comp)
    if (last) break;
    ++epoch;
    if (!poison && DTB_PUBREG == 0) {
      const int t1 = min(oy0 + bt, oy1), b0 = max(oy1 - bb, t1);
      publish_band<T, K, GT>(tile, xb, pitch, gx0, gy0, oy0, t1, b0, oy1, ox0, ox0 + bl,
                         max(ox1 - br, ox0 + bl), ox1);
    } else if (poison) {
      // poison mode publishes through smem (its sweeps run one step at a time)
      RectList<4> band;  // owned cells the neighbours' halos cover
      band.set(0, oy0, oy0 + bt, ox0, ox1);
      band.set(1, max(oy1 - bb, oy0 + bt), oy1, ox0, ox1);
      band.set(2, oy0 + bt, oy1 - bb, ox0, ox0 + bl);
      band.set(3, oy0 + bt, oy1 - bb, max(ox1 - br, ox0 + bl), ox1);
      s2g<T, K, 4, GT>(tile, xb, pitch, gx0, gy0, band);
    } else if (DTB_PUBREG == 1) {
      // side columns of the owned rows between the top/bottom bands
      publish_sides<T, K, GT>(tile, xb, pitch, gx0, gy0, oy0 + bt, oy1 - bb, ox0, ox0 + bl,
                          max(ox1 - br, ox0 + bl), ox1);
    }
#ifndef DTB_SKIPBAR
#define DTB_SKIPBAR 0  // 1: skip the post-publish CTA barrier in per-warp release modes (f64 +0.5 %, f32 -4 %)
#endif
#ifndef DTB_FENCE
#define DTB_FENCE 0  // 0: thread 0 st.release after the barrier; 1: every thread fences first;
                     // 9: no fence (timing experiments only - unsynchronised)
#endif
    DTB_MARK(t_pst)
    if (DTB_FENCE == 1) __threadfence();
    // per-warp release modes need no CTA barrier here: advance() closed with one
    if (flag_per_epoch == 1 || DTB_SKIPBAR == 0) gt_sync<GT>();
    DTB_MARK(t_pbar)
    if (gt_tid<GT>() == 0 && flag_per_epoch == 1) {
      if (DTB_FENCE == 9) *(volatile int*)(flags + vcta) = epoch;
      else st_release(flags + vcta, epoch);
    }
    DTB_MARK(t_pub)
    if (DTB_RING == 2) {
      // 2+3. per-direction: warp k waits for the neighbour owning halo region k
      // and immediately streams that region in (overlaps the 8 waits and loads)
      DTB_MARK(t_wait)
      unsigned long long t_poll = tc;
      if (DTB_CLUSTER && cl_on) cluster_arrive();  // my sweeps are done (partner may read)
      refresh_by_direction<T, K, GT>(tile, xb, pitch, gx0, gy0, flags, epoch * flag_per_epoch,
                                 geo.ntx, geo.nty, tx, ty, ry0, oy0, oy1, ry1, rx0, ox0, ox1,
                                 rx1, tracing ? &t_poll : nullptr, ptx, pbase, pdc);
      if (tracing) {
        const unsigned long long now_ = clock64();
        t_wait += t_poll - tc;   // warp 0: until its first neighbour flag arrived
        t_pst += now_ - t_poll;  // warp 0: its loads
        tc = now_;
      }
      if (DTB_CLUSTER && cl_on) cluster_wait();  // P2: the partner has read my seam columns
      gt_sync<GT>();
    } else {
    // 2. wait for the (up to 8) neighbours of this epoch
    if (gt_tid<GT>() < 9 && gt_tid<GT>() != 4) {
      const int dx = gt_tid<GT>() % 3 - 1, dy = gt_tid<GT>() / 3 - 1;
      const int nxt = tx + dx, nyt = ty + dy;
      if (nxt >= 0 && nxt < geo.ntx && nyt >= 0 && nyt < geo.nty) {
        const int* f = flags + nyt * geo.ntx + nxt;
        while (ld_acquire(f) < epoch * flag_per_epoch) __nanosleep(32);
      }
    }
    gt_sync<GT>();
    DTB_MARK(t_wait)
    // 3. refresh the halo ring (load region minus owned, domain ghost excluded)
    if (DTB_RING) {
      refresh_ring<T, K, GT>(tile, xb, pitch, gx0, gy0, ry0, oy0, oy1, ry1, rx0, ox0, ox1, rx1);
    } else {
      RectList<4> ring;
      ring.set(0, ry0, oy0, rx0, rx1);
      ring.set(1, oy1, ry1, rx0, rx1);
      ring.set(2, oy0, oy1, rx0, ox0);
      ring.set(3, oy0, oy1, ox1, rx1);
      g2s<T, K, 4, GT>(tile, xb, pitch, gx0, gy0, ring);
    }
    gt_sync<GT>();
    }
    DTB_MARK(t_ref)
  }
#undef DTB_MARK
  if (tracing) {
    unsigned long long* tr = trace + 8 * vcta;
    tr[0] = t_comp; tr[1] = t_pub; tr[2] = t_wait; tr[3] = t_ref; tr[4] = epoch;
    tr[5] = t_pst; tr[6] = t_pbar;
  }
  s2g_rows<T, K, GT>(tile, out, pitch, gx0, gy0, oy0 - !ht, oy1 + !hb, ox0 - !hl, ox1 + !hr);
}

// ---------------------------------------------------------------------------
// naive: one step, global memory (the T=1 HBM baseline)
// ---------------------------------------------------------------------------
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

// ---------------------------------------------------------------------------
// splitmix64 fill (prng.py:45-67): interior (x, y) = value i = y*nx + x
// ---------------------------------------------------------------------------
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

}  // namespace dtb

// ===========================================================================
// host runtime + C ABI
// ===========================================================================
namespace {

using namespace dtb;

thread_local std::string g_err;
thread_local int64_t g_launches = 0;
// set by solve_host_slabs around one slab's solve: the pipe kernel's final
// pass then feeds the neighbour slabs' halos in-kernel (HaloMirror)
thread_local const void* g_halo_mirror = nullptr;
thread_local std::vector<int64_t> g_trace;
thread_local unsigned g_flags = 0;

int fail(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CUDA_TRY(expr)                                                                   \
  do {                                                                                   \
    cudaError_t e_ = (expr);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return fail(DTB_ECUDA, "CUDA error %s (%s) at %s:%d", cudaGetErrorName(e_),        \
                  cudaGetErrorString(e_), __FILE__, __LINE__);                           \
  } while (0)

// Per-device scratch, grown on demand and kept (the solve is externally
// synchronous, so one arena per device suffices).
struct Arena {
  void* p = nullptr;
  size_t n = 0;
};
std::mutex g_mu;
Arena g_scratch[16];
Arena g_io[16];
Arena g_stage[16];  // aligned staging copies of misaligned grid origins (solve_dev)

int arena_get(Arena& a, size_t bytes, void** out) {
  if (a.n < bytes) {
    if (a.p) cudaFree(a.p);
    a.p = nullptr;
    a.n = 0;
    CUDA_TRY(cudaMalloc(&a.p, bytes));
    a.n = bytes;
  }
  *out = a.p;
  return DTB_OK;
}

// Per-call host work is on the critical path of short solves (C1: ~0.1 ms per
// solve), so device attributes, kernel smem attributes and occupancy are
// queried once per device / kernel and cached.
int query_dev_uncached(DevInfo& d, int dev);
int query_dev(DevInfo& d) {
  static std::mutex mu;
  static DevInfo cache[16];
  static bool have[16] = {};
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  if (!have[dev & 15]) {
    int rc = query_dev_uncached(cache[dev & 15], dev);
    if (rc) return rc;
    have[dev & 15] = true;
  }
  d = cache[dev & 15];
  return DTB_OK;
}

// cudaFuncSetAttribute(max dynamic smem) raised monotonically per (kernel,
// device) — a kernel's attribute is the max any call needed — and occupancy
// cached per (kernel, device, smem, threads)
int prepare_kernel(const void* kern, int device, int smem, int threads, int* per_sm) {
  struct A {
    const void* k;
    int dev, smem;
  };
  struct O {
    const void* k;
    int dev, smem, threads, per_sm;
  };
  static std::mutex mu;
  static std::vector<A> attrs;
  static std::vector<O> occ;
  std::lock_guard<std::mutex> lk(mu);
  A* a = nullptr;
  for (A& e : attrs)
    if (e.k == kern && e.dev == device) a = &e;
  if (!a || a->smem < smem) {
    CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    if (a) a->smem = smem;
    else attrs.push_back({kern, device, smem});
  }
  if (!per_sm) return DTB_OK;
  for (const O& e : occ)
    if (e.k == kern && e.dev == device && e.smem == smem && e.threads == threads) {
      *per_sm = e.per_sm;
      return DTB_OK;
    }
  int n = 0;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, threads, smem));
  occ.push_back({kern, device, smem, threads, n});
  *per_sm = n;
  return DTB_OK;
}

int query_dev_uncached(DevInfo& d, int dev) {
  int v = 0;
  CUDA_TRY(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev));
  d.sms = v;
  CUDA_TRY(cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  d.smem_optin = v;
  CUDA_TRY(cudaDeviceGetAttribute(&v, cudaDevAttrL2CacheSize, dev));
  d.l2_bytes = v;
  CUDA_TRY(cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev));
  d.smem_per_sm = v;
  return DTB_OK;
}

int fill_geometry(const Plan& p, Geometry& g) {
  if (p.sx.n > kMaxTiles || p.sy.n > kMaxTiles)
    return fail(DTB_EINFEASIBLE, "plan needs %d x %d tiles (max %d per dimension)", p.sx.n,
                p.sy.n, kMaxTiles);
  memset(&g, 0, sizeof g);
  g.ntx = p.sx.n;
  g.nty = p.sy.n;
  for (int i = 0; i < p.sx.n; ++i) g.col[i] = make_int4(p.sx.o0[i], p.sx.o1[i], p.sx.l0[i], p.sx.l1[i]);
  for (int j = 0; j < p.sy.n; ++j) g.row[j] = make_int4(p.sy.o0[j], p.sy.o1[j], p.sy.l0[j], p.sy.l1[j]);
  return DTB_OK;
}

template <typename T>
Weights<T> to_weights(const T w[5]) {
  Weights<T> k;
  k.w = w[0]; k.e = w[1]; k.s = w[2]; k.c = w[3]; k.n = w[4];
  k.nz = (T)-0.0;
  return k;
}

template <typename T, int K, int NW, bool DYN, int G = 1>
int launch_plan_kernels(const Plan& p, const Geometry& geo, const T* d_in, T* d_out,
                        int64_t pitch, int nx, int ny, const Weights<T>& wt,
                        int64_t steps, bool poison, cudaStream_t st) {
  const bool tracing = (g_flags & DTB_FLAG_TRACE) != 0;
  const int threads = NW * 32 * (p.mode == 0 ? G : 1);
  const int64_t tiles = (int64_t)p.ctas * (p.mode == 0 ? G : 1);
  const int smem = (int)p.smem_bytes;
  const int dev = 0;
  (void)dev;
  const size_t grid_bytes = (size_t)(ny + 2) * pitch * sizeof(T);
  int device;
  CUDA_TRY(cudaGetDevice(&device));
  if (p.mode == 0) {
    auto kern = resident_kernel<T, K, NW, DYN, G>;
    DevInfo di;
    if (int rc = query_dev(di)) return rc;
#ifndef DTB_BANDSYNC
#define DTB_BANDSYNC 0  // 1: band-to-band counters instead of CTA barriers inside an epoch (measured -1 %)
#endif
    // the band counters live after the tiles when the 1 KB of slack allows
    const int bs_bytes = 2 * NW * G * (int)sizeof(int);
    int bs_on = (DTB_BANDSYNC && !poison && smem + bs_bytes <= di.smem_optin) ? 1 : 0;
    const int smem_res = smem + (bs_on ? bs_bytes : 0);
    int per_sm = 0;
    if (int rc = prepare_kernel((const void*)kern, device, smem_res, threads, &per_sm)) return rc;
    const int sms = di.sms;
    if (per_sm < 1 || p.ctas > per_sm * sms)
      return fail(DTB_ECAPACITY, "resident plan needs %d co-resident CTAs, device holds %d",
                  p.ctas, per_sm * sms);
    void* scratch = nullptr;
    const size_t flag_bytes = 256 + (size_t)tiles * NW * sizeof(int);
    const size_t trace_bytes = (size_t)tiles * 8 * sizeof(unsigned long long);
    {
      std::lock_guard<std::mutex> lk(g_mu);
      int rc = arena_get(g_scratch[device & 15], 2 * grid_bytes + flag_bytes + trace_bytes + 256,
                         &scratch);
      if (rc) return rc;
    }
    T* xb0 = reinterpret_cast<T*>(scratch);
    T* xb1 = reinterpret_cast<T*>(reinterpret_cast<char*>(scratch) + grid_bytes);
    int* flags = reinterpret_cast<int*>(reinterpret_cast<char*>(scratch) + 2 * grid_bytes);
    CUDA_TRY(cudaMemsetAsync(flags, 0, (size_t)tiles * NW * sizeof(int), st));
    unsigned long long* trace = nullptr;
    if (tracing) {
      trace = reinterpret_cast<unsigned long long*>(
          reinterpret_cast<char*>(scratch) + ((2 * grid_bytes + flag_bytes + 255) & ~(size_t)255));
      CUDA_TRY(cudaMemsetAsync(trace, 0, trace_bytes, st));
    }
    int h = p.h;
    int pois = poison ? 1 : 0;
    int cl_on = 0;
    void* args[] = {(void*)&d_in, (void*)&d_out, (void*)&xb0, (void*)&xb1, (void*)&flags,
                    (void*)&pitch, (void*)&nx, (void*)&ny, (void*)&wt, (void*)&steps,
                    (void*)&h, (void*)&pois, (void*)&bs_on, (void*)&trace, (void*)&geo,
                    (void*)&cl_on};
    bool launched = false;
    if (DTB_CLUSTER && G == 1 && geo.ntx % 2 == 0 && p.ctas % 2 == 0 && !getenv("DTB_CLUSTER_OFF")) {
      // 2-CTA clusters along x, still a cooperative (co-resident) launch; if the
      // device cannot co-schedule them, fall back to the plain launch below
      cl_on = 1;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(p.ctas);
      cfg.blockDim = dim3(threads);
      cfg.dynamicSmemBytes = (size_t)smem_res;
      cfg.stream = st;
      cudaLaunchAttribute at[2];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 2;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      at[1].id = cudaLaunchAttributeCooperative;
      at[1].val.cooperative = 1;
      cfg.attrs = at;
      cfg.numAttrs = 2;
      int nclusters = 0;
      if (cudaOccupancyMaxActiveClusters(&nclusters, (const void*)kern, &cfg) == cudaSuccess &&
          nclusters * 2 >= p.ctas &&
          cudaLaunchKernelExC(&cfg, (const void*)kern, args) == cudaSuccess) {
        launched = true;
      } else {
        (void)cudaGetLastError();
        cl_on = 0;
      }
      if (getenv("DTB_CLUSTER_VERBOSE"))
        fprintf(stderr, "dtb: resident cluster launch %s (%d 2-CTA clusters co-resident, %d CTAs)\n",
                launched ? "used" : "not possible", nclusters, p.ctas);
    }
    if (!launched)
      CUDA_TRY(cudaLaunchCooperativeKernel((const void*)kern, dim3(p.ctas), dim3(threads), args,
                                           (size_t)smem_res, st));
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
  if (p.mode == 3) return DTB_EINFEASIBLE;  // handled by launch_pipe
  // streaming passes, ping-ponging dst between out and a scratch grid
  auto kern = stream_kernel<T, K, NW, DYN>;
  if (int rc = prepare_kernel((const void*)kern, device, smem * p.ctas_per_sm, threads, nullptr))
    return rc;
  const int64_t passes = (steps + p.h - 1) / p.h;
  T* tmp = nullptr;
  if (passes > 1) {
    void* scratch = nullptr;
    std::lock_guard<std::mutex> lk(g_mu);
    int rc = arena_get(g_scratch[device & 15], grid_bytes, &scratch);
    if (rc) return rc;
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
                                                       geo);
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

// pipelined streaming passes of h = 2S steps (mode 3), PW warps per CTA
template <typename T, int K, int PW, bool DYN>
int launch_pipe(const Plan& p, const Geometry& geo, const T* d_in, T* d_out, int64_t pitch,
                int nx, int ny, const Weights<T>& wt, int64_t steps, cudaStream_t st) {
#ifndef DTB_PIPE_STAGES
#define DTB_PIPE_STAGES 4
#endif
  constexpr int S = DTB_PIPE_STAGES, P = PW / S;
  auto kern = pipe_kernel<T, K, PW, S, DYN>;
  const int pipe_bytes = (PipeCfg<PW, T>::kRing0Rows + (S - 1) * PipeCfg<PW, T>::kRingRows) *
                         Tile<T, K>::ROW * (int)sizeof(T);
  const int psmem = P * pipe_bytes + (int)sizeof(PipeSmem<S>) * P;
  int device;
  CUDA_TRY(cudaGetDevice(&device));
  if (int rc = prepare_kernel((const void*)kern, device, psmem, PW * 32, nullptr)) return rc;
  const size_t grid_bytes = (size_t)(ny + 2) * pitch * sizeof(T);
  const int64_t passes = (steps + 2 * S - 1) / (2 * S);
  T* tmp = nullptr;
  if (passes > 1) {
    void* scratch = nullptr;
    std::lock_guard<std::mutex> lk(g_mu);
    int rc = arena_get(g_scratch[device & 15], grid_bytes, &scratch);
    if (rc) return rc;
    tmp = reinterpret_cast<T*>(scratch);
  }
  const int64_t ntiles = (int64_t)geo.ntx * geo.nty;
  DevInfo di;
  if (int rc = query_dev(di)) return rc;
  const int ctas = (int)std::min<int64_t>(di.sms, (ntiles + P - 1) / P);
  const HaloMirror<T>* mir = static_cast<const HaloMirror<T>*>(g_halo_mirror);
  HaloMirror<T> none;
  memset(&none, 0, sizeof none);
  if (mir) {
    auto kmir = pipe_kernel<T, K, PW, S, DYN, true>;
    if (int rc = prepare_kernel((const void*)kmir, device, psmem, PW * 32, nullptr)) return rc;
  }
  const T* src = d_in;
  int64_t done = 0;
  for (int64_t i = 0; i < passes; ++i) {
    const int s = (int)std::min<int64_t>(2 * S, steps - done);
    T* dst = ((passes - 1 - i) % 2 == 0) ? d_out : tmp;
    if (mir && i + 1 == passes)  // the epoch's result: also feed the neighbours' halos
      pipe_kernel<T, K, PW, S, DYN, true><<<ctas, PW * 32, psmem, st>>>(src, dst, pitch, nx, ny,
                                                                         wt, s, geo, *mir);
    else
      kern<<<ctas, PW * 32, psmem, st>>>(src, dst, pitch, nx, ny, wt, s, geo, none);
    g_launches += 1;
    CUDA_TRY(cudaGetLastError());
    src = dst;
    done += s;
  }
  return DTB_OK;
}

template <typename T, int K, int NW, int G = 1>
int dispatch_dyn(const Plan& p, const Geometry& geo, const T* d_in, T* d_out, int64_t pitch,
                 int nx, int ny, const Weights<T>& wt, int64_t steps, bool poison,
                 cudaStream_t st) {
  return p.dyn() ? launch_plan_kernels<T, K, NW, true, G>(p, geo, d_in, d_out, pitch, nx, ny, wt, steps, poison, st)
                 : launch_plan_kernels<T, K, NW, false, G>(p, geo, d_in, d_out, pitch, nx, ny, wt, steps, poison, st);
}

// kernel shapes compiled (must match the planner's candidates, dtb_plan.cpp)
template <typename T>
int dispatch(const Plan& p, const Geometry& geo, const T* d_in, T* d_out, int64_t pitch, int nx,
             int ny, const Weights<T>& wt, int64_t steps, bool poison, cudaStream_t st) {
  if (p.mode == 3) {
#ifndef DTB_PIPE_WARPS
#define DTB_PIPE_WARPS 16
#endif
    constexpr int KK = sizeof(T) == 8 ? 4 : 8;
    return p.dyn() ? launch_pipe<T, KK, DTB_PIPE_WARPS, true>(p, geo, d_in, d_out, pitch, nx, ny, wt, steps, st)
                   : launch_pipe<T, KK, DTB_PIPE_WARPS, false>(p, geo, d_in, d_out, pitch, nx, ny, wt, steps, st);
  }
  if (g_halo_mirror)
    return fail(DTB_EINVAL, "fused slab halos need the pipelined kernel (plan mode %d)", p.mode);
#define DTB_SHAPE(KK, WW)                                                                  \
  if (p.K == KK && p.warps == WW && p.groups == 1)                                         \
    return dispatch_dyn<T, KK, WW>(p, geo, d_in, d_out, pitch, nx, ny, wt, steps, poison, st);
  // two 4-warp tiles per CTA (resident only)
  if (p.mode == 0 && p.groups == 2 && p.warps == 4 && p.K == (sizeof(T) == 8 ? 4 : 8))
    return dispatch_dyn<T, sizeof(T) == 8 ? 4 : 8, 4, 2>(p, geo, d_in, d_out, pitch, nx, ny, wt,
                                                         steps, poison, st);
  if constexpr (sizeof(T) == 8) {
    DTB_SHAPE(4, 8)
#ifdef DTB_W12
    DTB_SHAPE(4, 12)
#endif
#ifdef DTB_W4
    DTB_SHAPE(4, 4)
#endif
#ifdef DTB_WIDE
    DTB_SHAPE(8, 8)
#endif
  } else {
    DTB_SHAPE(8, 8)
#ifdef DTB_WIDE
    DTB_SHAPE(16, 8)
#endif
  }
#undef DTB_SHAPE
  return fail(DTB_EINFEASIBLE, "no kernel instance for elem %d K %d warps %d", (int)sizeof(T),
              p.K, p.warps);
}

int validate(int64_t nx, int64_t ny, int64_t pitch, const double w[5], int64_t total_steps,
             int64_t t_depth, const dtb_rect* valid) {
  if (nx < 1 || ny < 1) return fail(DTB_EINVAL, "grid dims must be at least 1x1, got %lldx%lld", (long long)nx, (long long)ny);
  if (pitch < nx + 2) return fail(DTB_EINVAL, "pitch %lld smaller than nx+2 = %lld", (long long)pitch, (long long)(nx + 2));
  for (int i = 0; i < 5; ++i)
    if (!std::isfinite(w[i])) return fail(DTB_EINVAL, "non-finite stencil weight %c=%g", "wescn"[i], w[i]);
  if (t_depth < 1) return fail(DTB_EINVAL, "t_depth must be at least 1, got %lld", (long long)t_depth);
  if (total_steps < 1 || total_steps % t_depth)
    return fail(DTB_EINVAL, "total_steps %lld is not a positive multiple of t_depth %lld",
                (long long)total_steps, (long long)t_depth);
  if (valid) {
    if (valid->width < 0 || valid->height < 0)
      return fail(DTB_EINVAL, "negative rect dims: %lldx%lld", (long long)valid->width, (long long)valid->height);
    if (valid->width == 0 || valid->height == 0 || valid->x0 < 0 || valid->y0 < 0 ||
        valid->x0 + valid->width > nx || valid->y0 + valid->height > ny)
      return fail(DTB_EINVAL, "valid region (%lld, %lld, %lld, %lld) not within domain %lldx%lld",
                  (long long)valid->x0, (long long)valid->y0, (long long)valid->width,
                  (long long)valid->height, (long long)nx, (long long)ny);
  }
  return DTB_OK;
}

void fill_report(const Plan& p, int64_t nx, int64_t ny, int64_t steps, int elem, dtb_report* rep) {
  if (!rep) return;
  memset(rep, 0, sizeof *rep);
  rep->elem_bytes = elem;
  rep->useful_compute_cells = nx * ny * steps;
  if (p.mode == 2) {
    rep->global_load_cells = nx * ny * steps;
    rep->global_store_cells = nx * ny * steps;
    return;
  }
  const int64_t passes = (steps + p.h - 1) / p.h;
  int64_t load = 0, owned = nx * ny, halo_ring = 0;
  for (int i = 0; i < p.sx.n; ++i)
    for (int j = 0; j < p.sy.n; ++j) {
      const int64_t lw = p.sx.l1[i] - p.sx.l0[i], lh = p.sy.l1[j] - p.sy.l0[j];
      // domain cells of the load region (the ghost ring is not counted, metrics.py:3-6)
      const int64_t dw = std::min<int64_t>(p.sx.l1[i], nx) - std::max(p.sx.l0[i], 0);
      const int64_t dh = std::min<int64_t>(p.sy.l1[j], ny) - std::max(p.sy.l0[j], 0);
      load += dw * dh;
      halo_ring += dw * dh - (int64_t)(p.sx.o1[i] - p.sx.o0[i]) * (p.sy.o1[j] - p.sy.o0[j]);
      (void)lw; (void)lh;
    }
  if (p.mode == 0) {
    rep->global_load_cells = load + (passes - 1) * halo_ring;
    rep->global_store_cells = owned + (passes - 1) * halo_ring;
    rep->halo_exchanged_cells = (passes - 1) * halo_ring;
  } else {
    rep->global_load_cells = passes * load;
    rep->global_store_cells = passes * owned;
    rep->halo_exchanged_cells = 0;
  }
  rep->redundant_compute_cells = p.computed_cells_per_step * steps - nx * ny * steps;
  rep->scratchpad_peak_bytes = p.smem_bytes;
}

template <typename T>
int solve_dev(const T* d_in, T* d_out, int64_t nx, int64_t ny, int64_t pitch, const T w[5],
              int64_t total_steps, int64_t t_depth, const dtb_rect* valid, unsigned flags,
              cudaStream_t st, dtb_report* rep) {
  double wd[5];
  for (int i = 0; i < 5; ++i) wd[i] = (double)w[i];
  int rc = validate(nx, ny, pitch, wd, total_steps,
                    (flags & DTB_FLAG_FORCE_DEPTH) ? 1 : t_depth, valid);
  if (rc) return rc;
  if ((flags & DTB_FLAG_FORCE_DEPTH) && t_depth < 1)
    return fail(DTB_EINVAL, "forced depth must be at least 1, got %lld", (long long)t_depth);
  if (d_in == d_out) return fail(DTB_EINVAL, "input and output buffers alias");
  g_launches = 0;
  g_flags = flags;
  g_trace.clear();
  // valid-region runs: frozen cells outside `valid` are carried by a plain
  // copy, and the valid rectangle evolves as a standalone problem whose ghost
  // ring is the surrounding frozen cells (engine.py:26-30, grid.py:199-222).
  int64_t vx = 0, vy = 0, vnx = nx, vny = ny;
  if (valid && !(valid->x0 == 0 && valid->y0 == 0 && valid->width == nx && valid->height == ny)) {
    CUDA_TRY(cudaMemcpyAsync(d_out, d_in, (size_t)(ny + 2) * pitch * sizeof(T),
                             cudaMemcpyDeviceToDevice, st));
    vx = valid->x0; vy = valid->y0; vnx = valid->width; vny = valid->height;
  }
  const T* in_v = d_in + vy * pitch + vx;
  T* out_v = d_out + vy * pitch + vx;
  if ((reinterpret_cast<uintptr_t>(in_v) | reinterpret_cast<uintptr_t>(out_v)) & 15) {
    // the kernels move 16-byte chunks counted from the grid origin: solve a
    // misaligned origin (an odd-column valid window, an offset view) in an
    // aligned staging copy and copy the result back
    const int64_t spitch = (vnx + 2 + 31) / 32 * 32;
    const size_t sbytes = (size_t)(vny + 2) * spitch * sizeof(T), srow = (size_t)(vnx + 2) * sizeof(T);
    int device;
    CUDA_TRY(cudaGetDevice(&device));
    void* sp = nullptr;
    {
      std::lock_guard<std::mutex> lk(g_mu);
      if (int rc2 = arena_get(g_stage[device & 15], 2 * sbytes, &sp)) return rc2;
    }
    T* s_in = reinterpret_cast<T*>(sp);
    T* s_out = reinterpret_cast<T*>(reinterpret_cast<char*>(sp) + sbytes);
    CUDA_TRY(cudaMemcpy2DAsync(s_in, spitch * sizeof(T), in_v, pitch * sizeof(T), srow, vny + 2,
                               cudaMemcpyDeviceToDevice, st));
    if (int rc2 = solve_dev<T>(s_in, s_out, vnx, vny, spitch, w, total_steps, t_depth, nullptr,
                               flags, st, rep))
      return rc2;
    CUDA_TRY(cudaMemcpy2DAsync(out_v, pitch * sizeof(T), s_out, spitch * sizeof(T), srow, vny + 2,
                               cudaMemcpyDeviceToDevice, st));
    return DTB_OK;
  }
  DevInfo dev;
  rc = query_dev(dev);
  if (rc) return rc;
  int force = (flags & DTB_FLAG_FORCE_NAIVE) ? 2 : (flags & DTB_FLAG_FORCE_STREAM) ? 1
              : (flags & DTB_FLAG_FORCE_PIPE) ? 3 : (flags & DTB_FLAG_FORCE_RESIDENT) ? 4 : 0;
  int depth = (flags & DTB_FLAG_FORCE_DEPTH) ? (int)t_depth : 0;
  Plan p;
  char err[512];
  if (!make_plan(vnx, vny, (int)sizeof(T), total_steps, dev, force, depth, p, err, sizeof err))
    return fail(DTB_EINFEASIBLE, "%s", err);
  const Weights<T> wt = to_weights<T>(w);
  if (p.mode == 2) {
    // naive: total_steps launches ping-ponging between out and scratch
    const size_t grid_bytes = (size_t)(ny + 2) * pitch * sizeof(T);
    T* tmp = nullptr;
    if (total_steps > 1) {
      void* s = nullptr;
      int device;
      CUDA_TRY(cudaGetDevice(&device));
      std::lock_guard<std::mutex> lk(g_mu);
      rc = arena_get(g_scratch[device & 15], grid_bytes, &s);
      if (rc) return rc;
      tmp = reinterpret_cast<T*>(s);
      if (valid) CUDA_TRY(cudaMemcpyAsync(tmp, d_in, grid_bytes, cudaMemcpyDeviceToDevice, st));
    }
    T* tmp_v = tmp ? tmp + vy * pitch + vx : nullptr;
    const T* src = in_v;
    dim3 block(256), grid((unsigned)((vnx + 2 + 255) / 256), (unsigned)std::min<int64_t>(vny + 2, 65535));
    for (int64_t i = 0; i < total_steps; ++i) {
      T* dst = ((total_steps - 1 - i) % 2 == 0) ? out_v : tmp_v;
      naive_kernel<T><<<grid, block, 0, st>>>(src, dst, pitch, (int)vnx, (int)vny, wt);
      g_launches += 1;
      src = dst;
    }
    CUDA_TRY(cudaGetLastError());
  } else {
    Geometry geo;
    rc = fill_geometry(p, geo);
    if (rc) return rc;
    rc = dispatch<T>(p, geo, in_v, out_v, pitch, (int)vnx, (int)vny, wt, total_steps,
                     (flags & DTB_FLAG_POISON) != 0, st);
    if (rc) return rc;
  }
  fill_report(p, vnx, vny, total_steps, (int)sizeof(T), rep);
  return DTB_OK;
}

// ---------------------------------------------------------------------------
// n_gpus > 1 from the host entry: y-slabs (the native twin of
// slab.py). Slab g owns interior rows [y0, y1) and keeps a local padded grid
// of those rows plus kSlabDepth halo rows towards each neighbour (the global
// ghost row on the outer sides). Every epoch of s <= depth steps each slab
// advances its local grid s steps with its outer rows frozen (the trapezoid
// argument: owned rows stay exact), then receives depth rows from each
// neighbour into its halo by a device-to-device copy (P2P over NVLink when
// the slabs sit on different GPUs). Slabs go round-robin over the visible
// devices; slabs sharing a device run in order on that device's stream, so
// no kernel ever waits on another's. Bitwise equal to n_gpus = 1.
// ---------------------------------------------------------------------------
constexpr int kSlabDepth = 16;

struct DevBuffers {
  std::vector<std::pair<int, void*>> bufs;  // (device, pointer)
  std::vector<std::pair<int, cudaStream_t>> streams;
  std::vector<cudaEvent_t> events;
  int home = -1;  // the caller's device, restored on exit
  ~DevBuffers() {
    for (auto& s : streams) { cudaSetDevice(s.first); cudaStreamSynchronize(s.second); }
    for (auto& e : events) cudaEventDestroy(e);
    for (auto& s : streams) { cudaSetDevice(s.first); cudaStreamDestroy(s.second); }
    for (auto& b : bufs) { cudaSetDevice(b.first); cudaFree(b.second); }
    if (home >= 0) cudaSetDevice(home);
  }
};

template <typename T>
int solve_host_slabs(const T* in, T* out, int64_t nx, int64_t ny, int64_t pitch, const T w[5],
                     int64_t total_steps, unsigned flags, int n_slabs, dtb_report* rep) {
  if (ny < n_slabs)
    return fail(DTB_EINVAL, "%lld rows cannot be split over %d GPUs", (long long)ny, n_slabs);
  int ndev = 0, dev0 = 0;
  CUDA_TRY(cudaGetDeviceCount(&ndev));
  CUDA_TRY(cudaGetDevice(&dev0));
  if (ndev < 1) return fail(DTB_ECUDA, "no CUDA device");
  const int64_t base = ny / n_slabs, rem = ny % n_slabs;
  const int depth = (int)std::min<int64_t>(kSlabDepth, base);
  struct Slab { int dev; int64_t y0, own, ht, hb, lny, row0; T* a; T* b; };
  std::vector<Slab> sl(n_slabs);
  const int64_t dpitch = (nx + 2 + 31) / 32 * 32;
  const size_t hrow = (size_t)(nx + 2) * sizeof(T), drow = (size_t)dpitch * sizeof(T);
  DevBuffers res;
  res.home = dev0;
  std::vector<cudaStream_t> dstream(std::min(ndev, n_slabs));
  for (int d = 0; d < (int)dstream.size(); ++d) {
    CUDA_TRY(cudaSetDevice((dev0 + d) % ndev));
    CUDA_TRY(cudaStreamCreateWithFlags(&dstream[d], cudaStreamNonBlocking));
    res.streams.push_back({(dev0 + d) % ndev, dstream[d]});
    for (int e = 0; e < (int)dstream.size(); ++e)  // best effort: direct NVLink copies
      if (e != d && cudaDeviceEnablePeerAccess((dev0 + e) % ndev, 0) != cudaSuccess)
        cudaGetLastError();
  }
  int64_t y = 0;
  for (int g = 0; g < n_slabs; ++g) {
    Slab& s = sl[g];
    s.dev = g % (int)dstream.size();
    s.y0 = y;
    s.own = base + (g < rem ? 1 : 0);
    y += s.own;
    s.ht = g > 0 ? depth : 1;
    s.hb = g + 1 < n_slabs ? depth : 1;
    s.lny = s.own + s.ht + s.hb - 2;
    s.row0 = s.y0 + 1 - s.ht;  // padded global row of local row 0
    const size_t bytes = (size_t)(s.lny + 2) * drow;
    CUDA_TRY(cudaSetDevice((dev0 + s.dev) % ndev));
    void* p = nullptr;
    CUDA_TRY(cudaMalloc(&p, 2 * bytes));
    res.bufs.push_back({(dev0 + s.dev) % ndev, p});
    s.a = reinterpret_cast<T*>(p);
    s.b = reinterpret_cast<T*>(reinterpret_cast<char*>(p) + bytes);
    CUDA_TRY(cudaMemcpy2DAsync(s.a, drow, in + s.row0 * pitch, pitch * sizeof(T), hrow,
                               s.lny + 2, cudaMemcpyHostToDevice, dstream[s.dev]));
  }
  // exchange mode: fused (the pipe kernel's final pass of each epoch stores
  // the neighbours' halo rows straight into their next input, P2P when they
  // live on another GPU) whenever every slab runs the pipelined kernel; else
  // device-to-device copies after each epoch
  bool fused = (flags & DTB_FLAG_SLAB_COPY) == 0 && n_slabs > 1;
  for (int g = 0; g + 1 < n_slabs && fused; ++g) {  // in-kernel stores need peer access
    const int da = (dev0 + sl[g].dev) % ndev, db = (dev0 + sl[g + 1].dev) % ndev;
    int ab = 1, ba = 1;
    if (da != db) {
      CUDA_TRY(cudaDeviceCanAccessPeer(&ab, da, db));
      CUDA_TRY(cudaDeviceCanAccessPeer(&ba, db, da));
    }
    fused = ab && ba;
  }
  if (fused) {
    DevInfo di;
    if (int rc = query_dev(di)) return rc;
    const int force = (flags & DTB_FLAG_SLAB_FUSED) ? 3 : 0;
    for (int g = 0; g < n_slabs && fused; ++g) {
      Plan p;
      char err[256];
      fused = make_plan(nx, sl[g].lny, (int)sizeof(T), depth, di, force, 0, p, err, sizeof err) &&
              p.mode == 3;
    }
  }
  if ((flags & DTB_FLAG_SLAB_FUSED) && !fused)
    return fail(DTB_EINFEASIBLE, "fused slab halos need the pipelined kernel on every slab");
  std::vector<cudaEvent_t> solved(2 * n_slabs), copied(n_slabs);  // solved: epoch parity
  for (int g = 0; g < n_slabs; ++g) {
    CUDA_TRY(cudaSetDevice((dev0 + sl[g].dev) % ndev));
    for (int k = 0; k < 2; ++k) {
      CUDA_TRY(cudaEventCreateWithFlags(&solved[k * n_slabs + g], cudaEventDisableTiming));
      res.events.push_back(solved[k * n_slabs + g]);
    }
    CUDA_TRY(cudaEventCreateWithFlags(&copied[g], cudaEventDisableTiming));
    res.events.push_back(copied[g]);
  }
  struct MirrorScope {  // g_halo_mirror for exactly one slab solve
    explicit MirrorScope(const void* m) { g_halo_mirror = m; }
    ~MirrorScope() { g_halo_mirror = nullptr; }
  };
  dtb_report acc;
  memset(&acc, 0, sizeof acc);
  int64_t launches = 0, done = 0;
  int epoch = 0;
  const unsigned lflags = (flags & ~(unsigned)(DTB_FLAG_FORCE_DEPTH | DTB_FLAG_SLAB_COPY |
                                                DTB_FLAG_SLAB_FUSED)) |
                          (fused ? (unsigned)DTB_FLAG_FORCE_PIPE : 0u);
  std::vector<T*> next(n_slabs);
  while (done < total_steps) {
    const int64_t s_ep = std::min<int64_t>(depth, total_steps - done);
    const int cur = epoch & 1, prev = cur ^ 1;
    for (int g = 0; g < n_slabs; ++g) next[g] = sl[g].b;  // this epoch's outputs
    for (int g = 0; g < n_slabs; ++g) {
      Slab& s = sl[g];
      cudaStream_t st = dstream[s.dev];
      CUDA_TRY(cudaSetDevice((dev0 + s.dev) % ndev));
      if (epoch > 0) {
        if (fused) {
          // our halo rows in s.a came from the neighbours' previous epoch, and the
          // buffers we are about to write into were read by that epoch
          if (g > 0) CUDA_TRY(cudaStreamWaitEvent(st, solved[prev * n_slabs + g - 1], 0));
          if (g + 1 < n_slabs) CUDA_TRY(cudaStreamWaitEvent(st, solved[prev * n_slabs + g + 1], 0));
        } else {
          // the neighbours' last reads of our previous result buffer (their halo copies) are done
          if (g > 0) CUDA_TRY(cudaStreamWaitEvent(st, copied[g - 1], 0));
          if (g + 1 < n_slabs) CUDA_TRY(cudaStreamWaitEvent(st, copied[g + 1], 0));
        }
      }
      HaloMirror<T> m;
      memset(&m, 0, sizeof m);
      m.sw0 = g == 0 ? 0 : s.ht;
      m.sw1 = g + 1 == n_slabs ? s.lny + 2 : s.ht + s.own;
      if (g > 0) {  // our first owned rows -> the upper slab's bottom halo
        const Slab& u = sl[g - 1];
        m.peer[0] = next[g - 1];
        m.r0[0] = s.ht;
        m.r1[0] = s.ht + depth;
        m.p0[0] = u.ht + u.own;
      }
      if (g + 1 < n_slabs) {  // our last owned rows -> the lower slab's top halo
        m.peer[1] = next[g + 1];
        m.r0[1] = s.ht + s.own - depth;
        m.r1[1] = s.ht + s.own;
        m.p0[1] = 0;
      }
      dtb_report r;
      {
        MirrorScope scope(fused ? &m : nullptr);
        if (int rc = solve_dev<T>(s.a, s.b, nx, s.lny, dpitch, w, s_ep, 1, nullptr, lflags, st, &r))
          return rc;
      }
      launches += g_launches;
      acc.global_load_cells += r.global_load_cells;
      acc.global_store_cells += r.global_store_cells;
      acc.redundant_compute_cells += r.redundant_compute_cells + r.useful_compute_cells;
      acc.scratchpad_peak_bytes = std::max(acc.scratchpad_peak_bytes, r.scratchpad_peak_bytes);
      std::swap(s.a, s.b);
      CUDA_TRY(cudaEventRecord(solved[cur * n_slabs + g], st));
    }
    done += s_ep;
    ++epoch;
    if (done >= total_steps) break;
    if (fused) {
      acc.halo_exchanged_cells += 2 * (int64_t)(n_slabs - 1) * depth * nx;
      continue;
    }
    for (int g = 0; g < n_slabs; ++g) {  // halo rows from each neighbour's owned edge rows
      Slab& s = sl[g];
      cudaStream_t st = dstream[s.dev];
      CUDA_TRY(cudaSetDevice((dev0 + s.dev) % ndev));
      if (g > 0) {
        const Slab& u = sl[g - 1];
        CUDA_TRY(cudaStreamWaitEvent(st, solved[cur * n_slabs + g - 1], 0));
        CUDA_TRY(cudaMemcpy2DAsync(s.a, drow, u.a + (u.ht + u.own - depth) * dpitch, drow, hrow,
                                   depth, cudaMemcpyDefault, st));
        acc.halo_exchanged_cells += depth * nx;
      }
      if (g + 1 < n_slabs) {
        const Slab& d = sl[g + 1];
        CUDA_TRY(cudaStreamWaitEvent(st, solved[cur * n_slabs + g + 1], 0));
        CUDA_TRY(cudaMemcpy2DAsync(s.a + (s.ht + s.own) * dpitch, drow, d.a + d.ht * dpitch, drow,
                                   hrow, depth, cudaMemcpyDefault, st));
        acc.halo_exchanged_cells += depth * nx;
      }
      CUDA_TRY(cudaEventRecord(copied[g], st));
    }
  }
  for (int g = 0; g < n_slabs; ++g) {  // owned rows (and the global ghost rows) back
    const Slab& s = sl[g];
    CUDA_TRY(cudaSetDevice((dev0 + s.dev) % ndev));
    const int64_t r0 = g == 0 ? 0 : s.ht, r1 = s.ht + s.own + (g + 1 == n_slabs ? 1 : 0);
    CUDA_TRY(cudaMemcpy2DAsync(out + (s.row0 + r0) * pitch, pitch * sizeof(T), s.a + r0 * dpitch,
                               drow, hrow, r1 - r0, cudaMemcpyDeviceToHost, dstream[s.dev]));
  }
  for (int d = 0; d < (int)dstream.size(); ++d) {
    CUDA_TRY(cudaSetDevice((dev0 + d) % ndev));
    CUDA_TRY(cudaStreamSynchronize(dstream[d]));
  }
  g_launches = launches;
  if (rep) {
    *rep = acc;
    rep->elem_bytes = (int64_t)sizeof(T);
    rep->useful_compute_cells = nx * ny * total_steps;
    rep->redundant_compute_cells -= rep->useful_compute_cells;
  }
  return DTB_OK;
}

template <typename T>
int solve_host(const T* in, T* out, int64_t nx, int64_t ny, int64_t pitch, const T w[5],
               int64_t total_steps, int64_t t_depth, const dtb_rect* valid, int ilp, int n_gpus,
               unsigned flags, dtb_report* rep) {
  if (!in || !out) return fail(DTB_EINVAL, "null buffer");
  if (ilp < 1) return fail(DTB_EINVAL, "ilp must be at least 1, got %d", ilp);
  if (n_gpus < 1) return fail(DTB_EINVAL, "n_gpus must be at least 1, got %d", n_gpus);
  if (n_gpus > 1) {
    double wd[5];
    for (int i = 0; i < 5; ++i) wd[i] = (double)w[i];
    if (int rc = validate(nx, ny, pitch, wd, total_steps,
                          (flags & DTB_FLAG_FORCE_DEPTH) ? 1 : t_depth, valid))
      return rc;
    g_err.clear();
    if (valid && !(valid->x0 == 0 && valid->y0 == 0 && valid->width == nx && valid->height == ny)) {
      // cells outside `valid` are frozen: copy them, then slab-solve the valid
      // rectangle with its surrounding ring as ghost (engine.py:26-30, grid.py:199-222)
      for (int64_t r = 0; r < ny + 2; ++r)
        memcpy(out + r * pitch, in + r * pitch, (size_t)(nx + 2) * sizeof(T));
      const int64_t off = valid->y0 * pitch + valid->x0;
      return solve_host_slabs<T>(in + off, out + off, valid->width, valid->height, pitch, w,
                                 total_steps, flags, n_gpus, rep);
    }
    return solve_host_slabs<T>(in, out, nx, ny, pitch, w, total_steps, flags, n_gpus, rep);
  }
  double wd[5];
  for (int i = 0; i < 5; ++i) wd[i] = (double)w[i];
  int rc = validate(nx, ny, pitch, wd, total_steps,
                    (flags & DTB_FLAG_FORCE_DEPTH) ? 1 : t_depth, valid);
  if (rc) return rc;
  int device;
  CUDA_TRY(cudaGetDevice(&device));
  // device copy with a 128-byte-multiple pitch: 16-byte aligned tile copies
  const int64_t dpitch = (nx + 2 + 31) / 32 * 32;
  const size_t bytes = (size_t)(ny + 2) * dpitch * sizeof(T);
  void* io = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    rc = arena_get(g_io[device & 15], 2 * bytes, &io);
    if (rc) return rc;
  }
  T* d_in = reinterpret_cast<T*>(io);
  T* d_out = reinterpret_cast<T*>(reinterpret_cast<char*>(io) + bytes);
  cudaStream_t st = 0;
  const size_t row = (size_t)(nx + 2) * sizeof(T);
  CUDA_TRY(cudaMemcpy2DAsync(d_in, dpitch * sizeof(T), in, pitch * sizeof(T), row, ny + 2,
                             cudaMemcpyHostToDevice, st));
  rc = solve_dev<T>(d_in, d_out, nx, ny, dpitch, w, total_steps, t_depth, valid, flags, st, rep);
  if (rc) return rc;
  CUDA_TRY(cudaMemcpy2DAsync(out, pitch * sizeof(T), d_out, dpitch * sizeof(T), row, ny + 2,
                             cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return DTB_OK;
}

}  // namespace

extern "C" {

int dtb_j2d5pt_f64(const double* in, double* out, int64_t nx, int64_t ny, int64_t pitch,
                   const double w[5], int64_t total_steps, int64_t t_depth,
                   const dtb_rect* valid, int ilp, int n_gpus, unsigned flags,
                   dtb_report* rep) {
  g_err.clear();
  return solve_host<double>(in, out, nx, ny, pitch, w, total_steps, t_depth, valid, ilp, n_gpus,
                            flags, rep);
}

int dtb_j2d5pt_f32(const float* in, float* out, int64_t nx, int64_t ny, int64_t pitch,
                   const float w[5], int64_t total_steps, int64_t t_depth,
                   const dtb_rect* valid, int ilp, int n_gpus, unsigned flags,
                   dtb_report* rep) {
  g_err.clear();
  return solve_host<float>(in, out, nx, ny, pitch, w, total_steps, t_depth, valid, ilp, n_gpus,
                           flags, rep);
}

int dtb_j2d5pt_f64_dev(const double* d_in, double* d_out, int64_t nx, int64_t ny,
                       int64_t pitch, const double w[5], int64_t total_steps,
                       int64_t t_depth, const dtb_rect* valid, unsigned flags,
                       void* stream, dtb_report* rep) {
  g_err.clear();
  return solve_dev<double>(d_in, d_out, nx, ny, pitch, w, total_steps, t_depth, valid, flags,
                           (cudaStream_t)stream, rep);
}

int dtb_j2d5pt_f32_dev(const float* d_in, float* d_out, int64_t nx, int64_t ny,
                       int64_t pitch, const float w[5], int64_t total_steps,
                       int64_t t_depth, const dtb_rect* valid, unsigned flags,
                       void* stream, dtb_report* rep) {
  g_err.clear();
  return solve_dev<float>(d_in, d_out, nx, ny, pitch, w, total_steps, t_depth, valid, flags,
                          (cudaStream_t)stream, rep);
}

int dtb_plan(int64_t nx, int64_t ny, int32_t elem_bytes, int64_t total_steps, int64_t t_depth,
             unsigned flags, dtb_plan_info* out) {
  g_err.clear();
  if (!out) return fail(DTB_EINVAL, "null plan output");
  if (elem_bytes != 4 && elem_bytes != 8) return fail(DTB_EINVAL, "elem_bytes must be 4 or 8, got %d", elem_bytes);
  DevInfo dev;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) == cudaSuccess && ndev > 0) {
    int rc = query_dev(dev);
    if (rc) return rc;
  } else {
    cudaGetLastError();  // no GPU: plan for the B200 defaults (148 SMs, 227 KB)
  }
  int force = (flags & DTB_FLAG_FORCE_NAIVE) ? 2 : (flags & DTB_FLAG_FORCE_STREAM) ? 1
              : (flags & DTB_FLAG_FORCE_PIPE) ? 3 : (flags & DTB_FLAG_FORCE_RESIDENT) ? 4 : 0;
  int depth = (flags & DTB_FLAG_FORCE_DEPTH) ? (int)t_depth : 0;
  Plan p;
  char err[512];
  if (!make_plan(nx, ny, elem_bytes, total_steps, dev, force, depth, p, err, sizeof err))
    return fail(DTB_EINFEASIBLE, "%s", err);
  memset(out, 0, sizeof *out);
  out->mode = p.mode;
  out->elem_bytes = elem_bytes;
  out->lane_elems = p.K;
  out->warps = p.warps;
  out->halo = p.h;
  out->tiles_x = p.sx.n;
  out->tiles_y = p.sy.n;
  out->ctas = p.ctas;
  out->ctas_per_sm = p.ctas_per_sm;
  out->dyn = p.dyn() ? 1 : 0;
  out->smem_bytes = p.smem_bytes;
  for (int i = 0; i < p.sx.n; ++i) {
    out->tile_w = std::max<int64_t>(out->tile_w, p.sx.o1[i] - p.sx.o0[i]);
    out->load_w = std::max<int64_t>(out->load_w, p.sx.l1[i] - p.sx.l0[i]);
  }
  for (int j = 0; j < p.sy.n; ++j) {
    out->tile_h = std::max<int64_t>(out->tile_h, p.sy.o1[j] - p.sy.o0[j]);
    out->load_h = std::max<int64_t>(out->load_h, p.sy.l1[j] - p.sy.l0[j]);
  }
  out->computed_cells_per_step = p.computed_cells_per_step;
  out->est_cells_per_clk = p.cells_per_clk;
  return DTB_OK;
}

int64_t dtb_last_launch_count(void) { return g_launches; }

// debug builds (DTB_PIPE_PROBE): per pipe stage {wait_in, wait_out, total} SM cycles,
// summed over warps since the last call; resets the counters
extern "C" int dtb_debug_pipe_probe(uint64_t* out) {
#if DTB_PIPE_PROBE
  unsigned long long h[8][3];
  if (cudaMemcpyFromSymbol(h, dtb::g_pipe_probe, sizeof h) != cudaSuccess) return DTB_ECUDA;
  for (int i = 0; i < 24; ++i) out[i] = (&h[0][0])[i];
  unsigned long long z[8][3] = {};
  if (cudaMemcpyToSymbol(dtb::g_pipe_probe, z, sizeof z) != cudaSuccess) return DTB_ECUDA;
  return DTB_OK;
#else
  (void)out;
  return DTB_EINVAL;
#endif
}

int64_t dtb_last_trace(int64_t* out, int64_t n) {
  const int64_t m = std::min<int64_t>(n, (int64_t)g_trace.size());
  for (int64_t i = 0; i < m && out; ++i) out[i] = g_trace[(size_t)i];
  return (int64_t)g_trace.size() / 8;
}

int dtb_device_info(int32_t* sms, int64_t* smem_optin_per_block, int64_t* l2_bytes,
                    int32_t* cc_major, int32_t* cc_minor) {
  g_err.clear();
  DevInfo d;
  int rc = query_dev(d);
  if (rc) return rc;
  int dev = 0, maj = 0, mnr = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  CUDA_TRY(cudaDeviceGetAttribute(&maj, cudaDevAttrComputeCapabilityMajor, dev));
  CUDA_TRY(cudaDeviceGetAttribute(&mnr, cudaDevAttrComputeCapabilityMinor, dev));
  if (sms) *sms = d.sms;
  if (smem_optin_per_block) *smem_optin_per_block = d.smem_optin;
  if (l2_bytes) *l2_bytes = d.l2_bytes;
  if (cc_major) *cc_major = maj;
  if (cc_minor) *cc_minor = mnr;
  return DTB_OK;
}

int dtb_fill_random_f64(double* d_out, int64_t nx, int64_t ny, int64_t pitch, uint64_t seed,
                        double ghost, void* stream) {
  g_err.clear();
  if (nx < 1 || ny < 1 || pitch < nx + 2) return fail(DTB_EINVAL, "bad fill dims");
  fill_random_kernel<double><<<1184, 256, 0, (cudaStream_t)stream>>>(d_out, pitch, (int)nx, (int)ny, seed, ghost, 0, ny + 2);
  CUDA_TRY(cudaGetLastError());
  return DTB_OK;
}

int dtb_fill_random_f32(float* d_out, int64_t nx, int64_t ny, int64_t pitch, uint64_t seed,
                        double ghost, void* stream) {
  g_err.clear();
  if (nx < 1 || ny < 1 || pitch < nx + 2) return fail(DTB_EINVAL, "bad fill dims");
  fill_random_kernel<float><<<1184, 256, 0, (cudaStream_t)stream>>>(d_out, pitch, (int)nx, (int)ny, seed, ghost, 0, ny + 2);
  CUDA_TRY(cudaGetLastError());
  return DTB_OK;
}

int dtb_fill_random_rows_f64(double* d_out, int64_t nx, int64_t ny, int64_t pitch, uint64_t seed,
                             double ghost, int64_t row0, int64_t nrows, void* stream) {
  g_err.clear();
  if (nx < 1 || ny < 1 || pitch < nx + 2 || row0 < 0 || nrows < 0 || row0 + nrows > ny + 2)
    return fail(DTB_EINVAL, "bad fill rows");
  fill_random_kernel<double><<<1184, 256, 0, (cudaStream_t)stream>>>(d_out, pitch, (int)nx, (int)ny,
                                                                    seed, ghost, row0, nrows);
  CUDA_TRY(cudaGetLastError());
  return DTB_OK;
}

const char* dtb_last_error(void) { return g_err.c_str(); }

}  // extern "C"
