// dtb_tile_io.cuh — global <-> shared tile movement for the resident and
// tile-streaming kernels: whole-tile loads/stores, the resident halo refresh
// (per-neighbour epoch flags), and the NaN-poison debug mode.
#pragma once
#include "dtb_core.cuh"

namespace dtb {

__device__ __forceinline__ void cp_async(uint32_t dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async(uint32_t dst, const float* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// number of [a, b) that lie in [lo, hi) (counting domain cells of copies)
__device__ __forceinline__ long long span_in(long long a, long long b, long long lo, long long hi) {
  return max(0LL, min(b, hi) - max(a, lo));
}

__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int ld_relaxed_gpu(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Whole-rectangle tile copies, one warp per row, one 16-byte smem chunk per
// lane-iteration: tile rows [r0, r1) x cols [c0, c1) <-> global padded
// (gy0 + r, gx0 + c). When the global side is 16-byte aligned chunk-for-chunk
// (gx0 and pitch multiples of the chunk), whole chunks move as one 16-byte
// cp.async / STG; otherwise element by element. Loads are cp.async (the
// caller waits and synchronises).
template <typename T, int K>
__device__ __forceinline__ void g2s_rows(T* tile, const T* __restrict__ g, int64_t pitch, int gx0,
                                         int gy0, int r0, int r1, int c0, int c1) {
  typedef Tile<T, K> L;
  constexpr int E = L::EPC;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(tile);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
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

template <typename T, int K>
__device__ __forceinline__ void s2g_rows(const T* tile, T* __restrict__ g, int64_t pitch, int gx0,
                                         int gy0, int r0, int r1, int c0, int c1) {
  typedef Tile<T, K> L;
  typedef typename Arith<T>::vec_t V;
  constexpr int E = L::EPC;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
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

// Resident halo refresh, flattened: the ring — the full-width rows above and
// below the owned block, then the W / E columns beside it, row by row — in
// 16-byte chunks, split into NW equal contiguous shares, one per warp, after
// warp 0 has seen every neighbour's epoch flag (lanes 0..7 poll one each,
// acquire; a CTA barrier passes it on). Used for fp32 tiles (dtb_resident.cuh):
// the per-direction split (one warp per neighbour) leaves the W / E warps
// with ~30x the corner warps' chunks there (C3a 8 % slower); per-warp waits
// for only the neighbours of the warp's share measured 1.7 % slower than
// this barrier. `mark` (tracing): [0] flags seen, [1] warp 0's copy landed.
template <typename T, int K>
__device__ __forceinline__ void refresh_flat(T* tile, const T* __restrict__ g, int64_t pitch,
                                             int gx0, int gy0, const int* flags, int epoch,
                                             int ntx, int nty, int tx, int ty, int ry0, int oy0,
                                             int oy1, int ry1, int rx0, int ox0, int ox1, int rx1,
                                             unsigned long long* mark = nullptr,
                                             unsigned long long* cnt = nullptr) {
  typedef Tile<T, K> L;
  constexpr int E = L::EPC;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(tile);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  // whole 16-byte chunks move as one cp.async when the global rows are chunk-aligned
  const bool vec = ((gx0 % E) == 0) && ((pitch % E) == 0);
  // rects as scalars (a dynamically indexed array would land in local
  // memory, which the flag acquire's L1 invalidation evicts)
  const int qr = rx0 / E, nqr = rx1 > rx0 ? (rx1 + E - 1) / E - qr : 0;
  const int qw = rx0 / E, nqw = ox0 > rx0 ? (ox0 + E - 1) / E - qw : 0;
  const int qe = ox1 / E, nqe = rx1 > ox1 ? (rx1 + E - 1) / E - qe : 0;
  const int nt = max(0, oy0 - ry0) * nqr, nb = max(0, ry1 - oy1) * nqr;
  const int nm = max(0, oy1 - oy0);
  const int tot = nt + nb + nm * (nqw + nqe);
  const int i0 = (int)((int64_t)tot * warp / nw), i1 = (int)((int64_t)tot * (warp + 1) / nw);
  if (threadIdx.x < 8) {  // warp 0, one neighbour per lane: N S NW NE SW SE W E
    const int dx = lane == 0 || lane == 1 ? 0 : (lane == 2 || lane == 4 || lane == 6 ? -1 : 1);
    const int dy = lane == 6 || lane == 7 ? 0 : (lane == 0 || lane == 2 || lane == 3 ? -1 : 1);
    const bool rows = dy < 0 ? ry0 < oy0 : dy > 0 ? oy1 < ry1 : oy0 < oy1;
    const bool cols = dx < 0 ? rx0 < ox0 : dx > 0 ? ox1 < rx1 : ox0 < ox1;
    const int nxt = tx + dx, nyt = ty + dy;
    if (rows && cols && nxt >= 0 && nxt < ntx && nyt >= 0 && nyt < nty) {
      const int* f = flags + nyt * ntx + nxt;
      if (ld_acquire_gpu(f) < epoch) {
        // spin without the acquire's L1 invalidation, then acquire once
        while (ld_relaxed_gpu(f) < epoch) __nanosleep(32);
        (void)ld_acquire_gpu(f);
      }
    }
  }
  __syncthreads();  // every neighbour published (acquire by warp 0, barrier for the rest)
  if (mark) mark[0] = clock64();
  const uint64_t mr = nqr ? (0xFFFFFFFFull + (uint64_t)nqr) / (uint64_t)nqr : 0;
  const uint64_t mw = nqw + nqe ? (0xFFFFFFFFull + (uint64_t)(nqw + nqe)) / (uint64_t)(nqw + nqe) : 0;
  for (int i = i0 + lane; i < i1; i += 32) {
    int r, q, c0, c1;
    if (i < nt + nb) {  // a full-width row above or below the owned block
      const int j = i < nt ? i : i - nt;
      const uint32_t rr = (uint32_t)(((uint64_t)(uint32_t)j * mr) >> 32);
      r = (i < nt ? ry0 : oy1) + (int)rr;
      q = qr + j - (int)rr * nqr;
      c0 = rx0;
      c1 = rx1;
    } else {  // W then E chunks of one owned row
      const int j = i - nt - nb, w = nqw + nqe;
      const uint32_t rr = (uint32_t)(((uint64_t)(uint32_t)j * mw) >> 32);
      const int jj = j - (int)rr * w;
      r = oy0 + (int)rr;
      const bool west = jj < nqw;
      q = west ? qw + jj : qe + jj - nqw;
      c0 = west ? rx0 : ox1;
      c1 = west ? ox0 : rx1;
    }
    const int cb = q * E;
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
  if (cnt && threadIdx.x == 0) {  // refreshed halo cells: loads and exchanged cells
    const unsigned long long c =
        (unsigned long long)max(0, oy0 - ry0 + ry1 - oy1) * (unsigned long long)(rx1 - rx0) +
        (unsigned long long)max(0, oy1 - oy0) * (unsigned long long)(ox0 - rx0 + rx1 - ox1);
    atomicAdd(cnt + 0, c);
    atomicAdd(cnt + 2, c);
  }
  cp_async_wait_all();
  if (mark) mark[1] = clock64();
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

// Resident halo refresh, warp-specialised by direction: the ring is cut into
// 8 regions (N, S, the 4 corners, W, E), each owned by one neighbour; warp k
// polls that neighbour's epoch flag (acquire) and streams its region in with
// cp.async as soon as it is published, so the waits and loads of the eight
// directions overlap. `mark` (tracing): [0] when warp 0's first flag arrived.
// Chosen for fp64 (dtb_resident.cuh): C2 2 % faster than refresh_flat.
template <typename T, int K>
__device__ __forceinline__ void refresh_by_direction(T* tile, const T* __restrict__ g,
                                                     int64_t pitch, int gx0, int gy0,
                                                     const int* flags, int epoch, int ntx, int nty,
                                                     int tx, int ty, int ry0, int oy0, int oy1,
                                                     int ry1, int rx0, int ox0, int ox1, int rx1,
                                                     unsigned long long* mark = nullptr,
                                                     unsigned long long* cnt = nullptr) {
  typedef Tile<T, K> L;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(tile);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const bool vec = ((gx0 % L::EPC) == 0) && ((pitch % L::EPC) == 0);
  int polled = -1;  // neighbour this warp last waited for
  for (int k = warp; k < 8; k += nw) {
    int dx, dy, r0, r1, c0, c1;
    switch (k) {
      case 0: dx = 0; dy = -1; r0 = ry0; r1 = oy0; c0 = ox0; c1 = ox1; break;
      case 1: dx = 0; dy = 1; r0 = oy1; r1 = ry1; c0 = ox0; c1 = ox1; break;
      case 2: dx = -1; dy = -1; r0 = ry0; r1 = oy0; c0 = rx0; c1 = ox0; break;
      case 3: dx = 1; dy = -1; r0 = ry0; r1 = oy0; c0 = ox1; c1 = rx1; break;
      case 4: dx = -1; dy = 1; r0 = oy1; r1 = ry1; c0 = rx0; c1 = ox0; break;
      case 5: dx = 1; dy = 1; r0 = oy1; r1 = ry1; c0 = ox1; c1 = rx1; break;
      case 6: dx = -1; dy = 0; r0 = oy0; r1 = oy1; c0 = rx0; c1 = ox0; break;
      default: dx = 1; dy = 0; r0 = oy0; r1 = oy1; c0 = ox1; c1 = rx1; break;
    }
    const int nxt = tx + dx, nyt = ty + dy;
    if (r1 <= r0 || c1 <= c0 || nxt < 0 || nxt >= ntx || nyt < 0 || nyt >= nty) continue;
    const int nb = nyt * ntx + nxt;
    if (nb != polled) {
      if (lane == 0 && ld_acquire_gpu(flags + nb) < epoch) {
        while (ld_relaxed_gpu(flags + nb) < epoch) __nanosleep(32);
        (void)ld_acquire_gpu(flags + nb);
      }
      __syncwarp();
      if (mark && polled < 0) *mark = clock64();
      polled = nb;
    }
    warp_g2s_chunks<T, K>(sbase, g, pitch, gx0, gy0, r0, r1, c0, c1, vec, lane);
    if (cnt && lane == 0) {  // refreshed halo cells: loads and exchanged cells
      const unsigned long long n = (unsigned long long)(r1 - r0) * (unsigned long long)(c1 - c0);
      atomicAdd(cnt + 0, n);
      atomicAdd(cnt + 2, n);
    }
  }
  cp_async_wait_all();
}

// Poison (debug, DTB_FLAG_POISON): NaN every tile cell a correct schedule can
// no longer read after `done` steps of the epoch — the ring of width `done`
// along halo sides (the trapezoid rim, planner.py:272-286) plus the unused
// lane columns. A stale read anywhere then propagates NaN into the owned
// cells and fails the bitwise comparison (the reference's poison mode,
// engine.py:16-20,174-177). The domain's ghost ring is exempt: it is frozen
// and never refreshed, so a NaN there would be a stale value that a correct
// schedule keeps reading (where a halo side meets the domain edge).
template <typename T, int K>
__device__ void poison_rim(T* tile, int Lw, int Lh, int done, bool hl, bool hr, bool ht, bool hb) {
  typedef Tile<T, K> L;
  const T nanv = (T)NAN;
  for (int i = threadIdx.x; i < Lh * L::ROW; i += blockDim.x) {
    const int r = i / L::ROW, c = i % L::ROW;
    bool p = c >= Lw;
    p |= hl && c < done;
    p |= hr && c >= Lw - done;
    p |= ht && r < done;
    p |= hb && r >= Lh - done;
    const bool ghost = c < Lw && ((!ht && r == 0) || (!hb && r == Lh - 1) ||
                                  (!hl && c == 0) || (!hr && c == Lw - 1));
    if (p && !ghost) tile[L::at(r, c)] = nanv;
  }
}

// advance_tile, or in poison mode one step at a time with the stale rim
// NaN-ed after each step
template <typename T, int K, bool SYM, bool DYN>
__device__ void advance(T* tile, int Lw, int Lh, int steps, const Weights<T>& wt, bool poison,
                        bool hl, bool hr, bool ht, bool hb,
                        const Publisher<T, K>* pub = nullptr,
                        unsigned long long* cnt = nullptr, int owned_w = 0) {
  if (!poison) {
    advance_tile<T, K, SYM, DYN>(tile, Lw, Lh, steps, wt, pub, cnt, owned_w);
    return;
  }
  for (int s = 0; s < steps; ++s) {
    advance_tile<T, K, SYM, DYN>(tile, Lw, Lh, 1, wt, nullptr, cnt);
    poison_rim<T, K>(tile, Lw, Lh, s + 1, hl, hr, ht, hb);
    __syncthreads();
  }
}

}  // namespace dtb
