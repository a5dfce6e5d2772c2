// dtb_core.cuh — the shared-memory compute core of the B200 j2d5pt solver.
//
// One CTA owns a rectangular tile of the padded grid in shared memory (its
// "load region": owned cells dilated by the temporal halo, clipped to the
// domain plus its ghost ring). The tile's outermost row/column ring is the
// FROZEN FRAME: it is never written by a sweep. On domain edges that frame is
// the reference's frozen Dirichlet ghost ring (grid.py:1-12); on halo sides it
// is the outermost halo row, whose staleness eats one cell of the valid zone
// per step exactly like tile_active_region's trapezoid (planner.py:272-286).
//
// Every update is the reference's fixed-order, FMA-free expression
// (kernel.py:137-139):   ((((W*w + E*e) + S*s) + C*c) + N*n)
// with every product and sum separately rounded (__dmul_rn/__dadd_rn, built
// with -fmad=false), so every schedule below is bitwise equal to
// jacobi_reference (oracle.py:19-34).
//
// Streaming (running-sum) form. Rows flow through a "level" (one time step)
// in increasing y. When row x(r) arrives the level
//   * finishes row r-1:  out(r-1) = acc(r-1) + x(r)*n          (the N term)
//   * starts row r:      acc(r)   = ((x(r)[c-1]*w + x(r)[c+1]*e) + ps(r-1)) + x(r)*c
//   * keeps              ps(r)    = x(r)*s                      (row r+1's S term)
// Each product x*w, x*e, x*s, x*c, x*n is formed once, when its source row
// arrives, and each sum happens in exactly the reference's order — the same
// nine rounded operations per cell as kernel.py:137-139, in a different
// interleaving across cells, which cannot change any bit. A level carries two
// rows of state (ps, acc) instead of a 3-4 row window of raw values.
//
// Isotropic weights (SYM: w, e, s, n bitwise equal, e.g. the reference's
// StencilWeights.diffusive, grid.py:117-120): the four products x*w, x*e, x*s,
// x*n of one source cell are the same rounded number, so one multiply serves
// the cell's east neighbour (as its W term), its west neighbour (E term), the
// row below (S term) and the row above (N term): 2 products + 4 sums = 6
// rounded operations per cell update instead of 9, bit for bit the same.
//
// Layout (B200-first):
//  * a warp spans the whole tile width; lane l owns K consecutive columns
//    [l*K, l*K+K) in registers; smem rows have a fixed pitch of 32*K elements
//    and are moved as 16-byte chunks with an XOR chunk swizzle that makes
//    every LDS.128/STS.128 conflict-free;
//  * W/E neighbours across lanes come from 64-bit shuffles of the products;
//  * warps split the tile's rows into bands; a band sweep streams its rows
//    through TWO levels (t -> t+1 -> t+2), so each smem cell is read and
//    written once per two updates. Band seams are resolved by reading the two
//    foreign rows on each side BEFORE a CTA barrier and writing only owned
//    rows after it (in place, single buffer: smem holds exactly one copy of
//    the tile, which is what lets a 1900^2 fp64 grid live in 148 SMs' smem).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

// Steady rows per unrolled block of the band sweep, per element type (B200
// A/B on C2 / C3a: fp64 +1.8 % with 8-row blocks, fp32 -1 %)
#ifndef DTB_SWEEP_UNROLL
#define DTB_SWEEP_UNROLL(T) (sizeof(T) == 8 ? 8 : 4)
#endif

namespace dtb {

template <typename T> struct Arith;
template <> struct Arith<double> {
  typedef double2 vec_t;
  static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
  static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
};
template <> struct Arith<float> {
  typedef float4 vec_t;
  static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
  static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
};

template <typename T> struct Weights { T w, e, s, c, n; };

// The reference's update for one cell, kernel.py:137-139 / grid.py:95-116
// (used by the one-step-per-launch naive kernel).
template <typename T>
__device__ __forceinline__ T cell_update(T west, T east, T south, T center, T north,
                                         const Weights<T>& k) {
  typedef Arith<T> A;
  T acc = A::mul(west, k.w);
  acc = A::add(acc, A::mul(east, k.e));
  acc = A::add(acc, A::mul(south, k.s));
  acc = A::add(acc, A::mul(center, k.c));
  acc = A::add(acc, A::mul(north, k.n));
  return acc;
}

// Shared-memory tile of rows with pitch 32*K elements, 16-byte chunks
// XOR-swizzled within each 128-byte group.
template <typename T, int K>
struct Tile {
  static constexpr int EPC = 16 / (int)sizeof(T);  // elements per chunk
  static constexpr int CH = K / EPC;               // chunks per lane
  static constexpr int ROW = 32 * K;               // elements per row (pitch)
  static_assert(K % EPC == 0, "K must be a whole number of 16-byte chunks");
  static_assert(CH == 1 || CH == 2 || CH == 4 || CH == 8, "unsupported lane width");

  __device__ static __forceinline__ int swz(int c) { return c ^ ((c >> 3) & 7); }
  // physical element offset of tile cell (row r, column col)
  __device__ static __forceinline__ int at(int r, int col) {
    return r * ROW + swz(col / EPC) * EPC + (col % EPC);
  }
};

// Per-lane shared-memory addressing: 32-bit shared-window address of the
// tile plus this lane's (swizzled) chunk offsets, computed once per kernel so
// every row access in the sweeps is a single LDS/STS.128 at base + r*ROW + off.
template <typename T, int K>
struct LaneAddr {
  typedef Tile<T, K> L;
  uint32_t base;
  uint32_t off[L::CH];
  __device__ __forceinline__ LaneAddr(const T* tile, int lane) {
    base = (uint32_t)__cvta_generic_to_shared(tile);
#pragma unroll
    for (int j = 0; j < L::CH; ++j) off[j] = (uint32_t)(L::swz(lane * L::CH + j) * 16);
  }
  __device__ __forceinline__ uint32_t row(int r) const {
    return base + (uint32_t)r * (uint32_t)(L::ROW * sizeof(T));
  }
};

__device__ __forceinline__ void lds16(uint32_t a, double& x, double& y) {
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(a) : "memory");
}
__device__ __forceinline__ void lds16(uint32_t a, float& x, float& y, float& z, float& w) {
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(x), "=f"(y), "=f"(z), "=f"(w) : "r"(a) : "memory");
}
__device__ __forceinline__ void sts16(uint32_t a, double x, double y) {
  asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(x), "d"(y) : "memory");
}
__device__ __forceinline__ void sts16(uint32_t a, float x, float y, float z, float w) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(x), "f"(y), "f"(z),
               "f"(w) : "memory");
}

template <int CH>
__device__ __forceinline__ void load_row_at(uint32_t row, const uint32_t (&off)[CH], double (&v)[2 * CH]) {
#pragma unroll
  for (int j = 0; j < CH; ++j) lds16(row + off[j], v[2 * j], v[2 * j + 1]);
}
template <int CH>
__device__ __forceinline__ void load_row_at(uint32_t row, const uint32_t (&off)[CH], float (&v)[4 * CH]) {
#pragma unroll
  for (int j = 0; j < CH; ++j) lds16(row + off[j], v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
}
template <int CH>
__device__ __forceinline__ void store_row_at(uint32_t row, const uint32_t (&off)[CH], const double (&v)[2 * CH]) {
#pragma unroll
  for (int j = 0; j < CH; ++j) sts16(row + off[j], v[2 * j], v[2 * j + 1]);
}
template <int CH>
__device__ __forceinline__ void store_row_at(uint32_t row, const uint32_t (&off)[CH], const float (&v)[4 * CH]) {
#pragma unroll
  for (int j = 0; j < CH; ++j) sts16(row + off[j], v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
}

template <typename T, int K>
__device__ __forceinline__ void load_row(const LaneAddr<T, K>& la, int r, T (&v)[K]) {
  load_row_at<Tile<T, K>::CH>(la.row(r), la.off, v);
}
template <typename T, int K>
__device__ __forceinline__ void store_row(const LaneAddr<T, K>& la, int r, const T (&v)[K]) {
  store_row_at<Tile<T, K>::CH>(la.row(r), la.off, v);
}

template <typename T>
__device__ __forceinline__ T shfl_up1(T v) { return __shfl_up_sync(0xffffffffu, v, 1); }
template <typename T>
__device__ __forceinline__ T shfl_dn1(T v) { return __shfl_down_sync(0xffffffffu, v, 1); }
// fp64: the two 32-bit shuffles of one value in a single asm block, so the
// halves land in the register pair the DADD reads (the intrinsic left ptxas
// moving them: 11 fewer moves per 8 band rows, C2 +0.6 %, C4 +0.5 %)
template <>
__device__ __forceinline__ double shfl_up1<double>(double v) {
  double r;
  asm volatile("{ .reg .b32 lo, hi;\n mov.b64 {lo, hi}, %1;\n"
               " shfl.sync.up.b32 lo, lo, 1, 0, -1;\n shfl.sync.up.b32 hi, hi, 1, 0, -1;\n"
               " mov.b64 %0, {lo, hi}; }" : "=d"(r) : "d"(v));
  return r;
}
template <>
__device__ __forceinline__ double shfl_dn1<double>(double v) {
  double r;
  asm volatile("{ .reg .b32 lo, hi;\n mov.b64 {lo, hi}, %1;\n"
               " shfl.sync.down.b32 lo, lo, 1, 31, -1;\n shfl.sync.down.b32 hi, hi, 1, 31, -1;\n"
               " mov.b64 %0, {lo, hi}; }" : "=d"(r) : "d"(v));
  return r;
}

template <typename T, int K>
__device__ __forceinline__ void copy_row(const T (&a)[K], T (&b)[K]) {
#pragma unroll
  for (int e = 0; e < K; ++e) b[e] = a[e];
}

// Lane geometry of the frozen frame's columns: column 0 is lane 0 element 0,
// column Lw-1 is lane `last` element K-1 (the planner keeps Lw % K == 0).
// DYN: Lw % K != 0 (only when one tile spans the whole width), so the right
// frozen column sits at element last_e of its lane instead of element K-1.
struct LaneCtx {
  int lane;
  bool first;  // lane holds frozen column 0
  bool last;   // lane holds frozen column Lw-1
  int last_e;  // its element index (== K-1 unless DYN)
};

// ---------------------------------------------------------------------------
// One time level of the streaming form (see the header comment).
// ---------------------------------------------------------------------------
template <typename T, int K, bool SYM, bool DYN>
struct Level {
  T ps[K];             // previous row's S-term products x*s
  T acc[K];            // previous row's partial sums ((W + E) + S) + C
  T mid[DYN ? K : 2];  // previous row's raw values in the frozen columns
                       // (elements 0 and K-1; DYN: the whole row)

  __device__ __forceinline__ void keep_mid(const T (&x)[K]) {
    if (DYN) {
#pragma unroll
      for (int e = 0; e < K; ++e) mid[e] = x[e];
    } else {
      mid[0] = x[0];
      mid[DYN ? 0 : 1] = x[K - 1];
    }
  }
  // first row of the stream: no row above it is finished by it and its own
  // value cannot be finished (no S neighbour) — only its S products are kept
  __device__ __forceinline__ void start(const T (&x)[K], const Weights<T>& wt) {
#pragma unroll
    for (int e = 0; e < K; ++e) ps[e] = Arith<T>::mul(x[e], SYM ? wt.w : wt.s);
    keep_mid(x);
  }
  // Row x arrives. EMIT: finish the previous row into `out` (frozen columns
  // keep their value). ACC: start x's own partial sums (omit for the last row
  // of a stream: nothing below it will finish it).
  template <bool EMIT, bool ACC>
  __device__ __forceinline__ void push(const T (&x)[K], T (&out)[K], const Weights<T>& wt,
                                       const LaneCtx& lc) {
    typedef Arith<T> A;
    T pn[K];
#pragma unroll
    for (int e = 0; e < K; ++e) pn[e] = A::mul(x[e], SYM ? wt.w : wt.n);
    if (EMIT) {
#pragma unroll
      for (int e = 0; e < K; ++e) out[e] = A::add(acc[e], pn[e]);
      if (lc.first) out[0] = mid[0];
      if (DYN) {
        if (lc.last) {
#pragma unroll
          for (int e = 0; e < K; ++e)
            if (e == lc.last_e) out[e] = mid[e];
        }
      } else {
        if (lc.last) out[K - 1] = mid[DYN ? 0 : 1];
      }
    }
    if (ACC) {
      if constexpr (SYM) {
        const T west = shfl_up1(pn[K - 1]), east = shfl_dn1(pn[0]);
#pragma unroll
        for (int e = 0; e < K; ++e) {
          T a = A::add(e == 0 ? west : pn[e - 1], e == K - 1 ? east : pn[e + 1]);
          a = A::add(a, ps[e]);
          acc[e] = A::add(a, A::mul(x[e], wt.c));
        }
#pragma unroll
        for (int e = 0; e < K; ++e) ps[e] = pn[e];
      } else {
        T pw[K], pe[K];
#pragma unroll
        for (int e = 0; e < K; ++e) {
          pw[e] = A::mul(x[e], wt.w);
          pe[e] = A::mul(x[e], wt.e);
        }
        const T west = shfl_up1(pw[K - 1]), east = shfl_dn1(pe[0]);
#pragma unroll
        for (int e = 0; e < K; ++e) {
          T a = A::add(e == 0 ? west : pw[e - 1], e == K - 1 ? east : pe[e + 1]);
          a = A::add(a, ps[e]);
          acc[e] = A::add(a, A::mul(x[e], wt.c));
        }
#pragma unroll
        for (int e = 0; e < K; ++e) ps[e] = A::mul(x[e], wt.s);
      }
      keep_mid(x);
    }
  }
};

__device__ __forceinline__ int ld_acquire_cta(const int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared.s32 %0, [%1];"
               : "=r"(v)
               : "r"((uint32_t)__cvta_generic_to_shared(p))
               : "memory");
  return v;
}
__device__ __forceinline__ void st_release_cta(int* p, int v) {
  asm volatile("st.release.cta.shared.s32 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(p)),
               "r"(v)
               : "memory");
}

__device__ __forceinline__ void st_cg(double* a, double v) {
  asm volatile("st.global.cg.f64 [%0], %1;" ::"l"(a), "d"(v) : "memory");
}
__device__ __forceinline__ void st_cg(float* a, float v) {
  asm volatile("st.global.cg.f32 [%0], %1;" ::"l"(a), "f"(v) : "memory");
}
__device__ __forceinline__ void st_pred(bool p, double* a, double v) {
  asm volatile("{ .reg .pred q; setp.ne.u32 q, %0, 0; @q st.global.cg.f64 [%1], %2; }"
               ::"r"((unsigned)p), "l"(a), "d"(v) : "memory");
}
__device__ __forceinline__ void st_pred(bool p, float* a, float v) {
  asm volatile("{ .reg .pred q; setp.ne.u32 q, %0, 0; @q st.global.cg.f32 [%1], %2; }"
               ::"r"((unsigned)p), "l"(a), "f"(v) : "memory");
}

// Resident halo publisher: once a warp's band has finished the epoch's last
// sweep its rows are final (no other warp writes them), so the warp stores
// the cells of its band that the neighbours' halos cover straight into the
// L2 exchange buffer: whole owned rows of the top/bottom bands
// [own0, top1) / [bot0, own1) (K predicated stores per lane), and the side
// columns [cl0, cl0+wl) / [cr0, cr0+wr) of the rows in between flattened
// across lanes (one warp store covers 32 / (wl + wr) rows).
template <typename T, int K>
struct Publisher {
  T* g;             // exchange buffer at (tile row 0, this lane's first column)
  T* g0;            // exchange buffer at (tile row 0, tile column 0)
  int64_t pitch;
  int own0, own1, top1, bot0;
  uint32_t full_mask;     // this lane's owned columns (bit e = column lane*K + e)
  int cl0, wl, cr0, wr;
  int* flag;              // this CTA's epoch flag (one release-add per warp per epoch)

  __device__ __forceinline__ void put_sides(const LaneAddr<T, K>& la, int r0, int r1) const {
    typedef Tile<T, K> L;
    const int w = wl + wr, n = (r1 - r0) * w;
    if (w <= 0 || n <= 0) return;
    const int lane = threadIdx.x & 31;
    // element i = lane + 32 t of the (row, side column) list: (q, j) advance
    // incrementally (one division per call, none per element)
    const int dq = 32 / w, dj = 32 - dq * w;
    int q = lane / w, j = lane - q * w;
    for (int i = lane; i < n; i += 32) {
      const int r = r0 + q;
      const int c = j < wl ? cl0 + j : cr0 + (j - wl);
      T v;
      if constexpr (sizeof(T) == 8) {
        asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(la.base + (uint32_t)(L::at(r, c) * 8)));
      } else {
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(la.base + (uint32_t)(L::at(r, c) * 4)));
      }
      st_cg(g0 + (int64_t)r * pitch + c, v);
      q += dq;
      j += dj;
      if (j >= w) {
        j -= w;
        ++q;
      }
    }
  }
  __device__ __forceinline__ void put_rows(const LaneAddr<T, K>& la, int r0, int r1) const {
    if (full_mask == 0u || r0 >= r1) return;
    int row = r0;
    for (; row + 4 <= r1; row += 4) {  // 4 rows of LDS in flight, then the stores
      T v[4][K];
#pragma unroll
      for (int u = 0; u < 4; ++u) load_row<T, K>(la, row + u, v[u]);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        T* p = g + (int64_t)(row + u) * pitch;
#pragma unroll
        for (int e = 0; e < K; ++e) st_pred(((full_mask >> e) & 1u) != 0, p + e, v[u][e]);
      }
    }
    for (; row < r1; ++row) {
      T v[K];
      load_row<T, K>(la, row, v);
      T* p = g + (int64_t)row * pitch;
#pragma unroll
      for (int e = 0; e < K; ++e) st_pred(((full_mask >> e) & 1u) != 0, p + e, v[e]);
    }
  }
  // publish the part of band [ya, yb) the neighbours read; returns the cells
  // stored (whole owned rows: the owned width; sides: wl + wr per row)
  __device__ __forceinline__ int64_t put_band(const LaneAddr<T, K>& la, int ya, int yb,
                                              int owned_w) const {
    const int r0 = max(ya, own0), r1 = min(yb, own1);
    const int s0 = max(r0, top1), s1 = min(r1, bot0);
    if (s0 < s1) put_sides(la, s0, s1);
    put_rows(la, r0, min(r1, top1));
    put_rows(la, max(r0, bot0), r1);
    return (int64_t)max(0, s1 - s0) * (wl + wr) +
           (int64_t)(max(0, min(r1, top1) - r0) + max(0, r1 - max(r0, bot0))) * owned_w;
  }
};

// ---------------------------------------------------------------------------
// Two-step band sweep: rows [ya, yb) of the tile receive their t+2 values.
// 1 <= ya, yb <= Lh-1, yb - ya >= 2; rows 0 and Lh-1 are the frozen frame.
// Reads t rows [ya-2, yb+2) ∩ [0, Lh). The two foreign rows above are pushed
// into level 1 and the two below are held in registers BEFORE the CTA
// barrier inside; owned rows are written only after it. Every warp of the CTA
// must call this (idle warps with active=false).
//
// Stream of t rows into level 1, whose output rows feed level 2:
//   t(r) arrives  ->  level 1 finishes t+1 row r-1  ->  level 2 finishes t+2
//   row r-2, stored over row r-2 (no longer read: t(r-2) is consumed).
// The next row's LDS is issued before the current row's arithmetic.
// ---------------------------------------------------------------------------
template <typename T, int K, bool SYM, bool DYN>
__device__ __forceinline__ void sweep2(const LaneAddr<T, K>& la, int Lh, int ya, int yb,
                                       bool active, const Weights<T>& wt, const LaneCtx& lc) {
  typedef Level<T, K, SYM, DYN> Lv;
  constexpr int CH = Tile<T, K>::CH;
  constexpr uint32_t RB = (uint32_t)(Tile<T, K>::ROW * sizeof(T));
  Lv l1, l2;
  T x[K], y[K], b[K], o[K], h0[K], h1[K];
  const bool top_frozen = (ya == 1);       // row ya-1 is the frozen frame
  const bool bot_frozen = (yb == Lh - 1);  // row yb is the frozen frame
  if (active) {
    load_row<T, K>(la, yb, h0);
    if (!bot_frozen) load_row<T, K>(la, yb + 1, h1);
    if (top_frozen) {
      load_row<T, K>(la, 0, x);
      l1.start(x, wt);
      l2.start(x, wt);  // level 1's row 0 is the frozen row itself
    } else {
      load_row<T, K>(la, ya - 2, x);
      load_row<T, K>(la, ya - 1, y);
      l1.start(x, wt);
      l1.template push<false, true>(y, o, wt, lc);
    }
  }
  __syncthreads();  // every foreign row is now in registers; owned rows are ours
  if (!active) return;
  // owned rows ya, ya+1 complete the fill of level 2 (nothing stored yet)
  load_row<T, K>(la, ya, x);
  load_row<T, K>(la, ya + 1, y);
  if (top_frozen) {
    l1.template push<false, true>(x, b, wt, lc);  // row 0 was the start: no t+1 row 0 to finish
    l1.template push<true, true>(y, b, wt, lc);   // t+1 row 1
    l2.template push<false, true>(b, o, wt, lc);
  } else {
    l1.template push<true, true>(x, b, wt, lc);   // t+1 row ya-1
    l2.start(b, wt);
    l1.template push<true, true>(y, b, wt, lc);   // t+1 row ya
    l2.template push<false, true>(b, o, wt, lc);
  }
  // steady rows r = ya+2 .. yb-1: t+2 row r-2 stored
  int r = ya + 2;
  uint32_t rowp = la.row(r);
  if (r < yb) load_row_at<CH>(rowp, la.off, x);
#define DTB_SWEEP_ROW(X, Y)                                       \
  {                                                               \
    load_row_at<CH>(rowp + RB, la.off, Y);                        \
    l1.template push<true, true>(X, b, wt, lc);                   \
    l2.template push<true, true>(b, o, wt, lc);                   \
    store_row_at<CH>(rowp - 2 * RB, la.off, o);                   \
    rowp += RB;                                                   \
  }
  constexpr int U = DTB_SWEEP_UNROLL(T);
  for (; r + U < yb; r += U) {
#pragma unroll
    for (int u = 0; u < U / 2; ++u) {
      DTB_SWEEP_ROW(x, y)
      DTB_SWEEP_ROW(y, x)
    }
  }
  for (; r + 1 < yb; ++r) {
    DTB_SWEEP_ROW(x, y)
    copy_row<T, K>(y, x);
  }
#undef DTB_SWEEP_ROW
  if (r < yb) {  // last owned row: nothing to prefetch
    l1.template push<true, true>(x, b, wt, lc);
    l2.template push<true, true>(b, o, wt, lc);
    store_row_at<CH>(rowp - 2 * RB, la.off, o);
  }
  // the two pre-read rows below the band finish its last two rows
  if (bot_frozen) {
    l1.template push<true, false>(h0, b, wt, lc);  // t+1 row yb-1
    l2.template push<true, true>(b, o, wt, lc);
    store_row<T, K>(la, yb - 2, o);
    l2.template push<true, false>(h0, o, wt, lc);  // the frozen row is its own t+1 value
    store_row<T, K>(la, yb - 1, o);
  } else {
    l1.template push<true, true>(h0, b, wt, lc);   // t+1 row yb-1
    l2.template push<true, true>(b, o, wt, lc);
    store_row<T, K>(la, yb - 2, o);
    l1.template push<true, false>(h1, b, wt, lc);  // t+1 row yb
    l2.template push<true, false>(b, o, wt, lc);
    store_row<T, K>(la, yb - 1, o);
  }
}

// One-step band sweep (odd step counts): rows [ya, yb) get t+1;
// reads t rows [ya-1, yb+1). yb - ya >= 1.
template <typename T, int K, bool SYM, bool DYN>
__device__ __forceinline__ void sweep1(const LaneAddr<T, K>& la, int Lh, int ya, int yb,
                                       bool active, const Weights<T>& wt, const LaneCtx& lc) {
  typedef Level<T, K, SYM, DYN> Lv;
  (void)Lh;
  Lv l1;
  T x[K], h0[K], o[K];
  if (active) {
    load_row<T, K>(la, yb, h0);
    load_row<T, K>(la, ya - 1, x);
    l1.start(x, wt);
  }
  __syncthreads();
  if (!active) return;
  load_row<T, K>(la, ya, x);
  l1.template push<false, true>(x, o, wt, lc);
  for (int r = ya + 1; r < yb; ++r) {
    load_row<T, K>(la, r, x);
    l1.template push<true, true>(x, o, wt, lc);
    store_row<T, K>(la, r - 1, o);
  }
  l1.template push<true, false>(h0, o, wt, lc);
  store_row<T, K>(la, yb - 1, o);
}

// Split rows [1, Lh-1) into `nb` bands as evenly as possible; band b gets
// [ya, yb). Bands must be >= minh rows: the caller picks nb accordingly.
__device__ __forceinline__ void band_rows(int Lh, int nb, int b, int& ya, int& yb) {
  const int rows = Lh - 2;
  const int base = rows / nb, rem = rows % nb;
  ya = 1 + b * base + min(b, rem);
  yb = ya + base + (b < rem ? 1 : 0);
}

// Advance the tile `steps` time steps in place. All threads of the CTA call.
// With `pub` non-null each warp publishes its band right after its own last
// sweep and bumps the CTA's epoch flag with a release-add (neighbours wait for
// nwarps bumps per epoch). One CTA-level release by thread 0 after the
// closing barrier instead measured 7 % slower on C2 (10^4 steps, B200 A/B).
//
// cnt (DTB_FLAG_COUNT, else null): [1] += cells the publish stored, [3] +=
// cells each sweep updated (the band's rows at every level, Lw-2 columns;
// frozen rows and columns are not updates).
template <typename T, int K, bool SYM, bool DYN>
__device__ void advance_tile(T* __restrict__ tile, int Lw, int Lh, int steps,
                             const Weights<T>& wt, const Publisher<T, K>* pub = nullptr,
                             unsigned long long* cnt = nullptr, int owned_w = 0) {
  const int warp = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  LaneCtx lc;
  lc.lane = threadIdx.x & 31;
  const LaneAddr<T, K> la(tile, lc.lane);
  lc.first = (lc.lane == 0);
  lc.last = (lc.lane == (Lw - 1) / K);
  lc.last_e = (Lw - 1) % K;
  const int rows = Lh - 2;
  if (rows <= 0 || Lw <= 2) return;
  auto publish = [&](bool act, int ya, int yb) {
    if (act) {
      const int64_t n = pub->put_band(la, ya, yb, owned_w);
      if (cnt && lc.lane == 0 && n) atomicAdd(cnt + 1, (unsigned long long)n);
    }
    __syncwarp();
    if (lc.lane == 0)
      asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(pub->flag) : "memory");
  };
  int s = 0;
  if (steps >= 2 && rows >= 2) {
    const int nb2 = max(1, min(nw, rows / 2));
    int ya, yb;
    band_rows(Lh, nb2, min(warp, nb2 - 1), ya, yb);
    const bool act = warp < nb2;
    for (; s + 2 <= steps; s += 2) {
      sweep2<T, K, SYM, DYN>(la, Lh, ya, yb, act, wt, lc);
      if (cnt && act && lc.lane == 0)
        atomicAdd(cnt + 3, (unsigned long long)((2 * (yb - ya) + 2 - (ya == 1) -
                                                 (yb == Lh - 1)) * (Lw - 2)));
      if (pub && s + 2 == steps) publish(act, ya, yb);  // rows final: publish now
      __syncthreads();
    }
  }
  if (s < steps) {
    const int nb1 = max(1, min(nw, rows));
    int ya, yb;
    band_rows(Lh, nb1, min(warp, nb1 - 1), ya, yb);
    const bool act = warp < nb1;
    for (; s < steps; ++s) {
      sweep1<T, K, SYM, DYN>(la, Lh, ya, yb, act, wt, lc);
      if (cnt && act && lc.lane == 0)
        atomicAdd(cnt + 3, (unsigned long long)((yb - ya) * (Lw - 2)));
      if (pub && s + 1 == steps) publish(act, ya, yb);
      __syncthreads();
    }
  }
}

}  // namespace dtb
