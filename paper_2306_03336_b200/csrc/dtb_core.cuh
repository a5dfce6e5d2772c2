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
// written with __dmul_rn/__dadd_rn (never contracted) and compiled with
// -fmad=false, so every schedule below is bitwise equal to jacobi_reference
// (oracle.py:19-34).
//
// Layout and schedule (B200-first, not a port of engine.py):
//  * a warp spans the whole tile width; lane l owns K consecutive columns
//    [l*K, l*K+K) held in registers; smem rows have a fixed pitch of 32*K
//    elements and are read/written as 16-byte chunks with an XOR chunk
//    swizzle that makes every LDS.128/STS.128 conflict-free;
//  * W/E neighbours across lanes come from two 64-bit shuffles per row, never
//    from shared memory (the smem traffic is one load + one store per cell per
//    sweep);
//  * warps split the tile's rows into bands and march down them keeping a
//    rolling window of rows in registers (paper Listing 1's t[ILP+2],
//    PAPER.md:174-192) — and they advance TWO time steps per sweep: the t+1
//    row is produced from the t window and immediately consumed by the t+2
//    row one row behind, so each cell is loaded and stored once per two
//    updates. Band seams are resolved by reading the 2 foreign rows on each
//    side BEFORE a CTA barrier and writing only owned rows after it (the
//    in-place, single-buffered update: smem holds exactly one copy of the
//    tile, which is what lets a 1900^2 fp64 grid live in 148 SMs' smem).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

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

// The reference's update for one cell, kernel.py:137-139 / grid.py:95-116.
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

template <typename T, int K>
__device__ __forceinline__ void load_row(const T* __restrict__ tile, int r, int lane, T (&v)[K]) {
  typedef Tile<T, K> L;
  typedef typename Arith<T>::vec_t V;
  const T* row = tile + r * L::ROW;
#pragma unroll
  for (int j = 0; j < L::CH; ++j) {
    const int c = L::swz(lane * L::CH + j);
    V x = *reinterpret_cast<const V*>(row + c * L::EPC);
    const T* px = reinterpret_cast<const T*>(&x);
#pragma unroll
    for (int q = 0; q < L::EPC; ++q) v[j * L::EPC + q] = px[q];
  }
}

template <typename T, int K>
__device__ __forceinline__ void store_row(T* __restrict__ tile, int r, int lane, const T (&v)[K]) {
  typedef Tile<T, K> L;
  typedef typename Arith<T>::vec_t V;
  T* row = tile + r * L::ROW;
#pragma unroll
  for (int j = 0; j < L::CH; ++j) {
    const int c = L::swz(lane * L::CH + j);
    V x;
    T* px = reinterpret_cast<T*>(&x);
#pragma unroll
    for (int q = 0; q < L::EPC; ++q) px[q] = v[j * L::EPC + q];
    *reinterpret_cast<V*>(row + c * L::EPC) = x;
  }
}

template <typename T>
__device__ __forceinline__ T shfl_up1(T v) { return __shfl_up_sync(0xffffffffu, v, 1); }
template <typename T>
__device__ __forceinline__ T shfl_dn1(T v) { return __shfl_down_sync(0xffffffffu, v, 1); }

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

// One row of updates: out = stencil(up, mid, dn) for the lane's K columns;
// frozen columns keep `mid`.
template <typename T, int K, bool DYN>
__device__ __forceinline__ void row_update(const T (&up)[K], const T (&mid)[K], const T (&dn)[K],
                                           T (&out)[K], const Weights<T>& wt, const LaneCtx& lc) {
  const T west_edge = shfl_up1(mid[K - 1]);
  const T east_edge = shfl_dn1(mid[0]);
#pragma unroll
  for (int e = 0; e < K; ++e) {
    const T wv = (e == 0) ? west_edge : mid[e - 1];
    const T ev = (e == K - 1) ? east_edge : mid[e + 1];
    out[e] = cell_update(wv, ev, up[e], mid[e], dn[e], wt);
  }
  if (lc.first) out[0] = mid[0];
  if (DYN) {
    if (lc.last) {
#pragma unroll
      for (int e = 0; e < K; ++e)
        if (e == lc.last_e) out[e] = mid[e];
    }
  } else {
    if (lc.last) out[K - 1] = mid[K - 1];
  }
}

template <typename T, int K>
__device__ __forceinline__ void copy_row(const T (&a)[K], T (&b)[K]) {
#pragma unroll
  for (int e = 0; e < K; ++e) b[e] = a[e];
}

// ---------------------------------------------------------------------------
// Two-step band sweep. Rows [ya, yb) of the tile receive their t+2 values;
// 1 <= ya, yb <= Lh-1, yb - ya >= 2. Rows 0 and Lh-1 are the frozen frame.
// Reads t rows [ya-2, yb+2) ∩ [0, Lh). Foreign rows (outside [ya, yb)) are
// read before the CTA barrier the caller passes through `bar`; owned rows are
// written only after it. Every warp of the CTA must call this (idle warps
// with active=false) because of the barrier inside.
// ---------------------------------------------------------------------------
template <typename T, int K, bool DYN>
__device__ __forceinline__ void sweep2(T* __restrict__ tile, int Lh, int ya, int yb, bool active,
                                       const Weights<T>& wt, const LaneCtx& lc) {
  T a0[K], a1[K], a2[K];   // t rows (rolling)
  T b0[K], b1[K], b2[K];   // t+1 rows (rolling)
  T h0[K], h1[K];          // pre-read bottom halo (t rows yb, yb+1)
  T o[K];
  const bool top_frozen = (ya == 1);       // row ya-1 is the frozen frame
  const bool bot_frozen = (yb == Lh - 1);  // row yb is the frozen frame
  const int lane = lc.lane;
  if (active) {
    if (!top_frozen) load_row<T, K>(tile, ya - 2, lane, a0);
    load_row<T, K>(tile, ya - 1, lane, a1);
    load_row<T, K>(tile, yb, lane, h0);
    if (!bot_frozen) load_row<T, K>(tile, yb + 1, lane, h1);
  }
  __syncthreads();  // every foreign row is now in registers; owned rows are ours
  if (!active) return;

  load_row<T, K>(tile, ya, lane, a2);
  // level 1, row ya-1
  if (top_frozen) copy_row<T, K>(a1, b0);
  else row_update<T, K, DYN>(a0, a1, a2, b0, wt, lc);
  // level 1, row ya (needs t row ya+1: owned unless the band is 2 rows... yb-ya>=2 so ya+1 < yb)
  load_row<T, K>(tile, ya + 1, lane, a0);
  row_update<T, K, DYN>(a1, a2, a0, b1, wt, lc);
  // window now: t rows ya (a2), ya+1 (a0); t+1 rows ya-1 (b0), ya (b1)
  // Steady state: for r = ya+1 .. yb: level-1 row r needs t rows r-1,r,r+1;
  // then level-2 row r-1 from t+1 rows r-2,r-1,r. Unrolled by 3 so the
  // rolling windows rotate by renaming instead of register moves.
  int r = ya + 1;
#define DTB_STEP2(TM1, TC, TP1, BM2, BM1, BR)                                   \
  {                                                                              \
    const int q = r + 1;                                                         \
    if (q < yb) load_row<T, K>(tile, q, lane, TP1);                              \
    else if (q == yb) copy_row<T, K>(h0, TP1);                                   \
    else copy_row<T, K>(h1, TP1);                                                \
    if (r == yb && bot_frozen) copy_row<T, K>(TC, BR);                           \
    else row_update<T, K, DYN>(TM1, TC, TP1, BR, wt, lc);                             \
    row_update<T, K, DYN>(BM2, BM1, BR, o, wt, lc);                                   \
    store_row<T, K>(tile, r - 1, lane, o);                                       \
    ++r;                                                                         \
  }
  // rotation: (t rows) r-1=a2, r=a0, r+1 -> a1 ; (t+1) r-2=b0, r-1=b1, r -> b2
  while (r + 2 <= yb) {
    DTB_STEP2(a2, a0, a1, b0, b1, b2)
    DTB_STEP2(a0, a1, a2, b1, b2, b0)
    DTB_STEP2(a1, a2, a0, b2, b0, b1)
  }
  if (r <= yb) {
    DTB_STEP2(a2, a0, a1, b0, b1, b2)
    if (r <= yb) { DTB_STEP2(a0, a1, a2, b1, b2, b0) }
  }
#undef DTB_STEP2
}

// One-step band sweep (odd step counts): rows [ya, yb) get t+1;
// reads t rows [ya-1, yb+1). yb - ya >= 1.
template <typename T, int K, bool DYN>
__device__ __forceinline__ void sweep1(T* __restrict__ tile, int Lh, int ya, int yb, bool active,
                                       const Weights<T>& wt, const LaneCtx& lc) {
  T a0[K], a1[K], a2[K], h0[K], o[K];
  const int lane = lc.lane;
  (void)Lh;
  if (active) {
    load_row<T, K>(tile, ya - 1, lane, a0);
    load_row<T, K>(tile, yb, lane, h0);
  }
  __syncthreads();
  if (!active) return;
  load_row<T, K>(tile, ya, lane, a1);
  int r = ya;
#define DTB_STEP1(TM1, TC, TP1)                                                  \
  {                                                                              \
    const int q = r + 1;                                                         \
    if (q < yb) load_row<T, K>(tile, q, lane, TP1);                              \
    else copy_row<T, K>(h0, TP1);                                                \
    row_update<T, K, DYN>(TM1, TC, TP1, o, wt, lc);                                   \
    store_row<T, K>(tile, r, lane, o);                                           \
    ++r;                                                                         \
  }
  while (r + 3 <= yb) {
    DTB_STEP1(a0, a1, a2)
    DTB_STEP1(a1, a2, a0)
    DTB_STEP1(a2, a0, a1)
  }
  if (r < yb) {
    DTB_STEP1(a0, a1, a2)
    if (r < yb) { DTB_STEP1(a1, a2, a0) }
  }
#undef DTB_STEP1
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
template <typename T, int K, bool DYN>
__device__ void advance_tile(T* __restrict__ tile, int Lw, int Lh, int steps,
                             const Weights<T>& wt) {
  const int warp = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  LaneCtx lc;
  lc.lane = threadIdx.x & 31;
  lc.first = (lc.lane == 0);
  lc.last = (lc.lane == (Lw - 1) / K);
  lc.last_e = (Lw - 1) % K;
  const int rows = Lh - 2;
  if (rows <= 0 || Lw <= 2) return;
  int s = 0;
  if (steps >= 2 && rows >= 2) {
    const int nb2 = max(1, min(nw, rows / 2));
    int ya, yb;
    band_rows(Lh, nb2, min(warp, nb2 - 1), ya, yb);
    const bool act = warp < nb2;
    for (; s + 2 <= steps; s += 2) {
      sweep2<T, K, DYN>(tile, Lh, ya, yb, act, wt, lc);
      __syncthreads();
    }
  }
  if (s < steps) {
    const int nb1 = max(1, min(nw, rows));
    int ya, yb;
    band_rows(Lh, nb1, min(warp, nb1 - 1), ya, yb);
    for (; s < steps; ++s) {
      sweep1<T, K, DYN>(tile, Lh, ya, yb, warp < nb1, wt, lc);
      __syncthreads();
    }
  }
}

}  // namespace dtb
