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

// Schedule variants (compile-time, for A/B measurement; defaults are the product)
#ifndef DTB_ROW2
#define DTB_ROW2 0      // steady loop evaluates L1/L2 rows stage-major together
#endif
#ifndef DTB_FASTPATH
#define DTB_FASTPATH 1  // static sweep schedule for bands of 4k rows
#endif
#ifndef DTB_PUBREG
#define DTB_PUBREG 6    // resident publish: 0 smem pass after the epoch, 1 from registers
                        // inside the last sweep, 2 each warp right after its own last sweep,
                        // 3 as 2 with a per-warp release-add on the epoch flag (no CTA barrier),
                        // 4 every owned row from registers + release-add, 5 as 2 with one
                        // CTA-level release, 6 as 3 with the side columns flattened across
                        // lanes (fewest stores; the default)
#endif
#ifndef DTB_RING
#define DTB_RING 2      // resident halo refresh: 0 generic, 1 ring copy after one wait,
                        // 2 warp per direction: poll that neighbour, then copy its region
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

// nz: -0.0 supplied at run time (see f2mul: an opaque zero addend keeps
// ptxas from fusing a packed product into the following packed add)
template <typename T> struct Weights { T w, e, s, c, n, nz; };

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

// Lane geometry of the frozen frame's columns: column 0 is lane 0 element 0,
// column Lw-1 is lane `last` element K-1 (the planner keeps Lw % K == 0).
// DYN: Lw % K != 0 (only when one tile spans the whole width), so the right
// frozen column sits at element last_e of its lane instead of element K-1.
struct LaneCtx {
  int lane;
  bool first;  // lane holds frozen column 0
  bool last;   // lane holds frozen column Lw-1
  int last_e;  // its element index (== K-1 unless DYN)
  bool fz = true;  // warp-uniform: the tile has a frozen column at all (the
                   // resident kernel freezes only domain-ghost columns; a halo
                   // side's outer column may go stale — its error front moves
                   // one column per step like the frozen frame's, planner.py:272-286)
};

// Packed FP32 (sm_100a fma/add.rn.f32x2): two cells per instruction, each
// element rounded exactly like __fadd_rn/__fmul_rn (no fusion, no FTZ), so
// results are bitwise those of the scalar expression. On B200 a packed
// instruction issues at half rate, so the element rate equals scalar FP32
// (tools/microbench/f32x2.cu); it only frees issue slots. Measured no gain
// for the resident sweep and spills in the 128-register pipe: off by default.
#ifndef DTB_FZ_BRANCH
#define DTB_FZ_BRANCH 0  // 1: skip the frozen-column selects when the tile has none (no gain measured)
#endif
#ifndef DTB_F32X2
#define DTB_F32X2 0  // off: same element rate as scalar FP32 on B200 (packed ops issue at half rate)
#endif
__device__ __forceinline__ uint64_t f2pack(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void f2unpack(uint64_t v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
// x*w rounded once, as fma(x, w, -0.0) with the -0.0 a kernel argument: ptxas
// (12.9) contracts mul.rn.f32x2 + add.rn.f32x2 into one FFMA2 even with
// --fmad=false, and folds fma(x, w, constant -0) the same way; an addend it
// cannot see keeps the product and the sum separately rounded. fma(x, w, -0)
// equals round(x*w) bit for bit (exact product + -0 is the exact product,
// signed zeros included).
__device__ __forceinline__ uint64_t f2mul(uint64_t a, uint64_t b, uint64_t nz) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(nz));
  return d;
}
__device__ __forceinline__ uint64_t f2add(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
// cells (2p, 2p+1) of a row: ((((W*w + E*e) + S*s) + C*c) + N*n) per element
__device__ __forceinline__ uint64_t f2cell(uint64_t W, uint64_t E, uint64_t S, uint64_t C,
                                           uint64_t N, const uint64_t (&pw)[6]) {
  uint64_t acc = f2mul(W, pw[0], pw[5]);
  acc = f2add(acc, f2mul(E, pw[1], pw[5]));
  acc = f2add(acc, f2mul(S, pw[2], pw[5]));
  acc = f2add(acc, f2mul(C, pw[3], pw[5]));
  acc = f2add(acc, f2mul(N, pw[4], pw[5]));
  return acc;
}
template <int K>
__device__ __forceinline__ void row_update_f32x2(const float (&up)[K], const float (&mid)[K],
                                                 const float (&dn)[K], float (&out)[K],
                                                 float west_edge, float east_edge,
                                                 const uint64_t (&pw)[6]) {
#pragma unroll
  for (int p = 0; p < K / 2; ++p) {
    const int e0 = 2 * p, e1 = 2 * p + 1;
    const uint64_t W = f2pack(e0 == 0 ? west_edge : mid[e0 - 1], mid[e0]);
    const uint64_t E = f2pack(mid[e1], e1 == K - 1 ? east_edge : mid[e1 + 1]);
    const uint64_t acc = f2cell(W, E, f2pack(up[e0], up[e1]), f2pack(mid[e0], mid[e1]),
                                f2pack(dn[e0], dn[e1]), pw);
    f2unpack(acc, out[e0], out[e1]);
  }
}
__device__ __forceinline__ void f2weights(const Weights<float>& wt, uint64_t (&pw)[6]) {
  pw[0] = f2pack(wt.w, wt.w);
  pw[1] = f2pack(wt.e, wt.e);
  pw[2] = f2pack(wt.s, wt.s);
  pw[3] = f2pack(wt.c, wt.c);
  pw[4] = f2pack(wt.n, wt.n);
  pw[5] = f2pack(wt.nz, wt.nz);
}

// One row of updates: out = stencil(up, mid, dn) for the lane's K columns;
// frozen columns keep `mid`.
template <typename T, int K, bool DYN>
__device__ __forceinline__ void row_update(const T (&up)[K], const T (&mid)[K], const T (&dn)[K],
                                           T (&out)[K], const Weights<T>& wt, const LaneCtx& lc) {
  const T west_edge = shfl_up1(mid[K - 1]);
  const T east_edge = shfl_dn1(mid[0]);
  if constexpr (sizeof(T) == 4 && K % 2 == 0 && DTB_F32X2) {
    uint64_t pw[6];
    f2weights(wt, pw);
    row_update_f32x2<K>(up, mid, dn, out, west_edge, east_edge, pw);
  } else {
#pragma unroll
    for (int e = 0; e < K; ++e) {
      const T wv = (e == 0) ? west_edge : mid[e - 1];
      const T ev = (e == K - 1) ? east_edge : mid[e + 1];
      out[e] = cell_update(wv, ev, up[e], mid[e], dn[e], wt);
    }
  }
  if (DTB_FZ_BRANCH && !lc.fz) return;
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

// Two independent row updates evaluated stage-major: every accumulation
// stage (w, e, s, c, n) is issued for all 2K cells before the next, so the
// FP pipe always has 2K independent dependency chains in flight (the
// accumulation order within each cell is still W,E,S,C,N — only the
// interleaving across cells changes, which cannot change any result).
template <typename T, int K, bool DYN>
__device__ __forceinline__ void row_update2(const T (&ua)[K], const T (&ma)[K], const T (&da)[K],
                                            T (&oa)[K], const T (&ub)[K], const T (&mb)[K],
                                            const T (&db)[K], T (&ob)[K], const Weights<T>& wt,
                                            const LaneCtx& lc) {
  typedef Arith<T> A;
  const T wa = shfl_up1(ma[K - 1]), ea = shfl_dn1(ma[0]);
  const T wb = shfl_up1(mb[K - 1]), eb = shfl_dn1(mb[0]);
  if constexpr (sizeof(T) == 4 && K % 2 == 0 && DTB_F32X2) {
    uint64_t pw[6];
    f2weights(wt, pw);
    row_update_f32x2<K>(ua, ma, da, oa, wa, ea, pw);
    row_update_f32x2<K>(ub, mb, db, ob, wb, eb, pw);
  } else {
#pragma unroll
  for (int e = 0; e < K; ++e) {
    oa[e] = A::mul((e == 0) ? wa : ma[e - 1], wt.w);
    ob[e] = A::mul((e == 0) ? wb : mb[e - 1], wt.w);
  }
#pragma unroll
  for (int e = 0; e < K; ++e) {
    oa[e] = A::add(oa[e], A::mul((e == K - 1) ? ea : ma[e + 1], wt.e));
    ob[e] = A::add(ob[e], A::mul((e == K - 1) ? eb : mb[e + 1], wt.e));
  }
#pragma unroll
  for (int e = 0; e < K; ++e) {
    oa[e] = A::add(oa[e], A::mul(ua[e], wt.s));
    ob[e] = A::add(ob[e], A::mul(ub[e], wt.s));
  }
#pragma unroll
  for (int e = 0; e < K; ++e) {
    oa[e] = A::add(oa[e], A::mul(ma[e], wt.c));
    ob[e] = A::add(ob[e], A::mul(mb[e], wt.c));
  }
#pragma unroll
  for (int e = 0; e < K; ++e) {
    oa[e] = A::add(oa[e], A::mul(da[e], wt.n));
    ob[e] = A::add(ob[e], A::mul(db[e], wt.n));
  }
  }
  if (DTB_FZ_BRANCH && !lc.fz) return;
  if (lc.first) { oa[0] = ma[0]; ob[0] = mb[0]; }
  if (DYN) {
    if (lc.last) {
#pragma unroll
      for (int e = 0; e < K; ++e)
        if (e == lc.last_e) { oa[e] = ma[e]; ob[e] = mb[e]; }
    }
  } else {
    if (lc.last) { oa[K - 1] = ma[K - 1]; ob[K - 1] = mb[K - 1]; }
  }
}

template <typename T, int K>
__device__ __forceinline__ void copy_row(const T (&a)[K], T (&b)[K]) {
#pragma unroll
  for (int e = 0; e < K; ++e) b[e] = a[e];
}

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

// Band-to-band synchronisation of the two-step sweeps without CTA barriers
// (DTB_BANDSYNC): per-warp counters in shared memory. pre[w] = the sweep whose
// foreign rows warp w has read, done[w] = the last sweep warp w finished.
// A warp reads its neighbours' seam rows once they are done with the previous
// sweep, and overwrites its own seam rows only after the neighbour that reads
// them has; warps never wait for the whole CTA, so one band's prologue or
// epilogue overlaps the other bands' steady rows.
struct BandSync {
  int* pre;
  int* done;
  int seq;   // this sweep's number (1, 2, ...)
  int nb;    // active bands
};
__device__ __forceinline__ void bs_wait(const int* p, int v) {
  while (ld_acquire_cta(p) < v) {
  }
}
__device__ __forceinline__ void bs_post(int* p, int v) {
  __syncwarp();
  if ((threadIdx.x & 31) == 0) st_release_cta(p, v);
}

// Thread groups: GT == 0 is the whole CTA; GT > 0 splits the CTA into
// blockDim.x / GT independent groups of GT threads (the resident kernel's two
// tiles per CTA), each with its own named barrier 1 + group.
template <int GT>
__device__ __forceinline__ int gt_tid() {
  if constexpr (GT != 0) return (int)(threadIdx.x % GT);
  else return (int)threadIdx.x;
}
template <int GT>
__device__ __forceinline__ int gt_n() {
  if constexpr (GT != 0) return GT;
  else return (int)blockDim.x;
}
template <int GT>
__device__ __forceinline__ void gt_sync() {
  if constexpr (GT != 0)
    asm volatile("bar.sync %0, %1;" ::"r"(1 + (int)(threadIdx.x / GT)), "n"(GT) : "memory");
  else
    __syncthreads();
}

// Publisher: during the last sweep of a resident epoch, every freshly
// computed row that lies in the CTA's owned band (the cells its neighbours'
// halos cover) is also stored straight from registers to the L2 exchange
// buffer — the halo publish costs a few predicated STGs instead of a pass
// over shared memory. Rows [top0, top1) and [bot0, bot1) publish every owned
// column (full_mask); other owned rows [own0, own1) only the side columns.
__device__ __forceinline__ void st_pred(bool p, double* a, double v) {
  asm volatile("{ .reg .pred q; setp.ne.u32 q, %0, 0; @q st.global.cg.f64 [%1], %2; }"
               ::"r"((unsigned)p), "l"(a), "d"(v) : "memory");
}
__device__ __forceinline__ void st_pred(bool p, float* a, float v) {
  asm volatile("{ .reg .pred q; setp.ne.u32 q, %0, 0; @q st.global.cg.f32 [%1], %2; }"
               ::"r"((unsigned)p), "l"(a), "f"(v) : "memory");
}

// Publisher: during the last sweep of a resident epoch, rows of the owned
// top/bottom band (the rows the y-neighbours' halos cover, [own0, top1) and
// [bot0, own1)) are also stored straight from registers to the L2 exchange
// buffer (K predicated stores per lane, no branch). Only the warps whose band
// contains such rows run the publishing variant of the sweep; the narrow
// side columns are published from smem after the sweep.
template <typename T, int K>
struct Publisher {
  T* g;             // exchange buffer at (tile row 0, this lane's first column)
  int64_t pitch;
  int own0, own1, top1, bot0;
  uint32_t full_mask, side_mask;
  int* flag;        // modes 3/6: this CTA's epoch flag (per-warp release-add)
  // mode 2/3: publish the band's own rows [ya, yb) from smem (they are final once
  // the band's last sweep is done: no other warp writes them)
  // mode 6: side columns flattened across lanes (lane i -> element i of the
  // band's (row, side column) list), so one warp store covers 32 / (wl + wr)
  // rows instead of one
  T* g0;            // exchange buffer at (tile row 0, tile column 0)
  int cl0, wl, cr0, wr;  // side columns [cl0, cl0 + wl) and [cr0, cr0 + wr)
  __device__ __forceinline__ void put_sides(const LaneAddr<T, K>& la, int r0, int r1) const {
    typedef Tile<T, K> L;
    const int w = wl + wr, n = (r1 - r0) * w;
    const int lane = threadIdx.x & 31;
#pragma unroll 2
    for (int i = lane; i < n; i += 32) {
      const int q = i / w, j = i - q * w, r = r0 + q;
      const int c = j < wl ? cl0 + j : cr0 + (j - wl);
      T v;
      if (sizeof(T) == 8) {
        double d;
        asm volatile("ld.shared.f64 %0, [%1];" : "=d"(d) : "r"(la.base + (uint32_t)(L::at(r, c) * 8)));
        v = (T)d;
      } else {
        float f;
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(f) : "r"(la.base + (uint32_t)(L::at(r, c) * 4)));
        v = (T)f;
      }
      st_pred(true, g0 + (int64_t)r * pitch + c, v);
    }
  }
  __device__ __forceinline__ void put_band(const LaneAddr<T, K>& la, int ya, int yb) const {
    if (DTB_PUBREG == 6) {
      const int r0 = max(ya, own0), r1 = min(yb, own1);
      const int s0 = max(r0, top1), s1 = min(r1, bot0);
      if (s0 < s1) put_sides(la, s0, s1);
      put_rows(la, r0, min(r1, top1));
      put_rows(la, max(r0, bot0), r1);
      return;
    }
    put_rows(la, max(ya, own0), min(yb, own1));
  }
  __device__ __forceinline__ void put_rows(const LaneAddr<T, K>& la, int r0, int r1) const {
    // lanes with nothing to publish in any of these rows skip the loop
    if ((full_mask | side_mask) == 0u || r0 >= r1) return;
    int row = r0;
    for (; row + 4 <= r1; row += 4) {  // 4 rows of LDS in flight, then the stores
      T v[4][K];
#pragma unroll
      for (int u = 0; u < 4; ++u) load_row<T, K>(la, row + u, v[u]);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int rr = row + u;
        const uint32_t m = (rr < top1 || rr >= bot0) ? full_mask : side_mask;
        T* p = g + (int64_t)rr * pitch;
#pragma unroll
        for (int e = 0; e < K; ++e) st_pred(((m >> e) & 1u) != 0, p + e, v[u][e]);
      }
    }
    for (; row < r1; ++row) {
      T v[K];
      load_row<T, K>(la, row, v);
      const uint32_t m = (row < top1 || row >= bot0) ? full_mask : side_mask;
      T* p = g + (int64_t)row * pitch;
#pragma unroll
      for (int e = 0; e < K; ++e) st_pred(((m >> e) & 1u) != 0, p + e, v[e]);
    }
  }
  __device__ __forceinline__ bool covers(int ya, int yb) const {
    return (ya < top1 && yb > own0) || (ya < own1 && yb > bot0);
  }
  __device__ __forceinline__ void put(int row, const T (&v)[K]) const {
    uint32_t m;
    if (DTB_PUBREG == 4) {  // every owned row: full rows in the top/bottom band, else sides
      const bool own = row >= own0 && row < own1;
      m = own ? ((row < top1 || row >= bot0) ? full_mask : side_mask) : 0u;
    } else {
      const bool in = (row >= own0 && row < top1) || (row >= bot0 && row < own1);
      m = in ? full_mask : 0u;
    }
    T* p = g + (int64_t)row * pitch;
#pragma unroll
    for (int e = 0; e < K; ++e) st_pred(((m >> e) & 1u) != 0, p + e, v[e]);
  }
};

// ---------------------------------------------------------------------------
// Two-step band sweep. Rows [ya, yb) of the tile receive their t+2 values;
// 1 <= ya, yb <= Lh-1, yb - ya >= 2. Rows 0 and Lh-1 are the frozen frame.
// Reads t rows [ya-2, yb+2) ∩ [0, Lh). Foreign rows (outside [ya, yb)) are
// read before the CTA barrier inside; owned rows are written only after it.
// Every warp of the CTA must call this (idle warps with active=false).
//
// Software pipeline, one iteration per level-1 row r = ya-1 .. yb+1:
//   issue  LDS of t(r+2)                 (consumed one iteration later)
//   L1     b(r)   = stencil(t(r-1), t(r), t(r+1))
//   L2     out(r-2) = stencil(b(r-3), b(r-2), b(r-1))  -> STS row r-2
// L1 and L2 of one iteration are independent, doubling the ILP the FP64
// pipe sees. Rows live in 4-deep rotating register windows (t(q) in slot
// (q-ya+2)%4, b(q) in slot (q-ya+1)%4) unrolled 4x so every slot is static.
// Iterations j = r-ya+1 in [3, ...) whose loads hit owned rows run in a
// branch-free steady loop; the first three and the last few (frozen rows,
// pre-read halo rows) run through the general iteration.
// ---------------------------------------------------------------------------
template <typename T, int K, bool DYN, bool PUB, int GT = 0>
__device__ __forceinline__ void sweep2(const LaneAddr<T, K>& la, int Lh, int ya, int yb,
                                       bool active, const Weights<T>& wt, const LaneCtx& lc,
                                       const Publisher<T, K>& pub,
                                       const BandSync* bs = nullptr, int warp = 0) {
  T t0[K], t1[K], t2[K], t3[K];  // t rows
  T b0[K], b1[K], b2[K], b3[K];  // t+1 rows
  T h0[K], h1[K];                // pre-read bottom halo (t rows yb, yb+1)
  T o[K];
  const bool top_frozen = (ya == 1);       // row ya-1 is the frozen frame
  const bool bot_frozen = (yb == Lh - 1);  // row yb is the frozen frame
  if (bs && active) {  // the neighbours' seam rows are final
    if (warp > 0) bs_wait(bs->done + warp - 1, bs->seq - 1);
    if (warp + 1 < bs->nb) bs_wait(bs->done + warp + 1, bs->seq - 1);
  }
  if (active) {
    if (!top_frozen) load_row<T, K>(la, ya - 2, t0);
    load_row<T, K>(la, ya - 1, t1);
    load_row<T, K>(la, yb, h0);
    if (!bot_frozen) load_row<T, K>(la, yb + 1, h1);
  }
  if (bs) {
    if (!active) return;
    bs_post(bs->pre + warp, bs->seq);
  } else {
    gt_sync<GT>();  // every foreign row is now in registers; owned rows are ours
    if (!active) return;
  }
  load_row<T, K>(la, ya, t2);

  constexpr uint32_t kRowBytes = (uint32_t)(Tile<T, K>::ROW * sizeof(T));
  // steady iteration: r+2 < yb, ya+2 <= r < yb (no frozen row, owned loads)
#define DTB_STEADY(TM1, TC, TP1, TP2, BR, BM1, BM2, BM3)                         \
  {                                                                              \
    load_row_at<Tile<T, K>::CH>(rowp + 2 * kRowBytes, la.off, TP2);              \
    if (DTB_ROW2) {                                                              \
      row_update2<T, K, DYN>(TM1, TC, TP1, BR, BM3, BM2, BM1, o, wt, lc);        \
    } else {                                                                     \
      row_update<T, K, DYN>(TM1, TC, TP1, BR, wt, lc);                           \
      row_update<T, K, DYN>(BM3, BM2, BM1, o, wt, lc);                           \
    }                                                                            \
    store_row_at<Tile<T, K>::CH>(rowp - 2 * kRowBytes, la.off, o);               \
    if (PUB) pub.put(rr - 2, o);                                                 \
    rowp += kRowBytes;                                                           \
    ++rr;                                                                        \
  }
  const int H = yb - ya;
  if (DTB_FASTPATH && (H & 3) == 0 && H >= 4) {
    // ---- fast path: band height a multiple of 4 -> fully static schedule ----
    // j=0 (r=ya-1): L1(ya-1); load t(ya+1)
    load_row<T, K>(la, ya + 1, t3);
    if (top_frozen) copy_row<T, K>(t1, b0);
    else row_update<T, K, DYN>(t0, t1, t2, b0, wt, lc);
    // j=1 (r=ya): L1(ya); load t(ya+2)
    load_row<T, K>(la, ya + 2, t0);
    row_update<T, K, DYN>(t1, t2, t3, b1, wt, lc);
    // j=2 (r=ya+1): L1(ya+1); load t(ya+3)
    load_row<T, K>(la, ya + 3, t1);
    row_update<T, K, DYN>(t2, t3, t0, b2, wt, lc);
    // steady j=3 .. H-2 (r = ya+2 .. yb-3), (H-4)/4 blocks
    if (bs && warp > 0) bs_wait(bs->pre + warp - 1, bs->seq);  // rows ya, ya+1 read
    uint32_t rowp = la.row(ya + 2);
    int rr = ya + 2;
#ifndef DTB_UNROLL8
#define DTB_UNROLL8 (sizeof(T) == 8)  // 8-row steady blocks: fp64 +1.5 %, fp32 -2 % (B200 A/B)
#endif
    int blk = (H - 4) >> 2;
#ifndef DTB_UNROLL_X
#define DTB_UNROLL_X 2  // fp64 16-row steady blocks first (+0.6 % on C2 over 8-row blocks)
#endif
    if (DTB_UNROLL8 && DTB_UNROLL_X > 1) {
      for (; blk >= 2 * DTB_UNROLL_X; blk -= 2 * DTB_UNROLL_X) {
#pragma unroll
        for (int u = 0; u < DTB_UNROLL_X; ++u) {
          DTB_STEADY(t3, t0, t1, t2, b3, b2, b1, b0)
          DTB_STEADY(t0, t1, t2, t3, b0, b3, b2, b1)
          DTB_STEADY(t1, t2, t3, t0, b1, b0, b3, b2)
          DTB_STEADY(t2, t3, t0, t1, b2, b1, b0, b3)
          DTB_STEADY(t3, t0, t1, t2, b3, b2, b1, b0)
          DTB_STEADY(t0, t1, t2, t3, b0, b3, b2, b1)
          DTB_STEADY(t1, t2, t3, t0, b1, b0, b3, b2)
          DTB_STEADY(t2, t3, t0, t1, b2, b1, b0, b3)
        }
      }
    }
    if (DTB_UNROLL8) {
      for (; blk >= 2; blk -= 2) {
        DTB_STEADY(t3, t0, t1, t2, b3, b2, b1, b0)
        DTB_STEADY(t0, t1, t2, t3, b0, b3, b2, b1)
        DTB_STEADY(t1, t2, t3, t0, b1, b0, b3, b2)
        DTB_STEADY(t2, t3, t0, t1, b2, b1, b0, b3)
        DTB_STEADY(t3, t0, t1, t2, b3, b2, b1, b0)
        DTB_STEADY(t0, t1, t2, t3, b0, b3, b2, b1)
        DTB_STEADY(t1, t2, t3, t0, b1, b0, b3, b2)
        DTB_STEADY(t2, t3, t0, t1, b2, b1, b0, b3)
      }
    }
    for (; blk > 0; --blk) {
      DTB_STEADY(t3, t0, t1, t2, b3, b2, b1, b0)
      DTB_STEADY(t0, t1, t2, t3, b0, b3, b2, b1)
      DTB_STEADY(t1, t2, t3, t0, b1, b0, b3, b2)
      DTB_STEADY(t2, t3, t0, t1, b2, b1, b0, b3)
    }
    // tail j=H-1 (r=yb-2): t(yb) is h0; L1(yb-2), L2(yb-4)
    if (bs && warp + 1 < bs->nb) bs_wait(bs->pre + warp + 1, bs->seq);  // rows yb-2, yb-1 read
    row_update2<T, K, DYN>(t3, t0, t1, b3, b0, b1, b2, o, wt, lc);
    store_row<T, K>(la, yb - 4, o);
    if (PUB) pub.put(yb - 4, o);
    // r=yb-1: L1(yb-1) from (t0, t1, h0), L2(yb-3) from (b1, b2, b3)
    row_update2<T, K, DYN>(t0, t1, h0, b0, b1, b2, b3, o, wt, lc);
    store_row<T, K>(la, yb - 3, o);
    if (PUB) pub.put(yb - 3, o);
    // r=yb: L1(yb) (frozen row, or from (t1, h0, h1)), L2(yb-2) from (b2, b3, b0)
    if (bot_frozen) {
      copy_row<T, K>(h0, b1);
      row_update<T, K, DYN>(b2, b3, b0, o, wt, lc);
    } else {
      row_update2<T, K, DYN>(t1, h0, h1, b1, b2, b3, b0, o, wt, lc);
    }
    store_row<T, K>(la, yb - 2, o);
    if (PUB) pub.put(yb - 2, o);
    // r=yb+1: L2(yb-1) from (b3, b0, b1)
    row_update<T, K, DYN>(b3, b0, b1, o, wt, lc);
    store_row<T, K>(la, yb - 1, o);
    if (PUB) pub.put(yb - 1, o);
    if (bs) bs_post(bs->done + warp, bs->seq);
    return;
  }
  // general iteration (any r): sources and frozen rows resolved by branches
#define DTB_GEN(TM1, TC, TP1, TP2, BR, BM1, BM2, BM3)                            \
  {                                                                              \
    const int q = r + 2;                                                         \
    if (q < yb) load_row<T, K>(la, q, TP2);                                      \
    else if (q == yb) copy_row<T, K>(h0, TP2);                                   \
    else if (q == yb + 1 && !bot_frozen) copy_row<T, K>(h1, TP2);                \
    if (r <= yb) {                                                               \
      if ((r == ya - 1 && top_frozen) || (r == yb && bot_frozen))                \
        copy_row<T, K>(TC, BR);                                                  \
      else                                                                       \
        row_update<T, K, DYN>(TM1, TC, TP1, BR, wt, lc);                         \
    }                                                                            \
    if (r >= ya + 2) {                                                           \
      row_update<T, K, DYN>(BM3, BM2, BM1, o, wt, lc);                           \
      store_row<T, K>(la, r - 2, o);                                             \
      if (PUB) pub.put(r - 2, o);                                                \
    }                                                                            \
    ++r;                                                                         \
  }
  // slot pattern of iteration j (mod 4):
  //   j%4==0: (t0,t1,t2,t3, b0,b3,b2,b1)   j%4==1: (t1,t2,t3,t0, b1,b0,b3,b2)
  //   j%4==2: (t2,t3,t0,t1, b2,b1,b0,b3)   j%4==3: (t3,t0,t1,t2, b3,b2,b1,b0)
  // ---- general path (any band height >= 2) ----
  if (bs) {  // conservative: both seam neighbours have read before any store
    if (warp > 0) bs_wait(bs->pre + warp - 1, bs->seq);
    if (warp + 1 < bs->nb) bs_wait(bs->pre + warp + 1, bs->seq);
  }
  int r = ya - 1;
  DTB_GEN(t0, t1, t2, t3, b0, b3, b2, b1)  // j = 0
  DTB_GEN(t1, t2, t3, t0, b1, b0, b3, b2)  // j = 1
  DTB_GEN(t2, t3, t0, t1, b2, b1, b0, b3)  // j = 2
  // steady blocks of 4 starting at j = 3 (r = ya + 2): need r + 3 + 2 < yb
  uint32_t rowp = la.row(r);
  while (r + 5 < yb) {
    int rr = r;
    DTB_STEADY(t3, t0, t1, t2, b3, b2, b1, b0)
    DTB_STEADY(t0, t1, t2, t3, b0, b3, b2, b1)
    DTB_STEADY(t1, t2, t3, t0, b1, b0, b3, b2)
    DTB_STEADY(t2, t3, t0, t1, b2, b1, b0, b3)
    r += 4;
  }
  // tail from j = 3 (mod 4) until r > yb + 1
  while (r <= yb + 1) {
    DTB_GEN(t3, t0, t1, t2, b3, b2, b1, b0)
    if (r > yb + 1) break;
    DTB_GEN(t0, t1, t2, t3, b0, b3, b2, b1)
    if (r > yb + 1) break;
    DTB_GEN(t1, t2, t3, t0, b1, b0, b3, b2)
    if (r > yb + 1) break;
    DTB_GEN(t2, t3, t0, t1, b2, b1, b0, b3)
  }
  if (bs) bs_post(bs->done + warp, bs->seq);
#undef DTB_GEN
#undef DTB_STEADY
}

// One-step band sweep (odd step counts): rows [ya, yb) get t+1;
// reads t rows [ya-1, yb+1). yb - ya >= 1.
template <typename T, int K, bool DYN, bool PUB, int GT = 0>
__device__ __forceinline__ void sweep1(const LaneAddr<T, K>& la, int Lh, int ya, int yb,
                                       bool active, const Weights<T>& wt, const LaneCtx& lc,
                                       const Publisher<T, K>& pub) {
  T a0[K], a1[K], a2[K], h0[K], o[K];
  (void)Lh;
  if (active) {
    load_row<T, K>(la, ya - 1, a0);
    load_row<T, K>(la, yb, h0);
  }
  gt_sync<GT>();
  if (!active) return;
  load_row<T, K>(la, ya, a1);
  int r = ya;
#define DTB_STEP1(TM1, TC, TP1)                                                  \
  {                                                                              \
    const int q = r + 1;                                                         \
    if (q < yb) load_row<T, K>(la, q, TP1);                                      \
    else copy_row<T, K>(h0, TP1);                                                \
    row_update<T, K, DYN>(TM1, TC, TP1, o, wt, lc);                              \
    store_row<T, K>(la, r, o);                                                   \
    if (PUB) pub.put(r, o);                                                      \
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

// Two-step sweeps: band heights in whole multiples of 4 where possible (the
// static fast path of sweep2); the remainder rows go to the last band.
__device__ __forceinline__ void band_rows4(int Lh, int nb, int b, int& ya, int& yb) {
  const int rows = Lh - 2;
  const int q = rows >> 2;  // whole 4-row quads
  if (q < nb) {
    band_rows(Lh, nb, b, ya, yb);
    return;
  }
  const int base = q / nb, rem = q % nb;
  ya = 1 + 4 * (b * base + min(b, rem));
  yb = ya + 4 * (base + (b < rem ? 1 : 0));
  if (b == nb - 1) yb = Lh - 1;
}

// Advance the tile `steps` time steps in place. All threads of the CTA call.
// With `pub` non-null the final sweep also publishes the owned band.
template <typename T, int K, bool DYN, int GT = 0>
__device__ void advance_tile(T* __restrict__ tile, int Lw, int Lh, int steps,
                             const Weights<T>& wt, const Publisher<T, K>* pub = nullptr,
                             int* bsmem = nullptr, int* bseq = nullptr,
                             bool freeze_l = true, bool freeze_r = true) {
  const int warp = gt_tid<GT>() >> 5;
  const int nw = gt_n<GT>() >> 5;
  LaneCtx lc;
  lc.lane = threadIdx.x & 31;
  const LaneAddr<T, K> la(tile, lc.lane);
  lc.first = freeze_l && (lc.lane == 0);
  lc.last = freeze_r && (lc.lane == (Lw - 1) / K);
  lc.last_e = (Lw - 1) % K;
  lc.fz = freeze_l || freeze_r;
  const int rows = Lh - 2;
  if (rows <= 0 || Lw <= 2) return;
  Publisher<T, K> nopub;
  const Publisher<T, K>& pb = pub ? *pub : nopub;
  int s = 0;
  if (steps >= 2 && rows >= 2) {
    const int nb2 = max(1, min(nw, rows / 2));
    int ya, yb;
    band_rows4(Lh, nb2, min(warp, nb2 - 1), ya, yb);
    const bool act = warp < nb2;
    const bool band_pub = pub && ((DTB_PUBREG == 1 && pub->covers(ya, yb)) || DTB_PUBREG == 4);
    // band-to-band counters instead of CTA barriers between and inside the
    // two-step sweeps (not with in-sweep publishing); one barrier closes the run
    const bool use_bs = bsmem != nullptr && bseq != nullptr && !band_pub;
    BandSync bsync;
    bsync.pre = bsmem;
    bsync.done = bsmem + nw;
    bsync.nb = nb2;
    for (; s + 2 <= steps; s += 2) {
      bsync.seq = use_bs ? ++*bseq : 0;
      if (band_pub && s + 2 == steps) sweep2<T, K, DYN, true, GT>(la, Lh, ya, yb, act, wt, lc, pb);
      else sweep2<T, K, DYN, false, GT>(la, Lh, ya, yb, act, wt, lc, pb,
                                        use_bs ? &bsync : nullptr, warp);
      if (DTB_PUBREG >= 2 && pub && s + 2 == steps) {
        if (act && DTB_PUBREG != 4) pub->put_band(la, ya, yb);  // rows final: publish now
        if (DTB_PUBREG == 5) {
          // stores only; one CTA-level release after the closing barrier
        } else if (DTB_PUBREG == 2) {
          __threadfence();
        } else {
          // each warp releases its own stores and bumps the CTA's epoch flag;
          // neighbours wait for nwarps bumps per epoch (no CTA barrier first)
          __syncwarp();
          if (lc.lane == 0)
            asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(pub->flag) : "memory");
        }
      }
      if (!use_bs || s + 4 > steps) gt_sync<GT>();
    }
  }
  if (s < steps) {
    const int nb1 = max(1, min(nw, rows));
    int ya, yb;
    band_rows(Lh, nb1, min(warp, nb1 - 1), ya, yb);
    const bool band_pub = pub && ((DTB_PUBREG == 1 && pub->covers(ya, yb)) || DTB_PUBREG == 4);
    for (; s < steps; ++s) {
      if (band_pub && s + 1 == steps) sweep1<T, K, DYN, true, GT>(la, Lh, ya, yb, warp < nb1, wt, lc, pb);
      else sweep1<T, K, DYN, false, GT>(la, Lh, ya, yb, warp < nb1, wt, lc, pb);
      if (DTB_PUBREG >= 2 && pub && s + 1 == steps) {
        if (warp < nb1 && DTB_PUBREG != 4) pub->put_band(la, ya, yb);
        if (DTB_PUBREG == 5) {
        } else if (DTB_PUBREG == 2) {
          __threadfence();
        } else {
          __syncwarp();
          if (lc.lane == 0)
            asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(pub->flag) : "memory");
        }
      }
      gt_sync<GT>();
    }
  }
}

}  // namespace dtb
